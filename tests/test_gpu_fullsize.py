"""Size-independent properties at BASELINE.json's full sizes (configs 2
and 3: 512^3 / 512^2 and 2048^3 / 2048^2 geometry), on a few views of the
full scans so each case runs in seconds:

* adjoint identity <A x, y> = <x, A^T y> for the matched Atb;
* slab additivity of Ax and slab concatenation of Atb;
* angle-window invariance (windows are exact slices of the full scan);
* oracle parity on a thin window / slab of the full-size geometry (the
  oracle runs the same rays, so a 2-view x 8-plane case is cheap on CPU).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_l2, synth_geometry, to_oracle
from oracle import oracle as O
from paper_1905_03748_b200 import kernels as K

pytestmark = pytest.mark.gpu

CASES = [(512, 360, (0, 90, 181, 359)), (2048, 1024, (3, 517))]


def _dot(a, b):
    """<a, b> in fp64 without materialising fp64 copies (chunks of 64
    planes)."""
    t = 0.0
    for z in range(0, a.shape[0], 64):
        t += float((a[z:z + 64].double() * b[z:z + 64].double()).sum())
    return t


def _vol(n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.rand((n, n, n), device="cuda", generator=g)


@pytest.mark.parametrize("n,A,views", CASES)
def test_fullsize_adjoint(n, A, views):
    g = synth_geometry(n, A)
    x = _vol(n)
    gen = torch.Generator(device="cuda").manual_seed(1)
    for a in views:
        y = torch.randn((1, n, n), device="cuda", generator=gen)
        ax = torch.empty_like(y)
        K.fwd_interp(x, g, (a, a + 1), (0, n), ax)
        aty = torch.zeros_like(x)
        K.bwd_matched(y, g, (a, a + 1), (0, n), aty)
        lhs = _dot(ax, y)
        rhs = _dot(x, aty)
        scale = (_dot(ax, ax) * _dot(y, y)) ** 0.5
        assert abs(lhs - rhs) <= 1e-5 * scale, (a, lhs, rhs)
        del aty
    del x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,A,views", CASES)
def test_fullsize_slab_partition(n, A, views):
    g = synth_geometry(n, A)
    x = _vol(n)
    a0 = views[0]
    na = 2
    mono = torch.empty((na, n, n), device="cuda")
    K.fwd_interp(x, g, (a0, a0 + na), (0, n), mono)
    cuts = (0, n // 3, n // 2 + 7, n)
    acc = torch.empty_like(mono)
    for i, (z0, z1) in enumerate(zip(cuts[:-1], cuts[1:])):
        K.fwd_interp(x[z0:z1].contiguous(), g, (a0, a0 + na), (z0, z1), acc,
                     accumulate=i > 0)
    assert rel_l2(acc.cpu(), mono.cpu()) <= 1e-6
    # window invariance: the 2-view window is a slice of a 3-view window
    win = torch.empty((na + 1, n, n), device="cuda")
    K.fwd_interp(x, g, (a0 - 1 if a0 else a0, (a0 - 1 if a0 else a0) + na + 1),
                 (0, n), win)
    off = 1 if a0 else 0
    assert torch.equal(win[off:off + na], mono)
    del x
    torch.cuda.empty_cache()
    # Atb: slabs concatenate to the whole (central band of planes)
    y = torch.randn((na, n, n), device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(2))
    z0, z1 = n // 2 - 24, n // 2 + 24
    whole = torch.zeros((z1 - z0, n, n), device="cuda")
    K.bwd_matched(y, g, (a0, a0 + na), (z0, z1), whole)
    parts = torch.zeros_like(whole)
    for s0, s1 in ((z0, z0 + 5), (z0 + 5, z0 + 30), (z0 + 30, z1)):
        K.bwd_matched(y, g, (a0, a0 + na), (s0, s1), parts[s0 - z0:s1 - z0])
    assert rel_l2(parts.cpu(), whole.cpu()) <= 1e-6


def test_config2_window_vs_oracle():
    """Config 2 geometry: 2 views x full volume Ax and an 8-plane matched
    Atb slab, against the oracle (C restatement of _kernels.py)."""
    n, A = 512, 360
    g = synth_geometry(n, A)
    og = to_oracle(g)
    x = np.random.default_rng(0).random((n, n, n), dtype=np.float32)
    win = (45, 47)
    ax = torch.empty((2, n, n), device="cuda")
    K.fwd_interp(torch.from_numpy(x).cuda(), g, win, (0, n), ax)
    ref = O.fwd_interp(x, og, win)
    assert rel_l2(ax.cpu(), ref) <= 1e-5
    y = np.random.default_rng(1).standard_normal((2, n, n)).astype(np.float32)
    zr = (250, 258)
    acc = torch.zeros((8, n, n), device="cuda")
    K.bwd_matched(torch.from_numpy(y).cuda(), g, win, zr, acc)
    assert rel_l2(acc.cpu(), O.bwd_matched(y, og, win, zr)) <= 1e-5


def _crop_geometry(n, A, nu_full, crop, views):
    """A sub-rectangle (u0, v0, mu, mv) of the full n^3 / nu_full^2
    detector of synth_geometry(n, A), restricted to `views`: the same rays
    (up to rounding of the pixel centres) at a tracing cost the oracle can
    afford at full volume size."""
    import math
    import paper_1905_03748_b200 as cs
    full = synth_geometry(n, A)
    u0, v0, mu, mv = crop
    du, dv = full.detector.pixel_size
    off = ((u0 + 0.5 * (mu - 1) - 0.5 * (nu_full - 1)) * du,
           (v0 + 0.5 * (mv - 1) - 0.5 * (nu_full - 1)) * dv)
    det = cs.DetectorGrid(mu, mv, (du, dv), off)
    angles = tuple(full.angles[a] for a in views)
    return cs.ScanGeometry(full.dso, full.dsd, angles, full.voxel_grid, det)


@pytest.mark.parametrize("n,crop", [(512, (130, 200, 96, 64)),
                                    (2048, (700, 900, 64, 48))])
def test_fullsize_crop_vs_oracle(n, crop):
    """Config 2 / config 3 volumes: Ax over the full volume and matched Atb
    into a 16-plane slab, for a crop of the full detector in two views of
    the full scan, against the oracle (fp64 sample positions)."""
    import paper_1905_03748_b200 as cs
    A = 360 if n == 512 else 1024
    views = (17, A // 2 + 5)
    g = _crop_geometry(n, A, n, crop, views)
    og = to_oracle(g)
    vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                     device=torch.device("cuda", 0)).data
    x = vol.cpu().numpy()
    mu, mv = crop[2], crop[3]
    ax = torch.empty((2, mv, mu), device="cuda")
    K.fwd_interp(vol, g, (0, 2), (0, n), ax)
    del vol
    torch.cuda.empty_cache()
    ref = O.fwd_interp(x, og)
    e_ax = rel_l2(ax.cpu(), ref)
    del x
    y = np.random.default_rng(5).random((2, mv, mu)).astype(np.float32)
    v0 = crop[1]
    # the slab the crop's central rows cross near the rotation axis
    zc = int(n // 2 + (v0 + mv // 2 - n // 2) * 0.5 * 2.8284271247461903 * n / n)
    zr = (max(0, zc - 8), min(n, zc + 8))
    acc = torch.zeros((zr[1] - zr[0], n, n), device="cuda")
    K.bwd_matched(torch.from_numpy(y).cuda(), g, (0, 2), zr, acc)
    refb = O.bwd_matched(y, og, (0, 2), zr)
    assert float(np.abs(refb).sum()) > 0.0
    e_b = rel_l2(acc.cpu(), refb)
    # FDK-weighted Atb of the same crop into the same slab
    acc.zero_()
    K.bwd_fdk(torch.from_numpy(y).cuda(), g, (0, 2), zr, acc)
    reff = O.bwd_fdk(y, og, (0, 2), zr)
    e_f = rel_l2(acc.cpu(), reff)
    print(f"n={n}: Ax relL2 {e_ax:.3e}, matched relL2 {e_b:.3e}, "
          f"FDK relL2 {e_f:.3e}")
    assert e_ax <= 1e-5 and e_b <= 1e-5 and e_f <= 1e-5, (e_ax, e_b, e_f)


def test_config2_loops_properties():
    """The loops at config-2 size (60 of the 360-view scan for speed):
    CGLS residuals are monotone and drop; OS-SART and SART-TV
    reduce ||b - A x||; SART-TV lowers the TV norm of the OS-SART result."""
    import paper_1905_03748_b200 as cs
    n = 512
    full = synth_geometry(n, 360)
    g = full.with_angles(full.angles[::6])
    dev = torch.device("cuda", 0)
    x_true = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                        device=dev).data
    b = cs.forward_project_slab(cs.Volume(g.voxel_grid, x_true), g,
                                (0, g.n_angles),
                                cs.ProjectionMethod.INTERPOLATED)
    pool = cs.DevicePool.b200(1)
    r = cs.cgls(b, g, cs.ReconConfig(pool, cs.Algorithm.CGLS, 3))
    res = r.residuals
    assert all(b2 <= b1 * (1 + 1e-6) for b1, b2 in zip(res, res[1:])), res
    assert res[-1] < 0.5 * res[0]

    def resid(v):
        ax = cs.forward_project_slab(cs.Volume(g.voxel_grid, v), g,
                                     (0, g.n_angles),
                                     cs.ProjectionMethod.INTERPOLATED).data
        return float((ax - b.data).double().norm() / b.data.double().norm())

    xo = cs.os_sart(b, g, cs.ReconConfig(pool, cs.Algorithm.OSSART, 2, 12)).data
    assert resid(xo) < 0.5
    tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 10, 5e-2)
    xt = cs.os_sart(b, g, cs.ReconConfig(pool, cs.Algorithm.OSSART, 2, 12,
                                         tv=tv)).data
    assert resid(xt) < 0.6
    tvn = lambda v: cs.tv_norm(cs.Volume(g.voxel_grid, v))
    assert tvn(xt) < tvn(xo)
