"""CUDA path vs the oracle / reference goldens (the parity gate).

Tolerances (SURVEY 8(c), fp32 device accumulation vs fp64 reference):
  Ax interpolated  relL2 <= 1e-5, max-rel <= 1e-4
  Atb matched      relL2 <= 1e-5; adjoint identity <= 1e-5
  Atb FDK          relL2 <= 1e-5
  Siddon Ax        relL2 <= 1e-5
  TV step         relL2 <= 1e-5
  loops            relL2 <= 3e-5 (3x the operator tolerance)
  integer set-up   bit-exact (ray t0/step/n_steps, slab/angle ranges)
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K
from conftest import (max_rel, product_geometry, rel_l2, synth_geometry,
                      to_oracle)
from oracle import oracle as O

GEOS = ["g16", "ganiso", "g32"]
IP = cs.ProjectionMethod.INTERPOLATED
SD = cs.ProjectionMethod.SIDDON
TOL_OP = 1e-5
TOL_LOOP = 3e-5


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


@pytest.mark.parametrize("name", GEOS)
def test_ray_setup_bit_exact(golden, golden_meta, name):
    g = product_geometry(golden_meta["geometries"][name])
    t0, st, n = K.ray_table(g, (0, g.n_angles))
    np.testing.assert_array_equal(t0.cpu().numpy(), golden[f"{name}/ray_t0"])
    np.testing.assert_array_equal(st.cpu().numpy(), golden[f"{name}/ray_step"])
    np.testing.assert_array_equal(n.cpu().numpy(), golden[f"{name}/ray_n"])


@pytest.mark.parametrize("name", GEOS)
def test_forward_vs_reference(golden, golden_meta, name):
    d = golden_meta["geometries"][name]
    g = product_geometry(d)
    x = golden[f"{name}/x"]
    vol = cs.Volume(g.voxel_grid, x)
    A = g.n_angles
    got = cs.forward_project_slab(vol, g, (0, A), IP).data
    ref = golden[f"{name}/fwd_interp"]
    assert rel_l2(got, ref) <= TOL_OP and max_rel(got, ref) <= 1e-4
    got = cs.forward_project_slab(vol, g, (0, A), SD).data
    assert rel_l2(got, golden[f"{name}/fwd_siddon"]) <= TOL_OP
    z0, z1 = d["slab"]
    a0, a1 = d["window"]
    slab = cs.Volume(g.voxel_grid, x[z0:z1], (z0, z1))
    got = cs.forward_project_slab(slab, g, (a0, a1), IP).data
    assert rel_l2(got, golden[f"{name}/fwd_interp_slab"]) <= TOL_OP
    got = cs.forward_project_slab(slab, g, (a0, a1), SD).data
    assert rel_l2(got, golden[f"{name}/fwd_siddon_slab"]) <= TOL_OP


@pytest.mark.parametrize("name", GEOS)
def test_backward_vs_reference(golden, golden_meta, name):
    d = golden_meta["geometries"][name]
    g = product_geometry(d)
    x, y = golden[f"{name}/x"], golden[f"{name}/y"]
    A, nz = g.n_angles, g.voxel_grid.n_z
    stack = cs.ProjectionStack(g.detector, y, (0, A))
    for mode, key in ((cs.WeightMode.MATCHED, "bwd_matched"),
                      (cs.WeightMode.FDK, "bwd_fdk")):
        got = cs.backproject_slab(stack, g, (0, nz), mode).data
        assert rel_l2(got, golden[f"{name}/{key}"]) <= TOL_OP, key
        z0, z1 = d["slab"]
        a0, a1 = d["window"]
        sub = cs.ProjectionStack(g.detector, y[a0:a1], (a0, a1))
        acc = cs.Volume(g.voxel_grid, x[z0:z1] * 0.5, (z0, z1))
        got = cs.backproject_slab(sub, g, (z0, z1), mode,
                                  accumulate_into=acc).data
        assert rel_l2(got, golden[f"{name}/{key}_slab"]) <= TOL_OP, key


def test_kat_cube(golden, golden_meta):
    g = product_geometry(golden_meta["kat_cube"])
    vol = cs.Volume(g.voxel_grid, np.full((10, 10, 10), 0.02, np.float32))
    s = cs.forward_project_slab(vol, g, (0, 1), SD).data
    assert abs(s[0, 1, 1] - 0.2) < 1e-4
    i = cs.forward_project_slab(vol, g, (0, 1), IP).data
    np.testing.assert_allclose(i, golden["kat/cube_interp"], rtol=1e-5,
                               atol=1e-7)


@pytest.mark.parametrize("n,na", [(16, 8), (40, 13)])
def test_adjoint_identity(n, na):
    """<A x, y> == <x, A^T y>."""
    g = synth_geometry(n, na, nu=n + 8, nv=n + 4)
    rng = np.random.default_rng(3)
    for _ in range(5):
        x = dev(rng.random((n, n, n)))
        y = dev(rng.standard_normal((na, n + 4, n + 8)))
        ax = torch.empty_like(y)
        K.fwd_interp(x, g, (0, na), (0, n), ax)
        aty = torch.zeros_like(x)
        K.bwd_matched(y, g, (0, na), (0, n), aty)
        lhs = float((ax.double() * y.double()).sum())
        rhs = float((x.double() * aty.double()).sum())
        # random-sign y makes <.,.> cancel; scale by the Cauchy-Schwarz bound
        scale = float(ax.double().norm() * y.double().norm())
        assert abs(lhs - rhs) <= TOL_OP * scale


def test_dense_matrix_adjoint_8():
    """dense 8^3 matrix from unit basis vectors; A^T == A.T."""
    g = synth_geometry(8, 3, nu=10, nv=9)
    nvox = 8 ** 3
    cols = []
    basis = torch.zeros(nvox, device="cuda")
    out = torch.empty((3, 9, 10), device="cuda")
    for j in range(nvox):
        basis.zero_()
        basis[j] = 1.0
        K.fwd_interp(basis.view(8, 8, 8), g, (0, 3), (0, 8), out)
        cols.append(out.flatten().cpu().numpy().copy())
    Amat = np.stack(cols, 1).astype(np.float64)
    rows = []
    e = torch.zeros(3 * 9 * 10, device="cuda")
    acc = torch.zeros((8, 8, 8), device="cuda")
    for i in range(0, 3 * 9 * 10):
        e.zero_()
        e[i] = 1.0
        acc.zero_()
        K.bwd_matched(e.view(3, 9, 10), g, (0, 3), (0, 8), acc)
        rows.append(acc.flatten().cpu().numpy().copy())
    ATmat = np.stack(rows, 0).astype(np.float64)
    assert np.abs(Amat - ATmat).max() <= 1e-6 * np.abs(Amat).max()


def test_c1_operators_vs_oracle():
    """Config 1 (64^3, 64^2, 100 angles): full operators vs the oracle."""
    g = synth_geometry(64, 100)
    og = to_oracle(g)
    x = np.random.default_rng(0).random((64, 64, 64), dtype=np.float32)
    y = np.random.default_rng(1).standard_normal((100, 64, 64)).astype(
        np.float32)
    ax = torch.empty((100, 64, 64), device="cuda")
    K.fwd_interp(dev(x), g, (0, 100), (0, 64), ax)
    ref = O.fwd_interp(x, og)
    assert rel_l2(ax.cpu(), ref) <= TOL_OP
    assert max_rel(ax.cpu(), ref) <= 1e-4
    for fn, ofn in ((K.bwd_matched, O.bwd_matched), (K.bwd_fdk, O.bwd_fdk)):
        acc = torch.zeros((64, 64, 64), device="cuda")
        fn(dev(y), g, (0, 100), (0, 64), acc)
        assert rel_l2(acc.cpu(), ofn(y, og)) <= TOL_OP, fn.__name__


def test_slab_partition_transparency():
    """Forward slab partials sum to the monolithic projection; backward
    slabs concatenate to the monolithic volume."""
    n, na = 48, 36
    g = synth_geometry(n, na)
    x = dev(np.random.default_rng(0).random((n, n, n)))
    y = dev(np.random.default_rng(1).standard_normal((na, n, n)))
    mono = torch.empty((na, n, n), device="cuda")
    K.fwd_interp(x, g, (0, na), (0, n), mono)
    for cuts in [(0, 20, 41, 48), (0, 1, 2, 47, 48), (0, 16, 32, 48)]:
        acc = torch.empty_like(mono)
        for i, (z0, z1) in enumerate(zip(cuts[:-1], cuts[1:])):
            K.fwd_interp(x[z0:z1].contiguous(), g, (0, na), (z0, z1), acc,
                         accumulate=i > 0)
        assert rel_l2(acc.cpu(), mono.cpu()) <= 1e-6
    for fn in (K.bwd_matched, K.bwd_fdk):
        whole = torch.zeros((n, n, n), device="cuda")
        fn(y, g, (0, na), (0, n), whole)
        parts = torch.zeros_like(whole)
        for z0, z1 in [(0, 20), (20, 41), (41, 48)]:
            fn(y, g, (0, na), (z0, z1), parts[z0:z1])
        assert rel_l2(parts.cpu(), whole.cpu()) <= 1e-6


def test_angle_window_invariance():
    g = synth_geometry(32, 20)
    x = dev(np.random.default_rng(0).random((32, 32, 32)))
    full = torch.empty((20, 32, 32), device="cuda")
    K.fwd_interp(x, g, (0, 20), (0, 32), full)
    win = torch.empty((10, 32, 32), device="cuda")
    K.fwd_interp(x, g, (10, 20), (0, 32), win)
    assert torch.equal(win, full[10:20])


def test_edge_cases():
    """Rays missing the grid, single angle, zero projections."""
    grid = cs.VoxelGrid(8, 8, 8)
    det = cs.DetectorGrid(40, 30, (2.0, 2.0))  # panel much wider than shadow
    g = cs.ScanGeometry(40.0, 80.0, (0.3,), grid, det)
    og = to_oracle(g)
    x = np.random.default_rng(5).random((8, 8, 8), dtype=np.float32)
    got = cs.forward_project_slab(cs.Volume(grid, x), g, (0, 1), IP).data
    ref = O.fwd_interp(x, og)
    assert (ref == 0).sum() > 100  # many misses
    assert np.array_equal(got == 0, ref == 0)
    assert rel_l2(got, ref) <= TOL_OP
    zero = cs.ProjectionStack(det, np.zeros((1, 30, 40), np.float32))
    for mode in cs.WeightMode:
        out = cs.backproject_slab(zero, g, (0, 8), mode).data
        assert not out.any()


def test_tv_vs_reference(golden):
    f = golden["tv/f"]
    grid = cs.VoxelGrid(20, 18, 24)
    vol = cs.Volume(grid, f)
    assert abs(cs.tv_norm(vol) - float(golden["tv/norm"])) <= \
        1e-6 * float(golden["tv/norm"])
    single = np.zeros((3, 3, 3), np.float32)
    single[1, 1, 1] = 1.0
    assert abs(cs.tv_norm(cs.Volume(cs.VoxelGrid(3, 3, 3), single))
               - (math.sqrt(3) + 3)) < 1e-6
    GD, ROF = cs.TvMinimizer.GRADIENT_DESCENT, cs.TvMinimizer.ROF
    got = cs.minimize_tv_gradient(vol, cs.TvParams(GD, inner_iters=12,
                                                   step=0.05)).data
    assert rel_l2(got, golden["tv/gd"]) <= TOL_OP
    got = cs.minimize_rof(vol, cs.TvParams(ROF, inner_iters=12, lam=0.1)).data
    assert rel_l2(got, golden["tv/rof"]) <= TOL_OP
    for ndev in (1, 2, 3):
        pool = cs.DevicePool(tuple(cs.DeviceSpec(memory_budget=10 ** 9)
                                   for _ in range(ndev)))
        for minim, tag in ((GD, "gd"), (ROF, "rof")):
            for nm, ntag in ((cs.NormMode.EXACT_GLOBAL, "exact"),
                             (cs.NormMode.LOCAL_APPROX, "local")):
                if minim is ROF and ntag == "local":
                    continue
                p = cs.TvParams(minim, outer_syncs=2, inner_iters=4,
                                step=0.05, lam=0.1, norm_mode=nm,
                                halo_depth=5)
                got = cs.split_minimize(vol, pool, p).data
                key = f"tv/split_{tag}_{ntag}_d{ndev}"
                assert rel_l2(got, golden[key]) <= TOL_OP, key


def test_loops_vs_reference(golden, golden_meta):
    g = product_geometry(golden_meta["geometries"]["g16"])
    pool = cs.DevicePool((cs.DeviceSpec(memory_budget=2 ** 30),))
    b = cs.ProjectionStack(g.detector, golden["loops/b16"])
    res = cs.cgls(b, g, cs.ReconConfig(pool, iterations=4))
    assert rel_l2(res.volume.data, golden["loops/cgls_x"]) <= TOL_LOOP
    np.testing.assert_allclose(res.residuals, golden["loops/cgls_res"],
                               rtol=TOL_LOOP)
    got = cs.os_sart(b, g, cs.ReconConfig(pool, cs.Algorithm.OSSART, 3,
                                          g.n_angles)).data
    assert rel_l2(got, golden["loops/sirt_x"]) <= TOL_LOOP
    got = cs.os_sart(b, g, cs.ReconConfig(pool, cs.Algorithm.OSSART, 2, 3,
                                          0.8)).data
    assert rel_l2(got, golden["loops/ossart_x"]) <= TOL_LOOP
    tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, inner_iters=5,
                     step=0.01)
    got = cs.os_sart(b, g, cs.ReconConfig(pool, cs.Algorithm.OSSART, 2, 4,
                                          tv=tv)).data
    assert rel_l2(got, golden["loops/sarttv_x"]) <= TOL_LOOP
    got = cs.fdk(b, g, pool).data
    assert rel_l2(got, golden["loops/fdk_x"]) <= TOL_LOOP


def test_executor_split_transparency():
    """execute_forward / execute_backward == monolithic for {1,2,3}
    devices x forced splits, and traces respect budgets."""
    n, na = 24, 12
    g = synth_geometry(n, na)
    x = np.random.default_rng(0).random((n, n, n), dtype=np.float32)
    y = np.random.default_rng(1).standard_normal((na, n, n)).astype(
        np.float32)
    vol = cs.Volume(g.voxel_grid, x)
    stack = cs.ProjectionStack(g.detector, y)
    mono_f = cs.forward_project_slab(vol, g, (0, na), IP).data
    mono_b = cs.backproject_slab(stack, g, (0, n), cs.WeightMode.MATCHED).data
    plane = n * n * 4
    chunk = 9 * n * n * 4
    for ndev in (1, 2, 3):
        for budget in (10 ** 9, (n // 2) * plane + 4 * chunk,
                       (n // 3) * plane + 4 * chunk):
            pool = cs.DevicePool(tuple(cs.DeviceSpec(memory_budget=budget)
                                       for _ in range(ndev)))
            fplan = cs.plan_forward(g, pool)
            bplan = cs.plan_backward(g, pool)
            sink = []
            f = cs.execute_forward(vol, g, pool, fplan, IP, trace_sink=sink)
            assert rel_l2(f.data, mono_f) <= 1e-6
            b = cs.execute_backward(stack, g, pool, bplan,
                                    cs.WeightMode.MATCHED, trace_sink=sink)
            assert rel_l2(b.data, mono_b) <= 1e-6
            assert len(sink) == 2 and all(not t.simulated for t in sink)
            assert any(e.kind == "Kernel" for e in sink[0].events)


def test_host_backprojection_drains_in_pieces(monkeypatch):
    """backproject_slab on host projections into a fresh host volume: view
    chunks streamed up, the last chunk backprojected in z pieces that drain
    to the host while the next piece computes (projectors.py
    _backproject_to_host) -- forced here onto a small scan (3-view chunks,
    4 pieces), matched and FDK, against the oracle."""
    from paper_1905_03748_b200 import projectors as P
    monkeypatch.setattr(P, "_DRAIN_PIECE_MIN_BYTES", 0)
    monkeypatch.setattr(P, "_DRAIN_VIEWS", 3)
    g = synth_geometry(24, 10)
    y = np.random.default_rng(3).standard_normal(
        (10, g.detector.n_v, g.detector.n_u)).astype(np.float32)
    stack = cs.ProjectionStack(g.detector, y, (0, 10))
    for mode, ref_fn in ((cs.WeightMode.MATCHED, O.bwd_matched),
                         (cs.WeightMode.FDK, O.bwd_fdk)):
        got = cs.backproject_slab(stack, g, (0, 24), mode).data
        assert isinstance(got, np.ndarray)
        assert rel_l2(got, ref_fn(y, to_oracle(g))) <= TOL_OP, mode
        # a slab window of the grid: the same planes as the whole grid
        sl = cs.backproject_slab(stack, g, (5, 19), mode).data
        assert rel_l2(sl, got[5:19]) <= 1e-6, mode


def test_device_resident_roundtrip():
    """Device tensors in -> device tensors out, no host staging."""
    g = synth_geometry(32, 10)
    x = torch.rand((32, 32, 32), device="cuda")
    p = cs.forward_project_slab(cs.Volume(g.voxel_grid, x), g, (0, 10), IP)
    assert isinstance(p.data, torch.Tensor) and p.data.is_cuda
    v = cs.backproject_slab(p, g, (0, 32), cs.WeightMode.MATCHED)
    assert isinstance(v.data, torch.Tensor) and v.data.is_cuda
    ref = O.bwd_matched(p.data.cpu().numpy(), to_oracle(g))
    assert rel_l2(v.data.cpu(), ref) <= TOL_OP


def test_tigre_aliases():
    g = synth_geometry(16, 6)
    x = np.random.default_rng(0).random((16, 16, 16), dtype=np.float32)
    p = cs.Ax(x, g)
    assert rel_l2(p, O.fwd_interp(x, to_oracle(g))) <= TOL_OP
    v = cs.Atb(p, g, weight="fdk")
    assert rel_l2(v, O.bwd_fdk(p, to_oracle(g))) <= TOL_OP
    r = cs.sirt(p, g, niter=2)
    assert r.shape == (16, 16, 16)


def test_out_of_core_loops_match_in_core():
    """A device budget too small for the volume forces slab streaming
    (plan.n_splits > 1); CGLS / OS-SART through the out-of-core executor
    must match the in-core device loops."""
    n, na = 24, 12
    g = synth_geometry(n, na)
    x = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid).data
    b = cs.forward_project_slab(cs.Volume(g.voxel_grid, x), g, (0, na), IP)
    big = cs.DevicePool((cs.DeviceSpec(memory_budget=2 ** 30),))
    small = cs.DevicePool((cs.DeviceSpec(memory_budget=98000),))
    assert cs.plan_forward(g, small).n_splits > 1
    assert cs.plan_backward(g, small).n_splits > 1
    r_in = cs.cgls(b, g, cs.ReconConfig(big, iterations=3))
    sink = []
    r_out = cs.cgls(b, g, cs.ReconConfig(small, iterations=3), trace_sink=sink)
    assert rel_l2(r_out.volume.data, r_in.volume.data) <= TOL_LOOP
    np.testing.assert_allclose(r_out.residuals, r_in.residuals, rtol=TOL_LOOP)
    assert sink and all(max(t.high_water.values()) <= 98000 for t in sink)
    for t in sink:
        cs.check_trace(t, small)
    cfg_in = cs.ReconConfig(big, cs.Algorithm.OSSART, 2, 4)
    cfg_out = cs.ReconConfig(small, cs.Algorithm.OSSART, 2, 4)
    o_in = cs.os_sart(b, g, cfg_in).data
    o_out = cs.os_sart(b, g, cfg_out).data
    assert rel_l2(o_out, o_in) <= TOL_LOOP
    # the host loop's float32 vectors with V_S recomputed per block instead
    # of stored (HOST_WEIGHT_FRACTION = 0), and SART-TV out of core
    from paper_1905_03748_b200 import algorithms as ALG
    old = ALG.HOST_WEIGHT_FRACTION
    ALG.HOST_WEIGHT_FRACTION = 0.0
    try:
        o_re = cs.os_sart(b, g, cfg_out).data
    finally:
        ALG.HOST_WEIGHT_FRACTION = old
    assert rel_l2(o_re, o_in) <= TOL_LOOP
    tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 4, 1e-3)
    t_in = cs.os_sart(b, g, cs.ReconConfig(big, cs.Algorithm.OSSART, 2, 4,
                                           tv=tv)).data
    t_out = cs.os_sart(b, g, cs.ReconConfig(small, cs.Algorithm.OSSART, 2, 4,
                                            tv=tv)).data
    assert rel_l2(t_out, t_in) <= TOL_LOOP


def _odd_geometry(nx, ny, nz, nu, nv, na, voxel=(1.0, 0.9, 1.1),
                  offset=(0.3, -0.2, 0.1), pitch=None, det_off=(0.4, -0.3)):
    grid = cs.VoxelGrid(nx, ny, nz, voxel, offset)
    r = grid.bounding_radius()
    dso, dsd = 2.5 * r + 2.0, 5.0 * r + 4.0
    if pitch is None:
        ext = grid.extent
        mag = dsd / dso
        pitch = (1.3 * mag * max(ext[0], ext[1]) / nu,
                 1.3 * mag * ext[2] / nv)
    det = cs.DetectorGrid(nu, nv, pitch, det_off)
    angles = tuple(np.linspace(0.1, 0.1 + 2 * math.pi, na, endpoint=False))
    return cs.ScanGeometry(dso, dsd, angles, grid, det)


@pytest.mark.parametrize("shape", [(13, 11, 9, 17, 15, 7), (30, 26, 21, 33, 19, 11)])
def test_odd_sizes_vs_oracle(shape):
    """Sizes that are not multiples of 4 (scalar flush / load paths of the
    staged kernels), anisotropic voxels, offsets, slabs and windows."""
    nx, ny, nz, nu, nv, na = shape
    g = _odd_geometry(nx, ny, nz, nu, nv, na)
    og = to_oracle(g)
    rng = np.random.default_rng(11)
    x = rng.random((nz, ny, nx), dtype=np.float32)
    y = rng.standard_normal((na, nv, nu)).astype(np.float32)
    z0, z1 = nz // 3, nz - 2
    a0, a1 = 1, na - 1
    for (zr, ar) in (((0, nz), (0, na)), ((z0, z1), (a0, a1))):
        xs = x[zr[0]:zr[1]]
        got = cs.forward_project_slab(cs.Volume(g.voxel_grid, xs, zr), g, ar,
                                      IP).data
        assert rel_l2(got, O.fwd_interp(xs, og, ar, zr)) <= TOL_OP
        ys = y[ar[0]:ar[1]]
        st = cs.ProjectionStack(g.detector, ys, ar)
        for mode, ofn in ((cs.WeightMode.MATCHED, O.bwd_matched),
                          (cs.WeightMode.FDK, O.bwd_fdk)):
            got = cs.backproject_slab(st, g, zr, mode).data
            assert rel_l2(got, ofn(ys, og, ar, zr)) <= TOL_OP, mode


def test_fdk_oversized_footprint_direct_path():
    """Detector pixels much finer than voxels: a CTA's per-view footprint
    exceeds the shared staging buffer and the view is gathered directly."""
    g = _odd_geometry(16, 16, 16, 420, 400, 2, voxel=(1.0, 1.0, 1.0),
                      offset=(0.0, 0.0, 0.0), pitch=(0.1, 0.1),
                      det_off=(0.0, 0.0))
    og = to_oracle(g)
    y = np.random.default_rng(2).standard_normal((2, 400, 420)).astype(
        np.float32)
    got = cs.backproject_slab(cs.ProjectionStack(g.detector, y), g, (0, 16),
                              cs.WeightMode.FDK).data
    assert rel_l2(got, O.bwd_fdk(y, og)) <= TOL_OP


def test_staged_small_box_budget_subprocess():
    """With a tiny shared-memory box budget the staged matched kernel halves
    its chunk depth and then falls back to global reductions; results must
    not change (runs in a subprocess: the budget knob is read once)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path[:0] = [%r, %r]\n"
        "import numpy as np, paper_1905_03748_b200 as cs\n"
        "from conftest import synth_geometry, to_oracle, rel_l2\n"
        "from oracle import oracle as O\n"
        "g = synth_geometry(40, 12)\n"
        "y = np.random.default_rng(4).standard_normal((12, 40, 40)).astype(np.float32)\n"
        "got = cs.backproject_slab(cs.ProjectionStack(g.detector, y), g, (0, 40), cs.WeightMode.MATCHED).data\n"
        "e = rel_l2(got, O.bwd_matched(y, to_oracle(g)))\n"
        "print(e); assert e <= 1e-5\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
         os.path.dirname(os.path.abspath(__file__)))
    for kb in ("2", "6"):
        env = dict(os.environ, CS_STAGED_SMEM_KB=kb)
        r = subprocess.run([sys.executable, "-c", code], env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.parametrize("dims", [(1, 1, 1), (1, 3, 2), (3, 1, 5), (2, 2, 1)])
def test_tiny_grids_vs_oracle(dims):
    """Degenerate grids (single voxels / planes / rows): Ax, matched and FDK
    against the oracle, including slab launches of one plane."""
    nx, ny, nz = dims
    grid = cs.VoxelGrid(nx, ny, nz, (1.0, 1.2, 0.8))
    det = cs.DetectorGrid(9, 7, (0.7, 0.6))
    angles = tuple(np.linspace(0.05, 2 * math.pi, 6, endpoint=False))
    g = cs.ScanGeometry(12.0, 24.0, angles, grid, det)
    og = to_oracle(g)
    rng = np.random.default_rng(9)
    x = rng.random((nz, ny, nx), dtype=np.float32)
    y = rng.standard_normal((6, 7, 9)).astype(np.float32)
    got = cs.forward_project_slab(cs.Volume(grid, x), g, (0, 6), IP).data
    assert rel_l2(got, O.fwd_interp(x, og)) <= TOL_OP
    st = cs.ProjectionStack(det, y)
    for mode, ofn in ((cs.WeightMode.MATCHED, O.bwd_matched),
                      (cs.WeightMode.FDK, O.bwd_fdk)):
        got = cs.backproject_slab(st, g, (0, nz), mode).data
        assert rel_l2(got, ofn(y, og)) <= TOL_OP, mode
        got = cs.backproject_slab(st, g, (nz - 1, nz), mode).data
        assert rel_l2(got, ofn(y, og, (0, 6), (nz - 1, nz))) <= TOL_OP, mode


def test_unordered_angles_vs_oracle():
    """Views in arbitrary order, negative and beyond 2 pi, repeated: every
    view is independent (the per-view main axis, culling bands and view-id
    tables of the staged kernels must follow the given order)."""
    rng = np.random.default_rng(13)
    angles = tuple(float(a) for a in
                   np.concatenate([rng.uniform(-7.0, 13.0, 10), [0.0, 0.0,
                                   math.pi / 4, 3 * math.pi / 4]]))
    grid = cs.VoxelGrid(20, 18, 16)
    r = grid.bounding_radius()
    det = cs.DetectorGrid(26, 22, (2.0, 2.0))
    g = cs.ScanGeometry(2.5 * r, 5.0 * r, angles, grid, det)
    og = to_oracle(g)
    na = len(angles)
    x = rng.random((16, 18, 20), dtype=np.float32)
    y = rng.standard_normal((na, 22, 26)).astype(np.float32)
    got = cs.forward_project_slab(cs.Volume(grid, x), g, (0, na), IP).data
    assert rel_l2(got, O.fwd_interp(x, og)) <= TOL_OP
    st = cs.ProjectionStack(det, y)
    for mode, ofn in ((cs.WeightMode.MATCHED, O.bwd_matched),
                      (cs.WeightMode.FDK, O.bwd_fdk)):
        assert rel_l2(cs.backproject_slab(st, g, (0, 16), mode).data,
                      ofn(y, og)) <= TOL_OP, mode
        assert rel_l2(cs.backproject_slab(st, g, (5, 11), mode).data,
                      ofn(y, og, (0, na), (5, 11))) <= TOL_OP, mode


def test_wide_fan_and_cone_vs_oracle():
    """Source close to the grid with a panel spanning a +-60 degree fan and
    cone: edge rays travel mostly across the view's main axis (huge boxes,
    the staged kernels' half-depth / global fallbacks and mixed-direction
    tiles) -- Ax, matched and FDK against the oracle."""
    grid = cs.VoxelGrid(18, 16, 14, (1.0, 1.0, 1.0))
    r = grid.bounding_radius()
    dso, dsd = 1.15 * r, 2.3 * r
    width = 2.0 * dsd * math.tan(math.radians(60.0))
    det = cs.DetectorGrid(40, 36, (width / 40, width / 36))
    angles = tuple(np.linspace(0.3, 0.3 + 2 * math.pi, 8, endpoint=False))
    g = cs.ScanGeometry(dso, dsd, angles, grid, det)
    og = to_oracle(g)
    rng = np.random.default_rng(21)
    x = rng.random((14, 16, 18), dtype=np.float32)
    y = rng.standard_normal((8, 36, 40)).astype(np.float32)
    got = cs.forward_project_slab(cs.Volume(grid, x), g, (0, 8), IP).data
    assert rel_l2(got, O.fwd_interp(x, og)) <= TOL_OP
    st = cs.ProjectionStack(det, y)
    for mode, ofn in ((cs.WeightMode.MATCHED, O.bwd_matched),
                      (cs.WeightMode.FDK, O.bwd_fdk)):
        assert rel_l2(cs.backproject_slab(st, g, (0, 14), mode).data,
                      ofn(y, og)) <= TOL_OP, mode
        assert rel_l2(cs.backproject_slab(st, g, (3, 9), mode).data,
                      ofn(y, og, (0, 8), (3, 9))) <= TOL_OP, mode


def test_fine_detector_lane_strides_subprocess():
    """Pixels much finer than voxels: the staged matched kernel spreads a
    warp's lanes s pixels apart (s = 1, 2, 4, 8; forced with the
    CS_ST_LANE_STRIDE knob, read once, hence subprocesses) on a detector
    whose width / height are not multiples of 32 s / 8 / s; full volume and
    a slab / view window against the oracle."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path[:0] = [%r, %r]\n"
        "import numpy as np, paper_1905_03748_b200 as cs\n"
        "from conftest import to_oracle, rel_l2\n"
        "from oracle import oracle as O\n"
        "from test_gpu_parity import _odd_geometry\n"
        "g = _odd_geometry(12, 10, 9, 151, 133, 4, pitch=(0.09, 0.11))\n"
        "og = to_oracle(g)\n"
        "y = np.random.default_rng(6).standard_normal((4, 133, 151)).astype(np.float32)\n"
        "st = cs.ProjectionStack(g.detector, y)\n"
        "got = cs.backproject_slab(st, g, (0, 9), cs.WeightMode.MATCHED).data\n"
        "e1 = rel_l2(got, O.bwd_matched(y, og))\n"
        "st2 = cs.ProjectionStack(g.detector, y[1:3], (1, 3))\n"
        "got = cs.backproject_slab(st2, g, (2, 7), cs.WeightMode.MATCHED).data\n"
        "e2 = rel_l2(got, O.bwd_matched(y[1:3], og, (1, 3), (2, 7)))\n"
        "print(e1, e2); assert e1 <= 1e-5 and e2 <= 1e-5\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
         os.path.dirname(os.path.abspath(__file__)))
    for s in ("1", "2", "4", "8", ""):
        env = dict(os.environ, CS_ST_LANE_STRIDE=s)
        r = subprocess.run([sys.executable, "-c", code], env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, (s, r.stderr[-2000:])


def test_ax_texture_reuse_across_slab_heights():
    """The main-axis-layered Ax reuses a taller texture array for shorter
    slabs (rows past the slab are zeroed guard rows): a tall launch followed
    by short slab launches near the top / bottom / middle, each against
    the oracle; views of both main axes and a non-cubic grid (x- and
    y-layered arrays differ)."""
    for dims in ((20, 20, 24), (22, 18, 24)):
        nx, ny, nz = dims
        g = _odd_geometry(nx, ny, nz, 30, 28, 8)
        og = to_oracle(g)
        x = np.random.default_rng(17).random((nz, ny, nx), dtype=np.float32) + 0.5
        full = cs.forward_project_slab(cs.Volume(g.voxel_grid, x), g, (0, 8),
                                       IP).data
        assert rel_l2(full, O.fwd_interp(x, og)) <= TOL_OP
        for zr in ((nz - 3, nz), (0, 2), (9, 14), (5, 21)):
            xs = x[zr[0]:zr[1]]
            got = cs.forward_project_slab(cs.Volume(g.voxel_grid, xs, zr), g,
                                          (0, 8), IP).data
            assert rel_l2(got, O.fwd_interp(xs, og, (0, 8), zr)) <= TOL_OP, zr


def test_ax_z_layered_fallback_subprocess():
    """The z-layered Ax (used when nx or ny exceeds the layered-texture
    limit; forced here with CS_FWD_MLAYER=0, read once, hence a
    subprocess): full volume, slabs and the residual epilogue against the
    oracle."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path[:0] = [%r, %r]\n"
        "import numpy as np, torch, paper_1905_03748_b200 as cs\n"
        "from paper_1905_03748_b200 import kernels as K\n"
        "from conftest import to_oracle, rel_l2\n"
        "from oracle import oracle as O\n"
        "from test_gpu_parity import _odd_geometry\n"
        "g = _odd_geometry(30, 26, 21, 33, 19, 11)\n"
        "og = to_oracle(g)\n"
        "x = np.random.default_rng(3).random((21, 26, 30), dtype=np.float32)\n"
        "IP = cs.ProjectionMethod.INTERPOLATED\n"
        "got = cs.forward_project_slab(cs.Volume(g.voxel_grid, x), g, (0, 11), IP).data\n"
        "e1 = rel_l2(got, O.fwd_interp(x, og))\n"
        "xs = x[4:15]\n"
        "got = cs.forward_project_slab(cs.Volume(g.voxel_grid, xs, (4, 15)), g, (2, 9), IP).data\n"
        "e2 = rel_l2(got, O.fwd_interp(xs, og, (2, 9), (4, 15)))\n"
        "print(e1, e2); assert e1 <= 1e-5 and e2 <= 1e-5\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
         os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CS_FWD_MLAYER="0")
    r = subprocess.run([sys.executable, "-c", code], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


def test_release_cache_then_reuse():
    """cs_release_cache frees the cached texture arrays; the next calls
    re-create them and give identical results."""
    from paper_1905_03748_b200 import kernels as K
    import torch
    g = _odd_geometry(16, 14, 12, 20, 18, 6)
    x = torch.rand((12, 14, 16), device="cuda")
    p1 = torch.empty((6, 18, 20), device="cuda")
    K.fwd_interp(x, g, (0, 6), (0, 12), p1)
    K.release_cache()
    p2 = torch.empty_like(p1)
    K.fwd_interp(x, g, (0, 6), (0, 12), p2)
    assert torch.equal(p1, p2)
    K.release_cache()


def test_ax_subslabs_when_texture_does_not_fit_subprocess():
    """When the texture copy of a slab does not fit in device memory the Ax
    halves its sub-slab height and accumulates (simulated with the
    CS_TEX_MAX_MB knob, read once: subprocess); overwrite / accumulate Ax
    on both texture layouts against the oracle."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path[:0] = [%r, %r]\n"
        "import numpy as np, torch, paper_1905_03748_b200 as cs\n"
        "from paper_1905_03748_b200 import kernels as K\n"
        "from conftest import to_oracle, rel_l2\n"
        "from oracle import oracle as O\n"
        "from test_gpu_parity import _odd_geometry\n"
        "g = _odd_geometry(40, 36, 48, 44, 40, 5)\n"
        "og = to_oracle(g)\n"
        "x = np.random.default_rng(8).random((48, 36, 40), dtype=np.float32)\n"
        "xd = torch.from_numpy(x).cuda()\n"
        "p = torch.full((5, 40, 44), 7.0, device='cuda')\n"
        "n0 = K.launch_count()\n"
        "K.fwd_interp(xd, g, (0, 5), (0, 48), p)\n"
        "n1 = K.launch_count() - n0\n"
        "import os; assert n1 >= (16 if os.environ['CS_FWD_MLAYER'] == '1' else 4), n1\n"
        "ref = O.fwd_interp(x, og)\n"
        "e1 = rel_l2(p.cpu(), ref)\n"
        "K.fwd_interp(xd[10:40].contiguous(), g, (0, 5), (10, 40), p, accumulate=True)\n"
        "e2 = rel_l2(p.cpu(), ref + O.fwd_interp(x[10:40], og, (0, 5), (10, 40)))\n"
        "print(e1, e2, K.launch_count()); assert e1 <= 1e-5 and e2 <= 1e-5\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
         os.path.dirname(os.path.abspath(__file__)))
    for ml in ("1", "0"):
        # 48 planes x 40 x 36 floats = 270 KiB; cap 0.08 MiB -> 12-plane pieces
        env = dict(os.environ, CS_TEX_MAX_MB="0.08", CS_FWD_MLAYER=ml)
        r = subprocess.run([sys.executable, "-c", code], env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, (ml, r.stderr[-2000:])


def test_ax_layer_pieces_subprocess():
    """x / y extents over the layered-texture limit (forced low with the
    CS_MAX_LAYERS knob, read once: subprocess): the main-axis Ax goes through
    in layer pieces (k ranges clipped per piece, first piece overwrites,
    the rest accumulate), the z-layered Ax in sub-slabs; both against the
    oracle, full volume, a slab and an accumulate launch."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path[:0] = [%r, %r]\n"
        "import numpy as np, torch, paper_1905_03748_b200 as cs\n"
        "from paper_1905_03748_b200 import kernels as K\n"
        "from conftest import to_oracle, rel_l2\n"
        "from oracle import oracle as O\n"
        "from test_gpu_parity import _odd_geometry\n"
        "g = _odd_geometry(40, 36, 30, 44, 40, 7)\n"
        "og = to_oracle(g)\n"
        "x = np.random.default_rng(12).random((30, 36, 40), dtype=np.float32)\n"
        "xd = torch.from_numpy(x).cuda()\n"
        "p = torch.full((7, 40, 44), 3.0, device='cuda')\n"
        "n0 = K.launch_count()\n"
        "K.fwd_interp(xd, g, (0, 7), (0, 30), p)\n"
        "n1 = K.launch_count() - n0\n"
        "ref = O.fwd_interp(x, og)\n"
        "e1 = rel_l2(p.cpu(), ref)\n"
        "K.fwd_interp(xd[5:22].contiguous(), g, (0, 7), (5, 22), p, accumulate=True)\n"
        "e2 = rel_l2(p.cpu(), ref + O.fwd_interp(x[5:22], og, (0, 7), (5, 22)))\n"
        "print(e1, e2, n1); assert e1 <= 1e-5 and e2 <= 1e-5\n"
        "import os; assert n1 >= (12 if os.environ['CS_FWD_MLAYER'] == '1' else 2), n1\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
         os.path.dirname(os.path.abspath(__file__)))
    for ml in ("1", "0"):
        env = dict(os.environ, CS_MAX_LAYERS="16", CS_FWD_MLAYER=ml)
        r = subprocess.run([sys.executable, "-c", code], env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, (ml, r.stderr[-2000:])


@pytest.mark.parametrize("dims", [(22, 18, 15), (17, 26, 12)])
def test_ax_residual_epilogue_vs_oracle(dims):
    """Fused residual epilogue out = w * (b - A x) (the loops' Ax) on
    non-cubic grids (separate x- and y-layer arrays), with and without
    weights, against the oracle."""
    import torch
    from paper_1905_03748_b200 import kernels as K
    nx, ny, nz = dims
    g = _odd_geometry(nx, ny, nz, 25, 21, 9)
    og = to_oracle(g)
    rng = np.random.default_rng(31)
    x = rng.random((nz, ny, nx), dtype=np.float32)
    b = rng.standard_normal((9, 21, 25)).astype(np.float32)
    w = rng.random((9, 21, 25), dtype=np.float32) + 0.5
    ax = O.fwd_interp(x, og)
    xd, bd, wd = (torch.from_numpy(a).cuda() for a in (x, b, w))
    out = torch.empty_like(bd)
    K.fwd_interp_residual(xd, g, (0, 9), bd, None, out)
    assert rel_l2(out.cpu(), b - ax) <= TOL_OP
    K.fwd_interp_residual(xd, g, (0, 9), bd, wd, out)
    assert rel_l2(out.cpu(), w * (b - ax)) <= TOL_OP


def test_tv_grad_norm_and_sumsq_vs_oracle(golden):
    """cs_tv_grad_norm / cs_tv_grad_sumsq: ||g||_2 and its square for the
    TV subgradient g (regularization.py:127-130, :147), over the whole
    window and over a core band, against the oracle (fp64 numpy)."""
    import torch
    from paper_1905_03748_b200 import kernels as K
    f = np.asarray(golden["tv/f"], np.float32)
    g = O.tv_subgradient(f.astype(np.float64))
    ud = torch.from_numpy(f).cuda()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    K.tv_grad_norm(ud, (0, f.shape[0]), out)
    ref = float(np.linalg.norm(g))
    assert abs(float(out) - ref) <= 1e-5 * ref
    K.tv_grad_sumsq(ud, (5, 17), out)
    ref2 = float((g[5:17] ** 2).sum())
    assert abs(float(out) - ref2) <= 2e-5 * ref2


def test_tv_stored_g_pair_bit_identical():
    """cs_tv_grad_store + cs_tv_step_g (the production GD pieces) agree with
    cs_tv_grad_sumsq + cs_tv_step up to the grouping of the fp64 partial
    sums (different kernels); odd sizes exercise the scalar tail of the
    streaming step."""
    import torch
    from paper_1905_03748_b200 import kernels as K
    u = torch.rand((13, 11, 9), device="cuda")
    for core in ((0, 13), (3, 10)):
        s1 = torch.zeros(1, dtype=torch.float64, device="cuda")
        s2 = torch.zeros_like(s1)
        K.tv_grad_sumsq(u, core, s1)
        o1 = torch.empty_like(u)
        K.tv_step(u, o1, 0.05, s1, 1.3)
        g = torch.empty_like(u)
        K.tv_grad_store(u, g, core, s2)
        o2 = torch.empty_like(u)
        K.tv_step_g(u, g, o2, 0.05, s2, 1.3)
        # the two kernels group the (fp32 per-thread) partial sums
        # differently; the per-voxel g terms are the same bits
        assert abs(float(s1) - float(s2)) <= 1e-6 * float(s1)
        assert torch.allclose(o1, o2, rtol=1e-6, atol=1e-7)


def test_tv_gd_fused_bit_identical():
    """cs_tv_gd_fused (step i + gradient i+1 in one pass) gives exactly the
    bits of cs_tv_step_g followed by cs_tv_grad_store, on windows that are
    not multiples of the 31 x 15 x 32 tile (halo lanes / rows, partial z
    chunks) and with a core band; the zero-norm case leaves u unchanged."""
    import torch
    from paper_1905_03748_b200 import kernels as K
    gen = torch.Generator(device="cuda").manual_seed(7)
    # odd nx: single-voxel kernel; even nx: paired kernel (60 x 14 tiles)
    for shape, core in (((13, 11, 9), (0, 13)), ((70, 47, 65), (9, 61)),
                        ((33, 16, 32), (0, 33)), ((2, 2, 2), (0, 2)),
                        ((70, 47, 126), (9, 61)), ((35, 29, 62), (0, 35)),
                        ((37, 29, 132), (3, 30)), ((41, 19, 64), (0, 41))):
        u = torch.rand(shape, device="cuda", generator=gen)
        g = torch.empty_like(u)
        s0 = torch.zeros(1, dtype=torch.float64, device="cuda")
        K.tv_grad_store(u, g, core, s0)
        # two-pass reference: step, then gradient of the stepped volume
        u1 = torch.empty_like(u)
        K.tv_step_g(u, g, u1, 0.05, s0, 1.3)
        g1 = torch.empty_like(u)
        s1 = torch.zeros_like(s0)
        K.tv_grad_store(u1, g1, core, s1)
        # fused
        u2 = torch.empty_like(u)
        g2 = torch.empty_like(u)
        s2 = torch.zeros_like(s0)
        K.tv_gd_fused(u, g, u2, g2, core, 0.05, s0, 1.3, s2)
        assert torch.equal(u1, u2), shape
        assert torch.equal(g1, g2), shape
        assert torch.equal(s1, s2), shape
    # flat volume: ||g|| = 0 -> the step is skipped (regularization.py:148)
    u = torch.full((9, 10, 11), 0.25, device="cuda")
    g = torch.empty_like(u)
    s0 = torch.zeros(1, dtype=torch.float64, device="cuda")
    K.tv_grad_store(u, g, (0, 9), s0)
    assert float(s0) == 0.0
    u2, g2 = torch.empty_like(u), torch.empty_like(u)
    s2 = torch.ones_like(s0)
    K.tv_gd_fused(u, g, u2, g2, (0, 9), 0.05, s0, 1.0, s2)
    assert torch.equal(u2, u) and float(s2) == 0.0


def test_tv_gd_vs_oracle_tiles():
    """minimize_tv_gradient (grad pass, fused passes, final step) against the
    oracle on a volume spanning several 31 x 15 x 32 tiles with remainders,
    plus a 1-iteration and a 2-iteration run (no / one fused pass)."""
    rng = np.random.default_rng(11)
    for nx, iters in ((65, 1), (65, 2), (65, 9), (126, 9)):
        f = rng.random((70, 47, nx), dtype=np.float32)
        vol = cs.Volume(cs.VoxelGrid(nx, 47, 70), f)
        got = cs.minimize_tv_gradient(
            vol, cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT,
                             inner_iters=iters, step=0.5)).data
        want = O.minimize_tv_gradient(f, iters, 0.5)
        assert rel_l2(got, want) <= TOL_OP, (nx, iters)
        assert rel_l2(got, f) > 1e-4  # the step moved u


def test_tv_gd_fused_matches_tiled_kernel_subprocess():
    """The marching kernels' g equals the r01 tiled kernel's (CS_TV_TILED=1)
    bit for bit, paired (even nx) and single-voxel (CS_TV_PAIRS=0), on a
    window with tile remainders; the sums agree to partial-sum grouping and
    the fused pass between the paired and single-voxel kernels to that."""
    import os
    import subprocess
    import sys
    import tempfile
    code = (
        "import torch,sys;sys.path.insert(0,'.');"
        "from paper_1905_03748_b200 import kernels as K;"
        "gen=torch.Generator(device='cuda').manual_seed(3);"
        "u=torch.rand((45,38,int(sys.argv[2])),device='cuda',generator=gen);"
        "g=torch.empty_like(u);s=torch.zeros(1,dtype=torch.float64,"
        "device='cuda');K.tv_grad_store(u,g,(4,40),s);"
        "u2=torch.empty_like(u);g2=torch.empty_like(u);s2=torch.zeros_like(s);"
        "K.tv_gd_fused(u,g,u2,g2,(4,40),0.05,s,1.0,s2);"
        "torch.save((g.cpu(),s.cpu(),u2.cpu(),g2.cpu()),sys.argv[1])")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # nx = 70: paired kernel fed by cp.async; nx = 132: paired kernel fed by
    # TMA (nx % 4 == 0), against the cp.async feed (CS_TV_TMA=0)
    for nx, variants in ((70, (("pairs", {}), ("single", {"CS_TV_PAIRS": "0"}),
                               ("tiled", {"CS_TV_TILED": "1"}))),
                         (132, (("tma", {}), ("cpasync", {"CS_TV_TMA": "0"}),
                                ("tiled", {"CS_TV_TILED": "1"})))):
        with tempfile.TemporaryDirectory() as td:
            outs = []
            for tag, env_add in variants:
                f = os.path.join(td, f"{tag}.pt")
                env = dict(os.environ, **env_add)
                subprocess.run([sys.executable, "-c", code, f, str(nx)],
                               cwd=root, env=env, check=True)
                outs.append(torch_load(f))
        (gp, sp, up, g2p), (gs, ss, us, g2s), (gt, st, _, _) = outs
        assert (gp == gs).all() and (gp == gt).all(), nx
        # the fused step reads each kernel's own sum (fp32 partials grouped
        # per kernel): equal to fp32 rounding of the step coefficient
        assert torch.allclose(up, us, rtol=1e-6, atol=1e-7), nx
        assert torch.allclose(g2p, g2s, rtol=1e-5, atol=1e-6), nx
        for s_ in (ss, st):
            assert abs(float(sp) - float(s_)) <= 1e-6 * float(sp), nx


def test_rof_vs_oracle_tiles():
    """minimize_rof against the oracle on volumes spanning several 60 x 14 x
    32 tiles (marching kernel, even nx) and with odd nx (r01 kernel)."""
    rng = np.random.default_rng(12)
    for nx in (126, 65, 132):  # cp.async feed, r01 kernel, TMA feed
        f = rng.random((70, 47, nx), dtype=np.float32)
        vol = cs.Volume(cs.VoxelGrid(nx, 47, 70), f)
        got = cs.minimize_rof(vol, cs.TvParams(cs.TvMinimizer.ROF,
                                               inner_iters=7, lam=0.3)).data
        want = O.minimize_rof(f, 7, 0.3)
        assert rel_l2(got, want) <= TOL_OP, nx
        assert rel_l2(got, f) > 1e-3


def test_rof_march_bit_identical_subprocess():
    """The marching ROF kernel gives the r01 kernel's bits (CS_ROF_MARCH=0)
    for a dual field that is nonzero everywhere, faces included (halo
    windows carry interior p onto their faces), on a window with tile
    remainders."""
    import os
    import subprocess
    import sys
    import tempfile
    code = (
        "import torch,sys;sys.path.insert(0,'.');"
        "from paper_1905_03748_b200 import kernels as K;"
        "gen=torch.Generator(device='cuda').manual_seed(5);"
        "nx=int(sys.argv[2]);"
        "f=torch.rand((45,38,nx),device='cuda',generator=gen);"
        "p=torch.rand((3,45,38,nx),device='cuda',generator=gen)-0.5;"
        "q=torch.empty_like(p);K.rof_iter(f,p,q,0.2);"
        "q2=torch.empty_like(p);K.rof_iter(f,q,q2,0.2);"
        "torch.save((q.cpu(),q2.cpu()),sys.argv[1])")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    # nx = 70: cp.async feed; nx = 132: TMA feed (and its cp.async twin)
    for nx in (70, 132):
        with tempfile.TemporaryDirectory() as td:
            outs = []
            for tag, env_add in (("march", {}), ("cpasync", {"CS_TV_TMA": "0"}),
                                 ("r01", {"CS_ROF_MARCH": "0"})):
                fn = os.path.join(td, f"{tag}.pt")
                subprocess.run([sys.executable, "-c", code, fn, str(nx)],
                               cwd=root, env=dict(os.environ, **env_add),
                               check=True)
                outs.append(torch_load(fn))
        (a1, a2), (b1, b2), (c1, c2) = outs
        assert (a1 == c1).all() and (a2 == c2).all(), nx
        assert (b1 == c1).all() and (b2 == c2).all(), nx


def test_matched_transposed_frame_subprocess():
    """Matched Atb's x-major views run as y-major views of the transposed
    frame (staged.cu); the direct x-major launch (CS_ST_TRANSPOSE=0) gives
    the same box sums, so the two agree to fp32 summation order -- on odd,
    non-multiple-of-4 sizes with anisotropic voxels, offsets and a slab;
    likewise the transposed frame in z pieces (CS_ST_TPIECE)."""
    import os
    import subprocess
    import sys
    import tempfile
    code = (
        "import torch,sys,math,numpy as np;sys.path.insert(0,'.');"
        "sys.path.insert(0,'tests');"
        "import paper_1905_03748_b200 as cs;"
        "from paper_1905_03748_b200 import kernels as K;"
        "grid=cs.VoxelGrid(37,29,23,(1.0,0.9,1.1),(0.3,-0.2,0.1));"
        "det=cs.DetectorGrid(41,27,(2.1,2.3),(0.4,-0.3));"
        "ang=tuple(np.linspace(0.1,0.1+2*math.pi,19,endpoint=False));"
        "g=cs.ScanGeometry(90.0,180.0,ang,grid,det);"
        "y=torch.randn((19,27,41),device='cuda',"
        "generator=torch.Generator(device='cuda').manual_seed(2));"
        "acc=torch.zeros((23,29,37),device='cuda');"
        "K.bwd_matched(y,g,(0,19),(0,23),acc);"
        "sl=torch.zeros((9,29,37),device='cuda');"
        "K.bwd_matched(y,g,(0,19),(7,16),sl);"
        "torch.save((acc.cpu(),sl.cpu()),sys.argv[1])")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as td:
        outs = []
        for tag, env_add in (("t", {}), ("direct", {"CS_ST_TRANSPOSE": "0"}),
                             ("pieces", {"CS_ST_TPIECE": "4"})):
            fn = os.path.join(td, f"{tag}.pt")
            subprocess.run([sys.executable, "-c", code, fn], cwd=root,
                           env=dict(os.environ, **env_add), check=True)
            outs.append(torch_load(fn))
    (a1, a2), (b1, b2), (c1, c2) = outs
    assert rel_l2(a1.numpy(), b1.numpy()) <= 1e-6
    assert rel_l2(a2.numpy(), b2.numpy()) <= 1e-6
    assert rel_l2(a2.numpy(), b1.numpy()[7:16]) <= 1e-6
    # the transposed frame in z pieces of 4 planes (the path taken when a
    # slab-sized accumulator does not fit): pieces of 23 and of the 9-plane
    # slab, each accumulated and transposed-added in turn
    assert rel_l2(c1.numpy(), b1.numpy()) <= 1e-6
    assert rel_l2(c2.numpy(), b2.numpy()) <= 1e-6


def torch_load(path):
    import torch
    return torch.load(path)


def test_randomised_geometries_vs_oracle():
    """Seeded random sweep (tools/fuzz_parity.py): grids 3-40 per axis with
    anisotropic voxels and offsets, detectors 4-47 px with offsets, source
    distances from 1.3 grid radii, 1-12 arbitrary angles, random slab and
    view windows; interp / Siddon Ax, matched / FDK Atb against the oracle."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "tools", "fuzz_parity.py")
    spec = importlib.util.spec_from_file_location("fuzz_parity", path)
    fz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fz)
    rng = np.random.default_rng(2026)
    for _ in range(15):
        while True:
            try:
                g = fz.case(rng)
                break
            except ValueError:
                continue
        og = to_oracle(g)
        grid, det = g.voxel_grid, g.detector
        na, nz = g.n_angles, grid.n_z
        x = rng.random((nz, grid.n_y, grid.n_x), dtype=np.float32)
        y = rng.standard_normal((na, det.n_v, det.n_u)).astype(np.float32)
        z0 = int(rng.integers(0, nz))
        z1 = int(rng.integers(z0 + 1, nz + 1))
        a0 = int(rng.integers(0, na))
        a1 = int(rng.integers(a0 + 1, na + 1))
        xs = x[z0:z1]
        vol = cs.Volume(grid, xs, (z0, z1))
        assert rel_l2(cs.forward_project_slab(vol, g, (a0, a1), IP).data,
                      O.fwd_interp(xs, og, (a0, a1), (z0, z1))) <= TOL_OP
        assert rel_l2(cs.forward_project_slab(
            vol, g, (a0, a1), cs.ProjectionMethod.SIDDON).data,
            O.fwd_siddon(xs, og, (a0, a1), (z0, z1))) <= TOL_OP
        st = cs.ProjectionStack(det, y[a0:a1], (a0, a1))
        for mode, ofn in ((cs.WeightMode.MATCHED, O.bwd_matched),
                          (cs.WeightMode.FDK, O.bwd_fdk)):
            assert rel_l2(cs.backproject_slab(st, g, (z0, z1), mode).data,
                          ofn(y[a0:a1], og, (a0, a1), (z0, z1))) <= TOL_OP


def test_fdk_thin_slab_fine_pixels_regression():
    """Regression (found by tools/fuzz_parity.py with FUZZ_FINE): a 2-plane
    slab under pixels ~6x finer than voxels -- the staged FDK read planes
    past the slab outside its staged footprint (an illegal shared-memory
    address); they are no longer sampled."""
    grid = cs.VoxelGrid(38, 26, 28, (1.353254259269713, 0.7477279089896511,
                                     0.830182913402348),
                        (2.2413206723775714, -2.9684081726065514,
                         1.9273705102965977))
    det = cs.DetectorGrid(86, 35, (0.1323645593008397, 0.14701814799123764),
                          (0.031064659895868055, 0.1651667141129686))
    g = cs.ScanGeometry(109.23412942205707, 175.3939285422945,
                        (6.937003968081498, 4.097266868992543,
                         1.7105092121762766, 6.845442067546388), grid, det)
    og = to_oracle(g)
    y = np.random.default_rng(3).standard_normal((4, 35, 86)).astype(
        np.float32)
    for zr in ((26, 28), (0, 28), (5, 6)):
        st = cs.ProjectionStack(det, y[2:3], (2, 3))
        got = cs.backproject_slab(st, g, zr, cs.WeightMode.FDK).data
        assert rel_l2(got, O.bwd_fdk(y[2:3], og, (2, 3), zr)) <= TOL_OP, zr
