"""The kernel-level drop-in (paper_1905_03748_b200/refhook.py, INTEGRATION.md
section 2): the four replacements for the reference's numba kernels, called
exactly the way the reference's operators call them (projectors.py:265-315:
angle chunks of 9 / 32 views, float64 slab accumulators that are added to),
against the oracle.  On a GPU box the reference itself is absent, so the
call sites are restated here; test_host.py checks the signatures against
the reference where it is installed."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import refhook as R
from paper_1905_03748_b200.geometry import flat_geometry, grid6
from paper_1905_03748_b200.projectors import sample_step
from conftest import rel_l2, to_oracle
from oracle import oracle as O


def _geometry():
    grid = cs.VoxelGrid(21, 18, 15, (1.0, 0.9, 1.1), (0.3, -0.2, 0.1))
    r = grid.bounding_radius()
    det = cs.DetectorGrid(27, 19, (2.2, 2.4), (0.4, -0.3))
    angles = tuple(np.linspace(0.1, 0.1 + 2 * np.pi, 23, endpoint=False))
    return cs.ScanGeometry(2.5 * r + 2.0, 5.0 * r + 4.0, angles, grid, det)


def _split(fg):
    return fg[:, 0:3], fg[:, 3:6], fg[:, 6:9], fg[:, 9:12]


def test_refhook_kernels_vs_oracle():
    g = _geometry()
    og = to_oracle(g)
    grid, det = g.voxel_grid, g.detector
    nx, ny, nz = grid.n_x, grid.n_y, grid.n_z
    gp = tuple(float(v) for v in grid6(grid))
    rng = np.random.default_rng(4)
    x = rng.random((nz, ny, nx), dtype=np.float32)
    A = g.n_angles
    y = rng.standard_normal((A, det.n_v, det.n_u)).astype(np.float32)
    step = sample_step(grid)
    # Ax, interpolated and Siddon, in chunks of 9 views over a slab
    z0, z1 = 3, 12
    for name, ref in (("interp", O.fwd_interp), ("siddon", O.fwd_siddon)):
        out_all = np.empty((A, det.n_v, det.n_u), np.float32)
        for c0 in range(0, A, 9):
            c1 = min(c0 + 9, A)
            s, d0, us, vs = _split(flat_geometry(g, c0, c1))
            out = out_all[c0:c1]
            if name == "interp":
                R.interp_forward_chunk(x[z0:z1], s, d0, us, vs, *gp, nx, ny,
                                       nz, z0, z1, step, 8, 8, out)
            else:
                R.siddon_forward_chunk(x[z0:z1], s, d0, us, vs, *gp, nx, ny,
                                       nz, z0, z1, 8, 8, out)
        want = ref(x[z0:z1], og, slab=(z0, z1))
        assert rel_l2(out_all, want) <= 1e-5, name
    # Atb, matched and FDK, into a float64 slab accumulator that is ADDED to
    for mode, ref in (("matched", O.bwd_matched), ("fdk", O.bwd_fdk)):
        acc = np.full((z1 - z0, ny, nx), 0.25, np.float64)
        for c0 in range(0, A, 9):
            c1 = min(c0 + 9, A)
            if mode == "matched":
                s, d0, us, vs = _split(flat_geometry(g, c0, c1))
                R.matched_backward_chunk(acc, y[c0:c1], s, d0, us, vs, *gp,
                                         nx, ny, nz, z0, z1, step)
            else:
                th = np.array(g.angles[c0:c1])
                R.fdk_backward_chunk(acc, y[c0:c1], np.cos(th), np.sin(th),
                                     g.dso, g.dsd, *det.pixel_size,
                                     *det.detector_offset, *gp, z0, 8, 8)
        want = ref(y, og, slab=(z0, z1)) + 0.25
        assert rel_l2(acc, want) <= 1e-5, mode


def test_refhook_install_restores():
    import types
    mod = types.SimpleNamespace(**{k: None for k in R.HOOKS})
    old = R.install(mod)
    assert all(getattr(mod, k) is R.HOOKS[k] for k in R.HOOKS)
    for k, v in old.items():
        setattr(mod, k, v)
    assert all(getattr(mod, k) is None for k in R.HOOKS)
