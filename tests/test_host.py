"""Host-side logic of the product (no GPU): planner parity with the
reference's plans, geometry, the C-ABI library's exports, and the
no-CPU-fallback rule."""

from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np
import pytest
import torch

import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import _lib
from paper_1905_03748_b200.geometry import flat_geometry, grid6
from conftest import ROOT, product_geometry, to_oracle
from oracle import oracle as O


def _plan_case(c):
    grid = cs.VoxelGrid(c["n"], c["n"], c["nz"])
    det = cs.DetectorGrid(c["nu"], c["nv"])
    r = grid.bounding_radius()
    g = cs.ScanGeometry(3 * r + 1, 7 * r + 2, tuple(
        np.linspace(0, 2 * math.pi, c["A"], endpoint=False)), grid, det)
    pool = cs.DevicePool(tuple(cs.DeviceSpec(memory_budget=c["budget"])
                               for _ in range(c["dev"])))
    fn = cs.plan_forward if c["op"] == "forward" else cs.plan_backward
    return fn(g, pool, usable_fraction=c["uf"])


def test_planner_matches_reference(golden_meta):
    """Slab ranges, angle ranges, chunks, buffers, pin flag, peak bytes:
    bit-exact integers against the reference's plans."""
    for c in golden_meta["plans"]:
        ref = c["plan"]
        if ref is None:
            with pytest.raises(cs.InfeasiblePlanError):
                _plan_case(c)
            continue
        p = _plan_case(c)
        assert p.n_splits == ref["n_splits"]
        assert [list(t) for t in p.slab_ranges] == ref["slab_ranges"]
        assert [list(t) for t in p.angle_assignment] == \
            ref["angle_assignment"]
        assert p.chunk_angles == ref["chunk_angles"]
        assert p.buffer_count == ref["buffer_count"]
        assert p.pin_host_image == ref["pin_host_image"]
        assert p.per_device_bytes_peak == ref["per_device_bytes_peak"]


def test_planner_kat_512_256mib():
    """512^3, 256 MiB device -> 3 splits both ways."""
    grid = cs.VoxelGrid(512, 512, 512)
    det = cs.DetectorGrid(512, 512)
    g = cs.ScanGeometry(2048.0, 4096.0, tuple(
        np.linspace(0, 2 * math.pi, 512, endpoint=False)), grid, det)
    pool = cs.DevicePool((cs.DeviceSpec(memory_budget=256 * 2 ** 20),))
    pf = cs.plan_forward(g, pool, usable_fraction=1.0)
    pb = cs.plan_backward(g, pool, usable_fraction=1.0)
    assert pf.n_splits == 3 and pb.n_splits == 3
    assert pf.slab_ranges == ((0, 171), (171, 342), (342, 512))
    assert pf.buffer_count == 3 and pf.pin_host_image


def test_planner_infeasible():
    grid = cs.VoxelGrid(64, 64, 64)
    g = cs.ScanGeometry(200.0, 400.0, (0.0, 1.0), grid,
                        cs.DetectorGrid(64, 64))
    pool = cs.DevicePool((cs.DeviceSpec(memory_budget=20000),))
    with pytest.raises(cs.InfeasiblePlanError):
        cs.plan_forward(g, pool)


def test_slab_queues_round_robin():
    p = cs.SplitPlan(cs.OpKind.BACKWARD, 5, cs.scheduler.slab_ranges(10, 5),
                     ((0, 4),), 4, 2, True, 0)
    assert p.slab_queues(2) == [[0, 2, 4], [1, 3]]
    assert p.slab_queues(1) == [[0, 1, 2, 3, 4]]


def test_flat_geometry_bit_exact(golden_meta):
    for d in golden_meta["geometries"].values():
        g = product_geometry(d)
        og = to_oracle(g)
        np.testing.assert_array_equal(flat_geometry(g, 0, g.n_angles),
                                      O.flat_geometry(og, 0, og.n_angles))
        np.testing.assert_array_equal(grid6(g.voxel_grid), og.grid6())


def test_geometry_kats():
    """SPEC.md:56-58, :65-67."""
    grid = cs.VoxelGrid(8, 8, 8)
    det = cs.DetectorGrid(5, 5, (4.0, 4.0))
    g = cs.ScanGeometry(100.0, 200.0, (0.0, math.pi / 2, math.pi), grid, det)
    np.testing.assert_allclose(cs.source_position(g, 0), [100, 0, 0])
    np.testing.assert_allclose(cs.source_position(g, 1), [0, 100, 0],
                               atol=1e-9)
    r = cs.pixel_ray(g, 0, 2, 2)
    np.testing.assert_allclose(r.direction, [-1, 0, 0], atol=1e-15)
    assert r.hits
    # plane-distance property: origin + dsd * dir lies on the detector plane
    for (a, u, v) in [(0, 0, 4), (1, 3, 1), (2, 4, 0)]:
        ray = cs.pixel_ray(g, a, u, v)
        th = g.angles[a]
        axis = np.array([math.cos(th), math.sin(th), 0.0])
        cen = (g.dso - g.dsd) * axis
        p = np.array(ray.origin) + 1.0 * np.array(ray.direction) * (
            g.dsd / float(np.dot(-np.array(ray.direction), axis)))
        assert abs(float(np.dot(p - cen, axis))) < 1e-9 * g.dsd
    with pytest.raises(ValueError):
        cs.ScanGeometry(5.0, 200.0, (0.0,), grid, det)  # grid hits source
    with pytest.raises(ValueError):
        cs.ScanGeometry(100.0, 101.0, (0.0,), grid, det)  # hits detector
    with pytest.raises(IndexError):
        cs.source_position(g, 3)


def test_siddon_trace_kats():
    """axis-aligned 3x1x1 traversal; 45 deg diagonal."""
    grid = cs.VoxelGrid(3, 1, 1)
    ray = cs.Ray((10.0, 0.0, 0.0), (-1.0, 0.0, 0.0), 8.5, 11.5)
    tr = cs.siddon_trace(ray, grid)
    assert [i for i, _ in tr] == [(2, 0, 0), (1, 0, 0), (0, 0, 0)]
    np.testing.assert_allclose([l for _, l in tr], [1.0, 1.0, 1.0])
    g = cs.VoxelGrid(4, 4, 1)
    s = 1 / math.sqrt(2)
    ray = cs.Ray((-2.0 - 1.0, -2.0 - 1.0, 0.0), (s, s, 0.0),
                 math.sqrt(2), 5 * math.sqrt(2))
    tr = cs.siddon_trace(ray, g)
    assert len(tr) == 4
    np.testing.assert_allclose([l for _, l in tr], [math.sqrt(2)] * 4,
                               rtol=1e-9)
    assert cs.siddon_trace(cs.Ray((0, 0, 0), (1, 0, 0), 1.0, -1.0), g) == []


HEADER = os.path.join(ROOT, "include", "conesplit_b200.h")


def _header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    """The built C-ABI library loads without a GPU and exports every entry
    point include/conesplit_b200.h declares (and ctypes binds them all)."""
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build()"
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(L, name), name
    assert set(syms) == set(_lib.SYMBOLS), set(syms) ^ set(_lib.SYMBOLS)
    bound = _lib.load_library()
    assert bound.cs_version().decode().startswith("conesplit-b200")


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only check")
def test_no_cpu_fallback():
    """Operators fail loudly without a GPU instead of computing on CPU."""
    grid = cs.VoxelGrid(4, 4, 4)
    g = cs.ScanGeometry(20.0, 40.0, (0.0,), grid, cs.DetectorGrid(4, 4))
    vol = cs.Volume(grid, np.ones((4, 4, 4), np.float32))
    with pytest.raises(cs.NativeLibraryError):
        cs.forward_project_slab(vol, g, (0, 1),
                                cs.ProjectionMethod.INTERPOLATED)


def test_validation_errors():
    grid = cs.VoxelGrid(4, 4, 4)
    g = cs.ScanGeometry(20.0, 40.0, (0.0, 1.0), grid, cs.DetectorGrid(4, 4))
    vol = cs.Volume(grid, np.ones((4, 4, 4), np.float32))
    with pytest.raises(ValueError):
        cs.forward_project_slab(vol, g, (0, 3))
    other = cs.Volume(cs.VoxelGrid(4, 4, 5), np.ones((5, 4, 4), np.float32))
    with pytest.raises(ValueError):
        cs.forward_project_slab(other, g, (0, 1))
    with pytest.raises(ValueError):
        cs.Volume(grid, np.ones((3, 4, 4)), (0, 4))
    with pytest.raises(ValueError):
        cs.ProjectionStack(g.detector, np.ones((2, 4, 4)), (0, 3))
    with pytest.raises(ValueError):
        cs.backproject_slab(cs.ProjectionStack(g.detector,
                                               np.ones((2, 4, 4))),
                            g, (0, 5))
    with pytest.raises(ValueError):
        cs.ReconConfig(cs.DevicePool((cs.DeviceSpec(1),)), relaxation=2.0)


def test_halo_slabs_match_reference():
    for nz, n, d in [(32, 1, 8), (32, 3, 5), (17, 4, 2), (10, 10, 1)]:
        ours = [(s.core_range, s.window)
                for s in cs.regularization.make_halo_slabs(nz, n, d)]
        ref = O.make_halo_slabs(nz, n, d)
        assert ours == ref


def test_refine_for_overlap():
    """Executor slab refinement (execution._refine_for_overlap): the fewest
    equal parts (<= 4) letting two slab buffers fit beside fixed bytes;
    parts tile every slab exactly and keep the plan's order."""
    from paper_1905_03748_b200.execution import _refine_for_overlap
    plane = 1000  # elements per plane -> 4000 B
    slabs = ((0, 10), (10, 20), (20, 25))
    # two 10-plane buffers fit: unchanged
    assert _refine_for_overlap(slabs, plane, 1000, 2 * 10 * 4000 + 1000) == slabs
    # only 2 x 5 planes fit: halves
    out = _refine_for_overlap(slabs, plane, 0, 2 * 5 * 4000)
    assert out == ((0, 5), (5, 10), (10, 15), (15, 20), (20, 23), (23, 25))
    # nothing up to 4 parts fits: unchanged (the chunked path takes over)
    assert _refine_for_overlap(slabs, plane, 0, 2 * 2 * 4000) == slabs
    # a single slab is left alone
    assert _refine_for_overlap(((0, 7),), plane, 0, 10) == ((0, 7),)
    for budget in range(40000, 200000, 7000):
        out = _refine_for_overlap(slabs, plane, 3000, budget)
        flat = [z for s in out for z in s]
        assert flat[0] == 0 and flat[-1] == 25
        assert all(a[1] == b[0] for a, b in zip(out, out[1:]))
        assert all(b > a for a, b in out)


def test_bench_self_launch_command():
    """bench.py --gpus N (outside torchrun) starts N ranks through
    torch.distributed.run on 127.0.0.1 with its own arguments."""
    import importlib.util
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location(
        "bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    cmd = bench.launcher_cmd(["--gpus", "4", "--steps", "2"], 4, 29501)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert "--master-addr=127.0.0.1" in cmd and "--master-port=29501" in cmd
    i = cmd.index(os.path.join(root, "bench.py"))
    assert cmd[i + 1:] == ["--gpus", "4", "--steps", "2"]


def test_refhook_signatures_match_reference():
    """paper_1905_03748_b200.refhook's kernels take exactly the reference's
    arguments (conesplit/_kernels.py:154, :213, :278, :340), so install()
    can replace them in the reference's module.  Needs the reference
    source (this container; absent on GPU boxes)."""
    import importlib
    import inspect
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference source not present")
    sys.path.insert(0, src)
    try:
        try:
            ref = importlib.import_module("conesplit._kernels")
        except Exception as e:  # numba missing etc.
            pytest.skip(f"reference kernels not importable: {e}")
        from paper_1905_03748_b200 import refhook
        for name, fn in refhook.HOOKS.items():
            rf = getattr(ref, name)
            rf = getattr(rf, "py_func", rf)
            assert (list(inspect.signature(fn).parameters)
                    == list(inspect.signature(rf).parameters)), name
    finally:
        sys.path.remove(src)


def test_guarded_inverse_matches_numpy_bits():
    """_ginv (out-of-core OS-SART weights, algorithms.py:254-258 of the
    reference: a >= 1e-8 ? 1 / a : 0) gives numpy's fp32 bits, in place on
    writable input and on a copy of read-only input."""
    import numpy as np
    from paper_1905_03748_b200.algorithms import INVERSE_GUARD, _ginv
    rng = np.random.default_rng(5)
    a = rng.random(10007).astype(np.float32) * 3.0
    a[::7] = 0.0
    a[::11] = 5e-9
    a[::13] = np.float32(INVERSE_GUARD)
    want = np.zeros_like(a)
    m = a >= INVERSE_GUARD
    want[m] = np.float32(1.0) / a[m]
    got = _ginv(a.copy())
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    ro = a.copy()
    ro.flags.writeable = False
    got2 = _ginv(ro)
    assert np.array_equal(got2.view(np.uint32), want.view(np.uint32))
    assert np.array_equal(ro, a)
