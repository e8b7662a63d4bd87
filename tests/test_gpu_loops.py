"""Reconstruction loops on the GPU vs the oracle's loops (the reference's
algorithms.py:204-304 restated in oracle/oracle.py): randomised geometry
sweeps, BASELINE config 1's SIRT-10 / CGLS-10 and one config-2 OS-SART
iteration on a 36-view window.  Tolerance 3e-5 relL2 (3x the
operator tolerance)."""

from __future__ import annotations

import importlib.util
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1905_03748_b200 as cs
from conftest import rel_l2, synth_geometry, to_oracle
from oracle import oracle as O

TOL_LOOP = 3e-5
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _fuzz_module(**env):
    """tools/fuzz_parity.py with its FUZZ_* knobs (read at import)."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        spec = importlib.util.spec_from_file_location(
            "fuzz_parity_" + "_".join(f"{k}{v}" for k, v in env.items()),
            os.path.join(ROOT, "tools", "fuzz_parity.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        return mod
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _sweep(fz, seed, n_cases):
    """tools/fuzz_loops.py: random geometries, block sizes, relaxations and
    iteration counts; OS-SART, CGLS and (half the cases) SART-TV."""
    rng = np.random.default_rng(seed)
    pool = cs.DevicePool.b200(1)
    bad = []
    for i in range(n_cases):
        while True:
            try:
                g = fz.case(rng)
                if min(g.voxel_grid.counts) >= 2:
                    break
            except ValueError:
                continue
        og = to_oracle(g)
        grid, det, na = g.voxel_grid, g.detector, g.n_angles
        x = rng.random((grid.n_z, grid.n_y, grid.n_x), dtype=np.float32)
        b = O.fwd_interp(x, og).astype(np.float32)
        stack = cs.ProjectionStack(det, b)
        its = int(rng.integers(1, 4))
        block = int(rng.integers(1, na + 1))
        lam = float(rng.uniform(0.3, 1.5))
        errs = {}
        got = cs.os_sart(stack, g, cs.ReconConfig(
            pool, cs.Algorithm.OSSART, its, block, lam)).data
        errs["os_sart"] = rel_l2(got, O.os_sart(b, og, its, block, lam))
        r = cs.cgls(stack, g, cs.ReconConfig(pool, cs.Algorithm.CGLS, its))
        xo, _, _ = O.cgls(b, og, its)
        errs["cgls"] = rel_l2(r.volume.data, xo)
        if rng.random() < 0.5 and grid.n_z >= 4:
            tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 3, 1e-3)
            got = cs.os_sart(stack, g, cs.ReconConfig(
                pool, cs.Algorithm.OSSART, its, block, lam, tv=tv)).data
            ref = O.os_sart(b, og, its, block, lam,
                            tv=dict(n_slabs=1, minimizer="gd", outer_syncs=1,
                                    inner_iters=3, step=1e-3))
            errs["sart_tv"] = rel_l2(got, ref)
        worst = max(errs.values())
        if not worst <= TOL_LOOP:
            bad.append((i, list(grid.counts), na, block, errs))
    return bad


def test_loop_sweep_vs_oracle():
    """The 25-case sweep of tools/fuzz_loops.py (seed 3) that put OS-SART
    at 1.9e-3 in r01: low-coverage voxels (weight tails of the outermost
    rays) need the matched kernel's precise boxes."""
    bad = _sweep(_fuzz_module(FUZZ_MAXN="20"), 3, 25)
    assert not bad, bad


def test_loop_sweep_coarse_detectors_vs_oracle():
    """Large detectors (64-128 px) of coarse pixels, rays 1.6-3 voxels
    apart: interior voxels between rays see only weight tails, which the
    precise boxes' ray-gap rule covers for few-view blocks."""
    bad = _sweep(_fuzz_module(FUZZ_MAXN="20", FUZZ_COARSE="1"), 5, 10)
    assert not bad, bad


def _config1():
    g = synth_geometry(64, 100)
    x = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid).data
    og = to_oracle(g)
    return g, og, O.fwd_interp(x, og).astype(np.float32)


def test_config1_sirt10_vs_oracle():
    """BASELINE config 1: 64^3, 64^2 detector, 100 views, 10 SIRT
    iterations (os_sart with one block of all views)."""
    g, og, b = _config1()
    pool = cs.DevicePool.b200(1)
    got = cs.os_sart(cs.ProjectionStack(g.detector, b), g, cs.ReconConfig(
        pool, cs.Algorithm.OSSART, 10, 100)).data
    assert rel_l2(got, O.os_sart(b, og, 10, 100)) <= TOL_LOOP


def test_config1_cgls10_vs_oracle():
    g, og, b = _config1()
    pool = cs.DevicePool.b200(1)
    r = cs.cgls(cs.ProjectionStack(g.detector, b), g,
                cs.ReconConfig(pool, cs.Algorithm.CGLS, 10))
    xo, reso, _ = O.cgls(b, og, 10)
    assert rel_l2(r.volume.data, xo) <= TOL_LOOP
    np.testing.assert_allclose(r.residuals, reso, rtol=TOL_LOOP)


def test_config2_ossart_window_vs_oracle():
    """Config 2 geometry (512^3, 512^2 detector) on the first 36 views of
    the 360-view scan: one OS-SART iteration with one block of 36 (the
    bench's block size) against the oracle."""
    n = 512
    g360 = synth_geometry(n, 360)
    g = g360.with_angles(g360.angles[:36])
    og = to_oracle(g)
    x = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid).data
    b = O.fwd_interp(x, og).astype(np.float32)
    pool = cs.DevicePool.b200(1)
    got = cs.os_sart(cs.ProjectionStack(g.detector, b), g, cs.ReconConfig(
        pool, cs.Algorithm.OSSART, 1, 36)).data
    ref = O.os_sart(b, og, 1, 36)
    assert rel_l2(got, ref) <= TOL_LOOP
    assert math.isfinite(float(np.abs(got).max()))


def test_bench_self_launched_two_ranks_config3():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself; with
    CS_BENCH_BACKEND=gloo they share this GPU.  The line is the config-3
    slab/angle-split step (shrunk here) reported for 2 GPUs."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, CS_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
         "--steps", "2", "--warmup", "3", "--c3-size", "128",
         "--c3-angles", "64", "--c3-block", "16"],
        env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong"
    assert rec["config"]["workload"].startswith("config 3")
    assert rec["value"] > 0 and rec["gpu_launches"] > 0


def _dist_loop_worker(rank, world, port, q):
    import sys
    import torch
    import torch.distributed as dist
    for p in (ROOT, os.path.join(ROOT, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1905_03748_b200 as cs
    from conftest import rel_l2, synth_geometry, to_oracle
    from oracle import oracle as O
    g = synth_geometry(24, 10)
    og = to_oracle(g)
    x = np.random.default_rng(0).random((24, 24, 24), dtype=np.float32)
    b = O.fwd_interp(x, og).astype(np.float32)
    pool = cs.DevicePool(tuple(cs.DeviceSpec(memory_budget=2 ** 31)
                               for _ in range(world)))
    stack = cs.ProjectionStack(g.detector, b)
    errs = {}
    r = cs.cgls(stack, g, cs.ReconConfig(pool, cs.Algorithm.CGLS, 3))
    errs["cgls"] = rel_l2(r.volume.data, O.cgls(b, og, 3)[0])
    got = cs.os_sart(stack, g, cs.ReconConfig(pool, cs.Algorithm.OSSART, 2,
                                              3, 0.8)).data
    errs["os_sart"] = rel_l2(got, O.os_sart(b, og, 2, 3, 0.8))
    tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 3, 1e-3)
    got = cs.os_sart(stack, g, cs.ReconConfig(pool, cs.Algorithm.OSSART, 2,
                                              5, tv=tv)).data
    ref = O.os_sart(b, og, 2, 5, tv=dict(n_slabs=1, minimizer="gd",
                                         outer_syncs=1, inner_iters=3,
                                         step=1e-3))
    errs["sart_tv"] = rel_l2(got, ref)
    if rank == 0:
        q.put(errs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_loops_on_gpu_vs_oracle(world):
    """cgls / os_sart / SART-TV through the public API under
    torch.distributed (gloo, ranks sharing this GPU): x slab-sharded,
    projections angle-sharded, the sm_100a kernels per rank -- against the
    oracle's single-process loops."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_loop_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        errs = q.get(timeout=600)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    assert max(errs.values()) <= TOL_LOOP, errs
