#!/usr/bin/env python
"""Bench: cone-beam Ax / Atb GUPS on B200 (BASELINE.json metric).

One *step* = one pass of the loop hot path over one batch of views:
interpolated Ax + matched (exact-adjoint) Atb -- the operator pair every
OS-SART / SIRT / CGLS iteration applies (algorithms.py:213-216,
:280-283).  Unit: voxel x angle updates.  The Atb input is a DENSE stack
(every ray that meets the grid carries a non-zero value, like a loop
residual); the sparse Ax(phantom) stack, whose zero rays the reference
skips (_kernels.py:295-296), is reported beside it.

* N = 1 (default): BASELINE config 2 -- 512^3 volume, 512^2 detector, 360
  views; plus the config-3 block step on one GPU (``config3_step``, the
  N = 1 point of the scaling curve), FDK / TV / loop timings, the e2e
  number through the public API on host buffers, and the CPU oracle.
* N > 1: BASELINE config 3 -- 2048^3 volume, 2048^2 detector, 1024 views
  -- slab/angle split over the N ranks (sharded.py): each step is one
  64-view OS-SART block: every rank projects its 2048^3 / N slab for the
  block's views, one NCCL reduce-scatter per round sums the slab partials
  onto the view owners, the weighted residual is formed on the owner, one
  all-gather per round hands every rank the block, and every rank
  backprojects into its slab.  Total work per step is fixed (strong
  scaling).  ``python bench.py --gpus N`` launches the N ranks itself
  (torch.distributed.run, 127.0.0.1) unless it already runs under one.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_VOX = 512
N_ANG = 360
CHUNK = 90  # views per kernel launch
N_DET = 512
C3_VOX = 2048        # config 3
C3_ANG = 1024
C3_BLOCK = 64        # views per config-3 step (one OS-SART block)
METRIC = "Ax/Atb GUPS (voxel x angle updates/s), interp Ax + matched Atb"
UNIT = "GUPS"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", type=int, default=N_VOX)
    ap.add_argument("--angles", type=int, default=N_ANG)
    ap.add_argument("--no-extras", action="store_true",
                    help="skip OS-SART / e2e / CPU baseline (profiling runs)")
    ap.add_argument("--cpu-sample-angles", type=int, default=4)
    ap.add_argument("--c3-size", type=int, default=C3_VOX,
                    help="config-3 volume edge (tests shrink it)")
    ap.add_argument("--c3-angles", type=int, default=C3_ANG)
    ap.add_argument("--c3-block", type=int, default=C3_BLOCK)
    ap.add_argument("--no-c3", action="store_true",
                    help="N = 1: skip the config-3 block step")
    return ap.parse_args()


def launcher_cmd(argv, n_gpus, port):
    """torch.distributed.run command for N ranks on this node (rendezvous
    on 127.0.0.1: the container hostname may not resolve)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={n_gpus}", "--master-addr=127.0.0.1",
            f"--master-port={port}", os.path.abspath(__file__), *argv]


def self_launch(args):
    """--gpus N > 1 outside torchrun: start the N ranks and wait."""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")   # communicator init in the log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout: the JSON line
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(launcher_cmd(sys.argv[1:], args.gpus, port),
                           env=env)


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def make_geometry(n, n_angles, cs):
    """SURVEY 8(d) make_geo: dso = 2N, dsd = 4N, 1 mm voxels, pitch
    2 sqrt(2) N / N_det, angles over 2 pi."""
    import numpy as np
    mag = 2.0
    diag = math.sqrt(2.0) * n
    det = cs.DetectorGrid(n, n, (mag * diag / n, mag * max(diag, n) / n))
    angles = tuple(np.linspace(0.0, 2 * math.pi, n_angles, endpoint=False))
    return cs.ScanGeometry(2.0 * n, 4.0 * n, angles, cs.VoxelGrid(n, n, n),
                           det)


def bytes_per_update(n, n_det):
    """4 (1 + Nu Nv / Nvox) B per voxel-angle update."""
    return 4.0 * (1.0 + n_det * n_det / float(n ** 3))


class Clocks:
    """nvidia-smi sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 7:
                    rows.append(f)
        except OSError:
            pass
        finally:
            if self.path:
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        load = [r for r in rows if r[6] not in ("0", "[N/A]")] or rows
        sm = [float(r[0]) for r in load if r[0].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in load for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].isdigit()
                else None,
                "reasons": reasons, "samples": len(load)}


def cpu_oracle_sample(g, x_np, y_np, n_sample, threads, slab=None):
    """Oracle (C port, all host threads) on an angle window (and optionally
    a slab of planes): interpolated Ax + matched Atb of the dense stack
    y_np.  Returns (GUPS, seconds, updates)."""
    from oracle import oracle as O
    og = O.OGeom(g.dso, g.dsd, g.angles, g.voxel_grid.n_x, g.voxel_grid.n_y,
                 g.voxel_grid.n_z, nu=g.detector.n_u, nv=g.detector.n_v,
                 pixel=g.detector.pixel_size)
    win = (0, n_sample)
    z0, z1 = slab or (0, g.voxel_grid.n_z)
    t0 = time.perf_counter()
    O.fwd_interp(x_np, og, win, (z0, z1), threads=threads)
    O.bwd_matched(y_np[:n_sample], og, win, (z0, z1), threads=threads)
    dt = time.perf_counter() - t0
    upd = 2.0 * n_sample * float(x_np.size)
    return upd / dt / 1e9, dt, upd


def dense_stack(shape, dev, seed=1):
    """Dense Atb input (a residual-like stack: every ray non-zero)."""
    import torch
    return torch.randn(shape, device=dev,
                       generator=torch.Generator(device=dev).manual_seed(seed))


def load_traffic(kernel_key):
    """dram bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        return d.get(kernel_key)
    except (OSError, ValueError):
        return None


def load_limits(kernel_key):
    """ncu pipe utilisations of a kernel from the committed summary
    (profiles/ncu_limits.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_limits.json")))
        return d.get(kernel_key)
    except (OSError, ValueError):
        return None


def measured_peak():
    """HBM GB/s from MEASURED_PEAKS.json (driver-written), else the
    profiling guide's fallback."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback"


# --------------------------------------------------------------------------


def run_reference(args):
    """The reference's CPU path on this box's host cores: the oracle C port
    (bit-exact to the reference on every golden; the numba reference
    cannot travel to the GPU box).  Same metric / config as our arm; each
    step is a bounded sample of it (a view window, and at config 3 a slab
    of planes)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import numpy as np
    import paper_1905_03748_b200 as cs
    from oracle import oracle as O
    O.lib()
    c3 = world > 1 or args.gpus > 1
    n, na = (args.c3_size, args.c3_angles) if c3 else (args.size, args.angles)
    g = make_geometry(n, na, cs)
    threads = O.default_threads()
    n_s = 1 if c3 else max(1, min(args.cpu_sample_angles, na))
    slab = (n // 2 - 32, n // 2 + 32) if c3 else None
    x = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                   slab_range=slab).data
    y = np.random.default_rng(1).standard_normal(
        (n_s, n, n)).astype(np.float32)
    for _ in range(args.warmup):
        cpu_oracle_sample(g, x, y, n_s, threads, slab)
    times = []
    upd = 0.0
    for _ in range(args.steps):
        _, dt, upd = cpu_oracle_sample(g, x, y, n_s, threads, slab)
        times.append(dt)
    tot = sum(times)
    val = upd * args.steps / tot / 1e9
    sample = (f"{n_s}-view window" + (f" x planes {slab}" if slab else "")
              + " per step (window / slab outputs are exact slices of the "
              "full operators); dense Atb input")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": max(world, args.gpus), "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "strong" if c3 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (Shepp-Logan 3D phantom; dense "
        "standard-normal Atb input)",
        "config": {"workload": (f"config 3: {n}^3 volume, {n}^2 detector, "
                                f"{na} views" if c3 else
                                f"config 2: {n}^3 volume, {n}^2 detector, "
                                f"{na} views") +
                   "; interp Ax + matched Atb", "sample": sample},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class StepTimer:
    """Per-step CUDA events on the launching stream around the Ax and Atb
    halves of a step."""

    def __init__(self, steps):
        import torch
        self.ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)]
                   for _ in range(steps)]

    def mark(self, i, k, stream):
        if i is not None:
            self.ev[i][k].record(stream)

    def halves(self):
        n = len(self.ev)
        t_ax = sum(e[0].elapsed_time(e[1]) for e in self.ev) * 1e-3 / n
        t_atb = sum(e[1].elapsed_time(e[2]) for e in self.ev) * 1e-3 / n
        return t_ax, t_atb


def timed(steps, warmup, step, dist_on, dev_index, backend):
    """W untimed steps, then K steps between barriers + synchronize on the
    device clock (max over ranks).  Returns (seconds, clocks, launches)."""
    import torch
    import torch.distributed as dist
    from paper_1905_03748_b200 import kernels as K
    stream = torch.cuda.current_stream()
    for _ in range(max(3, warmup)):
        step(None)
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = K.launch_count()
    with Clocks(dev_index) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(steps):
            step(i)
        t_end.record(stream)
        torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    launches = K.launch_count() - launches0
    elapsed = t_start.elapsed_time(t_end) * 1e-3
    if dist_on:
        on_dev = backend == "nccl"
        t = torch.tensor([elapsed], dtype=torch.float64,
                         device=torch.device("cuda", dev_index) if on_dev
                         else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    return elapsed, clk.summary(), launches


def roofline(kname, t_launch, upd_launch, bpu):
    peak, peak_kind = measured_peak()
    achieved = upd_launch * bpu / t_launch / 1e9
    return {"bound": "hbm", "kernel": kname, "achieved": achieved,
            "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": load_traffic(kname), "peak_source": peak_kind,
            "bytes_per_update": bpu, "updates_per_launch": upd_launch,
            "launch_ms": t_launch * 1e3,
            # the pipe that actually bounds this gather kernel (ncu --set
            # full, committed summary)
            "ncu_pipes": load_limits(kname)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    # one rank per GPU; CS_BENCH_BACKEND=gloo lets several ranks share a GPU
    # to exercise the N>1 path on a 1-GPU box (timings then are not scaling)
    backend = os.environ.get("CS_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl",
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    try:
        if world == 1:
            line = run_config2(args, local)
        else:
            line = run_config3(args, rank, world, local, backend)
        if rank == 0:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            dist.destroy_process_group()
    return 0


def run_config2(args, local):
    """N = 1: config 2, 4 x 90-view launches of each operator per step."""
    import torch
    import paper_1905_03748_b200 as cs
    from paper_1905_03748_b200 import kernels as K

    n, A = args.size, args.angles
    g = make_geometry(n, A, cs)
    dev = torch.device("cuda", local)
    vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                     device=dev).data
    proj = torch.empty((A, n, n), dtype=torch.float32, device=dev)
    y = dense_stack((A, n, n), dev)                  # dense Atb input
    acc = torch.zeros((n, n, n), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    chunks = [(c, min(c + CHUNK, A)) for c in range(0, A, CHUNK)]
    tm = StepTimer(args.steps)

    def step(i):
        tm.mark(i, 0, stream)
        for c0, c1 in chunks:
            K.fwd_interp(vol, g, (c0, c1), (0, n), proj[c0:c1])
        tm.mark(i, 1, stream)
        K.fill(acc, 0.0)
        for c0, c1 in chunks:
            K.bwd_matched(y[c0:c1], g, (c0, c1), (0, n), acc)
        tm.mark(i, 2, stream)

    elapsed, clocks, launches = timed(args.steps, args.warmup, step, False,
                                      local, "nccl")
    t_ax, t_atb = tm.halves()
    upd = float(A) * n ** 3
    value = 2 * upd * args.steps / elapsed / 1e9
    bpu = bytes_per_update(n, n)
    if t_atb >= t_ax:
        kr = roofline("bwd_matched_kernel", t_atb / len(chunks),
                      upd / len(chunks), bpu)
    else:
        kr = roofline("fwd_mlayer_kernel", t_ax / len(chunks),
                      upd / len(chunks), bpu)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Shepp-Logan 3D phantom; dense standard-normal "
                "Atb input)",
        "config": {"workload": f"config 2: {n}^3 volume, {n}^2 detector, "
                   f"{A} views; interp Ax + matched Atb (dense input), "
                   f"{len(chunks)} launches of {CHUNK} views each",
                   "l2": "inputs > L2 (512 MiB volume, 360 MiB stacks)",
                   "parallelism": "1 GPU"},
        "ax_gups": upd / t_ax / 1e9,
        "atb_matched_gups": upd / t_atb / 1e9,
        "roofline": kr,
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if not args.no_extras:
        line.update(run_extras(args, cs, K, g, vol, y, dev))
    if not args.no_c3:
        line["config3_step"] = run_config3_single(args, local)
    return line


def c3_workload(args, world):
    return (f"config 3: {args.c3_size}^3 volume, {args.c3_size}^2 detector, "
            f"{args.c3_angles} views; step = one {args.c3_block}-view "
            f"OS-SART block (interp Ax of every slab + NCCL reduce-scatter "
            f"of the slab partials, weighted residual, all-gather, matched "
            f"Atb into every slab) over {world} rank(s)")


def c3_setup(args, rank, world, dev):
    """Config-3 state of one rank: its slab of the phantom, the block's
    measured projections (this rank's view shard; synthetic dense data),
    W = 1 (the step's arithmetic does not depend on W's values)."""
    import torch
    import paper_1905_03748_b200 as cs
    from paper_1905_03748_b200.sharded import ShardedOperators
    n = args.c3_size
    g = make_geometry(n, args.c3_angles, cs)
    ops = ShardedOperators(g, rank, world)
    z0, z1 = ops.slab
    x = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev,
                   slab_range=(z0, z1)).data
    return g, ops, x


def run_config3(args, rank, world, local, backend):
    """N > 1: config 3 slab/angle split (strong scaling of one block)."""
    import numpy as np
    import torch
    from paper_1905_03748_b200 import kernels as K

    dev = torch.device("cuda", local)
    g, ops, x = c3_setup(args, rank, world, dev)
    res = run_c3_steps(args, g, ops, x, dev, local, backend)
    res.update({
        "metric": METRIC, "unit": UNIT, "n_gpus": world,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (Shepp-Logan 3D phantom slabs; dense "
                "standard-normal measured projections)",
        "config": {"workload": c3_workload(args, world),
                   "l2": "inputs > L2 (volume slabs >= 4 GiB)",
                   "parallelism": f"slab x{world} / angle shard x{world}",
                   "backend": backend,
                   # peer: partial sums stored by the Ax kernels into the
                   # owners' memory, matched Atb reading the owners' views
                   # in place (peer.py); collective: NCCL reduce-scatter /
                   # all-gather per round (CS_EXCHANGE=nccl)
                   "exchange": ops.exchange_mode},
    })
    del np, K
    return res


def run_config3_single(args, local):
    """The config-3 block step on this one GPU (the N = 1 point of the
    scaling curve)."""
    import torch
    dev = torch.device("cuda", local)
    g, ops, x = c3_setup(args, 0, 1, dev)
    res = run_c3_steps(args, g, ops, x, dev, local, "nccl", steps=2,
                       warmup=1)
    res["config"] = {"workload": c3_workload(args, 1)}
    del x
    torch.cuda.empty_cache()
    from paper_1905_03748_b200 import kernels as K
    K.release_cache()
    return res


def run_c3_steps(args, g, ops, x, dev, local, backend, steps=None,
                 warmup=None):
    import torch
    from paper_1905_03748_b200 import kernels as K
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    det = g.detector
    nb = args.c3_block
    blocks = [(b0, b0 + nb) for b0 in range(0, args.c3_angles - nb + 1, nb)]
    s_lens = [ops.shard(b)[1] - ops.shard(b)[0] for b in blocks]
    m = max(s_lens)
    b_meas = dense_stack((m, det.n_v, det.n_u), dev, seed=1 + ops.rank)
    w = torch.ones_like(b_meas)
    res = torch.empty_like(b_meas)
    upd = torch.zeros_like(x)
    stream = torch.cuda.current_stream()
    tm = StepTimer(steps)
    counter = [0]

    def step(i):
        blk = blocks[counter[0] % len(blocks)]
        counter[0] += 1
        s0, s1 = ops.shard(blk)
        r = res[:s1 - s0]
        tm.mark(i, 0, stream)
        ops.forward_residual(x, b_meas[:s1 - s0], w[:s1 - s0], r, blk)
        tm.mark(i, 1, stream)
        ops.backward(r, upd, blk)
        tm.mark(i, 2, stream)

    dist_on = ops.world > 1
    elapsed, clocks, launches = timed(steps, warmup, step, dist_on, local,
                                      backend)
    t_ax, t_atb = tm.halves()
    n = g.voxel_grid.n_x
    upd_half = float(nb) * n ** 3            # whole volume, all ranks
    value = 2 * upd_half * steps / elapsed / 1e9
    out = {"value": value, "steps": steps, "warmup": max(3, warmup),
           "ms_per_step": 1e3 * elapsed / steps,
           "ax_gups": upd_half / t_ax / 1e9 if t_ax > 0 else None,
           "atb_matched_gups": upd_half / t_atb / 1e9 if t_atb > 0 else None,
           "ax_half_ms": t_ax * 1e3, "atb_half_ms": t_atb * 1e3,
           "clocks": clocks, "gpu_launches": launches,
           "roofline": roofline(
               "bwd_matched_kernel" if t_atb >= t_ax else "fwd_mlayer_kernel",
               max(t_atb, t_ax), upd_half / ops.world,
               bytes_per_update(n, n)),
           "e2e": c3_e2e(ops, x, b_meas, w, blocks, dev, backend,
                         upd=upd, res=res)}
    out["roofline"]["note"] = ("per-rank half-step (rank 0's share of the "
                               "block, incl. its collectives) as one launch")
    del K
    return out


def c3_e2e(ops, x, b_dev, w, blocks, dev, backend, reps=2, upd=None,
           res=None):
    """End to end per step through the public sharded API: the block's
    measured projections (this rank's shard) copied in from pinned host
    memory, the step, and the block's residual norm read back (the loop
    metric); slowest rank.  Reuses the device step's update and residual
    buffers: a second slab-sized update would take the memory the matched
    kernel's transposed frame needs (at N = 1 a 32 GiB volume) and time a
    different kernel path than the device step."""
    import torch
    import torch.distributed as dist
    from paper_1905_03748_b200.sharded import CudaVecOps
    m = b_dev.shape[0]
    host = torch.empty(b_dev.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(b_dev)
    b = torch.empty_like(b_dev)
    res = torch.empty_like(b_dev) if res is None else res
    upd = torch.zeros_like(x) if upd is None else upd
    blk = blocks[0]
    s0, s1 = ops.shard(blk)

    def step():
        b[:s1 - s0].copy_(host[:s1 - s0], non_blocking=True)
        r = res[:s1 - s0]
        ops.forward_residual(x, b[:s1 - s0], w[:s1 - s0], r, blk)
        nrm = ops.allreduce_(CudaVecOps.dot(r))
        ops.backward(r, upd, blk)
        return float(nrm.item())

    step()
    torch.cuda.synchronize()
    if ops.world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    if ops.world > 1:
        t = torch.tensor([dt], dtype=torch.float64,
                         device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    n = ops.geometry.voxel_grid.n_x
    upd_step = 2.0 * (blk[1] - blk[0]) * n ** 3
    return {"value": upd_step / dt / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": int((s1 - s0) * b_dev[0].numel() * 4),
            "d2h_bytes_per_step": 8, "ms_per_step": dt * 1e3,
            "api": "sharded.ShardedOperators forward_residual + backward; "
                   "block projections H2D from pinned host, residual norm "
                   "D2H", "scope": "rank 0's bytes; slowest rank's time"}


def run_extras(args, cs, K, g, vol, y, dev):
    """N = 1 extras: FDK and sparse-input matched Atb, TV, e2e through the
    public API, the loops (config 2 and config 1), the CPU baseline."""
    import numpy as np
    import torch
    out = {}
    n = g.voxel_grid.n_x
    A = g.n_angles
    peak, _ = measured_peak()
    acc = torch.zeros((n, n, n), dtype=torch.float32, device=dev)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)

    def rate(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1e-3 / reps

    upd = float(A) * n ** 3
    out["atb_fdk_gups"] = upd / rate(
        lambda: K.bwd_fdk(y, g, (0, A), (0, n), acc)) / 1e9
    # the sparse stack Ax(phantom): rays outside the head's shadow are zero
    # and skipped (the reference skips them too, _kernels.py:295-296)
    sparse = torch.empty_like(y)
    K.fwd_interp(vol, g, (0, A), (0, n), sparse)
    out["atb_matched_sparse_gups"] = upd / rate(
        lambda: K.bwd_matched(sparse, g, (0, A), (0, n), acc), 3) / 1e9
    del sparse
    # TV-GD iteration as the loops run it: in steady state one fused pass
    # per iteration (step i + gradient i+1 + Sigma g^2, tv.cu
    # tv_march_kernel); "tv_gd_run" times a whole 10-iteration
    # minimize_tv_gradient (gradient pass, 9 fused passes, final step, the
    # input copy).  ROF: one dual iteration.  512^3 volume; 12 /
    # 28 B per voxel-iteration algorithmic.
    from paper_1905_03748_b200 import regularization as REG
    u2 = torch.empty_like(vol)
    g2 = torch.empty_like(vol)
    g3 = torch.empty_like(vol)
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    ss2 = torch.zeros_like(ss)
    K.tv_grad_store(vol, g2, (0, n), ss)
    p3 = torch.zeros((3,) + tuple(vol.shape), device=dev)
    q3 = torch.empty_like(p3)
    for name, fn, bpv, its in (
            ("tv_gd", lambda: K.tv_gd_fused(vol, g2, u2, g3, (0, n), 1e-3,
                                            ss, 1.0, ss2), 12.0, 1),
            ("tv_gd_run", lambda: REG._gd_iterations(vol, 10, 1e-3), 12.0,
             10),
            ("tv_rof", lambda: K.rof_iter(vol, p3, q3, 0.1), 28.0, 1)):
        t = rate(fn, 5) / its
        out[f"{name}_gvox_iter_per_s"] = vol.numel() / t / 1e9
        out[f"{name}_hbm_frac"] = vol.numel() * bpv / t / (peak * 1e9)
    del u2, g2, g3, ss2, p3, q3, acc

    # end-to-end through the public API with pinned host buffers:
    # Ax(volume host) -> projections host; Atb(dense stack host) -> volume
    vol_h = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
    vol_h.copy_(vol)
    y_h = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
    y_h.copy_(y)
    vol_np, y_np = vol_h.numpy(), y_h.numpy()
    IP = cs.ProjectionMethod.INTERPOLATED

    def e2e_step():
        p = cs.forward_project_slab(cs.Volume(g.voxel_grid, vol_np), g,
                                    (0, A), IP)
        v = cs.backproject_slab(cs.ProjectionStack(g.detector, y_np, (0, A)),
                                g, (0, n), cs.WeightMode.MATCHED)
        return p, v
    # warm-up calls: results are held until the next call returns, so the
    # caching pinned-host allocator needs two sets of drain buffers before
    # it stops calling cudaHostAlloc, and the first reuse of a freed set is
    # still slow (tools/e2e_jitter.py: calls 0-2 slow, then steady), so
    # five calls reach the steady state of a user loop
    for _ in range(5):
        p, v = e2e_step()
    torch.cuda.synchronize()
    ne = 5
    iters = []
    t0 = time.perf_counter()
    for _ in range(ne):
        t1 = time.perf_counter()
        p, v = e2e_step()
        torch.cuda.synchronize()
        iters.append((time.perf_counter() - t1) * 1e3)
    dt = (time.perf_counter() - t0) / ne
    out["e2e"] = {"value": 2 * upd / dt / 1e9, "unit": "GUPS",
                  "h2d_bytes_per_step": int(vol_np.nbytes + y_np.nbytes),
                  "d2h_bytes_per_step": int(p.data.nbytes + v.data.nbytes),
                  "ms_per_step": dt * 1e3,
                  "iter_ms": [round(x, 1) for x in iters],
                  "api": "forward_project_slab + backproject_slab(MATCHED)"
                         " on host numpy (pinned), dense Atb input"}
    del vol_h, y_h

    # OS-SART s/iter (block 36, public API): (t(3 iters) - t(1 iter)) / 2
    # after a warm-up call (both include the same W / V set-up)
    pool = cs.DevicePool.b200(1)
    b = cs.ProjectionStack(g.detector, y)
    ts = {}
    for iters in (1, 1, 3):
        cfg = cs.ReconConfig(pool, cs.Algorithm.OSSART, iters, 36)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cs.os_sart(b, g, cfg)
        torch.cuda.synchronize()
        ts[iters] = time.perf_counter() - t0
    out["os_sart_s_per_iter"] = (ts[3] - ts[1]) / 2
    out["os_sart_setup_plus_1iter_s"] = ts[1]
    # SART-TV (SURVEY 8(d) C4 loop form: TV-GD 20 inner iterations,
    # ExactGlobal norm, after every OS-SART iteration) and the FDK
    # pipeline (cosine weight, ramp filter, FDK Atb) at config 2
    tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 20, 1e-3)
    for iters in (1, 1, 3):
        cfg = cs.ReconConfig(pool, cs.Algorithm.OSSART, iters, 36, tv=tv)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cs.os_sart(b, g, cfg)
        torch.cuda.synchronize()
        ts[iters] = time.perf_counter() - t0
    out["sart_tv_s_per_iter"] = (ts[3] - ts[1]) / 2
    for iters in (1, 1, 3):
        cfg = cs.ReconConfig(pool, cs.Algorithm.CGLS, iters)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cs.cgls(b, g, cfg)
        torch.cuda.synchronize()
        ts[iters] = time.perf_counter() - t0
    out["cgls_s_per_iter"] = (ts[3] - ts[1]) / 2
    cs.fdk(b, g, pool)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cs.fdk(b, g, pool)
    torch.cuda.synchronize()
    out["fdk_s"] = time.perf_counter() - t0

    # Config 1 loops end to end through the public API (host numpy in,
    # host numpy out), the reference's own timing case (BASELINE.md
    # section 2: SIRT 10 it 15.13 s, CGLS 10 it 15.66 s on 8 cores)
    g1 = make_geometry(64, 100, cs)
    x1 = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g1.voxel_grid).data
    b1 = cs.forward_project_slab(cs.Volume(g1.voxel_grid, x1), g1, (0, 100),
                                 cs.ProjectionMethod.INTERPOLATED)
    loops = {}
    for name, fn in (
            ("sirt_10it_s", lambda: cs.os_sart(b1, g1, cs.ReconConfig(
                pool, cs.Algorithm.OSSART, 10, 100))),
            ("cgls_10it_s", lambda: cs.cgls(b1, g1, cs.ReconConfig(
                pool, cs.Algorithm.CGLS, 10)))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        loops[name] = time.perf_counter() - t0
    out["config1_loops"] = {**loops, "api": "os_sart / cgls on host numpy, "
                            "64^3, 100 views (reference: SIRT 15.13 s, CGLS "
                            "15.66 s, 8 cores)"}

    from oracle import oracle as O
    threads = O.default_threads()
    x_np = vol.cpu().numpy()
    n_s = max(1, min(args.cpu_sample_angles, A))
    y_np = y[:n_s].cpu().numpy()
    cpu_oracle_sample(g, x_np, y_np, 1, threads)  # warm
    gups, dt, _ = cpu_oracle_sample(g, x_np, y_np, n_s, threads)
    out["cpu_baseline"] = {
        "value": gups, "unit": "GUPS", "cores": threads, "kind": "port",
        "sample": f"interp Ax + matched Atb (dense input) over a {n_s}-view "
                  f"window of config 2 ({dt:.1f} s; window outputs are exact "
                  "slices of the full scan)"}
    del np
    return out


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        sys.exit(run_reference(a))
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(a))
    sys.exit(run_ours(a))
