#!/usr/bin/env python
"""Bench: cone-beam Ax / Atb GUPS on B200 (BASELINE.json metric).

One *step* = one pass of the loop hot path over config 2:
interpolated Ax over the rank's 360 angles of a 512^3 volume onto a 512^2
detector + matched (exact-adjoint) Atb of those angles -- the operator pair
every OS-SART / SIRT / CGLS iteration applies (algorithms.py:213-216,
:280-283).  Unit: voxel x angle updates.

Multi-GPU (torchrun, one rank per GPU): weak scaling -- the scan has 360 x
N angles; rank r projects its own 360 angles of the full volume (angle
split, scheduler.py:164-166) and backprojects the same 360 angles into a
whole-volume partial; one NCCL reduce-scatter sums the partials so rank r
ends with planes [512 r / N, 512 (r+1) / N) of the full Atb (the paper's
slab split of Atb avoids this reduction over PCIe; over NVLink 5 it is ~1
ms of a ~300 ms step, while thin slabs cost 35% efficiency at 8 ranks).
Per-rank work is fixed.  Inputs (512 MiB volume, >= 360 MiB stack) exceed
the 126 MB L2, so no flush is needed between steps.

Also reported: per-operator GUPS (Ax, matched Atb, FDK Atb), OS-SART s/iter
(block 36, rank 0 at N=1), the roofline of the dominant kernel, the CPU
oracle on a bounded sample, the end-to-end number through the public API
with host buffers, SM clocks during the timed region.

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
    return ap.parse_args()


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


def atb_slabs(n, world, rank, per_rank=4):
    """The rank's share of the volume for the slab-split Atb: with N > 1 the
    n planes are cut into per_rank * N equal blocks dealt round-robin
    (rank r owns blocks r, r + N, ...), so every rank's planes span the
    whole height and the work balances whatever the data (the phantom's
    sinogram has zero rays -- skipped, _kernels.py:295-296 -- mostly above
    and below the head, which made the central contiguous slab the slowest
    rank).  Atb is slab-partition invariant, so any partition
    is the same operator."""
    if world == 1:
        return [(0, n)]
    nb = per_rank * world
    while nb > 1 and n % nb:
        nb //= 2
    nb = max(nb, world)
    edges = [n * i // nb for i in range(nb + 1)]
    return [(edges[b], edges[b + 1]) for b in range(rank, nb, world)]


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


def cpu_oracle_sample(g, x_np, n_sample, threads):
    """Oracle (C port, all host threads) on an angle window: interpolated
    Ax + matched Atb.  Returns (GUPS, seconds, updates)."""
    import numpy as np
    from oracle import oracle as O
    og = O.OGeom(g.dso, g.dsd, g.angles, g.voxel_grid.n_x, g.voxel_grid.n_y,
                 g.voxel_grid.n_z, nu=g.detector.n_u, nv=g.detector.n_v,
                 pixel=g.detector.pixel_size)
    win = (0, n_sample)
    t0 = time.perf_counter()
    p = O.fwd_interp(x_np, og, win, threads=threads)
    O.bwd_matched(p, og, win, threads=threads)
    dt = time.perf_counter() - t0
    upd = 2.0 * n_sample * float(x_np.size)
    del np
    return upd / dt / 1e9, dt, upd


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
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback"


# --------------------------------------------------------------------------


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import numpy as np
    import paper_1905_03748_b200 as cs
    from oracle import oracle as O
    O.lib()
    g = make_geometry(args.size, args.angles, cs)
    x = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid).data
    threads = O.default_threads()
    n_s = max(1, min(args.cpu_sample_angles, args.angles))
    for _ in range(args.warmup):
        cpu_oracle_sample(g, x, n_s, threads)
    times = []
    upd = 0.0
    for _ in range(args.steps):
        _, dt, upd = cpu_oracle_sample(g, x, n_s, threads)
        times.append(dt)
    tot = sum(times)
    val = upd * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Shepp-Logan 3D phantom)",
        "config": {"workload": f"config 2: {args.size}^3 volume, "
                   f"{args.size}^2 detector, {args.angles} angles; "
                   "interp Ax + matched Atb", "sample": f"{n_s}-angle window"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads,
                         "kind": "port",
                         "sample": f"{n_s}-angle window of the "
                         f"{args.angles}-angle scan per step (outputs are "
                         "exact slices of the full run)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    del np
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1905_03748_b200 as cs
    from paper_1905_03748_b200 import kernels as K

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
    n, A1 = args.size, args.angles
    A = A1 * world
    g = make_geometry(n, A, cs)
    dev = torch.device("cuda", local)
    a0, a1 = rank * A1, (rank + 1) * A1       # angle split (Ax and Atb)
    z0, z1 = n * rank // world, n * (rank + 1) // world
    nz_s = z1 - z0
    if world > 1 and n % world:
        raise SystemExit(f"--size {n} must be divisible by --gpus {world}")

    vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                     device=dev).data
    proj = torch.empty((A1, n, n), dtype=torch.float32, device=dev)
    y = torch.empty((A1, n, n), dtype=torch.float32, device=dev)
    K.fwd_interp(vol, g, (a0, a1), (0, n), y)                # Atb input
    # N = 1: Atb straight into the volume.  N > 1: every rank backprojects
    # ITS views into a full-volume partial and the partials are summed by
    # one NCCL reduce-scatter, rank r keeping planes [z0, z1).  The paper
    # slab-splits Atb instead (Alg. 2) to avoid that reduction over PCIe;
    # over NVLink 5 the 512 MiB reduce-scatter costs ~1 ms against ~140 ms
    # of backprojection, while thin slabs cost 35% efficiency at 8 ranks
    # (per-(ray, slab) overheads; tools/rank_share.py).
    acc = torch.zeros((n, n, n), dtype=torch.float32, device=dev)
    slab = acc if world == 1 else torch.empty((nz_s, n, n),
                                              dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def reduce_scatter():
        if backend == "nccl":
            dist.reduce_scatter_tensor(slab, acc)
        else:  # gloo (several ranks sharing one GPU, testing only)
            host = acc.cpu()
            dist.all_reduce(host)
            slab.copy_(host[z0:z1])

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)]
          for _ in range(args.steps)]

    # angle chunks of CHUNK views per launch (the paper's chunked launches;
    # one ncu capture == one bench launch)
    ax_chunks = [(c, min(c + CHUNK, a1)) for c in range(a0, a1, CHUNK)]
    atb_chunks = ax_chunks

    def step(e=None):
        if e:
            e[0].record(stream)
        for c0, c1 in ax_chunks:
            K.fwd_interp(vol, g, (c0, c1), (0, n), proj[c0 - a0:c1 - a0])
        if e:
            e[1].record(stream)
        K.fill(acc, 0.0)
        for c0, c1 in atb_chunks:
            K.bwd_matched(y[c0 - a0:c1 - a0], g, (c0, c1), (0, n), acc)
        if world > 1:
            reduce_scatter()
        if e:
            e[2].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = K.launch_count()
    with Clocks(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            step(ev[i])
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = K.launch_count() - launches0  # this library's kernels
    elapsed = t_start.elapsed_time(t_end) * 1e-3
    t_ax = sum(e[0].elapsed_time(e[1]) for e in ev) * 1e-3 / args.steps
    t_atb = sum(e[1].elapsed_time(e[2]) for e in ev) * 1e-3 / args.steps
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64,
                         device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    upd_ax = float(A1) * n ** 3
    upd_atb = float(A1) * n ** 3  # the rank's views into the whole volume
    upd_step_rank = upd_ax + upd_atb
    total_upd = upd_step_rank * world * args.steps   # weak: equal per rank
    value = total_upd / elapsed / 1e9
    clocks = clk.summary()

    extras = {}
    if not args.no_extras:
        extras = run_extras(args, cs, K, g, vol, y, dev, rank, world,
                            (a0, a1), (z0, z1))

    # dominant kernel roofline (bytes per SURVEY 8(d))
    bpu = bytes_per_update(n, n)
    if t_atb >= t_ax:
        kname, kt, kupd = ("bwd_matched_kernel", t_atb / len(atb_chunks),
                           upd_atb / len(atb_chunks))
    else:
        # main-axis-layered Ax (z-layered only past the layer limit)
        kname = ("fwd_mlayer_kernel" if n <= 2048 else "fwd_interp_kernel")
        kname, kt, kupd = (kname, t_ax / len(ax_chunks),
                           upd_ax / len(ax_chunks))
    peak, peak_kind = measured_peak()
    achieved = kupd * bpu / kt / 1e9
    traffic = load_traffic(kname)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Shepp-Logan 3D phantom; Atb input = its Ax)",
        "config": {"workload": f"config 2 per GPU: {n}^3 volume, {n}^2 "
                   f"detector, {A1} angles/GPU (scan of {A}); interp Ax + "
                   "matched Atb of the GPU's angles"
                   + ("" if world == 1 else
                      ", Atb partials reduce-scattered (NCCL) to slabs"),
                   "l2": "inputs > L2 (512 MiB volume, 360+ MiB stack)",
                   "parallelism": f"angle split x{world}"},
        "ax_gups": upd_ax / t_ax / 1e9,
        "atb_matched_gups": upd_atb / t_atb / 1e9,
        "roofline": {"bound": "hbm", "kernel": kname,
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_kind,
                     "bytes_per_update": bpu,
                     "updates_per_launch": kupd,
                     "launch_ms": kt * 1e3,
                     # the pipe that actually bounds this gather kernel
                     # (ncu --set full, committed summary)
                     "ncu_pipes": load_limits(kname)},
        "clocks": clocks,
        "gpu_launches": launches,
    }
    line.update(extras)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    del np
    return 0


def run_extras(args, cs, K, g, vol, y, dev, rank, world, arange, zrange):
    """FDK Atb GUPS, OS-SART s/iter, e2e through the public API, CPU
    baseline (rank 0, N = 1)."""
    import numpy as np
    import torch
    out = {}
    n = g.voxel_grid.n_x
    # every rank: its own views (y) into the whole volume
    va0, va1 = arange
    A = va1 - va0
    zrange = (0, n)
    z0, z1 = zrange
    slab = torch.zeros((z1 - z0, n, n), dtype=torch.float32, device=dev)
    # FDK-weighted Atb
    for _ in range(2):
        K.bwd_fdk(y, g, (va0, va1), zrange, slab)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    reps = 3
    for _ in range(reps):
        K.bwd_fdk(y, g, (va0, va1), zrange, slab)
    e.record()
    torch.cuda.synchronize()
    out["atb_fdk_gups"] = reps * float(A) * (z1 - z0) * n * n / (
        s.elapsed_time(e) * 1e-3) / 1e9
    # matched Atb on a dense (no zero pixels) stack: the bench input Ax(phantom)
    # has zeros outside the head's shadow, which the reference skips too
    # (_kernels.py:295-296); a residual stack is dense
    dense = torch.randn(y.shape, device=dev, generator=torch.Generator(
        device=dev).manual_seed(1))
    K.bwd_matched(dense, g, (va0, va1), zrange, slab)
    torch.cuda.synchronize()
    s.record()
    K.bwd_matched(dense, g, (va0, va1), zrange, slab)
    e.record()
    torch.cuda.synchronize()
    out["atb_matched_dense_gups"] = float(A) * (z1 - z0) * n * n / (
        s.elapsed_time(e) * 1e-3) / 1e9
    del dense
    # TV-GD iteration as the loops run it (g + Sigma g^2 pass, streaming
    # step pass) and ROF dual iteration on the 512^3 volume (SURVEY 8(d):
    # 12 / 28 B per voxel-iteration algorithmic)
    u2 = torch.empty_like(vol)
    g2 = torch.empty_like(vol)
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    p3 = torch.zeros((3,) + tuple(vol.shape), device=dev)
    q3 = torch.empty_like(p3)
    for name, fn, bpv in (
            ("tv_gd", lambda: (K.tv_grad_store(vol, g2, (0, n), ss),
                               K.tv_step_g(vol, g2, u2, 1e-3, ss, 1.0)), 12.0),
            ("tv_rof", lambda: K.rof_iter(vol, p3, q3, 0.1), 28.0)):
        fn()
        torch.cuda.synchronize()
        s.record()
        for _ in range(5):
            fn()
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) * 1e-3 / 5
        out[f"{name}_gvox_iter_per_s"] = vol.numel() / t / 1e9
        out[f"{name}_hbm_frac"] = vol.numel() * bpv / t / 6550.7e9
    del u2, p3, q3

    # end-to-end through the public API with pinned host buffers:
    # Ax(volume host) -> projections host; Atb(projections host) -> slab host
    a0, a1 = arange
    vol_h = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
    vol_h.copy_(vol)
    y_h = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
    y_h.copy_(y)
    vol_np, y_np = vol_h.numpy(), y_h.numpy()
    IP = cs.ProjectionMethod.INTERPOLATED

    def e2e_step():
        p = cs.forward_project_slab(cs.Volume(g.voxel_grid, vol_np), g,
                                    (a0, a1), IP)
        v = cs.backproject_slab(cs.ProjectionStack(g.detector, y_np,
                                                   (va0, va1)), g,
                                zrange, cs.WeightMode.MATCHED)
        return p, v
    # warm-up calls: results are held until the next call returns, so the
    # caching pinned-host allocator needs two sets of drain buffers before
    # it stops calling cudaHostAlloc (steady state of a user loop)
    for _ in range(3):
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
    if world > 1:
        # whole-job aggregate: every rank does equal work; slowest rank
        import torch.distributed as dist
        on_dev = os.environ.get("CS_BENCH_BACKEND", "nccl") == "nccl"
        tt = torch.tensor([dt], dtype=torch.float64,
                          device=dev if on_dev else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    upd = (float(a1 - a0) * n ** 3 + float(A) * (z1 - z0) * n * n) * world
    out["e2e"] = {"value": upd / dt / 1e9, "unit": "GUPS",
                  "h2d_bytes_per_step": int(vol_np.nbytes + y_np.nbytes),
                  "d2h_bytes_per_step": int(p.data.nbytes + v.data.nbytes),
                  "ms_per_step": dt * 1e3,
                  "iter_ms": [round(x, 1) for x in iters],
                  "scope": f"all {world} rank(s); slowest rank's time",
                  "api": "forward_project_slab + backproject_slab(MATCHED)"
                         " on host numpy (pinned)"}
    del vol_h, y_h

    if world == 1:
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
        for iters in (1, 1, 2):
            cfg = cs.ReconConfig(pool, cs.Algorithm.OSSART, iters, 36, tv=tv)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cs.os_sart(b, g, cfg)
            torch.cuda.synchronize()
            ts[iters] = time.perf_counter() - t0
        out["sart_tv_s_per_iter"] = ts[2] - ts[1]
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
        b1 = cs.forward_project_slab(cs.Volume(g1.voxel_grid, x1), g1,
                                     (0, 100),
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
        out["config1_loops"] = {**loops, "api": "os_sart / cgls on host "
                                "numpy, 64^3, 100 views (reference: SIRT "
                                "15.13 s, CGLS 15.66 s, 8 cores)"}

        from oracle import oracle as O
        threads = O.default_threads()
        x_np = vol.cpu().numpy()
        n_s = max(1, min(args.cpu_sample_angles, A))
        cpu_oracle_sample(g, x_np, 1, threads)  # warm
        gups, dt, upd = cpu_oracle_sample(g, x_np, n_s, threads)
        out["cpu_baseline"] = {
            "value": gups, "unit": "GUPS", "cores": threads, "kind": "port",
            "sample": f"interp Ax + matched Atb over a {n_s}-angle window of "
                      f"config 2 ({dt:.1f} s; window outputs are exact "
                      "slices of the full scan)"}
    del np
    return out


if __name__ == "__main__":
    a = parse()
    sys.exit(run_reference(a) if a.impl == "reference" else run_ours(a))
