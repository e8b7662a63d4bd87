"""Large-configuration measurements on ONE B200 (not the bench contract):

* ``c3``: the per-rank work of config 3 (2048^3 volume, 2048^2 detector,
  1024 views) at N GPUs under bench.py's decomposition -- interp Ax and
  matched Atb of the rank's 1024/N views over the whole volume, plus the
  reduce-scatter payload of the Atb partials (costed at 700 GB/s, the
  measured NVLink all-reduce bus bandwidth).
* ``ooc``: out-of-core streaming through execute_forward / execute_backward
  with a device budget below the volume size (slabs streamed H2D from
  page-locked host memory, Algorithm 1/2), against the same operators
  in-core.

* ``c5``: config 5 scale on ONE GPU without ever materialising the volume:
  a 4096^3 Shepp-Logan (256 GiB, > one B200's HBM) is generated slab by
  slab on the device, projected slab by slab with the partial projections
  accumulated in the kernel epilogue (Algorithm 1), then backprojected
  slab by slab (Algorithm 2) while the adjoint identity <A x, y> =
  <x, A^T y> is accumulated across slabs in fp64 -- a full-scale
  consistency check of both operators at 4096^3.

    python tools/bench_scale.py c3 [N=8] [views=1024]
    python tools/bench_scale.py c5 [n=4096] [views=32] [slab=256]
    python tools/bench_scale.py ooc [n=2048] [views=64] [budget_gib=12]
    python tools/bench_scale.py c4 [n=1024] [views=1024] [iters=2] [block=32]
    python tools/bench_scale.py oocloops [n=1536] [views=64] [budget_gib=6] [iters=3]

* ``oocloops``: BASELINE config 5's mechanism (a volume larger than the device
  budget reconstructed through slab streaming) with the loops themselves:
  CGLS and SART-TV on host float32 vectors with every operator pass planned
  and slab-streamed under a forced device budget, against the same loops
  in-core on the device (the volume fits a B200's HBM, so both run here).

Prints one JSON line per measurement.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e-3 / reps


def c3(N=8, A=1024, n=2048, rank=None):
    """Rank r's work at N ranks under bench.py's decomposition: interp Ax
    and matched Atb of its A/N views over the whole volume (Atb input: a
    dense stack, 1 + the phantom's sinogram), plus the reduce-scatter
    payload it would send (7/8 of the volume at N = 8)."""
    dev = torch.device("cuda", 0)
    rank = N // 2 if rank is None else rank
    g = bench.make_geometry(n, A, cs)
    vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                     device=dev).data
    a0, a1 = A * rank // N, A * (rank + 1) // N
    proj = torch.empty((a1 - a0, n, n), device=dev)
    chunk = 64
    t_ax = timed(lambda: [K.fwd_interp(vol, g, (c, min(c + chunk, a1)),
                                       (0, n), proj[c - a0:min(c + chunk, a1) - a0])
                          for c in range(a0, a1, chunk)])
    ax_upd = float(a1 - a0) * n ** 3
    y = proj.clone()
    y += 1.0  # dense: no zero pixels (the matched adjoint skips zeros)
    acc = torch.zeros((n, n, n), device=dev)
    del vol
    torch.cuda.empty_cache()

    def atb():
        for c in range(a0, a1, chunk):
            K.bwd_matched(y[c - a0:min(c + chunk, a1) - a0], g,
                          (c, min(c + chunk, a1)), (0, n), acc)
    t_atb = timed(atb)
    atb_upd = float(a1 - a0) * n ** 3
    rs_bytes = (N - 1) / N * n ** 3 * 4
    out = {"measure": "c3_rank_share", "N": N, "rank": rank, "n": n,
           "views": A, "views_per_rank": a1 - a0,
           "ax_gups": ax_upd / t_ax / 1e9, "ax_s": t_ax,
           "atb_matched_gups": atb_upd / t_atb / 1e9, "atb_s": t_atb,
           "reduce_scatter_bytes": rs_bytes,
           "reduce_scatter_s_at_700GBps": rs_bytes / 700e9,
           "step_gups_per_rank": (ax_upd + atb_upd) / (t_ax + t_atb) / 1e9}
    out["projected_N_gpu_gups"] = N * (ax_upd + atb_upd) / (
        t_ax + t_atb + rs_bytes / 700e9) / 1e9
    print(json.dumps(out), flush=True)


def ooc(n=2048, A=64, budget_gib=12.0):
    import numpy as np
    dev = torch.device("cuda", 0)
    g = bench.make_geometry(n, A, cs)
    vol_d = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                       device=dev).data
    IP = cs.ProjectionMethod.INTERPOLATED
    # in-core reference timings (device-resident operators)
    y_d = torch.empty((A, n, n), device=dev)
    t_fwd_in = timed(lambda: K.fwd_interp(vol_d, g, (0, A), (0, n), y_d))
    acc = torch.zeros_like(vol_d)
    t_bwd_in = timed(lambda: K.bwd_matched(y_d, g, (0, A), (0, n), acc))
    ref_f = y_d.cpu()
    ref_b = None
    acc.zero_()
    K.bwd_matched(y_d, g, (0, A), (0, n), acc)
    ref_b = acc.cpu()
    # host images (page-locked by the executor per plan.pin_host_image)
    vol_h = vol_d.cpu().numpy()
    y_h = ref_f.numpy()
    del acc, vol_d, y_d
    torch.cuda.empty_cache()
    pool = cs.DevicePool((cs.DeviceSpec(memory_budget=int(budget_gib * 2 ** 30),
                                        cuda_device=0),))
    fplan, bplan = cs.plan_forward(g, pool), cs.plan_backward(g, pool)
    vol = cs.Volume(g.voxel_grid, vol_h)
    stack = cs.ProjectionStack(g.detector, y_h)
    res = {}
    for name, fn in (
            ("fwd", lambda sink: cs.execute_forward(vol, g, pool, fplan, IP,
                                                    trace_sink=sink)),
            ("bwd", lambda sink: cs.execute_backward(
                stack, g, pool, bplan, cs.WeightMode.MATCHED,
                trace_sink=sink))):
        fn(None)
        torch.cuda.synchronize()
        sink = []
        t0 = time.perf_counter()
        r = fn(sink)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tr = sink[0]
        ker = sum(e.end - e.start for e in tr.events
                  if e.kind in ("Kernel", "Accumulate"))
        h2d = sum(e.bytes for e in tr.events if e.kind == "TransferIn")
        d2h = sum(e.bytes for e in tr.events if e.kind == "TransferOut")
        pin_s = sum(e.end - e.start for e in tr.events
                    if e.kind in ("Pin", "Unpin"))
        ref = (ref_f if name == "fwd" else ref_b).numpy()
        got = np.asarray(r.data)
        num = den = 0.0
        for z in range(0, ref.shape[0], 64):   # bounded host memory
            d = got[z:z + 64].astype(np.float64) - ref[z:z + 64]
            num += float((d * d).sum())
            den += float((ref[z:z + 64].astype(np.float64) ** 2).sum())
        rel = (num / den) ** 0.5
        del r, got
        res[name] = {"wall_s": dt, "kernel_s": ker, "pin_unpin_s": pin_s,
                     "in_core_s": t_fwd_in if name == "fwd" else t_bwd_in,
                     "gups": A * float(n) ** 3 / dt / 1e9,
                     "h2d_gib": h2d / 2 ** 30, "d2h_gib": d2h / 2 ** 30,
                     "n_splits": (fplan if name == "fwd" else bplan).n_splits,
                     "high_water_gib": max(tr.high_water.values()) / 2 ** 30,
                     "rel_l2_vs_in_core": rel}
    print(json.dumps({"measure": "out_of_core", "n": n, "views": A,
                      "budget_gib": budget_gib,
                      "volume_gib": n ** 3 * 4 / 2 ** 30, **res}), flush=True)


def _phantom_slab(g, z0, z1, dev):
    """Shepp-Logan values of planes [z0, z1) of g's grid (fp32 on the
    device; the same formula as paper_1905_03748_b200.phantoms)."""
    from paper_1905_03748_b200.phantoms import SHEPP_LOGAN_ELLIPSOIDS
    import math
    grid = g.voxel_grid
    ex, ey, ez = grid.extent
    vx, vy, vz = grid.voxel_size

    def centres(a, b, v, e):
        return ((torch.arange(a, b, dtype=torch.float64, device=dev) + 0.5)
                * v - 0.5 * e) / (0.5 * e)
    x = centres(0, grid.n_x, vx, ex).float()[None, None, :]
    y = centres(0, grid.n_y, vy, ey).float()[None, :, None]
    z = centres(z0, z1, vz, ez).float()[:, None, None]
    out = torch.zeros((z1 - z0, grid.n_y, grid.n_x), device=dev)
    for value, a, b, c, x0, y0, zc, phi_deg in SHEPP_LOGAN_ELLIPSOIDS:
        zz = ((z - zc) / c) ** 2
        if float(zz.min()) > 1.0:
            continue
        phi = math.radians(phi_deg)
        cp, sp = math.cos(phi), math.sin(phi)
        xr = (x - x0) * cp + (y - y0) * sp
        yr = -(x - x0) * sp + (y - y0) * cp
        out += value * (((xr / a) ** 2 + (yr / b) ** 2 + zz) <= 1.0)
    return out


def c5(n=4096, A=32, slab=256):
    dev = torch.device("cuda", 0)
    g = bench.make_geometry(n, A, cs)
    slabs = [(z, min(z + slab, n)) for z in range(0, n, slab)]
    proj = torch.empty((A, n, n), device=dev)
    torch.cuda.synchronize()
    t_gen = t_fwd = t_bwd = 0.0
    for si, (z0, z1) in enumerate(slabs):
        t0 = time.perf_counter()
        xs = _phantom_slab(g, z0, z1, dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        K.fwd_interp(xs, g, (0, A), (z0, z1), proj, accumulate=si > 0)
        torch.cuda.synchronize()
        t_fwd += time.perf_counter() - t1
        t_gen += t1 - t0
        del xs
    # y = a dense stack (no zero pixels); <A x, y> in fp64
    y = proj + 1.0
    lhs = sum(float((proj[a].double() * y[a].double()).sum())
              for a in range(A))
    rhs = 0.0
    acc = torch.empty((slab, n, n), device=dev)
    for z0, z1 in slabs:
        xs = _phantom_slab(g, z0, z1, dev)
        a_ = acc[:z1 - z0]
        a_.zero_()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        K.bwd_matched(y, g, (0, A), (z0, z1), a_)
        torch.cuda.synchronize()
        t_bwd += time.perf_counter() - t1
        rhs += sum(float((xs[k].double() * a_[k].double()).sum())
                   for k in range(z1 - z0))
        del xs
    upd = float(A) * n ** 3
    print(json.dumps({
        "measure": "c5_slab_streamed", "n": n, "views": A,
        "volume_gib": n ** 3 * 4 / 2 ** 30, "slab_planes": slab,
        "slabs": len(slabs), "ax_s": t_fwd, "ax_gups": upd / t_fwd / 1e9,
        "atb_matched_s": t_bwd, "atb_matched_gups": upd / t_bwd / 1e9,
        "phantom_gen_s": t_gen, "adjoint_lhs": lhs, "adjoint_rhs": rhs,
        "adjoint_rel_diff": abs(lhs - rhs) / abs(lhs)}), flush=True)


def c4(n=1024, A=1024, iters=2, block=32):
    """Config 4 loops on one GPU, in-core: SART-TV (OS-SART block `block`
    + TvParams(GD, inner 20, step 1e-3, ExactGlobal)) and CGLS on the
    Shepp-Logan sinogram of a 1024^3 volume x 1024 views of a 1024^2
    detector, device-resident inputs; seconds per
    iteration (after a setup+1-iteration run) and the residuals."""
    dev = torch.device("cuda", 0)
    g = bench.make_geometry(n, A, cs)
    x_true = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                        device=dev).data
    b = cs.forward_project_slab(cs.Volume(g.voxel_grid, x_true), g, (0, A),
                                cs.ProjectionMethod.INTERPOLATED)
    pool = cs.DevicePool.b200(1)
    tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 20, 1e-3)

    def resid(v):
        ax = cs.forward_project_slab(cs.Volume(g.voxel_grid, v), g, (0, A),
                                     cs.ProjectionMethod.INTERPOLATED).data
        return float((ax - b.data).double().norm() / b.data.double().norm())

    out = {"measure": "c4_loops", "n": n, "views": A, "block": block}
    for name, fn in (
            ("sart_tv", lambda it: cs.os_sart(b, g, cs.ReconConfig(
                pool, cs.Algorithm.OSSART, it, block, tv=tv)).data),
            ("cgls", lambda it: cs.cgls(b, g, cs.ReconConfig(
                pool, cs.Algorithm.CGLS, it)).volume.data)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(1)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        x = fn(1 + iters)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out[name] = {"s_per_iter": (t2 - t1 - (t1 - t0)) / iters,
                     "setup_plus_1iter_s": t1 - t0,
                     "rel_residual_after": resid(x)}
        del x
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


def oocloops(n=1536, A=64, budget_gib=6.0, iters=3):
    """Out-of-core CGLS / SART-TV (forced budget) vs in-core on one GPU."""
    import numpy as np
    g = bench.make_geometry(n, A, cs)
    dev = torch.device("cuda", 0)
    x_true = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid,
                        device=dev).data
    b_d = cs.forward_project_slab(cs.Volume(g.voxel_grid, x_true), g, (0, A),
                                  cs.ProjectionMethod.INTERPOLATED).data
    del x_true
    b_h = b_d.cpu().numpy()
    del b_d
    torch.cuda.empty_cache()
    big = cs.DevicePool.b200(1)
    small = cs.DevicePool((cs.DeviceSpec(
        memory_budget=int(budget_gib * 2 ** 30), cuda_device=0),))
    fplan, bplan = cs.plan_forward(g, small), cs.plan_backward(g, small)
    tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 8, 1e-3)
    out = {"measure": "ooc_loops", "n": n, "views": A, "iters": iters,
           "budget_gib": budget_gib, "volume_gib": n ** 3 * 4 / 2 ** 30,
           "fwd_splits": fplan.n_splits, "bwd_splits": bplan.n_splits}

    def rel(a, b):
        num = den = 0.0
        for z in range(0, b.shape[0], 64):
            d = a[z:z + 64].astype(np.float64) - b[z:z + 64]
            num += float((d * d).sum())
            den += float((b[z:z + 64].astype(np.float64) ** 2).sum())
        return (num / den) ** 0.5

    stack = cs.ProjectionStack(g.detector, b_h)
    for name, run in (
            ("cgls", lambda pool: cs.cgls(stack, g, cs.ReconConfig(
                pool, cs.Algorithm.CGLS, iters))),
            ("sart_tv", lambda pool: cs.os_sart(stack, g, cs.ReconConfig(
                pool, cs.Algorithm.OSSART, iters, 16, tv=tv)))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r_in = run(big)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        x_in = np.asarray((r_in.volume if name == "cgls" else r_in).data)
        res_in = list(r_in.residuals) if name == "cgls" else None
        del r_in
        torch.cuda.empty_cache()
        t2 = time.perf_counter()
        r_out = run(small)
        t3 = time.perf_counter()
        x_out = np.asarray((r_out.volume if name == "cgls" else r_out).data)
        ent = {"in_core_s": t1 - t0, "out_of_core_s": t3 - t2,
               "rel_l2_vs_in_core": rel(x_out, x_in)}
        if name == "cgls":
            ent["residuals_in"] = res_in
            ent["residuals_out"] = list(r_out.residuals)
        out[name] = ent
        del r_out, x_in, x_out
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    what = sys.argv[1]
    args = [float(a) for a in sys.argv[2:]]
    if what == "c3":
        c3(*[int(a) for a in args])
    elif what == "c5":
        c5(*[int(a) for a in args])
    elif what == "c4":
        c4(*[int(a) for a in args])
    elif what == "oocloops":
        oocloops(*([int(a) for a in args[:2]] + args[2:3] +
                   [int(a) for a in args[3:4]]))
    else:
        ooc(*([int(args[0])] if args else []) + ([int(args[1])] if len(args) > 1 else []) + (args[2:3]))
