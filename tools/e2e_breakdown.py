"""Where the end-to-end (public API, host numpy in / out) time goes at
config 2: times each stage of forward_project_slab / backproject_slab.

    python tools/e2e_breakdown.py
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
from paper_1905_03748_b200.projectors import to_device, to_host

n, A = 512, 360
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
y = torch.empty((A, n, n), device=dev)
K.fwd_interp(vol, g, (0, A), (0, n), y)
vol_h = torch.empty(vol.shape, pin_memory=True)
vol_h.copy_(vol)
y_h = torch.empty(y.shape, pin_memory=True)
y_h.copy_(y)
vol_np, y_np = vol_h.numpy(), y_h.numpy()
IP = cs.ProjectionMethod.INTERPOLATED


def sync_t():
    torch.cuda.synchronize()
    return time.perf_counter()


out = {}
for rep in range(3):
    t0 = sync_t()
    vd = to_device(vol_np)
    t1 = sync_t()
    p = torch.empty((A, n, n), device=dev)
    K.fwd_interp(vd, g, (0, A), (0, n), p)
    t2 = sync_t()
    ph = to_host(p)
    t3 = sync_t()
    yd = to_device(y_np)
    t4 = sync_t()
    acc = torch.zeros((n, n, n), device=dev)
    K.bwd_matched(yd, g, (0, A), (0, n), acc)
    t5 = sync_t()
    vh = to_host(acc)
    t6 = sync_t()
    api0 = sync_t()
    cs.forward_project_slab(cs.Volume(g.voxel_grid, vol_np), g, (0, A), IP)
    api1 = sync_t()
    cs.backproject_slab(cs.ProjectionStack(g.detector, y_np), g, (0, n),
                        cs.WeightMode.MATCHED)
    api2 = sync_t()
    out = {"h2d_vol_ms": (t1 - t0) * 1e3, "fwd_ms": (t2 - t1) * 1e3,
           "d2h_proj_ms": (t3 - t2) * 1e3, "h2d_proj_ms": (t4 - t3) * 1e3,
           "bwd_ms": (t5 - t4) * 1e3, "d2h_vol_ms": (t6 - t5) * 1e3,
           "api_fwd_ms": (api1 - api0) * 1e3,
           "api_bwd_ms": (api2 - api1) * 1e3}
    print(json.dumps(out), flush=True)


# the bench's e2e loop, per-iteration times (public API, host numpy in/out)
def e2e_step():
    p = cs.forward_project_slab(cs.Volume(g.voxel_grid, vol_np), g, (0, A), IP)
    v = cs.backproject_slab(cs.ProjectionStack(g.detector, y_np), g, (0, n),
                            cs.WeightMode.MATCHED)
    return p, v


ts = []
for i in range(8):
    t0 = sync_t()
    p_, v_ = e2e_step()
    ts.append((sync_t() - t0) * 1e3)
print(json.dumps({"e2e_iter_ms": ts}), flush=True)
