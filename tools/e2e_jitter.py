"""Per-iteration split of the bench's e2e step (public API on pinned host
numpy) into forward_project_slab / backproject_slab wall times, with the
pinned host allocator's counters, to locate host-side jitter.

    python tools/e2e_jitter.py
"""
import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K

n, A = 512, 360
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
y = torch.randn((A, n, n), device=dev,
                generator=torch.Generator(device=dev).manual_seed(1))
vol_h = torch.empty(vol.shape, pin_memory=True)
vol_h.copy_(vol)
y_h = torch.empty(y.shape, pin_memory=True)
y_h.copy_(y)
vol_np, y_np = vol_h.numpy(), y_h.numpy()
IP = cs.ProjectionMethod.INTERPOLATED
gc_mode = os.environ.get("JIT_GC", "on")
if gc_mode == "off":
    gc.disable()


def stats():
    try:
        s = torch.cuda.host_memory_stats()
        return {k: s[k] for k in ("num_host_alloc", "num_host_free")
                if k in s}
    except Exception:  # noqa: BLE001
        return {}


p = v = None
for i in range(14):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p_ = cs.forward_project_slab(cs.Volume(g.voxel_grid, vol_np), g, (0, A),
                                 IP)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    v_ = cs.backproject_slab(cs.ProjectionStack(g.detector, y_np), g, (0, n),
                             cs.WeightMode.MATCHED)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    p, v = p_, v_
    del p_, v_
    t3 = time.perf_counter()
    print(json.dumps({"it": i, "gc": gc_mode, "fwd_ms": round((t1 - t0) * 1e3, 1),
                      "bwd_ms": round((t2 - t1) * 1e3, 1),
                      "release_ms": round((t3 - t2) * 1e3, 1), **stats()}),
          flush=True)
