"""Config-3 block step at N = 1: device-timed pieces of the bench's
device step vs its e2e step (tools for the e2e gap), with free memory.

    python tools/c3_e2e_diag.py
"""
import json
import os
import sys
import time
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1905_03748_b200.sharded import CudaVecOps

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
args = SimpleNamespace(c3_size=2048, c3_angles=1024, c3_block=64)
g, ops, x = bench.c3_setup(args, 0, 1, dev)
det = g.detector
blk = (0, 64)
b = bench.dense_stack((64, det.n_v, det.n_u), dev, seed=1)
w = torch.ones_like(b)
res = torch.empty_like(b)
upd = torch.zeros_like(x)
host = torch.empty(b.shape, dtype=torch.float32, pin_memory=True)
host.copy_(b)


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3, out


for it in range(4):
    f, total = torch.cuda.mem_get_info()
    r = {"it": it, "free_gib": round(f / 2**30, 1)}
    r["h2d_ms"], _ = t(lambda: b.copy_(host, non_blocking=True))
    r["fwd_res_ms"], _ = t(lambda: ops.forward_residual(x, b, w, res, blk))
    r["dot_ms"], nrm = t(lambda: ops.allreduce_(CudaVecOps.dot(res)))
    r["bwd_ms"], _ = t(lambda: ops.backward(res, upd, blk))
    r["item_ms"], _ = t(lambda: float(nrm.item()))
    print(json.dumps(r), flush=True)
