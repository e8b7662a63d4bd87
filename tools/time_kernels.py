"""Time each hot kernel at config 2 with CUDA events (avg of R after warm)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K

n = int(os.environ.get("PROF_N", 512))
A = int(os.environ.get("PROF_A", 360))
R = int(os.environ.get("PROF_R", 3))
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
y = torch.empty((A, n, n), device=dev)
K.fwd_interp(vol, g, (0, A), (0, n), y)
acc = torch.zeros((n, n, n), device=dev)
dense = torch.randn((A, n, n), device=dev, generator=torch.Generator(
    device=dev).manual_seed(1))
ops = {
    "fwd": lambda: K.fwd_interp(vol, g, (0, A), (0, n), y),
    "matched": lambda: K.bwd_matched(y, g, (0, A), (0, n), acc),
    "fdk": lambda: K.bwd_fdk(y, g, (0, A), (0, n), acc),
    "matched_dense": lambda: K.bwd_matched(dense, g, (0, A), (0, n), acc),
}
out = {}
for name, fn in ops.items():
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(R):
        fn()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / R * 1e-3
    out[name] = {"ms": t * 1e3, "gups": A * n ** 3 / t / 1e9}
print(json.dumps({"tag": os.environ.get("TAG", ""), **out}))
