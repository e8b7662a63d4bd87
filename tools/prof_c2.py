"""Run each hot kernel at config 2 (512^3, 512^2, 360 angles) twice (warm
+ profiled) for ncu: fwd_interp, bwd_matched, bwd_fdk, tv step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K

n = int(os.environ.get("PROF_N", 512))
A = int(os.environ.get("PROF_A", 360))
which = os.environ.get("PROF_KERNELS", "fwd,matched,fdk").split(",")
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
y = torch.empty((A, n, n), device=dev)
K.fwd_interp(vol, g, (0, A), (0, n), y)
acc = torch.zeros((n, n, n), device=dev)
for rep in range(2):
    if "fwd" in which:
        K.fwd_interp(vol, g, (0, A), (0, n), y)
    if "matched" in which:
        K.bwd_matched(y, g, (0, A), (0, n), acc)
    if "fdk" in which:
        K.bwd_fdk(y, g, (0, A), (0, n), acc)
torch.cuda.synchronize()
print("done")
