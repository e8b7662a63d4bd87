"""Replays the bench's launches at config 2 (512^3, 512^2, 360 views) for
ncu: each hot kernel launched on its first CHUNK-view chunk exactly as
bench.py launches it (warm-up launch first, then the profiled one)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K

n = int(os.environ.get("PROF_N", bench.N_VOX))
A = int(os.environ.get("PROF_A", bench.N_ANG))
C = int(os.environ.get("PROF_CHUNK", bench.CHUNK))
which = os.environ.get("PROF_KERNELS", "fwd,matched,fdk").split(",")
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
y = torch.empty((A, n, n), device=dev)
K.fwd_interp(vol, g, (0, A), (0, n), y)
# the bench's matched input: a dense standard-normal stack (bench.py)
dense = torch.randn((C, n, n), device=dev, generator=torch.Generator(
    device=dev).manual_seed(1))
acc = torch.zeros((n, n, n), device=dev)
proj = torch.empty((C, n, n), device=dev)
u2 = torch.empty_like(vol)
g2 = torch.empty_like(vol)
ss = torch.zeros(1, dtype=torch.float64, device=dev)
ss2 = torch.zeros(1, dtype=torch.float64, device=dev)
g3 = torch.empty_like(vol)
p3 = torch.zeros((3, n, n, n), device=dev)
q3 = torch.empty_like(p3)
torch.cuda.synchronize()
for rep in range(2):
    if "tv" in which:  # GD: gradient pass, fused pass; ROF: dual iteration
        K.tv_grad_store(vol, g2, (0, n), ss)
        K.tv_gd_fused(vol, g2, u2, g3, (0, n), 1e-3, ss, 1.0, ss2)
        K.rof_iter(vol, p3, q3, 0.1)
    if "fwd" in which:
        K.fwd_interp(vol, g, (0, C), (0, n), proj)
    if "matched" in which:
        K.bwd_matched(dense, g, (0, C), (0, n), acc)
    if "fdk" in which:
        K.bwd_fdk(y[0:C], g, (0, C), (0, n), acc)
    if "siddon" in which:
        K.fwd_siddon(vol, g, (0, C), (0, n), proj)
torch.cuda.synchronize()
print("done")
