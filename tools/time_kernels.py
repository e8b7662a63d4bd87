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
    "siddon": lambda: K.fwd_siddon(vol, g, (0, A), (0, n), y),
}
only = os.environ.get("PROF_ONLY")
TVOPS = ("tv_gd_iter", "rof_iter", "tv_grad", "tv_fused", "tv_step",
         "tv_run10")
if not only or any(k in only for k in TVOPS):
    from paper_1905_03748_b200 import regularization as REG
    u2 = torch.empty_like(vol)
    g2 = torch.empty_like(vol)
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    ss2 = torch.zeros(1, dtype=torch.float64, device=dev)
    g3 = torch.empty_like(vol)
    p3 = torch.zeros((3, n, n, n), device=dev)
    q3 = torch.empty_like(p3)

    def tv_gd():
        K.tv_grad_store(vol, g2, (0, n), ss)
        K.tv_step_g(vol, g2, u2, 1e-3, ss, 1.0)

    ops["tv_gd_iter"] = tv_gd
    ops["tv_grad"] = lambda: K.tv_grad_store(vol, g2, (0, n), ss)
    ops["tv_fused"] = lambda: K.tv_gd_fused(vol, g2, u2, g3, (0, n), 1e-3,
                                            ss, 1.0, ss2)
    ops["tv_step"] = lambda: K.tv_step_g(vol, g2, u2, 1e-3, ss, 1.0)
    ops["tv_run10"] = lambda: REG._gd_iterations(vol, 10, 1e-3)
    ops["rof_iter"] = lambda: K.rof_iter(vol, p3, q3, 0.1)
if only:
    ops = {k: v for k, v in ops.items() if k in only.split(",")}
out = {}
for name, fn in ops.items():
    for _ in range(3 if name in TVOPS else 1):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    reps = R * 10 if name in TVOPS else R
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / reps * 1e-3
    if name in TVOPS:
        its = 10 if name == "tv_run10" else 1
        bpv = 28.0 if name == "rof_iter" else 12.0
        t /= its
        out[name] = {"ms": t * 1e3, "gvox_per_s": n ** 3 / t / 1e9,
                     "frac_hbm": n ** 3 * bpv / t / (bench.measured_peak()[0] * 1e9)}
    else:
        out[name] = {"ms": t * 1e3, "gups": A * n ** 3 / t / 1e9}
print(json.dumps({"tag": os.environ.get("TAG", ""), **out}))
