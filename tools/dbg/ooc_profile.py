"""cProfile of the out-of-core SART-TV loop (forced small device budget):
where the host-side time goes.  python tools/dbg/ooc_profile.py [n] [budget_gib]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))))
import torch

import bench
import paper_1905_03748_b200 as cs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
bud = float(sys.argv[2]) if len(sys.argv) > 2 else 1.5
A = 64
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
x_true = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
b = cs.forward_project_slab(cs.Volume(g.voxel_grid, x_true), g, (0, A),
                            cs.ProjectionMethod.INTERPOLATED).data.cpu().numpy()
del x_true
torch.cuda.empty_cache()
small = cs.DevicePool((cs.DeviceSpec(memory_budget=int(bud * 2 ** 30),
                                     cuda_device=0),))
tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 8, 1e-3)
stack = cs.ProjectionStack(g.detector, b)
cfg = cs.ReconConfig(small, cs.Algorithm.OSSART, 2, 16, tv=tv)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
cs.os_sart(stack, g, cfg)
torch.cuda.synchronize()
pr.disable()
print(f"total {time.perf_counter() - t0:.2f} s", flush=True)
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
st.sort_stats("tottime").print_stats(25)
