import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench, paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K
n, A = 512, 32
g = bench.make_geometry(n, A, cs)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=torch.device("cuda", 0)).data
y = torch.empty((A, n, n), device="cuda"); K.fwd_interp(vol, g, (0, A), (0, n), y)
vh = vol.cpu().numpy()
for budget in (2**30, 300 * 2**20):
    pool = cs.DevicePool((cs.DeviceSpec(memory_budget=budget, cuda_device=0),))
    plan = cs.plan_forward(g, pool)
    sink = []
    r = cs.execute_forward(cs.Volume(g.voxel_grid, vh), g, pool, plan, cs.ProjectionMethod.INTERPOLATED, trace_sink=sink)
    d = r.data.astype(np.float64) - y.cpu().numpy()
    print(budget, plan.n_splits, [e.payload for e in sink[0].events if e.kind == "TransferIn"][:10], "rel", np.linalg.norm(d) / np.linalg.norm(y.cpu().numpy()), "maxabs", np.abs(d).max())
