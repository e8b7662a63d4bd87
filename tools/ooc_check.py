import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench, paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
A = int(sys.argv[2]) if len(sys.argv) > 2 else 32
budgets = [int(float(b) * 2**30) for b in sys.argv[3:]] or [1, 300 / 1024]
budgets = [b if b > 1000 else int(b) for b in budgets]
g = bench.make_geometry(n, A, cs)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=torch.device("cuda", 0)).data
y = torch.empty((A, n, n), device="cuda"); K.fwd_interp(vol, g, (0, A), (0, n), y)
vh = vol.cpu().numpy()
for budget in budgets:
    pool = cs.DevicePool((cs.DeviceSpec(memory_budget=budget, cuda_device=0),))
    plan = cs.plan_forward(g, pool)
    sink = []
    r = cs.execute_forward(cs.Volume(g.voxel_grid, vh), g, pool, plan, cs.ProjectionMethod.INTERPOLATED, trace_sink=sink)
    ref = y.cpu().numpy()
    num = den = 0.0
    mx = 0.0
    for a in range(A):
        d = r.data[a].astype(np.float64) - ref[a]
        num += float((d * d).sum()); den += float((ref[a].astype(np.float64) ** 2).sum()); mx = max(mx, float(np.abs(d).max()))
    print(budget, plan.n_splits, [e.payload for e in sink[0].events if e.kind == "TransferIn"][:12], "rel", (num / den) ** 0.5, "maxabs", mx, flush=True)
