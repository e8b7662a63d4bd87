"""Siddon DDA A/B: config-2 timing and output difference between two library
builds (CS_LIB_PATH in the environment selects one; run twice)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K
n, A = 512, 360
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
y = torch.empty((A, n, n), device=dev)
run = lambda: [K.fwd_siddon(vol, g, (c, c + 90), (0, n), y[c:c + 90]) for c in range(0, A, 90)]
run(); torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); [run() for _ in range(3)]; e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e) / 3e3
np.save(sys.argv[2], y[::9].cpu().numpy())
print(json.dumps({"tag": sys.argv[1], "siddon_gups": A * n ** 3 / t / 1e9, "ms": t * 1e3}))
