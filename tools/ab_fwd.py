"""A/B of Ax implementations at config 2 (one process per variant, env
knobs are read once): times 4 x 90-view launches like bench.py and saves
the projections so variants can be compared bit for bit.

    python tools/ab_fwd.py TAG OUT.npy      (env selects the variant)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K

tag, path = sys.argv[1], sys.argv[2]
n = int(os.environ.get("PROF_N", 512))
A = int(os.environ.get("PROF_A", 360))
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
y = torch.empty((A, n, n), device=dev)


def run():
    for c in range(0, A, 90):
        K.fwd_interp(vol, g, (c, min(c + 90, A)), (0, n), y[c:c + 90])


run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
R = 3
s.record()
for _ in range(R):
    run()
e.record()
torch.cuda.synchronize()
t = s.elapsed_time(e) / R * 1e-3
# slab launch (accumulate mode, culled rows) for parity of the slab path
ys = torch.zeros((36, n, n), device=dev)
for z0, z1 in ((0, 100), (100, 300), (300, n)):
    K.fwd_interp(vol[z0:z1].contiguous(), g, (0, 36), (z0, z1), ys,
                 accumulate=z0 > 0)
np.save(path, y.cpu().numpy())
np.save(path.replace(".npy", "_slab.npy"), ys.cpu().numpy())
print(json.dumps({"tag": tag, "ms": t * 1e3, "gups": A * n ** 3 / t / 1e9}),
      flush=True)
