"""Per-rank work of bench.py at N ranks, on one GPU without contention:
interp Ax of the rank's 360 views of the full volume + matched Atb of all
360 N views into the rank's 512/N-plane slab (the bench's phantom-sinogram
input), against the N = 1 step.

    python tools/rank_share.py N [rank]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K

N = int(sys.argv[1])
rank = int(sys.argv[2]) if len(sys.argv) > 2 else N // 2
inter = len(sys.argv) > 3 and sys.argv[3] == "interleave"
n, A1 = 512, 360
A = A1 * N
g = bench.make_geometry(n, A, cs)
dev = torch.device("cuda", 0)
vol = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, g.voxel_grid, device=dev).data
y = torch.empty((A, n, n), device=dev)
for c in range(0, A, 360):
    K.fwd_interp(vol, g, (c, c + 360), (0, n), y[c:c + 360])
a0, a1 = rank * A1, (rank + 1) * A1
if inter:  # bench.atb_slabs: blocks r, r + N, r + 2N, r + 3N
    slabs = bench.atb_slabs(n, N, rank)
else:
    slabs = [(n * rank // N, n * (rank + 1) // N)]
nzr = sum(b - a for a, b in slabs)
z0, z1 = 0, nzr
proj = torch.empty((A1, n, n), device=dev)
slab = torch.zeros((nzr, n, n), device=dev)


def ax():
    for c in range(a0, a1, 90):
        K.fwd_interp(vol, g, (c, c + 90), (0, n), proj[c - a0:c - a0 + 90])


def atb():
    K.fill(slab, 0.0)
    for c in range(0, A, 90):
        o = 0
        for a_, b_ in slabs:
            K.bwd_matched(y[c:c + 90], g, (c, c + 90), (a_, b_),
                          slab[o:o + b_ - a_])
            o += b_ - a_


res = {"N": N, "rank": rank, "slabs": len(slabs)}
for name, fn, upd in (("ax", ax, A1 * n ** 3), ("atb", atb, A * (z1 - z0) * n * n)):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(3):
        fn()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 3 * 1e-3
    res[name + "_gups"] = upd / t / 1e9
    res[name + "_ms"] = t * 1e3
res["step_gups"] = (A1 * n ** 3 + A * (z1 - z0) * n * n) / (res["ax_ms"] + res["atb_ms"]) * 1e3 / 1e9
print(json.dumps(res), flush=True)
