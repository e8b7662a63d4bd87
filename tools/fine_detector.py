"""Matched Atb on a fine detector (pixels much smaller than voxels):
256^3 volume, 1024^2 detector, 90 views -- throughput of the int32 and
int64 box paths and parity on a window vs the oracle."""
import json, os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np, torch
import bench, paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K
from conftest import to_oracle, rel_l2
from oracle import oracle as O
n, nd, A = 256, int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 90
grid = cs.VoxelGrid(n, n, n)
full = bench.make_geometry(n, A, cs)
det = cs.DetectorGrid(nd, nd, (full.detector.pixel_size[0] * n / nd, full.detector.pixel_size[1] * n / nd))
g = cs.ScanGeometry(full.dso, full.dsd, full.angles, grid, det)
dev = torch.device("cuda", 0)
y = torch.randn((A, nd, nd), device=dev, generator=torch.Generator(device=dev).manual_seed(0))
acc = torch.zeros((n, n, n), device=dev)
K.bwd_matched(y, g, (0, A), (0, n), acc); torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); K.bwd_matched(y, g, (0, A), (0, n), acc); e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e) * 1e-3
# parity on a 2-view window, 8-plane slab
og = to_oracle(g)
yw = y[10:12].cpu().numpy()
zr = (120, 128)
a2 = torch.zeros((8, n, n), device=dev)
K.bwd_matched(y[10:12].contiguous(), g, (10, 12), zr, a2)
err = rel_l2(a2.cpu(), O.bwd_matched(yw, og, (10, 12), zr))
print(json.dumps({"n": n, "det": nd, "views": A, "gups": A * n ** 3 / t / 1e9, "ms": t * 1e3, "relL2_window": err}))
