import sys, os, math
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "tests")]
import numpy as np
import paper_1905_03748_b200 as cs
from conftest import to_oracle, rel_l2
from oracle import oracle as O
nx, ny, nz = 3, 1, 5
grid = cs.VoxelGrid(nx, ny, nz, (1.0, 1.2, 0.8))
det = cs.DetectorGrid(9, 7, (0.7, 0.6))
angles = tuple(np.linspace(0.05, 2 * math.pi, 6, endpoint=False))
g = cs.ScanGeometry(12.0, 24.0, angles, grid, det)
og = to_oracle(g)
rng = np.random.default_rng(9)
x = rng.random((nz, ny, nx), dtype=np.float32)
y = rng.standard_normal((6, 7, 9)).astype(np.float32)
st = cs.ProjectionStack(det, y)
for zr in ((0, nz), (nz - 1, nz), (0, 1), (2, 3)):
    got = cs.backproject_slab(st, g, zr, cs.WeightMode.MATCHED).data
    ref = O.bwd_matched(y, og, (0, 6), zr)
    print(os.environ.get("CS_STAGED_SMEM_KB", "64"), zr, rel_l2(got, ref), np.abs(got - ref).max(), np.abs(ref).max())
