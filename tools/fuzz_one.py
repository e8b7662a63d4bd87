"""Re-run one case of tools/fuzz_parity.py (same seed / index / env knobs)
and print its per-operator relL2:  python tools/fuzz_one.py SEED INDEX"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import importlib.util
import numpy as np

spec = importlib.util.spec_from_file_location(
    "fuzz_parity", os.path.join(ROOT, "tools", "fuzz_parity.py"))
fz = importlib.util.module_from_spec(spec)
spec.loader.exec_module(fz)
import paper_1905_03748_b200 as cs
from conftest import rel_l2, to_oracle
from oracle import oracle as O

seed, target = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
for i in range(target + 1):
    while True:
        try:
            g = fz.case(rng)
            break
        except ValueError:
            continue
    grid, det = g.voxel_grid, g.detector
    na, nz = g.n_angles, grid.n_z
    x = rng.random((nz, grid.n_y, grid.n_x), dtype=np.float32)
    y = rng.standard_normal((na, det.n_v, det.n_u)).astype(np.float32)
    z0 = int(rng.integers(0, nz))
    z1 = int(rng.integers(z0 + 1, nz + 1))
    a0 = int(rng.integers(0, na))
    a1 = int(rng.integers(a0 + 1, na + 1))
og = to_oracle(g)
xs = x[z0:z1]
ax = cs.forward_project_slab(cs.Volume(grid, xs, (z0, z1)), g, (a0, a1),
                             cs.ProjectionMethod.INTERPOLATED).data
axo = O.fwd_interp(xs, og, (a0, a1), (z0, z1))
st = cs.ProjectionStack(det, y[a0:a1], (a0, a1))
mb = cs.backproject_slab(st, g, (z0, z1), cs.WeightMode.MATCHED).data
mbo = O.bwd_matched(y[a0:a1], og, (a0, a1), (z0, z1))
print({"ax": rel_l2(ax, axo), "matched": rel_l2(mb, mbo),
       "ax_norm": float(np.linalg.norm(axo)), "pitch": det.pixel_size,
       "vox": grid.voxel_size, "dso": g.dso, "dsd": g.dsd,
       "slab": (z0, z1), "det": (det.n_u, det.n_v)})
