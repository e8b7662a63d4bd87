import importlib.util, json, os, sys
ROOT = "/root/repo"
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
os.environ.setdefault("FUZZ_MAXN", "20")
import numpy as np, torch
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K
from conftest import rel_l2, to_oracle
from oracle import oracle as O
spec = importlib.util.spec_from_file_location("fz", os.path.join(ROOT, "tools", "fuzz_parity.py"))
fz = importlib.util.module_from_spec(spec); spec.loader.exec_module(fz)
rng = np.random.default_rng(3)
pool = cs.DevicePool.b200(1)
target = int(sys.argv[1])
for i in range(target + 1):
    while True:
        try:
            g = fz.case(rng)
            if min(g.voxel_grid.counts) >= 2: break
        except ValueError: continue
    og = to_oracle(g); grid, det = g.voxel_grid, g.detector; na = g.n_angles
    x = rng.random((grid.n_z, grid.n_y, grid.n_x), dtype=np.float32)
    b = O.fwd_interp(x, og).astype(np.float32)
    its = int(rng.integers(1, 4)); block = int(rng.integers(1, na + 1)); lam = float(rng.uniform(0.3, 1.5))
    if i < target:
        if rng.random() < 0.5 and grid.n_z >= 4: pass
        continue
print("case", i, grid.counts, grid.voxel_size, det.n_u, det.n_v, det.pixel_size, "views", na, "block", block, "its", its, "lam", lam)
ones = np.ones((grid.n_z, grid.n_y, grid.n_x), np.float32)
row_o = O.fwd_interp(ones, og).astype(np.float64)
col_o = O.bwd_matched(np.ones((na, det.n_v, det.n_u), np.float32), og).astype(np.float64)
dev = torch.device("cuda", 0)
row_g = torch.empty((na, det.n_v, det.n_u), device=dev)
K.fwd_interp(torch.from_numpy(ones).to(dev), g, (0, na), (0, grid.n_z), row_g)
col_g = torch.zeros((grid.n_z, grid.n_y, grid.n_x), device=dev)
K.bwd_matched(torch.ones((na, det.n_v, det.n_u), device=dev), g, (0, na), (0, grid.n_z), col_g)
rg, cg = row_g.cpu().numpy().astype(np.float64), col_g.cpu().numpy().astype(np.float64)
print("row relL2", rel_l2(rg, row_o), "col relL2", rel_l2(cg, col_o))
m = row_o > 0
print("row min pos", row_o[m].min(), "max rel diff row", np.max(np.abs(rg[m] - row_o[m]) / row_o[m]))
mc = col_o > 0
print("col min pos", col_o[mc].min(), "max rel diff col", np.max(np.abs(cg[mc] - col_o[mc]) / col_o[mc]))
print("row zero mismatch", int(((row_o >= 1e-8) != (rg >= 1e-8)).sum()), "col zero mismatch", int(((col_o >= 1e-8) != (cg >= 1e-8)).sum()))
idx = np.argsort(np.abs(cg - col_o).ravel())[-5:]
print("worst col entries oracle/gpu", [(float(col_o.ravel()[j]), float(cg.ravel()[j])) for j in idx])
got = cs.os_sart(cs.ProjectionStack(det, b), g, cs.ReconConfig(pool, cs.Algorithm.OSSART, its, block, lam)).data
ref = O.os_sart(b, og, its, block, lam)
print("os_sart relL2", rel_l2(got, ref))
d = np.abs(got - ref); j = np.argmax(d); print("worst voxel", np.unravel_index(j, d.shape), got.ravel()[j], ref.ravel()[j], "col_o", col_o.ravel()[j])

# hypothesis test: OS-SART with the GPU operators but V (and W) from fp64
def blocks_of(na, bs):
    return O.angle_blocks(na, bs)

def sart(Vsrc):
    xg = np.zeros((grid.n_z, grid.n_y, grid.n_x), np.float64)
    bl = blocks_of(na, block)
    for _ in range(its):
        for (b0, b1) in bl:
            xt = torch.from_numpy(xg.astype(np.float32)).to(dev)
            ax = torch.empty((b1 - b0, det.n_v, det.n_u), device=dev)
            K.fwd_interp(xt, g, (b0, b1), (0, grid.n_z), ax)
            rowb = O.fwd_interp(ones, og, (b0, b1)).astype(np.float64)
            W = O.guarded_inverse(rowb)
            resid = (b[b0:b1].astype(np.float64) - ax.cpu().numpy()) * W
            acc = torch.zeros((grid.n_z, grid.n_y, grid.n_x), device=dev)
            K.bwd_matched(torch.from_numpy(resid.astype(np.float32)).to(dev), g, (b0, b1), (0, grid.n_z), acc)
            if Vsrc == "oracle":
                colb = O.bwd_matched(np.ones((b1 - b0, det.n_v, det.n_u), np.float32), og, (b0, b1)).astype(np.float64)
            else:
                cb = torch.zeros((grid.n_z, grid.n_y, grid.n_x), device=dev)
                K.bwd_matched(torch.ones((b1 - b0, det.n_v, det.n_u), device=dev), g, (b0, b1), (0, grid.n_z), cb)
                colb = cb.cpu().numpy().astype(np.float64)
            V = O.guarded_inverse(colb)
            xg += lam * V * acc.cpu().numpy()
    return xg.astype(np.float32)

print("emulated, V gpu:", rel_l2(sart("gpu"), ref), " V oracle:", rel_l2(sart("oracle"), ref))
