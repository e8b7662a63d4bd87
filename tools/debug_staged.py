import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K
from conftest import synth_geometry, to_oracle
from oracle import oracle as O
def run(g, x, ar, sr, label):
    og = to_oracle(g)
    out = torch.empty((ar[1]-ar[0], g.detector.n_v, g.detector.n_u), device="cuda")
    K.fwd_interp(torch.from_numpy(x[sr[0]:sr[1]].copy()).cuda(), g, ar, sr, out)
    got = out.cpu().numpy(); ref = O.fwd_interp(x[sr[0]:sr[1]], og, ar, sr)
    err = np.abs(got-ref); i = np.unravel_index(err.argmax(), err.shape)
    print(label, "relL2 %.3g" % (np.linalg.norm(got-ref)/max(np.linalg.norm(ref),1e-30)), "max at", i, got[i], ref[i],
          "bad views", sorted(set(np.nonzero(err > 1e-4*np.abs(ref).max())[0].tolist()))[:20])
g = synth_geometry(16, 8, nu=24, nv=20)
x = np.random.default_rng(0).random((16,16,16), dtype=np.float32)
run(g, x, (0, 8), (0, 16), "full")
run(g, x, (0, 8), (5, 11), "slab")
run(g, x, (1, 6), (0, 16), "window")
grid = cs.VoxelGrid(8, 8, 8)
det = cs.DetectorGrid(40, 30, (2.0, 2.0))
g2 = cs.ScanGeometry(40.0, 80.0, (0.3,), grid, det)
x2 = np.random.default_rng(5).random((8, 8, 8), dtype=np.float32)
run(g2, x2, (0, 1), (0, 8), "edge")
g3 = synth_geometry(48, 36)
x3 = np.random.default_rng(0).random((48,48,48), dtype=np.float32)
run(g3, x3, (0, 36), (0, 48), "48full")
run(g3, x3, (0, 36), (20, 41), "48slab")
