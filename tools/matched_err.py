"""Matched Atb error vs the oracle at config-2 geometry on thin windows
(dense random-sign stacks), for variant libraries (CS_LIB_PATH)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from conftest import rel_l2, synth_geometry, to_oracle
from oracle import oracle as O
from paper_1905_03748_b200 import kernels as K
n, A = 512, 360
g = synth_geometry(n, A); og = to_oracle(g)
res = {"lib": os.environ.get("CS_LIB_PATH", "prod")}
for win, zr in (((45, 47), (250, 258)), ((45, 47), (0, 8)), ((100, 101), (200, 264))):
    y = np.random.default_rng(1).standard_normal((win[1] - win[0], n, n)).astype(np.float32)
    acc = torch.zeros((zr[1] - zr[0], n, n), device="cuda")
    K.bwd_matched(torch.from_numpy(y).cuda(), g, win, zr, acc)
    ref = O.bwd_matched(y, og, win, zr)
    res[f"{win}{zr}"] = rel_l2(acc.cpu(), ref)
    yp = np.abs(y)
    acc.zero_()
    K.bwd_matched(torch.from_numpy(yp).cuda(), g, win, zr, acc)
    res[f"{win}{zr}abs"] = rel_l2(acc.cpu(), O.bwd_matched(yp, og, win, zr))
print(json.dumps(res))
