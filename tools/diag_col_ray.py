"""Trace a matched-Atb column-sum deviation to single rays: for a
tools/fuzz_loops.py case, find the voxel of A^T 1 (per OS-SART block) with
the largest relative GPU/oracle difference, then compare the GPU and oracle
contributions of every single ray (one-hot projection) to that voxel.

    python tools/diag_col_ray.py SEED CASE
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tools")]
os.environ.setdefault("FUZZ_MAXN", "20")
import numpy as np
import torch

from paper_1905_03748_b200 import kernels as K
from conftest import to_oracle
from oracle import oracle as O
from diag_loop_case import loop_cases


def main():
    seed, ci = int(sys.argv[1]), int(sys.argv[2])
    g, x0, its, block, lam = loop_cases(seed, ci + 1)[ci]
    og = to_oracle(g)
    grid, det, na = g.voxel_grid, g.detector, g.n_angles
    shp = (grid.n_z, grid.n_y, grid.n_x)
    dev = torch.device("cuda", 0)
    print(json.dumps({"case": ci, "grid": list(grid.counts),
                      "voxel": list(grid.voxel_size), "det": [det.n_u, det.n_v],
                      "pixel": list(det.pixel_size), "dso": g.dso, "dsd": g.dsd,
                      "angles": list(g.angles)}))
    for b0, b1 in O.angle_blocks(na, block):
        ones = np.ones((b1 - b0, det.n_v, det.n_u), np.float32)
        co = O.bwd_matched(ones, og, (b0, b1)).astype(np.float64)
        cg_t = torch.zeros(shp, device=dev)
        K.bwd_matched(torch.from_numpy(ones).to(dev), g, (b0, b1),
                      (0, grid.n_z), cg_t)
        cg = cg_t.cpu().numpy().astype(np.float64)
        m = co > 0
        rel = np.zeros_like(co)
        rel[m] = np.abs(cg[m] - co[m]) / co[m]
        j = int(np.argmax(rel))
        vz = np.unravel_index(j, shp)
        print(json.dumps({"block": [b0, b1], "worst_rel": float(rel.ravel()[j]),
                          "voxel": list(map(int, vz)), "col_oracle": float(co.ravel()[j]),
                          "col_gpu": float(cg.ravel()[j]),
                          "n_rel_gt_1e-4": int((rel > 1e-4).sum()),
                          "n_pos": int(m.sum())}))
        if rel.ravel()[j] < 1e-5:
            continue
        rows = []
        for a in range(b0, b1):
            for v in range(det.n_v):
                for u in range(det.n_u):
                    p = np.zeros((1, det.n_v, det.n_u), np.float32)
                    p[0, v, u] = 1.0
                    o = float(O.bwd_matched(p, og, (a, a + 1))[vz])
                    t = torch.zeros(shp, device=dev)
                    K.bwd_matched(torch.from_numpy(p).to(dev), g, (a, a + 1),
                                  (0, grid.n_z), t)
                    gv = float(t[vz].item())
                    if o != 0.0 or gv != 0.0:
                        rows.append({"a": a, "u": u, "v": v, "oracle": o,
                                     "gpu": gv,
                                     "rel": abs(gv - o) / max(abs(o), 1e-30)})
        rows.sort(key=lambda r: -abs(r["gpu"] - r["oracle"]))
        for r in rows[:12]:
            print(json.dumps(r))
        print(json.dumps({"sum_oracle": sum(r["oracle"] for r in rows),
                          "sum_gpu": sum(r["gpu"] for r in rows),
                          "n_rays": len(rows)}))


if __name__ == "__main__":
    main()
