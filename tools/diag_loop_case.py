"""Attribute an OS-SART deviation (GPU vs oracle) to its operators: replay
the reference's OS-SART in fp64 numpy with each of Ax, A^T(W r), W = 1/A1
and V = 1/A^T 1 taken from the GPU or from the oracle, one at a time.

    python tools/diag_loop_case.py SEED CASE [CASE ...]
(cases are the tools/fuzz_loops.py sequence for that seed)
"""
import importlib.util
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
os.environ.setdefault("FUZZ_MAXN", "20")
import numpy as np
import torch

import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K
from conftest import rel_l2, to_oracle
from oracle import oracle as O

spec = importlib.util.spec_from_file_location(
    "fz", os.path.join(ROOT, "tools", "fuzz_parity.py"))
fz = importlib.util.module_from_spec(spec)
spec.loader.exec_module(fz)


def loop_cases(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        while True:
            try:
                g = fz.case(rng)
                if min(g.voxel_grid.counts) >= 2:
                    break
            except ValueError:
                continue
        grid = g.voxel_grid
        x = rng.random((grid.n_z, grid.n_y, grid.n_x), dtype=np.float32)
        its = int(rng.integers(1, 4))
        block = int(rng.integers(1, g.n_angles + 1))
        lam = float(rng.uniform(0.3, 1.5))
        rng.random()
        out.append((g, x, its, block, lam))
    return out


def main():
    seed = int(sys.argv[1])
    want = [int(c) for c in sys.argv[2:]]
    cases = loop_cases(seed, max(want) + 1)
    dev = torch.device("cuda", 0)
    pool = cs.DevicePool.b200(1)
    for ci in want:
        g, x0, its, block, lam = cases[ci]
        og = to_oracle(g)
        grid, det, na = g.voxel_grid, g.detector, g.n_angles
        shp = (grid.n_z, grid.n_y, grid.n_x)
        b = O.fwd_interp(x0, og).astype(np.float32)
        ref = O.os_sart(b, og, its, block, lam)
        got = cs.os_sart(cs.ProjectionStack(det, b), g, cs.ReconConfig(
            pool, cs.Algorithm.OSSART, its, block, lam)).data

        def g_fwd(xx, a0, a1):
            out = torch.empty((a1 - a0, det.n_v, det.n_u), device=dev)
            K.fwd_interp(torch.from_numpy(np.asarray(xx, np.float32)).to(dev),
                         g, (a0, a1), (0, grid.n_z), out)
            return out.cpu().numpy().astype(np.float64)

        def g_bwd(yy, a0, a1):
            out = torch.zeros(shp, device=dev)
            K.bwd_matched(torch.from_numpy(np.asarray(yy, np.float32)).to(dev),
                          g, (a0, a1), (0, grid.n_z), out)
            return out.cpu().numpy().astype(np.float64)

        def o_fwd(xx, a0, a1):
            return O.fwd_interp(np.asarray(xx, np.float32), og,
                                (a0, a1)).astype(np.float64)

        def o_bwd(yy, a0, a1):
            return O.bwd_matched(np.asarray(yy, np.float32), og,
                                 (a0, a1)).astype(np.float64)

        def replay(src):
            fw = g_fwd if "ax" in src else o_fwd
            bw = g_bwd if "atb" in src else o_bwd
            wf = g_fwd if "w" in src else o_fwd
            vb = g_bwd if "v" in src else o_bwd
            blocks = O.angle_blocks(na, block)
            ws = []
            for b0, b1 in blocks:
                ws.append((O.guarded_inverse(wf(np.ones(shp), b0, b1)),
                           O.guarded_inverse(vb(np.ones((b1 - b0, det.n_v,
                                                         det.n_u)), b0, b1))))
            xx = np.zeros(shp)
            for _ in range(its):
                for (b0, b1), (w, v) in zip(blocks, ws):
                    r = b[b0:b1].astype(np.float64) - fw(xx, b0, b1)
                    xx += lam * v * bw(w * r, b0, b1)
            return xx.astype(np.float32)

        rep = {"case": ci, "grid": list(grid.counts), "views": na,
               "block": block, "its": its,
               "os_sart": rel_l2(got, ref)}
        for src in ([], ["ax"], ["atb"], ["w"], ["v"], ["atb", "v"],
                    ["ax", "atb", "w", "v"]):
            rep["+".join(src) or "oracle"] = rel_l2(replay(src), ref)
        d = np.abs(got - ref)
        j = int(np.argmax(d))
        rep["worst_voxel"] = [list(map(int, np.unravel_index(j, shp))),
                              float(got.ravel()[j]), float(ref.ravel()[j])]
        print(json.dumps(rep), flush=True)


if __name__ == "__main__":
    main()
