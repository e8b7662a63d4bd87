"""Randomised loop sweep: random small geometries (tools/fuzz_parity.case,
grids <= 20 per axis), random block sizes / relaxations / iterations,
optional TV-GD; os_sart and cgls (public API, host numpy) against the
oracle's loops.  Tolerance 3e-5 relL2 (3x the operator's).

    python tools/fuzz_loops.py [cases=20] [seed=0]
"""
import importlib.util
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
os.environ.setdefault("FUZZ_MAXN", "20")
import numpy as np

import paper_1905_03748_b200 as cs
from conftest import rel_l2, to_oracle
from oracle import oracle as O

spec = importlib.util.spec_from_file_location(
    "fuzz_parity", os.path.join(ROOT, "tools", "fuzz_parity.py"))
fz = importlib.util.module_from_spec(spec)
spec.loader.exec_module(fz)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    pool = cs.DevicePool.b200(1)
    fails, worst = 0, {}
    for i in range(n):
        while True:
            try:
                g = fz.case(rng)
                if min(g.voxel_grid.counts) >= 2:
                    break
            except ValueError:
                continue
        og = to_oracle(g)
        grid, det = g.voxel_grid, g.detector
        na = g.n_angles
        x = rng.random((grid.n_z, grid.n_y, grid.n_x), dtype=np.float32)
        b = O.fwd_interp(x, og).astype(np.float32)
        stack = cs.ProjectionStack(det, b)
        its = int(rng.integers(1, 4))
        block = int(rng.integers(1, na + 1))
        lam = float(rng.uniform(0.3, 1.5))
        res = {}
        got = cs.os_sart(stack, g, cs.ReconConfig(
            pool, cs.Algorithm.OSSART, its, block, lam)).data
        res["os_sart"] = rel_l2(got, O.os_sart(b, og, its, block, lam))
        r = cs.cgls(stack, g, cs.ReconConfig(pool, cs.Algorithm.CGLS, its))
        xo, reso, _ = O.cgls(b, og, its)
        res["cgls"] = rel_l2(r.volume.data, xo)
        if rng.random() < 0.5 and grid.n_z >= 4:
            tv = cs.TvParams(cs.TvMinimizer.GRADIENT_DESCENT, 1, 3, 1e-3)
            got = cs.os_sart(stack, g, cs.ReconConfig(
                pool, cs.Algorithm.OSSART, its, block, lam, tv=tv)).data
            ref = O.os_sart(b, og, its, block, lam,
                            tv=dict(n_slabs=1, minimizer="gd", outer_syncs=1,
                                    inner_iters=3, step=1e-3))
            res["sart_tv"] = rel_l2(got, ref)
        for k, v in res.items():
            worst[k] = max(worst.get(k, 0.0), v)
        bad = {k: v for k, v in res.items() if v > 3e-5}
        if bad:
            fails += 1
            print(json.dumps({"case": i, "bad": bad, "iters": its,
                              "block": block, "views": na,
                              "grid": list(grid.counts)}), flush=True)
    print(json.dumps({"cases": n, "failures": fails, "worst_relL2": worst}))


if __name__ == "__main__":
    main()
