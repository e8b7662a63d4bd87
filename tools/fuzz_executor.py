"""Randomised executor sweep: random geometries (tools/fuzz_parity.case),
pools of 1-3 budgeted devices (all on cuda:0) with budgets that force 1..8
slab splits, chunked windows; execute_forward / execute_backward (interp /
Siddon, matched / FDK) against the monolithic operators, traces checked.

    python tools/fuzz_executor.py [cases=30] [seed=0]
"""
import importlib.util
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np

import paper_1905_03748_b200 as cs
from conftest import rel_l2

spec = importlib.util.spec_from_file_location(
    "fuzz_parity", os.path.join(ROOT, "tools", "fuzz_parity.py"))
fz = importlib.util.module_from_spec(spec)
spec.loader.exec_module(fz)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    fails, worst = 0, {}
    for i in range(n):
        while True:
            try:
                g = fz.case(rng)
                break
            except ValueError:
                continue
        grid, det = g.voxel_grid, g.detector
        na = g.n_angles
        x = rng.random((grid.n_z, grid.n_y, grid.n_x), dtype=np.float32)
        y = rng.standard_normal((na, det.n_v, det.n_u)).astype(np.float32)
        vol, stack = cs.Volume(grid, x), cs.ProjectionStack(det, y)
        plane = grid.n_x * grid.n_y * 4
        sheet = det.n_u * det.n_v * 4
        splits = int(rng.integers(1, 9))
        nd = int(rng.integers(1, 4))
        slab = max(1, -(-grid.n_z // splits))
        budget = int((slab * plane + 4 * 32 * sheet) / 0.95) + 4096
        pool = cs.DevicePool(tuple(cs.DeviceSpec(memory_budget=budget)
                                   for _ in range(nd)))
        res = {}
        try:
            for meth, key in ((cs.ProjectionMethod.INTERPOLATED, "fwd_interp"),
                              (cs.ProjectionMethod.SIDDON, "fwd_siddon")):
                mono = cs.forward_project_slab(vol, g, (0, na), meth).data
                sink = []
                got = cs.execute_forward(vol, g, pool, cs.plan_forward(g, pool),
                                         meth, trace_sink=sink).data
                res[key] = rel_l2(got, mono)
            for mode, key in ((cs.WeightMode.MATCHED, "bwd_matched"),
                              (cs.WeightMode.FDK, "bwd_fdk")):
                mono = cs.backproject_slab(stack, g, (0, grid.n_z), mode).data
                got = cs.execute_backward(stack, g, pool,
                                          cs.plan_backward(g, pool), mode).data
                res[key] = rel_l2(got, mono)
        except cs.InfeasiblePlanError:
            continue
        for k, v in res.items():
            worst[k] = max(worst.get(k, 0.0), v)
        bad = {k: v for k, v in res.items() if v > 1e-6}
        if bad:
            fails += 1
            print(json.dumps({"case": i, "bad": bad, "splits": splits,
                              "devices": nd,
                              "grid": [grid.n_x, grid.n_y, grid.n_z]}),
                  flush=True)
    print(json.dumps({"cases": n, "failures": fails, "worst_relL2": worst}))


if __name__ == "__main__":
    main()
