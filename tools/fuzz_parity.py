"""Randomised parity sweep (GPU vs oracle): random grids (sizes, anisotropic
voxels, offsets), detectors (sizes, pitches, offsets), source distances,
angle sets, slab and view windows; Ax (interp, Siddon), matched and FDK Atb.
Prints one JSON line per failing case and a summary.

    python tools/fuzz_parity.py [cases=60] [seed=0]
    FUZZ_FINE=0.5 python tools/fuzz_parity.py ...   # half with fine pixels
    FUZZ_CLOSE=1 FUZZ_VIEWS=40 python tools/fuzz_parity.py ...  # wide fan
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np

import paper_1905_03748_b200 as cs
from conftest import rel_l2, to_oracle
from oracle import oracle as O

IP, SD = cs.ProjectionMethod.INTERPOLATED, cs.ProjectionMethod.SIDDON
FINE_FRACTION = float(os.environ.get("FUZZ_FINE", "0"))
CLOSE = os.environ.get("FUZZ_CLOSE") == "1"
MAX_VIEWS = int(os.environ.get("FUZZ_VIEWS", "12"))
MAX_N = int(os.environ.get("FUZZ_MAXN", "40"))
COARSE = os.environ.get("FUZZ_COARSE") == "1"


def case(rng):
    nx, ny, nz = (int(v) for v in rng.integers(3, MAX_N + 1, 3))
    vox = tuple(float(v) for v in rng.uniform(0.5, 1.6, 3))
    off = tuple(float(v) for v in rng.uniform(-3, 3, 3))
    grid = cs.VoxelGrid(nx, ny, nz, vox, off)
    r = grid.bounding_radius()
    lo = 1.05 if CLOSE else 1.3  # FUZZ_CLOSE: source near the grid (wide fan)
    dso = float(r * rng.uniform(lo, 1.4 if CLOSE else 4.0) + abs(off[0])
                + abs(off[1]) + 1.0)
    dsd = float(dso + r * rng.uniform(1.2, 3.0) + abs(off[0]) + abs(off[1]))
    fine = rng.random() < FINE_FRACTION  # pixels much finer than voxels
    nu, nv = (int(v) for v in rng.integers(4, 96 if fine else 48, 2))
    ext = grid.extent
    mag = dsd / dso
    span = rng.uniform(0.6, 1.6) * (rng.uniform(0.05, 0.3) if fine else 1.0)
    pitch = (float(span * mag * max(ext[0], ext[1]) / nu),
             float(span * mag * ext[2] / nv))
    if COARSE:  # large detectors of coarse pixels: rays 1.6-3 voxels apart
        nu, nv = (int(v) for v in rng.integers(64, 129, 2))
        fp = rng.uniform(1.6, 3.0, 2) * float(np.mean(vox))
        pitch = (float(fp[0] * mag), float(fp[1] * mag))
    doff = (float(rng.uniform(-0.3, 0.3) * nu * pitch[0]),
            float(rng.uniform(-0.3, 0.3) * nv * pitch[1]))
    na = int(rng.integers(1, MAX_VIEWS + 1))
    angles = tuple(float(a) for a in rng.uniform(-7, 7, na))
    det = cs.DetectorGrid(nu, nv, pitch, doff)
    return cs.ScanGeometry(dso, dsd, angles, grid, det)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    worst = {}
    fails = 0
    for i in range(n):
        while True:
            try:
                g = case(rng)
                break
            except ValueError:  # geometry rejected by the clearance check
                continue
        og = to_oracle(g)
        grid, det = g.voxel_grid, g.detector
        na, nz = g.n_angles, grid.n_z
        x = rng.random((nz, grid.n_y, grid.n_x), dtype=np.float32)
        y = rng.standard_normal((na, det.n_v, det.n_u)).astype(np.float32)
        z0 = int(rng.integers(0, nz))
        z1 = int(rng.integers(z0 + 1, nz + 1))
        a0 = int(rng.integers(0, na))
        a1 = int(rng.integers(a0 + 1, na + 1))
        print(json.dumps({"start": i, "grid": [grid.n_x, grid.n_y, nz],
                          "vox": grid.voxel_size, "off": grid.origin_offset,
                          "dso": g.dso, "dsd": g.dsd, "angles": g.angles,
                          "det": [det.n_u, det.n_v], "pitch": det.pixel_size,
                          "det_off": det.detector_offset, "slab": [z0, z1],
                          "views": [a0, a1]}), file=sys.stderr, flush=True)
        res = {}
        xs = x[z0:z1]
        res["ax"] = rel_l2(cs.forward_project_slab(
            cs.Volume(grid, xs, (z0, z1)), g, (a0, a1), IP).data,
            O.fwd_interp(xs, og, (a0, a1), (z0, z1)))
        res["siddon"] = rel_l2(cs.forward_project_slab(
            cs.Volume(grid, xs, (z0, z1)), g, (a0, a1), SD).data,
            O.fwd_siddon(xs, og, (a0, a1), (z0, z1)))
        st = cs.ProjectionStack(det, y[a0:a1], (a0, a1))
        res["matched"] = rel_l2(cs.backproject_slab(
            st, g, (z0, z1), cs.WeightMode.MATCHED).data,
            O.bwd_matched(y[a0:a1], og, (a0, a1), (z0, z1)))
        res["fdk"] = rel_l2(cs.backproject_slab(
            st, g, (z0, z1), cs.WeightMode.FDK).data,
            O.bwd_fdk(y[a0:a1], og, (a0, a1), (z0, z1)))
        for k, v in res.items():
            if not (v == v):  # nan: both sides zero (no ray hits the slab)
                continue
            worst[k] = max(worst.get(k, 0.0), v)
        bad = {k: v for k, v in res.items() if v == v and v > 1e-5}
        if bad:
            fails += 1
            print(json.dumps({"case": i, "bad": bad, "grid": [grid.n_x, grid.n_y, nz],
                              "vox": grid.voxel_size, "det": [det.n_u, det.n_v],
                              "slab": [z0, z1], "views": [a0, a1]}), flush=True)
    print(json.dumps({"cases": n, "failures": fails, "worst_relL2": worst}))


if __name__ == "__main__":
    main()
