"""Generate golden fixtures by running the REFERENCE implementation.

Run here (the container that mounts /root/reference), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/golden.npz (+ plans.json).  Every array is the output of
the reference's public API (conesplit.forward_project_slab,
backproject_slab, tv_norm, minimize_tv_gradient, minimize_rof,
split_minimize, cgls, os_sart, fdk, plan_forward/plan_backward) on seeded
inputs.  The product never reads these at run time; tests compare the
oracle (tests -m "not gpu") and the CUDA path (tests -m gpu) against them.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

import conesplit as cs
from conesplit import _kernels

HERE = os.path.dirname(os.path.abspath(__file__))


def geo_cases():
    """(name, ScanGeometry) pairs: the SURVEY 8(d) geometry at small sizes
    plus an off-centre, anisotropic one that exercises every offset."""
    out = []

    def make(n, a, nu, nv, voxel=(1.0, 1.0, 1.0), off=(0.0, 0.0, 0.0),
             det_off=(0.0, 0.0), span=2 * math.pi, nz=None):
        nz = n if nz is None else nz
        grid = cs.VoxelGrid(n, n, nz, voxel, off)
        ext = grid.extent
        dso, dsd = 2.0 * max(n, nz), 4.0 * max(n, nz)
        mag = dsd / dso
        diag = math.sqrt(ext[0] ** 2 + ext[1] ** 2)
        det = cs.DetectorGrid(nu, nv, (mag * diag / nu,
                                       mag * max(diag, ext[2]) / nv), det_off)
        angles = tuple(np.linspace(0.0, span, a, endpoint=False))
        return cs.ScanGeometry(dso, dsd, angles, grid, det)

    out.append(("g16", make(16, 8, 24, 20)))
    out.append(("ganiso", make(12, 7, 18, 16, voxel=(1.0, 0.8, 1.25),
                               off=(0.6, -0.35, 0.3), det_off=(0.9, -0.55),
                               span=3.0, nz=10)))
    out.append(("g32", make(32, 20, 32, 32)))
    return out


def geo_dict(g):
    return dict(dso=g.dso, dsd=g.dsd, angles=list(g.angles),
                nx=g.voxel_grid.n_x, ny=g.voxel_grid.n_y, nz=g.voxel_grid.n_z,
                voxel=list(g.voxel_grid.voxel_size),
                offset=list(g.voxel_grid.origin_offset),
                nu=g.detector.n_u, nv=g.detector.n_v,
                pixel=list(g.detector.pixel_size),
                det_offset=list(g.detector.detector_offset))


def main():
    _kernels.warm_up()
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"numpy": np.__version__,
                  "numba": __import__("numba").__version__,
                  "geometries": {}}
    IP, SD = cs.ProjectionMethod.INTERPOLATED, cs.ProjectionMethod.SIDDON
    for name, g in geo_cases():
        meta["geometries"][name] = geo_dict(g)
        grid = g.voxel_grid
        nz, A = grid.n_z, g.n_angles
        rng = np.random.default_rng(0)
        x = rng.random((nz, grid.n_y, grid.n_x), dtype=np.float32)
        y = np.random.default_rng(1).standard_normal(
            (A, g.detector.n_v, g.detector.n_u)).astype(np.float32)
        vol = cs.Volume(grid, x)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/y"] = y
        arrays[f"{name}/fwd_interp"] = cs.forward_project_slab(
            vol, g, (0, A), IP).data
        arrays[f"{name}/fwd_siddon"] = cs.forward_project_slab(
            vol, g, (0, A), SD).data
        # slab + angle-window variants (absolute ranges)
        z0, z1 = nz // 3, (2 * nz) // 3 + 1
        a0, a1 = 1, A - 2
        slab = cs.Volume(grid, x[z0:z1], (z0, z1))
        arrays[f"{name}/fwd_interp_slab"] = cs.forward_project_slab(
            slab, g, (a0, a1), IP).data
        arrays[f"{name}/fwd_siddon_slab"] = cs.forward_project_slab(
            slab, g, (a0, a1), SD).data
        stack = cs.ProjectionStack(g.detector, y, (0, A))
        arrays[f"{name}/bwd_matched"] = cs.backproject_slab(
            stack, g, (0, nz), cs.WeightMode.MATCHED).data
        arrays[f"{name}/bwd_fdk"] = cs.backproject_slab(
            stack, g, (0, nz), cs.WeightMode.FDK).data
        sub = cs.ProjectionStack(g.detector, y[a0:a1], (a0, a1))
        acc0 = cs.Volume(grid, x[z0:z1] * 0.5, (z0, z1))
        arrays[f"{name}/bwd_matched_slab"] = cs.backproject_slab(
            sub, g, (z0, z1), cs.WeightMode.MATCHED,
            accumulate_into=acc0.copy()).data
        arrays[f"{name}/bwd_fdk_slab"] = cs.backproject_slab(
            sub, g, (z0, z1), cs.WeightMode.FDK,
            accumulate_into=acc0.copy()).data
        meta["geometries"][name]["slab"] = [z0, z1]
        meta["geometries"][name]["window"] = [a0, a1]
        # per-ray fp64 set-up (t0, step, n_steps), _kernels.py:194-210
        from conesplit.projectors import _flat_geometry, _grid_params
        srcs, det00, ustep, vstep = _flat_geometry(g, range(A))
        gx0, gy0, gz0, vx, vy, vz, nx, ny, nzz = _grid_params(grid)
        det = g.detector
        t0s = np.zeros((A, det.n_v, det.n_u))
        sts = np.zeros_like(t0s)
        ns = np.zeros(t0s.shape, np.int64)
        for a in range(A):
            for v in range(det.n_v):
                for u in range(det.n_u):
                    # scalar replay of _kernels.py:234-243
                    d = [det00[a, i] + u * ustep[a, i] + v * vstep[a, i]
                         - srcs[a, i] for i in range(3)]
                    inv = 1.0 / math.sqrt(d[0] * d[0] + d[1] * d[1]
                                          + d[2] * d[2])
                    d = [c * inv for c in d]
                    r = _kernels._ray_steps(srcs[a, 0], srcs[a, 1], srcs[a, 2],
                                            d[0], d[1], d[2], gx0, gy0, gz0,
                                            vx, vy, vz, nx, ny, nzz,
                                            cs.projectors.sample_step(grid))
                    t0s[a, v, u], sts[a, v, u], ns[a, v, u] = r
        arrays[f"{name}/ray_t0"] = t0s
        arrays[f"{name}/ray_step"] = sts
        arrays[f"{name}/ray_n"] = ns

    # ---- KATs (SPEC.md examples) --------------------------------------
    grid = cs.VoxelGrid(10, 10, 10)
    det = cs.DetectorGrid(3, 3, (1.0, 1.0))
    g = cs.ScanGeometry(50.0, 100.0, (0.0,), grid, det)
    cube = cs.Volume(grid, np.full((10, 10, 10), 0.02, np.float32))
    arrays["kat/cube_siddon"] = cs.forward_project_slab(cube, g, (0, 1), SD).data
    arrays["kat/cube_interp"] = cs.forward_project_slab(cube, g, (0, 1), IP).data
    meta["kat_cube"] = geo_dict(g)

    # ---- TV ------------------------------------------------------------
    tv_grid = cs.VoxelGrid(20, 18, 24)
    blocks = cs.phantom(cs.PhantomKind.BLOCKS, tv_grid).data
    noisy = (blocks + 0.05 * np.random.default_rng(2).standard_normal(
        blocks.shape)).astype(np.float32)
    arrays["tv/f"] = noisy
    tvv = cs.Volume(tv_grid, noisy)
    arrays["tv/norm"] = np.array(cs.tv_norm(tvv))
    single = np.zeros((3, 3, 3), np.float32)
    single[1, 1, 1] = 1.0
    arrays["tv/single_voxel_norm"] = np.array(
        cs.tv_norm(cs.Volume(cs.VoxelGrid(3, 3, 3), single)))
    GD, ROF = cs.TvMinimizer.GRADIENT_DESCENT, cs.TvMinimizer.ROF
    arrays["tv/gd"] = cs.minimize_tv_gradient(
        tvv, cs.TvParams(GD, inner_iters=12, step=0.05)).data
    arrays["tv/rof"] = cs.minimize_rof(
        tvv, cs.TvParams(ROF, inner_iters=12, lam=0.1)).data
    budget = 6 * 20 * 18 * 4 * 2 * 5  # forces several slabs
    for dev in (1, 2, 3):
        pool = cs.DevicePool(tuple(cs.DeviceSpec(memory_budget=10 ** 9)
                                   for _ in range(dev)))
        for minim, tag in ((GD, "gd"), (ROF, "rof")):
            for nm, ntag in ((cs.NormMode.EXACT_GLOBAL, "exact"),
                             (cs.NormMode.LOCAL_APPROX, "local")):
                if minim is ROF and ntag == "local":
                    continue
                p = cs.TvParams(minim, outer_syncs=2, inner_iters=4,
                                step=0.05, lam=0.1, norm_mode=nm,
                                halo_depth=5)
                arrays[f"tv/split_{tag}_{ntag}_d{dev}"] = cs.split_minimize(
                    tvv, pool, p).data
    del budget

    # ---- loops -----------------------------------------------------------
    _, g16 = geo_cases()[0]
    pool1 = cs.DevicePool((cs.DeviceSpec(memory_budget=2 ** 30),))
    grid16 = g16.voxel_grid
    ph = cs.phantom(cs.PhantomKind.SHEPP_LOGAN_3D, grid16)
    arrays["loops/phantom16"] = ph.data
    b = cs.forward_project_slab(ph, g16, (0, g16.n_angles), IP)
    arrays["loops/b16"] = b.data
    res = cs.cgls(b, g16, cs.ReconConfig(pool1, iterations=4))
    arrays["loops/cgls_x"] = res.volume.data
    arrays["loops/cgls_res"] = np.array(res.residuals)
    arrays["loops/sirt_x"] = cs.os_sart(b, g16, cs.ReconConfig(
        pool1, cs.Algorithm.OSSART, iterations=3,
        block_size=g16.n_angles)).data
    arrays["loops/ossart_x"] = cs.os_sart(b, g16, cs.ReconConfig(
        pool1, cs.Algorithm.OSSART, iterations=2, block_size=3,
        relaxation=0.8)).data
    tvp = cs.TvParams(GD, inner_iters=5, step=0.01)
    arrays["loops/sarttv_x"] = cs.os_sart(b, g16, cs.ReconConfig(
        pool1, cs.Algorithm.OSSART, iterations=2, block_size=4, tv=tvp)).data
    arrays["loops/fdk_x"] = cs.fdk(b, g16, pool1).data

    # ---- planner ---------------------------------------------------------
    plans = []
    rng = np.random.default_rng(5)
    for i in range(60):
        n = int(rng.integers(8, 600))
        nzp = int(rng.integers(4, 600))
        A = int(rng.integers(1, 400))
        nu = int(rng.integers(4, 600))
        nv = int(rng.integers(4, 600))
        dev = int(rng.integers(1, 5))
        budget = int(rng.integers(2 ** 20, 2 ** 31))
        uf = float(rng.choice([0.85, 0.95, 1.0]))
        grid = cs.VoxelGrid(n, n, nzp)
        det = cs.DetectorGrid(nu, nv)
        r = grid.bounding_radius()
        gg = cs.ScanGeometry(3 * r + 1, 7 * r + 2, tuple(
            np.linspace(0, 2 * math.pi, A, endpoint=False)), grid, det)
        pool = cs.DevicePool(tuple(cs.DeviceSpec(memory_budget=budget)
                                   for _ in range(dev)))
        for op, fn in (("forward", cs.plan_forward),
                       ("backward", cs.plan_backward)):
            case = dict(op=op, n=n, nz=nzp, A=A, nu=nu, nv=nv, dev=dev,
                        budget=budget, uf=uf)
            try:
                p = fn(gg, pool, usable_fraction=uf)
                case["plan"] = dict(
                    n_splits=p.n_splits, slab_ranges=p.slab_ranges,
                    angle_assignment=p.angle_assignment,
                    chunk_angles=p.chunk_angles, buffer_count=p.buffer_count,
                    pin_host_image=p.pin_host_image,
                    per_device_bytes_peak=p.per_device_bytes_peak)
            except cs.InfeasiblePlanError:
                case["plan"] = None
            plans.append(case)
    meta["plans"] = plans

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, default=list)
    total = sum(a.nbytes for a in arrays.values())
    print(f"wrote {len(arrays)} arrays ({total / 1e6:.2f} MB raw)",
          file=sys.stderr)


if __name__ == "__main__":
    main()
