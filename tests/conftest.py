"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on
CPU (the oracle, planner, geometry, host logic, multi-process gloo tests)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden.npz"))


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def product_geometry(d):
    """Golden geometry dict -> paper_1905_03748_b200.ScanGeometry."""
    from paper_1905_03748_b200 import DetectorGrid, ScanGeometry, VoxelGrid
    grid = VoxelGrid(d["nx"], d["ny"], d["nz"], tuple(d["voxel"]),
                     tuple(d["offset"]))
    det = DetectorGrid(d["nu"], d["nv"], tuple(d["pixel"]),
                       tuple(d["det_offset"]))
    return ScanGeometry(d["dso"], d["dsd"], tuple(d["angles"]), grid, det)


def oracle_geometry(d):
    from oracle import oracle as O
    return O.OGeom(d["dso"], d["dsd"], tuple(d["angles"]), d["nx"], d["ny"],
                   d["nz"], tuple(d["voxel"]), tuple(d["offset"]), d["nu"],
                   d["nv"], tuple(d["pixel"]), tuple(d["det_offset"]))


def synth_geometry(n, n_angles, nu=None, nv=None):
    """SURVEY 8(d) make_geo as a product ScanGeometry."""
    import math
    from paper_1905_03748_b200 import DetectorGrid, ScanGeometry, VoxelGrid
    nu = n if nu is None else nu
    nv = n if nv is None else nv
    mag = 2.0
    diag = math.sqrt(2.0 * n * n)
    det = DetectorGrid(nu, nv, (mag * diag / nu, mag * max(diag, n) / nv))
    angles = tuple(np.linspace(0.0, 2 * math.pi, n_angles, endpoint=False))
    return ScanGeometry(2.0 * n, 4.0 * n, angles, VoxelGrid(n, n, n), det)


def to_oracle(g):
    from oracle import oracle as O
    grid, det = g.voxel_grid, g.detector
    return O.OGeom(g.dso, g.dsd, g.angles, grid.n_x, grid.n_y, grid.n_z,
                   tuple(grid.voxel_size), tuple(grid.origin_offset),
                   det.n_u, det.n_v, tuple(det.pixel_size),
                   tuple(det.detector_offset))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def max_rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))
