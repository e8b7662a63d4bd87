"""Golden files for the raw/sidecar format, written by the REFERENCE's own
writers (conesplit.fileio.write_volume / write_projections).

Run here (the container that mounts /root/reference), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_fileio_golden.py

tests/test_fileio.py reads them with the product reader and checks the
product writer reproduces them byte for byte.
"""

from __future__ import annotations

import math
import os

import numpy as np

import conesplit as cs
from conesplit import fileio

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fileio")


def main():
    os.makedirs(OUT, exist_ok=True)
    grid = cs.VoxelGrid(5, 4, 3, (1.0, 0.9, 1.1), (0.3, -0.2, 0.1))
    vol = np.random.default_rng(7).standard_normal((3, 4, 5)).astype(
        np.float32)
    fileio.write_volume(os.path.join(OUT, "vol.raw"), cs.Volume(grid, vol))
    det = cs.DetectorGrid(6, 3, (2.5, 2.25), (0.4, -0.3))
    angles = tuple(float(a) for a in np.linspace(0.1, 0.1 + 2 * math.pi, 4,
                                                 endpoint=False))
    geo = cs.ScanGeometry(20.0, 40.0, angles, grid, det)
    proj = np.random.default_rng(8).standard_normal((4, 3, 6)).astype(
        np.float32)
    fileio.write_projections(os.path.join(OUT, "proj.raw"),
                             cs.ProjectionStack(det, proj), geo)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
