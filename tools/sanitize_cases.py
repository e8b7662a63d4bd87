"""Small invocations of every kernel for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): odd sizes, slab and window launches,
the staged kernels' half-depth and global-memory fallbacks (small box
budget via CS_STAGED_SMEM_KB), FDK's direct path, TV and vector kernels.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch

import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import kernels as K


def geometry(nx, ny, nz, nu, nv, na, pitch=None):
    grid = cs.VoxelGrid(nx, ny, nz, (1.0, 0.9, 1.1), (0.3, -0.2, 0.1))
    r = grid.bounding_radius()
    dso, dsd = 2.5 * r + 2.0, 5.0 * r + 4.0
    ext = grid.extent
    if pitch is None:
        pitch = (1.3 * dsd / dso * max(ext[0], ext[1]) / nu,
                 1.3 * dsd / dso * ext[2] / nv)
    det = cs.DetectorGrid(nu, nv, pitch, (0.4, -0.3))
    angles = tuple(np.linspace(0.1, 0.1 + 2 * math.pi, na, endpoint=False))
    return cs.ScanGeometry(dso, dsd, angles, grid, det)


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    for shape in ((13, 11, 9, 17, 15, 7), (24, 24, 20, 30, 26, 9)):
        nx, ny, nz, nu, nv, na = shape
        g = geometry(*shape)
        x = torch.from_numpy(rng.random((nz, ny, nx), dtype=np.float32)).to(dev)
        y = torch.from_numpy(rng.standard_normal((na, nv, nu)).astype(
            np.float32)).to(dev)
        p = torch.empty((na, nv, nu), device=dev)
        K.fwd_interp(x, g, (0, na), (0, nz), p)
        K.fwd_interp(x[2:nz - 1].contiguous(), g, (1, na - 1), (2, nz - 1),
                     p[1:na - 1], accumulate=True)
        K.fwd_siddon(x, g, (0, na), (0, nz), p)
        if not os.environ.get("SAN_NO_RESIDUAL"):  # needs the whole slab
            K.fwd_interp_residual(x, g, (0, na), y, None, p)
        acc = torch.zeros_like(x)
        K.bwd_matched(y, g, (0, na), (0, nz), acc)
        K.bwd_matched(y, g, (0, na), (3, nz - 2), acc[3:nz - 2])
        K.bwd_fdk(y, g, (0, na), (0, nz), acc)
        u2 = torch.empty_like(x)
        ss = torch.zeros(1, dtype=torch.float64, device=dev)
        K.tv_grad_sumsq(x, (0, nz), ss)
        K.tv_step(x, u2, 1e-3, ss, 1.0)
        # marching GD kernels (paired for even nx, single-voxel for odd nx):
        # gradient pass, fused pass, final stream step
        g1, g2, u3 = (torch.empty_like(x) for _ in range(3))
        s2 = torch.zeros_like(ss)
        K.tv_grad_store(x, g1, (1, nz - 1), ss)
        K.tv_gd_fused(x, g1, u2, g2, (1, nz - 1), 1e-3, ss, 1.0, s2)
        K.tv_step_g(u2, g2, u3, 1e-3, s2, 1.0)
        p3 = torch.zeros((3,) + tuple(x.shape), device=dev)
        q3 = torch.empty_like(p3)
        K.rof_iter(x, p3, q3, 0.1)
        K.rof_finish(x, q3, u2, 0.1)
    # FDK direct path: pixels much finer than voxels
    g = geometry(8, 8, 8, 300, 280, 2, pitch=(0.1, 0.1))
    y = torch.from_numpy(rng.standard_normal((2, 280, 300)).astype(
        np.float32)).to(dev)
    acc = torch.zeros((8, 8, 8), device=dev)
    K.bwd_fdk(y, g, (0, 2), (0, 8), acc)
    # matched Atb with strided lanes (fine pixels: lane stride 8)
    K.bwd_matched(y, g, (0, 2), (0, 8), acc)
    K.bwd_matched(y, g, (0, 2), (3, 5), acc[3:5])
    # matched Atb on 512^2 planes: 14-plane chunks with 72 KB boxes, x-major
    # views in the transposed frame (CS_ST_TRANSPOSE=0: in their own frame)
    g = geometry(512, 512, 4, 96, 12, 3)
    y = torch.from_numpy(rng.standard_normal((3, 12, 96)).astype(
        np.float32)).to(dev)
    acc = torch.zeros((4, 512, 512), device=dev)
    K.bwd_matched(y, g, (0, 3), (0, 4), acc)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
