"""Kernel-level drop-in: the four numba kernels of
the reference (/root/reference/pkg/src/conesplit/_kernels.py:154, :213,
:278, :340) re-implemented over the sm_100a C-ABI with the SAME names,
signatures and in-place semantics, so that

    import conesplit._kernels as ref_kernels
    from paper_1905_03748_b200 import refhook
    refhook.install(ref_kernels)

runs the reference's own operators, executor and loops on the GPU (the
reference calls the kernels through the module attribute, projectors.py:272,
:277, :300, :310).  Arguments are the reference's host arrays; each call
uploads its inputs, launches, and writes the result back into ``out`` /
adds it into the float64 accumulator ``vol64`` (the reference's host-side
fp64 slab, which a device-resident caller would not need).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import check, lib

__all__ = ["interp_forward_chunk", "siddon_forward_chunk",
           "matched_backward_chunk", "fdk_backward_chunk", "install",
           "HOOKS"]


def _dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _geom12(srcs, det00, ustep, vstep) -> np.ndarray:
    """[n_a, 12] = src | det00 | ustep | vstep (the C-ABI's layout)."""
    return np.ascontiguousarray(np.hstack([np.asarray(srcs, np.float64),
                                           np.asarray(det00, np.float64),
                                           np.asarray(ustep, np.float64),
                                           np.asarray(vstep, np.float64)]))


def _grid6(gx0, gy0, gz0, vx, vy, vz) -> np.ndarray:
    return np.array([gx0, gy0, gz0, vx, vy, vz], dtype=np.float64)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data_as(ctypes.c_void_p).value


def interp_forward_chunk(vol, srcs, det00, ustep, vstep,
                         gx0, gy0, gz0, vx, vy, vz, nx, ny, nz, z_lo, z_hi,
                         step_max, tile_u, tile_v, out):
    """_kernels.py:213-275: out[a, v, u] = interpolated Ax of the slab
    vol[z_lo:z_hi] (tiles are a CPU scheduling detail and ignored)."""
    del tile_u, tile_v
    n_a, n_v, n_u = out.shape
    geom = _geom12(srcs, det00, ustep, vstep)
    g6 = _grid6(gx0, gy0, gz0, vx, vy, vz)
    dv = _dev(vol)
    do = torch.empty((n_a, n_v, n_u), dtype=torch.float32, device="cuda")
    check(lib().cs_fwd_interp(dv.data_ptr(), int(nx), int(ny), int(nz),
                              int(z_lo), int(z_hi), _ptr(g6), _ptr(geom),
                              n_a, n_u, n_v, float(step_max), do.data_ptr(),
                              0, _stream()))
    out[...] = do.cpu().numpy()


def siddon_forward_chunk(vol, srcs, det00, ustep, vstep,
                         gx0, gy0, gz0, vx, vy, vz, nx, ny, nz, z_lo, z_hi,
                         tile_u, tile_v, out):
    """_kernels.py:154-191: Siddon (exact intersection-length) Ax."""
    del tile_u, tile_v
    n_a, n_v, n_u = out.shape
    geom = _geom12(srcs, det00, ustep, vstep)
    g6 = _grid6(gx0, gy0, gz0, vx, vy, vz)
    dv = _dev(vol)
    do = torch.empty((n_a, n_v, n_u), dtype=torch.float32, device="cuda")
    check(lib().cs_fwd_siddon(dv.data_ptr(), int(nx), int(ny), int(nz),
                              int(z_lo), int(z_hi), _ptr(g6), _ptr(geom),
                              n_a, n_u, n_v, do.data_ptr(), 0, _stream()))
    out[...] = do.cpu().numpy()


def matched_backward_chunk(vol64, proj, srcs, det00, ustep, vstep,
                           gx0, gy0, gz0, vx, vy, vz, nx, ny, nz,
                           z_lo, z_hi, step_max):
    """_kernels.py:278-337: vol64 += A^T proj over the slab (exact adjoint
    of interp_forward_chunk); the device accumulates in fp32."""
    n_a, n_v, n_u = proj.shape
    geom = _geom12(srcs, det00, ustep, vstep)
    g6 = _grid6(gx0, gy0, gz0, vx, vy, vz)
    dp = _dev(proj)
    acc = torch.zeros((int(z_hi) - int(z_lo), int(ny), int(nx)),
                      dtype=torch.float32, device="cuda")
    check(lib().cs_bwd_matched(acc.data_ptr(), int(nx), int(ny), int(nz),
                               int(z_lo), int(z_hi), _ptr(g6), _ptr(geom),
                               n_a, n_u, n_v, float(step_max), dp.data_ptr(),
                               _stream()))
    vol64 += acc.cpu().numpy()


def fdk_backward_chunk(vol64, proj, coss, sins, dso, dsd,
                       du, dv, off_u, off_v,
                       gx0, gy0, gz0, vx, vy, vz, z_lo,
                       tile_x, tile_y):
    """_kernels.py:340-398: vol64 += FDK-weighted (dso/U)^2 bilinear
    backprojection over the slab vol64 (shape (z_hi - z_lo, ny, nx))."""
    del tile_x, tile_y
    n_a, n_v, n_u = proj.shape
    n_slab, ny, nx = vol64.shape
    cs_tab = np.ascontiguousarray(np.stack([np.asarray(coss, np.float64),
                                            np.asarray(sins, np.float64)], 1))
    g6 = _grid6(gx0, gy0, gz0, vx, vy, vz)
    dp = _dev(proj)
    acc = torch.zeros((n_slab, ny, nx), dtype=torch.float32, device="cuda")
    check(lib().cs_bwd_fdk(acc.data_ptr(), nx, ny, int(z_lo), n_slab,
                           _ptr(g6), _ptr(cs_tab), n_a, float(dso),
                           float(dsd), float(du), float(dv), float(off_u),
                           float(off_v), n_u, n_v, dp.data_ptr(), _stream()))
    vol64 += acc.cpu().numpy()


HOOKS = {f.__name__: f for f in (interp_forward_chunk, siddon_forward_chunk,
                                 matched_backward_chunk, fdk_backward_chunk)}


def install(module) -> dict:
    """Replace the four kernels on ``module`` (the reference's
    ``conesplit._kernels``); returns the originals so callers can restore
    them (``for k, v in old.items(): setattr(module, k, v)``)."""
    old = {}
    for name, fn in HOOKS.items():
        old[name] = getattr(module, name, None)
        setattr(module, name, fn)
    return old
