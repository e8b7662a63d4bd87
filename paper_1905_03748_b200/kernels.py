"""Thin typed wrappers over the C-ABI (one function per entry point).

Arguments are torch CUDA tensors (device buffers) plus host geometry;
every call is enqueued on ``stream`` (default: torch's current stream) and
never synchronises the host.  These are the building blocks the operator
layer (projectors, execution, regularization, algorithms) is written in.
"""

from __future__ import annotations

import numpy as np
import torch

from ._lib import check, dptr, hptr, lib, stream_ptr
from .geometry import ScanGeometry, VoxelGrid, flat_geometry, grid6

MAX_ANGLES_PER_LAUNCH = 65535  # grid.z limit of the ray kernels


def _checked_retry_oom(call):
    """check(call()); if the library ran out of device memory (its texture
    arrays and stream-ordered tables are allocated outside torch), release
    torch's cached blocks and the library's cached texture arrays, then
    retry once.  The C-ABI allocates before it launches anything, so a
    failed call left no partial result."""
    rc = call()
    if rc != 0:
        msg = lib().cs_last_error().decode()
        if "out of memory" in msg:
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            check(lib().cs_release_cache())
            rc = call()
    check(rc)


def release_cache() -> None:
    """Free the library's cached texture arrays on the current device."""
    check(lib().cs_release_cache())


def launch_count() -> int:
    """Kernels the library has launched since it was loaded."""
    return int(lib().cs_launch_count())


def _f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    return t


def _angle_chunks(a0: int, a1: int):
    for c0 in range(a0, a1, MAX_ANGLES_PER_LAUNCH):
        yield c0, min(a1, c0 + MAX_ANGLES_PER_LAUNCH)


def fwd_interp(vol: torch.Tensor, geometry: ScanGeometry, angle_range,
               slab_range, out: torch.Tensor, accumulate: bool = False,
               stream=None) -> torch.Tensor:
    """K1: out[a - a0] (+)= step * sum trilinear(vol) for a in angle_range.
    vol holds grid slices slab_range."""
    grid = geometry.voxel_grid
    det = geometry.detector
    z_lo, z_hi = slab_range
    a0, a1 = angle_range
    _f32(vol, "vol")
    _f32(out, "out")
    assert vol.shape == (z_hi - z_lo, grid.n_y, grid.n_x), vol.shape
    assert out.shape == (a1 - a0, det.n_v, det.n_u), out.shape
    g6 = grid6(grid)
    step = 0.5 * min(grid.voxel_size)
    L = lib()
    for c0, c1 in _angle_chunks(a0, a1):
        geom = flat_geometry(geometry, c0, c1)
        _checked_retry_oom(lambda: L.cs_fwd_interp(
            dptr(vol), grid.n_x, grid.n_y, grid.n_z, z_lo, z_hi, hptr(g6),
            hptr(geom), c1 - c0, det.n_u, det.n_v, step,
            dptr(out[c0 - a0:c1 - a0]), int(accumulate), stream_ptr(stream)))
    return out


def fwd_interp_residual(vol: torch.Tensor, geometry: ScanGeometry,
                        angle_range, b: torch.Tensor, w: torch.Tensor | None,
                        out: torch.Tensor, stream=None) -> torch.Tensor:
    """out = w * (b - A vol) over angle_range (full volume)."""
    grid = geometry.voxel_grid
    det = geometry.detector
    a0, a1 = angle_range
    _f32(vol, "vol")
    _f32(out, "out")
    _f32(b, "b")
    g6 = grid6(grid)
    step = 0.5 * min(grid.voxel_size)
    L = lib()
    for c0, c1 in _angle_chunks(a0, a1):
        geom = flat_geometry(geometry, c0, c1)
        sl = slice(c0 - a0, c1 - a0)
        _checked_retry_oom(lambda: L.cs_fwd_interp_residual(
            dptr(vol), grid.n_x, grid.n_y, grid.n_z, hptr(g6), hptr(geom),
            c1 - c0, det.n_u, det.n_v, step, dptr(b[sl]),
            None if w is None else dptr(w[sl]), dptr(out[sl]),
            stream_ptr(stream)))
    return out


def fwd_siddon(vol: torch.Tensor, geometry: ScanGeometry, angle_range,
               slab_range, out: torch.Tensor, accumulate: bool = False,
               stream=None) -> torch.Tensor:
    """K4: exact-intersection forward projection of a slab."""
    grid = geometry.voxel_grid
    det = geometry.detector
    z_lo, z_hi = slab_range
    a0, a1 = angle_range
    _f32(vol, "vol")
    _f32(out, "out")
    g6 = grid6(grid)
    L = lib()
    for c0, c1 in _angle_chunks(a0, a1):
        geom = flat_geometry(geometry, c0, c1)
        check(L.cs_fwd_siddon(
            dptr(vol), grid.n_x, grid.n_y, grid.n_z, z_lo, z_hi, hptr(g6),
            hptr(geom), c1 - c0, det.n_u, det.n_v,
            dptr(out[c0 - a0:c1 - a0]), int(accumulate), stream_ptr(stream)))
    return out


def bwd_matched(proj: torch.Tensor, geometry: ScanGeometry, angle_range,
                slab_range, vol_acc: torch.Tensor,
                stream=None) -> torch.Tensor:
    """K2: vol_acc += A^T proj restricted to slab_range (exact adjoint)."""
    grid = geometry.voxel_grid
    det = geometry.detector
    z_lo, z_hi = slab_range
    a0, a1 = angle_range
    _f32(proj, "proj")
    _f32(vol_acc, "vol_acc")
    assert vol_acc.shape == (z_hi - z_lo, grid.n_y, grid.n_x)
    assert proj.shape == (a1 - a0, det.n_v, det.n_u)
    g6 = grid6(grid)
    step = 0.5 * min(grid.voxel_size)
    L = lib()
    for c0, c1 in _angle_chunks(a0, a1):
        geom = flat_geometry(geometry, c0, c1)
        check(L.cs_bwd_matched(
            dptr(vol_acc), grid.n_x, grid.n_y, grid.n_z, z_lo, z_hi,
            hptr(g6), hptr(geom), c1 - c0, det.n_u, det.n_v, step,
            dptr(proj[c0 - a0:c1 - a0]), stream_ptr(stream)))
    return vol_acc


def set_deterministic(on: bool) -> None:
    """Bit-reproducible matched Atb (int64 fixed-point accumulation; see
    cs_set_deterministic) for every later bwd_matched in this process."""
    check(lib().cs_set_deterministic(int(bool(on))))


def bwd_fdk(proj: torch.Tensor, geometry: ScanGeometry, angle_range,
            slab_range, vol_acc: torch.Tensor, stream=None) -> torch.Tensor:
    """K3: vol_acc += FDK-weighted backprojection (dso/U)^2 * bilinear."""
    grid = geometry.voxel_grid
    det = geometry.detector
    z_lo, z_hi = slab_range
    a0, a1 = angle_range
    _f32(proj, "proj")
    _f32(vol_acc, "vol_acc")
    assert vol_acc.shape == (z_hi - z_lo, grid.n_y, grid.n_x)
    thetas = np.asarray(geometry.angles[a0:a1])
    cs = np.ascontiguousarray(np.stack([np.cos(thetas), np.sin(thetas)], 1))
    g6 = grid6(grid)
    du, dv = det.pixel_size
    off_u, off_v = det.detector_offset
    check(lib().cs_bwd_fdk(
        dptr(vol_acc), grid.n_x, grid.n_y, z_lo, z_hi - z_lo, hptr(g6),
        hptr(cs), a1 - a0, float(geometry.dso), float(geometry.dsd),
        float(du), float(dv), float(off_u), float(off_v), det.n_u, det.n_v,
        dptr(proj), stream_ptr(stream)))
    return vol_acc


def ray_table(geometry: ScanGeometry, angle_range, stream=None):
    """(t0, step, n) per ray from the device's fp64 set-up."""
    grid = geometry.voxel_grid
    det = geometry.detector
    a0, a1 = angle_range
    shape = (a1 - a0, det.n_v, det.n_u)
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = torch.empty(shape, dtype=torch.float64, device=dev)
    st = torch.empty_like(t0)
    n = torch.empty(shape, dtype=torch.int64, device=dev)
    geom = flat_geometry(geometry, a0, a1)
    g6 = grid6(grid)
    check(lib().cs_ray_table(
        grid.n_x, grid.n_y, grid.n_z, hptr(g6), hptr(geom), a1 - a0, det.n_u,
        det.n_v, 0.5 * min(grid.voxel_size), dptr(t0), dptr(st), dptr(n),
        stream_ptr(stream)))
    return t0, st, n


# ---------------------------------------------------------------- TV ----

def tv_grad_sumsq(u: torch.Tensor, core, out: torch.Tensor, stream=None):
    nz, ny, nx = u.shape
    check(lib().cs_tv_grad_sumsq(dptr(_f32(u, "u")), nx, ny, nz, core[0],
                                 core[1], dptr(out), stream_ptr(stream)))
    return out


def tv_grad_store(u: torch.Tensor, g: torch.Tensor, core, out: torch.Tensor,
                  stream=None):
    """g = TV subgradient over the whole window; out[0] = Σg² over the
    core planes (the first pass of a GD iteration, g kept for the step)."""
    nz, ny, nx = u.shape
    check(lib().cs_tv_grad_store(dptr(_f32(u, "u")), dptr(_f32(g, "g")), nx,
                                 ny, nz, core[0], core[1], dptr(out),
                                 stream_ptr(stream)))
    return g


def tv_step_g(u: torch.Tensor, g: torch.Tensor, u_out: torch.Tensor,
              step: float, sumsq: torch.Tensor, scale: float = 1.0,
              stream=None):
    """u_out = u - step g / (sqrt(sumsq) scale) (bit-identical to tv_step)."""
    check(lib().cs_tv_step_g(dptr(_f32(u, "u")), dptr(_f32(g, "g")),
                             dptr(_f32(u_out, "u_out")), u.numel(), step,
                             dptr(sumsq), scale, stream_ptr(stream)))
    return u_out


def tv_gd_fused(u: torch.Tensor, g: torch.Tensor, u_out: torch.Tensor,
                g_out: torch.Tensor, core, step: float, sumsq: torch.Tensor,
                scale: float, out: torch.Tensor, stream=None):
    """One GD iteration after the first in one pass: u_out = u - step g /
    (sqrt(sumsq) scale); g_out = TV subgradient of u_out; out[0] = Σg_out²
    over the core planes (= tv_step_g then tv_grad_store, bit for bit)."""
    nz, ny, nx = u.shape
    check(lib().cs_tv_gd_fused(dptr(_f32(u, "u")), dptr(_f32(g, "g")),
                               dptr(_f32(u_out, "u_out")),
                               dptr(_f32(g_out, "g_out")), nx, ny, nz,
                               core[0], core[1], float(step), dptr(sumsq),
                               float(scale), dptr(out), stream_ptr(stream)))
    return u_out


def tv_grad_norm(u: torch.Tensor, core, out: torch.Tensor, stream=None):
    """out[0] = ||g||_2 over the core planes (regularization.py:147)."""
    nz, ny, nx = u.shape
    check(lib().cs_tv_grad_norm(dptr(_f32(u, "u")), nx, ny, nz, core[0],
                                core[1], dptr(out), stream_ptr(stream)))
    return out


def tv_step(u: torch.Tensor, u_out: torch.Tensor, step: float,
            sumsq: torch.Tensor, scale: float = 1.0, stream=None):
    nz, ny, nx = u.shape
    check(lib().cs_tv_step(dptr(_f32(u, "u")), dptr(_f32(u_out, "u_out")),
                           nx, ny, nz, float(step), dptr(sumsq),
                           float(scale), stream_ptr(stream)))
    return u_out


def rof_iter(f: torch.Tensor, p_in: torch.Tensor, p_out: torch.Tensor,
             lam: float, stream=None):
    nz, ny, nx = f.shape
    check(lib().cs_rof_iter(dptr(_f32(f, "f")), dptr(_f32(p_in, "p_in")),
                            dptr(_f32(p_out, "p_out")), nx, ny, nz,
                            float(lam), stream_ptr(stream)))
    return p_out


def rof_finish(f: torch.Tensor, p: torch.Tensor, u: torch.Tensor,
               lam: float, stream=None):
    nz, ny, nx = f.shape
    check(lib().cs_rof_finish(dptr(_f32(f, "f")), dptr(_f32(p, "p")),
                              dptr(_f32(u, "u")), nx, ny, nz, float(lam),
                              stream_ptr(stream)))
    return u


def tv_norm(u: torch.Tensor, out: torch.Tensor, stream=None):
    nz, ny, nx = u.shape
    check(lib().cs_tv_norm(dptr(_f32(u, "u")), nx, ny, nz, dptr(out),
                           stream_ptr(stream)))
    return out


# ------------------------------------------------------- vector algebra --

def dot(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, stream=None):
    check(lib().cs_dot(dptr(a), dptr(b), a.numel(), dptr(out),
                       stream_ptr(stream)))
    return out


def axpy_ratio(y, x, num, den, sign: float, stream=None):
    check(lib().cs_axpy_ratio(dptr(y), dptr(x), y.numel(), dptr(num),
                              dptr(den), float(sign), stream_ptr(stream)))


def xpay_ratio(p, s, num, den, stream=None):
    check(lib().cs_xpay_ratio(dptr(p), dptr(s), p.numel(), dptr(num),
                              dptr(den), stream_ptr(stream)))


def guarded_inverse(a, out, stream=None):
    check(lib().cs_guarded_inverse(dptr(a), dptr(out), a.numel(),
                                   stream_ptr(stream)))
    return out


def sart_update(x, upd, v, lam: float, stream=None):
    check(lib().cs_sart_update(dptr(x), dptr(upd), dptr(v), float(lam),
                               x.numel(), stream_ptr(stream)))


def weighted_residual(r, b, w, stream=None):
    """r = w * (b - r) elementwise (w None: r = b - r)."""
    check(lib().cs_weighted_residual(dptr(r), dptr(b),
                                     None if w is None else dptr(w),
                                     r.numel(), stream_ptr(stream)))
    return r


def sum_slices(src: torch.Tensor, out: torch.Tensor,
               b: torch.Tensor | None = None, w: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    """out = sum_k src[k] in k order (src: (n_src,) + out.shape, each
    slice contiguous); with b: out = b - sum, with b and w: w * (b - sum)."""
    n = out.numel()
    _f32(out, "out")
    assert src.shape[1:] == out.shape, (src.shape, out.shape)
    assert src.shape[0] >= 1 and src.dtype == torch.float32
    assert src.shape[0] == 1 or src.stride(0) >= n
    for t, name in ((b, "b"), (w, "w")):
        if t is not None:
            _f32(t, name)
            assert t.shape == out.shape
    check(lib().cs_sum_slices(dptr(src[0]), src.shape[0], src.stride(0), n,
                              None if b is None else dptr(b),
                              None if w is None else dptr(w), dptr(out),
                              stream_ptr(stream)))
    return out


def peer_enable(device_index: int) -> None:
    """Let kernels on the current device reach memory of ``device_index``."""
    check(lib().cs_peer_enable(int(device_index)))


def fill(x, value: float, stream=None):
    check(lib().cs_fill(dptr(x), float(value), x.numel(), stream_ptr(stream)))
    return x


def grid_of(geometry_or_grid) -> VoxelGrid:
    return (geometry_or_grid.voxel_grid
            if isinstance(geometry_or_grid, ScanGeometry) else geometry_or_grid)
