"""CPU oracle for the cone-beam hot path -- TEST INFRASTRUCTURE ONLY.

Parity checker and CPU baseline ("kind": "port") for the B200 build.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module; the product package never
does (it fails loudly when its CUDA library is missing instead).

Contents, each restating the reference (/root/reference/pkg/src/conesplit):

* ``flat_geometry``  -- projectors.py:172-194 (per-angle src/det00/ustep/vstep)
* ``fwd_interp`` / ``bwd_matched`` / ``bwd_fdk`` / ``fwd_siddon`` -- the C
  restatement in cs_oracle.c of _kernels.py:213-275 / :278-337 / :340-398 /
  :154-191 with the float64 accumulators of projectors.py:246-348
* ``grad`` / ``div`` / ``tv_norm`` / ``tv_subgradient`` / ``minimize_tv_gradient``
  / ``minimize_rof`` / ``split_minimize`` -- regularization.py:88-280 (numpy)
* ``cgls`` / ``os_sart`` / ``fdk`` -- algorithms.py:146-304 (numpy, fp64 host
  vectors, monolithic operators: the reference's executor is bit-exact
  (backward) / 1e-7 (forward split) against monolithic)
* ``slab_ranges`` / ``even_angle_ranges`` / ``plan`` -- scheduler.py:158-210

Pinned against goldens produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libcs_oracle.so")
_lib = None


def build() -> str:
    """Compile the C restatement (gcc; no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i, d = ctypes.c_int, ctypes.c_double
        L.orc_fwd_interp.argtypes = [P, i, i, i, i, i, P, P, i, i, i, d, P, i]
        L.orc_bwd_matched.argtypes = [P, i, i, i, i, i, P, P, i, i, i, d, P, i]
        L.orc_bwd_fdk.argtypes = [P, i, i, i, i, P, P, i, d, d, d, d, d, d,
                                  i, i, P, i]
        L.orc_fwd_siddon.argtypes = [P, i, i, i, i, i, P, P, i, i, i, P, i]
        L.orc_ray_table.argtypes = [P, i, i, i, P, i, i, i, d, P, P, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") \
        else (os.cpu_count() or 1)


# --------------------------------------------------------------------------
# geometry (plain values, so the oracle does not depend on the product)


@dataclass(frozen=True)
class OGeom:
    dso: float
    dsd: float
    angles: tuple
    nx: int
    ny: int
    nz: int
    voxel: tuple = (1.0, 1.0, 1.0)
    offset: tuple = (0.0, 0.0, 0.0)
    nu: int = 1
    nv: int = 1
    pixel: tuple = (1.0, 1.0)
    det_offset: tuple = (0.0, 0.0)

    @property
    def n_angles(self):
        return len(self.angles)

    def grid6(self) -> np.ndarray:
        """geometry.py:55-68 min_corner + voxel sizes (projectors.py:197-202)."""
        ext = (self.nx * self.voxel[0], self.ny * self.voxel[1],
               self.nz * self.voxel[2])
        g0 = [self.offset[i] - 0.5 * ext[i] for i in range(3)]
        return np.array(g0 + list(self.voxel), dtype=np.float64)

    def step_max(self) -> float:
        """projectors.py:166-169."""
        return 0.5 * min(self.voxel)


def make_geo(n: int, n_angles: int, nu: int | None = None,
             nv: int | None = None) -> OGeom:
    """SURVEY 8(d) synthetic geometry: dso=2N, dsd=4N, pitch 2*sqrt(2)*N/Nu
    (the CLI default footprint cover, cli.py:122-130)."""
    nu = n if nu is None else nu
    nv = n if nv is None else nv
    dso, dsd = 2.0 * n, 4.0 * n
    mag = dsd / dso
    diag = math.sqrt(2.0 * n * n)
    pixel = (mag * diag / nu, mag * max(diag, float(n)) / nv)
    angles = tuple(float(a) for a in
                   np.linspace(0.0, 2 * math.pi, n_angles, endpoint=False))
    return OGeom(dso, dsd, angles, n, n, n, nu=nu, nv=nv, pixel=pixel)


def flat_geometry(g: OGeom, a0: int, a1: int) -> np.ndarray:
    """projectors.py:172-194, same numpy operation order -> [n, 12] f64."""
    n = a1 - a0
    out = np.empty((n, 12))
    du, dv = g.pixel
    off_u, off_v = g.det_offset
    for row, a in enumerate(range(a0, a1)):
        theta = g.angles[a]
        axis = np.array([math.cos(theta), math.sin(theta), 0.0])
        u_hat = np.array([-math.sin(theta), math.cos(theta), 0.0])
        v_hat = np.array([0.0, 0.0, 1.0])
        center = (g.dso - g.dsd) * axis
        u0 = (-0.5 * (g.nu - 1)) * du + off_u
        v0 = (-0.5 * (g.nv - 1)) * dv + off_v
        out[row, 0:3] = g.dso * axis
        out[row, 3:6] = center + u0 * u_hat + v0 * v_hat
        out[row, 6:9] = du * u_hat
        out[row, 9:12] = dv * v_hat
    return out


# --------------------------------------------------------------------------
# projectors (monolithic over an angle range; chunk-invariant in the reference)


def fwd_interp(vol: np.ndarray, g: OGeom, angle_range=None, slab=None,
               threads: int | None = None) -> np.ndarray:
    """forward_project_slab(..., INTERPOLATED), projectors.py:246-283."""
    a0, a1 = angle_range or (0, g.n_angles)
    z_lo, z_hi = slab or (0, g.nz)
    vol = np.ascontiguousarray(vol, dtype=np.float32)
    assert vol.shape == (z_hi - z_lo, g.ny, g.nx)
    geom = flat_geometry(g, a0, a1)
    grid = g.grid6()
    out = np.empty((a1 - a0, g.nv, g.nu), np.float32)
    lib().orc_fwd_interp(_ptr(vol), g.nx, g.ny, g.nz, z_lo, z_hi, _ptr(grid),
                         _ptr(geom), a1 - a0, g.nu, g.nv, g.step_max(),
                         _ptr(out), threads or default_threads())
    return out


def fwd_siddon(vol: np.ndarray, g: OGeom, angle_range=None, slab=None,
               threads: int | None = None) -> np.ndarray:
    """forward_project_slab(..., SIDDON), projectors.py:246-283."""
    a0, a1 = angle_range or (0, g.n_angles)
    z_lo, z_hi = slab or (0, g.nz)
    vol = np.ascontiguousarray(vol, dtype=np.float32)
    geom = flat_geometry(g, a0, a1)
    grid = g.grid6()
    out = np.empty((a1 - a0, g.nv, g.nu), np.float32)
    lib().orc_fwd_siddon(_ptr(vol), g.nx, g.ny, g.nz, z_lo, z_hi, _ptr(grid),
                         _ptr(geom), a1 - a0, g.nu, g.nv, _ptr(out),
                         threads or default_threads())
    return out


def bwd_matched(proj: np.ndarray, g: OGeom, angle_range=None, slab=None,
                acc: np.ndarray | None = None,
                threads: int | None = None) -> np.ndarray:
    """backproject_slab(..., MATCHED), projectors.py:318-348: f32 -> f64
    accumulator, kernel, cast back to f32."""
    a0, a1 = angle_range or (0, g.n_angles)
    z_lo, z_hi = slab or (0, g.nz)
    proj = np.ascontiguousarray(proj, dtype=np.float32)
    assert proj.shape == (a1 - a0, g.nv, g.nu)
    acc64 = (np.zeros((z_hi - z_lo, g.ny, g.nx)) if acc is None
             else np.asarray(acc, np.float32).astype(np.float64))
    geom = flat_geometry(g, a0, a1)
    grid = g.grid6()
    lib().orc_bwd_matched(_ptr(acc64), g.nx, g.ny, g.nz, z_lo, z_hi,
                          _ptr(grid), _ptr(geom), a1 - a0, g.nu, g.nv,
                          g.step_max(), _ptr(proj),
                          threads or default_threads())
    return acc64.astype(np.float32)


def bwd_fdk(proj: np.ndarray, g: OGeom, angle_range=None, slab=None,
            acc: np.ndarray | None = None,
            threads: int | None = None) -> np.ndarray:
    """backproject_slab(..., FDK), projectors.py:318-348 / :286-303."""
    a0, a1 = angle_range or (0, g.n_angles)
    z_lo, z_hi = slab or (0, g.nz)
    proj = np.ascontiguousarray(proj, dtype=np.float32)
    acc64 = (np.zeros((z_hi - z_lo, g.ny, g.nx)) if acc is None
             else np.asarray(acc, np.float32).astype(np.float64))
    thetas = np.array(g.angles[a0:a1])
    cs = np.ascontiguousarray(np.stack([np.cos(thetas), np.sin(thetas)], 1))
    grid = g.grid6()
    lib().orc_bwd_fdk(_ptr(acc64), g.nx, g.ny, z_hi - z_lo, z_lo, _ptr(grid),
                      _ptr(cs), a1 - a0, g.dso, g.dsd, g.pixel[0], g.pixel[1],
                      g.det_offset[0], g.det_offset[1], g.nu, g.nv,
                      _ptr(proj), threads or default_threads())
    return acc64.astype(np.float32)


def ray_table(g: OGeom, angle_range=None):
    """(t0, step, n_steps) per ray, _kernels.py:194-210."""
    a0, a1 = angle_range or (0, g.n_angles)
    geom = flat_geometry(g, a0, a1)
    grid = g.grid6()
    shape = (a1 - a0, g.nv, g.nu)
    t0 = np.empty(shape)
    st = np.empty(shape)
    n = np.empty(shape, np.int64)
    lib().orc_ray_table(_ptr(grid), g.nx, g.ny, g.nz, _ptr(geom), a1 - a0,
                        g.nu, g.nv, g.step_max(), _ptr(t0), _ptr(st), _ptr(n))
    return t0, st, n


# --------------------------------------------------------------------------
# TV (regularization.py:88-280), numpy, float64

TV_SMOOTH_EPS = 1e-8
ROF_DUAL_STEP = 1.0 / 12.0
ZERO_NORM = 1e-30


def grad(u):
    """regularization.py:88-95 forward differences, zero last plane."""
    gz = np.zeros_like(u)
    gy = np.zeros_like(u)
    gx = np.zeros_like(u)
    gz[:-1] = u[1:] - u[:-1]
    gy[:, :-1] = u[:, 1:] - u[:, :-1]
    gx[:, :, :-1] = u[:, :, 1:] - u[:, :, :-1]
    return gz, gy, gx


def div(pz, py, px):
    """regularization.py:98-110 negative adjoint of grad."""
    out = np.zeros_like(pz)
    out[0] = pz[0]
    out[1:-1] = pz[1:-1] - pz[:-2]
    out[-1] = -pz[-2]
    out[:, 0] += py[:, 0]
    out[:, 1:-1] += py[:, 1:-1] - py[:, :-2]
    out[:, -1] += -py[:, -2]
    out[:, :, 0] += px[:, :, 0]
    out[:, :, 1:-1] += px[:, :, 1:-1] - px[:, :, :-2]
    out[:, :, -1] += -px[:, :, -2]
    return out


def tv_norm(vol) -> float:
    """regularization.py:119-124."""
    gz, gy, gx = grad(np.asarray(vol, np.float32).astype(np.float64))
    return float(np.sum(np.sqrt(gz * gz + gy * gy + gx * gx)))


def tv_subgradient(u):
    """regularization.py:127-130."""
    gz, gy, gx = grad(u)
    mag = np.sqrt(gz * gz + gy * gy + gx * gx + TV_SMOOTH_EPS)
    return -div(gz / mag, gy / mag, gx / mag)


def minimize_tv_gradient(vol, inner_iters: int, step: float) -> np.ndarray:
    """regularization.py:133-151."""
    u = np.asarray(vol, np.float32).astype(np.float64)
    for _ in range(inner_iters):
        g = tv_subgradient(u)
        norm = np.sqrt(np.sum(g * g))
        if norm < ZERO_NORM:
            break
        u -= step * g / norm
    return u.astype(np.float32)


def rof_iterate(f, p, lam):
    """regularization.py:174-182."""
    u = f + lam * div(p[0], p[1], p[2])
    gz, gy, gx = grad(u)
    p[0] += (ROF_DUAL_STEP / lam) * gz
    p[1] += (ROF_DUAL_STEP / lam) * gy
    p[2] += (ROF_DUAL_STEP / lam) * gx
    mag = np.sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2])
    np.maximum(mag, 1.0, out=mag)
    p /= mag


def minimize_rof(vol, inner_iters: int, lam: float) -> np.ndarray:
    """regularization.py:154-171."""
    f = np.asarray(vol, np.float32).astype(np.float64)
    p = np.zeros((3,) + f.shape)
    for _ in range(inner_iters):
        rof_iterate(f, p, lam)
    return (f + lam * div(p[0], p[1], p[2])).astype(np.float32)


def make_halo_slabs(n_z: int, n_slabs: int, d: int):
    """regularization.py:185-194 -> list of (core, window)."""
    size = -(-n_z // n_slabs)
    return [((z0, min(z0 + size, n_z)),
             (max(0, z0 - d), min(n_z, min(z0 + size, n_z) + d)))
            for z0 in range(0, n_z, size)]


def split_minimize(vol, n_slabs: int, minimizer: str, outer_syncs: int,
                   inner_iters: int, step: float = 1e-3, lam: float = 0.1,
                   exact_global: bool = True, halo: int | None = None):
    """regularization.py:213-280 with an explicit slab count."""
    d = inner_iters if halo is None else halo
    slabs = make_halo_slabs(vol.shape[0], n_slabs, d)
    if minimizer == "gd":
        u = np.asarray(vol, np.float32).astype(np.float64)
        total_voxels = u.size
        for _ in range(outer_syncs):
            snap = u.copy()
            local = [snap[w0:w1].copy() for _, (w0, w1) in slabs]
            for _ in range(inner_iters):
                grads = [tv_subgradient(w) for w in local]
                if exact_global:
                    total = 0.0
                    for ((z0, z1), (w0, _)), gg in zip(slabs, grads):
                        core = gg[z0 - w0:z1 - w0]
                        total += np.sum(core * core)
                    norms = [np.sqrt(total)] * len(slabs)
                else:
                    norms = [np.sqrt(np.sum(gg * gg)) *
                             np.sqrt(total_voxels / w.size)
                             for w, gg in zip(local, grads)]
                for w, gg, nrm in zip(local, grads, norms):
                    if nrm >= ZERO_NORM:
                        w -= step * gg / nrm
            for ((z0, z1), (w0, _)), w in zip(slabs, local):
                u[z0:z1] = w[z0 - w0:z1 - w0]
        return u.astype(np.float32)
    f = np.asarray(vol, np.float32).astype(np.float64)
    p = np.zeros((3,) + f.shape)
    for _ in range(outer_syncs):
        p_snap = p.copy()
        for (z0, z1), (w0, w1) in slabs:
            f_loc = f[w0:w1]
            p_loc = p_snap[:, w0:w1].copy()
            for _ in range(inner_iters):
                rof_iterate(f_loc, p_loc, lam)
            p[:, z0:z1] = p_loc[:, z0 - w0:z1 - w0]
    return (f + lam * div(p[0], p[1], p[2])).astype(np.float32)


# --------------------------------------------------------------------------
# planner (scheduler.py:158-210)


def slab_ranges(n_z: int, n_splits: int):
    size = -(-n_z // n_splits)
    return tuple((z0, min(z0 + size, n_z)) for z0 in range(0, n_z, size))


def even_angle_ranges(n_angles: int, n_devices: int):
    b = [n_angles * k // n_devices for k in range(n_devices + 1)]
    return tuple((b[k], b[k + 1]) for k in range(n_devices))


def plan(op: str, g: OGeom, budgets, chunk_angles: int,
         usable_fraction: float = 0.95):
    """scheduler.py:169-210 -> dict of the SplitPlan fields."""
    n_angles = g.n_angles
    chunk = min(chunk_angles, n_angles)
    plane = g.nx * g.ny * 4
    chunk_bytes = chunk * g.nu * g.nv * 4
    usable = usable_fraction * min(budgets)
    if op == "forward" and g.nz * plane + 2 * chunk_bytes <= usable:
        n_splits, buffers = 1, 2
    else:
        buffers = 3 if op == "forward" else 2
        if op == "backward" and g.nz * plane + 2 * chunk_bytes <= usable:
            n_splits = 1
        else:
            max_slices = int((usable - buffers * chunk_bytes) // plane)
            if max_slices < 1:
                raise ValueError("infeasible")
            n_splits = -(-g.nz // max_slices)
    ranges = slab_ranges(g.nz, n_splits)
    peak = max(z1 - z0 for z0, z1 in ranges) * plane
    if op == "forward":
        assign = even_angle_ranges(n_angles, len(budgets))
    else:
        assign = tuple((c0, min(c0 + chunk, n_angles))
                       for c0 in range(0, n_angles, chunk))
    return dict(n_splits=n_splits, slab_ranges=ranges,
                angle_assignment=assign, chunk_angles=chunk,
                buffer_count=buffers,
                pin_host_image=(n_splits > 1) or len(budgets) > 2,
                per_device_bytes_peak=peak + buffers * chunk_bytes)


# --------------------------------------------------------------------------
# loops (algorithms.py), fp64 host vectors like the reference

INVERSE_GUARD = 1e-8
CG_BREAKDOWN = 1e-30


def _fwd64(x, g, ar=None, threads=None):
    return fwd_interp(x.astype(np.float32), g, ar, threads=threads
                      ).astype(np.float64)


def _bwd64(y, g, ar=None, threads=None):
    return bwd_matched(y.astype(np.float32), g, ar, threads=threads
                       ).astype(np.float64)


def cgls(b, g: OGeom, iterations: int, threads=None):
    """algorithms.py:204-246 -> (x f32, residuals, breakdown)."""
    b = np.asarray(b, np.float32).astype(np.float64)
    b_norm = float(np.linalg.norm(b))
    x = np.zeros((g.nz, g.ny, g.nx))
    res = []
    if b_norm == 0.0:
        return x.astype(np.float32), res, False
    r = b.copy()
    s = _bwd64(r, g, threads=threads)
    p = s.copy()
    gamma = float(np.vdot(s, s).real)
    breakdown = False
    for _ in range(iterations):
        q = _fwd64(p, g, threads=threads)
        delta = float(np.vdot(q, q).real)
        if delta < CG_BREAKDOWN or gamma < CG_BREAKDOWN:
            breakdown = True
            break
        alpha = gamma / delta
        x += alpha * p
        r -= alpha * q
        res.append(float(np.linalg.norm(r)) / b_norm)
        s = _bwd64(r, g, threads=threads)
        gamma_new = float(np.vdot(s, s).real)
        beta = gamma_new / gamma
        p = s + beta * p
        gamma = gamma_new
    return x.astype(np.float32), res, breakdown


def angle_blocks(n_angles: int, block_size: int):
    """algorithms.py:249-251."""
    return [(b0, min(b0 + block_size, n_angles))
            for b0 in range(0, n_angles, block_size)]


def guarded_inverse(a):
    """algorithms.py:254-258."""
    out = np.zeros_like(a)
    m = a >= INVERSE_GUARD
    out[m] = 1.0 / a[m]
    return out


def os_sart(b, g: OGeom, iterations: int, block_size: int,
            relaxation: float = 1.0, tv: dict | None = None, threads=None):
    """algorithms.py:261-304.  ``tv`` = kwargs of split_minimize (with
    n_slabs) applied once per outer iteration."""
    blocks = angle_blocks(g.n_angles, block_size)
    ones = np.ones((g.nz, g.ny, g.nx), np.float32)
    weights = []
    for b0, b1 in blocks:
        row = fwd_interp(ones, g, (b0, b1), threads=threads).astype(np.float64)
        col = bwd_matched(np.ones((b1 - b0, g.nv, g.nu), np.float32), g,
                          (b0, b1), threads=threads).astype(np.float64)
        weights.append((guarded_inverse(row), guarded_inverse(col)))
    b = np.asarray(b, np.float32).astype(np.float64)
    x = np.zeros((g.nz, g.ny, g.nx))
    for _ in range(iterations):
        for (b0, b1), (w, v) in zip(blocks, weights):
            resid = b[b0:b1] - _fwd64(x, g, (b0, b1), threads)
            upd = _bwd64(w * resid, g, (b0, b1), threads)
            x += relaxation * v * upd
        if tv is not None:
            x = split_minimize(x.astype(np.float32), **tv).astype(np.float64)
    return x.astype(np.float32)


def ramp_filter_rows(data, spacing):
    """algorithms.py:146-163."""
    n = data.shape[-1]
    pad = 1 << (2 * n - 1).bit_length()
    kernel = np.zeros(pad)
    kernel[0] = 1.0 / (4.0 * spacing * spacing)
    k = np.arange(1, pad // 2 + 1)
    odd = k[k % 2 == 1]
    kernel[odd] = -1.0 / (math.pi * odd * spacing) ** 2
    kernel[pad - odd] = kernel[odd]
    padded = np.zeros(data.shape[:-1] + (pad,))
    padded[..., :n] = data
    filtered = np.fft.irfft(np.fft.rfft(padded) * np.fft.rfft(kernel), pad)
    return filtered[..., :n] * spacing


def fdk(proj, g: OGeom, threads=None):
    """algorithms.py:166-201 (monolithic backward)."""
    du, dv = g.pixel
    off_u, off_v = g.det_offset
    u_pos = (np.arange(g.nu) - 0.5 * (g.nu - 1)) * du + off_u
    v_pos = (np.arange(g.nv) - 0.5 * (g.nv - 1)) * dv + off_v
    cosw = g.dsd / np.sqrt(g.dsd ** 2 + u_pos[None, :] ** 2
                           + v_pos[:, None] ** 2)
    weighted = np.asarray(proj, np.float32).astype(np.float64) * cosw[None]
    filt = ramp_filter_rows(weighted, du * g.dso / g.dsd)
    angles = np.asarray(g.angles)
    step = (2.0 * math.pi if len(angles) < 2
            else float(np.mean(np.diff(np.sort(angles)))))
    filt *= 0.5 * step
    return bwd_fdk(filt.astype(np.float32), g, threads=threads)
