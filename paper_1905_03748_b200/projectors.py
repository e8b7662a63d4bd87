"""Operators over one in-memory slab: the drop-in for conesplit.projectors
(/root/reference/pkg/src/conesplit/projectors.py).

Same names, signatures, defaults and errors as the reference
(boundary B2 of SURVEY 8(b)).  Data containers accept either host numpy
arrays (the reference's representation) or torch CUDA tensors
(device-resident, the B200-native representation); operators return the
representation they were given, so a numpy caller sees the reference's
behaviour and a device caller never leaves HBM.

The compute always runs in the sm_100a kernels (kernels.py -> C-ABI); there
is no CPU path.  Tile specs are accepted for API compatibility: the
reference's results are tile- and chunk-invariant and the
GPU launch shape is chosen for the hardware, not taken from them.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from ._lib import lib
from .geometry import DetectorGrid, Ray, ScanGeometry, VoxelGrid

__all__ = [
    "Volume",
    "ProjectionStack",
    "ForwardTileSpec",
    "BackwardTileSpec",
    "WeightMode",
    "ProjectionMethod",
    "siddon_trace",
    "forward_project_slab",
    "backproject_chunk_into",
    "backproject_slab",
    "sample_step",
    "to_device",
    "to_host",
]

DTYPE = np.float32


class WeightMode(enum.Enum):
    """projectors.py:39-44."""
    FDK = "fdk"
    MATCHED = "matched"


class ProjectionMethod(enum.Enum):
    """projectors.py:47-49."""
    SIDDON = "siddon"
    INTERPOLATED = "interpolated"


@dataclass(frozen=True)
class ForwardTileSpec:
    """projectors.py:52-62 (paper's N_u = N_v = N_angles = 9)."""
    tile_u: int = 9
    tile_v: int = 9
    chunk_angles: int = 9

    def __post_init__(self):
        if min(self.tile_u, self.tile_v, self.chunk_angles) < 1:
            raise ValueError("tile sizes must be >= 1")


@dataclass(frozen=True)
class BackwardTileSpec:
    """projectors.py:65-78 (paper's 16 x 32 x 32, N_z = 8)."""
    tile_x: int = 16
    tile_y: int = 32
    chunk_angles: int = 32
    voxels_per_unit: int = 8

    def __post_init__(self):
        if min(self.tile_x, self.tile_y, self.chunk_angles,
               self.voxels_per_unit) < 1:
            raise ValueError("tile sizes must be >= 1")


def _as_f32(data):
    if isinstance(data, torch.Tensor):
        if data.dtype != torch.float32:
            data = data.float()
        return data.contiguous()
    if isinstance(data, np.memmap) and data.dtype == DTYPE and \
            data.flags.c_contiguous:
        return data  # file-backed (fileio mmap): streamed, never pinned
    return np.ascontiguousarray(data, dtype=DTYPE)


def _device() -> torch.device:
    lib()  # no CUDA / no library -> NativeLibraryError (no CPU fallback)
    return torch.device("cuda", torch.cuda.current_device())


def to_device(data, stream=None) -> torch.Tensor:
    """float32 CUDA tensor view/copy of host or device data."""
    if isinstance(data, torch.Tensor):
        if data.is_cuda and data.dtype == torch.float32 and \
                data.is_contiguous():
            return data
        return data.to(device=_device(), dtype=torch.float32).contiguous()
    host = torch.from_numpy(np.ascontiguousarray(data, dtype=DTYPE))
    return host.to(_device(), non_blocking=False)


_PINNED_MIN_BYTES = 1 << 20


_DRAIN_VIEWS = 90  # views per chunk of an overlapped drain


def _chunked_to_host(launch, out: torch.Tensor, a0: int, a1: int):
    """Run launch(c0, c1) per view chunk on the current stream and copy each
    finished chunk of ``out`` (rows a - a0) to one pinned host array on a
    side stream, overlapping the device->host drain with the next chunk's
    kernels.  Returns the host array (a numpy view of the pinned buffer)."""
    cur = torch.cuda.current_stream(out.device)
    side = _side_stream(out.device)
    host = torch.empty(tuple(out.shape), dtype=torch.float32, pin_memory=True)
    for c0 in range(a0, a1, _DRAIN_VIEWS):
        c1 = min(a1, c0 + _DRAIN_VIEWS)
        launch(c0, c1)
        ev = torch.cuda.Event()
        ev.record(cur)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            host[c0 - a0:c1 - a0].copy_(out[c0 - a0:c1 - a0],
                                        non_blocking=True)
    out.record_stream(side)
    side.synchronize()
    return host.numpy()


def _chunked_from_host(data: np.ndarray, device, launch, a0: int, a1: int):
    """Upload host rows [a - a0] chunk by chunk on a side stream and run
    launch(chunk_tensor, c0, c1) on the current stream as each arrives."""
    cur = torch.cuda.current_stream(device)
    side = _side_stream(device)
    src = torch.from_numpy(np.ascontiguousarray(data, dtype=DTYPE))
    dev = torch.empty(tuple(src.shape), dtype=torch.float32, device=device)
    side.wait_stream(cur)  # dev's memory may be reused from cur's past work
    for c0 in range(a0, a1, _DRAIN_VIEWS):
        c1 = min(a1, c0 + _DRAIN_VIEWS)
        with torch.cuda.stream(side):
            dev[c0 - a0:c1 - a0].copy_(src[c0 - a0:c1 - a0],
                                       non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(side)
        cur.wait_event(ev)
        launch(dev[c0 - a0:c1 - a0], c0, c1)
    dev.record_stream(cur)
    side.synchronize()  # the host source may be released after return


# host-to-host backprojection: the last view chunk runs in this many z
# pieces, each drained to the host while the next one computes, when the
# slab is at least _DRAIN_PIECE_MIN_BYTES (the volume's device->host copy,
# ~10 ms per 512^3, otherwise follows the whole computation)
_DRAIN_PIECES = 4
_DRAIN_PIECE_MIN_BYTES = 64 << 20


def _backproject_to_host(data: np.ndarray, geometry, slab_range, bwd,
                         a0: int, a1: int, device) -> np.ndarray:
    """backproject_slab for host projections into a fresh host volume:
    view chunks uploaded on a side stream while the previous chunk
    backprojects (as _chunked_from_host); the last chunk's backprojection
    is cut into z pieces (Atb is additive over views and separable over
    slabs), and each finished piece of the volume drains to one pinned host
    array on the side stream while the next piece computes."""
    z0, z1 = slab_range
    grid = geometry.voxel_grid
    cur = torch.cuda.current_stream(device)
    side = _side_stream(device)
    target = torch.zeros((z1 - z0, grid.n_y, grid.n_x), dtype=torch.float32,
                         device=device)
    host = torch.empty(tuple(target.shape), dtype=torch.float32,
                       pin_memory=target.numel() * 4 >= _PINNED_MIN_BYTES)
    src = torch.from_numpy(np.ascontiguousarray(data, dtype=DTYPE))
    dev = torch.empty(tuple(src.shape), dtype=torch.float32, device=device)
    side.wait_stream(cur)  # dev / target memory may be reused from cur's work
    n_p = (_DRAIN_PIECES if target.numel() * 4 >= _DRAIN_PIECE_MIN_BYTES
           else 1)
    n_p = max(1, min(n_p, z1 - z0))
    starts = list(range(a0, a1, _DRAIN_VIEWS))
    for c0 in starts:
        c1 = min(a1, c0 + _DRAIN_VIEWS)
        with torch.cuda.stream(side):
            dev[c0 - a0:c1 - a0].copy_(src[c0 - a0:c1 - a0],
                                       non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(side)
        cur.wait_event(ev)
        chunk = dev[c0 - a0:c1 - a0]
        if c0 != starts[-1]:
            bwd(chunk, geometry, (c0, c1), (z0, z1), target)
            continue
        for i in range(n_p):
            p0 = z0 + (z1 - z0) * i // n_p
            p1 = z0 + (z1 - z0) * (i + 1) // n_p
            piece = target[p0 - z0:p1 - z0]
            bwd(chunk, geometry, (c0, c1), (p0, p1), piece)
            done = torch.cuda.Event()
            done.record(cur)
            side.wait_event(done)
            with torch.cuda.stream(side):
                host[p0 - z0:p1 - z0].copy_(piece, non_blocking=True)
    dev.record_stream(cur)
    target.record_stream(side)
    side.synchronize()  # the host source may be released after return
    return host.numpy()


_SIDE = {}


def _side_stream(device) -> torch.cuda.Stream:
    s = _SIDE.get(device)
    if s is None:
        s = _SIDE[device] = torch.cuda.Stream(device)
    return s


def to_host(t) -> np.ndarray:
    """Host numpy copy of a tensor.  Large device results drain through a
    page-locked buffer (torch's caching host allocator) at full PCIe rate;
    the returned array is a view that keeps that buffer alive."""
    if isinstance(t, torch.Tensor):
        t = t.detach()
        if t.is_cuda and t.numel() * t.element_size() >= _PINNED_MIN_BYTES:
            out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            out.copy_(t, non_blocking=True)
            torch.cuda.current_stream(t.device).synchronize()
            return out.numpy()
        return t.cpu().numpy()
    return np.asarray(t)


@dataclass
class Volume:
    """Attenuation on an axial slab: data[z, y, x] (x fastest), slab_range
    = [z_begin, z_end) of the grid (projectors.py:81-120).  ``data`` is a
    numpy array or a CUDA tensor."""

    grid: VoxelGrid
    data: object
    slab_range: tuple[int, int] | None = None

    def __post_init__(self):
        if self.slab_range is None:
            self.slab_range = (0, self.grid.n_z)
        z0, z1 = self.slab_range
        if not (0 <= z0 < z1 <= self.grid.n_z):
            raise ValueError(f"invalid slab range {self.slab_range}")
        self.slab_range = (int(z0), int(z1))
        self.data = _as_f32(self.data)
        expect = (z1 - z0, self.grid.n_y, self.grid.n_x)
        if tuple(self.data.shape) != expect:
            raise ValueError(
                f"volume data shape {tuple(self.data.shape)} != {expect}")

    @classmethod
    def zeros(cls, grid: VoxelGrid, slab_range=None,
              device=None) -> "Volume":
        z0, z1 = slab_range if slab_range is not None else (0, grid.n_z)
        shape = (z1 - z0, grid.n_y, grid.n_x)
        data = (torch.zeros(shape, dtype=torch.float32, device=device)
                if device is not None else np.zeros(shape, DTYPE))
        return cls(grid, data, (z0, z1))

    @property
    def n_slices(self) -> int:
        return self.slab_range[1] - self.slab_range[0]

    @property
    def nbytes(self) -> int:
        return self.n_slices * self.grid.n_y * self.grid.n_x * 4

    @property
    def on_device(self) -> bool:
        return isinstance(self.data, torch.Tensor) and self.data.is_cuda

    def copy(self) -> "Volume":
        d = self.data.clone() if isinstance(self.data, torch.Tensor) \
            else self.data.copy()
        return Volume(self.grid, d, self.slab_range)

    def numpy(self) -> np.ndarray:
        return to_host(self.data)


@dataclass
class ProjectionStack:
    """Line integrals data[angle, v, u] (u fastest) for the contiguous
    angle window angle_range (projectors.py:123-163)."""

    detector: DetectorGrid
    data: object
    angle_range: tuple[int, int] | None = None

    def __post_init__(self):
        if self.angle_range is None:
            self.angle_range = (0, int(self.data.shape[0]))
        a0, a1 = self.angle_range
        if not (0 <= a0 < a1):
            raise ValueError(f"invalid angle range {self.angle_range}")
        self.angle_range = (int(a0), int(a1))
        self.data = _as_f32(self.data)
        expect = (a1 - a0, self.detector.n_v, self.detector.n_u)
        if tuple(self.data.shape) != expect:
            raise ValueError(
                f"projection data shape {tuple(self.data.shape)} != {expect}")

    @classmethod
    def zeros(cls, detector, angle_range, device=None) -> "ProjectionStack":
        a0, a1 = angle_range
        shape = (a1 - a0, detector.n_v, detector.n_u)
        data = (torch.zeros(shape, dtype=torch.float32, device=device)
                if device is not None else np.zeros(shape, DTYPE))
        return cls(detector, data, (a0, a1))

    @property
    def n_angles(self) -> int:
        return self.angle_range[1] - self.angle_range[0]

    @property
    def nbytes(self) -> int:
        return self.n_angles * self.detector.n_u * self.detector.n_v * 4

    @property
    def on_device(self) -> bool:
        return isinstance(self.data, torch.Tensor) and self.data.is_cuda

    def copy(self) -> "ProjectionStack":
        d = self.data.clone() if isinstance(self.data, torch.Tensor) \
            else self.data.copy()
        return ProjectionStack(self.detector, d, self.angle_range)

    def numpy(self) -> np.ndarray:
        return to_host(self.data)


def sample_step(grid: VoxelGrid) -> float:
    """Half the smallest voxel edge (projectors.py:166-169)."""
    return 0.5 * min(grid.voxel_size)


def siddon_trace(ray: Ray, grid: VoxelGrid):
    """Ordered (voxel index, length) pairs along a ray (host utility,
    projectors.py:205-243): every grid-plane crossing inside the clipped
    segment cuts it, each piece is attributed to the voxel holding its
    midpoint, pieces of length <= 1e-12 are dropped."""
    if not ray.hits or ray.t_exit - ray.t_entry <= 1e-12:
        return []
    o = np.asarray(ray.origin, dtype=float)
    d = np.asarray(ray.direction, dtype=float)
    g0 = grid.min_corner()
    vox = np.asarray(grid.voxel_size, dtype=float)
    counts = np.asarray(grid.counts)
    t0, t1 = ray.t_entry, ray.t_exit
    cuts = {t0, t1}
    for k in range(3):
        if d[k] == 0.0:
            continue
        planes = g0[k] + np.arange(counts[k] + 1) * vox[k]
        ts = (planes - o[k]) / d[k]
        cuts.update(float(t) for t in ts if t0 < t < t1)
    cuts = sorted(cuts)
    out = []
    for ta, tb in zip(cuts[:-1], cuts[1:]):
        if tb - ta <= 1e-12:
            continue
        mid = o + 0.5 * (ta + tb) * d
        idx = np.floor((mid - g0) / vox).astype(int)
        if np.all(idx >= 0) and np.all(idx < counts):
            out.append(((int(idx[0]), int(idx[1]), int(idx[2])),
                        float(tb - ta)))
    return out


def forward_project_slab(volume: Volume, geometry: ScanGeometry,
                         angle_range: tuple[int, int],
                         method: ProjectionMethod = ProjectionMethod.SIDDON,
                         tiles: ForwardTileSpec = ForwardTileSpec(),
                         out=None) -> ProjectionStack:
    """Project an axial slab for a window of angles (projectors.py:246-283).

    Pixels integrate over the slab only; slab projections of a partition
    sum to the full-volume projection.  ``out`` (optional CUDA tensor of the
    stack shape) receives the result in place.
    """
    if volume.grid != geometry.voxel_grid:
        raise ValueError("volume grid does not match scan geometry")
    a0, a1 = angle_range
    if not (0 <= a0 < a1 <= geometry.n_angles):
        raise ValueError(f"angle range {angle_range} outside scan")
    if not isinstance(method, ProjectionMethod):
        raise ValueError(f"unknown projection method {method}")
    det = geometry.detector
    vol = to_device(volume.data)
    if out is None:
        out = torch.empty((a1 - a0, det.n_v, det.n_u), dtype=torch.float32,
                          device=vol.device)
    fwd = K.fwd_interp if method is ProjectionMethod.INTERPOLATED \
        else K.fwd_siddon
    if volume.on_device:
        fwd(vol, geometry, (a0, a1), volume.slab_range, out)
        return ProjectionStack(det, out, (a0, a1))
    # host caller: views in chunks, each chunk drained to pinned host memory
    # on a side stream while the next one projects
    return ProjectionStack(det, _chunked_to_host(
        lambda c0, c1: fwd(vol, geometry, (c0, c1), volume.slab_range,
                           out[c0 - a0:c1 - a0]), out, a0, a1), (a0, a1))


def backproject_chunk_into(acc, projections: ProjectionStack,
                           geometry: ScanGeometry,
                           slab_range: tuple[int, int], mode: WeightMode,
                           tiles: BackwardTileSpec = BackwardTileSpec()) -> None:
    """Add one angle window's backprojection into a slab accumulator
    (projectors.py:286-315).  ``acc`` is a CUDA float32 tensor (added to
    on device) or a host numpy array (float64 in the reference; updated in
    place through a device round trip)."""
    if not isinstance(mode, WeightMode):
        raise ValueError(f"unknown weight mode {mode}")
    a0, a1 = projections.angle_range
    if isinstance(acc, torch.Tensor) and acc.is_cuda:
        dev_acc = acc
    else:
        dev_acc = to_device(np.asarray(acc, dtype=np.float32))
    bwd = K.bwd_fdk if mode is WeightMode.FDK else K.bwd_matched
    if projections.on_device:
        bwd(to_device(projections.data), geometry, (a0, a1), slab_range,
            dev_acc)
    else:
        # host projections: view chunks uploaded on a side stream while the
        # previous chunk backprojects (Atb is additive over views)
        _chunked_from_host(
            projections.data, dev_acc.device,
            lambda p, c0, c1: bwd(p, geometry, (c0, c1), slab_range,
                                  dev_acc), a0, a1)
    if dev_acc is not acc:
        acc[...] = to_host(dev_acc).astype(acc.dtype)


def backproject_slab(projections: ProjectionStack, geometry: ScanGeometry,
                     slab_range: tuple[int, int],
                     mode: WeightMode = WeightMode.FDK,
                     tiles: BackwardTileSpec = BackwardTileSpec(),
                     accumulate_into: Volume | None = None) -> Volume:
    """Backproject a window of angles into one slab, adding onto
    ``accumulate_into`` (zeros when omitted), projectors.py:318-348."""
    z0, z1 = slab_range
    grid = geometry.voxel_grid
    if not (0 <= z0 < z1 <= grid.n_z):
        raise ValueError(f"invalid slab range {slab_range}")
    if projections.detector != geometry.detector:
        raise ValueError("projection detector does not match scan geometry")
    a0, a1 = projections.angle_range
    if not (0 <= a0 < a1 <= geometry.n_angles):
        raise ValueError(f"angle range {projections.angle_range} outside scan")
    if accumulate_into is None and not projections.on_device:
        if not isinstance(mode, WeightMode):
            raise ValueError(f"unknown weight mode {mode}")
        bwd = K.bwd_fdk if mode is WeightMode.FDK else K.bwd_matched
        return Volume(grid, _backproject_to_host(
            projections.data, geometry, (z0, z1), bwd, a0, a1, _device()),
            (z0, z1))
    if accumulate_into is None:
        # fresh accumulator: zeros on the device; host callers get host data
        target = torch.zeros((z1 - z0, grid.n_y, grid.n_x),
                             dtype=torch.float32, device=_device())
        backproject_chunk_into(target, projections, geometry, (z0, z1), mode,
                               tiles)
        return Volume(grid, target if projections.on_device
                      else to_host(target), (z0, z1))
    if accumulate_into.slab_range != (z0, z1):
        raise ValueError("accumulate_into does not cover the slab range")
    # device accumulators are added to in place; host ones round-trip
    target = to_device(accumulate_into.data)
    backproject_chunk_into(target, projections, geometry, (z0, z1), mode,
                           tiles)
    if not accumulate_into.on_device:
        accumulate_into.data[:] = to_host(target)
    return accumulate_into
