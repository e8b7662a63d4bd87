"""Raw little-endian float32 payloads with ``key = value`` sidecars -- the
drop-in for conesplit.fileio (/root/reference/pkg/src/conesplit/fileio.py).

Same on-disk format, names and errors as the reference:

* payload ``<path>``: float32 LE samples, x-fastest volumes ``[z][y][x]``,
  u-fastest projections ``[angle][v][u]`` (fileio.py:1-8);
* sidecar ``<path>.meta``: ASCII ``key = value`` lines; ``#`` comments and
  blank lines ignored (fileio.py:40-53); projection sidecars embed the scan
  geometry (fileio.py:104-117);
* writes are atomic: temp files, sidecar renamed into place first, then the
  payload (fileio.py:87-95).

B200-first additions for the out-of-core path (C5: volumes larger than one
GPU's HBM):

* ``read_volume(path, mmap=True)`` / ``read_projections(path, mmap=True)``
  return containers backed by a read-only ``np.memmap``; the executor
  (execution.py) streams slabs / angle chunks straight from the page cache
  into pinned staging buffers instead of page-locking the whole image;
* ``write_volume`` / ``write_projections`` accept CUDA tensors and drain
  them through a pinned buffer in bounded pieces, so a device-resident
  result is persisted without a full host copy;
* ``create_volume(path, grid)`` makes a writable memmap payload (zeros) to
  receive an out-of-core backprojection slab by slab; the sidecar lands
  when the payload is complete.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from .geometry import DetectorGrid, ScanGeometry, VoxelGrid
from .projectors import ProjectionStack, Volume

__all__ = [
    "read_volume",
    "write_volume",
    "read_projections",
    "write_projections",
    "read_sidecar",
    "read_geometry",
    "sidecar_path",
    "create_volume",
    "finish_volume",
]

DTYPE_TAG = "float32"
BYTE_ORDER_TAG = "little"
_LE_F32 = np.dtype("<f4")
_DRAIN_BYTES = 64 << 20  # pinned drain piece for device tensors


def sidecar_path(path: str) -> str:
    """``<path>.meta`` (fileio.py:36-37)."""
    return f"{path}.meta"


# --------------------------------------------------------------------------
# sidecar text


def _render(fields: dict) -> str:
    return "".join(f"{k} = {v}\n" for k, v in fields.items())


def read_sidecar(path: str) -> dict:
    """Parse ``<path>.meta`` into a str -> str dict (fileio.py:40-53);
    a non-comment line without ``=`` is a ValueError."""
    out: dict[str, str] = {}
    with open(sidecar_path(path), encoding="ascii") as fh:
        for raw in fh:
            text = raw.strip()
            if not text or text[0] == "#":
                continue
            key, sep, value = text.partition("=")
            if not sep:
                raise ValueError(f"malformed sidecar line: {text!r}")
            out[key.strip()] = value.strip()
    return out


def _words(text: str, cast):
    return tuple(cast(w) for w in text.split())


def _vec(values) -> str:
    return " ".join(repr(float(v)) for v in values)


def _require_tags(fields: dict, kind: str, layout: str):
    """fileio.py:64-76: kind, dtype, byte order and layout tags."""
    checks = (("kind", kind, "sidecar kind tag {!r} is not " + repr(kind)),
              ("dtype", DTYPE_TAG, "unknown dtype tag {!r}"),
              ("byte_order", BYTE_ORDER_TAG,
               "unsupported byte order tag {!r}"),
              ("layout", layout, "unexpected layout tag {!r}"))
    for key, want, msg in checks:
        got = fields.get(key)
        if got != want:
            raise ValueError(msg.format(got))


def _geometry_block(geometry: ScanGeometry) -> dict:
    """fileio.py:98-111 (repr round-trips every float64 exactly)."""
    grid, det = geometry.voxel_grid, geometry.detector
    return {
        "geometry.dso": repr(float(geometry.dso)),
        "geometry.dsd": repr(float(geometry.dsd)),
        "geometry.angles": _vec(geometry.angles),
        "grid.dims": f"{grid.n_x} {grid.n_y} {grid.n_z}",
        "grid.voxel_size": _vec(grid.voxel_size),
        "grid.origin_offset": _vec(grid.origin_offset),
        "detector.dims": f"{det.n_u} {det.n_v}",
        "detector.pixel_size": _vec(det.pixel_size),
        "detector.offset": _vec(det.detector_offset),
    }


def _volume_fields(grid: VoxelGrid) -> dict:
    """fileio.py:134-146."""
    return {
        "kind": "volume",
        "dims": f"{grid.n_x} {grid.n_y} {grid.n_z}",
        "dtype": DTYPE_TAG,
        "byte_order": BYTE_ORDER_TAG,
        "layout": "x-fastest",
        "voxel_size": _vec(grid.voxel_size),
        "origin_offset": _vec(grid.origin_offset),
    }


def read_geometry(path: str) -> ScanGeometry:
    """Scan geometry from a sidecar's geometry block (fileio.py:114-128)."""
    f = read_sidecar(path)
    if "geometry.dso" not in f:
        raise ValueError(f"{sidecar_path(path)} carries no geometry block")
    nx, ny, nz = _words(f["grid.dims"], int)
    nu, nv = _words(f["detector.dims"], int)
    grid = VoxelGrid(nx, ny, nz, _words(f["grid.voxel_size"], float),
                     _words(f["grid.origin_offset"], float))
    det = DetectorGrid(nu, nv, _words(f["detector.pixel_size"], float),
                       _words(f["detector.offset"], float))
    return ScanGeometry(float(f["geometry.dso"]), float(f["geometry.dsd"]),
                        _words(f["geometry.angles"], float), grid, det)


# --------------------------------------------------------------------------
# payloads


def _load_payload(path: str, shape: tuple, mmap: bool) -> np.ndarray:
    """Size-checked payload (fileio.py:79-84); memmap'd on request."""
    count = int(np.prod(shape))
    size = os.path.getsize(path)
    if size != count * 4:
        raise ValueError(
            f"payload holds {size} bytes, sidecar dims need {count * 4}")
    if mmap:
        return np.memmap(path, dtype=_LE_F32, mode="r", shape=shape)
    return np.fromfile(path, dtype=_LE_F32, count=count).reshape(shape)


def _emit_payload(fh, data):
    """Write float32 LE samples of a numpy array or a (CUDA) tensor; device
    data drains through one pinned buffer in bounded pieces."""
    if isinstance(data, torch.Tensor):
        flat = data.detach().reshape(-1)
        if not flat.is_cuda:
            np.ascontiguousarray(flat.float().numpy(), _LE_F32).tofile(fh)
            return
        step = max(1, _DRAIN_BYTES // 4)
        pin = torch.empty(min(step, flat.numel()), dtype=torch.float32,
                          pin_memory=True)
        for s in range(0, flat.numel(), step):
            n = min(step, flat.numel() - s)
            pin[:n].copy_(flat[s:s + n].float(), non_blocking=False)
            pin[:n].numpy().astype(_LE_F32, copy=False).tofile(fh)
        return
    arr = np.asarray(data)
    rows = arr.reshape(arr.shape[0], -1) if arr.ndim > 1 else arr[None]
    per = max(1, _DRAIN_BYTES // max(1, rows.shape[1] * 4))
    for s in range(0, rows.shape[0], per):
        np.ascontiguousarray(rows[s:s + per], _LE_F32).tofile(fh)


def _commit(path: str, sidecar: str, data):
    """Temp files, then sidecar rename, then payload rename
    (fileio.py:87-95): a payload never exists without its sidecar."""
    meta = sidecar_path(path)
    with open(meta + ".tmp", "w", encoding="ascii") as fh:
        fh.write(sidecar)
    with open(path + ".tmp", "wb") as fh:
        _emit_payload(fh, data)
    os.replace(meta + ".tmp", meta)
    os.replace(path + ".tmp", path)


def write_volume(path: str, volume: Volume):
    """fileio.py:131-147; only full volumes are persisted."""
    if volume.slab_range != (0, volume.grid.n_z):
        raise ValueError("only full volumes are persisted")
    _commit(path, _render(_volume_fields(volume.grid)), volume.data)


def read_volume(path: str, mmap: bool = False) -> Volume:
    """fileio.py:150-157 (+ ``mmap``: page-cache-backed, read-only)."""
    f = read_sidecar(path)
    _require_tags(f, "volume", "x-fastest")
    nx, ny, nz = _words(f["dims"], int)
    data = _load_payload(path, (nz, ny, nx), mmap)
    grid = VoxelGrid(nx, ny, nz, _words(f["voxel_size"], float),
                     _words(f["origin_offset"], float))
    return Volume(grid, data, (0, nz))


def write_projections(path: str, projections: ProjectionStack,
                      geometry: ScanGeometry):
    """fileio.py:160-174; the stack must cover every scan angle."""
    if projections.n_angles != geometry.n_angles:
        raise ValueError("projection stack does not cover the scan angles")
    det = projections.detector
    fields = {
        "kind": "projections",
        "dims": f"{det.n_u} {det.n_v} {projections.n_angles}",
        "dtype": DTYPE_TAG,
        "byte_order": BYTE_ORDER_TAG,
        "layout": "u-fastest",
        **_geometry_block(geometry),
    }
    _commit(path, _render(fields), projections.data)


def read_projections(path: str, mmap: bool = False
                     ) -> tuple[ProjectionStack, ScanGeometry]:
    """fileio.py:177-188: dims cross-checked against the geometry block."""
    f = read_sidecar(path)
    _require_tags(f, "projections", "u-fastest")
    nu, nv, n_angles = _words(f["dims"], int)
    geometry = read_geometry(path)
    if (geometry.detector.n_u, geometry.detector.n_v) != (nu, nv):
        raise ValueError("sidecar dims disagree with the geometry block")
    if geometry.n_angles != n_angles:
        raise ValueError("sidecar dims disagree with the angle list")
    data = _load_payload(path, (n_angles, nv, nu), mmap)
    return (ProjectionStack(geometry.detector, data, (0, n_angles)),
            geometry)


# --------------------------------------------------------------------------
# out-of-core outputs


def create_volume(path: str, grid: VoxelGrid) -> Volume:
    """A zero-filled, writable memmap volume at ``<path>.tmp`` (sparse file
    where the filesystem allows); fill it (e.g. as an execute_backward
    ``out``) and call :func:`finish_volume` to publish it atomically."""
    tmp = path + ".tmp"
    with open(tmp, "wb") as fh:
        fh.truncate(grid.n_voxels * 4)
    data = np.memmap(tmp, dtype=_LE_F32, mode="r+",
                     shape=(grid.n_z, grid.n_y, grid.n_x))
    return Volume(grid, data, (0, grid.n_z))


def finish_volume(path: str, volume: Volume):
    """Flush a :func:`create_volume` payload and publish sidecar + payload
    with the reference's ordering (sidecar first)."""
    data = volume.data
    if not isinstance(data, np.memmap):
        raise ValueError("finish_volume expects a create_volume() volume")
    data.flush()
    meta = sidecar_path(path)
    with open(meta + ".tmp", "w", encoding="ascii") as fh:
        fh.write(_render(_volume_fields(volume.grid)))
    os.replace(meta + ".tmp", meta)
    os.replace(path + ".tmp", path)
