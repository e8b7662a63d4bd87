"""Raw/sidecar persistence against files written by the
reference's own writers (tests/golden/make_fileio_golden.py)."""

from __future__ import annotations

import math
import os
import shutil

import numpy as np
import pytest

import paper_1905_03748_b200 as cs
from paper_1905_03748_b200 import fileio

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                    "fileio")


def _expected():
    grid = cs.VoxelGrid(5, 4, 3, (1.0, 0.9, 1.1), (0.3, -0.2, 0.1))
    vol = np.random.default_rng(7).standard_normal((3, 4, 5)).astype(
        np.float32)
    det = cs.DetectorGrid(6, 3, (2.5, 2.25), (0.4, -0.3))
    angles = tuple(float(a) for a in np.linspace(0.1, 0.1 + 2 * math.pi, 4,
                                                 endpoint=False))
    geo = cs.ScanGeometry(20.0, 40.0, angles, grid, det)
    proj = np.random.default_rng(8).standard_normal((4, 3, 6)).astype(
        np.float32)
    return grid, vol, det, geo, proj


def _same_file(a, b):
    with open(a, "rb") as fa, open(b, "rb") as fb:
        return fa.read() == fb.read()


@pytest.mark.parametrize("mmap", [False, True])
def test_read_reference_files(mmap):
    grid, vol, det, geo, proj = _expected()
    v = fileio.read_volume(os.path.join(GOLD, "vol.raw"), mmap=mmap)
    assert v.grid == grid and v.slab_range == (0, 3)
    assert np.array_equal(np.asarray(v.data), vol)
    assert isinstance(v.data, np.memmap) == mmap
    p, g = fileio.read_projections(os.path.join(GOLD, "proj.raw"), mmap=mmap)
    assert g == geo and p.detector == det and p.angle_range == (0, 4)
    assert np.array_equal(np.asarray(p.data), proj)
    assert fileio.read_geometry(os.path.join(GOLD, "proj.raw")) == geo


def test_writers_reproduce_reference_bytes(tmp_path):
    grid, vol, det, geo, proj = _expected()
    fileio.write_volume(str(tmp_path / "vol.raw"), cs.Volume(grid, vol))
    fileio.write_projections(str(tmp_path / "proj.raw"),
                             cs.ProjectionStack(det, proj), geo)
    for name in ("vol.raw", "vol.raw.meta", "proj.raw", "proj.raw.meta"):
        assert _same_file(tmp_path / name, os.path.join(GOLD, name)), name
    assert sorted(os.listdir(tmp_path)) == sorted(
        ["vol.raw", "vol.raw.meta", "proj.raw", "proj.raw.meta"])


def test_errors(tmp_path):
    grid, vol, det, geo, proj = _expected()
    for name in ("vol.raw", "vol.raw.meta", "proj.raw", "proj.raw.meta"):
        shutil.copy(os.path.join(GOLD, name), tmp_path / name)
    vp, pp = str(tmp_path / "vol.raw"), str(tmp_path / "proj.raw")
    with pytest.raises(ValueError, match="kind tag"):
        fileio.read_volume(pp)
    with pytest.raises(ValueError, match="no geometry block"):
        fileio.read_geometry(vp)
    with open(vp, "ab") as fh:
        fh.write(b"\0\0\0\0")
    with pytest.raises(ValueError, match="payload holds"):
        fileio.read_volume(vp)
    with open(fileio.sidecar_path(vp), "a") as fh:
        fh.write("no equals sign here\n")
    with pytest.raises(ValueError, match="malformed"):
        fileio.read_sidecar(vp)
    text = open(fileio.sidecar_path(pp)).read().replace(
        "dtype = float32", "dtype = float64")
    open(fileio.sidecar_path(pp), "w").write(text)
    with pytest.raises(ValueError, match="dtype"):
        fileio.read_projections(pp)
    with pytest.raises(ValueError, match="full volumes"):
        fileio.write_volume(str(tmp_path / "x.raw"),
                            cs.Volume(grid, vol[1:], (1, 3)))
    with pytest.raises(ValueError, match="scan angles"):
        fileio.write_projections(str(tmp_path / "y.raw"),
                                 cs.ProjectionStack(det, proj[:2]), geo)


def test_comments_and_blank_lines(tmp_path):
    shutil.copy(os.path.join(GOLD, "vol.raw"), tmp_path / "vol.raw")
    text = open(os.path.join(GOLD, "vol.raw.meta")).read()
    open(tmp_path / "vol.raw.meta", "w").write("# header\n\n" + text + "\n")
    v = fileio.read_volume(str(tmp_path / "vol.raw"))
    assert v.grid.counts == (5, 4, 3)


def test_create_finish_volume(tmp_path):
    grid, vol, *_ = _expected()
    path = str(tmp_path / "out.raw")
    v = fileio.create_volume(path, grid)
    assert not os.path.exists(path)
    v.data[:] = vol
    fileio.finish_volume(path, v)
    assert _same_file(path, os.path.join(GOLD, "vol.raw"))
    assert _same_file(path + ".meta", os.path.join(GOLD, "vol.raw.meta"))


@pytest.mark.gpu
def test_write_device_tensor(tmp_path):
    import torch
    grid, vol, det, geo, proj = _expected()
    fileio.write_volume(str(tmp_path / "vol.raw"),
                        cs.Volume(grid, torch.from_numpy(vol).cuda()))
    assert _same_file(tmp_path / "vol.raw", os.path.join(GOLD, "vol.raw"))
    fileio.write_projections(str(tmp_path / "proj.raw"),
                             cs.ProjectionStack(det,
                                                torch.from_numpy(proj).cuda()),
                             geo)
    assert _same_file(tmp_path / "proj.raw", os.path.join(GOLD, "proj.raw"))
