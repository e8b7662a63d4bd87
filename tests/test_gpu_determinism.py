"""Deterministic matched Atb (cs_set_deterministic / CS_ST_DETERMINISTIC=1,
staged.cu det_add): contributions summed as 64-bit fixed-point integers,
so repeated runs are bit-identical -- as the reference's fp64 host
accumulation is (_kernels.py:278-337) -- and the result still matches the
oracle within the operator tolerance (1e-5 relL2)."""

from __future__ import annotations

import math
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1905_03748_b200 as cs
from conftest import rel_l2, synth_geometry, to_oracle
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL_OP = 1e-5


def _odd_geometry(n_angles):
    grid = cs.VoxelGrid(37, 29, 23, (1.0, 0.9, 1.1), (0.3, -0.2, 0.1))
    det = cs.DetectorGrid(41, 27, (2.1, 2.3), (0.4, -0.3))
    ang = tuple(np.linspace(0.1, 0.1 + 2 * math.pi, n_angles, endpoint=False))
    return cs.ScanGeometry(90.0, 180.0, ang, grid, det)


@pytest.fixture
def deterministic():
    from paper_1905_03748_b200 import kernels as K
    K.set_deterministic(True)
    yield K
    K.set_deterministic(False)


@pytest.mark.parametrize("case", ["odd19", "few3", "cube64"])
def test_matched_deterministic_repeats_bit_identical(deterministic, case):
    import torch
    K = deterministic
    g = {"odd19": lambda: _odd_geometry(19), "few3": lambda: _odd_geometry(3),
         "cube64": lambda: synth_geometry(64, 48)}[case]()
    grid, det, na = g.voxel_grid, g.detector, g.n_angles
    y = torch.randn((na, det.n_v, det.n_u), device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(4))
    runs = []
    for _ in range(3):
        acc = torch.zeros((grid.n_z, grid.n_y, grid.n_x), device="cuda")
        K.bwd_matched(y, g, (0, na), (0, grid.n_z), acc)
        runs.append(acc.cpu().numpy())
    assert all(np.array_equal(runs[0], r) for r in runs[1:])
    # against the reference restatement (fp64) and the default mode
    ref = O.bwd_matched(y.cpu().numpy(), to_oracle(g))
    assert rel_l2(runs[0], ref) <= TOL_OP, rel_l2(runs[0], ref)
    K.set_deterministic(False)
    acc = torch.zeros_like(acc)
    K.bwd_matched(y, g, (0, na), (0, grid.n_z), acc)
    assert rel_l2(runs[0], acc.cpu().numpy()) <= 1e-6
    # a slab of the grid: the same planes as the whole-grid launch
    K.set_deterministic(True)
    sl = torch.zeros((9, grid.n_y, grid.n_x), device="cuda")
    K.bwd_matched(y, g, (0, na), (7, 16), sl)
    assert rel_l2(sl.cpu().numpy(), runs[0][7:16]) <= 1e-6


def test_matched_deterministic_global_fallback_subprocess():
    """A 2 KB box budget (CS_STAGED_SMEM_KB=2) sends most chunks down the
    global-memory path; with CS_ST_DETERMINISTIC=1 those taps go through the
    64-bit integer accumulator too: two processes, identical bits."""
    code = (
        "import torch,sys,math,numpy as np;sys.path.insert(0,'.');"
        "import paper_1905_03748_b200 as cs;"
        "from paper_1905_03748_b200 import kernels as K;"
        "grid=cs.VoxelGrid(37,29,23,(1.0,0.9,1.1),(0.3,-0.2,0.1));"
        "det=cs.DetectorGrid(41,27,(2.1,2.3),(0.4,-0.3));"
        "ang=tuple(np.linspace(0.1,0.1+2*math.pi,19,endpoint=False));"
        "g=cs.ScanGeometry(90.0,180.0,ang,grid,det);"
        "y=torch.randn((19,27,41),device='cuda',"
        "generator=torch.Generator(device='cuda').manual_seed(2));"
        "acc=torch.zeros((23,29,37),device='cuda');"
        "K.bwd_matched(y,g,(0,19),(0,23),acc);"
        "np.save(sys.argv[1],acc.cpu().numpy())")
    env = dict(os.environ, CS_ST_DETERMINISTIC="1", CS_STAGED_SMEM_KB="2")
    with tempfile.TemporaryDirectory() as td:
        outs = []
        for i in range(2):
            fn = os.path.join(td, f"r{i}.npy")
            subprocess.run([sys.executable, "-c", code, fn], cwd=ROOT,
                           env=env, check=True, timeout=300)
            outs.append(np.load(fn))
    assert np.array_equal(outs[0], outs[1])
    g = _odd_geometry(19)
    import torch
    y = torch.randn((19, 27, 41), device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(2))
    ref = O.bwd_matched(y.cpu().numpy(), to_oracle(g))
    assert rel_l2(outs[0], ref) <= TOL_OP


def test_matched_deterministic_transposed_frame_subprocess():
    """Deterministic mode runs the x-major views in the transposed frame
    into a second (transposed) int64 accumulator, finished together with
    the direct one (det_finish_t_kernel).  Against the x-major views in
    their own frame (CS_ST_TRANSPOSE=0): the same box sums in the same
    units of S, so the same volume up to chunks whose box fits in one
    frame's padded layout and not in the other's (global path)."""
    code = (
        "import torch,sys;sys.path.insert(0,'.');"
        "import numpy as np;"
        "from conftest import synth_geometry;"
        "from paper_1905_03748_b200 import kernels as K;"
        "g=synth_geometry(64,48);d=g.detector;"
        "y=torch.randn((48,d.n_v,d.n_u),device='cuda',"
        "generator=torch.Generator(device='cuda').manual_seed(4));"
        "acc=torch.zeros((64,64,64),device='cuda');"
        "K.bwd_matched(y,g,(0,48),(0,64),acc);"
        "np.save(sys.argv[1],acc.cpu().numpy())")
    outs = {}
    with tempfile.TemporaryDirectory() as td:
        for t in ("1", "0"):
            env = dict(os.environ, CS_ST_DETERMINISTIC="1",
                       CS_ST_TRANSPOSE=t,
                       PYTHONPATH=os.path.join(ROOT, "tests"))
            fn = os.path.join(td, f"t{t}.npy")
            subprocess.run([sys.executable, "-c", code, fn], cwd=ROOT,
                           env=env, check=True, timeout=300)
            outs[t] = np.load(fn)
    assert rel_l2(outs["1"], outs["0"]) <= 1e-7, rel_l2(outs["1"], outs["0"])
    import torch
    g = synth_geometry(64, 48)
    d = g.detector
    y = torch.randn((48, d.n_v, d.n_u), device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(4))
    ref = O.bwd_matched(y.cpu().numpy(), to_oracle(g))
    assert rel_l2(outs["1"], ref) <= TOL_OP
