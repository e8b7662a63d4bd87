"""TIGRE-style convenience entry points (SURVEY 8(b) "Python layer"):
``Ax(img, geo, angles)``, ``Atb(proj, geo, angles)``, ``sirt`` and
``asd_pocs`` over the conesplit-compatible API.  SIRT is os_sart with one
block of all angles (algorithms.py:267-268); "ASD-POCS" is os_sart with a
TV step per outer iteration (algorithms.py:299-303, SPEC's SART-TV glue).
Arrays in, arrays out (numpy or torch, matching the input)."""

from __future__ import annotations

from .algorithms import Algorithm, ReconConfig, os_sart
from .geometry import ScanGeometry
from .projectors import (ProjectionMethod, ProjectionStack, Volume,
                         WeightMode, backproject_slab, forward_project_slab)
from .regularization import NormMode, TvMinimizer, TvParams
from .scheduler import DevicePool

__all__ = ["Ax", "Atb", "sirt", "asd_pocs"]


def _geo(geo: ScanGeometry, angles) -> ScanGeometry:
    return geo if angles is None else geo.with_angles(tuple(angles))


def Ax(img, geo: ScanGeometry, angles=None, method: str = "interpolated"):
    """Forward projection of a full volume img[z, y, x] -> proj[a, v, u]."""
    g = _geo(geo, angles)
    vol = Volume(g.voxel_grid, img)
    m = ProjectionMethod(method)
    return forward_project_slab(vol, g, (0, g.n_angles), m).data


def Atb(proj, geo: ScanGeometry, angles=None, weight: str = "matched"):
    """Backprojection of proj[a, v, u] -> img[z, y, x]."""
    g = _geo(geo, angles)
    stack = ProjectionStack(g.detector, proj, (0, g.n_angles))
    return backproject_slab(stack, g, (0, g.voxel_grid.n_z),
                            WeightMode(weight)).data


def _pool(pool):
    return DevicePool.b200(1) if pool is None else pool


def sirt(proj, geo: ScanGeometry, angles=None, niter: int = 10,
         relaxation: float = 1.0, pool: DevicePool | None = None):
    g = _geo(geo, angles)
    cfg = ReconConfig(_pool(pool), Algorithm.OSSART, niter, g.n_angles,
                      relaxation)
    return os_sart(ProjectionStack(g.detector, proj), g, cfg).data


def asd_pocs(proj, geo: ScanGeometry, angles=None, niter: int = 10,
             block_size: int = 20, relaxation: float = 1.0,
             tv_iters: int = 20, tv_step: float = 1e-3,
             pool: DevicePool | None = None):
    g = _geo(geo, angles)
    tv = TvParams(TvMinimizer.GRADIENT_DESCENT, inner_iters=tv_iters,
                  step=tv_step, norm_mode=NormMode.EXACT_GLOBAL)
    cfg = ReconConfig(_pool(pool), Algorithm.OSSART, niter,
                      min(block_size, g.n_angles), relaxation, tv)
    return os_sart(ProjectionStack(g.detector, proj), g, cfg).data
