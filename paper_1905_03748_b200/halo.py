"""Distributed halo-slab TV: one slab per rank, ghosts over NCCL.

The multi-GPU form of split_minimize (regularization.py:213-280, paper
Sec. 2.3): rank r owns core [z0, z1) of the volume and a window
[w0, w1) = core +- halo.  Every epoch, ghost planes are refreshed from the
+-1 neighbours' cores with point-to-point send/recv (NCCL over
NVLink/NVSwitch: a contention-free ring); inside an epoch,
ExactGlobal norms cost one fp64 all_reduce per inner iteration and
LocalApprox none.  The stencil math is pluggable (``ops``) so the exchange
logic is testable with the gloo backend on CPU; the default ops are the
sm_100a kernels.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from . import kernels as K

__all__ = ["split_minimize_distributed", "minimize_sharded", "exchange_halos",
           "gather_cores", "CudaTvOps"]


class CudaTvOps:
    """TV stencils of csrc/tv.cu."""

    grad_sumsq = staticmethod(K.tv_grad_sumsq)
    step = staticmethod(K.tv_step)
    # the GD pair the loops use: g kept between the passes (bit-identical)
    grad_store = staticmethod(K.tv_grad_store)
    step_g = staticmethod(K.tv_step_g)
    rof_iter = staticmethod(K.rof_iter)
    rof_finish = staticmethod(K.rof_finish)


def exchange_halos(w: torch.Tensor, slabs, rank: int, zdim: int = 0) -> None:
    """Overwrite the ghost planes of window ``w`` (this rank's slab) with
    the neighbours' current core planes.  ``zdim`` is the plane axis of
    ``w`` (1 for the [3, z, y, x] ROF dual)."""
    s = slabs[rank]
    (z0, z1), (w0, w1) = s.core_range, s.window
    ops = []
    keep = []

    def planes(a, b):
        return w.narrow(zdim, a - w0, b - a)

    if rank > 0:
        prev = slabs[rank - 1]
        lo_ghost = (w0, z0)  # from rank-1's core top
        if lo_ghost[1] > lo_ghost[0]:
            buf = torch.empty_like(planes(*lo_ghost).contiguous())
            ops.append(dist.P2POp(dist.irecv, buf, rank - 1))
            keep.append((buf, lo_ghost))
        # rank-1 needs my first planes for its upper ghost
        send_hi = min(z1, prev.window[1])
        if send_hi > z0:
            ops.append(dist.P2POp(dist.isend,
                                  planes(z0, send_hi).contiguous(), rank - 1))
    if rank < len(slabs) - 1:
        nxt = slabs[rank + 1]
        hi_ghost = (z1, w1)
        if hi_ghost[1] > hi_ghost[0]:
            buf = torch.empty_like(planes(*hi_ghost).contiguous())
            ops.append(dist.P2POp(dist.irecv, buf, rank + 1))
            keep.append((buf, hi_ghost))
        send_lo = max(z0, nxt.window[0])
        if z1 > send_lo:
            ops.append(dist.P2POp(dist.isend,
                                  planes(send_lo, z1).contiguous(), rank + 1))
    if ops and w.is_cuda and dist.get_backend() != "nccl":
        # gloo (ranks sharing a GPU in tests) moves host tensors only
        staged = []
        for op in ops:
            h = op.tensor.cpu()
            staged.append((op, h))
        reqs = dist.batch_isend_irecv([dist.P2POp(op.op, h, op.peer)
                                       for op, h in staged])
        for req in reqs:
            req.wait()
        for op, h in staged:
            if op.op is dist.irecv:
                op.tensor.copy_(h)
    elif ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for buf, (a, b) in keep:
        planes(a, b).copy_(buf)


def gather_cores(w: torch.Tensor, slabs, rank: int, full_shape,
                 zdim: int = 0) -> torch.Tensor:
    """All ranks get the full array assembled from every rank's core."""
    s = slabs[rank]
    (z0, z1), (w0, _) = s.core_range, s.window
    core = w.narrow(zdim, z0 - w0, z1 - z0).contiguous()
    longest = max(t.core_range[1] - t.core_range[0] for t in slabs)
    shape = list(core.shape)
    shape[zdim] = longest
    pad = torch.zeros(shape, dtype=w.dtype, device=w.device)
    pad.narrow(zdim, 0, z1 - z0).copy_(core)
    if pad.is_cuda and dist.get_backend() != "nccl":
        hp = pad.cpu()
        parts = [torch.empty_like(hp) for _ in slabs]
        dist.all_gather(parts, hp)
        parts = [p.to(pad.device) for p in parts]
    else:
        parts = [torch.empty_like(pad) for _ in slabs]
        dist.all_gather(parts, pad)
    return torch.cat([p.narrow(zdim, 0, t.core_range[1] - t.core_range[0])
                      for p, t in zip(parts, slabs)], zdim)


def _check_halo(slabs):
    for i, s in enumerate(slabs):
        d = s.halo_depth
        if i > 0 and slabs[i - 1].core_range[1] - slabs[i - 1].core_range[0] < min(
                d, s.core_range[0] - s.window[0]):
            raise ValueError("halo deeper than a neighbour's core")
        if i + 1 < len(slabs) and slabs[i + 1].core_range[1] - \
                slabs[i + 1].core_range[0] < min(d, s.window[1] - s.core_range[1]):
            raise ValueError("halo deeper than a neighbour's core")


def split_minimize_distributed(u_full: torch.Tensor, slabs, params, rank: int,
                               ops=CudaTvOps) -> torch.Tensor:
    """Rank ``rank`` runs slab ``rank``; returns the full result on every
    rank.  Matches the single-process split_minimize slab for slab."""
    from .regularization import NormMode, TvMinimizer
    _check_halo(slabs)
    s = slabs[rank]
    (w0, w1) = s.window
    core = s.core_in_window
    total_voxels = u_full.numel()
    if params.minimizer is TvMinimizer.GRADIENT_DESCENT:
        w = u_full[w0:w1].clone()
        spare = torch.empty_like(w)
        ss = torch.zeros(1, dtype=torch.float64, device=w.device)
        exact = params.norm_mode is NormMode.EXACT_GLOBAL
        scale = 1.0 if exact else float(np.sqrt(total_voxels / w.numel()))
        stored = hasattr(ops, "grad_store")
        g = torch.empty_like(w) if stored else None
        for epoch in range(params.outer_syncs):
            if epoch > 0:
                exchange_halos(w, slabs, rank)
            for _ in range(params.inner_iters):
                band = (core.start, core.stop) if exact else (0, w.shape[0])
                if stored:
                    ops.grad_store(w, g, band, ss)
                else:
                    ops.grad_sumsq(w, band, ss)
                if exact:
                    dist.all_reduce(ss)
                if stored:
                    ops.step_g(w, g, spare, params.step, ss, scale)
                else:
                    ops.step(w, spare, params.step, ss, scale)
                w, spare = spare, w
        return gather_cores(w, slabs, rank, tuple(u_full.shape))
    f = u_full
    p = torch.zeros((3, w1 - w0) + tuple(f.shape[1:]), dtype=torch.float32,
                    device=f.device)
    q = torch.empty_like(p)
    f_loc = f[w0:w1].contiguous()
    for epoch in range(params.outer_syncs):
        if epoch > 0:
            exchange_halos(p, slabs, rank, zdim=1)
        for _ in range(params.inner_iters):
            ops.rof_iter(f_loc, p, q, params.lam)
            p, q = q, p
    # finish u = f + lam div p on this rank's core only: the ghost planes
    # refreshed from the neighbours' cores supply p at z0 - 1 (div reads
    # p at z - 1; the sub-slab's own first / last planes take the volume-
    # face formula and are dropped unless they are the volume's faces),
    # then one volume-sized gather of u instead of the 3-volume dual
    exchange_halos(p, slabs, rank, zdim=1)
    nz = f.shape[0]
    z0, z1 = s.core_range
    a, b = max(0, z0 - 1), min(nz, z1 + 1)
    if a >= w0 and b <= w1:
        ua = torch.empty((b - a,) + tuple(f.shape[1:]), dtype=f.dtype,
                         device=f.device)
        ops.rof_finish(f[a:b].contiguous(),
                       p.narrow(1, a - w0, b - a).contiguous(), ua,
                       params.lam)
        u_w = torch.zeros((w1 - w0,) + tuple(f.shape[1:]), dtype=f.dtype,
                          device=f.device)
        u_w[z0 - w0:z1 - w0] = ua[z0 - a:z1 - a]
        return gather_cores(u_w, slabs, rank, tuple(f.shape))
    # zero-depth halos: no ghost plane in the window, finish on the
    # gathered dual
    p_full = gather_cores(p, slabs, rank, None, zdim=1).contiguous()
    u = torch.empty_like(f)
    ops.rof_finish(f.contiguous(), p_full, u, params.lam)
    return u


def _halo_fits(slabs) -> bool:
    try:
        _check_halo(slabs)
    except ValueError:
        return False
    return all(t.core_range[1] > t.core_range[0] for t in slabs)


def minimize_sharded(core: torch.Tensor, cores, params, rank: int,
                     ops=CudaTvOps) -> torch.Tensor:
    """split_minimize on a slab-sharded volume: rank r holds planes
    ``cores[r]`` (``core``) and gets back its planes of the result -- the
    full volume is never assembled.  Ghost planes come from the +-1
    neighbours' cores (exchange_halos) when every halo fits inside the
    neighbouring core; otherwise (halo deeper than a neighbour's slab) each
    refresh all-gathers the cores and cuts the window from the full volume
    (correct for any partition, at a volume's worth of traffic).  Matches
    the single-process split_minimize on the same slab partition."""
    from .regularization import HaloSlab, NormMode, TvMinimizer
    d = params.effective_halo()
    n_z = cores[-1][1]
    slabs = [HaloSlab((z0, z1), d, (max(0, z0 - d), min(n_z, z1 + d)))
             for z0, z1 in cores]
    s = slabs[rank]
    (z0, z1), (w0, w1) = s.core_range, s.window
    c = s.core_in_window
    plane_shape = tuple(core.shape[1:])
    total = n_z * math.prod(plane_shape)
    exchange = _halo_fits(slabs)

    def refresh(w, zdim=0):
        if exchange:
            exchange_halos(w, slabs, rank, zdim)
        else:
            full = gather_cores(w, slabs, rank, None, zdim)
            w.copy_(full.narrow(zdim, w0, w1 - w0))

    if params.minimizer is TvMinimizer.GRADIENT_DESCENT:
        w = torch.zeros((w1 - w0,) + plane_shape, dtype=torch.float32,
                        device=core.device)
        w[c].copy_(core)
        spare = torch.empty_like(w)
        ss = torch.zeros(1, dtype=torch.float64, device=w.device)
        exact = params.norm_mode is NormMode.EXACT_GLOBAL
        scale = 1.0 if exact else float(np.sqrt(total / max(1, w.numel())))
        stored = hasattr(ops, "grad_store")
        g = torch.empty_like(w) if stored else None
        for _ in range(params.outer_syncs):
            refresh(w)
            for _ in range(params.inner_iters):
                band = (c.start, c.stop) if exact else (0, w.shape[0])
                if stored:
                    ops.grad_store(w, g, band, ss)
                else:
                    ops.grad_sumsq(w, band, ss)
                if exact:
                    if ss.is_cuda and dist.get_backend() != "nccl":
                        h = ss.cpu()
                        dist.all_reduce(h)
                        ss.copy_(h)
                    else:
                        dist.all_reduce(ss)
                if stored:
                    ops.step_g(w, g, spare, params.step, ss, scale)
                else:
                    ops.step(w, spare, params.step, ss, scale)
                w, spare = spare, w
        return w[c].contiguous()
    # ROF: f's window is fixed; the dual p gets fresh ghosts every epoch and
    # once more before the finish u = f + lam div p (div reads p at z - 1)
    f = torch.zeros((w1 - w0,) + plane_shape, dtype=torch.float32,
                    device=core.device)
    f[c].copy_(core)
    refresh(f)
    p = torch.zeros((3, w1 - w0) + plane_shape, dtype=torch.float32,
                    device=core.device)
    q = torch.empty_like(p)
    for epoch in range(params.outer_syncs):
        if epoch > 0:
            refresh(p, 1)
        for _ in range(params.inner_iters):
            ops.rof_iter(f, p, q, params.lam)
            p, q = q, p
    refresh(p, 1)
    u = torch.empty_like(f)
    ops.rof_finish(f, p, u, params.lam)
    return u[c].contiguous()
