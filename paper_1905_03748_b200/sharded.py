"""Slab-sharded multi-GPU operators and loops (one process per GPU).

The distributed form of the scheduled operators (execution.py:175-317,
scheduler.py:150-166) and of the loops built on them (algorithms.py:204-304),
laid out the way north_star asks: the volume is cut into axial slabs, one
per rank, and the projections into angle shards, one per rank --

* ``forward``: every rank projects ITS slab for every view of the range
  (slab-clipped partial projections, v-band culled: a slab's cone shadow
  covers only a band of detector rows) and the partials are summed by one
  reduce-scatter per round of views, which leaves each view's sum on the
  rank that owns the view (the reference's "partial projections summed
  across slabs", execution.py:224-235, done by NCCL over NVLink instead of
  through host memory);
* ``backward``: every rank needs every view for its slab, so the angle
  shards are all-gathered one round at a time and each rank backprojects
  into its own slab -- no reduction (Atb is slab-partition invariant,
  SURVEY 0.5).

Rounds are double-buffered: round j's collective runs on NCCL's stream
while round j+1's kernels run on the compute stream.  Nothing is ever
replicated: per rank the loops hold 1/N of every volume vector and 1/N of
every projection vector, so config 5 (4096^3, 256 GiB) runs in-core over 8
B200s.  Scalars (CGLS's gamma / delta / residual) are fp64
all-reduces.

The kernels and vector algebra are pluggable (``kernels``, ``vec``) so the
partition and exchange logic is tested with the gloo backend on CPU
(tests/test_distributed.py); the defaults are the sm_100a kernels.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import kernels as K
from .geometry import ScanGeometry
from .projectors import ProjectionMethod
from .scheduler import even_angle_ranges

__all__ = ["slab_partition", "view_shards", "ShardedOperators", "CudaVecOps",
           "cgls_sharded", "os_sart_sharded", "block_rows"]

INVERSE_GUARD = 1e-8
CG_BREAKDOWN = 1e-30
ROUND_BYTES = 512 << 20  # per-rank round of views (partials or gathered)


def slab_partition(n_z: int, world: int) -> list[tuple[int, int]]:
    """Axial slab of each rank: [n_z r // N, n_z (r+1) // N) (balanced;
    empty when n_z < N)."""
    return [(n_z * r // world, n_z * (r + 1) // world) for r in range(world)]


def view_shards(a0: int, a1: int, world: int) -> list[tuple[int, int]]:
    """Angle shard of each rank within [a0, a1): the reference's even split
    (scheduler.py:164-166) applied to the range."""
    return [(a0 + s0, a0 + s1) for s0, s1 in even_angle_ranges(a1 - a0, world)]


def block_rows(blocks, world: int, rank: int):
    """For OS-SART blocks: this rank's shard of each block and its row
    offset in the rank's local projection array (the shards concatenated in
    block order)."""
    out, off = [], 0
    for b0, b1 in blocks:
        s0, s1 = view_shards(b0, b1, world)[rank]
        out.append(((b0, b1), (s0, s1), off))
        off += s1 - s0
    return out, off


# ---------------------------------------------------------------- plumbing

class _Done:
    def wait(self):
        return None


def _nccl() -> bool:
    return dist.get_backend() == "nccl"


def _reduce_scatter(out: torch.Tensor, buf: torch.Tensor, rank: int,
                    world: int):
    """out = sum over ranks of buf[rank * C:(rank + 1) * C]; async on NCCL."""
    if _nccl():
        return dist.reduce_scatter_tensor(out, buf, async_op=True)
    # gloo (CPU tests, ranks sharing one GPU): same sums, synchronous,
    # through host memory
    h = buf.cpu() if buf.is_cuda else buf
    dist.all_reduce(h)
    c = out.shape[0]
    out.copy_(h[rank * c:(rank + 1) * c])
    return _Done()


def _all_gather(buf: torch.Tensor, mine: torch.Tensor, world: int):
    """buf[s * C:(s + 1) * C] = rank s's ``mine``; async on NCCL."""
    if _nccl():
        return dist.all_gather_into_tensor(buf, mine, async_op=True)
    c = mine.shape[0]
    if buf.is_cuda:  # gloo with ranks sharing one GPU: through host memory
        h = buf.cpu()
        dist.all_gather(list(h.split(c)), mine.cpu())
        buf.copy_(h)
    else:
        dist.all_gather(list(buf.split(c)), mine)
    return _Done()


def allreduce_(t: torch.Tensor) -> torch.Tensor:
    """In-place sum across ranks (fp64 scalars; device or host)."""
    if t.is_cuda and not _nccl():
        h = t.cpu()
        dist.all_reduce(h)
        t.copy_(h)
    else:
        dist.all_reduce(t)
    return t


class CudaVecOps:
    """Loop algebra of csrc/vector.cu (fp64 device scalars)."""

    @staticmethod
    def dot(a, b=None):
        out = torch.empty(1, dtype=torch.float64, device=a.device)
        if a.numel() == 0:
            return out.zero_()
        return K.dot(a, a if b is None else b, out)

    axpy_ratio = staticmethod(K.axpy_ratio)
    xpay_ratio = staticmethod(K.xpay_ratio)
    sart_update = staticmethod(K.sart_update)
    weighted_residual = staticmethod(K.weighted_residual)

    @staticmethod
    def guarded_inverse(a):
        return K.guarded_inverse(a, a)


class _CudaKernels:
    fwd_interp = staticmethod(lambda *a, **k: K.fwd_interp(*a, **k))
    fwd_siddon = staticmethod(lambda *a, **k: K.fwd_siddon(*a, **k))
    bwd_matched = staticmethod(lambda *a, **k: K.bwd_matched(*a, **k))


# --------------------------------------------------------------- operators

_EXCHANGES: dict = {}     # peer exchanges by (process group, rank, shape)
_HOST_GROUPS: dict = {}   # gloo group per NCCL process group (host barrier)


@dataclass
class ShardedOperators:
    """A / A^T with the volume slab-sharded and the views angle-sharded.

    ``forward(x_slab, out, (a0, a1))``: out (this rank's shard of the views,
    ``view_shards(a0, a1, N)[rank]``) = (A x)[shard].
    ``backward(y, out_slab, (a0, a1))``: out_slab += (A^T y) on this rank's
    planes; y = this rank's shard of [a0, a1).
    """

    geometry: ScanGeometry
    rank: int = 0
    world: int = 1
    method: ProjectionMethod = ProjectionMethod.INTERPOLATED
    round_views: int | None = None
    kernels: object = None

    def __post_init__(self):
        grid = self.geometry.voxel_grid
        self.slabs = slab_partition(grid.n_z, self.world)
        self.slab = self.slabs[self.rank]
        if self.kernels is None:
            self.kernels = _CudaKernels
        det = self.geometry.detector
        sheet = det.n_u * det.n_v * 4
        if self.round_views is None:
            self.round_views = max(1, min(64, ROUND_BYTES // max(
                1, self.world * sheet)))
        self._fwd = (self.kernels.fwd_interp
                     if self.method is ProjectionMethod.INTERPOLATED
                     else self.kernels.fwd_siddon)
        self._peer = None
        self._peer_tried = False

    def exchange(self, like: torch.Tensor | None = None):
        """The peer exchange (peer.py) when it is in use, else None (NCCL's
        collectives).  Set up on the first multi-rank operator call -- a
        collective, so every rank reaches it in the same call -- when the
        tensors are CUDA tensors and the kernels are the sm_100a ones."""
        if self._peer_tried or self.world == 1:
            return self._peer
        if like is None or not like.is_cuda or \
                self.kernels is not _CudaKernels:
            return None
        from .peer import PeerExchange, peer_mode_requested
        self._peer_tried = True
        if not peer_mode_requested():
            return None
        # one exchange (buffers, mappings, events, gloo group) per process
        # group and shape, shared by every ShardedOperators the loops
        # create: the ranks reach this point in the same order
        det = self.geometry.detector
        pg = dist.distributed_c10d._get_default_group()
        key = (id(pg), self.rank, self.world, like.device.index,
               self.round_views, det.n_v, det.n_u)
        if key not in _EXCHANGES:
            if _nccl():
                if id(pg) not in _HOST_GROUPS:
                    _HOST_GROUPS[id(pg)] = dist.new_group(backend="gloo")
                group = _HOST_GROUPS[id(pg)]
            else:
                group = None
            _EXCHANGES[key] = PeerExchange.create(
                self.rank, self.world, like.device, self.round_views,
                (det.n_v, det.n_u), group, self.geometry)
        self._peer = _EXCHANGES[key]
        return self._peer

    @property
    def exchange_mode(self) -> str:
        if self.world == 1:
            return "none"
        return "peer" if self._peer is not None else "collective"

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        """Sum a (scalar) tensor over the ranks; identity on one rank."""
        return allreduce_(t) if self.world > 1 else t

    # shapes ------------------------------------------------------------
    def slab_shape(self):
        g = self.geometry.voxel_grid
        return (self.slab[1] - self.slab[0], g.n_y, g.n_x)

    def shard(self, angle_range) -> tuple[int, int]:
        return view_shards(*angle_range, self.world)[self.rank]

    def _rounds(self, angle_range):
        shards = view_shards(*angle_range, self.world)
        longest = max(s1 - s0 for s0, s1 in shards)
        c = self.round_views
        return shards, c, -(-longest // c) if longest else 0

    def _sheet(self, n, like):
        det = self.geometry.detector
        return torch.empty((n, det.n_v, det.n_u), dtype=torch.float32,
                           device=like.device)

    # forward -----------------------------------------------------------
    def forward(self, x_slab: torch.Tensor, out: torch.Tensor,
                angle_range) -> torch.Tensor:
        a0, a1 = angle_range
        z0, z1 = self.slab
        if self.world == 1:
            if a1 > a0:
                self._fwd(x_slab, self.geometry, (a0, a1), (z0, z1), out)
            return out
        if self.exchange(x_slab) is not None:
            return self._forward_peer(x_slab, out, angle_range)
        shards, c, rounds = self._rounds(angle_range)
        m0, _ = shards[self.rank]
        bufs = [self._sheet(self.world * c, out) for _ in range(min(2, rounds))]
        recv = [self._sheet(c, out) for _ in range(min(2, rounds))]
        pending = [None, None]

        def land(p):
            work, rbuf, lo, hi = p
            work.wait()
            if hi > lo:
                out[lo - m0:hi - m0].copy_(rbuf[:hi - lo])

        for j in range(rounds):
            slot = j % 2
            if pending[slot] is not None:   # buffers of round j - 2
                land(pending[slot])
                pending[slot] = None
            buf = bufs[slot]
            for s, (s0, s1) in enumerate(shards):
                c0, c1 = s0 + j * c, min(s0 + (j + 1) * c, s1)
                if c1 <= c0:
                    continue
                part = buf[s * c:s * c + (c1 - c0)]
                if z1 > z0:
                    self._fwd(x_slab, self.geometry, (c0, c1), (z0, z1), part)
                else:
                    part.zero_()
            lo, hi = m0 + j * c, min(m0 + (j + 1) * c, shards[self.rank][1])
            work = _reduce_scatter(recv[slot], buf, self.rank, self.world)
            pending[slot] = (work, recv[slot], lo, max(lo, hi))
        for p in pending:
            if p is not None:
                land(p)
        return out

    def _forward_peer(self, x_slab, out, angle_range, b=None, w=None):
        """forward over peer memory (peer.py): per round, this rank's Ax
        kernels store the partials of shard s straight into rank s's inbox
        slot (P2P stores); after the round's barrier the side stream sums
        this rank's inbox in rank order into ``out`` (with b / w: the
        residual w o (b - sum)) while the compute stream moves on."""
        X = self._peer
        z0, z1 = self.slab
        shards, c, rounds = self._rounds(angle_range)
        m0, m1 = shards[self.rank]
        cur = torch.cuda.current_stream()
        X.side.wait_stream(cur)          # out / b / w are ready on cur
        for j in range(rounds):
            slot = X.next_slot("fwd")
            for s, (s0, s1) in enumerate(shards):
                c0, c1 = s0 + j * c, min(s0 + (j + 1) * c, s1)
                if c1 <= c0:
                    continue
                cur.wait_event(X.peer_ev[s]["consumed"][slot])
                part = X.inboxes[s][slot, self.rank, :c1 - c0]
                if z1 > z0:
                    self._fwd(x_slab, self.geometry, (c0, c1), (z0, z1), part)
                else:
                    K.fill(part, 0.0)
            X.record(cur, "written", slot)
            X.barrier()
            lo, hi = m0 + j * c, min(m0 + (j + 1) * c, m1)
            if hi > lo:
                X.wait_all(X.side, "written", slot)
                rows = slice(lo - m0, hi - m0)
                K.sum_slices(X.inbox[slot, :, :hi - lo], out[rows],
                             None if b is None else b[rows],
                             None if w is None else w[rows], stream=X.side)
            X.record(X.side, "consumed", slot)
        cur.wait_stream(X.side)
        return out

    def forward_residual(self, x_slab: torch.Tensor, b: torch.Tensor,
                         w: torch.Tensor | None, out: torch.Tensor,
                         angle_range) -> torch.Tensor:
        """out = w o (b - A x) on this rank's shard of angle_range.  One GPU
        with the interpolated projector: K1's fused residual epilogue (no
        separate pass over the projections); otherwise forward + cs_weighted_
        residual (also when the slab is too tall for the fused kernel's
        layered texture)."""
        if (self.world == 1 and self.kernels is _CudaKernels
                and self.method is ProjectionMethod.INTERPOLATED
                and angle_range[1] > angle_range[0]):
            from ._lib import ConesplitCudaError
            try:
                return K.fwd_interp_residual(x_slab, self.geometry,
                                             angle_range, b, w, out)
            except ConesplitCudaError as e:
                if e.code != -3:  # CS_ERR_UNSUPPORTED: nz > layer limit
                    raise
        if self.world > 1 and self.exchange(x_slab) is not None:
            return self._forward_peer(x_slab, out, angle_range, b, w)
        self.forward(x_slab, out, angle_range)
        return self._vec_residual(out, b, w)

    def _vec_residual(self, out, b, w):
        vec = getattr(self.kernels, "weighted_residual", None)
        if vec is None:
            return K.weighted_residual(out, b, w)
        return vec(out, b, w)

    # backward ----------------------------------------------------------
    def backward(self, y: torch.Tensor, out_slab: torch.Tensor,
                 angle_range) -> torch.Tensor:
        a0, a1 = angle_range
        z0, z1 = self.slab
        if self.world == 1:
            if a1 > a0:
                self.kernels.bwd_matched(y, self.geometry, (a0, a1), (z0, z1),
                                         out_slab)
            return out_slab
        if self.exchange(y) is not None:
            return self._backward_peer(y, out_slab, angle_range)
        shards, c, rounds = self._rounds(angle_range)
        m0, m1 = shards[self.rank]
        nbuf = min(2, rounds)
        gbufs = [self._sheet(self.world * c, y) for _ in range(nbuf)]
        sends = [self._sheet(c, y) for _ in range(nbuf)]

        def issue(j):
            slot = j % 2
            lo, hi = m0 + j * c, min(m0 + (j + 1) * c, m1)
            if hi > lo:
                sends[slot][:hi - lo].copy_(y[lo - m0:hi - m0])
            return _all_gather(gbufs[slot], sends[slot], self.world)

        work = issue(0) if rounds else None
        for j in range(rounds):
            nxt = issue(j + 1) if j + 1 < rounds else None  # prefetch
            work.wait()
            g = gbufs[j % 2]
            if z1 > z0:
                for s, (s0, s1) in enumerate(shards):
                    c0, c1 = s0 + j * c, min(s0 + (j + 1) * c, s1)
                    if c1 > c0:
                        self.kernels.bwd_matched(
                            g[s * c:s * c + (c1 - c0)], self.geometry,
                            (c0, c1), (z0, z1), out_slab)
            work = nxt
        return out_slab

    def _backward_peer(self, y, out_slab, angle_range):
        """backward over peer memory: per round, the side stream stages this
        rank's views in its outbox slot (once every reader of the slot's
        previous round is done); after the barrier the matched kernels read
        every owner's outbox in place (P2P loads)."""
        X = self._peer
        z0, z1 = self.slab
        shards, c, rounds = self._rounds(angle_range)
        m0, m1 = shards[self.rank]
        cur = torch.cuda.current_stream()
        X.side.wait_stream(cur)          # y is ready on cur
        for j in range(rounds):
            slot = X.next_slot("bwd")
            lo, hi = m0 + j * c, min(m0 + (j + 1) * c, m1)
            X.wait_all(X.side, "read", slot)
            if hi > lo:
                with torch.cuda.stream(X.side):
                    X.outbox[slot, :hi - lo].copy_(y[lo - m0:hi - m0])
            X.record(X.side, "staged", slot)
            X.barrier()
            for s, (s0, s1) in enumerate(shards):
                c0, c1 = s0 + j * c, min(s0 + (j + 1) * c, s1)
                if c1 > c0 and z1 > z0:
                    cur.wait_event(X.peer_ev[s]["staged"][slot])
                    self.kernels.bwd_matched(
                        X.outboxes[s][slot, :c1 - c0], self.geometry,
                        (c0, c1), (z0, z1), out_slab)
            X.record(cur, "read", slot)
        cur.wait_stream(X.side)
        return out_slab


# ------------------------------------------------------------------- loops

def _zeros(shape, like):
    return torch.zeros(shape, dtype=torch.float32, device=like.device)


def cgls_sharded(b: torch.Tensor, ops: ShardedOperators, iterations: int,
                 vec=CudaVecOps):
    """CGLS on the normal equations from zero (algorithms.py:204-246) with
    x, p, s slab-sharded and b, r, q angle-sharded (b = this rank's shard of
    all views).  Returns (x_slab, residuals, breakdown)."""
    na = ops.geometry.n_angles
    full = (0, na)
    b_norm = math.sqrt(float(ops.allreduce_(vec.dot(b)).item()))
    x = _zeros(ops.slab_shape(), b)
    residuals: list[float] = []
    if b_norm == 0.0:
        return x, residuals, False
    r = b.clone()
    s = _zeros(ops.slab_shape(), b)
    ops.backward(r, s, full)
    p = s.clone()
    gamma = ops.allreduce_(vec.dot(s))
    q = torch.empty_like(b)
    breakdown = False
    for _ in range(iterations):
        ops.forward(p, q, full)
        delta = ops.allreduce_(vec.dot(q))
        if float(delta.item()) < CG_BREAKDOWN or \
                float(gamma.item()) < CG_BREAKDOWN:
            breakdown = True
            break
        vec.axpy_ratio(x, p, gamma, delta, +1.0)    # x += alpha p
        vec.axpy_ratio(r, q, gamma, delta, -1.0)    # r -= alpha q
        rr = ops.allreduce_(vec.dot(r))
        residuals.append(math.sqrt(float(rr.item())) / b_norm)
        s.zero_()
        ops.backward(r, s, full)
        gamma_new = ops.allreduce_(vec.dot(s))
        vec.xpay_ratio(p, s, gamma_new, gamma)      # p = s + beta p
        gamma = gamma_new
    return x, residuals, breakdown


def os_sart_sharded(b_local: torch.Tensor, ops: ShardedOperators, blocks,
                    iterations: int, relaxation: float, tv=None,
                    tv_ops=None, vec=CudaVecOps,
                    weight_budget: int | None = None, tv_step=None):
    """OS-SART (algorithms.py:261-304): per block S,
    x += lambda V_S o A_S^T W_S (b_S - A_S x), x slab-sharded, the views of
    every block angle-sharded (``b_local`` = this rank's shards of the
    blocks in order, see block_rows).  W_S / V_S are the guarded inverses of
    A_S 1 / A_S^T 1; the V_S of all blocks are kept while they fit
    ``weight_budget`` bytes, else recomputed per block (one more A^T per
    block and iteration for the blocks beyond the budget, instead of
    n_blocks slab-sized buffers).  ``tv``
    (TvParams) runs the halo-exchanged TV step after every iteration
    (``tv_step(x) -> x`` replaces it, e.g. the single-GPU split_minimize)."""
    rows, n_local = block_rows(blocks, ops.world, ops.rank)
    assert b_local.shape[0] == n_local, (b_local.shape, n_local)
    shape = ops.slab_shape()
    # decided on the thickest slab: every rank must take the same branch
    # (the operators are collectives)
    slab_bytes = 4 * shape[1] * shape[2] * max(z1 - z0 for z0, z1 in ops.slabs)
    if weight_budget is None:
        weight_budget = 1 << 62
    # as many blocks' V_S as fit are kept, the rest recomputed per block
    n_keep = min(len(blocks), int(weight_budget // max(slab_bytes, 1)))
    ones_slab = torch.ones(shape, dtype=torch.float32, device=b_local.device)
    w_all = torch.empty_like(b_local)

    def col_inverse(b0, b1, s0, s1):
        ones = torch.ones((s1 - s0,) + tuple(b_local.shape[1:]),
                          dtype=torch.float32, device=b_local.device)
        v = _zeros(shape, b_local)
        ops.backward(ones, v, (b0, b1))
        return vec.guarded_inverse(v)

    vs = []
    for (b0, b1), (s0, s1), off in rows:
        w = w_all[off:off + s1 - s0]
        ops.forward(ones_slab, w, (b0, b1))
        vec.guarded_inverse(w)
        vs.append(col_inverse(b0, b1, s0, s1) if len(vs) < n_keep else None)
    del ones_slab
    x = _zeros(shape, b_local)
    upd = torch.zeros_like(x)
    longest = max((s1 - s0 for _, (s0, s1), _ in rows), default=0)
    res_buf = torch.empty((longest,) + tuple(b_local.shape[1:]),
                          dtype=torch.float32, device=b_local.device)
    for _ in range(iterations):
        for i, ((b0, b1), (s0, s1), off) in enumerate(rows):
            res = res_buf[:s1 - s0]
            if vec is CudaVecOps:
                ops.forward_residual(x, b_local[off:off + s1 - s0],
                                     w_all[off:off + s1 - s0], res, (b0, b1))
            else:
                ops.forward(x, res, (b0, b1))
                vec.weighted_residual(res, b_local[off:off + s1 - s0],
                                      w_all[off:off + s1 - s0])
            ops.backward(res, upd, (b0, b1))
            v = vs[i] if vs[i] is not None else col_inverse(b0, b1, s0, s1)
            vec.sart_update(x, upd, v, relaxation)
        if tv_step is not None:
            x = tv_step(x)
        elif tv is not None:
            from .halo import minimize_sharded
            x = minimize_sharded(x, ops.slabs, tv, ops.rank,
                                 **({} if tv_ops is None else {"ops": tv_ops}))
    return x
