"""Planned execution of Ax / Atb over a device pool on CUDA streams -- the
paper's Algorithms 1 and 2 rebuilt B200-first; drop-in for
conesplit.execution (/root/reference/pkg/src/conesplit/execution.py).

Per device (one host thread per GPU of the pool; with torch.distributed
initialised and world_size == len(pool), rank r is device r):

* three streams -- ``h2d`` (slab / projection uploads), ``compute``
  (kernels), ``d2h`` (drains) -- ordered by CUDA events, so slab s+1 uploads
  while slab s projects and slab s-1 drains (double buffering);
* forward (Alg. 1, execution.py:175-246): the device's angle window
  (``plan.angle_assignment``) stays resident in HBM as an fp32 accumulator;
  slab 0 overwrites it and later slabs add into it inside the Ax epilogue
  (the reference's host-side TransferIn-partial + Accumulate of
  execution.py:224-235 fused into K1);
* backward (Alg. 2, execution.py:249-317): projections are uploaded once
  when they fit beside the slab buffers (else streamed in plan chunks per
  slab); each owned slab is zeroed, backprojected over every angle and
  drained on the host while the next slab computes.
  Slabs are dealt round-robin over ``max(plan.n_splits, n_devices)`` equal
  slabs, so every GPU works even when one slab would fit (SURVEY 0.6 --
  legal because Atb is slab-partition invariant);
* host images (numpy or file-backed memmaps) stream through a bounded
  ring of pinned slots with multi-threaded host copies (no page-locking of
  whole images); device-resident inputs skip the transfers;
* every transfer and kernel is bracketed by CUDA events and reported as an
  :class:`ExecutionTrace` (``simulated=False``) whose per-device high-water
  is the executor's own allocation ledger -- check_trace() applies.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .geometry import ScanGeometry
from .projectors import (
    BackwardTileSpec,
    ForwardTileSpec,
    ProjectionMethod,
    ProjectionStack,
    Volume,
    WeightMode,
)
from .scheduler import (
    HOST,
    SCALAR_BYTES,
    BudgetExceededError,
    DevicePool,
    ExecutionTrace,
    OpKind,
    SplitPlan,
    TraceEvent,
    slab_ranges,
)

__all__ = ["execute_forward", "execute_backward", "dist_info"]


def dist_info():
    """(rank, world) when torch.distributed is initialised, else (0, 1)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


# --------------------------------------------------------------------------
# per-device worker state


@dataclass
class _Ev:
    kind: str
    payload: str
    nbytes: int
    start: torch.cuda.Event
    end: torch.cuda.Event


@dataclass
class _Device:
    index: int
    cuda: torch.device
    budget: int
    allocated: int = 0
    high_water: int = 0
    events: list = field(default_factory=list)

    def __post_init__(self):
        with torch.cuda.device(self.cuda):
            self.compute = torch.cuda.Stream(self.cuda)
            self.h2d = torch.cuda.Stream(self.cuda)
            self.d2h = torch.cuda.Stream(self.cuda)
            self.t_zero = torch.cuda.Event(enable_timing=True)
            self.t_zero.record(torch.cuda.current_stream(self.cuda))

    @property
    def name(self) -> str:
        return f"dev{self.index}"

    def alloc(self, shape, nbytes=None) -> torch.Tensor:
        nbytes = int(np.prod(shape)) * SCALAR_BYTES if nbytes is None \
            else nbytes
        self.allocated += nbytes
        self.high_water = max(self.high_water, self.allocated)
        if self.allocated > self.budget:
            raise BudgetExceededError(
                f"{self.name}: {self.allocated} B allocated exceeds budget "
                f"{self.budget} B")
        return torch.empty(shape, dtype=torch.float32, device=self.cuda)

    def free(self, nbytes: int):
        self.allocated -= nbytes

    def begin(self, stream, kind, payload, nbytes=0) -> _Ev:
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ev = _Ev(kind, payload, nbytes, s, e)
        self.events.append((ev, stream))
        return ev

    @staticmethod
    def end(ev: _Ev, stream):
        ev.end.record(stream)

    def trace_events(self) -> list[TraceEvent]:
        out = []
        for ev, _ in self.events:
            ev.end.synchronize()
            out.append(TraceEvent(
                self.name, ev.kind, ev.payload,
                self.t_zero.elapsed_time(ev.start) * 1e-3,
                self.t_zero.elapsed_time(ev.end) * 1e-3, ev.nbytes))
        return out


def _cuda_device(pool: DevicePool, i: int) -> torch.device:
    n = torch.cuda.device_count()
    if n == 0:
        raise RuntimeError("no CUDA device visible (no CPU fallback)")
    # abstract pools larger than the box share GPUs (like the reference's
    # host-backed virtual devices)
    return torch.device("cuda", pool.cuda_index(i) % n)


_COPY_POOL = None
_COPY_LOCK = threading.Lock()
_PIECE_BYTES = 64 << 20   # one pinned ring slot
_RING_SLOTS = 4


def _copy_pool():
    global _COPY_POOL
    with _COPY_LOCK:
        if _COPY_POOL is None:
            import concurrent.futures
            import os
            _COPY_POOL = concurrent.futures.ThreadPoolExecutor(
                max_workers=max(2, min(16, os.cpu_count() or 2)),
                thread_name_prefix="cs-copy")
        return _COPY_POOL


def _par_copy(dst: np.ndarray, src: np.ndarray):
    """dst[:] = src for 1-D float32 arrays, split over the copy pool (numpy
    releases the GIL): host memcpy at ~10 GB/s per core would otherwise be
    the bottleneck of streamed passes."""
    n = src.shape[0]
    parts = min(16, max(1, (n * 4) >> 22))  # >= 4 MiB per part
    if parts == 1:
        np.copyto(dst, src)
        return
    step = -(-n // parts)
    futs = [_copy_pool().submit(np.copyto, dst[j:j + step], src[j:j + step])
            for j in range(0, n, step)]
    for f in futs:
        f.result()


class _HostLink:
    """Host <-> device streaming through a bounded ring of pinned slots
    (4 x 64 MiB, cached by torch's pinned allocator across passes): every
    piece is copied between the host array and a slot by the copy pool and
    moved by DMA on the caller's stream; a slot is refilled only after its
    DMA completed.  Nothing is page-locked in place, so host images of any
    size -- including file-backed memmaps (fileio) -- stream at host-memcpy
    speed with bounded pinned memory (the paper's pinned double buffers,
    PAPER.md:106-110, instead of registering the whole image)."""

    def __init__(self):
        n = _PIECE_BYTES // 4
        self.slots = [torch.empty(n, dtype=torch.float32, pin_memory=True)
                      for _ in range(_RING_SLOTS)]
        self.busy = [None] * _RING_SLOTS
        self.next = 0

    def _slot(self) -> int:
        b = self.next % _RING_SLOTS
        self.next += 1
        if self.busy[b] is not None:
            self.busy[b].synchronize()
            self.busy[b] = None
        return b

    def h2d(self, dst: torch.Tensor, src: np.ndarray, stream):
        """Enqueue dst <- src (returns once every piece is in a slot)."""
        flat_d = dst.view(-1)
        flat_s = np.ascontiguousarray(src).reshape(-1)
        n = flat_s.shape[0]
        step = self.slots[0].numel()
        for off in range(0, n, step):
            m = min(step, n - off)
            b = self._slot()
            _par_copy(self.slots[b][:m].numpy(), flat_s[off:off + m])
            with torch.cuda.stream(stream):
                flat_d[off:off + m].copy_(self.slots[b][:m],
                                          non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            self.busy[b] = ev

    def d2h(self, dst: np.ndarray, src: torch.Tensor, stream):
        """dst <- src after the work already enqueued on ``stream``;
        returns when dst holds the data (DMA of piece k+1 overlaps the
        host copy of piece k)."""
        flat_s = src.reshape(-1)
        flat_d = dst.reshape(-1)
        assert np.shares_memory(flat_d, dst), "d2h needs a contiguous dst"
        n = flat_s.numel()
        step = self.slots[0].numel()
        pending = None

        def land(p):
            b, off, m, ev = p
            ev.synchronize()
            _par_copy(flat_d[off:off + m], self.slots[b][:m].numpy())

        for off in range(0, n, step):
            m = min(step, n - off)
            b = self._slot()
            with torch.cuda.stream(stream):
                self.slots[b][:m].copy_(flat_s[off:off + m],
                                        non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            self.busy[b] = ev
            if pending is not None:
                land(pending)
            pending = (b, off, m, ev)
        if pending is not None:
            land(pending)


def _upload(dst: torch.Tensor, src, stream, link: "_HostLink | None"):
    """H2D (host numpy via the pinned ring) or D2D of one slab / chunk."""
    if isinstance(src, np.ndarray):
        link.h2d(dst, src, stream)
        return
    with torch.cuda.stream(stream):
        dst.copy_(src, non_blocking=True)


def _refine_for_overlap(slabs, plane: int, fixed_bytes: int, budget: int,
                        max_factor: int = 4):
    """The plan's slabs are the fewest that fit one slab beside the other
    buffers (scheduler.py:169-210); with one slab buffer the upload of slab
    s+1 cannot overlap slab s's kernels.  Split every slab into the
    smallest number of equal parts (<= max_factor) for which two slab
    buffers fit beside ``fixed_bytes``, so transfers double-buffer.  (Slab
    results concatenate / add up exactly as the plan's -- Atb is
    slab-partition invariant, Ax partials differ by fp32 rounding only.)"""
    if len(slabs) < 2:
        return slabs
    longest = max(z1 - z0 for z0, z1 in slabs)
    if fixed_bytes + 2 * longest * plane * SCALAR_BYTES <= budget:
        return slabs
    for r in range(2, max_factor + 1):
        part = -(-longest // r)
        if fixed_bytes + 2 * part * plane * SCALAR_BYTES <= budget:
            out = []
            for z0, z1 in slabs:
                step = -(-(z1 - z0) // r)
                out.extend((z, min(z + step, z1)) for z in range(z0, z1, step))
            return tuple(out)
    return slabs


def _join_streams(dev: _Device):
    """Order the caller's stream after the worker streams, so buffers the
    caching allocator hands back (allocated on the current stream) are not
    reused while side-stream work is in flight."""
    cur = torch.cuda.current_stream(dev.cuda)
    for s in (dev.h2d, dev.compute, dev.d2h):
        cur.wait_stream(s)


def _run_devices(work, n_devices: int):
    """Run work(i) for every device, one host thread each (ctypes and torch
    release the GIL while enqueuing); first failure is re-raised after all
    joined (execution.py:126-150)."""
    rank, world = dist_info()
    if world > 1 and world == n_devices:
        work(rank)
        return
    errors: list = [None] * n_devices
    if n_devices == 1:
        work(0)
        return

    def runner(i):
        try:
            work(i)
        except BaseException as e:  # noqa: BLE001 -- propagated below
            errors[i] = e

    threads = [threading.Thread(target=runner, args=(i,), name=f"dev{i}")
               for i in range(n_devices)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errors:
        if e is not None:
            raise e


def _validate(plan: SplitPlan, op: OpKind, geometry: ScanGeometry,
              pool: DevicePool):
    """execution.py:153-172."""
    if plan.op_kind is not op:
        raise ValueError(f"plan is for {plan.op_kind}, not {op}")
    if plan.n_z != geometry.voxel_grid.n_z:
        raise ValueError("plan slab ranges do not cover the volume")
    if op is OpKind.FORWARD:
        if len(plan.angle_assignment) != len(pool):
            raise ValueError("plan angle assignment does not match the pool")
        pos = 0
        for a0, a1 in sorted(plan.angle_assignment):
            if a0 != pos:
                raise ValueError("forward plan angles are not a partition")
            pos = max(pos, a1)
        if pos != geometry.n_angles:
            raise ValueError("forward plan does not cover all angles")
    elif plan.angle_assignment[-1][1] != geometry.n_angles:
        raise ValueError("backward plan does not cover all angles")


def _finish(devs, host_events, trace_sink):
    events = list(host_events)
    high = {}
    for d in devs:
        if d is None:
            continue
        events.extend(d.trace_events())
        high[d.name] = d.high_water
    events.sort(key=lambda e: (e.start, e.device))
    span = (max(e.end for e in events) - min(e.start for e in events)
            if events else 0.0)
    trace = ExecutionTrace(events, high, span, simulated=False)
    if trace_sink is not None:
        trace_sink.append(trace)
    return trace


def _allgather_rows(t: torch.Tensor, ranges, rank: int) -> torch.Tensor:
    """Assemble a tensor partitioned along dim 0 by ``ranges`` (one per
    rank) on every rank: pad to the largest part, all_gather, trim."""
    import torch.distributed as dist
    longest = max(b - a for a, b in ranges)
    mine = ranges[rank][1] - ranges[rank][0]
    pad = torch.zeros((longest,) + tuple(t.shape[1:]), dtype=t.dtype,
                      device=t.device)
    if mine:
        pad[:mine].copy_(t[:mine])
    parts = [torch.empty_like(pad) for _ in ranges]
    dist.all_gather(parts, pad)
    return torch.cat([p[:b - a] for p, (a, b) in zip(parts, ranges)], 0)


# --------------------------------------------------------------------------
# forward (Algorithm 1)


def execute_forward(volume: Volume, geometry: ScanGeometry, pool: DevicePool,
                    plan: SplitPlan,
                    method: ProjectionMethod = ProjectionMethod.SIDDON,
                    tiles: ForwardTileSpec = ForwardTileSpec(),
                    trace_sink: list | None = None) -> ProjectionStack:
    """Run a planned forward pass (execution.py:175-246); equals the
    monolithic projection of the full volume.

    Per device: when its angle window fits beside two slab buffers, the
    window stays resident as the accumulator (slab s+1 uploads while slab s
    projects; later slabs accumulate in the kernel epilogue).  Otherwise the
    window is processed in ``plan.chunk_angles`` chunks exactly as
    Algorithm 1: per slab, per chunk, the partial projection is staged back
    in (TransferIn), accumulated by the kernel and drained (TransferOut).
    Host images that are not page-locked (file-backed memmaps) stream
    through pinned staging buffers."""
    _validate(plan, OpKind.FORWARD, geometry, pool)
    grid, det = geometry.voxel_grid, geometry.detector
    if volume.slab_range != (0, grid.n_z):
        raise ValueError("forward execution needs the full host volume")
    on_dev = volume.on_device
    n_angles = geometry.n_angles
    plane = grid.n_x * grid.n_y
    sheet = det.n_u * det.n_v
    parts: list = [None] * len(pool)
    devs: list = [None] * len(pool)
    host_events: list = []
    fwd = K.fwd_interp if method is ProjectionMethod.INTERPOLATED \
        else K.fwd_siddon
    def work(i: int):
        a0, a1 = plan.angle_assignment[i]
        if a1 <= a0:
            return
        dev = _Device(i, _cuda_device(pool, i), pool.devices[i].memory_budget)
        devs[i] = dev
        with torch.cuda.device(dev.cuda):
            src = volume.data
            if on_dev and src.device == dev.cuda and plan.n_splits == 1:
                # device-resident input that fits: no staging
                acc = dev.alloc((a1 - a0, det.n_v, det.n_u))
                ev = dev.begin(dev.compute, "Kernel", "s0.c0")
                with torch.cuda.stream(dev.compute):
                    dev.compute.wait_stream(torch.cuda.current_stream(
                        dev.cuda))
                    fwd(src, geometry, (a0, a1), (0, grid.n_z), acc,
                        False, dev.compute)
                dev.end(ev, dev.compute)
                parts[i] = acc
                _join_streams(dev)
                return
            window = (a1 - a0) * sheet * SCALAR_BYTES
            slabs = _refine_for_overlap(plan.slab_ranges, plane, window,
                                        dev.budget)
            longest = max(z1 - z0 for z0, z1 in slabs)
            nbuf = 1 if len(slabs) == 1 else 2
            staging = _HostLink() if isinstance(src, np.ndarray) else None
            slab_bytes = longest * plane * SCALAR_BYTES
            if window + nbuf * slab_bytes <= dev.budget:
                parts[i] = _forward_resident(dev, src, slabs, nbuf, longest,
                                             staging, (a0, a1), on_dev)
            else:
                cbytes = 3 * plan.chunk_angles * sheet * SCALAR_BYTES
                if nbuf * slab_bytes + cbytes > dev.budget:
                    nbuf = 1  # the reference's one slab + three chunks
                parts[i] = _forward_chunked(dev, src, slabs, nbuf, longest,
                                            staging, (a0, a1),
                                            plan.chunk_angles)
            _join_streams(dev)

    def _forward_resident(dev, src, slabs, nbuf, longest, staging, window,
                          dev_out):
        a0, a1 = window
        acc = dev.alloc((a1 - a0, det.n_v, det.n_u))
        bufs = [dev.alloc((longest, grid.n_y, grid.n_x)) for _ in range(nbuf)]
        ready = [torch.cuda.Event() for _ in range(nbuf)]
        free = [None] * nbuf
        for si, (z0, z1) in enumerate(slabs):
            b = si % nbuf
            buf = bufs[b][:z1 - z0]
            if free[b] is not None:
                dev.h2d.wait_event(free[b])
            ev = dev.begin(dev.h2d, "TransferIn", f"slab{si}",
                           (z1 - z0) * plane * SCALAR_BYTES)
            _upload(buf, src[z0:z1], dev.h2d, staging)
            dev.end(ev, dev.h2d)
            ready[b].record(dev.h2d)
            dev.compute.wait_event(ready[b])
            ev = dev.begin(dev.compute, "Kernel" if si == 0 else "Accumulate",
                           f"s{si}.c0")
            fwd(buf, geometry, (a0, a1), (z0, z1), acc, si > 0, dev.compute)
            dev.end(ev, dev.compute)
            fe = torch.cuda.Event()
            fe.record(dev.compute)
            free[b] = fe
        if dev_out:
            return acc
        out = np.empty(tuple(acc.shape), np.float32)
        dev.d2h.wait_stream(dev.compute)
        ev = dev.begin(dev.d2h, "TransferOut", "out",
                       acc.numel() * SCALAR_BYTES)
        (staging or _HostLink()).d2h(out, acc, dev.d2h)
        dev.end(ev, dev.d2h)
        return out

    def _forward_chunked(dev, src, slabs, nbuf, longest, staging, window,
                         chunk_angles):
        """Algorithm 1 proper: the device holds slab buffers and three chunk
        buffers; partial projections live on the host between slabs."""
        a0, a1 = window
        chunks = [(c, min(c + chunk_angles, a1))
                  for c in range(a0, a1, chunk_angles)]
        csize = chunk_angles * sheet
        res = np.empty((a1 - a0, det.n_v, det.n_u), np.float32)
        bufs = [dev.alloc((longest, grid.n_y, grid.n_x)) for _ in range(nbuf)]
        cbufs = [dev.alloc((csize,)) for _ in range(3)]
        pins = [torch.empty(csize, dtype=torch.float32, pin_memory=True)
                for _ in range(3)]
        slab_ready = [torch.cuda.Event() for _ in range(nbuf)]
        slab_free = [None] * nbuf
        cfree = [None] * 3       # compute done with a chunk buffer
        pending = []             # (pinned idx, event, c0, c1) drains
        k = 0

        def drain(upto_len):
            while len(pending) > upto_len:
                pb, e, c0, c1 = pending.pop(0)
                e.synchronize()
                n = (c1 - c0) * sheet
                res[c0 - a0:c1 - a0] = pins[pb][:n].numpy().reshape(
                    c1 - c0, det.n_v, det.n_u)

        for si, (z0, z1) in enumerate(slabs):
            b = si % nbuf
            buf = bufs[b][:z1 - z0]
            if slab_free[b] is not None:
                dev.h2d.wait_event(slab_free[b])
            ev = dev.begin(dev.h2d, "TransferIn", f"slab{si}",
                           (z1 - z0) * plane * SCALAR_BYTES)
            _upload(buf, src[z0:z1], dev.h2d, staging)
            dev.end(ev, dev.h2d)
            slab_ready[b].record(dev.h2d)
            drain(0)  # partials of slab si-1 are on the host
            for ci, (c0, c1) in enumerate(chunks):
                cb = k % 3
                k += 1
                n = (c1 - c0) * sheet
                cbuf = cbufs[cb][:n].view(c1 - c0, det.n_v, det.n_u)
                drain(2)  # pinned buffer cb is free once its drain is done
                if cfree[cb] is not None:
                    dev.h2d.wait_event(cfree[cb])
                if si > 0:
                    pins[cb][:n].numpy()[:] = res[c0 - a0:c1 - a0].reshape(-1)
                    ev = dev.begin(dev.h2d, "TransferIn", f"partial{ci}",
                                   n * SCALAR_BYTES)
                    with torch.cuda.stream(dev.h2d):
                        cbuf.view(-1).copy_(pins[cb][:n], non_blocking=True)
                    dev.end(ev, dev.h2d)
                dev.compute.wait_stream(dev.h2d)
                dev.compute.wait_event(slab_ready[b])
                ev = dev.begin(dev.compute,
                               "Kernel" if si == 0 else "Accumulate",
                               f"s{si}.c{ci}")
                fwd(buf, geometry, (c0, c1), (z0, z1), cbuf, si > 0,
                    dev.compute)
                dev.end(ev, dev.compute)
                dev.d2h.wait_stream(dev.compute)
                ev = dev.begin(dev.d2h, "TransferOut", f"chunk{ci}",
                               n * SCALAR_BYTES)
                with torch.cuda.stream(dev.d2h):
                    pins[cb][:n].copy_(cbuf.view(-1), non_blocking=True)
                dev.end(ev, dev.d2h)
                de = torch.cuda.Event()
                de.record(dev.d2h)
                cfree[cb] = de
                pending.append((cb, de, c0, c1))
            fe = torch.cuda.Event()
            fe.record(dev.compute)
            slab_free[b] = fe
        drain(0)
        return res

    _run_devices(work, len(pool))
    rank, world = dist_info()
    if world > 1 and world == len(pool):
        # every rank gets every rank's views, one bounded piece at a time,
        # straight into the output (a device tensor only for device input)
        shape = (n_angles, det.n_v, det.n_u)
        data = (torch.empty(shape, dtype=torch.float32,
                            device=volume.data.device) if on_dev
                else np.empty(shape, np.float32))
        _bcast_rows(data, parts[rank], plan.angle_assignment, rank)
    elif on_dev:
        data = torch.cat([torch.as_tensor(p).to(volume.data.device)
                          for p in parts if p is not None], 0)
    else:
        data = np.concatenate([p for p in parts if p is not None], 0)
    _finish(devs, host_events, trace_sink)
    return ProjectionStack(det, data, (0, n_angles))


# --------------------------------------------------------------------------
# backward (Algorithm 2)


def backward_slabs(plan: SplitPlan, n_devices: int):
    """Slab list actually executed: the plan's slabs, refined to at least
    one slab per device."""
    n = max(plan.n_splits, n_devices)
    return slab_ranges(plan.n_z, min(n, plan.n_z))


def execute_backward(projections: ProjectionStack, geometry: ScanGeometry,
                     pool: DevicePool, plan: SplitPlan,
                     mode: WeightMode = WeightMode.FDK,
                     tiles: BackwardTileSpec = BackwardTileSpec(),
                     trace_sink: list | None = None,
                     out: Volume | None = None) -> Volume:
    """Run a planned backward pass (execution.py:249-317); equals the
    monolithic backprojection.

    Per device: when the whole projection set fits beside two slab
    buffers it is uploaded once; otherwise every owned slab streams all
    angle chunks through two chunk buffers (Algorithm 2 proper).  ``out``
    (optional, host or file-backed ``fileio.create_volume``) receives the
    result slab by slab instead of a fresh array."""
    _validate(plan, OpKind.BACKWARD, geometry, pool)
    grid, det = geometry.voxel_grid, geometry.detector
    if projections.angle_range != (0, geometry.n_angles):
        raise ValueError("backward execution needs the full projection set")
    on_dev = projections.on_device
    D = len(pool)
    slabs = backward_slabs(plan, D)
    queues = [list(range(d, len(slabs), D)) for d in range(D)]
    plane = grid.n_x * grid.n_y
    sheet = det.n_u * det.n_v
    if out is not None:
        if out.grid != grid or out.slab_range != (0, grid.n_z):
            raise ValueError("out must be a full volume on the scan grid")
        res = out.data
    elif on_dev:
        res = torch.zeros((grid.n_z, grid.n_y, grid.n_x), dtype=torch.float32,
                          device=projections.data.device)
    else:
        res = np.zeros((grid.n_z, grid.n_y, grid.n_x), np.float32)
    res_dev = isinstance(res, torch.Tensor) and res.is_cuda
    devs: list = [None] * D
    host_events: list = []
    bwd = K.bwd_fdk if mode is WeightMode.FDK else K.bwd_matched
    A = geometry.n_angles

    def work(i: int):
        if not queues[i]:
            return
        dev = _Device(i, _cuda_device(pool, i), pool.devices[i].memory_budget)
        devs[i] = dev
        with torch.cuda.device(dev.cuda):
            src = projections.data
            local = on_dev and src.device == dev.cuda
            # this device's slabs, refined for double buffering when the
            # budget only holds one slab beside the projections (uploaded
            # once when they fit, else streamed in plan chunks)
            C0 = min(plan.chunk_angles, A)
            mine = tuple(slabs[q] for q in queues[i])
            proj_bytes = 0 if local else A * sheet * SCALAR_BYTES
            cand = _refine_for_overlap(mine, plane, proj_bytes, dev.budget)
            if proj_bytes + 2 * max(z1 - z0 for z0, z1 in cand) * plane * \
                    SCALAR_BYTES > dev.budget and len(cand) > 1:
                cand = _refine_for_overlap(
                    mine, plane, 2 * C0 * sheet * SCALAR_BYTES, dev.budget)
            mine = list(cand)
            longest = max(z1 - z0 for z0, z1 in mine)
            nbuf = 1 if len(mine) == 1 else 2
            slab_bytes = longest * plane * SCALAR_BYTES
            whole = local or (A * sheet * SCALAR_BYTES + nbuf * slab_bytes
                              <= dev.budget)
            if not whole and nbuf * slab_bytes + 2 * min(
                    plan.chunk_angles, A) * sheet * SCALAR_BYTES > dev.budget:
                nbuf = 1  # the reference's one slab + two chunks
            link = _HostLink() if (isinstance(src, np.ndarray)
                                   or not res_dev) else None
            proj = None
            if local:
                proj = src
                dev.compute.wait_stream(torch.cuda.current_stream(dev.cuda))
            elif whole:
                proj = dev.alloc(tuple(src.shape))
                ev = dev.begin(dev.h2d, "TransferIn", "chunk.all",
                               proj.numel() * SCALAR_BYTES)
                _upload(proj, src, dev.h2d, link)
                dev.end(ev, dev.h2d)
                dev.compute.wait_stream(dev.h2d)
            else:
                C = min(plan.chunk_angles, A)
                cbufs = [dev.alloc((C * sheet,)) for _ in range(2)]
                cdone = [None, None]
            bufs = [dev.alloc((longest, grid.n_y, grid.n_x))
                    for _ in range(nbuf)]
            drained = [None] * nbuf
            k = 0
            waiting = None   # (buffer, z0, z1, event) not yet on the host

            def drain(item):
                b_, z0_, z1_, ev_, si_ = item
                dev.d2h.wait_event(ev_)
                tev = dev.begin(dev.d2h, "TransferOut", f"slab{si_}",
                                (z1_ - z0_) * plane * SCALAR_BYTES)
                if res_dev:
                    with torch.cuda.stream(dev.d2h):
                        res[z0_:z1_].copy_(bufs[b_][:z1_ - z0_],
                                           non_blocking=True)
                else:
                    link.d2h(res[z0_:z1_], bufs[b_][:z1_ - z0_], dev.d2h)
                dev.end(tev, dev.d2h)
                de = torch.cuda.Event()
                de.record(dev.d2h)
                drained[b_] = de

            for qi, (z0, z1) in enumerate(mine):
                si = qi
                b = qi % nbuf
                if waiting is not None and waiting[0] == b:
                    drain(waiting)   # single buffer: drain before reuse
                    waiting = None
                if drained[b] is not None:
                    dev.compute.wait_event(drained[b])
                buf = bufs[b][:z1 - z0]
                with torch.cuda.stream(dev.compute):
                    buf.zero_()
                if proj is not None:
                    ev = dev.begin(dev.compute, "Kernel", f"s{si}.c0")
                    bwd(proj, geometry, (0, A), (z0, z1), buf, dev.compute)
                    dev.end(ev, dev.compute)
                else:
                    for ci, c0 in enumerate(range(0, A, C)):
                        c1 = min(c0 + C, A)
                        cb = k % 2
                        k += 1
                        cbuf = cbufs[cb][:(c1 - c0) * sheet].view(
                            c1 - c0, det.n_v, det.n_u)
                        if cdone[cb] is not None:
                            dev.h2d.wait_event(cdone[cb])
                        ev = dev.begin(dev.h2d, "TransferIn", f"chunk{ci}",
                                       (c1 - c0) * sheet * SCALAR_BYTES)
                        _upload(cbuf, src[c0:c1], dev.h2d, link)
                        dev.end(ev, dev.h2d)
                        dev.compute.wait_stream(dev.h2d)
                        ev = dev.begin(dev.compute, "Kernel", f"s{si}.c{ci}")
                        bwd(cbuf, geometry, (c0, c1), (z0, z1), buf,
                            dev.compute)
                        dev.end(ev, dev.compute)
                        ce = torch.cuda.Event()
                        ce.record(dev.compute)
                        cdone[cb] = ce
                done = torch.cuda.Event()
                done.record(dev.compute)
                # the previous slab drains on the host while this one computes
                if waiting is not None:
                    drain(waiting)
                waiting = (b, z0, z1, done, si)
            if waiting is not None:
                drain(waiting)
            dev.d2h.synchronize()
            _join_streams(dev)

    _run_devices(work, D)
    rank, world = dist_info()
    if world > 1 and world == D:
        _gather_slabs(res, slabs, queues, rank, res_dev)
    _finish(devs, host_events, trace_sink)
    if out is not None:
        if isinstance(out.data, np.memmap):
            out.data.flush()
        return out
    return Volume(grid, res, (0, grid.n_z))


def _gather_slabs(out, slabs, queues, rank, on_dev, device=None):
    """Every rank ends with the full volume: each slab is broadcast from
    its owner in bounded pieces straight into ``out`` (host or device), so
    no rank stages more than one piece beyond its output."""
    for owner, q in enumerate(queues):
        for si in q:
            z0, z1 = slabs[si]
            _bcast_range(out, out[z0:z1] if owner == rank else None,
                         (z0, z1), owner, rank, device)
    return out


PIECE_BYTES = 256 << 20


def _bcast_range(out, mine, rng, owner, rank, device=None):
    """out[r0:r1] = the owner's ``mine`` (rows r0..r1) on every rank, in
    pieces of <= PIECE_BYTES.  NCCL broadcasts device buffers (NVLink);
    gloo (tests) broadcasts host tensors."""
    import torch.distributed as dist
    r0, r1 = rng
    if r1 <= r0:
        return
    row = int(np.prod(out.shape[1:])) * 4
    step = max(1, PIECE_BYTES // max(1, row))
    nccl = dist.get_backend() == "nccl"
    if device is None and nccl:
        device = torch.device("cuda", torch.cuda.current_device())
    for p0 in range(r0, r1, step):
        p1 = min(r1, p0 + step)
        if owner == rank:
            src = mine[p0 - r0:p1 - r0]
            piece = (torch.as_tensor(src) if not isinstance(src, torch.Tensor)
                     else src)
            piece = piece.to(device if nccl else "cpu").contiguous()
        else:
            piece = torch.empty((p1 - p0,) + tuple(out.shape[1:]),
                                dtype=torch.float32,
                                device=device if nccl else "cpu")
        dist.broadcast(piece, src=owner)
        if isinstance(out, torch.Tensor):
            out[p0:p1].copy_(piece)
        else:
            out[p0:p1] = piece.cpu().numpy()


def _bcast_rows(out, mine, ranges, rank):
    """Row-partitioned gather (ranges[r] owned by rank r; empty ranges and
    missing parts allowed)."""
    for owner, rng in enumerate(ranges):
        _bcast_range(out, mine if owner == rank else None, rng, owner, rank)
