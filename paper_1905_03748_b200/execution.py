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
* backward (Alg. 2, execution.py:249-317): projections are uploaded once,
  each owned slab is zeroed, backprojected over every angle and drained.
  Slabs are dealt round-robin over ``max(plan.n_splits, n_devices)`` equal
  slabs, so every GPU works even when one slab would fit (SURVEY 0.6 --
  legal because Atb is slab-partition invariant);
* host images are page-locked for the pass when ``plan.pin_host_image``
  (Pin/Unpin events), device-resident inputs skip the transfers;
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


class _Pinned:
    """Page-lock a host numpy image for the pass (execution.py:117-124)."""

    def __init__(self, arr: np.ndarray | None, enabled: bool, events: list):
        self.arr = arr if (enabled and isinstance(arr, np.ndarray)
                           and arr.nbytes > 0) else None
        self.events = events
        self.ok = False

    def __enter__(self):
        if self.arr is not None:
            import time
            t0 = time.perf_counter()
            rc = torch.cuda.cudart().cudaHostRegister(
                self.arr.ctypes.data, self.arr.nbytes, 0)
            self.ok = (int(rc) == 0) if not hasattr(rc, "value") else \
                (rc.value == 0)
            self.events.append(TraceEvent(HOST, "Pin", "image", 0.0,
                                          time.perf_counter() - t0,
                                          self.arr.nbytes))
        return self

    def __exit__(self, *exc):
        if self.arr is not None and self.ok:
            import time
            t0 = time.perf_counter()
            torch.cuda.cudart().cudaHostUnregister(self.arr.ctypes.data)
            self.events.append(TraceEvent(HOST, "Unpin", "image", 0.0,
                                          time.perf_counter() - t0,
                                          self.arr.nbytes))
        return False


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
    monolithic projection of the full volume."""
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
            acc = dev.alloc((a1 - a0, det.n_v, det.n_u))
            src = volume.data
            if on_dev and src.device == dev.cuda and plan.n_splits == 1:
                # device-resident input that fits: no staging
                ev = dev.begin(dev.compute, "Kernel", "s0.c0")
                with torch.cuda.stream(dev.compute):
                    dev.compute.wait_stream(torch.cuda.current_stream(
                        dev.cuda))
                    fwd(src, geometry, (a0, a1), (0, grid.n_z), acc,
                        False, dev.compute)
                dev.end(ev, dev.compute)
            else:
                slabs = plan.slab_ranges
                longest = max(z1 - z0 for z0, z1 in slabs)
                nbuf = 1 if len(slabs) == 1 else 2
                bufs = [dev.alloc((longest, grid.n_y, grid.n_x))
                        for _ in range(nbuf)]
                ready = [torch.cuda.Event() for _ in range(nbuf)]
                free = [None] * nbuf
                for si, (z0, z1) in enumerate(slabs):
                    b = si % nbuf
                    buf = bufs[b][:z1 - z0]
                    nbytes = (z1 - z0) * plane * SCALAR_BYTES
                    if free[b] is not None:
                        dev.h2d.wait_event(free[b])
                    ev = dev.begin(dev.h2d, "TransferIn", f"slab{si}", nbytes)
                    with torch.cuda.stream(dev.h2d):
                        chunk = src[z0:z1]
                        if isinstance(chunk, np.ndarray):
                            chunk = torch.from_numpy(chunk)
                        buf.copy_(chunk, non_blocking=True)
                    dev.end(ev, dev.h2d)
                    ready[b].record(dev.h2d)
                    dev.compute.wait_event(ready[b])
                    ev = dev.begin(dev.compute,
                                   "Kernel" if si == 0 else "Accumulate",
                                   f"s{si}.c0")
                    fwd(buf, geometry, (a0, a1), (z0, z1), acc, si > 0,
                        dev.compute)
                    dev.end(ev, dev.compute)
                    fe = torch.cuda.Event()
                    fe.record(dev.compute)
                    free[b] = fe
            if not on_dev:
                out = torch.empty(acc.shape, dtype=torch.float32,
                                  pin_memory=True)
                dev.d2h.wait_stream(dev.compute)
                ev = dev.begin(dev.d2h, "TransferOut", "out",
                               acc.numel() * SCALAR_BYTES)
                with torch.cuda.stream(dev.d2h):
                    out.copy_(acc, non_blocking=True)
                dev.end(ev, dev.d2h)
                dev.d2h.synchronize()
                parts[i] = out.numpy()
            else:
                parts[i] = acc
            _join_streams(dev)

    with _Pinned(volume.data if not on_dev else None, plan.pin_host_image,
                 host_events):
        _run_devices(work, len(pool))
    rank, world = dist_info()
    if world > 1 and world == len(pool):
        mine = parts[rank]
        t = mine if isinstance(mine, torch.Tensor) else torch.from_numpy(mine)
        dev = torch.device("cuda", torch.cuda.current_device())
        full = _allgather_rows(t.to(dev), plan.angle_assignment, rank)
        data = full if on_dev else full.cpu().numpy()
    elif on_dev:
        data = torch.cat([p.to(volume.data.device) for p in parts
                          if p is not None], 0)
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
                     trace_sink: list | None = None) -> Volume:
    """Run a planned backward pass (execution.py:249-317); equals the
    monolithic backprojection."""
    _validate(plan, OpKind.BACKWARD, geometry, pool)
    grid, det = geometry.voxel_grid, geometry.detector
    if projections.angle_range != (0, geometry.n_angles):
        raise ValueError("backward execution needs the full projection set")
    on_dev = projections.on_device
    D = len(pool)
    slabs = backward_slabs(plan, D)
    queues = [list(range(d, len(slabs), D)) for d in range(D)]
    plane = grid.n_x * grid.n_y
    if on_dev:
        out = torch.zeros((grid.n_z, grid.n_y, grid.n_x), dtype=torch.float32,
                          device=projections.data.device)
    else:
        out = np.zeros((grid.n_z, grid.n_y, grid.n_x), np.float32)
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
            if on_dev and src.device == dev.cuda:
                proj = src
                dev.compute.wait_stream(torch.cuda.current_stream(dev.cuda))
            else:
                proj = dev.alloc(tuple(src.shape))
                ev = dev.begin(dev.h2d, "TransferIn", "chunk.all",
                               proj.numel() * SCALAR_BYTES)
                with torch.cuda.stream(dev.h2d):
                    s = torch.from_numpy(src) if isinstance(src, np.ndarray) \
                        else src
                    proj.copy_(s, non_blocking=True)
                dev.end(ev, dev.h2d)
                dev.compute.wait_stream(dev.h2d)
            longest = max(slabs[s][1] - slabs[s][0] for s in queues[i])
            nbuf = 1 if len(queues[i]) == 1 else 2
            bufs = [dev.alloc((longest, grid.n_y, grid.n_x))
                    for _ in range(nbuf)]
            drained = [None] * nbuf
            pinned_out = None
            if not on_dev:
                pinned_out = [torch.empty((longest, grid.n_y, grid.n_x),
                                          dtype=torch.float32,
                                          pin_memory=True)
                              for _ in range(nbuf)]
            pending = []
            for qi, si in enumerate(queues[i]):
                z0, z1 = slabs[si]
                b = qi % nbuf
                if drained[b] is not None:
                    dev.compute.wait_event(drained[b])
                    # host copy of the previous user of this buffer
                    _flush(pending, out, b)
                buf = bufs[b][:z1 - z0]
                with torch.cuda.stream(dev.compute):
                    buf.zero_()
                ev = dev.begin(dev.compute, "Kernel", f"s{si}.c0")
                bwd(proj, geometry, (0, A), (z0, z1), buf, dev.compute)
                dev.end(ev, dev.compute)
                nbytes = (z1 - z0) * plane * SCALAR_BYTES
                dev.d2h.wait_stream(dev.compute)
                ev = dev.begin(dev.d2h, "TransferOut", f"slab{si}", nbytes)
                with torch.cuda.stream(dev.d2h):
                    if on_dev:
                        out[z0:z1].copy_(buf, non_blocking=True)
                    else:
                        pinned_out[b][:z1 - z0].copy_(buf, non_blocking=True)
                dev.end(ev, dev.d2h)
                de = torch.cuda.Event()
                de.record(dev.d2h)
                drained[b] = de
                if not on_dev:
                    pending.append((b, de, pinned_out[b], z0, z1))
            dev.d2h.synchronize()
            _flush(pending, out, None)
            _join_streams(dev)

    _run_devices(work, D)
    rank, world = dist_info()
    if world > 1 and world == D:
        out = _gather_slabs(out, slabs, queues, rank, on_dev)
    _finish(devs, host_events, trace_sink)
    return Volume(grid, out, (0, grid.n_z))


def _flush(pending, out, only_buf):
    """Copy drained pinned slabs into the host volume (after their event)."""
    keep = []
    for item in pending:
        b, ev, pin, z0, z1 = item
        if only_buf is None or b == only_buf:
            ev.synchronize()
            out[z0:z1] = pin[:z1 - z0].numpy()
        else:
            keep.append(item)
    pending[:] = keep


def _gather_slabs(out, slabs, queues, rank, on_dev, device=None):
    """Every rank ends with the full volume: broadcast each slab from its
    owner (NCCL over NVLink between ranks; ``device`` is where host volumes
    are staged for the collective, default the current GPU)."""
    import torch.distributed as dist
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    full = out if on_dev else torch.from_numpy(out).to(device)
    for owner, q in enumerate(queues):
        for si in q:
            z0, z1 = slabs[si]
            part = full[z0:z1].contiguous()
            dist.broadcast(part, src=owner)
            full[z0:z1].copy_(part)
    return full if on_dev else full.cpu().numpy()
