"""Peer-memory exchange for the slab-sharded operators (one process per GPU).

The sharded forward (sharded.py) sums every rank's slab-partial projections
of a round of views onto the rank that owns those views, and the sharded
backward needs every rank's shard of the round on every rank: with NCCL a
reduce-scatter and an all-gather per round, issued after the kernels that
produce / consume them.  Here the transfers are folded into the kernels:

* forward: each rank's Ax kernels store their partial projections straight
  into the OWNER's inbox -- device memory of the peer GPU mapped into this
  process with CUDA IPC, reached over NVLink / NVSwitch by the kernel's own
  coalesced stores, tile by tile as the rays finish -- at the writing
  rank's slot.  The owner sums its slots in rank order (cs_sum_slices,
  fused with OS-SART's residual w o (b - sum) when asked) on a side stream
  while its compute stream starts the next round;
* backward: each rank stages its shard of the round in its outbox (a local
  copy) and every rank's matched Atb kernels read the owners' outboxes
  directly (peer loads, once per ray), so no gathered copy exists.

This replaces the reference's host-side sum of slab partials
(execution.py:224-235) and the per-device full upload of the projections
(execution.py:249-317).

Ordering uses inter-process CUDA events, one per slot and direction: a
writer's stream waits on the owner's "consumed" event before storing into
that slot, the owner's side stream waits on every writer's "written" event
before summing (and the same for "staged" / "read" in the backward).  One
host-only barrier per round (a gloo group: no device synchronisation, the
GPUs keep running) orders every rank's event records before any rank's
waits.  Slots alternate over every round of a direction, across calls as
well, so a slot's "consumed" / "read" event -- recorded after its round's
barrier -- is waited on by the slot's next user only after the barrier of
the round in between, which no rank passes before recording it: every wait
resolves to the record of the intended round.

The mapping is validated at set-up through the launch paths the operators
use: each rank's fill kernel stores a marker row and its Ax kernel (the
v-band memset included) a probe view of a small volume into every peer's
inbox, and its matched kernel backprojects every peer's outbox pattern; the
owners / readers compare with the same launches on local memory.
``PeerExchange.create`` returns None on every rank when CUDA IPC or P2P is
unavailable or a probe disagrees anywhere, and the operators keep NCCL's
collectives.
"""

from __future__ import annotations

import os
import warnings

import torch
import torch.distributed as dist

from . import kernels as K

__all__ = ["PeerExchange", "peer_mode_requested"]


def peer_mode_requested() -> bool:
    """CS_EXCHANGE=nccl selects the collectives (A/B); default peer."""
    return os.environ.get("CS_EXCHANGE", "peer").lower() != "nccl"


class PeerExchange:
    """Double-buffered inbox / outbox with peer mappings and IPC events."""

    KINDS = ("written", "consumed", "staged", "read")

    def __init__(self, rank: int, world: int, device: torch.device,
                 round_views: int, sheet: tuple[int, int], group=None,
                 geometry=None):
        self.rank, self.world, self.c = rank, world, round_views
        self.probe = None if geometry is None else _probe_geometry(geometry)
        self.device = device
        self.group = group
        n_v, n_u = sheet
        f32 = dict(dtype=torch.float32, device=device)
        self.inbox = torch.empty((2, world, round_views, n_v, n_u), **f32)
        self.outbox = torch.empty((2, round_views, n_v, n_u), **f32)
        self.side = torch.cuda.Stream(device)
        self.ev = {k: [torch.cuda.Event(interprocess=True) for _ in range(2)]
                   for k in self.KINDS}
        # rounds of each direction since set-up: slots alternate across
        # calls too, so between a slot's "consumed" / "read" record (after
        # its round's barrier) and the next wait on it there is always
        # another round's barrier
        self._seq = {"fwd": 1, "bwd": 0}
        self.inboxes: list[torch.Tensor] = []
        self.outboxes: list[torch.Tensor] = []
        self.peer_ev: list[dict] = []

    # ---------------------------------------------------------- set-up
    @classmethod
    def create(cls, rank, world, device, round_views, sheet, group=None,
               geometry=None):
        """Collective over the ranks; None (on every rank) when the peer
        path is unavailable on any of them.  Each stage ends in an
        all-gather, so a rank that fails still takes part in every
        collective the others enter."""
        def agree(ok):
            flags = [None] * world
            dist.all_gather_object(flags, bool(ok), group=group)
            return all(flags)

        ex, mine = None, None
        try:
            ex = cls(rank, world, device, round_views, sheet, group,
                     geometry)
            mine = ex._handles()
        except Exception as e:  # noqa: BLE001 - reported, then agreed on
            warnings.warn(f"peer exchange unavailable on rank {rank}: {e!r}")
        every = [None] * world
        dist.all_gather_object(every, mine, group=group)
        if any(m is None for m in every):
            return None
        ok = True
        try:
            ex._open(every)
        except Exception as e:  # noqa: BLE001
            warnings.warn(f"peer mapping failed on rank {rank}: {e!r}")
            ok = False
        if not agree(ok):
            ex.close()
            return None
        ok = True
        try:
            ex._mark_peers()
        except Exception as e:  # noqa: BLE001
            warnings.warn(f"peer stores failed on rank {rank}: {e!r}")
            ok = False
        ex.barrier()
        try:
            ok = ex._check_marks() and ok
        except Exception as e:  # noqa: BLE001
            warnings.warn(f"peer self-check failed on rank {rank}: {e!r}")
            ok = False
        if not agree(ok):
            ex.close()
            return None
        return ex

    def _handles(self):
        from torch.multiprocessing.reductions import reduce_tensor
        with torch.cuda.device(self.device):
            for evs in self.ev.values():   # create the events on this device
                for e in evs:
                    e.record()
            torch.cuda.synchronize(self.device)
            return (self.device.index, reduce_tensor(self.inbox),
                    reduce_tensor(self.outbox),
                    {k: [e.ipc_handle() for e in v]
                     for k, v in self.ev.items()})

    def _open(self, every):
        for s, (dev_s, rin, rout, handles) in enumerate(every):
            if s == self.rank:
                self.inboxes.append(self.inbox)
                self.outboxes.append(self.outbox)
                self.peer_ev.append(self.ev)
                continue
            with torch.cuda.device(self.device):
                K.peer_enable(dev_s)
            self.inboxes.append(rin[0](*rin[1]))
            self.outboxes.append(rout[0](*rout[1]))
            self.peer_ev.append({
                k: [torch.cuda.Event.from_ipc_handle(
                    torch.device("cuda", dev_s), h) for h in hs]
                for k, hs in handles.items()})

    def _marker(self, writer: int, owner: int) -> float:
        return float(1 + writer * self.world + owner)

    def _pattern(self, rank: int) -> float:
        return 0.25 * (rank + 1)

    def _mark_peers(self):
        """Set-up check, part 1 (peer stores): the fill kernel writes a
        marker row into this rank's slot of every owner's inbox (slot 0),
        the Ax kernel a probe view (slot 1); the outbox gets this rank's
        pattern for the readers."""
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream()
            for s in range(self.world):
                K.fill(self.inboxes[s][0, self.rank, 0, 0],
                       self._marker(self.rank, s))
            if self.probe is not None:
                g, vol = self.probe, self._probe_volume()
                for s in range(self.world):
                    K.fwd_interp(vol, g, (0, 1), (0, vol.shape[0]),
                                 self.inboxes[s][1, self.rank, :1])
            K.fill(self.outbox[0, :1], self._pattern(self.rank))
            self.ev["written"][0].record(cur)
            self.ev["staged"][0].record(cur)

    def _probe_volume(self):
        n = self.probe.voxel_grid.n_x
        i = torch.arange(n ** 3, dtype=torch.float32, device=self.device)
        return (1.0 + (i % 7) / 7.0).reshape(n, n, n)

    def _check_marks(self) -> bool:
        """Part 2 (after a barrier): the owner reads every writer's marker
        and probe view (bit-identical to its own launch of the same Ax),
        and backprojects every peer's outbox with the matched kernel
        (against the same launch on a local copy of the pattern)."""
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream()
            self.wait_all(cur, "written", 0)
            self.wait_all(cur, "staged", 0)
            got = self.inbox[0, :, 0, 0].cpu()
            ok = True
            if self.probe is not None:
                g, vol = self.probe, self._probe_volume()
                nz = vol.shape[0]
                mine = torch.empty_like(self.inbox[1, 0, :1])
                K.fwd_interp(vol, g, (0, 1), (0, nz), mine)
                ok = bool((self.inbox[1, :, :1] == mine).all().item())
                for s in range(self.world):
                    far = torch.zeros_like(vol)
                    K.bwd_matched(self.outboxes[s][0, :1], g, (0, 1),
                                  (0, nz), far)
                    near = torch.zeros_like(vol)
                    K.bwd_matched(K.fill(torch.empty_like(mine),
                                         self._pattern(s)),
                                  g, (0, 1), (0, nz), near)
                    err = (far - near).norm() / near.norm().clamp_min(1e-30)
                    ok = ok and float(err.item()) <= 1e-6
            self.ev["consumed"][0].record(cur)
            self.ev["consumed"][1].record(cur)
            self.ev["read"][0].record(cur)
        want = torch.tensor([self._marker(s, self.rank)
                             for s in range(self.world)])
        return ok and bool((got == want[:, None]).all())

    def barrier(self):
        """Host-only rendezvous (no device synchronisation)."""
        dist.barrier(group=self.group)

    def close(self):
        self.inboxes.clear()
        self.outboxes.clear()
        self.peer_ev.clear()

    # ------------------------------------------------------- protocol
    def next_slot(self, direction: str) -> int:
        n = self._seq[direction]
        self._seq[direction] = n + 1
        return n % 2

    def wait_all(self, stream, kind: str, slot: int, ranks=None):
        for s in (range(self.world) if ranks is None else ranks):
            stream.wait_event(self.peer_ev[s][kind][slot])

    def record(self, stream, kind: str, slot: int):
        self.ev[kind][slot].record(stream)


def _probe_geometry(geometry):
    """One view of the operators' geometry on an 8^3 grid spanning the
    same field of view (every detector row of the probe sees the cone)."""
    from .geometry import ScanGeometry, VoxelGrid
    g = geometry.voxel_grid
    n = 8
    vs = tuple(float(v) * c / n for v, c in zip(g.voxel_size, g.counts))
    return ScanGeometry(geometry.dso, geometry.dsd, (float(geometry.angles[0]),),
                        VoxelGrid(n, n, n, vs, tuple(g.origin_offset)),
                        geometry.detector)
