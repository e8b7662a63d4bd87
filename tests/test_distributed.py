"""Multi-process (world_size 2-3, gloo on CPU) tests of the N>1 host logic:
halo exchange + scalar all-reduce of the distributed TV split, the
row/slab gathers behind the angle-split Ax and slab-split Atb, and the
distributed ScheduledOperators partition.  Stencil / projector math is
injected as CPU stand-ins (the CUDA kernels are covered by -m gpu tests);
what is tested here is who computes what and how the pieces are
exchanged -- checked against the oracle."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys
    for p in (ROOT, os.path.join(ROOT, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ------------------------------------------------------------ TV ops (CPU)

def _grad(u):
    gz = torch.zeros_like(u)
    gy = torch.zeros_like(u)
    gx = torch.zeros_like(u)
    gz[:-1] = u[1:] - u[:-1]
    gy[:, :-1] = u[:, 1:] - u[:, :-1]
    gx[:, :, :-1] = u[:, :, 1:] - u[:, :, :-1]
    return gz, gy, gx


def _div(pz, py, px):
    out = torch.zeros_like(pz)
    out[0] = pz[0]
    out[1:-1] = pz[1:-1] - pz[:-2]
    out[-1] = -pz[-2]
    out[:, 0] += py[:, 0]
    out[:, 1:-1] += py[:, 1:-1] - py[:, :-2]
    out[:, -1] += -py[:, -2]
    out[:, :, 0] += px[:, :, 0]
    out[:, :, 1:-1] += px[:, :, 1:-1] - px[:, :, :-2]
    out[:, :, -1] += -px[:, :, -2]
    return out


def _subgrad(u):
    gz, gy, gx = _grad(u)
    mag = torch.sqrt(gz * gz + gy * gy + gx * gx + 1e-8)
    return -_div(gz / mag, gy / mag, gx / mag)


class CpuTvOps:
    @staticmethod
    def grad_sumsq(w, core, out):
        g = _subgrad(w.double())[core[0]:core[1]]
        out[0] = (g * g).sum()

    @staticmethod
    def step(w, out, step, ss, scale):
        norm = float(np.sqrt(float(ss[0]))) * scale
        if norm < 1e-30:
            out.copy_(w)
        else:
            out.copy_(w.double() - step * _subgrad(w.double()) / norm)

    @staticmethod
    def rof_iter(f, p, q, lam):
        p64 = p.double()
        u = f.double() + lam * _div(p64[0], p64[1], p64[2])
        g = torch.stack(_grad(u))
        pn = p64 + (1.0 / 12.0 / lam) * g
        mag = torch.clamp(torch.sqrt((pn * pn).sum(0)), min=1.0)
        q.copy_(pn / mag)

    @staticmethod
    def rof_finish(f, p, u, lam):
        p64 = p.double()
        u.copy_(f.double() + lam * _div(p64[0], p64[1], p64[2]))


class CpuTvOpsStored(CpuTvOps):
    """Adds the stored-g GD pair (CudaTvOps.grad_store / step_g)."""

    @staticmethod
    def grad_store(w, g, core, out):
        g.copy_(_subgrad(w.double()))
        gc = g.double()[core[0]:core[1]]
        out[0] = (gc * gc).sum()

    @staticmethod
    def step_g(w, g, out, step, ss, scale):
        norm = float(np.sqrt(float(ss[0]))) * scale
        if norm < 1e-30:
            out.copy_(w)
        else:
            out.copy_(w.double() - step * g.double() / norm)


def _tv_worker(rank, world, port, f, params_kw, q, stored=False):
    _init(rank, world, port)
    from paper_1905_03748_b200 import halo
    from paper_1905_03748_b200.regularization import (TvParams,
                                                      make_halo_slabs)
    params = TvParams(**params_kw)
    slabs = make_halo_slabs(f.shape[0], world, params.effective_halo())
    out = halo.split_minimize_distributed(
        torch.from_numpy(f), slabs, params, rank,
        ops=CpuTvOpsStored if stored else CpuTvOps)
    if rank == 0:
        q.put(out.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _run(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["gd_exact", "gd_local", "rof",
                                  "gd_exact_stored", "gd_local_stored"])
def test_distributed_tv_split_matches_oracle(world, case):
    from paper_1905_03748_b200.regularization import NormMode, TvMinimizer
    from oracle import oracle as O
    rng = np.random.default_rng(7)
    f = (np.repeat(np.linspace(0, 1, 18)[:, None, None], 1, 0)
         * np.ones((18, 10, 12)) + 0.05 * rng.standard_normal((18, 10, 12))
         ).astype(np.float32)
    if case == "rof":
        kw = dict(minimizer=TvMinimizer.ROF, outer_syncs=3, inner_iters=3,
                  lam=0.1, halo_depth=4)
        ref = O.split_minimize(f, world, "rof", 3, 3, lam=0.1, halo=4)
    else:
        exact = case.startswith("gd_exact")
        kw = dict(minimizer=TvMinimizer.GRADIENT_DESCENT, outer_syncs=3,
                  inner_iters=3, step=0.05, halo_depth=4,
                  norm_mode=NormMode.EXACT_GLOBAL if exact
                  else NormMode.LOCAL_APPROX)
        ref = O.split_minimize(f, world, "gd", 3, 3, step=0.05,
                               exact_global=exact, halo=4)
    if case.endswith("_stored"):
        got = _run(_tv_worker_stored, world, f, kw)
    else:
        got = _run(_tv_worker, world, f, kw)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err < 1e-6, err


def _tv_worker_stored(rank, world, port, f, params_kw, q):
    _tv_worker(rank, world, port, f, params_kw, q, stored=True)


def _gather_worker(rank, world, port, q):
    _init(rank, world, port)
    from paper_1905_03748_b200.execution import _allgather_rows, _gather_slabs
    ranges = [(0, 5), (5, 7), (7, 13)][:world]
    if world == 2:
        ranges = [(0, 6), (6, 13)]
    full = torch.arange(13 * 4, dtype=torch.float32).reshape(13, 4)
    a, b = ranges[rank]
    part = full[a:b].clone()
    got = _allgather_rows(part, ranges, rank)
    ok1 = torch.equal(got, full)
    # slab gather: every rank owns round-robin slabs of a 10-plane volume
    slabs = [(0, 3), (3, 6), (6, 9), (9, 10)]
    queues = [list(range(d, len(slabs), world)) for d in range(world)]
    vol = torch.zeros(10, 2, 2)
    ref = torch.arange(40, dtype=torch.float32).reshape(10, 2, 2)
    for si in queues[rank]:
        z0, z1 = slabs[si]
        vol[z0:z1] = ref[z0:z1]
    got2 = _gather_slabs(vol.numpy(), slabs, queues, rank, on_dev=False,
                         device=torch.device("cpu"))
    ok2 = np.array_equal(got2, ref.numpy())
    flag = torch.tensor([int(ok1 and ok2)])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        q.put(int(flag.item()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_gathers(world):
    assert _run(_gather_worker, world) == 1


def _ops_worker(rank, world, port, q):
    """Distributed ScheduledOperators: rank r projects its angle range and
    backprojects its slab; the gathered results must equal the monolithic
    oracle operators."""
    _init(rank, world, port)
    import paper_1905_03748_b200 as cs
    from paper_1905_03748_b200 import algorithms as AL
    from paper_1905_03748_b200 import kernels as K
    from oracle import oracle as O
    from conftest import synth_geometry, to_oracle
    g = synth_geometry(12, 7)
    og = to_oracle(g)

    def fake_fwd(x, geometry, ar, sr, out, accumulate=False, stream=None):
        assert sr == (0, 12)
        out.copy_(torch.from_numpy(O.fwd_interp(x.numpy(), og, ar)))
        return out

    def fake_bwd(y, geometry, ar, sr, out, stream=None):
        out += torch.from_numpy(O.bwd_matched(y.numpy(), og, ar, sr))
        return out

    K.fwd_interp = fake_fwd
    K.bwd_matched = fake_bwd
    AL.K.fwd_interp = fake_fwd
    AL.K.bwd_matched = fake_bwd
    pool = cs.DevicePool(tuple(cs.DeviceSpec(memory_budget=2 ** 30)
                               for _ in range(world)))
    ops = AL.ScheduledOperators(g, pool, cs.ProjectionMethod.INTERPOLATED,
                                cs.WeightMode.MATCHED)
    assert ops.distributed
    x = np.random.default_rng(0).random((12, 12, 12), dtype=np.float32)
    y = np.random.default_rng(1).standard_normal((7, 12, 12)).astype(
        np.float32)
    fx = torch.empty((7, 12, 12))
    ops.fwd_dev(torch.from_numpy(x), fx)
    by = torch.zeros((12, 12, 12))
    ops.bwd_dev(torch.from_numpy(y), by)
    ok = (np.array_equal(fx.numpy(), O.fwd_interp(x, og))
          and np.allclose(by.numpy(), O.bwd_matched(y, og), rtol=1e-6,
                          atol=1e-7))
    flag = torch.tensor([int(ok)])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        q.put(int(flag.item()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_operator_partition(world):
    assert _run(_ops_worker, world) == 1
