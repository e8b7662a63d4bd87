"""The CPU oracle (oracle/) is pinned against goldens produced by the
reference implementation itself (tests/golden/make_golden.py): every
operator, TV routine, loop and plan must reproduce the reference's bits."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import oracle_geometry
from oracle import oracle as O

GEOS = ["g16", "ganiso", "g32"]


@pytest.mark.parametrize("name", GEOS)
def test_projectors_bit_exact(golden, golden_meta, name):
    d = golden_meta["geometries"][name]
    g = oracle_geometry(d)
    x, y = golden[f"{name}/x"], golden[f"{name}/y"]
    z0, z1 = d["slab"]
    a0, a1 = d["window"]
    eq = np.testing.assert_array_equal
    eq(O.fwd_interp(x, g), golden[f"{name}/fwd_interp"])
    eq(O.fwd_siddon(x, g), golden[f"{name}/fwd_siddon"])
    eq(O.fwd_interp(x[z0:z1], g, (a0, a1), (z0, z1)),
       golden[f"{name}/fwd_interp_slab"])
    eq(O.fwd_siddon(x[z0:z1], g, (a0, a1), (z0, z1)),
       golden[f"{name}/fwd_siddon_slab"])
    eq(O.bwd_matched(y, g), golden[f"{name}/bwd_matched"])
    eq(O.bwd_fdk(y, g), golden[f"{name}/bwd_fdk"])
    acc = x[z0:z1] * 0.5
    eq(O.bwd_matched(y[a0:a1], g, (a0, a1), (z0, z1), acc=acc),
       golden[f"{name}/bwd_matched_slab"])
    eq(O.bwd_fdk(y[a0:a1], g, (a0, a1), (z0, z1), acc=acc),
       golden[f"{name}/bwd_fdk_slab"])


@pytest.mark.parametrize("name", GEOS)
def test_ray_setup_bit_exact(golden, golden_meta, name):
    g = oracle_geometry(golden_meta["geometries"][name])
    t0, st, n = O.ray_table(g)
    np.testing.assert_array_equal(t0, golden[f"{name}/ray_t0"])
    np.testing.assert_array_equal(st, golden[f"{name}/ray_step"])
    np.testing.assert_array_equal(n, golden[f"{name}/ray_n"])


def test_matched_thread_count_invariant(golden, golden_meta):
    """z-band threading replays the reference's single-thread order."""
    g = oracle_geometry(golden_meta["geometries"]["g32"])
    y = golden["g32/y"]
    ref = O.bwd_matched(y, g, threads=1)
    for t in (2, 3, 7):
        np.testing.assert_array_equal(O.bwd_matched(y, g, threads=t), ref)


def test_kat_cube(golden, golden_meta):
    """10 mm cube of 0.02/mm, central ray -> 0.2 (Siddon);
    the interpolated projector gives 0.195 (zero-padded faces)."""
    g = oracle_geometry(golden_meta["kat_cube"])
    x = np.full((10, 10, 10), 0.02, np.float32)
    s = O.fwd_siddon(x, g)
    np.testing.assert_array_equal(s, golden["kat/cube_siddon"])
    assert abs(s[0, 1, 1] - 0.2) < 1e-4
    np.testing.assert_array_equal(O.fwd_interp(x, g), golden["kat/cube_interp"])


def test_tv(golden):
    f = golden["tv/f"]
    assert float(golden["tv/norm"]) == O.tv_norm(f)
    single = np.zeros((3, 3, 3), np.float32)
    single[1, 1, 1] = 1.0
    assert abs(O.tv_norm(single) - (np.sqrt(3) + 3)) < 1e-12
    np.testing.assert_array_equal(O.minimize_tv_gradient(f, 12, 0.05),
                                  golden["tv/gd"])
    np.testing.assert_array_equal(O.minimize_rof(f, 12, 0.1), golden["tv/rof"])
    for dev in (1, 2, 3):
        for tag in ("gd", "rof"):
            for nt in ("exact", "local"):
                if tag == "rof" and nt == "local":
                    continue
                got = O.split_minimize(f, dev, tag, 2, 4, 0.05, 0.1,
                                       nt == "exact", 5)
                np.testing.assert_array_equal(
                    got, golden[f"tv/split_{tag}_{nt}_d{dev}"])


def test_loops(golden, golden_meta):
    g = oracle_geometry(golden_meta["geometries"]["g16"])
    b = golden["loops/b16"]
    x, res, bd = O.cgls(b, g, 4)
    np.testing.assert_array_equal(x, golden["loops/cgls_x"])
    np.testing.assert_array_equal(np.array(res), golden["loops/cgls_res"])
    assert not bd
    np.testing.assert_array_equal(O.os_sart(b, g, 3, g.n_angles),
                                  golden["loops/sirt_x"])
    np.testing.assert_array_equal(O.os_sart(b, g, 2, 3, 0.8),
                                  golden["loops/ossart_x"])
    tv = dict(n_slabs=1, minimizer="gd", outer_syncs=1, inner_iters=5,
              step=0.01)
    np.testing.assert_array_equal(O.os_sart(b, g, 2, 4, tv=tv),
                                  golden["loops/sarttv_x"])
    np.testing.assert_array_equal(O.fdk(b, g), golden["loops/fdk_x"])


def test_plans(golden_meta):
    for c in golden_meta["plans"]:
        g = O.OGeom(1.0, 2.0, tuple(range(c["A"])), c["n"], c["n"], c["nz"],
                    nu=c["nu"], nv=c["nv"])
        chunk = 9 if c["op"] == "forward" else 32
        try:
            p = O.plan(c["op"], g, [c["budget"]] * c["dev"], chunk, c["uf"])
        except ValueError:
            p = None
        ref = c["plan"]
        if ref is None:
            assert p is None
            continue
        for k, v in ref.items():
            got = p[k]
            if isinstance(v, list):
                got = [list(t) for t in got]
            assert got == v, (c, k)
