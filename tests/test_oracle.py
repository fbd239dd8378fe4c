"""Pin the oracle (oracle/eik_oracle.c) against the reference's own
known-answer values and golden fields (tests/golden/, generated from the
unmodified reference by tests/golden/make_golden.py), and -- where
oracle/_ref is built -- against the reference run live.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from oracle import oracle as O
from tests.golden.make_golden import SMALL_CASES, sha

GOLD = os.path.join(os.path.dirname(__file__), "golden")
INF = math.inf


def _kat():
    with open(os.path.join(GOLD, "kat.json")) as f:
        return json.load(f)


def _nb(v):
    return np.array(v, dtype=np.float64).ctypes.data_as(O._dp)


def test_local_update_kats():
    k = _kat()
    for a, b, f, h, want in k["quadrant"]:
        assert O.olib.orc_quadrant_update(a, b, f, h) == float.fromhex(want)
    for nb, f, h, want in k["node"]:
        assert O.olib.orc_node_update(_nb(nb), f, h) == float.fromhex(want)
    for nb, d, f, h, want in k["directional"]:
        assert O.olib.orc_directional_update(_nb(nb), d, f, h) == float.fromhex(want)


def test_local_update_pinned_values():
    # test_local_update.cpp:31-46 (values restated; tolerance as there)
    q = O.olib.orc_quadrant_update
    assert q(0.0, 0.0, 1.0, 1.0) == pytest.approx(math.sqrt(2.0) / 2.0, rel=1e-14)
    assert q(0.0, INF, 2.0, 0.1) == pytest.approx(0.05)
    assert q(0.0, 10.0, 1.0, 1.0) == pytest.approx(1.0)
    assert q(INF, INF, 1.0, 1.0) == INF
    assert q(1.0, 2.0, 1.0, 2.0) == pytest.approx(1.5 + math.sqrt(7.0) / 2.0, rel=1e-12)


def test_random_node_update_hash():
    k = _kat()["random_node_update"]
    rng = np.random.default_rng(k["seed"])
    n = k["n"]
    vals = np.where(rng.random((n, 4)) < 0.15, INF, 10.0 * rng.random((n, 4)) - 2.0)
    fs = 0.05 + 3.0 * rng.random(n)
    hs = 0.01 + rng.random(n)
    res = np.array([O.olib.orc_node_update(_nb(vals[i]), fs[i], hs[i]) for i in range(n)])
    assert sha(res) == k["sha256"]


def _small():
    with open(os.path.join(GOLD, "small.json")) as f:
        meta = json.load(f)
    return np.load(os.path.join(GOLD, "small.npz")), meta


@pytest.mark.parametrize("cid,make,cells", SMALL_CASES, ids=[c[0] for c in SMALL_CASES])
def test_oracle_matches_reference_golden_fields(cid, make, cells):
    arrays, meta = _small()
    p = make()
    runs = [(m, None) for m in ("fmm", "fsm", "lsm")]
    runs += [(m, c) for c in cells for m in ("hcm", "fhcm", "fmsm")]
    for method, c in runs:
        key = f"{cid}/{method}" + (f"/{c}" if c else "")
        got = O.oracle_solve(p, method, E.build_cells(p.grid, c, c) if c else None)
        want = arrays[key]
        assert np.array_equal(got.u.view(np.int64), want.view(np.int64)), key
        m = meta[key]
        assert (got.sweeps, got.node_updates, got.heap_removals, got.mon_checks,
                got.mon_single) == (m["sweeps"], m["node_updates"], m["heap_removals"],
                                    m["mon_checks"], m["mon_single"]), key


def test_oracle_acceptance_sweep_counts():
    # acceptance.cpp:133-146: constant 176 -> 5, checker11 176 -> 16, checker41 164 -> 44
    with open(os.path.join(GOLD, "big.json")) as f:
        acc = json.load(f)["acceptance_fsm_sweeps"]
    for name, m, sp in [("constant", 176, E.speed_constant()),
                        ("checker11", 176, E.speed_checkerboard(11)),
                        ("checker41", 164, E.speed_checkerboard(41))]:
        p = E.build_problem(E.Grid.unit_square(m), sp, E.ExitSpec.point_source((0.5, 0.5)))
        r = O.oracle_solve(p, "fsm")
        want = acc[f"{name}/{m}"]
        assert r.sweeps == want["published"] == want["sweeps"]
        assert sha(r.u) == want["sha256"]


def test_oracle_c1_matches_reference_hash_and_error():
    from paper_1110_6220_b200 import configs
    with open(os.path.join(GOLD, "big.json")) as f:
        big = json.load(f)
    p = configs.config1().problem
    g = p.grid
    xs = g.x0 + np.arange(g.m) * g.h
    X, Y = np.meshgrid(xs, xs)
    exact = np.hypot(X, Y).reshape(-1)
    for key, method, cs in [("c1/fsm", "fsm", 0), ("c1/fmm", "fmm", 0), ("c1/fmsm/16", "fmsm", 16)]:
        r = O.oracle_solve(p, method, E.build_cells(g, g.m // cs, g.m // cs) if cs else None)
        assert sha(r.u) == big[key]["sha256"], key
        assert r.sweeps == big[key]["sweeps"]
        assert float(np.abs(r.u - exact).max()) == pytest.approx(1.272e-2, abs=5e-6)


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_native_fields_match_reference_speed_fields():
    # our C restatement of speed_fields.cpp vs the reference's SpeedSpec
    named = {"constant": E.speed_constant(), "checker11": E.speed_checkerboard(11),
             "checker41": E.speed_checkerboard(41), "sinusoidA": E.speed_sinusoid(0.5, 20),
             "sinusoidB": E.speed_sinusoid(0.99, 2), "comb4": E.speed_comb_maze(4),
             "comb8": E.speed_comb_maze(8)}
    g = E.Grid.unit_square(97)
    rng = np.random.default_rng(0)
    extra = rng.random((500, 2))
    for name, sp in named.items():
        F = sp.sample(g)
        ref = np.array([O.rlib.ref_named_speed(name.encode(), g.x(i), g.y(j))
                        for j in range(g.n) for i in range(g.m)])
        assert np.array_equal(F, ref), name
        ref2 = np.array([O.rlib.ref_named_speed(name.encode(), x, y) for x, y in extra])
        assert np.array_equal(sp(extra[:, 0], extra[:, 1]), ref2), name


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_oracle_vs_live_reference_remainder_and_exits():
    # remainder decompositions (cells.cpp:7-19) and multi-node exit sets
    g = E.Grid.unit_square(45)
    p = E.build_problem(g, E.speed_sinusoid(0.5, 20),
                        E.ExitSpec.node_set([(3, 4), (40, 2), (20, 30), (3, 4)], [0.1, 0.0, 0.2, 0.05]))
    for method in ("fmm", "fsm", "lsm"):
        a, b = O.oracle_solve(p, method), O.ref_solve(p, method)
        assert np.array_equal(a.u, b.u) and a.sweeps == b.sweeps
    for c in (7, 6, 2):
        for method in ("hcm", "fhcm", "fmsm"):
            a = O.oracle_solve(p, method, E.build_cells(g, c, c))
            b = O.ref_solve(p, method, c, c)
            assert np.array_equal(a.u.view(np.int64), b.u.view(np.int64)), (method, c)
            assert (a.sweeps, a.node_updates, a.heap_removals, a.mon_checks) == \
                (b.sweeps, b.node_updates, b.heap_removals, b.mon_checks), (method, c)
