"""GPU parity for the two-scale methods (kernels 2 and 3).

FMSM must be bitwise-identical to the reference with identical counters
(SURVEY.md finding 4: the DAG-respecting schedule reproduces the one-pass
order exactly).  Golden values come from the unmodified reference
(tests/golden/make_golden.py); random cases use the oracle, which is pinned
to the reference by tests/test_oracle.py.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs
from oracle import oracle as O
from tests.golden.make_golden import SMALL_CASES

pytestmark = pytest.mark.gpu
# bit-exact parity with the reference's HCM needs the exact replay of its heap
# order ("hcm_exact"); "hcm" itself runs the band scheduler (test_gpu_hcm_band.py)
EXACT = {"hcm": "hcm_exact"}
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(u):
    return hashlib.sha256(np.ascontiguousarray(u, dtype=np.float64).tobytes()).hexdigest()


def bitwise(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def _big():
    with open(os.path.join(GOLD, "big.json")) as f:
        return json.load(f)


def _small():
    with open(os.path.join(GOLD, "small.json")) as f:
        return np.load(os.path.join(GOLD, "small.npz")), json.load(f)


@pytest.mark.parametrize("cid,make,cells", SMALL_CASES, ids=[c[0] for c in SMALL_CASES])
def test_fmsm_small_golden_fields(cid, make, cells):
    arrays, meta = _small()
    p = make()
    for c in cells:
        key = f"{cid}/fmsm/{c}"
        out = E.fmsm_solve(p, E.build_cells(p.grid, c, c))
        assert bitwise(out.values, arrays[key]), key
        m = meta[key]
        assert (out.sweeps, out.node_updates, out.heap_removals) == \
            (m["sweeps"], m["node_updates"], m["heap_removals"]), key


def test_fmsm_c1_bitwise():
    big = _big()["c1/fmsm/16"]
    p = configs.config1().problem
    out = E.fmsm_solve(p, E.build_cells(p.grid, 16, 16))
    assert sha(out.values) == big["sha256"]
    assert (out.sweeps, out.node_updates, out.heap_removals) == \
        (big["sweeps"], big["node_updates"], big["heap_removals"])


@pytest.mark.parametrize("cs", [8, 16, 32, 64])
def test_fmsm_c2_bitwise_full_size(cs):
    big = _big()[f"c2/fmsm/{cs}"]
    p = configs.config2().problem
    out = E.fmsm_solve(p, E.build_cells(p.grid, big["cells"], big["cells"]))
    assert sha(out.values) == big["sha256"]
    assert (out.sweeps, out.node_updates, out.heap_removals) == \
        (big["sweeps"], big["node_updates"], big["heap_removals"])


@pytest.mark.parametrize("seed", range(8))
def test_fmsm_random_against_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    m, n = int(rng.integers(12, 160)), int(rng.integers(12, 160))
    g = E.Grid(m, n, float(rng.uniform(0.002, 0.05)), -0.1, 0.3)
    F = rng.uniform(0.1, 3.0, size=(n, m))
    sp = lambda x, y, F=F, g=g: F[np.rint((y - g.y0) / g.h).astype(int),  # noqa: E731
                                  np.rint((x - g.x0) / g.h).astype(int)]
    if seed % 3 == 0:
        ex = E.ExitSpec.point_source((g.x(int(rng.integers(0, m))) + 0.3 * g.h,
                                      g.y(int(rng.integers(0, n))) - 0.2 * g.h))
    elif seed % 3 == 1:
        k = int(rng.integers(2, 9))
        ex = E.ExitSpec.node_set([(int(rng.integers(0, m)), int(rng.integers(0, n)))
                                  for _ in range(k)], list(rng.uniform(0, 0.2, size=k)))
    else:
        ex = E.ExitSpec.full_boundary()
    p = E.build_problem(g, sp, ex)
    for cx, cy in [(2, 2), (int(rng.integers(2, 9)), int(rng.integers(2, 9))),
                   (max(2, m // 8), max(2, n // 8))]:
        cells = E.build_cells(g, cx, cy)
        a = E.fmsm_solve(p, cells)
        b = O.oracle_solve(p, "fmsm", cells)
        assert bitwise(a.values, b.u), (cx, cy)
        assert (a.sweeps, a.node_updates, a.heap_removals) == \
            (b.sweeps, b.node_updates, b.heap_removals), (cx, cy)


def test_fmsm_rejects_degenerate_decompositions():
    # test_fmsm.cpp:99-103
    p = E.build_problem(E.Grid.unit_square(16), E.speed_constant(), E.ExitSpec.point_source((0.5, 0.5)))
    with pytest.raises(E.ConfigError):
        E.fmsm_solve(p, E.build_cells(p.grid, 1, 1))
    with pytest.raises(E.ConfigError):
        E.fmsm_solve(p, E.build_cells(p.grid, 1, 4))


def test_fmsm_exact_for_constant_speed():
    # test_fmsm.cpp:128-136: FMSM within 1e-13 of FMM for constant speed
    p = E.build_problem(E.Grid.unit_square(56), E.speed_constant(), E.ExitSpec.point_source((0.5, 0.5)))
    exact = O.oracle_solve(p, "fmm").u
    for c in (4, 7, 8):
        out = E.fmsm_solve(p, E.build_cells(p.grid, c, c))
        rel = np.abs(out.values - exact) / np.maximum(np.abs(exact), 1e-300)
        assert float(rel.max()) < 1e-13


# ---- heap-cell methods (exact device replay of heap_cell.cpp) ---------------

@pytest.mark.parametrize("cid,make,cells", SMALL_CASES, ids=[c[0] for c in SMALL_CASES])
def test_hcm_fhcm_small_golden_fields(cid, make, cells):
    arrays, meta = _small()
    p = make()
    for c in cells:
        for method in ("hcm", "fhcm"):
            key = f"{cid}/{method}/{c}"
            out = E.solve(p, EXACT.get(method, method), E.build_cells(p.grid, c, c))
            assert bitwise(out.values, arrays[key]), key
            m = meta[key]
            assert (out.sweeps, out.node_updates, out.heap_removals, out.hybrid.mon_checks,
                    out.hybrid.mon_single) == (m["sweeps"], m["node_updates"], m["heap_removals"],
                                               m["mon_checks"], m["mon_single"]), key


@pytest.mark.parametrize("method", ["hcm", "fhcm"])
@pytest.mark.parametrize("cs", [8, 16, 32, 64])
def test_heapcell_c2_bitwise_full_size(method, cs):
    big = _big()[f"c2/{method}/{cs}"]
    p = configs.config2().problem
    out = E.solve(p, EXACT.get(method, method), E.build_cells(p.grid, big["cells"], big["cells"]))
    assert sha(out.values) == big["sha256"]
    assert (out.sweeps, out.node_updates, out.heap_removals, out.hybrid.mon_checks,
            out.hybrid.mon_single) == (big["sweeps"], big["node_updates"], big["heap_removals"],
                                       big["mon_checks"], big["mon_single"])


@pytest.mark.parametrize("seed", range(6))
def test_heapcell_random_against_oracle(seed):
    rng = np.random.default_rng(300 + seed)
    m, n = int(rng.integers(10, 120)), int(rng.integers(10, 120))
    g = E.Grid(m, n, float(rng.uniform(0.002, 0.05)), 0.2, -0.4)
    F = rng.uniform(0.05, 3.0, size=(n, m))
    sp = lambda x, y, F=F, g=g: F[np.clip(np.rint((y - g.y0) / g.h).astype(int), 0, g.n - 1),  # noqa: E731
                                  np.clip(np.rint((x - g.x0) / g.h).astype(int), 0, g.m - 1)]
    k = int(rng.integers(1, 6))
    ex = E.ExitSpec.node_set([(int(rng.integers(0, m)), int(rng.integers(0, n))) for _ in range(k)],
                             list(rng.uniform(0, 0.1, size=k)))
    p = E.build_problem(g, sp, ex)
    for cx, cy in [(1, 1), (2, 3), (int(rng.integers(2, 10)), int(rng.integers(2, 10)))]:
        cells = E.build_cells(g, cx, cy)
        for method in ("hcm", "fhcm"):
            a = E.solve(p, EXACT.get(method, method), cells)
            b = O.oracle_solve(p, method, cells)
            assert bitwise(a.values, b.u), (method, cx, cy)
            assert (a.sweeps, a.node_updates, a.heap_removals, a.hybrid.mon_checks,
                    a.hybrid.mon_single) == (b.sweeps, b.node_updates, b.heap_removals,
                                             b.mon_checks, b.mon_single), (method, cx, cy)


def test_hcm_single_cell_is_lsm():
    # test_heap_cell.cpp:80-90: one cell -> HCM == LSM bit for bit, incl. counters
    p = E.build_problem(E.Grid.unit_square(33), E.speed_checkerboard(11),
                        E.ExitSpec.point_source((0.5, 0.5)))
    out = E.hcm_solve(p, E.build_cells(p.grid, 1, 1))
    lsm = O.oracle_solve(p, "lsm")
    assert out.heap_removals == 1 and out.hybrid.avhr == 1.0
    assert (out.sweeps, out.node_updates) == (lsm.sweeps, lsm.node_updates)
    assert bitwise(out.values, lsm.u)


def test_fhcm_exact_for_constant_speed():
    # test_heap_cell.cpp:142-151
    p = E.build_problem(E.Grid.unit_square(56), E.speed_constant(), E.ExitSpec.point_source((0.5, 0.5)))
    exact = O.oracle_solve(p, "fmm").u
    for c in (4, 8):
        out = E.fhcm_solve(p, E.build_cells(p.grid, c, c))
        rel = np.abs(out.values - exact) / np.maximum(np.abs(exact), 1e-300)
        assert float(rel.max()) < 1e-13
        assert out.hybrid.mon_pct == 100.0 and out.hybrid.avhr == 1.0


def test_heapcell_all_exit_and_first_removal():
    # test_heap_cell.cpp:153-185
    ex = E.ExitSpec.node_set([(i, j) for j in range(8) for i in range(8)])
    p = E.build_problem(E.Grid.unit_square(8), E.speed_constant(), ex)
    out = E.hcm_solve(p, E.build_cells(p.grid, 2, 2))
    assert out.node_updates == 0 and np.all(out.values == 0.0)
    ex = E.ExitSpec.node_set([(i, j) for j in range(4) for i in range(4)])
    p = E.build_problem(E.Grid.unit_square(8), E.speed_constant(), ex)
    exact = O.oracle_solve(p, "fmm").u
    for method in ("hcm", "fhcm"):
        out = E.solve(p, method, E.build_cells(p.grid, 2, 2))
        assert np.all(np.isfinite(out.values))
    out = E.hcm_solve(p, E.build_cells(p.grid, 2, 2))
    assert float(np.max(np.abs(out.values - exact) / np.maximum(exact, 1e-300))) < 1e-12


@pytest.mark.parametrize("env", [{"EIK_HC_HEAP_CAP": "2"}, {"EIK_HC_GLOBAL_HEAP": "1"},
                                 {"EIK_HC_CHAIN": "0"}, {"EIK_HC_CHAIN": "2"},
                                 {"EIK_HC_CTAS": "1"}, {"EIK_HC_WARPS": "1"},
                                 {"EIK_HC_SKIP_FROM": "0"}, {"EIK_HC_SKIP_FROM": "9"},
                                 {"EIK_HC_MIN_SMEM": "0", "EIK_HC_WARPS": "2"}],
                         ids=["heap-overflow-fallback", "global-heap", "no-chain", "chain-all",
                              "committer-only", "no-queue-helper", "skip-engine-all",
                              "skip-engine-none", "packed-ctas"])
def test_heapcell_engine_variants_bitwise(env, monkeypatch):
    """Every scheduling variant of the heap-cell kernel -- a committer heap that
    overflows shared memory and falls back to global memory, the global heap,
    plain-only / all-neighbour chained speculation, the committer alone, one
    warp per CTA (no queue helper), either in-cell engine for HCM's sweeps,
    CTAs packed several per SM -- must give the reference's bits and counters
    (C2 at 16x16-node cells)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    E.lib.eik_debug_reload_knobs()  # the library reads its knobs once
    try:
        _engine_variant_bitwise(env)
    finally:
        for k in env:
            monkeypatch.delenv(k)
        E.lib.eik_debug_reload_knobs()


def _engine_variant_bitwise(env):
    p = configs.config2(257).problem
    cells = E.build_cells(p.grid, 16, 16)
    for method in ("hcm", "fhcm"):
        a = E.solve(p, EXACT.get(method, method), cells)
        b = O.oracle_solve(p, method, cells)
        assert bitwise(a.values, b.u), (method, env)
        assert (a.sweeps, a.node_updates, a.heap_removals, a.hybrid.mon_checks,
                a.hybrid.mon_single) == (b.sweeps, b.node_updates, b.heap_removals,
                                         b.mon_checks, b.mon_single), (method, env)
