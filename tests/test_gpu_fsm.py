"""GPU parity for kernel (1), the wavefront FSM, and the FMM row it serves.

FSM must be bitwise-identical to the reference with identical sweep and
node-update counts (the wavefront is a topological order of the reference's
dependency DAG, SURVEY.md finding 2).  FMM values must match the reference's
FMM to L-inf <= 1e-10 (BASELINE.json north_star tolerance, fp64).
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _big():
    with open(os.path.join(GOLD, "big.json")) as f:
        return json.load(f)


def sha(u):
    return hashlib.sha256(np.ascontiguousarray(u, dtype=np.float64).tobytes()).hexdigest()


def bitwise(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def test_fsm_c1_bitwise_and_error():
    big = _big()["c1/fsm"]
    p = configs.config1().problem
    out = E.fsm_solve(p)
    assert sha(out.values) == big["sha256"]
    assert out.sweeps == big["sweeps"] == 5
    assert out.node_updates == big["node_updates"]
    g = p.grid
    xs = g.x0 + np.arange(g.m) * g.h
    X, Y = np.meshgrid(xs, xs)
    err = np.abs(out.values - np.hypot(X, Y).ravel())
    assert float(err.max()) == big["linf_vs_abs"]
    assert float(err.mean()) == pytest.approx(big["l1_vs_abs"], rel=1e-12)
    assert out.kernel_launches >= 1


def test_fsm_c2_bitwise_full_size():
    big = _big()["c2/fsm"]
    out = E.fsm_solve(configs.config2().problem)
    assert out.sweeps == big["sweeps"] == 47
    assert out.node_updates == big["node_updates"]
    assert sha(out.values) == big["sha256"]


def test_fmm_c2_matches_reference_fmm():
    big = _big()["c2/fmm"]
    p = configs.config2().problem
    out = E.fmm_solve(p)
    ref = O.oracle_solve(p, "fmm")
    assert sha(ref.u) == big["sha256"]  # the oracle is the reference here
    assert float(np.max(np.abs(out.values - ref.u))) <= 1e-10
    assert out.heap_removals == big["heap_removals"]


@pytest.mark.parametrize("m,n", [(2, 2), (3, 40), (40, 3), (33, 31), (31, 33), (64, 64),
                                 (65, 97), (200, 31), (17, 257)])
def test_fsm_shapes_bitwise(m, n):
    # strips of 32 rows: partial last strip, single strip, thin/tall grids
    g = E.Grid(m, n, 0.01, -0.3, 0.2)
    rng = np.random.default_rng(m * 1000 + n)
    src = (int(rng.integers(0, m)), int(rng.integers(0, n)))
    p = E.build_problem(g, E.speed_sinusoid(0.9, 3), E.ExitSpec.node_set([src]))
    a = E.fsm_solve(p)
    b = O.oracle_solve(p, "fsm")
    assert bitwise(a.values, b.u)
    assert (a.sweeps, a.node_updates) == (b.sweeps, b.node_updates)


@pytest.mark.parametrize("seed", range(6))
def test_fsm_random_fields_and_exit_sets_bitwise(seed):
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(20, 300)), int(rng.integers(20, 300))
    g = E.Grid(m, n, float(rng.uniform(0.001, 0.1)), 0.0, 0.0)
    k = int(rng.integers(1, 12))
    nodes = [(int(rng.integers(0, m)), int(rng.integers(0, n))) for _ in range(k)]
    costs = list(rng.uniform(0, 0.5, size=k))
    F = rng.uniform(0.05, 3.0, size=(n, m))
    mask = rng.random((n, m)) < 0.1
    F[mask] = 0.01  # slow obstacles, many sweeps
    sp = lambda x, y, F=F, g=g: F[np.rint((y - g.y0) / g.h).astype(int),  # noqa: E731
                                  np.rint((x - g.x0) / g.h).astype(int)]
    p = E.build_problem(g, sp, E.ExitSpec.node_set(nodes, costs))
    a = E.fsm_solve(p)
    b = O.oracle_solve(p, "fsm")
    assert bitwise(a.values, b.u)
    assert (a.sweeps, a.node_updates) == (b.sweeps, b.node_updates)


def test_fsm_all_exit_problem_one_sweep():
    # test_classic_solvers.cpp:66-84: every node an exit -> FSM sweeps == 1
    g = E.Grid.unit_square(7)
    p = E.build_problem(g, E.speed_constant(), E.ExitSpec.node_set(
        [(i, j) for j in range(7) for i in range(7)]))
    out = E.fsm_solve(p)
    assert out.sweeps == 1 and np.all(out.values == 0.0)


def test_fsm_boundary_exits_and_acceptance_sweeps():
    big = _big()["acceptance_fsm_sweeps"]
    for name, m, sp in [("constant", 1408, E.speed_constant()),
                        ("checker11", 176, E.speed_checkerboard(11)),
                        ("checker41", 164, E.speed_checkerboard(41))]:
        p = E.build_problem(E.Grid.unit_square(m), sp, E.ExitSpec.point_source((0.5, 0.5)))
        out = E.fsm_solve(p)
        assert out.sweeps == big[f"{name}/{m}"]["published"]
        assert sha(out.values) == big[f"{name}/{m}"]["sha256"]
    p = E.build_problem(E.Grid.unit_square(45), E.speed_sinusoid(0.5, 20), E.ExitSpec.full_boundary())
    a, b = E.fsm_solve(p), O.oracle_solve(p, "fsm")
    assert bitwise(a.values, b.u) and a.sweeps == b.sweeps


def test_plan_resident_reruns_are_identical():
    p = configs.config2(513).problem
    plan = E.Plan(p, "fsm")
    u1 = np.empty(p.grid.size())
    u2 = np.empty(p.grid.size())
    o1 = plan.run(u1)
    o2 = plan.run(u2)
    assert bitwise(u1, u2) and o1.sweeps == o2.sweeps
    assert bitwise(u1, O.oracle_solve(p, "fsm").u)
    plan.close()


def test_bad_speed_is_rejected():
    g = E.Grid.unit_square(9)
    p = E.build_problem(g, lambda x, y: np.where(x > 0.5, 0.0, 1.0), E.ExitSpec.point_source((0.5, 0.5)))
    with pytest.raises(ValueError):
        E.fsm_solve(p)


def test_cost_outside_the_square_roots_domain_is_rejected():
    """h / F beyond [2^-480, 2^500] is refused loudly (the wavefront's
    straight-line square root has no out-of-range path), not solved wrongly."""
    g = E.Grid.unit_square(9)
    for f in (1e150, 1e-152):
        p = E.build_problem(g, lambda x, y, f=f: np.full_like(x, f), E.ExitSpec.point_source((0.5, 0.5)))
        with pytest.raises(ValueError):
            E.fsm_solve(p)
    # well inside the domain, far from 1: still the reference's bits
    for f in (1e100, 1e-100):
        p = E.build_problem(g, lambda x, y, f=f: np.full_like(x, f), E.ExitSpec.point_source((0.5, 0.5)))
        a = E.fsm_solve(p)
        b = O.oracle_solve(p, "fsm")
        assert bitwise(a.values, b.u)


def test_set_device_selects_and_rejects():
    """eik_set_device: the library's own CUDA runtime follows the caller's
    device choice (one process per GPU); an absent device is a ConfigError."""
    E.set_device(0)
    p = E.build_problem(E.Grid.unit_square(33), E.speed_constant(), E.ExitSpec.point_source((0.5, 0.5)))
    assert E.fsm_solve(p).sweeps >= 2
    with pytest.raises(E.ConfigError):
        E.set_device(E.device_count() + 7)


def _knob(name, value):
    if value is None:
        os.environ.pop(name, None)
    else:
        os.environ[name] = value
    E.lib.eik_debug_reload_knobs()


@pytest.mark.parametrize("seed", range(4))
def test_super_block_skipping_equals_plain_wavefront_every_sweep(seed):
    """EIK_FSM_SB=0 (no super-block skipping) and the default agree sweep by
    sweep: the change flag of every sweep and the field after K sweeps."""
    rng = np.random.default_rng(100 + seed)
    m, n = int(rng.integers(40, 700)), int(rng.integers(40, 300))
    g = E.Grid(m, n, 0.01, 0.0, 0.0)
    F = rng.uniform(0.2, 3.0, size=(n, m))
    F[rng.random((n, m)) < 0.08] = 0.02
    sp = lambda x, y, F=F, g=g: F[np.rint((y - g.y0) / g.h).astype(int),  # noqa: E731
                                  np.rint((x - g.x0) / g.h).astype(int)]
    nodes = [(int(rng.integers(0, m)), int(rng.integers(0, n))) for _ in range(3)]
    p = E.build_problem(g, sp, E.ExitSpec.node_set(nodes))
    from paper_1110_6220_b200.distributed import DeviceStripSweeper

    def run(sb, K):
        _knob("EIK_FSM_SB", sb)
        try:
            s = DeviceStripSweeper(p)
            flags = s.plan.sweep(0, K)
            out = np.zeros((n, m))
            s.get_rows(0, n, out)
            s.close()
        finally:
            _knob("EIK_FSM_SB", None)
        return flags, out

    for K in (40, 7, 13):
        f1, u1 = run(None, K)
        f0, u0 = run("0", K)
        assert f1 == f0
        assert bitwise(u1, u0)


@pytest.mark.parametrize("seed", range(3))
def test_sweep_by_sweep_launches_carry_change_bits(seed):
    """One launch per sweep with rows rewritten in between (the sharded path's
    rounds): carrying the change bits across launches (default) equals
    evaluating every node in every launch (EIK_FSM_CONT=0), flag by flag."""
    rng = np.random.default_rng(200 + seed)
    m, n = int(rng.integers(60, 500)), int(rng.integers(70, 260))
    g = E.Grid(m, n, 0.01, 0.0, 0.0)
    F = rng.uniform(0.3, 2.0, size=(n, m))
    sp = lambda x, y, F=F, g=g: F[np.rint((y - g.y0) / g.h).astype(int),  # noqa: E731
                                  np.rint((x - g.x0) / g.h).astype(int)]
    # frozen first and last rows (a strip's ghost rows) plus one source
    nodes = [(i, 0) for i in range(m)] + [(i, n - 1) for i in range(m)] + [(m // 3, n // 2)]
    costs = [math.inf] * (2 * m) + [0.0]
    from paper_1110_6220_b200.distributed import DeviceStripSweeper
    p = E.build_problem(g, sp, E.ExitSpec.node_set(nodes, [5.0] * (2 * m) + [0.0]))
    del costs
    lo = rng.uniform(0.5, 3.0, size=m)
    hi = rng.uniform(0.5, 3.0, size=m)

    def run(cont):
        _knob("EIK_FSM_CONT", cont)
        try:
            s = DeviceStripSweeper(p)
            flags = []
            for k in range(80):
                flags.append(s.sweep(k))
                if k == 3:   # the neighbours' edge rows arrive
                    s.set_rows(0, 1, lo)
                if k == 6:
                    s.set_rows(n - 1, 1, hi)
                if k == 9:   # ... and improve in a few columns only
                    lo2 = lo.copy()
                    lo2[m // 2: m // 2 + 5] *= 0.5
                    s.set_rows(0, 1, lo2)
            out = np.zeros((n, m))
            s.get_rows(0, n, out)
            s.close()
        finally:
            _knob("EIK_FSM_CONT", None)
        return flags, out

    f1, u1 = run(None)
    f0, u0 = run("0")
    assert f1 == f0
    assert bitwise(u1, u0)
    assert not f1[-1]  # converged: the comparison covers the whole solve


def test_rows_longer_than_the_dirty_map_keep_the_plain_wavefront():
    """Rows beyond 131 k columns do not fit the kernel's shared-memory dirty
    map: super-block skipping is off and the result is still the reference's."""
    m, n = 140001, 37
    g = E.Grid(m, n, 1e-3, 0.0, 0.0)
    p = E.build_problem(g, lambda x, y: 1.0 + 0.5 * np.sin(40 * x) * np.cos(3 * y),
                        E.ExitSpec.node_set([(70000, 18), (5, 3)], [0.0, 0.25]))
    a = E.fsm_solve(p)
    b = O.oracle_solve(p, "fsm")
    assert bitwise(a.values, b.u)
    assert (a.sweeps, a.node_updates) == (b.sweeps, b.node_updates)


def test_wide_grid_with_skipping_is_bitwise():
    """A long thin grid (many super-blocks per strip, two strips)."""
    m, n = 20011, 50
    g = E.Grid(m, n, 1e-3, 0.0, 0.0)
    p = E.build_problem(g, lambda x, y: 1.0 + 0.7 * np.sin(25 * x) * np.sin(31 * y),
                        E.ExitSpec.node_set([(10, 10), (15000, 40)]))
    a = E.fsm_solve(p)
    b = O.oracle_solve(p, "fsm")
    assert bitwise(a.values, b.u)
    assert (a.sweeps, a.node_updates) == (b.sweeps, b.node_updates)
