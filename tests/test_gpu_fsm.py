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


def test_set_device_selects_and_rejects():
    """eik_set_device: the library's own CUDA runtime follows the caller's
    device choice (one process per GPU); an absent device is a ConfigError."""
    E.set_device(0)
    p = E.build_problem(E.Grid.unit_square(33), E.speed_constant(), E.ExitSpec.point_source((0.5, 0.5)))
    assert E.fsm_solve(p).sweeps >= 2
    with pytest.raises(E.ConfigError):
        E.set_device(E.device_count() + 7)
