"""GPU parity for the LSM and FMM rows of the exact solvers, and the ABI's
argument checks.

* lsm_solve (classic_solvers.cpp:160-212) runs in kernel (1) with its lock
  logic counted exactly: field and sweeps are fsm_solve's, node_updates the
  reference's count of unlocked nodes processed -- bit for bit and counter for
  counter against the C restatement (pinned to the reference,
  tests/test_oracle.py) on small grids and against the reference's own
  goldens (tests/golden/extra.json) at full size.
* fmm_solve's counters (sweeps 0, node_updates = candidate evaluations,
  heap_removals = M - |Q|) and its record_acceptance_order option.
* negative exit costs are refused (EIK_ERR_DOMAIN) instead of solved wrongly;
  grids taller than one device's FSM wavefront get EIK_ERR_NOT_IMPL up front.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(u):
    return hashlib.sha256(np.ascontiguousarray(u, dtype=np.float64).tobytes()).hexdigest()


def bitwise(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def _extra():
    with open(os.path.join(GOLD, "extra.json")) as f:
        return json.load(f)


def _random_problem(m, n, seed, n_src=3, field=None):
    g = E.Grid(m, n, 0.01, -0.3, 0.2)
    rng = np.random.default_rng(seed)
    flat = rng.choice(m * n, size=min(n_src, m * n - 1), replace=False)
    nodes = [(int(k % m), int(k // m)) for k in flat]
    sp = field or E.speed_sinusoid(0.9, 3)
    return E.build_problem(g, sp, E.ExitSpec.node_set(nodes))


@pytest.mark.parametrize("m,n,src", [(2, 2, 1), (3, 40, 1), (40, 3, 2), (33, 31, 3),
                                     (65, 97, 5), (200, 31, 2), (17, 257, 4), (129, 130, 9)])
def test_lsm_shapes_bitwise_with_counters(m, n, src):
    p = _random_problem(m, n, m * 7 + n, src)
    a = E.lsm_solve(p)
    b = O.oracle_solve(p, "lsm")
    assert bitwise(a.values, b.u)
    assert (a.sweeps, a.node_updates, a.heap_removals) == (b.sweeps, b.node_updates, 0)


def test_lsm_small_configs_against_oracle():
    cases = [configs.config1().problem, configs.config2(257).problem,
             configs.config3(257).problem, configs.config4(257).problem,
             configs.config5(257).problem]
    # boundary exit rows, a checkerboard, a maze with many direction changes
    g = E.Grid.unit_square(150)
    cases.append(E.build_problem(g, E.speed_checkerboard(11), E.ExitSpec.full_boundary()))
    for p in cases:
        a = E.lsm_solve(p)
        b = O.oracle_solve(p, "lsm")
        assert bitwise(a.values, b.u)
        assert (a.sweeps, a.node_updates) == (b.sweeps, b.node_updates)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5_2049"])
def test_lsm_full_size_against_reference_goldens(name):
    want = _extra()["lsm"][name]
    cfg = {"c1": configs.config1, "c2": configs.config2, "c3": configs.config3,
           "c4": configs.config4, "c5_2049": lambda: configs.config5(2049)}[name]()
    out = E.lsm_solve(cfg.problem)
    assert sha(out.values) == want["sha256"]
    assert (out.sweeps, out.node_updates) == (want["sweeps"], want["node_updates"])


def test_lsm_in_a_batch_equals_alone():
    p = configs.config2(513).problem
    alone = E.lsm_solve(p)
    outs, _ = E.solve_batch([(p, "lsm", None, None), (p, "fsm", None, None),
                             (p, "lsm", None, None)])
    for o in (outs[0], outs[2]):
        assert bitwise(o.values, alone.values)
        assert (o.sweeps, o.node_updates) == (alone.sweeps, alone.node_updates)
    assert bitwise(outs[1].values, alone.values)  # LSM's field is FSM's


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_fmm_row_counters_and_distance_to_reference_fmm(name):
    """The GPU FMM row is the exact fixed point, bitwise the reference FSM
    field; its distance to the reference FMM is therefore exactly the stored
    L-inf(reference FMM - reference FSM), which must be <= 1e-10.  Counters
    are fmm_solve's own."""
    want = _extra()["fmm_vs_fsm"][name]
    cfg = {"c2": configs.config2, "c3": configs.config3, "c4": configs.config4}[name]()
    out = E.fmm_solve(cfg.problem)
    assert sha(out.values) == want["fsm_sha256"]
    assert want["linf"] <= 1e-10
    ref = want["fmm"]
    assert (out.sweeps, out.node_updates, out.heap_removals) == (
        ref["sweeps"], ref["node_updates"], ref["heap_removals"])


@pytest.mark.parametrize("m,n,src", [(2, 2, 1), (33, 31, 3), (65, 97, 40), (200, 31, 2)])
def test_fmm_counters_small(m, n, src):
    p = _random_problem(m, n, m + n, src)
    a = E.fmm_solve(p)
    b = O.oracle_solve(p, "fmm")
    assert float(np.max(np.abs(a.values - b.u))) <= 1e-10
    assert (a.sweeps, a.node_updates, a.heap_removals) == (0, b.node_updates, b.heap_removals)


def test_fmm_acceptance_order():
    # test_classic_solvers.cpp:99-111: M - |Q| entries, non-decreasing values
    g = E.Grid.unit_square(33)
    p = E.build_problem(g, E.speed_checkerboard(11), E.ExitSpec.point_source((0.5, 0.5)))
    out = E.fmm_solve(p, E.FmmOptions(record_acceptance_order=True))
    order = out.acceptance_order
    assert order.size == g.size() - 1
    assert np.all(np.diff(out.values[order]) >= 0.0)
    assert sorted(order.tolist()) == sorted(set(range(g.size())) - set(p.exit_nodes))
    plain = E.fmm_solve(p)
    assert bitwise(plain.values, out.values) and plain.acceptance_order is None


def test_negative_exit_cost_is_refused():
    g = E.Grid.unit_square(40)
    p = E.build_problem(g, E.speed_constant(), E.ExitSpec.node_set([(3, 4), (20, 30)], [0.0, -1.0]))
    for method, cells in (("fsm", None), ("fmm", None), ("lsm", None),
                          ("hcm", E.build_cells(g, 4, 4)), ("fhcm", E.build_cells(g, 4, 4))):
        with pytest.raises(ValueError, match="negative exit costs"):
            E.solve(p, method, cells)


def test_too_tall_grid_fails_up_front():
    g = E.Grid(2, 48001, 1e-3, 0.0, 0.0)
    p = E.build_problem(g, E.speed_constant(), E.ExitSpec.node_set([(0, 0)]))
    with pytest.raises(NotImplementedError, match="rows"):
        E.fsm_solve(p)
