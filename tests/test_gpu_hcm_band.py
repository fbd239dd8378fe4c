"""GPU tests of the HCM band scheduler (north_star item 3; k_heapcell.cu
hcm_band_kernel): every round processes the in-band queued cells that are
local minima among their in-band queued neighbours, so HCM runs with a
different pop order.  HCM ends at the discrete fixed point whatever the order,
so the field must match the reference's hcm_solve within the north_star
tolerance (1e-10, fp64); pops / sweeps / node updates are the band order's
own and are reported beside the reference's.  Rounds are a deterministic
function of the values (selection depends on sets, not on list order), so a
solve is bit-reproducible.
"""
import json
import os

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs
from oracle import oracle as O
from tests.golden.make_golden import SMALL_CASES

pytestmark = pytest.mark.gpu
TOL = 1e-10


def bitwise(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


@pytest.mark.parametrize("cid,make,cells", SMALL_CASES, ids=[c[0] for c in SMALL_CASES])
def test_band_small_cases_against_reference_hcm(cid, make, cells):
    p = make()
    for c in cells:
        cl = E.build_cells(p.grid, c, c)
        band = E.solve(p, "hcm", cl)
        ref = O.oracle_solve(p, "hcm", cl)  # pinned to the reference (test_oracle.py)
        assert float(np.max(np.abs(band.values - ref.u))) <= TOL, (cid, c)
        assert band.heap_removals >= 1 and band.rounds >= 1
        assert band.rounds <= band.heap_removals


@pytest.mark.parametrize("seed", range(6))
def test_band_random_grids(seed):
    rng = np.random.default_rng(900 + seed)
    m, n = int(rng.integers(10, 120)), int(rng.integers(10, 120))
    g = E.Grid(m, n, float(rng.uniform(0.002, 0.05)), 0.2, -0.4)
    F = rng.uniform(0.05, 3.0, size=(n, m))
    sp = lambda x, y, F=F, g=g: F[np.clip(np.rint((y - g.y0) / g.h).astype(int), 0, g.n - 1),  # noqa: E731
                                  np.clip(np.rint((x - g.x0) / g.h).astype(int), 0, g.m - 1)]
    k = int(rng.integers(1, 6))
    ex = E.ExitSpec.node_set([(int(rng.integers(0, m)), int(rng.integers(0, n))) for _ in range(k)],
                             list(rng.uniform(0, 0.1, size=k)))
    p = E.build_problem(g, sp, ex)
    for cx, cy in [(1, 1), (2, 3), (int(rng.integers(2, 12)), int(rng.integers(2, 12)))]:
        cells = E.build_cells(g, cx, cy)
        a = E.solve(p, "hcm", cells)
        b = O.oracle_solve(p, "hcm", cells)
        scale = max(1.0, float(np.max(b.u)))
        assert float(np.max(np.abs(a.values - b.u))) <= TOL * scale, (cx, cy)


@pytest.mark.parametrize("cs", [8, 16, 32, 64])
def test_band_c2_full_size(cs):
    """C2 at 2049^2: the band field against the exact replay (bitwise the
    reference, test_gpu_cells.py) and the fixed point FSM computes."""
    p = configs.config2().problem
    cells = E.build_cells(p.grid, p.grid.m // cs, p.grid.m // cs)
    band = E.solve(p, "hcm", cells)
    exact = E.solve(p, "hcm_exact", cells)
    fsm = E.fsm_solve(p)
    assert float(np.max(np.abs(band.values - exact.values))) <= TOL
    assert float(np.max(np.abs(band.values - fsm.values))) <= TOL
    again = E.solve(p, "hcm", cells)
    assert bitwise(again.values, band.values)  # deterministic
    assert (again.heap_removals, again.sweeps, again.node_updates, again.rounds) == (
        band.heap_removals, band.sweeps, band.node_updates, band.rounds)
    assert band.rounds < exact.heap_removals


@pytest.mark.parametrize("name,cs", [("c3", 16), ("c3", 48), ("c4", 16), ("c4", 32)])
def test_band_c3_c4_full_size(name, cs):
    with open(os.path.join(os.path.dirname(__file__), "golden", "c34.json")) as f:
        gold = json.load(f)[f"{name}/hcm/{cs}"]
    p = (configs.config3 if name == "c3" else configs.config4)().problem
    cells = E.build_cells(p.grid, gold["cells"], gold["cells"])
    band = E.solve(p, "hcm", cells)
    exact = E.solve(p, "hcm_exact", cells)  # bitwise the reference (test_gpu_configs.py)
    assert exact.heap_removals == gold["heap_removals"]
    assert float(np.max(np.abs(band.values - exact.values))) <= TOL


def test_band_in_a_batch_equals_alone():
    p = configs.config2(513).problem
    cells = E.build_cells(p.grid, 32, 32)
    alone = E.solve(p, "hcm", cells)
    outs, _ = E.solve_batch([(p, "hcm", cells, None), (p, "fhcm", cells, None),
                             (p, "hcm", cells, None)])
    for o in (outs[0], outs[2]):
        assert bitwise(o.values, alone.values)
        assert (o.heap_removals, o.rounds) == (alone.heap_removals, alone.rounds)


def test_default_mode_switch():
    p = configs.config2(257).problem
    cells = E.build_cells(p.grid, 16, 16)
    ref = O.oracle_solve(p, "hcm", cells)
    E.set_hcm_mode("exact")
    try:
        ex = E.solve(p, "hcm", cells)
    finally:
        E.set_hcm_mode("band")
    assert bitwise(ex.values, ref.u) and ex.heap_removals == ref.heap_removals
    assert ex.rounds == 0
    band = E.solve(p, "hcm", cells)
    assert band.rounds > 0


@pytest.mark.parametrize("seed", range(4))
def test_band_walls_widen_the_band(seed):
    """A maze-like field (walls of F = 1e-3, 1000x the base h/F): the adaptive
    width grows to its cap on narrow fronts; the field still lands on the
    reference HCM's fixed point, and the solve is reproducible."""
    rng = np.random.default_rng(1700 + seed)
    m = n = int(rng.integers(60, 160))
    g = E.Grid(m, n, 1.0 / (m - 1), 0.0, 0.0)
    F = np.ones((n, m))
    for _ in range(int(rng.integers(3, 9))):  # walls with a gap
        if rng.integers(0, 2):
            j = int(rng.integers(2, n - 2))
            F[j:j + 2, :] = 1e-3
            a = int(rng.integers(0, m - 6))
            F[j:j + 2, a:a + 5] = 1.0
        else:
            i = int(rng.integers(2, m - 2))
            F[:, i:i + 2] = 1e-3
            a = int(rng.integers(0, n - 6))
            F[a:a + 5, i:i + 2] = 1.0
    sp = lambda x, y, F=F, g=g: F[np.clip(np.rint((y - g.y0) / g.h).astype(int), 0, g.n - 1),  # noqa: E731
                                  np.clip(np.rint((x - g.x0) / g.h).astype(int), 0, g.m - 1)]
    p = E.build_problem(g, sp, E.ExitSpec.node_set([(0, 0)], [0.0]))
    for c in (4, 8, 16):
        cells = E.build_cells(g, max(1, m // c), max(1, n // c))
        a = E.solve(p, "hcm", cells)
        b = O.oracle_solve(p, "hcm", cells)
        scale = max(1.0, float(np.max(b.u)))
        assert float(np.max(np.abs(a.values - b.u))) <= TOL * scale, c
        again = E.solve(p, "hcm", cells)
        assert bitwise(again.values, a.values) and again.rounds == a.rounds
