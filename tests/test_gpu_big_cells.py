"""Any cell decomposition the reference accepts (build_cells, cells.cpp:32-47):
cells taller than the register engine's 128 rows or too large for a
shared-memory tile are swept in place in the padded field by the
band-splitting engine (k_cellsweep.cuh big_cell_sweep) -- FMSM by its
dataflow kernel, HCM/FHCM by the exact serial heap loop
(k_heapcell.cu heapcell_serial_kernel).  Bit-exact with identical counters
against the C restatement (pinned to the reference, tests/test_oracle.py).
"""
import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import configs
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def bitwise(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def _check(p, method, cells):
    dev = "hcm_exact" if method == "hcm" else method
    a = E.solve(p, dev, cells)
    b = O.oracle_solve(p, method, cells)
    assert bitwise(a.values, b.u), (method, cells.cells_x, cells.cells_y)
    assert (a.sweeps, a.node_updates, a.heap_removals, a.hybrid.mon_checks,
            a.hybrid.mon_single) == (b.sweeps, b.node_updates, b.heap_removals, b.mon_checks,
                                     b.mon_single), (method, cells.cells_x, cells.cells_y)
    return a


@pytest.mark.parametrize("method", ["hcm", "fhcm", "fmsm"])
def test_c1_two_by_two_cells(method):
    # the verdict's example: 257^2 in 2x2 cells (the last cells 129 rows tall)
    p = configs.config1().problem
    _check(p, method, E.build_cells(p.grid, 2, 2))


@pytest.mark.parametrize("m,n,cx,cy", [(200, 150, 1, 1), (150, 301, 1, 2), (300, 300, 2, 2),
                                       (413, 270, 3, 2), (130, 500, 1, 3), (270, 129, 2, 1)])
def test_random_big_cells(m, n, cx, cy):
    rng = np.random.default_rng(m * 7 + n * 3 + cx)
    g = E.Grid(m, n, 0.004, -0.3, 0.1)
    F = rng.uniform(0.2, 3.0, size=(n, m))
    sp = lambda x, y, F=F, g=g: F[np.clip(np.rint((y - g.y0) / g.h).astype(int), 0, g.n - 1),  # noqa: E731
                                  np.clip(np.rint((x - g.x0) / g.h).astype(int), 0, g.m - 1)]
    k = int(rng.integers(1, 5))
    ex = E.ExitSpec.node_set([(int(rng.integers(0, m)), int(rng.integers(0, n))) for _ in range(k)],
                             list(rng.uniform(0, 0.05, size=k)))
    p = E.build_problem(g, sp, ex)
    cells = E.build_cells(g, cx, cy)
    for method in ("hcm", "fhcm") + (("fmsm",) if cx >= 2 and cy >= 2 else ()):
        _check(p, method, cells)
    band = E.solve(p, "hcm", cells)  # big cells: the band default falls back to the exact loop
    assert float(np.max(np.abs(band.values - O.oracle_solve(p, "hcm", cells).u))) <= 1e-10


def test_one_cell_hcm_is_lsm_big():
    # test_heap_cell.cpp:80-90 with a cell too large for a tile
    g = E.Grid.unit_square(180)
    p = E.build_problem(g, E.speed_sinusoid(0.5, 4), E.ExitSpec.point_source((0.3, 0.6)))
    out = E.solve(p, "hcm_exact", E.build_cells(g, 1, 1))
    lsm = O.oracle_solve(p, "lsm")
    assert bitwise(out.values, lsm.u)
    assert (out.sweeps, out.node_updates) == (lsm.sweeps, lsm.node_updates)


@pytest.mark.parametrize("method", ["hcm", "fhcm", "fmsm"])
def test_c2_128_node_cells(method):
    """C2 (2049^2) in 16x16 cells: 128-node cells with a 129-node last row and
    column, too large for a shared-memory tile."""
    p = configs.config2().problem
    _check(p, method, E.build_cells(p.grid, 16, 16))


@pytest.mark.parametrize("h", [33, 40, 47, 63, 64, 65, 95, 96, 97, 127, 128])
def test_cells_of_33_to_128_rows_as_bands(h):
    """Cells of 33-128 rows go through the locked engine band by band (32 rows
    each, k_cellsweep.cuh cell_sweep_lock_bands) in the replay and the HCM band
    kernel: every height class, with a shorter last band and a remainder cell
    row, against the C restatement -- values and every counter (exact replay),
    and <= 1e-10 for the band scheduler."""
    rng = np.random.default_rng(1000 + h)
    m, n = 3 * 37 + 5, 3 * h + 7  # cells_y = 3: two cells of h rows, the last h + 7
    g = E.Grid(m, n, 0.003, -0.1, 0.2)
    F = rng.uniform(0.3, 2.5, size=(n, m))
    F[rng.random((n, m)) < 0.05] = 0.05
    sp = lambda x, y, F=F, g=g: F[np.clip(np.rint((y - g.y0) / g.h).astype(int), 0, g.n - 1),  # noqa: E731
                                  np.clip(np.rint((x - g.x0) / g.h).astype(int), 0, g.m - 1)]
    ex = E.ExitSpec.node_set([(int(rng.integers(0, m)), int(rng.integers(0, n))) for _ in range(3)],
                             list(rng.uniform(0, 0.05, size=3)))
    p = E.build_problem(g, sp, ex)
    cells = E.build_cells(g, 3, 3)
    for method in ("hcm", "fhcm"):
        _check(p, method, cells)
    band = E.solve(p, "hcm", cells)
    assert float(np.max(np.abs(band.values - O.oracle_solve(p, "hcm", cells).u))) <= 1e-10
