"""Host-side logic and the C-ABI library, without a GPU: the library loads,
exports every symbol include/eikonal_b200.h declares, validates arguments
with the reference's error semantics, and the Python mirror of the
reference's problem construction agrees with the reference."""
import ctypes as C
import math
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1110_6220_b200 as E
from paper_1110_6220_b200 import _native as N
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "eikonal_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eik_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = _header_functions()
    assert len(names) >= 14
    lib = C.CDLL(N.LIB_PATH)
    for nm in names:
        assert hasattr(lib, nm), nm
    syms = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                          text=True).stdout
    for nm in names:
        assert re.search(rf"\bT {nm}$", syms, flags=re.M), nm


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_abi_version():
    assert N.lib.eik_abi_version() == 4


def _c_problem(p):
    from paper_1110_6220_b200.solvers import _c_problem
    return _c_problem(p, p.sampled_speed())


def test_config_errors_before_any_device_work():
    g = E.Grid.unit_square(8)
    p = E.build_problem(g, E.speed_constant(), E.ExitSpec.point_source((0.5, 0.5)))
    cp, keep = _c_problem(p)
    out = N.eik_output()
    u = np.empty(64)
    out.u = N.dptr(u)
    # fmsm with < 2x2 cells -> ConfigError (fmsm.cpp:124-125)
    cells = N.eik_cells(1, 4)
    rc = N.lib.eik_solve(C.byref(cp), C.byref(cells), N.EIK_FMSM, C.byref(out))
    assert rc == N.EIK_ERR_CONFIG and "2x2" in N.lib.eik_last_error().decode()
    # too many cells (cells.cpp:35)
    rc = N.lib.eik_solve(C.byref(cp), C.byref(N.eik_cells(9, 2)), N.EIK_HCM, C.byref(out))
    assert rc == N.EIK_ERR_CONFIG
    # empty exit set (grid.cpp:77)
    cp.n_exit = 0
    assert N.lib.eik_solve(C.byref(cp), None, N.EIK_FSM, C.byref(out)) == N.EIK_ERR_CONFIG


def test_no_cpu_fallback_without_device():
    if E.device_count() > 0:
        pytest.skip("a device is visible")
    p = E.build_problem(E.Grid.unit_square(8), E.speed_constant(), E.ExitSpec.point_source((0.5, 0.5)))
    with pytest.raises(RuntimeError, match="CUDA"):
        E.fsm_solve(p)


def test_build_problem_mirrors_reference():
    with pytest.raises(E.ConfigError):
        E.Grid(1, 5, 1.0)
    with pytest.raises(ValueError):
        E.snap_point_to_node(E.Grid.unit_square(5), (1.5, 0.5))
    g = E.Grid.unit_square(5)
    p = E.build_problem(g, E.speed_constant(),
                        E.ExitSpec.node_set([(1, 1), (0, 0), (1, 1)], [0.5, 0.2, 0.1]))
    assert list(p.exit_nodes) == [0, 6] and list(p.exit_cost) == [0.2, 0.1]
    pb = E.build_problem(g, E.speed_constant(), E.ExitSpec.full_boundary())
    assert len(pb.exit_nodes) == 16


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_snap_matches_reference():
    rng = np.random.default_rng(3)
    for m in (5, 64, 257):
        g = E.Grid.centered(m)
        pts = rng.uniform(-1, 1, size=(300, 2))
        # exact ties: half-way points resolve toward the smaller index
        pts[:20] = (np.floor(pts[:20] / g.h) + 0.5) * g.h
        for x, y in pts:
            i = C.c_int64()
            j = C.c_int64()
            assert O.rlib.ref_snap(C.byref(g.c()), x, y, C.byref(i), C.byref(j)) == 0
            assert E.snap_point_to_node(g, (x, y)) == (i.value, j.value)


def test_build_cells_and_geometry():
    # cells.cpp:7-47 / test_cells.cpp:9-35
    d = E.build_cells(E.Grid.unit_square(176), 22, 22)
    assert all(e - b == 8 for b, e in zip(d.i_begin, d.i_end))
    assert d.hc_x == pytest.approx(8.0 / 175.0)
    d = E.build_cells(E.Grid.unit_square(9), 2, 2)
    assert d.i_end[0] - d.i_begin[0] == 4 and d.i_end[1] - d.i_begin[1] == 5
    with pytest.raises(E.ConfigError):
        E.build_cells(E.Grid.unit_square(8), 0, 2)
    with pytest.raises(E.ConfigError):
        E.build_cells(E.Grid.unit_square(8), 2, 9)
    g = E.Grid.centered(2049)
    J = N.lib.eik_cell_centers(C.byref(g.c()), 128, 128, N.dptr(None))
    xy = np.empty((J, 2))
    N.lib.eik_cell_centers(C.byref(g.c()), 128, 128, N.dptr(xy))
    # last cell is 17 wide (remainder): centre of nodes 1905..2048...
    d = E.build_cells(g, 128, 128)
    last = 127
    want = 0.5 * (g.x(d.i_begin[last]) + g.x(d.i_end[last] - 1))
    assert xy[last, 0] == want
    for side in range(4):
        cnt = N.lib.eik_cell_probe_points(C.byref(g.c()), 128, 128, side, N.dptr(None))
        pts = np.empty((cnt, 2))
        N.lib.eik_cell_probe_points(C.byref(g.c()), 128, 128, side, N.dptr(pts))
        assert np.all(pts >= -1.0) and np.all(pts <= 1.0)


def test_field_sampling_is_bitwise_on_demand_evaluation():
    from paper_1110_6220_b200 import configs
    g = E.Grid.centered(129)
    p, q, phi = configs.sinsum_coeffs(5)
    fields = [E.speed_sinusoid(0.5, 20), E.speed_sinsum(p, q, phi),
              E.speed_blocks(np.array([[1.0, 2.0], [2.0, 1.0]]), -1, -1, 1.0),
              E.speed_nodemask(g, configs.maze_mask(129, 1), 0.01, 1.0)]
    xs = g.x0 + np.arange(g.m) * g.h
    X, Y = np.meshgrid(xs, xs)
    for f in fields:
        F = f.sample(g)
        assert np.array_equal(F, f(X.ravel(), Y.ravel())), f.name
        assert np.all(F > 0)
    Fs = fields[1].sample(g)
    assert 0.5 <= Fs.min() and Fs.max() <= 1.5


def test_python_callable_speed_sampling():
    g = E.Grid.unit_square(17)
    p = E.build_problem(g, lambda x, y: 1.0 + 0.0 * x, E.ExitSpec.point_source((0.5, 0.5)))
    assert np.array_equal(p.sampled_speed(), np.ones(17 * 17))


def test_maze_config_shape():
    from paper_1110_6220_b200 import configs
    mk = configs.maze_mask(1025, 4)
    frac = mk.mean()
    assert 0.05 <= frac < 0.07
    assert mk[0, 0] == 0
