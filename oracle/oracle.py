"""ORACLE -- TEST INFRASTRUCTURE ONLY.

ctypes access to the checkers: oracle/liboracle.so (C restatement) and
oracle/_ref/libeikref.so (the unmodified reference, built from
/root/reference by oracle/Makefile).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from paper_1110_6220_b200 import _native as N
from paper_1110_6220_b200.problem import CellDecomposition, CellTables, Problem, SpeedField

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libeikref.so")
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class orc_problem(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("h", C.c_double), ("x0", C.c_double),
                ("y0", C.c_double), ("F", _dp), ("exit_nodes", _i64p), ("exit_cost", _dp),
                ("n_exit", C.c_int64), ("exit_points_xy", _dp), ("exit_point_cost", _dp),
                ("n_exit_points", C.c_int64)]


class orc_cells(C.Structure):
    _fields_ = [("cells_x", C.c_int32), ("cells_y", C.c_int32), ("probe_w", _dp),
                ("probe_e", _dp), ("probe_s", _dp), ("probe_n", _dp), ("center_F", _dp)]


class orc_stats(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("node_updates", C.c_int64),
                ("heap_removals", C.c_int64), ("mon_checks", C.c_int64),
                ("mon_single", C.c_int64)]


class ref_stats(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("node_updates", C.c_int64),
                ("heap_removals", C.c_int64), ("cell_removals", C.c_int64),
                ("cell_sweeps", C.c_int64), ("mon_checks", C.c_int64),
                ("mon_single", C.c_int64), ("avhr", C.c_double), ("avs", C.c_double),
                ("mon_pct", C.c_double), ("elapsed_ms", C.c_double)]


@dataclass
class Result:
    u: np.ndarray
    sweeps: int
    node_updates: int
    heap_removals: int
    mon_checks: int = 0
    mon_single: int = 0
    elapsed_ms: float = 0.0


def _load_oracle():
    lib = C.CDLL(ORACLE_SO)
    for nm in ("orc_fmm", "orc_fsm", "orc_lsm"):
        getattr(lib, nm).argtypes = [C.POINTER(orc_problem), _dp, C.POINTER(orc_stats)]
        getattr(lib, nm).restype = C.c_int
    for nm in ("orc_hcm", "orc_fhcm", "orc_fmsm"):
        getattr(lib, nm).argtypes = [C.POINTER(orc_problem), C.POINTER(orc_cells), _dp,
                                     C.POINTER(orc_stats)]
        getattr(lib, nm).restype = C.c_int
    lib.orc_fmsm_ex.argtypes = [C.POINTER(orc_problem), C.POINTER(orc_cells), _dp,
                                C.POINTER(orc_stats), C.c_void_p]
    lib.orc_fmsm_ex.restype = C.c_int
    lib.orc_quadrant_update.argtypes = [C.c_double] * 4
    lib.orc_quadrant_update.restype = C.c_double
    lib.orc_node_update.argtypes = [_dp, C.c_double, C.c_double]
    lib.orc_node_update.restype = C.c_double
    lib.orc_directional_update.argtypes = [_dp, C.c_int, C.c_double, C.c_double]
    lib.orc_directional_update.restype = C.c_double
    lib.orc_fsm_sweep.argtypes = [C.c_int64, C.c_int64, C.c_double, _dp, C.c_void_p, _dp, C.c_int]
    lib.orc_fsm_sweep.restype = C.c_int
    return lib


def _load_ref():
    if not os.path.exists(REF_SO):
        return None
    lib = C.CDLL(REF_SO)
    lib.ref_solve.argtypes = [C.c_int, C.POINTER(N.eik_grid), C.POINTER(N.eik_field), _i64p, _dp,
                              C.c_int64, _dp, _dp, C.c_int64, C.c_int, C.c_int, _dp,
                              C.POINTER(ref_stats)]
    lib.ref_solve.restype = C.c_int
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_quadrant_update.argtypes = [C.c_double] * 4
    lib.ref_quadrant_update.restype = C.c_double
    lib.ref_node_update.argtypes = [_dp, C.c_double, C.c_double]
    lib.ref_node_update.restype = C.c_double
    lib.ref_directional_update.argtypes = [_dp, C.c_int, C.c_double, C.c_double]
    lib.ref_dump_field.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_char_p, C.c_int]
    lib.ref_dump_field.restype = C.c_int
    lib.ref_csv_line.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, _dp, _i64p, C.c_char_p,
                                 C.c_int]
    lib.ref_csv_line.restype = C.c_int
    lib.ref_csv_header.argtypes = []
    lib.ref_csv_header.restype = C.c_char_p
    lib.ref_directional_update.restype = C.c_double
    lib.ref_snap.argtypes = [C.POINTER(N.eik_grid), C.c_double, C.c_double, _i64p, _i64p]
    lib.ref_snap.restype = C.c_int
    lib.ref_metrics.argtypes = [C.POINTER(N.eik_grid), C.POINTER(N.eik_field), _i64p, _dp,
                                C.c_int64, C.c_int, _dp, _dp, _dp]
    lib.ref_metrics.restype = C.c_int
    lib.ref_named_speed.argtypes = [C.c_char_p, C.c_double, C.c_double]
    lib.ref_named_speed.restype = C.c_double
    return lib


olib = _load_oracle()
rlib = _load_ref()


def have_ref() -> bool:
    return rlib is not None


def _orc_problem(p: Problem):
    F = p.sampled_speed()
    en = np.ascontiguousarray(p.exit_nodes, dtype=np.int64)
    ec = np.ascontiguousarray(p.exit_cost, dtype=np.float64)
    pts = np.ascontiguousarray(p.exit_points, dtype=np.float64).reshape(-1)
    pc = np.ascontiguousarray(p.exit_point_cost, dtype=np.float64)
    g = p.grid
    op = orc_problem(g.m, g.n, g.h, g.x0, g.y0, F.ctypes.data_as(_dp), en.ctypes.data_as(_i64p),
                     ec.ctypes.data_as(_dp), len(en),
                     pts.ctypes.data_as(_dp) if pts.size else _dp(),
                     pc.ctypes.data_as(_dp) if pc.size else _dp(), len(pc))
    return op, (F, en, ec, pts, pc)


def oracle_solve(p: Problem, method: str, cells: CellDecomposition = None,
                 tables: CellTables = None) -> Result:
    """C restatement (oracle/eik_oracle.c)."""
    from paper_1110_6220_b200.problem import cell_tables
    op, keep = _orc_problem(p)
    u = np.empty(p.grid.size(), dtype=np.float64)
    st = orc_stats()
    if method in ("fmm", "fsm", "lsm"):
        rc = getattr(olib, "orc_" + method)(C.byref(op), u.ctypes.data_as(_dp), C.byref(st))
    else:
        if tables is None:
            tables = cell_tables(p, cells)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (tables.probe_w, tables.probe_e, tables.probe_s, tables.probe_n, tables.center)]
        oc = orc_cells(cells.cells_x, cells.cells_y, *[a.ctypes.data_as(_dp) for a in arrs])
        rc = getattr(olib, "orc_" + method)(C.byref(op), C.byref(oc), u.ctypes.data_as(_dp),
                                            C.byref(st))
    if rc == 1:
        raise N.ConfigError("oracle: bad configuration")
    if rc == 3:
        raise N.BudgetError("heap-cell removal budget exceeded")
    return Result(u, st.sweeps, st.node_updates, st.heap_removals, st.mon_checks, st.mon_single)


def oracle_fmsm_order(p: Problem, cells: CellDecomposition, tables: CellTables = None):
    """FMSM Part I only (fmsm.cpp:126-162): the quantised cell order and the
    coarse Fast March's heap removals and node updates."""
    from paper_1110_6220_b200.problem import cell_tables
    op, keep = _orc_problem(p)
    if tables is None:
        tables = cell_tables(p, cells)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
            (tables.probe_w, tables.probe_e, tables.probe_s, tables.probe_n, tables.center)]
    oc = orc_cells(cells.cells_x, cells.cells_y, *[a.ctypes.data_as(_dp) for a in arrs])
    order = np.empty(cells.cells_x * cells.cells_y, dtype=np.int64)
    st = orc_stats()
    rc = olib.orc_fmsm_ex(C.byref(op), C.byref(oc), None, C.byref(st), order.ctypes.data)
    if rc == 1:
        raise N.ConfigError("oracle: bad configuration")
    return order, st.heap_removals, st.node_updates


def oracle_fsm_sweep(m: int, n: int, h: float, F: np.ndarray, frozen: np.ndarray, u: np.ndarray,
                     direction: int) -> bool:
    """One FSM sweep in place (classic_solvers.cpp:140-155); frozen nodes are
    skipped.  Test infrastructure for the strip-Jacobi emulation."""
    assert F.dtype == np.float64 and u.dtype == np.float64 and frozen.dtype == np.uint8
    return bool(olib.orc_fsm_sweep(m, n, h, F.ctypes.data_as(_dp), frozen.ctypes.data,
                                   u.ctypes.data_as(_dp), direction))


def ref_dump_field(u: np.ndarray, m: int, n: int, h: float, path: str, ascii: bool) -> None:
    """The reference's dump_field (field_io.cpp:20-45)."""
    uu = np.ascontiguousarray(u, dtype=np.float64)
    if rlib.ref_dump_field(uu.ctypes.data_as(_dp), m, n, h, path.encode(), 1 if ascii else 0):
        raise RuntimeError(rlib.ref_last_error().decode())


_METHOD_ENUM = {"fmm": 0, "fsm": 1, "lsm": 2, "hcm": 3, "fhcm": 4, "fmsm": 5}  # experiment.hpp:11


def ref_csv_line(problem: str, method: str, grid_m: int, cells_x: int, d9, c3) -> str:
    """The reference's csv_line (experiment.cpp:319-329)."""
    d = np.ascontiguousarray(d9, dtype=np.float64)
    c = np.ascontiguousarray(c3, dtype=np.int64)
    buf = C.create_string_buffer(1024)
    rlib.ref_csv_line(problem.encode(), _METHOD_ENUM[method], grid_m, cells_x,
                      d.ctypes.data_as(_dp), c.ctypes.data_as(_i64p), buf, 1024)
    return buf.value.decode()


def ref_csv_header() -> str:
    return rlib.ref_csv_header().decode()


_REF_METHOD = {"fmm": 0, "fsm": 1, "lsm": 2, "hcm": 3, "fhcm": 4, "fmsm": 5}


def ref_solve(p: Problem, method: str, cells_x: int = 0, cells_y: int = 0) -> Result:
    """The UNMODIFIED reference (oracle/_ref) with an on-demand SpeedFn."""
    if rlib is None:
        raise RuntimeError("oracle/_ref/libeikref.so not built")
    if not isinstance(p.speed, SpeedField):
        raise TypeError("ref_solve needs a native SpeedField")
    g = p.grid.c()
    en = np.ascontiguousarray(p.exit_nodes, dtype=np.int64)
    ec = np.ascontiguousarray(p.exit_cost, dtype=np.float64)
    pts = np.ascontiguousarray(p.exit_points, dtype=np.float64).reshape(-1)
    pc = np.ascontiguousarray(p.exit_point_cost, dtype=np.float64)
    u = np.empty(p.grid.size(), dtype=np.float64)
    st = ref_stats()
    rc = rlib.ref_solve(_REF_METHOD[method], C.byref(g), C.byref(p.speed.cfield),
                        en.ctypes.data_as(_i64p), ec.ctypes.data_as(_dp), len(en),
                        pts.ctypes.data_as(_dp) if pts.size else _dp(),
                        pc.ctypes.data_as(_dp) if pc.size else _dp(), len(pc),
                        cells_x, cells_y, u.ctypes.data_as(_dp), C.byref(st))
    if rc == 1:
        raise N.ConfigError(rlib.ref_last_error().decode())
    if rc == 3:
        raise N.BudgetError(rlib.ref_last_error().decode())
    if rc:
        raise ValueError(rlib.ref_last_error().decode())
    return Result(u, st.sweeps, st.node_updates, st.heap_removals, st.mon_checks,
                  st.mon_single, st.elapsed_ms)


def ref_metrics(p: Problem, u_method: np.ndarray, u_exact: np.ndarray, refine: int = 4):
    """(l_inf, l_1, R, rho, R_ratio, m_plus, x_plus_empty) of metrics.cpp against
    refine-x FMM truth."""
    g = p.grid.c()
    en = np.ascontiguousarray(p.exit_nodes, dtype=np.int64)
    ec = np.ascontiguousarray(p.exit_cost, dtype=np.float64)
    out = np.zeros(7)
    um = np.ascontiguousarray(u_method, dtype=np.float64)
    ue = np.ascontiguousarray(u_exact, dtype=np.float64)
    rc = rlib.ref_metrics(C.byref(g), C.byref(p.speed.cfield), en.ctypes.data_as(_i64p),
                          ec.ctypes.data_as(_dp), len(en), refine, um.ctypes.data_as(_dp),
                          ue.ctypes.data_as(_dp), out.ctypes.data_as(_dp))
    if rc:
        raise ValueError(rlib.ref_last_error().decode())
    return tuple(out)
