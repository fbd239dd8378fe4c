"""Solver entry points mirroring the reference's L2 API.

    fmm_solve(problem, opts)      classic_solvers.hpp:18
    fsm_solve(problem)            classic_solvers.hpp:33
    lsm_solve(problem)            classic_solvers.hpp:38
    hcm_solve(problem, cells)     heap_cell.hpp:36
    fhcm_solve(problem, cells)    heap_cell.hpp:41
    fmsm_solve(problem, cells)    fmsm.hpp:36

Every call crosses the C-ABI (include/eikonal_b200.h) into the sm_100a
kernels; there is no CPU solver behind these names.  Errors map to the
reference's exception types (ConfigError, BudgetError ~ runtime_error,
ValueError ~ domain_error).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N
from .problem import CellDecomposition, CellTables, Problem, cell_tables


@dataclass
class HybridStats:
    """grid.hpp:132-140."""
    avhr: float = 0.0
    avs: float = 0.0
    mon_pct: float = 0.0
    cell_removals: int = 0
    cell_sweeps: int = 0
    mon_checks: int = 0
    mon_single: int = 0


@dataclass
class SolverOutput:
    """grid.hpp:142-149; `values` is the m*n row-major field (index j*m+i)."""
    values: np.ndarray
    m: int
    n: int
    sweeps: int = 0
    node_updates: int = 0
    heap_removals: int = 0
    hybrid: HybridStats = field(default_factory=HybridStats)
    device_ms: float = 0.0
    host_ms: float = 0.0
    kernel_launches: int = 0
    spec: tuple = (0, 0, 0)  # heap-cell replay: (hits, waits, self-processed)
    rounds: int = 0          # HCM band scheduler: rounds
    ctas: int = 0            # CTAs of the persistent solve kernel
    acceptance_order: Optional[np.ndarray] = None  # FMM only, when requested (grid.hpp:148)

    def at(self, i: int, j: int) -> float:
        return float(self.values[j * self.m + i])

    def as_2d(self) -> np.ndarray:
        return self.values.reshape(self.n, self.m)


def _c_problem(problem: Problem, F: np.ndarray):
    p = N.eik_problem()
    p.grid = problem.grid.c()
    p.speed = N.dptr(F)
    p.speed_on_device = 0
    en = np.ascontiguousarray(problem.exit_nodes, dtype=np.int64)
    ec = np.ascontiguousarray(problem.exit_cost, dtype=np.float64)
    pts = np.ascontiguousarray(problem.exit_points, dtype=np.float64).reshape(-1)
    pc = np.ascontiguousarray(problem.exit_point_cost, dtype=np.float64)
    p.exit_nodes = N.i64ptr(en)
    p.exit_cost = N.dptr(ec)
    p.n_exit = len(en)
    p.exit_points_xy = N.dptr(pts) if pts.size else N.dptr(None)
    p.exit_point_cost = N.dptr(pc) if pc.size else N.dptr(None)
    p.n_exit_points = len(pc)
    return p, (en, ec, pts, pc, F)


def _c_cells(cells: Optional[CellDecomposition], tabs: Optional[CellTables]):
    if cells is None:
        return None, ()
    c = N.eik_cells()
    c.cells_x = cells.cells_x
    c.cells_y = cells.cells_y
    keep = ()
    if tabs is not None:
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (tabs.probe_w, tabs.probe_e, tabs.probe_s, tabs.probe_n, tabs.center)]
        c.probe_speed_w, c.probe_speed_e, c.probe_speed_s, c.probe_speed_n, c.center_speed = \
            [N.dptr(a) for a in arrs]
        keep = tuple(arrs)
    return c, keep


def _pack(out: N.eik_output, values: np.ndarray, g) -> SolverOutput:
    return SolverOutput(values=values, m=g.m, n=g.n, sweeps=out.sweeps,
                        node_updates=out.node_updates, heap_removals=out.heap_removals,
                        hybrid=HybridStats(out.avhr, out.avs, out.mon_pct, out.cell_removals,
                                           out.cell_sweeps, out.mon_checks, out.mon_single),
                        device_ms=out.device_ms, host_ms=out.host_ms,
                        kernel_launches=out.kernel_launches,
                        spec=(out.spec_hits, out.spec_waits, out.spec_self),
                        ctas=out.grid_ctas, rounds=out.rounds)


def solve(problem: Problem, method: str, cells: Optional[CellDecomposition] = None,
          tables: Optional[CellTables] = None, out: Optional[np.ndarray] = None) -> SolverOutput:
    """One solve through eik_solve (host buffers in, host values out).
    `out` may be a caller-owned (e.g. pinned) float64 buffer of m*n values."""
    code = N.METHOD_NAMES[method]
    F = problem.sampled_speed()
    p, keep_p = _c_problem(problem, F)
    if cells is not None and tables is None:
        tables = cell_tables(problem, cells)
    c, keep_c = _c_cells(cells, tables)
    u = out if out is not None else np.empty(problem.grid.size(), dtype=np.float64)
    res = N.eik_output()
    res.u = N.dptr(u)
    res.u_on_device = 0
    rc = N.lib.eik_solve(C.byref(p), C.byref(c) if c is not None else None, code, C.byref(res))
    N.raise_for(rc)
    return _pack(res, u, problem.grid)


@dataclass
class FmmOptions:
    """classic_solvers.hpp:10-13."""
    record_acceptance_order: bool = False


def fmm_solve(problem: Problem, opts: Optional[FmmOptions] = None) -> SolverOutput:
    if opts is None or not opts.record_acceptance_order:
        return solve(problem, "fmm")
    plan = Plan(problem, "fmm")
    try:
        out = plan.run(np.empty(problem.grid.size(), dtype=np.float64))
        order = np.empty(problem.grid.size() - len(problem.exit_nodes), dtype=np.int32)
        N.raise_for(N.lib.eik_plan_acceptance_order(
            plan._h, order.ctypes.data_as(C.POINTER(C.c_int32)), 0))
        out.acceptance_order = order
    finally:
        plan.close()
    return out


def fsm_solve(problem: Problem) -> SolverOutput:
    return solve(problem, "fsm")


def lsm_solve(problem: Problem) -> SolverOutput:
    return solve(problem, "lsm")


def hcm_solve(problem: Problem, cells: CellDecomposition) -> SolverOutput:
    return solve(problem, "hcm", cells)


def set_hcm_mode(mode: str) -> None:
    """Default HCM ordering for later solves/plans: "band" (the band
    scheduler, default) or "exact" (the exact replay; also method "hcm_exact")."""
    N.raise_for(N.lib.eik_set_hcm_mode({"band": 0, "exact": 1}[mode]))


def fhcm_solve(problem: Problem, cells: CellDecomposition) -> SolverOutput:
    return solve(problem, "fhcm", cells)


def fmsm_solve(problem: Problem, cells: CellDecomposition) -> SolverOutput:
    return solve(problem, "fmsm", cells)


def solve_multi(problem: Problem, method: str = "fsm", devices=None) -> SolverOutput:
    """fsm_solve / the FMM row over several GPUs of this process
    (eik_solve_multi): row strips, one per device, strip-Jacobi rounds with
    the edge rows exchanged by peer copies.  `devices` lists CUDA ordinals (a
    device may appear more than once: its strips then share it)."""
    devs = list(devices) if devices is not None else [0]
    F = problem.sampled_speed()
    p, keep_p = _c_problem(problem, F)
    u = np.empty(problem.grid.size(), dtype=np.float64)
    res = N.eik_output()
    res.u = N.dptr(u)
    res.u_on_device = 0
    dv = (C.c_int32 * len(devs))(*devs)
    N.raise_for(N.lib.eik_solve_multi(C.byref(p), N.METHOD_NAMES[method], dv, len(devs),
                                      C.byref(res)))
    return _pack(res, u, problem.grid)


class Plan:
    """Resident solve (eik_plan_*): inputs uploaded once, values stay in HBM."""

    def __init__(self, problem: Problem, method: str,
                 cells: Optional[CellDecomposition] = None,
                 tables: Optional[CellTables] = None):
        self.problem = problem
        self.method = method
        F = problem.sampled_speed()
        p, keep_p = _c_problem(problem, F)
        if cells is not None and tables is None:
            tables = cell_tables(problem, cells)
        c, keep_c = _c_cells(cells, tables)
        self._h = N.lib.eik_plan_create(C.byref(p), C.byref(c) if c is not None else None,
                                        N.METHOD_NAMES[method])
        if not self._h:
            N.raise_for(N.lib.eik_last_status() or N.EIK_ERR_CUDA)

    def run(self, u_host: Optional[np.ndarray] = None, u_device_ptr: int = 0) -> SolverOutput:
        out = N.eik_output()
        if u_host is not None:
            out.u = N.dptr(u_host)
            out.u_on_device = 0
        elif u_device_ptr:
            out.u = C.cast(C.c_void_p(u_device_ptr), C.POINTER(C.c_double))
            out.u_on_device = 1
        else:
            out.u = N.dptr(None)
        N.raise_for(N.lib.eik_plan_run(self._h, C.byref(out)))
        return _pack(out, u_host, self.problem.grid)

    def set_ctas(self, max_ctas: int) -> None:
        """Cap the CTAs of this plan's persistent kernel (0 = whole device)."""
        N.raise_for(N.lib.eik_plan_set_ctas(self._h, int(max_ctas)))

    def set_partitions(self, part_rows: int) -> None:
        """FSM/FMM plans: strip-Jacobi parts of `part_rows` rows (multiple of
        32) swept side by side on the device; 0 = one exact Gauss-Seidel
        wavefront (the default, fsm_solve's order bit for bit)."""
        N.raise_for(N.lib.eik_plan_set_partitions(self._h, int(part_rows)))

    def capacity(self):
        """(CTAs of the persistent kernel the device holds, fixed grid or 0)."""
        d, f = C.c_int32(), C.c_int32()
        N.raise_for(N.lib.eik_plan_capacity(self._h, C.byref(d), C.byref(f)))
        return d.value, f.value

    def values_ptr(self) -> int:
        return N.lib.eik_plan_values(self._h)

    def sweep(self, first_sweep: int, count: int = 1):
        """FSM/FMM plans: exactly `count` more sweeps on the current values
        (eik_plan_sweep); per-sweep "changed" flags."""
        ch = (C.c_int32 * count)()
        N.raise_for(N.lib.eik_plan_sweep(self._h, first_sweep, count, ch))
        return [bool(x) for x in ch]

    def close(self):
        lib = getattr(N, "lib", None)  # None during interpreter shutdown
        if getattr(self, "_h", None) and lib is not None:
            lib.eik_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def run_batch(plans, u_hosts=None):
    """Run distinct plans concurrently on their device (eik_plan_run_batch):
    the device-side counterpart of the reference's --jobs thread pool
    (experiment.cpp:284-310).  Returns (outputs, batch device ms)."""
    n = len(plans)
    outs = (N.eik_output * n)()
    for k in range(n):
        outs[k].u = N.dptr(u_hosts[k] if u_hosts is not None else None)
        outs[k].u_on_device = 0
    hs = (C.c_void_p * n)(*[p._h for p in plans])
    ms = C.c_double()
    N.raise_for(N.lib.eik_plan_run_batch(hs, n, outs, C.byref(ms)))
    return [_pack(outs[k], u_hosts[k] if u_hosts is not None else None, plans[k].problem.grid)
            for k in range(n)], ms.value


def solve_batch(jobs, outs=None):
    """Several solve() calls at once (eik_solve_batch): jobs are
    (problem, method, cells, tables) tuples (cells/tables None for FMM/FSM);
    `outs` optional caller-owned float64 buffers.  Returns (outputs, batch
    device ms)."""
    n = len(jobs)
    keep, pp, cc, us = [], (C.POINTER(N.eik_problem) * n)(), (C.POINTER(N.eik_cells) * n)(), []
    meth = (C.c_int32 * n)()
    res = (N.eik_output * n)()
    for k, (problem, method, cells, tables) in enumerate(jobs):
        F = problem.sampled_speed()
        p, kp = _c_problem(problem, F)
        if cells is not None and tables is None:
            tables = cell_tables(problem, cells)
        c, kc = _c_cells(cells, tables)
        keep += [p, kp, c, kc]
        pp[k] = C.pointer(p)
        cc[k] = C.pointer(c) if c is not None else C.POINTER(N.eik_cells)()
        meth[k] = N.METHOD_NAMES[method]
        u = outs[k] if outs is not None else np.empty(problem.grid.size(), dtype=np.float64)
        us.append(u)
        res[k].u = N.dptr(u)
        res[k].u_on_device = 0
    ms = C.c_double()
    N.raise_for(N.lib.eik_solve_batch(pp, cc, meth, n, res, C.byref(ms)))
    return [_pack(res[k], us[k], jobs[k][0].grid) for k in range(n)], ms.value
