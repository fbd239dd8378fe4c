"""Ground truth and error metrics on the device:
the reference's metrics.cpp -- ground_truth (:77-99), error_fields (:11-32),
error_ratios (:34-69), method_metrics (:71-75).

ground_truth solves the refined problem with this package's FMM row (the
exact discrete fixed point on the device; it agrees with the reference's FMM
to ~1e-15, acceptance.cpp C1) and subsamples it; method_metrics reduces the
error fields in one device pass (eik_metrics).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .problem import Grid, Problem


@dataclass
class MetricsReport:
    """metrics.hpp MetricsReport."""
    l_inf: float
    l_1: float
    max_error_ratio: float
    avg_error_ratio: float
    ratio_of_max: float
    m_plus: int
    x_plus_empty: bool


def method_metrics(u_method, u_exact, u_truth, exit_nodes) -> MetricsReport:
    """error_ratios(error_fields(...)) on the device.  Fields: m*n arrays
    (numpy on the host; torch CUDA tensors stay on the device)."""
    def ptr(a):
        if isinstance(a, np.ndarray):
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError("fields must be C-contiguous float64")
            return a.ctypes.data_as(C.POINTER(C.c_double)), 0, a.size
        return C.cast(C.c_void_p(a.data_ptr()), C.POINTER(C.c_double)), 1, a.numel()
    pm, dm, M = ptr(u_method)
    pe, de, Me = ptr(u_exact)
    pt, dt, Mt = ptr(u_truth)
    if not (M == Me == Mt) or not (dm == de == dt):
        raise ValueError("error_fields: shape mismatch")  # metrics.cpp:15-18
    ex = np.ascontiguousarray(exit_nodes, dtype=np.int64)
    out = N.eik_metrics_out()
    N.raise_for(N.lib.eik_metrics(pm, pe, pt, M, 1, ex.ctypes.data_as(C.POINTER(C.c_int64)),
                                  len(ex), dm, C.byref(out)))
    return MetricsReport(out.l_inf, out.l_1, out.max_error_ratio, out.avg_error_ratio,
                         out.ratio_of_max, int(out.m_plus), bool(out.x_plus_empty))


def refined_problem(problem: Problem, refine: int) -> Problem:
    """metrics.cpp:80-93: the grid refined `refine` times, exits mapped to
    (refine*i, refine*j) with their costs (the index map is monotone)."""
    if refine < 1:
        raise ValueError("refine must be >= 1")
    g = problem.grid
    fine = Grid(refine * (g.m - 1) + 1, refine * (g.n - 1) + 1, g.h / refine, g.x0, g.y0)
    ex = np.asarray(problem.exit_nodes, dtype=np.int64)
    i, j = ex % g.m, ex // g.m
    nodes = (refine * j) * fine.m + refine * i
    return Problem(fine, problem.speed, nodes, np.asarray(problem.exit_cost, dtype=np.float64))


def ground_truth(problem: Problem, refine: int = 4) -> np.ndarray:
    """metrics.cpp:77-99: the refined solve subsampled at the coarse nodes."""
    from .solvers import fmm_solve
    g = problem.grid
    fp = refined_problem(problem, refine)
    u = fmm_solve(fp).values.reshape(fp.grid.n, fp.grid.m)
    return np.ascontiguousarray(u[::refine, ::refine][: g.n, : g.m]).reshape(-1)
