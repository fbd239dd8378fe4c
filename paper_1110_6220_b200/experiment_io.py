"""Field dumps and experiment rows in the reference's formats (SURVEY.md
section 8(f) row 3): field_io.cpp (dump_field / load_field, raw and ascii)
and experiment.cpp's row (run_row, :198-253) and CSV schema (csv_header /
csv_line, :314-329), so B200 results drop into the reference's tables.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from .metrics import method_metrics
from .problem import Problem, build_cells

METHODS = ("fmm", "fsm", "lsm", "hcm", "fhcm", "fmsm")  # experiment.hpp:11 order
HYBRID = ("hcm", "fhcm", "fmsm")


# ---- field_io.cpp -----------------------------------------------------------

def dump_field(values: np.ndarray, m: int, n: int, h: float, path: str,
               fmt: str = "raw") -> None:
    """field_io.cpp:20-45.  raw: int64 {m, n} then m*n doubles (row j major);
    ascii: "%d %d %.17g" header, then one line per row of "%.17g" values."""
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    if v.size != m * n:
        raise ValueError("dump_field: size mismatch")
    if fmt == "raw":
        with open(path, "wb") as f:
            f.write(np.array([m, n], dtype=np.int64).tobytes())
            f.write(v.tobytes())
    elif fmt == "ascii":
        with open(path, "w") as f:
            f.write("%d %d %.17g\n" % (m, n, h))
            rows = v.reshape(n, m)
            for j in range(n):
                f.write(" ".join("%.17g" % x for x in rows[j]) + "\n")
    else:
        raise ValueError("fmt must be 'raw' or 'ascii'")


def load_field(path: str, fmt: str = "raw") -> Tuple[np.ndarray, int, int, float]:
    """field_io.cpp:47-77: (values m*n, m, n, h); raw dumps carry no h (0)."""
    if fmt == "raw":
        with open(path, "rb") as f:
            head = f.read(16)
            if len(head) < 16:
                raise RuntimeError(f"bad raw header: {path}")
            m, n = (int(x) for x in np.frombuffer(head, dtype=np.int64))
            data = f.read(8 * m * n)
            if len(data) < 8 * m * n:
                raise RuntimeError(f"truncated raw dump: {path}")
            return np.frombuffer(data, dtype=np.float64).copy(), m, n, 0.0
    if fmt == "ascii":
        with open(path) as f:
            toks = f.read().split()
        if len(toks) < 3:
            raise RuntimeError(f"bad ascii header: {path}")
        m, n, h = int(toks[0]), int(toks[1]), float(toks[2])
        if len(toks) < 3 + m * n:
            raise RuntimeError(f"truncated ascii dump: {path}")
        return np.array([float(t) for t in toks[3:3 + m * n]]), m, n, h  # strtod: "inf"
    raise ValueError("fmt must be 'raw' or 'ascii'")


# ---- experiment.cpp ---------------------------------------------------------

@dataclass
class ExperimentRow:
    """experiment.hpp:39-49."""
    problem: str
    method: str
    grid_m: int
    cells_x: int = 0
    elapsed_ms: float = 0.0
    l_inf: float = 0.0
    l_1: float = 0.0
    max_ratio: float = 1.0
    rho: float = 1.0
    ratio_of_max: float = 1.0
    avhr: float = 0.0
    avs: float = 0.0
    mon_pct: float = 0.0
    sweeps: int = 0
    node_updates: int = 0
    heap_removals: int = 0


def csv_header() -> str:
    """experiment.cpp:314-317."""
    return ("problem,method,grid_m,cells_x,elapsed_ms,l_inf,l_1,R_max_ratio,"
            "rho,R_ratio,avhr,avs,mon_pct,sweeps,node_updates,heap_removals")


def csv_line(r: ExperimentRow) -> str:
    """experiment.cpp:319-329 (C printf formats)."""
    return ("%s,%s,%d,%d,%.3f,%.6e,%.6e,%.6f,%.6f,%.6f,%.4f,%.4f,%.2f,%d,%d,%d" % (
        r.problem, r.method, r.grid_m, r.cells_x, r.elapsed_ms, r.l_inf, r.l_1, r.max_ratio,
        r.rho, r.ratio_of_max, r.avhr, r.avs, r.mon_pct, r.sweeps, r.node_updates,
        r.heap_removals))


def run_row(problem_name: str, problem: Problem, method: str, cells: int,
            exact: np.ndarray, truth: np.ndarray, repeat: int = 1,
            dump_dir: Optional[str] = None) -> ExperimentRow:
    """experiment.cpp:198-253 over the device solvers: best-of-`repeat` wall
    time of the solve, counters, and the metrics against `exact` (the FMM
    field on the same grid) and `truth` (ground_truth) -- exact methods keep
    the ratio columns at 1."""
    from .solvers import solve
    if method not in METHODS:
        raise ValueError(f"unknown method {method}")
    decomp = build_cells(problem.grid, cells, cells) if method in HYBRID else None
    best, out = math.inf, None
    for _ in range(max(1, repeat)):
        t0 = time.perf_counter()
        out = solve(problem, method, decomp)
        best = min(best, (time.perf_counter() - t0) * 1e3)
    row = ExperimentRow(problem_name, method, problem.grid.m, cells if decomp else 0, best)
    row.sweeps, row.node_updates, row.heap_removals = out.sweeps, out.node_updates, \
        out.heap_removals
    row.avhr, row.avs, row.mon_pct = out.hybrid.avhr, out.hybrid.avs, out.hybrid.mon_pct
    if method in HYBRID:
        rep = method_metrics(out.values, exact, truth, problem.exit_nodes)
        row.max_ratio, row.rho, row.ratio_of_max = rep.max_error_ratio, rep.avg_error_ratio, \
            rep.ratio_of_max
    else:
        rep = method_metrics(out.values, out.values, truth, problem.exit_nodes)
    row.l_inf, row.l_1 = rep.l_inf, rep.l_1
    if dump_dir:
        name = f"{problem_name}_{method}_m{problem.grid.m}" + (f"_c{cells}" if decomp else "")
        dump_field(out.values, problem.grid.m, problem.grid.n, problem.grid.h,
                   f"{dump_dir}/{name}.txt", "ascii")
    return row
