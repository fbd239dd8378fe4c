"""B200-native hot path of the two-scale Eikonal solvers (arXiv 1110.6220).

Python mirror of the reference solver interface
(/root/reference/proj/include/eikonal/*.hpp) over the C-ABI in
include/eikonal_b200.h.  The solves run in hand-written sm_100a kernels
(paper_1110_6220_b200/csrc/); there is no CPU fallback.
"""
# Concurrent solves (run_batch / solve_batch) run best with one hardware
# work queue per stream: export CUDA_DEVICE_MAX_CONNECTIONS=32 before anything
# in the process creates the CUDA context (bench.py does).  Neither the
# package nor the library changes the process environment.

from ._native import BudgetError, ConfigError, LIB_PATH, lib
from .problem import (CellDecomposition, CellTables, ExitSpec, Grid, Problem, SpeedField,
                      build_cells, build_problem, cell_tables, snap_point_to_node,
                      speed_blocks, speed_checkerboard, speed_comb_maze, speed_constant,
                      speed_nodemask, speed_sinsum, speed_sinusoid)
from .solvers import (FmmOptions, HybridStats, Plan, SolverOutput, fhcm_solve, fmm_solve,
                      fmsm_solve, fsm_solve, hcm_solve, lsm_solve, run_batch, set_hcm_mode, solve,
                      solve_batch, solve_multi)
from .distributed import (FmsmStripSolve, StripSolve, fmsm_schedule, fmsm_solve_strips,
                          fsm_solve_strips, strip_bounds)
from .metrics import MetricsReport, ground_truth, method_metrics, refined_problem
from . import experiment_io


def device_count() -> int:
    return int(lib.eik_device_count())


def set_device(device: int) -> None:
    """Device for this thread's later solves/plans (eik_set_device): the
    library has its own CUDA runtime, so torch.cuda.set_device does not
    reach it."""
    from ._native import raise_for
    raise_for(lib.eik_set_device(int(device)))


__all__ = [
    "BudgetError", "ConfigError", "LIB_PATH", "CellDecomposition", "CellTables", "ExitSpec",
    "Grid", "Problem", "SpeedField", "build_cells", "build_problem", "cell_tables",
    "snap_point_to_node", "speed_blocks", "speed_checkerboard", "speed_comb_maze",
    "speed_constant", "speed_nodemask", "speed_sinsum", "speed_sinusoid", "HybridStats",
    "Plan", "SolverOutput", "FmmOptions", "fhcm_solve", "fmm_solve", "fmsm_solve",
    "fsm_solve", "lsm_solve", "hcm_solve", "set_hcm_mode", "solve", "solve_multi", "run_batch", "solve_batch", "device_count", "set_device", "StripSolve", "fsm_solve_strips", "FmsmStripSolve", "fmsm_solve_strips", "fmsm_schedule",
    "strip_bounds", "MetricsReport", "ground_truth", "method_metrics", "refined_problem",
    "experiment_io",
]
