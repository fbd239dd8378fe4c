"""ctypes binding of the C-ABI in include/eikonal_b200.h.

The product path has no CPU fallback: if libeikonal_b200.so is missing the
import fails loudly, and on a host without a CUDA device every solve returns
EIK_ERR_CUDA (raised as RuntimeError).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libeikonal_b200.so")

EIK_FMM, EIK_FSM, EIK_LSM, EIK_HCM, EIK_FHCM, EIK_FMSM, EIK_HCM_EXACT = range(7)
# "hcm" runs the band scheduler (default, eik_set_hcm_mode); "hcm_exact" the
# exact replay of hcm_solve's heap order (bit-identical field and counters)
METHOD_NAMES = {"fmm": EIK_FMM, "fsm": EIK_FSM, "lsm": EIK_LSM, "hcm": EIK_HCM,
                "fhcm": EIK_FHCM, "fmsm": EIK_FMSM, "hcm_exact": EIK_HCM_EXACT}

EIK_OK, EIK_ERR_CONFIG, EIK_ERR_CUDA, EIK_ERR_BUDGET, EIK_ERR_NOT_IMPL, EIK_ERR_DOMAIN = range(6)

EIK_FIELD_CONSTANT, EIK_FIELD_SINUSOID, EIK_FIELD_CHECKER, EIK_FIELD_COMB, \
    EIK_FIELD_BLOCKS, EIK_FIELD_NODEMASK, EIK_FIELD_SINSUM = range(7)

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class eik_grid(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("h", C.c_double),
                ("x0", C.c_double), ("y0", C.c_double)]


class eik_problem(C.Structure):
    _fields_ = [("grid", eik_grid), ("speed", _dp), ("speed_on_device", C.c_int32),
                ("exit_nodes", _i64p), ("exit_cost", _dp), ("n_exit", C.c_int64),
                ("exit_points_xy", _dp), ("exit_point_cost", _dp),
                ("n_exit_points", C.c_int64)]


class eik_cells(C.Structure):
    _fields_ = [("cells_x", C.c_int32), ("cells_y", C.c_int32),
                ("probe_speed_w", _dp), ("probe_speed_e", _dp),
                ("probe_speed_s", _dp), ("probe_speed_n", _dp),
                ("center_speed", _dp)]


class eik_output(C.Structure):
    _fields_ = [("u", _dp), ("u_on_device", C.c_int32),
                ("sweeps", C.c_int64), ("node_updates", C.c_int64),
                ("heap_removals", C.c_int64), ("cell_removals", C.c_int64),
                ("cell_sweeps", C.c_int64), ("mon_checks", C.c_int64),
                ("mon_single", C.c_int64), ("avhr", C.c_double), ("avs", C.c_double),
                ("mon_pct", C.c_double), ("device_ms", C.c_double), ("host_ms", C.c_double),
                ("kernel_launches", C.c_int64), ("spec_hits", C.c_int64),
                ("spec_waits", C.c_int64), ("spec_self", C.c_int64), ("grid_ctas", C.c_int64),
                ("rounds", C.c_int64)]


class eik_field(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value", C.c_double),
                ("amp", C.c_double), ("freq", C.c_int32),
                ("checkers", C.c_int32), ("slow", C.c_double), ("fast", C.c_double),
                ("n_barriers", C.c_int32), ("barrier_speed", C.c_double),
                ("barrier_width", C.c_double), ("gap_fraction", C.c_double),
                ("nb", C.c_int32), ("bx0", C.c_double), ("by0", C.c_double),
                ("bscale", C.c_double), ("block_speed", _dp),
                ("mask_grid", eik_grid), ("mask", C.POINTER(C.c_uint8)),
                ("K", C.c_int32), ("kp", _dp), ("kq", _dp), ("kphi", _dp)]


class eik_metrics_out(C.Structure):
    _fields_ = [("l_inf", C.c_double), ("l_1", C.c_double), ("max_error_ratio", C.c_double),
                ("avg_error_ratio", C.c_double), ("ratio_of_max", C.c_double),
                ("m_plus", C.c_int64), ("x_plus_empty", C.c_int32)]


EXPORTS = {
    # name: (restype, argtypes)
    "eik_solve": (C.c_int, [C.POINTER(eik_problem), C.POINTER(eik_cells), C.c_int32,
                            C.POINTER(eik_output)]),
    "eik_plan_create": (C.c_void_p, [C.POINTER(eik_problem), C.POINTER(eik_cells), C.c_int32]),
    "eik_plan_run": (C.c_int, [C.c_void_p, C.POINTER(eik_output)]),
    "eik_plan_values": (C.c_void_p, [C.c_void_p]),
    "eik_plan_pitch": (C.c_int64, [C.c_void_p]),
    "eik_plan_destroy": (None, [C.c_void_p]),
    "eik_plan_prepare": (C.c_int, [C.c_void_p]),
    "eik_plan_acceptance_order": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32]),
    "eik_plan_sweep": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_int32)]),
    "eik_plan_get_rows": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int32]),
    "eik_plan_set_rows": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int32]),
    "eik_plan_sweep_async": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    "eik_plan_rows_async": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int32,
                                      C.c_void_p]),
    "eik_plan_set_ctas": (C.c_int, [C.c_void_p, C.c_int32]),
    "eik_fmsm_schedule": (C.c_int, [C.POINTER(eik_problem), C.POINTER(eik_cells), C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "eik_plan_create_fmsm_strip": (C.c_void_p, [C.POINTER(eik_problem), C.c_int32, C.c_int32,
                                                C.c_int64, C.c_int64, C.c_int64]),
    "eik_plan_fmsm_levels": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "eik_plan_fmsm_level_async": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "eik_plan_fmsm_counters": (C.c_int, [C.c_void_p, C.c_void_p]),
    "eik_set_hcm_mode": (C.c_int, [C.c_int32]),
    "eik_plan_set_hcm_mode": (C.c_int, [C.c_void_p, C.c_int32]),
    "eik_plan_set_partitions": (C.c_int, [C.c_void_p, C.c_int32]),
    "eik_plan_capacity": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "eik_plan_run_batch": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(eik_output),
                                     C.POINTER(C.c_double)]),
    "eik_solve_multi": (C.c_int, [C.POINTER(eik_problem), C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                  C.POINTER(eik_output)]),
    "eik_field_sample_rows": (C.c_int, [C.POINTER(eik_field), C.POINTER(eik_grid), C.c_int64,
                                        C.c_int64, _dp, C.c_int32]),
    "eik_solve_batch": (C.c_int, [C.POINTER(C.POINTER(eik_problem)), C.POINTER(C.POINTER(eik_cells)),
                                  C.POINTER(C.c_int32), C.c_int32, C.POINTER(eik_output),
                                  C.POINTER(C.c_double)]),
    "eik_last_error": (C.c_char_p, []),
    "eik_last_status": (C.c_int, []),
    "eik_abi_version": (C.c_int, []),
    "eik_debug_reload_knobs": (None, []),
    "eik_device_count": (C.c_int, []),
    "eik_set_device": (C.c_int, [C.c_int32]),
    "eik_release_cached": (None, []),
    "eik_metrics": (C.c_int, [_dp, _dp, _dp, C.c_int64, C.c_int64, _i64p, C.c_int64, C.c_int32,
                              C.POINTER(eik_metrics_out)]),
    "eik_cell_probe_points": (C.c_int64, [C.POINTER(eik_grid), C.c_int32, C.c_int32,
                                          C.c_int32, _dp]),
    "eik_cell_centers": (C.c_int64, [C.POINTER(eik_grid), C.c_int32, C.c_int32, _dp]),
    "eik_field_eval": (C.c_double, [C.POINTER(eik_field), C.c_double, C.c_double]),
    "eik_field_sample": (C.c_int, [C.POINTER(eik_field), C.POINTER(eik_grid), _dp, C.c_int32]),
    "eik_field_eval_points": (C.c_int, [C.POINTER(eik_field), _dp, C.c_int64, _dp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the Eikonal hot path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def dptr(arr):
    """double* of a C-contiguous float64 numpy array (or NULL for None)."""
    if arr is None:
        return _dp()
    return arr.ctypes.data_as(_dp)


def i64ptr(arr):
    if arr is None:
        return _i64p()
    return arr.ctypes.data_as(_i64p)


class ConfigError(RuntimeError):
    """Mirror of eikonal::ConfigError (grid.hpp:16-19)."""


class BudgetError(RuntimeError):
    """Mirror of std::runtime_error("heap-cell removal budget exceeded")."""


def raise_for(code: int, what: str = ""):
    if code == EIK_OK:
        return
    msg = lib.eik_last_error().decode() or what
    if code == EIK_ERR_CONFIG:
        raise ConfigError(msg)
    if code == EIK_ERR_BUDGET:
        raise BudgetError(msg)
    if code == EIK_ERR_DOMAIN:
        raise ValueError(msg)
    if code == EIK_ERR_NOT_IMPL:
        raise NotImplementedError(msg)
    raise RuntimeError(f"CUDA: {msg}")
