"""ctypes view of include/babplan_cuda.h (the C-ABI of the sm_100a hot path).

The structs here mirror the header field for field; `load()` opens the
in-tree libbabplan_cuda.so and fails loudly when it is missing -- there is
no CPU fallback behind this module.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BP_LIB_PATH") or os.path.join(_HERE, "_lib", "libbabplan_cuda.so")  # override: dev variants

BP_OK, BP_INVALID_ARGUMENT, BP_LOGIC, BP_RUNTIME, BP_CUDA, BP_NCCL, BP_UNSUPPORTED = range(7)
BP_FEATURE_RELATIVE, BP_FEATURE_ABSOLUTE, BP_FEATURE_NETWORK = 0, 1, 2
BP_VAL_X, BP_VAL_U, BP_VAL_P, BP_VAL_OP0 = 0, 1, 2, 3
(BP_OP_LINEAR, BP_OP_RELU, BP_OP_SUM, BP_OP_SCALAR_AFFINE, BP_OP_SQDIST, BP_OP_HINGE,
 BP_OP_SLICE) = range(7)
BP_STOP_LAST_RELU, BP_STOP_EVERY_STEP_OUTPUT, BP_STOP_CUSTOM = 0, 1, 2
BP_BOUND_FULL_CROWN, BP_BOUND_EMPIRICAL, BP_BOUND_INTERVAL = 0, 1, 2
BP_ALPHA_ADAPTIVE, BP_ALPHA_ZERO, BP_ALPHA_ONE = 0, 1, 2
BP_SEARCH_CEM, BP_SEARCH_MPPI, BP_SEARCH_GD = 0, 1, 2
BP_SPLIT_SAMPLES, BP_SPLIT_WIDTH = 0, 1

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_fp = C.POINTER(C.c_float)


class CostOp(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("src0", C.c_int), ("src1", C.c_int), ("dim", C.c_int),
        ("in_dim", C.c_int), ("begin", C.c_int), ("W", _dp), ("b", _dp),
        ("scale", C.c_double), ("offset", C.c_double), ("target", _dp), ("weight", _dp),
        ("weight_by_step", C.c_int), ("center", _dp), ("radius", C.c_double),
        ("penalty", C.c_double), ("is_term", C.c_int),
    ]


class ObjectiveDesc(C.Structure):
    _fields_ = [
        ("ks", C.c_int), ("ka", C.c_int), ("kd", C.c_int), ("horizon", C.c_int),
        ("feature_mode", C.c_int), ("n_layers", C.c_int), ("widths", _ip),
        ("W", C.POINTER(_dp)), ("b", C.POINTER(_dp)), ("relu_after", _ip),
        ("x0", _dp), ("p0", _dp), ("u_lower", _dp), ("u_upper", _dp), ("step_weight", _dp),
        ("n_ops", C.c_int), ("ops", C.POINTER(CostOp)), ("stop_rule", C.c_int),
        ("n_custom_stops", C.c_int), ("custom_stop_steps", _ip),
    ]


class SearchConfig(C.Structure):
    _fields_ = [
        ("method", C.c_int), ("samples_per_iter", C.c_int), ("iterations", C.c_int),
        ("top_capacity", C.c_int), ("seed", C.c_uint64), ("cem_agents", C.c_int),
        ("cem_elites", C.c_int), ("cem_jitter", C.c_double), ("cem_init_sigma", C.c_double),
        ("mppi_noise_frac", C.c_double), ("mppi_temperature", C.c_double),
        ("mppi_n_noise", C.c_int), ("mppi_n_temp", C.c_int), ("mppi_noise_ratios", _dp),
        ("mppi_temperature_ratios", _dp), ("gd_base_step", C.c_double),
        ("gd_n_ratios", C.c_int), ("gd_step_ratios", _dp),
    ]


class PlannerConfig(C.Structure):
    _fields_ = [
        ("batch", C.c_int), ("eta", C.c_double), ("temperature", C.c_double),
        ("top_percent", C.c_double), ("min_width", C.c_double), ("bound_mode", C.c_int),
        ("alpha", C.c_int), ("split_rule", C.c_int), ("seed", C.c_uint64),
        ("search", SearchConfig), ("max_iterations", C.c_int), ("wall_clock_ms", C.c_double),
        ("target_objective", C.c_double),
    ]


class TraceRow(C.Structure):
    _fields_ = [
        ("iter", C.c_int), ("uf", C.c_double), ("min_lf", C.c_double),
        ("pruned_vol", C.c_double), ("selected_vol", C.c_double), ("pool_size", C.c_int64),
        ("samples", C.c_int64), ("wall_ms", C.c_double),
    ]


EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
ALLTOALL_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p, C.POINTER(C.c_int64))


class PoolMeta(C.Structure):
    _fields_ = [("lf", C.c_double), ("uf", C.c_double), ("id", C.c_int64), ("log_vol", C.c_double)]


# Every symbol the header declares (tests check the library exports them all).
EXPORTS = [
    "bp_init", "bp_destroy", "bp_get_last_error", "bp_set_exchange", "bp_set_alltoall", "bp_nccl_unique_id", "bp_set_nccl", "bp_nccl_selftest", "bp_set_stream", "bp_set_rollout_path", "bp_rollout_info", "bp_io_bytes", "bp_node_bounds", "bp_gradient",
    "bp_load_objective", "bp_load_synthetic",
    "bp_stat_layout", "bp_rollout", "bp_batch_search", "bp_search_update", "bp_search_counters", "bp_set_plan_log", "bp_plan_log_size", "bp_plan_log_get", "bp_report_summary", "bp_report_top",
    "bp_report_stats", "bp_batch_bound", "bp_bound_boxes", "bp_plan", "bp_planner_create", "bp_planner_step",
    "bp_planner_finish", "bp_planner_destroy", "bp_result_summary", "bp_result_best",
    "bp_result_trace", "bp_result_free", "bp_timing", "bp_rng_new", "bp_rng_free",
    "bp_rng_uniform", "bp_rng_normal", "bp_rng_bits", "bp_rng_fill", "bp_mix_seed", "bp_pick_out",
    "bp_pool_split", "bp_pool_merge", "bp_generate_model", "bp_measure_fp32_peak", "bp_measure_tf32_peak",
]

_lib = None
_lock = threading.Lock()


class BabplanError(RuntimeError):
    pass


def load() -> C.CDLL:
    """Opens the in-tree CUDA library (raises if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise BabplanError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback for the hot path)")
        lib = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        sig = {
            "bp_init": (C.c_int, [C.c_int, C.POINTER(vp)]),
            "bp_destroy": (C.c_int, [vp]),
            "bp_get_last_error": (C.c_size_t, [C.c_char_p, C.c_size_t]),
            "bp_set_exchange": (C.c_int, [vp, C.c_int, C.c_int, EXCHANGE_FN, vp]),
            "bp_set_alltoall": (C.c_int, [vp, ALLTOALL_FN]),
            "bp_nccl_unique_id": (C.c_int, [C.c_char_p]),
            "bp_set_nccl": (C.c_int, [vp, C.c_int, C.c_int, C.c_char_p]),
            "bp_nccl_selftest": (C.c_int, [vp, C.c_int64, C.POINTER(C.c_int)]),
            "bp_set_stream": (C.c_int, [vp, vp]),
            "bp_set_rollout_path": (C.c_int, [vp, C.c_int, _ip]),
            "bp_rollout_info": (C.c_int, [vp, _ip, _ip, _ip, C.POINTER(C.c_int64)]),
            "bp_node_bounds": (C.c_int, [vp, _dp, _dp]),
            "bp_gradient": (C.c_int, [vp, C.c_int64, _fp, _fp]),
            "bp_io_bytes": (C.c_int, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "bp_load_objective": (C.c_int, [vp, C.POINTER(ObjectiveDesc)]),
            "bp_load_synthetic": (C.c_int, [vp, C.c_int]),
            "bp_stat_layout": (C.c_int, [vp, _ip, _ip, _ip, _ip, _ip, _ip, C.c_int]),
            "bp_rollout": (C.c_int, [vp, C.c_int, C.c_int, _fp, _fp, _fp, _fp, _fp, _ip]),
            "bp_batch_search": (C.c_int, [vp, C.c_int, _dp, _dp, _dp, C.POINTER(SearchConfig)]),
            "bp_search_update": (C.c_int, [vp, C.c_int, C.POINTER(SearchConfig), _dp, _dp, C.c_int, _fp, _fp, _fp,
                                           _fp, _fp, _fp, _ip, _fp, _ip, _fp]),
            "bp_report_summary": (C.c_int, [vp, _dp, _dp, C.POINTER(C.c_int64), _ip, _ip]),
            "bp_report_top": (C.c_int, [vp, C.c_int, _dp, _dp, C.c_int]),
            "bp_report_stats": (C.c_int, [vp, C.c_int, _fp, _fp]),
            "bp_batch_bound": (C.c_int, [vp, C.c_int, C.c_int, _dp]),
            "bp_bound_boxes": (C.c_int, [vp, C.c_int, _dp, _dp, C.c_int, C.c_int, _dp]),
            "bp_plan": (C.c_int, [vp, C.POINTER(PlannerConfig), _dp, C.c_int, C.POINTER(vp)]),
            "bp_planner_create": (C.c_int, [vp, C.POINTER(PlannerConfig), _dp, C.POINTER(vp)]),
            "bp_planner_step": (C.c_int, [vp, _ip, _ip, _ip]),
            "bp_planner_finish": (C.c_int, [vp, C.POINTER(vp)]),
            "bp_planner_destroy": (C.c_int, [vp]),
            "bp_result_summary": (C.c_int, [vp, _dp, _dp, _ip, C.POINTER(C.c_int64), _ip,
                                            C.c_char_p, C.c_size_t, _ip, _ip]),
            "bp_result_best": (C.c_int, [vp, _dp]),
            "bp_result_trace": (C.c_int, [vp, C.POINTER(TraceRow), C.c_int]),
            "bp_result_free": (C.c_int, [vp]),
            "bp_search_counters": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
            "bp_set_plan_log": (C.c_int, [vp, C.c_int]),
            "bp_plan_log_size": (C.c_int, [vp, _ip, _ip]),
            "bp_plan_log_get": (C.c_int, [vp, _ip, _dp, _dp, _dp, _dp, _dp, _ip, _dp, _dp, C.POINTER(C.c_int64), _ip]),
            "bp_timing": (C.c_int, [vp, _dp, C.POINTER(C.c_int64), _dp, _dp, C.POINTER(C.c_int64)]),
            "bp_rng_new": (C.c_int, [C.c_uint64, C.POINTER(vp)]),
            "bp_rng_free": (C.c_int, [vp]),
            "bp_rng_uniform": (C.c_int, [vp, _dp]),
            "bp_rng_normal": (C.c_int, [vp, _dp]),
            "bp_rng_bits": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
            "bp_rng_fill": (C.c_int, [vp, C.c_int, C.c_int64, _dp]),
            "bp_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "bp_pick_out": (C.c_int, [C.POINTER(PoolMeta), C.c_int, C.c_int, C.c_double,
                                      C.c_double, vp, _ip, _ip]),
            "bp_pool_split": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _ip, _fp, _fp,
                                        C.POINTER(C.c_int64), C.c_double, C.c_double, C.c_int, _ip, _dp, _dp,
                                        _ip, _fp, _fp]),
            "bp_pool_merge": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, _ip, _fp, _fp, _ip, _fp, _fp,
                                        _fp, _fp, _ip, _ip, _fp, _fp, _fp, _ip, _fp]),
            "bp_generate_model": (C.c_int, [C.c_uint64, C.c_int, _ip, _dp]),
            "bp_measure_fp32_peak": (C.c_int, [C.c_int, _dp, _dp]),
            "bp_measure_tf32_peak": (C.c_int, [C.c_int, _dp, _dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


_EXC = {BP_INVALID_ARGUMENT: ValueError, BP_LOGIC: RuntimeError, BP_RUNTIME: RuntimeError,
        BP_CUDA: BabplanError, BP_NCCL: BabplanError, BP_UNSUPPORTED: NotImplementedError}


def check(status: int) -> None:
    """Raises the Python analogue of the reference's exception for a failed call."""
    if status == BP_OK:
        return
    lib = load()
    buf = C.create_string_buffer(1024)
    lib.bp_get_last_error(buf, 1024)
    raise _EXC.get(status, BabplanError)(buf.value.decode(errors="replace"))


def dptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def fptr(a):
    return a.ctypes.data_as(_fp) if a is not None else None


def iptr(a):
    return a.ctypes.data_as(_ip) if a is not None else None
