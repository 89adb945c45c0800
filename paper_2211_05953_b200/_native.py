"""ctypes binding of libbfpp.so (the C ABI in include/bfpp.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2211_05953_b200/csrc``). There is no Python fallback: if the
library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BFPP_LIB_PATH", os.path.join(_HERE, "libbfpp.so"))  # override: A/B runs


class ModelSpecC(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("n_layers", "s_hidden", "n_heads", "s_head", "s_mlp", "s_seq", "s_voc")]


class ParallelConfigC(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_dp", "n_tp", "n_pp", "n_mb", "s_mb", "n_loop")] + \
               [("dp_variant", C.c_int32), ("schedule", C.c_int32)]


class ClusterSpecC(C.Structure):
    _fields_ = [("n_node", C.c_int64), ("s_node", C.c_int64)] + \
               [(n, C.c_double) for n in ("peak_flops", "bw_intra", "bw_inter", "pp_latency",
                                          "mem_capacity", "kernel_efficiency")]


class TimingModelC(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("t_fwd_stage", "bwd_ratio", "t_pp_transfer", "pp_latency",
                                          "t_dp_reduce_stage", "t_dp_reconstruct_stage")]


class TaskC(C.Structure):
    _fields_ = [("id", C.c_int32), ("lane", C.c_int32), ("kind", C.c_int32), ("priority", C.c_int32),
                ("device", C.c_int64), ("peer_device", C.c_int64), ("micro_batch", C.c_int64),
                ("stage", C.c_int64)]


class MeasuredRatesC(C.Structure):
    _fields_ = [("fwd_layer_seq", C.c_double), ("bwd_ratio", C.c_double), ("pp_s_per_byte", C.c_double),
                ("pp_latency", C.c_double), ("reduce_s_per_param", C.c_double),
                ("reconstruct_s_per_param", C.c_double)]


class RankedConfigC(C.Structure):
    _fields_ = [("config", ParallelConfigC), ("score", C.c_double), ("memory_bytes", C.c_double),
                ("bubble", C.c_double), ("timing", TimingModelC)]


class ExecOptsC(C.Structure):
    _fields_ = [("device", C.c_int32), ("record_timeline", C.c_int32), ("seed", C.c_uint64),
                ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("init_std", C.c_float), ("flags", C.c_int32)]


_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)
_DP = C.POINTER(C.c_double)

_PROTOS = {
    # schedule
    "bfpp_last_error": (C.c_char_p, []),
    "bfpp_validate": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC), C.POINTER(ClusterSpecC)]),
    "bfpp_place_stages": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC), _I64P, C.c_int64,
                                    _I64P, _I64P]),
    "bfpp_build_tasks": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC), C.POINTER(_P)]),
    "bfpp_build_accumulation_tasks": (C.c_int, [C.POINTER(ModelSpecC), C.c_int32, C.c_int32, C.c_int64,
                                                C.POINTER(_P)]),
    "bfpp_graph_from_arrays": (C.c_int, [C.c_int64, C.c_int64, C.POINTER(TaskC), _I32P, _I32P, _I32P, _I32P,
                                         C.POINTER(_P)]),
    "bfpp_graph_n_devices": (C.c_int64, [_P]),
    "bfpp_graph_n_tasks": (C.c_int64, [_P]),
    "bfpp_graph_n_deps": (C.c_int64, [_P]),
    "bfpp_graph_n_program_steps": (C.c_int64, [_P]),
    "bfpp_graph_tasks": (C.c_int, [_P, C.POINTER(TaskC), C.c_int64]),
    "bfpp_graph_deps": (C.c_int, [_P, _I32P, _I32P]),
    "bfpp_graph_programs": (C.c_int, [_P, _I32P, _I32P]),
    "bfpp_graph_destroy": (None, [_P]),
    "bfpp_simulate": (C.c_int, [_P, C.POINTER(TimingModelC), C.POINTER(_P)]),
    "bfpp_simulate_durations": (C.c_int, [_P, _DP, C.POINTER(_P)]),
    "bfpp_timeline_n_events": (C.c_int64, [_P]),
    "bfpp_timeline_n_devices": (C.c_int64, [_P]),
    "bfpp_timeline_makespan": (C.c_double, [_P]),
    "bfpp_timeline_events": (C.c_int, [_P, _DP, _DP, _DP]),
    "bfpp_timeline_from_arrays": (C.c_int, [_P, _DP, _DP, C.POINTER(_P)]),
    "bfpp_timeline_destroy": (None, [_P]),
    "bfpp_bubble_fraction": (C.c_double, [_P]),
    "bfpp_peak_inflight": (C.c_int, [_P, _P, C.c_int64, _I64P]),
    "bfpp_compute_per_gpu": (C.c_double, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC)]),
    "bfpp_total_memory": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC), C.c_double, _DP]),
    "bfpp_feasible": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC), C.POINTER(ClusterSpecC),
                                C.c_double, C.c_double, _I32P]),
    "bfpp_cluster_preset": (C.c_int, [C.c_char_p, C.POINTER(ClusterSpecC)]),
    "bfpp_rates_from_timing": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC),
                                         C.POINTER(TimingModelC), C.POINTER(MeasuredRatesC)]),
    "bfpp_rank_configs": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ClusterSpecC), _I32P, C.c_int64, _I32P,
                                    C.c_int64] + [_I64P, C.c_int64] * 5
                          + [C.c_int32, C.POINTER(MeasuredRatesC), C.c_double, C.c_double, C.c_int32, C.c_int64,
                             C.POINTER(RankedConfigC), _I64P]),
    "bfpp_chrome_trace_json": (C.c_int, [_P, _P, C.c_char_p, C.c_int64, _I64P]),
    "bfpp_gantt_svg": (C.c_int, [_P, _P, C.c_char_p, C.c_int64, _I64P]),
    "bfpp_measured_timing_model": (C.c_int, [_P, _P, C.POINTER(TimingModelC)]),
    "bfpp_plan_rank": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int64] + [_I32P] * 6
                       + [_I64P, _I64P]),
}

_lib = None


def lib():
    """Loads libbfpp.so once; raises loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(make -C paper_2211_05953_b200/csrc); there is no fallback")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _bind_optional(L)
        _lib = L
    return _lib


def _bind_optional(L):
    """Prototypes of the device-side entry points (executor, kernels)."""
    from . import _native_dev
    _native_dev.bind(L)


def declared_symbols():
    """Every function name declared in include/bfpp.h (for the export test)."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "bfpp.h")
    with open(hdr) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bfpp_[a-z0-9_]+)\s*\(", text)))
