"""Prototypes of the device-side C ABI entry points (kernels + executor)."""
from __future__ import annotations

import ctypes as C

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32


class GemmArgsC(C.Structure):
    _fields_ = [("M", _I64), ("N", _I64), ("K", _I64),
                ("A", _P), ("lda", _I64), ("a_mn_major", _I32),
                ("B", _P), ("ldb", _I64), ("b_mn_major", _I32),
                ("D", _P), ("ldd", _I64),
                ("aux", _P), ("ldaux", _I64),
                ("aux_out", _P), ("ldaux_out", _I64),
                ("epilogue", _I32), ("accumulate", _I32)]


PROTOS: dict = {
    "bfpp_gemm_bf16": (C.c_int, [C.POINTER(GemmArgsC), _P]),
    "bfpp_gemm_config": (C.c_int, [C.c_int32, C.c_int32, C.c_int32]),
    "bfpp_gemm_schedule": (C.c_int, [C.c_int32]),
    "bfpp_gemm_sm_limit": (C.c_int, [C.c_int32]),
    "bfpp_attention_config": (C.c_int, [C.c_int32]),
    "bfpp_gemm_bf16_pair": (C.c_int, [C.POINTER(GemmArgsC), C.POINTER(GemmArgsC), _P]),
    "bfpp_kernel_variant_count": (C.c_int64, [C.c_int32]),
    "bfpp_kernel_variant_reset": (None, []),
}


def bind(L):
    for name, (res, args) in PROTOS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args

_F = C.c_float
_FP = C.c_void_p  # float* passed as raw pointers
PROTOS.update({
    "bfpp_attention_fwd": (C.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _P]),
    "bfpp_attention_bwd": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _P]),
    "bfpp_layernorm_fwd": (C.c_int, [_P, _P, _P, _P, _P, _P, _I32, _I32, _F, _P]),
    "bfpp_layernorm_bwd": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _P]),
    "bfpp_embed_fwd": (C.c_int, [_P, _P, _P, _P, _I32, _I32, _I32, _P]),
    "bfpp_embed_bwd": (C.c_int, [_P, _P, _P, _P, _I32, _I32, _I32, _P]),
    "bfpp_softmax_xent": (C.c_int, [_P, _I64, _P, _P, _I32, _I32, _F, _P]),
    "bfpp_adam_update": (C.c_int, [_P, _P, _P, _P, _P, _I64, _F, _F, _F, _F, _F, _I32, _I32, _P]),
})

from ._native import ModelSpecC, ParallelConfigC, ExecOptsC  # noqa: E402

PROTOS.update({
    "bfpp_nccl_unique_id": (C.c_int, [_P]),
    "bfpp_exec_n_comm_ids": (_I64, [C.POINTER(ParallelConfigC)]),
    "bfpp_exec_create": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC), C.POINTER(ExecOptsC), _I32,
                                   _I32, _P, C.POINTER(_P)]),
    "bfpp_exec_create_graph": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC), _P, C.POINTER(ExecOptsC),
                                         _I32, _I32, _P, C.POINTER(_P)]),
    "bfpp_exec_step": (C.c_int, [_P, _P, C.POINTER(C.c_float)]),
    "bfpp_exec_step_device": (C.c_int, [_P, _P, _P]),
    "bfpp_exec_sync": (C.c_int, [_P]),
    "bfpp_exec_destroy": (None, [_P]),
    "bfpp_exec_graph": (C.c_int, [_P, C.POINTER(_P)]),
    "bfpp_exec_n_local_stages": (_I64, [_P]),
    "bfpp_exec_local_stage": (_I64, [_P, _I64]),
    "bfpp_exec_stage_numel": (_I64, [_P, _I64]),
    "bfpp_exec_device_bytes": (_I64, [_P]),
    "bfpp_exec_memory_plan": (C.c_int, [C.POINTER(ModelSpecC), C.POINTER(ParallelConfigC), C.POINTER(ExecOptsC), _I32,
                                        C.POINTER(_I64), C.POINTER(_I64)]),
    "bfpp_exec_memory": (C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I64)]),
    "bfpp_exec_set_params": (C.c_int, [_P, _I64, _P, _I64]),
    "bfpp_exec_get_params": (C.c_int, [_P, _I64, _P, _I64, C.POINTER(_I64), C.POINTER(_I64)]),
    "bfpp_exec_get_grads": (C.c_int, [_P, _I64, _P, _I64, C.POINTER(_I64), C.POINTER(_I64)]),
    "bfpp_exec_zero_grads": (C.c_int, [_P]),
    "bfpp_exec_get_weights16": (C.c_int, [_P, _I64, _P, _I64, C.POINTER(_I64), C.POINTER(_I64)]),
    "bfpp_exec_timeline": (C.c_int, [_P, _P, _P]),
    "bfpp_exec_stream": (_P, [_P]),
    "bfpp_exec_set_flags": (C.c_int, [_P, _I32, _I32]),
    "bfpp_exec_kernel_stats": (C.c_int, [_P, _I32, C.POINTER(_I64), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]),
})
