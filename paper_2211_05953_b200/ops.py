"""Thin torch-tensor front end over the device kernels of libbfpp.so.

Tensors are used only as device memory (data_ptr) and for the current CUDA
stream; every computation happens in the hand-written sm_100a kernels behind
the C ABI. There is no fallback path: a failed launch raises.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as _nat
from ._native_dev import GemmArgsC

EPI_BF16, EPI_GELU, EPI_RESID, EPI_DGELU, EPI_F32 = 0, 1, 2, 3, 4


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check(st):
    if st != 0:
        raise RuntimeError(_nat.lib().bfpp_last_error().decode())


def _ptr(t):
    return t.data_ptr() if t is not None else None


def gemm(a: torch.Tensor, b: torch.Tensor, *, a_mn_major=False, b_mn_major=False, out=None,
         epilogue=EPI_BF16, aux=None, aux_out=None, accumulate=False):
    """out[M,N] = sum_k A[m,k] B[n,k].

    a: [M,K] (or [K,M] if a_mn_major); b: [N,K] (or [K,N] if b_mn_major); bf16, row-major
    (unit stride in the last dimension, any leading stride).
    """
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    assert a.stride(1) == 1 and b.stride(1) == 1
    M, K = (a.shape[1], a.shape[0]) if a_mn_major else a.shape
    N = b.shape[1] if b_mn_major else b.shape[0]
    assert (b.shape[0] if b_mn_major else b.shape[1]) == K
    if out is None:
        out = torch.empty(M, N, device=a.device,
                          dtype=torch.float32 if epilogue == EPI_F32 else torch.bfloat16)
    args = GemmArgsC(M, N, K, a.data_ptr(), a.stride(0), int(a_mn_major), b.data_ptr(), b.stride(0),
                     int(b_mn_major), out.data_ptr(), out.stride(0),
                     _ptr(aux), aux.stride(0) if aux is not None else 0,
                     _ptr(aux_out), aux_out.stride(0) if aux_out is not None else 0, epilogue, int(accumulate))
    _check(_nat.lib().bfpp_gemm_bf16(C.byref(args), _stream()))
    return out
