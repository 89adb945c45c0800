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

def _gemm_args(a, b, a_mn_major, b_mn_major, out, epilogue, aux, aux_out, accumulate):
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
    return args, out


def gemm_pair(first: dict, second: dict):
    """Two independent GEMMs in one grouped launch; each dict holds gemm()'s arguments
    (a, b, and optionally a_mn_major, b_mn_major, out, epilogue, aux, aux_out, accumulate)."""
    def unpack(d):
        return _gemm_args(d["a"], d["b"], d.get("a_mn_major", False), d.get("b_mn_major", False), d.get("out"),
                          d.get("epilogue", EPI_BF16), d.get("aux"), d.get("aux_out"), d.get("accumulate", False))
    (x, ox), (y, oy) = unpack(first), unpack(second)
    _check(_nat.lib().bfpp_gemm_bf16_pair(C.byref(x), C.byref(y), _stream()))
    return ox, oy


def attention_config(fwd_tiles: int = 0):
    """Query tiles per attention-forward CTA: 0 auto, 1, 2."""
    _check(_nat.lib().bfpp_attention_config(fwd_tiles))


def gemm_config(mode: int = -1, bn2: int = 0, stream_k: int = -1):
    """Process-wide GEMM variant selection (tests / benchmarks): mode -1 auto, 1 one-CTA, 2 two-CTA;
    bn2 = two-CTA tile width (0 default 256, 128); stream_k -1 auto, 0 off, 1 forced."""
    _check(_nat.lib().bfpp_gemm_config(mode, bn2, stream_k))


def gemm_schedule(dynamic: bool = False):
    """Tile schedule of the persistent 2-CTA GEMM: static (default) or dynamic (device tile counter)."""
    _check(_nat.lib().bfpp_gemm_schedule(1 if dynamic else 0))


def attention_fwd(qkv, batch, seq, heads, head_dim=128):
    T = batch * seq
    o = torch.empty(T, heads * head_dim, device=qkv.device, dtype=torch.bfloat16)
    lse = torch.empty(batch * heads, seq, device=qkv.device, dtype=torch.float32)
    _check(_nat.lib().bfpp_attention_fwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), batch, seq, heads,
                                         head_dim, _stream()))
    return o, lse


def attention_bwd(qkv, o, dout, lse, batch, seq, heads, head_dim=128):
    T = batch * seq
    delta = torch.empty(batch * heads, seq, device=qkv.device, dtype=torch.float32)
    dq_acc = torch.empty(T, heads * head_dim, device=qkv.device, dtype=torch.float32)
    dqkv = torch.empty_like(qkv)
    _check(_nat.lib().bfpp_attention_bwd(qkv.data_ptr(), o.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                         delta.data_ptr(), dq_acc.data_ptr(), dqkv.data_ptr(), batch, seq, heads,
                                         head_dim, _stream()))
    return dqkv


def layernorm_fwd(x, gamma, beta, eps=1e-5):
    rows, width = x.shape
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=x.device, dtype=torch.float32)
    rstd = torch.empty(rows, device=x.device, dtype=torch.float32)
    _check(_nat.lib().bfpp_layernorm_fwd(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(),
                                         mean.data_ptr(), rstd.data_ptr(), rows, width, eps, _stream()))
    return y, mean, rstd


def layernorm_bwd(dy, x, gamma, mean, rstd, dgamma, dbeta, dres=None):
    rows, width = x.shape
    dx = torch.empty_like(x)
    _check(_nat.lib().bfpp_layernorm_bwd(dy.data_ptr(), x.data_ptr(), gamma.data_ptr(), mean.data_ptr(),
                                         rstd.data_ptr(), _ptr(dres), dx.data_ptr(), dgamma.data_ptr(),
                                         dbeta.data_ptr(), rows, width, _stream()))
    return dx


def embed_fwd(tok, wte, wpe, seq):
    T, h = tok.numel(), wte.shape[1]
    x = torch.empty(T, h, device=wte.device, dtype=torch.bfloat16)
    _check(_nat.lib().bfpp_embed_fwd(tok.data_ptr(), wte.data_ptr(), wpe.data_ptr(), x.data_ptr(), T, seq, h,
                                     _stream()))
    return x


def embed_bwd(tok, dx, dwte, dwpe, seq):
    T, h = dx.shape
    _check(_nat.lib().bfpp_embed_bwd(tok.data_ptr(), dx.data_ptr(), dwte.data_ptr(), dwpe.data_ptr(), T, seq, h,
                                     _stream()))


def softmax_xent_(logits, labels, grad_scale):
    T, V = logits.shape
    loss = torch.empty(T, device=logits.device, dtype=torch.float32)
    _check(_nat.lib().bfpp_softmax_xent(logits.data_ptr(), logits.stride(0), labels.data_ptr(), loss.data_ptr(),
                                        T, V, grad_scale, _stream()))
    return loss


def adam_update_(p, m, v, g, w16, lr, beta1, beta2, eps, wd, step, zero_grad=False):
    _check(_nat.lib().bfpp_adam_update(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), w16.data_ptr(),
                                       p.numel(), lr, beta1, beta2, eps, wd, step, int(zero_grad), _stream()))
