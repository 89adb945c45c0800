"""Micro-benchmark of the tcgen05 GEMM on the exact GEMMs of one training step
(CUDA events, median of 20, L2 flushed between iterations), next to cuBLAS."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05953_b200 import ops  # noqa: E402


def bench(fn, iters=20, flush=True):
    buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush:
            buf.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e-3


def step_gemms(T, h, V):
    m = 4 * h
    E = ops
    # name, M, N, K, a_mn, b_mn, epilogue
    return [("fwd qkv", T, 3 * h, h, 0, 0, E.EPI_BF16), ("fwd o+res", T, h, h, 0, 0, E.EPI_RESID),
            ("fwd fc1+gelu", T, m, h, 0, 0, E.EPI_GELU), ("fwd fc2+res", T, h, m, 0, 0, E.EPI_RESID),
            ("wgrad fc2", h, m, T, 1, 1, E.EPI_F32), ("dgrad fc2+dgelu", T, m, h, 0, 1, E.EPI_DGELU),
            ("wgrad fc1", m, h, T, 1, 1, E.EPI_F32), ("dgrad fc1", T, h, m, 0, 1, E.EPI_BF16),
            ("wgrad o", h, h, T, 1, 1, E.EPI_F32), ("dgrad o", T, h, h, 0, 1, E.EPI_BF16),
            ("wgrad qkv", 3 * h, h, T, 1, 1, E.EPI_F32), ("dgrad qkv", T, h, 3 * h, 0, 1, E.EPI_BF16),
            ("head fwd", T, V, h, 0, 0, E.EPI_BF16), ("head dgrad", T, h, V, 0, 1, E.EPI_BF16),
            ("head wgrad", V, h, T, 1, 1, E.EPI_F32)]


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    V = 50304
    tot_ours = tot_cb = tot_fl = 0.0
    for name, M, N, K, amn, bmn, epi in step_gemms(T, h, V):
        A = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
        B = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == ops.EPI_F32 else torch.bfloat16)
        aux = torch.randn(M, N, device="cuda").bfloat16()
        kw = dict(a_mn_major=bool(amn), b_mn_major=bool(bmn), out=out, epilogue=epi)
        if epi in (ops.EPI_RESID, ops.EPI_DGELU):
            kw["aux"] = aux
        if epi == ops.EPI_GELU:
            kw["aux_out"] = aux
        if epi == ops.EPI_F32:
            kw["accumulate"] = True
        t = bench(lambda: ops.gemm(A, B, **kw))
        Am = A.t() if amn else A
        Bm = B if bmn else B.t()
        o2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        tc = bench(lambda: torch.matmul(Am, Bm, out=o2))
        fl = 2.0 * M * N * K
        tot_ours += t
        tot_cb += tc
        tot_fl += fl
        print(f"{name:16s} M={M:6d} N={N:6d} K={K:6d}  ours {fl / t / 1e12:7.1f} TF/s ({t * 1e6:7.1f} us)"
              f"  cublas {fl / tc / 1e12:7.1f} TF/s ({tc * 1e6:7.1f} us)", flush=True)
    print(f"TOTAL ours {tot_fl / tot_ours / 1e12:.1f} TF/s  cublas {tot_fl / tot_cb / 1e12:.1f} TF/s")


if __name__ == "__main__":
    main()
