"""Micro-benchmark of the tcgen05 GEMM on transformer shapes (CUDA events, L2-flushed)."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2211_05953_b200 import ops  # noqa: E402


def bench(fn, iters=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e-3


def main():
    T = 2048 * int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    shapes = []
    for h in (2048, 4096):
        shapes += [("fwd qkv h%d" % h, T, 3 * h, h, 0, 0), ("fwd fc1 h%d" % h, T, 4 * h, h, 0, 0),
                   ("fwd fc2 h%d" % h, T, h, 4 * h, 0, 0), ("dgrad fc1 h%d" % h, T, h, 4 * h, 0, 1),
                   ("wgrad fc1 h%d" % h, 4 * h, h, T, 1, 1)]
    shapes.append(("lm head", T, 50304, 4096, 0, 0))
    for name, M, N, K, amn, bmn in shapes:
        A = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
        B = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t = bench(lambda: ops.gemm(A, B, a_mn_major=bool(amn), b_mn_major=bool(bmn), out=out))
        Am = A.t() if amn else A
        Bm = B if bmn else B.t()
        tc = bench(lambda: torch.matmul(Am, Bm, out=out))
        fl = 2.0 * M * N * K
        print(f"{name:18s} M={M:6d} N={N:6d} K={K:6d}  ours {fl / t / 1e12:7.1f} TF/s ({t * 1e6:8.1f} us)"
              f"  cublas {fl / tc / 1e12:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
