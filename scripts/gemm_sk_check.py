"""Stream-K vs data-parallel 2-CTA GEMM on the step's shapes: exactness (same result up to f32
summation order) and time (CUDA graph of 20 launches)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05953_b200 import ops  # noqa: E402


SIDE = torch.cuda.Stream()


def bench(fn, reps=20, iters=5):
    with torch.cuda.stream(SIDE):  # warm up (and allocate per-stream workspaces) on the capture stream
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=SIDE):
        for _ in range(reps):
            fn()
    ts = []
    for _ in range(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / reps)
    return sorted(ts)[len(ts) // 2] * 1e3


E = ops
T, h = 2048, int(sys.argv[1]) if len(sys.argv) > 1 else 2048
m = 4 * h
shapes = [("qkv", T, 3 * h, h, 0, 0, E.EPI_BF16), ("o+res", T, h, h, 0, 0, E.EPI_RESID),
          ("fc1+gelu", T, m, h, 0, 0, E.EPI_GELU), ("fc2+res", T, h, m, 0, 0, E.EPI_RESID),
          ("wgrad fc2", h, m, T, 1, 1, E.EPI_F32), ("dgrad fc2", T, m, h, 0, 1, E.EPI_DGELU),
          ("wgrad fc1", m, h, T, 1, 1, E.EPI_F32), ("dgrad fc1", T, h, m, 0, 1, E.EPI_BF16),
          ("wgrad o", h, h, T, 1, 1, E.EPI_F32), ("dgrad qkv", T, h, 3 * h, 0, 1, E.EPI_BF16)]
tot = {0: 0.0, 1: 0.0}
for name, M, N, K, amn, bmn, epi in shapes:
    A = (torch.randn((K, M) if amn else (M, K), device="cuda") * 0.5).bfloat16()
    B = (torch.randn((K, N) if bmn else (N, K), device="cuda") * 0.5).bfloat16()
    aux = torch.randn(M, N, device="cuda").bfloat16()
    outs, times = {}, {}
    for sk in (0, 1):
        ops.gemm_config(2, 256, sk)
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == E.EPI_F32 else torch.bfloat16)
        pre = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi == E.EPI_GELU else None
        kw = dict(a_mn_major=bool(amn), b_mn_major=bool(bmn), out=out, epilogue=epi,
                  aux=aux if epi in (E.EPI_RESID, E.EPI_DGELU) else None, aux_out=pre)
        ops.gemm(A, B, **kw)
        torch.cuda.synchronize()
        outs[sk] = out.float().clone()
        times[sk] = bench(lambda: ops.gemm(A, B, **kw))
        tot[sk] += times[sk]
    err = (outs[0] - outs[1]).abs().max().item() / (outs[0].abs().max().item() + 1e-6)
    fl = 2.0 * M * N * K
    print(f"{name:10s} {M:5d}x{N:5d}x{K:5d}  dp {times[0]:7.1f} us ({fl / times[0] / 1e6:6.0f} TF/s)  "
          f"sk {times[1]:7.1f} us ({fl / times[1] / 1e6:6.0f} TF/s)  rel diff {err:.2e}", flush=True)
print(f"TOTAL dp {tot[0]:.1f} us  sk {tot[1]:.1f} us")
