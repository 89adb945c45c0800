"""Per-CTA start/end spread of one 2-CTA GEMM launch (scripts/gemm_trace.cu), alone and with the
optimizer kernel streaming on a low-priority stream (the in-step co-running case). Shows whether
the co-running slowdown is uniform or concentrated on the SMs that host optimizer blocks."""
import ctypes as C
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2211_05953_b200 import ops  # noqa: E402

L = C.CDLL(os.path.join(HERE, "libgemmtrace.so"))
M, N, K = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (2048, 8192, 2048)
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
hi = torch.cuda.Stream(priority=-5)
lo = torch.cuda.Stream(priority=0)
n_param = 300 << 20
p = torch.randn(n_param, device="cuda")
mm, vv, g = torch.zeros_like(p), torch.ones_like(p), torch.randn_like(p)
w16 = torch.empty(n_param, device="cuda", dtype=torch.bfloat16)


def run(with_adam):
    torch.cuda.synchronize()
    if with_adam:
        with torch.cuda.stream(lo):
            for _ in range(3):
                ops.adam_update_(p, mm, vv, g, w16, 1e-4, 0.9, 0.95, 1e-8, 0.0, 1)
        torch.cuda._sleep(2_000_000)  # let the optimizer fill the GPU first
    with torch.cuda.stream(hi):
        if with_adam:
            hi.wait_stream(torch.cuda.current_stream())
        L.trace_gemm(M, N, K, C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(D.data_ptr()),
                     C.c_void_p(hi.cuda_stream))
    torch.cuda.synchronize()
    buf = np.zeros((512, 4), dtype=np.uint64)
    assert L.trace_read(buf.ctypes.data_as(C.c_void_p)) == 0
    return buf


for label, adam in (("alone", False), ("alone", False), ("beside adam", True)):
    buf = run(adam)
    used = buf[:, 0] > 0
    st, en, tiles, sm = (buf[used, i].astype(np.int64) for i in range(4))
    t0 = st.min()
    dur = (en - t0) / 1e3
    start = (st - t0) / 1e3
    span = dur.max()
    flops = 2.0 * M * N * K
    print(f"{label}: {used.sum()} CTAs, span {span:.1f} us ({flops / span / 1e6:.0f} TF/s); start max {start.max():.1f} us; "
          f"end min/median/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us; tiles/CTA {tiles.min()}-{tiles.max()}")
    order = np.argsort(dur)
    print("   earliest ends (sm, tiles, us):", [(int(sm[i]), int(tiles[i]), round(float(dur[i]), 1)) for i in order[:6]])
    print("   latest ends   (sm, tiles, us):", [(int(sm[i]), int(tiles[i]), round(float(dur[i]), 1)) for i in order[-6:]])
    # per-tile time of each CTA (end - start) / tiles
    per = (en - st) / np.maximum(tiles, 1) / 1e3
    print(f"   us per tile: min {per.min():.2f} median {np.median(per):.2f} max {per.max():.2f}")
