"""LayerNorm kernels alone at the step's shapes (CUDA events, median of 50)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05953_b200 import ops  # noqa: E402


def bench(fn, iters=10, reps=20):
    """fn x reps captured in a CUDA graph (no host launch overhead in the measurement)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e3 / reps


for rows, width in [(2048, 2048), (8192, 2048), (2048, 4096), (4096, 4096), (2048, 5120), (2048, 8192)]:
    x = torch.randn(rows, width, device="cuda").bfloat16()
    g = torch.ones(width, device="cuda").bfloat16()
    b = torch.zeros(width, device="cuda").bfloat16()
    y, mean, rstd = ops.layernorm_fwd(x, g, b)
    dy = torch.randn_like(x)
    dres = torch.randn_like(x)
    dg = torch.zeros(width, device="cuda")
    db = torch.zeros(width, device="cuda")
    tf = bench(lambda: ops.layernorm_fwd(x, g, b))
    tb = bench(lambda: ops.layernorm_bwd(dy, x, g, mean, rstd, dg, db, dres=dres))
    nb = rows * width * 2  # bytes of one bf16 [rows, width] tensor
    print(f"rows {rows} width {width}: fwd {tf:6.1f} us ({2 * nb / tf / 1e6:5.2f} TB/s)  "
          f"bwd {tb:6.1f} us ({4 * nb / tb / 1e6:5.2f} TB/s)")
