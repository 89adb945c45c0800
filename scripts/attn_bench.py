"""Times the attention kernels at a given shape (CUDA graph of 20 calls, median of 5 replays)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05953_b200 import ops  # noqa: E402

B, S, H = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (1, 2048, 16)
qkv = torch.randn(B * S, 3 * H * 128, device="cuda").bfloat16()
dout = torch.randn(B * S, H * 128, device="cuda").bfloat16()
o, lse = ops.attention_fwd(qkv, B, S, H)
SIDE = torch.cuda.Stream()


def t(fn, reps=20):
    with torch.cuda.stream(SIDE):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=SIDE):
        for _ in range(reps):
            fn()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    return sorted(ts)[2]


fl = 2.0 * B * S * (S + 1) * H * 128
tf = t(lambda: ops.attention_fwd(qkv, B, S, H))
tb = t(lambda: ops.attention_bwd(qkv, o, dout, lse, B, S, H))
print(f"B={B} S={S} H={H}: fwd {tf * 1e3:.1f} us ({fl / tf / 1e9:.0f} TF/s)  "
      f"bwd {tb * 1e3:.1f} us ({2.5 * fl / tb / 1e9:.0f} TF/s)")
