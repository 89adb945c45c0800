"""Times the attention kernels at a given shape (CUDA events, median of 20)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05953_b200 import ops
B, S, H = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (1, 2048, 16)
qkv = torch.randn(B * S, 3 * H * 128, device="cuda").bfloat16()
dout = torch.randn(B * S, H * 128, device="cuda").bfloat16()
o, lse = ops.attention_fwd(qkv, B, S, H)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[n // 2]
fl = 2.0 * B * S * (S + 1) * H * 128
tf = t(lambda: ops.attention_fwd(qkv, B, S, H)); tb = t(lambda: ops.attention_bwd(qkv, o, dout, lse, B, S, H))
print(f"B={B} S={S} H={H}: fwd {tf*1e3:.1f} us ({fl/tf/1e9:.0f} TF/s)  bwd {tb*1e3:.1f} us ({2.5*fl/tb/1e9:.0f} TF/s)")
