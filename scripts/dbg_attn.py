import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05953_b200 import ops
B, S, H = [int(x) for x in sys.argv[1:4]]
qkv = torch.randn(B * S, 3 * H * 128, device="cuda").bfloat16()
o, lse = ops.attention_fwd(qkv, B, S, H); torch.cuda.synchronize(); print("fwd ok", flush=True)
dout = torch.randn(B * S, H * 128, device="cuda").bfloat16()
d = ops.attention_bwd(qkv, o, dout, lse, B, S, H); torch.cuda.synchronize(); print("bwd ok", flush=True)
