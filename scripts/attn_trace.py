"""Prints the per-query-block timeline (clock64, relative cycles) of CTA (0,0,0) of the attention
backward kernel built with BFPP_ATTN_TRACE (scripts/attn_trace.cu)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
L = C.CDLL(os.path.join(HERE, "libattntrace.so"))
B, S, H = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (1, 2048, 16)
qkv = torch.randn(B * S, 3 * H * 128, device="cuda").bfloat16()
o = torch.empty(B * S, H * 128, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H, S, device="cuda")
L.trace_fwd(C.c_void_p(qkv.data_ptr()), C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()), B, S, H)
dout = torch.randn(B * S, H * 128, device="cuda").bfloat16()
delta = torch.empty(B * H, S, device="cuda")
dq = torch.empty(B * S, H * 128, device="cuda")
dqkv = torch.empty_like(qkv)
for _ in range(3):
    L.trace_clear()
    L.trace_bwd(*[C.c_void_p(t.data_ptr()) for t in (qkv, o, dout, lse, delta, dq, dqkv)], B, S, H)
torch.cuda.synchronize()
buf = np.zeros((8, 64, 16), dtype=np.uint64)
assert L.trace_read(buf.ctypes.data_as(C.c_void_p)) == 0
t0 = buf[buf > 0].min()
rel = np.where(buf > 0, buf.astype(np.int64) - int(t0), -1)
names = {0: ["q_issue", "oA_issue", "oB_issue"],
         1: ["q_full", "dq_empty", "o_full", "s_commit", "-", "-", "-", "p0", "-", "p1", "dq_commit", "end"],
         2: ["wait", "dq_full", "tma0", "tma1"],
         3: ["barA", "barA_done", "sA", "pA"], 4: ["barB", "barB_done", "sB", "pB"]}
role = ["producer", "mma", "drain", "elemA", "elemB"]
n_it = (S + 127) // 128
for it in range(n_it):
    print(f"--- block {it}")
    for r in range(5):
        print(f"  {role[r]:8s} " + " ".join(f"{n}={rel[r, it, k]}" for k, n in enumerate(names[r]) if n != "-"))
