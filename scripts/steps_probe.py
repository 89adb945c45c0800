"""Runs N single-GPU training steps printing the loss (hang/NaN probe)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2211_05953_b200 import pipesim as ps
from paper_2211_05953_b200.executor import Executor
from paper_2211_05953_b200.model import GPTConfig
model = sys.argv[1] if len(sys.argv) > 1 else "gpt-1.3b"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
skip = len(sys.argv) > 3 and sys.argv[3] == "skip"
cfg = GPTConfig.preset(model)
c = ps.ParallelConfig(n_loop=4, n_mb=1, schedule=ps.Schedule.BreadthFirst)
ex = Executor(cfg, c, skip_optimizer=skip, lr=1e-4)
tok = torch.randint(0, cfg.s_voc, (1, 1, cfg.s_seq + 1), dtype=torch.int32).pin_memory()
t0 = time.time()
for i in range(n):
    loss = ex.step(tok)
    print(i, f"{loss:.5f}", f"{time.time()-t0:.2f}s", flush=True)
