"""Prints the measured per-task timeline of one N=1 step (after warm-up) for a bench config."""
import argparse
import torch

from paper_2211_05953_b200 import pipesim as ps
from paper_2211_05953_b200.executor import Executor
from paper_2211_05953_b200.model import GPTConfig

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="gpt-1.3b")
ap.add_argument("--loops", type=int, default=4)
ap.add_argument("--n-mb", type=int, default=1)
ap.add_argument("--schedule", default="BreadthFirst")
ap.add_argument("--skip-opt", action="store_true")
ap.add_argument("--quiet", action="store_true")
args = ap.parse_args()
cfg = GPTConfig.preset(args.model)
config = ps.ParallelConfig(n_dp=1, n_pp=1, n_loop=args.loops, n_mb=args.n_mb, dp_variant=ps.DpVariant.DP_FS,
                           schedule=ps.Schedule[args.schedule])
ex = Executor(cfg, config, lr=1e-4, skip_optimizer=args.skip_opt)
tok = torch.randint(0, cfg.s_voc, (args.n_mb, 1, cfg.s_seq + 1), device="cuda", dtype=torch.int32)
loss = torch.zeros(1, device="cuda")
for _ in range(4):
    ex.step_device(tok, loss)
ex.set_flags(record_timeline=True, profile_kernels=False)
for _ in range(2):
    ex.step_device(tok, loss)
ex.sync()
s, e = ex.task_times()
rows = []
for t in ex.graph.tasks:
    if s[t.id] == s[t.id]:
        rows.append((s[t.id], e[t.id], t.kind.name, t.stage, t.micro_batch, t.id))
rows.sort()
for a, b, k, st, mb, i in ([] if args.quiet else rows):
    print(f"{a * 1e3:9.3f} {b * 1e3:9.3f} {(b - a) * 1e3:8.3f} ms  {k:12s} stage {st} mb {mb} id {i}")
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
stream = torch.cuda.ExternalStream(ex.stream_handle)
ex.set_flags(False, False)
e0.record(stream)
for _ in range(5):
    ex.step_device(tok, loss)
e1.record(stream)
torch.cuda.synchronize()
print("ms/step", e0.elapsed_time(e1) / 5)
ex.set_flags(False, True)
ex.step_device(tok, loss)
ex.sync()
for k, (n, ms, work) in ex.kernel_stats().items():
    print(f"{k:14s} launches {n:5d}  {ms:8.3f} ms  {work / ms / 1e9 if ms else 0:10.1f} (G work/s)")
ex.close()
