"""Schedule x batch-per-GPU sweep on one box (launches bench.py under torchrun per point).

    python scripts/sweep.py --gpus 4 --model gpt-6.7b --pp 4 --loops 2 --betas 1 2 4 8 \
        --schedules breadth_first depth_first 1f1b gpipe --out profiles/sweep.jsonl
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--model", default="gpt-6.7b")
    ap.add_argument("--pp", type=int, default=4)
    ap.add_argument("--loops", type=int, default=2)
    ap.add_argument("--betas", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--schedules", nargs="+", default=["breadth_first", "depth_first", "1f1b", "gpipe"])
    ap.add_argument("--dp-variant", default="dp_fs")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", required=True)
    ap.add_argument("--timeout", type=int, default=400)
    a = ap.parse_args()
    port = 29600
    with open(a.out, "a") as f:
        for beta in a.betas:
            for sched in a.schedules:
                port += 1
                loops = a.loops if sched in ("breadth_first", "depth_first") else 1  # GPipe / 1F1B: no loops
                cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
                       "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
                       "--gpus", str(a.gpus), "--model", a.model, "--schedule", sched, "--pp", str(a.pp),
                       "--loops", str(loops), "--beta", str(beta), "--dp-variant", a.dp_variant,
                       "--steps", str(a.steps), "--warmup", str(a.warmup), "--no-e2e", "--no-cpu-baseline"]
                if a.gpus == 1:
                    cmd = cmd[:1] + cmd[cmd.index(os.path.join(ROOT, "bench.py")):]
                try:
                    r = subprocess.run(cmd, capture_output=True, text=True, timeout=a.timeout)
                    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
                    rec = json.loads(lines[-1]) if lines else {"error": (r.stderr or r.stdout)[-600:]}
                except subprocess.TimeoutExpired:
                    rec = {"error": "timeout"}
                rec.update({"sweep_schedule": sched, "sweep_beta": beta, "sweep_model": a.model})
                f.write(json.dumps(rec) + "\n")
                f.flush()
                v = rec.get("value")
                print(f"{a.model} {sched:14s} beta={beta}: "
                      + (f"{v:,.0f} tok/s  mfu={rec['mfu']['vs_spec_2250TF']:.3f}  bubble={rec['bubble_fraction']}"
                         if v else rec.get("error", "?")[:300]), flush=True)


if __name__ == "__main__":
    main()
