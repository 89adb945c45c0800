"""Benchmark of the breadth-first pipeline executor (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--model M] ...
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Workload (BASELINE.json configs[1]): GPT-1.3B (L24, h2048, 16 heads of 128, V 50304, seq 2048),
breadth-first looping schedule with 4 loops, fully sharded DP, 1 sequence per GPU:
  N=1: PP1 x 4 loops;  N=2: PP2 x 4 loops, DP1;  N=4: PP2 x 4 loops x DP2;  N=8: PP2 x 4 loops x DP4.
A step = one full training step (forward, backward, FSDP reduce-scatter, Adam) over the global batch.
Inputs are synthetic token ids; weights are random-initialised on device.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import time

import numpy as np

# executor streams need their own hardware work queues (paper_2211_05953_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # one hardware queue per executor stream (see executor.py)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCHEDULES = {"breadth_first": 4, "depth_first": 3, "1f1b": 2, "gpipe": 1, "no_pipeline": 0}
SPEC_BF16_FLOPS = 2.25e15


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="gpt-1.3b")
    ap.add_argument("--schedule", default="breadth_first", choices=list(SCHEDULES))
    ap.add_argument("--beta", type=int, default=1, help="sequences per GPU")
    ap.add_argument("--pp", type=int, default=None)
    ap.add_argument("--loops", type=int, default=4)
    ap.add_argument("--dp-variant", default="dp_fs", choices=["dp0", "dp_ps", "dp_fs"])
    ap.add_argument("--s-mb", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-timeline", action="store_true")
    ap.add_argument("--recompute", action="store_true", help="activation checkpointing (recompute in the backward)")
    return ap.parse_args()


def layout(args, n):
    pp = args.pp if args.pp is not None else (1 if n == 1 else 2)
    if n % pp:
        raise SystemExit(f"--gpus {n} is not a multiple of pp {pp}")
    dp = n // pp
    loops = args.loops if SCHEDULES[args.schedule] in (3, 4) else 1
    sched = args.schedule
    if pp == 1 and sched in ("gpipe", "1f1b"):
        sched = "no_pipeline" if loops == 1 else sched
    n_mb = args.beta * n // (dp * args.s_mb)
    if n_mb < pp:
        n_mb = pp
    return pp, dp, loops, n_mb, sched


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r.split(",") for r in (getattr(self, "out", "") or "").strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def config_dict(args, cfg, pp, dp, loops, n_mb, sched):
    """The workload keys both arms print (identical, so the driver can pair the lines)."""
    return {"workload": f"BASELINE configs[1]: {args.model} seq {cfg.s_seq}, {sched} PP{pp}x{loops} loops"
                        f" x DP{dp} {args.dp_variant}, {args.beta} seq/GPU",
            "model": args.model, "global_batch": n_mb * args.s_mb * dp, "seq_len": cfg.s_seq,
            "parallelism": f"pp{pp}x{loops}loops-dp{dp}-{args.dp_variant}", "schedule": sched,
            "n_mb": n_mb, "s_mb": args.s_mb,
            "l2": "inputs larger than L2 (bf16 weights + activations >> 126 MB)"}


def reference_arm(args):
    """CPU reference arm: the oracle port (the reference has no model executor) on
    the host cores. Each step is one bounded sample of the workload (oracle/cpu_baseline.py
    SampleStep: one layer + an LM-head slice, model-flop weighted into tokens), really executed, so
    ms_per_step x steps is the wall time the arm spends; value = sample tokens / sample seconds."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cpu_baseline as CB
    from paper_2211_05953_b200.model import GPTConfig
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.gpus
    cfg = GPTConfig.preset(args.model)
    pp, dp, loops, n_mb, sched = layout(args, n)
    sample = CB.SampleStep(cfg)
    times = []
    t_all = time.perf_counter()
    for i in range(args.warmup + args.steps):
        t = sample.run()
        if i >= args.warmup:
            times.append(t)
    wall = time.perf_counter() - t_all
    sec = float(np.mean(times))
    tps = sample.tokens_equiv / sec
    threads = CB.blas_threads()
    line = {"impl": "reference", "metric": "tokens/sec", "value": tps, "unit": "tokens/s", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, cfg, pp, dp, loops, n_mb, sched),
            "tokens_per_step": sample.tokens_equiv,
            "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "port",
                             "sample": sample.desc + "; the reference (pipesim) has no CPU model executor"},
            "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


NVLINK_GBS_PER_DIR = 770.0  # measured NVLink 5 peer-copy bandwidth per direction


def comm_rates(ex, cfg, config, tl, s_mb):
    """Achieved bandwidth of the measured timeline's communication tasks (NCCL / peer
    copies are NVLink-bound): each Transfer moves one [s_mb*seq, h] bf16 activation (or gradient)
    to the ring neighbour; each Reconstruct all-gathers a stage's bf16 weights, (n_dp-1)/n_dp of
    which arrive over NVLink per rank. Under the per-segment early reduce the Reduce tasks only hold
    the tail segments, so they are not rated."""
    from paper_2211_05953_b200 import pipesim as ps
    out = {}
    ev = tl.events
    tasks = ex.graph.tasks
    xfer = [ev[t.id].end - ev[t.id].start for t in tasks if t.kind == ps.TaskKind.Transfer]
    if xfer:
        b = 2.0 * s_mb * cfg.s_seq * cfg.s_hidden
        med = float(np.median(xfer))
        out["transfer"] = {"count": len(xfer), "bytes": b, "median_us": med * 1e6,
                           "gbs_median": b / med / 1e9 if med > 0 else None,
                           "frac_of_nvlink_dir": b / med / 1e9 / NVLINK_GBS_PER_DIR if med > 0 else None}
    if config.n_dp >= 2:
        rec = [(t, ev[t.id].end - ev[t.id].start) for t in tasks if t.kind == ps.TaskKind.Reconstruct
               and t.stage in ex.local_stages]
        if rec:
            rates = [2.0 * ex.stage_numel(t.stage) * (config.n_dp - 1) / config.n_dp / d / 1e9 for t, d in rec if d > 0]
            out["reconstruct"] = {"count": len(rec), "gbs_median": float(np.median(rates)),
                                  "frac_of_nvlink_dir": float(np.median(rates)) / NVLINK_GBS_PER_DIR,
                                  "median_us": float(np.median([d for _, d in rec])) * 1e6}
    return out or None


def memory_report(ex, cfg, config, recompute, used):
    """Allocated device bytes by category (== the host-side plan), the device's used bytes (incl.
    CUDA context and NCCL buffers), and the reference's analytic total_memory / feasible for the
    same config on the B200 preset (memory.cpp:72-86)."""
    from paper_2211_05953_b200 import pipesim as ps
    from paper_2211_05953_b200.executor import memory_plan
    m = ps.ModelSpec(n_layers=cfg.n_layers, s_hidden=cfg.s_hidden, n_heads=cfg.n_heads, s_seq=cfg.s_seq,
                     s_voc=cfg.s_voc)
    live = ex.memory()
    plan = memory_plan(cfg, config, ex.rank, recompute=recompute)
    ref = ps.total_memory(m, config)
    b200 = ps.cluster_preset("b200")
    return {"allocated": live, "plan_total": plan["total"], "plan_matches": plan == live, "device_used": used,
            "recompute": recompute,
            "reference_total_memory": {"state": ref.state_bytes, "activation": ref.activation_bytes,
                                       "checkpoint": ref.checkpoint_bytes, "total": ref.total_bytes},
            "reference_feasible_b200": ps.feasible(m, config, b200),
            "allocated_over_reference": live["total"] / ref.total_bytes if ref.total_bytes else None,
            "allocated_frac_of_hbm": live["total"] / b200.mem_capacity}


def _progress(msg):
    if os.environ.get("BFPP_BENCH_VERBOSE"):
        print(f"[rank {os.environ.get('RANK', '0')}] {msg}", file=sys.stderr, flush=True)


def main():
    args = parse()
    if os.environ.get("BFPP_HANG_DUMP_S"):
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["BFPP_HANG_DUMP_S"]), exit=True)
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist
    from paper_2211_05953_b200 import pipesim as ps
    from paper_2211_05953_b200.executor import Executor, comm_ids, measured_timeline
    from paper_2211_05953_b200.model import GPTConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.gpus
    if world != n and world != 1:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {n}")
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    cfg = GPTConfig.preset(args.model)
    pp, dp, loops, n_mb, sched = layout(args, world)
    config = ps.ParallelConfig(n_dp=dp, n_pp=pp, n_loop=loops, n_mb=n_mb, s_mb=args.s_mb,
                               dp_variant=ps.DpVariant[{"dp0": "DP0", "dp_ps": "DP_PS", "dp_fs": "DP_FS"}[args.dp_variant]],
                               schedule=ps.Schedule(SCHEDULES[sched]))
    uids = None
    if world > 1:
        obj = [comm_ids(config) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uids = obj[0]
    ex = Executor(cfg, config, rank=rank, world=world, device=local, uids=uids, lr=1e-4, recompute=args.recompute)
    stream = torch.cuda.ExternalStream(ex.stream_handle)
    T = args.s_mb * cfg.s_seq
    g = torch.Generator(device="cuda").manual_seed(1234 + rank // pp)
    tokens_dev = torch.randint(0, cfg.s_voc, (n_mb, args.s_mb, cfg.s_seq + 1), device="cuda", dtype=torch.int32,
                               generator=g)
    loss_dev = torch.zeros(1, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    _progress('warmup')
    for _ in range(args.warmup):
        ex.step_device(tokens_dev, loss_dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            ex.step_device(tokens_dev, loss_dev)
        e1.record(stream)
        barrier()
    _progress('timed done')
    free_b, total_b = torch.cuda.mem_get_info(local)
    mem_used = total_b - free_b
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    launches_step = sum(v[0] for v in ex.kernel_stats().values())
    tokens_per_step = n_mb * args.s_mb * dp * cfg.s_seq
    value = tokens_per_step / (ms * 1e-3)
    loss_val = float(loss_dev.item())
    if world > 1:  # the loss lives on each replica's last-stage rank: mean over the DP replicas
        last = rank % pp == (pp * loops - 1) % pp
        t = torch.tensor([loss_val if last else 0.0], dtype=torch.float64)
        dist.all_reduce(t)
        loss_val = float(t.item()) / dp

    # ---- end-to-end through the public API: pinned host tokens in, loss out, every step ----
    _progress('e2e start')
    e2e = None
    if not args.no_e2e:
        host = tokens_dev.cpu().pin_memory()
        for _ in range(2):
            ex.step(host)
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            ex.step(host)
        e1.record(stream)
        barrier()
        e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3)) / args.steps
        first_or_last = (rank % pp == 0) or (rank % pp == (pp * loops - 1) % pp)
        h2d = host.numel() * 4 * (1 if first_or_last else 0)
        d2h = 4 if rank % pp == (pp * loops - 1) % pp else 0
        if world > 1:
            t = torch.tensor([h2d, d2h], dtype=torch.float64)
            dist.all_reduce(t)
            h2d, d2h = int(t[0]), int(t[1])
        e2e = {"value": tokens_per_step / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms}

    _progress('diagnostics')
    # ---- untimed diagnostic steps: per-kernel CUDA events, measured timeline ----
    ex.set_flags(record_timeline=False, profile_kernels=True)
    ex.step_device(tokens_dev, loss_dev)
    ex.sync()
    kst = ex.kernel_stats()
    bubble = None
    comm = None
    measured_timing = None
    sim_bubble = None
    replay_bubble = None
    task_replay_bubble = None
    peak_layers = None
    _progress('timeline')
    if not args.no_timeline:
        ex.set_flags(record_timeline=True, profile_kernels=False)
        ex.step_device(tokens_dev, loss_dev)
        ex.sync()
        s, e = ex.task_times()
        if world > 1:
            gathered = [None] * world
            dist.all_gather_object(gathered, (rank, s, e))
        else:
            gathered = [(0, s, e)]
        rep0 = [(st, en) for r, st, en in gathered if r // pp == 0]
        tl = measured_timeline(ex.graph, [a for a, _ in rep0], [b for _, b in rep0])
        bubble = ps.bubble_fraction(tl)
        sim_bubble = (pp - 1) / (n_mb * loops)
        # the same graph simulated with the measured per-kind task durations
        mtm = ps.measured_timing_model(ex.graph, tl)
        replay_bubble = ps.bubble_fraction(ps.simulate(ex.graph, mtm))
        # the same graph replayed with every task's own measured duration: the bubble a zero-overhead
        # executor would show with these task times (measured - this = executor overhead)
        task_replay_bubble = ps.bubble_fraction(
            ps.simulate_durations(ex.graph, [e.end - e.start for e in tl.events]))
        mspec = ps.ModelSpec(n_layers=cfg.n_layers, s_hidden=cfg.s_hidden, n_heads=cfg.n_heads, s_seq=cfg.s_seq,
                             s_voc=cfg.s_voc)
        measured_timing = {"timing_model": dataclasses.asdict(mtm),
                           "rates": dataclasses.asdict(ps.rates_from_timing(mspec, config, mtm))}
        peak_layers = max(ps.peak_inflight(tl, ex.graph, ps.place_stages(ex.model, config)))
        comm = comm_rates(ex, cfg, config, tl, args.s_mb)
    ex.set_flags(False, False)

    pk, pk_kind = peaks()
    gemm_n, gemm_ms, gemm_flops = kst["gemm"]
    achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    step_kernel_ms = sum(v[1] for v in kst.values())
    roofline = {"bound": "tensor", "kernel": "tcgen05 bf16 GEMM (gemm_sm100.cu)", "achieved": achieved,
                "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                "frac": achieved / pk["bf16_tflops_sustained"] if achieved else None,
                "peak_source": f"{pk_kind} bf16_tflops_sustained (kernel timed inside a long step)",
                "traffic": None, "launches_per_step": gemm_n,
                "share_of_kernel_time": gemm_ms / step_kernel_ms if step_kernel_ms else None,
                "kernels": {k: {"launches": v[0], "ms": v[1],
                                "rate": (v[2] / (v[1] * 1e-3) / (1e12 if k in ("gemm", "attention_fwd",
                                                                                "attention_bwd") else 1e9))
                                if v[1] > 0 else None,
                                "rate_unit": "TFLOP/s" if k.startswith(("gemm", "attention")) else "GB/s"}
                            for k, v in kst.items()}}
    traffic_file = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(traffic_file):
        try:
            with open(traffic_file) as f:
                roofline["traffic"] = json.load(f).get("bytes_per_launch")
        except Exception:
            pass

    fpt = cfg.model_flops_per_token()
    mfu = value * fpt / world / SPEC_BF16_FLOPS
    mfu_meas = value * fpt / world / (pk["bf16_tflops"] * 1e12)
    eq11 = ps.compute_per_gpu(ps.ModelSpec(n_layers=cfg.n_layers, s_hidden=cfg.s_hidden, n_heads=cfg.n_heads,
                                           s_seq=cfg.s_seq, s_voc=cfg.s_voc), config) / (ms * 1e-3)
    clocks = clk.summary()
    gpu_launches = launches_step * args.steps
    if world > 1:
        t = torch.tensor([gpu_launches], dtype=torch.float64)
        dist.all_reduce(t)
        gpu_launches = int(t.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        try:
            import cpu_baseline as CB
            smp = CB.SampleStep(cfg)
            smp.run()
            sec = min(smp.run() for _ in range(2))
            tps = smp.tokens_equiv / sec
            cpu = {"value": tps, "unit": "tokens/s", "cores": CB.blas_threads(), "kind": "port",
                   "sample": smp.desc + f"; best of 2 after 1 warm-up, {sec:.2f} s per sample"}
            from paper_2211_05953_b200 import _native as NN
            mspec = ps.ModelSpec(n_layers=cfg.n_layers, s_hidden=cfg.s_hidden, n_heads=cfg.n_heads,
                                 s_seq=cfg.s_seq, s_voc=cfg.s_voc)
            sp = CB.reference_schedule_path(mspec._c(), config._c(), NN.TimingModelC(1.0, 2.0, 0.0, 0.0, 0.0, 0.0))
            if sp:
                cpu["reference_schedule_path"] = sp
            # the reference's own CPU search (rank_configs, simulate scoring) on all host threads
            ss = CB.reference_search_path(mspec._c(), 8, os.cpu_count() or 1)
            if ss:
                cpu["reference_search_path"] = ss
        except Exception as exc:  # the baseline must never break the bench line
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": "tokens/sec", "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config_dict(args, cfg, pp, dp, loops, n_mb, sched),
            "mfu": {"vs_spec_2250TF": mfu, "vs_measured_burst": mfu_meas,
                    "model_flops_per_token": fpt, "eq11_tflops_per_gpu": eq11 / 1e12},
            "bubble_fraction": {"measured": bubble, "eq7": sim_bubble,
                                "simulated_with_measured_timing": replay_bubble,
                                "simulated_with_measured_task_durations": task_replay_bubble,
                                "peak_inflight_layers_measured": peak_layers},
            "loss": loss_val,
            "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clocks, "roofline": roofline,
            "cpu_baseline": cpu,
            "device_bytes_per_rank": ex.device_bytes,
            "memory": memory_report(ex, cfg, config, args.recompute, mem_used),
            "comm": comm,
            "measured_timing": measured_timing,
            "executor_options": {
                "defer_wgrad": pp >= 2 and not args.recompute and os.environ.get("BFPP_DEFER_WGRAD", "1") != "0"
                and os.environ.get("BFPP_WGRAD_STREAM", "0") == "0",
                "lazy_token_table_update": dp == 1 and os.environ.get("BFPP_LAZY_WTE", "1") != "0",
                "gemm_tile_schedule": "dynamic" if os.environ.get("BFPP_GEMM_DYN") == "1" else "static",
                "dp_copy_engine_allgather": dp >= 2 and os.environ.get("BFPP_DP_CE_ALLGATHER") == "1"},
        }
        print(json.dumps(line), flush=True)
    ex.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
