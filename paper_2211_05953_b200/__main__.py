"""Command line: the reference CLI's `simulate` (tools/pipesim.cpp:60-91) plus `execute`.

  python -m paper_2211_05953_b200 simulate --model gpt-6.7b --schedule breadth_first --pp 4 --loops 2 \\
      --dp 2 --n-mb 8 [--trace t.json] [--gantt g.svg]
  python -m paper_2211_05953_b200 execute  --model gpt-1.3b --schedule breadth_first --pp 1 --loops 4 \\
      --n-mb 1 --steps 5 [--trace t.json] [--gantt g.svg]
  (N > 1 ranks: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 -m paper_2211_05953_b200 execute ...)

  python -m paper_2211_05953_b200 search --model gpt-6.7b --cluster b200 --batch 8 16 \
      [--scoring measured --rates-from bench_line.json] [--top 20]

`search` ranks the feasible configurations of a search space like the reference's `rank_configs`
(search.cpp:136-188; simulate scoring = TimingModel::derive), or with per-kind task costs
measured on B200s (`--scoring measured`: the `measured_timing.rates` of a bench.py JSON line, or
--rates f,b,pp,lat,red,rec), printing one CSV row per configuration; exit 3 when nothing is
feasible (the reference's empty-result code).
`simulate` prints the reference's summary lines (makespan, bubble, peak in-flight layers, lane busy
times; report.cpp:214-232) for the analytic timing model; `execute` runs the same task graph on the local B200(s),
prints the measured step time, tokens/s, the measured bubble fraction and the bubble of the
graph simulated with the measured per-kind task durations, and writes the measured timeline as
a Chrome trace / Gantt chart. Exit codes follow the reference CLI: 2 spec error, 4 execution error.
"""
from __future__ import annotations

import argparse
import os
import sys

from . import pipesim as ps
from .model import PRESETS, GPTConfig

SCHEDULES = {"no_pipeline": ps.Schedule.NoPipeline, "gpipe": ps.Schedule.GPipe, "1f1b": ps.Schedule.OneFOneB,
             "depth_first": ps.Schedule.DepthFirst, "breadth_first": ps.Schedule.BreadthFirst}
VARIANTS = {"dp0": ps.DpVariant.DP0, "dp_ps": ps.DpVariant.DP_PS, "dp_fs": ps.DpVariant.DP_FS}


def _args(argv):
    ap = argparse.ArgumentParser(prog="python -m paper_2211_05953_b200")
    ap.add_argument("command", choices=["simulate", "execute", "search"])
    ap.add_argument("--model", default="gpt-1.3b", choices=sorted(PRESETS))
    ap.add_argument("--schedule", default="breadth_first", choices=sorted(SCHEDULES))
    ap.add_argument("--dp-variant", default="dp_fs", choices=sorted(VARIANTS))
    ap.add_argument("--pp", type=int, default=1)
    ap.add_argument("--loops", type=int, default=1)
    ap.add_argument("--dp", type=int, default=1)
    ap.add_argument("--n-mb", type=int, default=1)
    ap.add_argument("--s-mb", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5, help="execute: timed steps (after 3 warm-up steps)")
    ap.add_argument("--t-fwd", type=float, default=1.0, help="simulate: forward time of one stage")
    ap.add_argument("--bwd-ratio", type=float, default=2.0)
    ap.add_argument("--t-pp", type=float, default=0.0)
    ap.add_argument("--t-reduce", type=float, default=0.0)
    ap.add_argument("--t-reconstruct", type=float, default=0.0)
    ap.add_argument("--trace", help="write the (simulated / measured) timeline as Chrome trace JSON")
    ap.add_argument("--gantt", help="write the timeline as an SVG Gantt chart")
    # search
    ap.add_argument("--cluster", default="b200", help="search: cluster preset (a100, v100-dgx1, b200)")
    ap.add_argument("--gpus", type=int, default=None, help="search: GPUs per node (overrides the preset)")
    ap.add_argument("--schedules", nargs="+", default=["gpipe", "1f1b", "depth_first", "breadth_first"])
    ap.add_argument("--variants", nargs="+", default=["dp0", "dp_ps", "dp_fs"])
    ap.add_argument("--pp-choices", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--loop-choices", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--mb-choices", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32])
    ap.add_argument("--smb-choices", type=int, nargs="+", default=[1])
    ap.add_argument("--batch", type=int, nargs="+", default=[8, 16])
    ap.add_argument("--scoring", default="simulate", choices=["simulate", "measured"])
    ap.add_argument("--rates-from", help="search: bench.py JSON line(s); the last measured_timing.rates is used")
    ap.add_argument("--rates", type=float, nargs=6, help="search: fwd_layer_seq bwd_ratio pp_s_per_byte "
                                                          "pp_latency reduce_s_per_param reconstruct_s_per_param")
    ap.add_argument("--top", type=int, default=0, help="search: print only the best N per batch size")
    return ap.parse_args(argv)


def _write(path, text):
    if path:
        with open(path, "w") as f:
            f.write(text)


def _summary(model, config, graph, tl):
    pl = ps.place_stages(model, config)
    peak = max(ps.peak_inflight(tl, graph, pl))  # live checkpointed layers
    print(f"makespan_seconds,{tl.makespan:.9f}")
    print(f"bubble_fraction,{ps.bubble_fraction(tl):.9f}")
    print(f"peak_inflight_layers,{peak}")
    for d in range(tl.n_devices):
        print(f"busy_device{d}," + ",".join(f"{n}={v:.9f}" for n, v in zip(("compute", "dp-net", "pp-net"),
                                                                           tl.lane_busy[d])))


def main(argv=None) -> int:
    a = _args(argv if argv is not None else sys.argv[1:])
    cfg = GPTConfig.preset(a.model)
    model = ps.ModelSpec(n_layers=cfg.n_layers, s_hidden=cfg.s_hidden, n_heads=cfg.n_heads, s_seq=cfg.s_seq,
                         s_voc=cfg.s_voc)
    config = ps.ParallelConfig(n_dp=a.dp, n_pp=a.pp, n_loop=a.loops, n_mb=a.n_mb, s_mb=a.s_mb,
                               dp_variant=VARIANTS[a.dp_variant], schedule=SCHEDULES[a.schedule])
    try:
        if a.command == "simulate":
            graph = ps.build_tasks(model, config)
            tl = ps.simulate(graph, ps.TimingModel(a.t_fwd, a.bwd_ratio, a.t_pp, 0.0, a.t_reduce, a.t_reconstruct))
            _summary(model, config, graph, tl)
            _write(a.trace, ps.chrome_trace_json(tl, graph))
            _write(a.gantt, ps.gantt_svg(tl, graph))
            return 0
        if a.command == "search":
            return _search(a, model)
        return _execute(a, cfg, model, config)
    except ps.SpecError as e:
        print(e, file=sys.stderr)
        return 2
    except ps.SimError as e:
        print(e, file=sys.stderr)
        return 4


def _search(a, model) -> int:
    import json
    k = ps.cluster_preset(a.cluster)
    if a.gpus:
        k = ps.ClusterSpec(1, a.gpus, k.peak_flops, k.bw_intra, k.bw_inter, k.pp_latency, k.mem_capacity,
                           k.kernel_efficiency)
    rates = None
    if a.scoring == "measured":
        if a.rates:
            rates = ps.MeasuredRates(*a.rates)
        elif a.rates_from:
            for line in open(a.rates_from):
                line = line.strip()
                if line.startswith("{") and '"measured_timing"' in line:
                    mt = json.loads(line).get("measured_timing")
                    if mt:
                        rates = ps.MeasuredRates(**mt["rates"])
        if rates is None:
            raise ps.SpecError("error[invalid-spec]: search: measured scoring needs --rates or --rates-from "
                               "with a measured_timing line")
    ranked = ps.rank_configs(model, k, schedules=[int(SCHEDULES[x]) for x in a.schedules],
                             dp_variants=[int(VARIANTS[x]) for x in a.variants], n_pp=a.pp_choices,
                             s_mb=a.smb_choices, n_mb=a.mb_choices, n_loop=a.loop_choices, batch_sizes=a.batch,
                             scoring=a.scoring, rates=rates)
    if not ranked:
        print("pipesim: error[empty-result]: every configuration of the search space is infeasible", file=sys.stderr)
        return 3
    names = {v: n for n, v in SCHEDULES.items()}
    print("rank,batch,schedule,dp_variant,n_pp,n_loop,n_dp,n_mb,s_mb,flops_per_gpu,tokens_per_second_per_gpu,"
          "bubble,memory_bytes")
    shown = {}
    for i, r in enumerate(ranked, 1):
        c = r.config
        if a.top and shown.get(c.batch_size(), 0) >= a.top:
            continue
        shown[c.batch_size()] = shown.get(c.batch_size(), 0) + 1
        tok = r.score / ps.compute_per_gpu(model, c) * c.batch_size() * model.s_seq / k.n_gpu()
        print(f"{i},{c.batch_size()},{names[c.schedule]},{c.dp_variant.name},{c.n_pp},{c.n_loop},{c.n_dp},{c.n_mb},"
              f"{c.s_mb},{r.score:.6e},{tok:.1f},{r.bubble:.6f},{r.memory_bytes:.0f}")
    return 0


def _execute(a, cfg, model, config) -> int:
    import torch
    import torch.distributed as dist

    from .executor import Executor, comm_ids, measured_timeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != config.n_dp * config.n_pp:
        raise ps.SpecError(f"error[invalid-spec]: execute: {world} ranks for n_dp * n_pp = "
                           f"{config.n_dp * config.n_pp}")
    uids = None
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        obj = [comm_ids(config) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uids = obj[0]
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ex = Executor(cfg, config, rank=rank, world=world, device=local, uids=uids)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank // config.n_pp)
    tokens = torch.randint(0, cfg.s_voc, (config.n_mb, config.s_mb, cfg.s_seq + 1), device="cuda",
                           dtype=torch.int32, generator=g)
    loss = torch.zeros(1, device="cuda")
    for _ in range(3):
        ex.step_device(tokens, loss)
    ex.sync()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.ExternalStream(ex.stream_handle)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        ex.step_device(tokens, loss)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    ex.set_flags(record_timeline=True)
    ex.step_device(tokens, loss)
    ex.sync()
    s, e = ex.task_times()
    gathered = [(rank, s, e)]
    times = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, s, e))
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    if rank == 0:
        rep0 = [(st, en) for r, st, en in gathered if r // config.n_pp == 0]
        tl = measured_timeline(ex.graph, [x for x, _ in rep0], [y for _, y in rep0])
        replay = ps.simulate(ex.graph, ps.measured_timing_model(ex.graph, tl))
        tokens_per_step = config.n_dp * config.n_mb * config.s_mb * cfg.s_seq
        ms = float(times.item())
        print(f"step_ms,{ms:.4f}")
        print(f"tokens_per_second,{tokens_per_step / (ms * 1e-3):.1f}")
        print(f"loss,{float(loss.item()):.6f}" if config.n_pp == 1 else "loss,(last-stage rank)")
        _summary(model, config, ex.graph, tl)
        print(f"bubble_fraction_simulated_with_measured_timing,{ps.bubble_fraction(replay):.9f}")
        _write(a.trace, ps.chrome_trace_json(tl, ex.graph))
        _write(a.gantt, ps.gantt_svg(tl, ex.graph))
    ex.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
