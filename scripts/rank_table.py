"""Ranked configuration table for GPT-6.7B on one 8 x B200 node: the reference's
simulate scoring (TimingModel::derive on the b200 preset) next to measured scoring (per-kind task
costs from a B200 run, carried to every candidate by rates_from_timing / timing_from_rates).

    python scripts/rank_table.py profiles/r02_sweep_pp2dp2.jsonl > profiles/r02_rank_configs_gpt6.7b.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05953_b200 import pipesim as ps  # noqa: E402

S, V = ps.Schedule, ps.DpVariant
NAMES = {0: "no_pipeline", 1: "gpipe", 2: "1f1b", 3: "depth_first", 4: "breadth_first"}


def measured_rates(path):
    """Rates of the breadth-first beta = 2 point of a sweep file (its measured timing model)."""
    for line in open(path):
        d = json.loads(line)
        if d.get("sweep_schedule") == "breadth_first" and d.get("sweep_beta") == 2 and d.get("measured_timing"):
            r = d["measured_timing"]["rates"]
            return ps.MeasuredRates(**r), d["config"]["parallelism"], d["value"]
    raise SystemExit("no breadth_first beta=2 point with a measured timing in " + path)


def main():
    path = sys.argv[1]
    rates, where, tps = measured_rates(path)
    model = ps.ModelSpec(n_layers=32, s_hidden=4096, n_heads=32, s_seq=2048, s_voc=50304)
    k = ps.cluster_preset("b200")
    space = dict(schedules=[1, 2, 3, 4], dp_variants=[0, 1, 2], n_pp=[1, 2, 4, 8], s_mb=[1],
                 n_mb=[2, 4, 8, 16], n_loop=[1, 2, 4], batch_sizes=[8, 16])
    sim = ps.rank_configs(model, k, threads=0, **space)
    meas = ps.rank_configs(model, k, scoring="measured", rates=rates, threads=0, **space)
    print("# GPT-6.7B on one 8 x B200 node: ranked configurations\n")
    print(f"Measured rates from `{os.path.basename(path)}` (breadth-first, {where}, beta 2, {tps:,.0f} tok/s "
          f"on 4 B200s): forward {rates.fwd_layer_seq * 1e3:.3f} ms per layer per sequence, backward/forward "
          f"{rates.bwd_ratio:.2f}, hand-off {1 / rates.pp_s_per_byte / 1e9:.0f} GB/s, DP reduce "
          f"{rates.reduce_s_per_param * 1e12:.2f} ps/param, reconstruct {rates.reconstruct_s_per_param * 1e12:.2f} "
          "ps/param.\n")
    print("Search space: GPipe / 1F1B / looped DF / BF x DP0 / DP_PS / DP_FS (the reference's sharding policy) "
          "x n_pp {1,2,4,8} x n_mb {2,4,8,16} x loops {1,2,4}, s_mb 1, batch 8 or 16 sequences (beta 1 / 2); "
          "feasibility = the reference's total_memory on the b200 preset.\n")
    for name, ranked in (("measured scoring", meas), ("simulate scoring (reference, TimingModel::derive)", sim)):
        for batch in (8, 16):
            rows = [r for r in ranked if r.config.batch_size() == batch][:12]
            print(f"## {name}, batch {batch} (beta {batch // 8})\n")
            print("| rank | schedule | DP variant | PP x loops x DP | n_mb | tok/s/GPU | MFU (spec) | bubble |")
            print("|---|---|---|---|---|---|---|---|")
            fpt = 72 * 32 * 4096 ** 2 + 12 * 32 * 2048 * 4096 + 6 * 4096 * 50304
            for i, r in enumerate(rows, 1):
                c = r.config
                tok = r.score / ps.compute_per_gpu(model, c) * c.batch_size() * 2048 / 8 if r.score else 0
                print(f"| {i} | {NAMES[int(c.schedule)]} | {c.dp_variant.name} | {c.n_pp} x {c.n_loop} x {c.n_dp} | "
                      f"{c.n_mb} | {tok:,.0f} | {tok * fpt / 2.25e15:.3f} | {r.bubble:.3f} |")
            print()
        best = {}
        for r in ranked:
            best.setdefault((int(r.config.schedule), r.config.batch_size()), r)
        print(f"Best per schedule ({name}):\n")
        print("| schedule | batch 8 tok/s/GPU | batch 16 tok/s/GPU |")
        print("|---|---|---|")
        for s in (4, 3, 2, 1):
            cells = []
            for batch in (8, 16):
                r = best.get((s, batch))
                cells.append(f"{r.score / ps.compute_per_gpu(model, r.config) * batch * 2048 / 8:,.0f}" if r else "-")
            print(f"| {NAMES[s]} | {cells[0]} | {cells[1]} |")
        print()


if __name__ == "__main__":
    main()
