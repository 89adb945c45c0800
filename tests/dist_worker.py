"""TEST INFRASTRUCTURE: one rank of a multi-GPU executor run (launched by torchrun from
tests/test_multi_gpu.py). Writes its run_rank() result to <out>/rank<r>.pkl."""
import argparse
import os
import pickle
import sys
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # one hardware queue per executor stream (see executor.py)

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import exec_harness as H  # noqa: E402
from paper_2211_05953_b200 import pipesim as ps  # noqa: E402

CASES = {
    # BASELINE configs[0]: tiny BF, 2 stages x 2 loops, 4 micro-batches, 2 DP ranks (fully sharded)
    "tiny_bf_pp2x2_dp2_fs": dict(n_dp=2, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP_FS", schedule="BreadthFirst"),
    "bf_pp2x2_mb4": dict(n_dp=1, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP0", schedule="BreadthFirst"),
    "df_pp2x2_mb4": dict(n_dp=1, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP0", schedule="DepthFirst"),
    "gpipe_pp2_mb3": dict(n_dp=1, n_pp=2, n_loop=1, n_mb=3, dp_variant="DP0", schedule="GPipe"),
    "1f1b_pp2_mb4": dict(n_dp=1, n_pp=2, n_loop=1, n_mb=4, dp_variant="DP0", schedule="OneFOneB"),
    "bf_pp1x4_dp2_fs": dict(n_dp=2, n_pp=1, n_loop=4, n_mb=2, dp_variant="DP_FS", schedule="BreadthFirst"),
    "np_dp2_dp0": dict(n_dp=2, n_pp=1, n_loop=1, n_mb=2, dp_variant="DP0", schedule="NoPipeline"),
    "np_dp2_ps": dict(n_dp=2, n_pp=1, n_loop=1, n_mb=2, dp_variant="DP_PS", schedule="NoPipeline"),
    "gpipe_dp2_fs_mb2": dict(n_dp=2, n_pp=1, n_loop=1, n_mb=2, dp_variant="DP_FS", schedule="GPipe"),
    "df_pp2x2_dp2_fs": dict(n_dp=2, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP_FS", schedule="DepthFirst"),
    "bf_pp4x1_mb4": dict(n_dp=1, n_pp=4, n_loop=1, n_mb=4, dp_variant="DP0", schedule="BreadthFirst"),
    "1f1b_pp2_dp2_fs": dict(n_dp=2, n_pp=2, n_loop=1, n_mb=2, dp_variant="DP_FS", schedule="OneFOneB"),
    # four-way data parallelism (the DP group size of bench.py at N = 8)
    "bf_pp1x2_dp4_fs": dict(n_dp=4, n_pp=1, n_loop=2, n_mb=2, dp_variant="DP_FS", schedule="BreadthFirst"),
    "np_dp4_dp0": dict(n_dp=4, n_pp=1, n_loop=1, n_mb=1, dp_variant="DP0", schedule="NoPipeline"),
    # three ranks: layer segments do not split into 8-element slices -> one segment per stage
    "bf_pp1x2_dp3_fs": dict(n_dp=3, n_pp=1, n_loop=2, n_mb=2, dp_variant="DP_FS", schedule="BreadthFirst"),
    # gradient-accumulation graphs (build_accumulation_tasks, schedule.cpp:454-500; PAPER App. C):
    # one layer per stage, data parallel; breadth-first reduces per layer, depth-first per micro-batch
    "acc_bf_dp2_fs_mb3": dict(n_dp=2, n_mb=3, dp_variant="DP_FS", accumulation="BreadthFirst"),
    "acc_df_dp2_fs_mb2": dict(n_dp=2, n_mb=2, dp_variant="DP_FS", accumulation="DepthFirst"),
    "acc_bf_dp2_dp0_mb2": dict(n_dp=2, n_mb=2, dp_variant="DP0", accumulation="BreadthFirst"),
    # three optimizer steps on one executor per rank (receive-slot / flag reuse across steps, the
    # run-ahead ring, per-segment early reduce-scatter + Adam moments from step 2 on)
    "steps3_tiny_bf_pp2x2_dp2_fs": dict(n_dp=2, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP_FS",
                                        schedule="BreadthFirst", steps=3),
    "steps3_tiny_df_pp2x2_dp2_fs": dict(n_dp=2, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP_FS",
                                        schedule="DepthFirst", steps=3),
    "steps3_tiny_bf_pp2x2_mb4": dict(n_dp=1, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP0", schedule="BreadthFirst",
                                     steps=3),
    "steps3_tiny_np_dp2_ps": dict(n_dp=2, n_pp=1, n_loop=1, n_mb=2, dp_variant="DP_PS", schedule="NoPipeline",
                                  steps=3),
    # production kernel paths (2-CTA / grouped GEMMs, multi-head multi-block attention) across GPUs
    "small_bf_pp2x1_dp1_mb2": dict(n_dp=1, n_pp=2, n_loop=1, n_mb=2, s_mb=2, dp_variant="DP0",
                                   schedule="BreadthFirst", model="small"),
    "steps3_small_bf_pp1x2_dp2_fs": dict(n_dp=2, n_pp=1, n_loop=2, n_mb=2, dp_variant="DP_FS",
                                         schedule="BreadthFirst", model="small", steps=3),
    "steps3_small_bf_pp2x1_dp2_fs": dict(n_dp=2, n_pp=2, n_loop=1, n_mb=2, dp_variant="DP_FS",
                                         schedule="BreadthFirst", model="small", steps=3),
    # activation checkpointing (recompute in the backward) with the pooled sharded gradients,
    # pipeline hand-offs and several optimizer steps; and a multi-unit (depth-first) DP_FS stage
    "steps3_tiny_bf_pp2x2_dp2_fs_rc": dict(n_dp=2, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP_FS",
                                           schedule="BreadthFirst", steps=3, recompute=True),
    "tiny_df_pp2x2_dp2_fs_rc": dict(n_dp=2, n_pp=2, n_loop=2, n_mb=4, dp_variant="DP_FS", schedule="DepthFirst",
                                    recompute=True),
    "steps3_small_1f1b_pp2_dp2_fs_rc": dict(n_dp=2, n_pp=2, n_loop=1, n_mb=4, dp_variant="DP_FS",
                                            schedule="OneFOneB", model="small", steps=3, recompute=True),
}


def model_of(name):
    return H.GPTConfig.preset(CASES[name].get("model", "tiny"))


def steps_of(name):
    return CASES[name].get("steps", 0)


def recompute_of(name):
    return CASES[name].get("recompute", False)


def accumulation_graph(name):
    """The gradient-accumulation task graph of an accumulation case (None for build_tasks cases)."""
    c = CASES[name]
    if "accumulation" not in c:
        return None
    from paper_2211_05953_b200.executor import model_spec
    return ps.build_accumulation_tasks(model_spec(model_of(name)), ps.DpVariant[c["dp_variant"]],
                                       ps.AccumulationOrder[c["accumulation"]], c["n_mb"])


def config_of(name):
    c = dict(CASES[name])
    c.pop("model", None)
    c.pop("steps", None)
    c.pop("recompute", None)
    if "accumulation" in c:
        from paper_2211_05953_b200.executor import accumulation_config
        return accumulation_config(model_of(name), ps.DpVariant[c["dp_variant"]], c["n_mb"], c["n_dp"])
    c["dp_variant"] = ps.DpVariant[c["dp_variant"]]
    c["schedule"] = ps.Schedule[c["schedule"]]
    return ps.ParallelConfig(**c)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("BFPP_HANG_DUMP_S", "100")), exit=True)
    import torch
    import torch.distributed as dist
    from paper_2211_05953_b200.executor import Executor, comm_ids
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    config = config_of(a.case)
    cfg = model_of(a.case)
    n_steps = steps_of(a.case)

    def factory(**kw):
        obj = [comm_ids(config) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return Executor(cfg, config, rank=rank, world=world, device=local, uids=obj[0],
                        graph=accumulation_graph(a.case), recompute=recompute_of(a.case), **kw)

    if n_steps:
        params, tokens = H.make_steps_case(cfg, config, n_steps)
        res = H.run_rank_steps(factory, cfg, config, params, tokens, rank)
    else:
        params, tokens = H.make_case(cfg, config)
        res = H.run_rank(factory, cfg, config, params, tokens, rank)
    with open(os.path.join(a.out, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
