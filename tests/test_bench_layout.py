"""bench.py's parallel layouts (host only): BASELINE configs[1] at 1/2/4/8 GPUs, weak scaling,
and every layout is a valid reference configuration whose graph builds."""
import argparse
import importlib.util
import os

import pytest

import paper_2211_05953_b200 as ps
from paper_2211_05953_b200.model import GPTConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)


def _args(**kw):
    a = dict(gpus=1, steps=10, warmup=3, impl="ours", model="gpt-1.3b", schedule="breadth_first", beta=1, pp=None,
             loops=4, dp_variant="dp_fs", s_mb=1)
    a.update(kw)
    return argparse.Namespace(**a)


@pytest.mark.parametrize("n,want", [(1, (1, 1, 4, 1)), (2, (2, 1, 4, 2)), (4, (2, 2, 4, 2)), (8, (2, 4, 4, 2))])
def test_default_layouts_are_baseline_config1(n, want):
    pp, dp, loops, n_mb, sched = bench.layout(_args(gpus=n), n)
    assert (pp, dp, loops, n_mb) == want and sched == "breadth_first"
    # one sequence per GPU: tokens per step grow with the GPU count (weak scaling)
    assert n_mb * dp == n


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("schedule", ["breadth_first", "depth_first", "1f1b", "gpipe"])
def test_layouts_build_valid_graphs(n, schedule):
    a = _args(gpus=n, schedule=schedule, beta=2)
    pp, dp, loops, n_mb, sched = bench.layout(a, n)
    cfg = GPTConfig.preset("gpt-1.3b")
    model = ps.ModelSpec(n_layers=cfg.n_layers, s_hidden=cfg.s_hidden, n_heads=cfg.n_heads, s_seq=cfg.s_seq,
                         s_voc=cfg.s_voc)
    config = ps.ParallelConfig(n_dp=dp, n_pp=pp, n_loop=loops, n_mb=n_mb, dp_variant=ps.DpVariant.DP_FS,
                               schedule=ps.Schedule(bench.SCHEDULES[sched]))
    g = ps.build_tasks(model, config)
    assert len(g.compute_program) == pp
    assert sum(len(p) for p in g.compute_program) == 2 * pp * loops * n_mb
