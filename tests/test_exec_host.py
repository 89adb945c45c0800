"""Executor argument validation (host side, no GPU): the checks run before any CUDA call."""
import pytest

import paper_2211_05953_b200 as ps
from paper_2211_05953_b200.executor import Executor, accumulation_config, model_spec
from paper_2211_05953_b200.model import GPTConfig

TINY = GPTConfig.preset("tiny")


def test_accumulation_graph_needs_data_parallel_ranks():
    g = ps.build_accumulation_tasks(model_spec(TINY), ps.DpVariant.DP_FS, ps.AccumulationOrder.BreadthFirst, 2)
    with pytest.raises(ps.SpecError, match="data-parallel tasks but n_dp < 2"):
        Executor(TINY, accumulation_config(TINY, ps.DpVariant.DP_FS, 2, 1), graph=g)


def test_graph_must_match_config():
    g = ps.build_accumulation_tasks(model_spec(TINY), ps.DpVariant.DP_FS, ps.AccumulationOrder.BreadthFirst, 3)
    with pytest.raises(ps.SpecError, match="micro-batch"):  # config says 2 micro-batches, graph has 3
        Executor(TINY, accumulation_config(TINY, ps.DpVariant.DP_FS, 2, 2), rank=0, world=2, graph=g)
    g2 = ps.build_tasks(model_spec(TINY), ps.ParallelConfig(n_pp=2, n_loop=2, n_mb=2,
                                                            schedule=ps.Schedule.BreadthFirst))
    with pytest.raises(ps.SpecError, match="devices"):
        Executor(TINY, accumulation_config(TINY, ps.DpVariant.DP_FS, 2, 2), rank=0, world=2, graph=g2)


def test_executor_rejects_tensor_parallel_and_rank_mismatch():
    with pytest.raises(ps.SpecError, match="number of ranks"):
        Executor(TINY, ps.ParallelConfig(n_dp=2, n_pp=1, n_mb=1), rank=0, world=1)
