"""Executor numerics vs the CPU oracle on one B200 (tiny GPT), every schedule
that fits one device, plus timeline/metric checks. Tolerances: tests/exec_harness.compare."""
import numpy as np
import pytest

import exec_harness as H
from paper_2211_05953_b200 import pipesim as ps

pytestmark = pytest.mark.gpu
S = ps.Schedule

CONFIGS = {
    "nopipe_mb4": ps.ParallelConfig(n_mb=4, schedule=S.NoPipeline),
    "bf_loop4_mb3": ps.ParallelConfig(n_mb=3, n_loop=4, schedule=S.BreadthFirst),
    "df_loop2_mb2": ps.ParallelConfig(n_mb=2, n_loop=2, schedule=S.DepthFirst),
    "gpipe_mb2_smb2": ps.ParallelConfig(n_mb=2, s_mb=2, schedule=S.GPipe),
    "1f1b_mb2": ps.ParallelConfig(n_mb=2, schedule=S.OneFOneB),
}


SMALL = H.GPTConfig.preset("small")
# production kernel paths inside the composed step (kernel variant -> minimum launches)
PROD = {"gemm_2cta": 1, "gemm_2cta_pair": 1, "attn_fwd_multi": 1, "attn_bwd_multi": 1}
SMALL_CONFIGS = {
    "small_bf_loop2_mb2_smb2": ps.ParallelConfig(n_mb=2, s_mb=2, n_loop=2, schedule=S.BreadthFirst),
    "small_df_loop2_mb2": ps.ParallelConfig(n_mb=2, n_loop=2, schedule=S.DepthFirst),
    "small_nopipe_mb2_smb2": ps.ParallelConfig(n_mb=2, s_mb=2, schedule=S.NoPipeline),
}


def _variants():
    from paper_2211_05953_b200.executor import kernel_variant_counts
    return kernel_variant_counts()


@pytest.mark.parametrize("name", list(SMALL_CONFIGS))
def test_executor_small_production_kernels(cuda_device, name):
    """Executor vs oracle at a preset where every GEMM takes the 2-CTA path (weight gradients as
    grouped pairs) and attention runs several heads x several 128-row blocks (multi-tile online
    softmax, lazy O rescale, per-head QKV slicing); the launch counters prove those ran."""
    from paper_2211_05953_b200.executor import Executor, kernel_variant_counts
    config = SMALL_CONFIGS[name]
    params, tokens = H.make_case(SMALL, config)
    kernel_variant_counts(reset=True)
    res = H.run_rank(lambda **kw: Executor(SMALL, config, **kw), SMALL, config, params, tokens, 0)
    used = _variants()
    for k, n in PROD.items():
        assert used[k] >= n, (k, used)
    assert used["gemm_1cta"] == 0, used  # every GEMM of this preset is a 2-CTA problem
    rep = H.compare(SMALL, config, [res], params, tokens)
    print(name, used, rep["losses"], max(rep["grad_rel"].values()))


def test_executor_large_vocab_head_raster(cuda_device):
    """LM head with V = 50304: the weight-gradient operand dlogits^T (V x tokens, 103 MB) exceeds
    L2, so the 2-CTA GEMM walks its tiles N-fastest; checked against the oracle in the step."""
    from paper_2211_05953_b200.executor import Executor, kernel_variant_counts
    cfg = H.GPTConfig.preset("small-v50k")
    config = ps.ParallelConfig(n_mb=1, s_mb=2, schedule=S.NoPipeline)
    params, tokens = H.make_case(cfg, config)
    kernel_variant_counts(reset=True)
    res = H.run_rank(lambda **kw: Executor(cfg, config, **kw), cfg, config, params, tokens, 0)
    used = _variants()
    assert used["gemm_2cta_nfast"] >= 1 and used["attn_bwd_multi"] >= 1, used
    rep = H.compare(cfg, config, [res], params, tokens)
    print(used, rep["losses"], max(rep["grad_rel"].values()))


STEP_CONFIGS = {
    "tiny_bf_loop4_mb3": (H.TINY, ps.ParallelConfig(n_mb=3, n_loop=4, schedule=S.BreadthFirst)),
    "small_bf_loop2_mb2_smb2": (SMALL, SMALL_CONFIGS["small_bf_loop2_mb2_smb2"]),
    "small_df_loop2_mb2": (SMALL, SMALL_CONFIGS["small_df_loop2_mb2"]),
}


@pytest.mark.parametrize("name", list(STEP_CONFIGS))
def test_executor_multi_step_matches_oracle(cuda_device, name):
    """Three optimizer steps on one executor (a fresh batch per step) vs the oracle looping
    loss/grad/Adam: per-step losses and the final weights (tolerances: H.compare_steps)."""
    from paper_2211_05953_b200.executor import Executor
    cfg, config = STEP_CONFIGS[name]
    params, tokens = H.make_steps_case(cfg, config, n_steps=3)
    res = H.run_rank_steps(lambda **kw: Executor(cfg, config, **kw), cfg, config, params, tokens, 0)
    rep = H.compare_steps(cfg, config, [res], params, tokens)
    print(name, rep["losses"], min(rep["weights_frac_close"].values()), max(rep["weights_max_dev_lr"].values()))


@pytest.mark.parametrize("name", list(CONFIGS))
def test_executor_matches_oracle(cuda_device, name):
    from paper_2211_05953_b200.executor import Executor
    config = CONFIGS[name]
    cfg = H.TINY
    params, tokens = H.make_case(cfg, config)
    res = H.run_rank(lambda **kw: Executor(cfg, config, **kw), cfg, config, params, tokens, 0)
    rep = H.compare(cfg, config, [res], params, tokens)
    print(name, rep["losses"], max(rep["grad_rel"].values()))


def test_schedules_agree_with_each_other(cuda_device):
    """Same model/batch: every schedule's gradients agree (f32 accumulation, ascending micro-batches)."""
    from paper_2211_05953_b200.executor import Executor
    cfg = H.TINY
    base = ps.ParallelConfig(n_mb=4, schedule=S.NoPipeline)
    params, tokens = H.make_case(cfg, base)
    out = {}
    for name, c in [("np", base), ("bf", ps.ParallelConfig(n_mb=4, n_loop=4, schedule=S.BreadthFirst)),
                    ("df", ps.ParallelConfig(n_mb=4, n_loop=2, schedule=S.DepthFirst))]:
        r = H.run_rank(lambda **kw: Executor(cfg, c, **kw), cfg, c, params, tokens, 0)
        n_stage = c.n_loop
        flat = {}
        for s in range(n_stage):
            flat.update(H.unflatten_stage(r["grads"][s][0], cfg, s, n_stage))
        out[name] = (r["loss"], flat)
    for name in ("bf", "df"):
        assert abs(out[name][0] - out["np"][0]) <= 1e-6 * abs(out["np"][0])
        for k, v in out["np"][1].items():
            np.testing.assert_allclose(out[name][1][k], v, rtol=2e-3, atol=1e-6, err_msg=(name, k))


def test_measured_timeline_contract(cuda_device):
    from paper_2211_05953_b200.executor import Executor, measured_timeline
    cfg = H.TINY
    c = ps.ParallelConfig(n_mb=4, n_loop=4, schedule=S.BreadthFirst)
    params, tokens = H.make_case(cfg, c)
    ex = Executor(cfg, c, record_timeline=True)
    ex.step(tokens[0])
    ex.step(tokens[0])
    s, e = ex.task_times()
    tl = measured_timeline(ex.graph, [s], [e])
    for t in ex.graph.tasks:
        ev = tl.events[t.id]
        assert ev.end >= ev.start >= 0
        for d in t.deps:
            assert tl.events[d].end <= ev.start + 1e-6
    prog = ex.graph.compute_program[0]
    for a, b in zip(prog, prog[1:]):
        assert tl.events[a].end <= tl.events[b].start + 1e-6
    assert 0 <= ps.bubble_fraction(tl) < 1.0


@pytest.mark.gpu
def test_cli_execute_writes_measured_trace(tmp_path, capsys, cuda_device):
    """`python -m paper_2211_05953_b200 execute`: measured timeline -> bubble, replayed bubble, trace, Gantt."""
    import json
    from paper_2211_05953_b200.__main__ import main
    trace, svg = tmp_path / "t.json", tmp_path / "g.svg"
    assert main(["execute", "--model", "tiny", "--pp", "1", "--loops", "2", "--n-mb", "2", "--steps", "2",
                 "--trace", str(trace), "--gantt", str(svg)]) == 0
    out = dict(line.split(",", 1) for line in capsys.readouterr().out.splitlines())
    assert float(out["tokens_per_second"]) > 0 and 0.0 <= float(out["bubble_fraction"]) < 1.0
    assert 0.0 <= float(out["bubble_fraction_simulated_with_measured_timing"]) < 1.0
    doc = json.loads(trace.read_text())
    assert sum(e["ph"] == "X" for e in doc["traceEvents"]) == 2 * 2 * 2  # (fwd + bwd) x 2 stages x 2 mb
    assert svg.read_text().startswith("<svg")


RC_CONFIGS = {
    "tiny_bf_loop2_mb3_rc": (H.TINY, ps.ParallelConfig(n_mb=3, n_loop=2, schedule=S.BreadthFirst)),
    "tiny_df_loop2_mb2_rc": (H.TINY, ps.ParallelConfig(n_mb=2, n_loop=2, schedule=S.DepthFirst)),
    "small_bf_loop2_mb2_smb2_rc": (SMALL, ps.ParallelConfig(n_mb=2, s_mb=2, n_loop=2, schedule=S.BreadthFirst)),
}


@pytest.mark.parametrize("name", list(RC_CONFIGS))
def test_executor_recompute_matches_oracle(cuda_device, name):
    """Activation checkpointing: each layer's forward recomputed from its checkpoint inside the
    backward (and the LM head's logits), gradients and a 3-step trajectory vs the oracle."""
    from paper_2211_05953_b200.executor import Executor
    cfg, config = RC_CONFIGS[name]
    params, tokens = H.make_case(cfg, config)
    res = H.run_rank(lambda **kw: Executor(cfg, config, recompute=True, **kw), cfg, config, params, tokens, 0)
    rep = H.compare(cfg, config, [res], params, tokens)
    params, tokens = H.make_steps_case(cfg, config, n_steps=3)
    res = H.run_rank_steps(lambda **kw: Executor(cfg, config, recompute=True, **kw), cfg, config, params, tokens, 0)
    rep2 = H.compare_steps(cfg, config, [res], params, tokens)
    print(name, rep["losses"], max(rep["grad_rel"].values()), rep2["losses"])


@pytest.mark.parametrize("recompute", [False, True])
def test_executor_memory_matches_plan(cuda_device, recompute):
    """The live executor allocates exactly what the host-side plan (bfpp_exec_memory_plan, no GPU)
    says, category by category."""
    from paper_2211_05953_b200.executor import Executor, memory_plan
    for cfg, config in ((SMALL, ps.ParallelConfig(n_mb=2, n_loop=2, schedule=S.BreadthFirst)),
                        (H.TINY, ps.ParallelConfig(n_mb=4, n_loop=2, schedule=S.DepthFirst))):
        ex = Executor(cfg, config, recompute=recompute)
        live = ex.memory()
        assert live == memory_plan(cfg, config, 0, recompute=recompute)
        assert live["total"] == ex.device_bytes
        ex.close()
