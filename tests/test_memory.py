"""Memory: the reference's analytic model restated (total_memory / feasible / cluster_preset,
memory.cpp:7-86, types.cpp:206-231) checked against the compiled reference, and the executor's own
per-rank allocation plan (bfpp_exec_memory_plan: its allocation code in sizing mode, no GPU)
checked against the paper's structure (pooled activation sets = peak_inflight, checkpoints of
2 s h bytes under recompute, one pooled gradient buffer under DP_FS) and against HBM capacity."""
import ctypes as C
import itertools

import pytest

import ref_oracle as R
from paper_2211_05953_b200 import _native as N
from paper_2211_05953_b200 import pipesim as ps
from paper_2211_05953_b200.executor import memory_plan, model_spec
from paper_2211_05953_b200.model import GPTConfig

S, V = ps.Schedule, ps.DpVariant
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")


def _grid():
    models = [ps.ModelSpec(n_layers=16, s_hidden=1024, n_heads=16, s_seq=1024, s_voc=30592),
              ps.ModelSpec(n_layers=64, s_hidden=8192, n_heads=64, s_seq=1024, s_voc=30592)]
    for m, p, v, mb, dv, sc in itertools.product(models, (1, 2, 4), (1, 2), (1, 4, 8), list(V),
                                                 (S.NoPipeline, S.GPipe, S.OneFOneB, S.DepthFirst, S.BreadthFirst)):
        if v > 1 and sc not in (S.DepthFirst, S.BreadthFirst):
            continue
        if p == 1 and sc in (S.GPipe, S.OneFOneB):
            continue
        if sc == S.NoPipeline and (p > 1 or v > 1):
            continue
        if sc == S.DepthFirst and mb % p:
            continue
        try:
            c = ps.ParallelConfig(n_dp=2, n_pp=p, n_loop=v, n_mb=mb, dp_variant=dv, schedule=sc)
        except ps.SpecError:
            continue
        yield m, c


@needs_ref
def test_total_memory_matches_reference():
    L = R.ref()
    n = 0
    for m, c in _grid():
        for dp0 in (12.0, 20.0):
            ours = ps.total_memory(m, c, ps.MemoryOptions(dp0_bytes_per_param=dp0))
            out = (C.c_double * 4)()
            assert L.ref_total_memory(C.byref(m._c()), C.byref(c._c()), dp0, out) == 0
            assert (ours.state_bytes, ours.activation_bytes, ours.checkpoint_bytes, ours.total_bytes) == tuple(out)
            for cap, head in ((80.0 * 2 ** 30, 0.85), (180e9, 0.85), (32.0 * 2 ** 30, 0.5)):
                r = C.c_int32()
                assert L.ref_feasible(C.byref(m._c()), C.byref(c._c()), cap, dp0, head, C.byref(r)) == 0
                k = ps.ClusterSpec(1, 8, 1.0, 1.0, 1.0, mem_capacity=cap)
                assert ps.feasible(m, c, k, ps.MemoryOptions(dp0, head)) == bool(r.value)
            n += 1
    assert n > 50


@needs_ref
def test_cluster_presets_match_reference():
    L = R.ref()
    for name in ("a100", "v100-dgx1"):
        k = N.ClusterSpecC()
        assert L.ref_cluster_preset(name.encode(), C.byref(k)) == 0
        ours = ps.cluster_preset(name)
        assert ours == ps.ClusterSpec(k.n_node, k.s_node, k.peak_flops, k.bw_intra, k.bw_inter, k.pp_latency,
                                      k.mem_capacity, k.kernel_efficiency)
    b = ps.cluster_preset("b200")
    assert (b.n_gpu(), b.peak_flops, b.mem_capacity) == (8, 2.25e15, 180e9)
    with pytest.raises(ps.SpecError):
        ps.cluster_preset("h100")


def _per_rank(cfg, c, **kw):
    return [memory_plan(cfg, c, r, **kw) for r in range(c.n_pp * c.n_dp)]


def test_52b_fully_sharded_fits_b200():
    """BASELINE configs[4]: 52B (64 layers, h 8192), PP4 x 2 loops x DP2 fully sharded, breadth-first,
    one sequence per GPU, with activation checkpoints: every rank within 0.85 x 180 GB (the
    reference's headroom, memory.cpp:82-86), which the round-1 layout (a full f32 gradient per
    local stage, a landing buffer per stage, all activations) exceeded at ~219 GB of state alone."""
    cfg = GPTConfig.preset("52b")
    b200 = ps.cluster_preset("b200")
    c = ps.ParallelConfig(n_dp=2, n_pp=4, n_loop=2, n_mb=4, dp_variant=V.DP_FS, schedule=S.BreadthFirst)
    plans = _per_rank(cfg, c, recompute=True)
    worst = max(p["total"] for p in plans)
    assert worst <= 0.85 * b200.mem_capacity, worst / 1e9
    for p in plans:
        # fp32 master + m + v of this rank's 1/8 of the model (the part no layout can shrink)
        assert p["optimizer"] > 0.5 * p["total"]
        # one pooled f32 gradient buffer of the largest local stage (not one per stage)
        assert p["grads"] < 0.2 * p["total"]
    # without checkpoints the activations alone push the same layout past the limit
    assert max(p["total"] for p in _per_rank(cfg, c, recompute=False)) > 0.85 * b200.mem_capacity
    # more loops = smaller stages = smaller reconstruction slots and gradient buffer
    c4 = ps.ParallelConfig(n_dp=2, n_pp=4, n_loop=4, n_mb=8, dp_variant=V.DP_FS, schedule=S.BreadthFirst)
    assert max(p["total"] for p in _per_rank(cfg, c4, recompute=True)) < worst


@pytest.mark.parametrize("sched,p,v,mb", [(S.BreadthFirst, 2, 2, 4), (S.DepthFirst, 2, 2, 4), (S.DepthFirst, 2, 2, 8),
                                          (S.OneFOneB, 4, 1, 8), (S.GPipe, 2, 1, 4), (S.NoPipeline, 1, 1, 3)])
def test_activation_pool_is_peak_inflight(sched, p, v, mb):
    """The pooled activation sets of each rank equal the reference's peak_inflight (live
    checkpointed stages, simulate.cpp:166-191) divided by layers per stage."""
    cfg = GPTConfig.preset("tiny")
    m = model_spec(cfg)
    m = ps.ModelSpec(n_layers=8, s_hidden=m.s_hidden, n_heads=m.n_heads, s_seq=m.s_seq, s_voc=m.s_voc)
    c = ps.ParallelConfig(n_pp=p, n_loop=v, n_mb=mb, schedule=sched)
    pl = ps.place_stages(m, c)
    g = ps.build_tasks(m, c, pl)
    tl = ps.simulate(g, ps.TimingModel(t_fwd_stage=1.0, bwd_ratio=2.0, t_pp_transfer=0.1))
    peak = ps.peak_inflight(tl, g, pl)
    for d in range(p):
        plan = memory_plan(m, c, d)
        assert plan["activation_sets"] * pl.layers_per_stage == peak[d], (d, plan, peak)


def test_recompute_keeps_checkpoints_only():
    """Under recompute an activation set holds one 2 T h-byte checkpoint per layer (the reference's
    per-checkpoint size, memory.cpp:64-70) and the per-layer working set lives in scratch once."""
    cfg = GPTConfig.preset("gpt-1.3b")
    c = ps.ParallelConfig(n_pp=2, n_loop=4, n_mb=4, schedule=S.BreadthFirst)
    T, h = c.s_mb * cfg.s_seq, cfg.s_hidden
    for rank in range(2):
        full, rc = memory_plan(cfg, c, rank), memory_plan(cfg, c, rank, recompute=True)
        lps = cfg.n_layers // (c.n_pp * c.n_loop)
        ckpt = rc["activation_sets"] * lps * 2 * T * h
        emb = 2 * T * h * c.n_mb if rank == 0 else 0  # stage-0 embedding outputs (layer-0 inputs)
        assert rc["activations"] == ckpt + emb
        assert full["activations"] > 8 * rc["activations"]
        assert rc["total"] < full["total"]


def test_reference_model_vs_executor_plan():
    """The reference's DP_FS state term (8 P / L: two bf16 layers of weights + gradients on an
    'arbitrarily large' DP group) leaves out the fp32 master / Adam shard that
    dominates a 2-way DP group: the executor's real per-rank bytes are far above total_memory."""
    cfg = GPTConfig.preset("52b")
    m = model_spec(cfg)
    c = ps.ParallelConfig(n_dp=2, n_pp=4, n_loop=2, n_mb=4, dp_variant=V.DP_FS, schedule=S.BreadthFirst)
    ref = ps.total_memory(m, c)
    ours = max(p["total"] for p in _per_rank(cfg, c, recompute=True))
    assert ours > 10 * ref.total_bytes
    assert ps.feasible(m, c, ps.cluster_preset("b200"))


def test_deferred_wgrad_and_lazy_table_scratch(monkeypatch):
    """The per-layer gradient scratch of deferred weight gradients (n_pp >= 2: dpre, dqkv, gmid, gout
    per layer of a stage) and the lazy token-table update's row marks / list (n_dp = 1, the rank of
    stage 0) are in the plan, with exactly these sizes; the A/B switches remove them."""
    cfg = GPTConfig.preset("gpt-1.3b")
    T, h, mlp, V = cfg.s_seq, cfg.s_hidden, cfg.s_mlp, cfg.s_voc
    c = ps.ParallelConfig(n_pp=2, n_loop=4, n_mb=2, schedule=S.BreadthFirst)
    lps = cfg.n_layers // (c.n_pp * c.n_loop)

    def rnd(n):  # the executor's allocator rounds each buffer up to >= 256 bytes
        return max(n, 256)

    defer_bytes = lps * (rnd(2 * T * mlp) + rnd(2 * 3 * T * h) + 2 * rnd(2 * T * h))
    lazy_bytes = rnd(4 * V) + rnd(4 * c.n_mb * T) + rnd(4)
    base = {}
    for defer in ("1", "0"):
        for lazy in ("1", "0"):
            monkeypatch.setenv("BFPP_DEFER_WGRAD", defer)
            monkeypatch.setenv("BFPP_LAZY_WTE", lazy)
            base[defer, lazy] = [memory_plan(cfg, c, r)["scratch"] for r in range(2)]
    for r in range(2):
        assert base["1", "0"][r] - base["0", "0"][r] == defer_bytes
        lazy_here = lazy_bytes if r == 0 else 0  # stage 0 lives on rank 0
        assert base["0", "1"][r] - base["0", "0"][r] == lazy_here
        assert base["1", "1"][r] - base["0", "0"][r] == defer_bytes + lazy_here
    # recompute keeps one working set per rank: no deferral scratch
    monkeypatch.setenv("BFPP_DEFER_WGRAD", "1")
    monkeypatch.setenv("BFPP_LAZY_WTE", "0")
    rc = memory_plan(cfg, c, 1, recompute=True)["scratch"]
    monkeypatch.setenv("BFPP_DEFER_WGRAD", "0")
    assert memory_plan(cfg, c, 1, recompute=True)["scratch"] == rc
