"""Configuration search: the reference's enumerate_configs + rank_configs in
simulate mode (search.cpp:62-188) restated, checked against the compiled reference (same configs,
same order, identical scores), and the "measured" scoring mode: candidates simulated with
per-kind task costs measured at one configuration. Given the reference's own derived timing as
the "measurement", measured scoring must reproduce the reference's ranking."""
import ctypes as C

import pytest

import ref_oracle as R
from paper_2211_05953_b200 import _native as N
from paper_2211_05953_b200 import pipesim as ps

S, V = ps.Schedule, ps.DpVariant
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")

SPACES = {
    "gpt6.7b_8gpu": (ps.ModelSpec(n_layers=32, s_hidden=4096, n_heads=32, s_seq=2048, s_voc=50304),
                     dict(schedules=[1, 2, 3, 4], dp_variants=[0, 1, 2], n_pp=[1, 2, 4, 8], s_mb=[1, 2],
                          n_mb=[2, 4, 8, 16, 32], n_loop=[1, 2, 4], batch_sizes=[16, 32, 64])),
    "52b_8gpu": (ps.ModelSpec(n_layers=64, s_hidden=8192, n_heads=64, s_seq=1024, s_voc=30592),
                 dict(schedules=[0, 1, 2, 3, 4], dp_variants=[0, 2], n_pp=[2, 4, 8], s_mb=[1],
                      n_mb=[4, 8, 16], n_loop=[1, 2, 4, 8], batch_sizes=[16, 32])),
}


def _ref_rank(model, cluster, sp):
    L = R.ref()
    i32 = lambda xs: (C.c_int32 * len(xs))(*xs)  # noqa: E731
    i64 = lambda xs: (C.c_int64 * len(xs))(*xs)  # noqa: E731
    arrays = [i32(sp["schedules"]), len(sp["schedules"]), i32(sp["dp_variants"]), len(sp["dp_variants"])]
    for k in ("n_pp", "s_mb", "n_mb", "n_loop", "batch_sizes"):
        arrays += [i64(sp[k]), len(sp[k])]
    n = C.c_int64()
    assert L.ref_rank_configs(C.byref(model._c()), C.byref(cluster._c()), *arrays, 4, 0, None, None,
                              C.byref(n)) == 0, L.ref_last_error()
    cfgs = (N.ParallelConfigC * n.value)()
    scores = (C.c_double * n.value)()
    assert L.ref_rank_configs(C.byref(model._c()), C.byref(cluster._c()), *arrays, 4, n.value, cfgs, scores,
                              C.byref(n)) == 0
    key = lambda c: (c.n_dp, c.n_tp, c.n_pp, c.n_mb, c.s_mb, c.n_loop, c.dp_variant, c.schedule)  # noqa: E731
    return [(key(c), s) for c, s in zip(cfgs, scores)]


def _key(c: ps.ParallelConfig):
    return (c.n_dp, c.n_tp, c.n_pp, c.n_mb, c.s_mb, c.n_loop, int(c.dp_variant), int(c.schedule))


@needs_ref
@pytest.mark.parametrize("name", list(SPACES))
@pytest.mark.parametrize("cluster", ["a100", "b200"])
def test_simulate_ranking_matches_reference(name, cluster):
    model, sp = SPACES[name]
    k = ps.cluster_preset(cluster)
    if cluster == "a100":  # the reference's 32-GPU preset: search one 8-GPU node of it
        k = ps.ClusterSpec(1, 8, k.peak_flops, k.bw_intra, k.bw_inter, k.pp_latency, k.mem_capacity,
                           k.kernel_efficiency)
    ours = ps.rank_configs(model, k, threads=4, **sp)
    ref = _ref_rank(model, k, sp)
    assert len(ours) == len(ref) and len(ref) > 5
    assert [_key(r.config) for r in ours] == [c for c, _ in ref]
    assert [r.score for r in ours] == [s for _, s in ref]


@needs_ref
@pytest.mark.parametrize("name", list(SPACES))
def test_measured_scoring_reproduces_reference_given_its_timing(name):
    """Rates taken from TimingModel::derive at one configuration carry to every other one (forward
    time linear in layers per stage and s_mb, hand-off time in message bytes, DP time in stage
    parameters), so measured scoring with them ranks exactly as the reference's simulate mode."""
    model, sp = SPACES[name]
    k = ps.cluster_preset("b200")
    ref = _ref_rank(model, k, sp)
    at = ps.ParallelConfig(n_dp=2, n_pp=4, n_loop=1, n_mb=8, dp_variant=V.DP0, schedule=S.OneFOneB)
    ranked_sim = ps.rank_configs(model, k, threads=4, **sp)
    base = next(r for r in ranked_sim if r.config.n_dp >= 2 and r.config.n_pp >= 2)
    rates = ps.rates_from_timing(model, base.config, base.timing)
    meas = ps.rank_configs(model, k, scoring="measured", rates=rates, threads=4, **sp)
    assert len(meas) == len(ref)
    for r, (c, s) in zip(meas, ref):
        assert r.score == pytest.approx(s, rel=1e-9)
    # ties broken identically up to the floating-point noise of the rate round trip
    assert sorted(_key(r.config) for r in meas) == sorted(c for c, _ in ref)
    del at


def test_measured_rates_round_trip():
    model, _ = SPACES["gpt6.7b_8gpu"]
    c0 = ps.ParallelConfig(n_dp=2, n_pp=4, n_loop=2, n_mb=8, dp_variant=V.DP_FS, schedule=S.BreadthFirst)
    t0 = ps.TimingModel(t_fwd_stage=0.012, bwd_ratio=2.1, t_pp_transfer=4e-5, pp_latency=5e-6,
                        t_dp_reduce_stage=0.02, t_dp_reconstruct_stage=0.006)
    r = ps.rates_from_timing(model, c0, t0)
    # a config with stages half as deep and twice the micro-batch size has the same stage cost
    c1 = ps.ParallelConfig(n_dp=2, n_pp=4, n_loop=4, n_mb=4, s_mb=2, dp_variant=V.DP_FS, schedule=S.BreadthFirst)
    got = ps.rank_configs(model, ps.cluster_preset("b200"), schedules=[4], dp_variants=[2], n_pp=[4], s_mb=[2],
                          n_mb=[4], n_loop=[4], batch_sizes=[16], scoring="measured", rates=r)
    assert len(got) == 1 and got[0].config == c1
    t1 = got[0].timing
    assert t1.t_fwd_stage == pytest.approx(t0.t_fwd_stage) and t1.bwd_ratio == t0.bwd_ratio
    assert t1.t_pp_transfer == pytest.approx(2 * t0.t_pp_transfer)
    assert t1.t_dp_reduce_stage == pytest.approx(t0.t_dp_reduce_stage / 2)
    with pytest.raises(ps.SpecError):
        ps.rank_configs(model, ps.cluster_preset("b200"), schedules=[4], dp_variants=[2], n_pp=[4], s_mb=[1],
                        n_mb=[8], n_loop=[2], batch_sizes=[16], scoring="measured")


def test_simulate_durations_replays_simulate():
    """simulate_durations with each task's simulated duration reproduces simulate() exactly, and a
    uniformly slower task set stretches the makespan proportionally."""
    m = ps.ModelSpec(n_layers=16, s_hidden=256, n_heads=2, s_seq=128, s_voc=1000)
    for sched, dv in ((S.BreadthFirst, V.DP_FS), (S.DepthFirst, V.DP0), (S.OneFOneB, V.DP_PS)):
        loops = 2 if sched in (S.BreadthFirst, S.DepthFirst) else 1
        c = ps.ParallelConfig(n_dp=2, n_pp=4, n_loop=loops, n_mb=8, dp_variant=dv, schedule=sched)
        g = ps.build_tasks(m, c)
        tm = ps.TimingModel(t_fwd_stage=1.0, bwd_ratio=2.0, t_pp_transfer=0.125, t_dp_reduce_stage=0.5,
                            t_dp_reconstruct_stage=0.25)
        a = ps.simulate(g, tm)
        dur = [e.end - e.start for e in a.events]
        b = ps.simulate_durations(g, dur)
        assert [(e.start, e.end) for e in a.events] == [(e.start, e.end) for e in b.events]
        assert ps.simulate_durations(g, [2 * x for x in dur]).makespan == 2 * a.makespan
    with pytest.raises(ps.SpecError):
        ps.simulate_durations(g, dur[:-1])
    with pytest.raises(ps.SpecError):
        ps.simulate_durations(g, [-1.0] + dur[1:])


def test_cli_search(tmp_path, capsys):
    """`python -m paper_2211_05953_b200 search`: simulate ranking, measured ranking from a bench line,
    and the reference's empty-result exit code."""
    import json
    from paper_2211_05953_b200.__main__ import main
    assert main(["search", "--model", "gpt-6.7b", "--batch", "16", "--top", "3"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0].startswith("rank,batch,schedule") and len(rows) == 4
    line = {"measured_timing": {"rates": {"fwd_layer_seq": 7.7e-4, "bwd_ratio": 2.2, "pp_s_per_byte": 2.5e-12,
                                          "pp_latency": 0.0, "reduce_s_per_param": 2.7e-13,
                                          "reconstruct_s_per_param": 3.3e-12}}}
    f = tmp_path / "bench.jsonl"
    f.write_text("noise\n" + json.dumps(line) + "\n")
    assert main(["search", "--model", "gpt-6.7b", "--batch", "8", "--scoring", "measured", "--rates-from", str(f)]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    assert len(out) > 5 and float(out[1].split(",")[10]) >= float(out[-1].split(",")[10])
    assert main(["search", "--model", "gpt-6.7b", "--scoring", "measured"]) == 2
    assert main(["search", "--model", "52b", "--gpus", "2", "--batch", "1"]) == 3
