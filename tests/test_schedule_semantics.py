"""The reference's schedule known-answer tests (proj/tests/test_schedule.cpp,
tests/python/test_smoke.py:40-51), restated against the bfpp Python mirror."""
import random

import pytest

import paper_2211_05953_b200 as ps
from paper_2211_05953_b200 import DpVariant as V, Schedule as S, TaskKind as K


def layers_model(n, seq=128):  # test_schedule.cpp:15-17
    return ps.ModelSpec(n_layers=n, s_hidden=64, n_heads=4, s_seq=seq, s_voc=1000, s_head=16)


def cfg(s, v, pp, loop, mb, dp=1):
    return ps.ParallelConfig(n_dp=dp, n_pp=pp, n_loop=loop, n_mb=mb, dp_variant=v, schedule=s)


def run(m, c, t):
    return ps.simulate(ps.build_tasks(m, c, ps.place_stages(m, c)), t)


def unit(t_fwd=1.0, ratio=2.0):
    return ps.TimingModel(t_fwd_stage=t_fwd, bwd_ratio=ratio)


def test_placement_loops_around_ring():
    pl = ps.place_stages(layers_model(16), cfg(S.BreadthFirst, V.DP0, 4, 4, 4))
    assert pl.n_stage == 16 and pl.layers_per_stage == 1
    assert pl.assignment == [s % 4 for s in range(16)]
    pl = ps.place_stages(layers_model(16), cfg(S.GPipe, V.DP0, 4, 1, 4))
    assert pl.assignment == [0, 1, 2, 3] and pl.layers_per_stage == 4
    assert list(pl.layers_of(2)) == [8, 9, 10, 11]


def test_divisibility_error():
    with pytest.raises(ps.SpecError, match="divisibility"):
        ps.place_stages(layers_model(16), cfg(S.BreadthFirst, V.DP0, 5, 1, 5))


def test_hand_checked_makespans():
    assert run(layers_model(2), cfg(S.GPipe, V.DP0, 2, 1, 2), unit()).makespan == 9.0
    assert run(layers_model(4), cfg(S.BreadthFirst, V.DP0, 2, 2, 2), unit(0.5)).makespan == 7.5


def test_bubble_closed_form_grid():
    for p in (2, 4):
        for v in (1, 2, 4):
            for mb in range(p, 4 * p + 1):
                for s in (S.GPipe, S.OneFOneB, S.DepthFirst, S.BreadthFirst):
                    if s in (S.GPipe, S.OneFOneB) and v != 1:
                        continue
                    if s == S.DepthFirst and mb % p:
                        continue
                    tl = run(layers_model(p * v), cfg(s, V.DP0, p, v, mb), unit())
                    assert ps.bubble_fraction(tl) == pytest.approx((p - 1) / (mb * v), rel=1e-9)


def test_python_smoke_bubble():  # test_smoke.py:40-51
    m = ps.ModelSpec(n_layers=16, s_hidden=64, n_heads=4, s_seq=128, s_voc=1000, s_head=16)
    c = ps.ParallelConfig(n_pp=4, n_mb=8, n_loop=4, schedule=S.BreadthFirst)
    assert ps.bubble_fraction(ps.simulate_config(m, c, ps.TimingModel())) == pytest.approx(3 / 32, abs=1e-12)


def test_checkpoint_residency():
    for p in (2, 4):
        for v in (1, 2, 4):
            for mb in range(p, 4 * p + 1, p):
                m = layers_model(p * v)
                L = p * v
                for s in (S.GPipe, S.OneFOneB, S.DepthFirst, S.BreadthFirst):
                    if s in (S.GPipe, S.OneFOneB) and v != 1:
                        continue
                    c = cfg(s, V.DP0, p, v, mb)
                    pl = ps.place_stages(m, c)
                    g = ps.build_tasks(m, c, pl)
                    peak = max(ps.peak_inflight(ps.simulate(g, unit()), g, pl))
                    if s in (S.GPipe, S.BreadthFirst):
                        assert peak == mb * L // p
                    elif s == S.OneFOneB:
                        assert peak <= (2 * p - 1) * L // p
                    else:
                        assert peak <= L + p - 1


def test_program_prefixes_16_layers_4_devices_8_mb():
    m = layers_model(16)

    def prefix(s, loop, n):
        g = ps.build_tasks(m, cfg(s, V.DP0, 4, loop, 8))
        return [(g.tasks[i].kind, g.tasks[i].micro_batch, g.tasks[i].stage) for i in g.compute_program[0][:n]]

    bf = prefix(S.BreadthFirst, 4, 10)
    assert bf[:8] == [(K.Fwd, mb, 0) for mb in range(8)] and bf[8:] == [(K.Fwd, 0, 4), (K.Fwd, 1, 4)]
    df = prefix(S.DepthFirst, 4, 8)
    assert df[:4] == [(K.Fwd, mb, 0) for mb in range(4)] and df[4] == (K.Fwd, 0, 4)
    gp = prefix(S.GPipe, 1, 9)
    assert gp[:8] == [(K.Fwd, mb, 0) for mb in range(8)] and gp[8][0] == K.Bwd
    ob = prefix(S.OneFOneB, 1, 6)
    assert ob[0] == (K.Fwd, 0, 0) and ob[3] == (K.Fwd, 3, 0) and ob[4] == (K.Bwd, 0, 0) and ob[5] == (K.Fwd, 4, 0)


def test_fully_sharded_counts():
    p, v, mb = 4, 4, 8
    m = layers_model(p * v)
    cnt = lambda g, k: len(g.tasks_of_kind(k))  # noqa: E731
    g = ps.build_tasks(m, cfg(S.BreadthFirst, V.DP_FS, p, v, mb, 2))
    assert cnt(g, K.Reconstruct) == 2 * p * v and cnt(g, K.Reduce) == p * v
    g = ps.build_tasks(m, cfg(S.DepthFirst, V.DP_FS, p, v, mb, 2))
    assert cnt(g, K.Reconstruct) == 2 * p * v * (mb // p) and cnt(g, K.Reduce) == p * v * (mb // p)
    g = ps.build_tasks(layers_model(p), cfg(S.GPipe, V.DP_FS, p, 1, mb, 2))
    assert cnt(g, K.Reconstruct) == 2 * p * mb and cnt(g, K.Reduce) == p * mb
    g = ps.build_tasks(m, cfg(S.BreadthFirst, V.DP_FS, p, v, mb, 1))
    assert cnt(g, K.Reconstruct) == 0 and cnt(g, K.Reduce) == 0
    g = ps.build_tasks(m, cfg(S.DepthFirst, V.DP0, p, v, mb, 2))
    assert cnt(g, K.Reconstruct) == 0 and cnt(g, K.Reduce) == p * v


def test_reduction_overlap_ordering():
    rng = random.Random(17)
    for _ in range(12):
        p, v = rng.choice((2, 4, 8)), rng.choice((2, 4))
        mb = p * (2 + rng.randrange(3))
        L = p * v
        red = rng.uniform(0.05, 3.0)

        def timing(loops):
            lps = L / (p * loops)
            return ps.TimingModel(t_fwd_stage=lps, bwd_ratio=2.0, t_dp_reduce_stage=red * lps)

        m = layers_model(L)
        bf = run(m, cfg(S.BreadthFirst, V.DP0, p, v, mb, 2), timing(v)).makespan
        df = run(m, cfg(S.DepthFirst, V.DP0, p, v, mb, 2), timing(v)).makespan
        gp = run(m, cfg(S.GPipe, V.DP0, p, 1, mb, 2), timing(1)).makespan
        assert bf <= df + 1e-9 and df <= gp + 1e-9


def test_timeline_contract_and_determinism():
    rng = random.Random(51)
    for _ in range(24):
        p, v = rng.choice((2, 4, 8)), rng.choice((1, 2, 4))
        mb = p * (1 + rng.randrange(3))
        s = rng.choice((S.GPipe, S.OneFOneB, S.DepthFirst, S.BreadthFirst))
        if s in (S.GPipe, S.OneFOneB) and v != 1:
            continue
        fs = rng.randrange(2) == 0
        c = cfg(s, V.DP_FS if fs else V.DP0, p, v, mb, 2)
        m = layers_model(p * v)
        t = ps.TimingModel(1.0, 2.0 + rng.randrange(2), 0.01 * rng.randrange(8), 0.01 * rng.randrange(4),
                           0.1 * rng.randrange(12), 0.1 * rng.randrange(6))
        g = ps.build_tasks(m, c)
        tl = ps.simulate(g, t)
        assert tl.makespan == max(e.end for e in tl.events)
        lanes = {}
        for task in g.tasks:
            ev = tl.events[task.id]
            for d in task.deps:
                assert tl.events[d].end <= ev.start + 1e-12
            lanes.setdefault((task.device, int(task.lane)), []).append((ev.start, ev.end))
            if task.kind == K.Transfer:
                lanes.setdefault((task.peer_device, 2), []).append((ev.start, ev.end))
        for iv in lanes.values():
            iv.sort()
            for a, b in zip(iv, iv[1:]):
                assert b[0] >= a[1] - 1e-12
        tl2 = ps.simulate(ps.build_tasks(m, c), t)
        assert [(e.start, e.end) for e in tl.events] == [(e.start, e.end) for e in tl2.events]


def test_deadlock_detection():
    a = ps.Task(0, 0, -1, ps.Lane.Compute, K.Fwd, 0, 0, 0, [1])
    b = ps.Task(1, 0, -1, ps.Lane.Compute, K.Bwd, 0, 0, 1, [])
    g = ps.TaskGraph.from_tasks(1, [a, b], [[0, 1]])
    with pytest.raises(ps.SimError, match="deadlock"):
        ps.simulate(g, unit())


def test_accumulation_timelines():
    m = layers_model(4)
    t = ps.TimingModel(t_dp_reduce_stage=0.7, t_dp_reconstruct_stage=0.3)
    df = ps.accumulation_timeline(m, V.DP_FS, ps.AccumulationOrder.DepthFirst, 4, t)
    bf = ps.accumulation_timeline(m, V.DP_FS, ps.AccumulationOrder.BreadthFirst, 4, t)
    assert df.lane_busy[0][1] == pytest.approx(4.0 * bf.lane_busy[0][1])
    for mb in (2, 4):
        for red in (0.2, 1.5, 4.0):
            tt = ps.TimingModel(t_dp_reduce_stage=red)
            d = ps.accumulation_timeline(m, V.DP0, ps.AccumulationOrder.DepthFirst, mb, tt)
            b = ps.accumulation_timeline(m, V.DP0, ps.AccumulationOrder.BreadthFirst, mb, tt)
            assert b.makespan <= d.makespan + 1e-9


def test_measured_timeline_metrics():
    """Metrics applied to an externally measured timeline (the executor's path)."""
    m = layers_model(4)
    c = cfg(S.BreadthFirst, V.DP0, 2, 2, 2)
    g = ps.build_tasks(m, c)
    sim = ps.simulate(g, unit(0.5))
    tl = ps.Timeline.from_intervals(g, [e.start for e in sim.events], [e.end for e in sim.events])
    assert tl.makespan == sim.makespan
    assert ps.bubble_fraction(tl) == ps.bubble_fraction(sim)


def test_throughput_eq11():
    m = ps.ModelSpec(n_layers=32, s_hidden=4096, n_heads=32, s_seq=2048, s_voc=50304)
    c = ps.ParallelConfig(n_dp=2, n_pp=4, n_loop=2, n_mb=8, dp_variant=V.DP_FS, schedule=S.BreadthFirst)
    cl = ps.ClusterSpec(n_node=1, s_node=8, peak_flops=2.25e15, bw_intra=1.8e12, bw_inter=1.8e12)
    tl = ps.simulate_config(m, c, ps.TimingModel(t_fwd_stage=0.01, bwd_ratio=2.0))
    pp = ps.throughput(m, c, tl, cl)
    assert pp.throughput == pytest.approx(ps.compute_per_gpu(m, c) / tl.makespan)
    assert pp.beta == 2.0


def test_param_count_and_compute_per_gpu_closed_forms():
    """param_count = 12 L h^2 (types.cpp:132-134); compute_per_gpu = Eq. 11 (types.cpp:136-146):
    s * 96 * n_mb * s_mb * L * h * (h + s/6 + V/(16 L)) / (n_pp * n_tp)."""
    m = ps.ModelSpec(n_layers=24, s_hidden=2048, n_heads=16, s_seq=2048, s_voc=50304)
    assert ps.param_count(m) == 12 * 24 * 2048 * 2048
    c = ps.ParallelConfig(n_dp=1, n_pp=2, n_loop=4, n_mb=2, schedule=S.BreadthFirst)
    L, h, s, V = 24, 2048.0, 2048.0, 50304.0
    want = s * 96 * 2 * 1 * L * h * (h + s / 6 + V / (16 * L)) / 2
    assert ps.compute_per_gpu(m, c) == pytest.approx(want, rel=1e-12)
