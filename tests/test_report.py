"""Timeline exporters and the measured timing model (CPU).

chrome_trace_json must parse to the same document as the reference's (report.cpp:160-212;
the reference pretty-prints with nlohmann, ours writes the JSON directly) and gantt_svg must
be byte-identical (report.cpp:248-290): against tests/golden/report_golden.json (generated
from the compiled reference by tests/golden/make_report_golden.py) and, when oracle/_ref is
present, live over a grid of schedules with random timings.
"""
import ctypes as C
import json
import os
import random

import pytest

import ref_oracle as R
import paper_2211_05953_b200 as ps
from paper_2211_05953_b200 import _native as N

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "report_golden.json")
with open(GOLDEN) as f:
    CASES = json.load(f)


def _graph(m, c):
    h = C.c_void_p()
    assert N.lib().bfpp_build_tasks(C.byref(N.ModelSpecC(*m)), C.byref(N.ParallelConfigC(*c)), C.byref(h)) == 0
    return ps.TaskGraph(h.value)


def _ours(m, c, t):
    g = _graph(m, c)
    tl = ps.simulate(g, ps.TimingModel(*t))
    return ps.chrome_trace_json(tl, g), ps.gantt_svg(tl, g)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_exporters_match_golden(case):
    trace, svg = _ours(case["model"], case["config"], case["timing"])
    assert json.loads(trace) == json.loads(case["chrome_trace_json"])
    assert svg == case["gantt_svg"]


def test_trace_structure():
    case = CASES[0]  # tiny BF DP_FS: 68 tasks, 24 of them transfers (mirrored)
    doc = json.loads(_ours(case["model"], case["config"], case["timing"])[0])
    ev = doc["traceEvents"]
    assert doc["displayTimeUnit"] == "ms"
    assert sum(e["ph"] == "M" for e in ev) == 2 * 4  # per device: process + 3 lanes
    assert sum(e["ph"] == "X" for e in ev) == 68 + 24
    xs = [e for e in ev if e["ph"] == "X"]
    assert all(a["ts"] <= b["ts"] for a, b in zip(xs, xs[1:]))  # start order (mirrors follow their send)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_exporters_live_vs_reference():
    rnd = random.Random(7)
    m = (8, 64, 4, 16, 256, 128, 1000)
    configs = [(1, 1, 2, 4, 1, 2, 0, 4), (2, 1, 2, 4, 1, 2, 2, 4), (1, 1, 4, 8, 1, 2, 0, 3),
               (2, 1, 4, 8, 1, 2, 2, 3), (1, 1, 4, 8, 1, 1, 0, 1), (2, 1, 2, 6, 1, 1, 2, 2), (1, 1, 1, 3, 1, 1, 0, 0)]
    for c in configs:
        t = (rnd.uniform(0.5, 2), rnd.uniform(1.5, 3), rnd.uniform(0, 0.3), rnd.uniform(0, 0.05),
             rnd.uniform(0, 0.5), rnd.uniform(0, 0.5))
        h = C.c_void_p()
        assert R.ref().ref_build_tasks(C.byref(N.ModelSpecC(*m)), C.byref(N.ParallelConfigC(*c)), C.byref(h)) == 0
        tm = N.TimingModelC(*t)
        ref_trace, ref_svg = R.ref_timeline_text(h, tm, 0), R.ref_timeline_text(h, tm, 1)
        R.ref().ref_graph_destroy(h)
        trace, svg = _ours(m, c, t)
        assert json.loads(trace) == json.loads(ref_trace), c
        assert svg == ref_svg, c


@pytest.mark.parametrize("sched,variant,dp,loops", [(ps.Schedule.BreadthFirst, ps.DpVariant.DP_FS, 2, 2),
                                                    (ps.Schedule.DepthFirst, ps.DpVariant.DP0, 1, 2),
                                                    (ps.Schedule.OneFOneB, ps.DpVariant.DP_FS, 2, 1)])
def test_measured_timing_model_roundtrip(sched, variant, dp, loops):
    """Per-kind means of a simulated timeline recover its timing model, and replaying the graph with
    the recovered model reproduces the timeline (zero latency, so transfer duration = t_pp)."""
    model = ps.ModelSpec(n_layers=8, s_hidden=64, n_heads=4, s_seq=128, s_voc=1000)
    cfg = ps.ParallelConfig(n_dp=dp, n_pp=2, n_loop=loops, n_mb=4, dp_variant=variant, schedule=sched)
    g = ps.build_tasks(model, cfg)
    tm = ps.TimingModel(t_fwd_stage=1.25, bwd_ratio=2.5, t_pp_transfer=0.125, pp_latency=0.0,
                        t_dp_reduce_stage=0.375 if dp > 1 else 0.0, t_dp_reconstruct_stage=0.25 if dp > 1 else 0.0)
    tl = ps.simulate(g, tm)
    got = ps.measured_timing_model(g, tl)
    assert got.t_fwd_stage == pytest.approx(1.25) and got.bwd_ratio == pytest.approx(2.5)
    assert got.t_pp_transfer == pytest.approx(0.125)
    if dp > 1:
        assert got.t_dp_reduce_stage == pytest.approx(0.375)
        assert got.t_dp_reconstruct_stage == pytest.approx(0.25)
    replay = ps.simulate(g, got)
    assert replay.makespan == pytest.approx(tl.makespan, rel=1e-12)
    assert ps.bubble_fraction(replay) == pytest.approx(ps.bubble_fraction(tl), abs=1e-12)


def test_measured_timing_model_needs_forward_tasks():
    model = ps.ModelSpec(n_layers=4, s_hidden=64, n_heads=4, s_seq=128, s_voc=1000)
    g = ps.build_tasks(model, ps.ParallelConfig(n_pp=2, n_loop=1, n_mb=2, schedule=ps.Schedule.GPipe))
    tl = ps.Timeline.from_intervals(g, [0.0] * len(g.tasks), [0.0] * len(g.tasks))
    with pytest.raises(ps.SimError):
        ps.measured_timing_model(g, tl)


def test_cli_simulate(tmp_path, capsys):
    from paper_2211_05953_b200.__main__ import main
    trace, svg = tmp_path / "t.json", tmp_path / "g.svg"
    assert main(["simulate", "--model", "gpt-6.7b", "--pp", "4", "--loops", "2", "--dp", "2", "--n-mb", "8",
                 "--trace", str(trace), "--gantt", str(svg)]) == 0
    out = dict(line.split(",", 1) for line in capsys.readouterr().out.splitlines())
    assert float(out["bubble_fraction"]) == pytest.approx(3 / 16)  # (p - 1) / (n_mb * v), Eq. 7
    assert json.loads(trace.read_text())["displayTimeUnit"] == "ms"
    assert svg.read_text().startswith("<svg")
    assert main(["simulate", "--model", "gpt-6.7b", "--pp", "5", "--loops", "2", "--n-mb", "8"]) == 2
    assert "divisibility" in capsys.readouterr().err
