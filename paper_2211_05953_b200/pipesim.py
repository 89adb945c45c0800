"""Host-side mirror of the reference's ``pipesim`` Python module for the hot path.

Same names, argument meaning and error behaviour as the reference's pybind
module (proj/bindings/module.cpp:28-379) for the schedule/stage API:
``ModelSpec``, ``ParallelConfig``, ``ClusterSpec``, ``TimingModel``,
``place_stages``, ``build_tasks``, ``build_accumulation_tasks``, ``simulate``,
``simulate_config``, ``bubble_fraction``, ``peak_inflight``,
``accumulation_timeline``, ``compute_per_gpu``, ``param_count``,
``throughput``; ``SpecError``/``SimError`` exceptions. Everything computes in
libbfpp.so (C ABI, include/bfpp.h); this file only marshals. Unlike the
reference binding, ``Task.priority`` is exposed (module.cpp:185-193 omits it).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List

from . import _native as N


class SpecError(ValueError):
    """Invalid model/cluster/config (reference error.hpp:8-12; exit code 2)."""


class SimError(RuntimeError):
    """Wedged program / execution failure (reference error.hpp:14-18; exit code 4)."""


class DpVariant(enum.IntEnum):
    DP0 = 0
    DP_PS = 1
    DP_FS = 2


class Schedule(enum.IntEnum):
    NoPipeline = 0
    GPipe = 1
    OneFOneB = 2
    DepthFirst = 3
    BreadthFirst = 4


class Lane(enum.IntEnum):
    Compute = 0
    DpNet = 1
    PpNet = 2


class TaskKind(enum.IntEnum):
    Fwd = 0
    Bwd = 1
    Reduce = 2
    Reconstruct = 3
    Transfer = 4


class AccumulationOrder(enum.IntEnum):
    DepthFirst = 0
    BreadthFirst = 1


def _check(status: int):
    if status == 0:
        return
    msg = N.lib().bfpp_last_error().decode()
    if status == 2:
        raise SpecError(msg)
    raise SimError(msg)


@dataclass(frozen=True)
class ModelSpec:
    """pipesim::ModelSpec; constructor validates like ModelSpec::make (types.cpp:57-68)."""
    n_layers: int
    s_hidden: int
    n_heads: int
    s_seq: int
    s_voc: int
    s_mlp: int = -1
    s_head: int = -1

    def __post_init__(self):
        if self.s_head <= 0:
            object.__setattr__(self, "s_head", self.s_hidden // self.n_heads if self.n_heads > 0 else 0)
        if self.s_mlp <= 0:
            object.__setattr__(self, "s_mlp", 4 * self.s_hidden)
        _check(_validate_model(self))

    def _c(self) -> N.ModelSpecC:
        return N.ModelSpecC(self.n_layers, self.s_hidden, self.n_heads, self.s_head, self.s_mlp,
                            self.s_seq, self.s_voc)


def _validate_model(m: ModelSpec) -> int:
    # A 1-stage, 1-micro-batch config only checks the model fields.
    one = N.ParallelConfigC(1, 1, 1, 1, 1, 1, 0, 0)
    mc = N.ModelSpecC(m.n_layers, m.s_hidden, m.n_heads, m.s_head, m.s_mlp, m.s_seq, m.s_voc)
    return N.lib().bfpp_validate(C.byref(mc), C.byref(one), None)


@dataclass(frozen=True)
class ClusterSpec:
    n_node: int
    s_node: int
    peak_flops: float
    bw_intra: float
    bw_inter: float
    pp_latency: float = 0.0
    mem_capacity: float = 0.0
    kernel_efficiency: float = 0.6

    def n_gpu(self) -> int:
        return self.n_node * self.s_node

    def _c(self) -> N.ClusterSpecC:
        return N.ClusterSpecC(self.n_node, self.s_node, self.peak_flops, self.bw_intra, self.bw_inter,
                              self.pp_latency, self.mem_capacity, self.kernel_efficiency)


@dataclass(frozen=True)
class ParallelConfig:
    """pipesim::ParallelConfig; internal consistency checked on construction
    (pybind ctor, module.cpp:114-121; types.cpp:92-108)."""
    n_dp: int = 1
    n_tp: int = 1
    n_pp: int = 1
    n_mb: int = 1
    s_mb: int = 1
    n_loop: int = 1
    dp_variant: DpVariant = DpVariant.DP0
    schedule: Schedule = Schedule.NoPipeline

    def __post_init__(self):
        # Model-independent checks: use a model whose layer count every stage count divides.
        big = N.ModelSpecC(max(1, self.n_pp * self.n_loop), 1, 1, 1, 4, 1, 1)
        _check(N.lib().bfpp_validate(C.byref(big), C.byref(self._c()), None))

    def n_stage(self) -> int:
        return self.n_pp * self.n_loop

    def batch_size(self) -> int:
        return self.n_dp * self.n_mb * self.s_mb

    def validate(self, model: ModelSpec, cluster: ClusterSpec | None = None):
        _check(N.lib().bfpp_validate(C.byref(model._c()), C.byref(self._c()),
                                     C.byref(cluster._c()) if cluster is not None else None))

    def _c(self) -> N.ParallelConfigC:
        return N.ParallelConfigC(self.n_dp, self.n_tp, self.n_pp, self.n_mb, self.s_mb, self.n_loop,
                                 int(self.dp_variant), int(self.schedule))


@dataclass
class TimingModel:
    t_fwd_stage: float = 1.0
    bwd_ratio: float = 2.0
    t_pp_transfer: float = 0.0
    pp_latency: float = 0.0
    t_dp_reduce_stage: float = 0.0
    t_dp_reconstruct_stage: float = 0.0

    def _c(self) -> N.TimingModelC:
        return N.TimingModelC(self.t_fwd_stage, self.bwd_ratio, self.t_pp_transfer, self.pp_latency,
                              self.t_dp_reduce_stage, self.t_dp_reconstruct_stage)


@dataclass(frozen=True)
class StagePlacement:
    n_stage: int
    n_pp: int
    layers_per_stage: int
    assignment: List[int]

    def device_of(self, stage: int) -> int:
        return self.assignment[stage]

    def layers_of(self, stage: int) -> range:
        """Explicit layer range of a stage: [s*lps, (s+1)*lps)."""
        return range(stage * self.layers_per_stage, (stage + 1) * self.layers_per_stage)


@dataclass
class Task:
    id: int
    device: int
    peer_device: int
    lane: Lane
    kind: TaskKind
    micro_batch: int
    stage: int
    priority: int
    deps: List[int] = field(default_factory=list)


class TaskGraph:
    """pipesim::TaskGraph backed by a native handle (passed to the executor)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        L = N.lib()
        n = L.bfpp_graph_n_tasks(self._h)
        nd = L.bfpp_graph_n_devices(self._h)
        raw = (N.TaskC * max(n, 1))()
        _check(L.bfpp_graph_tasks(self._h, raw, n))
        doff = (C.c_int32 * (n + 1))()
        dids = (C.c_int32 * max(1, L.bfpp_graph_n_deps(self._h)))()
        _check(L.bfpp_graph_deps(self._h, doff, dids))
        poff = (C.c_int32 * (nd + 1))()
        pids = (C.c_int32 * max(1, L.bfpp_graph_n_program_steps(self._h)))()
        _check(L.bfpp_graph_programs(self._h, poff, pids))
        self.n_devices = int(nd)
        self.tasks = [Task(t.id, t.device, t.peer_device, Lane(t.lane), TaskKind(t.kind), t.micro_batch,
                           t.stage, t.priority, list(dids[doff[i]:doff[i + 1]]))
                      for i, t in enumerate(raw[:n])]
        self.compute_program = [list(pids[poff[d]:poff[d + 1]]) for d in range(nd)]

    def tasks_of_kind(self, kind: TaskKind) -> List[int]:
        return [t.id for t in self.tasks if t.kind == kind]

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                N.lib().bfpp_graph_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @staticmethod
    def from_tasks(n_devices: int, tasks: List[Task], compute_program: List[List[int]]) -> "TaskGraph":
        n = len(tasks)
        raw = (N.TaskC * max(n, 1))(*[N.TaskC(t.id, int(t.lane), int(t.kind), t.priority, t.device,
                                              t.peer_device, t.micro_batch, t.stage) for t in tasks])
        offs, ids = [0], []
        for t in tasks:
            ids += t.deps
            offs.append(len(ids))
        poffs, pids = [0], []
        for p in compute_program:
            pids += p
            poffs.append(len(pids))
        h = C.c_void_p()
        arr = lambda xs: (C.c_int32 * max(1, len(xs)))(*xs)  # noqa: E731
        _check(N.lib().bfpp_graph_from_arrays(n_devices, n, raw, arr(offs), arr(ids), arr(poffs), arr(pids),
                                              C.byref(h)))
        return TaskGraph(h.value)


@dataclass
class TimelineEvent:
    task: int
    start: float
    end: float


class Timeline:
    """pipesim::Timeline (simulated or measured), backed by a native handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        L = N.lib()
        n = L.bfpp_timeline_n_events(self._h)
        nd = L.bfpp_timeline_n_devices(self._h)
        st = (C.c_double * max(n, 1))()
        en = (C.c_double * max(n, 1))()
        lb = (C.c_double * (3 * nd))()
        _check(L.bfpp_timeline_events(self._h, st, en, lb))
        self.n_devices = int(nd)
        self.events = [TimelineEvent(i, st[i], en[i]) for i in range(n)]
        self.makespan = float(L.bfpp_timeline_makespan(self._h))
        self.lane_busy = [[lb[3 * d + l] for l in range(3)] for d in range(nd)]

    def compute_busy_max(self) -> float:
        return max([lb[0] for lb in self.lane_busy] + [0.0])

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                N.lib().bfpp_timeline_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @staticmethod
    def from_intervals(graph: TaskGraph, start: List[float], end: List[float]) -> "Timeline":
        n = len(graph.tasks)
        h = C.c_void_p()
        _check(N.lib().bfpp_timeline_from_arrays(graph.handle, (C.c_double * max(n, 1))(*start),
                                                 (C.c_double * max(n, 1))(*end), C.byref(h)))
        return Timeline(h.value)


@dataclass
class PerfPoint:
    beta: float = 0.0
    throughput: float = 0.0
    utilization: float = 0.0
    config: ParallelConfig | None = None


def place_stages(model: ModelSpec, config: ParallelConfig) -> StagePlacement:
    ns = config.n_pp * config.n_loop
    out = (C.c_int64 * max(ns, 1))()
    n_stage, lps = C.c_int64(), C.c_int64()
    _check(N.lib().bfpp_place_stages(C.byref(model._c()), C.byref(config._c()), out, ns, C.byref(n_stage),
                                     C.byref(lps)))
    return StagePlacement(n_stage.value, config.n_pp, lps.value, list(out[:n_stage.value]))


def build_tasks(model: ModelSpec, config: ParallelConfig, placement: StagePlacement | None = None) -> TaskGraph:
    if placement is not None and (placement.n_stage != config.n_stage() or placement.n_pp != config.n_pp):
        raise SpecError("error[invalid-spec]: schedule: placement does not match the configuration")
    h = C.c_void_p()
    _check(N.lib().bfpp_build_tasks(C.byref(model._c()), C.byref(config._c()), C.byref(h)))
    return TaskGraph(h.value)


def build_accumulation_tasks(model: ModelSpec, dp_variant: DpVariant, order: AccumulationOrder,
                             n_mb: int) -> TaskGraph:
    h = C.c_void_p()
    _check(N.lib().bfpp_build_accumulation_tasks(C.byref(model._c()), int(dp_variant), int(order), n_mb,
                                                 C.byref(h)))
    return TaskGraph(h.value)


def simulate(graph: TaskGraph, timing: TimingModel) -> Timeline:
    h = C.c_void_p()
    _check(N.lib().bfpp_simulate(graph.handle, C.byref(timing._c()), C.byref(h)))
    return Timeline(h.value)


def simulate_durations(graph: TaskGraph, durations) -> Timeline:
    """simulate() with one duration per task (e.g. a measured timeline's own task times)."""
    durations = list(durations)
    if len(durations) != len(graph.tasks):
        raise SpecError("error[invalid-spec]: simulate_durations: one duration per task expected")
    d = (C.c_double * len(graph.tasks))(*[float(x) for x in durations])
    h = C.c_void_p()
    _check(N.lib().bfpp_simulate_durations(graph.handle, d, C.byref(h)))
    return Timeline(h.value)


def simulate_config(model: ModelSpec, config: ParallelConfig, timing: TimingModel) -> Timeline:
    return simulate(build_tasks(model, config, place_stages(model, config)), timing)


def accumulation_timeline(model, dp_variant, order, n_mb, timing) -> Timeline:
    return simulate(build_accumulation_tasks(model, dp_variant, order, n_mb), timing)


def bubble_fraction(timeline: Timeline) -> float:
    return float(N.lib().bfpp_bubble_fraction(timeline.handle))


def peak_inflight(timeline: Timeline, graph: TaskGraph, placement: StagePlacement) -> List[int]:
    out = (C.c_int64 * timeline.n_devices)()
    _check(N.lib().bfpp_peak_inflight(timeline.handle, graph.handle, placement.layers_per_stage, out))
    return list(out)


def _text(fn, timeline: Timeline, graph: TaskGraph) -> str:
    n = C.c_int64()
    _check(fn(timeline.handle, graph.handle, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(timeline.handle, graph.handle, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def chrome_trace_json(timeline: Timeline, graph: TaskGraph) -> str:
    """Chrome trace-event JSON of a simulated or measured timeline (reference report.cpp:160-212)."""
    return _text(N.lib().bfpp_chrome_trace_json, timeline, graph)


def gantt_svg(timeline: Timeline, graph: TaskGraph) -> str:
    """SVG Gantt chart, one row per device lane (reference report.cpp:248-290)."""
    return _text(N.lib().bfpp_gantt_svg, timeline, graph)


def measured_timing_model(graph: TaskGraph, timeline: Timeline) -> TimingModel:
    """Per-kind mean task durations of a (measured) timeline as a TimingModel."""
    t = N.TimingModelC()
    _check(N.lib().bfpp_measured_timing_model(graph.handle, timeline.handle, C.byref(t)))
    return TimingModel(t.t_fwd_stage, t.bwd_ratio, t.t_pp_transfer, t.pp_latency, t.t_dp_reduce_stage,
                       t.t_dp_reconstruct_stage)


def compute_per_gpu(model: ModelSpec, config: ParallelConfig) -> float:
    return float(N.lib().bfpp_compute_per_gpu(C.byref(model._c()), C.byref(config._c())))


@dataclass(frozen=True)
class MemoryBreakdown:
    state_bytes: float
    activation_bytes: float
    checkpoint_bytes: float
    total_bytes: float


@dataclass(frozen=True)
class MemoryOptions:
    dp0_bytes_per_param: float = 20.0
    headroom: float = 0.85


def total_memory(model: ModelSpec, config: ParallelConfig, opts: MemoryOptions = MemoryOptions()) -> MemoryBreakdown:
    """Analytic bytes per device (memory.cpp:72-80)."""
    out = (C.c_double * 4)()
    _check(N.lib().bfpp_total_memory(C.byref(model._c()), C.byref(config._c()), opts.dp0_bytes_per_param, out))
    return MemoryBreakdown(*out)


def feasible(model: ModelSpec, config: ParallelConfig, cluster: ClusterSpec,
             opts: MemoryOptions = MemoryOptions()) -> bool:
    """total_memory <= headroom * mem_capacity (memory.cpp:82-86)."""
    r = C.c_int32()
    _check(N.lib().bfpp_feasible(C.byref(model._c()), C.byref(config._c()), C.byref(cluster._c()),
                                 opts.dp0_bytes_per_param, opts.headroom, C.byref(r)))
    return bool(r.value)


def cluster_preset(name: str) -> ClusterSpec:
    """The reference's presets (types.cpp:206-231: "a100", "v100-dgx1") plus "b200"."""
    k = N.ClusterSpecC()
    _check(N.lib().bfpp_cluster_preset(name.encode(), C.byref(k)))
    return ClusterSpec(k.n_node, k.s_node, k.peak_flops, k.bw_intra, k.bw_inter, k.pp_latency, k.mem_capacity,
                       k.kernel_efficiency)


@dataclass(frozen=True)
class MeasuredRates:
    """Per-kind task costs measured at one configuration, in units that carry to another
    (forward s per layer per sequence, backward/forward, s per hand-off byte, DP s per stage param)."""
    fwd_layer_seq: float
    bwd_ratio: float
    pp_s_per_byte: float
    pp_latency: float
    reduce_s_per_param: float
    reconstruct_s_per_param: float

    def _c(self):
        return N.MeasuredRatesC(self.fwd_layer_seq, self.bwd_ratio, self.pp_s_per_byte, self.pp_latency,
                                self.reduce_s_per_param, self.reconstruct_s_per_param)


def rates_from_timing(model: ModelSpec, config: ParallelConfig, timing: TimingModel) -> MeasuredRates:
    """Rates of a (measured) TimingModel at `config` (divides out stage size, s_mb, message sizes)."""
    r = N.MeasuredRatesC()
    _check(N.lib().bfpp_rates_from_timing(C.byref(model._c()), C.byref(config._c()), C.byref(timing._c()),
                                          C.byref(r)))
    return MeasuredRates(r.fwd_layer_seq, r.bwd_ratio, r.pp_s_per_byte, r.pp_latency, r.reduce_s_per_param,
                         r.reconstruct_s_per_param)


@dataclass(frozen=True)
class RankedConfig:
    config: ParallelConfig
    score: float          # flop/s per GPU (Eq. 11 over the simulated makespan)
    memory_bytes: float   # total_memory
    bubble: float
    timing: TimingModel


def rank_configs(model: ModelSpec, cluster: ClusterSpec, *, schedules, dp_variants, n_pp, s_mb, n_mb, n_loop,
                 batch_sizes, scoring: str = "simulate", rates: MeasuredRates | None = None,
                 memory: MemoryOptions = MemoryOptions(), threads: int = 0) -> List[RankedConfig]:
    """enumerate_configs + rank_configs (search.cpp:62-188, n_tp = 1): the feasible configurations of
    the space, best first. scoring "simulate" = the reference's (TimingModel::derive); "measured" =
    simulated with timing_from_rates(rates) (per-kind durations measured on B200s)."""
    if scoring not in ("simulate", "measured"):
        raise SpecError(f"unknown scoring mode '{scoring}' (expected simulate or measured)")
    if scoring == "measured" and rates is None:
        raise SpecError("measured scoring needs rates")
    i32 = lambda xs: (C.c_int32 * len(xs))(*[int(x) for x in xs])  # noqa: E731
    i64 = lambda xs: (C.c_int64 * len(xs))(*[int(x) for x in xs])  # noqa: E731
    arrays = [i32(schedules), len(schedules), i32(dp_variants), len(dp_variants), i64(n_pp), len(n_pp), i64(s_mb),
              len(s_mb), i64(n_mb), len(n_mb), i64(n_loop), len(n_loop), i64(batch_sizes), len(batch_sizes)]
    rc = C.byref(rates._c()) if rates is not None else None
    n = C.c_int64()
    L = N.lib()
    args = lambda cap, out: [C.byref(model._c()), C.byref(cluster._c())] + arrays + [  # noqa: E731
        1 if scoring == "measured" else 0, rc, memory.dp0_bytes_per_param, memory.headroom, threads, cap, out,
        C.byref(n)]
    _check(L.bfpp_rank_configs(*args(0, None)))
    buf = (N.RankedConfigC * max(1, n.value))()
    _check(L.bfpp_rank_configs(*args(n.value, buf)))
    out = []
    for r in buf[:n.value]:
        c = r.config
        cfg = ParallelConfig(n_dp=c.n_dp, n_tp=c.n_tp, n_pp=c.n_pp, n_mb=c.n_mb, s_mb=c.s_mb, n_loop=c.n_loop,
                             dp_variant=DpVariant(c.dp_variant), schedule=Schedule(c.schedule))
        t = r.timing
        out.append(RankedConfig(cfg, r.score, r.memory_bytes, r.bubble,
                                TimingModel(t.t_fwd_stage, t.bwd_ratio, t.t_pp_transfer, t.pp_latency,
                                            t.t_dp_reduce_stage, t.t_dp_reconstruct_stage)))
    return out


def param_count(model: ModelSpec) -> int:
    return 12 * model.n_layers * model.s_hidden * model.s_hidden


def throughput(model: ModelSpec, config: ParallelConfig, timeline: Timeline, cluster: ClusterSpec) -> PerfPoint:
    """Eq. 11 flop/s per GPU over the (simulated or measured) makespan (perf.cpp:8-20)."""
    config.validate(model, cluster)
    if timeline.makespan <= 0:
        raise SpecError("error[invalid-spec]: throughput: timeline has no extent")
    tput = compute_per_gpu(model, config) / timeline.makespan
    return PerfPoint(config.batch_size() / cluster.n_gpu(), tput, tput / cluster.peak_flops, config)
