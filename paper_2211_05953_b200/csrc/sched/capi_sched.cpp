// extern "C" boundary for the schedule layer (include/bfpp.h, schedule section).
#include <algorithm>
#include <cstring>
#include <string>

#include "../../../include/bfpp.h"
#include "capi_util.hpp"
#include "report.hpp"
#include "schedule.hpp"

namespace bfpp {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

ModelSpec to_model(const bfpp_model_spec* m) {
    ModelSpec s;
    s.n_layers = m->n_layers;
    s.s_hidden = m->s_hidden;
    s.n_heads = m->n_heads;
    s.s_head = m->s_head;
    s.s_mlp = m->s_mlp;
    s.s_seq = m->s_seq;
    s.s_voc = m->s_voc;
    return s;
}

ParallelConfig to_config(const bfpp_parallel_config* c) {
    ParallelConfig p;
    p.n_dp = c->n_dp;
    p.n_tp = c->n_tp;
    p.n_pp = c->n_pp;
    p.n_mb = c->n_mb;
    p.s_mb = c->s_mb;
    p.n_loop = c->n_loop;
    if (c->dp_variant < 0 || c->dp_variant > 2) throw SpecError("config: unknown data-parallel variant");
    if (c->schedule < 0 || c->schedule > 4) throw SpecError("config: unknown schedule");
    p.dp_variant = static_cast<DpVariant>(c->dp_variant);
    p.schedule = static_cast<Schedule>(c->schedule);
    return p;
}

const TaskGraph& graph_of(const bfpp_graph* g) { return g->g; }

bfpp_timeline* wrap_timeline(Timeline&& tl) { return new bfpp_timeline{std::move(tl)}; }

}  // namespace bfpp

using namespace bfpp;

extern "C" {

const char* bfpp_last_error(void) { return g_last_error.c_str(); }

int bfpp_validate(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_cluster_spec* cl) {
    return guarded([&] {
        if (!cl) {
            to_config(c).validate(to_model(m));
            return;
        }
        ClusterSpec k;
        k.n_node = cl->n_node;
        k.s_node = cl->s_node;
        k.peak_flops = cl->peak_flops;
        k.bw_intra = cl->bw_intra;
        k.bw_inter = cl->bw_inter;
        k.pp_latency = cl->pp_latency;
        k.mem_capacity = cl->mem_capacity;
        k.kernel_efficiency = cl->kernel_efficiency;
        to_config(c).validate(to_model(m), k);
    });
}

int bfpp_place_stages(const bfpp_model_spec* m, const bfpp_parallel_config* c, int64_t* assignment_out, int64_t cap,
                      int64_t* n_stage, int64_t* layers_per_stage) {
    return guarded([&] {
        StagePlacement pl = place_stages(to_model(m), to_config(c));
        if (cap < pl.n_stage) throw SpecError("place_stages: output buffer too small");
        for (i64 s = 0; s < pl.n_stage; ++s) assignment_out[s] = pl.assignment[static_cast<size_t>(s)];
        if (n_stage) *n_stage = pl.n_stage;
        if (layers_per_stage) *layers_per_stage = pl.layers_per_stage;
    });
}

int bfpp_build_tasks(const bfpp_model_spec* m, const bfpp_parallel_config* c, bfpp_graph** out) {
    *out = nullptr;
    return guarded([&] {
        ModelSpec ms = to_model(m);
        ParallelConfig pc = to_config(c);
        *out = new bfpp_graph{build_tasks(ms, pc, place_stages(ms, pc))};
    });
}

int bfpp_build_accumulation_tasks(const bfpp_model_spec* m, int32_t dp_variant, int32_t order, int64_t n_mb,
                                  bfpp_graph** out) {
    *out = nullptr;
    return guarded([&] {
        if (dp_variant < 0 || dp_variant > 2) throw SpecError("accumulation: unknown data-parallel variant");
        if (order < 0 || order > 1) throw SpecError("accumulation: unknown order");
        *out = new bfpp_graph{build_accumulation_tasks(to_model(m), static_cast<DpVariant>(dp_variant),
                                                       static_cast<AccumulationOrder>(order), n_mb)};
    });
}

int bfpp_graph_from_arrays(int64_t n_devices, int64_t n_tasks, const bfpp_task* tasks, const int32_t* dep_offsets,
                           const int32_t* dep_ids, const int32_t* prog_offsets, const int32_t* prog_ids,
                           bfpp_graph** out) {
    *out = nullptr;
    return guarded([&] {
        if (n_devices < 1 || n_tasks < 0) throw SpecError("graph: bad sizes");
        TaskGraph g;
        g.n_devices = n_devices;
        for (int64_t i = 0; i < n_tasks; ++i) {
            Task t;
            t.id = tasks[i].id;
            if (t.id != i) throw SpecError("graph: task ids must equal their index");
            t.lane = static_cast<Lane>(tasks[i].lane);
            t.kind = static_cast<TaskKind>(tasks[i].kind);
            t.priority = tasks[i].priority;
            t.device = tasks[i].device;
            t.peer_device = tasks[i].peer_device;
            t.micro_batch = tasks[i].micro_batch;
            t.stage = tasks[i].stage;
            for (int32_t k = dep_offsets[i]; k < dep_offsets[i + 1]; ++k) {
                if (dep_ids[k] < 0 || dep_ids[k] >= n_tasks) throw SpecError("graph: dependency out of range");
                t.deps.push_back(dep_ids[k]);
            }
            g.tasks.push_back(std::move(t));
        }
        g.compute_program.resize(static_cast<size_t>(n_devices));
        for (int64_t d = 0; d < n_devices; ++d)
            for (int32_t k = prog_offsets[d]; k < prog_offsets[d + 1]; ++k)
                g.compute_program[static_cast<size_t>(d)].push_back(prog_ids[k]);
        *out = new bfpp_graph{std::move(g)};
    });
}

int64_t bfpp_graph_n_devices(const bfpp_graph* g) { return g->g.n_devices; }
int64_t bfpp_graph_n_tasks(const bfpp_graph* g) { return static_cast<int64_t>(g->g.tasks.size()); }
int64_t bfpp_graph_n_deps(const bfpp_graph* g) {
    int64_t n = 0;
    for (const Task& t : g->g.tasks) n += static_cast<int64_t>(t.deps.size());
    return n;
}
int64_t bfpp_graph_n_program_steps(const bfpp_graph* g) {
    int64_t n = 0;
    for (const auto& p : g->g.compute_program) n += static_cast<int64_t>(p.size());
    return n;
}

int bfpp_graph_tasks(const bfpp_graph* g, bfpp_task* out, int64_t cap) {
    return guarded([&] {
        if (cap < static_cast<int64_t>(g->g.tasks.size())) throw SpecError("graph: output buffer too small");
        for (size_t i = 0; i < g->g.tasks.size(); ++i) {
            const Task& t = g->g.tasks[i];
            out[i] = bfpp_task{t.id, static_cast<int32_t>(t.lane), static_cast<int32_t>(t.kind), t.priority,
                               t.device, t.peer_device, t.micro_batch, t.stage};
        }
    });
}

int bfpp_graph_deps(const bfpp_graph* g, int32_t* offsets, int32_t* ids) {
    return guarded([&] {
        int32_t k = 0;
        for (size_t i = 0; i < g->g.tasks.size(); ++i) {
            offsets[i] = k;
            for (TaskId d : g->g.tasks[i].deps) ids[k++] = d;
        }
        offsets[g->g.tasks.size()] = k;
    });
}

int bfpp_graph_programs(const bfpp_graph* g, int32_t* offsets, int32_t* ids) {
    return guarded([&] {
        int32_t k = 0;
        for (size_t d = 0; d < g->g.compute_program.size(); ++d) {
            offsets[d] = k;
            for (TaskId id : g->g.compute_program[d]) ids[k++] = id;
        }
        offsets[g->g.compute_program.size()] = k;
    });
}

void bfpp_graph_destroy(bfpp_graph* g) { delete g; }

int bfpp_simulate_durations(const bfpp_graph* g, const double* durations, bfpp_timeline** out) {
    *out = nullptr;
    return guarded([&] {
        std::vector<double> d(durations, durations + g->g.tasks.size());
        *out = new bfpp_timeline{simulate_durations(g->g, d)};
    });
}

int bfpp_simulate(const bfpp_graph* g, const bfpp_timing_model* t, bfpp_timeline** out) {
    *out = nullptr;
    return guarded([&] {
        TimingModel tm;
        tm.t_fwd_stage = t->t_fwd_stage;
        tm.bwd_ratio = t->bwd_ratio;
        tm.t_pp_transfer = t->t_pp_transfer;
        tm.pp_latency = t->pp_latency;
        tm.t_dp_reduce_stage = t->t_dp_reduce_stage;
        tm.t_dp_reconstruct_stage = t->t_dp_reconstruct_stage;
        *out = new bfpp_timeline{simulate(g->g, tm)};
    });
}

int64_t bfpp_timeline_n_events(const bfpp_timeline* tl) { return static_cast<int64_t>(tl->tl.events.size()); }
int64_t bfpp_timeline_n_devices(const bfpp_timeline* tl) { return tl->tl.n_devices; }
double bfpp_timeline_makespan(const bfpp_timeline* tl) { return tl->tl.makespan; }

int bfpp_timeline_events(const bfpp_timeline* tl, double* start, double* end, double* lane_busy) {
    return guarded([&] {
        for (size_t i = 0; i < tl->tl.events.size(); ++i) {
            if (start) start[i] = tl->tl.events[i].start;
            if (end) end[i] = tl->tl.events[i].end;
        }
        if (lane_busy)
            for (size_t d = 0; d < tl->tl.lane_busy.size(); ++d)
                for (int l = 0; l < 3; ++l) lane_busy[d * 3 + l] = tl->tl.lane_busy[d][l];
    });
}

int bfpp_timeline_from_arrays(const bfpp_graph* g, const double* start, const double* end, bfpp_timeline** out) {
    *out = nullptr;
    return guarded([&] { *out = new bfpp_timeline{timeline_from_intervals(g->g, start, end)}; });
}

void bfpp_timeline_destroy(bfpp_timeline* tl) { delete tl; }

double bfpp_bubble_fraction(const bfpp_timeline* tl) { return bubble_fraction(tl->tl); }

namespace {
int copy_text(const std::string& text, char* buf, int64_t cap, int64_t* len) {
    *len = static_cast<int64_t>(text.size());
    if (buf && cap > 0) {
        const size_t n = std::min(static_cast<size_t>(cap - 1), text.size());
        std::memcpy(buf, text.data(), n);
        buf[n] = 0;
    }
    return 0;
}
}  // namespace

int bfpp_chrome_trace_json(const bfpp_timeline* tl, const bfpp_graph* g, char* buf, int64_t cap, int64_t* len) {
    return guarded([&] { copy_text(chrome_trace_json(tl->tl, g->g), buf, cap, len); });
}

int bfpp_gantt_svg(const bfpp_timeline* tl, const bfpp_graph* g, char* buf, int64_t cap, int64_t* len) {
    return guarded([&] { copy_text(gantt_svg(tl->tl, g->g), buf, cap, len); });
}

int bfpp_measured_timing_model(const bfpp_graph* g, const bfpp_timeline* tl, bfpp_timing_model* out) {
    return guarded([&] {
        const TimingModel tm = measured_timing_model(g->g, tl->tl);
        out->t_fwd_stage = tm.t_fwd_stage;
        out->bwd_ratio = tm.bwd_ratio;
        out->t_pp_transfer = tm.t_pp_transfer;
        out->pp_latency = tm.pp_latency;
        out->t_dp_reduce_stage = tm.t_dp_reduce_stage;
        out->t_dp_reconstruct_stage = tm.t_dp_reconstruct_stage;
    });
}

int bfpp_peak_inflight(const bfpp_timeline* tl, const bfpp_graph* g, int64_t layers_per_stage, int64_t* out) {
    return guarded([&] {
        auto p = peak_inflight(tl->tl, g->g, layers_per_stage);
        for (size_t i = 0; i < p.size(); ++i) out[i] = p[i];
    });
}

int bfpp_total_memory(const bfpp_model_spec* m, const bfpp_parallel_config* c, double dp0_bytes_per_param,
                      double* out) {
    return guarded([&] {
        MemoryOptions o;
        o.dp0_bytes_per_param = dp0_bytes_per_param;
        const MemoryBreakdown b = total_memory(to_model(m), to_config(c), o);
        out[0] = b.state_bytes;
        out[1] = b.activation_bytes;
        out[2] = b.checkpoint_bytes;
        out[3] = b.total_bytes;
    });
}

int bfpp_feasible(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_cluster_spec* cl,
                  double dp0_bytes_per_param, double headroom, int32_t* out) {
    return guarded([&] {
        MemoryOptions o;
        o.dp0_bytes_per_param = dp0_bytes_per_param;
        o.headroom = headroom;
        ClusterSpec k;
        k.mem_capacity = cl->mem_capacity;
        *out = feasible(to_model(m), to_config(c), k, o) ? 1 : 0;
    });
}

int bfpp_cluster_preset(const char* name, bfpp_cluster_spec* out) {
    return guarded([&] {
        const ClusterSpec k = cluster_preset(name ? name : "");
        out->n_node = k.n_node;
        out->s_node = k.s_node;
        out->peak_flops = k.peak_flops;
        out->bw_intra = k.bw_intra;
        out->bw_inter = k.bw_inter;
        out->pp_latency = k.pp_latency;
        out->mem_capacity = k.mem_capacity;
        out->kernel_efficiency = k.kernel_efficiency;
    });
}

int bfpp_rates_from_timing(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_timing_model* t,
                           bfpp_measured_rates* out) {
    return guarded([&] {
        TimingModel tm;
        tm.t_fwd_stage = t->t_fwd_stage;
        tm.bwd_ratio = t->bwd_ratio;
        tm.t_pp_transfer = t->t_pp_transfer;
        tm.pp_latency = t->pp_latency;
        tm.t_dp_reduce_stage = t->t_dp_reduce_stage;
        tm.t_dp_reconstruct_stage = t->t_dp_reconstruct_stage;
        const MeasuredRates r = rates_from_timing(to_model(m), to_config(c), tm);
        *out = {r.fwd_layer_seq, r.bwd_ratio, r.pp_s_per_byte, r.pp_latency, r.reduce_s_per_param,
                r.reconstruct_s_per_param};
    });
}

int bfpp_rank_configs(const bfpp_model_spec* m, const bfpp_cluster_spec* k, const int32_t* schedules, int64_t n_sched,
                      const int32_t* dp_variants, int64_t n_var, const int64_t* n_pp, int64_t n_n_pp,
                      const int64_t* s_mb, int64_t n_s_mb, const int64_t* n_mb, int64_t n_n_mb,
                      const int64_t* n_loop, int64_t n_n_loop, const int64_t* batch_sizes, int64_t n_batch,
                      int32_t scoring, const bfpp_measured_rates* rates, double dp0_bytes_per_param, double headroom,
                      int32_t threads, int64_t cap, bfpp_ranked_config* out, int64_t* n_out) {
    return guarded([&] {
        SearchSpace sp;
        sp.schedules.assign(schedules, schedules + n_sched);
        sp.dp_variants.assign(dp_variants, dp_variants + n_var);
        sp.n_pp.assign(n_pp, n_pp + n_n_pp);
        sp.n_tp = {1};
        sp.s_mb.assign(s_mb, s_mb + n_s_mb);
        sp.n_mb.assign(n_mb, n_mb + n_n_mb);
        sp.n_loop.assign(n_loop, n_loop + n_n_loop);
        sp.batch_sizes.assign(batch_sizes, batch_sizes + n_batch);
        for (int32_t s : sp.schedules)
            if (s < 0 || s > 4) throw SpecError("search: unknown schedule");
        for (int32_t v : sp.dp_variants)
            if (v < 0 || v > 2) throw SpecError("search: unknown data-parallel variant");
        if (scoring == 1 && !rates) throw SpecError("search: measured scoring needs rates");
        ClusterSpec kc;
        kc.n_node = k->n_node;
        kc.s_node = k->s_node;
        kc.peak_flops = k->peak_flops;
        kc.bw_intra = k->bw_intra;
        kc.bw_inter = k->bw_inter;
        kc.pp_latency = k->pp_latency;
        kc.mem_capacity = k->mem_capacity;
        kc.kernel_efficiency = k->kernel_efficiency;
        MeasuredRates r;
        if (rates)
            r = {rates->fwd_layer_seq, rates->bwd_ratio, rates->pp_s_per_byte, rates->pp_latency,
                 rates->reduce_s_per_param, rates->reconstruct_s_per_param};
        MemoryOptions mo;
        mo.dp0_bytes_per_param = dp0_bytes_per_param;
        mo.headroom = headroom;
        const ModelSpec mm = to_model(m);
        const std::vector<RankedConfig> ranked =
            rank_configs(enumerate_configs(sp, mm, kc), mm, kc, scoring == 1, r, mo, threads);
        *n_out = static_cast<int64_t>(ranked.size());
        if (cap == 0) return;
        if (cap < *n_out) throw SpecError("search: output array smaller than the ranked list");
        for (size_t i = 0; i < ranked.size(); ++i) {
            const RankedConfig& rc = ranked[i];
            bfpp_ranked_config& o = out[i];
            o.config = {rc.config.n_dp, rc.config.n_tp, rc.config.n_pp, rc.config.n_mb, rc.config.s_mb,
                        rc.config.n_loop, static_cast<int32_t>(rc.config.dp_variant),
                        static_cast<int32_t>(rc.config.schedule)};
            o.score = rc.score;
            o.memory_bytes = rc.memory_bytes;
            o.bubble = rc.bubble;
            o.timing = {rc.timing.t_fwd_stage, rc.timing.bwd_ratio, rc.timing.t_pp_transfer, rc.timing.pp_latency,
                        rc.timing.t_dp_reduce_stage, rc.timing.t_dp_reconstruct_stage};
        }
    });
}

double bfpp_compute_per_gpu(const bfpp_model_spec* m, const bfpp_parallel_config* c) {
    try {
        return compute_per_gpu(to_model(m), to_config(c));
    } catch (const std::exception& e) {
        set_error(e.what());
        return -1.0;
    }
}

}  // extern "C"
