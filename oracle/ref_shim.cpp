// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// extern "C" shim over the UNMODIFIED reference schedule/simulator sources
// (/root/reference/proj/src/{types,memory,network,perf,schedule,simulate,report,search}.cpp),
// compiled by oracle/Makefile into oracle/_ref/libpipesim_ref.so. It exposes the
// reference's build_tasks / simulate results (including Task::priority, which
// the reference's own Python binding omits, bindings/module.cpp:185-193) with
// the same POD layout as include/bfpp.h so tests can compare field by field.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <string>

#include "../include/bfpp.h"
#include "pipesim/memory.hpp"
#include "pipesim/perf.hpp"
#include "pipesim/report.hpp"
#include "pipesim/search.hpp"
#include "pipesim/schedule.hpp"
#include "pipesim/simulate.hpp"

using namespace pipesim;

namespace {
thread_local std::string err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const SpecError& e) {
        err = e.what();
        return 2;
    } catch (const SimError& e) {
        err = e.what();
        return 4;
    } catch (const std::exception& e) {
        err = e.what();
        return 4;
    }
}

ModelSpec model_of(const bfpp_model_spec* m) {
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

ParallelConfig config_of(const bfpp_parallel_config* c) {
    ParallelConfig p;
    p.n_dp = c->n_dp;
    p.n_tp = c->n_tp;
    p.n_pp = c->n_pp;
    p.n_mb = c->n_mb;
    p.s_mb = c->s_mb;
    p.n_loop = c->n_loop;
    p.dp_variant = static_cast<DpVariant>(c->dp_variant);
    p.schedule = static_cast<Schedule>(c->schedule);
    return p;
}

TimingModel timing_of(const bfpp_timing_model* t) {
    TimingModel tm;
    tm.t_fwd_stage = t->t_fwd_stage;
    tm.bwd_ratio = t->bwd_ratio;
    tm.t_pp_transfer = t->t_pp_transfer;
    tm.pp_latency = t->pp_latency;
    tm.t_dp_reduce_stage = t->t_dp_reduce_stage;
    tm.t_dp_reconstruct_stage = t->t_dp_reconstruct_stage;
    return tm;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return err.c_str(); }

int ref_validate(const bfpp_model_spec* m, const bfpp_parallel_config* c) {
    return guard([&] { config_of(c).validate(model_of(m)); });
}

int ref_place_stages(const bfpp_model_spec* m, const bfpp_parallel_config* c, int64_t* out, int64_t cap,
                     int64_t* n_stage, int64_t* lps) {
    return guard([&] {
        StagePlacement pl = place_stages(model_of(m), config_of(c));
        if (cap < pl.n_stage) throw SpecError("buffer too small");
        for (count_t s = 0; s < pl.n_stage; ++s) out[s] = pl.assignment[static_cast<size_t>(s)];
        *n_stage = pl.n_stage;
        *lps = pl.layers_per_stage;
    });
}

int ref_build_tasks(const bfpp_model_spec* m, const bfpp_parallel_config* c, void** out) {
    *out = nullptr;
    return guard([&] {
        ModelSpec ms = model_of(m);
        ParallelConfig pc = config_of(c);
        *out = new TaskGraph(build_tasks(ms, pc, place_stages(ms, pc)));
    });
}

int ref_build_accumulation_tasks(const bfpp_model_spec* m, int32_t v, int32_t order, int64_t n_mb, void** out) {
    *out = nullptr;
    return guard([&] {
        *out = new TaskGraph(build_accumulation_tasks(model_of(m), static_cast<DpVariant>(v),
                                                      static_cast<AccumulationOrder>(order), n_mb));
    });
}

int64_t ref_graph_n_tasks(void* g) { return static_cast<int64_t>(static_cast<TaskGraph*>(g)->tasks.size()); }
int64_t ref_graph_n_devices(void* g) { return static_cast<TaskGraph*>(g)->n_devices; }
int64_t ref_graph_n_deps(void* g) {
    int64_t n = 0;
    for (const Task& t : static_cast<TaskGraph*>(g)->tasks) n += static_cast<int64_t>(t.deps.size());
    return n;
}
int64_t ref_graph_n_program_steps(void* g) {
    int64_t n = 0;
    for (const auto& p : static_cast<TaskGraph*>(g)->compute_program) n += static_cast<int64_t>(p.size());
    return n;
}

void ref_graph_dump(void* gp, bfpp_task* tasks, int32_t* dep_off, int32_t* dep_ids, int32_t* prog_off,
                    int32_t* prog_ids) {
    const TaskGraph& g = *static_cast<TaskGraph*>(gp);
    int32_t k = 0;
    for (size_t i = 0; i < g.tasks.size(); ++i) {
        const Task& t = g.tasks[i];
        tasks[i] = bfpp_task{t.id, static_cast<int32_t>(t.lane), static_cast<int32_t>(t.kind), t.priority,
                             t.device, t.peer_device, t.micro_batch, t.stage};
        dep_off[i] = k;
        for (TaskId d : t.deps) dep_ids[k++] = d;
    }
    dep_off[g.tasks.size()] = k;
    k = 0;
    for (size_t d = 0; d < g.compute_program.size(); ++d) {
        prog_off[d] = k;
        for (TaskId id : g.compute_program[d]) prog_ids[k++] = id;
    }
    prog_off[g.compute_program.size()] = k;
}

void ref_graph_destroy(void* g) { delete static_cast<TaskGraph*>(g); }

int ref_simulate(void* g, const bfpp_timing_model* t, double* start, double* end, double* lane_busy,
                 double* makespan, double* bubble) {
    return guard([&] {
        const TaskGraph& graph = *static_cast<TaskGraph*>(g);
        Timeline tl = simulate(graph, timing_of(t));
        for (size_t i = 0; i < tl.events.size(); ++i) {
            start[i] = tl.events[i].start;
            end[i] = tl.events[i].end;
        }
        for (size_t d = 0; d < tl.lane_busy.size(); ++d)
            for (int l = 0; l < 3; ++l) lane_busy[d * 3 + l] = tl.lane_busy[d][static_cast<size_t>(l)];
        *makespan = tl.makespan;
        *bubble = bubble_fraction(tl);
    });
}

// The reference's chrome_trace_json / gantt_svg of the simulated timeline of graph g
// (which: 0 trace JSON, 1 SVG). Two-call pattern like the product's text exporters.
int ref_timeline_text(void* g, const bfpp_timing_model* t, int32_t which, char* buf, int64_t cap, int64_t* len) {
    return guard([&] {
        const TaskGraph& graph = *static_cast<TaskGraph*>(g);
        Timeline tl = simulate(graph, timing_of(t));
        const std::string text = which == 0 ? chrome_trace_json(tl, graph) : gantt_svg(tl, graph);
        *len = static_cast<int64_t>(text.size());
        if (buf && cap > 0) {
            const size_t n = std::min(static_cast<size_t>(cap - 1), text.size());
            std::memcpy(buf, text.data(), n);
            buf[n] = 0;
        }
    });
}

int ref_peak_inflight(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_timing_model* t,
                      int64_t* out) {
    return guard([&] {
        ModelSpec ms = model_of(m);
        ParallelConfig pc = config_of(c);
        StagePlacement pl = place_stages(ms, pc);
        TaskGraph g = build_tasks(ms, pc, pl);
        Timeline tl = simulate(g, timing_of(t));
        auto p = peak_inflight(tl, g, pl);
        for (size_t i = 0; i < p.size(); ++i) out[i] = p[i];
    });
}

double ref_compute_per_gpu(const bfpp_model_spec* m, const bfpp_parallel_config* c) {
    return compute_per_gpu(model_of(m), config_of(c));
}

// total_memory / feasible / cluster_preset (memory.cpp:72-86, types.cpp:206-231)
int ref_total_memory(const bfpp_model_spec* m, const bfpp_parallel_config* c, double dp0_bytes_per_param,
                     double* out) {
    return guard([&] {
        MemoryOptions o;
        o.dp0_bytes_per_param = dp0_bytes_per_param;
        const MemoryBreakdown b = total_memory(model_of(m), config_of(c), o);
        out[0] = b.state_bytes;
        out[1] = b.activation_bytes;
        out[2] = b.checkpoint_bytes;
        out[3] = b.total_bytes;
    });
}

int ref_feasible(const bfpp_model_spec* m, const bfpp_parallel_config* c, double mem_capacity,
                 double dp0_bytes_per_param, double headroom, int32_t* out) {
    return guard([&] {
        MemoryOptions o;
        o.dp0_bytes_per_param = dp0_bytes_per_param;
        o.headroom = headroom;
        ClusterSpec k;
        k.mem_capacity = mem_capacity;
        *out = feasible(model_of(m), config_of(c), k, o) ? 1 : 0;
    });
}

// enumerate_configs + rank_configs(Scoring::Simulate) of the reference (search.cpp:62-188), n_tp = 1
int ref_rank_configs(const bfpp_model_spec* m, const bfpp_cluster_spec* k, const int32_t* schedules, int64_t n_sched,
                     const int32_t* dp_variants, int64_t n_var, const int64_t* n_pp, int64_t n_n_pp,
                     const int64_t* s_mb, int64_t n_s_mb, const int64_t* n_mb, int64_t n_n_mb, const int64_t* n_loop,
                     int64_t n_n_loop, const int64_t* batch_sizes, int64_t n_batch, int32_t threads, int64_t cap,
                     bfpp_parallel_config* configs, double* scores, int64_t* n_out) {
    return guard([&] {
        SearchSpace sp;
        for (int64_t i = 0; i < n_sched; ++i) sp.schedules.insert(static_cast<Schedule>(schedules[i]));
        for (int64_t i = 0; i < n_var; ++i) sp.dp_variants.insert(static_cast<DpVariant>(dp_variants[i]));
        sp.n_pp_choices.insert(n_pp, n_pp + n_n_pp);
        sp.n_tp_choices = {1};
        sp.s_mb_choices.insert(s_mb, s_mb + n_s_mb);
        sp.n_mb_choices.insert(n_mb, n_mb + n_n_mb);
        sp.n_loop_choices.insert(n_loop, n_loop + n_n_loop);
        sp.batch_sizes.insert(batch_sizes, batch_sizes + n_batch);
        ClusterSpec c;
        c.n_node = k->n_node;
        c.s_node = k->s_node;
        c.peak_flops = k->peak_flops;
        c.bw_intra = k->bw_intra;
        c.bw_inter = k->bw_inter;
        c.pp_latency = k->pp_latency;
        c.mem_capacity = k->mem_capacity;
        c.kernel_efficiency = k->kernel_efficiency;
        const ModelSpec mm = model_of(m);
        SearchOptions so;
        so.threads = threads;
        const std::vector<RankedConfig> r = rank_configs(enumerate_configs(sp, mm, c), mm, c, Scoring::Simulate, so);
        *n_out = static_cast<int64_t>(r.size());
        if (cap < *n_out) return;
        for (size_t i = 0; i < r.size(); ++i) {
            const ParallelConfig& p = r[i].config;
            configs[i] = {p.n_dp, p.n_tp, p.n_pp, p.n_mb, p.s_mb, p.n_loop, static_cast<int32_t>(p.dp_variant),
                          static_cast<int32_t>(p.schedule)};
            scores[i] = r[i].score;
        }
    });
}

int ref_cluster_preset(const char* name, bfpp_cluster_spec* out) {
    return guard([&] {
        const ClusterSpec k = cluster_preset(name);
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

// CPU baseline: seconds per place_stages+build_tasks and per simulate, median-free
// mean over `reps` repetitions (single thread).
int ref_time_schedule_path(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_timing_model* t,
                           int reps, double* build_s, double* sim_s, int64_t* n_tasks) {
    return guard([&] {
        ModelSpec ms = model_of(m);
        ParallelConfig pc = config_of(c);
        TimingModel tm = timing_of(t);
        double b = 0, s = 0;
        for (int r = 0; r < reps; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            TaskGraph g = build_tasks(ms, pc, place_stages(ms, pc));
            auto t1 = std::chrono::steady_clock::now();
            Timeline tl = simulate(g, tm);
            auto t2 = std::chrono::steady_clock::now();
            b += std::chrono::duration<double>(t1 - t0).count();
            s += std::chrono::duration<double>(t2 - t1).count();
            *n_tasks = static_cast<int64_t>(g.tasks.size());
        }
        *build_s = b / reps;
        *sim_s = s / reps;
    });
}

// The reference's configuration search in simulate mode (search.cpp:136-188) over a GPT model on
// one node of n_gpu B200s: enumerate_configs + rank_configs(Scoring::Simulate) with `threads`
// workers, timed wall-clock. Returns the number of enumerated / ranked configurations.
int ref_time_rank_configs(const bfpp_model_spec* m, int64_t n_gpu, int threads, double* seconds,
                          int64_t* n_enumerated, int64_t* n_ranked) {
    return guard([&] {
        ModelSpec ms = model_of(m);
        ClusterSpec cl;
        cl.n_node = 1;
        cl.s_node = n_gpu;
        cl.peak_flops = 2.25e15;
        cl.bw_intra = 9.0e11;
        cl.bw_inter = 5.0e10;
        cl.pp_latency = 5e-6;
        cl.mem_capacity = 180e9;
        SearchSpace sp;
        sp.schedules = {Schedule::NoPipeline, Schedule::GPipe, Schedule::OneFOneB, Schedule::DepthFirst,
                        Schedule::BreadthFirst};
        sp.n_pp_choices = {1, 2, 4, 8};
        sp.n_tp_choices = {1};
        sp.s_mb_choices = {1, 2};
        sp.n_mb_choices = {1, 2, 4, 8, 16, 32};
        sp.n_loop_choices = {1, 2, 4, 8};
        sp.dp_variants = {DpVariant::DP0, DpVariant::DP_PS, DpVariant::DP_FS};
        sp.batch_sizes = {8, 16, 32, 64};
        sp.scoring = Scoring::Simulate;
        SearchOptions opts;
        opts.threads = threads;
        auto t0 = std::chrono::steady_clock::now();
        const std::vector<ParallelConfig> all = enumerate_configs(sp, ms, cl);
        const std::vector<RankedConfig> ranked = rank_configs(all, ms, cl, Scoring::Simulate, opts);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *n_enumerated = static_cast<int64_t>(all.size());
        *n_ranked = static_cast<int64_t>(ranked.size());
    });
}

}  // extern "C"
