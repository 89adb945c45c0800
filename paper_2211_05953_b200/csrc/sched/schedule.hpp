// bfpp schedule layer: the drop-in replacement for the reference's
// schedule/stage API (pipesim `types.hpp`, `schedule.hpp`, `simulate.hpp`,
// `perf.hpp`). Enum integer values are the wire format shared with the C ABI
// in include/bfpp.h and with the reference (types.hpp:14-15,
// schedule.hpp:41-42).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace bfpp {

using i64 = std::int64_t;
using TaskId = int;

// Reference error.hpp:8-18: SpecError (invalid description, exit 2) and
// SimError (wedged program, exit 4).
struct SpecError : std::runtime_error {
    explicit SpecError(const std::string& m) : std::runtime_error(m) {}
};
struct SimError : std::runtime_error {
    explicit SimError(const std::string& m) : std::runtime_error(m) {}
};

enum class DpVariant : int { DP0 = 0, DP_PS = 1, DP_FS = 2 };
enum class Schedule : int { NoPipeline = 0, GPipe = 1, OneFOneB = 2, DepthFirst = 3, BreadthFirst = 4 };
enum class Lane : int { Compute = 0, DpNet = 1, PpNet = 2 };
enum class TaskKind : int { Fwd = 0, Bwd = 1, Reduce = 2, Reconstruct = 3, Transfer = 4 };
enum class AccumulationOrder : int { DepthFirst = 0, BreadthFirst = 1 };

const char* kind_name(TaskKind k);
const char* schedule_name(Schedule s);

struct ModelSpec {
    i64 n_layers = 1, s_hidden = 1, n_heads = 1, s_head = 1, s_mlp = 4, s_seq = 1, s_voc = 1;
    void validate() const;
};

struct ClusterSpec {
    i64 n_node = 1, s_node = 8;
    double peak_flops = 1.0, bw_intra = 1.0, bw_inter = 1.0, pp_latency = 0.0,
           mem_capacity = 0.0, kernel_efficiency = 0.6;
    i64 n_gpu() const { return n_node * s_node; }
    void validate() const;
};

struct ParallelConfig {
    i64 n_dp = 1, n_tp = 1, n_pp = 1, n_mb = 1, s_mb = 1, n_loop = 1;
    DpVariant dp_variant = DpVariant::DP0;
    Schedule schedule = Schedule::NoPipeline;
    i64 n_stage() const { return n_pp * n_loop; }
    i64 batch_size() const { return n_dp * n_mb * s_mb; }
    i64 grid_size() const { return n_dp * n_tp * n_pp; }
    void validate() const;
    void validate(const ModelSpec& m) const;
    void validate(const ModelSpec& m, const ClusterSpec& c) const;
};

struct StagePlacement {
    i64 n_stage = 1, n_pp = 1, layers_per_stage = 1;
    std::vector<i64> assignment;  // stage -> pipeline rank
    i64 device_of(i64 s) const { return assignment[static_cast<size_t>(s)]; }
    // Explicit layer range of stage s: [first_layer(s), first_layer(s)+layers_per_stage).
    i64 first_layer(i64 s) const { return s * layers_per_stage; }
};

struct TimingModel {
    double t_fwd_stage = 1.0, bwd_ratio = 2.0, t_pp_transfer = 0.0, pp_latency = 0.0,
           t_dp_reduce_stage = 0.0, t_dp_reconstruct_stage = 0.0;
    void validate() const;
};

struct Task {
    TaskId id = -1;
    i64 device = 0;
    i64 peer_device = -1;
    Lane lane = Lane::Compute;
    TaskKind kind = TaskKind::Fwd;
    i64 micro_batch = -1;
    i64 stage = -1;
    int priority = 0;
    std::vector<TaskId> deps;
};

struct TaskGraph {
    i64 n_devices = 1;
    std::vector<Task> tasks;
    std::vector<std::vector<TaskId>> compute_program;
};

struct TimelineEvent {
    TaskId task = -1;
    double start = 0.0, end = 0.0;
};

struct Timeline {
    i64 n_devices = 1;
    std::vector<TimelineEvent> events;  // indexed by task id
    double makespan = 0.0;
    std::vector<std::array<double, 3>> lane_busy;  // [device][lane]
    double compute_busy_max() const;
};

StagePlacement place_stages(const ModelSpec& m, const ParallelConfig& c);
TaskGraph build_tasks(const ModelSpec& m, const ParallelConfig& c, const StagePlacement& pl);
TaskGraph build_accumulation_tasks(const ModelSpec& m, DpVariant v, AccumulationOrder o, i64 n_mb);
Timeline simulate(const TaskGraph& g, const TimingModel& t);
Timeline simulate_durations(const TaskGraph& g, const std::vector<double>& durations);
double bubble_fraction(const Timeline& tl);
std::vector<i64> peak_inflight(const Timeline& tl, const TaskGraph& g, i64 layers_per_stage);
// A measured timeline: events from per-task intervals, lane busy time summed
// per (device, lane) with transfers charged to both endpoints, makespan = the
// latest end (the simulator's accounting, ref simulate.cpp:87-96).
Timeline timeline_from_intervals(const TaskGraph& g, const double* start, const double* end);

// Eq. 11 accounting (reference types.cpp:136-146) and throughput (perf.cpp:8-20).
double compute_per_gpu(const ModelSpec& m, const ParallelConfig& c);
i64 param_count(const ModelSpec& m);

// Analytic memory model (reference memory.hpp / memory.cpp, restated in memory.cpp).
struct MemoryOptions {
    double dp0_bytes_per_param = 20.0;
    double headroom = 0.85;
};
struct MemoryBreakdown {
    double state_bytes = 0.0, activation_bytes = 0.0, checkpoint_bytes = 0.0, total_bytes = 0.0;
};
double state_memory(const ModelSpec& m, const ParallelConfig& c, const MemoryOptions& o = {});
double activation_memory(const ModelSpec& m, const ParallelConfig& c);
double checkpoint_count(const ModelSpec& m, const ParallelConfig& c);
double checkpoint_memory(const ModelSpec& m, const ParallelConfig& c);
MemoryBreakdown total_memory(const ModelSpec& m, const ParallelConfig& c, const MemoryOptions& o = {});
bool feasible(const ModelSpec& m, const ParallelConfig& c, const ClusterSpec& k, const MemoryOptions& o = {});
// "a100", "v100-dgx1" (the reference's, types.cpp:206-231) and "b200"
ClusterSpec cluster_preset(const std::string& name);

// Configuration search (search.cpp, restated in search.cpp) + measured scoring.
TimingModel derive_timing(const ModelSpec& m, const ParallelConfig& c, const ClusterSpec& k, bool recompute = true);
// Per-kind task costs measured at one configuration, in units that carry to another:
// forward seconds per layer per sequence, the backward/forward ratio, seconds per hand-off byte,
// DP seconds per stage parameter (reduce-scatter of the f32 gradient / all-gather of bf16 weights).
struct MeasuredRates {
    double fwd_layer_seq = 0, bwd_ratio = 2, pp_s_per_byte = 0, pp_latency = 0, reduce_s_per_param = 0,
           reconstruct_s_per_param = 0;
};
MeasuredRates rates_from_timing(const ModelSpec& m, const ParallelConfig& c, const TimingModel& t);
TimingModel timing_from_rates(const ModelSpec& m, const ParallelConfig& c, const MeasuredRates& r);
struct SearchSpace {
    std::vector<int> schedules, dp_variants;
    std::vector<i64> n_pp, n_tp, s_mb, n_mb, n_loop, batch_sizes;
};
struct RankedConfig {
    ParallelConfig config;
    double score = 0.0;  // flop/s per GPU (Eq. 11 over the simulated makespan)
    double memory_bytes = 0.0, bubble = 0.0;
    TimingModel timing;
};
std::vector<ParallelConfig> enumerate_configs(const SearchSpace& sp, const ModelSpec& m, const ClusterSpec& k);
// measured = false: the reference's simulate scoring (TimingModel::derive); true: timing_from_rates
std::vector<RankedConfig> rank_configs(const std::vector<ParallelConfig>& configs, const ModelSpec& m,
                                       const ClusterSpec& k, bool measured, const MeasuredRates& rates,
                                       const MemoryOptions& mo, int threads);

}  // namespace bfpp
