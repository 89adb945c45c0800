// Per-rank B200 executor of a bfpp TaskGraph (the reference's simulate(),
// simulate.cpp:41-158, replaced by real execution).
//
// One process per GPU. Lanes become CUDA streams: Compute -> compute stream
// (program order), DpNet -> low-priority DP stream (priority order: NCCL all-gather /
// reduce-scatter / all-reduce + sharded Adam, per layer segment), PpNet -> send / receive
// streams per direction (copy-engine peer copies into the receiver's CUDA-IPC-mapped slots,
// flag writes / waits with stream memory operations). Cross-stream dependencies are CUDA
// events; the per-rank plan (stream, waits, enqueue order) is plan_rank (plan.hpp).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "../sched/schedule.hpp"

namespace bfpp {

struct ExecOptions {
    int device = 0;
    bool record_timeline = false;
    uint64_t seed = 1234;
    float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.f, init_std = 0.02f;
    bool skip_optimizer = false;
    bool profile_kernels = false;  // CUDA events around every kernel of the step (per-category stats)
};

// Kernel categories for per-step statistics (launch counts always; times when profiling).
enum KernelCat : int { K_GEMM = 0, K_ATTN_FWD, K_ATTN_BWD, K_LAYERNORM, K_MISC, K_ADAM, K_NCAT };
struct KernelStats {
    double ms[K_NCAT] = {};
    double work[K_NCAT] = {};  // flops (GEMM, attention) or bytes (HBM-bound kernels)
    int64_t launches[K_NCAT] = {};
};

// Element offsets of one transformer layer inside a stage's flat parameter vector.
struct LayerParams {
    int64_t ln1_g, ln1_b, qkv, o, ln2_g, ln2_b, fc1, fc2;
};

// Flat parameter layout of one stage: [wte][wpe] (stage 0) + layers + [lnf_g][lnf_b][head] (last).
struct StageLayout {
    bool first = false, last = false;
    int64_t wte = -1, wpe = -1, lnf_g = -1, lnf_b = -1, head = -1;
    std::vector<LayerParams> layers;
    int64_t numel = 0;   // logical parameter count
    int64_t padded = 0;  // multiple of 64 * n_dp (shardable, 128-B aligned shards)
};

StageLayout make_stage_layout(const ModelSpec& m, i64 stage, i64 n_stage, i64 layers_per_stage, i64 n_dp);

class Executor {
public:
    // graph: run this task graph instead of build_tasks(m, c) (e.g. build_accumulation_tasks);
    // c must describe its placement (n_pp, n_loop, n_mb, n_dp, dp_variant).
    Executor(const ModelSpec& m, const ParallelConfig& c, const ExecOptions& o, int rank, int world,
             const std::vector<ncclUniqueId>& uids, const TaskGraph* graph = nullptr);
    ~Executor();

    // tokens: [n_mb][s_mb][seq+1] int32 of this rank's DP replica (host or device pointer).
    void step(const int32_t* tokens, bool tokens_on_host, float* loss_host, float* loss_dev);
    void sync();

    const TaskGraph& graph() const { return graph_; }
    i64 n_local_stages() const { return v_; }
    i64 local_stage(i64 c) const { return c * p_ + pp_rank_; }
    const StageLayout& layout(i64 stage) const { return layouts_[static_cast<size_t>(stage)]; }
    void set_params(i64 stage, const float* host, int64_t n);
    void get_params(i64 stage, float* host, int64_t n, int64_t* lo, int64_t* hi);
    void get_grads(i64 stage, float* host, int64_t n, int64_t* lo, int64_t* hi);
    void zero_grads();
    // bf16 compute weights: resident copy (full) or this rank's all-gather source shard (DP_FS)
    void get_weights16(i64 stage, uint16_t* host, int64_t n, int64_t* lo, int64_t* hi);
    // per-task [start,end] seconds of the last step (tasks of other devices: NaN)
    void timeline(double* start, double* end) const;
    size_t device_bytes() const { return dev_bytes_; }
    const KernelStats& kernel_stats() const;  // of the last step
    cudaStream_t compute_stream() const;
    void set_flags(bool record_timeline, bool profile_kernels);

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
    ModelSpec m_;
    ParallelConfig c_;
    ExecOptions o_;
    TaskGraph graph_;
    StagePlacement pl_;
    std::vector<StageLayout> layouts_;
    int rank_, world_;
    i64 p_, v_, pp_rank_, dp_rank_;
    size_t dev_bytes_ = 0;
};

}  // namespace bfpp
