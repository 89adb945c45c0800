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
    // activation checkpointing: a forward keeps only each layer's output
    // (2 T h bytes, the reference's checkpoint, memory.cpp:64-70); the backward recomputes the
    // layer's forward into one working set (and the LM head's logits) before differentiating it
    bool recompute = false;
    // size the rank's buffers without touching the GPU (memory_plan)
    bool dry_run = false;
};

// Device bytes of one rank by category (allocation sizes as the executor requests them).
enum MemCat : int {
    M_WEIGHTS = 0,     // bf16 compute weights: resident stages, or the two DP_FS reconstruction slots
    M_GRADS,           // f32 gradient accumulation: per stage, or one pooled buffer (sharded variants)
    M_OPTIMIZER,       // f32 master weights + Adam m, v (this rank's shards)
    M_GRAD_SHARDS,     // reduced-gradient shards, reduce-scatter landing / per-segment buffers
    M_WEIGHT_SHARDS,   // bf16 all-gather source shards (sharded variants)
    M_ACTIVATIONS,     // activation sets of the live (micro-batch, stage) pairs: full or checkpoints
    M_PP_BUFFERS,      // pipeline receive arena + per-(micro-batch, stage) backward send buffers
    M_SCRATCH,         // per-layer working sets, attention temporaries, logits (recompute), tokens
    M_NCAT
};
struct MemoryPlan {
    size_t bytes[M_NCAT] = {};
    int64_t activation_sets = 0;  // pooled (micro-batch, local stage) activation sets = peak live in program order
    int64_t head_sets = 0;        // pooled logits sets of the last stage (0 with recompute)
    size_t total() const {
        size_t t = 0;
        for (size_t b : bytes) t += b;
        return t;
    }
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
    // completes deferred optimizer work (the lazy token-table update) before parameters are read
    void flush_lazy_updates();
    void get_grads(i64 stage, float* host, int64_t n, int64_t* lo, int64_t* hi);
    void zero_grads();
    // bf16 compute weights: resident copy (full) or this rank's all-gather source shard (DP_FS)
    void get_weights16(i64 stage, uint16_t* host, int64_t n, int64_t* lo, int64_t* hi);
    // per-task [start,end] seconds of the last step (tasks of other devices: NaN)
    void timeline(double* start, double* end) const;
    size_t device_bytes() const { return dev_bytes_; }
    const MemoryPlan& memory_plan() const { return mem_; }
    const KernelStats& kernel_stats() const;  // of the last step
    cudaStream_t compute_stream() const;
    void set_flags(bool record_timeline, bool profile_kernels);

private:
    struct Impl;
    void wait_step_event(cudaEvent_t ev, int step);
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
    MemoryPlan mem_;
};

}  // namespace bfpp
