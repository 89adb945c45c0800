// Per-rank executor: runs one pipeline rank's slice of a bfpp TaskGraph on a B200 with the
// sm_100a stage kernels, copy-engine peer copies over NVLink for the pipeline hand-offs (CUDA IPC
// + stream memory operations) and NCCL for the (fully sharded) data-parallel traffic.
// See executor.hpp and DESIGN.md §3.
#include "executor.hpp"

#include <cuda.h>

#include <cuda_bf16.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>

#include "../kernels/gemm.hpp"
#include "../kernels/kernels.hpp"
#include "plan.hpp"

namespace bfpp {

#define CK(x)                                                                                                     \
    do {                                                                                                          \
        cudaError_t e_ = (x);                                                                                     \
        if (e_ != cudaSuccess)                                                                                    \
            throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " #x);         \
    } while (0)
#define NK(x)                                                                                                     \
    do {                                                                                                          \
        ncclResult_t r_ = (x);                                                                                    \
        if (r_ != ncclSuccess)                                                                                    \
            throw std::runtime_error(std::string("NCCL error ") + ncclGetErrorString(r_) + " at " #x);         \
    } while (0)

using bf16 = __nv_bfloat16;

StageLayout make_stage_layout(const ModelSpec& m, i64 stage, i64 n_stage, i64 lps, i64 n_dp) {
    StageLayout L;
    const int64_t h = m.s_hidden, mlp = m.s_mlp, V = m.s_voc, S = m.s_seq;
    int64_t off = 0;
    auto take = [&](int64_t n) {
        const int64_t o = off;
        off += (n + 63) / 64 * 64;  // 128-byte aligned sub-tensors (TMA needs 16 B)
        return o;
    };
    L.first = stage == 0;
    L.last = stage == n_stage - 1;
    if (L.first) {
        L.wte = take(V * h);
        L.wpe = take(S * h);
    }
    for (i64 l = 0; l < lps; ++l) {
        LayerParams p;
        p.ln1_g = take(h);
        p.ln1_b = take(h);
        p.qkv = take(3 * h * h);
        p.o = take(h * h);
        p.ln2_g = take(h);
        p.ln2_b = take(h);
        p.fc1 = take(mlp * h);
        p.fc2 = take(h * mlp);
        L.layers.push_back(p);
    }
    if (L.last) {
        L.lnf_g = take(h);
        L.lnf_b = take(h);
        L.head = take(V * h);
    }
    L.numel = off;
    const int64_t q = 64 * n_dp;
    L.padded = (off + q - 1) / q * q;
    return L;
}

namespace {

// Stream memory operations (driver API, resolved at run time): the pipeline hand-off is a
// copy-engine peer copy followed by a 32-bit flag write into the receiver's memory; the
// receiver's stream waits on the flag. No SMs, no communicator-ordering hazards.
using PFN_waitv32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_writev32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct StreamMemOps {
    PFN_waitv32 wait = nullptr;
    PFN_writev32 write = nullptr;
};
const StreamMemOps& memops() {
    static StreamMemOps ops;
    static bool init = false;
    if (!init) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.wait = reinterpret_cast<PFN_waitv32>(p);
        p = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.write = reinterpret_cast<PFN_writev32>(p);
        init = true;
    }
    if (!ops.wait || !ops.write) throw std::runtime_error("executor: stream memory operations unavailable");
    return ops;
}

// Kinds of parameter sub-tensors for initialisation.
struct Segment {
    int64_t off, n;
    float mean, std;
};

std::vector<Segment> init_segments(const StageLayout& L, const ModelSpec& m, float std) {
    const int64_t h = m.s_hidden, mlp = m.s_mlp, V = m.s_voc, S = m.s_seq;
    const float out_std = std / std::sqrt(2.f * static_cast<float>(m.n_layers));
    std::vector<Segment> s;
    if (L.first) {
        s.push_back({L.wte, V * h, 0.f, std});
        s.push_back({L.wpe, S * h, 0.f, std});
    }
    for (const auto& p : L.layers) {
        s.push_back({p.ln1_g, h, 1.f, 0.f});
        s.push_back({p.ln1_b, h, 0.f, 0.f});
        s.push_back({p.qkv, 3 * h * h, 0.f, std});
        s.push_back({p.o, h * h, 0.f, out_std});
        s.push_back({p.ln2_g, h, 1.f, 0.f});
        s.push_back({p.ln2_b, h, 0.f, 0.f});
        s.push_back({p.fc1, mlp * h, 0.f, std});
        s.push_back({p.fc2, h * mlp, 0.f, out_std});
    }
    if (L.last) {
        s.push_back({L.lnf_g, h, 1.f, 0.f});
        s.push_back({L.lnf_b, h, 0.f, 0.f});
        s.push_back({L.head, V * h, 0.f, std});
    }
    return s;
}

__global__ void add_f32_kernel(float* __restrict__ dst, const float* __restrict__ src, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] += src[i];
}

}  // namespace

// ---------------------------------------------------------------------------------------------
struct LayerActs {
    bf16 *x_in, *ln1, *qkv, *o, *x_mid, *ln2, *pre, *act, *x_out;
    float *mu1, *rs1, *mu2, *rs2, *lse;
};
struct StageActs {
    std::vector<LayerActs> layers;
    bf16* in = nullptr;    // stage input (recv target / embedding output / previous stage output)
    bf16* out = nullptr;   // stage output (= last layer x_out; forward send source)
    bf16 *lnf = nullptr, *logits = nullptr;
    float *muf = nullptr, *rsf = nullptr;
    bf16* gin = nullptr;   // grad wrt stage output (backward recv target / next stage's gout)
    bf16* gout = nullptr;  // grad wrt stage input (backward send source)
};

struct LocalStage {
    i64 stage = 0;
    int64_t shard_n = 0;
    // Sharded variants (n_dp >= 2, DP_FS / DP_PS): the stage vector is cut into segments (the
    // embeddings, each layer, the head) and every segment is sharded across the DP ranks, so a
    // rank's optimizer shard is the concatenation of its 1/n_dp slice of every segment. One
    // segment's gradients can then be reduce-scattered (and its weights all-gathered) on their
    // own, as soon as that layer's backward is done. seg = boundaries in the stage vector;
    // segment s of rank r = [seg[s] + r * len_s / n_dp, + len_s / n_dp) -> shard offset seg[s] / n_dp.
    std::vector<int64_t> seg;
    std::vector<char> seg_done;  // segments already reduced (and updated) in the current step
    std::vector<cudaEvent_t> seg_ev;  // per segment: its latest reduce-scatter has read the gradient
    int64_t nd = 1, r = 0;       // shard degree and this rank's slice (1, 0 when not sharded)
    int n_units = 0;             // reduction units of this stage per step (Reduce tasks)
    bf16* w16 = nullptr;      // resident compute weights (not DP_FS with n_dp >= 2)
    float* grad = nullptr;    // full f32 gradient (accumulated across micro-batches; pooled: inside gbuf)
    float *master = nullptr, *m = nullptr, *v = nullptr;  // f32 optimizer shard
    float* gshard = nullptr;  // reduced gradient shard (sharded variants; null = transient per segment)
    bf16* w16_shard = nullptr;
};

// Segment boundaries of a stage for per-segment sharding: embeddings | each layer | head, when
// every segment splits into n_dp slices of whole 8-element groups; otherwise the whole stage.
std::vector<int64_t> shard_segments(const StageLayout& L, i64 n_dp) {
    std::vector<int64_t> b{0};
    for (const LayerParams& P : L.layers)
        if (P.ln1_g > b.back()) b.push_back(P.ln1_g);
    if (L.last && L.lnf_g > b.back()) b.push_back(L.lnf_g);
    b.push_back(L.padded);
    for (size_t i = 0; i + 1 < b.size(); ++i)
        if ((b[i + 1] - b[i]) % (8 * n_dp) != 0) return {0, L.padded};
    return b;
}

// f(full-vector offset, length, shard offset) for each slice this rank owns
template <class F>
void for_each_chunk(const LocalStage& ls, F&& f) {
    for (size_t s = 0; s + 1 < ls.seg.size(); ++s) {
        const int64_t len = (ls.seg[s + 1] - ls.seg[s]) / ls.nd;
        f(ls.seg[s] + ls.r * len, len, ls.seg[s] / ls.nd);
    }
}

// bf16 weights of segments [s0, s1): every rank's slices -> the full vector dst (all ranks)
void all_gather_segments(const LocalStage& ls, bf16* dst, size_t s0, size_t s1, ncclComm_t comm, cudaStream_t st) {
    NK(ncclGroupStart());
    for (size_t s = s0; s < s1; ++s) {
        const size_t n = static_cast<size_t>((ls.seg[s + 1] - ls.seg[s]) / ls.nd);
        NK(ncclAllGather(ls.w16_shard + ls.seg[s] / ls.nd, dst + ls.seg[s], n, ncclBfloat16, comm, st));
    }
    NK(ncclGroupEnd());
}

// f32 gradients of segments [s0, s1): summed over the ranks, this rank's slices -> dst (shard
// layout, shifted down by `shift` elements); each segment's event is recorded once they are read
void reduce_scatter_segments(const LocalStage& ls, float* dst, size_t s0, size_t s1, ncclComm_t comm,
                             cudaStream_t st, int64_t shift = 0) {
    NK(ncclGroupStart());
    for (size_t s = s0; s < s1; ++s) {
        const size_t n = static_cast<size_t>((ls.seg[s + 1] - ls.seg[s]) / ls.nd);
        NK(ncclReduceScatter(ls.grad + ls.seg[s], dst + ls.seg[s] / ls.nd - shift, n, ncclFloat32, ncclSum, comm,
                             st));
    }
    NK(ncclGroupEnd());
    for (size_t s = s0; s < s1; ++s)
        if (s < ls.seg_ev.size()) CK(cudaEventRecord(ls.seg_ev[s], st));
}

using TaskExec = PlanTask;

struct Executor::Impl {
    int dev = 0;
    cudaStream_t st[S_N] = {};
    ncclComm_t world_comm = nullptr, dp_comm = nullptr;
    std::vector<std::pair<size_t, ncclComm_t>> comm_ids;  // (global uid index, comm) for ordered teardown
    // pipeline hand-off: receive arena (all activation / gradient receive slots of this rank) and
    // its ready flags, both exported by CUDA IPC to the two ring neighbours
    bf16* recv_arena = nullptr;
    uint32_t* recv_flags = nullptr;
    std::map<int, bf16*> peer_arena;       // rank -> mapped receive arena
    std::map<int, uint32_t*> peer_flags;   // rank -> mapped flags
    std::vector<void*> ipc_opened;
    uint32_t xfer_seq = 0;                 // step sequence number written into the flags
    std::vector<void*> allocs;
    // DP_FS all-gather through the copy engines (opt-in): the bf16 shard and full-weight slot buffers are
    // ncclMemAlloc'd and registered as symmetric windows of a CTAPolicy-ZERO DP communicator, so
    // NCCL moves them with copy engines instead of taking SMs from the compute stream
    // (scripts/nccl_sym.cu: 544 vs 407 GB/s per direction at n_dp = 2, no SM kernel)
    bool sym = false;
    std::vector<std::pair<void*, size_t>> sym_bufs;
    std::vector<ncclWindow_t> wins;
    std::vector<LocalStage> local;  // index c
    bf16* slots[2] = {nullptr, nullptr};
    std::vector<std::vector<StageActs>> acts;  // [mb][c]
    // scratch: tmp_h is compute-stream private; the per-layer sets [2] are read by the wgrad
    // stream and alternate by backward layer counter (event hand-offs in both directions)
    bf16* tmp_h = nullptr;
    bf16 *gmid_s[2] = {}, *dpre_s[2] = {}, *dqkv_s[2] = {}, *gout_s[2] = {}, *g_head = nullptr;
    cudaEvent_t ev_a[2] = {}, ev_b[2] = {}, ev_wg[2] = {};
    cudaEvent_t ev_opt[2] = {};  // segment-wise optimizer hand-off (compute, wgrad stream)
    std::vector<cudaEvent_t> rec_ev[2];  // DP_FS: per weight slot, one event per all-gathered segment
    std::vector<cudaEvent_t> done_g;  // per Bwd task: its gradients are complete (compute + wgrad streams)
    // Deferred weight gradients: a backward whose input gradient goes to another device runs its
    // data-gradient chain first and records done_dx, so the send (and the peer's backward) starts
    // before this stage's weight-gradient GEMMs, which then fill the wait for the next task.
    // Per-layer gradient scratch of one stage keeps the chain's outputs until those GEMMs run.
    bool defer_wgrad = false;
    // Lazy token-embedding update (n_dp == 1, stage 0 on this rank): step k's Adam of the wte table
    // runs at the start of step k + 1 — the rows of step k + 1's tokens first, on the compute stream
    // before the lookup, every other row on the DP stream beside the forward — instead of in the
    // step's tail. Each row is still updated once per step with step k's gradient and moments.
    bool lazy_wte = false, wte_pending = false, wte_armed = false, wte_rest = false;
    int wte_step = 0;
    int32_t *wte_mark = nullptr, *wte_list = nullptr, *wte_count = nullptr;
    cudaEvent_t ev_wte_mark = nullptr, ev_wte_done = nullptr;
    std::vector<cudaEvent_t> done_dx;  // per deferring Bwd task: its input gradient is ready
    std::vector<bf16*> dpre_d, dqkv_d, gmid_d, gout_d;  // [layer of the stage]
    float *dq_acc = nullptr, *delta = nullptr;
    int32_t *inputs = nullptr, *labels = nullptr;
    float *row_loss = nullptr, *loss_dev = nullptr, *loss_pinned = nullptr;
    std::vector<TaskExec> order;
    std::vector<cudaEvent_t> done;                // per task id (local tasks)
    std::vector<cudaEvent_t> t_start, t_end;      // timing events
    cudaEvent_t origin = nullptr, step_end = nullptr, stream_end[S_N] = {};
    cudaEvent_t step_done[2] = {};  // ring: the host waits for step k-2 before enqueuing step k
    std::vector<double> tl_start, tl_end;
    int step_no = 0;
    int bwd_layers = 0;  // backward layers processed in the current step (scratch set parity)
    bool wgrad_stream = false;
    bool debug = false;
    bool watchdog = false;  // BFPP_EXEC_WATCHDOG: stall reports without the debug mode's serialisation
    std::vector<int> task_c;                      // local stage index of compute tasks
    KernelStats stats;
    struct Mark {
        int cat;
        double work;
        size_t ev;
    };
    std::vector<cudaEvent_t> ev_pool;
    std::vector<Mark> marks;

    // pooled f32 gradient buffer of the sharded variants + transient shard buffers (DP stream)
    float* gbuf = nullptr;
    int64_t gbuf_n = 0;
    float* gtmp = nullptr;  // reduce-scatter landing buffer of stages that reduce several times
    float* gseg = nullptr;  // per-segment reduced gradient of single-unit stages (then Adam)

    bool dry = false;  // sizing only (ExecOptions::dry_run): no device memory is touched
    uintptr_t fake = 0x10000;
    MemoryPlan* mem = nullptr;
    size_t* total = nullptr;
    template <class T>
    T* alloc(size_t n, int cat, bool window = false) {
        const size_t bytes = std::max<size_t>(n * sizeof(T), 256);
        mem->bytes[cat] += bytes;
        *total += bytes;
        if (dry) {
            void* p = reinterpret_cast<void*>(fake);
            fake += (bytes + 255) / 256 * 256;
            return static_cast<T*>(p);
        }
        void* p = nullptr;
        if (window && sym) {
            NK(ncclMemAlloc(&p, bytes));
            sym_bufs.push_back({p, bytes});
            return static_cast<T*>(p);
        }
        CK(cudaMalloc(&p, bytes));
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
};

Executor::Executor(const ModelSpec& m, const ParallelConfig& c, const ExecOptions& o, int rank, int world,
                   const std::vector<ncclUniqueId>& uids, const TaskGraph* graph)
    : impl_(new Impl), m_(m), c_(c), o_(o), rank_(rank), world_(world) {
    c_.validate(m_);
    if (c_.n_tp != 1) throw SpecError("executor: tensor parallelism (n_tp > 1) is not supported");
    if (c_.grid_size() != world) throw SpecError("executor: n_dp * n_pp must equal the number of ranks");
    if (m_.s_head != 128) throw SpecError("executor: attention kernels need s_head = 128");
    if (m_.s_hidden % 64 || m_.s_mlp % 64 || m_.s_voc % 8)
        throw SpecError("executor: s_hidden and s_mlp must be multiples of 64, s_voc of 8");
    p_ = c_.n_pp;
    v_ = c_.n_loop;
    pp_rank_ = rank % p_;
    dp_rank_ = rank / p_;
    pl_ = place_stages(m_, c_);
    if (graph) {
        // an externally built graph (e.g. the breadth-/depth-first gradient-accumulation graphs of
        // build_accumulation_tasks, schedule.cpp:454-500) must match the placement of c
        if (graph->n_devices != p_ || graph->compute_program.size() != static_cast<size_t>(p_))
            throw SpecError("executor: graph has " + std::to_string(graph->n_devices) + " devices, config n_pp = " +
                            std::to_string(p_));
        i64 n_compute = 0;
        for (const Task& t : graph->tasks) {
            if (t.stage < 0 || t.stage >= pl_.n_stage)
                throw SpecError("executor: graph stage " + std::to_string(t.stage) + " outside the config's " +
                                std::to_string(pl_.n_stage) + " stages");
            if (t.micro_batch >= c_.n_mb)
                throw SpecError("executor: graph micro-batch outside the config's n_mb");
            if ((t.kind == TaskKind::Reduce || t.kind == TaskKind::Reconstruct) && c_.n_dp < 2)
                throw SpecError("executor: graph has data-parallel tasks but n_dp < 2");
            if (t.kind == TaskKind::Reconstruct && c_.dp_variant != DpVariant::DP_FS)
                throw SpecError("executor: graph reconstructs weights but the config is not DP_FS");
            if (t.lane == Lane::Compute) ++n_compute;
        }
        if (n_compute != 2 * pl_.n_stage * c_.n_mb)
            throw SpecError("executor: graph must hold one Fwd and one Bwd per (stage, micro-batch)");
        graph_ = *graph;
    } else {
        graph_ = build_tasks(m_, c_, pl_);
    }
    for (i64 s = 0; s < pl_.n_stage; ++s)
        layouts_.push_back(make_stage_layout(m_, s, pl_.n_stage, pl_.layers_per_stage, c_.n_dp));

    Impl& I = *impl_;
    I.dev = o.device;
    I.dry = o.dry_run;
    I.mem = &mem_;
    I.total = &dev_bytes_;
    if (const char* e = getenv("BFPP_WGRAD_STREAM")) I.wgrad_stream = atoi(e) != 0;
    if (const char* e = getenv("BFPP_EXEC_DEBUG")) I.debug = atoi(e) != 0;
    if (const char* e = getenv("BFPP_EXEC_WATCHDOG")) I.watchdog = atoi(e) != 0;
    // recompute: one working set per rank, so weight gradients stay on the compute stream
    if (o_.recompute) I.wgrad_stream = false;
    const bool fs = c_.n_dp >= 2 && c_.dp_variant == DpVariant::DP_FS;
    // sharded variants: gradients are consumed by reduce-scatters, so the rank's stages share one
    // f32 gradient buffer (reused per segment as the previous unit's reduce-scatters drain it)
    const bool pooled = c_.n_dp >= 2 && c_.dp_variant != DpVariant::DP0;
    // opt-in (BFPP_DP_CE_ALLGATHER=1): +3.6% at N = 4, but 3 of 14 GPT-1.3B N = 4 bench runs hung
    // inside an all-gather on both DP peers ("Copy-engine all-gather")
    if (const char* e = getenv("BFPP_DP_CE_ALLGATHER")) I.sym = fs && !I.dry && atoi(e) != 0;
    if (!I.dry) CK(cudaSetDevice(I.dev));

    // ---- per-task execution plan (host only) ----
    I.order = plan_rank(graph_, pp_rank_, c_.n_dp, pooled);

    // ---- parameters, gradients, optimizer shards ----
    int64_t max_padded = 0;
    std::vector<int> n_units(static_cast<size_t>(v_), 0);  // reduction units per local stage
    for (const Task& t : graph_.tasks)
        if (t.kind == TaskKind::Reduce && t.device == pp_rank_) ++n_units[static_cast<size_t>(t.stage / p_)];
    for (i64 cc = 0; cc < v_; ++cc) max_padded = std::max(max_padded, layouts_[static_cast<size_t>(local_stage(cc))].padded);
    int64_t gtmp_n = 0, gseg_n = 0;
    for (i64 cc = 0; cc < v_; ++cc) {
        LocalStage ls;
        ls.stage = local_stage(cc);
        const StageLayout& L = layouts_[static_cast<size_t>(ls.stage)];
        ls.shard_n = pooled ? L.padded / c_.n_dp : L.padded;
        ls.seg = pooled ? shard_segments(L, c_.n_dp) : std::vector<int64_t>{0, L.padded};
        ls.seg_done.assign(ls.seg.size() - 1, 0);
        ls.nd = pooled ? c_.n_dp : 1;
        ls.r = pooled ? dp_rank_ : 0;
        ls.n_units = n_units[static_cast<size_t>(cc)];
        if (!fs) ls.w16 = I.alloc<bf16>(static_cast<size_t>(L.padded), M_WEIGHTS);
        if (!pooled) ls.grad = I.alloc<float>(static_cast<size_t>(L.padded), M_GRADS);
        ls.master = I.alloc<float>(static_cast<size_t>(ls.shard_n), M_OPTIMIZER);
        ls.m = I.alloc<float>(static_cast<size_t>(ls.shard_n), M_OPTIMIZER);
        ls.v = I.alloc<float>(static_cast<size_t>(ls.shard_n), M_OPTIMIZER);
        if (pooled) {
            // the reduced gradient persists across units only when the stage reduces more than
            // once (DF / GPipe / 1F1B units); a single unit is reduced and updated segment by
            // segment through a transient buffer (kept whole when the optimizer is skipped, so
            // the gradients can be read back)
            if (ls.n_units > 1 || o_.skip_optimizer) {
                ls.gshard = I.alloc<float>(static_cast<size_t>(ls.shard_n), M_GRAD_SHARDS);
            } else {
                for (size_t si = 0; si + 1 < ls.seg.size(); ++si)
                    gseg_n = std::max(gseg_n, (ls.seg[si + 1] - ls.seg[si]) / ls.nd);
            }
            if (ls.n_units > 1) gtmp_n = std::max(gtmp_n, ls.shard_n);
            ls.w16_shard = I.alloc<bf16>(static_cast<size_t>(ls.shard_n), M_WEIGHT_SHARDS, true);
        }
        I.local.push_back(ls);
    }
    if (pooled) {
        I.gbuf = I.alloc<float>(static_cast<size_t>(max_padded), M_GRADS);
        I.gbuf_n = max_padded;
        for (auto& ls : I.local)  // right-aligned: every stage's gradient ends at the buffer end
            ls.grad = I.gbuf + (max_padded - layouts_[static_cast<size_t>(ls.stage)].padded);
        if (gtmp_n) I.gtmp = I.alloc<float>(static_cast<size_t>(gtmp_n), M_GRAD_SHARDS);
        if (gseg_n) I.gseg = I.alloc<float>(static_cast<size_t>(gseg_n), M_GRAD_SHARDS);
    }
    if (fs)
        for (auto& sl : I.slots) sl = I.alloc<bf16>(static_cast<size_t>(max_padded), M_WEIGHTS, true);

    // ---- activations: pooled sets of the live (micro-batch, local stage) pairs ----
    // A forward takes a set, the backward of the same (micro-batch, stage) returns it; set ids are
    // assigned once by walking this device's compute program (the same every step), so the pool
    // holds peak_inflight sets (simulate.cpp:166-191) and reuse is ordered by the compute stream.
    const int64_t T = c_.s_mb * m_.s_seq, h = m_.s_hidden, mlp = m_.s_mlp, V = m_.s_voc, H = m_.n_heads;
    const size_t Th = static_cast<size_t>(T * h);
    const i64 last_stage = pl_.n_stage - 1;
    const bool has_last = pl_.device_of(last_stage) == pp_rank_;
    std::vector<int> set_of(static_cast<size_t>(c_.n_mb * v_), -1), head_of(static_cast<size_t>(c_.n_mb), -1);
    {
        std::vector<int> used, hused;
        auto take = [](std::vector<int>& u) {
            for (size_t k = 0; k < u.size(); ++k)
                if (!u[k]) {
                    u[k] = 1;
                    return static_cast<int>(k);
                }
            u.push_back(1);
            return static_cast<int>(u.size() - 1);
        };
        for (TaskId id : graph_.compute_program[static_cast<size_t>(pp_rank_)]) {
            const Task& t = graph_.tasks[static_cast<size_t>(id)];
            const size_t key = static_cast<size_t>(t.micro_batch * v_ + t.stage / p_);
            const bool head = t.stage == last_stage && !o_.recompute;
            if (t.kind == TaskKind::Fwd) {
                set_of[key] = take(used);
                if (head) head_of[static_cast<size_t>(t.micro_batch)] = take(hused);
            } else {
                used[static_cast<size_t>(set_of[key])] = 0;
                if (head) hused[static_cast<size_t>(head_of[static_cast<size_t>(t.micro_batch)])] = 0;
            }
        }
        mem_.activation_sets = static_cast<int64_t>(used.size());
        mem_.head_sets = static_cast<int64_t>(hused.size());
    }
    const i64 lps = pl_.layers_per_stage;
    // one activation set: per layer either everything the backward reads (no recompute) or only
    // the layer output (the checkpoint; the next layer's input)
    struct LayerSet {
        std::vector<LayerActs> layers;
    };
    auto make_layer_acts = [&](int cat) {
        LayerActs la{};
        la.ln1 = I.alloc<bf16>(Th, cat);
        la.qkv = I.alloc<bf16>(3 * Th, cat);
        la.o = I.alloc<bf16>(Th, cat);
        la.x_mid = I.alloc<bf16>(Th, cat);
        la.ln2 = I.alloc<bf16>(Th, cat);
        la.pre = I.alloc<bf16>(static_cast<size_t>(T * mlp), cat);
        la.act = I.alloc<bf16>(static_cast<size_t>(T * mlp), cat);
        la.mu1 = I.alloc<float>(static_cast<size_t>(T), cat);
        la.rs1 = I.alloc<float>(static_cast<size_t>(T), cat);
        la.mu2 = I.alloc<float>(static_cast<size_t>(T), cat);
        la.rs2 = I.alloc<float>(static_cast<size_t>(T), cat);
        la.lse = I.alloc<float>(static_cast<size_t>(T * H), cat);
        return la;
    };
    LayerActs work{};  // recompute: the one working set
    if (o_.recompute) work = make_layer_acts(M_SCRATCH);
    std::vector<LayerSet> sets(static_cast<size_t>(mem_.activation_sets));
    for (auto& st : sets)
        for (i64 l = 0; l < lps; ++l) {
            LayerActs la = o_.recompute ? work : make_layer_acts(M_ACTIVATIONS);
            la.x_out = I.alloc<bf16>(Th, M_ACTIVATIONS);
            st.layers.push_back(la);
        }
    struct HeadSet {
        bf16 *lnf, *logits;
        float *muf, *rsf;
    };
    auto make_head = [&](int cat) {
        HeadSet hs{};
        hs.lnf = I.alloc<bf16>(Th, cat);
        hs.muf = I.alloc<float>(static_cast<size_t>(T), cat);
        hs.rsf = I.alloc<float>(static_cast<size_t>(T), cat);
        hs.logits = I.alloc<bf16>(static_cast<size_t>(T * V), cat);
        return hs;
    };
    std::vector<HeadSet> heads;
    if (has_last) {
        if (o_.recompute)
            heads.push_back(make_head(M_SCRATCH));
        else
            for (int64_t k = 0; k < mem_.head_sets; ++k) heads.push_back(make_head(M_ACTIVATIONS));
    }

    I.acts.assign(static_cast<size_t>(c_.n_mb), std::vector<StageActs>(static_cast<size_t>(v_)));
    // receive slot (dir 0 = forward activation, 1 = backward gradient) of (mb, local stage c)
    auto slot = [&](int dir, i64 mb, i64 cc) { return static_cast<size_t>((mb * v_ + cc) * 2 + dir); };
    const size_t n_slots = static_cast<size_t>(c_.n_mb * v_ * 2);
    if (p_ >= 2) {
        const size_t arena = n_slots * Th * sizeof(bf16), flags = n_slots * sizeof(uint32_t) + 256;
        if (!I.dry) {
            CK(cudaSetDevice(I.dev));
            CK(cudaMalloc(&I.recv_arena, arena));
            CK(cudaMalloc(&I.recv_flags, flags));
            CK(cudaMemset(I.recv_flags, 0, n_slots * sizeof(uint32_t)));
        }
        mem_.bytes[M_PP_BUFFERS] += arena + flags;
        dev_bytes_ += arena + flags;
    }
    for (i64 mb = 0; mb < c_.n_mb; ++mb) {
        for (i64 cc = 0; cc < v_; ++cc) {
            StageActs& a = I.acts[static_cast<size_t>(mb)][static_cast<size_t>(cc)];
            const i64 s = local_stage(cc);
            const StageLayout& L = layouts_[static_cast<size_t>(s)];
            const LayerSet& set = sets[static_cast<size_t>(set_of[static_cast<size_t>(mb * v_ + cc)])];
            // input: aliases the previous stage's output when both live on this device
            if (s > 0 && pl_.device_of(s - 1) == pp_rank_)
                a.in = I.acts[static_cast<size_t>(mb)][static_cast<size_t>(cc - 1)].out;
            else if (s > 0)
                a.in = I.recv_arena + slot(0, mb, cc) * Th;  // written by the previous rank's copy engine
            else
                a.in = I.alloc<bf16>(Th, M_ACTIVATIONS);     // embedding output
            bf16* x = a.in;
            for (size_t l = 0; l < L.layers.size(); ++l) {
                LayerActs la = set.layers[l];
                la.x_in = x;
                x = la.x_out;
                a.layers.push_back(la);
            }
            a.out = x;
            if (L.last) {
                const HeadSet& hs = heads[o_.recompute ? 0 : static_cast<size_t>(head_of[static_cast<size_t>(mb)])];
                a.lnf = hs.lnf;
                a.muf = hs.muf;
                a.rsf = hs.rsf;
                a.logits = hs.logits;
            }
            if (!L.first) a.gout = I.alloc<bf16>(Th, M_PP_BUFFERS);
        }
        // gin: the next stage's gout when it lives on this device, else a receive buffer
        for (i64 cc = 0; cc < v_; ++cc) {
            StageActs& a = I.acts[static_cast<size_t>(mb)][static_cast<size_t>(cc)];
            const i64 s = local_stage(cc);
            if (s == pl_.n_stage - 1) continue;
            if (pl_.device_of(s + 1) == pp_rank_)
                a.gin = I.acts[static_cast<size_t>(mb)][static_cast<size_t>(cc + 1)].gout;
            else
                a.gin = I.recv_arena + slot(1, mb, cc) * Th;
        }
    }
    I.tmp_h = I.alloc<bf16>(Th, M_SCRATCH);
    I.g_head = I.alloc<bf16>(Th, M_SCRATCH);
    for (int k = 0; k < 2; ++k) {
        I.gmid_s[k] = I.alloc<bf16>(Th, M_SCRATCH);
        I.gout_s[k] = I.alloc<bf16>(Th, M_SCRATCH);
        I.dpre_s[k] = I.alloc<bf16>(static_cast<size_t>(T * mlp), M_SCRATCH);
        I.dqkv_s[k] = I.alloc<bf16>(3 * Th, M_SCRATCH);
    }
    I.lazy_wte = c_.n_dp == 1 && !o_.skip_optimizer && pl_.device_of(0) == pp_rank_;
    if (const char* e = getenv("BFPP_LAZY_WTE")) I.lazy_wte = I.lazy_wte && atoi(e) != 0;  // A/B switch
    if (I.lazy_wte) {
        I.wte_mark = I.alloc<int32_t>(static_cast<size_t>(V), M_SCRATCH);
        I.wte_list = I.alloc<int32_t>(static_cast<size_t>(c_.n_mb * T), M_SCRATCH);
        I.wte_count = I.alloc<int32_t>(1, M_SCRATCH);
    }
    I.defer_wgrad = p_ >= 2 && !I.wgrad_stream && !o_.recompute;
    if (const char* e = getenv("BFPP_DEFER_WGRAD")) I.defer_wgrad = I.defer_wgrad && atoi(e) != 0;  // A/B switch
    if (I.defer_wgrad)
        for (i64 j = 0; j < pl_.layers_per_stage; ++j) {
            I.dpre_d.push_back(I.alloc<bf16>(static_cast<size_t>(T * mlp), M_SCRATCH));
            I.dqkv_d.push_back(I.alloc<bf16>(3 * Th, M_SCRATCH));
            I.gmid_d.push_back(I.alloc<bf16>(Th, M_SCRATCH));
            I.gout_d.push_back(I.alloc<bf16>(Th, M_SCRATCH));
        }
    I.dq_acc = I.alloc<float>(Th, M_SCRATCH);
    I.delta = I.alloc<float>(static_cast<size_t>(T * H), M_SCRATCH);
    I.inputs = I.alloc<int32_t>(static_cast<size_t>(c_.n_mb * T), M_SCRATCH);
    I.labels = I.alloc<int32_t>(static_cast<size_t>(c_.n_mb * T), M_SCRATCH);
    I.row_loss = I.alloc<float>(static_cast<size_t>(c_.n_mb * T), M_SCRATCH);
    I.loss_dev = I.alloc<float>(4, M_SCRATCH);
    if (I.dry) return;  // sizing only: no streams, communicators, initialisation or events

    CK(cudaSetDevice(I.dev));
    // The pipeline receive streams block in cuStreamWaitValue32 until a peer's copy lands; a send
    // stream that shares their hardware queue would wait behind them and the ring would hang.
    // CUDA maps streams onto CUDA_DEVICE_MAX_CONNECTIONS queues (default 8); the package sets 32
    // before CUDA initialises, but a user value (1 is common in Megatron setups) wins.
    if (p_ >= 2) {
        const char* e = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
        const int conns = e ? atoi(e) : 8;
        if (conns < S_N)
            throw SpecError("executor: CUDA_DEVICE_MAX_CONNECTIONS=" + std::to_string(conns) +
                            " gives the executor's " + std::to_string(S_N) +
                            " streams fewer hardware queues than streams; pipeline hand-offs (n_pp >= 2) can "
                            "deadlock. Set it to >= 32 before CUDA initialises (import the package first).");
    }
    // Stream priorities: compute and pipeline hand-offs high, the DP lane (all-gather,
    // reduce-scatter, Adam) low, so bandwidth-bound optimizer blocks fill gaps instead of
    // delaying the compute stream's CTAs.
    {
        int least = 0, greatest = 0;
        CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        const int wgrad_prio = greatest + 1 <= least ? greatest + 1 : greatest;
        for (int s = 0; s < S_N; ++s)
            CK(cudaStreamCreateWithPriority(&I.st[s], cudaStreamNonBlocking,
                                            s == S_DP ? least : s == S_WGRAD ? wgrad_prio : greatest));
    }

    // ---- NCCL communicators (uid layout: see bfpp_exec_n_comm_ids): world (IPC handle exchange,
    // teardown barrier) and one DP group per pipeline rank. Pipeline hand-offs do not use NCCL.
    {
        const size_t need = static_cast<size_t>(1 + p_);
        if (world > 1 && uids.size() < need) throw SpecError("executor: not enough NCCL unique ids");
        NK(ncclGroupStart());
        if (world > 1) NK(ncclCommInitRank(&I.world_comm, world, uids[0], rank));
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        if (I.sym) cfg.CTAPolicy = NCCL_CTA_POLICY_ZERO;  // copy-engine all-gathers on the windows below
        if (c_.n_dp >= 2)
            NK(ncclCommInitRankConfig(&I.dp_comm, static_cast<int>(c_.n_dp),
                                      uids[static_cast<size_t>(1 + pp_rank_)], static_cast<int>(dp_rank_), &cfg));
        NK(ncclGroupEnd());
        // symmetric windows: every DP peer allocated the same buffers in the same order
        for (auto& b : I.sym_bufs) {
            ncclWindow_t w;
            NK(ncclCommWindowRegister(I.dp_comm, b.first, b.second, &w, NCCL_WIN_COLL_SYMMETRIC));
            I.wins.push_back(w);
        }
        if (I.world_comm) I.comm_ids.push_back({0, I.world_comm});
        if (I.dp_comm) I.comm_ids.push_back({static_cast<size_t>(1 + pp_rank_), I.dp_comm});
    }
    if (I.gbuf) CK(cudaMemset(I.gbuf, 0, static_cast<size_t>(max_padded) * 4));
    for (auto& ls : I.local) {
        if (!pooled) CK(cudaMemset(ls.grad, 0, static_cast<size_t>(layouts_[static_cast<size_t>(ls.stage)].padded) * 4));
        CK(cudaMemset(ls.m, 0, static_cast<size_t>(ls.shard_n) * 4));
        CK(cudaMemset(ls.v, 0, static_cast<size_t>(ls.shard_n) * 4));
        ls.seg_ev.resize(ls.seg.size() - 1);
        for (auto& e : ls.seg_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (fs) {
        size_t max_seg = 1;
        for (const auto& ls : I.local) max_seg = std::max(max_seg, ls.seg.size() - 1);
        for (auto& evs : I.rec_ev) {
            evs.resize(max_seg);
            for (auto& e : evs) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    // default initialisation: N(0, std), output projections std/sqrt(2L), LayerNorm (1, 0)
    for (auto& ls : I.local) {
        const StageLayout& L = layouts_[static_cast<size_t>(ls.stage)];
        int64_t gbase = 0;  // global element offset of this stage (model order, split-independent)
        for (i64 s = 0; s < ls.stage; ++s) gbase += layouts_[static_cast<size_t>(s)].numel;
        CK(cudaMemset(ls.master, 0, static_cast<size_t>(ls.shard_n) * 4));
        for (const Segment& sg : init_segments(L, m_, o.init_std))
            for_each_chunk(ls, [&](int64_t off, int64_t n, int64_t soff) {
                const int64_t lo = std::max(sg.off, off), hi = std::min(sg.off + sg.n, off + n);
                if (lo >= hi) return;
                init_normal(ls.master + soff + (lo - off), nullptr, hi - lo, sg.mean, sg.std, o.seed,
                            static_cast<uint64_t>(gbase + lo), I.st[S_COMPUTE]);
            });
        if (ls.w16_shard) f32_to_bf16(ls.master, ls.w16_shard, ls.shard_n, I.st[S_COMPUTE]);
        if (ls.w16) {
            if (ls.w16_shard)  // DP_PS: replicated weights assembled from the optimizer shards
                all_gather_segments(ls, ls.w16, 0, ls.seg.size() - 1, I.dp_comm, I.st[S_COMPUTE]);
            else
                f32_to_bf16(ls.master, ls.w16, ls.shard_n, I.st[S_COMPUTE]);
        }
    }
    for (int k = 0; k < 2; ++k) {
        CK(cudaEventCreateWithFlags(&I.ev_a[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&I.ev_b[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&I.ev_wg[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&I.ev_opt[k], cudaEventDisableTiming));
    }
    CK(cudaMallocHost(&I.loss_pinned, sizeof(float)));

    // ---- CUDA IPC: map the ring neighbours' receive arenas and flags ----
    if (p_ >= 2) {
        struct Handles {
            cudaIpcMemHandle_t arena, flags;
        };
        Handles mine{};
        CK(cudaIpcGetMemHandle(&mine.arena, I.recv_arena));
        CK(cudaIpcGetMemHandle(&mine.flags, I.recv_flags));
        uint8_t *d_all = nullptr, *d_mine = nullptr;
        CK(cudaMalloc(&d_all, sizeof(Handles) * static_cast<size_t>(world)));
        CK(cudaMalloc(&d_mine, sizeof(Handles)));
        CK(cudaMemcpy(d_mine, &mine, sizeof(Handles), cudaMemcpyHostToDevice));
        NK(ncclAllGather(d_mine, d_all, sizeof(Handles), ncclUint8, I.world_comm, I.st[S_COMPUTE]));
        std::vector<Handles> all(static_cast<size_t>(world));
        CK(cudaMemcpyAsync(all.data(), d_all, sizeof(Handles) * static_cast<size_t>(world), cudaMemcpyDeviceToHost,
                           I.st[S_COMPUTE]));
        CK(cudaStreamSynchronize(I.st[S_COMPUTE]));
        CK(cudaFree(d_all));
        CK(cudaFree(d_mine));
        for (i64 nb : {(pp_rank_ + 1) % p_, (pp_rank_ - 1 + p_) % p_}) {
            const int r = static_cast<int>(dp_rank_ * p_ + nb);
            if (I.peer_arena.count(r)) continue;
            void *pa = nullptr, *pf = nullptr;
            CK(cudaIpcOpenMemHandle(&pa, all[static_cast<size_t>(r)].arena, cudaIpcMemLazyEnablePeerAccess));
            CK(cudaIpcOpenMemHandle(&pf, all[static_cast<size_t>(r)].flags, cudaIpcMemLazyEnablePeerAccess));
            I.peer_arena[r] = static_cast<bf16*>(pa);
            I.peer_flags[r] = static_cast<uint32_t*>(pf);
            I.ipc_opened.push_back(pa);
            I.ipc_opened.push_back(pf);
        }
    }

    // ---- per-task events ----
    const size_t n = graph_.tasks.size();
    I.done.assign(n, nullptr);
    I.done_g.assign(n, nullptr);
    I.done_dx.assign(n, nullptr);
    I.t_start.assign(n, nullptr);
    I.t_end.assign(n, nullptr);
    I.task_c.assign(n, -1);
    I.tl_start.assign(n, NAN);
    I.tl_end.assign(n, NAN);
    for (const TaskExec& te : I.order) {
        const Task& t = graph_.tasks[static_cast<size_t>(te.id)];
        if (t.lane == Lane::Compute) I.task_c[static_cast<size_t>(te.id)] = static_cast<int>(t.stage / p_);
        CK(cudaEventCreateWithFlags(&I.done[static_cast<size_t>(te.id)], cudaEventDisableTiming));
        if (t.kind == TaskKind::Bwd)
            CK(cudaEventCreateWithFlags(&I.done_g[static_cast<size_t>(te.id)], cudaEventDisableTiming));
        if (t.kind == TaskKind::Bwd && I.defer_wgrad && t.stage > 0 && pl_.device_of(t.stage - 1) != pp_rank_)
            CK(cudaEventCreateWithFlags(&I.done_dx[static_cast<size_t>(te.id)], cudaEventDisableTiming));
    }
    set_flags(o.record_timeline, o.profile_kernels);
    CK(cudaEventCreate(&I.origin));
    if (I.lazy_wte) {
        CK(cudaEventCreateWithFlags(&I.ev_wte_mark, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&I.ev_wte_done, cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&I.step_end, cudaEventDisableTiming));
    for (auto& e : I.step_done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
    for (auto& e : I.stream_end) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(I.step_end, I.st[S_COMPUTE]));
    CK(cudaStreamSynchronize(I.st[S_COMPUTE]));
}


Executor::~Executor() {
    Impl& I = *impl_;
    if (I.dry) return;
    cudaSetDevice(I.dev);
    cudaDeviceSynchronize();
    // Tear communicators down in ascending global id order so that the two members of
    // every 2-rank edge communicator finalise it at the same point (the forward ring
    // d -> d+1 and its wrap cross, so per-rank "out before in" orders would cycle).
    if (I.world_comm) {  // no peer may still be copying into this rank's arena
        float* one = nullptr;
        if (cudaMalloc(&one, sizeof(float)) == cudaSuccess) {
            ncclAllReduce(one, one, 1, ncclFloat32, ncclSum, I.world_comm, I.st[S_COMPUTE]);
            cudaStreamSynchronize(I.st[S_COMPUTE]);
            cudaFree(one);
        }
    }
    for (void* p : I.ipc_opened) cudaIpcCloseMemHandle(p);
    if (I.recv_arena) cudaFree(I.recv_arena);
    if (I.recv_flags) cudaFree(I.recv_flags);
    std::vector<std::pair<size_t, ncclComm_t>> comms(I.comm_ids.begin(), I.comm_ids.end());
    std::sort(comms.begin(), comms.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (ncclWindow_t w : I.wins) ncclCommWindowDeregister(I.dp_comm, w);
    for (auto& kv : comms) ncclCommDestroy(kv.second);
    for (auto& b : I.sym_bufs) ncclMemFree(b.first);
    for (auto e : I.done)
        if (e) cudaEventDestroy(e);
    for (auto e : I.t_start)
        if (e) cudaEventDestroy(e);
    for (auto e : I.t_end)
        if (e) cudaEventDestroy(e);
    for (auto e : I.ev_pool) cudaEventDestroy(e);
    for (auto& evs : I.rec_ev)
        for (auto e : evs)
            if (e) cudaEventDestroy(e);
    for (auto e : I.done_dx)
        if (e) cudaEventDestroy(e);
    for (auto e : I.done_g)
        if (e) cudaEventDestroy(e);
    for (auto& ls : I.local)
        for (auto e : ls.seg_ev)
            if (e) cudaEventDestroy(e);
    for (int k = 0; k < 2; ++k)
        for (cudaEvent_t e : {I.ev_a[k], I.ev_b[k], I.ev_wg[k], I.ev_opt[k]})
            if (e) cudaEventDestroy(e);
    if (I.origin) cudaEventDestroy(I.origin);
    for (cudaEvent_t e : {I.ev_wte_mark, I.ev_wte_done})
        if (e) cudaEventDestroy(e);
    if (I.step_end) cudaEventDestroy(I.step_end);
    for (auto e : I.step_done)
        if (e) cudaEventDestroy(e);
    for (auto e : I.stream_end)
        if (e) cudaEventDestroy(e);
    for (void* p : I.allocs) cudaFree(p);
    if (I.loss_pinned) cudaFreeHost(I.loss_pinned);
    for (auto s : I.st)
        if (s) cudaStreamDestroy(s);
}

// ---------------------------------------------------------------------------------------------
namespace {

void gemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int amn, const void* B,
          int64_t ldb, int bmn, void* D, int64_t ldd, int epi, const void* aux = nullptr, int64_t ldaux = 0,
          void* aux_out = nullptr, int64_t ldaux_out = 0, int accumulate = 0) {
    GemmArgs g;
    g.M = M, g.N = N, g.K = K;
    g.A = A, g.lda = lda, g.a_mn_major = amn;
    g.B = B, g.ldb = ldb, g.b_mn_major = bmn;
    g.D = D, g.ldd = ldd;
    g.aux = aux, g.ldaux = ldaux, g.aux_out = aux_out, g.ldaux_out = ldaux_out;
    g.epilogue = epi, g.accumulate = accumulate;
    gemm_bf16(g, st);
}

}  // namespace

void Executor::step(const int32_t* tokens, bool on_host, float* loss_host, float* loss_dev) {
    Impl& I = *impl_;
    CK(cudaSetDevice(I.dev));
    cudaStream_t cs = I.st[S_COMPUTE], ds = I.st[S_DP];
    ++I.step_no;
    ++I.xfer_seq;
    // Cap the host's run-ahead at two steps ("frequent non-blocking syncs to cap
    // the kernel queue"): a rank that does not read the loss could otherwise enqueue steps until
    // its launch queue / NCCL proxy FIFOs fill while its peers still wait for this step's sends.
    if (I.debug) fprintf(stderr, "[bfpp rank %d] step %d begin\n", rank_, I.step_no);
    // debug mode: no run-ahead at all, so a stalled step is reported by the watchdog below
    const int cap_slot = I.debug ? (I.step_no - 1) & 1 : I.step_no & 1;
    if (I.step_no >= (I.debug ? 2 : 3)) wait_step_event(I.step_done[cap_slot], I.step_no - 2);
    if (I.debug) fprintf(stderr, "[bfpp rank %d] step %d run-ahead cap passed\n", rank_, I.step_no);
    for (int s = 0; s < S_N; ++s) CK(cudaStreamWaitEvent(I.st[s], I.step_end, 0));
    const int64_t T = c_.s_mb * m_.s_seq, h = m_.s_hidden, mlp = m_.s_mlp, V = m_.s_voc;
    const int H = static_cast<int>(m_.n_heads), S = static_cast<int>(m_.s_seq), B = static_cast<int>(c_.s_mb);
    const bool has_first = pl_.device_of(0) == pp_rank_, has_last = pl_.device_of(pl_.n_stage - 1) == pp_rank_;
    if (has_first || has_last) {
        const size_t rows = static_cast<size_t>(c_.n_mb * c_.s_mb);
        const size_t w = static_cast<size_t>(m_.s_seq) * 4, pitch = static_cast<size_t>(m_.s_seq + 1) * 4;
        const cudaMemcpyKind k = on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        CK(cudaMemcpy2DAsync(I.inputs, w, tokens, pitch, w, rows, k, cs));
        CK(cudaMemcpy2DAsync(I.labels, w, tokens + 1, pitch, w, rows, k, cs));
    }
    if (o_.record_timeline) {
        // A common time origin for the ranks' timelines: every compute stream passes a 1-float
        // all-reduce on the world communicator before recording its origin (residual skew = the
        // all-reduce's completion skew, microseconds), and this rank's other streams start after it.
        if (I.world_comm)
            NK(ncclAllReduce(I.loss_dev + 2, I.loss_dev + 2, 1, ncclFloat32, ncclSum, I.world_comm, cs));
        CK(cudaEventRecord(I.origin, cs));
        for (int s = 1; s < S_N; ++s) CK(cudaStreamWaitEvent(I.st[s], I.origin, 0));
    }
    const float grad_scale = 1.f / static_cast<float>(c_.n_dp * c_.n_mb * T);
    const bool fs = c_.n_dp >= 2 && c_.dp_variant == DpVariant::DP_FS;

    I.stats = KernelStats{};
    I.marks.clear();
    I.bwd_layers = 0;
    size_t ev_next = 0;
    // every kernel of the step goes through K(): counts launches, optionally brackets with events
    auto K = [&](int cat, double work, int n_launch, cudaStream_t st, auto&& fn) {
        I.stats.launches[cat] += n_launch;
        if (!o_.profile_kernels) {
            fn();
            return;
        }
        while (I.ev_pool.size() < ev_next + 2) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            I.ev_pool.push_back(e);
        }
        CK(cudaEventRecord(I.ev_pool[ev_next], st));
        fn();
        CK(cudaEventRecord(I.ev_pool[ev_next + 1], st));
        I.marks.push_back({cat, work, ev_next});
        ev_next += 2;
    };
    auto G = [&](cudaStream_t st, int64_t M, int64_t N, int64_t Kd, const void* A, int64_t lda, int amn,
                 const void* Bp, int64_t ldb, int bmn, void* D, int64_t ldd, int epi, const void* aux = nullptr,
                 int64_t ldaux = 0, void* aux_out = nullptr, int64_t ldaux_out = 0, int acc = 0) {
        K(K_GEMM, 2.0 * M * N * Kd, 1, st,
          [&] { gemm(st, M, N, Kd, A, lda, amn, Bp, ldb, bmn, D, ldd, epi, aux, ldaux, aux_out, ldaux_out, acc); });
    };
    // two independent f32 weight-gradient GEMMs (store or reduce-add) in one grouped launch
    struct WG {
        int64_t M, N, Kd;
        const void* A;
        int64_t lda;
        int amn;
        const void* B;
        int64_t ldb;
        int bmn;
        void* D;
        int64_t ldd;
    };
    auto G2 = [&](cudaStream_t st, const WG& x, const WG& y, int acc) {
        auto args = [&](const WG& w) {
            GemmArgs a;
            a.M = w.M;
            a.N = w.N;
            a.K = w.Kd;
            a.A = w.A;
            a.lda = w.lda;
            a.a_mn_major = w.amn;
            a.B = w.B;
            a.ldb = w.ldb;
            a.b_mn_major = w.bmn;
            a.D = w.D;
            a.ldd = w.ldd;
            a.epilogue = GEMM_EPI_F32;
            a.accumulate = acc;
            return a;
        };
        const GemmArgs ax = args(x), ay = args(y);
        K(K_GEMM, 2.0 * (x.M * x.N * x.Kd + y.M * y.N * y.Kd), gemm_pairable(ax, ay) ? 1 : 2, st,
          [&] { gemm_bf16_pair(ax, ay, st); });
    };
    const double Th2 = 2.0 * static_cast<double>(T * h);  // bytes of one [T,h] bf16 activation
    const double attn_flops = 2.0 * B * static_cast<double>(S) * (S + 1) * static_cast<double>(h);  // causal, fwd
    auto LNF = [&](cudaStream_t st, const bf16* x, const bf16* g, const bf16* b, bf16* y, float* mu, float* rs) {
        K(K_LAYERNORM, 2 * Th2, 1, st,
          [&] { layernorm_fwd(x, g, b, y, mu, rs, static_cast<int>(T), static_cast<int>(h), 1e-5f, st); });
    };
    auto LNB = [&](cudaStream_t st, const bf16* dy, const bf16* x, const bf16* g, const float* mu, const float* rs,
                   const bf16* dres, bf16* dx, float* dg, float* db, int acc) {
        K(K_LAYERNORM, (dres ? 6 : 5) * Th2, layernorm_bwd_launches(static_cast<int>(h)), st, [&] {
            layernorm_bwd(dy, x, g, mu, rs, dres, dx, dg, db, static_cast<int>(T), static_cast<int>(h), st, acc);
        });
    };

    auto weights = [&](const TaskExec& te, int cidx) -> const bf16* {
        if (fs) return I.slots[te.slot];
        return I.local[static_cast<size_t>(cidx)].w16;
    };
    // Adam over elements [lo, hi) of a stage's (shard of) master weights / moments; gradient = g
    // (elements lo..hi) or, by default, the stage's gradient shard / full gradient at lo
    auto adam = [&](LocalStage& ls, cudaStream_t st, int64_t lo = 0, int64_t hi = -1, size_t s0 = 0,
                    size_t s1 = SIZE_MAX, const float* g = nullptr) {
        if (o_.skip_optimizer) return;
        if (hi < 0) hi = ls.shard_n;
        if (s1 == SIZE_MAX) s1 = ls.seg.size() - 1;
        const bool sharded = ls.w16_shard != nullptr;
        if (!g) g = (sharded ? ls.gshard : ls.grad) + lo;
        bf16* w = sharded ? ls.w16_shard : ls.w16;
        K(K_ADAM, 30.0 * static_cast<double>(hi - lo), 1, st, [&] {
            adam_update(ls.master + lo, ls.m + lo, ls.v + lo, const_cast<float*>(g), w + lo, hi - lo, o_.lr, o_.beta1,
                        o_.beta2, o_.eps, o_.weight_decay, I.step_no, 0, st);
        });
        if (sharded && c_.dp_variant == DpVariant::DP_PS) all_gather_segments(ls, ls.w16, s0, s1, I.dp_comm, st);
    };
    // Reduction of one stage segment (sharded variants): reduce-scatter its gradients into this
    // rank's slice, fold in earlier units, and (last unit) update it — on stream st. A stage with
    // a single unit and no persistent shard goes through the transient per-segment buffer.
    auto reduce_segment = [&](LocalStage& ls, cudaStream_t st, size_t si, bool first_unit, bool update) {
        const int64_t lo = ls.seg[si] / ls.nd, hi = ls.seg[si + 1] / ls.nd;
        if (!ls.gshard) {
            reduce_scatter_segments(ls, I.gseg, si, si + 1, I.dp_comm, st, lo);
            if (update) adam(ls, st, lo, hi, si, si + 1, I.gseg);
        } else {
            reduce_scatter_segments(ls, first_unit ? ls.gshard : I.gtmp, si, si + 1, I.dp_comm, st);
            if (!first_unit)
                K(K_MISC, 12.0 * static_cast<double>(hi - lo), 1, st,
                  [&] { add_f32_kernel<<<296, 256, 0, st>>>(ls.gshard + lo, I.gtmp + lo, hi - lo); });
            if (update) adam(ls, st, lo, hi, si, si + 1);
        }
        ls.seg_done[si] = 1;
    };
    // Under DP_FS / DP_PS every reduction unit runs segment by segment inside the backward that
    // completes it: each layer is reduce-scattered (and, in the stage's last unit, updated) on the
    // DP stream as soon as its gradients are final, leaving only the last segments for the Reduce
    // task, and the pooled gradient buffer drains in the order the next unit refills it.
    auto early_segment = [&](LocalStage& ls, cudaStream_t st, cudaStream_t ws, int64_t seg_start, bool first_unit,
                             bool update) {
        size_t si = 0;
        while (si + 1 < ls.seg.size() && ls.seg[si] != seg_start) ++si;
        if (si + 1 >= ls.seg.size()) return;  // single-segment layout: the Reduce task does it all
        CK(cudaEventRecord(I.ev_opt[0], st));
        CK(cudaStreamWaitEvent(ds, I.ev_opt[0], 0));
        if (ws != st) {
            CK(cudaEventRecord(I.ev_opt[1], ws));
            CK(cudaStreamWaitEvent(ds, I.ev_opt[1], 0));
        }
        reduce_segment(ls, ds, si, first_unit, update);
    };
    // Pooled gradients: before a unit's first backward overwrites stage-vector range [lo, hi) of
    // its stage, wait until every reduce-scatter still reading that part of the shared buffer
    // (any local stage's segment overlapping it) has finished.
    auto guard_grads = [&](const LocalStage& ls, cudaStream_t st, cudaStream_t ws, int64_t lo, int64_t hi) {
        if (!I.gbuf) return;
        const int64_t blo = (ls.grad - I.gbuf) + lo, bhi = (ls.grad - I.gbuf) + hi;
        for (const LocalStage& o2 : I.local) {
            const int64_t base = o2.grad - I.gbuf;
            for (size_t si = 0; si + 1 < o2.seg.size(); ++si)
                if (base + o2.seg[si] < bhi && base + o2.seg[si + 1] > blo) {
                    CK(cudaStreamWaitEvent(st, o2.seg_ev[si], 0));
                    if (ws != st) CK(cudaStreamWaitEvent(ws, o2.seg_ev[si], 0));
                }
        }
    };
    // n_dp == 1: a parameter segment's gradient is final as soon as the stage's last backward
    // has produced it, so the optimizer runs segment by segment (a layer at a time) on the DP
    // stream, overlapping the rest of the backward; only the last segment is left as a tail.
    auto adam_segment = [&](LocalStage& ls, cudaStream_t st, cudaStream_t ws, int64_t lo, int64_t hi) {
        if (o_.skip_optimizer || hi <= lo) return;
        CK(cudaEventRecord(I.ev_opt[0], st));
        CK(cudaStreamWaitEvent(ds, I.ev_opt[0], 0));
        if (ws != st) {
            CK(cudaEventRecord(I.ev_opt[1], ws));
            CK(cudaStreamWaitEvent(ds, I.ev_opt[1], 0));
        }
        adam(ls, ds, lo, hi);
    };

    for (const TaskExec& te : I.order) {
        const Task& t = graph_.tasks[static_cast<size_t>(te.id)];
        cudaStream_t st = I.st[te.stream];
        // DP_FS: a compute task waits for its weights segment by segment (right before each layer
        // uses them), so it starts as soon as the first segment has been all-gathered
        bool seg_wait = false;
        for (TaskId d : te.waits) {
            const TaskKind dk = graph_.tasks[static_cast<size_t>(d)].kind;
            if (fs && dk == TaskKind::Reconstruct && (t.kind == TaskKind::Fwd || t.kind == TaskKind::Bwd)) {
                seg_wait = true;
                continue;
            }
            // gradient consumers (Reduce) need the wgrad stream's half of a backward task too; a
            // send of a deferring backward needs only its data-gradient chain
            const bool grads = dk == TaskKind::Bwd && t.kind == TaskKind::Reduce;
            cudaEvent_t ev = grads ? I.done_g[static_cast<size_t>(d)] : I.done[static_cast<size_t>(d)];
            if (t.kind == TaskKind::Transfer && dk == TaskKind::Bwd && I.done_dx[static_cast<size_t>(d)])
                ev = I.done_dx[static_cast<size_t>(d)];
            CK(cudaStreamWaitEvent(st, ev, 0));
        }
        // wait for the all-gather of the weight segment that holds stage-vector offset `off`
        auto need_weights = [&](const LocalStage& ls, int64_t off) {
            if (!seg_wait) return;
            size_t si = 0;
            while (si + 2 < ls.seg.size() && ls.seg[si + 1] <= off) ++si;
            CK(cudaStreamWaitEvent(st, I.rec_ev[te.slot][si], 0));
        };
        if (o_.record_timeline) CK(cudaEventRecord(I.t_start[static_cast<size_t>(te.id)], st));
        const int cidx = I.task_c[static_cast<size_t>(te.id)];
        switch (t.kind) {
        case TaskKind::Fwd: {
            const StageLayout& L = layouts_[static_cast<size_t>(t.stage)];
            StageActs& a = I.acts[static_cast<size_t>(t.micro_batch)][static_cast<size_t>(cidx)];
            const bf16* W = weights(te, cidx);
            const LocalStage& lsw = I.local[static_cast<size_t>(cidx)];
            const int32_t* inp = I.inputs + t.micro_batch * T;
            if (L.first) need_weights(lsw, L.wte);
            if (L.first && I.wte_pending) {
                // the previous step's table update: this step's token rows now, the rest beside the forward
                LocalStage& l0 = I.local[static_cast<size_t>(cidx)];
                const int ntok = static_cast<int>(c_.n_mb * T);
                const int64_t base = L.wte;
                auto rows = [&](int listed, cudaStream_t s2) {
                    adam_rows(l0.master + base, l0.m + base, l0.v + base, l0.grad + base, l0.w16 + base, V,
                              static_cast<int>(h), I.wte_mark, I.wte_list, I.wte_count, ntok, listed, o_.lr, o_.beta1,
                              o_.beta2, o_.eps, o_.weight_decay, I.wte_step, s2);
                };
                K(K_MISC, 8.0 * ntok, 1, st,
                  [&] { mark_rows(I.inputs, ntok, I.wte_mark, I.wte_list, I.wte_count, V, st); });
                K(K_ADAM, 30.0 * static_cast<double>(ntok) * h, 1, st, [&] { rows(1, st); });
                CK(cudaEventRecord(I.ev_wte_mark, st));
                I.wte_pending = false;
                I.wte_rest = true;  // the other rows: issued with the step's first backward (below)
                I.wte_armed = true;
            }
            if (L.first)
                K(K_MISC, 3 * Th2, 1, st, [&] {
                    embed_fwd(inp, W + L.wte, W + L.wpe, a.in, static_cast<int>(T), S, static_cast<int>(h), st);
                });
            for (size_t l = 0; l < L.layers.size(); ++l) {
                const LayerParams& P = L.layers[l];
                LayerActs& x = a.layers[l];
                need_weights(lsw, P.ln1_g);
                LNF(st, x.x_in, W + P.ln1_g, W + P.ln1_b, x.ln1, x.mu1, x.rs1);
                G(st, T, 3 * h, h, x.ln1, h, 0, W + P.qkv, h, 0, x.qkv, 3 * h, GEMM_EPI_BF16);
                K(K_ATTN_FWD, attn_flops, 1, st, [&] { attention_fwd(x.qkv, x.o, x.lse, B, S, H, 128, st); });
                G(st, T, h, h, x.o, h, 0, W + P.o, h, 0, x.x_mid, h, GEMM_EPI_RESID, x.x_in, h);
                LNF(st, x.x_mid, W + P.ln2_g, W + P.ln2_b, x.ln2, x.mu2, x.rs2);
                G(st, T, mlp, h, x.ln2, h, 0, W + P.fc1, h, 0, x.act, mlp, GEMM_EPI_GELU, nullptr, 0, x.pre, mlp);
                G(st, T, h, mlp, x.act, mlp, 0, W + P.fc2, mlp, 0, x.x_out, h, GEMM_EPI_RESID, x.x_mid, h);
            }
            if (L.last) {
                need_weights(lsw, L.lnf_g);
                LNF(st, a.out, W + L.lnf_g, W + L.lnf_b, a.lnf, a.muf, a.rsf);
                G(st, T, V, h, a.lnf, h, 0, W + L.head, h, 0, a.logits, V, GEMM_EPI_BF16);
                K(K_MISC, 4.0 * static_cast<double>(T * V), 1, st, [&] {
                    softmax_xent(a.logits, V, I.labels + t.micro_batch * T, I.row_loss + t.micro_batch * T,
                                 static_cast<int>(T), static_cast<int>(V), grad_scale, st);
                });
            }
            break;
        }
        case TaskKind::Bwd: {
            const StageLayout& L = layouts_[static_cast<size_t>(t.stage)];
            StageActs& a = I.acts[static_cast<size_t>(t.micro_batch)][static_cast<size_t>(cidx)];
            LocalStage& ls = I.local[static_cast<size_t>(cidx)];
            const bf16* W = weights(te, cidx);
            float* G_ = ls.grad;
            if (I.wte_rest) {
                // the lazy table update's other rows go on the DP stream at the start of the backward,
                // where it is idle until the first layer's gradients exist, instead of beside the
                // forward (which has no optimizer work to hide behind)
                I.wte_rest = false;
                for (LocalStage& l0 : I.local) {
                    const StageLayout& L0 = layouts_[static_cast<size_t>(l0.stage)];
                    if (!L0.first) continue;
                    const int64_t base = L0.wte;
                    // device order, not host order: the DP stream waits for the compute stream to
                    // reach this backward (after every forward of the step, and after the row marks)
                    CK(cudaEventRecord(I.ev_wte_mark, st));
                    CK(cudaStreamWaitEvent(ds, I.ev_wte_mark, 0));
                    K(K_ADAM, 30.0 * static_cast<double>(V * h), 1, ds, [&] {
                        adam_rows(l0.master + base, l0.m + base, l0.v + base, l0.grad + base, l0.w16 + base, V,
                                  static_cast<int>(h), I.wte_mark, I.wte_list, I.wte_count,
                                  static_cast<int>(c_.n_mb * T), 0, o_.lr, o_.beta1, o_.beta2, o_.eps,
                                  o_.weight_decay, I.wte_step, ds);
                    });
                    CK(cudaEventRecord(I.ev_wte_done, ds));
                }
            }
            // weight-gradient GEMMs: same stream by default (measured faster at T = 2048, where two
            // persistent GEMM grids only interleave at CTA granularity); BFPP_WGRAD_STREAM=1 runs
            // them on a separate stream overlapping the data-gradient chain
            cudaStream_t ws = I.wgrad_stream ? I.st[S_WGRAD] : st;
            const int acc = te.first_in_unit ? 0 : 1;  // the unit's first contribution overwrites
            const bool seg_opt = te.adam_after;  // only set on a backward task when n_dp == 1
            // sharded variants: the backward that completes a reduction unit reduce-scatters it
            // segment by segment (and updates it in the stage's last unit)
            const bool early = te.unit_end_bwd && ls.w16_shard != nullptr && ls.seg.size() > 2;
            const bool guard = te.first_in_unit && I.gbuf != nullptr;
            const size_t nl = L.layers.size();
            // deferred weight gradients: chain first, then (after done_dx) the weight-gradient GEMMs
            // and the per-segment optimizer / reduce-scatter work in the original order
            const bool defer = I.done_dx[static_cast<size_t>(te.id)] != nullptr;
            struct LaterLayer {
                size_t li;
                const bf16 *g, *dpre, *gmid, *dqkv;
            };
            std::vector<LaterLayer> later;
            bool head_later = false;
            // end of layer li's parameters in the stage vector (the last layer of a non-last stage
            // runs to the padded end; n_dp == 1 here for the optimizer segments, so shard = stage)
            auto layer_end = [&](size_t li) -> int64_t {
                return li + 1 < nl ? L.layers[li + 1].ln1_g : (L.last ? L.lnf_g : L.padded);
            };
            // the wgrad stream also writes this stage's gradient buffer: honour the same
            // resource waits (previous unit's reduce-scatter) as the compute stream
            for (TaskId d : te.waits)
                if (graph_.tasks[static_cast<size_t>(d)].kind == TaskKind::Reduce)
                    CK(cudaStreamWaitEvent(ws, I.done[static_cast<size_t>(d)], 0));
            auto wait_wgrad_latest = [&] {
                if (I.bwd_layers > 0) CK(cudaStreamWaitEvent(st, I.ev_wg[(I.bwd_layers - 1) & 1], 0));
            };
            const bf16* g;
            if (L.last) {
                need_weights(ls, L.lnf_g);
                if (o_.recompute) {  // the LM head's logits and dlogits were not kept: recompute them
                    LNF(st, a.out, W + L.lnf_g, W + L.lnf_b, a.lnf, a.muf, a.rsf);
                    G(st, T, V, h, a.lnf, h, 0, W + L.head, h, 0, a.logits, V, GEMM_EPI_BF16);
                    K(K_MISC, 4.0 * static_cast<double>(T * V), 1, st, [&] {
                        softmax_xent(a.logits, V, I.labels + t.micro_batch * T, I.row_loss + t.micro_batch * T,
                                     static_cast<int>(T), static_cast<int>(V), grad_scale, st);
                    });
                }
                if (guard) guard_grads(ls, st, ws, L.lnf_g, L.padded);
                G(st, T, h, V, a.logits, V, 0, W + L.head, h, 1, I.tmp_h, h, GEMM_EPI_BF16);
                CK(cudaEventRecord(I.ev_a[0], st));  // logits/lnf are persistent; only ordering matters
                CK(cudaStreamWaitEvent(ws, I.ev_a[0], 0));
                if (defer)
                    head_later = true;
                else
                    G(ws, V, h, T, a.logits, V, 1, a.lnf, h, 1, G_ + L.head, h, GEMM_EPI_F32, nullptr, 0, nullptr, 0,
                      acc);
                wait_wgrad_latest();  // g_head was last read by an earlier layer's wgrad
                LNB(st, I.tmp_h, a.out, W + L.lnf_g, a.muf, a.rsf, nullptr, I.g_head, G_ + L.lnf_g, G_ + L.lnf_b,
                    acc);
                g = I.g_head;
                if (!defer && seg_opt) adam_segment(ls, st, ws, L.lnf_g, ls.shard_n);
                if (!defer && early) early_segment(ls, st, ws, L.lnf_g, te.reduce_first_unit, te.last_unit_bwd);
            } else {
                g = a.gin;
            }
            for (size_t li = L.layers.size(); li-- > 0;) {
                const LayerParams& P = L.layers[li];
                LayerActs& x = a.layers[li];
                need_weights(ls, P.ln1_g);
                const int lc = I.bwd_layers++;
                const int k = lc & 1;
                // set k was last read by the wgrads of layer lc-2
                if (lc >= 2) CK(cudaStreamWaitEvent(st, I.ev_wg[k], 0));
                if (o_.recompute) {
                    // the layer's forward from its checkpointed input into the working set (its
                    // output x_out is the checkpoint itself and is not recomputed)
                    LNF(st, x.x_in, W + P.ln1_g, W + P.ln1_b, x.ln1, x.mu1, x.rs1);
                    G(st, T, 3 * h, h, x.ln1, h, 0, W + P.qkv, h, 0, x.qkv, 3 * h, GEMM_EPI_BF16);
                    K(K_ATTN_FWD, attn_flops, 1, st, [&] { attention_fwd(x.qkv, x.o, x.lse, B, S, H, 128, st); });
                    G(st, T, h, h, x.o, h, 0, W + P.o, h, 0, x.x_mid, h, GEMM_EPI_RESID, x.x_in, h);
                    LNF(st, x.x_mid, W + P.ln2_g, W + P.ln2_b, x.ln2, x.mu2, x.rs2);
                    G(st, T, mlp, h, x.ln2, h, 0, W + P.fc1, h, 0, x.act, mlp, GEMM_EPI_GELU, nullptr, 0, x.pre, mlp);
                }
                if (guard) guard_grads(ls, st, ws, P.ln1_g, layer_end(li));
                bf16 *gmid = defer ? I.gmid_d[li] : I.gmid_s[k], *dpre = defer ? I.dpre_d[li] : I.dpre_s[k],
                     *dqkv = defer ? I.dqkv_d[li] : I.dqkv_s[k];
                bf16* gnext = (li == 0 && !L.first) ? a.gout : (defer ? I.gout_d[li] : I.gout_s[k]);
                // MLP: x_out = x_mid + gelu(ln2 W1^T) W2^T
                G(st, T, mlp, h, g, h, 0, W + P.fc2, mlp, 1, dpre, mlp, GEMM_EPI_DGELU, x.pre, mlp);
                CK(cudaEventRecord(I.ev_a[k], st));
                CK(cudaStreamWaitEvent(ws, I.ev_a[k], 0));
                // weight gradients of fc2 and fc1: independent, one grouped launch
                if (!defer)
                    G2(ws, {h, mlp, T, g, h, 1, x.act, mlp, 1, G_ + P.fc2, mlp},
                       {mlp, h, T, dpre, mlp, 1, x.ln2, h, 1, G_ + P.fc1, h}, acc);
                G(st, T, h, mlp, dpre, mlp, 0, W + P.fc1, h, 1, I.tmp_h, h, GEMM_EPI_BF16);
                LNB(st, I.tmp_h, x.x_mid, W + P.ln2_g, x.mu2, x.rs2, g, gmid, G_ + P.ln2_g, G_ + P.ln2_b, acc);
                // attention: x_mid = x_in + attn(ln1 Wqkv^T) Wo^T
                G(st, T, h, h, gmid, h, 0, W + P.o, h, 1, I.tmp_h, h, GEMM_EPI_BF16);
                K(K_ATTN_BWD, 2.5 * attn_flops, 3, st, [&] {
                    attention_bwd(x.qkv, x.o, I.tmp_h, x.lse, I.delta, I.dq_acc, dqkv, B, S, H, 128, st);
                });
                CK(cudaEventRecord(I.ev_b[k], st));
                CK(cudaStreamWaitEvent(ws, I.ev_b[k], 0));
                if (defer)
                    later.push_back({li, g, dpre, gmid, dqkv});
                else
                    G2(ws, {h, h, T, gmid, h, 1, x.o, h, 1, G_ + P.o, h},
                       {3 * h, h, T, dqkv, 3 * h, 1, x.ln1, h, 1, G_ + P.qkv, h}, acc);
                CK(cudaEventRecord(I.ev_wg[k], ws));
                G(st, T, h, 3 * h, dqkv, 3 * h, 0, W + P.qkv, h, 1, I.tmp_h, h, GEMM_EPI_BF16);
                // gnext (set k) was last read as g_in by the wgrad of layer lc-1
                if (gnext == I.gout_s[k] && lc >= 1) CK(cudaStreamWaitEvent(st, I.ev_wg[(lc - 1) & 1], 0));
                LNB(st, I.tmp_h, x.x_in, W + P.ln1_g, x.mu1, x.rs1, gmid, gnext, G_ + P.ln1_g, G_ + P.ln1_b, acc);
                g = gnext;
                if (!defer && seg_opt) adam_segment(ls, st, ws, P.ln1_g, layer_end(li));
                if (!defer && early) early_segment(ls, st, ws, P.ln1_g, te.reduce_first_unit, te.last_unit_bwd);
            }
            if (defer) {
                // the input gradient (a.gout) is final: the send may start; then the weight gradients
                CK(cudaEventRecord(I.done_dx[static_cast<size_t>(te.id)], st));
                if (head_later) {
                    G(ws, V, h, T, a.logits, V, 1, a.lnf, h, 1, G_ + L.head, h, GEMM_EPI_F32, nullptr, 0, nullptr, 0,
                      acc);
                    if (seg_opt) adam_segment(ls, st, ws, L.lnf_g, ls.shard_n);
                    if (early) early_segment(ls, st, ws, L.lnf_g, te.reduce_first_unit, te.last_unit_bwd);
                }
                for (const LaterLayer& d : later) {
                    const LayerParams& P = L.layers[d.li];
                    const LayerActs& x = a.layers[d.li];
                    G2(ws, {h, mlp, T, d.g, h, 1, x.act, mlp, 1, G_ + P.fc2, mlp},
                       {mlp, h, T, d.dpre, mlp, 1, x.ln2, h, 1, G_ + P.fc1, h}, acc);
                    G2(ws, {h, h, T, d.gmid, h, 1, x.o, h, 1, G_ + P.o, h},
                       {3 * h, h, T, d.dqkv, 3 * h, 1, x.ln1, h, 1, G_ + P.qkv, h}, acc);
                    if (seg_opt) adam_segment(ls, st, ws, P.ln1_g, layer_end(d.li));
                    if (early) early_segment(ls, st, ws, P.ln1_g, te.reduce_first_unit, te.last_unit_bwd);
                }
            }
            if (L.first && guard) guard_grads(ls, st, ws, 0, L.layers[0].ln1_g);
            if (L.first && I.wte_armed) {  // the lazy table update still reads the previous gradient
                CK(cudaStreamWaitEvent(st, I.ev_wte_done, 0));
                I.wte_armed = false;
            }
            if (L.first && acc == 0) {  // scatter-added gradients need a zeroed start
                CK(cudaMemsetAsync(G_ + L.wte, 0, static_cast<size_t>(V * h) * 4, st));
                CK(cudaMemsetAsync(G_ + L.wpe, 0, static_cast<size_t>(m_.s_seq * h) * 4, st));
            }
            if (L.first)  // iota, radix sort (1-2 launches), per-token and per-position sums
                K(K_MISC, 2 * Th2, 4, st, [&] {
                    embed_bwd(I.inputs + t.micro_batch * T, g, G_ + L.wte, G_ + L.wpe, static_cast<int>(T), S,
                              static_cast<int>(h), st);
                });
            // gradients complete = compute-stream part (LN, embedding) joined into the wgrad stream
            CK(cudaEventRecord(I.done[static_cast<size_t>(te.id)], st));
            CK(cudaStreamWaitEvent(ws, I.done[static_cast<size_t>(te.id)], 0));
            CK(cudaEventRecord(I.done_g[static_cast<size_t>(te.id)], ws));
            if (seg_opt && L.first) {  // embeddings (the token table lazily, at the next step's start)
                if (I.lazy_wte) {
                    adam_segment(ls, st, ws, L.wpe, L.layers[0].ln1_g);
                    I.wte_pending = true;
                    I.wte_step = I.step_no;
                } else {
                    adam_segment(ls, st, ws, 0, L.layers[0].ln1_g);
                }
            }
            break;
        }
        case TaskKind::Transfer: {
            // Copy-engine peer copy straight into the receiver's slot, then a flag write carrying
            // the step sequence number; the receiver's stream waits for the flag (stream memory
            // operations: no SM is held while waiting).
            const bool fwd = graph_.tasks[static_cast<size_t>(t.deps[0])].kind == TaskKind::Fwd;
            const size_t bytes = static_cast<size_t>(T * h) * sizeof(bf16);
            const i64 dst_stage = fwd ? t.stage + 1 : t.stage - 1;
            const size_t sl = static_cast<size_t>((t.micro_batch * v_ + dst_stage / p_) * 2 + (fwd ? 0 : 1));
            if (I.debug)
                fprintf(stderr, "[bfpp rank %d] step %d task %d %s %s mb %lld s %lld\n", rank_, I.step_no, te.id,
                        te.send ? "send" : "recv", fwd ? "fwd" : "bwd", (long long)t.micro_batch, (long long)t.stage);
            if (te.send) {
                const StageActs& a = I.acts[static_cast<size_t>(t.micro_batch)][static_cast<size_t>(t.stage / p_)];
                const int peer = static_cast<int>(dp_rank_ * p_ + t.peer_device);
                bf16* dst = I.peer_arena.at(peer) + sl * static_cast<size_t>(T * h);
                CK(cudaMemcpyAsync(dst, fwd ? a.out : a.gout, bytes, cudaMemcpyDeviceToDevice, st));
                if (memops().write(st, reinterpret_cast<CUdeviceptr>(I.peer_flags.at(peer) + sl), I.xfer_seq,
                                   CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
                    throw std::runtime_error("executor: cuStreamWriteValue32 failed");
            } else {
                if (memops().wait(st, reinterpret_cast<CUdeviceptr>(I.recv_flags + sl), I.xfer_seq,
                                  CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                    throw std::runtime_error("executor: cuStreamWaitValue32 failed");
            }
            break;
        }
        case TaskKind::Reconstruct: {
            LocalStage& ls = I.local[static_cast<size_t>(t.stage / p_)];
            for (size_t si = 0; si + 1 < ls.seg.size(); ++si) {
                all_gather_segments(ls, I.slots[te.slot], si, si + 1, I.dp_comm, st);
                CK(cudaEventRecord(I.rec_ev[te.slot][si], st));
            }
            break;
        }
        case TaskKind::Reduce: {
            LocalStage& ls = I.local[static_cast<size_t>(t.stage / p_)];
            const int64_t full = layouts_[static_cast<size_t>(t.stage)].padded;
            if (c_.dp_variant == DpVariant::DP0) {
                NK(ncclAllReduce(ls.grad, ls.grad, static_cast<size_t>(full), ncclFloat32, ncclSum, I.dp_comm, st));
            } else if (std::find(ls.seg_done.begin(), ls.seg_done.end(), 1) != ls.seg_done.end()) {
                // the backward already reduced and updated some segments: finish the others
                for (size_t si = 0; si + 1 < ls.seg.size(); ++si)
                    if (!ls.seg_done[si]) reduce_segment(ls, st, si, te.first_unit, te.adam_after);
                std::fill(ls.seg_done.begin(), ls.seg_done.end(), 0);
                break;
            } else if (!ls.gshard) {  // single unit, transient shard buffer (segments, or the whole stage)
                for (size_t si = 0; si + 1 < ls.seg.size(); ++si)
                    reduce_segment(ls, st, si, true, te.adam_after);
                std::fill(ls.seg_done.begin(), ls.seg_done.end(), 0);
                break;
            } else {
                float* dst = te.first_unit ? ls.gshard : I.gtmp;
                reduce_scatter_segments(ls, dst, 0, ls.seg.size() - 1, I.dp_comm, st);
                if (!te.first_unit)
                    K(K_MISC, 12.0 * ls.shard_n, 1, st, [&] { add_f32_kernel<<<296, 256, 0, st>>>(ls.gshard, I.gtmp, ls.shard_n); });
                // no re-zeroing: the next unit's first backward overwrites the gradient buffer
            }
            if (te.adam_after) adam(ls, st);
            break;
        }
        }
        if (o_.record_timeline) CK(cudaEventRecord(I.t_end[static_cast<size_t>(te.id)], st));
        CK(cudaEventRecord(I.done[static_cast<size_t>(te.id)], st));
    }
    // loss of this replica (last-stage device): mean over its n_mb * T tokens
    if (has_last)
        K(K_MISC, 4.0 * c_.n_mb * T, 1, cs,
          [&] { sum_f32(I.row_loss, c_.n_mb * T, 1.f / static_cast<float>(c_.n_mb * T), I.loss_dev, 0, cs); });
    for (int s = 1; s < S_N; ++s) {
        CK(cudaEventRecord(I.stream_end[s], I.st[s]));
        CK(cudaStreamWaitEvent(cs, I.stream_end[s], 0));
    }
    CK(cudaEventRecord(I.step_end, cs));
    CK(cudaEventRecord(I.step_done[I.step_no & 1], cs));
    if (loss_dev && has_last) CK(cudaMemcpyAsync(loss_dev, I.loss_dev, 4, cudaMemcpyDeviceToDevice, cs));
    if (loss_host) {
        if (has_last) {
            CK(cudaMemcpyAsync(I.loss_pinned, I.loss_dev, 4, cudaMemcpyDeviceToHost, cs));
            if (I.debug) fprintf(stderr, "[bfpp rank %d] step %d loss sync\n", rank_, I.step_no);
            CK(cudaStreamSynchronize(cs));
            *loss_host = *I.loss_pinned;
        } else {
            *loss_host = NAN;
        }
    }
    CK(cudaPeekAtLastError());
    if (I.debug) fprintf(stderr, "[bfpp rank %d] step %d enqueued\n", rank_, I.step_no);
    if (o_.profile_kernels) {
        wait_step_event(I.step_end, I.step_no);
        for (const auto& mk : I.marks) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, I.ev_pool[mk.ev], I.ev_pool[mk.ev + 1]));
            I.stats.ms[mk.cat] += ms;
            I.stats.work[mk.cat] += mk.work;
        }
    }
    if (o_.record_timeline) {
        wait_step_event(I.step_end, I.step_no);
        for (const TaskExec& te : I.order) {
            float a = 0, b = 0;
            CK(cudaEventElapsedTime(&a, I.origin, I.t_start[static_cast<size_t>(te.id)]));
            CK(cudaEventElapsedTime(&b, I.origin, I.t_end[static_cast<size_t>(te.id)]));
            const Task& t = graph_.tasks[static_cast<size_t>(te.id)];
            // a transfer is reported by its sender; the receiver keeps its own view only if it is the sender
            if (t.kind == TaskKind::Transfer && !te.send) continue;
            I.tl_start[static_cast<size_t>(te.id)] = a * 1e-3;
            I.tl_end[static_cast<size_t>(te.id)] = b * 1e-3;
        }
    }
}

// Host wait for a step's completion event. With the watchdog on (debug mode, or
// BFPP_EXEC_WATCHDOG=1) the event is polled and, after 20 s without progress, the first
// unfinished tasks and the state of every stream are reported once (then the wait continues).
void Executor::wait_step_event(cudaEvent_t ev, int step) {
    Impl& I = *impl_;
    if (!I.debug && !I.watchdog) {
        CK(cudaEventSynchronize(ev));
        return;
    }
    auto t0 = std::chrono::steady_clock::now();
    bool reported = false;
    cudaError_t q;
    while ((q = cudaEventQuery(ev)) == cudaErrorNotReady) {
        if (!reported && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20)) {
            fprintf(stderr, "[bfpp rank %d] STALL waiting for step %d; unfinished tasks:\n", rank_, step);
            int shown = 0;
            for (const TaskExec& te : I.order) {
                if (cudaEventQuery(I.done[static_cast<size_t>(te.id)]) == cudaErrorNotReady && shown < 12) {
                    const Task& tt = graph_.tasks[static_cast<size_t>(te.id)];
                    fprintf(stderr, "  task %d kind %s mb %lld stage %lld stream %d\n", te.id, kind_name(tt.kind),
                            (long long)tt.micro_batch, (long long)tt.stage, te.stream);
                    ++shown;
                }
            }
            for (int s = 0; s < S_N; ++s)
                fprintf(stderr, "  stream %d query %d\n", s, static_cast<int>(cudaStreamQuery(I.st[s])));
            fflush(stderr);
            reported = true;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
    CK(q);
}

const KernelStats& Executor::kernel_stats() const { return impl_->stats; }

void Executor::set_flags(bool record_timeline, bool profile_kernels) {
    Impl& I = *impl_;
    CK(cudaSetDevice(I.dev));
    o_.record_timeline = record_timeline;
    o_.profile_kernels = profile_kernels;
    if (record_timeline)
        for (const TaskExec& te : I.order) {
            const size_t id = static_cast<size_t>(te.id);
            if (!I.t_start[id]) CK(cudaEventCreate(&I.t_start[id]));
            if (!I.t_end[id]) CK(cudaEventCreate(&I.t_end[id]));
        }
}
cudaStream_t Executor::compute_stream() const { return impl_->st[S_COMPUTE]; }

void Executor::sync() {
    CK(cudaSetDevice(impl_->dev));
    CK(cudaStreamSynchronize(impl_->st[S_COMPUTE]));
    ncclResult_t async_err = ncclSuccess;
    for (ncclComm_t cm : {impl_->world_comm, impl_->dp_comm})
        if (cm && ncclCommGetAsyncError(cm, &async_err) == ncclSuccess && async_err != ncclSuccess)
            throw std::runtime_error(std::string("NCCL async error: ") + ncclGetErrorString(async_err));
}

void Executor::timeline(double* start, double* end) const {
    for (size_t i = 0; i < impl_->tl_start.size(); ++i) {
        start[i] = impl_->tl_start[i];
        end[i] = impl_->tl_end[i];
    }
}

namespace {
// this rank's slices of a device shard -> host[0, numel) (NaN where another rank owns the element)
void scatter_shard(const LocalStage& ls, const StageLayout& L, const float* dev, float* host, int64_t* lo,
                   int64_t* hi) {
    std::vector<float> sh(static_cast<size_t>(ls.shard_n));
    CK(cudaMemcpy(sh.data(), dev, static_cast<size_t>(ls.shard_n) * 4, cudaMemcpyDeviceToHost));
    std::fill(host, host + L.numel, std::numeric_limits<float>::quiet_NaN());
    for_each_chunk(ls, [&](int64_t off, int64_t len, int64_t soff) {
        const int64_t m = std::max<int64_t>(0, std::min(len, L.numel - off));
        if (m > 0) std::memcpy(host + off, sh.data() + soff, static_cast<size_t>(m) * 4);
    });
    *lo = 0;
    *hi = L.numel;
}

LocalStage& find_local(std::vector<LocalStage>& v, i64 stage) {
    for (auto& ls : v)
        if (ls.stage == stage) return ls;
    throw SpecError("executor: stage is not hosted by this rank");
}
}  // namespace

void Executor::set_params(i64 stage, const float* host, int64_t n) {
    // All copies are stream-ordered on the compute stream: a synchronous cudaMemcpy from
    // pageable memory may return before its DMA lands, and the executor's streams do not
    // synchronise with the legacy default stream.
    Impl& I = *impl_;
    CK(cudaSetDevice(I.dev));
    sync();
    I.wte_pending = I.wte_armed = I.wte_rest = false;  // the optimizer restarts: no deferred update carries over
    cudaStream_t cs = I.st[S_COMPUTE];
    LocalStage& ls = find_local(I.local, stage);
    const StageLayout& L = layouts_[static_cast<size_t>(stage)];
    if (n != L.numel) throw SpecError("set_params: size mismatch with the stage layout");
    std::vector<float> padded(static_cast<size_t>(L.padded), 0.f);
    std::memcpy(padded.data(), host, static_cast<size_t>(n) * 4);
    std::vector<float> shard(static_cast<size_t>(ls.shard_n));
    for_each_chunk(ls, [&](int64_t off, int64_t len, int64_t soff) {
        std::memcpy(shard.data() + soff, padded.data() + off, static_cast<size_t>(len) * 4);
    });
    CK(cudaMemcpyAsync(ls.master, shard.data(), static_cast<size_t>(ls.shard_n) * 4, cudaMemcpyHostToDevice, cs));
    CK(cudaMemsetAsync(ls.m, 0, static_cast<size_t>(ls.shard_n) * 4, cs));
    CK(cudaMemsetAsync(ls.v, 0, static_cast<size_t>(ls.shard_n) * 4, cs));
    if (ls.w16_shard) f32_to_bf16(ls.master, ls.w16_shard, ls.shard_n, cs);
    float* tmp = nullptr;
    if (ls.w16) {
        if (ls.shard_n == L.padded) {
            f32_to_bf16(ls.master, ls.w16, L.padded, cs);
        } else {  // replicated weights with a sharded optimizer (DP_PS): convert the full vector
            CK(cudaMalloc(&tmp, static_cast<size_t>(L.padded) * 4));
            CK(cudaMemcpyAsync(tmp, padded.data(), static_cast<size_t>(L.padded) * 4, cudaMemcpyHostToDevice, cs));
            f32_to_bf16(tmp, ls.w16, L.padded, cs);
        }
    }
    CK(cudaStreamSynchronize(cs));
    if (tmp) CK(cudaFree(tmp));
    I.step_no = 0;
}

// Completes a pending lazy token-table update (all rows, the pending step's bias corrections) so
// the parameters read back are those after the last step.
void Executor::flush_lazy_updates() {
    Impl& I = *impl_;
    if (!I.wte_pending) return;
    CK(cudaSetDevice(I.dev));
    for (LocalStage& ls : I.local) {
        const StageLayout& L = layouts_[static_cast<size_t>(ls.stage)];
        if (!L.first) continue;
        const int64_t base = L.wte, n = L.wpe - L.wte;
        adam_update(ls.master + base, ls.m + base, ls.v + base, ls.grad + base, ls.w16 + base, n, o_.lr, o_.beta1,
                    o_.beta2, o_.eps, o_.weight_decay, I.wte_step, 0, I.st[S_COMPUTE]);
    }
    I.wte_pending = false;
    CK(cudaStreamSynchronize(I.st[S_COMPUTE]));
}

void Executor::get_params(i64 stage, float* host, int64_t n, int64_t* lo, int64_t* hi) {
    Impl& I = *impl_;
    sync();
    flush_lazy_updates();
    CK(cudaDeviceSynchronize());
    LocalStage& ls = find_local(I.local, stage);
    const StageLayout& L = layouts_[static_cast<size_t>(stage)];
    if (n < L.numel) throw SpecError("get_params: buffer too small");
    scatter_shard(ls, L, ls.master, host, lo, hi);
}

void Executor::get_grads(i64 stage, float* host, int64_t n, int64_t* lo, int64_t* hi) {
    Impl& I = *impl_;
    sync();
    CK(cudaDeviceSynchronize());
    LocalStage& ls = find_local(I.local, stage);
    const StageLayout& L = layouts_[static_cast<size_t>(stage)];
    if (n < L.numel) throw SpecError("get_grads: buffer too small");
    if (ls.w16_shard && !ls.gshard)
        throw SpecError("get_grads: this stage's reduced gradients are transient (one reduction unit); "
                        "create the executor with skip_optimizer to keep them");
    if (ls.gshard) {
        scatter_shard(ls, L, ls.gshard, host, lo, hi);
    } else {
        CK(cudaMemcpy(host, ls.grad, static_cast<size_t>(L.numel) * 4, cudaMemcpyDeviceToHost));
        *lo = 0;
        *hi = L.numel;
    }
}

void Executor::get_weights16(i64 stage, uint16_t* host, int64_t n, int64_t* lo, int64_t* hi) {
    Impl& I = *impl_;
    sync();
    flush_lazy_updates();
    CK(cudaDeviceSynchronize());
    LocalStage& ls = find_local(I.local, stage);
    const StageLayout& L = layouts_[static_cast<size_t>(stage)];
    if (n < L.numel) throw SpecError("get_weights16: buffer too small");
    if (ls.w16) {
        CK(cudaMemcpy(host, ls.w16, static_cast<size_t>(L.numel) * 2, cudaMemcpyDeviceToHost));
        *lo = 0;
        *hi = L.numel;
    } else {
        std::vector<uint16_t> sh(static_cast<size_t>(ls.shard_n));
        CK(cudaMemcpy(sh.data(), ls.w16_shard, static_cast<size_t>(ls.shard_n) * 2, cudaMemcpyDeviceToHost));
        std::fill(host, host + L.numel, static_cast<uint16_t>(0x7FC0));  // bf16 NaN where not owned
        for_each_chunk(ls, [&](int64_t off, int64_t len, int64_t soff) {
            const int64_t m = std::max<int64_t>(0, std::min(len, L.numel - off));
            if (m > 0) std::memcpy(host + off, sh.data() + soff, static_cast<size_t>(m) * 2);
        });
        *lo = 0;
        *hi = L.numel;
    }
}

void Executor::zero_grads() {
    Impl& I = *impl_;
    sync();
    if (I.gbuf) CK(cudaMemset(I.gbuf, 0, static_cast<size_t>(I.gbuf_n) * 4));
    for (auto& ls : I.local) {
        if (!I.gbuf) CK(cudaMemset(ls.grad, 0, static_cast<size_t>(layouts_[static_cast<size_t>(ls.stage)].padded) * 4));
        if (ls.gshard) CK(cudaMemset(ls.gshard, 0, static_cast<size_t>(ls.shard_n) * 4));
    }
    CK(cudaDeviceSynchronize());
}

}  // namespace bfpp
