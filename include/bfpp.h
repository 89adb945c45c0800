/*
 * bfpp.h — C ABI of the B200-native breadth-first pipeline executor.
 *
 * Schedule section: drop-in replacement for the reference's schedule/stage API
 * (pipesim; C++ signatures in proj/include/pipesim/schedule.hpp and
 * simulate.hpp). Exceptions cannot cross a C ABI, so every function returns a
 * status code (BFPP_OK, BFPP_SPEC_ERROR = the CLI's exit code 2 for SpecError,
 * BFPP_EXEC_ERROR = exit code 4 for SimError / execution failures;
 * reference tools/pipesim.cpp:214-226) and the message is available from
 * bfpp_last_error() (thread-local).
 *
 * Enum integer values are the reference's declaration order (wire format):
 *   DpVariant  DP0=0 DP_PS=1 DP_FS=2                       (types.hpp:14)
 *   Schedule   NoPipeline=0 GPipe=1 OneFOneB=2 DepthFirst=3 BreadthFirst=4 (types.hpp:15)
 *   Lane       Compute=0 DpNet=1 PpNet=2                   (schedule.hpp:41)
 *   TaskKind   Fwd=0 Bwd=1 Reduce=2 Reconstruct=3 Transfer=4 (schedule.hpp:42)
 */
#ifndef BFPP_H
#define BFPP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFPP_OK 0
#define BFPP_SPEC_ERROR 2
#define BFPP_EXEC_ERROR 4

/* ---- value types (POD mirrors of the reference structs) ------------------ */

/* mirrors pipesim::ModelSpec (types.hpp:29-43) */
typedef struct bfpp_model_spec {
    int64_t n_layers, s_hidden, n_heads, s_head, s_mlp, s_seq, s_voc;
} bfpp_model_spec;

/* mirrors pipesim::ParallelConfig (types.hpp:64-84) */
typedef struct bfpp_parallel_config {
    int64_t n_dp, n_tp, n_pp, n_mb, s_mb, n_loop;
    int32_t dp_variant, schedule;
} bfpp_parallel_config;

/* mirrors pipesim::ClusterSpec (types.hpp:47-59) */
typedef struct bfpp_cluster_spec {
    int64_t n_node, s_node;
    double peak_flops, bw_intra, bw_inter, pp_latency, mem_capacity, kernel_efficiency;
} bfpp_cluster_spec;

/* mirrors pipesim::TimingModel (schedule.hpp:24-39) */
typedef struct bfpp_timing_model {
    double t_fwd_stage, bwd_ratio, t_pp_transfer, pp_latency, t_dp_reduce_stage, t_dp_reconstruct_stage;
} bfpp_timing_model;

/* mirrors pipesim::Task (schedule.hpp:46-56) without deps (CSR accessors) */
typedef struct bfpp_task {
    int32_t id, lane, kind, priority;
    int64_t device, peer_device, micro_batch, stage;
} bfpp_task;

typedef struct bfpp_graph bfpp_graph;       /* pipesim::TaskGraph */
typedef struct bfpp_timeline bfpp_timeline; /* pipesim::Timeline  */
typedef struct bfpp_exec bfpp_exec;         /* per-rank executor   */

const char* bfpp_last_error(void);

/* ---- schedule API ---------------------------------------------------------- */

/* replaces ParallelConfig::validate(model[, cluster]) (types.cpp:92-130); cluster may be NULL */
int bfpp_validate(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_cluster_spec* cl);

/* replaces total_memory (memory.hpp / memory.cpp:72-80): out[4] = state, activation, checkpoint,
 * total bytes per device of the reference's analytic model (MemoryOptions::dp0_bytes_per_param) */
int bfpp_total_memory(const bfpp_model_spec* m, const bfpp_parallel_config* c, double dp0_bytes_per_param,
                      double* out);
/* replaces feasible (memory.cpp:82-86): *out = total <= headroom * cl->mem_capacity */
int bfpp_feasible(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_cluster_spec* cl,
                  double dp0_bytes_per_param, double headroom, int32_t* out);
/* replaces cluster_preset (types.cpp:206-231): "a100", "v100-dgx1", and "b200" (new) */
int bfpp_cluster_preset(const char* name, bfpp_cluster_spec* out);

/* Configuration search (replaces enumerate_configs + rank_configs, search.cpp:62-188; n_tp = 1).
 * Measured per-kind task costs in units that carry across configurations (see rates_from_timing). */
typedef struct bfpp_measured_rates {
    double fwd_layer_seq;           /* forward seconds per layer per sequence (s_mb = 1) */
    double bwd_ratio;               /* backward / forward */
    double pp_s_per_byte, pp_latency;
    double reduce_s_per_param;      /* DP reduction seconds per stage parameter */
    double reconstruct_s_per_param; /* DP_FS reconstruction seconds per stage parameter */
} bfpp_measured_rates;
typedef struct bfpp_ranked_config {
    bfpp_parallel_config config;
    double score;        /* flop/s per GPU: Eq. 11 over the simulated makespan (perf.cpp:8-20) */
    double memory_bytes; /* total_memory (memory.cpp:72-80) */
    double bubble;       /* bubble_fraction of the simulated timeline */
    bfpp_timing_model timing;
} bfpp_ranked_config;
/* rates of a (measured) timing model at configuration c: divides out c's stage size, micro-batch
 * size and message sizes */
int bfpp_rates_from_timing(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_timing_model* t,
                           bfpp_measured_rates* out);
/* Enumerates the space (choice arrays; the reference's sharding policy and grid rules), keeps the
 * feasible configs (total_memory <= headroom * mem_capacity), simulates each with
 * TimingModel::derive (scoring 0, the reference's "simulate" mode) or with the measured rates
 * (scoring 1), and returns them best first (ties: lower memory, less model parallelism).
 * Two-phase sizing: cap = 0 returns the count in *n_out. */
int bfpp_rank_configs(const bfpp_model_spec* m, const bfpp_cluster_spec* k, const int32_t* schedules, int64_t n_sched,
                      const int32_t* dp_variants, int64_t n_var, const int64_t* n_pp, int64_t n_n_pp,
                      const int64_t* s_mb, int64_t n_s_mb, const int64_t* n_mb, int64_t n_n_mb,
                      const int64_t* n_loop, int64_t n_n_loop, const int64_t* batch_sizes, int64_t n_batch,
                      int32_t scoring, const bfpp_measured_rates* rates, double dp0_bytes_per_param, double headroom,
                      int32_t threads, int64_t cap, bfpp_ranked_config* out, int64_t* n_out);

/* replaces place_stages (schedule.hpp:20, schedule.cpp:23-33). assignment_out
 * receives n_stage entries (cap must be >= n_pp*n_loop). */
int bfpp_place_stages(const bfpp_model_spec* m, const bfpp_parallel_config* c, int64_t* assignment_out,
                      int64_t cap, int64_t* n_stage, int64_t* layers_per_stage);

/* replaces build_tasks (schedule.hpp:73-74, schedule.cpp:422-452); the
 * placement is recomputed from (m, c) exactly as place_stages does. */
int bfpp_build_tasks(const bfpp_model_spec* m, const bfpp_parallel_config* c, bfpp_graph** out);

/* replaces build_accumulation_tasks (schedule.hpp:80-81, schedule.cpp:454-500); order 0 = DF, 1 = BF */
int bfpp_build_accumulation_tasks(const bfpp_model_spec* m, int32_t dp_variant, int32_t order, int64_t n_mb,
                                  bfpp_graph** out);

/* Builds a graph from raw arrays (deadlock / malformed-program tests; ref test_schedule.cpp:393-406). */
int bfpp_graph_from_arrays(int64_t n_devices, int64_t n_tasks, const bfpp_task* tasks, const int32_t* dep_offsets,
                           const int32_t* dep_ids, const int32_t* prog_offsets, const int32_t* prog_ids,
                           bfpp_graph** out);

int64_t bfpp_graph_n_devices(const bfpp_graph* g);
int64_t bfpp_graph_n_tasks(const bfpp_graph* g);
int64_t bfpp_graph_n_deps(const bfpp_graph* g);
int64_t bfpp_graph_n_program_steps(const bfpp_graph* g);
/* copy-out: tasks[n_tasks]; dep CSR (offsets[n_tasks+1], ids[n_deps]); program CSR (offsets[n_devices+1], ids[...]) */
int bfpp_graph_tasks(const bfpp_graph* g, bfpp_task* out, int64_t cap);
int bfpp_graph_deps(const bfpp_graph* g, int32_t* offsets, int32_t* ids);
int bfpp_graph_programs(const bfpp_graph* g, int32_t* offsets, int32_t* ids);
void bfpp_graph_destroy(bfpp_graph* g);

/* replaces simulate (simulate.hpp:28, simulate.cpp:41-158) */
int bfpp_simulate(const bfpp_graph* g, const bfpp_timing_model* t, bfpp_timeline** out);
/* the same list scheduler with one duration per task id (durations[n_tasks]): replays a measured
 * timeline's own task times with zero executor overhead (new; no reference counterpart) */
int bfpp_simulate_durations(const bfpp_graph* g, const double* durations, bfpp_timeline** out);
int64_t bfpp_timeline_n_events(const bfpp_timeline* tl);
int64_t bfpp_timeline_n_devices(const bfpp_timeline* tl);
double bfpp_timeline_makespan(const bfpp_timeline* tl);
/* start/end[n_events] (seconds), lane_busy[n_devices*3] */
int bfpp_timeline_events(const bfpp_timeline* tl, double* start, double* end, double* lane_busy);
/* Builds a timeline from measured per-task intervals (executor output, or tests). */
int bfpp_timeline_from_arrays(const bfpp_graph* g, const double* start, const double* end, bfpp_timeline** out);
void bfpp_timeline_destroy(bfpp_timeline* tl);

/* replaces bubble_fraction (simulate.cpp:160-164) */
double bfpp_bubble_fraction(const bfpp_timeline* tl);
/* replace chrome_trace_json (report.cpp:160-212; pybind module.cpp:375) and gantt_svg
 * (report.cpp:248-290; module.cpp:376) for any timeline, simulated or measured. Two-call text
 * pattern: *len = length without the terminator; up to cap-1 bytes + NUL written to buf (may be NULL). */
int bfpp_chrome_trace_json(const bfpp_timeline* tl, const bfpp_graph* g, char* buf, int64_t cap, int64_t* len);
int bfpp_gantt_svg(const bfpp_timeline* tl, const bfpp_graph* g, char* buf, int64_t cap, int64_t* len);
/* Per-kind mean durations of a measured timeline as a TimingModel (closes the loop of
 * TimingModel::derive, schedule.cpp:43-86: simulate the same graph with measured timings). */
int bfpp_measured_timing_model(const bfpp_graph* g, const bfpp_timeline* tl, bfpp_timing_model* out);
/* replaces peak_inflight (simulate.cpp:166-191); out[n_devices] */
int bfpp_peak_inflight(const bfpp_timeline* tl, const bfpp_graph* g, int64_t layers_per_stage, int64_t* out);
/* replaces compute_per_gpu (types.cpp:136-146; Eq. 11) */
double bfpp_compute_per_gpu(const bfpp_model_spec* m, const bfpp_parallel_config* c);

/* ---- device kernels (device pointers; stream is a cudaStream_t, NULL = default) --------
 * The reference has no kernels (stage compute is the scalar
 * TimingModel::t_fwd_stage, schedule.hpp:25-26); these are the stage executor's
 * building blocks, exported for parity tests and micro-benchmarks. */

/* epilogues of bfpp_gemm_bf16 */
#define BFPP_EPI_BF16 0  /* D = acc (bf16)                                   */
#define BFPP_EPI_GELU 1  /* aux_out = acc (bf16), D = gelu(aux_out) (bf16)   */
#define BFPP_EPI_RESID 2 /* D = acc + aux (bf16)                             */
#define BFPP_EPI_DGELU 3 /* D = acc * gelu'(aux) (bf16)                      */
#define BFPP_EPI_F32 4   /* D (+)= acc (f32, accumulate flag)                */

typedef struct bfpp_gemm_args {
    int64_t M, N, K;
    const void* A; int64_t lda; int32_t a_mn_major; /* 0: A[M][lda]; 1: A stored as [K][lda] */
    const void* B; int64_t ldb; int32_t b_mn_major; /* 0: B[N][ldb]; 1: B stored as [K][ldb] */
    void* D; int64_t ldd;
    const void* aux; int64_t ldaux;
    void* aux_out; int64_t ldaux_out;
    int32_t epilogue, accumulate;
} bfpp_gemm_args;

/* D[M,N] = sum_k A[m,k] B[n,k] on tcgen05 (TMA + TMEM), bf16 in, f32 accumulate */
int bfpp_gemm_bf16(const bfpp_gemm_args* args, void* stream);
/* Two independent GEMMs in one launch (one persistent tile space: the pair fills the SMs' waves
 * together and pays one prologue); same operand majors and M, N >= 256 required for the grouped
 * kernel, otherwise (or with BFPP_GEMM_PAIR=0) two ordinary launches. Results equal bfpp_gemm_bf16. */
int bfpp_gemm_bf16_pair(const bfpp_gemm_args* a, const bfpp_gemm_args* b, void* stream);
/* GEMM variant selection for benchmarks and tests (process-wide): mode -1 auto, 1 one-CTA
 * 128-row tiles, 2 two-CTA 256-row tiles; bn2 = pair-tile width (0 default = 256, 128 opt-in);
 * stream_k = 0 off (default), 1 forced, -1 auto (only when the last tile wave leaves pairs idle).
 * Defaults come from BFPP_GEMM_MODE / BFPP_GEMM_BN2 / BFPP_GEMM_SK. */
int bfpp_gemm_config(int32_t mode, int32_t bn2, int32_t stream_k);
/* tile schedule of the persistent 2-CTA GEMM: 0 static (tile t, t + pairs, ...; default), 1 dynamic
 * (a pair's later tiles come from a per-stream device counter, so a pair that starts late or runs
 * slow takes fewer tiles; CUDA-graph captures always use the static schedule). BFPP_GEMM_DYN. */
int bfpp_gemm_schedule(int32_t dynamic);
/* attention forward: query tiles per CTA (0 auto, 1, 2 = two tiles sharing K/V, ping-pong softmax) */
int bfpp_attention_config(int32_t fwd_tiles);
/* persistent GEMM grids use at most n SMs (0 = all): for streams confined to an SM partition */
int bfpp_gemm_sm_limit(int32_t n);
/* Process-wide launch counters per kernel variant (0 1-CTA GEMM, 1 2-CTA GEMM, 2 grouped 2-CTA
 * pair, 3 N-fastest raster, 4 stream-K, 5 attention fwd with > 1 head and > 1 query block,
 * 6 attention bwd with > 1 head and > 1 key block); -1 for an unknown variant. Host-side, no GPU
 * access: used by the parity tests to show which production kernels a composed step ran. */
int64_t bfpp_kernel_variant_count(int32_t variant);
void bfpp_kernel_variant_reset(void);

/* causal multi-head attention, head_dim 128 (flash-style; never materialises T x T).
 * qkv [B*S][3*H*128] bf16 (Q | K | V column blocks), o [B*S][H*128] bf16,
 * lse [B*H][S] f32 (log2-sum-exp of scaled scores). Backward scratch: delta [B*H][S],
 * dq_acc [B*S][H*128] f32; dqkv has qkv's layout. */
int bfpp_attention_fwd(const void* qkv, void* o, float* lse, int32_t batch, int32_t seq, int32_t heads,
                       int32_t head_dim, void* stream);
int bfpp_attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse, float* delta,
                       float* dq_acc, void* dqkv, int32_t batch, int32_t seq, int32_t heads, int32_t head_dim,
                       void* stream);

/* LayerNorm over rows of `width` (bf16 x/y/gamma/beta, f32 mean/rstd). The backward
 * adds dres (may be NULL) to dx and ACCUMULATES dgamma/dbeta. */
int bfpp_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd,
                       int32_t rows, int32_t width, float eps, void* stream);
int bfpp_layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                       const void* dres, void* dx, float* dgamma, float* dbeta, int32_t rows, int32_t width,
                       void* stream);

/* x[t] = wte[tok[t]] + wpe[t mod S] (bf16); backward scatter-adds into f32 dwte/dwpe */
int bfpp_embed_fwd(const int32_t* tok, const void* wte, const void* wpe, void* x, int32_t T, int32_t S, int32_t h,
                   void* stream);
int bfpp_embed_bwd(const int32_t* tok, const void* dx, float* dwte, float* dwpe, int32_t T, int32_t S, int32_t h,
                   void* stream);

/* row_loss[t] = logsumexp(logits[t]) - logits[t][label[t]];
 * logits[t] <- (softmax(logits[t]) - onehot(label[t])) * grad_scale   (in place, bf16) */
int bfpp_softmax_xent(void* logits, int64_t ld, const int32_t* labels, float* row_loss, int32_t T, int32_t V,
                      float grad_scale, void* stream);

/* Adam (bias-corrected, decoupled weight decay) on f32 p/m/v with gradient g;
 * writes the bf16 copy w16; zeroes g if zero_grad. */
int bfpp_adam_update(float* p, float* m, float* v, float* g, void* w16, int64_t n, float lr, float beta1,
                     float beta2, float eps, float weight_decay, int32_t step, int32_t zero_grad, void* stream);

/* ---- executor: the reference's simulate() replaced by real execution --------------------
 * One process per GPU, rank = dp * n_pp + pp (reference placement convention,
 * types.hpp:110-113 with n_tp = 1). The executor builds the same TaskGraph as
 * bfpp_build_tasks and runs this rank's slice: Compute lane -> compute stream in
 * program order; DpNet lane -> DP stream in priority order (NCCL all-gather for
 * Reconstruct, reduce-scatter / all-reduce + sharded Adam for Reduce); PpNet ->
 * copy-engine peer copies into the receiver's CUDA-IPC-mapped slots, signalled with stream
 * memory operations (no NCCL on the pipeline path).
 * The model is a pre-LN GPT (bias-free linears, GeLU MLP, untied embeddings; the
 * embedding is folded into stage 0 and final LN + LM head + loss into the last
 * stage). */

#define BFPP_NCCL_UID_BYTES 128
#define BFPP_EXEC_SKIP_OPTIMIZER 1  /* flags: keep gradients, do not run Adam */
#define BFPP_EXEC_PROFILE_KERNELS 2 /* flags: CUDA events around every kernel -> bfpp_exec_kernel_stats */
#define BFPP_EXEC_RECOMPUTE 4       /* flags: activation checkpointing -- keep each layer's output only,
                                       recompute the layer (and LM-head logits) in the backward
                                       (checkpoint = 2 s h bytes, memory.cpp:64-70) */

typedef struct bfpp_exec_opts {
    int32_t device;          /* CUDA ordinal of this rank */
    int32_t record_timeline; /* 1: per-task CUDA events -> bfpp_exec_timeline */
    uint64_t seed;           /* Philox seed of the default N(0, init_std) initialisation */
    float lr, beta1, beta2, eps, weight_decay, init_std;
    int32_t flags;
} bfpp_exec_opts;

/* Fills 128 bytes with a fresh ncclUniqueId (generated on one rank, broadcast by the caller). */
int bfpp_nccl_unique_id(void* out);
/* Number of unique ids bfpp_exec_create expects: 1 + n_pp; id[0] = the world communicator (IPC
 * handle exchange, teardown barrier, timeline origin), id[1 + d] = DP group of pipeline rank d. */
int64_t bfpp_exec_n_comm_ids(const bfpp_parallel_config* c);
int bfpp_exec_create(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_exec_opts* o,
                     int32_t rank, int32_t world, const void* uids, bfpp_exec** out);
/* Same, running the given task graph instead of build_tasks(m, c) -- e.g. the gradient-accumulation
 * graphs of bfpp_build_accumulation_tasks (schedule.cpp:454-500, PAPER Appendix C), executed with
 * c = {n_pp 1, n_loop n_layers, n_mb, n_dp = ranks, dp_variant}. Validated against c (status 2). */
int bfpp_exec_create_graph(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_graph* g,
                           const bfpp_exec_opts* o, int32_t rank, int32_t world, const void* uids,
                           bfpp_exec** out);
/* Device bytes one rank of (m, c, o->flags) allocates, by category (bytes[8]: 0 bf16 compute
 * weights / DP_FS reconstruction slots, 1 f32 gradient buffers, 2 f32 master + Adam moments,
 * 3 reduced-gradient shards and reduce-scatter buffers, 4 bf16 all-gather source shards,
 * 5 activation sets (full, or checkpoints with BFPP_EXEC_RECOMPUTE), 6 pipeline receive arena and
 * send buffers, 7 scratch) and sets[2] = {pooled activation sets (= peak live (micro-batch, stage)
 * pairs in program order, simulate.cpp:166-191's peak_inflight in stages), pooled logits sets}.
 * Sizing only: no GPU is needed (the executor's allocation code run without allocating); the
 * figure to hold against the reference's total_memory / feasible (memory.cpp:72-86). */
int bfpp_exec_memory_plan(const bfpp_model_spec* m, const bfpp_parallel_config* c, const bfpp_exec_opts* o,
                          int32_t rank, int64_t* bytes, int64_t* sets);
/* the same breakdown of a live executor (its allocations) */
int bfpp_exec_memory(const bfpp_exec* e, int64_t* bytes, int64_t* sets);
/* One training step (forward, backward, gradient reduction, Adam) over this replica's
 * tokens [n_mb][s_mb][s_seq+1] int32 (inputs = [..., :-1], labels = [..., 1:]).
 * bfpp_exec_step takes HOST tokens and returns the replica's mean token loss on the
 * last-stage rank (NaN elsewhere); bfpp_exec_step_device takes DEVICE tokens, writes
 * the loss to a device float (may be NULL) and does not synchronise. */
int bfpp_exec_step(bfpp_exec* e, const int32_t* tokens_host, float* loss);
int bfpp_exec_step_device(bfpp_exec* e, const int32_t* tokens_dev, float* loss_dev);
int bfpp_exec_sync(bfpp_exec* e);
void bfpp_exec_destroy(bfpp_exec* e);
/* a copy of the executor's task graph (identical to bfpp_build_tasks) */
int bfpp_exec_graph(const bfpp_exec* e, bfpp_graph** out);
int64_t bfpp_exec_n_local_stages(const bfpp_exec* e);
int64_t bfpp_exec_local_stage(const bfpp_exec* e, int64_t c);
int64_t bfpp_exec_stage_numel(const bfpp_exec* e, int64_t stage);
int64_t bfpp_exec_device_bytes(const bfpp_exec* e);
/* Parameter I/O in the stage's flat layout. set_params takes the full stage
 * vector on every DP rank; get_params / get_grads write the f32 master weights / reduced
 * gradients this rank holds into a full-size buffer, NaN where another DP rank owns the element
 * (sharded variants own a 1/n_dp slice of every layer segment); [lo, hi) = [0, numel). */
int bfpp_exec_set_params(bfpp_exec* e, int64_t stage, const float* host, int64_t n);
int bfpp_exec_get_params(bfpp_exec* e, int64_t stage, float* host, int64_t n, int64_t* lo, int64_t* hi);
int bfpp_exec_get_grads(bfpp_exec* e, int64_t stage, float* host, int64_t n, int64_t* lo, int64_t* hi);
int bfpp_exec_zero_grads(bfpp_exec* e);
/* bf16 compute weights (resident copy, or this rank's all-gather source slices under DP_FS;
 * bf16 NaN 0x7FC0 where another rank owns the element) */
int bfpp_exec_get_weights16(bfpp_exec* e, int64_t stage, uint16_t* host, int64_t n, int64_t* lo, int64_t* hi);
/* measured [start, end] (seconds from the step origin) of this rank's tasks in the last
 * step; tasks of other devices are NaN. Arrays have bfpp_graph_n_tasks entries. */
int bfpp_exec_timeline(const bfpp_exec* e, double* start, double* end);
/* The executor's per-rank plan (host only, no GPU needed): for pipeline rank pp_rank of a
 * build_tasks graph, the local tasks in host enqueue order with their stream
 * (0 compute, 1 DP, 2/3 forward send/receive, 4/5 backward send/receive), flags
 * (1 send, 2 first reduce unit, 4 last reduce unit, 8 optimizer after, 16 first gradient
 * contribution of its unit, 32 last optimizer update of the step, 64 backward completing its
 * stage's last reduction unit, 128 ... whose reduction is also the first unit), DP_FS weight slot and the
 * cross-stream waits (CSR). Two-phase sizing: call with cap = 0 to get *n_tasks and *n_waits,
 * then pass cap >= n_tasks (ids, streams, flags, slots: cap entries; wait_offsets: cap + 1) and
 * wait_cap >= n_waits (wait_ids); smaller capacities fail with status 2 and write nothing. */
int bfpp_plan_rank(const bfpp_graph* g, int64_t pp_rank, int64_t n_dp, int32_t dp_variant, int64_t cap,
                   int64_t wait_cap, int32_t* ids, int32_t* streams, int32_t* flags, int32_t* slots,
                   int32_t* wait_offsets, int32_t* wait_ids, int64_t* n_tasks, int64_t* n_waits);

/* toggles per-task timeline events and per-kernel profiling for subsequent steps */
int bfpp_exec_set_flags(bfpp_exec* e, int32_t record_timeline, int32_t profile_kernels);
/* the executor's compute stream (cudaStream_t); every step starts on it and ends on it with
 * all of the step's streams joined (events recorded on it after a step bracket the whole step) */
void* bfpp_exec_stream(const bfpp_exec* e);
/* kernel statistics of the last step for category cat (0 GEMM, 1 attention fwd,
 * 2 attention bwd, 3 LayerNorm, 4 misc (embedding, cross-entropy, reductions), 5 Adam):
 * launches (always), summed device ms and algorithmic work (flops for 0-2, bytes for 3-5;
 * both only with BFPP_EXEC_PROFILE_KERNELS). */
int bfpp_exec_kernel_stats(const bfpp_exec* e, int32_t cat, int64_t* launches, double* ms, double* work);

#ifdef __cplusplus
}
#endif
#endif /* BFPP_H */
