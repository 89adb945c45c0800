// Causal flash attention forward and backward on the 5th-gen tensor cores (sm_100a), head_dim
// 128. Forward below; the backward's warp roles are described above attn_bwd_tc_kernel.
//
// One CTA per (128-query block, head, sample). Warp roles (192 threads):
//   warp 0      TMA producer: Q once, then K and V tiles of 128 keys (2-stage rings)
//   warp 1      MMA issuer (one elected thread) + TMEM owner:
//                 S_j = Q K_j^T  -> TMEM (double-buffered, so S_{j+1} overlaps softmax_j)
//                 O  += P_j V_j  -> TMEM (A = P_j read from TMEM, where it overwrote S_j;
//                                   B = V MN-major)
//   warps 2..5  softmax: thread = query row (TMEM lane); the whole 128-key row of S is in
//               registers, so max / sum need no shuffles. Online softmax in the log2
//               domain with a lazily updated running max (O in TMEM is rescaled only when
//               the max grows by more than 2^8), P packed as bf16 pairs into the S_j columns
//               (the A operand of the PV MMA). The exps of tile j run while PV_{j-1} is on the
//               tensor pipe: only an O rescale waits for it.
// Layouts as attention.cu: qkv [B*S][3*H*128], o [B*S][H*128], lse [B*H][S] (log2 domain).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>
#include <stdexcept>

#include "gemm.hpp"
#include "kernels.hpp"
#include "sm100_ptx.cuh"

namespace bfpp {
namespace {

constexpr int D = 128, BQ = 128, BKV = 128;

// Per-iteration clock64 stamps of one CTA's warp roles (scripts/attn_trace.cu builds this file
// with BFPP_ATTN_TRACE); compiled out of the product library.
#ifdef BFPP_ATTN_TRACE
__device__ unsigned long long g_attn_trace[8][64][16];
#define ATRACE(role, it, ev)                                                                     \
    do {                                                                                         \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (it) < 64)                  \
            g_attn_trace[role][it][ev] = clock64();                                              \
    } while (0)
#else
#define ATRACE(role, it, ev) \
    do {                     \
    } while (0)
#endif
constexpr int kTile = 128 * 128 * 2;  // one [128 rows][128 dims] bf16 tile = 2 x [128][64] SW128 blocks
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.f;  // log2 units

struct FwdSmem {
    static constexpr int kQ = 0;
    static constexpr int kK = kQ + kTile;          // 2 stages
    static constexpr int kV = kK + 2 * kTile;      // 2 stages
    static constexpr int kBar = kV + 2 * kTile;
    static constexpr int kBytes = kBar + 256 + 1024;
};

// K-major SW128 operand inside a [2 blocks][128 rows][128 B] tile: k-step kk (16 elements).
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t tile, int kk) {
    return ptx::sdesc_sw128(tile + (kk >> 2) * (kTile / 2) + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 operand (V as B of P.V): 128 keys x 128 dims, k-step kk = 16 keys.
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t tile, int kk) {
    return ptx::sdesc_sw128(tile + kk * 16 * 128, kTile / 2, 1024);
}

__global__ void __launch_bounds__(192, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, __nv_bfloat16* __restrict__ o,
                       float* __restrict__ lse, int S, int H, float scale_log2) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + FwdSmem::kBar);
    uint64_t* q_full = bar + 0;
    uint64_t* k_full = bar + 1;   // [2]
    uint64_t* k_empty = bar + 3;  // [2]
    uint64_t* v_full = bar + 5;   // [2]
    uint64_t* v_empty = bar + 7;  // [2]
    uint64_t* s_full = bar + 9;   // [2]
    uint64_t* p_full = bar + 11;
    uint64_t* o_done = bar + 12;  // PV_j complete (O stable)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

    // grid (H, query blocks, B): x (heads) varies fastest, so the longest query blocks (most
    // key tiles under the causal mask) of every head are scheduled first
    const int n_qb = (S + BQ - 1) / BQ;
    const int qb = n_qb - 1 - blockIdx.y;
    const int head = blockIdx.x, b = blockIdx.z;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int HD = H * D;
    const int row0 = b * S;
    const int n_kv = min((qb + 1) * BQ, S);
    const int n_tiles = (n_kv + BKV - 1) / BKV;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tm_qkv);
        ptx::mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&k_full[i], 1);
            ptx::mbar_init(&k_empty[i], 1);
            ptx::mbar_init(&v_full[i], 1);
            ptx::mbar_init(&v_empty[i], 1);
            ptx::mbar_init(&s_full[i], 1);
        }
        ptx::mbar_init(p_full, 4);
        ptx::mbar_init(o_done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_o = tmem, t_s = tmem + 128;  // O: cols [0,128); S buffers: [128,256), [256,384)

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            const int qcol = head * D, kcol = HD + head * D, vcol = 2 * HD + head * D;
            ptx::mbar_expect_tx(q_full, kTile);
            for (int h2 = 0; h2 < 2; ++h2)
                ptx::tma_load_2d(sm + FwdSmem::kQ + h2 * (kTile / 2), &tm_qkv, q_full, qcol + 64 * h2, row0 + qb * BQ);
            for (int j = 0; j < n_tiles; ++j) {
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                ptx::mbar_wait(&k_empty[st], ph ^ 1);
                ptx::mbar_expect_tx(&k_full[st], kTile);
                for (int h2 = 0; h2 < 2; ++h2)
                    ptx::tma_load_2d(sm + FwdSmem::kK + st * kTile + h2 * (kTile / 2), &tm_qkv, &k_full[st],
                                     kcol + 64 * h2, row0 + j * BKV);
                ptx::mbar_wait(&v_empty[st], ph ^ 1);
                ptx::mbar_expect_tx(&v_full[st], kTile);
                for (int h2 = 0; h2 < 2; ++h2)
                    ptx::tma_load_2d(sm + FwdSmem::kV + st * kTile + h2 * (kTile / 2), &tm_qkv, &v_full[st],
                                     vcol + 64 * h2, row0 + j * BKV);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer =====
            constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, 128, 0, 0);   // Q K^T: both K-major
            constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(128, 128, 0, 1);  // P V: V is MN-major
            const uint32_t sq = ptx::smem_u32(sm + FwdSmem::kQ);
            ptx::mbar_wait(q_full, 0);
            // S_j reuses the columns of P_{j-2}: issued after p_full_{j-1} (so softmax is done with
            // them) and after PV_{j-2} (the tensor pipe runs this thread's MMAs in issue order)
            auto issue_s = [&](int j) {
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                ptx::mbar_wait(&k_full[st], ph);
                ptx::tc_fence_after();
                const uint32_t sk = ptx::smem_u32(sm + FwdSmem::kK + st * kTile);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    ptx::umma_f16(t_s + st * 128, kmajor_desc(sq, kk), kmajor_desc(sk, kk), idesc_s, kk != 0);
                ptx::umma_commit(&k_empty[st]);
                ptx::umma_commit(&s_full[st]);
            };
            issue_s(0);
            for (int j = 0; j < n_tiles; ++j) {
                if (j + 1 < n_tiles) issue_s(j + 1);
                const int st = j & 1;
                ptx::mbar_wait(p_full, j & 1);
                ptx::mbar_wait(&v_full[st], (j >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t sv = ptx::smem_u32(sm + FwdSmem::kV + st * kTile);
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk)  // P: 16 keys = 8 packed columns per K-step
                    ptx::umma_f16_ts(t_o, t_s + st * 128 + kk * 8, mnmajor_desc(sv, kk), idesc_pv, (j | kk) != 0);
                ptx::umma_commit(&v_empty[st]);
                ptx::umma_commit(o_done);
            }
        }
    } else {
        // ===== softmax warps: thread = query row =====
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;          // row within the tile (= TMEM lane)
        const int qrow = qb * BQ + r;          // query position within the sequence
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        float m_used = -INFINITY, l = 0.f;
        for (int j = 0; j < n_tiles; ++j) {
            const int st = j & 1;
            ptx::mbar_wait(&s_full[st], (j >> 1) & 1);
            ptx::tc_fence_after();
            float s[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t rr[32];
                ptx::tmem_ld_32x32b_x32(t_s + st * 128 + lane_off + c * 32, rr);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(rr[i]);
            }
            const int k0 = j * BKV;
            const bool diag = k0 + BKV - 1 > qb * BQ || k0 + BKV > S;
            // keys k0 + i with i < lim are visible to this query row (k <= q, k < S)
            const int lim = diag ? min(qrow + 1, S) - k0 : BKV;
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < 128; ++i) {
                const float v = i < lim ? s[i] * scale_log2 : -INFINITY;
                s[i] = v;
                mx = fmaxf(mx, v);
            }
            // The rescale decision is per row, but tcgen05.ld/st are warp-collective
            // (.sync.aligned): if any row of the warp needs it, the whole warp rescales (rows
            // that do not need it use alpha = 1), so the TMEM accesses never diverge.
            const bool mine = mx > m_used + kRescaleThreshold;
            const bool rescale = __any_sync(0xffffffffu, mine);
            float alpha = 1.f;
            if (rescale) {
                alpha = mine ? (m_used == -INFINITY ? 0.f : ptx::ex2_fast(m_used - mx)) : 1.f;
                if (mine) m_used = mx;
                l *= alpha;
            }
            float sum = 0.f;
            uint32_t pw[64];
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                const float p0 = ptx::ex2_fast(s[2 * i] - m_used);
                const float p1 = ptx::ex2_fast(s[2 * i + 1] - m_used);
                sum += p0 + p1;
                __nv_bfloat162 hb = __floats2bfloat162_rn(p0, p1);
                pw[i] = *reinterpret_cast<uint32_t*>(&hb);
            }
            l += sum;
            if (rescale && j > 0) {
                // O is stable once PV_{j-1} has completed (PV_j waits for this tile's p_full)
                ptx::mbar_wait(o_done, (j - 1) & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t rr[32];
                    ptx::tmem_ld_32x32b_x32(t_o + lane_off + c * 32, rr);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) rr[i] = __float_as_uint(__uint_as_float(rr[i]) * alpha);
                    ptx::tmem_st_32x32b_x32(t_o + lane_off + c * 32, rr);
                }
            }
            // P_j packed into the first 64 columns of S_j's buffer (all of S_j is in registers)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t w[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) w[i] = pw[c * 16 + i];
                ptx::tmem_st_32x32b_x16(t_s + st * 128 + lane_off + c * 16, w);
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(p_full);
        }
        // epilogue: O / l -> bf16 -> global; lse = m + log2(l). Passing s_full_{n-1} only proves
        // PV_{n-3} done, so wait for the phases of PV_{n-2} and PV_{n-1} in turn (a parity wait
        // must not skip a phase)
        if (n_tiles >= 2) ptx::mbar_wait(o_done, (n_tiles - 2) & 1);
        ptx::mbar_wait(o_done, (n_tiles - 1) & 1);
        ptx::tc_fence_after();
        const float inv = 1.f / l;
        __nv_bfloat16* orow = o + static_cast<int64_t>(row0 + qrow) * HD + head * D;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t rr[32];
            ptx::tmem_ld_32x32b_x32(t_o + lane_off + c * 32, rr);
            ptx::tmem_ld_wait();
            if (qrow < S) {
#pragma unroll
                for (int i = 0; i < 32; i += 8) {
                    uint4 pk;
                    uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        __nv_bfloat162 hb = __floats2bfloat162_rn(__uint_as_float(rr[i + 2 * u]) * inv,
                                                                  __uint_as_float(rr[i + 2 * u + 1]) * inv);
                        w[u] = *reinterpret_cast<uint32_t*>(&hb);
                    }
                    *reinterpret_cast<uint4*>(orow + c * 32 + i) = pk;
                }
            }
        }
        if (qrow < S) lse[(static_cast<int64_t>(b) * H + head) * S + qrow] = m_used + __log2f(l);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<512>(tmem);
}

// -------------------------------------------------------------------------------------
// Forward, two query tiles per CTA (adjacent 128-query blocks 2p, 2p+1 of one head), sharing every
// K / V tile; 10 warps:
//   warp 0      TMA: Q0, Q1 once, K_j and V_j through 2-stage rings
//   warp 1      MMA issuer: S_t,0 for both tiles, then per key tile j and tile t:
//                 O_t += P_t,j V_j (A = P read from TMEM over S_t), then S_t,j+1 = Q_t K_j+1^T
//   warps 2..5  softmax of tile 0, warps 6..9 softmax of tile 1 (thread = query row): while one
//               tile's softmax runs, the tensor pipe works on the other tile (ping-pong)
// TMEM: O0 [0,128), O1 [128,256), S0/P0 [256,384), S1/P1 [384,512). S_t,j+1 is issued after PV_t,j,
// so when softmax t sees S_t,j+1 the previous PV has completed and O_t may be rescaled at once.
struct Fwd2Smem {
    static constexpr int kQ = 0;               // [2 tiles]
    static constexpr int kK = kQ + 2 * kTile;  // 2 stages
    static constexpr int kV = kK + 2 * kTile;  // 2 stages
    static constexpr int kBar = kV + 2 * kTile;
    static constexpr int kBytes = kBar + 256 + 1024;
};

__global__ void __launch_bounds__(320, 1)
    attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tm_qkv, __nv_bfloat16* __restrict__ o,
                        float* __restrict__ lse, int S, int H, float scale_log2) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + Fwd2Smem::kBar);
    uint64_t* q_full = bar + 0;
    uint64_t* k_full = bar + 1;   // [2]
    uint64_t* k_empty = bar + 3;  // [2]
    uint64_t* v_full = bar + 5;   // [2]
    uint64_t* v_empty = bar + 7;  // [2]
    uint64_t* s_full = bar + 9;   // [tile]
    uint64_t* p_full = bar + 11;  // [tile]
    uint64_t* o_done = bar + 13;  // [tile] PV_t,j complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

    // grid (H, query-block pairs, B), longest pairs first
    const int n_qb = (S + BQ - 1) / BQ;
    const int n_pairs = (n_qb + 1) / 2;
    const int pr = n_pairs - 1 - blockIdx.y;
    const int head = blockIdx.x, b = blockIdx.z;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int HD = H * D;
    const int row0 = b * S;
    const int n_tq = 2 * pr + 1 < n_qb ? 2 : 1;  // query tiles of this CTA
    auto tiles_of = [&](int t) { return (min((2 * pr + t + 1) * BQ, S) + BKV - 1) / BKV; };
    const int n_max = tiles_of(n_tq - 1);

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tm_qkv);
        ptx::mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&k_full[i], 1);
            ptx::mbar_init(&k_empty[i], 1);
            ptx::mbar_init(&v_full[i], 1);
            ptx::mbar_init(&v_empty[i], 1);
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&p_full[i], 4);
            ptx::mbar_init(&o_done[i], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const int qcol = head * D, kcol = HD + head * D, vcol = 2 * HD + head * D;
            ptx::mbar_expect_tx(q_full, n_tq * kTile);
            for (int t = 0; t < n_tq; ++t)
                for (int h2 = 0; h2 < 2; ++h2)
                    ptx::tma_load_2d(sm + Fwd2Smem::kQ + t * kTile + h2 * (kTile / 2), &tm_qkv, q_full,
                                     qcol + 64 * h2, row0 + (2 * pr + t) * BQ);
            for (int j = 0; j < n_max; ++j) {
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                ptx::mbar_wait(&k_empty[st], ph ^ 1);
                ptx::mbar_expect_tx(&k_full[st], kTile);
                for (int h2 = 0; h2 < 2; ++h2)
                    ptx::tma_load_2d(sm + Fwd2Smem::kK + st * kTile + h2 * (kTile / 2), &tm_qkv, &k_full[st],
                                     kcol + 64 * h2, row0 + j * BKV);
                ptx::mbar_wait(&v_empty[st], ph ^ 1);
                ptx::mbar_expect_tx(&v_full[st], kTile);
                for (int h2 = 0; h2 < 2; ++h2)
                    ptx::tma_load_2d(sm + Fwd2Smem::kV + st * kTile + h2 * (kTile / 2), &tm_qkv, &v_full[st],
                                     vcol + 64 * h2, row0 + j * BKV);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(128, 128, 0, 0);   // Q K^T: both K-major
            constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(128, 128, 0, 1);  // P V: V is MN-major
            ptx::mbar_wait(q_full, 0);
            auto issue_s = [&](int t, int j) {
                const int st = j & 1;
                ptx::mbar_wait(&k_full[st], (j >> 1) & 1);
                ptx::tc_fence_after();
                const uint32_t sq = ptx::smem_u32(sm + Fwd2Smem::kQ + t * kTile);
                const uint32_t sk = ptx::smem_u32(sm + Fwd2Smem::kK + st * kTile);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    ptx::umma_f16(tmem + 256 + t * 128, kmajor_desc(sq, kk), kmajor_desc(sk, kk), idesc_s, kk != 0);
                ptx::umma_commit(&s_full[t]);
            };
            for (int t = 0; t < n_tq; ++t) issue_s(t, 0);
            for (int j = 0; j < n_max; ++j) {
                const int st = j & 1;
                for (int t = 0; t < n_tq; ++t) {
                    const int nt = tiles_of(t);
                    if (j >= nt) continue;
                    ptx::mbar_wait(&p_full[t], j & 1);
                    ptx::mbar_wait(&v_full[st], (j >> 1) & 1);
                    ptx::tc_fence_after();
                    const uint32_t sv = ptx::smem_u32(sm + Fwd2Smem::kV + st * kTile);
#pragma unroll
                    for (int kk = 0; kk < BKV / 16; ++kk)  // P: 16 keys = 8 packed columns per K-step
                        ptx::umma_f16_ts(tmem + t * 128, tmem + 256 + t * 128 + kk * 8, mnmajor_desc(sv, kk),
                                         idesc_pv, (j | kk) != 0);
                    ptx::umma_commit(&o_done[t]);
                    if (j + 1 < nt) issue_s(t, j + 1);
                }
                ptx::umma_commit(&k_empty[st]);
                ptx::umma_commit(&v_empty[st]);
            }
        }
    } else {
        // ===== softmax warps: tile t = (warp - 2) / 4, thread = query row =====
        const int t = (warp - 2) >> 2;
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const int qb = 2 * pr + t;
        const int qrow = qb * BQ + r;
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        const uint32_t t_o = tmem + t * 128, t_s = tmem + 256 + t * 128;
        if (t < n_tq) {
            const int n_tiles = tiles_of(t);
            float m_used = -INFINITY, l = 0.f;
            for (int j = 0; j < n_tiles; ++j) {
                ptx::mbar_wait(&s_full[t], j & 1);
                ptx::tc_fence_after();
                float s[128];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t rr[32];
                    ptx::tmem_ld_32x32b_x32(t_s + lane_off + c * 32, rr);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(rr[i]);
                }
                const int k0 = j * BKV;
                const bool diag = k0 + BKV - 1 > qb * BQ || k0 + BKV > S;
                const int lim = diag ? min(qrow + 1, S) - k0 : BKV;
                float mx = -INFINITY;
#pragma unroll
                for (int i = 0; i < 128; ++i) {
                    const float v = i < lim ? s[i] * scale_log2 : -INFINITY;
                    s[i] = v;
                    mx = fmaxf(mx, v);
                }
                // warp-uniform rescale (tcgen05.ld/st are .sync.aligned); O_t is stable: S_t,j was
                // issued after PV_t,j-1 and s_full fired once every earlier MMA had completed
                const bool mine = mx > m_used + kRescaleThreshold;
                if (__any_sync(0xffffffffu, mine)) {
                    const float alpha = mine ? (m_used == -INFINITY ? 0.f : ptx::ex2_fast(m_used - mx)) : 1.f;
                    if (mine) m_used = mx;
                    l *= alpha;
                    if (j > 0) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            uint32_t rr[32];
                            ptx::tmem_ld_32x32b_x32(t_o + lane_off + c * 32, rr);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 32; ++i) rr[i] = __float_as_uint(__uint_as_float(rr[i]) * alpha);
                            ptx::tmem_st_32x32b_x32(t_o + lane_off + c * 32, rr);
                        }
                    }
                }
                float sum = 0.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t w[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float p0 = ptx::ex2_fast(s[c * 32 + 2 * i] - m_used);
                        const float p1 = ptx::ex2_fast(s[c * 32 + 2 * i + 1] - m_used);
                        sum += p0 + p1;
                        __nv_bfloat162 hb = __floats2bfloat162_rn(p0, p1);
                        w[i] = *reinterpret_cast<uint32_t*>(&hb);
                    }
                    ptx::tmem_st_32x32b_x16(t_s + lane_off + c * 16, w);
                }
                l += sum;
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&p_full[t]);
            }
            // epilogue: passing s_full_t(n-1) proved PV_t(n-2) done; wait for PV_t(n-1)
            ptx::mbar_wait(&o_done[t], (n_tiles - 1) & 1);
            ptx::tc_fence_after();
            const float inv = 1.f / l;
            __nv_bfloat16* orow = o + static_cast<int64_t>(row0 + qrow) * HD + head * D;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t rr[32];
                ptx::tmem_ld_32x32b_x32(t_o + lane_off + c * 32, rr);
                ptx::tmem_ld_wait();
                if (qrow < S) {
#pragma unroll
                    for (int i = 0; i < 32; i += 8) {
                        uint4 pk;
                        uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            __nv_bfloat162 hb = __floats2bfloat162_rn(__uint_as_float(rr[i + 2 * u]) * inv,
                                                                      __uint_as_float(rr[i + 2 * u + 1]) * inv);
                            w[u] = *reinterpret_cast<uint32_t*>(&hb);
                        }
                        *reinterpret_cast<uint4*>(orow + c * 32 + i) = pk;
                    }
                }
            }
            if (qrow < S) lse[(static_cast<int64_t>(b) * H + head) * S + qrow] = m_used + __log2f(l);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace

int attn_fwd_tiles = 0;  // query tiles per forward CTA: 0 auto, 1, 2 (tests / benchmarks)

void attention_fwd_tc(const void* qkv, void* o, float* lse, int batch, int seq, int heads, int head_dim,
                      cudaStream_t st) {
    if (head_dim != D) throw std::runtime_error("attention: head_dim must be 128");
    static bool cfg = false;
    if (!cfg) {
        cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem::kBytes);
        cfg = true;
    }
    const int64_t T = static_cast<int64_t>(batch) * seq, h3 = 3LL * heads * head_dim;
    const CUtensorMap tm = make_tma_2d(qkv, h3, T, h3, 128, false);
    dim3 grid(heads, (seq + BQ - 1) / BQ, batch);
    if (heads > 1 && seq > BQ) count_variant(KV_ATTN_FWD_MULTI);
    const float scale_log2 = kLog2e / sqrtf(static_cast<float>(head_dim));
    // two query tiles per CTA halve the CTA count; with fewer than ~2 waves of pairs the causal
    // imbalance (the longest pair has 2x the key tiles of the longest single block) outweighs the
    // ping-pong (measured: 1x2048x16 heads 28.9 vs 46.4 us; 4x2048x32 218 vs 208 us; 1x4096x16 90
    // vs 87 us). BFPP_ATTN_FWD=1 / 2 forces one / two tiles.
    const int n_qb = (seq + BQ - 1) / BQ;
    const int64_t pair_ctas = static_cast<int64_t>(heads) * batch * ((n_qb + 1) / 2);
    static const int env = getenv("BFPP_ATTN_FWD") ? atoi(getenv("BFPP_ATTN_FWD")) : 0;
    const int force = attn_fwd_tiles ? attn_fwd_tiles : env;
    const bool one_tile = force == 1 || (force != 2 && pair_ctas < 256);
    if (one_tile) {
        attn_fwd_tc_kernel<<<grid, 192, FwdSmem::kBytes, st>>>(tm, static_cast<__nv_bfloat16*>(o), lse, seq, heads,
                                                               scale_log2);
        return;
    }
    static bool cfg2 = false;
    if (!cfg2) {
        cudaFuncSetAttribute(attn_fwd_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Smem::kBytes);
        cfg2 = true;
    }
    dim3 grid2(heads, (n_qb + 1) / 2, batch);
    attn_fwd_tc2_kernel<<<grid2, 320, Fwd2Smem::kBytes, st>>>(tm, static_cast<__nv_bfloat16*>(o), lse, seq, heads,
                                                              scale_log2);
}


// =====================================================================================
namespace {

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// -------------------------------------------------------------------------------------
// Backward: one CTA per (128-key block, head, sample), 18 warps (576 threads). Every MMA is
// 128 x 128 x 16 (an N = 64 MMA takes as long as N = 128); the elementwise work of a query block
// is split into two 64-query halves h = A, B so dV_A / dK_A start while half B is computed:
//   warp 0      TMA: K, V once; Q_i (2-stage ring) and dO_i per query block (one buffer per
//               64-row half, refilled as soon as that half's dV MMAs have read it)
//   warp 1      MMA issuer (one thread), per query block i, in issue order:
//                 S^T = K Q_i^T -> TMEM[0,128)   dP^T = V dO_i^T -> TMEM[128,256)
//                 for h: dV += P_h^T dO_h   (A = P_h^T read from TMEM, packed over S_h^T)
//                        (h = B: dQ^T = K^T dS^T -> TMEM[128,256), lanes = head dims)
//                        dK += dS_h^T Q_h   (A = dS^T from shared memory)
//   warps 2..9  dQ drain, two per TMEM lane quadrant: thread = head dim d; a warp takes its 32
//               dims x 64 queries out of TMEM at once (releasing the columns), then stages them as
//               two SWIZZLE_128B [32 queries][32 dims] f32 boxes, each added to the f32 dQ
//               accumulator with one TMA reduce-add (cp.reduce.async.bulk.tensor)
//   warps 10..17: elementwise, two per TMEM lane quadrant (thread = key row), one per 64-query
//               half h of each block, 16 queries at a time: P^T = exp2(S^T*scale_log2 - lse)
//               packed bf16 into TMEM over the half's own S^T columns, dS^T = P^T (dP^T - delta)
//               bf16 into shared memory (packed f32x2 arithmetic; the causal selects only on
//               diagonal / partial blocks); finally dK, dV.
// Shared memory: K, V, Q[2], dO, dS^T, dQ staging (8 x [32][32] f32) = 7 x 32 KB + lse/delta
// (exactly fits 227 KB; the dynamic shared window is 1024-byte aligned, checked at run time).
struct BwdSmem {
    static constexpr int kK = 0, kV = kTile, kQ = 2 * kTile, kO = 4 * kTile, kS = 5 * kTile, kDQ = 6 * kTile;
    static constexpr int kStat = 7 * kTile;  // [half][iteration parity][-lse 64 | -delta 64] f32
    static constexpr int kBar = kStat + 2048;
    static constexpr int kBytes = kBar + 160;  // 17 mbarriers + the TMEM address
};
static_assert(BwdSmem::kBytes <= 232448, "attention backward shared memory");

// Elementwise core of the backward for N queries of one key row: rs = S^T, rd = dP^T (TMEM
// words), nl / nd = -lse / -delta of the N queries (shared memory, broadcast), [lo, hi) = the
// visible query range (MASK only) -> P^T and dS^T as packed bf16 pairs.
template <bool MASK, int N>
__device__ __forceinline__ void bwd_elementwise(const uint32_t (&rs)[N], const uint32_t (&rd)[N], const float* nl,
                                                const float* nd, float scale_log2, int q_base, int lo, int hi,
                                                uint32_t (&pw)[N / 2], uint32_t (&dw)[N / 2]) {
    const uint64_t sc = ptx::pack2(scale_log2, scale_log2);
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        const float2 nl2 = *reinterpret_cast<const float2*>(nl + j);
        const float2 nd2 = *reinterpret_cast<const float2*>(nd + j);
        const float2 t = ptx::unpack2(ptx::ffma2(ptx::pack2(__uint_as_float(rs[j]), __uint_as_float(rs[j + 1])), sc,
                                                 ptx::pack2(nl2.x, nl2.y)));
        float p0 = ptx::ex2_fast(t.x), p1 = ptx::ex2_fast(t.y);
        if (MASK) {
            const int q = q_base + j;
            p0 = ((q >= lo) & (q < hi)) ? p0 : 0.f;
            p1 = ((q + 1 >= lo) & (q + 1 < hi)) ? p1 : 0.f;
        }
        const uint64_t pp = ptx::pack2(p0, p1);
        const float2 d = ptx::unpack2(
            ptx::fmul2(pp, ptx::fadd2(ptx::pack2(__uint_as_float(rd[j]), __uint_as_float(rd[j + 1])),
                                      ptx::pack2(nd2.x, nd2.y))));
        __nv_bfloat162 hp = __floats2bfloat162_rn(p0, p1), hd = __floats2bfloat162_rn(d.x, d.y);
        pw[j / 2] = *reinterpret_cast<uint32_t*>(&hp);
        dw[j / 2] = *reinterpret_cast<uint32_t*>(&hd);
    }
}

__global__ void __launch_bounds__(576, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                        const __grid_constant__ CUtensorMap tm_dq, const float* __restrict__ lse,
                        const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, int S, int H, float scale,
                        float scale_log2) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw;
    if (threadIdx.x == 0 && (ptx::smem_u32(sm) & 1023u)) __trap();
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BwdSmem::kBar);
    uint64_t* kv_full = bar + 0;
    uint64_t* q_full = bar + 1;    // [2]
    uint64_t* q_empty = bar + 3;   // [2]
    uint64_t* s_full = bar + 5;
    uint64_t* p_full = bar + 7;    // [half]
    uint64_t* dq_full = bar + 9;
    uint64_t* dq_empty = bar + 11;
    uint64_t* o_full = bar + 13;   // [half]
    uint64_t* o_empty = bar + 15;  // [half]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);

    const int kb = blockIdx.y;
    const int head = blockIdx.x, b = blockIdx.z;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int HD = H * D;
    const int row0 = b * S;
    const int i0 = kb;  // first query block that sees this key block (BQ == BKV)
    const int n_qb = (S + BQ - 1) / BQ;
    const int n_it = n_qb - i0;
    constexpr int kHalf = kTile / 4;  // 64 rows x 128 B: row offset of the second half of a tile

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tm_qkv);
        ptx::tma_prefetch(&tm_do);
        ptx::tma_prefetch(&tm_dq);
        ptx::mbar_init(kv_full, 1);
        ptx::mbar_init(s_full, 1);
        ptx::mbar_init(dq_full, 1);
        ptx::mbar_init(dq_empty, 8);
        for (int k = 0; k < 2; ++k) {
            ptx::mbar_init(&q_full[k], 1);
            ptx::mbar_init(&q_empty[k], 1);
            ptx::mbar_init(&p_full[k], 4);
            ptx::mbar_init(&o_full[k], 1);
            ptx::mbar_init(&o_empty[k], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t t_s = tmem, t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 384;

    if (warp == 0) {
        if (lane == 0) {
            const int qcol = head * D, kcol = HD + head * D, vcol = 2 * HD + head * D;
            ptx::mbar_expect_tx(kv_full, 2 * kTile);
            for (int h2 = 0; h2 < 2; ++h2) {
                ptx::tma_load_2d(sm + BwdSmem::kK + h2 * (kTile / 2), &tm_qkv, kv_full, kcol + 64 * h2, row0 + kb * BKV);
                ptx::tma_load_2d(sm + BwdSmem::kV + h2 * (kTile / 2), &tm_qkv, kv_full, vcol + 64 * h2, row0 + kb * BKV);
            }
            for (int it = 0; it < n_it; ++it) {
                const int st = it & 1, i = i0 + it;
                if (it >= 2) ptx::mbar_wait(&q_empty[st], ((it >> 1) & 1) ^ 1);
                ATRACE(0, it, 0);
                ptx::mbar_expect_tx(&q_full[st], kTile);
                for (int h2 = 0; h2 < 2; ++h2)
                    ptx::tma_load_2d(sm + BwdSmem::kQ + st * kTile + h2 * (kTile / 2), &tm_qkv, &q_full[st],
                                     qcol + 64 * h2, row0 + i * BQ);
                for (int h = 0; h < 2; ++h) {  // dO rows 64h..64h+63: [2 dim blocks][64 rows][128 B]
                    if (it >= 1) ptx::mbar_wait(&o_empty[h], (it - 1) & 1);
                    ATRACE(0, it, 1 + h);
                    ptx::mbar_expect_tx(&o_full[h], kTile / 2);
                    for (int h2 = 0; h2 < 2; ++h2)
                        ptx::tma_load_2d(sm + BwdSmem::kO + h2 * (kTile / 2) + h * kHalf, &tm_do, &o_full[h],
                                         head * D + 64 * h2, row0 + i * BQ + 64 * h);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id_kk = ptx::idesc_bf16_f32(128, 128, 0, 0);  // S^T, dP^T: A, B K-major
            constexpr uint32_t id_kn = ptx::idesc_bf16_f32(128, 128, 0, 1);  // dV, dK: B MN-major
            constexpr uint32_t id_nn = ptx::idesc_bf16_f32(128, 128, 1, 1);  // dQ^T: A, B MN-major
            const uint32_t sk = ptx::smem_u32(sm + BwdSmem::kK), sv = ptx::smem_u32(sm + BwdSmem::kV);
            const uint32_t so = ptx::smem_u32(sm + BwdSmem::kO), sds = ptx::smem_u32(sm + BwdSmem::kS);
            ptx::mbar_wait(kv_full, 0);
            for (int it = 0; it < n_it; ++it) {
                const int st = it & 1;
                const uint32_t sq = ptx::smem_u32(sm + BwdSmem::kQ + st * kTile);
                ptx::mbar_wait(&q_full[st], (it >> 1) & 1);
                ATRACE(1, it, 0);
                ptx::tc_fence_after();
                // S^T overwrites P^T of the previous block: issued after that block's dV (the
                // tensor pipe executes one thread's MMAs in issue order). All MMAs are 128 x 128:
                // N = 64 costs as much tensor time as N = 128.
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    ptx::umma_f16(t_s, kmajor_desc(sk, kk), kmajor_desc(sq, kk), id_kk, kk != 0);
                if (it > 0) ptx::mbar_wait(dq_empty, (it - 1) & 1);  // dQ of block i-1 drained
                ATRACE(1, it, 1);
                ptx::mbar_wait(&o_full[0], it & 1);
                ptx::mbar_wait(&o_full[1], it & 1);
                ATRACE(1, it, 2);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    ptx::umma_f16(t_dp, kmajor_desc(sv, kk), kmajor_desc(so, kk), id_kk, kk != 0);
                ptx::umma_commit(s_full);
                ATRACE(1, it, 3);
                for (int h = 0; h < 2; ++h) {
                    ptx::mbar_wait(&p_full[h], it & 1);
                    ATRACE(1, it, 7 + 2 * h);
                    ptx::tc_fence_after();
                    // dV += P_h^T dO_h: K-step kk = queries 16kk..16kk+15 of the block; P_h^T packed
                    // in TMEM at columns 64h + 8 (kk % 4)
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4) {
                        const int kk = h * 4 + k4;
                        ptx::umma_f16_ts(t_dv, t_s + h * 64 + k4 * 8, mnmajor_desc(so, kk), id_kn, (it | kk) != 0);
                    }
                    ptx::umma_commit(&o_empty[h]);  // dO rows of this half: read by dP^T and dV only (the
                                                    // refill overlaps the rest of the block)
                    if (h == 1) {
                        // dQ^T [d][q] = sum_key K[key][d] dS[q][key]: A = K (MN-major over d),
                        // B = dS^T tile (MN-major over q), K-step = 16 keys; before dK_B so the
                        // drain overlaps dK_B and the next S^T
#pragma unroll
                        for (int kk = 0; kk < BKV / 16; ++kk)
                            ptx::umma_f16(t_dp, mnmajor_desc(sk, kk), mnmajor_desc(sds, kk), id_nn, kk != 0);
                        ptx::umma_commit(dq_full);
                        ATRACE(1, it, 10);
                    }
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4) {
                        const int kk = h * 4 + k4;
                        ptx::umma_f16(t_dk, kmajor_desc(sds, kk), mnmajor_desc(sq, kk), id_kn, (it | kk) != 0);
                    }
                }
                ptx::umma_commit(&q_empty[st]);
                ATRACE(1, it, 11);
            }
        }
    } else if (warp < 10) {
        // ===== dQ drain: thread = head dim d (TMEM lane); warp (q4, dh) owns dims q4*32..+31 of
        // queries 64dh..64dh+63 and stages them as two [32 queries][32 dims] f32 boxes =====
        const int q4 = warp & 3, dh = (warp - 2) >> 2;
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        uint8_t* box_ptr = sm + BwdSmem::kDQ + (warp - 2) * 4096;  // [32 queries][32 dims] f32, SWIZZLE_128B
        const uint32_t box = ptx::smem_u32(box_ptr);
        const uint32_t col = static_cast<uint32_t>(lane & 3) * 4;
        for (int it = 0; it < n_it; ++it) {
            const int q0 = (i0 + it) * BQ + dh * 64;
            if (warp == 2 && lane == 0) ATRACE(2, it, 0);
            ptx::mbar_wait(dq_full, it & 1);
            if (warp == 2 && lane == 0) ATRACE(2, it, 1);
            ptx::tc_fence_after();
            uint32_t v[2][32];
            ptx::tmem_ld_32x32b_x32(t_dp + lane_off + dh * 64, v[0]);
            ptx::tmem_ld_32x32b_x32(t_dp + lane_off + dh * 64 + 32, v[1]);
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(dq_empty);  // this warp's share of dQ^T is in registers
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
                if (lane == 0) ptx::bulk_wait_read<0>();  // the previous reduce has read the box
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 32; ++j)  // row j of the box = query q0 + 32 c2 + j
                    ptx::st_shared_f32(box + j * 128 + ((((lane >> 2) ^ j) & 7) << 4) + col,
                                       __uint_as_float(v[c2][j]) * scale);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::tma_reduce_add_2d(&tm_dq, box_ptr, head * D + q4 * 32, row0 + q0 + c2 * 32);
                    ptx::bulk_commit();
                    if (warp == 2) ATRACE(2, it, 2 + c2);
                }
            }
        }
        if (lane == 0) ptx::bulk_wait<0>();
    } else {
        // ===== elementwise: thread = key row r, query half h (64 queries) of every block =====
        const int q4 = warp & 3, h = (warp - 10) >> 2;
        const int r = q4 * 32 + lane;
        const int key = kb * BKV + r;
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        const int e = threadIdx.x - (10 + 4 * h) * 32;  // 0..127 within the half: lse (< 64) or delta
        const uint32_t sds_base = ptx::smem_u32(sm + BwdSmem::kS);
        const int64_t stat_base = (static_cast<int64_t>(b) * H + head) * S;
        const float* stat = e < 64 ? lse : delta;
        const int eq = e & 63;
        float nxt = 0.f;
        {
            const int q = i0 * BQ + h * 64 + eq;
            if (q < S) nxt = stat[stat_base + q];
        }
        for (int it = 0; it < n_it; ++it) {
            const int i = i0 + it;
            const int qh = i * BQ + h * 64;  // first query of this half
            // [parity][lse 64 | delta 64]: a warp one iteration ahead never overwrites values a
            // slower warp of the half still reads (nobody passes the barrier two iterations ahead)
            reinterpret_cast<float*>(sm + BwdSmem::kStat + h * 1024 + (it & 1) * 512)[e] = -nxt;  // -lse | -delta
            if (it + 1 < n_it) {
                const int q = qh + BQ + eq;
                nxt = q < S ? stat[stat_base + q] : 0.f;
            }
            if (lane == 0 && (warp == 10 || warp == 14)) ATRACE(3 + h, it, 0);
            named_bar_sync(1 + h, 128);
            if (lane == 0 && (warp == 10 || warp == 14)) ATRACE(3 + h, it, 1);
            // s_full(i) also orders after every MMA of block i-1 (the readers of dS^T)
            ptx::mbar_wait(s_full, it & 1);
            if (lane == 0 && (warp == 10 || warp == 14)) ATRACE(3 + h, it, 2);
            ptx::tc_fence_after();
            const bool mask = (i == i0) || (i * BQ + BQ > S) || (kb * BKV + BKV > S);
            // valid queries of this thread's key row: key <= q < S, as a [lo, hi) range of the
            // half's query index (empty when key >= S); a select per element, no branches
            const int lo = mask ? key - qh : INT_MIN, hi = mask ? S - qh : INT_MAX;
            const float* Lp = reinterpret_cast<const float*>(sm + BwdSmem::kStat + h * 1024 + (it & 1) * 512);
            const float* Dp = Lp + 64;
#pragma unroll 1
            for (int sub = 0; sub < 4; ++sub) {
                const int qc = sub * 16;  // first query of the 16 within the half
                uint32_t rs[16], rd[16];
                ptx::tmem_ld_32x32b_x16(t_s + lane_off + h * 64 + qc, rs);
                ptx::tmem_ld_32x32b_x16(t_dp + lane_off + h * 64 + qc, rd);
                ptx::tmem_ld_wait();
                uint32_t pw[8], dw[8];
                if (mask)  // warp-uniform: only diagonal / partial blocks pay for the selects
                    bwd_elementwise<true, 16>(rs, rd, Lp + qc, Dp + qc, scale_log2, qc, lo, hi, pw, dw);
                else
                    bwd_elementwise<false, 16>(rs, rd, Lp + qc, Dp + qc, scale_log2, qc, lo, hi, pw, dw);
                // P^T packed over this half's S^T columns 64h + [8 sub, 8 sub + 8): all read already
                ptx::tmem_st_32x32b_x8(t_s + lane_off + h * 64 + sub * 8, pw);
                // dS^T row r of the [2 q-halves][128 keys][128 B] SW128 tile: 16-byte chunks qc / 8 + {0, 1}
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int ch = qc / 8 + u;
                    const uint32_t off = h * (kTile / 2) + r * 128 + ((ch ^ (r & 7)) << 4);
                    ptx::st_shared_v4(sds_base + off, dw[4 * u], dw[4 * u + 1], dw[4 * u + 2], dw[4 * u + 3]);
                }
            }
            ptx::tmem_st_wait();
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&p_full[h]);
            if (lane == 0 && (warp == 10 || warp == 14)) ATRACE(3 + h, it, 3);
        }
        // dK (scaled) and dV: every MMA has completed once the last block's q_empty commit fires
        // (its previous phase, block n-3, completed before s_full of block n-1)
        {
            const int last = n_it - 1;
            ptx::mbar_wait(&q_empty[last & 1], (last >> 1) & 1);
        }
        ptx::tc_fence_after();
        __nv_bfloat16* dkr = dqkv + static_cast<int64_t>(row0 + key) * 3 * HD + HD + head * D;
        __nv_bfloat16* dvr = dqkv + static_cast<int64_t>(row0 + key) * 3 * HD + 2 * HD + head * D;
#pragma unroll 1
        for (int sub = 0; sub < 4; ++sub) {
            const int c0 = h * 64 + sub * 16;
            uint32_t rk[16], rv[16];
            ptx::tmem_ld_32x32b_x16(t_dk + lane_off + c0, rk);
            ptx::tmem_ld_32x32b_x16(t_dv + lane_off + c0, rv);
            ptx::tmem_ld_wait();
            if (key >= S) continue;
#pragma unroll
            for (int j = 0; j < 16; j += 8) {
                uint4 ok, ov;
                uint32_t* wk = reinterpret_cast<uint32_t*>(&ok);
                uint32_t* wv = reinterpret_cast<uint32_t*>(&ov);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    __nv_bfloat162 a = __floats2bfloat162_rn(__uint_as_float(rk[j + 2 * u]) * scale,
                                                             __uint_as_float(rk[j + 2 * u + 1]) * scale);
                    __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(rv[j + 2 * u]),
                                                             __uint_as_float(rv[j + 2 * u + 1]));
                    wk[u] = *reinterpret_cast<uint32_t*>(&a);
                    wv[u] = *reinterpret_cast<uint32_t*>(&v);
                }
                *reinterpret_cast<uint4*>(dkr + c0 + j) = ok;
                *reinterpret_cast<uint4*>(dvr + c0 + j) = ov;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<512>(tmem);
}

}  // namespace

void attention_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* delta, float* dq_acc,
                      void* dqkv, int batch, int seq, int heads, int head_dim, cudaStream_t st) {
    if (head_dim != D) throw std::runtime_error("attention: head_dim must be 128");
    static bool cfg = false;
    if (!cfg) {
        cudaFuncSetAttribute(attn_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BwdSmem::kBytes);
        cfg = true;
    }
    const int64_t T = static_cast<int64_t>(batch) * seq, HD = static_cast<int64_t>(heads) * head_dim;
    const CUtensorMap tq = make_tma_2d(qkv, 3 * HD, T, 3 * HD, 128, false);
    const CUtensorMap to64 = make_tma_2d(dout, HD, T, HD, 64, false);  // dO loaded per 64-row half
    dim3 grid(heads, (seq + BKV - 1) / BKV, batch);
    if (heads > 1 && seq > BKV) count_variant(KV_ATTN_BWD_MULTI);
    const float scale = 1.f / sqrtf(static_cast<float>(head_dim));
    const CUtensorMap tdq = make_tma_2d(dq_acc, HD, T, HD, 32, true);  // [32 queries][32 dims] boxes
    attn_bwd_tc_kernel<<<grid, 576, BwdSmem::kBytes, st>>>(tq, to64, tdq, lse, delta,
                                                             static_cast<__nv_bfloat16*>(dqkv), seq, heads, scale,
                                                             scale * kLog2e);
}

}  // namespace bfpp
