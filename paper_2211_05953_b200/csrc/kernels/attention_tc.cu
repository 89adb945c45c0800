// Causal flash attention forward on the 5th-gen tensor cores (sm_100a), head_dim 128.
//
// One CTA per (128-query block, head, sample). Warp roles (192 threads):
//   warp 0      TMA producer: Q once, then K and V tiles of 128 keys (2-stage rings)
//   warp 1      MMA issuer (one elected thread) + TMEM owner:
//                 S_j = Q K_j^T  -> TMEM (double-buffered, so S_{j+1} overlaps softmax_j)
//                 O  += P_j V_j  -> TMEM (A = P from shared memory, B = V MN-major)
//   warps 2..5  softmax: thread = query row (TMEM lane); the whole 128-key row of S is in
//               registers, so max / sum need no shuffles. Online softmax in the log2
//               domain with a lazily updated running max (O in TMEM is rescaled only when
//               the max grows by more than 2^8), P written as bf16 into a SWIZZLE_128B
//               K-major tile for the PV MMA.
// Layouts as attention.cu: qkv [B*S][3*H*128], o [B*S][H*128], lse [B*H][S] (log2 domain).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdexcept>

#include "gemm.hpp"
#include "kernels.hpp"
#include "sm100_ptx.cuh"

namespace bfpp {
namespace {

constexpr int D = 128, BQ = 128, BKV = 128;
constexpr int kTile = 128 * 128 * 2;  // one [128 rows][128 dims] bf16 tile = 2 x [128][64] SW128 blocks
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.f;  // log2 units

struct FwdSmem {
    static constexpr int kQ = 0;
    static constexpr int kK = kQ + kTile;          // 2 stages
    static constexpr int kV = kK + 2 * kTile;      // 2 stages
    static constexpr int kP = kV + 2 * kTile;
    static constexpr int kBar = kP + kTile;
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
    uint64_t* s_empty = bar + 11; // [2]
    uint64_t* p_full = bar + 13;
    uint64_t* o_done = bar + 14;  // PV_j complete (P buffer free, O stable)
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
            ptx::mbar_init(&s_empty[i], 4);
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
            const uint32_t sp = ptx::smem_u32(sm + FwdSmem::kP);
            ptx::mbar_wait(q_full, 0);
            auto issue_s = [&](int j) {
                const int st = j & 1;
                const uint32_t ph = (j >> 1) & 1;
                ptx::mbar_wait(&k_full[st], ph);
                ptx::mbar_wait(&s_empty[st], ph ^ 1);
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
                for (int kk = 0; kk < BKV / 16; ++kk)
                    ptx::umma_f16(t_o, kmajor_desc(sp, kk), mnmajor_desc(sv, kk), idesc_pv, (j | kk) != 0);
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
        const uint32_t prow = ptx::smem_u32(sm + FwdSmem::kP) + r * 128;
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
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&s_empty[st]);
            const int k0 = j * BKV;
            const bool diag = k0 + BKV - 1 > qb * BQ || k0 + BKV > S;
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < 128; ++i) {
                float v = s[i] * scale_log2;
                if (diag && (k0 + i > qrow || k0 + i >= S)) v = -INFINITY;
                s[i] = v;
                mx = fmaxf(mx, v);
            }
            // P buffer and O are free once PV_{j-1} has completed
            if (j > 0) ptx::mbar_wait(o_done, (j - 1) & 1);
            // The rescale decision is per row, but tcgen05.ld/st are warp-collective
            // (.sync.aligned): if any row of the warp needs it, the whole warp rescales (rows
            // that do not need it use alpha = 1), so the TMEM accesses never diverge.
            const bool mine = mx > m_used + kRescaleThreshold;
            if (__any_sync(0xffffffffu, mine)) {
                const float m_new = mine ? mx : m_used;
                const float alpha = mine ? (m_used == -INFINITY ? 0.f : ptx::ex2_fast(m_used - mx)) : 1.f;
                l *= alpha;
                if (j > 0) {
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
                    ptx::tmem_st_wait();
                }
                m_used = m_new;
            }
            float sum = 0.f;
#pragma unroll
            for (int c = 0; c < 16; ++c) {  // 16 chunks of 8 keys = 16 B of bf16
                uint4 pk;
                uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float p0 = ptx::ex2_fast(s[8 * c + 2 * u] - m_used);
                    const float p1 = ptx::ex2_fast(s[8 * c + 2 * u + 1] - m_used);
                    sum += p0 + p1;
                    __nv_bfloat162 hb = __floats2bfloat162_rn(p0, p1);
                    w[u] = *reinterpret_cast<uint32_t*>(&hb);
                }
                // [2 key-blocks][128 rows][128 B], 16-byte chunk swizzled by row & 7
                const int blk = c >> 3, ch = c & 7;
                ptx::st_shared_v4(prow + blk * (kTile / 2) + ((ch ^ (r & 7)) << 4), pk);
            }
            l += sum;
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(p_full);
        }
        // epilogue: O / l -> bf16 -> global; lse = m + log2(l)
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

}  // namespace

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
    attn_fwd_tc_kernel<<<grid, 192, FwdSmem::kBytes, st>>>(tm, static_cast<__nv_bfloat16*>(o), lse, seq, heads,
                                                           scale_log2);
}


// =====================================================================================
// Backward: one CTA per (128-key block, head, sample), looping over the query blocks at or
// after the diagonal. Warp roles (192 threads):
//   warp 0      TMA: K, V once; Q_i and dO_i per query block (single buffer, reloaded as soon
//               as the MMAs that read them have completed)
//   warp 1      MMA: S^T = K Q_i^T and dP^T = V dO_i^T (TMEM, lanes = keys);
//               dV += P^T dO_i, dK += dS^T Q_i (TMEM accumulators); dQ_i = dS K (TMEM, lanes = q)
//   warps 2..5  thread = key row: P^T = exp2(S^T*scale_log2 - lse), dS^T = P^T (dP^T - delta),
//               both to shared memory as bf16 (K-major over q); then drain dQ_i (thread = q row)
//               with red.global.add.v4.f32; finally write dK, dV.
// TMEM columns: [0,128) S^T, [128,256) dP^T / dQ, [256,384) dV, [384,512) dK.
namespace {

struct BwdSmem {
    static constexpr int kK = 0, kV = kTile, kQ = 2 * kTile, kO = 3 * kTile, kP = 4 * kTile, kS = 5 * kTile;
    static constexpr int kLse = 6 * kTile;         // [2][128] f32 (double-buffered by iteration)
    static constexpr int kDelta = kLse + 1024;     // [2][128] f32
    static constexpr int kBar = kDelta + 1024;
    static constexpr int kBytes = kBar + 256 + 1024;
};

__device__ __forceinline__ void red_add_v4(float* dst, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

__global__ void __launch_bounds__(192, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                       const float* __restrict__ lse, const float* __restrict__ delta, float* __restrict__ dq_acc,
                       __nv_bfloat16* __restrict__ dqkv, int S, int H, float scale, float scale_log2) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BwdSmem::kBar);
    uint64_t* kv_full = bar + 0;
    uint64_t* qo_full = bar + 1;
    uint64_t* qo_empty = bar + 2;
    uint64_t* s_full = bar + 3;
    uint64_t* p_full = bar + 4;
    uint64_t* dq_full = bar + 5;
    uint64_t* dq_empty = bar + 6;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);
    const uint32_t s_lse = ptx::smem_u32(sm + BwdSmem::kLse);
    const uint32_t s_del = ptx::smem_u32(sm + BwdSmem::kDelta);

    // grid (H, key blocks, B): the block scheduler walks x fastest, so every head's key block 0
    // (which sees the most query blocks under the causal mask) starts in the first wave
    const int n_kb = (S + BKV - 1) / BKV;
    const int kb = blockIdx.y;
    const int head = blockIdx.x, b = blockIdx.z;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int HD = H * D;
    const int row0 = b * S;
    const int i0 = kb;  // first query block that sees this key block (BQ == BKV)
    const int n_qb = (S + BQ - 1) / BQ;
    (void)n_kb;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tm_qkv);
        ptx::tma_prefetch(&tm_do);
        ptx::mbar_init(kv_full, 1);
        ptx::mbar_init(qo_full, 1);
        ptx::mbar_init(qo_empty, 1);
        ptx::mbar_init(s_full, 1);
        ptx::mbar_init(p_full, 4);
        ptx::mbar_init(dq_full, 1);
        ptx::mbar_init(dq_empty, 4);
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
            for (int i = i0; i < n_qb; ++i) {
                if (i > i0) ptx::mbar_wait(qo_empty, (i - i0 - 1) & 1);
                ptx::mbar_expect_tx(qo_full, 2 * kTile);
                for (int h2 = 0; h2 < 2; ++h2) {
                    ptx::tma_load_2d(sm + BwdSmem::kQ + h2 * (kTile / 2), &tm_qkv, qo_full, qcol + 64 * h2, row0 + i * BQ);
                    ptx::tma_load_2d(sm + BwdSmem::kO + h2 * (kTile / 2), &tm_do, qo_full, head * D + 64 * h2, row0 + i * BQ);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id_kk = ptx::idesc_bf16_f32(128, 128, 0, 0);  // A, B K-major
            constexpr uint32_t id_kn = ptx::idesc_bf16_f32(128, 128, 0, 1);  // B MN-major
            constexpr uint32_t id_nn = ptx::idesc_bf16_f32(128, 128, 1, 1);  // A, B MN-major
            const uint32_t sk = ptx::smem_u32(sm + BwdSmem::kK), sv = ptx::smem_u32(sm + BwdSmem::kV);
            const uint32_t sq = ptx::smem_u32(sm + BwdSmem::kQ), so = ptx::smem_u32(sm + BwdSmem::kO);
            const uint32_t sp = ptx::smem_u32(sm + BwdSmem::kP), sds = ptx::smem_u32(sm + BwdSmem::kS);
            ptx::mbar_wait(kv_full, 0);
            for (int i = i0; i < n_qb; ++i) {
                const int it = i - i0;
                // S^T_i right away (the tensor pipe runs it while dQ_{i-1} drains); dP^T_i into the
                // dQ_{i-1} columns once those are drained
                ptx::mbar_wait(qo_full, it & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    ptx::umma_f16(t_s, kmajor_desc(sk, kk), kmajor_desc(sq, kk), id_kk, kk != 0);
                if (it > 0) ptx::mbar_wait(dq_empty, (it - 1) & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    ptx::umma_f16(t_dp, kmajor_desc(sv, kk), kmajor_desc(so, kk), id_kk, kk != 0);
                ptx::umma_commit(s_full);
                ptx::mbar_wait(p_full, it & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < BQ / 16; ++kk) {
                    ptx::umma_f16(t_dv, kmajor_desc(sp, kk), mnmajor_desc(so, kk), id_kn, (it | kk) != 0);
                    ptx::umma_f16(t_dk, kmajor_desc(sds, kk), mnmajor_desc(sq, kk), id_kn, (it | kk) != 0);
                }
                ptx::umma_commit(qo_empty);
                // dQ_i into the dP^T columns (consumed once p_full fired)
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk)
                    ptx::umma_f16(t_dp, mnmajor_desc(sds, kk), mnmajor_desc(sk, kk), id_nn, kk != 0);
                ptx::umma_commit(dq_full);
            }
        }
    } else {
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;  // TMEM lane: key row (S^T, dP^T, dK, dV) or q row (dQ)
        const int key = kb * BKV + r;
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        const int tid = threadIdx.x - 64;
        const uint32_t sp_base = ptx::smem_u32(sm + BwdSmem::kP), sds_base = ptx::smem_u32(sm + BwdSmem::kS);
        const int64_t stat_base = (static_cast<int64_t>(b) * H + head) * S;
        // LSE / delta of the next query block are loaded one iteration ahead (their global-load
        // latency was exposed at the top of every iteration)
        float nxt_l = 0.f, nxt_d = 0.f;
        {
            const int q = i0 * BQ + tid;
            if (q < S) {
                nxt_l = lse[stat_base + q];
                nxt_d = delta[stat_base + q];
            }
        }
        for (int i = i0; i < n_qb; ++i) {
            const int it = i - i0;
            const int q0 = i * BQ;
            // double-buffered by iteration: a warp one iteration ahead never overwrites values a
            // slower warp is still reading (nobody gets two ahead past the barrier below)
            const uint32_t L = s_lse + (it & 1) * 512;
            const uint32_t Dl = s_del + (it & 1) * 512;
            ptx::st_shared_f32(L + 4 * tid, nxt_l);
            ptx::st_shared_f32(Dl + 4 * tid, nxt_d);
            if (i + 1 < n_qb) {
                const int q = q0 + BQ + tid;
                nxt_l = q < S ? lse[stat_base + q] : 0.f;
                nxt_d = q < S ? delta[stat_base + q] : 0.f;
            }
            named_bar_sync(1, 128);
            ptx::mbar_wait(s_full, it & 1);
            ptx::tc_fence_after();
            const bool mask = (i == i0) || (q0 + BQ > S) || (kb * BKV + BKV > S);
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t rs[32], rd[32];
                ptx::tmem_ld_32x32b_x32(t_s + lane_off + c * 32, rs);
                ptx::tmem_ld_32x32b_x32(t_dp + lane_off + c * 32, rd);
                ptx::tmem_ld_wait();
                uint32_t pw[16], dw[16];
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    float p[2], d[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int ql = c * 32 + j + e;
                        float pv = ptx::ex2_fast(__uint_as_float(rs[j + e]) * scale_log2 - ptx::ld_shared_f32(L + 4 * ql));
                        if (mask && (key > q0 + ql || q0 + ql >= S || key >= S)) pv = 0.f;
                        p[e] = pv;
                        d[e] = pv * (__uint_as_float(rd[j + e]) - ptx::ld_shared_f32(Dl + 4 * ql));
                    }
                    __nv_bfloat162 hp = __floats2bfloat162_rn(p[0], p[1]), hd = __floats2bfloat162_rn(d[0], d[1]);
                    pw[j / 2] = *reinterpret_cast<uint32_t*>(&hp);
                    dw[j / 2] = *reinterpret_cast<uint32_t*>(&hd);
                }
                // row r of the [2 q-blocks][128 keys][128 B] tiles; chunk c covers q 32c..32c+31
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int blk = c >> 1, ch = (c & 1) * 4 + u;
                    const uint32_t off = blk * (kTile / 2) + r * 128 + ((ch ^ (r & 7)) << 4);
                    ptx::st_shared_v4(sp_base + off, pw[4 * u], pw[4 * u + 1], pw[4 * u + 2], pw[4 * u + 3]);
                    ptx::st_shared_v4(sds_base + off, dw[4 * u], dw[4 * u + 1], dw[4 * u + 2], dw[4 * u + 3]);
                }
            }
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(p_full);
            // drain dQ_i (TMEM lane = q row) into the f32 accumulator
            ptx::mbar_wait(dq_full, it & 1);
            ptx::tc_fence_after();
            const int q = q0 + r;
            float* dst = dq_acc + static_cast<int64_t>(row0 + q) * HD + head * D;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t rq[32];
                ptx::tmem_ld_32x32b_x32(t_dp + lane_off + c * 32, rq);
                ptx::tmem_ld_wait();
                if (q < S) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        red_add_v4(dst + c * 32 + j, __uint_as_float(rq[j]) * scale, __uint_as_float(rq[j + 1]) * scale,
                                   __uint_as_float(rq[j + 2]) * scale, __uint_as_float(rq[j + 3]) * scale);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(dq_empty);
        }
        // dK (scaled) and dV for this thread's key row. tcgen05.ld is warp-collective
        // (.sync.aligned): every lane loads, only rows inside the sequence store.
        ptx::tc_fence_after();
        __nv_bfloat16* dkr = dqkv + static_cast<int64_t>(row0 + key) * 3 * HD + HD + head * D;
        __nv_bfloat16* dvr = dqkv + static_cast<int64_t>(row0 + key) * 3 * HD + 2 * HD + head * D;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t rk[32], rv[32];
            ptx::tmem_ld_32x32b_x32(t_dk + lane_off + c * 32, rk);
            ptx::tmem_ld_32x32b_x32(t_dv + lane_off + c * 32, rv);
            ptx::tmem_ld_wait();
            if (key >= S) continue;
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
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
                *reinterpret_cast<uint4*>(dkr + c * 32 + j) = ok;
                *reinterpret_cast<uint4*>(dvr + c * 32 + j) = ov;
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
    const CUtensorMap to = make_tma_2d(dout, HD, T, HD, 128, false);
    dim3 grid(heads, (seq + BKV - 1) / BKV, batch);
    if (heads > 1 && seq > BKV) count_variant(KV_ATTN_BWD_MULTI);
    const float scale = 1.f / sqrtf(static_cast<float>(head_dim));
    attn_bwd_tc_kernel<<<grid, 192, BwdSmem::kBytes, st>>>(tq, to, lse, delta, dq_acc,
                                                           static_cast<__nv_bfloat16*>(dqkv), seq, heads, scale,
                                                           scale * kLog2e);
}

}  // namespace bfpp
