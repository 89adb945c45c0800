// Causal multi-head attention forward/backward for head_dim 128 (flash-style,
// online softmax in the log2 domain, never materialising the T x T scores).
//
// Layouts (per micro-batch of B samples x S tokens, T = B*S rows):
//   qkv  [T][3h] bf16   Q at cols [0,h), K at [h,2h), V at [2h,3h); head j = cols j*128..
//   o    [T][h]  bf16
//   lse  [B*H][S] f32   log2-sum-exp of the scaled scores (saved for backward)
//   dqkv [T][3h] bf16   gradients, same layout as qkv
// Tensor-core work uses mma.sync m16n8k16 (bf16 -> f32) with ldmatrix from
// XOR-swizzled shared memory and cp.async double buffering.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdexcept>

#include "kernels.hpp"

namespace bfpp {
namespace {

constexpr int D = 128;  // head dim
constexpr float kLog2e = 1.4426950408889634f;

// [rows][128] bf16 tile, 16 chunks of 16 B per row, chunk XOR-swizzled by row&7.
__device__ __forceinline__ uint32_t swz(int row, int chunk) { return row * 256 + ((chunk ^ (row & 7)) << 4); }
// [rows][64] bf16 tile (8 chunks per row).
__device__ __forceinline__ uint32_t swz64(int row, int chunk) { return row * 128 + ((chunk ^ (row & 7)) << 4); }

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Cooperative async load of a [rows][128] bf16 tile (row stride ld elements) into swizzled smem.
template <int ROWS, int NT>
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* g, int64_t ld, int tid) {
#pragma unroll
    for (int i = tid; i < ROWS * 16; i += NT) {
        const int r = i >> 4, c = i & 15;
        cp_async16(sbase + swz(r, c), g + r * ld + c * 8);
    }
}

// ============================== forward ==========================================
constexpr int F_BR = 128, F_BC = 64, F_WARPS = 8;

__global__ void __launch_bounds__(F_WARPS * 32, 1)
    attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                    int S, int H, float scale_log2) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int qb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int h3 = 3 * H * D;
    const int64_t row0 = static_cast<int64_t>(b) * S;
    const __nv_bfloat16* Qg = qkv + (row0 + qb * F_BR) * h3 + head * D;
    const __nv_bfloat16* Kg = qkv + row0 * h3 + H * D + head * D;
    const __nv_bfloat16* Vg = qkv + row0 * h3 + 2 * H * D + head * D;
    const uint32_t sQ = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const uint32_t sK = sQ + F_BR * 256;
    const uint32_t sV = sK + 2 * F_BC * 256;

    const int q_hi = min(S, (qb + 1) * F_BR);  // exclusive
    const int n_kv = (q_hi + F_BC - 1) / F_BC;
    const int q_rows = min(F_BR, S - qb * F_BR);

    // Q (rows beyond S are never written back; load clamped rows)
    for (int i = tid; i < F_BR * 16; i += F_WARPS * 32) {
        const int r = i >> 4, c = i & 15;
        const int rr = r < q_rows ? r : 0;
        cp_async16(sQ + swz(r, c), Qg + static_cast<int64_t>(rr) * h3 + c * 8);
    }
    auto load_kv = [&](int j, int buf) {
        for (int i = tid; i < F_BC * 16; i += F_WARPS * 32) {
            const int r = i >> 4, c = i & 15;
            const int kr = min(j * F_BC + r, S - 1);
            cp_async16(sK + buf * F_BC * 256 + swz(r, c), Kg + static_cast<int64_t>(kr) * h3 + c * 8);
            cp_async16(sV + buf * F_BC * 256 + swz(r, c), Vg + static_cast<int64_t>(kr) * h3 + c * 8);
        }
    };
    load_kv(0, 0);
    cp_commit();

    const int g = lane >> 2, cq = lane & 3;
    const int wq0 = qb * F_BR + warp * 16;  // first query row of this warp
    float acc[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
    uint32_t qf[8][4];

    for (int j = 0; j < n_kv; ++j) {
        const int buf = j & 1;
        if (j + 1 < n_kv) load_kv(j + 1, buf ^ 1);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        if (j == 0) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int r = warp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
                ldsm_x4(sQ + swz(r, 2 * kk + (lane >> 4)), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
            }
        }
        const int k0 = j * F_BC;
        if (k0 <= wq0 + 15) {  // some key of this tile is visible to this warp
            const uint32_t kb = sK + buf * F_BC * 256, vb = sV + buf * F_BC * 256;
            float s[8][4];
#pragma unroll
            for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
                for (int np = 0; np < 4; ++np) {
                    uint32_t b0, b1, b2, b3;
                    const int r = np * 16 + (lane & 7) + 8 * (lane >> 4);
                    ldsm_x4(kb + swz(r, 2 * kk + ((lane >> 3) & 1)), b0, b1, b2, b3);
                    mma16816(s[2 * np], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
                    mma16816(s[2 * np + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
                }
            }
            const bool need_mask = k0 + F_BC - 1 > wq0 || k0 + F_BC > S;
            float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
            for (int n = 0; n < 8; ++n) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float v = s[n][e] * scale_log2;
                    if (need_mask) {
                        const int key = k0 + n * 8 + 2 * cq + (e & 1);
                        const int q = wq0 + g + 8 * (e >> 1);
                        if (key > q || key >= S) v = -INFINITY;
                    }
                    s[n][e] = v;
                    mx[e >> 1] = fmaxf(mx[e >> 1], v);
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffff, mx[i], 1));
                mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffff, mx[i], 2));
            }
            float alpha[2], rs[2] = {0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                alpha[i] = m_r[i] == -INFINITY ? 0.f : ex2(m_r[i] - mx[i]);
                m_r[i] = mx[i];
            }
            uint32_t pf[4][4];
#pragma unroll
            for (int n = 0; n < 8; ++n) {
                const float p0 = ex2(s[n][0] - mx[0]), p1 = ex2(s[n][1] - mx[0]);
                const float p2 = ex2(s[n][2] - mx[1]), p3 = ex2(s[n][3] - mx[1]);
                rs[0] += p0 + p1;
                rs[1] += p2 + p3;
                pf[n >> 1][(n & 1) * 2 + 0] = pack_bf16(p0, p1);
                pf[n >> 1][(n & 1) * 2 + 1] = pack_bf16(p2, p3);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) l_r[i] = l_r[i] * alpha[i] + rs[i];
#pragma unroll
            for (int n = 0; n < 16; ++n) {
                acc[n][0] *= alpha[0];
                acc[n][1] *= alpha[0];
                acc[n][2] *= alpha[1];
                acc[n][3] *= alpha[1];
            }
            // O += P V   (A = P: 16 x 64 keys; B[k=key][n=dim] = V via transposed ldmatrix)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
                for (int np = 0; np < 8; ++np) {
                    uint32_t b0, b1, b2, b3;
                    const int r = kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
                    ldsm_x4_t(vb + swz(r, 2 * np + (lane >> 4)), b0, b1, b2, b3);
                    mma16816(acc[2 * np], pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3], b0, b1);
                    mma16816(acc[2 * np + 1], pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3], b2, b3);
                }
            }
        }
        __syncthreads();
    }
    // finalize: quad-reduce the row sums, normalise, store O and LSE
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        l_r[i] += __shfl_xor_sync(0xffffffff, l_r[i], 1);
        l_r[i] += __shfl_xor_sync(0xffffffff, l_r[i], 2);
    }
    const int HD = H * D;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int q = wq0 + g + 8 * i;
        if (q >= S) continue;
        const float inv = 1.f / l_r[i];
        __nv_bfloat16* orow = o + (row0 + q) * HD + head * D;
#pragma unroll
        for (int n = 0; n < 16; ++n)
            *reinterpret_cast<uint32_t*>(orow + n * 8 + 2 * cq) = pack_bf16(acc[n][2 * i] * inv, acc[n][2 * i + 1] * inv);
        if (cq == 0) lse[(static_cast<int64_t>(b) * H + head) * S + q] = m_r[i] + log2f(l_r[i]);
    }
}

// ============================== backward =========================================
// D_i = sum_d dO[i,d] * O[i,d]; also zeroes the f32 dQ accumulator.
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                     float* __restrict__ delta, float* __restrict__ dq_acc, int S, int H, int T) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= T * H) return;
    const int row = warp / H, head = warp % H;
    const int64_t off = static_cast<int64_t>(row) * H * D + head * D + lane * 4;
    const uint2 a = *reinterpret_cast<const uint2*>(o + off);
    const uint2 c = *reinterpret_cast<const uint2*>(dout + off);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(c2[i]);
        s += x.x * y.x + x.y * y.y;
    }
#pragma unroll
    for (int k = 16; k; k >>= 1) s += __shfl_xor_sync(0xffffffff, s, k);
    *reinterpret_cast<float4*>(dq_acc + off) = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lane == 0) {
        const int b = row / S, q = row % S;
        delta[(static_cast<int64_t>(b) * H + head) * S + q] = s;
    }
}

constexpr int B_BC = 64, B_BR = 64, B_WARPS = 4;

__global__ void __launch_bounds__(B_WARPS * 32, 2)
    attn_bwd_kernel(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
                    const float* __restrict__ lse, const float* __restrict__ delta, float* __restrict__ dq_acc,
                    __nv_bfloat16* __restrict__ dqkv, int S, int H, float scale, float scale_log2) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int kb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, cq = lane & 3;
    const int h3 = 3 * H * D, HD = H * D;
    const int64_t row0 = static_cast<int64_t>(b) * S;
    const __nv_bfloat16* Qg = qkv + row0 * h3 + head * D;
    const __nv_bfloat16* Kg = qkv + row0 * h3 + HD + head * D;
    const __nv_bfloat16* Vg = qkv + row0 * h3 + 2 * HD + head * D;
    const __nv_bfloat16* dOg = dout + row0 * HD + head * D;
    const float* lse_g = lse + (static_cast<int64_t>(b) * H + head) * S;
    const float* del_g = delta + (static_cast<int64_t>(b) * H + head) * S;

    const uint32_t sK = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const uint32_t sV = sK + B_BC * 256;
    const uint32_t sQ = sV + B_BC * 256;         // 2 buffers
    const uint32_t sdO = sQ + 2 * B_BR * 256;    // 2 buffers
    const uint32_t sdS = sdO + 2 * B_BR * 256;   // [64 keys][64 q] bf16
    float* sL = reinterpret_cast<float*>(sm + (sdS - sK) + B_BC * 128);  // [2][64] lse
    float* sD = sL + 2 * B_BR;                                          // [2][64] delta

    const int k0 = kb * B_BC;
    const int k_rows = min(B_BC, S - k0);
    for (int i = tid; i < B_BC * 16; i += B_WARPS * 32) {
        const int r = i >> 4, c = i & 15;
        const int rr = r < k_rows ? r : 0;
        cp_async16(sK + swz(r, c), Kg + static_cast<int64_t>(k0 + rr) * h3 + c * 8);
        cp_async16(sV + swz(r, c), Vg + static_cast<int64_t>(k0 + rr) * h3 + c * 8);
    }
    const int i_begin = k0 / B_BR;
    const int i_end = (S + B_BR - 1) / B_BR;
    auto load_q = [&](int i, int buf) {
        for (int t = tid; t < B_BR * 16; t += B_WARPS * 32) {
            const int r = t >> 4, c = t & 15;
            const int q = min(i * B_BR + r, S - 1);
            cp_async16(sQ + buf * B_BR * 256 + swz(r, c), Qg + static_cast<int64_t>(q) * h3 + c * 8);
            cp_async16(sdO + buf * B_BR * 256 + swz(r, c), dOg + static_cast<int64_t>(q) * HD + c * 8);
        }
        for (int t = tid; t < B_BR; t += B_WARPS * 32) {
            const int q = i * B_BR + t;
            sL[buf * B_BR + t] = q < S ? lse_g[q] : 0.f;
            sD[buf * B_BR + t] = q < S ? del_g[q] : 0.f;
        }
    };
    load_q(i_begin, 0);
    cp_commit();

    float dk[16][4], dv[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[n][e] = dv[n][e] = 0.f;
    const int wk0 = k0 + warp * 16;  // first key of this warp

    for (int i = i_begin; i < i_end; ++i) {
        const int buf = (i - i_begin) & 1;
        if (i + 1 < i_end) load_q(i + 1, buf ^ 1);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const uint32_t qb_s = sQ + buf * B_BR * 256, ob_s = sdO + buf * B_BR * 256;
        const float* L = sL + buf * B_BR;
        const float* Dl = sD + buf * B_BR;
        const int q0 = i * B_BR;
        // S^T (16 keys x 64 q) and dP^T = V dO^T
        float st[8][4], dp[8][4];
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) st[n][e] = dp[n][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t a[4], v[4];
            const int ar = warp * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
            ldsm_x4(sK + swz(ar, 2 * kk + (lane >> 4)), a[0], a[1], a[2], a[3]);
            ldsm_x4(sV + swz(ar, 2 * kk + (lane >> 4)), v[0], v[1], v[2], v[3]);
#pragma unroll
            for (int np = 0; np < 4; ++np) {
                uint32_t b0, b1, b2, b3;
                const int r = np * 16 + (lane & 7) + 8 * (lane >> 4);
                ldsm_x4(qb_s + swz(r, 2 * kk + ((lane >> 3) & 1)), b0, b1, b2, b3);
                mma16816(st[2 * np], a[0], a[1], a[2], a[3], b0, b1);
                mma16816(st[2 * np + 1], a[0], a[1], a[2], a[3], b2, b3);
                ldsm_x4(ob_s + swz(r, 2 * kk + ((lane >> 3) & 1)), b0, b1, b2, b3);
                mma16816(dp[2 * np], v[0], v[1], v[2], v[3], b0, b1);
                mma16816(dp[2 * np + 1], v[0], v[1], v[2], v[3], b2, b3);
            }
        }
        // P^T = exp2(scale_log2 * S^T - lse[q]) masked; dS^T = P^T (dP^T - delta[q])
        uint32_t pa[4][4], da[4][4];
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            float p[4], d[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int ql = n * 8 + 2 * cq + (e & 1);
                const int q = q0 + ql;
                const int key = wk0 + g + 8 * (e >> 1);
                float pv = ex2(st[n][e] * scale_log2 - L[ql]);
                if (key > q || q >= S || key >= S) pv = 0.f;
                p[e] = pv;
                d[e] = pv * (dp[n][e] - Dl[ql]);
            }
            pa[n >> 1][(n & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
            pa[n >> 1][(n & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
            da[n >> 1][(n & 1) * 2 + 0] = pack_bf16(d[0], d[1]);
            da[n >> 1][(n & 1) * 2 + 1] = pack_bf16(d[2], d[3]);
        }
        // stash dS^T (bf16) for the dQ product: rows = keys, cols = q
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            const uint32_t* src = &da[n >> 1][(n & 1) * 2];
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) {
                const int r = warp * 16 + g + 8 * hr;
                const int col = n * 8 + 2 * cq;  // element column
                const uint32_t addr = sdS + swz64(r, col >> 3) + (col & 7) * 2;
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(src[hr]));
            }
        }
        // dV += P^T dO ; dK += dS^T Q   (B[k=q][n=dim] via transposed ldmatrix)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int np = 0; np < 8; ++np) {
                uint32_t b0, b1, b2, b3;
                const int r = kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
                ldsm_x4_t(ob_s + swz(r, 2 * np + (lane >> 4)), b0, b1, b2, b3);
                mma16816(dv[2 * np], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b0, b1);
                mma16816(dv[2 * np + 1], pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3], b2, b3);
                ldsm_x4_t(qb_s + swz(r, 2 * np + (lane >> 4)), b0, b1, b2, b3);
                mma16816(dk[2 * np], da[kk][0], da[kk][1], da[kk][2], da[kk][3], b0, b1);
                mma16816(dk[2 * np + 1], da[kk][0], da[kk][1], da[kk][2], da[kk][3], b2, b3);
            }
        }
        __syncthreads();
        // dQ[q rows of this warp] += dS K   (A[m=q][k=key] = dS^T[key][q] via transposed ldmatrix)
        {
            uint32_t af[4][4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                // matrices: (keys kk*16+0..7, q w*16+0..7), (keys +0..7, q +8..15), (keys +8..15, q 0..7), (keys +8.., q +8..)
                const int key = kk * 16 + (lane & 7) + 8 * (lane >> 4);
                const int qc = warp * 16 + 8 * ((lane >> 3) & 1);
                uint32_t r0, r1, r2, r3;
                ldsm_x4_t(sdS + swz64(key, qc >> 3), r0, r1, r2, r3);
                // a0: (q g, keys 2c..) = m(keys 0-7, q 0-7)^T ; a1: (q g+8, keys 2c) = m(keys 0-7, q 8-15)^T
                // a2: (q g, keys 8+2c) = m(keys 8-15, q 0-7)^T ; a3: m(keys 8-15, q 8-15)^T
                af[kk][0] = r0;
                af[kk][1] = r1;
                af[kk][2] = r2;
                af[kk][3] = r3;
            }
            const int qa = q0 + warp * 16 + g;
#pragma unroll
            for (int np = 0; np < 8; ++np) {
                float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    uint32_t b0, b1, b2, b3;
                    const int r = kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
                    ldsm_x4_t(sK + swz(r, 2 * np + (lane >> 4)), b0, b1, b2, b3);
                    mma16816(c0, af[kk][0], af[kk][1], af[kk][2], af[kk][3], b0, b1);
                    mma16816(c1, af[kk][0], af[kk][1], af[kk][2], af[kk][3], b2, b3);
                }
#pragma unroll
                for (int hr = 0; hr < 2; ++hr) {
                    const int q = qa + 8 * hr;
                    if (q >= S) continue;
                    float* dst = dq_acc + (row0 + q) * HD + head * D + np * 16 + 2 * cq;
                    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dst), "f"(c0[2 * hr] * scale),
                                 "f"(c0[2 * hr + 1] * scale)
                                 : "memory");
                    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dst + 8), "f"(c1[2 * hr] * scale),
                                 "f"(c1[2 * hr + 1] * scale)
                                 : "memory");
                }
            }
        }
        __syncthreads();
    }
    // write dK (scaled) and dV for this warp's 16 keys
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int key = wk0 + g + 8 * hr;
        if (key >= S) continue;
        __nv_bfloat16* dkr = dqkv + (row0 + key) * h3 + HD + head * D;
        __nv_bfloat16* dvr = dqkv + (row0 + key) * h3 + 2 * HD + head * D;
#pragma unroll
        for (int n = 0; n < 16; ++n) {
            *reinterpret_cast<uint32_t*>(dkr + n * 8 + 2 * cq) =
                pack_bf16(dk[n][2 * hr] * scale, dk[n][2 * hr + 1] * scale);
            *reinterpret_cast<uint32_t*>(dvr + n * 8 + 2 * cq) = pack_bf16(dv[n][2 * hr], dv[n][2 * hr + 1]);
        }
    }
}

__global__ void attn_dq_convert_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int T,
                                       int HD) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i >= static_cast<int64_t>(T) * HD) return;
    const int64_t row = i / HD, col = i % HD;
    const float4 v = *reinterpret_cast<const float4*>(dq_acc + i);
    uint2 o;
    o.x = pack_bf16(v.x, v.y);
    o.y = pack_bf16(v.z, v.w);
    *reinterpret_cast<uint2*>(dqkv + row * 3 * HD + col) = o;
}

constexpr int kFwdSmem = (F_BR + 4 * F_BC) * 256;
constexpr int kBwdSmem = (2 * B_BC + 4 * B_BR) * 256 + B_BC * 128 + 4 * B_BR * 4;

}  // namespace

void attention_fwd_mma(const void* qkv, void* o, float* lse, int batch, int seq, int heads, int head_dim,
                       cudaStream_t st) {
    if (head_dim != D) throw std::runtime_error("attention: head_dim must be 128");
    static bool cfg = false;
    if (!cfg) {
        cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
        cfg = true;
    }
    dim3 grid((seq + F_BR - 1) / F_BR, heads, batch);
    const float scale_log2 = kLog2e / sqrtf(static_cast<float>(head_dim));
    attn_fwd_kernel<<<grid, F_WARPS * 32, kFwdSmem, st>>>(static_cast<const __nv_bfloat16*>(qkv),
                                                          static_cast<__nv_bfloat16*>(o), lse, seq, heads,
                                                          scale_log2);
}

// forward entry point: the tcgen05/TMEM kernel (attention_tc.cu)
void attention_fwd(const void* qkv, void* o, float* lse, int batch, int seq, int heads, int head_dim,
                   cudaStream_t st) {
    attention_fwd_tc(qkv, o, lse, batch, seq, heads, head_dim, st);
}

void attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse, float* delta, float* dq_acc,
                   void* dqkv, int batch, int seq, int heads, int head_dim, cudaStream_t st) {
    if (head_dim != D) throw std::runtime_error("attention: head_dim must be 128");
    const int T = batch * seq;
    const int warps = T * heads;
    attn_bwd_prep_kernel<<<(warps + 7) / 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                                          static_cast<const __nv_bfloat16*>(dout), delta, dq_acc, seq,
                                                          heads, T);
    attention_bwd_tc(qkv, dout, lse, delta, dq_acc, dqkv, batch, seq, heads, head_dim, st);
    const int64_t n4 = static_cast<int64_t>(T) * heads * head_dim / 4;
    attn_dq_convert_kernel<<<static_cast<unsigned>((n4 + 255) / 256), 256, 0, st>>>(
        dq_acc, static_cast<__nv_bfloat16*>(dqkv), T, heads * head_dim);
}

}  // namespace bfpp
