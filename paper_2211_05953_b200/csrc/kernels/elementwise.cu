// HBM-bound kernels of the stage executor: token/position embedding (fwd +
// scatter-add bwd), fused softmax cross-entropy (loss + dlogits in place),
// sharded Adam with bf16 emission, Philox normal init, reductions.
// All use 128-bit vector accesses and grid sizes in multiples of the SM count.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <cstdlib>
#include <stdexcept>

#include "kernels.hpp"

namespace bfpp {
namespace {

int sm_count() {
    static int n = 0;
    if (!n) {
        int d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    }
    return n;
}

__device__ __forceinline__ void bf8_to_f(const uint4& raw, float (&v)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        float2 f = __bfloat1622float2(h[u]);
        v[2 * u] = f.x;
        v[2 * u + 1] = f.y;
    }
}
__device__ __forceinline__ uint4 f_to_bf8(const float (&v)[8]) {
    uint4 o;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int u = 0; u < 4; ++u) h[u] = __floats2bfloat162_rn(v[2 * u], v[2 * u + 1]);
    return o;
}

// x[t] = wte[tok[t]] + wpe[t % S]; one warp per row.
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ wte,
                                 const __nv_bfloat16* __restrict__ wpe, __nv_bfloat16* __restrict__ x, int T, int S,
                                 int h) {
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (row >= T) return;
    const int id = tok[row], pos = row % S;
    for (int c = lane * 8; c < h; c += 256) {
        float a[8], b[8];
        bf8_to_f(*reinterpret_cast<const uint4*>(wte + static_cast<int64_t>(id) * h + c), a);
        bf8_to_f(*reinterpret_cast<const uint4*>(wpe + static_cast<int64_t>(pos) * h + c), b);
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += b[u];
        *reinterpret_cast<uint4*>(x + static_cast<int64_t>(row) * h + c) = f_to_bf8(a);
    }
}

// Embedding backward without atomics (bit-reproducible): the T (token, row) pairs are radix-sorted
// by token (stable, so equal tokens keep row order), then one warp per distinct token adds that
// token's rows of dx in row order to dwte[token], and one warp per position adds the s_mb samples of
// that position to dwpe[pos]. dwte / dwpe hold the running sums (the executor zeroes them at the
// start of a reduction unit).
__global__ void iota_kernel(int32_t* __restrict__ v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

__global__ void embed_wte_bwd_kernel(const int32_t* __restrict__ sk, const int32_t* __restrict__ sv,
                                     const __nv_bfloat16* __restrict__ dx, float* __restrict__ dwte, int T, int h) {
    const int i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (i >= T || (i > 0 && sk[i] == sk[i - 1])) return;  // segment heads only
    const int id = sk[i];
    int end = i + 1;
    while (end < T && sk[end] == id) ++end;
    for (int c = lane * 8; c < h; c += 256) {
        float* dst = dwte + static_cast<int64_t>(id) * h + c;
        float acc[8];
        const float4 a0 = *reinterpret_cast<const float4*>(dst), a1 = *reinterpret_cast<const float4*>(dst + 4);
        acc[0] = a0.x, acc[1] = a0.y, acc[2] = a0.z, acc[3] = a0.w, acc[4] = a1.x, acc[5] = a1.y, acc[6] = a1.z,
        acc[7] = a1.w;
        for (int k = i; k < end; ++k) {
            float a[8];
            bf8_to_f(*reinterpret_cast<const uint4*>(dx + static_cast<int64_t>(sv[k]) * h + c), a);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += a[u];
        }
        *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
}

__global__ void embed_wpe_bwd_kernel(const __nv_bfloat16* __restrict__ dx, float* __restrict__ dwpe, int T, int S,
                                     int h) {
    const int pos = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (pos >= S) return;
    for (int c = lane * 8; c < h; c += 256) {
        float* dst = dwpe + static_cast<int64_t>(pos) * h + c;
        float acc[8];
        const float4 a0 = *reinterpret_cast<const float4*>(dst), a1 = *reinterpret_cast<const float4*>(dst + 4);
        acc[0] = a0.x, acc[1] = a0.y, acc[2] = a0.z, acc[3] = a0.w, acc[4] = a1.x, acc[5] = a1.y, acc[6] = a1.z,
        acc[7] = a1.w;
        for (int row = pos; row < T; row += S) {
            float a[8];
            bf8_to_f(*reinterpret_cast<const uint4*>(dx + static_cast<int64_t>(row) * h + c), a);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += a[u];
        }
        *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
}

// One 256-thread block per row: online max/sum-exp, then dlogits = (softmax - onehot) * gscale in place.
__global__ void __launch_bounds__(256) xent_kernel(__nv_bfloat16* __restrict__ logits, int64_t ld,
                                                   const int32_t* __restrict__ labels, float* __restrict__ row_loss,
                                                   int V, float gscale) {
    const int row = blockIdx.x;
    __nv_bfloat16* lr = logits + static_cast<int64_t>(row) * ld;
    float m = -INFINITY, s = 0.f;
    for (int c = threadIdx.x * 8; c < V; c += 256 * 8) {
        float v[8];
        bf8_to_f(*reinterpret_cast<const uint4*>(lr + c), v);
        float mx = v[0];
#pragma unroll
        for (int u = 1; u < 8; ++u) mx = fmaxf(mx, v[u]);
        const float nm = fmaxf(m, mx);
        float acc = s * __expf(m - nm);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __expf(v[u] - nm);
        m = nm;
        s = acc;
    }
#pragma unroll
    for (int k = 16; k; k >>= 1) {
        const float om = __shfl_xor_sync(0xffffffff, m, k), os = __shfl_xor_sync(0xffffffff, s, k);
        const float nm = fmaxf(m, om);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
        m = nm;
    }
    __shared__ float sm_m[8], sm_s[8];
    if ((threadIdx.x & 31) == 0) sm_m[threadIdx.x >> 5] = m, sm_s[threadIdx.x >> 5] = s;
    __syncthreads();
    float M = sm_m[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) M = fmaxf(M, sm_m[i]);
    float Ssum = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) Ssum += sm_s[i] * __expf(sm_m[i] - M);
    const float lse = M + __logf(Ssum);
    const int label = labels[row];
    if (threadIdx.x == 0) row_loss[row] = lse - __bfloat162float(lr[label]);
    __syncthreads();  // the label logit is read before it is overwritten
    const float inv = 1.f / Ssum;
    for (int c = threadIdx.x * 8; c < V; c += 256 * 8) {
        float v[8];
        bf8_to_f(*reinterpret_cast<const uint4*>(lr + c), v);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (__expf(v[u] - M) * inv - (c + u == label ? 1.f : 0.f)) * gscale;
        *reinterpret_cast<uint4*>(lr + c) = f_to_bf8(v);
    }
}

// p, m, v f32 shards; g f32 gradient (zeroed after use if zero_grad); w16 bf16 copy of p.
// Launched with one 256-thread block per SM so it co-resides with the compute stream's
// GEMM CTAs; each thread keeps ILP float4 groups of all four arrays in flight.
// One float4 of parameters per thread, one contiguous 1024-parameter chunk per 256-thread block,
// the grid covering the tensor (measured on B200: 5.4 TB/s, vs 3.3 TB/s for 4-way ILP and
// 4.5 TB/s for a grid-stride layout, scripts/adam_variants.cu). Blocks are short-lived and light
// (~32 registers, no shared memory), so up to four fit on an SM beside a resident GEMM CTA
// (96 regs x 320 threads) and retire within microseconds: the block scheduler keeps placing the
// high-priority compute stream's CTAs while Adam on the low-priority DP stream streams HBM under
// the tensor-core work.

// Optimizer streams: L1 bypass + an L2 evict-first policy (measured 6.1 TB/s for Adam alone vs
// 5.4 TB/s with .cs hints and 5.6 TB/s with default caching; scripts/overlap_bench.py).
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float4 ld4_stream(const float4* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st4_stream(float4* p, float4 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void st2_stream(uint2* p, uint2 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u32 [%0], {%1,%2}, %3;"
                 :: "l"(p), "r"(v.x), "r"(v.y), "l"(pol) : "memory");
}

// 256-thread blocks: two fit beside a persistent GEMM CTA. (512-thread blocks, which cannot
// co-reside with an attention-backward CTA, measured: GEMMs 1030 vs 930 TF/s in-step, but the
// optimizer dropped to 2.3 TB/s and its tail made the N = 1 step 7 % longer.)
constexpr int kAdamThreads = 256;
__global__ void __launch_bounds__(kAdamThreads) adam_kernel(float* __restrict__ p, float* __restrict__ m,
                                                            float* __restrict__ v, float* __restrict__ g,
                                                            __nv_bfloat16* __restrict__ w16, int64_t n, float lr,
                                                            float b1, float b2, float eps, float wd, float bc1,
                                                            float bc2, int zero_grad) {
    const int64_t n4 = n / 4;
    const uint64_t pol = evict_first_policy();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kAdamThreads + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * kAdamThreads) {
        float4 P = ld4_stream(reinterpret_cast<const float4*>(p) + i, pol);
        float4 M = ld4_stream(reinterpret_cast<const float4*>(m) + i, pol);
        float4 Vv = ld4_stream(reinterpret_cast<const float4*>(v) + i, pol);
        const float4 G = ld4_stream(reinterpret_cast<const float4*>(g) + i, pol);
        float* pp = &P.x;
        float* mm = &M.x;
        float* vv = &Vv.x;
        const float* gg = &G.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            mm[k] = b1 * mm[k] + (1.f - b1) * gg[k];
            vv[k] = b2 * vv[k] + (1.f - b2) * gg[k] * gg[k];
            // bc1/bc2 are the reciprocal bias corrections; approximate division (2 ulp) keeps the
            // instruction count low for the SMs shared with GEMMs (GEMM 850 -> 947 TF/s co-running)
            pp[k] -= lr * (__fdividef(mm[k] * bc1, sqrtf(vv[k] * bc2) + eps) + wd * pp[k]);
        }
        st4_stream(reinterpret_cast<float4*>(p) + i, P, pol);
        st4_stream(reinterpret_cast<float4*>(m) + i, M, pol);
        st4_stream(reinterpret_cast<float4*>(v) + i, Vv, pol);
        if (zero_grad) st4_stream(reinterpret_cast<float4*>(g) + i, make_float4(0.f, 0.f, 0.f, 0.f), pol);
        __nv_bfloat162 lo = __floats2bfloat162_rn(P.x, P.y), hi = __floats2bfloat162_rn(P.z, P.w);
        uint2 o;
        o.x = *reinterpret_cast<uint32_t*>(&lo);
        o.y = *reinterpret_cast<uint32_t*>(&hi);
        st2_stream(reinterpret_cast<uint2*>(w16) + i, o, pol);
    }
    // scalar tail (n % 4 elements) on the last block
    const int64_t t = n4 * 4 + threadIdx.x;
    if (blockIdx.x == gridDim.x - 1 && t < n) {
        m[t] = b1 * m[t] + (1.f - b1) * g[t];
        v[t] = b2 * v[t] + (1.f - b2) * g[t] * g[t];
        p[t] -= lr * ((m[t] * bc1) / (sqrtf(v[t] * bc2) + eps) + wd * p[t]);
        if (zero_grad) g[t] = 0.f;
        w16[t] = __float2bfloat16_rn(p[t]);
    }
}

// ---- row-wise Adam over an embedding table [rows][h] (h % 4 == 0), same math as adam_kernel ----
// The next step's token rows are updated first (list pass, before the embedding lookup) and every
// other row afterwards (masked pass, off the critical path); each row is updated exactly once.
__device__ __forceinline__ void adam_group(float* p, float* m, float* v, const float* g, __nv_bfloat16* w16,
                                           int64_t i, float lr, float b1, float b2, float eps, float wd, float bc1,
                                           float bc2, uint64_t pol) {
    float4 P = ld4_stream(reinterpret_cast<const float4*>(p) + i, pol);
    float4 M = ld4_stream(reinterpret_cast<const float4*>(m) + i, pol);
    float4 Vv = ld4_stream(reinterpret_cast<const float4*>(v) + i, pol);
    const float4 G = ld4_stream(reinterpret_cast<const float4*>(g) + i, pol);
    float* pp = &P.x;
    float* mm = &M.x;
    float* vv = &Vv.x;
    const float* gg = &G.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        mm[k] = b1 * mm[k] + (1.f - b1) * gg[k];
        vv[k] = b2 * vv[k] + (1.f - b2) * gg[k] * gg[k];
        pp[k] -= lr * (__fdividef(mm[k] * bc1, sqrtf(vv[k] * bc2) + eps) + wd * pp[k]);
    }
    st4_stream(reinterpret_cast<float4*>(p) + i, P, pol);
    st4_stream(reinterpret_cast<float4*>(m) + i, M, pol);
    st4_stream(reinterpret_cast<float4*>(v) + i, Vv, pol);
    __nv_bfloat162 lo = __floats2bfloat162_rn(P.x, P.y), hi = __floats2bfloat162_rn(P.z, P.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&lo);
    o.y = *reinterpret_cast<uint32_t*>(&hi);
    st2_stream(reinterpret_cast<uint2*>(w16) + i, o, pol);
}

// mark[tok] = 1 for every token; the first marker of a row appends it to list (order irrelevant:
// rows are independent)
__global__ void mark_rows_kernel(const int32_t* __restrict__ tok, int n, int32_t* __restrict__ mark,
                                 int32_t* __restrict__ list, int32_t* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = tok[i];
    if (atomicExch(&mark[r], 1) == 0) list[atomicAdd(count, 1)] = r;
}

__global__ void __launch_bounds__(256) adam_rows_list_kernel(float* p, float* m, float* v, const float* g,
                                                             __nv_bfloat16* w16, const int32_t* __restrict__ list,
                                                             const int32_t* __restrict__ count, int max_rows, int h4,
                                                             float lr, float b1, float b2, float eps, float wd,
                                                             float bc1, float bc2) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int li = static_cast<int>(idx / h4);
    if (li >= max_rows || li >= *count) return;
    const int64_t i = static_cast<int64_t>(list[li]) * h4 + idx % h4;
    adam_group(p, m, v, g, w16, i, lr, b1, b2, eps, wd, bc1, bc2, evict_first_policy());
}

__global__ void __launch_bounds__(256) adam_rows_unmarked_kernel(float* p, float* m, float* v, const float* g,
                                                                 __nv_bfloat16* w16, const int32_t* __restrict__ mark,
                                                                 int64_t rows, int h4, float lr, float b1, float b2,
                                                                 float eps, float wd, float bc1, float bc2) {
    // one float4 per thread and short-lived blocks, like adam_kernel (it runs beside the GEMMs)
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < rows * h4 && !mark[i / h4]) adam_group(p, m, v, g, w16, i, lr, b1, b2, eps, wd, bc1, bc2, evict_first_policy());
}

__global__ void init_normal_kernel(float* __restrict__ p, __nv_bfloat16* __restrict__ w16, int64_t n, float mean,
                                   float std, uint64_t seed, uint64_t offset) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * 4;
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
        curandStatePhilox4_32_10_t st;
        curand_init(seed, (offset + i) / 4, 0, &st);
        const float4 r = curand_normal4(&st);
        const float vals[4] = {mean + std * r.x, mean + std * r.y, mean + std * r.z, mean + std * r.w};
        for (int u = 0; u < 4 && i + u < n; ++u) {
            if (p) p[i + u] = vals[u];
            if (w16) w16[i + u] = __float2bfloat16_rn(vals[u]);
        }
    }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = __float2bfloat16_rn(src[i]);
}

__global__ void sum_kernel(const float* __restrict__ x, int64_t n, float scale, float* __restrict__ out,
                           int accumulate) {
    float s = 0.f;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
#pragma unroll
    for (int k = 16; k; k >>= 1) s += __shfl_xor_sync(0xffffffff, s, k);
    __shared__ float part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int i = 0; i < static_cast<int>(blockDim.x / 32); ++i) t += part[i];
        *out = (accumulate ? *out : 0.f) + t * scale;
    }
}

}  // namespace

void embed_fwd(const int32_t* tok, const void* wte, const void* wpe, void* x, int T, int S, int h, cudaStream_t st) {
    if (h % 8) throw std::runtime_error("embedding: hidden size must be a multiple of 8");
    embed_fwd_kernel<<<(T + 7) / 8, 256, 0, st>>>(tok, static_cast<const __nv_bfloat16*>(wte),
                                                  static_cast<const __nv_bfloat16*>(wpe),
                                                  static_cast<__nv_bfloat16*>(x), T, S, h);
}

void embed_bwd(const int32_t* tok, const void* dx, float* dwte, float* dwpe, int T, int S, int h, cudaStream_t st) {
    if (h % 8) throw std::runtime_error("embed_bwd: hidden size must be a multiple of 8");
    // per-device workspace: row ids, sorted keys / values, radix-sort temporary storage
    static thread_local void* ws[64] = {};
    static thread_local size_t ws_bytes[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, tok, static_cast<int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), T, 0, 32, st);
    const size_t ids = (static_cast<size_t>(T) * 4 + 255) / 256 * 256;
    const size_t need = 3 * ids + tmp;
    if (need > ws_bytes[dev]) {
        if (ws[dev]) cudaFree(ws[dev]);
        if (cudaMalloc(&ws[dev], need) != cudaSuccess) throw std::runtime_error("embed_bwd: workspace allocation failed");
        ws_bytes[dev] = need;
    }
    auto* base = static_cast<uint8_t*>(ws[dev]);
    auto* rows = reinterpret_cast<int32_t*>(base);
    auto* sk = reinterpret_cast<int32_t*>(base + ids);
    auto* sv = reinterpret_cast<int32_t*>(base + 2 * ids);
    iota_kernel<<<(T + 255) / 256, 256, 0, st>>>(rows, T);
    if (cub::DeviceRadixSort::SortPairs(base + 3 * ids, tmp, tok, sk, rows, sv, T, 0, 32, st) != cudaSuccess)
        throw std::runtime_error("embed_bwd: radix sort failed");
    const auto* d = static_cast<const __nv_bfloat16*>(dx);
    embed_wte_bwd_kernel<<<(T + 7) / 8, 256, 0, st>>>(sk, sv, d, dwte, T, h);
    embed_wpe_bwd_kernel<<<(S + 7) / 8, 256, 0, st>>>(d, dwpe, T, S, h);
}

void softmax_xent(void* logits, int64_t ld, const int32_t* labels, float* row_loss, int T, int V, float grad_scale,
                  cudaStream_t st) {
    if (V % 8 || ld % 8) throw std::runtime_error("xent: vocab and ld must be multiples of 8");
    xent_kernel<<<T, 256, 0, st>>>(static_cast<__nv_bfloat16*>(logits), ld, labels, row_loss, V, grad_scale);
}

void adam_update(float* p, float* m, float* v, float* g, void* w16, int64_t n, float lr, float b1, float b2,
                 float eps, float wd, int step, int zero_grad, cudaStream_t st) {
    // the vector kernel multiplies by the reciprocals of the bias corrections
    const float bc1 = 1.f / (1.f - powf(b1, static_cast<float>(step)));
    const float bc2 = 1.f / (1.f - powf(b2, static_cast<float>(step)));
    static const bool once = [] {
        // max shared-memory carveout: an SM running optimizer blocks stays configurable for a GEMM CTA
        cudaFuncSetAttribute(adam_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        return true;
    }();
    (void)once;
    static const int64_t grid_cap = [] {  // experiment knob: grid-stride over at most this many blocks
        const char* e = getenv("BFPP_ADAM_GRID");
        return e ? static_cast<int64_t>(atoll(e)) : int64_t{0};
    }();
    int64_t blocks = (n / 4 + kAdamThreads - 1) / kAdamThreads;
    if (grid_cap > 0 && blocks > grid_cap) blocks = grid_cap;
    adam_kernel<<<static_cast<unsigned>(blocks > 0 ? blocks : 1), kAdamThreads, 0, st>>>(
        p, m, v, g, static_cast<__nv_bfloat16*>(w16), n, lr, b1, b2, eps, wd, bc1, bc2, zero_grad);
}

void mark_rows(const int32_t* tok, int n, int32_t* mark, int32_t* list, int32_t* count, int64_t rows,
               cudaStream_t st) {
    cudaMemsetAsync(mark, 0, static_cast<size_t>(rows) * 4, st);
    cudaMemsetAsync(count, 0, 4, st);
    mark_rows_kernel<<<(n + 255) / 256, 256, 0, st>>>(tok, n, mark, list, count);
}

void adam_rows(float* p, float* m, float* v, const float* g, void* w16, int64_t rows, int h, const int32_t* mark,
               const int32_t* list, const int32_t* count, int max_rows, int listed, float lr, float b1, float b2,
               float eps, float wd, int step, cudaStream_t st) {
    if (h % 4) throw std::runtime_error("adam_rows: row width must be a multiple of 4");
    const float bc1 = 1.f / (1.f - powf(b1, static_cast<float>(step)));
    const float bc2 = 1.f / (1.f - powf(b2, static_cast<float>(step)));
    const int h4 = h / 4;
    auto* w = static_cast<__nv_bfloat16*>(w16);
    if (listed) {
        const int64_t n = static_cast<int64_t>(max_rows) * h4;
        adam_rows_list_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
            p, m, v, g, w, list, count, max_rows, h4, lr, b1, b2, eps, wd, bc1, bc2);
    } else {
        const int64_t n = rows * h4;
        adam_rows_unmarked_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(p, m, v, g, w, mark, rows, h4,
                                                                                        lr, b1, b2, eps, wd, bc1, bc2);
    }
}

void init_normal(float* p, void* w16, int64_t n, float mean, float std, uint64_t seed, uint64_t offset,
                 cudaStream_t st) {
    const int64_t want = (n / 4 + 255) / 256;
    const int blocks = static_cast<int>(want < 8 * sm_count() ? (want > 0 ? want : 1) : 8 * sm_count());
    init_normal_kernel<<<blocks, 256, 0, st>>>(p, static_cast<__nv_bfloat16*>(w16), n, mean, std, seed, offset);
}

void f32_to_bf16(const float* src, void* dst, int64_t n, cudaStream_t st) {
    const int64_t want = (n + 255) / 256;
    const int blocks = static_cast<int>(want < 8 * sm_count() ? (want > 0 ? want : 1) : 8 * sm_count());
    f32_to_bf16_kernel<<<blocks, 256, 0, st>>>(src, static_cast<__nv_bfloat16*>(dst), n);
}

void sum_f32(const float* x, int64_t n, float scale, float* out, int accumulate, cudaStream_t st) {
    sum_kernel<<<1, 1024, 0, st>>>(x, n, scale, out, accumulate);
}

}  // namespace bfpp
