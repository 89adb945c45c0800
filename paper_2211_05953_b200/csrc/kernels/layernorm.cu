// LayerNorm forward/backward (HBM-bound). One 128-thread block per row (a
// block-stride loop over rows in the backward), 128-bit vector loads, f32
// statistics, warp-shuffle + shared-memory reductions.
//   fwd: y = (x - mean) * rstd * gamma + beta       (bf16 in/out; mean/rstd f32 saved)
//   bwd: dx = rstd * (g - mean(g) - xhat * mean(g * xhat)) [+ dres],  g = dy * gamma
//        dgamma += sum_rows dy * xhat, dbeta += sum_rows dy   (f32, accumulated across calls)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdexcept>

#include "kernels.hpp"

namespace bfpp {
namespace {

constexpr int NT = 128;

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
    uint4 raw = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        float2 f = __bfloat1622float2(h[u]);
        v[2 * u] = f.x;
        v[2 * u + 1] = f.y;
    }
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&v)[8]) {
    uint4 o;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int u = 0; u < 4; ++u) h[u] = __floats2bfloat162_rn(v[2 * u], v[2 * u + 1]);
    *reinterpret_cast<uint4*>(p) = o;
}
__device__ __forceinline__ void load8f(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}

// Sum of two values over the 128-thread block.
__device__ __forceinline__ float2 block_sum2(float a, float b, float2* red) {
#pragma unroll
    for (int k = 16; k; k >>= 1) {
        a += __shfl_xor_sync(0xffffffff, a, k);
        b += __shfl_xor_sync(0xffffffff, b, k);
    }
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = make_float2(a, b);
    __syncthreads();
    float2 s = red[0];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i) s.x += red[i].x, s.y += red[i].y;
    return s;
}

template <int V>  // 8-element vectors per thread; covers widths up to 1024 * V
__global__ void __launch_bounds__(NT) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                    const __nv_bfloat16* __restrict__ gamma,
                                                    const __nv_bfloat16* __restrict__ beta, __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
                                                    float* __restrict__ rstd_out, int width, float eps) {
    __shared__ float2 red[NT / 32];
    const int64_t off = static_cast<int64_t>(blockIdx.x) * width;
    float v[V][8];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int c = (i * NT + threadIdx.x) * 8;
        if (c < width) {
            load8(x + off + c, v[i]);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[i][u];
        }
    }
    const float mean = block_sum2(s, 0.f, red).x / width;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int c = (i * NT + threadIdx.x) * 8;
        if (c < width)
#pragma unroll
            for (int u = 0; u < 8; ++u) q += (v[i][u] - mean) * (v[i][u] - mean);
    }
    const float rstd = rsqrtf(block_sum2(q, 0.f, red).x / width + eps);
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int c = (i * NT + threadIdx.x) * 8;
        if (c >= width) continue;
        float g[8], b[8], o[8];
        load8(gamma + c, g);
        load8(beta + c, b);
#pragma unroll
        for (int u = 0; u < 8; ++u) o[u] = (v[i][u] - mean) * rstd * g[u] + b[u];
        store8(y + off + c, o);
    }
    if (threadIdx.x == 0) {
        mean_out[blockIdx.x] = mean;
        rstd_out[blockIdx.x] = rstd;
    }
}

template <int V>
__global__ void __launch_bounds__(NT) ln_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                                    const __nv_bfloat16* __restrict__ x,
                                                    const __nv_bfloat16* __restrict__ gamma, const float* __restrict__ mean,
                                                    const float* __restrict__ rstd,
                                                    const __nv_bfloat16* __restrict__ dres,
                                                    __nv_bfloat16* __restrict__ dx, float* __restrict__ ws,
                                                    int rows, int width) {
    __shared__ float2 red[NT / 32];
    float pg[V][8], pb[V][8], g[V][8];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int c = (i * NT + threadIdx.x) * 8;
#pragma unroll
        for (int u = 0; u < 8; ++u) pg[i][u] = pb[i][u] = 0.f;
        if (c < width) load8(gamma + c, g[i]);
    }
    for (int row = blockIdx.x; row < rows; row += gridDim.x) {
        const int64_t off = static_cast<int64_t>(row) * width;
        const float mu = mean[row], rs = rstd[row];
        float xh[V][8], gd[V][8];
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int i = 0; i < V; ++i) {
            const int c = (i * NT + threadIdx.x) * 8;
            if (c >= width) continue;
            float xv[8], dv[8];
            load8(x + off + c, xv);
            load8(dy + off + c, dv);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                xh[i][u] = (xv[u] - mu) * rs;
                gd[i][u] = dv[u] * g[i][u];
                pg[i][u] += dv[u] * xh[i][u];
                pb[i][u] += dv[u];
                s1 += gd[i][u];
                s2 += gd[i][u] * xh[i][u];
            }
        }
        const float2 s = block_sum2(s1, s2, red);
        const float m1 = s.x / width, m2 = s.y / width;
#pragma unroll
        for (int i = 0; i < V; ++i) {
            const int c = (i * NT + threadIdx.x) * 8;
            if (c >= width) continue;
            float r[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) r[u] = rs * (gd[i][u] - m1 - xh[i][u] * m2);
            if (dres) {
                float rr[8];
                load8(dres + off + c, rr);
#pragma unroll
                for (int u = 0; u < 8; ++u) r[u] += rr[u];
            }
            store8(dx + off + c, r);
        }
    }
    // per-block partial column sums -> workspace [gridDim.x][2][width] (reduced by ln_colsum_kernel)
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int c = (i * NT + threadIdx.x) * 8;
        if (c >= width) continue;
        float* wg = ws + static_cast<int64_t>(blockIdx.x) * 2 * width + c;
        *reinterpret_cast<float4*>(wg) = make_float4(pg[i][0], pg[i][1], pg[i][2], pg[i][3]);
        *reinterpret_cast<float4*>(wg + 4) = make_float4(pg[i][4], pg[i][5], pg[i][6], pg[i][7]);
        *reinterpret_cast<float4*>(wg + width) = make_float4(pb[i][0], pb[i][1], pb[i][2], pb[i][3]);
        *reinterpret_cast<float4*>(wg + width + 4) = make_float4(pb[i][4], pb[i][5], pb[i][6], pb[i][7]);
    }
}

// dgamma/dbeta (+)= column sums of the per-block partials; one thread per output column,
// coalesced across the block, deterministic order.
__global__ void ln_colsum_kernel(const float* __restrict__ ws, int nblk, int width, float* __restrict__ dgamma,
                                 float* __restrict__ dbeta) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 2 * width) return;
    float s = 0.f;
    for (int b = 0; b < nblk; ++b) s += ws[static_cast<int64_t>(b) * 2 * width + c];
    if (c < width)
        dgamma[c] += s;
    else
        dbeta[c - width] += s;
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    }
    return n;
}

}  // namespace

void layernorm_fwd(const void* x, const void* gamma_, const void* beta_, void* y, float* mean, float* rstd, int rows,
                   int width, float eps, cudaStream_t st) {
    if (width % 8) throw std::runtime_error("layernorm: width must be a multiple of 8");
    auto X = static_cast<const __nv_bfloat16*>(x);
    auto Y = static_cast<__nv_bfloat16*>(y);
    auto gamma = static_cast<const __nv_bfloat16*>(gamma_);
    auto beta = static_cast<const __nv_bfloat16*>(beta_);
    const int v = (width + 1023) / 1024;
#define LNF(V_) \
    if (v <= V_) return ln_fwd_kernel<V_><<<rows, NT, 0, st>>>(X, gamma, beta, Y, mean, rstd, width, eps);
    LNF(1) LNF(2) LNF(4) LNF(8) LNF(16)
#undef LNF
    throw std::runtime_error("layernorm: width too large");
}

void layernorm_bwd(const void* dy, const void* x, const void* gamma_, const float* mean, const float* rstd,
                   const void* dres, void* dx, float* dgamma, float* dbeta, int rows, int width, cudaStream_t st) {
    if (width % 8) throw std::runtime_error("layernorm: width must be a multiple of 8");
    auto DY = static_cast<const __nv_bfloat16*>(dy);
    auto X = static_cast<const __nv_bfloat16*>(x);
    auto R = static_cast<const __nv_bfloat16*>(dres);
    auto DX = static_cast<__nv_bfloat16*>(dx);
    auto gamma = static_cast<const __nv_bfloat16*>(gamma_);
    const int v = (width + 1023) / 1024;
    // one block per SM: partial dgamma/dbeta stay in registers over ~rows/148 rows, then a
    // deterministic column reduction (no contended atomics)
    const int blocks = rows < sm_count() ? rows : sm_count();
    static float* ws = nullptr;
    static size_t ws_bytes = 0;
    const size_t need = static_cast<size_t>(blocks) * 2 * width * sizeof(float);
    if (need > ws_bytes) {
        if (ws) cudaFree(ws);
        if (cudaMalloc(&ws, need) != cudaSuccess) throw std::runtime_error("layernorm: workspace allocation failed");
        ws_bytes = need;
    }
#define LNB(V_)                                                                                           \
    if (v <= V_) {                                                                                        \
        ln_bwd_kernel<V_><<<blocks, NT, 0, st>>>(DY, X, gamma, mean, rstd, R, DX, ws, rows, width);        \
        ln_colsum_kernel<<<(2 * width + 255) / 256, 256, 0, st>>>(ws, blocks, width, dgamma, dbeta);     \
        return;                                                                                           \
    }
    LNB(1) LNB(2) LNB(4) LNB(8)
#undef LNB
    throw std::runtime_error("layernorm: width too large for backward");
}

}  // namespace bfpp
