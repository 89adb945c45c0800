// LayerNorm forward/backward (HBM-bound). One warp per row, 8 rows per 256-thread
// block, 128-bit vector accesses, f32 statistics via warp shuffles; two passes per
// row (the second pass re-reads the row from L1) so no per-thread row arrays are
// held in registers at any width. The parameter gradients are a separate
// two-level column reduction over 8-row chunks (coalesced, deterministic).
//   fwd: y = (x - mean) * rstd * gamma + beta       (bf16 in/out; mean/rstd f32 saved)
//   bwd: dx = rstd * (g - mean(g) - xhat * mean(g * xhat)) [+ dres],  g = dy * gamma
//        dgamma += sum_rows dy * xhat, dbeta += sum_rows dy   (f32, accumulated across calls)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdexcept>

#include "kernels.hpp"

namespace bfpp {
namespace {

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
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int k = 16; k; k >>= 1) v += __shfl_xor_sync(0xffffffff, v, k);
    return v;
}

__global__ void __launch_bounds__(256) ln_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ gamma,
                                                     const __nv_bfloat16* __restrict__ beta,
                                                     __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
                                                     float* __restrict__ rstd_out, int rows, int width, float eps) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= rows) return;
    const __nv_bfloat16* xr = x + static_cast<int64_t>(row) * width;
    float s = 0.f, q = 0.f;
    for (int c = lane * 8; c < width; c += 256) {
        float v[8];
        load8(xr + c, v);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s += v[u];
            q += v[u] * v[u];
        }
    }
    s = warp_sum(s);
    q = warp_sum(q);
    const float mean = s / width;
    const float rstd = rsqrtf(fmaxf(q / width - mean * mean, 0.f) + eps);
    __nv_bfloat16* yr = y + static_cast<int64_t>(row) * width;
    for (int c = lane * 8; c < width; c += 256) {
        float v[8], g[8], b[8];
        load8(xr + c, v);
        load8(gamma + c, g);
        load8(beta + c, b);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (v[u] - mean) * rstd * g[u] + b[u];
        store8(yr + c, v);
    }
    if (lane == 0) {
        mean_out[row] = mean;
        rstd_out[row] = rstd;
    }
}

__global__ void __launch_bounds__(256) ln_bwd_dx_kernel(const __nv_bfloat16* __restrict__ dy,
                                                        const __nv_bfloat16* __restrict__ x,
                                                        const __nv_bfloat16* __restrict__ gamma,
                                                        const float* __restrict__ mean,
                                                        const float* __restrict__ rstd,
                                                        const __nv_bfloat16* __restrict__ dres,
                                                        __nv_bfloat16* __restrict__ dx, int rows, int width) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int64_t off = static_cast<int64_t>(row) * width;
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane * 8; c < width; c += 256) {
        float xv[8], dv[8], g[8];
        load8(x + off + c, xv);
        load8(dy + off + c, dv);
        load8(gamma + c, g);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float gd = dv[u] * g[u];
            s1 += gd;
            s2 += gd * (xv[u] - mu) * rs;
        }
    }
    const float m1 = warp_sum(s1) / width, m2 = warp_sum(s2) / width;
    for (int c = lane * 8; c < width; c += 256) {
        float xv[8], dv[8], g[8], r[8];
        load8(x + off + c, xv);
        load8(dy + off + c, dv);
        load8(gamma + c, g);
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = rs * (dv[u] * g[u] - m1 - (xv[u] - mu) * rs * m2);
        if (dres) {
            float rr[8];
            load8(dres + off + c, rr);
#pragma unroll
            for (int u = 0; u < 8; ++u) r[u] += rr[u];
        }
        store8(dx + off + c, r);
    }
}

// Per (row chunk, 8-column group): partial sums of dy * xhat and dy over the chunk's rows,
// written to ws[chunk][2][width]; ln_colsum_kernel then adds the chunk sums into dgamma/dbeta
// (deterministic, no atomics).
__global__ void __launch_bounds__(256) ln_bwd_param_kernel(const __nv_bfloat16* __restrict__ dy,
                                                           const __nv_bfloat16* __restrict__ x,
                                                           const float* __restrict__ mean,
                                                           const float* __restrict__ rstd, float* __restrict__ ws,
                                                           int rows, int width, int rows_per_chunk) {
    const int c = (blockIdx.x * 256 + threadIdx.x) * 8;
    if (c >= width) return;
    const int r0 = blockIdx.y * rows_per_chunk, r1 = min(rows, r0 + rows_per_chunk);
    float pg[8] = {}, pb[8] = {};
    for (int r = r0; r < r1; ++r) {
        const int64_t off = static_cast<int64_t>(r) * width + c;
        float xv[8], dv[8];
        load8(x + off, xv);
        load8(dy + off, dv);
        const float mu = mean[r], rs = rstd[r];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            pg[u] += dv[u] * (xv[u] - mu) * rs;
            pb[u] += dv[u];
        }
    }
    float* w = ws + static_cast<int64_t>(blockIdx.y) * 2 * width + c;
    *reinterpret_cast<float4*>(w) = make_float4(pg[0], pg[1], pg[2], pg[3]);
    *reinterpret_cast<float4*>(w + 4) = make_float4(pg[4], pg[5], pg[6], pg[7]);
    *reinterpret_cast<float4*>(w + width) = make_float4(pb[0], pb[1], pb[2], pb[3]);
    *reinterpret_cast<float4*>(w + width + 4) = make_float4(pb[4], pb[5], pb[6], pb[7]);
}

// column sums over chunks: blockIdx.y takes every gridDim.y-th chunk (short, unrolled,
// independent loads), then one atomic per (column, y) — gridDim.y-way contention only
__global__ void ln_colsum_kernel(const float* __restrict__ ws, int chunks, int width, float* __restrict__ dgamma,
                                 float* __restrict__ dbeta) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 2 * width) return;
    float s = 0.f;
#pragma unroll 8
    for (int b = blockIdx.y; b < chunks; b += gridDim.y) s += ws[static_cast<int64_t>(b) * 2 * width + c];
    atomicAdd(c < width ? dgamma + c : dbeta + (c - width), s);
}

}  // namespace

void layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int rows,
                   int width, float eps, cudaStream_t st) {
    if (width % 8) throw std::runtime_error("layernorm: width must be a multiple of 8");
    ln_fwd_kernel<<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x),
                                                  static_cast<const __nv_bfloat16*>(gamma),
                                                  static_cast<const __nv_bfloat16*>(beta),
                                                  static_cast<__nv_bfloat16*>(y), mean, rstd, rows, width, eps);
}

void layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                   const void* dres, void* dx, float* dgamma, float* dbeta, int rows, int width, cudaStream_t st,
                   int accumulate) {
    if (width % 8) throw std::runtime_error("layernorm: width must be a multiple of 8");
    auto DY = static_cast<const __nv_bfloat16*>(dy);
    auto X = static_cast<const __nv_bfloat16*>(x);
    ln_bwd_dx_kernel<<<(rows + 7) / 8, 256, 0, st>>>(DY, X, static_cast<const __nv_bfloat16*>(gamma), mean, rstd,
                                                     static_cast<const __nv_bfloat16*>(dres),
                                                     static_cast<__nv_bfloat16*>(dx), rows, width);
    // (column group, 8-row chunk) work items: enough parallelism to cover DRAM latency
    const int col_blocks = (width + 2047) / 2048;
    const int per = 8;
    const int chunks = (rows + per - 1) / per;
    static float* ws = nullptr;
    static size_t ws_bytes = 0;
    const size_t need = static_cast<size_t>(chunks) * 2 * width * sizeof(float);
    if (need > ws_bytes) {
        if (ws) cudaFree(ws);
        if (cudaMalloc(&ws, need) != cudaSuccess) throw std::runtime_error("layernorm: workspace allocation failed");
        ws_bytes = need;
    }
    ln_bwd_param_kernel<<<dim3(col_blocks, chunks), 256, 0, st>>>(DY, X, mean, rstd, ws, rows, width, per);
    if (!accumulate) {  // first contribution of this gradient unit: overwrite instead of add
        cudaMemsetAsync(dgamma, 0, static_cast<size_t>(width) * sizeof(float), st);
        cudaMemsetAsync(dbeta, 0, static_cast<size_t>(width) * sizeof(float), st);
    }
    ln_colsum_kernel<<<dim3((2 * width + 255) / 256, 32), 256, 0, st>>>(ws, chunks, width, dgamma, dbeta);
}

}  // namespace bfpp
