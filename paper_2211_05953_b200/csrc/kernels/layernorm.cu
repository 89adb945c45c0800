// LayerNorm forward/backward (HBM-bound), bf16 rows, f32 statistics.
//   fwd: y = (x - mean) * rstd * gamma + beta       (bf16 in/out; mean/rstd f32 saved)
//   bwd: dx = rstd * (g - mean(g) - xhat * mean(g * xhat)) [+ dres],  g = dy * gamma
//        dgamma += sum_rows dy * xhat, dbeta += sum_rows dy   (f32, accumulated across calls)
// Dispatch by row width:
//   backward, width <= 8192: bulk-staged kernel (cp.async.bulk rows into shared memory, column
//     partials per block) + one deterministic partial-sum kernel;
//   forward, width <= 4096: register-resident rows (one warp per row, or two for > 2048);
//     forward 4096 < width <= 8192: bulk-staged kernel;
//   wider rows: generic two-pass kernels (the row re-read from L1) with a two-level column
//     reduction for the parameter gradients. No atomics in any gradient path except the
//     generic column sum.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <set>
#include <stdexcept>
#include <type_traits>

#include "kernels.hpp"
#include "sm100_ptx.cuh"

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


// ---- register-resident variants (width <= 256 * NCH): one warp per row, the whole row held in
// registers as packed bf16 (NCH x 16 B per lane), all loads of a row in flight at once, exact
// two-pass statistics from registers; the backward also emits the block's dgamma/dbeta partials
// (shared-memory reduction over its 8 rows), so a LayerNorm backward is 2 launches, not 3 + 2 memsets.
__device__ __forceinline__ void unpack8(const uint4& raw, float (&v)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        float2 f = __bfloat1622float2(h[u]);
        v[2 * u] = f.x;
        v[2 * u + 1] = f.y;
    }
}

template <int NCH>
__global__ void __launch_bounds__(256) ln_fwd_reg_kernel(const __nv_bfloat16* __restrict__ x,
                                                         const __nv_bfloat16* __restrict__ gamma,
                                                         const __nv_bfloat16* __restrict__ beta,
                                                         __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
                                                         float* __restrict__ rstd_out, int rows, int width, float eps) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= rows) return;
    const __nv_bfloat16* xr = x + static_cast<int64_t>(row) * width;
    uint4 raw[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        const int c = (k * 32 + lane) * 8;
        if (c < width) raw[k] = *reinterpret_cast<const uint4*>(xr + c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        if ((k * 32 + lane) * 8 >= width) continue;
        float v[8];
        unpack8(raw[k], v);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    const float mean = warp_sum(s) / width;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        if ((k * 32 + lane) * 8 >= width) continue;
        float v[8];
        unpack8(raw[k], v);
#pragma unroll
        for (int u = 0; u < 8; ++u) q += (v[u] - mean) * (v[u] - mean);
    }
    const float rstd = rsqrtf(warp_sum(q) / width + eps);
    __nv_bfloat16* yr = y + static_cast<int64_t>(row) * width;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        const int c = (k * 32 + lane) * 8;
        if (c >= width) continue;
        float v[8], g[8], b[8];
        unpack8(raw[k], v);
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

// dx for 8 rows per block + the block's column partials ws[block][0..width) = sum dy*xhat,
// ws[block][width..2 width) = sum dy: per 256-column chunk the 8 warps stage their values in
// shared memory and each thread sums one column over the block's rows (no atomics).
template <int NCH>
__global__ void __launch_bounds__(256, 1) ln_bwd_reg_kernel(const __nv_bfloat16* __restrict__ dy,
                                                         const __nv_bfloat16* __restrict__ x,
                                                         const __nv_bfloat16* __restrict__ gamma,
                                                         const float* __restrict__ mean,
                                                         const float* __restrict__ rstd,
                                                         const __nv_bfloat16* __restrict__ dres,
                                                         __nv_bfloat16* __restrict__ dx, float* __restrict__ ws,
                                                         int rows, int width) {
    __shared__ __align__(16) float red[8][2][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * 8 + warp;
    const bool valid = row < rows;
    const int64_t off = static_cast<int64_t>(valid ? row : 0) * width;
    // every load of the row up front (x, dy, gamma, and the residual gradient for small rows)
    constexpr bool kPrefetch = NCH <= 8;
    uint4 rx[NCH], rd[NCH], rg[kPrefetch ? NCH : 1], rr[kPrefetch ? NCH : 1];
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        const int c = (k * 32 + lane) * 8;
        if (valid && c < width) {
            rx[k] = *reinterpret_cast<const uint4*>(x + off + c);
            rd[k] = *reinterpret_cast<const uint4*>(dy + off + c);
        } else {
            rx[k] = make_uint4(0, 0, 0, 0);
            rd[k] = make_uint4(0, 0, 0, 0);
        }
        if constexpr (kPrefetch) {
            rg[k] = c < width ? *reinterpret_cast<const uint4*>(gamma + c) : make_uint4(0, 0, 0, 0);
            rr[k] = (dres && valid && c < width) ? *reinterpret_cast<const uint4*>(dres + off + c)
                                                 : make_uint4(0, 0, 0, 0);
        }
    }
    const float mu = valid ? mean[row] : 0.f, rs = valid ? rstd[row] : 0.f;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        const int c = (k * 32 + lane) * 8;
        if (c >= width) continue;
        float xv[8], dv[8], g[8];
        unpack8(rx[k], xv);
        unpack8(rd[k], dv);
        if constexpr (kPrefetch) unpack8(rg[k], g);
        else load8(gamma + c, g);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float gd = dv[u] * g[u];
            s1 += gd;
            s2 += gd * (xv[u] - mu) * rs;
        }
    }
    const float m1 = warp_sum(s1) / width, m2 = warp_sum(s2) / width;
    // dx: independent chunks (no barriers), so the residual-gradient loads are all in flight together
    if (valid) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const int c = (k * 32 + lane) * 8;
            if (c >= width) continue;
            float xv[8], dv[8], g[8], r[8];
            unpack8(rx[k], xv);
            unpack8(rd[k], dv);
            if constexpr (kPrefetch) unpack8(rg[k], g);
            else load8(gamma + c, g);
#pragma unroll
            for (int u = 0; u < 8; ++u) r[u] = rs * (dv[u] * g[u] - m1 - (xv[u] - mu) * rs * m2);
            if (dres) {
                float rv[8];
                if constexpr (kPrefetch) unpack8(rr[k], rv);
                else load8(dres + off + c, rv);
#pragma unroll
                for (int u = 0; u < 8; ++u) r[u] += rv[u];
            }
            store8(dx + off + c, r);
        }
    }
    // column partials over the block's 8 rows, one 256-column chunk at a time
    float* wout = ws + static_cast<int64_t>(blockIdx.x) * 2 * width;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        float xv[8], dv[8];
        unpack8(rx[k], xv);
        unpack8(rd[k], dv);
        float4* rg = reinterpret_cast<float4*>(&red[warp][0][lane * 8]);
        float4* rb = reinterpret_cast<float4*>(&red[warp][1][lane * 8]);
        // rows past the end hold zeros in rx/rd, so they contribute nothing
        rg[0] = make_float4(dv[0] * (xv[0] - mu) * rs, dv[1] * (xv[1] - mu) * rs, dv[2] * (xv[2] - mu) * rs,
                            dv[3] * (xv[3] - mu) * rs);
        rg[1] = make_float4(dv[4] * (xv[4] - mu) * rs, dv[5] * (xv[5] - mu) * rs, dv[6] * (xv[6] - mu) * rs,
                            dv[7] * (xv[7] - mu) * rs);
        rb[0] = make_float4(dv[0], dv[1], dv[2], dv[3]);
        rb[1] = make_float4(dv[4], dv[5], dv[6], dv[7]);
        __syncthreads();
        const int col = k * 256 + threadIdx.x;
        if (col < width) {
            float tg = 0.f, tb = 0.f;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                tg += red[w][0][threadIdx.x];
                tb += red[w][1][threadIdx.x];
            }
            wout[col] = tg;
            wout[width + col] = tb;
        }
        __syncthreads();
    }
}

// dgamma/dbeta (=, or += when accumulating) = column sums of the n_part block partials: 32
// columns per block (one per lane, 128-byte rows per warp access), 16 warps split the partials
// and a fixed-order shared-memory sum combines them. Deterministic, no atomics, no memsets.
constexpr int kPartsumWarps = 16;
__global__ void __launch_bounds__(kPartsumWarps * 32) ln_partsum_kernel(const float* __restrict__ ws, int n_part,
                                                                        int width, float* __restrict__ dgamma,
                                                                        float* __restrict__ dbeta, int accumulate) {
    __shared__ float red[kPartsumWarps][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * 32 + lane;  // column in [0, 2 width)
    float s = 0.f;
    if (c < 2 * width) {
#pragma unroll 8
        for (int b = warp; b < n_part; b += kPartsumWarps) s += ws[static_cast<int64_t>(b) * 2 * width + c];
    }
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && c < 2 * width) {
        float t = red[0][lane];
#pragma unroll
        for (int w = 1; w < kPartsumWarps; ++w) t += red[w][lane];
        float* dst = c < width ? dgamma + c : dbeta + (c - width);
        *dst = accumulate ? *dst + t : t;
    }
}
void launch_partsum(const float* ws, int n_part, int width, float* dgamma, float* dbeta, int accumulate,
                    cudaStream_t st) {
    ln_partsum_kernel<<<(2 * width + 31) / 32, kPartsumWarps * 32, 0, st>>>(ws, n_part, width, dgamma, dbeta,
                                                                          accumulate);
}

// chunks of 8 elements per lane: NCH = 1, 2, 4, 8, 12, 16, 20, 24 (width <= 256 NCH), up to MAX
template <int MAX, typename F>
bool ln_dispatch(int width, F&& f) {
    const int n = (width + 255) / 256;
    if (n <= 1) { f(std::integral_constant<int, 1>{}); return true; }
    if (n <= 2) { f(std::integral_constant<int, 2>{}); return true; }
    if (n <= 4) { f(std::integral_constant<int, 4>{}); return true; }
    if (n <= 8) { f(std::integral_constant<int, 8>{}); return true; }
    if (n <= 12) { f(std::integral_constant<int, 12>{}); return true; }
    if (n <= 16) { f(std::integral_constant<int, 16>{}); return true; }
    if constexpr (MAX >= 24) {
        if (n <= 20) { f(std::integral_constant<int, 20>{}); return true; }
        if (n <= 24) { f(std::integral_constant<int, 24>{}); return true; }
    }
    return false;
}


// ---- wide rows (2048 < width <= 4096): W warps per row, 8 chunks of 8 elements per lane each,
// R = 8 / W rows per block; the row statistics are combined through shared memory.
template <int W>
struct MwShape {
    static constexpr int R = W == 3 ? 2 : 8 / W;  // rows per block
    static constexpr int kThreads = 32 * W * R;
};

template <int W>
__global__ void __launch_bounds__(MwShape<W>::kThreads) ln_fwd_mw_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ gamma,
    const __nv_bfloat16* __restrict__ beta, __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
    float* __restrict__ rstd_out, int rows, int width, float eps) {
    constexpr int R = MwShape<W>::R;
    __shared__ float red[R][W];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int part = warp % W, ri = warp / W;
    const int row = blockIdx.x * R + ri;
    const bool valid = row < rows;
    const __nv_bfloat16* xr = x + static_cast<int64_t>(valid ? row : 0) * width;
    uint4 raw[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int c = ((part * 8 + k) * 32 + lane) * 8;
        raw[k] = (valid && c < width) ? *reinterpret_cast<const uint4*>(xr + c) : make_uint4(0, 0, 0, 0);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float v[8];
        unpack8(raw[k], v);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
    }
    s = warp_sum(s);
    if (lane == 0) red[ri][part] = s;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) tot += red[ri][w];
    const float mean = tot / width;
    __syncthreads();
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (((part * 8 + k) * 32 + lane) * 8 >= width) continue;
        float v[8];
        unpack8(raw[k], v);
#pragma unroll
        for (int u = 0; u < 8; ++u) q += (v[u] - mean) * (v[u] - mean);
    }
    q = warp_sum(q);
    if (lane == 0) red[ri][part] = q;
    __syncthreads();
    float qt = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) qt += red[ri][w];
    const float rstd = rsqrtf(qt / width + eps);
    if (!valid) return;
    __nv_bfloat16* yr = y + static_cast<int64_t>(row) * width;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int c = ((part * 8 + k) * 32 + lane) * 8;
        if (c >= width) continue;
        float v[8], g[8], b[8];
        unpack8(raw[k], v);
        load8(gamma + c, g);
        load8(beta + c, b);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (v[u] - mean) * rstd * g[u] + b[u];
        store8(yr + c, v);
    }
    if (lane == 0 && part == 0) {
        mean_out[row] = mean;
        rstd_out[row] = rstd;
    }
}

template <int W>
__global__ void __launch_bounds__(MwShape<W>::kThreads, 1) ln_bwd_mw_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ gamma,
    const float* __restrict__ mean, const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ dres,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ ws, int rows, int width) {
    constexpr int R = MwShape<W>::R;
    __shared__ float st[R][W][2];
    __shared__ __align__(16) float red[W * R][2][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int part = warp % W, ri = warp / W;
    const int row = blockIdx.x * R + ri;
    const bool valid = row < rows;
    const int64_t off = static_cast<int64_t>(valid ? row : 0) * width;
    uint4 rx[8], rd[8], rg[8], rr[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int c = ((part * 8 + k) * 32 + lane) * 8;
        const bool in = valid && c < width;
        rx[k] = in ? *reinterpret_cast<const uint4*>(x + off + c) : make_uint4(0, 0, 0, 0);
        rd[k] = in ? *reinterpret_cast<const uint4*>(dy + off + c) : make_uint4(0, 0, 0, 0);
        rg[k] = c < width ? *reinterpret_cast<const uint4*>(gamma + c) : make_uint4(0, 0, 0, 0);
        rr[k] = (dres && in) ? *reinterpret_cast<const uint4*>(dres + off + c) : make_uint4(0, 0, 0, 0);
    }
    const float mu = valid ? mean[row] : 0.f, rs = valid ? rstd[row] : 0.f;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float xv[8], dv[8], g[8];
        unpack8(rx[k], xv);
        unpack8(rd[k], dv);
        unpack8(rg[k], g);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float gd = dv[u] * g[u];
            s1 += gd;
            s2 += gd * (xv[u] - mu) * rs;
        }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
        st[ri][part][0] = s1;
        st[ri][part][1] = s2;
    }
    __syncthreads();
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        t1 += st[ri][w][0];
        t2 += st[ri][w][1];
    }
    const float m1 = t1 / width, m2 = t2 / width;
    if (valid) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int c = ((part * 8 + k) * 32 + lane) * 8;
            if (c >= width) continue;
            float xv[8], dv[8], g[8], r[8], rv[8];
            unpack8(rx[k], xv);
            unpack8(rd[k], dv);
            unpack8(rg[k], g);
            unpack8(rr[k], rv);
#pragma unroll
            for (int u = 0; u < 8; ++u) r[u] = rs * (dv[u] * g[u] - m1 - (xv[u] - mu) * rs * m2) + rv[u];
            store8(dx + off + c, r);
        }
    }
    // column partials over the block's R rows: round k covers chunk (w * 8 + k) of every part w
    float* wout = ws + static_cast<int64_t>(blockIdx.x) * 2 * width;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float xv[8], dv[8];
        unpack8(rx[k], xv);
        unpack8(rd[k], dv);
        float4* pg = reinterpret_cast<float4*>(&red[warp][0][lane * 8]);
        float4* pb = reinterpret_cast<float4*>(&red[warp][1][lane * 8]);
        pg[0] = make_float4(dv[0] * (xv[0] - mu) * rs, dv[1] * (xv[1] - mu) * rs, dv[2] * (xv[2] - mu) * rs,
                            dv[3] * (xv[3] - mu) * rs);
        pg[1] = make_float4(dv[4] * (xv[4] - mu) * rs, dv[5] * (xv[5] - mu) * rs, dv[6] * (xv[6] - mu) * rs,
                            dv[7] * (xv[7] - mu) * rs);
        pb[0] = make_float4(dv[0], dv[1], dv[2], dv[3]);
        pb[1] = make_float4(dv[4], dv[5], dv[6], dv[7]);
        __syncthreads();
        for (int i = threadIdx.x; i < W * 256; i += MwShape<W>::kThreads) {
            const int w = i / 256, t = i % 256;
            const int col = (w * 8 + k) * 256 + t;
            if (col < width) {
                float tg = 0.f, tb = 0.f;
#pragma unroll
                for (int r2 = 0; r2 < R; ++r2) {
                    tg += red[r2 * W + w][0][t];
                    tb += red[r2 * W + w][1][t];
                }
                wout[col] = tg;
                wout[width + col] = tb;
            }
        }
        __syncthreads();
    }
}

template <typename F>
bool ln_dispatch_wide(int width, F&& f) {
    if (width <= 2048) return false;
    if (width <= 4096) { f(std::integral_constant<int, 2>{}); return true; }
    // W = 3 measured slower than the two-pass kernels at width 5120 (scripts/ln_bench.py); wider
    // rows keep the generic path
    return false;
}

using namespace ptx;

// ---- bulk-staged variants (scripts/ln_bench.py, backward at 2048 x 2048: 13.6 vs 16.3 us; at
// 2048 x 8192: 44 vs 101 us): a block's R rows (and gamma / beta) are fetched with one-shot
// cp.async.bulk copies into shared memory, completing on one mbarrier, so every load of the block
// is in flight at once with no register cost; two or more blocks per SM then overlap one block's
// arithmetic with the next block's loads. W = 8 / R warps per row.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ uint4 lds16(const __nv_bfloat16* p) { return *reinterpret_cast<const uint4*>(p); }

// the rows [r0, r0 + nr) of each of the n_src tensors, then the n_vec width-vectors, issued by warp 0
__device__ __forceinline__ void bulk_rows(uint64_t* bar, const __nv_bfloat16* const* src, __nv_bfloat16* const* dst,
                                          int n_src, const __nv_bfloat16* const* vsrc, __nv_bfloat16* const* vdst,
                                          int n_vec, int64_t r0, int nr, int width) {
    const int lane = threadIdx.x & 31;
    const uint32_t rb = static_cast<uint32_t>(width) * 2;
    if (lane == 0) mbar_expect_tx(bar, rb * static_cast<uint32_t>(n_src * nr + n_vec));
    __syncwarp();
    for (int i = lane; i < n_src * nr + n_vec; i += 32) {
        if (i < n_src * nr) {
            const int t = i / nr, r = i % nr;
            bulk_g2s(dst[t] + static_cast<int64_t>(r) * width, src[t] + (r0 + r) * width, rb, bar);
        } else {
            bulk_g2s(vdst[i - n_src * nr], vsrc[i - n_src * nr], rb, bar);
        }
    }
}

template <int R>
__global__ void __launch_bounds__(256) ln_fwd_bulk_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const __nv_bfloat16* __restrict__ beta,
                                                          __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
                                                          float* __restrict__ rstd_out, int rows, int width, float eps) {
    constexpr int W = 8 / R;
    extern __shared__ __align__(128) uint8_t ln_smem[];
    __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(ln_smem);
    __nv_bfloat16* sg = sx + R * width;
    __nv_bfloat16* sb = sg + width;
    __shared__ __align__(8) uint64_t bar;
    __shared__ float st[R][W];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * R;
    const int nr = min(R, static_cast<int>(rows - r0));
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == 0) {
        const __nv_bfloat16* src[1] = {x};
        __nv_bfloat16* dst[1] = {sx};
        const __nv_bfloat16* vs[2] = {gamma, beta};
        __nv_bfloat16* vd[2] = {sg, sb};
        bulk_rows(&bar, src, dst, 1, vs, vd, 2, r0, nr, width);
    }
    mbar_wait(&bar, 0);
    const int ri = warp / W, part = warp % W;
    const bool valid = ri < nr;
    const __nv_bfloat16* xr = sx + ri * width;
    float s = 0.f;
    if (valid)
        for (int c = (part * 32 + lane) * 8; c < width; c += W * 256) {
            float v[8];
            unpack8(lds16(xr + c), v);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
    s = warp_sum(s);
    if constexpr (W > 1) {
        if (lane == 0) st[ri][part] = s;
        __syncthreads();
        s = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) s += st[ri][w];
        __syncthreads();
    }
    const float mean = s / width;
    float q = 0.f;
    if (valid)
        for (int c = (part * 32 + lane) * 8; c < width; c += W * 256) {
            float v[8];
            unpack8(lds16(xr + c), v);
#pragma unroll
            for (int u = 0; u < 8; ++u) q += (v[u] - mean) * (v[u] - mean);
        }
    q = warp_sum(q);
    if constexpr (W > 1) {
        if (lane == 0) st[ri][part] = q;
        __syncthreads();
        q = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) q += st[ri][w];
    }
    const float rstd = rsqrtf(q / width + eps);
    if (!valid) return;
    __nv_bfloat16* yr = y + (r0 + ri) * width;
    for (int c = (part * 32 + lane) * 8; c < width; c += W * 256) {
        float v[8], g[8], b[8];
        unpack8(lds16(xr + c), v);
        unpack8(lds16(sg + c), g);
        unpack8(lds16(sb + c), b);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (v[u] - mean) * rstd * g[u] + b[u];
        store8(yr + c, v);
    }
    if (lane == 0 && part == 0) {
        mean_out[r0 + ri] = mean;
        rstd_out[r0 + ri] = rstd;
    }
}

// dx of R-row groups (block-strided loop, one group staged at a time), and the block's column
// partials ws[block][0..width) = sum dy * xhat, ws[block][width..2 width) = sum dy accumulated
// in registers across its groups (C 2048-column slices per thread) and written once, so the
// partial traffic is gridDim.x (<= 2 per SM) rows, not one per group
template <int R, int C, bool RES>
__global__ void __launch_bounds__(256) ln_bwd_bulk_kernel(const __nv_bfloat16* __restrict__ dy,
                                                          const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ rstd,
                                                          const __nv_bfloat16* __restrict__ dres,
                                                          __nv_bfloat16* __restrict__ dx, float* __restrict__ ws,
                                                          int rows, int width) {
    constexpr int W = 8 / R;
    extern __shared__ __align__(128) uint8_t ln_smem[];
    __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(ln_smem);
    __nv_bfloat16* sd = sx + R * width;
    __nv_bfloat16* sg = sd + R * width;
    __nv_bfloat16* sr = sg + width;  // RES only
    __shared__ __align__(8) uint64_t bar;
    __shared__ float s_mu[R], s_rs[R];
    __shared__ float st[R][W][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ri = warp / W, part = warp % W;
    const int n_groups = (rows + R - 1) / R;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    float pg[C][8] = {}, pb[C][8] = {};
    int it = 0;
    for (int grp = blockIdx.x; grp < n_groups; grp += gridDim.x, ++it) {
        const int64_t r0 = static_cast<int64_t>(grp) * R;
        const int nr = min(R, static_cast<int>(rows - r0));
        __syncthreads();  // the previous group's rows and statistics are no longer read
        if (threadIdx.x < R) {
            const bool v = static_cast<int>(threadIdx.x) < nr;
            s_mu[threadIdx.x] = v ? mean[r0 + threadIdx.x] : 0.f;
            s_rs[threadIdx.x] = v ? rstd[r0 + threadIdx.x] : 0.f;
        }
        if (warp == 0) {
            const __nv_bfloat16* src[3] = {x, dy, dres};
            __nv_bfloat16* dst[3] = {sx, sd, sr};
            const __nv_bfloat16* vs[1] = {gamma};
            __nv_bfloat16* vd[1] = {sg};
            bulk_rows(&bar, src, dst, RES ? 3 : 2, vs, vd, it == 0 ? 1 : 0, r0, nr, width);
        }
        __syncthreads();  // s_mu / s_rs
        mbar_wait(&bar, it & 1);
        const bool valid = ri < nr;
        const float mu = s_mu[ri], rs = s_rs[ri];
        const __nv_bfloat16* xr = sx + ri * width;
        const __nv_bfloat16* dr = sd + ri * width;
        float s1 = 0.f, s2 = 0.f;
        if (valid)
            for (int c = (part * 32 + lane) * 8; c < width; c += W * 256) {
                float xv[8], dv[8], g[8];
                unpack8(lds16(xr + c), xv);
                unpack8(lds16(dr + c), dv);
                unpack8(lds16(sg + c), g);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float gd = dv[u] * g[u];
                    s1 += gd;
                    s2 += gd * (xv[u] - mu) * rs;
                }
            }
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        if constexpr (W > 1) {
            if (lane == 0) {
                st[ri][part][0] = s1;
                st[ri][part][1] = s2;
            }
            __syncthreads();
            s1 = s2 = 0.f;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                s1 += st[ri][w][0];
                s2 += st[ri][w][1];
            }
        }
        const float m1 = s1 / width, m2 = s2 / width;
        if (valid) {
            __nv_bfloat16* dxr = dx + (r0 + ri) * width;
            for (int c = (part * 32 + lane) * 8; c < width; c += W * 256) {
                float xv[8], dv[8], g[8], r[8];
                unpack8(lds16(xr + c), xv);
                unpack8(lds16(dr + c), dv);
                unpack8(lds16(sg + c), g);
#pragma unroll
                for (int u = 0; u < 8; ++u) r[u] = rs * (dv[u] * g[u] - m1 - (xv[u] - mu) * rs * m2);
                if constexpr (RES) {
                    float rv[8];
                    unpack8(lds16(sr + ri * width + c), rv);
#pragma unroll
                    for (int u = 0; u < 8; ++u) r[u] += rv[u];
                }
                store8(dxr + c, r);
            }
        }
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const int c = k * 2048 + threadIdx.x * 8;
            if (c >= width) continue;
            for (int r = 0; r < nr; ++r) {
                float xv[8], dv[8];
                unpack8(lds16(sx + r * width + c), xv);
                unpack8(lds16(sd + r * width + c), dv);
                const float m = s_mu[r], q = s_rs[r];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    pg[k][u] += dv[u] * (xv[u] - m) * q;
                    pb[k][u] += dv[u];
                }
            }
        }
    }
    float* wout = ws + static_cast<int64_t>(blockIdx.x) * 2 * width;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        const int c = k * 2048 + threadIdx.x * 8;
        if (c >= width) continue;
        *reinterpret_cast<float4*>(wout + c) = make_float4(pg[k][0], pg[k][1], pg[k][2], pg[k][3]);
        *reinterpret_cast<float4*>(wout + c + 4) = make_float4(pg[k][4], pg[k][5], pg[k][6], pg[k][7]);
        *reinterpret_cast<float4*>(wout + width + c) = make_float4(pb[k][0], pb[k][1], pb[k][2], pb[k][3]);
        *reinterpret_cast<float4*>(wout + width + c + 4) = make_float4(pb[k][4], pb[k][5], pb[k][6], pb[k][7]);
    }
}

// rows per block of the bulk kernels (8 / R warps per row); 0 = row too wide for them
int ln_bulk_rows(int width) {
    static const int mode = [] {
        const char* e = getenv("BFPP_LN_BULK");  // A/B switch: 0 = register-resident kernels
        return e ? atoi(e) : 1;
    }();
    if (!mode) return 0;
    return width <= 2048 ? 8 : width <= 4096 ? 4 : width <= 8192 ? 2 : 0;
}
template <typename F>
void ln_bulk_dispatch(int R, F&& f) {
    switch (R) {
        case 8: f(std::integral_constant<int, 8>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        case 2: f(std::integral_constant<int, 2>{}); break;
        default: f(std::integral_constant<int, 2>{}); break;
    }
}
// raise a kernel's dynamic shared-memory limit once (host calls come from one thread per device)
template <class K>
void ln_smem_optin(K kernel) {
    static std::set<const void*> done;
    if (done.insert(reinterpret_cast<const void*>(kernel)).second)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

float* ln_workspace(size_t bytes) {
    // one workspace per device (the executor runs every LayerNorm backward on one stream)
    static thread_local float* ws[64] = {};
    static thread_local size_t ws_bytes[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (bytes > ws_bytes[dev]) {
        if (ws[dev]) cudaFree(ws[dev]);
        if (cudaMalloc(&ws[dev], bytes) != cudaSuccess) throw std::runtime_error("layernorm: workspace allocation failed");
        ws_bytes[dev] = bytes;
    }
    return ws[dev];
}

}  // namespace

void layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int rows,
                   int width, float eps, cudaStream_t st) {
    if (width % 8) throw std::runtime_error("layernorm: width must be a multiple of 8");
    // forward: the register-resident kernels are as fast up to 4096 columns (scripts/ln_bench.py:
    // 5.1 vs 5.3 us at 2048 x 2048); the bulk kernel takes the wider rows (11.0 vs 14.8 us at 5120)
    if (const int R = width > 4096 ? ln_bulk_rows(width) : 0) {
        ln_bulk_dispatch(R, [&](auto r) {
            constexpr int RR = decltype(r)::value;
            const size_t smem = static_cast<size_t>(RR + 2) * width * 2;
            ln_smem_optin(ln_fwd_bulk_kernel<RR>);
            ln_fwd_bulk_kernel<RR><<<(rows + RR - 1) / RR, 256, smem, st>>>(
                static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(gamma),
                static_cast<const __nv_bfloat16*>(beta), static_cast<__nv_bfloat16*>(y), mean, rstd, rows, width, eps);
        });
        return;
    }
    const bool wide = ln_dispatch_wide(width, [&](auto w) {
        constexpr int W = decltype(w)::value;
        using Sh = MwShape<W>;
        ln_fwd_mw_kernel<W><<<(rows + Sh::R - 1) / Sh::R, Sh::kThreads, 0, st>>>(
            static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(gamma),
            static_cast<const __nv_bfloat16*>(beta), static_cast<__nv_bfloat16*>(y), mean, rstd, rows, width, eps);
    });
    if (wide) return;
    const bool done = ln_dispatch<24>(width, [&](auto nch) {
        ln_fwd_reg_kernel<decltype(nch)::value><<<(rows + 7) / 8, 256, 0, st>>>(
            static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(gamma),
            static_cast<const __nv_bfloat16*>(beta), static_cast<__nv_bfloat16*>(y), mean, rstd, rows, width, eps);
    });
    if (done) return;
    ln_fwd_kernel<<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x),
                                                  static_cast<const __nv_bfloat16*>(gamma),
                                                  static_cast<const __nv_bfloat16*>(beta),
                                                  static_cast<__nv_bfloat16*>(y), mean, rstd, rows, width, eps);
}

int layernorm_bwd_launches(int width) { return ln_bulk_rows(width) || width <= 4096 ? 2 : 3; }

void layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                   const void* dres, void* dx, float* dgamma, float* dbeta, int rows, int width, cudaStream_t st,
                   int accumulate) {
    if (width % 8) throw std::runtime_error("layernorm: width must be a multiple of 8");
    auto DY = static_cast<const __nv_bfloat16*>(dy);
    auto X = static_cast<const __nv_bfloat16*>(x);
    if (const int R = ln_bulk_rows(width)) {
        static int sm_of[64] = {};  // SM count per device, queried once
        int dev = 0;
        cudaGetDevice(&dev);
        if (!sm_of[dev & 63]) cudaDeviceGetAttribute(&sm_of[dev & 63], cudaDevAttrMultiProcessorCount, dev);
        const int n_sm = sm_of[dev & 63] > 0 ? sm_of[dev & 63] : 148;
        const int parts = std::min((rows + R - 1) / R, 2 * n_sm);  // two resident blocks per SM
        float* part = ln_workspace(static_cast<size_t>(parts) * 2 * width * sizeof(float));
        ln_bulk_dispatch(R, [&](auto r) {
            constexpr int RR = decltype(r)::value, CC = 8 / RR;
            auto launch = [&](auto kernel, int n_src) {
                const size_t smem = static_cast<size_t>(n_src * RR + 1) * width * 2;
                ln_smem_optin(kernel);
                kernel<<<parts, 256, smem, st>>>(DY, X, static_cast<const __nv_bfloat16*>(gamma), mean, rstd,
                                                 static_cast<const __nv_bfloat16*>(dres),
                                                 static_cast<__nv_bfloat16*>(dx), part, rows, width);
            };
            if (dres) launch(ln_bwd_bulk_kernel<RR, CC, true>, 3);
            else launch(ln_bwd_bulk_kernel<RR, CC, false>, 2);
        });
        launch_partsum(part, parts, width, dgamma, dbeta, accumulate, st);
        return;
    }
    {
        int parts = 0;
        const bool wide = ln_dispatch_wide(width, [&](auto w) {
            constexpr int W = decltype(w)::value;
            using Sh = MwShape<W>;
            parts = (rows + Sh::R - 1) / Sh::R;
            float* part = ln_workspace(static_cast<size_t>(parts) * 2 * width * sizeof(float));
            ln_bwd_mw_kernel<W><<<parts, Sh::kThreads, 0, st>>>(
                DY, X, static_cast<const __nv_bfloat16*>(gamma), mean, rstd, static_cast<const __nv_bfloat16*>(dres),
                static_cast<__nv_bfloat16*>(dx), part, rows, width);
            launch_partsum(part, parts, width, dgamma, dbeta, accumulate, st);
        });
        if (wide) return;
    }
    const int blocks = (rows + 7) / 8;
    {
        float* part = ln_workspace(static_cast<size_t>(blocks) * 2 * width * sizeof(float));
        const bool done = ln_dispatch<16>(width, [&](auto nch) {
            ln_bwd_reg_kernel<decltype(nch)::value><<<blocks, 256, 0, st>>>(
                DY, X, static_cast<const __nv_bfloat16*>(gamma), mean, rstd, static_cast<const __nv_bfloat16*>(dres),
                static_cast<__nv_bfloat16*>(dx), part, rows, width);
        });  // x and dy both register-resident: up to 16 chunks per lane without spills
        if (done) {
            launch_partsum(part, blocks, width, dgamma, dbeta, accumulate, st);
            return;
        }
    }
    ln_bwd_dx_kernel<<<(rows + 7) / 8, 256, 0, st>>>(DY, X, static_cast<const __nv_bfloat16*>(gamma), mean, rstd,
                                                     static_cast<const __nv_bfloat16*>(dres),
                                                     static_cast<__nv_bfloat16*>(dx), rows, width);
    // (column group, 8-row chunk) work items: enough parallelism to cover DRAM latency
    const int col_blocks = (width + 2047) / 2048;
    const int per = 8;
    const int chunks = (rows + per - 1) / per;
    float* ws = ln_workspace(static_cast<size_t>(chunks) * 2 * width * sizeof(float));
    ln_bwd_param_kernel<<<dim3(col_blocks, chunks), 256, 0, st>>>(DY, X, mean, rstd, ws, rows, width, per);
    if (!accumulate) {  // first contribution of this gradient unit: overwrite instead of add
        cudaMemsetAsync(dgamma, 0, static_cast<size_t>(width) * sizeof(float), st);
        cudaMemsetAsync(dbeta, 0, static_cast<size_t>(width) * sizeof(float), st);
    }
    ln_colsum_kernel<<<dim3((2 * width + 255) / 256, 32), 256, 0, st>>>(ws, chunks, width, dgamma, dbeta);
}

}  // namespace bfpp
