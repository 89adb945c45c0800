// Causal multi-head attention entry points (head_dim 128). The tensor-core work is the
// tcgen05/TMEM flash-attention pair in attention_tc.cu; this file holds the two small
// HBM-bound kernels around the backward (delta = rowsum(dO * O), dQ f32 -> bf16; the dQ
// accumulator is zeroed with a memset) and the host entry points.
//
// Layouts (per micro-batch of B samples x S tokens, T = B*S rows):
//   qkv  [T][3h] bf16   Q at cols [0,h), K at [h,2h), V at [2h,3h); head j = cols j*128..
//   o    [T][h]  bf16
//   lse  [B*H][S] f32   log2-sum-exp of the scaled scores (saved for backward)
//   dqkv [T][3h] bf16   gradients, same layout as qkv
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdexcept>

#include "kernels.hpp"

namespace bfpp {
namespace {

constexpr int D = 128;  // head dim

// delta_i = sum_d dO[i,d] * O[i,d]: half a warp per (token, head), 16-byte loads (8 bf16 per lane).
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                     float* __restrict__ delta, int S, int H, int T) {
    const int pair = (blockIdx.x * blockDim.x + threadIdx.x) >> 4, l16 = threadIdx.x & 15;
    const bool ok = pair < T * H;
    float s = 0.f;
    if (ok) {
        const int row = pair / H, head = pair % H;
        const int64_t off = static_cast<int64_t>(row) * H * D + head * D + l16 * 8;
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(o + off));
        const uint4 c = __ldg(reinterpret_cast<const uint4*>(dout + off));
        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
        const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(c2[i]);
            s += x.x * y.x + x.y * y.y;
        }
    }
#pragma unroll
    for (int k = 8; k; k >>= 1) s += __shfl_xor_sync(0xffffffff, s, k);
    if (ok && l16 == 0) {
        const int row = pair / H, head = pair % H;
        const int b = row / S, q = row % S;
        delta[(static_cast<int64_t>(b) * H + head) * S + q] = s;
    }
}

// dQ (f32, accumulated by the backward kernel's TMA reduce-adds) -> bf16 into the Q columns of
// dqkv; 8 elements per thread (two 16-byte loads, one 16-byte store).
__global__ void attn_dq_convert_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int T,
                                       int HD) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
    if (i >= static_cast<int64_t>(T) * HD) return;
    const int64_t row = i / HD, col = i % HD;
    const float4 v0 = __ldcs(reinterpret_cast<const float4*>(dq_acc + i));
    const float4 v1 = __ldcs(reinterpret_cast<const float4*>(dq_acc + i + 4));
    __nv_bfloat162 p[4] = {__floats2bfloat162_rn(v0.x, v0.y), __floats2bfloat162_rn(v0.z, v0.w),
                           __floats2bfloat162_rn(v1.x, v1.y), __floats2bfloat162_rn(v1.z, v1.w)};
    *reinterpret_cast<uint4*>(dqkv + row * 3 * HD + col) = *reinterpret_cast<const uint4*>(p);
}

}  // namespace

void attention_fwd(const void* qkv, void* o, float* lse, int batch, int seq, int heads, int head_dim,
                   cudaStream_t st) {
    attention_fwd_tc(qkv, o, lse, batch, seq, heads, head_dim, st);
}

void attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse, float* delta, float* dq_acc,
                   void* dqkv, int batch, int seq, int heads, int head_dim, cudaStream_t st) {
    if (head_dim != D) throw std::runtime_error("attention: head_dim must be 128");
    const int T = batch * seq;
    const int64_t n = static_cast<int64_t>(T) * heads * head_dim;
    if (cudaMemsetAsync(dq_acc, 0, static_cast<size_t>(n) * sizeof(float), st) != cudaSuccess)
        throw std::runtime_error("attention: dQ accumulator memset failed");
    const int pairs = T * heads;
    attn_bwd_prep_kernel<<<(pairs + 15) / 16, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                                            static_cast<const __nv_bfloat16*>(dout), delta, seq, heads, T);
    attention_bwd_tc(qkv, dout, lse, delta, dq_acc, dqkv, batch, seq, heads, head_dim, st);
    attn_dq_convert_kernel<<<static_cast<unsigned>((n / 8 + 255) / 256), 256, 0, st>>>(
        dq_acc, static_cast<__nv_bfloat16*>(dqkv), T, heads * head_dim);
}

}  // namespace bfpp
