// Causal multi-head attention entry points (head_dim 128). The tensor-core work is the
// tcgen05/TMEM flash-attention pair in attention_tc.cu; this file holds the two small
// HBM-bound kernels around the backward and the host entry points.
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

// delta_i = sum_d dO[i,d] * O[i,d] (one warp per (token, head)); also zeroes the f32 dQ accumulator.
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

// dQ (f32, accumulated by the backward kernel's red.global.add) -> bf16 into the Q columns of dqkv.
__global__ void attn_dq_convert_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int T,
                                       int HD) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i >= static_cast<int64_t>(T) * HD) return;
    const int64_t row = i / HD, col = i % HD;
    const float4 v = *reinterpret_cast<const float4*>(dq_acc + i);
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 out;
    out.x = *reinterpret_cast<uint32_t*>(&lo);
    out.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dqkv + row * 3 * HD + col) = out;
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
