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
                                     float* __restrict__ delta, float* __restrict__ dq_acc, int S, int H, int T) {
    // a half-warp per two (token, head) pairs: all four 16-byte loads in flight before the math;
    // the same threads zero the pairs' dQ accumulator rows (no separate memset)
    const int base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 4) * 2, l16 = threadIdx.x & 15;
    uint4 a[2], c[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int pair = base + k;
        if (pair < T * H) {
            const int64_t off = static_cast<int64_t>(pair) * D + l16 * 8;  // [T][H][D] = pair * D
            a[k] = __ldg(reinterpret_cast<const uint4*>(o + off));
            c[k] = __ldg(reinterpret_cast<const uint4*>(dout + off));
            __stcs(reinterpret_cast<float4*>(dq_acc + off), make_float4(0.f, 0.f, 0.f, 0.f));
            __stcs(reinterpret_cast<float4*>(dq_acc + off + 4), make_float4(0.f, 0.f, 0.f, 0.f));
        } else {
            a[k] = c[k] = make_uint4(0, 0, 0, 0);
        }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a[k]);
        const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c[k]);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(c2[i]);
            s += x.x * y.x + x.y * y.y;
        }
#pragma unroll
        for (int m = 8; m; m >>= 1) s += __shfl_xor_sync(0xffffffff, s, m);
        const int pair = base + k;
        if (pair < T * H && l16 == 0) {
            const int row = pair / H, head = pair % H;
            const int bb = row / S, q = row % S;
            delta[(static_cast<int64_t>(bb) * H + head) * S + q] = s;
        }
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
    const int pairs = T * heads;
    attn_bwd_prep_kernel<<<(pairs + 31) / 32, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                                            static_cast<const __nv_bfloat16*>(dout), delta, dq_acc,
                                                            seq, heads, T);
    attention_bwd_tc(qkv, dout, lse, delta, dq_acc, dqkv, batch, seq, heads, head_dim, st);
    attn_dq_convert_kernel<<<static_cast<unsigned>((n / 8 + 255) / 256), 256, 0, st>>>(
        dq_acc, static_cast<__nv_bfloat16*>(dqkv), T, heads * head_dim);
}

}  // namespace bfpp
