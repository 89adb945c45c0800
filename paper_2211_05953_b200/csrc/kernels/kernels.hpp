// Host interfaces of the HBM-bound and attention kernels (device pointers, async on `st`).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace bfpp {

// attention.cu — causal MHA, head_dim 128; qkv [B*S][3*H*128], o [B*S][H*128], lse [B*H][S] (log2 domain)
void attention_fwd(const void* qkv, void* o, float* lse, int batch, int seq, int heads, int head_dim, cudaStream_t st);
// query tiles per forward CTA: 0 auto (two when there are >= 256 tile pairs), 1, 2
extern int attn_fwd_tiles;
// tcgen05/TMEM version of attention_fwd (attention_tc.cu); same inputs/outputs
void attention_fwd_tc(const void* qkv, void* o, float* lse, int batch, int seq, int heads, int head_dim,
                      cudaStream_t st);
void attention_bwd_tc(const void* qkv, const void* dout, const float* lse, const float* delta, float* dq_acc,
                      void* dqkv, int batch, int seq, int heads, int head_dim, cudaStream_t st);
// delta [B*H][S] and dq_acc [B*S][H*128] f32 are scratch; dqkv receives dQ, dK, dV.
void attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse, float* delta, float* dq_acc,
                   void* dqkv, int batch, int seq, int heads, int head_dim, cudaStream_t st);

// layernorm.cu
void layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd, int rows,
                   int width, float eps, cudaStream_t st);
void layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                   const void* dres, void* dx, float* dgamma, float* dbeta, int rows, int width, cudaStream_t st,
                   int accumulate = 1);
// kernel launches of one layernorm_bwd call at this width (register-resident paths: 2; generic: 3)
int layernorm_bwd_launches(int width);

// elementwise.cu
void embed_fwd(const int32_t* tok, const void* wte, const void* wpe, void* x, int T, int S, int h, cudaStream_t st);
void embed_bwd(const int32_t* tok, const void* dx, float* dwte, float* dwpe, int T, int S, int h, cudaStream_t st);
void softmax_xent(void* logits, int64_t ld, const int32_t* labels, float* row_loss, int T, int V, float grad_scale,
                  cudaStream_t st);
void adam_update(float* p, float* m, float* v, float* g, void* w16, int64_t n, float lr, float b1, float b2,
                 float eps, float wd, int step, int zero_grad, cudaStream_t st);
// Row-wise Adam over an embedding table (same math as adam_update): mark_rows marks the rows of
// `tok` in mark[rows] and lists them once each; adam_rows updates the listed rows (listed = 1) or
// every unmarked row (listed = 0)
void mark_rows(const int32_t* tok, int n, int32_t* mark, int32_t* list, int32_t* count, int64_t rows,
               cudaStream_t st);
void adam_rows(float* p, float* m, float* v, const float* g, void* w16, int64_t rows, int h, const int32_t* mark,
               const int32_t* list, const int32_t* count, int max_rows, int listed, float lr, float b1, float b2,
               float eps, float wd, int step, cudaStream_t st);
void init_normal(float* p, void* w16, int64_t n, float mean, float std, uint64_t seed, uint64_t offset,
                 cudaStream_t st);
void f32_to_bf16(const float* src, void* dst, int64_t n, cudaStream_t st);
void sum_f32(const float* x, int64_t n, float scale, float* out, int accumulate, cudaStream_t st);

}  // namespace bfpp
