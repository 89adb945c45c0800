// extern "C" entry points of the device kernels (include/bfpp.h, kernel section).
#include <cuda_runtime.h>

#include <atomic>
#include <stdexcept>
#include <string>

#include "../../../include/bfpp.h"
#include "../sched/capi_util.hpp"
#include "gemm.hpp"
#include "kernels.hpp"

using namespace bfpp;

namespace {
std::atomic<int64_t> g_variant_count[KV_N];
}  // namespace
void bfpp::count_variant(int v) {
    if (v >= 0 && v < KV_N) g_variant_count[v].fetch_add(1, std::memory_order_relaxed);
}

namespace {
void check_launch() {
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA launch failed: ") + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

int64_t bfpp_kernel_variant_count(int32_t v) {
    return v >= 0 && v < KV_N ? g_variant_count[v].load(std::memory_order_relaxed) : -1;
}
void bfpp_kernel_variant_reset(void) {
    for (auto& c : g_variant_count) c.store(0, std::memory_order_relaxed);
}

int bfpp_gemm_config(int32_t mode, int32_t bn2, int32_t stream_k) {
    return guarded([&] {
        if (mode != -1 && mode != 1 && mode != 2) throw SpecError("gemm_config: mode must be -1, 1 or 2");
        if (bn2 != 0 && bn2 != 128 && bn2 != 256) throw SpecError("gemm_config: bn2 must be 0, 128 or 256");
        if (stream_k < -1 || stream_k > 1) throw SpecError("gemm_config: stream_k must be -1, 0 or 1");
        bfpp::gemm_bf16_configure(mode, bn2, stream_k);
    });
}

int bfpp_gemm_schedule(int32_t dynamic) {
    return guarded([&] {
        if (dynamic != 0 && dynamic != 1) throw SpecError("gemm_schedule: dynamic must be 0 or 1");
        bfpp::gemm_dyn = dynamic;
    });
}

int bfpp_attention_config(int32_t fwd_tiles) {
    return guarded([&] {
        if (fwd_tiles < 0 || fwd_tiles > 2) throw SpecError("attention_config: fwd_tiles must be 0, 1 or 2");
        bfpp::attn_fwd_tiles = fwd_tiles;
    });
}

int bfpp_gemm_sm_limit(int32_t n) {
    return guarded([&] {
        if (n < 0) throw SpecError("gemm_sm_limit: must be >= 0 (0 = all SMs)");
        bfpp::gemm_sm_limit = n;
    });
}

namespace {
GemmArgs to_gemm(const bfpp_gemm_args* a) {
    GemmArgs g;
    g.M = a->M;
    g.N = a->N;
    g.K = a->K;
    g.A = a->A;
    g.lda = a->lda;
    g.a_mn_major = a->a_mn_major;
    g.B = a->B;
    g.ldb = a->ldb;
    g.b_mn_major = a->b_mn_major;
    g.D = a->D;
    g.ldd = a->ldd;
    g.aux = a->aux;
    g.ldaux = a->ldaux;
    g.aux_out = a->aux_out;
    g.ldaux_out = a->ldaux_out;
    g.epilogue = a->epilogue;
    g.accumulate = a->accumulate;
    return g;
}
}  // namespace

int bfpp_gemm_bf16(const bfpp_gemm_args* a, void* stream) {
    return guarded([&] {
        gemm_bf16(to_gemm(a), static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

int bfpp_gemm_bf16_pair(const bfpp_gemm_args* a, const bfpp_gemm_args* b, void* stream) {
    return guarded([&] {
        gemm_bf16_pair(to_gemm(a), to_gemm(b), static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

}  // extern "C"

extern "C" {

int bfpp_attention_fwd(const void* qkv, void* o, float* lse, int32_t batch, int32_t seq, int32_t heads,
                       int32_t head_dim, void* stream) {
    return guarded([&] {
        attention_fwd(qkv, o, lse, batch, seq, heads, head_dim, static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

int bfpp_attention_bwd(const void* qkv, const void* o, const void* dout, const float* lse, float* delta,
                       float* dq_acc, void* dqkv, int32_t batch, int32_t seq, int32_t heads, int32_t head_dim,
                       void* stream) {
    return guarded([&] {
        attention_bwd(qkv, o, dout, lse, delta, dq_acc, dqkv, batch, seq, heads, head_dim,
                      static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

int bfpp_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, float* mean, float* rstd,
                       int32_t rows, int32_t width, float eps, void* stream) {
    return guarded([&] {
        layernorm_fwd(x, gamma, beta, y, mean, rstd, rows, width, eps, static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

int bfpp_layernorm_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
                       const void* dres, void* dx, float* dgamma, float* dbeta, int32_t rows, int32_t width,
                       void* stream) {
    return guarded([&] {
        layernorm_bwd(dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, rows, width,
                      static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

int bfpp_embed_fwd(const int32_t* tok, const void* wte, const void* wpe, void* x, int32_t T, int32_t S, int32_t h,
                   void* stream) {
    return guarded([&] {
        embed_fwd(tok, wte, wpe, x, T, S, h, static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

int bfpp_embed_bwd(const int32_t* tok, const void* dx, float* dwte, float* dwpe, int32_t T, int32_t S, int32_t h,
                   void* stream) {
    return guarded([&] {
        embed_bwd(tok, dx, dwte, dwpe, T, S, h, static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

int bfpp_softmax_xent(void* logits, int64_t ld, const int32_t* labels, float* row_loss, int32_t T, int32_t V,
                      float grad_scale, void* stream) {
    return guarded([&] {
        softmax_xent(logits, ld, labels, row_loss, T, V, grad_scale, static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

int bfpp_adam_update(float* p, float* m, float* v, float* g, void* w16, int64_t n, float lr, float beta1,
                     float beta2, float eps, float weight_decay, int32_t step, int32_t zero_grad, void* stream) {
    return guarded([&] {
        adam_update(p, m, v, g, w16, n, lr, beta1, beta2, eps, weight_decay, step, zero_grad,
                    static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

}  // extern "C"
