// Host interface of the sm_100a bf16 GEMM (gemm_sm100.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace bfpp {

enum GemmEpilogue : int {
    GEMM_EPI_BF16 = 0,   // D = acc                                (bf16)
    GEMM_EPI_GELU = 1,   // aux_out = acc (bf16), D = gelu(aux_out) (bf16)
    GEMM_EPI_RESID = 2,  // D = acc + aux                          (bf16)
    GEMM_EPI_DGELU = 3,  // D = acc * gelu'(aux)                   (bf16)
    GEMM_EPI_F32 = 4,    // D (+)= acc                             (f32; accumulate flag)
};

struct GemmArgs {
    int64_t M = 0, N = 0, K = 0;
    const void* A = nullptr;  // bf16
    int64_t lda = 0;
    int a_mn_major = 0;       // 0: A is [M][lda] (K contiguous); 1: A is [K][lda] (M contiguous)
    const void* B = nullptr;  // bf16
    int64_t ldb = 0;
    int b_mn_major = 0;       // 0: B is [N][ldb]; 1: B is [K][ldb]
    void* D = nullptr;
    int64_t ldd = 0;
    const void* aux = nullptr;
    int64_t ldaux = 0;
    void* aux_out = nullptr;
    int64_t ldaux_out = 0;
    int epilogue = GEMM_EPI_BF16;
    int accumulate = 0;
};

void gemm_bf16(const GemmArgs& g, cudaStream_t stream);
extern int gemm_mode;
extern int gemm_sm_limit;  // > 0: persistent grids sized to this many SMs (SM partition of the launching stream)  // -1 auto (2-CTA tiles when M, N >= 256), 1 force 1-CTA, 2 force 2-CTA
void gemm_bf16_configure(int mode, int bn2, int stream_k);
// Two independent GEMMs (same operand majors) in one grouped 2-CTA launch when eligible, else two launches.
void gemm_bf16_pair(const GemmArgs& a, const GemmArgs& b, cudaStream_t st);
bool gemm_pairable(const GemmArgs& a, const GemmArgs& b);  // one grouped launch (else two)
extern int gemm_pair;  // grouped pair launches (default 1; BFPP_GEMM_PAIR=0 disables)  // overrides the environment defaults
extern int gemm_bn2;   // 2-CTA pair-tile width: 0 default (256), 128 opt-in
extern int gemm_pdl;   // programmatic dependent launch of the GEMM kernels (default 0, BFPP_GEMM_PDL=1)
extern int gemm_sk;    // stream-K in the 2-CTA kernel: -1 auto, 0 off, 1 forced (BFPP_GEMM_SK)
extern int gemm_dyn;   // dynamic tile schedule in the 2-CTA kernel (default 0, BFPP_GEMM_DYN=1)

// Host-side launch counters per kernel variant (process-wide, reset by bfpp_kernel_variant_reset):
// lets the composed-step parity tests assert which production paths actually ran.
enum KernelVariant : int {
    KV_GEMM_1CTA = 0,     // gemm_kernel (128 x BN tiles)
    KV_GEMM_2CTA,         // gemm2_kernel, one problem (256 x 256 cta_group::2 tiles)
    KV_GEMM_2CTA_PAIR,    // gemm2_kernel, two problems in one grouped launch
    KV_GEMM_2CTA_NFAST,   // gemm2 launch with the N-fastest tile raster
    KV_GEMM_2CTA_STREAMK, // gemm2 launch with stream-K ranges
    KV_ATTN_FWD_MULTI,    // attention forward with > 1 head and > 1 query block
    KV_ATTN_BWD_MULTI,    // attention backward with > 1 head and > 1 key block
    KV_N
};
void count_variant(int v);

// 2-D TMA descriptor over a row-major [rows][ld] matrix (bf16, or f32 if `f32`) with `inner`
// valid columns; box = {128 bytes of the inner dimension, box_rows}, SWIZZLE_128B, OOB -> 0.
CUtensorMap make_tma_2d(const void* ptr, int64_t inner, int64_t rows, int64_t ld, int box_rows, bool f32);

}  // namespace bfpp
