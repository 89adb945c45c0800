// Timeline probe of the attention backward kernel: builds attention_tc.cu with BFPP_ATTN_TRACE
// (clock64 stamps of one CTA's warp roles per query block) into scripts/libattntrace.so.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -cudart static \
//        scripts/attn_trace.cu paper_2211_05953_b200/csrc/kernels/attention.cu \
//        paper_2211_05953_b200/csrc/kernels/gemm_sm100.cu -o scripts/libattntrace.so -ldl
// and run scripts/attn_trace.py.
#define BFPP_ATTN_TRACE
#include "../paper_2211_05953_b200/csrc/kernels/attention_tc.cu"

extern "C" int trace_read(unsigned long long* out) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, bfpp::g_attn_trace, sizeof(bfpp::g_attn_trace)));
}
extern "C" int trace_clear() {
    static unsigned long long zero[8 * 64 * 16] = {};
    return static_cast<int>(cudaMemcpyToSymbol(bfpp::g_attn_trace, zero, sizeof(zero)));
}
extern "C" void trace_bwd(const void* qkv, const void* o, const void* dout, const float* lse, float* delta, float* dq,
                          void* dqkv, int B, int S, int H) {
    bfpp::attention_bwd(qkv, o, dout, lse, delta, dq, dqkv, B, S, H, 128, 0);
}
extern "C" void trace_fwd(const void* qkv, void* o, float* lse, int B, int S, int H) {
    bfpp::attention_fwd(qkv, o, lse, B, S, H, 128, 0);
}
namespace bfpp {
void count_variant(int) {}  // capi_kernels.cpp's launch counters are not part of this probe
}
