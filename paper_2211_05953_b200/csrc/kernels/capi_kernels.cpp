// extern "C" entry points of the device kernels (include/bfpp.h, kernel section).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../../include/bfpp.h"
#include "../sched/capi_util.hpp"
#include "gemm.hpp"
#include "kernels.hpp"

using namespace bfpp;

namespace {
void check_launch() {
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA launch failed: ") + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

int bfpp_gemm_bf16(const bfpp_gemm_args* a, void* stream) {
    return guarded([&] {
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
        gemm_bf16(g, static_cast<cudaStream_t>(stream));
        check_launch();
    });
}

}  // extern "C"
