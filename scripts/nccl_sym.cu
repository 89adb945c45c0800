// DP_FS collective microbenchmark on 2 GPUs of one box (single process, ncclCommInitAll):
// all-gather of bf16 weight shards and reduce-scatter of f32 gradients at the sizes of one
// GPT-1.3B stage, under four buffer / policy modes:
//   0 cudaMalloc buffers, default communicator (what the executor does today)
//   1 cudaMalloc buffers registered with ncclCommRegister (zero-copy P2P)
//   2 ncclMemAlloc buffers in symmetric windows, CTAPolicy default
//   3 ... CTAPolicy EFFICIENCY      4 ... CTAPolicy ZERO (copy-engine collectives where supported)
//   5 CTAPolicy ZERO, only the all-gather buffers in windows (reduce-scatter on plain cudaMalloc)
// For each: time alone, and the slowdown of a concurrent all-SM FMA kernel (the SMs the collective
// takes away from the compute stream).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/nccl_sym.cu -I$NCCL/include -L$NCCL/lib -l:libnccl.so.2
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <nccl.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
#define NK(x) do { ncclResult_t e = (x); if (e != ncclSuccess) { printf("NCCL %s @%d\n", ncclGetErrorString(e), __LINE__); exit(1); } } while (0)

__global__ void spin(float* out, int iters) {
    float a = threadIdx.x, b = 1.0001f;
    for (int i = 0; i < iters; ++i) a = fmaf(a, b, 1e-7f);
    if (a == -1.f) out[0] = a;
}

int main(int argc, char** argv) {
    const int ND = 2;
    const size_t n_ag = argc > 1 ? atol(argv[1]) : 75000000;  // bf16 elements per rank shard
    const size_t n_rs = n_ag;                                   // f32 elements per rank result
    int devs[ND] = {0, 1};
    const int m0 = argc > 2 ? atoi(argv[2]) : 0, m1 = argc > 2 ? m0 : 5;  // one mode per process: see below
    for (int mode = m0; mode <= m1; ++mode) {
        ncclComm_t comm[ND];
        if (mode < 2) {
            NK(ncclCommInitAll(comm, ND, devs));
        } else {
            ncclUniqueId id;
            NK(ncclGetUniqueId(&id));
            NK(ncclGroupStart());
            for (int d = 0; d < ND; ++d) {
                CK(cudaSetDevice(d));
                ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
                cfg.CTAPolicy = mode == 2 ? NCCL_CTA_POLICY_DEFAULT : mode == 3 ? NCCL_CTA_POLICY_EFFICIENCY
                                                                                : NCCL_CTA_POLICY_ZERO;
                NK(ncclCommInitRankConfig(&comm[d], ND, id, d, &cfg));
            }
            NK(ncclGroupEnd());
        }
        void *wsh[ND], *wfull[ND], *g[ND], *gsh[ND];
        const size_t b_wsh = n_ag * 2, b_wfull = n_ag * 2 * ND, b_g = n_rs * 4 * ND, b_gsh = n_rs * 4;
        std::vector<void*> regs;
        std::vector<ncclWindow_t> wins;
        for (int d = 0; d < ND; ++d) {
            CK(cudaSetDevice(d));
            if (mode >= 2) {
                NK(ncclMemAlloc(&wsh[d], b_wsh)); NK(ncclMemAlloc(&wfull[d], b_wfull));
                if (mode == 5) {
                    CK(cudaMalloc(&g[d], b_g)); CK(cudaMalloc(&gsh[d], b_gsh));
                } else {
                    NK(ncclMemAlloc(&g[d], b_g)); NK(ncclMemAlloc(&gsh[d], b_gsh));
                }
            } else {
                CK(cudaMalloc(&wsh[d], b_wsh)); CK(cudaMalloc(&wfull[d], b_wfull));
                CK(cudaMalloc(&g[d], b_g)); CK(cudaMalloc(&gsh[d], b_gsh));
            }
            CK(cudaMemset(wsh[d], 0, b_wsh)); CK(cudaMemset(g[d], 0, b_g));
        }
        if (mode == 1) {
            for (int d = 0; d < ND; ++d) {
                CK(cudaSetDevice(d));
                void* h;
                NK(ncclCommRegister(comm[d], wsh[d], b_wsh, &h)); regs.push_back(h);
                NK(ncclCommRegister(comm[d], wfull[d], b_wfull, &h)); regs.push_back(h);
                NK(ncclCommRegister(comm[d], g[d], b_g, &h)); regs.push_back(h);
                NK(ncclCommRegister(comm[d], gsh[d], b_gsh, &h)); regs.push_back(h);
            }
        }
        if (mode >= 2) {
            void** bufs[4] = {wsh, wfull, g, gsh};
            size_t sz[4] = {b_wsh, b_wfull, b_g, b_gsh};
            for (int k = 0; k < (mode == 5 ? 2 : 4); ++k) {
                NK(ncclGroupStart());
                for (int d = 0; d < ND; ++d) {
                    CK(cudaSetDevice(d));
                    ncclWindow_t w;
                    NK(ncclCommWindowRegister(comm[d], bufs[k][d], sz[k], &w, NCCL_WIN_COLL_SYMMETRIC));
                    wins.push_back(w);
                }
                NK(ncclGroupEnd());
            }
        }
        cudaStream_t cs[ND], ks[ND];
        cudaEvent_t e0[ND], e1[ND], k0[ND], k1[ND];
        float* junk[ND];
        for (int d = 0; d < ND; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaStreamCreateWithFlags(&cs[d], cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&ks[d], cudaStreamNonBlocking));
            CK(cudaEventCreate(&e0[d])); CK(cudaEventCreate(&e1[d]));
            CK(cudaEventCreate(&k0[d])); CK(cudaEventCreate(&k1[d]));
            CK(cudaMalloc(&junk[d], 16));
        }
        auto run = [&](int which, int reps) {
            for (int r = 0; r < reps; ++r) {
                NK(ncclGroupStart());
                for (int d = 0; d < ND; ++d) {
                    CK(cudaSetDevice(d));
                    if (which == 0)
                        NK(ncclAllGather(wsh[d], wfull[d], n_ag, ncclBfloat16, comm[d], cs[d]));
                    else
                        NK(ncclReduceScatter(g[d], gsh[d], n_rs, ncclFloat32, ncclSum, comm[d], cs[d]));
                }
                NK(ncclGroupEnd());
            }
        };
        const int spin_iters = 800000;  // longer than the 8 collectives
        for (int which = 0; which < 2; ++which) {
            run(which, 3);
            for (int d = 0; d < ND; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
            // alone
            for (int d = 0; d < ND; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], cs[d])); }
            run(which, 10);
            for (int d = 0; d < ND; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e1[d], cs[d])); }
            for (int d = 0; d < ND; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
            float ms = 0;
            CK(cudaSetDevice(0));
            CK(cudaEventElapsedTime(&ms, e0[0], e1[0]));
            const double us = ms * 100.0;
            const double bytes = which == 0 ? (double)n_ag * 2 * (ND - 1) : (double)n_rs * 4 * (ND - 1);
            // spin alone
            CK(cudaEventRecord(k0[0], ks[0]));
            spin<<<148 * 8, 256, 0, ks[0]>>>(junk[0], spin_iters);
            CK(cudaEventRecord(k1[0], ks[0]));
            CK(cudaDeviceSynchronize());
            float ks_alone = 0;
            CK(cudaEventElapsedTime(&ks_alone, k0[0], k1[0]));
            // spin with the collective looping beside it
            for (int d = 0; d < ND; ++d) { CK(cudaSetDevice(d)); }
            run(which, 8);
            CK(cudaSetDevice(0));
            CK(cudaEventRecord(k0[0], ks[0]));
            spin<<<148 * 8, 256, 0, ks[0]>>>(junk[0], spin_iters);
            CK(cudaEventRecord(k1[0], ks[0]));
            for (int d = 0; d < ND; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
            float ks_co = 0;
            CK(cudaEventElapsedTime(&ks_co, k0[0], k1[0]));
            printf("mode %d %s: %.1f us  %.1f GB/s per direction;  spin alone %.2f ms, beside %.2f ms (x%.3f)\n", mode,
                   which == 0 ? "all-gather    " : "reduce-scatter", us, bytes / us * 1e-3, ks_alone, ks_co,
                   ks_co / ks_alone);
            fflush(stdout);
        }
        for (int d = 0; d < ND; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
        if (mode >= 2) break;  // window teardown is left to process exit (run one symmetric mode per process)
        for (size_t i = 0; i < regs.size(); ++i) NK(ncclCommDeregister(comm[i / 4], regs[i]));
        for (int d = 0; d < ND; ++d) {
            CK(cudaSetDevice(d));
            cudaFree(wsh[d]); cudaFree(wfull[d]); cudaFree(g[d]); cudaFree(gsh[d]);
            NK(ncclCommDestroy(comm[d]));
        }
    }
    return 0;
}
