// Standalone sweep of Adam kernel variants (bandwidth alone): nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int ILP, bool CS>
__global__ void __launch_bounds__(256, 2) adam_v(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                                                 const float* __restrict__ g, __nv_bfloat16* __restrict__ w, long n4,
                                                 float lr, float b1, float b2, float eps, float bc1, float bc2) {
    const long stride = (long)gridDim.x * blockDim.x;
    for (long base = (long)blockIdx.x * blockDim.x + threadIdx.x; base < n4; base += stride * ILP) {
        float4 P[ILP], M[ILP], V[ILP], G[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            long i = base + u * stride;
            if (i < n4) {
                if (CS) {
                    P[u] = __ldcs((const float4*)p + i); M[u] = __ldcs((const float4*)m + i);
                    V[u] = __ldcs((const float4*)v + i); G[u] = __ldcs((const float4*)g + i);
                } else {
                    P[u] = ((const float4*)p)[i]; M[u] = ((const float4*)m)[i];
                    V[u] = ((const float4*)v)[i]; G[u] = ((const float4*)g)[i];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < ILP; ++u) {
            long i = base + u * stride;
            if (i >= n4) continue;
            float* pp = &P[u].x; float* mm = &M[u].x; float* vv = &V[u].x; const float* gg = &G[u].x;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                mm[k] = b1 * mm[k] + (1.f - b1) * gg[k];
                vv[k] = b2 * vv[k] + (1.f - b2) * gg[k] * gg[k];
                pp[k] -= lr * ((mm[k] / bc1) / (sqrtf(vv[k] / bc2) + eps));
            }
            __nv_bfloat162 lo = __floats2bfloat162_rn(P[u].x, P[u].y), hi = __floats2bfloat162_rn(P[u].z, P[u].w);
            uint2 o; o.x = *(uint32_t*)&lo; o.y = *(uint32_t*)&hi;
            if (CS) {
                __stcs((float4*)p + i, P[u]); __stcs((float4*)m + i, M[u]); __stcs((float4*)v + i, V[u]);
                __stcs((uint2*)w + i, o);
            } else {
                ((float4*)p)[i] = P[u]; ((float4*)m)[i] = M[u]; ((float4*)v)[i] = V[u]; ((uint2*)w)[i] = o;
            }
        }
    }
}


template <int ILP, int NT>
__global__ void __launch_bounds__(NT) adam_bc(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                                              const float* __restrict__ g, __nv_bfloat16* __restrict__ w, long n4,
                                              float lr, float b1, float b2, float eps, float bc1, float bc2) {
    const long base = (long)blockIdx.x * NT * ILP + threadIdx.x;
    float4 P[ILP], M[ILP], V[ILP], G[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
        long i = base + u * NT;
        if (i < n4) {
            P[u] = ((const float4*)p)[i]; M[u] = ((const float4*)m)[i];
            V[u] = ((const float4*)v)[i]; G[u] = ((const float4*)g)[i];
        }
    }
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
        long i = base + u * NT;
        if (i >= n4) continue;
        float* pp = &P[u].x; float* mm = &M[u].x; float* vv = &V[u].x; const float* gg = &G[u].x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            mm[k] = b1 * mm[k] + (1.f - b1) * gg[k];
            vv[k] = b2 * vv[k] + (1.f - b2) * gg[k] * gg[k];
            pp[k] -= lr * ((mm[k] / bc1) / (sqrtf(vv[k] / bc2) + eps));
        }
        __nv_bfloat162 lo = __floats2bfloat162_rn(P[u].x, P[u].y), hi = __floats2bfloat162_rn(P[u].z, P[u].w);
        uint2 o; o.x = *(uint32_t*)&lo; o.y = *(uint32_t*)&hi;
        ((float4*)p)[i] = P[u]; ((float4*)m)[i] = M[u]; ((float4*)v)[i] = V[u]; ((uint2*)w)[i] = o;
    }
}

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, long n4) {
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) b[i] = a[i];
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 10;
}

int main() {
    const long n = 300L << 20, n4 = n / 4;
    float *p, *m, *v, *g; __nv_bfloat16* w;
    cudaMalloc(&p, n * 4); cudaMalloc(&m, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&g, n * 4); cudaMalloc(&w, n * 2);
    cudaMemset(p, 0, n * 4); cudaMemset(m, 0, n * 4); cudaMemset(v, 0, n * 4); cudaMemset(g, 0, n * 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double bytes = 30.0 * n;
    float t = timeit([&] { copy_k<<<sms * 8, 256>>>((const float4*)p, (float4*)m, n4); });
    printf("copy f32 %.0f GB/s\n", 8.0 * n / t / 1e6);
#define RUN(ILP, CS, GRID, NAME) { long grid = GRID; float t = timeit([&] { adam_v<ILP, CS><<<grid, 256>>>(p, m, v, g, w, n4, 1e-4f, .9f, .95f, 1e-8f, .1f, .05f); }); \
    printf("%-28s ILP %d cs %d grid %8ld: %.0f GB/s\n", NAME, ILP, (int)CS, grid, bytes / t / 1e6); }
    RUN(4, true, (n4 + 1023) / 1024, "short-lived");
    RUN(4, false, (n4 + 1023) / 1024, "short-lived");
    RUN(2, true, (n4 + 511) / 512, "short-lived");
    RUN(2, false, (n4 + 511) / 512, "short-lived");
    RUN(1, false, (n4 + 255) / 256, "short-lived");
    RUN(4, true, sms * 2, "persistent 2/SM");
    RUN(4, false, sms * 2, "persistent 2/SM");
    RUN(2, false, sms * 4, "persistent 4/SM");
    RUN(8, false, (n4 + 2047) / 2048, "short-lived");
#define RUNBC(ILP, NT) { long grid = (n4 + NT * ILP - 1) / (NT * ILP); float t = timeit([&] { adam_bc<ILP, NT><<<grid, NT>>>(p, m, v, g, w, n4, 1e-4f, .9f, .95f, 1e-8f, .1f, .05f); }); \
    printf("block-contiguous ILP %d NT %d: %.0f GB/s\n", ILP, NT, bytes / t / 1e6); }
    RUNBC(1, 256) RUNBC(2, 256) RUNBC(4, 256) RUNBC(8, 256) RUNBC(1, 512) RUNBC(2, 512) RUNBC(4, 128) RUNBC(2, 128) RUNBC(1, 1024)
    return 0;
}
