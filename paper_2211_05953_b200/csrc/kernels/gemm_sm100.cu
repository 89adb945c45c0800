// Persistent warp-specialised bf16 GEMM for sm_100a: TMA -> SMEM (SWIZZLE_128B)
// -> tcgen05.mma (accumulator in TMEM, double-buffered) -> fused epilogue ->
// SMEM staging -> TMA store (or TMA reduce-add for f32 gradient accumulation).
//
//   D[M,N] = sum_k A[m,k] * B[n,k]      (f32 accumulate)
//
// A is either K-major (row-major [M][lda]) or MN-major (row-major [K][lda], i.e.
// A^T stored); likewise B ([N][ldb] or [K][ldb]). The three transformer GEMM
// forms are then: forward X.W^T (K,K), data-grad dY.W (K,MN) and weight-grad
// dY^T.X (MN,MN), with no explicit transposes.
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = MMA issuer (+ TMEM
// owner), warps 2..9 = epilogue. Epilogue warp w reads TMEM lane quarter w % 4
// and every other 128-byte column strip of the tile ("half" = (w - 2) / 4).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>

#include "gemm.hpp"
#include "sm100_ptx.cuh"

namespace bfpp {

// ---- host side -----------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return fn;
}

namespace {
CUtensorMap encode_tma_2d(const void* ptr, int64_t inner, int64_t rows, int64_t ld, int box_rows, bool f32);
}  // namespace

// 2-D tensor map over a row-major [rows][ld] matrix with `inner` valid columns;
// box = {128 B of inner, box_rows}, SWIZZLE_128B, OOB loads -> zero, OOB stores dropped.
// Cached by (address, shape, box): the executor's buffers are persistent, so every launch of a step
// after the first reuses its descriptors instead of encoding ~3 per GEMM launch on the host.
CUtensorMap make_tma_2d(const void* ptr, int64_t inner, int64_t rows, int64_t ld, int box_rows, bool f32) {
    using Key = std::tuple<const void*, int64_t, int64_t, int64_t, int, bool>;
    static std::mutex mu;
    static std::map<Key, CUtensorMap> cache;
    const Key k{ptr, inner, rows, ld, box_rows, f32};
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(k);
    if (it != cache.end()) return it->second;
    if (cache.size() >= 8192) cache.clear();  // bounded (tests allocate many short-lived buffers)
    const CUtensorMap m = encode_tma_2d(ptr, inner, rows, ld, box_rows, f32);
    cache.emplace(k, m);
    return m;
}

namespace {
CUtensorMap encode_tma_2d(const void* ptr, int64_t inner, int64_t rows, int64_t ld, int box_rows, bool f32) {
    CUtensorMap m;
    const int esz = f32 ? 4 : 2;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esz)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                             const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}
}  // namespace


namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStageBytesOut = 32 * 128;  // one [32 rows x 128 B] TMA store box per epilogue warp

__device__ __forceinline__ float gelu_f(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    return 0.5f * x * (1.f + ptx::tanh_fast(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float dgelu_f(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float t = ptx::tanh_fast(k0 * (x + k1 * x * x * x));
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

struct EpiArgs {
    const __nv_bfloat16* aux;  // residual / gelu pre-activation input
    int64_t ldaux;
    __nv_bfloat16* aux_out;    // gelu pre-activation output
    int64_t ldaux_out;
    int epi;
    int accumulate;
    int n_fast = 0;  // 2-CTA kernel: tile raster with N fastest (A is reused by the pairs of a wave)
};

// Stream-K (2-CTA kernel; opt-in, BFPP_GEMM_SK=1 / bfpp_gemm_config): correct and tested, but
// measured 15-90 % slower than data-parallel tiles on the step's shapes (scripts/gemm_sk_check.py):
// the owner's partial reads/writes are latency-bound at the very end of every pair's range.
// The (tile, k-block) iteration space is split into one contiguous
// range per CTA pair, so every pair does the same number of MMA k-blocks (no partially filled
// last wave). A tile whose k-blocks straddle ranges is finished by the pair holding its last
// k-block (the "owner"); the other pairs ("producers") write their f32 partial accumulators to
// a workspace slot and publish a flag. Each pair walks its range backwards, so its producer
// segment (the end of its range) is published first and its owner segment (the start) is
// drained last: an owner never waits on a pair that is itself still waiting.
struct SkArgs {
    float* ws;    // [pair][cta][128][256] f32 partials (nullptr: data-parallel tiles)
    int* flags;   // [pair][cta] epoch of the last published partial
    int epoch;
    // dynamic tile scheduler (data-parallel tiles): a pair's first tile is its index, every later
    // tile is n_pairs + (atomicAdd(tctr, 1) - tbase); nullptr = static t += n_pairs schedule
    unsigned long long* tctr;
    unsigned long long tbase;
};

struct Seg {
    int tile, kb0, kb1;
};

// Second problem of a grouped launch (two independent GEMMs with the same operand majors, e.g.
// the weight gradients of fc2 and fc1): its tiles follow the first problem's in one persistent
// tile space, so the pair fills the SM pairs' waves together and pays one prologue.
struct Second {
    CUtensorMap A, B, D;
    int M, N, K;
    EpiArgs ep;
};

struct WorkIter {
    bool sk;
    int t, step, num_tiles, nk;  // data-parallel: tiles t, t + step, ...
    long long u0, u;             // stream-K: this pair's range [u0, u1), walked down from u1
    __device__ WorkIter(bool sk_, int pair, int n_pairs, int num_tiles_, int nk_)
        : sk(sk_), t(pair), step(n_pairs), num_tiles(num_tiles_), nk(nk_) {
        const long long total = static_cast<long long>(num_tiles_) * nk_;
        u0 = total * pair / n_pairs;
        u = total * (pair + 1) / n_pairs;
    }
    __device__ bool next(Seg& g) {
        if (!sk) {
            if (t >= num_tiles) return false;
            g = {t, 0, nk};
            t += step;
            return true;
        }
        if (u <= u0) return false;
        const int tile = static_cast<int>((u - 1) / nk);
        const long long ts = static_cast<long long>(tile) * nk;
        const long long lo = u0 > ts ? u0 : ts;
        g = {tile, static_cast<int>(lo - ts), static_cast<int>(u - ts)};
        u = lo;
        return true;
    }
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int BN>
struct Smem {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kOutOffset = kStages * kStageBytes;
    static constexpr int kBarOffset = kOutOffset + kEpiWarps * kStageBytesOut;
    static constexpr int kBytes = kBarOffset + 256 + 1024;  // barriers + alignment slack
};

__device__ __forceinline__ void load_row32_bf16(const __nv_bfloat16* p, int valid, float (&v)[32]) {
    if (valid >= 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            uint4 raw = *reinterpret_cast<const uint4*>(p + j);
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float2 f = __bfloat1622float2(h[u]);
                v[j + 2 * u] = f.x;
                v[j + 2 * u + 1] = f.y;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = j < valid ? __bfloat162float(p[j]) : 0.f;
    }
}

// One 128-byte column strip of a warp's 32 accumulator rows: TMEM -> registers -> fused op ->
// swizzled staging row at `rowa`. Works in 32-column halves so the epilogue stays within the
// kernel's 104-register budget (which leaves room on the SM for another stream's block).
// `release` runs right after this warp's last TMEM read of the tile when `last` is set.
// n_parts stream-K partials (f32 rows, already offset to this strip's first column) are added
// to the accumulator before the fused op.
__device__ __forceinline__ void add_part(float (&v)[32], const float* part) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        const float4 w = __ldcg(reinterpret_cast<const float4*>(part + j));
        v[j] += w.x;
        v[j + 1] += w.y;
        v[j + 2] += w.z;
        v[j + 3] += w.w;
    }
}

template <typename Release>
__device__ __forceinline__ void epilogue_strip(const EpiArgs& ep, uint32_t tcol, int row, int col0, int valid_all,
                                               uint32_t rowa, int lane, bool last, Release release,
                                               const float* part0, const float* part1) {
    if (ep.epi == GEMM_EPI_F32) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tcol, r);
        ptx::tmem_ld_wait();
        if (last) release();
        if (part0) {
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            add_part(v, part0);
            if (part1) add_part(v, part1);
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(v[j]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
            ptx::st_shared_v4(rowa + ((c ^ (lane & 7)) << 4), r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
        return;
    }
    const bool need_aux = (ep.epi == GEMM_EPI_RESID || ep.epi == GEMM_EPI_DGELU);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int valid = max(0, min(32, valid_all - 32 * h));
        float a[32];
        // issue the aux loads before the TMEM load so both latencies overlap
        if (need_aux) {
            if (valid > 0) {
                load_row32_bf16(ep.aux + static_cast<int64_t>(row) * ep.ldaux + col0 + 32 * h, valid, a);
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) a[j] = 0.f;
            }
        }
        float v[32];
        {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(tcol + 32 * h, r);
            ptx::tmem_ld_wait();
            if (h == 1 && last) release();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        }
        if (part0) {
            add_part(v, part0 + 32 * h);
            if (part1) add_part(v, part1 + 32 * h);
        }
        if (ep.epi == GEMM_EPI_RESID) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += a[j];
        } else if (ep.epi == GEMM_EPI_DGELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= dgelu_f(a[j]);
        } else if (ep.epi == GEMM_EPI_GELU) {
            // pre-activation stored as bf16; gelu evaluated on the stored value
            __nv_bfloat16* pre = ep.aux_out + static_cast<int64_t>(row) * ep.ldaux_out + col0 + 32 * h;
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
                uint4 o;
                __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    hh[u] = __floats2bfloat162_rn(v[j + 2 * u], v[j + 2 * u + 1]);
                    const float2 f = __bfloat1622float2(hh[u]);
                    v[j + 2 * u] = gelu_f(f.x);
                    v[j + 2 * u + 1] = gelu_f(f.y);
                }
                if (valid >= j + 8) {
                    *reinterpret_cast<uint4*>(pre + j) = o;
                } else {
                    for (int u = 0; u < 8; ++u)
                        if (j + u < valid) pre[j + u] = reinterpret_cast<__nv_bfloat16*>(&o)[u];
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint4 o;
            __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int u = 0; u < 4; ++u) hh[u] = __floats2bfloat162_rn(v[8 * c + 2 * u], v[8 * c + 2 * u + 1]);
            ptx::st_shared_v4(rowa + (((4 * h + c) ^ (lane & 7)) << 4), o);
        }
    }
}

template <int BN, int A_MN, int B_MN>
__global__ void __maxnreg__(96)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, int M, int N, int K, EpiArgs ep) {
    using S = Smem<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int m_tiles = (M + BM - 1) / BM;
    const int n_tiles = (N + BN - 1) / BN;
    const int num_tiles = m_tiles * n_tiles;
    const int nk = (K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        ptx::tma_prefetch(&tmD);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], kEpiWarps);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<2 * BN>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: everything above overlapped the previous kernel's tail; inputs/outputs are touched below
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                const int m0 = (t % m_tiles) * BM, n0 = (t / m_tiles) * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * S::kStageBytes;
                    uint8_t* sb = sa + S::kABytes;
                    ptx::mbar_expect_tx(&full[stage], S::kStageBytes);
                    const int k0 = kb * BK;
                    if (A_MN) {
#pragma unroll
                        for (int i = 0; i < BM / 64; ++i)
                            ptx::tma_load_2d(sa + i * 64 * BK * 2, &tmA, &full[stage], m0 + 64 * i, k0);
                    } else {
                        ptx::tma_load_2d(sa, &tmA, &full[stage], k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int i = 0; i < BN / 64; ++i)
                            ptx::tma_load_2d(sb + i * 64 * BK * 2, &tmB, &full[stage], n0 + 64 * i, k0);
                    } else {
                        ptx::tma_load_2d(sb, &tmB, &full[stage], k0, n0);
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer =====
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t sa = ptx::smem_u32(smem + stage * S::kStageBytes);
                    const uint32_t sb = sa + S::kABytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // K-major: advance 32 B inside the 128 B swizzle row; MN-major: 16 K-rows of 128 B.
                        const uint64_t ad = A_MN ? ptx::sdesc_sw128(sa + k * 2048, 64 * BK * 2, 1024)
                                                 : ptx::sdesc_sw128(sa + k * 32, 16, 1024);
                        const uint64_t bd = B_MN ? ptx::sdesc_sw128(sb + k * 2048, 64 * BK * 2, 1024)
                                                 : ptx::sdesc_sw128(sb + k * 32, 16, 1024);
                        ptx::umma_f16(d_tmem, ad, bd, idesc, (kb | k) != 0);
                    }
                    ptx::umma_commit(&empty[stage]);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::umma_commit(&tfull[acc]);
            }
        }
    } else {
        // ===== epilogue: TMEM -> registers -> fused op -> swizzled SMEM -> TMA store =====
        const int ew = warp - 2;
        const int q = warp & 3;        // TMEM lane quarter (hardware: warp id % 4)
        const int half = ew >> 2;      // which alternate 128-byte column strips this warp owns
        uint8_t* stage_out = smem + S::kOutOffset + ew * kStageBytesOut;
        const bool f32_out = ep.epi == GEMM_EPI_F32;
        const int cw = f32_out ? 32 : 64;  // tile columns per 128-byte strip
        const int n_strips = BN / cw;
        int it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            const int m0 = (t % m_tiles) * BM, n0 = (t / m_tiles) * BN;
            const int row = m0 + q * 32 + lane;
            const bool row_ok = row < M;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            for (int sidx = half; sidx < n_strips; sidx += 2) {
                const int col0 = n0 + sidx * cw;
                const uint32_t tcol = tmem_base + ((q * 32) << 16) + acc * BN + sidx * cw;
                const int valid = row_ok ? min(cw, N - col0) : 0;
                // staging buffer reuse: the previous TMA store must have finished reading it
                if (lane == 0) ptx::bulk_wait_read<0>();
                __syncwarp();
                const uint32_t rowa = ptx::smem_u32(stage_out) + lane * 128;
                epilogue_strip(ep, tcol, row, col0, valid, rowa, lane, sidx + 2 >= n_strips, [&] {
                    // this warp's last TMEM read of the tile: hand the accumulator back to the MMA warp
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
                }, nullptr, nullptr);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0 && col0 < N && m0 + q * 32 < M) {
                    if (f32_out && ep.accumulate)
                        ptx::tma_reduce_add_2d(&tmD, stage_out, col0, m0 + q * 32);
                    else
                        ptx::tma_store_2d(&tmD, stage_out, col0, m0 + q * 32);
                    ptx::bulk_commit();
                }
            }
        }
        if (lane == 0) ptx::bulk_wait<0>();
    }
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<2 * BN>(tmem_base);
}


// ===================================================================================
// 2-CTA variant (cta_group::2): a cluster of two CTAs on neighbouring SMs computes a 256 x 256
// tile; each CTA stages its own 128 rows of A and 128 rows (half the N extent) of B per
// k-block (32 KB instead of 48 KB per SM for the same flops per SM), the leader CTA issues
// tcgen05.mma.cta_group::2 (M = 256) over both CTAs' shared memory, and each CTA's TMEM holds
// its 128 x 256 half of the accumulator, drained by its own 8 epilogue warps.
// 5 stages: 197 KB + the 1 KB per-CTA reservation leaves room on the SM for an optimizer or NCCL
// block from another stream to run beside the GEMM CTA (6 stages filled the SM).
// BN = 128 (each CTA stages 64 rows of B, 24 KB/stage, 7 stages): opt-in variant (see gemm_bf16).
template <int BN>
struct Smem2 {
#ifndef BFPP_GEMM2_STAGES
#define BFPP_GEMM2_STAGES 5  // experiments build other depths (scripts/gemm_stages.sh)
#endif
    static constexpr int kStages = BN == 256 ? BFPP_GEMM2_STAGES : 7;
    static constexpr int kABytes = 128 * BK * 2;
    static constexpr int kBBytes = (BN / 2) * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kOutOffset = kStages * kStageBytes;
    static constexpr int kBarOffset = kOutOffset + kEpiWarps * kStageBytesOut;
    static constexpr int kBytes = kBarOffset + 256 + 1024;
};

// Per-CTA timing probe (scripts/gemm_trace.cu builds this file with BFPP_GEMM_TRACE): start and
// end (%globaltimer, ns), tiles drained and SM id of every CTA of the last gemm2 launch.
#ifdef BFPP_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[512][4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define GTRACE_START()                                             \
    if (threadIdx.x == 64) {                                       \
        unsigned smid;                                             \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));          \
        g_gemm_trace[blockIdx.x][0] = gtimer();                    \
        g_gemm_trace[blockIdx.x][3] = smid;                        \
    }
#define GTRACE_END(n)                                              \
    if (threadIdx.x == 64) {                                       \
        g_gemm_trace[blockIdx.x][1] = gtimer();                    \
        g_gemm_trace[blockIdx.x][2] = static_cast<unsigned long long>(n); \
    }
#else
#define GTRACE_START()
#define GTRACE_END(n)
#endif

template <int BN, int A_MN, int B_MN, bool SK, bool GROUP>
__global__ void __maxnreg__(96)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmD, int M, int N, int K, EpiArgs ep, SkArgs sk,
                 const __grid_constant__ Second p2) {
    using S = Smem2<BN>;
    constexpr int kStages2 = S::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
    uint64_t* empty = full + kStages2;
    uint64_t* tfull = empty + kStages2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    // dynamic schedule: a 4-deep ring of tile indices the leader's producer fills for the pair
    // (its own MMA and epilogue warps, the peer's producer and epilogue warps)
    uint64_t* tq_full = tempty + 3;
    uint64_t* tq_empty = tq_full + 4;
    int* tq = reinterpret_cast<int*>(tq_empty + 4);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int m_tiles0 = (M + 255) / 256;
    const int tiles0 = m_tiles0 * ((N + BN - 1) / BN);
    const int nk0 = (K + BK - 1) / BK;
    const int m_tiles1 = GROUP ? (p2.M + 255) / 256 : 1;
    const int nk1 = GROUP ? (p2.K + BK - 1) / BK : 1;
    const int num_tiles = tiles0 + (GROUP ? m_tiles1 * ((p2.N + BN - 1) / BN) : 0);
    const int nk = nk0;  // stream-K (never grouped) splits the first problem's k-blocks
    const bool use_sk = SK && !GROUP && BN == 256 && sk.ws != nullptr;  // stream-K instantiation only
    const bool dyn = !use_sk && sk.tctr != nullptr;
    // problem of global tile t: tensor maps, shape, epilogue, tile index within the problem
    struct Prob {
        const CUtensorMap *A, *B, *D;
        int M, N, nk, m_tiles, t;
        const EpiArgs* ep;
        int mi, ni;  // tile coordinates (raster: M fastest, or N fastest when A is the big operand)
    };
    auto prob = [&](int t) -> Prob {
        Prob p = (GROUP && t >= tiles0) ? Prob{&p2.A, &p2.B, &p2.D, p2.M, p2.N, nk1, m_tiles1, t - tiles0, &p2.ep, 0, 0}
                                        : Prob{&tmA, &tmB, &tmD, M, N, nk0, m_tiles0, t, &ep, 0, 0};
        if (p.ep->n_fast) {
            const int nt = (p.N + BN - 1) / BN;
            p.mi = p.t / nt;
            p.ni = p.t % nt;
        } else {
            p.mi = p.t % p.m_tiles;
            p.ni = p.t / p.m_tiles;
        }
        return p;
    };

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        ptx::tma_prefetch(&tmD);
        if (GROUP) {
            ptx::tma_prefetch(&p2.A);
            ptx::tma_prefetch(&p2.B);
            ptx::tma_prefetch(&p2.D);
        }
        for (int s = 0; s < kStages2; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], 2 * kEpiWarps);
        }
        for (int b = 0; b < 4; ++b) {
            ptx::mbar_init(&tq_full[b], 1);
            ptx::mbar_init(&tq_empty[b], 2 * kEpiWarps + 2);  // both CTAs' epilogue warps, MMA, peer producer
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc_2sm<2 * BN>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: everything above overlapped the previous kernel's tail; inputs/outputs are touched below
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();
    GTRACE_START();
    // tile-ring consumer: index of ring entry i (every consumer reads every entry once, in order)
    auto read_tile = [&](int i) -> int {
        const int slot = i & 3;
        ptx::mbar_wait_cluster(&tq_full[slot], (i >> 2) & 1);
        const int t = *reinterpret_cast<volatile int*>(&tq[slot]);
        // the slot is rewritten four tiles later; a release here would hold the MMA thread until
        // its in-flight MMAs drain
        ptx::mbar_arrive_cluster_relaxed(ptx::mapa_shared(ptx::smem_u32(&tq_empty[slot]), 0));
        return t;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer (both CTAs): own 128 rows of A and own 128-row half of B =====
            int stage = 0;
            uint32_t phase = 0;
            WorkIter wi(use_sk, pair, n_pairs, num_tiles, nk);
            Seg g;
            int qi = 0;
            unsigned long long fetched = 0;  // counter value drawn one tile ahead (latency hidden)
            // leader: take the next tile (static first tile, then the shared counter) and publish
            // it to both CTAs' rings; peer: read it from its own ring
            auto next = [&](Seg& sg) -> bool {
                if (!dyn) return wi.next(sg);
                int t;
                if (rank == 0) {
                    if (qi == 0) {
                        t = pair < num_tiles ? pair : num_tiles;
                    } else {
                        t = n_pairs + static_cast<int>(fetched - sk.tbase);
                        if (t > num_tiles) t = num_tiles;
                    }
                    // draw the following tile now; its value is first used at the next call
                    if (t < num_tiles) fetched = atomicAdd(sk.tctr, 1ull);
                    const int slot = qi & 3;
                    ptx::mbar_wait_cluster(&tq_empty[slot], ((qi >> 2) & 1) ^ 1);
                    tq[slot] = t;
                    ptx::st_shared_cluster_u32(ptx::mapa_shared(ptx::smem_u32(&tq[slot]), 1), static_cast<uint32_t>(t));
                    ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tq_full[slot]), 0));
                    ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tq_full[slot]), 1));
                    ++qi;
                } else {
                    t = read_tile(qi++);
                }
                if (t >= num_tiles) return false;
                sg = {t, 0, nk};
                return true;
            };
            while (next(g)) {
                const Prob pb = prob(g.tile);
                if (!use_sk) g.kb1 = pb.nk;
                const int m0 = pb.mi * 256 + 128 * rank, n0 = pb.ni * BN + (BN / 2) * rank;
                for (int kb = g.kb0; kb < g.kb1; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * S::kStageBytes;
                    uint8_t* sb = sa + S::kABytes;
                    if (rank == 0) ptx::mbar_expect_tx(&full[stage], 2 * S::kStageBytes);
                    const int k0 = kb * BK;
                    if (A_MN) {
#pragma unroll
                        for (int i = 0; i < 2; ++i)
                            ptx::tma_load_2d_2sm(sa + i * 64 * BK * 2, pb.A, &full[stage], m0 + 64 * i, k0);
                    } else {
                        ptx::tma_load_2d_2sm(sa, pb.A, &full[stage], k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int i = 0; i < BN / 128; ++i)
                            ptx::tma_load_2d_2sm(sb + i * 64 * BK * 2, pb.B, &full[stage], n0 + 64 * i, k0);
                    } else {
                        ptx::tma_load_2d_2sm(sb, pb.B, &full[stage], k0, n0);
                    }
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // ===== MMA issuer (leader CTA only) =====
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(256, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            WorkIter wi(use_sk, pair, n_pairs, num_tiles, nk);
            Seg g;
            auto next = [&](Seg& sg) -> bool {
                if (!dyn) return wi.next(sg);
                const int t = read_tile(it);
                if (t >= num_tiles) return false;
                sg = {t, 0, nk};
                return true;
            };
            for (; next(g); ++it) {
                if (!use_sk) g.kb1 = prob(g.tile).nk;
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = g.kb0; kb < g.kb1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t sa = ptx::smem_u32(smem + stage * S::kStageBytes);
                    const uint32_t sb = sa + S::kABytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t ad = A_MN ? ptx::sdesc_sw128(sa + k * 2048, 64 * BK * 2, 1024)
                                                 : ptx::sdesc_sw128(sa + k * 32, 16, 1024);
                        const uint64_t bd = B_MN ? ptx::sdesc_sw128(sb + k * 2048, 64 * BK * 2, 1024)
                                                 : ptx::sdesc_sw128(sb + k * 32, 16, 1024);
                        ptx::umma_f16_2sm(d_tmem, ad, bd, idesc, (kb != g.kb0) || k != 0);
                    }
                    ptx::umma_commit_2sm(&empty[stage], 0x3);
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::umma_commit_2sm(&tfull[acc], 0x3);
            }
        }
    } else {
        // ===== epilogue: TMEM -> registers -> fused op -> swizzled SMEM -> TMA store =====
        const int ew = warp - 2;
        const int q = warp & 3;        // TMEM lane quarter (hardware: warp id % 4)
        const int half = ew >> 2;      // which alternate 128-byte column strips this warp owns
        uint8_t* stage_out = smem + S::kOutOffset + ew * kStageBytesOut;
        int it = 0;
        const int lr = q * 32 + lane;  // this thread's accumulator row within the CTA's 128 rows
        WorkIter wi(use_sk, pair, n_pairs, num_tiles, nk);
        Seg g;
        auto next = [&](Seg& sg) -> bool {
            if (!dyn) return wi.next(sg);
            int t = 0;
            if (lane == 0) t = read_tile(it);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= num_tiles) return false;
            sg = {t, 0, nk};
            return true;
        };
        for (; next(g); ++it) {
            const Prob pb = prob(g.tile);
            if (!use_sk) g.kb1 = pb.nk;
            const EpiArgs& ep_t = *pb.ep;
            const CUtensorMap* td = pb.D;
            const bool f32_out = ep_t.epi == GEMM_EPI_F32;
            const int cw = f32_out ? 32 : 64;  // tile columns per 128-byte strip
            const int n_strips = BN / cw;
            const int t = pb.t;
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            const int m0 = pb.mi * 256 + 128 * rank, n0 = pb.ni * BN;
            const int row = m0 + q * 32 + lane;
            const bool row_ok = row < pb.M;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            auto release = [&] {
                // this warp's last TMEM read of the segment: hand the accumulator back to the MMA warp
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tempty[acc]), 0));
            };
            if (use_sk && g.kb1 < nk) {
                // ---- stream-K producer: f32 partial to this pair's workspace slot, then publish ----
                float* dst = sk.ws + ((static_cast<size_t>(pair) * 2 + rank) * 128 + lr) * 256;
                for (int sidx = half; sidx < BN / 32; sidx += 2) {
                    uint32_t r[32];
                    ptx::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * BN + sidx * 32, r);
                    ptx::tmem_ld_wait();
                    if (sidx + 2 >= BN / 32) release();
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        __stcg(reinterpret_cast<float4*>(dst + sidx * 32 + j),
                               make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                           __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
                }
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
                if (ew == 0 && lane == 0) st_release_gpu(sk.flags + pair * 2 + rank, sk.epoch);
                continue;
            }
            // ---- full tile, or stream-K owner: add the partials of the pairs before this one ----
            const float* part0 = nullptr;
            const float* part1 = nullptr;
            if (g.kb0 > 0) {
                // producers: pair - 1, and pair - 2 when pair - 1's range starts inside this tile
                const long long total = static_cast<long long>(num_tiles) * nk, ts = static_cast<long long>(t) * nk;
                const int q1 = pair - 1;
                while (ld_acquire_gpu(sk.flags + q1 * 2 + rank) != sk.epoch) {
                }
                part0 = sk.ws + ((static_cast<size_t>(q1) * 2 + rank) * 128 + lr) * 256;
                if (total * q1 / n_pairs > ts) {
                    const int q2 = pair - 2;
                    while (ld_acquire_gpu(sk.flags + q2 * 2 + rank) != sk.epoch) {
                    }
                    part1 = sk.ws + ((static_cast<size_t>(q2) * 2 + rank) * 128 + lr) * 256;
                }
            }
            for (int sidx = half; sidx < n_strips; sidx += 2) {
                const int col0 = n0 + sidx * cw;
                const uint32_t tcol = tmem_base + ((q * 32) << 16) + acc * BN + sidx * cw;
                const int valid = row_ok ? min(cw, pb.N - col0) : 0;
                // staging buffer reuse: the previous TMA store must have finished reading it
                if (lane == 0) ptx::bulk_wait_read<0>();
                __syncwarp();
                const uint32_t rowa = ptx::smem_u32(stage_out) + lane * 128;
                epilogue_strip(ep_t, tcol, row, col0, valid, rowa, lane, sidx + 2 >= n_strips, release,
                               part0 ? part0 + sidx * cw : nullptr, part1 ? part1 + sidx * cw : nullptr);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0 && col0 < pb.N && m0 + q * 32 < pb.M) {
                    if (f32_out && ep_t.accumulate)
                        ptx::tma_reduce_add_2d(td, stage_out, col0, m0 + q * 32);
                    else
                        ptx::tma_store_2d(td, stage_out, col0, m0 + q * 32);
                    ptx::bulk_commit();
                }
            }
        }
        if (lane == 0) ptx::bulk_wait<0>();
        GTRACE_END(it);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) ptx::tmem_dealloc_2sm<2 * BN>(tmem_base);
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    // persistent grids launched into an SM partition (green context) size to the partition
    return gemm_sm_limit > 0 && gemm_sm_limit < n ? gemm_sm_limit : n;
}

template <int BN, int A_MN, int B_MN>
void launch(const GemmArgs& g, cudaStream_t st) {
    CUtensorMap ta = A_MN ? make_tma_2d(g.A, g.M, g.K, g.lda, BK, false) : make_tma_2d(g.A, g.K, g.M, g.lda, BM, false);
    CUtensorMap tb = B_MN ? make_tma_2d(g.B, g.N, g.K, g.ldb, BK, false) : make_tma_2d(g.B, g.K, g.N, g.ldb, BN, false);
    const bool f32 = g.epilogue == GEMM_EPI_F32;
    CUtensorMap td = make_tma_2d(g.D, g.N, g.M, g.ldd, 32, f32);
    EpiArgs ep{static_cast<const __nv_bfloat16*>(g.aux), g.ldaux, static_cast<__nv_bfloat16*>(g.aux_out),
               g.ldaux_out, g.epilogue, g.accumulate};
    auto kern = gemm_kernel<BN, A_MN, B_MN>;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<BN>::kBytes);
        configured = true;
    }
    const int tiles = static_cast<int>(((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN));
    const int grid = tiles < num_sms() ? tiles : num_sms();
    count_variant(KV_GEMM_1CTA);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Smem<BN>::kBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = gemm_pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, ta, tb, td, static_cast<int>(g.M), static_cast<int>(g.N), static_cast<int>(g.K),
                       ep);
}

// Stream-K partial workspace, one per stream (GEMMs of one stream run in order; two streams
// never share a slot): [pairs][2 CTAs][128][256] f32 + [pairs][2] int flags, epochs per launch.
struct SkWorkspace {
    float* ws = nullptr;
    int* flags = nullptr;
    int epoch = 0;
};
SkWorkspace& sk_workspace(cudaStream_t st, int pairs) {
    static std::map<std::pair<int, cudaStream_t>, SkWorkspace> all;
    int dev = 0;
    cudaGetDevice(&dev);
    SkWorkspace& w = all[{dev, st}];
    if (!w.ws) {
        if (cudaMalloc(&w.ws, static_cast<size_t>(pairs) * 2 * 128 * 256 * sizeof(float)) != cudaSuccess ||
            cudaMalloc(&w.flags, static_cast<size_t>(pairs) * 2 * sizeof(int)) != cudaSuccess)
            throw std::runtime_error("gemm: stream-K workspace allocation failed");
        cudaMemset(w.flags, 0, static_cast<size_t>(pairs) * 2 * sizeof(int));
    }
    return w;
}

// Dynamic-schedule tile counter, one per (device, stream): a launch that fetches draws exactly
// `tiles` values from it (every pair's failing fetch included), so the host knows each launch's
// base without resetting the counter. GEMMs of one stream run in order (PDL launches fetch only
// after griddepcontrol.wait), so launches never interleave on a counter.
struct TileCounter {
    unsigned long long* ctr = nullptr;
    unsigned long long next = 0;
};
TileCounter* tile_counter(cudaStream_t st) {
    static std::map<std::pair<int, cudaStream_t>, TileCounter> all;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return nullptr;  // a captured launch replays with a fixed base: static schedule
    int dev = 0;
    cudaGetDevice(&dev);
    TileCounter& c = all[{dev, st}];
    if (!c.ctr) {
        if (cudaMalloc(&c.ctr, sizeof(unsigned long long)) != cudaSuccess)
            throw std::runtime_error("gemm: tile counter allocation failed");
        cudaMemset(c.ctr, 0, sizeof(unsigned long long));
    }
    return &c;
}

template <int BN, int A_MN, int B_MN>
void launch2(const GemmArgs& g, cudaStream_t st, const GemmArgs* second = nullptr) {
    auto maps = [](const GemmArgs& a, CUtensorMap& ta, CUtensorMap& tb, CUtensorMap& td) {
        ta = A_MN ? make_tma_2d(a.A, a.M, a.K, a.lda, BK, false) : make_tma_2d(a.A, a.K, a.M, a.lda, 128, false);
        tb = B_MN ? make_tma_2d(a.B, a.N, a.K, a.ldb, BK, false) : make_tma_2d(a.B, a.K, a.N, a.ldb, BN / 2, false);
        td = make_tma_2d(a.D, a.N, a.M, a.ldd, 32, a.epilogue == GEMM_EPI_F32);
    };
    auto epi = [](const GemmArgs& a) {
        // N-fastest raster when A does not stay in L2 across the N passes (e.g. the LM-head weight
        // gradient, A = dlogits^T: 206 MB, read once instead of once per N tile)
        const bool n_fast = a.M * a.K * 2 > (int64_t(64) << 20) && a.N > BN;
        return EpiArgs{static_cast<const __nv_bfloat16*>(a.aux), a.ldaux, static_cast<__nv_bfloat16*>(a.aux_out),
                       a.ldaux_out, a.epilogue, a.accumulate, n_fast ? 1 : 0};
    };
    CUtensorMap ta, tb, td;
    maps(g, ta, tb, td);
    const EpiArgs ep = epi(g);
    Second p2{};
    if (second) {
        maps(*second, p2.A, p2.B, p2.D);
        p2.M = static_cast<int>(second->M);
        p2.N = static_cast<int>(second->N);
        p2.K = static_cast<int>(second->K);
        p2.ep = epi(*second);
    }
    static bool configured = false;
    if (!configured) {
        for (auto* k : {gemm2_kernel<BN, A_MN, B_MN, false, false>, gemm2_kernel<BN, A_MN, B_MN, true, false>,
                        gemm2_kernel<BN, A_MN, B_MN, false, true>})
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem2<BN>::kBytes);
        configured = true;
    }
    int tiles = static_cast<int>(((g.M + 255) / 256) * ((g.N + BN - 1) / BN));
    if (second) tiles += static_cast<int>(((second->M + 255) / 256) * ((second->N + BN - 1) / BN));
    const int nk = static_cast<int>((g.K + BK - 1) / BK);
    int pairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
    SkArgs sk{nullptr, nullptr, 0, nullptr, 0};
    {
        // stream-K when the data-parallel tile waves leave pairs idle and every pair's range is at
        // least half a tile (so a tile has at most two producers)
        const int all = num_sms() / 2;
        const long long total = static_cast<long long>(tiles) * nk;
        const int waves = (tiles + all - 1) / all;
        const double eff = static_cast<double>(tiles) / (static_cast<double>(waves) * all);
        const bool want = !second && (gemm_sk == 1 || (gemm_sk < 0 && eff < 0.92));
        if (want && BN == 256 && total / all >= (nk + 1) / 2 && nk >= 2) {
            SkWorkspace& w = sk_workspace(st, all);
            sk = SkArgs{w.ws, w.flags, ++w.epoch, nullptr, 0};
            pairs = all;
        }
    }
    // dynamic tiles (opt-in) when a pair runs more than one tile: a pair that starts late (its SMs
    // still busy with another stream's blocks) or runs slow takes fewer tiles. scripts/gemm_trace.py,
    // 2048 x 8192 x 2048 launched while the optimizer saturates the GPU: 1224 vs 969 TF/s (one
    // cluster of the static grid starts ~40 us late); alone 1425 vs 1535 TF/s (the tile ring costs
    // ~1 us per tile); in the N = 1 step GEMMs 1006 vs 1037 TF/s, so static stays the default.
    if (!sk.ws && gemm_dyn && tiles > pairs)
        if (TileCounter* c = tile_counter(st)) {
            sk.tctr = c->ctr;
            sk.tbase = c->next;
            c->next += static_cast<unsigned long long>(tiles);
        }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Smem2<BN>::kBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see griddep_wait)
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = gemm_pdl ? 2 : 1;
    const int M = static_cast<int>(g.M), N = static_cast<int>(g.N), K = static_cast<int>(g.K);
    count_variant(second ? KV_GEMM_2CTA_PAIR : KV_GEMM_2CTA);
    if (ep.n_fast || (second && p2.ep.n_fast)) count_variant(KV_GEMM_2CTA_NFAST);
    if (sk.ws) count_variant(KV_GEMM_2CTA_STREAMK);
    if (second)
        cudaLaunchKernelEx(&cfg, gemm2_kernel<BN, A_MN, B_MN, false, true>, ta, tb, td, M, N, K, ep, sk, p2);
    else if (sk.ws)
        cudaLaunchKernelEx(&cfg, gemm2_kernel<BN, A_MN, B_MN, true, false>, ta, tb, td, M, N, K, ep, sk, p2);
    else
        cudaLaunchKernelEx(&cfg, gemm2_kernel<BN, A_MN, B_MN, false, false>, ta, tb, td, M, N, K, ep, sk, p2);
}

}  // namespace

int gemm_sk = 0;     // stream-K for the 2-CTA kernel: 0 off (default), 1 forced, -1 auto (BFPP_GEMM_SK)
int gemm_mode = -1;  // -1 auto, 1 force 1-CTA, 2 force 2-CTA (benchmarks / tests)
int gemm_sm_limit = 0;  // > 0: persistent grids sized to this many SMs (a green-context partition)
int gemm_pdl = 0;    // programmatic dependent launch (BFPP_GEMM_PDL=1): measured no gain in-step (optimizer co-running)
int gemm_bn2 = 0;    // 2-CTA pair-tile width: 0 / 256 default, 128 opt-in (BFPP_GEMM_BN2; tests)
int gemm_pair = 1;   // grouped launches of independent GEMM pairs (BFPP_GEMM_PAIR=0: two launches)
int gemm_dyn = 0;    // dynamic tile schedule of the 2-CTA kernel (opt-in: BFPP_GEMM_DYN=1, bfpp_gemm_schedule)

static bool env_read = false;

void gemm_bf16_configure(int mode, int bn2, int stream_k) {
    env_read = true;
    gemm_mode = mode;
    gemm_bn2 = bn2;
    gemm_sk = stream_k;
}

static void read_env() {
    if (env_read) return;
    if (const char* e = getenv("BFPP_GEMM_MODE")) gemm_mode = atoi(e);
    if (const char* e = getenv("BFPP_GEMM_BN2")) gemm_bn2 = atoi(e);
    if (const char* e = getenv("BFPP_GEMM_PDL")) gemm_pdl = atoi(e);
    if (const char* e = getenv("BFPP_GEMM_SK")) gemm_sk = atoi(e);
    if (const char* e = getenv("BFPP_GEMM_PAIR")) gemm_pair = atoi(e);
    if (const char* e = getenv("BFPP_GEMM_DYN")) gemm_dyn = atoi(e);
    if (const char* e = getenv("BFPP_GEMM_SMS")) gemm_sm_limit = atoi(e);
    env_read = true;
}

void gemm_bf16(const GemmArgs& g, cudaStream_t st) {
    read_env();
    if (g.M <= 0 || g.N <= 0 || g.K <= 0) throw std::runtime_error("gemm: empty problem");
    if (g.K % 8 || g.lda % 8 || g.ldb % 8 || g.ldd % 8) throw std::runtime_error("gemm: K and leading dims must be multiples of 8");
    const bool small_n = g.N <= 128;
    const int a = g.a_mn_major ? 1 : 0, b = g.b_mn_major ? 1 : 0;
    const bool pair = gemm_mode == 2 || (gemm_mode < 0 && g.M >= 256 && g.N >= 256);
    if (pair) {
        // 256 x 128 pair tiles even out wave counts but measured 25-30 % slower per flop than
        // 256 x 256 on the 2048 x 8192 GEMMs (scripts/gemm_bench.py), so they are opt-in only
        const bool narrow = gemm_bn2 == 128;
        if (narrow) {
            if (a == 0 && b == 0) return launch2<128, 0, 0>(g, st);
            if (a == 0 && b == 1) return launch2<128, 0, 1>(g, st);
            if (a == 1 && b == 0) return launch2<128, 1, 0>(g, st);
            return launch2<128, 1, 1>(g, st);
        }
        if (a == 0 && b == 0) return launch2<256, 0, 0>(g, st);
        if (a == 0 && b == 1) return launch2<256, 0, 1>(g, st);
        if (a == 1 && b == 0) return launch2<256, 1, 0>(g, st);
        return launch2<256, 1, 1>(g, st);
    }
#define BFPP_GEMM_CASE(BN_, A_, B_) \
    if (a == A_ && b == B_) return launch<BN_, A_, B_>(g, st);
    if (small_n) {
        BFPP_GEMM_CASE(128, 0, 0)
        BFPP_GEMM_CASE(128, 0, 1)
        BFPP_GEMM_CASE(128, 1, 0)
        BFPP_GEMM_CASE(128, 1, 1)
    } else {
        BFPP_GEMM_CASE(256, 0, 0)
        BFPP_GEMM_CASE(256, 0, 1)
        BFPP_GEMM_CASE(256, 1, 0)
        BFPP_GEMM_CASE(256, 1, 1)
    }
#undef BFPP_GEMM_CASE
}

bool gemm_pairable(const GemmArgs& a, const GemmArgs& b) {
    read_env();
    const bool same = a.a_mn_major == b.a_mn_major && a.b_mn_major == b.b_mn_major;
    return gemm_pair && same && gemm_mode != 1 && gemm_bn2 != 128 && a.M >= 256 && a.N >= 256 && b.M >= 256 &&
           b.N >= 256;
}

void gemm_bf16_pair(const GemmArgs& a, const GemmArgs& b, cudaStream_t st) {
    if (!gemm_pairable(a, b)) {
        gemm_bf16(a, st);
        gemm_bf16(b, st);
        return;
    }
    for (const GemmArgs* g : {&a, &b}) {
        if (g->M <= 0 || g->N <= 0 || g->K <= 0) throw std::runtime_error("gemm: empty problem");
        if (g->K % 8 || g->lda % 8 || g->ldb % 8 || g->ldd % 8)
            throw std::runtime_error("gemm: K and leading dims must be multiples of 8");
    }
    const int am = a.a_mn_major ? 1 : 0, bm = a.b_mn_major ? 1 : 0;
    if (am == 0 && bm == 0) return launch2<256, 0, 0>(a, st, &b);
    if (am == 0 && bm == 1) return launch2<256, 0, 1>(a, st, &b);
    if (am == 1 && bm == 0) return launch2<256, 1, 0>(a, st, &b);
    return launch2<256, 1, 1>(a, st, &b);
}

}  // namespace bfpp
