// bf16 GEMM on the 5th-generation tensor cores (tcgen05, kind::f16 with bf16
// operands, fp32 accumulation in TMEM, fp32 output) with a fused epilogue, for
// the input projections of the bf16-I/O layers: S6 B_k / C_k / the low-rank
// delta projection (layers.py:1020-1027) and the RG-LRU gate projections
// (layers.py:1212-1218).
//
//   C[M, N] = act(alpha * A[M, K] . Bt[N, K]^T + bias[n]) + beta * Cin[M, N]
//   act in {identity, softplus (threshold 30, numerics.py:36-39), sigmoid}
//
// A and Bt bf16 row-major K-contiguous (A = activations, Bt = the weight as
// [out, in]); C / Cin fp32.  bf16 x bf16 products are exact in fp32, so the
// only rounding besides the operands' is the accumulation.
//
// CTA = 6 warps, persistent over 128 x BN output tiles (M fastest):
//   warp 0      TMA producer: k-blocks of 64 (128-byte rows, 128B swizzle =
//               the UMMA K-major SW128 canonical layout) of A and Bt into a
//               ring of stages
//   warp 1      MMA issuer (one thread; 4 UMMA k-steps of 16 per k-block)
//   warps 2..5  epilogue: tcgen05.ld of its 32 TMEM lanes (= rows) in chunks
//               of 32 columns, bias + activation (+ Cin, which lands by TMA
//               in the warp's 32 x 32 box first), one TMA store per box
// The accumulator is double-buffered in TMEM (2 x BN columns): the epilogue
// of tile i overlaps the mainloop of tile i + 1.
#include "lrx_host.h"
#include "lrx_tma.cuh"

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

namespace lrx {
namespace gemm16 {

constexpr int BM = 128;
constexpr int BK = 64;  // bf16 per 128-byte row
constexpr int THREADS = 192;

enum Act : int { ACT_NONE = 0, ACT_SOFTPLUS = 1, ACT_SIGMOID = 2 };

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    // K-major SWIZZLE_128B: 8-row groups of 128-byte rows = 1024 B (SBO), layout type 2
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

template <int BN>
__host__ __device__ constexpr uint32_t idesc_bf16() {
    // D F32 [4,6) = 1, A BF16 [7,10) = 1, B BF16 [10,13) = 1, K-major both,
    // N >> 3 at [17,23), M >> 4 at [24,29)
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     tma::smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ float act(float x, int a) {
    // MUFU forms (ex2 / lg2 / rcp, ~2 ulp): softplus keeps its relative
    // precision for e^x << 1 through the log1p series (as the S6 scan's
    // softplus); threshold 30 (numerics.py:36-39)
    if (a == 1) {
        float e, lg;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fminf(x, 30.f) * 1.4426950408889634f));
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(1.f + e));
        const float ser = e * (1.f - e * (0.5f - e * (1.f / 3.f)));
        return x > 30.f ? x : (e < 1e-2f ? ser : lg * 0.6931471805599453f);
    }
    if (a == 2) {
        float e, r;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-x * 1.4426950408889634f));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + e));
        return r;
    }
    return x;
}

template <int BN>
struct Lay {
    static constexpr int A = BM * BK * 2;  // 16 KB
    static constexpr int B = BN * BK * 2;
    static constexpr int STAGE = A + B;
    static constexpr int STAGES = BN >= 256 ? 4 : 6;
    static constexpr int EPI = 4 * 4096;  // one 32 x 32 fp32 box per epilogue warp
    static constexpr size_t smem() { return 2048 + (size_t)STAGES * STAGE + EPI; }
};

template <int BN, bool OB>  // OB: bf16 output (no Cin)
__global__ void __launch_bounds__(THREADS, 1) gemm_bf16_kernel(
    const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
    const __grid_constant__ CUtensorMap mC, const __grid_constant__ CUtensorMap mCin, const float* Cin,
    const float* __restrict__ bias, int M, int N, int K, float alpha, float beta, int act_kind) {
    using LY = Lay<BN>;
    constexpr int STAGES = LY::STAGES;
    constexpr int CW = BN < 32 ? BN : 32;  // epilogue box width (columns)
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base);  // [STAGES] TMA landed
    uint64_t* empty = full + STAGES;                     // [STAGES] MMAs done with the stage
    uint64_t* tfull = empty + STAGES;                    // [2] accumulator ready
    uint64_t* tempty = tfull + 2;                        // [2] accumulator drained
    uint64_t* cbar = tempty + 2;                         // [4] Cin box landed (per epilogue warp)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cbar + 4);
    unsigned char* stages = base + 1024;
    float* epi = reinterpret_cast<float*>(stages + STAGES * LY::STAGE);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (K + BK - 1) / BK;
    const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN, ntiles = tm * tn;
    constexpr uint32_t kCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;

    if (threadIdx.x == 0) {
        tma::prefetch_map(&mA);
        tma::prefetch_map(&mB);
        tma::prefetch_map(&mC);
        for (int i = 0; i < STAGES; ++i) {
            tma::mbar_init(&full[i], 1);
            tma::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tma::mbar_init(&tfull[i], 1);
            tma::mbar_init(&tempty[i], 128);
        }
        for (int i = 0; i < 4; ++i) tma::mbar_init(&cbar[i], 1);
        if (Cin) tma::prefetch_map(&mCin);
        tma::fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tma::smem_u32(tmem_slot)),
                     "r"(kCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------------------------------------- producer
            int it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int m0 = (tile % tm) * BM, n0 = (tile / tm) * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    if (it >= STAGES) tma::mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
                    unsigned char* sp = stages + st * LY::STAGE;
                    tma::mbar_arrive_expect_tx(&full[st], LY::STAGE);
                    tma::load_2d(sp, &mA, kb * BK, m0, &full[st]);
                    tma::load_2d(sp + LY::A, &mB, kb * BK, n0, &full[st]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------------------------------------- MMA issuer
            constexpr uint32_t idesc = idesc_bf16<BN>();
            int it = 0, ti = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
                const int acc = ti & 1;
                if (ti >= 2) tma::mbar_wait(&tempty[acc], ((ti >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t td = tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    tma::mbar_wait(&full[st], (it / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sa = tma::smem_u32(stages + st * LY::STAGE), sb = sa + LY::A;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)  // 16 bf16 = 32 bytes per UMMA k-step
                        mma_bf16(td, sw128_desc(sa + 32 * k), sw128_desc(sb + 32 * k), idesc, (kb | k) != 0);
                    mma_commit(&empty[st]);
                }
                mma_commit(&tfull[acc]);
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue
        const int q = warp & 3;  // TMEM lane quarter this warp may access (warps 2..5)
        float* buf = epi + (warp - 2) * 1024;
        uint64_t* cb = &cbar[warp - 2];
        uint32_t cph = 0;
        int ti = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
            const int m0 = (tile % tm) * BM, n0 = (tile / tm) * BN;
            const int acc = ti & 1;
            const int rbase = m0 + 32 * q;
            tma::mbar_wait(&tfull[acc], (ti >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += CW) {
                if (lane == 0) tma::bulk_wait_read<0>();  // the last store has read the box
                __syncwarp();
                if (Cin && lane == 0) {
                    tma::mbar_arrive_expect_tx(cb, 32 * CW * 4);
                    tma::load_2d(buf, &mCin, n0 + c0, rbase, cb);
                }
                uint32_t r[CW];
                const uint32_t taddr = tmem + acc * BN + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
                if constexpr (CW == 32) {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]),
                          "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                        : "r"(taddr));
                } else {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15}, [%16];"
                        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                          "=r"(r[14]), "=r"(r[15])
                        : "r"(taddr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c0 + CW >= BN) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    tma::mbar_arrive(&tempty[acc]);
                }
                if (Cin) tma::mbar_wait(cb, (cph++) & 1);
                if constexpr (OB) {  // bf16 row of CW values: 64-byte rows, 64B swizzle (CW = 32)
                    unsigned char* rb = reinterpret_cast<unsigned char*>(buf) + lane * CW * 2;
#pragma unroll
                    for (int g = 0; g < CW / 8; ++g) {
                        const int col = n0 + c0 + 8 * g;
                        uint32_t pk[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float x0 = alpha * __uint_as_float(r[8 * g + 2 * e]);
                            float x1 = alpha * __uint_as_float(r[8 * g + 2 * e + 1]);
                            if (bias) {
                                x0 += __ldg(bias + min(col + 2 * e, N - 1));
                                x1 += __ldg(bias + min(col + 2 * e + 1, N - 1));
                            }
                            const __nv_bfloat162 h2 = __floats2bfloat162_rn(act(x0, act_kind), act(x1, act_kind));
                            pk[e] = *reinterpret_cast<const uint32_t*>(&h2);
                        }
                        const int chunk = CW == 32 ? (g ^ ((lane >> 1) & 3)) : g;
                        *reinterpret_cast<uint4*>(rb + 16 * chunk) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    }
                } else {
                float* rowp = buf + lane * CW;  // this lane's row: CW / 4 16-byte chunks (swizzled at CW = 32)
#pragma unroll
                for (int g = 0; g < CW / 4; ++g) {
                    float4* p4 = reinterpret_cast<float4*>(rowp + 4 * (CW == 32 ? (g ^ (lane & 7)) : g));
                    const int col = n0 + c0 + 4 * g;
                    float v[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float x = alpha * __uint_as_float(r[4 * g + e]);
                        if (bias) x += __ldg(bias + min(col + e, N - 1));
                        v[e] = act(x, act_kind);
                    }
                    if (Cin) {
                        const float4 c = *p4;
                        v[0] += beta * c.x;
                        v[1] += beta * c.y;
                        v[2] += beta * c.z;
                        v[3] += beta * c.w;
                    }
                    *p4 = make_float4(v[0], v[1], v[2], v[3]);
                }
                }
                tma::fence_proxy_async();  // generic smem writes -> the TMA store's reads
                __syncwarp();
                if (lane == 0) {
                    tma::store_2d(&mC, buf, n0 + c0, rbase);
                    tma::bulk_commit();
                }
            }
        }
        if (lane == 0) tma::bulk_wait<0>();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 enc_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// [rows, cols] bf16 row-major, box [box_rows, 64 cols = 128 B], 128-byte swizzle
static bool enc_bf16(CUtensorMap* m, const void* p, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    auto fn = enc_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(p) & 15) || ((cols * 2) & 15)) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {BK, box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// C / Cin boxes: 32 rows x cw fp32; cw = 32 (128 B rows, 128-byte swizzle) or
// 16 (narrow outputs, unswizzled)
static bool enc_out(CUtensorMap* m, const void* p, uint64_t rows, uint64_t cols, uint32_t cw) {
    auto fn = enc_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(p) & 15) || ((cols * 4) & 15)) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {cw, 32};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(p), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, cw == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// bf16 C boxes: 32 rows x cw bf16 (64-byte rows, 64B swizzle at cw = 32)
static bool enc_out16(CUtensorMap* m, const void* p, uint64_t rows, uint64_t cols, uint32_t cw) {
    auto fn = enc_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(p) & 15) || ((cols * 2) & 15)) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {cw, 32};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, cw == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <int BN>
static int launch(const void* A, const void* Bt, void* C, const float* Cin, const float* bias, int64_t M, int64_t N,
                  int64_t K, float alpha, float beta, int act_kind, bool out_bf16, cudaStream_t st) {
    CUtensorMap mA, mB, mC, mCin;
    constexpr uint32_t cw = BN < 32 ? BN : 32;
    const bool oc = out_bf16 ? enc_out16(&mC, C, M, N, cw) : enc_out(&mC, C, M, N, cw);
    if (!enc_bf16(&mA, A, M, K, BM) || !enc_bf16(&mB, Bt, N, K, BN) || !oc ||
        (Cin && !enc_out(&mCin, Cin, M, N, cw))) {
        set_error("gemm_bf16: TMA descriptor rejected (K %% 8 == 0, N %% 4 == 0 and 16-byte aligned rows required)");
        return LRX_ERR_VALUE;
    }
    if (!Cin) mCin = mC;
    const size_t smem = Lay<BN>::smem();
    auto k = out_bf16 ? gemm_bf16_kernel<BN, true> : gemm_bf16_kernel<BN, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        set_error("gemm_bf16: cannot reserve %zu B of shared memory", smem);
        return LRX_ERR_CUDA;
    }
    const int64_t tiles = cdiv(M, BM) * cdiv(N, BN);
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, sm_count());
    k<<<grid, THREADS, smem, st>>>(mA, mB, mC, mCin, Cin, bias, (int)M, (int)N, (int)K, alpha, beta, act_kind);
    return launched(out_bf16 ? "lrx_gemm_bf16/tcgen05 (bf16 out)" : "lrx_gemm_bf16/tcgen05");
}

}  // namespace gemm16
}  // namespace lrx

using namespace lrx;

extern "C" {

int lrx_gemm_bf16(const void* A, const void* Bt, void* C, const void* Cin, const void* bias, int64_t M, int64_t N,
                  int64_t K, float alpha, float beta, int act, int out_bf16, void* stream) {
    LRX_REQUIRE(M >= 1 && N >= 1 && K >= 1, LRX_ERR_SHAPE, "gemm_bf16: bad extents M=%lld N=%lld K=%lld",
                (long long)M, (long long)N, (long long)K);
    LRX_REQUIRE(act >= 0 && act <= 2, LRX_ERR_VALUE, "gemm_bf16: unknown activation %d", act);
    LRX_REQUIRE(!(out_bf16 && Cin), LRX_ERR_VALUE, "gemm_bf16: Cin needs the fp32 output");
    // the whole K is accumulated in TMEM (not round-to-nearest; the bf16
    // operands' own rounding dominates), N is tiled by 32-column boxes
    LRX_REQUIRE(M < (1ll << 31) && N <= (1 << 16) && N % 4 == 0 && K <= 16384, LRX_ERR_UNSUPPORTED,
                "gemm_bf16: extents unsupported (N %% 4 == 0, K <= 16384)");
    cudaStream_t st = (cudaStream_t)stream;
    void* c = C;
    const bool ob = out_bf16 != 0;
    const float *cin = (const float*)Cin, *b = (const float*)bias;
    if (N <= 16) return gemm16::launch<16>(A, Bt, c, cin, b, M, N, K, alpha, beta, act, ob, st);
    if (N <= 32) return gemm16::launch<32>(A, Bt, c, cin, b, M, N, K, alpha, beta, act, ob, st);
    if (N <= 64) return gemm16::launch<64>(A, Bt, c, cin, b, M, N, K, alpha, beta, act, ob, st);
    if (N <= 128) return gemm16::launch<128>(A, Bt, c, cin, b, M, N, K, alpha, beta, act, ob, st);
    return gemm16::launch<256>(A, Bt, c, cin, b, M, N, K, alpha, beta, act, ob, st);
}

}  // extern "C"
