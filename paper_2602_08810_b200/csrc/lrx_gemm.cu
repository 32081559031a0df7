// fp32 GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32) with the
// 3xTF32 split, for the dense projections of the MIMO layers (S5 / LRU:
// layers.py:650-704, bu = B u, y = Re(C x) + D u and their pullbacks).
//
//   C[M, N] = alpha * A[M, K] . Bt[N, K]^T + (colscale ? colscale[n] : beta) * Cin[M, N]
//
// All operands fp32 row-major, both A and Bt K-contiguous ("K-major").  TF32
// keeps 10 mantissa bits, far from the 1e-4 fp32 parity bar, so each product
// is split: a = a_hi + a_lo with a_hi the TF32 truncation (what the tensor core
// reads from an fp32 word) and a_lo = a - a_hi (exact in fp32), and
//   a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi        (error ~2^-20 |a b|)
// i.e. three MMAs per k-step into one fp32 TMEM accumulator.  Bt (a small
// weight) arrives pre-split from the host (Bt, Bt_lo); A's low part is made
// in shared memory from the TMA-landed tile by the split warps.
//
// CTA = 6 warps, one 128 x BN output tile:
//   warp 0      TMA producer (A, Bt, Bt_lo k-blocks of 32 into a 3-stage ring,
//               128-byte swizzle = the UMMA K-major SW128 canonical layout)
//   warp 1      MMA issuer (one thread; 4 k-steps x 3 products per k-block,
//               tcgen05.commit frees the stage / signals the epilogue)
//   warps 2..5  split (A_lo = A - trunc_tf32(A), same swizzled offsets), then
//               the epilogue: tcgen05.ld of its 32 TMEM lanes (= rows),
//               alpha / colscale / Cin, direct 128-byte row stores.
#include "lrx_host.h"
#include "lrx_tma.cuh"

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>
#include <string.h>

#include <algorithm>

namespace lrx {
namespace gemm {

constexpr int BM = 128;
constexpr int BKT = 16;  // K-block of the tall kernel: 64-byte rows, 64B swizzle, 4 stages in flight

__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
    // K-major SWIZZLE_64B: 8-row groups of 64-byte rows = 512 B (SBO), layout type 4
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}


template <int BN>
__host__ __device__ constexpr uint32_t idesc_tf32() {
    // c_format F32 (1) [4,6), a/b format TF32 (2) [7,10) [10,13), K-major both,
    // N >> 3 at [17,23), M >> 4 at [24,29)
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// multicast flavours for 2-CTA clusters (MC = 2): the B / B_lo k-blocks land
// in both CTAs' shared memory from one TMA each, and every MMA commit frees
// the stage in both CTAs
__device__ __forceinline__ void load_2d_mc(void* dst, const CUtensorMap* m, int c0, int r0, uint64_t* bar,
                                           uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(tma::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(r0), "r"(tma::smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     tma::smem_u32(bar)),
                 "h"(mask)
                 : "memory");
}
__device__ __forceinline__ int cluster_rank() {
    int r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     tma::smem_u32(bar))
                 : "memory");
}

// epilogue activation (the projection's nonlinearity fused into the GEMM):
// 1 softplus (threshold 30, numerics.py:36-39), 2 sigmoid
__device__ __forceinline__ float epi_act(float x, int a) {
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

template <int BN, bool TE = false>
struct Lay {
    static constexpr int A = BM * BKT * 4;  // 8 KB
    static constexpr int B = BN * BKT * 4;
    static constexpr int STAGE = 2 * A + 2 * B;  // A, A_lo, Bt, Bt_lo
    static constexpr int STAGES = BN >= 256 ? 4 : 6;
    // per epilogue warp: TE = one 32 x 32 fp32 TMA box (128B-swizzled, 4 KB);
    // else a 32 x 32 transpose tile (padded)
    static constexpr int EPI = TE ? 8 * 4096 : 8 * 32 * 33 * 4;
    // 1 KB alignment slack + 1 KB barrier block + the stage ring + epilogue tiles
    static constexpr size_t smem() { return 2048 + (size_t)STAGES * STAGE + EPI; }
};

// Persistent: CTA c walks output tiles c, c + grid, ... (M-fastest).  Warps:
// 0 TMA producer, 1 MMA issuer, 2..5 split (A_lo), 6..9 epilogue.  The
// accumulator is double-buffered in TMEM (2 x BN columns), so the epilogue of
// tile i (tcgen05.ld -> smem transpose -> coalesced alpha/colscale/Cin
// row stores) overlaps the mainloop of tile i+1.
constexpr int THREADS_P = 448;  // + 8 epilogue warps (2 per TMEM lane quarter)

// TE: TMA epilogue.  Each epilogue warp owns one 4 KB box buffer (32 rows x
// 32 columns, 128-byte swizzle): the skip input Cin lands there by TMA
// (issued before the accumulator wait, so the first chunk's read overlaps
// the mainloop), the lane of row r combines it with its accumulator row in
// place (16-byte accesses at the swizzled chunk: conflict-free), and one
// TMA store writes the box (out-of-bounds rows / columns clipped).  The
// direct-store epilogue kept 32 loads of 128 B in flight per warp, which
// bounded the skip-input GEMMs at ~2 TB/s.
template <int BN, bool TE, int MC>
__global__ void __launch_bounds__(THREADS_P, 1) gemm_tf32x3_kernel(
    const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
    const __grid_constant__ CUtensorMap mBl, const __grid_constant__ CUtensorMap mC,
    const __grid_constant__ CUtensorMap mCin, float* C, const float* Cin,
    const float* __restrict__ colscale, const float* __restrict__ bias, int act_kind, int M, int N, int K, float alpha,
    float beta) {
    using LY = Lay<BN, TE>;
    constexpr int STAGES = LY::STAGES;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base);     // [STAGES] TMA landed
    uint64_t* split = full + STAGES;                         // [STAGES] A_lo written
    uint64_t* empty = split + STAGES;                        // [STAGES] MMAs done with the stage
    uint64_t* tfull = empty + STAGES;                        // [2] accumulator ready
    uint64_t* tempty = tfull + 2;                            // [2] accumulator drained
    uint64_t* cbar = tempty + 2;                             // [8] TE: Cin box landed (per epilogue warp)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cbar + 8);
    unsigned char* stages = base + 1024;
    float* epi = reinterpret_cast<float*>(stages + STAGES * LY::STAGE);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (K + BKT - 1) / BKT;
    const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
    // tile schedule: a cluster of MC CTAs walks units of MC adjacent M-tiles
    // (same N-tile) in lockstep; CTA rank r takes M-tile MC * (unit % tmp) + r
    const int crank = MC == 2 ? cluster_rank() : 0;
    const int cid = blockIdx.x / MC, ncl = gridDim.x / MC;
    const int tmp = (tm + MC - 1) / MC, ntiles = tmp * tn;
    constexpr uint32_t kCols = 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;

    if (threadIdx.x == 0) {
        tma::prefetch_map(&mA);
        tma::prefetch_map(&mB);
        tma::prefetch_map(&mBl);
        for (int i = 0; i < STAGES; ++i) {
            tma::mbar_init(&full[i], 1);
            tma::mbar_init(&split[i], 128);
            tma::mbar_init(&empty[i], MC);  // MC = 2: both CTAs' MMAs release a stage
        }
        for (int i = 0; i < 2; ++i) {
            tma::mbar_init(&tfull[i], 1);
            tma::mbar_init(&tempty[i], 256);
        }
        for (int i = 0; i < 8; ++i) tma::mbar_init(&cbar[i], 1);
        if (TE) {
            tma::prefetch_map(&mC);
            if (Cin) tma::prefetch_map(&mCin);
        }
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
    if (MC == 2) cluster_sync();  // the peer's barriers exist before any multicast reaches them
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ------------------------------------------ producer
            int it = 0;
            for (int tile = cid; tile < ntiles; tile += ncl) {
                const int m0 = ((tile % tmp) * MC + crank) * BM, n0 = (tile / tmp) * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    if (it >= STAGES) tma::mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
                    unsigned char* sp = stages + st * LY::STAGE;
                    tma::mbar_arrive_expect_tx(&full[st], LY::A + 2 * LY::B);
                    tma::load_2d(sp, &mA, kb * BKT, m0, &full[st]);
                    if (MC == 2) {  // rank 0 brings B, rank 1 B_lo, each to both CTAs
                        if (crank == 0) load_2d_mc(sp + 2 * LY::A, &mB, kb * BKT, n0, &full[st], 0x3);
                        else load_2d_mc(sp + 2 * LY::A + LY::B, &mBl, kb * BKT, n0, &full[st], 0x3);
                    } else {
                        tma::load_2d(sp + 2 * LY::A, &mB, kb * BKT, n0, &full[st]);
                        tma::load_2d(sp + 2 * LY::A + LY::B, &mBl, kb * BKT, n0, &full[st]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ------------------------------------------ MMA issuer
            constexpr uint32_t idesc = idesc_tf32<BN>();
            int it = 0, ti = 0;
            for (int tile = cid; tile < ntiles; tile += ncl, ++ti) {
                const int acc = ti & 1;
                if (ti >= 2) tma::mbar_wait(&tempty[acc], ((ti >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t td = tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    tma::mbar_wait(&split[st], (it / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sa = tma::smem_u32(stages + st * LY::STAGE);
                    const uint32_t sal = sa + LY::A, sb = sa + 2 * LY::A, sbl = sb + LY::B;
#pragma unroll
                    for (int k = 0; k < BKT / 8; ++k) {  // 8 tf32 = 32 bytes per UMMA k-step
                        const uint32_t off = k * 32;
                        const uint64_t dA = sw64_desc(sa + off), dAl = sw64_desc(sal + off);
                        const uint64_t dB = sw64_desc(sb + off), dBl = sw64_desc(sbl + off);
                        mma_tf32(td, dA, dB, idesc, (kb | k) != 0);
                        mma_tf32(td, dA, dBl, idesc, 1);
                        mma_tf32(td, dAl, dB, idesc, 1);
                    }
                    if (MC == 2) mma_commit_mc(&empty[st], 0x3);  // frees the stage in both CTAs
                    else mma_commit(&empty[st]);  // stage reusable once these MMAs have read it
                }
                mma_commit(&tfull[acc]);
            }
        }
    } else if (warp < 6) {
        // ---------------------------------------------------------- split
        const int t = threadIdx.x - 64;  // 0..127
        int it = 0;
        for (int tile = cid; tile < ntiles; tile += ncl)
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int st = it % STAGES;
                tma::mbar_wait(&full[st], (it / STAGES) & 1);
                const float4* a4 = reinterpret_cast<const float4*>(stages + st * LY::STAGE);
                float4* l4 = reinterpret_cast<float4*>(stages + st * LY::STAGE + LY::A);
#pragma unroll
                for (int i = 0; i < LY::A / 16 / 128; ++i) {
                    const float4 v = a4[t + 128 * i];
                    float4 lo;
                    lo.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                    lo.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                    lo.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                    lo.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                    l4[t + 128 * i] = lo;
                }
                tma::fence_proxy_async();  // generic writes -> async-proxy (MMA) reads
                tma::mbar_arrive(&split[st]);
            }
    } else if (TE) {
        // ------------------------------------------------- epilogue (TMA)
        const int q = warp & 3;
        const int half = (warp - 6) >> 2;
        float* buf = epi + (warp - 6) * 1024;  // 4 KB, 1 KB aligned
        uint64_t* cb = &cbar[warp - 6];
        uint32_t cph = 0;
        int ti = 0;
        for (int tile = cid; tile < ntiles; tile += ncl, ++ti) {
            const int m0 = ((tile % tmp) * MC + crank) * BM, n0 = (tile / tmp) * BN;
            const int acc = ti & 1;
            const int rbase = m0 + 32 * q;
            auto issue_cin = [&](int c0) {
                if (lane == 0) {
                    tma::mbar_arrive_expect_tx(cb, 4096);
                    tma::load_2d(buf, &mCin, n0 + c0, rbase, cb);
                }
            };
            if (lane == 0) tma::bulk_wait_read<0>();  // the last store has read the buffer
            __syncwarp();
            if (Cin) issue_cin(32 * half);
            tma::mbar_wait(&tfull[acc], (ti >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int c0 = 32 * half; c0 < BN; c0 += 64) {
                uint32_t r[32];
                const uint32_t taddr = tmem + acc * BN + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                    "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                      "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                      "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                // the skip input's per-column scale: lane j loads column c0 + j once and
                // the row lanes take it by shuffle (S5 skip GEMM 104 -> 98 us)
                const float csj = colscale ? __ldg(colscale + min(n0 + c0 + lane, N - 1)) : beta;
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c0 + 64 >= BN) {
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    tma::mbar_arrive(&tempty[acc]);
                }
                if (Cin) tma::mbar_wait(cb, (cph++) & 1);
                float* rowp = buf + lane * 32;  // this lane's row: 8 swizzled 16-byte chunks
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    float4* p4 = reinterpret_cast<float4*>(rowp + 4 * (g ^ (lane & 7)));
                    float4 v;
                    v.x = alpha * __uint_as_float(r[4 * g]);
                    v.y = alpha * __uint_as_float(r[4 * g + 1]);
                    v.z = alpha * __uint_as_float(r[4 * g + 2]);
                    v.w = alpha * __uint_as_float(r[4 * g + 3]);
                    if (bias || act_kind) {  // broadcast L1 loads (shuffles measured slower here)
                        const int col = n0 + c0 + 4 * g;
                        const float b0 = bias ? __ldg(bias + min(col, N - 1)) : 0.f;
                        const float b1 = bias ? __ldg(bias + min(col + 1, N - 1)) : 0.f;
                        const float b2 = bias ? __ldg(bias + min(col + 2, N - 1)) : 0.f;
                        const float b3 = bias ? __ldg(bias + min(col + 3, N - 1)) : 0.f;
                        v.x = epi_act(v.x + b0, act_kind);
                        v.y = epi_act(v.y + b1, act_kind);
                        v.z = epi_act(v.z + b2, act_kind);
                        v.w = epi_act(v.w + b3, act_kind);
                    }
                    if (Cin) {
                        const float4 c = *p4;
                        v.x += __shfl_sync(0xffffffffu, csj, 4 * g) * c.x;
                        v.y += __shfl_sync(0xffffffffu, csj, 4 * g + 1) * c.y;
                        v.z += __shfl_sync(0xffffffffu, csj, 4 * g + 2) * c.z;
                        v.w += __shfl_sync(0xffffffffu, csj, 4 * g + 3) * c.w;
                    }
                    *p4 = v;
                }
                tma::fence_proxy_async();  // generic smem writes -> the TMA store's reads
                __syncwarp();
                if (lane == 0) {
                    tma::store_2d(&mC, buf, n0 + c0, rbase);
                    tma::bulk_commit();
                }
                if (c0 + 64 < BN) {
                    if (lane == 0) tma::bulk_wait_read<0>();
                    __syncwarp();
                    if (Cin) issue_cin(c0 + 64);
                }
            }
        }
        if (lane == 0) tma::bulk_wait<0>();
    } else {
        // ---------------------------------------------------------- epilogue
        const int q = warp & 3;            // TMEM lane quarter this warp may access
        const int half = (warp - 6) >> 2;  // which of the interleaved 32-column chunks
        float* tp = epi + (warp - 6) * 32 * 33;
        int ti = 0;
        for (int tile = cid; tile < ntiles; tile += ncl, ++ti) {
            const int m0 = ((tile % tmp) * MC + crank) * BM, n0 = (tile / tmp) * BN;
            const int acc = ti & 1;
            const int rbase = m0 + 32 * q;
            // skip-input rows for column chunk c0 (lane = column: coalesced);
            // the next chunk's loads are issued before this chunk is stored
            float cin[32], cnext[32];
            auto load_cin = [&](int c0, float* dst) {
                const int col = n0 + c0 + lane;
                const bool colok = col < N;
                const float cs = colok ? (colscale ? colscale[col] : beta) : 0.f;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    dst[i] = (colok && rbase + i < M) ? cs * __ldcs(Cin + (int64_t)(rbase + i) * N + col) : 0.f;
            };
            if (Cin) load_cin(32 * half, cnext);
            tma::mbar_wait(&tfull[acc], (ti >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int c0 = 32 * half; c0 < BN; c0 += 64) {
                uint32_t r[32];
                const uint32_t taddr = tmem + acc * BN + ((uint32_t)(32 * q) << 16) + (uint32_t)c0;
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                    "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                      "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                      "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (c0 + 64 >= BN) {  // this warp's last chunk: accumulator reads done
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    tma::mbar_arrive(&tempty[acc]);
                }
                // transpose through shared memory: lane holds row (32q + lane), 32 columns;
                // write back rows with the lane index on the column (coalesced)
#pragma unroll
                for (int j = 0; j < 32; ++j) tp[lane * 33 + j] = __uint_as_float(r[j]);
                __syncwarp();
                const int col = n0 + c0 + lane;
                const bool colok = col < N;
                if (Cin) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) cin[i] = cnext[i];
                    if (c0 + 64 < BN) load_cin(c0 + 64, cnext);
                }
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int row = rbase + i;
                    if (row < M && colok) {
                        float v = alpha * tp[i * 33 + lane];
                        if (bias || act_kind) v = epi_act(v + (bias ? bias[col] : 0.f), act_kind);
                        if (Cin) v += cin[i];
                        __stcs(C + (int64_t)row * N + col, v);
                    }
                }
                __syncwarp();
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (MC == 2) cluster_sync();  // no CTA leaves while its peer may still multicast into it
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols) : "memory");
}

// ============================================================================
// "TN" reduction GEMM for the weight gradients (R = gy^T x, R2 = g^T u):
//   part[kz][m][n] = alpha * sum_{k in split kz} A[k, m] B[k, n]
// A [K, M] and B [K, N] row-major: both operands are MN-major for the MMA.
// K (= B*L tokens, 1e5+) is split across CTAs; the partial tiles are summed
// in a fixed order by lrx_reduce_rows (deterministic).  Both operands are
// activations, so the split warps make both low parts.
//
// MN-major tf32 operands use the 128B swizzle with 32-byte atoms: a TMA box
// of 32 K-rows x 32 fp32 (128 B) is 8 atoms of 4 K-rows x 128 B stacked at
// 512 B (SBO); the next 32-wide MN chunk is the next box, 4 KB on (LBO).  One
// UMMA k-step of 8 tf32 rows = two atoms: advance the start address by 1 KB.
constexpr int BKN = 16;  // K-block (rows) of the TN kernel: boxes of 16 rows x 128 B
constexpr int kMaxSpan = 4096;  // K rows one TN CTA accumulates in TMEM (see tn_plan)
constexpr int THREADS_TN = 320;  // TMA, MMA, 8 split warps (the first 4 also run the epilogue)

__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr) {
    // MN-major tf32 needs the 128B swizzle with 32-byte atoms (layout type 1,
    // SWIZZLE_128B_BASE32B; TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 4-row
    // swizzle period, SBO = 512 B between 4-row K groups, LBO = one box
    // (BKN rows x 128 B) between 32-element MN chunks
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((BKN * 128) >> 4) << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;
    return d;
}

template <int BN>
__host__ __device__ constexpr uint32_t idesc_tf32_mn() {
    return idesc_tf32<BN>() | (1u << 15) | (1u << 16);  // A and B MN-major
}

template <int BN, int MT>
struct LayTN {
    static constexpr int A = MT * BM * BKN * 4;  // 4 MT boxes of BKN x 32
    static constexpr int B = BN * BKN * 4;       // BN/32 boxes
    static constexpr int STAGE = 2 * A + 2 * B;
    static constexpr int STAGES = STAGE >= 64 * 1024 ? 3 : STAGE >= 48 * 1024 ? 4 : 6;
    static constexpr size_t smem() { return 2048 + (size_t)STAGES * STAGE; }
};

__device__ __forceinline__ float4 tf32_low4(float4 v) {
    float4 lo;
    lo.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    lo.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    lo.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    lo.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    return lo;
}

// MT M-tiles of 128 per CTA share every B stage (MT = 2 halves the B traffic
// of the weight-gradient reductions, whose M = N = 256)
template <int BN, int MT>
__global__ void __launch_bounds__(THREADS_TN, 1) gemm_tn_kernel(
    const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, float* __restrict__ part,
    int M, int N, int K, int kb_per_split, float alpha) {
    using LY = LayTN<BN, MT>;
    constexpr int STAGES = LY::STAGES;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base);
    uint64_t* split = full + STAGES;
    uint64_t* empty = split + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
    unsigned char* stages = base + 1024;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM * MT, n0 = blockIdx.y * BN, kz = blockIdx.z;
    const int nk_all = (K + BKN - 1) / BKN;
    const int kb0 = kz * kb_per_split, kb1 = min(nk_all, kb0 + kb_per_split);
    const int nk = max(0, kb1 - kb0);
    constexpr uint32_t kTmemCols = MT * BN <= 32 ? 32 : MT * BN <= 64 ? 64 : MT * BN <= 128 ? 128 : MT * BN <= 256 ? 256 : 512;

    if (threadIdx.x == 0) {
        tma::prefetch_map(&mA);
        tma::prefetch_map(&mB);
        for (int i = 0; i < STAGES; ++i) {
            tma::mbar_init(&full[i], 1);
            tma::mbar_init(&split[i], 256);
            tma::mbar_init(&empty[i], 1);
        }
        tma::mbar_init(tfull, 1);
        tma::fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tma::smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < nk; ++i) {
                const int st = i % STAGES;
                if (i >= STAGES) tma::mbar_wait(&empty[st], ((i / STAGES) & 1) ^ 1);
                unsigned char* sp = stages + st * LY::STAGE;
                const int k0 = (kb0 + i) * BKN;
                tma::mbar_arrive_expect_tx(&full[st], LY::A + LY::B);
#pragma unroll
                for (int c = 0; c < MT * BM / 32; ++c) tma::load_2d(sp + c * BKN * 128, &mA, m0 + 32 * c, k0, &full[st]);
#pragma unroll
                for (int c = 0; c < BN / 32; ++c)
                    tma::load_2d(sp + 2 * LY::A + c * BKN * 128, &mB, n0 + 32 * c, k0, &full[st]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32_mn<BN>();
            for (int i = 0; i < nk; ++i) {
                const int st = i % STAGES;
                tma::mbar_wait(&split[st], (i / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t sa = tma::smem_u32(stages + st * LY::STAGE);
                const uint32_t sal = sa + LY::A, sb = sa + 2 * LY::A, sbl = sb + LY::B;
#pragma unroll
                for (int k = 0; k < BKN / 8; ++k) {
                    const uint32_t off = k * 1024;  // 8 K-rows x 128 B
                    const uint64_t dB = sw128_mn_desc(sb + off), dBl = sw128_mn_desc(sbl + off);
#pragma unroll
                    for (int h = 0; h < MT; ++h) {  // M half h: its 4 boxes of 32 columns
                        const uint32_t ah = h * 4 * BKN * 128;
                        const uint64_t dA = sw128_mn_desc(sa + ah + off), dAl = sw128_mn_desc(sal + ah + off);
                        const uint32_t td = tmem + h * BN;
                        mma_tf32(td, dA, dB, idesc, (i | k) != 0);
                        mma_tf32(td, dA, dBl, idesc, 1);
                        mma_tf32(td, dAl, dB, idesc, 1);
                    }
                }
                mma_commit(&empty[st]);
            }
            mma_commit(tfull);
        }
    } else {
        const int t = threadIdx.x - 64;  // 8 split warps: 0..255
        for (int i = 0; i < nk; ++i) {
            const int st = i % STAGES;
            tma::mbar_wait(&full[st], (i / STAGES) & 1);
            unsigned char* sp = stages + st * LY::STAGE;
            const float4* a4 = reinterpret_cast<const float4*>(sp);
            float4* al4 = reinterpret_cast<float4*>(sp + LY::A);
            const float4* b4 = reinterpret_cast<const float4*>(sp + 2 * LY::A);
            float4* bl4 = reinterpret_cast<float4*>(sp + 2 * LY::A + LY::B);
#pragma unroll
            for (int j = 0; j < LY::A / 16 / 256; ++j) al4[t + 256 * j] = tf32_low4(a4[t + 256 * j]);
#pragma unroll
            for (int j = 0; j < LY::B / 16 / 256; ++j) bl4[t + 256 * j] = tf32_low4(b4[t + 256 * j]);
            tma::fence_proxy_async();
            tma::mbar_arrive(&split[st]);
        }
        if (warp >= 6) goto done;  // warps 2..5 cover the four TMEM lane quarters
        {
        const int q = warp & 3;
        if (nk > 0) {
            tma::mbar_wait(tfull, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        for (int h = 0; h < MT; ++h) {
        const int row = m0 + h * BM + 32 * q + lane;
        float* dst = part + ((int64_t)kz * M + row) * N;
        if (nk == 0) {
            if (row < M)
                for (int c = n0; c < min(N, n0 + BN); ++c) dst[c] = 0.f;
        } else {
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(h * BN + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                    "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                      "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                      "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (row < M)
                    for (int j = 0; j < 32; ++j) {
                        const int col = n0 + c0 + j;
                        if (col < N) dst[col] = alpha * __uint_as_float(r[j]);
                    }
            }
        }
        }
        }
    }
done:
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

static bool enc_k(CUtensorMap* m, const void* p, uint64_t rows, uint64_t cols, uint32_t box_rows);

static bool enc_epi(CUtensorMap* m, const void* p, uint64_t rows, uint64_t cols);

template <int BN>
static int launch(const float* A, const float* Bt, const float* Btl, float* C, const float* Cin, const float* cs,
                  const float* bias, int act, int64_t M, int64_t N, int64_t K, float alpha, float beta,
                  cudaStream_t st) {
    CUtensorMap mA, mB, mBl, mC, mCin;
    if (!enc_k(&mA, A, M, K, BM) || !enc_k(&mB, Bt, N, K, BN) || !enc_k(&mBl, Btl, N, K, BN)) {
        set_error("gemm: TMA descriptor rejected (K %% 4 == 0 and 16-byte aligned rows required)");
        return LRX_ERR_VALUE;
    }
    // TMA epilogue when C / Cin rows are 16-byte aligned (LRX_GEMM_EPI=direct forces the old one)
    const char* ee = getenv("LRX_GEMM_EPI");
    const bool te = !(ee && !strcmp(ee, "direct")) && enc_epi(&mC, C, M, N) && (!Cin || enc_epi(&mCin, Cin, M, N));
    if (!te) mC = mA, mCin = mA;  // unused
    else if (!Cin) mCin = mC;
    const size_t smem = te ? Lay<BN, true>::smem() : Lay<BN, false>::smem();
    // 2-CTA clusters sharing the B / B_lo stream (LRX_GEMM_MC=1 disables)
    const char* em = getenv("LRX_GEMM_MC");
    const bool mc = !(em && !strcmp(em, "1")) && cdiv(M, BM) >= 2;
    auto k = te ? (mc ? gemm_tf32x3_kernel<BN, true, 2> : gemm_tf32x3_kernel<BN, true, 1>)
                : (mc ? gemm_tf32x3_kernel<BN, false, 2> : gemm_tf32x3_kernel<BN, false, 1>);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        set_error("gemm: cannot reserve %zu B of shared memory", smem);
        return LRX_ERR_CUDA;
    }
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    if (mc) {
        const int64_t units = cdiv(cdiv(M, BM), 2) * cdiv(N, BN);
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(THREADS_P);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // persistent: only as many pairs as can be co-resident (an odd SM
        // count per GPC leaves SMs no pair can use)
        static int max_cl = 0;
        if (!max_cl) {
            cfg.gridDim = dim3(sms);
            if (cudaOccupancyMaxActiveClusters(&max_cl, (void*)k, &cfg) != cudaSuccess || max_cl < 1) max_cl = sms / 2;
        }
        cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(units, max_cl)));
        if (cudaLaunchKernelEx(&cfg, k, mA, mB, mBl, mC, mCin, C, Cin, cs, bias, act, (int)M, (int)N, (int)K, alpha,
                               beta) !=
            cudaSuccess) {
            set_error("gemm: cluster launch failed");
            return LRX_ERR_CUDA;
        }
        return launched(te ? "lrx_gemm_f32/tcgen05x2+tma_epilogue" : "lrx_gemm_f32/tcgen05x2");
    }
    const int64_t tiles = cdiv(M, BM) * cdiv(N, BN);
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
    k<<<grid, THREADS_P, smem, st>>>(mA, mB, mBl, mC, mCin, C, Cin, cs, bias, act, (int)M, (int)N, (int)K, alpha,
                                     beta);
    return launched(te ? "lrx_gemm_f32/tcgen05+tma_epilogue" : "lrx_gemm_f32/tcgen05");
}

}  // namespace gemm
}  // namespace lrx

#include <cudaTypedefs.h>

namespace lrx {
namespace gemm {

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


// [rows, cols] fp32 row-major, box [box_rows, BKT = 16 cols = 64 B], 64-byte swizzle
// C / Cin boxes of the TMA epilogue: 32 rows x 32 fp32 (128 B), 128B swizzle.
static bool enc_epi(CUtensorMap* m, const void* p, uint64_t rows, uint64_t cols) {
    auto fn = enc_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(p) & 15) || ((cols * 4) & 15)) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(p), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool enc_k(CUtensorMap* m, const void* p, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    auto fn = enc_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(p) & 15) || ((cols * 4) & 15)) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {BKT, box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(p), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [rows, cols] fp32 row-major, box [32 rows, 32 cols = 128 B], 128-byte
// swizzle with 32-byte atoms (the MN-major tf32 UMMA layout)
static bool enc_sw128_box32(CUtensorMap* m, const void* p, uint64_t rows, uint64_t cols) {
    auto fn = enc_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(p) & 15) || ((cols * 4) & 15)) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 4};
    cuuint32_t box[2] = {32, BKN};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(p), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct TNPlan {
    int BN, MT, ks, kb_per_split;
};
static TNPlan tn_plan(int64_t M, int64_t N, int64_t K) {
    TNPlan p;
    p.BN = N <= 64 ? 64 : N <= 128 ? 128 : 256;
    // MT = 2 (both M halves per CTA sharing each B stage) halves the B traffic
    // but measured slower on the S5 shapes (192 vs 137 us for 256x256x131072:
    // fewer stages in flight); kept selectable for other shapes
    p.MT = getenv("LRX_GEMM_TN_MT2") && M > BM ? 2 : 1;
    const int64_t tiles = cdiv(M, BM * p.MT) * cdiv(N, p.BN);
    const int64_t nk = cdiv(K, BKN);
    // split-K CTAs over the GPU: one wave (measured 256x256x131072: 148 CTAs
    // 104 us, 296 136 us, 592 194 us: each extra wave re-pays the pipeline
    // fill and writes more partial tiles)
    const char* ew = getenv("LRX_GEMM_TN_CTAS");
    const int64_t ctas = ew ? std::max(1, atoi(ew)) : 148;
    int64_t ks = std::max<int64_t>(1, std::min<int64_t>(cdiv(ctas, tiles), nk / 4 > 0 ? nk / 4 : 1));
    // accuracy: the tensor core's fp32 accumulation is not round-to-nearest;
    // its error grows ~6e-8 per accumulated 8-row MMA step, so one CTA spans
    // at most kMaxSpan rows of K (3e-5) and longer sums split further
    const int64_t ks_acc = cdiv(nk * BKN, (int64_t)kMaxSpan);
    if (!ew && tiles >= ctas) {
        // more tiles than SMs: pick the split (1..4) with the least wave
        // quantisation (2560 x 2560 outputs = 200 tiles: ks 2 fills 90% of 3 waves
        // where ks 1 fills 68% of 2)
        double best = 0;
        for (int64_t k = 1; k <= 4 && k <= std::max<int64_t>(1, nk / 4); ++k) {
            const int64_t n = tiles * k;
            const double eff = (double)n / (double)(cdiv(n, ctas) * ctas);
            if (eff > best + 0.02) best = eff, ks = k;
        }
    }
    ks = std::max(ks, std::min(ks_acc, nk));
    p.kb_per_split = (int)cdiv(nk, ks);
    p.ks = (int)cdiv(nk, p.kb_per_split);
    return p;
}

template <int BN, int MT>
static int launch_tn(const float* A, const float* B, float* part, const TNPlan& pl, int64_t M, int64_t N, int64_t K,
                     float alpha, cudaStream_t st) {
    CUtensorMap mA, mB;
    if (!enc_sw128_box32(&mA, A, K, M) || !enc_sw128_box32(&mB, B, K, N)) {
        set_error("gemm_tn: TMA descriptor rejected (M, N %% 4 == 0 and 16-byte aligned rows required)");
        return LRX_ERR_VALUE;
    }
    const size_t smem = LayTN<BN, MT>::smem();
    auto k = gemm_tn_kernel<BN, MT>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        set_error("gemm_tn: cannot reserve %zu B of shared memory", smem);
        return LRX_ERR_CUDA;
    }
    const dim3 grid((unsigned)cdiv(M, BM * MT), (unsigned)cdiv(N, BN), (unsigned)pl.ks);
    k<<<grid, THREADS_TN, smem, st>>>(mA, mB, part, (int)M, (int)N, (int)K, pl.kb_per_split, alpha);
    return launched("lrx_gemm_f32_tn/tcgen05");
}

}  // namespace gemm
}  // namespace lrx

using namespace lrx;

extern "C" {

int lrx_gemm_f32(const void* A, const void* Bt, const void* Bt_lo, void* C, const void* Cin, const void* colscale,
                 const void* bias, int act, int64_t M, int64_t N, int64_t K, float alpha, float beta, void* stream) {
    LRX_REQUIRE(M >= 1 && N >= 1 && K >= 1, LRX_ERR_SHAPE, "gemm: bad extents M=%lld N=%lld K=%lld", (long long)M,
                (long long)N, (long long)K);
    // K <= 8192: the whole K is accumulated in TMEM (not round-to-nearest:
    // ~6e-8 per 8-wide step, 6e-5 at the cap); longer sums go to the library
    LRX_REQUIRE(M < (1ll << 31) && N <= (1 << 16) && K <= 8192, LRX_ERR_UNSUPPORTED, "gemm: extents too large");
    LRX_REQUIRE(act >= 0 && act <= 2, LRX_ERR_VALUE, "gemm: unknown activation %d", act);
    cudaStream_t st = (cudaStream_t)stream;
    const float *a = (const float*)A, *b = (const float*)Bt, *bl = (const float*)Bt_lo, *bs = (const float*)bias;
    if (N <= 64) return gemm::launch<64>(a, b, bl, (float*)C, (const float*)Cin, (const float*)colscale, bs, act, M, N, K, alpha,
                                         beta, st);
    const char* e = getenv("LRX_GEMM_BN");
    const int bn_cap = e ? atoi(e) : 256;
    if (N <= 128 || bn_cap <= 128) return gemm::launch<128>(a, b, bl, (float*)C, (const float*)Cin, (const float*)colscale, bs, act, M, N, K,
                                           alpha, beta, st);
    return gemm::launch<256>(a, b, bl, (float*)C, (const float*)Cin, (const float*)colscale, bs, act, M, N, K, alpha, beta, st);
}

int lrx_gemm_f32_tn_splits(int64_t M, int64_t N, int64_t K, int64_t* n_splits) {
    LRX_REQUIRE(M >= 1 && N >= 1 && K >= 1, LRX_ERR_SHAPE, "gemm_tn: bad extents");
    *n_splits = gemm::tn_plan(M, N, K).ks;
    return LRX_OK;
}

int lrx_gemm_f32_tn(const void* A, const void* B, void* part, int64_t M, int64_t N, int64_t K, float alpha,
                    void* stream) {
    LRX_REQUIRE(M >= 1 && N >= 1 && K >= 1, LRX_ERR_SHAPE, "gemm_tn: bad extents M=%lld N=%lld K=%lld",
                (long long)M, (long long)N, (long long)K);
    LRX_REQUIRE(M <= (1 << 16) && N <= (1 << 16) && K < (1ll << 31), LRX_ERR_UNSUPPORTED, "gemm_tn: extents too large");
    const gemm::TNPlan pl = gemm::tn_plan(M, N, K);
    cudaStream_t st = (cudaStream_t)stream;
    const float *a = (const float*)A, *b = (const float*)B;
    if (pl.MT == 2) {
        if (pl.BN == 64) return gemm::launch_tn<64, 2>(a, b, (float*)part, pl, M, N, K, alpha, st);
        if (pl.BN == 128) return gemm::launch_tn<128, 2>(a, b, (float*)part, pl, M, N, K, alpha, st);
        return gemm::launch_tn<256, 2>(a, b, (float*)part, pl, M, N, K, alpha, st);
    }
    if (pl.BN == 64) return gemm::launch_tn<64, 1>(a, b, (float*)part, pl, M, N, K, alpha, st);
    if (pl.BN == 128) return gemm::launch_tn<128, 1>(a, b, (float*)part, pl, M, N, K, alpha, st);
    return gemm::launch_tn<256, 1>(a, b, (float*)part, pl, M, N, K, alpha, st);
}

}  // extern "C"
