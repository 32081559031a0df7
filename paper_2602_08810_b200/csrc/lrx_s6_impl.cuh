// S6 / Mamba selective scan, fused forward / backward.
//
// Reference: pkg/src/linrec/layers.py S6 (983-1168): _projections 1020-1027,
// _forward_tape 1051-1066, _backward 1068-1118; with the pullback of
// autograd._scan_pullback 113-140 and numerics.softplus/sigmoid 86-105.
//
//   delta_k[d] = softplus(pre_k[d] + b_delta[d]),  a[d,n] = -exp(a_log[d,n])
//   x_k[d,n]   = exp(delta_k[d] a[d,n]) x_{k-1}[d,n] + delta_k[d] u_k[d] B_k[n]
//   y_k[d]     = sum_n C_k[n] x_k[d,n] + D[d] u_k[d]
//
// pre = (u W_delta) W_delta_proj and B_k = W_B u, C_k = W_C u are the layer's
// GEMMs (cuBLAS); everything from the bias add to the readout is fused here.
// Activations u / y / gy / gu use the I/O type (bf16, f32 or f64); the
// projection outputs pre, B_k, C_k and the pre-gradient use the compute type
// (f32 for bf16 I/O): the kernel is MUFU-bound, so keeping delta's argument
// unrounded costs no time and keeps d b_delta inside the bf16 tolerance.
//
// Mapping: one thread owns one (b, d) channel with its NS states in registers
// and walks the whole sequence; a CTA holds THREADS consecutive channels of
// one batch row so B_k / C_k rows are staged once in shared memory and read
// as broadcasts.  The forward saves the state every CK steps.  The backward
// walks CK-chunks right-to-left: it recomputes the chunk forward keeping the
// state at every SUB-step boundary in shared memory, then per SUB-block
// recomputes x_{k-1} into shared memory and runs the reverse recurrence.  The
// cross-channel sums dB_k[n] = sum_d g delta u and dC_k[n] = sum_d gy x are
// reduced inside each warp by a register transpose-reduction (one shuffle
// per value), across the CTA's warps in shared memory, and across CTAs as
// per-channel-block partials reduced in a fixed order (deterministic).
#pragma once
#include <stdlib.h>
#include "lrx_common.cuh"
#include "lrx_host.h"

namespace lrx {
namespace s6 {

constexpr int kTT = 16;  // forward time tile (B/C rows staged in smem)

template <typename C, int NS>
struct Cfg {
    static constexpr int THREADS = (sizeof(C) * NS >= 256) ? 32 : 64;
    static constexpr int SUB = NS >= 64 ? 4 : 8;
    static constexpr int CK = NS >= 64 ? 16 : (NS >= 32 ? 32 : 64);
    static constexpr int NSUB = CK / SUB;
    static constexpr int WARPS = THREADS / 32;
    static constexpr size_t smem_bwd() {
        return sizeof(C) * ((size_t)NSUB * NS * THREADS + (size_t)SUB * NS * THREADS + 2 * (size_t)SUB * NS +
                            (size_t)SUB * WARPS * 2 * NS);
    }
};

template <bool FAST> struct Exp;
template <> struct Exp<true> {
    __device__ static float f(float x) { return __expf(x); }
    __device__ static double f(double x) { return ::exp(x); }
};
template <> struct Exp<false> {
    __device__ static float f(float x) { return expf(x); }
    __device__ static double f(double x) { return ::exp(x); }
};

template <typename IO, typename C, int NS>
__global__ void __launch_bounds__(Cfg<C, NS>::THREADS) fwd_kernel(
    const IO* __restrict__ u, const C* __restrict__ pre, const C* __restrict__ bdelta, const C* __restrict__ a_log,
    const C* __restrict__ Bk, const C* __restrict__ Ck, const C* __restrict__ Dskip, const C* __restrict__ x0,
    IO* __restrict__ y, C* __restrict__ ckpt, int64_t L, int64_t D, int N, int n_ck) {
    using CF = Cfg<C, NS>;
    using E = Exp<sizeof(IO) == 2>;
    using M = Math<C>;
    __shared__ C sB[kTT][NS], sC[kTT][NS];
    const int b = blockIdx.y;
    const int64_t d = (int64_t)blockIdx.x * CF::THREADS + threadIdx.x;
    const bool valid = d < D;
    C a[NS], x[NS];
#pragma unroll
    for (int n = 0; n < NS; ++n) {
        a[n] = (valid && n < N) ? -M::exp(a_log[d * N + n]) : C(0);
        x[n] = (x0 && valid && n < N) ? x0[((int64_t)b * D + d) * N + n] : C(0);
    }
    const C bd = valid ? bdelta[d] : C(0), Dd = valid ? Dskip[d] : C(0);
    for (int64_t t0 = 0; t0 < L; t0 += kTT) {
        const int nt = (int)min((int64_t)kTT, L - t0);
        __syncthreads();
        for (int i = threadIdx.x; i < kTT * NS; i += CF::THREADS) {
            const int k = i / NS, n = i % NS;
            const bool ok = k < nt && n < N;
            const int64_t off = ((int64_t)b * L + t0 + k) * N + n;
            sB[k][n] = ok ? C(cvt(Bk[off])) : C(0);
            sC[k][n] = ok ? C(cvt(Ck[off])) : C(0);
        }
        __syncthreads();
        IO uu[kTT];
        C pp[kTT];
#pragma unroll
        for (int k = 0; k < kTT; ++k) {
            const bool ok = valid && k < nt;
            const int64_t off = ((int64_t)b * L + t0 + k) * D + d;
            uu[k] = ok ? ld_stream(u + off) : IO(0);
            pp[k] = ok ? ld_stream(pre + off) : C(0);
        }
#pragma unroll
        for (int k = 0; k < kTT; ++k) {
            if (k < nt) {
                const int64_t t = t0 + k;
                if (valid && ckpt != nullptr && (t % CF::CK) == 0) {
                    C* cp = ckpt + (((int64_t)b * (n_ck + 1) + t / CF::CK) * D + d) * N;
#pragma unroll
                    for (int n = 0; n < NS; ++n)
                        if (n < N) cp[n] = x[n];
                }
                const C uk = cvt(uu[k]);
                const C delta = M::softplus(C(cvt(pp[k])) + bd);
                const C du = delta * uk;
                C yv = C(0);
#pragma unroll
                for (int n = 0; n < NS; ++n) {
                    const C ab = E::f(delta * a[n]);
                    x[n] = ab * x[n] + du * sB[k][n];
                    yv += x[n] * sC[k][n];
                }
                if (valid) st_io(y + ((int64_t)b * L + t) * D + d, yv + Dd * uk);
            }
        }
    }
    if (valid && ckpt != nullptr) {  // final state (prefill / return_state) in the last slot
        C* cp = ckpt + (((int64_t)b * (n_ck + 1) + n_ck) * D + d) * N;
#pragma unroll
        for (int n = 0; n < NS; ++n)
            if (n < N) cp[n] = x[n];
    }
}

// In-warp transpose reduction of NV values (NV a power of two <= 32): on
// return v[0] in lane l holds the warp-wide sum of value index (l % NV).
template <int NV>
__device__ __forceinline__ void tr_reduce(float* v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int m = NV / 2; m >= 1; m >>= 1) {
        const bool up = lane & m;
#pragma unroll
        for (int i = 0; i < m; ++i) {
            const float send = up ? v[i] : v[i + m];
            const float keep = up ? v[i + m] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
    }
#pragma unroll
    for (int m = NV; m < 32; m <<= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
}
template <int NV>
__device__ __forceinline__ void tr_reduce(double* v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int m = NV / 2; m >= 1; m >>= 1) {
        const bool up = lane & m;
#pragma unroll
        for (int i = 0; i < m; ++i) {
            const double send = up ? v[i] : v[i + m];
            const double keep = up ? v[i + m] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
    }
#pragma unroll
    for (int m = NV; m < 32; m <<= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
}

template <typename IO, typename C, int NS>
__global__ void __launch_bounds__(Cfg<C, NS>::THREADS) bwd_kernel(
    const IO* __restrict__ u, const C* __restrict__ pre, const C* __restrict__ bdelta, const C* __restrict__ a_log,
    const C* __restrict__ Bk, const C* __restrict__ Ck, const C* __restrict__ Dskip, const C* __restrict__ ckpt,
    const IO* __restrict__ gy, const C* __restrict__ h_in, IO* __restrict__ gu, C* __restrict__ gpre,
    C* __restrict__ gB_part, C* __restrict__ gC_part, C* __restrict__ ga_part, C* __restrict__ gD_part,
    C* __restrict__ gb_part, C* __restrict__ h_out, int64_t B, int64_t L, int64_t D, int N, int n_ck) {
    using CF = Cfg<C, NS>;
    using E = Exp<sizeof(IO) == 2>;
    using M = Math<C>;
    constexpr int TH = CF::THREADS, SUB = CF::SUB, NV = 2 * NS;
    constexpr int NVW = NV < 32 ? NV : 32;  // values per transpose-reduction round
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* subx = reinterpret_cast<C*>(smem_raw);            // [NSUB][NS][TH]
    C* xs = subx + (size_t)CF::NSUB * NS * TH;           // [SUB][NS][TH]
    C* sB = xs + (size_t)SUB * NS * TH;                  // [SUB][NS]
    C* sC = sB + (size_t)SUB * NS;                       // [SUB][NS]
    C* red = sC + (size_t)SUB * NS;                      // [SUB][WARPS][NV]

    const int b = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t d = (int64_t)blockIdx.x * TH + tid;
    const bool valid = d < D;
    C a[NS], h[NS], gacc[NS];
#pragma unroll
    for (int n = 0; n < NS; ++n) {
        a[n] = (valid && n < N) ? -M::exp(a_log[d * N + n]) : C(0);
        h[n] = (h_in && valid && n < N) ? h_in[((int64_t)b * D + d) * N + n] : C(0);
        gacc[n] = C(0);
    }
    const C bd = valid ? bdelta[d] : C(0), Dd = valid ? Dskip[d] : C(0);
    C gD_acc = 0, gb_acc = 0;

    for (int ci = n_ck - 1; ci >= 0; --ci) {
        const int64_t tc0 = (int64_t)ci * CF::CK;
        const int ncs = (int)min((int64_t)CF::CK, L - tc0);
        const int nsub = (ncs + SUB - 1) / SUB;
        C x[NS];
        {
            const C* cp = ckpt + (((int64_t)b * (n_ck + 1) + ci) * D + (valid ? d : 0)) * N;
#pragma unroll
            for (int n = 0; n < NS; ++n) x[n] = (valid && n < N) ? cp[n] : C(0);
        }
        // pass 1: chunk forward, keep the state entering every SUB block
        for (int j = 0; j < nsub; ++j) {
#pragma unroll
            for (int n = 0; n < NS; ++n) subx[((size_t)j * NS + n) * TH + tid] = x[n];
            const int64_t ts0 = tc0 + (int64_t)j * SUB;
            const int nts = (int)min((int64_t)SUB, L - ts0);
            for (int k = 0; k < nts; ++k) {
                const int64_t t = ts0 + k;
                const int64_t off = ((int64_t)b * L + t) * D + d;
                const C uk = valid ? C(cvt(u[off])) : C(0);
                const C delta = M::softplus((valid ? C(cvt(pre[off])) : C(0)) + bd);
                const C du = delta * uk;
                const C* brow = Bk + ((int64_t)b * L + t) * N;
#pragma unroll
                for (int n = 0; n < NS; ++n) {
                    const C bn = n < N ? C(cvt(brow[n])) : C(0);
                    x[n] = E::f(delta * a[n]) * x[n] + du * bn;
                }
            }
        }
        // pass 2: SUB blocks right-to-left
        for (int j = nsub - 1; j >= 0; --j) {
            const int64_t ts0 = tc0 + (int64_t)j * SUB;
            const int nts = (int)min((int64_t)SUB, L - ts0);
            __syncthreads();
            for (int i = tid; i < SUB * NS; i += TH) {
                const int k = i / NS, n = i % NS;
                const bool ok = k < nts && n < N;
                const int64_t off = ((int64_t)b * L + ts0 + k) * N + n;
                sB[i] = ok ? C(cvt(Bk[off])) : C(0);
                sC[i] = ok ? C(cvt(Ck[off])) : C(0);
            }
            __syncthreads();
            C uk[SUB], dl[SUB], gk[SUB], pk[SUB];
#pragma unroll
            for (int n = 0; n < NS; ++n) x[n] = subx[((size_t)j * NS + n) * TH + tid];
#pragma unroll
            for (int k = 0; k < SUB; ++k) {
                const bool ok = valid && k < nts;
                const int64_t off = ((int64_t)b * L + ts0 + k) * D + d;
                uk[k] = ok ? C(cvt(u[off])) : C(0);
                pk[k] = (ok ? C(cvt(pre[off])) : C(0)) + bd;
                gk[k] = ok ? C(cvt(gy[off])) : C(0);
                dl[k] = M::softplus(pk[k]);
            }
#pragma unroll
            for (int k = 0; k < SUB; ++k) {
                if (k < nts) {
                    const C du = dl[k] * uk[k];
#pragma unroll
                    for (int n = 0; n < NS; ++n) {
                        xs[((size_t)k * NS + n) * TH + tid] = x[n];
                        x[n] = E::f(dl[k] * a[n]) * x[n] + du * sB[k * NS + n];
                    }
                }
            }
#pragma unroll
            for (int k = SUB - 1; k >= 0; --k) {
                if (k < nts) {
                    const C du = dl[k] * uk[k];
                    C sa = 0, sb = 0;
                    C cv[NV];
#pragma unroll
                    for (int n = 0; n < NS; ++n) {
                        const C ab = E::f(dl[k] * a[n]);
                        const C xp = xs[((size_t)k * NS + n) * TH + tid];
                        const C bn = sB[k * NS + n], cn = sC[k * NS + n];
                        const C g = gk[k] * cn + h[n];
                        const C term = ab * (g * xp);       // abar * (g conj(x_{k-1}))
                        sa += term * a[n];
                        gacc[n] += term * dl[k];
                        sb += g * bn;
                        cv[n] = g * du;                      // -> dB_k[n]
                        cv[NS + n] = gk[k] * (ab * xp + du * bn);  // gy * x_k -> dC_k[n]
                        h[n] = ab * g;
                    }
                    const C gdelta = sa + sb * uk[k];
                    const C gp = M::sigmoid(pk[k]) * gdelta;
                    if (valid) {
                        const int64_t off = ((int64_t)b * L + ts0 + k) * D + d;
                        st_io(gu + off, Dd * gk[k] + dl[k] * sb);
                        st_io(gpre + off, gp);
                        gD_acc += gk[k] * uk[k];
                        gb_acc += gp;
                    } else {
#pragma unroll
                        for (int i = 0; i < NV; ++i) cv[i] = C(0);
                    }
#pragma unroll
                    for (int q = 0; q < NV; q += NVW) {
                        tr_reduce<NVW>(cv + q);
                        if (lane < NVW) red[((size_t)k * CF::WARPS + warp) * NV + q + lane] = cv[q];
                    }
                }
            }
            __syncthreads();
            const int64_t dblk = blockIdx.x;
            for (int i = tid; i < nts * NV; i += TH) {
                const int k = i / NV, v = i % NV;
                C sum = 0;
#pragma unroll
                for (int w = 0; w < CF::WARPS; ++w) sum += red[((size_t)k * CF::WARPS + w) * NV + v];
                const int n = v < NS ? v : v - NS;
                if (n < N) {
                    C* dst = v < NS ? gB_part : gC_part;
                    dst[((dblk * B + b) * L + ts0 + k) * N + n] = sum;
                }
            }
        }
    }
    if (valid) {
#pragma unroll
        for (int n = 0; n < NS; ++n)
            if (n < N) ga_part[((int64_t)b * D + d) * N + n] = a[n] * gacc[n];
        gD_part[(int64_t)b * D + d] = gD_acc;
        gb_part[(int64_t)b * D + d] = gb_acc;
        if (h_out) {
#pragma unroll
            for (int n = 0; n < NS; ++n)
                if (n < N) h_out[((int64_t)b * D + d) * N + n] = h[n];
        }
    }
}

// ============================================================================
// v2 (fp32 compute, d_state 16 / 32): TPC = 4 threads per channel, NPT states
// each.  4x the warps of the thread-per-channel mapping (C3 has only
// B*D = 24576 channels), softplus once per channel-step shared by shuffle,
// MUFU ex2 discretisation with a*log2(e) folded in, pairwise readout.
template <int NST>
struct V2 {
    static constexpr int TPC = 4;
    static constexpr int NPT = NST / TPC;
    static constexpr int FWD_T = 128;                 // threads per forward CTA
    static constexpr int BWD_T = 256;                 // = Cfg<float,NST>::THREADS channels * TPC
    static constexpr int CK = Cfg<float, NST>::CK;
    static constexpr int SUB = Cfg<float, NST>::SUB;
    static constexpr int NSUB = CK / SUB;
    static constexpr int NV = 2 * NPT;                // dB/dC values per thread per step
    static constexpr size_t smem_bwd() {
        return sizeof(float) * ((size_t)NSUB * NPT * BWD_T + (size_t)SUB * NPT * BWD_T + 2 * (size_t)SUB * NST +
                                (size_t)SUB * (BWD_T / 32) * TPC * NV);
    }
};
static_assert(V2<16>::BWD_T / V2<16>::TPC == Cfg<float, 16>::THREADS, "v2/v1 channel blocks must match");
static_assert(V2<32>::BWD_T / V2<32>::TPC == Cfg<float, 32>::THREADS, "v2/v1 channel blocks must match");

constexpr float kLog2e = 1.4426950408889634f;

// softplus for the compute path: x > 30 -> x; small e = e^x uses the series
// of log1p so delta keeps full relative precision (numerics.py:86-94).
__device__ __forceinline__ float softplus_fast(float x) {
    const float e = Fast<float>::ex2(fminf(x, 30.f) * kLog2e);
    const float lg = __log2f(1.f + e) * 0.6931471805599453f;
    const float ser = e * (1.f - e * (0.5f - e * (1.f / 3.f)));
    return x > 30.f ? x : (e < 1e-2f ? ser : lg);
}

// Transpose-reduction of NV values over the 8 lanes that share lane bits
// outside [2, 5) (the 8 channels of one state group in a warp).  On return
// v[chunk] holds, for value index chunk*8 + ((lane >> 2) & 7), the 8-lane sum.
template <int NV>
__device__ __forceinline__ void tr_reduce8(float* v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < NV; c += 8) {
#pragma unroll
        for (int m = 4; m >= 1; m >>= 1) {
            const bool up = (lane >> 2) & m;
#pragma unroll
            for (int i = 0; i < m; ++i) {
                const float send = up ? v[c + i] : v[c + i + m];
                const float keep = up ? v[c + i + m] : v[c + i];
                v[c + i] = keep + __shfl_xor_sync(0xffffffffu, send, m << 2);
            }
        }
        v[c / 8] = v[c];
    }
}

template <typename IO, int NST>
__global__ void __launch_bounds__(V2<NST>::FWD_T) fwd_v2_kernel(
    const IO* __restrict__ u, const float* __restrict__ pre, const float* __restrict__ bdelta,
    const float* __restrict__ a_log, const float* __restrict__ Bk, const float* __restrict__ Ck,
    const float* __restrict__ Dskip, const float* __restrict__ x0, IO* __restrict__ y, float* __restrict__ ckpt,
    int64_t L, int64_t D, int N, int n_ck) {
    using G = V2<NST>;
    constexpr int TPC = G::TPC, NPT = G::NPT, CPB = G::FWD_T / TPC;
    __shared__ float sB[kTT][NST], sC[kTT][NST];
    const int tid = threadIdx.x, lane = tid & 31, q = tid % TPC;
    const int b = blockIdx.y;
    const int64_t d = (int64_t)blockIdx.x * CPB + tid / TPC;
    const bool valid = d < D;
    const int n0 = q * NPT;
    float a2[NPT], x[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const int n = n0 + j;
        a2[j] = (valid && n < N) ? -__expf(a_log[d * N + n]) * kLog2e : 0.f;
        x[j] = (x0 && valid && n < N) ? x0[((int64_t)b * D + d) * N + n] : 0.f;
    }
    const float bd = valid ? bdelta[d] : 0.f, Dd = valid ? Dskip[d] : 0.f;
    const int gbase = lane & ~(TPC - 1);
    for (int64_t t0 = 0; t0 < L; t0 += kTT) {
        const int nt = (int)min((int64_t)kTT, L - t0);
        __syncthreads();
        for (int i = tid; i < kTT * NST; i += G::FWD_T) {
            const int k = i / NST, n = i % NST;
            const bool ok = k < nt && n < N;
            const int64_t off = ((int64_t)b * L + t0 + k) * N + n;
            sB[k][n] = ok ? Bk[off] : 0.f;
            sC[k][n] = ok ? Ck[off] : 0.f;
        }
        __syncthreads();
        IO uu[kTT];
        float dl_own[kTT / TPC];
#pragma unroll
        for (int k = 0; k < kTT; ++k) {
            const bool ok = valid && k < nt;
            uu[k] = ok ? u[((int64_t)b * L + t0 + k) * D + d] : IO(0);
        }
#pragma unroll
        for (int kk = 0; kk < kTT / TPC; ++kk) {
            const int k = kk * TPC + q;
            const bool ok = valid && k < nt;
            const float p = ok ? pre[((int64_t)b * L + t0 + k) * D + d] : 0.f;
            dl_own[kk] = softplus_fast(p + bd);
        }
#pragma unroll
        for (int k = 0; k < kTT; ++k) {
            const float delta = __shfl_sync(0xffffffffu, dl_own[k / TPC], gbase | (k % TPC));
            if (k < nt) {
                const int64_t t = t0 + k;
                if (valid && ckpt != nullptr && (t % G::CK) == 0) {
                    float* cp = ckpt + (((int64_t)b * (n_ck + 1) + t / G::CK) * D + d) * N + n0;
#pragma unroll
                    for (int j = 0; j < NPT; ++j)
                        if (n0 + j < N) cp[j] = x[j];
                }
                const float uk = cvt(uu[k]);
                const float du = delta * uk;
                float yp[NPT];
#pragma unroll
                for (int j = 0; j < NPT; ++j) {
                    const float ab = Fast<float>::ex2(delta * a2[j]);
                    x[j] = fmaf(ab, x[j], du * sB[k][n0 + j]);
                    yp[j] = x[j] * sC[k][n0 + j];
                }
#pragma unroll
                for (int w2 = NPT / 2; w2 >= 1; w2 >>= 1)
#pragma unroll
                    for (int j = 0; j < w2; ++j) yp[j] += yp[j + w2];
                float yv = yp[0];
                yv += __shfl_xor_sync(0xffffffffu, yv, 1);
                yv += __shfl_xor_sync(0xffffffffu, yv, 2);
                if (valid && q == 0) st_io(y + ((int64_t)b * L + t) * D + d, yv + Dd * uk);
            }
        }
    }
    if (valid && ckpt != nullptr) {
        float* cp = ckpt + (((int64_t)b * (n_ck + 1) + n_ck) * D + d) * N + n0;
#pragma unroll
        for (int j = 0; j < NPT; ++j)
            if (n0 + j < N) cp[j] = x[j];
    }
}

template <typename IO, int NST>
__global__ void __launch_bounds__(V2<NST>::BWD_T) bwd_v2_kernel(
    const IO* __restrict__ u, const float* __restrict__ pre, const float* __restrict__ bdelta,
    const float* __restrict__ a_log, const float* __restrict__ Bk, const float* __restrict__ Ck,
    const float* __restrict__ Dskip, const float* __restrict__ ckpt, const IO* __restrict__ gy,
    const float* __restrict__ h_in, IO* __restrict__ gu, float* __restrict__ gpre, float* __restrict__ gB_part,
    float* __restrict__ gC_part, float* __restrict__ ga_part, float* __restrict__ gD_part,
    float* __restrict__ gb_part, float* __restrict__ h_out, int64_t B, int64_t L, int64_t D, int N, int n_ck) {
    using G = V2<NST>;
    constexpr int TH = G::BWD_T, TPC = G::TPC, NPT = G::NPT, SUB = G::SUB, NV = G::NV, WARPS = TH / 32;
    constexpr int CPB = TH / TPC;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* subx = reinterpret_cast<float*>(smem_raw);             // [NSUB][NPT][TH]
    float* xs = subx + (size_t)G::NSUB * NPT * TH;                // [SUB][NPT][TH]
    float* sB = xs + (size_t)SUB * NPT * TH;                      // [SUB][NST]
    float* sC = sB + (size_t)SUB * NST;                           // [SUB][NST]
    float* red = sC + (size_t)SUB * NST;                          // [SUB][WARPS][TPC*NV]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q = tid % TPC;
    const int b = blockIdx.y;
    const int64_t d = (int64_t)blockIdx.x * CPB + tid / TPC;
    const bool valid = d < D;
    const int n0 = q * NPT;
    const int gbase = lane & ~(TPC - 1);
    float a[NPT], a2[NPT], h[NPT], gacc[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const int n = n0 + j;
        a[j] = (valid && n < N) ? -__expf(a_log[d * N + n]) : 0.f;
        a2[j] = a[j] * kLog2e;
        h[j] = (h_in && valid && n < N) ? h_in[((int64_t)b * D + d) * N + n] : 0.f;
        gacc[j] = 0.f;
    }
    const float bd = valid ? bdelta[d] : 0.f, Dd = valid ? Dskip[d] : 0.f;
    float gD_acc = 0.f, gb_acc = 0.f;

    // delta for step t (shared by the TPC lanes of a channel): lane q computes
    // the steps k with k % TPC == q of a SUB block
    auto deltas = [&](int64_t ts0, int nts, float* dl_own) {
#pragma unroll
        for (int kk = 0; kk < SUB / TPC; ++kk) {
            const int k = kk * TPC + q;
            const bool ok = valid && k < nts;
            const float p = ok ? pre[((int64_t)b * L + ts0 + k) * D + d] : 0.f;
            dl_own[kk] = softplus_fast(p + bd);
        }
    };

    for (int ci = n_ck - 1; ci >= 0; --ci) {
        const int64_t tc0 = (int64_t)ci * G::CK;
        const int ncs = (int)min((int64_t)G::CK, L - tc0);
        const int nsub = (ncs + SUB - 1) / SUB;
        float x[NPT];
        {
            const float* cp = ckpt + (((int64_t)b * (n_ck + 1) + ci) * D + (valid ? d : 0)) * N + n0;
#pragma unroll
            for (int j = 0; j < NPT; ++j) x[j] = (valid && n0 + j < N) ? cp[j] : 0.f;
        }
        // pass 1: chunk forward, keep the state entering every SUB block
        for (int jb = 0; jb < nsub; ++jb) {
#pragma unroll
            for (int j = 0; j < NPT; ++j) subx[((size_t)jb * NPT + j) * TH + tid] = x[j];
            const int64_t ts0 = tc0 + (int64_t)jb * SUB;
            const int nts = (int)min((int64_t)SUB, L - ts0);
            float dl_own[SUB / TPC];
            deltas(ts0, nts, dl_own);
#pragma unroll
            for (int k = 0; k < SUB; ++k) {
                const float delta = __shfl_sync(0xffffffffu, dl_own[k / TPC], gbase | (k % TPC));
                if (k < nts) {
                    const int64_t t = ts0 + k;
                    const float uk = valid ? float(cvt(u[((int64_t)b * L + t) * D + d])) : 0.f;
                    const float du = delta * uk;
                    const float* brow = Bk + ((int64_t)b * L + t) * N + n0;
#pragma unroll
                    for (int j = 0; j < NPT; ++j) {
                        const float bn = n0 + j < N ? brow[j] : 0.f;
                        x[j] = fmaf(Fast<float>::ex2(delta * a2[j]), x[j], du * bn);
                    }
                }
            }
        }
        // pass 2: SUB blocks right-to-left
        for (int jb = nsub - 1; jb >= 0; --jb) {
            const int64_t ts0 = tc0 + (int64_t)jb * SUB;
            const int nts = (int)min((int64_t)SUB, L - ts0);
            __syncthreads();
            for (int i = tid; i < SUB * NST; i += TH) {
                const int k = i / NST, n = i % NST;
                const bool ok = k < nts && n < N;
                const int64_t off = ((int64_t)b * L + ts0 + k) * N + n;
                sB[i] = ok ? Bk[off] : 0.f;
                sC[i] = ok ? Ck[off] : 0.f;
            }
            __syncthreads();
            float dl_own[SUB / TPC], uk[SUB], gk[SUB];
            deltas(ts0, nts, dl_own);
#pragma unroll
            for (int j = 0; j < NPT; ++j) x[j] = subx[((size_t)jb * NPT + j) * TH + tid];
#pragma unroll
            for (int k = 0; k < SUB; ++k) {
                const bool ok = valid && k < nts;
                const int64_t off = ((int64_t)b * L + ts0 + k) * D + d;
                uk[k] = ok ? float(cvt(u[off])) : 0.f;
                gk[k] = ok ? float(cvt(gy[off])) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < SUB; ++k) {
                const float delta = __shfl_sync(0xffffffffu, dl_own[k / TPC], gbase | (k % TPC));
                if (k < nts) {
                    const float du = delta * uk[k];
#pragma unroll
                    for (int j = 0; j < NPT; ++j) {
                        xs[((size_t)k * NPT + j) * TH + tid] = x[j];
                        x[j] = fmaf(Fast<float>::ex2(delta * a2[j]), x[j], du * sB[k * NST + n0 + j]);
                    }
                }
            }
#pragma unroll
            for (int k = SUB - 1; k >= 0; --k) {
                const float delta = __shfl_sync(0xffffffffu, dl_own[k / TPC], gbase | (k % TPC));
                if (k < nts) {
                    const float du = delta * uk[k];
                    float sa = 0.f, sb = 0.f;
                    float cv[NV];
#pragma unroll
                    for (int j = 0; j < NPT; ++j) {
                        const float ab = Fast<float>::ex2(delta * a2[j]);
                        const float xp = xs[((size_t)k * NPT + j) * TH + tid];
                        const float bn = sB[k * NST + n0 + j], cn = sC[k * NST + n0 + j];
                        const float g = fmaf(gk[k], cn, h[j]);
                        const float term = ab * (g * xp);
                        sa = fmaf(term, a[j], sa);
                        gacc[j] = fmaf(term, delta, gacc[j]);
                        sb = fmaf(g, bn, sb);
                        cv[j] = g * du;
                        cv[NPT + j] = gk[k] * fmaf(ab, xp, du * bn);
                        h[j] = ab * g;
                    }
                    sa += __shfl_xor_sync(0xffffffffu, sa, 1);
                    sb += __shfl_xor_sync(0xffffffffu, sb, 1);
                    sa += __shfl_xor_sync(0xffffffffu, sa, 2);
                    sb += __shfl_xor_sync(0xffffffffu, sb, 2);
                    if (valid && q == 0) {
                        const float p = pre[((int64_t)b * L + ts0 + k) * D + d] + bd;
                        const float gp = Fast<float>::sigmoid(p) * fmaf(sb, uk[k], sa);
                        const int64_t off = ((int64_t)b * L + ts0 + k) * D + d;
                        st_io(gu + off, fmaf(Dd, gk[k], delta * sb));
                        gpre[off] = gp;
                        gD_acc = fmaf(gk[k], uk[k], gD_acc);
                        gb_acc += gp;
                    }
                    if (!valid) {
#pragma unroll
                        for (int i = 0; i < NV; ++i) cv[i] = 0.f;
                    }
                    tr_reduce8<NV>(cv);
                    const int c = (lane >> 2) & 7;
#pragma unroll
                    for (int ch = 0; ch < NV / 8; ++ch)
                        red[((size_t)k * WARPS + warp) * (TPC * NV) + q * NV + ch * 8 + c] = cv[ch];
                }
            }
            __syncthreads();
            const int64_t dblk = blockIdx.x;
            for (int i = tid; i < nts * TPC * NV; i += TH) {
                const int k = i / (TPC * NV), r = i % (TPC * NV);
                float sum = 0.f;
#pragma unroll
                for (int w = 0; w < WARPS; ++w) sum += red[((size_t)k * WARPS + w) * (TPC * NV) + r];
                const int qq = r / NV, v = r % NV;
                const int n = qq * NPT + (v < NPT ? v : v - NPT);
                if (n < N) {
                    float* dst = v < NPT ? gB_part : gC_part;
                    dst[((dblk * B + b) * L + ts0 + k) * N + n] = sum;
                }
            }
        }
    }
    if (valid) {
#pragma unroll
        for (int j = 0; j < NPT; ++j)
            if (n0 + j < N) ga_part[((int64_t)b * D + d) * N + n0 + j] = a[j] * gacc[j];
        if (q == 0) {
            gD_part[(int64_t)b * D + d] = gD_acc;
            gb_part[(int64_t)b * D + d] = gb_acc;
        }
        if (h_out) {  // carry to the left of step 0: abar_0 g_0 (= d loss / d x0)
#pragma unroll
            for (int j = 0; j < NPT; ++j)
                if (n0 + j < N) h_out[((int64_t)b * D + d) * N + n0 + j] = h[j];
        }
    }
}

template <typename C>
static int pick_ns(int64_t N) {
    if (N <= 4) return 4;
    if (N <= 8) return 8;
    if (N <= 16) return 16;
    if (N <= 32) return 32;
    if (N <= 64) return 64;
    return 0;
}

template <typename C, int NS>
static void geom(int64_t L, int64_t D, int* ck, int* n_ck, int* n_dblk) {
    *ck = Cfg<C, NS>::CK;
    *n_ck = (int)cdiv(L, Cfg<C, NS>::CK);
    *n_dblk = (int)cdiv(D, Cfg<C, NS>::THREADS);
}

template <typename C>
static int geom_rt(int64_t L, int64_t D, int64_t N, int* ck, int* n_ck, int* n_dblk) {
    switch (pick_ns<C>(N)) {
        case 4: geom<C, 4>(L, D, ck, n_ck, n_dblk); return 4;
        case 8: geom<C, 8>(L, D, ck, n_ck, n_dblk); return 8;
        case 16: geom<C, 16>(L, D, ck, n_ck, n_dblk); return 16;
        case 32: geom<C, 32>(L, D, ck, n_ck, n_dblk); return 32;
        case 64: geom<C, 64>(L, D, ck, n_ck, n_dblk); return 64;
    }
    return 0;
}

template <typename IO, typename C, int NS>
static int fwd_launch(const void* u, const void* pre, const void* bd, const void* al, const void* Bk, const void* Ck,
                      const void* Dk, const void* x0, void* y, void* ckpt, int64_t B, int64_t L, int64_t D,
                      int64_t N, cudaStream_t st) {
    using CF = Cfg<C, NS>;
    if constexpr (sizeof(C) == 4 && (NS == 16 || NS == 32)) {
        if (!getenv("LRX_S6_V1")) {
            using G = V2<NS>;
            const dim3 grid((unsigned)cdiv(D, G::FWD_T / G::TPC), (unsigned)B);
            fwd_v2_kernel<IO, NS><<<grid, G::FWD_T, 0, st>>>((const IO*)u, (const float*)pre, (const float*)bd,
                                                              (const float*)al, (const float*)Bk, (const float*)Ck,
                                                              (const float*)Dk, (const float*)x0, (IO*)y,
                                                              (float*)ckpt, L, D, (int)N, (int)cdiv(L, G::CK));
            return launched("lrx_s6_fwd/v2");
        }
    }
    const dim3 grid((unsigned)cdiv(D, CF::THREADS), (unsigned)B);
    fwd_kernel<IO, C, NS><<<grid, CF::THREADS, 0, st>>>((const IO*)u, (const C*)pre, (const C*)bd, (const C*)al,
                                                        (const C*)Bk, (const C*)Ck, (const C*)Dk, (const C*)x0,
                                                        (IO*)y, (C*)ckpt, L, D, (int)N, (int)cdiv(L, CF::CK));
    return launched("lrx_s6_fwd");
}

template <typename IO, typename C, int NS>
static int bwd_launch(const void* u, const void* pre, const void* bd, const void* al, const void* Bk, const void* Ck,
                      const void* Dk, const void* ckpt, const void* gy, const void* h_in, void* gu, void* gpre,
                      void* gBp, void* gCp, void* gap, void* gDp, void* gbp, void* h_out, int64_t B, int64_t L,
                      int64_t D, int64_t N, cudaStream_t st) {
    using CF = Cfg<C, NS>;
    if constexpr (sizeof(C) == 4 && (NS == 16 || NS == 32)) {
        if (!getenv("LRX_S6_V1")) {
            using G = V2<NS>;
            const size_t smem2 = G::smem_bwd();
            auto k2 = bwd_v2_kernel<IO, NS>;
            if (cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2) != cudaSuccess) {
                set_error("s6 bwd: cannot reserve %zu bytes of shared memory", smem2);
                return LRX_ERR_CUDA;
            }
            const dim3 grid((unsigned)cdiv(D, G::BWD_T / G::TPC), (unsigned)B);
            k2<<<grid, G::BWD_T, smem2, st>>>((const IO*)u, (const float*)pre, (const float*)bd, (const float*)al,
                                              (const float*)Bk, (const float*)Ck, (const float*)Dk,
                                              (const float*)ckpt, (const IO*)gy, (const float*)h_in, (IO*)gu,
                                              (float*)gpre, (float*)gBp, (float*)gCp, (float*)gap, (float*)gDp,
                                              (float*)gbp, (float*)h_out, B, L, D, (int)N, (int)cdiv(L, G::CK));
            return launched("lrx_s6_bwd/v2");
        }
    }
    const size_t smem = CF::smem_bwd();
    auto kfn = bwd_kernel<IO, C, NS>;
    if (smem > 48 * 1024) {
        if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
            set_error("s6 bwd: cannot reserve %zu bytes of shared memory", smem);
            return LRX_ERR_CUDA;
        }
    }
    const dim3 grid((unsigned)cdiv(D, CF::THREADS), (unsigned)B);
    kfn<<<grid, CF::THREADS, smem, st>>>((const IO*)u, (const C*)pre, (const C*)bd, (const C*)al, (const C*)Bk,
                                         (const C*)Ck, (const C*)Dk, (const C*)ckpt, (const IO*)gy,
                                         (const C*)h_in, (IO*)gu, (C*)gpre, (C*)gBp, (C*)gCp, (C*)gap, (C*)gDp,
                                         (C*)gbp, (C*)h_out, B, L, D, (int)N, (int)cdiv(L, CF::CK));
    return launched("lrx_s6_bwd");
}

#define S6_NS_SWITCH(C, N, CALL)                                                \
    switch (pick_ns<C>(N)) {                                                     \
        case 4: { constexpr int NS = 4; return CALL; }                           \
        case 8: { constexpr int NS = 8; return CALL; }                           \
        case 16: { constexpr int NS = 16; return CALL; }                         \
        case 32: { constexpr int NS = 32; return CALL; }                         \
        case 64: { constexpr int NS = 64; return CALL; }                         \
        default: set_error("s6: d_state %lld > 64 is not compiled", (long long)N); \
            return LRX_ERR_UNSUPPORTED;                                          \
    }

#define LRX_S6_FWD_PARAMS const void* u, const void* pre, const void* bd, const void* al, const void* Bk, \
    const void* Ck, const void* Dk, const void* x0, void* y, void* ckpt, int64_t B, int64_t L, int64_t D,  \
    int64_t N, cudaStream_t st
#define LRX_S6_BWD_PARAMS const void* u, const void* pre, const void* bd, const void* al, const void* Bk, \
    const void* Ck, const void* Dk, const void* ckpt, const void* gy, const void* h_in, void* gu, void* gpre, \
    void* gBp, void* gCp, void* gap, void* gDp, void* gbp, void* h_out, int64_t B, int64_t L, int64_t D,   \
    int64_t N, cudaStream_t st

template <typename IO, typename C>
static int fwd_t(LRX_S6_FWD_PARAMS) {
    S6_NS_SWITCH(C, N, (fwd_launch<IO, C, NS>(u, pre, bd, al, Bk, Ck, Dk, x0, y, ckpt, B, L, D, N, st)))
}

template <typename IO, typename C>
static int bwd_t(LRX_S6_BWD_PARAMS) {
    S6_NS_SWITCH(C, N, (bwd_launch<IO, C, NS>(u, pre, bd, al, Bk, Ck, Dk, ckpt, gy, h_in, gu, gpre, gBp, gCp, gap,
                                              gDp, gbp, h_out, B, L, D, N, st)))
}

// per-I/O-dtype entry points, each compiled in its own translation unit
int fwd_f32(LRX_S6_FWD_PARAMS);
int fwd_bf16(LRX_S6_FWD_PARAMS);
int fwd_f64(LRX_S6_FWD_PARAMS);
int bwd_f32(LRX_S6_BWD_PARAMS);
int bwd_bf16(LRX_S6_BWD_PARAMS);
int bwd_f64(LRX_S6_BWD_PARAMS);

}  // namespace s6
}  // namespace lrx

