// S4D (per-channel complex diagonal LTI, constant step) fused forward /
// backward: the scan, the input map w u and the readout Re(sum_n c x) + d u
// in one pass, without the [B, L, H, N] complex planes of the generic path.
//
// Reference: pkg/src/linrec/layers.py S4D 352-546: _forward_tape 453-473
// (x_n = abar_n x_n + w_n u, y = Re(sum_n c_n x_n) + d u with w = scale b,
// discretize.py:59-142), _backward 477-546 (g_n = conj(c_n) gy +
// conj(abar_n) g_n(next); d abar = sum g conj(x_prev), d w-path = sum g u,
// dc = sum gy conj(x), du = d gy + Re(sum_n g conj(w)), dd = sum gy u).
//
// Lanes (b, h, n) with n fastest.  A warp is one channel (N = 64: two states
// per lane) or 32/N channels (N = 8, 16, 32).  Time runs in tiles of TT = 16
// steps: the per-step readout partials of a lane stay in registers for the
// tile, then one transposed butterfly over the channel's lanes leaves each
// lane with whole sums for 16/G of the steps (G = lanes per channel).  The
// forward writes the entering state of every tile (checkpoints); the backward
// walks tiles right to left, recomputes the tile's states from its checkpoint
// into registers and runs the reverse recurrence.  Parameter-gradient sums
// are per (b, h, n) partials, summed over b by the caller in fixed order.
#include "lrx_common.cuh"
#include "lrx_host.h"

namespace lrx {
namespace s4d {

constexpr int TT = 16;  // steps per tile (checkpoint interval)

// transposed butterfly over lane bits HI..LO (see lrx_s6v3.cu tr_reduce)
// (one level per template instance: the halves are compile-time, so the
// per-lane selection stays a value select and the arrays stay in registers)
template <typename T, int CNT, int M, int LO>
__device__ __forceinline__ void tr_level(T* v) {
    if constexpr (M >= LO && CNT >= 2) {
        constexpr int half = CNT / 2;
        const bool up = (threadIdx.x & 31) & M;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const T a = v[i], b = v[i + half];
            const T send = up ? a : b;
            const T keep = up ? b : a;
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, M);
        }
        tr_level<T, half, M / 2, LO>(v);
    }
}
template <typename T, int V, int HI, int LO>
__device__ __forceinline__ void tr_reduce(T* v) {
    tr_level<T, V, HI, LO>(v);
}

// G = lanes per channel (min(N, 32)), NPL = states per lane (N / G)
// After the reduction lane r holds whole-channel sums in v[0 .. PER) for
// steps step0(r) + i; G = 32 (more lanes than steps): lane pairs hold the
// same step and the even lane writes it.
template <typename T, int G>
__device__ __forceinline__ void reduce_tile(T* v) {
    if constexpr (G == 32) {
        tr_reduce<T, TT, 16, 2>(v);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    } else if constexpr (G == 16) {
        tr_reduce<T, TT, 8, 1>(v);
    } else {
        tr_reduce<T, TT, 4, 1>(v);
    }
}
template <int G> struct Out {
    static constexpr int PER = G == 32 ? 1 : TT / G;
    __device__ static bool writer(int r) { return G == 32 ? !(r & 1) : true; }
    __device__ static int step0(int r) { return G == 32 ? r >> 1 : r * PER; }
};

template <typename T, int G, int NPL>
__global__ void __launch_bounds__(128) fwd_kernel(const T* __restrict__ u, const cplx<T>* __restrict__ abar,
                                                  const cplx<T>* __restrict__ w, const cplx<T>* __restrict__ c,
                                                  const T* __restrict__ d, T* __restrict__ y,
                                                  cplx<T>* __restrict__ ckpt, cplx<T>* __restrict__ xlast, int64_t B,
                                                  int64_t L, int64_t H) {
    constexpr int N = G * NPL;
    const int64_t lane_id = (int64_t)blockIdx.x * 128 + threadIdx.x;  // (b, h, r) with r = lane in channel
    const int64_t n_lanes = B * H * G;
    const bool live = lane_id < n_lanes;
    const int64_t ch = (live ? lane_id : n_lanes - 1) / G;  // (b, h)
    const int r = (int)(lane_id % G);
    const int64_t b = ch / H, h = ch % H;
    cplx<T> ab[NPL], ww[NPL], cc[NPL], x[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
        const int64_t n = h * N + r * NPL + j;
        ab[j] = abar[n], ww[j] = w[n], cc[j] = c[n];
        x[j] = Traits<cplx<T>>::zero();
    }
    const T dd = d[h];
    const T* up = u + b * L * H + h;
    T* yp = y + b * L * H + h;
    const int64_t n_ck = (L + TT - 1) / TT;
    for (int64_t t0 = 0; t0 < L; t0 += TT) {
        if (live) {
#pragma unroll
            for (int j = 0; j < NPL; ++j)
                ckpt[((b * n_ck + t0 / TT) * H + h) * N + r * NPL + j] = x[j];
        }
        const int nt = (int)min((int64_t)TT, L - t0);
        T uu[TT], part[TT];
#pragma unroll
        for (int k = 0; k < TT; ++k) uu[k] = k < nt ? up[(t0 + k) * H] : T(0);
#pragma unroll
        for (int k = 0; k < TT; ++k) {
            T s = 0;
#pragma unroll
            for (int j = 0; j < NPL; ++j) {
                if (k < nt) x[j] = ab[j] * x[j] + uu[k] * ww[j];  // ragged last tile: state stops at L-1
                s += cc[j].re * x[j].re - cc[j].im * x[j].im;
            }
            part[k] = s;
        }
        reduce_tile<T, G>(part);
        if (live && Out<G>::writer(r)) {
#pragma unroll
            for (int i = 0; i < Out<G>::PER; ++i) {
                const int k = Out<G>::step0(r) + i;
                if (k < nt) yp[(t0 + k) * H] = part[i] + dd * up[(t0 + k) * H];
            }
        }
    }
    if (xlast && live) {
#pragma unroll
        for (int j = 0; j < NPL; ++j) xlast[(b * H + h) * N + r * NPL + j] = x[j];
    }
}

template <typename T, int G, int NPL>
__global__ void __launch_bounds__(128) bwd_kernel(const T* __restrict__ u, const T* __restrict__ gy,
                                                  const cplx<T>* __restrict__ abar, const cplx<T>* __restrict__ w,
                                                  const cplx<T>* __restrict__ c, const T* __restrict__ d,
                                                  const cplx<T>* __restrict__ ckpt, T* __restrict__ gu,
                                                  cplx<T>* __restrict__ gab_p, cplx<T>* __restrict__ gw_p,
                                                  cplx<T>* __restrict__ gc_p, T* __restrict__ gd_p, int64_t B,
                                                  int64_t L, int64_t H) {
    constexpr int N = G * NPL;
    const int64_t lane_id = (int64_t)blockIdx.x * 128 + threadIdx.x;
    const int64_t n_lanes = B * H * G;
    const bool live = lane_id < n_lanes;
    const int64_t ch = (live ? lane_id : n_lanes - 1) / G;
    const int r = (int)(lane_id % G);
    const int64_t b = ch / H, h = ch % H;
    cplx<T> ab[NPL], abc[NPL], wc[NPL], ccc[NPL], hc[NPL], sab[NPL], sw[NPL], sc[NPL];
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
        const int64_t n = h * N + r * NPL + j;
        ab[j] = abar[n], abc[j] = conj(ab[j]), wc[j] = conj(w[n]), ccc[j] = conj(c[n]);
        hc[j] = sab[j] = sw[j] = sc[j] = Traits<cplx<T>>::zero();
    }
    const T dd = d[h];
    T sd = 0;
    const T* up = u + b * L * H + h;
    const T* gp = gy + b * L * H + h;
    T* gup = gu + b * L * H + h;
    const int64_t n_ck = (L + TT - 1) / TT;
    for (int64_t t0 = (n_ck - 1) * TT; t0 >= 0; t0 -= TT) {
        const int nt = (int)min((int64_t)TT, L - t0);
        T uu[TT], gg[TT], part[TT];
#pragma unroll
        for (int k = 0; k < TT; ++k) {
            uu[k] = k < nt ? up[(t0 + k) * H] : T(0);
            gg[k] = k < nt ? gp[(t0 + k) * H] : T(0);
        }
        // states of the tile: hist[k] = x_{t0+k-1}; xe = x_{t0+nt-1}
        cplx<T> hist[TT][NPL], xs[NPL];
#pragma unroll
        for (int j = 0; j < NPL; ++j) xs[j] = ckpt[((b * n_ck + t0 / TT) * H + h) * N + r * NPL + j];
#pragma unroll
        for (int k = 0; k < TT; ++k)
#pragma unroll
            for (int j = 0; j < NPL; ++j) {
                hist[k][j] = xs[j];
                if (k < nt) xs[j] = ab[j] * xs[j] + uu[k] * conj(wc[j]);
            }
#pragma unroll
        for (int k = TT - 1; k >= 0; --k) {
            T s = 0;
            if (k < nt) {
#pragma unroll
                for (int j = 0; j < NPL; ++j) {
                    const cplx<T> xk = k + 1 < TT ? hist[k + 1 < TT ? k + 1 : 0][j] : xs[j];
                    const cplx<T> xcur = (k == nt - 1) ? xs[j] : xk;
                    const cplx<T> g = gg[k] * ccc[j] + hc[j];
                    hc[j] = abc[j] * g;
                    sab[j] = sab[j] + g * conj(hist[k][j]);
                    sw[j] = sw[j] + uu[k] * g;
                    sc[j] = sc[j] + gg[k] * conj(xcur);
                    const cplx<T> gwc = g * wc[j];
                    s += gwc.re;
                }
                if (r == 0) sd += gg[k] * uu[k];
            }
            part[k] = s;
        }
        reduce_tile<T, G>(part);
        if (live && Out<G>::writer(r)) {
#pragma unroll
            for (int i = 0; i < Out<G>::PER; ++i) {
                const int k = Out<G>::step0(r) + i;
                if (k < nt) gup[(t0 + k) * H] = part[i] + dd * gp[(t0 + k) * H];
            }
        }
    }
    if (!live) return;
#pragma unroll
    for (int j = 0; j < NPL; ++j) {
        const int64_t o = (b * H + h) * N + r * NPL + j;
        gab_p[o] = sab[j];
        gw_p[o] = sw[j];
        gc_p[o] = sc[j];
    }
    if (r == 0) gd_p[b * H + h] = sd;
}

template <typename T>
static int fwd_t(const void* u, const void* abar, const void* w, const void* c, const void* d, void* y, void* ckpt,
                 void* xlast, int64_t B, int64_t L, int64_t H, int64_t N, cudaStream_t st) {
    const int64_t G = N < 32 ? N : 32;
    const unsigned grid = (unsigned)cdiv(B * H * G, 128);
#define S4D_FWD(G_, NPL_)                                                                                       \
    fwd_kernel<T, G_, NPL_><<<grid, 128, 0, st>>>((const T*)u, (const cplx<T>*)abar, (const cplx<T>*)w,        \
                                                   (const cplx<T>*)c, (const T*)d, (T*)y, (cplx<T>*)ckpt,           \
                                                   (cplx<T>*)xlast, B, L, H)
    switch (N) {
        case 8: S4D_FWD(8, 1); break;
        case 16: S4D_FWD(16, 1); break;
        case 32: S4D_FWD(32, 1); break;
        case 64: S4D_FWD(32, 2); break;
        default: set_error("s4d fused: d_state %lld not in {8, 16, 32, 64}", (long long)N); return LRX_ERR_UNSUPPORTED;
    }
#undef S4D_FWD
    return launched("lrx_s4d_fwd");
}

template <typename T>
static int bwd_t(const void* u, const void* gy, const void* abar, const void* w, const void* c, const void* d,
                 const void* ckpt, void* gu, void* gab, void* gw, void* gc, void* gd, int64_t B, int64_t L, int64_t H,
                 int64_t N, cudaStream_t st) {
    const int64_t G = N < 32 ? N : 32;
    const unsigned grid = (unsigned)cdiv(B * H * G, 128);
#define S4D_BWD(G_, NPL_)                                                                                        \
    bwd_kernel<T, G_, NPL_><<<grid, 128, 0, st>>>((const T*)u, (const T*)gy, (const cplx<T>*)abar,              \
                                                   (const cplx<T>*)w, (const cplx<T>*)c, (const T*)d,           \
                                                   (const cplx<T>*)ckpt, (T*)gu, (cplx<T>*)gab, (cplx<T>*)gw,   \
                                                   (cplx<T>*)gc, (T*)gd, B, L, H)
    switch (N) {
        case 8: S4D_BWD(8, 1); break;
        case 16: S4D_BWD(16, 1); break;
        case 32: S4D_BWD(32, 1); break;
        case 64: S4D_BWD(32, 2); break;
        default: set_error("s4d fused: d_state %lld not in {8, 16, 32, 64}", (long long)N); return LRX_ERR_UNSUPPORTED;
    }
#undef S4D_BWD
    return launched("lrx_s4d_bwd");
}

}  // namespace s4d
}  // namespace lrx

using namespace lrx;

extern "C" {

int lrx_s4d_chunking(int64_t L, int64_t* chunk_len, int64_t* n_chunks) {
    LRX_REQUIRE(L >= 1, LRX_ERR_SHAPE, "length must be >= 1");
    *chunk_len = s4d::TT;
    *n_chunks = cdiv(L, (int64_t)s4d::TT);
    return LRX_OK;
}

int lrx_s4d_fwd(int dtype, const void* u, const void* abar, const void* w, const void* c, const void* d, void* y,
                void* ckpt, void* xlast, int64_t B, int64_t L, int64_t H, int64_t N, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && H >= 1 && N >= 1, LRX_ERR_SHAPE, "s4d: bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == LRX_F32) return s4d::fwd_t<float>(u, abar, w, c, d, y, ckpt, xlast, B, L, H, N, st);
    if (dtype == LRX_F64) return s4d::fwd_t<double>(u, abar, w, c, d, y, ckpt, xlast, B, L, H, N, st);
    set_error("s4d: dtype %d (f32 / f64)", dtype);
    return LRX_ERR_VALUE;
}

int lrx_s4d_bwd(int dtype, const void* u, const void* gy, const void* abar, const void* w, const void* c,
                const void* d, const void* ckpt, void* gu, void* gabar_part, void* gw_part, void* gc_part,
                void* gd_part, int64_t B, int64_t L, int64_t H, int64_t N, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && H >= 1 && N >= 1, LRX_ERR_SHAPE, "s4d: bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == LRX_F32)
        return s4d::bwd_t<float>(u, gy, abar, w, c, d, ckpt, gu, gabar_part, gw_part, gc_part, gd_part, B, L, H, N,
                                 st);
    if (dtype == LRX_F64)
        return s4d::bwd_t<double>(u, gy, abar, w, c, d, ckpt, gu, gabar_part, gw_part, gc_part, gd_part, B, L, H, N,
                                  st);
    set_error("s4d: dtype %d (f32 / f64)", dtype);
    return LRX_ERR_VALUE;
}

}  // extern "C"
