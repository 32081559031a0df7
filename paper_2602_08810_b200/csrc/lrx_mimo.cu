// Complex diagonal LTI scan between the dense projections of S5 / LRU.
//
// Reference: pkg/src/linrec/layers.py _MIMOBase (616-783):
// _shared_tape_forward 666-686 (v = scale * bu, x = scan(abar, v)),
// _mimo_head_pullback 691-699, _mimo_input_pullback 701-704,
// S5._backward 836-895, LRU._backward 945-980, and the scan pullback
// autograd._scan_pullback 113-140 with constant coefficients.
//
// Lanes are the flattened (b, p) pairs of the [B, L, P] complex state, so any
// P packs densely into 128-lane CTAs; every step of a warp is one contiguous
// run of interleaved complex values.  The forward fuses the input scaling
// v = scale * bu into the load; the backward fuses gbu = conj(scale) g and the
// two per-coefficient reductions sum_k g conj(x_{k-1}) (-> d abar) and
// sum_k conj(bu_k) g_k (-> d scale) into the reverse pass, written as
// per-chunk partials that lrx_reduce_rows folds in a fixed order.
#include "lrx_common.cuh"
#include "lrx_host.h"

namespace lrx {
namespace mimo {

constexpr int kThreads = 128;
template <typename T> struct Tile { static constexpr int K = 16; };
template <> struct Tile<double> { static constexpr int K = 8; };

template <typename T> __device__ __forceinline__ cplx<T> ldc(const cplx<T>* p);
template <> __device__ __forceinline__ cplx<float> ldc(const cplx<float>* p) {
    float2 v = __ldcs(reinterpret_cast<const float2*>(p));
    return {v.x, v.y};
}
template <> __device__ __forceinline__ cplx<double> ldc(const cplx<double>* p) {
    double2 v = __ldcs(reinterpret_cast<const double2*>(p));
    return {v.x, v.y};
}
template <typename T> __device__ __forceinline__ void stc(cplx<T>* p, cplx<T> v);
template <> __device__ __forceinline__ void stc(cplx<float>* p, cplx<float> v) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v.re, v.im));
}
template <> __device__ __forceinline__ void stc(cplx<double>* p, cplx<double> v) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v.re, v.im));
}

template <typename T>
__global__ void __launch_bounds__(kThreads) fwd_kernel(const cplx<T>* __restrict__ abar,
                                                       const cplx<T>* __restrict__ scale,
                                                       const cplx<T>* __restrict__ bu, cplx<T>* __restrict__ x,
                                                       int64_t B, int64_t L, int64_t P, int n_blk, LookbackWS ws) {
    using V = cplx<T>;
    using Tr = Traits<V>;
    constexpr int K = Tile<T>::K;
    const int tile = next_tile(ws.ticket);
    const int c = tile / n_blk, blk = tile % n_blk;
    const int64_t n_lanes = B * P;
    const int64_t lane = (int64_t)blk * kThreads + threadIdx.x;
    const bool valid = lane < n_lanes;
    const int64_t b = valid ? lane / P : 0, p = valid ? lane % P : 0;
    const int64_t t0 = (int64_t)c * K;
    const int nt = (int)min((int64_t)K, L - t0);
    const V ab = valid ? abar[p] : Tr::one();
    const V sc = valid ? scale[p] : Tr::zero();
    V v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const bool ok = valid && k < nt;
        v[k] = ok ? sc * ldc(bu + (b * L + t0 + k) * P + p) : Tr::zero();
    }
    V A = Tr::one(), X = Tr::zero();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (k < nt) {
            X = ab * X + v[k];
            A = ab * A;
        }
    }
    V* agg_a = static_cast<V*>(ws.agg_a);
    V* agg_x = static_cast<V*>(ws.agg_x);
    V* inc_x = static_cast<V*>(ws.inc_x);
    const int64_t woff = (int64_t)c * n_lanes + lane;
    int* sw = ws.status + (int64_t)c * n_blk + blk;
    V xin = Tr::zero();
    if (c > 0) {
        lb_publish<V>(sw, LB_AGG, agg_a + woff, A, agg_x + woff, X, valid);
        xin = lb_lookback<V>(ws, c, blk, n_blk, lane, n_lanes, valid);
    }
    if ((c % kAnchor) == 0)
        lb_publish<V>(sw, LB_INC, (V*)nullptr, A, inc_x + woff, A * xin + X, valid);
    V xs = xin;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (valid && k < nt) {
            xs = ab * xs + v[k];
            stc(x + (b * L + t0 + k) * P + p, xs);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) bwd_kernel(const cplx<T>* __restrict__ abar,
                                                       const cplx<T>* __restrict__ scale,
                                                       const cplx<T>* __restrict__ bu,
                                                       const cplx<T>* __restrict__ x, const cplx<T>* __restrict__ gx,
                                                       cplx<T>* __restrict__ gbu, cplx<T>* __restrict__ gabar_part,
                                                       cplx<T>* __restrict__ gscale_part, int64_t B, int64_t L,
                                                       int64_t P, int n_blk, int n_chunks, LookbackWS ws) {
    using V = cplx<T>;
    using Tr = Traits<V>;
    constexpr int K = Tile<T>::K;
    const int tile = next_tile(ws.ticket);
    const int s = tile / n_blk, blk = tile % n_blk;
    const int c = n_chunks - 1 - s;
    const int64_t n_lanes = B * P;
    const int64_t lane = (int64_t)blk * kThreads + threadIdx.x;
    const bool valid = lane < n_lanes;
    const int64_t b = valid ? lane / P : 0, p = valid ? lane % P : 0;
    const int64_t t0 = (int64_t)c * K;
    const int nt = (int)min((int64_t)K, L - t0);
    const V abc = valid ? conj(abar[p]) : Tr::one();
    const V scc = valid ? conj(scale[p]) : Tr::zero();
    V gxv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const bool ok = valid && k < nt;
        gxv[k] = ok ? ldc(gx + (b * L + t0 + k) * P + p) : Tr::zero();
    }
    V A = Tr::one(), H = Tr::zero();
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
        if (k < nt) {
            const V g = gxv[k] + H;
            H = abc * g;
            A = abc * A;
        }
    }
    V* agg_a = static_cast<V*>(ws.agg_a);
    V* agg_x = static_cast<V*>(ws.agg_x);
    V* inc_x = static_cast<V*>(ws.inc_x);
    const int64_t woff = (int64_t)s * n_lanes + lane;
    int* sw = ws.status + (int64_t)s * n_blk + blk;
    V hin = Tr::zero();
    if (s > 0) {
        lb_publish<V>(sw, LB_AGG, agg_a + woff, A, agg_x + woff, H, valid);
        hin = lb_lookback<V>(ws, s, blk, n_blk, lane, n_lanes, valid);
    }
    if ((s % kAnchor) == 0)
        lb_publish<V>(sw, LB_INC, (V*)nullptr, A, inc_x + woff, A * hin + H, valid);
    V h = hin, sa = Tr::zero(), ss = Tr::zero();
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
        if (valid && k < nt) {
            const int64_t off = (b * L + t0 + k) * P + p;
            const V g = gxv[k] + h;
            h = abc * g;
            stc(gbu + off, scc * g);
            const V xp = (t0 + k == 0) ? Tr::zero() : ldc(x + off - P);
            sa = sa + g * conj(xp);
            ss = ss + conj(ldc(bu + off)) * g;
        }
    }
    if (valid) {
        gabar_part[(int64_t)c * n_lanes + lane] = sa;
        gscale_part[(int64_t)c * n_lanes + lane] = ss;
    }
}

template <typename T>
static size_t ws_bytes(int64_t B, int64_t L, int64_t P) {
    const int64_t nc = cdiv(L, Tile<T>::K), nb = cdiv(B * P, kThreads);
    Carver cv(nullptr);
    cv.take<int>(1);
    cv.take<int>((size_t)(nc * nb));
    for (int i = 0; i < 3; ++i) cv.take<cplx<T>>((size_t)(nc * B * P));
    return cv.off;
}

template <typename T>
static int carve(void* w, size_t wb, int64_t B, int64_t L, int64_t P, LookbackWS* ws, cudaStream_t st) {
    const int64_t nc = cdiv(L, Tile<T>::K), nb = cdiv(B * P, kThreads);
    const size_t need = ws_bytes<T>(B, L, P);
    LRX_REQUIRE(w && wb >= need, LRX_ERR_VALUE, "mimo workspace too small: %zu < %zu", wb, need);
    Carver cv(w);
    ws->ticket = cv.take<int>(1);
    ws->status = cv.take<int>((size_t)(nc * nb));
    const size_t head = cv.off;
    ws->agg_a = cv.take<cplx<T>>((size_t)(nc * B * P));
    ws->agg_x = cv.take<cplx<T>>((size_t)(nc * B * P));
    ws->inc_x = cv.take<cplx<T>>((size_t)(nc * B * P));
    LRX_REQUIRE(cudaMemsetAsync(w, 0, head, st) == cudaSuccess, LRX_ERR_CUDA, "workspace memset failed");
    return LRX_OK;
}

template <typename T>
static int fwd_t(const void* abar, const void* scale, const void* bu, void* x, int64_t B, int64_t L, int64_t P,
                 void* w, size_t wb, cudaStream_t st) {
    LookbackWS ws;
    if (int rc = carve<T>(w, wb, B, L, P, &ws, st)) return rc;
    const int64_t nc = cdiv(L, Tile<T>::K), nb = cdiv(B * P, kThreads);
    fwd_kernel<T><<<(unsigned)(nc * nb), kThreads, 0, st>>>((const cplx<T>*)abar, (const cplx<T>*)scale,
                                                            (const cplx<T>*)bu, (cplx<T>*)x, B, L, P, (int)nb, ws);
    return launched("lrx_mimo_fwd");
}

template <typename T>
static int bwd_t(const void* abar, const void* scale, const void* bu, const void* x, const void* gx, void* gbu,
                 void* gap, void* gsp, int64_t B, int64_t L, int64_t P, void* w, size_t wb, cudaStream_t st) {
    LookbackWS ws;
    if (int rc = carve<T>(w, wb, B, L, P, &ws, st)) return rc;
    const int64_t nc = cdiv(L, Tile<T>::K), nb = cdiv(B * P, kThreads);
    bwd_kernel<T><<<(unsigned)(nc * nb), kThreads, 0, st>>>(
        (const cplx<T>*)abar, (const cplx<T>*)scale, (const cplx<T>*)bu, (const cplx<T>*)x, (const cplx<T>*)gx,
        (cplx<T>*)gbu, (cplx<T>*)gap, (cplx<T>*)gsp, B, L, P, (int)nb, (int)nc, ws);
    return launched("lrx_mimo_bwd");
}

}  // namespace mimo
}  // namespace lrx

using namespace lrx;

extern "C" {

int lrx_mimo_chunking(int dtype, int64_t L, int64_t* chunk_len, int64_t* n_chunks) {
    LRX_REQUIRE(L >= 1, LRX_ERR_SHAPE, "length must be >= 1");
    const int K = dtype == LRX_C128 ? mimo::Tile<double>::K : mimo::Tile<float>::K;
    *chunk_len = K;
    *n_chunks = cdiv(L, K);
    return LRX_OK;
}

size_t lrx_mimo_workspace_bytes(int dtype, int64_t B, int64_t L, int64_t P) {
    if (B < 1 || L < 1 || P < 1) return 256;
    return dtype == LRX_C128 ? mimo::ws_bytes<double>(B, L, P) : mimo::ws_bytes<float>(B, L, P);
}

size_t lrx_mimo_bwd_workspace_bytes(int dtype, int64_t B, int64_t L, int64_t P) {
    return lrx_mimo_workspace_bytes(dtype, B, L, P);
}

int lrx_mimo_fwd(int dtype, const void* abar, const void* scale, const void* bu, void* x, int64_t B, int64_t L,
                 int64_t P, void* workspace, size_t workspace_bytes, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && P >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == LRX_C64) return mimo::fwd_t<float>(abar, scale, bu, x, B, L, P, workspace, workspace_bytes, st);
    if (dtype == LRX_C128) return mimo::fwd_t<double>(abar, scale, bu, x, B, L, P, workspace, workspace_bytes, st);
    set_error("mimo: dtype must be C64 or C128, got %d", dtype);
    return LRX_ERR_VALUE;
}

int lrx_mimo_bwd(int dtype, const void* abar, const void* scale, const void* bu, const void* x, const void* gx,
                 void* gbu, void* gabar_part, void* gscale_part, int64_t B, int64_t L, int64_t P, void* workspace,
                 size_t workspace_bytes, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && P >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == LRX_C64)
        return mimo::bwd_t<float>(abar, scale, bu, x, gx, gbu, gabar_part, gscale_part, B, L, P, workspace,
                                  workspace_bytes, st);
    if (dtype == LRX_C128)
        return mimo::bwd_t<double>(abar, scale, bu, x, gx, gbu, gabar_part, gscale_part, B, L, P, workspace,
                                   workspace_bytes, st);
    set_error("mimo: dtype must be C64 or C128, got %d", dtype);
    return LRX_ERR_VALUE;
}

}  // extern "C"
