// Shared device-side building blocks for the lrx sm_100a kernels.
//
//  * value types: real float/double, complex cplx<float>/cplx<double> with the
//    plain (non-Annex-G) product the reference's numba kernels use;
//  * I/O element conversion (bf16 / f32 / f64 storage -> compute precision);
//  * the overflow-safe softplus / sigmoid of the reference
//    (pkg/src/linrec/numerics.py:36-39, 86-105);
//  * the decoupled look-back that chains time chunks of a first-order
//    recurrence across CTAs: each (lane block, chunk) tile publishes its
//    aggregate (A = prod a, X = local state from zero) and, once its carry is
//    known, the inclusive state; successors fold a FIXED set of predecessor
//    aggregates and one anchor's inclusive value (bitwise deterministic).
//    Tiles are handed out in launch order by an atomic ticket, so every awaited
//    predecessor is already resident or done (forward progress without
//    cooperative launch).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace lrx {

// ---------------------------------------------------------------- complex
template <typename T>
struct cplx {
    T re, im;
};

template <typename T> __host__ __device__ __forceinline__ cplx<T> mk(T r, T i) { return cplx<T>{r, i}; }
template <typename T> __device__ __forceinline__ cplx<T> operator+(cplx<T> a, cplx<T> b) { return {a.re + b.re, a.im + b.im}; }
template <typename T> __device__ __forceinline__ cplx<T> operator-(cplx<T> a, cplx<T> b) { return {a.re - b.re, a.im - b.im}; }
template <typename T> __device__ __forceinline__ cplx<T> operator*(cplx<T> a, cplx<T> b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
template <typename T> __device__ __forceinline__ cplx<T> operator*(T s, cplx<T> b) { return {s * b.re, s * b.im}; }
template <typename T> __device__ __forceinline__ cplx<T> conj(cplx<T> a) { return {a.re, -a.im}; }

template <typename V> struct Traits;
template <> struct Traits<float> {
    using R = float;
    static constexpr bool complex = false;
    __device__ static float one() { return 1.f; }
    __device__ static float zero() { return 0.f; }
    __device__ static float cj(float a) { return a; }
};
template <> struct Traits<double> {
    using R = double;
    static constexpr bool complex = false;
    __device__ static double one() { return 1.0; }
    __device__ static double zero() { return 0.0; }
    __device__ static double cj(double a) { return a; }
};
template <typename T> struct Traits<cplx<T>> {
    using R = T;
    static constexpr bool complex = true;
    __device__ static cplx<T> one() { return {T(1), T(0)}; }
    __device__ static cplx<T> zero() { return {T(0), T(0)}; }
    __device__ static cplx<T> cj(cplx<T> a) { return conj(a); }
};

// ---------------------------------------------------------------- I/O
__device__ __forceinline__ float ld_io(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float ld_io(const float* p) { return *p; }
__device__ __forceinline__ double ld_io(const double* p) { return *p; }
template <typename C> __device__ __forceinline__ void st_io(__nv_bfloat16* p, C v) { *p = __float2bfloat16_rn(float(v)); }
template <typename C> __device__ __forceinline__ void st_io(float* p, C v) { *p = float(v); }
template <typename C> __device__ __forceinline__ void st_io(double* p, C v) { *p = double(v); }

// register value -> compute precision
__device__ __forceinline__ float cvt(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float cvt(float v) { return v; }
__device__ __forceinline__ double cvt(double v) { return v; }

// streaming (read-once) loads: keep them out of L1
template <typename X> __device__ __forceinline__ X ld_stream(const X* p) { return __ldcs(p); }
__device__ __forceinline__ __nv_bfloat16 ld_stream(const __nv_bfloat16* p) {
    unsigned short r = __ldcs(reinterpret_cast<const unsigned short*>(p));
    return *reinterpret_cast<__nv_bfloat16*>(&r);
}

// ---------------------------------------------------------------- math
template <typename C> struct Math;
template <> struct Math<float> {
    static constexpr float SOFTPLUS_T = 30.f;  // numerics.py:36-39 (float32)
    __device__ static float exp(float x) { return expf(x); }
    __device__ static float log1p(float x) { return log1pf(x); }
    __device__ static float expm1(float x) { return expm1f(x); }
    __device__ static float sqrt(float x) { return sqrtf(x); }
    __device__ static float softplus(float x) { return x > SOFTPLUS_T ? x : log1pf(expf(fminf(x, SOFTPLUS_T))); }
    __device__ static float sigmoid(float x) {  // numerics.py:97-105
        float e = expf(x >= 0.f ? -x : x);
        return x >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
    }
};
template <> struct Math<double> {
    static constexpr double SOFTPLUS_T = 50.0;  // numerics.py:36-39 (float64)
    __device__ static double exp(double x) { return ::exp(x); }
    __device__ static double log1p(double x) { return ::log1p(x); }
    __device__ static double expm1(double x) { return ::expm1(x); }
    __device__ static double sqrt(double x) { return ::sqrt(x); }
    __device__ static double softplus(double x) { return x > SOFTPLUS_T ? x : ::log1p(::exp(fmin(x, SOFTPLUS_T))); }
    __device__ static double sigmoid(double x) {
        double e = ::exp(x >= 0.0 ? -x : x);
        return x >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
    }
};

// Fast fp32 math for the hot loops (MUFU ex2 / rcp based).  Accuracy is
// ~2 ulp, well inside the 1e-4 fp32 parity bar; expm1 keeps full relative
// accuracy near 0 with a short Taylor polynomial (sqrt(1 - a^2) for a -> 1 is
// exactly where a naive exp(x) - 1 cancels, layers.py:1217).
template <typename C> struct Fast;
template <> struct Fast<float> {
    __device__ static float ex2(float x) {
        float y;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    __device__ static float exp(float x) { return ex2(x * 1.4426950408889634f); }
    __device__ static float rcp(float x) {
        float y;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    __device__ static float div(float a, float b) { return a * rcp(b); }
    __device__ static float sqrt(float x) {
        float y;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    // 1/(1+e^-x): saturates cleanly (e^-x -> inf gives rcp -> 0)
    __device__ static float sigmoid(float x) { return rcp(1.f + exp(-x)); }
    // Relative-accurate e^x - 1 without branches: for |x| < 0.7 a degree-6
    // Taylor polynomial at h = x/2 and the doubling expm1(x) = p (p + 2);
    // otherwise e^x - 1 carries no cancellation.
    __device__ static float expm1(float x) {
        const float h = 0.5f * x;
        float p = 1.f / 720.f;
        p = fmaf(p, h, 1.f / 120.f);
        p = fmaf(p, h, 1.f / 24.f);
        p = fmaf(p, h, 1.f / 6.f);
        p = fmaf(p, h, 0.5f);
        p = fmaf(p, h, 1.f);
        p *= h;
        const float small = p * (p + 2.f);
        const float big = exp(x) - 1.f;
        return fabsf(x) < 0.7f ? small : big;
    }
    // expm1(x) when e^x is already known (ex): no extra MUFU op
    __device__ static float expm1_known(float x, float ex) {
        const float h = 0.5f * x;
        float p = 1.f / 720.f;
        p = fmaf(p, h, 1.f / 120.f);
        p = fmaf(p, h, 1.f / 24.f);
        p = fmaf(p, h, 1.f / 6.f);
        p = fmaf(p, h, 0.5f);
        p = fmaf(p, h, 1.f);
        p *= h;
        return fabsf(x) < 0.7f ? p * (p + 2.f) : ex - 1.f;
    }
};
template <> struct Fast<double> {
    __device__ static double exp(double x) { return ::exp(x); }
    __device__ static double rcp(double x) { return 1.0 / x; }
    __device__ static double div(double a, double b) { return a / b; }
    __device__ static double sqrt(double x) { return ::sqrt(x); }
    __device__ static double sigmoid(double x) { return Math<double>::sigmoid(x); }
    __device__ static double expm1(double x) { return ::expm1(x); }
    __device__ static double expm1_known(double x, double) { return ::expm1(x); }
};

// ---------------------------------------------------------------- per-step discretisation
// (asynchronous S4D / S5: lrx_s4d.cu, lrx_mimo.cu)  discretize.py:59-93 and
// autograd.py:186-211 (scheme_partials), evaluated per step in the kernels.
// ZOH: scale = (abar - 1) / lam and d scale / d lam = (dt abar lam - (abar - 1)) / lam^2
// cancel catastrophically for small |z| = |dt lam| (f32 at z ~ 1e-4 keeps ~3
// digits), so below a threshold they run as the series
//   scale = dt phi1(z),  phi1 = sum z^k / (k+1)!,
//   dsl   = dt^2 phi2(z), phi2 = sum z^k (k+1) / (k+2)!
// (f32: |z| < 0.5, 9 terms; f64: |z| < 0.05, 11 terms -- truncation below the
// unit roundoff); the reference's small-pole branch is the z -> 0 limit.
template <typename T> __device__ __forceinline__ T small_pole_eps();
template <> __device__ __forceinline__ float small_pole_eps<float>() { return 1e-4f; }   // discretize.py:39-42
template <> __device__ __forceinline__ double small_pole_eps<double>() { return 1e-8; }
template <typename T> struct ZohSeries;
template <> struct ZohSeries<float> { static constexpr float R = 0.5f; static constexpr int K = 9; };
template <> struct ZohSeries<double> { static constexpr double R = 0.05; static constexpr int K = 11; };
__device__ __forceinline__ void sc_(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ void sc_(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ float ex_(float x) { return expf(x); }
__device__ __forceinline__ double ex_(double x) { return exp(x); }

template <typename T>
__device__ __forceinline__ cplx<T> cdiv_(cplx<T> a, cplx<T> b) {
    const T den = b.re * b.re + b.im * b.im;
    return {(a.re * b.re + a.im * b.im) / den, (a.im * b.re - a.re * b.im) / den};
}

// phi1(z) = sum_{k<K} z^k / (k+1)!, phi2(z) = sum_{k<K} z^k (k+1) / (k+2)! (Horner)
template <typename T>
__device__ __forceinline__ void zoh_series(cplx<T> z, cplx<T>& p1, cplx<T>& p2) {
    constexpr int K = ZohSeries<T>::K;
    T f1[K], f2[K];
    T fact = T(1);  // (k+1)!
#pragma unroll
    for (int k = 0; k < K; ++k) {
        fact *= T(k + 1);
        f1[k] = T(1) / fact;
        f2[k] = T(k + 1) / (fact * T(k + 2));
    }
    p1 = {f1[K - 1], T(0)};
    p2 = {f2[K - 1], T(0)};
#pragma unroll
    for (int k = K - 2; k >= 0; --k) {
        p1 = p1 * z + cplx<T>{f1[k], T(0)};
        p2 = p2 * z + cplx<T>{f2[k], T(0)};
    }
}

enum { SCHEME_ZOH = 0, SCHEME_BILINEAR = 1, SCHEME_DIRAC = 2 };

template <typename T>
__device__ __forceinline__ bool small_pole(cplx<T> lam) {  // the reference's branch (discretize.py:59-68)
    return sqrt(lam.re * lam.re + lam.im * lam.im) < small_pole_eps<T>();
}
template <typename T>
__device__ __forceinline__ bool zoh_small(cplx<T> z) {
    return z.re * z.re + z.im * z.im < ZohSeries<T>::R * ZohSeries<T>::R;
}

// (abar, scale) of one step dt for pole lam (discretize.py:59-93)
template <typename T>
__device__ __forceinline__ void disc(int scheme, cplx<T> lam, T dt, cplx<T>& ab, cplx<T>& sc) {
    const cplx<T> z = dt * lam;
    if (scheme == SCHEME_BILINEAR) {
        const cplx<T> den = {T(1) - T(0.5) * z.re, -T(0.5) * z.im};
        ab = cdiv_(cplx<T>{T(1) + T(0.5) * z.re, T(0.5) * z.im}, den);
        sc = cdiv_(cplx<T>{dt, T(0)}, den);
        return;
    }
    T sn, cs;
    sc_(z.im, &sn, &cs);
    const T e = ex_(z.re);
    ab = {e * cs, e * sn};
    if (scheme == SCHEME_DIRAC) {
        sc = {T(1), T(0)};
    } else if (small_pole(lam)) {
        sc = {dt, T(0)};
    } else if (zoh_small(z)) {
        cplx<T> p1, p2;
        zoh_series(z, p1, p2);
        sc = dt * p1;
    } else {
        sc = cdiv_(ab - cplx<T>{T(1), T(0)}, lam);
    }
}

// partials d abar / d lam, d abar / d dt, d scale / d lam, d scale / d dt
template <typename T>
__device__ __forceinline__ void disc_partials(int scheme, cplx<T> lam, T dt, cplx<T> ab, cplx<T>& dal, cplx<T>& dad,
                                              cplx<T>& dsl, cplx<T>& dsd) {
    if (scheme == SCHEME_BILINEAR) {
        const cplx<T> den = {T(1) - T(0.5) * dt * lam.re, -T(0.5) * dt * lam.im};
        const cplx<T> inv2 = cdiv_(cplx<T>{T(1), T(0)}, den * den);
        dal = dt * inv2;
        dad = lam * inv2;
        dsl = (T(0.5) * dt * dt) * inv2;
        dsd = inv2;
        return;
    }
    dal = dt * ab;
    dad = lam * ab;
    if (scheme == SCHEME_DIRAC) {
        dsl = dsd = cplx<T>{T(0), T(0)};
        return;
    }
    const cplx<T> z = dt * lam;
    if (small_pole(lam)) {
        dsl = {T(0.5) * dt * dt, T(0)};
        dsd = {T(1), T(0)};
        return;
    }
    dsd = ab;
    if (zoh_small(z)) {
        cplx<T> p1, p2;
        zoh_series(z, p1, p2);
        dsl = (dt * dt) * p2;
    } else {
        dsl = cdiv_(dt * (ab * lam) - (ab - cplx<T>{T(1), T(0)}), lam * lam);
    }
}

// ---------------------------------------------------------------- look-back
// Status words per tile: 0 = nothing yet, 1 = aggregate published,
// 2 = inclusive published.  Tiles are (chunk, lane block); values are per lane.
enum : int { LB_EMPTY = 0, LB_AGG = 1, LB_INC = 2 };

struct LookbackWS {
    int* ticket;   // [1]
    int* status;   // [n_chunks * n_blk]
    void* agg_a;   // [n_chunks * n_lanes] of V
    void* agg_x;   // [n_chunks * n_lanes] of V
    void* inc_x;   // [n_chunks * n_lanes] of V  (state leaving the chunk)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// CTA-wide: obtain this CTA's tile index in launch order.
__device__ __forceinline__ int next_tile(int* ticket) {
    __shared__ int s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    return s_tile;
}

// Publish per-lane values, then the tile status (CTA-wide call).
template <typename V> __device__ __forceinline__ V ldcg(const V* p) { return __ldcg(p); }
template <> __device__ __forceinline__ cplx<float> ldcg(const cplx<float>* p) {
    float2 v = __ldcg(reinterpret_cast<const float2*>(p));
    return {v.x, v.y};
}
template <> __device__ __forceinline__ cplx<double> ldcg(const cplx<double>* p) {
    double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    return {v.x, v.y};
}
__device__ __forceinline__ void stcg_v(cplx<float>* p, cplx<float> v) { __stcg(reinterpret_cast<float2*>(p), make_float2(v.re, v.im)); }
__device__ __forceinline__ void stcg_v(cplx<double>* p, cplx<double> v) { __stcg(reinterpret_cast<double2*>(p), make_double2(v.re, v.im)); }
__device__ __forceinline__ void stcg_v(float* p, float v) { __stcg(p, v); }
__device__ __forceinline__ void stcg_v(double* p, double v) { __stcg(p, v); }

// Publish per-lane values (a may be skipped), then the tile status.  CTA-wide.
template <typename V>
__device__ __forceinline__ void lb_publish(int* status_word, int flag, V* dst_a, V a, V* dst_x, V x,
                                           bool valid) {
    if (valid) {
        if (dst_a) stcg_v(dst_a, a);
        stcg_v(dst_x, x);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(status_word, flag);
}

// Anchored look-back: return the carry entering scan-order chunk c (c >= 1)
// for this thread's lane.  Chunk c folds the aggregates of chunks
// anchor+1 .. c-1 and then the INCLUSIVE value of its anchor, where
// anchor = the nearest multiple of kAnchor below c.  The fold set is a fixed
// function of c, so the result is bitwise reproducible run to run (unlike a
// classic decoupled look-back whose fold depth depends on timing); the
// serial dependency only runs through the anchors (1 in kAnchor chunks).
// CTA-wide call.
constexpr int kAnchor = 8;

__device__ __forceinline__ int lb_wait(const int* w, int want) {
    __shared__ int s_flag;
    if (threadIdx.x == 0) {
        int f;
        while ((f = ld_acquire(w)) < want) __nanosleep(20);
        s_flag = f;
    }
    __syncthreads();
    const int f = s_flag;
    __syncthreads();
    return f;
}

template <typename V>
__device__ V lb_lookback(const LookbackWS& ws, int c, int blk, int n_blk, int64_t lane, int64_t n_lanes,
                         bool valid) {
    using Tr = Traits<V>;
    const V* agg_a = static_cast<const V*>(ws.agg_a);
    const V* agg_x = static_cast<const V*>(ws.agg_x);
    const V* inc_x = static_cast<const V*>(ws.inc_x);
    const int anchor = ((c - 1) / kAnchor) * kAnchor;
    V A = Tr::one(), X = Tr::zero();
    for (int p = c - 1; p > anchor; --p) {
        lb_wait(ws.status + (int64_t)p * n_blk + blk, LB_AGG);
        if (valid) {
            const int64_t off = (int64_t)p * n_lanes + lane;
            const V pa = ldcg(agg_a + off), px = ldcg(agg_x + off);
            X = A * px + X;
            A = A * pa;
        }
    }
    lb_wait(ws.status + (int64_t)anchor * n_blk + blk, LB_INC);
    if (valid) X = A * ldcg(inc_x + (int64_t)anchor * n_lanes + lane) + X;
    return X;
}

template <typename V>
__device__ __forceinline__ void lb_store(V* base, int64_t off, V v, bool valid) {
    if (valid) stcg_v(base + off, v);
}

}  // namespace lrx
