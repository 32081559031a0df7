// Parameter-sized coefficient work of the MIMO LTI layers (S5, LRU), fused.
//
// Reference: pkg/src/linrec/layers.py S5._lam/_abar_scale 823-834 and
// S5._backward 836-895 (glam / glog_delta through scheme_partials,
// autograd.py:186-211); LRU._lambda/_abar_scale 936-943 and LRU._backward
// 945-980; discretize.py:59-142 (zoh / dirac factors).
//
// Per step the layer needs, from ~8 parameter tensors of size [P] / [P, m]:
//   abar[P], scale[P] (complex, compute dtype) discretised in f64,
//   the four real layouts of the complex projections the GEMMs consume,
// and after the scan the coefficient gradients from (sum_k g conj x_{k-1},
// sum_k conj(bu) g) plus the B / C gradient planes from the two weight GEMMs.
// Done with torch ops that is ~40 launches of a few microseconds each (a
// third of the C1 step); here it is one launch forward and one backward.
//
// extra[P][8] (f64, kept by the caller between forward and backward):
//   lam.re, lam.im, abar.re, abar.im, scale.re, scale.im, delta, 0
#include "lrx_common.cuh"
#include "lrx_host.h"

namespace lrx {
namespace coef {

using z64 = cplx<double>;

__device__ __forceinline__ z64 zexp(z64 a) {
    const double e = exp(a.re);
    double s, c;
    sincos(a.im, &s, &c);
    return {e * c, e * s};
}
__device__ __forceinline__ z64 zdiv(z64 a, z64 b) {
    const double d = b.re * b.re + b.im * b.im;
    return {(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
}
__device__ __forceinline__ double zabs(z64 a) { return hypot(a.re, a.im); }

template <typename T> __device__ __forceinline__ double ld(const void* p, int64_t i) {
    return (double)static_cast<const T*>(p)[i];
}
template <typename T> __device__ __forceinline__ void st(void* p, int64_t i, double v) {
    static_cast<T*>(p)[i] = (T)v;
}

// layout element (and, for fp32 with lo set, its 3xTF32 low part
// v - tf32(v) one plane of n elements further: ops.tf32_lo)
template <typename T>
__device__ __forceinline__ void put(void* p, int64_t i, double v, int lo, int64_t n) {
    if (!p) return;
    const T t = (T)v;
    static_cast<T*>(p)[i] = t;
    if constexpr (sizeof(T) == 4) {
        if (lo) static_cast<float*>(p)[n + i] = t - __int_as_float(__float_as_int(t) & -8192);
    }
}

constexpr double kZohEps = 1e-8;  // discretize.py:39-44 (f64 poles)

// kind 0 = S5 (p0 lambda_re_log, p1 lambda_im, p2 log_delta),
// kind 1 = LRU (p0 nu_log, p1 theta_log, p2 gamma_log).
template <typename T>
__global__ void coef_fwd_kernel(int kind, int scheme, const void* p0, const void* p1, const void* p2,
                                const void* b_re, const void* b_im, const void* c_re, const void* c_im, int64_t P,
                                int64_t m, void* abar, void* scale, double* extra, void* wbt, void* wb, void* wct,
                                void* wgt, int lo) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = tid; p < P; p += nth) {
        z64 lam, ab, sc;
        double delta = 0;
        if (kind == 0) {
            lam = {-exp(ld<T>(p0, p)), ld<T>(p1, p)};
            delta = exp(ld<T>(p2, p));
            ab = zexp(delta * lam);
            if (scheme == LRX_DIRAC) {
                sc = {1.0, 0.0};
            } else {  // zoh: (abar - 1) / lam, delta for a vanishing pole
                sc = zabs(lam) < kZohEps ? z64{delta, 0.0} : zdiv(ab - z64{1.0, 0.0}, lam);
            }
        } else {
            lam = zexp(z64{-exp(ld<T>(p0, p)), exp(ld<T>(p1, p))});
            ab = lam;
            // gamma = exp(gamma_log) in the layer dtype (layers.py:941)
            sc = {(double)(T)exp((T)ld<T>(p2, p)), 0.0};
        }
        st<T>(abar, 2 * p, ab.re);
        st<T>(abar, 2 * p + 1, ab.im);
        st<T>(scale, 2 * p, sc.re);
        st<T>(scale, 2 * p + 1, sc.im);
        double* e = extra + 8 * p;
        e[0] = lam.re, e[1] = lam.im, e[2] = ab.re, e[3] = ab.im, e[4] = sc.re, e[5] = sc.im, e[6] = delta, e[7] = 0;
    }
    // real layouts of B [P, m] and C [m, P] (interleaved re/im state columns):
    //   wbt [2P, m]: rows (B_re[p], B_im[p])      u @ wbt^T  = interleaved B u
    //   wb  [m, 2P]: wbt^T
    //   wct [m, 2P]: (C_re[h,p], -C_im[h,p])      x2 @ wct^T = Re(C x)
    //   wgt [2P, m]: wct^T
    for (int64_t i = tid; i < P * m; i += nth) {
        const int64_t p = i / m, h = i % m;  // B index [p, h]
        const double br = ld<T>(b_re, i), bi = ld<T>(b_im, i);
        const int64_t hc = i / P, pc = i % P;  // C index [h, p]
        const double cr = ld<T>(c_re, i), ci = ld<T>(c_im, i);
        put<T>(wbt, (2 * p) * m + h, br, lo, 2 * P * m);
        put<T>(wbt, (2 * p + 1) * m + h, bi, lo, 2 * P * m);
        put<T>(wb, h * 2 * P + 2 * p, br, lo, 2 * P * m);
        put<T>(wb, h * 2 * P + 2 * p + 1, bi, lo, 2 * P * m);
        put<T>(wct, hc * 2 * P + 2 * pc, cr, lo, 2 * P * m);
        put<T>(wct, hc * 2 * P + 2 * pc + 1, -ci, lo, 2 * P * m);
        put<T>(wgt, (2 * pc) * m + hc, cr, lo, 2 * P * m);
        put<T>(wgt, (2 * pc + 1) * m + hc, -ci, lo, 2 * P * m);
    }
}

// ga = sum g conj(x_{k-1}) (per state, summed over batch and time), gsc = sum
// conj(bu) g; R [m, 2P] = gy^T x2; R2 [2P, m] = gbu2^T u2.
template <typename T>
__global__ void coef_bwd_kernel(int kind, int scheme, const void* p0, const void* p1, const void* p2,
                                const double* extra, const void* ga, const void* gsc, const void* R, const void* R2,
                                double osc, void* g0, void* g1, void* g2, void* gb_re, void* gb_im, void* gc_re,
                                void* gc_im, int64_t P, int64_t m) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = tid; p < P; p += nth) {
        const double* e = extra + 8 * p;
        const z64 lam{e[0], e[1]}, ab{e[2], e[3]};
        const double delta = e[6];
        const z64 a{ld<T>(ga, 2 * p), ld<T>(ga, 2 * p + 1)};
        const z64 s{ld<T>(gsc, 2 * p), ld<T>(gsc, 2 * p + 1)};
        if (kind == 0) {
            // scheme_partials (autograd.py:186-211): d abar / d lam, d abar / d delta,
            // d scale / d lam, d scale / d delta
            const z64 dal = delta * ab, dad = lam * ab;
            z64 dsl{0, 0}, dsd{0, 0};
            if (scheme != LRX_DIRAC) {
                if (zabs(lam) < kZohEps) {
                    dsl = {delta * delta / 2.0, 0.0};
                    dsd = {1.0, 0.0};
                } else {
                    dsl = zdiv(delta * (ab * lam) - (ab - z64{1.0, 0.0}), lam * lam);
                    dsd = ab;
                }
            }
            const z64 glam = conj(dal) * a + conj(dsl) * s;
            const double gdel = (conj(dad) * a).re + (conj(dsd) * s).re;
            st<T>(g0, p, -exp(ld<T>(p0, p)) * glam.re);
            st<T>(g1, p, glam.im);
            st<T>(g2, p, gdel * delta);
        } else {
            const z64 cl = conj(lam) * a;
            st<T>(g0, p, -exp(ld<T>(p0, p)) * cl.re);
            st<T>(g1, p, exp(ld<T>(p1, p)) * cl.im);
            st<T>(g2, p, exp(ld<T>(p2, p)) * s.re);
        }
    }
    for (int64_t i = tid; i < P * m; i += nth) {
        const int64_t p = i / m, h = i % m;  // gB [p, h] from R2 [2P, m]
        st<T>(gb_re, i, ld<T>(R2, (2 * p) * m + h));
        st<T>(gb_im, i, ld<T>(R2, (2 * p + 1) * m + h));
        const int64_t hc = i / P, pc = i % P;  // gC [h, p] from R [m, 2P]
        st<T>(gc_re, i, osc * ld<T>(R, hc * 2 * P + 2 * pc));
        st<T>(gc_im, i, -osc * ld<T>(R, hc * 2 * P + 2 * pc + 1));
    }
}

static unsigned grid_for(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (unsigned)(b < 1 ? 1 : b > 1184 ? 1184 : b);
}

}  // namespace coef
}  // namespace lrx

using namespace lrx;

extern "C" {

int lrx_mimo_coef(int kind, int scheme, int dtype, const void* p0, const void* p1, const void* p2, const void* b_re,
                  const void* b_im, const void* c_re, const void* c_im, int64_t P, int64_t m, void* abar, void* scale,
                  double* extra, void* wbt, void* wb, void* wct, void* wgt, int lo_planes, void* stream) {
    LRX_REQUIRE(P >= 1 && m >= 1, LRX_ERR_SHAPE, "mimo coef: bad extents P=%lld m=%lld", (long long)P, (long long)m);
    LRX_REQUIRE(kind == 0 || kind == 1, LRX_ERR_VALUE, "mimo coef: kind %d (0 = s5, 1 = lru)", kind);
    LRX_REQUIRE(kind == 1 || scheme == LRX_ZOH || scheme == LRX_DIRAC, LRX_ERR_VALUE,
                "mimo coef: scheme %d is not fused (bilinear checks its singular set on the host)", scheme);
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = coef::grid_for(P * m);
    if (dtype == LRX_F32)
        coef::coef_fwd_kernel<float><<<g, 256, 0, st>>>(kind, scheme, p0, p1, p2, b_re, b_im, c_re, c_im, P, m, abar,
                                                        scale, extra, wbt, wb, wct, wgt, lo_planes);
    else if (dtype == LRX_F64)
        coef::coef_fwd_kernel<double><<<g, 256, 0, st>>>(kind, scheme, p0, p1, p2, b_re, b_im, c_re, c_im, P, m, abar,
                                                         scale, extra, wbt, wb, wct, wgt, lo_planes);
    else {
        set_error("mimo coef: parameter dtype %d (f32 or f64)", dtype);
        return LRX_ERR_VALUE;
    }
    return launched("lrx_mimo_coef");
}

int lrx_mimo_coef_grads(int kind, int scheme, int dtype, const void* p0, const void* p1, const void* p2,
                        const double* extra, const void* ga, const void* gsc, const void* R, const void* R2,
                        double out_scale, void* g0, void* g1, void* g2, void* gb_re, void* gb_im, void* gc_re,
                        void* gc_im, int64_t P, int64_t m, void* stream) {
    LRX_REQUIRE(P >= 1 && m >= 1, LRX_ERR_SHAPE, "mimo coef grads: bad extents");
    LRX_REQUIRE(kind == 0 || kind == 1, LRX_ERR_VALUE, "mimo coef grads: kind %d", kind);
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = coef::grid_for(P * m);
    if (dtype == LRX_F32)
        coef::coef_bwd_kernel<float><<<g, 256, 0, st>>>(kind, scheme, p0, p1, p2, extra, ga, gsc, R, R2, out_scale,
                                                        g0, g1, g2, gb_re, gb_im, gc_re, gc_im, P, m);
    else if (dtype == LRX_F64)
        coef::coef_bwd_kernel<double><<<g, 256, 0, st>>>(kind, scheme, p0, p1, p2, extra, ga, gsc, R, R2, out_scale,
                                                         g0, g1, g2, gb_re, gb_im, gc_re, gc_im, P, m);
    else {
        set_error("mimo coef grads: parameter dtype %d (f32 or f64)", dtype);
        return LRX_ERR_VALUE;
    }
    return launched("lrx_mimo_coef_grads");
}

}  // extern "C"
