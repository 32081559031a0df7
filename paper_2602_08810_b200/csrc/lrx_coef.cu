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

#include <algorithm>

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
                                void* wgt, void* wbf, void* wgf, int lo) {
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
    //   wbf [256, m]: the fused projection + scan layout (lrx_mimo_fused_fwd):
    //   Re rows p, Im rows 128 + p, zero rows past P (all 256 rows written)
    //   wgf [256, m]: wgt in that layout (the fused backward's gx projection)
    if (wbf || wgf)
        for (int64_t i = tid; i < 128 * m; i += nth) {
            const int64_t p = i / m, h = i % m;
            const bool in = p < P;
            put<T>(wbf, p * m + h, in ? ld<T>(b_re, p * m + h) : 0.0, lo, 256 * m);
            put<T>(wbf, (128 + p) * m + h, in ? ld<T>(b_im, p * m + h) : 0.0, lo, 256 * m);
            put<T>(wgf, p * m + h, in ? ld<T>(c_re, h * P + p) : 0.0, lo, 256 * m);
            put<T>(wgf, (128 + p) * m + h, in ? -ld<T>(c_im, h * P + p) : 0.0, lo, 256 * m);
        }
}

// ga = sum g conj(x_{k-1}) (per state, summed over batch and time), gsc = sum
// conj(bu) g; R [m, 2P] = gy^T x2; R2 [2P, m] = gbu2^T u2.
//
// gsc == NULL (the fused forward stores no bu): gsc = sum_k conj(bu_k) g_k =
// sum_h conj(B[p, h]) (gbu^T u)[p, h] / conj(scale_p) from R2, one warp per
// state (lane-strided over h, fixed xor tree: deterministic).
template <typename T>
__global__ void coef_bwd_kernel(int kind, int scheme, const void* p0, const void* p1, const void* p2,
                                const double* extra, const void* ga, int64_t ga_rows, const void* gsc,
                                int64_t gsc_rows, const void* R, const void* R2, const void* b_re, const void* b_im,
                                double osc, void* g0, void* g1, void* g2, void* gb_re, void* gb_im, void* gc_re,
                                void* gc_im, int64_t P, int64_t m) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (int64_t p = tid >> 5; p < P; p += nth >> 5) {  // warp per state
        const double* e = extra + 8 * p;
        const z64 lam{e[0], e[1]}, ab{e[2], e[3]};
        const double delta = e[6];
        // the scan's per-chunk partial rows [rows, P], summed here in f64 (lane-
        // strided rows, then the fixed xor tree)
        auto rowsum = [&](const void* v, int64_t rows) {
            z64 acc{0.0, 0.0};
            for (int64_t r = lane; r < rows; r += 32) acc = acc + z64{ld<T>(v, 2 * (r * P + p)), ld<T>(v, 2 * (r * P + p) + 1)};
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                acc.re += __shfl_xor_sync(0xffffffffu, acc.re, o);
                acc.im += __shfl_xor_sync(0xffffffffu, acc.im, o);
            }
            return acc;
        };
        const z64 a = rowsum(ga, ga_rows);
        z64 s;
        if (gsc) {
            s = rowsum(gsc, gsc_rows);
        } else {
            z64 acc{0.0, 0.0};
            for (int64_t h = lane; h < m; h += 32) {
                const z64 w{ld<T>(b_re, p * m + h), ld<T>(b_im, p * m + h)};
                const z64 r{ld<T>(R2, (2 * p) * m + h), ld<T>(R2, (2 * p + 1) * m + h)};
                acc = acc + conj(w) * r;
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                acc.re += __shfl_xor_sync(0xffffffffu, acc.re, o);
                acc.im += __shfl_xor_sync(0xffffffffu, acc.im, o);
            }
            s = zdiv(acc, conj(z64{e[4], e[5]}));
        }
        if (lane) continue;
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

namespace lrx {
namespace coef {

// ---- S4D (layers.py:352-546): per (h, n) coefficients and their gradients --
// Forward: lam = -exp(lambda_re_log) + i lambda_im, delta = exp(log_delta[h]),
// (abar, scale) = scheme(lam, delta) in f64 (lrx_common.cuh disc), w = scale b.
template <typename T>
__global__ void s4d_coef_kernel(int scheme, const T* lre, const T* lim, const T* bre, const T* bim, const T* ldl,
                                int64_t H, int64_t N, cplx<T>* abar, cplx<T>* w) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= H * N) return;
    const z64 lam = {-exp((double)lre[i]), (double)lim[i]};
    const double delta = exp((double)ldl[i / N]);
    z64 ab, sc;
    disc<double>(scheme, lam, delta, ab, sc);
    const z64 wv = sc * z64{(double)bre[i], (double)bim[i]};
    abar[i] = {(T)ab.re, (T)ab.im};
    w[i] = {(T)wv.re, (T)wv.im};
}

// Backward, block per channel h (threads over n): from gabar = sum g conj(x_prev)
// and gpsi = sum u g (the fused kernel's partial sums):
//   gscale = conj(b) gpsi, gb = conj(scale) gpsi,
//   glam = conj(dal) gabar + conj(dsl) gscale,
//   glog_delta[h] = delta sum_n Re(conj(dad) gabar) + Re(conj(dsd) gscale)
// (S4D._backward, layers.py:520-546; the n-sum is a fixed-order tree).
template <typename T>
__global__ void s4d_coef_grads_kernel(int scheme, const T* lre, const T* lim, const T* bre, const T* bim,
                                      const T* ldl, const cplx<T>* gabar, const cplx<T>* gpsi, int64_t H, int64_t N,
                                      T* g_lre, T* g_lim, T* g_bre, T* g_bim, T* g_ldl) {
    __shared__ double red[64];
    const int64_t h = blockIdx.x;
    const int n = threadIdx.x;
    double gd = 0.0;
    if (n < N) {
        const int64_t i = h * N + n;
        const z64 lam = {-exp((double)lre[i]), (double)lim[i]};
        const double delta = exp((double)ldl[h]);
        z64 ab, sc, dal, dad, dsl, dsd;
        disc<double>(scheme, lam, delta, ab, sc);
        disc_partials<double>(scheme, lam, delta, ab, dal, dad, dsl, dsd);
        const z64 ga = {(double)gabar[i].re, (double)gabar[i].im}, gp = {(double)gpsi[i].re, (double)gpsi[i].im};
        const z64 b = {(double)bre[i], (double)bim[i]};
        const z64 gsc = conj(b) * gp, gb = conj(sc) * gp;
        const z64 glam = conj(dal) * ga + conj(dsl) * gsc;
        g_lre[i] = (T)(lam.re * glam.re);  // d lam.re / d lambda_re_log = -exp(.) = lam.re
        g_lim[i] = (T)glam.im;
        g_bre[i] = (T)gb.re;
        g_bim[i] = (T)gb.im;
        gd = ((conj(dad) * ga).re + (conj(dsd) * gsc).re) * delta;
    }
    red[n] = gd;
    __syncthreads();
    for (int s2 = 32; s2 >= 1; s2 >>= 1) {
        if (n < s2) red[n] += red[n + s2];
        __syncthreads();
    }
    if (n == 0) g_ldl[h] = (T)red[0];
}

}  // namespace coef
}  // namespace lrx

extern "C" {

int lrx_mimo_coef(int kind, int scheme, int dtype, const void* p0, const void* p1, const void* p2, const void* b_re,
                  const void* b_im, const void* c_re, const void* c_im, int64_t P, int64_t m, void* abar, void* scale,
                  double* extra, void* wbt, void* wb, void* wct, void* wgt, void* wbf, void* wgf, int lo_planes,
                  void* stream) {
    LRX_REQUIRE(P >= 1 && m >= 1, LRX_ERR_SHAPE, "mimo coef: bad extents P=%lld m=%lld", (long long)P, (long long)m);
    LRX_REQUIRE(kind == 0 || kind == 1, LRX_ERR_VALUE, "mimo coef: kind %d (0 = s5, 1 = lru)", kind);
    LRX_REQUIRE(kind == 1 || scheme == LRX_ZOH || scheme == LRX_DIRAC, LRX_ERR_VALUE,
                "mimo coef: scheme %d is not fused (bilinear checks its singular set on the host)", scheme);
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = coef::grid_for(P * m);
    if (dtype == LRX_F32)
        coef::coef_fwd_kernel<float><<<g, 256, 0, st>>>(kind, scheme, p0, p1, p2, b_re, b_im, c_re, c_im, P, m, abar,
                                                        scale, extra, wbt, wb, wct, wgt, wbf, wgf, lo_planes);
    else if (dtype == LRX_F64)
        coef::coef_fwd_kernel<double><<<g, 256, 0, st>>>(kind, scheme, p0, p1, p2, b_re, b_im, c_re, c_im, P, m, abar,
                                                         scale, extra, wbt, wb, wct, wgt, wbf, wgf, lo_planes);
    else {
        set_error("mimo coef: parameter dtype %d (f32 or f64)", dtype);
        return LRX_ERR_VALUE;
    }
    return launched("lrx_mimo_coef");
}

int lrx_mimo_coef_grads(int kind, int scheme, int dtype, const void* p0, const void* p1, const void* p2,
                        const double* extra, const void* ga, int64_t ga_rows, const void* gsc, int64_t gsc_rows,
                        const void* R, const void* R2, const void* b_re, const void* b_im, double out_scale,
                        void* g0, void* g1, void* g2, void* gb_re, void* gb_im, void* gc_re, void* gc_im, int64_t P,
                        int64_t m, void* stream) {
    LRX_REQUIRE(P >= 1 && m >= 1, LRX_ERR_SHAPE, "mimo coef grads: bad extents");
    LRX_REQUIRE(kind == 0 || kind == 1, LRX_ERR_VALUE, "mimo coef grads: kind %d", kind);
    cudaStream_t st = (cudaStream_t)stream;
    LRX_REQUIRE(gsc || (b_re && b_im), LRX_ERR_VALUE, "mimo coef grads: gsc or (b_re, b_im) required");
    LRX_REQUIRE(ga_rows >= 1 && (!gsc || gsc_rows >= 1), LRX_ERR_SHAPE, "mimo coef grads: partial rows");
    const unsigned g = std::max(coef::grid_for(P * m), (unsigned)cdiv(P, 8));  // >= one warp per state
    if (dtype == LRX_F32)
        coef::coef_bwd_kernel<float><<<g, 256, 0, st>>>(kind, scheme, p0, p1, p2, extra, ga, ga_rows, gsc, gsc_rows, R, R2, b_re, b_im,
                                                        out_scale, g0, g1, g2, gb_re, gb_im, gc_re, gc_im, P, m);
    else if (dtype == LRX_F64)
        coef::coef_bwd_kernel<double><<<g, 256, 0, st>>>(kind, scheme, p0, p1, p2, extra, ga, ga_rows, gsc, gsc_rows, R, R2, b_re, b_im,
                                                         out_scale, g0, g1, g2, gb_re, gb_im, gc_re, gc_im, P, m);
    else {
        set_error("mimo coef grads: parameter dtype %d (f32 or f64)", dtype);
        return LRX_ERR_VALUE;
    }
    return launched("lrx_mimo_coef_grads");
}

int lrx_s4d_coef(int dtype, int scheme, const void* lambda_re_log, const void* lambda_im, const void* b_re,
                 const void* b_im, const void* log_delta, int64_t H, int64_t N, void* abar, void* w, void* stream) {
    LRX_REQUIRE(H >= 1 && N >= 1, LRX_ERR_SHAPE, "s4d coef: bad extents");
    LRX_REQUIRE(scheme >= 0 && scheme <= 2, LRX_ERR_VALUE, "s4d coef: scheme %d", scheme);
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = (unsigned)cdiv(H * N, 128);
    if (dtype == LRX_F32)
        coef::s4d_coef_kernel<float><<<grid, 128, 0, st>>>(scheme, (const float*)lambda_re_log, (const float*)lambda_im,
                                                            (const float*)b_re, (const float*)b_im,
                                                            (const float*)log_delta, H, N, (cplx<float>*)abar,
                                                            (cplx<float>*)w);
    else if (dtype == LRX_F64)
        coef::s4d_coef_kernel<double><<<grid, 128, 0, st>>>(scheme, (const double*)lambda_re_log,
                                                             (const double*)lambda_im, (const double*)b_re,
                                                             (const double*)b_im, (const double*)log_delta, H, N,
                                                             (cplx<double>*)abar, (cplx<double>*)w);
    else {
        set_error("s4d coef: dtype %d (f32 / f64)", dtype);
        return LRX_ERR_VALUE;
    }
    return launched("lrx_s4d_coef");
}

int lrx_s4d_coef_grads(int dtype, int scheme, const void* lambda_re_log, const void* lambda_im, const void* b_re,
                       const void* b_im, const void* log_delta, const void* gabar, const void* gpsi, int64_t H,
                       int64_t N, void* g_lambda_re_log, void* g_lambda_im, void* g_b_re, void* g_b_im,
                       void* g_log_delta, void* stream) {
    LRX_REQUIRE(H >= 1 && N >= 1 && N <= 64, LRX_ERR_SHAPE, "s4d coef grads: bad extents (N <= 64)");
    LRX_REQUIRE(scheme >= 0 && scheme <= 2, LRX_ERR_VALUE, "s4d coef: scheme %d", scheme);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == LRX_F32)
        coef::s4d_coef_grads_kernel<float><<<(unsigned)H, 64, 0, st>>>(
            scheme, (const float*)lambda_re_log, (const float*)lambda_im, (const float*)b_re, (const float*)b_im,
            (const float*)log_delta, (const cplx<float>*)gabar, (const cplx<float>*)gpsi, H, N,
            (float*)g_lambda_re_log, (float*)g_lambda_im, (float*)g_b_re, (float*)g_b_im, (float*)g_log_delta);
    else if (dtype == LRX_F64)
        coef::s4d_coef_grads_kernel<double><<<(unsigned)H, 64, 0, st>>>(
            scheme, (const double*)lambda_re_log, (const double*)lambda_im, (const double*)b_re, (const double*)b_im,
            (const double*)log_delta, (const cplx<double>*)gabar, (const cplx<double>*)gpsi, H, N,
            (double*)g_lambda_re_log, (double*)g_lambda_im, (double*)g_b_re, (double*)g_b_im, (double*)g_log_delta);
    else {
        set_error("s4d coef: dtype %d (f32 / f64)", dtype);
        return LRX_ERR_VALUE;
    }
    return launched("lrx_s4d_coef_grads");
}

}  // extern "C"
