// Single-step (decode) kernels: one recurrence update per call on a
// device-resident state, for the step-mode API (Layer.step, layers.py:251-269
// with the per-kind _step: S4D 578-613, _MIMOBase 748-783, S6 1145-1168,
// RG-LRU 1310-1336).  One token per sequence: the work is a handful of small
// GEMVs and an elementwise update, so each kernel fuses its GEMV with the
// state update (warp per output row, lanes over the contraction, shuffle
// reduction) and no kernel allocates.
#include "lrx_common.cuh"
#include "lrx_host.h"

namespace lrx {
namespace step {

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

// S4D: x[b,h,n] = abar[h,n] x + w[h,n] u[b,h];  y[b,h] = Re(sum_n c x) + d u
template <typename T>
__global__ void s4d_step_kernel(cplx<T>* __restrict__ x, const cplx<T>* __restrict__ abar,
                                const cplx<T>* __restrict__ w, const cplx<T>* __restrict__ c,
                                const T* __restrict__ d, const T* __restrict__ u, T* __restrict__ y, int64_t Bn,
                                int64_t H, int64_t N) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // (b, h)
    const int lane = threadIdx.x & 31;
    if (row >= Bn * H) return;
    const int64_t h = row % H;
    const T uk = u[row];
    T acc = 0;
    for (int64_t n = lane; n < N; n += 32) {
        const int64_t p = h * N + n;
        cplx<T> xv = x[row * N + n];
        xv = abar[p] * xv + uk * w[p];
        x[row * N + n] = xv;
        acc += c[p].re * xv.re - c[p].im * xv.im;
    }
    acc = warp_sum(acc);
    if (lane == 0) y[row] = acc + d[h] * uk;
}

// MIMO input: x[b,p] = abar[p] x + scale[p] (sum_h B[p,h] u[b,h])
template <typename T>
__global__ void mimo_step_in_kernel(cplx<T>* __restrict__ x, const cplx<T>* __restrict__ abar,
                                    const cplx<T>* __restrict__ scale, const T* __restrict__ Bre,
                                    const T* __restrict__ Bim, const T* __restrict__ u, int64_t Bn, int64_t P,
                                    int64_t H) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // (b, p)
    const int lane = threadIdx.x & 31;
    if (row >= Bn * P) return;
    const int64_t b = row / P, p = row % P;
    T sr = 0, si = 0;
    for (int64_t h = lane; h < H; h += 32) {
        const T uu = u[b * H + h];
        sr += Bre[p * H + h] * uu;
        si += Bim[p * H + h] * uu;
    }
    sr = warp_sum(sr);
    si = warp_sum(si);
    if (lane == 0) x[row] = abar[p] * x[row] + scale[p] * mk(sr, si);
}

// MIMO output: y[b,h] = osc * Re(sum_p C[h,p] x[b,p]) + D[h] u[b,h]
template <typename T>
__global__ void mimo_step_out_kernel(const cplx<T>* __restrict__ x, const T* __restrict__ Cre,
                                     const T* __restrict__ Cim, const T* __restrict__ D, const T* __restrict__ u,
                                     T* __restrict__ y, T osc, int64_t Bn, int64_t P, int64_t H) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // (b, h)
    const int lane = threadIdx.x & 31;
    if (row >= Bn * H) return;
    const int64_t b = row / H, h = row % H;
    T acc = 0;
    for (int64_t p = lane; p < P; p += 32) {
        const cplx<T> xv = x[b * P + p];
        acc += Cre[h * P + p] * xv.re - Cim[h * P + p] * xv.im;
    }
    acc = warp_sum(acc);
    if (lane == 0) y[row] = osc * acc + D[h] * u[row];
}

// S6: delta = softplus(pre + b), x[b,d,n] = exp(delta a) x + delta u B_k[n],
// y = sum_n C_k[n] x + D u   (thread per (b, d); exact exp / log1p)
template <typename IO, typename C>
__global__ void s6_step_kernel(C* __restrict__ x, const IO* __restrict__ u, const C* __restrict__ pre,
                               const C* __restrict__ Bk, const C* __restrict__ Ck, const C* __restrict__ bdelta,
                               const C* __restrict__ a_log, const C* __restrict__ Dskip, IO* __restrict__ y,
                               int64_t Bn, int64_t D, int64_t N) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (b, d)
    if (i >= Bn * D) return;
    const int64_t b = i / D, d = i % D;
    const C uk = cvt(u[i]);
    const C delta = Math<C>::softplus(pre[i] + bdelta[d]);
    const C du = delta * uk;
    C acc = 0;
    for (int64_t n = 0; n < N; ++n) {
        const C a = -Math<C>::exp(a_log[d * N + n]);
        C xv = x[i * N + n];
        xv = Math<C>::exp(delta * a) * xv + du * Bk[b * N + n];
        x[i * N + n] = xv;
        acc += Ck[b * N + n] * xv;
    }
    st_io(y + i, acc + Dskip[d] * uk);
}

// RG-LRU: gates, x = a x + sqrt(1 - a^2) i u, y = x   (thread per (b, w))
template <typename IO, typename C>
__global__ void rglru_step_kernel(C* __restrict__ x, const IO* __restrict__ u, const IO* __restrict__ qr,
                                  const IO* __restrict__ qi, const C* __restrict__ lam, const C* __restrict__ b_r,
                                  const C* __restrict__ b_i, IO* __restrict__ y, int64_t Bn, int64_t W) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Bn * W) return;
    const int64_t w = i % W;
    const C uk = cvt(u[i]);
    const C r = Math<C>::sigmoid(C(cvt(qr[i])) + b_r[w]);
    const C ig = Math<C>::sigmoid(C(cvt(qi[i])) + b_i[w]);
    const C loga = (C(8) * r) * (-Math<C>::softplus(-lam[w]));  // GATE_POWER 8, layers.py:1208-1210
    const C a = Math<C>::exp(loga);
    const C s = Math<C>::sqrt(-Math<C>::expm1(C(2) * loga));
    const C xv = a * x[i] + (s * ig) * uk;
    x[i] = xv;
    st_io(y + i, xv);
}

static unsigned warps_grid(int64_t rows, int wpb) { return (unsigned)cdiv(rows, wpb); }

// operator-level step (scan.py:232-250): x <- a x + b, a and b each either
// full (period n), lane-periodic (period p: index i % p) or scalar (period 1)
template <typename V>
__global__ void scan_step_kernel(V* __restrict__ x, const V* __restrict__ a, const V* __restrict__ b, int64_t n,
                                 int64_t pa, int64_t pb) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = a[i % pa] * x[i] + b[i % pb];
}

}  // namespace step
}  // namespace lrx

using namespace lrx;

extern "C" {

int lrx_scan_step(int dtype, void* x, const void* a, const void* b, int64_t n, int64_t a_period, int64_t b_period,
                  void* stream) {
    LRX_REQUIRE(n >= 1 && a_period >= 1 && b_period >= 1 && n % a_period == 0 && n % b_period == 0, LRX_ERR_SHAPE,
                "scan step: operand periods %lld / %lld do not tile the state (%lld)", (long long)a_period,
                (long long)b_period, (long long)n);
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (unsigned)cdiv(n, 256);
    switch (dtype) {
        case LRX_F32: step::scan_step_kernel<float><<<g, 256, 0, st>>>((float*)x, (const float*)a, (const float*)b, n,
                                                                      a_period, b_period); break;
        case LRX_F64: step::scan_step_kernel<double><<<g, 256, 0, st>>>((double*)x, (const double*)a,
                                                                       (const double*)b, n, a_period, b_period); break;
        case LRX_C64:
            step::scan_step_kernel<cplx<float>><<<g, 256, 0, st>>>((cplx<float>*)x, (const cplx<float>*)a,
                                                                   (const cplx<float>*)b, n, a_period, b_period);
            break;
        case LRX_C128:
            step::scan_step_kernel<cplx<double>><<<g, 256, 0, st>>>((cplx<double>*)x, (const cplx<double>*)a,
                                                                    (const cplx<double>*)b, n, a_period, b_period);
            break;
        default: set_error("scan step: unsupported dtype %d", dtype); return LRX_ERR_VALUE;
    }
    return launched("lrx_scan_step");
}

int lrx_s4d_step(int dtype, void* x, const void* abar, const void* w, const void* c, const void* d, const void* u,
                 void* y, int64_t B, int64_t H, int64_t N, void* stream) {
    LRX_REQUIRE(B >= 1 && H >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = step::warps_grid(B * H, 8);
    if (dtype == LRX_C64)
        step::s4d_step_kernel<float><<<g, 256, 0, st>>>((cplx<float>*)x, (const cplx<float>*)abar,
                                                        (const cplx<float>*)w, (const cplx<float>*)c,
                                                        (const float*)d, (const float*)u, (float*)y, B, H, N);
    else if (dtype == LRX_C128)
        step::s4d_step_kernel<double><<<g, 256, 0, st>>>((cplx<double>*)x, (const cplx<double>*)abar,
                                                         (const cplx<double>*)w, (const cplx<double>*)c,
                                                         (const double*)d, (const double*)u, (double*)y, B, H, N);
    else {
        set_error("s4d step: state dtype must be c64 or c128, got %d", dtype);
        return LRX_ERR_VALUE;
    }
    return launched("lrx_s4d_step");
}

int lrx_mimo_step(int dtype, void* x, const void* abar, const void* scale, const void* Bre, const void* Bim,
                  const void* Cre, const void* Cim, const void* D, const void* u, void* y, double out_scale,
                  int64_t B, int64_t P, int64_t H, void* stream) {
    LRX_REQUIRE(B >= 1 && P >= 1 && H >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == LRX_C64) {
        step::mimo_step_in_kernel<float><<<step::warps_grid(B * P, 8), 256, 0, st>>>(
            (cplx<float>*)x, (const cplx<float>*)abar, (const cplx<float>*)scale, (const float*)Bre,
            (const float*)Bim, (const float*)u, B, P, H);
        step::mimo_step_out_kernel<float><<<step::warps_grid(B * H, 8), 256, 0, st>>>(
            (const cplx<float>*)x, (const float*)Cre, (const float*)Cim, (const float*)D, (const float*)u,
            (float*)y, (float)out_scale, B, P, H);
    } else if (dtype == LRX_C128) {
        step::mimo_step_in_kernel<double><<<step::warps_grid(B * P, 8), 256, 0, st>>>(
            (cplx<double>*)x, (const cplx<double>*)abar, (const cplx<double>*)scale, (const double*)Bre,
            (const double*)Bim, (const double*)u, B, P, H);
        step::mimo_step_out_kernel<double><<<step::warps_grid(B * H, 8), 256, 0, st>>>(
            (const cplx<double>*)x, (const double*)Cre, (const double*)Cim, (const double*)D, (const double*)u,
            (double*)y, out_scale, B, P, H);
    } else {
        set_error("mimo step: state dtype must be c64 or c128, got %d", dtype);
        return LRX_ERR_VALUE;
    }
    return launched("lrx_mimo_step", 2);
}

int lrx_s6_step(int io_dtype, void* x, const void* u, const void* pre, const void* Bk, const void* Ck,
                const void* b_delta, const void* a_log, const void* Dskip, void* y, int64_t B, int64_t D, int64_t N,
                void* stream) {
    LRX_REQUIRE(B >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (unsigned)cdiv(B * D, 128);
    switch (io_dtype) {
        case LRX_F32:
            step::s6_step_kernel<float, float><<<g, 128, 0, st>>>(
                (float*)x, (const float*)u, (const float*)pre, (const float*)Bk, (const float*)Ck,
                (const float*)b_delta, (const float*)a_log, (const float*)Dskip, (float*)y, B, D, N);
            break;
        case LRX_BF16:
            step::s6_step_kernel<__nv_bfloat16, float><<<g, 128, 0, st>>>(
                (float*)x, (const __nv_bfloat16*)u, (const float*)pre, (const float*)Bk, (const float*)Ck,
                (const float*)b_delta, (const float*)a_log, (const float*)Dskip, (__nv_bfloat16*)y, B, D, N);
            break;
        case LRX_F64:
            step::s6_step_kernel<double, double><<<g, 128, 0, st>>>(
                (double*)x, (const double*)u, (const double*)pre, (const double*)Bk, (const double*)Ck,
                (const double*)b_delta, (const double*)a_log, (const double*)Dskip, (double*)y, B, D, N);
            break;
        default: set_error("s6 step: unsupported io dtype %d", io_dtype); return LRX_ERR_VALUE;
    }
    return launched("lrx_s6_step");
}

int lrx_rglru_step(int io_dtype, void* x, const void* u, const void* qr, const void* qi, const void* lambda_param,
                   const void* b_r, const void* b_i, void* y, int64_t B, int64_t W, void* stream) {
    LRX_REQUIRE(B >= 1 && W >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (unsigned)cdiv(B * W, 128);
    switch (io_dtype) {
        case LRX_F32:
            step::rglru_step_kernel<float, float><<<g, 128, 0, st>>>(
                (float*)x, (const float*)u, (const float*)qr, (const float*)qi, (const float*)lambda_param,
                (const float*)b_r, (const float*)b_i, (float*)y, B, W);
            break;
        case LRX_BF16:
            step::rglru_step_kernel<__nv_bfloat16, float><<<g, 128, 0, st>>>(
                (float*)x, (const __nv_bfloat16*)u, (const __nv_bfloat16*)qr, (const __nv_bfloat16*)qi,
                (const float*)lambda_param, (const float*)b_r, (const float*)b_i, (__nv_bfloat16*)y, B, W);
            break;
        case LRX_F64:
            step::rglru_step_kernel<double, double><<<g, 128, 0, st>>>(
                (double*)x, (const double*)u, (const double*)qr, (const double*)qi, (const double*)lambda_param,
                (const double*)b_r, (const double*)b_i, (double*)y, B, W);
            break;
        default: set_error("rglru step: unsupported io dtype %d", io_dtype); return LRX_ERR_VALUE;
    }
    return launched("lrx_rglru_step");
}

}  // extern "C"
