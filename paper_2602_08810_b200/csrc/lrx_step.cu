// Single-step (decode) kernels: one recurrence update per call on a
// device-resident state, for the step-mode API (Layer.step, layers.py:251-269
// with the per-kind _step: S4D 578-613, _MIMOBase 748-783, S6 1145-1168,
// RG-LRU 1310-1336).  One token per sequence: the work is a handful of small
// GEMVs and an elementwise update, so each kernel fuses its GEMV with the
// state update (warp per output row, lanes over the contraction, shuffle
// reduction) and no kernel allocates.
#include <algorithm>

#include "lrx_common.cuh"
#include "lrx_host.h"
#include "lrx_tma.cuh"

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

// S6 token in two kernels (fp32 weights, batch <= 16; layers.py:1020-1027 +
// 1145-1168).  (1) the input projections p1 = u W_delta [B, r], B_k = u W_B^T,
// C_k = u W_C^T [B, n]: CTA per output column, its 8 warps split the model
// width, u staged in shared memory; (2) thread per (b, d): pre = p1 . W_dp[:, d]
// then the update of the channel's N states.
template <typename IO>
__global__ void __launch_bounds__(256) s6_step_proj_kernel(const IO* __restrict__ u, const float* __restrict__ Wd,
                                                           const float* __restrict__ WB,
                                                           const float* __restrict__ WC, float* __restrict__ out,
                                                           int Bn, int m, int r, int n) {
    // u [Bn][m] lands by one bulk copy (IO dtype); [8 warps][16] partials after it
    extern __shared__ __align__(128) unsigned char smp[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smp);
    const IO* us = reinterpret_cast<const IO*>(smp + 128);
    float* part = reinterpret_cast<float*>(smp + 128 + (((size_t)Bn * m * sizeof(IO) + 15) & ~(size_t)15));
    if (threadIdx.x == 0) {
        tma::mbar_init(bar, 1);
        tma::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)Bn * m * sizeof(IO);
        tma::mbar_arrive_expect_tx(bar, bytes);
        tma::load_1d(smp + 128, u, bytes, bar);
    }
    tma::mbar_wait(bar, 0);
    const int c = blockIdx.x;  // output column: [0, r) p1, [r, r+n) B_k, [r+n, r+2n) C_k
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float acc[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) acc[b] = 0.f;
    for (int i = warp * 32 + lane; i < m; i += 256) {
        float wv = c < r ? Wd[(int64_t)i * r + c] : c < r + n ? WB[(int64_t)(c - r) * m + i]
                                                             : WC[(int64_t)(c - r - n) * m + i];
        // bf16 layers multiply bf16 activations by bf16-cast weights (layers._mm)
        if constexpr (sizeof(IO) == 2) wv = __bfloat162float(__float2bfloat16_rn(wv));
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (b < Bn) acc[b] = fmaf(wv, float(cvt(us[b * m + i])), acc[b]);
    }
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        if (b < Bn) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], o);
        }
    }
    if (lane < Bn) {
        float v = 0.f;
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (lane == b) v = acc[b];
        part[warp * 16 + lane] = v;
    }
    __syncthreads();
    if (threadIdx.x < Bn) {
        float v = 0.f;
        for (int w = 0; w < 8; ++w) v += part[w * 16 + threadIdx.x];  // fixed order
        out[(int64_t)threadIdx.x * (r + 2 * n) + c] = v;
    }
}

template <typename IO>
__global__ void s6_step_fused_kernel(float* __restrict__ x, const IO* __restrict__ u,
                                     const float* __restrict__ proj, const float* __restrict__ Wdp,
                                     const float* __restrict__ bdelta, const float* __restrict__ a_log,
                                     const float* __restrict__ Dskip, IO* __restrict__ y, int Bn, int D, int r,
                                     int N) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (b, d)
    if (i >= (int64_t)Bn * D) return;
    const int b = (int)(i / D), d = (int)(i % D);
    const float* pb = proj + (int64_t)b * (r + 2 * N);
    float pre = 0.f;
    for (int j = 0; j < r; ++j) pre = fmaf(pb[j], Wdp[(int64_t)j * D + d], pre);
    const float uk = float(cvt(u[i]));
    const float delta = Math<float>::softplus(pre + bdelta[d]);
    const float du = delta * uk;
    float acc = 0.f;
    for (int k = 0; k < N; ++k) {
        const float a = -Math<float>::exp(a_log[(int64_t)d * N + k]);
        float xv = x[i * N + k];
        xv = Math<float>::exp(delta * a) * xv + du * pb[r + k];
        x[i * N + k] = xv;
        acc += pb[r + N + k] * xv;
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

// RG-LRU token in ONE kernel (fp32 gate weights, batch <= 16): the two gate
// GEMVs qr = u W_r^T, qi = u W_i^T (layers.py:1213-1214) and the gated update.
// The batch's u rows land in shared memory with one bulk copy; each warp owns
// CPW = 2 channels and streams their rows of W_r and W_i (16-byte loads, 4
// rows x 4 iterations in flight per lane), butterfly-reduces the dot
// products and lane b applies the update of (b, w).  Bound: reading the
// weights once per token (2 W^2 fp32).
constexpr int kCPW = 2;

template <typename IO, int BM>
__global__ void __launch_bounds__(256) rglru_step_fused_kernel(float* __restrict__ x, const IO* __restrict__ u,
                                                               const float* __restrict__ Wr,
                                                               const float* __restrict__ Wi,
                                                               const float* __restrict__ lam,
                                                               const float* __restrict__ b_r,
                                                               const float* __restrict__ b_i, IO* __restrict__ y,
                                                               int Bn, int W) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    const IO* us = reinterpret_cast<const IO*>(smem + 128);  // [Bn][W]
    if (threadIdx.x == 0) {
        tma::mbar_init(bar, 1);
        tma::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)Bn * W * sizeof(IO);
        tma::mbar_arrive_expect_tx(bar, bytes);
        tma::load_1d(smem + 128, u, bytes, bar);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w0 = (blockIdx.x * 8 + warp) * kCPW;
    if (w0 >= W) return;  // (after the copy is issued: thread 0 is in warp 0)
    float ar[kCPW][BM], ai[kCPW][BM];
#pragma unroll
    for (int c = 0; c < kCPW; ++c)
#pragma unroll
        for (int b = 0; b < BM; ++b) ar[c][b] = ai[c][b] = 0.f;
    const float4* wr[kCPW];
    const float4* wi[kCPW];
#pragma unroll
    for (int c = 0; c < kCPW; ++c) {
        const int w = min(w0 + c, W - 1);
        wr[c] = reinterpret_cast<const float4*>(Wr + (int64_t)w * W);
        wi[c] = reinterpret_cast<const float4*>(Wi + (int64_t)w * W);
    }
    tma::mbar_wait(bar, 0);
#pragma unroll 4
    for (int k4 = lane; k4 < W / 4; k4 += 32) {
        float4 r4[kCPW], i4[kCPW];
#pragma unroll
        for (int c = 0; c < kCPW; ++c) r4[c] = __ldcs(wr[c] + k4), i4[c] = __ldcs(wi[c] + k4);
#pragma unroll
        for (int b = 0; b < BM; ++b) {
            if (b < Bn) {
                float4 u4;
                if constexpr (sizeof(IO) == 4) {
                    u4 = reinterpret_cast<const float4*>(us + b * W)[k4];
                } else {
                    const uint2 h = reinterpret_cast<const uint2*>(us + b * W)[k4];
                    u4.x = __uint_as_float(h.x << 16), u4.y = __uint_as_float(h.x & 0xFFFF0000u);
                    u4.z = __uint_as_float(h.y << 16), u4.w = __uint_as_float(h.y & 0xFFFF0000u);
                }
#pragma unroll
                for (int c = 0; c < kCPW; ++c) {
                    ar[c][b] += r4[c].x * u4.x + r4[c].y * u4.y + r4[c].z * u4.z + r4[c].w * u4.w;
                    ai[c][b] += i4[c].x * u4.x + i4[c].y * u4.y + i4[c].z * u4.z + i4[c].w * u4.w;
                }
            }
        }
    }
#pragma unroll
    for (int c = 0; c < kCPW; ++c) {
        float qr = 0.f, qi = 0.f;
#pragma unroll
        for (int b = 0; b < BM; ++b) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ar[c][b] += __shfl_xor_sync(0xffffffffu, ar[c][b], o);
                ai[c][b] += __shfl_xor_sync(0xffffffffu, ai[c][b], o);
            }
            if (lane == b) qr = ar[c][b], qi = ai[c][b];
        }
        const int w = w0 + c;
        if (lane < Bn && w < W) {
            const int64_t i = (int64_t)lane * W + w;
            const float uk = float(cvt(us[lane * W + w]));
            const float r = Math<float>::sigmoid(qr + b_r[w]);
            const float ig = Math<float>::sigmoid(qi + b_i[w]);
            const float loga = (8.f * r) * (-Math<float>::softplus(-lam[w]));  // GATE_POWER 8
            const float a = Math<float>::exp(loga);
            const float s = Math<float>::sqrt(-Math<float>::expm1(2.f * loga));
            const float xv = a * x[i] + (s * ig) * uk;
            x[i] = xv;
            st_io(y + i, xv);
        }
    }
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

int lrx_s6_step_fused(int io_dtype, void* x, const void* u, const void* W_delta, const void* W_delta_proj,
                      const void* W_B, const void* W_C, const void* b_delta, const void* a_log, const void* Dskip,
                      void* y, void* proj_ws, int64_t B, int64_t D, int64_t R, int64_t N, void* stream) {
    LRX_REQUIRE(B >= 1 && D >= 1 && R >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    const size_t esz = io_dtype == LRX_BF16 ? 2 : 4;
    const size_t ubytes = (size_t)B * D * esz;
    const size_t smem = 128 + ((ubytes + 15) & ~(size_t)15) + 8 * 16 * 4;
    LRX_REQUIRE(B <= 16 && smem <= 200 * 1024 && (io_dtype == LRX_F32 || io_dtype == LRX_BF16) && ubytes % 16 == 0 &&
                    (reinterpret_cast<uintptr_t>(u) & 15) == 0,
                LRX_ERR_UNSUPPORTED, "s6 fused step: batch <= 16, 16-byte u rows, f32 / bf16 I/O");
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g2 = (unsigned)cdiv(B * D, 128);
#define LRX_S6_FUSED(IO_)                                                                                         \
    do {                                                                                                          \
        auto k = step::s6_step_proj_kernel<IO_>;                                                                 \
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {   \
            set_error("s6 fused step: cannot reserve %zu B of shared memory", smem);                              \
            return LRX_ERR_CUDA;                                                                                 \
        }                                                                                                         \
        k<<<(unsigned)(R + 2 * N), 256, smem, st>>>((const IO_*)u, (const float*)W_delta, (const float*)W_B,      \
                                                    (const float*)W_C, (float*)proj_ws, (int)B, (int)D, (int)R,  \
                                                    (int)N);                                                      \
        step::s6_step_fused_kernel<IO_><<<g2, 128, 0, st>>>(                                                     \
            (float*)x, (const IO_*)u, (const float*)proj_ws, (const float*)W_delta_proj, (const float*)b_delta,  \
            (const float*)a_log, (const float*)Dskip, (IO_*)y, (int)B, (int)D, (int)R, (int)N);                  \
    } while (0)
    if (io_dtype == LRX_F32) LRX_S6_FUSED(float);
    else LRX_S6_FUSED(__nv_bfloat16);
#undef LRX_S6_FUSED
    return launched("lrx_s6_step_fused", 2);
}

int lrx_rglru_step_fused(int io_dtype, void* x, const void* u, const void* W_r, const void* W_i,
                         const void* lambda_param, const void* b_r, const void* b_i, void* y, int64_t B, int64_t W,
                         void* stream) {
    LRX_REQUIRE(B >= 1 && W >= 1, LRX_ERR_SHAPE, "bad extents");
    const size_t esz = io_dtype == LRX_BF16 ? 2 : 4;
    const size_t smem = 128 + (size_t)B * W * esz;
    LRX_REQUIRE(B <= 16 && W % 8 == 0 && smem <= 200 * 1024 && (io_dtype == LRX_F32 || io_dtype == LRX_BF16) &&
                    (reinterpret_cast<uintptr_t>(u) & 15) == 0,
                LRX_ERR_UNSUPPORTED, "rglru fused step: batch <= 16, width %% 8 == 0, f32 / bf16 I/O");
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (unsigned)cdiv(W, 8 * step::kCPW);
#define LRX_RG_FUSED(IO_, BM_)                                                                                  \
    do {                                                                                                        \
        auto k = step::rglru_step_fused_kernel<IO_, BM_>;                                                      \
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) { \
            set_error("rglru fused step: cannot reserve %zu B of shared memory", smem);                         \
            return LRX_ERR_CUDA;                                                                               \
        }                                                                                                       \
        k<<<g, 256, smem, st>>>((float*)x, (const IO_*)u, (const float*)W_r, (const float*)W_i,                 \
                                (const float*)lambda_param, (const float*)b_r, (const float*)b_i, (IO_*)y, (int)B, \
                                (int)W);                                                                        \
    } while (0)
#define LRX_RG_FUSED_B(IO_)                \
    do {                                   \
        if (B <= 1) LRX_RG_FUSED(IO_, 1);  \
        else if (B <= 2) LRX_RG_FUSED(IO_, 2);  \
        else if (B <= 4) LRX_RG_FUSED(IO_, 4);  \
        else if (B <= 8) LRX_RG_FUSED(IO_, 8);  \
        else LRX_RG_FUSED(IO_, 16);        \
    } while (0)
    if (io_dtype == LRX_F32) LRX_RG_FUSED_B(float);
    else LRX_RG_FUSED_B(__nv_bfloat16);
#undef LRX_RG_FUSED_B
#undef LRX_RG_FUSED
    return launched("lrx_rglru_step_fused");
}

}  // extern "C"
