// Generic diagonal scan operator on time-major [L, N] arrays.
//
// Replaces the reference's scan operator: scan_sequential / scan_parallel
// (pkg/src/linrec/scan.py:127-201) over the numba loops scan_const,
// scan_var, compose_*, local_scan_*, fixup_* (_scan_kernels.py:17-128), and
// the pullback backward_const / backward_var + _scan_pullback
// (_scan_kernels.py:131-153, autograd.py:113-140).
//
// B200 design: one thread per lane (consecutive threads = consecutive lanes,
// so every step is one coalesced 128 B+ row segment per warp), a register
// tile of T time steps per thread, and time chunks chained across CTAs by a
// decoupled look-back (lrx_common.cuh).  One read of a/b and one write of
// out per element: the HBM minimum.  The reference's three passes
// (local scan, serial stitch, fixup) collapse into this single pass.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <stdlib.h>
#include <type_traits>

#include "lrx_common.cuh"

#include <algorithm>
#include "lrx_host.h"

namespace lrx {

static thread_local char g_err[512];
std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

constexpr int kLanes = 128;  // threads (= lanes) per CTA

template <typename V> struct Tile;            // register tile length per type
template <> struct Tile<float> { static constexpr int T = 32; };
template <> struct Tile<double> { static constexpr int T = 16; };
template <> struct Tile<cplx<float>> { static constexpr int T = 16; };
template <> struct Tile<cplx<double>> { static constexpr int T = 8; };

template <typename V> __device__ __forceinline__ V ld(const V* p) { return *p; }
template <> __device__ __forceinline__ cplx<float> ld(const cplx<float>* p) {
    float2 v = __ldcs(reinterpret_cast<const float2*>(p));
    return {v.x, v.y};
}
template <> __device__ __forceinline__ cplx<double> ld(const cplx<double>* p) {
    double2 v = __ldcs(reinterpret_cast<const double2*>(p));
    return {v.x, v.y};
}
template <> __device__ __forceinline__ float ld(const float* p) { return __ldcs(p); }
template <> __device__ __forceinline__ double ld(const double* p) { return __ldcs(p); }
template <typename V> __device__ __forceinline__ void st(V* p, V v) { *p = v; }
template <> __device__ __forceinline__ void st(cplx<float>* p, cplx<float> v) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v.re, v.im));
}
template <> __device__ __forceinline__ void st(cplx<double>* p, cplx<double> v) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v.re, v.im));
}
template <> __device__ __forceinline__ void st(float* p, float v) { __stcs(p, v); }
template <> __device__ __forceinline__ void st(double* p, double v) { __stcs(p, v); }

// ---------------------------------------------------------------- forward
template <typename V, bool PER_STEP>
__global__ void __launch_bounds__(kLanes) scan_fwd_kernel(const V* __restrict__ a, const V* __restrict__ b,
                                                          const V* __restrict__ x0, V* __restrict__ out,
                                                          int64_t L, int64_t N, int n_blk, LookbackWS ws) {
    using Tr = Traits<V>;
    constexpr int T = Tile<V>::T;
    const int tile = next_tile(ws.ticket);
    const int c = tile / n_blk, blk = tile % n_blk;
    const int64_t lane = (int64_t)blk * kLanes + threadIdx.x;
    const bool valid = lane < N;
    const int64_t t0 = (int64_t)c * T;
    const int nt = (int)min((int64_t)T, L - t0);

    V av[T], bv[T];
    const V ac = (!PER_STEP && valid) ? ld(a + lane) : Tr::one();
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const bool ok = valid && k < nt;
        const int64_t off = (t0 + k) * N + lane;
        bv[k] = ok ? ld(b + off) : Tr::zero();
        av[k] = ok ? (PER_STEP ? ld(a + off) : ac) : Tr::one();
    }
    V A = Tr::one(), X = Tr::zero();
#pragma unroll
    for (int k = 0; k < T; ++k) {
        X = av[k] * X + bv[k];
        A = av[k] * A;
    }
    V* agg_a = static_cast<V*>(ws.agg_a);
    V* agg_x = static_cast<V*>(ws.agg_x);
    V* inc_x = static_cast<V*>(ws.inc_x);
    const int64_t woff = (int64_t)c * N + lane;
    int* sw = ws.status + (int64_t)c * n_blk + blk;
    V xin;
    if (c == 0) {
        xin = (x0 && valid) ? ld(x0 + lane) : Tr::zero();
    } else {
        lb_publish<V>(sw, LB_AGG, agg_a + woff, A, agg_x + woff, X, valid);
        xin = lb_lookback<V>(ws, c, blk, n_blk, lane, N, valid);
    }
    if ((c % kAnchor) == 0)
        lb_publish<V>(sw, LB_INC, (V*)nullptr, A, inc_x + woff, A * xin + X, valid);
    V x = xin;
#pragma unroll
    for (int k = 0; k < T; ++k) {
        x = av[k] * x + bv[k];
        if (valid && k < nt) st(out + (t0 + k) * N + lane, x);
    }
}

// ---------------------------------------------------------------- streaming
// When the lanes alone fill the GPU (>= ~32 warps per SM), one thread walks
// its lane over the whole sequence: no chunk aggregates, no look-back, each
// array streamed exactly once (3 streams forward, 5 backward); loads run a
// T-step register tile ahead of the recurrence.
// register tile of the streaming walk: short enough for ~40 resident warps per SM
template <typename V> struct STile { static constexpr int T = 8; };
template <> struct STile<cplx<double>> { static constexpr int T = 4; };

template <typename V, bool PER_STEP, bool AGG>
__global__ void __launch_bounds__(kLanes) scan_fwd_stream_kernel(const V* __restrict__ a, const V* __restrict__ b,
                                                                 const V* __restrict__ x0, V* __restrict__ out,
                                                                 V* __restrict__ mapA, V* __restrict__ mapX,
                                                                 int64_t L, int64_t N, int64_t seg_len) {
    // segment s = blockIdx.y walks [s seg_len, (s+1) seg_len); AGG: its map
    // (prod a, state from 0) -> mapA / mapX; main: folds the maps of the
    // segments to its left in a fixed order, then writes the states
    using Tr = Traits<V>;
    constexpr int T = STile<V>::T;
    const int64_t lane = (int64_t)blockIdx.x * kLanes + threadIdx.x;
    if (lane >= N) return;
    const int s = blockIdx.y;
    const int64_t tb = (int64_t)s * seg_len, te = min(L, tb + seg_len);
    const V ac = PER_STEP ? Tr::one() : ld(a + lane);
    V x = Tr::zero(), A = Tr::one();
    if (!AGG) {
        x = x0 ? ld(x0 + lane) : Tr::zero();
        for (int r = 0; r < s; ++r) x = mapA[(int64_t)r * N + lane] * x + mapX[(int64_t)r * N + lane];
    }
    for (int64_t t0 = tb; t0 < te; t0 += T) {
        const int nt = (int)min((int64_t)T, te - t0);
        V av[T], bv[T];
#pragma unroll
        for (int k = 0; k < T; ++k) {
            const int64_t off = (t0 + k) * N + lane;
            bv[k] = k < nt ? ld(b + off) : Tr::zero();
            av[k] = PER_STEP ? (k < nt ? ld(a + off) : Tr::one()) : ac;
        }
#pragma unroll
        for (int k = 0; k < T; ++k) {
            if (k < nt) {
                x = av[k] * x + bv[k];
                if (AGG) A = av[k] * A;
                else st(out + (t0 + k) * N + lane, x);
            }
        }
    }
    if (AGG) {
        mapA[(int64_t)s * N + lane] = A;
        mapX[(int64_t)s * N + lane] = x;
    }
}

// backward aggregate of segment s: its cotangent map (prod conj a, the carry
// leaving to the left from a zero carry entering on the right)
template <typename V, bool PER_STEP>
__global__ void __launch_bounds__(kLanes) scan_bwd_agg_kernel(const V* __restrict__ a, const V* __restrict__ gx,
                                                              V* __restrict__ mapA, V* __restrict__ mapH, int64_t L,
                                                              int64_t N, int64_t seg_len) {
    using Tr = Traits<V>;
    constexpr int T = STile<V>::T;
    const int64_t lane = (int64_t)blockIdx.x * kLanes + threadIdx.x;
    if (lane >= N) return;
    const int s = blockIdx.y + 1;  // segment 0's map is never folded
    const int64_t tb = (int64_t)s * seg_len, te = min(L, tb + seg_len);
    const V acst = PER_STEP ? Tr::one() : Tr::cj(ld(a + lane));
    V h = Tr::zero(), A = Tr::one();
    for (int64_t t1 = te; t1 > tb; t1 -= T) {
        const int64_t t0 = max(tb, t1 - T);
        const int nt = (int)(t1 - t0);
        V acv[T], gxv[T];
#pragma unroll
        for (int k = 0; k < T; ++k) {
            const int64_t off = (t0 + k) * N + lane;
            gxv[k] = k < nt ? ld(gx + off) : Tr::zero();
            acv[k] = PER_STEP ? (k < nt ? Tr::cj(ld(a + off)) : Tr::one()) : acst;
        }
#pragma unroll
        for (int k = T - 1; k >= 0; --k) {
            if (k < nt) {
                h = acv[k] * (gxv[k] + h);
                A = acv[k] * A;
            }
        }
    }
    mapA[(int64_t)s * N + lane] = A;
    mapH[(int64_t)s * N + lane] = h;
}

// backward main: segment s walks right to left after folding the maps of the
// segments to its right (fixed order); for a constant a its sum of
// g conj(x_prev) lands in ga[s N + lane] (summed over segments by the caller)
template <typename V, bool PER_STEP>
__global__ void __launch_bounds__(kLanes) scan_bwd_stream_kernel(const V* __restrict__ a, const V* __restrict__ x,
                                                                 const V* __restrict__ x0, const V* __restrict__ gx,
                                                                 V* __restrict__ gb, V* __restrict__ ga,
                                                                 V* __restrict__ gx0, const V* __restrict__ mapA,
                                                                 const V* __restrict__ mapH, int64_t L, int64_t N,
                                                                 int64_t seg_len) {
    using Tr = Traits<V>;
    constexpr int T = STile<V>::T;
    const int64_t lane = (int64_t)blockIdx.x * kLanes + threadIdx.x;
    if (lane >= N) return;
    const int s = blockIdx.y, S = gridDim.y;
    const int64_t tb = (int64_t)s * seg_len, te = min(L, tb + seg_len);
    const V acst = PER_STEP ? Tr::one() : Tr::cj(ld(a + lane));
    const V x0v = x0 ? ld(x0 + lane) : Tr::zero();
    V h = Tr::zero(), gsum = Tr::zero();
    for (int r = S - 1; r > s; --r) h = mapA[(int64_t)r * N + lane] * h + mapH[(int64_t)r * N + lane];
    for (int64_t t1 = te; t1 > tb; t1 -= T) {
        const int64_t t0 = max(tb, t1 - T);
        const int nt = (int)(t1 - t0);
        V acv[T], gxv[T], xpv[T];
#pragma unroll
        for (int k = 0; k < T; ++k) {
            const int64_t off = (t0 + k) * N + lane;
            const bool ok = k < nt;
            gxv[k] = ok ? ld(gx + off) : Tr::zero();
            acv[k] = PER_STEP ? (ok ? Tr::cj(ld(a + off)) : Tr::one()) : acst;
            if (ga) xpv[k] = !ok ? Tr::zero() : (t0 + k == 0) ? x0v : ld(x + off - N);
        }
#pragma unroll
        for (int k = T - 1; k >= 0; --k) {
            if (k < nt) {
                const V g = gxv[k] + h;
                h = acv[k] * g;
                const int64_t off = (t0 + k) * N + lane;
                st(gb + off, g);
                if (ga) {
                    const V contrib = g * Tr::cj(xpv[k]);
                    if constexpr (PER_STEP) st(ga + off, contrib);
                    else gsum = gsum + contrib;
                }
            }
        }
    }
    if (!PER_STEP && ga) st(ga + (int64_t)s * N + lane, gsum);
    if (gx0 && s == 0) st(gx0 + lane, h);
}

// Time segments of the streaming walk (S = 1: the whole sequence, one pass);
// segments of >= 64 steps.
// LRX_SCAN_SEGS overrides.
static int64_t stream_segs(int64_t L, int64_t N, int64_t* seg_len) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t warps = cdiv(N, (int64_t)kLanes) * (kLanes / 32);
    // lanes alone at >= 16 warps per SM stream best in one pass (c64 x 131072:
    // 2.1 ms unsegmented vs 2.8 ms in 2 segments); fewer: ~32 warps per SM
    int64_t S = warps >= (int64_t)sms * 16 ? 1 : cdiv((int64_t)sms * 32, warps);
    if (const char* e = getenv("LRX_SCAN_SEGS")) S = std::max<int64_t>(1, atoll(e));
    S = std::min<int64_t>(S, std::max<int64_t>(1, L / 64));
    *seg_len = cdiv(cdiv(L, S), (int64_t)8) * 8;
    return cdiv(L, *seg_len);
}

// The streaming walk (time-segmented when the lanes are few) is the default;
// LRX_SCAN_STREAM=0 selects the single-pass chunked look-back kernels.
static bool stream_ok() {
    const char* e = getenv("LRX_SCAN_STREAM");
    return !(e && atoi(e) == 0);
}

// ---------------------------------------------------------------- backward
// Reverse chunks in scan order s = n_chunks-1-c.  Within chunk c the carry
// entering from the right is h = conj(a[t1]) g[t1] (t1 = first step of chunk
// c+1); the chunk publishes h_out = conj(a[t0]) g[t0].  For chunk 0 that is
// exactly grad_x0 = conj(a_0) g_0.
template <typename V, bool PER_STEP>
__global__ void __launch_bounds__(kLanes) scan_bwd_kernel(const V* __restrict__ a, const V* __restrict__ x,
                                                          const V* __restrict__ x0, const V* __restrict__ gx,
                                                          V* __restrict__ gb, V* __restrict__ ga,
                                                          V* __restrict__ ga_part, V* __restrict__ gx0,
                                                          int64_t L, int64_t N, int n_blk, int n_chunks,
                                                          LookbackWS ws) {
    using Tr = Traits<V>;
    constexpr int T = Tile<V>::T;
    const int tile = next_tile(ws.ticket);
    const int s = tile / n_blk, blk = tile % n_blk;
    const int c = n_chunks - 1 - s;
    const int64_t lane = (int64_t)blk * kLanes + threadIdx.x;
    const bool valid = lane < N;
    const int64_t t0 = (int64_t)c * T;
    const int nt = (int)min((int64_t)T, L - t0);

    V acv[T], gxv[T];
    const V acst = (!PER_STEP && valid) ? Tr::cj(ld(a + lane)) : Tr::one();
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const bool ok = valid && k < nt;
        const int64_t off = (t0 + k) * N + lane;
        gxv[k] = ok ? ld(gx + off) : Tr::zero();
        acv[k] = ok ? (PER_STEP ? Tr::cj(ld(a + off)) : acst) : Tr::one();
    }
    // local aggregate from h_in = 0
    V A = Tr::one(), H = Tr::zero();
#pragma unroll
    for (int k = T - 1; k >= 0; --k) {
        const V g = gxv[k] + H;
        H = acv[k] * g;
        A = acv[k] * A;
    }
    V* agg_a = static_cast<V*>(ws.agg_a);
    V* agg_x = static_cast<V*>(ws.agg_x);
    V* inc_x = static_cast<V*>(ws.inc_x);
    const int64_t woff = (int64_t)s * N + lane;
    int* sw = ws.status + (int64_t)s * n_blk + blk;
    V hin;
    if (s == 0) {
        hin = Tr::zero();
    } else {
        lb_publish<V>(sw, LB_AGG, agg_a + woff, A, agg_x + woff, H, valid);
        hin = lb_lookback<V>(ws, s, blk, n_blk, lane, N, valid);
    }
    if ((s % kAnchor) == 0)
        lb_publish<V>(sw, LB_INC, (V*)nullptr, A, inc_x + woff, A * hin + H, valid);

    V h = hin, gsum = Tr::zero();
#pragma unroll
    for (int k = T - 1; k >= 0; --k) {
        if (valid && k < nt) {
            const V g = gxv[k] + h;
            h = acv[k] * g;
            const int64_t off = (t0 + k) * N + lane;
            st(gb + off, g);
            if (ga || ga_part) {
                const int64_t tk = t0 + k;
                V xp = (tk == 0) ? (x0 ? ld(x0 + lane) : Tr::zero()) : ld(x + off - N);
                const V contrib = g * Tr::cj(xp);
                if constexpr (PER_STEP) st(ga + off, contrib);
                else gsum = gsum + contrib;
            }
        }
    }
    if (!PER_STEP && ga_part && valid) st(ga_part + (int64_t)c * N + lane, gsum);
    if (c == 0 && gx0 && valid) st(gx0 + lane, h);
}

// ---------------------------------------------------------------- reduce
template <typename V>
__global__ void reduce_rows_kernel(const V* __restrict__ in, V* __restrict__ out, int64_t R, int64_t N) {
    // block = 32 columns x RL row lanes; lane r folds rows r, r+RL, ... then
    // the RL partial sums are combined by a fixed tree: deterministic, and
    // coalesced over the 32 columns of every row
    extern __shared__ __align__(16) unsigned char red_raw[];
    V* red = reinterpret_cast<V*>(red_raw);
    const int RL = blockDim.x / 32;
    const int c = threadIdx.x & 31, r0 = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * 32 + c;
    V acc = Traits<V>::zero();
    if (j < N)
        for (int64_t r = r0; r < R; r += RL) acc = acc + in[r * N + j];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int h = RL / 2; h >= 1; h >>= 1) {
        if (r0 < h) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + 32 * h];
        __syncthreads();
    }
    if (r0 == 0 && j < N) out[j] = red[c];
}

// Few rows, many columns (the S6 dB_k / dC_k channel-block partials: 24-32
// rows of B*L*N columns): thread per 4 columns, 8 rows' 16-byte loads in
// flight, summed in row order (deterministic).
__global__ void reduce_cols4_kernel(const float4* __restrict__ in, float4* __restrict__ out, int64_t R, int64_t N4) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N4) return;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t r = 0;
    for (; r + 8 <= R; r += 8) {
        float4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldcs(in + (r + i) * N4 + j);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc.x += v[i].x, acc.y += v[i].y, acc.z += v[i].z, acc.w += v[i].w;
    }
    for (; r < R; ++r) {
        const float4 v = __ldcs(in + r * N4 + j);
        acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
    out[j] = acc;
}

// launch: many row lanes when there are few columns (the S5/LRU parameter
// partials: R ~ 1e4 rows of P columns), 8 when columns are plentiful
template <typename V>
static void reduce_rows_launch(const V* in, V* out, int64_t R, int64_t N, cudaStream_t st) {
    if constexpr (std::is_same<V, float>::value) {
        if (R <= 64 && N % 4 == 0 && N >= 4 * 256 * 148 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
            (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
            const int64_t n4 = N / 4;
            reduce_cols4_kernel<<<(unsigned)cdiv(n4, 256), 256, 0, st>>>(reinterpret_cast<const float4*>(in),
                                                                         reinterpret_cast<float4*>(out), R, n4);
            return;
        }
    }
    const int64_t blocks = cdiv(N, 32);
    int RL = 8;
    while (RL < 32 && blocks * RL < 148 * 64 && RL * 8 < R) RL *= 2;
    reduce_rows_kernel<V><<<(unsigned)blocks, 32 * RL, 32 * RL * sizeof(V), st>>>(in, out, R, N);
}

// Two-stage variant for long columns: stage 1 folds row groups of `rpg`
// rows (optionally of the elementwise product in[r,j] * in2[r,j]) into
// partials [G, N]; stage 2 is reduce_rows_kernel over the G partials.  Fixed
// order throughout (deterministic for given R, N).
template <typename V>
__global__ void reduce_rows_part_kernel(const V* __restrict__ in, const V* __restrict__ in2, V* __restrict__ part,
                                        int64_t R, int64_t N, int64_t rpg) {
    __shared__ V red[256];
    const int c = threadIdx.x & 31, r0 = threadIdx.x >> 5;  // 8 row lanes
    const int64_t j = (int64_t)blockIdx.x * 32 + c;
    const int64_t rb = (int64_t)blockIdx.y * rpg, re = min(R, rb + rpg);
    V acc = Traits<V>::zero();
    if (j < N) {
        // four independent partial sums keep four rows' loads in flight
        V a1 = Traits<V>::zero(), a2 = a1, a3 = a1;
        int64_t r = rb + r0;
        if (in2) {
            for (; r + 24 < re; r += 32) {
                acc = acc + in[r * N + j] * in2[r * N + j];
                a1 = a1 + in[(r + 8) * N + j] * in2[(r + 8) * N + j];
                a2 = a2 + in[(r + 16) * N + j] * in2[(r + 16) * N + j];
                a3 = a3 + in[(r + 24) * N + j] * in2[(r + 24) * N + j];
            }
            for (; r < re; r += 8) acc = acc + in[r * N + j] * in2[r * N + j];
        } else {
            for (; r + 24 < re; r += 32) {
                acc = acc + in[r * N + j];
                a1 = a1 + in[(r + 8) * N + j];
                a2 = a2 + in[(r + 16) * N + j];
                a3 = a3 + in[(r + 24) * N + j];
            }
            for (; r < re; r += 8) acc = acc + in[r * N + j];
        }
        acc = (acc + a1) + (a2 + a3);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int h = 4; h >= 1; h >>= 1) {
        if (r0 < h) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + 32 * h];
        __syncthreads();
    }
    if (r0 == 0 && j < N) part[(int64_t)blockIdx.y * N + j] = red[c];
}

// float, N % 4 == 0: float4 loads (a warp reads 512 contiguous bytes per row),
// so four times the bytes are in flight per load instruction
__global__ void reduce_rows_part4_kernel(const float4* __restrict__ in, const float4* __restrict__ in2,
                                         float4* __restrict__ part, int64_t R, int64_t N4, int64_t rpg) {
    __shared__ float4 red[256];
    const int c = threadIdx.x & 31, r0 = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * 32 + c;
    const int64_t rb = (int64_t)blockIdx.y * rpg, re = min(R, rb + rpg);
    float4 a0 = make_float4(0, 0, 0, 0), a1 = a0;
    auto fma4 = [](float4 acc, float4 x, float4 y) {
        return make_float4(fmaf(x.x, y.x, acc.x), fmaf(x.y, y.y, acc.y), fmaf(x.z, y.z, acc.z), fmaf(x.w, y.w, acc.w));
    };
    auto add4 = [](float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); };
    if (j < N4) {
        int64_t r = rb + r0;
        if (in2) {
            for (; r + 8 < re; r += 16) {
                a0 = fma4(a0, __ldcs(in + r * N4 + j), __ldcs(in2 + r * N4 + j));
                a1 = fma4(a1, __ldcs(in + (r + 8) * N4 + j), __ldcs(in2 + (r + 8) * N4 + j));
            }
            for (; r < re; r += 8) a0 = fma4(a0, __ldcs(in + r * N4 + j), __ldcs(in2 + r * N4 + j));
        } else {
            for (; r + 8 < re; r += 16) {
                a0 = add4(a0, __ldcs(in + r * N4 + j));
                a1 = add4(a1, __ldcs(in + (r + 8) * N4 + j));
            }
            for (; r < re; r += 8) a0 = add4(a0, __ldcs(in + r * N4 + j));
        }
    }
    red[threadIdx.x] = add4(a0, a1);
    __syncthreads();
    for (int h = 4; h >= 1; h >>= 1) {
        if (r0 < h) red[threadIdx.x] = add4(red[threadIdx.x], red[threadIdx.x + 32 * h]);
        __syncthreads();
    }
    if (r0 == 0 && j < N4) part[(int64_t)blockIdx.y * N4 + j] = red[c];
}

static int64_t reduce_groups4(int64_t R, int64_t N) {  // float4 plan (N % 4 == 0)
    const int64_t cb = cdiv(N / 4, 32);
    return std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * 148, cb), R / 256));
}

static int64_t reduce_groups(int64_t R, int64_t N) {
    const int64_t cb = cdiv(N, 32);
    int64_t G = cdiv(4 * 148, cb);                 // ~4 blocks of 256 threads per SM
    G = std::min<int64_t>(G, std::max<int64_t>(1, R / 256));
    return std::max<int64_t>(1, G);
}


template <typename V>
static size_t reduce_ws(int64_t R, int64_t N) {
    int64_t G = reduce_groups(R, N);
    if (sizeof(V) == 4 && !Traits<V>::complex && N % 4 == 0) G = std::max(G, reduce_groups4(R, N));
    return G > 1 ? (size_t)G * N * sizeof(V) : 0;
}

template <typename V>
static int reduce_rows2(const V* in, const V* in2, V* out, int64_t R, int64_t N, void* ws, size_t wb,
                        cudaStream_t st) {
    if constexpr (sizeof(V) == 4 && !Traits<V>::complex) {
        const bool al = !((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(in2) |
                           reinterpret_cast<uintptr_t>(out)) & 15);
        if (N % 4 == 0 && al) {
            const int64_t N4 = N / 4, cb = cdiv(N4, 32);
            const int64_t G = reduce_groups4(R, N);
            const int64_t rpg = cdiv(R, G);
            if (G == 1) {
                reduce_rows_part4_kernel<<<dim3((unsigned)cb, 1), 256, 0, st>>>(
                    (const float4*)in, (const float4*)in2, (float4*)out, R, N4, rpg);
                return launched("lrx_reduce_rows_ws");
            }
            LRX_REQUIRE(ws && wb >= (size_t)G * N * sizeof(V), LRX_ERR_VALUE,
                        "reduce_rows: workspace of %zu bytes needed", (size_t)G * N * sizeof(V));
            reduce_rows_part4_kernel<<<dim3((unsigned)cb, (unsigned)G), 256, 0, st>>>(
                (const float4*)in, (const float4*)in2, (float4*)ws, R, N4, rpg);
            reduce_rows_launch<V>(static_cast<V*>(ws), out, G, N, st);
            return launched("lrx_reduce_rows_ws", 2);
        }
    }
    const int64_t G = reduce_groups(R, N);
    const int64_t rpg = cdiv(R, G);
    if (G == 1) {
        reduce_rows_part_kernel<V><<<dim3((unsigned)cdiv(N, 32), 1), 256, 0, st>>>(in, in2, out, R, N, rpg);
        return launched("lrx_reduce_rows_ws");
    }
    LRX_REQUIRE(ws && wb >= (size_t)G * N * sizeof(V), LRX_ERR_VALUE, "reduce_rows: workspace of %zu bytes needed",
                (size_t)G * N * sizeof(V));
    V* part = static_cast<V*>(ws);
    reduce_rows_part_kernel<V><<<dim3((unsigned)cdiv(N, 32), (unsigned)G), 256, 0, st>>>(in, in2, part, R, N, rpg);
    reduce_rows_launch<V>(part, out, G, N, st);
    return launched("lrx_reduce_rows_ws", 2);
}

// ---------------------------------------------------------------- host side
template <typename V>
static void chunking(int64_t L, int64_t N, int* n_chunks, int* n_blk) {
    *n_chunks = (int)cdiv(L, Tile<V>::T);
    *n_blk = (int)cdiv(N, kLanes);
}

template <typename V>
static size_t ws_bytes(int64_t L, int64_t N, bool bwd) {
    int nc, nb;
    chunking<V>(L, N, &nc, &nb);
    Carver cv(nullptr);
    cv.take<int>(1);
    cv.take<int>((size_t)nc * nb);
    cv.take<V>((size_t)nc * N);
    cv.take<V>((size_t)nc * N);
    cv.take<V>((size_t)nc * N);
    if (bwd) cv.take<V>((size_t)nc * N);
    return cv.off;
}

template <typename V>
static int carve(void* w, size_t wb, int64_t L, int64_t N, bool bwd, LookbackWS* ws, V** part,
                 cudaStream_t st) {
    int nc, nb;
    chunking<V>(L, N, &nc, &nb);
    const size_t need = ws_bytes<V>(L, N, bwd);
    LRX_REQUIRE(w != nullptr && wb >= need, LRX_ERR_VALUE, "workspace too small: %zu < %zu", wb, need);
    Carver cv(w);
    ws->ticket = cv.take<int>(1);
    ws->status = cv.take<int>((size_t)nc * nb);
    const size_t head = cv.off;
    ws->agg_a = cv.take<V>((size_t)nc * N);
    ws->agg_x = cv.take<V>((size_t)nc * N);
    ws->inc_x = cv.take<V>((size_t)nc * N);
    if (part) *part = bwd ? cv.take<V>((size_t)nc * N) : nullptr;
    if (cudaMemsetAsync(w, 0, head, st) != cudaSuccess) {
        set_error("workspace memset failed");
        return LRX_ERR_CUDA;
    }
    return LRX_OK;
}

template <typename V>
static int fwd_t(int per_step, const void* a, const void* b, const void* x0, void* out, int64_t L, int64_t N,
                 void* w, size_t wb, cudaStream_t st) {
    if (stream_ok()) {
        int64_t seg;
        const int64_t S = stream_segs(L, N, &seg);
        LRX_REQUIRE(S == 1 || (w && wb >= (size_t)2 * S * N * sizeof(V)), LRX_ERR_VALUE, "scan workspace too small");
        V* mA = static_cast<V*>(w);
        V* mX = mA + S * N;
        const unsigned g = (unsigned)cdiv(N, kLanes);
        int n = 1;
        if (S > 1) {
            if (per_step)
                scan_fwd_stream_kernel<V, true, true><<<dim3(g, (unsigned)(S - 1)), kLanes, 0, st>>>(
                    (const V*)a, (const V*)b, nullptr, nullptr, mA, mX, L, N, seg);
            else
                scan_fwd_stream_kernel<V, false, true><<<dim3(g, (unsigned)(S - 1)), kLanes, 0, st>>>(
                    (const V*)a, (const V*)b, nullptr, nullptr, mA, mX, L, N, seg);
            ++n;
        }
        if (per_step)
            scan_fwd_stream_kernel<V, true, false><<<dim3(g, (unsigned)S), kLanes, 0, st>>>(
                (const V*)a, (const V*)b, (const V*)x0, (V*)out, mA, mX, L, N, seg);
        else
            scan_fwd_stream_kernel<V, false, false><<<dim3(g, (unsigned)S), kLanes, 0, st>>>(
                (const V*)a, (const V*)b, (const V*)x0, (V*)out, mA, mX, L, N, seg);
        return launched("lrx_scan_fwd/stream", n);
    }
    int nc, nb;
    chunking<V>(L, N, &nc, &nb);
    LookbackWS ws;
    int rc = carve<V>(w, wb, L, N, false, &ws, nullptr, st);
    if (rc) return rc;
    const dim3 grid((unsigned)((int64_t)nc * nb));
    if (per_step)
        scan_fwd_kernel<V, true><<<grid, kLanes, 0, st>>>((const V*)a, (const V*)b, (const V*)x0, (V*)out, L, N,
                                                          nb, ws);
    else
        scan_fwd_kernel<V, false><<<grid, kLanes, 0, st>>>((const V*)a, (const V*)b, (const V*)x0, (V*)out, L, N,
                                                           nb, ws);
    return launched("lrx_scan_fwd");
}

template <typename V>
static int bwd_t(int per_step, const void* a, const void* x, const void* x0, const void* gx, void* gb, void* ga,
                 void* gx0, int64_t L, int64_t N, void* w, size_t wb, cudaStream_t st) {
    if (stream_ok()) {
        int64_t seg;
        const int64_t S = stream_segs(L, N, &seg);
        const bool part = !per_step && ga && S > 1;  // constant a: per-segment partial sums
        const size_t need = (size_t)(S > 1 ? 2 * S * N : 0) * sizeof(V) + (part ? (size_t)S * N * sizeof(V) : 0);
        LRX_REQUIRE(need == 0 || (w && wb >= need), LRX_ERR_VALUE, "scan workspace too small");
        V* mA = static_cast<V*>(w);
        V* mH = mA + S * N;
        V* gap = part ? mH + S * N : (V*)ga;
        const unsigned g = (unsigned)cdiv(N, kLanes);
        int n = 1;
        if (S > 1) {  // maps of segments 1 .. S-1
            if (per_step)
                scan_bwd_agg_kernel<V, true><<<dim3(g, (unsigned)(S - 1)), kLanes, 0, st>>>((const V*)a, (const V*)gx,
                                                                                          mA, mH, L, N, seg);
            else
                scan_bwd_agg_kernel<V, false><<<dim3(g, (unsigned)(S - 1)), kLanes, 0, st>>>((const V*)a, (const V*)gx,
                                                                                           mA, mH, L, N, seg);
            ++n;
        }
        if (per_step)
            scan_bwd_stream_kernel<V, true><<<dim3(g, (unsigned)S), kLanes, 0, st>>>(
                (const V*)a, (const V*)x, (const V*)x0, (const V*)gx, (V*)gb, (V*)ga, (V*)gx0, mA, mH, L, N, seg);
        else
            scan_bwd_stream_kernel<V, false><<<dim3(g, (unsigned)S), kLanes, 0, st>>>(
                (const V*)a, (const V*)x, (const V*)x0, (const V*)gx, (V*)gb, (V*)gap, (V*)gx0, mA, mH, L, N, seg);
        if (int rc = launched("lrx_scan_bwd/stream", n)) return rc;
        if (!part) return LRX_OK;
        reduce_rows_launch<V>(gap, (V*)ga, S, N, st);
        return launched("lrx_scan_bwd/reduce");
    }
    int nc, nb;
    chunking<V>(L, N, &nc, &nb);
    LookbackWS ws;
    V* part = nullptr;
    int rc = carve<V>(w, wb, L, N, true, &ws, &part, st);
    if (rc) return rc;
    const dim3 grid((unsigned)((int64_t)nc * nb));
    if (per_step) {
        scan_bwd_kernel<V, true><<<grid, kLanes, 0, st>>>((const V*)a, (const V*)x, (const V*)x0, (const V*)gx,
                                                          (V*)gb, (V*)ga, nullptr, (V*)gx0, L, N, nb, nc, ws);
        return launched("lrx_scan_bwd");
    }
    scan_bwd_kernel<V, false><<<grid, kLanes, 0, st>>>((const V*)a, (const V*)x, (const V*)x0, (const V*)gx,
                                                       (V*)gb, nullptr, ga ? part : nullptr, (V*)gx0, L, N, nb,
                                                       nc, ws);
    rc = launched("lrx_scan_bwd");
    if (rc || !ga) return rc;
    reduce_rows_launch<V>(part, (V*)ga, nc, N, st);
    return launched("lrx_scan_bwd/reduce");
}

}  // namespace lrx

using namespace lrx;

#define LRX_DISPATCH(dt, FN, ...)                                         \
    switch (dt) {                                                         \
        case LRX_F32: return FN<float>(__VA_ARGS__);                      \
        case LRX_F64: return FN<double>(__VA_ARGS__);                     \
        case LRX_C64: return FN<cplx<float>>(__VA_ARGS__);                \
        case LRX_C128: return FN<cplx<double>>(__VA_ARGS__);              \
        default: set_error("unsupported dtype %d", dt); return LRX_ERR_VALUE; \
    }

#define LRX_DISPATCH_SZ(dt, FN, ...)                                      \
    switch (dt) {                                                         \
        case LRX_F32: return FN<float>(__VA_ARGS__);                      \
        case LRX_F64: return FN<double>(__VA_ARGS__);                     \
        case LRX_C64: return FN<cplx<float>>(__VA_ARGS__);                \
        case LRX_C128: return FN<cplx<double>>(__VA_ARGS__);              \
        default: return 0;                                                \
    }

extern "C" {

const char* lrx_last_error(void) { return g_err; }
int lrx_version(void) { return 1; }
int64_t lrx_launch_count(void) { return g_launches.load(); }

size_t lrx_scan_workspace_bytes(int dtype, int64_t L, int64_t N) {
    if (L < 1 || N < 1) return 256;
    LRX_DISPATCH_SZ(dtype, ws_bytes, L, N, false)
}

size_t lrx_scan_bwd_workspace_bytes(int dtype, int64_t L, int64_t N) {
    if (L < 1 || N < 1) return 256;
    LRX_DISPATCH_SZ(dtype, ws_bytes, L, N, true)
}

int lrx_scan_fwd(int dtype, int a_per_step, const void* a, const void* b, const void* x0, void* out, int64_t L,
                 int64_t N, void* workspace, size_t workspace_bytes, void* stream) {
    LRX_REQUIRE(L >= 1, LRX_ERR_SHAPE, "length must be >= 1, got %lld", (long long)L);
    LRX_REQUIRE(N >= 1, LRX_ERR_SHAPE, "lane count must be >= 1, got %lld", (long long)N);
    LRX_REQUIRE(a && b && out, LRX_ERR_VALUE, "null array argument");
    LRX_DISPATCH(dtype, fwd_t, a_per_step, a, b, x0, out, L, N, workspace, workspace_bytes, (cudaStream_t)stream)
}

int lrx_scan_bwd(int dtype, int a_per_step, const void* a, const void* x, const void* x0, const void* gx, void* gb,
                 void* ga, void* gx0, int64_t L, int64_t N, void* workspace, size_t workspace_bytes, void* stream) {
    LRX_REQUIRE(L >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents L=%lld N=%lld", (long long)L, (long long)N);
    LRX_REQUIRE(a && gx && gb, LRX_ERR_VALUE, "null array argument");
    LRX_REQUIRE(!ga || x, LRX_ERR_VALUE, "grad_a needs the forward states x");
    LRX_DISPATCH(dtype, bwd_t, a_per_step, a, x, x0, gx, gb, ga, gx0, L, N, workspace, workspace_bytes,
                 (cudaStream_t)stream)
}

size_t lrx_reduce_rows_ws_bytes(int dtype, int64_t R, int64_t N) {
    if (R < 1 || N < 1) return 0;
    LRX_DISPATCH_SZ(dtype, reduce_ws, R, N)
}

int lrx_reduce_rows_ws(int dtype, const void* in, const void* in2, void* out, int64_t R, int64_t N, void* ws,
                       size_t ws_bytes, void* stream) {
    LRX_REQUIRE(R >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents R=%lld N=%lld", (long long)R, (long long)N);
    cudaStream_t st = (cudaStream_t)stream;
    switch (dtype) {
        case LRX_F32: return reduce_rows2<float>((const float*)in, (const float*)in2, (float*)out, R, N, ws, ws_bytes, st);
        case LRX_F64:
            return reduce_rows2<double>((const double*)in, (const double*)in2, (double*)out, R, N, ws, ws_bytes, st);
        case LRX_C64:
            return reduce_rows2<cplx<float>>((const cplx<float>*)in, (const cplx<float>*)in2, (cplx<float>*)out, R, N,
                                             ws, ws_bytes, st);
        case LRX_C128:
            return reduce_rows2<cplx<double>>((const cplx<double>*)in, (const cplx<double>*)in2, (cplx<double>*)out,
                                              R, N, ws, ws_bytes, st);
    }
    set_error("unsupported dtype %d", dtype);
    return LRX_ERR_VALUE;
}

int lrx_reduce_rows(int dtype, const void* in, void* out, int64_t R, int64_t N, void* stream) {
    LRX_REQUIRE(R >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents R=%lld N=%lld", (long long)R, (long long)N);
    cudaStream_t st = (cudaStream_t)stream;
    switch (dtype) {
        case LRX_F32: reduce_rows_launch<float>((const float*)in, (float*)out, R, N, st); break;
        case LRX_F64: reduce_rows_launch<double>((const double*)in, (double*)out, R, N, st); break;
        case LRX_C64: reduce_rows_launch<cplx<float>>((const cplx<float>*)in, (cplx<float>*)out, R, N, st); break;
        case LRX_C128: reduce_rows_launch<cplx<double>>((const cplx<double>*)in, (cplx<double>*)out, R, N, st); break;
        default: set_error("unsupported dtype %d", dtype); return LRX_ERR_VALUE;
    }
    return launched("lrx_reduce_rows");
}

}  // extern "C"
