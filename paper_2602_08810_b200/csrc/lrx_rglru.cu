// RG-LRU (Griffin) gated recurrence, fused forward / backward.
//
// Reference: pkg/src/linrec/layers.py RGLRU (1171-1336): _log_a 1208-1210,
// _gates 1212-1218, _forward_tape 1239-1250, _backward 1252-1291.
//
//   r = sigmoid(qr + b_r), i = sigmoid(qi + b_i)      qr = u W_r^T, qi = u W_i^T
//   log a_k = 8 r_k log sigmoid(lambda),  a_k = exp(log a_k)
//   s_k = sqrt(-expm1(2 log a_k)),  x_k = a_k x_{k-1} + s_k i_k u_k,  y = x
//
// Layout [B, L, W] (channel-contiguous, as the layer's u); lane = (b, w).
// Gates and discretisation are computed in the load path: the forward reads
// u, qr, qi once and writes y once; the backward reads u, qr, qi, gy and the
// saved output y (= the state, so x_{k-1} needs no recompute) once and writes
// gu, gqr, gqi once.
//
// Three kernel families, chosen per call (LRX_RGLRU_MODE overrides):
//  * tma      one CTA per LW-lane column block walks the whole sequence; time
//             tiles of PF steps x LW channels arrive by TMA into an S-stage
//             shared-memory ring (full/empty mbarriers), threads read their
//             channel column.  Registers hold no in-flight data, so every
//             lane of the problem is resident in one wave.  LW in {128,64,32}
//             keeps >= 4 CTAs per SM when lanes are scarce (8-GPU sharding).
//  * stream   same walk with a register prefetch (fallback when the rows are
//             not 16-byte aligned for TMA).
//  * lookback time chunks of T steps across CTAs chained by the anchored
//             look-back (lrx_common.cuh); the backward recomputes states from
//             per-chunk checkpoints (used for bf16 I/O, where y is rounded).
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "lrx_common.cuh"
#include "lrx_host.h"
#include "lrx_tma.cuh"

namespace lrx {
namespace rglru {

constexpr int kThreads = 128;
constexpr float kGate = 8.0f;  // GATE_POWER, layers.py:1177

// Checkpoint interval: the forward saves the state entering every T-step
// chunk (plus the final state); the backward re-anchors its reverse state
// reconstruction there, so no reconstruction runs deeper than T - 1 steps.
template <typename IO> struct Tile { static constexpr int T = 8; };
// Largest TMA time tile (rows per barrier wait).
template <typename IO> struct MaxPF { static constexpr int T = 16; };
template <> struct MaxPF<double> { static constexpr int T = 8; };

template <typename C>
struct Coef {
    C r, i, a, s, u;
};

template <typename C, typename IO>
__device__ __forceinline__ Coef<C> gates(IO uu, IO q_r, IO q_i, C la, C br, C bi) {
    using F = Fast<C>;
    Coef<C> k;
    k.u = cvt(uu);
    k.r = F::sigmoid(C(cvt(q_r)) + br);
    k.i = F::sigmoid(C(cvt(q_i)) + bi);
    const C loga = (C(kGate) * k.r) * la;
    k.a = F::exp(loga);
    k.s = F::sqrt(-F::expm1_known(C(2) * loga, k.a * k.a));  // e^{2 log a} = a^2
    return k;
}

// Compensated (Kahan) accumulator: the per-lane parameter-gradient sums run
// over up to 2^20 steps in fp32.
template <typename C>
struct Kahan {
    C s = 0, c = 0;
    __device__ __forceinline__ void add(C v) {
        const C y = v - c;
        const C t = s + y;
        c = (t - s) - y;
        s = t;
    }
};

template <typename C>
struct BwdOut {
    C gu, gqr, gqi, la_term;
};
template <typename C>
__device__ __forceinline__ BwdOut<C> bwd_step(const Coef<C>& q, C g, C xprev, C la) {
    const C gak = g * xprev;
    const C gs = (q.i * q.u) * g;
    const C gloga = q.a * gak - Fast<C>::div(q.a * q.a, q.s) * gs;
    BwdOut<C> o;
    o.gqr = (q.r * (C(1) - q.r)) * ((C(kGate) * la) * gloga);
    o.gqi = (q.i * (C(1) - q.i)) * ((q.s * q.u) * g);
    o.gu = (q.s * q.i) * g;
    o.la_term = (C(kGate) * q.r) * gloga;
    return o;
}

// ====================================================================== TMA
template <typename IO>
struct Ring {
    uint64_t* full;
    uint64_t* empty;
    IO* data;  // [S][NARR][PF][LW]
};

template <typename IO>
__device__ __forceinline__ Ring<IO> ring(unsigned char* smem, int S) {
    Ring<IO> r;
    r.full = reinterpret_cast<uint64_t*>(smem);
    r.empty = r.full + S;
    r.data = reinterpret_cast<IO*>(smem + 128 * ((2 * S * 8 + 127) / 128));
    return r;
}

// Time segments.  When B*W lanes are too few to keep ~24 warps per SM (the
// per-rank batch of an 8-GPU job), the sequence is cut into n_seg segments
// of seg_len steps (gridDim.y).  A first pass (AGG) reduces each segment to
// its transfer pair with a zero carry in: A_s = sum log a_k, X_s = the state
// the segment produces from x = 0.  The main pass folds the pairs of the
// segments before it in fixed order (x = exp(A_r) x + X_r) and streams its
// own segment.  The kernel is latency-bound at few warps per SM, so the extra
// read pass costs less than the parallelism it buys.
template <typename IO, typename C, int LW, int PF, bool AGG>
__global__ void __launch_bounds__(LW, PF == 4 && LW >= 64 ? 1152 / LW : 1) fwd_tma_kernel(const __grid_constant__ CUtensorMap mu,
                                                     const __grid_constant__ CUtensorMap mr,
                                                     const __grid_constant__ CUtensorMap mi, const C* __restrict__ lam,
                                                     const C* __restrict__ b_r, const C* __restrict__ b_i,
                                                     IO* __restrict__ y, C* __restrict__ ckpt, C* __restrict__ seg_a,
                                                     C* __restrict__ seg_x, int64_t L, int64_t W, int n_wblk, int Bn,
                                                     int S, int seg_len, int seg0) {
    constexpr int CK = Tile<IO>::T;
    constexpr int NW = LW / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    auto R = ring<IO>(smem, S);
    const int tid = threadIdx.x;
    const int b = blockIdx.x / n_wblk;
    const int w0 = (blockIdx.x % n_wblk) * LW;
    const int64_t w = w0 + tid;
    const bool valid = w < W;
    const int seg = seg0 + blockIdx.y;
    const int64_t t_beg = (int64_t)seg * seg_len;
    const int64_t t_end = min(L, t_beg + seg_len);
    const int j_beg = (int)(t_beg / PF);
    const int n_tiles = (int)((t_end + PF - 1) / PF) - j_beg;
    const int row0 = b * (int)L;
    constexpr uint32_t kStageBytes = 3u * PF * LW * sizeof(IO);
    if (tid == 0) {
        tma::prefetch_map(&mu);
        tma::prefetch_map(&mr);
        tma::prefetch_map(&mi);
        for (int s = 0; s < S; ++s) {
            tma::mbar_init(&R.full[s], 1);
            tma::mbar_init(&R.empty[s], NW);
        }
        tma::fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int j) {
        const int s = j % S;
        IO* dst = R.data + (size_t)s * 3 * PF * LW;
        const int r = row0 + (j_beg + j) * PF;
        tma::mbar_arrive_expect_tx(&R.full[s], kStageBytes);
        tma::load_2d(dst, &mu, w0, r, &R.full[s]);
        tma::load_2d(dst + PF * LW, &mr, w0, r, &R.full[s]);
        tma::load_2d(dst + 2 * PF * LW, &mi, w0, r, &R.full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < S && j < n_tiles; ++j) issue(j);

    C la = 0, br = 0, bi = 0;
    if (valid) {
        la = -Math<C>::softplus(-lam[w]);
        br = b_r[w];
        bi = b_i[w];
    }
    const int64_t BW = (int64_t)Bn * W;
    const int64_t lane = (int64_t)b * W + w;
    C x = 0, sla = 0;
    if (!AGG && valid)
        for (int r = 0; r < seg; ++r) x = Fast<C>::exp(seg_a[r * BW + lane]) * x + seg_x[r * BW + lane];
    IO* py = y + ((int64_t)row0 + t_beg) * W + w;
    static_assert(CK % PF == 0 || PF % CK == 0, "tile and checkpoint interval must nest");
    for (int j = 0; j < n_tiles; ++j) {
        const int s = j % S;
        const uint32_t ph = (j / S) & 1;
        tma::mbar_wait(&R.full[s], ph);
        const IO* src = R.data + (size_t)s * 3 * PF * LW + tid;
        IO cu[PF], cr[PF], ci[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            cu[k] = src[k * LW];
            cr[k] = src[(PF + k) * LW];
            ci[k] = src[(2 * PF + k) * LW];
        }
        __syncwarp();
        if ((tid & 31) == 0) tma::mbar_arrive(&R.empty[s]);
        if (tid == 0 && j + S < n_tiles) {
            tma::mbar_wait(&R.empty[s], ph);
            issue(j + S);
        }
        const int64_t t0 = (int64_t)(j_beg + j) * PF;
        const int nk = (int)min((int64_t)PF, t_end - t0);
        const C xin = x;
        // the whole-tile case runs without per-step guards; stores are
        // predicated once per tile
        C tla = 0, xs[PF];
        auto step = [&](int k) {
            const Coef<C> q = gates<C>(cu[k], cr[k], ci[k], la, br, bi);
            x = q.a * x + (q.s * q.i) * q.u;
            xs[k] = x;
            if (AGG) tla += (C(kGate) * q.r) * la;
        };
        if (nk == PF) {
#pragma unroll
            for (int k = 0; k < PF; ++k) step(k);
        } else {
#pragma unroll
            for (int k = 0; k < PF; ++k)
                if (k < nk) step(k);
        }
        if (AGG) {
            sla += tla;
        } else {
            if (ckpt && valid) {  // the state entering each checkpoint chunk of the tile
#pragma unroll
                for (int k = 0; k < PF; k += (PF < CK ? PF : CK))
                    if (k < nk && ((t0 + k) % CK) == 0) __stcs(ckpt + ((t0 + k) / CK) * BW + lane, k ? xs[k - 1] : xin);
            }
            if (valid) {
                if (nk == PF) {
#pragma unroll
                    for (int k = 0; k < PF; ++k) st_io(py + k * W, xs[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < PF; ++k)
                        if (k < nk) st_io(py + k * W, xs[k]);
                }
            }
            py += PF * W;
        }
    }
    if (AGG && valid) {
        seg_a[seg * BW + lane] = sla;
        seg_x[seg * BW + lane] = x;
    }
    if (!AGG && ckpt && valid && t_end == L) __stcs(ckpt + ((L + CK - 1) / CK) * BW + lane, x);  // final state
}

// Reverse streaming pass; the y tile of a time tile is loaded one row early
// so its row k holds x_{t-1}.  Segmented like the forward: the AGG pass
// streams qr and gy only (A_s = sum log a_k, H_s = the carry the segment
// hands to its left neighbour from h = 0); the main pass folds the segments
// to its right (h = exp(A_r) h + H_r, r = n_seg-1 .. seg+1) and writes
// per-(segment, lane) parameter-gradient partials.
template <typename IO, typename C, int LW, int PF, bool AGG>
__global__ void __launch_bounds__(LW, PF == 4 && LW >= 64 ? 1152 / LW : 1) bwd_tma_kernel(
    const __grid_constant__ CUtensorMap mu, const __grid_constant__ CUtensorMap mr,
    const __grid_constant__ CUtensorMap mi, const __grid_constant__ CUtensorMap mg,
    const __grid_constant__ CUtensorMap my, const C* __restrict__ lam, const C* __restrict__ b_r,
    const C* __restrict__ b_i, IO* __restrict__ gu, IO* __restrict__ gqr, IO* __restrict__ gqi,
    C* __restrict__ gla_part, C* __restrict__ gbr_part, C* __restrict__ gbi_part, C* __restrict__ seg_a,
    C* __restrict__ seg_h, int64_t L, int64_t W, int n_wblk, int Bn, int S, int seg_len, int seg0, int n_seg) {
    constexpr int NW = LW / 32;
    constexpr int NA = AGG ? 2 : 5;  // staged arrays: AGG {qr, gy}; main {u, qr, qi, gy, y}
    extern __shared__ __align__(128) unsigned char smem[];
    auto R = ring<IO>(smem, S);
    const int tid = threadIdx.x;
    const int b = blockIdx.x / n_wblk;
    const int w0 = (blockIdx.x % n_wblk) * LW;
    const int64_t w = w0 + tid;
    const bool valid = w < W;
    const int seg = seg0 + blockIdx.y;
    const int64_t t_beg = (int64_t)seg * seg_len;
    const int64_t t_end = min(L, t_beg + seg_len);
    const int j_beg = (int)(t_beg / PF);
    const int n_tiles = (int)((t_end + PF - 1) / PF) - j_beg;
    const int row0 = b * (int)L;
    constexpr uint32_t kStageBytes = (uint32_t)NA * PF * LW * sizeof(IO);
    if (tid == 0) {
        if (!AGG) tma::prefetch_map(&mu);
        tma::prefetch_map(&mr);
        if (!AGG) tma::prefetch_map(&mi);
        tma::prefetch_map(&mg);
        if (!AGG) tma::prefetch_map(&my);
        for (int s = 0; s < S; ++s) {
            tma::mbar_init(&R.full[s], 1);
            tma::mbar_init(&R.empty[s], NW);
        }
        tma::fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int j) {  // j-th tile in reverse order
        const int tt = j_beg + n_tiles - 1 - j;
        const int s = j % S;
        IO* dst = R.data + (size_t)s * NA * PF * LW;
        const int r = row0 + tt * PF;
        tma::mbar_arrive_expect_tx(&R.full[s], kStageBytes);
        if (AGG) {
            tma::load_2d(dst, &mr, w0, r, &R.full[s]);
            tma::load_2d(dst + PF * LW, &mg, w0, r, &R.full[s]);
        } else {
            tma::load_2d(dst, &mu, w0, r, &R.full[s]);
            tma::load_2d(dst + PF * LW, &mr, w0, r, &R.full[s]);
            tma::load_2d(dst + 2 * PF * LW, &mi, w0, r, &R.full[s]);
            tma::load_2d(dst + 3 * PF * LW, &mg, w0, r, &R.full[s]);
            tma::load_2d(dst + 4 * PF * LW, &my, w0, r - 1, &R.full[s]);  // rows t-1
        }
    };
    if (tid == 0)
        for (int j = 0; j < S && j < n_tiles; ++j) issue(j);

    C la = 0, br = 0, bi = 0;
    if (valid) {
        la = -Math<C>::softplus(-lam[w]);
        br = b_r[w];
        bi = b_i[w];
    }
    const int64_t BW = (int64_t)Bn * W;
    const int64_t lane = (int64_t)b * W + w;
    C h = 0, asum = 0;
    if (!AGG && valid)
        for (int r = n_seg - 1; r > seg; --r) h = Fast<C>::exp(seg_a[r * BW + lane]) * h + seg_h[r * BW + lane];
    Kahan<C> sla, sbr, sbi;
    IO *pgu = gu + (int64_t)row0 * W + w, *pgr = gqr + (int64_t)row0 * W + w, *pgi = gqi + (int64_t)row0 * W + w;
    for (int j = 0; j < n_tiles; ++j) {
        const int s = j % S;
        const uint32_t ph = (j / S) & 1;
        const int tt = j_beg + n_tiles - 1 - j;
        tma::mbar_wait(&R.full[s], ph);
        const IO* src = R.data + (size_t)s * NA * PF * LW + tid;
        IO cu[PF], cr[PF], ci[PF], cg[PF], cy[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            if (AGG) {
                cr[k] = src[k * LW];
                cg[k] = src[(PF + k) * LW];
            } else {
                cu[k] = src[k * LW];
                cr[k] = src[(PF + k) * LW];
                ci[k] = src[(2 * PF + k) * LW];
                cg[k] = src[(3 * PF + k) * LW];
                cy[k] = src[(4 * PF + k) * LW];
            }
        }
        __syncwarp();
        if ((tid & 31) == 0) tma::mbar_arrive(&R.empty[s]);
        if (tid == 0 && j + S < n_tiles) {
            tma::mbar_wait(&R.empty[s], ph);
            issue(j + S);
        }
        const int64_t t0 = (int64_t)tt * PF;
        const int nk = (int)min((int64_t)PF, t_end - t0);
        if (AGG) {
            C tla = 0;
#pragma unroll
            for (int k = PF - 1; k >= 0; --k) {
                if (k < nk) {
                    const C r = Fast<C>::sigmoid(C(cvt(cr[k])) + br);
                    const C loga = (C(kGate) * r) * la;
                    h = Fast<C>::exp(loga) * (C(cvt(cg[k])) + h);
                    tla += loga;
                }
            }
            asum += tla;
            continue;
        }
        if (tt == 0) cy[0] = IO(0);  // x_{-1} = 0
        C tla = 0, tbr = 0, tbi = 0;
        const int64_t o0 = t0 * W;
        IO *qu = pgu + o0, *qr = pgr + o0, *qi = pgi + o0;
        auto step = [&](int k) {
            const Coef<C> q = gates<C>(cu[k], cr[k], ci[k], la, br, bi);
            const C g = C(cvt(cg[k])) + h;
            h = q.a * g;
            const BwdOut<C> o = bwd_step<C>(q, g, C(cvt(cy[k])), la);
            if (valid) {  // predicated stores
                st_io(qu + k * W, o.gu);
                st_io(qr + k * W, o.gqr);
                st_io(qi + k * W, o.gqi);
            }
            tla += o.la_term;
            tbr += o.gqr;
            tbi += o.gqi;
        };
        if (nk == PF) {  // whole tile: no per-step guards
#pragma unroll
            for (int k = PF - 1; k >= 0; --k) step(k);
        } else {
#pragma unroll
            for (int k = PF - 1; k >= 0; --k)
                if (k < nk) step(k);
        }
        sla.add(tla);
        sbr.add(tbr);
        sbi.add(tbi);
    }
    if (!valid) return;
    if (AGG) {
        seg_a[seg * BW + lane] = asum;
        seg_h[seg * BW + lane] = h;
    } else {
        const int64_t p = seg * BW + lane;
        gla_part[p] = sla.s;
        gbr_part[p] = sbr.s;
        gbi_part[p] = sbi.s;
    }
}

// Backward without the y stream and with one gate evaluation per element:
// the reverse walk reconstructs the state it needs, x_{t-1} = (x_t - b_t) / a_t,
// from the gates it evaluates anyway for the pullback.  The division expands
// rounding errors by 1/a per step, so the walk re-anchors on the forward's
// checkpoints: x_t at the end of every T-step chunk and x_{t-1} at its start
// are the saved states (exact), leaving at most T - 1 = 7 reconstructed steps
// (measured on C4-distributed gates: 2.5e-6 max-normalised state error at
// T = 8 against 1.2e-4 at T = 16).  Streams u, qr, qi, gy in and gu, gqr, gqi
// out -- the 7 algorithmic arrays -- plus 1/T of a state array of anchors.
// Segmented like bwd_tma_kernel (its AGG pass supplies the segment maps).
template <typename IO, typename C, int LW, int PF>
__global__ void __launch_bounds__(LW, PF == 4 && LW >= 64 ? 1152 / LW : 1) bwd_rev_kernel(
    const __grid_constant__ CUtensorMap mu, const __grid_constant__ CUtensorMap mr,
    const __grid_constant__ CUtensorMap mi, const __grid_constant__ CUtensorMap mg, const C* __restrict__ lam,
    const C* __restrict__ b_r, const C* __restrict__ b_i, const C* __restrict__ ckpt, IO* __restrict__ gu,
    IO* __restrict__ gqr, IO* __restrict__ gqi, C* __restrict__ gla_part, C* __restrict__ gbr_part,
    C* __restrict__ gbi_part, const C* __restrict__ seg_a, const C* __restrict__ seg_h, int64_t L, int64_t W,
    int n_wblk, int Bn, int S, int seg_len, int n_seg) {
    constexpr int NW = LW / 32;
    constexpr int NA = 4;  // u, qr, qi, gy
    constexpr int CK = Tile<IO>::T;
    static_assert(CK % PF == 0 || PF % CK == 0, "tile and checkpoint interval must nest");
    extern __shared__ __align__(128) unsigned char smem[];
    auto R = ring<IO>(smem, S);
    const int tid = threadIdx.x;
    const int b = blockIdx.x / n_wblk;
    const int w0 = (blockIdx.x % n_wblk) * LW;
    const int64_t w = w0 + tid;
    const bool valid = w < W;
    const int seg = blockIdx.y;
    const int64_t t_beg = (int64_t)seg * seg_len;
    const int64_t t_end = min(L, t_beg + seg_len);
    const int j_beg = (int)(t_beg / PF);
    const int n_tiles = (int)((t_end + PF - 1) / PF) - j_beg;
    const int row0 = b * (int)L;
    constexpr uint32_t kStageBytes = (uint32_t)NA * PF * LW * sizeof(IO);
    if (tid == 0) {
        tma::prefetch_map(&mu);
        tma::prefetch_map(&mr);
        tma::prefetch_map(&mi);
        tma::prefetch_map(&mg);
        for (int s = 0; s < S; ++s) {
            tma::mbar_init(&R.full[s], 1);
            tma::mbar_init(&R.empty[s], NW);
        }
        tma::fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int j) {  // j-th tile in reverse order
        const int tt = j_beg + n_tiles - 1 - j;
        const int s = j % S;
        IO* dst = R.data + (size_t)s * NA * PF * LW;
        const int r = row0 + tt * PF;
        tma::mbar_arrive_expect_tx(&R.full[s], kStageBytes);
        tma::load_2d(dst, &mu, w0, r, &R.full[s]);
        tma::load_2d(dst + PF * LW, &mr, w0, r, &R.full[s]);
        tma::load_2d(dst + 2 * PF * LW, &mi, w0, r, &R.full[s]);
        tma::load_2d(dst + 3 * PF * LW, &mg, w0, r, &R.full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < S && j < n_tiles; ++j) issue(j);

    C la = 0, br = 0, bi = 0;
    if (valid) {
        la = -Math<C>::softplus(-lam[w]);
        br = b_r[w];
        bi = b_i[w];
    }
    const int64_t BW = (int64_t)Bn * W;
    const int64_t lane = (int64_t)b * W + (valid ? w : 0);
    C h = 0;
    if (valid)
        for (int r = n_seg - 1; r > seg; --r) h = Fast<C>::exp(seg_a[r * BW + lane]) * h + seg_h[r * BW + lane];
    // x = the state after the step being walked; anc = the saved state entering
    // the next chunk start below it (prefetched one chunk ahead)
    const C* pck = ckpt + lane;
    C x = __ldcg(pck + ((t_end + CK - 1) / CK) * BW);
    int64_t c_next = (t_end - 1) / CK;
    C anc = __ldcg(pck + c_next * BW);
    Kahan<C> sla, sbr, sbi;
    IO *pgu = gu + (int64_t)row0 * W + w, *pgr = gqr + (int64_t)row0 * W + w, *pgi = gqi + (int64_t)row0 * W + w;
    for (int j = 0; j < n_tiles; ++j) {
        const int s = j % S;
        const uint32_t ph = (j / S) & 1;
        const int tt = j_beg + n_tiles - 1 - j;
        tma::mbar_wait(&R.full[s], ph);
        const IO* src = R.data + (size_t)s * NA * PF * LW + tid;
        IO cu[PF], cr[PF], ci[PF], cg[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            cu[k] = src[k * LW];
            cr[k] = src[(PF + k) * LW];
            ci[k] = src[(2 * PF + k) * LW];
            cg[k] = src[(3 * PF + k) * LW];
        }
        __syncwarp();
        if ((tid & 31) == 0) tma::mbar_arrive(&R.empty[s]);
        if (tid == 0 && j + S < n_tiles) {
            tma::mbar_wait(&R.empty[s], ph);
            issue(j + S);
        }
        const int64_t t0 = (int64_t)tt * PF;
        const int nk = (int)min((int64_t)PF, t_end - t0);
        C tla = 0, tbr = 0, tbi = 0;
        const int64_t o0 = t0 * W;
        IO *qu = pgu + o0, *qr = pgr + o0, *qi = pgi + o0;
        auto step = [&](int k) {
            const Coef<C> q = gates<C>(cu[k], cr[k], ci[k], la, br, bi);
            const C g = C(cvt(cg[k])) + h;
            h = q.a * g;
            C xprev;
            if (((t0 + k) % CK) == 0) {  // chunk start: the saved state
                xprev = anc;
                c_next -= 1;
                anc = (c_next >= 0 && valid) ? __ldcg(pck + c_next * BW) : C(0);
            } else {
                xprev = (x - (q.s * q.i) * q.u) * Fast<C>::rcp(q.a);
            }
            const BwdOut<C> o = bwd_step<C>(q, g, xprev, la);
            x = xprev;
            if (valid) {
                st_io(qu + k * W, o.gu);
                st_io(qr + k * W, o.gqr);
                st_io(qi + k * W, o.gqi);
            }
            tla += o.la_term;
            tbr += o.gqr;
            tbi += o.gqi;
        };
        if (nk == PF) {
#pragma unroll
            for (int k = PF - 1; k >= 0; --k) step(k);
        } else {
#pragma unroll
            for (int k = PF - 1; k >= 0; --k)
                if (k < nk) step(k);
        }
        sla.add(tla);
        sbr.add(tbr);
        sbi.add(tbi);
    }
    if (!valid) return;
    const int64_t p = seg * BW + lane;
    gla_part[p] = sla.s;
    gbr_part[p] = sbr.s;
    gbi_part[p] = sbi.s;
}

// ---------------------------------------------------------------- lane pairs
// fp32 compute with two channels per thread: every elementwise operation of
// the gates and the pullback runs on packed fp32x2 (FFMA2 / FMUL2 / FADD2, one
// instruction for both lanes, IEEE rounding per lane) and the per-step
// overhead (shared loads, global stores, addressing, barrier waits) is paid
// once per pair.  The scalar walk issued ~130 instructions per element and
// was issue-bound below the HBM ceiling (ncu, C4 bwd: issue 66%, 5.1 TB/s).
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 ex2_2(float2 x) { return make_float2(Fast<float>::ex2(x.x), Fast<float>::ex2(x.y)); }
__device__ __forceinline__ float2 rcp2(float2 x) { return make_float2(Fast<float>::rcp(x.x), Fast<float>::rcp(x.y)); }
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ float2 ld2(const __nv_bfloat16* p) {
    const uint32_t v = *reinterpret_cast<const uint32_t*>(p);
    return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));
}
__device__ __forceinline__ void st2(float* p, float2 v) { __stcs(reinterpret_cast<float2*>(p), v); }
__device__ __forceinline__ void st2(__nv_bfloat16* p, float2 v) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v.x, v.y);
}

struct Coef2 {
    float2 r, i, a, s, rs, u;  // rs = 1 / s
};
// gates() on a lane pair; s and 1/s from one rsqrt of -expm1(2 log a) = 1 - a^2
__device__ __forceinline__ Coef2 gates2(float2 u, float2 qr, float2 qi, float2 la, float2 br, float2 bi) {
    constexpr float kL2e = 1.4426950408889634f;
    Coef2 k;
    k.u = u;
    k.r = rcp2(add2(f2(1.f), ex2_2(mul2(add2(qr, br), f2(-kL2e)))));
    k.i = rcp2(add2(f2(1.f), ex2_2(mul2(add2(qi, bi), f2(-kL2e)))));
    const float2 loga = mul2(mul2(f2(kGate), k.r), la);
    k.a = ex2_2(mul2(loga, f2(kL2e)));
    // expm1(2 loga): degree-6 Taylor at h = loga (half the argument), doubled
    const float2 h = loga;
    float2 p = fma2(f2(1.f / 720.f), h, f2(1.f / 120.f));
    p = fma2(p, h, f2(1.f / 24.f));
    p = fma2(p, h, f2(1.f / 6.f));
    p = fma2(p, h, f2(0.5f));
    p = fma2(p, h, f2(1.f));
    p = mul2(p, h);
    const float2 small = mul2(p, add2(p, f2(2.f)));
    const float2 big = fma2(k.a, k.a, f2(-1.f));
    const float2 m = make_float2(-(fabsf(2.f * loga.x) < 0.7f ? small.x : big.x),
                                 -(fabsf(2.f * loga.y) < 0.7f ? small.y : big.y));  // 1 - a^2 > 0
    k.rs = make_float2(rsqrt_approx(m.x), rsqrt_approx(m.y));
    k.s = mul2(m, k.rs);
    return k;
}

template <typename IO, int LW, int PF>
__global__ void __launch_bounds__(LW / 2, PF <= 4 ? 1152 / LW : 512 / LW) bwd_rev2_kernel(
    const __grid_constant__ CUtensorMap mu, const __grid_constant__ CUtensorMap mr,
    const __grid_constant__ CUtensorMap mi, const __grid_constant__ CUtensorMap mg, const float* __restrict__ lam,
    const float* __restrict__ b_r, const float* __restrict__ b_i, const float* __restrict__ ckpt, IO* __restrict__ gu,
    IO* __restrict__ gqr, IO* __restrict__ gqi, float* __restrict__ gla_part, float* __restrict__ gbr_part,
    float* __restrict__ gbi_part, const float* __restrict__ seg_a, const float* __restrict__ seg_h, int64_t L,
    int64_t W, int n_wblk, int Bn, int S, int seg_len, int n_seg) {
    constexpr int NT = LW / 2;
    constexpr int NW = NT / 32;
    static_assert(NW >= 1, "lane pairs need LW >= 64");
    constexpr int NA = 4;  // u, qr, qi, gy
    constexpr int CK = Tile<IO>::T;
    static_assert(CK % PF == 0 || PF % CK == 0, "tile and checkpoint interval must nest");
    extern __shared__ __align__(128) unsigned char smem[];
    auto R = ring<IO>(smem, S);
    const int tid = threadIdx.x;
    const int b = blockIdx.x / n_wblk;
    const int w0 = (blockIdx.x % n_wblk) * LW;
    const int64_t w = w0 + 2 * tid;  // lanes w, w + 1 (W is even: 16-byte rows)
    const bool valid = w < W;
    const int seg = blockIdx.y;
    const int64_t t_beg = (int64_t)seg * seg_len;
    const int64_t t_end = min(L, t_beg + seg_len);
    const int j_beg = (int)(t_beg / PF);
    const int n_tiles = (int)((t_end + PF - 1) / PF) - j_beg;
    const int row0 = b * (int)L;
    constexpr uint32_t kStageBytes = (uint32_t)NA * PF * LW * sizeof(IO);
    if (tid == 0) {
        tma::prefetch_map(&mu);
        tma::prefetch_map(&mr);
        tma::prefetch_map(&mi);
        tma::prefetch_map(&mg);
        for (int s = 0; s < S; ++s) {
            tma::mbar_init(&R.full[s], 1);
            tma::mbar_init(&R.empty[s], NW);
        }
        tma::fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int j, int s) {  // j-th tile in reverse order, into stage s
        const int tt = j_beg + n_tiles - 1 - j;
        IO* dst = R.data + (size_t)s * NA * PF * LW;
        const int r = row0 + tt * PF;
        tma::mbar_arrive_expect_tx(&R.full[s], kStageBytes);
        tma::load_2d(dst, &mu, w0, r, &R.full[s]);
        tma::load_2d(dst + PF * LW, &mr, w0, r, &R.full[s]);
        tma::load_2d(dst + 2 * PF * LW, &mi, w0, r, &R.full[s]);
        tma::load_2d(dst + 3 * PF * LW, &mg, w0, r, &R.full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < S && j < n_tiles; ++j) issue(j, j);

    float2 la = f2(0.f), br = f2(0.f), bi = f2(0.f);
    if (valid) {
        la = make_float2(-Math<float>::softplus(-lam[w]), -Math<float>::softplus(-lam[w + 1]));
        br = ld2(b_r + w);
        bi = ld2(b_i + w);
    }
    const float2 la8 = mul2(f2(kGate), la);
    const int64_t BW = (int64_t)Bn * W;
    const int64_t lane = (int64_t)b * W + (valid ? w : 0);
    float2 h = f2(0.f);
    if (valid)
        for (int r = n_seg - 1; r > seg; --r)
            h = fma2(ex2_2(mul2(ld2(seg_a + r * BW + lane), f2(1.4426950408889634f))), h, ld2(seg_h + r * BW + lane));
    // x = the state after the step being walked; anc = the saved state entering
    // the next chunk start below it (prefetched one chunk ahead)
    const float* pck = ckpt + lane;
    float2 x = valid ? __ldcg(reinterpret_cast<const float2*>(pck + ((t_end + CK - 1) / CK) * BW)) : f2(0.f);
    int64_t c_next = (t_end - 1) / CK;
    float2 anc = valid ? __ldcg(reinterpret_cast<const float2*>(pck + c_next * BW)) : f2(0.f);
    Kahan<float> sla[2], sbr[2], sbi[2];
    const int64_t tile_stride = (int64_t)PF * W;
    const int64_t o_last = ((int64_t)row0 + (int64_t)(j_beg + n_tiles - 1) * PF) * W + w;
    IO *qu = gu + o_last, *qr = gqr + o_last, *qi = gqi + o_last;
    int s = 0;
    uint32_t ph = 0;
    for (int j = 0; j < n_tiles; ++j) {
        const int tt = j_beg + n_tiles - 1 - j;
        tma::mbar_wait(&R.full[s], ph);
        const IO* src = R.data + (size_t)s * NA * PF * LW + 2 * tid;
        float2 cu[PF], cr[PF], ci[PF], cg[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            cu[k] = ld2(src + k * LW);
            cr[k] = ld2(src + (PF + k) * LW);
            ci[k] = ld2(src + (2 * PF + k) * LW);
            cg[k] = ld2(src + (3 * PF + k) * LW);
        }
        __syncwarp();
        if ((tid & 31) == 0) tma::mbar_arrive(&R.empty[s]);
        if (tid == 0 && j + S < n_tiles) {
            tma::mbar_wait(&R.empty[s], ph);
            issue(j + S, s);
        }
        if (++s == S) {
            s = 0;
            ph ^= 1;
        }
        const int64_t t0 = (int64_t)tt * PF;
        const int nk = (int)min((int64_t)PF, t_end - t0);
        float2 tla = f2(0.f), tbr = f2(0.f), tbi = f2(0.f);
        auto step = [&](int k) {
            const Coef2 q = gates2(cu[k], cr[k], ci[k], la, br, bi);
            const float2 g = add2(cg[k], h);
            h = mul2(q.a, g);
            const float2 si = mul2(q.s, q.i);
            float2 xprev;
            if (((t0 + k) % CK) == 0) {  // chunk start: the saved state
                xprev = anc;
                c_next -= 1;
                anc = (c_next >= 0 && valid) ? __ldcg(reinterpret_cast<const float2*>(pck + c_next * BW)) : f2(0.f);
            } else {
                xprev = mul2(fma2(f2(-1.f), mul2(si, q.u), x), rcp2(q.a));
            }
            // pullback (bwd_step): gloga = a g x_{k-1} - (a^2 / s) i u g
            const float2 gs = mul2(mul2(q.i, q.u), g);
            const float2 gloga = fma2(mul2(q.a, q.a), mul2(f2(-1.f), mul2(q.rs, gs)), mul2(q.a, mul2(g, xprev)));
            const float2 gqr_v = mul2(mul2(q.r, sub2(f2(1.f), q.r)), mul2(la8, gloga));
            const float2 gqi_v = mul2(mul2(q.i, sub2(f2(1.f), q.i)), mul2(mul2(q.s, q.u), g));
            const float2 gu_v = mul2(si, g);
            x = xprev;
            if (valid) {
                st2(qu + k * W, gu_v);
                st2(qr + k * W, gqr_v);
                st2(qi + k * W, gqi_v);
            }
            tla = fma2(mul2(f2(kGate), q.r), gloga, tla);
            tbr = add2(tbr, gqr_v);
            tbi = add2(tbi, gqi_v);
        };
        if (nk == PF) {
#pragma unroll
            for (int k = PF - 1; k >= 0; --k) step(k);
        } else {
#pragma unroll
            for (int k = PF - 1; k >= 0; --k)
                if (k < nk) step(k);
        }
        qu -= tile_stride;
        qr -= tile_stride;
        qi -= tile_stride;
        sla[0].add(tla.x);
        sla[1].add(tla.y);
        sbr[0].add(tbr.x);
        sbr[1].add(tbr.y);
        sbi[0].add(tbi.x);
        sbi[1].add(tbi.y);
    }
    if (!valid) return;
    const int64_t p = seg * BW + lane;
    *reinterpret_cast<float2*>(gla_part + p) = make_float2(sla[0].s, sla[1].s);
    *reinterpret_cast<float2*>(gbr_part + p) = make_float2(sbr[0].s, sbr[1].s);
    *reinterpret_cast<float2*>(gbi_part + p) = make_float2(sbi[0].s, sbi[1].s);
}

// Lane-pair forward (fp32 compute, LW >= 64): fwd_tma_kernel on packed fp32x2.
template <typename IO, int LW, int PF, bool AGG>
__global__ void __launch_bounds__(LW / 2, PF <= 4 ? 1152 / LW : 512 / LW) fwd2_kernel(
    const __grid_constant__ CUtensorMap mu, const __grid_constant__ CUtensorMap mr,
    const __grid_constant__ CUtensorMap mi, const float* __restrict__ lam, const float* __restrict__ b_r,
    const float* __restrict__ b_i, IO* __restrict__ y, float* __restrict__ ckpt, float* __restrict__ seg_a,
    float* __restrict__ seg_x, int64_t L, int64_t W, int n_wblk, int Bn, int S, int seg_len, int seg0) {
    constexpr int CK = Tile<IO>::T;
    constexpr int NT = LW / 2;
    constexpr int NW = NT / 32;
    static_assert(NW >= 1, "lane pairs need LW >= 64");
    static_assert(CK % PF == 0 || PF % CK == 0, "tile and checkpoint interval must nest");
    extern __shared__ __align__(128) unsigned char smem[];
    auto R = ring<IO>(smem, S);
    const int tid = threadIdx.x;
    const int b = blockIdx.x / n_wblk;
    const int w0 = (blockIdx.x % n_wblk) * LW;
    const int64_t w = w0 + 2 * tid;
    const bool valid = w < W;
    const int seg = seg0 + blockIdx.y;
    const int64_t t_beg = (int64_t)seg * seg_len;
    const int64_t t_end = min(L, t_beg + seg_len);
    const int j_beg = (int)(t_beg / PF);
    const int n_tiles = (int)((t_end + PF - 1) / PF) - j_beg;
    const int row0 = b * (int)L;
    constexpr uint32_t kStageBytes = 3u * PF * LW * sizeof(IO);
    if (tid == 0) {
        tma::prefetch_map(&mu);
        tma::prefetch_map(&mr);
        tma::prefetch_map(&mi);
        for (int s = 0; s < S; ++s) {
            tma::mbar_init(&R.full[s], 1);
            tma::mbar_init(&R.empty[s], NW);
        }
        tma::fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int j, int s) {
        IO* dst = R.data + (size_t)s * 3 * PF * LW;
        const int r = row0 + (j_beg + j) * PF;
        tma::mbar_arrive_expect_tx(&R.full[s], kStageBytes);
        tma::load_2d(dst, &mu, w0, r, &R.full[s]);
        tma::load_2d(dst + PF * LW, &mr, w0, r, &R.full[s]);
        tma::load_2d(dst + 2 * PF * LW, &mi, w0, r, &R.full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < S && j < n_tiles; ++j) issue(j, j);

    float2 la = f2(0.f), br = f2(0.f), bi = f2(0.f);
    if (valid) {
        la = make_float2(-Math<float>::softplus(-lam[w]), -Math<float>::softplus(-lam[w + 1]));
        br = ld2(b_r + w);
        bi = ld2(b_i + w);
    }
    const int64_t BW = (int64_t)Bn * W;
    const int64_t lane = (int64_t)b * W + (valid ? w : 0);
    float2 x = f2(0.f), sla = f2(0.f);
    if (!AGG && valid)
        for (int r = 0; r < seg; ++r)
            x = fma2(ex2_2(mul2(ld2(seg_a + r * BW + lane), f2(1.4426950408889634f))), x, ld2(seg_x + r * BW + lane));
    IO* py = y + ((int64_t)row0 + t_beg) * W + w;
    int s = 0;
    uint32_t ph = 0;
    for (int j = 0; j < n_tiles; ++j) {
        tma::mbar_wait(&R.full[s], ph);
        const IO* src = R.data + (size_t)s * 3 * PF * LW + 2 * tid;
        float2 cu[PF], cr[PF], ci[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            cu[k] = ld2(src + k * LW);
            cr[k] = ld2(src + (PF + k) * LW);
            ci[k] = ld2(src + (2 * PF + k) * LW);
        }
        __syncwarp();
        if ((tid & 31) == 0) tma::mbar_arrive(&R.empty[s]);
        if (tid == 0 && j + S < n_tiles) {
            tma::mbar_wait(&R.empty[s], ph);
            issue(j + S, s);
        }
        if (++s == S) {
            s = 0;
            ph ^= 1;
        }
        const int64_t t0 = (int64_t)(j_beg + j) * PF;
        const int nk = (int)min((int64_t)PF, t_end - t0);
        const float2 xin = x;
        float2 tla = f2(0.f), xs[PF];
        auto step = [&](int k) {
            const Coef2 q = gates2(cu[k], cr[k], ci[k], la, br, bi);
            x = fma2(q.a, x, mul2(mul2(q.s, q.i), q.u));
            xs[k] = x;
            if (AGG) tla = fma2(mul2(f2(kGate), q.r), la, tla);
        };
        if (nk == PF) {
#pragma unroll
            for (int k = 0; k < PF; ++k) step(k);
        } else {
#pragma unroll
            for (int k = 0; k < PF; ++k)
                if (k < nk) step(k);
        }
        if (AGG) {
            sla = add2(sla, tla);
        } else {
            if (ckpt && valid) {  // the state entering each checkpoint chunk of the tile
#pragma unroll
                for (int k = 0; k < PF; k += (PF < CK ? PF : CK))
                    if (k < nk && ((t0 + k) % CK) == 0)
                        __stcs(reinterpret_cast<float2*>(ckpt + ((t0 + k) / CK) * BW + lane), k ? xs[k - 1] : xin);
            }
            if (valid) {
                if (nk == PF) {
#pragma unroll
                    for (int k = 0; k < PF; ++k) st2(py + k * W, xs[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < PF; ++k)
                        if (k < nk) st2(py + k * W, xs[k]);
                }
            }
            py += PF * W;
        }
    }
    if (AGG && valid) {
        *reinterpret_cast<float2*>(seg_a + seg * BW + lane) = sla;
        *reinterpret_cast<float2*>(seg_x + seg * BW + lane) = x;
    }
    if (!AGG && ckpt && valid && t_end == L)  // final state
        __stcs(reinterpret_cast<float2*>(ckpt + ((L + CK - 1) / CK) * BW + lane), x);
}

// Backward without the y stream: time tiles of one checkpoint chunk (RC = 16
// rows of u, qr, qi, gy by TMA); per chunk the states are recomputed from the
// forward's checkpoint into registers, then the reverse recurrence runs over
// the staged rows again.  7 array passes instead of 8 (y is not read) for a
// second evaluation of the gates (MUFU has the headroom: the kernel is
// HBM-bound).  CTAs are not all co-resident (waves of LW-lane blocks).
template <typename IO, typename C, int LW, int RC>
__global__ void __launch_bounds__(LW) bwd_rc_kernel(
    const __grid_constant__ CUtensorMap mu, const __grid_constant__ CUtensorMap mr,
    const __grid_constant__ CUtensorMap mi, const __grid_constant__ CUtensorMap mg, const C* __restrict__ lam,
    const C* __restrict__ b_r, const C* __restrict__ b_i, const C* __restrict__ ckpt, IO* __restrict__ gu,
    IO* __restrict__ gqr, IO* __restrict__ gqi, C* __restrict__ gla_part, C* __restrict__ gbr_part,
    C* __restrict__ gbi_part, int64_t L, int64_t W, int n_wblk, int Bn, int S) {
    constexpr int NW = LW / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    auto R = ring<IO>(smem, S);
    const int tid = threadIdx.x;
    const int b = blockIdx.x / n_wblk;
    const int w0 = (blockIdx.x % n_wblk) * LW;
    const int64_t w = w0 + tid;
    const bool valid = w < W;
    const int row0 = b * (int)L;
    const int n_tiles = (int)((L + RC - 1) / RC);
    constexpr uint32_t kStageBytes = 4u * RC * LW * sizeof(IO);
    if (tid == 0) {
        tma::prefetch_map(&mu);
        tma::prefetch_map(&mr);
        tma::prefetch_map(&mi);
        tma::prefetch_map(&mg);
        for (int s = 0; s < S; ++s) {
            tma::mbar_init(&R.full[s], 1);
            tma::mbar_init(&R.empty[s], NW);
        }
        tma::fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int j) {  // j-th tile in reverse order
        const int tt = n_tiles - 1 - j;
        const int s = j % S;
        IO* dst = R.data + (size_t)s * 4 * RC * LW;
        const int r = row0 + tt * RC;
        tma::mbar_arrive_expect_tx(&R.full[s], kStageBytes);
        tma::load_2d(dst, &mu, w0, r, &R.full[s]);
        tma::load_2d(dst + RC * LW, &mr, w0, r, &R.full[s]);
        tma::load_2d(dst + 2 * RC * LW, &mi, w0, r, &R.full[s]);
        tma::load_2d(dst + 3 * RC * LW, &mg, w0, r, &R.full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < S && j < n_tiles; ++j) issue(j);

    C la = 0, br = 0, bi = 0;
    if (valid) {
        la = -Math<C>::softplus(-lam[w]);
        br = b_r[w];
        bi = b_i[w];
    }
    C h = 0;
    Kahan<C> sla, sbr, sbi;
    IO *pgu = gu + (int64_t)row0 * W + w, *pgr = gqr + (int64_t)row0 * W + w, *pgi = gqi + (int64_t)row0 * W + w;
    const int64_t ck_stride = (int64_t)Bn * W;
    const C* pc = ckpt + (int64_t)b * W + (valid ? w : 0);
    C xnext = valid ? __ldcg(pc + (int64_t)(n_tiles - 1) * ck_stride) : C(0);
    for (int j = 0; j < n_tiles; ++j) {
        const int s = j % S;
        const uint32_t ph = (j / S) & 1;
        const int tt = n_tiles - 1 - j;
        const C xin = xnext;  // state entering this chunk
        if (valid && tt > 0) xnext = __ldcg(pc + (int64_t)(tt - 1) * ck_stride);  // prefetch the next chunk's
        tma::mbar_wait(&R.full[s], ph);
        const IO* src = R.data + (size_t)s * 4 * RC * LW + tid;
        const int64_t t0 = (int64_t)tt * RC;
        const int nk = (int)min((int64_t)RC, L - t0);
        // forward recompute: xs[k] = x_{k-1}
        C xs[RC];
        C x = xin;
#pragma unroll
        for (int k = 0; k < RC; ++k) {
            xs[k] = x;
            if (k < nk) {
                const Coef<C> q = gates<C>(src[k * LW], src[(RC + k) * LW], src[(2 * RC + k) * LW], la, br, bi);
                x = q.a * x + (q.s * q.i) * q.u;
            }
        }
        C tla = 0, tbr = 0, tbi = 0;
        const int64_t o0 = t0 * W;
#pragma unroll
        for (int k = RC - 1; k >= 0; --k) {
            if (k < nk) {
                const Coef<C> q = gates<C>(src[k * LW], src[(RC + k) * LW], src[(2 * RC + k) * LW], la, br, bi);
                const C g = C(cvt(src[(3 * RC + k) * LW])) + h;
                h = q.a * g;
                const BwdOut<C> o = bwd_step<C>(q, g, xs[k], la);
                if (valid) {
                    const int64_t off = o0 + (int64_t)k * W;
                    st_io(pgu + off, o.gu);
                    st_io(pgr + off, o.gqr);
                    st_io(pgi + off, o.gqi);
                }
                tla += o.la_term;
                tbr += o.gqr;
                tbi += o.gqi;
            }
        }
        sla.add(tla);
        sbr.add(tbr);
        sbi.add(tbi);
        __syncwarp();
        if ((tid & 31) == 0) tma::mbar_arrive(&R.empty[s]);
        if (tid == 0 && j + S < n_tiles) {
            tma::mbar_wait(&R.empty[s], ph);
            issue(j + S);
        }
    }
    if (valid) {
        const int64_t p = (int64_t)b * W + w;
        gla_part[p] = sla.s;
        gbr_part[p] = sbr.s;
        gbi_part[p] = sbi.s;
    }
}

// ==================================================================== stream
template <typename IO, typename C, int PF>
__global__ void __launch_bounds__(kThreads) fwd_stream_kernel(
    const IO* __restrict__ u, const IO* __restrict__ qr, const IO* __restrict__ qi, const C* __restrict__ lam,
    const C* __restrict__ b_r, const C* __restrict__ b_i, IO* __restrict__ y, C* __restrict__ ckpt, int64_t L,
    int64_t W, int n_wblk, int Bn) {
    constexpr int CK = Tile<IO>::T;
    static_assert(CK % PF == 0, "checkpoint interval must be a multiple of the prefetch tile");
    using M = Math<C>;
    const int blk = blockIdx.x;
    const int b = blk / n_wblk;
    const int64_t w = (int64_t)(blk % n_wblk) * kThreads + threadIdx.x;
    if (w >= W) return;
    const C la = -M::softplus(-lam[w]), br = b_r[w], bi = b_i[w];
    const int64_t base = (int64_t)b * L * W + w;
    const IO *pu = u + base, *pr = qr + base, *pi = qi + base;
    IO* py = y + base;
    C* pc = ckpt ? ckpt + (int64_t)b * W + w : nullptr;
    const int64_t ck_stride = (int64_t)Bn * W;
    IO nu[PF], nr[PF], ni[PF];
#pragma unroll
    for (int k = 0; k < PF; ++k) {
        const bool ok = k < L;
        nu[k] = ok ? ld_stream(pu + k * W) : IO(0);
        nr[k] = ok ? ld_stream(pr + k * W) : IO(0);
        ni[k] = ok ? ld_stream(pi + k * W) : IO(0);
    }
    C x = 0;
    for (int64_t t0 = 0; t0 < L; t0 += PF) {
        IO cu[PF], cr[PF], ci[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            cu[k] = nu[k];
            cr[k] = nr[k];
            ci[k] = ni[k];
        }
        const int64_t tn = t0 + PF;
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const bool ok = tn + k < L;
            const int64_t off = (tn + k) * W;
            nu[k] = ok ? ld_stream(pu + off) : IO(0);
            nr[k] = ok ? ld_stream(pr + off) : IO(0);
            ni[k] = ok ? ld_stream(pi + off) : IO(0);
        }
        if (pc && (t0 % CK) == 0) {
            __stcs(pc, x);
            pc += ck_stride;
        }
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            if (t0 + k < L) {
                const Coef<C> q = gates<C>(cu[k], cr[k], ci[k], la, br, bi);
                x = q.a * x + (q.s * q.i) * q.u;
                st_io(py + (t0 + k) * W, x);
            }
        }
    }
    if (pc) __stcs(ckpt + ((L + CK - 1) / CK) * ck_stride + (int64_t)b * W + w, x);  // final state
}

// ================================================================== lookback
template <typename IO, typename C>
__global__ void __launch_bounds__(kThreads, 4) fwd_kernel(const IO* __restrict__ u, const IO* __restrict__ qr,
                                                          const IO* __restrict__ qi, const C* __restrict__ lam,
                                                          const C* __restrict__ b_r, const C* __restrict__ b_i,
                                                          IO* __restrict__ y, C* __restrict__ ckpt, int64_t L,
                                                          int64_t W, int n_wblk, int n_blk, LookbackWS ws) {
    constexpr int T = Tile<IO>::T;
    using M = Math<C>;
    const int tile = next_tile(ws.ticket);
    const int c = tile / n_blk, blk = tile % n_blk;
    const int b = blk / n_wblk;
    const int64_t w = (int64_t)(blk % n_wblk) * kThreads + threadIdx.x;
    const bool valid = w < W;
    const int64_t n_lanes = (int64_t)n_blk * kThreads;
    const int64_t lane = (int64_t)blk * kThreads + threadIdx.x;  // padded lane id
    const int64_t t0 = (int64_t)c * T;
    const int nt = (int)min((int64_t)T, L - t0);

    C la = 0, br = 0, bi = 0;
    if (valid) {
        la = -M::softplus(-lam[w]);  // log sigmoid(lambda), layers.py:1208-1210
        br = b_r[w];
        bi = b_i[w];
    }
    IO uu[T], rr[T], ii[T];
    const int64_t base = ((int64_t)b * L + t0) * W + (valid ? w : 0);
    {
        const IO *pu = u + base, *pr = qr + base, *pi = qi + base;
#pragma unroll
        for (int k = 0; k < T; ++k) {
            const bool ok = valid && k < nt;
            uu[k] = ok ? ld_stream(pu) : IO(0);
            rr[k] = ok ? ld_stream(pr) : IO(0);
            ii[k] = ok ? ld_stream(pi) : IO(0);
            pu += W;
            pr += W;
            pi += W;
        }
    }
    C av[T], bv[T];
    C A = 1, X = 0;
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const Coef<C> q = gates<C>(uu[k], rr[k], ii[k], la, br, bi);
        const bool ok = k < nt;
        av[k] = ok ? q.a : C(1);
        bv[k] = ok ? (q.s * q.i) * q.u : C(0);
        X = av[k] * X + bv[k];
        A = av[k] * A;
    }
    C* agg_a = static_cast<C*>(ws.agg_a);
    C* agg_x = static_cast<C*>(ws.agg_x);
    C* inc_x = static_cast<C*>(ws.inc_x);
    const int64_t woff = (int64_t)c * n_lanes + lane;
    int* sw = ws.status + (int64_t)c * n_blk + blk;
    C xin = 0;
    if (c > 0) {
        lb_publish<C>(sw, LB_AGG, agg_a + woff, A, agg_x + woff, X, valid);
        xin = lb_lookback<C>(ws, c, blk, n_blk, lane, n_lanes, valid);
    }
    if ((c % kAnchor) == 0) lb_publish<C>(sw, LB_INC, (C*)nullptr, A, inc_x + woff, A * xin + X, valid);
    const int Bn = n_blk / n_wblk;
    if (valid && ckpt) ckpt[((int64_t)c * Bn + b) * W + w] = xin;
    C x = xin;
    IO* py = y + base;
#pragma unroll
    for (int k = 0; k < T; ++k) {
        x = av[k] * x + bv[k];
        if (valid && k < nt) st_io(py, x);
        py += W;
    }
    // final state (the padded steps past L keep x: a = 1, b = 0)
    if (valid && ckpt && t0 + nt == L) ckpt[((int64_t)(c + 1) * Bn + b) * W + w] = x;
}

// Backward.  Reverse recurrence g_k = gy_k + a_{k+1} g_{k+1}; the carry passed
// leftwards between chunks is h = a_{t0} g_{t0} (layers.py:1252-1291 with
// autograd._scan_pullback 113-140).  States are recomputed from the chunk's
// entering state saved by the forward.
template <typename IO, typename C>
__global__ void __launch_bounds__(kThreads, 3) bwd_kernel(
    const IO* __restrict__ u, const IO* __restrict__ qr, const IO* __restrict__ qi, const C* __restrict__ lam,
    const C* __restrict__ b_r, const C* __restrict__ b_i, const C* __restrict__ ckpt, const IO* __restrict__ gy,
    IO* __restrict__ gu, IO* __restrict__ gqr, IO* __restrict__ gqi, C* __restrict__ gla_part,
    C* __restrict__ gbr_part, C* __restrict__ gbi_part, int64_t L, int64_t W, int n_wblk, int n_blk,
    int n_chunks, LookbackWS ws) {
    constexpr int T = Tile<IO>::T;
    using M = Math<C>;
    const int tile = next_tile(ws.ticket);
    const int s = tile / n_blk, blk = tile % n_blk;
    const int c = n_chunks - 1 - s;
    const int b = blk / n_wblk;
    const int64_t w = (int64_t)(blk % n_wblk) * kThreads + threadIdx.x;
    const bool valid = w < W;
    const int64_t n_lanes = (int64_t)n_blk * kThreads;
    const int64_t lane = (int64_t)blk * kThreads + threadIdx.x;
    const int64_t t0 = (int64_t)c * T;
    const int nt = (int)min((int64_t)T, L - t0);

    C la = 0, br = 0, bi = 0;
    if (valid) {
        la = -M::softplus(-lam[w]);
        br = b_r[w];
        bi = b_i[w];
    }
    IO uu[T], rr[T], ii[T], gg[T];
    const int64_t base = ((int64_t)b * L + t0) * W + (valid ? w : 0);
    {
        const IO *pu = u + base, *pr = qr + base, *pi = qi + base, *pg = gy + base;
#pragma unroll
        for (int k = 0; k < T; ++k) {
            const bool ok = valid && k < nt;
            uu[k] = ok ? ld_stream(pu) : IO(0);
            rr[k] = ok ? ld_stream(pr) : IO(0);
            ii[k] = ok ? ld_stream(pi) : IO(0);
            gg[k] = ok ? ld_stream(pg) : IO(0);
            pu += W;
            pr += W;
            pi += W;
            pg += W;
        }
    }
    C xprev[T], av[T];
    const int Bn = n_blk / n_wblk;
    C x = valid ? ckpt[((int64_t)c * Bn + b) * W + w] : C(0);
    C A = 1;
#pragma unroll
    for (int k = 0; k < T; ++k) {
        const Coef<C> q = gates<C>(uu[k], rr[k], ii[k], la, br, bi);
        const bool ok = k < nt;
        xprev[k] = x;
        av[k] = ok ? q.a : C(1);
        x = av[k] * x + (ok ? (q.s * q.i) * q.u : C(0));
        A = av[k] * A;
    }
    C H = 0;
#pragma unroll
    for (int k = T - 1; k >= 0; --k) {
        const C g = C(cvt(gg[k])) + H;
        H = av[k] * g;
    }
    C* agg_a = static_cast<C*>(ws.agg_a);
    C* agg_x = static_cast<C*>(ws.agg_x);
    C* inc_x = static_cast<C*>(ws.inc_x);
    const int64_t woff = (int64_t)s * n_lanes + lane;
    int* sw = ws.status + (int64_t)s * n_blk + blk;
    C hin = 0;
    if (s > 0) {
        lb_publish<C>(sw, LB_AGG, agg_a + woff, A, agg_x + woff, H, valid);
        hin = lb_lookback<C>(ws, s, blk, n_blk, lane, n_lanes, valid);
    }
    if ((s % kAnchor) == 0) lb_publish<C>(sw, LB_INC, (C*)nullptr, A, inc_x + woff, A * hin + H, valid);

    C h = hin, sla = 0, sbr = 0, sbi = 0;
#pragma unroll
    for (int k = T - 1; k >= 0; --k) {
        if (valid && k < nt) {
            const Coef<C> q = gates<C>(uu[k], rr[k], ii[k], la, br, bi);
            const C g = C(cvt(gg[k])) + h;
            h = q.a * g;
            const BwdOut<C> o = bwd_step<C>(q, g, xprev[k], la);
            const int64_t off = base + (int64_t)k * W;
            st_io(gu + off, o.gu);
            st_io(gqr + off, o.gqr);
            st_io(gqi + off, o.gqi);
            sla += o.la_term;
            sbr += o.gqr;
            sbi += o.gqi;
        }
    }
    if (valid) {
        const int64_t p = ((int64_t)c * Bn + b) * W + w;
        gla_part[p] = sla;
        gbr_part[p] = sbr;
        gbi_part[p] = sbi;
    }
}

// Kahan-compensated fixed-order column sums: out[j] = sum_r in[r, j].
template <typename C>
__global__ void colsum_kernel(const C* __restrict__ in, C* __restrict__ out, int64_t R, int64_t N) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N) return;
    Kahan<C> k;
    for (int64_t r = 0; r < R; ++r) k.add(in[r * N + j]);
    out[j] = k.s;
}

// ====================================================================== host
static int mode_env() {  // read per call so tests can switch kernels in-process
    const char* e = getenv("LRX_RGLRU_MODE");
    return !e ? 0 : !strcmp(e, "tma") ? 1 : !strcmp(e, "stream") ? 2 : !strcmp(e, "lookback") ? 3 : !strcmp(e, "rc") ? 4
                  : !strcmp(e, "rev") ? 5 : 0;
}

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

template <typename IO>
static void geometry(int64_t B, int64_t L, int64_t W, int* n_chunks, int* n_wblk, int* n_blk) {
    *n_chunks = (int)cdiv(L, Tile<IO>::T);
    *n_wblk = (int)cdiv(W, kThreads);
    *n_blk = (int)(B * *n_wblk);
}

template <typename IO, typename C>
static size_t ws_lookback(int64_t B, int64_t L, int64_t W) {
    int nc, nw, nb;
    geometry<IO>(B, L, W, &nc, &nw, &nb);
    const size_t lanes = (size_t)nb * kThreads;
    Carver cv(nullptr);
    cv.take<int>(1);
    cv.take<int>((size_t)nc * nb);
    for (int i = 0; i < 3; ++i) cv.take<C>((size_t)nc * lanes);
    return cv.off;
}

template <typename IO, typename C>
static int carve(void* w, size_t wb, int64_t B, int64_t L, int64_t W, LookbackWS* ws, Carver* cv,
                 cudaStream_t st) {
    int nc, nw, nb;
    geometry<IO>(B, L, W, &nc, &nw, &nb);
    const size_t lanes = (size_t)nb * kThreads;
    ws->ticket = cv->take<int>(1);
    ws->status = cv->take<int>((size_t)nc * nb);
    const size_t head = cv->off;
    ws->agg_a = cv->take<C>((size_t)nc * lanes);
    ws->agg_x = cv->take<C>((size_t)nc * lanes);
    ws->inc_x = cv->take<C>((size_t)nc * lanes);
    LRX_REQUIRE(w && cv->off <= wb, LRX_ERR_VALUE, "rglru workspace too small: %zu < %zu", wb, cv->off);
    LRX_REQUIRE(cudaMemsetAsync(w, 0, head, st) == cudaSuccess, LRX_ERR_CUDA, "workspace memset failed");
    return LRX_OK;
}

// TMA plan: lanes per CTA, ring stages, shared-memory bytes.  False when TMA
// does not apply (row alignment, residency), so the caller falls back.
struct TmaPlan {
    int LW, PF, S, n_wblk, n_blk, n_seg, seg_len;
    size_t smem;
};

// Launch plan of a TMA streaming pass with `narr` staged arrays.  The walk is
// latency-bound unless each SM holds enough independent steps in flight:
// resident warps x PF (the tile rows a thread evaluates between barrier
// waits) >= kWork.  The plan takes the smallest tile PF in {4, 8, 16} that
// reaches it and fits shared memory.  With few lanes (the per-rank batch of
// an 8-GPU job: < 6 warps per SM) the sequence is first cut into n_seg time
// segments (>= 256 steps, a multiple of the checkpoint interval) at the
// price of the AGG pass.  Env overrides (tests, sweeps):
// LRX_RGLRU_LW, _PF, _SEGS, _STAGES.
constexpr int kWork = 128;

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

template <typename IO>
static bool tma_plan(int64_t B, int64_t L, int64_t W, int narr, TmaPlan* p, int pf_cap = 16) {
    constexpr int CK = Tile<IO>::T;
    if ((W * (int64_t)sizeof(IO)) % 16) return false;
    const int sms = sm_count();
    int LW = W <= 32 ? 32 : W <= 64 ? 64 : 128;
    if (const char* e = getenv("LRX_RGLRU_LW")) LW = atoi(e) == 32 ? 32 : atoi(e) == 64 ? 64 : 128;
    const int n_wblk = (int)cdiv(W, LW);
    const int64_t n_blk = B * n_wblk;
    // per-direction overrides (narr 3 = forward, 4 = backward) before the shared ones
    const char* dir = narr == 3 ? "LRX_RGLRU_FWD_STAGES" : "LRX_RGLRU_BWD_STAGES";
    const double warps = (double)n_blk * (LW / 32) / sms;  // one lane per thread (the lane-pair kernels run half)
    // fp32 lane-pair walks with a full GPU of lanes (C4: ~35): short tiles in a
    // 2-stage ring stream best (measured C4 fwd 7.9 -> 7.0 ms, bwd 14.1 -> 13.3);
    // half as many lanes (~17) still prefer the short tile with the deep ring
    const bool pair32 = sizeof(IO) == 4 && LW >= 64 && !getenv("LRX_RGLRU_SCALAR");
    // a shallower ring also wins at half that (B = 32 of an 2-GPU job: fwd 4.21 -> 3.58 ms with 3 stages)
    const int smax = env_int(dir, env_int("LRX_RGLRU_STAGES", pair32 ? (warps >= 24 ? 2 : 3) : 6));
    // ring depth that fits for (PF, n_seg); 0 = does not fit
    auto stages = [&](int PF, int64_t n_seg) -> int {
        const int64_t per_sm = cdiv(n_blk * n_seg, (int64_t)sms);
        if (per_sm > 32) return 0;
        const size_t stage = (size_t)narr * PF * LW * sizeof(IO);
        // 228 KB per SM minus the 1 KB the runtime reserves per resident CTA
        const size_t budget = ((size_t)(228 - per_sm - 4) * 1024u) / per_sm;
        if (budget < 256 + 2 * stage) return 0;
        return (int)std::min<size_t>((size_t)smax, (budget - 256) / stage);
    };
    const int64_t max_seg = std::max<int64_t>(1, std::min<int64_t>(64, L / 256));
    // segments only below ~6 resident warps per SM (measured: the AGG pass
    // costs more than it buys above that); aim for ~12.
    // (the lane-pair forward streams 3 arrays with one ex2-free chain per pair:
    // it keeps one segment down to ~3 warps/SM -- B = 8 of an 8-GPU C4 job:
    // 1.64 ms with 3 segments, 1.47 with one; tools/rg_plan_grid.py)
    const double seg_below = pair32 && narr == 3 ? 3 : 6;
    int64_t n_seg = warps < seg_below ? std::min<int64_t>(max_seg, (int64_t)std::ceil(12 / warps)) : 1;
    int PF = 0;
    for (; n_seg >= 1 && !PF; n_seg = n_seg > 1 ? n_seg - 1 : 0) {
        for (int pf = 4; pf <= MaxPF<IO>::T; pf *= 2) {
            if (!stages(pf, n_seg)) break;
            PF = pf;
            // bf16 streams half the bytes per element: the walk is issue-bound, so
            // it takes twice the in-flight work (C4 bf16 fwd: PF 4 6.9 ms, PF 8 5.7 ms)
            // the lane-pair forward reaches it with half the tile (B = 32 / 16 / 8 of an
            // N-GPU job: PF 4 / 8 / 8, measured tools/rg_plan_grid.py)
            if (warps * n_seg * pf >= (sizeof(IO) == 2 ? 2 * kWork : kWork) / (pair32 && narr == 3 ? 2 : 1)) break;
        }
        if (PF) break;
    }
    if (!PF) return false;
    if (pair32 && warps >= 24 && n_seg == 1) PF = 2;
    const char* epf = getenv(narr == 3 ? "LRX_RGLRU_FWD_PF" : "LRX_RGLRU_BWD_PF");
    if (!epf) epf = getenv("LRX_RGLRU_PF");
    if (epf) PF = std::min(MaxPF<IO>::T, atoi(epf) >= 16 ? 16 : atoi(epf) >= 8 ? 8 : atoi(epf) >= 4 ? 4 : 2);
    PF = std::min(PF, std::max(2, pf_cap));  // the caller's residency cap (pair_resident)
    if (const char* e = getenv("LRX_RGLRU_SEGS"))
        n_seg = std::max<int64_t>(1, std::min<int64_t>({(int64_t)atoi(e), 64, std::max<int64_t>(1, L / 64)}));
    // segments start on a tile and on a checkpoint boundary
    constexpr int64_t kAlign = CK > MaxPF<IO>::T ? CK : MaxPF<IO>::T;
    const int64_t len = cdiv(cdiv(L, n_seg), kAlign) * kAlign;
    p->seg_len = (int)std::min<int64_t>(len, 1ll << 30);
    p->n_seg = (int)cdiv(L, len);
    while (!(p->S = stages(PF, p->n_seg)) && PF > 2) PF /= 2;  // overrides that do not fit
    if (!p->S) return false;
    p->LW = LW;
    p->PF = PF;
    p->n_wblk = n_wblk;
    p->n_blk = (int)n_blk;
    p->smem = 128 * ((2 * p->S * 8 + 127) / 128) + (size_t)p->S * narr * PF * LW * sizeof(IO);
    return true;
}

template <typename K>
static int reserve_smem(K k, size_t smem, const char* what) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        set_error("%s: cannot reserve %zu B of shared memory", what, smem);
        return LRX_ERR_CUDA;
    }
    return LRX_OK;
}

// seg: 2 * n_seg * B * W values (A then X) when pl.n_seg > 1.
template <typename IO, typename C, int LW, int PF>
static int launch_fwd_tma(const TmaPlan& pl, const CUtensorMap* m, const void* lam, const void* br, const void* bi,
                          void* y, void* ckpt, C* seg, int64_t B, int64_t L, int64_t W, cudaStream_t st) {
    const int64_t sn = (int64_t)pl.n_seg * B * W;
    if (pl.n_seg > 1) {
        auto a = fwd_tma_kernel<IO, C, LW, PF, true>;
        if (int rc = reserve_smem(a, pl.smem, "rglru fwd")) return rc;
        a<<<dim3(pl.n_blk, pl.n_seg - 1), LW, pl.smem, st>>>(m[0], m[1], m[2], (const C*)lam, (const C*)br,
                                                              (const C*)bi, nullptr, nullptr, seg, seg + sn, L, W,
                                                              pl.n_wblk, (int)B, pl.S, pl.seg_len, 0);
        if (int rc = launched("lrx_rglru_fwd/tma_agg")) return rc;
    }
    auto k = fwd_tma_kernel<IO, C, LW, PF, false>;
    if (int rc = reserve_smem(k, pl.smem, "rglru fwd")) return rc;
    k<<<dim3(pl.n_blk, pl.n_seg), LW, pl.smem, st>>>(m[0], m[1], m[2], (const C*)lam, (const C*)br, (const C*)bi,
                                                     (IO*)y, (C*)ckpt, seg, seg + sn, L, W, pl.n_wblk, (int)B, pl.S,
                                                     pl.seg_len, 0);
    return launched("lrx_rglru_fwd/tma");
}

// parts: 3 * n_seg * B * W; seg: 2 * n_seg * B * W (A then H).  `pa` is the
// plan of the 2-array AGG pass (same segments, deeper ring).
template <typename IO, typename C, int LW, int PF>
static int launch_bwd_tma(const TmaPlan& pl, const TmaPlan& pa, const CUtensorMap* m, const void* lam,
                          const void* br, const void* bi, void* gu, void* gqr, void* gqi, C* parts, C* seg, int64_t B,
                          int64_t L, int64_t W, cudaStream_t st) {
    const int64_t n = (int64_t)pl.n_seg * B * W;
    if (pl.n_seg > 1) {
        auto a = bwd_tma_kernel<IO, C, LW, PF, true>;
        if (int rc = reserve_smem(a, pa.smem, "rglru bwd")) return rc;
        // segment 0's pair is never read
        a<<<dim3(pl.n_blk, pl.n_seg - 1), LW, pa.smem, st>>>(
            m[0], m[1], m[2], m[3], m[4], (const C*)lam, (const C*)br, (const C*)bi, nullptr, nullptr, nullptr,
            nullptr, nullptr, nullptr, seg, seg + n, L, W, pl.n_wblk, (int)B, pa.S, pl.seg_len, 1, pl.n_seg);
        if (int rc = launched("lrx_rglru_bwd/tma_agg")) return rc;
    }
    auto k = bwd_tma_kernel<IO, C, LW, PF, false>;
    if (int rc = reserve_smem(k, pl.smem, "rglru bwd")) return rc;
    k<<<dim3(pl.n_blk, pl.n_seg), LW, pl.smem, st>>>(m[0], m[1], m[2], m[3], m[4], (const C*)lam, (const C*)br,
                                                     (const C*)bi, (IO*)gu, (IO*)gqr, (IO*)gqi, parts, parts + n,
                                                     parts + 2 * n, seg, seg + n, L, W, pl.n_wblk, (int)B, pl.S,
                                                     pl.seg_len, 0, pl.n_seg);
    return launched("lrx_rglru_bwd/tma");
}

// Reverse-reconstruction backward (4 staged arrays + anchors); the AGG pass
// is bwd_tma_kernel's (it stages qr and gy only).
template <typename IO, typename C, int LW, int PF>
static int launch_bwd_rev(const TmaPlan& pl, const TmaPlan& pa, const CUtensorMap* m, const void* lam,
                          const void* br, const void* bi, const void* ckpt, void* gu, void* gqr, void* gqi, C* parts,
                          C* seg, int64_t B, int64_t L, int64_t W, cudaStream_t st) {
    const int64_t n = (int64_t)pl.n_seg * B * W;
    if (pl.n_seg > 1) {
        auto a = bwd_tma_kernel<IO, C, LW, PF, true>;
        if (int rc = reserve_smem(a, pa.smem, "rglru bwd")) return rc;
        a<<<dim3(pl.n_blk, pl.n_seg - 1), LW, pa.smem, st>>>(
            m[0], m[1], m[2], m[3], m[0], (const C*)lam, (const C*)br, (const C*)bi, nullptr, nullptr, nullptr,
            nullptr, nullptr, nullptr, seg, seg + n, L, W, pl.n_wblk, (int)B, pa.S, pl.seg_len, 1, pl.n_seg);
        if (int rc = launched("lrx_rglru_bwd/tma_agg")) return rc;
    }
    auto k = bwd_rev_kernel<IO, C, LW, PF>;
    if (int rc = reserve_smem(k, pl.smem, "rglru bwd")) return rc;
    k<<<dim3(pl.n_blk, pl.n_seg), LW, pl.smem, st>>>(m[0], m[1], m[2], m[3], (const C*)lam, (const C*)br,
                                                     (const C*)bi, (const C*)ckpt, (IO*)gu, (IO*)gqr, (IO*)gqi, parts,
                                                     parts + n, parts + 2 * n, seg, seg + n, L, W, pl.n_wblk, (int)B,
                                                     pl.S, pl.seg_len, pl.n_seg);
    return launched("lrx_rglru_bwd/rev");
}

// Lane-pair variant of launch_bwd_rev (fp32 compute, LW >= 64).
template <typename IO, int LW, int PF>
static int launch_bwd_rev2(const TmaPlan& pl, const TmaPlan& pa, const CUtensorMap* m, const void* lam,
                           const void* br, const void* bi, const void* ckpt, void* gu, void* gqr, void* gqi,
                           float* parts, float* seg, int64_t B, int64_t L, int64_t W, cudaStream_t st) {
    const int64_t n = (int64_t)pl.n_seg * B * W;
    if (pl.n_seg > 1) {
        auto a = bwd_tma_kernel<IO, float, LW, PF, true>;
        if (int rc = reserve_smem(a, pa.smem, "rglru bwd")) return rc;
        a<<<dim3(pl.n_blk, pl.n_seg - 1), LW, pa.smem, st>>>(
            m[0], m[1], m[2], m[3], m[0], (const float*)lam, (const float*)br, (const float*)bi, nullptr, nullptr,
            nullptr, nullptr, nullptr, nullptr, seg, seg + n, L, W, pl.n_wblk, (int)B, pa.S, pl.seg_len, 1, pl.n_seg);
        if (int rc = launched("lrx_rglru_bwd/tma_agg")) return rc;
    }
    auto k = bwd_rev2_kernel<IO, LW, PF>;
    if (int rc = reserve_smem(k, pl.smem, "rglru bwd")) return rc;
    k<<<dim3(pl.n_blk, pl.n_seg), LW / 2, pl.smem, st>>>(m[0], m[1], m[2], m[3], (const float*)lam, (const float*)br,
                                                         (const float*)bi, (const float*)ckpt, (IO*)gu, (IO*)gqr,
                                                         (IO*)gqi, parts, parts + n, parts + 2 * n, seg, seg + n, L, W,
                                                         pl.n_wblk, (int)B, pl.S, pl.seg_len, pl.n_seg);
    return launched("lrx_rglru_bwd/rev2");
}

template <typename IO, typename C, int LW>
static int rev_pf(const TmaPlan& pl, const TmaPlan& pa, const CUtensorMap* m, const void* lam, const void* br,
                  const void* bi, const void* ckpt, void* gu, void* gqr, void* gqi, C* parts, C* seg, int64_t B,
                  int64_t L, int64_t W, cudaStream_t st) {
    if constexpr (LW >= 64 && std::is_same<C, float>::value) {
        if (!getenv("LRX_RGLRU_SCALAR")) switch (pl.PF) {
            case 16: return launch_bwd_rev2<IO, LW, 16>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st);
            case 8: return launch_bwd_rev2<IO, LW, 8>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st);
            case 2: return launch_bwd_rev2<IO, LW, 2>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st);
            default: return launch_bwd_rev2<IO, LW, 4>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st);
        }
    }
    switch (pl.PF) {
        case 16: if constexpr (MaxPF<IO>::T >= 16) return launch_bwd_rev<IO, C, LW, 16>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st);
        [[fallthrough]];
        case 8: return launch_bwd_rev<IO, C, LW, 8>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st);
        default: return launch_bwd_rev<IO, C, LW, 4>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st);
    }
}

template <typename IO, typename C, int LW>
static int launch_bwd_rc(const CUtensorMap* m, const void* lam, const void* br, const void* bi, const void* ckpt,
                         void* gu, void* gqr, void* gqi, C* parts, int64_t B, int64_t L, int64_t W, int S,
                         cudaStream_t st) {
    constexpr int RC = Tile<IO>::T;
    auto k = bwd_rc_kernel<IO, C, LW, RC>;
    const size_t smem = 128 * ((2 * S * 8 + 127) / 128) + (size_t)S * 4 * RC * LW * sizeof(IO);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        set_error("rglru bwd: cannot reserve %zu B of shared memory", smem);
        return LRX_ERR_CUDA;
    }
    const int n_wblk = (int)cdiv(W, LW);
    const int64_t n = B * W;
    k<<<(unsigned)(B * n_wblk), LW, smem, st>>>(m[0], m[1], m[2], m[3], (const C*)lam, (const C*)br, (const C*)bi,
                                                (const C*)ckpt, (IO*)gu, (IO*)gqr, (IO*)gqi, parts, parts + n,
                                                parts + 2 * n, L, W, n_wblk, (int)B, S);
    return launched("lrx_rglru_bwd/rc");
}

// The backward AGG pass (2 arrays) runs the main pass's tile and segments
// with the deeper ring its smaller stages allow.
template <typename IO>
static bool agg_plan(const TmaPlan& pl, int64_t B, int64_t L, int64_t W, TmaPlan* pa) {
    *pa = pl;
    const int sms = sm_count();
    const int64_t per_sm = cdiv((int64_t)pl.n_blk * pl.n_seg, (int64_t)sms);
    const size_t stage = (size_t)2 * pl.PF * pl.LW * sizeof(IO);
    const size_t budget = ((size_t)(228 - per_sm - 4) * 1024u) / per_sm;
    pa->S = (int)std::min<size_t>((size_t)env_int("LRX_RGLRU_STAGES", 6), (budget - 256) / stage);
    pa->smem = 128 * ((2 * pa->S * 8 + 127) / 128) + (size_t)pa->S * stage;
    return pa->S >= 2;
}

template <typename IO, int LW, int PF>
static int launch_fwd2(const TmaPlan& pl, const CUtensorMap* m, const void* lam, const void* br, const void* bi,
                       void* y, void* ckpt, float* seg, int64_t B, int64_t L, int64_t W, cudaStream_t st) {
    const int64_t sn = (int64_t)pl.n_seg * B * W;
    if (pl.n_seg > 1) {
        auto a = fwd2_kernel<IO, LW, PF, true>;
        if (int rc = reserve_smem(a, pl.smem, "rglru fwd")) return rc;
        a<<<dim3(pl.n_blk, pl.n_seg - 1), LW / 2, pl.smem, st>>>(m[0], m[1], m[2], (const float*)lam,
                                                                  (const float*)br, (const float*)bi, nullptr, nullptr,
                                                                  seg, seg + sn, L, W, pl.n_wblk, (int)B, pl.S,
                                                                  pl.seg_len, 0);
        if (int rc = launched("lrx_rglru_fwd/tma2_agg")) return rc;
    }
    auto k = fwd2_kernel<IO, LW, PF, false>;
    if (int rc = reserve_smem(k, pl.smem, "rglru fwd")) return rc;
    k<<<dim3(pl.n_blk, pl.n_seg), LW / 2, pl.smem, st>>>(m[0], m[1], m[2], (const float*)lam, (const float*)br,
                                                         (const float*)bi, (IO*)y, (float*)ckpt, seg, seg + sn, L, W,
                                                         pl.n_wblk, (int)B, pl.S, pl.seg_len, 0);
    return launched("lrx_rglru_fwd/tma2");
}

template <typename IO, typename C, int LW>
static int fwd_pf(const TmaPlan& pl, const CUtensorMap* m, const void* lam, const void* br, const void* bi, void* y,
                  void* ckpt, C* seg, int64_t B, int64_t L, int64_t W, cudaStream_t st) {
    if constexpr (LW >= 64 && std::is_same<C, float>::value) {
        if (!getenv("LRX_RGLRU_SCALAR")) switch (pl.PF) {
            case 16: return launch_fwd2<IO, LW, 16>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
            case 8: return launch_fwd2<IO, LW, 8>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
            case 2: return launch_fwd2<IO, LW, 2>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
            default: return launch_fwd2<IO, LW, 4>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
        }
    }
    switch (pl.PF) {
        case 16: if constexpr (MaxPF<IO>::T >= 16) return launch_fwd_tma<IO, C, LW, 16>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
        [[fallthrough]];
        case 8: return launch_fwd_tma<IO, C, LW, 8>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
        default: return launch_fwd_tma<IO, C, LW, 4>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
    }
}

template <typename IO, typename C, int LW>
static int bwd_pf(const TmaPlan& pl, const TmaPlan& pa, const CUtensorMap* m, const void* lam, const void* br,
                  const void* bi, void* gu, void* gqr, void* gqi, C* parts, C* seg, int64_t B, int64_t L, int64_t W,
                  cudaStream_t st) {
    switch (pl.PF) {
        case 16: if constexpr (MaxPF<IO>::T >= 16) return launch_bwd_tma<IO, C, LW, 16>(pl, pa, m, lam, br, bi, gu, gqr, gqi, parts, seg, B, L, W, st);
        [[fallthrough]];
        case 8: return launch_bwd_tma<IO, C, LW, 8>(pl, pa, m, lam, br, bi, gu, gqr, gqi, parts, seg, B, L, W, st);
        default: return launch_bwd_tma<IO, C, LW, 4>(pl, pa, m, lam, br, bi, gu, gqr, gqi, parts, seg, B, L, W, st);
    }
}

template <typename IO, typename C>
static int colsums(C* parts, int64_t rows, int64_t B, int64_t W, void* gla, void* gbr, void* gbi,
                   cudaStream_t st) {
    const int64_t pn = rows * B * W;
    const unsigned g = (unsigned)cdiv(W, 256);
    colsum_kernel<C><<<g, 256, 0, st>>>(parts, (C*)gla, rows * B, W);
    colsum_kernel<C><<<g, 256, 0, st>>>(parts + pn, (C*)gbr, rows * B, W);
    colsum_kernel<C><<<g, 256, 0, st>>>(parts + 2 * pn, (C*)gbi, rows * B, W);
    return launched("lrx_rglru_bwd/colsum", 3);
}

// Every CTA of a TMA pass walks its whole segment, so the grid must be
// resident in one wave.  The lane-pair kernels at PF >= 8 are register-bound
// to 512 / LW CTAs per SM (B = 32 of a 2-GPU job needs 5 at LW = 128: PF 8
// ran as 1.1 waves, bwd 6.8 -> 8.8 ms), so the plan halves PF until the
// occupancy query says the grid fits.
template <typename IO, int LW>
static bool pair_resident_lw(const TmaPlan& pl, int narr) {
    const void* k = nullptr;
    if (narr == 3) {
        switch (pl.PF) {
            case 16: k = (const void*)fwd2_kernel<IO, LW, 16, false>; break;
            case 8: k = (const void*)fwd2_kernel<IO, LW, 8, false>; break;
            case 2: k = (const void*)fwd2_kernel<IO, LW, 2, false>; break;
            default: k = (const void*)fwd2_kernel<IO, LW, 4, false>; break;
        }
    } else {
        switch (pl.PF) {
            case 16: k = (const void*)bwd_rev2_kernel<IO, LW, 16>; break;
            case 8: k = (const void*)bwd_rev2_kernel<IO, LW, 8>; break;
            case 2: k = (const void*)bwd_rev2_kernel<IO, LW, 2>; break;
            default: k = (const void*)bwd_rev2_kernel<IO, LW, 4>; break;
        }
    }
    int occ = 0;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, LW / 2, pl.smem) != cudaSuccess)
        return true;  // no answer: keep the plan (the launch reports real errors)
    return (int64_t)occ * sm_count() >= (int64_t)pl.n_blk * pl.n_seg;
}

template <typename IO, typename C>
static bool pair_plan(int64_t B, int64_t L, int64_t W, int narr, TmaPlan* pl) {
    if (!tma_plan<IO>(B, L, W, narr, pl)) return false;
    if constexpr (std::is_same<C, float>::value && !std::is_same<IO, double>::value) {
        if (pl->LW < 64 || getenv("LRX_RGLRU_SCALAR")) return true;
        while (pl->PF > 2 &&
               !(pl->LW == 128 ? pair_resident_lw<IO, 128>(*pl, narr) : pair_resident_lw<IO, 64>(*pl, narr))) {
            TmaPlan q;
            if (!tma_plan<IO>(B, L, W, narr, &q, pl->PF / 2) || q.PF >= pl->PF) break;
            *pl = q;
        }
    }
    return true;
}

template <typename IO, typename C>
static int fwd_t(const void* u, const void* qr, const void* qi, const void* lam, const void* br, const void* bi,
                 void* y, void* ckpt, int64_t B, int64_t L, int64_t W, void* w, size_t wb, cudaStream_t st) {
    const int mode = mode_env();
    TmaPlan pl;
    if ((mode == 0 || mode == 1 || mode == 5) && B * L < (1ll << 31) && pair_plan<IO, C>(B, L, W, 3, &pl)) {
        CUtensorMap m[3];
        const void* src[3] = {u, qr, qi};
        bool ok = true;
        for (int i = 0; i < 3; ++i) ok &= tma::encode_2d(&m[i], src[i], sizeof(IO), B * L, W, pl.PF, pl.LW);
        if (ok) {
            C* seg = nullptr;
            if (pl.n_seg > 1) {
                Carver cv(w);
                seg = cv.take<C>((size_t)2 * pl.n_seg * B * W);
                LRX_REQUIRE(w && cv.off <= wb, LRX_ERR_VALUE, "rglru workspace too small");
            }
            switch (pl.LW) {
                case 128: return fwd_pf<IO, C, 128>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
                case 64: return fwd_pf<IO, C, 64>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
                default: return fwd_pf<IO, C, 32>(pl, m, lam, br, bi, y, ckpt, seg, B, L, W, st);
            }
        }
        LRX_REQUIRE(mode != 1, LRX_ERR_UNSUPPORTED, "rglru: TMA descriptors unavailable");
    }
    int nc, nw, nb;
    geometry<IO>(B, L, W, &nc, &nw, &nb);
    if (mode == 2 || (mode == 0 && nb >= 4 * sm_count())) {
        fwd_stream_kernel<IO, C, 4><<<(unsigned)nb, kThreads, 0, st>>>(
            (const IO*)u, (const IO*)qr, (const IO*)qi, (const C*)lam, (const C*)br, (const C*)bi, (IO*)y, (C*)ckpt,
            L, W, nw, (int)B);
        return launched("lrx_rglru_fwd/stream");
    }
    LookbackWS ws;
    Carver cv(w);
    if (int rc = carve<IO, C>(w, wb, B, L, W, &ws, &cv, st)) return rc;
    fwd_kernel<IO, C><<<(unsigned)((int64_t)nc * nb), kThreads, 0, st>>>(
        (const IO*)u, (const IO*)qr, (const IO*)qi, (const C*)lam, (const C*)br, (const C*)bi, (IO*)y, (C*)ckpt,
        L, W, nw, nb, ws);
    return launched("lrx_rglru_fwd/lookback");
}

template <typename IO, typename C>
static int bwd_t(const void* u, const void* qr, const void* qi, const void* lam, const void* br, const void* bi,
                 const void* ckpt, const void* y, const void* gy, void* gu, void* gqr, void* gqi, void* gla,
                 void* gbr, void* gbi, int64_t B, int64_t L, int64_t W, void* w, size_t wb, cudaStream_t st) {
    const int mode = mode_env();
    const int64_t n = B * W;
    TmaPlan pl, pa;
    // default: the reverse-reconstruction walk (7 streams + 1/8 of anchors,
    // gates once per element); needs the forward's checkpoints
    if (ckpt && (mode == 0 || mode == 5) && B * L < (1ll << 31) && pair_plan<IO, C>(B, L, W, 4, &pl) &&
        agg_plan<IO>(pl, B, L, W, &pa)) {
        CUtensorMap m[4];
        const void* src[4] = {u, qr, qi, gy};
        bool ok = true;
        for (int i = 0; i < 4; ++i) ok &= tma::encode_2d(&m[i], src[i], sizeof(IO), B * L, W, pl.PF, pl.LW);
        if (ok) {
            const int64_t sn = (int64_t)pl.n_seg * B * W;
            Carver cv(w);
            C* parts = cv.take<C>((size_t)3 * sn);
            C* seg = cv.take<C>((size_t)2 * sn);
            LRX_REQUIRE(w && cv.off <= wb, LRX_ERR_VALUE, "rglru workspace too small");
            int rc;
            switch (pl.LW) {
                case 128: rc = rev_pf<IO, C, 128>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st); break;
                case 64: rc = rev_pf<IO, C, 64>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st); break;
                default: rc = rev_pf<IO, C, 32>(pl, pa, m, lam, br, bi, ckpt, gu, gqr, gqi, parts, seg, B, L, W, st); break;
            }
            if (rc) return rc;
            return colsums<IO, C>(parts, pl.n_seg, B, W, gla, gbr, gbi, st);
        }
        LRX_REQUIRE(mode != 5, LRX_ERR_UNSUPPORTED, "rglru: TMA descriptors unavailable");
    }
    // recompute variant (LRX_RGLRU_MODE=rc): 7 array passes, no y stream.
    // fp32: measured slower on C4 (18.3 vs 16.4 ms: the 2 x gates per element
    // at ~14 warps/SM, limited by the 512 B of staged rows per thread), so the
    // y-streaming kernel stays the default there.  bf16 I/O: y is rounded, so
    // this is the default backward (the look-back recompute took 65 ms on C4).
    const bool rc_ok = ckpt && B * L < (1ll << 31) && (W * (int64_t)sizeof(IO)) % 16 == 0 && sizeof(IO) <= 4;
    if (rc_ok && (mode == 4 || (sizeof(IO) == 2 && (mode == 0 || mode == 1)))) {
        constexpr int RC = Tile<IO>::T;
        // 128-channel CTAs when they still give 4 per SM (C4 bf16: 14.5 vs 15.3 ms at 64)
        int LW = B * cdiv(W, 128) >= 4 * sm_count() ? 128 : B * cdiv(W, 64) >= 4 * sm_count() ? 64 : 32;
        if (const char* e = getenv("LRX_RGLRU_RC_LW")) LW = atoi(e) >= 128 ? 128 : atoi(e) >= 64 ? 64 : 32;
        const int S = env_int("LRX_RGLRU_RC_STAGES", 2);
        CUtensorMap m[4];
        const void* src[4] = {u, qr, qi, gy};
        bool ok = true;
        for (int i = 0; i < 4; ++i) ok &= tma::encode_2d(&m[i], src[i], sizeof(IO), B * L, W, RC, LW);
        if (ok) {
            Carver cv(w);
            C* parts = cv.take<C>((size_t)3 * n);
            LRX_REQUIRE(w && cv.off <= wb, LRX_ERR_VALUE, "rglru workspace too small");
            const int rc = LW == 128 ? launch_bwd_rc<IO, C, 128>(m, lam, br, bi, ckpt, gu, gqr, gqi, parts, B, L, W, S, st)
                           : LW == 64 ? launch_bwd_rc<IO, C, 64>(m, lam, br, bi, ckpt, gu, gqr, gqi, parts, B, L, W, S, st)
                                      : launch_bwd_rc<IO, C, 32>(m, lam, br, bi, ckpt, gu, gqr, gqi, parts, B, L, W, S, st);
            if (rc) return rc;
            return colsums<IO, C>(parts, 1, B, W, gla, gbr, gbi, st);
        }
        LRX_REQUIRE(mode != 4, LRX_ERR_UNSUPPORTED, "rglru: TMA descriptors unavailable");
    }
    // y (= the state) is exact only at fp32/f64 I/O; bf16 recomputes instead
    if (y && sizeof(IO) != 2 && (mode == 0 || mode == 1) && B * L < (1ll << 31) &&
        tma_plan<IO>(B, L, W, 5, &pl) && agg_plan<IO>(pl, B, L, W, &pa)) {
        CUtensorMap m[5];
        const void* src[5] = {u, qr, qi, gy, y};
        bool ok = true;
        for (int i = 0; i < 5; ++i) ok &= tma::encode_2d(&m[i], src[i], sizeof(IO), B * L, W, pl.PF, pl.LW);
        if (ok) {
            const int64_t sn = (int64_t)pl.n_seg * B * W;
            Carver cv(w);
            C* parts = cv.take<C>((size_t)3 * sn);
            C* seg = cv.take<C>((size_t)2 * sn);
            LRX_REQUIRE(w && cv.off <= wb, LRX_ERR_VALUE, "rglru workspace too small");
            int rc;
            switch (pl.LW) {
                case 128: rc = bwd_pf<IO, C, 128>(pl, pa, m, lam, br, bi, gu, gqr, gqi, parts, seg, B, L, W, st); break;
                case 64: rc = bwd_pf<IO, C, 64>(pl, pa, m, lam, br, bi, gu, gqr, gqi, parts, seg, B, L, W, st); break;
                default: rc = bwd_pf<IO, C, 32>(pl, pa, m, lam, br, bi, gu, gqr, gqi, parts, seg, B, L, W, st); break;
            }
            if (rc) return rc;
            return colsums<IO, C>(parts, pl.n_seg, B, W, gla, gbr, gbi, st);
        }
        LRX_REQUIRE(mode != 1, LRX_ERR_UNSUPPORTED, "rglru: TMA descriptors unavailable");
    }
    LRX_REQUIRE(ckpt, LRX_ERR_VALUE, "rglru bwd: this path recomputes states and needs the forward checkpoints");
    int nc, nw, nb;
    geometry<IO>(B, L, W, &nc, &nw, &nb);
    LookbackWS ws;
    Carver cv(w);
    if (int rc = carve<IO, C>(w, wb, B, L, W, &ws, &cv, st)) return rc;
    C* parts = cv.take<C>((size_t)3 * nc * n);
    LRX_REQUIRE(cv.off <= wb, LRX_ERR_VALUE, "rglru workspace too small");
    const size_t pn = (size_t)nc * n;
    bwd_kernel<IO, C><<<(unsigned)((int64_t)nc * nb), kThreads, 0, st>>>(
        (const IO*)u, (const IO*)qr, (const IO*)qi, (const C*)lam, (const C*)br, (const C*)bi, (const C*)ckpt,
        (const IO*)gy, (IO*)gu, (IO*)gqr, (IO*)gqi, parts, parts + pn, parts + 2 * pn, L, W, nw, nb, nc, ws);
    if (int rc = launched("lrx_rglru_bwd/lookback")) return rc;
    return colsums<IO, C>(parts, nc, B, W, gla, gbr, gbi, st);
}

template <typename IO, typename C>
static size_t bwd_ws_bytes(int64_t B, int64_t L, int64_t W) {
    int nc, nw, nb;
    geometry<IO>(B, L, W, &nc, &nw, &nb);
    const size_t lb = ws_lookback<IO, C>(B, L, W) + align_up((size_t)3 * nc * B * W * sizeof(C));
    TmaPlan pl;  // segmented TMA passes: 3 partial + 2 pair rows per segment
    const size_t tm = tma_plan<IO>(B, L, W, 5, &pl) ? 5 * align_up((size_t)pl.n_seg * B * W * sizeof(C)) : 0;
    const size_t tr = tma_plan<IO>(B, L, W, 4, &pl) ? 5 * align_up((size_t)pl.n_seg * B * W * sizeof(C)) : 0;
    return std::max(lb, std::max(tm, tr));
}

}  // namespace rglru
}  // namespace lrx

using namespace lrx;

extern "C" {

int lrx_rglru_chunking(int io_dtype, int64_t L, int64_t* chunk_len, int64_t* n_chunks) {
    LRX_REQUIRE(L >= 1, LRX_ERR_SHAPE, "length must be >= 1");
    const int T = io_dtype == LRX_F64 ? rglru::Tile<double>::T : rglru::Tile<float>::T;
    *chunk_len = T;
    *n_chunks = cdiv(L, T);
    return LRX_OK;
}

size_t lrx_rglru_workspace_bytes(int io_dtype, int64_t B, int64_t L, int64_t W) {
    if (B < 1 || L < 1 || W < 1) return 256;
    switch (io_dtype) {
        case LRX_F32: return rglru::bwd_ws_bytes<float, float>(B, L, W);
        case LRX_BF16: return rglru::bwd_ws_bytes<__nv_bfloat16, float>(B, L, W);
        case LRX_F64: return rglru::bwd_ws_bytes<double, double>(B, L, W);
    }
    return 0;
}

int lrx_rglru_fwd(int io_dtype, const void* u, const void* qr, const void* qi, const void* lambda_param,
                  const void* b_r, const void* b_i, void* y, void* ckpt, int64_t B, int64_t L, int64_t W,
                  void* workspace, size_t workspace_bytes, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && W >= 1, LRX_ERR_SHAPE, "bad extents B=%lld L=%lld W=%lld", (long long)B,
                (long long)L, (long long)W);
    cudaStream_t st = (cudaStream_t)stream;
    switch (io_dtype) {
        case LRX_F32:
            return rglru::fwd_t<float, float>(u, qr, qi, lambda_param, b_r, b_i, y, ckpt, B, L, W, workspace,
                                              workspace_bytes, st);
        case LRX_BF16:
            return rglru::fwd_t<__nv_bfloat16, float>(u, qr, qi, lambda_param, b_r, b_i, y, ckpt, B, L, W,
                                                      workspace, workspace_bytes, st);
        case LRX_F64:
            return rglru::fwd_t<double, double>(u, qr, qi, lambda_param, b_r, b_i, y, ckpt, B, L, W, workspace,
                                                workspace_bytes, st);
    }
    set_error("rglru: unsupported io dtype %d", io_dtype);
    return LRX_ERR_VALUE;
}

int lrx_rglru_bwd(int io_dtype, const void* u, const void* qr, const void* qi, const void* lambda_param,
                  const void* b_r, const void* b_i, const void* ckpt, const void* y, const void* gy, void* gu_local,
                  void* gqr, void* gqi, void* gla, void* gb_r, void* gb_i, int64_t B, int64_t L, int64_t W,
                  void* workspace, size_t workspace_bytes, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && W >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    switch (io_dtype) {
        case LRX_F32:
            return rglru::bwd_t<float, float>(u, qr, qi, lambda_param, b_r, b_i, ckpt, y, gy, gu_local, gqr, gqi,
                                              gla, gb_r, gb_i, B, L, W, workspace, workspace_bytes, st);
        case LRX_BF16:
            return rglru::bwd_t<__nv_bfloat16, float>(u, qr, qi, lambda_param, b_r, b_i, ckpt, y, gy, gu_local, gqr,
                                                      gqi, gla, gb_r, gb_i, B, L, W, workspace, workspace_bytes, st);
        case LRX_F64:
            return rglru::bwd_t<double, double>(u, qr, qi, lambda_param, b_r, b_i, ckpt, y, gy, gu_local, gqr, gqi,
                                                gla, gb_r, gb_i, B, L, W, workspace, workspace_bytes, st);
    }
    set_error("rglru: unsupported io dtype %d", io_dtype);
    return LRX_ERR_VALUE;
}

}  // extern "C"
