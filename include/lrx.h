/*
 * lrx — B200-native (sm_100a) diagonal linear-recurrence scan: the C-ABI.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `linrec` (arxiv 2602.08810, /root/reference/pkg/src/linrec).  Every entry
 * point below replaces one reference interface; the citation is given per
 * function.  Conventions (mirroring the reference's native loops,
 * _scan_kernels.py:1-8):
 *
 *   - plain device pointers and sizes, no framework types;
 *   - the CALLER allocates every output and the workspace (the reference's
 *     kernels also write into a caller-allocated `out`), sized with the
 *     matching *_workspace_bytes() query;
 *   - every call is stream-ordered and asynchronous on `stream`
 *     (a cudaStream_t passed as void*); nothing synchronises the host;
 *   - calls are reentrant across streams and devices (the reference's
 *     kernels are nogil and write disjoint slices);
 *   - return value: LRX_OK or an error code; lrx_last_error() returns a
 *     thread-local message for the last failure.  Shape/value errors are
 *     detected before any launch.
 *
 * Layouts: generic operator arrays are time-major [L, N] C-contiguous, as in
 * _scan_kernels.py.  Fused layer kernels take the layer-level layout
 * [B, L, H] (batch, time, channel) of Layer.forward(u[B, L, d_model])
 * (layers.py:218-249); parameters keep the shapes of Layer.parameters().
 * Complex arrays are interleaved (re, im) pairs.
 */
#ifndef LRX_H
#define LRX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (map to ShapeError / ValueError / SingularBilinear in Python) */
#define LRX_OK 0
#define LRX_ERR_SHAPE 1       /* numerics.py:42 ShapeError                  */
#define LRX_ERR_VALUE 2       /* ValueError (bad mode / scheme / dtype)      */
#define LRX_ERR_SINGULAR 3    /* discretize.py:47 SingularBilinear           */
#define LRX_ERR_CUDA 4        /* CUDA launch / runtime failure               */
#define LRX_ERR_UNSUPPORTED 5 /* size outside the compiled kernel range      */

/* element types */
#define LRX_F32 0
#define LRX_F64 1
#define LRX_C64 2
#define LRX_C128 3
#define LRX_BF16 4

/* discretization schemes (discretize.py:118-128 SCHEMES) */
#define LRX_ZOH 0
#define LRX_BILINEAR 1
#define LRX_DIRAC 2

const char* lrx_last_error(void);
int lrx_version(void);
/* number of kernels launched by this library in this process (monotonic) */
int64_t lrx_launch_count(void);

/* ------------------------------------------------------------------------ *
 * Generic operator.  Replaces scan.scan_sequential / scan.scan_parallel
 * (scan.py:127-201) and the numba loops scan_const/scan_var,
 * compose_*, local_scan_*, fixup_* (_scan_kernels.py:17-128): one pass,
 * chunks chained by a decoupled look-back instead of the 3-phase thread pool.
 *   out[k] = a_k * out[k-1] + b[k],  out[-1] = x0 (zeros when x0 == NULL)
 * a is [N] (a_per_step = 0) or [L, N]; dtype in {F32, F64, C64, C128}.
 * ------------------------------------------------------------------------ */
size_t lrx_scan_workspace_bytes(int dtype, int64_t L, int64_t N);
int lrx_scan_fwd(int dtype, int a_per_step, const void* a, const void* b, const void* x0,
                 void* out, int64_t L, int64_t N, void* workspace, size_t workspace_bytes,
                 void* stream);

/* Reverse-mode pullback.  Replaces autograd._scan_pullback / scan_backward
 * (autograd.py:113-179) and backward_const/backward_var
 * (_scan_kernels.py:131-153).  `a` is NOT conjugated by the caller (the
 * conjugation of the reference's callers happens inside):
 *   g[k]   = gx[k] + conj(a_{k+1}) g[k+1]          -> gb   [L, N]
 *   ga     = g[k] conj(x[k-1])  ([L,N] per-step; summed over k to [N] for
 *            constant a)                            -> ga   (NULL to skip; needs x)
 *   gx0    = conj(a_0) g[0]                         -> gx0  (NULL to skip)
 * x is the forward state [L, N]; x0 the forward seed (NULL = zeros). */
size_t lrx_scan_bwd_workspace_bytes(int dtype, int64_t L, int64_t N);
int lrx_scan_bwd(int dtype, int a_per_step, const void* a, const void* x, const void* x0,
                 const void* gx, void* gb, void* ga, void* gx0, int64_t L, int64_t N,
                 void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * RG-LRU gated scan, fused (layers.py:1171-1291: _log_a 1208-1210, _gates
 * 1212-1218, _forward_tape 1239-1250, _backward 1252-1291).
 *   r = sigmoid(qr + b_r), i = sigmoid(qi + b_i), log a = 8 r log sigmoid(lambda)
 *   x_k = a_k x_{k-1} + sqrt(-expm1(2 log a_k)) i_k u_k ,  y = x
 * qr = u W_r^T and qi = u W_i^T are the layer's gate GEMM outputs (bias not
 * added).  io_dtype in {F32, F64, BF16}; params (lambda, b_r, b_i) are F32 for
 * F32/BF16 I/O and F64 for F64 I/O.  ckpt receives the state entering every
 * time chunk and, in its last row, the final state ([n_chunks + 1, B*W],
 * compute precision): the backward's reconstruction anchors.
 * ------------------------------------------------------------------------ */
int lrx_rglru_chunking(int io_dtype, int64_t L, int64_t* chunk_len, int64_t* n_chunks);
size_t lrx_rglru_workspace_bytes(int io_dtype, int64_t B, int64_t L, int64_t W);
int lrx_rglru_fwd(int io_dtype, const void* u, const void* qr, const void* qi, const void* lambda_param,
                  const void* b_r, const void* b_i, void* y, void* ckpt, int64_t B, int64_t L, int64_t W,
                  void* workspace, size_t workspace_bytes, void* stream);
/* Backward.  Outputs gu_local = sqrt(1-a^2) i g (the GEMM terms gqr W_r +
 * gqi W_i are the caller's), gqr, gqi ([B, L, W], io dtype), and the
 * parameter-gradient sums over batch and time gla = sum 8 r dlog(a),
 * gb_r = sum gqr, gb_i = sum gqi ([W], compute precision; fixed-order,
 * compensated).  The default walk reconstructs x_{t-1} = (x_t - b_t) / a_t
 * from the gates it evaluates for the pullback, re-anchored on ckpt at every
 * chunk boundary (<= 7 reconstructed steps).  y (the forward output = the
 * state) is read only by the y-streaming variant (LRX_RGLRU_MODE=tma, f32/f64
 * I/O) and may be NULL.  Workspace: lrx_rglru_workspace_bytes(). */
int lrx_rglru_bwd(int io_dtype, const void* u, const void* qr, const void* qi, const void* lambda_param,
                  const void* b_r, const void* b_i, const void* ckpt, const void* y, const void* gy,
                  void* gu_local, void* gqr, void* gqi, void* gla, void* gb_r, void* gb_i, int64_t B,
                  int64_t L, int64_t W, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * S6 selective scan, fused (layers.py:983-1118: _projections 1020-1027,
 * _forward_tape 1051-1066, _backward 1068-1118).
 *   delta = softplus(pre + b_delta), abar = exp(delta * a), a = -exp(a_log)
 *   x_k[d,n] = abar x_{k-1} + delta u B_k[n],  y = sum_n C_k[n] x_k + D u
 * pre [B,L,D] = (u W_delta) W_delta_proj (bias not added); Bk, Ck [B,L,N].
 * u / y / gy / gu_local use io_dtype; pre, Bk, Ck and gpre use the compute
 * precision (F32 for F32/BF16 io, F64 for F64 io).
 * io_dtype in {F32, F64, BF16}; params (b_delta [D], a_log [D,N], Dskip [D])
 * F32 (F64 for F64 I/O).  ckpt receives the state at
 * every ckpt_len-step boundary and, in its last slot, the final state:
 * [B, n_ckpt, D, N] compute precision (n_ckpt = ceil(L/ckpt_len) + 1).
 * ------------------------------------------------------------------------ */
/* Geometry for these extents: out[0] ckpt_len, out[1] n_ckpt, out[2] n_dblk
 * (rows of the gBk/gCk partials), out[3] n_seg (time segments run
 * concurrently when B*D alone cannot fill the GPU), out[4] part_rows (rows of
 * the ga/gD/gb partials = n_seg*B), out[5] workspace bytes. */
int lrx_s6_geometry(int io_dtype, int64_t B, int64_t L, int64_t D, int64_t N, int64_t* out6);
/* flags for lrx_s6_fwd / lrx_s6_bwd */
#define LRX_S6_DELTA_IN 2  /* `pre` already holds delta = softplus(pre + b_delta)
                              (the projection GEMM's epilogue): no softplus in the
                              scan, sigmoid(pre) = 1 - exp(-delta) in the backward;
                              b_delta is ignored; gpre stays d loss / d pre */
#define LRX_S6_REUSE_AGG 1 /* ws already holds the per-segment maps from a
                              preceding lrx_s6_{fwd,bwd}_carry on the same inputs */
/* x0 [B, D, N] (compute precision, NULL = zeros) seeds the state: the
 * sequence-parallel mode continues a scan another rank started.
 * ws: caller-allocated device workspace of out[5] bytes (transient). */
int lrx_s6_fwd(int io_dtype, const void* u, const void* pre, const void* b_delta, const void* a_log,
               const void* Bk, const void* Ck, const void* Dskip, const void* x0, void* y, void* ckpt,
               int64_t B, int64_t L, int64_t D, int64_t N, void* ws, int64_t ws_bytes, int flags, void* stream);
/* Outputs: gu_local = D gy + delta * sum_n g B   (GEMM terms are the
 * caller's) [B,L,D] io dtype; gpre = sigmoid(pre+b) * gdelta [B,L,D]
 * compute precision;
 * gBk_part, gCk_part [n_dblk, B, L, N] per channel-block partials;
 * ga_part (d/d a_log, already times a) [part_rows, D, N]; gD_part, gb_part
 * [part_rows, D] (compute precision).  Reduce the partial axes with
 * lrx_reduce_rows. */
/* h_in [B, D, N] (NULL = zeros) is the cotangent carry entering from the
 * right (abar_{L} g_{L} of the next slice); h_out [B, D, N] (NULL to skip)
 * receives abar_0 g_0 = d loss / d x0 (the carry for the slice to the left). */
int lrx_s6_bwd(int io_dtype, const void* u, const void* pre, const void* b_delta, const void* a_log,
               const void* Bk, const void* Ck, const void* Dskip, const void* ckpt, const void* gy,
               const void* h_in, void* gu_local, void* gpre, void* gBk_part, void* gCk_part, void* ga_part,
               void* gD_part, void* gb_part, void* h_out, int64_t B, int64_t L, int64_t D, int64_t N,
               void* ws, int64_t ws_bytes, int flags, void* stream);
/* Sequence-parallel carry exchange (config C5; F32/BF16 io, N = 16).
 * fwd_carry: the slice's affine map x_end = prod(abar) x_in + x_agg, returned
 * as x_agg [B, D, N] (state reached from a zero start) and sd_agg [B, D]
 * (sum of delta; prod abar = exp(a * sd_agg)).  bwd_carry: the same for the
 * cotangent carry travelling right to left (h_agg = d loss / d x_in with a
 * zero carry entering on the right).  Both leave the per-segment maps in ws
 * for a following lrx_s6_fwd / lrx_s6_bwd with LRX_S6_REUSE_AGG. */
int lrx_s6_fwd_carry(int io_dtype, const void* u, const void* pre, const void* b_delta, const void* a_log,
                     const void* Bk, void* x_agg, void* sd_agg, int64_t B, int64_t L, int64_t D, int64_t N,
                     void* ws, int64_t ws_bytes, void* stream);
int lrx_s6_bwd_carry(int io_dtype, const void* gy, const void* pre, const void* b_delta, const void* a_log,
                     const void* Ck, void* h_agg, void* sd_agg, int64_t B, int64_t L, int64_t D, int64_t N,
                     void* ws, int64_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * Single-step (decode) updates on a device-resident state, one token per
 * sequence (Layer.step, layers.py:251-269; per kind S4D 578-613, S5/LRU
 * 748-783, S6 1145-1168, RG-LRU 1310-1336).  x is updated in place, y is
 * written; nothing is allocated.
 * ------------------------------------------------------------------------ */
/* Operator-level step (scan.py:232-250): x[n] <- a x + b, with a / b of
 * period a_period / b_period (n = full, 1 = scalar, p = trailing lanes). */
int lrx_scan_step(int dtype, void* x, const void* a, const void* b, int64_t n, int64_t a_period, int64_t b_period,
                  void* stream);
/* S4D: x[B,H,N] = abar[H,N] x + w[H,N] u[B,H]; y[B,H] = Re(sum_n c x) + d u.
 * dtype C64 / C128 (x, abar, w, c complex; d, u, y the matching real type). */
int lrx_s4d_step(int dtype, void* x, const void* abar, const void* w, const void* c, const void* d, const void* u,
                 void* y, int64_t B, int64_t H, int64_t N, void* stream);
/* S5 / LRU: x[B,P] = abar[P] x + scale[P] (B u); y[B,H] = out_scale Re(C x) + D u
 * with B = Bre + i Bim [P,H], C = Cre + i Cim [H,P] real planes. */
int lrx_mimo_step(int dtype, void* x, const void* abar, const void* scale, const void* Bre, const void* Bim,
                  const void* Cre, const void* Cim, const void* D, const void* u, void* y, double out_scale,
                  int64_t B, int64_t P, int64_t H, void* stream);
/* ---- S4D fused scan (layers.py:352-546) ------------------------------------
 * u, y, gy, gu [B, L, H] real (F32 / F64); c [H, N] complex of that
 * precision; d [H].  N in {8, 16, 32, 64} (LRX_ERR_UNSUPPORTED otherwise: the
 * generic operator path).  Steps:
 *   constant  (deltas == NULL): abar, w (= scale b) [H, N] complex
 *             (lam / b / delta unused);
 *   per step  (asynchronous S4D, layers.py:402-440, discretize.py:59-93):
 *             deltas [B, L] real, delta [H] = exp(log_delta), lam, b [H, N]
 *             complex, scheme 0 ZOH / 1 bilinear / 2 dirac -- abar_k, scale_k
 *             are computed in the kernel (abar / w unused).
 * ckpt [B, n_chunks, H, N] complex = the state entering every chunk
 * (lrx_s4d_chunking); xlast [B, H, N] (or NULL) = the final state.  Long
 * sequences over few lanes run in time segments: workspace lrx_s4d_geometry
 * geo[1] bytes, partial rows R = geo[0] (segments) x B.
 * Backward partials [R, H, N] (R x [H] for gd_part), summed by the caller:
 *   constant: p1 = sum g conj(x_prev) (d abar), p2 = sum u g (d w-path);
 *   per step: p1 = d lambda, p2 = d b, p3 (real) = sum_k deltas_k d delta_k
 *             (times delta[h] and summed over n: d log_delta);
 *   gc_part = sum gy conj(x), gd_part = sum gy u. */
int lrx_s4d_chunking(int64_t L, int64_t* chunk_len, int64_t* n_chunks);
int lrx_s4d_geometry(int dtype, int64_t B, int64_t L, int64_t H, int64_t N, int64_t* geo);
int lrx_s4d_fwd(int dtype, const void* u, const void* abar, const void* w, const void* lam, const void* b,
                const void* delta, const void* deltas, int scheme, const void* c, const void* d, void* y, void* ckpt,
                void* xlast, int64_t B, int64_t L, int64_t H, int64_t N, void* workspace, size_t workspace_bytes,
                void* stream);
int lrx_s4d_bwd(int dtype, const void* u, const void* gy, const void* abar, const void* w, const void* lam,
                const void* b, const void* delta, const void* deltas, int scheme, const void* c, const void* d,
                const void* ckpt, void* gu, void* p1_part, void* p2_part, void* p3_part, void* gc_part, void* gd_part,
                int64_t B, int64_t L, int64_t H, int64_t N, void* workspace, size_t workspace_bytes, void* stream);

/* ---- MIMO scan with per-step steps (asynchronous S5, layers.py:650-658) ----
 * x_k = abar_k x_{k-1} + scale_k bu_k with (abar_k, scale_k) = scheme(lam[p],
 * deltas[b, k] delta[p]) computed in the kernel (scheme 0 ZOH / 1 bilinear /
 * 2 dirac; discretize.py:59-93).  lam [P] complex, delta [P] = exp(log_delta)
 * and deltas [B, L] real of the matching precision; bu, x, gx, gbu [B, L, P].
 * Backward partials [n_chunks * B, P] (lrx_mimo_chunking): glam (complex) and
 * gdl = sum_k deltas_k d delta_k (real; times delta[p]: d log_delta). */
size_t lrx_mimo_ps_workspace_bytes(int dtype, int64_t B, int64_t L, int64_t P);
int lrx_mimo_fwd_ps(int dtype, const void* lam, const void* delta, const void* deltas, int scheme, const void* bu,
                    void* x, int64_t B, int64_t L, int64_t P, void* workspace, size_t workspace_bytes, void* stream);
int lrx_mimo_bwd_ps(int dtype, const void* lam, const void* delta, const void* deltas, int scheme, const void* bu,
                    const void* x, const void* gx, void* gbu, void* glam_part, void* gdl_part, int64_t B, int64_t L,
                    int64_t P, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Fused MIMO projection + scan (S5 / LRU, constant steps, fp32;
 * layers.py:650-704 _stream_build / _shared_tape_forward and the pullbacks
 * _mimo_head_pullback / _mimo_input_pullback, autograd.py:113-140) ----
 * One kernel per direction: the tcgen05 3xTF32 projection lands in TMEM with
 * the state on the TMEM lane and is scanned there (bu / gx never reach HBM).
 * A, A_lo [256, m] = the projection's [2P, m] rows permuted to
 * [Re rows p (128, zero padded) ; Im rows p (128)] and their TF32 low parts.
 * Forward:  x = scan(abar, scale * (u A^T)) [B, L, P] complex; bu (or NULL)
 *           receives u A^T.
 * Backward: gx = alpha gy A^T, g_k = gx_k + conj(abar) g_{k+1};
 *           gbu = conj(scale) g; ga_part [units, P] complex = sum_k g
 *           conj(x_{k-1}) per unit (units = lrx_mimo_fused_units: B x
 *           ceil(L / 128)), summed by the caller.  d scale = sum_k conj(bu_k)
 *           g_k is the caller's: sum_h conj(W[p, h]) (gbu^T u)[p, h] /
 *           conj(scale_p) from its weight-gradient GEMM (bu is not needed).
 * Requires P <= 128, m % 16 == 0, L <= 8192 (LRX_ERR_UNSUPPORTED otherwise:
 * the separate GEMM + lrx_mimo_fwd / bwd path).  Workspace:
 * lrx_mimo_fused_workspace_bytes. */
int lrx_mimo_fused_workspace_bytes(int64_t B, int64_t L, int64_t P, int64_t* bytes);
int lrx_mimo_fused_units(int64_t B, int64_t L, int64_t* units);
int lrx_mimo_fused_fwd(const void* A, const void* A_lo, const void* u, const void* abar, const void* scale, void* x,
                       void* bu, int64_t B, int64_t L, int64_t m, int64_t P, void* workspace, size_t workspace_bytes,
                       void* stream);
int lrx_mimo_fused_bwd(const void* A, const void* A_lo, const void* gy, float alpha, const void* abar,
                       const void* scale, const void* x, void* gbu, void* ga_part, int64_t B, int64_t L, int64_t m,
                       int64_t P, void* workspace, size_t workspace_bytes, void* stream);

/* ---- bf16 <-> fp32 conversion of activation planes (n elements, 16-byte
 * aligned): the bf16 layers' fp32 GEMM operands and results. */
int lrx_cast(int dtype_in, int dtype_out, const void* in, void* out, int64_t n, void* stream);

/* ---- S4D coefficient work (constant steps), one launch each way ----------
 * S4D._lam / scheme_factors and the coefficient part of S4D._backward through
 * scheme_partials (layers.py:382-386, 520-546; discretize.py:59-93;
 * autograd.py:186-211), in f64 on the device: parameters [H, N] (log_delta
 * [H]) of the layer dtype (F32 / F64) -> abar, w = scale b [H, N] complex of
 * that precision; backward from the fused kernel's gabar / gw sums to the
 * parameter gradients (N <= 64). */
int lrx_s4d_coef(int dtype, int scheme, const void* lambda_re_log, const void* lambda_im, const void* b_re,
                 const void* b_im, const void* log_delta, int64_t H, int64_t N, void* abar, void* w, void* stream);
int lrx_s4d_coef_grads(int dtype, int scheme, const void* lambda_re_log, const void* lambda_im, const void* b_re,
                       const void* b_im, const void* log_delta, const void* gabar, const void* gpsi, int64_t H,
                       int64_t N, void* g_lambda_re_log, void* g_lambda_im, void* g_b_re, void* g_b_im,
                       void* g_log_delta, void* stream);

/* ---- MIMO LTI coefficient work (S5 / LRU), one launch each way ------------
 * Replaces the parameter-sized torch glue of S5._abar_scale / LRU._abar_scale
 * (layers.py:823-834, 936-943) and the coefficient + B/C gradient assembly of
 * S5._backward / LRU._backward (layers.py:836-895, 945-980) with
 * scheme_partials (autograd.py:186-211).
 * kind 0 = S5 (p0 lambda_re_log, p1 lambda_im, p2 log_delta; scheme ZOH or
 * DIRAC: bilinear keeps its host-side singular check), kind 1 = LRU (p0
 * nu_log, p1 theta_log, p2 gamma_log).  dtype = parameter dtype (F32 / F64);
 * abar, scale: complex [P] of that precision; extra: f64 [P][8] kept for the
 * gradient call; wbt [2P,m], wb [m,2P], wct [m,2P], wgt [2P,m]: real layouts
 * of B [P,m] and C [m,P] for the projection GEMMs, and wbf [256,m] = B in
 * the lrx_mimo_fused_fwd layout (Re rows p, Im rows 128 + p, zero rows past
 * P; P <= 128) and wgf [256,m] = wgt in that layout (lrx_mimo_fused_bwd)
 * (any may be NULL); with lo_planes (F32 only) each is followed
 * by a second plane holding the 3xTF32 low parts v - tf32(v) (the Bt_lo
 * operand of lrx_gemm_f32). */
int lrx_mimo_coef(int kind, int scheme, int dtype, const void* p0, const void* p1, const void* p2, const void* b_re,
                  const void* b_im, const void* c_re, const void* c_im, int64_t P, int64_t m, void* abar, void* scale,
                  double* extra, void* wbt, void* wb, void* wct, void* wgt, void* wbf, void* wgf, int lo_planes,
                  void* stream);
/* ga, gsc: complex [ga_rows, P] / [gsc_rows, P] partial rows of sum g
 * conj(x_prev) and sum conj(bu) g (the scans' per-chunk partials; summed
 * here in f64, fixed order); R [m,2P] = gy^T x, R2 [2P,m] = gbu^T u.  gsc
 * may be NULL (no bu stored, after
 * lrx_mimo_fused_fwd): then gsc = sum_h conj(B[p,h]) R2c[p,h] / conj(scale_p)
 * from b_re / b_im [P,m].  g0..g2: [P] coefficient grads (keys as p0..p2),
 * gb_re/gb_im [P,m], gc_re/gc_im [m,P] = out_scale (R_re, -R_im). */
int lrx_mimo_coef_grads(int kind, int scheme, int dtype, const void* p0, const void* p1, const void* p2,
                        const double* extra, const void* ga, int64_t ga_rows, const void* gsc, int64_t gsc_rows,
                        const void* R, const void* R2, const void* b_re, const void* b_im, double out_scale,
                        void* g0, void* g1, void* g2, void* gb_re, void* gb_im, void* gc_re, void* gc_im, int64_t P,
                        int64_t m, void* stream);
/* S6: x[B,D,N] compute precision; u, y io dtype; pre [B,D] = the delta
 * projection (bias not added), Bk, Ck [B,N] compute precision. */
int lrx_s6_step(int io_dtype, void* x, const void* u, const void* pre, const void* Bk, const void* Ck,
                const void* b_delta, const void* a_log, const void* Dskip, void* y, int64_t B, int64_t D, int64_t N,
                void* stream);
/* RG-LRU: x[B,W] compute precision; u, qr, qi, y io dtype. */
int lrx_rglru_step(int io_dtype, void* x, const void* u, const void* qr, const void* qi, const void* lambda_param,
                   const void* b_r, const void* b_i, void* y, int64_t B, int64_t W, void* stream);
/* S6 token in two kernels: the input projections p1 = u W_delta [B, R],
 * B_k = u W_B^T, C_k = u W_C^T [B, N] into proj_ws ([B][R + 2N] fp32, caller
 * allocated), then pre = p1 W_delta_proj and the update (fp32 weights;
 * batch <= 16, f32 / bf16 I/O; LRX_ERR_UNSUPPORTED otherwise). */
int lrx_s6_step_fused(int io_dtype, void* x, const void* u, const void* W_delta, const void* W_delta_proj,
                      const void* W_B, const void* W_C, const void* b_delta, const void* a_log, const void* Dskip,
                      void* y, void* proj_ws, int64_t B, int64_t D, int64_t R, int64_t N, void* stream);
/* RG-LRU token in one kernel: the gate GEMVs qr = u W_r^T, qi = u W_i^T
 * (fp32 weights [W, W]) fused with the update; batch <= 16, W % 8 == 0,
 * f32 / bf16 I/O (LRX_ERR_UNSUPPORTED otherwise: use lrx_rglru_step). */
int lrx_rglru_step_fused(int io_dtype, void* x, const void* u, const void* W_r, const void* W_i,
                         const void* lambda_param, const void* b_r, const void* b_i, void* y, int64_t B, int64_t W,
                         void* stream);

/* ------------------------------------------------------------------------ *
 * fp32 GEMM on the tcgen05 tensor cores with the 3xTF32 split (the dense
 * projections of S5 / LRU, layers.py:650-704):
 *   C[M,N] = act(alpha A[M,K] Bt[N,K]^T + bias[n]) + (colscale ? colscale[n] : beta) Cin[M,N]
 * fp32 row-major, K contiguous in both A and Bt; Bt_lo = Bt - tf32(Bt) is the
 * caller's pre-split low part of the (small) right operand.  Cin / bias may
 * be NULL, Cin may alias C; act 0 identity / 1 softplus / 2 sigmoid (the S6
 * delta projection's softplus(. + b_delta), layers.py:1020-1027, fused).
 * Rows must be 16-byte aligned (K % 4 == 0).
 * ------------------------------------------------------------------------ */
int lrx_gemm_f32(const void* A, const void* Bt, const void* Bt_lo, void* C, const void* Cin, const void* colscale,
                 const void* bias, int act, int64_t M, int64_t N, int64_t K, float alpha, float beta, void* stream);
/* Reduction ("TN") GEMM for the weight gradients: with A [K, M] and B [K, N]
 * row-major (K = tokens, long), part[s, M, N] = alpha sum_{k in split s}
 * A[k, m] B[k, n] for s < n_splits; sum the split axis with lrx_reduce_rows.
 * M, N % 4 == 0. */
int lrx_gemm_f32_tn_splits(int64_t M, int64_t N, int64_t K, int64_t* n_splits);
int lrx_gemm_f32_tn(const void* A, const void* B, void* part, int64_t M, int64_t N, int64_t K, float alpha,
                    void* stream);

/* ------------------------------------------------------------------------ *
 * bf16 GEMM on the tcgen05 tensor cores (kind::f16, fp32 accumulation) with a
 * fused epilogue, for the input projections of the bf16-I/O layers (S6
 * _projections layers.py:1020-1027: B_k, C_k, the low-rank delta input;
 * RG-LRU _gates layers.py:1212-1218):
 *   C[M,N] = act(alpha A[M,K] Bt[N,K]^T + bias[n]) + beta Cin[M,N]
 * A, Bt bf16 row-major K-contiguous; C fp32 (or bf16 with out_bf16, then no
 * Cin), Cin fp32 (Cin / bias may be NULL);
 * act: 0 identity, 1 softplus (numerics.py:36-39), 2 sigmoid (:97-105).
 * K % 8 == 0, N % 4 == 0 (N % 8 == 0 for bf16 out), 16-byte aligned rows.  Replaces the numpy matmuls
 * of those reference lines (cuBLAS in round 1).
 * ------------------------------------------------------------------------ */
#define LRX_ACT_NONE 0
#define LRX_ACT_SOFTPLUS 1
#define LRX_ACT_SIGMOID 2
int lrx_gemm_bf16(const void* A, const void* Bt, void* C, const void* Cin, const void* bias, int64_t M, int64_t N,
                  int64_t K, float alpha, float beta, int act, int out_bf16, void* stream);

/* ------------------------------------------------------------------------ *
 * MIMO complex diagonal scan for S5 / LRU (layers.py:616-980): the recurrence
 * between the dense projections bu = B u and y = Re(C x) (cuBLAS GEMMs):
 *   x_k[b,p] = abar[p] x_{k-1} + scale[p] bu_k[b,p]        (lanes b*P + p)
 * bu, x: [B, L, P] complex (C64/C128); abar, scale: [P] complex.
 * ------------------------------------------------------------------------ */
size_t lrx_mimo_workspace_bytes(int dtype, int64_t B, int64_t L, int64_t P);
int lrx_mimo_fwd(int dtype, const void* abar, const void* scale, const void* bu, void* x, int64_t B,
                 int64_t L, int64_t P, void* workspace, size_t workspace_bytes, void* stream);
/* Reverse pass, fused with the LTI coefficient reductions
 * (_MIMOBase._mimo_input_pullback 701-704, S5._backward 836-895,
 * LRU._backward 945-980):
 *   g_k = gx_k + conj(abar) g_{k+1};  gbu = conj(scale) g  -> gbu [B,L,P]
 *   gabar_part[c, b*P+p] = sum_{k in chunk c} g_k conj(x_{k-1})
 *   gscale_part[c, b*P+p] = sum_{k in chunk c} conj(bu_k) g_k   (not written
 *   when bu is NULL: the caller takes d scale from its weight-gradient GEMM,
 *   as after lrx_mimo_fused_fwd, which stores no bu)
 * (reduce the [n_chunks*B, P] partials with lrx_reduce_rows). */
int lrx_mimo_chunking(int dtype, int64_t B, int64_t L, int64_t P, int64_t* chunk_len, int64_t* n_chunks);
size_t lrx_mimo_bwd_workspace_bytes(int dtype, int64_t B, int64_t L, int64_t P);
int lrx_mimo_bwd(int dtype, const void* abar, const void* scale, const void* bu, const void* x,
                 const void* gx, void* gbu, void* gabar_part, void* gscale_part, int64_t B, int64_t L,
                 int64_t P, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * Deterministic fixed-order reduction: out[j] = sum_r in[r, j]  (dtype any
 * of F32/F64/C64/C128).  Used for every parameter-gradient partial above so
 * training is bitwise reproducible (test_acceptance.py:249-250).
 * ------------------------------------------------------------------------ */
int lrx_reduce_rows(int dtype, const void* in, void* out, int64_t R, int64_t N, void* stream);
/* Same with row groups spread over the GPU (long columns): out[j] =
 * sum_r in[r,j] (* in2[r,j] when in2 is not NULL: a column-wise dot
 * product).  Workspace: lrx_reduce_rows_ws_bytes() (0 = none needed). */
size_t lrx_reduce_rows_ws_bytes(int dtype, int64_t R, int64_t N);
int lrx_reduce_rows_ws(int dtype, const void* in, const void* in2, void* out, int64_t R, int64_t N, void* ws,
                       size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LRX_H */
