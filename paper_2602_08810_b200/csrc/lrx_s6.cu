// S6 selective scan: C-ABI entry points.  fp32-compute I/O (bf16, f32) with
// d_state 16 runs the v3 kernels (lrx_s6v3.cu: TMA tiles, channel-pair
// threads, time segments); f64 and other state sizes run the generic kernels
// (lrx_s6_impl.cuh, instantiated per I/O dtype in lrx_s6_{f32,bf16,f64}.cu).
#include "lrx_s6_impl.cuh"

using namespace lrx;

namespace lrx {
namespace s6v3 {
struct Geo {
    int64_t n_ck, n_dblk, n_seg, seg_len, ws_bytes;
};
bool eligible(int io, int64_t D, int64_t N);
Geo geometry(int64_t B, int64_t L, int64_t D);
template <typename IO>
int fwd(const void*, const void*, const void*, const void*, const void*, const void*, const void*, const void*,
        void*, void*, int64_t, int64_t, int64_t, void*, int64_t, int, cudaStream_t);
template <typename IO>
int bwd(const void*, const void*, const void*, const void*, const void*, const void*, const void*, const void*,
        const void*, const void*, void*, void*, void*, void*, void*, void*, void*, void*, int64_t, int64_t, int64_t,
        void*, int64_t, int, cudaStream_t);
template <typename IO>
int fwd_carry(const void*, const void*, const void*, const void*, const void*, void*, void*, int64_t, int64_t,
              int64_t, void*, int64_t, cudaStream_t);
template <typename IO>
int bwd_carry(const void*, const void*, const void*, const void*, const void*, void*, void*, int64_t, int64_t,
              int64_t, void*, int64_t, cudaStream_t);
}  // namespace s6v3
}  // namespace lrx

extern "C" {

int lrx_s6_geometry(int io_dtype, int64_t B, int64_t L, int64_t D, int64_t N, int64_t* out) {
    LRX_REQUIRE(B >= 1 && L >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    LRX_REQUIRE(io_dtype == LRX_F32 || io_dtype == LRX_BF16 || io_dtype == LRX_F64, LRX_ERR_VALUE,
                "s6: unsupported io dtype %d", io_dtype);
    if (s6v3::eligible(io_dtype, D, N)) {
        const s6v3::Geo g = s6v3::geometry(B, L, D);
        out[0] = 8;
        out[1] = g.n_ck + 1;
        out[2] = g.n_dblk;
        out[3] = g.n_seg;
        out[4] = g.n_seg * B;
        out[5] = g.ws_bytes;
        return LRX_OK;
    }
    int ck = 0, nck = 0, ndb = 0, ns;
    if (io_dtype == LRX_F64) ns = s6::geom_rt<double>(L, D, N, &ck, &nck, &ndb);
    else ns = s6::geom_rt<float>(L, D, N, &ck, &nck, &ndb);
    LRX_REQUIRE(ns > 0, LRX_ERR_UNSUPPORTED, "s6: d_state %lld > 64 is not compiled", (long long)N);
    out[0] = ck;
    out[1] = nck + 1;  // the last slot receives the final state
    out[2] = ndb;
    out[3] = 1;
    out[4] = B;
    out[5] = 0;
    return LRX_OK;
}

int lrx_s6_fwd(int io_dtype, const void* u, const void* pre, const void* b_delta, const void* a_log, const void* Bk,
               const void* Ck, const void* Dskip, const void* x0, void* y, void* ckpt, int64_t B, int64_t L,
               int64_t D, int64_t N, void* ws, int64_t ws_bytes, int flags, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    if (s6v3::eligible(io_dtype, D, N)) {
        if (io_dtype == LRX_BF16)
            return s6v3::fwd<__nv_bfloat16>(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0, y, ckpt, B, L, D, ws,
                                            ws_bytes, flags, st);
        return s6v3::fwd<float>(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0, y, ckpt, B, L, D, ws, ws_bytes, flags,
                                st);
    }
    LRX_REQUIRE(!(flags & LRX_S6_DELTA_IN), LRX_ERR_UNSUPPORTED,
                "s6: LRX_S6_DELTA_IN needs the v3 kernels (d_state 16, f32 / bf16 I/O)");
    switch (io_dtype) {
        case LRX_F32: return s6::fwd_f32(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0, y, ckpt, B, L, D, N, st);
        case LRX_BF16: return s6::fwd_bf16(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0, y, ckpt, B, L, D, N, st);
        case LRX_F64: return s6::fwd_f64(u, pre, b_delta, a_log, Bk, Ck, Dskip, x0, y, ckpt, B, L, D, N, st);
    }
    set_error("s6: unsupported io dtype %d", io_dtype);
    return LRX_ERR_VALUE;
}

int lrx_s6_bwd(int io_dtype, const void* u, const void* pre, const void* b_delta, const void* a_log, const void* Bk,
               const void* Ck, const void* Dskip, const void* ckpt, const void* gy, const void* h_in, void* gu_local,
               void* gpre, void* gBk_part, void* gCk_part, void* ga_part, void* gD_part, void* gb_part, void* h_out,
               int64_t B, int64_t L, int64_t D, int64_t N, void* ws, int64_t ws_bytes, int flags, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
    if (s6v3::eligible(io_dtype, D, N)) {
        if (io_dtype == LRX_BF16)
            return s6v3::bwd<__nv_bfloat16>(u, pre, b_delta, a_log, Bk, Ck, Dskip, ckpt, gy, h_in, gu_local, gpre,
                                            gBk_part, gCk_part, ga_part, gD_part, gb_part, h_out, B, L, D, ws,
                                            ws_bytes, flags, st);
        return s6v3::bwd<float>(u, pre, b_delta, a_log, Bk, Ck, Dskip, ckpt, gy, h_in, gu_local, gpre, gBk_part,
                                gCk_part, ga_part, gD_part, gb_part, h_out, B, L, D, ws, ws_bytes, flags, st);
    }
    LRX_REQUIRE(!(flags & LRX_S6_DELTA_IN), LRX_ERR_UNSUPPORTED,
                "s6: LRX_S6_DELTA_IN needs the v3 kernels (d_state 16, f32 / bf16 I/O)");
    switch (io_dtype) {
        case LRX_F32:
            return s6::bwd_f32(u, pre, b_delta, a_log, Bk, Ck, Dskip, ckpt, gy, h_in, gu_local, gpre, gBk_part,
                               gCk_part, ga_part, gD_part, gb_part, h_out, B, L, D, N, st);
        case LRX_BF16:
            return s6::bwd_bf16(u, pre, b_delta, a_log, Bk, Ck, Dskip, ckpt, gy, h_in, gu_local, gpre, gBk_part,
                                gCk_part, ga_part, gD_part, gb_part, h_out, B, L, D, N, st);
        case LRX_F64:
            return s6::bwd_f64(u, pre, b_delta, a_log, Bk, Ck, Dskip, ckpt, gy, h_in, gu_local, gpre, gBk_part,
                               gCk_part, ga_part, gD_part, gb_part, h_out, B, L, D, N, st);
    }
    set_error("s6: unsupported io dtype %d", io_dtype);
    return LRX_ERR_VALUE;
}

int lrx_s6_fwd_carry(int io_dtype, const void* u, const void* pre, const void* b_delta, const void* a_log,
                     const void* Bk, void* x_agg, void* sd_agg, int64_t B, int64_t L, int64_t D, int64_t N, void* ws,
                     int64_t ws_bytes, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    LRX_REQUIRE(s6v3::eligible(io_dtype, D, N), LRX_ERR_UNSUPPORTED,
                "s6 carry: needs f32/bf16 io, d_state 16 and an aligned channel count");
    cudaStream_t st = (cudaStream_t)stream;
    if (io_dtype == LRX_BF16)
        return s6v3::fwd_carry<__nv_bfloat16>(u, pre, b_delta, a_log, Bk, x_agg, sd_agg, B, L, D, ws, ws_bytes, st);
    return s6v3::fwd_carry<float>(u, pre, b_delta, a_log, Bk, x_agg, sd_agg, B, L, D, ws, ws_bytes, st);
}

int lrx_s6_bwd_carry(int io_dtype, const void* gy, const void* pre, const void* b_delta, const void* a_log,
                     const void* Ck, void* h_agg, void* sd_agg, int64_t B, int64_t L, int64_t D, int64_t N, void* ws,
                     int64_t ws_bytes, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    LRX_REQUIRE(s6v3::eligible(io_dtype, D, N), LRX_ERR_UNSUPPORTED,
                "s6 carry: needs f32/bf16 io, d_state 16 and an aligned channel count");
    cudaStream_t st = (cudaStream_t)stream;
    if (io_dtype == LRX_BF16)
        return s6v3::bwd_carry<__nv_bfloat16>(gy, pre, b_delta, a_log, Ck, h_agg, sd_agg, B, L, D, ws, ws_bytes, st);
    return s6v3::bwd_carry<float>(gy, pre, b_delta, a_log, Ck, h_agg, sd_agg, B, L, D, ws, ws_bytes, st);
}

}  // extern "C"
