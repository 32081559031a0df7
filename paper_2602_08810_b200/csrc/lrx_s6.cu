// S6 selective scan: C-ABI entry points (kernels: lrx_s6_impl.cuh, instantiated
// per I/O dtype in lrx_s6_{f32,bf16,f64}.cu).
#include "lrx_s6_impl.cuh"

using namespace lrx;

extern "C" {

int lrx_s6_ckpt_len(int io_dtype, int64_t L, int64_t D, int64_t N, int64_t* ckpt_len, int64_t* n_ckpt,
                    int64_t* n_dblk) {
    LRX_REQUIRE(L >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    int ck = 0, nck = 0, ndb = 0, ns;
    if (io_dtype == LRX_F64) ns = s6::geom_rt<double>(L, D, N, &ck, &nck, &ndb);
    else ns = s6::geom_rt<float>(L, D, N, &ck, &nck, &ndb);
    LRX_REQUIRE(ns > 0, LRX_ERR_UNSUPPORTED, "s6: d_state %lld > 64 is not compiled", (long long)N);
    *ckpt_len = ck;
    *n_ckpt = nck + 1;  // the last slot receives the final state
    *n_dblk = ndb;
    return LRX_OK;
}

int lrx_s6_fwd(int io_dtype, const void* u, const void* pre, const void* b_delta, const void* a_log, const void* Bk,
               const void* Ck, const void* Dskip, const void* x0, void* y, void* ckpt, int64_t B, int64_t L,
               int64_t D, int64_t N, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
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
               int64_t B, int64_t L, int64_t D, int64_t N, void* stream) {
    LRX_REQUIRE(B >= 1 && L >= 1 && D >= 1 && N >= 1, LRX_ERR_SHAPE, "bad extents");
    cudaStream_t st = (cudaStream_t)stream;
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

}  // extern "C"
