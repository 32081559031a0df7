// S6 kernels instantiated for bf16 I/O (see lrx_s6_impl.cuh).
#include "lrx_s6_impl.cuh"

namespace lrx {
namespace s6 {

int fwd_bf16(LRX_S6_FWD_PARAMS) {
    return fwd_t<__nv_bfloat16, float>(u, pre, bd, al, Bk, Ck, Dk, x0, y, ckpt, B, L, D, N, st);
}

int bwd_bf16(LRX_S6_BWD_PARAMS) {
    return bwd_t<__nv_bfloat16, float>(u, pre, bd, al, Bk, Ck, Dk, ckpt, gy, h_in, gu, gpre, gBp, gCp, gap, gDp, gbp, h_out, B, L,
                            D, N, st);
}

}  // namespace s6
}  // namespace lrx
