// S6 kernels instantiated for f64 I/O (see lrx_s6_impl.cuh).
#include "lrx_s6_impl.cuh"

namespace lrx {
namespace s6 {

int fwd_f64(LRX_S6_FWD_PARAMS) {
    return fwd_t<double, double>(u, pre, bd, al, Bk, Ck, Dk, x0, y, ckpt, B, L, D, N, st);
}

int bwd_f64(LRX_S6_BWD_PARAMS) {
    return bwd_t<double, double>(u, pre, bd, al, Bk, Ck, Dk, ckpt, gy, h_in, gu, gpre, gBp, gCp, gap, gDp, gbp, h_out, B, L,
                            D, N, st);
}

}  // namespace s6
}  // namespace lrx
