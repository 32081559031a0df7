// S6 kernels instantiated for bf16 I/O (see lrx_s6_impl.cuh).
#include "lrx_s6_impl.cuh"

namespace lrx {
namespace s6 {

int fwd_bf16(const void* u, const void* pre, const void* bd, const void* al, const void* Bk, const void* Ck,
            const void* Dk, void* y, void* ckpt, int64_t B, int64_t L, int64_t D, int64_t N, cudaStream_t st) {
    return fwd_t<__nv_bfloat16, float>(u, pre, bd, al, Bk, Ck, Dk, y, ckpt, B, L, D, N, st);
}

int bwd_bf16(const void* u, const void* pre, const void* bd, const void* al, const void* Bk, const void* Ck,
            const void* Dk, const void* ckpt, const void* gy, void* gu, void* gpre, void* gBp, void* gCp, void* gap,
            void* gDp, void* gbp, int64_t B, int64_t L, int64_t D, int64_t N, cudaStream_t st) {
    return bwd_t<__nv_bfloat16, float>(u, pre, bd, al, Bk, Ck, Dk, ckpt, gy, gu, gpre, gBp, gCp, gap, gDp, gbp, B, L, D, N, st);
}

}  // namespace s6
}  // namespace lrx
