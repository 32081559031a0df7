// bf16 <-> fp32 conversion of activation planes (the bf16 layers' fp32
// projection / gradient GEMMs read and write fp32): 8 elements per thread per
// step with 16-byte bf16 and 2 x 16-byte fp32 accesses, grid-stride over the
// GPU (streaming, HBM-bound).  torch's generic conversion ran at ~2.3 TB/s on
// the S6 layer's 805 MB planes (profiles/r2a_launches_s6_layer.json).
#include <cuda_bf16.h>

#include "lrx_host.h"

namespace lrx {
namespace cast {

__global__ void __launch_bounds__(256) bf16_to_f32(const uint4* __restrict__ in, float4* __restrict__ out, int64_t n8) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
        const uint4 v = __ldcs(in + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        float f[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            f[2 * k] = __uint_as_float(w[k] << 16);
            f[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
        }
        __stcs(out + 2 * i, make_float4(f[0], f[1], f[2], f[3]));
        __stcs(out + 2 * i + 1, make_float4(f[4], f[5], f[6], f[7]));
    }
}

__global__ void __launch_bounds__(256) f32_to_bf16(const float4* __restrict__ in, uint4* __restrict__ out, int64_t n8) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
        const float4 a = __ldcs(in + 2 * i), b = __ldcs(in + 2 * i + 1);
        const __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w);
        const __nv_bfloat162 p2 = __floats2bfloat162_rn(b.x, b.y), p3 = __floats2bfloat162_rn(b.z, b.w);
        __stcs(out + i, make_uint4(*reinterpret_cast<const uint32_t*>(&p0), *reinterpret_cast<const uint32_t*>(&p1),
                                   *reinterpret_cast<const uint32_t*>(&p2), *reinterpret_cast<const uint32_t*>(&p3)));
    }
}

__global__ void tail_kernel(const void* in, void* out, int64_t i0, int64_t n, int to_f32) {
    const int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (to_f32) static_cast<float*>(out)[i] = __bfloat162float(static_cast<const __nv_bfloat16*>(in)[i]);
    else static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(static_cast<const float*>(in)[i]);
}

}  // namespace cast
}  // namespace lrx

using namespace lrx;

extern "C" {

int lrx_cast(int dtype_in, int dtype_out, const void* in, void* out, int64_t n, void* stream) {
    LRX_REQUIRE(n >= 0, LRX_ERR_SHAPE, "cast: negative size");
    const bool to_f32 = dtype_in == LRX_BF16 && dtype_out == LRX_F32;
    LRX_REQUIRE(to_f32 || (dtype_in == LRX_F32 && dtype_out == LRX_BF16), LRX_ERR_VALUE,
                "cast: bf16 -> f32 or f32 -> bf16 only");
    LRX_REQUIRE(((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0, LRX_ERR_VALUE,
                "cast: 16-byte aligned buffers required");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n8 = n / 8;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n8, 256), (int64_t)sms * 8));
    int launches = 0;
    if (n8 > 0) {
        if (to_f32) cast::bf16_to_f32<<<grid, 256, 0, st>>>((const uint4*)in, (float4*)out, n8);
        else cast::f32_to_bf16<<<grid, 256, 0, st>>>((const float4*)in, (uint4*)out, n8);
        ++launches;
    }
    if (n8 * 8 < n) {
        cast::tail_kernel<<<1, 8, 0, st>>>(in, out, n8 * 8, n, to_f32);
        ++launches;
    }
    return launches ? launched("lrx_cast", launches) : LRX_OK;
}

}  // extern "C"
