// Achievable HBM bandwidth for the RG-LRU stream mixes (no arithmetic):
//   copy   1 read  + 1 write   (the MEASURED_PEAKS copy test)
//   fwd    3 reads + 1 write   (u, qr, qi -> y)
//   bwd    5 reads + 3 writes  (u, qr, qi, gy, y -> gu, gqr, gqi)
// Grid-stride float4 streams over C4-sized arrays (64 x 16384 x 2560 fp32 =
// 10.7 GB each; --small for a 1/8 size), best of 5 with CUDA events.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a streams.cu -o streams
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

template <int R, int W>
__global__ void __launch_bounds__(256) mix(const float4* const* in, float4* const* out, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float4 v = __ldcs(in[r] + i);
            s.x += v.x, s.y += v.y, s.z += v.z, s.w += v.w;
        }
#pragma unroll
        for (int w = 0; w < W; ++w) __stcs(out[w] + i, s);
    }
}

template <int R, int W>
static void run(const char* name, float4** bufs, long long n, int sms) {
    const float4** din;
    float4** dout;
    cudaMalloc(&din, sizeof(void*) * 8);
    cudaMalloc(&dout, sizeof(void*) * 8);
    cudaMemcpy(din, bufs, sizeof(void*) * R, cudaMemcpyHostToDevice);
    cudaMemcpy(dout, bufs + R, sizeof(void*) * W, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
        cudaEventRecord(a);
        mix<R, W><<<sms * 8, 256>>>(din, dout, n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 0 && ms < best) best = ms;
    }
    const double bytes = (double)(R + W) * n * 16;
    printf("%-5s %d reads + %d writes: %.3f ms  %.0f GB/s\n", name, R, W, best, bytes / best / 1e6);
    cudaFree(din);
    cudaFree(dout);
}

int main(int argc, char** argv) {
    long long elems = 64LL * 16384 * 2560;
    if (argc > 1 && !strcmp(argv[1], "--small")) elems /= 8;
    const long long n = elems / 4;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float4* bufs[8];
    for (int i = 0; i < 8; ++i) {
        if (cudaMalloc(&bufs[i], n * 16) != cudaSuccess) {
            printf("alloc failed\n");
            return 1;
        }
        cudaMemset(bufs[i], 0, n * 16);
    }
    run<1, 1>("copy", bufs, n, sms);
    run<3, 1>("fwd", bufs, n, sms);
    run<5, 3>("bwd", bufs, n, sms);
    run<4, 3>("bwd7", bufs, n, sms);
    return 0;
}
