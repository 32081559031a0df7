// MUFU ex2 throughput vs independent chains per thread (the round-1 mufu.cu
// ran 8 dependent chains, which is latency-bound): ex2 ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(float* out, int iters, float seed) {
    float v[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = seed + threadIdx.x * 1e-6f + i * 1e-3f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += v[i];
    if (s == 12345.f) out[0] = s;
}
template <int CH>
void run(float* o, int sms, int threads, int warps_per_sm) {
    int blocks = sms * warps_per_sm * 32 / threads;
    int iters = 32768 / CH;
    k<CH><<<blocks, threads>>>(o, 16, 0.5f);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<CH><<<blocks, threads>>>(o, iters, 0.5f);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * iters * CH;
    printf("ex2 chains %2d warps/SM %2d: %.3f Tex2/s = %.1f per clk per SM at 1.965 GHz\n", CH, warps_per_sm,
           ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
    float* o; cudaMalloc(&o, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {8, 16, 32, 64}) { run<8>(o, sms, 256, w); run<16>(o, sms, 256, w); run<32>(o, sms, 256, w); }
    return 0;
}
