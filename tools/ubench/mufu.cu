// MUFU / FMA throughput microbenchmark: ops per clock per SM for ex2, lg2, rcp, and FFMA.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters, float seed) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = seed + threadIdx.x * 1e-3f + i * 1e-2f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
            if (OP == 1) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
            if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
            if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(v[i]));
            if (OP == 4) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(*reinterpret_cast<unsigned*>(&v[i])));
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 12345.f) out[0] = s;
}
int main() {
    float* o; cudaMalloc(&o, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char* names[] = {"ex2.f32", "lg2.f32", "rcp.f32", "ffma", "ex2.f16x2"};
    for (int op = 0; op < 5; ++op) {
        for (int threads : {256, 1024}) {
            int blocks = sms * (2048 / threads);
            int iters = 4096;
            void (*kf)(float*, int, float) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : k<4>;
            kf<<<blocks, threads>>>(o, 16, 0.5f);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            kf<<<blocks, threads>>>(o, iters, 0.5f);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * threads * iters * 8;
            printf("%-10s threads/blk %4d: %.3f Tops/s = %.2f per clk per SM (at %d MHz nominal)\n", names[op], threads,
                   ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
