// Per-kernel cost of a chain of small dependent kernels replayed from a CUDA
// graph, with and without programmatic dependent launch (PDL): the launch
// floor that bounds the LRU C1 step (~18 kernels of a few us each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl pdl.cu
#include <cstdio>
#include <cuda_runtime.h>

// each CTA reads what the previous kernel wrote (a real dependency), does a
// little smem work (prologue) and writes its slice
__global__ void step_kernel(const float* in, float* out, int n, int pdl, int early) {
    __shared__ float s[256];
    s[threadIdx.x] = threadIdx.x * 0.5f;  // prologue independent of the predecessor
    __syncthreads();
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (pdl && early) asm volatile("griddepcontrol.launch_dependents;");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i] * 0.999f + s[threadIdx.x ^ 1];
}

int main() {
    const int n = 148 * 256 * 4;
    float *a, *b;
    cudaMalloc(&a, n * 4);
    cudaMalloc(&b, n * 4);
    cudaMemset(a, 0, n * 4);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int grid : {148, 592}) {
        for (int mode = 0; mode < 3; ++mode) {  // 0 plain, 1 PDL (implicit trigger), 2 PDL + early trigger
            const int chain = 20;
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
            for (int k = 0; k < chain; ++k) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = st;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = mode ? 1 : 0;
                const float* in = (k & 1) ? b : a;
                float* out = (k & 1) ? a : b;
                cudaLaunchKernelEx(&cfg, step_kernel, in, out, grid * 256 < n ? grid * 256 : n, mode ? 1 : 0,
                                   mode == 2 ? 1 : 0);
            }
            cudaStreamEndCapture(st, &g);
            if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
                printf("instantiate failed mode %d\n", mode);
                continue;
            }
            for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, st);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, st);
            const int reps = 50;
            for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, st);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("grid %4d %-22s: %.2f us per kernel (chain of %d in one graph)\n", grid,
                   mode == 0 ? "plain" : mode == 1 ? "PDL" : "PDL + early trigger", ms * 1e3 / reps / chain, chain);
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
