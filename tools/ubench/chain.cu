// Launch/handoff floor: CUDA graph of K back-to-back kernels, with and without PDL.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k(int* p, int early) {
    if (early) asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}
int main() {
    int* p; cudaMalloc(&p, 4); cudaMemset(p, 0, 4);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const int K = 1000;
    for (int grid : {1, 144, 296}) {
        for (int mode = 0; mode < 3; ++mode) {  // 0: no PDL, 1: PDL attr, wait at start, 2: PDL + early trigger
            cudaGraph_t g; cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < K; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.stream = s;
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                a[0].val.programmaticStreamSerializationAllowed = mode > 0;
                cfg.attrs = a; cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, empty_k, p, mode == 2 ? 1 : 0);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("grid %3d mode %d: %.3f us per kernel\n", grid, mode, ms * 1e3 / K);
            cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
