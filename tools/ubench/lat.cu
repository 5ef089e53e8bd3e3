// Microbenchmarks of the latencies that bound the BiQGEMM tail (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const float* __restrict__ buf, double* out, long long* cyc, int n) {
    long long t0 = clock64();
    // DADD dependent chain
    double a = out[0];
    for (int i = 0; i < n; ++i) a = a + 1.0000001;
    long long t1 = clock64();
    // FADD chain
    float f = (float)a;
    for (int i = 0; i < n; ++i) f = f * 1.0000001f + 0.5f;
    long long t2 = clock64();
    // dependent L2 loads (pointer chase through buf indices)
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) idx = __float_as_int(__ldcg(buf + idx)) & 0xfffff;
    long long t3 = clock64();
    // SHFL chain
    float s = f;
    for (int i = 0; i < n; ++i) s = __shfl_xor_sync(0xffffffff, s, 1) + 1.0f;
    long long t4 = clock64();
    // F2F chain
    float g = f;
    for (int i = 0; i < n; ++i) g = (float)((double)g * 1.5);
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    }
    out[1 + threadIdx.x] = a + f + idx + s + g;
}
int main() {
    float* buf; double* out; long long* cyc;
    cudaMalloc(&buf, 4 << 22); cudaMalloc(&out, 8 * 64); cudaMallocManaged(&cyc, 8 * 8);
    cudaMemset(buf, 0, 4 << 22); cudaMemset(out, 0, 8 * 64);
    int n = 1000;
    for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(buf, out, cyc, n); cudaDeviceSynchronize(); }
    printf("cycles per op: DADD %.1f  FFMA %.1f  LDG.cg(L2) %.1f  SHFL+FADD %.1f  F2F pair %.1f\n",
           cyc[0] / (double)n, cyc[1] / (double)n, cyc[2] / (double)n, cyc[3] / (double)n, cyc[4] / (double)n);
    return 0;
}
