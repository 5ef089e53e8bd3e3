// Throughput microbenchmarks: DADD / FADD / F2F per SM (full occupancy, independent chains).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void add_thr(T* out, int n) {
    T a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const T c = (T)1.0000001;
    for (int i = 0; i < n; ++i) {
        a0 += c; a1 += c; a2 += c; a3 += c; a4 += c; a5 += c; a6 += c; a7 += c;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void cvt_thr(float* out, int n) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    double d = 0;
    for (int i = 0; i < n; ++i) {
        d += (double)a0; d += (double)a1; d += (double)a2; d += (double)a3;
        a0 += 1.f; a1 += 1.f; a2 += 1.f; a3 += 1.f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)d;
}
int main() {
    int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* od; float* of; cudaMalloc(&od, 8 << 24); cudaMalloc(&of, 4 << 24);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int n = 4096, blocks = sms * 4, threads = 256;
    float ms;
    add_thr<double><<<blocks, threads>>>(od, n); cudaEventRecord(e0); add_thr<double><<<blocks, threads>>>(od, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); double dflops = 8.0 * n * blocks * threads / (ms * 1e-3);
    add_thr<float><<<blocks, threads>>>(of, n); cudaEventRecord(e0); add_thr<float><<<blocks, threads>>>(of, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); double fflops = 8.0 * n * blocks * threads / (ms * 1e-3);
    cvt_thr<<<blocks, threads>>>(of, n); cudaEventRecord(e0); cvt_thr<<<blocks, threads>>>(of, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); double cvt = 4.0 * n * blocks * threads / (ms * 1e-3);
    printf("DADD %.2f T/s (%.1f per SM per clk@1.9GHz)  FADD %.2f T/s (%.1f)  F2F+DADD %.2f T/s (%.1f)\n",
           dflops / 1e12, dflops / sms / 1.9e9, fflops / 1e12, fflops / sms / 1.9e9, cvt / 1e12, cvt / sms / 1.9e9);
    return 0;
}
