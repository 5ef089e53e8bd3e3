// Is straight-line code fetch-bound at kernel start?  A kernel with a long
// unrolled body, timed by globaltimer from entry to exit, on repeated launches.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
template <int N>
__global__ void body(float* out, unsigned long long* t, float s) {
    unsigned long long t0 = gt();
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = s * (threadIdx.x + i);
#pragma unroll
    for (int i = 0; i < N; ++i) a[i & 7] = a[i & 7] * 1.0001f + (float)i;
    unsigned long long t1 = gt();
    float r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}
template <int N>
void run(float* out, unsigned long long* t) {
    for (int rep = 0; rep < 5; ++rep) { body<N><<<148, 128>>>(out, t, 1.0f); cudaDeviceSynchronize(); }
    double m = 0; for (int i = 0; i < 148; ++i) m += t[i];
    printf("N=%5d FFMA straight-line: %.0f ns (%.2f ns per instr; ~%.0f KB code)\n", N, m / 148, m / 148 / N, N * 16 / 1024.0);
}
int main() {
    float* out; unsigned long long* t;
    cudaMalloc(&out, 1 << 20); cudaMallocManaged(&t, 148 * 8);
    run<256>(out, t); run<1024>(out, t); run<2048>(out, t); run<4096>(out, t); run<8192>(out, t);
    return 0;
}
