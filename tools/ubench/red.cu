// Reproduce the cluster reduction's global pattern: 8 ranks write partials
// [rank][plane][row] (stcg), cluster barrier, thread-per-row loads of 8x3
// partials at 48 KB stride.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
template <int MODE>
__global__ void __cluster_dims__(8, 1, 1) k(float* part, const float* alpha, float* y, unsigned long long* out) {
    uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int cid = blockIdx.x / 8;
    const int rows = 4096, beta = 3;
    // each CTA writes partial[rank][i][row] for rows of its cluster range (512 rows)
    for (int idx = threadIdx.x; idx < 512 * beta; idx += blockDim.x) {
        const int i = idx / 512, r = cid * 512 + idx % 512;
        float* dst = part + ((long)rank * beta + i) * rows + r;
        if (MODE == 0) __stcg(dst, 1.0f + r); else *dst = 1.0f + r;
    }
    unsigned long long t0 = gt();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    unsigned long long t1 = gt();
    float s = 0;
    if (threadIdx.x < 64) {
        const int r = cid * 512 + rank * 64 + threadIdx.x;
        float v[24];
#pragma unroll
        for (int q = 0; q < 24; ++q) v[q] = MODE == 0 ? __ldcg(part + ((long)(q % 8) * beta + q / 8) * rows + r) : part[((long)(q % 8) * beta + q / 8) * rows + r];
        float a = __ldg(alpha + r);
#pragma unroll
        for (int q = 0; q < 24; ++q) s += v[q] * a;
        y[r] = s;
    }
    unsigned long long t2 = gt();
    if (threadIdx.x == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t1; }
}
int main() {
    float *part, *alpha, *y; unsigned long long* out;
    cudaMalloc(&part, 64 << 20); cudaMalloc(&alpha, 1 << 20); cudaMalloc(&y, 1 << 20); cudaMallocManaged(&out, 64 * 16);
    cudaMemset(part, 0, 64 << 20); cudaMemset(alpha, 0, 1 << 20);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            if (mode == 0) k<0><<<64, 512>>>(part, alpha, y, out); else k<1><<<64, 512>>>(part, alpha, y, out);
            cudaDeviceSynchronize();
        }
        double b = 0, l = 0;
        for (int i = 0; i < 64; ++i) { b += out[2 * i]; l += out[2 * i + 1]; }
        printf("mode %d (%s): barrier %.0f ns, reduce %.0f ns\n", mode, mode == 0 ? "cg" : "default", b / 64, l / 64);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
