// Latency of reading data another SM just wrote (cluster barrier handoff).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void __cluster_dims__(8, 1, 1) k(float* buf, unsigned long long* out, int mode) {
    uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    float* mine = buf + (blockIdx.x) * 1024;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) __stcg(mine + i, (float)(i + blockIdx.x));
    unsigned long long t0 = gt();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    unsigned long long t1 = gt();
    const int other = (blockIdx.x / 8) * 8 + (rank + 1) % 8;
    const float* src = mode == 0 ? buf + other * 1024 : (mode == 1 ? mine : buf + (blockIdx.x + 4096) * 1024);
    float v = 0;
    for (int rep = 0; rep < 4; ++rep) v += __ldcg(src + threadIdx.x + rep * 256);
    unsigned long long t2 = gt();
    float w = __ldcg(src + 1023 - threadIdx.x);  // second dependent-ish round
    unsigned long long t3 = gt();
    if (threadIdx.x == 0) { out[blockIdx.x * 4 + 0] = t1 - t0; out[blockIdx.x * 4 + 1] = t2 - t1; out[blockIdx.x * 4 + 2] = t3 - t2; }
    if (v + w == 12345.f) buf[0] = 0;
}
int main() {
    float* buf; unsigned long long* out;
    cudaMalloc(&buf, 8192 * 1024 * 4); cudaMallocManaged(&out, 128 * 4 * 8);
    cudaMemset(buf, 0, 8192 * 1024 * 4);
    const char* names[3] = {"other CTA's data", "own data", "untouched data"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int r = 0; r < 3; ++r) { k<<<112, 256>>>(buf, out, mode); cudaDeviceSynchronize(); }
        double b = 0, l1 = 0, l2 = 0;
        for (int i = 0; i < 112; ++i) { b += out[i * 4]; l1 += out[i * 4 + 1]; l2 += out[i * 4 + 2]; }
        printf("%-18s: barrier %.0f ns, first loads %.0f ns, second load %.0f ns\n", names[mode], b / 112, l1 / 112, l2 / 112);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
