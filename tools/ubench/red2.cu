// Cluster reduction pattern microbenchmark: cluster size CS (8 or 16), 1 CTA/SM (big smem),
// partials in smem (DSMEM path) or global (L2 path).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void k(float* part, const float* alpha, float* y, unsigned long long* out, int cs) {
    extern __shared__ float sm[];
    uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int cid = blockIdx.x / cs, beta = 3, nrl = 608;
    for (int idx = threadIdx.x; idx < nrl * beta; idx += blockDim.x) {
        if (MODE == 0) sm[idx] = 1.0f + idx; else part[((long)rank * beta + idx / nrl) * 4096 + cid * nrl + idx % nrl] = 1.0f + idx;
    }
    unsigned long long t0 = gt();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    unsigned long long t1 = gt();
    const int o_lo = nrl * rank / cs, o_hi = nrl * (rank + 1) / cs;
    for (int o = o_lo + threadIdx.x; o < o_hi; o += blockDim.x) {
        double acc = 0;
        float v[48];
        for (int q = 0; q < 48; ++q) {
            const int kk = q % 16, i = q / 16;
            if (MODE == 0) {
                uint32_t a = smem_u32(sm + i * nrl + o), r;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(kk % cs));
                asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v[q]) : "r"(r));
            } else {
                v[q] = part[((long)(kk % cs) * beta + i) * 4096 + cid * nrl + o];
            }
        }
        for (int q = 0; q < 48; ++q) acc += v[q] * alpha[q];
        y[cid * nrl + o] = acc;
    }
    unsigned long long t2 = gt();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    if (threadIdx.x == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t1; }
}
int main() {
    float *part, *alpha, *y; unsigned long long* out;
    cudaMalloc(&part, 64 << 20); cudaMalloc(&alpha, 1 << 20); cudaMalloc(&y, 1 << 20); cudaMallocManaged(&out, 256 * 16);
    cudaMemset(part, 0, 64 << 20); cudaMemset(alpha, 0, 1 << 20);
    for (int cs : {8, 16}) for (int mode = 0; mode < 2; ++mode) {
        auto kern = mode == 0 ? k<0> : k<1>;
        const int smem = 192 * 1024;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs == 16 ? 112 : 128); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        for (int rep = 0; rep < 3; ++rep) { cudaLaunchKernelEx(&cfg, kern, part, (const float*)alpha, y, out, cs); cudaDeviceSynchronize(); }
        double b = 0, l = 0; int n = cfg.gridDim.x;
        for (int i = 0; i < n; ++i) { b += out[2 * i]; l += out[2 * i + 1]; }
        printf("cs %2d mode %s: barrier %.0f ns, reduce %.0f ns  (%s)\n", cs, mode == 0 ? "dsmem " : "global", b / n, l / n, cudaGetErrorString(cudaGetLastError()));
    }
}
