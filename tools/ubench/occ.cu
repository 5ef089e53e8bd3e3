// Cluster scheduling facts on this part: max active clusters per size and
// smem footprint, and how many distinct SMs a grid of clusters lands on.
#include <cstdio>
#include <cstdint>
#include <set>
#include <cuda_runtime.h>

__global__ void probe(int* smid_out) {
    extern __shared__ unsigned char s[];
    uint32_t id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    if (threadIdx.x == 0) smid_out[blockIdx.x] = id;
    s[threadIdx.x] = 1;
    // hold the SM a little so the whole grid is resident together
    unsigned long long t0 = clock64();
    while (clock64() - t0 < 200000) {}
}

int main() {
    int* d;
    cudaMallocManaged(&d, 4096 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int smem_kb : {60, 100, 110, 150, 200}) {
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = smem_kb * 1024;
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = cs;
            a[0].val.clusterDim.y = 1;
            a[0].val.clusterDim.z = 1;
            cfg.attrs = a;
            cfg.numAttrs = 1;
            cfg.gridDim = dim3(cs);
            int n = 0;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
            if (e != cudaSuccess) { printf("smem %d cs %d: %s\n", smem_kb, cs, cudaGetErrorString(e)); cudaGetLastError(); continue; }
            cfg.gridDim = dim3(n * cs);
            for (int i = 0; i < 4096; ++i) d[i] = -1;
            e = cudaLaunchKernelEx(&cfg, probe, d);
            cudaDeviceSynchronize();
            std::set<int> sms;
            for (int i = 0; i < n * cs; ++i) sms.insert(d[i]);
            printf("smem %3d KB cluster %2d: max active clusters %3d -> %4d CTAs on %3zu SMs (%s)\n", smem_kb, cs, n,
                   n * cs, sms.size(), cudaGetErrorString(e));
        }
    }
    return 0;
}
