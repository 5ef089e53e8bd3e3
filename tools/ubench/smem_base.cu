// Where does the dynamic shared-memory window start (shared-space address),
// for plain and cluster launches?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(unsigned* out) {
    extern __shared__ __align__(1024) unsigned char s[];
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)__cvta_generic_to_shared(s);
}
int main() {
    unsigned* d;
    cudaMallocManaged(&d, 64 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {0, 1, 2, 4, 8, 16})
        for (int smem_kb : {100, 227}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(16);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = smem_kb * 1024;
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = cs ? cs : 1;
            a[0].val.clusterDim.y = 1;
            a[0].val.clusterDim.z = 1;
            cfg.attrs = a;
            cfg.numAttrs = cs ? 1 : 0;
            cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
            cudaDeviceSynchronize();
            printf("cluster %2d smem %3d KB: base 0x%x 0x%x (%s)\n", cs, smem_kb, d[0], d[15], cudaGetErrorString(e));
        }
    return 0;
}
