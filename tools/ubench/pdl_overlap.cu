// Does a PDL successor's CTA become resident on an SM while the
// predecessor's CTA still runs there (2 CTAs/SM by smem)?  And how long after
// the predecessor's last CTA exits does griddepcontrol.wait return?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void kern(unsigned long long* t, int spin_ns, int idx) {
    extern __shared__ unsigned char s[];
    unsigned long long t0 = gt();
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    unsigned long long t1 = gt();
    s[threadIdx.x] = 1;
    while (gt() - t1 < (unsigned long long)spin_ns) {}
    __syncthreads();
    unsigned long long t2 = gt();
    if (threadIdx.x == 0) {
        t[(idx * 1024 + blockIdx.x) * 3 + 0] = t0;
        t[(idx * 1024 + blockIdx.x) * 3 + 1] = t1;
        t[(idx * 1024 + blockIdx.x) * 3 + 2] = t2;
    }
}
int main() {
    unsigned long long* t;
    cudaMallocManaged(&t, 8 * 1024 * 3 * 8);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int smem_kb : {100, 200}) {
        for (int rep = 0; rep < 2; ++rep) {
            for (int i = 0; i < 4; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(148);
                cfg.blockDim = dim3(256);
                cfg.dynamicSmemBytes = smem_kb * 1024;
                cfg.stream = s;
                cudaLaunchAttribute a[1];
                a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                a[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = a;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, kern, t, 5000, i);
            }
            cudaStreamSynchronize(s);
        }
        printf("smem %d KB (4 kernels x 148 CTAs, 5 us body):\n", smem_kb);
        unsigned long long base = ~0ull;
        for (int i = 0; i < 148; ++i) base = t[i * 3] < base ? t[i * 3] : base;
        for (int k = 0; k < 4; ++k) {
            unsigned long long smin = ~0ull, smax = 0, wmin = ~0ull, wmax = 0, emax = 0, emin = ~0ull;
            for (int i = 0; i < 148; ++i) {
                unsigned long long* r = t + (k * 1024 + i) * 3;
                smin = r[0] < smin ? r[0] : smin;
                smax = r[0] > smax ? r[0] : smax;
                wmin = r[1] < wmin ? r[1] : wmin;
                wmax = r[1] > wmax ? r[1] : wmax;
                emax = r[2] > emax ? r[2] : emax;
                emin = r[2] < emin ? r[2] : emin;
            }
            printf("  k%d start [%6llu,%6llu] wait-return [%6llu,%6llu] end [%6llu,%6llu] ns\n", k, smin - base,
                   smax - base, wmin - base, wmax - base, emin - base, emax - base);
        }
    }
    return 0;
}
