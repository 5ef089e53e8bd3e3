// How fast does a one-shot burst of TMA bulk copies land per SM?  (The
// single-call latency form's key stream: each CTA issues ~7 x 8 KiB at once.)
// Variants: cluster size (1 / 8), grid (120 / 148), dynamic smem size.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_burst tools/ubench/tma_burst.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void burst(const unsigned char* src, size_t per_cta, int pieces, unsigned long long* out, int spin) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    unsigned char* dst = sm + 1024;
    const unsigned long long t0 = gt();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t piece = static_cast<uint32_t>(per_cta / pieces);
    if (warp == 0) {
        for (int p = lane; p < pieces; p += 32) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[p])), "r"(1) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int p = lane; p < pieces; p += 32) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[p])), "r"(piece) : "memory");
            if (spin & 4) {
                uint64_t pol;
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                                 smem_u32(dst + p * piece)),
                             "l"(src + blockIdx.x * per_cta + p * piece), "r"(piece), "r"(smem_u32(&bar[p])), "l"(pol)
                             : "memory");
            } else {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(dst + p * piece)),
                             "l"(src + blockIdx.x * per_cta + p * piece), "r"(piece), "r"(smem_u32(&bar[p]))
                             : "memory");
            }
        }
    }
    const unsigned long long t1 = gt();
    if (spin & 2) asm volatile("griddepcontrol.launch_dependents;" :::);
    if (spin & 2) asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    if ((spin & 1) && warp > 0) {  // the latency form's gather warps: spin on the pieces meanwhile
        const int p = (warp - 1) % pieces;
        asm volatile("{\n\t.reg .pred q;\nS_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t@!q bra S_%=;\n}" ::"r"(
                         smem_u32(&bar[p]))
                     : "memory");
    }
    if (threadIdx.x == 0) {
        for (int p = 0; p < pieces; ++p)
            asm volatile("{\n\t.reg .pred q;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n\t@!q bra W_%=;\n}" ::"r"(
                             smem_u32(&bar[p]))
                         : "memory");
        const unsigned long long t2 = gt();
        out[blockIdx.x * 3 + 0] = t0;
        out[blockIdx.x * 3 + 1] = t1;
        out[blockIdx.x * 3 + 2] = t2;
    }
}

int main() {
    const size_t per_cta = 56 * 1024;
    const int copies = 40;
    unsigned char* src;
    cudaMalloc(&src, per_cta * 148 * copies);
    cudaMemset(src, 1, per_cta * 148 * copies);
    unsigned long long* out;
    cudaMalloc(&out, 148 * 3 * 8);
    cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(burst, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    struct V { int grid, cs, smem_kb, pieces, threads, spin; };
    std::vector<V> vs = {{120, 1, 227, 7, 576, 0}, {120, 8, 227, 7, 576, 0}, {148, 1, 227, 7, 576, 0},
                         {120, 8, 64, 7, 576, 0},  {120, 1, 64, 7, 576, 0},  {120, 8, 227, 28, 576, 0},
                         {120, 1, 227, 28, 576, 0}, {120, 8, 227, 7, 128, 0}, {120, 8, 227, 7, 576, 1},
                         {120, 1, 227, 7, 576, 1}, {120, 8, 227, 7, 576, 2}, {120, 8, 227, 7, 576, 3},
                         {120, 8, 227, 7, 576, 4}, {120, 8, 227, 7, 576, 6}};
    for (auto v : vs) {
        std::vector<double> issued, landed;
        for (int rep = 0; rep < 30; ++rep) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(v.grid);
            cfg.blockDim = dim3(v.threads);
            cfg.dynamicSmemBytes = v.smem_kb * 1024;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = v.cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[1].val.programmaticStreamSerializationAllowed = (v.spin & 2) ? 1 : 0;
            cfg.attrs = at;
            cfg.numAttrs = 2;
            const unsigned char* s = src + (rep % copies) * per_cta * 148;
            if (v.spin & 2) {  // a PDL chain of 20 launches; the last one is recorded
                for (int k = 0; k < 20; ++k)
                    cudaLaunchKernelEx(&cfg, burst, src + ((rep * 20 + k) % copies) * per_cta * 148, per_cta, v.pieces, out, v.spin);
            } else {
                cudaLaunchKernelEx(&cfg, burst, s, per_cta, v.pieces, out, v.spin);
            }
            cudaDeviceSynchronize();
            if (rep < 10) continue;
            std::vector<unsigned long long> h(148 * 3);
            cudaMemcpy(h.data(), out, 148 * 3 * 8, cudaMemcpyDeviceToHost);
            unsigned long long t0 = ~0ull;
            for (int i = 0; i < v.grid; ++i) t0 = std::min(t0, h[i * 3]);
            for (int i = 0; i < v.grid; ++i) {
                issued.push_back((h[i * 3 + 1] - t0) * 1e-3);
                landed.push_back((h[i * 3 + 2] - t0) * 1e-3);
            }
        }
        std::sort(issued.begin(), issued.end());
        std::sort(landed.begin(), landed.end());
        printf("spin %d grid %3d cluster %d smem %3d KB pieces %2d threads %3d: issued med %.2f  landed med %.2f max %.2f us  (%.1f GB/s/SM)\n",
               v.spin, v.grid, v.cs, v.smem_kb, v.pieces, v.threads, issued[issued.size() / 2], landed[landed.size() / 2],
               landed.back(), per_cta / (landed[landed.size() / 2] * 1e3));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
