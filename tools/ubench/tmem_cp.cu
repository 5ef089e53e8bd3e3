// Can key chunks reach registers through TMEM instead of LDS?  smem chunk
// (32 rows x 32 B, row l's 16-byte pieces at l*16 and 512 + l*16) ->
// tcgen05.cp.32x128b.warpx4 (x2) -> TMEM -> tcgen05.ld.32x32b.x4 (x2) in each
// warp's lane quarter.  Checks the bytes and measures the cp issue rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_k_interleave(uint32_t saddr, uint32_t sbo_bytes, uint32_t lbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
    return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__global__ void k(int* bad, unsigned long long* cyc, int ncp, int issuers) {
    __shared__ __align__(1024) unsigned char chunk[1024];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) chunk[i] = (unsigned char)(i * 7 + 3);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // make the generic-proxy smem writes visible to the async (tensor) proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tbase;
    if (threadIdx.x == 0) {
        const uint64_t d0 = desc_k_interleave(smem_u32(chunk), 128, 0);
        const uint64_t d1 = desc_k_interleave(smem_u32(chunk + 512), 128, 0);
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tb), "l"(d0));
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tb + 4), "l"(d1));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    asm volatile("{\n\t.reg .pred p;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n}" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[8];
    const uint32_t ta = tb | ((uint32_t)(32 * (warp & 3)) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(ta + 4));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const uint32_t* s0 = reinterpret_cast<const uint32_t*>(chunk + lane * 16);
    const uint32_t* s1 = reinterpret_cast<const uint32_t*>(chunk + 512 + lane * 16);
    int b = 0;
    for (int i = 0; i < 4; ++i) {
        b += r[i] != s0[i];
        b += r[4 + i] != s1[i];
    }
    if (b) atomicAdd(bad, b);
    // issue rate: lane 0 of warps 0..issuers-1 each issue ncp/issuers copies
    __syncthreads();
    __shared__ __align__(8) uint64_t bars[8];
    if (threadIdx.x < 8) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[threadIdx.x])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned long long t0 = clock64();
    if (lane == 0 && warp < issuers) {
        const uint64_t d0 = desc_k_interleave(smem_u32(chunk), 128, 0);
        const int per = ncp / issuers;
        for (int i = 0; i < per; ++i)
            asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tb + (uint32_t)(((warp * per + i) * 4) & 511)), "l"(d0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[warp])));
        asm volatile("{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n}" ::"r"(
                         smem_u32(&bars[warp]))
                     : "memory");
    }
    __syncthreads();
    unsigned long long t2 = clock64();
    if (threadIdx.x == 0) {
        cyc[blockIdx.x * 2 + 0] = t2 - t0;
        cyc[blockIdx.x * 2 + 1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
    int* bad;
    unsigned long long* cyc;
    cudaMallocManaged(&bad, 4);
    cudaMallocManaged(&cyc, 148 * 2 * 8);
    for (int issuers : {1, 2, 4, 8}) {
        const int ncp = 1024;
        *bad = 0;
        k<<<148, 256>>>(bad, cyc, ncp, issuers);
        cudaError_t e = cudaDeviceSynchronize();
        printf("issuers %d ncp %4d: mismatching words %d (%s); all copies done in %llu cycles (%.1f per cp)\n", issuers,
               ncp, *bad, cudaGetErrorString(e), cyc[0], (double)cyc[0] / ncp);
    }
    return 0;
}
