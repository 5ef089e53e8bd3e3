// Raw HBM read bandwidth of a per-SM TMA bulk-copy ring (cp.async.bulk ->
// mbarrier), vs stage size and ring depth, with trivial consumers; and a
// plain LDG.128 streaming kernel for reference.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                     smem_u32(b)),
                 "r"(par)
                 : "memory");
}

template <int POLICY>
__global__ void __launch_bounds__(256, 1) tma_ring(const unsigned char* src, size_t per_cta, int stage, int nst,
                                                   unsigned* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + 32;
    unsigned char* ring = sm + 1024;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 7); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned char* base = src + blockIdx.x * per_cta;
    const long long nstages = per_cta / stage;
    if (warp == 0) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (long long s = 0; s < nstages; ++s) {
                const int slot = s % nst;
                if (s >= nst) mbar_wait(&empty[slot], ((s / nst) - 1) & 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])), "r"(stage) : "memory");
                if (POLICY)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                                     smem_u32(ring + slot * stage)),
                                 "l"(base + s * stage), "r"(stage), "r"(smem_u32(&full[slot])), "l"(pol)
                                 : "memory");
                else
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     smem_u32(ring + slot * stage)),
                                 "l"(base + s * stage), "r"(stage), "r"(smem_u32(&full[slot]))
                                 : "memory");
            }
        }
        return;
    }
    unsigned acc = 0;
    for (long long s = 0; s < nstages; ++s) {
        const int slot = s % nst;
        mbar_wait(&full[slot], (s / nst) & 1);
        acc += ring[slot * stage + (warp * 32 + lane) * 4];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
}

// Same ring, stage copied as `split` pieces, stages issued round-robin by `lanes` producer lanes.
__global__ void __launch_bounds__(256, 1) tma_ring2(const unsigned char* src, size_t per_cta, int stage, int nst,
                                                    int split, int lanes, unsigned* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + 32;
    unsigned char* ring = sm + 1024;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 7); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned char* base = src + blockIdx.x * per_cta;
    const long long nstages = per_cta / stage;
    if (warp == 0) {
        if (lane < lanes) {
            const int piece = stage / split;
            for (long long s = lane; s < nstages; s += lanes) {
                const int slot = s % nst;
                if (s >= nst) mbar_wait(&empty[slot], ((s / nst) - 1) & 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])), "r"(stage) : "memory");
                for (int q = 0; q < split; ++q)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     smem_u32(ring + slot * stage + q * piece)),
                                 "l"(base + s * stage + q * piece), "r"(piece), "r"(smem_u32(&full[slot]))
                                 : "memory");
            }
        }
        return;
    }
    unsigned acc = 0;
    for (long long s = 0; s < nstages; ++s) {
        const int slot = s % nst;
        mbar_wait(&full[slot], (s / nst) & 1);
        acc += ring[slot * stage + (warp * 32 + lane) * 4];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
    }
    if (acc == 0xdeadbeef) sink[0] = acc;
}

__global__ void ldg_stream(const uint4* src, size_t n16, unsigned* sink) {
    uint4 acc = {0, 0, 0, 0};
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(src + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0xdeadbeef) sink[0] = 1;
}

int main() {
    const size_t total = size_t(1) << 31;  // 2 GiB, >> L2
    unsigned char* buf;
    unsigned* sink;
    cudaMalloc(&buf, total);
    cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, total);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148;
    const size_t per_cta = (total / grid) & ~size_t(65535);
    cudaFuncSetAttribute(tma_ring<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(tma_ring<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(tma_ring2, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int stage : {8192, 16384, 32768})
        for (int split : {1, 2, 4, 8})
            for (int lanes : {1, 2, 4}) {
                const int nst = 128 * 1024 / stage;
                if (stage / split < 1024) continue;
                const size_t pc = per_cta / stage * stage;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(e0);
                    tma_ring2<<<grid, 256, 1024 + nst * stage>>>(buf, pc, stage, nst, split, lanes, sink);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("ring2 stage %5d split %d (piece %5d) lanes %d: %7.1f GB/s %s\n", stage, split, stage / split, lanes,
                       pc * grid / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
    for (int pol = 0; pol < 0; ++pol)
        for (int stage : {4096, 8192, 12288, 16384, 32768}) {
            for (int ring_kb : {32, 64, 96, 128, 192}) {
                const int nst = ring_kb * 1024 / stage;
                if (nst < 2 || nst > 32) continue;
                const size_t pc = per_cta / stage * stage;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(e0);
                    if (pol) tma_ring<1><<<grid, 256, 1024 + nst * stage>>>(buf, pc, stage, nst, sink);
                    else tma_ring<0><<<grid, 256, 1024 + nst * stage>>>(buf, pc, stage, nst, sink);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("tma %s stage %5d B ring %3d KB (%2d stages): %7.1f GB/s  %s\n", pol ? "evict_first" : "no-hint    ",
                       stage, ring_kb, nst, pc * grid / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
        }
    for (int blocks : {1184}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            ldg_stream<<<blocks, 512>>>(reinterpret_cast<const uint4*>(buf), total / 16, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("ldg.128 grid %4d x 512: %7.1f GB/s\n", blocks, total / ms / 1e6);
    }
    return 0;
}
