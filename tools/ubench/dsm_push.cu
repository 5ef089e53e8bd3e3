// Cross-CTA partial-sum exchange inside a cluster: push with
// st.async...mbarrier::complete_tx into the owner's shared memory, vs a full
// cluster barrier followed by DSMEM pulls.  Timed per CTA with globaltimer.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
template <int CS>
__global__ void push(unsigned long long* out, int mode) {
    __shared__ __align__(16) float slots[CS][3][64];  // [src rank][plane][row]
    __shared__ __align__(8) uint64_t bar;
    const uint32_t rank = ctarank();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // everyone's barrier must be initialised before anyone pushes
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"(CS * 3 * 64 * 4) : "memory");
    __syncthreads();
    const unsigned long long t0 = gt();
    if (mode == 0) {
        // push: thread (dst, plane, row-pair)...: 32 threads per (dst rank) each sending 3*64 floats / 32
        for (int e = threadIdx.x; e < CS * 3 * 16; e += blockDim.x) {
            const int dst = e / 48, rem = e % 48;  // 48 float4 per (dst): 3 planes x 16 float4
            const float v = (float)(rank * 1000 + rem);
            const uint32_t laddr = smem_u32(&slots[rank][rem / 16][(rem % 16) * 4]);
            const uint32_t raddr = mapa(laddr, dst);
            const uint32_t rbar = mapa(smem_u32(&bar), dst);
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(raddr),
                         "f"(v), "f"(v), "f"(v), "f"(v), "r"(rbar)
                         : "memory");
        }
        // wait for all CS pushes into my slots
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
    } else {
        // local store + cluster barrier + pull
        for (int e = threadIdx.x; e < 3 * 64; e += blockDim.x) slots[rank][e / 64][e % 64] = (float)e;
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        float acc = 0;
        for (int e = threadIdx.x; e < CS * 3 * 64 / CS; e += blockDim.x) {
            for (int r = 0; r < CS; ++r) {
                float v;
                asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(mapa(smem_u32(&slots[r][0][0]) + e * 4, r)));
                acc += v;
            }
        }
        slots[0][0][threadIdx.x % 64] += acc;
    }
    const unsigned long long t1 = gt();
    float s = 0;
    for (int r = 0; r < CS; ++r) s += slots[r][threadIdx.x % 3][threadIdx.x % 64];
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0 + (s == 1.2345f);
}
template <int CS>
void run(unsigned long long* out, int mode) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS * (CS == 16 ? 7 : 18));
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = CS;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(push<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int r = 0; r < 5; ++r) cudaLaunchKernelEx(&cfg, push<CS>, out, mode);
    cudaError_t e = cudaDeviceSynchronize();
    double m = 0, mx = 0;
    for (unsigned i = 0; i < cfg.gridDim.x; ++i) {
        m += out[i];
        mx = out[i] > mx ? out[i] : mx;
    }
    printf("cluster %2d %s: mean %.0f ns max %.0f ns (%s)\n", CS, mode == 0 ? "push st.async+mbarrier" : "barrier+pull   ",
           m / cfg.gridDim.x, mx, cudaGetErrorString(e));
}
int main() {
    unsigned long long* out;
    cudaMallocManaged(&out, 4096 * 8);
    for (int mode = 0; mode < 2; ++mode) {
        run<4>(out, mode);
        run<8>(out, mode);
        run<16>(out, mode);
    }
    return 0;
}
