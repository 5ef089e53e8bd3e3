// common.cuh -- shared device helpers for the BiQGEMM sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

namespace bqg {

// ---- host-side per-device launch state ---------------------------------------

// Kernel attributes (cudaFuncSetAttribute), occupancy answers and the SM
// count belong to a DEVICE, not to the process: a process that drives two
// GPUs must configure each one.  Every launcher keeps its one-time state in
// a PerDevice table indexed by the current device ordinal, initialised under
// std::call_once (thread-safe).
constexpr int kMaxDevices = 64;
struct PerDeviceOnce {
    std::once_flag flag[kMaxDevices];
    cudaError_t err[kMaxDevices] = {};
};
inline int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return -1;
    return d;
}
// Runs f() once per device; later calls return f()'s first result.
template <class F>
inline cudaError_t once_per_device(PerDeviceOnce& o, int dev, F&& f) {
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    std::call_once(o.flag[dev], [&] { o.err[dev] = f(); });
    return o.err[dev];
}
inline int device_sms(int dev) {
    static std::atomic<int> sms[kMaxDevices];
    if (dev < 0 || dev >= kMaxDevices) return 148;
    int v = sms[dev].load(std::memory_order_relaxed);
    if (v == 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        sms[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// ---- launch-level helpers ---------------------------------------------------

// Programmatic dependent launch (PDL).  A kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor on the stream is still running; griddepcontrol.wait blocks
// until the predecessor grid has completed and its memory is visible.
// Everything placed before pdl_wait() must not read memory the predecessor
// writes (here: only the packed weight keys, which are immutable).
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// ---- streaming loads ----------------------------------------------------------

// L2 eviction policy "evict first": the packed-key stream is read exactly
// once per call and must not push the LUT inputs / workspace out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 256-bit read-only streaming load (sm_100: ld.v8.b32), no L1 allocation,
// L2 evict-first.  `p` must be 32-byte aligned.
struct U8x32 {
    uint32_t w[8];
};
__device__ __forceinline__ U8x32 ld_stream_u8x32(const void* p) {
    U8x32 v;
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]),
          "=r"(v.w[6]), "=r"(v.w[7])
        : "l"(p));
    return v;
}

// 128-bit read-only streaming load with an explicit L2 cache policy.
__device__ __forceinline__ uint4 ld_stream_u4(const void* p, uint64_t pol) {
    uint4 v;
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p), "l"(pol));
    return v;
}

// L2-coherent load (bypasses L1) that the compiler may schedule freely.
__device__ __forceinline__ float ld_cg_f32(const float* p) { return __ldcg(p); }

// Release/acquire fence at GPU scope (lighter than __threadfence's SC fence):
// orders this thread's partial stores before its ticket atomic, and the
// finaliser's ticket observation before its partial loads.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// ---- shared memory --------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ float2 lds_f32x2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

__device__ __forceinline__ float4 lds_f32x4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// Exact IEEE fp32 add that ptxas may not contract or reorder: the LUT entries
// must follow the DP recurrence of lut.hpp:50-69 operation for operation.
__device__ __forceinline__ float fadd_rn(float a, float b) { return __fadd_rn(a, b); }

// ---- mbarrier + bulk copy (TMA engine, non-tensor) ---------------------------

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}"
        ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// Non-blocking test: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Wait by polling with a fixed sleep between tests: for warps that wait a
// long time (many microseconds) off the critical path.  Each poll costs ~4
// issue slots; the hardware-suspended try_wait of mbar_wait_sleep (below)
// wakes far more often than that (measured: ~10 polls per gathered unit in
// the texture form).
__device__ __forceinline__ void mbar_wait_poll(uint64_t* bar, uint32_t parity, unsigned sleep_ns) {
    while (!mbar_test(bar, parity)) __nanosleep(sleep_ns);
}
// Like mbar_wait, but the thread may sleep until the phase completes (suspend-time
// hint): for warps that wait long (producers, builders, loaders) so that
// their retries do not take issue slots from the gather warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
#ifdef BQG_NO_SLEEP_WAIT
    mbar_wait(bar, parity);
    return;
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}"
        ::"r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
}
// Global -> shared bulk copy completed on `bar` (complete_tx), L2 policy hint.
// bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// Same without an L2 policy (data other CTAs re-read: x, alpha).
__device__ __forceinline__ void bulk_g2s_plain(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst_smem)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Named barrier over `count` threads (the consumer warps only).
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// Arrive without waiting (the producer side of a named-barrier handoff).
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- thread-block clusters ---------------------------------------------------

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// Distributed shared memory: the address of the same shared-memory offset in
// CTA `rank` of this cluster, and a load through it.
__device__ __forceinline__ uint32_t dsmem_map(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t caddr) {
    float v;
    asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(caddr));
    return v;
}

// Cluster-wide barrier with release/acquire semantics: global-memory writes of
// every CTA in the cluster before the arrive are visible to every CTA after
// the wait.  All threads of every CTA must execute it.
__device__ __forceinline__ void cluster_sync_acqrel() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Cluster barrier without memory ordering (e.g. "nobody exits while others
// still read my shared memory").
__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

}  // namespace bqg
