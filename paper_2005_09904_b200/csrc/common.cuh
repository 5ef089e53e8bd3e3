// common.cuh -- shared device helpers for the BiQGEMM sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bqg {

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

__device__ __forceinline__ float ld_cg_f32(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

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

}  // namespace bqg
