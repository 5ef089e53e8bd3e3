// kernels.h -- internal launcher declarations shared by the C-ABI layer.
//
// Device data layouts (all row-major unless stated):
//   W        m x n f32
//   planes   beta x m x ceil(n/32) u32 words, LSB-first, bit 1 = +1
//            (BinaryPlane, packing.hpp:16-57)
//   alpha    beta x m f32 (QuantizedLinear::alphas, quantize.hpp:16-22)
//   keys     beta x m x G, u8 for mu <= 8, u16 for mu > 8, pad bits 0
//            (KeyMatrix, packing.hpp:61-73; the BQGM on-disk key payload,
//            model_io.cpp:77-87)
//   tiled    (mu <= 8) NB x beta x MT x 32 x 32 bytes, NB = ceil(G/32),
//            MT = ceil(m/32): for group block gb, plane i, row tile t the
//            1 KiB chunk holds, for lane gl (group gb*32+gl), the 32 keys of
//            rows t*32 .. t*32+31 at byte position rr ^ gl.  A warp streams
//            one contiguous 1 KiB chunk per (plane, row tile); the XOR
//            swizzle lets the cross-lane reduction run without selects.
//   x        x_rows x b f32 (x_rows <= G*mu; missing rows are zero)
//   y        m x b f32
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bqg {

struct QueryParams {
    const uint8_t* keys;    // tiled
    const float* alpha;     // beta x m or nullptr (plane mode: alpha = 1)
    const float* x;         // x_rows x b
    float* y;               // m x b
    float* partial;         // NB x beta x (MT*32) x b   (workspace)
    unsigned* counters;     // MT                        (workspace, zero, left zero)
    long long x_rows;
    int m, G, NB, MT, beta, b, cpb;
};

// Workspace for the fast path (bytes).
size_t fast_workspace_bytes(long long m, long long groups, int beta, long long b);
// Grid planner: CTAs per 32-group block.
int plan_cpb(long long m, long long groups, int beta, long long b, int num_sms);

cudaError_t launch_quantize_greedy(const float* w, long long m, long long n, int beta,
                                   uint32_t* planes, float* alpha, double* alpha_d,
                                   cudaStream_t stream);
cudaError_t launch_pack_keys(const uint32_t* plane, long long m, long long n, int mu, void* keys,
                             cudaStream_t stream);
cudaError_t launch_tile_keys(const uint8_t* keys, long long m, long long groups, int beta,
                             uint8_t* tiled, cudaStream_t stream);

// Fast path (mu <= 8): fused LUT build -> query -> alpha epilogue.
cudaError_t launch_biqgemm_fast(const QueryParams& p, int mu, bool pdl, cudaStream_t stream);

// Fast-path LUT builder exposed for parity (same device code as the fused kernel).
cudaError_t launch_build_lut_f32(const float* x, long long x_rows, long long b, int mu,
                                 long long g0, long long count, bool key_major, float* out,
                                 cudaStream_t stream);

// Exact path (any mu in 1..16, any b): fp64 LUT (global memory), fp64
// accumulation in the reference's order -> bit-identical to
// biqgemm::detail::run (kernel.hpp:116-204).  T is float or double.
template <typename T>
cudaError_t launch_build_lut_exact(const T* x, long long x_rows, long long b, int mu, long long g0,
                                   long long count, bool key_major, double* out,
                                   cudaStream_t stream);
template <typename T>
cudaError_t launch_biqgemm_exact(const void* keys_rowmajor, const T* alpha, const T* x,
                                 long long x_rows, T* y, long long m, long long n, int beta,
                                 int mu, long long b, void* workspace, size_t workspace_bytes,
                                 cudaStream_t stream);
size_t exact_workspace_bytes(long long m, long long n, int beta, int mu, long long b);

}  // namespace bqg
