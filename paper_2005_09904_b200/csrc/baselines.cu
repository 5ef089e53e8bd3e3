// baselines.cu -- GPU versions of the reference's comparison methods
// (/root/reference/proj/core/include/biqgemm/baselines.hpp), used by the
// benchmark to show where BiQGEMM stands on B200 (paper
// Fig. 10 / Table IV analogs).  Not on the BiQGEMM path.
//
//  * gemm_unpack (baselines.hpp:40-52, Alg. 3 of the paper): y = sum_i
//    alpha_i * (B_i x) computed straight from the packed sign bits
//    (BinaryPlane words, bit 1 = +1), no lookup tables: a warp owns 32 rows
//    (lane = row), x is staged in shared memory and read as a broadcast, and
//    each bit costs one sign-select + one FMA per column.
//  * bandwidth_probe (baselines.hpp:56-87): multiplies each packed word as a
//    scalar against an x fragment -- values intentionally meaningless; it
//    measures the packed-word traffic with plain coalesced loads.
#include <algorithm>

#include "kernels.h"

namespace bqg {
namespace {

constexpr int kUW = 8;  // warps per CTA (split the words of the row tile)

template <int BMAX>
__global__ void __launch_bounds__(kUW * 32) unpack_gemv_kernel(const uint32_t* __restrict__ planes,
                                                               const float* __restrict__ alpha,
                                                               const float* __restrict__ x, long long x_rows,
                                                               float* __restrict__ y, long long m, long long n,
                                                               int b, int beta) {
    extern __shared__ float xs[];  // [n][b]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (long long i = threadIdx.x; i < n * b; i += blockDim.x)
        xs[i] = (i / b) < x_rows ? x[i] : 0.0f;
    __syncthreads();
    __shared__ float part[kUW][32][BMAX];
    const long long r = static_cast<long long>(blockIdx.x) * 32 + lane;
    const long long wpr = (n + 31) / 32;
    float yacc[BMAX];
#pragma unroll
    for (int c = 0; c < BMAX; ++c) yacc[c] = 0.0f;
    for (int i = 0; i < beta; ++i) {
        float acc[BMAX];
#pragma unroll
        for (int c = 0; c < BMAX; ++c) acc[c] = 0.0f;
        if (r < m) {
            const uint32_t* row = planes + (static_cast<long long>(i) * m + r) * wpr;
            for (long long w = warp; w < wpr; w += kUW) {
                const uint32_t word = __ldg(row + w);
                const int kmax = static_cast<int>(min(32LL, n - w * 32));
                for (int k = 0; k < kmax; ++k) {
                    // +1 for a set bit, -1 otherwise (packing.hpp:16-57)
                    const float s = __int_as_float(0x3f800000 | ((~(word >> k) & 1u) << 31));
#pragma unroll
                    for (int c = 0; c < BMAX; ++c)
                        if (c < b) acc[c] = fmaf(s, xs[(w * 32 + k) * b + c], acc[c]);
                }
            }
        }
        // reduce the kUW word-partials of each row, then scale by alpha_i
#pragma unroll
        for (int c = 0; c < BMAX; ++c) part[warp][lane][c] = acc[c];
        __syncthreads();
        if (warp == 0 && r < m) {
            const float a = alpha ? alpha[static_cast<long long>(i) * m + r] : 1.0f;
#pragma unroll
            for (int c = 0; c < BMAX; ++c) {
                float s = 0.0f;
#pragma unroll
                for (int q = 0; q < kUW; ++q) s += part[q][lane][c];
                yacc[c] += a * s;
            }
        }
        __syncthreads();
    }
    if (warp == 0 && r < m)
        for (int c = 0; c < b; ++c) y[r * b + c] = yacc[c];
}

__global__ void probe_kernel(const uint32_t* __restrict__ words, long long m, long long wpr,
                             const float* __restrict__ x, long long x_rows, float* __restrict__ out) {
    // one thread per row: acc += word * x((w*32) % x_rows), the reference's arithmetic
    const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= m) return;
    // rows are read word-interleaved across the warp for coalescing: thread t
    // of the warp reads word (t + 32j) of the 32-row block
    double acc = 0.0;
    const uint32_t* row = words + r * wpr;
    for (long long w = 0; w < wpr; ++w) acc += static_cast<double>(__ldcs(row + w)) * x[(w * 32) % x_rows];
    out[r] = static_cast<float>(acc);
}

__global__ void probe_stream_kernel(const uint4* __restrict__ words, long long n16, const float* __restrict__ x,
                                    long long x_rows, float* __restrict__ out) {
    // the same traffic with 16-byte coalesced streaming loads (the probe's
    // bandwidth, not the reference's loop order)
    float acc = 0.0f;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcs(words + i);
        const float xv = x[(i * 128) % x_rows];
        acc = fmaf(static_cast<float>(v.x ^ v.y ^ v.z ^ v.w), xv, acc);
    }
    out[static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x] = acc;
}

}  // namespace

cudaError_t launch_gemm_unpack(const uint32_t* planes, const float* alpha, const float* x, long long x_rows, float* y,
                               long long m, long long n, int b, int beta, cudaStream_t stream) {
    const size_t smem = static_cast<size_t>(n) * b * sizeof(float);
    if (smem > 200 * 1024 || b > 8) return cudaErrorInvalidValue;
    const dim3 grid(static_cast<unsigned>((m + 31) / 32));
#define BQG_UNPACK(BM)                                                                                          \
    {                                                                                                           \
        auto k = unpack_gemv_kernel<BM>;                                                                        \
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);      \
        if (e != cudaSuccess) return e;                                                                         \
        k<<<grid, kUW * 32, smem, stream>>>(planes, alpha, x, x_rows, y, m, n, b, beta);                        \
        return cudaGetLastError();                                                                              \
    }
    if (b == 1) BQG_UNPACK(1)
    if (b <= 2) BQG_UNPACK(2)
    if (b <= 4) BQG_UNPACK(4)
    BQG_UNPACK(8)
#undef BQG_UNPACK
}

cudaError_t launch_bandwidth_probe(const uint32_t* words, long long m, long long n, const float* x, long long x_rows,
                                   float* out, bool streaming, cudaStream_t stream) {
    const long long wpr = (n + 31) / 32;
    if (!streaming) {
        probe_kernel<<<static_cast<unsigned>((m + 255) / 256), 256, 0, stream>>>(words, m, wpr, x, x_rows, out);
        return cudaGetLastError();
    }
    const long long n16 = m * wpr / 4;  // whole 16-byte groups (the tail is not part of the probe)
    probe_stream_kernel<<<1184, 512, 0, stream>>>(reinterpret_cast<const uint4*>(words), n16, x, x_rows, out);
    return cudaGetLastError();
}

}  // namespace bqg
