// biqgemm_exact.cu -- the exact path: fp64 LUT in global memory (L2), fp64
// accumulation in the reference's order, any mu in 1..16, any batch b, T in
// {float, double}.
//
// It reproduces biqgemm::detail::run (/root/reference/proj/core/include/
// biqgemm/kernel.hpp:116-204) operation for operation:
//   - tables: build_lut_dp in double (lut.hpp:50-69), e[k] evaluated as
//     e0 + ascending set-bit steps (the DP's own addition order);
//   - acc_i(r, col) += entry, groups ascending, starting from +0.0
//     (query_rows, kernel.hpp:83-108; tiling never changes this order);
//   - y(r, col) = T(sum_i alpha_i[r] * acc_i(r, col)) in double, planes
//     ascending (kernel.hpp:183-195),
// so y is bit-identical to the reference CPU path.  It is the path for
// mu > 8 (2^mu-entry tables do not fit shared memory) and for T = double, and
// the debug "exact mode" for fp32.  It is not the fast path.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace bqg {

namespace {

constexpr size_t kLutTileBudget = size_t(256) << 20;  // bytes of fp64 tables per tile

// One thread per (table (gl, col), k < 2^(mu-1)).  layout: 0 table-major,
// 1 key-major, within the tile (LutBlock::index, lut.hpp:90-97).
// naive = 0: build_lut_dp order (lut.hpp:50-69); naive = 1: build_lut_naive
// (lut.hpp:31-43), every entry an explicit signed sum, t ascending.
template <typename T>
__global__ void build_lut_exact_kernel(const T* __restrict__ x, long long x_rows, long long b, int mu,
                                       long long g0, long long count, int key_major, int naive,
                                       double* __restrict__ out) {
    const long long half = 1LL << (mu - 1);
    const long long table = 1LL << mu;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= count * b * half) return;
    const long long k = idx % half;
    const long long tbl = idx / half;  // gl * b + col
    const long long gl = tbl / b, col = tbl - gl * b;
    const long long g = g0 + gl;
    double e = 0.0;
    for (int t = 0; t < mu; ++t) {
        const long long r = g * mu + t;
        const double xv = r < x_rows ? static_cast<double>(x[r * b + col]) : 0.0;
        e = __dsub_rn(e, xv);
    }
    for (int t = 0; t < mu - 1; ++t) {
        if ((k >> t) & 1) {
            const long long r = g * mu + t;
            const double xv = r < x_rows ? static_cast<double>(x[r * b + col]) : 0.0;
            e = __dadd_rn(e, __dmul_rn(2.0, xv));
        }
    }
    const long long base = gl * b * table;
    const long long kk = table - 1 - k;
    if (naive) {
        // both halves computed directly: acc += s_t * x_t, t ascending, from +0.0
        double e1 = 0.0, e2 = 0.0;
        for (int t = 0; t < mu; ++t) {
            const long long r = g * mu + t;
            const double xv = r < x_rows ? static_cast<double>(x[r * b + col]) : 0.0;
            e1 = __dadd_rn(e1, __dmul_rn(((k >> t) & 1) ? 1.0 : -1.0, xv));
            e2 = __dadd_rn(e2, __dmul_rn(((kk >> t) & 1) ? 1.0 : -1.0, xv));
        }
        e = e1;
        if (key_major) {
            out[base + k * b + col] = e1;
            out[base + kk * b + col] = e2;
        } else {
            out[base + col * table + k] = e1;
            out[base + col * table + kk] = e2;
        }
        return;
    }
    if (key_major) {
        out[base + k * b + col] = e;
        out[base + kk * b + col] = -e;
    } else {
        out[base + col * table + k] = e;
        out[base + col * table + kk] = -e;
    }
}

// acc_i(r, col) += sum over groups of the tile, ascending.  One thread per
// (plane, row, col).
template <typename K>
__global__ void query_exact_kernel(const K* __restrict__ keys, const double* __restrict__ lut,
                                   long long m, long long groups, int beta, int mu, long long b,
                                   long long g0, long long count, double* __restrict__ acc) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<long long>(beta) * m * b) return;
    const long long col = idx % b;
    const long long ir = idx / b;  // i * m + r
    const long long table = 1LL << mu;
    const K* kp = keys + ir * groups + g0;
    double a = acc[idx];
    for (long long gl = 0; gl < count; ++gl) {
        const long long key = static_cast<long long>(kp[gl]);
        a = __dadd_rn(a, lut[(gl * b + col) * table + key]);
    }
    acc[idx] = a;
}

template <typename T>
__global__ void epilogue_exact_kernel(const double* __restrict__ acc, const T* __restrict__ alpha,
                                      long long m, int beta, long long b, T* __restrict__ y) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= m * b) return;
    const long long r = idx / b;
    double s = 0.0;
    for (int i = 0; i < beta; ++i) {
        const double a = alpha ? static_cast<double>(alpha[static_cast<long long>(i) * m + r]) : 1.0;
        s = __dadd_rn(s, __dmul_rn(a, acc[static_cast<long long>(i) * m * b + idx]));
    }
    y[idx] = static_cast<T>(s);
}

long long tile_groups(long long groups, int mu, long long b) {
    const long long per_group = (1LL << mu) * b * static_cast<long long>(sizeof(double));
    return std::max<long long>(1, std::min<long long>(groups, static_cast<long long>(kLutTileBudget) / per_group));
}

unsigned blocks_for(long long n, int threads) { return static_cast<unsigned>((n + threads - 1) / threads); }

}  // namespace

size_t exact_workspace_bytes(long long m, long long n, int beta, int mu, long long b) {
    const long long groups = (n + mu - 1) / mu;
    const size_t acc = static_cast<size_t>(beta) * m * b * sizeof(double);
    const size_t lut = static_cast<size_t>(tile_groups(groups, mu, b)) * b * (size_t(1) << mu) * sizeof(double);
    return ((acc + 255) / 256) * 256 + lut;
}

template <typename T>
cudaError_t launch_build_lut_exact(const T* x, long long x_rows, long long b, int mu, long long g0,
                                   long long count, bool key_major, double* out, cudaStream_t stream,
                                   bool naive) {
    const long long work = count * b * (1LL << (mu - 1));
    build_lut_exact_kernel<T><<<blocks_for(work, 256), 256, 0, stream>>>(x, x_rows, b, mu, g0, count,
                                                                        key_major ? 1 : 0, naive ? 1 : 0, out);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_biqgemm_exact(const void* keys, const T* alpha, const T* x, long long x_rows, T* y,
                                 long long m, long long n, int beta, int mu, long long b, void* workspace,
                                 size_t workspace_bytes, cudaStream_t stream, bool naive, const PhaseMarks* marks) {
    auto mark = [&](int phase) {
        if (marks) marks->mark(marks->ctx, phase, stream);
    };
    if (workspace_bytes < exact_workspace_bytes(m, n, beta, mu, b)) return cudaErrorInvalidValue;
    const long long groups = (n + mu - 1) / mu;
    const size_t acc_bytes = static_cast<size_t>(beta) * m * b * sizeof(double);
    double* acc = static_cast<double*>(workspace);
    double* lut = reinterpret_cast<double*>(static_cast<char*>(workspace) + ((acc_bytes + 255) / 256) * 256);
    cudaError_t e = cudaMemsetAsync(acc, 0, acc_bytes, stream);
    if (e != cudaSuccess) return e;
    const long long tg = tile_groups(groups, mu, b);
    for (long long g0 = 0; g0 < groups; g0 += tg) {
        const long long count = std::min(tg, groups - g0);
        mark(0);
        e = launch_build_lut_exact<T>(x, x_rows, b, mu, g0, count, false, lut, stream, naive);
        if (e != cudaSuccess) return e;
        mark(1);
        const long long work = static_cast<long long>(beta) * m * b;
        if (mu <= 8) {
            query_exact_kernel<uint8_t><<<blocks_for(work, 256), 256, 0, stream>>>(
                static_cast<const uint8_t*>(keys), lut, m, groups, beta, mu, b, g0, count, acc);
        } else {
            query_exact_kernel<uint16_t><<<blocks_for(work, 256), 256, 0, stream>>>(
                static_cast<const uint16_t*>(keys), lut, m, groups, beta, mu, b, g0, count, acc);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    mark(2);
    epilogue_exact_kernel<T><<<blocks_for(m * b, 256), 256, 0, stream>>>(acc, alpha, m, beta, b, y);
    return cudaGetLastError();
}

template cudaError_t launch_build_lut_exact<float>(const float*, long long, long long, int, long long,
                                                   long long, bool, double*, cudaStream_t, bool);
template cudaError_t launch_build_lut_exact<double>(const double*, long long, long long, int, long long,
                                                    long long, bool, double*, cudaStream_t, bool);
template cudaError_t launch_biqgemm_exact<float>(const void*, const float*, const float*, long long, float*,
                                                 long long, long long, int, int, long long, void*, size_t,
                                                 cudaStream_t, bool, const PhaseMarks*);
template cudaError_t launch_biqgemm_exact<double>(const void*, const double*, const double*, long long,
                                                  double*, long long, long long, int, int, long long, void*,
                                                  size_t, cudaStream_t, bool, const PhaseMarks*);

}  // namespace bqg
