// quantize.cu -- offline producers of the hot path's inputs, on the GPU.
//
//   quantize_greedy_kernel : quantize.hpp:27-58 (greedy binary coding, per-row alpha)
//   pack_keys_kernel       : packing.hpp:84-107 (mu-bit keys, row-major, u8/u16)
//   tile_keys_kernel       : row-major keys -> the query kernel's tiled layout
//
// Bit-exactness: quantize_greedy sums |residual| sequentially in fp64 per row
// (quantize.hpp:46-47).  One thread owns one row and walks its columns in
// ascending order, so alpha is the same double the reference computes; the
// residual of plane i is recomputed as ((w - a0*s0) - a1*s1) ... - a_{i-1}*s_{i-1}
// in the reference's order (a_j*s_j is exact since s_j = +-1), so every sign
// bit matches.  W is staged through shared memory 32x32 tiles so global reads
// are coalesced while each thread still sees its own row in order.
#include "common.cuh"
#include "kernels.h"

namespace bqg {

namespace {

constexpr int kQWarps = 4;  // warps per CTA; each warp owns 32 rows

template <typename T>
__global__ void __launch_bounds__(kQWarps * 32)
    quantize_greedy_kernel(const T* __restrict__ w, long long m, long long n, int beta,
                           uint32_t* __restrict__ planes, T* __restrict__ alpha,
                           double* __restrict__ alpha_d) {
    __shared__ T tile[kQWarps][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r0 = (static_cast<long long>(blockIdx.x) * kQWarps + warp) * 32;
    if (r0 >= m) return;
    const long long r = r0 + lane;
    const bool row_ok = r < m;
    const long long wpr = (n + 31) / 32;
    T(*t)[33] = tile[warp];

    for (int i = 0; i < beta; ++i) {
        // pass A: alpha_i = (sequential sum |res_i|) / n
        double abs_sum = 0.0;
        for (long long c0 = 0; c0 < n; c0 += 32) {
            __syncwarp();
#pragma unroll 4
            for (int rr = 0; rr < 32; ++rr) {
                const long long rg = r0 + rr, c = c0 + lane;
                t[rr][lane] = (rg < m && c < n) ? w[rg * n + c] : T(0);
            }
            __syncwarp();
            if (row_ok) {
                const int cols = static_cast<int>(min(32LL, n - c0));
                for (int j = 0; j < cols; ++j) {
                    double res = static_cast<double>(t[lane][j]);
                    for (int p = 0; p < i; ++p) {
                        const uint32_t word = planes[(static_cast<long long>(p) * m + r) * wpr + c0 / 32];
                        const double s = ((word >> j) & 1u) ? 1.0 : -1.0;
                        res = __dsub_rn(res, __dmul_rn(alpha_d[static_cast<long long>(p) * m + r], s));
                    }
                    abs_sum = __dadd_rn(abs_sum, fabs(res));
                }
            }
        }
        double a = 0.0;
        if (row_ok) {
            a = __ddiv_rn(abs_sum, static_cast<double>(n));
            alpha_d[static_cast<long long>(i) * m + r] = a;
            alpha[static_cast<long long>(i) * m + r] = static_cast<T>(a);  // T(alpha), round to nearest
        }
        // pass B: sign bits of res_i (sign(0) = +1, quantize.hpp:51)
        for (long long c0 = 0; c0 < n; c0 += 32) {
            __syncwarp();
#pragma unroll 4
            for (int rr = 0; rr < 32; ++rr) {
                const long long rg = r0 + rr, c = c0 + lane;
                t[rr][lane] = (rg < m && c < n) ? w[rg * n + c] : T(0);
            }
            __syncwarp();
            if (row_ok) {
                const int cols = static_cast<int>(min(32LL, n - c0));
                uint32_t word = 0;
                for (int j = 0; j < cols; ++j) {
                    double res = static_cast<double>(t[lane][j]);
                    for (int p = 0; p < i; ++p) {
                        const uint32_t pw = planes[(static_cast<long long>(p) * m + r) * wpr + c0 / 32];
                        const double s = ((pw >> j) & 1u) ? 1.0 : -1.0;
                        res = __dsub_rn(res, __dmul_rn(alpha_d[static_cast<long long>(p) * m + r], s));
                    }
                    if (!(res < 0.0)) word |= 1u << j;
                }
                planes[(static_cast<long long>(i) * m + r) * wpr + c0 / 32] = word;
            }
        }
    }
}

// keys(r, g) = sum_{t < mu, g*mu+t < n} bit(r, g*mu+t) << t   (packing.hpp:84-107)
template <typename K>
__global__ void pack_keys_kernel(const uint32_t* __restrict__ plane, long long m, long long n,
                                 int mu, long long groups, K* __restrict__ keys) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= m * groups) return;
    const long long r = idx / groups, g = idx - r * groups;
    const long long wpr = (n + 31) / 32;
    const uint32_t* row = plane + r * wpr;
    uint32_t key = 0;
    for (int t = 0; t < mu; ++t) {
        const long long c = g * mu + t;
        if (c < n && ((row[c >> 5] >> (c & 31)) & 1u)) key |= 1u << t;
    }
    keys[idx] = static_cast<K>(key);
}

// Row-major u8 keys [beta][m][G] -> tiled layout (see kernels.h):
//   chunk(gb, t, i) = ((gb*MT + t)*beta + i) * 1024 bytes
//   within a chunk, lane l (row t*32 + l) owns the 16-byte pieces at l*16 and
//   512 + l*16; its byte j (piece j>>4, byte j&15) is the key of group
//   gb*32 + ((l + j) mod 32).
// Padding rows/groups are 0.  One thread per output byte (coalesced writes).
__global__ void tile_keys_kernel(const uint8_t* __restrict__ keys, long long m, long long groups,
                                 int beta, long long MT, long long NB, uint8_t* __restrict__ out) {
    const long long total = NB * MT * beta * 1024;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const int within = static_cast<int>(idx & 1023);
    const int l = (within >> 4) & 31;
    const int j = ((within >> 9) << 4) | (within & 15);
    const int gl = (l + j) & 31;
    long long chunk = idx >> 10;
    const int i = static_cast<int>(chunk % beta);
    chunk /= beta;
    const long long t = chunk % MT;
    const long long gb = chunk / MT;
    const long long r = t * 32 + l, g = gb * 32 + gl;
    uint8_t v = 0;
    if (r < m && g < groups) v = keys[(static_cast<long long>(i) * m + r) * groups + g];
    out[idx] = v;
}

// Re-key mu-bit keys (u8 for mu <= 8, u16 above) to mu = 8: byte g8 of row r
// holds the sign bits of weights 8*g8 .. 8*g8+7 (bit t = weight 8*g8 + t,
// packing.hpp:61-81's order), i.e. bit (8*g8 + t) % mu of key (8*g8 + t) / mu;
// bits past the G*mu bits of a row are 0 -- exactly the pad bits the keys
// carry past n, so every x row the mu-keys accept meets the same sign.
template <typename K>
__global__ void rekey_mu8_kernel(const K* __restrict__ keys, long long rows, long long groups, int mu,
                                 long long groups8, uint8_t* __restrict__ out) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows * groups8) return;
    const long long r = idx / groups8, g8 = idx - r * groups8;
    const K* kr = keys + r * groups;
    unsigned v = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const long long w = g8 * 8 + t, g = w / mu;
        if (g < groups) v |= ((static_cast<unsigned>(kr[g]) >> static_cast<int>(w - g * mu)) & 1u) << t;
    }
    out[idx] = static_cast<uint8_t>(v);
}

}  // namespace

cudaError_t launch_rekey_mu8(const void* keys, long long rows, long long groups, int mu, long long groups8,
                             uint8_t* out, cudaStream_t stream) {
    const long long total = rows * groups8;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    if (mu <= 8)
        rekey_mu8_kernel<uint8_t><<<grid, 256, 0, stream>>>(static_cast<const uint8_t*>(keys), rows, groups, mu, groups8, out);
    else
        rekey_mu8_kernel<uint16_t><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(keys), rows, groups, mu, groups8,
                                                            out);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_quantize_greedy(const T* w, long long m, long long n, int beta,
                                   uint32_t* planes, T* alpha, double* alpha_d,
                                   cudaStream_t stream) {
    const long long rows_per_cta = kQWarps * 32;
    const unsigned grid = static_cast<unsigned>((m + rows_per_cta - 1) / rows_per_cta);
    quantize_greedy_kernel<T><<<grid, kQWarps * 32, 0, stream>>>(w, m, n, beta, planes, alpha, alpha_d);
    return cudaGetLastError();
}
template cudaError_t launch_quantize_greedy<float>(const float*, long long, long long, int, uint32_t*, float*,
                                                   double*, cudaStream_t);
template cudaError_t launch_quantize_greedy<double>(const double*, long long, long long, int, uint32_t*, double*,
                                                    double*, cudaStream_t);

cudaError_t launch_pack_keys(const uint32_t* plane, long long m, long long n, int mu,
                             void* keys, cudaStream_t stream) {
    const long long groups = (n + mu - 1) / mu;
    const long long total = m * groups;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    if (mu <= 8) {
        pack_keys_kernel<uint8_t><<<grid, 256, 0, stream>>>(plane, m, n, mu, groups,
                                                            static_cast<uint8_t*>(keys));
    } else {
        pack_keys_kernel<uint16_t><<<grid, 256, 0, stream>>>(plane, m, n, mu, groups,
                                                             static_cast<uint16_t*>(keys));
    }
    return cudaGetLastError();
}

cudaError_t launch_tile_keys(const uint8_t* keys, long long m, long long groups, int beta,
                             uint8_t* tiled, cudaStream_t stream) {
    const long long MT = (m + 31) / 32, NB = (groups + 31) / 32;
    const long long total = NB * beta * MT * 1024;
    const unsigned grid = static_cast<unsigned>((total + 255) / 256);
    tile_keys_kernel<<<grid, 256, 0, stream>>>(keys, m, groups, beta, MT, NB, tiled);
    return cudaGetLastError();
}

}  // namespace bqg
