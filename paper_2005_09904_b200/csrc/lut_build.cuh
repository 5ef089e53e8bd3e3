// lut_build.cuh -- in-shared-memory LUT construction (replaces
// build_lut_block / build_lut_dp, /root/reference/proj/core/include/biqgemm/
// lut.hpp:50-69,109-154).
//
// Placement ("bank-owned"): one CTA owns a block of 32 consecutive groups and
// BT input columns.  The BT tables of group gb*32+l are interleaved per key
// and live in the bank(s) lane l owns:
//     word((k, l, c)) = k * KROW + l * BT + c          (k = key, c = column)
// with KROW = 32*BT (or 64 for BT = 1, see the query kernel).
// During the query lane l (which handles group gb*32+l) gathers BT
// consecutive floats at (k*32+l)*BT: a warp-wide gather touches every bank
// exactly once per wavefront (LDS.32 / .64 / .128 for BT = 1 / 2 / 4), i.e.
// it is conflict-free.  Building is conflict-free too: lane l writes a
// BT-vector into its own slot (STS.32 / .64 / .128).
//
// Order of operations (bit-exact with lut.hpp:50-69 evaluated in fp32):
//   e[0] = ((0 - x0) - x1) - ... - x_{mu-1}
//   e[k] = e[k - 2^top(k)] + 2*x_top(k)            for 0 < k < 2^(mu-1)
//   e[2^mu - 1 - k] = -e[k]
// Unrolled, e[k] = e0 + s_{b1} + s_{b2} + ... over the set bits of k in
// ascending order, left-associated.  The NW warps of the CTA split the first
// half into 2^(mu-1-L) chunks of 2^L consecutive keys: warp w runs the DP over
// the low L bits (identical to the reference's first L rounds), then adds the
// steps of the chunk index bits in ascending order -- exactly the additions
// the sequential DP performs for those entries.
#pragma once

#include "common.cuh"

namespace bqg {

template <int N>
struct Log2 {
    static constexpr int value = 1 + Log2<N / 2>::value;
};
template <>
struct Log2<1> {
    static constexpr int value = 0;
};

template <int BT>
struct VecT;
template <>
struct VecT<1> {
    using type = float;
};
template <>
struct VecT<2> {
    using type = float2;
};
template <>
struct VecT<4> {
    using type = float4;
};

template <int BT>
__device__ __forceinline__ void store_vec(float* dst, const float (&v)[BT], bool negate) {
    if constexpr (BT == 1) {
        *dst = negate ? -v[0] : v[0];
    } else if constexpr (BT == 2) {
        *reinterpret_cast<float2*>(dst) = negate ? make_float2(-v[0], -v[1]) : make_float2(v[0], v[1]);
    } else {
        *reinterpret_cast<float4*>(dst) = negate ? make_float4(-v[0], -v[1], -v[2], -v[3])
                                                 : make_float4(v[0], v[1], v[2], v[3]);
    }
}

// Builds, for this lane's group g and input columns col0 .. col0+BT-1, all
// 2^MU entries into the bank-owned block at `lut` (shared memory).
//   x : input, x_rows x b row-major (x(r, c) at r*b + c); rows >= x_rows are
//       zero (lut.hpp:133-136; kernel.hpp:132 lets x be shorter than n).
//       Columns >= b are clamped to b-1 (their outputs are never stored).
// Called by all NW warps of the CTA with the same g per lane; warp `warp`
// writes its chunk.  Caller must __syncthreads() afterwards.
// KROW: words per key row (>= 32*BT).  The query kernel uses KROW = 64 for
// BT = 1 so that a key sits at bit 8 of the byte address (PRMT addressing).
template <int MU, int NW, int BT, int KROW = 32 * BT>
__device__ __forceinline__ void build_bank_owned_tables(float* lut, const float* __restrict__ x,
                                                        long long x_rows, long long b, long long g,
                                                        long long col0, int warp, int lane) {
    constexpr int L = (MU - 1) < 2 ? (MU - 1) : 2;  // low bits per chunk (chunk = 2^L keys)
    constexpr int NCH = 1 << (MU - 1 - L);           // chunks in the first half
    constexpr int TABLE = 1 << MU;
    if (warp >= NCH) return;

    float xv[MU][BT];
    if constexpr (BT == 1 && MU % 4 == 0) {
        // b == 1 here (BT = 1 is only used for one input column): the group's
        // MU inputs are contiguous -> 16-byte loads.
        const long long r0 = g * MU;
        if (b == 1 && r0 + MU <= x_rows && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < MU / 4; ++q) {
                const float4 v = __ldcg(reinterpret_cast<const float4*>(x + r0 + 4 * q));
                xv[4 * q + 0][0] = v.x;
                xv[4 * q + 1][0] = v.y;
                xv[4 * q + 2][0] = v.z;
                xv[4 * q + 3][0] = v.w;
            }
        } else {
#pragma unroll
            for (int t = 0; t < MU; ++t) {
                const long long r = r0 + t;
                xv[t][0] = r < x_rows ? ld_cg_f32(x + r * b + min(col0, b - 1)) : 0.0f;
            }
        }
    } else {
#pragma unroll
        for (int t = 0; t < MU; ++t) {
            const long long r = g * MU + t;
#pragma unroll
            for (int c = 0; c < BT; ++c) {
                const long long col = min(col0 + c, b - 1);
                xv[t][c] = r < x_rows ? ld_cg_f32(x + r * b + col) : 0.0f;
            }
        }
    }
    // e0 and the low-chunk DP (identical to the reference's first L rounds)
    float low[1 << L][BT];
#pragma unroll
    for (int c = 0; c < BT; ++c) {
        float e0 = 0.0f;
#pragma unroll
        for (int t = 0; t < MU; ++t) e0 = __fsub_rn(e0, xv[t][c]);
        low[0][c] = e0;
#pragma unroll
        for (int i = 1; i <= L; ++i) {
            const float step = 2.0f * xv[i - 1][c];
            const int half = 1 << (i - 1);
#pragma unroll
            for (int j = 0; j < half; ++j) low[j + half][c] = fadd_rn(low[j][c], step);
        }
    }
#pragma unroll 1
    for (int ch = warp; ch < NCH; ch += NW) {
#pragma unroll
        for (int j = 0; j < (1 << L); ++j) {
            float v[BT];
#pragma unroll
            for (int c = 0; c < BT; ++c) {
                float e = low[j][c];
#pragma unroll
                for (int t = L; t < MU - 1; ++t) {
                    const float st = 2.0f * xv[t][c];
                    e = ((ch >> (t - L)) & 1) ? fadd_rn(e, st) : e;
                }
                v[c] = e;
            }
            const int k = (ch << L) + j;
            store_vec<BT>(lut + k * KROW + lane * BT, v, false);
            store_vec<BT>(lut + (TABLE - 1 - k) * KROW + lane * BT, v, true);
        }
    }
}

// x staged once per CTA: xs[(rl)*BT + c] = x(gb*32*MU + rl, col0 + c) for the
// block's 32*MU input rows (0 past x_rows or past b).  Coalesced cooperative
// load by `nthreads` threads; caller synchronises before the build.
template <int MU, int BT>
__device__ __forceinline__ void stage_x_tile(float* xs, const float* __restrict__ x, long long x_rows, long long b,
                                             long long gb, long long col0, int tid, int nthreads) {
    const long long r0 = gb * 32 * MU;
    for (int idx = tid; idx < 32 * MU * BT; idx += nthreads) {
        const int rl = idx / BT, c = idx - (idx / BT) * BT;
        const long long r = r0 + rl, col = col0 + c;
        xs[idx] = (r < x_rows && col < b) ? __ldcg(x + r * b + col) : 0.0f;
    }
}

// The staged x tile in shared memory: lane l's MU x BT inputs (its group's
// rows, BT columns) at xs + l*XS.  XS = BT * (MU rounded up to odd): with an
// odd number of BT-vectors per lane the build's per-lane vector reads hit
// distinct banks (an unpadded 32*BT-word stride put all 32 lanes on one bank
// group: 32-way conflicts, ~1.6 us of a 2.2 us BT = 4 build).
__host__ __device__ constexpr int xs_stride(int mu, int bt) { return bt * (mu % 2 == 0 ? mu + 1 : mu); }
__host__ __device__ constexpr int xs_words(int mu, int bt) { return 32 * xs_stride(mu, bt); }
// Slot of element idx = (block row rl) * BT + column of the unpadded tile.
template <int MU, int BT>
__device__ __forceinline__ int xs_slot(int idx) {
    const int rl = idx / BT, c = idx - (idx / BT) * BT;
    return (rl / MU) * xs_stride(MU, BT) + (rl - (rl / MU) * MU) * BT + c;
}

// build_bank_owned_tables with x read from the staged shared-memory tile
// (identical arithmetic and order; lane l owns group gb*32 + l).
template <int MU, int NW, int BT, int KROW = 32 * BT>
__device__ __forceinline__ void build_bank_owned_tables_smem(float* lut, const float* xs, int warp, int lane) {
    constexpr int L = (MU - 1) < 2 ? (MU - 1) : 2;
    constexpr int NCH = 1 << (MU - 1 - L);
    constexpr int TABLE = 1 << MU;
    if (warp >= NCH) return;
    float xv[MU][BT];
    const float* xl = xs + lane * xs_stride(MU, BT);  // 16-byte aligned for BT = 4, 8 for BT = 2
#pragma unroll
    for (int t = 0; t < MU; ++t) {
        if constexpr (BT == 4) {
            const float4 v = *reinterpret_cast<const float4*>(xl + t * 4);
            xv[t][0] = v.x;
            xv[t][1] = v.y;
            xv[t][2] = v.z;
            xv[t][3] = v.w;
        } else if constexpr (BT == 2) {
            const float2 v = *reinterpret_cast<const float2*>(xl + t * 2);
            xv[t][0] = v.x;
            xv[t][1] = v.y;
        } else {
            xv[t][0] = xl[t];
        }
    }
    float low[1 << L][BT];
#pragma unroll
    for (int c = 0; c < BT; ++c) {
        float e0 = 0.0f;
#pragma unroll
        for (int t = 0; t < MU; ++t) e0 = __fsub_rn(e0, xv[t][c]);
        low[0][c] = e0;
#pragma unroll
        for (int i = 1; i <= L; ++i) {
            const float step = 2.0f * xv[i - 1][c];
            const int half = 1 << (i - 1);
#pragma unroll
            for (int j = 0; j < half; ++j) low[j + half][c] = fadd_rn(low[j][c], step);
        }
    }
#pragma unroll 1
    for (int ch = warp; ch < NCH; ch += NW) {
#pragma unroll
        for (int j = 0; j < (1 << L); ++j) {
            float v[BT];
#pragma unroll
            for (int c = 0; c < BT; ++c) {
                float e = low[j][c];
#pragma unroll
                for (int t = L; t < MU - 1; ++t) {
                    const float st = 2.0f * xv[t][c];
                    e = ((ch >> (t - L)) & 1) ? fadd_rn(e, st) : e;
                }
                v[c] = e;
            }
            const int k = (ch << L) + j;
            store_vec<BT>(lut + k * KROW + lane * BT, v, false);
            store_vec<BT>(lut + (TABLE - 1 - k) * KROW + lane * BT, v, true);
        }
    }
}

}  // namespace bqg
