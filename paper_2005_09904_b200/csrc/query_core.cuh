// query_core.cuh -- the per-chunk LUT gather shared by the fast kernels.
#pragma once

#include "common.cuh"

namespace bqg {

// Words per key row of the shared-memory LUT.  BT = 1 uses 64 (half the row
// unused) so the key lands at bit 8 of the byte address: one PRMT builds the
// whole address (key byte -> byte 1, rotated bank offset -> byte 0).  BT = 2
// is byte-aligned natively (row = 256 bytes); BT = 4 (512-byte rows) uses
// SHF + LOP3.
template <int BT>
struct LutGeom {
    static constexpr int KROW = BT == 1 ? 64 : 32 * BT;
    static constexpr bool PRMT = BT <= 2;
};

template <int BT>
__device__ __forceinline__ void lds_vec(uint32_t addr, float (&e)[BT]) {
    if constexpr (BT == 1) {
        asm("ld.shared.f32 %0, [%1];" : "=f"(e[0]) : "r"(addr));
    } else if constexpr (BT == 2) {
        asm("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(e[0]), "=f"(e[1]) : "r"(addr));
    } else {
        asm("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(e[0]), "=f"(e[1]), "=f"(e[2]), "=f"(e[3]) : "r"(addr));
    }
}

// One 1 KiB chunk (32 rows x 32 groups of one plane), BT input columns.
// Lane l holds the 32 keys of row l: byte j = key(row l, group (l+j) mod 32).
// goff[j] = the lane's rotated bank offset for step j (the same for every
// chunk, kept in registers).  Sums are kept in 4 interleaved accumulators and
// combined pairwise at the end.
// ABS = true: goff already holds the LUT's 64 KiB-aligned shared address in
// bits 16..31 (PRMT keeps them), so the gather address needs no add.
template <int MU, int BT, bool ABS = false>
__device__ __forceinline__ void gather_chunk(const uint32_t (&w)[8], uint32_t lut_s, const uint32_t (&goff)[32],
                                             float (&out)[BT]) {
    float acc[4][BT];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < BT; ++c) acc[a][c] = 0.0f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t wv = w[j >> 2];
        const int bi = j & 3;
        uint32_t off;
        if constexpr (LutGeom<BT>::PRMT) {
            // byte0 <- goff.b0, byte1 <- key byte bi, bytes 2,3 <- goff.b2,b3
            off = __byte_perm(goff[j], wv, 0x3200u | ((4u + bi) << 4));
        } else {
            constexpr int SH = 9;
            constexpr uint32_t MASK = ((1u << MU) - 1u) << SH;
            const int sft = 8 * bi - SH;
            const uint32_t sh = sft >= 0 ? (wv >> sft) : (wv << (-sft));
            off = (sh & MASK) | goff[j];
        }
        float e[BT];
        lds_vec<BT>(ABS ? off : lut_s + off, e);
#pragma unroll
        for (int c = 0; c < BT; ++c) acc[j & 3][c] += e[c];
    }
#pragma unroll
    for (int c = 0; c < BT; ++c) out[c] = (acc[0][c] + acc[1][c]) + (acc[2][c] + acc[3][c]);
}

}  // namespace bqg
