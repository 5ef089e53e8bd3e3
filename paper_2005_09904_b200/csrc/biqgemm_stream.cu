// biqgemm_stream.cu -- the grouped ("stream") BiQGEMM form: b == 1, mu == 8,
// 1 <= beta <= 4, for a GROUP of independent calls that share (m, n, beta,
// mu) -- e.g. the Q/K/V or gate/up projections of one layer, or the
// per-request GEMVs of a serving batch.  Each call is a full
// biqgemm::biqgemm (/root/reference/proj/core/include/biqgemm/kernel.hpp:
// 246-258 -> detail::run 116-204): its own x, its own LUT build
// (lut.hpp:50-69,109-154), its own key stream and alpha epilogue
// (kernel.hpp:183-195).  Nothing is shared or skipped between calls; the
// group exists so that consecutive calls overlap on the device instead of
// paying a kernel boundary (~1 us of handoff, tools/ubench/pdl_overlap.cu)
// each.
//
// Work split.  A call's keys are NB x MT "units" (unit = one 32-group block
// x one 32-row tile x all beta planes = beta KiB of the tiled layout, and
// unit u = gb*MT + t sits at byte u*beta*1024: kernels.h).  CTA c owns the
// contiguous unit range [c*W/grid, (c+1)*W/grid) of EVERY call (W = NB*MT,
// grid >= NB so a range spans at most two group blocks).  Per CTA:
//
//   key warp   : one lane streams the CTA's unit range of call 0, 1, 2, ...
//                global -> shared with cp.async.bulk (TMA bulk engine,
//                L2::evict_first) through an R-stage mbarrier ring that
//                runs ahead across call boundaries -- HBM never waits for a
//                call boundary.
//   x warp     : loads x of call c+1 (the <= 2 blocks' 256 rows each) into a
//                double-buffered shared tile one call ahead.
//   15 consumer warps, per call c:
//       one named barrier (everybody is done with call c-1 and LUT(c) is
//       complete), build their share of LUT(c+1) into the other of two
//       64 KiB LUT buffers (bank-owned DP tables, bit-exact with the fp32
//       DP, lut_build.cuh), then gather their units of call c: lane l = row
//       l of the tile, step j reads table (l+j) mod 32 -> one conflict-free
//       wavefront per 32 lookups; address = ONE PRMT (key byte -> bits
//       8..15, rotated bank -> bits 2..6, buffer base -> bits 16..31; the
//       second block of a CTA that spans two sits at +128 B, an LDS
//       immediate).  Per unit the beta plane sums are combined with alpha in
//       fp64 and stored as ONE fp32 partial per (call, block, row).
//   stream_finalize_kernel (PDL-chained): y_c[r] = sum over blocks (fp64,
//       blocks ascending) -> f32.
//
// Every output's reduction tree is a function of (n, mu) only (gather order
// within a block, planes ascending, blocks ascending), so y is bitwise
// independent of the grid, the group size and any 32-row-aligned row
// sharding.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "lut_build.cuh"  // Log2

namespace bqg {

namespace {

constexpr int kMU = 8;
constexpr int kTable = 1 << kMU;
#ifndef BQG_STREAM_NC
#define BQG_STREAM_NC 18
#endif
constexpr int kNC = BQG_STREAM_NC;               // consumer (gather) warps
constexpr int kWKey = kNC;                       // key-stream warp
constexpr int kWX = kNC + 1, kWA = kNC + 2;      // x loader, alpha loader
constexpr int kWBuild = kNC + 3;                 // LUT builder warps
#ifndef BQG_STREAM_NBUILD
#define BQG_STREAM_NBUILD 4
#endif
constexpr int kNBuild = BQG_STREAM_NBUILD;       // 1, 2, 4 or 8
constexpr int kSThreads = (kNC + 3 + kNBuild) * 32;
constexpr uint32_t kAlphaBudget = 48 * 1024;     // all alpha buffers together
constexpr int kMaxStages = 24;
constexpr int kStreamSmem = 227 * 1024;          // opt-in maximum per CTA
constexpr int kXBlock = 32 * kMU;                // x rows per group block

struct StreamArgs {
    int ncalls;
    long long x_rows;
    int m, NB, MT, cpb, grid, ups;
    int debug;       // BQG_DEBUG_FLAGS (profiling / A/B switches; 0 in production)
    float* partial;  // ncalls x NB x (MT*32), fp32
    StreamCall calls[kStreamMaxGroup];
};

// ---------------------------------------------------------------- LUT build
// The table of group gb*32 + lane lives in bank `lane`: entry k of buffer
// half h at byte  base + k*256 + h*128 + lane*4.  The first half (keys <
// 128) is the DP recurrence of lut.hpp:50-69 evaluated in fp32,
//     e[0] = ((0 - x0) - x1) - ... - x7,   e[k] = e[k - 2^top(k)] + 2*x_top(k),
// and the second half its negation, e[255 - k] = -e[k] (lut.hpp:63-66).  The
// recurrence tree is walked depth-first at compile time (parent -> child =
// one fadd), so every entry is produced by exactly the reference's addition
// and the live state is one value per tree level.  With NB builder warps
// (NB = 2^h, h <= 3), builder q owns the keys whose top h first-half bits
// (bits 7-h .. 6) equal q:
//     e[j | q << (7-h)] = ((e[j] (+ 2*x_{7-h})) ...) (+ 2*x6)     for j < 2^(7-h),
// the recurrence's own order (each builder re-walks the j < 2^(7-h) subtree).
__device__ __forceinline__ void sts_pair(uint32_t col, int k, float v) {
    sts_f32(col + static_cast<uint32_t>(k) * 256u, v);
    sts_f32(col + static_cast<uint32_t>(kTable - 1 - k) * 256u, -v);
}

template <int K, int I, int Q, int LB>  // LB = low bits walked by the DFS (7 - h)
struct Dfs {
    static __device__ __forceinline__ void children(float v, const float (&s)[kMU], uint32_t col) {
        if constexpr (I < LB) {
            Dfs<(K | (1 << I)), I + 1, Q, LB>::node(fadd_rn(v, s[I]), s, col);
            Dfs<K, I + 1, Q, LB>::children(v, s, col);
        }
    }
    static __device__ __forceinline__ void node(float v, const float (&s)[kMU], uint32_t col) {
        float e = v;
#pragma unroll
        for (int t = LB; t < 7; ++t)
            if ((Q >> (t - LB)) & 1) e = fadd_rn(e, s[t]);
        sts_pair(col, K | (Q << LB), e);
        children(v, s, col);
    }
};

template <int NBW>
__device__ __forceinline__ void build_tables(int which, uint32_t col, const float* xb, int lane) {
    constexpr int LB = 7 - Log2<NBW>::value;
    float x[kMU], s[kMU];
#pragma unroll
    for (int t = 0; t < kMU; ++t) x[t] = xb[lane * kMU + t];
    float e0 = 0.0f;
#pragma unroll
    for (int t = 0; t < kMU; ++t) e0 = __fsub_rn(e0, x[t]);
#pragma unroll
    for (int t = 0; t < kMU; ++t) s[t] = 2.0f * x[t];
    switch (which) {
        case 0: Dfs<0, 0, 0, LB>::node(e0, s, col); break;
        case 1: if constexpr (NBW > 1) Dfs<0, 0, 1, LB>::node(e0, s, col); break;
        case 2: if constexpr (NBW > 2) Dfs<0, 0, 2, LB>::node(e0, s, col); break;
        case 3: if constexpr (NBW > 3) Dfs<0, 0, 3, LB>::node(e0, s, col); break;
        case 4: if constexpr (NBW > 4) Dfs<0, 0, 4, LB>::node(e0, s, col); break;
        case 5: if constexpr (NBW > 5) Dfs<0, 0, 5, LB>::node(e0, s, col); break;
        case 6: if constexpr (NBW > 6) Dfs<0, 0, 6, LB>::node(e0, s, col); break;
        default: if constexpr (NBW > 7) Dfs<0, 0, 7, LB>::node(e0, s, col); break;
    }
}

// ---------------------------------------------------------------- gather
// One 1 KiB chunk (32 rows x 32 groups of one plane): lane l sums its row's
// 32 lookups (4 interleaved accumulators combined pairwise, the order of
// gather_chunk in query_core.cuh).  The shared address of lookup j is ONE
// PRMT: byte 0 = the lane's rotated bank offset 4*((l+j) mod 32) (byte j%4
// of rot[j/4]), byte 1 = key byte j%4 of w[j/4], bytes 2-3 = the sign of a
// rot byte (< 128, so 0); the LUT base (64 KiB, kLutBase) and the buffer
// half (+128 B) are the LDS immediate.
constexpr uint32_t kLutBase = 0x10000u;

template <int IMM>
__device__ __forceinline__ float lds_lut(uint32_t rotw, uint32_t w, uint32_t sel) {
    uint32_t off;  // PTX prmt (not __byte_perm, which drops the sign-replicate bit of a selector nibble)
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(off) : "r"(rotw), "r"(w), "r"(sel));
    float e;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(e) : "r"(off), "n"(kLutBase + IMM));
    return e;
}

// The 4 interleaved accumulators acc[j % 4] are kept as two f32x2 pairs
// (acc0, acc1) and (acc2, acc3): one FADD2 adds lookups j and j+1 of the same
// 4-step group -- the same additions, in the same order, as 4 scalar chains.
__device__ __forceinline__ uint64_t pack2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float2 unpack2(uint64_t a) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(a));
    return r;
}

template <int IMM>
__device__ __forceinline__ float stream_gather(const uint32_t (&w)[8], const uint32_t (&rot)[8]) {
    uint64_t acc01 = 0, acc23 = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // lookups j = 4q .. 4q+3
        const float e0 = lds_lut<IMM>(rot[q], w[q], 0x8840u);
        const float e1 = lds_lut<IMM>(rot[q], w[q], 0x8851u);
        const float e2 = lds_lut<IMM>(rot[q], w[q], 0x8862u);
        const float e3 = lds_lut<IMM>(rot[q], w[q], 0x8873u);
        if (q == 0) {  // 0 + e == e (up to the sign of a zero sum)
            acc01 = pack2(e0, e1);
            acc23 = pack2(e2, e3);
        } else {
            acc01 = fadd2(acc01, pack2(e0, e1));
            acc23 = fadd2(acc23, pack2(e2, e3));
        }
    }
    const float2 a = unpack2(acc01), b = unpack2(acc23);
    return (a.x + a.y) + (b.x + b.y);
}

// beta chunks of one unit, combined with alpha in fp64 (planes ascending).
template <int BETA, int IMM>
__device__ __forceinline__ double stream_unit(uint32_t kbase, int lane, const uint32_t (&rot)[8],
                                              const float (&a)[BETA]) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < BETA; ++i) {
        uint32_t w[8];
        const uint32_t p = kbase + static_cast<uint32_t>(i) * 1024u + static_cast<uint32_t>(lane) * 16u;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(p));
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+512];" : "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "r"(p));
        const float P = stream_gather<IMM>(w, rot);
        s += static_cast<double>(a[i]) * static_cast<double>(P);
    }
    return s;
}

template <int BETA>
__global__ void __launch_bounds__(kSThreads, 1) biqgemm_stream_kernel(const __grid_constant__ StreamArgs A) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pdl_launch_dependents();

    // ---- this CTA's work: tiles [t0, t0+U) of group block gb, every call
    const int gb = blockIdx.x / A.cpb, jb = blockIdx.x - gb * A.cpb;
    const int t0 = static_cast<int>(static_cast<long long>(jb) * A.MT / A.cpb);
    const int U = static_cast<int>(static_cast<long long>(jb + 1) * A.MT / A.cpb) - t0;
    const long long u0 = static_cast<long long>(gb) * A.MT + t0;
    const int ncalls = A.ncalls;
    const int spc = (U + A.ups - 1) / A.ups;  // ring stages per call
    // alpha of the CTA's rows, staged per call in nab buffers ([BETA][U*32]):
    // 4 when they fit the budget (loads run up to 3 calls ahead), else 2; if
    // even 2 do not fit, gather warps load alpha themselves
    const uint32_t abuf_bytes = static_cast<uint32_t>(U) * BETA * 128u;
    // (2 buffers: measured faster than 4 -- the key ring keeps the room)
    const int nab = 2;
    const bool alpha_smem = static_cast<uint32_t>(nab) * abuf_bytes <= kAlphaBudget;

    // ---- shared memory:
    //   [bars 1K | x bufs 4x1K | alpha bufs | stages.. | LUT 64K | ..stages]
    // LUT buffer lb = (64 KiB region lb/2, half lb%2); the code supports up to
    // 4 buffers (two regions), the kernel uses nlb = 2.
    const uint32_t sbase = smem_u32(smem);
    // the LUT sits at offset kLutBase of the CTA's shared window (the
    // gather's LDS immediate); no cluster here, so no rank bits
    const uint32_t lut_abs = (sbase & 0xFF000000u) | kLutBase;
    const uint32_t send = sbase + kStreamSmem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    uint64_t* xfull = empty + kMaxStages;  // [4] x(c) loaded                (32 x-loader lanes)
    uint64_t* xempty = xfull + 4;          // [4] x(c) consumed               (kNBuild builders)
    uint64_t* lfull = xempty + 4;          // [4] LUT(c) built                (kNBuild builders)
    uint64_t* ldone = lfull + 4;           // [4] call c gathered: LUT free   (kNC consumers)
    uint64_t* afull = ldone + 4;           // [4] alpha(c) loaded             (32 alpha-loader lanes)
    uint64_t* adone = afull + 4;           // [4] call c gathered: alpha free (kNC consumers)
    // issued[slot] = 1 + the ring round last issued into the slot (release by
    // the key warp, acquire by a consumer before its parity wait on full[]):
    // slots refill independently, so without it a warp far ahead could wait
    // on a slot two rounds early, which the mbarrier parity cannot tell apart
    uint32_t* issued = reinterpret_cast<uint32_t*>(adone + 4);  // [kMaxStages]
    float* xs = reinterpret_cast<float*>(smem + 1024);                    // [4][kXBlock]
    float* as = reinterpret_cast<float*>(smem + 1024 + 4 * kXBlock * 4);  // [nab][BETA][U*32]
    const uint32_t stage_bytes = static_cast<uint32_t>(A.ups) * BETA * 1024u;
    const uint32_t lo0 =
        (sbase + 1024u + 4u * kXBlock * 4u + (alpha_smem ? static_cast<uint32_t>(nab) * abuf_bytes : 0u) + 127u) & ~127u;
    const int nlo = lo0 + stage_bytes <= lut_abs ? static_cast<int>((lut_abs - lo0) / stage_bytes) : 0;
    auto nhi_at = [&](uint32_t hi) { return hi + stage_bytes <= send ? static_cast<int>((send - hi) / stage_bytes) : 0; };
    // 2 LUT buffers (the halves of one 64 KiB region); 4 (a second region)
    // is supported by the protocol but measured slower: ring bytes matter more
    const int nlb = 2;
    const uint32_t hi0 = lut_abs + (nlb == 4 ? 0x20000u : 0x10000u);
    const int nst = min(kMaxStages, nlo + nhi_at(hi0));
    // layout assumption: dynamic shared memory starts below 64 KiB, so the
    // LUT sits at kLutBase (the gather's LDS immediate)
    if (sbase > lut_abs || lo0 > lut_abs || hi0 > send || nst < 2) __trap();
    auto stage_addr = [&](int slot) -> uint32_t {
        return slot < nlo ? lo0 + static_cast<uint32_t>(slot) * stage_bytes
                          : hi0 + static_cast<uint32_t>(slot - nlo) * stage_bytes;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], A.ups * 32);  // every lane of a unit's warp arrives
        }
        for (int b = 0; b < 4; ++b) {
            mbar_init(&xfull[b], 32);
            mbar_init(&xempty[b], kNBuild * 32);
            mbar_init(&lfull[b], kNBuild * 32);
            mbar_init(&ldone[b], kNC * 32);
        }
        for (int b = 0; b < 4; ++b) {
            mbar_init(&afull[b], 32);
            mbar_init(&adone[b], kNC * 32);
        }
        for (int s = 0; s < kMaxStages; ++s) issued[s] = 0;
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kWKey) {
        // ---------------------------------------------------- key stream
        // Stages are call-aligned: call c's U units fill spc = ceil(U/ups)
        // stages (the last one possibly partial), stage s = c*spc + j.
        // Lane L owns ring slot L (stages L, L+nst, ...): the bulk copies of
        // different stages are issued by different lanes, in parallel (one
        // issuing thread caps the copy rate at ~3 TB/s chip-wide with 8-12
        // KiB copies; several reach ~7 TB/s: tools/ubench/tma_stream.cu).
        // The issued-round guard (issued[]) is what keeps the protocol sound;
        // stages need no gating on the calls' LUT/alpha readiness
        // (tools/stream_protocol_sim.py models the protocol).
        if (lane < nst) {
            const uint64_t pol = policy_evict_first();
            const long long nstages_total = static_cast<long long>(ncalls) * spc;
            const int slot = lane;
            auto issue = [&](long long s) {
                const int c = static_cast<int>(s / spc), j = static_cast<int>(s - static_cast<long long>(c) * spc);
                const int k0 = j * A.ups, len = min(A.ups, U - k0);
                const uint32_t bytes = static_cast<uint32_t>(len) * BETA * 1024u;
                mbar_arrive_expect_tx(&full[slot], bytes);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
                    "[%0], [%1], %2, [%3], %4;" ::"r"(stage_addr(slot)),
                    "l"(A.calls[c].keys + (u0 + k0) * BETA * 1024), "r"(bytes), "r"(smem_u32(&full[slot])), "l"(pol)
                    : "memory");
                // issued[slot] = round + 1 (one increment per round), as an atomic
                asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;" ::"r"(smem_u32(&issued[slot])) : "memory");
            };
            long long s0 = lane;
            // Stage 0 lands ALONE before the other lanes request theirs: a
            // whole-ring request from every CTA delays the first stage (C4
            // single call 12.67 -> 12.06 us, C2 group of one 6.68 -> 6.24;
            // BQG_DEBUG_FLAGS bit 21 restores the old order).  Every issuing
            // lane sees phase 0 of slot 0 before lane 0 can refill the slot
            // (the __syncwarp), so no lane tests a later phase of the same parity.
            if (nstages_total > 1 && !(A.debug & (1 << 21))) {
                if (lane == 0) issue(0);
                mbar_wait(&full[0], 0);
                __syncwarp(nst >= 32 ? 0xffffffffu : ((1u << nst) - 1u));
                if (lane == 0) s0 = nst;
            }
            for (long long s = s0; s < nstages_total; s += nst) {
                const long long round = s / nst;
                if (round > 0) mbar_wait_sleep(&empty[slot], static_cast<uint32_t>((round - 1) & 1));
                issue(s);
            }
        }
        return;
    }
    if (warp == kWX) {
        // ------------------------------ x(c) into buffer c%4, ahead of use
        // TMA bulk copy when the block's rows are 16-byte aligned and
        // complete; otherwise the 32 lanes copy (zero past x_rows).
        pdl_wait();
        const long long r0 = static_cast<long long>(gb) * kXBlock;
        for (int c = 0; c < ncalls; ++c) {
            const int buf = c & 3;
            if (c >= 4) mbar_wait_sleep(&xempty[buf], static_cast<uint32_t>(((c >> 2) - 1) & 1));
            const float* x = A.calls[c].x;
            float* xd = xs + buf * kXBlock;
            if (r0 + kXBlock <= A.x_rows && (reinterpret_cast<uintptr_t>(x + r0) & 15) == 0) {
                if (lane == 0) {
                    mbar_arrive_expect_tx(&xfull[buf], kXBlock * 4);
                    bulk_g2s_plain(xd, x + r0, kXBlock * 4, &xfull[buf]);
                } else {
                    mbar_arrive(&xfull[buf]);
                }
            } else {
                float v[kXBlock / 32];
#pragma unroll
                for (int q = 0; q < kXBlock / 32; ++q) {
                    const long long r = r0 + q * 32 + lane;
                    v[q] = r < A.x_rows ? __ldcg(x + r) : 0.0f;
                }
#pragma unroll
                for (int q = 0; q < kXBlock / 32; ++q) xd[q * 32 + lane] = v[q];
                mbar_arrive(&xfull[buf]);
            }
        }
        return;
    }
    if (warp == kWA) {
        // ------------------------- alpha(c) into buffer c % nab ([BETA][U*32])
        const long long ra = static_cast<long long>(t0) * 32;
        const long long arows = min(static_cast<long long>(U) * 32, static_cast<long long>(A.m) - ra);
        for (int c = 0; c < ncalls; ++c) {
            const int buf = c % nab;
            // afull runs at most nab phases ahead of the consumers (even when
            // alpha is not staged), so its parity waits never alias
            if (c >= nab) mbar_wait_sleep(&adone[buf], static_cast<uint32_t>((c / nab - 1) & 1));
            if (alpha_smem) {
                const float* al = A.calls[c].alpha;
                float* ad = as + buf * (abuf_bytes / 4);
                const uint32_t nbytes = static_cast<uint32_t>(arows) * 4u;
                const bool tma = al && (nbytes & 15) == 0 && (A.m & 3) == 0 &&
                                 (reinterpret_cast<uintptr_t>(al + ra) & 15) == 0;
                if (tma) {
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&afull[buf], nbytes * BETA);
#pragma unroll
                        for (int i = 0; i < BETA; ++i)
                            bulk_g2s_plain(ad + i * U * 32, al + static_cast<long long>(i) * A.m + ra, nbytes, &afull[buf]);
                    } else {
                        mbar_arrive(&afull[buf]);
                    }
                } else {
                    for (int i = 0; i < BETA; ++i) {
                        for (int k0 = 0; k0 < U * 32; k0 += 32 * 8) {
                            float v[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const long long rl = k0 + q * 32 + lane;
                                v[q] = (rl < arows) ? (al ? __ldg(al + static_cast<long long>(i) * A.m + ra + rl) : 1.0f)
                                                    : 0.0f;
                            }
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                if (k0 + q * 32 + lane < U * 32) ad[i * U * 32 + k0 + q * 32 + lane] = v[q];
                        }
                    }
                    mbar_arrive(&afull[buf]);
                }
            } else {
                mbar_arrive(&afull[buf]);
            }
        }
        return;
    }
    if (warp >= kWBuild) {
        // ------------------------------------ LUT(c) into buffer c % nlb
        const int which = warp - kWBuild;
        for (int c = 0; c < ncalls; ++c) {
            const int lb = c % nlb, xb = c & 3;
            mbar_wait(&xfull[xb], static_cast<uint32_t>((c >> 2) & 1));
            if (c >= nlb) mbar_wait(&ldone[lb], static_cast<uint32_t>((c / nlb - 1) & 1));
            build_tables<kNBuild>(which, lut_abs + static_cast<uint32_t>(lb >> 1) * 0x10000u + static_cast<uint32_t>(lb & 1) * 128u +
                                    static_cast<uint32_t>(lane) * 4u,
                         xs + xb * kXBlock, lane);
            // every lane releases its own table stores / x reads
            mbar_arrive(&xempty[xb]);
            mbar_arrive(&lfull[lb]);
        }
        return;
    }

    // ---------------------------------------------------------- consumers
    uint64_t pol_keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    uint32_t rot[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        rot[q] = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) rot[q] |= (static_cast<uint32_t>((lane + 4 * q + b) & 31) * 4u) << (8 * b);
    }
    pdl_wait();  // partials of the previous launch may still be read by its finaliser
    const long long MTP = static_cast<long long>(A.MT) * 32;
    // This warp's units are gu = warp, warp + kNC, ... of the CTA's (call,
    // unit) sequence (continuous across calls: balanced however U and kNC
    // relate).  Unit k of call c is in stage c*spc + k/ups at position
    // k%ups; the ring slot and phase advance incrementally.
    int gu = warp;
    long long st_cur = 0;  // global stage index that (slot, kround) describe
    int slot = 0;
    uint32_t kround = 0;
    for (int c = 0; c < ncalls; ++c) {
        const int lb = c % nlb;
        const int ab_i = c % nab;
        mbar_wait(&lfull[lb], static_cast<uint32_t>((c / nlb) & 1));
        mbar_wait(&afull[ab_i], static_cast<uint32_t>((c / nab) & 1));
        const float* alpha = A.calls[c].alpha;
        const float* ab = as + ab_i * (abuf_bytes / 4);
        float* part = A.partial + (static_cast<long long>(c) * A.NB + gb) * MTP;
        const int cbase = c * U;
        for (; gu < cbase + U; gu += kNC) {
            const int k = gu - cbase;
            const long long r = static_cast<long long>(t0 + k) * 32 + lane;
            const int sj = k / A.ups, pos = k - sj * A.ups;
            float a[BETA];
#pragma unroll
            for (int i = 0; i < BETA; ++i) {
                if (alpha_smem) a[i] = ab[(i * U + k) * 32 + lane];
                else a[i] = alpha ? (r < A.m ? __ldg(alpha + static_cast<long long>(i) * A.m + r) : 0.0f) : 1.0f;
            }
            const long long st = static_cast<long long>(c) * spc + sj;
            {
                long long d = st - st_cur;
                if (d >= nst) {
                    slot = static_cast<int>(st % nst);
                    kround = static_cast<uint32_t>(st / nst);
                } else {
                    slot += static_cast<int>(d);
                    if (slot >= nst) {
                        slot -= nst;
                        ++kround;
                    }
                }
                st_cur = st;
            }
            {
                uint32_t iss;
                do {
                    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(iss) : "r"(smem_u32(&issued[slot])) : "memory");
                } while (iss <= kround);
            }
            mbar_wait(&full[slot], kround & 1u);
            const uint32_t kbase = stage_addr(slot) + static_cast<uint32_t>(pos) * BETA * 1024u;
            // LUT buffer lb = half lb of the 64 KiB region (nlb = 2): +128 B
            const double sum = lb == 0 ? stream_unit<BETA, 0>(kbase, lane, rot, a)
                                       : stream_unit<BETA, 128>(kbase, lane, rot, a);
            {
                // every lane releases its key reads; the last unit of a
                // partial (call-final) stage completes the stage's count
                const int nin = min(A.ups, U - sj * A.ups);
                mbar_arrive_cnt(&empty[slot], pos == nin - 1 ? static_cast<uint32_t>(A.ups - nin + 1) : 1u);
            }
            if (r < A.m) {
                // partials stay in L2 for the epilogue (the key stream is evict_first)
                asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(part + r), "f"(static_cast<float>(sum)),
                             "l"(pol_keep)
                             : "memory");
            }
        }
        mbar_arrive(&ldone[lb]);  // every lane: its LUT and alpha reads of call c are done
        mbar_arrive(&adone[ab_i]);
    }
}

__global__ void __launch_bounds__(256) stream_finalize_kernel(const __grid_constant__ StreamArgs A) {
    // the next grouped launch may start now: its key stream does not depend
    // on us, and its x / partial accesses wait (griddepcontrol.wait) for this
    // grid to complete
    pdl_launch_dependents();
    pdl_wait();
    const int c = blockIdx.y;
    const long long r = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
    if (r >= A.m) return;
    const long long MTP = static_cast<long long>(A.MT) * 32;
    const float* p = A.partial + static_cast<long long>(c) * A.NB * MTP + r;
    double s = 0.0;
    for (int gb = 0; gb < A.NB; ++gb) s += static_cast<double>(__ldcs(p + gb * MTP));  // read once: evict first
    A.calls[c].y[r] = static_cast<float>(s);
}

template <int BETA>
cudaError_t launch_stream_beta(const StreamArgs& A, bool pdl, cudaStream_t stream) {
    static PerDeviceOnce configured;
    cudaError_t ea = once_per_device(configured, current_device(), [] {
        return cudaFuncSetAttribute(biqgemm_stream_kernel<BETA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kStreamSmem);
    });
    if (ea != cudaSuccess) return ea;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(A.grid));
    cfg.blockDim = dim3(kSThreads);
    cfg.dynamicSmemBytes = kStreamSmem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, biqgemm_stream_kernel<BETA>, A);
    if (e != cudaSuccess) return e;
    // finaliser: always PDL-chained behind the stream kernel
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(static_cast<unsigned>((A.m + 255) / 256), static_cast<unsigned>(A.ncalls));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    return cudaLaunchKernelEx(&cfg, stream_finalize_kernel, A);
}

}  // namespace

bool stream_supported(int mu, int beta, long long b) { return mu == kMU && b == 1 && beta >= 1 && beta <= 4; }

size_t stream_workspace_bytes(long long m, long long groups, int count) {
    const long long NB = (groups + 31) / 32, MT = (m + 31) / 32;
    const long long per = static_cast<long long>(std::min(count, kStreamMaxGroup));
    return kTexCounterBytes + static_cast<size_t>(per * NB * MT * 32) * sizeof(float);
}

int debug_flags_stream() {
    static const int f = [] {
        const char* e = getenv("BQG_DEBUG_FLAGS");
        return e ? atoi(e) : 0;
    }();
    return f;
}

int tex_min_group(long long m) {
    // Crossovers measured after the ring-start change (per call, PDL-chained
    // grouped launches, `profiles/ab_grouped_crossover_r2e.txt`): ~9 calls at
    // m = 4096 (beta 1 and 3), 13-16 at m = 8192-11008, 16-24 at 16384 -- the
    // texture form's fixed cost (the last calls' finalisation, one CTA per
    // call) grows with m.  9 * sqrt(m / 4096), at least kTexMinGroup.
    const double t = 9.0 * std::sqrt(static_cast<double>(m) / 4096.0);
    return std::max(kTexMinGroup, static_cast<int>(std::lround(t)));
}

cudaError_t launch_biqgemm_stream(const StreamCall* calls, int count, long long x_rows, int m, int G, int beta,
                                  float* ws, bool pdl, cudaStream_t stream) {
    static const int impl = [] {
        const char* v = getenv("BQG_STREAM_IMPL");
        return (v && v[0] == 't' && v[1] == 'm') ? 1 : 0;  // "tma": the TMA-ring form below
    }();
    // The texture form finalises in-kernel (the last CTA to finish a call sums
    // its partials), which pays off over a group; a call or two alone keeps
    // this TMA-ring form, whose finaliser is a separate wide kernel.
    if (impl == 0 && count >= tex_min_group(m) && tex_stream_applies(m, G, beta))
        return launch_biqgemm_tex(calls, count, x_rows, m, G, beta, ws, pdl, stream);
    // A group of one is a single call: the latency form where it applies
    // (same arithmetic, y bitwise equal; C2 6.1 -> 5.4 us)
    if (impl == 0 && count == 1 && !(debug_flags_stream() & 16384)) {
        QueryParams p{};
        p.keys = calls[0].keys;
        p.alpha = calls[0].alpha;
        p.x = calls[0].x;
        p.y = calls[0].y;
        p.x_rows = x_rows;
        p.m = m;
        p.G = G;
        p.NB = (G + 31) / 32;
        p.MT = (m + 31) / 32;
        p.beta = beta;
        p.b = 1;
        p.debug = debug_flags_stream();
        if (latency_applies(p)) {
            bool used = false;
            const cudaError_t e = launch_biqgemm_latency(p, pdl, stream, &used);
            if (e != cudaSuccess || used) return e;
        }
    }
    const int sms = device_sms(current_device());
    StreamArgs A{};
    static const int debug_flags = [] {
        const char* e = getenv("BQG_DEBUG_FLAGS");
        return e ? atoi(e) : 0;
    }();
    A.debug = debug_flags;
    A.x_rows = x_rows;
    A.m = m;
    A.NB = (G + 31) / 32;
    A.MT = (m + 31) / 32;
    // cpb CTAs per 32-group block, each a contiguous range of >= 1 row
    // tiles of that block; one CTA per SM when NB <= #SMs
    A.cpb = std::max(1, std::min(A.MT, sms / A.NB));
    A.grid = A.cpb * A.NB;
#ifndef BQG_STREAM_STAGE_KB
#define BQG_STREAM_STAGE_KB 16
#endif
    A.ups = std::max(1, BQG_STREAM_STAGE_KB / beta);  // ~16 KiB ring stages (TMA bulk copies)
    A.partial = ws + kTexCounterBytes / sizeof(float);  // the counters stay the texture form's
    for (int done = 0; done < count; done += kStreamMaxGroup) {
        A.ncalls = std::min(kStreamMaxGroup, count - done);
        for (int i = 0; i < A.ncalls; ++i) A.calls[i] = calls[done + i];
        cudaError_t e;
        switch (beta) {
            case 1: e = launch_stream_beta<1>(A, pdl || done > 0, stream); break;
            case 2: e = launch_stream_beta<2>(A, pdl || done > 0, stream); break;
            case 3: e = launch_stream_beta<3>(A, pdl || done > 0, stream); break;
            case 4: e = launch_stream_beta<4>(A, pdl || done > 0, stream); break;
            default: return cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace bqg
