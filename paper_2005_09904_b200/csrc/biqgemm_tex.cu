// biqgemm_tex.cu -- the grouped BiQGEMM form, keys through the TEXTURE pipe.
// b == 1, mu == 8, 1 <= beta <= 4; a GROUP of independent calls sharing
// (m, n, beta, mu), each a full biqgemm::biqgemm
// (/root/reference/proj/core/include/biqgemm/kernel.hpp:246-258 ->
// detail::run 116-204): its own x, its own LUT build (lut.hpp:50-69,
// 109-154), its own key stream and alpha epilogue (kernel.hpp:183-195).
//
// Why the texture pipe.  The LUT gather is one shared-memory wavefront per
// 32 lookups, and at b = 1 it alone needs ~70% of the HBM time of the key
// stream, so every other user of the SM's LSU data pipe eats directly into
// the roofline.  The TMA-ring form (biqgemm_stream.cu) lands keys in shared
// memory and reads them back with LDS.128 (+25% LSU wavefronts) and builds
// every call's tables in every CTA (+19%).  Measured on this B200
// (tools/ubench/lsu_tex.cu): a conflict-free LDS gather keeps 0.96-0.98
// wavefronts/clk/SM while other warps stream 21 B/clk/SM through
// tex1Dfetch (TLD) -- the two do not share a pipe; the same stream through
// LDG.128 costs the gather 10%.  So keys go HBM -> L2 -> TEX -> registers,
// prefetched UD units ahead, and never touch shared memory.
//
// Work split.  The group's units are ONE sequence u = (c*NB + gb)*MT + t
// (call c, 32-group block gb, 32-row tile t; unit = beta KiB of the tiled
// layout, kernels.h) and CTA i owns the contiguous range [i*T/grid,
// (i+1)*T/grid): every SM gets the same number of units (+-1), and a CTA
// walks whole (call, block) runs of MT units, so it builds one set of 32
// tables per MT units (C2: 2% of its shared-memory traffic instead of 19%).
// Per CTA:
//   NW gather warps : unit k of the CTA goes to warp k % NW.  Lane l = row
//                     l of the tile; step j reads table (l+j) mod 32 (one
//                     conflict-free wavefront per 32 lookups; address = ONE
//                     PRMT, query_core.cuh / biqgemm_stream.cu); per unit the
//                     beta plane sums are combined with alpha in fp64 and
//                     stored as ONE fp32 partial per (call, block, row).
//   NBW builder warps: the tables of (call, block) run q+1.. into LUT buffer
//                     q % NL while the gather warps are on run q (x read
//                     straight from global/L2; the DFS DP builder, bit-exact
//                     with the fp32 DP of lut.hpp:50-69).
//   stream_finalize (PDL-chained): y_c[r] = sum over blocks (fp64, blocks
//                     ascending) -> f32.
// The partial and finalize arithmetic is the TMA-ring form's, operation for
// operation, so y is bitwise identical to it and to the single-call forms,
// and bitwise independent of the grid, the group size and 32-row-aligned
// row sharding.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "lut_build.cuh"  // Log2

namespace bqg {

namespace {

constexpr int kMU = 8;
constexpr int kTable = 1 << kMU;
#ifndef BQG_TEX_NW
#define BQG_TEX_NW 28
#endif
#ifndef BQG_TEX_UD3
#define BQG_TEX_UD3 1
#endif
constexpr int kNWDefault = BQG_TEX_NW;   // gather warps (beta <= 3; fewer for beta = 4: registers)
#ifndef BQG_TEX_NBW
#define BQG_TEX_NBW 4
#endif
// L2 prefetch distance, in a warp's own unit strides (0 = off): when a warp
// fetches unit u into registers it also asks L2 for unit u + PF*NW of the
// same call (cp.async.bulk.prefetch, one lane), so the next fetches hit L2.
#ifndef BQG_TEX_PF
#define BQG_TEX_PF 0
#endif
constexpr int kNBW = BQG_TEX_NBW;   // builder warps (1, 2 or 4)
template <int NW>
struct TexGeom {
    static constexpr int threads = (NW + kNBW) * 32;
};
// LUT buffers: the two halves of one 64 KiB region.  Shared
// memory is kept small on purpose: texture fetches in flight occupy L1
// lines, and L1 is what the shared-memory carve-out leaves of 256 KiB.
constexpr int kNL = 2;
// Profiling switches, compile time (a variant build): 1 no LUT protocol,
// 2 no gather, 4 no key fetch.
#ifndef BQG_TEX_DBG
#define BQG_TEX_DBG 0
#endif
constexpr int kTexDbg = BQG_TEX_DBG;
// Builder warps poll for a free LUT buffer this often (a run lasts ~10 us at
// C2; a poll is ~4 issue slots taken from the gather warps' SM sub-partition)
constexpr unsigned kBuilderPollNs = 1000;
#ifndef BQG_TEX_BPOLL
#define BQG_TEX_BPOLL 1
#endif
#ifndef BQG_TEX_BFIRST
#define BQG_TEX_BFIRST 1
#endif
__device__ __forceinline__ void builder_wait(uint64_t* bar, uint32_t parity) {
    if (BQG_TEX_BPOLL)
        mbar_wait_poll(bar, parity, kBuilderPollNs);
    else
        mbar_wait_sleep(bar, parity);
}
constexpr uint32_t kLutBase = 0x10000u;
constexpr int kTexSmem = 0x20000;  // >= the end of the LUT region

struct TexCall {
    int toff;                // texel (16 B) offset of the call's tiled keys in its window's texture
    int win;                 // which of the launch's texture windows (0..kWin-1)
    const float* alpha;      // beta x m or nullptr
    const float* x;          // x_rows x 1
    float* y;                // m x 1
};

struct TexArgs {
    unsigned long long tex[4];  // texture objects over <= 4 address windows that hold every call's
                             // keys.  Each is read with a CONSTANT index (a switch on the call's
                             // window), so the handle is uniform: a handle picked with a per-warp
                             // index makes ptxas wrap each TLD in a waterfall loop that serialises
                             // the fetches (2.3 vs 6.4 TB/s, tools/ubench/tex_pattern.cu).
    unsigned long long wbase[4];  // byte address of each window's first texel (L2 prefetch addresses)
    int ncalls;
    long long x_rows;
    int m, NB, MT, grid;
    long long total;  // ncalls * NB * MT units
    float* partial;   // ncalls x NB x (MT*32), fp32
    unsigned* cnt;    // [kStreamMaxGroup] completion counters (zero between launches)
    // Fused all-gather (row-sharded calls): y rows are also stored at the
    // same offset from each peer's gather buffer -- NVLink stores into the
    // other GPUs' memory, issued by the finaliser as each call completes.
    // npeer = 0: the local y only.  local_base: this rank's gather buffer.
    int npeer;
    const float* local_base;
    float* peer_base[kMaxPeers];
    TexCall calls[kStreamMaxGroup];
};

// Per-CTA finalisation queue (shared memory).  y_c is summed in-kernel by
// the CTA whose completion count for call c is the last to arrive.
struct FinQueue {
    int posted;        // tasks posted so far (builder lane 0 writes, everyone reads)
    int call[kStreamMaxGroup];
    int next[kStreamMaxGroup];  // next 128-row chunk of task t to hand out
};
constexpr int kFinRows = 128;  // rows per chunk: 32 lanes x 4

// ---------------------------------------------------------------- LUT build
// The table of group gb*32 + lane lives in bank `lane`: entry k of buffer
// half h at byte  region + k*256 + h*128 + lane*4; e[k] for k < 128 is the
// fp32 DP (lut.hpp:50-69: e[0] = ((0 - x0) - x1) ... - x7, e[k] = e[k -
// 2^top(k)] + 2*x_top(k)), e[255 - k] = -e[k].  Walked depth-first at
// compile time: every entry is produced by exactly the reference's addition.
// Builder q of NBW = 2^h owns the first-half keys whose top h bits are q
// (the same decomposition as biqgemm_stream.cu, hence the same bits).
__device__ __forceinline__ void sts_pair(uint32_t col, int k, float v) {
    sts_f32(col + static_cast<uint32_t>(k) * 256u, v);
    sts_f32(col + static_cast<uint32_t>(kTable - 1 - k) * 256u, -v);
}

template <int K, int I, int Q, int LB>
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
__device__ __forceinline__ void build_tables_reg(int which, uint32_t col, const float (&x)[kMU]) {
    constexpr int LB = 7 - Log2<NBW>::value;
    float s[kMU];
    float e0 = 0.0f;
#pragma unroll
    for (int t = 0; t < kMU; ++t) e0 = __fsub_rn(e0, x[t]);
#pragma unroll
    for (int t = 0; t < kMU; ++t) s[t] = 2.0f * x[t];
    switch (which) {
        case 0: Dfs<0, 0, 0, LB>::node(e0, s, col); break;
        case 1: if constexpr (NBW > 1) Dfs<0, 0, 1, LB>::node(e0, s, col); break;
        case 2: if constexpr (NBW > 2) Dfs<0, 0, 2, LB>::node(e0, s, col); break;
        default: if constexpr (NBW > 3) Dfs<0, 0, 3, LB>::node(e0, s, col); break;
    }
}

// ---------------------------------------------------------------- gather
template <int IMM>
__device__ __forceinline__ float lds_lut(uint32_t rotw, uint32_t w, uint32_t sel) {
    uint32_t off;  // PTX prmt: the selector's sign-replicate nibble zeroes bytes 2-3
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(off) : "r"(rotw), "r"(w), "r"(sel));
    float e;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(e) : "r"(off), "n"(IMM));
    return e;
}
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

// One 1 KiB chunk: the same additions in the same order as stream_gather
// (biqgemm_stream.cu) -- 4 interleaved chains as two f32x2 pairs.
template <int IMM>
__device__ __forceinline__ float tex_gather(const uint4& lo, const uint4& hi, const uint32_t (&rot)[8]) {
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint64_t acc01 = 0, acc23 = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float e0 = lds_lut<IMM>(rot[q], w[q], 0x8840u);
        const float e1 = lds_lut<IMM>(rot[q], w[q], 0x8851u);
        const float e2 = lds_lut<IMM>(rot[q], w[q], 0x8862u);
        const float e3 = lds_lut<IMM>(rot[q], w[q], 0x8873u);
        if (q == 0) {
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

template <int BETA, int IMM>
__device__ __forceinline__ double tex_unit(const uint4 (&k)[BETA][2], const float (&a)[BETA],
                                           const uint32_t (&rot_in)[8]) {
#ifndef BQG_TEX_ROTREG
    // rot[q] byte b = 4*((lane + 4q + b) mod 32) = (rot[0] + 16q per byte) mod 128:
    // two ALU ops per unit and register instead of 8 live registers (at 64
    // registers per thread ptxas otherwise rematerialises all 8 from the lane
    // id, ~40 instructions per unit; measured C2 1.39 -> 1.26 us per call)
    uint32_t rot[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) rot[q] = (rot_in[0] + 0x10101010u * q) & 0x7C7C7C7Cu;
#else
    const uint32_t (&rot)[8] = rot_in;
#endif
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < BETA; ++i) {
        const float P = tex_gather<IMM>(k[i][0], k[i][1], rot);
        s += static_cast<double>(a[i]) * static_cast<double>(P);
    }
    return s;
}

// One prefetched unit: its keys, alpha, the index of its partial (~0u when
// the row is past m) and its run.  Computed at fetch time so that the
// gather loop keeps only one full cursor live (64 registers per thread:
// the 8 rotation registers must stay resident, not be rematerialised).
template <int BETA>
struct Slot {
    uint4 k[BETA][2];
    float a[BETA];
    uint32_t pidx;
    int q;
};

// Position of a unit in the sequence: run q (relative to the CTA's first
// (call, block) run), call c, block gb, tile t.  Advanced incrementally (no
// 64-bit divisions in the unit loop).
struct Cursor {
    int q, c, gb, t;
    int toff, win;           // the call's texel offset, window and alpha, reloaded only when c
    const float* al;         // changes (a dynamically indexed kernel parameter is a constant-cache load)
};
__device__ __forceinline__ void load_call(const TexArgs& A, Cursor& p) {
    if (p.c < A.ncalls) {
        p.toff = A.calls[p.c].toff;
        p.win = A.calls[p.c].win;
        p.al = A.calls[p.c].alpha;
    }
}
__device__ __forceinline__ void advance(const TexArgs& A, Cursor& p, int by) {
    p.t += by;
    const int c0 = p.c;
    while (p.t >= A.MT) {
        p.t -= A.MT;
        ++p.q;
        if (++p.gb == A.NB) {
            p.gb = 0;
            ++p.c;
        }
    }
    if (p.c != c0) load_call(A, p);
}

// Texel index of lane `lane`'s first 16 bytes of unit p (plane 0, low half).
template <int BETA>
__device__ __forceinline__ int unit_base(const TexArgs& A, const Cursor& p, int lane) {
    return p.toff + ((p.gb * A.MT + p.t) * BETA) * 64 + lane;
}

// Plane i of a unit: the lane's two 16-byte pieces (bytes l*16 and 512 + l*16
// of the plane's 1 KiB chunk).
__device__ __forceinline__ void fetch_plane(const TexArgs& A, int win, int base, int i, uint4 (&k)[2]) {
    auto fetch = [&](cudaTextureObject_t tex) {
        k[0] = tex1Dfetch<uint4>(tex, base + i * 64);
        k[1] = tex1Dfetch<uint4>(tex, base + i * 64 + 32);
    };
    switch (win) {  // warp-uniform branch, constant-index (uniform) handle in each arm
        case 0: fetch(A.tex[0]); break;
        case 1: fetch(A.tex[1]); break;
        case 2: fetch(A.tex[2]); break;
        default: fetch(A.tex[3]); break;
    }
}

// Everything of a unit but its keys: alpha, partial index, run; and the
// optional L2 prefetch of a unit further ahead.
template <int BETA, int NW>
__device__ __forceinline__ void unit_meta(const TexArgs& A, const Cursor& p, int lane, float (&a)[BETA],
                                          uint32_t& pidx, int& q) {
#if BQG_TEX_PF > 0
    const int uic = p.gb * A.MT + p.t;  // unit index inside the call
    if (lane == 0 && uic + BQG_TEX_PF * NW < A.NB * A.MT) {
        const unsigned long long addr =
            A.wbase[p.win] + 16ull * static_cast<unsigned long long>(p.toff + ((uic + BQG_TEX_PF * NW) * BETA) * 64);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(addr), "r"(BETA * 1024) : "memory");
    }
#endif
    const int r = p.t * 32 + lane;
#pragma unroll
    for (int i = 0; i < BETA; ++i)
        a[i] = r < A.m ? (p.al ? __ldg(p.al + static_cast<long long>(i) * A.m + r) : 1.0f) : 0.0f;
    pidx = r < A.m ? static_cast<uint32_t>((p.c * A.NB + p.gb) * A.MT) * 32u + static_cast<uint32_t>(r) : ~0u;
    q = p.q;
}

template <int BETA, int NW>
__device__ __forceinline__ void fetch_unit(const TexArgs& A, const Cursor& p, int lane, Slot<BETA>& sl) {
    const int base = unit_base<BETA>(A, p, lane);
#pragma unroll
    for (int i = 0; i < BETA; ++i) fetch_plane(A, p.win, base, i, sl.k[i]);
    unit_meta<BETA, NW>(A, p, lane, sl.a, sl.pidx, sl.q);
}

__device__ __forceinline__ int ld_volatile_s32(const int* p) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

// y_c[r] for the 128 rows of chunk ch: f32( sum_gb partial[c][gb][r] ),
// fp64, blocks ascending (the TMA-ring form's finaliser, operation for
// operation).  Lane l owns rows ch*128 + 4l .. +3 (one 16-byte load per
// block, 8 blocks in flight; run by the builder warps between builds and
// by every warp once its gather work is done).  .cg loads: the partials were written by
// other SMs (L1 is not coherent).
__device__ __forceinline__ void fin_chunk(const TexArgs& A, int c, int ch, int lane) {
    const long long r0 = static_cast<long long>(ch) * kFinRows + lane * 4;
    if (r0 >= A.m) return;
    const long long MTP = static_cast<long long>(A.MT) * 32;
    const float4* p = reinterpret_cast<const float4*>(A.partial + static_cast<long long>(c) * A.NB * MTP + r0);
    const long long st = MTP / 4;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int gb = 0;
    for (; gb + 8 <= A.NB; gb += 8) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcg(p + (gb + k) * st);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            s0 += static_cast<double>(v[k].x);
            s1 += static_cast<double>(v[k].y);
            s2 += static_cast<double>(v[k].z);
            s3 += static_cast<double>(v[k].w);
        }
    }
    for (; gb < A.NB; ++gb) {
        const float4 v = __ldcg(p + gb * st);
        s0 += static_cast<double>(v.x);
        s1 += static_cast<double>(v.y);
        s2 += static_cast<double>(v.z);
        s3 += static_cast<double>(v.w);
    }
    float* y = A.calls[c].y + r0;
    const long long left = A.m - r0;
    auto put = [&](float* d) {
        d[0] = static_cast<float>(s0);
        if (left > 1) d[1] = static_cast<float>(s1);
        if (left > 2) d[2] = static_cast<float>(s2);
        if (left > 3) d[3] = static_cast<float>(s3);
    };
    put(y);
    if (A.npeer > 0) {  // the same rows into every peer's gather buffer (fire-and-forget stores)
        const long long off = y - A.local_base;
        for (int k = 0; k < A.npeer; ++k) put(A.peer_base[k] + off);
    }
}

// One finalisation chunk if any is available: returns false when the queue
// holds no work for this warp right now.  tcur = the warp's task cursor.
__device__ __forceinline__ bool fin_one(const TexArgs& A, FinQueue* fq, int& tcur, int lane) {
    const int nch = (A.m + kFinRows - 1) / kFinRows;
    while (tcur < ld_volatile_s32(&fq->posted)) {
        int ch = 0;
        if (lane == 0) ch = atomicAdd(&fq->next[tcur], 1);
        ch = __shfl_sync(0xffffffffu, ch, 0);
        if (ch < nch) {
            fin_chunk(A, fq->call[tcur], ch, lane);
            return true;
        }
        ++tcur;
    }
    return false;
}

// Finish every chunk posted so far.
__device__ __forceinline__ void fin_drain(const TexArgs& A, FinQueue* fq, int& tcur, int lane) {
    while (fin_one(A, fq, tcur, lane)) {
    }
}

template <int BETA, int UD, int kNW>
__global__ void __launch_bounds__(TexGeom<kNW>::threads, 1) biqgemm_tex_kernel(const __grid_constant__ TexArgs A) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pdl_launch_dependents();

    const long long U0 = static_cast<long long>(blockIdx.x) * A.total / A.grid;
    const long long U1 = static_cast<long long>(blockIdx.x + 1) * A.total / A.grid;
    if (U0 >= U1) return;
    const long long cb0 = U0 / A.MT;
    const int nruns = static_cast<int>((U1 - 1) / A.MT - cb0 + 1);  // (call, block) runs touched

    const uint32_t sbase = smem_u32(smem);
    const uint32_t lut_abs = (sbase & 0xFF000000u) | kLutBase;
    if (sbase + 1024u > lut_abs || lut_abs + 0x10000u > sbase + kTexSmem) __trap();
    uint64_t* lfull = reinterpret_cast<uint64_t*>(smem);  // [kNL] LUT(q) built       (kNBW*32 lanes)
    uint64_t* ldone = lfull + kNL;                        // [kNL] run q gathered      (kNW*32 lanes)
    FinQueue* fq = reinterpret_cast<FinQueue*>(smem + 64);
    if (threadIdx.x == 0) {
        for (int b = 0; b < kNL; ++b) {
            mbar_init(&lfull[b], kNBW * 32);
            mbar_init(&ldone[b], kNW * 32);
        }
        fq->posted = 0;
        fence_mbar_init();
    }
    __syncthreads();
    const long long W = static_cast<long long>(A.NB) * A.MT;  // units per call
    int tcur = 0;  // this warp's finalisation-task cursor

    if (warp >= kNW) {
        // ------------------------------------------------ builders
        const int which = warp - kNW;
        if (kTexDbg & 1) return;
        // Run q's gather is complete (its ldone phase): if it is the CTA's
        // last run of call c, add the CTA's unit count of c to c's counter;
        // the CTA that completes the count owns y_c's finalisation.
        // Memory order: gather warps' partial stores -> mbarrier arrive
        // (release.cta) -> this thread's wait (acquire.cta) -> fence.acq_rel.gpu
        // -> counter atomic; the finaliser: atomic -> fence.acq_rel.gpu -> .cg loads.
        auto signal_run = [&](int q) {
            const long long cb = cb0 + q;
            const int c = static_cast<int>(cb / A.NB);
            const bool last = q == nruns - 1 || (cb + 1) / A.NB != c;
            if (!last || which != 0 || lane != 0) return;
            const long long lo = max(U0, static_cast<long long>(c) * W), hi = min(U1, static_cast<long long>(c + 1) * W);
            const unsigned mine = static_cast<unsigned>(hi - lo);
            fence_acq_rel_gpu();
            const unsigned old = atomicAdd(A.cnt + c, mine);
            if (old + mine == static_cast<unsigned>(W)) {
                fence_acq_rel_gpu();
                A.cnt[c] = 0;  // every CTA has added: reset for the next launch
                const int t = fq->posted;
                fq->call[t] = c;
                fq->next[t] = 0;
                __threadfence_block();
                *reinterpret_cast<volatile int*>(&fq->posted) = t + 1;
            }
        };
        pdl_wait();  // x may be the predecessor's output; the counters its finaliser's
        for (int q = 0; q < nruns; ++q) {
            const long long cb = cb0 + q;
            const int c = static_cast<int>(cb / A.NB), gb = static_cast<int>(cb - static_cast<long long>(c) * A.NB);
            const float* x = A.calls[c].x;
            float xv[kMU];
            const long long r0 = (static_cast<long long>(gb) * 32 + lane) * kMU;
            if (r0 + kMU <= A.x_rows && (reinterpret_cast<uintptr_t>(x + r0) & 15) == 0) {
                const float4 v0 = __ldg(reinterpret_cast<const float4*>(x + r0));
                const float4 v1 = __ldg(reinterpret_cast<const float4*>(x + r0) + 1);
                xv[0] = v0.x; xv[1] = v0.y; xv[2] = v0.z; xv[3] = v0.w;
                xv[4] = v1.x; xv[5] = v1.y; xv[6] = v1.z; xv[7] = v1.w;
            } else {
#pragma unroll
                for (int t = 0; t < kMU; ++t) xv[t] = r0 + t < A.x_rows ? __ldg(x + r0 + t) : 0.0f;
            }
            const int buf = q % kNL;
            // LUT buffer `buf` is free once run q - kNL is gathered; the gather
            // warps are then on run q - 1, which lasts far longer than a poll
            if (q >= kNL) {
                // one builder warp polls; the others sleep on a named barrier
                // (a blocked warp issues nothing: 4x fewer polling slots)
                if (which == 0) builder_wait(&ldone[buf], static_cast<uint32_t>((q / kNL - 1) & 1));
                named_bar_sync(2, kNBW * 32);
            }
#if !BQG_TEX_BFIRST
            if (q >= kNL) {
                signal_run(q - kNL);
                named_bar_sync(1, kNBW * 32);
                fin_drain(A, fq, tcur, lane);
            }
#endif
            build_tables_reg<kNBW>(which,
                                   lut_abs + static_cast<uint32_t>(buf >> 1) * 0x10000u +
                                       static_cast<uint32_t>(buf & 1) * 128u + static_cast<uint32_t>(lane) * 4u,
                                   xv);
            mbar_arrive(&lfull[buf]);
            // only then signal run q - kNL and finalise what became ready: a
            // finalisation (up to a whole call) must never delay a LUT
            if (BQG_TEX_BFIRST && q >= kNL) {
                signal_run(q - kNL);
                named_bar_sync(1, kNBW * 32);  // every builder sees a task posted just now
                fin_drain(A, fq, tcur, lane);  // builders finalise while the gather warps run on
            }
        }
        for (int q = max(0, nruns - kNL); q < nruns; ++q) {
            if (which == 0) builder_wait(&ldone[q % kNL], static_cast<uint32_t>((q / kNL) & 1));
            signal_run(q);
        }
        named_bar_sync(1, kNBW * 32);
        // release: the queue is final (the gather warps sleep on barrier 3)
        if (which == 0) named_bar_arrive(3, (kNW + 1) * 32);
        fin_drain(A, fq, tcur, lane);
        if (A.npeer > 0) __threadfence_system();  // peer stores (other GPUs' memory) performed before the CTA retires
        return;
    }

    // ---------------------------------------------------- gather warps
    uint32_t rot[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        rot[q] = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) rot[q] |= (static_cast<uint32_t>((lane + 4 * q + b) & 31) * 4u) << (8 * b);
    }
    uint64_t pol_keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    // this warp's units: u_k = U0 + warp + k*kNW, k < nk; the next UD are in
    // registers (slot k % UD), fetched UD units ahead of their gather
    const int nk = U1 - U0 > warp ? static_cast<int>((U1 - U0 - warp + kNW - 1) / kNW) : 0;
    Cursor pf{0, 0, 0, 0, 0, 0, nullptr};
    if (nk > 0) {
        const long long u = U0 + warp, cb = u / A.MT;
        pf.q = static_cast<int>(cb - cb0);
        pf.t = static_cast<int>(u - cb * A.MT);
        pf.c = static_cast<int>(cb / A.NB);
        pf.gb = static_cast<int>(cb - static_cast<long long>(pf.c) * A.NB);
        load_call(A, pf);
    }
    // Every warp walks EVERY run of the CTA in order -- wait LUT(q) built,
    // gather its units of run q (maybe none), release run q -- so a release
    // of run q + kNL always follows the build of run q + kNL, which follows
    // the completion of run q's release phase: no mbarrier over-arrival or
    // parity aliasing however few units a run has.
    int cur = -1;  // run whose LUT this warp waited for and has not released
    auto move_to = [&](int q) {
        while (cur < q) {
            if (cur >= 0) mbar_arrive(&ldone[cur % kNL]);
            ++cur;
            mbar_wait(&lfull[cur % kNL], static_cast<uint32_t>((cur / kNL) & 1));
        }
    };
    auto store_partial = [&](uint32_t pidx, double s) {
        if (pidx != ~0u) {
            // partials stay in L2 for the finaliser (L2 evict_last)
            asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(A.partial + pidx),
                         "f"(static_cast<float>(s)), "l"(pol_keep)
                         : "memory");
        }
    };
    Slot<BETA> S[UD];
#pragma unroll
    for (int d = 0; d < UD; ++d) {
        if (d < nk) fetch_unit<BETA, kNW>(A, pf, lane, S[d]);
        advance(A, pf, kNW);
    }
    pdl_wait();  // the previous launch may still read the partials / counters
    for (int k0 = 0; k0 < nk; k0 += UD) {
#pragma unroll
        for (int d = 0; d < UD; ++d) {
            if (k0 + d < nk) {
                if (!(kTexDbg & 1)) move_to(S[d].q);
                double s;
                if (kTexDbg & 2) {
                    uint32_t h = 0;
#pragma unroll
                    for (int i = 0; i < BETA; ++i) h ^= S[d].k[i][0].x ^ S[d].k[i][0].y ^ S[d].k[i][1].z ^ S[d].k[i][1].w;
                    s = h;
                } else if (S[d].q % kNL == 0) {  // LUT buffer = the LDS immediate (region base + half)
                    s = tex_unit<BETA, kLutBase>(S[d].k, S[d].a, rot);
                } else {
                    s = tex_unit<BETA, kLutBase + 128>(S[d].k, S[d].a, rot);
                }
                const uint32_t pidx = S[d].pidx;
                if (k0 + d + UD < nk && !(kTexDbg & 4)) fetch_unit<BETA, kNW>(A, pf, lane, S[d]);
                advance(A, pf, kNW);
                store_partial(pidx, s);
            }
        }
    }
    if (kTexDbg & 1) return;
    move_to(nruns - 1);
    mbar_arrive(&ldone[cur % kNL]);
    named_bar_sync(3, (kNW + 1) * 32);  // the CTA's last tasks are posted: everyone helps finish them
    fin_drain(A, fq, tcur, lane);
    if (A.npeer > 0) __threadfence_system();  // peer stores (other GPUs' memory) performed before the CTA retires
}

// Per-device caches (cudaFuncSetAttribute and the SM count are per device).
constexpr int kMaxDev = kMaxDevices;

template <int BETA, int UD, int NW>
cudaError_t launch_tex_beta(const TexArgs& A, int dev, bool pdl, cudaStream_t stream) {
    static PerDeviceOnce configured;
    const cudaError_t ea = once_per_device(configured, dev, [] {
        return cudaFuncSetAttribute(biqgemm_tex_kernel<BETA, UD, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kTexSmem);
    });
    if (ea != cudaSuccess) return ea;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(A.grid));
    cfg.blockDim = dim3(TexGeom<NW>::threads);
    cfg.dynamicSmemBytes = kTexSmem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, biqgemm_tex_kernel<BETA, UD, NW>, A);
    if (e != cudaSuccess) return e;
    return cudaSuccess;
}

// Texture objects over address windows, created on first use and cached by
// (device, base, bytes).  A linear texture object only describes memory
// (address, texel format, size) and owns nothing, and the driver accepts a
// window that spans several allocations (tools/ubench/tex_span.cu); the
// kernel only fetches inside the calls' key buffers.  Windows are rounded
// out to 2 MiB so that recurring groups hit the cache.
struct TexKey {
    int dev;
    uintptr_t base;
    size_t bytes;
    bool operator==(const TexKey& o) const { return dev == o.dev && base == o.base && bytes == o.bytes; }
};
struct TexKeyHash {
    size_t operator()(const TexKey& k) const { return std::hash<uintptr_t>()(k.base) ^ (k.bytes * 0x9E3779B97F4A7C15ull) ^ k.dev; }
};
std::mutex g_tex_mu;
std::unordered_map<TexKey, cudaTextureObject_t, TexKeyHash> g_tex;
constexpr size_t kTexCacheMax = 4096;
constexpr uintptr_t kWinAlign = 2u << 20;

cudaError_t window_texture(int dev, uintptr_t base, size_t bytes, cudaTextureObject_t* out) {
    std::lock_guard<std::mutex> lk(g_tex_mu);
    const TexKey key{dev, base, bytes};
    auto it = g_tex.find(key);
    if (it != g_tex.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    if (g_tex.size() >= kTexCacheMax) {  // bounded: drop everything (rare; objects are cheap to remake)
        for (auto& kv : g_tex) cudaDestroyTextureObject(kv.second);
        g_tex.clear();
    }
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = reinterpret_cast<void*>(base);
    rd.res.linear.desc = cudaCreateChannelDesc(32, 32, 32, 32, cudaChannelFormatKindUnsigned);
    rd.res.linear.sizeInBytes = bytes;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t = 0;
    // object creation is not a stream operation: allowed while a stream of
    // this thread is being captured into a CUDA graph (relaxed mode)
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    cudaError_t e = cudaCreateTextureObject(&t, &rd, &td, nullptr);
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (e != cudaSuccess) return e;
    g_tex.emplace(key, t);
    *out = t;
    return cudaSuccess;
}

long long g_max_texels[kMaxDev];
std::once_flag g_texels_once[kMaxDev];

long long max_texels(int dev) {
    std::call_once(g_texels_once[dev], [&] {
        int w = 0;
        if (cudaDeviceGetAttribute(&w, cudaDevAttrMaxTexture1DLinearWidth, dev) != cudaSuccess || w <= 0) w = 1 << 27;
        g_max_texels[dev] = std::min<long long>(w, 1ll << 30);
    });
    return g_max_texels[dev];
}

}  // namespace

bool tex_stream_applies(long long m, int G, int beta) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return false;
    const long long bytes = ((G + 31) / 32) * ((m + 31) / 32) * static_cast<long long>(beta) * 1024;
    return bytes / 16 + 2 * (kWinAlign / 16) <= max_texels(dev);
}

cudaError_t zero_counters_once(void* ws, int dev, cudaStream_t stream) {
    // The counters must be zero before a workspace's first launch (the C ABI
    // documents it; the library's own allocators zero-fill).  As a safety net
    // a workspace not seen before is zeroed on the stream -- inside a graph
    // capture the memset becomes a graph node.
    static std::mutex mu;
    static std::unordered_map<uintptr_t, int> seen;
    const uintptr_t key = reinterpret_cast<uintptr_t>(ws) ^ (static_cast<uintptr_t>(dev) << 56);
    std::lock_guard<std::mutex> lk(mu);
    if (seen.count(key)) return cudaSuccess;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cs);
    const cudaError_t e = cudaMemsetAsync(ws, 0, kTexCounterBytes, stream);
    if (e != cudaSuccess) return e;
    if (cs == cudaStreamCaptureStatusNone) seen.emplace(key, 1);
    return cudaSuccess;
}

cudaError_t launch_biqgemm_tex(const StreamCall* calls, int count, long long x_rows, int m, int G, int beta,
                               float* ws, bool pdl, cudaStream_t stream, const float* local_base,
                               float* const* peer_base, int npeer) {
    if (npeer < 0 || npeer > kMaxPeers) return cudaErrorInvalidValue;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    std::vector<TexArgs> buf(1);  // ~12 KiB: keep it off the caller's stack
    TexArgs& A = buf[0];
    A.x_rows = x_rows;
    A.npeer = npeer;
    A.local_base = local_base;
    for (int k = 0; k < kMaxPeers; ++k) A.peer_base[k] = k < npeer ? peer_base[k] : nullptr;
    A.m = m;
    A.NB = (G + 31) / 32;
    A.MT = (m + 31) / 32;
    A.cnt = reinterpret_cast<unsigned*>(ws);  // kTexCounterBytes, then the partials
    e = zero_counters_once(ws, dev, stream);
    if (e != cudaSuccess) return e;
    A.partial = ws + kTexCounterBytes / sizeof(float);
    static const bool verbose = getenv("BQG_TEX_VERBOSE") != nullptr;
    const size_t key_bytes = static_cast<size_t>(A.NB) * A.MT * beta * 1024;
    const long long texels = max_texels(dev);
    // Address windows: greedy over the calls' key buffers sorted by address,
    // each window (rounded out to 2 MiB) at most `texels` texels.
    std::vector<std::pair<uintptr_t, int>> order(count);
    for (int i = 0; i < count; ++i) {
        const uintptr_t p = reinterpret_cast<uintptr_t>(calls[i].keys);
        if (p & 15) return cudaErrorMisalignedAddress;  // the C ABI checks 16-byte alignment first
        order[i] = {p, i};
    }
    std::sort(order.begin(), order.end());
    std::vector<int> win_of(count);
    std::vector<std::pair<uintptr_t, uintptr_t>> wins;  // [base, top)
    static const bool exact_win = getenv("BQG_TEX_EXACTWIN") != nullptr;  // diagnostics
    for (const auto& pr : order) {
        const uintptr_t lo = exact_win ? pr.first : pr.first & ~(kWinAlign - 1);
        const uintptr_t hi = exact_win ? pr.first + key_bytes : (pr.first + key_bytes + kWinAlign - 1) & ~(kWinAlign - 1);
        if (!exact_win && !wins.empty() &&
            static_cast<long long>((std::max(hi, wins.back().second) - wins.back().first) / 16) <= texels) {
            wins.back().second = std::max(hi, wins.back().second);
        } else {
            wins.push_back({lo, hi});
        }
        win_of[pr.second] = static_cast<int>(wins.size()) - 1;
    }
    int done = 0;
    while (done < count) {
        // the longest run of calls (<= kStreamMaxGroup) that needs <= 4 windows
        int slot_of_win[4] = {-1, -1, -1, -1}, nw = 0, n = 0;
        while (done + n < count && n < kStreamMaxGroup) {
            const int w = win_of[done + n];
            int slot = -1;
            for (int k = 0; k < nw; ++k)
                if (slot_of_win[k] == w) slot = k;
            if (slot < 0) {
                if (nw == 4) break;
                slot = nw;
                slot_of_win[nw++] = w;
            }
            const StreamCall& sc = calls[done + n];
            A.calls[n] = {static_cast<int>((reinterpret_cast<uintptr_t>(sc.keys) - wins[w].first) / 16), slot, sc.alpha,
                          sc.x, sc.y};
            ++n;
        }
        for (int k = 0; k < 4; ++k) {
            cudaTextureObject_t t = 0;
            if (k < nw) {
                e = window_texture(dev, wins[slot_of_win[k]].first, wins[slot_of_win[k]].second - wins[slot_of_win[k]].first, &t);
                if (e != cudaSuccess) return e;
            }
            A.tex[k] = static_cast<unsigned long long>(t);
            A.wbase[k] = k < nw ? static_cast<unsigned long long>(wins[slot_of_win[k]].first) : 0ull;
        }
        A.ncalls = n;
        if (verbose) fprintf(stderr, "[bqg tex] launch of %d calls, %d windows\n", n, nw);
        A.total = static_cast<long long>(A.ncalls) * A.NB * A.MT;
        A.grid = static_cast<int>(std::min<long long>(device_sms(dev), A.total));
        const bool p = pdl || done > 0;
        switch (beta) {
            case 1: e = launch_tex_beta<1, 3, kNWDefault>(A, dev, p, stream); break;
            case 2: e = launch_tex_beta<2, 1, kNWDefault>(A, dev, p, stream); break;
            case 3: e = launch_tex_beta<3, BQG_TEX_UD3, kNWDefault>(A, dev, p, stream); break;
            case 4: e = launch_tex_beta<4, 1, 24>(A, dev, p, stream); break;
            default: return cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return e;
        done += n;
    }
    return cudaSuccess;
}

}  // namespace bqg
