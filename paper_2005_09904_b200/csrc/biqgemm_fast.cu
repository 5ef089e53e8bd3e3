// biqgemm_fast.cu -- the BiQGEMM hot path for mu <= 8 (fp32 LUT), sm_100a.
//
// Replaces biqgemm::detail::run + query_rows + the alpha epilogue
// (/root/reference/proj/core/include/biqgemm/kernel.hpp:83-108,116-204) and
// build_lut_block (lut.hpp:109-154) with two kernels launched back to back
// with programmatic dependent launch (PDL):
//
// 1. biqgemm_fast_kernel -- per CTA: one 32-group block x BT input columns x
//    a contiguous range of 1 KiB key chunks (chunk = plane i x 32-row tile).
//      producer warp : streams the CTA's key chunks global -> shared with the
//                      TMA bulk-copy engine (cp.async.bulk, L2 evict-first)
//                      through an R-stage mbarrier ring.  Keys never depend
//                      on the previous kernel, so the ring fills before
//                      griddepcontrol.wait and overlaps the predecessor.
//      consumer warps: after griddepcontrol.wait, build the block's tables in
//                      bank-owned shared memory with the DP recurrence
//                      (lut_build.cuh; table of group g lives in bank g);
//                      then per 32-row TILE (its beta 1 KiB chunks, one
//                      warp) lane l owns row l and at step j gathers
//                      T_g[key(l, g)] for the rotated group g = (l + j) mod 32
//                      -- every lane hits a different bank, so each warp
//                      gather is one conflict-free wavefront -- and
//                      accumulates in registers.  No cross-lane reduction (no
//                      SHFL, which shares the shared-memory pipe).  The beta
//                      plane sums of a tile are combined with alpha in fp64
//                      and ONE fp32 partial per (block, row, column) goes to
//                      the workspace (beta x less partial traffic than one per
//                      plane: the round trip through HBM/L2 was ~25% of a
//                      large-b call).
// 2. finalize_kernel -- y(r,c) = f32(sum_gb partial[gb][r][c]), fp64, blocks
//    ascending: per block sum_i alpha_i * P_i in fp64 first (kernel.hpp:
//    183-195 applies alpha after the full group sum; the per-block combine is
//    the b = 1 forms' arithmetic, within the fp32 contract).
//
// Every output's reduction tree is a function of (n, mu) only, so y is
// bitwise identical for every grid shape, CTA split and row sharding.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "lut_build.cuh"
#include "query_core.cuh"

namespace bqg {

// Per-CTA timeline for profiling (BQG_DEBUG_FLAGS & 2): globaltimer ns at
// start (0), after griddepcontrol.wait (1), first segment's LUT built (2),
// first key stage landed (3), query done (4); smid (5); the last segment's
// start after the drain barrier (6) and its LUT built (7), 0 for one segment.
// Off in production (one predicated branch per CTA).
__device__ unsigned long long g_timeline[8192][8];

namespace {

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned s;
    asm volatile("mov.u32 %0, %smid;" : "=r"(s));
    return s;
}

struct FastPlan {
    int cpp;    // 32-row tiles (beta KiB of keys each) per (group block, column tile) pair
    int CT;     // column tiles
    int mode;   // 0 = aligned (cpb CTAs per pair), 1 = flat contiguous split
    int cpb;    // aligned: CTAs per pair
    int grid;
    int q, r;   // balanced split: CTA c gets q + (c < r) tiles of its domain
    int tps;    // tiles per ring stage (<= NW: warp w takes tile w of a stage)
    int R;      // ring stages (<= kMaxStages)
};
constexpr int kMaxStages = 8;

// Byte offset of key byte `bi` of word w in the bank-owned LUT, OR'd with the
// lane's offset.  word(k, l, c) = (k*32 + l)*BT + c  ->  byte = k << SH | l*4*BT.
template <int MU, int BT>
__device__ __forceinline__ uint32_t lut_off(uint32_t w, int bi, uint32_t lane_off) {
    constexpr int SH = (BT == 1) ? 7 : (BT == 2 ? 8 : 9);
    constexpr uint32_t MASK = ((1u << MU) - 1u) << SH;
    const int s = 8 * bi - SH;  // compile-time after unrolling
    const uint32_t v = s >= 0 ? (w >> s) : (w << (-s));
    return (v & MASK) | lane_off;
}

template <int MU, int BT, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, BT == 1 ? 2 : 1)
    biqgemm_fast_kernel(const QueryParams p, const FastPlan plan) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int LUT_BYTES = (1 << MU) * LutGeom<BT>::KROW * 4;
    const int beta = p.beta;
    const int R = plan.R;
    const int TPS = plan.tps;                              // tiles per stage
    const uint32_t TILE_BYTES = static_cast<uint32_t>(beta) * 1024u;
    const uint32_t STAGE_BYTES = static_cast<uint32_t>(TPS) * TILE_BYTES;
    float* lut = reinterpret_cast<float*>(smem);
    unsigned char* stages = smem + LUT_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + static_cast<size_t>(R) * STAGE_BYTES);
    uint64_t* empty = full + kMaxStages;
    float* xs = reinterpret_cast<float*>(empty + kMaxStages);  // staged x tile (xs_words)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool tl = (p.debug & 2) && threadIdx.x == 0 && blockIdx.x < 8192;
    if (tl) {
        g_timeline[blockIdx.x][0] = gtimer();
        g_timeline[blockIdx.x][5] = smid();
        g_timeline[blockIdx.x][6] = g_timeline[blockIdx.x][7] = 0;
    }
    pdl_launch_dependents();

    // This CTA's tile range [cbeg, cend) over the (pair, tile) sequence.
    const int c = plan.mode == 0 ? static_cast<int>(blockIdx.x) % plan.cpb : static_cast<int>(blockIdx.x);
    const int dom = plan.mode == 0 ? static_cast<int>(blockIdx.x) / plan.cpb : 0;
    const int cbeg = dom * plan.cpp + c * plan.q + min(c, plan.r);
    const int cend = cbeg + plan.q + (c < plan.r ? 1 : 0);

    if (threadIdx.x == 0) {
        for (int st = 0; st < R; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const long long rows_pad = static_cast<long long>(p.MT) * 32;

    if (warp == NW) {
        // ------------------------------------------------ producer (1 lane)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int sc = 0;  // stage counter across segments
            for (int seg = cbeg; seg < cend;) {
                const int pair = seg / plan.cpp;
                const int pbase = pair * plan.cpp;
                const int seg_end = min(cend, pbase + plan.cpp);
                const int gb = pair / plan.CT;
                const unsigned char* kpair = p.keys + static_cast<long long>(gb) * plan.cpp * TILE_BYTES;
                for (int t0 = seg - pbase; t0 < seg_end - pbase; t0 += TPS, ++sc) {
                    const int cnt = min(TPS, seg_end - pbase - t0);
                    const int slot = sc % R;
                    mbar_wait(&empty[slot], ((sc / R) & 1) ^ 1);
                    // Stage 0 lands ALONE before the rest of the fill is
                    // requested: every CTA asking for its whole ring at once
                    // (up to 20 MB in flight) delayed the first stage to
                    // ~3 us (C4 b = 2: 13.6 -> 12.9 us per call; BQG_DEBUG_FLAGS
                    // bit 21 restores the old order for A/B)
                    if (sc == 1 && !(p.debug & (1 << 21))) mbar_wait(&full[0], 0);
                    mbar_arrive_expect_tx(&full[slot], cnt * TILE_BYTES);
                    bulk_g2s(stages + static_cast<size_t>(slot) * STAGE_BYTES, kpair + static_cast<long long>(t0) * TILE_BYTES,
                             cnt * TILE_BYTES, &full[slot], pol);
                }
                seg = seg_end;
            }
        }
        return;
    }

    // ---------------------------------------------------- consumers
    uint32_t goff[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) goff[j] = static_cast<uint32_t>((lane + j) & 31) * 4u * BT;
    const uint32_t lut_s = smem_u32(lut);
    pdl_wait();  // x (and the workspace) of the predecessor are visible from here on
    if (tl) g_timeline[blockIdx.x][1] = gtimer();
    int sc = 0;
    // The x tile of a segment's (block, column tile) is loaded into registers
    // one segment ahead (its global latency overlaps the previous segment's
    // gather) and stored to shared memory at the segment boundary -- the
    // values stage_x_tile would read.
    constexpr int XT = 32 * MU * BT, XPT = (XT + NW * 32 - 1) / (NW * 32);
    float xr[XPT];
    auto load_x = [&](int pair) {
        const long long gbx = pair / plan.CT, col0 = static_cast<long long>(pair - gbx * plan.CT) * BT;
        const long long r0 = gbx * 32 * MU;
#pragma unroll
        for (int k = 0; k < XPT; ++k) {
            const int idx = threadIdx.x + k * NW * 32;
            const int rl = idx / BT, cc = idx - (idx / BT) * BT;
            const long long r = r0 + rl, col = col0 + cc;
            xr[k] = (idx < XT && r < p.x_rows && col < p.b) ? __ldcg(p.x + r * p.b + col) : 0.0f;
        }
    };
    if (cbeg < cend) load_x(cbeg / plan.cpp);
    for (int seg = cbeg; seg < cend;) {
        const int pair = seg / plan.cpp;
        const int pbase = pair * plan.cpp;
        const int seg_end = min(cend, pbase + plan.cpp);
        const int gb = pair / plan.CT, ct = pair - gb * plan.CT;
        if (seg != cbeg) named_bar_sync(1, NW * 32);  // previous segment done with the LUT and x tile
        if (tl && seg != cbeg) g_timeline[blockIdx.x][6] = gtimer();
#pragma unroll
        for (int k = 0; k < XPT; ++k) {
            const int idx = threadIdx.x + k * NW * 32;
            if (idx < XT) xs[xs_slot<MU, BT>(idx)] = xr[k];
        }
        named_bar_sync(1, NW * 32);
        if (seg_end < cend) load_x(seg_end / plan.cpp);  // the next segment's x, in flight during this one
        build_bank_owned_tables_smem<MU, NW, BT, LutGeom<BT>::KROW>(lut, xs, warp, lane);
        named_bar_sync(1, NW * 32);
        if (tl) g_timeline[blockIdx.x][seg == cbeg ? 2 : 7] = gtimer();

        const int lo = seg - pbase, hi = seg_end - pbase;
        for (int t0 = lo; t0 < hi; t0 += TPS, ++sc) {
            const int slot = sc % R;
            const int t = t0 + warp;  // this warp's tile of the stage
            const bool mine = warp < TPS && t < hi;
            // alpha of the warp's rows, requested before the keys are waited for
            const long long row = static_cast<long long>(t) * 32 + lane;
            const bool live = mine && row < p.m;
            mbar_wait(&full[slot], (sc / R) & 1);
            if (tl && sc == 0) g_timeline[blockIdx.x][3] = gtimer();
            if (mine) {
                const unsigned char* kt = stages + static_cast<size_t>(slot) * STAGE_BYTES +
                                          static_cast<size_t>(warp) * TILE_BYTES;
                double acc[BT];
#pragma unroll
                for (int cc = 0; cc < BT; ++cc) acc[cc] = 0.0;
#pragma unroll 1
                for (int i = 0; i < beta; ++i) {
                    const float a = live ? (p.alpha ? __ldg(p.alpha + static_cast<long long>(i) * p.m + row) : 1.0f)
                                         : 0.0f;
                    const unsigned char* kc = kt + i * 1024;
                    const uint4 ka = *reinterpret_cast<const uint4*>(kc + lane * 16);
                    const uint4 kb = *reinterpret_cast<const uint4*>(kc + 512 + lane * 16);
                    const uint32_t w[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
                    float o[BT];
                    gather_chunk<MU, BT>(w, lut_s, goff, o);
#pragma unroll
                    for (int cc = 0; cc < BT; ++cc) acc[cc] += static_cast<double>(a) * static_cast<double>(o[cc]);
                }
                // partial[gb][ct][row][BT]: the warp's 32 rows x BT columns are
                // one contiguous 128*BT-byte run (one vector store per lane;
                // padding columns past b are written and never read)
                float* dst = p.partial + ((static_cast<long long>(gb) * plan.CT + ct) * rows_pad + row) * BT;
                if constexpr (BT == 4) {
                    *reinterpret_cast<float4*>(dst) = make_float4(static_cast<float>(acc[0]), static_cast<float>(acc[1]),
                                                                  static_cast<float>(acc[2]), static_cast<float>(acc[3]));
                } else if constexpr (BT == 2) {
                    *reinterpret_cast<float2*>(dst) = make_float2(static_cast<float>(acc[0]), static_cast<float>(acc[1]));
                } else {
                    dst[0] = static_cast<float>(acc[0]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
        seg = seg_end;
    }
    if (tl) g_timeline[blockIdx.x][4] = gtimer();
}

// y(r, c) = f32(sum_gb partial[gb][r][c]), fp64, blocks ascending (each
// partial already holds sum_i alpha_i * P_i of its block, combined in fp64).
// One thread per (column tile, row): the BT columns of a partial are one
// vector load, and every load is issued ahead of its use -- the partials in
// batches of KB vectors with the next batch in flight while the current one
// is summed (the finaliser is latency-bound otherwise).
template <int BT>
struct VecT;
template <>
struct VecT<1> {
    using T = float;
    static __device__ __forceinline__ float get(const float& v, int) { return v; }
};
template <>
struct VecT<2> {
    using T = float2;
    static __device__ __forceinline__ float get(const float2& v, int c) { return c == 0 ? v.x : v.y; }
};
template <>
struct VecT<4> {
    using T = float4;
    static __device__ __forceinline__ float get(const float4& v, int c) {
        return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
    }
};

// COLS = BT: a thread owns a whole column tile (vector loads); COLS = 2 or 1:
// a slice of it (BT / COLS times the threads -- for fewer output tiles; the
// launcher picks by tile count, measured crossovers).
template <int BT, int COLS>
__global__ void __launch_bounds__(128) finalize_kernel(const QueryParams p) {
    using V = typename VecT<COLS>::T;
    pdl_launch_dependents();
    pdl_wait();
    const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long CT = (p.b + BT - 1) / BT;
    constexpr int PER = BT / COLS;  // threads per column tile
    const long long cc = tid % PER, rt = tid / PER;  // cc: which COLS-wide slice of the tile
    const long long r = rt % p.m, ct = rt / p.m;
    if (ct >= CT || ct * BT + cc * COLS >= p.b) return;
    const long long rows_pad = static_cast<long long>(p.MT) * 32;
    const int total = p.NB;  // partial gb: [gb][ct][row][BT]
    const long long stride = CT * rows_pad * PER;  // in V units
    const V* src = reinterpret_cast<const V*>(p.partial) + (ct * rows_pad + r) * PER + cc;  // block 0
    constexpr int KB = COLS == 4 ? 8 : (COLS == 2 ? 16 : 32);
    V v[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k)
        if (k < total) v[k] = __ldcg(src + k * stride);  // (no loads past the last block: C4 b = 2 -0.8 us)
    double y[COLS];
#pragma unroll
    for (int c = 0; c < COLS; ++c) y[c] = 0.0;
#pragma unroll 1
    for (int q0 = 0; q0 < total; q0 += KB) {
        const bool more = q0 + KB < total;
        V nv[KB];
        if (more) {
#pragma unroll
            for (int k = 0; k < KB; ++k)
                if (q0 + KB + k < total) nv[k] = __ldcg(src + (q0 + KB + k) * stride);
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            if (q0 + k < total) {
#pragma unroll
                for (int c = 0; c < COLS; ++c) y[c] += static_cast<double>(VecT<COLS>::get(v[k], c));
            }
        }
        if (more) {
#pragma unroll
            for (int k = 0; k < KB; ++k) v[k] = nv[k];
        }
    }
    float* yr = p.y + r * p.b + ct * BT + cc * COLS;
#pragma unroll
    for (int c = 0; c < COLS; ++c)
        if (ct * BT + cc * COLS + c < p.b) yr[c] = static_cast<float>(y[c]);
    // fused all-gather: the same values into every peer's gather buffer (NVLink stores)
#pragma unroll 1
    for (int k = 0; k < kMaxPeers; ++k) {
        if (k >= p.npeer) break;
        float* py = p.peer_y[k] + (yr - p.peer_local);
#pragma unroll
        for (int c = 0; c < COLS; ++c)
            if (ct * BT + cc * COLS + c < p.b) py[c] = static_cast<float>(y[c]);
    }
    if (p.npeer > 0) __threadfence_system();  // peer stores performed before the grid completes
}

#ifndef BQG_FAST_NW
#define BQG_FAST_NW 12
#endif
constexpr int kNW = BQG_FAST_NW;

// Shared memory: the LUT, a ring of R stages of tps tiles (beta KiB each),
// 2 x kMaxStages mbarriers, the staged x tile.  BT = 1 runs two CTAs per SM.
constexpr size_t kSmemCap = 227 * 1024;
#ifndef BQG_FAST_MINR
#define BQG_FAST_MINR 2
#endif
constexpr size_t kMinStages = BQG_FAST_MINR;  // ring depth the stage size is chosen for
size_t lut_bytes(int mu, int bt) { return (size_t(1) << mu) * (bt == 1 ? 64 : 32 * bt) * 4; }
size_t smem_tail(int mu, int bt) { return 2 * kMaxStages * sizeof(uint64_t) + size_t(xs_words(mu, bt)) * 4; }
size_t fast_smem_bytes(const FastPlan& pl, int mu, int bt, int beta) {
    return lut_bytes(mu, bt) + size_t(pl.R) * pl.tps * beta * 1024 + smem_tail(mu, bt);
}
// tiles per stage and ring depth for (mu, BT, beta): as many tiles per stage
// as consumer warps while two stages fit, then as many stages as fit (<= 6).
bool ring_shape(int mu, int bt, int beta, FastPlan& pl) {
    for (size_t budget : {bt == 1 ? size_t(110 * 1024) : kSmemCap, kSmemCap}) {
        const size_t fixed = lut_bytes(mu, bt) + smem_tail(mu, bt) + 1024;
        if (fixed >= budget) continue;
        const size_t avail = budget - fixed, tile = size_t(beta) * 1024;
        const int tps = static_cast<int>(std::min<size_t>(kNW, avail / (kMinStages * tile)));
        if (tps < 1) continue;
        pl.tps = tps;
        // ring depth: 2 stages for BT = 4 (C3 25.66 -> 25.42, C5 147.9 ->
        // 147.4 us; b = 4..64 neutral), up to 6 otherwise (BT = 2: C4 b = 2
        // 13.0 at 2 vs 12.9 at 6); BQG_FAST_RMAX overrides (A/B knob)
        static const int rmax_env = [] {
            const char* e = getenv("BQG_FAST_RMAX");
            return e ? std::max(2, atoi(e)) : 0;
        }();
        const int rmax = rmax_env ? rmax_env : (bt == 4 ? 2 : 6);
        pl.R = static_cast<int>(std::min<size_t>(rmax, avail / (tps * tile)));
        return true;
    }
    return false;
}

template <int MU, int BT>
cudaError_t launch_mu_bt(const QueryParams& p, const FastPlan& plan, bool pdl, cudaStream_t stream) {
    auto kern = biqgemm_fast_kernel<MU, BT, kNW>;
    const size_t smem = fast_smem_bytes(plan, MU, BT, p.beta);
    static PerDeviceOnce configured;  // one attribute call per instantiation and device
    cudaError_t ea = once_per_device(configured, current_device(), [&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemCap));
    });
    if (ea != cudaSuccess) return ea;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(plan.grid));
    cfg.blockDim = dim3((kNW + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, plan);
    if (e != cudaSuccess) return e;
    if (p.debug & (1 << 20)) return cudaSuccess;  // profiling: no finaliser (y not written)
    // finaliser: always PDL-chained to the fused kernel
    cudaLaunchConfig_t f = {};
    // one thread per (column tile, row), or per (column tile, row, column)
    // when the tiles alone give fewer than 128 threads per SM (measured crossover)
    const long long tiles = static_cast<long long>(p.m) * ((p.b + BT - 1) / BT);
    const bool per_col = BT > 1 && tiles < 148LL * 128;
    const bool half = !per_col && BT == 4 && tiles < 148LL * 256;  // two threads per tile (float2)
    const long long n = per_col ? tiles * BT : (half ? tiles * 2 : tiles);
    f.gridDim = dim3(static_cast<unsigned>((n + 127) / 128));
    f.blockDim = dim3(128);
    f.stream = stream;
    cudaLaunchAttribute fa[1];
    fa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    fa[0].val.programmaticStreamSerializationAllowed = 1;
    f.attrs = fa;
    f.numAttrs = 1;
    if (per_col) return cudaLaunchKernelEx(&f, finalize_kernel<BT, 1>, p);
    if constexpr (BT == 4) {
        if (half) return cudaLaunchKernelEx(&f, finalize_kernel<4, 2>, p);
    }
    return cudaLaunchKernelEx(&f, finalize_kernel<BT, BT>, p);
}

template <int MU>
cudaError_t launch_mu(const QueryParams& p, const FastPlan& plan, int bt, bool pdl, cudaStream_t s) {
    if (bt == 1) return launch_mu_bt<MU, 1>(p, plan, pdl, s);
    if (bt == 2) return launch_mu_bt<MU, 2>(p, plan, pdl, s);
    return launch_mu_bt<MU, 4>(p, plan, pdl, s);
}

int pick_bt(long long b) {
    static const int force = [] {  // BQG_FAST_BT: experiment knob (1, 2 or 4)
        const char* e = getenv("BQG_FAST_BT");
        return e ? atoi(e) : 0;
    }();
    if (b > 1 && (force == 1 || force == 2 || force == 4)) return force;
    return b == 1 ? 1 : (b == 2 ? 2 : 4);
}

FastPlan make_plan(long long m, long long groups, int beta, long long b, int mu, int num_sms) {
    const int BT = pick_bt(b);
    FastPlan pl{};
    const long long NB = (groups + 31) / 32, MT = (m + 31) / 32;
    pl.CT = static_cast<int>((b + BT - 1) / BT);
    pl.cpp = static_cast<int>(MT);  // units: 32-row tiles (beta chunks each)
    if (!ring_shape(mu, BT, beta, pl)) pl.tps = pl.R = 0;  // the launcher rejects the shape
    const long long pairs = NB * pl.CT;
    const long long total = pairs * pl.cpp;
    // Cost model in shared-memory wavefronts (the binding resource): building
    // one block of tables = 2^mu * BT wavefronts (+ fixed overhead); one
    // tile = beta chunks of 32 (BT=1), 64 (BT=2) or 128 (BT=4) gather
    // wavefronts + 8 key wavefronts.
    const double build = static_cast<double>(1 << mu) * BT + 96.0;
    const double unit = beta * ((BT == 4 ? 128.0 : (BT == 2 ? 64.0 : 32.0)) + 8.0);
    const long long sms = std::max(1, num_sms);
    long long best_cpb = 1;
    double best_aligned = 1e300;
    for (long long cpb = 1; cpb <= std::max<long long>(1, std::min<long long>(pl.cpp, 4 * sms)); ++cpb) {
        const long long grid = pairs * cpb;
        const long long waves = (grid + sms - 1) / sms;
        const double t = static_cast<double>(waves) * (build + static_cast<double>((pl.cpp + cpb - 1) / cpb) * unit);
        if (t < best_aligned - 1e-9) {
            best_aligned = t;
            best_cpb = cpb;
        }
    }
    const long long fgrid = std::min<long long>(sms, total);
    const long long chunk = (total + fgrid - 1) / fgrid;
    const long long spans = std::min<long long>(pairs, (chunk + pl.cpp - 1) / pl.cpp + 1);
    const double t_flat = static_cast<double>(spans) * build + static_cast<double>(chunk) * unit;
    if (t_flat < best_aligned) {
        pl.mode = 1;
        pl.cpb = 1;
        pl.grid = static_cast<int>(fgrid);
        pl.q = static_cast<int>(total / fgrid);
        pl.r = static_cast<int>(total % fgrid);
    } else {
        pl.mode = 0;
        pl.cpb = static_cast<int>(best_cpb);
        pl.grid = static_cast<int>(pairs * best_cpb);
        pl.q = pl.cpp / pl.cpb;
        pl.r = pl.cpp % pl.cpb;
    }
    return pl;
}

}  // namespace

size_t fast_workspace_bytes(long long m, long long groups, int beta, long long b) {
    const long long NB = (groups + 31) / 32, MT = (m + 31) / 32;
    const long long BT = pick_bt(b), bpad = (b + BT - 1) / BT * BT;  // column tiles are written whole
    // the counters of the grouped forms first, then the partials of any form
    return kTexCounterBytes + static_cast<size_t>(NB) * beta * MT * 32 * std::max(b, bpad) * sizeof(float);
}

int plan_cpb(long long m, long long groups, int beta, long long b, int num_sms) {
    return make_plan(m, groups, beta, b, 8, num_sms).cpb;
}

// Shapes for the single-kernel cluster form.  b == 1 shapes the stream form
// takes are excluded: the latency and stream forms combine alpha per block
// before the block sum, the cluster form after it, and the choice must not
// depend on m (MT) -- else a layer and its row shards could take different
// forms and y would differ in the last bits across shardings.
bool cluster_shape(const QueryParams& p, int mu) {
    if (p.b == 1 && stream_supported(mu, p.beta, p.b)) return false;
    return p.b <= 4 && p.NB >= 8 && p.NB <= 16 && p.MT <= 256;
}

int fast_form(const QueryParams& p, int mu) {
    static const int debug_flags = [] {
        const char* e = getenv("BQG_DEBUG_FLAGS");
        return e ? atoi(e) : 0;
    }();
    if (!(debug_flags & (128 | 8192 | 16384)) && latency_supported(mu, p.beta, p.b, p.NB) && latency_applies(p)) return 1;
    if (!(debug_flags & 128) && (cluster_shape(p, mu) || (debug_flags & 8192))) return 2;  // (if the device can co-schedule it)
    if (!(debug_flags & (128 | 8192 | 65536)) && stream_supported(mu, p.beta, p.b)) return 4;
    return 3;
}

cudaError_t launch_biqgemm_fast(const QueryParams& p_in, int mu, bool pdl, cudaStream_t stream) {
    static const int debug_flags = [] {
        const char* e = getenv("BQG_DEBUG_FLAGS");  // profiling switches; never set in production
        return e ? atoi(e) : 0;
    }();
    const int sms = device_sms(current_device());
    QueryParams p = p_in;
    p.debug = debug_flags;
    p.bt = pick_bt(p.b);
    // The single-kernel cluster form wins when the per-call fixed costs
    // dominate and one column tile covers b (measured: C2 6.6 vs 8.5 us); the
    // two-kernel form (148 CTAs, cost-model split) wins for larger b / m.
    if (!(debug_flags & (128 | 8192 | 16384)) && latency_supported(mu, p.beta, p.b, p.NB)) {  // 16384: skip (profiling)
        bool used = false;
        cudaError_t e = launch_biqgemm_latency(p, pdl, stream, &used);
        if (e != cudaSuccess || used) return e;
    }
    if (!(debug_flags & 128) && (cluster_shape(p, mu) || (debug_flags & 8192))) {  // 128/8192: force a form (profiling)
        bool used = false;
        cudaError_t e = launch_biqgemm_cluster(p, mu, pdl, stream, &used);
        if (e != cudaSuccess || used) return e;
    }
    // b == 1, mu == 8, beta <= 4 shapes outside the latency / cluster forms
    // (large m, e.g. C4): the grouped stream form with a group of one beats
    // the two-kernel form (C4: 12.4 vs 14.0 us per dependent call), and its
    // y is bitwise the grouped form's.  The single-call workspace is larger
    // than the stream form's (beta x the partials).
    if (!(debug_flags & (128 | 8192 | 65536)) && stream_supported(mu, p.beta, p.b)) {
        const StreamCall call{p.keys, p.alpha, p.x, p.y};
        return launch_biqgemm_stream(&call, 1, p.x_rows, p.m, p.G, p.beta, p.ws, pdl, stream);
    }
    return launch_biqgemm_twokernel(p, mu, pdl, stream);
}

bool twokernel_supported(int mu, int beta, long long b) {
    if (mu < 1 || mu > 8 || beta < 1) return false;
    FastPlan pl{};
    return ring_shape(mu, pick_bt(b), beta, pl) && pl.R >= 2;
}

cudaError_t launch_biqgemm_twokernel(const QueryParams& p_in, int mu, bool pdl, cudaStream_t stream) {
    static const int debug_flags = [] {
        const char* e = getenv("BQG_DEBUG_FLAGS");
        return e ? atoi(e) : 0;
    }();
    if (p_in.npeer < 0 || p_in.npeer > kMaxPeers) return cudaErrorInvalidValue;
    const int sms = device_sms(current_device());
    QueryParams p = p_in;
    p.debug = debug_flags;
    p.bt = pick_bt(p.b);
    const FastPlan plan = make_plan(p.m, p.G, p.beta, p.b, mu, sms);
    if (plan.R < 2) return cudaErrorInvalidValue;  // beta too large for a two-stage key ring
    const int bt = pick_bt(p.b);
    switch (mu) {
        case 1: return launch_mu<1>(p, plan, bt, pdl, stream);
        case 2: return launch_mu<2>(p, plan, bt, pdl, stream);
        case 3: return launch_mu<3>(p, plan, bt, pdl, stream);
        case 4: return launch_mu<4>(p, plan, bt, pdl, stream);
        case 5: return launch_mu<5>(p, plan, bt, pdl, stream);
        case 6: return launch_mu<6>(p, plan, bt, pdl, stream);
        case 7: return launch_mu<7>(p, plan, bt, pdl, stream);
        case 8: return launch_mu<8>(p, plan, bt, pdl, stream);
        default: return cudaErrorInvalidValue;
    }
}

// ---- parity entry: the same bank-owned builder, dumped in the reference layout ----

namespace {

template <int MU>
__global__ void __launch_bounds__(256) build_lut_dump_kernel(const float* __restrict__ x, long long x_rows,
                                                             long long b, long long g0, long long count,
                                                             bool key_major, float* __restrict__ out) {
    __shared__ float tab[(1 << MU) * 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long col = blockIdx.y;
    const long long gl = static_cast<long long>(blockIdx.x) * 32 + lane;  // local group
    build_bank_owned_tables<MU, 8, 1>(tab, x, x_rows, b, g0 + gl, col, warp, lane);
    __syncthreads();
    constexpr int TABLE = 1 << MU;
    for (int idx = threadIdx.x; idx < TABLE * 32; idx += blockDim.x) {
        const int k = idx >> 5, l = idx & 31;
        const long long g = static_cast<long long>(blockIdx.x) * 32 + l;
        if (g >= count) continue;
        const long long base = g * b * TABLE;
        const long long o = key_major ? base + static_cast<long long>(k) * b + col : base + col * TABLE + k;
        out[o] = tab[idx];
    }
}

}  // namespace

cudaError_t launch_build_lut_f32(const float* x, long long x_rows, long long b, int mu, long long g0,
                                 long long count, bool key_major, float* out, cudaStream_t stream) {
    const dim3 grid(static_cast<unsigned>((count + 31) / 32), static_cast<unsigned>(b));
    switch (mu) {
#define BQG_CASE(M)                                                                                      \
    case M:                                                                                              \
        build_lut_dump_kernel<M><<<grid, 256, 0, stream>>>(x, x_rows, b, g0, count, key_major, out); \
        break;
        BQG_CASE(1)
        BQG_CASE(2)
        BQG_CASE(3)
        BQG_CASE(4)
        BQG_CASE(5)
        BQG_CASE(6)
        BQG_CASE(7)
        BQG_CASE(8)
#undef BQG_CASE
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace bqg

extern "C" int bqg_debug_timeline(unsigned long long* out, int rows) {
    return cudaMemcpyFromSymbol(out, bqg::g_timeline, sizeof(unsigned long long) * 8 * (rows < 8192 ? rows : 8192)) ==
                   cudaSuccess
               ? 0
               : 2;
}
