// biqgemm_latency.cu -- the single-call latency form: b == 1, mu == 8,
// 1 <= beta <= 4, NB = ceil(G/32) <= 16 (n <= 4096).  One BiQGEMM call
// (/root/reference/proj/core/include/biqgemm/kernel.hpp:246-258 ->
// detail::run 116-204) as ONE kernel whose critical path after
// griddepcontrol.wait is: x -> LUT -> gather -> in-cluster push reduction ->
// y.  Everything that does not depend on x (keys, alpha, barrier setup, the
// cluster rendezvous) is issued before the wait, overlapping the predecessor.
//
// Decomposition: a cluster of CS CTAs owns a contiguous range of 32-row
// tiles and ALL NB group blocks; CTA rank s owns blocks s*bpc .. s*bpc+bpc-1
// (bpc = NB/CS = 1 or 2; the two blocks' tables are the two halves of one
// 64 KiB bank-owned LUT region, as in biqgemm_stream.cu).
//   - key lanes issue the CTA's whole key range (contiguous per block in the
//     tiled layout) as <= 8 KiB TMA bulk copies from parallel lanes, each on
//     its own single-use mbarrier; one lane copies the alpha rows;
//   - after the wait, every warp builds a share of the tables (the DP
//     recurrence walked depth-first, bit-exact with lut.hpp:50-69);
//   - warps gather chunks (tile, plane) w, w+16, ... (FADD2 pairs, the
//     stream form's order) into per-chunk sums;
//   - per (block, row) the plane sums are combined with alpha in fp64 and the
//     fp32 partial is pushed with st.async into the shared memory of the CTA
//     that owns the row, completing a transaction count on its mbarrier;
//   - the owner sums the NB partials of its rows in ascending block order in
//     fp64 and stores y.
// The arithmetic is the stream form's (per block: sum_i alpha_i * P_i in
// fp64 -> fp32; blocks ascending in fp64), so y is bitwise identical to
// bqg_biqgemm_grouped_f32 and independent of the cluster split.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "lut_build.cuh"  // Log2

#ifndef BQG_LAT_PIECE
#define BQG_LAT_PIECE 8
#endif

namespace bqg {

// Per-CTA timeline (BQG_DEBUG_FLAGS & 2): globaltimer ns at start, after the
// cluster rendezvous, after griddepcontrol.wait, LUT built, gather done,
// partials pushed, y stored, prologue barrier; thread 0: x loaded, its DFS
// done, first key piece landed, its last chunk gathered.  Off in production.
__device__ unsigned long long g_timeline_lat[1024][16];

namespace {

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// The timer read is ordered after v is available (v is an asm input).
__device__ __forceinline__ unsigned long long gtime_after(float v) {
    unsigned long long t;
    asm volatile("{\n\t.reg .f32 d;\n\tmov.f32 d, %1;\n\tmov.u64 %0, %%globaltimer;\n}" : "=l"(t) : "f"(v));
    return t;
}

constexpr int kMU = 8;
constexpr int kTable = 1 << kMU;
constexpr int kLW = 18;                    // warps per CTA (all gather; the first 16 build)
constexpr int kLB = 16;                    // builder warps
constexpr int kLThreads = kLW * 32;
constexpr int kPieceChunks = BQG_LAT_PIECE;  // chunks (KiB) per key copy
constexpr int kMaxPieces = 64;
constexpr int kBarBytes = 1024;  // kbar[kMaxPieces] + abar + pbar
constexpr uint32_t kLutBytes = 0x10000u;  // 256 key rows x 256 B (32 tables x 2 blocks x fp32)
constexpr int kLatSmem = 227 * 1024;      // the most a CTA may ask for
constexpr int kLatSmemMin = 116 * 1024;   // > half an SM's 228 KiB: one CTA per SM

struct LatArgs {
    int debug;            // BQG_DEBUG_FLAGS & 2: per-CTA globaltimer timeline
    const uint8_t* keys;  // tiled
    const float* alpha;   // beta x m or nullptr
    const float* x;
    float* y;
    long long x_rows;
    int m, NB, MT, CS, bpc, tq, tr;
    int smem;             // dynamic shared memory bytes: LUT + bars/alpha/sums/slots + keys
};

__device__ __forceinline__ void sts_pair(uint32_t col, int k, float v) {
    sts_f32(col + static_cast<uint32_t>(k) * 256u, v);
    sts_f32(col + static_cast<uint32_t>(kTable - 1 - k) * 256u, -v);
}

// DFS over the low LB key bits; builder q owns the keys whose bits LB..6 equal
// q (the recurrence's own order: e[j | q<<LB] = ((e[j] + s_LB?) ...) + s_6?).
// One code path for all builders: q is a warp-uniform runtime value (the
// high-bit adds are uniformly predicated), so the cold code fetched per call
// is one DFS, not one per builder.
template <int K, int I, int LB>
struct LDfs {
    static __device__ __forceinline__ void children(float v, const float (&s)[kMU], uint32_t col, int q) {
        if constexpr (I < LB) {
            LDfs<(K | (1 << I)), I + 1, LB>::node(fadd_rn(v, s[I]), s, col, q);
            LDfs<K, I + 1, LB>::children(v, s, col, q);
        }
    }
    static __device__ __forceinline__ void node(float v, const float (&s)[kMU], uint32_t col, int q) {
        float e = v;
#pragma unroll
        for (int t = LB; t < 7; ++t)
            if ((q >> (t - LB)) & 1) e = fadd_rn(e, s[t]);
        sts_pair(col, K | (q << LB), e);
        children(v, s, col, q);
    }
};

// Builder `which` of NBW for the tables of groups gb*32 + lane (x rows
// gb*256 + lane*8 .. +7, zero past x_rows) into the LUT half at col.
template <int NBW>
__device__ __forceinline__ void build_share(int which, uint32_t col, const float* __restrict__ x, long long x_rows,
                                            int gb, int lane, unsigned long long* tl) {
    float xv[kMU], s[kMU];
    const long long r0 = static_cast<long long>(gb) * 32 * kMU + lane * kMU;
    if (r0 + kMU <= x_rows && (reinterpret_cast<uintptr_t>(x + r0) & 15) == 0) {
        const float4 a = __ldcg(reinterpret_cast<const float4*>(x + r0));
        const float4 b = __ldcg(reinterpret_cast<const float4*>(x + r0 + 4));
        xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
        xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
    } else {
#pragma unroll
        for (int t = 0; t < kMU; ++t) xv[t] = r0 + t < x_rows ? __ldcg(x + r0 + t) : 0.0f;
    }
    float e0 = 0.0f;
#pragma unroll
    for (int t = 0; t < kMU; ++t) e0 = __fsub_rn(e0, xv[t]);
    if (tl) tl[8] = gtime_after(e0);  // x has arrived
#pragma unroll
    for (int t = 0; t < kMU; ++t) s[t] = 2.0f * xv[t];
    LDfs<0, 0, 7 - Log2<NBW>::value>::node(e0, s, col, which);
    if (tl) tl[9] = gtime();
}

// ---- gather (identical arithmetic to biqgemm_stream.cu) -------------------
// base = the LUT's shared address (warp-uniform; ptxas keeps it in a
// uniform register and folds it into the LDS address: [R + UR + imm]).
template <int IMM>
__device__ __forceinline__ float lds_lut(uint32_t rotw, uint32_t w, uint32_t sel, uint32_t base) {
    uint32_t off;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(off) : "r"(rotw), "r"(w), "r"(sel));
    float e;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(e) : "r"(off + base), "n"(IMM));
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
template <int IMM>
__device__ __forceinline__ float gather_chunk_l(uint32_t kaddr, int lane, const uint32_t (&rot)[8], uint32_t base) {
    uint32_t w[8];
    const uint32_t p = kaddr + static_cast<uint32_t>(lane) * 16u;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(p));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+512];" : "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "r"(p));
    uint64_t acc01 = 0, acc23 = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float e0 = lds_lut<IMM>(rot[q], w[q], 0x8840u, base);
        const float e1 = lds_lut<IMM>(rot[q], w[q], 0x8851u, base);
        const float e2 = lds_lut<IMM>(rot[q], w[q], 0x8862u, base);
        const float e3 = lds_lut<IMM>(rot[q], w[q], 0x8873u, base);
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

__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(remote_addr),
                 "r"(__float_as_uint(v)), "r"(remote_bar)
                 : "memory");
}

template <int BETA>
__global__ void __launch_bounds__(kLThreads, 1) biqgemm_latency_kernel(const __grid_constant__ LatArgs A) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool tl = (A.debug & 2) && threadIdx.x == 0 && blockIdx.x < 1024;
    if (tl) g_timeline_lat[blockIdx.x][0] = gtime();
    const int CS = A.CS, bpc = A.bpc;
    const int s_rank = static_cast<int>(cluster_ctarank());
    const int cid = blockIdx.x / CS;
    const int T0 = cid * A.tq + min(cid, A.tr);
    const int nt = A.tq + (cid < A.tr ? 1 : 0);                  // tiles of this cluster
    const int rows = min(nt * 32, A.m - T0 * 32);                 // real rows
    const int rpo = (rows + CS - 1) / CS;                          // rows per owner rank
    const int own0 = min(s_rank * rpo, rows), own1 = min(own0 + rpo, rows);
    const int nchunk_b = nt * BETA;                                // chunks per block
    const int nchunk = nchunk_b * bpc;
    const int npb = (nchunk_b + kPieceChunks - 1) / kPieceChunks;  // key pieces per block
    const int npieces = npb * bpc;

    // ---- shared memory: [LUT 64 KiB | bars | alpha | psum | push slots | keys]
    // sized to what the call needs (A.smem, at least kLatSmemMin: one CTA per
    // SM).  The LUT is at the start of the dynamic window; the gather
    // addresses it as [PRMT result + LUT base (uniform) + imm].
    const uint32_t sbase = smem_u32(smem);
    const uint32_t lut_abs = sbase;
    uint64_t* kbar = reinterpret_cast<uint64_t*>(smem + kLutBytes);  // [kMaxPieces]
    uint64_t* abar = kbar + kMaxPieces;                              // alpha landed
    uint64_t* pbar = abar + 1;                                       // pushes into this CTA landed
    float* as = reinterpret_cast<float*>(smem + kLutBytes + kBarBytes);  // [BETA][nt*32]
    float* psum = as + BETA * nt * 32;                                   // [nchunk][32]
    float* slots = psum + nchunk * 32;                                   // [NB][rpo]
    const uint32_t lo_end = smem_u32(slots + A.NB * rpo);
    const uint32_t keys_at = (lo_end + 127u) & ~127u;
    const uint32_t kbytes = static_cast<uint32_t>(nchunk) * 1024u;
    if ((sbase & 127u) != 0 || keys_at + kbytes > sbase + static_cast<uint32_t>(A.smem) || npieces > kMaxPieces) __trap();

    const uint32_t own_bytes = static_cast<uint32_t>(own1 - own0) * 4u * static_cast<uint32_t>(A.NB);
    if (threadIdx.x == 0) {
        for (int p = 0; p < npieces; ++p) mbar_init(&kbar[p], 1);
        const uint32_t ab = static_cast<uint32_t>(rows) * 4u;
        const bool atma = A.alpha && (ab & 15) == 0 && (A.m & 3) == 0 &&
                          (reinterpret_cast<uintptr_t>(A.alpha) & 15) == 0;
        mbar_init(abar, atma ? BETA : 1);
        mbar_init(pbar, 1);
        fence_mbar_init();
        // arm the push barrier before any peer can push (cluster barrier below)
        mbar_arrive_expect_tx(pbar, own_bytes);
    }
    __syncthreads();
    if (tl) g_timeline_lat[blockIdx.x][7] = gtime();
    pdl_launch_dependents();

    // ---- pre-wait: keys and alpha (immutable) stream in from parallel lanes
    if (warp == kLW - 1) {
        const uint64_t pol = policy_evict_first();
        for (int p = lane; p < npieces; p += 32) {
            const int b = p / npb, j = p - b * npb;
            const int c0 = j * kPieceChunks, cn = min(kPieceChunks, nchunk_b - c0);
            const long long gb = static_cast<long long>(s_rank) * bpc + b;
            const unsigned char* src = A.keys + ((gb * A.MT + T0) * BETA + c0) * 1024;
            mbar_arrive_expect_tx(&kbar[p], static_cast<uint32_t>(cn) * 1024u);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                    keys_at + static_cast<uint32_t>(b * nchunk_b + c0) * 1024u),
                "l"(src), "r"(static_cast<uint32_t>(cn) * 1024u), "r"(smem_u32(&kbar[p])), "l"(pol)
                : "memory");
        }
        if ((A.debug & 2) && lane == 0 && blockIdx.x < 1024) g_timeline_lat[blockIdx.x][12] = gtime();
        // alpha: one plane per lane (lanes 31, 30, ...), all on abar
        {
            const uint32_t ab = static_cast<uint32_t>(rows) * 4u;
            const bool tma = A.alpha && (ab & 15) == 0 && (A.m & 3) == 0 &&
                             (reinterpret_cast<uintptr_t>(A.alpha) & 15) == 0;
            const int i = 31 - lane;
            if (tma && i < BETA) {
                if (i == 0) mbar_arrive_expect_tx(abar, ab * BETA);
                else mbar_arrive(abar);
                bulk_g2s_plain(as + i * nt * 32, A.alpha + static_cast<long long>(i) * A.m + T0 * 32, ab, abar);
            } else if (!tma && lane == 31) {
                mbar_arrive(abar);  // alpha loaded by the threads below
            }
        }
    }
    {
        const uint32_t ab = static_cast<uint32_t>(rows) * 4u;
        const bool tma = A.alpha && (ab & 15) == 0 && (A.m & 3) == 0 &&
                         (reinterpret_cast<uintptr_t>(A.alpha) & 15) == 0;
        if (!tma) {
            for (int idx = threadIdx.x; idx < BETA * nt * 32; idx += kLThreads) {
                const int i = idx / (nt * 32), rl = idx - i * nt * 32;
                as[idx] = (rl < rows) ? (A.alpha ? __ldg(A.alpha + static_cast<long long>(i) * A.m + T0 * 32 + rl) : 1.0f)
                                      : 0.0f;
            }
        }
    }
    // every CTA's push barrier is initialised before any peer pushes: arrive
    // now, wait just before the push phase.  fence.mbarrier_init (above)
    // publishes the init; the arrive can be relaxed (a release arrive would
    // wait for this CTA's outstanding memory operations: ~1.3 us measured).
    __syncwarp();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    if (tl) g_timeline_lat[blockIdx.x][1] = gtime();
    uint32_t rot[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        rot[q] = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) rot[q] |= (static_cast<uint32_t>((lane + 4 * q + b) & 31) * 4u) << (8 * b);
    }

    pdl_wait();  // x of the predecessor is visible from here on
    if (tl) g_timeline_lat[blockIdx.x][2] = gtime();

    // ---- LUT: bpc blocks, kLB / bpc builder warps each
    if (warp < kLB) {
        const int b = warp / (kLB / bpc), which = warp - b * (kLB / bpc);
        const uint32_t col = lut_abs + static_cast<uint32_t>(b) * 128u + static_cast<uint32_t>(lane) * 4u;
        const int gb = s_rank * bpc + b;
        unsigned long long* tlw = (tl && warp == 0) ? g_timeline_lat[blockIdx.x] : nullptr;
        if (bpc == 1) build_share<16>(which, col, A.x, A.x_rows, gb, lane, tlw);
        else build_share<8>(which, col, A.x, A.x_rows, gb, lane, tlw);
    }
    __syncthreads();
    if (tl) g_timeline_lat[blockIdx.x][3] = gtime();

    // ---- gather: chunk q = (block b, tile k, plane i), warps take q = w, w+kLW, ...
    for (int q = warp; q < nchunk; q += kLW) {
        const int b = q / nchunk_b, c = q - b * nchunk_b;
        mbar_wait(&kbar[b * npb + c / kPieceChunks], 0);
        if (tl && q == 0) g_timeline_lat[blockIdx.x][10] = gtime();
        const uint32_t ka = keys_at + static_cast<uint32_t>(q) * 1024u;
        const float P = b == 0 ? gather_chunk_l<0>(ka, lane, rot, lut_abs) : gather_chunk_l<128>(ka, lane, rot, lut_abs);
        psum[q * 32 + lane] = P;
    }
    if (tl) {
        g_timeline_lat[blockIdx.x][11] = gtime();
        for (int p = 0; p < npieces; ++p) mbar_wait(&kbar[p], 0);
        g_timeline_lat[blockIdx.x][13] = gtime();
    }
    mbar_wait(abar, 0);
    __syncthreads();
    if (tl) g_timeline_lat[blockIdx.x][4] = gtime();

    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    // ---- per (block, row): alpha-combine in fp64, push the fp32 partial to the row's owner
    for (int idx = threadIdx.x; idx < bpc * nt * 32; idx += kLThreads) {
        const int b = idx / (nt * 32), rl = idx - b * nt * 32;
        if (rl >= rows) continue;
        const int k = rl >> 5, l = rl & 31;
        double sacc = 0.0;
#pragma unroll
        for (int i = 0; i < BETA; ++i)
            sacc += static_cast<double>(as[i * nt * 32 + rl]) *
                    static_cast<double>(psum[((b * nt + k) * BETA + i) * 32 + l]);
        const int o = rl / rpo;  // owner rank
        const int gb = s_rank * bpc + b;
        const uint32_t local = smem_u32(slots + gb * rpo + (rl - o * rpo));
        st_async_f32(dsmem_map(local, static_cast<uint32_t>(o)), static_cast<float>(sacc),
                     dsmem_map(smem_u32(pbar), static_cast<uint32_t>(o)));
    }

    // ---- owner: sum the NB partials of its rows, blocks ascending
    if (tl) g_timeline_lat[blockIdx.x][5] = gtime();
    if (own1 > own0) {
        mbar_wait(pbar, 0);
        for (int rl = own0 + threadIdx.x; rl < own1; rl += kLThreads) {
            double yv = 0.0;
            for (int gb = 0; gb < A.NB; ++gb) yv += static_cast<double>(slots[gb * rpo + (rl - own0)]);
            A.y[static_cast<long long>(T0) * 32 + rl] = static_cast<float>(yv);
        }
    }
    if (tl) g_timeline_lat[blockIdx.x][6] = gtime();
}

template <int BETA>
cudaError_t set_lat_attributes(int dev) {
    static PerDeviceOnce configured;
    return once_per_device(configured, dev, [] {
        auto kern = biqgemm_latency_kernel<BETA>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kLatSmem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return e;
    });
}

template <int BETA>
cudaError_t launch_lat_beta(const LatArgs& A, int nclusters, bool pdl, cudaStream_t stream) {
    auto kern = biqgemm_latency_kernel<BETA>;
    cudaError_t ea = set_lat_attributes<BETA>(current_device());
    if (ea != cudaSuccess) return ea;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(A.CS);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(nclusters * A.CS));
    cfg.blockDim = dim3(kLThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(A.smem);
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, A);
}

template <int BETA>
int max_clusters(int cs) {
    static std::atomic<int> cache[kMaxDevices][17];
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) return -1;
    const int have = cache[dev][cs].load(std::memory_order_relaxed);
    if (have != 0) return have;
    auto kern = biqgemm_latency_kernel<BETA>;
    if (set_lat_attributes<BETA>(dev) != cudaSuccess) return -1;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(cs));
    cfg.blockDim = dim3(kLThreads);
    cfg.dynamicSmemBytes = kLatSmem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = -1;
    }
    const int v = n > 0 ? n : -1;
    cache[dev][cs].store(v, std::memory_order_relaxed);
    return v;
}

}  // namespace

// NB group blocks split over a cluster of CS CTAs, NB / CS = 1 or 2 blocks each
// (CS <= 16: NB <= 16, i.e. n <= 4096 at mu = 8; any NB -- clusters of 3, 5,
// 6, 7, ... CTAs included, e.g. n = 3072: NB = 12, clusters of 6 or 12)
bool latency_supported(int mu, int beta, long long b, int NB) {
    return mu == kMU && b == 1 && beta >= 1 && beta <= 4 && NB >= 1 && NB <= 16;
}

namespace {
bool plan_latency(const QueryParams& p, LatArgs& A, int& nclusters);
}

bool latency_applies(const QueryParams& p) {
    if (!latency_supported(8, p.beta, p.b, p.NB)) return false;
    LatArgs A{};
    int nc = 0;
    return plan_latency(p, A, nc);
}

cudaError_t launch_biqgemm_latency(const QueryParams& p, bool pdl, cudaStream_t stream, bool* used) {
    *used = false;
    LatArgs A{};
    int nclusters = 0;
    if (!plan_latency(p, A, nclusters)) return cudaSuccess;
    *used = true;
    switch (p.beta) {
        case 1: return launch_lat_beta<1>(A, nclusters, pdl, stream);
        case 2: return launch_lat_beta<2>(A, nclusters, pdl, stream);
        case 3: return launch_lat_beta<3>(A, nclusters, pdl, stream);
        default: return launch_lat_beta<4>(A, nclusters, pdl, stream);
    }
}

namespace {
bool plan_latency(const QueryParams& p, LatArgs& A, int& nclusters) {
    A.debug = p.debug;
    A.keys = p.keys;
    A.alpha = p.alpha;
    A.x = p.x;
    A.y = p.y;
    A.x_rows = p.x_rows;
    A.m = p.m;
    A.NB = p.NB;
    A.MT = p.MT;
    // cluster of CS CTAs x bpc blocks per CTA: the shape that covers the most SMs
    int best_cs = 0, best_n = 0;
    for (int cs = 16; cs >= 1; --cs) {
        if (cs > A.NB || A.NB % cs != 0 || A.NB / cs > 2) continue;
        int n = 0;
        switch (p.beta) {
            case 1: n = max_clusters<1>(cs); break;
            case 2: n = max_clusters<2>(cs); break;
            case 3: n = max_clusters<3>(cs); break;
            default: n = max_clusters<4>(cs); break;
        }
        if (n > 0 && n * cs > best_n * best_cs) {
            best_cs = cs;
            best_n = n;
        }
    }
    if (best_cs == 0) return false;
    A.CS = best_cs;
    A.bpc = A.NB / best_cs;
    nclusters = std::min(best_n, A.MT);
    A.tq = A.MT / nclusters;
    A.tr = A.MT % nclusters;
    // shared memory of the largest cluster range: LUT, bars, alpha, sums, slots, keys
    {
        const long long nt = A.tq + (A.tr ? 1 : 0);
        const long long lo = kBarBytes + 4 * nt * 32 * p.beta + 4 * nt * 32 * p.beta * A.bpc +
                             4LL * A.NB * ((nt * 32 + A.CS - 1) / A.CS);
        const long long keys = nt * p.beta * A.bpc * 1024;
        const long long need = (static_cast<long long>(kLutBytes) + lo + 128 + keys + 1023) / 1024 * 1024;
        if (need > kLatSmem || (nt * p.beta + kPieceChunks - 1) / kPieceChunks * A.bpc > kMaxPieces) return false;
        // At least kLatSmemMin: one CTA per SM.  A second CTA on the SM (a
        // smaller request) was measured SLOWER (beta = 1: 4.87 vs 4.04 us per
        // dependent call, beta = 2: 6.29 vs 4.97): the cluster scheduler then
        // packs a call's own CTAs two per SM.  Asking for less than the
        // whole 227 KiB leaves L1 for x and the alpha rows (BQG_LAT_SMEM=full:
        // the old 227 KiB request, for A/B).
        static const bool full = [] {
            const char* e = getenv("BQG_LAT_SMEM");
            return e && e[0] == 'f';
        }();
        A.smem = full ? kLatSmem : static_cast<int>(std::max<long long>(need, kLatSmemMin));
    }
    return true;
}
}  // namespace

}  // namespace bqg

extern "C" int bqg_debug_timeline_latency(unsigned long long* out, int rows) {
    return cudaMemcpyFromSymbol(out, bqg::g_timeline_lat, sizeof(unsigned long long) * 16 * (rows < 1024 ? rows : 1024)) ==
                   cudaSuccess
               ? 0
               : 2;
}
