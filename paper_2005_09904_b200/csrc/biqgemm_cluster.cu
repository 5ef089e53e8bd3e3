// biqgemm_cluster.cu -- single-kernel BiQGEMM (mu <= 8) with the cross-SM
// reduction done inside a thread-block cluster.
//
// Same algorithm and data layout as biqgemm_fast.cu (see there and
// kernels.h), different work decomposition:
//   - a cluster of CS CTAs (CS = min(NB, 16), one CTA per SM) owns a
//     contiguous range of 32-row tiles and ALL group blocks: CTA rank r
//     handles group blocks r, r+CS, r+2CS, ... (one LUT build each) and
//     accumulates its blocks' partial sums (fp32, blocks ascending) into
//     partial[r][plane][row][col] in global memory (L2-resident);
//   - one cluster barrier (release/acquire at cluster scope) publishes them;
//   - every CTA of the cluster then finalises an equal slice of the
//     cluster's outputs: y = sum_i alpha_i * sum_r partial[r][i] in fp64,
//     planes and ranks ascending (kernel.hpp:183-195).
// No second kernel, no atomics, no "last CTA" tail: every CTA does the same
// work.  The reduction order of an output is a function of (n, mu) only
// (through NB and CS), so y is bitwise identical for every row split and
// row sharding with 32-row-aligned boundaries.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "lut_build.cuh"
#include "query_core.cuh"

namespace bqg {

// Per-CTA timeline for profiling (BQG_DEBUG_FLAGS & 2); see biqgemm_fast.cu.
__device__ unsigned long long g_timeline_c[8192][16];

namespace {

__device__ __forceinline__ unsigned long long gtimer_c() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct ClusterPlan {
    int cs;         // CTAs per cluster (= group-block stride)
    int nclusters;
    int CT;         // column tiles of BT columns
    int tq, tr;     // 32-row tiles per cluster: cluster c gets tq + (c < tr)
    int dsm;        // 1: partial sums stay in shared memory (DSMEM reduction)
};

constexpr int kPSUM = 24 * 1024;  // bytes of shared memory for per-CTA partial sums (DSMEM mode)

template <int MU, int BT, int NW, int R>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    biqgemm_cluster_kernel(const QueryParams p, const ClusterPlan plan) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int LUT_BYTES = (1 << MU) * LutGeom<BT>::KROW * 4;
    constexpr int STAGE_BYTES = NW * 1024;
    constexpr int STAGE_AREA = R * STAGE_BYTES + 2 * R * 8;
    // BT <= 2: place the LUT at a 64 KiB-aligned shared address so PRMT
    // builds the complete gather address (no add per lookup).  The other
    // regions (key stages + barriers, partial sums) go into the alignment
    // gap in front of the LUT when they fit, else behind it.
    constexpr bool ABS = LutGeom<BT>::PRMT;
    const uint32_t sbase = smem_u32(smem);
    uint32_t lut_abs = 0, gap = 0;
    if constexpr (ABS) {
        lut_abs = (sbase + 0xFFFFu) & ~0xFFFFu;
        gap = lut_abs - sbase;
    }
    float* lut = reinterpret_cast<float*>(smem + gap);
    uint32_t lo_cur = 0, hi_cur = gap + LUT_BYTES;
    auto place = [&](uint32_t bytes) -> unsigned char* {
        if (lo_cur + bytes <= gap) {
            unsigned char* a = smem + lo_cur;
            lo_cur += bytes;
            return a;
        }
        unsigned char* a = smem + hi_cur;
        hi_cur += bytes;
        return a;
    };
    unsigned char* stages = place(STAGE_AREA);
    float* psum = reinterpret_cast<float*>(place(kPSUM));
    float* xs = reinterpret_cast<float*>(place(xs_words(MU, BT) * 4));  // staged x tile of the current segment
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + R * STAGE_BYTES);
    uint64_t* empty = full + R;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool tl = (p.debug & 2) && threadIdx.x == 0 && blockIdx.x < 8192;
    if (tl) {
        g_timeline_c[blockIdx.x][0] = gtimer_c();
    }
    pdl_launch_dependents();

    const int cs = plan.cs;
    const int rank = static_cast<int>(cluster_ctarank());
    const int cid = static_cast<int>(blockIdx.x) / cs;
    const int T0 = cid * plan.tq + min(cid, plan.tr);
    const int T1 = T0 + plan.tq + (cid < plan.tr ? 1 : 0);
    const int beta = p.beta;
    const int cps = (T1 - T0) * beta;  // key chunks per (group block, column tile) segment
    const long long rows_pad = static_cast<long long>(p.MT) * 32;
    const int nblk = (p.NB - rank + cs - 1) / cs;  // group blocks of this rank
    const int nrl = (T1 - T0) * 32;                 // rows of this cluster (padded to tiles)
    const int nseg = nblk * plan.CT;

    if (threadIdx.x == 0) {
        for (int s = 0; s < R; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
        if (tl) g_timeline_c[blockIdx.x][14] = gtimer_c();
    }
    __syncthreads();
    if (tl) g_timeline_c[blockIdx.x][15] = gtimer_c();

    // This CTA's slice of the cluster's outputs (row-major over rows x b).
    const int nr = max(0, min(T1 * 32, p.m) - T0 * 32);  // real rows of this cluster
    const long long nout = static_cast<long long>(nr) * p.b;
    const long long o_lo = nout * rank / cs, o_hi = nout * (rank + 1) / cs;

    if (warp == NW) {
        // ------------------------------------------------ producer (1 lane)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int sc = 0;
            for (int sg = 0; sg < nseg; ++sg) {
                const int gb = rank + (sg % nblk) * cs;
                const unsigned char* kseg =
                    p.keys + ((static_cast<long long>(gb) * p.MT + T0) * beta) * 1024;
                for (int c0 = 0; c0 < cps; c0 += NW, ++sc) {
                    const int cnt = min(NW, cps - c0);
                    const int slot = sc % R;
                    if (sc >= R) mbar_wait(&empty[slot], ((sc / R) & 1) ^ 1);  // first R stages are free
                    // stage 0 lands alone before the rest of the fill is requested
                    // (C2 b = 2 7.94 -> 7.82 us, b = 3 / 4 neutral; bit 21: old order)
                    if (sc == 1 && !(p.debug & (1 << 21))) mbar_wait(&full[0], 0);
                    if ((p.debug & 2) && blockIdx.x < 8192 && sc == 0) g_timeline_c[blockIdx.x][13] = gtimer_c();
                    mbar_arrive_expect_tx(&full[slot], cnt * 1024);
                    bulk_g2s(stages + slot * STAGE_BYTES, kseg + static_cast<long long>(c0) * 1024, cnt * 1024,
                             &full[slot], pol);
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------------------------------------------- consumers
        uint32_t goff[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) goff[j] = lut_abs | (static_cast<uint32_t>((lane + j) & 31) * 4u * BT);
        const uint32_t lut_s = smem_u32(lut);
        if (tl) g_timeline_c[blockIdx.x][12] = gtimer_c();
        pdl_wait();  // x (and the workspace) of the predecessor are visible from here on
        if (tl) {
            g_timeline_c[blockIdx.x][1] = gtimer_c();
            if (p.debug & 1024) {  // profiling: latency of one x load right now
                const unsigned long long a = gtimer_c();
                const float v = __ldcg(p.x + (blockIdx.x * 64) % p.x_rows);
                const unsigned long long bb = gtimer_c();
                g_timeline_c[blockIdx.x][8] = bb - a + (v == 1234.5f ? 1 : 0);
                const unsigned long long c2 = gtimer_c();
                const float v2 = __ldcg(reinterpret_cast<const float*>(p.keys) + (blockIdx.x * 999) % 1000);
                g_timeline_c[blockIdx.x][9] = gtimer_c() - c2 + (v2 == 1234.5f ? 1 : 0);
            }
        }
        const int dq = NW / beta, dr = NW - (NW / beta) * beta;
        int sc = 0;
        // x tile of segment sg+1 loaded into registers during segment sg (the
        // values stage_x_tile would read), stored at the segment boundary
        constexpr int XT = 32 * MU * BT, XPT = (XT + NW * 32 - 1) / (NW * 32);
        float xr[XPT];
        auto load_x = [&](int sgx) {
            const int ctx = sgx / nblk;
            const long long gbx = rank + (sgx - ctx * nblk) * cs, col0 = static_cast<long long>(ctx) * BT;
            const long long r0 = gbx * 32 * MU;
#pragma unroll
            for (int k = 0; k < XPT; ++k) {
                const int idx = threadIdx.x + k * NW * 32;
                const int rl = idx / BT, c = idx - (idx / BT) * BT;
                const long long r = r0 + rl, col = col0 + c;
                xr[k] = (idx < XT && r < p.x_rows && col < p.b) ? __ldcg(p.x + r * p.b + col) : 0.0f;
            }
        };
        if (nseg > 0) load_x(0);
        for (int sg = 0; sg < nseg; ++sg) {
            const int ct = sg / nblk;
            const int bi = sg - ct * nblk;
            const int gb = rank + bi * cs;
            const bool first = bi == 0;  // first group block of this rank for this column tile
            if (sg != 0) named_bar_sync(1, NW * 32);  // previous segment done with the LUT and x tile
#pragma unroll
            for (int k = 0; k < XPT; ++k) {
                const int idx = threadIdx.x + k * NW * 32;
                if (idx < XT) xs[xs_slot<MU, BT>(idx)] = xr[k];
            }
            named_bar_sync(1, NW * 32);
            if (sg + 1 < nseg) load_x(sg + 1);
            build_bank_owned_tables_smem<MU, NW, BT, LutGeom<BT>::KROW>(lut, xs, warp, lane);
            named_bar_sync(1, NW * 32);
            if (tl && sg == 0) g_timeline_c[blockIdx.x][2] = gtimer_c();
            int ti = warp / beta, ii = warp - (warp / beta) * beta;
            for (int c0 = 0; c0 < cps; c0 += NW, ++sc) {
                const int slot = sc % R;
                mbar_wait(&full[slot], (sc / R) & 1);
                if (tl && sc == 0) g_timeline_c[blockIdx.x][3] = gtimer_c();
                if (c0 + warp < cps && !(p.debug & 2048)) {
                    const unsigned char* kc = stages + slot * STAGE_BYTES + warp * 1024;
                    const uint4 ka = *reinterpret_cast<const uint4*>(kc + lane * 16);
                    const uint4 kb = *reinterpret_cast<const uint4*>(kc + 512 + lane * 16);
                    const uint32_t w[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
                    float o[BT];
                    gather_chunk<MU, BT, ABS>(w, lut_s, goff, o);
                    if (plan.dsm) {
                        float* dst = psum + (static_cast<long long>(ii) * nrl + ti * 32 + lane) * p.b + ct * BT;
#pragma unroll
                        for (int c = 0; c < BT; ++c)
                            if (ct * BT + c < p.b) dst[c] = first ? o[c] : dst[c] + o[c];
                    } else {
                        float* dst = p.partial +
                                     ((static_cast<long long>(rank) * beta + ii) * rows_pad + (T0 + ti) * 32 + lane) * p.b +
                                     static_cast<long long>(ct) * BT;
#pragma unroll
                        for (int c = 0; c < BT; ++c)
                            if (ct * BT + c < p.b) dst[c] = first ? o[c] : dst[c] + o[c];
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                ti += dq;
                ii += dr;
                if (ii >= beta) {
                    ii -= beta;
                    ++ti;
                }
            }
        }
        if (tl) g_timeline_c[blockIdx.x][4] = gtimer_c();
    }

    // -------------------------------------------- cluster-wide reduction
    cluster_sync_acqrel();
    if (tl) {
        g_timeline_c[blockIdx.x][6] = gtimer_c();
        if (p.debug & 1024) {
            const unsigned long long a = gtimer_c();
            const float v = p.alpha ? __ldg(p.alpha + (blockIdx.x * 64) % p.m) : 0.f;
            g_timeline_c[blockIdx.x][10] = gtimer_c() - a + (v == 1234.5f ? 1 : 0);
            const unsigned long long c2 = gtimer_c();
            const float v2 = __ldcg(p.partial + (blockIdx.x * 64) % p.m);
            g_timeline_c[blockIdx.x][11] = gtimer_c() - c2 + (v2 == 1234.5f ? 1 : 0);
        }
    }
    const int nrk = min(cs, p.NB);
    const long long pstride = rows_pad * p.b;                          // next plane
    const long long rstride = static_cast<long long>(beta) * pstride;  // next rank
    if (plan.dsm) {
        // Partials live in the shared memory of the cluster's CTAs: one
        // thread per output reads all beta x nrk of them through DSMEM plus
        // its beta alphas in one batch, then sums in a fixed order (ranks
        // ascending within a plane in fp64, planes ascending).
        const uint32_t ps = smem_u32(psum);
        for (long long o = o_lo + threadIdx.x; o < o_hi; o += blockDim.x) {
            const int rl = static_cast<int>(o / p.b);
            const int col = static_cast<int>(o - static_cast<long long>(rl) * p.b);
            const long long r = static_cast<long long>(T0) * 32 + rl;
            double y = 0.0;
            for (int i0 = 0; i0 < beta; i0 += 2) {
                const int i1 = min(i0 + 1, beta - 1);
                const uint32_t off0 = ps + static_cast<uint32_t>(((i0 * nrl + rl) * p.b + col) * 4);
                const uint32_t off1 = ps + static_cast<uint32_t>(((i1 * nrl + rl) * p.b + col) * 4);
                float v0[16], v1[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const uint32_t rk = static_cast<uint32_t>(min(k, nrk - 1));
                    v0[k] = ld_dsmem_f32(dsmem_map(off0, rk));
                    v1[k] = ld_dsmem_f32(dsmem_map(off1, rk));
                }
                const float a0 = p.alpha ? p.alpha[static_cast<long long>(i0) * p.m + r] : 1.0f;
                const float a1 = p.alpha ? p.alpha[static_cast<long long>(i1) * p.m + r] : 1.0f;
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    s0 += k < nrk ? static_cast<double>(v0[k]) : 0.0;
                    s1 += k < nrk ? static_cast<double>(v1[k]) : 0.0;
                }
                y += static_cast<double>(a0) * s0;
                if (i0 + 1 < beta) y += static_cast<double>(a1) * s1;
            }
            p.y[r * p.b + col] = static_cast<float>(y);
            if (tl && o == o_lo) g_timeline_c[blockIdx.x][7] = gtimer_c();
        }
        cluster_sync_relaxed();  // no CTA may exit while others read its shared memory
    } else {
    // One thread per output; its beta*nrk partials and beta alphas are
        // loaded in one batch (one L2 round trip; plain loads are safe after the
        // acquire above), then summed in a fixed order: ranks ascending within a
        // plane (fp64), planes ascending.  No branches between the loads, so they
        // all stay in flight together.
        for (long long o = o_lo + threadIdx.x; o < o_hi; o += blockDim.x) {
            const long long rr = o / p.b;
            const long long r = static_cast<long long>(T0) * 32 + rr;
            const long long col = o - rr * p.b;
            const float* src = p.partial + r * p.b + col;
            double y = 0.0;
            for (int i0 = 0; i0 < beta; i0 += 2) {
                const int i1 = min(i0 + 1, beta - 1);
                float v0[16], v1[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const long long kk = min(k, nrk - 1);
                    v0[k] = src[kk * rstride + i0 * pstride];
                    v1[k] = src[kk * rstride + i1 * pstride];
                }
                const float a0 = p.alpha ? p.alpha[static_cast<long long>(i0) * p.m + r] : 1.0f;
                const float a1 = p.alpha ? p.alpha[static_cast<long long>(i1) * p.m + r] : 1.0f;
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    s0 += k < nrk ? static_cast<double>(v0[k]) : 0.0;
                    s1 += k < nrk ? static_cast<double>(v1[k]) : 0.0;
                }
                y += static_cast<double>(a0) * s0;
                if (i0 + 1 < beta) y += static_cast<double>(a1) * s1;
            }
            p.y[r * p.b + col] = static_cast<float>(y);
            if (tl && o == o_lo) g_timeline_c[blockIdx.x][7] = gtimer_c();
        }
    }
    if (tl) g_timeline_c[blockIdx.x][5] = gtimer_c();
}

constexpr int kCNW = 15;  // consumer warps per CTA (+1 producer = 16 warps: 4 per SMSP, <= 128 regs)
constexpr int kCR = 4;    // pipeline stages (16 KiB each)

template <int MU, int BT>
size_t cluster_smem_bytes() {
    const size_t lut = static_cast<size_t>(1u << MU) * LutGeom<BT>::KROW * 4;
    const size_t stages = static_cast<size_t>(kCR) * kCNW * 1024 + 2 * kCR * sizeof(uint64_t);
    // BT <= 2 aligns the LUT to 64 KiB inside the allocation (<= 64 KiB - 1 slack)
    return (LutGeom<BT>::PRMT ? 65535 : 0) + lut + stages + kPSUM + xs_words(MU, BT) * 4;
}

template <int MU, int BT>
cudaError_t launch_cluster_mu_bt(const QueryParams& p, int cs, bool pdl, cudaStream_t stream, bool* used) {
    auto kern = biqgemm_cluster_kernel<MU, BT, kCNW, kCR>;
    const size_t smem = cluster_smem_bytes<MU, BT>();
    static PerDeviceOnce configured;
    static std::atomic<int> max_active[kMaxDevices][17];
    const int dev = current_device();
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3((kCNW + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t ea = once_per_device(configured, dev, [&] {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return e;
    });
    if (ea != cudaSuccess) return ea;
    int active = max_active[dev][cs].load(std::memory_order_relaxed);
    if (active == 0) {  // occupancy of this cluster size on this device (racing threads compute the same answer)
        int n = 0;
        cfg.gridDim = dim3(static_cast<unsigned>(cs));
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            n = -1;
        }
        active = n > 0 ? n : -1;
        max_active[dev][cs].store(active, std::memory_order_relaxed);
    }
    if (active < 1) {
        *used = false;
        return cudaSuccess;
    }
    ClusterPlan plan{};
    plan.cs = cs;
    plan.CT = (p.b + BT - 1) / BT;
    plan.nclusters = std::min(active, p.MT);
    plan.tq = p.MT / plan.nclusters;
    plan.tr = p.MT % plan.nclusters;
    {
        const long long nrl = static_cast<long long>(plan.tq + (plan.tr ? 1 : 0)) * 32;
        const long long need = (nrl * p.beta * p.b + static_cast<long long>(p.beta) * (nrl / cs + 2)) * 4;
        plan.dsm = (need <= kPSUM && cs <= 16) ? 1 : 0;
    }
    cfg.gridDim = dim3(static_cast<unsigned>(plan.nclusters * cs));
    *used = true;
    return cudaLaunchKernelEx(&cfg, kern, p, plan);
}

template <int MU>
cudaError_t launch_cluster_mu(const QueryParams& p, int cs, int bt, bool pdl, cudaStream_t s, bool* used) {
    if (bt == 1) return launch_cluster_mu_bt<MU, 1>(p, cs, pdl, s, used);
    if (bt == 2) return launch_cluster_mu_bt<MU, 2>(p, cs, pdl, s, used);
    return launch_cluster_mu_bt<MU, 4>(p, cs, pdl, s, used);
}

}  // namespace

cudaError_t launch_biqgemm_cluster(const QueryParams& p, int mu, bool pdl, cudaStream_t stream, bool* used) {
    const int cs = std::min(p.NB, 16);
    const int bt = p.b == 1 ? 1 : (p.b == 2 ? 2 : 4);
    *used = false;
    switch (mu) {
        case 1: return launch_cluster_mu<1>(p, cs, bt, pdl, stream, used);
        case 2: return launch_cluster_mu<2>(p, cs, bt, pdl, stream, used);
        case 3: return launch_cluster_mu<3>(p, cs, bt, pdl, stream, used);
        case 4: return launch_cluster_mu<4>(p, cs, bt, pdl, stream, used);
        case 5: return launch_cluster_mu<5>(p, cs, bt, pdl, stream, used);
        case 6: return launch_cluster_mu<6>(p, cs, bt, pdl, stream, used);
        case 7: return launch_cluster_mu<7>(p, cs, bt, pdl, stream, used);
        case 8: return launch_cluster_mu<8>(p, cs, bt, pdl, stream, used);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace bqg

extern "C" int bqg_debug_timeline_cluster(unsigned long long* out, int rows) {
    return cudaMemcpyFromSymbol(out, bqg::g_timeline_c,
                                sizeof(unsigned long long) * 16 * (rows < 8192 ? rows : 8192)) == cudaSuccess
               ? 0
               : 2;
}
