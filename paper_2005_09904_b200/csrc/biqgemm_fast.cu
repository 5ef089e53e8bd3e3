// biqgemm_fast.cu -- the fused BiQGEMM hot path for mu <= 8 (fp32 LUT).
//
// Replaces biqgemm::detail::run + query_rows + the alpha epilogue
// (/root/reference/proj/core/include/biqgemm/kernel.hpp:83-108,116-204) and
// build_lut_block (lut.hpp:109-154) with ONE kernel:
//
//   prologue   : each warp issues 128-bit evict-first loads for its first D
//                work units of packed keys (keys never depend on the previous
//                kernel, so this runs before griddepcontrol.wait and overlaps
//                the predecessor's tail under PDL);
//   LUT build  : after griddepcontrol.wait, the CTA builds the tables of its
//                32-group block (x BT input columns) in bank-owned shared
//                memory with the DP recurrence (lut_build.cuh);
//   query      : per unit (plane i, row tile, group block) lane l gathers
//                T_{gb*32+l}[key] for 32 (BT=1) or 16 (BT>1) rows from its own
//                bank -- conflict-free, one wavefront per warp gather -- then a
//                swizzled butterfly (31 SHFL+FADD per 1024 lookups) sums the
//                32 groups per row;
//   epilogue   : the per-(block, plane) partial goes to a workspace; the warp
//                that completes the last unit of a 32-row tile (atomic ticket)
//                reduces the tile in a FIXED order -- fp64 over group blocks
//                ascending, then y = sum_i alpha_i * acc_i in fp64 over planes
//                ascending (kernel.hpp:183-195) -- and resets the ticket.
//
// The reduction tree of every output is a function of (n, mu) only, so y is
// bitwise identical for every grid shape, CTA split and row sharding.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "lut_build.cuh"

namespace bqg {

namespace {

struct FastPlan {
    long long upp;    // units per (group block, column tile) pair
    long long total;  // total units
    int CT;           // column tiles
    int H;            // units per (tile, plane): 1 for BT=1 (32 rows), 2 otherwise (16 rows)
    int mode;         // 0 = aligned (cpb CTAs per pair), 1 = flat contiguous split
    int cpb;
    int grid;
};

// Byte offset of key byte `bi` of word w in the bank-owned LUT, OR'd with the
// lane's column offset.  BT=1: word = k*32 + l  -> byte k<<7 | l<<2.
template <int MU, int BT>
__device__ __forceinline__ uint32_t lut_off(uint32_t w, int bi, uint32_t lane_off) {
    constexpr int SH = (BT == 1) ? 7 : (BT == 2 ? 8 : 9);
    constexpr uint32_t MASK = ((1u << MU) - 1u) << SH;
    const int s = 8 * bi - SH;  // compile-time after unrolling
    const uint32_t v = s >= 0 ? (w >> s) : (w << (-s));
    return (v & MASK) | lane_off;
}

// One unit of keys for this lane: 32 bytes (BT=1) or 16 bytes (BT>1).
template <int KPU>
__device__ __forceinline__ void load_keys(uint32_t (&w)[4 * KPU], const uint8_t* a, uint64_t pol) {
    if constexpr (KPU == 2) {
        const U8x32 v = ld_stream_u8x32(a);
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = v.w[q];
    } else {
        const uint4 v = ld_stream_u4(a, pol);
        w[0] = v.x;
        w[1] = v.y;
        w[2] = v.z;
        w[3] = v.w;
    }
}

template <int MU, int BT, int NW, int D>
__global__ void __launch_bounds__(NW * 32, BT == 1 ? 2 : 1)
    biqgemm_fast_kernel(const QueryParams p, const FastPlan plan) {
    extern __shared__ __align__(16) float lut[];
    constexpr int KPU = (BT == 1) ? 2 : 1;  // uint4 of keys per lane per unit
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    pdl_launch_dependents();

    long long ubeg, uend;
    if (plan.mode == 0) {
        const long long pair = blockIdx.x / plan.cpb, c = blockIdx.x % plan.cpb;
        ubeg = pair * plan.upp + plan.upp * c / plan.cpb;
        uend = pair * plan.upp + plan.upp * (c + 1) / plan.cpb;
    } else {
        ubeg = plan.total * blockIdx.x / plan.grid;
        uend = plan.total * (blockIdx.x + 1) / plan.grid;
    }

    const int beta = p.beta, H = plan.H;
    const long long MT = p.MT, rows_pad = MT * 32;
    const uint32_t lane_off = static_cast<uint32_t>(lane) * 4u * BT;
    const char* lutc = reinterpret_cast<const char*>(lut);
    const uint64_t pol = policy_evict_first();
    bool waited = false;

    for (long long seg = ubeg; seg < uend;) {
        const long long pair = seg / plan.upp;
        const long long seg_end = min(uend, (pair + 1) * plan.upp);
        const int gb = static_cast<int>(pair / plan.CT), ct = static_cast<int>(pair % plan.CT);
        const long long base_local = pair * plan.upp;

        // Address of this lane's keys for unit u (global index).
        auto key_addr = [&](long long u) -> const uint8_t* {
            const long long local = u - base_local;
            const long long t = local / (static_cast<long long>(beta) * H);
            const int rem = static_cast<int>(local - t * beta * H);
            const int i = rem / H, h = rem - (rem / H) * H;
            const uint8_t* chunk =
                p.keys + ((((static_cast<long long>(gb) * beta + i) * MT + t) * 32 + lane) * 32);
            if (BT == 1) return chunk;
            return chunk + 16 * (h ^ (lane >> 4));
        };

        uint32_t kr[D][4 * KPU];
#pragma unroll
        for (int s = 0; s < D; ++s) {
            const long long u = seg + warp + static_cast<long long>(s) * NW;
            if (u < seg_end) load_keys<KPU>(kr[s], key_addr(u), pol);
        }
        if (!waited) {
            pdl_wait();
            waited = true;
        }
        __syncthreads();  // previous segment's gathers are done with the LUT
        build_bank_owned_tables<MU, NW, BT>(lut, p.x, p.x_rows, p.b,
                                            static_cast<long long>(gb) * 32 + lane,
                                            static_cast<long long>(ct) * BT, warp, lane);
        __syncthreads();

        for (long long ub = seg + warp; ub < seg_end; ub += static_cast<long long>(D) * NW) {
#pragma unroll
            for (int s = 0; s < D; ++s) {
                const long long u = ub + static_cast<long long>(s) * NW;
                if (u >= seg_end) break;
                uint32_t w[4 * KPU];
#pragma unroll
                for (int q = 0; q < 4 * KPU; ++q) w[q] = kr[s][q];
                {
                    const long long un = u + static_cast<long long>(D) * NW;
                    if (un < seg_end) load_keys<KPU>(kr[s], key_addr(un), pol);
                }
                const long long local = u - base_local;
                const long long t = local / (static_cast<long long>(beta) * H);
                const int rem = static_cast<int>(local - t * beta * H);
                const int i = rem / H, h = rem - (rem / H) * H;

                if constexpr (BT == 1) {
                    float v[32];
#pragma unroll
                    for (int wi = 0; wi < 8; ++wi) {
#pragma unroll
                        for (int bi = 0; bi < 4; ++bi) {
                            const uint32_t off = lut_off<MU, 1>(w[wi], bi, lane_off);
                            v[wi * 4 + bi] = *reinterpret_cast<const float*>(lutc + off);
                        }
                    }
                    // swizzled butterfly: slot s holds row s ^ lane
#pragma unroll
                    for (int hw = 16; hw >= 1; hw >>= 1) {
#pragma unroll
                        for (int s2 = 0; s2 < hw; ++s2)
                            v[s2] += __shfl_xor_sync(0xffffffffu, v[s2 + hw], hw);
                    }
                    const long long r = t * 32 + lane;
                    p.partial[(static_cast<long long>(gb) * beta + i) * rows_pad + r] = v[0];
                } else {
                    float v[16][BT];
#pragma unroll
                    for (int wi = 0; wi < 4; ++wi) {
#pragma unroll
                        for (int bi = 0; bi < 4; ++bi) {
                            const uint32_t off = lut_off<MU, BT>(w[wi], bi, lane_off);
                            if constexpr (BT == 2) {
                                const float2 e = *reinterpret_cast<const float2*>(lutc + off);
                                v[wi * 4 + bi][0] = e.x;
                                v[wi * 4 + bi][1] = e.y;
                            } else {
                                const float4 e = *reinterpret_cast<const float4*>(lutc + off);
                                v[wi * 4 + bi][0] = e.x;
                                v[wi * 4 + bi][1] = e.y;
                                v[wi * 4 + bi][2] = e.z;
                                v[wi * 4 + bi][3] = e.w;
                            }
                        }
                    }
                    // slot s holds row 16h + (s ^ (lane & 15))
#pragma unroll
                    for (int hw = 8; hw >= 1; hw >>= 1) {
#pragma unroll
                        for (int s2 = 0; s2 < hw; ++s2) {
#pragma unroll
                            for (int c = 0; c < BT; ++c)
                                v[s2][c] += __shfl_xor_sync(0xffffffffu, v[s2 + hw][c], hw);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < BT; ++c) v[0][c] += __shfl_xor_sync(0xffffffffu, v[0][c], 16);
                    if (lane < 16) {
                        const long long r = t * 32 + 16 * h + lane;
                        float* dst = p.partial +
                                     ((static_cast<long long>(gb) * beta + i) * rows_pad + r) * p.b +
                                     static_cast<long long>(ct) * BT;
#pragma unroll
                        for (int c = 0; c < BT; ++c) {
                            if (ct * BT + c < p.b) dst[c] = v[0][c];
                        }
                    }
                }

                // ---- completion ticket for (tile t, column tile ct) ----
                __threadfence();
                __syncwarp();
                unsigned ticket = 0;
                unsigned* ctr = p.counters + t * plan.CT + ct;
                if (lane == 0) ticket = atomicAdd(ctr, 1u);
                ticket = __shfl_sync(0xffffffffu, ticket, 0);
                const unsigned expect = static_cast<unsigned>(p.NB) * beta * H;
                if (ticket == expect - 1) {
                    __threadfence();
                    const long long r = t * 32 + lane;
                    if (r < p.m) {
                        for (int c = 0; c < BT; ++c) {
                            const long long col = static_cast<long long>(ct) * BT + c;
                            if (col >= p.b) break;
                            double y = 0.0;
                            for (int pi = 0; pi < beta; ++pi) {
                                double acc = 0.0;
                                for (int g2 = 0; g2 < p.NB; ++g2) {
                                    acc += static_cast<double>(ld_cg_f32(
                                        p.partial +
                                        ((static_cast<long long>(g2) * beta + pi) * rows_pad + r) * p.b +
                                        col));
                                }
                                const double a =
                                    p.alpha ? static_cast<double>(p.alpha[static_cast<long long>(pi) * p.m + r])
                                            : 1.0;
                                y += a * acc;
                            }
                            p.y[r * p.b + col] = static_cast<float>(y);
                        }
                    }
                    if (lane == 0) *ctr = 0u;
                }
            }
        }
        seg = seg_end;
    }
    if (!waited) pdl_wait();
}

template <int MU, int BT>
cudaError_t launch_mu_bt(const QueryParams& p, const FastPlan& plan, bool pdl, cudaStream_t stream) {
    constexpr int NW = 8, D = 4;
    auto kern = biqgemm_fast_kernel<MU, BT, NW, D>;
    const size_t smem = static_cast<size_t>(1u << MU) * 32 * BT * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(plan.grid));
    cfg.blockDim = dim3(NW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p, plan);
}

template <int MU>
cudaError_t launch_mu(const QueryParams& p, const FastPlan& plan, int bt, bool pdl, cudaStream_t s) {
    if (bt == 1) return launch_mu_bt<MU, 1>(p, plan, pdl, s);
    if (bt == 2) return launch_mu_bt<MU, 2>(p, plan, pdl, s);
    return launch_mu_bt<MU, 4>(p, plan, pdl, s);
}

int pick_bt(long long b) { return b == 1 ? 1 : (b == 2 ? 2 : 4); }

FastPlan make_plan(long long m, long long groups, int beta, long long b, int mu, int num_sms) {
    const int BT = pick_bt(b);
    FastPlan pl{};
    const long long NB = (groups + 31) / 32, MT = (m + 31) / 32;
    pl.CT = static_cast<int>((b + BT - 1) / BT);
    pl.H = BT == 1 ? 1 : 2;
    pl.upp = MT * beta * pl.H;
    const long long pairs = NB * pl.CT;
    pl.total = pairs * pl.upp;
    // Cost model in shared-memory wavefronts (the binding resource):
    // building one block of tables = 2^mu * BT wavefronts; one unit =
    // 32 (BT<=2) or 64 (BT=4) gather wavefronts.
    const double build = static_cast<double>(1 << mu) * BT + 64.0;
    const double unit = BT == 4 ? 64.0 : 32.0;
    const long long sms = std::max(1, num_sms);
    // aligned: cpb CTAs per pair
    long long best_cpb = 1;
    double best_aligned = 1e300;
    for (long long cpb = 1; cpb <= std::max<long long>(1, std::min<long long>(pl.upp, 4 * sms)); ++cpb) {
        const long long grid = pairs * cpb;
        const long long waves = (grid + sms - 1) / sms;
        const double t = static_cast<double>(waves) *
                         (build + static_cast<double>((pl.upp + cpb - 1) / cpb) * unit);
        if (t < best_aligned - 1e-9) {
            best_aligned = t;
            best_cpb = cpb;
        }
    }
    // flat: one CTA per SM, contiguous chunks (may span several pairs)
    const long long fgrid = std::min<long long>(sms, pl.total);
    const long long chunk = (pl.total + fgrid - 1) / fgrid;
    const long long spans = std::min<long long>(pairs, (chunk + pl.upp - 1) / pl.upp + 1);
    const double t_flat = static_cast<double>(spans) * build + static_cast<double>(chunk) * unit;
    if (t_flat < best_aligned) {
        pl.mode = 1;
        pl.cpb = 1;
        pl.grid = static_cast<int>(fgrid);
    } else {
        pl.mode = 0;
        pl.cpb = static_cast<int>(best_cpb);
        pl.grid = static_cast<int>(pairs * best_cpb);
    }
    return pl;
}

}  // namespace

size_t fast_workspace_bytes(long long m, long long groups, int beta, long long b) {
    const long long NB = (groups + 31) / 32, MT = (m + 31) / 32;
    const int BT = pick_bt(b);
    const long long CT = (b + BT - 1) / BT;
    const size_t partial = static_cast<size_t>(NB) * beta * MT * 32 * b * sizeof(float);
    const size_t counters = static_cast<size_t>(MT * CT) * sizeof(unsigned);
    return ((counters + 255) / 256) * 256 + partial;
}

int plan_cpb(long long m, long long groups, int beta, long long b, int num_sms) {
    return make_plan(m, groups, beta, b, 8, num_sms).cpb;
}

cudaError_t launch_biqgemm_fast(const QueryParams& p, int mu, bool pdl, cudaStream_t stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const FastPlan plan = make_plan(p.m, p.G, p.beta, p.b, mu, sms);
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
        const long long o = key_major ? base + static_cast<long long>(k) * b + col
                                      : base + col * TABLE + k;
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
