// kernels.h -- internal launcher declarations shared by the C-ABI layer.
//
// Device data layouts (all row-major unless stated):
//   W        m x n f32
//   planes   beta x m x ceil(n/32) u32 words, LSB-first, bit 1 = +1
//            (BinaryPlane, packing.hpp:16-57)
//   alpha    beta x m f32 (QuantizedLinear::alphas, quantize.hpp:16-22)
//   keys     beta x m x G, u8 for mu <= 8, u16 for mu > 8, pad bits 0
//            (KeyMatrix, packing.hpp:61-73; the BQGM on-disk key payload,
//            model_io.cpp:77-87)
//   tiled    (mu <= 8) 1 KiB chunks, chunk(gb, t, i) at ((gb*MT + t)*beta + i)
//            KiB, NB = ceil(G/32), MT = ceil(m/32): group block gb, row tile
//            t, plane i.  Inside a chunk, lane l (row t*32 + l) owns the
//            16-byte pieces at l*16 and 512 + l*16; its byte j (piece j>>4,
//            byte j&15) is the key of group gb*32 + ((l + j) mod 32).  A CTA's
//            chunk range is one contiguous byte range (one TMA bulk copy per
//            pipeline stage); a warp's 16-byte shared-memory reads are
//            conflict-free; the rotation makes lane l read bank (l+j) mod 32
//            at step j, so the LUT gather never conflicts.
//   x        x_rows x b f32 (x_rows <= G*mu; missing rows are zero)
//   y        m x b f32
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bqg {

constexpr int kStreamMaxGroup = 512;  // calls per launch (kernel-parameter array, 16 KiB)
// EVERY fast-path workspace starts with one completion counter per call of a
// grouped launch (zero between launches: the texture form resets what it
// uses); every form's partial sums start after them, so forms that share a
// workspace (a layer handle's, the grouped host pipeline's) never clobber the
// counters.
constexpr size_t kTexCounterBytes = kStreamMaxGroup * sizeof(unsigned);
// Zero the counters of a workspace the library has not seen before (on
// `stream`; a graph node under capture) -- a safety net behind the C ABI's
// zero-at-allocation rule.
cudaError_t zero_counters_once(void* ws, int dev, cudaStream_t stream);

// Fused all-gather (biqgemm_tex.cu's finaliser, the two-kernel form's
// finalize_kernel): every y row is also stored at the same offset from a
// local base in each of up to kMaxPeers peer gather buffers.
constexpr int kMaxPeers = 8;

struct QueryParams {
    const uint8_t* keys;    // tiled
    const float* alpha;     // beta x m or nullptr (plane mode: alpha = 1)
    const float* x;         // x_rows x b
    float* y;               // m x b
    float* ws;              // workspace base: kTexCounterBytes of completion counters (grouped/texture forms)
    float* partial;         // = ws + kTexCounterBytes: partial sums (layout per form)
    long long x_rows;
    int m, G, NB, MT, beta, b, cpb;
    int bt;     // fast form: input columns per column tile (1, 2 or 4)
    int debug;  // profiling switches (BQG_DEBUG_FLAGS); 0 in production
    // two-kernel form only: y(r, c) is also stored at peer_y[k] + (&y(r, c) - peer_local)
    int npeer;
    const float* peer_local;
    float* peer_y[kMaxPeers];
};

// Grouped ("stream") form: a group of independent calls sharing (m, n, beta,
// mu); b == 1, mu == 8, beta <= 4 (biqgemm_stream.cu).
struct StreamCall {
    const uint8_t* keys;  // tiled
    const float* alpha;   // beta x m or nullptr
    const float* x;       // x_rows x 1
    float* y;             // m x 1
};
bool stream_supported(int mu, int beta, long long b);
size_t stream_workspace_bytes(long long m, long long groups, int count);
cudaError_t launch_biqgemm_stream(const StreamCall* calls, int count, long long x_rows, int m, int G, int beta,
                                  float* ws, bool pdl, cudaStream_t stream);
// The same grouped computation with the keys fetched through the texture
// pipe (biqgemm_tex.cu); launch_biqgemm_stream dispatches to it when
// tex_stream_applies (texel range) unless BQG_STREAM_IMPL=tma.
bool tex_stream_applies(long long m, int G, int beta);
#ifndef BQG_TEX_MIN_GROUP
#define BQG_TEX_MIN_GROUP 4
#endif
constexpr int kTexMinGroup = BQG_TEX_MIN_GROUP;  // smaller groups take the TMA-ring form
// The group size from which the texture form beats the TMA-ring form for
// m rows (>= kTexMinGroup; measured crossovers, tools/ab_tex_min_group3.sh).
int tex_min_group(long long m);
// peer_base / npeer (<= kMaxPeers): the finaliser also stores every y row at
// the same offset from local_base in each peer gather buffer (fused
// all-gather over NVLink; npeer = 0: local y only).
cudaError_t launch_biqgemm_tex(const StreamCall* calls, int count, long long x_rows, int m, int G, int beta,
                               float* ws, bool pdl, cudaStream_t stream, const float* local_base = nullptr,
                               float* const* peer_base = nullptr, int npeer = 0);

// Single-call latency form (biqgemm_latency.cu): b == 1, mu == 8, beta <= 4,
// NB in {1,2,4,8,16}; one kernel, in-cluster push reduction.  *used = false
// when the shape does not fit (caller falls back).
bool latency_supported(int mu, int beta, long long b, int NB);
cudaError_t launch_biqgemm_latency(const QueryParams& p, bool pdl, cudaStream_t stream, bool* used);
bool latency_applies(const QueryParams& p);
// Which single-call form launch_biqgemm_fast picks: 1 latency, 2 cluster, 3 two-kernel,
// 4 stream form with a group of one.
int fast_form(const QueryParams& p, int mu);

// Comparison baselines (baselines.cu; reference baselines.hpp:40-87).
cudaError_t launch_gemm_unpack(const uint32_t* planes, const float* alpha, const float* x, long long x_rows, float* y,
                               long long m, long long n, int b, int beta, cudaStream_t stream);
cudaError_t launch_bandwidth_probe(const uint32_t* words, long long m, long long n, const float* x, long long x_rows,
                                   float* out, bool streaming, cudaStream_t stream);

// Workspace for the fast path (bytes).
size_t fast_workspace_bytes(long long m, long long groups, int beta, long long b);
// Grid planner: CTAs per 32-group block.
int plan_cpb(long long m, long long groups, int beta, long long b, int num_sms);

template <typename T>
cudaError_t launch_quantize_greedy(const T* w, long long m, long long n, int beta,
                                   uint32_t* planes, T* alpha, double* alpha_d,
                                   cudaStream_t stream);
cudaError_t launch_pack_keys(const uint32_t* plane, long long m, long long n, int mu, void* keys,
                             cudaStream_t stream);
// keys (rows x groups, mu-bit, u8 / u16) -> the same sign bits as mu = 8 keys
// (rows x groups8 bytes, groups8 >= ceil(groups*mu / 8)); rows = beta*m.
cudaError_t launch_rekey_mu8(const void* keys, long long rows, long long groups, int mu, long long groups8,
                             uint8_t* out, cudaStream_t stream);
cudaError_t launch_tile_keys(const uint8_t* keys, long long m, long long groups, int beta,
                             uint8_t* tiled, cudaStream_t stream);

// Fast path (mu <= 8): fused LUT build -> query -> alpha epilogue.
// Tries the single-kernel cluster form first, else two PDL-chained kernels.
cudaError_t launch_biqgemm_fast(const QueryParams& p, int mu, bool pdl, cudaStream_t stream);
// The two-kernel form (form 3) directly, whatever fast_form would pick: the
// row-sharded entries use it for every shard so y is bitwise the same for any
// shard count, and its finaliser honours p.npeer / p.peer_y.
bool twokernel_supported(int mu, int beta, long long b);
cudaError_t launch_biqgemm_twokernel(const QueryParams& p, int mu, bool pdl, cudaStream_t stream);
// Single-kernel form with an in-cluster reduction; *used = false when the
// device cannot co-schedule the cluster (caller falls back).
cudaError_t launch_biqgemm_cluster(const QueryParams& p, int mu, bool pdl, cudaStream_t stream, bool* used);

// Fast-path LUT builder exposed for parity (same device code as the fused kernel).
cudaError_t launch_build_lut_f32(const float* x, long long x_rows, long long b, int mu,
                                 long long g0, long long count, bool key_major, float* out,
                                 cudaStream_t stream);

// Exact path (any mu in 1..16, any b): fp64 LUT (global memory), fp64
// accumulation in the reference's order -> bit-identical to
// biqgemm::detail::run (kernel.hpp:116-204).  T is float or double.
template <typename T>
cudaError_t launch_build_lut_exact(const T* x, long long x_rows, long long b, int mu, long long g0,
                                   long long count, bool key_major, double* out,
                                   cudaStream_t stream, bool naive = false);
// Phase marks for KernelStats (kernel.hpp:41-46,156-159): mark(ctx, phase)
// is called on the host right before the launches of each phase are queued
// (phase 0 = a tile's LUT build, 1 = its query, 2 = the alpha epilogue), so
// the caller can record an event on the stream there.
struct PhaseMarks {
    void* ctx;
    void (*mark)(void* ctx, int phase, cudaStream_t stream);
};
template <typename T>
cudaError_t launch_biqgemm_exact(const void* keys_rowmajor, const T* alpha, const T* x,
                                 long long x_rows, T* y, long long m, long long n, int beta,
                                 int mu, long long b, void* workspace, size_t workspace_bytes,
                                 cudaStream_t stream, bool naive = false,
                                 const PhaseMarks* marks = nullptr);
size_t exact_workspace_bytes(long long m, long long n, int beta, int mu, long long b);

}  // namespace bqg
