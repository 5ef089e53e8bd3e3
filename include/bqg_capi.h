/*
 * bqg_capi.h -- C ABI of the B200-native BiQGEMM library (libbiqgemm_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/core/include/biqgemm/, "proj/core"): every entry point
 * below replaces one reference function, cited as file:line.  The C++ host
 * library in include/biqgemm_b200/ re-presents the reference's C++ API
 * (Matrix, BinaryPlane, KeyMatrix, PackedLinear, biqgemm, ...) on top of
 * these calls; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "d_" pointers are device memory,
 *     "h_" pointers are host memory.  All matrices are row-major.
 *   - Device entry points are stream-ordered and asynchronous; `stream` is a
 *     cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every function returns a bqg_status; nothing throws across the ABI.
 *     bqg_last_error_message() gives the per-thread detail text.  The C++
 *     wrapper maps BQG_ERR_INVALID_ARGUMENT to std::invalid_argument and the
 *     format codes to the reference's FormatError hierarchy
 *     (model_io.hpp:14-32), exactly like the reference throws.
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point returns BQG_ERR_NO_DEVICE.
 *
 * Data layouts: see paper_2005_09904_b200/csrc/kernels.h and DESIGN.md.
 */
#ifndef BQG_CAPI_H
#define BQG_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BQG_ABI_VERSION 1

typedef enum bqg_status {
    BQG_OK = 0,
    BQG_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    BQG_ERR_CUDA = 2,             /* a CUDA runtime call failed */
    BQG_ERR_NO_DEVICE = 3,        /* no usable CUDA device (no CPU fallback) */
    BQG_ERR_OUT_OF_MEMORY = 4,
    BQG_ERR_FORMAT = 5,           /* reference: FormatError (model_io.hpp:14) */
    BQG_ERR_BAD_MAGIC = 6,        /* reference: BadMagicError (model_io.hpp:18) */
    BQG_ERR_BAD_VERSION = 7,      /* reference: BadVersionError (model_io.hpp:22) */
    BQG_ERR_TRUNCATED = 8,        /* reference: TruncatedError (model_io.hpp:26) */
    BQG_ERR_RANGE = 9,            /* reference: RangeError (model_io.hpp:30) */
    BQG_ERR_IO = 10,              /* reference: std::runtime_error (model_io.cpp:169,175) */
    BQG_ERR_WORKSPACE = 11,       /* workspace too small */
    BQG_ERR_COMM = 12             /* a collective failed or NCCL is unavailable */
} bqg_status;

/* LutLayout (lut.hpp:71) and LutBuilder (lut.hpp:73). */
enum { BQG_LUT_TABLE_MAJOR = 0, BQG_LUT_KEY_MAJOR = 1 };
enum { BQG_LUT_DP = 0, BQG_LUT_NAIVE = 1 };
/* forward path selector (the `exact` argument of the layer entry points) */
enum { BQG_FORWARD_FAST = 0, BQG_FORWARD_EXACT = 1, BQG_FORWARD_EXACT_NAIVE = 2 };

const char* bqg_status_string(int status);
const char* bqg_last_error_message(void);
int bqg_abi_version(void);

/* ---------------------------------------------------------------- host-only
 * (no GPU needed) */

/* Matrix<float>::random_uniform / random_normal (matrix.hpp:63-79): libstdc++
 * mt19937_64 + uniform_real_distribution<float>(lo, hi) /
 * normal_distribution<float>(0, 1), row-major fill of rows*cols values. */
int bqg_random_uniform_f32(float* h_out, size_t rows, size_t cols, uint64_t seed, float lo, float hi);
int bqg_random_normal_f32(float* h_out, size_t rows, size_t cols, uint64_t seed);
int bqg_random_uniform_f64(double* h_out, size_t rows, size_t cols, uint64_t seed, double lo, double hi);
int bqg_random_normal_f64(double* h_out, size_t rows, size_t cols, uint64_t seed);

/* plan_tiles (kernel.hpp:58-70).  On the GPU the TileShape does not change the
 * result or the launch (the device planner sizes its own work units); it is
 * kept for API fidelity and validated like the reference does. */
int bqg_plan_tiles(size_t m, size_t groups, size_t b, unsigned mu, size_t budget_bytes,
                   size_t entry_bytes, size_t* t_w, size_t* t_h);

/* footprint (model_io.cpp:182-194): out[0..3] = weight, activation, output,
 * alpha bytes. */
int bqg_footprint(uint64_t m, uint64_t n, unsigned weight_bits, uint64_t batch,
                  unsigned activation_bits, unsigned output_bits, uint64_t* out4);

/* Exact op counters (kernel.hpp:23-36, laws at 179-180 and lut.hpp:62-68):
 * out[0] lut_build_ops = (2^mu + mu - 1)*G*b (DP) or 2^mu*mu*G*b (naive),
 * out[1] lookups = out[2] accumulate_ops = m*G*b*beta, out[3] fma_ops = 0. */
int bqg_op_counters(size_t m, size_t n, size_t b, unsigned beta, unsigned mu, int builder,
                    uint64_t* out4);

/* Bytes of the tiled device key layout for beta planes (mu <= 8). */
size_t bqg_tiled_key_bytes(size_t m, size_t n, unsigned beta, unsigned mu);

/* BQGM model file (model_io.cpp:65-141, format README.md:88-108), host side.
 * bqg_bqgm_parse validates exactly like load() (magic, version, dims, mu,
 * per-plane alpha + keys with range check, no trailing bytes) and reports the
 * header; with non-NULL outputs it also copies alpha (beta x m f32) and keys
 * (beta x m x G, u8 if mu <= 8 else u16, i.e. the file's own payload). */
int bqg_bqgm_parse(const uint8_t* h_bytes, size_t len, size_t* m, size_t* n, unsigned* beta,
                   unsigned* mu, float* h_alpha, void* h_keys);
/* save() from packed keys (rowmajor u8/u16 as above) and alpha. *len is the
 * buffer size on entry and the file size on return; h_out may be NULL. */
int bqg_bqgm_serialize(const void* h_keys, const float* h_alpha, size_t m, size_t n, unsigned beta,
                       unsigned mu, uint8_t* h_out, size_t* len);

/* ----------------------------------------------------------- device primitives */

/* quantize_greedy<float> (quantize.hpp:27-58), bit-exact.
 * d_w: m x n f32.  d_planes: beta x m x ceil(n/32) u32 (BinaryPlane words).
 * d_alpha: beta x m f32.  Uses a temporary fp64 buffer of beta*m doubles. */
int bqg_quantize_greedy_f32(const float* d_w, size_t m, size_t n, unsigned beta,
                            uint32_t* d_planes, float* d_alpha, void* stream);
/* quantize_greedy<double>: same algorithm, double W, double alpha. */
int bqg_quantize_greedy_f64(const double* d_w, size_t m, size_t n, unsigned beta,
                            uint32_t* d_planes, double* d_alpha, void* stream);

/* pack_keys (packing.hpp:84-107), bit-exact, for one plane.
 * d_plane: m x ceil(n/32) words.  d_keys: m x G, u8 (mu <= 8) or u16. */
int bqg_pack_keys(const uint32_t* d_plane, size_t m, size_t n, unsigned mu, void* d_keys,
                  void* stream);

/* Row-major u8 keys of beta planes (beta x m x G) -> the fast path's tiled
 * layout (bqg_tiled_key_bytes bytes).  mu <= 8 only. */
int bqg_tile_keys(const uint8_t* d_keys, size_t m, size_t n, unsigned beta, unsigned mu,
                  uint8_t* d_tiled, void* stream);

/* mu != 8 on the fast path: the sign bits of mu-bit keys (beta x m x G, u16
 * for mu > 8, u8 otherwise) re-keyed as mu = 8 keys over
 * bqg_rekey_mu8_columns(n, mu) = 8*ceil(G*mu/8) columns (beta x m x that/8
 * bytes, row-major; bits past G*mu are 0, like the keys' own pad bits).
 * y = sum_i alpha_i * W_i x does not depend on the grouping, so these keys
 * (then bqg_tile_keys with mu = 8 and n = that column count) run the mu <= 8
 * kernels -- fp32 tables, within the fast path's contract of the reference's
 * mu result; the exact path keeps the mu-bit keys and stays bit-identical.
 * The key stream shrinks too: 1 bit per weight instead of 16/mu. */
size_t bqg_rekey_mu8_columns(size_t n, unsigned mu);
int bqg_rekey_mu8(const void* d_keys, size_t m, size_t n, unsigned beta, unsigned mu, uint8_t* d_keys8,
                  void* stream);

/* build_lut_block (lut.hpp:109-154) for groups [g0, g0+count) of x
 * (x_rows x b), in the reference's LutBlock layout (lut.hpp:90-97).
 *   _f32: the fast path's bank-owned shared-memory builder (mu <= 8),
 *         fp32, DP order; bit-exact with the DP evaluated in fp32.
 *   _f64: the exact path's builder, fp64, bit-exact with the reference;
 *         builder BQG_LUT_DP (lut.hpp:50-69) or BQG_LUT_NAIVE (lut.hpp:31-43).
 *   _f64x: as _f64 for a double x (Matrix<double>).
 * The _f32 builder is DP only.
 * *ops (may be NULL) receives the reference's counted ops. */
int bqg_build_lut_f32(const float* d_x, size_t x_rows, size_t b, unsigned mu, size_t g0,
                      size_t count, int layout, int builder, float* d_entries, uint64_t* ops,
                      void* stream);
int bqg_build_lut_f64(const float* d_x, size_t x_rows, size_t b, unsigned mu, size_t g0,
                      size_t count, int layout, int builder, double* d_entries, uint64_t* ops,
                      void* stream);
int bqg_build_lut_f64x(const double* d_x, size_t x_rows, size_t b, unsigned mu, size_t g0,
                       size_t count, int layout, int builder, double* d_entries, uint64_t* ops,
                       void* stream);

typedef struct bqg_kernel_stats {
    /* OpCounters (kernel.hpp:23-36), exact, computed analytically with the
     * builder's law (Dp: 2^mu + mu - 1, Naive: 2^mu * mu per table) */
    uint64_t lut_build_ops, lookups, accumulate_ops, fma_ops;
    /* KernelStats phase seconds (kernel.hpp:41-46), CUDA-event timed.
     * Exact path: build = the LUT kernels, query = the lookup kernels,
     * replace = setup + alpha epilogue + H2D of x + D2H of y.  Fast path: the
     * LUT build runs INSIDE the query kernel (builder warps overlap the
     * gather), so build_seconds stays 0 and query_seconds is that kernel. */
    double build_seconds, query_seconds, replace_seconds;
} bqg_kernel_stats;

/* The BiQGEMM multiply, biqgemm (kernel.hpp:246-258) / biqgemm_plane
 * (kernel.hpp:209-215 when d_alpha == NULL, alpha = 1):
 *     y(r, c) = sum_i alpha_i[r] * sum_g LUT_g,c[key_i(r, g)]
 * Fast path (mu <= 8): d_keys is the TILED layout (bqg_tile_keys); fused
 *   LUT build -> query -> alpha epilogue; fp32 LUT, fp32 group sums, fp64
 *   cross-block/plane epilogue.  Deterministic and grid-invariant.
 *   Workspace: bqg_biqgemm_workspace_bytes() bytes (per-block partial sums;
 *   no initialisation needed).  Two kernels are launched (fused LUT
 *   build/query, then the fixed-order epilogue), chained with programmatic
 *   dependent launch.  pdl != 0 also launches the first one with
 *   programmatic stream serialization (overlaps the predecessor's tail).
 * x_rows <= G*mu (rows beyond x_rows are zero; kernel.hpp:132-134). */
size_t bqg_biqgemm_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu);
int bqg_biqgemm_f32(const uint8_t* d_keys_tiled, const float* d_alpha, const float* d_x,
                    size_t x_rows, float* d_y, size_t m, size_t n, size_t b, unsigned beta,
                    unsigned mu, void* d_workspace, size_t workspace_bytes, int pdl, void* stream);

/* Which single-call kernel form bqg_biqgemm_f32 uses for this shape on the
 * current device: 1 = latency form (b == 1, mu == 8, beta <= 4, n <= 4096:
 * one kernel, in-cluster push reduction, y bitwise equal to the grouped
 * form), 2 = cluster form, 3 = two-kernel form, 4 = the grouped stream form
 * with a group of one (b == 1, mu == 8, beta <= 4 shapes outside forms 1-2,
 * e.g. large m; y bitwise equal to the grouped form); 0 = no fast path. */
int bqg_biqgemm_form(size_t m, size_t n, size_t b, unsigned beta, unsigned mu);

/* Grouped calls: `count` independent biqgemm calls (kernel.hpp:246-258, one
 * per entry) that share (m, n, b, beta, mu) but have their own weights,
 * alpha, x and y -- the Q/K/V or gate/up projections of one layer, or one
 * GEMV per request of a serving batch.  Equivalent to calling
 * bqg_biqgemm_f32 once per entry; the difference is only on the device:
 * for b == 1, mu == 8, beta <= 4 and count >= 4 the calls run in ONE
 * persistent kernel per 512 calls (keys through the texture pipe, the last
 * CTA to finish a call sums its partials: biqgemm_tex.cu); fewer calls run
 * the TMA-ring kernel plus its epilogue kernel.  Other shapes run the
 * single-call kernels back to back.  h_calls is a HOST array (copied into
 * the launch; graph-capturable); entries' device pointers must stay valid
 * until the stream reaches the work; d_keys_tiled 16-byte aligned.  y is
 * bitwise identical to the single-call stream form and deterministic.
 * Workspace: bqg_biqgemm_grouped_workspace_bytes(); its first 2 KiB hold
 * per-call completion counters that must be ZERO before the workspace's
 * first use (cudaMemset at allocation; the kernels leave them zero).  A
 * workspace address the library has not seen before is zeroed on `stream`
 * as a safety net. */
typedef struct bqg_call {
    const uint8_t* d_keys_tiled;
    const float* d_alpha; /* NULL = plane mode (alpha = 1) */
    const float* d_x;
    float* d_y;
} bqg_call;
size_t bqg_biqgemm_grouped_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                           size_t count);
int bqg_biqgemm_grouped_f32(const bqg_call* h_calls, size_t count, size_t x_rows, size_t m, size_t n,
                            size_t b, unsigned beta, unsigned mu, void* d_workspace,
                            size_t workspace_bytes, int pdl, void* stream);

/* Exact path: any mu in 1..16, any b; d_keys ROW-MAJOR (beta x m x G, u8 for
 * mu <= 8 else u16); fp64 LUT and accumulation in the reference's order, so y
 * is bit-identical to the reference.  Workspace from
 * bqg_biqgemm_exact_workspace_bytes (no zero-fill requirement). */
size_t bqg_biqgemm_exact_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu);
int bqg_biqgemm_exact_f32(const void* d_keys, const float* d_alpha, const float* d_x, size_t x_rows,
                          float* d_y, size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                          void* d_workspace, size_t workspace_bytes, void* stream);
int bqg_biqgemm_exact_f64(const void* d_keys, const double* d_alpha, const double* d_x,
                          size_t x_rows, double* d_y, size_t m, size_t n, size_t b, unsigned beta,
                          unsigned mu, void* d_workspace, size_t workspace_bytes, void* stream);
/* The same with the reference's KernelOptions::builder (kernel.hpp:51,158):
 * BQG_LUT_DP or BQG_LUT_NAIVE (lut.hpp:31-43) -- y is bit-identical to the
 * reference run with that builder.  stats (may be NULL) ACCUMULATES like
 * KernelStats (kernel.hpp:197-202): the builder's op law, and the phase split
 * of kernel.hpp:148-190 event-timed on `stream` (build = each group tile's
 * LUT kernel, query = its lookup kernel, replace = accumulator zero-fill +
 * alpha epilogue); with stats the call synchronises `stream`. */
int bqg_biqgemm_exact_ex_f32(const void* d_keys, const float* d_alpha, const float* d_x, size_t x_rows,
                             float* d_y, size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                             int builder, void* d_workspace, size_t workspace_bytes,
                             struct bqg_kernel_stats* stats, void* stream);
int bqg_biqgemm_exact_ex_f64(const void* d_keys, const double* d_alpha, const double* d_x,
                             size_t x_rows, double* d_y, size_t m, size_t n, size_t b, unsigned beta,
                             unsigned mu, int builder, void* d_workspace, size_t workspace_bytes,
                             struct bqg_kernel_stats* stats, void* stream);

/* Comparison baselines on the GPU (reference baselines.hpp; not the BiQGEMM
 * path).  gemm_unpack (baselines.hpp:40-52): y = sum_i alpha_i * (B_i x)
 * straight from the sign-plane words (beta x m x ceil(n/32) u32, bit 1 =
 * +1), fp32, b <= 8 and n*b*4 <= 200 KiB.  bandwidth_probe
 * (baselines.hpp:65-87): one multiply-add per packed word (values
 * meaningless); streaming != 0 reads the words with coalesced 16-byte loads
 * and writes one value per thread of a 1184 x 512 grid into d_out. */
int bqg_gemm_unpack_f32(const uint32_t* d_planes, const float* d_alpha, const float* d_x, size_t x_rows,
                        float* d_y, size_t m, size_t n, size_t b, unsigned beta, void* stream);
int bqg_bandwidth_probe(const uint32_t* d_words, size_t m, size_t n, const float* d_x, size_t x_rows,
                        float* d_out, int streaming, void* stream);

/* ------------------------------------------------------------ layer handle
 * A device-resident PackedLinear<float> (kernel.hpp:217-241) with its
 * workspace and a private stream: what the reference's callers hold. */
typedef struct bqg_layer bqg_layer;


/* quantize_greedy + pack_linear on the device from host weights W (m x n). */
int bqg_layer_create_from_weights(const float* h_w, size_t m, size_t n, unsigned beta, unsigned mu,
                                  bqg_layer** out);
/* From device weights (no H2D). */
int bqg_layer_create_from_device_weights(const float* d_w, size_t m, size_t n, unsigned beta,
                                         unsigned mu, bqg_layer** out);
/* From an already packed model (PackedLinear / a loaded BQGM payload):
 * h_keys row-major beta x m x G (u8 if mu <= 8 else u16), h_alpha beta x m
 * (NULL = plane mode, alpha = 1). */
int bqg_layer_create_from_keys(const void* h_keys, const float* h_alpha, size_t m, size_t n,
                               unsigned beta, unsigned mu, bqg_layer** out);
/* load() (model_io.cpp:92-141) straight onto the device. */
int bqg_layer_load_bqgm(const uint8_t* h_bytes, size_t len, bqg_layer** out);
void bqg_layer_destroy(bqg_layer* layer);

int bqg_layer_shape(const bqg_layer* layer, size_t* m, size_t* n, unsigned* beta, unsigned* mu);
/* Download keys (row-major, u8/u16) and alpha; plane words too if non-NULL. */
int bqg_layer_export(const bqg_layer* layer, void* h_keys, float* h_alpha, uint32_t* h_planes);
/* The fast path's view of a layer: (n, 8) for mu = 8; for every other mu
 * the re-keyed (bqg_rekey_mu8_columns(n, mu), 8) -- the shape its tiled keys
 * have (environment BQG_REKEY_SMALL_MU=0 at layer creation keeps mu < 8
 * layers on (n, mu)).  A call whose x has at most 8*ceil(n/8) rows runs with
 * that many columns (a prefix of the tiled layout: group blocks are its outer
 * index), so a mu != 8 layer of n columns takes the forms a mu = 8 layer takes. */
int bqg_layer_fast_shape(const bqg_layer* layer, size_t* n_fast, unsigned* mu_fast);
/* Device views (for device-resident timing and the sharded driver); the
 * tiled keys are in the fast view (bqg_layer_fast_shape). */
const uint8_t* bqg_layer_device_tiled_keys(const bqg_layer* layer);
const void* bqg_layer_device_keys(const bqg_layer* layer);
const float* bqg_layer_device_alpha(const bqg_layer* layer);

/* biqgemm(model, x) with HOST x (x_rows x b) and HOST y (m x b): H2D of x,
 * the fused kernel, D2H of y, synchronised before return -- the reference
 * call's contract.  exact selects the path: BQG_FORWARD_FAST (0; any mu,
 * mu > 8 through the re-keyed mu = 8 kernels), or the
 * exact (fp64, bit-identical) path with the reference's Dp builder
 * (BQG_FORWARD_EXACT, any nonzero value) or its Naive builder
 * (BQG_FORWARD_EXACT_NAIVE; KernelOptions::builder, kernel.hpp:51,158).
 * stats (may be NULL) ACCUMULATES like KernelStats (kernel.hpp:197-202). */
int bqg_layer_forward_host(bqg_layer* layer, const float* h_x, size_t x_rows, size_t b, float* h_y,
                           int exact, bqg_kernel_stats* stats);
/* biqgemm over a GROUP of layers that share (m, n, beta, mu) -- one call per
 * layer, each with its own x -- with HOST buffers: h_x is count x (x_rows x
 * b) contiguous, h_y is count x (m x b).  H2D of x, the grouped kernels
 * (bqg_biqgemm_grouped_f32) and D2H of y are pipelined in sub-groups sized
 * by host I/O (C2: 64, 128, 256 ... 128, 64 calls) on three streams;
 * synchronised before return.  When the same layers (by identity, not
 * address), the same pinned h_x / h_y and the same shape recur, the
 * pipeline is captured on the second occurrence and from then on replayed
 * as one CUDA graph launch.  Runs on a per-device library stream with its
 * own staging and workspace (thread-safe; calls are serialised).  exact != 0:
 * the exact path per layer.  stats (may be NULL) accumulates the counters of
 * all calls (stats calls are never captured). */
int bqg_layers_forward_host(bqg_layer* const* layers, size_t count, const float* h_x, size_t x_rows,
                            size_t b, float* h_y, int exact, bqg_kernel_stats* stats);
/* Device-resident forward on a caller stream (no copies, no sync).  The
 * layer's workspace is shared by its calls: calls on DIFFERENT streams must
 * not overlap in time (order them, or give each stream its own layer). */
int bqg_layer_forward_device(bqg_layer* layer, const float* d_x, size_t x_rows, size_t b, float* d_y,
                             int exact, int pdl, void* stream);

/* ---------------------------------------------------------------- multi-GPU
 * Output rows (m) sharded across ranks, one process per GPU (north_star;
 * the reference's row-partitioned workers, kernel.hpp:80-82,162-176).
 * Rank r owns rows [r*R, min(m, (r+1)*R)), R = 32*ceil(ceil(m/32)/nranks):
 * 32-row aligned, so y is bitwise identical for any nranks. */
int bqg_shard_rows(size_t m, int nranks, int rank, size_t* row_begin, size_t* row_end,
                   size_t* rows_per_rank);

/* Collectives used by the sharded call, stream-ordered on `stream`:
 * broadcast `bytes` of d_buf from `root` in place; all-gather
 * `bytes_per_rank` from d_send into d_recv (rank r's bytes at offset
 * r*bytes_per_rank; d_send may alias that slot).  bqg_nccl_collectives()
 * fills it with NCCL (ncclBroadcast / ncclAllGather over NVLink); tests can
 * plug in their own (e.g. gloo with host staging). */
typedef struct bqg_collectives {
    void* ctx;
    int (*broadcast)(void* ctx, void* d_buf, size_t bytes, int root, void* stream);
    int (*allgather)(void* ctx, const void* d_send, void* d_recv, size_t bytes_per_rank, void* stream);
} bqg_collectives;

/* NCCL, resolved at run time (dlopen libnccl.so.2; no link-time dependency).
 * The 128-byte unique id is created on one rank and passed to all (e.g. via
 * torch.distributed); the communicator binds to the current CUDA device. */
int bqg_nccl_available(void);
int bqg_nccl_unique_id(void* h_id128);
int bqg_nccl_comm_init(const void* h_id128, int nranks, int rank, void** comm_out);
int bqg_nccl_comm_destroy(void* comm);
int bqg_nccl_collectives(void* comm, bqg_collectives* out);

/* One row-sharded biqgemm call (kernel.hpp:246-258 over all m rows):
 *   1. broadcast d_x (x_rows x b) from rank 0, in place;
 *   2. this rank's rows [row_begin, row_end) with bqg_biqgemm_f32 on its
 *      shard (d_keys_tiled_shard / d_alpha_shard: the tiled keys and alpha of
 *      those rows, e.g. a layer built from W[row_begin:row_end]) into block
 *      `rank` of d_y_gather;
 *   3. all-gather the nranks blocks of R*b floats into d_y_gather.
 * d_y_gather holds nranks*R*b floats; its first m*b floats are y (m x b).
 * Workspace: bqg_biqgemm_sharded_workspace_bytes().  Every rank calls it
 * with the same (m, n, b, beta, mu). */
size_t bqg_biqgemm_sharded_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                           int nranks);
int bqg_biqgemm_sharded_f32(const uint8_t* d_keys_tiled_shard, const float* d_alpha_shard, float* d_x,
                            size_t x_rows, float* d_y_gather, size_t m, size_t n, size_t b,
                            unsigned beta, unsigned mu, int rank, int nranks,
                            const bqg_collectives* coll, void* d_workspace, size_t workspace_bytes,
                            void* stream);

/* A GROUP of row-sharded calls (the serving batch of bqg_biqgemm_grouped_f32,
 * each layer row-sharded): one broadcast of all calls' x, the grouped kernel
 * on this rank's rows of every call, one all-gather.
 *   d_x: count x (x_rows x b) contiguous; rank 0's contents are broadcast.
 *   d_y_gather: nranks x count x (R x b): block (r, i) holds rows
 *     [r*R, r*R + rows_r) of call i's y (R from bqg_shard_rows), so call i's
 *     y is the concatenation over r of the first rows_r rows of block (r, i).
 * h_calls: HOST array of this rank's shards (keys tiled, alpha or NULL).
 * Workspace: bqg_biqgemm_grouped_sharded_workspace_bytes(). */
typedef struct bqg_shard_call {
    const uint8_t* d_keys_tiled_shard;
    const float* d_alpha_shard;
} bqg_shard_call;
size_t bqg_biqgemm_grouped_sharded_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta,
                                                   unsigned mu, size_t count, int nranks);
int bqg_biqgemm_grouped_sharded_f32(const bqg_shard_call* h_calls, size_t count, float* d_x,
                                    size_t x_rows, float* d_y_gather, size_t m, size_t n, size_t b,
                                    unsigned beta, unsigned mu, int rank, int nranks,
                                    const bqg_collectives* coll, void* d_workspace,
                                    size_t workspace_bytes, int pdl, void* stream);

/* The same with the all-gather FUSED into the kernel (north_star's y
 * assembly over NVLink without a collective on the data): h_y_gather_peers
 * is a HOST array of nranks device pointers -- every rank's gather buffer
 * (nranks x count x R x b floats, same layout as above) as mapped in THIS
 * process (bqg_ipc_*; entry [rank] is the local buffer).  The texture
 * kernel's finaliser stores each y row into every rank's buffer as its call
 * completes; a 16-byte-per-rank all-gather through `coll` then orders every
 * rank's stores before later reads (a barrier).  Shapes the texture form
 * does not take fall back to the collective all-gather.  Workspace:
 * bqg_biqgemm_grouped_sharded_p2p_workspace_bytes(). */
size_t bqg_biqgemm_grouped_sharded_p2p_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta,
                                                       unsigned mu, size_t count, int nranks);
int bqg_biqgemm_grouped_sharded_p2p_f32(const bqg_shard_call* h_calls, size_t count, float* d_x,
                                        size_t x_rows, float* const* h_y_gather_peers, size_t m,
                                        size_t n, size_t b, unsigned beta, unsigned mu, int rank,
                                        int nranks, const bqg_collectives* coll, void* d_workspace,
                                        size_t workspace_bytes, int pdl, void* stream);
/* One row-sharded call with the all-gather fused into the kernels (the
 * north_star C5 decomposition): broadcast x, then the two-kernel form on this
 * rank's rows -- every shard count takes that form, so y is bitwise
 * independent of nranks -- whose finaliser stores each y value into every
 * rank's gather buffer (h_y_gather_peers as above; each buffer nranks x R x b
 * floats, the first m*b are y), then the 16-byte barrier.  b = 1 shapes the
 * latency / stream forms serve, and shapes the two-kernel form does not take,
 * run the rank's rows with bqg_biqgemm_f32 and gather through `coll`.
 * Workspace: bqg_biqgemm_sharded_p2p_workspace_bytes(). */
size_t bqg_biqgemm_sharded_p2p_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                               int nranks);
int bqg_biqgemm_sharded_p2p_f32(const uint8_t* d_keys_tiled_shard, const float* d_alpha_shard, float* d_x,
                                size_t x_rows, float* const* h_y_gather_peers, size_t m, size_t n,
                                size_t b, unsigned beta, unsigned mu, int rank, int nranks,
                                const bqg_collectives* coll, void* d_workspace, size_t workspace_bytes,
                                void* stream);
/* Peer buffers across processes: the cudaIpcMemHandle_t (64 opaque bytes)
 * of the allocation containing d_ptr plus d_ptr's offset in it (any device
 * pointer, e.g. a caching-allocator tensor); open maps a peer process's
 * buffer (lazy peer access) and returns the same offset into it; close
 * unmaps what open mapped. */
int bqg_ipc_get_handle(void* d_ptr, void* h_handle64, size_t* offset);
int bqg_ipc_open_handle(const void* h_handle64, size_t offset, void** d_ptr);
int bqg_ipc_close_handle(void* d_ptr);

#ifdef __cplusplus
}
#endif

#endif /* BQG_CAPI_H */
