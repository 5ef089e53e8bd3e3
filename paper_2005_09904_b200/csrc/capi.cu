// capi.cu -- implementation of include/bqg_capi.h.
//
// Host-side validation mirrors the reference's exceptions one for one (the
// reference file:line is given at each check); compute goes to the sm_100a
// kernels in quantize.cu / biqgemm_fast.cu / biqgemm_exact.cu.  There is no
// CPU compute path: without a CUDA device every compute entry point fails
// with BQG_ERR_NO_DEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <random>
#include <string>
#include <vector>

#include "../../include/bqg_capi.h"
#include "kernels.h"

namespace {

thread_local std::string g_msg;

int set_err(int st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_msg = buf;
    return st;
}

int cuda_err(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) {
        return set_err(BQG_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
    }
    return set_err(BQG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define BQG_CUDA(call)                                        \
    do {                                                      \
        cudaError_t _e = (call);                              \
        if (_e != cudaSuccess) return cuda_err(_e, #call);    \
    } while (0)

int ensure_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return set_err(BQG_ERR_NO_DEVICE,
                       "no usable CUDA device (%s); the library has no CPU fallback",
                       e == cudaSuccess ? "device count 0" : cudaGetErrorString(e));
    }
    return BQG_OK;
}

#define BQG_NEED_DEVICE()                    \
    do {                                     \
        int _s = ensure_device();            \
        if (_s != BQG_OK) return _s;         \
    } while (0)

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

size_t groups_of(size_t n, unsigned mu) { return (n + mu - 1) / mu; }

int check_mu(unsigned mu, const char* who) {
    // packing.hpp:85-87, lut.hpp:16-18: mu in [1, 16]
    if (mu < 1 || mu > 16) return set_err(BQG_ERR_INVALID_ARGUMENT, "%s: mu out of range [1,16]", who);
    return BQG_OK;
}

int check_dims(size_t m, size_t n, const char* who) {
    // matrix.hpp:23-25 / packing.hpp:28-31: dimensions must be nonzero
    if (m == 0 || n == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "%s: dimensions must be nonzero", who);
    return BQG_OK;
}

int check_x(size_t x_rows, size_t b, size_t n, unsigned mu, const char* who) {
    if (x_rows == 0 || b == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "%s: x dimensions must be nonzero", who);
    // kernel.hpp:132-134: the key matrix must cover x's rows
    if (static_cast<size_t>(mu) * groups_of(n, mu) < x_rows)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "%s: key matrix too narrow for input", who);
    return BQG_OK;
}

template <typename T, typename Dist>
int fill_random(T* out, size_t rows, size_t cols, uint64_t seed, Dist dist) {
    if (!out) return set_err(BQG_ERR_INVALID_ARGUMENT, "random fill: null output");
    if (rows == 0 || cols == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "Matrix: dimensions must be nonzero");
    std::mt19937_64 rng(seed);
    const size_t count = rows * cols;
    for (size_t i = 0; i < count; ++i) out[i] = dist(rng);
    return BQG_OK;
}

}  // namespace

// ============================================================== status / misc

extern "C" const char* bqg_status_string(int status) {
    switch (status) {
        case BQG_OK: return "ok";
        case BQG_ERR_INVALID_ARGUMENT: return "invalid argument";
        case BQG_ERR_CUDA: return "CUDA error";
        case BQG_ERR_NO_DEVICE: return "no CUDA device";
        case BQG_ERR_OUT_OF_MEMORY: return "out of device memory";
        case BQG_ERR_FORMAT: return "format error";
        case BQG_ERR_BAD_MAGIC: return "bad magic";
        case BQG_ERR_BAD_VERSION: return "bad version";
        case BQG_ERR_TRUNCATED: return "truncated";
        case BQG_ERR_RANGE: return "value out of range";
        case BQG_ERR_IO: return "I/O error";
        case BQG_ERR_WORKSPACE: return "workspace too small";
        case BQG_ERR_COMM: return "collective communication error";
        default: return "unknown status";
    }
}

extern "C" const char* bqg_last_error_message(void) { return g_msg.c_str(); }

extern "C" int bqg_abi_version(void) { return BQG_ABI_VERSION; }

// ============================================================== host-only

extern "C" int bqg_random_uniform_f32(float* out, size_t rows, size_t cols, uint64_t seed, float lo, float hi) {
    return fill_random(out, rows, cols, seed, std::uniform_real_distribution<float>(lo, hi));
}
extern "C" int bqg_random_normal_f32(float* out, size_t rows, size_t cols, uint64_t seed) {
    return fill_random(out, rows, cols, seed, std::normal_distribution<float>(0.0f, 1.0f));
}
extern "C" int bqg_random_uniform_f64(double* out, size_t rows, size_t cols, uint64_t seed, double lo, double hi) {
    return fill_random(out, rows, cols, seed, std::uniform_real_distribution<double>(lo, hi));
}
extern "C" int bqg_random_normal_f64(double* out, size_t rows, size_t cols, uint64_t seed) {
    return fill_random(out, rows, cols, seed, std::normal_distribution<double>(0.0, 1.0));
}

extern "C" int bqg_plan_tiles(size_t m, size_t groups, size_t b, unsigned mu, size_t budget, size_t entry_bytes,
                              size_t* t_w, size_t* t_h) {
    if (mu > 63) return set_err(BQG_ERR_INVALID_ARGUMENT, "plan_tiles: mu too large");
    const size_t per_group = (size_t(1) << mu) * b * entry_bytes;
    // kernel.hpp:62-64
    if (per_group == 0 || budget < per_group)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "plan_tiles: budget below one group's tables");
    const size_t tw = std::min(groups, budget / per_group);
    if (tw == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "plan_tiles: zero groups");
    const size_t th = std::clamp<size_t>(budget / (tw * sizeof(uint32_t)), 1, std::max<size_t>(m, 1));
    if (t_w) *t_w = tw;
    if (t_h) *t_h = th;
    return BQG_OK;
}

extern "C" int bqg_footprint(uint64_t m, uint64_t n, unsigned bits, uint64_t batch, unsigned abits, unsigned obits,
                             uint64_t* out) {
    // model_io.cpp:185-187
    if (bits == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "footprint: weight bits must be >= 1");
    out[0] = (m * n * bits + 7) / 8;
    out[1] = (n * batch * abits + 7) / 8;
    out[2] = (m * batch * obits + 7) / 8;
    out[3] = bits >= 32 ? 0 : uint64_t(4) * m * bits;
    return BQG_OK;
}

extern "C" int bqg_op_counters(size_t m, size_t n, size_t b, unsigned beta, unsigned mu, int builder,
                               uint64_t* out) {
    int s = check_mu(mu, "op_counters");
    if (s) return s;
    const uint64_t G = groups_of(n, mu);
    const uint64_t table = uint64_t(1) << mu;
    out[0] = (builder == BQG_LUT_NAIVE ? table * mu : table + mu - 1) * G * b;
    out[1] = uint64_t(m) * G * b * beta;
    out[2] = out[1];
    out[3] = 0;
    return BQG_OK;
}

extern "C" size_t bqg_tiled_key_bytes(size_t m, size_t n, unsigned beta, unsigned mu) {
    if (mu < 1 || mu > 8) return 0;
    const size_t G = groups_of(n, mu);
    return ((G + 31) / 32) * beta * ((m + 31) / 32) * 1024;
}

extern "C" size_t bqg_rekey_mu8_columns(size_t n, unsigned mu) {
    if (mu < 1 || mu > 16 || n == 0) return 0;
    return 8 * ((groups_of(n, mu) * mu + 7) / 8);
}

extern "C" int bqg_rekey_mu8(const void* d_keys, size_t m, size_t n, unsigned beta, unsigned mu, uint8_t* d_keys8,
                             void* stream) {
    int s = check_mu(mu, "rekey_mu8");
    if (s) return s;
    s = check_dims(m, n, "rekey_mu8");
    if (s) return s;
    if (beta == 0 || !d_keys || !d_keys8) return set_err(BQG_ERR_INVALID_ARGUMENT, "rekey_mu8: bad argument");
    BQG_NEED_DEVICE();
    const size_t n8 = bqg_rekey_mu8_columns(n, mu);
    cudaError_t e = bqg::launch_rekey_mu8(d_keys, static_cast<long long>(beta) * static_cast<long long>(m),
                                          static_cast<long long>(groups_of(n, mu)), static_cast<int>(mu),
                                          static_cast<long long>(n8 / 8), d_keys8, as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "rekey_mu8 kernel");
    return BQG_OK;
}

// ---- BQGM (model_io.cpp:65-141) ----

namespace {

constexpr uint8_t kMagic[4] = {'B', 'Q', 'G', 'M'};
constexpr uint16_t kVersion = 1;

struct Cursor {
    const uint8_t* p;
    size_t len, pos;
    bool need(size_t k) const { return pos + k <= len; }
};

int truncated(const Cursor& c) {
    return set_err(BQG_ERR_TRUNCATED, "model file truncated at offset %zu", c.pos);
}

}  // namespace

extern "C" int bqg_bqgm_parse(const uint8_t* bytes, size_t len, size_t* m_out, size_t* n_out, unsigned* beta_out,
                              unsigned* mu_out, float* alpha, void* keys) {
    Cursor c{bytes, len, 0};
    if (!c.need(4)) return truncated(c);
    if (std::memcmp(bytes, kMagic, 4) != 0) return set_err(BQG_ERR_BAD_MAGIC, "bad magic, expected BQGM");
    c.pos = 4;
    if (!c.need(2)) return truncated(c);
    const uint16_t version = uint16_t(bytes[4] | (uint16_t(bytes[5]) << 8));
    c.pos = 6;
    if (version != kVersion) return set_err(BQG_ERR_BAD_VERSION, "unsupported version %u", unsigned(version));
    auto u32 = [&](uint32_t& v) {
        if (!c.need(4)) return false;
        v = 0;
        for (int i = 0; i < 4; ++i) v |= uint32_t(bytes[c.pos + i]) << (8 * i);
        c.pos += 4;
        return true;
    };
    uint32_t m = 0, n = 0;
    if (!u32(m)) return truncated(c);
    if (!u32(n)) return truncated(c);
    if (!c.need(1)) return truncated(c);
    const unsigned beta = bytes[c.pos++];
    if (!c.need(1)) return truncated(c);
    const unsigned mu = bytes[c.pos++];
    // model_io.cpp:108-113
    if (m == 0 || n == 0 || beta == 0) return set_err(BQG_ERR_RANGE, "zero dimension in header");
    if (mu < 1 || mu > 16) return set_err(BQG_ERR_RANGE, "mu out of range [1,16]");
    const size_t G = groups_of(n, mu);
    const uint32_t limit = 1u << mu;
    const bool wide = mu > 8;
    for (unsigned i = 0; i < beta; ++i) {
        for (size_t r = 0; r < m; ++r) {
            uint32_t bits;
            if (!u32(bits)) return truncated(c);
            if (alpha) std::memcpy(alpha + size_t(i) * m + r, &bits, 4);
        }
        const size_t count = size_t(m) * G;
        for (size_t k = 0; k < count; ++k) {
            uint32_t key;
            if (wide) {
                if (!c.need(2)) return truncated(c);
                key = uint32_t(bytes[c.pos]) | (uint32_t(bytes[c.pos + 1]) << 8);
                c.pos += 2;
            } else {
                if (!c.need(1)) return truncated(c);
                key = bytes[c.pos++];
            }
            if (key >= limit) return set_err(BQG_ERR_RANGE, "key out of range for mu=%u", mu);
            if (keys) {
                if (wide) static_cast<uint16_t*>(keys)[size_t(i) * count + k] = uint16_t(key);
                else static_cast<uint8_t*>(keys)[size_t(i) * count + k] = uint8_t(key);
            }
        }
    }
    // model_io.cpp:137-139
    if (c.pos != len) return set_err(BQG_ERR_FORMAT, "trailing bytes after payload");
    *m_out = m;
    *n_out = n;
    *beta_out = beta;
    *mu_out = mu;
    return BQG_OK;
}

extern "C" int bqg_bqgm_serialize(const void* keys, const float* alpha, size_t m, size_t n, unsigned beta,
                                  unsigned mu, uint8_t* out, size_t* len) {
    int s = check_mu(mu, "save");  // model_io.cpp:66-68
    if (s) return s;
    if (m == 0 || n == 0 || beta == 0 || beta > 255 || m > 0xffffffffu || n > 0xffffffffu)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "save: dimensions out of range");
    const size_t G = groups_of(n, mu);
    const bool wide = mu > 8;
    const size_t total = 16 + size_t(beta) * (4 * m + m * G * (wide ? 2 : 1));
    if (out) {
        if (*len < total) return set_err(BQG_ERR_INVALID_ARGUMENT, "save: buffer too small");
        size_t pos = 0;
        std::memcpy(out, kMagic, 4);
        pos = 4;
        out[pos++] = uint8_t(kVersion & 0xff);
        out[pos++] = uint8_t(kVersion >> 8);
        for (int i = 0; i < 4; ++i) out[pos++] = uint8_t(uint32_t(m) >> (8 * i));
        for (int i = 0; i < 4; ++i) out[pos++] = uint8_t(uint32_t(n) >> (8 * i));
        out[pos++] = uint8_t(beta);
        out[pos++] = uint8_t(mu);
        for (unsigned i = 0; i < beta; ++i) {
            for (size_t r = 0; r < m; ++r) {
                const float a = alpha ? alpha[size_t(i) * m + r] : 1.0f;
                uint32_t bits;
                std::memcpy(&bits, &a, 4);
                for (int k = 0; k < 4; ++k) out[pos++] = uint8_t(bits >> (8 * k));
            }
            const size_t count = m * G;
            for (size_t k = 0; k < count; ++k) {
                if (wide) {
                    const uint16_t v = static_cast<const uint16_t*>(keys)[size_t(i) * count + k];
                    out[pos++] = uint8_t(v & 0xff);
                    out[pos++] = uint8_t(v >> 8);
                } else {
                    out[pos++] = static_cast<const uint8_t*>(keys)[size_t(i) * count + k];
                }
            }
        }
    }
    *len = total;
    return BQG_OK;
}

// ============================================================== device primitives

template <typename T>
static int quantize_impl(const T* d_w, size_t m, size_t n, unsigned beta, uint32_t* d_planes, T* d_alpha,
                         void* stream) {
    // quantize.hpp:29-31
    if (beta == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "quantize_greedy: beta must be >= 1");
    int s = check_dims(m, n, "quantize_greedy");
    if (s) return s;
    if (!d_w || !d_planes || !d_alpha) return set_err(BQG_ERR_INVALID_ARGUMENT, "quantize_greedy: null pointer");
    BQG_NEED_DEVICE();
    cudaStream_t st = as_stream(stream);
    double* alpha_d = nullptr;
    BQG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&alpha_d), sizeof(double) * beta * m, st));
    cudaError_t e = bqg::launch_quantize_greedy<T>(d_w, static_cast<long long>(m), static_cast<long long>(n),
                                                   static_cast<int>(beta), d_planes, d_alpha, alpha_d, st);
    cudaFreeAsync(alpha_d, st);
    if (e != cudaSuccess) return cuda_err(e, "quantize_greedy kernel");
    return BQG_OK;
}

extern "C" int bqg_quantize_greedy_f32(const float* d_w, size_t m, size_t n, unsigned beta, uint32_t* d_planes,
                                       float* d_alpha, void* stream) {
    return quantize_impl<float>(d_w, m, n, beta, d_planes, d_alpha, stream);
}

extern "C" int bqg_quantize_greedy_f64(const double* d_w, size_t m, size_t n, unsigned beta, uint32_t* d_planes,
                                       double* d_alpha, void* stream) {
    return quantize_impl<double>(d_w, m, n, beta, d_planes, d_alpha, stream);
}

extern "C" int bqg_pack_keys(const uint32_t* d_plane, size_t m, size_t n, unsigned mu, void* d_keys, void* stream) {
    int s = check_mu(mu, "pack_keys");
    if (s) return s;
    s = check_dims(m, n, "pack_keys");
    if (s) return s;
    if (!d_plane || !d_keys) return set_err(BQG_ERR_INVALID_ARGUMENT, "pack_keys: null pointer");
    BQG_NEED_DEVICE();
    cudaError_t e = bqg::launch_pack_keys(d_plane, static_cast<long long>(m), static_cast<long long>(n),
                                          static_cast<int>(mu), d_keys, as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "pack_keys kernel");
    return BQG_OK;
}

extern "C" int bqg_tile_keys(const uint8_t* d_keys, size_t m, size_t n, unsigned beta, unsigned mu,
                             uint8_t* d_tiled, void* stream) {
    if (mu < 1 || mu > 8) return set_err(BQG_ERR_INVALID_ARGUMENT, "tile_keys: tiled layout needs mu in [1,8]");
    int s = check_dims(m, n, "tile_keys");
    if (s) return s;
    if (beta == 0 || !d_keys || !d_tiled) return set_err(BQG_ERR_INVALID_ARGUMENT, "tile_keys: bad argument");
    BQG_NEED_DEVICE();
    cudaError_t e = bqg::launch_tile_keys(d_keys, static_cast<long long>(m),
                                          static_cast<long long>(groups_of(n, mu)), static_cast<int>(beta),
                                          d_tiled, as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "tile_keys kernel");
    return BQG_OK;
}

namespace {
int check_lut_args(size_t x_rows, size_t b, unsigned mu, size_t count, int layout, int builder, const char* who,
                   bool allow_naive = false) {
    int s = check_mu(mu, who);
    if (s) return s;
    if (count == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "build_lut_block: empty tile");  // lut.hpp:114-116
    if (x_rows == 0 || b == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "%s: x dimensions must be nonzero", who);
    if (layout != BQG_LUT_TABLE_MAJOR && layout != BQG_LUT_KEY_MAJOR)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "%s: unknown layout", who);
    if (builder != BQG_LUT_DP && !(allow_naive && builder == BQG_LUT_NAIVE))
        return set_err(BQG_ERR_INVALID_ARGUMENT, "%s: unsupported builder", who);
    return BQG_OK;
}
}  // namespace

extern "C" int bqg_build_lut_f32(const float* d_x, size_t x_rows, size_t b, unsigned mu, size_t g0, size_t count,
                                 int layout, int builder, float* d_entries, uint64_t* ops, void* stream) {
    int s = check_lut_args(x_rows, b, mu, count, layout, builder, "build_lut_f32");
    if (s) return s;
    if (mu > 8) return set_err(BQG_ERR_INVALID_ARGUMENT, "build_lut_f32: shared-memory builder needs mu <= 8");
    BQG_NEED_DEVICE();
    cudaError_t e = bqg::launch_build_lut_f32(d_x, static_cast<long long>(x_rows), static_cast<long long>(b),
                                              static_cast<int>(mu), static_cast<long long>(g0),
                                              static_cast<long long>(count), layout == BQG_LUT_KEY_MAJOR,
                                              d_entries, as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "build_lut_f32 kernel");
    if (ops) *ops += ((uint64_t(1) << mu) + mu - 1) * count * b;
    return BQG_OK;
}

template <typename T>
static int build_lut_exact_impl(const T* d_x, size_t x_rows, size_t b, unsigned mu, size_t g0, size_t count,
                                int layout, int builder, double* d_entries, uint64_t* ops, void* stream,
                                const char* who) {
    int s = check_lut_args(x_rows, b, mu, count, layout, builder, who, true);
    if (s) return s;
    if (!d_x || !d_entries) return set_err(BQG_ERR_INVALID_ARGUMENT, "%s: null pointer", who);
    BQG_NEED_DEVICE();
    cudaError_t e = bqg::launch_build_lut_exact<T>(
        d_x, static_cast<long long>(x_rows), static_cast<long long>(b), static_cast<int>(mu),
        static_cast<long long>(g0), static_cast<long long>(count), layout == BQG_LUT_KEY_MAJOR, d_entries,
        as_stream(stream), builder == BQG_LUT_NAIVE);
    if (e != cudaSuccess) return cuda_err(e, "build_lut exact kernel");
    // lut.hpp:42 (naive: 2^mu * mu per table), lut.hpp:68 (dp: 2^mu + mu - 1)
    const uint64_t per = builder == BQG_LUT_NAIVE ? (uint64_t(1) << mu) * mu : (uint64_t(1) << mu) + mu - 1;
    if (ops) *ops += per * count * b;
    return BQG_OK;
}

extern "C" int bqg_build_lut_f64(const float* d_x, size_t x_rows, size_t b, unsigned mu, size_t g0, size_t count,
                                 int layout, int builder, double* d_entries, uint64_t* ops, void* stream) {
    return build_lut_exact_impl<float>(d_x, x_rows, b, mu, g0, count, layout, builder, d_entries, ops, stream,
                                       "build_lut_f64");
}

extern "C" int bqg_build_lut_f64x(const double* d_x, size_t x_rows, size_t b, unsigned mu, size_t g0,
                                  size_t count, int layout, int builder, double* d_entries, uint64_t* ops,
                                  void* stream) {
    return build_lut_exact_impl<double>(d_x, x_rows, b, mu, g0, count, layout, builder, d_entries, ops, stream,
                                        "build_lut_f64x");
}

extern "C" size_t bqg_biqgemm_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu) {
    if (mu < 1 || mu > 8 || m == 0 || n == 0 || b == 0 || beta == 0) return 0;
    return bqg::fast_workspace_bytes(static_cast<long long>(m), static_cast<long long>(groups_of(n, mu)),
                                     static_cast<int>(beta), static_cast<long long>(b));
}

namespace {
bqg::QueryParams make_params(const uint8_t* keys, const float* alpha, const float* x, size_t x_rows, float* y,
                             size_t m, size_t n, size_t b, unsigned beta, unsigned mu, void* ws) {
    bqg::QueryParams p{};
    const long long G = static_cast<long long>(groups_of(n, mu));
    p.keys = keys;
    p.alpha = alpha;
    p.x = x;
    p.y = y;
    p.ws = static_cast<float*>(ws);
    p.partial = p.ws + bqg::kTexCounterBytes / sizeof(float);
    p.x_rows = static_cast<long long>(x_rows);
    p.m = static_cast<int>(m);
    p.G = static_cast<int>(G);
    p.NB = static_cast<int>((G + 31) / 32);
    p.MT = static_cast<int>((static_cast<long long>(m) + 31) / 32);
    p.beta = static_cast<int>(beta);
    p.b = static_cast<int>(b);
    p.cpb = 1;
    return p;
}
}  // namespace

extern "C" int bqg_biqgemm_f32(const uint8_t* d_keys, const float* d_alpha, const float* d_x, size_t x_rows,
                               float* d_y, size_t m, size_t n, size_t b, unsigned beta, unsigned mu, void* d_ws,
                               size_t ws_bytes, int pdl, void* stream) {
    int s = check_mu(mu, "biqgemm");
    if (s) return s;
    if (mu > 8) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_f32: fast path needs mu <= 8 (use the exact path)");
    s = check_dims(m, n, "biqgemm");
    if (s) return s;
    if (beta == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: beta must be >= 1");
    s = check_x(x_rows, b, n, mu, "biqgemm");
    if (s) return s;
    if (m > 0x7fffffff || b > 0x7fffffff) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: dimension too large");
    {
        const unsigned long long chunks = ((groups_of(n, mu) + 31) / 32) * ((m + 31) / 32) * beta *
                                          ((b + 3) / 4 + 1);
        if (chunks > 0x7fffffffull) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: problem too large for one call");
    }
    if (!d_keys || !d_x || !d_y || !d_ws) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: null pointer");
    if (ws_bytes < bqg_biqgemm_workspace_bytes(m, n, b, beta, mu))
        return set_err(BQG_ERR_WORKSPACE, "biqgemm: workspace %zu < %zu bytes", ws_bytes,
                       bqg_biqgemm_workspace_bytes(m, n, b, beta, mu));
    BQG_NEED_DEVICE();
    const bqg::QueryParams p = make_params(d_keys, d_alpha, d_x, x_rows, d_y, m, n, b, beta, mu, d_ws);
    cudaError_t e = bqg::launch_biqgemm_fast(p, static_cast<int>(mu), pdl != 0, as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "biqgemm fast kernel");
    return BQG_OK;
}

extern "C" size_t bqg_biqgemm_grouped_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                                      size_t count) {
    if (mu < 1 || mu > 8 || m == 0 || n == 0 || b == 0 || beta == 0 || count == 0) return 0;
    const size_t single = bqg_biqgemm_workspace_bytes(m, n, b, beta, mu);
    if (!bqg::stream_supported(static_cast<int>(mu), static_cast<int>(beta), static_cast<long long>(b)))
        return single;
    const size_t grouped = bqg::stream_workspace_bytes(static_cast<long long>(m),
                                                       static_cast<long long>(groups_of(n, mu)),
                                                       static_cast<int>(std::min<size_t>(count, 1u << 30)));
    return std::max(single, grouped);
}

extern "C" int bqg_biqgemm_grouped_f32(const bqg_call* h_calls, size_t count, size_t x_rows, size_t m, size_t n,
                                       size_t b, unsigned beta, unsigned mu, void* d_ws, size_t ws_bytes, int pdl,
                                       void* stream) {
    int s = check_mu(mu, "biqgemm");
    if (s) return s;
    if (mu > 8) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_grouped: fast path needs mu <= 8 (use the exact path)");
    s = check_dims(m, n, "biqgemm");
    if (s) return s;
    if (beta == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: beta must be >= 1");
    s = check_x(x_rows, b, n, mu, "biqgemm");
    if (s) return s;
    if (count == 0) return BQG_OK;
    if (!h_calls || !d_ws) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_grouped: null pointer");
    for (size_t i = 0; i < count; ++i)
        if (!h_calls[i].d_keys_tiled || !h_calls[i].d_x || !h_calls[i].d_y)
            return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_grouped: null pointer in call %zu", i);
    if (ws_bytes < bqg_biqgemm_grouped_workspace_bytes(m, n, b, beta, mu, count))
        return set_err(BQG_ERR_WORKSPACE, "biqgemm_grouped: workspace %zu < %zu bytes", ws_bytes,
                       bqg_biqgemm_grouped_workspace_bytes(m, n, b, beta, mu, count));
    if (m > 0x7fffffff || count > 0x7fffffff) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: dimension too large");
    BQG_NEED_DEVICE();
    if (!bqg::stream_supported(static_cast<int>(mu), static_cast<int>(beta), static_cast<long long>(b))) {
        for (size_t i = 0; i < count; ++i) {
            s = bqg_biqgemm_f32(h_calls[i].d_keys_tiled, h_calls[i].d_alpha, h_calls[i].d_x, x_rows, h_calls[i].d_y,
                                m, n, b, beta, mu, d_ws, ws_bytes, pdl || i > 0, stream);
            if (s) return s;
        }
        return BQG_OK;
    }
    std::vector<bqg::StreamCall> calls(count);
    for (size_t i = 0; i < count; ++i)
        calls[i] = {h_calls[i].d_keys_tiled, h_calls[i].d_alpha, h_calls[i].d_x, h_calls[i].d_y};
    cudaError_t e = bqg::launch_biqgemm_stream(calls.data(), static_cast<int>(count), static_cast<long long>(x_rows),
                                               static_cast<int>(m), static_cast<int>(groups_of(n, mu)),
                                               static_cast<int>(beta), static_cast<float*>(d_ws), pdl != 0,
                                               as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "biqgemm grouped kernels");
    return BQG_OK;
}

extern "C" int bqg_biqgemm_form(size_t m, size_t n, size_t b, unsigned beta, unsigned mu) {
    if (mu < 1 || mu > 8 || m == 0 || n == 0 || b == 0 || beta == 0) return 0;
    if (ensure_device() != BQG_OK) return 0;
    const bqg::QueryParams p = make_params(nullptr, nullptr, nullptr, n, nullptr, m, n, b, beta, mu, nullptr);
    return bqg::fast_form(p, static_cast<int>(mu));
}

extern "C" size_t bqg_biqgemm_exact_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu) {
    if (mu < 1 || mu > 16 || m == 0 || n == 0 || b == 0 || beta == 0) return 0;
    return bqg::exact_workspace_bytes(static_cast<long long>(m), static_cast<long long>(n), static_cast<int>(beta),
                                      static_cast<int>(mu), static_cast<long long>(b));
}

namespace {
// Event trail of one exact call: an event before the call, one per phase
// mark (bqg::PhaseMarks), one after.  The reference's phase split
// (kernel.hpp:156-159): build = each tile's LUT build, query = each tile's
// lookups, replace = accumulator setup + the alpha epilogue.
struct EventTrail {
    std::vector<cudaEvent_t> ev;
    std::vector<int> phase;
    cudaError_t err = cudaSuccess;
    static void mark(void* ctx, int ph, cudaStream_t s) {
        auto* t = static_cast<EventTrail*>(ctx);
        cudaEvent_t e = nullptr;
        cudaError_t r = cudaEventCreate(&e);
        if (r == cudaSuccess) r = cudaEventRecord(e, s);
        if (r != cudaSuccess) {
            if (t->err == cudaSuccess) t->err = r;
            if (e) cudaEventDestroy(e);
            return;
        }
        t->ev.push_back(e);
        t->phase.push_back(ph);
    }
    ~EventTrail() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
    // seconds[0..2] += build, query, replace
    void accumulate(double* seconds) const {
        for (size_t i = 0; i + 1 < ev.size(); ++i) {
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            const int ph = phase[i];
            seconds[ph == 0 ? 0 : (ph == 1 ? 1 : 2)] += ms * 1e-3;
        }
    }
};
}  // namespace

template <typename T>
static int biqgemm_exact_impl(const void* d_keys, const T* d_alpha, const T* d_x, size_t x_rows, T* d_y, size_t m,
                              size_t n, size_t b, unsigned beta, unsigned mu, int builder, void* d_ws,
                              size_t ws_bytes, bqg_kernel_stats* stats, void* stream) {
    int s = check_mu(mu, "biqgemm");
    if (s) return s;
    s = check_dims(m, n, "biqgemm");
    if (s) return s;
    if (beta == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: beta must be >= 1");
    s = check_x(x_rows, b, n, mu, "biqgemm");
    if (s) return s;
    if (!d_keys || !d_x || !d_y || !d_ws) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: null pointer");
    if (builder != BQG_LUT_DP && builder != BQG_LUT_NAIVE)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: unsupported builder");
    if (ws_bytes < bqg_biqgemm_exact_workspace_bytes(m, n, b, beta, mu))
        return set_err(BQG_ERR_WORKSPACE, "biqgemm_exact: workspace too small");
    BQG_NEED_DEVICE();
    cudaStream_t st = as_stream(stream);
    EventTrail trail;
    const bqg::PhaseMarks marks{&trail, &EventTrail::mark};
    if (stats) EventTrail::mark(&trail, 2, st);  // accumulator zero-fill: "replace" (kernel.hpp:148-150)
    cudaError_t e = bqg::launch_biqgemm_exact<T>(d_keys, d_alpha, d_x, static_cast<long long>(x_rows), d_y,
                                                 static_cast<long long>(m), static_cast<long long>(n),
                                                 static_cast<int>(beta), static_cast<int>(mu),
                                                 static_cast<long long>(b), d_ws, ws_bytes, st,
                                                 builder == BQG_LUT_NAIVE, stats ? &marks : nullptr);
    if (e != cudaSuccess) return cuda_err(e, "biqgemm exact kernels");
    if (stats) {
        EventTrail::mark(&trail, 3, st);
        if (trail.err != cudaSuccess) return cuda_err(trail.err, "biqgemm exact: phase events");
        BQG_CUDA(cudaStreamSynchronize(st));
        uint64_t ops[4];
        bqg_op_counters(m, n, b, beta, mu, builder, ops);
        stats->lut_build_ops += ops[0];
        stats->lookups += ops[1];
        stats->accumulate_ops += ops[2];
        stats->fma_ops += ops[3];
        double sec[3] = {0.0, 0.0, 0.0};
        trail.accumulate(sec);
        stats->build_seconds += sec[0];
        stats->query_seconds += sec[1];
        stats->replace_seconds += sec[2];
    }
    return BQG_OK;
}

extern "C" int bqg_biqgemm_exact_f32(const void* d_keys, const float* d_alpha, const float* d_x, size_t x_rows,
                                     float* d_y, size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                     void* d_ws, size_t ws_bytes, void* stream) {
    return biqgemm_exact_impl<float>(d_keys, d_alpha, d_x, x_rows, d_y, m, n, b, beta, mu, BQG_LUT_DP, d_ws,
                                     ws_bytes, nullptr, stream);
}

extern "C" int bqg_biqgemm_exact_f64(const void* d_keys, const double* d_alpha, const double* d_x, size_t x_rows,
                                     double* d_y, size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                     void* d_ws, size_t ws_bytes, void* stream) {
    return biqgemm_exact_impl<double>(d_keys, d_alpha, d_x, x_rows, d_y, m, n, b, beta, mu, BQG_LUT_DP, d_ws,
                                      ws_bytes, nullptr, stream);
}

extern "C" int bqg_biqgemm_exact_ex_f32(const void* d_keys, const float* d_alpha, const float* d_x, size_t x_rows,
                                        float* d_y, size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                        int builder, void* d_ws, size_t ws_bytes, bqg_kernel_stats* stats,
                                        void* stream) {
    return biqgemm_exact_impl<float>(d_keys, d_alpha, d_x, x_rows, d_y, m, n, b, beta, mu, builder, d_ws, ws_bytes,
                                     stats, stream);
}

extern "C" int bqg_biqgemm_exact_ex_f64(const void* d_keys, const double* d_alpha, const double* d_x,
                                        size_t x_rows, double* d_y, size_t m, size_t n, size_t b, unsigned beta,
                                        unsigned mu, int builder, void* d_ws, size_t ws_bytes,
                                        bqg_kernel_stats* stats, void* stream) {
    return biqgemm_exact_impl<double>(d_keys, d_alpha, d_x, x_rows, d_y, m, n, b, beta, mu, builder, d_ws,
                                      ws_bytes, stats, stream);
}

// ============================================================== comparison baselines

extern "C" int bqg_gemm_unpack_f32(const uint32_t* d_planes, const float* d_alpha, const float* d_x, size_t x_rows,
                                   float* d_y, size_t m, size_t n, size_t b, unsigned beta, void* stream) {
    int s = check_dims(m, n, "gemm_unpack");
    if (s) return s;
    if (beta == 0 || b == 0 || b > 8 || x_rows == 0 || x_rows > n || n * b * 4 > 200 * 1024)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "gemm_unpack: needs 1 <= b <= 8, x_rows <= n, n*b*4 <= 200 KiB");
    if (!d_planes || !d_x || !d_y) return set_err(BQG_ERR_INVALID_ARGUMENT, "gemm_unpack: null pointer");
    BQG_NEED_DEVICE();
    cudaError_t e = bqg::launch_gemm_unpack(d_planes, d_alpha, d_x, static_cast<long long>(x_rows), d_y,
                                            static_cast<long long>(m), static_cast<long long>(n), static_cast<int>(b),
                                            static_cast<int>(beta), as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "gemm_unpack kernel");
    return BQG_OK;
}

extern "C" int bqg_bandwidth_probe(const uint32_t* d_words, size_t m, size_t n, const float* d_x, size_t x_rows,
                                   float* d_out, int streaming, void* stream) {
    int s = check_dims(m, n, "gemm_bandwidth_probe");
    if (s) return s;
    if (!d_words || !d_x || !d_out || x_rows == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "bandwidth_probe: bad argument");
    BQG_NEED_DEVICE();
    cudaError_t e = bqg::launch_bandwidth_probe(d_words, static_cast<long long>(m), static_cast<long long>(n), d_x,
                                                static_cast<long long>(x_rows), d_out, streaming != 0,
                                                as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "bandwidth_probe kernel");
    return BQG_OK;
}

// ============================================================== layer handle

struct bqg_layer {
    uint64_t uid = 0;  // process-unique (a new layer at a freed layer's address is a different layer)
    size_t m = 0, n = 0, G = 0;
    unsigned beta = 0, mu = 0;
    // The fast path's view: mu <= 8 -> (n, mu); mu > 8 -> the sign bits
    // re-keyed to mu = 8 over fn = bqg_rekey_mu8_columns(n, mu) columns (the
    // fast kernels' u8 keys and shared-memory tables; y within the fp32
    // contract of the reference's mu, the exact path stays bit-identical).
    size_t fn = 0;
    unsigned fmu = 0;
    bool plane_mode = false;
    cudaStream_t stream = nullptr;
    uint32_t* d_planes = nullptr;  // only when created from weights
    void* d_keys = nullptr;        // row-major u8/u16
    uint8_t* d_tiled = nullptr;    // tiled u8 keys of the fast view (fn, fmu)
    float* d_alpha = nullptr;
    // forward scratch (grown on demand)
    void* d_ws = nullptr;
    size_t ws_bytes = 0;
    void* d_ws_exact = nullptr;
    size_t ws_exact_bytes = 0;
    float* d_x = nullptr;
    size_t x_cap = 0;
    float* d_y = nullptr;
    size_t y_cap = 0;
    float* h_x_pin = nullptr;  // pinned staging for pageable caller buffers (forward_host)
    size_t hx_cap = 0;
    float* h_y_pin = nullptr;
    size_t hy_cap = 0;
    // cached CUDA graph of one host forward (H2D -> kernels -> D2H) for the
    // last (x_rows, b, exact) shape; captured on the second call of a shape
    cudaGraphExec_t gexec = nullptr;
    size_t g_xrows = 0, g_b = 0;
    int g_exact = -1, g_seen = 0;
    unsigned buf_gen = 0, g_gen = 0;  // bumped whenever a buffer the graph uses is reallocated
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    std::mutex mu_lock;

    size_t key_bytes_per_plane() const { return m * G * (mu > 8 ? 2 : 1); }
};

namespace {

void layer_free(bqg_layer* L) {
    if (!L) return;
    if (L->stream) cudaStreamSynchronize(L->stream);
    cudaFree(L->d_planes);
    cudaFree(L->d_keys);
    cudaFree(L->d_tiled);
    cudaFree(L->d_alpha);
    cudaFree(L->d_ws);
    cudaFree(L->d_ws_exact);
    cudaFree(L->d_x);
    cudaFree(L->d_y);
    cudaFreeHost(L->h_x_pin);
    cudaFreeHost(L->h_y_pin);
    if (L->gexec) cudaGraphExecDestroy(L->gexec);
    for (auto& e : L->ev)
        if (e) cudaEventDestroy(e);
    if (L->stream) cudaStreamDestroy(L->stream);
    delete L;
}

int layer_alloc(size_t m, size_t n, unsigned beta, unsigned mu, bool plane_mode, bqg_layer** out) {
    if (!out) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null output");
    int s = check_mu(mu, "pack_linear");
    if (s) return s;
    s = check_dims(m, n, "pack_linear");
    if (s) return s;
    if (beta == 0) return set_err(BQG_ERR_INVALID_ARGUMENT, "quantize_greedy: beta must be >= 1");
    if (m > 0x7fffffff) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: m too large");
    BQG_NEED_DEVICE();
    bqg_layer* L = new (std::nothrow) bqg_layer();
    if (!L) return set_err(BQG_ERR_OUT_OF_MEMORY, "layer: host allocation failed");
    static std::atomic<uint64_t> next_uid{1};
    L->uid = next_uid.fetch_add(1, std::memory_order_relaxed);
    L->m = m;
    L->n = n;
    L->beta = beta;
    L->mu = mu;
    L->G = groups_of(n, mu);
    // mu != 8: the same sign bits re-keyed to mu = 8 (mu > 8: u16 keys the
    // fast kernels do not take; mu < 8: the mu = 8 forms -- latency, texture,
    // stream -- are several times faster than the mu < 8 two-kernel form;
    // BQG_REKEY_SMALL_MU=0 keeps mu < 8 layers on their own keys, for A/B)
    static const bool keep_small_mu = [] {
        const char* v = getenv("BQG_REKEY_SMALL_MU");
        return v && v[0] == '0';
    }();
    const bool native = mu == 8 || (mu < 8 && keep_small_mu);
    L->fn = native ? n : bqg_rekey_mu8_columns(n, mu);
    L->fmu = native ? mu : 8;
    L->plane_mode = plane_mode;
    cudaError_t e = cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&L->d_keys, L->key_bytes_per_plane() * beta);
    if (e == cudaSuccess)
        e = cudaMalloc(reinterpret_cast<void**>(&L->d_tiled), bqg_tiled_key_bytes(m, L->fn, beta, L->fmu));
    if (e == cudaSuccess && !plane_mode) e = cudaMalloc(reinterpret_cast<void**>(&L->d_alpha), sizeof(float) * beta * m);
    for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&L->ev[i]);
    if (e != cudaSuccess) {
        layer_free(L);
        return cuda_err(e, "layer allocation");
    }
    *out = L;
    return BQG_OK;
}

int layer_finish_tiling(bqg_layer* L) {
    if (L->fmu == L->mu) {
        cudaError_t e = bqg::launch_tile_keys(static_cast<const uint8_t*>(L->d_keys), static_cast<long long>(L->m),
                                              static_cast<long long>(L->G), static_cast<int>(L->beta), L->d_tiled,
                                              L->stream);
        if (e != cudaSuccess) return cuda_err(e, "tile_keys kernel");
    } else {
        // mu != 8: the same sign bits as mu = 8 keys, then the fast path's tiling
        uint8_t* k8 = nullptr;
        const size_t g8 = L->fn / 8;
        BQG_CUDA(cudaMalloc(reinterpret_cast<void**>(&k8), size_t(L->beta) * L->m * g8));
        int s = bqg_rekey_mu8(L->d_keys, L->m, L->n, L->beta, L->mu, k8, L->stream);
        cudaError_t e = s ? cudaSuccess
                          : bqg::launch_tile_keys(k8, static_cast<long long>(L->m), static_cast<long long>(g8),
                                                  static_cast<int>(L->beta), L->d_tiled, L->stream);
        cudaError_t e2 = cudaStreamSynchronize(L->stream);
        cudaFree(k8);
        if (s) return s;
        if (e != cudaSuccess) return cuda_err(e, "tile_keys kernel");
        if (e2 != cudaSuccess) return cuda_err(e2, "rekey");
    }
    BQG_CUDA(cudaStreamSynchronize(L->stream));
    return BQG_OK;
}

int layer_from_device_weights(const float* d_w, size_t m, size_t n, unsigned beta, unsigned mu, bqg_layer* L) {
    const size_t wpr = (n + 31) / 32;
    BQG_CUDA(cudaMalloc(reinterpret_cast<void**>(&L->d_planes), sizeof(uint32_t) * beta * m * wpr));
    int s = bqg_quantize_greedy_f32(d_w, m, n, beta, L->d_planes, L->d_alpha, L->stream);
    if (s) return s;
    for (unsigned i = 0; i < beta; ++i) {
        s = bqg_pack_keys(L->d_planes + size_t(i) * m * wpr, m, n, mu,
                          static_cast<char*>(L->d_keys) + L->key_bytes_per_plane() * i, L->stream);
        if (s) return s;
    }
    return layer_finish_tiling(L);
}

// Grow a library-owned device buffer.  The zero fill is queued on the stream
// that will use the buffer: the library's streams are non-blocking, so a
// legacy-stream cudaMemset is NOT ordered before their kernels and could land
// in the middle of (or after) the first call that uses the buffer -- seen as
// a wrong first result when another process shares the GPU.
template <typename P>
int grow(P*& ptr, size_t& cap, size_t need, cudaStream_t stream) {
    if (need <= cap) return BQG_OK;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    BQG_CUDA(cudaStreamIsCapturing(stream, &cs));
    if (cs != cudaStreamCaptureStatusNone)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "workspace growth while the stream is being captured: run the "
                                                 "call once before capturing it");
    if (ptr) BQG_CUDA(cudaStreamSynchronize(stream));  // queued work may still read the old buffer
    cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    BQG_CUDA(cudaMalloc(reinterpret_cast<void**>(&ptr), need));
    BQG_CUDA(cudaMemsetAsync(ptr, 0, need, stream));  // workspaces start zero-filled (grouped counters)
    cap = need;
    return BQG_OK;
}

}  // namespace

extern "C" int bqg_layer_create_from_device_weights(const float* d_w, size_t m, size_t n, unsigned beta, unsigned mu,
                                                    bqg_layer** out) {
    bqg_layer* L = nullptr;
    int s = layer_alloc(m, n, beta, mu, false, &L);
    if (s) return s;
    s = layer_from_device_weights(d_w, m, n, beta, mu, L);
    if (s) {
        layer_free(L);
        return s;
    }
    *out = L;
    return BQG_OK;
}

extern "C" int bqg_layer_create_from_weights(const float* h_w, size_t m, size_t n, unsigned beta, unsigned mu,
                                             bqg_layer** out) {
    if (!h_w) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null weights");
    bqg_layer* L = nullptr;
    int s = layer_alloc(m, n, beta, mu, false, &L);
    if (s) return s;
    float* d_w = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&d_w), sizeof(float) * m * n);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_w, h_w, sizeof(float) * m * n, cudaMemcpyHostToDevice, L->stream);
    if (e != cudaSuccess) {
        cudaFree(d_w);
        layer_free(L);
        return cuda_err(e, "layer weights upload");
    }
    s = layer_from_device_weights(d_w, m, n, beta, mu, L);
    cudaStreamSynchronize(L->stream);
    cudaFree(d_w);
    if (s) {
        layer_free(L);
        return s;
    }
    *out = L;
    return BQG_OK;
}

extern "C" int bqg_layer_create_from_keys(const void* h_keys, const float* h_alpha, size_t m, size_t n,
                                          unsigned beta, unsigned mu, bqg_layer** out) {
    if (!h_keys) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null keys");
    {
        int s = check_mu(mu, "pack_linear");
        if (s) return s;
    }
    // Keys index 2^mu-entry tables: reject out-of-range keys up front
    // (model_io.cpp:130-132 does the same for loaded files).
    const size_t G = groups_of(n, mu);
    const size_t count = size_t(beta) * m * G;
    const uint32_t limit = 1u << mu;
    for (size_t k = 0; k < count; ++k) {
        const uint32_t v = mu > 8 ? static_cast<const uint16_t*>(h_keys)[k] : static_cast<const uint8_t*>(h_keys)[k];
        if (v >= limit) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: key %u out of range for mu=%u", v, mu);
    }
    bqg_layer* L = nullptr;
    int s = layer_alloc(m, n, beta, mu, h_alpha == nullptr, &L);
    if (s) return s;
    cudaError_t e = cudaMemcpyAsync(L->d_keys, h_keys, L->key_bytes_per_plane() * beta, cudaMemcpyHostToDevice,
                                    L->stream);
    if (e == cudaSuccess && h_alpha)
        e = cudaMemcpyAsync(L->d_alpha, h_alpha, sizeof(float) * beta * m, cudaMemcpyHostToDevice, L->stream);
    if (e != cudaSuccess) {
        layer_free(L);
        return cuda_err(e, "layer upload");
    }
    s = layer_finish_tiling(L);
    if (s) {
        layer_free(L);
        return s;
    }
    *out = L;
    return BQG_OK;
}

extern "C" int bqg_layer_load_bqgm(const uint8_t* bytes, size_t len, bqg_layer** out) {
    size_t m, n;
    unsigned beta, mu;
    int s = bqg_bqgm_parse(bytes, len, &m, &n, &beta, &mu, nullptr, nullptr);
    if (s) return s;
    const size_t G = groups_of(n, mu);
    std::vector<float> alpha(size_t(beta) * m);
    std::vector<uint8_t> keys(size_t(beta) * m * G * (mu > 8 ? 2 : 1));
    s = bqg_bqgm_parse(bytes, len, &m, &n, &beta, &mu, alpha.data(), keys.data());
    if (s) return s;
    return bqg_layer_create_from_keys(keys.data(), alpha.data(), m, n, beta, mu, out);
}

extern "C" void bqg_layer_destroy(bqg_layer* layer) { layer_free(layer); }

extern "C" int bqg_layer_shape(const bqg_layer* L, size_t* m, size_t* n, unsigned* beta, unsigned* mu) {
    if (!L) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null");
    if (m) *m = L->m;
    if (n) *n = L->n;
    if (beta) *beta = L->beta;
    if (mu) *mu = L->mu;
    return BQG_OK;
}

extern "C" int bqg_layer_export(const bqg_layer* L, void* h_keys, float* h_alpha, uint32_t* h_planes) {
    if (!L) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null");
    if (h_keys) BQG_CUDA(cudaMemcpy(h_keys, L->d_keys, L->key_bytes_per_plane() * L->beta, cudaMemcpyDeviceToHost));
    if (h_alpha) {
        if (L->d_alpha) {
            BQG_CUDA(cudaMemcpy(h_alpha, L->d_alpha, sizeof(float) * L->beta * L->m, cudaMemcpyDeviceToHost));
        } else {
            for (size_t i = 0; i < size_t(L->beta) * L->m; ++i) h_alpha[i] = 1.0f;
        }
    }
    if (h_planes) {
        if (!L->d_planes) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: no sign planes (created from keys)");
        BQG_CUDA(cudaMemcpy(h_planes, L->d_planes, sizeof(uint32_t) * L->beta * L->m * ((L->n + 31) / 32),
                            cudaMemcpyDeviceToHost));
    }
    return BQG_OK;
}

extern "C" int bqg_layer_fast_shape(const bqg_layer* L, size_t* n_fast, unsigned* mu_fast) {
    if (!L) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null");
    if (n_fast) *n_fast = L->fn;
    if (mu_fast) *mu_fast = L->fmu;
    return BQG_OK;
}
extern "C" const uint8_t* bqg_layer_device_tiled_keys(const bqg_layer* L) { return L ? L->d_tiled : nullptr; }
extern "C" const void* bqg_layer_device_keys(const bqg_layer* L) { return L ? L->d_keys : nullptr; }
extern "C" const float* bqg_layer_device_alpha(const bqg_layer* L) { return L ? L->d_alpha : nullptr; }

namespace {

// Columns of the fast view a call with x_rows input rows needs: mu <= 8 ->
// n; mu > 8 -> 8*ceil(n/8) when x reaches no further (its groups are a prefix
// of the re-keyed tiling: blocks are the layout's outer index), else the
// whole re-keyed width (x rows past n meet the pad bits' sign).  A call
// covering n keeps the group blocks a mu = 8 layer of n columns has (C2:
// 16, the latency form's shape) instead of one more nearly empty block.
size_t fast_columns(const bqg_layer* L, size_t x_rows) {
    if (L->fmu == L->mu) return L->n;
    const size_t n8 = 8 * ((L->n + 7) / 8);
    return x_rows <= n8 ? n8 : L->fn;
}

// exact: BQG_FORWARD_FAST (0), BQG_FORWARD_EXACT (fp64 DP tables) or
// BQG_FORWARD_EXACT_NAIVE (fp64 naive tables: KernelOptions::builder = Naive,
// kernel.hpp:51,158).  xstats (exact path only) receives the exact path's
// counters and build/query/replace split; it synchronises the stream.
int layer_forward(bqg_layer* L, const float* d_x, size_t x_rows, size_t b, float* d_y, int exact, int pdl,
                  cudaStream_t st, bqg_kernel_stats* xstats = nullptr) {
    if (exact) {
        const size_t need = bqg_biqgemm_exact_workspace_bytes(L->m, L->n, b, L->beta, L->mu);
        if (need > L->ws_exact_bytes) ++L->buf_gen;
        int s = grow(L->d_ws_exact, L->ws_exact_bytes, need, st);
        if (s) return s;
        return biqgemm_exact_impl<float>(L->d_keys, L->d_alpha, d_x, x_rows, d_y, L->m, L->n, b, L->beta, L->mu,
                                         exact == BQG_FORWARD_EXACT_NAIVE ? BQG_LUT_NAIVE : BQG_LUT_DP,
                                         L->d_ws_exact, L->ws_exact_bytes, xstats, st);
    }
    // the fast view (mu > 8: the re-keyed mu = 8 tiles over fn >= G*mu columns)
    const size_t fn = fast_columns(L, x_rows);
    const size_t need = bqg_biqgemm_workspace_bytes(L->m, fn, b, L->beta, L->fmu);
    if (need > L->ws_bytes) {
        ++L->buf_gen;
        int s = grow(L->d_ws, L->ws_bytes, need, st);
        if (s) return s;
    }
    return bqg_biqgemm_f32(L->d_tiled, L->d_alpha, d_x, x_rows, d_y, L->m, fn, b, L->beta, L->fmu, L->d_ws,
                           L->ws_bytes, pdl, st);
}

}  // namespace

extern "C" int bqg_layer_forward_device(bqg_layer* L, const float* d_x, size_t x_rows, size_t b, float* d_y,
                                        int exact, int pdl, void* stream) {
    if (!L) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null");
    int s = check_x(x_rows, b, L->n, L->mu, "biqgemm");
    if (s) return s;
    std::lock_guard<std::mutex> g(L->mu_lock);
    return layer_forward(L, d_x, x_rows, b, d_y, exact, pdl, as_stream(stream));
}

namespace {
bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}
template <typename P>
int grow_host(P*& ptr, size_t& cap, size_t need) {
    if (need <= cap) return BQG_OK;
    cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
    BQG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ptr), need, cudaHostAllocDefault));
    cap = need;
    return BQG_OK;
}
}  // namespace

extern "C" int bqg_layer_forward_host(bqg_layer* L, const float* h_x, size_t x_rows, size_t b, float* h_y,
                                      int exact, bqg_kernel_stats* stats) {
    if (!L || !h_x || !h_y) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: null argument");
    int s = check_x(x_rows, b, L->n, L->mu, "biqgemm");
    if (s) return s;
    std::lock_guard<std::mutex> g(L->mu_lock);
    const size_t xbytes = sizeof(float) * x_rows * b, ybytes = sizeof(float) * L->m * b;
    if (xbytes > L->x_cap || ybytes > L->y_cap || xbytes > L->hx_cap || ybytes > L->hy_cap) ++L->buf_gen;
    s = grow(L->d_x, L->x_cap, xbytes, L->stream);
    if (s) return s;
    s = grow(L->d_y, L->y_cap, ybytes, L->stream);
    if (s) return s;
    // Steady state (no stats requested): the caller's x is copied into the
    // layer's pinned staging, one cached CUDA graph runs H2D -> kernels ->
    // D2H, and y is copied out -- one API launch per call instead of five.
    if (!stats) {
        const bool same = L->g_xrows == x_rows && L->g_b == b && L->g_exact == exact && L->g_gen == L->buf_gen;
        if (!same) {
            if (L->gexec) cudaGraphExecDestroy(L->gexec);
            L->gexec = nullptr;
            L->g_xrows = x_rows;
            L->g_b = b;
            L->g_exact = exact;
            L->g_gen = L->buf_gen;
            L->g_seen = 0;
        }
        s = grow_host(L->h_x_pin, L->hx_cap, xbytes);
        if (s) return s;
        s = grow_host(L->h_y_pin, L->hy_cap, ybytes);
        if (s) return s;
        std::memcpy(L->h_x_pin, h_x, xbytes);
        cudaStream_t st = L->stream;
        if (!L->gexec && L->g_seen >= 1) {  // second call of this shape: capture
            cudaGraph_t graph = nullptr;
            BQG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            cudaError_t e = cudaMemcpyAsync(L->d_x, L->h_x_pin, xbytes, cudaMemcpyHostToDevice, st);
            int fs = e == cudaSuccess ? layer_forward(L, L->d_x, x_rows, b, L->d_y, exact, 0, st) : BQG_OK;
            if (e == cudaSuccess && fs == BQG_OK)
                e = cudaMemcpyAsync(L->h_y_pin, L->d_y, ybytes, cudaMemcpyDeviceToHost, st);
            cudaError_t e2 = cudaStreamEndCapture(st, &graph);
            if (fs) {
                if (graph) cudaGraphDestroy(graph);
                return fs;
            }
            if (e != cudaSuccess || e2 != cudaSuccess) {
                if (graph) cudaGraphDestroy(graph);
                return cuda_err(e != cudaSuccess ? e : e2, "forward graph capture");
            }
            e = cudaGraphInstantiate(&L->gexec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) return cuda_err(e, "forward graph instantiate");
        }
        if (L->gexec) {
            BQG_CUDA(cudaGraphLaunch(L->gexec, st));
        } else {
            BQG_CUDA(cudaMemcpyAsync(L->d_x, L->h_x_pin, xbytes, cudaMemcpyHostToDevice, st));
            s = layer_forward(L, L->d_x, x_rows, b, L->d_y, exact, 0, st);
            if (s) return s;
            BQG_CUDA(cudaMemcpyAsync(L->h_y_pin, L->d_y, ybytes, cudaMemcpyDeviceToHost, st));
            ++L->g_seen;
        }
        BQG_CUDA(cudaStreamSynchronize(st));
        std::memcpy(h_y, L->h_y_pin, ybytes);
        return BQG_OK;
    }
    // With stats: the same work step by step, event-timed.  Pageable caller
    // buffers are staged through the layer's pinned buffers.
    const bool xpin = is_pinned(h_x), ypin = is_pinned(h_y);
    if (!xpin) {
        s = grow_host(L->h_x_pin, L->hx_cap, xbytes);
        if (s) return s;
        std::memcpy(L->h_x_pin, h_x, xbytes);
    }
    if (!ypin) {
        s = grow_host(L->h_y_pin, L->hy_cap, ybytes);
        if (s) return s;
    }
    cudaStream_t st = L->stream;
    if (stats) BQG_CUDA(cudaEventRecord(L->ev[0], st));
    BQG_CUDA(cudaMemcpyAsync(L->d_x, xpin ? h_x : L->h_x_pin, xbytes, cudaMemcpyHostToDevice, st));
    if (stats) BQG_CUDA(cudaEventRecord(L->ev[1], st));
    const bool exact_path = exact != 0;
    bqg_kernel_stats xs{};
    s = layer_forward(L, L->d_x, x_rows, b, L->d_y, exact, 0, st, exact_path ? &xs : nullptr);
    if (s) return s;
    if (stats) BQG_CUDA(cudaEventRecord(L->ev[2], st));
    BQG_CUDA(cudaMemcpyAsync(ypin ? h_y : L->h_y_pin, L->d_y, ybytes, cudaMemcpyDeviceToHost, st));
    if (stats) BQG_CUDA(cudaEventRecord(L->ev[3], st));
    BQG_CUDA(cudaStreamSynchronize(st));
    if (!ypin) std::memcpy(h_y, L->h_y_pin, ybytes);
    if (stats) {
        float t01 = 0, t12 = 0, t23 = 0;
        cudaEventElapsedTime(&t01, L->ev[0], L->ev[1]);
        cudaEventElapsedTime(&t12, L->ev[1], L->ev[2]);
        cudaEventElapsedTime(&t23, L->ev[2], L->ev[3]);
        if (exact_path) {
            // separate build / query kernels: the reference's phase split
            stats->lut_build_ops += xs.lut_build_ops;
            stats->lookups += xs.lookups;
            stats->accumulate_ops += xs.accumulate_ops;
            stats->fma_ops += xs.fma_ops;
            stats->build_seconds += xs.build_seconds;
            stats->query_seconds += xs.query_seconds;
            stats->replace_seconds += xs.replace_seconds;
        } else {
            // fast path: the LUT build runs inside the query kernel (builder
            // warps overlap the gather), so its time is part of query_seconds
            uint64_t ops[4];
            bqg_op_counters(L->m, L->n, b, L->beta, L->mu, BQG_LUT_DP, ops);
            stats->lut_build_ops += ops[0];
            stats->lookups += ops[1];
            stats->accumulate_ops += ops[2];
            stats->fma_ops += ops[3];
            stats->query_seconds += t12 * 1e-3;
        }
        stats->replace_seconds += (t01 + t23) * 1e-3;
    }
    return BQG_OK;
}

namespace {
// Process-wide per-device context for grouped host calls: a stream, event
// pairs and grown-on-demand staging/workspace buffers, so a group's call does
// not depend on which layer comes first.
struct GroupContext {
    std::mutex lock;
    cudaStream_t stream = nullptr;  // kernels
    cudaStream_t copy = nullptr;    // H2D
    cudaStream_t down = nullptr;    // D2H
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> chunk_ev;  // 2 per sub-group (H2D landed, kernels done), grown on demand
    float* d_x = nullptr;
    size_t x_cap = 0;
    float* d_y = nullptr;
    size_t y_cap = 0;
    void* d_ws = nullptr;
    size_t ws_cap = 0;
    cudaEvent_t fork = nullptr, join_cp = nullptr, join_dp = nullptr;  // the three streams as one capturable unit
    // Captured pipelines (H2D -> grouped kernels -> D2H), replayed as one
    // graph launch when the same layers, host buffers and shape recur (the
    // steady state of a serving loop).  Keyed by layer uids (not addresses)
    // and by the context's device buffers (a regrow invalidates).
    struct Captured {
        std::vector<uint64_t> uids;
        const float* h_x = nullptr;
        float* h_y = nullptr;
        size_t x_rows = 0, b = 0;
        const void *d_x = nullptr, *d_y = nullptr, *d_ws = nullptr;
        int seen = 0;
        cudaGraphExec_t exec = nullptr;
    };
    std::vector<Captured> captured;  // most recent last, at most kMaxCaptured
};
constexpr size_t kMaxCaptured = 8;
GroupContext g_group_ctx[16];
}  // namespace

extern "C" int bqg_layers_forward_host(bqg_layer* const* layers, size_t count, const float* h_x, size_t x_rows,
                                       size_t b, float* h_y, int exact, bqg_kernel_stats* stats) {
    if (!layers || !h_x || !h_y) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: null argument");
    if (count == 0) return BQG_OK;
    bqg_layer* L0 = layers[0];
    if (!L0) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null");
    for (size_t i = 1; i < count; ++i) {
        const bqg_layer* L = layers[i];
        if (!L) return set_err(BQG_ERR_INVALID_ARGUMENT, "layer: null");
        // kernel.hpp:127-131: every call of the group has the same shape
        if (L->m != L0->m || L->n != L0->n || L->beta != L0->beta || L->mu != L0->mu)
            return set_err(BQG_ERR_INVALID_ARGUMENT, "layers_forward: layers must share (m, n, beta, mu)");
    }
    int s = check_x(x_rows, b, L0->n, L0->mu, "biqgemm");
    if (s) return s;
    if (exact) {
        for (size_t i = 0; i < count; ++i) {
            s = bqg_layer_forward_host(layers[i], h_x + i * x_rows * b, x_rows, b, h_y + i * L0->m * b, exact, stats);
            if (s) return s;
        }
        return BQG_OK;
    }
    int dev = 0;
    BQG_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 16) return set_err(BQG_ERR_INVALID_ARGUMENT, "layers_forward: device index >= 16");
    GroupContext& G = g_group_ctx[dev];
    std::lock_guard<std::mutex> g(G.lock);
    if (!G.stream) {
        BQG_CUDA(cudaStreamCreateWithFlags(&G.stream, cudaStreamNonBlocking));
        BQG_CUDA(cudaStreamCreateWithFlags(&G.copy, cudaStreamNonBlocking));
        BQG_CUDA(cudaStreamCreateWithFlags(&G.down, cudaStreamNonBlocking));
        for (auto& e : G.ev) BQG_CUDA(cudaEventCreate(&e));
        BQG_CUDA(cudaEventCreateWithFlags(&G.fork, cudaEventDisableTiming));
        BQG_CUDA(cudaEventCreateWithFlags(&G.join_cp, cudaEventDisableTiming));
        BQG_CUDA(cudaEventCreateWithFlags(&G.join_dp, cudaEventDisableTiming));
    }
    const size_t xs = x_rows * b, ys = L0->m * b;
    s = grow(G.d_x, G.x_cap, sizeof(float) * xs * count, G.stream);
    if (s) return s;
    s = grow(G.d_y, G.y_cap, sizeof(float) * ys * count, G.stream);
    if (s) return s;
    // Pipelined in sub-groups: the H2D of sub-group k+1 (copy stream) and the
    // D2H of sub-group k-1 (down stream) overlap the kernels of sub-group k
    // (compute stream); consecutive grouped launches are PDL-chained.  The
    // sub-groups ramp up (each H2D lands while the previous, half-size
    // sub-group computes) to kSub calls (grouped-launch efficiency) and ramp
    // down at the end (the last D2H is short) when there is room.  Sizes
    // follow the calls' host I/O: the first sub-group moves ~2 MiB of x + y,
    // the steady ones ~8 MiB (C2: 64 -> 128 -> 256 ... 256 -> 128 -> 64 calls,
    // measured best of 16/32/64 x 128/256; a b = 256 call is its own
    // sub-group).  y is the same as one grouped call.
    size_t kFirst, kSub;
    {
        static const long long e_first = [] {
            const char* e = getenv("BQG_E2E_FIRST");
            return e ? atoll(e) : 0LL;
        }();
        static const long long e_sub = [] {
            const char* e = getenv("BQG_E2E_SUB");
            return e ? atoll(e) : 0LL;
        }();
        const size_t io = std::max<size_t>(1, sizeof(float) * (xs + ys));  // host bytes per call
        kFirst = e_first > 0 ? static_cast<size_t>(e_first) : std::clamp<size_t>((2u << 20) / io, 1, 64);
        kSub = e_sub > 0 ? static_cast<size_t>(e_sub) : std::clamp<size_t>((8u << 20) / io, 1, 256);
    }
    std::vector<size_t> starts{0};
    static const std::vector<size_t> e_sched = [] {  // BQG_E2E_SCHEDULE="16,48,...": tuning runs only
        std::vector<size_t> v;
        const char* e = getenv("BQG_E2E_SCHEDULE");
        while (e && *e) {
            const long long k = atoll(e);
            if (k > 0) v.push_back(static_cast<size_t>(k));
            e = strchr(e, ',');
            if (e) ++e;
        }
        return v;
    }();
    if (!e_sched.empty()) {
        size_t rem = count;
        for (size_t i = 0; rem; ++i) {
            const size_t c = std::min(rem, e_sched[std::min(i, e_sched.size() - 1)]);
            starts.push_back(starts.back() + c);
            rem -= c;
        }
        kSub = std::max(kSub, *std::max_element(e_sched.begin(), e_sched.end()));
    } else {
        size_t rem = count;
        auto take = [&](size_t c) {
            c = std::min(c, rem);
            if (c) starts.push_back(starts.back() + c), rem -= c;
        };
        for (size_t sz = kFirst; sz < kSub && rem; sz *= 2) take(sz);
        std::vector<size_t> down;
        size_t dsum = 0;
        for (size_t sz = kFirst; sz < kSub; sz *= 2) down.push_back(sz), dsum += sz;
        if (rem >= dsum + kSub) {
            while (rem > dsum) take(std::min(kSub, rem - dsum));
            for (auto it = down.rbegin(); it != down.rend(); ++it) take(*it);
        }
        while (rem) take(kSub);
    }
    const size_t nsub = starts.size() - 1;
    while (G.chunk_ev.size() < 2 * nsub) {
        cudaEvent_t e;
        BQG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        G.chunk_ev.push_back(e);
    }
    s = grow(G.d_ws, G.ws_cap,
             bqg_biqgemm_grouped_workspace_bytes(L0->m, fast_columns(L0, x_rows), b, L0->beta, L0->fmu,
                                                 std::min(count, kSub)),
             G.stream);
    if (s) return s;
    std::vector<bqg_call> calls(count);
    for (size_t i = 0; i < count; ++i) calls[i] = {layers[i]->d_tiled, layers[i]->d_alpha, G.d_x + i * xs, G.d_y + i * ys};
    cudaStream_t st = G.stream, cp = G.copy, dp = G.down;
    // The pipeline forks from the kernel stream and joins back into it, so
    // it can be captured as one graph.  Everything queued reads h_x and
    // writes h_y: on an error part-way the queued copies must land before
    // control returns (the caller may free or reuse its host buffers, and the
    // next call may regrow G.d_x / G.d_y).
    auto enqueue = [&]() -> int {
        BQG_CUDA(cudaEventRecord(G.fork, st));
        BQG_CUDA(cudaStreamWaitEvent(cp, G.fork, 0));
        BQG_CUDA(cudaStreamWaitEvent(dp, G.fork, 0));
        if (stats) BQG_CUDA(cudaEventRecord(G.ev[0], cp));
        // all H2D copies are queued first (the copy stream runs ahead of the kernels)
        for (size_t k = 0; k < nsub; ++k) {
            const size_t i0 = starts[k], cnt = starts[k + 1] - i0;
            BQG_CUDA(cudaMemcpyAsync(G.d_x + i0 * xs, h_x + i0 * xs, sizeof(float) * xs * cnt, cudaMemcpyHostToDevice, cp));
            BQG_CUDA(cudaEventRecord(G.chunk_ev[2 * k], cp));
        }
        for (size_t k = 0; k < nsub; ++k) {
            const size_t i0 = starts[k], cnt = starts[k + 1] - i0;
            cudaEvent_t h2d = G.chunk_ev[2 * k], done = G.chunk_ev[2 * k + 1];
            BQG_CUDA(cudaStreamWaitEvent(st, h2d, 0));
            if (stats && k == 0) BQG_CUDA(cudaEventRecord(G.ev[1], st));
            const int rc = bqg_biqgemm_grouped_f32(calls.data() + i0, cnt, x_rows, L0->m, fast_columns(L0, x_rows), b,
                                                   L0->beta, L0->fmu,
                                                   G.d_ws, G.ws_cap, k > 0 ? 1 : 0, st);
            if (rc) return rc;
            BQG_CUDA(cudaEventRecord(done, st));
            BQG_CUDA(cudaStreamWaitEvent(dp, done, 0));
            BQG_CUDA(cudaMemcpyAsync(h_y + i0 * ys, G.d_y + i0 * ys, sizeof(float) * ys * cnt, cudaMemcpyDeviceToHost, dp));
        }
        if (stats) {
            BQG_CUDA(cudaEventRecord(G.ev[2], st));
            BQG_CUDA(cudaEventRecord(G.ev[3], dp));
        }
        BQG_CUDA(cudaEventRecord(G.join_cp, cp));
        BQG_CUDA(cudaEventRecord(G.join_dp, dp));
        BQG_CUDA(cudaStreamWaitEvent(st, G.join_cp, 0));
        BQG_CUDA(cudaStreamWaitEvent(st, G.join_dp, 0));
        return BQG_OK;
    };
    auto drain = [&](int rc) {
        cudaStreamSynchronize(cp);  // status ignored: rc is the error reported
        cudaStreamSynchronize(st);
        cudaStreamSynchronize(dp);
        return rc;
    };
    // Replay a captured pipeline when this exact call recurs (no stats,
    // pinned caller buffers: graph memcpy nodes need page-locked memory).
    GroupContext::Captured* cap = nullptr;
    if (!stats && is_pinned(h_x) && is_pinned(h_y)) {
        for (auto& c : G.captured) {
            if (c.h_x != h_x || c.h_y != h_y || c.x_rows != x_rows || c.b != b || c.uids.size() != count) continue;
            bool same = c.d_x == G.d_x && c.d_y == G.d_y && c.d_ws == G.d_ws;
            for (size_t i = 0; same && i < count; ++i) same = c.uids[i] == layers[i]->uid;
            if (same) {
                cap = &c;
                break;
            }
            if (c.exec && !(c.d_x == G.d_x && c.d_y == G.d_y && c.d_ws == G.d_ws)) {  // stale device buffers
                cudaGraphExecDestroy(c.exec);
                c.exec = nullptr;
                c.seen = 0;
            }
        }
        if (!cap) {
            if (G.captured.size() >= kMaxCaptured) {
                if (G.captured.front().exec) cudaGraphExecDestroy(G.captured.front().exec);
                G.captured.erase(G.captured.begin());
            }
            GroupContext::Captured c;
            c.uids.resize(count);
            for (size_t i = 0; i < count; ++i) c.uids[i] = layers[i]->uid;
            c.h_x = h_x;
            c.h_y = h_y;
            c.x_rows = x_rows;
            c.b = b;
            c.d_x = G.d_x;
            c.d_y = G.d_y;
            c.d_ws = G.d_ws;
            G.captured.push_back(std::move(c));
            cap = &G.captured.back();
        }
        if (!cap->exec && cap->seen >= 1) {  // second occurrence: capture once
            cudaGraph_t graph = nullptr;
            BQG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            const int rc = enqueue();
            const cudaError_t ee = cudaStreamEndCapture(st, &graph);
            if (rc == BQG_OK && ee == cudaSuccess && graph) {
                if (cudaGraphInstantiate(&cap->exec, graph, 0) != cudaSuccess) cap->exec = nullptr;
            }
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            if (rc) return drain(rc);
        }
        ++cap->seen;
        if (cap->exec) {
            BQG_CUDA(cudaGraphLaunch(cap->exec, st));
            const cudaError_t se = cudaStreamSynchronize(st);
            if (se != cudaSuccess) return drain(cuda_err(se, "layers_forward graph"));
            return BQG_OK;
        }
    }
    s = enqueue();
    if (s) return drain(s);
    {
        const cudaError_t se = cudaStreamSynchronize(st);
        if (se != cudaSuccess) return drain(cuda_err(se, "layers_forward"));
    }
    if (stats) {
        uint64_t ops[4];
        bqg_op_counters(L0->m, L0->n, b, L0->beta, L0->mu, BQG_LUT_DP, ops);
        stats->lut_build_ops += ops[0] * count;
        stats->lookups += ops[1] * count;
        stats->accumulate_ops += ops[2] * count;
        stats->fma_ops += ops[3] * count;
        float t01 = 0, t12 = 0, t03 = 0;
        cudaEventElapsedTime(&t01, G.ev[0], G.ev[1]);
        cudaEventElapsedTime(&t12, G.ev[1], G.ev[2]);
        cudaEventElapsedTime(&t03, G.ev[0], G.ev[3]);
        stats->query_seconds += t12 * 1e-3;
        stats->replace_seconds += (t03 - t12 > 0 ? t03 - t12 : 0) * 1e-3;
    }
    return BQG_OK;
}

// ============================================================ multi-GPU
// Row sharding (north_star): rank r owns output rows
// [r*R, min(m, (r+1)*R)), R = 32*ceil(ceil(m/32)/nranks).  Row tiles never
// straddle ranks, so every output's reduction tree -- and y -- is bitwise
// identical for any number of ranks, and with EQUAL blocks the all-gathered
// buffer's first m*b floats are y (m x b row-major) with no compaction.
// The reference partitions rows the same way across its worker threads
// (kernel.hpp:80-82,162-176).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): the library has no
// link-time NCCL dependency, and inside a PyTorch process it shares the NCCL
// torch already loaded.

#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi& nccl() {
    std::call_once(g_nccl_once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            g_nccl.why = dlerror() ? dlerror() : "libnccl.so.2 not found";
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(sym("ncclGetUniqueId"));
        g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(sym("ncclCommInitRank"));
        g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(sym("ncclCommDestroy"));
        g_nccl.CommGetAsyncError = reinterpret_cast<decltype(g_nccl.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
        g_nccl.Broadcast = reinterpret_cast<decltype(g_nccl.Broadcast)>(sym("ncclBroadcast"));
        g_nccl.AllGather = reinterpret_cast<decltype(g_nccl.AllGather)>(sym("ncclAllGather"));
        g_nccl.GetErrorString = reinterpret_cast<decltype(g_nccl.GetErrorString)>(sym("ncclGetErrorString"));
        g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.Broadcast &&
                    g_nccl.AllGather && g_nccl.GetErrorString && g_nccl.CommGetAsyncError;
        if (!g_nccl.ok) g_nccl.why = "libnccl.so.2 lacks an expected symbol";
    });
    return g_nccl;
}

int nccl_err(ncclResult_t r, const char* what) {
    return set_err(BQG_ERR_COMM, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
}

int nccl_bcast(void* ctx, void* d_buf, size_t bytes, int root, void* stream) {
    const ncclResult_t r = nccl().Broadcast(d_buf, d_buf, bytes, ncclUint8, root, static_cast<ncclComm_t>(ctx),
                                            as_stream(stream));
    return r == ncclSuccess ? BQG_OK : nccl_err(r, "ncclBroadcast");
}

int nccl_allgather(void* ctx, const void* d_send, void* d_recv, size_t bytes_per_rank, void* stream) {
    const ncclResult_t r = nccl().AllGather(d_send, d_recv, bytes_per_rank, ncclUint8, static_cast<ncclComm_t>(ctx),
                                            as_stream(stream));
    return r == ncclSuccess ? BQG_OK : nccl_err(r, "ncclAllGather");
}

}  // namespace

extern "C" int bqg_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int bqg_nccl_unique_id(void* h_id) {
    if (!h_id) return set_err(BQG_ERR_INVALID_ARGUMENT, "nccl_unique_id: null pointer");
    if (!nccl().ok) return set_err(BQG_ERR_COMM, "NCCL unavailable: %s", nccl().why.c_str());
    ncclUniqueId id;
    const ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_err(r, "ncclGetUniqueId");
    std::memcpy(h_id, &id, sizeof(id));
    return BQG_OK;
}

extern "C" int bqg_nccl_comm_init(const void* h_id, int nranks, int rank, void** comm_out) {
    if (!h_id || !comm_out) return set_err(BQG_ERR_INVALID_ARGUMENT, "nccl_comm_init: null pointer");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "nccl_comm_init: rank %d of %d", rank, nranks);
    if (!nccl().ok) return set_err(BQG_ERR_COMM, "NCCL unavailable: %s", nccl().why.c_str());
    BQG_NEED_DEVICE();
    ncclUniqueId id;
    std::memcpy(&id, h_id, sizeof(id));
    ncclComm_t c = nullptr;
    const ncclResult_t r = nccl().CommInitRank(&c, nranks, id, rank);  // on the current device
    if (r != ncclSuccess) return nccl_err(r, "ncclCommInitRank");
    *comm_out = c;
    return BQG_OK;
}

extern "C" int bqg_nccl_comm_destroy(void* comm) {
    if (!comm) return BQG_OK;
    if (!nccl().ok) return set_err(BQG_ERR_COMM, "NCCL unavailable: %s", nccl().why.c_str());
    const ncclResult_t r = nccl().CommDestroy(static_cast<ncclComm_t>(comm));
    return r == ncclSuccess ? BQG_OK : nccl_err(r, "ncclCommDestroy");
}

extern "C" int bqg_nccl_collectives(void* comm, bqg_collectives* out) {
    if (!comm || !out) return set_err(BQG_ERR_INVALID_ARGUMENT, "nccl_collectives: null pointer");
    if (!nccl().ok) return set_err(BQG_ERR_COMM, "NCCL unavailable: %s", nccl().why.c_str());
    out->ctx = comm;
    out->broadcast = nccl_bcast;
    out->allgather = nccl_allgather;
    return BQG_OK;
}

extern "C" int bqg_shard_rows(size_t m, int nranks, int rank, size_t* row_begin, size_t* row_end,
                              size_t* rows_per_rank) {
    if (m == 0 || nranks < 1 || rank < 0 || rank >= nranks)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "shard_rows: m %zu, rank %d of %d", m, rank, nranks);
    const size_t tiles = (m + 31) / 32;
    const size_t R = 32 * ((tiles + static_cast<size_t>(nranks) - 1) / static_cast<size_t>(nranks));
    if (row_begin) *row_begin = std::min(m, static_cast<size_t>(rank) * R);
    if (row_end) *row_end = std::min(m, static_cast<size_t>(rank + 1) * R);
    if (rows_per_rank) *rows_per_rank = R;
    return BQG_OK;
}

extern "C" size_t bqg_biqgemm_sharded_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                                      int nranks) {
    size_t R = 0;
    if (bqg_shard_rows(m, nranks, 0, nullptr, nullptr, &R) != BQG_OK) return 0;
    return bqg_biqgemm_workspace_bytes(std::min(R, m), n, b, beta, mu);
}

extern "C" int bqg_biqgemm_sharded_f32(const uint8_t* d_keys_tiled_shard, const float* d_alpha_shard, float* d_x,
                                       size_t x_rows, float* d_y_gather, size_t m, size_t n, size_t b,
                                       unsigned beta, unsigned mu, int rank, int nranks,
                                       const bqg_collectives* coll, void* d_ws, size_t ws_bytes, void* stream) {
    size_t lo = 0, hi = 0, R = 0;
    int s = bqg_shard_rows(m, nranks, rank, &lo, &hi, &R);
    if (s) return s;
    if (!coll || !coll->broadcast || !coll->allgather)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: collectives missing");
    if (!d_x || !d_y_gather) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null pointer");
    s = check_x(x_rows, b, n, mu, "biqgemm");
    if (s) return s;
    // 1. x from rank 0 to every rank (in place; a 1-rank group runs it too,
    //    so the collective path is exercised on a single GPU)
    s = coll->broadcast(coll->ctx, d_x, x_rows * b * sizeof(float), 0, stream);
    if (s) return s;
    // 2. this rank's rows into its block of the gather buffer
    float* y_mine = d_y_gather + static_cast<size_t>(rank) * R * b;
    if (hi > lo) {
        s = bqg_biqgemm_f32(d_keys_tiled_shard, d_alpha_shard, d_x, x_rows, y_mine, hi - lo, n, b, beta, mu, d_ws,
                            ws_bytes, 0, stream);
        if (s) return s;
    }
    // 3. the row blocks to every rank: the buffer's first m*b floats are y
    return coll->allgather(coll->ctx, y_mine, d_y_gather, R * b * sizeof(float), stream);
}

extern "C" size_t bqg_biqgemm_grouped_sharded_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta,
                                                              unsigned mu, size_t count, int nranks) {
    size_t R = 0;
    if (bqg_shard_rows(m, nranks, 0, nullptr, nullptr, &R) != BQG_OK) return 0;
    return bqg_biqgemm_grouped_workspace_bytes(std::min(R, m), n, b, beta, mu, count);
}

extern "C" int bqg_biqgemm_grouped_sharded_f32(const bqg_shard_call* h_calls, size_t count, float* d_x, size_t x_rows,
                                               float* d_y_gather, size_t m, size_t n, size_t b, unsigned beta,
                                               unsigned mu, int rank, int nranks, const bqg_collectives* coll,
                                               void* d_ws, size_t ws_bytes, int pdl, void* stream) {
    size_t lo = 0, hi = 0, R = 0;
    int s = bqg_shard_rows(m, nranks, rank, &lo, &hi, &R);
    if (s) return s;
    if (!coll || !coll->broadcast || !coll->allgather)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: collectives missing");
    if (!d_x || !d_y_gather || (count && !h_calls))
        return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null pointer");
    s = check_x(x_rows, b, n, mu, "biqgemm");
    if (s) return s;
    if (count == 0) return BQG_OK;
    const size_t xs = x_rows * b, block = R * b;
    // 1. every call's x from rank 0, one broadcast of the contiguous batch
    s = coll->broadcast(coll->ctx, d_x, count * xs * sizeof(float), 0, stream);
    if (s) return s;
    // 2. the group on this rank's rows: call i -> block (rank, i) of the gather buffer
    float* y_mine = d_y_gather + static_cast<size_t>(rank) * count * block;
    if (hi > lo) {
        std::vector<bqg_call> calls(count);
        for (size_t i = 0; i < count; ++i) {
            if (!h_calls[i].d_keys_tiled_shard)
                return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null keys in call %zu", i);
            calls[i] = {h_calls[i].d_keys_tiled_shard, h_calls[i].d_alpha_shard, d_x + i * xs, y_mine + i * block};
        }
        s = bqg_biqgemm_grouped_f32(calls.data(), count, x_rows, hi - lo, n, b, beta, mu, d_ws, ws_bytes, pdl, stream);
        if (s) return s;
    }
    // 3. the rank blocks to every rank
    return coll->allgather(coll->ctx, y_mine, d_y_gather, count * block * sizeof(float), stream);
}

// ============================================================ fused all-gather over peer memory

namespace {
// cuMemGetAddressRange through the runtime's driver entry point (no link-time
// libcuda dependency): the base of the allocation that contains p.
int allocation_base(void* p, char** base) {
    using Fn = int (*)(unsigned long long*, size_t*, unsigned long long);
    static Fn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<Fn>(f);
        cudaGetLastError();
    });
    if (!fn) return set_err(BQG_ERR_CUDA, "ipc: cuMemGetAddressRange unavailable");
    unsigned long long b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "ipc: pointer is not in a device allocation");
    *base = reinterpret_cast<char*>(b);
    return BQG_OK;
}
}  // namespace

extern "C" int bqg_ipc_get_handle(void* d_ptr, void* h_handle, size_t* offset) {
    if (!d_ptr || !h_handle || !offset) return set_err(BQG_ERR_INVALID_ARGUMENT, "ipc_get_handle: null pointer");
    char* base = nullptr;
    int s = allocation_base(d_ptr, &base);
    if (s) return s;
    cudaIpcMemHandle_t hd;
    BQG_CUDA(cudaIpcGetMemHandle(&hd, base));
    static_assert(sizeof(hd) <= 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(h_handle, &hd, sizeof(hd));
    *offset = static_cast<size_t>(static_cast<char*>(d_ptr) - base);
    return BQG_OK;
}

extern "C" int bqg_ipc_open_handle(const void* h_handle, size_t offset, void** d_ptr) {
    if (!h_handle || !d_ptr) return set_err(BQG_ERR_INVALID_ARGUMENT, "ipc_open_handle: null pointer");
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, h_handle, sizeof(hd));
    void* base = nullptr;
    BQG_CUDA(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess));
    *d_ptr = static_cast<char*>(base) + offset;
    return BQG_OK;
}

extern "C" int bqg_ipc_close_handle(void* d_ptr) {
    if (!d_ptr) return BQG_OK;
    char* base = nullptr;
    int s = allocation_base(d_ptr, &base);
    if (s) return s;
    BQG_CUDA(cudaIpcCloseMemHandle(base));
    return BQG_OK;
}

namespace {
constexpr size_t kBarrierBytesPerRank = 16;
size_t barrier_offset(size_t grouped_ws) { return (grouped_ws + 255) & ~size_t(255); }
}  // namespace

extern "C" size_t bqg_biqgemm_grouped_sharded_p2p_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta,
                                                                  unsigned mu, size_t count, int nranks) {
    const size_t g = bqg_biqgemm_grouped_sharded_workspace_bytes(m, n, b, beta, mu, count, nranks);
    if (g == 0) return 0;
    return barrier_offset(g) + kBarrierBytesPerRank * static_cast<size_t>(nranks);
}

extern "C" int bqg_biqgemm_grouped_sharded_p2p_f32(const bqg_shard_call* h_calls, size_t count, float* d_x,
                                                   size_t x_rows, float* const* h_y_gather_peers, size_t m, size_t n,
                                                   size_t b, unsigned beta, unsigned mu, int rank, int nranks,
                                                   const bqg_collectives* coll, void* d_ws, size_t ws_bytes, int pdl,
                                                   void* stream) {
    size_t lo = 0, hi = 0, R = 0;
    int s = bqg_shard_rows(m, nranks, rank, &lo, &hi, &R);
    if (s) return s;
    if (!coll || !coll->broadcast || !coll->allgather)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: collectives missing");
    if (!d_x || !h_y_gather_peers || (count && !h_calls))
        return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null pointer");
    for (int r = 0; r < nranks; ++r)
        if (!h_y_gather_peers[r]) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null peer buffer %d", r);
    s = check_x(x_rows, b, n, mu, "biqgemm");
    if (s) return s;
    const size_t gws = bqg_biqgemm_grouped_sharded_workspace_bytes(m, n, b, beta, mu, std::max<size_t>(count, 1), nranks);
    if (!d_ws || ws_bytes < barrier_offset(gws) + kBarrierBytesPerRank * static_cast<size_t>(nranks))
        return set_err(BQG_ERR_WORKSPACE, "biqgemm_sharded_p2p: workspace too small");
    if (count == 0) return BQG_OK;
    const size_t xs = x_rows * b, block = R * b;
    float* y_local = h_y_gather_peers[rank];
    // 1. every call's x from rank 0
    s = coll->broadcast(coll->ctx, d_x, count * xs * sizeof(float), 0, stream);
    if (s) return s;
    // the same decision on every rank (it picks the collective that follows)
    const bool fused = nranks - 1 <= bqg::kMaxPeers && count >= static_cast<size_t>(bqg::kTexMinGroup) &&
                       bqg::stream_supported(static_cast<int>(mu), static_cast<int>(beta), static_cast<long long>(b)) &&
                       bqg::tex_stream_applies(static_cast<long long>(R), static_cast<int>(groups_of(n, mu)),
                                               static_cast<int>(beta));
    if (hi > lo) {
        std::vector<bqg::StreamCall> calls(count);
        for (size_t i = 0; i < count; ++i) {
            if (!h_calls[i].d_keys_tiled_shard)
                return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null keys in call %zu", i);
            calls[i] = {h_calls[i].d_keys_tiled_shard, h_calls[i].d_alpha_shard, d_x + i * xs,
                        y_local + (static_cast<size_t>(rank) * count + i) * block};
        }
        if (fused) {
            // 2+3. the grouped texture kernel on this rank's rows; its
            // finaliser stores every y row into every peer's gather buffer
            std::vector<float*> peers;
            for (int r = 0; r < nranks; ++r)
                if (r != rank) peers.push_back(h_y_gather_peers[r]);
            cudaError_t e = bqg::launch_biqgemm_tex(calls.data(), static_cast<int>(count), static_cast<long long>(x_rows),
                                                    static_cast<int>(hi - lo), static_cast<int>(groups_of(n, mu)),
                                                    static_cast<int>(beta), static_cast<float*>(d_ws), pdl != 0,
                                                    as_stream(stream), y_local, peers.data(),
                                                    static_cast<int>(peers.size()));
            if (e != cudaSuccess) return cuda_err(e, "biqgemm grouped p2p kernel");
        } else {
            std::vector<bqg_call> gc(count);
            for (size_t i = 0; i < count; ++i) gc[i] = {calls[i].keys, calls[i].alpha, calls[i].x, calls[i].y};
            s = bqg_biqgemm_grouped_f32(gc.data(), count, x_rows, hi - lo, n, b, beta, mu, d_ws, gws, pdl, stream);
            if (s) return s;
        }
    }
    if (!fused) {  // shapes the texture form does not take: the gather through the collectives
        float* y_mine = y_local + static_cast<size_t>(rank) * count * block;
        return coll->allgather(coll->ctx, y_mine, y_local, count * block * sizeof(float), stream);
    }
    // 4. a barrier (an all-gather of 16 bytes per rank): every rank's kernel
    //    -- and with it every peer store into this rank's buffer -- is
    //    complete before work queued after this call reads y
    char* bar = static_cast<char*>(d_ws) + barrier_offset(gws);
    return coll->allgather(coll->ctx, bar + static_cast<size_t>(rank) * kBarrierBytesPerRank, bar,
                           kBarrierBytesPerRank, stream);
}

extern "C" size_t bqg_biqgemm_sharded_p2p_workspace_bytes(size_t m, size_t n, size_t b, unsigned beta, unsigned mu,
                                                          int nranks) {
    const size_t g = bqg_biqgemm_sharded_workspace_bytes(m, n, b, beta, mu, nranks);
    if (g == 0) return 0;
    return barrier_offset(g) + kBarrierBytesPerRank * static_cast<size_t>(nranks);
}

extern "C" int bqg_biqgemm_sharded_p2p_f32(const uint8_t* d_keys_tiled_shard, const float* d_alpha_shard, float* d_x,
                                           size_t x_rows, float* const* h_y_gather_peers, size_t m, size_t n,
                                           size_t b, unsigned beta, unsigned mu, int rank, int nranks,
                                           const bqg_collectives* coll, void* d_ws, size_t ws_bytes, void* stream) {
    size_t lo = 0, hi = 0, R = 0;
    int s = bqg_shard_rows(m, nranks, rank, &lo, &hi, &R);
    if (s) return s;
    if (!coll || !coll->broadcast || !coll->allgather)
        return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: collectives missing");
    if (!d_x || !h_y_gather_peers) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null pointer");
    for (int r = 0; r < nranks; ++r)
        if (!h_y_gather_peers[r]) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null peer buffer %d", r);
    s = check_mu(mu, "biqgemm");
    if (s) return s;
    s = check_x(x_rows, b, n, mu, "biqgemm");
    if (s) return s;
    const size_t gws = bqg_biqgemm_sharded_workspace_bytes(m, n, b, beta, mu, nranks);
    if (!d_ws || gws == 0 || ws_bytes < barrier_offset(gws) + kBarrierBytesPerRank * static_cast<size_t>(nranks))
        return set_err(BQG_ERR_WORKSPACE, "biqgemm_sharded_p2p: workspace too small");
    float* y_local = h_y_gather_peers[rank];
    float* y_mine = y_local + static_cast<size_t>(rank) * R * b;
    // 1. x from rank 0 to every rank
    s = coll->broadcast(coll->ctx, d_x, x_rows * b * sizeof(float), 0, stream);
    if (s) return s;
    // the same decision on every rank (it picks the collective that follows):
    // shapes the two-kernel form takes, except the b = 1 shapes the latency /
    // stream forms serve
    const bool fused = nranks - 1 <= bqg::kMaxPeers && mu <= 8 &&
                       !bqg::stream_supported(static_cast<int>(mu), static_cast<int>(beta), static_cast<long long>(b)) &&
                       bqg::twokernel_supported(static_cast<int>(mu), static_cast<int>(beta), static_cast<long long>(b));
    if (!fused) {  // the rank's rows, then the gather through the collectives
        if (hi > lo) {
            s = bqg_biqgemm_f32(d_keys_tiled_shard, d_alpha_shard, d_x, x_rows, y_mine, hi - lo, n, b, beta, mu, d_ws,
                                gws, 0, stream);
            if (s) return s;
        }
        return coll->allgather(coll->ctx, y_mine, y_local, R * b * sizeof(float), stream);
    }
    if (hi > lo) {
        if (!d_keys_tiled_shard) return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm_sharded: null keys");
        if (hi - lo > 0x7fffffff || b > 0x7fffffff)
            return set_err(BQG_ERR_INVALID_ARGUMENT, "biqgemm: dimension too large");
        BQG_NEED_DEVICE();
        // 2+3. the two-kernel form on this rank's rows (every shard count
        // takes the same form, so y is bitwise independent of nranks); its
        // finaliser stores every y value into every peer's gather buffer
        bqg::QueryParams p = make_params(d_keys_tiled_shard, d_alpha_shard, d_x, x_rows, y_mine, hi - lo, n, b, beta,
                                         mu, d_ws);
        p.peer_local = y_local;
        for (int r = 0; r < nranks; ++r)
            if (r != rank) p.peer_y[p.npeer++] = h_y_gather_peers[r];
        cudaError_t e = bqg::launch_biqgemm_twokernel(p, static_cast<int>(mu), false, as_stream(stream));
        if (e != cudaSuccess) return cuda_err(e, "biqgemm sharded p2p kernels");
    }
    // 4. the barrier: every rank's kernels, and their peer stores into this
    //    rank's buffer, are complete before work queued after this call reads y
    char* bar = static_cast<char*>(d_ws) + barrier_offset(gws);
    return coll->allgather(coll->ctx, bar + static_cast<size_t>(rank) * kBarrierBytesPerRank, bar,
                           kBarrierBytesPerRank, stream);
}
