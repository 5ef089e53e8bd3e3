// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// headers (/root/reference/proj/core/include/biqgemm/*.hpp) and the
// reference's only compiled TU (model_io.cpp), built by oracle/Makefile into
// oracle/_ref/libbqg_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C restatement
// (bqg_oracle.c) and to make golden fixtures, and by bench.py's
// --impl reference / cpu_baseline leg to time the reference's own CPU path.
// The product library never links or loads it.  No reference source is
// copied here: this file only calls the reference API.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "biqgemm/baselines.hpp"
#include "biqgemm/kernel.hpp"
#include "biqgemm/lut.hpp"
#include "biqgemm/matrix.hpp"
#include "biqgemm/model_io.hpp"
#include "biqgemm/packing.hpp"
#include "biqgemm/quantize.hpp"

using namespace biqgemm;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return 1;
}

PackedLinear<float> make_model(const std::uint32_t* keys, const float* alpha,
                               std::size_t m, std::size_t n, unsigned beta,
                               unsigned mu) {
    PackedLinear<float> p;
    p.m = m;
    p.n = n;
    p.beta = beta;
    p.mu = mu;
    const std::size_t groups = (n + mu - 1) / mu;
    for (unsigned i = 0; i < beta; ++i) {
        KeyMatrix k;
        k.m = m;
        k.groups = groups;
        k.mu = mu;
        k.pad = groups * mu - n;
        k.keys.assign(keys + std::size_t(i) * m * groups,
                      keys + std::size_t(i + 1) * m * groups);
        p.keys.push_back(std::move(k));
        if (alpha) {
            p.alphas.emplace_back(alpha + std::size_t(i) * m,
                                  alpha + std::size_t(i + 1) * m);
        } else {
            p.alphas.emplace_back(m, 1.0f);
        }
    }
    return p;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_random_uniform_f32(std::size_t rows, std::size_t cols, std::uint64_t seed,
                           float lo, float hi, float* out) {
    try {
        auto m = Matrix<float>::random_uniform(rows, cols, seed, lo, hi);
        std::memcpy(out, m.data(), sizeof(float) * rows * cols);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_random_normal_f32(std::size_t rows, std::size_t cols, std::uint64_t seed,
                          float* out) {
    try {
        auto m = Matrix<float>::random_normal(rows, cols, seed);
        std::memcpy(out, m.data(), sizeof(float) * rows * cols);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// quantize_greedy + pack_linear.  planes: beta x m x ceil(n/32) words,
// alpha: beta x m, keys: beta x m x G (u32).  Any output may be NULL.
int ref_quantize_pack_f32(const float* w, std::size_t m, std::size_t n, unsigned beta,
                          unsigned mu, std::uint32_t* planes, float* alpha,
                          std::uint32_t* keys) {
    try {
        Matrix<float> W(m, n, std::vector<float>(w, w + m * n));
        auto q = quantize_greedy(W, beta);
        const std::size_t wpr = (n + 31) / 32;
        for (unsigned i = 0; i < beta; ++i) {
            if (planes) {
                const auto& words = q.planes[i].words();
                std::memcpy(planes + std::size_t(i) * m * wpr, words.data(),
                            sizeof(std::uint32_t) * m * wpr);
            }
            if (alpha) {
                std::memcpy(alpha + std::size_t(i) * m, q.alphas[i].data(),
                            sizeof(float) * m);
            }
        }
        if (keys) {
            auto p = pack_linear(q, mu);
            const std::size_t groups = p.keys[0].groups;
            for (unsigned i = 0; i < beta; ++i) {
                std::memcpy(keys + std::size_t(i) * m * groups, p.keys[i].keys.data(),
                            sizeof(std::uint32_t) * m * groups);
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_pack_keys(const std::uint32_t* plane_words, std::size_t m, std::size_t n,
                  unsigned mu, std::uint32_t* keys) {
    try {
        const std::size_t wpr = (n + 31) / 32;
        auto plane = unpack_plane_words(
            std::vector<std::uint32_t>(plane_words, plane_words + m * wpr), m, n);
        auto k = pack_keys(plane, mu);
        std::memcpy(keys, k.keys.data(), sizeof(std::uint32_t) * k.keys.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// build_lut_block over a float x (x_rows x b), double entries.
int ref_build_lut_block(const float* x, std::size_t x_rows, std::size_t b,
                        std::size_t g0, std::size_t count, unsigned mu, int key_major,
                        int naive, double* entries, std::uint64_t* ops) {
    try {
        Matrix<float> X(x_rows, b, std::vector<float>(x, x + x_rows * b));
        std::uint64_t o = 0;
        auto blk = build_lut_block(X, g0, count, mu,
                                   key_major ? LutLayout::KeyMajor : LutLayout::TableMajor,
                                   &o, naive ? LutBuilder::Naive : LutBuilder::Dp);
        std::memcpy(entries, blk.entries.data(), sizeof(double) * blk.entries.size());
        if (ops) *ops = o;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// biqgemm (alpha != NULL) or biqgemm_plane semantics (alpha == NULL, beta == 1).
// stats: [build_ops, lookups, accumulate_ops, fma_ops] + [build_s, query_s, replace_s]
int ref_biqgemm_builder_f32(const std::uint32_t* keys, const float* alpha, std::size_t m,
                            std::size_t n, unsigned beta, unsigned mu, const float* x,
                            std::size_t x_rows, std::size_t b, std::size_t t_w, std::size_t t_h,
                            std::size_t threads, std::size_t budget, int naive, float* y,
                            double* stats);

int ref_biqgemm_f32(const std::uint32_t* keys, const float* alpha, std::size_t m,
                    std::size_t n, unsigned beta, unsigned mu, const float* x,
                    std::size_t x_rows, std::size_t b, std::size_t t_w, std::size_t t_h,
                    std::size_t threads, std::size_t budget, float* y, double* stats) {
    return ref_biqgemm_builder_f32(keys, alpha, m, n, beta, mu, x, x_rows, b, t_w, t_h, threads,
                                   budget, 0, y, stats);
}

// The same with KernelOptions::builder = Naive when naive != 0.
int ref_biqgemm_builder_f32(const std::uint32_t* keys, const float* alpha, std::size_t m,
                            std::size_t n, unsigned beta, unsigned mu, const float* x,
                            std::size_t x_rows, std::size_t b, std::size_t t_w, std::size_t t_h,
                            std::size_t threads, std::size_t budget, int naive, float* y,
                            double* stats) {
    try {
        auto model = make_model(keys, alpha, m, n, beta, mu);
        Matrix<float> X(x_rows, b, std::vector<float>(x, x + x_rows * b));
        KernelStats st;
        KernelOptions opts;
        opts.threads = threads;
        opts.budget_bytes = budget;
        if (naive) opts.builder = LutBuilder::Naive;
        Matrix<float> Y = alpha ? biqgemm::biqgemm(model, X, TileShape{t_w, t_h}, &st, opts)
                                : biqgemm_plane(model.keys[0], X, TileShape{t_w, t_h}, &st, opts);
        std::memcpy(y, Y.data(), sizeof(float) * m * b);
        if (stats) {
            stats[0] = double(st.ops.lut_build_ops);
            stats[1] = double(st.ops.lookups);
            stats[2] = double(st.ops.accumulate_ops);
            stats[3] = double(st.ops.fma_ops);
            stats[4] = st.build_seconds;
            stats[5] = st.query_seconds;
            stats[6] = st.replace_seconds;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Timing leg for the CPU baseline (bench_cli.cpp:160-166 protocol): warmup
// calls, then `repeats` timed calls of the reference biqgemm on a prepared
// model; returns every per-call wall time in seconds (caller takes the median)
// and the checksum (fp64 sum of y) of the last call.
int ref_time_biqgemm_f32(const std::uint32_t* keys, const float* alpha, std::size_t m,
                         std::size_t n, unsigned beta, unsigned mu, const float* x,
                         std::size_t b, std::size_t threads, int warmup, int repeats,
                         double* seconds, double* checksum) {
    try {
        auto model = make_model(keys, alpha, m, n, beta, mu);
        Matrix<float> X(n, b, std::vector<float>(x, x + n * b));
        const std::size_t groups = model.keys[0].groups;
        const std::size_t budget =
            std::max<std::size_t>(32 * 1024, (std::size_t(1) << mu) * b * sizeof(float));
        KernelOptions opts;
        opts.threads = threads;
        opts.budget_bytes = budget;
        const TileShape tile = plan_tiles(m, groups, b, mu, budget, sizeof(float));
        double sum = 0.0;
        auto once = [&]() {
            auto Y = biqgemm::biqgemm(model, X, tile, nullptr, opts);
            sum = 0.0;
            for (std::size_t i = 0; i < m * b; ++i) sum += double(Y.data()[i]);
        };
        for (int i = 0; i < warmup; ++i) once();
        for (int i = 0; i < repeats; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            auto Y = biqgemm::biqgemm(model, X, tile, nullptr, opts);
            seconds[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (i == repeats - 1) {
                sum = 0.0;
                for (std::size_t k = 0; k < m * b; ++k) sum += double(Y.data()[k]);
            }
        }
        if (checksum) *checksum = sum;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// gemm_dense(dequantize(q), x): the reference's own oracle (acceptance_test.cpp:62-63).
int ref_gemm_dense_dequant_f32(const std::uint32_t* planes, const float* alpha,
                               std::size_t m, std::size_t n, unsigned beta,
                               const float* x, std::size_t b, float* y) {
    try {
        QuantizedLinear<float> q;
        q.m = m;
        q.n = n;
        q.beta = beta;
        const std::size_t wpr = (n + 31) / 32;
        for (unsigned i = 0; i < beta; ++i) {
            q.planes.push_back(unpack_plane_words(
                std::vector<std::uint32_t>(planes + std::size_t(i) * m * wpr,
                                           planes + std::size_t(i + 1) * m * wpr),
                m, n));
            q.alphas.emplace_back(alpha + std::size_t(i) * m, alpha + std::size_t(i + 1) * m);
        }
        Matrix<float> X(n, b, std::vector<float>(x, x + n * b));
        auto Y = gemm_dense(dequantize(q), X);
        std::memcpy(y, Y.data(), sizeof(float) * m * b);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// model_io save(): serialise quantize_greedy(W, beta) at mu.  Returns byte
// count in *len; out may be NULL to query the size.
int ref_save_bqgm(const float* w, std::size_t m, std::size_t n, unsigned beta,
                  unsigned mu, std::uint8_t* out, std::size_t* len) {
    try {
        Matrix<float> W(m, n, std::vector<float>(w, w + m * n));
        auto bytes = save(quantize_greedy(W, beta), mu);
        if (out) std::memcpy(out, bytes.data(), std::min(*len, bytes.size()));
        *len = bytes.size();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// model_io load(): returns 0, or 2 bad magic, 3 bad version, 4 truncated,
// 5 range, 6 other FormatError, 1 other.
int ref_load_bqgm(const std::uint8_t* bytes, std::size_t len, std::size_t* m_out,
                  std::size_t* n_out, unsigned* beta_out, unsigned* mu_out,
                  std::uint32_t* keys, float* alpha) {
    try {
        auto p = load(std::span<const std::uint8_t>(bytes, len));
        *m_out = p.m;
        *n_out = p.n;
        *beta_out = p.beta;
        *mu_out = p.mu;
        const std::size_t groups = (p.n + p.mu - 1) / p.mu;
        for (unsigned i = 0; i < p.beta; ++i) {
            if (keys) {
                std::memcpy(keys + std::size_t(i) * p.m * groups, p.keys[i].keys.data(),
                            sizeof(std::uint32_t) * p.m * groups);
            }
            if (alpha) {
                std::memcpy(alpha + std::size_t(i) * p.m, p.alphas[i].data(),
                            sizeof(float) * p.m);
            }
        }
        return 0;
    } catch (const BadMagicError& e) {
        g_err = e.what();
        return 2;
    } catch (const BadVersionError& e) {
        g_err = e.what();
        return 3;
    } catch (const TruncatedError& e) {
        g_err = e.what();
        return 4;
    } catch (const RangeError& e) {
        g_err = e.what();
        return 5;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 6;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// footprint() (model_io.cpp:182-194): out[0..3] = weight, activation, output, alpha bytes.
int ref_footprint(std::uint64_t m, std::uint64_t n, unsigned bits, std::uint64_t batch,
                  std::uint64_t* out) {
    try {
        auto f = footprint(m, n, bits, batch);
        out[0] = f.weight_bytes;
        out[1] = f.activation_bytes;
        out[2] = f.output_bytes;
        out[3] = f.alpha_bytes;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
