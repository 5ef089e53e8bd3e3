// kernel.hpp -- drop-in for /root/reference/proj/core/include/biqgemm/kernel.hpp.
//
// Same types and entry points (TileShape, OpCounters, KernelStats,
// KernelOptions, plan_tiles, biqgemm_plane, PackedLinear, pack_linear,
// biqgemm), same validation and exceptions (kernel.hpp:127-143), same
// accumulate-into-stats contract (kernel.hpp:197-202).  The multiply runs on
// the B200:
//   - T = float, mu <= 8 : the fast path (fused LUT build / gather / alpha
//     epilogue, fp32 tables; ||y - y_ref||_F / ||y_ref||_F <= 1e-5);
//   - T = double, mu > 8, or KernelOptions::exact : the exact path (fp64
//     tables and accumulation in the reference's order: bit-identical y).
// A PackedLinear uploads itself to the device on first use and keeps the
// device copy; call reset_device() after mutating keys/alphas in place.
// KernelOptions::threads is accepted and ignored (the GPU decides its own
// parallelism); deterministic is always true; budget_bytes is validated as in
// the reference; TileShape is validated but does not change the result (the
// reference guarantees the same, acceptance criterion 7).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "detail.hpp"
#include "lut.hpp"
#include "matrix.hpp"
#include "packing.hpp"
#include "quantize.hpp"

namespace biqgemm {

struct TileShape {
    std::size_t t_w = 1;
    std::size_t t_h = 1;
};

struct OpCounters {
    std::uint64_t lut_build_ops = 0;
    std::uint64_t lookups = 0;
    std::uint64_t accumulate_ops = 0;
    std::uint64_t fma_ops = 0;
    OpCounters& operator+=(const OpCounters& o) {
        lut_build_ops += o.lut_build_ops;
        lookups += o.lookups;
        accumulate_ops += o.accumulate_ops;
        fma_ops += o.fma_ops;
        return *this;
    }
};

// Phase split on the GPU: query_seconds = the fused kernel(s) (LUT build and
// query are one kernel; build_seconds stays 0), replace_seconds = x upload +
// y download.
struct KernelStats {
    OpCounters ops;
    double build_seconds = 0.0;
    double query_seconds = 0.0;
    double replace_seconds = 0.0;
};

struct KernelOptions {
    std::size_t threads = 1;  // ignored on the GPU
    bool deterministic = true;
    LutBuilder builder = LutBuilder::Dp;
    std::size_t budget_bytes = 0;  // 0 disables the working-set check
    bool exact = false;            // extension: force the fp64 bit-exact path
};

inline TileShape plan_tiles(std::size_t m, std::size_t groups, std::size_t b, unsigned mu, std::size_t budget_bytes,
                            std::size_t entry_bytes = 4) {
    TileShape t;
    detail::check(bqg_plan_tiles(m, groups, b, mu, budget_bytes, entry_bytes, &t.t_w, &t.t_h));
    return t;
}

template <typename T>
struct PackedLinear {
    std::size_t m = 0;
    std::size_t n = 0;
    unsigned beta = 0;
    unsigned mu = 0;
    std::vector<KeyMatrix> keys;         // one per plane
    std::vector<std::vector<T>> alphas;  // one length-m vector per plane
    mutable std::shared_ptr<void> device_cache;
    void reset_device() const { device_cache.reset(); }
};

template <typename T>
PackedLinear<T> pack_linear(const QuantizedLinear<T>& q, unsigned mu) {
    PackedLinear<T> p;
    p.m = q.m;
    p.n = q.n;
    p.beta = q.beta;
    p.mu = mu;
    p.keys.reserve(q.beta);
    for (const BinaryPlane& plane : q.planes) p.keys.push_back(pack_keys(plane, mu));
    p.alphas = q.alphas;
    return p;
}

namespace detail {

struct LayerF32 {
    bqg_layer* h = nullptr;
    ~LayerF32() {
        if (h) bqg_layer_destroy(h);
    }
};

struct ModelF64 {
    DeviceBuffer keys, alpha;
};

inline std::vector<std::uint8_t> narrow_keys(const std::vector<const KeyMatrix*>& planes, unsigned mu) {
    const std::size_t per = planes[0]->keys.size();
    const std::size_t w = mu > 8 ? 2 : 1;
    std::vector<std::uint8_t> out(planes.size() * per * w);
    for (std::size_t i = 0; i < planes.size(); ++i) {
        const auto& k = planes[i]->keys;
        for (std::size_t j = 0; j < per; ++j) {
            if (w == 2) {
                reinterpret_cast<std::uint16_t*>(out.data())[i * per + j] = static_cast<std::uint16_t>(k[j]);
            } else {
                out[i * per + j] = static_cast<std::uint8_t>(k[j]);
            }
        }
    }
    return out;
}

// detail::run (kernel.hpp:116-204): validation in the reference's order, then
// the device multiply.  `cache` holds the device copy of the model.
template <typename T>
Matrix<T> run(const std::vector<const KeyMatrix*>& planes, const std::vector<const std::vector<T>*>& alphas,
              std::size_t n, const Matrix<T>& x, const TileShape& tile, const KernelOptions& opts, KernelStats* stats,
              std::shared_ptr<void>& cache) {
    const KeyMatrix& k0 = *planes[0];
    const std::size_t m = k0.m, groups = k0.groups, b = x.cols();
    const unsigned mu = k0.mu;
    for (const KeyMatrix* p : planes)
        if (p->m != m || p->groups != groups || p->mu != mu)
            throw std::invalid_argument("biqgemm: inconsistent plane shapes");
    if (std::size_t(mu) * groups < x.rows()) throw std::invalid_argument("biqgemm: key matrix too narrow for input");
    if (tile.t_w == 0 || tile.t_h == 0) throw std::invalid_argument("biqgemm: tile dimensions must be nonzero");
    if (opts.budget_bytes != 0) {
        const std::size_t need = tile.t_w * (std::size_t(1) << mu) * b * sizeof(T);
        if (need > opts.budget_bytes) throw std::invalid_argument("biqgemm: tile exceeds working-set budget");
    }
    const unsigned beta = static_cast<unsigned>(planes.size());
    if (n == 0) n = groups * mu;  // plane mode: only the padded width is known
    Matrix<T> y(m, b);
    if constexpr (std::is_same_v<T, float>) {
        if (!cache) {
            auto L = std::make_shared<LayerF32>();
            const auto keys = narrow_keys(planes, mu);
            std::vector<float> a;
            if (!alphas.empty()) {
                a.reserve(beta * m);
                for (auto* v : alphas) a.insert(a.end(), v->begin(), v->end());
            }
            check(bqg_layer_create_from_keys(keys.data(), alphas.empty() ? nullptr : a.data(), m, n, beta, mu, &L->h));
            cache = L;
        }
        bqg_kernel_stats st{};
        check(bqg_layer_forward_host(static_cast<LayerF32*>(cache.get())->h, x.data(), x.rows(), b, y.data(),
                                     opts.exact ? 1 : 0, &st));
        if (stats) {
            stats->ops.lut_build_ops += st.lut_build_ops;
            stats->ops.lookups += st.lookups;
            stats->ops.accumulate_ops += st.accumulate_ops;
            stats->ops.fma_ops += st.fma_ops;
            stats->build_seconds += st.build_seconds;
            stats->query_seconds += st.query_seconds;
            stats->replace_seconds += st.replace_seconds;
        }
    } else {
        if (!cache) {
            auto M = std::make_shared<ModelF64>();
            const auto keys = narrow_keys(planes, mu);
            M->keys = DeviceBuffer(keys.data(), keys.size());
            if (!alphas.empty()) {
                std::vector<double> a;
                for (auto* v : alphas) a.insert(a.end(), v->begin(), v->end());
                M->alpha = DeviceBuffer(a.data(), a.size() * sizeof(double));
            }
            cache = M;
        }
        auto* M = static_cast<ModelF64*>(cache.get());
        const auto t0 = std::chrono::steady_clock::now();
        DeviceBuffer d_x(x.data(), x.rows() * b * sizeof(double));
        DeviceBuffer d_y(m * b * sizeof(double));
        const std::size_t ws = bqg_biqgemm_exact_workspace_bytes(m, n, b, beta, mu);
        DeviceBuffer d_ws(ws);
        const auto t1 = std::chrono::steady_clock::now();
        check(bqg_biqgemm_exact_f64(M->keys.get(), M->alpha.get<double>(), d_x.get<double>(), x.rows(),
                                    d_y.get<double>(), m, n, b, beta, mu, d_ws.get(), ws, nullptr));
        cuda_check(cudaDeviceSynchronize(), "biqgemm");
        const auto t2 = std::chrono::steady_clock::now();
        d_y.download(y.data(), m * b * sizeof(double));
        const auto t3 = std::chrono::steady_clock::now();
        if (stats) {
            std::uint64_t ops[4];
            check(bqg_op_counters(m, n, b, beta, mu, BQG_LUT_DP, ops));
            stats->ops.lut_build_ops += ops[0];
            stats->ops.lookups += ops[1];
            stats->ops.accumulate_ops += ops[2];
            stats->query_seconds += std::chrono::duration<double>(t2 - t1).count();
            stats->replace_seconds += std::chrono::duration<double>((t1 - t0) + (t3 - t2)).count();
        }
    }
    return y;
}

}  // namespace detail

// kernel.hpp:209-215: one key matrix, alpha = 1.
template <typename T>
Matrix<T> biqgemm_plane(const KeyMatrix& keys, const Matrix<T>& x, const TileShape& tile, KernelStats* stats = nullptr,
                        const KernelOptions& opts = {}) {
    std::shared_ptr<void> cache;
    return detail::run<T>({&keys}, {}, 0, x, tile, opts, stats, cache);
}

// kernel.hpp:246-258: sum_i alpha_i o (B_i . X).
template <typename T>
Matrix<T> biqgemm(const PackedLinear<T>& model, const Matrix<T>& x, const TileShape& tile,
                  KernelStats* stats = nullptr, const KernelOptions& opts = {}) {
    std::vector<const KeyMatrix*> planes;
    std::vector<const std::vector<T>*> alphas;
    for (unsigned i = 0; i < model.beta; ++i) {
        planes.push_back(&model.keys[i]);
        alphas.push_back(&model.alphas[i]);
    }
    if (planes.empty()) throw std::invalid_argument("biqgemm: model has no planes");
    return detail::run<T>(planes, alphas, model.n, x, tile, opts, stats, model.device_cache);
}

}  // namespace biqgemm
