// kernel.hpp -- drop-in for /root/reference/proj/core/include/biqgemm/kernel.hpp.
//
// Same types and entry points (TileShape, OpCounters, KernelStats,
// KernelOptions, plan_tiles, biqgemm_plane, PackedLinear, pack_linear,
// biqgemm), same validation and exceptions (kernel.hpp:127-143), same
// accumulate-into-stats contract (kernel.hpp:197-202).  The multiply runs on
// the B200:
//   - T = float : the fast path (fused LUT build / gather / alpha epilogue,
//     fp32 tables; ||y - y_ref||_F / ||y_ref||_F <= 1e-5); mu > 8 runs the
//     same kernels on the sign bits re-keyed to mu = 8 (bqg_rekey_mu8);
//   - T = double, or KernelOptions::exact : the exact path (fp64 tables and
//     accumulation in the reference's order: bit-identical y).
// A PackedLinear (and a KeyMatrix used with biqgemm_plane) uploads itself to
// the device on first use and keeps the device copy; call reset_device()
// after mutating keys/alphas in place.  KernelOptions::builder = Naive runs
// the exact path with the reference's naive tables.
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

// Phase split on the GPU (kernel.hpp:41-46).  Exact path (double,
// KernelOptions::exact, or builder = Naive): build = the LUT kernels, query =
// the lookup kernels, replace = setup + alpha epilogue + x upload + y
// download -- the reference's split.  Fast path: the LUT build runs inside the
// query kernel (builder warps overlap the gather), so build_seconds stays 0
// and query_seconds is the fused kernel.
struct KernelStats {
    OpCounters ops;
    double build_seconds = 0.0;
    double query_seconds = 0.0;
    double replace_seconds = 0.0;
};

struct KernelOptions {
    std::size_t threads = 1;  // ignored on the GPU
    bool deterministic = true;
    // Dp: the fast path (fp32 DP tables) or, with `exact`, fp64 DP tables.
    // Naive (the reference's ablation builder, lut.hpp:31-43): fp64 naive
    // tables on the exact path -- y bit-identical to the reference run with
    // LutBuilder::Naive, lut_build_ops = 2^mu * mu per table (kernel.hpp:158).
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
    detail::DeviceCache device_cache;    // device copy, made on the first multiply (copies start empty)
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
// the device multiply.  `cache` holds the device copy of the model, tagged
// with the first plane's key storage.
template <typename T>
Matrix<T> run(const std::vector<const KeyMatrix*>& planes, const std::vector<const std::vector<T>*>& alphas,
              std::size_t n, const Matrix<T>& x, const TileShape& tile, const KernelOptions& opts, KernelStats* stats,
              const DeviceCache& cache) {
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
    const bool naive = opts.builder == LutBuilder::Naive;
    const void* tag = k0.keys.data();
    const std::size_t tag_size = k0.keys.size() * beta + (alphas.empty() ? 0 : alphas[0]->size());
    Matrix<T> y(m, b);
    bqg_kernel_stats st{};
    if constexpr (std::is_same_v<T, float>) {
        auto L = cache.get(tag, tag_size, [&] {
            auto h = std::make_shared<LayerF32>();
            const auto keys = narrow_keys(planes, mu);
            std::vector<float> a;
            if (!alphas.empty()) {
                a.reserve(beta * m);
                for (auto* v : alphas) a.insert(a.end(), v->begin(), v->end());
            }
            check(bqg_layer_create_from_keys(keys.data(), alphas.empty() ? nullptr : a.data(), m, n, beta, mu, &h->h));
            return std::static_pointer_cast<void>(h);
        });
        const int path = naive ? BQG_FORWARD_EXACT_NAIVE : (opts.exact ? BQG_FORWARD_EXACT : BQG_FORWARD_FAST);
        check(bqg_layer_forward_host(static_cast<LayerF32*>(L.get())->h, x.data(), x.rows(), b, y.data(), path,
                                     stats ? &st : nullptr));
    } else {
        auto Mp = cache.get(tag, tag_size, [&] {
            auto M = std::make_shared<ModelF64>();
            const auto keys = narrow_keys(planes, mu);
            M->keys = DeviceBuffer(keys.data(), keys.size());
            if (!alphas.empty()) {
                std::vector<double> a;
                for (auto* v : alphas) a.insert(a.end(), v->begin(), v->end());
                M->alpha = DeviceBuffer(a.data(), a.size() * sizeof(double));
            }
            return std::static_pointer_cast<void>(M);
        });
        auto* M = static_cast<ModelF64*>(Mp.get());
        const auto t0 = std::chrono::steady_clock::now();
        DeviceBuffer d_x(x.data(), x.rows() * b * sizeof(double));
        DeviceBuffer d_y(m * b * sizeof(double));
        const std::size_t ws = bqg_biqgemm_exact_workspace_bytes(m, n, b, beta, mu);
        DeviceBuffer d_ws(ws);
        const auto t1 = std::chrono::steady_clock::now();
        check(bqg_biqgemm_exact_ex_f64(M->keys.get(), M->alpha.get<double>(), d_x.get<double>(), x.rows(),
                                       d_y.get<double>(), m, n, b, beta, mu, naive ? BQG_LUT_NAIVE : BQG_LUT_DP,
                                       d_ws.get(), ws, stats ? &st : nullptr, nullptr));
        cuda_check(cudaDeviceSynchronize(), "biqgemm");
        const auto t2 = std::chrono::steady_clock::now();
        d_y.download(y.data(), m * b * sizeof(double));
        const auto t3 = std::chrono::steady_clock::now();
        st.replace_seconds += std::chrono::duration<double>((t1 - t0) + (t3 - t2)).count();
    }
    if (stats) {
        stats->ops.lut_build_ops += st.lut_build_ops;
        stats->ops.lookups += st.lookups;
        stats->ops.accumulate_ops += st.accumulate_ops;
        stats->ops.fma_ops += st.fma_ops;
        stats->build_seconds += st.build_seconds;
        stats->query_seconds += st.query_seconds;
        stats->replace_seconds += st.replace_seconds;
    }
    return y;
}

}  // namespace detail

// kernel.hpp:209-215: one key matrix, alpha = 1.
// The key matrix keeps its device copy (KeyMatrix::device_cache), so
// repeated calls on one plane upload its keys once.
template <typename T>
Matrix<T> biqgemm_plane(const KeyMatrix& keys, const Matrix<T>& x, const TileShape& tile, KernelStats* stats = nullptr,
                        const KernelOptions& opts = {}) {
    return detail::run<T>({&keys}, {}, 0, x, tile, opts, stats, keys.device_cache);
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
