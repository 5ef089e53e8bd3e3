// lut.hpp -- drop-in for /root/reference/proj/core/include/biqgemm/lut.hpp.
//
// Table construction runs on the GPU (bqg_build_lut_f64 / _f64x, the exact
// builder: fp64 entries, the DP recurrence of lut.hpp:50-69 or the naive
// signed sums of lut.hpp:31-43, bit-identical to the reference).  LutBlock
// keeps the reference's layouts (table-major / key-major, lut.hpp:71-105).
// The fused fast path builds its fp32 tables in shared memory instead; those
// are exposed for parity through bqg_build_lut_f32.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "detail.hpp"
#include "matrix.hpp"
#include "packing.hpp"

namespace biqgemm {

inline BinaryPlane make_m_mu(unsigned mu) {
    if (mu < 1 || mu > kMaxLutUnit) throw std::invalid_argument("make_m_mu: mu out of range [1,16]");
    const std::size_t table = std::size_t(1) << mu;
    BinaryPlane m(table, mu);
    for (std::size_t k = 0; k < table; ++k)
        for (unsigned t = 0; t < mu; ++t) m.set(k, t, ((k >> t) & 1u) ? +1 : -1);
    return m;
}

enum class LutLayout { TableMajor, KeyMajor };
enum class LutBuilder { Dp, Naive };

namespace detail {
// One GPU table build for an x_rows x b input (device copy made here).
template <typename T>
inline std::uint64_t gpu_build(const T* x_host, std::size_t x_rows, std::size_t b, std::size_t g0, std::size_t count,
                               unsigned mu, LutLayout layout, LutBuilder builder, double* out_host) {
    DeviceBuffer d_x(x_host, x_rows * b * sizeof(T));
    const std::size_t n_entries = count * b * (std::size_t(1) << mu);
    DeviceBuffer d_out(n_entries * sizeof(double));
    std::uint64_t ops = 0;
    const int lay = layout == LutLayout::KeyMajor ? BQG_LUT_KEY_MAJOR : BQG_LUT_TABLE_MAJOR;
    const int bld = builder == LutBuilder::Naive ? BQG_LUT_NAIVE : BQG_LUT_DP;
    if constexpr (std::is_same_v<T, float>) {
        check(bqg_build_lut_f64(d_x.get<float>(), x_rows, b, mu, g0, count, lay, bld, d_out.get<double>(), &ops, nullptr));
    } else {
        check(bqg_build_lut_f64x(d_x.get<double>(), x_rows, b, mu, g0, count, lay, bld, d_out.get<double>(), &ops,
                                 nullptr));
    }
    d_out.download(out_host, n_entries * sizeof(double));
    return ops;
}
}  // namespace detail

// lut.hpp:31-43: 2^mu explicit dot products; returns 2^mu * mu.
template <typename T>
std::uint64_t build_lut_naive(const T* x, unsigned mu, double* out) {
    if (mu < 1 || mu > kMaxLutUnit) throw std::invalid_argument("build_lut_naive: mu out of range [1,16]");
    return detail::gpu_build<T>(x, mu, 1, 0, 1, mu, LutLayout::TableMajor, LutBuilder::Naive, out);
}

// lut.hpp:50-69: dynamic programming; returns 2^mu + mu - 1.
template <typename T>
std::uint64_t build_lut_dp(const T* x, unsigned mu, double* out) {
    if (mu < 1 || mu > kMaxLutUnit) throw std::invalid_argument("build_lut_dp: mu out of range [1,16]");
    return detail::gpu_build<T>(x, mu, 1, 0, 1, mu, LutLayout::TableMajor, LutBuilder::Dp, out);
}

struct LutBlock {
    unsigned mu = 0;
    std::size_t batch = 0;
    std::size_t group_count = 0;
    LutLayout layout = LutLayout::TableMajor;
    std::vector<double> entries;  // group_count * batch * 2^mu
    std::size_t table_size() const { return std::size_t(1) << mu; }
    std::size_t index(std::size_t group, std::size_t table, std::uint32_t key) const {
        const std::size_t base = group * batch * table_size();
        if (layout == LutLayout::KeyMajor) return base + std::size_t(key) * batch + table;
        return base + table * table_size() + key;
    }
    double at(std::size_t group, std::size_t table, std::uint32_t key) const { return entries[index(group, table, key)]; }
    const double* group_base(std::size_t group) const { return entries.data() + group * batch * table_size(); }
};

// lut.hpp:109-154.
template <typename T>
LutBlock build_lut_block(const Matrix<T>& x, std::size_t group_begin, std::size_t group_count, unsigned mu,
                         LutLayout layout, std::uint64_t* build_ops = nullptr, LutBuilder builder = LutBuilder::Dp) {
    if (group_count == 0) throw std::invalid_argument("build_lut_block: empty tile");
    if (mu < 1 || mu > kMaxLutUnit) throw std::invalid_argument("build_lut_block: mu out of range [1,16]");
    LutBlock block;
    block.mu = mu;
    block.batch = x.cols();
    block.group_count = group_count;
    block.layout = layout;
    block.entries.resize(group_count * x.cols() * (std::size_t(1) << mu));
    const std::uint64_t ops = detail::gpu_build<T>(x.data(), x.rows(), x.cols(), group_begin, group_count, mu, layout,
                                                   builder, block.entries.data());
    if (build_ops) *build_ops += ops;
    return block;
}

}  // namespace biqgemm
