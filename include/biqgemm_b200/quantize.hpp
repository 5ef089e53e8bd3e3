// quantize.hpp -- drop-in for /root/reference/proj/core/include/biqgemm/quantize.hpp.
//
// quantize_greedy (quantize.hpp:27-58) runs on the GPU
// (bqg_quantize_greedy_f32 / _f64) and is bit-exact with the reference:
// per-row sequential fp64 |residual| sums, sign(0) = +1, alpha stored as T.
// dequantize / quantization_error are host utilities (test oracles in the
// reference).
#pragma once

#include <cstddef>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "detail.hpp"
#include "matrix.hpp"
#include "packing.hpp"

namespace biqgemm {

template <typename T>
struct QuantizedLinear {
    std::size_t m = 0;
    std::size_t n = 0;
    unsigned beta = 0;
    std::vector<BinaryPlane> planes;     // beta planes, each m x n
    std::vector<std::vector<T>> alphas;  // beta vectors, each length m
};

template <typename T>
QuantizedLinear<T> quantize_greedy(const Matrix<T>& w, unsigned beta) {
    if (beta == 0) throw std::invalid_argument("quantize_greedy: beta must be >= 1");
    const std::size_t m = w.rows(), n = w.cols();
    QuantizedLinear<T> q;
    q.m = m;
    q.n = n;
    q.beta = beta;
    q.planes.assign(beta, BinaryPlane(m, n));
    q.alphas.assign(beta, std::vector<T>(m, T(0)));
    const std::size_t wpr = (n + 31) / 32;
    detail::DeviceBuffer d_w(w.data(), m * n * sizeof(T));
    detail::DeviceBuffer d_planes(beta * m * wpr * sizeof(std::uint32_t));
    detail::DeviceBuffer d_alpha(beta * m * sizeof(T));
    if constexpr (std::is_same_v<T, float>) {
        detail::check(bqg_quantize_greedy_f32(d_w.get<float>(), m, n, beta, d_planes.get<std::uint32_t>(),
                                              d_alpha.get<float>(), nullptr));
    } else {
        detail::check(bqg_quantize_greedy_f64(d_w.get<double>(), m, n, beta, d_planes.get<std::uint32_t>(),
                                              d_alpha.get<double>(), nullptr));
    }
    std::vector<std::uint32_t> words(beta * m * wpr);
    d_planes.download(words.data(), words.size() * sizeof(std::uint32_t));
    std::vector<T> alpha(beta * m);
    d_alpha.download(alpha.data(), alpha.size() * sizeof(T));
    for (unsigned i = 0; i < beta; ++i) {
        auto& pw = q.planes[i].mutable_words();
        std::copy(words.begin() + i * m * wpr, words.begin() + (i + 1) * m * wpr, pw.begin());
        std::copy(alpha.begin() + i * m, alpha.begin() + (i + 1) * m, q.alphas[i].begin());
    }
    return q;
}

template <typename T>
Matrix<T> dequantize(const QuantizedLinear<T>& q) {
    Matrix<T> w(q.m, q.n);
    for (std::size_t r = 0; r < q.m; ++r)
        for (std::size_t c = 0; c < q.n; ++c) {
            double acc = 0.0;
            for (unsigned i = 0; i < q.beta; ++i) acc += double(q.alphas[i][r]) * double(q.planes[i].get(r, c));
            w(r, c) = T(acc);
        }
    return w;
}

template <typename T>
double quantization_error(const Matrix<T>& w, const QuantizedLinear<T>& q) {
    if (w.rows() != q.m || w.cols() != q.n) throw std::invalid_argument("quantization_error: shape mismatch");
    return frobenius_distance(w, dequantize(q));
}

}  // namespace biqgemm
