// model_io.hpp -- drop-in for /root/reference/proj/core/include/biqgemm/model_io.hpp
// (+ core/src/model_io.cpp).  BQGM serialisation/validation is the library's
// host code (bqg_bqgm_serialize / bqg_bqgm_parse), byte-identical files and
// the same typed errors, in the same order of checks.
#pragma once

#include <cstdint>
#include <fstream>
#include <iterator>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "detail.hpp"
#include "kernel.hpp"
#include "quantize.hpp"

namespace biqgemm {

inline std::vector<std::uint8_t> save(const QuantizedLinear<float>& q, unsigned mu) {
    if (mu < 1 || mu > kMaxLutUnit) throw std::invalid_argument("save: mu out of range [1,16]");
    const PackedLinear<float> p = pack_linear(q, mu);
    std::vector<const KeyMatrix*> planes;
    for (const auto& k : p.keys) planes.push_back(&k);
    const auto keys = detail::narrow_keys(planes, mu);
    std::vector<float> alpha;
    for (const auto& a : q.alphas) alpha.insert(alpha.end(), a.begin(), a.end());
    std::size_t len = 0;
    detail::check(bqg_bqgm_serialize(keys.data(), alpha.data(), q.m, q.n, q.beta, mu, nullptr, &len));
    std::vector<std::uint8_t> out(len);
    detail::check(bqg_bqgm_serialize(keys.data(), alpha.data(), q.m, q.n, q.beta, mu, out.data(), &len));
    return out;
}

inline PackedLinear<float> load(std::span<const std::uint8_t> bytes) {
    std::size_t m = 0, n = 0;
    unsigned beta = 0, mu = 0;
    detail::check(bqg_bqgm_parse(bytes.data(), bytes.size(), &m, &n, &beta, &mu, nullptr, nullptr));
    const std::size_t G = (n + mu - 1) / mu;
    std::vector<float> alpha(std::size_t(beta) * m);
    std::vector<std::uint8_t> keys(std::size_t(beta) * m * G * (mu > 8 ? 2 : 1));
    detail::check(bqg_bqgm_parse(bytes.data(), bytes.size(), &m, &n, &beta, &mu, alpha.data(), keys.data()));
    PackedLinear<float> p;
    p.m = m;
    p.n = n;
    p.beta = beta;
    p.mu = mu;
    for (unsigned i = 0; i < beta; ++i) {
        KeyMatrix k;
        k.m = m;
        k.groups = G;
        k.mu = mu;
        k.pad = G * mu - n;
        k.keys.resize(m * G);
        for (std::size_t j = 0; j < m * G; ++j)
            k.keys[j] = mu > 8 ? reinterpret_cast<const std::uint16_t*>(keys.data())[i * m * G + j]
                               : keys[i * m * G + j];
        p.keys.push_back(std::move(k));
        p.alphas.emplace_back(alpha.begin() + i * m, alpha.begin() + (i + 1) * m);
    }
    return p;
}

inline QuantizedLinear<float> to_quantized_linear(const PackedLinear<float>& p) {
    QuantizedLinear<float> q;
    q.m = p.m;
    q.n = p.n;
    q.beta = p.beta;
    q.alphas = p.alphas;
    for (const KeyMatrix& keys : p.keys) {
        BinaryPlane plane(p.m, p.n);
        for (std::size_t r = 0; r < p.m; ++r)
            for (std::size_t g = 0; g < keys.groups; ++g) {
                const std::uint32_t key = keys.key(r, g);
                for (unsigned t = 0; t < p.mu; ++t) {
                    const std::size_t c = g * p.mu + t;
                    if (c < p.n) plane.set(r, c, ((key >> t) & 1u) ? +1 : -1);
                }
            }
        q.planes.push_back(std::move(plane));
    }
    return q;
}

inline void save_file(const QuantizedLinear<float>& q, unsigned mu, const std::string& path) {
    const auto bytes = save(q, mu);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("save_file: cannot open " + path);
    out.write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(bytes.size()));
}

inline PackedLinear<float> load_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("load_file: cannot open " + path);
    std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return load(bytes);
}

struct Footprint {
    std::uint64_t weight_bytes = 0, activation_bytes = 0, output_bytes = 0, alpha_bytes = 0;
    std::uint64_t total_bytes() const { return weight_bytes + activation_bytes + output_bytes; }
    double weight_mb() const { return double(weight_bytes) / 1e6; }
    double activation_mb() const { return double(activation_bytes) / 1e6; }
    double output_mb() const { return double(output_bytes) / 1e6; }
    double total_mb() const { return double(total_bytes()) / 1e6; }
};

inline Footprint footprint(std::uint64_t m, std::uint64_t n, unsigned weight_bits, std::uint64_t batch = 18,
                           unsigned activation_bits = 32, unsigned output_bits = 32) {
    std::uint64_t o[4];
    detail::check(bqg_footprint(m, n, weight_bits, batch, activation_bits, output_bits, o));
    return Footprint{o[0], o[1], o[2], o[3]};
}

}  // namespace biqgemm
