// dropin_test.cpp -- the reference's own unit tests and acceptance criteria
// (/root/reference/proj/tests/test_*.cpp, acceptance_test.cpp), re-expressed
// against the drop-in C++ API (include/biqgemm_b200/) that runs on the B200.
// The test bodies are written like the reference's so the parity is easy to
// audit; each cites the reference test it mirrors.
//
//   dropin_test             all tests (needs a CUDA device)
//   dropin_test --host-only only the tests that need no device
// Exit code = number of failed checks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "biqgemm_b200/kernel.hpp"
#include "biqgemm_b200/lut.hpp"
#include "biqgemm_b200/matrix.hpp"
#include "biqgemm_b200/model_io.hpp"
#include "biqgemm_b200/packing.hpp"
#include "biqgemm_b200/quantize.hpp"

using namespace biqgemm;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                 \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(c)) {                                                              \
            ++g_fail;                                                            \
            std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);           \
        }                                                                        \
    } while (0)
#define CHECK_THROWS_AS(expr, exc)                                               \
    do {                                                                         \
        ++g_checks;                                                              \
        bool ok_ = false;                                                        \
        try {                                                                    \
            (void)(expr);                                                        \
        } catch (const exc&) {                                                   \
            ok_ = true;                                                          \
        } catch (...) {                                                          \
        }                                                                        \
        if (!ok_) {                                                              \
            ++g_fail;                                                            \
            std::printf("  FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #exc); \
        }                                                                        \
    } while (0)

namespace {

BinaryPlane plane_from_signs(std::size_t rows, std::size_t cols, const std::vector<int>& signs) {
    BinaryPlane p(rows, cols);
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t c = 0; c < cols; ++c) p.set(r, c, signs[r * cols + c]);
    return p;
}

BinaryPlane random_plane(std::size_t rows, std::size_t cols, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    BinaryPlane p(rows, cols);
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t c = 0; c < cols; ++c) p.set(r, c, (rng() & 1) ? +1 : -1);
    return p;
}

template <typename T>
Matrix<T> plane_to_dense(const BinaryPlane& p) {
    Matrix<T> d(p.rows(), p.cols());
    for (std::size_t r = 0; r < p.rows(); ++r)
        for (std::size_t c = 0; c < p.cols(); ++c) d(r, c) = T(p.get(r, c));
    return d;
}

// gemm_dense (baselines.hpp:14-36) restated: the test oracle.
template <typename T>
Matrix<T> gemm_dense(const Matrix<T>& a, const Matrix<T>& x) {
    Matrix<T> y(a.rows(), x.cols());
    for (std::size_t r = 0; r < a.rows(); ++r)
        for (std::size_t col = 0; col < x.cols(); ++col) {
            double acc = 0.0;
            for (std::size_t k = 0; k < a.cols(); ++k) acc += double(a(r, k)) * double(x(k, col));
            y(r, col) = T(acc);
        }
    return y;
}

// ---------------------------------------------------------------- host only

void host_tests() {
    // matrix.hpp:21-41
    CHECK_THROWS_AS(Matrix<float>(0, 3), std::invalid_argument);
    CHECK_THROWS_AS(Matrix<float>(2, 2, {1.f, 2.f, NAN, 4.f}), std::invalid_argument);
    CHECK_THROWS_AS(Matrix<float>(2, 2, {1.f, 2.f, 3.f}), std::invalid_argument);
    CHECK(Matrix<double>::identity(3)(1, 1) == 1.0 && Matrix<double>::identity(3)(0, 1) == 0.0);
    // seeded fills are deterministic
    CHECK(Matrix<float>::random_uniform(5, 7, 11) == Matrix<float>::random_uniform(5, 7, 11));
    CHECK(!(Matrix<float>::random_uniform(5, 7, 11) == Matrix<float>::random_uniform(5, 7, 12)));
    // test_packing.cpp:59-95
    for (int s : unpack_word(0)) CHECK(s == -1);
    auto w1 = unpack_word(1);
    CHECK(w1[0] == 1 && w1[1] == -1);
    BinaryPlane p32(1, 32);
    for (std::size_t c = 0; c < 32; ++c) p32.set(0, c, +1);
    CHECK(pack_plane_words(p32).size() == 1 && pack_plane_words(p32)[0] == 0xFFFFFFFFu);
    for (std::uint64_t seed = 0; seed < 10; ++seed) {
        auto p = random_plane(2, 64, seed);
        CHECK(unpack_plane_words(pack_plane_words(p), 2, 64) == p);
    }
    // test_packing.cpp:96-109 codec bijection
    for (unsigned mu = 1; mu <= 8; ++mu) {
        std::set<std::uint32_t> seen;
        for (std::uint32_t k = 0; k < (1u << mu); ++k) {
            std::vector<int> signs(mu);
            for (unsigned t = 0; t < mu; ++t) signs[t] = (k >> t) & 1u ? +1 : -1;
            CHECK(encode_key(signs.data(), mu) == k);
            seen.insert(encode_key(signs.data(), mu));
        }
        CHECK(seen.size() == (1u << mu));
    }
    // test_lut.cpp:12-31
    auto m2 = make_m_mu(2);
    const int expected[4][2] = {{-1, -1}, {+1, -1}, {-1, +1}, {+1, +1}};
    for (std::size_t k = 0; k < 4; ++k) CHECK(m2.get(k, 0) == expected[k][0] && m2.get(k, 1) == expected[k][1]);
    CHECK_THROWS_AS(make_m_mu(17), std::invalid_argument);
    // test_kernel.cpp:98-106
    CHECK(plan_tiles(1024, 128, 1, 8, 64 * 1024, 4).t_w == 64);
    CHECK(plan_tiles(1024, 128, 64, 8, 64 * 1024, 4).t_w == 1);
    CHECK_THROWS_AS(plan_tiles(1024, 128, 64, 8, 1024, 4), std::invalid_argument);
    // acceptance criterion 5 / test_model_io.cpp:82-97
    const unsigned bits[] = {32, 8, 6, 4, 3, 2};
    const double want[] = {1.049, 0.262, 0.197, 0.131, 0.098, 0.066};
    for (int i = 0; i < 6; ++i) CHECK(std::round(footprint(512, 512, bits[i]).weight_mb() * 1000.0) / 1000.0 == want[i]);
    CHECK(footprint(512, 512, 4).weight_bytes == 131072);
    CHECK_THROWS_AS(footprint(1, 1, 0), std::invalid_argument);
    // model_io typed errors on hand-made files (test_model_io.cpp:56-78)
    std::vector<std::uint8_t> good = {'B', 'Q', 'G', 'M', 1, 0, 1, 0, 0, 0, 4, 0, 0, 0, 1, 3};
    const float a = 0.5f;
    std::uint8_t ab[4];
    std::memcpy(ab, &a, 4);
    good.insert(good.end(), ab, ab + 4);
    good.push_back(5);  // G = ceil(4/3) = 2 keys of mu=3
    good.push_back(2);
    CHECK(load(good).keys[0].keys == (std::vector<std::uint32_t>{5, 2}));
    auto bad = good;
    bad[0] = 'X';
    CHECK_THROWS_AS(load(bad), BadMagicError);
    bad = good;
    bad[4] = 99;
    CHECK_THROWS_AS(load(bad), BadVersionError);
    bad = good;
    bad.resize(bad.size() - 1);
    CHECK_THROWS_AS(load(bad), TruncatedError);
    bad = good;
    bad.back() = 0xFF;
    CHECK_THROWS_AS(load(bad), RangeError);
    bad = good;
    bad.push_back(0);
    CHECK_THROWS_AS(load(bad), FormatError);
}

// ---------------------------------------------------------------- device

void packing_tests() {
    CHECK(pack_keys(plane_from_signs(1, 4, {-1, +1, +1, -1}), 4).key(0, 0) == 6);  // test_packing.cpp:37-42
    CHECK(pack_keys(plane_from_signs(1, 4, {+1, +1, +1, +1}), 4).key(0, 0) == 15);
    auto k = pack_keys(plane_from_signs(1, 6, {+1, -1, +1, -1, -1, +1}), 4);  // :49-57
    CHECK(k.groups == 2 && k.pad == 2 && k.key(0, 0) == 5 && k.key(0, 1) == 2);
    for (std::uint64_t seed = 0; seed < 5; ++seed) {  // :111-128
        auto p = random_plane(3, 16, seed);
        BinaryPlane f(3, 16);
        for (std::size_t r = 0; r < 3; ++r)
            for (std::size_t c = 0; c < 16; ++c) f.set(r, c, -p.get(r, c));
        for (unsigned mu : {2u, 4u, 8u}) {
            auto kp = pack_keys(p, mu), kf = pack_keys(f, mu);
            for (std::size_t i = 0; i < kp.keys.size(); ++i) CHECK(kf.keys[i] == ((1u << mu) - 1) - kp.keys[i]);
        }
    }
    BinaryPlane p(1, 4);
    CHECK_THROWS_AS(pack_keys(p, 0), std::invalid_argument);  // :130-134
    CHECK_THROWS_AS(pack_keys(p, 17), std::invalid_argument);
}

void lut_tests() {
    const double x[2] = {1.0, 2.0};
    double out[4];
    CHECK(build_lut_naive(x, 2, out) == 8);  // test_lut.cpp:33-42
    CHECK(out[0] == -3.0 && out[1] == -1.0 && out[2] == 1.0 && out[3] == 3.0);
    CHECK(build_lut_dp(x, 2, out) == 5);  // :56-65
    CHECK(out[0] == -3.0 && out[1] == -1.0 && out[2] == 1.0 && out[3] == 3.0);
    auto xr = Matrix<double>::random_uniform(4, 1, 3);  // :67-75
    double o16[16];
    build_lut_dp(xr.data(), 4, o16);
    for (std::uint32_t k = 0; k < 8; ++k) CHECK(o16[15 - k] == -o16[k]);
    std::mt19937_64 rng(0x5EED);  // :77-92 and acceptance criterion 2
    std::uniform_real_distribution<double> dist(-10.0, 10.0);
    for (unsigned mu = 1; mu <= 8; ++mu) {
        const std::size_t table = std::size_t(1) << mu;
        std::vector<double> xv(mu), dp(table), nv(table);
        for (int rep = 0; rep < 10; ++rep) {
            for (auto& v : xv) v = dist(rng);
            build_lut_dp(xv.data(), mu, dp.data());
            build_lut_naive(xv.data(), mu, nv.data());
            for (std::size_t kk = 0; kk < table; ++kk)
                CHECK(std::abs(dp[kk] - nv[kk]) / std::max(1.0, std::abs(nv[kk])) <= 1e-12);
            for (std::size_t kk = 0; kk < table / 2; ++kk) CHECK(dp[table - 1 - kk] == -dp[kk]);
        }
    }
    auto x1 = Matrix<double>::random_uniform(4, 1, 11);  // :94-100
    CHECK(build_lut_block(x1, 0, 1, 4, LutLayout::TableMajor).entries ==
          build_lut_block(x1, 0, 1, 4, LutLayout::KeyMajor).entries);
    auto x4 = Matrix<double>::random_uniform(4, 4, 12);  // :102-109
    auto blk = build_lut_block(x4, 0, 1, 4, LutLayout::KeyMajor);
    for (std::uint32_t kk = 0; kk < 16; ++kk)
        for (std::size_t t = 0; t < 4; ++t) CHECK(blk.index(0, t, kk) == std::size_t(kk) * 4 + t);
    auto x12 = Matrix<double>::random_uniform(12, 2, 13);  // :111-128
    for (auto layout : {LutLayout::TableMajor, LutLayout::KeyMajor}) {
        auto block = build_lut_block(x12, 0, 3, 4, layout);
        double expv[16], sub[4];
        for (std::size_t g = 0; g < 3; ++g)
            for (std::size_t col = 0; col < 2; ++col) {
                for (unsigned t = 0; t < 4; ++t) sub[t] = x12(g * 4 + t, col);
                build_lut_naive(sub, 4, expv);
                for (std::uint32_t kk = 0; kk < 16; ++kk) CHECK(std::abs(block.at(g, col, kk) - expv[kk]) < 1e-12);
            }
    }
    auto x16 = Matrix<double>::random_uniform(16, 3, 15);  // :149-157
    std::uint64_t ops = 0;
    build_lut_block(x16, 0, 4, 4, LutLayout::KeyMajor, &ops);
    CHECK(ops == (16 + 4 - 1) * 4 * 3);
    CHECK_THROWS_AS(build_lut_block(x16, 0, 0, 4, LutLayout::KeyMajor), std::invalid_argument);
    Matrix<double> x6(6, 1, {1, 2, 3, 4, 5, 6});  // :159-169
    auto b6 = build_lut_block(x6, 0, 2, 4, LutLayout::TableMajor);
    double s6[4] = {5, 6, 0, 0}, e6[16];
    build_lut_naive(s6, 4, e6);
    for (std::uint32_t kk = 0; kk < 16; ++kk) CHECK(std::abs(b6.at(1, 0, kk) - e6[kk]) < 1e-12);
}

void kernel_tests() {
    BinaryPlane pp(2, 4);  // test_kernel.cpp:40-49
    for (std::size_t r = 0; r < 2; ++r)
        for (std::size_t c = 0; c < 4; ++c) pp.set(r, c, +1);
    auto ycs = biqgemm_plane(pack_keys(pp, 4), Matrix<double>(4, 1, {1, 2, 3, 4}), TileShape{1, 2});
    CHECK(ycs(0, 0) == 10.0 && ycs(1, 0) == 10.0);
    auto x83 = Matrix<double>::random_normal(8, 3, 21);  // :51-59
    for (unsigned mu : {2u, 4u, 8u}) {
        auto p = random_plane(8, 8, mu);
        CHECK(frobenius_distance(biqgemm_plane(pack_keys(p, mu), x83, TileShape{2, 4}),
                                 gemm_dense(plane_to_dense<double>(p), x83)) < 1e-12);
    }
    {  // :61-68 (fp32 fast path)
        auto p = random_plane(512, 512, 7);
        auto x = Matrix<float>::random_normal(512, 18, 8);
        KernelStats stats;
        biqgemm_plane(pack_keys(p, 8), x, TileShape{16, 64}, &stats);
        CHECK(stats.ops.lookups == 589824ull);
    }
    {  // :70-79
        auto w = Matrix<double>::random_uniform(8, 8, 31);
        auto q = quantize_greedy(w, 1);
        auto x = Matrix<double>::random_normal(8, 2, 32);
        auto model = pack_linear(q, 4);
        std::fill(model.alphas[0].begin(), model.alphas[0].end(), 1.0);
        CHECK(biqgemm::biqgemm(model, x, TileShape{1, 8}) == biqgemm_plane(model.keys[0], x, TileShape{1, 8}));
    }
    {  // :81-87
        Matrix<double> w(2, 2, {3, 1, -3, -1});
        auto model = pack_linear(quantize_greedy(w, 2), 2);
        CHECK(frobenius_distance(biqgemm::biqgemm(model, Matrix<double>::identity(2), TileShape{1, 2}), w) < 1e-12);
    }
    {  // :89-96
        auto w = Matrix<float>::random_uniform(16, 16, 41);
        auto q = quantize_greedy(w, 3);
        auto x = Matrix<float>::random_normal(16, 4, 42);
        auto y = biqgemm::biqgemm(pack_linear(q, 4), x, TileShape{2, 8});
        auto ref = gemm_dense(dequantize(q), x);
        CHECK(frobenius_distance(y, ref) / frobenius_norm(ref) < 1e-4);
    }
    {  // KernelOptions::builder (kernel.hpp:51,158): Naive = 2^mu*mu build ops per table on the exact
       // path; a copy of a model starts without a device copy (its own keys/alphas are used)
        auto w = Matrix<float>::random_uniform(64, 96, 51);
        auto model = pack_linear(quantize_greedy(w, 2), 6);
        auto x = Matrix<float>::random_normal(96, 2, 52);
        KernelOptions naive;
        naive.builder = LutBuilder::Naive;
        KernelOptions ex;
        ex.exact = true;
        KernelStats sn, sd;
        auto yn = biqgemm::biqgemm(model, x, TileShape{4, 8}, &sn, naive);
        auto yd = biqgemm::biqgemm(model, x, TileShape{4, 8}, &sd, ex);
        const std::uint64_t G = model.keys[0].groups;
        CHECK(sn.ops.lut_build_ops == 64ull * 6 * G * 2);
        CHECK(sd.ops.lut_build_ops == (64ull + 6 - 1) * G * 2);
        CHECK(frobenius_distance(yn, yd) <= 1e-6 * frobenius_norm(yd));
        CHECK(sn.build_seconds > 0 && sn.query_seconds > 0);
        auto copy = model;
        for (auto& a : copy.alphas) std::fill(a.begin(), a.end(), 0.0f);
        auto yz = biqgemm::biqgemm(copy, x, TileShape{1, 1});
        for (std::size_t i = 0; i < yz.rows(); ++i) CHECK(yz(i, 0) == 0.0f && yz(i, 1) == 0.0f);
        CHECK(frobenius_norm(biqgemm::biqgemm(model, x, TileShape{1, 1})) > 0.0);
        // biqgemm_plane keeps the key matrix's device copy: same answer on reuse
        auto y1 = biqgemm_plane(model.keys[0], x, TileShape{1, 1});
        CHECK(biqgemm_plane(model.keys[0], x, TileShape{2, 2}) == y1);
    }
    {  // :108-134 + acceptance criterion 7: bitwise invariance over tiles/workers
        std::mt19937_64 rng(0x5EED);
        for (int rep = 0; rep < 10; ++rep) {
            const std::size_t m = 1 + rng() % 48, n = 1 + rng() % 48, b = 1 + rng() % 6;
            const unsigned beta = 1 + unsigned(rng() % 3), mu = 1u << (rng() % 4);
            auto model = pack_linear(quantize_greedy(Matrix<float>::random_uniform(m, n, rng()), beta), mu);
            auto x = Matrix<float>::random_normal(n, b, rng());
            const std::size_t groups = model.keys[0].groups;
            const TileShape shapes[] = {{1, 1}, {groups, m}, {(groups + 1) / 2, (m + 1) / 2}, {2, 3}};
            KernelOptions opts;
            auto ref = biqgemm::biqgemm(model, x, shapes[0], nullptr, opts);
            for (const auto& tile : shapes)
                for (std::size_t threads : {1, 2, 4}) {
                    opts.threads = threads;
                    CHECK(biqgemm::biqgemm(model, x, tile, nullptr, opts) == ref);
                }
        }
    }
    {  // :136-151 padding neutrality
        auto p = random_plane(4, 10, 51);
        auto k = pack_keys(p, 4);
        auto x = Matrix<double>::random_normal(10, 2, 52);
        Matrix<double> xp(12, 2);
        for (std::size_t r = 0; r < 10; ++r)
            for (std::size_t c = 0; c < 2; ++c) xp(r, c) = x(r, c);
        auto y = biqgemm_plane(k, x, TileShape{1, 4});
        CHECK(y == biqgemm_plane(k, xp, TileShape{1, 4}));
        CHECK(frobenius_distance(y, gemm_dense(plane_to_dense<double>(p), x)) < 1e-12);
    }
    {  // :153-161
        auto w = Matrix<float>::random_uniform(24, 32, 61);
        auto x = Matrix<float>::random_normal(32, 3, 62);
        KernelStats s1, s3;
        biqgemm::biqgemm(pack_linear(quantize_greedy(w, 1), 8), x, TileShape{2, 8}, &s1);
        biqgemm::biqgemm(pack_linear(quantize_greedy(w, 3), 8), x, TileShape{2, 8}, &s3);
        CHECK(s3.ops.lookups == 3 * s1.ops.lookups && s3.ops.lut_build_ops == s1.ops.lut_build_ops);
    }
    {  // :163-182 and acceptance criterion 3
        std::mt19937_64 rng(77);
        for (int rep = 0; rep < 20; ++rep) {
            const std::size_t m = 1 + rng() % 40, n = 1 + rng() % 70, b = 1 + rng() % 5;
            const unsigned beta = 1 + unsigned(rng() % 3), mu = 1 + unsigned(rng() % 8);
            const std::size_t groups = (n + mu - 1) / mu;
            auto w = Matrix<float>::random_uniform(m, n, rng());
            auto x = Matrix<float>::random_normal(n, b, rng());
            KernelStats stats;
            biqgemm::biqgemm(pack_linear(quantize_greedy(w, beta), mu), x,
                             TileShape{1 + rng() % groups, 1 + rng() % m}, &stats);
            CHECK(stats.ops.lookups == std::uint64_t(m) * groups * b * beta);
            CHECK(stats.ops.lut_build_ops == ((std::uint64_t(1) << mu) + mu - 1) * groups * b);
        }
    }
    {  // :184-196
        auto k = pack_keys(random_plane(4, 8, 81), 4);
        CHECK_THROWS_AS(biqgemm_plane(k, Matrix<double>::random_normal(16, 1, 82), TileShape{1, 4}),
                        std::invalid_argument);
        KernelOptions opts;
        opts.budget_bytes = 8;
        CHECK_THROWS_AS(biqgemm_plane(k, Matrix<double>::random_normal(8, 1, 83), TileShape{2, 4}, nullptr, opts),
                        std::invalid_argument);
    }
}

void acceptance_tests() {
    // criterion 1: 200 random cases vs gemm_dense(dequantize(q), x)
    std::mt19937_64 rng(0x5EED);
    const unsigned mus[] = {1, 2, 4, 8};
    auto cases = [&](auto tag, int n_cases, double tol) {
        using T = decltype(tag);
        for (int i = 0; i < n_cases; ++i) {
            const std::size_t m = 1 + rng() % 64, n = 1 + rng() % 64, b = 1 + rng() % 8;
            const unsigned mu = mus[rng() % 4], beta = 1 + unsigned(rng() % 3);
            auto w = Matrix<T>::random_uniform(m, n, rng());
            auto x = Matrix<T>::random_normal(n, b, rng());
            auto q = quantize_greedy(w, beta);
            auto model = pack_linear(q, mu);
            const std::size_t groups = model.keys[0].groups;
            const TileShape tile{1 + rng() % groups, 1 + rng() % m};
            auto y = biqgemm::biqgemm(model, x, tile);
            auto ref = gemm_dense(dequantize(q), x);
            const double nrm = frobenius_norm(ref), err = frobenius_distance(y, ref);
            CHECK((nrm > 0 ? err / nrm : err) <= tol);
        }
    };
    cases(double{}, 100, 1e-12);
    cases(float{}, 100, 1e-4);
    // criterion 6: monotone residual, exact 1-bit alpha
    std::mt19937_64 r6(0x5EED);
    for (int i = 0; i < 30; ++i) {
        const std::size_t m = 1 + r6() % 12, n = 1 + r6() % 16;
        auto w = Matrix<double>::random_uniform(m, n, r6());
        double prev = frobenius_norm(w);
        for (unsigned beta = 1; beta <= 4; ++beta) {
            const double err = quantization_error(w, quantize_greedy(w, beta));
            CHECK(err <= prev + 1e-12);
            prev = err;
        }
        auto q1 = quantize_greedy(w, 1);
        for (std::size_t r = 0; r < m; ++r) {
            double mean_abs = 0.0;
            for (std::size_t c = 0; c < n; ++c) mean_abs += std::abs(w(r, c));
            CHECK(q1.alphas[0][r] == mean_abs / double(n));
        }
    }
    // criterion 9: model round trips
    std::mt19937_64 r9(0x5EED);
    for (int i = 0; i < 20; ++i) {
        const std::size_t m = 1 + r9() % 16, n = 1 + r9() % 32;
        const unsigned beta = 1 + unsigned(r9() % 3), mu = 1 + unsigned(r9() % 16);
        auto q = quantize_greedy(Matrix<float>::random_uniform(m, n, r9()), beta);
        auto loaded = load(save(q, mu));
        auto packed = pack_linear(q, mu);
        for (unsigned pl = 0; pl < beta; ++pl) {
            CHECK(loaded.keys[pl].keys == packed.keys[pl].keys);
            CHECK(loaded.alphas[pl] == q.alphas[pl]);
        }
        auto back = to_quantized_linear(loaded);
        for (unsigned pl = 0; pl < beta; ++pl) CHECK(back.planes[pl] == q.planes[pl]);
    }
}

}  // namespace

int main(int argc, char** argv) {
    const bool host_only = argc > 1 && std::string(argv[1]) == "--host-only";
    struct Group {
        const char* name;
        std::function<void()> fn;
        bool device;
    };
    const Group groups[] = {{"host", host_tests, false},     {"packing", packing_tests, true},
                            {"lut", lut_tests, true},        {"kernel", kernel_tests, true},
                            {"acceptance", acceptance_tests, true}};
    for (const auto& g : groups) {
        if (g.device && host_only) continue;
        const int before = g_fail;
        try {
            g.fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("  FAIL %s: exception %s\n", g.name, e.what());
        }
        std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", g.name);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail;
}
