/*
 * bqg_oracle.c -- CPU restatement of the reference BiQGEMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2005_09904_b200/) links, loads or calls this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may use it, and only as the checker.
 *
 * Each function restates one reference function in plain C99 and cites the
 * file:line of /root/reference/proj/core/include/biqgemm/ it follows.  The
 * restatement is pinned against the reference itself (oracle/_ref, built
 * from the reference headers by oracle/Makefile) and against the
 * reference's known-answer tests (tests/golden/, tests/test_oracle.py).
 *
 * Conventions (same as the reference):
 *   - matrices are row-major; x is n x b (x(r,c) at r*b+c), y is m x b;
 *   - a BinaryPlane row holds ceil(cols/32) little-endian u32 words,
 *     LSB-first, bit 1 = +1 (packing.hpp:16-57);
 *   - a key matrix is m x G row-major, G = ceil(n/mu), pad bits 0
 *     (packing.hpp:61-107).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BQO_OK 0
#define BQO_EINVAL 1

static size_t words_per_row(size_t cols) { return (cols + 31u) / 32u; }

/* quantize.hpp:27-58 quantize_greedy<float>.  Per row: residual in double;
 * for each plane alpha = (sequential sum |res|)/n, stored as float; sign =
 * res < 0 ? -1 : +1 (sign(0) = +1); res -= alpha*sign.
 * planes: beta x m x wpr words (zeroed here); alpha: beta x m floats. */
int bqo_quantize_greedy_f32(const float* w, size_t m, size_t n, unsigned beta,
                            uint32_t* planes, float* alpha) {
    if (beta == 0 || m == 0 || n == 0) return BQO_EINVAL;
    const size_t wpr = words_per_row(n);
    memset(planes, 0, sizeof(uint32_t) * beta * m * wpr);
    double* res = (double*)malloc(sizeof(double) * n);
    if (!res) return BQO_EINVAL;
    for (size_t r = 0; r < m; ++r) {
        for (size_t c = 0; c < n; ++c) res[c] = (double)w[r * n + c];
        for (unsigned i = 0; i < beta; ++i) {
            double abs_sum = 0.0;
            for (size_t c = 0; c < n; ++c) abs_sum += fabs(res[c]);
            const double a = abs_sum / (double)n;
            alpha[(size_t)i * m + r] = (float)a;
            uint32_t* row = planes + ((size_t)i * m + r) * wpr;
            for (size_t c = 0; c < n; ++c) {
                const int positive = !(res[c] < 0.0);
                if (positive) row[c / 32] |= 1u << (c % 32);
                res[c] -= a * (positive ? 1.0 : -1.0);
            }
        }
    }
    free(res);
    return BQO_OK;
}

/* quantize.hpp:61-74 dequantize<float>: W-hat(r,c) = float(sum_i alpha_i[r]*s),
 * accumulated in double over ascending i. */
int bqo_dequantize_f32(const uint32_t* planes, const float* alpha, size_t m,
                       size_t n, unsigned beta, float* w_out) {
    const size_t wpr = words_per_row(n);
    for (size_t r = 0; r < m; ++r) {
        for (size_t c = 0; c < n; ++c) {
            double acc = 0.0;
            for (unsigned i = 0; i < beta; ++i) {
                const uint32_t word = planes[((size_t)i * m + r) * wpr + c / 32];
                const double s = ((word >> (c % 32)) & 1u) ? 1.0 : -1.0;
                acc += (double)alpha[(size_t)i * m + r] * s;
            }
            w_out[r * n + c] = (float)acc;
        }
    }
    return BQO_OK;
}

/* packing.hpp:84-107 pack_keys: key(r,g) = sum_{t<mu, g*mu+t<n} bit(r, g*mu+t) << t.
 * Output as u32 (the reference's in-memory type). */
int bqo_pack_keys(const uint32_t* plane, size_t m, size_t n, unsigned mu,
                  uint32_t* keys) {
    if (mu < 1 || mu > 16) return BQO_EINVAL;
    const size_t wpr = words_per_row(n);
    const size_t groups = (n + mu - 1) / mu;
    for (size_t r = 0; r < m; ++r) {
        const uint32_t* row = plane + r * wpr;
        for (size_t g = 0; g < groups; ++g) {
            uint32_t key = 0;
            for (unsigned t = 0; t < mu; ++t) {
                const size_t c = g * mu + t;
                if (c < n && ((row[c / 32] >> (c % 32)) & 1u)) key |= 1u << t;
            }
            keys[r * groups + g] = key;
        }
    }
    return BQO_OK;
}

/* lut.hpp:31-43 build_lut_naive: out[k] = sum_t (bit t of k ? +x_t : -x_t),
 * double accumulation.  Returns 2^mu * mu. */
uint64_t bqo_build_lut_naive_f64(const double* x, unsigned mu, double* out) {
    const size_t table = (size_t)1 << mu;
    for (size_t k = 0; k < table; ++k) {
        double acc = 0.0;
        for (unsigned t = 0; t < mu; ++t) acc += (((k >> t) & 1u) ? 1.0 : -1.0) * x[t];
        out[k] = acc;
    }
    return (uint64_t)table * mu;
}

/* lut.hpp:50-69 build_lut_dp (double): out[0] = -sum x (sequential
 * subtraction from 0); for i = 1..mu-1, j < 2^(i-1): out[j + 2^(i-1)] =
 * out[j] + 2*x_(i-1); then out[2^mu-1-k] = -out[k] for k < 2^(mu-1).
 * Returns 2^mu + mu - 1. */
uint64_t bqo_build_lut_dp_f64(const double* x, unsigned mu, double* out) {
    double e0 = 0.0;
    for (unsigned t = 0; t < mu; ++t) e0 -= x[t];
    out[0] = e0;
    for (unsigned i = 1; i < mu; ++i) {
        const double step = 2.0 * x[i - 1];
        const size_t half = (size_t)1 << (i - 1);
        for (size_t j = 0; j < half; ++j) out[j + half] = out[j] + step;
    }
    const size_t table = (size_t)1 << mu;
    for (size_t k = 0; k < table / 2; ++k) out[table - 1 - k] = -out[k];
    return (uint64_t)table + mu - 1;
}

/* The same DP recurrence evaluated in fp32 (the precision the GPU LUT is
 * held in).  This is the bit-exact target for the CUDA LUT builder: the
 * entry order of additions is exactly lut.hpp:50-69's, only the type
 * differs. */
uint64_t bqo_build_lut_dp_f32(const float* x, unsigned mu, float* out) {
    float e0 = 0.0f;
    for (unsigned t = 0; t < mu; ++t) e0 -= x[t];
    out[0] = e0;
    for (unsigned i = 1; i < mu; ++i) {
        const float step = 2.0f * x[i - 1];
        const size_t half = (size_t)1 << (i - 1);
        for (size_t j = 0; j < half; ++j) out[j + half] = out[j] + step;
    }
    const size_t table = (size_t)1 << mu;
    for (size_t k = 0; k < table / 2; ++k) out[table - 1 - k] = -out[k];
    return (uint64_t)table + mu - 1;
}

/* lut.hpp:71-105 LutBlock::index: table-major (layout 0) = group*b*2^mu +
 * t*2^mu + k; key-major (layout 1) = group*b*2^mu + k*b + t. */
static size_t lut_index(size_t group, size_t t, uint32_t k, size_t b, unsigned mu,
                        int key_major) {
    const size_t ts = (size_t)1 << mu;
    const size_t base = group * b * ts;
    return key_major ? base + (size_t)k * b + t : base + t * ts + k;
}

/* lut.hpp:109-154 build_lut_block: tables for groups [g0, g0+count) of an
 * x_rows x b input; sub-vector rows >= x_rows are zero.  builder 0 = DP,
 * 1 = naive.  double entries.  Returns counted ops. */
uint64_t bqo_build_lut_block_f64(const float* x, size_t x_rows, size_t b,
                                 size_t g0, size_t count, unsigned mu,
                                 int key_major, int naive, double* entries) {
    const size_t table = (size_t)1 << mu;
    double sub[16];
    double* tmp = (double*)malloc(sizeof(double) * table);
    uint64_t ops = 0;
    for (size_t gl = 0; gl < count; ++gl) {
        const size_t g = g0 + gl;
        for (size_t col = 0; col < b; ++col) {
            for (unsigned t = 0; t < mu; ++t) {
                const size_t r = g * mu + t;
                sub[t] = r < x_rows ? (double)x[r * b + col] : 0.0;
            }
            ops += naive ? bqo_build_lut_naive_f64(sub, mu, tmp)
                         : bqo_build_lut_dp_f64(sub, mu, tmp);
            for (size_t k = 0; k < table; ++k)
                entries[lut_index(gl, col, (uint32_t)k, b, mu, key_major)] = tmp[k];
        }
    }
    free(tmp);
    return ops;
}

/* Same block build, DP in fp32 (GPU precision), for bit-exact LUT parity. */
uint64_t bqo_build_lut_block_f32(const float* x, size_t x_rows, size_t b,
                                 size_t g0, size_t count, unsigned mu,
                                 int key_major, float* entries) {
    const size_t table = (size_t)1 << mu;
    float sub[16];
    float* tmp = (float*)malloc(sizeof(float) * table);
    uint64_t ops = 0;
    for (size_t gl = 0; gl < count; ++gl) {
        const size_t g = g0 + gl;
        for (size_t col = 0; col < b; ++col) {
            for (unsigned t = 0; t < mu; ++t) {
                const size_t r = g * mu + t;
                sub[t] = r < x_rows ? x[r * b + col] : 0.0f;
            }
            ops += bqo_build_lut_dp_f32(sub, mu, tmp);
            for (size_t k = 0; k < table; ++k)
                entries[lut_index(gl, col, (uint32_t)k, b, mu, key_major)] = tmp[k];
        }
    }
    free(tmp);
    return ops;
}

/* kernel.hpp:116-204 detail::run<float> (+ biqgemm 246-258, biqgemm_plane
 * 209-215 when alpha == NULL).  Per plane i the accumulator acc_i(r,col) is
 * the fp64 sum of LUT entries over ascending group index; the epilogue
 * y(r,col) = float(sum_i alpha_i[r] * acc_i(r,col)) in fp64 over ascending i
 * (alpha = 1 in plane mode).  Tiling and threading do not change the result
 * (criterion 7), so the restatement uses one tile covering all groups.
 * keys: beta x m x G (u32).  counters[0..2] = build ops, lookups,
 * accumulate ops (kernel.hpp:179-180). */
int bqo_biqgemm_ex_f32(const uint32_t* keys, const float* alpha, size_t m, size_t n,
                       unsigned beta, unsigned mu, const float* x, size_t x_rows,
                       size_t b, int naive, float* y, uint64_t* counters);

int bqo_biqgemm_f32(const uint32_t* keys, const float* alpha, size_t m, size_t n,
                    unsigned beta, unsigned mu, const float* x, size_t x_rows,
                    size_t b, float* y, uint64_t* counters) {
    return bqo_biqgemm_ex_f32(keys, alpha, m, n, beta, mu, x, x_rows, b, 0, y, counters);
}

/* The same with KernelOptions::builder (kernel.hpp:51,158): naive != 0
 * builds every table with build_lut_naive (lut.hpp:31-43) instead of the DP. */
int bqo_biqgemm_ex_f32(const uint32_t* keys, const float* alpha, size_t m, size_t n,
                       unsigned beta, unsigned mu, const float* x, size_t x_rows,
                       size_t b, int naive, float* y, uint64_t* counters) {
    if (mu < 1 || mu > 16 || beta == 0) return BQO_EINVAL;
    const size_t groups = (n + mu - 1) / mu;
    if ((size_t)mu * groups < x_rows) return BQO_EINVAL; /* kernel.hpp:132-134 */
    const size_t table = (size_t)1 << mu;
    const int key_major = b > 1; /* kernel.hpp:146 */
    double* lut = (double*)malloc(sizeof(double) * groups * b * table);
    double* acc = (double*)calloc((size_t)beta * m * b, sizeof(double));
    if (!lut || !acc) { free(lut); free(acc); return BQO_EINVAL; }
    const uint64_t ops = bqo_build_lut_block_f64(x, x_rows, b, 0, groups, mu,
                                                 key_major, naive, lut);
    for (unsigned i = 0; i < beta; ++i) {
        const uint32_t* kp = keys + (size_t)i * m * groups;
        double* ai = acc + (size_t)i * m * b;
        for (size_t r = 0; r < m; ++r) {
            for (size_t g = 0; g < groups; ++g) {
                const uint32_t k = kp[r * groups + g];
                for (size_t col = 0; col < b; ++col)
                    ai[r * b + col] += lut[lut_index(g, col, k, b, mu, key_major)];
            }
        }
    }
    for (size_t r = 0; r < m; ++r) {
        for (size_t col = 0; col < b; ++col) {
            double s = 0.0;
            for (unsigned i = 0; i < beta; ++i) {
                const double a = alpha ? (double)alpha[(size_t)i * m + r] : 1.0;
                s += a * acc[((size_t)i * m + r) * b + col];
            }
            y[r * b + col] = (float)s;
        }
    }
    if (counters) {
        counters[0] = ops;
        counters[1] = (uint64_t)m * groups * b * beta;
        counters[2] = counters[1];
    }
    free(lut);
    free(acc);
    return BQO_OK;
}

/* baselines.hpp:14-36 gemm_dense<float>: y(r,c) = float(sum_k double(a)*double(x)). */
int bqo_gemm_dense_f32(const float* a, size_t m, size_t n, const float* x,
                       size_t b, float* y) {
    for (size_t r = 0; r < m; ++r) {
        for (size_t col = 0; col < b; ++col) {
            double acc = 0.0;
            for (size_t k = 0; k < n; ++k) acc += (double)a[r * n + k] * (double)x[k * b + col];
            y[r * b + col] = (float)acc;
        }
    }
    return BQO_OK;
}

/* kernel.hpp:58-70 plan_tiles. Returns 0 and fills t_w/t_h, or EINVAL
 * when the budget is below one group's tables. */
int bqo_plan_tiles(size_t m, size_t groups, size_t b, unsigned mu, size_t budget,
                   size_t entry_bytes, size_t* t_w, size_t* t_h) {
    const size_t per_group = ((size_t)1 << mu) * b * entry_bytes;
    if (per_group == 0 || budget < per_group) return BQO_EINVAL;
    size_t tw = budget / per_group;
    if (tw > groups) tw = groups;
    size_t th = budget / (tw * 4u);
    if (th < 1) th = 1;
    if (th > m) th = m;
    *t_w = tw;
    *t_h = th;
    return BQO_OK;
}

/* matrix.hpp:87-110 frobenius_distance / frobenius_norm (fp64). */
double bqo_frobenius_distance_f32(const float* a, const float* b, size_t count) {
    double acc = 0.0;
    for (size_t i = 0; i < count; ++i) {
        const double d = (double)a[i] - (double)b[i];
        acc += d * d;
    }
    return sqrt(acc);
}

double bqo_frobenius_norm_f32(const float* a, size_t count) {
    double acc = 0.0;
    for (size_t i = 0; i < count; ++i) acc += (double)a[i] * (double)a[i];
    return sqrt(acc);
}
