/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the SWARM boundary codec.
 *
 * This file is a plain-C restatement of the reference's numeric operators
 * (swarmsim::compress, /root/reference/proj/src/compression.cpp).  It exists so
 * that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can CHECK
 * the CUDA path.  Nothing in paper_2301_11913_b200/ links, imports or calls it;
 * the product path fails loudly when its CUDA library is missing.
 *
 * Parity pinning: every function here is checked (tests/test_oracle.py) against
 *   (1) the known-answer vectors of P/tests/test_compression.cpp:14-136,
 *   (2) the reference itself compiled from /root/reference sources into
 *       oracle/_ref/libswarmsim_ref.so (oracle/Makefile), through the golden
 *       fixtures committed in tests/golden/ (tests/golden/make_golden.py).
 *
 * Citations use P/ = /root/reference/proj/.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#define ORC_OK 0
#define ORC_E_INVALID 1
#define ORC_E_NONFINITE 2

/* ---------------------------------------------------------------------------
 * std::mt19937_64 (the generator every reference test uses, e.g.
 * P/tests/acceptance.cpp:356, P/tests/test_compression.cpp:54), restated so the
 * reference's seeded inputs can be regenerated without C++.
 * ------------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} orc_mt64;

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* g) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    if (g->idx >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ MAG[x & 1ULL];
        }
        for (; i < 311; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[i + 1] & LM);
            g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ MAG[x & 1ULL];
        }
        uint64_t x = (g->mt[311] & UM) | (g->mt[0] & LM);
        g->mt[311] = g->mt[155] ^ (x >> 1) ^ MAG[x & 1ULL];
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

static double u53(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }

/* P/tests/acceptance.cpp:356-362: 10^6 values, seed 2026, every ~11th scaled 1000. */
void orc_gen_acceptance(uint64_t seed, size_t n, double* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) {
        const double u = u53(&g);
        out[i] = (u - 0.5) * ((orc_mt64_next(&g) % 11 == 0) ? 1000.0 : 2.0);
    }
}

/* P/tests/test_compression.cpp:54-61: 100k heavy-tailed values, seed 123. */
void orc_gen_heavy_tailed(uint64_t seed, size_t n, double* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) {
        const double u = u53(&g);
        out[i] = (u - 0.5) * ((orc_mt64_next(&g) % 7 == 0) ? 100.0 : 1.0);
    }
}

/*
 * Codec-sweep input: uniform(-1,1), every 11th value
 * x500, plus, per `block`-sized block, an anchor of exactly 508 at the block
 * start and exact/near half-step ties (x = ±2(2m+1), 127x/508 = m+0.5) every
 * 13th element, so the tie-breaking rule of compression.cpp:24 is exercised.
 */
void orc_gen_sweep_f32(uint64_t seed, size_t n, size_t block, float* out) {
    orc_mt64 g;
    orc_mt64_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) {
        double v = 2.0 * u53(&g) - 1.0;
        if (i % 11 == 0) v *= 500.0;
        float f = (float)v;
        const size_t j = block ? (i % block) : i;
        if (j == 0) {
            f = 508.0f;
        } else if (j % 13 == 0) {
            const uint64_t r = orc_mt64_next(&g);
            const int m = (int)(r % 127);             /* 0..126 */
            float t = (float)(2 * (2 * m + 1));       /* exact tie */
            const int variant = (int)((r >> 8) % 3);  /* tie, just above, just below */
            if (variant == 1) t = nextafterf(t, INFINITY);
            if (variant == 2) t = nextafterf(t, 0.0f);
            f = ((r >> 16) & 1) ? -t : t;
        }
        out[i] = f;
    }
}

/* ---------------------------------------------------------------------------
 * quantize_blockwise — P/src/compression.cpp:10-29.
 * Validation order follows :11-14 (block_size first, then any non-finite).
 * Per block: absmax = max |x| (:21); code = round(127*x/absmax) with C round()
 * (half away from zero), clamped to [-127,127], 0 for an all-zero block (:23-25).
 * ------------------------------------------------------------------------- */
int orc_quantize_f64(const double* x, size_t n, size_t bs, int8_t* codes, double* absmax_out) {
    if (bs == 0) return ORC_E_INVALID;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return ORC_E_NONFINITE;
    size_t b = 0;
    for (size_t begin = 0; begin < n; begin += bs, ++b) {
        const size_t end = begin + bs < n ? begin + bs : n;
        double a = 0.0;
        for (size_t i = begin; i < end; ++i) {
            const double m = fabs(x[i]);
            a = a < m ? m : a; /* std::max(a, m) */
        }
        absmax_out[b] = a;
        for (size_t i = begin; i < end; ++i) {
            double c = a > 0.0 ? round(127.0 * x[i] / a) : 0.0;
            if (c < -127.0) c = -127.0;
            if (c > 127.0) c = 127.0;
            codes[i] = (int8_t)c;
        }
    }
    return ORC_OK;
}

/* fp32 wire variant: identical math on the exactly-promoted inputs; the per-block
 * scale is the fp32 absmax (exact, since max|x| of fp32 values is an fp32 value). */
int orc_quantize_f32(const float* x, size_t n, size_t bs, int8_t* codes, float* scales) {
    if (bs == 0) return ORC_E_INVALID;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return ORC_E_NONFINITE;
    size_t b = 0;
    for (size_t begin = 0; begin < n; begin += bs, ++b) {
        const size_t end = begin + bs < n ? begin + bs : n;
        double a = 0.0;
        for (size_t i = begin; i < end; ++i) {
            const double m = fabs((double)x[i]);
            a = a < m ? m : a;
        }
        scales[b] = (float)a;
        for (size_t i = begin; i < end; ++i) {
            double c = a > 0.0 ? round(127.0 * (double)x[i] / a) : 0.0;
            if (c < -127.0) c = -127.0;
            if (c > 127.0) c = 127.0;
            codes[i] = (int8_t)c;
        }
    }
    return ORC_OK;
}

static float bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* round-to-nearest-even of a double to bf16 (no double rounding through fp32) */
static uint16_t f64_to_bf16(double d) {
    if (isnan(d)) return 0x7FC0;
    uint64_t u;
    memcpy(&u, &d, 8);
    const uint64_t sign = u >> 63;
    const double ad = fabs(d);
    if (ad == 0.0) return (uint16_t)(sign << 15);
    /* bf16 has 8 exponent bits like fp32; compute via exact scaling */
    int e;
    double m = frexp(ad, &e); /* ad = m * 2^e, m in [0.5,1) */
    /* normal bf16 range: exponent (e-1) in [-126, 127] */
    int ue = e - 1;
    double q;
    if (ue < -126) { /* subnormal: step 2^-133 */
        q = ldexp(ad, 133);
        double r = nearbyint(q); /* ties-to-even under default rounding mode */
        float f = (float)ldexp(r, -133);
        uint32_t fu;
        memcpy(&fu, &f, 4);
        return (uint16_t)((sign << 15) | (fu >> 16));
    }
    q = ldexp(m, 8); /* 8 significant bits: [128, 256) */
    double r = nearbyint(q);
    double v = ldexp(r, e - 8);
    if (v > 3.3895313892515355e38) v = INFINITY; /* overflow past bf16 max */
    float f = (float)v; /* exact: v has 8 significant bits */
    uint32_t fu;
    memcpy(&fu, &f, 4);
    return (uint16_t)((sign << 15) | (fu >> 16));
}

int orc_quantize_bf16(const uint16_t* x, size_t n, size_t bs, int8_t* codes, float* scales) {
    if (bs == 0) return ORC_E_INVALID;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(bf16_to_f32(x[i]))) return ORC_E_NONFINITE;
    size_t b = 0;
    for (size_t begin = 0; begin < n; begin += bs, ++b) {
        const size_t end = begin + bs < n ? begin + bs : n;
        double a = 0.0;
        for (size_t i = begin; i < end; ++i) {
            const double m = fabs((double)bf16_to_f32(x[i]));
            a = a < m ? m : a;
        }
        scales[b] = (float)a;
        for (size_t i = begin; i < end; ++i) {
            double c = a > 0.0 ? round(127.0 * (double)bf16_to_f32(x[i]) / a) : 0.0;
            if (c < -127.0) c = -127.0;
            if (c > 127.0) c = 127.0;
            codes[i] = (int8_t)c;
        }
    }
    return ORC_OK;
}

/* dequantize_blockwise — P/src/compression.cpp:31-37: x = code * absmax[i/bs] / 127.0 */
void orc_dequantize_f64(const int8_t* codes, size_t n, const double* absmax, size_t bs, double* out) {
    for (size_t i = 0; i < n; ++i) out[i] = (double)codes[i] * absmax[i / bs] / 127.0;
}

/* fp32 / bf16 outputs: the reference's fp64 value rounded once to the output type. */
void orc_dequantize_f32(const int8_t* codes, size_t n, const float* scales, size_t bs, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = (float)((double)codes[i] * (double)scales[i / bs] / 127.0);
}

void orc_dequantize_bf16(const int8_t* codes, size_t n, const float* scales, size_t bs, uint16_t* out) {
    for (size_t i = 0; i < n; ++i)
        out[i] = f64_to_bf16((double)codes[i] * (double)scales[i / bs] / 127.0);
}

uint16_t orc_f64_to_bf16(double d) { return f64_to_bf16(d); }

/* maxout_k — P/src/compression.cpp:39-50. std::max(m, v) keeps m unless m < v,
 * so the earliest of tied maxima wins; `argmax` (optional) records which. */
int orc_maxout_f64(const double* x, size_t n, size_t k, double* out, uint8_t* argmax) {
    if (k == 0 || n % k != 0) return ORC_E_INVALID;
    for (size_t j = 0; j < n / k; ++j) {
        double m = x[j * k];
        size_t am = 0;
        for (size_t i = 1; i < k; ++i) {
            if (m < x[j * k + i]) {
                m = x[j * k + i];
                am = i;
            }
        }
        out[j] = m;
        if (argmax) argmax[j] = (uint8_t)am;
    }
    return ORC_OK;
}

/* layer_norm — P/src/compression.cpp:52-74: two-pass mean / biased variance,
 * (x-mean)/sqrt(var+eps), then optional gain and bias (NULL = ones / zeros). */
int orc_layer_norm_f64(const double* x, size_t n, const double* gain, const double* bias, double eps,
                       double* out) {
    if (n == 0) return ORC_E_INVALID;
    double mean = 0.0;
    for (size_t i = 0; i < n; ++i) mean += x[i];
    mean /= (double)n;
    double var = 0.0;
    for (size_t i = 0; i < n; ++i) var += (x[i] - mean) * (x[i] - mean);
    var /= (double)n;
    const double inv = 1.0 / sqrt(var + eps);
    for (size_t i = 0; i < n; ++i) {
        double o = (x[i] - mean) * inv;
        if (gain) o *= gain[i];
        if (bias) o += bias[i];
        out[i] = o;
    }
    return ORC_OK;
}

/* bottleneck matvec — P/src/compression.cpp:78-101: out[j] = sum_i x[i] * w[i][j],
 * accumulated in i order; w is row-major rows x cols. */
void orc_matvec_f64(const double* x, size_t rows, const double* w, size_t cols, double* out) {
    for (size_t j = 0; j < cols; ++j) out[j] = 0.0;
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) out[j] += x[i] * w[i * cols + j];
}
