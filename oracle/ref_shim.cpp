// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference.
//
// oracle/Makefile compiles this file together with the reference's own
// P/src/compression.cpp (P/ = /root/reference/proj/, read in place, never
// copied) into oracle/_ref/libswarmsim_ref.so.  Tests use it to pin the C
// restatement (codec_oracle.c) and to generate tests/golden/; bench.py's
// `--impl reference` / cpu_baseline leg times it on the host cores.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "swarmsim/compression.hpp"
#include "swarmsim/errors.hpp"

using namespace swarmsim;

extern "C" {

// 0 ok, 1 ConfigError (any message), 3 other exception
int ref_quantize_blockwise(const double* x, size_t n, size_t bs, int8_t* codes, double* absmax,
                           size_t* n_blocks) {
    try {
        std::vector<double> v(x, x + n);
        const auto q = compress::quantize_blockwise(v, bs);
        std::memcpy(codes, q.codes.data(), q.codes.size());
        std::memcpy(absmax, q.absmax.data(), q.absmax.size() * sizeof(double));
        if (n_blocks) *n_blocks = q.n_blocks();
        return 0;
    } catch (const ConfigError&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

int ref_dequantize_blockwise(const int8_t* codes, size_t n, const double* absmax, size_t n_blocks,
                             size_t bs, double* out) {
    try {
        compress::QuantizedTensor q;
        q.codes.assign(codes, codes + n);
        q.absmax.assign(absmax, absmax + n_blocks);
        q.block_size = bs;
        const auto y = compress::dequantize_blockwise(q);
        std::memcpy(out, y.data(), n * sizeof(double));
        return 0;
    } catch (...) {
        return 3;
    }
}

int ref_maxout_k(const double* x, size_t n, size_t k, double* out) {
    try {
        std::vector<double> v(x, x + n);
        const auto y = compress::maxout_k(v, k);
        std::memcpy(out, y.data(), y.size() * sizeof(double));
        return 0;
    } catch (const ConfigError&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

int ref_layer_norm(const double* x, size_t n, const double* gain, const double* bias, double eps,
                   double* out) {
    try {
        std::vector<double> v(x, x + n);
        compress::LayerNormParams p;
        if (gain) p.gain.assign(gain, gain + n);
        if (bias) p.bias.assign(bias, bias + n);
        p.epsilon = eps;
        const auto y = compress::layer_norm(v, p);
        std::memcpy(out, y.data(), n * sizeof(double));
        return 0;
    } catch (const ConfigError&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

int ref_bottleneck_forward(const double* x, size_t m, const double* w_c, size_t c, double eps,
                           double* out) {
    try {
        std::vector<double> v(x, x + m);
        std::vector<std::vector<double>> w(m, std::vector<double>(c));
        for (size_t i = 0; i < m; ++i) std::copy(w_c + i * c, w_c + (i + 1) * c, w[i].begin());
        compress::LayerNormParams p;
        p.epsilon = eps;
        const auto y = compress::bottleneck_forward(v, w, p);
        std::memcpy(out, y.data(), y.size() * sizeof(double));
        return 0;
    } catch (const ConfigError&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

double ref_payload_bits(int64_t d_model, int64_t seq_len, int64_t batch, double act_bytes,
                        int kind, double factor) {
    cost_model::LayerShape s;
    s.d_model = d_model;
    s.d_ffn = 4 * d_model;
    s.n_heads = 1;
    s.seq_len = seq_len;
    s.batch = batch;
    s.activation_bytes_per_element = act_bytes;
    try {
        return compress::payload_bits(s, {static_cast<compress::Kind>(kind), factor});
    } catch (...) {
        return -1.0;
    }
}

// std::mt19937_64 stream, to pin the C restatement of the generator.
void ref_mt64(uint64_t seed, size_t n, uint64_t* out) {
    std::mt19937_64 rng(seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng();
}

// ---------------------------------------------------------------------------
// CPU baseline: the reference codec, unmodified, on block-aligned chunks over
// `threads` host threads (bit-identical to one call because blocks are
// independent).  Inputs are prepared as the reference's own argument type
// (std::vector<double>) BEFORE the timed call by ref_codec_prepare.
struct RefCodecJob {
    std::vector<std::vector<double>> chunks;
    std::vector<compress::QuantizedTensor> out;
    size_t bs = 0;
};

void* ref_codec_prepare(const float* x, size_t n, size_t bs, int threads) {
    auto* job = new RefCodecJob;
    job->bs = bs;
    const size_t n_blocks = (n + bs - 1) / bs;
    const size_t per = (n_blocks + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const size_t b0 = std::min(n_blocks, per * t), b1 = std::min(n_blocks, per * (t + 1));
        const size_t e0 = std::min(n, b0 * bs), e1 = std::min(n, b1 * bs);
        job->chunks.emplace_back(x + e0, x + e1);
    }
    job->out.resize(job->chunks.size());
    return job;
}

// Runs quantize (+ dequantize when `roundtrip`) on all chunks; returns codes
// checksum so the work cannot be elided.
uint64_t ref_codec_run(void* handle, int roundtrip) {
    auto* job = static_cast<RefCodecJob*>(handle);
    std::vector<std::thread> pool;
    std::vector<uint64_t> sums(job->chunks.size(), 0);
    for (size_t t = 0; t < job->chunks.size(); ++t) {
        pool.emplace_back([job, t, roundtrip, &sums] {
            job->out[t] = compress::quantize_blockwise(job->chunks[t], job->bs);
            uint64_t s = 0;
            for (int8_t c : job->out[t].codes) s = s * 31 + static_cast<uint8_t>(c);
            if (roundtrip) {
                const auto y = compress::dequantize_blockwise(job->out[t]);
                s += static_cast<uint64_t>(y.empty() ? 0.0 : y.back() * 1e6);
            }
            sums[t] = s;
        });
    }
    for (auto& th : pool) th.join();
    uint64_t s = 0;
    for (auto v : sums) s ^= v;
    return s;
}

void ref_codec_codes(void* handle, int8_t* codes, float* scales) {
    auto* job = static_cast<RefCodecJob*>(handle);
    size_t off = 0, boff = 0;
    for (auto& q : job->out) {
        std::memcpy(codes + off, q.codes.data(), q.codes.size());
        for (size_t b = 0; b < q.absmax.size(); ++b) scales[boff + b] = static_cast<float>(q.absmax[b]);
        off += q.codes.size();
        boff += q.absmax.size();
    }
}

void ref_codec_free(void* handle) { delete static_cast<RefCodecJob*>(handle); }

}  // extern "C"
