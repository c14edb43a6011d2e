// swarmsim::compress / cost_model compatibility layer over the C-ABI.
//
// Same signatures, defaults, validation order and exception types as the
// reference (P/include/swarmsim/compression.hpp, P/src/compression.cpp), but
// every numeric operator runs on the B200: host vector -> H2D -> sm_100a kernel
// -> D2H, returned by value like the reference.  There is no CPU fallback: if
// the device path fails, the call throws std::runtime_error.
#include <algorithm>
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "swarm_b200.h"
#include "swarmsim/compression.hpp"
#include "swarmsim/errors.hpp"

namespace swarmsim {
namespace {

[[noreturn]] void raise(int rc, const char* what) {
    std::string msg = swarm_last_error();
    if (msg.empty()) msg = what;
    if (rc == SWARM_E_INVALID || rc == SWARM_E_NONFINITE) throw ConfigError(msg);
    throw std::runtime_error(std::string(what) + ": device path failed: " + msg);
}

void check(int rc, const char* what) {
    if (rc != SWARM_OK) raise(rc, what);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer for the by-value compat calls (not on the training hot path)
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

std::vector<double> matvec(const std::vector<double>& x, const std::vector<std::vector<double>>& w, const char* who) {
    // validation order of compression.cpp:80-84
    if (w.size() != x.size()) throw ConfigError(std::string(who) + ": weight row count mismatch");
    const size_t cols = w.empty() ? 0 : w.front().size();
    for (const auto& row : w)
        if (row.size() != cols) throw ConfigError(std::string(who) + ": ragged weight matrix");
    std::vector<double> out(cols, 0.0);
    if (cols == 0) return out;
    const size_t rows = x.size();
    std::vector<double> flat(rows * cols);
    for (size_t i = 0; i < rows; ++i) std::copy(w[i].begin(), w[i].end(), flat.begin() + i * cols);
    DevBuf dx(rows * sizeof(double)), dw(flat.size() * sizeof(double)), dout(cols * sizeof(double));
    if (rows) {
        cuda_check(cudaMemcpy(dx.p, x.data(), rows * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(dw.p, flat.data(), flat.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    }
    check(swarm_matvec_f64(dx.as<double>(), rows, dw.as<double>(), cols, dout.as<double>(), nullptr), who);
    cuda_check(cudaMemcpy(out.data(), dout.p, cols * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    return out;
}

}  // namespace

namespace compress {

QuantizedTensor quantize_blockwise(const std::vector<double>& x, std::size_t block_size) {
    if (block_size == 0) throw ConfigError("quantize_blockwise: block_size must be positive");
    QuantizedTensor q;
    q.block_size = block_size;
    q.codes.resize(x.size());
    q.absmax.resize((x.size() + block_size - 1) / block_size);
    const int rc = swarm_quantize_blockwise_host(x.data(), SWARM_DTYPE_F64, x.size(), block_size, q.codes.data(),
                                                 q.absmax.data());
    if (rc == SWARM_E_NONFINITE) throw ConfigError("quantize_blockwise: non-finite input");
    check(rc, "quantize_blockwise");
    return q;
}

std::vector<double> dequantize_blockwise(const QuantizedTensor& q) {
    std::vector<double> x(q.codes.size());
    if (q.codes.empty()) return x;
    if (q.block_size == 0) throw ConfigError("dequantize_blockwise: block_size must be positive");
    if (q.absmax.size() < (q.codes.size() + q.block_size - 1) / q.block_size)
        throw ConfigError("dequantize_blockwise: absmax has fewer entries than blocks");
    check(swarm_dequantize_blockwise_host(q.codes.data(), q.absmax.data(), SWARM_DTYPE_F64, q.codes.size(),
                                          q.block_size, x.data(), SWARM_DTYPE_F64),
          "dequantize_blockwise");
    return x;
}

std::vector<double> maxout_k(const std::vector<double>& x, std::size_t k) {
    if (k == 0 || x.size() % k != 0) throw ConfigError("maxout_k: k must divide the input length");
    std::vector<double> out(x.size() / k);
    if (out.empty()) return out;
    DevBuf dx(x.size() * sizeof(double)), dout(out.size() * sizeof(double));
    cuda_check(cudaMemcpy(dx.p, x.data(), x.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    check(swarm_maxout_forward(dx.p, SWARM_DTYPE_F64, x.size(), k, dout.p, nullptr, nullptr), "maxout_k");
    cuda_check(cudaMemcpy(out.data(), dout.p, out.size() * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    return out;
}

std::vector<double> layer_norm(const std::vector<double>& x, const LayerNormParams& params) {
    if (x.empty()) throw ConfigError("layer_norm: empty input");
    if (!params.gain.empty() && params.gain.size() != x.size()) throw ConfigError("layer_norm: gain size mismatch");
    if (!params.bias.empty() && params.bias.size() != x.size()) throw ConfigError("layer_norm: bias size mismatch");
    const size_t n = x.size(), bytes = n * sizeof(double);
    DevBuf dx(bytes), dg(params.gain.empty() ? 0 : bytes), db(params.bias.empty() ? 0 : bytes), dout(bytes);
    cuda_check(cudaMemcpy(dx.p, x.data(), bytes, cudaMemcpyHostToDevice), "H2D");
    if (dg.p) cuda_check(cudaMemcpy(dg.p, params.gain.data(), bytes, cudaMemcpyHostToDevice), "H2D");
    if (db.p) cuda_check(cudaMemcpy(db.p, params.bias.data(), bytes, cudaMemcpyHostToDevice), "H2D");
    check(swarm_layer_norm_forward(dx.p, SWARM_DTYPE_F64, 1, n, dg.p, db.p, params.epsilon, dout.p, nullptr, nullptr,
                                   nullptr),
          "layer_norm");
    std::vector<double> out(n);
    cuda_check(cudaMemcpy(out.data(), dout.p, bytes, cudaMemcpyDeviceToHost), "D2H");
    return out;
}

std::vector<double> bottleneck_forward(const std::vector<double>& x, const std::vector<std::vector<double>>& w_c,
                                       const LayerNormParams& params) {
    return matvec(layer_norm(x, params), w_c, "bottleneck_forward");
}

std::vector<double> bottleneck_decompress(const std::vector<double>& y, const std::vector<std::vector<double>>& w_d) {
    return matvec(y, w_d, "bottleneck_decompress");
}

void CompressionSpec::validate() const {
    if (kind == Kind::Bottleneck && (factor <= 0.0 || factor > 1.0))
        throw ConfigError("CompressionSpec: bottleneck factor must be in (0,1]");
    if (kind == Kind::Maxout && (factor < 1.0 || factor != std::floor(factor)))
        throw ConfigError("CompressionSpec: maxout factor must be an integer >= 1");
}

Kind kind_from_name(const std::string& name) {
    static const std::pair<const char*, Kind> table[] = {
        {"none", Kind::None}, {"int8", Kind::Int8}, {"bottleneck", Kind::Bottleneck}, {"maxout", Kind::Maxout}};
    for (const auto& [n, k] : table)
        if (name == n) return k;
    throw ConfigError("unknown compression kind: " + name);
}

std::string kind_name(Kind k) {
    switch (k) {
        case Kind::Int8: return "int8";
        case Kind::Bottleneck: return "bottleneck";
        case Kind::Maxout: return "maxout";
        default: return "none";
    }
}

// Bits per microbatch on the wire (compression.cpp:139-152): int8 counts one
// byte per element (scales excluded, so it is exactly half of fp16).
double payload_bits(const cost_model::LayerShape& shape, const CompressionSpec& spec) {
    spec.validate();
    const double elems = static_cast<double>(shape.batch) * static_cast<double>(shape.seq_len) *
                         static_cast<double>(shape.d_model);
    const double base = elems * shape.activation_bytes_per_element * 8.0;
    switch (spec.kind) {
        case Kind::Int8: return elems * 8.0;
        case Kind::Bottleneck: return base * spec.factor;
        case Kind::Maxout: return base / spec.factor;
        default: return base;
    }
}

}  // namespace compress

namespace cost_model {

void LayerShape::validate() const {
    const bool positive = d_model > 0 && d_ffn > 0 && n_heads > 0 && seq_len > 0 && batch > 0 &&
                          layers_per_stage > 0 && activation_bytes_per_element > 0.0;
    if (!positive) throw ConfigError("LayerShape: all fields must be strictly positive");
    if (d_model % n_heads != 0) throw ConfigError("LayerShape: n_heads must divide d_model");
}

// Wqkv (d x 3d) + Wo (d x d) + W1 (d x d_ffn) + W2 (d_ffn x d), no biases (cost_model.cpp:31-35)
std::int64_t params_per_layer(const LayerShape& s) {
    s.validate();
    return 4 * s.d_model * s.d_model + 2 * s.d_model * s.d_ffn;
}

// 2 FLOP per parameter per token forward; backward = 2x forward (cost_model.cpp:37-42)
double flops_per_stage(const LayerShape& s, bool include_backward) {
    const double fwd = 2.0 * static_cast<double>(params_per_layer(s)) * static_cast<double>(s.batch) *
                       static_cast<double>(s.seq_len) * static_cast<double>(s.layers_per_stage);
    return include_backward ? 3.0 * fwd : fwd;
}

double activation_payload_bits(const LayerShape& s) {
    s.validate();
    return static_cast<double>(s.batch) * static_cast<double>(s.seq_len) * static_cast<double>(s.d_model) *
           s.activation_bytes_per_element * 8.0;
}

void DeviceProfile::validate() const {
    if (effective_flops <= 0.0 || upload_bps <= 0.0 || download_bps <= 0.0)
        throw ConfigError("DeviceProfile: flops and bandwidths must be positive");
    if (rtt_seconds < 0.0) throw ConfigError("DeviceProfile: rtt_seconds must be nonnegative");
}

// compute = stage FLOPs / effective FLOP/s; comm = activations out + gradients back
// plus one latency each way; overlapped -> max (cost_model.cpp:50-66)
CostBreakdown stage_cost(const LayerShape& shape, const DeviceProfile& device, bool overlap) {
    device.validate();
    CostBreakdown out;
    out.compute_seconds = flops_per_stage(shape, true) / device.effective_flops;
    const double payload = activation_payload_bits(shape);
    out.comm_seconds = payload / device.upload_bps + payload / device.download_bps + 2.0 * device.rtt_seconds;
    out.total_seconds = overlap ? std::max(out.compute_seconds, out.comm_seconds) : out.compute_seconds + out.comm_seconds;
    out.utilization = out.compute_seconds / out.total_seconds;
    out.idle_fraction = 1.0 - out.utilization;
    return out;
}

double square_cube_ratio(const LayerShape& shape) {
    return flops_per_stage(shape, true) / activation_payload_bits(shape);
}

DeviceProfile calibrated_profile(const LayerShape& shape, double measured_visit_seconds, double link_bps,
                                 double link_rtt_seconds) {
    if (!(measured_visit_seconds > 0.0)) throw ConfigError("calibrated_profile: visit time must be positive");
    DeviceProfile d;
    d.effective_flops = flops_per_stage(shape, true) / measured_visit_seconds;
    d.upload_bps = link_bps;
    d.download_bps = link_bps;
    d.rtt_seconds = link_rtt_seconds;
    d.validate();
    return d;
}

// PAPER:292 / cost_model.cpp:72-80 presets ("ours" ships int8 activations)
LayerShape preset(std::string_view name) {
    LayerShape s;
    if (name == "base") s = {768, 3072, 12, 512, 1, 1, 2.0};
    else if (name == "xxlarge") s = {4096, 16384, 32, 512, 1, 1, 2.0};
    else if (name == "gpt3") s = {12288, 49152, 96, 512, 1, 1, 2.0};
    else if (name == "ours") s = {4096, 16384, 32, 512, 1, 3, 1.0};
    else throw ConfigError("unknown preset: " + std::string(name));
    return s;
}

std::vector<std::string> preset_names() { return {"base", "xxlarge", "gpt3", "ours"}; }

}  // namespace cost_model
}  // namespace swarmsim
