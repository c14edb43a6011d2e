// Training building blocks around the GEMMs of the stage executor (sm_100a):
// token embedding, attention softmax forward/backward, fused LM-head
// cross-entropy, fused AdamW over the flat parameter arena, and init.
// All are bandwidth-bound; each touches its operands once with coalesced,
// vectorised accesses where the layout allows.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace swarm {
namespace {

unsigned grid_for(size_t work, unsigned per_block, unsigned cap = 148u * 32u) {
    const size_t g = (work + per_block - 1) / per_block;
    return static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(g, cap)));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------- embedding --
__global__ void k_embed_fwd(const int32_t* __restrict__ tok, int n, const uint4* __restrict__ table, int vocab,
                            int d8, uint4* __restrict__ out) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += warps) {
        const int id = tok[t];
        const bool ok = id >= 0 && id < vocab;
        for (int c = lane; c < d8; c += 32)
            out[static_cast<size_t>(t) * d8 + c] = ok ? table[static_cast<size_t>(id) * d8 + c] : make_uint4(0, 0, 0, 0);
    }
}

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__global__ void k_embed_bwd(const int32_t* __restrict__ tok, int n, const T* __restrict__ dout,
                            int vocab, int d, float* __restrict__ dtable) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += warps) {
        const int id = tok[t];
        if (id < 0 || id >= vocab) continue;
        for (int c = lane; c < d; c += 32)
            atomicAdd(dtable + static_cast<size_t>(id) * d + c, to_f(dout[static_cast<size_t>(t) * d + c]));
    }
}

// --------------------------------------------------------------- softmax --
constexpr int kMaxLPerLane = 32;  // L <= 1024

template <typename T>
__global__ void k_softmax_fwd(const float* __restrict__ S, int rows, int L, int causal, T* __restrict__ P) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const float log2e = 1.4426950408889634f;
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += warps) {
        const float* s = S + static_cast<size_t>(row) * L;
        const int qi = row % L;
        float v[kMaxLPerLane];
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < kMaxLPerLane; ++k) {
            const int j = k * 32 + lane;
            float x = -INFINITY;
            if (j < L) {
                x = s[j];
                if (causal && j > qi) x = -INFINITY;
            }
            v[k] = x;
            m = fmaxf(m, x);
        }
        m = warp_max(m);
        float sum = 0.f;
#pragma unroll
        for (int k = 0; k < kMaxLPerLane; ++k) {
            // fp32 output (the fp32 arithmetic mode): expf of the difference, as the oracle
            const float e = (v[k] == -INFINITY) ? 0.f : (sizeof(T) == 4 ? expf(v[k] - m) : exp2f((v[k] - m) * log2e));
            v[k] = e;
            sum += e;
        }
        const float inv = 1.f / warp_sum(sum);
        T* p = P + static_cast<size_t>(row) * L;
#pragma unroll
        for (int k = 0; k < kMaxLPerLane; ++k) {
            const int j = k * 32 + lane;
            if (j < L) p[j] = from_f<T>(v[k] * inv);
        }
    }
}

template <typename T>
__global__ void k_softmax_bwd(const T* __restrict__ P, const float* __restrict__ dP, int rows, int L, float scale,
                              T* __restrict__ dS) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += warps) {
        const size_t base = static_cast<size_t>(row) * L;
        float p[kMaxLPerLane], g[kMaxLPerLane];
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < kMaxLPerLane; ++k) {
            const int j = k * 32 + lane;
            p[k] = j < L ? to_f(P[base + j]) : 0.f;
            g[k] = j < L ? dP[base + j] : 0.f;
            acc += p[k] * g[k];
        }
        acc = warp_sum(acc);
#pragma unroll
        for (int k = 0; k < kMaxLPerLane; ++k) {
            const int j = k * 32 + lane;
            if (j < L) dS[base + j] = from_f<T>(scale * p[k] * (g[k] - acc));
        }
    }
}

// ---------------------------------------------------------- cross-entropy --
constexpr int kCeThreads = 512;

template <typename T>
__device__ __forceinline__ float ce_exp(float x) {
    return sizeof(T) == 4 ? expf(x) : __expf(x);  // fp32 mode: the accurate exponential
}

template <typename T>
__global__ void __launch_bounds__(kCeThreads) k_cross_entropy(const float* __restrict__ logits,
                                                              const int32_t* __restrict__ targets, int vocab,
                                                              float grad_scale, float* __restrict__ loss_sum,
                                                              T* __restrict__ dlogits) {
    __shared__ float sm[kCeThreads / 32], ss[kCeThreads / 32];
    const int row = blockIdx.x;
    const float* x = logits + static_cast<size_t>(row) * vocab;
    float m = -INFINITY, s = 0.f;
    for (int j = threadIdx.x; j < vocab; j += kCeThreads) {
        const float v = x[j];
        if (v > m) {
            s = s * ce_exp<T>(m - v) + 1.f;
            m = v;
        } else {
            s += ce_exp<T>(v - m);
        }
    }
    // combine (m, s) pairs: warp then block
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const float mm = fmaxf(m, m2);
        s = (mm == -INFINITY) ? 0.f : s * ce_exp<T>(m - mm) + s2 * ce_exp<T>(m2 - mm);
        m = mm;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sm[warp] = m;
        ss[warp] = s;
    }
    __syncthreads();
    float M = -INFINITY;
    for (int w = 0; w < kCeThreads / 32; ++w) M = fmaxf(M, sm[w]);
    float Ssum = 0.f;
    for (int w = 0; w < kCeThreads / 32; ++w) Ssum += ss[w] * ce_exp<T>(sm[w] - M);
    const float lse = M + logf(Ssum);
    const int tgt = targets[row];
    if (threadIdx.x == 0 && loss_sum) atomicAdd(loss_sum, lse - x[tgt]);
    if (dlogits) {
        T* d = dlogits + static_cast<size_t>(row) * vocab;
        for (int j = threadIdx.x; j < vocab; j += kCeThreads) {
            const float p = ce_exp<T>(x[j] - lse);
            d[j] = from_f<T>(grad_scale * (p - (j == tgt ? 1.f : 0.f)));
        }
    }
}

// vocab % 8 == 0 and 16-B aligned rows: float4 loads, 16-B stores of 8 bf16
// gradients (the scalar kernel above moved 2-B stores and ran at ~half of HBM
// bandwidth on the 50304-word head); same arithmetic per element.
__global__ void __launch_bounds__(kCeThreads) k_cross_entropy_v(const float4* __restrict__ logits,
                                                                const int32_t* __restrict__ targets, int vocab,
                                                                float grad_scale, float* __restrict__ loss_sum,
                                                                uint4* __restrict__ dlogits) {
    __shared__ float sm[kCeThreads / 32], ss[kCeThreads / 32];
    const int row = blockIdx.x;
    const int v4 = vocab >> 2;
    const float4* x = logits + static_cast<size_t>(row) * v4;
    float m = -INFINITY, s = 0.f;
    auto fold = [&](const float4 v) {
        const float mx = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
        const float mm = fmaxf(m, mx);
        s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + __expf(v.x - mm) + __expf(v.y - mm) + __expf(v.z - mm) +
            __expf(v.w - mm);
        m = mm;
    };
    int j = threadIdx.x;
    for (; j + 3 * kCeThreads < v4; j += 4 * kCeThreads) {  // four 16-B loads in flight per thread
        const float4 a = x[j], b = x[j + kCeThreads], c = x[j + 2 * kCeThreads], e = x[j + 3 * kCeThreads];
        fold(a);
        fold(b);
        fold(c);
        fold(e);
    }
    for (; j < v4; j += kCeThreads) fold(x[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const float mm = fmaxf(m, m2);
        s = (mm == -INFINITY) ? 0.f : s * __expf(m - mm) + s2 * __expf(m2 - mm);
        m = mm;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sm[warp] = m;
        ss[warp] = s;
    }
    __syncthreads();
    float M = -INFINITY;
    for (int w = 0; w < kCeThreads / 32; ++w) M = fmaxf(M, sm[w]);
    float Ssum = 0.f;
    for (int w = 0; w < kCeThreads / 32; ++w) Ssum += ss[w] * __expf(sm[w] - M);
    const float lse = M + logf(Ssum);
    const int tgt = targets[row];
    const float* xs = reinterpret_cast<const float*>(x);
    if (threadIdx.x == 0 && loss_sum) atomicAdd(loss_sum, lse - xs[tgt]);
    if (dlogits) {
        uint4* d = dlogits + static_cast<size_t>(row) * (vocab >> 3);
        for (int j = threadIdx.x; j < (vocab >> 3); j += kCeThreads) {
            const float4 a = x[2 * j], b = x[2 * j + 1];
            const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c0 = 8 * j + 2 * q;
                const float g0 = grad_scale * (__expf(v[2 * q] - lse) - (c0 == tgt ? 1.f : 0.f));
                const float g1 = grad_scale * (__expf(v[2 * q + 1] - lse) - (c0 + 1 == tgt ? 1.f : 0.f));
                const __nv_bfloat162 h = __floats2bfloat162_rn(g0, g1);
                w[q] = *reinterpret_cast<const uint32_t*>(&h);
            }
            d[j] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

// ------------------------------------------------------------------ AdamW --
__global__ void k_adamw(float* __restrict__ p32, __nv_bfloat16* __restrict__ p16, float* __restrict__ grad,
                        float* __restrict__ m, float* __restrict__ v, size_t n, float lr, float b1, float b2,
                        float eps, float wd, float bc1, float bc2, float gscale, int zero_grad) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float g = grad[i] * gscale;
        const float mi = b1 * m[i] + (1.f - b1) * g;
        const float vi = b2 * v[i] + (1.f - b2) * g * g;
        m[i] = mi;
        v[i] = vi;
        float p = p32[i];
        p -= lr * ((mi / bc1) / (sqrtf(vi / bc2) + eps) + wd * p);
        p32[i] = p;
        if (p16) p16[i] = __float2bfloat16_rn(p);
        if (zero_grad) grad[i] = 0.f;
    }
}

// 4 parameters per thread per iteration: 16-B loads of p32 / grad / m / v and an
// 8-B store of the bf16 shadow (the scalar kernel ran at ~65% of HBM bandwidth)
__global__ void k_adamw4(float4* __restrict__ p32, uint2* __restrict__ p16, float4* __restrict__ grad,
                         float4* __restrict__ m, float4* __restrict__ v, size_t n4, float lr, float b1, float b2,
                         float eps, float wd, float inv_bc1, float inv_sqrt_bc2, float gscale, int zero_grad) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float4 g4 = grad[i], m4 = m[i], v4 = v[i], p4 = p32[i];
        const float gs[4] = {g4.x, g4.y, g4.z, g4.w}, ms[4] = {m4.x, m4.y, m4.z, m4.w};
        const float vs[4] = {v4.x, v4.y, v4.z, v4.w}, ps[4] = {p4.x, p4.y, p4.z, p4.w};
        float mo[4], vo[4], po[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float g = gs[k] * gscale;
            mo[k] = b1 * ms[k] + (1.f - b1) * g;
            vo[k] = b2 * vs[k] + (1.f - b2) * g * g;
            po[k] = ps[k] - lr * ((mo[k] * inv_bc1) / (sqrtf(vo[k]) * inv_sqrt_bc2 + eps) + wd * ps[k]);
        }
        m[i] = make_float4(mo[0], mo[1], mo[2], mo[3]);
        v[i] = make_float4(vo[0], vo[1], vo[2], vo[3]);
        p32[i] = make_float4(po[0], po[1], po[2], po[3]);
        if (p16) {
            const __nv_bfloat162 a = __floats2bfloat162_rn(po[0], po[1]), b = __floats2bfloat162_rn(po[2], po[3]);
            p16[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
        }
        if (zero_grad) grad[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// ------------------------------------------------------------------- init --
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void k_fill_normal(float* __restrict__ p, size_t n, float mean, float stdv, uint64_t seed) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = splitmix64(seed * 0xD1B54A32D192ED03ull + i);
        const float u1 = (static_cast<float>(r >> 40) + 1.f) * (1.f / 16777217.f);  // (0,1]
        const float u2 = static_cast<float>((r >> 16) & 0xffffffull) * (1.f / 16777216.f);
        p[i] = mean + stdv * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
    }
}

__global__ void k_add4(float4* __restrict__ dst, const float4* __restrict__ src, size_t n4) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float4 a = dst[i], b = src[i];
        dst[i] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
}
__global__ void k_add(float* __restrict__ dst, const float* __restrict__ src, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        dst[i] += src[i];
}

__global__ void k_cast(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(in[i]);
}

}  // namespace
}  // namespace swarm

using namespace swarm;

extern "C" {

int swarm_embedding_forward_ex(const int32_t* tokens, size_t n, const void* table, size_t vocab, size_t d, void* out,
                               int dtype, swarm_stream_t stream) {
    if (dtype != SWARM_DTYPE_BF16 && dtype != SWARM_DTYPE_F32) return invalid("embedding: dtype must be f32 or bf16");
    const size_t row_bytes = d * (dtype == SWARM_DTYPE_F32 ? 4 : 2);
    if (row_bytes % 16) return invalid("embedding: rows must be a multiple of 16 bytes");
    if (n == 0) return SWARM_OK;
    k_embed_fwd<<<grid_for(n * 32, 256), 256, 0, as_stream(stream)>>>(
        tokens, static_cast<int>(n), static_cast<const uint4*>(table), static_cast<int>(vocab),
        static_cast<int>(row_bytes / 16), static_cast<uint4*>(out));
    SWARM_LAUNCH_CHECK("k_embed_fwd");
    return SWARM_OK;
}

int swarm_embedding_forward(const int32_t* tokens, size_t n, const void* table, size_t vocab, size_t d, void* out,
                            swarm_stream_t stream) {
    if (d % 8) return invalid("embedding: d must be a multiple of 8");
    return swarm_embedding_forward_ex(tokens, n, table, vocab, d, out, SWARM_DTYPE_BF16, stream);
}

int swarm_embedding_backward_ex(const int32_t* tokens, size_t n, const void* dout, size_t vocab, size_t d,
                                float* dtable, int dtype, swarm_stream_t stream) {
    if (n == 0) return SWARM_OK;
    const unsigned g = grid_for(n * 32, 256);
    if (dtype == SWARM_DTYPE_F32)
        k_embed_bwd<float><<<g, 256, 0, as_stream(stream)>>>(tokens, static_cast<int>(n),
                                                             static_cast<const float*>(dout), static_cast<int>(vocab),
                                                             static_cast<int>(d), dtable);
    else if (dtype == SWARM_DTYPE_BF16)
        k_embed_bwd<__nv_bfloat16><<<g, 256, 0, as_stream(stream)>>>(
            tokens, static_cast<int>(n), static_cast<const __nv_bfloat16*>(dout), static_cast<int>(vocab),
            static_cast<int>(d), dtable);
    else
        return invalid("embedding backward: dtype must be f32 or bf16");
    SWARM_LAUNCH_CHECK("k_embed_bwd");
    return SWARM_OK;
}

int swarm_embedding_backward(const int32_t* tokens, size_t n, const void* dout, size_t vocab, size_t d, float* dtable,
                             swarm_stream_t stream) {
    return swarm_embedding_backward_ex(tokens, n, dout, vocab, d, dtable, SWARM_DTYPE_BF16, stream);
}

int swarm_attn_softmax_forward_ex(const float* s, size_t rows, size_t L, int causal, void* p, int p_dtype,
                                  swarm_stream_t stream) {
    if (L == 0 || L > 32 * kMaxLPerLane) return invalid("attn softmax: L must be in [1, 1024]");
    if (rows == 0) return SWARM_OK;
    const unsigned g = grid_for(rows * 32, 256);
    if (p_dtype == SWARM_DTYPE_F32)
        k_softmax_fwd<float><<<g, 256, 0, as_stream(stream)>>>(s, static_cast<int>(rows), static_cast<int>(L), causal,
                                                               static_cast<float*>(p));
    else if (p_dtype == SWARM_DTYPE_BF16)
        k_softmax_fwd<__nv_bfloat16><<<g, 256, 0, as_stream(stream)>>>(s, static_cast<int>(rows), static_cast<int>(L),
                                                                       causal, static_cast<__nv_bfloat16*>(p));
    else
        return invalid("attn softmax: dtype must be f32 or bf16");
    SWARM_LAUNCH_CHECK("k_softmax_fwd");
    return SWARM_OK;
}

int swarm_attn_softmax_forward(const float* s, size_t rows, size_t L, int causal, void* p, swarm_stream_t stream) {
    return swarm_attn_softmax_forward_ex(s, rows, L, causal, p, SWARM_DTYPE_BF16, stream);
}

int swarm_attn_softmax_backward_ex(const void* p, const float* dp, size_t rows, size_t L, float scale, void* ds,
                                   int dtype, swarm_stream_t stream) {
    if (L == 0 || L > 32 * kMaxLPerLane) return invalid("attn softmax bwd: L must be in [1, 1024]");
    if (rows == 0) return SWARM_OK;
    const unsigned g = grid_for(rows * 32, 256);
    if (dtype == SWARM_DTYPE_F32)
        k_softmax_bwd<float><<<g, 256, 0, as_stream(stream)>>>(static_cast<const float*>(p), dp, static_cast<int>(rows),
                                                               static_cast<int>(L), scale, static_cast<float*>(ds));
    else if (dtype == SWARM_DTYPE_BF16)
        k_softmax_bwd<__nv_bfloat16><<<g, 256, 0, as_stream(stream)>>>(
            static_cast<const __nv_bfloat16*>(p), dp, static_cast<int>(rows), static_cast<int>(L), scale,
            static_cast<__nv_bfloat16*>(ds));
    else
        return invalid("attn softmax bwd: dtype must be f32 or bf16");
    SWARM_LAUNCH_CHECK("k_softmax_bwd");
    return SWARM_OK;
}

int swarm_attn_softmax_backward(const void* p, const float* dp, size_t rows, size_t L, float scale, void* ds,
                                swarm_stream_t stream) {
    return swarm_attn_softmax_backward_ex(p, dp, rows, L, scale, ds, SWARM_DTYPE_BF16, stream);
}

int swarm_cross_entropy_ex(const float* logits, const int32_t* targets, size_t rows, size_t vocab, float grad_scale,
                           float* loss_sum, void* dlogits, int dlogits_dtype, swarm_stream_t stream) {
    if (vocab == 0) return invalid("cross_entropy: empty vocab");
    if (rows == 0) return SWARM_OK;
    if (dlogits_dtype == SWARM_DTYPE_F32) {
        k_cross_entropy<float><<<static_cast<unsigned>(rows), kCeThreads, 0, as_stream(stream)>>>(
            logits, targets, static_cast<int>(vocab), grad_scale, loss_sum, static_cast<float*>(dlogits));
        SWARM_LAUNCH_CHECK("k_cross_entropy");
        return SWARM_OK;
    }
    if (dlogits_dtype != SWARM_DTYPE_BF16) return invalid("cross_entropy: dlogits dtype must be f32 or bf16");
    if (vocab % 8 == 0 && !(reinterpret_cast<uintptr_t>(logits) & 15) && !(reinterpret_cast<uintptr_t>(dlogits) & 15)) {
        // at most 2 rows per SM in flight (the unused dynamic smem only caps occupancy): 296 rows x
        // 200 KB stay L2-resident between the two passes over a row, 4 per SM would not
        static const int ce_smem = [] {
            const int b = 96 * 1024;
            cudaFuncSetAttribute(k_cross_entropy_v, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
            return b;
        }();
        k_cross_entropy_v<<<static_cast<unsigned>(rows), kCeThreads, ce_smem, as_stream(stream)>>>(
            reinterpret_cast<const float4*>(logits), targets, static_cast<int>(vocab), grad_scale, loss_sum,
            static_cast<uint4*>(dlogits));
        SWARM_LAUNCH_CHECK("k_cross_entropy_v");
        return SWARM_OK;
    }
    k_cross_entropy<__nv_bfloat16><<<static_cast<unsigned>(rows), kCeThreads, 0, as_stream(stream)>>>(
        logits, targets, static_cast<int>(vocab), grad_scale, loss_sum, static_cast<__nv_bfloat16*>(dlogits));
    SWARM_LAUNCH_CHECK("k_cross_entropy");
    return SWARM_OK;
}

int swarm_cross_entropy(const float* logits, const int32_t* targets, size_t rows, size_t vocab, float grad_scale,
                        float* loss_sum, void* dlogits, swarm_stream_t stream) {
    return swarm_cross_entropy_ex(logits, targets, rows, vocab, grad_scale, loss_sum, dlogits, SWARM_DTYPE_BF16,
                                  stream);
}

int swarm_adamw_step(float* p32, void* p16, float* grad, float* m, float* v, size_t n, float lr, float beta1,
                     float beta2, float eps, float weight_decay, int step, float grad_scale, int zero_grad,
                     swarm_stream_t stream) {
    if (step < 1) return invalid("adamw: step must be >= 1");
    if (n == 0) return SWARM_OK;
    const float bc1 = 1.f - std::pow(beta1, static_cast<float>(step));
    const float bc2 = 1.f - std::pow(beta2, static_cast<float>(step));
    const bool vec = n % 4 == 0 && !((reinterpret_cast<uintptr_t>(p32) | reinterpret_cast<uintptr_t>(grad) |
                                      reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) &&
                     !(reinterpret_cast<uintptr_t>(p16) & 7);
    if (vec) {
        // m / bc1 / (sqrt(v / bc2) + eps) == m * (1/bc1) / (sqrt(v) * (1/sqrt(bc2)) + eps)
        k_adamw4<<<grid_for(n / 4, 256, 148u * 16u), 256, 0, as_stream(stream)>>>(
            reinterpret_cast<float4*>(p32), static_cast<uint2*>(p16), reinterpret_cast<float4*>(grad),
            reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n / 4, lr, beta1, beta2, eps, weight_decay,
            1.f / bc1, 1.f / std::sqrt(bc2), grad_scale, zero_grad);
        SWARM_LAUNCH_CHECK("k_adamw4");
        return SWARM_OK;
    }
    k_adamw<<<grid_for(n, 256, 148u * 16u), 256, 0, as_stream(stream)>>>(
        p32, static_cast<__nv_bfloat16*>(p16), grad, m, v, n, lr, beta1, beta2, eps, weight_decay, bc1, bc2,
        grad_scale, zero_grad);
    SWARM_LAUNCH_CHECK("k_adamw");
    return SWARM_OK;
}

int swarm_fill_normal(float* p, size_t n, float mean, float stdv, uint64_t seed, swarm_stream_t stream) {
    if (n == 0) return SWARM_OK;
    k_fill_normal<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(p, n, mean, stdv, seed);
    SWARM_LAUNCH_CHECK("k_fill_normal");
    return SWARM_OK;
}

int swarm_add_f32(float* dst, const float* src, size_t n, swarm_stream_t stream) {
    if (n == 0) return SWARM_OK;
    if (n % 4 == 0 && !((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15)) {
        k_add4<<<grid_for(n / 4, 256, 148u * 16u), 256, 0, as_stream(stream)>>>(
            reinterpret_cast<float4*>(dst), reinterpret_cast<const float4*>(src), n / 4);
        SWARM_LAUNCH_CHECK("k_add4");
        return SWARM_OK;
    }
    k_add<<<grid_for(n, 256, 148u * 16u), 256, 0, as_stream(stream)>>>(dst, src, n);
    SWARM_LAUNCH_CHECK("k_add");
    return SWARM_OK;
}

int swarm_cast_f32_bf16(const float* in, void* out, size_t n, swarm_stream_t stream) {
    if (n == 0) return SWARM_OK;
    k_cast<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(in, static_cast<__nv_bfloat16*>(out), n);
    SWARM_LAUNCH_CHECK("k_cast");
    return SWARM_OK;
}

}  // extern "C"
