// K1 / K2: blockwise int8 absmax codec for SWARM stage boundaries (sm_100a).
//
// Replaces swarmsim::compress::quantize_blockwise / dequantize_blockwise
// (/root/reference/proj/src/compression.cpp:10-37).  HBM-bound byte work:
// one CTA owns one quantization block, keeps it in registers (single pass
// over HBM), reduces |x| with an integer max over the IEEE bit patterns
// (warp REDUX + one smem hop; NaN/Inf surface as bit patterns >= 0x7f800000,
// so the same reduction is the non-finite check of compression.cpp:12-14),
// then writes packed codes with streaming stores.
//
// Bit-exactness vs the reference's fp64 `round(127.0*x/absmax)`: a fp32
// candidate from x*(127/a) is within 1.5e-5 of the exact quotient, so it is
// already correct unless its fractional part is within 1e-4 of one half; only
// then an exact fp64 boundary test 127|x| >= (m+0.5)a decides (both products
// are exact in fp64 for fp32/bf16 inputs).  Ties round away from zero like C
// round().  The fp64 API path repeats the reference's fp64 operations verbatim.
//
// Dequantize with fp32 scales to f32/bf16 (k_dequant_blocks / _words) is pure
// fp32 arithmetic proven equal to the reference's fp64 value rounded once (see
// DeqSplit); it replaced a per-block smem codebook whose random-bank
// lookups made the kernel MIO-bound (ncu: mio_throttle 14.5, 0.70 of HBM).
// The codebook kernel (k_dequant_table: table[c] = (OutT)(c*a/127.0) in fp64)
// remains for fp64 scales and non-power-of-two block sizes.
#include <algorithm>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace swarm {
namespace {

constexpr uint32_t kF32AbsMask = 0x7fffffffu;
constexpr uint32_t kF32Inf = 0x7f800000u;

// Slow, exact path (taken with probability ~2e-4): 127|x| vs (fl+0.5)*a,
// both products exact in fp64 for fp32/bf16 x and fp32 a.
__device__ __noinline__ int code_exact(float x, float a, float inv) {
    const float ax = fabsf(x);
    const float fl = floorf(__fmul_rn(ax, inv));
    const double t = __dmul_rn(127.0, static_cast<double>(ax));
    const double bnd = __dmul_rn(static_cast<double>(fl) + 0.5, static_cast<double>(a));
    int m = static_cast<int>(fl) + (t >= bnd ? 1 : 0);
    m = m > 127 ? 127 : m;
    return x < 0.f ? -m : m;
}

// Fast path without F2I/FRND (those issue on the narrow XU pipe and made this
// kernel issue-bound): y = x*(127/a) is within 1.5e-5 of the exact quotient;
// adding 1.5*2^23 rounds it to the nearest integer inside the mantissa, which
// equals round-half-away-from-zero unless y is within 1e-4 of a half-integer.
__device__ __forceinline__ int code_from_f32(float x, float a, float inv) {
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
    const float y = __fmul_rn(x, inv);
    const float t = __fadd_rn(y, kMagic);
    const float r = __fsub_rn(t, kMagic);
    const float d = __fsub_rn(y, r);
    if (fabsf(fabsf(d) - 0.5f) < 1e-4f) return code_exact(x, a, inv);
    const int m = __float_as_int(t) - 0x4B400000;
    return max(-127, min(127, m));
}

__device__ __forceinline__ uint32_t pack4(int c0, int c1, int c2, int c3) {
    return (static_cast<uint32_t>(c0) & 0xffu) | ((static_cast<uint32_t>(c1) & 0xffu) << 8) |
           ((static_cast<uint32_t>(c2) & 0xffu) << 16) | ((static_cast<uint32_t>(c3) & 0xffu) << 24);
}

template <int THREADS>
__device__ __forceinline__ uint32_t block_max_u32(uint32_t m, uint32_t* red) {
    m = __reduce_max_sync(0xffffffffu, m);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = m;
    __syncthreads();
    uint32_t r = red[0];
#pragma unroll
    for (int w = 1; w < THREADS / 32; ++w) r = max(r, red[w]);
    return r;
}

// ---- fp32 fast path: bs = THREADS * 4 * V, full blocks, 16B-aligned -------
template <int THREADS, int V>
__global__ void __launch_bounds__(THREADS) k_quant_f32(const float4* __restrict__ x,
                                                       uint32_t* __restrict__ codes,
                                                       float* __restrict__ scales,
                                                       uint32_t* __restrict__ flags) {
    constexpr int BS4 = THREADS * V;
    __shared__ uint32_t red[THREADS / 32];
    const size_t b = blockIdx.x;
    const float4* xb = x + b * BS4;
    float4 v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __ldcs(xb + threadIdx.x + i * THREADS);
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        m = max(m, __float_as_uint(v[i].x) & kF32AbsMask);
        m = max(m, __float_as_uint(v[i].y) & kF32AbsMask);
        m = max(m, __float_as_uint(v[i].z) & kF32AbsMask);
        m = max(m, __float_as_uint(v[i].w) & kF32AbsMask);
    }
    m = block_max_u32<THREADS>(m, red);
    const float a = __uint_as_float(m);
    if (m >= kF32Inf && threadIdx.x == 0 && flags) atomicOr(flags, SWARM_FLAG_NONFINITE);
    const float inv = m != 0 ? __fdiv_rn(127.f, a) : 0.f;
    uint32_t* cb = codes + b * BS4;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const uint32_t p = pack4(code_from_f32(v[i].x, a, inv), code_from_f32(v[i].y, a, inv),
                                 code_from_f32(v[i].z, a, inv), code_from_f32(v[i].w, a, inv));
        __stcs(cb + threadIdx.x + i * THREADS, p);
    }
    if (threadIdx.x == 0) scales[b] = a;
}

// ---- bf16 fast path: bs = THREADS * 8 * V ---------------------------------
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <int THREADS, int V>
__global__ void __launch_bounds__(THREADS) k_quant_bf16(const uint4* __restrict__ x,
                                                        uint2* __restrict__ codes,
                                                        float* __restrict__ scales,
                                                        uint32_t* __restrict__ flags) {
    constexpr int BS8 = THREADS * V;
    __shared__ uint32_t red[THREADS / 32];
    const size_t b = blockIdx.x;
    const uint4* xb = x + b * BS8;
    uint4 v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __ldcs(xb + threadIdx.x + i * THREADS);
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            m = max(m, (w[j] << 16) & kF32AbsMask);
            m = max(m, w[j] & 0x7fff0000u);
        }
    }
    m = block_max_u32<THREADS>(m, red);
    const float a = __uint_as_float(m);
    if (m >= kF32Inf && threadIdx.x == 0 && flags) atomicOr(flags, SWARM_FLAG_NONFINITE);
    const float inv = m != 0 ? __fdiv_rn(127.f, a) : 0.f;
    uint2* cb = codes + b * BS8;
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        uint2 p;
        p.x = pack4(code_from_f32(bf16lo(w[0]), a, inv), code_from_f32(bf16hi(w[0]), a, inv),
                    code_from_f32(bf16lo(w[1]), a, inv), code_from_f32(bf16hi(w[1]), a, inv));
        p.y = pack4(code_from_f32(bf16lo(w[2]), a, inv), code_from_f32(bf16hi(w[2]), a, inv),
                    code_from_f32(bf16lo(w[3]), a, inv), code_from_f32(bf16hi(w[3]), a, inv));
        __stcs(cb + threadIdx.x + i * THREADS, p);
    }
    if (threadIdx.x == 0) scales[b] = a;
}

// ---- generic path: any block size / alignment / dtype, and ragged tails ----
template <typename T>
struct Elem;
template <>
struct Elem<float> {
    static __device__ __forceinline__ uint64_t absbits(float v) { return __float_as_uint(v) & kF32AbsMask; }
    static __device__ __forceinline__ bool nonfinite(uint64_t m) { return m >= kF32Inf; }
};
template <>
struct Elem<__nv_bfloat16> {
    static __device__ __forceinline__ uint64_t absbits(__nv_bfloat16 v) {
        return (static_cast<uint32_t>(__bfloat16_as_ushort(v)) << 16) & kF32AbsMask;
    }
    static __device__ __forceinline__ bool nonfinite(uint64_t m) { return m >= kF32Inf; }
};
template <>
struct Elem<double> {
    static __device__ __forceinline__ uint64_t absbits(double v) {
        return static_cast<uint64_t>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
    }
    static __device__ __forceinline__ bool nonfinite(uint64_t m) { return m >= 0x7ff0000000000000ull; }
};

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T, typename ScaleT>
__global__ void k_quant_generic(const T* __restrict__ x, size_t n, size_t bs, size_t first_block,
                                int8_t* __restrict__ codes, ScaleT* __restrict__ scales,
                                uint32_t* __restrict__ flags) {
    __shared__ uint64_t red[32];
    const size_t b = first_block + blockIdx.x;
    const size_t begin = b * bs;
    const size_t end = min(n, begin + bs);
    uint64_t m = 0;
    for (size_t i = begin + threadIdx.x; i < end; i += blockDim.x) m = max(m, Elem<T>::absbits(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = m;
    __syncthreads();
    m = red[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = max(m, red[w]);
    if (Elem<T>::nonfinite(m) && threadIdx.x == 0 && flags) atomicOr(flags, SWARM_FLAG_NONFINITE);
    if constexpr (sizeof(T) == 8) {
        const double a = __longlong_as_double(static_cast<long long>(m));
        // verbatim reference arithmetic: round(127.0 * x / absmax), clamp (compression.cpp:24-25)
        for (size_t i = begin + threadIdx.x; i < end; i += blockDim.x) {
            double c = a > 0.0 ? round(__ddiv_rn(__dmul_rn(127.0, x[i]), a)) : 0.0;
            c = fmin(fmax(c, -127.0), 127.0);
            codes[i] = static_cast<int8_t>(static_cast<int>(c));
        }
        if (threadIdx.x == 0) scales[b] = static_cast<ScaleT>(a);
    } else {
        const float a = __uint_as_float(static_cast<uint32_t>(m));
        const float inv = m != 0 ? __fdiv_rn(127.f, a) : 0.f;
        for (size_t i = begin + threadIdx.x; i < end; i += blockDim.x)
            codes[i] = static_cast<int8_t>(code_from_f32(to_f(x[i]), a, inv));
        if (threadIdx.x == 0) scales[b] = static_cast<ScaleT>(a);
    }
}

// ---- dequantize ------------------------------------------------------------
__device__ __forceinline__ uint16_t f64_to_bf16_bits(double d) {
    // round-to-odd to fp32, then round-to-nearest-even to bf16 == single RN of d
    float f = __double2float_rz(d);
    if (static_cast<double>(f) != d) f = __uint_as_float(__float_as_uint(f) | 1u);
    uint32_t u = __float_as_uint(f);
    if ((u & kF32AbsMask) > kF32Inf) return 0x7fc0;
    u = u + 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

template <typename OutT>
__device__ __forceinline__ OutT from_f64(double d);
template <>
__device__ __forceinline__ float from_f64<float>(double d) { return __double2float_rn(d); }
template <>
__device__ __forceinline__ double from_f64<double>(double d) { return d; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double d) {
    return __ushort_as_bfloat16(f64_to_bf16_bits(d));
}

__device__ __forceinline__ double deq(int c, double a) {
    return __ddiv_rn(__dmul_rn(static_cast<double>(c), a), 127.0);  // compression.cpp:34
}

// one CTA per full block; bs % 16 == 0; codes 16B aligned; out 16B aligned
template <typename OutT, typename ScaleT, int THREADS>
__global__ void __launch_bounds__(THREADS) k_dequant_table(const uint4* __restrict__ codes,
                                                           const ScaleT* __restrict__ scales, size_t bs,
                                                           OutT* __restrict__ out) {
    __shared__ OutT table[256];
    const size_t b = blockIdx.x;
    const size_t n16 = bs / 16;
    const uint4* cb = codes + b * n16;
    OutT* ob = out + b * bs;
    // issue this thread's first code load before the codebook build so the
    // HBM latency overlaps the 256 fp64 divides
    const uint4 first = threadIdx.x < n16 ? __ldcs(cb + threadIdx.x) : make_uint4(0, 0, 0, 0);
    const double a = static_cast<double>(scales[b]);
    if (threadIdx.x < 256) table[threadIdx.x] = from_f64<OutT>(deq(static_cast<int>(threadIdx.x) - 128, a));
    __syncthreads();
    for (size_t j = threadIdx.x; j < n16; j += THREADS) {
        const uint4 c = j == threadIdx.x ? first : __ldcs(cb + j);
        const uint32_t w[4] = {c.x, c.y, c.z, c.w};
        OutT vals[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int code = static_cast<int8_t>((w[q] >> (8 * r)) & 0xffu);
                vals[q * 4 + r] = table[code + 128];
            }
        }
        uint4* dst = reinterpret_cast<uint4*>(ob + j * 16);
        constexpr int kVecs = 16 * sizeof(OutT) / 16;
#pragma unroll
        for (int q = 0; q < kVecs; ++q) __stcs(dst + q, reinterpret_cast<const uint4*>(vals)[q]);
    }
}

// Arithmetic dequantize for fp32 scales (no codebook, no smem): the exact
// value x = c*a/127 has, in units of the fp32 ulp of x, a fractional part that
// is a multiple of 1/127 (c*mant(a) is an integer and x < 2^24 ulps), so it
// lies >= 1/254 ulp from every fp32 rounding midpoint and the reference's
// fl32(fl64(x)) equals RN32(x).  Per block a/127 is split as A1 + A2 (A1 =
// a*(1/127), A2 = (a - 127*A1)*(1/127) from the exact fma remainder), so
// c*A1 + c*A2 misses x by ~2^-40 ulp and q = fma(c, A1, c*A2) -- one
// rounding -- is RN32(x).  Exhaustively checked over every code and every fp32
// mantissa in several binades (scripts/deq_exhaustive.c, 0 mismatches); the
// derivation is scale-invariant while nothing leaves the normal range, hence the
// a in [2^-64, 2^65) guard -- other scales take the fp64 path.  bf16 output:
// RN16(q) == RN16(x) unless q is itself a bf16 midpoint (low 16 bits 0x8000;
// ~1.8e-5 of (a, c) pairs), which takes the fp64 path.
struct DeqSplit {
    float a1, a2;
    bool fast;
    __device__ __forceinline__ explicit DeqSplit(float a) {
        constexpr float kInv127 = 1.0f / 127.0f;
        fast = a >= 5.421010862427522e-20f && a < 3.6893488147419103e19f;  // [2^-64, 2^65)
        a1 = __fmul_rn(a, kInv127);
        a2 = __fmul_rn(__fmaf_rn(-a1, 127.0f, a), kInv127);
    }
    // byte r of the biased word (codes ^ 0x80808080): 0x4B0000XX = 2^23 + (c + 128)
    __device__ __forceinline__ float operator()(uint32_t wb, int r) const {
        const float cf = __fsub_rn(__int_as_float(__byte_perm(wb, 0x4B000000u, 0x7540u | r)), 8388736.0f);
        return __fmaf_rn(cf, a1, __fmul_rn(cf, a2));
    }
};

template <typename OutT>
struct DeqWord;
template <>
struct DeqWord<float> {
    using V = float4;
    __device__ __forceinline__ static V run(uint32_t w, const DeqSplit& d, float a) {
        float v[4];
        if (d.fast) {
            const uint32_t wb = w ^ 0x80808080u;
#pragma unroll
            for (int r = 0; r < 4; ++r) v[r] = d(wb, r);
        } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
                v[r] = __double2float_rn(deq(static_cast<int8_t>((w >> (8 * r)) & 0xffu), static_cast<double>(a)));
        }
        return make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <>
struct DeqWord<__nv_bfloat16> {
    using V = uint2;
    __device__ __forceinline__ static V run(uint32_t w, const DeqSplit& d, float a) {
        uint32_t h[4];
        const uint32_t wb = w ^ 0x80808080u;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t u = __float_as_uint(d(wb, r));
            if (d.fast && (u & 0xffffu) != 0x8000u) h[r] = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
            else h[r] = f64_to_bf16_bits(deq(static_cast<int8_t>((w >> (8 * r)) & 0xffu), static_cast<double>(a)));
        }
        return make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
    }
};

// block sizes 1024 * WPT: one CTA per block; every thread loads its WPT code
// words (lane-contiguous, 512 B per warp load) before any math, splits the
// block's scale once, and stores 16-B (f32) / 8-B (bf16) vectors
template <typename OutT, int WPT>
__global__ void __launch_bounds__(256) k_dequant_blocks(const uint32_t* __restrict__ codes,
                                                        const float* __restrict__ scales, size_t nblocks,
                                                        typename DeqWord<OutT>::V* __restrict__ out) {
    using V = typename DeqWord<OutT>::V;
    constexpr int WPB = 256 * WPT;
    for (size_t b = blockIdx.x; b < nblocks; b += gridDim.x) {  // one pass per CTA unless grid.x is capped
        uint32_t w[WPT];
#pragma unroll
        for (int k = 0; k < WPT; ++k) w[k] = __ldcs(codes + b * WPB + threadIdx.x + k * 256);
        const float a = __ldg(scales + b);
        const DeqSplit d(a);
        V* ob = out + b * WPB + threadIdx.x;
#pragma unroll
        for (int k = 0; k < WPT; ++k) __stcs(ob + k * 256, DeqWord<OutT>::run(w[k], d, a));
    }
}

// any power-of-two block size: flat over 32-bit words, scale of word i = scales[i >> wshift]
template <typename OutT, int U>
__global__ void __launch_bounds__(256) k_dequant_words(const uint32_t* __restrict__ codes,
                                                       const float* __restrict__ scales, size_t nwords,
                                                       unsigned wshift, typename DeqWord<OutT>::V* __restrict__ out) {
    using V = typename DeqWord<OutT>::V;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < nwords; i += U * stride) {
        uint32_t w[U];
        float a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) w[u] = __ldcs(codes + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = __ldg(scales + ((i + u * stride) >> wshift));
#pragma unroll
        for (int u = 0; u < U; ++u) __stcs(out + i + u * stride, DeqWord<OutT>::run(w[u], DeqSplit(a[u]), a[u]));
    }
    for (; i < nwords; i += stride) {
        const float a = __ldg(scales + (i >> wshift));
        __stcs(out + i, DeqWord<OutT>::run(__ldcs(codes + i), DeqSplit(a), a));
    }
}

template <typename OutT, typename ScaleT>
__global__ void k_dequant_generic(const int8_t* __restrict__ codes, const ScaleT* __restrict__ scales,
                                  size_t n, size_t bs, size_t first, OutT* __restrict__ out) {
    for (size_t i = first + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = from_f64<OutT>(deq(codes[i], static_cast<double>(scales[i / bs])));
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

unsigned grid_for(size_t work, unsigned per_block, unsigned cap = 148u * 16u) {
    const size_t g = (work + per_block - 1) / per_block;
    return static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(g, cap)));
}

template <typename T, typename ScaleT>
int launch_generic_quant(const T* x, size_t n, size_t bs, size_t first_block, size_t nblocks, int8_t* codes,
                         ScaleT* scales, uint32_t* flags, cudaStream_t st) {
    if (nblocks == 0) return SWARM_OK;
    const unsigned threads = bs >= 1024 ? 256 : (bs >= 128 ? 128 : 32);
    size_t done = 0;
    while (done < nblocks) {  // grid.x limit
        const size_t g = std::min<size_t>(nblocks - done, 0x7fffffffu);
        k_quant_generic<T, ScaleT><<<static_cast<unsigned>(g), threads, 0, st>>>(x, n, bs, first_block + done,
                                                                                 codes, scales, flags);
        SWARM_LAUNCH_CHECK("k_quant_generic");
        done += g;
    }
    return SWARM_OK;
}

}  // namespace

int quantize_device(const void* x, int dtype, size_t n, size_t bs, int8_t* codes, void* scales, uint32_t* flags,
                    cudaStream_t st) {
    if (bs == 0) return invalid("quantize_blockwise: block_size must be positive");
    if (n == 0) return SWARM_OK;
    if (!x || !codes || !scales) return invalid("quantize_blockwise: null buffer");
    const size_t nfull = n / bs;
    const size_t nblocks = (n + bs - 1) / bs;
    size_t fast = 0;  // number of leading full blocks handled by a fast kernel
    if (dtype == SWARM_DTYPE_F32) {
        auto* xf = static_cast<const float*>(x);
        auto* sf = static_cast<float*>(scales);
        if (nfull > 0 && aligned(x, 16) && aligned(codes, 4) && (bs == 4096 || bs == 2048 || bs == 1024)) {
            const unsigned g = static_cast<unsigned>(nfull);
            auto* x4 = reinterpret_cast<const float4*>(x);
            auto* c4 = reinterpret_cast<uint32_t*>(codes);
            if (bs == 4096) k_quant_f32<256, 4><<<g, 256, 0, st>>>(x4, c4, sf, flags);
            else if (bs == 2048) k_quant_f32<256, 2><<<g, 256, 0, st>>>(x4, c4, sf, flags);
            else k_quant_f32<256, 1><<<g, 256, 0, st>>>(x4, c4, sf, flags);
            SWARM_LAUNCH_CHECK("k_quant_f32");
            fast = nfull;
        }
        return launch_generic_quant<float, float>(xf, n, bs, fast, nblocks - fast, codes, sf, flags, st);
    }
    if (dtype == SWARM_DTYPE_BF16) {
        auto* xb = static_cast<const __nv_bfloat16*>(x);
        auto* sf = static_cast<float*>(scales);
        if (nfull > 0 && aligned(x, 16) && aligned(codes, 8) && (bs == 4096 || bs == 2048)) {
            const unsigned g = static_cast<unsigned>(nfull);
            auto* x8 = reinterpret_cast<const uint4*>(x);
            auto* c8 = reinterpret_cast<uint2*>(codes);
            if (bs == 4096) k_quant_bf16<256, 2><<<g, 256, 0, st>>>(x8, c8, sf, flags);
            else k_quant_bf16<256, 1><<<g, 256, 0, st>>>(x8, c8, sf, flags);
            SWARM_LAUNCH_CHECK("k_quant_bf16");
            fast = nfull;
        }
        return launch_generic_quant<__nv_bfloat16, float>(xb, n, bs, fast, nblocks - fast, codes, sf, flags, st);
    }
    if (dtype == SWARM_DTYPE_F64)
        return launch_generic_quant<double, double>(static_cast<const double*>(x), n, bs, 0, nblocks, codes,
                                                    static_cast<double*>(scales), flags, st);
    set_error("quantize_blockwise: unsupported dtype");
    return SWARM_E_UNSUPPORTED;
}

namespace {
template <typename OutT, typename ScaleT>
int launch_dequant(const int8_t* codes, const ScaleT* scales, size_t n, size_t bs, OutT* out, cudaStream_t st) {
    const size_t nfull = n / bs;
    size_t first = 0;
    constexpr bool kArith = std::is_same<ScaleT, float>::value &&
                            (std::is_same<OutT, float>::value || std::is_same<OutT, __nv_bfloat16>::value);
    if constexpr (kArith) {
        using V = typename DeqWord<OutT>::V;
        if (nfull > 0 && bs >= 4 && (bs & (bs - 1)) == 0 && aligned(codes, 4) && aligned(out, sizeof(V))) {
            const auto* c32 = reinterpret_cast<const uint32_t*>(codes);
            auto* ov = reinterpret_cast<V*>(out);
            // one CTA per block: measured 6.68 TB/s vs 5.29 for persistent CTAs walking
            // blocks (1 GiB f32; the hardware CTA scheduler balances the write stream better)
            const unsigned g = grid_for(nfull, 1, 0x7fffffffu);
            if (bs == 4096) k_dequant_blocks<OutT, 4><<<g, 256, 0, st>>>(c32, scales, nfull, ov);
            else if (bs == 2048) k_dequant_blocks<OutT, 2><<<g, 256, 0, st>>>(c32, scales, nfull, ov);
            else if (bs == 8192) k_dequant_blocks<OutT, 8><<<g, 256, 0, st>>>(c32, scales, nfull, ov);
            else if (bs == 1024) k_dequant_blocks<OutT, 1><<<g, 256, 0, st>>>(c32, scales, nfull, ov);
            else {
                const size_t nwords = nfull * bs / 4;
                const unsigned wshift = static_cast<unsigned>(__builtin_ctzll(bs / 4));
                k_dequant_words<OutT, 4><<<grid_for(nwords, 256 * 4, 0x7fffffffu), 256, 0, st>>>(c32, scales, nwords,
                                                                                                 wshift, ov);
            }
            SWARM_LAUNCH_CHECK("k_dequant_blocks/words");
            first = nfull * bs;
        }
    }
    if (first == 0 && nfull > 0 && bs % 16 == 0 && bs >= 512 && aligned(codes, 16) && aligned(out, 16)) {
        k_dequant_table<OutT, ScaleT, 256><<<static_cast<unsigned>(nfull), 256, 0, st>>>(
            reinterpret_cast<const uint4*>(codes), scales, bs, out);
        SWARM_LAUNCH_CHECK("k_dequant_table");
        first = nfull * bs;
    }
    if (first < n) {
        k_dequant_generic<OutT, ScaleT><<<grid_for(n - first, 256), 256, 0, st>>>(codes, scales, n, bs, first, out);
        SWARM_LAUNCH_CHECK("k_dequant_generic");
    }
    return SWARM_OK;
}

template <typename ScaleT>
int dequant_out(const int8_t* codes, const ScaleT* scales, size_t n, size_t bs, void* out, int out_dtype,
                cudaStream_t st) {
    switch (out_dtype) {
        case SWARM_DTYPE_F32: return launch_dequant<float, ScaleT>(codes, scales, n, bs, static_cast<float*>(out), st);
        case SWARM_DTYPE_BF16:
            return launch_dequant<__nv_bfloat16, ScaleT>(codes, scales, n, bs, static_cast<__nv_bfloat16*>(out), st);
        case SWARM_DTYPE_F64: return launch_dequant<double, ScaleT>(codes, scales, n, bs, static_cast<double*>(out), st);
    }
    set_error("dequantize_blockwise: unsupported output dtype");
    return SWARM_E_UNSUPPORTED;
}
}  // namespace

int dequantize_device(const int8_t* codes, const void* scales, int scale_dtype, size_t n, size_t bs, void* out,
                      int out_dtype, cudaStream_t st) {
    if (bs == 0) return invalid("dequantize_blockwise: block_size must be positive");
    if (n == 0) return SWARM_OK;
    if (!codes || !scales || !out) return invalid("dequantize_blockwise: null buffer");
    if (scale_dtype == SWARM_DTYPE_F32)
        return dequant_out<float>(codes, static_cast<const float*>(scales), n, bs, out, out_dtype, st);
    if (scale_dtype == SWARM_DTYPE_F64)
        return dequant_out<double>(codes, static_cast<const double*>(scales), n, bs, out, out_dtype, st);
    set_error("dequantize_blockwise: unsupported scale dtype");
    return SWARM_E_UNSUPPORTED;
}

// ---- host end-to-end path ------------------------------------------------
// Per-host-thread workspace so the by-value API stays reentrant
// without a global lock: two streams ping-pong chunks so the
// H2D of chunk i+1 overlaps the kernel and D2H of chunk i.
namespace {
size_t dtype_size(int dt) { return dt == SWARM_DTYPE_BF16 ? 2 : (dt == SWARM_DTYPE_F64 ? 8 : 4); }

struct HostWorkspace {
    cudaStream_t stream[2] = {nullptr, nullptr};
    void* buf[2] = {nullptr, nullptr};
    size_t cap = 0;
    uint32_t* flags = nullptr;
    int device = -1;
    ~HostWorkspace() = default;  // process-lifetime; freed by the driver at exit
    int ensure(size_t bytes_per_slot) {
        int dev = 0;
        SWARM_CUDA_TRY(cudaGetDevice(&dev));
        if (device != dev) {  // first use on this device (or device switched)
            for (int i = 0; i < 2; ++i) SWARM_CUDA_TRY(cudaStreamCreateWithFlags(&stream[i], cudaStreamNonBlocking));
            SWARM_CUDA_TRY(cudaMalloc(&flags, 2 * sizeof(uint32_t)));
            cap = 0;
            buf[0] = buf[1] = nullptr;
            device = dev;
        }
        if (bytes_per_slot > cap) {
            for (int i = 0; i < 2; ++i) {
                if (buf[i]) SWARM_CUDA_TRY(cudaFree(buf[i]));
                SWARM_CUDA_TRY(cudaMalloc(&buf[i], bytes_per_slot));
            }
            cap = bytes_per_slot;
        }
        return SWARM_OK;
    }
};
thread_local HostWorkspace g_ws;

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
constexpr size_t kChunkTarget = 32u << 20;  // ~32 MiB of input per pipelined chunk
}  // namespace

int quantize_host(const void* x, int dtype, size_t n, size_t bs, int8_t* codes, void* scales) {
    if (bs == 0) return invalid("quantize_blockwise: block_size must be positive");
    if (n == 0) return SWARM_OK;
    const size_t es = dtype_size(dtype);
    const size_t ss = dtype == SWARM_DTYPE_F64 ? 8 : 4;
    // chunk = whole blocks, about kChunkTarget bytes of input
    size_t blocks_per_chunk = std::max<size_t>(1, kChunkTarget / std::max<size_t>(1, bs * es));
    const size_t nblocks = (n + bs - 1) / bs;
    blocks_per_chunk = std::min(blocks_per_chunk, nblocks);
    const size_t chunk = blocks_per_chunk * bs;
    const size_t in_b = round_up(std::min(chunk, n) * es, 256);
    const size_t code_b = round_up(std::min(chunk, n), 256);
    const size_t sc_b = round_up(blocks_per_chunk * ss, 256);
    if (int rc = g_ws.ensure(in_b + code_b + sc_b)) return rc;
    SWARM_CUDA_TRY(cudaMemsetAsync(g_ws.flags, 0, 2 * sizeof(uint32_t), g_ws.stream[0]));
    SWARM_CUDA_TRY(cudaStreamSynchronize(g_ws.stream[0]));
    size_t ci = 0;
    for (size_t off = 0; off < n; off += chunk, ++ci) {
        const int s = static_cast<int>(ci & 1);
        cudaStream_t st = g_ws.stream[s];
        const size_t len = std::min(chunk, n - off);
        const size_t nb = (len + bs - 1) / bs;
        char* base = static_cast<char*>(g_ws.buf[s]);
        void* dx = base;
        int8_t* dc = reinterpret_cast<int8_t*>(base + in_b);
        void* dsc = base + in_b + code_b;
        SWARM_CUDA_TRY(cudaMemcpyAsync(dx, static_cast<const char*>(x) + off * es, len * es,
                                       cudaMemcpyHostToDevice, st));
        if (int rc = quantize_device(dx, dtype, len, bs, dc, dsc, g_ws.flags + s, st)) return rc;
        SWARM_CUDA_TRY(cudaMemcpyAsync(codes + off, dc, len, cudaMemcpyDeviceToHost, st));
        SWARM_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(scales) + (off / bs) * ss, dsc, nb * ss,
                                       cudaMemcpyDeviceToHost, st));
    }
    uint32_t fl[2] = {0, 0};
    SWARM_CUDA_TRY(cudaStreamSynchronize(g_ws.stream[0]));
    SWARM_CUDA_TRY(cudaStreamSynchronize(g_ws.stream[1]));
    SWARM_CUDA_TRY(cudaMemcpy(fl, g_ws.flags, sizeof(fl), cudaMemcpyDeviceToHost));
    if ((fl[0] | fl[1]) & SWARM_FLAG_NONFINITE) {
        set_error("quantize_blockwise: non-finite input");
        return SWARM_E_NONFINITE;
    }
    return SWARM_OK;
}

int dequantize_host(const int8_t* codes, const void* scales, int scale_dtype, size_t n, size_t bs, void* out,
                    int out_dtype) {
    if (bs == 0) return invalid("dequantize_blockwise: block_size must be positive");
    if (n == 0) return SWARM_OK;
    const size_t os = dtype_size(out_dtype);
    const size_t ss = scale_dtype == SWARM_DTYPE_F64 ? 8 : 4;
    size_t blocks_per_chunk = std::max<size_t>(1, kChunkTarget / std::max<size_t>(1, bs * os));
    const size_t nblocks = (n + bs - 1) / bs;
    blocks_per_chunk = std::min(blocks_per_chunk, nblocks);
    const size_t chunk = blocks_per_chunk * bs;
    const size_t out_b = round_up(std::min(chunk, n) * os, 256);
    const size_t code_b = round_up(std::min(chunk, n), 256);
    const size_t sc_b = round_up(blocks_per_chunk * ss, 256);
    if (int rc = g_ws.ensure(out_b + code_b + sc_b)) return rc;
    size_t ci = 0;
    for (size_t off = 0; off < n; off += chunk, ++ci) {
        const int s = static_cast<int>(ci & 1);
        cudaStream_t st = g_ws.stream[s];
        const size_t len = std::min(chunk, n - off);
        const size_t nb = (len + bs - 1) / bs;
        char* base = static_cast<char*>(g_ws.buf[s]);
        void* dout = base;
        int8_t* dc = reinterpret_cast<int8_t*>(base + out_b);
        void* dsc = base + out_b + code_b;
        SWARM_CUDA_TRY(cudaMemcpyAsync(dc, codes + off, len, cudaMemcpyHostToDevice, st));
        SWARM_CUDA_TRY(cudaMemcpyAsync(dsc, static_cast<const char*>(scales) + (off / bs) * ss, nb * ss,
                                       cudaMemcpyHostToDevice, st));
        if (int rc = dequantize_device(dc, dsc, scale_dtype, len, bs, dout, out_dtype, st)) return rc;
        SWARM_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(out) + off * os, dout, len * os, cudaMemcpyDeviceToHost, st));
    }
    SWARM_CUDA_TRY(cudaStreamSynchronize(g_ws.stream[0]));
    SWARM_CUDA_TRY(cudaStreamSynchronize(g_ws.stream[1]));
    return SWARM_OK;
}

}  // namespace swarm

extern "C" {

int swarm_quantize_blockwise(const void* x, int dtype, size_t n, size_t block_size, int8_t* codes, void* scales,
                             uint32_t* flags, swarm_stream_t stream) {
    return swarm::quantize_device(x, dtype, n, block_size, codes, scales, flags, swarm::as_stream(stream));
}

int swarm_dequantize_blockwise(const int8_t* codes, const void* scales, int scale_dtype, size_t n, size_t block_size,
                               void* out, int out_dtype, swarm_stream_t stream) {
    return swarm::dequantize_device(codes, scales, scale_dtype, n, block_size, out, out_dtype,
                                    swarm::as_stream(stream));
}

int swarm_quantize_blockwise_host(const void* x, int dtype, size_t n, size_t block_size, int8_t* codes,
                                  void* scales) {
    return swarm::quantize_host(x, dtype, n, block_size, codes, scales);
}

int swarm_dequantize_blockwise_host(const int8_t* codes, const void* scales, int scale_dtype, size_t n,
                                    size_t block_size, void* out, int out_dtype) {
    return swarm::dequantize_host(codes, scales, scale_dtype, n, block_size, out, out_dtype);
}

}  // extern "C"
