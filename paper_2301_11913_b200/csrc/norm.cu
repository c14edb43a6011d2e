// K3 maxout and K4 LayerNorm (sm_100a).
//
// maxout_k  — replaces compress::maxout_k (/root/reference/proj/src/compression.cpp:39-50);
//             adds the argmax the training backward needs (no reference).
// layer_norm — replaces compress::layer_norm (compression.cpp:52-74), row-wise over a
//             [rows, cols] activation: the row lives in registers, two-pass mean /
//             biased variance like the reference, fp32 statistics for f32/bf16 I/O
//             (fp64 for the f64 API path).  Backward is the standard LN gradient with
//             deterministic two-stage column reductions for dgain/dbias.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace swarm {
namespace {

template <typename T>
__device__ __forceinline__ float ld_f(const T* p);
template <>
__device__ __forceinline__ float ld_f<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T>
__device__ __forceinline__ T st_t(float v);
template <>
__device__ __forceinline__ float st_t<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 st_t<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// ---------------------------------------------------------------- maxout ----
template <typename T>
__device__ __forceinline__ bool less(T a, T b) {
    return a < b;
}
template <>
__device__ __forceinline__ bool less<__nv_bfloat16>(__nv_bfloat16 a, __nv_bfloat16 b) {
    return __bfloat162float(a) < __bfloat162float(b);
}

template <typename T>
__global__ void k_maxout_fwd(const T* __restrict__ x, size_t nout, int k, T* __restrict__ out,
                             uint8_t* __restrict__ argmax) {
    for (size_t j = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; j < nout;
         j += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const T* w = x + j * k;
        T m = w[0];
        int am = 0;
        for (int i = 1; i < k; ++i) {
            const T v = w[i];
            if (less(m, v)) {  // std::max(m, v) keeps m unless m < v
                m = v;
                am = i;
            }
        }
        out[j] = m;
        if (argmax) argmax[j] = static_cast<uint8_t>(am);
    }
}

template <typename T>
__global__ void k_maxout_bwd(const T* __restrict__ gout, const uint8_t* __restrict__ argmax, size_t nin, int k,
                             T* __restrict__ gin) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nin;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t j = i / k;
        const int r = static_cast<int>(i - j * k);
        gin[i] = (r == argmax[j]) ? gout[j] : T(0);
    }
}

unsigned grid_1d(size_t n, unsigned threads) {
    const size_t g = (n + threads - 1) / threads;
    return static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(g, 148u * 32u)));
}

// ------------------------------------------------------------- layernorm ----
constexpr int kLnThreads = 256;
constexpr int kLnMaxPerThread = 32;  // cols <= 8192

template <int THREADS>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // protect red from a previous use
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = 0.f;
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) r += red[w];
    return r;
}

// column owned by (thread, slot): col = slot*THREADS*VEC + threadIdx.x*VEC + v
template <typename T, int VEC>
__device__ __forceinline__ void load_row(const T* __restrict__ row, int cols, float (&v)[kLnMaxPerThread]) {
#pragma unroll
    for (int s = 0; s < kLnMaxPerThread / VEC; ++s) {
        const int c0 = s * kLnThreads * VEC + threadIdx.x * VEC;
        if (c0 < cols) {
            if constexpr (VEC == 8) {  // bf16 x8
                const uint4 q = *reinterpret_cast<const uint4*>(row + c0);
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    v[s * 8 + 2 * j] = __uint_as_float(w[j] << 16);
                    v[s * 8 + 2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
                }
            } else if constexpr (VEC == 4) {  // f32 x4
                const float4 q = *reinterpret_cast<const float4*>(row + c0);
                v[s * 4 + 0] = q.x;
                v[s * 4 + 1] = q.y;
                v[s * 4 + 2] = q.z;
                v[s * 4 + 3] = q.w;
            } else {
                v[s] = ld_f<T>(row + c0);
            }
        }
    }
}

template <typename T, int VEC>
__device__ __forceinline__ void store_row(T* __restrict__ row, int cols, const float (&v)[kLnMaxPerThread]) {
#pragma unroll
    for (int s = 0; s < kLnMaxPerThread / VEC; ++s) {
        const int c0 = s * kLnThreads * VEC + threadIdx.x * VEC;
        if (c0 < cols) {
            if constexpr (VEC == 8) {
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const __nv_bfloat162 p = __floats2bfloat162_rn(v[s * 8 + 2 * j], v[s * 8 + 2 * j + 1]);
                    w[j] = *reinterpret_cast<const uint32_t*>(&p);
                }
                *reinterpret_cast<uint4*>(row + c0) = make_uint4(w[0], w[1], w[2], w[3]);
            } else if constexpr (VEC == 4) {
                *reinterpret_cast<float4*>(row + c0) = make_float4(v[s * 4], v[s * 4 + 1], v[s * 4 + 2], v[s * 4 + 3]);
            } else {
                row[c0] = st_t<T>(v[s]);
            }
        }
    }
}

template <int VEC>
__device__ __forceinline__ int col_of(int s, int j) {
    return s * kLnThreads * VEC + threadIdx.x * VEC + j;
}

template <typename T, int VEC>
__global__ void __launch_bounds__(kLnThreads) k_ln_fwd(const T* __restrict__ x, int rows, int cols,
                                                       const float* __restrict__ gain, const float* __restrict__ bias,
                                                       float eps, T* __restrict__ out, float* __restrict__ mean_out,
                                                       float* __restrict__ rstd_out) {
    __shared__ float red[kLnThreads / 32];
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        float v[kLnMaxPerThread];
        load_row<T, VEC>(x + static_cast<size_t>(r) * cols, cols, v);
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < kLnMaxPerThread / VEC; ++q)
#pragma unroll
            for (int j = 0; j < VEC; ++j)
                if (col_of<VEC>(q, j) < cols) s += v[q * VEC + j];
        const float mean = block_sum<kLnThreads>(s, red) / static_cast<float>(cols);
        float s2 = 0.f;
#pragma unroll
        for (int q = 0; q < kLnMaxPerThread / VEC; ++q)
#pragma unroll
            for (int j = 0; j < VEC; ++j)
                if (col_of<VEC>(q, j) < cols) {
                    const float d = v[q * VEC + j] - mean;
                    s2 += d * d;
                }
        const float var = block_sum<kLnThreads>(s2, red) / static_cast<float>(cols);
        const float rstd = 1.0f / sqrtf(var + eps);
#pragma unroll
        for (int q = 0; q < kLnMaxPerThread / VEC; ++q)
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const int c = col_of<VEC>(q, j);
                if (c < cols) {
                    float o = (v[q * VEC + j] - mean) * rstd;
                    if (gain) o *= gain[c];
                    if (bias) o += bias[c];
                    v[q * VEC + j] = o;
                }
            }
        store_row<T, VEC>(out + static_cast<size_t>(r) * cols, cols, v);
        if (threadIdx.x == 0) {
            if (mean_out) mean_out[r] = mean;
            if (rstd_out) rstd_out[r] = rstd;
        }
    }
}

// rows handled per CTA in the backward: partial dgain/dbias rows = gridDim.x
template <typename T, int VEC>
__global__ void __launch_bounds__(kLnThreads) k_ln_bwd(const T* __restrict__ dy, const T* __restrict__ x, int rows,
                                                       int cols, const float* __restrict__ gain,
                                                       const float* __restrict__ mean, const float* __restrict__ rstd,
                                                       const T* __restrict__ dres, T* __restrict__ dx,
                                                       float* __restrict__ part_g,
                                                       float* __restrict__ part_b, int rows_per_cta) {
    __shared__ float red[kLnThreads / 32];
    float acc_g[kLnMaxPerThread], acc_b[kLnMaxPerThread];
#pragma unroll
    for (int i = 0; i < kLnMaxPerThread; ++i) acc_g[i] = acc_b[i] = 0.f;
    const int r0 = blockIdx.x * rows_per_cta;
    const int r1 = min(rows, r0 + rows_per_cta);
    for (int r = r0; r < r1; ++r) {
        float xv[kLnMaxPerThread], gv[kLnMaxPerThread];
        load_row<T, VEC>(x + static_cast<size_t>(r) * cols, cols, xv);
        load_row<T, VEC>(dy + static_cast<size_t>(r) * cols, cols, gv);
        const float mu = mean[r], rs = rstd[r];
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int q = 0; q < kLnMaxPerThread / VEC; ++q)
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                const int c = col_of<VEC>(q, j);
                const int i = q * VEC + j;
                if (c < cols) {
                    const float xh = (xv[i] - mu) * rs;
                    const float d = gv[i];
                    acc_g[i] += d * xh;
                    acc_b[i] += d;
                    const float gy = gain ? d * gain[c] : d;
                    xv[i] = xh;
                    gv[i] = gy;
                    s1 += gy * xh;
                    s2 += gy;
                }
            }
        const float c1 = block_sum<kLnThreads>(s1, red) / static_cast<float>(cols);
        const float c2 = block_sum<kLnThreads>(s2, red) / static_cast<float>(cols);
#pragma unroll
        for (int i = 0; i < kLnMaxPerThread; ++i) xv[i] = rs * (gv[i] - c2 - xv[i] * c1);
        if (dres) {
            load_row<T, VEC>(dres + static_cast<size_t>(r) * cols, cols, gv);
#pragma unroll
            for (int i = 0; i < kLnMaxPerThread; ++i) xv[i] += gv[i];
        }
        store_row<T, VEC>(dx + static_cast<size_t>(r) * cols, cols, xv);
    }
    float* pg = part_g + static_cast<size_t>(blockIdx.x) * cols;
    float* pb = part_b + static_cast<size_t>(blockIdx.x) * cols;
#pragma unroll
    for (int q = 0; q < kLnMaxPerThread / VEC; ++q)
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const int c = col_of<VEC>(q, j);
            if (c < cols) {
                pg[c] = acc_g[q * VEC + j];
                pb[c] = acc_b[q * VEC + j];
            }
        }
}

__global__ void k_col_reduce(const float* __restrict__ part, int nparts, int cols, float* __restrict__ out,
                             int accumulate) {
    pdl_trigger();
    pdl_wait();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    float s = 0.f;
    for (int p = 0; p < nparts; ++p) s += part[static_cast<size_t>(p) * cols + c];
    // accumulate with an atomic add: one add per element per call (same value as a plain
    // read-modify-write), but safe when two visits of a stage run concurrently (lanes)
    if (accumulate) atomicAdd(out + c, s);
    else out[c] = s;
}

// fp64 API path: one CTA per row, three passes over global, verbatim formula.
__global__ void k_ln_fwd_f64(const double* __restrict__ x, int rows, int cols, const double* __restrict__ gain,
                             const double* __restrict__ bias, double eps, double* __restrict__ out) {
    __shared__ double red[32];
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        const double* xr = x + static_cast<size_t>(r) * cols;
        double s = 0.0;
        for (int c = threadIdx.x; c < cols; c += blockDim.x) s += xr[c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
        __syncthreads();
        s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w];
        const double mean = s / static_cast<double>(cols);
        double v = 0.0;
        for (int c = threadIdx.x; c < cols; c += blockDim.x) v += (xr[c] - mean) * (xr[c] - mean);
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        v = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) v += red[w];
        const double var = v / static_cast<double>(cols);
        const double inv = 1.0 / sqrt(var + eps);
        for (int c = threadIdx.x; c < cols; c += blockDim.x) {
            double o = (xr[c] - mean) * inv;
            if (gain) o *= gain[c];
            if (bias) o += bias[c];
            out[static_cast<size_t>(r) * cols + c] = o;
        }
    }
}

__global__ void k_matvec_f64(const double* __restrict__ x, int rows, const double* __restrict__ w, int cols,
                             double* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    double s = 0.0;
    for (int i = 0; i < rows; ++i) s = __dadd_rn(s, __dmul_rn(x[i], w[static_cast<size_t>(i) * cols + j]));
    out[j] = s;
}

bool al(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// ---------------------------------------------- warp-per-row bf16 LayerNorm --
// Small CTAs (2 warps = 2 rows) so the single wave of rows spreads evenly over
// the SMs (8-warp CTAs left some SMs with twice the rows of others).
constexpr int kLnWarpThreads = 64;
constexpr int kLnRowsPerCta = kLnWarpThreads / 32;
// cols = 256*NV: each lane holds NV 16-byte vectors (8 bf16) of the row, so a
// row needs no block barrier and each warp keeps 2*NV loads in flight.  This is
// the training path (d_model 256..4096); the block-per-row kernels above remain
// for fp32 / odd widths.
__device__ __forceinline__ void unpack8(const uint4& q, float* v) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        v[2 * j] = __uint_as_float(w[j] << 16);
        v[2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
    }
}
__device__ __forceinline__ uint4 pack8(const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162 p = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        w[j] = *reinterpret_cast<const uint32_t*>(&p);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// 8 consecutive fp32 (16-B aligned) or `dflt` when p is null
__device__ __forceinline__ void load8f(const float* __restrict__ p, int c0, float dflt, float (&v)[8]) {
    if (!p) {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = dflt;
        return;
    }
    const float4 a = __ldg(reinterpret_cast<const float4*>(p + c0));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p + c0) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NV>
__global__ void __launch_bounds__(kLnWarpThreads) k_ln_fwd_w(const uint4* __restrict__ x, int rows, const float* __restrict__ g,
                                                  const float* __restrict__ b, float eps, uint4* __restrict__ out,
                                                  float* __restrict__ mean_out, float* __restrict__ rstd_out) {
    pdl_trigger();
    pdl_wait();
    constexpr int C8 = 32 * NV;
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const float inv_n = 1.f / (256.f * NV);
    if constexpr (NV > 8) {
        // wide rows (d = 4096): a float copy of the row would not fit the register
        // file; three passes re-read it (L1 hits after the first)
        for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
            const uint4* xr = x + static_cast<size_t>(r) * C8;
            float s = 0.f;
#pragma unroll 4
            for (int i = 0; i < NV; ++i) {
                float v[8];
                unpack8(xr[lane + 32 * i], v);
#pragma unroll
                for (int j = 0; j < 8; ++j) s += v[j];
            }
            const float mean = wsum(s) * inv_n;
            float s2 = 0.f;
#pragma unroll 4
            for (int i = 0; i < NV; ++i) {
                float v[8];
                unpack8(xr[lane + 32 * i], v);
#pragma unroll
                for (int j = 0; j < 8; ++j) s2 += (v[j] - mean) * (v[j] - mean);
            }
            const float rstd = 1.0f / sqrtf(wsum(s2) * inv_n + eps);
            uint4* orow = out + static_cast<size_t>(r) * C8;
#pragma unroll 4
            for (int i = 0; i < NV; ++i) {
                const int c0 = (lane + 32 * i) * 8;
                float v[8], o[8], gv[8], bv[8];
                unpack8(xr[lane + 32 * i], v);
                load8f(g, c0, 1.f, gv);
                load8f(b, c0, 0.f, bv);
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = (v[j] - mean) * rstd * gv[j] + bv[j];
                orow[lane + 32 * i] = pack8(o);
            }
            if (lane == 0) {
                if (mean_out) mean_out[r] = mean;
                if (rstd_out) rstd_out[r] = rstd;
            }
        }
        return;
    }
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
        const uint4* xr = x + static_cast<size_t>(r) * C8;
        float v[NV * 8];
#pragma unroll
        for (int i = 0; i < NV; ++i) unpack8(xr[lane + 32 * i], v + 8 * i);
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < NV * 8; ++i) s += v[i];
        const float mean = wsum(s) * inv_n;
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < NV * 8; ++i) s2 += (v[i] - mean) * (v[i] - mean);
        const float rstd = 1.0f / sqrtf(wsum(s2) * inv_n + eps);
        uint4* orow = out + static_cast<size_t>(r) * C8;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int c0 = (lane + 32 * i) * 8;
            float o[8];
            float gv[8], bv[8];
            load8f(g, c0, 1.f, gv);  // 2 x 16-B loads (scalar loads here were the kernel's bottleneck)
            load8f(b, c0, 0.f, bv);
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = (v[8 * i + j] - mean) * rstd * gv[j] + bv[j];
            orow[lane + 32 * i] = pack8(o);
        }
        if (lane == 0) {
            if (mean_out) mean_out[r] = mean;
            if (rstd_out) rstd_out[r] = rstd;
        }
    }
}

// dx = rstd * (g*dy - mean(g*dy) - xhat * mean(g*dy*xhat)) (+ dres)
template <int NV>
__global__ void __launch_bounds__(kLnWarpThreads) k_ln_bwd_dx_w(const uint4* __restrict__ dy, const uint4* __restrict__ x, int rows,
                                                     const float* __restrict__ g, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, const uint4* __restrict__ dres,
                                                     uint4* __restrict__ dx) {
    pdl_trigger();
    pdl_wait();
    constexpr int C8 = 32 * NV;
    constexpr bool KEEP = NV <= 8;  // keep the row in registers, else re-read it (L1/L2 hits)
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const float inv_n = 1.f / (256.f * NV);
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
        const size_t base = static_cast<size_t>(r) * C8;
        const float mu = mean[r], rs = rstd[r];
        float xh[KEEP ? NV * 8 : 8], gy[KEEP ? NV * 8 : 8];
        float s1 = 0.f, s2 = 0.f;
#pragma unroll(KEEP ? NV : 4)
        for (int i = 0; i < NV; ++i) {
            float xv[8], dv[8];
            unpack8(x[base + lane + 32 * i], xv);
            unpack8(dy[base + lane + 32 * i], dv);
            const int c0 = (lane + 32 * i) * 8;
            float gv[8];
            load8f(g, c0, 1.f, gv);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float h = (xv[j] - mu) * rs;
                const float q = dv[j] * gv[j];
                s1 += q * h;
                s2 += q;
                if constexpr (KEEP) {
                    xh[8 * i + j] = h;
                    gy[8 * i + j] = q;
                }
            }
        }
        const float c1 = wsum(s1) * inv_n, c2 = wsum(s2) * inv_n;
#pragma unroll(KEEP ? NV : 4)
        for (int i = 0; i < NV; ++i) {
            const int c0 = (lane + 32 * i) * 8;
            float o[8];
            if constexpr (KEEP) {
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = rs * (gy[8 * i + j] - c2 - xh[8 * i + j] * c1);
            } else {
                float xv[8], dv[8], gv[8];
                unpack8(x[base + lane + 32 * i], xv);
                unpack8(dy[base + lane + 32 * i], dv);
                load8f(g, c0, 1.f, gv);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float h = (xv[j] - mu) * rs;
                    o[j] = rs * (dv[j] * gv[j] - c2 - h * c1);
                }
            }
            if (dres) {
                float rv[8];
                unpack8(dres[base + lane + 32 * i], rv);
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] += rv[j];
            }
            dx[base + lane + 32 * i] = pack8(o);
        }
    }
}

// dgain/dbias partials: CTA (column strip of 64, row split) with 8 column
// vectors x 32 row lanes; deterministic (fixed reduction order).
// The last CTA of each 64-column strip to finish (a self-resetting arrival
// counter per strip) sums the strip's split partials in split order and writes
// / accumulates dgain, dbias: one launch, still deterministic.
__global__ void __launch_bounds__(256) k_ln_bwd_dgb(const uint4* __restrict__ dy, const uint4* __restrict__ x, int rows,
                                                    int cols, const float* __restrict__ mean,
                                                    const float* __restrict__ rstd, int rows_per_split,
                                                    float* __restrict__ part_g, float* __restrict__ part_b,
                                                    int* __restrict__ strip_count, float* __restrict__ dg,
                                                    float* __restrict__ db, int accumulate) {
    pdl_trigger();
    pdl_wait();
    __shared__ float sg[32][65], sb[32][65];
    const int cv = threadIdx.x & 7, rl = threadIdx.x >> 3;
    const int c8 = blockIdx.x * 8 + cv;  // column vector
    const int cols8 = cols / 8;
    const int r0 = blockIdx.y * rows_per_split, r1 = min(rows, r0 + rows_per_split);
    float ag[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, ab[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (c8 < cols8) {
#pragma unroll 4
        for (int r = r0 + rl; r < r1; r += 32) {
            float xv[8], dv[8];
            unpack8(x[static_cast<size_t>(r) * cols8 + c8], xv);
            unpack8(dy[static_cast<size_t>(r) * cols8 + c8], dv);
            const float mu = mean[r], rs = rstd[r];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                ag[j] += dv[j] * (xv[j] - mu) * rs;
                ab[j] += dv[j];
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        sg[rl][cv * 8 + j] = ag[j];
        sb[rl][cv * 8 + j] = ab[j];
    }
    __syncthreads();
    if (threadIdx.x < 128) {
        const int col = threadIdx.x & 63;
        const bool isg = threadIdx.x < 64;
        float acc = 0.f;
        for (int k = 0; k < 32; ++k) acc += isg ? sg[k][col] : sb[k][col];
        const int gcol = blockIdx.x * 64 + col;
        if (gcol < cols) (isg ? part_g : part_b)[static_cast<size_t>(blockIdx.y) * cols + gcol] = acc;
    }
    __threadfence();
    __syncthreads();
    __shared__ int is_last;
    if (threadIdx.x == 0) is_last = atomicAdd(&strip_count[blockIdx.x], 1) == static_cast<int>(gridDim.y) - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // 128 outputs (64 columns x {gain, bias}) x 2 halves of the splits; each half
    // keeps 4 loads in flight, the halves meet in smem in a fixed order
    {
        const int o = threadIdx.x & 127, hsel = threadIdx.x >> 7;
        const int col = o & 63;
        const bool isg = o < 64;
        const int gcol = blockIdx.x * 64 + col;
        const int ns = static_cast<int>(gridDim.y), k0 = hsel ? ns / 2 : 0, k1 = hsel ? ns : ns / 2;
        float acc = 0.f;
        if (gcol < cols) {
            const float* part = (isg ? part_g : part_b) + gcol;
            int k = k0;
            for (; k + 4 <= k1; k += 4) {
                const float a0 = __ldcg(part + static_cast<size_t>(k) * cols);
                const float a1 = __ldcg(part + static_cast<size_t>(k + 1) * cols);
                const float a2 = __ldcg(part + static_cast<size_t>(k + 2) * cols);
                const float a3 = __ldcg(part + static_cast<size_t>(k + 3) * cols);
                acc += ((a0 + a1) + (a2 + a3));
            }
            for (; k < k1; ++k) acc += __ldcg(part + static_cast<size_t>(k) * cols);
        }
        float* red = &sg[0][0];  // reuse the partial tile (32 x 65 floats) for the 2 x 128 half sums
        red[hsel * 128 + o] = acc;
        __syncthreads();
        if (hsel == 0 && gcol < cols) {
            float* out = isg ? dg : db;
            const float t = red[o] + red[128 + o];
            if (out) {
                if (accumulate) atomicAdd(out + gcol, t);  // see k_col_reduce
                else out[gcol] = t;
            }
        }
    }
    if (threadIdx.x == 0) strip_count[blockIdx.x] = 0;  // ready for the next launch
}

template <int NV>
void ln_fwd_w(const __nv_bfloat16* x, int rows, const float* g, const float* b, float eps, __nv_bfloat16* out,
              float* mean, float* rstd, cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>(std::min((rows + kLnRowsPerCta - 1) / kLnRowsPerCta, 148 * 32));
    launch_pdl(k_ln_fwd_w<NV>, dim3(grid), dim3(kLnWarpThreads), 0, st, reinterpret_cast<const uint4*>(x), rows, g, b, eps,
               reinterpret_cast<uint4*>(out), mean, rstd);
}

template <int NV>
void ln_bwd_dx_w(const __nv_bfloat16* dy, const __nv_bfloat16* x, int rows, const float* g, const float* mean,
                 const float* rstd, const __nv_bfloat16* dres, __nv_bfloat16* dx, cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>(std::min((rows + kLnRowsPerCta - 1) / kLnRowsPerCta, 148 * 32));
    launch_pdl(k_ln_bwd_dx_w<NV>, dim3(grid), dim3(kLnWarpThreads), 0, st, reinterpret_cast<const uint4*>(dy),
               reinterpret_cast<const uint4*>(x), rows, g, mean, rstd, reinterpret_cast<const uint4*>(dres),
               reinterpret_cast<uint4*>(dx));
}

bool warp_ln_ok(int cols) { return cols % 256 == 0 && cols <= 4096 && (cols / 256) <= 16; }

template <typename F>
bool dispatch_nv(int nv, F&& f) {
    switch (nv) {
        case 1: f(std::integral_constant<int, 1>{}); return true;
        case 2: f(std::integral_constant<int, 2>{}); return true;
        case 4: f(std::integral_constant<int, 4>{}); return true;
        case 8: f(std::integral_constant<int, 8>{}); return true;
        case 12: f(std::integral_constant<int, 12>{}); return true;
        case 16: f(std::integral_constant<int, 16>{}); return true;
        default: return false;
    }
}

template <typename T>
int ln_fwd_launch(const T* x, int rows, int cols, const float* g, const float* b, float eps, T* out, float* mean,
                  float* rstd, cudaStream_t st) {
    if constexpr (sizeof(T) == 2) {
        if (warp_ln_ok(cols) && al(x, 16) && al(out, 16) && (!g || al(g, 16)) && (!b || al(b, 16)) &&
            dispatch_nv(cols / 256, [&](auto nv) { ln_fwd_w<decltype(nv)::value>(x, rows, g, b, eps, out, mean, rstd, st); })) {
            SWARM_LAUNCH_CHECK("k_ln_fwd_w");
            return SWARM_OK;
        }
    }
    const unsigned grid = static_cast<unsigned>(std::min(rows, 148 * 8));
    constexpr int V = sizeof(T) == 2 ? 8 : 4;
    if (cols % V == 0 && al(x, 16) && al(out, 16))
        k_ln_fwd<T, V><<<grid, kLnThreads, 0, st>>>(x, rows, cols, g, b, eps, out, mean, rstd);
    else
        k_ln_fwd<T, 1><<<grid, kLnThreads, 0, st>>>(x, rows, cols, g, b, eps, out, mean, rstd);
    SWARM_LAUNCH_CHECK("k_ln_fwd");
    return SWARM_OK;
}

constexpr size_t kLnCounterBytes = 4096;
int ln_bwd_parts(size_t rows) { return static_cast<int>(std::min<size_t>(rows, 2 * 148)); }

template <typename T>
int ln_bwd_launch(const T* dy, const T* x, int rows, int cols, const float* g, const float* mean, const float* rstd,
                  const T* dres, T* dx, float* dg, float* db, int accumulate, float* ws, cudaStream_t st) {
    if constexpr (sizeof(T) == 2) {
        if (warp_ln_ok(cols) && al(x, 16) && al(dy, 16) && al(dx, 16) && (!dres || al(dres, 16)) && (!g || al(g, 16)) &&
            dispatch_nv(cols / 256, [&](auto nv) {
                if (dx) ln_bwd_dx_w<decltype(nv)::value>(dy, x, rows, g, mean, rstd, dres, dx, st);
            })) {
            if (dx) SWARM_LAUNCH_CHECK("k_ln_bwd_dx_w");
            if (dg || db) {
                // row splits of SWARM_LN_DGB_ROWS (128) rows: fatter CTAs than the 64-row split, whose
                // per-CTA reduction + arrival counter cost dominated (ncu 12.3 us for 16 MB of reads);
                // measured dx + dgain/dbias at 2048 x 2048: 13.6 (64) / 12.05 (128) / 12.9 (256) / 15.5 (512) us
                static const int rows_per = [] {
                    const char* e = getenv("SWARM_LN_DGB_ROWS");
                    return e ? std::max(32, atoi(e)) : 128;
                }();
                const int splits = std::max(1, std::min(ln_bwd_parts(rows), (rows + rows_per - 1) / rows_per));
                const int rps = (rows + splits - 1) / splits;
                int* strips = reinterpret_cast<int*>(ws);  // fixed counter area, see swarm_layer_norm_backward_workspace
                float* pg = ws + kLnCounterBytes / sizeof(float);
                float* pb = pg + static_cast<size_t>(splits) * cols;
                launch_pdl(k_ln_bwd_dgb, dim3((cols + 63) / 64, splits), dim3(256), 0, st,
                           reinterpret_cast<const uint4*>(dy), reinterpret_cast<const uint4*>(x), rows, cols, mean,
                           rstd, rps, pg, pb, strips, dg, db, accumulate);
                SWARM_LAUNCH_CHECK("k_ln_bwd_dgb");
            }
            return SWARM_OK;
        }
    }
    if (!dx) return invalid("layer_norm backward: dx may be omitted only for bf16 rows of width 256k <= 4096");
    const int parts = ln_bwd_parts(rows);
    const int rpc = (rows + parts - 1) / parts;
    const int grid = (rows + rpc - 1) / rpc;
    float* pg = ws + kLnCounterBytes / sizeof(float);
    float* pb = pg + static_cast<size_t>(parts) * cols;
    constexpr int V = sizeof(T) == 2 ? 8 : 4;
    if (cols % V == 0 && al(x, 16) && al(dy, 16) && al(dx, 16) && (!dres || al(dres, 16)))
        k_ln_bwd<T, V><<<grid, kLnThreads, 0, st>>>(dy, x, rows, cols, g, mean, rstd, dres, dx, pg, pb, rpc);
    else
        k_ln_bwd<T, 1><<<grid, kLnThreads, 0, st>>>(dy, x, rows, cols, g, mean, rstd, dres, dx, pg, pb, rpc);
    SWARM_LAUNCH_CHECK("k_ln_bwd");
    const unsigned cg = static_cast<unsigned>((cols + 255) / 256);
    if (dg) {
        k_col_reduce<<<cg, 256, 0, st>>>(pg, grid, cols, dg, accumulate);
        SWARM_LAUNCH_CHECK("k_col_reduce");
    }
    if (db) {
        k_col_reduce<<<cg, 256, 0, st>>>(pb, grid, cols, db, accumulate);
        SWARM_LAUNCH_CHECK("k_col_reduce");
    }
    return SWARM_OK;
}

}  // namespace
}  // namespace swarm

using namespace swarm;

extern "C" {

int swarm_maxout_forward(const void* x, int dtype, size_t n, size_t k, void* out, uint8_t* argmax,
                         swarm_stream_t stream) {
    if (k == 0 || n % k != 0) return invalid("maxout_k: k must divide the input length");
    if (k > 255) return invalid("maxout_k: k must be <= 255 on the device path");
    if (n == 0) return SWARM_OK;
    const size_t nout = n / k;
    cudaStream_t st = as_stream(stream);
    const unsigned g = grid_1d(nout, 256);
    switch (dtype) {
        case SWARM_DTYPE_F32:
            k_maxout_fwd<float><<<g, 256, 0, st>>>(static_cast<const float*>(x), nout, static_cast<int>(k),
                                                   static_cast<float*>(out), argmax);
            break;
        case SWARM_DTYPE_BF16:
            k_maxout_fwd<__nv_bfloat16><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), nout,
                                                           static_cast<int>(k), static_cast<__nv_bfloat16*>(out),
                                                           argmax);
            break;
        case SWARM_DTYPE_F64:
            k_maxout_fwd<double><<<g, 256, 0, st>>>(static_cast<const double*>(x), nout, static_cast<int>(k),
                                                    static_cast<double*>(out), argmax);
            break;
        default: set_error("maxout_k: unsupported dtype"); return SWARM_E_UNSUPPORTED;
    }
    SWARM_LAUNCH_CHECK("k_maxout_fwd");
    return SWARM_OK;
}

int swarm_maxout_backward(const void* grad_out, int dtype, const uint8_t* argmax, size_t n_out, size_t k,
                          void* grad_in, swarm_stream_t stream) {
    if (k == 0 || k > 255) return invalid("maxout backward: bad k");
    if (n_out == 0) return SWARM_OK;
    const size_t nin = n_out * k;
    cudaStream_t st = as_stream(stream);
    const unsigned g = grid_1d(nin, 256);
    switch (dtype) {
        case SWARM_DTYPE_F32:
            k_maxout_bwd<float><<<g, 256, 0, st>>>(static_cast<const float*>(grad_out), argmax, nin,
                                                   static_cast<int>(k), static_cast<float*>(grad_in));
            break;
        case SWARM_DTYPE_BF16:
            k_maxout_bwd<__nv_bfloat16><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(grad_out), argmax, nin,
                                                           static_cast<int>(k), static_cast<__nv_bfloat16*>(grad_in));
            break;
        case SWARM_DTYPE_F64:
            k_maxout_bwd<double><<<g, 256, 0, st>>>(static_cast<const double*>(grad_out), argmax, nin,
                                                    static_cast<int>(k), static_cast<double*>(grad_in));
            break;
        default: set_error("maxout backward: unsupported dtype"); return SWARM_E_UNSUPPORTED;
    }
    SWARM_LAUNCH_CHECK("k_maxout_bwd");
    return SWARM_OK;
}

int swarm_layer_norm_forward(const void* x, int dtype, size_t rows, size_t cols, const void* gain, const void* bias,
                             double eps, void* out, float* mean, float* rstd, swarm_stream_t stream) {
    if (cols == 0) return invalid("layer_norm: empty input");
    if (rows == 0) return SWARM_OK;
    cudaStream_t st = as_stream(stream);
    if (dtype == SWARM_DTYPE_F64) {
        k_ln_fwd_f64<<<static_cast<unsigned>(std::min<size_t>(rows, 148 * 8)), 256, 0, st>>>(
            static_cast<const double*>(x), static_cast<int>(rows), static_cast<int>(cols),
            static_cast<const double*>(gain), static_cast<const double*>(bias), eps, static_cast<double*>(out));
        SWARM_LAUNCH_CHECK("k_ln_fwd_f64");
        return SWARM_OK;
    }
    if (cols > static_cast<size_t>(kLnThreads * kLnMaxPerThread)) return invalid("layer_norm: cols > 8192 unsupported");
    const float* g = static_cast<const float*>(gain);
    const float* b = static_cast<const float*>(bias);
    if (dtype == SWARM_DTYPE_F32)
        return ln_fwd_launch<float>(static_cast<const float*>(x), static_cast<int>(rows), static_cast<int>(cols), g,
                                    b, static_cast<float>(eps), static_cast<float*>(out), mean, rstd, st);
    if (dtype == SWARM_DTYPE_BF16)
        return ln_fwd_launch<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(x), static_cast<int>(rows),
                                            static_cast<int>(cols), g, b, static_cast<float>(eps),
                                            static_cast<__nv_bfloat16*>(out), mean, rstd, st);
    set_error("layer_norm: unsupported dtype");
    return SWARM_E_UNSUPPORTED;
}

int swarm_matvec_f64(const double* x, size_t rows, const double* w, size_t cols, double* out, swarm_stream_t stream) {
    if (cols == 0) return SWARM_OK;
    k_matvec_f64<<<static_cast<unsigned>((cols + 127) / 128), 128, 0, as_stream(stream)>>>(
        x, static_cast<int>(rows), w, static_cast<int>(cols), out);
    SWARM_LAUNCH_CHECK("k_matvec_f64");
    return SWARM_OK;
}

size_t swarm_layer_norm_backward_workspace(size_t rows, size_t cols) {
    // a fixed area of arrival counters (one per 64-column strip, any width up to 64K
    // columns, so one workspace serves calls of different widths), then the split
    // partials of dgain and dbias
    return kLnCounterBytes + 2 * static_cast<size_t>(ln_bwd_parts(rows)) * cols * sizeof(float);
}

int swarm_layer_norm_backward(const void* dy, const void* x, int dtype, size_t rows, size_t cols, const float* gain,
                              const float* mean, const float* rstd, const void* dres, void* dx, float* dgain,
                              float* dbias, int accumulate, void* workspace, swarm_stream_t stream) {
    if (cols == 0 || cols > static_cast<size_t>(kLnThreads * kLnMaxPerThread))
        return invalid("layer_norm backward: bad cols");
    if (rows == 0) return SWARM_OK;
    cudaStream_t st = as_stream(stream);
    float* ws = static_cast<float*>(workspace);
    if (dtype == SWARM_DTYPE_F32)
        return ln_bwd_launch<float>(static_cast<const float*>(dy), static_cast<const float*>(x), static_cast<int>(rows),
                                    static_cast<int>(cols), gain, mean, rstd, static_cast<const float*>(dres),
                                    static_cast<float*>(dx), dgain, dbias, accumulate, ws, st);
    if (dtype == SWARM_DTYPE_BF16)
        return ln_bwd_launch<__nv_bfloat16>(
            static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), static_cast<int>(rows),
            static_cast<int>(cols), gain, mean, rstd, static_cast<const __nv_bfloat16*>(dres),
            static_cast<__nv_bfloat16*>(dx), dgain, dbias, accumulate, ws, st);
    set_error("layer_norm backward: unsupported dtype");
    return SWARM_E_UNSUPPORTED;
}

}  // extern "C"
