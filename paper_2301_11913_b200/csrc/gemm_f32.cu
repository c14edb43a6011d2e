// fp32 GEMM (SIMT FFMA, fp32 accumulate) behind swarm_gemm_f32: the stage
// executor's fp32 arithmetic mode (swarm_stage_config.fp32, BASELINE configs[0]
// "tiny ... fp32"), whose results are compared with the fp64 CPU oracle at
// 1e-5 relative.  tcgen05 has no fp32-input MMA kind with fp32 rounding of the
// products (kind::tf32 truncates operands to 10 mantissa bits), so this path runs
// on the FMA pipes: 64x64 CTA tiles, 16-deep K slices staged in shared memory,
// 4x4 accumulators per thread.  It carries the exact swarm_gemm_args semantics
// of the bf16 kernel (layouts, batch offsets, second K segment, epilogues), so
// the stage code issues the same calls in both modes.
#include <algorithm>

#include "common.cuh"

namespace swarm {
namespace {

constexpr int kTm = 64, kTn = 64, kTk = 16, kThreads = 256;

__device__ __forceinline__ float gelu32(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float dgelu32(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float t = tanhf(k0 * (x + k1 * x * x * x));
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

// one operand tile (rows of the output dimension x kTk) into smem as s[k][i]
__device__ __forceinline__ void load_tile(float (*s)[kTm + 4], const float* base, const float* base2, int ld, bool mn,
                                          long long roff, long long coff, int i0, int n_i, int k0, int K, int kseg) {
    for (int e = threadIdx.x; e < kTm * kTk; e += kThreads) {
        int ii, kk;
        if (mn) {  // stored K x I, I contiguous: consecutive threads walk I
            kk = e / kTm;
            ii = e % kTm;
        } else {   // stored I x K, K contiguous: consecutive threads walk K
            ii = e / kTk;
            kk = e % kTk;
        }
        const int i = i0 + ii, k = k0 + kk;
        float v = 0.f;
        if (i < n_i && k < K) {
            const float* p = base;
            int kl = k;
            if (base2 && k >= kseg) {
                p = base2;
                kl = k - kseg;
            }
            const long long r = mn ? kl + roff : i + roff;
            const long long c = mn ? i + coff : kl + coff;
            v = p[r * ld + c];
        }
        s[kk][ii] = v;
    }
}

__global__ void __launch_bounds__(kThreads) k_gemm_f32(const swarm_gemm_args g) {
    __shared__ float As[kTk][kTm + 4], Bs[kTk][kTn + 4];
    const int z = blockIdx.z, zb = z / g.bh, zh = z % g.bh;
    const long long ar = static_cast<long long>(g.ra0) * zb + static_cast<long long>(g.ra1) * zh;
    const long long ac = static_cast<long long>(g.ca0) * zb + static_cast<long long>(g.ca1) * zh;
    const long long br = static_cast<long long>(g.rb0) * zb + static_cast<long long>(g.rb1) * zh;
    const long long bc = static_cast<long long>(g.cb0) * zb + static_cast<long long>(g.cb1) * zh;
    const long long dr = static_cast<long long>(g.rd0) * zb + static_cast<long long>(g.rd1) * zh;
    const long long dc = static_cast<long long>(g.cd0) * zb + static_cast<long long>(g.cd1) * zh;
    const int m0 = blockIdx.y * kTm, n0 = blockIdx.x * kTn;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const bool two = g.a2 && g.b2;
    const int kseg = two ? g.k / 2 : g.k;
    const float* A = static_cast<const float*>(g.a);
    const float* B = static_cast<const float*>(g.b);
    const float* A2 = two ? static_cast<const float*>(g.a2) : nullptr;
    const float* B2 = two ? static_cast<const float*>(g.b2) : nullptr;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < g.k; k0 += kTk) {
        load_tile(As, A, A2, g.lda, g.a_mn_major, ar, ac, m0, g.m, k0, g.k, kseg);
        load_tile(Bs, B, B2, g.ldb, g.b_mn_major, br, bc, n0, g.n, k0, g.k, kseg);
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kTk; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* D = static_cast<float*>(g.d);
    float* U = const_cast<float*>(static_cast<const float*>(g.aux));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty + 16 * i;
        if (m >= g.m) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx + 16 * j;
            if (n >= g.n) continue;
            const long long o = (m + dr) * g.ldd + n + dc;
            const float v = g.alpha * acc[i][j];
            switch (g.epilogue) {
                case SWARM_EPI_ACCUM_F32: atomicAdd(D + o, v); break;  // lanes may accumulate concurrently
                case SWARM_EPI_RESIDUAL: D[o] = v + U[o]; break;
                case SWARM_EPI_GELU:
                    U[o] = v;
                    D[o] = gelu32(v);
                    break;
                case SWARM_EPI_DGELU: D[o] = v * dgelu32(U[o]); break;
                case SWARM_EPI_GELU_DERIV:
                    U[o] = dgelu32(v);
                    D[o] = gelu32(v);
                    break;
                case SWARM_EPI_MUL: D[o] = v * U[o]; break;
                default: D[o] = v; break;  // STORE_BF16 (an fp32 activation here) / STORE_F32
            }
        }
    }
}

}  // namespace
}  // namespace swarm

using namespace swarm;

extern "C" int swarm_gemm_f32(const swarm_gemm_args* a, swarm_stream_t stream) {
    if (!a) return invalid("gemm_f32: null args");
    if (a->m <= 0 || a->n <= 0 || a->k <= 0 || a->batch <= 0 || a->bh <= 0) return invalid("gemm_f32: bad shape");
    if (!a->a || !a->b || !a->d) return invalid("gemm_f32: null operand");
    if (a->epilogue < 0 || a->epilogue > SWARM_EPI_MUL) return invalid("gemm_f32: bad epilogue");
    if ((a->epilogue == SWARM_EPI_RESIDUAL || a->epilogue == SWARM_EPI_GELU || a->epilogue == SWARM_EPI_DGELU ||
         a->epilogue == SWARM_EPI_GELU_DERIV || a->epilogue == SWARM_EPI_MUL) &&
        !a->aux)
        return invalid("gemm_f32: epilogue needs aux");
    if ((a->a2 || a->b2) && (!a->a2 || !a->b2 || a->batch != 1 || a->k % 2))
        return invalid("gemm_f32: two K segments need a2 and b2, batch 1 and an even K");
    if (a->batch > 65535) return invalid("gemm_f32: batch too large");
    const dim3 grid(static_cast<unsigned>((a->n + kTn - 1) / kTn), static_cast<unsigned>((a->m + kTm - 1) / kTm),
                    static_cast<unsigned>(a->batch));
    k_gemm_f32<<<grid, kThreads, 0, as_stream(stream)>>>(*a);
    SWARM_LAUNCH_CHECK("k_gemm_f32");
    return SWARM_OK;
}
