// K5: persistent, warp-specialised tcgen05 bf16 GEMM for sm_100a.
//
// Every dense contraction of the transformer block (QKV, O, FFN1, FFN2 and
// their dgrad/wgrad; attention S = QK^T, O = PV and their backward) goes
// through this kernel.  The reference only counts these FLOPs
// (/root/reference/proj/src/cost_model.cpp:31-42); it never executes them.
//
// Structure (one CTA per SM, 256 threads):
//   warp 0  TMA producer: 128x64 A tile + BNx64 B tile per stage, SWIZZLE_128B,
//           STAGES-deep smem ring guarded by full/empty mbarriers;
//   warp 1  MMA issuer: one elected thread issues tcgen05.mma (M=128, N=BN, K=16)
//           into a double-buffered fp32 accumulator in TMEM (2 x BN columns),
//           tcgen05.commit frees smem slots and signals the epilogue;
//   warp 2  TMEM allocator;
//   warps 4-7 epilogue: tcgen05.ld (32 lanes x 32 columns) -> fused op (scale,
//           residual add, GeLU / GeLU', fp32 accumulate) -> global stores, then
//           release the TMEM buffer so the next tile's MMAs overlap this drain.
// Operands may be K-major or MN-major (transposed) on either side, so dgrad and
// wgrad read activations/weights in place with no transpose pass.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "sm100.cuh"

namespace swarm {
namespace gemm {

using namespace swarm::sm100;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;
constexpr int kEpiSlot = 4096;                   // one 32x32 fp32 (or 2 x 32x32 bf16) chunk
constexpr int kEpiSmem = 4 * 2 * kEpiSlot;       // 4 epilogue warps x double buffer

struct Params {
    int m, n, k, bh;
    int tiles_m, tiles_n, tiles_per_batch, total_tiles, k_blocks;
    int ra0, ra1, ca0, ca1, rb0, rb1, cb0, cb1;
    void* d;
    long long ldd;
    int rd0, rd1, cd0, cd1;
    const void* aux;
    float alpha;
    int epi;
    int vec_ok;
    int tma_epi;  // stage output chunks in smem and write them with TMA (store / reduce-add)
    // stream-K (pair kernel): tiles [0, dp_tiles) are whole-tile units dealt
    // round-robin to the clusters; the sk_tiles after them are cut into
    // sk_tiles * k_blocks k-block iterations split evenly over the clusters
    int dp_tiles, sk_tiles, sk_iters;
    float* ws;      // per-cluster partial accumulators: [cluster][first|last][half][128][256] fp32
    int* sk_cnt;    // [sk_tile][half][warp] arrival counters (self-resetting)
    int* sk_ready;  // [cluster][first|last][half][warp] partial-ready flags (self-resetting)
    int k_tri;    // swarm_gemm_args.k_tri (1-CTA kernel): skip all-zero k-blocks of a triangular A
    int kb_half;  // two-segment K (pair kernel): k-blocks >= kb_half come from tma_a2 / tma_b2 (0 = one segment)
    int aux_prefetch;  // epilogue: request R / U before the TMEM drain (SWARM_GEMM_AUX_PREFETCH=0: after)
    int dbg;      // SWARM_GEMM_DBG (experiments only): 1 skip output stores, 2 skip MMAs, 4 skip TMA loads,
                  // 8 stream-K units store directly (no fixup), 16 fixup without waiting for partials
};

// MINB = 2: a short-K variant with two CTAs per SM (2 stages), for many small tiles (the batched
// attention GEMMs: 256 tiles of 128 x 128 x <= 512): one CTA's prologue / epilogue overlaps the
// other's MMAs instead of each tile paying its pipeline fill alone
template <int BN, int MINB = 1>
struct Cfg {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGES = MINB == 2 ? 2 : (BN == 256 ? 4 : 6);
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + kEpiSmem + 1024 + 256;
    static_assert(SMEM <= 232448, "GEMM exceeds the 227 KB dynamic smem limit");
    static_assert(2 * STAGES * 8 + 4 * 8 + 4 <= 256, "barrier area overflow");
};

// tanh on the SFU (MUFU.TANH, max relative error ~2^-11): the GeLU epilogues round to bf16
// (2^-8), so the accurate tanhf -- ~20 FMA-pipe instructions per element -- only cost issue
// slots (the live per-shape table showed the DGELU GEMM at 689 TFLOP/s against ~1100 for the
// same shape with a plain epilogue).  The fp32 mode's GEMM (gemm_f32.cu) keeps tanhf.
__device__ __forceinline__ float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float gelu_f(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float hx = 0.5f * x;
    return fmaf(hx, tanh_approx(k0 * fmaf(k1 * x, x * x, x)), hx);
}
// gelu(x) and gelu'(x) from one tanh (SWARM_EPI_GELU_DERIV)
__device__ __forceinline__ void gelu_both(float x, float& g, float& dg) {
    // gelu'(x) = 0.5 (1 + t) + 0.5 x (1 - t^2) k0 (1 + 3 k1 x^2), t = tanh(k0 (x + k1 x^3)); the
    // x^2 of the tanh argument reused, k0 folded into the polynomial (7 FMA-pipe ops after the tanh)
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float xx = x * x;
    const float t = tanh_approx(k0 * fmaf(k1 * x, xx, x));
    const float hx = 0.5f * x;
    g = fmaf(hx, t, hx);
    dg = fmaf(hx * fmaf(-t, t, 1.f), fmaf(3.f * k0 * k1, xx, k0), fmaf(0.5f, t, 0.5f));
}
__device__ __forceinline__ float dgelu_f(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float t = tanh_approx(k0 * fmaf(k1 * x, x * x, x));
    return fmaf(0.5f, 1.f + t, 0.5f * x * fmaf(-t, t, 1.f) * k0 * fmaf(3.f * k1, x * x, 1.f));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&p);
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// Apply the fused epilogue to 32 consecutive columns [col0, col0+32) of one row.
__device__ __forceinline__ void epilogue_chunk(const Params& p, float (&v)[32], long long off, int ncols_valid) {
    const bool full = p.vec_ok && ncols_valid >= 32;
    switch (p.epi) {
        case SWARM_EPI_STORE_BF16:
        case SWARM_EPI_RESIDUAL: {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.d) + off;
            if (p.epi == SWARM_EPI_RESIDUAL) {
                const __nv_bfloat16* r = static_cast<const __nv_bfloat16*>(p.aux) + off;
                if (full) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 w = reinterpret_cast<const uint4*>(r)[q];
                        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            v[q * 8 + 2 * j] += bf_lo(ws[j]);
                            v[q * 8 + 2 * j + 1] += bf_hi(ws[j]);
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < ncols_valid) v[j] += __bfloat162float(r[j]);
                }
            }
            if (full) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    reinterpret_cast<uint4*>(dst)[q] =
                        make_uint4(pack_bf16(v[q * 8 + 0], v[q * 8 + 1]), pack_bf16(v[q * 8 + 2], v[q * 8 + 3]),
                                   pack_bf16(v[q * 8 + 4], v[q * 8 + 5]), pack_bf16(v[q * 8 + 6], v[q * 8 + 7]));
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < ncols_valid) dst[j] = __float2bfloat16_rn(v[j]);
            }
            break;
        }
        case SWARM_EPI_STORE_F32:
        case SWARM_EPI_ACCUM_F32: {
            float* dst = static_cast<float*>(p.d) + off;
            if (full) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    // accumulation is a vector atomic (red.global.add.v4.f32): two lanes of a stage
                    // may accumulate into one gradient concurrently (swarm_stage_enable_lanes)
                    if (p.epi == SWARM_EPI_ACCUM_F32) atomicAdd(reinterpret_cast<float4*>(dst) + q, o);
                    else reinterpret_cast<float4*>(dst)[q] = o;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < ncols_valid) {
                        if (p.epi == SWARM_EPI_ACCUM_F32) atomicAdd(dst + j, v[j]);
                        else dst[j] = v[j];
                    }
            }
            break;
        }
        case SWARM_EPI_GELU: {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.d) + off;
            __nv_bfloat16* u = const_cast<__nv_bfloat16*>(static_cast<const __nv_bfloat16*>(p.aux)) + off;
            if (full) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    reinterpret_cast<uint4*>(u)[q] =
                        make_uint4(pack_bf16(v[q * 8 + 0], v[q * 8 + 1]), pack_bf16(v[q * 8 + 2], v[q * 8 + 3]),
                                   pack_bf16(v[q * 8 + 4], v[q * 8 + 5]), pack_bf16(v[q * 8 + 6], v[q * 8 + 7]));
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    reinterpret_cast<uint4*>(dst)[q] =
                        make_uint4(pack_bf16(v[q * 8 + 0], v[q * 8 + 1]), pack_bf16(v[q * 8 + 2], v[q * 8 + 3]),
                                   pack_bf16(v[q * 8 + 4], v[q * 8 + 5]), pack_bf16(v[q * 8 + 6], v[q * 8 + 7]));
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (j >= ncols_valid) continue;
                    u[j] = __float2bfloat16_rn(v[j]);
                    dst[j] = __float2bfloat16_rn(gelu_f(v[j]));
                }
            }
            break;
        }
        case SWARM_EPI_DGELU: {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.d) + off;
            const __nv_bfloat16* u = static_cast<const __nv_bfloat16*>(p.aux) + off;
            if (full) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint4 w = reinterpret_cast<const uint4*>(u)[q];
                    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        v[q * 8 + 2 * j] *= dgelu_f(bf_lo(ws[j]));
                        v[q * 8 + 2 * j + 1] *= dgelu_f(bf_hi(ws[j]));
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    reinterpret_cast<uint4*>(dst)[q] =
                        make_uint4(pack_bf16(v[q * 8 + 0], v[q * 8 + 1]), pack_bf16(v[q * 8 + 2], v[q * 8 + 3]),
                                   pack_bf16(v[q * 8 + 4], v[q * 8 + 5]), pack_bf16(v[q * 8 + 6], v[q * 8 + 7]));
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < ncols_valid) dst[j] = __float2bfloat16_rn(v[j] * dgelu_f(__bfloat162float(u[j])));
            }
            break;
        }
        case SWARM_EPI_GELU_DERIV:
        case SWARM_EPI_MUL: {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.d) + off;
            __nv_bfloat16* u = const_cast<__nv_bfloat16*>(static_cast<const __nv_bfloat16*>(p.aux)) + off;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j >= ncols_valid) continue;
                if (p.epi == SWARM_EPI_MUL) {
                    dst[j] = __float2bfloat16_rn(v[j] * __bfloat162float(u[j]));
                } else {
                    float g, dg;
                    gelu_both(v[j], g, dg);
                    u[j] = __float2bfloat16_rn(dg);
                    dst[j] = __float2bfloat16_rn(g);
                }
            }
            break;
        }
        default: break;
    }
}


// Swizzled staging of one 32 x 32 chunk (this warp's 32 rows; thread = row):
// fp32 rows are 128 B (TMA SWIZZLE_128B: 16-B chunk j at j ^ (row & 7)), bf16
// rows 64 B (SWIZZLE_64B: j ^ ((row >> 1) & 3)); both bank-conflict free.
__device__ __forceinline__ void stage_f32(uint8_t* slot, int row, const float (&v)[32]) {
    const uint32_t base = smem_u32(slot) + row * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        st_shared_v4(base + ((j ^ (row & 7)) << 4), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                     __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
}
__device__ __forceinline__ void stage_bf16(uint8_t* slot, int row, const float (&v)[32]) {
    const uint32_t base = smem_u32(slot) + row * 64;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        st_shared_v4(base + ((j ^ ((row >> 1) & 3)) << 4), pack_bf16(v[8 * j], v[8 * j + 1]),
                     pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                     pack_bf16(v[8 * j + 6], v[8 * j + 7]));
}

// Drain this warp's 32 rows x BN_TILE columns of one accumulator tile.
// Stream-K fixup: `fix_slots` packs (8 bits each) the workspace slots holding
// the other clusters' partial sums of this tile; `fix_row` is this warp's
// 32-row block inside a slot.  A block is stored as [chunk c][float4 j][lane]
// so that each warp access is 512 contiguous bytes (row-per-thread addressing
// would scatter every store over 32 rows).
__device__ __forceinline__ const float4* sk_part(const Params& p, uint64_t slots, int f, size_t row_off) {
    const int sl = static_cast<int>((slots >> (8 * f)) & 0xff);
    return reinterpret_cast<const float4*>(p.ws + static_cast<size_t>(sl) * 2 * 128 * 256 + row_off);
}
template <int BN_TILE>
__device__ __forceinline__ void drain_tile(const Params& p, const CUtensorMap* md, const CUtensorMap* mu,
                                           uint8_t* stg, int& slot_idx, uint32_t taddr, int row_base, long long rd,
                                           long long cd, int col_tile0, int lane, uint64_t fix_slots = 0,
                                           int nfix = 0, size_t fix_row = 0, int c_begin = 0,
                                           int c_end = BN_TILE / 32, int nslots = 2) {
    const int row = row_base + lane;
    // epilogues that read a bf16 operand (R, U): this chunk's 64 B of it are requested before the
    // TMEM load, and the next chunk's are pulled into L2, so the global latency overlaps the
    // accumulator drain instead of serialising once per 32-column chunk
    const bool reads_aux = p.tma_epi && p.aux &&
                           (p.epi == SWARM_EPI_RESIDUAL || p.epi == SWARM_EPI_DGELU || p.epi == SWARM_EPI_MUL);
    const bool pre = reads_aux && p.aux_prefetch;
#pragma unroll 1
    for (int c = c_begin; c < c_end; ++c) {
        const int col0 = col_tile0 + c * 32;
        uint4 a4[4];
        if (pre && row < p.m && col0 < p.n) {
            const uint4* src =
                reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.aux) + (rd + row) * p.ldd + cd + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q) a4[q] = src[q];
            if (c + 1 < BN_TILE / 32 && col0 + 32 < p.n)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 4));
        }
        uint32_t rr[32];
        tmem_ld_32x32b_x32(taddr + static_cast<uint32_t>(c * 32), rr);
        tmem_ld_wait();
        if (col0 >= p.n) continue;  // warp-uniform
        if (reads_aux && !pre && row < p.m) {  // SWARM_GEMM_AUX_PREFETCH=0: load after the drain
            const uint4* src =
                reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.aux) + (rd + row) * p.ldd + cd + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q) a4[q] = src[q];
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
        for (int f = 0; f < nfix; ++f) {
            const float4* src = sk_part(p, fix_slots, f, fix_row) + c * 256 + lane;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 w = __ldcg(src + j * 32);
                v[4 * j] += w.x;
                v[4 * j + 1] += w.y;
                v[4 * j + 2] += w.z;
                v[4 * j + 3] += w.w;
            }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= p.alpha;
        const long long off = (rd + row) * p.ldd + cd + col0;
        if (!p.tma_epi) {
            if (row < p.m) epilogue_chunk(p, v, off, min(32, p.n - col0));
            continue;
        }
        uint8_t* slot = stg + (nslots == 2 ? slot_idx : 0) * kEpiSlot;
        slot_idx ^= 1;
        if (lane == 0) {  // the store issued from this slot (two chunks ago; one with a single slot) has read it
            if (nslots == 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
        }
        __syncwarp();
        const bool row_ok = row < p.m;
        const int gc = static_cast<int>(cd) + col0, gr = static_cast<int>(rd) + row_base;
        switch (p.epi) {
            case SWARM_EPI_STORE_F32:
            case SWARM_EPI_ACCUM_F32:
                stage_f32(slot, lane, v);
                break;
            case SWARM_EPI_RESIDUAL:
                if (row_ok) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 w = a4[q];
                        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            v[q * 8 + 2 * j] += bf_lo(ws[j]);
                            v[q * 8 + 2 * j + 1] += bf_hi(ws[j]);
                        }
                    }
                }
                stage_bf16(slot, lane, v);
                break;
            case SWARM_EPI_GELU:
                stage_bf16(slot + 2048, lane, v);  // U = pre-activation
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
                stage_bf16(slot, lane, v);
                break;
            case SWARM_EPI_DGELU:
                if (row_ok) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 w = a4[q];
                        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            v[q * 8 + 2 * j] *= dgelu_f(bf_lo(ws[j]));
                            v[q * 8 + 2 * j + 1] *= dgelu_f(bf_hi(ws[j]));
                        }
                    }
                }
                stage_bf16(slot, lane, v);
                break;
            case SWARM_EPI_GELU_DERIV: {  // U = gelu'(pre-activation), D = gelu(pre-activation)
                float dg[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) gelu_both(v[j], v[j], dg[j]);
                stage_bf16(slot + 2048, lane, dg);
                stage_bf16(slot, lane, v);
                break;
            }
            case SWARM_EPI_MUL:  // D = acc * U (U = gelu' saved by the forward)
                if (row_ok) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 w = a4[q];
                        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            v[q * 8 + 2 * j] *= bf_lo(ws[j]);
                            v[q * 8 + 2 * j + 1] *= bf_hi(ws[j]);
                        }
                    }
                }
                stage_bf16(slot, lane, v);
                break;
            default:
                stage_bf16(slot, lane, v);
                break;
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0 && row_base < p.m && !(p.dbg & 1)) {
            if (p.epi == SWARM_EPI_ACCUM_F32) tma_reduce_add_2d(md, slot, gc, gr);
            else tma_store_2d(md, slot, gc, gr);
            if (p.epi == SWARM_EPI_GELU || p.epi == SWARM_EPI_GELU_DERIV) tma_store_2d(mu, slot + 2048, gc, gr);
            bulk_commit();
        }
    }
}

// k-block range of m-tile mt (all of K unless A is triangular, see k_tri)
__device__ __forceinline__ void k_range(const Params& p, int mt, int& kb0, int& kb1) {
    kb0 = 0;
    kb1 = p.k_blocks;
    if (p.k_tri == 1) kb1 = min(p.k_blocks, ((mt + 1) * BM + BK - 1) / BK);
    else if (p.k_tri == 2) kb0 = (mt * BM) / BK;
}

template <int BN, bool A_MN, bool B_MN, int MINB = 1>
__global__ void __launch_bounds__(kThreads, MINB)
    k_gemm(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
           const __grid_constant__ CUtensorMap tma_d, const __grid_constant__ CUtensorMap tma_u, const Params p) {
    using C = Cfg<BN, MINB>;
    pdl_trigger();
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw & 1023)) & 1023);
    uint8_t* sa = smem;
    uint8_t* sb = smem + C::STAGES * C::A_BYTES;
    uint8_t* stg_all = sb + C::STAGES * C::B_BYTES;  // epilogue staging, 1024-aligned
    uint64_t* full = reinterpret_cast<uint64_t*>(stg_all + kEpiSmem);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 4);
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        tmem_alloc(tmem_slot, C::TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // the previous kernel's outputs (our operands) are complete from here on

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
                const int z = t / p.tiles_per_batch;
                const int r = t - z * p.tiles_per_batch;
                const int mt = r % p.tiles_m, nt = r / p.tiles_m;
                const int zb = z / p.bh, zh = z - zb * p.bh;
                const int ra = p.ra0 * zb + p.ra1 * zh, ca = p.ca0 * zb + p.ca1 * zh;
                const int rb = p.rb0 * zb + p.rb1 * zh, cb = p.cb0 * zb + p.cb1 * zh;
                int kb0, kb1;
                k_range(p, mt, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
                    uint8_t* a_dst = sa + stage * C::A_BYTES;
                    uint8_t* b_dst = sb + stage * C::B_BYTES;
                    if constexpr (!A_MN) {
                        tma_load_2d(a_dst, &tma_a, &full[stage], ca + kb * BK, ra + mt * BM);
                    } else {
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j)
                            tma_load_2d(a_dst + j * (64 * BK * 2), &tma_a, &full[stage], ca + mt * BM + j * 64,
                                        ra + kb * BK);
                    }
                    if constexpr (!B_MN) {
                        tma_load_2d(b_dst, &tma_b, &full[stage], cb + kb * BK, rb + nt * BN);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            tma_load_2d(b_dst + j * (64 * BK * 2), &tma_b, &full[stage], cb + nt * BN + j * 64,
                                        rb + kb * BK);
                    }
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
                const int r = t % p.tiles_per_batch;
                int kb0, kb1;
                k_range(p, r % p.tiles_m, kb0, kb1);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sa + stage * C::A_BYTES);
                    const uint32_t b_base = smem_u32(sb + stage * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t ad = A_MN ? make_sdesc(a_base + k * 2048, 64 * BK * 2, 1024)
                                                 : make_sdesc(a_base + k * 32, 16, 1024);
                        const uint64_t bd = B_MN ? make_sdesc(b_base + k * 2048, 64 * BK * 2, 1024)
                                                 : make_sdesc(b_base + k * 32, 16, 1024);
                        mma_bf16(d_tmem, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue (TMEM -> HBM)
        const int q = warp - 4;  // TMEM lane quarter owned by this warp (warp % 4)
        uint8_t* stg = stg_all + q * 2 * kEpiSlot;
        int slot_idx = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
            const int z = t / p.tiles_per_batch;
            const int r = t - z * p.tiles_per_batch;
            const int mt = r % p.tiles_m, nt = r / p.tiles_m;
            const int zb = z / p.bh, zh = z - zb * p.bh;
            const long long rd = p.rd0 * zb + p.rd1 * zh, cd = p.cd0 * zb + p.cd1 * zh;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            drain_tile<BN>(p, &tma_d, &tma_u, stg, slot_idx,
                           tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN),
                           mt * BM + q * 32, rd, cd, nt * BN, lane);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (lane == 0) bulk_wait_all();  // TMA stores drained before the CTA exits
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, C::TMEM_COLS);
    }
}

// ------------------------------------------------- 2-CTA pair variant (M=256)
// A cluster of two CTAs on one TPC computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2: each CTA stages its own 128 rows of A and its own
// 128 rows (N) of B, so per-SM operand traffic (TMA ingest and smem reads) is
// half of the single-CTA 128 x 256 tile for the same MMA rate.  The leader
// (rank 0) issues the MMAs; both CTAs' TMA loads complete on the leader's full
// barrier; commits multicast to both CTAs' empty / tmem-full barriers; both
// CTAs' epilogue warps release the accumulator on the leader's tmem-empty.
constexpr int PAIR_BN = 256;
constexpr int kMaxSkParts = 8;  // host keeps every stream-K tile within this many clusters

// One work unit of a cluster: k-blocks [kb0, kb1) of `tile`.  Whole tiles come
// first (data-parallel waves), then this cluster's contiguous stream-K range.
struct Unit {
    int tile, kb0, kb1;
    int sk;     // stream-K tile index (tile - dp_tiles), -1 for a data-parallel tile
    int first;  // 1 when the unit opens this cluster's stream-K range
};
__device__ __forceinline__ int sk_bound(const Params& p, int c, int n_clusters) {
    return static_cast<int>(static_cast<long long>(c) * p.sk_iters / n_clusters);
}
struct UnitIter {
    int c, nc, t, i, e, b;
    __device__ UnitIter(const Params& p, int cluster, int n_clusters)
        : c(cluster), nc(n_clusters), t(cluster), i(sk_bound(p, cluster, n_clusters)),
          e(sk_bound(p, cluster + 1, n_clusters)), b(i) {}
    __device__ bool next(const Params& p, Unit& u) {
        if (t < p.dp_tiles) {
            u = Unit{t, 0, p.k_blocks, -1, 0};
            t += nc;
            return true;
        }
        if (i >= e) return false;
        const int st = i / p.k_blocks, k0 = i - st * p.k_blocks;
        const int k1 = min(p.k_blocks, k0 + (e - i));
        u = Unit{p.dp_tiles + st, k0, k1, st, i == b ? 1 : 0};
        i += k1 - k0;
        return true;
    }
};
// Partial-sum slot of the segment of stream-K tile `st` computed by cluster cc:
// a cluster owns at most one segment that opens its range (slot 0) and one that
// closes it mid-tile (slot 1).  Returns -1 when cc has no segment of st.
__device__ __forceinline__ int sk_slot(const Params& p, int st, int cc, int n_clusters) {
    const int lo = st * p.k_blocks, hi = lo + p.k_blocks;
    const int b0 = sk_bound(p, cc, n_clusters), b1 = sk_bound(p, cc + 1, n_clusters);
    const int s0 = max(b0, lo), s1 = min(b1, hi);
    if (s0 >= s1) return -1;
    return cc * 2 + (s0 == b0 ? 0 : 1);
}

struct Cfg2 {
    static constexpr int A_BYTES = 128 * BK * 2;  // this CTA's half of A
    static constexpr int B_BYTES = 128 * BK * 2;  // this CTA's half of B
    static constexpr int STAGES = 6;
    static constexpr int TMEM_COLS = 2 * PAIR_BN;
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + kEpiSmem + 1024 + 256;
    static_assert(SMEM <= 232448, "pair GEMM exceeds the 227 KB dynamic smem limit");
    static_assert(2 * STAGES * 8 + 4 * 8 + 4 <= 256, "barrier area overflow");
};

// EPI8: eight epilogue warps (2-9, two per TMEM lane quarter, each group half of a tile's columns,
// one staging slot each) instead of four (4-7): the fused epilogues' arithmetic is halved per warp
template <bool A_MN, bool B_MN, int NPAIR, bool EPI8 = false>
__global__ void __launch_bounds__(EPI8 ? 320 : kThreads, 1)
    k_gemm2(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
            const __grid_constant__ CUtensorMap tma_d, const __grid_constant__ CUtensorMap tma_u,
            const __grid_constant__ CUtensorMap tma_a2, const __grid_constant__ CUtensorMap tma_b2, const Params p) {
    using C = Cfg2;
    pdl_trigger();
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw & 1023)) & 1023);
    uint8_t* sa = smem;
    uint8_t* sb = smem + C::STAGES * C::A_BYTES;
    uint8_t* stg_all = sb + C::STAGES * C::B_BYTES;  // epilogue staging, 1024-aligned
    uint64_t* full = reinterpret_cast<uint64_t*>(stg_all + kEpiSmem);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // cluster = NPAIR CTA pairs side by side in N; CTA rank = 2*pair + half
    const uint32_t rank = cluster_ctarank();
    const int pair = static_cast<int>(rank >> 1);
    const int half = static_cast<int>(rank & 1);
    const bool leader = half == 0;
    const int cluster = blockIdx.x / (2 * NPAIR);
    const int n_clusters = gridDim.x / (2 * NPAIR);
    const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pair));
    const uint16_t all_mask = static_cast<uint16_t>((1u << (2 * NPAIR)) - 1);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        if (p.kb_half) {
            tma_prefetch(&tma_a2);
            tma_prefetch(&tma_b2);
        }
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NPAIR);  // every pair's MMA frees a stage its A multicast wrote
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], EPI8 ? 16 : 8);  // epilogue warps x 2 CTAs (only the leader's is used)
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
        tmem_relinquish_pair();
    }
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // the previous kernel's outputs (our operands) are complete from here on

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            UnitIter it(p, cluster, n_clusters);
            Unit u;
            while (it.next(p, u)) {
                const int z = u.tile / p.tiles_per_batch;
                const int r = u.tile - z * p.tiles_per_batch;
                const int mt = r % p.tiles_m, nt = r / p.tiles_m;
                const int zb = z / p.bh, zh = z - zb * p.bh;
                const int ra = p.ra0 * zb + p.ra1 * zh, ca = p.ca0 * zb + p.ca1 * zh;
                const int rb = p.rb0 * zb + p.rb1 * zh, cb = p.cb0 * zb + p.cb1 * zh;
                const int m0 = mt * 256 + half * 128;
                const int n0 = (nt * NPAIR + pair) * PAIR_BN + half * 128;
                for (int kb = u.kb0; kb < u.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (p.dbg & 4) {  // experiment: no operand traffic
                        if (leader) mbar_arrive(&full[stage]);
                        if (++stage == C::STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
                    const uint32_t bar = pair_leader_addr(&full[stage]);
                    uint8_t* a_dst = sa + stage * C::A_BYTES;
                    uint8_t* b_dst = sb + stage * C::B_BYTES;
                    // two-segment K (paired microbatches): the second half of K lives in other buffers
                    const bool seg2 = p.kb_half && kb >= p.kb_half;
                    const CUtensorMap* ma = seg2 ? &tma_a2 : &tma_a;
                    const CUtensorMap* mb = seg2 ? &tma_b2 : &tma_b;
                    const int kk = seg2 ? kb - p.kb_half : kb;
                    if constexpr (NPAIR == 1) {
                        if constexpr (!A_MN) {
                            tma_load_2d_pair(a_dst, ma, bar, ca + kk * BK, ra + m0);
                        } else {
#pragma unroll
                            for (int j = 0; j < 2; ++j)
                                tma_load_2d_pair(a_dst + j * (64 * BK * 2), ma, bar, ca + m0 + j * 64, ra + kk * BK);
                        }
                    } else {
                        // both pairs need this A half: each pair loads one 64-row (K-major) or
                        // 64-column (MN-major) piece and multicasts it to the same half of every pair
                        const uint16_t mc = static_cast<uint16_t>(0x5u << half);
                        if constexpr (!A_MN)
                            tma_load_2d_pair_mc(a_dst + pair * (64 * 128), ma, bar, ca + kk * BK, ra + m0 + pair * 64,
                                                mc);
                        else
                            tma_load_2d_pair_mc(a_dst + pair * (64 * BK * 2), ma, bar, ca + m0 + pair * 64,
                                                ra + kk * BK, mc);
                    }
                    if constexpr (!B_MN) {
                        tma_load_2d_pair(b_dst, mb, bar, cb + kk * BK, rb + n0);
                    } else {
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            tma_load_2d_pair(b_dst + j * (64 * BK * 2), mb, bar, cb + n0 + j * 64, rb + kk * BK);
                    }
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ------------------------------------------------ MMA issuer (leader only)
            constexpr uint32_t idesc = make_idesc_bf16(256, PAIR_BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            UnitIter it(p, cluster, n_clusters);
            Unit u;
            while (it.next(p, u)) {
                const int kb0 = u.kb0, kb1 = u.kb1;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * PAIR_BN);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sa + stage * C::A_BYTES);
                    const uint32_t b_base = smem_u32(sb + stage * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t ad = A_MN ? make_sdesc(a_base + k * 2048, 64 * BK * 2, 1024)
                                                 : make_sdesc(a_base + k * 32, 16, 1024);
                        const uint64_t bd = B_MN ? make_sdesc(b_base + k * 2048, 64 * BK * 2, 1024)
                                                 : make_sdesc(b_base + k * 32, 16, 1024);
                        if (!(p.dbg & 2)) mma_bf16_pair(d_tmem, ad, bd, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                    }
                    mma_commit_pair(&empty[stage], all_mask);
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit_pair(&tfull[acc], pair_mask);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (EPI8 ? warp >= 2 : warp >= 4) {
        // ------------------------------------------------ epilogue (both CTAs, own 128 rows)
        const int q = warp & 3;
        const int grp = EPI8 ? (warp - 2) >> 2 : 0;  // EPI8: column half of the tile
        const uint32_t tempty_leader[2] = {map_to_cta(&tempty[0], rank & ~1u), map_to_cta(&tempty[1], rank & ~1u)};
        uint8_t* stg = stg_all + (EPI8 ? (warp - 2) : 2 * q) * kEpiSlot;
        int slot_idx = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        UnitIter it(p, cluster, n_clusters);
        Unit u;
        while (it.next(p, u)) {
            const int z = u.tile / p.tiles_per_batch;
            const int r = u.tile - z * p.tiles_per_batch;
            const int mt = r % p.tiles_m, nt = r / p.tiles_m;
            const int zb = z / p.bh, zh = z - zb * p.bh;
            const long long rd = p.rd0 * zb + p.rd1 * zh, cd = p.cd0 * zb + p.cd1 * zh;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr =
                tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * PAIR_BN);
            uint64_t fix_slots = 0;  // other contributors' slots, 8 bits each
            int nfix = 0;
            const size_t fix_row = static_cast<size_t>(half * 128 + q * 32) * PAIR_BN;
            bool drain = true;
            if (!EPI8 && u.sk >= 0 && (u.kb0 != 0 || u.kb1 != p.k_blocks) && !(p.dbg & 8)) {
                // stream-K partial tile: the last of its clusters to arrive (per warp
                // quarter) sums everyone's partials and runs the epilogue; the others
                // park their fp32 partial in the workspace.  Nobody waits on a
                // cluster that has not arrived, so co-residency is never assumed.
                const int wq = half * 4 + q;
                int* cnt = p.sk_cnt + u.sk * 8 + wq;
                int order = 0;
                if (lane == 0) order = atomicAdd(cnt, 1);
                order = __shfl_sync(0xffffffffu, order, 0);
                const int lo = u.sk * p.k_blocks;
                int c_lo = static_cast<int>(static_cast<long long>(lo) * n_clusters / p.sk_iters);
                while (c_lo > 0 && sk_bound(p, c_lo, n_clusters) > lo) --c_lo;
                int parts = 0, my_slot = cluster * 2 + (u.first ? 0 : 1);
                for (int cc = c_lo; cc < n_clusters && sk_bound(p, cc, n_clusters) < lo + p.k_blocks; ++cc) {
                    const int sl = sk_slot(p, u.sk, cc, n_clusters);
                    if (sl < 0) continue;
                    ++parts;
                    if (sl != my_slot && nfix < kMaxSkParts) fix_slots |= static_cast<uint64_t>(sl) << (8 * nfix++);
                }
                if (order < parts - 1) {
                    float* dst = p.ws + static_cast<size_t>(my_slot) * 2 * 128 * PAIR_BN + fix_row;
#pragma unroll 1
                    for (int c = 0; c < PAIR_BN / 32; ++c) {
                        uint32_t rr[32];
                        tmem_ld_32x32b_x32(taddr + static_cast<uint32_t>(c * 32), rr);
                        tmem_ld_wait();
                        float4* d4 = reinterpret_cast<float4*>(dst) + c * 256 + lane;
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            __stcg(d4 + j * 32, make_float4(__uint_as_float(rr[4 * j]), __uint_as_float(rr[4 * j + 1]),
                                                       __uint_as_float(rr[4 * j + 2]), __uint_as_float(rr[4 * j + 3])));
                    }
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) st_release_gpu(p.sk_ready + my_slot * 8 + wq, 1);
                    drain = false;
                    nfix = 0;
                } else {
                    if (lane == 0) *cnt = 0;  // every contributor has arrived: reset for the next launch
                    for (int f = 0; f < nfix; ++f) {
                        const int sl = static_cast<int>((fix_slots >> (8 * f)) & 0xff);
                        while (!(p.dbg & 16) && ld_acquire_gpu(p.sk_ready + sl * 8 + wq) == 0) {
                        }
                    }
                }
            }
            if (drain)
                drain_tile<PAIR_BN>(p, &tma_d, &tma_u, stg, slot_idx, taddr, mt * 256 + half * 128 + q * 32, rd, cd,
                                    (nt * NPAIR + pair) * PAIR_BN, lane, fix_slots, nfix, fix_row,
                                    EPI8 ? grp * (PAIR_BN / 64) : 0, EPI8 ? (grp + 1) * (PAIR_BN / 64) : PAIR_BN / 32,
                                    EPI8 ? 1 : 2);
            __syncwarp();
            if (lane == 0)
                for (int f = 0; f < nfix; ++f)
                    p.sk_ready[static_cast<int>((fix_slots >> (8 * f)) & 0xff) * 8 + half * 4 + q] = 0;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    cluster_sync();  // both CTAs finished every MMA / TMEM read before the pair frees TMEM
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
    }
}

// ---------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(ptr);
    });
    return fn;
}

// Descriptor cache: a training step re-issues the same few hundred
// (pointer, shape, box) operands every microbatch, so encode each once.
struct MapKey {
    const void* ptr;
    long long rows, cols, ld;
    int bi, bo;
    bool operator==(const MapKey& o) const {
        return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && bi == o.bi && bo == o.bo;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        size_t h = reinterpret_cast<uintptr_t>(k.ptr);
        for (long long v : {k.rows, k.cols, k.ld, static_cast<long long>(k.bi) << 16 | k.bo})
            h = h * 0x9E3779B97F4A7C15ull + static_cast<size_t>(v);
        return h;
    }
};

int encode_2d_uncached(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box_inner,
                       int box_outer);

int encode_2d(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box_inner,
              int box_outer) {
    thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    const MapKey key{ptr, rows, cols, ld, box_inner, box_outer};
    auto it = cache.find(key);
    if (it != cache.end()) {
        *m = it->second;
        return SWARM_OK;
    }
    const int rc = encode_2d_uncached(m, ptr, rows, cols, ld, box_inner, box_outer);
    if (rc == SWARM_OK) {
        if (cache.size() > 16384) cache.clear();  // bounded: pointers of freed buffers age out
        cache.emplace(key, *m);
    }
    return rc;
}

int encode_2d_uncached(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box_inner,
                       int box_outer) {
    EncodeFn enc = get_encode();
    if (!enc) {
        set_error("gemm: cuTensorMapEncodeTiled unavailable");
        return SWARM_E_CUDA;
    }
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("gemm: cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
        return SWARM_E_INVALID;
    }
    return SWARM_OK;
}

// Output map for the TMA epilogue: 32 x 32 boxes, fp32 (128-B rows, SWIZZLE_128B)
// or bf16 (64-B rows, SWIZZLE_64B), matching stage_f32 / stage_bf16.
int encode_2d_out_uncached(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, bool f32);

int encode_2d_out(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, bool f32) {
    thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    const MapKey key{ptr, rows, cols, ld, f32 ? -32 : -16, 32};  // negative box tags: output maps
    auto it = cache.find(key);
    if (it != cache.end()) {
        *m = it->second;
        return SWARM_OK;
    }
    const int rc = encode_2d_out_uncached(m, ptr, rows, cols, ld, f32);
    if (rc == SWARM_OK) {
        if (cache.size() > 16384) cache.clear();
        cache.emplace(key, *m);
    }
    return rc;
}

int encode_2d_out_uncached(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, bool f32) {
    EncodeFn enc = get_encode();
    if (!enc) return SWARM_E_CUDA;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * (f32 ? 4 : 2)};
    const cuuint32_t box[2] = {32, 32};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? SWARM_OK : SWARM_E_INVALID;
}

// Stream-K runs only when the caller passes a workspace; see the policy in
// swarm_gemm_bf16 and the measurements in profiles/r01_gemm_experiments.md.
// Stream-K scratch layout (caller-owned, see swarm_gemm_args.workspace):
// [arrival counters | ready flags | partial accumulators].
constexpr int kMaxClusters = 128;
constexpr size_t kSkFlagBytes = 65536;
static_assert(kMaxClusters * 8 * 3 * sizeof(int) <= kSkFlagBytes, "flag area");
int streamk_mode() {  // SWARM_GEMM_STREAMK: 0 never, 1 whenever shorter, unset: when it pays >= 25%
    static const int m = [] {
        const char* e = getenv("SWARM_GEMM_STREAMK");
        return e ? (e[0] == '0' ? 0 : 1) : 2;
    }();
    return m;
}

size_t sk_bytes(int clusters) {
    return kSkFlagBytes + static_cast<size_t>(clusters) * 2 * 2 * 128 * PAIR_BN * sizeof(float);
}

bool tma_epi_enabled() {
    static const bool on = [] {
        const char* e = getenv("SWARM_GEMM_TMA_EPI");
        return !(e && e[0] == '0');
    }();
    return on;
}

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = kNumSMs;
    }
    return n;
}

template <int BN, bool A_MN, bool B_MN, int MINB = 1>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td, const CUtensorMap& tu, const Params& p,
           cudaStream_t st) {
    auto kern = k_gemm<BN, A_MN, B_MN, MINB>;
    static bool attr = false;
    if (!attr) {
        SWARM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN, MINB>::SMEM));
        attr = true;
    }
    const int grid = std::min(p.total_tiles, num_sms() * MINB);
    SWARM_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(kThreads), Cfg<BN, MINB>::SMEM, st, ta, tb, td, tu, p));
    SWARM_LAUNCH_CHECK("k_gemm");
    return SWARM_OK;
}

// SWARM_GEMM_EPI8: 0 = four epilogue warps, 1 = eight, 2 (default) = eight for bf16 outputs only
// (an fp32 chunk fills a warp's whole staging slot, so with eight warps and one slot each
// the reduce-add / store of chunk c must finish reading before chunk c+1 is staged:
// fp32 outputs measured 2.5-3.5% faster with four double-buffered warps, scripts/ffn_epi_probe.py)
int epi8_mode() {
    static const int m = [] {
        const char* e = getenv("SWARM_GEMM_EPI8");
        return e ? atoi(e) : 2;
    }();
    return m;
}
bool epi8_for(int epi) {
    const int m = epi8_mode();
    if (m == 0) return false;
    return m != 2 || (epi != SWARM_EPI_STORE_F32 && epi != SWARM_EPI_ACCUM_F32);
}

template <bool A_MN, bool B_MN, int NPAIR, bool EPI8>
int launch_pair_k(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td, const CUtensorMap& tu,
                  const CUtensorMap& ta2, const CUtensorMap& tb2, const Params& p, int clusters, cudaStream_t st);

template <bool A_MN, bool B_MN, int NPAIR>
int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td, const CUtensorMap& tu,
                const CUtensorMap& ta2, const CUtensorMap& tb2, const Params& p, int clusters, cudaStream_t st) {
    // eight epilogue warps unless stream-K partial tiles are in play (their fix-up is per warp quarter)
    if (epi8_for(p.epi) && p.sk_tiles == 0)
        return launch_pair_k<A_MN, B_MN, NPAIR, true>(ta, tb, td, tu, ta2, tb2, p, clusters, st);
    return launch_pair_k<A_MN, B_MN, NPAIR, false>(ta, tb, td, tu, ta2, tb2, p, clusters, st);
}

template <bool A_MN, bool B_MN, int NPAIR, bool EPI8>
int launch_pair_k(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td, const CUtensorMap& tu,
                  const CUtensorMap& ta2, const CUtensorMap& tb2, const Params& p, int clusters, cudaStream_t st) {
    auto kern = k_gemm2<A_MN, B_MN, NPAIR, EPI8>;
    static bool attr = false;
    if (!attr) {
        SWARM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2::SMEM));
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * NPAIR * clusters);
    cfg.blockDim = dim3(EPI8 ? 320 : kThreads);
    cfg.dynamicSmemBytes = Cfg2::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2 * NPAIR;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1 + pdl_attr(&attrs[1]);
    SWARM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, td, tu, ta2, tb2, p));
    SWARM_LAUNCH_CHECK("k_gemm2");
    return SWARM_OK;
}

// How many 2-CTA clusters of the pair kernel can be resident at once.  On B200
// this is below num_sms / 2 (GPCs with an odd number of usable SMs strand one
// SM each), and a persistent grid larger than it runs its extra clusters as a
// second wave — doubling a stream-K launch, whose clusters all get equal work.
template <int NPAIR>
int query_clusters() {
    const int cap = num_sms() / (2 * NPAIR);
    auto kern = k_gemm2<false, false, NPAIR>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2::SMEM) != cudaSuccess) {
        cudaGetLastError();
        return cap;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * NPAIR * cap);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg2::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2 * NPAIR;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess || c <= 0) {
        cudaGetLastError();
        return cap;
    }
    return std::min(c, cap);
}

int max_pair_clusters() {
    static const int n = query_clusters<1>();
    return n;
}
int max_quad_clusters() {  // 4-CTA clusters of the multicast variant
    static const int n = query_clusters<2>();
    return n;
}

template <int NPAIR>
int dispatch_pair(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td,
                  const CUtensorMap& tu, const CUtensorMap& ta2, const CUtensorMap& tb2, const Params& p, int clusters,
                  cudaStream_t st) {
    if (!amn && !bmn) return launch_pair<false, false, NPAIR>(ta, tb, td, tu, ta2, tb2, p, clusters, st);
    if (!amn && bmn) return launch_pair<false, true, NPAIR>(ta, tb, td, tu, ta2, tb2, p, clusters, st);
    if (amn && !bmn) return launch_pair<true, false, NPAIR>(ta, tb, td, tu, ta2, tb2, p, clusters, st);
    return launch_pair<true, true, NPAIR>(ta, tb, td, tu, ta2, tb2, p, clusters, st);
}

// 4-CTA clusters (two pairs side by side in N sharing each A sub-tile by TMA
// multicast) are the default where N splits into an even number of 256-wide
// tiles (SWARM_GEMM_MCAST=0 disables them).  Only 33 such clusters are resident
// on B200 (132 SMs, GPC packing), yet halving the A operand feed wins on most
// block shapes, most of all on the MN-major weight-gradient GEMMs
// (profiles/r01_gemm_experiments.md).
int multicast_mode() {
    static const int on = [] {
        const char* e = getenv("SWARM_GEMM_MCAST");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool pair_enabled() {
    static const bool on = [] {
        const char* e = getenv("SWARM_GEMM_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int BN>
int dispatch(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td,
             const CUtensorMap& tu, const Params& p, cudaStream_t st) {
    if constexpr (BN == 128) {
        static const bool two = [] {
            const char* e = getenv("SWARM_GEMM_TWO_CTA");
            return !(e && e[0] == '0');
        }();
        if (two && p.k_blocks <= 16 && p.total_tiles > num_sms()) {  // many short tiles
            if (!amn && !bmn) return launch<BN, false, false, 2>(ta, tb, td, tu, p, st);
            if (!amn && bmn) return launch<BN, false, true, 2>(ta, tb, td, tu, p, st);
            if (amn && !bmn) return launch<BN, true, false, 2>(ta, tb, td, tu, p, st);
            return launch<BN, true, true, 2>(ta, tb, td, tu, p, st);
        }
    }
    if (!amn && !bmn) return launch<BN, false, false>(ta, tb, td, tu, p, st);
    if (!amn && bmn) return launch<BN, false, true>(ta, tb, td, tu, p, st);
    if (amn && !bmn) return launch<BN, true, false>(ta, tb, td, tu, p, st);
    return launch<BN, true, true>(ta, tb, td, tu, p, st);
}

}  // namespace gemm
}  // namespace swarm

extern "C" int swarm_gemm_pair_clusters(void) {
    return swarm::gemm::multicast_mode() ? swarm::gemm::max_quad_clusters() : swarm::gemm::max_pair_clusters();
}

extern "C" size_t swarm_gemm_workspace_bytes(void) {
    using namespace swarm::gemm;
    return sk_bytes(std::min(num_sms() / 2, kMaxClusters));
}

extern "C" int swarm_gemm_bf16(const swarm_gemm_args* a, swarm_stream_t stream) {
    using namespace swarm;
    using namespace swarm::gemm;
    if (!a) return invalid("gemm: null args");
    if (a->m <= 0 || a->n <= 0 || a->k <= 0 || a->batch <= 0 || a->bh <= 0) return invalid("gemm: bad shape");
    if (!a->a || !a->b || !a->d) return invalid("gemm: null operand");
    if ((a->epilogue == SWARM_EPI_RESIDUAL || a->epilogue == SWARM_EPI_GELU || a->epilogue == SWARM_EPI_DGELU ||
         a->epilogue == SWARM_EPI_GELU_DERIV || a->epilogue == SWARM_EPI_MUL) &&
        !a->aux)
        return invalid("gemm: epilogue needs aux");
    if (a->epilogue < 0 || a->epilogue > SWARM_EPI_MUL) return invalid("gemm: bad epilogue");
    if (a->k_tri < 0 || a->k_tri > 2 || (a->k_tri && a->m != a->k)) return invalid("gemm: k_tri needs M == K");
    if (a->lda % 8 || a->ldb % 8 || (reinterpret_cast<uintptr_t>(a->a) & 15) || (reinterpret_cast<uintptr_t>(a->b) & 15))
        return invalid("gemm: A/B rows must be 16-byte aligned");
    const bool two_seg = a->a2 || a->b2;
    if (two_seg) {
        if (!a->a2 || !a->b2 || a->batch != 1 || a->k % (2 * BK) || a->k_tri ||
            (reinterpret_cast<uintptr_t>(a->a2) & 15) || (reinterpret_cast<uintptr_t>(a->b2) & 15))
            return invalid("gemm: two K segments need a2 and b2, batch 1, K a multiple of 128, no k_tri");
        if (!(a->m > 128 && a->n > 128 && pair_enabled())) {
            // the 1-CTA kernel has no second segment: two launches, the second accumulating
            if (a->epilogue != SWARM_EPI_ACCUM_F32 && a->epilogue != SWARM_EPI_STORE_F32)
                return invalid("gemm: two K segments on small tiles need an fp32 epilogue");
            swarm_gemm_args h = *a;
            h.a2 = h.b2 = nullptr;
            h.k = a->k / 2;
            int rc = swarm_gemm_bf16(&h, stream);
            if (rc) return rc;
            h.a = a->a2;
            h.b = a->b2;
            h.epilogue = SWARM_EPI_ACCUM_F32;
            return swarm_gemm_bf16(&h, stream);
        }
    }
    // storage extents (per K segment)
    const long long kseg = two_seg ? a->k / 2 : a->k;
    long long ar = a->a_rows, ac = a->a_cols, br = a->b_rows, bc = a->b_cols;
    if (ar == 0 || ac == 0) {
        ar = a->a_mn_major ? kseg : a->m;
        ac = a->a_mn_major ? a->m : kseg;
    }
    if (br == 0 || bc == 0) {
        br = a->b_mn_major ? kseg : a->n;
        bc = a->b_mn_major ? a->n : kseg;
    }
    // 2-CTA pair tiles (256 x 256) when both M and N fill them; else one CTA, 128 x BN
    bool pair = pair_enabled() && a->m > 128 && a->n > 128;
    bool narrow = false;  // one-CTA 128 x 128 tiles instead of pair tiles (few-tile shapes, below)
    // two pairs per cluster sharing A by TMA multicast when N splits into an even
    // number of 256-wide tiles (halves the A traffic from L2 per SM)
    const int pair_tiles_n = (a->n + PAIR_BN - 1) / PAIR_BN;
    // Stream-K tail (pair tiles, needs the caller's workspace): whole waves of 256x256
    // tiles stay data-parallel, the last partial wave's tiles are cut into k-block
    // ranges spread evenly over every cluster.  It pays when a GEMM has few tiles and a
    // long K (configs[3]: 512 x 4096 x 16384 = 32 tiles of 256 k-blocks on 74 clusters);
    // for the configs[2] shapes the data-parallel tail is cheaper than it looks (the
    // last wave runs with the L2 feed to itself) and the fixup costs ~40 k-block times,
    // so by default stream-K is chosen only when it still wins by 10% after paying for
    // the fixup (SWARM_GEMM_STREAMK=0 never, =1 whenever the k-block path is shorter).
    const int kblocks = (a->k + BK - 1) / BK;
    bool use_sk = false;
    int sk_C = 0, sk_waves = 0, sk_rem = 0;
    if (pair && a->workspace && streamk_mode() != 0 &&
        a->workspace_bytes >= sk_bytes(std::min(num_sms() / 2, kMaxClusters)) &&
        (reinterpret_cast<uintptr_t>(a->workspace) & 255) == 0) {
        const long long tiles1 = static_cast<long long>((a->m + 255) / 256) * pair_tiles_n * a->batch;
        sk_C = std::min(max_pair_clusters(), kMaxClusters);
        sk_waves = static_cast<int>(tiles1 / sk_C);
        sk_rem = static_cast<int>(tiles1 % sk_C);
        const long long w = static_cast<long long>(sk_rem) * kblocks;
        const long long per = w / sk_C;
        const long long t_dp = static_cast<long long>(sk_waves + (sk_rem ? 1 : 0)) * kblocks;
        const long long t_sk = static_cast<long long>(sk_waves) * kblocks + (w + sk_C - 1) / sk_C;
        // the fixup (every split tile's fp32 partials written and read back through L2)
        // measured ~10-13 us on B200 = ~40 k-block times (scripts/streamk_diag_D.py)
        const bool pays = streamk_mode() == 1 ? t_sk + 2 < t_dp : 10 * (t_sk + 40) <= 9 * t_dp;
        use_sk = sk_rem && per >= 4 && per * (kMaxSkParts - 1) >= kblocks && pays;
    }
    // Few-tile shapes without a paying stream-K split (configs[3]'s o / o-dgrad: 512 x 4096,
    // 32 pair tiles on 74 clusters) fill more SMs with one-CTA 128 x 128 tiles.  Measured
    // per-SM rate of those is ~0.62 of a pair tile's (610 vs 760 TFLOP/s on 512x4096x4096,
    // scripts/gemm_shapes.py), so they are chosen when wave utilisation x 0.62 still wins.
    if (pair && !use_sk && !two_seg) {
        const long long pt = static_cast<long long>((a->m + 255) / 256) * pair_tiles_n * a->batch;
        const long long nt = static_cast<long long>((a->m + 127) / 128) * ((a->n + 127) / 128) * a->batch;
        const long long pc = max_pair_clusters(), sc = num_sms();
        const double u_pair = static_cast<double>(pt) / (((pt + pc - 1) / pc) * pc);
        const double u_narrow = static_cast<double>(nt) / (((nt + sc - 1) / sc) * sc);
        if (u_narrow * 0.62 > u_pair) {
            pair = false;
            narrow = true;
        }
    }
    const int npair = (pair && !use_sk && multicast_mode() && pair_tiles_n % 2 == 0) ? 2 : 1;
    const int BN = pair ? PAIR_BN : (a->n <= 128 || narrow ? 128 : 256);
    const int TM = pair ? 256 : BM;
    CUtensorMap ta, tb;
    const int box_a = a->a_mn_major ? BK : (npair == 2 ? 64 : BM), box_b = a->b_mn_major ? BK : (pair ? 128 : BN);
    int rc = encode_2d(&ta, a->a, ar, ac, a->lda, 64, box_a);
    if (rc) return rc;
    rc = encode_2d(&tb, a->b, br, bc, a->ldb, 64, box_b);
    if (rc) return rc;
    CUtensorMap ta2 = ta, tb2 = tb;
    if (two_seg) {
        rc = encode_2d(&ta2, a->a2, ar, ac, a->lda, 64, box_a);
        if (rc) return rc;
        rc = encode_2d(&tb2, a->b2, br, bc, a->ldb, 64, box_b);
        if (rc) return rc;
    }
    Params p{};
    p.m = a->m;
    p.n = a->n;
    p.k = a->k;
    p.bh = a->bh;
    p.tiles_m = (a->m + TM - 1) / TM;
    p.tiles_n = (a->n + BN - 1) / BN / (pair ? npair : 1);  // cluster tiles along N
    p.tiles_per_batch = p.tiles_m * p.tiles_n;
    p.total_tiles = p.tiles_per_batch * a->batch;
    p.k_blocks = (a->k + BK - 1) / BK;
    p.ra0 = a->ra0; p.ra1 = a->ra1; p.ca0 = a->ca0; p.ca1 = a->ca1;
    p.rb0 = a->rb0; p.rb1 = a->rb1; p.cb0 = a->cb0; p.cb1 = a->cb1;
    p.d = a->d;
    p.ldd = a->ldd;
    p.rd0 = a->rd0; p.rd1 = a->rd1; p.cd0 = a->cd0; p.cd1 = a->cd1;
    p.aux = a->aux;
    p.k_tri = pair ? 0 : a->k_tri;  // the pair kernel computes the zero blocks (still exact)
    p.kb_half = two_seg ? static_cast<int>(kseg / BK) : 0;
    p.alpha = a->alpha;
    p.epi = a->epilogue;
    const int esz = (a->epilogue == SWARM_EPI_STORE_F32 || a->epilogue == SWARM_EPI_ACCUM_F32) ? 4 : 2;
    const int vec_elems = 16 / esz;
    const bool cd_ok = (a->cd0 % vec_elems == 0) && (a->cd1 % vec_elems == 0);
    p.vec_ok = (a->ldd % vec_elems == 0) && cd_ok && ((reinterpret_cast<uintptr_t>(a->d) & 15) == 0) &&
               (!a->aux || (reinterpret_cast<uintptr_t>(a->aux) & 15) == 0);
    // TMA-store epilogue: output extents from the batch offsets; exact tiles or
    // a single batch (so TMA's bounds clipping never writes another batch's rows)
    const int nb = (a->batch + a->bh - 1) / a->bh;
    const long long d_rows = static_cast<long long>(a->rd0) * (nb - 1) + static_cast<long long>(a->rd1) * (a->bh - 1) + a->m;
    const long long d_cols = static_cast<long long>(a->cd0) * (nb - 1) + static_cast<long long>(a->cd1) * (a->bh - 1) + a->n;
    const bool exact = (a->m % TM == 0) && (a->n % 32 == 0);
    {
        static const int dbg = [] {
            const char* e = getenv("SWARM_GEMM_DBG");
            return e ? atoi(e) : 0;
        }();
        p.dbg = dbg;
        static const int pf = [] {
            const char* e = getenv("SWARM_GEMM_AUX_PREFETCH");
            return e && e[0] == '0' ? 0 : 1;
        }();
        p.aux_prefetch = pf;
    }
    p.tma_epi = tma_epi_enabled() && (a->batch == 1 || exact) && d_cols <= a->ldd &&
                ((reinterpret_cast<uintptr_t>(a->d) & 15) == 0) && ((a->ldd * esz) % 16 == 0) &&
                (!a->aux || (reinterpret_cast<uintptr_t>(a->aux) & 15) == 0);
    CUtensorMap td{}, tu{};
    if (p.tma_epi) {
        const bool f32 = esz == 4;
        rc = encode_2d_out(&td, a->d, d_rows, d_cols, a->ldd, f32);
        if (rc == SWARM_OK && (a->epilogue == SWARM_EPI_GELU || a->epilogue == SWARM_EPI_GELU_DERIV))
            rc = encode_2d_out(&tu, a->aux, d_rows, d_cols, a->ldd, false);
        if (rc != SWARM_OK) p.tma_epi = 0;  // fall back to direct stores
    }
    p.dp_tiles = p.total_tiles;
    p.sk_tiles = 0;
    p.sk_iters = 0;
    cudaStream_t st = as_stream(stream);
    const int resident = npair == 1 ? max_pair_clusters() : max_quad_clusters();
    int grid_clusters = std::min(p.total_tiles, resident);
    if (use_sk) {
        p.dp_tiles = sk_waves * sk_C;
        p.sk_tiles = sk_rem;
        p.sk_iters = sk_rem * p.k_blocks;
        p.sk_cnt = static_cast<int*>(a->workspace);
        p.sk_ready = p.sk_cnt + kMaxClusters * 8;
        p.ws = reinterpret_cast<float*>(static_cast<uint8_t*>(a->workspace) + kSkFlagBytes);
        grid_clusters = sk_C;
    }
    if (pair && npair == 2)
        return dispatch_pair<2>(a->a_mn_major, a->b_mn_major, ta, tb, td, tu, ta2, tb2, p, grid_clusters, st);
    if (pair) return dispatch_pair<1>(a->a_mn_major, a->b_mn_major, ta, tb, td, tu, ta2, tb2, p, grid_clusters, st);
    if (BN == 128) return dispatch<128>(a->a_mn_major, a->b_mn_major, ta, tb, td, tu, p, st);
    return dispatch<256>(a->a_mn_major, a->b_mn_major, ta, tb, td, tu, p, st);
}
