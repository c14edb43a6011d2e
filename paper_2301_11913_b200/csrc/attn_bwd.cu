// Fused attention backward (sm_100a, tcgen05 + TMEM + TMA), d_head 128:
//
//   dP = dO V^T,  dS = scale * P * (dP - dO.O),  dV = P^T dO,  dK = dS^T Q,  dQ = dS K
//
// for z = b*H + h, with P the forward's bf16 probabilities.  It replaces the
// score-gradient kernel + three batched GEMMs of the unfused backward: dS never
// leaves shared memory, and dV / dK / dQ come out of this one kernel.
//
// One CTA owns key blocks of 128 keys of one (b, h) and streams the query blocks
// that see them (causal: query blocks >= the key block).  Per query block j:
//   TMA      dO_j, Q_j, P_j (three [128 x 128] bf16 tiles, SWIZZLE_128B 64-column boxes)
//   MMA      dP = dO_j V_i^T            (TMEM columns   0-127, M = queries)
//            dV += P_j^T dO_j           (TMEM columns 384-511, M = keys; P_j read MN-major)
//   rows     dS_j = scale * P_j * (dP - D_j), written over P_j in shared memory
//            (one query row per thread; D_j = dO_j . O_j per row from warp 3)
//   MMA      dK += dS_j^T Q_j           (TMEM columns 256-383; dS read MN-major)
//            dQ_j = dS_j K_i            (TMEM columns 128-255; dS read K-major)
//   rows     dQ_j -> red.global.add into an fp32 accumulator; the last key block to
//            add to query block j (an arrival counter) converts it to bf16 into dqkv
//            and re-zeroes the accumulator and the counter
// and once per key block the dK / dV accumulators go to dqkv in bf16.  The same
// shared-memory tile serves as K-major and MN-major operand (SWIZZLE_128B atoms are
// 8 rows x 128 B either way; only the descriptor's reading of them differs).
//
// Causal work is paired: a CTA takes key blocks t and nkb-1-t, so every CTA streams
// nkb + 1 query blocks (configs[2]: L = 512 -> 2 CTAs per (b, h), 128 CTAs, one wave).
// TMEM: all 512 columns, so one CTA per SM.
//
// Warp roles: warp 0 TMA, warp 1 MMA issuer, warps 2-3 dQ conversion (warp 2 also allocates
// TMEM), warps 4-7 dS rows and warps 8-11 dQ rows, one row per thread (TMEM lane quarter =
// warp % 4).
//
// dQ's fp32 sum over key blocks is taken with atomics, so its order (<= L/128 terms)
// is not fixed; SWARM_ATTN_BWD_FUSED=0 selects the unfused path (csrc/attention.cu +
// batched GEMMs), whose results are order-deterministic.  Parity: tests/test_attention_gpu.py
// (torch fp32 reference of the same op) and the stage tests against the fp64 oracle.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <utility>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"

namespace swarm {
namespace attn {
int map_bf16(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int bi, int bo,
             CUtensorMapSwizzle sw);
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encoder();
}
namespace attn_bwd {

using namespace swarm::sm100;

constexpr int kThreads = 384;
constexpr int kBlk = 128;         // keys per key block = queries per query block
constexpr int kDh = 128;          // d_head
constexpr int kBox = kBlk * 128;  // one [128 rows x 64 columns] bf16 SWIZZLE_128B box: 16 KB
constexpr int kTile = 2 * kBox;   // [128 x 128] bf16: 32 KB
constexpr int kBars = 12;
constexpr int kMaxBlocks = 24;  // query blocks one CTA streams (causal pair: nkb + 1 <= 9; else nkb <= 8)
constexpr int kStg = kBlk * 128;  // dQ staging: [128 rows x 32] fp32, SWIZZLE_128B (16 KB)
constexpr int kSmem = 6 * kTile + 2 * kStg + kBars * 8 + 16 + 4 * kMaxBlocks + 1024;
constexpr uint32_t kColDP = 0, kColDQ = 128, kColDK = 256, kColDV = 384;
static_assert(kSmem <= 232448, "attention backward: shared memory");

struct Params {
    int B, H, L, causal;
    float scale;
    int q_col0, k_col0, v_col0;  // head-0 columns of Q, K, V in the qkv storage
    const __nv_bfloat16* o;      // forward output O [B*L, ld_o], head h at column h*128
    int ld_o;
    float* dq_acc;  // fp32 dQ accumulator [B*L, ld_acc] (zero on entry, left zero)
    int ld_acc;
    int* counters;  // [B*H*(L/128)] key-block arrivals per query block (zero on entry, left zero)
    __nv_bfloat16* dqkv;
    int ld_dqkv, dq_col0, dk_col0, dv_col0;
    int dbg;  // experiments (SWARM_ATTN_BWD_DBG): 1 skips the dQ reductions, 2 the dQ write-out
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&p);
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* m, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void dq_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// 128 fp32 TMEM columns of this thread's lane -> 128 bf16 at dst (16-B aligned)
__device__ __forceinline__ void tmem_row_to_bf16(uint32_t taddr, __nv_bfloat16* dst) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + 32 * c, r);
        tmem_ld_wait();
#pragma unroll
        for (int w = 0; w < 4; ++w)
            d4[4 * c + w] = make_uint4(pack2(__uint_as_float(r[8 * w]), __uint_as_float(r[8 * w + 1])),
                                       pack2(__uint_as_float(r[8 * w + 2]), __uint_as_float(r[8 * w + 3])),
                                       pack2(__uint_as_float(r[8 * w + 4]), __uint_as_float(r[8 * w + 5])),
                                       pack2(__uint_as_float(r[8 * w + 6]), __uint_as_float(r[8 * w + 7])));
    }
}

// the key blocks CTA `t` of a (b, h) owns: causal pairs (t, nkb-1-t), else one
__device__ __forceinline__ int key_blocks(const Params& p, int t, int (&kb)[2]) {
    const int nkb = p.L / kBlk;
    kb[0] = t;
    if (p.causal && nkb - 1 - t != t) {
        kb[1] = nkb - 1 - t;
        return 2;
    }
    return 1;
}

// per-CTA timeline for experiments (SWARM_ATTN_BWD_DBG & 4): globaltimer at fixed points of
// thread 128 (row 0)
constexpr int kTr = 96;
__device__ unsigned long long g_abwd_trace[256][kTr];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TR(i)                                                                            \
    do {                                                                                 \
        if ((p.dbg & 4) && r == 0 && blockIdx.x < 256 && (i) < kTr) g_abwd_trace[blockIdx.x][(i)] = gtime(); \
    } while (0)
#define TRL(i)                                                                                   \
    do {                                                                                         \
        if ((p.dbg & 4) && lane == 0 && blockIdx.x < 256 && (i) < kTr) g_abwd_trace[blockIdx.x][(i)] = gtime(); \
    } while (0)
#define TR0(i)                                                                                        \
    do {                                                                                              \
        if ((p.dbg & 4) && threadIdx.x == 128 && blockIdx.x < 256) g_abwd_trace[blockIdx.x][(i)] = gtime(); \
    } while (0)

__global__ void __launch_bounds__(kThreads, 1)
    k_attn_bwd(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
               const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_o,
               const __grid_constant__ CUtensorMap tm_acc, const Params p) {
    pdl_trigger();
    TR0(0);
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw & 1023)) & 1023);
    uint8_t* sK = smem;
    uint8_t* sV = sK + kTile;
    uint8_t* sDO = sV + kTile;
    uint8_t* sQ = sDO + kTile;
    uint8_t* sP = sQ + kTile;  // P_j, then dS_j in place
    uint8_t* sO = sP + kTile;
    uint8_t* sStg = sO + kTile;  // two dQ staging buffers
    uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + 2 * kStg);
    uint64_t* kv_full = bars + 0;      // TMA: K_i, V_i landed
    uint64_t* kv_free = bars + 1;      // MMA: done with K_i, V_i
    uint64_t* ld_full = bars + 2;      // TMA: dO_j, Q_j, P_j, O_j landed
    uint64_t* ld_free = bars + 3;      // MMA (after the rows' dS): done with dO_j, Q_j, dS_j, O_j
    uint64_t* mma12 = bars + 4;        // dP, dV updated
    uint64_t* ds_ready = bars + 5;     // dS rows: dS_j written (4 warps)
    uint64_t* mma34 = bars + 6;        // dK updated, dQ_j ready
    uint64_t* dq_free = bars + 7;      // dQ rows: dQ_j read out of TMEM (4 warps)
    uint64_t* acc_full = bars + 8;     // dK, dV of the key block complete
    uint64_t* acc_free = bars + 9;     // dK (dS rows) and dV (dQ rows) read out (8 warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kBars);
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
    // dQ rows -> converter: per block, whether this CTA was the last to add to its query block
    volatile int* conv_posted = reinterpret_cast<volatile int*>(tmem_slot + 2);
    int* conv_flag = reinterpret_cast<int*>(tmem_slot + 4);  // [kMaxBlocks]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nz = p.B * p.H, nqb = p.L / kBlk;
    const int z = static_cast<int>(blockIdx.x) % nz, t = static_cast<int>(blockIdx.x) / nz;
    const int zb = z / p.H, zh = z - zb * p.H;
    int kbs[2] = {0, 0};
    const int nk = key_blocks(p, t, kbs);

    if (warp == 0 && lane == 0) {
        mbar_init(kv_full, 1);
        mbar_init(kv_free, 1);
        mbar_init(ld_full, 1);
        mbar_init(ld_free, 1);
        mbar_init(mma12, 1);
        mbar_init(ds_ready, 4);
        mbar_init(mma34, 1);
        mbar_init(dq_free, 4);
        mbar_init(acc_full, 1);
        mbar_init(acc_free, 8);
        *conv_posted = 0;
        fence_barrier_init();
    }
    if (warp == 2) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
                TR0(1);
    pdl_wait();

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA
            int n = 0;
            for (int ti = 0; ti < nk; ++ti) {
                const int kb = kbs[ti];
                if (ti > 0) mbar_wait(kv_free, (ti - 1) & 1);
                if (ti > 0) TRL(90);
                mbar_arrive_expect_tx(kv_full, 2 * kTile);
                const int krow = zb * p.L + kb * kBlk;
                for (int b = 0; b < 2; ++b) {
                    tma_load_2d(sK + b * kBox, &tm_qkv, kv_full, p.k_col0 + zh * kDh + 64 * b, krow);
                    tma_load_2d(sV + b * kBox, &tm_qkv, kv_full, p.v_col0 + zh * kDh + 64 * b, krow);
                }
                if (ti == 0 && nk == 2)  // the second key block's K, V: to L2 now, to smem at the switch
                    for (int b = 0; b < 2; ++b) {
                        const int krow2 = zb * p.L + kbs[1] * kBlk;
                        tma_prefetch_l2(&tm_qkv, p.k_col0 + zh * kDh + 64 * b, krow2);
                        tma_prefetch_l2(&tm_qkv, p.v_col0 + zh * kDh + 64 * b, krow2);
                    }
                for (int j = p.causal ? kb : 0; j < nqb; ++j, ++n) {
                    if (j + 1 < nqb)  // the next query block's tiles to L2 while this one computes
                        for (int b = 0; b < 2; ++b) {
                            const int qrow2 = zb * p.L + (j + 1) * kBlk;
                            tma_prefetch_l2(&tm_do, zh * kDh + 64 * b, qrow2);
                            tma_prefetch_l2(&tm_qkv, p.q_col0 + zh * kDh + 64 * b, qrow2);
                            tma_prefetch_l2(&tm_p, kb * kBlk + 64 * b, z * p.L + (j + 1) * kBlk);
                            tma_prefetch_l2(&tm_o, zh * kDh + 64 * b, qrow2);
                        }
                    if (n > 0) mbar_wait(ld_free, (n - 1) & 1);
                    if (ti > 0) TRL(91);
                    mbar_arrive_expect_tx(ld_full, 4 * kTile);
                    const int qrow = zb * p.L + j * kBlk;
                    for (int b = 0; b < 2; ++b) {
                        tma_load_2d(sDO + b * kBox, &tm_do, ld_full, zh * kDh + 64 * b, qrow);
                        tma_load_2d(sQ + b * kBox, &tm_qkv, ld_full, p.q_col0 + zh * kDh + 64 * b, qrow);
                        tma_load_2d(sP + b * kBox, &tm_p, ld_full, kb * kBlk + 64 * b, z * p.L + j * kBlk);
                        tma_load_2d(sO + b * kBox, &tm_o, ld_full, zh * kDh + 64 * b, qrow);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------------------ MMA
            constexpr uint32_t id_kk = make_idesc_bf16(kBlk, kDh, false, false);
            constexpr uint32_t id_mm = make_idesc_bf16(kBlk, kDh, true, true);
            constexpr uint32_t id_km = make_idesc_bf16(kBlk, kDh, false, true);
            const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aDO = smem_u32(sDO), aQ = smem_u32(sQ),
                           aP = smem_u32(sP);
            // K-major operand: k-step kk (16 columns) sits in box kk/4 at +32 B per step; MN-major
            // operand: k-step kk is rows 16kk.. (+2048 B), the two 64-wide MN chunks one box apart
            auto kmaj = [](uint32_t base, int kk) { return make_sdesc(base + (kk >> 2) * kBox + (kk & 3) * 32, 16, 1024); };
            auto mnmaj = [](uint32_t base, int kk) { return make_sdesc(base + kk * 2048, kBox, 1024); };
            int n = 0;
            for (int ti = 0; ti < nk; ++ti) {
                const int kb = kbs[ti];
                mbar_wait(kv_full, ti & 1);
                if (ti > 0) TRL(92);
                if (ti > 0) mbar_wait(acc_free, (ti - 1) & 1);  // the previous key block's dK, dV were read out
                if (ti > 0) TRL(93);
                tc_fence_after();
                for (int j = p.causal ? kb : 0, jj = 0; j < nqb; ++j, ++jj, ++n) {
                    mbar_wait(ld_full, n & 1);
                    TRL(8 + 9 * n + 5);
                    tc_fence_after();
                    for (int kk = 0; kk < kDh / 16; ++kk)  // dP = dO_j V_i^T (K = d_head)
                        mma_bf16(tmem + kColDP, kmaj(aDO, kk), kmaj(aV, kk), id_kk, kk != 0 ? 1u : 0u);
                    for (int kk = 0; kk < kBlk / 16; ++kk)  // dV += P_j^T dO_j (K = queries)
                        mma_bf16(tmem + kColDV, mnmaj(aP, kk), mnmaj(aDO, kk), id_mm, (jj | kk) != 0 ? 1u : 0u);
                    mma_commit(mma12);
                    if (p.dbg & 4) {
                        mbar_wait(mma12, n & 1);
                        TRL(8 + 9 * n + 7);
                    }
                    mbar_wait(ds_ready, n & 1);
                    tc_fence_after();
                    for (int kk = 0; kk < kBlk / 16; ++kk)  // dK += dS_j^T Q_j (K = queries)
                        mma_bf16(tmem + kColDK, mnmaj(aP, kk), mnmaj(aQ, kk), id_mm, (jj | kk) != 0 ? 1u : 0u);
                    if (n > 0) {
                        mbar_wait(dq_free, (n - 1) & 1);
                        tc_fence_after();
                    }
                    for (int kk = 0; kk < kBlk / 16; ++kk)  // dQ_j = dS_j K_i (K = keys)
                        mma_bf16(tmem + kColDQ, kmaj(aP, kk), mnmaj(aK, kk), id_km, kk != 0 ? 1u : 0u);
                    mma_commit(mma34);
                    mma_commit(ld_free);
                    if (p.dbg & 4) {
                        mbar_wait(mma34, n & 1);
                        TRL(8 + 9 * n + 8);
                    }
                }
                mma_commit(acc_full);
                mma_commit(kv_free);
            }
        }
    } else if (warp == 2 || warp == 3) {
        // ------------------------------------------------ converter: dQ_j fp32 -> bf16 (+ re-zero)
        // for the query blocks this CTA completed last; coalesced, warp w rows 64(w-2).., lane l
        // columns 4l..4l+3
        int n = 0;
        for (int ti = 0; ti < nk; ++ti)
            for (int j = p.causal ? kbs[ti] : 0; j < nqb; ++j, ++n) {
                while (*conv_posted <= n) __nanosleep(64);
                __threadfence_block();
                if (!conv_flag[n] || (p.dbg & 2)) continue;
                const size_t row0 = static_cast<size_t>(zb) * p.L + j * kBlk + 64 * (warp - 2);
                float* a0 = p.dq_acc + row0 * p.ld_acc + zh * kDh + 4 * lane;
                __nv_bfloat16* o0 = p.dqkv + row0 * p.ld_dqkv + p.dq_col0 + zh * kDh + 4 * lane;
#pragma unroll 1
                for (int hh = 0; hh < 4; ++hh) {
                    float4 x[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        x[i] = __ldcg(reinterpret_cast<const float4*>(a0 + static_cast<size_t>(16 * hh + i) * p.ld_acc));
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const size_t rr = 16 * hh + i;
                        *reinterpret_cast<uint2*>(o0 + rr * p.ld_dqkv) = make_uint2(pack2(x[i].x, x[i].y), pack2(x[i].z, x[i].w));
                        __stcg(reinterpret_cast<float4*>(a0 + rr * p.ld_acc), make_float4(0.f, 0.f, 0.f, 0.f));
                    }
                }
                asm volatile("bar.sync 2, 64;" ::: "memory");
                if (warp == 2 && lane == 0) p.counters[z * nqb + j] = 0;
            }
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ dS rows: one query row per thread
        const int r = (warp - 4) * 32 + lane;
        const uint32_t trow = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        int n = 0;
        for (int ti = 0; ti < nk; ++ti) {
            const int kb = kbs[ti];
            for (int j = p.causal ? kb : 0; j < nqb; ++j, ++n) {
                // D = dO_j[r] . O_j[r] (both rows from shared memory) while the MMAs run
                mbar_wait(ld_full, n & 1);
                float D = 0.f;
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const uint32_t ra = smem_u32(sDO + b * kBox) + r * 128, rb = smem_u32(sO + b * kBox) + r * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        uint32_t a[4], o[4];
                        const uint32_t off = (c ^ (r & 7)) << 4;
                        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                                     : "r"(ra + off));
                        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3])
                                     : "r"(rb + off));
#pragma unroll
                        for (int k = 0; k < 4; ++k) D += lo(a[k]) * lo(o[k]) + hi(a[k]) * hi(o[k]);
                    }
                }
                // dS_j row r = scale * P * (dP - D) over P in place
                mbar_wait(mma12, n & 1);
                TR(8 + 9 * n + 0);
                tc_fence_after();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t ra[32], rb[32];
                    tmem_ld_32x32b_x32(trow + kColDP + 64 * h, ra);
                    tmem_ld_32x32b_x32(trow + kColDP + 64 * h + 32, rb);
                    tmem_ld_wait();
                    const uint32_t prow = smem_u32(sP + h * kBox) + r * 128;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t addr = prow + ((k ^ (r & 7)) << 4);
                        uint32_t w0, w1, w2, w3;
                        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                                     : "r"(addr));
                        const uint32_t w[4] = {w0, w1, w2, w3};
                        float o[8];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int c = k * 8 + 2 * e;
                            const float d0 = __uint_as_float(c < 32 ? ra[c] : rb[c - 32]);
                            const float d1 = __uint_as_float(c + 1 < 32 ? ra[c + 1] : rb[c - 31]);
                            o[2 * e] = p.scale * lo(w[e]) * (d0 - D);
                            o[2 * e + 1] = p.scale * hi(w[e]) * (d1 - D);
                        }
                        st_shared_v4(addr, pack2(o[0], o[1]), pack2(o[2], o[3]), pack2(o[4], o[5]),
                                     pack2(o[6], o[7]));
                    }
                }
                fence_async_smem();  // dS (generic-proxy writes) -> the MMA's operand reads
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(ds_ready);
                TR(8 + 9 * n + 1);
            }
            // dK rows of key block kb
            mbar_wait(acc_full, ti & 1);
            TR(2 + 2 * ti);
            tc_fence_after();
            const size_t krow = static_cast<size_t>(zb) * p.L + kb * kBlk + r;
            tmem_row_to_bf16(trow + kColDK, p.dqkv + krow * p.ld_dqkv + p.dk_col0 + zh * kDh);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free);
            TR(3 + 2 * ti);
        }
    } else if (warp >= 8) {
        // ------------------------------------------------ dQ rows (off the dS critical path)
        const int r = (warp - 8) * 32 + lane;
        const uint32_t trow = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        int n = 0;
        for (int ti = 0; ti < nk; ++ti) {
            const int kb = kbs[ti];
            for (int j = p.causal ? kb : 0; j < nqb; ++j, ++n) {
                mbar_wait(mma34, n & 1);
                TR(8 + 9 * n + 2);
                tc_fence_after();
                uint32_t v[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(trow + kColDQ + 32 * c, v[c]);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(dq_free);  // the next dQ MMA may overwrite TMEM now
                // dQ_j -> the fp32 accumulator by TMA reduce-add, 32 columns at a time through two
                // SWIZZLE_128B staging buffers (16-B piece k of row r at k ^ (r & 7))
                if (!(p.dbg & 1)) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint8_t* stg = sStg + (c & 1) * kStg;
                        if (c >= 2) {
                            if (r == 0) bulk_wait_read<1>();  // the reduce issued from this buffer has read it
                            dq_bar();
                        } else if (c == 0 && n > 0) {
                            dq_bar();  // row 0 has waited for the previous block's reduces (bulk wait below)
                        }
                        const uint32_t row = smem_u32(stg) + r * 128;
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            st_shared_v4(row + ((k ^ (r & 7)) << 4), v[c][4 * k], v[c][4 * k + 1], v[c][4 * k + 2],
                                         v[c][4 * k + 3]);
                        fence_async_smem();
                        dq_bar();
                        if (r == 0) {
                            tma_reduce_add_2d(&tm_acc, stg, zh * kDh + 32 * c, zb * p.L + j * kBlk);
                            bulk_commit();
                        }
                    }
                }
                TR(8 + 9 * n + 3);
                // the last key block to add to query block j converts dQ_j to bf16 and re-zeroes it:
                // the reduces complete (bulk wait), one gpu-scope fence, the arrival
                int* cnt = p.counters + z * nqb + j;
                if (r == 0) {
                    bulk_wait_all();
                    const int need = p.causal ? j + 1 : nqb;
                    __threadfence();
                    const int last = atomicAdd(cnt, 1) == need - 1;
                    if (last) __threadfence();
                    *last_flag = last;
                }
                TR(8 + 9 * n + 4);
                if (r == 0) {
                    conv_flag[n] = *last_flag;
                    __threadfence_block();
                    *conv_posted = n + 1;
                }
            }
            // dV rows of key block kb
            mbar_wait(acc_full, ti & 1);
            tc_fence_after();
            const size_t krow = static_cast<size_t>(zb) * p.L + kb * kBlk + r;
            tmem_row_to_bf16(trow + kColDV, p.dqkv + krow * p.ld_dqkv + p.dv_col0 + zh * kDh);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free);
        }
    }
    TR0(6);
    tc_fence_before();
    __syncthreads();
    TR0(7);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// fp32 [rows x cols] (row stride cols), 32 x 128 boxes, SWIZZLE_128B; cached per (ptr, rows, cols)
int map_f32(CUtensorMap* m, const void* ptr, long long rows, long long cols) {
    struct Key {
        const void* p;
        long long r, c;
    };
    thread_local std::vector<std::pair<Key, CUtensorMap>> cache;
    for (const auto& [k, v] : cache)
        if (k.p == ptr && k.r == rows && k.c == cols) {
            *m = v;
            return SWARM_OK;
        }
    auto enc = swarm::attn::encoder();
    if (!enc) return SWARM_E_CUDA;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
    const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(kBlk)};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return SWARM_E_INVALID;
    if (cache.size() > 64) cache.clear();
    cache.push_back({Key{ptr, rows, cols}, *m});
    return SWARM_OK;
}

int launch(const Params& p, const void* qkv, int ld_qkv, int qkv_cols, const void* dO, int ld_do, const void* P,
           cudaStream_t st) {
    // (O's tensor map is built from p.o / p.ld_o)
    using swarm::attn::map_bf16;
    const long long T = static_cast<long long>(p.B) * p.L, rows_p = static_cast<long long>(p.B) * p.H * p.L;
    CUtensorMap tq, td, tp, to, ta;
    if (map_bf16(&tq, qkv, T, qkv_cols, ld_qkv, 64, kBlk, CU_TENSOR_MAP_SWIZZLE_128B) ||
        map_bf16(&td, dO, T, static_cast<long long>(p.H) * kDh, ld_do, 64, kBlk, CU_TENSOR_MAP_SWIZZLE_128B) ||
        map_bf16(&tp, P, rows_p, p.L, p.L, 64, kBlk, CU_TENSOR_MAP_SWIZZLE_128B) ||
        map_bf16(&to, p.o, T, static_cast<long long>(p.H) * kDh, p.ld_o, 64, kBlk, CU_TENSOR_MAP_SWIZZLE_128B))
        return invalid("attention backward: tensor map encoding failed");
    if (map_f32(&ta, p.dq_acc, T, p.ld_acc))
        return invalid("attention backward: tensor map encoding failed (dQ accumulator)");
    static bool attr = false;
    if (!attr) {
        SWARM_CUDA_TRY(cudaFuncSetAttribute(k_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        attr = true;
    }
    const int nkb = p.L / kBlk;
    const int per_z = p.causal ? (nkb + 1) / 2 : nkb;
    k_attn_bwd<<<p.B * p.H * per_z, kThreads, kSmem, st>>>(tq, td, tp, to, ta, p);
    SWARM_LAUNCH_CHECK("k_attn_bwd");
    return SWARM_OK;
}

bool al16(const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; }

}  // namespace attn_bwd
}  // namespace swarm

extern "C" {

// experiments only (not in the public header): the last traced launch's per-CTA timeline
int swarm_debug_abwd_trace(uint64_t* host, int n_ctas) {
    if (n_ctas > 256) n_ctas = 256;
    return cudaMemcpyFromSymbol(host, swarm::attn_bwd::g_abwd_trace, sizeof(uint64_t) * swarm::attn_bwd::kTr * n_ctas) ==
                   cudaSuccess
               ? SWARM_OK
               : SWARM_E_CUDA;
}

size_t swarm_attn_backward_workspace(int B, int H, int L, int d_head) {
    if (B <= 0 || H <= 0 || L <= 0 || d_head <= 0) return 0;
    const size_t acc = static_cast<size_t>(B) * L * H * d_head * sizeof(float);
    const size_t cnt = static_cast<size_t>(B) * H * ((L + 127) / 128) * sizeof(int);
    return acc + ((cnt + 255) / 256) * 256;
}

int swarm_attn_backward(const void* dO, int ld_do, const void* qkv, int ld_qkv, int qkv_cols, int k_col0, int v_col0,
                        const void* O, int ld_o, const void* P, int B, int H, int L, int d_head, float scale,
                        int causal, void* dqkv, int ld_dqkv, int dk_col0, int dv_col0, void* workspace,
                        swarm_stream_t stream) {
    using namespace swarm::attn_bwd;
    if (d_head != kDh || L % kBlk || L <= 0 || B <= 0 || H <= 0)
        return swarm::invalid("attention backward: need d_head 128 and L % 128 == 0");
    if (!dO || !qkv || !O || !P || !dqkv || !workspace)
        return swarm::invalid("attention backward: null operand or workspace");
    if (!al16(dO) || !al16(qkv) || !al16(O) || !al16(P) || !al16(dqkv) || !al16(workspace) || ld_do % 8 ||
        ld_qkv % 8 || ld_o % 8 || ld_dqkv % 8 || k_col0 % 8 || v_col0 % 8 || dk_col0 % 8 || dv_col0 % 8)
        return swarm::invalid("attention backward: operands must be 16-byte aligned bf16 rows");
    if (qkv_cols < v_col0 + H * kDh || qkv_cols < k_col0 + H * kDh || ld_qkv < qkv_cols || ld_do < H * kDh ||
        ld_o < H * kDh || ld_dqkv < dv_col0 + H * kDh || ld_dqkv < dk_col0 + H * kDh)
        return swarm::invalid("attention backward: row strides too small for H heads");
    Params p{};
    p.B = B;
    p.H = H;
    p.L = L;
    p.causal = causal ? 1 : 0;
    p.scale = scale;
    p.q_col0 = 0;
    p.k_col0 = k_col0;
    p.v_col0 = v_col0;
    p.o = static_cast<const __nv_bfloat16*>(O);
    p.ld_o = ld_o;
    p.dq_acc = static_cast<float*>(workspace);
    p.ld_acc = H * kDh;
    p.counters = reinterpret_cast<int*>(static_cast<char*>(workspace) +
                                        static_cast<size_t>(B) * L * H * kDh * sizeof(float));
    p.dqkv = static_cast<__nv_bfloat16*>(dqkv);
    p.ld_dqkv = ld_dqkv;
    p.dq_col0 = 0;
    p.dk_col0 = dk_col0;
    p.dv_col0 = dv_col0;
    static const int dbg = [] {
        const char* e = getenv("SWARM_ATTN_BWD_DBG");
        return e ? atoi(e) : 0;
    }();
    p.dbg = dbg;
    return launch(p, qkv, ld_qkv, qkv_cols, dO, ld_do, P, swarm::as_stream(stream));
}

}  // extern "C"
