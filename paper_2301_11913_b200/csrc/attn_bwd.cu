// Fused attention backward (sm_100a, tcgen05 + TMEM + TMA), d_head 128:
//
//   dP = dO V^T,  dS = scale * P * (dP - D),  dV = P^T dO,  dK = dS^T Q,  dQ = dS K
//
// for z = b*H + h, with P the forward's bf16 probabilities and D = rowsum(dO * O) (=
// rowsum(P * dP)).  It replaces the score-gradient kernel + three batched GEMMs of the
// unfused backward: dP and dS never leave the SM.  Three launches:
//   k_attn_rowdot  D per (z, query)                          (reads dO, O once: 16 MB at configs[2])
//   k_attn_bwd     dK, dV (bf16, into dqkv) and dQ partials  (TMA reduce-add into an fp32 accumulator)
//   k_attn_dq_out  the accumulator -> bf16 dQ into dqkv, and back to zero
//
// k_attn_bwd: one CTA owns key blocks of 128 keys of one (b, h) and streams the query
// blocks that see them (causal: query blocks >= the key block).  Per query block j:
//   TMA    dO_j, Q_j, P_j ([128 x 128] bf16 tiles as two SWIZZLE_128B 64-column boxes; P
//          double-buffered, dO reloaded as soon as its MMAs are issued, Q after dK's)
//   MMA    dP = dO_j V_i^T        (TMEM columns   0-127, M = queries)
//          dV += P_j^T dO_j       (TMEM columns 384-511, M = keys; P_j read MN-major)
//   rows   dS_j = scale * P_j * (dP - D_j) over P_j in shared memory (warps 4-7, one query
//          row per thread)
//   MMA    dK += dS_j^T Q_j       (TMEM columns 256-383; dS read MN-major)
//          dQ_j = dS_j K_i        (TMEM columns 128-255; dS read K-major)
//   rows   dQ_j -> shared staging -> TMA reduce-add (warps 8-11, off the dS critical path)
// and per key block dK, dV: TMEM -> bf16 over K_i / V_i in shared memory -> TMA stores.
// One shared-memory tile serves as K-major and MN-major operand: SWIZZLE_128B atoms are
// 8 rows x 128 B either way; only the descriptor's reading of them differs.
//
// Causal work is paired: a CTA takes key blocks t and nkb-1-t, so every CTA streams nkb + 1
// query blocks (configs[2]: L 512 -> 2 CTAs per (b, h), 128 CTAs, one wave).  Everything a
// CTA reads after its first block is prefetched to L2 at entry.  TMEM: all 512 columns
// (one CTA per SM).  Warps: 0 TMA, 1 MMA issuer, 2 TMEM allocator, 4-7 dS rows, 8-11 dQ rows.
//
// dQ's fp32 sum over key blocks uses reduce-add, so its order (<= L/128 terms) is not
// fixed; SWARM_ATTN_BWD_FUSED=0 selects the unfused, order-deterministic path
// (csrc/attention.cu + batched GEMMs).  Parity: tests/test_attention_gpu.py (torch fp32 of
// the same op; the unfused kernels) and the stage tests against the fp64 oracle.
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
constexpr int kBars = 20;  // (+ the TMEM slot after them)
constexpr int kStg = kBlk * 128;  // dQ staging: [128 rows x 32] fp32, SWIZZLE_128B (16 KB)
constexpr int kSmem = 6 * kTile + 2 * kStg + kBars * 8 + 16 + 1024;
constexpr uint32_t kColDP = 0, kColDQ = 128, kColDK = 256, kColDV = 384;
static_assert(kSmem <= 232448, "attention backward: shared memory");

struct Params {
    int B, H, L, causal;
    float scale;
    int q_col0, k_col0, v_col0;  // head-0 columns of Q, K, V in the qkv storage
    const float* D;              // rowsum(dO * O) per (z, query) [B*H*L] (k_attn_rowdot)
    const float* lse;            // RECOMP: the forward's log2-sum-exp per (z, query) [B*H*L]
    float* dq_acc;               // fp32 dQ accumulator [B*L, ld_acc] (zero on entry, left zero)
    int ld_acc;
    __nv_bfloat16* dqkv;
    int ld_dqkv, dq_col0, dk_col0, dv_col0;
    int dbg;  // experiments (SWARM_ATTN_BWD_DBG): 1 skips the dQ reductions, 2 the dQ write-out, 4 traces
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&p);
}
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* m, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void dq_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

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

// per-CTA timeline for experiments (SWARM_ATTN_BWD_DBG & 4): globaltimer at fixed points
constexpr int kTr = 96;
__device__ unsigned long long g_abwd_trace[256][kTr];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TR(cond, i)                                                                                              \
    do {                                                                                                         \
        if ((p.dbg & 4) && (cond) && blockIdx.x < 256 && (i) < kTr) g_abwd_trace[blockIdx.x][(i)] = gtime();    \
    } while (0)

// D[z*L + q] = dO[b*L + q, h*128 ..] . O[b*L + q, h*128 ..]: 16 threads per (row, head)
__global__ void __launch_bounds__(256) k_attn_rowdot(const __nv_bfloat16* __restrict__ dO, int ld_do,
                                                     const __nv_bfloat16* __restrict__ O, int ld_o, int B, int H,
                                                     int L, float* __restrict__ D) {
    pdl_trigger();
    pdl_wait();
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = gid >> 4, part = gid & 15;
    const int rows = B * L;
    const bool ok = item < rows * H;
    const int row = ok ? item / H : 0, h = ok ? item - (item / H) * H : 0;
    float acc = 0.f;
    if (ok) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(dO + static_cast<size_t>(row) * ld_do + h * kDh) + part);
        const uint4 o = __ldg(reinterpret_cast<const uint4*>(O + static_cast<size_t>(row) * ld_o + h * kDh) + part);
        const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wo[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) acc += lo(wa[k]) * lo(wo[k]) + hi(wa[k]) * hi(wo[k]);
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (ok && part == 0) {
        const int b = row / L, q = row - b * L;
        D[(static_cast<size_t>(b) * H + h) * L + q] = acc;
    }
}

// dQ: the fp32 accumulator -> bf16 into dqkv, and back to zero for the next launch (8 columns per thread)
__global__ void __launch_bounds__(256) k_attn_dq_out(float* __restrict__ acc, int rows, int cols,
                                                     __nv_bfloat16* __restrict__ dqkv, int ld_dqkv) {
    pdl_trigger();
    pdl_wait();
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c8 = cols / 8;
    if (i >= static_cast<long long>(rows) * c8) return;
    const long long row = i / c8, c = (i - row * c8) * 8;
    float4* a = reinterpret_cast<float4*>(acc + row * cols + c);
    const float4 x = __ldcg(a), y = __ldcg(a + 1);
    *reinterpret_cast<uint4*>(dqkv + row * ld_dqkv + c) = make_uint4(pack2(x.x, x.y), pack2(x.z, x.w), pack2(y.x, y.y), pack2(y.z, y.w));
    __stcg(a, make_float4(0.f, 0.f, 0.f, 0.f));
    __stcg(a + 1, make_float4(0.f, 0.f, 0.f, 0.f));
}

// 2^x on the SFU (ex2.approx.ftz: 2 ulp; P is rounded to bf16)
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// RECOMP = false: P_j is the forward's stored probabilities, TMA-loaded (double-buffered).
// RECOMP = true:  the forward stored only each row's log2-sum-exp (swarm_attn_forward_lse);
//                 S_j = Q_j K_i^T is recomputed into the dP columns and the dS rows write
//                 P_j = 2^(S_j * scale * log2 e - lse) into the (single) P buffer; Q is
//                 double-buffered instead, since S needs it at the start of the block.
template <bool RECOMP>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_bwd(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
               const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_acc,
               const __grid_constant__ CUtensorMap tm_out, const Params p) {
    pdl_trigger();
    TR(threadIdx.x == 128, 0);
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw & 1023)) & 1023);
    uint8_t* sK = smem;
    uint8_t* sV = sK + kTile;
    uint8_t* sDO = sV + kTile;
    uint8_t* sX = sDO + kTile;  // 3 tiles: Q + P[2], or (RECOMP) Q[2] + P
    auto sQb = [&](int n) { return RECOMP ? sX + (n & 1) * kTile : sX; };
    auto sPb = [&](int n) { return RECOMP ? sX + 2 * kTile : sX + kTile + (n & 1) * kTile; };
    uint8_t* sStg = sX + 3 * kTile;  // two dQ staging buffers
    uint64_t* bars = reinterpret_cast<uint64_t*>(sStg + 2 * kStg);
    uint64_t* kv_full = bars + 0;   // TMA: K_i, V_i landed
    uint64_t* kv_free = bars + 1;   // dS rows: dK, dV staged through sK / sV and stored (TMA read them)
    uint64_t* do_full = bars + 2;   // TMA: dO_j landed
    uint64_t* do_free = bars + 3;   // MMA: done with dO_j (dP, dV issued)
    uint64_t* q_full = bars + 4;    // [2] TMA: Q_j landed (buffer n % 2; one buffer unless RECOMP)
    uint64_t* q_free = bars + 6;    // [2] MMA: done with Q_j
    uint64_t* p_full = bars + 8;    // [2] TMA: P_j landed in buffer n % 2 (not RECOMP)
    uint64_t* p_free = bars + 10;   // [2] MMA: done with dS_j in its buffer
    uint64_t* mma12 = bars + 12;    // dP, dV updated
    uint64_t* ds_ready = bars + 13; // dS rows: dS_j written (4 warps)
    uint64_t* mma34 = bars + 14;    // dK updated, dQ_j ready
    uint64_t* dq_free = bars + 15;  // dQ rows: dQ_j read out of TMEM (4 warps)
    uint64_t* acc_full = bars + 16; // dK, dV of the key block complete
    uint64_t* acc_free = bars + 17; // dS rows: dK, dV read out (4 warps)
    uint64_t* s_full = bars + 18;   // RECOMP: S_j = Q_j K_i^T in TMEM
    uint64_t* p_ready = bars + 19;  // RECOMP: dS rows: P_j written (4 warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kBars);
    const int qbuf = RECOMP ? 2 : 1;  // Q buffers

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nz = p.B * p.H, nqb = p.L / kBlk;
    const int z = static_cast<int>(blockIdx.x) % nz, t = static_cast<int>(blockIdx.x) / nz;
    const int zb = z / p.H, zh = z - zb * p.H;
    int kbs[2] = {0, 0};
    const int nk = key_blocks(p, t, kbs);
    auto j0 = [&](int ti) { return p.causal ? kbs[ti] : 0; };

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kBars; ++i) mbar_init(bars + i, (i == 13 || i == 15 || i == 17 || i == 19) ? 4 : 1);
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
    TR(threadIdx.x == 128, 1);
    pdl_wait();

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA
            const int qcol = p.q_col0 + zh * kDh;
            auto qrow = [&](int j) { return zb * p.L + j * kBlk; };
            // everything this CTA reads after its first block, to L2 now (in order of use)
            if (nk == 2)
                for (int b = 0; b < 2; ++b) {
                    tma_prefetch_l2(&tm_qkv, p.k_col0 + zh * kDh + 64 * b, qrow(kbs[1]));
                    tma_prefetch_l2(&tm_qkv, p.v_col0 + zh * kDh + 64 * b, qrow(kbs[1]));
                }
            for (int ti = 0; ti < nk; ++ti)
                for (int j = j0(ti) + (ti == 0); j < nqb; ++j)
                    for (int b = 0; b < 2; ++b) {
                        if (!RECOMP) tma_prefetch_l2(&tm_p, kbs[ti] * kBlk + 64 * b, z * p.L + j * kBlk);
                        if (ti == 0) {
                            tma_prefetch_l2(&tm_do, zh * kDh + 64 * b, qrow(j));
                            tma_prefetch_l2(&tm_qkv, qcol + 64 * b, qrow(j));
                        }
                    }
            int n = 0;
            for (int ti = 0; ti < nk; ++ti) {
                const int kb = kbs[ti];
                if (ti > 0) mbar_wait(kv_free, (ti - 1) & 1);
                mbar_arrive_expect_tx(kv_full, 2 * kTile);
                for (int b = 0; b < 2; ++b) {
                    tma_load_2d(sK + b * kBox, &tm_qkv, kv_full, p.k_col0 + zh * kDh + 64 * b, qrow(kb));
                    tma_load_2d(sV + b * kBox, &tm_qkv, kv_full, p.v_col0 + zh * kDh + 64 * b, qrow(kb));
                }
                for (int j = j0(ti); j < nqb; ++j, ++n) {
                    // RECOMP: Q_j first (the score MMA needs it at the block's start), into the
                    // buffer block n-2 used; dO_j once dP, dV of the previous block are issued.
                    // Else: dO_j, then P_j into the buffer block n-2 used, then Q_j once the
                    // previous dK is issued (needed only after this block's dS)
                    const int qb = RECOMP ? (n & 1) : 0;
                    auto load_q = [&]() {
                        if (RECOMP ? n > 1 : n > 0)
                            mbar_wait(&q_free[qb], RECOMP ? (((n >> 1) - 1) & 1) : ((n - 1) & 1));
                        mbar_arrive_expect_tx(&q_full[qb], kTile);
                        for (int b = 0; b < 2; ++b)
                            tma_load_2d(sQb(n) + b * kBox, &tm_qkv, &q_full[qb], qcol + 64 * b, qrow(j));
                    };
                    if (RECOMP) load_q();
                    if (n > 0) mbar_wait(do_free, (n - 1) & 1);
                    mbar_arrive_expect_tx(do_full, kTile);
                    for (int b = 0; b < 2; ++b) tma_load_2d(sDO + b * kBox, &tm_do, do_full, zh * kDh + 64 * b, qrow(j));
                    if (!RECOMP) {
                        const int pb = n & 1;
                        if (n > 1) mbar_wait(&p_free[pb], ((n >> 1) - 1) & 1);
                        mbar_arrive_expect_tx(&p_full[pb], kTile);
                        for (int b = 0; b < 2; ++b)
                            tma_load_2d(sPb(n) + b * kBox, &tm_p, &p_full[pb], kb * kBlk + 64 * b, z * p.L + j * kBlk);
                        load_q();
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
            const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aDO = smem_u32(sDO);
            // K-major operand: k-step kk (16 columns) sits in box kk/4 at +32 B per step; MN-major
            // operand: k-step kk is rows 16kk.. (+2048 B), the two 64-wide MN chunks one box apart
            auto kmaj = [](uint32_t base, int kk) { return make_sdesc(base + (kk >> 2) * kBox + (kk & 3) * 32, 16, 1024); };
            auto mnmaj = [](uint32_t base, int kk) { return make_sdesc(base + kk * 2048, kBox, 1024); };
            // RECOMP: block n's S, dP and dQ share TMEM region rg(n) (columns 0 or 128, alternating), so
            // the next block's S = Q K^T can be issued into the other region right after this block's
            // dP / dV -- while the rows compute dS -- and the rows' next exponentials overlap dK / dQ
            auto rg = [&](int m) -> uint32_t { return RECOMP ? ((m & 1) ? kColDQ : kColDP) : kColDP; };
            auto rq = [&](int m) -> uint32_t { return RECOMP ? rg(m) : kColDQ; };
            auto issue_s = [&](int m, uint32_t aQm) {  // S_m = Q_m K_i^T (K = d_head)
                mbar_wait(&q_full[m & 1], (m >> 1) & 1);
                tc_fence_after();
                for (int kk = 0; kk < kDh / 16; ++kk)
                    mma_bf16(tmem + rg(m), kmaj(aQm, kk), kmaj(aK, kk), id_kk, kk != 0 ? 1u : 0u);
                mma_commit(s_full);
            };
            int n = 0;
            for (int ti = 0; ti < nk; ++ti) {
                mbar_wait(kv_full, ti & 1);
                if (ti > 0) mbar_wait(acc_free, (ti - 1) & 1);  // the previous key block's dK, dV were read out
                tc_fence_after();
                const int jn = nqb - j0(ti);  // blocks of this key block
                for (int j = j0(ti), jj = 0; j < nqb; ++j, ++jj, ++n) {
                    const int qb = RECOMP ? (n & 1) : 0, pb = RECOMP ? 0 : (n & 1);
                    const uint32_t aP = smem_u32(sPb(n)), aQ = smem_u32(sQb(n));
                    const uint32_t q_par = RECOMP ? ((n >> 1) & 1) : (n & 1);
                    if constexpr (RECOMP) {
                        // (the first block of a key block: S was not issued ahead -- K changed; its region
                        // last held dQ_{n-2}, whose read-out was awaited before dQ_{n-1}'s MMA)
                        if (jj == 0) issue_s(n, aQ);
                        mbar_wait(p_ready, n & 1);  // P_j written (and S_j read) by the rows
                        TR(true, 8 + 9 * n + 7);
                    } else {
                        mbar_wait(&p_full[pb], (n >> 1) & 1);
                    }
                    mbar_wait(do_full, n & 1);
                    tc_fence_after();
                    for (int kk = 0; kk < kDh / 16; ++kk)  // dP = dO_j V_i^T (K = d_head), over S_j
                        mma_bf16(tmem + rg(n), kmaj(aDO, kk), kmaj(aV, kk), id_kk, kk != 0 ? 1u : 0u);
                    for (int kk = 0; kk < kBlk / 16; ++kk)  // dV += P_j^T dO_j (K = queries)
                        mma_bf16(tmem + kColDV, mnmaj(aP, kk), mnmaj(aDO, kk), id_mm, (jj | kk) != 0 ? 1u : 0u);
                    mma_commit(mma12);
                    mma_commit(do_free);
                    // dQ_{n-1} read out of its region (also the region S_{n+1} goes to): observed before
                    // every dQ MMA, so the dQ rows are never two phases ahead of this wait
                    if (n > 0) {
                        mbar_wait(dq_free, (n - 1) & 1);
                        tc_fence_after();
                    }
                    if (RECOMP && jj + 1 < jn) issue_s(n + 1, smem_u32(sQb(n + 1)));
                    mbar_wait(ds_ready, n & 1);
                    if (!RECOMP) mbar_wait(&q_full[0], q_par);
                    tc_fence_after();
                    for (int kk = 0; kk < kBlk / 16; ++kk)  // dK += dS_j^T Q_j (K = queries)
                        mma_bf16(tmem + kColDK, mnmaj(aP, kk), mnmaj(aQ, kk), id_mm, (jj | kk) != 0 ? 1u : 0u);
                    mma_commit(&q_free[qb]);
                    for (int kk = 0; kk < kBlk / 16; ++kk)  // dQ_j = dS_j K_i (K = keys), over dP_j (RECOMP)
                        mma_bf16(tmem + rq(n), kmaj(aP, kk), mnmaj(aK, kk), id_km, kk != 0 ? 1u : 0u);
                    mma_commit(mma34);
                    mma_commit(&p_free[pb]);
                    TR(true, 8 + 9 * n + 5);
                }
                mma_commit(acc_full);  // (every MMA reading K_i, V_i is complete too)
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ dS rows: one query row per thread
        const int r = (warp - 4) * 32 + lane;
        const uint32_t trow = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        const float cs = p.scale * 1.4426950408889634f;
        int n = 0;
        for (int ti = 0; ti < nk; ++ti) {
            const int kb = kbs[ti];
            for (int j = j0(ti); j < nqb; ++j, ++n) {
                const int pb = RECOMP ? 0 : (n & 1);
                uint8_t* sPn = sPb(n);
                const size_t qz = static_cast<size_t>(z) * p.L + j * kBlk + r;
                const float D = __ldg(p.D + qz);
                if constexpr (RECOMP) {
                    // P_j row r = 2^(S * cs - lse), keys past the query masked (causal diagonal block); the
                    // exponentials are taken while dK / dQ of the previous block may still read its dS
                    // out of the P buffer, and written once that buffer is free
                    const float lse = __ldg(p.lse + qz);
                    const int valid = (p.causal && kb == j) ? r + 1 : kBlk;  // columns < valid are unmasked
                    const uint32_t rgn = (n & 1) ? kColDQ : kColDP;
                    mbar_wait(s_full, n & 1);
                    TR(r == 0, 8 + 9 * n + 6);
                    tc_fence_after();
                    uint32_t pk[64];  // P_j row, packed bf16 pairs
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t ra[32], rb[32];
                        tmem_ld_32x32b_x32(trow + rgn + 64 * h, ra);
                        tmem_ld_32x32b_x32(trow + rgn + 64 * h + 32, rb);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const int c = 2 * e;  // column inside the half
                            const float s0 = __uint_as_float(c < 32 ? ra[c] : rb[c - 32]);
                            const float s1 = __uint_as_float(c + 1 < 32 ? ra[c + 1] : rb[c - 31]);
                            const float p0 = (64 * h + c < valid) ? fast_exp2(fmaf(s0, cs, -lse)) : 0.f;
                            const float p1 = (64 * h + c + 1 < valid) ? fast_exp2(fmaf(s1, cs, -lse)) : 0.f;
                            pk[32 * h + e] = pack2(p0, p1);
                        }
                    }
                    tc_fence_before();
                    if (n > 0) mbar_wait(&p_free[0], (n - 1) & 1);  // dS_{j-1} consumed by dK, dQ
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t prow = smem_u32(sPn + h * kBox) + r * 128;
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            st_shared_v4(prow + ((k ^ (r & 7)) << 4), pk[32 * h + 4 * k], pk[32 * h + 4 * k + 1],
                                         pk[32 * h + 4 * k + 2], pk[32 * h + 4 * k + 3]);
                    }
                    fence_async_smem();  // P (generic-proxy writes) -> the dV MMA's operand reads
                    __syncwarp();
                    if (lane == 0) mbar_arrive(p_ready);
                    TR(r == 0, 8 + 9 * n + 4);
                } else {
                    mbar_wait(&p_full[pb], (n >> 1) & 1);  // (TMA writes visible to these threads)
                }
                mbar_wait(mma12, n & 1);
                TR(r == 0, 8 + 9 * n + 0);
                tc_fence_after();
                // dS_j row r = scale * P * (dP - D) over P in place
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t ra[32], rb[32];
                    const uint32_t rgd = (RECOMP && (n & 1)) ? kColDQ : kColDP;
                    tmem_ld_32x32b_x32(trow + rgd + 64 * h, ra);
                    tmem_ld_32x32b_x32(trow + rgd + 64 * h + 32, rb);
                    tmem_ld_wait();
                    const uint32_t prow = smem_u32(sPn + h * kBox) + r * 128;
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
                TR(r == 0, 8 + 9 * n + 1);
            }
            // dK, dV of key block kb: TMEM -> bf16 rows over K_i / V_i in shared memory (the key
            // block's MMAs are complete) -> TMA stores; then the next K, V may load there
            mbar_wait(acc_full, ti & 1);
            TR(r == 0, 2 + 2 * ti);
            tc_fence_after();
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                uint32_t v[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(trow + (g ? kColDV : kColDK) + 32 * c, v[c]);
                tmem_ld_wait();
                uint8_t* dst = g ? sV : sK;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const int k16 = 4 * c + w;  // 16-B piece of the 256-B row: box k16 / 8, piece k16 % 8
                        const uint32_t addr = smem_u32(dst + (k16 >> 3) * kBox) + r * 128 + (((k16 & 7) ^ (r & 7)) << 4);
                        st_shared_v4(addr, pack2(__uint_as_float(v[c][8 * w]), __uint_as_float(v[c][8 * w + 1])),
                                     pack2(__uint_as_float(v[c][8 * w + 2]), __uint_as_float(v[c][8 * w + 3])),
                                     pack2(__uint_as_float(v[c][8 * w + 4]), __uint_as_float(v[c][8 * w + 5])),
                                     pack2(__uint_as_float(v[c][8 * w + 6]), __uint_as_float(v[c][8 * w + 7])));
                    }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free);
            fence_async_smem();
            asm volatile("bar.sync 3, 128;" ::: "memory");
            if (r == 0) {
                const int krow = zb * p.L + kb * kBlk;
                for (int b = 0; b < 2; ++b) {
                    tma_store_2d(&tm_out, sK + b * kBox, p.dk_col0 + zh * kDh + 64 * b, krow);
                    tma_store_2d(&tm_out, sV + b * kBox, p.dv_col0 + zh * kDh + 64 * b, krow);
                }
                bulk_commit();
                bulk_wait_read<0>();
                mbar_arrive(kv_free);
                if (ti == nk - 1) bulk_wait_all();
            }
            TR(r == 0, 3 + 2 * ti);
        }
    } else if (warp >= 8) {
        // ------------------------------------------------ dQ rows (off the dS critical path)
        const int r = (warp - 8) * 32 + lane;
        const uint32_t trow = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        int n = 0;
        for (int ti = 0; ti < nk; ++ti)
            for (int j = j0(ti); j < nqb; ++j, ++n) {
                mbar_wait(mma34, n & 1);
                TR(r == 0, 8 + 9 * n + 2);
                tc_fence_after();
                uint32_t v[4][32];
#pragma unroll
                const uint32_t rgq = (RECOMP && !(n & 1)) ? kColDP : kColDQ;  // RECOMP: dQ_j sits in block j's region
                for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(trow + rgq + 32 * c, v[c]);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(dq_free);  // the region may be overwritten now
                // dQ_j -> the fp32 accumulator by TMA reduce-add, 32 columns at a time through two
                // SWIZZLE_128B staging buffers (16-B piece k of row r at k ^ (r & 7))
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint8_t* stg = sStg + (c & 1) * kStg;
                    if (n > 0 || c >= 2) {
                        if (r == 0) bulk_wait_read<1>();  // the reduce issued from this buffer has read it
                        dq_bar();
                    }
                    const uint32_t row = smem_u32(stg) + r * 128;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        st_shared_v4(row + ((k ^ (r & 7)) << 4), v[c][4 * k], v[c][4 * k + 1], v[c][4 * k + 2],
                                     v[c][4 * k + 3]);
                    fence_async_smem();
                    dq_bar();
                    if (r == 0) {
                        if (!(p.dbg & 1)) tma_reduce_add_2d(&tm_acc, stg, zh * kDh + 32 * c, zb * p.L + j * kBlk);
                        bulk_commit();
                    }
                }
                TR(r == 0, 8 + 9 * n + 3);
            }
        if (r == 0) bulk_wait_all();  // the reduces complete before the CTA retires
    }
    TR(threadIdx.x == 128, 6);
    tc_fence_before();
    __syncthreads();
    TR(threadIdx.x == 128, 7);
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

int launch(const Params& p, const void* qkv, int ld_qkv, int qkv_cols, const void* dO, int ld_do, const void* O,
           int ld_o, const void* P, cudaStream_t st) {
    using swarm::attn::map_bf16;
    const long long T = static_cast<long long>(p.B) * p.L, rows_p = static_cast<long long>(p.B) * p.H * p.L;
    CUtensorMap tq, td, tp, ta, tout;
    if (map_bf16(&tq, qkv, T, qkv_cols, ld_qkv, 64, kBlk, CU_TENSOR_MAP_SWIZZLE_128B) ||
        map_bf16(&td, dO, T, static_cast<long long>(p.H) * kDh, ld_do, 64, kBlk, CU_TENSOR_MAP_SWIZZLE_128B) ||
        (P ? map_bf16(&tp, P, rows_p, p.L, p.L, 64, kBlk, CU_TENSOR_MAP_SWIZZLE_128B) : 0) ||
        map_bf16(&tout, p.dqkv, T, p.ld_dqkv, p.ld_dqkv, 64, kBlk, CU_TENSOR_MAP_SWIZZLE_128B))
        return invalid("attention backward: tensor map encoding failed");
    if (map_f32(&ta, p.dq_acc, T, p.ld_acc))
        return invalid("attention backward: tensor map encoding failed (dQ accumulator)");
    if (!P) tp = td;  // (unused: P is recomputed from the log2-sum-exp)
    static bool attr = false;
    if (!attr) {
        SWARM_CUDA_TRY(cudaFuncSetAttribute(k_attn_bwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        SWARM_CUDA_TRY(cudaFuncSetAttribute(k_attn_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        attr = true;
    }
    const long long items = T * p.H * 16;
    launch_pdl(k_attn_rowdot, dim3(static_cast<unsigned>((items + 255) / 256)), dim3(256), 0, st,
               static_cast<const __nv_bfloat16*>(dO), ld_do, static_cast<const __nv_bfloat16*>(O), ld_o, p.B, p.H,
               p.L, const_cast<float*>(p.D));
    SWARM_LAUNCH_CHECK("k_attn_rowdot");
    const int nkb = p.L / kBlk;
    const int per_z = p.causal ? (nkb + 1) / 2 : nkb;
    if (p.lse) k_attn_bwd<true><<<p.B * p.H * per_z, kThreads, kSmem, st>>>(tq, td, tp, ta, tout, p);
    else k_attn_bwd<false><<<p.B * p.H * per_z, kThreads, kSmem, st>>>(tq, td, tp, ta, tout, p);
    SWARM_LAUNCH_CHECK("k_attn_bwd");
    if (!(p.dbg & 2)) {
        const long long n8 = T * p.ld_acc / 8;
        launch_pdl(k_attn_dq_out, dim3(static_cast<unsigned>((n8 + 255) / 256)), dim3(256), 0, st, p.dq_acc,
                   static_cast<int>(T), p.ld_acc, p.dqkv + p.dq_col0, p.ld_dqkv);
        SWARM_LAUNCH_CHECK("k_attn_dq_out");
    }
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
    return acc + static_cast<size_t>(B) * H * L * sizeof(float);  // + D
}

static int attn_backward(const void* dO, int ld_do, const void* qkv, int ld_qkv, int qkv_cols, int k_col0,
                         int v_col0, const void* O, int ld_o, const void* P, const float* lse, int B, int H, int L,
                         int d_head, float scale, int causal, void* dqkv, int ld_dqkv, int dk_col0, int dv_col0,
                         void* workspace, swarm_stream_t stream) {
    using namespace swarm::attn_bwd;
    if (d_head != kDh || L % kBlk || L <= 0 || B <= 0 || H <= 0)
        return swarm::invalid("attention backward: need d_head 128 and L % 128 == 0");
    if (!dO || !qkv || !O || !(P || lse) || !dqkv || !workspace)
        return swarm::invalid("attention backward: null operand or workspace");
    if (!al16(dO) || !al16(qkv) || !al16(O) || (P && !al16(P)) || !al16(dqkv) || !al16(workspace) || ld_do % 8 ||
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
    p.lse = lse;
    p.dq_acc = static_cast<float*>(workspace);
    p.ld_acc = H * kDh;
    p.D = reinterpret_cast<const float*>(static_cast<char*>(workspace) + static_cast<size_t>(B) * L * H * kDh * sizeof(float));
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
    return launch(p, qkv, ld_qkv, qkv_cols, dO, ld_do, O, ld_o, P, swarm::as_stream(stream));
}

int swarm_attn_backward(const void* dO, int ld_do, const void* qkv, int ld_qkv, int qkv_cols, int k_col0, int v_col0,
                        const void* O, int ld_o, const void* P, int B, int H, int L, int d_head, float scale,
                        int causal, void* dqkv, int ld_dqkv, int dk_col0, int dv_col0, void* workspace,
                        swarm_stream_t stream) {
    if (!P) return swarm::invalid("attention backward: null P");
    return attn_backward(dO, ld_do, qkv, ld_qkv, qkv_cols, k_col0, v_col0, O, ld_o, P, nullptr, B, H, L, d_head, scale,
                         causal, dqkv, ld_dqkv, dk_col0, dv_col0, workspace, stream);
}

int swarm_attn_backward_lse(const void* dO, int ld_do, const void* qkv, int ld_qkv, int qkv_cols, int k_col0,
                            int v_col0, const void* O, int ld_o, const float* lse, int B, int H, int L, int d_head,
                            float scale, int causal, void* dqkv, int ld_dqkv, int dk_col0, int dv_col0,
                            void* workspace, swarm_stream_t stream) {
    if (!lse) return swarm::invalid("attention backward: null lse");
    return attn_backward(dO, ld_do, qkv, ld_qkv, qkv_cols, k_col0, v_col0, O, ld_o, nullptr, lse, B, H, L, d_head,
                         scale, causal, dqkv, ld_dqkv, dk_col0, dv_col0, workspace, stream);
}

}  // extern "C"
