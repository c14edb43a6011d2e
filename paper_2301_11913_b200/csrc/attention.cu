// Fused attention-score kernels (sm_100a, tcgen05 + TMEM + TMA).
//
// Forward:  P[z, i, :] = softmax(scale * Q_z[i] K_z^T)        (causal optional)
// Backward: dS[z, i, :] = scale * P (dP - rowsum(P * dP)),  dP = dO_z[i] V_z^T
// for z = b*H + h.  One CTA owns 128 query rows of one (b, h) and streams the
// keys in 64-wide chunks: a 3-stage TMA ring of K (or V) chunks feeds
// tcgen05.mma (M=128, N=64) into two 64-column TMEM accumulators, so the MMA
// of chunk j+1 overlaps the softmax of chunk j.  Two passes over the chunks:
// pass 0 gathers the row statistics (online max / sum for the forward,
// rowsum(P * dP) for the backward), pass 1 recomputes each chunk's scores and
// writes the bf16 probabilities (score gradients) with TMA stores.  Recomputing
// the 128 x 64 x d_head product is cheaper than keeping 128 x L scores resident,
// and the small footprint (~99 KB smem, 128 TMEM columns) puts two CTAs on every
// SM, so one CTA's softmax overlaps the other's loads and MMAs.  No fp32 score
// matrix and no separate softmax kernel (csrc/train_ops.cu keeps the unfused
// kernels for reference/tests).  The reference has no attention at all (SPEC:90
// folds it into 6*P*T); parity is against the fp64 block oracle.
//
// Warp roles: warp 0 TMA, warp 1 MMA issuer, warp 2 TMEM allocator, warps 4-7
// one query row per thread (TMEM lane quarter = warp % 4).  CTAs are ordered
// heaviest first (causal: the last query blocks see the most keys).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <unordered_map>
#include <utility>

#include "common.cuh"
#include "sm100.cuh"

namespace swarm {
namespace attn {

using namespace swarm::sm100;

constexpr int kThreads = 256;
constexpr int BQ = 128;        // query rows per CTA
constexpr int BKV = 64;        // keys per chunk (MMA N)
constexpr int kMaxL = 1024;
constexpr int kMaxDh = 128;    // K extent of the score GEMM (<= 2 x 64-wide boxes)
constexpr int kSlot = 2048;    // one 32 x 32 bf16 staging box

struct Params {
    int B, H, L, dh, causal;
    int a_col0, b_col0;  // column of head 0 in the A / B storages
    float scale;
    const __nv_bfloat16* o;  // backward: O = P V [B*L, ld_o] (head h at column h*dh)
    int ld_o;
    int trace;  // record the per-CTA timeline (experiments)
    float* lse;  // PV forward: when set, P is not stored; lse[z*L + i] = the row's log2-sum-exp of scale * q.k * log2(e)
};

constexpr int kABytes = (kMaxDh / 64) * BQ * 128;       // 32 KB: Q / dO block
constexpr int kChunkBytes = (kMaxDh / 64) * BKV * 128;  // 16 KB: K / V chunk
constexpr int kPChunkBytes = BQ * BKV * 2;              // 16 KB: P chunk (backward), dS written in place
// forward: 3-stage K ring + 4 row warps x 2 staging slots; backward: 2-stage
// (V chunk, P chunk) ring, dS staged in place of the P chunk it replaces
// PV (forward with O = P V fused, d_head = 128): 2-stage (K chunk, V chunk) ring; each chunk's P is
// written over its stage's K chunk once the score MMA has read it, stored from there, and read
// there by the P V MMA (A operand); the O accumulator takes TMEM columns 128-255
template <bool BWD, bool PV = false>
struct Lay {
    static constexpr int kStages = BWD || PV ? 2 : 3;
    static constexpr int kStageBytes = kChunkBytes + (BWD ? kPChunkBytes : (PV ? kChunkBytes : 0));
    static constexpr int kStgBytes = BWD || PV ? 0 : 4 * 2 * kSlot;
    static constexpr int kSmem = kABytes + kStages * kStageBytes + kStgBytes + 1024 + 256;
    static constexpr int kTmemCols = PV ? 4 * BKV : 2 * BKV;
    static_assert(2 * (kSmem + 1024) <= 233472, "two attention CTAs must fit one SM");
};

// 2^x on the SFU (ex2.approx.ftz: 2 ulp; the probabilities are rounded to bf16 anyway)
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x for x <= 0 on the FMA pipe (FlashAttention-4's trick to relieve the SFU):
// x = n + f with n = rint(x) via the 1.5 * 2^23 magic add, 2^f on [-0.5, 0.5] by a
// degree-3 minimax polynomial (max relative error 2.1e-4, far below bf16's 2^-8),
// then n is added to the exponent field.  x is clamped at -125 (result ~2^-125).
__device__ __forceinline__ float poly_exp2(float x) {
    x = fmaxf(x, -125.f);
    const float t = __fadd_rn(x, 12582912.f);
    const float f = __fsub_rn(x, __fsub_rn(t, 12582912.f));
    const float p = fmaf(fmaf(fmaf(5.484800413e-02f, f, 2.418066114e-01f), f, 6.932482123e-01f), f, 9.999886751e-01f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// a quarter of the exponentials go to the FMA pipe, the rest to the SFU
template <int J>
__device__ __forceinline__ float mixed_exp2(float x) {
    if constexpr ((J & 3) == 0) return poly_exp2(x);
    else return fast_exp2(x);
}

template <int... J>
__device__ __forceinline__ float sum_exp2_impl(const uint32_t (&ra)[32], const uint32_t (&rb)[32], float cs, float nb,
                                               std::integer_sequence<int, J...>) {
    float acc[2] = {0.f, 0.f};
    ((acc[J & 1] += mixed_exp2<J>(fmaf(__uint_as_float(ra[J]), cs, nb)) +
                    mixed_exp2<J + 1>(fmaf(__uint_as_float(rb[J]), cs, nb))),
     ...);
    return acc[0] + acc[1];
}
// sum over the 64 scores of a chunk of 2^(s * cs + nb)
__device__ __forceinline__ float sum_exp2_64(const uint32_t (&ra)[32], const uint32_t (&rb)[32], float cs, float nb) {
    return sum_exp2_impl(ra, rb, cs, nb, std::make_integer_sequence<int, 32>{});
}
template <int... J>
__device__ __forceinline__ void exp2_impl(const uint32_t (&ra)[32], const uint32_t (&rb)[32], float cs, float nb,
                                          float* v, std::integer_sequence<int, J...>) {
    ((v[J] = mixed_exp2<J>(fmaf(__uint_as_float(ra[J]), cs, nb)),
      v[32 + J] = mixed_exp2<J + 2>(fmaf(__uint_as_float(rb[J]), cs, nb))),
     ...);
}
__device__ __forceinline__ void exp2_64(const uint32_t (&ra)[32], const uint32_t (&rb)[32], float cs, float nb,
                                        float* v) {
    exp2_impl(ra, rb, cs, nb, v, std::make_integer_sequence<int, 32>{});
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&p);
}

// 32 x 32 bf16 box, SWIZZLE_64B (16-B chunk j of row r at j ^ ((r >> 1) & 3))
__device__ __forceinline__ void stage_bf16(uint8_t* slot, int row, const float* v) {
    const uint32_t base = smem_u32(slot) + row * 64;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        st_shared_v4(base + ((j ^ ((row >> 1) & 3)) << 4), pack_bf16(v[8 * j], v[8 * j + 1]),
                     pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                     pack_bf16(v[8 * j + 6], v[8 * j + 7]));
}

// Per-CTA timeline for experiments (SWARM_ATTN_TRACE=1, scripts/attn_trace.py):
// globaltimer at entry, after the prologue, after the statistics pass, at the end
// of the output pass, and the CTA's SM id.
constexpr int kTraceCtas = 4096;
__device__ unsigned long long g_attn_trace[kTraceCtas][6];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace(const Params& p, int slot) {
    if (p.trace && blockIdx.x < kTraceCtas) g_attn_trace[blockIdx.x][slot] = gtimer();
}

template <bool BWD, bool PV = false, bool ONE = false>
__global__ void __launch_bounds__(kThreads, 2)
    k_attn_chunks(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                  const __grid_constant__ CUtensorMap tma_p, const __grid_constant__ CUtensorMap tma_out,
                  const Params p) {
    // PV: tma_p maps V (the forward reads no P), O goes to p.o_out
    // forward: pass 0 row max / sum, pass 1 probabilities; backward: one pass, the
    // row statistic rowsum(P * dP) = dO . O comes from the forward output
    // PV with an lse output: one pass with an online row max (O rescaled in TMEM when the max
    // grows by more than 2^8; the final O divided by the row sum), no statistics pass
    constexpr bool one = PV && ONE;
    constexpr int kPasses = (BWD || one) ? 1 : 2;
    pdl_trigger();
    if (threadIdx.x == 128) {
        trace(p, 0);
        if (p.trace && blockIdx.x < kTraceCtas) {
            unsigned smid;
            asm("mov.u32 %0, %%smid;" : "=r"(smid));
            g_attn_trace[blockIdx.x][5] = smid;
        }
    }
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw & 1023)) & 1023);
    using Y = Lay<BWD, PV>;
    constexpr int kStages = Y::kStages;
    uint8_t* sa = smem;
    uint8_t* sb = sa + kABytes;  // stage s: K / V chunk, then (backward) the P chunk
    uint8_t* stg_all = sb + kStages * Y::kStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(stg_all + Y::kStgBytes);
    uint64_t* qfull = bars;
    uint64_t* full = bars + 1;
    uint64_t* empty = full + kStages;
    uint64_t* sfull = empty + kStages;
    uint64_t* sempty = sfull + 2;
    // PV: per stage, the 4 row warps wrote that stage's chunk P (over its K chunk).  One barrier per
    // stage, not one overall: the row warps may finish two chunks' P before the MMA thread polls, and a
    // single barrier would then have moved two phases past the waiter's parity
    uint64_t* pfull = sempty + 2;
    uint64_t* ofull = pfull + 2;  // PV: the last P V MMA committed
    uint64_t* pvdone = ofull + 1;  // one pass: each P V MMA committed (the rows rescale O after it)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pvdone + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = p.L / BQ, nz = p.B * p.H;
    const int mt = nqb - 1 - static_cast<int>(blockIdx.x) / nz;  // heaviest query blocks first
    const int z = static_cast<int>(blockIdx.x) % nz;
    const int zb = z / p.H, zh = z - zb * p.H;
    const int kboxes = p.dh / 64;
    const int kv_len = p.causal ? (mt + 1) * BQ : p.L;  // keys past the block's last query are masked
    const int nch = kv_len / BKV;

    if (warp == 0 && lane == 0) {
        mbar_init(qfull, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            // bwd: the MMA and the 4 row warps (P read, dS stored); PV: the MMA (scores, or P V) and
            // the 4 row warps (S read in pass 0, P stored from the stage in pass 1)
            mbar_init(&empty[s], BWD || PV ? 5 : 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sfull[b], 1);
            mbar_init(&sempty[b], 4);
        }
        mbar_init(&pfull[0], 4);
        mbar_init(&pfull[1], 4);
        mbar_init(ofull, 1);
        mbar_init(pvdone, 1);
        fence_barrier_init();
    }
    if (warp == 2) {
        tmem_alloc(tmem_slot, Y::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();

    if (warp == 0 && lane == 0) {
        // ------------------------------------------------------------ TMA
        const int arow = zb * p.L + mt * BQ, acol = p.a_col0 + zh * p.dh;
        const int brow = zb * p.L, bcol = p.b_col0 + zh * p.dh;
        mbar_arrive_expect_tx(qfull, kboxes * BQ * 128);
        for (int kb = 0; kb < kboxes; ++kb) tma_load_2d(sa + kb * BQ * 128, &tma_a, qfull, acol + kb * 64, arow);
        int stage = 0;
        uint32_t phase = 0;
        for (int pass = 0; pass < kPasses; ++pass)
            for (int j = 0; j < nch; ++j) {
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sst = sb + stage * Y::kStageBytes;
                const bool load_v = PV && pass == kPasses - 1;
                mbar_arrive_expect_tx(&full[stage], kboxes * BKV * 128 * (load_v ? 2 : 1) + (BWD ? kPChunkBytes : 0));
                for (int kb = 0; kb < kboxes; ++kb)
                    tma_load_2d(sst + kb * BKV * 128, &tma_b, &full[stage], bcol + kb * 64, brow + j * BKV);
                if (load_v)  // V chunk (MN-major B of the P V MMA): [64 keys x 64 d_head] boxes after the K chunk
                    for (int kb = 0; kb < kboxes; ++kb)
                        tma_load_2d(sst + kChunkBytes + kb * BKV * 128, &tma_p, &full[stage], bcol + kb * 64,
                                    brow + j * BKV);
                if constexpr (BWD)  // P[z, mt*128 .. +128, j*64 .. +64]
                    tma_load_2d(sst + kChunkBytes, &tma_p, &full[stage], j * BKV, z * p.L + mt * BQ);
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------------------ MMA
        constexpr uint32_t idesc = make_idesc_bf16(BQ, BKV, false, false);
        mbar_wait(qfull, 0);
        int stage = 0, buf = 0;
        uint32_t phase = 0, bphase = 0;
        const int ksteps = p.dh / 16;
        // PV: O += P_j V_j (M 128, N d_head, K 64 keys): A = P_j over the K chunk, B = V_j MN-major
        constexpr uint32_t idesc_pv = make_idesc_bf16(BQ, kMaxDh, false, true);
        uint32_t pphase[2] = {0, 0};
        auto issue_pv = [&](int st_pv, int jj) {
            mbar_wait(&pfull[st_pv], pphase[st_pv]);
            pphase[st_pv] ^= 1;
            tc_fence_after();
            const uint32_t p_base = smem_u32(sb + st_pv * Y::kStageBytes);
            const uint32_t v_base = p_base + kChunkBytes;
            for (int kk = 0; kk < BKV / 16; ++kk) {
                const uint64_t ad = make_sdesc(p_base + kk * 32, 16, 1024);
                const uint64_t bd = make_sdesc(v_base + kk * 2048, BKV * 128, 1024);
                mma_bf16(tmem + 2 * BKV, ad, bd, idesc_pv, (jj != 0 || kk != 0) ? 1u : 0u);
            }
            mma_commit(&empty[st_pv]);
            if constexpr (one) mma_commit(pvdone);
        };
        int prev_stage = -1;
        for (int pass = 0; pass < kPasses; ++pass)
            for (int j = 0; j < nch; ++j) {
                mbar_wait(&full[stage], phase);
                mbar_wait(&sempty[buf], bphase ^ 1);
                tc_fence_after();
                const uint32_t a_base = smem_u32(sa), b_base = smem_u32(sb + stage * Y::kStageBytes);
                for (int kk = 0; kk < ksteps; ++kk) {
                    const uint64_t ad = make_sdesc(a_base + (kk >> 2) * (BQ * 128) + (kk & 3) * 32, 16, 1024);
                    const uint64_t bd = make_sdesc(b_base + (kk >> 2) * (BKV * 128) + (kk & 3) * 32, 16, 1024);
                    mma_bf16(tmem + buf * BKV, ad, bd, idesc, kk != 0 ? 1u : 0u);
                }
                const bool pv_pass = PV && pass == kPasses - 1;
                if (!pv_pass) mma_commit(&empty[stage]);  // (PV pass: the stage is released after P V)
                mma_commit(&sfull[buf]);
                if (pv_pass) {  // the previous chunk's P V overlaps this chunk's softmax
                    if (j > 0) issue_pv(prev_stage, j - 1);
                    prev_stage = stage;
                }
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
                if (++buf == 2) {
                    buf = 0;
                    bphase ^= 1;
                }
            }
        if constexpr (PV) {
            issue_pv(prev_stage, nch - 1);
            mma_commit(ofull);
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ one query row per thread
        const int q = warp - 4;
        const int r = q * 32 + lane;
        const int qi = mt * BQ + r;
        const int valid = p.causal ? qi + 1 : p.L;  // columns < valid are unmasked
        const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
        uint8_t* stg = stg_all + q * 2 * kSlot;
        int slot_idx = 0;
        const int out_row = z * p.L + mt * BQ + q * 32;
        int buf = 0;
        uint32_t bphase = 0;
        // scores are raw q.k; softmax works in log2 units u = s * cs
        const float cs = p.scale * 1.4426950408889634f;
        if (r == 0) trace(p, 1);
        float bias = 0.f;  // fwd pass 1: max(u) + log2(sum), so p = 2^(u - bias); bwd: dO . O
        int stage = 0;
        uint32_t sphase = 0;
        float m_used = -INFINITY, l_run = 0.f;  // one pass: the exponent offset in use, the running sum
        float resc = 1.f;                         // one pass: this chunk's O rescale factor
        if constexpr (!BWD && !one) {
            // ---------------- pass 0: online row max / sum
            float mu = -INFINITY, l = 0.f;
            for (int j = 0; j < nch; ++j) {
                uint32_t ra[32], rb[32];
                mbar_wait(&sfull[buf], bphase);
                tc_fence_after();
                tmem_ld_32x32b_x32(trow + buf * BKV, ra);
                tmem_ld_32x32b_x32(trow + buf * BKV + 32, rb);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sempty[buf]);
                    if (PV) mbar_arrive(&empty[stage]);  // (PV: a stage is freed by the MMA and the 4 row warps)
                }
                if (++stage == kStages) {
                    stage = 0;
                    sphase ^= 1;
                }
                if (++buf == 2) {
                    buf = 0;
                    bphase ^= 1;
                }
                const int c0 = j * BKV;
                if (c0 >= valid) continue;  // fully masked for this row
                const bool full = c0 + BKV <= valid;
                float cm = -INFINITY;
                if (full) {
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj)
                        cm = fmaxf(cm, fmaxf(__uint_as_float(ra[jj]), __uint_as_float(rb[jj])));
                } else {
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        if (c0 + jj < valid) cm = fmaxf(cm, __uint_as_float(ra[jj]));
                        if (c0 + 32 + jj < valid) cm = fmaxf(cm, __uint_as_float(rb[jj]));
                    }
                }
                const float nmu = fmaxf(mu, cm * cs);
                float add = 0.f;
                if (full) {
                    add = sum_exp2_64(ra, rb, cs, -nmu);
                } else {
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        if (c0 + jj < valid) add += fast_exp2(fmaf(__uint_as_float(ra[jj]), cs, -nmu));
                        if (c0 + 32 + jj < valid) add += fast_exp2(fmaf(__uint_as_float(rb[jj]), cs, -nmu));
                    }
                }
                l = (mu == -INFINITY ? 0.f : l * fast_exp2(mu - nmu)) + add;
                mu = nmu;
            }
            bias = mu + __log2f(l);
        } else if (BWD) {
            // D = dO[row] . O[row] over this head's d_head columns (= rowsum(P * dP))
            const size_t grow = static_cast<size_t>(zb) * p.L + qi;
            // dO[row] from the A tile (2 x 128-B SWIZZLE_128B boxes), O[row] from global in 2 batches
            const uint4* o4 = reinterpret_cast<const uint4*>(p.o + grow * p.ld_o + zh * p.dh);
            mbar_wait(qfull, 0);
            float acc = 0.f;
            for (int half = 0; half < p.dh / 64; ++half) {
                uint4 b[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) b[c] = __ldg(o4 + half * 8 + c);
                const uint32_t arow_s = smem_u32(sa + half * BQ * 128) + r * 128;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint32_t a0, a1, a2, a3;
                    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                                 : "r"(arow_s + ((c ^ (r & 7)) << 4)));
                    const uint32_t wa[4] = {a0, a1, a2, a3}, wb[4] = {b[c].x, b[c].y, b[c].z, b[c].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        acc += __uint_as_float(wa[k] << 16) * __uint_as_float(wb[k] << 16) +
                               __uint_as_float(wa[k] & 0xffff0000u) * __uint_as_float(wb[k] & 0xffff0000u);
                }
            }
            bias = acc;
        }
        if (r == 0) trace(p, 2);
        // ---------------- probabilities (fwd pass 1) / score gradients (bwd)
        for (int j = 0; j < nch; ++j) {
            const int c0 = j * BKV;
            uint32_t ra[32], rb[32];
            mbar_wait(&sfull[buf], bphase);
            tc_fence_after();
            tmem_ld_32x32b_x32(trow + buf * BKV, ra);
            tmem_ld_32x32b_x32(trow + buf * BKV + 32, rb);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sempty[buf]);
            if (++buf == 2) {
                buf = 0;
                bphase ^= 1;
            }
            if constexpr (!BWD) {
                float v[64];
                if constexpr (one) {
                    // online max: a chunk whose max exceeds the offset in use by more than 2^8 moves it,
                    // rescaling the running sum and this row's O accumulator (after the P V MMAs issued so
                    // far completed: by the in-order tensor pipe, all but P V of the previous chunk)
                    float f = 1.f;
                    if (c0 < valid) {
                        float cm = -INFINITY;
                        if (c0 + BKV <= valid) {
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj)
                                cm = fmaxf(cm, fmaxf(__uint_as_float(ra[jj]), __uint_as_float(rb[jj])));
                        } else {
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) {
                                if (c0 + jj < valid) cm = fmaxf(cm, __uint_as_float(ra[jj]));
                                if (c0 + 32 + jj < valid) cm = fmaxf(cm, __uint_as_float(rb[jj]));
                            }
                        }
                        const float cmu = cm * cs;
                        if (m_used == -INFINITY) {
                            m_used = cmu;
                        } else if (cmu > m_used + 8.f) {
                            f = fast_exp2(m_used - cmu);
                            l_run *= f;
                            m_used = cmu;
                        }
                    }
                    resc = f;  // (O itself is rescaled after P_j is written, before P V_j may start)
                    bias = m_used;
                }
                if (c0 + BKV <= valid) {
                    exp2_64(ra, rb, cs, -bias, v);
                } else {
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        v[jj] = (c0 + jj < valid) ? fast_exp2(fmaf(__uint_as_float(ra[jj]), cs, -bias)) : 0.f;
                        v[32 + jj] = (c0 + 32 + jj < valid) ? fast_exp2(fmaf(__uint_as_float(rb[jj]), cs, -bias)) : 0.f;
                    }
                }
                if constexpr (one) {
                    float add = 0.f;
#pragma unroll
                    for (int jj = 0; jj < 64; ++jj) add += v[jj];
                    l_run += add;
                }
                if constexpr (PV) {
                    // P_j over this stage's K chunk (the score MMA has read it: sfull), in the
                    // SWIZZLE_128B K-major layout the P V MMA reads as its A operand (128-B rows, 16-B
                    // piece k of row r at k ^ (r & 7)); stored to global from there too
                    uint8_t* pt = sb + stage * Y::kStageBytes;
                    const uint32_t prow = smem_u32(pt) + r * 128;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        st_shared_v4(prow + ((k ^ (r & 7)) << 4), pack_bf16(v[8 * k], v[8 * k + 1]),
                                     pack_bf16(v[8 * k + 2], v[8 * k + 3]), pack_bf16(v[8 * k + 4], v[8 * k + 5]),
                                     pack_bf16(v[8 * k + 6], v[8 * k + 7]));
                    if constexpr (one) {
                        // the offset moved for some row of the warp: rescale the warp's O rows once every
                        // P V MMA issued so far completed (by the in-order tensor pipe, all but the previous
                        // chunk's are: the score MMA of this chunk followed them)
                        if (__any_sync(0xffffffffu, resc != 1.f)) {
                            if (j > 0) mbar_wait(pvdone, (j - 1) & 1);
                            tc_fence_after();
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                uint32_t ro[32];
                                tmem_ld_32x32b_x32(trow + 2 * BKV + 32 * c, ro);
                                tmem_ld_wait();
#pragma unroll
                                for (int w = 0; w < 32; ++w) ro[w] = __float_as_uint(__uint_as_float(ro[w]) * resc);
                                tmem_st_32x32b_x32(trow + 2 * BKV + 32 * c, ro);
                            }
                            tmem_st_wait();
                            tc_fence_before();
                        }
                    }
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (!p.lse) {
                            tma_store_2d(&tma_out, pt + q * 32 * 128, c0, out_row);
                            bulk_commit();
                        }
                        mbar_arrive(&pfull[stage]);
                        if (!p.lse) bulk_wait_read<0>();  // the box has left smem: the stage may be refilled
                        mbar_arrive(&empty[stage]);
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        sphase ^= 1;
                    }
                    continue;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint8_t* slot = stg + slot_idx * kSlot;
                    slot_idx ^= 1;
                    if (lane == 0) bulk_wait_read<1>();  // the store issued from this slot two boxes ago has read it
                    __syncwarp();
                    stage_bf16(slot, lane, v + 32 * h);
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&tma_out, slot, c0 + 32 * h, out_row);
                        bulk_commit();
                    }
                }
            } else {
                // this row's 64 P values sit in the stage's P chunk (128-B rows, SWIZZLE_128B:
                // 16-B piece k of row r at k ^ (r & 7)); dS overwrites them in place and
                // the warp's 32 x 64 box is stored from there
                const uint32_t prow_s = smem_u32(sb + stage * Y::kStageBytes + kChunkBytes) + r * 128;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t addr = prow_s + ((k ^ (r & 7)) << 4);
                    uint32_t w0, w1, w2, w3;
                    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                                 : "r"(addr));
                    const uint32_t w[4] = {w0, w1, w2, w3};
                    float o[8];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int c = k * 8 + 2 * e;  // column inside the chunk
                        const float d0 = __uint_as_float(c < 32 ? ra[c] : rb[c - 32]);
                        const float d1 = __uint_as_float(c + 1 < 32 ? ra[c + 1] : rb[c - 31]);
                        o[2 * e] = p.scale * __uint_as_float(w[e] << 16) * (d0 - bias);
                        o[2 * e + 1] = p.scale * __uint_as_float(w[e] & 0xffff0000u) * (d1 - bias);
                    }
                    st_shared_v4(addr, pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]),
                                 pack_bf16(o[6], o[7]));
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tma_out, sb + stage * Y::kStageBytes + kChunkBytes + q * 32 * 128, c0, out_row);
                    bulk_commit();
                    bulk_wait_read<0>();  // the box has left smem: the stage may be refilled
                    mbar_arrive(&empty[stage]);
                }
                if (++stage == kStages) {
                    stage = 0;
                    sphase ^= 1;
                }
            }
        }
        if constexpr (PV) {
            const float inv_l = one ? 1.f / l_run : 1.f;
            if (one) p.lse[static_cast<size_t>(z) * p.L + qi] = m_used + __log2f(l_run);
            // O row (d_head = 128 fp32 accumulators, TMEM columns 128-255) -> bf16 at O[b*L + qi, h*dh]
            mbar_wait(ofull, 0);
            tc_fence_after();
            __nv_bfloat16* orow = const_cast<__nv_bfloat16*>(p.o) + (static_cast<size_t>(zb) * p.L + qi) * p.ld_o +
                                  zh * p.dh;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t ro[32];
                tmem_ld_32x32b_x32(trow + 2 * BKV + 32 * c, ro);
                tmem_ld_wait();
                uint4* dst = reinterpret_cast<uint4*>(orow + 32 * c);
#pragma unroll
                for (int w = 0; w < 4; ++w)
                    dst[w] = make_uint4(pack_bf16(__uint_as_float(ro[8 * w]) * inv_l, __uint_as_float(ro[8 * w + 1]) * inv_l),
                                        pack_bf16(__uint_as_float(ro[8 * w + 2]) * inv_l, __uint_as_float(ro[8 * w + 3]) * inv_l),
                                        pack_bf16(__uint_as_float(ro[8 * w + 4]) * inv_l, __uint_as_float(ro[8 * w + 5]) * inv_l),
                                        pack_bf16(__uint_as_float(ro[8 * w + 6]) * inv_l, __uint_as_float(ro[8 * w + 7]) * inv_l));
            }
            tc_fence_before();
        }
        // keys past the causal block are never written (nothing on the hot path
        // reads them; the stage executor zeroes P / dS once at creation)
        if (lane == 0) bulk_wait_all();
        if (r == 0) trace(p, 3);
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, Y::kTmemCols);
    }
    if (threadIdx.x == 128) trace(p, 4);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeFn>(nullptr);
        return reinterpret_cast<EncodeFn>(ptr);
    }();
    return fn;
}

int map_bf16_uncached(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int bi, int bo,
                      CUtensorMapSwizzle sw);

// Descriptor cache (the same few operands recur every layer and microbatch):
// encoding costs microseconds of host time per map, which an eager visit would
// otherwise spend with the GPU idle.
struct MapKey {
    const void* ptr;
    long long rows, cols, ld;
    int bi, bo, sw;
    bool operator==(const MapKey& o) const {
        return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && bi == o.bi && bo == o.bo && sw == o.sw;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        size_t h = reinterpret_cast<uintptr_t>(k.ptr);
        for (long long v : {k.rows, k.cols, k.ld, static_cast<long long>(k.bi) << 32 | k.bo << 8 | k.sw})
            h = h * 0x9E3779B97F4A7C15ull + static_cast<size_t>(v);
        return h;
    }
};

int map_bf16(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int bi, int bo,
             CUtensorMapSwizzle sw) {
    thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    const MapKey key{ptr, rows, cols, ld, bi, bo, static_cast<int>(sw)};
    auto it = cache.find(key);
    if (it != cache.end()) {
        *m = it->second;
        return SWARM_OK;
    }
    const int rc = map_bf16_uncached(m, ptr, rows, cols, ld, bi, bo, sw);
    if (rc == SWARM_OK) {
        if (cache.size() > 4096) cache.clear();
        cache.emplace(key, *m);
    }
    return rc;
}

int map_bf16_uncached(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int bi, int bo,
                      CUtensorMapSwizzle sw) {
    EncodeFn enc = encoder();
    if (!enc) return SWARM_E_CUDA;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(bi), static_cast<cuuint32_t>(bo)};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
               ? SWARM_OK
               : SWARM_E_INVALID;
}

bool trace_enabled() {
    static const bool on = [] {
        const char* e = getenv("SWARM_ATTN_TRACE");
        return e && e[0] == '1';
    }();
    return on;
}

template <bool BWD, bool PV = false>
int launch(const void* a, int lda, int a_cols, int a_col0, const void* b, int ldb, int b_cols, int b_col0,
           const void* pin, const void* o, int ld_o, void* out, int B, int H, int L, int dh, float scale, int causal,
           cudaStream_t st, float* lse = nullptr) {
    // PV: pin = V (same storage geometry as K), o = the O output [B*L, ld_o]
    if (L % BQ || L > kMaxL || dh % 64 || dh > kMaxDh || B <= 0 || H <= 0)
        return invalid("attention: need L % 128 == 0, L <= 1024, dh % 64 == 0, dh <= 128");
    if (BWD && (!pin || (reinterpret_cast<uintptr_t>(pin) & 15)))
        return invalid("attention: P must be a 16-byte aligned bf16 [B*H*L, L] array");
    if (BWD && (!o || (reinterpret_cast<uintptr_t>(o) & 15) || (reinterpret_cast<uintptr_t>(a) & 15) || ld_o % 8 ||
                lda % 8))
        return invalid("attention: dO and O must be 16-byte aligned bf16 rows");
    const long long T = static_cast<long long>(B) * L, rows_out = static_cast<long long>(B) * H * L;
    CUtensorMap ta, tb, tp{}, to;
    // forward P: 32 x 32 boxes (SWIZZLE_64B staging); backward dS: 32 rows x 64 keys, in place of
    // the P chunk loaded with 128 x 64 boxes (SWIZZLE_128B)
    if (PV && (dh != kMaxDh || !pin || !o || (reinterpret_cast<uintptr_t>(o) & 15) || ld_o % 8))
        return invalid("attention P V: needs d_head 128, V, and a 16-byte aligned O");
    if (!out && !(PV && lse)) return invalid("attention: null output");
    if (map_bf16(&ta, a, T, a_cols, lda, 64, BQ, CU_TENSOR_MAP_SWIZZLE_128B) ||
        map_bf16(&tb, b, T, b_cols, ldb, 64, BKV, CU_TENSOR_MAP_SWIZZLE_128B) ||
        (out && (BWD || PV ? map_bf16(&to, out, rows_out, L, L, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B)
                           : map_bf16(&to, out, rows_out, L, L, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))))
        return invalid("attention: tensor map encoding failed");
    if (!out) to = ta;  // (unused: the LSE forward stores no P)
    if (BWD && map_bf16(&tp, pin, rows_out, L, L, 64, BQ, CU_TENSOR_MAP_SWIZZLE_128B))
        return invalid("attention: tensor map encoding failed (P)");
    if (PV && map_bf16(&tp, pin, T, b_cols, ldb, 64, BKV, CU_TENSOR_MAP_SWIZZLE_128B))
        return invalid("attention: tensor map encoding failed (V)");
    auto kern = (PV && lse) ? k_attn_chunks<BWD, PV, true> : k_attn_chunks<BWD, PV, false>;
    constexpr int kSmem = Lay<BWD, PV>::kSmem;
    static bool attr = false;
    if (!attr) {
        for (auto kf : {k_attn_chunks<BWD, PV, false>, k_attn_chunks<BWD, PV, true>}) {
            SWARM_CUDA_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
            SWARM_CUDA_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        }
        attr = true;
    }
    Params p{B, H, L, dh, causal, a_col0, b_col0, scale, static_cast<const __nv_bfloat16*>(o), ld_o,
             trace_enabled() ? 1 : 0, lse};
    // launched without programmatic serialization: letting the next-but-one grid's
    // CTAs claim the free slots early measured ~1 us slower per launch here
    // (scripts/launch_overhead.py); the kernel still triggers its own dependents
    kern<<<B * H * (L / BQ), kThreads, kSmem, st>>>(ta, tb, tp, to, p);
    SWARM_LAUNCH_CHECK("k_attn_chunks");
    return SWARM_OK;
}

}  // namespace attn
}  // namespace swarm

extern "C" {

int swarm_attn_scores_softmax(const void* q, const void* k, int ld, int n_cols, int B, int H, int L, int dh,
                              float scale, int causal, void* P, swarm_stream_t stream) {
    return swarm::attn::launch<false>(q, ld, n_cols, 0, k, ld, n_cols, 0, nullptr, nullptr, 0, P, B, H, L, dh, scale,
                                      causal, swarm::as_stream(stream));
}

int swarm_attn_forward_pv(const void* q, const void* k, const void* v, int ld, int n_cols, int B, int H, int L,
                          int dh, float scale, int causal, void* P, void* O, int ld_o, swarm_stream_t stream) {
    return swarm::attn::launch<false, true>(q, ld, n_cols, 0, k, ld, n_cols, 0, v, O, ld_o, P, B, H, L, dh, scale,
                                            causal, swarm::as_stream(stream));
}

int swarm_attn_forward_lse(const void* q, const void* k, const void* v, int ld, int n_cols, int B, int H, int L,
                           int dh, float scale, int causal, float* lse, void* O, int ld_o, swarm_stream_t stream) {
    if (!lse) return swarm::invalid("attention: null lse");
    return swarm::attn::launch<false, true>(q, ld, n_cols, 0, k, ld, n_cols, 0, v, O, ld_o, nullptr, B, H, L, dh, scale,
                                            causal, swarm::as_stream(stream), lse);
}

int swarm_attn_scores_softmax_backward(const void* dO, int ld_do, const void* v, int ld_v, int v_cols, const void* o,
                                       int ld_o, const void* P, int B, int H, int L, int dh, float scale, int causal,
                                       void* dS, swarm_stream_t stream) {
    return swarm::attn::launch<true>(dO, ld_do, H * dh, 0, v, ld_v, v_cols, 0, P, o, ld_o, dS, B, H, L, dh, scale,
                                     causal, swarm::as_stream(stream));
}

// experiments only (not in the public header): copy the last traced launch's
// per-CTA timeline, n_ctas x 6 u64 (t_entry, t_prologue, t_stats, t_out, t_exit, smid)
int swarm_debug_attn_trace(uint64_t* host, int n_ctas) {
    if (n_ctas > swarm::attn::kTraceCtas) n_ctas = swarm::attn::kTraceCtas;
    return cudaMemcpyFromSymbol(host, swarm::attn::g_attn_trace, sizeof(uint64_t) * 6 * n_ctas) == cudaSuccess
               ? SWARM_OK
               : SWARM_E_CUDA;
}

}  // extern "C"
