// Fused attention-score kernels (sm_100a, tcgen05 + TMEM + TMA).
//
// Forward:  P[z, i, :] = softmax(scale * Q_z[i] K_z^T)        (causal optional)
// Backward: dS[z, i, :] = scale * P (dP - rowsum(P * dP)),  dP = dO_z[i] V_z^T
// for z = b*H + h.  One CTA owns 128 query rows of one (b, h): the full
// 128 x L score block (L <= 512) is accumulated in TMEM (up to all 512
// columns), so the softmax (or its gradient) is applied straight out of TMEM
// and only the bf16 probabilities / score gradients reach HBM — no fp32 S or
// dP round trip and no separate softmax kernel (csrc/train_ops.cu keeps the
// unfused kernels for reference/tests).  The reference has no attention at all
// (SPEC:90 folds it into 6*P*T); parity is against the fp64 block oracle.
//
// Warp roles: warp 0 TMA (Q/dO block, K/V rows, and in the backward the P block
// after the MMAs), warp 1 MMA issuer, warp 2 TMEM allocator; then all 8 warps
// run the softmax epilogue (one row per thread, key columns split between warps
// 4-7 and 0-3, row statistics combined through smem), staged through swizzled
// smem and written with TMA stores.
#include <cudaTypedefs.h>

#include <algorithm>
#include <unordered_map>

#include "common.cuh"
#include "sm100.cuh"

namespace swarm {
namespace attn {

using namespace swarm::sm100;

constexpr int kThreads = 256;
constexpr int BQ = 128;      // query rows per CTA
constexpr int kMaxL = 512;   // TMEM columns
constexpr int kMaxDh = 128;  // K extent of the score GEMM (2 x 64-wide k-blocks)
constexpr int kSlot = 4096;

struct Params {
    int B, H, L, dh, causal;
    int a_col0, b_col0;  // column of head 0 in the A / B storages
    float scale;
};

// smem: A [dh/64][128 x 64] bf16 | B [dh/64][L x 64] bf16 (reused for the P tile
// in the backward) | staging 8 warps x 2 x 4 KB | barriers
constexpr int kABytes = (kMaxDh / 64) * BQ * 64 * 2;       // 32 KB
constexpr int kBBytes = (kMaxDh / 64) * kMaxL * 64 * 2;    // 128 KB (>= the 128 x 512 P tile)
constexpr int kStgBytes = 8 * 2 * kSlot;                   // 64 KB: 8 warps x double buffer
constexpr int kSmem = kABytes + kBBytes + kStgBytes + 1024 + 128;
static_assert(kSmem <= 232448, "attention kernel exceeds 227 KB smem");

// 2^x on the SFU (ex2.approx.ftz: 2 ulp; the probabilities are rounded to bf16 anyway)
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&p);
}

__device__ __forceinline__ void stage_bf16(uint8_t* slot, int row, const float (&v)[32]) {
    const uint32_t base = smem_u32(slot) + row * 64;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        st_shared_v4(base + ((j ^ ((row >> 1) & 3)) << 4), pack_bf16(v[8 * j], v[8 * j + 1]),
                     pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                     pack_bf16(v[8 * j + 6], v[8 * j + 7]));
}

// P tile in smem: [L/64 boxes][128 rows x 128 B], SWIZZLE_128B: 16-B chunk j of
// row r at j ^ (r & 7).  Returns 32 consecutive P values of row r from column c0.
__device__ __forceinline__ void load_p32(const uint8_t* ptile, int r, int c0, float (&p)[32]) {
    const uint8_t* box = ptile + (c0 >> 6) * (BQ * 128);
    const uint32_t rowbase = smem_u32(box) + r * 128;
    const int j0 = (c0 & 63) >> 3;  // first 16-B chunk inside the 128-B row
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t w0, w1, w2, w3;
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                     : "r"(rowbase + (((j0 + q) ^ (r & 7)) << 4)));
        const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            p[q * 8 + 2 * k] = __uint_as_float(w[k] << 16);
            p[q * 8 + 2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
        }
    }
}

template <bool BWD>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_rows(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                const __grid_constant__ CUtensorMap tma_p_in, const __grid_constant__ CUtensorMap tma_out,
                const Params p) {
    pdl_trigger();
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw & 1023)) & 1023);
    uint8_t* sa = smem;
    uint8_t* sb = smem + kABytes;
    uint8_t* stg_all = sb + kBBytes;
    uint64_t* bar_ab = reinterpret_cast<uint64_t*>(stg_all + kStgBytes);
    uint64_t* bar_mma = bar_ab + 1;
    uint64_t* bar_p = bar_ab + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_ab + 3);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = p.L / BQ;
    const int z = blockIdx.x / nqb, mt = blockIdx.x - z * nqb;
    const int zb = z / p.H, zh = z - zb * p.H;
    const int kblocks = p.dh / 64;
    const int nmma = p.L < 256 ? p.L : 256;  // MMA N per instruction
    // causal: keys beyond the last query row of this block are fully masked
    const int kv_len = p.causal ? min(p.L, (mt + 1) * BQ) : p.L;
    const int n_halves = (kv_len + nmma - 1) / nmma;

    if (warp == 0 && lane == 0) {
        mbar_init(bar_ab, 1);
        mbar_init(bar_mma, 1);
        mbar_init(bar_p, 1);
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
    pdl_wait();

    if (warp == 0 && lane == 0) {
        // ------------------------------------------------------------ TMA
        const int arow = zb * p.L + mt * BQ, acol = p.a_col0 + zh * p.dh;
        const int brow = zb * p.L, bcol = p.b_col0 + zh * p.dh;
        const uint32_t bytes = kblocks * (BQ * 128 + n_halves * nmma * 128);
        mbar_arrive_expect_tx(bar_ab, bytes);
        for (int kb = 0; kb < kblocks; ++kb) {
            tma_load_2d(sa + kb * BQ * 128, &tma_a, bar_ab, acol + kb * 64, arow);
            for (int h = 0; h < n_halves; ++h)
                tma_load_2d(sb + kb * (kMaxL * 128) + h * nmma * 128, &tma_b, bar_ab, bcol + kb * 64, brow + h * nmma);
        }
        if constexpr (BWD) {
            // after the MMAs have consumed B, bring the P block into the same space
            mbar_wait(bar_mma, 0);
            mbar_arrive_expect_tx(bar_p, (kv_len / 64) * BQ * 128);
            for (int c = 0; c < kv_len / 64; ++c)
                tma_load_2d(sb + c * BQ * 128, &tma_p_in, bar_p, c * 64, z * p.L + mt * BQ);
        }
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------------------ MMA
        mbar_wait(bar_ab, 0);
        tc_fence_after();
        const uint32_t idesc = make_idesc_bf16(BQ, nmma, false, false);
        for (int kb = 0; kb < kblocks; ++kb) {
            const uint32_t a_base = smem_u32(sa + kb * BQ * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t ad = make_sdesc(a_base + k * 32, 16, 1024);
                for (int h = 0; h < n_halves; ++h) {
                    const uint32_t b_base = smem_u32(sb + kb * (kMaxL * 128) + h * nmma * 128);
                    const uint64_t bd = make_sdesc(b_base + k * 32, 16, 1024);
                    mma_bf16(tmem + h * nmma, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
                }
            }
        }
        mma_commit(bar_mma);
    }
    __syncwarp();  // lanes of warps 0/1 re-converge after their single-thread roles
    {
        // ------------------------------------------------------------ softmax epilogue
        // All 8 warps: warp w owns TMEM lane quarter w % 4 (32 rows, one per
        // thread); warps 4-7 take the first half of the key chunks, warps 0-3 the
        // second half (and the all-masked tail); row statistics meet in smem.
        // row statistics live in the A (Q / dO) tile, dead once the MMAs completed
        float (*st_a)[BQ] = reinterpret_cast<float (*)[BQ]>(sa);
        float (*st_b)[BQ] = reinterpret_cast<float (*)[BQ]>(sa + 2 * BQ * sizeof(float));
        const int q = warp & 3;
        const int grp = warp >= 4 ? 0 : 1;
        const int r = q * 32 + lane;            // row inside the block
        const int qi = mt * BQ + r;             // query position in the sequence
        const int valid = p.causal ? qi + 1 : p.L;
        const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
        uint8_t* stg = stg_all + (warp & 7) * 2 * kSlot;  // two 4 KB slots per warp
        int slot_idx = 0;
        const int out_row = z * p.L + mt * BQ + q * 32;
        const int n32 = kv_len / 32;
        const int split = (n32 / 2) * 32;
        const int c_lo = grp == 0 ? 0 : split, c_hi = grp == 0 ? split : kv_len;
        mbar_wait(bar_mma, 0);
        tc_fence_after();
        const float l2e = 1.4426950408889634f;
        float stat_a = 0.f, stat_b = 0.f;  // fwd: row max / 1/sum; bwd: rowsum(P*dP)
        if constexpr (!BWD) {
            float m = -INFINITY, s = 0.f;
            for (int c0 = c_lo; c0 < c_hi; c0 += 64) {
                uint32_t ra[32], rb[32];
                tmem_ld_32x32b_x32(trow + c0, ra);
                tmem_ld_32x32b_x32(trow + c0 + 32, rb);
                tmem_ld_wait();
                float cm = -INFINITY;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (c0 + j < valid) cm = fmaxf(cm, __uint_as_float(ra[j]));
                    if (c0 + 32 + j < valid) cm = fmaxf(cm, __uint_as_float(rb[j]));
                }
                const float nm = fmaxf(m, cm * p.scale);
                if (nm != -INFINITY) {
                    float add = 0.f;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (c0 + j < valid) add += fast_exp2((__uint_as_float(ra[j]) * p.scale - nm) * l2e);
                        if (c0 + 32 + j < valid) add += fast_exp2((__uint_as_float(rb[j]) * p.scale - nm) * l2e);
                    }
                    s = (m == -INFINITY ? 0.f : s * fast_exp2((m - nm) * l2e)) + add;
                    m = nm;
                }
            }
            st_a[grp][r] = m;
            st_b[grp][r] = s;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            const float m0 = st_a[0][r], m1 = st_a[1][r];
            const float mm = fmaxf(m0, m1);
            const float ss = (m0 == -INFINITY ? 0.f : st_b[0][r] * fast_exp2((m0 - mm) * l2e)) +
                             (m1 == -INFINITY ? 0.f : st_b[1][r] * fast_exp2((m1 - mm) * l2e));
            stat_a = mm;
            stat_b = 1.f / ss;
        } else {
            mbar_wait(bar_p, 0);
            float acc = 0.f;
            for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
                uint32_t rr[32];
                tmem_ld_32x32b_x32(trow + c0, rr);
                tmem_ld_wait();
                float pv[32];
                load_p32(sb, r, c0, pv);
#pragma unroll
                for (int j = 0; j < 32; ++j) acc += pv[j] * __uint_as_float(rr[j]);
            }
            st_a[grp][r] = acc;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            stat_a = st_a[0][r] + st_a[1][r];
        }
        // second pass: normalise (fwd) / form dS (bwd); masked / skipped columns write 0
        const int w_hi = grp == 0 ? c_hi : p.L;
        for (int c0 = c_lo; c0 < w_hi; c0 += 32) {
            float v[32];
            if (c0 < kv_len) {
                uint32_t rr[32];
                tmem_ld_32x32b_x32(trow + c0, rr);
                tmem_ld_wait();
                if constexpr (!BWD) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        v[j] = (c0 + j < valid) ? fast_exp2((__uint_as_float(rr[j]) * p.scale - stat_a) * l2e) * stat_b
                                                : 0.f;
                } else {
                    float pv[32];
                    load_p32(sb, r, c0, pv);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = p.scale * pv[j] * (__uint_as_float(rr[j]) - stat_a);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
            uint8_t* slot = stg + slot_idx * kSlot;
            slot_idx ^= 1;
            if (lane == 0) bulk_wait_read<1>();  // the store issued from this slot two chunks ago has read it
            __syncwarp();
            stage_bf16(slot, lane, v);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(&tma_out, slot, c0, out_row);
                bulk_commit();
            }
        }
        if (lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
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

template <bool BWD>
int launch(const void* a, int lda, int a_cols, int a_col0, const void* b, int ldb, int b_cols, int b_col0,
           const void* pin, void* out, int B, int H, int L, int dh, float scale, int causal, cudaStream_t st) {
    if (L % BQ || L > kMaxL || dh % 64 || dh > kMaxDh || B <= 0 || H <= 0)
        return invalid("attention: need L % 128 == 0, L <= 512, dh % 64 == 0, dh <= 128");
    const long long T = static_cast<long long>(B) * L, rows_out = static_cast<long long>(B) * H * L;
    const int nmma = L < 256 ? L : 256;
    CUtensorMap ta, tb, tp{}, to;
    if (map_bf16(&ta, a, T, a_cols, lda, 64, BQ, CU_TENSOR_MAP_SWIZZLE_128B) ||
        map_bf16(&tb, b, T, b_cols, ldb, 64, nmma, CU_TENSOR_MAP_SWIZZLE_128B) ||
        map_bf16(&to, out, rows_out, L, L, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
        return invalid("attention: tensor map encoding failed");
    if (BWD && map_bf16(&tp, pin, rows_out, L, L, 64, BQ, CU_TENSOR_MAP_SWIZZLE_128B))
        return invalid("attention: tensor map encoding failed (P)");
    auto kern = k_attn_rows<BWD>;
    static bool attr = false;
    if (!attr) {
        SWARM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        attr = true;
    }
    Params p{B, H, L, dh, causal, a_col0, b_col0, scale};
    SWARM_CUDA_TRY(launch_pdl(kern, dim3(B * H * (L / BQ)), dim3(kThreads), kSmem, st, ta, tb, tp, to, p));
    SWARM_LAUNCH_CHECK("k_attn_rows");
    return SWARM_OK;
}

}  // namespace attn
}  // namespace swarm

extern "C" {

int swarm_attn_scores_softmax(const void* q, const void* k, int ld, int n_cols, int B, int H, int L, int dh,
                              float scale, int causal, void* P, swarm_stream_t stream) {
    return swarm::attn::launch<false>(q, ld, n_cols, 0, k, ld, n_cols, 0, nullptr, P, B, H, L, dh, scale, causal,
                                      swarm::as_stream(stream));
}

int swarm_attn_scores_softmax_backward(const void* dO, int ld_do, const void* v, int ld_v, int v_cols, const void* P,
                                       int B, int H, int L, int dh, float scale, int causal, void* dS,
                                       swarm_stream_t stream) {
    return swarm::attn::launch<true>(dO, ld_do, H * dh, 0, v, ld_v, v_cols, 0, P, dS, B, H, L, dh, scale, causal,
                                     swarm::as_stream(stream));
}

}  // extern "C"
