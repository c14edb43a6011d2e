// Stage executor: the real forward / backward visit of one SWARM pipeline
// stage on one B200 (the reference simulates it as a constant service time,
// /root/reference/proj/src/sim.cpp:361-364 and :395-403).
//
// Host C++ that only enqueues sm_100a kernels through the C-ABI on the
// caller's stream; every buffer is allocated once at creation, so a visit
// performs no allocation and no host synchronisation.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <tuple>
#include <string>
#include <unordered_map>
#include <vector>

#include "swarm_b200.h"

namespace {

using bf16 = uint16_t;  // storage only; kernels interpret it

// Element pointer into an activation buffer.  Its element is bf16 (2 B) or, in
// the fp32 arithmetic mode (swarm_stage_config.fp32), fp32 (4 B); offsets are in
// elements of the stage's dtype, so the visit code is the same in both modes.
struct EP {
    char* p = nullptr;
    int es = 2;
    EP() = default;
    EP(std::nullptr_t) {}
    EP(void* q, int e) : p(static_cast<char*>(q)), es(e) {}
    EP operator+(size_t n) const { return p ? EP(p + n * es, es) : EP(); }
    operator void*() const { return p; }
};

struct TensorInfo {
    std::string name;
    size_t off, rows, cols;
};

// one layer's backward gradients that its weight gradients read (paired mode)
struct Stash {
    EP dy, du, dhid, dqkv;
};

struct LayerW {
    size_t wqkv, wo, w1, w2, ln1g, ln1b, ln2g, ln2b;
};

struct Act {
    EP x, a, qkv, P, o, h, c, u, g;  // P: the forward's probabilities (not on the log2-sum-exp path)
    float *mu1, *rs1, *mu2, *rs2;
    float* lse = nullptr;  // the attention rows' log2-sum-exp [B*H*L] (the backward recomputes P from it)
};

struct Slot {
    std::vector<Act> layer;  // n_layers entries; layer[l].x is the input of application l
    EP out;               // output of the last application (input of the next stage / final LN)
    EP xf;                // final LN output (last stage)
    float *muf, *rsf;
    EP dxf;               // d loss / d xf, produced by the fused LM-head backward
    int32_t* tokens;         // first stage: the microbatch's token ids (embedding backward)
    // maxout bottleneck: sender keeps LN_c(out), its stats and the argmax;
    // receiver keeps the dequantized wire tensor, LN_d of it and its stats
    EP z;
    float *muc, *rsc;
    EP mo;
    uint8_t* am;
    EP mi, ni;
    float *mud, *rsd;
};

// One visit's workspaces (+ its side stream and fork/join events).  A stage
// keeps the active set in its fields; with lanes, set_lane swaps another set in,
// so two visits of the stage can be in flight on two streams.
struct Work {
    float *S = nullptr, *dP = nullptr, *logits = nullptr;
    EP dS, gy[2], dhid, dc, du, dqkv, dO, da, dlogits, wtmp;
    void* lnws = nullptr;
    void* abws = nullptr;
    cudaStream_t side = nullptr;
    void* skws[2] = {nullptr, nullptr};
    cudaEvent_t ev_fork[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_join = nullptr, ev_dq = nullptr;
};

}  // namespace

struct swarm_stage {
    swarm_stage_config cfg{};
    int T = 0, d = 0, H = 0, dh = 0, F = 0, V = 0, L = 0, B = 0;
    size_t nparams = 0;
    std::vector<TensorInfo> tensors;
    std::vector<LayerW> layers;
    size_t emb = 0, lnfg = 0, lnfb = 0, head = 0;
    bool f32 = false;    // fp32 arithmetic mode (swarm_stage_config.fp32)
    int es = 2;          // activation element size: 2 (bf16) or 4 (fp32)
    int dt = SWARM_DTYPE_BF16;  // activation dtype passed to the kernels
    bool bneck = false;  // maxout bottleneck at the boundaries
    bool stacked = false;  // layer-shared: stacked weight-gradient inputs (one K = n_layers*T GEMM per weight)
    int wire_w = 0;      // features per token on the wire (d, or d / maxout_k)
    size_t bn_in_g = 0, bn_in_b = 0, bn_wd = 0, bn_out_g = 0, bn_out_b = 0;
    float *p32 = nullptr, *grad = nullptr, *m = nullptr, *v = nullptr;
    bf16* p16 = nullptr;
    // delayed parameter updates: two shadow / gradient banks; p16 / grad point at the current one
    bf16* p16b[2] = {nullptr, nullptr};
    float* gradb[2] = {nullptr, nullptr};
    bool banks = false;
    int bank = 0;
    // LayerNorm gains / biases are read in fp32 from the master; with banks each
    // bank keeps its own compact copy (the master is being updated concurrently)
    // paired weight gradients: per layer, the backward's dY tensors of a deferred
    // visit (>= two sets: the pending visit's and the current one's; the
    // engine-driven executor keeps one set per trainer)
    std::vector<std::vector<Stash>> stash;
    std::vector<std::pair<size_t, size_t>> ln_slices;  // (arena offset, elements)
    std::unordered_map<size_t, size_t> ln_compact;    // arena offset -> compact offset
    size_t ln_total = 0;
    float* lnv[2] = {nullptr, nullptr};
    std::vector<Slot> slots;
    // workspaces (one visit at a time per stage)
    float *S = nullptr, *dP = nullptr, *logits = nullptr;
    void* wire_hdr = nullptr;  // device copy of this stage's swarm_wire_header
    EP dS, gy[2], dhid, dc, du, dqkv, dO, da, dlogits, wtmp;
    void* lnws = nullptr;
    std::vector<void*> allocations;
    int step = 0;
    bool fused_attn = false;  // scores+softmax in one tcgen05 kernel (csrc/attention.cu)
    bool fused_bwd = false;   // the attention backward in one kernel (csrc/attn_bwd.cu)
    bool attn_lse = false;    // forward stores log2-sum-exp, not P; the backward recomputes P
    void* abws = nullptr;     // its dQ accumulator + arrival counters (zeroed once; kernels leave it zeroed)
    // weight-gradient GEMMs run on a side stream forked/joined per layer, so they
    // fill the SMs the data-gradient chain leaves idle (GEMM wave tails)
    cudaStream_t side = nullptr;
    void* skws[2] = {nullptr, nullptr};  // GEMM stream-K scratch: visit stream, side stream
    cudaEvent_t ev_fork[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_join = nullptr;
    cudaEvent_t ev_dq = nullptr;  // dQ (side stream) complete
    EP last_dx;                   // the input gradient the last backward visit encoded (tests: "dx_last")
    std::vector<Work> lanes;      // all workspace sets when lanes are enabled (lanes[lane] is stale while active)
    int lane = 0;
    // visit profiling (bench.py's live roofline and step breakdown): event pairs
    // around each GEMM (category 0) and each other kernel call of a profiled visit
    bool prof_on = false;
    std::vector<cudaEvent_t> prof_events;
    std::vector<double> prof_flops;
    std::vector<int> prof_cat;
    std::vector<double> prof_w;  // weight of each event pair (visits of this kind per step)
    std::vector<std::string> prof_shape;  // GEMM events: "MxNxK batch epi" (per-shape table)
    std::string prof_table;               // the last read's per-shape GEMM table
    double prof_weight = 1.0;
    size_t prof_used = 0;
    double prof_last_ms[SWARM_PROF_CATEGORIES] = {};
    uint64_t prof_last_n[SWARM_PROF_CATEGORIES] = {};
};

namespace {

thread_local std::string g_err;

int fail(const std::string& m) {
    g_err = m;
    return SWARM_E_INVALID;
}

#define TRY(expr)                   \
    do {                            \
        int _rc = (expr);           \
        if (_rc != SWARM_OK) return _rc; \
    } while (0)

int dmalloc(swarm_stage* s, void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    cudaError_t e = cudaMalloc(p, bytes);
    // zero-filled once: e.g. the causal attention kernels never write P / dS past
    // a query block's causal extent, so those regions must start (and stay) zero
    if (e == cudaSuccess) e = cudaMemset(*p, 0, bytes);
    if (e != cudaSuccess) {
        g_err = std::string("stage: cudaMalloc failed: ") + cudaGetErrorString(e);
        return SWARM_E_CUDA;
    }
    s->allocations.push_back(*p);
    return SWARM_OK;
}

// the fused attention backward's workspace (zero-filled; the kernel leaves it zeroed)
int attn_ws_alloc(swarm_stage* s, void** p) {
    return dmalloc(s, p, swarm_attn_backward_workspace(s->B, s->H, s->L, s->dh));
}

template <typename T>
int alloc(swarm_stage* s, T** p, size_t count) {
    void* q = nullptr;
    TRY(dmalloc(s, &q, count * sizeof(T)));
    *p = static_cast<T*>(q);
    return SWARM_OK;
}

// an activation buffer of `count` elements of the stage's dtype
int alloc(swarm_stage* s, EP* p, size_t count) {
    void* q = nullptr;
    TRY(dmalloc(s, &q, count * s->es));
    *p = EP(q, s->es);
    return SWARM_OK;
}

// the weights the visit's GEMMs read: the bf16 shadow of the current bank, or the
// fp32 master itself in the fp32 mode
EP wts(const swarm_stage* s) { return s->f32 ? EP(s->p32, 4) : EP(s->p16, 2); }

// fp32 LayerNorm parameter at arena offset `off` as the current visit must read it
const float* ln_param(const swarm_stage* s, size_t off) {
    if (!s->banks) return s->p32 + off;
    return s->lnv[s->bank] + s->ln_compact.at(off);
}

// refresh bank b's compact LayerNorm copy from the fp32 master
int refresh_ln(swarm_stage* s, int b, cudaStream_t st) {
    for (const auto& [off, n] : s->ln_slices)
        if (cudaMemcpyAsync(s->lnv[b] + s->ln_compact.at(off), s->p32 + off, n * sizeof(float),
                            cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return SWARM_E_CUDA;
    return SWARM_OK;
}

size_t add_tensor(swarm_stage* s, const std::string& name, size_t rows, size_t cols) {
    const size_t off = s->nparams;
    s->tensors.push_back({name, off, rows, cols});
    if (rows == 1) {  // LayerNorm gain / bias
        s->ln_compact[off] = s->ln_total;
        s->ln_slices.emplace_back(off, cols);
        s->ln_total += (cols + 63) & ~size_t(63);
    }
    s->nparams += (rows * cols + 63) & ~size_t(63);  // 256-byte aligned fp32 / 128-byte bf16 slices
    return off;
}

// ------------------------------------------------------------------ GEMMs --
struct Op {  // one operand in its 2-D storage
    const void* p;
    int ld, rows, cols;
    bool mn;  // MN-major (the operand is stored transposed)
};

thread_local swarm_stage* t_prof = nullptr;  // stage whose visit is being profiled, if any
thread_local swarm_stage* t_cur = nullptr;   // stage whose visit is being issued

struct ProfScope {
    explicit ProfScope(swarm_stage* s) {
        t_prof = s->prof_on ? s : nullptr;
        t_cur = s;
    }
    ~ProfScope() { t_prof = t_cur = nullptr; }
};

// Begin / end one profiled kernel call (no-ops outside a profiled visit).
int prof_begin(int cat, cudaStream_t st) {
    swarm_stage* s = t_prof;
    if (!s) return SWARM_OK;
    while (s->prof_events.size() < 2 * (s->prof_used + 1)) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return SWARM_E_CUDA;
        s->prof_events.push_back(e);
    }
    cudaEventRecord(s->prof_events[2 * s->prof_used], st);
    s->prof_cat.push_back(cat);
    s->prof_shape.emplace_back();
    s->prof_flops.push_back(0.0);
    s->prof_w.push_back(s->prof_weight);
    return SWARM_OK;
}
void prof_end(cudaStream_t st) {
    swarm_stage* s = t_prof;
    if (!s) return;
    cudaEventRecord(s->prof_events[2 * s->prof_used + 1], st);
    s->prof_used += 1;
}
struct ProfOp {
    cudaStream_t st;
    ProfOp(int cat, cudaStream_t st_) : st(st_) { prof_begin(cat, st); }
    ~ProfOp() { prof_end(st); }
};
#define PTRY(cat, st, expr)        \
    do {                           \
        ProfOp _po((cat), (st));   \
        TRY(expr);                 \
    } while (0)

int run_gemm(swarm_gemm_args g, cudaStream_t st) {
    if (t_cur) {  // the visit stream and the side stream each own a stream-K scratch
        g.workspace = t_cur->skws[st == t_cur->side ? 1 : 0];
        g.workspace_bytes = swarm_gemm_workspace_bytes();
    }
    auto gemm = (t_cur && t_cur->f32) ? swarm_gemm_f32 : swarm_gemm_bf16;
    swarm_stage* s = t_prof;
    if (!s) return gemm(&g, st);
    TRY(prof_begin(SWARM_PROF_GEMM, st));
    const int rc = gemm(&g, st);
    prof_end(st);
    s->prof_used -= 1;  // fill in the FLOPs of the pair just closed
    double kfrac = 1.0;  // executed share of K when a causal A lets the kernel skip zero k-blocks
    const bool pair_kernel = g.m > 128 && g.n > 128;  // csrc/gemm.cu ignores k_tri there
    if (g.k_tri && !pair_kernel) {
        const int tm = (g.m + 127) / 128, kb = (g.k + 63) / 64;
        long long done = 0;
        for (int mt = 0; mt < tm; ++mt)
            done += g.k_tri == 1 ? std::min(kb, ((mt + 1) * 128 + 63) / 64) : kb - (mt * 128) / 64;
        kfrac = static_cast<double>(done) / (static_cast<double>(tm) * kb);
    }
    s->prof_flops.back() = 2.0 * g.m * g.n * static_cast<double>(g.k) * g.batch * kfrac;
    s->prof_shape.back() = std::to_string(g.m) + "x" + std::to_string(g.n) + "x" + std::to_string(g.k) + " b" +
                           std::to_string(g.batch) + " e" + std::to_string(g.epilogue) + (g.a_mn_major ? " Amn" : "") +
                           (g.b_mn_major ? " Bmn" : "") + (g.a2 ? " 2seg" : "") + (g.k_tri ? " tri" : "");
    s->prof_used += 1;
    return rc;
}

int mm(int M, int N, int K, Op a, Op b, void* d, int ldd, int epi, const void* aux, float alpha, cudaStream_t st) {
    swarm_gemm_args g{};
    g.m = M;
    g.n = N;
    g.k = K;
    g.batch = 1;
    g.bh = 1;
    g.a = a.p;
    g.lda = a.ld;
    g.a_mn_major = a.mn;
    g.a_rows = a.rows;
    g.a_cols = a.cols;
    g.b = b.p;
    g.ldb = b.ld;
    g.b_mn_major = b.mn;
    g.b_rows = b.rows;
    g.b_cols = b.cols;
    g.d = d;
    g.ldd = ldd;
    g.aux = aux;
    g.alpha = alpha;
    g.epilogue = epi;
    return run_gemm(g, st);
}

// Weight gradient over two microbatches: K = 2T split into (a, b) then (a2, b2)
int mm2(int M, int N, int K2, Op a, Op b, const void* a2, const void* b2, float* d, int ldd, cudaStream_t st) {
    swarm_gemm_args g{};
    g.m = M;
    g.n = N;
    g.k = K2;
    g.batch = 1;
    g.bh = 1;
    g.a = a.p;
    g.lda = a.ld;
    g.a_mn_major = a.mn;
    g.a_rows = a.rows;
    g.a_cols = a.cols;
    g.b = b.p;
    g.ldb = b.ld;
    g.b_mn_major = b.mn;
    g.b_rows = b.rows;
    g.b_cols = b.cols;
    g.a2 = a2;
    g.b2 = b2;
    g.d = d;
    g.ldd = ldd;
    g.alpha = 1.f;
    g.epilogue = SWARM_EPI_ACCUM_F32;
    return run_gemm(g, st);
}

// Attention GEMM batched over z = b*H + h.  Offsets in storage coordinates:
// token-major operands move by L rows per batch and dh columns per head;
// [B*H*L, L] score-like operands move by H*L rows per batch and L per head.
struct BOp {
    Op op;
    int r0, r1, c0, c1;
};

int bmm(swarm_stage* s, int M, int N, int K, BOp a, BOp b, void* d, int ldd, int rd0, int rd1, int cd0, int cd1,
        int epi, float alpha, cudaStream_t st, int k_tri = 0) {
    swarm_gemm_args g{};
    g.k_tri = s->cfg.causal ? k_tri : 0;  // causal P / dS: skip the all-zero key blocks
    g.m = M;
    g.n = N;
    g.k = K;
    g.batch = s->B * s->H;
    g.bh = s->H;
    g.a = a.op.p;
    g.lda = a.op.ld;
    g.a_mn_major = a.op.mn;
    g.a_rows = a.op.rows;
    g.a_cols = a.op.cols;
    g.ra0 = a.r0;
    g.ra1 = a.r1;
    g.ca0 = a.c0;
    g.ca1 = a.c1;
    g.b = b.op.p;
    g.ldb = b.op.ld;
    g.b_mn_major = b.op.mn;
    g.b_rows = b.op.rows;
    g.b_cols = b.op.cols;
    g.rb0 = b.r0;
    g.rb1 = b.r1;
    g.cb0 = b.c0;
    g.cb1 = b.c1;
    g.d = d;
    g.ldd = ldd;
    g.rd0 = rd0;
    g.rd1 = rd1;
    g.cd0 = cd0;
    g.cd1 = cd1;
    g.alpha = alpha;
    g.epilogue = epi;
    return run_gemm(g, st);
}

const LayerW& weights(const swarm_stage* s, int l) { return s->layers[s->cfg.shared_layers ? 0 : l]; }

// Profiled (eager) visits keep every GEMM on the visit stream so the events
// around each GEMM time that kernel alone; other visits overlap the two streams.
cudaStream_t side_of(swarm_stage* s, cudaStream_t main) { return t_prof ? main : s->side; }

// side stream waits for everything enqueued on `main` so far
int fork_side(swarm_stage* s, cudaStream_t main, int i) {
    if (t_prof) return SWARM_OK;
    if (cudaEventRecord(s->ev_fork[i], main) != cudaSuccess) return SWARM_E_CUDA;
    return cudaStreamWaitEvent(s->side, s->ev_fork[i], 0) == cudaSuccess ? SWARM_OK : SWARM_E_CUDA;
}
// main waits for the side stream up to this point (event `e` recorded on it)
int wait_side(swarm_stage* s, cudaStream_t main, cudaEvent_t e) {
    if (t_prof) return SWARM_OK;
    if (cudaEventRecord(e, s->side) != cudaSuccess) return SWARM_E_CUDA;
    return cudaStreamWaitEvent(main, e, 0) == cudaSuccess ? SWARM_OK : SWARM_E_CUDA;
}
// main waits for everything enqueued on the side stream so far
int join_side(swarm_stage* s, cudaStream_t main) {
    if (t_prof) return SWARM_OK;
    if (cudaEventRecord(s->ev_join, s->side) != cudaSuccess) return SWARM_E_CUDA;
    return cudaStreamWaitEvent(main, s->ev_join, 0) == cudaSuccess ? SWARM_OK : SWARM_E_CUDA;
}

// the forward's P V inside the attention kernel (d_head 128; SWARM_ATTN_PV=0 keeps the separate GEMM)
bool attn_pv(const swarm_stage* s) {
    static const bool on = [] {
        const char* e = getenv("SWARM_ATTN_PV");
        return !(e && e[0] == '0');
    }();
    return on && s->dh == 128;
}

bool gelu_deriv() {
    static const bool on = [] {
        const char* e = getenv("SWARM_GELU_DERIV");
        return !(e && e[0] == '0');
    }();
    return on;
}

// ---------------------------------------------------------- block forward --
int block_forward(swarm_stage* s, Act& A, EP y, const LayerW& W, cudaStream_t st) {
    const int T = s->T, d = s->d, H = s->H, dh = s->dh, F = s->F, L = s->L;
    const EP p16 = wts(s);
    PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_forward(A.x, s->dt, T, d, ln_param(s, W.ln1g), ln_param(s, W.ln1b), 1e-5, A.a, A.mu1, A.rs1, st));
    TRY(mm(T, 3 * d, d, {A.a, d, T, d, false}, {p16 + W.wqkv, d, 3 * d, d, false}, A.qkv, 3 * d,
           SWARM_EPI_STORE_BF16, nullptr, 1.f, st));
    const float scale = 1.f / std::sqrt(static_cast<float>(dh));
    if (s->attn_lse) {
        // O = softmax(scale * Q K^T) V in one kernel (scores and O in TMEM); only each row's log2-sum-exp
        // is kept for the backward
        PTRY(SWARM_PROF_ATTENTION, st, swarm_attn_forward_lse(A.qkv, A.qkv + d, A.qkv + 2 * d, 3 * d, d, s->B, H, L, dh,
                                                              scale, s->cfg.causal, A.lse, A.o, d, st));
    } else if (s->fused_attn && attn_pv(s)) {
        // P = softmax(scale * Q K^T) and O = P V in one kernel (scores and O in TMEM)
        PTRY(SWARM_PROF_ATTENTION, st, swarm_attn_forward_pv(A.qkv, A.qkv + d, A.qkv + 2 * d, 3 * d, d, s->B, H, L, dh,
                                                             scale, s->cfg.causal, A.P, A.o, d, st));
    } else if (s->fused_attn) {
        // P = softmax(scale * Q K^T) per (b, h), scores kept in TMEM
        PTRY(SWARM_PROF_ATTENTION, st, swarm_attn_scores_softmax(A.qkv, A.qkv + d, 3 * d, d, s->B, H, L, dh, scale, s->cfg.causal, A.P, st));
    } else {
        // S = scale * Q K^T per (b, h), then a row softmax
        TRY(bmm(s, L, L, dh, {{A.qkv, 3 * d, T, d, false}, L, 0, 0, dh},
                {{A.qkv + d, 3 * d, T, d, false}, L, 0, 0, dh}, s->S, L, H * L, L, 0, 0, SWARM_EPI_STORE_F32, scale,
                st));
        PTRY(SWARM_PROF_ATTENTION, st, swarm_attn_softmax_forward_ex(s->S, static_cast<size_t>(s->B) * H * L, L, s->cfg.causal, A.P, s->dt, st));
    }
    // O = P V  (V read MN-major straight from the qkv buffer), unless the attention kernel did it
    if (!(s->fused_attn && attn_pv(s)))
        TRY(bmm(s, L, dh, L, {{A.P, L, s->B * H * L, L, false}, H * L, L, 0, 0},
                {{A.qkv + 2 * d, 3 * d, T, d, true}, L, 0, 0, dh}, A.o, d, L, 0, 0, dh, SWARM_EPI_STORE_BF16, 1.f, st,
                1));
    // h = x + O Wo^T
    TRY(mm(T, d, d, {A.o, d, T, d, false}, {p16 + W.wo, d, d, d, false}, A.h, d, SWARM_EPI_RESIDUAL, A.x, 1.f, st));
    PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_forward(A.h, s->dt, T, d, ln_param(s, W.ln2g), ln_param(s, W.ln2b), 1e-5, A.c, A.mu2, A.rs2, st));
    // u = c W1^T, g = gelu(u)
    // g = gelu(c W1^T); u keeps gelu'(c W1^T) for the backward (one tanh for both;
    // SWARM_GELU_DERIV=0: u keeps the pre-activation and the backward recomputes gelu')
    TRY(mm(T, F, d, {A.c, d, T, d, false}, {p16 + W.w1, d, F, d, false}, A.g, F,
           gelu_deriv() ? SWARM_EPI_GELU_DERIV : SWARM_EPI_GELU, A.u, 1.f, st));
    // y = h + g W2^T
    TRY(mm(T, d, F, {A.g, F, T, F, false}, {p16 + W.w2, F, d, F, false}, y, d, SWARM_EPI_RESIDUAL, A.h, 1.f, st));
    return SWARM_OK;
}

// --------------------------------------------------------- block backward --
// dy: gradient w.r.t. the block output; dx: gradient w.r.t. the block input.
// The four weight-gradient GEMMs of a block: dW += dY^T X.  mode SWARM_WGRAD_NOW:
// this microbatch alone; DEFER: none (the dY tensors stay stashed for the next
// visit); PAIR: K = 2T over the pending visit's stash (first) and this one's.
struct WgradPlan {
    int mode = SWARM_WGRAD_NOW;
    const Act* prev = nullptr;  // the pending visit's activations of this layer
    const Stash* ps = nullptr;  // ... and its stashed dY
};

int wgrad(swarm_stage* s, const WgradPlan& wp, int M, int N, Op dy, Op x, Op dy_prev, Op x_prev, float* out, int ldo,
          cudaStream_t sd) {
    const int T = s->T;
    if (wp.mode == SWARM_WGRAD_DEFER) return SWARM_OK;
    if (wp.mode == SWARM_WGRAD_NOW) return mm(M, N, T, dy, x, out, ldo, SWARM_EPI_ACCUM_F32, nullptr, 1.f, sd);
    return mm2(M, N, 2 * T, dy_prev, x_prev, dy.p, x.p, out, ldo, sd);
}

// LayerNorm backward of a block: dx = LN'(dy) + dres on the visit stream, the gain /
// bias gradients (a second pass over dy and x, off the critical path) on the side
// stream after fork `fork_i`.  The fp32 mode's generic kernel computes both in one
// call on the visit stream.
int ln_backward_split(swarm_stage* s, EP dy, EP x, const float* gain, const float* mu, const float* rs, EP dres,
                      EP dx, float* dgain, float* dbias, cudaStream_t st, int fork_i) {
    const int T = s->T, d = s->d;
    if (s->f32) {
        PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_backward(dy, x, s->dt, T, d, gain, mu, rs, dres, dx, dgain, dbias,
                                                                 1, s->lnws, st));
        return SWARM_OK;
    }
    PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_backward(dy, x, s->dt, T, d, gain, mu, rs, dres, dx, nullptr,
                                                             nullptr, 1, s->lnws, st));
    TRY(fork_side(s, st, fork_i));
    cudaStream_t sd = side_of(s, st);
    PTRY(SWARM_PROF_LAYERNORM, sd, swarm_layer_norm_backward(dy, x, s->dt, T, d, gain, mu, rs, nullptr, nullptr, dgain,
                                                             dbias, 1, s->lnws, sd));
    return SWARM_OK;
}

// The unfused attention backward: score gradients (fused softmax-backward kernel, or a GEMM
// + row kernel), then dQ, dK, dV as batched GEMMs over dS / P (SWARM_ATTN_BWD_FUSED=0, d_head != 128)
int attn_backward_unfused(swarm_stage* s, const Act& A, EP dqkv, float scale, cudaStream_t st) {
    const int T = s->T, d = s->d, H = s->H, dh = s->dh, L = s->L, BHL = s->B * s->H * s->L;
    if (s->fused_attn) {
        PTRY(SWARM_PROF_ATTENTION, st, swarm_attn_scores_softmax_backward(s->dO, d, A.qkv + 2 * d, 3 * d, d, A.o, d, A.P, s->B, H, L, dh, scale,
                                               s->cfg.causal, s->dS, st));
    } else {
        TRY(bmm(s, L, L, dh, {{s->dO, d, T, d, false}, L, 0, 0, dh},
                {{A.qkv + 2 * d, 3 * d, T, d, false}, L, 0, 0, dh}, s->dP, L, H * L, L, 0, 0, SWARM_EPI_STORE_F32,
                1.f, st));
        PTRY(SWARM_PROF_ATTENTION, st, swarm_attn_softmax_backward_ex(A.P, s->dP, BHL, L, scale, s->dS, s->dt, st));
    }
    // dQ = dS K ; dK = dS^T Q ; dV = P^T dO   (all read in place, written into dqkv); dQ runs on the
    // side stream beside dK, dV (three independent GEMMs of 1.7 waves each fill each other's tails)
    TRY(fork_side(s, st, 4));
    TRY(bmm(s, L, dh, L, {{s->dS, L, BHL, L, false}, H * L, L, 0, 0}, {{A.qkv + d, 3 * d, T, d, true}, L, 0, 0, dh},
            dqkv, 3 * d, L, 0, 0, dh, SWARM_EPI_STORE_BF16, 1.f, side_of(s, st), 1));
    TRY(bmm(s, L, dh, L, {{s->dS, L, BHL, L, true}, H * L, L, 0, 0}, {{A.qkv, 3 * d, T, d, true}, L, 0, 0, dh},
            dqkv + d, 3 * d, L, 0, 0, dh, SWARM_EPI_STORE_BF16, 1.f, st, 2));
    TRY(bmm(s, L, dh, L, {{A.P, L, BHL, L, true}, H * L, L, 0, 0}, {{s->dO, d, T, d, true}, L, 0, 0, dh},
            dqkv + 2 * d, 3 * d, L, 0, 0, dh, SWARM_EPI_STORE_BF16, 1.f, st, 2));
    TRY(wait_side(s, st, s->ev_dq));  // dqkv complete on main (the dWqkv fork below then carries it to the side)
    return SWARM_OK;
}

int block_backward(swarm_stage* s, const Act& A, EP dy, EP dx, const LayerW& W, cudaStream_t st,
                   const WgradPlan& wp = WgradPlan{}, const Stash* cs = nullptr) {
    const int T = s->T, d = s->d, H = s->H, dh = s->dh, F = s->F, L = s->L;
    const EP p16 = wts(s);
    float* G = s->grad;
    cudaStream_t sd = side_of(s, st);  // weight gradients
    // dY tensors the weight gradients read: per-visit workspaces, or this layer's stash
    EP du = cs ? cs->du : s->du;
    EP dhid = cs ? cs->dhid : s->dhid;
    EP dqkv = cs ? cs->dqkv : s->dqkv;
    const Act* PA = wp.prev;
    const Stash* ps = wp.ps;
    const bool pr = wp.mode == SWARM_WGRAD_PAIR;
    // MLP: du = (dy W2) * gelu'(u); dW2 += dy^T g; dc = du W1; dW1 += du^T c
    TRY(fork_side(s, st, 0));
    TRY(wgrad(s, wp, d, F, {dy, d, T, d, true}, {A.g, F, T, F, true}, {pr ? ps->dy : nullptr, d, T, d, true},
              {pr ? PA->g : nullptr, F, T, F, true}, G + W.w2, F, sd));
    TRY(mm(T, F, d, {dy, d, T, d, false}, {p16 + W.w2, F, d, F, true}, du, F,
           gelu_deriv() ? SWARM_EPI_MUL : SWARM_EPI_DGELU, A.u, 1.f, st));
    TRY(fork_side(s, st, 1));
    TRY(wgrad(s, wp, F, d, {du, F, T, F, true}, {A.c, d, T, d, true}, {pr ? ps->du : nullptr, F, T, F, true},
              {pr ? PA->c : nullptr, d, T, d, true}, G + W.w1, d, sd));
    TRY(mm(T, d, F, {du, F, T, F, false}, {p16 + W.w1, d, F, d, true}, s->dc, d, SWARM_EPI_STORE_BF16, nullptr, 1.f,
           st));
    // dh = LN2'(dc) + dy on the visit stream; LN2's gain / bias gradients (a second pass
    // over dc and h, off the critical path) on the side stream
    TRY(ln_backward_split(s, s->dc, A.h, ln_param(s, W.ln2g), A.mu2, A.rs2, dy, dhid, G + W.ln2g, G + W.ln2b, st, 5));
    // attention output projection
    TRY(fork_side(s, st, 2));
    TRY(wgrad(s, wp, d, d, {dhid, d, T, d, true}, {A.o, d, T, d, true}, {pr ? ps->dhid : nullptr, d, T, d, true},
              {pr ? PA->o : nullptr, d, T, d, true}, G + W.wo, d, sd));
    TRY(mm(T, d, d, {dhid, d, T, d, false}, {p16 + W.wo, d, d, d, true}, s->dO, d, SWARM_EPI_STORE_BF16, nullptr, 1.f,
           st));
    // dP = dO V^T ; dS = scale * P (dP - rowsum(P dP))
    const float scale = 1.f / std::sqrt(static_cast<float>(dh));
    if (s->attn_lse) {
        // the attention backward with P recomputed on chip from the forward's log2-sum-exp
        PTRY(SWARM_PROF_ATTENTION, st, swarm_attn_backward_lse(s->dO, d, A.qkv, 3 * d, 3 * d, d, 2 * d, A.o, d, A.lse,
                                                               s->B, H, L, dh, scale, s->cfg.causal, dqkv, 3 * d, d,
                                                               2 * d, s->abws, st));
    } else if (s->fused_bwd) {
        // the whole attention backward in one kernel: dP, dS on chip, dQ | dK | dV into dqkv
        PTRY(SWARM_PROF_ATTENTION, st, swarm_attn_backward(s->dO, d, A.qkv, 3 * d, 3 * d, d, 2 * d, A.o, d, A.P, s->B, H, L,
                                                           dh, scale, s->cfg.causal, dqkv, 3 * d, d, 2 * d, s->abws,
                                                           st));
    } else {
        TRY(attn_backward_unfused(s, A, dqkv, scale, st));
    }
    // da = dqkv Wqkv ; dWqkv += dqkv^T a
    TRY(fork_side(s, st, 3));
    TRY(wgrad(s, wp, 3 * d, d, {dqkv, 3 * d, T, 3 * d, true}, {A.a, d, T, d, true},
              {pr ? ps->dqkv : nullptr, 3 * d, T, 3 * d, true}, {pr ? PA->a : nullptr, d, T, d, true}, G + W.wqkv, d,
              sd));
    TRY(mm(T, d, 3 * d, {dqkv, 3 * d, T, 3 * d, false}, {p16 + W.wqkv, d, 3 * d, d, true}, s->da, d,
           SWARM_EPI_STORE_BF16, nullptr, 1.f, st));
    // dx = LN1'(da) + dh; LN1's gain / bias gradients on the side stream
    TRY(ln_backward_split(s, s->da, A.x, ln_param(s, W.ln1g), A.mu1, A.rs1, dhid, dx, G + W.ln1g, G + W.ln1b, st, 6));
    // the next layer overwrites the workspaces the weight gradients read
    return join_side(s, st);
}

// Wire message: payload (int8 codes, 16-B padded, then fp32 per-block scales;
// or raw bf16) followed by a 16-byte swarm_wire_header.
size_t wire_payload_bytes(const swarm_stage* s) {
    const size_t n = static_cast<size_t>(s->T) * s->wire_w;
    if (s->cfg.wire == SWARM_WIRE_INT8) {
        const size_t bs = static_cast<size_t>(s->cfg.block_size);
        return ((n + 15) & ~size_t(15)) + (((n + bs - 1) / bs) * sizeof(float) + 15) / 16 * 16;
    }
    return (n * s->es + 15) / 16 * 16;  // raw activations in the stage's dtype
}

size_t wire_bytes(const swarm_stage* s) { return wire_payload_bytes(s) + sizeof(swarm_wire_header); }

int wire_decode(swarm_stage* s, const void* msg, EP out, cudaStream_t st) {
    const size_t n = static_cast<size_t>(s->T) * s->wire_w;
    if (s->cfg.wire == SWARM_WIRE_INT8) {
        const int8_t* codes = static_cast<const int8_t*>(msg);
        const void* scales = static_cast<const char*>(msg) + ((n + 15) & ~size_t(15));
        return swarm_dequantize_blockwise(codes, scales, SWARM_DTYPE_F32, n, s->cfg.block_size, out, s->dt,
                                          st);
    }
    const cudaError_t e = cudaMemcpyAsync(out, msg, n * s->es, cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SWARM_OK : SWARM_E_CUDA;
}

int wire_encode(swarm_stage* s, EP x, void* msg, cudaStream_t st) {
    const size_t n = static_cast<size_t>(s->T) * s->wire_w;
    // header first (a 16-byte device-to-device copy of the stage's prebuilt header)
    if (cudaMemcpyAsync(static_cast<char*>(msg) + wire_payload_bytes(s), s->wire_hdr, sizeof(swarm_wire_header),
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return SWARM_E_CUDA;
    if (s->cfg.wire == SWARM_WIRE_INT8) {
        int8_t* codes = static_cast<int8_t*>(msg);
        void* scales = static_cast<char*>(msg) + ((n + 15) & ~size_t(15));
        return swarm_quantize_blockwise(x, s->dt, n, s->cfg.block_size, codes, scales, nullptr, st);
    }
    const cudaError_t e = cudaMemcpyAsync(msg, x, n * s->es, cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SWARM_OK : SWARM_E_CUDA;
}

int init_params(swarm_stage* s, cudaStream_t st) {
    const uint64_t base = s->cfg.seed * 1000003ull;
    if (cudaMemsetAsync(s->p32, 0, s->nparams * 4, st) != cudaSuccess) return SWARM_E_CUDA;  // alignment padding
    for (size_t i = 0; i < s->tensors.size(); ++i) {
        const auto& t = s->tensors[i];
        const size_t n = t.rows * t.cols;
        const bool is_gain = t.name.find("_g") != std::string::npos && t.rows == 1;
        const bool is_bias = t.name.find("_b") != std::string::npos && t.rows == 1;
        const float mean = is_gain ? 1.f : 0.f;
        const float stdv = (is_gain || is_bias) ? 0.f : s->cfg.init_std;
        TRY(swarm_fill_normal(s->p32 + t.off, n, mean, stdv, base + i, st));
    }
    if (!s->f32) TRY(swarm_cast_f32_bf16(s->p32, s->p16, s->nparams, st));
    if (cudaMemsetAsync(s->grad, 0, s->nparams * 4, st) != cudaSuccess ||
        cudaMemsetAsync(s->m, 0, s->nparams * 4, st) != cudaSuccess ||
        cudaMemsetAsync(s->v, 0, s->nparams * 4, st) != cudaSuccess)
        return SWARM_E_CUDA;
    return SWARM_OK;
}

int create(const swarm_stage_config* c, swarm_stage* s) {
    s->cfg = *c;
    s->f32 = c->fp32 != 0;
    s->es = s->f32 ? 4 : 2;
    s->dt = s->f32 ? SWARM_DTYPE_F32 : SWARM_DTYPE_BF16;
    s->d = c->d_model;
    s->H = c->n_heads;
    s->F = c->d_ffn;
    s->L = c->seq_len;
    s->B = c->micro_batch;
    s->V = c->vocab;
    s->T = s->B * s->L;
    if (s->d <= 0 || s->H <= 0 || s->d % s->H || s->F <= 0 || s->L <= 0 || s->B <= 0 || c->n_layers <= 0 ||
        c->max_slots <= 0)
        return fail("stage: bad shape");
    s->dh = s->d / s->H;
    if (s->d % 64 || s->F % 64 || s->dh % 64 || s->L % 64) return fail("stage: d, d_ffn, d_head, seq_len must be multiples of 64");
    if (s->L > 1024) return fail("stage: seq_len > 1024 unsupported");
    if ((c->is_first || c->is_last) && (s->V <= 0 || s->V % 8)) return fail("stage: vocab must be a positive multiple of 8");
    if (c->wire == SWARM_WIRE_INT8 && c->block_size <= 0) return fail("stage: block_size must be positive");
    const int d = s->d, F = s->F;
    // parameter layout
    s->bneck = c->maxout_k > 1;
    s->stacked = c->shared_layers && c->n_layers > 1;
    if (s->bneck && (d % c->maxout_k || (d / c->maxout_k) % 64 || c->maxout_k > 255))
        return fail("stage: maxout_k must divide d_model into a multiple of 64");
    s->wire_w = s->bneck ? d / c->maxout_k : d;
    if (c->is_first) s->emb = add_tensor(s, "embedding", s->V, d);
    if (s->bneck && !c->is_first) {  // receiving side of the bottleneck
        s->bn_in_g = add_tensor(s, "bneck_in_ln_g", 1, s->wire_w);
        s->bn_in_b = add_tensor(s, "bneck_in_ln_b", 1, s->wire_w);
        s->bn_wd = add_tensor(s, "bneck_wd", d, s->wire_w);
    }
    const int nw = c->shared_layers ? 1 : c->n_layers;
    for (int l = 0; l < nw; ++l) {
        const std::string p = "layer" + std::to_string(l) + ".";
        LayerW w{};
        w.wqkv = add_tensor(s, p + "wqkv", 3 * d, d);
        w.wo = add_tensor(s, p + "wo", d, d);
        w.w1 = add_tensor(s, p + "w1", F, d);
        w.w2 = add_tensor(s, p + "w2", d, F);
        w.ln1g = add_tensor(s, p + "ln1_g", 1, d);
        w.ln1b = add_tensor(s, p + "ln1_b", 1, d);
        w.ln2g = add_tensor(s, p + "ln2_g", 1, d);
        w.ln2b = add_tensor(s, p + "ln2_b", 1, d);
        s->layers.push_back(w);
    }
    if (s->bneck && !c->is_last) {  // sending side
        s->bn_out_g = add_tensor(s, "bneck_out_ln_g", 1, d);
        s->bn_out_b = add_tensor(s, "bneck_out_ln_b", 1, d);
    }
    if (c->is_last) {
        s->lnfg = add_tensor(s, "lnf_g", 1, d);
        s->lnfb = add_tensor(s, "lnf_b", 1, d);
        s->head = add_tensor(s, "head", s->V, d);
    }
    TRY(alloc(s, &s->p32, s->nparams));
    TRY(alloc(s, &s->grad, s->nparams));
    TRY(alloc(s, &s->m, s->nparams));
    TRY(alloc(s, &s->v, s->nparams));
    if (!s->f32) TRY(alloc(s, &s->p16, s->nparams));
    // activation slots
    const size_t T = s->T, Td = T * d, TF = T * F, BHLL = static_cast<size_t>(s->B) * s->H * s->L * s->L;
    // attention path: fused score kernels; the one-kernel backward (d_head 128); with it, the
    // forward stores each row's log2-sum-exp instead of P and the backward recomputes P on chip
    // (SWARM_ATTN_FUSED / SWARM_ATTN_BWD_FUSED / SWARM_ATTN_LSE = 0 turn each off)
    {
        const char* e = getenv("SWARM_ATTN_FUSED");
        s->fused_attn = !s->f32 && !(e && e[0] == '0') && s->L % 128 == 0 && s->L <= 512 && s->dh % 64 == 0 && s->dh <= 128;
    }
    {
        const char* e = getenv("SWARM_ATTN_BWD_FUSED");
        s->fused_bwd = s->fused_attn && s->dh == 128 && !(e && e[0] == '0');
    }
    {
        const char* e = getenv("SWARM_ATTN_LSE");
        s->attn_lse = s->fused_bwd && attn_pv(s) && !(e && e[0] == '0');
    }
    s->slots.resize(c->max_slots);
    // layer-shared stages keep the weight-gradient inputs (a, o, c, g) of all
    // applications stacked in application order, so one GEMM with K = n_layers * T
    // computes a shared weight's gradient (stacked_wgrad)
    const size_t nl = static_cast<size_t>(c->n_layers);
    for (auto& sl : s->slots) {
        sl.layer.resize(c->n_layers);
        EP sa, so, sc, sg;
        if (s->stacked) {
            TRY(alloc(s, &sa, nl * Td));
            TRY(alloc(s, &so, nl * Td));
            TRY(alloc(s, &sc, nl * Td));
            TRY(alloc(s, &sg, nl * TF));
        }
        for (size_t l = 0; l < nl; ++l) {
            Act& A = sl.layer[l];
            TRY(alloc(s, &A.x, Td));
            if (s->stacked) A.a = sa + l * Td;
            else TRY(alloc(s, &A.a, Td));
            TRY(alloc(s, &A.qkv, 3 * Td));
            if (s->attn_lse) TRY(alloc(s, &A.lse, static_cast<size_t>(s->B) * s->H * s->L));
            else TRY(alloc(s, &A.P, BHLL));
            if (s->stacked) A.o = so + l * Td;
            else TRY(alloc(s, &A.o, Td));
            TRY(alloc(s, &A.h, Td));
            if (s->stacked) A.c = sc + l * Td;
            else TRY(alloc(s, &A.c, Td));
            TRY(alloc(s, &A.u, TF));
            if (s->stacked) A.g = sg + l * TF;
            else TRY(alloc(s, &A.g, TF));
            TRY(alloc(s, &A.mu1, T));
            TRY(alloc(s, &A.rs1, T));
            TRY(alloc(s, &A.mu2, T));
            TRY(alloc(s, &A.rs2, T));
        }
        TRY(alloc(s, &sl.out, Td));
        if (c->is_last) {
            TRY(alloc(s, &sl.xf, Td));
            TRY(alloc(s, &sl.muf, T));
            TRY(alloc(s, &sl.rsf, T));
            TRY(alloc(s, &sl.dxf, Td));
        }
        if (c->is_first) TRY(alloc(s, &sl.tokens, T));
        if (s->bneck && !c->is_last) {
            TRY(alloc(s, &sl.z, Td));
            TRY(alloc(s, &sl.muc, T));
            TRY(alloc(s, &sl.rsc, T));
            TRY(alloc(s, &sl.mo, T * s->wire_w));
            TRY(alloc(s, &sl.am, T * s->wire_w));
        }
        if (s->bneck && !c->is_first) {
            TRY(alloc(s, &sl.mi, T * s->wire_w));
            TRY(alloc(s, &sl.ni, T * s->wire_w));
            TRY(alloc(s, &sl.mud, T));
            TRY(alloc(s, &sl.rsd, T));
        }
    }
    // workspaces (fp32 scores only for the unfused attention path)
    if (!s->fused_attn) {
        TRY(alloc(s, &s->S, BHLL));
        TRY(alloc(s, &s->dP, BHLL));
    }
    if (s->fused_bwd) TRY(attn_ws_alloc(s, &s->abws));
    else TRY(alloc(s, &s->dS, BHLL));
    TRY(alloc(s, &s->gy[0], Td));
    TRY(alloc(s, &s->gy[1], Td));
    TRY(alloc(s, &s->dhid, Td));
    TRY(alloc(s, &s->dc, Td));
    TRY(alloc(s, &s->du, TF));
    TRY(alloc(s, &s->dqkv, 3 * Td));
    TRY(alloc(s, &s->dO, Td));
    TRY(alloc(s, &s->da, Td));
    TRY(alloc(s, &s->wtmp, T * s->wire_w));
    {
        swarm_wire_header h{};
        h.magic = SWARM_WIRE_MAGIC;
        h.n_elems = static_cast<uint32_t>(T * s->wire_w);
        h.block_size = static_cast<uint32_t>(c->block_size);
        h.kind = static_cast<uint8_t>(c->wire);
        h.maxout_k = static_cast<uint8_t>(s->bneck ? c->maxout_k : 1);
        h.version = 1;
        TRY(dmalloc(s, &s->wire_hdr, sizeof(h)));
        if (cudaMemcpy(s->wire_hdr, &h, sizeof(h), cudaMemcpyHostToDevice) != cudaSuccess) return SWARM_E_CUDA;
    }
    TRY(dmalloc(s, &s->lnws, swarm_layer_norm_backward_workspace(T, d)));
    if (c->is_last) {
        TRY(alloc(s, &s->logits, T * s->V));
        TRY(alloc(s, &s->dlogits, T * s->V));
    }
    if (cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking) != cudaSuccess) return SWARM_E_CUDA;
    for (void*& w : s->skws) {
        TRY(dmalloc(s, &w, swarm_gemm_workspace_bytes()));
        if (cudaMemset(w, 0, swarm_gemm_workspace_bytes()) != cudaSuccess) return SWARM_E_CUDA;
    }
    for (auto& e : s->ev_fork)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SWARM_E_CUDA;
    if (cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming) != cudaSuccess) return SWARM_E_CUDA;
    if (cudaEventCreateWithFlags(&s->ev_dq, cudaEventDisableTiming) != cudaSuccess) return SWARM_E_CUDA;
    TRY(init_params(s, nullptr));
    if (cudaStreamSynchronize(nullptr) != cudaSuccess) return SWARM_E_CUDA;
    return SWARM_OK;
}

}  // namespace

namespace {
#define SWARM_WORK_FIELDS(X) X(S) X(dP) X(logits) X(dS) X(dhid) X(dc) X(du) X(dqkv) X(dO) X(da) X(dlogits) X(wtmp) \
    X(lnws) X(abws) X(side) X(ev_join) X(ev_dq)
void work_save(const swarm_stage* s, Work& w) {
#define X(f) w.f = s->f;
    SWARM_WORK_FIELDS(X)
#undef X
    for (int i = 0; i < 2; ++i) w.gy[i] = s->gy[i], w.skws[i] = s->skws[i];
    for (int i = 0; i < 7; ++i) w.ev_fork[i] = s->ev_fork[i];
}
void work_load(swarm_stage* s, const Work& w) {
#define X(f) s->f = w.f;
    SWARM_WORK_FIELDS(X)
#undef X
    for (int i = 0; i < 2; ++i) s->gy[i] = w.gy[i], s->skws[i] = w.skws[i];
    for (int i = 0; i < 7; ++i) s->ev_fork[i] = w.ev_fork[i];
}
// a second (third, ...) workspace set, sized as create() sizes the first
int work_alloc(swarm_stage* s, Work& w) {
    const size_t T = s->T, d = s->d, Td = T * d, TF = T * s->F, BHLL = static_cast<size_t>(s->B) * s->H * s->L * s->L;
    if (!s->fused_attn) {
        TRY(alloc(s, &w.S, BHLL));
        TRY(alloc(s, &w.dP, BHLL));
    }
    if (s->fused_bwd) TRY(attn_ws_alloc(s, &w.abws));
    else TRY(alloc(s, &w.dS, BHLL));
    TRY(alloc(s, &w.gy[0], Td));
    TRY(alloc(s, &w.gy[1], Td));
    TRY(alloc(s, &w.dhid, Td));
    TRY(alloc(s, &w.dc, Td));
    TRY(alloc(s, &w.du, TF));
    TRY(alloc(s, &w.dqkv, 3 * Td));
    TRY(alloc(s, &w.dO, Td));
    TRY(alloc(s, &w.da, Td));
    TRY(alloc(s, &w.wtmp, T * s->wire_w));
    TRY(dmalloc(s, &w.lnws, swarm_layer_norm_backward_workspace(T, d)));
    if (s->cfg.is_last) {
        TRY(alloc(s, &w.logits, T * s->V));
        TRY(alloc(s, &w.dlogits, T * s->V));
    }
    if (cudaStreamCreateWithFlags(&w.side, cudaStreamNonBlocking) != cudaSuccess) return SWARM_E_CUDA;
    for (void*& x : w.skws) {
        TRY(dmalloc(s, &x, swarm_gemm_workspace_bytes()));
        if (cudaMemset(x, 0, swarm_gemm_workspace_bytes()) != cudaSuccess) return SWARM_E_CUDA;
    }
    for (auto& e : w.ev_fork)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SWARM_E_CUDA;
    if (cudaEventCreateWithFlags(&w.ev_join, cudaEventDisableTiming) != cudaSuccess) return SWARM_E_CUDA;
    if (cudaEventCreateWithFlags(&w.ev_dq, cudaEventDisableTiming) != cudaSuccess) return SWARM_E_CUDA;
    return cudaDeviceSynchronize() == cudaSuccess ? SWARM_OK : SWARM_E_CUDA;
}
}  // namespace

extern "C" {

int swarm_stage_create(const swarm_stage_config* cfg, swarm_stage_t* out) {
    if (!cfg || !out) return fail("stage: null argument");
    auto* s = new (std::nothrow) swarm_stage;
    if (!s) return fail("stage: out of host memory");
    const int rc = create(cfg, s);
    if (rc != SWARM_OK) {
        swarm_stage_destroy(s);
        return rc;
    }
    *out = s;
    return SWARM_OK;
}

void swarm_stage_destroy(swarm_stage_t s) {
    if (!s) return;
    cudaDeviceSynchronize();
    for (cudaEvent_t e : s->prof_events) cudaEventDestroy(e);
    if (!s->lanes.empty()) work_save(s, s->lanes[s->lane]);
    else s->lanes.resize(1), work_save(s, s->lanes[0]);
    for (Work& w : s->lanes) {
        for (cudaEvent_t e : w.ev_fork)
            if (e) cudaEventDestroy(e);
        if (w.ev_join) cudaEventDestroy(w.ev_join);
        if (w.ev_dq) cudaEventDestroy(w.ev_dq);
        if (w.side) cudaStreamDestroy(w.side);
    }
    for (void* p : s->allocations) cudaFree(p);
    delete s;
}

size_t swarm_stage_wire_bytes(swarm_stage_t s) { return wire_bytes(s); }

int swarm_wire_parse_header(const void* header, uint32_t* n_elems, uint32_t* block_size, int* kind, int* maxout_k) {
    const auto* h = static_cast<const swarm_wire_header*>(header);
    if (!h || h->magic != SWARM_WIRE_MAGIC || h->version != 1) return fail("wire: bad header");
    if (n_elems) *n_elems = h->n_elems;
    if (block_size) *block_size = h->block_size;
    if (kind) *kind = h->kind;
    if (maxout_k) *maxout_k = h->maxout_k;
    return SWARM_OK;
}

void swarm_stage_profile(swarm_stage_t s, int enable) { s->prof_on = enable != 0; }
void swarm_stage_profile_weight(swarm_stage_t s, double weight) { s->prof_weight = weight; }

int swarm_stage_profile_read(swarm_stage_t s, double* gemm_ms, double* gemm_flops, uint64_t* gemm_launches) {
    double fl = 0.0;
    double ms[SWARM_PROF_CATEGORIES] = {};
    uint64_t n[SWARM_PROF_CATEGORIES] = {};
    std::map<std::string, std::tuple<double, double, int>> shapes;  // key -> (ms, flops, launches)
    for (size_t i = 0; i < s->prof_used; ++i) {
        if (cudaEventSynchronize(s->prof_events[2 * i + 1]) != cudaSuccess) return SWARM_E_CUDA;
        float e = 0.f;
        cudaEventElapsedTime(&e, s->prof_events[2 * i], s->prof_events[2 * i + 1]);
        ms[s->prof_cat[i]] += e * s->prof_w[i];
        n[s->prof_cat[i]] += 1;
        fl += s->prof_flops[i] * s->prof_w[i];
        if (s->prof_cat[i] == SWARM_PROF_GEMM) {
            auto& t = shapes[s->prof_shape[i]];
            std::get<0>(t) += e * s->prof_w[i];
            std::get<1>(t) += s->prof_flops[i] * s->prof_w[i];
            std::get<2>(t) += 1;
        }
    }
    if (gemm_ms) *gemm_ms = ms[SWARM_PROF_GEMM];
    if (gemm_flops) *gemm_flops = fl;
    if (gemm_launches) *gemm_launches = n[SWARM_PROF_GEMM];
    for (int c = 0; c < SWARM_PROF_CATEGORIES; ++c) {
        s->prof_last_ms[c] = ms[c];
        s->prof_last_n[c] = n[c];
    }
    s->prof_used = 0;
    s->prof_flops.clear();
    s->prof_cat.clear();
    s->prof_w.clear();
    s->prof_shape.clear();
    s->prof_table.clear();
    for (const auto& [k, t] : shapes) {  // "shape;ms;flops;launches" lines
        char line[256];
        snprintf(line, sizeof(line), "%s;%.6f;%.6e;%d\n", k.c_str(), std::get<0>(t), std::get<1>(t), std::get<2>(t));
        s->prof_table += line;
    }
    return SWARM_OK;
}

const char* swarm_stage_profile_shapes(swarm_stage_t s) { return s->prof_table.c_str(); }

void swarm_stage_profile_breakdown(swarm_stage_t s, double* ms, uint64_t* launches) {
    for (int c = 0; c < SWARM_PROF_CATEGORIES; ++c) {
        if (ms) ms[c] = s->prof_last_ms[c];
        if (launches) launches[c] = s->prof_last_n[c];
    }
}
size_t swarm_stage_num_params(swarm_stage_t s) { return s->nparams; }
float* swarm_stage_grads(swarm_stage_t s) { return s->grad; }
float* swarm_stage_params(swarm_stage_t s) { return s->p32; }
void* swarm_stage_params_bf16(swarm_stage_t s) { return s->p16; }

int swarm_stage_sync_shadow(swarm_stage_t s, swarm_stream_t stream) {
    if (s->f32) return SWARM_OK;  // the GEMMs read the fp32 master itself
    if (!s->banks) return swarm_cast_f32_bf16(s->p32, s->p16, s->nparams, stream);
    for (bf16* p : s->p16b) TRY(swarm_cast_f32_bf16(s->p32, p, s->nparams, stream));
    for (int b = 0; b < 2; ++b) TRY(refresh_ln(s, b, static_cast<cudaStream_t>(stream)));
    return SWARM_OK;
}

int swarm_stage_enable_banks(swarm_stage_t s, swarm_stream_t stream) {
    if (s->banks) return SWARM_OK;
    if (s->f32) return fail("enable_banks: delayed-update banks need the bf16 mode");
    s->p16b[0] = s->p16;
    s->gradb[0] = s->grad;
    TRY(alloc(s, &s->p16b[1], s->nparams));
    TRY(alloc(s, &s->gradb[1], s->nparams));  // zero-filled by dmalloc
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (float*& l : s->lnv) TRY(alloc(s, &l, s->ln_total));
    TRY(refresh_ln(s, 0, st));
    TRY(refresh_ln(s, 1, st));
    if (cudaMemcpyAsync(s->p16b[1], s->p16b[0], s->nparams * sizeof(bf16), cudaMemcpyDeviceToDevice, st) !=
        cudaSuccess)
        return SWARM_E_CUDA;
    s->banks = true;
    return SWARM_OK;
}

int swarm_stage_set_bank(swarm_stage_t s, int bank) {
    if (bank < 0 || bank > 1 || (bank == 1 && !s->banks)) return fail("set_bank: bank must be 0, or 1 after enable_banks");
    s->bank = bank;
    s->p16 = s->banks ? s->p16b[bank] : s->p16;
    s->grad = s->banks ? s->gradb[bank] : s->grad;
    return SWARM_OK;
}

void* swarm_stage_params_bf16_bank(swarm_stage_t s, int bank) {
    if (!s->banks) return bank == 0 ? s->p16 : nullptr;
    return (bank == 0 || bank == 1) ? s->p16b[bank] : nullptr;
}

float* swarm_stage_grads_bank(swarm_stage_t s, int bank) {
    if (!s->banks) return bank == 0 ? s->grad : nullptr;
    return (bank == 0 || bank == 1) ? s->gradb[bank] : nullptr;
}

int swarm_stage_optimizer_step_bank(swarm_stage_t s, int bank, float grad_scale, swarm_stream_t stream) {
    if (!s->banks) return bank == 0 ? swarm_stage_optimizer_step(s, grad_scale, stream) : fail("optimizer_step_bank: no banks");
    if (bank < 0 || bank > 1) return fail("optimizer_step_bank: bank must be 0 or 1");
    s->step += 1;
    const auto& c = s->cfg;
    TRY(swarm_adamw_step(s->p32, s->p16b[bank], s->gradb[bank], s->m, s->v, s->nparams, c.lr, c.beta1, c.beta2,
                         c.eps, c.weight_decay, s->step, grad_scale, 1, stream));
    return refresh_ln(s, bank, static_cast<cudaStream_t>(stream));
}

int swarm_stage_param_info(swarm_stage_t s, int index, const char** name, size_t* offset, size_t* rows, size_t* cols) {
    if (index < 0 || index >= static_cast<int>(s->tensors.size())) return SWARM_E_INVALID;
    const auto& t = s->tensors[index];
    if (name) *name = t.name.c_str();
    if (offset) *offset = t.off;
    if (rows) *rows = t.rows;
    if (cols) *cols = t.cols;
    return SWARM_OK;
}

int swarm_stage_activation(swarm_stage_t s, int slot, int layer, const char* name, void** ptr, size_t* numel) {
    if (slot < 0 || slot >= static_cast<int>(s->slots.size())) return fail("activation: bad slot");
    Slot& sl = s->slots[slot];
    const size_t Td = static_cast<size_t>(s->T) * s->d;
    const std::string n = name ? name : "";
    if (n == "out") return *ptr = sl.out, *numel = Td, SWARM_OK;
    if (n == "xf") return *ptr = sl.xf, *numel = sl.xf ? Td : 0, SWARM_OK;
    if (n == "dxf") return *ptr = sl.dxf, *numel = sl.dxf ? Td : 0, SWARM_OK;
    if (n == "dx_last") return *ptr = s->last_dx, *numel = s->last_dx ? static_cast<size_t>(s->T) * s->wire_w : 0, SWARM_OK;
    if (n == "wire_in") return *ptr = s->bneck ? sl.mi : sl.layer[0].x, *numel = static_cast<size_t>(s->T) * s->wire_w, SWARM_OK;
    if (n == "wire_out") return *ptr = s->bneck ? sl.mo : sl.out, *numel = static_cast<size_t>(s->T) * s->wire_w, SWARM_OK;
    if (layer < 0 || layer >= static_cast<int>(sl.layer.size())) return fail("activation: bad layer");
    Act& A = sl.layer[layer];
    const size_t TF = static_cast<size_t>(s->T) * s->F;
    struct {
        const char* k;
        void* p;
        size_t n;
    } table[] = {{"x", A.x, Td}, {"a", A.a, Td}, {"qkv", A.qkv, 3 * Td},
                 {"P", A.P, A.P ? static_cast<size_t>(s->B) * s->H * s->L * s->L : 0},
                 {"lse", A.lse, A.lse ? static_cast<size_t>(s->B) * s->H * s->L : 0},
                 {"o", A.o, Td}, {"h", A.h, Td}, {"c", A.c, Td}, {"u", A.u, TF}, {"g", A.g, TF}};
    for (auto& e : table)
        if (n == e.k) return *ptr = e.p, *numel = e.n, SWARM_OK;
    return fail("activation: unknown name " + n);
}

int swarm_stage_forward(swarm_stage_t s, int slot, const void* in, const int32_t* targets, void* out, float* loss_sum,
                        float loss_scale, swarm_stream_t stream) {
    if (slot < 0 || slot >= static_cast<int>(s->slots.size())) return fail("forward: bad slot");
    if (!in) return fail("forward: null input");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ProfScope prof(s);
    Slot& sl = s->slots[slot];
    const int T = s->T, d = s->d, n = s->cfg.n_layers;
    if (s->cfg.is_first) {
        if (cudaMemcpyAsync(sl.tokens, in, T * sizeof(int32_t), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return SWARM_E_CUDA;
        PTRY(SWARM_PROF_OTHER, st, swarm_embedding_forward_ex(sl.tokens, T, wts(s) + s->emb, s->V, d, sl.layer[0].x, s->dt, st));
    } else if (s->bneck) {
        // receiver: x0 = LN_d(dequant(wire)) W_d^T   (d/k -> d)
        const int w = s->wire_w;
        PTRY(SWARM_PROF_OTHER, st, wire_decode(s, in, sl.mi, st));
        PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_forward(sl.mi, s->dt, T, w, ln_param(s, s->bn_in_g), ln_param(s, s->bn_in_b), 1e-5,
                                     sl.ni, sl.mud, sl.rsd, st));
        TRY(mm(T, d, w, {sl.ni, w, T, w, false}, {wts(s) + s->bn_wd, w, d, w, false}, sl.layer[0].x, d,
               SWARM_EPI_STORE_BF16, nullptr, 1.f, st));
    } else {
        PTRY(SWARM_PROF_OTHER, st, wire_decode(s, in, sl.layer[0].x, st));
    }
    for (int l = 0; l < n; ++l) {
        EP y = (l + 1 < n) ? sl.layer[l + 1].x : sl.out;
        TRY(block_forward(s, sl.layer[l], y, weights(s, l), st));
    }
    if (!s->cfg.is_last) {
        if (!out) return fail("forward: null output message");
        if (!s->bneck) {
            ProfOp po(SWARM_PROF_OTHER, st);
            return wire_encode(s, sl.out, out, st);
        }
        // sender: wire = int8(maxout_k(LN_c(out)))
        PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_forward(sl.out, s->dt, T, d, ln_param(s, s->bn_out_g), ln_param(s, s->bn_out_b), 1e-5,
                                     sl.z, sl.muc, sl.rsc, st));
        PTRY(SWARM_PROF_OTHER, st, swarm_maxout_forward(sl.z, s->dt, static_cast<size_t>(T) * d, s->cfg.maxout_k, sl.mo, sl.am,
                                 st));
        ProfOp po(SWARM_PROF_OTHER, st);
        return wire_encode(s, sl.mo, out, st);
    }
    if (!targets) return fail("forward: last stage needs targets");
    // final LN + LM head + cross-entropy, with the head's backward fused in
    PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_forward(sl.out, s->dt, T, d, ln_param(s, s->lnfg), ln_param(s, s->lnfb), 1e-5, sl.xf,
                                 sl.muf, sl.rsf, st));
    TRY(mm(T, s->V, d, {sl.xf, d, T, d, false}, {wts(s) + s->head, d, s->V, d, false}, s->logits, s->V,
           SWARM_EPI_STORE_F32, nullptr, 1.f, st));
    PTRY(SWARM_PROF_OTHER, st, swarm_cross_entropy_ex(s->logits, targets, T, s->V, loss_scale, loss_sum, s->dlogits, s->dt, st));
    TRY(fork_side(s, st, 0));
    TRY(mm(s->V, d, T, {s->dlogits, s->V, T, s->V, true}, {sl.xf, d, T, d, true}, s->grad + s->head, d,
           SWARM_EPI_ACCUM_F32, nullptr, 1.f, side_of(s, st)));
    TRY(mm(T, d, s->V, {s->dlogits, s->V, T, s->V, false}, {wts(s) + s->head, d, s->V, d, true}, sl.dxf, d,
           SWARM_EPI_STORE_BF16, nullptr, 1.f, st));
    return join_side(s, st);
}

int swarm_stage_enable_lanes(swarm_stage_t s, int n) {
    if (!s || n < 1) return fail("enable_lanes: need at least one lane");
    if (!s->lanes.empty()) return static_cast<int>(s->lanes.size()) >= n ? SWARM_OK : fail("enable_lanes: already enabled");
    if (n == 1) return SWARM_OK;
    // build every set first and commit only when all succeeded: a failed call leaves the
    // stage without lanes (its device buffers stay owned by s->allocations)
    std::vector<Work> sets(n);
    work_save(s, sets[0]);
    for (int i = 1; i < n; ++i) {
        const int rc = work_alloc(s, sets[i]);
        if (rc != SWARM_OK) {
            for (int j = 1; j <= i; ++j) {
                for (cudaEvent_t& e : sets[j].ev_fork)
                    if (e) cudaEventDestroy(e);
                if (sets[j].ev_join) cudaEventDestroy(sets[j].ev_join);
                if (sets[j].ev_dq) cudaEventDestroy(sets[j].ev_dq);
                if (sets[j].side) cudaStreamDestroy(sets[j].side);
            }
            return rc;
        }
    }
    s->lanes = std::move(sets);
    s->lane = 0;
    return SWARM_OK;
}

int swarm_stage_set_lane(swarm_stage_t s, int lane) {
    if (!s) return fail("set_lane: null stage");
    if (s->lanes.empty()) return lane == 0 ? SWARM_OK : fail("set_lane: lanes not enabled");
    if (lane < 0 || lane >= static_cast<int>(s->lanes.size())) return fail("set_lane: bad lane");
    if (lane == s->lane) return SWARM_OK;
    work_save(s, s->lanes[s->lane]);
    work_load(s, s->lanes[lane]);
    s->lane = lane;
    return SWARM_OK;
}

int swarm_stage_backward(swarm_stage_t s, int slot, const void* grad_in, void* grad_out, swarm_stream_t stream) {
    return swarm_stage_backward_ex(s, slot, grad_in, grad_out, SWARM_WGRAD_NOW, 0, -1, 0, stream);
}

int swarm_stage_enable_wgrad_pairing(swarm_stage_t s) { return swarm_stage_enable_wgrad_pairing_sets(s, 2); }

int swarm_stage_enable_wgrad_pairing_sets(swarm_stage_t s, int n_sets) {
    if (n_sets < 2) return fail("enable_wgrad_pairing: need at least two stash sets");
    if (!s->stash.empty()) return static_cast<int>(s->stash.size()) >= n_sets
                                      ? SWARM_OK
                                      : fail("enable_wgrad_pairing: already enabled with fewer sets");
    const size_t T = s->T, d = s->d, F = s->F, nl = static_cast<size_t>(s->cfg.n_layers);
    s->stash.resize(n_sets);
    for (auto& set : s->stash) {
        set.resize(nl);
        if (s->stacked) {  // application order, contiguous: the stacked GEMMs read each as one K = n*T operand
            EP dy, du, dh, dq;
            TRY(alloc(s, &dy, nl * T * d));
            TRY(alloc(s, &du, nl * T * F));
            TRY(alloc(s, &dh, nl * T * d));
            TRY(alloc(s, &dq, nl * 3 * T * d));
            for (size_t l = 0; l < nl; ++l)
                set[l] = Stash{dy + l * T * d, du + l * T * F, dh + l * T * d, dq + l * 3 * T * d};
            continue;
        }
        for (Stash& x : set) {
            TRY(alloc(s, &x.dy, T * d));
            TRY(alloc(s, &x.du, T * F));
            TRY(alloc(s, &x.dhid, T * d));
            TRY(alloc(s, &x.dqkv, 3 * T * d));
        }
    }
    return SWARM_OK;
}

namespace {
// Layer-shared stage: the shared weights' gradients over every application of a
// visit (or of a pending visit and this one) as one GEMM per weight, dW += sum_l
// dY_l^T X_l with K = n_layers * T (2 n_layers T for a pair), reading the stacked
// activations and stash.  Replaces n_layers K = T GEMMs that each read and wrote
// the whole fp32 gradient of the weight (configs[3]: 16 x 268 MB per FFN weight).
int stacked_wgrad(swarm_stage* s, const Slot& cur, const std::vector<Stash>& cs, const Slot* prev,
                  const std::vector<Stash>* ps, cudaStream_t sd) {
    const int d = s->d, F = s->F, nT = s->cfg.n_layers * s->T;
    float* G = s->grad;
    const LayerW& W = weights(s, 0);
    auto one = [&](int M, int N, int ldy, EP dy, EP pdy, int ldx, EP x, EP px,
                   size_t off, int ldo) {
        if (!prev) return mm(M, N, nT, {dy, ldy, nT, ldy, true}, {x, ldx, nT, ldx, true}, G + off, ldo,
                             SWARM_EPI_ACCUM_F32, nullptr, 1.f, sd);
        return mm2(M, N, 2 * nT, {pdy, ldy, nT, ldy, true}, {px, ldx, nT, ldx, true}, dy, x, G + off, ldo, sd);
    };
    const Act& A = cur.layer[0];
    const Act* P = prev ? &prev->layer[0] : nullptr;
    const Stash& c0 = cs[0];
    const Stash* p0 = ps ? &(*ps)[0] : nullptr;
    TRY(one(d, F, d, c0.dy, p0 ? p0->dy : nullptr, F, A.g, P ? P->g : nullptr, W.w2, F));
    TRY(one(F, d, F, c0.du, p0 ? p0->du : nullptr, d, A.c, P ? P->c : nullptr, W.w1, d));
    TRY(one(d, d, d, c0.dhid, p0 ? p0->dhid : nullptr, d, A.o, P ? P->o : nullptr, W.wo, d));
    return one(3 * d, d, 3 * d, c0.dqkv, p0 ? p0->dqkv : nullptr, d, A.a, P ? P->a : nullptr, W.wqkv, d);
}
}  // namespace

int swarm_stage_flush_wgrad(swarm_stage_t s, int slot, int set, swarm_stream_t stream) {
    if (s->stash.empty()) return fail("flush_wgrad: pairing not enabled");
    if (slot < 0 || slot >= static_cast<int>(s->slots.size()) || set < 0 || set >= static_cast<int>(s->stash.size()))
        return fail("flush_wgrad: bad slot/set");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ProfScope prof(s);
    const int T = s->T, d = s->d, F = s->F, n = s->cfg.n_layers;
    float* G = s->grad;
    if (s->stacked) return stacked_wgrad(s, s->slots[slot], s->stash[set], nullptr, nullptr, st);
    for (int l = 0; l < n; ++l) {
        const Act& A = s->slots[slot].layer[l];
        const Stash& x = s->stash[set][l];
        const LayerW& W = weights(s, l);
        TRY(mm(d, F, T, {x.dy, d, T, d, true}, {A.g, F, T, F, true}, G + W.w2, F, SWARM_EPI_ACCUM_F32, nullptr, 1.f, st));
        TRY(mm(F, d, T, {x.du, F, T, F, true}, {A.c, d, T, d, true}, G + W.w1, d, SWARM_EPI_ACCUM_F32, nullptr, 1.f, st));
        TRY(mm(d, d, T, {x.dhid, d, T, d, true}, {A.o, d, T, d, true}, G + W.wo, d, SWARM_EPI_ACCUM_F32, nullptr, 1.f, st));
        TRY(mm(3 * d, d, T, {x.dqkv, 3 * d, T, 3 * d, true}, {A.a, d, T, d, true}, G + W.wqkv, d, SWARM_EPI_ACCUM_F32,
               nullptr, 1.f, st));
    }
    return SWARM_OK;
}

int swarm_stage_backward_ex(swarm_stage_t s, int slot, const void* grad_in, void* grad_out, int wgrad_mode, int set,
                            int prev_slot, int prev_set, swarm_stream_t stream) {
    if (slot < 0 || slot >= static_cast<int>(s->slots.size())) return fail("backward: bad slot");
    if (wgrad_mode < SWARM_WGRAD_NOW || wgrad_mode > SWARM_WGRAD_PAIR) return fail("backward: bad wgrad mode");
    if (wgrad_mode != SWARM_WGRAD_NOW) {
        const int nsets = static_cast<int>(s->stash.size());
        if (nsets == 0) return fail("backward: wgrad pairing not enabled");
        if (set < 0 || set >= nsets) return fail("backward: bad stash set");
        if (wgrad_mode == SWARM_WGRAD_PAIR &&
            (prev_slot < 0 || prev_slot >= static_cast<int>(s->slots.size()) || prev_set < 0 || prev_set >= nsets ||
             prev_set == set || prev_slot == slot))
            return fail("backward: pairing needs a distinct pending slot and stash set");
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ProfScope prof(s);
    Slot& sl = s->slots[slot];
    const int T = s->T, d = s->d, n = s->cfg.n_layers;
    const bool stashed = wgrad_mode != SWARM_WGRAD_NOW;
    // the gradient entering the last layer: a workspace, or that layer's stash
    EP g_in = stashed ? s->stash[set][n - 1].dy : s->gy[0];
    int cur = 0;
    if (s->cfg.is_last) {
        PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_backward(sl.dxf, sl.out, s->dt, T, d, ln_param(s, s->lnfg), sl.muf, sl.rsf, nullptr,
                                      g_in, s->grad + s->lnfg, s->grad + s->lnfb, 1, s->lnws, st));
    } else {
        if (!grad_in) return fail("backward: null gradient message");
        if (s->bneck) {
            // d out = LN_c'(maxout'(dequant(grad)))
            PTRY(SWARM_PROF_OTHER, st, wire_decode(s, grad_in, s->wtmp, st));
            PTRY(SWARM_PROF_OTHER, st, swarm_maxout_backward(s->wtmp, s->dt, sl.am, static_cast<size_t>(T) * s->wire_w,
                                      s->cfg.maxout_k, s->dc, st));
            PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_backward(s->dc, sl.out, s->dt, T, d, ln_param(s, s->bn_out_g), sl.muc, sl.rsc,
                                          nullptr, g_in, s->grad + s->bn_out_g, s->grad + s->bn_out_b, 1, s->lnws,
                                          st));
        } else {
            PTRY(SWARM_PROF_OTHER, st, wire_decode(s, grad_in, g_in, st));
        }
    }
    if (!stashed) {
        for (int l = n - 1; l >= 0; --l) {
            TRY(block_backward(s, sl.layer[l], s->gy[cur], s->gy[cur ^ 1], weights(s, l), st));
            cur ^= 1;
        }
    } else {
        // layer l's input gradient lives in stash[set][l].dy (its weight gradients read it);
        // layer 0's output gradient goes to the workspace the tail below consumes
        for (int l = n - 1; l >= 0; --l) {
            WgradPlan wp;
            wp.mode = s->stacked ? SWARM_WGRAD_DEFER : wgrad_mode;  // stacked: all applications at once, below
            if (wp.mode == SWARM_WGRAD_PAIR) {
                wp.prev = &s->slots[prev_slot].layer[l];
                wp.ps = &s->stash[prev_set][l];
            }
            EP dx = l > 0 ? s->stash[set][l - 1].dy : s->gy[0];
            TRY(block_backward(s, sl.layer[l], s->stash[set][l].dy, dx, weights(s, l), st, wp, &s->stash[set][l]));
        }
        if (s->stacked && wgrad_mode == SWARM_WGRAD_PAIR) {
            TRY(fork_side(s, st, 0));
            TRY(stacked_wgrad(s, sl, s->stash[set], &s->slots[prev_slot], &s->stash[prev_set], side_of(s, st)));
            TRY(join_side(s, st));
        }
        cur = 0;
    }
    if (s->cfg.is_first) {
        ProfOp po(SWARM_PROF_OTHER, st);
        return swarm_embedding_backward_ex(sl.tokens, T, s->gy[cur], s->V, d, s->grad + s->emb, s->dt, st);
    }
    if (!grad_out) return fail("backward: null output gradient message");
    if (!s->bneck) {
        ProfOp po(SWARM_PROF_OTHER, st);
        s->last_dx = s->gy[cur];
        return wire_encode(s, s->gy[cur], grad_out, st);
    }
    // receiver side of the bottleneck: dW_d += dx0^T ni ; dni = dx0 W_d ; dmi = LN_d'(dni)
    const int w = s->wire_w;
    EP dx0 = s->gy[cur];
    TRY(mm(d, w, T, {dx0, d, T, d, true}, {sl.ni, w, T, w, true}, s->grad + s->bn_wd, w, SWARM_EPI_ACCUM_F32, nullptr,
           1.f, st));
    TRY(mm(T, w, d, {dx0, d, T, d, false}, {wts(s) + s->bn_wd, w, d, w, true}, s->wtmp, w, SWARM_EPI_STORE_BF16,
           nullptr, 1.f, st));
    PTRY(SWARM_PROF_LAYERNORM, st, swarm_layer_norm_backward(s->wtmp, sl.mi, s->dt, T, w, ln_param(s, s->bn_in_g), sl.mud, sl.rsd, nullptr,
                                  s->dqkv, s->grad + s->bn_in_g, s->grad + s->bn_in_b, 1, s->lnws, st));
    ProfOp po(SWARM_PROF_OTHER, st);
    s->last_dx = s->dqkv;
    return wire_encode(s, s->dqkv, grad_out, st);
}

int swarm_stage_optimizer_state(swarm_stage_t s, float** m, float** v, int* step) {
    if (m) *m = s->m;
    if (v) *v = s->v;
    if (step) *step = s->step;
    return SWARM_OK;
}

int swarm_stage_set_step(swarm_stage_t s, int step) {
    if (step < 0) return fail("set_step: negative step");
    s->step = step;
    return SWARM_OK;
}

int swarm_stage_optimizer_step(swarm_stage_t s, float grad_scale, swarm_stream_t stream) {
    s->step += 1;
    const auto& c = s->cfg;
    return swarm_adamw_step(s->p32, s->p16, s->grad, s->m, s->v, s->nparams, c.lr, c.beta1, c.beta2, c.eps,
                            c.weight_decay, s->step, grad_scale, 1, stream);
}

}  // extern "C"
