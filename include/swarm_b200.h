/*
 * swarm_b200.h — the drop-in C-ABI of the B200-native SWARM per-stage hot path.
 *
 * Library: paper_2301_11913_b200/libswarm_b200.so (sm_100a, built by
 * paper_2301_11913_b200/csrc/Makefile).  Plain pointers and sizes only.
 *
 * Conventions:
 *   - every "device" pointer is CUDA device memory owned by the caller;
 *     every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and allocates nothing on the hot path;
 *   - "_host" entry points take HOST buffers and do H2D -> kernel -> D2H
 *     themselves (the reference's own by-value contract), blocking until done;
 *   - return codes: SWARM_OK, SWARM_E_INVALID (maps to swarmsim::ConfigError),
 *     SWARM_E_NONFINITE (ConfigError "quantize_blockwise: non-finite input"),
 *     SWARM_E_CUDA, SWARM_E_UNSUPPORTED.  swarm_last_error() gives the message
 *     of the calling thread's last failure;
 *   - device-side errors (non-finite input) are reported through an optional
 *     device word `flags` that the kernel ORs SWARM_FLAG_NONFINITE into; the
 *     caller reads it at its next sync point.
 *
 * P/ = /root/reference/proj/ (the reference; each entry cites what it replaces).
 */
#ifndef SWARM_B200_H
#define SWARM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWARM_OK 0
#define SWARM_E_INVALID 1
#define SWARM_E_NONFINITE 2
#define SWARM_E_CUDA 3
#define SWARM_E_UNSUPPORTED 4
#define SWARM_E_NO_PEER 5 /* maps to swarmsim::NoPeerAvailable */

#define SWARM_DTYPE_F32 0
#define SWARM_DTYPE_BF16 1
#define SWARM_DTYPE_F64 2

#define SWARM_FLAG_NONFINITE 1u

typedef void* swarm_stream_t; /* cudaStream_t */

/* ---- library ----------------------------------------------------------- */
const char* swarm_last_error(void);
int swarm_version(void);
/* number of kernels this library has launched in this process (for bench's gpu_launches) */
uint64_t swarm_launch_count(void);

/* ---- K1: blockwise int8 absmax quantizer --------------------------------
 * Replaces compress::quantize_blockwise (P/src/compression.cpp:10-29,
 * declared P/include/swarmsim/compression.hpp:23).
 *   x       : n values of `dtype` (F32 | BF16 | F64), device
 *   codes   : n int8, device;  code = round_half_away(127*x/absmax), bit-exact
 *             to the reference's fp64 formula for every input dtype
 *   scales  : ceil(n/block_size) per-block absmax, device; float for F32/BF16
 *             input (exact), double for F64 input
 *   flags   : optional device uint32 (SWARM_FLAG_NONFINITE on NaN/Inf input)
 * block_size == 0 -> SWARM_E_INVALID (compression.cpp:11). */
int swarm_quantize_blockwise(const void* x, int dtype, size_t n, size_t block_size, int8_t* codes,
                             void* scales, uint32_t* flags, swarm_stream_t stream);

/* ---- K2: blockwise dequantizer ------------------------------------------
 * Replaces compress::dequantize_blockwise (P/src/compression.cpp:31-37).
 * out[i] = code[i]*absmax[i/bs]/127.0 evaluated in fp64 and rounded once to
 * `out_dtype` (F32 | BF16 | F64).  scale_dtype: F32 or F64. */
int swarm_dequantize_blockwise(const int8_t* codes, const void* scales, int scale_dtype, size_t n,
                               size_t block_size, void* out, int out_dtype, swarm_stream_t stream);

/* Host-buffer end-to-end variants (the reference's by-value API shape):
 * chunked, pipelined H2D -> kernel -> D2H over an internal device workspace.
 * Returns SWARM_E_NONFINITE when the input holds NaN/Inf (codes undefined). */
int swarm_quantize_blockwise_host(const void* x, int dtype, size_t n, size_t block_size,
                                  int8_t* codes, void* scales);
int swarm_dequantize_blockwise_host(const int8_t* codes, const void* scales, int scale_dtype,
                                    size_t n, size_t block_size, void* out, int out_dtype);

/* ---- K3: maxout ----------------------------------------------------------
 * Replaces compress::maxout_k (P/src/compression.cpp:39-50): out[j] = max of
 * x[j*k .. j*k+k-1], earliest element wins ties (std::max semantics); argmax
 * (optional, uint8 window index) feeds the backward scatter.  k must divide n. */
int swarm_maxout_forward(const void* x, int dtype, size_t n, size_t k, void* out, uint8_t* argmax,
                         swarm_stream_t stream);
/* grad_in[j*k+i] = (i == argmax[j]) ? grad_out[j] : 0 (no reference) */
int swarm_maxout_backward(const void* grad_out, int dtype, const uint8_t* argmax, size_t n_out,
                          size_t k, void* grad_in, swarm_stream_t stream);

/* ---- K4: LayerNorm -------------------------------------------------------
 * Replaces compress::layer_norm (P/src/compression.cpp:52-74) row-wise:
 * two-pass mean / biased variance, (x-mean)/sqrt(var+eps)*gain+bias.
 * dtype F32 | BF16 (fp32 statistics) or F64 (fp64 throughout); gain/bias are
 * float for F32/BF16 and double for F64, NULL = ones/zeros.  mean/rstd
 * (optional, float, `rows` each) are saved for the backward. */
int swarm_layer_norm_forward(const void* x, int dtype, size_t rows, size_t cols, const void* gain,
                             const void* bias, double eps, void* out, float* mean, float* rstd,
                             swarm_stream_t stream);
/* dx = LN'(dy) (+ dres when non-NULL: the residual branch's gradient, fused),
 * dgain/dbias (float, cols) written, or added when `accumulate` != 0 (gradient
 * accumulation over microbatches).  Either part may be skipped: dgain = dbias =
 * NULL computes dx only; dx = NULL (bf16 rows of width 256k <= 4096) computes the
 * gain/bias gradients only, so they can run on another stream.  `workspace` >= swarm_layer_norm_backward_workspace()
 * bytes of device memory, zero-filled before its first use (the call leaves it zeroed
 * again; it must not be shared by concurrent calls). */
size_t swarm_layer_norm_backward_workspace(size_t rows, size_t cols);
int swarm_layer_norm_backward(const void* dy, const void* x, int dtype, size_t rows, size_t cols,
                              const float* gain, const float* mean, const float* rstd, const void* dres,
                              void* dx, float* dgain, float* dbias, int accumulate, void* workspace,
                              swarm_stream_t stream);

/* ---- bottleneck projection (fp64 API path) -------------------------------
 * Replaces the private matvec behind compress::bottleneck_forward /
 * bottleneck_decompress (P/src/compression.cpp:78-101): out[j] = sum_i x[i]*w[i][j]
 * accumulated in ascending i with unfused fp64 multiply/add, i.e. bit-identical
 * to the reference.  w is row-major rows x cols (device). */
int swarm_matvec_f64(const double* x, size_t rows, const double* w, size_t cols, double* out,
                     swarm_stream_t stream);

/* ---- K5: tcgen05 / TMEM / TMA bf16 GEMM ---------------------------------
 * The block's dense contractions (cost_model.cpp:31-42 counts them; the
 * reference never executes them).  Computes, for z in [0, batch):
 *   D_z = alpha * op(A_z) . op(B_z)^T   (M x N, fp32 accumulate in TMEM)
 * A is M x K: K-contiguous rows (a_mn_major=0, row stride lda) or stored
 * K x M with M contiguous (a_mn_major=1).  Same for B (N x K).
 * Batch offsets (elements) for operand X in {a,b,d}: z -> (z/bh, z%bh) with
 * row offset rX0*(z/bh) + rX1*(z%bh) and column offset cX0*(z/bh) + cX1*(z%bh)
 * applied to the operand's 2D storage.  `epilogue` selects the fused op:    */
#define SWARM_EPI_STORE_BF16 0  /* D = bf16(alpha*acc)                         */
#define SWARM_EPI_STORE_F32 1   /* D = alpha*acc (float)                       */
#define SWARM_EPI_ACCUM_F32 2   /* D += alpha*acc (float; gradient accumulate) */
#define SWARM_EPI_RESIDUAL 3    /* D = bf16(alpha*acc + R)                     */
#define SWARM_EPI_GELU 4        /* U = bf16(acc); D = bf16(gelu(acc))          */
#define SWARM_EPI_DGELU 5       /* D = bf16(acc * gelu'(U))                    */
#define SWARM_EPI_GELU_DERIV 6  /* U = bf16(gelu'(acc)); D = bf16(gelu(acc))   (one tanh for both) */
#define SWARM_EPI_MUL 7         /* D = bf16(acc * U)   (the MLP backward with U = gelu' saved) */
typedef struct {
    int m, n, k, batch, bh;
    /* operand storage: a_rows x a_cols row-major with row stride lda (0,0 =
       derive from m,k for an unbatched call); bf16, 16-byte aligned rows */
    const void* a; int lda; int a_mn_major; int a_rows, a_cols; int ra0, ra1, ca0, ca1;
    const void* b; int ldb; int b_mn_major; int b_rows, b_cols; int rb0, rb1, cb0, cb1;
    void* d; int ldd; int rd0, rd1, cd0, cd1;
    const void* aux; /* R (RESIDUAL) or U (DGELU): bf16, same layout as D; U output for GELU */
    float alpha;
    int epilogue;
    /* causal structure of A per batch entry (M == K): 0 dense; 1 A[i][j] == 0 for
       j > i (P, dS: k-blocks past the tile's last row are skipped); 2 A[i][j] == 0
       for j < i (P^T, dS^T: k-blocks before the tile's first row are skipped) */
    int k_tri;
    /* optional second K segment (batch == 1): when both are non-NULL, K splits into
       two equal halves (K/2 a multiple of 64); k-indices [K/2, K) read a2 / b2, which
       share the layout (ld, majorness, per-segment extents) of a / b.  This pairs the
       weight-gradient GEMMs of two microbatches whose activations live in separate
       buffers (one K = 2T GEMM instead of two K = T ones). */
    const void* a2;
    const void* b2;
    /* optional stream-K scratch (NULL = whole tiles only): at least
       swarm_gemm_workspace_bytes(), zero-filled once before its first use (the
       kernel leaves it zeroed again); never shared by GEMMs that can run
       concurrently.  With it, the last partial wave of 256x256 tiles is split
       along K across every SM pair (results identical up to fp32 summation
       order).  The kernel uses it only where it wins after paying for the fixup
       (few tiles, long K); SWARM_GEMM_STREAMK=0 / 1 force never / whenever the
       k-block path is shorter. */
    void* workspace;
    size_t workspace_bytes;
} swarm_gemm_args;
int swarm_gemm_bf16(const swarm_gemm_args* args, swarm_stream_t stream);
/* The same contraction with fp32 operands (SIMT FFMA, fp32 accumulate): the stage
 * executor's fp32 arithmetic mode (swarm_stage_config.fp32; BASELINE configs[0] is
 * specified fp32).  Every epilogue keeps its meaning with fp32 in place of bf16
 * (STORE_BF16 stores fp32; R / U are fp32); ACCUM_F32 adds atomically.  No
 * alignment requirement beyond fp32. */
int swarm_gemm_f32(const swarm_gemm_args* args, swarm_stream_t stream);
size_t swarm_gemm_workspace_bytes(void);
/* resident 2-CTA clusters of the 256x256 pair kernel on the current device (its
   persistent grid size; below SMs / 2 when GPCs strand SMs); 4-CTA clusters
   for the multicast variant (the default; SWARM_GEMM_MCAST=0 selects pairs) */
int swarm_gemm_pair_clusters(void);

/* ---- training building blocks (stage executor internals, exported for tests)
 * None of these has a reference counterpart: the reference only models the
 * block's cost (cost_model.cpp:31-42, sim.cpp:361-364).  bf16 tensors are
 * passed as void*. */
/* out[t,:] = table[tokens[t],:]  (bf16 [vocab,d] -> bf16 [n,d]); out-of-range ids give 0 */
int swarm_embedding_forward(const int32_t* tokens, size_t n_tokens, const void* table, size_t vocab, size_t d,
                            void* out, swarm_stream_t stream);
/* dtable[tokens[t],:] += dout[t,:]  (fp32 accumulate) */
int swarm_embedding_backward(const int32_t* tokens, size_t n_tokens, const void* dout, size_t vocab, size_t d,
                             float* dtable, swarm_stream_t stream);
/* the same for dtype F32 | BF16 tables / activations (fp32 mode: the fp32 master is the table) */
int swarm_embedding_forward_ex(const int32_t* tokens, size_t n_tokens, const void* table, size_t vocab, size_t d,
                               void* out, int dtype, swarm_stream_t stream);
int swarm_embedding_backward_ex(const int32_t* tokens, size_t n_tokens, const void* dout, size_t vocab, size_t d,
                                float* dtable, int dtype, swarm_stream_t stream);
/* P = softmax(S) row-wise over L columns (rows = batch*heads*L); causal masks
 * column j > (row % L).  S fp32 (already scaled), P bf16. */
int swarm_attn_softmax_forward(const float* s, size_t rows, size_t L, int causal, void* p, swarm_stream_t stream);
/* dS = scale * P * (dP - rowsum(P*dP)), bf16 */
int swarm_attn_softmax_backward(const void* p, const float* dp, size_t rows, size_t L, float scale, void* ds,
                                swarm_stream_t stream);
/* the same with P / dS of dtype F32 | BF16 (fp32 mode: accurate expf) */
int swarm_attn_softmax_forward_ex(const float* s, size_t rows, size_t L, int causal, void* p, int p_dtype,
                                  swarm_stream_t stream);
int swarm_attn_softmax_backward_ex(const void* p, const float* dp, size_t rows, size_t L, float scale, void* ds,
                                   int dtype, swarm_stream_t stream);
/* Fused attention scores (tcgen05; L % 128 == 0, L <= 1024, d_head % 64 == 0, d_head <= 128):
 *   P[z*L + i, j] = softmax_j(scale * q_z[i] . k_z[j])  (bf16 [B*H*L, L], causal masks j > i)
 * with q_z = q[b*L + i, h*d_head : (h+1)*d_head] for z = b*H + h (row stride ld, n_cols
 * valid columns; k likewise); scores stay in TMEM.  When causal, columns at or past a
 * query block's causal extent ((i/128 + 1) * 128) are not written. */
int swarm_attn_scores_softmax(const void* q, const void* k, int ld, int n_cols, int B, int H, int L, int d_head,
                              float scale, int causal, void* P, swarm_stream_t stream);
/* The same probabilities P plus the attention output O = P V in one kernel (d_head 128): each key
 * chunk's P is written over its K chunk in shared memory once the score MMA has read it, stored to
 * P from there, and multiplied by the V chunk (tcgen05, O accumulated in TMEM); O[b*L + i, h*d_head
 * .. +d_head] (row stride ld_o) in bf16.  v has q's storage geometry (ld, n_cols). */
int swarm_attn_forward_pv(const void* q, const void* k, const void* v, int ld, int n_cols, int B, int H, int L,
                          int d_head, float scale, int causal, void* P, void* O, int ld_o, swarm_stream_t stream);
/* The same forward storing no P: lse[z*L + i] (float, [B*H*L]) = log2 sum_j 2^(scale * q_z[i] . k_z[j] *
 * log2(e)) over the unmasked keys -- the row's log-sum-exp in base 2 -- and O as above (bit-identical
 * to swarm_attn_forward_pv's O).  The backward recomputes P from it (swarm_attn_backward_lse), so
 * no [B*H*L, L] buffer exists on this path. */
int swarm_attn_forward_lse(const void* q, const void* k, const void* v, int ld, int n_cols, int B, int H, int L,
                           int d_head, float scale, int causal, float* lse, void* O, int ld_o, swarm_stream_t stream);
/* dS = scale * P * (dP - rowsum(P * dP)) with dP = dO_z V_z^T computed in TMEM (bf16 out); the
 * row statistic is taken as dO . O (O = P V, the forward's attention output, [B*L, ld_o] with
 * head h at column h*d_head), which equals rowsum(P * dP) and saves a second pass.
 * Columns at or past a query block's causal extent ((i/128 + 1) * 128) are not written
 * (the forward likewise leaves them untouched when causal): callers that read them keep
 * them zeroed. */
int swarm_attn_scores_softmax_backward(const void* dO, int ld_do, const void* v, int ld_v, int v_cols, const void* o,
                                       int ld_o, const void* P, int B, int H, int L, int d_head, float scale,
                                       int causal, void* dS, swarm_stream_t stream);
/* The attention backward with dP and dS on chip (tcgen05, d_head 128, L % 128 == 0): with dO
 * [B*L, ld_do] (head h at column h*128), the forward's qkv storage (Q at column 0, K at k_col0,
 * V at v_col0, row stride ld_qkv, qkv_cols valid columns), O [B*L, ld_o] and the forward's P
 * (bf16 [B*H*L, L]), writes dQ | dK | dV (bf16) into dqkv at columns 0 | dk_col0 | dv_col0
 * (+ h*128, row stride ld_dqkv):
 *   dV = P^T dO,  dS = scale * P * (dO V^T - dO.O),  dK = dS^T Q,  dQ = dS K
 * workspace: swarm_attn_backward_workspace(B, H, L, 128) bytes, zeroed by the caller once (every
 * call leaves its fp32 dQ accumulator, the head B*L*H*128*4 bytes, zeroed); one call in flight per
 * workspace.  dQ's fp32 sum over key blocks uses reduce-add (summation order not fixed).
 * Replaces swarm_attn_scores_softmax_backward + the three dS / P GEMMs (csrc/attn_bwd.cu). */
size_t swarm_attn_backward_workspace(int B, int H, int L, int d_head);
/* The same with P recomputed on chip from the forward's log2-sum-exp (swarm_attn_forward_lse):
 * S = Q K^T per (query, key) block in TMEM, P = 2^(S * scale * log2(e) - lse) in bf16 (causal
 * mask on the diagonal blocks), then as above.  Same workspace. */
int swarm_attn_backward_lse(const void* dO, int ld_do, const void* qkv, int ld_qkv, int qkv_cols, int k_col0,
                            int v_col0, const void* O, int ld_o, const float* lse, int B, int H, int L, int d_head,
                            float scale, int causal, void* dqkv, int ld_dqkv, int dk_col0, int dv_col0,
                            void* workspace, swarm_stream_t stream);
int swarm_attn_backward(const void* dO, int ld_do, const void* qkv, int ld_qkv, int qkv_cols, int k_col0, int v_col0,
                        const void* O, int ld_o, const void* P, int B, int H, int L, int d_head, float scale,
                        int causal, void* dqkv, int ld_dqkv, int dk_col0, int dv_col0, void* workspace,
                        swarm_stream_t stream);
/* token cross-entropy on fp32 logits [rows, vocab]: loss_sum += sum_t (lse_t - logit_t[target_t]);
 * dlogits (bf16, optional) = grad_scale * (softmax - onehot) */
int swarm_cross_entropy(const float* logits, const int32_t* targets, size_t rows, size_t vocab, float grad_scale,
                        float* loss_sum, void* dlogits, swarm_stream_t stream);
/* dlogits of dtype F32 | BF16 (F32: accurate expf, the fp32 mode) */
int swarm_cross_entropy_ex(const float* logits, const int32_t* targets, size_t rows, size_t vocab, float grad_scale,
                           float* loss_sum, void* dlogits, int dlogits_dtype, swarm_stream_t stream);
/* fused AdamW over a flat fp32 arena; refreshes the bf16 shadow (p16, optional)
 * and zeroes the gradient when zero_grad != 0.  step >= 1 (bias correction). */
int swarm_adamw_step(float* p32, void* p16, float* grad, float* m, float* v, size_t n, float lr, float beta1,
                     float beta2, float eps, float weight_decay, int step, float grad_scale, int zero_grad,
                     swarm_stream_t stream);
/* p[i] = mean + std * N(0,1) from a counter-based hash of (seed, i) */
int swarm_fill_normal(float* p, size_t n, float mean, float std, uint64_t seed, swarm_stream_t stream);
int swarm_cast_f32_bf16(const float* in, void* out, size_t n, swarm_stream_t stream);
/* dst[i] += src[i] (fp32): sums the gradient arenas of a stage's peers that share a GPU */
int swarm_add_f32(float* dst, const float* src, size_t n, swarm_stream_t stream);

/* ---- stage executor -------------------------------------------------------
 * One SWARM pipeline stage on one GPU: a contiguous range of pre-LN
 * transformer blocks (Wqkv d x 3d, Wo d x d, W1 d x d_ffn, W2 d_ffn x d, no
 * biases: P/src/cost_model.cpp:31-35; GeLU MLP with residual: PAPER:787), the
 * embedding on the first stage and final LN + LM head + cross-entropy on the
 * last.  It is the real work behind the reference's simulated stage visit
 * (Engine::visit_seconds / start_service, P/src/sim.cpp:361-364, 395-403):
 * forward = one forward visit, backward = one backward visit.  Boundary
 * tensors cross stages as a "wire message": bf16 activations, or int8 codes
 * followed by fp32 per-block scales (the codec above; payload as
 * QuantizedTensor::payload_bits, compression.hpp:20).  Weights, fp32 master
 * copy, fp32 gradients and AdamW moments live in flat device arenas owned by
 * the stage; activations for up to max_slots in-flight microbatches too.  */
#define SWARM_WIRE_BF16 0
#define SWARM_WIRE_INT8 1
/* Wire message = payload ‖ header.  INT8 payload: codes[n] (padded to 16 B) then
 * fp32 scales[ceil(n/block)] (padded to 16 B); BF16 payload: bf16[n] (padded).
 * The last 16 bytes are this header (one self-describing message
 * per hop, one NCCL call). */
#define SWARM_WIRE_MAGIC 0x314D5753u /* "SWM1" */
typedef struct {
    uint32_t magic;
    uint32_t n_elems;
    uint32_t block_size;
    uint8_t kind; /* SWARM_WIRE_* */
    uint8_t maxout_k;
    uint8_t version;
    uint8_t reserved;
} swarm_wire_header;
/* parse a header copied to host memory (last sizeof(swarm_wire_header) bytes of a message) */
int swarm_wire_parse_header(const void* header, uint32_t* n_elems, uint32_t* block_size, int* kind, int* maxout_k);
typedef struct swarm_stage* swarm_stage_t;
typedef struct {
    int d_model, n_heads, d_ffn, seq_len, micro_batch;
    int n_layers;      /* block applications in this stage */
    int shared_layers; /* 1: one weight set applied n_layers times (layer sharing) */
    int vocab;
    int is_first, is_last;
    int causal;
    int max_slots;     /* microbatches in flight (activation slots) */
    int wire;          /* SWARM_WIRE_BF16 | SWARM_WIRE_INT8 */
    int block_size;    /* int8 codec block */
    int maxout_k;      /* > 1: maxout bottleneck at the boundaries: the sender sends
                          maxout_k(LN(y)) (d/k wide), the receiver applies LN then W_d (d/k -> d) */
    float lr, beta1, beta2, eps, weight_decay, init_std;
    uint64_t seed;
    int fp32;          /* 1: fp32 arithmetic mode — fp32 activations and wire tensors, fp32 GEMMs
                          (swarm_gemm_f32) reading the fp32 master weights, unfused attention;
                          0 (default): bf16 storage, tcgen05 bf16 GEMMs, fp32 accumulation.
                          Delayed-update banks need the bf16 mode. */
} swarm_stage_config;

int swarm_stage_create(const swarm_stage_config* cfg, swarm_stage_t* out);
void swarm_stage_destroy(swarm_stage_t st);
size_t swarm_stage_wire_bytes(swarm_stage_t st);
size_t swarm_stage_num_params(swarm_stage_t st);
/* forward visit of microbatch `slot`.  in: int32 tokens [B*L] on the first
 * stage, else a wire message.  out: wire message for the next stage (unused on
 * the last).  Last stage: targets int32 [B*L]; loss_sum (device float) += the
 * token losses; the LM-head backward runs here too (dlogits scaled by
 * loss_scale, so backward needs no second pass over the vocabulary). */
int swarm_stage_forward(swarm_stage_t st, int slot, const void* in, const int32_t* targets, void* out,
                        float* loss_sum, float loss_scale, swarm_stream_t stream);
/* backward visit: grad_in = wire message from the next stage (unused on the
 * last), grad_out = wire message for the previous stage (unused on the first).
 * Parameter gradients accumulate into the fp32 gradient arena. */
int swarm_stage_backward(swarm_stage_t st, int slot, const void* grad_in, void* grad_out, swarm_stream_t stream);
/* Paired weight gradients: the four weight-gradient GEMMs of every block run once
 * per two backward visits with K = 2T (measured 10-24% faster than two K = T
 * GEMMs, and half the fp32 reduce-add traffic into the gradient arena).
 * enable_wgrad_pairing allocates two stash sets of the blocks' dY tensors.
 * backward_ex(wgrad_mode): SWARM_WGRAD_NOW = swarm_stage_backward; DEFER = compute
 * the data gradients, keep this visit's dY tensors in stash `set`, no weight
 * gradients; PAIR = also issue the weight gradients of the pending visit
 * (prev_slot, prev_set) and this one as two-segment GEMMs.  flush_wgrad issues a
 * still-pending visit's weight gradients alone (before the all-reduce).  The
 * calls are stateless: the caller tracks the pending visit (CUDA-graph safe). */
#define SWARM_WGRAD_NOW 0
#define SWARM_WGRAD_DEFER 1
#define SWARM_WGRAD_PAIR 2
int swarm_stage_enable_wgrad_pairing(swarm_stage_t st);
/* the same with n_sets >= 2 stash sets (set / prev_set index them); the
 * engine-driven executor keeps one per trainer so a deferred visit's dY survives
 * other trainers' visits */
int swarm_stage_enable_wgrad_pairing_sets(swarm_stage_t st, int n_sets);
/* Lanes: n sets of visit workspaces (+ side stream / events) so that n visits of
 * one stage can be in flight on n streams; set_lane selects the set the next
 * visit call uses.  Visits on different lanes must use different slots; their
 * gradient accumulation (TMA reduce-add GEMM epilogues, atomic LayerNorm and
 * embedding gradients) is safe concurrently.  The caller orders visits that
 * share a slot or a stash set. */
int swarm_stage_enable_lanes(swarm_stage_t st, int n);
int swarm_stage_set_lane(swarm_stage_t st, int lane);
int swarm_stage_backward_ex(swarm_stage_t st, int slot, const void* grad_in, void* grad_out, int wgrad_mode, int set,
                            int prev_slot, int prev_set, swarm_stream_t stream);
int swarm_stage_flush_wgrad(swarm_stage_t st, int slot, int set, swarm_stream_t stream);
/* AdamW over the whole stage; grads are multiplied by grad_scale first, then zeroed. */
int swarm_stage_optimizer_step(swarm_stage_t st, float grad_scale, swarm_stream_t stream);
float* swarm_stage_grads(swarm_stage_t st);  /* fp32 [num_params]: intra-stage all-reduce buffer */
float* swarm_stage_params(swarm_stage_t st); /* fp32 master [num_params] */
void* swarm_stage_params_bf16(swarm_stage_t st);
/* migration state (params() + AdamW m, v, step): what a peer moving to this stage
 * downloads from a stage-mate (P/src/rebalancer.cpp:71-75 counts these bytes) */
int swarm_stage_optimizer_state(swarm_stage_t st, float** m, float** v, int* step);
int swarm_stage_set_step(swarm_stage_t st, int step);
/* re-derive the bf16 shadow from the fp32 master (after loading / receiving weights);
 * with two banks enabled, both shadows */
int swarm_stage_sync_shadow(swarm_stage_t st, swarm_stream_t stream);
/* Delayed parameter updates.  enable_banks allocates a
 * second bf16 shadow and a second gradient arena (both copies of bank 0).  Visits
 * read the weights of, and accumulate gradients into, the bank selected by
 * set_bank; optimizer_step_bank applies bank b's gradients to the fp32 master,
 * writes the result into bank b's shadow and zeroes bank b's gradients.  Step t
 * uses bank t % 2, so the optimizer of step t (bank t % 2) can run while step t+1
 * computes on the other bank: step t+1 sees the weights of step t-1's update. */
int swarm_stage_enable_banks(swarm_stage_t st, swarm_stream_t stream);
int swarm_stage_set_bank(swarm_stage_t st, int bank);
float* swarm_stage_grads_bank(swarm_stage_t st, int bank);
void* swarm_stage_params_bf16_bank(swarm_stage_t st, int bank); /* bank b's bf16 weight shadow */
int swarm_stage_optimizer_step_bank(swarm_stage_t st, int bank, float grad_scale, swarm_stream_t stream);
/* enumerate parameter tensors: index -> name, offset (elements), rows, cols */
int swarm_stage_param_info(swarm_stage_t st, int index, const char** name, size_t* offset, size_t* rows,
                           size_t* cols);
/* Visit profiling for the live roofline: while enabled, every kernel call of
 * this stage's visits is bracketed by CUDA events on the visit's stream (the
 * weight-gradient side stream is folded onto it);
 * profile_read synchronises, returns the summed GEMM time (ms), executed
 * FLOPs (2*M*N*K*batch, less the k-blocks a causal k_tri skips) and launch
 * count recorded since the last read, and resets.  profile_breakdown returns
 * the per-category time / call counts of that last read. */
#define SWARM_PROF_GEMM 0
#define SWARM_PROF_ATTENTION 1  /* fused score/softmax kernels (their GEMMs count as GEMM) */
#define SWARM_PROF_LAYERNORM 2
#define SWARM_PROF_OTHER 3      /* embedding, codec / wire, maxout, cross-entropy */
#define SWARM_PROF_CATEGORIES 4
void swarm_stage_profile(swarm_stage_t st, int enable);
/* weight applied to the time / FLOPs of events recorded from now on (profile_read
 * returns weighted sums): the number of visits of the profiled kind per step, so
 * one profiled visit per kind stands for all of them */
void swarm_stage_profile_weight(swarm_stage_t st, double weight);
int swarm_stage_profile_read(swarm_stage_t st, double* gemm_ms, double* gemm_flops, uint64_t* gemm_launches);
/* measurement utility: occupy `stream` for `ns` nanoseconds (one spinning
   thread) so the kernels issued behind it run back to back, free of host
   launch gaps, while an eagerly issued visit is being profiled */
int swarm_gpu_spin(uint64_t ns, swarm_stream_t stream);
void swarm_stage_profile_breakdown(swarm_stage_t st, double* ms /* [SWARM_PROF_CATEGORIES] */,
                                   uint64_t* launches /* [SWARM_PROF_CATEGORIES] */);
/* the last read's GEMM time per shape: lines "MxNxK bBATCH eEPILOGUE[ Amn][ Bmn][ 2seg][ tri];ms;flops;launches" */
const char* swarm_stage_profile_shapes(swarm_stage_t st);
/* saved activation of (slot, layer) by name ("x","a","qkv","P","o","h","c","u","g","xf","dxf"), for tests;
 * also "wire_out" (the tensor the last forward of `slot` encoded), "wire_in" (the decoded input wire
 * tensor) and "dx_last" (the input gradient the stage's last backward visit encoded).  Elements are
 * bf16, or fp32 in the fp32 mode. */
int swarm_stage_activation(swarm_stage_t st, int slot, int layer, const char* name, void** ptr, size_t* numel);

/* ---- host control plane: stochastic wiring + rebalancing ------------------
 * Replace wiring::RoutingState (P/include/swarmsim/wiring.hpp:19-90,
 * P/src/wiring.cpp:33-120) and rebalancer::decide (P/src/rebalancer.cpp:25-69)
 * with decision-identical host C++ (no GPU).  Peers are the reference's PeerId
 * values (uint64).  Errors: SWARM_E_INVALID (ConfigError), SWARM_E_NO_PEER. */
typedef struct swarm_router* swarm_router_t;
const char* swarm_router_last_error(void);
int swarm_router_create(size_t n_stages, double gamma, double epsilon, swarm_router_t* out);
void swarm_router_destroy(swarm_router_t r);
int swarm_router_add_server(swarm_router_t r, uint64_t peer, const size_t* stages, size_t n_stages, double phase);
int swarm_router_ban_server(swarm_router_t r, uint64_t peer);
void swarm_router_remove_server(swarm_router_t r, uint64_t peer);
int swarm_router_is_banned(swarm_router_t r, uint64_t peer);
int swarm_router_choose_server(swarm_router_t r, size_t stage, uint64_t* peer);
int swarm_router_record_response(swarm_router_t r, uint64_t peer, double elapsed_seconds);
int swarm_router_peer_state(swarm_router_t r, uint64_t peer, double* ema, double* priority);
int swarm_rebalance_decide(size_t n_stages, const size_t* offsets, const uint64_t* peers, const double* queues,
                           uint64_t* mover, size_t* from_stage, size_t* to_stage, size_t* op_count);

/* ---- engine-driven executor schedule ----------------------
 * The reference's discrete-event engine (P/src/sim.cpp:199-761: Engine::run,
 * start_service :395-403, dispatch_current :405-436, on_stage_complete
 * :472-491, advance_trainer :493-510, AllReduceTick :245-250) restated for a
 * static population, with the real executor attached where the reference
 * advances simulated time.  Records come out in event-processing order; every
 * rank running the same engine on the same seed sees the same sequence.
 * Workers are SimConfig::initial_peers flattened stage by stage (PeerId ==
 * index, as Engine::add_worker assigns them). */
#define SWARM_ENG_START 0      /* worker begins the visit (trainer, stage, backward); time..end_time modeled */
#define SWARM_ENG_HOP 1        /* trainer's input dispatched to `worker`'s queue; from_worker produced it (-1: new
                                  microbatch; -2: not given -- the driver derives it from the START records) */
#define SWARM_ENG_DONE 2       /* trainer's microbatch finished (backward at stage 0 on `worker`) */
#define SWARM_ENG_ALLREDUCE 3  /* stage-wide all-reduce tick; starts stall until end_time */
/* membership records (churn and rebalancing, P/src/sim.cpp:527-719) */
#define SWARM_ENG_LEAVE 4      /* `worker` died (kill_worker; backward = 1: it was migrating); its queued jobs
                                  follow as HOP records to other peers (requeue) */
#define SWARM_ENG_JOIN 5       /* new `worker` joined `stage` (on_peer_join); its trainers start */
#define SWARM_ENG_MIGRATE 6    /* `worker` leaves stage `from_worker` for `stage` (begin_migration); it downloads
                                  the destination's state until end_time */
#define SWARM_ENG_MIGRATED 7   /* `worker` serves `stage` again (on_migration_complete) */
#define SWARM_ENG_REBALANCE 8  /* Alg. 2 decision: from stage `from_worker` to `stage`, mover `worker` (-1: none;
                                  backward = 1: skipped on a stale table) */
typedef struct {
    double time;
    double end_time;
    int32_t kind;
    int32_t backward;
    uint32_t trainer;
    uint32_t stage;
    int64_t worker;
    int64_t from_worker;
    uint64_t microbatch; /* the trainer's microbatch counter */
} swarm_engine_record;
typedef struct swarm_engine* swarm_engine_t;
const char* swarm_engine_last_error(void);
/* The reference SimConfig (P/include/swarmsim/sim.hpp:21-54) with an explicit initial population
 * and churn trace (trace::Trace of (t, delta), trace.hpp:10-16): */
typedef struct {
    size_t n_stages;
    size_t n_workers;            /* initial_peers flattened stage by stage */
    const size_t* worker_stage;
    const double* worker_speed;  /* NULL = 1.0 */
    size_t n_churn;              /* churn trace: delta > 0 joins, < 0 leaves, at time t */
    const double* churn_t;
    const int64_t* churn_delta;
    double forward_seconds, backward_multiplier;
    size_t trainers_per_peer;
    double allreduce_period, allreduce_stall;
    int rebalance_periodic;      /* RebalanceMode::Periodic (else None) */
    double rebalance_period, straggler_timeout, propagation_delay, announce_ttl;
    uint64_t state_transfer_bytes;
    double download_bps;         /* DeviceProfile::download_bps: migration downtime = bytes * 8 / bps */
    double duration_seconds, bucket_seconds;
} swarm_sim_config;
swarm_sim_config swarm_sim_config_default(void); /* the reference's defaults */
int swarm_engine_create_ex(const swarm_sim_config* cfg, uint64_t seed, swarm_engine_t* out);
/* SimResult::requeued / abandoned, workers ever created and alive now */
int swarm_engine_counts(swarm_engine_t e, uint64_t* requeued, uint64_t* abandoned, size_t* n_workers, int64_t* alive);
int swarm_engine_worker(swarm_engine_t e, size_t worker, size_t* stage, int* alive, int* migrating);
/* SimConfig fields: n_stages, initial_peers (worker_stage/worker_speed, speed may be NULL = 1.0),
 * forward_service_seconds, backward_multiplier, trainers_per_peer, allreduce_period/_stall,
 * duration_seconds, bucket_seconds; seed = sim::run's seed.  Errors: SWARM_E_INVALID (ConfigError). */
int swarm_engine_create(size_t n_stages, size_t n_workers, const size_t* worker_stage, const double* worker_speed,
                        double forward_seconds, double backward_multiplier, size_t trainers_per_peer,
                        double allreduce_period, double allreduce_stall, double duration_seconds,
                        double bucket_seconds, uint64_t seed, swarm_engine_t* out);
void swarm_engine_destroy(swarm_engine_t e);
size_t swarm_engine_n_trainers(swarm_engine_t e);
/* up to `cap` next records (n = 0: the run reached duration_seconds) */
int swarm_engine_next(swarm_engine_t e, swarm_engine_record* records, size_t cap, size_t* n);
/* SimResult::dispatched / completed / throughput.completed (per bucket) so far */
int swarm_engine_summary(swarm_engine_t e, uint64_t* dispatched, uint64_t* completed, double* buckets,
                         size_t n_buckets, double* now);

/* ---- NCCL transport: stage-to-stage hops and intra-stage all-reduce ------
 * Raw NCCL (resolved at run time: the process's libnccl.so.2, SWARM_NCCL_LIB to
 * override).  One process per GPU; the caller sets the CUDA device first.
 * SWARM_E_UNSUPPORTED when no NCCL library is found. */
typedef struct swarm_comm* swarm_comm_t;
const char* swarm_comm_last_error(void);
int swarm_comm_nccl_version(void);
int swarm_comm_unique_id(void* id /* 128 bytes, ncclUniqueId */);
int swarm_comm_create(const void* id, int nranks, int rank, swarm_comm_t* out); /* ncclCommInitRank */
/* ncclCommSplit: collective over `parent`; color < 0 leaves this rank out (*out = NULL) */
int swarm_comm_split(swarm_comm_t parent, int color, int key, swarm_comm_t* out);
/* the same with ncclConfig_t.maxCTAs = max_ctas (> 0): the CTAs (SMs) its kernels may occupy */
int swarm_comm_split_ex(swarm_comm_t parent, int color, int key, int max_ctas, swarm_comm_t* out);
void swarm_comm_destroy(swarm_comm_t c);
int swarm_comm_size(swarm_comm_t c, int* nranks, int* rank);
int swarm_comm_group_start(void);
int swarm_comm_group_end(void);
/* The stage-to-stage hop (replaces Engine::dispatch_current's queue move,
 * P/src/sim.cpp:405-436, and the link-time model of cost_model.cpp:55-59): one
 * wire message [payload | swarm_wire_header] (swarm_stage_wire_bytes) as a single
 * ncclSend / ncclRecv to / from `peer` (rank in `c`), stream-ordered. */
int swarm_send_compressed(swarm_comm_t c, const void* msg, size_t bytes, int peer, swarm_stream_t stream);
int swarm_recv_compressed(swarm_comm_t c, void* msg, size_t bytes, int peer, swarm_stream_t stream);
/* in-place SUM all-reduce of `count` F32 | BF16 elements */
int swarm_allreduce_sum(swarm_comm_t c, void* buf, size_t count, int dtype, swarm_stream_t stream);
/* The intra-stage gradient averaging (replaces the AllReduceTick stall,
 * P/src/sim.cpp:245-250, :352): SUM of the stage's fp32 gradient arena over the
 * stage's peers (`stage_comm`; NULL or one member: no-op).  The optimizer step that
 * follows divides by the microbatches the stage served (grad_scale). */
int swarm_stage_allreduce(swarm_stage_t st, swarm_comm_t stage_comm, swarm_stream_t stream);

/* ---- host driver: the engine-driven SWARM executor in C++ ------------------
 * Walks engine records (START / HOP / ALLREDUCE / DONE, above) and issues the
 * real work where the reference advances simulated time: visits at START
 * (Engine::start_service, sim.cpp:395-403), transfers for cross-rank HOPs
 * (dispatch_current, :405-436; both halves issued at the consumer's START),
 * all-reduce + AdamW at ALLREDUCE (:245-250, :352).  Placement:
 * world >= n_stages: peer id == rank, `layout[s]` peers on stage s (NULL: even);
 * world < n_stages: each rank hosts n_stages / world consecutive stages.  Every
 * rank runs the same engine on the same seed. */
typedef struct {
    swarm_stage_config model; /* every stage's shapes / wire / optimizer; is_first, is_last, max_slots
                                 (= trainers) and seed (= seed * 1000 + stage) are set per peer */
    int n_stages;
    int world, rank;
    const int* layout;
    double forward_seconds, backward_multiplier, allreduce_period, allreduce_stall, duration_seconds;
    int trainers_per_peer;
    uint64_t seed;
    int lanes;           /* visits a peer serves concurrently (swarm_stage_enable_lanes) */
    int pair_wgrad;      /* paired weight gradients over a peer's consecutive backward visits */
    int use_graphs;      /* CUDA-graph replay of every (peer, kind, trainer, pair, lane) visit */
    int stream_per_peer; /* 0: every local peer shares one stream */
    int n_pool;          /* synthetic token pool size (microbatch (t, k) uses entry (7 t + k) % n_pool) */
    swarm_comm_t comm;   /* world communicator (NULL when world == 1) */
    /* optional full SimConfig (churn trace, rebalancing, peer speeds): when set, it replaces the
       engine fields above and its initial_peers give the layout.  Peer pid lives on rank
       pid * world / n_initial (joiners: pid % world), so any layout runs on any world size
       (peers sharing a GPU sum their gradients locally before the NCCL all-reduce). */
    const swarm_sim_config* sim;
    /* delayed parameter updates: 1 = each tick's all-reduce + AdamW run on an
       update stream, overlapped with the next interval, whose visits use the other weight / gradient bank
       (swarm_stage_enable_banks): one optimizer step of delay */
    int dpu;
    /* optional: the rank of each initial peer (peer ids in stage order, as `layout` / sim's
       initial_peers give them); NULL = pid * world / n_initial.  Lets a caller balance the ranks'
       loads, e.g. spread a heavier stage's peers over several GPUs next to lighter stages' peers. */
    const int* peer_rank;
} swarm_driver_config;
typedef struct {
    uint64_t records, visits, ticks, optimizer_steps, completed, captures, kernels;
    uint32_t n_trainers;
    size_t wire_bytes;
    size_t visit_log_size;
    uint64_t recomputes;   /* backward visits that first recomputed the stage forward (peer changed) */
    uint64_t migrations;   /* MIGRATE records */
    uint64_t state_bytes;  /* params + AdamW state moved to migrating / joining peers */
    size_t n_peers;        /* peers ever created */
} swarm_driver_counters;
typedef struct swarm_driver* swarm_driver_t;
const char* swarm_driver_last_error(void);
int swarm_driver_create(const swarm_driver_config* cfg, swarm_driver_t* out);
void swarm_driver_destroy(swarm_driver_t d);
/* process the driver's own engine records until n more microbatches completed */
int swarm_driver_run(swarm_driver_t d, uint64_t n_microbatches, uint64_t* completed);
/* the same, stopping early right after a record of kind `stop_kind` (>= 0), e.g. SWARM_ENG_LEAVE, or,
 * for stop_kind = -2, right *before* a membership record (LEAVE / JOIN / MIGRATE / MIGRATED) once at
 * least one microbatch completed (the record is processed first by the next call) */
int swarm_driver_run_until(swarm_driver_t d, uint64_t n_microbatches, int stop_kind, uint64_t* completed);
/* membership as the records left it: the peer's stage, liveness, migration state and rank */
int swarm_driver_peer_info(swarm_driver_t d, int peer, int* stage, int* alive, int* migrating, int* rank);
/* the additive hook: one record from any engine that emits the same records in the same
 * order (the driver's own, or the reference Engine patched as INTEGRATION.md §4 shows) */
int swarm_driver_on_record(swarm_driver_t d, const swarm_engine_record* record);
/* every peer stream waits for `stream` (start of a region) / `stream` waits for every peer
 * stream and outstanding transfer (end of a region) */
int swarm_driver_fork(swarm_driver_t d, swarm_stream_t stream);
int swarm_driver_finish(swarm_driver_t d, swarm_stream_t stream);
int swarm_driver_flush_wgrad(swarm_driver_t d);
/* replace the token pool: device copy (host = 0), or pinned host buffers read by each
 * consuming visit (host = 1: end-to-end mode; NULL pointers switch it off) */
int swarm_driver_set_pool(swarm_driver_t d, const int32_t* tokens, const int32_t* targets, int n_pool, int host);
int swarm_driver_pool(swarm_driver_t d, int32_t** tokens, int32_t** targets, int* n_pool, int* tokens_per_microbatch);
float* swarm_driver_loss_sum(swarm_driver_t d); /* device float: token cross-entropy sum x loss scale */
swarm_stage_t swarm_driver_stage(swarm_driver_t d, int peer); /* NULL when the peer is not on this rank */
/* the peer's stream after joining its lanes (e.g. to read its loss) */
swarm_stream_t swarm_driver_peer_stream(swarm_driver_t d, int peer);
swarm_engine_t swarm_driver_engine(swarm_driver_t d);
int swarm_driver_stats(swarm_driver_t d, swarm_driver_counters* stats);
/* Tick cost on this rank's compute streams, cumulative: the GPU time (ms) the peers' streams spent
 * in a tick (the stage gradient sum + all-reduce + AdamW on the lead's stream, the stage-mates
 * waiting for it) or, with dpu, blocked at the first visit after a tick on that bank's update;
 * `spans` = the number of such stretches.  Waits for the GPU to reach the last one. */
int swarm_driver_tick_time(swarm_driver_t d, double* ms, uint64_t* spans);
int swarm_driver_visit_log(swarm_driver_t d, size_t i, uint32_t* trainer, uint64_t* microbatch, uint32_t* stage,
                           int* backward, int64_t* peer);
int swarm_driver_peer_of_rank(swarm_driver_t d, int peer); /* the rank hosting `peer` */
/* Profiled region (bench.py's live roofline): until profile_end every visit runs eagerly on
 * one stream behind a `spin_ns` GPU spin, with the stages' per-kernel CUDA events on
 * (swarm_stage_profile), so each kernel is timed alone.  profile_end sums, over the local
 * stages, the GEMM time (ms), executed GEMM FLOPs and launches, and the per-category
 * time / launches (SWARM_PROF_*), and restores the normal streams. */
int swarm_driver_profile_begin(swarm_driver_t d, uint64_t spin_ns);
int swarm_driver_profile_end(swarm_driver_t d, double* gemm_ms, double* gemm_flops, uint64_t* gemm_launches,
                             double* cat_ms /* [SWARM_PROF_CATEGORIES] */, uint64_t* cat_launches);
/* the profiled region's per-shape GEMM lines over the local stages (swarm_stage_profile_shapes format) */
const char* swarm_driver_profile_shapes(swarm_driver_t d);

#ifdef __cplusplus
}
#endif
#endif /* SWARM_B200_H */
