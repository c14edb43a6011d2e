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
/* dx (dtype), dgain/dbias (float, cols; written, not accumulated) from dy,
 * x and the saved statistics.  `workspace` >= swarm_layer_norm_backward_workspace()
 * bytes of device memory. */
size_t swarm_layer_norm_backward_workspace(size_t rows, size_t cols);
int swarm_layer_norm_backward(const void* dy, const void* x, int dtype, size_t rows, size_t cols,
                              const float* gain, const float* mean, const float* rstd, void* dx,
                              float* dgain, float* dbias, void* workspace, swarm_stream_t stream);

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
} swarm_gemm_args;
int swarm_gemm_bf16(const swarm_gemm_args* args, swarm_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SWARM_B200_H */
