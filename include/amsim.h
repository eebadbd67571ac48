/*
 * amsim.h -- C ABI of libamsim: the AMSim approximate-multiply GEMM /
 * convolution hot path of ApproxTrain (arXiv 2209.04161) on NVIDIA B200
 * (sm_100a).  Citations "PAPER.md:L" are lines of the paper's LaTeX source.
 *
 * What the library computes
 *   Every FP32 product a*b inside a GEMM or a 2-D convolution pass is replaced
 *   by AMSim (Alg. 2): the operands' top m mantissa bits
 *   index a 2^(2m)-entry mantissa-product lookup table built from a C
 *   functional model of the multiplier (Alg. 1); exponents
 *   add, signs XOR, and zero / underflow / overflow follow Alg. 2.
 *   Products accumulate in FP32.
 *
 * Readings of silent/garbled passages (DESIGN.md lists all of them):
 *   - M_MASK is the top-m mantissa mask (C1); operands are truncated, the
 *     product keeps the table's full 23-bit mantissa (C15).
 *   - Exp <= 0 -> +0 before the carry is added (C4); Exp >= 255, or Exp = 254
 *     plus a carry, -> (sa^sb)*Inf (C5, C6); zero results are +0 (C6);
 *     zero/subnormal operands give +0 (C8); Inf/NaN operands follow Alg. 2's
 *     literal integer arithmetic (C7).
 *   - Operand order (the table need not be symmetric, C11): the FIRST operand
 *     a indexes the table row.  Conv fwd: a = x, b = w (Alg. 3 l.5);
 *     wgrad: a = x, b = dy (Alg. 4 l.5); dgrad: a = dy, b = w (Alg. 4 l.8).
 *
 * Conventions (all entry points)
 *   - Return AMSIM_OK (0) or an error code; amsim_last_error() gives a
 *     thread-local message.  No C++ exception crosses the ABI.
 *   - Arguments are validated synchronously.  An invalid call returns before
 *     any launch and writes nothing.
 *   - Tensor pointers are DEVICE pointers on the current CUDA device, owned by
 *     the caller; kernels are enqueued on `stream` (NULL = legacy default
 *     stream) and the call returns without synchronising.  Launch failures
 *     return AMSIM_ERR_CUDA; asynchronous faults surface at the caller's next
 *     synchronisation.
 *   - No CPU fallback: without an sm_100 device every compute call returns
 *     AMSIM_ERR_UNSUPPORTED.
 *   - Table placement: a table that fits shared memory (every m <= 7, and
 *     m = 8 with 8/16-bit entries) is replicated in each SM's shared memory;
 *     larger ones (m = 8 with 32-bit entries, m = 9..11: 512 KB - 16 MB) are
 *     read from global memory and stay L2-resident.  Same bits either way.
 *   - Results are deterministic: the same call on the same inputs gives the
 *     same bits (fixed accumulation order per output; split-K partials are
 *     reduced in a fixed order).
 */
#ifndef AMSIM_H
#define AMSIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMSIM_ABI_VERSION 1

typedef enum {
    AMSIM_OK = 0,
    AMSIM_ERR_INVALID_ARG = 1,  /* null pointer, negative size, bad leading dim, bad descriptor */
    AMSIM_ERR_UNSUPPORTED = 2,  /* no sm_100 device, or m outside [1, 11] */
    AMSIM_ERR_MODEL = 3,        /* functional model broke Alg. 1's assumptions at (k, j) */
    AMSIM_ERR_NOMEM = 4,        /* host or device allocation failed */
    AMSIM_ERR_CUDA = 5,         /* CUDA launch / runtime error */
    AMSIM_ERR_IO = 6            /* LUT file: open, magic, version, size or truncation error */
} amsim_status;

/* CUDA stream handle (binary-compatible with cudaStream_t / CUstream). */
typedef struct CUstream_st *amsim_stream_t;

/* ---------------------------------------------------------------------- */
/* Multiplier functional model and lookup table (Alg. 1)                    */

/* The user's approximate multiplier: two FP32 in, the
 * approximate FP32 product out.  Must be pure and deterministic, approximate
 * only the significand product (sign = XOR, exponent = sum),
 * and produce a carry of at most 1. */
typedef float (*amsim_mul_fn)(float a, float b);

/* Opaque LUT handle.  Immutable after creation; safe to share between host
 * threads and to use on several devices (each device gets its own copy,
 * uploaded lazily under a mutex on first use; the upload is a synchronous
 * host operation on a private stream, so a first call made inside a CUDA graph
 * capture works and the graph contains only the compute launches). */
typedef struct amsim_lut amsim_lut;

/* Alg. 1.  For every (k, j) in [0, 2^m)^2 the probe
 * operands A = +1.k and B = +1.j (exponent field 127, k and j in the top m
 * mantissa bits; reading C9) are passed to `model`; the entry is
 *   (carry << 23) | mantissa(C),  carry = exponent(C) > 127.
 * m in [1, 11].  Errors: AMSIM_ERR_INVALID_ARG (null),
 * AMSIM_ERR_UNSUPPORTED (m out of range), AMSIM_ERR_MODEL if C is not a
 * positive normal number with exponent field 127 or 128 (message names k, j).
 * On success *out owns a new handle (free with amsim_lut_destroy). */
amsim_status amsim_lut_build(amsim_mul_fn model, int m_bits, amsim_lut **out);

/* Wrap an existing table of 2^(2m) entries (copied).  Every entry must have
 * bits 31..24 clear else AMSIM_ERR_INVALID_ARG. */
amsim_status amsim_lut_from_entries(const uint32_t *entries, int m_bits, amsim_lut **out);

/* Host view of the 2^(2m) entries, row k = first operand (borrowed pointer,
 * valid until amsim_lut_destroy). */
amsim_status amsim_lut_entries(const amsim_lut *lut, const uint32_t **entries, size_t *count);

/* m, and the device entry width the kernels use: 8 when m >= 7 and every
 * entry's low 16 mantissa bits are zero (carry + 7 fraction bits suffice, e.g.
 * Mitchell at m = 7: a 128-byte row, one shared-memory wavefront), else 16 when
 * every entry's low 8 bits are zero (carry + 15 fraction bits; rows of up to
 * 64 entries already fit one wavefront), else 32.  The width changes the
 * kernels' speed, never their bits. */
amsim_status amsim_lut_info(const amsim_lut *lut, int *m_bits, int *device_entry_bits);

/* LUT binary file ("LUTs are written into binary files"),
 * little-endian: "AMLT", version byte 1, m byte, 2 zero bytes, then the
 * 2^(2m) entries as uint32.  Load errors -> AMSIM_ERR_IO. */
amsim_status amsim_lut_save(const amsim_lut *lut, const char *path);
amsim_status amsim_lut_load(const char *path, amsim_lut **out);

void amsim_lut_destroy(amsim_lut *lut);

/* Exponent casting to a (1, e, m) format ("the bits of the
 * exponent e can be varied from 1 to 8 provided that a proper exponent casting
 * function is given"; reading C23).  Creates a new handle with a
 * copy of src's table whose compute calls first cast BOTH operands of every
 * product to e exponent bits: with bias B = 2^(e-1) - 1, a normal operand of
 * unbiased exponent above B becomes +-Inf, below 1 - B +-0; zeros,
 * subnormals, Inf and NaN are unchanged.  Products and sums stay FP32.
 * e = 8 (the default of every other constructor) is the identity.
 * Errors: AMSIM_ERR_INVALID_ARG (null, e outside [1, 8]), AMSIM_ERR_NOMEM. */
amsim_status amsim_lut_with_exponent_bits(const amsim_lut *src, int e_bits, amsim_lut **out);

/* The exponent width of a handle (8 unless set by amsim_lut_with_exponent_bits). */
amsim_status amsim_lut_exponent_bits(const amsim_lut *lut, int *e_bits);

/* Thread-local description of the last error on this thread ("" if none). */
const char *amsim_last_error(void);

/* Built-in functional models (independent of the test oracle):
 *   exact    -- true product of the operands, rounded once (bfloat16 by
 *               truncation at m = 7),
 *   mitchell -- Mitchell's logarithmic multiplier (MIT16),
 *   mbm      -- AFM16/MBM stand-in (Mitchell + constant bias compensation;
 *               PAPER.md:782-785 only cites it; fidelity unpinned). */
float amsim_model_exact(float a, float b);
float amsim_model_mitchell(float a, float b);
float amsim_model_mbm(float a, float b);

/* ---------------------------------------------------------------------- */
/* GEMM (dense layers)                      */

/* C[i][j] = (accumulate ? C[i][j] : 0) + S[i][j],
 *   S[i][j] = FP32 sum over t of amsim(op(A)[i][t], op(B)[t][j]),
 * row-major storage; op(A) is M x K (A stored M x K with leading dimension
 * lda, or K x M when trans_a), op(B) is K x N (B stored K x N, ldb, or
 * N x K when trans_b), C is M x N with ldc >= N.  S is formed from +0 in
 * increasing t; the tile planner may split t into contiguous chunks to
 * balance the SMs (partials then added in increasing chunk order, on a
 * stream-ordered scratch allocation; policy bit 1 disables splitting).
 * M, N or K = 0 is valid (K = 0 sets C to +0, or leaves it with accumulate).
 * Dense layers: fwd Y = X W (a = x, b = w), wgrad dW = X^T dY (trans_a,
 * a = x, b = dy), dgrad dX = dY W^T (trans_b, a = dy, b = w).
 * Errors: AMSIM_ERR_INVALID_ARG (null pointer with nonzero size, negative
 * size, leading dimension too small), AMSIM_ERR_UNSUPPORTED, AMSIM_ERR_CUDA. */
amsim_status amsim_gemm(const amsim_lut *lut, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
                        const float *A, int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc,
                        int accumulate, amsim_stream_t stream);

/* ---------------------------------------------------------------------- */
/* 2-D convolution (AMCONV2D), TF Conv2D semantics        */

/* Input x: NHWC [N][H][W][C].  Weights w: HWIO [R][S][C][K] (KH = R,
 * KW = S, Cout = K).  Output y / dy: NHWC [N][OH][OW][K] with
 * OH = (H + 2 pad_h - R) / stride_h + 1 (floor), likewise OW.  Symmetric zero
 * padding with pad_h <= R - 1 and pad_w <= S - 1. */
typedef struct {
    int32_t N, H, W, C;
    int32_t K, R, S;
    int32_t stride_h, stride_w, pad_h, pad_w;
} amsim_conv2d_desc;

/* Forward (Alg. 3): y = IM2COL(x) . w as an implicit GEMM
 * (no Columns buffer); a = x, b = w; each output sums over (kh, kw, ci) in
 * increasing order.  Padded taps are exact zeros (reading C14). */
amsim_status amsim_conv2d_fwd(const amsim_lut *lut, const amsim_conv2d_desc *d, const float *x, const float *w,
                              float *y, amsim_stream_t stream);

/* Preceding-layer gradient (Alg. 4 l.6-8):
 * dx = IM2COL_PLG(pad(dilate(dy))) . reverse_transpose(w), computed by
 * implicit GEMM over the taps (kh', kw', co) in the paper's increasing order
 * with the dilated / padded zeros skipped exactly (C14, C16); a = dy, b = w. */
amsim_status amsim_conv2d_bwd_data(const amsim_lut *lut, const amsim_conv2d_desc *d, const float *dy,
                                   const float *w, float *dx, amsim_stream_t stream);

/* Workspace bytes amsim_conv2d_bwd_filter needs for this descriptor (split-K
 * partial sums); 0 when no split is used. */
amsim_status amsim_conv2d_bwd_filter_workspace(const amsim_lut *lut, const amsim_conv2d_desc *d, size_t *bytes);

/* Weight gradient (Alg. 4 l.4-5): dw = IM2COL_W(x) . dy
 * with the error's dilation done by skipping; a = x, b = dy.
 * The reduction over (n, oh, ow) may be split; partials go to `workspace`
 * (>= amsim_conv2d_bwd_filter_workspace bytes, device memory owned by the
 * caller) and are reduced in fixed order.  AMSIM_ERR_INVALID_ARG if the
 * workspace is too small. */
amsim_status amsim_conv2d_bwd_filter(const amsim_lut *lut, const amsim_conv2d_desc *d, const float *x,
                                     const float *dy, float *dw, void *workspace, size_t workspace_bytes,
                                     amsim_stream_t stream);

/* ---------------------------------------------------------------------- */
/* Test and measurement hooks                                               */

/* Execution policy (bit set of the CALLING THREAD, default 0; other threads'
 * calls are unaffected):
 *   bit 0 -- force the literal Alg. 2 careful path everywhere (default: per
 *            smem tile, the FTZ fast path when the tile's exponent ranges make
 *            it bit-identical to Alg. 2, else the careful path);
 *   bit 1 -- never split K: every output is then the FP32 sum from +0 in
 *            increasing k, bit-identical to a sequential reference (default:
 *            the tile planner may split K to balance the SMs; partials are
 *            reduced in a fixed order, so results stay deterministic);
 *   bit 2 -- use the 32-bit device table layout even when the table fits 8
 *            or 16 bits (tests: the layout changes speed, never bits);
 *   bit 3 -- stage every operand tile with cp.async gathers (default: tiles
 *            that are boxes of a tensor -- GEMM operands, conv weights, wgrad
 *            errors, im2col boxes of activations / errors -- are loaded by TMA);
 *   bit 4 -- never use the transposed kernel orientation (default: for a
 *            symmetric table and N << M the planner may make the output
 *            channels the warp-shared rows; same bits);
 *   bit 5 -- gather with cp.async the operand tiles that need several im2col
 *            descriptors or boxes (default TMA: wgrad activation tiles spanning
 *            taps of a power-of-two C >= 32, one box per tap; stride-2 dgrad
 *            error tiles, one descriptor per stride phase).
 * Errors: AMSIM_ERR_INVALID_ARG outside [0, 63]. */
amsim_status amsim_set_path_policy(int policy);

/* Multiply mode (of the calling thread, default AMSIM_MUL_LUT).  The two other modes
 * are measurement instruments for the paper's comparisons, not AMSim:
 *   AMSIM_MUL_LUT    -- AMSim: the table lookup of Alg. 2 (the product path);
 *   AMSIM_MUL_NATIVE -- the same GEMM / conv kernels with the native IEEE FP32
 *                       multiply-add of the UNtruncated operands (ApproxTrain
 *                       with native multiplication, "ATnG");
 *                       the table is not read;
 *   AMSIM_MUL_DIRECT -- the table's functional model evaluated per product on
 *                       the device with no table ("direct simulation",
 *                       PAPER.md:345-349, 398); same bits as AMSIM_MUL_LUT.
 *                       Only for tables built by amsim_lut_build from a
 *                       built-in model, else AMSIM_ERR_UNSUPPORTED at the call.
 * Errors: AMSIM_ERR_INVALID_ARG for an unknown mode. */
#define AMSIM_MUL_LUT 0
#define AMSIM_MUL_NATIVE 1
#define AMSIM_MUL_DIRECT 2
amsim_status amsim_set_multiply_mode(int mode);

/* Kernel launches issued by this library in this process (all entry points). */
uint64_t amsim_launch_count(void);

/* Roofline instrument: shared-memory LUT-lookup microbenchmark.  Runs the
 * lookup pattern of the GEMM inner loop (lanes of a warp share the table
 * row, columns drawn from `b_idx`; m bits, `entry_bits` 8, 16 or 32) for
 * `iters` iterations on every SM and writes the achieved lookups per second
 * to *lookups_per_s (synchronises `stream`). */
amsim_status amsim_bench_lut_lookup(int m_bits, int entry_bits, int iters, const uint32_t *b_idx_host,
                                    size_t n_idx, double *lookups_per_s, amsim_stream_t stream);

int amsim_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* AMSIM_H */
