/*
 * oracle/amsim_oracle.c -- CPU ORACLE for the AMSim hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2209_04161_b200/csrc); neither side includes the other.
 *
 * What it computes (citations are lines of /root/reference/PAPER.md):
 *   - the multiplier functional models `approx_mul(float,float)->float`
 *     (Alg. 1 input; exact = bfloat16-by-truncation, PAPER.md:726-727;
 *     Mitchell = MIT16; MBM = AFM16 stand-in),
 *   - oracle_mul: one approximate product, following Alg. 2
 *     step by step but calling the functional model DIRECTLY per product
 *     ("direct C/C++ simulation") -- no lookup table,
 *   - oracle_gemm: C[i][j] = sum_t mul(A[i][t], B[t][j]) with FP32 accumulation
 *      in increasing t, plus the FP64 sum and sum |p|,
 *   - the convolution passes as the paper formulates them, with every
 *     intermediate materialised: IM2COL + GEMM (Alg. 3),
 *     dilate + IM2COL_Weight + GEMM (Alg. 4 l.4-5),
 *     dilate + pad + IM2COL_PLG + reverse_transpose + GEMM (Alg. 4 l.6-8,
 *     PAPER.md:572-584).
 *
 * Readings of silent / garbled passages are the SURVEY.md section 8(c) readings
 * C1-C22, listed in DESIGN.md; each is cited where it is applied below.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * except the MBM model's FIDELITY to Saadat et al. 2018 ("parity unpinned",
 * reading C17) -- the model is a documented stand-in.
 *
 * Build: gcc -O2 -fopenmp -fPIC -shared -ffp-contract=off (no fast-math: IEEE
 * single-precision adds, no FTZ/DAZ).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* FP32 field access (Alg. 2 masks S_MASK / E_MASK / M_MASK) */

static uint32_t bits_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float float_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t sign_field(uint32_t u) { return u >> 31; }
static uint32_t exp_field(uint32_t u) { return (u >> 23) & 0xFFu; }
static uint32_t mant_field(uint32_t u) { return u & 0x7FFFFFu; }

/* ------------------------------------------------------------------ */
/* Multiplier functional models (the user's approx_mul).
 * Each approximates only the significand product; sign is the XOR and the
 * exponent is the sum.  They are called only on normal
 * operands whose product exponent is in range (Alg. 2 handles the rest).   */

/* Exact multiplier: the true product of the (already truncated) operands,
 * rounded once to FP32.  With m <= 11 mantissa bits per operand the 24-bit
 * significand product is exact in FP32 (bfloat16 = (1,8,7)
 * by bit truncation). */
float oracle_model_exact(float a, float b)
{
    double p = (double)a * (double)b;
    return (float)p;
}

/* Split a normal float into sign, unbiased exponent and fraction x in [0,1):
 * |v| = (1 + x) * 2^E. */
static void split_normal(float v, int *sign, int *E, double *x)
{
    uint32_t u = bits_of(v);
    *sign = (int)sign_field(u);
    *E = (int)exp_field(u) - 127;
    *x = (double)mant_field(u) / 8388608.0; /* 2^23 */
}

/* Mitchell's logarithmic multiplier (MIT16; Mitchell 1962):
 * log2(1+x) ~ x, so log2|AB| ~ Ea + Eb + x + y, and the antilog
 * 2^(n+f) ~ 2^n (1+f) gives
 *     x + y <  1 :  (1 + x + y)   * 2^(Ea+Eb)
 *     x + y >= 1 :  (x + y)       * 2^(Ea+Eb+1)      (carry)
 * Evaluated in double (exact for 23-bit fractions) and rounded once to FP32. */
float oracle_model_mitchell(float a, float b)
{
    int sa, sb, Ea, Eb;
    double x, y;
    split_normal(a, &sa, &Ea, &x);
    split_normal(b, &sb, &Eb, &y);
    double s = x + y, mag;
    if (s < 1.0)
        mag = ldexp(1.0 + s, Ea + Eb);
    else
        mag = ldexp(s, Ea + Eb + 1);
    float r = (float)mag;
    return (sa ^ sb) ? -r : r;
}

/* MBM / AFM16 STAND-IN (reading C17 -- FIDELITY UNPINNED).  The paper only
 * cites Saadat et al. 2018.  Stand-in: Mitchell plus a
 * constant bias-compensation term on the significand,
 *     x + y <  1 :  sig = 1 + x + y + 5/64,  renormalised (carry) if sig >= 2
 *     x + y >= 1 :  sig = x + y + 5/128  (carry), saturated at 2 - 2^-15
 * 5/64 ~ 1/12 = E[xy | x+y<1] (Mitchell's mean deficit), 5/128 ~ 1/24 its
 * normalised counterpart.  The saturation keeps the carry at most 1 (the
 * Alg. 1 contract). */
float oracle_model_mbm(float a, float b)
{
    int sa, sb, Ea, Eb;
    double x, y;
    split_normal(a, &sa, &Ea, &x);
    split_normal(b, &sb, &Eb, &y);
    double s = x + y, sig;
    int e;
    if (s < 1.0) {
        sig = 1.0 + s + 5.0 / 64.0;
        e = Ea + Eb;
        if (sig >= 2.0) { sig = sig / 2.0; e = e + 1; }
    } else {
        sig = s + 5.0 / 128.0;
        e = Ea + Eb + 1;
        if (sig > 2.0 - ldexp(1.0, -15)) sig = 2.0 - ldexp(1.0, -15);
    }
    float r = (float)ldexp(sig, e);
    return (sa ^ sb) ? -r : r;
}

/* Test-only ASYMMETRIC model: exact product of a's significand with b's
 * significand truncated to 3 fraction bits.  Valid under Alg. 1's contract
 * (carry <= 1, sign XOR) but model(a,b) != model(b,a), so any swapped operand
 * order (reading C11) changes results. */
float oracle_model_asym(float a, float b)
{
    uint32_t ub = bits_of(b) & 0xFFF00000u; /* keep sign, exponent, 3 fraction bits */
    double p = (double)a * (double)float_of(ub);
    return (float)p;
}

typedef float (*oracle_model_fn)(float, float);

static oracle_model_fn model_by_id(int id)
{
    switch (id) {
    case 0: return oracle_model_exact;
    case 1: return oracle_model_mitchell;
    case 2: return oracle_model_mbm;
    case 3: return oracle_model_asym;
    default: return 0;
    }
}

/* ------------------------------------------------------------------ */
/* oracle_mul -- one approximate product (SURVEY.md 8(c) "oracle_mul").
 * Returns 0 on success, 1 if the model broke the Alg. 1 contract
 * (reading C10), 2 on a bad model id / m.                                */

enum { ORC_OK = 0, ORC_MODEL = 1, ORC_ARG = 2 };

/* truncation to (1,8,m): clear the low 23-m mantissa bits (PAPER.md:727,
 * reading C1: M_MASK = top-m mantissa bits). */
static uint32_t truncate_m(uint32_t u, int m)
{
    uint32_t low = (m >= 23) ? 0u : ((1u << (23 - m)) - 1u);
    return u & ~low;
}

static int mul_impl(float a, float b, oracle_model_fn model, int m, float *out)
{
    uint32_t ua = bits_of(a), ub = bits_of(b);
    uint32_t sa = sign_field(ua), sb = sign_field(ub);
    int ea = (int)exp_field(ua), eb = (int)exp_field(ub);
    uint32_t s = (sa ^ sb) << 31;                     /* Alg. 2 l.5: (a XOR b) & S_MASK */

    /* step 2: a & E_MASK == 0 or b & E_MASK == 0 -> c = 0;
     * zero and subnormal operands flush (C8); the zero is +0 (C6). */
    if (ea == 0 || eb == 0) { *out = 0.0f; return ORC_OK; }

    /* step 3: Exp = ((a&E_MASK) + (b&E_MASK)) >> 23) - 127 (l.6, reading C2) */
    int Exp = ea + eb - 127;
    if (Exp <= 0) { *out = 0.0f; return ORC_OK; }      /* l.12, before the carry (C4) */
    if (Exp >= 255) { *out = float_of(s | 0x7F800000u); return ORC_OK; } /* l.14-15, signed (C6) */

    if (ea == 255 || eb == 255) {
        /* step 7 (reading C7): an Inf/NaN operand with an in-range Exp.  The
         * model cannot be called on it, so Alg. 2's literal integer arithmetic
         * is followed with (carry, mantissa) taken from one model call on the
         * Alg. 1 probe operands 1.k and 1.j (exponent field 127, sign +,
         * reading C9).  No table is built or read. */
        uint32_t k = mant_field(truncate_m(ua, m)), j = mant_field(truncate_m(ub, m));
        float pa = float_of((127u << 23) | k), pb = float_of((127u << 23) | j);
        uint32_t uc = bits_of(model(pa, pb));
        int ec = (int)exp_field(uc);
        if (sign_field(uc) != 0 || (ec != 127 && ec != 128)) return ORC_MODEL;
        int E = Exp + (ec - 127);                        /* l.16: Exp + Carry (C3) */
        if (E >= 255) { *out = float_of(s | 0x7F800000u); return ORC_OK; } /* C5 */
        *out = float_of(s | ((uint32_t)E << 23) | mant_field(uc));
        return ORC_OK;
    }

    /* step 4: truncate both operands to m mantissa bits. */
    float at = float_of(truncate_m(ua, m)), bt = float_of(truncate_m(ub, m));
    /* step 5: call the functional model directly. */
    uint32_t uc = bits_of(model(at, bt));
    int ec = (int)exp_field(uc);
    /* step 6 */
    if (ec == 255) {
        /* carry overflowed at Exp = 254 (model returned Inf or, for bitwise
         * models, a NaN pattern): +-Inf (reading C5). */
        if (Exp + 1 != 255) return ORC_MODEL;
        *out = float_of(s | 0x7F800000u);
        return ORC_OK;
    }
    if (ec != Exp && ec != Exp + 1) return ORC_MODEL;  /* C10 */
    if ((sign_field(uc) << 31) != s) return ORC_MODEL;
    *out = float_of(uc);
    return ORC_OK;
}

int oracle_mul(float a, float b, int model_id, int m, float *out)
{
    oracle_model_fn model = model_by_id(model_id);
    if (!model || m < 1 || m > 23) return ORC_ARG;
    return mul_impl(a, b, model, m, out);
}

/* Vectorised helper for tests: out[i] = mul(a[i], b[i]). */
int oracle_mul_vec(const float *a, const float *b, int64_t n, int model_id, int m, float *out)
{
    oracle_model_fn model = model_by_id(model_id);
    if (!model || m < 1 || m > 23) return ORC_ARG;
    int err = ORC_OK;
#pragma omp parallel for schedule(static) reduction(max : err)
    for (int64_t i = 0; i < n; i++) {
        int e = mul_impl(a[i], b[i], model, m, &out[i]);
        if (e > err) err = e;
    }
    return err;
}

/* ------------------------------------------------------------------ */
/* Exponent casting to a (1, e, m) format ("the bits of the
 * exponent e can be varied from 1 to 8 provided that a proper exponent casting
 * function is given"; the paper gives none -- reading C23):
 * bias B = 2^(e-1) - 1, normal unbiased exponents [1 - B, B].  A normal FP32
 * operand whose unbiased exponent is above B becomes +-Inf (overflow), below
 * 1 - B +-0 (no subnormals, as Alg. 2 flushes them); zeros,
 * subnormals, Inf and NaN pass unchanged.  e = 8 is the identity.  The cast is
 * applied to both operands before Alg. 2; products and sums stay FP32.     */
float oracle_cast_e(float x, int e)
{
    uint32_t u = bits_of(x);
    int ef = (int)exp_field(u);
    if (e >= 8 || ef == 0 || ef == 255) return x;
    int B = (1 << (e - 1)) - 1;
    int unb = ef - 127;
    if (unb > B) return float_of((u & 0x80000000u) | 0x7F800000u);
    if (unb < 1 - B) return float_of(u & 0x80000000u);
    return x;
}

void oracle_cast_e_vec(const float *in, int64_t n, int e, float *out)
{
    for (int64_t i = 0; i < n; i++) out[i] = oracle_cast_e(in[i], e);
}

/* Direct model call (for the LUT-vs-model exhaustive pins). */
float oracle_model_call(int model_id, float a, float b)
{
    oracle_model_fn model = model_by_id(model_id);
    return model ? model(a, b) : NAN;
}

/* ------------------------------------------------------------------ */
/* oracle_gemm: for each selected row i of A (M x K,
 * row-major) and every column j of B (K x N, row-major):
 *   c32[i][j] = FP32 sequential sum over increasing t from +0.0
 *   c64[i][j] = double sum of the same products
 *   abs64[i][j] = sum |p_t|
 * `rows` (length nrows) selects rows of A; NULL means all M rows in order.
 * Outputs are [nrows][N].  Parallel over rows only (order within a sum is
 * untouched).                                                              */
int oracle_gemm(int model_id, int m, int64_t M, int64_t N, int64_t K,
                const float *A, const float *B, const int64_t *rows, int64_t nrows,
                float *c32, double *c64, double *abs64)
{
    oracle_model_fn model = model_by_id(model_id);
    if (!model || m < 1 || m > 23 || M < 0 || N < 0 || K < 0) return ORC_ARG;
    if (!rows) nrows = M;
    int err = ORC_OK;
#pragma omp parallel for schedule(dynamic, 1) reduction(max : err)
    for (int64_t r = 0; r < nrows; r++) {
        int64_t i = rows ? rows[r] : r;
        for (int64_t j = 0; j < N; j++) {
            float s32 = 0.0f;
            double s64 = 0.0, a64 = 0.0;
            for (int64_t t = 0; t < K; t++) {
                float p;
                int e = mul_impl(A[i * K + t], B[t * N + j], model, m, &p);
                if (e > err) err = e;
                s32 = s32 + p;
                s64 += (double)p;
                a64 += fabs((double)p);
            }
            c32[r * N + j] = s32;
            if (c64) c64[r * N + j] = s64;
            if (abs64) abs64[r * N + j] = a64;
        }
    }
    return err;
}

/* ------------------------------------------------------------------ */
/* Convolution descriptor (TF Conv2D semantics: NHWC input,
 * HWIO weights [R][S][C][K], symmetric zero padding). */
typedef struct {
    int32_t N, H, W, C; /* input NHWC */
    int32_t K, R, S;    /* Cout, KH, KW */
    int32_t stride_h, stride_w, pad_h, pad_w;
} oracle_conv_desc;

static int64_t out_h(const oracle_conv_desc *d) { return (d->H + 2 * d->pad_h - d->R) / d->stride_h + 1; }
static int64_t out_w(const oracle_conv_desc *d) { return (d->W + 2 * d->pad_w - d->S) / d->stride_w + 1; }

static int desc_ok(const oracle_conv_desc *d)
{
    return d->N >= 0 && d->H > 0 && d->W > 0 && d->C > 0 && d->K > 0 && d->R > 0 && d->S > 0 &&
           d->stride_h > 0 && d->stride_w > 0 && d->pad_h >= 0 && d->pad_w >= 0 &&
           d->H + 2 * d->pad_h >= d->R && d->W + 2 * d->pad_w >= d->S;
}

/* IM2COL (Alg. 3 line 4): row r = (n, oh, ow) holds the
 * receptive field of output (oh, ow) in (kh, kw, ci) order, ci fastest;
 * padded taps read 0.  Only the selected rows are materialised.          */
static void im2col_rows(const oracle_conv_desc *d, const float *x, const int64_t *rows, int64_t nrows,
                        float *cols)
{
    int64_t OH = out_h(d), OW = out_w(d), KC = (int64_t)d->R * d->S * d->C;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; r++) {
        int64_t row = rows ? rows[r] : r;
        int64_t n = row / (OH * OW), oh = (row / OW) % OH, ow = row % OW;
        float *dst = cols + r * KC;
        for (int kh = 0; kh < d->R; kh++)
            for (int kw = 0; kw < d->S; kw++)
                for (int ci = 0; ci < d->C; ci++) {
                    int64_t ih = oh * d->stride_h - d->pad_h + kh, iw = ow * d->stride_w - d->pad_w + kw;
                    float v = 0.0f;
                    if (ih >= 0 && ih < d->H && iw >= 0 && iw < d->W)
                        v = x[((n * d->H + ih) * d->W + iw) * d->C + ci];
                    dst[((int64_t)kh * d->S + kw) * d->C + ci] = v;
                }
    }
}

/* Forward pass, Alg. 3: A^l = GEMM(IM2COL(A^{l-1}), W^l); a = activation,
 * b = weight.  W (HWIO) is already the (KH*KW*C) x K matrix.
 * `rows` selects output rows (n, oh, ow); outputs are [nrows][K].          */
int oracle_conv_fwd(int model_id, int m, const oracle_conv_desc *d, const float *x, const float *w,
                    const int64_t *rows, int64_t nrows, float *y32, double *y64, double *abs64)
{
    if (!desc_ok(d)) return ORC_ARG;
    int64_t M = (int64_t)d->N * out_h(d) * out_w(d), KC = (int64_t)d->R * d->S * d->C;
    if (!rows) nrows = M;
    float *cols = (float *)malloc((size_t)(nrows * KC > 0 ? nrows * KC : 1) * sizeof(float));
    if (!cols) return ORC_ARG;
    im2col_rows(d, x, rows, nrows, cols);
    int e = oracle_gemm(model_id, m, nrows, d->K, KC, cols, w, NULL, nrows, y32, y64, abs64);
    free(cols);
    return e;
}

/* Dilation ("inserting zeros between elements based on the
 * stride"): E [N][OH][OW][K] -> D [N][(OH-1)s_h+1][(OW-1)s_w+1][K].        */
static float *dilate(const oracle_conv_desc *d, const float *dy, int64_t *DH, int64_t *DW)
{
    int64_t OH = out_h(d), OW = out_w(d);
    *DH = (OH - 1) * d->stride_h + 1;
    *DW = (OW - 1) * d->stride_w + 1;
    size_t n = (size_t)d->N * (size_t)(*DH) * (size_t)(*DW) * (size_t)d->K;
    float *D = (float *)calloc(n > 0 ? n : 1, sizeof(float));
    if (!D) return NULL;
    for (int64_t n_ = 0; n_ < d->N; n_++)
        for (int64_t oh = 0; oh < OH; oh++)
            for (int64_t ow = 0; ow < OW; ow++)
                for (int64_t k = 0; k < d->K; k++)
                    D[((n_ * (*DH) + oh * d->stride_h) * (*DW) + ow * d->stride_w) * d->K + k] =
                        dy[((n_ * OH + oh) * OW + ow) * d->K + k];
    return D;
}

/* Weight gradient, Alg. 4 lines 4-5 with the dilation
 * materialised ("a naive method ... a separate GPU kernel to perform the
 * dilation"; the paper's fused kernel skips exactly these
 * zeros, reading C14):
 *   Columns[(kh,kw,ci)][(n,y,x)] = Xpad[n][kh+y][kw+x][ci]  over the dilated
 *   grid (y,x) in [0,DH)x[0,DW);  W'[(kh,kw,ci)][co] = GEMM(Columns, D),
 *   a = activation, b = error.
 * `rows` selects rows (kh,kw,ci) of W'; outputs [nrows][K].                 */
int oracle_conv_bwd_filter(int model_id, int m, const oracle_conv_desc *d, const float *x, const float *dy,
                           const int64_t *rows, int64_t nrows, float *dw32, double *dw64, double *abs64)
{
    if (!desc_ok(d)) return ORC_ARG;
    int64_t DH, DW;
    float *D = dilate(d, dy, &DH, &DW);
    if (!D) return ORC_ARG;
    int64_t KC = (int64_t)d->R * d->S * d->C, L = (int64_t)d->N * DH * DW;
    if (!rows) nrows = KC;
    float *cols = (float *)malloc((size_t)(nrows * L > 0 ? nrows * L : 1) * sizeof(float));
    if (!cols) { free(D); return ORC_ARG; }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; r++) {
        int64_t row = rows ? rows[r] : r;
        int64_t kh = row / ((int64_t)d->S * d->C), kw = (row / d->C) % d->S, ci = row % d->C;
        for (int64_t n_ = 0; n_ < d->N; n_++)
            for (int64_t y = 0; y < DH; y++)
                for (int64_t xx = 0; xx < DW; xx++) {
                    int64_t ih = kh + y - d->pad_h, iw = kw + xx - d->pad_w;
                    float v = 0.0f;
                    if (ih >= 0 && ih < d->H && iw >= 0 && iw < d->W)
                        v = x[((n_ * d->H + ih) * d->W + iw) * d->C + ci];
                    cols[r * L + (n_ * DH + y) * DW + xx] = v;
                }
    }
    int e = oracle_gemm(model_id, m, nrows, d->K, L, cols, D, NULL, nrows, dw32, dw64, abs64);
    free(cols);
    free(D);
    return e;
}

/* Preceding-layer gradient, Alg. 4 lines 6-8:
 *   PD = pad(dilate(E)) with pad_top = KH-1-P, pad_bottom = H-1+P-(OH-1)S
 *        per axis (reading C16; PAPER.md:679 leaves it unexplained),
 *   Columns_PLG = IM2COL(PD) with a KHxKW window, stride 1 -> N*H*W rows,
 *   W_r = reverse_transpose(W): W_r[kh'][kw'][co][ci] = W[KH-1-kh'][KW-1-kw'][ci][co]
 *        (PAPER.md:582, 684-685),
 *   Errors^l = GEMM(Columns_PLG, W_r), a = error, b = weight.
 * `rows` selects rows (n,h,w) of dX; outputs [nrows][C].                    */
int oracle_conv_bwd_data(int model_id, int m, const oracle_conv_desc *d, const float *dy, const float *w,
                         const int64_t *rows, int64_t nrows, float *dx32, double *dx64, double *abs64)
{
    if (!desc_ok(d)) return ORC_ARG;
    if (d->pad_h > d->R - 1 || d->pad_w > d->S - 1) return ORC_ARG; /* C16 needs P <= KH-1 */
    int64_t OH = out_h(d), OW = out_w(d), DH, DW;
    float *D = dilate(d, dy, &DH, &DW);
    if (!D) return ORC_ARG;
    int64_t pt = d->R - 1 - d->pad_h, pb = d->H - 1 + d->pad_h - (OH - 1) * d->stride_h;
    int64_t pl = d->S - 1 - d->pad_w, pr = d->W - 1 + d->pad_w - (OW - 1) * d->stride_w;
    int64_t PH = pt + DH + pb, PW = pl + DW + pr; /* = H + KH - 1, W + KW - 1 */
    size_t npd = (size_t)d->N * PH * PW * d->K;
    float *PD = (float *)calloc(npd > 0 ? npd : 1, sizeof(float));
    if (!PD) { free(D); return ORC_ARG; }
    for (int64_t n_ = 0; n_ < d->N; n_++)
        for (int64_t y = 0; y < DH; y++)
            for (int64_t xx = 0; xx < DW; xx++)
                for (int64_t k = 0; k < d->K; k++)
                    PD[((n_ * PH + pt + y) * PW + pl + xx) * d->K + k] = D[((n_ * DH + y) * DW + xx) * d->K + k];
    free(D);

    /* W_r as a (KH*KW*K) x C matrix */
    int64_t KW_ = (int64_t)d->R * d->S * d->K;
    float *Wr = (float *)malloc((size_t)KW_ * d->C * sizeof(float));
    if (!Wr) { free(PD); return ORC_ARG; }
    for (int64_t kh = 0; kh < d->R; kh++)
        for (int64_t kw = 0; kw < d->S; kw++)
            for (int64_t co = 0; co < d->K; co++)
                for (int64_t ci = 0; ci < d->C; ci++)
                    Wr[((kh * d->S + kw) * d->K + co) * d->C + ci] =
                        w[(((d->R - 1 - kh) * d->S + (d->S - 1 - kw)) * d->C + ci) * d->K + co];

    int64_t M = (int64_t)d->N * d->H * d->W;
    if (!rows) nrows = M;
    float *cols = (float *)malloc((size_t)(nrows * KW_ > 0 ? nrows * KW_ : 1) * sizeof(float));
    if (!cols) { free(PD); free(Wr); return ORC_ARG; }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; r++) {
        int64_t row = rows ? rows[r] : r;
        int64_t n_ = row / ((int64_t)d->H * d->W), h = (row / d->W) % d->H, ww = row % d->W;
        for (int64_t kh = 0; kh < d->R; kh++)
            for (int64_t kw = 0; kw < d->S; kw++)
                for (int64_t co = 0; co < d->K; co++)
                    cols[r * KW_ + (kh * d->S + kw) * d->K + co] = PD[((n_ * PH + h + kh) * PW + ww + kw) * d->K + co];
    }
    free(PD);
    int e = oracle_gemm(model_id, m, nrows, d->C, KW_, cols, Wr, NULL, nrows, dx32, dx64, abs64);
    free(cols);
    free(Wr);
    return e;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
