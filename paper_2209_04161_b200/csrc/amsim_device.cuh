// libamsim device code: the AMSim LUT GEMM core (persistent, one CTA per SM)
// and its operand address maps for dense GEMM and NHWC conv fwd / bwd-data /
// bwd-filter (implicit GEMM).  Citations "PAPER.md:L" are lines of
// /root/reference/PAPER.md; DESIGN.md has the derivation.
//
//  * The CTA holds the 2^(2m)-entry mantissa-product table in shared memory
//    for the whole launch (the paper used texture memory).
//  * Operand k-tiles are staged into shared memory asynchronously (cp.async
//    with zero fill for padding / ragged edges; completion tracked by one
//    mbarrier per stage, STAGES deep) and DECODED ONCE per tile into
//    (alpha, offset) pairs: alpha = sign|exponent bits = +-2^(e-127) or +-0,
//    offset = the top-m mantissa bits pre-scaled to a table byte offset
//    (Alg. 2 l.1-2; reading C1).  The paper decodes inside
//    AMSim for every product.
//  * The 32 lanes of a warp share the A element (same table row) and take
//    32*TN different B columns, so one warp-wide lookup touches a single
//    2^m-entry row (m = 7, 16-bit entries: 64 words on 32 banks, <= 2
//    wavefronts; 8-bit entries -- tables whose mantissas fit 7 bits, e.g.
//    Mitchell at m <= 7: 32 words, 1 wavefront).
//  * Fast path per product: e = LUT[rowoff(a) + off(b)]; x = e*mul_b + alpha_b
//    (integer add into the exponent field: x = +-(1.mant*2^carry)*2^(eb-127);
//    mul_b = 0 makes x = +-0 when b is zero); acc = fma.rn.ftz(x, alpha_a, acc).
//    FTZ realises Alg. 2's Exp <= 0 -> 0.  Taken only for smem tiles whose
//    exponent ranges make it bit-identical to Alg. 2; otherwise the careful
//    path evaluates Alg. 2 literally.
//  * acc starts at +0 and adds products in increasing k (FP32).
#pragma once

#include <cuda.h>  // CUtensorMap (type only; descriptors are encoded through the runtime's driver entry point)
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

namespace amsim {
namespace dev {

#ifndef AMSIM_PACK
#define AMSIM_PACK 1
#endif
#ifndef AMSIM_SKIP
#define AMSIM_SKIP 1
#endif
#ifndef AMSIM_KK_UNROLL_SMALL
#define AMSIM_KK_UNROLL_SMALL 2   // fast-path k unroll for register tiles of <= 64 products
#endif
#ifndef AMSIM_KK_UNROLL_LARGE
#define AMSIM_KK_UNROLL_LARGE 2   // fast-path k unroll for larger register tiles (1 / 4: +0.6 % / +12 %
                                  // on the step, profiles/r02c_ab_unroll_*.jsonl)
#endif
#ifndef AMSIM_PACK8
#define AMSIM_PACK8 0
#endif
#ifndef AMSIM_PACK8A
#define AMSIM_PACK8A 0   // 8-bit tables: pack only the warp-shared A side (alpha | offset)
#endif
#ifndef AMSIM_ROWPRED
#define AMSIM_ROWPRED 0   // zero-row skipping: one predicate per row (lut_row_if16) instead of per lookup
                          // (fewer SASS instructions, but measured 0.7 % slower on the step: off)
#endif
#ifndef AMSIM_DGRAD_SKIP
#define AMSIM_DGRAD_SKIP 1   // zero-row skipping also in the dgrad kernels (dense errors; measured 0.4 %
                             // faster on dgrad than the plain lookups, same box, tools/ab_bench.py)
#endif
#ifndef AMSIM_DECODE_LATE
// 1: every kernel decodes k-tile g right before its lookups (the round-1 order);
// 0: only the 8-bit-table conv fwd / wgrad kernels (issue-bound on layer inputs:
// measured 2-3 % faster there, 1-2 % slower everywhere else, tools/ab_bench.py)
#define AMSIM_DECODE_LATE 0
#endif
#ifndef AMSIM_SKIP_BRANCH
// conv fwd / wgrad in the normal orientation: a zero warp-shared row (ReLU zero)
// is skipped by a warp-uniform branch -- lookups, IMAD and FFMA -- instead of
// predicating only its lookups (measured: ResNet-50 MBM step 729.0 -> 716.0 ms,
// fwd -4.5 %, wgrad -0.9 %; Mitchell 600.6 -> 594.3 ms; profiles/r02b_ab_skipb_tree_*.jsonl)
#define AMSIM_SKIP_BRANCH 1
#endif
#ifndef AMSIM_PACK_ACT
#define AMSIM_PACK_ACT 1      // packed operand words also for the conv fwd / wgrad (layer-input) kernels
                              // (0 measured 2.6 % slower on the step)
#endif
#ifndef AMSIM_ADDR_OR
// table address = row offset | column offset (an ALU-pipe LOP3) instead of + (an
// FMA-pipe IMAD.IADD): measured ResNet-50 MBM step 717.3 -> 707.0 ms, Mitchell
// 594.3 -> 585.4 ms, 16384^3 Mitchell GEMM 5.64 -> 5.79 T/s (same box,
// profiles/r02b_ab_addror_*.jsonl).  Round 1 measured it 3-6 % slower, when the
// per-element decode kept the ALU pipe busy.
#define AMSIM_ADDR_OR 1
#endif
#ifndef AMSIM_SK_TREE
#define AMSIM_SK_TREE 1   // stream-K pieces summed by a binary tree (0: by the last piece, serially)
#endif
#ifndef AMSIM_DA
// interleave the decode of k-tile g+1 with the fast-path lookups of k-tile g
// (1: the configurations where it measured faster with the round-2 per-element
// decode; 2: every 16-row tile; 0: never -- since the quad decode the
// un-interleaved order is 1 % faster on the ResNet-50 step, DA = 1 / 2 / 0:
// 731.8 / 753.1 / 724.8 ms, profiles/r02b_ab_da_mbm.jsonl)
#define AMSIM_DA 0
#endif
#ifndef AMSIM_LATE8
#define AMSIM_LATE8 1   // 8-bit-table conv fwd / wgrad kernels decode each k-tile right before its lookups
#endif

constexpr int BK = 16;
constexpr int STAGES = 3;
constexpr int RAW_PAD = 4;    // row padding of k-contiguous raw tiles (keeps 16-B alignment)
constexpr int MAX_SUB = 9;    // sub-problems per launch (stride phases of dgrad, S <= 3)
constexpr int SK_LEVELS = 9;  // stream-K fix-up tree levels (<= 512 pieces per tile)

// ---------------------------------------------------------------------------
// PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const float *src, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 4 : 0));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const float *src, bool valid)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}

__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar));
}

// TMA: expect `bytes` more transaction bytes on the stage barrier (no arrival),
// then a 2-D tile load that completes them (the tensor map lives in the
// __grid_constant__ kernel parameters).
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

// im2col-mode TMA: pixelsPerColumn output pixels traversed from (w, h, n), each
// reading channelsPerPixel channels from c at the tap offset (offw, offh)
__device__ __forceinline__ void tma_load_im2col_4d(uint32_t dst, const CUtensorMap *map, int c, int w, int h, int n,
                                                   int offw, int offh, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6], {%7, %8};\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar), "h"(uint16_t(offw)),
        "h"(uint16_t(offh))
        : "memory");
}

__device__ __forceinline__ float lds_f32(uint32_t addr)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ float fma_ftz(float a, float b, float c)
{
    float d;
    asm("fma.rn.ftz.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

__device__ __forceinline__ float add_ftz(float a, float b)
{
    float d;
    asm("add.rn.ftz.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// Shared-memory table entry at `addr`, loaded only when `act` != 0 (else `v`
// keeps its previous value): a predicated-off LDS requests no shared-memory
// wavefront.
template <int EB>
__device__ __forceinline__ void lut_entry_if(uint32_t &v, uint32_t addr, uint32_t act)
{
    if constexpr (EB == 16)
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.u16 %0, [%1];\n\t}"
                     : "+r"(v) : "r"(addr), "r"(act));
    else
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.u32 %0, [%1];\n\t}"
                     : "+r"(v) : "r"(addr), "r"(act));
}

// One warp-shared row's TN lookups (TN = 4 or 8, 16-bit entries), all
// predicated on the row's A element being nonzero (`act` != 0): one predicate
// per row instead of one per lookup; an inactive row keeps v[] unchanged.
template <int TN>
__device__ __forceinline__ void lut_row_if16(uint32_t (&v)[TN], const uint32_t (&a)[TN], uint32_t act)
{
    static_assert(TN == 4 || TN == 8, "row-predicated lookups for 4 or 8 columns");
    if constexpr (TN == 4) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %8, 0;\n\t"
                     "@q ld.shared.u16 %0, [%4];\n\t@q ld.shared.u16 %1, [%5];\n\t"
                     "@q ld.shared.u16 %2, [%6];\n\t@q ld.shared.u16 %3, [%7];\n\t}"
                     : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(act));
    } else {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %16, 0;\n\t"
                     "@q ld.shared.u16 %0, [%8];\n\t@q ld.shared.u16 %1, [%9];\n\t"
                     "@q ld.shared.u16 %2, [%10];\n\t@q ld.shared.u16 %3, [%11];\n\t"
                     "@q ld.shared.u16 %4, [%12];\n\t@q ld.shared.u16 %5, [%13];\n\t"
                     "@q ld.shared.u16 %6, [%14];\n\t@q ld.shared.u16 %7, [%15];\n\t}"
                     : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]),
                       "r"(act));
    }
}

// Table entry at byte offset `addr`: a shared-memory address (GL = false) or
// an offset from `gbase`, the global (L2-resident) table (GL = true: tables
// too large for shared memory, m >= 8).
template <int EB, bool GL = false>
__device__ __forceinline__ uint32_t lut_entry(uint32_t addr, const unsigned char *gbase)
{
    uint32_t v;
    if constexpr (!GL) {
        if constexpr (EB == 8)
            asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
        else if constexpr (EB == 16)
            asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
        else
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    } else {
        const unsigned char *q = gbase + addr;
        if constexpr (EB == 8)
            asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(q));
        else if constexpr (EB == 16)
            asm volatile("ld.global.nc.u16 %0, [%1];" : "=r"(v) : "l"(q));
        else
            asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(q));
    }
    return v;
}

// Unsigned division by a runtime constant (n < 2^31).
struct FastDiv {
    uint32_t d, mul, shr;
    __host__ void init(uint32_t div)
    {
        d = div ? div : 1;
        shr = 0;
        while ((1ull << shr) < d) shr++;
        mul = uint32_t(((1ull << 32) * ((1ull << shr) - d)) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const
    {
        return uint32_t((uint64_t(__umulhi(n, mul)) + n) >> shr);
    }
};

// ---------------------------------------------------------------------------
// Problem description: up to MAX_SUB independent sub-GEMMs sharing N (the
// stride phases of dgrad).  Tiles are numbered sub by sub (tile_begin), n
// fastest.  Schedule (amsim_mm_kernel): tiles [0, n_dp) round-robin over the
// grid whole ("data-parallel"), tiles [n_dp, ntiles) by STREAM-K -- their
// k-tiles laid end to end (a tile with K = 0 counts as one position) and cut
// into sk_G equal contiguous ranges, CTA c taking [c W / sk_G, (c+1) W / sk_G).
// A tile cut by a range boundary is computed in pieces whose FP32 partial sums
// are added in increasing k order by the piece that finishes last.

struct SubP {
    int M, K;             // rows and reduction length of this sub-problem
    int tiles_m;
    int kt;               // k-tiles per tile (0 when K = 0)
    int tile_begin;       // first global tile index
    int sk_tile;          // first stream-K tile of this sub (>= tile_begin; tile_end if none)
    int sk_pos;           // stream-K position of tile sk_tile
};

struct OpDesc {
    int kcontig;          // raw tile stored [mn][BK + RAW_PAD] (k contiguous, 1), [BK][BMN] (0), or
                          // [mn][BK] with TMA's 64-byte swizzle (k contiguous, TMA-loaded, 2), or
                          // tap-blocked [BMN / 2^cblk_log2][BK][2^cblk_log2] (one im2col box per tap, 3)
    int vec_log2;         // 0 (4-byte copies) or 2 (16-byte copies along the contiguous dim)
    int cblk_log2;        // kcontig 3: channels per tap block (log2)
};

struct KParams {
    // TMA descriptors of the operands whose smem tile is a box of a tensor
    // (tma_on[0] = A, [1] = B: 0 = gathered with cp.async, 2 / 3 = 2-D / 3-D
    // box, 4 = 4-D im2col box, at the coordinates the operand map's
    // tma_coords() gives).
    CUtensorMap tma[2];
    int tma_on[2];
    int N, tiles_n, nsub, ntiles;
    SubP sub[MAX_SUB];
    int n_dp;             // tiles [0, n_dp) data-parallel (round-robin), the rest stream-K
    int sk_G, sk_W;       // stream-K: CTAs taking part, total positions (k-tiles)
    int grid;             // CTAs launched
    float *C;             // output (ldc-strided rows, A map's out_row)
    float *ws;            // stream-K partial tiles [2 sk_G][TM * TN][NT], then uint32 counters [ntiles - n_dp]
    int64_t ws_elems;     // workspace size in 4-byte words (0: no stream-K)
    int cfg;              // host-side tile configuration id
    int64_t ldc;
    int accumulate;
    OpDesc da, db;
    const void *lut;      // device table (global); copied to shared memory
    int m_bits;
    uint32_t lut_bytes;
    int policy;           // 1 = force the careful path
    int lut_global;       // table read from global memory / L2 (too large for shared memory)
    int ecast_lo, ecast_hi;  // exponent casting (reading C23): normal exponent fields outside [lo, hi] -> 0 / Inf
    int mul;              // MulMode
    int trn;              // transposed orientation (see amsim_mm_kernel)
};

// ---------------------------------------------------------------------------
// Operand address maps: at(s, mn, k) -> address of element (mn, k) of
// sub-problem s (mn = GEMM row for A, column for B) or nullptr for an implicit
// zero (padding, dilation, ragged edge).  A maps also give the output row
// offset of GEMM row `row` (out_row).

struct GemmOp {
    const float *p;
    int64_t ld;
    int MN, K;
    int kcontig;
    __device__ __forceinline__ const float *at(int, int mn, int k) const
    {
        if (mn >= MN || k >= K) return nullptr;
        return kcontig ? p + int64_t(mn) * ld + k : p + int64_t(k) * ld + mn;
    }
    __device__ __forceinline__ int64_t out_row(int, int row, int64_t ldc) const { return int64_t(row) * ldc; }
    // TMA box origin (innermost coordinate first): [k][mn] with mn contiguous, or [mn][k]
    __device__ __forceinline__ void tma_coords(int, int mn0, int k0, int *c) const
    {
        c[0] = kcontig ? k0 : mn0;
        c[1] = kcontig ? mn0 : k0;
        c[2] = 0;
    }
};

struct ConvGeom {
    int N, H, W, C, K, R, S, sh, sw, ph, pw, OH, OW;
    FastDiv fOHOW, fOW, fSC, fC;
};

// fwd A: element (m = (n,oh,ow), k = (kh,kw,ci)) of IM2COL(x) (Alg. 3 l.4)
struct FwdX {
    const float *x;
    ConvGeom g;
    int M, Kd;
    __device__ __forceinline__ const float *at(int, int m, int k) const
    {
        if (m >= M || k >= Kd) return nullptr;
        uint32_t n = g.fOHOW.div(m), r = m - n * uint32_t(g.OH * g.OW);
        uint32_t oh = g.fOW.div(r), ow = r - oh * g.OW;
        uint32_t kh = g.fSC.div(k), r2 = k - kh * uint32_t(g.S * g.C);
        uint32_t kw = g.fC.div(r2), ci = r2 - kw * g.C;
        int ih = int(oh) * g.sh - g.ph + int(kh), iw = int(ow) * g.sw - g.pw + int(kw);
        if (ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) return nullptr;
        return x + ((int64_t(n) * g.H + ih) * g.W + iw) * g.C + ci;
    }
    __device__ __forceinline__ int64_t out_row(int, int row, int64_t ldc) const { return int64_t(row) * ldc; }
    // TMA box origin.  1x1 / stride 1 / unpadded: IM2COL(x) is x viewed as
    // [pixels][C] (2-D).  Otherwise im2col mode (C % BK == 0): the tile's first
    // output pixel (n, oh, ow) gives the base (ow*sw - pw, oh*sh - ph, n), the
    // k-tile's tap (kh, kw) the offsets, its channel chunk c.
    __device__ __forceinline__ void tma_coords(int, int m0, int k0, int *c) const
    {
        if (g.R == 1 && g.S == 1 && g.sh == 1 && g.sw == 1 && g.ph == 0 && g.pw == 0) {
            c[0] = k0;
            c[1] = m0;
            c[2] = 0;
            return;
        }
        uint32_t n = g.fOHOW.div(uint32_t(m0)), r = uint32_t(m0) - n * uint32_t(g.OH * g.OW);
        uint32_t oh = g.fOW.div(r), ow = r - oh * g.OW;
        uint32_t kh = g.fSC.div(uint32_t(k0)), r2 = uint32_t(k0) - kh * uint32_t(g.S * g.C);
        uint32_t kw = g.fC.div(r2), ci = r2 - kw * g.C;
        c[0] = int(ci);
        c[1] = int(ow) * g.sw - g.pw;
        c[2] = int(oh) * g.sh - g.ph;
        c[3] = int(n);
        c[4] = int(kw);
        c[5] = int(kh);
    }
};

// wgrad A: element (mn = (kh,kw,ci), k = (n,oh,ow)) = x[n][oh*s-p+kh][ow*s-p+kw][ci]
// (IM2COL_Weight with the error's dilation skipped)
struct WgX {
    const float *x;
    ConvGeom g;
    int M, Kd;
    __device__ __forceinline__ const float *at(int, int mn, int k) const
    {
        if (mn >= M || k >= Kd) return nullptr;
        uint32_t kh = g.fSC.div(mn), r2 = mn - kh * uint32_t(g.S * g.C);
        uint32_t kw = g.fC.div(r2), ci = r2 - kw * g.C;
        uint32_t n = g.fOHOW.div(k), r = k - n * uint32_t(g.OH * g.OW);
        uint32_t oh = g.fOW.div(r), ow = r - oh * g.OW;
        int ih = int(oh) * g.sh - g.ph + int(kh), iw = int(ow) * g.sw - g.pw + int(kw);
        if (ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) return nullptr;
        return x + ((int64_t(n) * g.H + ih) * g.W + iw) * g.C + ci;
    }
    __device__ __forceinline__ int64_t out_row(int, int row, int64_t ldc) const { return int64_t(row) * ldc; }
    // TMA box origin.  1x1 / stride 1 / unpadded: element (ci, pixel) of x as
    // [pixels][C] (2-D).  Otherwise im2col mode (C % BM == 0, so a row tile lies
    // in one tap): BK output pixels from the k-tile's first (n, oh, ow), BM
    // channels from the row tile's (kh, kw, ci0) -- smem [BK][BM].  When BM is a
    // multiple of C instead (multi-tap, kcontig 3), one box of C channels per tap
    // of the row tile, called with mn0 = the tap block's first row.
    __device__ __forceinline__ void tma_coords(int, int mn0, int k0, int *c) const
    {
        if (g.R == 1 && g.S == 1 && g.sh == 1 && g.sw == 1 && g.ph == 0 && g.pw == 0) {
            c[0] = mn0;
            c[1] = k0;
            c[2] = 0;
            return;
        }
        uint32_t kh = g.fSC.div(uint32_t(mn0)), r2 = uint32_t(mn0) - kh * uint32_t(g.S * g.C);
        uint32_t kw = g.fC.div(r2), ci = r2 - kw * g.C;
        uint32_t n = g.fOHOW.div(uint32_t(k0)), r = uint32_t(k0) - n * uint32_t(g.OH * g.OW);
        uint32_t oh = g.fOW.div(r), ow = r - oh * g.OW;
        if (mn0 >= M) {   // tap block past the last tap (multi-tap boxes): channels out of range, zero-filled
            kh = kw = 0;
            ci = uint32_t(g.C);
        }
        c[0] = int(ci);
        c[1] = int(ow) * g.sw - g.pw;
        c[2] = int(oh) * g.sh - g.ph;
        c[3] = int(n);
        c[4] = int(kw);
        c[5] = int(kh);
    }
};

// dgrad, per stride phase (a, b) in [0,sh) x [0,sw): the output pixels
// h = sh*u + ch with ch = (a - ph) mod sh receive contributions only from the
// taps kh = a, a+sh, ... (the other taps of IM2COL_PLG(pad(dilate(dy))) read
// the dilated zeros, and are skipped exactly, reading C14).
// Taps run in the paper's order: kh' = R-1-kh increasing (reverse_transpose,
// PAPER.md:582), then kw', then co.
struct DgPhase {
    int a, b, ch, cw;     // phase and first output row / column of the phase
    int th, tw;           // valid taps per axis
    int lo_h, lo_w;       // dy row / column read by the phase's output (0, 0) at its tap offset 0 (im2col lower corner)
    int Hp, Wp;           // output rows / columns of the phase
    FastDiv fHpWp, fWp, fTwK;
};

constexpr int MAX_PH_TMA = 4;   // stride-2 dgrad: one im2col descriptor per phase
struct DgDY {
    CUtensorMap ph_map[MAX_PH_TMA];   // per-phase im2col descriptors (strided dgrad, TMA mode 6)
    int ph_tma;                       // ph_map encoded for every phase with taps
    const float *dy;
    ConvGeom g;
    DgPhase ph[MAX_SUB];
    FastDiv fK;
    __device__ __forceinline__ const float *at(int s, int m, int k) const
    {
        const DgPhase &P = ph[s];
        if (m >= g.N * P.Hp * P.Wp || k >= P.th * P.tw * g.K) return nullptr;
        uint32_t n = P.fHpWp.div(m), r = m - n * uint32_t(P.Hp * P.Wp);
        uint32_t u = P.fWp.div(r), v = r - u * P.Wp;
        uint32_t i = P.fTwK.div(k), r2 = k - i * uint32_t(P.tw * g.K);
        uint32_t j = fK.div(r2), co = r2 - j * g.K;
        int kh = P.a + g.sh * (P.th - 1 - int(i)), kw = P.b + g.sw * (P.tw - 1 - int(j));
        int h = g.sh * int(u) + P.ch, w = g.sw * int(v) + P.cw;
        int oh = (h + g.ph - kh) / g.sh, ow = (w + g.pw - kw) / g.sw;  // exact by construction
        if (h + g.ph - kh < 0 || w + g.pw - kw < 0 || oh >= g.OH || ow >= g.OW) return nullptr;
        return dy + ((int64_t(n) * g.OH + oh) * g.OW + ow) * g.K + co;
    }
    __device__ __forceinline__ int64_t out_row(int s, int row, int64_t ldc) const
    {
        const DgPhase &P = ph[s];
        uint32_t n = P.fHpWp.div(row), r = row - n * uint32_t(P.Hp * P.Wp);
        uint32_t u = P.fWp.div(r), v = r - u * P.Wp;
        int h = g.sh * int(u) + P.ch, w = g.sw * int(v) + P.cw;
        return ((int64_t(n) * g.H + h) * g.W + w) * ldc;
    }
    // TMA box origin (stride 1: one phase; 1x1 unpadded at any stride, whose
    // only phase with a tap is (0, 0); stride 2: one im2col descriptor per phase,
    // ph_map[s], mode 6).  1x1 unpadded: dy as [pixels][K].  Otherwise im2col mode over dy (K % BK == 0): output pixel
    // (n, h, w) has base (w + pw - (S-1), h + ph - (R-1), n) and tap (i, j) of the
    // reverse_transpose order reads dy[h + ph - kh] with kh = R-1-i: offsets (j, i).
    __device__ __forceinline__ void tma_coords(int s, int m0, int k0, int *c) const
    {
        if (g.R == 1 && g.S == 1 && g.ph == 0 && g.pw == 0) {
            c[0] = k0;
            c[1] = m0;
            c[2] = 0;
            return;
        }
        const DgPhase &P = ph[s];
        uint32_t n = P.fHpWp.div(uint32_t(m0)), r = uint32_t(m0) - n * uint32_t(P.Hp * P.Wp);
        uint32_t h = P.fWp.div(r), w = r - h * P.Wp;
        uint32_t i = P.fTwK.div(uint32_t(k0)), r2 = uint32_t(k0) - i * uint32_t(P.tw * g.K);
        uint32_t j = fK.div(r2), co = r2 - j * g.K;
        c[0] = int(co);
        c[1] = int(w) + P.lo_w;   // stride 1: pw - (S-1)
        c[2] = int(h) + P.lo_h;   // stride 1: ph - (R-1)
        c[3] = int(n);
        c[4] = int(j);
        c[5] = int(i);
    }
};

// dgrad B: reverse_transpose(w) restricted to the phase's taps:
// element (mn = ci, k = (i, j, co)) = w[kh][kw][ci][co]
struct DgW {
    const float *w;
    ConvGeom g;
    DgPhase ph[MAX_SUB];
    FastDiv fK;
    __device__ __forceinline__ const float *at(int s, int ci, int k) const
    {
        const DgPhase &P = ph[s];
        if (ci >= g.C || k >= P.th * P.tw * g.K) return nullptr;
        uint32_t i = P.fTwK.div(k), r2 = k - i * uint32_t(P.tw * g.K);
        uint32_t j = fK.div(r2), co = r2 - j * g.K;
        int kh = P.a + g.sh * (P.th - 1 - int(i)), kw = P.b + g.sw * (P.tw - 1 - int(j));
        return w + ((int64_t(kh) * g.S + kw) * g.C + ci) * g.K + co;
    }
    // TMA (K % BK == 0, so a k-tile lies inside one tap): box {co, ci, tap} of w
    // viewed as [R*S][C][K]
    __device__ __forceinline__ void tma_coords(int s, int ci0, int k0, int *c) const
    {
        const DgPhase &P = ph[s];
        uint32_t i = P.fTwK.div(uint32_t(k0)), r2 = uint32_t(k0) - i * uint32_t(P.tw * g.K);
        uint32_t j = fK.div(r2), co = r2 - j * g.K;
        int kh = P.a + g.sh * (P.th - 1 - int(i)), kw = P.b + g.sw * (P.tw - 1 - int(j));
        c[0] = int(co);
        c[1] = ci0;
        c[2] = kh * g.S + kw;
    }
};

// ---------------------------------------------------------------------------

// NT threads as WM x WN warps (WN = warps side by side along N); each warp owns
// TM rows x 32*TN columns of the BM x BN CTA tile.
// NP ("narrow"): raw tiles without row padding and one packed word per decoded
// element -- only for launches whose operands are all TMA boxes (no k-contiguous
// cp.async layout) with packed (16/32-bit shared) tables; lets the 64 x 512
// tile (Flat8) fit shared memory.
template <int NT_, int TM_, int TN_, int WN_ = 1, bool NP_ = false>
struct KCfg {
    static constexpr bool NP = NP_;
    static constexpr int NT = NT_;
    static constexpr int NWARPS = NT / 32;
    static constexpr int TM = TM_;
    static constexpr int TN = TN_;
    static constexpr int WN = WN_;
    static constexpr int WM = NWARPS / WN;
    static_assert(WM * WN == NWARPS, "warp grid must cover the CTA");
    static constexpr int BM = WM * TM;
    static constexpr int BN = WN * 32 * TN;
    // first row / column of warp w's sub-tile
    static constexpr __host__ __device__ int wrow(int w) { return (w / WN) * TM; }
    static constexpr __host__ __device__ int wcol(int w) { return (w % WN) * 32 * TN; }
    // a lane owns columns lane * CG + col(c), c < TN: groups of 4 consecutive
    // columns 128 apart when TN is a multiple of 4 (conflict-free LDS.128), else
    // TN consecutive (TN = 2, 3, 5: scalar loads at an odd or 2-word lane stride)
    static constexpr bool G4 = TN % 4 == 0;
    static constexpr int CG = G4 ? 4 : TN;
    static constexpr __host__ __device__ int col(int c) { return G4 ? (c >> 2) * 128 + (c & 3) : c; }
    static constexpr int RAW_A = BM * (BK + (NP ? 0 : RAW_PAD));
    static constexpr int RAW_B = BN * (BK + (NP ? 0 : RAW_PAD));
    static constexpr int RAW_STAGE = RAW_A + RAW_B;        // floats
    static constexpr int DEC = (NP ? 1 : 2) * BK * (BM + BN);   // u32 per buffer (alpha + offset, or packed)
    static size_t smem_bytes(uint32_t lut_bytes)
    {
        // + 1 KB: room to align the shared table to 1 KB (OR-formed table addresses)
        size_t lut = lut_bytes ? ((lut_bytes + 127) & ~size_t(127)) + 1024 : 0;
        return lut + sizeof(float) * RAW_STAGE * STAGES + sizeof(uint32_t) * DEC * 2 + sizeof(uint32_t) * NWARPS * 2 +
               8 * STAGES + 16 + 128;
    }
};

// dgrad operand maps (dense error operands: no zero-row skipping to protect)
template <class Op> struct is_dgrad_op { static constexpr bool value = false; };
template <> struct is_dgrad_op<DgDY> { static constexpr bool value = true; };
template <> struct is_dgrad_op<DgW> { static constexpr bool value = true; };

// conv fwd / wgrad operand maps (layer inputs: ReLU zeros)
template <class Op> struct is_act_op { static constexpr bool value = false; };
template <> struct is_act_op<FwdX> { static constexpr bool value = true; };
template <> struct is_act_op<WgX> { static constexpr bool value = true; };

// Descriptor of sub-problem s: the operand's own per-phase map (DgDY, mode 6)
// or the launch-wide one.
template <class Op>
__device__ __forceinline__ const CUtensorMap *phase_map(const Op &, int, const CUtensorMap *dflt) { return dflt; }
__device__ __forceinline__ const CUtensorMap *phase_map(const DgDY &op, int s, const CUtensorMap *) { return &op.ph_map[s]; }

template <int NT, int ROWS, class Op>
__device__ __forceinline__ void issue_operand(const Op &op, const OpDesc &d, float *raw, int s, int mn0, int k0,
                                              int kend, const float *dummy)
{
    static_assert(ROWS % 4 == 0, "tile rows must be a multiple of 4");
    const int tid = threadIdx.x;
    const int vl = d.vec_log2;
    if constexpr (std::is_same<Op, FwdX>::value) {
        // conv fwd input with C % 4 != 0 (the RGB stem, LeNet): 4-byte gathers, one
        // output pixel per thread -- its (n, oh, ow) decomposed once, the k-tile's
        // (kh, kw, ci) stepped incrementally -- instead of two fast divisions and a
        // 64-bit address per element (~100 SASS instructions each, ncu on the stem)
        if (d.kcontig == 1 && vl == 0) {
            const ConvGeom &g = op.g;
            uint32_t kh = g.fSC.div(uint32_t(k0)), r2 = uint32_t(k0) - kh * uint32_t(g.S * g.C);
            uint32_t kw0 = g.fC.div(r2), ci0 = r2 - kw0 * g.C;
            for (int i = tid; i < ROWS; i += NT) {
                const int m = mn0 + i;
                const bool rowok = m < op.M;
                const uint32_t mm = rowok ? uint32_t(m) : 0u;
                const uint32_t n = g.fOHOW.div(mm), r = mm - n * uint32_t(g.OH * g.OW);
                const uint32_t oh = g.fOW.div(r), ow = r - oh * g.OW;
                const int ihb = int(oh) * g.sh - g.ph, iwb = int(ow) * g.sw - g.pw;
                const float *xb = op.x + int64_t(n) * g.H * g.W * g.C;
                int h = int(kh), w = int(kw0), c = int(ci0);
                const uint32_t dst0 = smem_u32(raw + i * (BK + RAW_PAD));
#pragma unroll
                for (int kk = 0; kk < BK; kk++) {
                    const int ih = ihb + h, iw = iwb + w;
                    const bool ok = rowok && k0 + kk < kend && k0 + kk < op.Kd && unsigned(ih) < unsigned(g.H) &&
                                    unsigned(iw) < unsigned(g.W);
                    const float *src = ok ? xb + (ih * g.W + iw) * g.C + c : dummy;
                    cp_async4(dst0 + kk * 4, src, ok);
                    if (++c == g.C) {
                        c = 0;
                        if (++w == g.S) {
                            w = 0;
                            ++h;
                        }
                    }
                }
            }
            return;
        }
    }
    if constexpr (std::is_same<Op, WgX>::value) {
        // wgrad input with C % 4 != 0 (the RGB stem): raw [BK][ROWS], one weight row
        // (kh, kw, ci) per thread, decomposed once; the k-tile's output pixels
        // (n, oh, ow) stepped incrementally (lanes take consecutive rows: the smem
        // writes stay conflict-free)
        if (d.kcontig == 0 && vl == 0) {
            const ConvGeom &g = op.g;
            const uint32_t kq = uint32_t(min(k0, max(op.Kd - 1, 0)));
            const uint32_t n0 = g.fOHOW.div(kq), rq = kq - n0 * uint32_t(g.OH * g.OW);
            const uint32_t oh0 = g.fOW.div(rq), ow0 = rq - oh0 * g.OW;
            for (int i = tid; i < ROWS; i += NT) {
                const int m = mn0 + i;
                const bool rowok = m < op.M;
                const uint32_t mm = rowok ? uint32_t(m) : 0u;
                const uint32_t kh = g.fSC.div(mm), r2 = mm - kh * uint32_t(g.S * g.C);
                const uint32_t kw = g.fC.div(r2), ci = r2 - kw * g.C;
                int n = int(n0), oh = int(oh0), ow = int(ow0);
                const float *xc = op.x + ci;
#pragma unroll
                for (int kk = 0; kk < BK; kk++) {
                    const int ih = oh * g.sh - g.ph + int(kh), iw = ow * g.sw - g.pw + int(kw);
                    const bool ok = rowok && k0 + kk < kend && k0 + kk < op.Kd && unsigned(ih) < unsigned(g.H) &&
                                    unsigned(iw) < unsigned(g.W);
                    const float *src = ok ? xc + ((int64_t(n) * g.H + ih) * g.W + iw) * g.C : dummy;
                    cp_async4(smem_u32(raw + kk * ROWS + i), src, ok);
                    if (++ow == g.OW) {
                        ow = 0;
                        if (++oh == g.OH) {
                            oh = 0;
                            ++n;
                        }
                    }
                }
            }
            return;
        }
    }
    if (d.kcontig) {  // raw [ROWS][BK + RAW_PAD]
        const int cpr_log2 = 4 - vl;  // chunks per row, BK = 16
        const int total = ROWS << cpr_log2;
        for (int c = tid; c < total; c += NT) {
            int i = c >> cpr_log2, kk = (c & ((1 << cpr_log2) - 1)) << vl;
            int k = k0 + kk;
            const float *src = (k < kend) ? op.at(s, mn0 + i, k) : nullptr;
            uint32_t dst = smem_u32(raw + i * (BK + RAW_PAD) + kk);
            if (vl == 2)
                cp_async16(dst, src ? src : dummy, src != nullptr);
            else
                cp_async4(dst, src ? src : dummy, src != nullptr);
        }
    } else {  // raw [BK][ROWS]
        const int total = (BK * ROWS) >> vl;
        for (int c = tid; c < total; c += NT) {
            // chunks per row: ROWS or ROWS / 4 (compile-time divisors)
            int kk = vl ? c / (ROWS / 4) : c / ROWS;
            int i = (vl ? c % (ROWS / 4) : c % ROWS) << vl;
            int k = k0 + kk;
            const float *src = (k < kend) ? op.at(s, mn0 + i, k) : nullptr;
            uint32_t dst = smem_u32(raw + kk * ROWS + i);
            if (vl == 2)
                cp_async16(dst, src ? src : dummy, src != nullptr);
            else
                cp_async4(dst, src ? src : dummy, src != nullptr);
        }
    }
}

// Decode of one raw operand tile into (alpha, offset) arrays laid out
// [BK][rows], four elements per call (a "quad", one 16-byte shared load):
//  * raw [BK][rows] (kcontig 0) and tap-blocked [rows >> cbl][BK][1 << cbl]
//    (kcontig 3): 4 consecutive rows at one k -> one 16-byte store per array;
//  * k-contiguous raw [rows][BK + RAW_PAD] (cp.async, kcontig 1) and TMA tiles
//    [rows][BK] with the 64-byte swizzle (16-B chunk ^= address bits 8..7,
//    kcontig 2): 4 consecutive k of one row -> 4 coalesced word stores (lanes
//    take consecutive rows, so the 16-byte loads are conflict-free).
// Quad q of the BK * ROWS / 4.  Tracks, over the nonzero exponent fields,
// tmax = max(bits & 0x7F800000) and tmin = min((bits & 0x7F800000) - 1)
// (zeros wrap to 0xFFFFFFFF and drop out of the min).
// PACK: one word per element, alpha (bits 31..23) | offset (bits 22..0;
// shared-memory table offsets are < 2^18), halving the inner loop's operand loads.
struct DecArgs {
    int shift;            // 23 - m
    uint32_t mask;        // 2^m - 1
    int off_shift;        // table offset = off_base + (index << off_shift)
    uint32_t off_base;
    bool ecast;           // exponent casting (reading C23) active: elo > 1 or ehi < 254
    uint32_t elo, ehi;
};

template <int ROWS, bool RAW_ALPHA = false, bool PACK = false>
__device__ __forceinline__ void decode_quad(const float *raw, int kcontig, int cbl, int q, uint32_t *al, uint32_t *off,
                                            const DecArgs &da, uint32_t &tmin, uint32_t &tmax)
{
    static_assert(ROWS % 4 == 0, "tile rows must be a multiple of 4");
    uint32_t u[4];
    int e[4];
    const bool rowq = kcontig == 0 || kcontig == 3;
    if (rowq) {   // 4 consecutive rows at one k
        const int kk = q / (ROWS / 4), i = (q % (ROWS / 4)) * 4;
        const int src = kcontig == 0 ? kk * ROWS + i : (((i >> cbl) * BK + kk) << cbl) | (i & ((1 << cbl) - 1));
        const uint4 v = *reinterpret_cast<const uint4 *>(raw + src);
        u[0] = v.x; u[1] = v.y; u[2] = v.z; u[3] = v.w;
#pragma unroll
        for (int j = 0; j < 4; j++) e[j] = kk * ROWS + i + j;
    } else {      // 4 consecutive k of one row
        const int i = q % ROWS, k4 = (q / ROWS) * 4;
        uint32_t a;
        if (kcontig == 2) {
            a = smem_u32(raw) + uint32_t(i * BK + k4) * 4u;
            a ^= ((a >> 7) & 3u) << 4;
        } else {
            a = smem_u32(raw + i * (BK + RAW_PAD) + k4);
        }
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
        u[0] = v.x; u[1] = v.y; u[2] = v.z; u[3] = v.w;
#pragma unroll
        for (int j = 0; j < 4; j++) e[j] = (k4 + j) * ROWS + i;
    }
    uint32_t A[4], O[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        uint32_t x = u[j];
        if (da.ecast) {   // exponent cast to (1, e, m), reading C23
            const uint32_t ex = (x >> 23) & 0xFFu;
            if (ex != 0 && ex != 255 && (ex < da.elo || ex > da.ehi)) x = (x & 0x80000000u) | (ex > da.ehi ? 0x7F800000u : 0u);
        }
        const uint32_t o = da.off_base + (((x >> da.shift) & da.mask) << da.off_shift);
        const uint32_t t = x & 0x7F800000u;
        tmax = max(tmax, t);
        tmin = min(tmin, t - 1u);
        if constexpr (PACK) {
            A[j] = (x & 0xFF800000u) | o;
        } else {
            A[j] = RAW_ALPHA ? x : (x & 0xFF800000u);
            O[j] = o;
        }
    }
    if (rowq) {
        *reinterpret_cast<uint4 *>(al + e[0]) = make_uint4(A[0], A[1], A[2], A[3]);
        if constexpr (!PACK) *reinterpret_cast<uint4 *>(off + e[0]) = make_uint4(O[0], O[1], O[2], O[3]);
    } else {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            al[e[j]] = A[j];
            if constexpr (!PACK) off[e[j]] = O[j];
        }
    }
}

// Multiply modes (amsim_set_multiply_mode): the AMSim table lookup (the
// product path), or -- measurement instruments for the paper's comparisons --
// the native FP32 multiply (ATnG analog) and direct
// per-product evaluation of a built-in functional model with no table
// (PAPER.md:345-349, 398).
enum MulMode { MUL_LUT = 0, MUL_NATIVE = 1, MUL_DIRECT_EXACT = 2, MUL_DIRECT_MITCHELL = 3, MUL_DIRECT_MBM = 4 };

// Direct evaluation of a model's Alg. 1 entry (carry << 23) | mantissa from
// the operands' truncated fractions.  MUL_DIRECT_EXACT receives the fractions
// as floats 1.f (exponent field 127), the others the in-place 23-bit
// fractions.  Each mirrors the host model of the same name (amsim_host.cpp).
template <int MUL>
__device__ __forceinline__ uint32_t direct_entry(uint32_t oa, uint32_t ob)
{
    if constexpr (MUL == MUL_DIRECT_EXACT) {
        // (1.fa)(1.fb) in [1, 4) is exact in FP32 for m <= 11; exponent 127 or 128
        return __float_as_uint(__fmul_rn(__uint_as_float(oa), __uint_as_float(ob))) - 0x3F800000u;
    } else if constexpr (MUL == MUL_DIRECT_MITCHELL) {
        return oa + ob;  // fa + fb: the carry lands in bit 23
    } else {
        const uint32_t one = 1u << 23;
        uint32_t s = oa + ob;
        if (s < one) {
            uint32_t sig = one + s + (5u << 17);  // 1 + fa + fb + 5/64
            if (sig >= 2 * one) {                 // renormalise (round to nearest even): carry
                uint32_t h = sig >> 1;
                return h + (sig & h & 1u);        // in [2^23, 2^24): (1 << 23) | mantissa
            }
            return sig - one;
        }
        return min(s + (5u << 16), 2 * one - (1u << 8));  // (fa + fb) + 5/128, saturated; carry = 1
    }
}

// TRN (transposed orientation): the kernel computes C^T = op(B)^T op(A)^T for
// a skinny-N problem -- opa is the ORIGINAL B operand's map (its elements are
// the warp-shared rows), opb the original A operand's (lanes), the table is
// used transposed (only symmetric tables, so LUT^T = LUT), and the epilogue /
// reduction write C[opb.out_row(col) + row]: each lane stores TM consecutive
// output channels of one pixel (32-64 contiguous bytes).
template <class Cf, int EB, class OpA, class OpB, bool GL = false, int MUL = MUL_LUT, bool TRN = false>
__global__ void __launch_bounds__(Cf::NT, 1) amsim_mm_kernel(const __grid_constant__ KParams p,
                                                             const __grid_constant__ OpA opa,
                                                             const __grid_constant__ OpB opb)
{
    constexpr int NT = Cf::NT, NWARPS = Cf::NWARPS, TM = Cf::TM, TN = Cf::TN, BM = Cf::BM, BN = Cf::BN;
    constexpr int CG = Cf::CG;
    // packed (alpha | offset) operand words for the LSU-bound 16/32-bit tables in
    // shared memory (global table offsets can exceed 23 bits; the 8-bit path is
    // issue-bound and loses more to the unpacking than it gains: measured
    // +5.7 % / -3.8 % on the ResNet-50 step)
    constexpr bool PK = AMSIM_PACK && MUL == MUL_LUT && !GL && (EB >= 16 || AMSIM_PACK8) &&
                        (AMSIM_PACK_ACT || Cf::NP || !(is_act_op<OpA>::value || is_act_op<OpB>::value));
    // A side packed (the warp-shared rows: broadcast loads); the B side keeps
    // separate alpha / offset arrays unless PK
    constexpr bool PKA = PK || (AMSIM_PACK8A && MUL == MUL_LUT && !GL && EB == 8);
    // Zero-row skipping (normal orientation, LSU-bound 16/32-bit shared tables):
    // a warp-shared A element with a zero exponent field (+-0, subnormal) has
    // alpha_a = +-0, so its products add +-0 to acc (never -0: it starts at +0)
    // and leave it unchanged whatever the entry -- the lookup is predicated off
    // (no wavefront) and the FFMA reuses the column's last entry, a valid table
    // value, so x stays finite under the fast-path conditions.  Same bits.
    // Only for TN >= 4: the per-row predicate costs one LOP3 per row and k,
    // which 1- and 2-column tiles cannot amortise (LeNet-5: +17 % measured).
    constexpr int KK_UNROLL = TM * TN <= 64 ? AMSIM_KK_UNROLL_SMALL : AMSIM_KK_UNROLL_LARGE;
    // dgrad's A operand is the layer error (dense): AMSIM_DGRAD_SKIP = 0 would
    // give its kernels the plain lookups (measured slower, so off)
    constexpr bool DGRAD = is_dgrad_op<OpA>::value || is_dgrad_op<OpB>::value;
    constexpr bool SKIP = AMSIM_SKIP && MUL == MUL_LUT && !GL && EB >= 16 && !TRN && TN >= 4 && (!DGRAD || AMSIM_DGRAD_SKIP);
    constexpr bool ROWPRED = SKIP && AMSIM_ROWPRED && EB == 16 && (TN == 4 || TN == 8);
    // branch-skipping of zero rows (layer-input A operands in the normal
    // orientation: conv fwd / wgrad), also for 8-bit tables
    // (16 x 8 tiles only: with 4 columns per row the branch is not amortised --
    // l2.x.conv2 wgrad on 16 x 4 tiles 7.10 -> 8.07 ms, profiles/r02b_cfg_sweep_b256*.jsonl)
    constexpr bool SKIPB = AMSIM_SKIP_BRANCH && MUL == MUL_LUT && !GL && !TRN && TN >= 8 &&
                           (is_act_op<OpA>::value || is_act_op<OpB>::value);
    constexpr uint32_t AMASK = 0xFF800000u, OMASK = 0x007FFFFFu;
    // table address = row offset + column offset; with AMSIM_ADDR_OR the two are
    // OR-ed (an ALU-pipe LOP3 instead of an FMA-pipe IMAD.IADD): exact because the
    // shared table is aligned to its row size (checked on the host) and the
    // column offset is < the row size
    auto ADDR = [](uint32_t ro, uint32_t co) { return (AMSIM_ADDR_OR && !GL) ? (ro | co) : (ro + co); };
    extern __shared__ __align__(128) unsigned char smem[];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lut_pad = (GL || MUL != MUL_LUT) ? 0u : ((p.lut_bytes + 127u) & ~127u);
    const unsigned char *lut_g = reinterpret_cast<const unsigned char *>(p.lut);
    // the shared table starts 1 KB-aligned (dynamic shared memory already is on
    // sm_100, so this offset is 0 in practice; smem_bytes reserves the room)
    const uint32_t lut_align = lut_pad ? ((1024u - (smem_u32(smem) & 1023u)) & 1023u) : 0u;
    unsigned char *lut_s = smem + lut_align;
    float *raw = reinterpret_cast<float *>(smem + lut_align + lut_pad);
    uint32_t *dec = reinterpret_cast<uint32_t *>(raw + Cf::RAW_STAGE * STAGES);
    uint32_t *wflags = dec + Cf::DEC * 2;  // [2][NWARPS]
    uint64_t *bars = reinterpret_cast<uint64_t *>(wflags + NWARPS * 2);
    volatile int *sk_last = reinterpret_cast<volatile int *>(bars + STAGES);   // stream-K: this CTA adds the last piece

    // table -> shared memory, once per persistent CTA
    if constexpr (!GL && MUL == MUL_LUT) {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.lut);
        uint4 *dst = reinterpret_cast<uint4 *>(lut_s);
        for (uint32_t i = tid; i < p.lut_bytes / 16; i += NT) dst[i] = src[i];
        for (uint32_t i = (p.lut_bytes / 16) * 16 + tid; i < p.lut_bytes; i += NT)
            lut_s[i] = reinterpret_cast<const unsigned char *>(p.lut)[i];
    }
    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) mbar_init(smem_u32(&bars[s]), NT);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int m = p.m_bits;
    const int shift = 23 - m;
    const uint32_t mask = (1u << m) - 1u;
    constexpr int ebytes_log2 = EB == 8 ? 0 : (EB == 16 ? 1 : 2);
    const uint32_t lut_base = GL ? 0u : smem_u32(lut_s);
    // ADDR_OR needs the shared table aligned to its row size (<= 512 B for every
    // shared-memory table): lut_s is 1 KB-aligned above, and a violation would fail
    // loudly instead of reading wrong entries
    if (AMSIM_ADDR_OR && !GL && MUL == MUL_LUT && (lut_base & ((1u << (m + ebytes_log2)) - 1u))) __trap();
    // entry << (32 - EB) restores the Alg. 1 layout (carry << 23) | mantissa
    constexpr uint32_t MULV = MUL != MUL_LUT ? 1u : (EB == 8 ? 65536u : (EB == 16 ? 256u : 1u));
    // decode: table byte offsets (LUT) or in-place truncated fractions (direct)
    const int a_off_shift = MUL == MUL_LUT ? m + ebytes_log2 : shift;
    const int b_off_shift = MUL == MUL_LUT ? ebytes_log2 : shift;
    const uint32_t a_off_base = MUL == MUL_LUT ? lut_base : (MUL == MUL_DIRECT_EXACT ? 0x3F800000u : 0u);
    const uint32_t b_off_base = MUL == MUL_DIRECT_EXACT ? 0x3F800000u : 0u;
    const uint32_t elo = uint32_t(p.ecast_lo), ehi = uint32_t(p.ecast_hi);
    const DecArgs dargs_a{shift, mask, a_off_shift, a_off_base, elo > 1u || ehi < 254u, elo, ehi};
    const DecArgs dargs_b{shift, mask, b_off_shift, b_off_base, elo > 1u || ehi < 254u, elo, ehi};
    const float *dummy = reinterpret_cast<const float *>(p.lut);  // valid global address for 0-byte copies

    // Work units: (tile t, k-tile range [k0, k1)); see SubP for the schedule.
    struct Unit {
        int t, k0, k1, P;   // P: stream-K position of tile t (stream-K units only)
        bool sk;
    };
    struct Sched {
        Unit u;             // u.t < 0: no more work
        int lo, hi;         // this CTA's stream-K position range
    };
    auto sub_of = [&](int t) {
        int s = 0;
        while (s + 1 < p.nsub && t >= p.sub[s + 1].tile_begin) s++;
        return s;
    };
    // stream-K position -> unit (first unit of the CTA's range)
    auto sk_begin = [&](Sched &S) {
        S.u.t = -1;
        S.u.sk = true;
        if (int(blockIdx.x) >= p.sk_G) return;
        S.lo = int(int64_t(blockIdx.x) * p.sk_W / p.sk_G);
        S.hi = int(int64_t(blockIdx.x + 1) * p.sk_W / p.sk_G);
        if (S.lo >= S.hi) return;
        for (int s = 0; s < p.nsub; s++) {
            const SubP &B = p.sub[s];
            const int w = max(B.kt, 1);
            const int tend = s + 1 < p.nsub ? p.sub[s + 1].tile_begin : p.ntiles;
            if (B.sk_tile < tend && S.lo < B.sk_pos + (tend - B.sk_tile) * w) {
                const int i = (S.lo - B.sk_pos) / w;
                S.u.t = B.sk_tile + i;
                S.u.P = B.sk_pos + i * w;
                S.u.k0 = min(S.lo - S.u.P, B.kt);
                S.u.k1 = min(min(S.hi - S.u.P, w), B.kt);
                return;
            }
        }
    };
    auto sched_start = [&](Sched &S) {
        if (int(blockIdx.x) < p.n_dp) {
            S.u.t = blockIdx.x;
            S.u.k0 = 0;
            S.u.k1 = p.sub[sub_of(S.u.t)].kt;
            S.u.sk = false;
        } else {
            sk_begin(S);
        }
    };
    auto sched_next = [&](Sched &S) {
        if (!S.u.sk) {
            const int t = S.u.t + int(gridDim.x);
            if (t < p.n_dp) {
                S.u.t = t;
                S.u.k1 = p.sub[sub_of(t)].kt;
            } else {
                sk_begin(S);
            }
            return;
        }
        const int P = S.u.P + max(p.sub[sub_of(S.u.t)].kt, 1);
        if (P >= S.hi) {
            S.u.t = -1;
            return;
        }
        S.u.t++;
        S.u.P = P;
        const int kt = p.sub[sub_of(S.u.t)].kt;
        S.u.k0 = 0;
        S.u.k1 = min(min(S.hi - P, max(kt, 1)), kt);
    };

    struct Tile {
        int s, m0, n0, kb, ke;
        bool partial;     // a stream-K piece of the tile (partial sums, fixed-order fix-up)
    };
    auto tile_of = [&](const Unit &u) {
        Tile T;
        const int s = sub_of(u.t);
        const SubP &S = p.sub[s];
        const int local = u.t - S.tile_begin;
        T.s = s;
        T.m0 = (local / p.tiles_n) * BM;
        T.n0 = (local % p.tiles_n) * BN;
        T.kb = u.k0 * BK;
        T.ke = min(S.K, u.k1 * BK);
        T.partial = u.sk && (u.k0 > 0 || u.k1 < S.kt);
        return T;
    };
    auto ktiles_of = [&](const Tile &T) { return T.ke > T.kb ? (T.ke - T.kb + BK - 1) / BK : 0; };

    // issue cursor (runs STAGES-1 k-tiles ahead of the compute cursor)
    int ik = 0, ig = 0;
    Sched IS;
    sched_start(IS);
    Tile IT;
    if (IS.u.t >= 0) IT = tile_of(IS.u);
    auto issue_next = [&]() {
        while (IS.u.t >= 0) {
            int kt = ktiles_of(IT);
            if (ik >= kt) {  // empty k range
                sched_next(IS);
                ik = 0;
                if (IS.u.t >= 0) IT = tile_of(IS.u);
                continue;
            }
            int stage = ig % STAGES;
            float *ra = raw + stage * Cf::RAW_STAGE;
            float *rb = ra + Cf::RAW_A;
            int k0 = IT.kb + ik * BK;
            const uint32_t bar = smem_u32(&bars[stage]);
            if (p.tma_on[0] | p.tma_on[1]) {
                if (tid == 0) {
                    // the stage's previous contents were read (generic proxy) before the
                    // last __syncthreads; order those reads before the async-proxy writes
                    fence_proxy_async_smem();
                    mbar_expect_tx(bar, (p.tma_on[0] ? BM * BK * 4 : 0) + (p.tma_on[1] ? BN * BK * 4 : 0));
                    int c[6];
                    auto load = [&](int mode, const CUtensorMap *map, uint32_t dst) {
                        if (mode == 4) tma_load_im2col_4d(dst, map, c[0], c[1], c[2], c[3], c[4], c[5], bar);
                        else if (mode == 3) tma_load_3d(dst, map, c[0], c[1], c[2], bar);
                        else tma_load_2d(dst, map, c[0], c[1], bar);
                    };
                    // mode 5: one im2col box of 2^cblk_log2 channels per tap block of the tile
                    auto load_op = [&](int mode, const CUtensorMap *map, uint32_t dst, const auto &op, int mn0,
                                       int rows, int cbl) {
                        if (mode == 6) {   // per-phase im2col descriptor held by the operand map
                            for (int j = 0; j < rows; j += 256) {
                                op.tma_coords(IT.s, mn0 + j, k0, c);
                                load(4, phase_map(op, IT.s, map), dst + uint32_t(j * BK) * 4u);
                            }
                        } else if (mode == 5) {
                            for (int t = 0; t < (rows >> cbl); t++) {
                                op.tma_coords(IT.s, mn0 + (t << cbl), k0, c);
                                load(4, map, dst + uint32_t(t * (BK << cbl)) * 4u);
                            }
                        } else {
                            // a box holds <= 256 rows: taller tiles (k-contiguous [rows][BK] only) take
                            // several boxes, 256 rows (16 KB, a multiple of the swizzle span) apart
                            for (int j = 0; j < rows; j += 256) {
                                op.tma_coords(IT.s, mn0 + j, k0, c);
                                load(mode, map, dst + uint32_t(j * BK) * 4u);
                            }
                        }
                    };
                    if (p.tma_on[0]) load_op(p.tma_on[0], &p.tma[0], smem_u32(ra), opa, IT.m0, BM, p.da.cblk_log2);
                    if (p.tma_on[1]) load_op(p.tma_on[1], &p.tma[1], smem_u32(rb), opb, IT.n0, BN, p.db.cblk_log2);
                }
            }
            if (!p.tma_on[0]) issue_operand<NT, BM>(opa, p.da, ra, IT.s, IT.m0, k0, IT.ke, dummy);
            if (!p.tma_on[1]) issue_operand<NT, BN>(opb, p.db, rb, IT.s, IT.n0, k0, IT.ke, dummy);
            cp_async_arrive_noinc(bar);
            ig++;
            if (++ik == kt) {
                ik = 0;
                sched_next(IS);
                if (IS.u.t >= 0) IT = tile_of(IS.u);
            }
            return;
        }
    };
    for (int s = 0; s < STAGES - 1; s++) issue_next();

    // Decode-ahead: k-tile g+1 is decoded into the other (alpha, offset) buffer
    // -- interleaved with the lookups of k-tile g on the fast path -- and its
    // exponent ranges are published before the one barrier per k-tile, so the
    // decode's shared-memory latency hides behind the lookups instead of
    // stalling the whole CTA between k-tiles.
    // quads (4 elements, decode_quad) per thread and k-tile; the last round may be partial
    constexpr int TQA = BK * BM / 4, TQB = BK * BN / 4;
    constexpr int NQA = (TQA + NT - 1) / NT, NQB = (TQB + NT - 1) / NT;
    // Interleaving pays for the transposed orientation's 16-row tiles (Big^T /
    // Flat^T / Huge^T: 1.5-3.5 % faster on dense operands, neutral on layer
    // inputs) and for the normal 16 x 8 tile on dense errors (dgrad, 1 %); it
    // costs 2-7 % in the normal orientation's zero-row-skipping loop on layer
    // inputs and for 8-row tiles (tools/cfg_sweep.py with AMSIM_DA = 0 / 1,
    // profiles/r02_cfg_da*.jsonl); elsewhere k-tile g+1 is decoded after the
    // lookups of k-tile g, before the barrier.
    constexpr bool DA = AMSIM_DA != 0 && MUL == MUL_LUT && TM == 16 &&
                        (AMSIM_DA == 2 || (TRN ? TN % 4 == 0 : (DGRAD && TN == 8)));
    static_assert(NQA + NQB <= BK || !DA, "decode-ahead: one quad per kk step");
    static_assert(!Cf::NP || PK, "narrow (NP) tile configurations need the packed operand words");
    constexpr int DSTR = PKA ? 1 : 2;   // decoded words per A element (packed: alpha | offset)
    auto dec_a = [&](int gg) { return dec + (gg & 1) * Cf::DEC; };
    auto raw_of = [&](int gg) { return raw + (gg % STAGES) * Cf::RAW_STAGE; };
    auto wait_raw = [&](int gg) { mbar_wait(smem_u32(&bars[gg % STAGES]), uint32_t((gg / STAGES) & 1)); };
    auto dec_quad_a = [&](int gg, int j, uint32_t &mn, uint32_t &mx) {
        const int q = j * NT + tid;
        if (TQA % NT == 0 || q < TQA) {
            uint32_t *d = dec_a(gg);
            decode_quad<BM, MUL == MUL_NATIVE, PKA>(raw_of(gg), p.da.kcontig, p.da.cblk_log2, q, d, d + BK * BM, dargs_a,
                                                    mn, mx);
        }
    };
    auto dec_quad_b = [&](int gg, int j, uint32_t &mn, uint32_t &mx) {
        const int q = j * NT + tid;
        if (TQB % NT == 0 || q < TQB) {
            uint32_t *d = dec_a(gg) + DSTR * BK * BM;
            decode_quad<BN, MUL == MUL_NATIVE, PK>(raw_of(gg) + Cf::RAW_A, p.db.kcontig, p.db.cblk_log2, q, d, d + BK * BN,
                                                   dargs_b, mn, mx);
        }
    };
    // per-warp exponent ranges of k-tile gg -> wflags[gg & 1][warp]: bytes
    // (Amin, Amax, Bmin, Bmax) of the nonzero exponent fields (decode_quad's
    // tmin / tmax encoding; empty: min 255, max 0)
    auto publish = [&](int gg, uint32_t tamin, uint32_t tamax, uint32_t tbmin, uint32_t tbmax) {
        const uint32_t amin = __reduce_min_sync(0xffffffffu, (min(tamin, 0x7F7FFFFFu) + 1u) >> 23);
        const uint32_t amax = __reduce_max_sync(0xffffffffu, tamax >> 23);
        const uint32_t bmin = __reduce_min_sync(0xffffffffu, (min(tbmin, 0x7F7FFFFFu) + 1u) >> 23);
        const uint32_t bmax = __reduce_max_sync(0xffffffffu, tbmax >> 23);
        if (lane == 0) wflags[(gg & 1) * NWARPS + warp] = amin | (amax << 8) | (bmin << 16) | (bmax << 24);
    };
    auto decode_all = [&](int gg) {
        uint32_t amin = 0xFFFFFFFFu, amax = 0, bmin = 0xFFFFFFFFu, bmax = 0;
#pragma unroll
        for (int j = 0; j < NQA; j++) dec_quad_a(gg, j, amin, amax);
#pragma unroll
        for (int j = 0; j < NQB; j++) dec_quad_b(gg, j, bmin, bmax);
        publish(gg, amin, amax, bmin, bmax);
    };

    float acc[TM][TN];
    uint32_t ecur[TN];   // SKIP: last entry loaded per column
#pragma unroll
    for (int c = 0; c < TN; c++) ecur[c] = 0;
    int g = 0;
    constexpr bool LATE = AMSIM_DECODE_LATE != 0 ||
                          (AMSIM_LATE8 && EB == 8 && MUL == MUL_LUT && (is_act_op<OpA>::value || is_act_op<OpB>::value));
    if (!LATE && ig > 0) {   // the CTA's first k-tile
        wait_raw(0);
        decode_all(0);
        __syncthreads();
    }
    Sched CS;
    sched_start(CS);
    for (; CS.u.t >= 0; sched_next(CS)) {
        const Tile T = tile_of(CS.u);
        const int KT = ktiles_of(T);
#pragma unroll
        for (int r = 0; r < TM; r++)
#pragma unroll
            for (int c = 0; c < TN; c++) acc[r][c] = 0.0f;

        for (int kt = 0; kt < KT; kt++, g++) {
            issue_next();
            const bool has_next = !LATE && ig > g + 1;   // k-tile g+1 exists (the issue cursor has issued it)
            if (LATE) {   // the round-1 order: this k-tile's decode, then the barrier, then its lookups
                wait_raw(g);
                decode_all(g);
                __syncthreads();
            }
            uint32_t *d = dec_a(g);
            uint32_t *a_al = d, *a_off = d + BK * BM, *b_al = d + DSTR * BK * BM, *b_off = b_al + BK * BN;
            // the CTA's exponent ranges: lane w < NWARPS reads warp w's word, one
            // warp-wide reduction per field
            const uint32_t fw = lane < NWARPS ? wflags[(g & 1) * NWARPS + lane] : 0x00FF00FFu;
            const int Amin = int(__reduce_min_sync(0xffffffffu, fw & 0xFFu));
            const int Amax = int(__reduce_max_sync(0xffffffffu, (fw >> 8) & 0xFFu));
            const int Bmin = int(__reduce_min_sync(0xffffffffu, (fw >> 16) & 0xFFu));
            const int Bmax = int(__reduce_max_sync(0xffffffffu, fw >> 24));
            // The fast path equals Alg. 2 bit-for-bit when alpha_a is finite
            // (ea <= 254), x = entry * 2^(eb-127) is finite (eb <= 253) and,
            // for every pair of nonzero operands, 1 <= Exp (ea + eb >= 128)
            // and Exp + carry <= 254 (ea + eb <= 380).  Min / max run over the
            // nonzero elements of the two smem tiles (conservative).
            const bool fast = p.policy == 0 && Amax <= 254 && Bmax <= 253 &&
                              (Amax == 0 || Bmax == 0 || (Amin + Bmin >= 128 && Amax + Bmax <= 380));
            if (has_next) wait_raw(g + 1);
            uint32_t namin = 0xFFFFFFFFu, namax = 0, nbmin = 0xFFFFFFFFu, nbmax = 0;   // k-tile g+1's exponent ranges (fast path)

            const uint32_t *A_al = a_al + Cf::wrow(warp), *A_off = a_off + Cf::wrow(warp);
            // lane columns: groups of 4 consecutive columns, group g at g * 128
            // (TN >= 4: each LDS.128 of a group covers 512 contiguous bytes), else TN consecutive
            const uint32_t *B_al = b_al + Cf::wcol(warp) + lane * CG, *B_off = b_off + Cf::wcol(warp) + lane * CG;
            if constexpr (MUL == MUL_NATIVE) {
                // native FP32 multiply-add of the untruncated operands (IEEE, no FTZ)
#pragma unroll 2
                for (int kk = 0; kk < BK; kk++) {
                    float av[TM], bv[TN];
#pragma unroll
                    for (int r = 0; r < TM; r += 4) {
                        float4 v = *reinterpret_cast<const float4 *>(A_al + kk * BM + r);
                        av[r] = v.x; av[r + 1] = v.y; av[r + 2] = v.z; av[r + 3] = v.w;
                    }
                    if constexpr (TN % 4 == 0) {
#pragma unroll
                        for (int c = 0; c < TN; c += 4) {
                            float4 v = *reinterpret_cast<const float4 *>(B_al + kk * BN + c * 32);
                            bv[c] = v.x; bv[c + 1] = v.y; bv[c + 2] = v.z; bv[c + 3] = v.w;
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < TN; c++) bv[c] = __uint_as_float(B_al[kk * BN + c]);
                    }
#pragma unroll
                    for (int r = 0; r < TM; r++)
#pragma unroll
                        for (int c = 0; c < TN; c++) acc[r][c] = __fmaf_rn(av[r], bv[c], acc[r][c]);
                }
            } else if (fast) {
#pragma unroll KK_UNROLL
                for (int kk = 0; kk < BK; kk++) {
                    if (DA && has_next) {   // decode-ahead slice of k-tile g+1: quad kk
                        if (kk < NQA) dec_quad_a(g + 1, kk, namin, namax);
                        else if (kk < NQA + NQB) dec_quad_b(g + 1, kk - NQA, nbmin, nbmax);
                    }
                    uint32_t aal[TM], aof[TM], bal[TN], bof[TN], mul[TN];
#pragma unroll
                    for (int r = 0; r < TM; r += 4) {
                        uint4 v = *reinterpret_cast<const uint4 *>(A_al + kk * BM + r);
                        if constexpr (PKA) {
                            aal[r] = v.x & AMASK; aal[r + 1] = v.y & AMASK; aal[r + 2] = v.z & AMASK; aal[r + 3] = v.w & AMASK;
                            aof[r] = v.x & OMASK; aof[r + 1] = v.y & OMASK; aof[r + 2] = v.z & OMASK; aof[r + 3] = v.w & OMASK;
                        } else {
                            uint4 o = *reinterpret_cast<const uint4 *>(A_off + kk * BM + r);
                            aal[r] = v.x; aal[r + 1] = v.y; aal[r + 2] = v.z; aal[r + 3] = v.w;
                            aof[r] = o.x; aof[r + 1] = o.y; aof[r + 2] = o.z; aof[r + 3] = o.w;
                        }
                    }
                    if constexpr (TN % 4 == 0) {
#pragma unroll
                        for (int c = 0; c < TN; c += 4) {
                            uint4 v = *reinterpret_cast<const uint4 *>(B_al + kk * BN + c * 32);
                            if constexpr (PK) {
                                bal[c] = v.x & AMASK; bal[c + 1] = v.y & AMASK; bal[c + 2] = v.z & AMASK; bal[c + 3] = v.w & AMASK;
                                bof[c] = v.x & OMASK; bof[c + 1] = v.y & OMASK; bof[c + 2] = v.z & OMASK; bof[c + 3] = v.w & OMASK;
                            } else {
                                uint4 o = *reinterpret_cast<const uint4 *>(B_off + kk * BN + c * 32);
                                bal[c] = v.x; bal[c + 1] = v.y; bal[c + 2] = v.z; bal[c + 3] = v.w;
                                bof[c] = o.x; bof[c + 1] = o.y; bof[c + 2] = o.z; bof[c + 3] = o.w;
                            }
                        }
                    } else if constexpr (TN == 2 && PK) {
                        uint2 v = *reinterpret_cast<const uint2 *>(B_al + kk * BN);
                        bal[0] = v.x & AMASK; bal[1] = v.y & AMASK;
                        bof[0] = v.x & OMASK; bof[1] = v.y & OMASK;
                    } else if constexpr (TN == 2) {
                        uint2 v = *reinterpret_cast<const uint2 *>(B_al + kk * BN);
                        uint2 o = *reinterpret_cast<const uint2 *>(B_off + kk * BN);
                        bal[0] = v.x; bal[1] = v.y;
                        bof[0] = o.x; bof[1] = o.y;
                    } else {
#pragma unroll
                        for (int c = 0; c < TN; c++) {
                            bal[c] = PK ? (B_al[kk * BN + c] & AMASK) : B_al[kk * BN + c];
                            bof[c] = PK ? (B_al[kk * BN + c] & OMASK) : B_off[kk * BN + c];
                        }
                    }
#pragma unroll
                    for (int c = 0; c < TN; c++) mul[c] = min(bal[c] << 1, MULV);
#pragma unroll
                    for (int r = 0; r < TM; r++) {
                        if constexpr (SKIPB) {
                            // a zero warp-shared element: the whole row (lookups, IMAD,
                            // FFMA) is skipped by a warp-uniform branch -- its products
                            // are +-0 and acc + (+-0) = acc (acc is never -0).  (Measured
                            // slower: a vote to mark the branch uniform, 717 -> 740 ms;
                            // issuing row r+1's lookups before row r's math, -> 808 ms;
                            // rows in pairs (both rows' lookups together), 699 -> 895 ms.)
                            if ((aal[r] << 1) == 0u) continue;
#pragma unroll
                            for (int c = 0; c < TN; c++) {
                                const uint32_t e = lut_entry<EB, GL>(ADDR(aof[r], bof[c]), lut_g);
                                const uint32_t x = e * mul[c] + bal[c];
                                acc[r][c] = fma_ftz(__uint_as_float(x), __uint_as_float(aal[r]), acc[r][c]);
                            }
                            continue;
                        }
                        if constexpr (ROWPRED) {
                            uint32_t ad[TN];
#pragma unroll
                            for (int c = 0; c < TN; c++) ad[c] = aof[r] + bof[c];
                            lut_row_if16<TN>(ecur, ad, aal[r] << 1);
                        }
#pragma unroll
                        for (int c = 0; c < TN; c++) {
                            uint32_t e;
                            if constexpr (ROWPRED) {
                                e = ecur[c];
                            } else if constexpr (SKIP) {
                                lut_entry_if<EB>(ecur[c], ADDR(aof[r], bof[c]), aal[r] << 1);
                                e = ecur[c];
                            } else {
                                e = MUL == MUL_LUT ? lut_entry<EB, GL>(ADDR(aof[r], bof[c]), lut_g)
                                                   : direct_entry<MUL>(aof[r], bof[c]);
                            }
                            uint32_t x = e * mul[c] + bal[c];
                            acc[r][c] = fma_ftz(__uint_as_float(x), __uint_as_float(aal[r]), acc[r][c]);
                        }
                    }
                }
            } else {
                // careful path: Alg. 2 literally, readings C4-C7
                for (int kk = 0; kk < BK; kk++) {
#pragma unroll
                    for (int r = 0; r < TM; r++) {
                        uint32_t aal = A_al[kk * BM + r], aof = PKA ? (aal & OMASK) : A_off[kk * BM + r];
                        if (PKA) aal &= AMASK;
                        uint32_t ea = (aal >> 23) & 0xFFu;
#pragma unroll
                        for (int c = 0; c < TN; c++) {
                            uint32_t bal = B_al[kk * BN + Cf::col(c)];
                            uint32_t bof = PK ? (bal & OMASK) : B_off[kk * BN + Cf::col(c)];
                            if (PK) bal &= AMASK;
                            uint32_t eb = (bal >> 23) & 0xFFu;
                            uint32_t ent = (MUL == MUL_LUT ? lut_entry<EB, GL>(aof + bof, lut_g)
                                                           : direct_entry<MUL>(aof, bof)) * MULV;  // (carry << 23) | mantissa
                            uint32_t sgn = (aal ^ bal) & 0x80000000u;
                            int Exp = int(ea + eb) - 127;
                            uint32_t pbits;
                            if (ea == 0 || eb == 0 || Exp <= 0) {
                                pbits = 0u;                                    // +0 (C4, C6, C8)
                            } else if (Exp >= 255) {
                                pbits = sgn | 0x7F800000u;                     // +-Inf (C6)
                            } else {
                                int E = Exp + int((ent >> 23) & 1u);           // Exp + Carry (C3)
                                pbits = (E >= 255) ? (sgn | 0x7F800000u)       // C5
                                                   : (sgn | (uint32_t(E) << 23) | (ent & 0x7FFFFFu));
                            }
                            acc[r][c] = add_ftz(acc[r][c], __uint_as_float(pbits));
                        }
                    }
                }
            }
            if (has_next) {
                if (MUL == MUL_NATIVE || !fast || !DA) decode_all(g + 1);   // not interleaved
                else publish(g + 1, namin, namax, nbmin, nbmax);
            }
            // k-tile g+1 decoded and published; dec[g & 1] and raw stage g free
            if (!LATE) __syncthreads();
        }

        const SubP &S = p.sub[T.s];
        if (T.partial) {
            // Stream-K piece: the tile's pieces (CTAs ca..cb, in k order) are
            // summed by a binary tree fixed by the plan -- node (level l, n)
            // adds the sums of pieces [n 2^l, n 2^l + 2^(l-1)) and
            // [n 2^l + 2^(l-1), (n+1) 2^l) -- so the result is deterministic
            // and nothing waits on another CTA: a CTA stores its subtree's sum
            // in the subtree's leftmost slot ([TM * TN][NT], coalesced; slot 2c
            // for CTA c's first stream-K unit, 2c + 1 for its last) and bumps
            // the node's counter; the second arrival adds the two and climbs.
            // The root's last arrival writes the tile.  (A single last-piece
            // fix-up read all pieces serially: 74 pieces of 128 KB for a
            // 2-tile wgrad at batch 32; the tree's critical path is
            // ceil(log2 P) reads and writes.)
            const int P = CS.u.P, w = max(S.kt, 1);
            auto cta_of = [&](int pos) { return int((int64_t(pos + 1) * p.sk_G - 1) / p.sk_W); };
            auto lo_of = [&](int c) { return int(int64_t(c) * p.sk_W / p.sk_G); };
            auto pid = [&](int c) { return 2 * c + (lo_of(c) < P ? 1 : 0); };
            auto slot = [&](int c) { return p.ws + size_t(pid(c)) * (TM * TN) * NT + tid; };
            const int ca = cta_of(P), cb = cta_of(P + w - 1), np = cb - ca + 1, j = int(blockIdx.x) - ca;
            unsigned *cnt = reinterpret_cast<unsigned *>(p.ws + size_t(2 * p.sk_G) * (TM * TN) * NT);
            bool done = true;   // this CTA ends up holding the whole tile's sum
            if constexpr (!AMSIM_SK_TREE) {
                // round-2 first version: every piece stores its partial sums; the last
                // to arrive (one counter per tile) reads all pieces in increasing k
                float *mine = slot(blockIdx.x);
#pragma unroll
                for (int r = 0; r < TM; r++)
#pragma unroll
                    for (int c = 0; c < TN; c++) __stcg(mine + (r * TN + c) * NT, acc[r][c]);
                __threadfence();
                __syncthreads();
                if (tid == 0) *sk_last = atomicAdd(cnt + pid(ca), 1u) + 1 == unsigned(np);
                __syncthreads();
                if (!*sk_last) continue;
                __threadfence();
#pragma unroll
                for (int r = 0; r < TM; r++)
#pragma unroll
                    for (int c = 0; c < TN; c++) acc[r][c] = 0.0f;
                for (int q = ca; q <= cb; q++) {
                    const float *src = slot(q);
#pragma unroll
                    for (int r = 0; r < TM; r++)
#pragma unroll
                        for (int c = 0; c < TN; c++) acc[r][c] += __ldcg(src + (r * TN + c) * NT);
                }
            }
            for (int l = 1; AMSIM_SK_TREE && (1 << (l - 1)) < np; l++) {
                const int left = (j >> l) << l, right = left + (1 << (l - 1));
                if (right >= np) continue;   // no right subtree: the sum passes through
                const bool mine_left = j < right;
                float *dst = slot(ca + (mine_left ? left : right));   // my subtree's leftmost slot
#pragma unroll
                for (int r = 0; r < TM; r++)
#pragma unroll
                    for (int c = 0; c < TN; c++) __stcg(dst + (r * TN + c) * NT, acc[r][c]);
                __threadfence();
                __syncthreads();
                if (tid == 0) *sk_last = atomicAdd(cnt + (l - 1) * (2 * p.sk_G) + pid(ca + left), 1u) == 1u;
                __syncthreads();
                if (!*sk_last) {
                    done = false;
                    break;
                }
                __threadfence();
                const float *src = slot(ca + (mine_left ? right : left));
#pragma unroll
                for (int r = 0; r < TM; r++)
#pragma unroll
                    for (int c = 0; c < TN; c++) acc[r][c] += __ldcg(src + (r * TN + c) * NT);
            }
            if (!done) continue;
        }
        // epilogue: this thread's TM x TN outputs
        if constexpr (TRN) {
            const int row0 = T.m0 + Cf::wrow(warp);
#pragma unroll
            for (int c = 0; c < TN; c++) {
                int col = T.n0 + Cf::wcol(warp) + lane * CG + Cf::col(c);
                if (col >= p.N) continue;
                float *dst = p.C + opb.out_row(T.s, col, p.ldc) + row0;
                if (row0 + TM <= S.M && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && !p.accumulate) {
#pragma unroll
                    for (int r = 0; r < TM; r += 4)
                        *reinterpret_cast<float4 *>(dst + r) =
                            make_float4(acc[r][c], acc[r + 1][c], acc[r + 2][c], acc[r + 3][c]);
                } else {
#pragma unroll
                    for (int r = 0; r < TM; r++)
                        if (row0 + r < S.M) dst[r] = p.accumulate ? dst[r] + acc[r][c] : acc[r][c];
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < TM; r++) {
                int row = T.m0 + Cf::wrow(warp) + r;
                if (row >= S.M) continue;
                float *dst = p.C + opa.out_row(T.s, row, p.ldc);
                if constexpr (Cf::G4) {
                    // a lane's 4-column groups are contiguous: one 16-byte store per group
#pragma unroll
                    for (int c = 0; c < TN; c += 4) {
                        const int col = T.n0 + Cf::wcol(warp) + lane * CG + Cf::col(c);
                        float *q = dst + col;
                        if (col + 3 < p.N && !p.accumulate && (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
                            *reinterpret_cast<float4 *>(q) = make_float4(acc[r][c], acc[r][c + 1], acc[r][c + 2], acc[r][c + 3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; j++)
                                if (col + j < p.N) q[j] = p.accumulate ? (q[j] + acc[r][c + j]) : acc[r][c + j];
                        }
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < TN; c++) {
                        int col = T.n0 + Cf::wcol(warp) + lane * CG + Cf::col(c);
                        if (col >= p.N) continue;
                        dst[col] = p.accumulate ? (dst[col] + acc[r][c]) : acc[r][c];
                    }
                }
            }
        }
    }
}

}  // namespace dev
}  // namespace amsim
