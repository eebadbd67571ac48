// libamsim device side: the AMSim LUT GEMM core and its operand loaders for
// dense GEMM and NHWC conv fwd / bwd-data / bwd-filter (implicit GEMM).
//
// Citations "PAPER.md:L" are lines of /root/reference/PAPER.md.
//
// Design (DESIGN.md has the full derivation):
//  * Persistent CTAs, one per SM (256 threads = 8 warps), each holding the
//    2^(2m)-entry mantissa-product table in shared memory for the whole
//    launch (the paper used texture memory).
//  * Operand k-tiles are staged into shared memory asynchronously
//    (cp.async with zero-fill for padding / ragged edges, completion tracked
//    by an mbarrier per stage, STAGES deep), then DECODED ONCE per tile into
//    (alpha, offset) pairs: alpha = sign|exponent bits = +-2^(e-127) or +-0,
//    offset = the operand's top-m mantissa bits pre-scaled to a table byte
//    offset (Alg. 2 l.1-2; reading C1).  The paper
//    decodes inside AMSim for every product.
//  * Warp layout: the 32 lanes of a warp share the A element (same table
//    row) and take 32*TN different B columns, so one warp-wide lookup touches
//    a single 2^m-entry row (at m = 7 with 16-bit entries: 64 words over 32
//    banks -> <= 2 wavefronts).
//  * Per product (fast path): e = LUT[rowoff(a) + off(b)]; x = e*mul_b +
//    alpha_b (integer add of the exponent field: x = +-(1.mant * 2^carry) *
//    2^(eb-127), and x = +-0 when b is zero since mul_b = 0); acc =
//    fma.rn.ftz(x, alpha_a, acc).  The FTZ flush of alpha_a*x realises Alg. 2's
//    Exp <= 0 -> 0 rule; the fast path is taken only for smem tiles whose
//    exponent ranges make it bit-identical to Alg. 2 (1 <= Exp and
//    Exp + carry <= 254 for every nonzero pair, no Inf/NaN), else the
//    careful path evaluates Alg. 2 literally.
//  * acc starts at +0 and adds products in increasing k (FP32).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "amsim_internal.h"

namespace amsim {
namespace dev {

constexpr int NT = 256;        // threads per CTA
constexpr int NWARPS = NT / 32;
constexpr int TM = 8;          // rows per warp (all lanes share them)
constexpr int BM = NWARPS * TM;  // 64
constexpr int BK = 16;
constexpr int STAGES = 3;
constexpr int RAW_PAD = 4;     // row padding of k-contiguous raw tiles (keeps 16-B alignment)

// ---------------------------------------------------------------------------
// small PTX helpers

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

template <int EB>
__device__ __forceinline__ uint32_t lds_entry(uint32_t addr)
{
    uint32_t v;
    if constexpr (EB == 16)
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    else
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// Unsigned division by a runtime constant (n < 2^31).
struct FastDiv {
    uint32_t d, mul, shr;
    __host__ void init(uint32_t div)
    {
        d = div;
        shr = 0;
        while ((1ull << shr) < div) shr++;
        mul = uint32_t(((1ull << 32) * ((1ull << shr) - div)) / div + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const
    {
        return uint32_t((uint64_t(__umulhi(n, mul)) + n) >> shr);
    }
};

// ---------------------------------------------------------------------------
// Operand address maps.  at(mn, k) returns the address of operand element
// (mn, k) (mn = GEMM row for A / column for B) or nullptr for an implicit
// zero (padding, dilation, ragged edge).  kcontig: memory is contiguous along
// k (else along mn); vec: elements per copy along the contiguous dimension.

struct GemmOp {
    const float *p;
    int64_t ld;
    int MN, K;
    int kcontig;
    __device__ __forceinline__ const float *at(int mn, int k) const
    {
        if (mn >= MN || k >= K) return nullptr;
        return kcontig ? p + int64_t(mn) * ld + k : p + int64_t(k) * ld + mn;
    }
};

struct ConvGeom {
    int N, H, W, C, K, R, S, sh, sw, ph, pw, OH, OW;
    FastDiv fOHOW, fOW, fSC, fC, fHW, fW;
};

// fwd A: element (m = (n,oh,ow), k = (kh,kw,ci)) of IM2COL(x) (Alg. 3 l.4)
struct FwdX {
    const float *x;
    ConvGeom g;
    int M, Kd;
    __device__ __forceinline__ const float *at(int m, int k) const
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
};

// wgrad A: element (mn = (kh,kw,ci), k = (n,oh,ow)) = x[n][oh*s-p+kh][ow*s-p+kw][ci]
// (IM2COL_Weight with the error's dilation skipped)
struct WgX {
    const float *x;
    ConvGeom g;
    int M, Kd;
    __device__ __forceinline__ const float *at(int mn, int k) const
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
};

// dgrad A: element (m = (n,h,w), k = (kh',kw',co)) of IM2COL_PLG(pad(dilate(dy)))
// (Alg. 4 l.6): tap kh = R-1-kh' reads dy[(h+ph-kh)/sh] when
// the division is exact and in range, else the dilated / padded zero (C16).
struct DgDY {
    const float *dy;
    ConvGeom g;
    int M, Kd;
    __device__ __forceinline__ const float *at(int m, int k) const
    {
        if (m >= M || k >= Kd) return nullptr;
        uint32_t n = g.fHW.div(m), r = m - n * uint32_t(g.H * g.W);
        uint32_t h = g.fW.div(r), w = r - h * g.W;
        uint32_t khp = g.fSC.div(k), r2 = k - khp * uint32_t(g.S * g.K);  // fSC holds S*K here
        uint32_t kwp = g.fC.div(r2), co = r2 - kwp * g.K;                   // fC holds K here
        int kh = g.R - 1 - int(khp), kw = g.S - 1 - int(kwp);
        int th = int(h) + g.ph - kh, tw = int(w) + g.pw - kw;
        if (th < 0 || tw < 0) return nullptr;
        int oh = th / g.sh, ow = tw / g.sw;
        if (oh * g.sh != th || ow * g.sw != tw || oh >= g.OH || ow >= g.OW) return nullptr;
        return dy + ((int64_t(n) * g.OH + oh) * g.OW + ow) * g.K + co;
    }
};

// dgrad B: reverse_transpose(w): element (mn = ci, k = (kh',kw',co))
// = w[R-1-kh'][S-1-kw'][ci][co]
struct DgW {
    const float *w;
    ConvGeom g;
    int Nn, Kd;
    __device__ __forceinline__ const float *at(int ci, int k) const
    {
        if (ci >= Nn || k >= Kd) return nullptr;
        uint32_t khp = g.fSC.div(k), r2 = k - khp * uint32_t(g.S * g.K);
        uint32_t kwp = g.fC.div(r2), co = r2 - kwp * g.K;
        int kh = g.R - 1 - int(khp), kw = g.S - 1 - int(kwp);
        return w + ((int64_t(kh) * g.S + kw) * g.C + ci) * g.K + co;
    }
};

// ---------------------------------------------------------------------------

struct OpDesc {
    int kcontig;  // raw tile stored [mn][BK+PAD] (k contiguous) or [BK][BMN]
    int vec;      // 1 or 4
};

struct KParams {
    int M, N, K;          // GEMM problem (op(A) M x K, op(B) K x N)
    int tiles_m, tiles_n, splits, kchunk;
    float *C;             // output (or split workspace [splits][M][N] when splits > 1)
    int64_t ldc;
    int accumulate;
    OpDesc da, db;
    const void *lut;      // device table (global); copied to smem
    int m_bits;
    uint32_t lut_bytes;
    int policy;           // 1 = force careful
};

template <int TN>
struct Cfg {
    static constexpr int BN = 32 * TN;
    static constexpr int RAW_A = BM * (BK + RAW_PAD) > BK * BM ? BM * (BK + RAW_PAD) : BK * BM;
    static constexpr int RAW_B = BN * (BK + RAW_PAD) > BK * BN ? BN * (BK + RAW_PAD) : BK * BN;
    static constexpr int RAW_STAGE = RAW_A + RAW_B;              // floats
    static constexpr int DEC = 2 * BK * (BM + BN);               // u32 per buffer (al + off)
};

template <int TN>
__host__ size_t smem_bytes(uint32_t lut_bytes)
{
    using C = Cfg<TN>;
    size_t lut = (lut_bytes + 127) & ~size_t(127);
    return lut + sizeof(float) * C::RAW_STAGE * STAGES + sizeof(uint32_t) * C::DEC * 2 +
           sizeof(uint32_t) * NWARPS * 2 + 8 * STAGES + 128;
}

template <class Op>
__device__ __forceinline__ void issue_operand(const Op &op, const OpDesc &d, float *raw, int rows, int mn0, int k0,
                                              int kend, const float *dummy)
{
    const int tid = threadIdx.x;
    // raw layout: kcontig -> [rows][BK + RAW_PAD], else [BK][rows]
    if (d.kcontig) {
        const int cpr = BK / d.vec;  // chunks per row
        const int total = rows * cpr;
        for (int c = tid; c < total; c += NT) {
            int i = c / cpr, kk = (c - i * cpr) * d.vec;
            int k = k0 + kk;
            const float *src = (k < kend) ? op.at(mn0 + i, k) : nullptr;
            uint32_t dst = smem_u32(raw + i * (BK + RAW_PAD) + kk);
            if (d.vec == 4)
                cp_async16(dst, src ? src : dummy, src != nullptr);
            else
                cp_async4(dst, src ? src : dummy, src != nullptr);
        }
    } else {
        const int cpr = rows / d.vec;
        const int total = BK * cpr;
        for (int c = tid; c < total; c += NT) {
            int kk = c / cpr, i = (c - kk * cpr) * d.vec;
            int k = k0 + kk;
            const float *src = (k < kend) ? op.at(mn0 + i, k) : nullptr;
            uint32_t dst = smem_u32(raw + kk * rows + i);
            if (d.vec == 4)
                cp_async16(dst, src ? src : dummy, src != nullptr);
            else
                cp_async4(dst, src ? src : dummy, src != nullptr);
        }
    }
}

// Decode one raw operand tile into (alpha, offset) arrays laid out [BK][rows];
// tracks the min / max exponent field over nonzero elements.
__device__ __forceinline__ void decode_operand(const float *raw, const OpDesc &d, int rows, uint32_t *al,
                                               uint32_t *off, int shift, uint32_t mask, int off_shift,
                                               uint32_t off_base, uint32_t &emin, uint32_t &emax)
{
    const int total = BK * rows;
    for (int e = threadIdx.x; e < total; e += NT) {
        int kk = e / rows, i = e - kk * rows;
        float v = d.kcontig ? raw[i * (BK + RAW_PAD) + kk] : raw[kk * rows + i];
        uint32_t u = __float_as_uint(v);
        uint32_t ex = (u >> 23) & 0xFFu;
        al[e] = u & 0xFF800000u;
        off[e] = off_base + (((u >> shift) & mask) << off_shift);
        if (ex) {
            emin = min(emin, ex);
            emax = max(emax, ex);
        }
    }
}

template <int TN, int EB, class OpA, class OpB>
__global__ void __launch_bounds__(NT, 1) amsim_mm_kernel(const __grid_constant__ KParams p,
                                                         const __grid_constant__ OpA opa,
                                                         const __grid_constant__ OpB opb)
{
    using Cf = Cfg<TN>;
    constexpr int BN = Cf::BN;
    extern __shared__ __align__(128) unsigned char smem[];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lut_pad = (p.lut_bytes + 127u) & ~127u;
    unsigned char *lut_s = smem;
    float *raw = reinterpret_cast<float *>(smem + lut_pad);
    uint32_t *dec = reinterpret_cast<uint32_t *>(raw + Cf::RAW_STAGE * STAGES);
    uint32_t *wflags = dec + Cf::DEC * 2;                        // [2][NWARPS]
    uint64_t *bars = reinterpret_cast<uint64_t *>(wflags + NWARPS * 2);

    // table -> shared memory (once per persistent CTA)
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.lut);
        uint4 *dst = reinterpret_cast<uint4 *>(lut_s);
        for (uint32_t i = tid; i < p.lut_bytes / 16; i += NT) dst[i] = src[i];
        if (p.lut_bytes % 16) {
            for (uint32_t i = (p.lut_bytes / 16) * 16 + tid; i < p.lut_bytes; i += NT)
                lut_s[i] = reinterpret_cast<const unsigned char *>(p.lut)[i];
        }
    }
    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) mbar_init(smem_u32(&bars[s]), NT);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int m = p.m_bits;
    const int shift = 23 - m;
    const uint32_t mask = (1u << m) - 1u;
    constexpr int ebytes_log2 = EB == 16 ? 1 : 2;
    const uint32_t lut_base = smem_u32(lut_s);
    constexpr uint32_t MULV = EB == 16 ? 256u : 1u;

    const int ntiles = p.tiles_m * p.tiles_n * p.splits;
    auto tile_coords = [&](int t, int &m0, int &n0, int &kb, int &ke) {
        int tn = t % p.tiles_n;
        int r = t / p.tiles_n;
        int tm = r % p.tiles_m;
        int s = r / p.tiles_m;
        m0 = tm * BM;
        n0 = tn * BN;
        kb = s * p.kchunk;
        ke = min(p.K, kb + p.kchunk);
    };
    auto ktiles_of = [&](int kb, int ke) { return ke > kb ? (ke - kb + BK - 1) / BK : 0; };

    // issue cursor
    int itile = blockIdx.x, ik = 0, ig = 0;
    auto issue_next = [&]() {
        while (itile < ntiles) {
            int m0, n0, kb, ke;
            tile_coords(itile, m0, n0, kb, ke);
            int kt = ktiles_of(kb, ke);
            if (ik >= kt) {  // (only for empty k ranges)
                itile += gridDim.x;
                ik = 0;
                continue;
            }
            int stage = ig % STAGES;
            float *ra = raw + stage * Cf::RAW_STAGE;
            float *rb = ra + Cf::RAW_A;
            int k0 = kb + ik * BK;
            const float *dummy = reinterpret_cast<const float *>(p.lut);  // valid global address for 0-byte copies
            issue_operand(opa, p.da, ra, BM, m0, k0, ke, dummy);
            issue_operand(opb, p.db, rb, BN, n0, k0, ke, dummy);
            cp_async_arrive_noinc(smem_u32(&bars[stage]));
            ig++;
            if (++ik == kt) {
                ik = 0;
                itile += gridDim.x;
            }
            return;
        }
    };
    for (int s = 0; s < STAGES - 1; s++) issue_next();

    float acc[TM][TN];
    int g = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int m0, n0, kb, ke;
        tile_coords(tile, m0, n0, kb, ke);
        const int KT = ktiles_of(kb, ke);
#pragma unroll
        for (int r = 0; r < TM; r++)
#pragma unroll
            for (int c = 0; c < TN; c++) acc[r][c] = 0.0f;

        for (int kt = 0; kt < KT; kt++, g++) {
            issue_next();
            const int stage = g % STAGES;
            mbar_wait(smem_u32(&bars[stage]), uint32_t((g / STAGES) & 1));
            const float *ra = raw + stage * Cf::RAW_STAGE;
            const float *rb = ra + Cf::RAW_A;
            uint32_t *d = dec + (g & 1) * Cf::DEC;
            uint32_t *a_al = d, *a_off = d + BK * BM, *b_al = d + 2 * BK * BM, *b_off = b_al + BK * BN;
            uint32_t amin = 255, amax = 0, bmin = 255, bmax = 0;
            decode_operand(ra, p.da, BM, a_al, a_off, shift, mask, m + ebytes_log2, lut_base, amin, amax);
            decode_operand(rb, p.db, BN, b_al, b_off, shift, mask, ebytes_log2, 0u, bmin, bmax);
            amin = __reduce_min_sync(0xffffffffu, amin);
            amax = __reduce_max_sync(0xffffffffu, amax);
            bmin = __reduce_min_sync(0xffffffffu, bmin);
            bmax = __reduce_max_sync(0xffffffffu, bmax);
            uint32_t *wf = wflags + (g & 1) * NWARPS;
            if (lane == 0) wf[warp] = amin | (amax << 8) | (bmin << 16) | (bmax << 24);
            __syncthreads();

            uint32_t f = wf[0];
            uint32_t lo = f & 0x00FF00FFu, hi = f & 0xFF00FF00u;  // mins, maxs
#pragma unroll
            for (int w = 1; w < NWARPS; w++) {
                uint32_t v = wf[w];
                lo = __vminu4(lo | 0xFF00FF00u, v | 0xFF00FF00u) & 0x00FF00FFu;
                hi = __vmaxu4(hi, v & 0xFF00FF00u);
            }
            const int Amin = lo & 0xFF, Bmin = (lo >> 16) & 0xFF, Amax = (hi >> 8) & 0xFF, Bmax = hi >> 24;
            // The fast path is bit-identical to Alg. 2 when alpha_a is finite
            // (ea <= 254), x = entry * 2^(eb-127) is finite (eb <= 253) and,
            // for every pair of nonzero operands, 1 <= Exp (ea + eb >= 128)
            // and Exp + carry <= 254 (ea + eb <= 380).  Min/max run over the
            // nonzero elements of the two smem tiles (conservative).
            const bool fast = p.policy == 0 && Amax <= 254 && Bmax <= 253 &&
                              (Amax == 0 || Bmax == 0 || (Amin + Bmin >= 128 && Amax + Bmax <= 380));

            const uint32_t *A_al = a_al + warp * TM, *A_off = a_off + warp * TM;
            const uint32_t *B_al = b_al + lane * TN, *B_off = b_off + lane * TN;
            if (fast) {
#pragma unroll 2
                for (int kk = 0; kk < BK; kk++) {
                    uint32_t aal[TM], aof[TM], bal[TN], bof[TN], mul[TN];
#pragma unroll
                    for (int r = 0; r < TM; r += 4) {
                        uint4 v = *reinterpret_cast<const uint4 *>(A_al + kk * BM + r);
                        uint4 o = *reinterpret_cast<const uint4 *>(A_off + kk * BM + r);
                        aal[r] = v.x; aal[r + 1] = v.y; aal[r + 2] = v.z; aal[r + 3] = v.w;
                        aof[r] = o.x; aof[r + 1] = o.y; aof[r + 2] = o.z; aof[r + 3] = o.w;
                    }
                    if constexpr (TN == 4) {
                        uint4 v = *reinterpret_cast<const uint4 *>(B_al + kk * BN);
                        uint4 o = *reinterpret_cast<const uint4 *>(B_off + kk * BN);
                        bal[0] = v.x; bal[1] = v.y; bal[2] = v.z; bal[3] = v.w;
                        bof[0] = o.x; bof[1] = o.y; bof[2] = o.z; bof[3] = o.w;
                    } else if constexpr (TN == 2) {
                        uint2 v = *reinterpret_cast<const uint2 *>(B_al + kk * BN);
                        uint2 o = *reinterpret_cast<const uint2 *>(B_off + kk * BN);
                        bal[0] = v.x; bal[1] = v.y;
                        bof[0] = o.x; bof[1] = o.y;
                    } else {
                        bal[0] = B_al[kk * BN];
                        bof[0] = B_off[kk * BN];
                    }
#pragma unroll
                    for (int c = 0; c < TN; c++) mul[c] = min(bal[c] << 1, MULV);
#pragma unroll
                    for (int r = 0; r < TM; r++)
#pragma unroll
                        for (int c = 0; c < TN; c++) {
                            uint32_t e = lds_entry<EB>(aof[r] + bof[c]);
                            uint32_t x = e * mul[c] + bal[c];
                            acc[r][c] = fma_ftz(__uint_as_float(x), __uint_as_float(aal[r]), acc[r][c]);
                        }
                }
            } else {
                // careful path: Alg. 2 literally with the
                // readings C4-C7.
                for (int kk = 0; kk < BK; kk++) {
#pragma unroll
                    for (int r = 0; r < TM; r++) {
                        uint32_t aal = A_al[kk * BM + r], aof = A_off[kk * BM + r];
                        uint32_t ea = (aal >> 23) & 0xFFu;
#pragma unroll
                        for (int c = 0; c < TN; c++) {
                            uint32_t bal = B_al[kk * BN + c], bof = B_off[kk * BN + c];
                            uint32_t eb = (bal >> 23) & 0xFFu;
                            uint32_t ent = lds_entry<EB>(aof + bof) * MULV;   // (carry << 23) | mantissa
                            uint32_t sgn = (aal ^ bal) & 0x80000000u;
                            int Exp = int(ea + eb) - 127;
                            uint32_t pbits;
                            if (ea == 0 || eb == 0 || Exp <= 0) {
                                pbits = 0u;                                   // +0 (C4, C6, C8)
                            } else if (Exp >= 255) {
                                pbits = sgn | 0x7F800000u;                    // +-Inf (C6)
                            } else {
                                int E = Exp + int((ent >> 23) & 1u);          // Exp + Carry (C3)
                                pbits = (E >= 255) ? (sgn | 0x7F800000u)      // C5
                                                   : (sgn | (uint32_t(E) << 23) | (ent & 0x7FFFFFu));
                            }
                            acc[r][c] = add_ftz(acc[r][c], __uint_as_float(pbits));
                        }
                    }
                }
            }
        }

        // epilogue: this thread's TM x TN outputs
        {
            int split = tile / (p.tiles_m * p.tiles_n);
            float *Cb = p.C + (p.splits > 1 ? int64_t(split) * p.M * p.N : 0);
#pragma unroll
            for (int r = 0; r < TM; r++) {
                int row = m0 + warp * TM + r;
                if (row >= p.M) continue;
#pragma unroll
                for (int c = 0; c < TN; c++) {
                    int col = n0 + lane * TN + c;
                    if (col >= p.N) continue;
                    float *dst = Cb + int64_t(row) * p.ldc + col;
                    *dst = (p.accumulate && p.splits == 1) ? (*dst + acc[r][c]) : acc[r][c];
                }
            }
        }
    }
}

// Deterministic split-K reduction: C[i][j] (+)= sum_s ws[s][i][j] in
// increasing s.
__global__ void splitk_reduce_kernel(const float *__restrict__ ws, int splits, int M, int N, float *C, int64_t ldc,
                                     int accumulate)
{
    int64_t total = int64_t(M) * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        float s = 0.0f;
        for (int k = 0; k < splits; k++) s += ws[int64_t(k) * total + e];
        int64_t i = e / N, j = e % N;
        float *dst = C + i * ldc + j;
        *dst = accumulate ? (*dst + s) : s;
    }
}

__global__ void fill_zero_kernel(float *C, int M, int N, int64_t ldc)
{
    int64_t total = int64_t(M) * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x)
        C[(e / N) * ldc + e % N] = 0.0f;
}

// ---------------------------------------------------------------------------
// LUT-lookup microbenchmark (roofline instrument): the fast path's lookup
// pattern (row shared by the warp, per-lane column offsets) without operand
// traffic: each iteration does TM x TN lookups + IMAD + FFMA.
template <int EB>
__global__ void __launch_bounds__(NT, 1) lut_bench_kernel(const void *lut, uint32_t lut_bytes, int m,
                                                          const uint32_t *bidx, int nidx, int iters, float *out)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const uint4 *src = reinterpret_cast<const uint4 *>(lut);
    for (uint32_t i = threadIdx.x; i < lut_bytes / 16; i += NT) reinterpret_cast<uint4 *>(smem)[i] = src[i];
    __syncthreads();
    constexpr int ebl = EB == 16 ? 1 : 2;
    const uint32_t base = smem_u32(smem);
    const int warp = threadIdx.x >> 5;
    const uint32_t rmask = (1u << m) - 1u;
    uint32_t bof[4], row[TM];
    for (int c = 0; c < 4; c++) bof[c] = base + (bidx[(blockIdx.x * NT + threadIdx.x * 4 + c) % nidx] << ebl);
    for (int r = 0; r < TM; r++) row[r] = ((warp * 37 + r * 11 + blockIdx.x) * 13) & rmask;
    float acc[TM][4] = {};
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < TM; r++) {
            const uint32_t aof = ((row[r] + uint32_t(it)) & rmask) << (m + ebl);  // warp-uniform row walk
#pragma unroll
            for (int c = 0; c < 4; c++) {
                uint32_t e = lds_entry<EB>(aof + bof[c]);
                acc[r][c] = fma_ftz(__uint_as_float(e * 256u + 0x3F800000u), 1.0f, acc[r][c]);
            }
        }
    }
    float s = 0.f;
    for (int r = 0; r < TM; r++)
        for (int c = 0; c < 4; c++) s += acc[r][c];
    out[blockIdx.x * NT + threadIdx.x] = s;
}

}  // namespace dev

// ===========================================================================
// Host dispatch

using namespace dev;

static int g_num_sms = 0;
static int num_sms()
{
    if (!g_num_sms) {
        int d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, d);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

static amsim_status cuda_check(cudaError_t e, const char *what)
{
    if (e == cudaSuccess) return AMSIM_OK;
    return set_error(AMSIM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <int TN, int EB, class OpA, class OpB>
static amsim_status launch_mm(KParams p, const OpA &a, const OpB &b, cudaStream_t st)
{
    size_t smem = smem_bytes<TN>(p.lut_bytes);
    auto kern = amsim_mm_kernel<TN, EB, OpA, OpB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute");
    int ntiles = p.tiles_m * p.tiles_n * p.splits;
    int grid = std::min(ntiles, num_sms());
    if (grid <= 0) return AMSIM_OK;
    kern<<<grid, NT, smem, st>>>(p, a, b);
    count_launch();
    return cuda_check(cudaGetLastError(), "amsim_mm_kernel launch");
}

template <int EB, class OpA, class OpB>
static amsim_status launch_tn(KParams p, const OpA &a, const OpB &b, cudaStream_t st)
{
    if (p.N <= 32) {
        p.tiles_n = (p.N + 31) / 32;
        return launch_mm<1, EB>(p, a, b, st);
    }
    if (p.N <= 64) {
        p.tiles_n = (p.N + 63) / 64;
        return launch_mm<2, EB>(p, a, b, st);
    }
    p.tiles_n = (p.N + 127) / 128;
    return launch_mm<4, EB>(p, a, b, st);
}

static int bn_for(int N) { return N <= 32 ? 32 : (N <= 64 ? 64 : 128); }

// Common problem setup: table, tiles, split-K.
static amsim_status prepare(const amsim_lut *lut, KParams &p, int M, int N, int K, int max_splits)
{
    const void *tab = nullptr;
    int eb = 32;
    amsim_status s = device_table(lut, &tab, &eb);
    if (s != AMSIM_OK) return s;
    int mbits = 0;
    amsim_lut_info(lut, &mbits, nullptr);
    uint32_t bytes = uint32_t((size_t(1) << (2 * mbits)) * (eb / 8));
    if (smem_bytes<4>(bytes) > 227 * 1024)
        return set_error(AMSIM_ERR_UNSUPPORTED, "table of m = " + std::to_string(mbits) +
                                                    " does not fit in shared memory (global-memory table: future work)");
    p.M = M;
    p.N = N;
    p.K = K;
    p.lut = tab;
    p.m_bits = mbits;
    p.lut_bytes = bytes;
    p.policy = path_policy();
    p.tiles_m = (M + BM - 1) / BM;
    int bn = bn_for(N);
    p.tiles_n = (N + bn - 1) / bn;
    p.splits = 1;
    p.kchunk = std::max(K, 1);
    if (max_splits > 1) {
        long tiles = long(p.tiles_m) * p.tiles_n;
        long want = (2L * num_sms() + tiles - 1) / tiles;
        long maxs = std::max(1L, long(K) / (BK * 16));
        long sp = std::min({want, maxs, long(max_splits)});
        if (sp > 1) {
            int kc = (K + int(sp) - 1) / int(sp);
            kc = (kc + BK - 1) / BK * BK;
            p.splits = (K + kc - 1) / kc;
            p.kchunk = kc;
        }
    }
    return AMSIM_OK;
}

static int entry_bits_of(const amsim_lut *lut)
{
    int eb = 32;
    amsim_lut_info(lut, nullptr, &eb);
    return eb;
}

template <class OpA, class OpB>
static amsim_status run(const amsim_lut *lut, KParams p, const OpA &a, const OpB &b, cudaStream_t st)
{
    if (entry_bits_of(lut) == 16) return launch_tn<16>(p, a, b, st);
    return launch_tn<32>(p, a, b, st);
}

static amsim_status finish_split(const KParams &p, float *C, int64_t ldc, int accumulate, cudaStream_t st)
{
    if (p.splits <= 1) return AMSIM_OK;
    int64_t total = int64_t(p.M) * p.N;
    int blocks = int(std::min<int64_t>((total + 255) / 256, 4L * num_sms()));
    splitk_reduce_kernel<<<std::max(blocks, 1), 256, 0, st>>>(p.C, p.splits, p.M, p.N, C, ldc, accumulate);
    count_launch();
    return cuda_check(cudaGetLastError(), "splitk_reduce launch");
}

static void init_geom(ConvGeom &g, const amsim_conv2d_desc *d)
{
    g.N = d->N; g.H = d->H; g.W = d->W; g.C = d->C; g.K = d->K; g.R = d->R; g.S = d->S;
    g.sh = d->stride_h; g.sw = d->stride_w; g.ph = d->pad_h; g.pw = d->pad_w;
    g.OH = (d->H + 2 * d->pad_h - d->R) / d->stride_h + 1;
    g.OW = (d->W + 2 * d->pad_w - d->S) / d->stride_w + 1;
    g.fOHOW.init(uint32_t(g.OH * g.OW));
    g.fOW.init(uint32_t(g.OW));
    g.fSC.init(uint32_t(g.S * g.C));
    g.fC.init(uint32_t(g.C));
    g.fHW.init(uint32_t(g.H * g.W));
    g.fW.init(uint32_t(g.W));
}

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static amsim_status check_desc(const amsim_conv2d_desc *d)
{
    if (!d) return set_error(AMSIM_ERR_INVALID_ARG, "null conv descriptor");
    if (d->N < 0 || d->H <= 0 || d->W <= 0 || d->C <= 0 || d->K <= 0 || d->R <= 0 || d->S <= 0 ||
        d->stride_h <= 0 || d->stride_w <= 0 || d->pad_h < 0 || d->pad_w < 0 || d->pad_h > d->R - 1 ||
        d->pad_w > d->S - 1 || d->H + 2 * d->pad_h < d->R || d->W + 2 * d->pad_w < d->S)
        return set_error(AMSIM_ERR_INVALID_ARG, "invalid conv descriptor (sizes > 0, stride >= 1, 0 <= pad <= kernel-1, "
                                                "kernel fits the padded input)");
    int64_t OH = (int64_t(d->H) + 2 * d->pad_h - d->R) / d->stride_h + 1;
    int64_t OW = (int64_t(d->W) + 2 * d->pad_w - d->S) / d->stride_w + 1;
    if (int64_t(d->N) * d->H * d->W * d->C >= (1LL << 31) || int64_t(d->N) * OH * OW * d->K >= (1LL << 31) ||
        int64_t(d->N) * OH * OW >= (1LL << 31) || int64_t(d->R) * d->S * d->C * d->K >= (1LL << 31))
        return set_error(AMSIM_ERR_INVALID_ARG, "conv tensor too large (each tensor < 2^31 elements)");
    return AMSIM_OK;
}

}  // namespace amsim

using namespace amsim;

extern "C" {

amsim_status amsim_gemm(const amsim_lut *lut, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K,
                        const float *A, int64_t lda, const float *B, int64_t ldb, float *C, int64_t ldc,
                        int accumulate, amsim_stream_t stream)
{
    clear_error();
    if (!lut) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: null lut");
    if (M < 0 || N < 0 || K < 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: negative size");
    if (M >= (1LL << 31) || N >= (1LL << 31) || K >= (1LL << 31))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: dimensions must be < 2^31");
    if (M == 0 || N == 0) return AMSIM_OK;
    if (!C || ldc < N) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: C null or ldc < N");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (K == 0) {
        const void *tab;
        int eb;
        amsim_status s = device_table(lut, &tab, &eb);  // device check
        if (s != AMSIM_OK) return s;
        if (accumulate) return AMSIM_OK;
        fill_zero_kernel<<<std::max(1, int(std::min<int64_t>((M * N + 255) / 256, 1024))), 256, 0, st>>>(C, int(M), int(N), ldc);
        count_launch();
        return cuda_check(cudaGetLastError(), "fill_zero launch");
    }
    if (!A || !B) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: null operand");
    if ((!trans_a && lda < K) || (trans_a && lda < M))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: lda too small");
    if ((!trans_b && ldb < N) || (trans_b && ldb < K))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: ldb too small");
    KParams p{};
    amsim_status s = prepare(lut, p, int(M), int(N), int(K), 1);
    if (s != AMSIM_OK) return s;
    GemmOp a{A, lda, int(M), int(K), trans_a ? 0 : 1};
    GemmOp b{B, ldb, int(N), int(K), trans_b ? 1 : 0};
    // 16-byte copies need 4 contiguous elements with 16-B aligned rows
    bool va = aligned16(A) && lda % 4 == 0 && (trans_a ? M % 4 == 0 : K % 4 == 0);
    bool vb = aligned16(B) && ldb % 4 == 0 && (trans_b ? K % 4 == 0 : N % 4 == 0);
    p.da = OpDesc{a.kcontig, va ? 4 : 1};
    p.db = OpDesc{b.kcontig, vb ? 4 : 1};
    p.C = C;
    p.ldc = ldc;
    p.accumulate = accumulate;
    return run(lut, p, a, b, st);
}

amsim_status amsim_conv2d_fwd(const amsim_lut *lut, const amsim_conv2d_desc *d, const float *x, const float *w,
                              float *y, amsim_stream_t stream)
{
    clear_error();
    if (!lut) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_fwd: null lut");
    amsim_status s = check_desc(d);
    if (s != AMSIM_OK) return s;
    if (d->N == 0) return AMSIM_OK;
    if (!x || !w || !y) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_fwd: null tensor");
    ConvGeom g;
    init_geom(g, d);
    int M = d->N * g.OH * g.OW, N = d->K, K = d->R * d->S * d->C;
    KParams p{};
    s = prepare(lut, p, M, N, K, 1);
    if (s != AMSIM_OK) return s;
    FwdX a{x, g, M, K};
    GemmOp b{w, N, N, K, 0};
    p.da = OpDesc{1, (d->C % 4 == 0 && aligned16(x)) ? 4 : 1};
    p.db = OpDesc{0, (N % 4 == 0 && aligned16(w)) ? 4 : 1};
    p.C = y;
    p.ldc = N;
    p.accumulate = 0;
    return run(lut, p, a, b, reinterpret_cast<cudaStream_t>(stream));
}

amsim_status amsim_conv2d_bwd_data(const amsim_lut *lut, const amsim_conv2d_desc *d, const float *dy,
                                   const float *w, float *dx, amsim_stream_t stream)
{
    clear_error();
    if (!lut) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_data: null lut");
    amsim_status s = check_desc(d);
    if (s != AMSIM_OK) return s;
    if (d->N == 0) return AMSIM_OK;
    if (!dy || !w || !dx) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_data: null tensor");
    ConvGeom g;
    init_geom(g, d);
    // k = (kh', kw', co): reuse fSC / fC as divisors S*K and K
    g.fSC.init(uint32_t(d->S * d->K));
    g.fC.init(uint32_t(d->K));
    int M = d->N * d->H * d->W, N = d->C, K = d->R * d->S * d->K;
    KParams p{};
    s = prepare(lut, p, M, N, K, 1);
    if (s != AMSIM_OK) return s;
    DgDY a{dy, g, M, K};
    DgW b{w, g, N, K};
    bool v = d->K % 4 == 0;
    p.da = OpDesc{1, (v && aligned16(dy)) ? 4 : 1};
    p.db = OpDesc{1, (v && aligned16(w)) ? 4 : 1};
    p.C = dx;
    p.ldc = N;
    p.accumulate = 0;
    return run(lut, p, a, b, reinterpret_cast<cudaStream_t>(stream));
}

static amsim_status wgrad_params(const amsim_lut *lut, const amsim_conv2d_desc *d, KParams &p, ConvGeom &g)
{
    init_geom(g, d);
    int M = d->R * d->S * d->C, N = d->K, K = d->N * g.OH * g.OW;
    return prepare(lut, p, M, N, K, 1024);
}

amsim_status amsim_conv2d_bwd_filter_workspace(const amsim_lut *lut, const amsim_conv2d_desc *d, size_t *bytes)
{
    clear_error();
    if (!lut || !bytes) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_filter_workspace: null argument");
    amsim_status s = check_desc(d);
    if (s != AMSIM_OK) return s;
    KParams p{};
    ConvGeom g;
    s = wgrad_params(lut, d, p, g);
    if (s != AMSIM_OK) return s;
    *bytes = p.splits > 1 ? size_t(p.splits) * p.M * p.N * sizeof(float) : 0;
    return AMSIM_OK;
}

amsim_status amsim_conv2d_bwd_filter(const amsim_lut *lut, const amsim_conv2d_desc *d, const float *x,
                                     const float *dy, float *dw, void *workspace, size_t workspace_bytes,
                                     amsim_stream_t stream)
{
    clear_error();
    if (!lut) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_filter: null lut");
    amsim_status s = check_desc(d);
    if (s != AMSIM_OK) return s;
    if (!x || !dy || !dw) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_filter: null tensor");
    KParams p{};
    ConvGeom g;
    s = wgrad_params(lut, d, p, g);
    if (s != AMSIM_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (p.K == 0) {
        fill_zero_kernel<<<64, 256, 0, st>>>(dw, p.M, p.N, p.N);
        count_launch();
        return cuda_check(cudaGetLastError(), "fill_zero launch");
    }
    size_t need = p.splits > 1 ? size_t(p.splits) * p.M * p.N * sizeof(float) : 0;
    if (need > 0 && (!workspace || workspace_bytes < need))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_filter: workspace too small (need " +
                                                    std::to_string(need) + " bytes)");
    WgX a{x, g, p.M, p.K};
    GemmOp b{dy, d->K, p.N, p.K, 0};
    p.da = OpDesc{0, (d->C % 4 == 0 && aligned16(x)) ? 4 : 1};
    p.db = OpDesc{0, (d->K % 4 == 0 && aligned16(dy)) ? 4 : 1};
    p.C = p.splits > 1 ? static_cast<float *>(workspace) : dw;
    p.ldc = p.splits > 1 ? p.N : p.N;
    p.accumulate = 0;
    s = run(lut, p, a, b, st);
    if (s != AMSIM_OK) return s;
    return finish_split(p, dw, p.N, 0, st);
}

amsim_status amsim_bench_lut_lookup(int m_bits, int entry_bits, int iters, const uint32_t *b_idx_host, size_t n_idx,
                                    double *lookups_per_s, amsim_stream_t stream)
{
    clear_error();
    if (m_bits < 1 || m_bits > 8 || (entry_bits != 16 && entry_bits != 32) || iters <= 0 || !b_idx_host || !n_idx ||
        !lookups_per_s)
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_bench_lut_lookup: bad argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint32_t bytes = uint32_t((size_t(1) << (2 * m_bits)) * (entry_bits / 8));
    if (bytes > 200 * 1024) return set_error(AMSIM_ERR_UNSUPPORTED, "table too large for shared memory");
    void *tab = nullptr;
    uint32_t *idx = nullptr;
    float *out = nullptr;
    int sms = num_sms();
    amsim_status s = AMSIM_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    do {
        if ((s = cuda_check(cudaMalloc(&tab, bytes), "cudaMalloc")) != AMSIM_OK) break;
        if ((s = cuda_check(cudaMemsetAsync(tab, 0, bytes, st), "memset")) != AMSIM_OK) break;
        if ((s = cuda_check(cudaMalloc(&idx, n_idx * 4), "cudaMalloc")) != AMSIM_OK) break;
        if ((s = cuda_check(cudaMemcpyAsync(idx, b_idx_host, n_idx * 4, cudaMemcpyHostToDevice, st), "memcpy")) != AMSIM_OK) break;
        if ((s = cuda_check(cudaMalloc(&out, size_t(sms) * NT * 4), "cudaMalloc")) != AMSIM_OK) break;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto launch = [&]() {
            if (entry_bits == 16) {
                cudaFuncSetAttribute(lut_bench_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
                lut_bench_kernel<16><<<sms, NT, bytes, st>>>(tab, bytes, m_bits, idx, int(n_idx), iters, out);
            } else {
                cudaFuncSetAttribute(lut_bench_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
                lut_bench_kernel<32><<<sms, NT, bytes, st>>>(tab, bytes, m_bits, idx, int(n_idx), iters, out);
            }
            count_launch();
        };
        launch();  // warm-up
        cudaEventRecord(e0, st);
        launch();
        cudaEventRecord(e1, st);
        if ((s = cuda_check(cudaEventSynchronize(e1), "bench sync")) != AMSIM_OK) break;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        double lookups = double(sms) * NT * iters * TM * 4;
        *lookups_per_s = lookups / (ms * 1e-3);
    } while (0);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(tab);
    cudaFree(idx);
    cudaFree(out);
    return s;
}

}  // extern "C"
