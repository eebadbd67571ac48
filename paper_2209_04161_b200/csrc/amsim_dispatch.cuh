// libamsim dispatch shared by the per-entry-point translation units
// (amsim_gemm.cu, amsim_conv_*.cu, amsim_bench.cu): tile configurations,
// the tile planner and the launch helpers.  Internal; not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "amsim_device.cuh"
#include "amsim_internal.h"

#ifndef AMSIM_NT_BIG
#define AMSIM_NT_BIG 256
#endif
#ifndef AMSIM_TM_BIG
#define AMSIM_TM_BIG 16
#endif
#ifndef AMSIM_NT_MID
#define AMSIM_NT_MID 256
#endif
#ifndef AMSIM_TM_MID
#define AMSIM_TM_MID 16
#endif

namespace amsim {
namespace dev {

static __global__ void fill_zero_kernel(float *C, int M, int N, int64_t ldc)
{
    int64_t total = int64_t(M) * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x)
        C[(e / N) * ldc + e % N] = 0.0f;
}

// LUT-lookup microbenchmark (roofline instrument): the fast path's lookup
// pattern -- table row shared by the warp, per-lane column offsets drawn from
// `bidx`, 8 rows x 4 columns per thread -- with no operand traffic.
constexpr int BENCH_NT = 256, BENCH_TM = 8;
template <int EB>
__global__ void __launch_bounds__(BENCH_NT, 1) lut_bench_kernel(const void *lut, uint32_t lut_bytes, int m,
                                                                const uint32_t *bidx, int nidx, int iters, float *out)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const uint4 *src = reinterpret_cast<const uint4 *>(lut);
    for (uint32_t i = threadIdx.x; i < lut_bytes / 16; i += BENCH_NT) reinterpret_cast<uint4 *>(smem)[i] = src[i];
    __syncthreads();
    constexpr int ebl = EB == 8 ? 0 : (EB == 16 ? 1 : 2);
    const uint32_t base = smem_u32(smem);
    const int warp = threadIdx.x >> 5;
    const uint32_t rmask = (1u << m) - 1u;
    uint32_t bof[4], row[BENCH_TM];
    for (int c = 0; c < 4; c++) bof[c] = base + (bidx[(blockIdx.x * BENCH_NT + threadIdx.x * 4 + c) % nidx] << ebl);
    for (int r = 0; r < BENCH_TM; r++) row[r] = ((warp * 37 + r * 11 + blockIdx.x) * 13) & rmask;
    float acc[BENCH_TM][4] = {};
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int r = 0; r < BENCH_TM; r++) {
            const uint32_t aof = ((row[r] + uint32_t(it)) & rmask) << (m + ebl);  // warp-uniform row walk
#pragma unroll
            for (int c = 0; c < 4; c++) {
                uint32_t e = lut_entry<EB>(aof + bof[c], nullptr);
                acc[r][c] = fma_ftz(__uint_as_float(e * (EB == 8 ? 65536u : 256u) + 0x3F800000u), 1.0f, acc[r][c]);
            }
        }
    }
    float s = 0.f;
    for (int r = 0; r < BENCH_TM; r++)
        for (int c = 0; c < 4; c++) s += acc[r][c];
    out[blockIdx.x * BENCH_NT + threadIdx.x] = s;
}

}  // namespace dev

// ===========================================================================
// Host dispatch

using namespace dev;

using CfgSmall = KCfg<256, 8, 1>;                        // N <= 32
using CfgMid = KCfg<AMSIM_NT_MID, AMSIM_TM_MID, 2>;      // N <= 64, M > 64
#ifndef AMSIM_TN_BIG
#define AMSIM_TN_BIG 4
#endif
using CfgBig = KCfg<AMSIM_NT_BIG, AMSIM_TM_BIG, AMSIM_TN_BIG>;  // N > 64, M > 64
using CfgLean = KCfg<256, 8, 2>;                         // N <= 64, M <= 64; and tables too large for the others
using CfgWide = KCfg<256, 8, 4>;                         // N > 64, M <= 64
#ifndef AMSIM_SK_ALIGN_PCT
#define AMSIM_SK_ALIGN_PCT 0   // stream-K CTA count aligned to the tile count when it costs <= this % of the SMs
#endif
#ifndef AMSIM_HUGE8
#define AMSIM_HUGE8 1   // offer the 16 x 8 tile to 8-bit tables too
#endif
using CfgHuge = KCfg<256, 16, 8>;                        // N >= 256, 16/32-bit tables (fewer operand loads per lookup)
using CfgFlat = KCfg<256, 16, 4, 2>;                     // 64 x 256: 64-row problems (64-channel layers, transposed)
                                                         // with Big's 16 x 4 register tile instead of Wide's 8 x 4
using CfgTall = KCfg<256, 20, 2>;
using CfgTallT = KCfg<256, 8, 5>;                        // 64 x 160, transposed only: 129..160 lanes (stem wgrad, 147)
using CfgFlat3 = KCfg<256, 16, 3, 2>;                    // 64 x 192, transposed only: lanes = 576 = 3 x 192 (3x3 x 64-channel wgrad)
using CfgFlat8 = KCfg<256, 16, 8, 2, true>;              // 64 x 512, transposed only: Huge's 16 x 8 register tile for
                                                         // the 64-channel layers; narrow shared-memory layout (NP), so
                                                         // both operands must be k-contiguous TMA boxes

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

// A problem before tiling: sub-problems (M_s, K_s) sharing N.
struct Problem {
    int N = 0;
    int nsub = 1;
    int M[MAX_SUB] = {0};
    int K[MAX_SUB] = {0};
    // the original A operand (the lanes in the transposed orientation) is loaded
    // as k-contiguous TMA boxes and B as TMA boxes: the narrow Flat8 tile may be used
    bool tma_lanes = false;
    // the A operand is a layer input (ReLU activations in a network): in the
    // transposed orientation it is read by the lanes, where its zeros share one
    // table word and cut bank conflicts (measured +7 % on ResNet-50 l2.1.conv1
    // fwd at equal tile shape), so the planner favours that orientation by 5 %
    bool a_is_activation = false;
};

enum class CfgId { Small, Mid, Big, Lean, Wide, Huge, Flat, Tall, Flat3, TallT, Flat8 };
static constexpr size_t kSmemMax = 227 * 1024;

static void cfg_shape(CfgId c, int &BM, int &BN, int &NT, size_t &smem, uint32_t lut_bytes)
{
    switch (c) {
    case CfgId::Small: BM = CfgSmall::BM; BN = CfgSmall::BN; NT = CfgSmall::NT; smem = CfgSmall::smem_bytes(lut_bytes); break;
    case CfgId::Mid: BM = CfgMid::BM; BN = CfgMid::BN; NT = CfgMid::NT; smem = CfgMid::smem_bytes(lut_bytes); break;
    case CfgId::Lean: BM = CfgLean::BM; BN = CfgLean::BN; NT = CfgLean::NT; smem = CfgLean::smem_bytes(lut_bytes); break;
    case CfgId::Wide: BM = CfgWide::BM; BN = CfgWide::BN; NT = CfgWide::NT; smem = CfgWide::smem_bytes(lut_bytes); break;
    case CfgId::Huge: BM = CfgHuge::BM; BN = CfgHuge::BN; NT = CfgHuge::NT; smem = CfgHuge::smem_bytes(lut_bytes); break;
    case CfgId::Flat: BM = CfgFlat::BM; BN = CfgFlat::BN; NT = CfgFlat::NT; smem = CfgFlat::smem_bytes(lut_bytes); break;
    case CfgId::Tall: BM = CfgTall::BM; BN = CfgTall::BN; NT = CfgTall::NT; smem = CfgTall::smem_bytes(lut_bytes); break;
    case CfgId::TallT: BM = CfgTallT::BM; BN = CfgTallT::BN; NT = CfgTallT::NT; smem = CfgTallT::smem_bytes(lut_bytes); break;
    case CfgId::Flat3: BM = CfgFlat3::BM; BN = CfgFlat3::BN; NT = CfgFlat3::NT; smem = CfgFlat3::smem_bytes(lut_bytes); break;
    case CfgId::Flat8: BM = CfgFlat8::BM; BN = CfgFlat8::BN; NT = CfgFlat8::NT; smem = CfgFlat8::smem_bytes(lut_bytes); break;
    default: BM = CfgBig::BM; BN = CfgBig::BN; NT = CfgBig::NT; smem = CfgBig::smem_bytes(lut_bytes); break;
    }
}

// Tile plan with a small cost model (cost unit: one k-tile of one BM x BN
// tile on one SM).  Two schedules (see SubP):
//  * data-parallel: CTAs take whole tiles round-robin (t = blockIdx.x + i*grid);
//    a CTA's time is the sum of its tiles' k-tiles plus a per-tile overhead;
//    every output is the FP32 sum from +0 in increasing k (policy bit 1 forces it);
//  * stream-K: every SM gets the same number of k-tiles (W / G), whatever the
//    tile count -- no wave quantisation -- at the price of <= 2 partial tiles per
//    CTA written, re-read and added in a fixed order by the last piece.
// The cheaper one is taken.  Deterministic for a given problem and device.
static double tile_plan(KParams &p, const Problem &pr, int BM, int BN, int policy, int NT)
{
    const int G = num_sms();
    p.N = pr.N;
    p.tiles_n = (pr.N + BN - 1) / BN;
    p.nsub = pr.nsub;
    const double tile_overhead = 2.0;
    const double ktile_s = double(BM) * BN * BK / (20.0 * 1.9e9);     // ~20 approx-MAC/clk/SM
    const double hbm_per_unit = 5.0e12 * ktile_s;                     // HBM bytes per cost unit (whole chip)
    const double l2_per_unit_sm = 150.0e9 * ktile_s;                  // L2 bytes one SM reads per cost unit
    int begin = 0;
    int64_t W = 0;
    for (int s = 0; s < pr.nsub; s++) {
        SubP &S = p.sub[s];
        S.M = pr.M[s];
        S.K = pr.K[s];
        S.tiles_m = (S.M + BM - 1) / BM;
        S.kt = S.K > 0 ? (S.K + BK - 1) / BK : 0;
        S.tile_begin = begin;
        begin += S.tiles_m * p.tiles_n;
        W += int64_t(S.tiles_m) * p.tiles_n * std::max(S.kt, 1);
    }
    p.ntiles = begin;
    // data-parallel makespan: round-robin simulation
    std::vector<double> load(G, 0.0);
    for (int s = 0, t = 0; s < pr.nsub; s++) {
        const double cost = tile_overhead + p.sub[s].kt;
        const long n = long(p.sub[s].tiles_m) * p.tiles_n;
        const long full = n / G, rem = n % G;
        if (full)
            for (int g = 0; g < G; g++) load[g] += cost * full;
        for (long r = 0; r < rem; r++) load[(t + full * G + r) % G] += cost;
        t = int((t + n) % G);
    }
    const double dp = *std::max_element(load.begin(), load.end());
    // stream-K makespan: W / Gsk k-tiles, the per-unit overhead of the tiles a
    // range touches, partial tiles through HBM, and the fix-up tree's critical
    // path (one partial tile written and one read per level, ceil(log2 pieces) levels)
    // small problems may use fewer CTAs than SMs (each at least `chunk` k-tiles):
    // the count that minimises the modelled time
    const double tile_bytes = 4.0 * BM * BN;
    auto sk_cost = [&](int g) {
        const double per_cta = double(W) / g;
        const double units = double(p.ntiles) / g + 1.0;
        double pieces_max = 1.0;
        for (int s = 0; s < pr.nsub; s++)
            pieces_max = std::max(pieces_max, std::ceil(std::max(p.sub[s].kt, 1) / per_cta) + 1.0);
        return std::ceil(per_cta) + tile_overhead * units + 2.0 * 2.0 * g * tile_bytes / hbm_per_unit +
               2.0 * std::ceil(std::log2(pieces_max)) * tile_bytes / l2_per_unit_sm;
    };
    int Gsk = 1;
    double sk = 1e300;
    for (int chunk : {1, 2, 4, 8}) {
        const int g = int(std::max<int64_t>(1, std::min<int64_t>(G, W / chunk)));
        const double c = sk_cost(g);
        if (c < sk * 0.99) {
            sk = c;
            Gsk = g;
        }
    }
    // Few tiles, each split over several CTAs (wgrad: a handful of weight tiles,
    // K = N * OH * OW): with G not a multiple of the tile count, the CTAs of
    // different tiles start at different k offsets, so tiles that share an
    // operand slice (the error / activation rows of the same pixels) read it
    // hundreds of k-tiles apart and L2 cannot serve the second read.  A CTA
    // count that is a multiple of the tile count aligns every tile's pieces in
    // k, at the cost of up to AMSIM_SK_ALIGN_PCT % of the SMs.
    if (p.nsub == 1 && p.ntiles > 1 && p.ntiles * 2 <= Gsk && Gsk % p.ntiles != 0) {
        const int Ga = (Gsk / p.ntiles) * p.ntiles;
        if ((Gsk - Ga) * 100 <= Gsk * AMSIM_SK_ALIGN_PCT) {
            sk = sk * Gsk / Ga;
            Gsk = Ga;
        }
    }
    bool use_sk = sk < dp * 0.98;
    // AMSIM_SCHED=dp|sk forces a schedule (tests and tuning only; policy bit 1 still wins)
    if (const char *f = std::getenv("AMSIM_SCHED"); f && *f) use_sk = f[0] == 's';
    use_sk = use_sk && !(policy & 2) && W < (int64_t(1) << 30);
    p.n_dp = use_sk ? 0 : p.ntiles;
    p.sk_G = use_sk ? Gsk : 0;
    p.sk_W = use_sk ? int(W) : 0;
    for (int s = 0, pos = 0; s < pr.nsub; s++) {
        SubP &S = p.sub[s];
        const int tend = S.tile_begin + S.tiles_m * p.tiles_n;
        S.sk_tile = std::min(tend, std::max(S.tile_begin, p.n_dp));
        S.sk_pos = pos;
        pos += (tend - S.sk_tile) * std::max(S.kt, 1);
    }
    p.grid = std::max(p.n_dp > 0 ? std::min(p.n_dp, G) : 0, p.sk_G);
    // workspace: 2 partial tiles per stream-K CTA, then the fix-up tree's counters
    p.ws = nullptr;
    p.ws_elems = use_sk ? int64_t(2) * Gsk * BM * BN + int64_t(SK_LEVELS) * 2 * Gsk : 0;
    (void)NT;
    return use_sk ? sk : dp;
}

// Shared-memory wavefronts per warp-wide lookup, including the operand loads
// of the inner loop: the table row (2^m entries) read by
// 32 lanes at random columns costs ~row_bytes / 128 wavefronts (>= 1); the A
// side adds 1/TN (broadcast LDS.128, 2 wavefronts per 4 values, two arrays),
// the B side 2/TM.  Relative only -- it ranks the tile configurations.
static double wf_per_lookup(CfgId c, int eb, int mbits, bool table_in_smem)
{
    int TM = 16, TN = 4;
    switch (c) {
    case CfgId::Small: TM = 8; TN = 1; break;
    case CfgId::Mid: TM = 16; TN = 2; break;
    case CfgId::Lean: TM = 8; TN = 2; break;
    case CfgId::Wide: TM = 8; TN = 4; break;
    case CfgId::Huge: TM = 16; TN = 8; break;
    case CfgId::Flat: TM = 16; TN = 4; break;
    case CfgId::Tall: TM = 20; TN = 2; break;
    case CfgId::Flat3: TM = 16; TN = 3; break;
    case CfgId::Flat8: TM = 16; TN = 8; break;
    case CfgId::TallT: TM = 8; TN = 5; break;
    default: break;
    }
    double row = double(size_t(1) << mbits) * (eb / 8);
    double lk = table_in_smem ? std::max(1.0, row / 128.0 * 1.025) : 1.0;
    return lk + 1.0 / TN + 2.0 / TM;
}

// Measured cost per padded approx-MAC (ns per G) of each tile configuration
// with a 16-bit shared-memory table (MBM m = 7) under the stream-K schedule,
// median over the ResNet-50 b256 passes of `tools/cfg_sweep.py`
// (profiles/r02b_cfg_sweep_b256_final.jsonl, refit in round 2): dense operands (dgrad) and layer-input
// A operands (fwd / wgrad: zero-row skipping in the normal orientation, sparse
// lanes in the transposed one).  The wavefront model below under-prices the
// instruction overhead of the smaller register tiles (Big 16x4 measures 1.13x
// Huge 16x8 per MAC where the wavefronts predict 1.05x).  < 0: not measured.
static double measured_cost16(CfgId c, bool trn, bool act)
{
    // refitted after the quad decode, the zero-row branch skipping (16 x 8) and the
    // OR table addresses (profiles/r02b_cfg_sweep_b256_final.jsonl, tools/fit_costs.py)
    if (trn) {
        switch (c) {
        case CfgId::Huge: return act ? 0.2352 : 0.2571;
        case CfgId::Big: return act ? 0.2602 : 0.2770;
        case CfgId::Flat: return act ? 0.2652 : 0.2825;
        case CfgId::Flat3: return act ? 0.2758 : 0.2939;
        case CfgId::Flat8: return act ? 0.2445 : 0.2626;
        case CfgId::TallT: return act ? 0.2377 : 0.2375;
        case CfgId::Wide: return act ? 0.2828 : 0.3045;
        default: return -1.0;
        }
    }
    switch (c) {
    case CfgId::Huge: return act ? 0.1814 : 0.2551;
    case CfgId::Big: return act ? 0.2427 : 0.2816;
    case CfgId::Flat: return act ? 0.2437 : 0.2809;
    case CfgId::Mid: return act ? 0.3079 : 0.3174;
    case CfgId::Lean: return act ? 0.3641 : 0.3736;
    case CfgId::Small: return act ? 0.4882 : 0.5227;
    // offered only for <= 64 (Wide) / 129..160 rows (Tall), absent from the sweep's
    // shapes: the round-2 guesses scaled by the sweeps' mean change (x 0.91)
    case CfgId::Tall: return act ? 0.3100 : 0.3280;
    case CfgId::Wide: return act ? 0.2730 : 0.3000;
    default: return -1.0;
    }
}

static int cfg_tn(CfgId c)
{
    switch (c) {
    case CfgId::Small: return 1;
    case CfgId::Mid: case CfgId::Lean: case CfgId::Tall: return 2;
    case CfgId::Flat3: return 3;
    case CfgId::TallT: return 5;
    case CfgId::Huge: case CfgId::Flat8: return 8;
    default: return 4;
    }
}

static bool tma_disabled() { return (path_policy() & 8) != 0; }   // policy bit 3: cp.async for every operand

// Plan cache: the same problem (shape, table width, mode, policy) is planned
// once per process.
struct PlanRec {
    int cfg, tiles_n, nsub, ntiles, trn, n_dp, sk_G, sk_W, grid;
    int64_t ws_elems;
    SubP sub[MAX_SUB];
};
static std::mutex g_plan_mu;
static std::map<std::vector<int64_t>, PlanRec> g_plans;
static constexpr size_t kPlanCacheMax = 4096;

// Table, tile configuration and split plan for a problem.
// mode / policy < 0: the process-wide multiply mode / path policy.
static amsim_status prepare(const amsim_lut *lut, KParams &p, const Problem &pr, int &eb, int mode = -1,
                            int policy = -1)
{
    if (mode < 0) mode = multiply_mode();
    if (policy < 0) policy = path_policy();
    const void *tab = nullptr;
    amsim_status s = device_table(lut, &tab, &eb, policy);
    if (s != AMSIM_OK) return s;
    int mbits = 0;
    amsim_lut_info(lut, &mbits, nullptr);
    uint32_t bytes = uint32_t((size_t(1) << (2 * mbits)) * (eb / 8));
    // Tables too large for shared memory (m >= 8 with 32-bit entries, m >= 9)
    // are read from global memory, where they stay L2-resident (<= 16 MB).
    p.lut_global = CfgLean::smem_bytes(bytes) > kSmemMax ? 1 : 0;
    p.mul = MUL_LUT;
    if (mode == AMSIM_MUL_NATIVE) {
        p.mul = MUL_NATIVE;
    } else if (mode == AMSIM_MUL_DIRECT) {
        if (lut->model_id < 0)
            return set_error(AMSIM_ERR_UNSUPPORTED, "AMSIM_MUL_DIRECT needs a table built from a built-in model");
        p.mul = MUL_DIRECT_EXACT + lut->model_id;
    }
    if (p.mul != MUL_LUT) p.lut_global = 0;
    {   // exponent casting (reading C23): kept normal exponent fields [128 - B, 127 + B], B = 2^(e-1) - 1
        const int B = (1 << (lut->e_bits - 1)) - 1;
        p.ecast_lo = lut->e_bits >= 8 ? 1 : 128 - B;
        p.ecast_hi = lut->e_bits >= 8 ? 254 : 127 + B;
    }
    p.lut = tab;
    p.m_bits = mbits;
    p.lut_bytes = bytes;
    p.policy = policy & 1;
    const bool smem_table = !p.lut_global && p.mul == MUL_LUT;
    const uint32_t smem_lut = smem_table ? bytes : 0u;
    int force = -1;   // AMSIM_FORCE_CFG: tuning experiments only (>= 10: transposed orientation, cfg - 10)
    if (const char *f = std::getenv("AMSIM_FORCE_CFG"); f && *f) force = std::atoi(f);
    int sched = 0;     // AMSIM_SCHED (tile_plan): part of the cache key
    if (const char *f = std::getenv("AMSIM_SCHED"); f && *f) sched = f[0];
    // lut->symmetric decides whether the transposed orientation (which reads
    // LUT^T) may be planned, so it is part of the key
    std::vector<int64_t> key = {pr.N, pr.nsub, pr.a_is_activation, eb, p.lut_global, p.mul, policy & (3 | 8 | 16 | 32),
                                mbits, num_sms(), force, lut->symmetric ? 1 : 0, sched, pr.tma_lanes ? 1 : 0};
    for (int i = 0; i < pr.nsub; i++) {
        key.push_back(pr.M[i]);
        key.push_back(pr.K[i]);
    }
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        auto it = g_plans.find(key);
        if (it != g_plans.end()) {
            const PlanRec &r = it->second;
            p.cfg = r.cfg; p.trn = r.trn; p.N = r.trn ? pr.M[0] : pr.N; p.tiles_n = r.tiles_n; p.nsub = r.nsub;
            p.ntiles = r.ntiles; p.n_dp = r.n_dp; p.sk_G = r.sk_G; p.sk_W = r.sk_W; p.grid = r.grid;
            p.ws_elems = r.ws_elems; p.ws = nullptr;
            std::memcpy(p.sub, r.sub, sizeof(r.sub));
            return AMSIM_OK;
        }
    }
    // Candidate tile configurations (the non-table modes and global tables use Big / Lean
    // only); cost = planned makespan in k-tiles x lookups per k-tile x wavefronts per lookup.
    std::vector<CfgId> cands;
    if (smem_table) {
        cands = {CfgId::Small, CfgId::Mid, CfgId::Big, CfgId::Lean, CfgId::Flat};
        // Wide (8 x 4) only for <= 64-row problems, its purpose: on larger ones the
        // wavefront model under-prices its instruction overhead (7.3 instructions
        // per approx-MAC vs 5.1 for 16 x 8, ncu) and it measured 5-18 % slower
        // than Big / Huge on every ResNet-18 pass where it was picked
        int mmax = 0;
        for (int i = 0; i < pr.nsub; i++) mmax = std::max(mmax, pr.M[i]);
        if (mmax <= 64) cands.push_back(CfgId::Wide);
        if (eb >= 16 || AMSIM_HUGE8) cands.push_back(CfgId::Huge);
        // one 160-row tile for 129..160 rows (Mid / Lean would pad 147 rows to 256 / 192)
        if (pr.nsub == 1 && pr.M[0] > 128 && pr.M[0] <= CfgTall::BM) cands.push_back(CfgId::Tall);
    } else {
        cands = {CfgId::Big, CfgId::Lean};
    }
    if (force >= 0) {
        for (CfgId c : cands)
            if (int(c) == force) {
                cands = {c};
                break;
            }
    }
    const bool trn_ok = smem_table && lut->symmetric && pr.nsub == 1 && eb <= 16 &&
                        int64_t(pr.M[0]) * 4 >= pr.N && !(policy & 16) && !(force >= 0 && force < 10);
    if (force >= 10 && trn_ok) cands.clear();
    double best = 1e300;
    KParams bestp = p;
    // 16-bit shared-memory tables at m = 7 (MBM / exact): measured per-configuration
    // costs; otherwise the wavefront model, scaled to the same units (Huge: 2.30
    // wavefronts per lookup <-> 0.2732)
    const bool measured16 = smem_table && eb == 16 && mbits == 7 && p.mul == MUL_LUT;
    const double wf_to_cost16 = 0.2732 / 2.30;
    for (CfgId c : cands) {
        int BM, BN, NT;
        size_t smem;
        cfg_shape(c, BM, BN, NT, smem, smem_lut);
        if (smem > kSmemMax) continue;
        KParams q = p;
        q.cfg = int(c);
        q.trn = 0;
        const double m16 = measured16 ? measured_cost16(c, false, pr.a_is_activation) : -1.0;
        double cost = tile_plan(q, pr, BM, BN, policy, NT) * double(BM) * BN *
                      (m16 > 0 ? m16 : wf_per_lookup(c, eb, mbits, smem_table) * wf_to_cost16);
        // zero-row skipping (SKIP in amsim_mm_kernel): in this orientation a layer
        // input's zeros (ReLU) are warp-shared rows whose lookups are predicated
        // off.  The saving grows with the columns per lane (the predicate and the
        // operand loads are per row): measured on ResNet-50 (MBM, m = 7) at
        // 0.87-0.89 of Huge^T for Huge (16 x 8), 0.96-1.04 for Big (16 x 4),
        // none for 2-column tiles -- factors calibrated on those ratios
        // (the measured 16-bit costs include it).
        if (m16 < 0 && pr.a_is_activation && AMSIM_SKIP && smem_table && eb >= 16 && p.mul == MUL_LUT)
            cost *= cfg_tn(c) >= 8 ? 0.84 : cfg_tn(c) >= 4 ? 0.92 : 1.0;
        if (cost < best * 0.999) {
            best = cost;
            bestp = q;
        }
    }
    // Transposed orientation (the output channels become the warp-shared rows,
    // the pixels the lanes): symmetric shared-memory tables, one sub-problem,
    // N well below M (policy bit 4 disables it).  It wins for skinny N (fewer
    // operand loads per lookup) and, at equal tile shape, whenever the A
    // operand is a layer input (sparse lanes, see Problem::a_is_activation).
    if (trn_ok) {
        Problem pt = pr;
        pt.N = pr.M[0];
        pt.M[0] = pr.N;
        std::vector<CfgId> tc = {CfgId::Wide, CfgId::Big, CfgId::Flat};
        // 192 lanes where they tile the lane dimension exactly and 256 would not
        // (3x3 x 64-channel wgrad: 576 = 3 x 192, vs 768 = 3 x 256 for Flat)
        if (pr.M[0] % CfgFlat3::BN == 0 && pr.M[0] % CfgFlat::BN != 0) tc.push_back(CfgId::Flat3);
        if (pr.M[0] > 128 && pr.M[0] <= CfgTallT::BN) tc.push_back(CfgId::TallT);
        if (eb >= 16) tc.push_back(CfgId::Huge);
        // 64 x 512 for <= 64 output channels when every operand tile is a TMA box
        if (eb == 16 && pr.tma_lanes && !tma_disabled() && pr.N <= 64) tc.push_back(CfgId::Flat8);
        if (force >= 10) tc = {CfgId(force - 10)};
        if (force >= 10 && CfgId(force - 10) == CfgId::Flat8 && !(eb == 16 && pr.tma_lanes && !tma_disabled()))
            tc = {CfgId::Flat};
        if (force >= 10 && CfgId(force - 10) == CfgId::Huge && eb < 16) tc = {CfgId::Big};
        for (CfgId c : tc) {
            int BM, BN, NT;
            size_t smem;
            cfg_shape(c, BM, BN, NT, smem, smem_lut);
            if (smem > kSmemMax) continue;
            KParams q = p;
            q.cfg = int(c);
            q.trn = 1;
            const double m16 = measured16 ? measured_cost16(c, true, pr.a_is_activation) : -1.0;
            double cost = tile_plan(q, pt, BM, BN, policy, NT) * double(BM) * BN *
                          (m16 > 0 ? m16 : wf_per_lookup(c, eb, mbits, smem_table) * wf_to_cost16 *
                                               (pr.a_is_activation ? 0.95 : 1.0));
            if (cost < best * 0.999) {
                best = cost;
                bestp = q;
            }
        }
    }
    if (best >= 1e299) return set_error(AMSIM_ERR_UNSUPPORTED, "no tile configuration fits shared memory");
    p = bestp;
    if (const char *dbg = std::getenv("AMSIM_DEBUG_PLAN"); dbg && *dbg && *dbg != '0')
        std::fprintf(stderr, "[amsim plan] N=%d M0=%d K0=%d nsub=%d eb=%d mul=%d -> cfg=%d trn=%d tiles=%d n_dp=%d "
                     "sk_G=%d sk_W=%d ws=%lld\n",
                     pr.N, pr.M[0], pr.K[0], pr.nsub, eb, p.mul, p.cfg, p.trn, p.ntiles, p.n_dp, p.sk_G, p.sk_W,
                     (long long)p.ws_elems);
    PlanRec r;
    r.cfg = p.cfg; r.trn = p.trn; r.tiles_n = p.tiles_n; r.nsub = p.nsub; r.ntiles = p.ntiles; r.ws_elems = p.ws_elems;
    r.n_dp = p.n_dp; r.sk_G = p.sk_G; r.sk_W = p.sk_W; r.grid = p.grid;
    std::memcpy(r.sub, p.sub, sizeof(r.sub));
    std::lock_guard<std::mutex> g(g_plan_mu);
    if (g_plans.size() >= kPlanCacheMax) g_plans.clear();   // bounded: a process planning many shapes re-plans
    g_plans.emplace(std::move(key), r);
    return AMSIM_OK;
}

template <class Cf, int EB, class OpA, class OpB, bool GL = false, int MUL = MUL_LUT, bool TRN = false>
static amsim_status launch_cfg(const KParams &p, const OpA &a, const OpB &b, cudaStream_t st)
{
    size_t smem = Cf::smem_bytes((GL || MUL != MUL_LUT) ? 0u : p.lut_bytes);
    auto kern = amsim_mm_kernel<Cf, EB, OpA, OpB, GL, MUL, TRN>;
    // opt in to the full shared-memory carve-out once per instantiation and device
    // (a launch may then use any size up to it); per-call attribute setting cost ~us
    static std::atomic<uint64_t> opted{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(opted.load(std::memory_order_relaxed) & (1ull << (dev & 63)))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemMax));
        if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute");
        opted.fetch_or(1ull << (dev & 63));
    }
    const int grid = p.grid;
    if (grid <= 0) return AMSIM_OK;
    kern<<<grid, Cf::NT, smem, st>>>(p, a, b);
    count_launch();
    return cuda_check(cudaGetLastError(), "amsim_mm_kernel launch");
}

template <int MUL, class OpA, class OpB>
static amsim_status launch_mode(const KParams &p, const OpA &a, const OpB &b, cudaStream_t st)
{
    return CfgId(p.cfg) == CfgId::Lean ? launch_cfg<CfgLean, 32, OpA, OpB, false, MUL>(p, a, b, st)
                                       : launch_cfg<CfgBig, 32, OpA, OpB, false, MUL>(p, a, b, st);
}

template <int EB, class OpA, class OpB>
static amsim_status launch_eb(const KParams &p, const OpA &a, const OpB &b, cudaStream_t st)
{
    switch (p.mul) {
    case MUL_NATIVE: return launch_mode<MUL_NATIVE>(p, a, b, st);
    case MUL_DIRECT_EXACT: return launch_mode<MUL_DIRECT_EXACT>(p, a, b, st);
    case MUL_DIRECT_MITCHELL: return launch_mode<MUL_DIRECT_MITCHELL>(p, a, b, st);
    case MUL_DIRECT_MBM: return launch_mode<MUL_DIRECT_MBM>(p, a, b, st);
    default: break;
    }
    if (p.lut_global) {
        if constexpr (EB == 8) return set_error(AMSIM_ERR_UNSUPPORTED, "8-bit tables always fit shared memory");
        else return CfgId(p.cfg) == CfgId::Lean ? launch_cfg<CfgLean, EB, OpA, OpB, true>(p, a, b, st)
                                                 : launch_cfg<CfgBig, EB, OpA, OpB, true>(p, a, b, st);
    }
    switch (CfgId(p.cfg)) {
    case CfgId::Small: return launch_cfg<CfgSmall, EB>(p, a, b, st);
    case CfgId::Mid: return launch_cfg<CfgMid, EB>(p, a, b, st);
    case CfgId::Lean: return launch_cfg<CfgLean, EB>(p, a, b, st);
    case CfgId::Wide: return launch_cfg<CfgWide, EB>(p, a, b, st);
    case CfgId::Flat: return launch_cfg<CfgFlat, EB>(p, a, b, st);
    case CfgId::Tall: return launch_cfg<CfgTall, EB>(p, a, b, st);
    case CfgId::Huge:
        if constexpr (EB >= 16 || AMSIM_HUGE8) return launch_cfg<CfgHuge, EB>(p, a, b, st);
        else return set_error(AMSIM_ERR_UNSUPPORTED, "internal: Huge tiles need 16/32-bit tables");
    default: return launch_cfg<CfgBig, EB>(p, a, b, st);
    }
}

// ---------------------------------------------------------------------------
// TMA descriptors for operand tiles that are plain boxes of a row-major matrix:
// a GemmOp read with k strided (smem tile [BK][rows], rows contiguous), i.e.
// the B operand of conv fwd (w) and wgrad (dy), GEMM B (no transpose) and GEMM
// A when transposed.  The box is rows x BK elements at (row0, k0); out-of-range
// elements are zero-filled by the TMA unit, like the cp.async path's zero fill.
static PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// Encode a tensor map over FP32 `base` with `rank` dims (innermost first),
// byte strides of dims 1.., box `box`; kcontig tiles use the 64-byte swizzle
// (the decode applies the same XOR).  Returns the TMA mode (2 / 3 = 2-D / 3-D)
// or 0 when the tensor cannot be described (alignment) -> cp.async.
static int encode_tma(CUtensorMap *map, const float *base, int rank, const cuuint64_t *dims,
                      const cuuint64_t *strides, const cuuint32_t *box, bool swizzle)
{
    auto fn = tma_encode_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(base) & 15)) return 0;
    for (int d = 0; d < rank; d++)
        if (dims[d] == 0 || (d > 0 && strides[d - 1] % 16)) return 0;
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cuuint32_t(rank), const_cast<float *>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? rank : 0;
}


static PFN_cuTensorMapEncodeIm2col_v12000 tma_im2col_fn()
{
    static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f);
    });
    return fn;
}

// im2col-mode descriptor over an NHWC tensor [n][h][w][c]: `rows` pixels per
// box (traversed w, h, n inside the bounding box [lower, dim - 1 + upper] with
// the given traversal strides), BK channels per pixel, 64-byte swizzle.
static int encode_im2col(CUtensorMap *map, const float *base, int N, int H, int W, int C, int lower_h, int lower_w,
                         int upper_h, int upper_w, int sh, int sw, int rows, int chans = BK)
{
    auto fn = tma_im2col_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || C % chans || N <= 0) return 0;
    cuuint64_t dims[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
    cuuint64_t st[3] = {cuuint64_t(C) * 4, cuuint64_t(W) * C * 4, cuuint64_t(H) * W * C * 4};
    int lo[2] = {lower_w, lower_h}, hi[2] = {upper_w, upper_h};
    cuuint32_t estr[4] = {1, cuuint32_t(sw), cuuint32_t(sh), 1};
    // k-contiguous tiles (BK channels per pixel) use the 64-byte swizzle; wgrad's
    // [BK pixels][BM channels] tiles are stored plainly
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(base), dims, st, lo, hi,
                    cuuint32_t(chans), cuuint32_t(rows), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    chans == BK ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 4 : 0;
}

// A row-major matrix (GemmOp): [k][mn] (mn contiguous) or [mn][k] (k contiguous, swizzled).
static int setup_tma(CUtensorMap *map, const GemmOp &op, int rows, OpDesc &d)
{
    if (tma_disabled() || op.MN <= 0 || op.K <= 0) return 0;
    cuuint64_t st[1] = {cuuint64_t(op.ld) * 4};
    if (!op.kcontig) {
        cuuint64_t dims[2] = {cuuint64_t(op.MN), cuuint64_t(op.K)};
        cuuint32_t box[2] = {cuuint32_t(rows), cuuint32_t(BK)};
        return encode_tma(map, op.p, 2, dims, st, box, false);
    }
    cuuint64_t dims[2] = {cuuint64_t(op.K), cuuint64_t(op.MN)};
    cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(rows)};
    int m = encode_tma(map, op.p, 2, dims, st, box, true);
    if (m) d.kcontig = 2;
    return m;
}

static bool is_1x1_s1(const ConvGeom &g) { return g.R == 1 && g.S == 1 && g.sh == 1 && g.sw == 1 && g.ph == 0 && g.pw == 0; }

// conv fwd A: for a 1x1 / stride-1 / unpadded conv, IM2COL(x) is x as [pixels][C];
// otherwise TMA's im2col mode (bounding box lower = -pad, upper = pad - (R-1),
// traversal stride = conv stride) when C % BK == 0
static int setup_tma(CUtensorMap *map, const FwdX &op, int rows, OpDesc &d)
{
    if (tma_disabled()) return 0;
    if (!is_1x1_s1(op.g)) {
        const ConvGeom &g = op.g;
        int m = encode_im2col(map, op.x, g.N, g.H, g.W, g.C, -g.ph, -g.pw, g.ph - (g.R - 1), g.pw - (g.S - 1), g.sh,
                              g.sw, rows);
        if (m) d.kcontig = 2;
        return m;
    }
    cuuint64_t dims[2] = {cuuint64_t(op.g.C), cuuint64_t(op.M)};
    cuuint64_t st[1] = {cuuint64_t(op.g.C) * 4};
    cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(rows)};
    int m = encode_tma(map, op.x, 2, dims, st, box, true);
    if (m) d.kcontig = 2;
    return m;
}

// conv wgrad A: for 1x1 / stride 1 / unpadded, element (ci, pixel) of x as [pixels][C];
// otherwise im2col mode with BK pixels x `rows` channels per box when C % rows == 0
static int setup_tma(CUtensorMap *map, const WgX &op, int rows, OpDesc &d)
{
    if (tma_disabled()) return 0;
    if (!is_1x1_s1(op.g)) {
        const ConvGeom &g = op.g;
        if (rows > 256) return 0;
        if (g.C % rows == 0)
            return encode_im2col(map, op.x, g.N, g.H, g.W, g.C, -g.ph, -g.pw, g.ph - (g.R - 1), g.pw - (g.S - 1),
                                 g.sh, g.sw, BK, rows);
        // multi-tap: a row tile spans rows / C whole taps (C a power of two, >= 32 so
        // the plain [BK][C] box needs no swizzle): one im2col box per tap, smem
        // tap-blocked [rows / C][BK][C] (kcontig 3, tap-block loop in the kernel)
        if (rows % g.C || (g.C & (g.C - 1)) || g.C < 32 || (path_policy() & 32)) return 0;
        int m = encode_im2col(map, op.x, g.N, g.H, g.W, g.C, -g.ph, -g.pw, g.ph - (g.R - 1), g.pw - (g.S - 1), g.sh,
                              g.sw, BK, g.C);
        if (!m) return 0;
        d.kcontig = 3;
        d.cblk_log2 = __builtin_ctz(unsigned(g.C));
        return 5;
    }
    cuuint64_t dims[2] = {cuuint64_t(op.g.C), cuuint64_t(op.Kd)};
    cuuint64_t st[1] = {cuuint64_t(op.g.C) * 4};
    cuuint32_t box[2] = {cuuint32_t(rows), cuuint32_t(BK)};
    return encode_tma(map, op.x, 2, dims, st, box, false);
}

// conv dgrad A: for 1x1 / unpadded (any stride: one phase with a tap), dy as [pixels][K];
// other stride-1 convs: im2col mode over dy (lower = pad - (R-1),
// upper = pad - (R-1) + H - OH) when K % BK == 0
static int setup_tma(CUtensorMap *map, const DgDY &op, int rows, OpDesc &d)
{
    if (tma_disabled()) return 0;
    const ConvGeom &g = op.g;
    // 1x1 unpadded, any stride: only phase (0, 0) has a tap, and its rows are
    // dy's pixels in order (Hp = OH, Wp = OW) -- the plain 2-D box below
    if (!(g.R == 1 && g.S == 1 && g.ph == 0 && g.pw == 0)) {
        if (g.sh != 1 || g.sw != 1) {   // per-phase descriptors encoded by the entry point (encode_dgrad_phases)
            if (!op.ph_tma) return 0;
            d.kcontig = 2;
            return 6;
        }
        int m = encode_im2col(map, op.dy, g.N, g.OH, g.OW, g.K, g.ph - (g.R - 1), g.pw - (g.S - 1),
                              g.ph - (g.R - 1) + g.H - g.OH, g.pw - (g.S - 1) + g.W - g.OW, 1, 1, rows);
        if (m) d.kcontig = 2;
        return m;
    }
    cuuint64_t dims[2] = {cuuint64_t(op.g.K), cuuint64_t(int64_t(op.g.N) * op.g.OH * op.g.OW)};
    cuuint64_t st[1] = {cuuint64_t(op.g.K) * 4};
    cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(rows)};
    int m = encode_tma(map, op.dy, 2, dims, st, box, true);
    if (m) d.kcontig = 2;
    return m;
}

// Strided dgrad (2 x 2 phases): one im2col descriptor over dy per phase with
// lower corner (lo_h, lo_w) and upper = lower + (Hp, Wp) - (OH, OW), so the box
// walks the phase's Hp x Wp output pixels and the tap offsets (j, i) reach the
// dy pixels of the phase's taps (reverse_transpose order, as for stride 1).
// Returns false (cp.async gathers) when any phase cannot be encoded.
static bool encode_dgrad_phases(DgDY &op, int nsub, int rows)
{
    const ConvGeom &g = op.g;
    if (tma_disabled() || (path_policy() & 32) || nsub > MAX_PH_TMA || g.K % BK) return false;
    for (int s = 0; s < nsub; s++) {
        const DgPhase &P = op.ph[s];
        if (P.th == 0 || P.tw == 0 || P.Hp == 0 || P.Wp == 0) continue;   // no k-tiles / rows: never loaded
        if (!encode_im2col(&op.ph_map[s], op.dy, g.N, g.OH, g.OW, g.K, P.lo_h, P.lo_w, P.lo_h + P.Hp - g.OH,
                           P.lo_w + P.Wp - g.OW, 1, 1, rows))
            return false;
    }
    return true;
}

// conv dgrad B: the reverse-transposed weight taps, a 3-D box {co, ci, tap} of w
// as [R*S][C][K] when every k-tile lies inside one tap (K % BK == 0)
static int setup_tma(CUtensorMap *map, const DgW &op, int rows, OpDesc &d)
{
    if (tma_disabled() || op.g.K % BK) return 0;
    cuuint64_t dims[3] = {cuuint64_t(op.g.K), cuuint64_t(op.g.C), cuuint64_t(op.g.R) * op.g.S};
    cuuint64_t st[2] = {cuuint64_t(op.g.K) * 4, cuuint64_t(op.g.C) * op.g.K * 4};
    cuuint32_t box[3] = {cuuint32_t(BK), cuuint32_t(rows), 1};
    int m = encode_tma(map, op.w, 3, dims, st, box, true);
    if (m) d.kcontig = 2;
    return m;
}

// Transposed orientation: the row operand is the original B (opr), the lanes'
// the original A (opc); shared-memory tables of 8 / 16 bits only.
template <int EB, class OpR, class OpC>
static amsim_status launch_trn(const KParams &p, const OpR &r, const OpC &c, cudaStream_t st)
{
    switch (CfgId(p.cfg)) {
    case CfgId::Wide: return launch_cfg<CfgWide, EB, OpR, OpC, false, MUL_LUT, true>(p, r, c, st);
    case CfgId::Flat: return launch_cfg<CfgFlat, EB, OpR, OpC, false, MUL_LUT, true>(p, r, c, st);
    case CfgId::Flat3: return launch_cfg<CfgFlat3, EB, OpR, OpC, false, MUL_LUT, true>(p, r, c, st);
    case CfgId::Flat8:
        if constexpr (EB == 16) return launch_cfg<CfgFlat8, EB, OpR, OpC, false, MUL_LUT, true>(p, r, c, st);
        else break;
    case CfgId::TallT: return launch_cfg<CfgTallT, EB, OpR, OpC, false, MUL_LUT, true>(p, r, c, st);
    case CfgId::Big: return launch_cfg<CfgBig, EB, OpR, OpC, false, MUL_LUT, true>(p, r, c, st);
    case CfgId::Huge:
        if constexpr (EB >= 16) return launch_cfg<CfgHuge, EB, OpR, OpC, false, MUL_LUT, true>(p, r, c, st);
        else break;
    default: break;
    }
    return set_error(AMSIM_ERR_UNSUPPORTED, "internal: transposed orientation with this tile configuration");
}

// Launch the GEMM core.  A stream-K plan needs `ws` (partial tiles and tile
// counters, p.ws_elems words): the caller's workspace or, when nullptr, a
// stream-ordered allocation; its counters are zeroed on the stream first.
template <class OpA, class OpB>
static amsim_status run(int eb, KParams p, const OpA &a, const OpB &b, cudaStream_t st, float *ws = nullptr)
{
    bool own = false;
    if (p.ws_elems > 0) {
        if (!ws) {
            void *q = nullptr;
            amsim_status s = scratch_alloc(&q, size_t(p.ws_elems) * sizeof(float), st);
            if (s != AMSIM_OK) return s;
            ws = static_cast<float *>(q);
            own = true;
        }
        p.ws = ws;
        // stream-K fix-up tree counters start at zero (SK_LEVELS x 2 per stream-K CTA,
        // after the partial slots)
        const int64_t ncnt = int64_t(SK_LEVELS) * 2 * p.sk_G;
        cudaError_t e = cudaMemsetAsync(ws + (p.ws_elems - ncnt), 0, size_t(ncnt) * 4, st);
        if (e != cudaSuccess) {
            if (own) scratch_free(ws, st);
            return cuda_check(e, "stream-K counter reset");
        }
    }
    int BM, BN, NT;
    size_t smem;
    cfg_shape(CfgId(p.cfg), BM, BN, NT, smem, 0);
    amsim_status s;
    if (p.trn) {   // rows = original B operand, lanes = original A operand
        std::swap(p.da, p.db);
        p.tma_on[0] = setup_tma(&p.tma[0], b, std::min(BM, 256), p.da);
        p.tma_on[1] = setup_tma(&p.tma[1], a, std::min(BN, 256), p.db);   // taller tiles: several boxes
        if (CfgId(p.cfg) == CfgId::Flat8 &&
            !(p.tma_on[0] && p.tma_on[1] && p.da.kcontig != 1 && p.db.kcontig == 2 && p.tma_on[1] != 5)) {
            if (own) scratch_free(ws, st);
            return set_error(AMSIM_ERR_UNSUPPORTED, "internal: the 64 x 512 tile needs TMA-staged operands");
        }
        s = eb == 8 ? launch_trn<8>(p, b, a, st) : launch_trn<16>(p, b, a, st);
    } else {
        p.tma_on[0] = setup_tma(&p.tma[0], a, BM, p.da);
        p.tma_on[1] = setup_tma(&p.tma[1], b, BN, p.db);
        s = (eb == 8 && p.mul == MUL_LUT)    ? launch_eb<8>(p, a, b, st)
            : (eb == 16 && p.mul == MUL_LUT) ? launch_eb<16>(p, a, b, st)
                                             : launch_eb<32>(p, a, b, st);
    }
    if (own) scratch_free(ws, st);
    return s;
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
    if (d->stride_h * d->stride_w > MAX_SUB)
        return set_error(AMSIM_ERR_UNSUPPORTED, "stride_h * stride_w > 9 is not supported");
    return AMSIM_OK;
}

// Stride phases of the preceding-layer gradient (see DgPhase).
static void dgrad_phases(const amsim_conv2d_desc *d, Problem &pr, DgPhase *ph)
{
    const int sh = d->stride_h, sw = d->stride_w;
    pr.N = d->C;
    pr.nsub = sh * sw;
    for (int a = 0; a < sh; a++)
        for (int b = 0; b < sw; b++) {
            DgPhase &P = ph[a * sw + b];
            P.a = a;
            P.b = b;
            P.ch = ((a - d->pad_h) % sh + sh) % sh;
            P.cw = ((b - d->pad_w) % sw + sw) % sw;
            P.th = a < d->R ? (d->R - a + sh - 1) / sh : 0;
            P.tw = b < d->S ? (d->S - b + sw - 1) / sw : 0;
            P.Hp = P.ch < d->H ? (d->H - P.ch + sh - 1) / sh : 0;
            P.Wp = P.cw < d->W ? (d->W - P.cw + sw - 1) / sw : 0;
            P.fHpWp.init(uint32_t(std::max(1, P.Hp * P.Wp)));
            P.fWp.init(uint32_t(std::max(1, P.Wp)));
            P.fTwK.init(uint32_t(std::max(1, P.tw * d->K)));
            // dy row read by output row u at tap offset i: u + lo_h + i, lo_h = (ch + ph - a) / sh - (th - 1)
            P.lo_h = (P.ch + d->pad_h - a) / sh - (P.th - 1);
            P.lo_w = (P.cw + d->pad_w - b) / sw - (P.tw - 1);
            pr.M[a * sw + b] = d->N * P.Hp * P.Wp;
            pr.K[a * sw + b] = P.th * P.tw * d->K;
        }
}

}  // namespace amsim
