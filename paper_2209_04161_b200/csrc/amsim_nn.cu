// libamsim: the non-approximated layers of a full training / inference step
// (include/amsim_nn.h).  Native FP32 arithmetic
// (PAPER.md:480 approximates only Conv2D / Dense multiplications).  All of
// these are HBM-bound: NHWC rows with the channel dimension innermost, float4
// accesses when C % 4 == 0, per-channel reductions in two deterministic stages
// (per-block partials in FP64, then a fixed-order sum per channel).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "../../include/amsim_nn.h"
#include "amsim_internal.h"

namespace amsim {
namespace nn {

constexpr int NT = 256;

static int64_t reduce_blocks(int64_t P)
{
    // depends only on P (not on the device), so results are reproducible everywhere
    return std::max<int64_t>(1, std::min<int64_t>((P + 63) / 64, 512));
}

static amsim_status check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return AMSIM_OK;
    return set_error(AMSIM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static size_t ws_need(int64_t P, int32_t C)
{
    // partials [G][C] x (2 doubles) + per-channel coefficients [4][C] floats
    return size_t(reduce_blocks(P)) * C * 16 + size_t(C) * 16 + 256;
}

// ---------------------------------------------------------------------------
// Per-channel reduction of two quantities over P rows: partial[g][c] =
// (sum_a, sum_b) over the rows of block g.  F(row, c) -> float2.
template <class F>
__global__ void __launch_bounds__(NT) channel_partials(int64_t P, int32_t C, F f, double2 *part)
{
    __shared__ double2 red[NT];
    const int64_t G = gridDim.x;
    const int64_t r0 = P * blockIdx.x / G, r1 = P * (blockIdx.x + 1) / G;
    const int tid = threadIdx.x;
    if (C >= NT) {
        for (int c = tid; c < C; c += NT) {
            float a = 0.f, b = 0.f;
            for (int64_t r = r0; r < r1; r++) {
                float2 v = f(r, c);
                a += v.x;
                b += v.y;
            }
            part[blockIdx.x * int64_t(C) + c] = make_double2(a, b);
        }
        return;
    }
    const int rp = NT / C;  // rows in parallel
    const int c = tid % C, rl = tid / C;
    float a = 0.f, b = 0.f;
    if (rl < rp)
        for (int64_t r = r0 + rl; r < r1; r += rp) {
            float2 v = f(r, c);
            a += v.x;
            b += v.y;
        }
    red[tid] = make_double2(a, b);
    __syncthreads();
    if (tid < C) {
        double sa = 0, sb = 0;
        for (int i = 0; i < rp; i++) {
            sa += red[i * C + tid].x;
            sb += red[i * C + tid].y;
        }
        part[blockIdx.x * int64_t(C) + tid] = make_double2(sa, sb);
    }
}

// Same with 4 channels per thread (C % 4 == 0, 16-byte aligned tensors):
// F(row, c4, a, b) accumulates channels 4*c4 .. 4*c4+3; rows are processed two
// at a time for memory-level parallelism.
template <class F>
__global__ void __launch_bounds__(NT) channel_partials4(int64_t P, int32_t C, F f, double2 *part)
{
    __shared__ float4 red[2][NT];
    const int64_t G = gridDim.x;
    const int64_t r0 = P * blockIdx.x / G, r1 = P * (blockIdx.x + 1) / G;
    const int tid = threadIdx.x, C4 = C / 4;
    auto store = [&](int c4, const float4 &a, const float4 &b) {
        double2 *o = part + blockIdx.x * int64_t(C) + 4 * c4;
        o[0] = make_double2(a.x, b.x);
        o[1] = make_double2(a.y, b.y);
        o[2] = make_double2(a.z, b.z);
        o[3] = make_double2(a.w, b.w);
    };
    if (C4 >= NT) {
        for (int c4 = tid; c4 < C4; c4 += NT) {
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, a2 = a, b2 = a;
            int64_t r = r0;
            for (; r + 1 < r1; r += 2) {
                f(r, c4, a, b);
                f(r + 1, c4, a2, b2);
            }
            if (r < r1) f(r, c4, a, b);
            a.x += a2.x; a.y += a2.y; a.z += a2.z; a.w += a2.w;
            b.x += b2.x; b.y += b2.y; b.z += b2.z; b.w += b2.w;
            store(c4, a, b);
        }
        return;
    }
    const int rp = NT / C4;
    const int c4 = tid % C4, rl = tid / C4;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, a2 = a, b2 = a;
    if (rl < rp) {
        int64_t r = r0 + rl;
        for (; r + rp < r1; r += 2 * rp) {
            f(r, c4, a, b);
            f(r + rp, c4, a2, b2);
        }
        if (r < r1) f(r, c4, a, b);
    }
    a.x += a2.x; a.y += a2.y; a.z += a2.z; a.w += a2.w;
    b.x += b2.x; b.y += b2.y; b.z += b2.z; b.w += b2.w;
    red[0][tid] = a;
    red[1][tid] = b;
    __syncthreads();
    if (tid < C4) {
        double sa[4] = {0, 0, 0, 0}, sb[4] = {0, 0, 0, 0};
        for (int i = 0; i < rp; i++) {
            float4 u = red[0][i * C4 + tid], v = red[1][i * C4 + tid];
            sa[0] += u.x; sa[1] += u.y; sa[2] += u.z; sa[3] += u.w;
            sb[0] += v.x; sb[1] += v.y; sb[2] += v.z; sb[3] += v.w;
        }
        double2 *o = part + blockIdx.x * int64_t(C) + 4 * tid;
        for (int j = 0; j < 4; j++) o[j] = make_double2(sa[j], sb[j]);
    }
}

__device__ __forceinline__ void acc4(float4 &a, float x0, float x1, float x2, float x3)
{
    a.x += x0; a.y += x1; a.z += x2; a.w += x3;
}

// fixed-order sum of the partials of channel c
__device__ __forceinline__ double2 sum_partials(const double2 *part, int64_t G, int32_t C, int c)
{
    double a = 0, b = 0;
    for (int64_t g = 0; g < G; g++) {
        double2 v = part[g * C + c];
        a += v.x;
        b += v.y;
    }
    return make_double2(a, b);
}

struct StatsF {
    const float *x;
    int32_t C;
    __device__ float2 operator()(int64_t r, int c) const
    {
        float v = x[r * C + c];
        return make_float2(v, v * v);
    }
};

__global__ void bn_stats_finalize(const double2 *part, int64_t G, int64_t P, int32_t C, const float *gamma,
                                  const float *beta, float eps, float *save_mean, float *save_invstd,
                                  float *running_mean, float *running_var, float momentum, float *scale,
                                  float *shift)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double2 s = sum_partials(part, G, C, c);
    double mean = s.x / double(P);
    double var = fmax(0.0, s.y / double(P) - mean * mean);
    float invstd = float(1.0 / sqrt(var + double(eps)));
    save_mean[c] = float(mean);
    save_invstd[c] = invstd;
    float sc = gamma[c] * invstd;
    scale[c] = sc;
    shift[c] = beta[c] - float(mean) * sc;
    if (running_mean) running_mean[c] = (1.f - momentum) * running_mean[c] + momentum * float(mean);
    if (running_var)
        running_var[c] = (1.f - momentum) * running_var[c] +
                         momentum * float(P > 1 ? var * double(P) / double(P - 1) : var);
}

__global__ void bn_infer_coeffs(int32_t C, const float *gamma, const float *beta, const float *rmean,
                                const float *rvar, float eps, float *scale, float *shift)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    float sc = gamma[c] / sqrtf(rvar[c] + eps);
    scale[c] = sc;
    shift[c] = beta[c] - rmean[c] * sc;
}

// y = [relu](x * scale_c + shift_c [+ res])
template <int V>
__global__ void __launch_bounds__(NT) bn_apply(const float *x, int64_t n, int32_t C, const float *scale,
                                               const float *shift, const float *res, int relu, float *y)
{
    for (int64_t i = (blockIdx.x * int64_t(NT) + threadIdx.x) * V; i < n; i += int64_t(gridDim.x) * NT * V) {
        const int c = int(i % C);
        if constexpr (V == 4) {
            float4 v = *reinterpret_cast<const float4 *>(x + i);
            float4 s = *reinterpret_cast<const float4 *>(scale + c);
            float4 t = *reinterpret_cast<const float4 *>(shift + c);
            float4 o = make_float4(fmaf(v.x, s.x, t.x), fmaf(v.y, s.y, t.y), fmaf(v.z, s.z, t.z), fmaf(v.w, s.w, t.w));
            if (res) {
                float4 r = *reinterpret_cast<const float4 *>(res + i);
                o.x += r.x; o.y += r.y; o.z += r.z; o.w += r.w;
            }
            if (relu) {
                o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
            }
            *reinterpret_cast<float4 *>(y + i) = o;
        } else {
            float o = fmaf(x[i], scale[c], shift[c]);
            if (res) o += res[i];
            if (relu) o = fmaxf(o, 0.f);
            y[i] = o;
        }
    }
}

struct StatsF4 {
    const float *x;
    int32_t C;
    __device__ __forceinline__ void operator()(int64_t r, int c4, float4 &a, float4 &b) const
    {
        float4 v = *reinterpret_cast<const float4 *>(x + r * C + 4 * c4);
        acc4(a, v.x, v.y, v.z, v.w);
        acc4(b, v.x * v.x, v.y * v.y, v.z * v.z, v.w * v.w);
    }
};

struct BnBwdF {
    const float *dy, *y, *x, *mean, *invstd;
    int32_t C;
    int relu;
    __device__ float2 operator()(int64_t r, int c) const
    {
        int64_t i = r * C + c;
        float dz = (relu && !(y[i] > 0.f)) ? 0.f : dy[i];
        float xh = (x[i] - mean[c]) * invstd[c];
        return make_float2(dz, dz * xh);
    }
};

__global__ void bn_bwd_finalize(const double2 *part, int64_t G, int64_t P, int32_t C, const float *gamma,
                                const float *invstd, float *dgamma, float *dbeta, float *k1, float *mdz,
                                float *mdzx)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    double2 s = sum_partials(part, G, C, c);
    dbeta[c] = float(s.x);
    dgamma[c] = float(s.y);
    k1[c] = gamma[c] * invstd[c];
    mdz[c] = float(s.x / double(P));
    mdzx[c] = float(s.y / double(P));
}

__global__ void __launch_bounds__(NT) bn_bwd_apply4(const float *dy, const float *y, const float *x, int64_t n,
                                                    int32_t C, const float *mean, const float *invstd,
                                                    const float *k1, const float *mdz, const float *mdzx, int relu,
                                                    float *dx, float *dres)
{
    for (int64_t i = (blockIdx.x * int64_t(NT) + threadIdx.x) * 4; i < n; i += int64_t(gridDim.x) * NT * 4) {
        const int c = int(i % C);
        float4 g = *reinterpret_cast<const float4 *>(dy + i);
        if (relu) {
            float4 o = *reinterpret_cast<const float4 *>(y + i);
            g.x = o.x > 0.f ? g.x : 0.f; g.y = o.y > 0.f ? g.y : 0.f;
            g.z = o.z > 0.f ? g.z : 0.f; g.w = o.w > 0.f ? g.w : 0.f;
        }
        float4 v = *reinterpret_cast<const float4 *>(x + i);
        float4 m = *reinterpret_cast<const float4 *>(mean + c), s = *reinterpret_cast<const float4 *>(invstd + c);
        float4 k = *reinterpret_cast<const float4 *>(k1 + c), z = *reinterpret_cast<const float4 *>(mdz + c);
        float4 w = *reinterpret_cast<const float4 *>(mdzx + c);
        float4 r;
        r.x = k.x * (g.x - z.x - (v.x - m.x) * s.x * w.x);
        r.y = k.y * (g.y - z.y - (v.y - m.y) * s.y * w.y);
        r.z = k.z * (g.z - z.z - (v.z - m.z) * s.z * w.z);
        r.w = k.w * (g.w - z.w - (v.w - m.w) * s.w * w.w);
        *reinterpret_cast<float4 *>(dx + i) = r;
        if (dres) *reinterpret_cast<float4 *>(dres + i) = g;
    }
}

__global__ void __launch_bounds__(NT) bn_bwd_apply(const float *dy, const float *y, const float *x, int64_t n,
                                                   int32_t C, const float *mean, const float *invstd,
                                                   const float *k1, const float *mdz, const float *mdzx, int relu,
                                                   float *dx, float *dres)
{
    for (int64_t i = blockIdx.x * int64_t(NT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * NT) {
        const int c = int(i % C);
        float dz = (relu && !(y[i] > 0.f)) ? 0.f : dy[i];
        float xh = (x[i] - mean[c]) * invstd[c];
        dx[i] = k1[c] * (dz - mdz[c] - xh * mdzx[c]);
        if (dres) dres[i] = dz;
    }
}

// ---------------------------------------------------------------------------
// bias + activation

__global__ void __launch_bounds__(NT) bias_act_fwd_k(const float *x, int64_t n, int32_t C, const float *bias,
                                                     int relu, float *y)
{
    for (int64_t i = blockIdx.x * int64_t(NT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * NT) {
        float o = x[i] + bias[i % C];
        y[i] = relu ? fmaxf(o, 0.f) : o;
    }
}

struct BnBwdF4 {
    const float *dy, *y, *x, *mean, *invstd;
    int32_t C;
    int relu;
    __device__ __forceinline__ void operator()(int64_t r, int c4, float4 &a, float4 &b) const
    {
        const int64_t i = r * C + 4 * c4;
        float4 g = *reinterpret_cast<const float4 *>(dy + i);
        float4 v = *reinterpret_cast<const float4 *>(x + i);
        float4 m = *reinterpret_cast<const float4 *>(mean + 4 * c4);
        float4 s = *reinterpret_cast<const float4 *>(invstd + 4 * c4);
        if (relu) {
            float4 o = *reinterpret_cast<const float4 *>(y + i);
            g.x = o.x > 0.f ? g.x : 0.f; g.y = o.y > 0.f ? g.y : 0.f;
            g.z = o.z > 0.f ? g.z : 0.f; g.w = o.w > 0.f ? g.w : 0.f;
        }
        acc4(a, g.x, g.y, g.z, g.w);
        acc4(b, g.x * ((v.x - m.x) * s.x), g.y * ((v.y - m.y) * s.y), g.z * ((v.z - m.z) * s.z),
             g.w * ((v.w - m.w) * s.w));
    }
};

struct BiasBwdF {  // writes dx while reducing (each element is visited exactly once)
    const float *dy, *y;
    float *dx;
    int32_t C;
    int relu;
    __device__ float2 operator()(int64_t r, int c) const
    {
        int64_t i = r * C + c;
        float dz = (relu && !(y[i] > 0.f)) ? 0.f : dy[i];
        dx[i] = dz;
        return make_float2(dz, 0.f);
    }
};

__global__ void bias_bwd_finalize(const double2 *part, int64_t G, int32_t C, float *dbias)
{
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    dbias[c] = float(sum_partials(part, G, C, c).x);
}

// ---------------------------------------------------------------------------
// pooling

__global__ void __launch_bounds__(NT) maxpool_fwd_k(const float *x, int N, int H, int W, int C, int R, int S, int st,
                                                    int pad, int OH, int OW, float *y, uint8_t *am)
{
    const int64_t n_out = int64_t(N) * OH * OW * C;
    for (int64_t i = blockIdx.x * int64_t(NT) + threadIdx.x; i < n_out; i += int64_t(gridDim.x) * NT) {
        int c = int(i % C);
        int64_t p = i / C;
        int ow = int(p % OW);
        p /= OW;
        int oh = int(p % OH);
        int n = int(p / OH);
        float best = -INFINITY;
        int arg = 0;
        bool any = false;
        for (int kh = 0; kh < R; kh++) {
            int h = oh * st - pad + kh;
            if (h < 0 || h >= H) continue;
            for (int kw = 0; kw < S; kw++) {
                int w = ow * st - pad + kw;
                if (w < 0 || w >= W) continue;
                float v = x[((int64_t(n) * H + h) * W + w) * C + c];
                if (!any || v > best || (v != v && best == best)) {  // first maximum; NaN propagates
                    best = v;
                    arg = kh * S + kw;
                    any = true;
                }
            }
        }
        y[i] = best;
        am[i] = uint8_t(arg);
    }
}

__global__ void __launch_bounds__(NT) maxpool_bwd_k(const float *dy, const uint8_t *am, int N, int H, int W, int C,
                                                    int R, int S, int st, int pad, int OH, int OW, float *dx)
{
    const int64_t n_in = int64_t(N) * H * W * C;
    for (int64_t i = blockIdx.x * int64_t(NT) + threadIdx.x; i < n_in; i += int64_t(gridDim.x) * NT) {
        int c = int(i % C);
        int64_t p = i / C;
        int w = int(p % W);
        p /= W;
        int h = int(p % H);
        int n = int(p / H);
        // output rows oh with oh*st - pad <= h <= oh*st - pad + R - 1
        int oh0 = max(0, (h + pad - R + st) / st), oh1 = min(OH - 1, (h + pad) / st);
        int ow0 = max(0, (w + pad - S + st) / st), ow1 = min(OW - 1, (w + pad) / st);
        if (h + pad - R + 1 < 0) oh0 = 0;
        if (w + pad - S + 1 < 0) ow0 = 0;
        float s = 0.f;
        for (int oh = oh0; oh <= oh1; oh++) {
            int kh = h - (oh * st - pad);
            if (kh < 0 || kh >= R) continue;
            for (int ow = ow0; ow <= ow1; ow++) {
                int kw = w - (ow * st - pad);
                if (kw < 0 || kw >= S) continue;
                int64_t o = ((int64_t(n) * OH + oh) * OW + ow) * C + c;
                if (am[o] == kh * S + kw) s += dy[o];
            }
        }
        dx[i] = s;
    }
}

__global__ void __launch_bounds__(NT) avgpool_fwd_k(const float *x, int N, int HW, int C, float *y)
{
    const int64_t n_out = int64_t(N) * C;
    for (int64_t i = blockIdx.x * int64_t(NT) + threadIdx.x; i < n_out; i += int64_t(gridDim.x) * NT) {
        int c = int(i % C);
        int64_t n = i / C;
        const float *p = x + n * HW * C + c;
        float s = 0.f;
        for (int j = 0; j < HW; j++) s += p[int64_t(j) * C];
        y[i] = s / float(HW);
    }
}

__global__ void __launch_bounds__(NT) avgpool_bwd_k(const float *dy, int N, int HW, int C, float *dx)
{
    const int64_t n_in = int64_t(N) * HW * C;
    const float inv = 1.f / float(HW);
    for (int64_t i = blockIdx.x * int64_t(NT) + threadIdx.x; i < n_in; i += int64_t(gridDim.x) * NT) {
        int c = int(i % C);
        int64_t n = i / (int64_t(HW) * C);
        dx[i] = dy[n * C + c] * inv;
    }
}

// ---------------------------------------------------------------------------
// softmax cross-entropy (one block per row), then a fixed-order mean

__device__ float block_reduce(float v, bool is_max, float *sh)
{
    for (int o = 16; o > 0; o >>= 1) {
        float u = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmaxf(v, u) : v + u;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    float r = sh[0];
    for (int i = 1; i < NT / 32; i++) r = is_max ? fmaxf(r, sh[i]) : r + sh[i];
    return r;
}

__global__ void __launch_bounds__(NT) softmax_xent_k(const float *z, const int32_t *labels, int N, int K,
                                                     float inv_n, float *dz, float *row_loss)
{
    __shared__ float sh[NT / 32];
    const int n = blockIdx.x;
    const float *zr = z + int64_t(n) * K;
    float m = -INFINITY;
    for (int k = threadIdx.x; k < K; k += NT) m = fmaxf(m, zr[k]);
    m = block_reduce(m, true, sh);
    float s = 0.f;
    for (int k = threadIdx.x; k < K; k += NT) s += __expf(zr[k] - m);
    s = block_reduce(s, false, sh);
    const int lab = labels[n];
    for (int k = threadIdx.x; k < K; k += NT) {
        float p = __expf(zr[k] - m) / s;
        dz[int64_t(n) * K + k] = (p - (k == lab ? 1.f : 0.f)) * inv_n;
    }
    if (threadIdx.x == 0) row_loss[n] = logf(s) + m - ((lab >= 0 && lab < K) ? zr[lab] : m + logf(s));
}

__global__ void mean_k(const float *v, int N, float *out)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0;
        for (int i = 0; i < N; i++) s += v[i];
        out[0] = float(s / N);
    }
}

__global__ void __launch_bounds__(NT) add_k(const float *a, const float *b, float *o, int64_t n)
{
    const int64_t n4 = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(o)) & 15)
                           ? 0 : n / 4;
    for (int64_t i = blockIdx.x * int64_t(NT) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * NT) {
        float4 u = reinterpret_cast<const float4 *>(a)[i], v = reinterpret_cast<const float4 *>(b)[i];
        reinterpret_cast<float4 *>(o)[i] = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
    }
    for (int64_t i = n4 * 4 + blockIdx.x * int64_t(NT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * NT)
        o[i] = a[i] + b[i];
}

__global__ void __launch_bounds__(NT) sgd_k(float *w, const float *g, float *v, int64_t n, float lr, float mom,
                                            float wd)
{
    for (int64_t i = blockIdx.x * int64_t(NT) + threadIdx.x; i < n; i += int64_t(gridDim.x) * NT) {
        float vi = mom * v[i] + (g[i] + wd * w[i]);
        v[i] = vi;
        w[i] -= lr * vi;
    }
}

static int grid_for(int64_t n)
{
    return int(std::max<int64_t>(1, std::min<int64_t>((n + NT - 1) / NT, 148 * 16)));
}

static bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace nn
}  // namespace amsim

using namespace amsim;
using namespace amsim::nn;

extern "C" {

size_t amsim_nn_workspace_bytes(int64_t P, int32_t C) { return ws_need(P, C); }

static amsim_status check_pc(int64_t P, int32_t C, const void *ws, size_t ws_bytes, const char *fn)
{
    if (P < 0 || C <= 0) return set_error(AMSIM_ERR_INVALID_ARG, std::string(fn) + ": P >= 0 and C > 0 required");
    if (ws_bytes < ws_need(P, C) || !ws)
        return set_error(AMSIM_ERR_INVALID_ARG, std::string(fn) + ": workspace too small (need " +
                                                    std::to_string(ws_need(P, C)) + " bytes)");
    return AMSIM_OK;
}

amsim_status amsim_bn_fwd_train(const float *x, int64_t P, int32_t C, const float *gamma, const float *beta,
                                float eps, const float *res, int relu, float *y, float *save_mean,
                                float *save_invstd, float *running_mean, float *running_var, float momentum,
                                void *ws, size_t ws_bytes, amsim_stream_t stream)
{
    clear_error();
    amsim_status s = check_pc(P, C, ws, ws_bytes, "amsim_bn_fwd_train");
    if (s != AMSIM_OK) return s;
    if (P == 0) return AMSIM_OK;
    if (!x || !gamma || !beta || !y || !save_mean || !save_invstd)
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_bn_fwd_train: null tensor");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t G = reduce_blocks(P);
    double2 *part = static_cast<double2 *>(ws);
    float *scale = reinterpret_cast<float *>(static_cast<char *>(ws) + G * C * 16);
    float *shift = scale + C;
    if (C % 4 == 0 && al16(x))
        channel_partials4<<<int(G), NT, 0, st>>>(P, C, StatsF4{x, C}, part);
    else
        channel_partials<<<int(G), NT, 0, st>>>(P, C, StatsF{x, C}, part);
    bn_stats_finalize<<<(C + 127) / 128, 128, 0, st>>>(part, G, P, C, gamma, beta, eps, save_mean, save_invstd,
                                                       running_mean, running_var, momentum, scale, shift);
    const int64_t n = P * C;
    bool v4 = C % 4 == 0 && al16(x) && al16(y) && (!res || al16(res)) && al16(scale);
    if (v4)
        bn_apply<4><<<grid_for(n / 4), NT, 0, st>>>(x, n, C, scale, shift, res, relu, y);
    else
        bn_apply<1><<<grid_for(n), NT, 0, st>>>(x, n, C, scale, shift, res, relu, y);
    count_launch(3);
    return check_launch("amsim_bn_fwd_train");
}

amsim_status amsim_bn_fwd_infer(const float *x, int64_t P, int32_t C, const float *gamma, const float *beta,
                                const float *running_mean, const float *running_var, float eps,
                                const float *res, int relu, float *y, amsim_stream_t stream)
{
    clear_error();
    if (P < 0 || C <= 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_bn_fwd_infer: P >= 0 and C > 0 required");
    if (P == 0) return AMSIM_OK;
    if (!x || !gamma || !beta || !running_mean || !running_var || !y)
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_bn_fwd_infer: null tensor");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    float *coef = nullptr;
    if (scratch_alloc(reinterpret_cast<void **>(&coef), size_t(C) * 8 + 16, st) != AMSIM_OK)
        return set_error(AMSIM_ERR_NOMEM, "amsim_bn_fwd_infer: scratch allocation");
    float *scale = coef, *shift = coef + ((C + 3) & ~3);
    bn_infer_coeffs<<<(C + 127) / 128, 128, 0, st>>>(C, gamma, beta, running_mean, running_var, eps, scale, shift);
    const int64_t n = P * C;
    bool v4 = C % 4 == 0 && al16(x) && al16(y) && (!res || al16(res));
    if (v4)
        bn_apply<4><<<grid_for(n / 4), NT, 0, st>>>(x, n, C, scale, shift, res, relu, y);
    else
        bn_apply<1><<<grid_for(n), NT, 0, st>>>(x, n, C, scale, shift, res, relu, y);
    scratch_free(coef, st);
    count_launch(2);
    return check_launch("amsim_bn_fwd_infer");
}

amsim_status amsim_bn_bwd(const float *dy, const float *y, const float *x, int64_t P, int32_t C,
                          const float *gamma, const float *save_mean, const float *save_invstd, int relu,
                          float *dx, float *dres, float *dgamma, float *dbeta, void *ws, size_t ws_bytes,
                          amsim_stream_t stream)
{
    clear_error();
    amsim_status s = check_pc(P, C, ws, ws_bytes, "amsim_bn_bwd");
    if (s != AMSIM_OK) return s;
    if (P == 0) return AMSIM_OK;
    if (!dy || !x || !gamma || !save_mean || !save_invstd || !dx || !dgamma || !dbeta || (relu && !y))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_bn_bwd: null tensor");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t G = reduce_blocks(P);
    double2 *part = static_cast<double2 *>(ws);
    float *k1 = reinterpret_cast<float *>(static_cast<char *>(ws) + G * C * 16);
    float *mdz = k1 + C, *mdzx = mdz + C;
    const bool v4 = C % 4 == 0 && al16(dy) && al16(x) && (!y || al16(y)) && al16(dx) && (!dres || al16(dres)) &&
                    al16(save_mean) && al16(save_invstd);
    if (v4)
        channel_partials4<<<int(G), NT, 0, st>>>(P, C, BnBwdF4{dy, y, x, save_mean, save_invstd, C, relu}, part);
    else
        channel_partials<<<int(G), NT, 0, st>>>(P, C, BnBwdF{dy, y, x, save_mean, save_invstd, C, relu}, part);
    bn_bwd_finalize<<<(C + 127) / 128, 128, 0, st>>>(part, G, P, C, gamma, save_invstd, dgamma, dbeta, k1, mdz, mdzx);
    if (v4 && al16(k1))
        bn_bwd_apply4<<<grid_for(P * C / 4), NT, 0, st>>>(dy, y, x, P * C, C, save_mean, save_invstd, k1, mdz, mdzx,
                                                          relu, dx, dres);
    else
        bn_bwd_apply<<<grid_for(P * C), NT, 0, st>>>(dy, y, x, P * C, C, save_mean, save_invstd, k1, mdz, mdzx, relu,
                                                     dx, dres);
    count_launch(3);
    return check_launch("amsim_bn_bwd");
}

amsim_status amsim_bias_act_fwd(const float *x, int64_t P, int32_t C, const float *bias, int relu, float *y,
                                amsim_stream_t stream)
{
    clear_error();
    if (P < 0 || C <= 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_bias_act_fwd: P >= 0 and C > 0 required");
    if (P == 0) return AMSIM_OK;
    if (!x || !bias || !y) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_bias_act_fwd: null tensor");
    bias_act_fwd_k<<<grid_for(P * C), NT, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, P * C, C, bias, relu, y);
    count_launch();
    return check_launch("amsim_bias_act_fwd");
}

amsim_status amsim_bias_act_bwd(const float *dy, const float *y, int64_t P, int32_t C, int relu, float *dx,
                                float *dbias, void *ws, size_t ws_bytes, amsim_stream_t stream)
{
    clear_error();
    amsim_status s = check_pc(P, C, ws, ws_bytes, "amsim_bias_act_bwd");
    if (s != AMSIM_OK) return s;
    if (P == 0) return AMSIM_OK;
    if (!dy || !dx || !dbias || (relu && !y)) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_bias_act_bwd: null tensor");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t G = reduce_blocks(P);
    double2 *part = static_cast<double2 *>(ws);
    channel_partials<<<int(G), NT, 0, st>>>(P, C, BiasBwdF{dy, y, dx, C, relu}, part);
    bias_bwd_finalize<<<(C + 127) / 128, 128, 0, st>>>(part, G, C, dbias);
    count_launch(2);
    return check_launch("amsim_bias_act_bwd");
}

static amsim_status pool_args(int32_t N, int32_t H, int32_t W, int32_t C, int32_t R, int32_t S, int32_t st,
                              int32_t pad, int &OH, int &OW, const char *fn)
{
    if (N < 0 || H <= 0 || W <= 0 || C <= 0 || R <= 0 || S <= 0 || st <= 0 || pad < 0 || pad >= R || pad >= S ||
        R * S > 255 || H + 2 * pad < R || W + 2 * pad < S)
        return set_error(AMSIM_ERR_INVALID_ARG, std::string(fn) + ": invalid pooling geometry");
    OH = (H + 2 * pad - R) / st + 1;
    OW = (W + 2 * pad - S) / st + 1;
    return AMSIM_OK;
}

amsim_status amsim_maxpool_fwd(const float *x, int32_t N, int32_t H, int32_t W, int32_t C, int32_t R, int32_t S,
                               int32_t stride, int32_t pad, float *y, uint8_t *argmax, amsim_stream_t stream)
{
    clear_error();
    int OH, OW;
    amsim_status s = pool_args(N, H, W, C, R, S, stride, pad, OH, OW, "amsim_maxpool_fwd");
    if (s != AMSIM_OK) return s;
    if (N == 0) return AMSIM_OK;
    if (!x || !y || !argmax) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_maxpool_fwd: null tensor");
    maxpool_fwd_k<<<grid_for(int64_t(N) * OH * OW * C), NT, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        x, N, H, W, C, R, S, stride, pad, OH, OW, y, argmax);
    count_launch();
    return check_launch("amsim_maxpool_fwd");
}

amsim_status amsim_maxpool_bwd(const float *dy, const uint8_t *argmax, int32_t N, int32_t H, int32_t W, int32_t C,
                               int32_t R, int32_t S, int32_t stride, int32_t pad, float *dx, amsim_stream_t stream)
{
    clear_error();
    int OH, OW;
    amsim_status s = pool_args(N, H, W, C, R, S, stride, pad, OH, OW, "amsim_maxpool_bwd");
    if (s != AMSIM_OK) return s;
    if (N == 0) return AMSIM_OK;
    if (!dy || !argmax || !dx) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_maxpool_bwd: null tensor");
    maxpool_bwd_k<<<grid_for(int64_t(N) * H * W * C), NT, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        dy, argmax, N, H, W, C, R, S, stride, pad, OH, OW, dx);
    count_launch();
    return check_launch("amsim_maxpool_bwd");
}

amsim_status amsim_avgpool_fwd(const float *x, int32_t N, int32_t HW, int32_t C, float *y, amsim_stream_t stream)
{
    clear_error();
    if (N < 0 || HW <= 0 || C <= 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_avgpool_fwd: bad sizes");
    if (N == 0) return AMSIM_OK;
    if (!x || !y) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_avgpool_fwd: null tensor");
    avgpool_fwd_k<<<grid_for(int64_t(N) * C), NT, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, N, HW, C, y);
    count_launch();
    return check_launch("amsim_avgpool_fwd");
}

amsim_status amsim_avgpool_bwd(const float *dy, int32_t N, int32_t HW, int32_t C, float *dx, amsim_stream_t stream)
{
    clear_error();
    if (N < 0 || HW <= 0 || C <= 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_avgpool_bwd: bad sizes");
    if (N == 0) return AMSIM_OK;
    if (!dy || !dx) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_avgpool_bwd: null tensor");
    avgpool_bwd_k<<<grid_for(int64_t(N) * HW * C), NT, 0, reinterpret_cast<cudaStream_t>(stream)>>>(dy, N, HW, C, dx);
    count_launch();
    return check_launch("amsim_avgpool_bwd");
}

amsim_status amsim_softmax_xent(const float *logits, const int32_t *labels, int32_t N, int32_t K,
                                int32_t grad_denominator, float *loss, float *dlogits, void *ws, size_t ws_bytes,
                                amsim_stream_t stream)
{
    clear_error();
    if (N <= 0 || K <= 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_softmax_xent: N > 0 and K > 0 required");
    if (grad_denominator < 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_softmax_xent: grad_denominator < 0");
    if (!logits || !labels || !loss || !dlogits) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_softmax_xent: null tensor");
    if (!ws || ws_bytes < ws_need(N, 1))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_softmax_xent: workspace too small");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    float *row_loss = static_cast<float *>(ws);
    softmax_xent_k<<<N, NT, 0, st>>>(logits, labels, N, K, 1.f / float(grad_denominator ? grad_denominator : N),
                                     dlogits, row_loss);
    mean_k<<<1, 32, 0, st>>>(row_loss, N, loss);
    count_launch(2);
    return check_launch("amsim_softmax_xent");
}

amsim_status amsim_add(const float *a, const float *b, float *out, int64_t n, amsim_stream_t stream)
{
    clear_error();
    if (n < 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_add: n < 0");
    if (n == 0) return AMSIM_OK;
    if (!a || !b || !out) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_add: null tensor");
    add_k<<<grid_for(n), NT, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a, b, out, n);
    count_launch();
    return check_launch("amsim_add");
}

amsim_status amsim_sgd_momentum(float *w, const float *g, float *v, int64_t n, float lr, float momentum,
                                float weight_decay, amsim_stream_t stream)
{
    clear_error();
    if (n < 0) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_sgd_momentum: n < 0");
    if (n == 0) return AMSIM_OK;
    if (!w || !g || !v) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_sgd_momentum: null tensor");
    sgd_k<<<grid_for(n), NT, 0, reinterpret_cast<cudaStream_t>(stream)>>>(w, g, v, n, lr, momentum, weight_decay);
    count_launch();
    return check_launch("amsim_sgd_momentum");
}

}  // extern "C"
