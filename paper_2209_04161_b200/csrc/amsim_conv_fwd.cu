// libamsim: conv forward, Alg. 3 (C-ABI entry points of include/amsim.h).
// Citations "PAPER.md:L" are lines of /root/reference/PAPER.md.
#include "amsim_dispatch.cuh"

using namespace amsim;
using namespace amsim::dev;

extern "C" {

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
    Problem pr;
    pr.a_is_activation = true;
    pr.N = d->K;
    pr.M[0] = d->N * g.OH * g.OW;
    pr.K[0] = d->R * d->S * d->C;
    // TMA boxes for both operands (setup_tma): x as [pixels][C] (1x1 / stride 1 /
    // unpadded) or im2col boxes of 16 channels, w as [k][Cout]
    pr.tma_lanes = aligned16(x) && aligned16(w) && d->K % 4 == 0 && (is_1x1_s1(g) ? d->C % 4 == 0 : d->C % BK == 0);
    KParams p{};
    int eb = 32;
    s = prepare(lut, p, pr, eb);
    if (s != AMSIM_OK) return s;
    FwdX a{x, g, pr.M[0], pr.K[0]};
    GemmOp b{w, pr.N, pr.N, pr.K[0], 0};
    p.da = OpDesc{1, (d->C % 4 == 0 && aligned16(x)) ? 2 : 0};
    p.db = OpDesc{0, (pr.N % 4 == 0 && aligned16(w)) ? 2 : 0};
    p.C = y;
    p.ldc = pr.N;
    p.accumulate = 0;
    return run(eb, p, a, b, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
