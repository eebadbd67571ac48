// libamsim: conv preceding-layer gradient, Alg. 4 l.6-8 (C-ABI entry points of include/amsim.h).
// Citations "PAPER.md:L" are lines of /root/reference/PAPER.md.
#include "amsim_dispatch.cuh"

using namespace amsim;
using namespace amsim::dev;

extern "C" {

amsim_status amsim_conv2d_bwd_data(const amsim_lut *lut, const amsim_conv2d_desc *d, const float *dy,
                                   const float *w, float *dx, amsim_stream_t stream)
{
    clear_error();
    if (!lut) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_data: null lut");
    amsim_status s = check_desc(d);
    if (s != AMSIM_OK) return s;
    if (d->N == 0) return AMSIM_OK;
    if (!dy || !w || !dx) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_data: null tensor");
    DgDY a{};
    DgW b{};
    init_geom(a.g, d);
    Problem pr;
    dgrad_phases(d, pr, a.ph);
    // TMA boxes for both operands (setup_tma): dy as [pixels][K] (1x1 unpadded),
    // im2col boxes (stride 1) or per-phase im2col boxes (stride 2); w taps as 3-D boxes
    const bool one = d->R == 1 && d->S == 1 && d->pad_h == 0 && d->pad_w == 0;
    const bool s1 = d->stride_h == 1 && d->stride_w == 1;
    pr.tma_lanes = aligned16(dy) && aligned16(w) && d->K % BK == 0 &&
                   (one || s1 || (pr.nsub <= MAX_PH_TMA && !(path_policy() & 32)));
    a.dy = dy;
    a.fK.init(uint32_t(d->K));
    b.w = w;
    b.g = a.g;
    b.fK = a.fK;
    std::memcpy(b.ph, a.ph, sizeof(a.ph));
    KParams p{};
    int eb = 32;
    s = prepare(lut, p, pr, eb);
    if (s != AMSIM_OK) return s;
    if (d->stride_h > 1 || d->stride_w > 1) {   // per-phase im2col TMA descriptors for the dy tiles
        int BM, BN, NT;
        size_t smem;
        cfg_shape(CfgId(p.cfg), BM, BN, NT, smem, 0);
        a.ph_tma = encode_dgrad_phases(a, pr.nsub, std::min(p.trn ? BN : BM, 256)) ? 1 : 0;
    }
    bool v = d->K % 4 == 0;
    p.da = OpDesc{1, (v && aligned16(dy)) ? 2 : 0};
    p.db = OpDesc{1, (v && aligned16(w)) ? 2 : 0};
    p.C = dx;
    p.ldc = d->C;
    p.accumulate = 0;
    return run(eb, p, a, b, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
