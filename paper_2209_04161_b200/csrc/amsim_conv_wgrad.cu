// libamsim: conv weight gradient, Alg. 4 l.4-5 (C-ABI entry points of include/amsim.h).
// Citations "PAPER.md:L" are lines of /root/reference/PAPER.md.
#include "amsim_dispatch.cuh"

using namespace amsim;
using namespace amsim::dev;

extern "C" {

static amsim_status wgrad_plan(const amsim_lut *lut, const amsim_conv2d_desc *d, KParams &p, ConvGeom &g, int &eb,
                               int mode = -1, int policy = -1)
{
    init_geom(g, d);
    Problem pr;
    pr.a_is_activation = true;
    pr.N = d->K;
    pr.M[0] = d->R * d->S * d->C;
    pr.K[0] = d->N * g.OH * g.OW;
    return prepare(lut, p, pr, eb, mode, policy);
}

amsim_status amsim_conv2d_bwd_filter_workspace(const amsim_lut *lut, const amsim_conv2d_desc *d, size_t *bytes)
{
    clear_error();
    if (!lut || !bytes) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_filter_workspace: null argument");
    amsim_status s = check_desc(d);
    if (s != AMSIM_OK) return s;
    // The plan (hence the workspace) depends on the multiply mode and the
    // table layout policy; report the maximum so one allocation serves all.
    // A variant with no plan (a forced tile configuration that only fits some
    // table layouts, AMSIM_FORCE_CFG) is skipped; an error only if none plans.
    int64_t need = 0;
    bool any = false;
    amsim_status last = AMSIM_OK;
    const int pol = path_policy() & 3;   // bits 2 (table layout) and 4 (orientation) are varied below
    for (int mode : {AMSIM_MUL_LUT, AMSIM_MUL_NATIVE})
        for (int policy : {pol, pol | 4, pol | 16, pol | 4 | 16}) {
            KParams p{};
            ConvGeom g;
            int eb;
            s = wgrad_plan(lut, d, p, g, eb, mode, policy);
            if (s != AMSIM_OK) {
                last = s;
                continue;
            }
            any = true;
            need = std::max<int64_t>(need, p.ws_elems);
        }
    if (!any) return last;
    clear_error();
    *bytes = size_t(need) * sizeof(float);
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
    int eb;
    s = wgrad_plan(lut, d, p, g, eb);
    if (s != AMSIM_OK) return s;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    // original problem dims (the plan's sub-problem / N are transposed when the
    // planner picked the transposed orientation)
    const int Mo = d->R * d->S * d->C, No = d->K, Ko = d->N * g.OH * g.OW;
    if (Ko == 0) {
        fill_zero_kernel<<<64, 256, 0, st>>>(dw, Mo, No, No);
        count_launch();
        return cuda_check(cudaGetLastError(), "fill_zero launch");
    }
    size_t need = size_t(p.ws_elems) * sizeof(float);
    if (need > 0 && (!workspace || workspace_bytes < need))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_conv2d_bwd_filter: workspace too small (need " +
                                                    std::to_string(need) + " bytes)");
    WgX a{x, g, Mo, Ko};
    GemmOp b{dy, d->K, No, Ko, 0};
    p.da = OpDesc{0, (d->C % 4 == 0 && aligned16(x)) ? 2 : 0};
    p.db = OpDesc{0, (d->K % 4 == 0 && aligned16(dy)) ? 2 : 0};
    p.C = dw;
    p.ldc = No;
    p.accumulate = 0;
    return run(eb, p, a, b, st, static_cast<float *>(workspace));
}

}  // extern "C"
