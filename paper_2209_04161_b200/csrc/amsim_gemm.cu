// libamsim: dense GEMM (C-ABI entry points of include/amsim.h).
// Citations "PAPER.md:L" are lines of /root/reference/PAPER.md.
#include "amsim_dispatch.cuh"

using namespace amsim;
using namespace amsim::dev;

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
        fill_zero_kernel<<<std::max(1, int(std::min<int64_t>((M * N + 255) / 256, 1024))), 256, 0, st>>>(C, int(M),
                                                                                                         int(N), ldc);
        count_launch();
        return cuda_check(cudaGetLastError(), "fill_zero launch");
    }
    if (!A || !B) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: null operand");
    if ((!trans_a && lda < K) || (trans_a && lda < M))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: lda too small");
    if ((!trans_b && ldb < N) || (trans_b && ldb < K))
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_gemm: ldb too small");
    Problem pr;
    pr.N = int(N);
    pr.M[0] = int(M);
    pr.K[0] = int(K);
    // TMA boxes for both operands, A k-contiguous (setup_tma)
    pr.tma_lanes = !trans_a && aligned16(A) && aligned16(B) && lda % 4 == 0 && ldb % 4 == 0;
    KParams p{};
    int eb = 32;
    amsim_status s = prepare(lut, p, pr, eb);
    if (s != AMSIM_OK) return s;
    GemmOp a{A, lda, int(M), int(K), trans_a ? 0 : 1};
    GemmOp b{B, ldb, int(N), int(K), trans_b ? 1 : 0};
    // 16-byte copies need 4 contiguous elements with 16-B aligned rows
    bool va = aligned16(A) && lda % 4 == 0 && (trans_a ? M % 4 == 0 : K % 4 == 0);
    bool vb = aligned16(B) && ldb % 4 == 0 && (trans_b ? K % 4 == 0 : N % 4 == 0);
    p.da = OpDesc{a.kcontig, va ? 2 : 0};
    p.db = OpDesc{b.kcontig, vb ? 2 : 0};
    p.C = C;
    p.ldc = ldc;
    p.accumulate = accumulate;
    return run(eb, p, a, b, st);
}

}  // extern "C"
