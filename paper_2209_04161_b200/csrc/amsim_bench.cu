// libamsim: LUT-lookup microbenchmark (roofline instrument) (C-ABI entry points of include/amsim.h).
// Citations "PAPER.md:L" are lines of /root/reference/PAPER.md.
#include "amsim_dispatch.cuh"

using namespace amsim;
using namespace amsim::dev;

extern "C" {

amsim_status amsim_bench_lut_lookup(int m_bits, int entry_bits, int iters, const uint32_t *b_idx_host, size_t n_idx,
                                    double *lookups_per_s, amsim_stream_t stream)
{
    clear_error();
    if (m_bits < 1 || m_bits > 8 || (entry_bits != 8 && entry_bits != 16 && entry_bits != 32) || iters <= 0 ||
        !b_idx_host || !n_idx ||
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
        if ((s = cuda_check(cudaMemcpyAsync(idx, b_idx_host, n_idx * 4, cudaMemcpyHostToDevice, st), "memcpy")) !=
            AMSIM_OK)
            break;
        if ((s = cuda_check(cudaMalloc(&out, size_t(sms) * BENCH_NT * 4), "cudaMalloc")) != AMSIM_OK) break;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto launch = [&]() {
            if (entry_bits == 8) {
                cudaFuncSetAttribute(lut_bench_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
                lut_bench_kernel<8><<<sms, BENCH_NT, bytes, st>>>(tab, bytes, m_bits, idx, int(n_idx), iters, out);
            } else if (entry_bits == 16) {
                cudaFuncSetAttribute(lut_bench_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
                lut_bench_kernel<16><<<sms, BENCH_NT, bytes, st>>>(tab, bytes, m_bits, idx, int(n_idx), iters, out);
            } else {
                cudaFuncSetAttribute(lut_bench_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
                lut_bench_kernel<32><<<sms, BENCH_NT, bytes, st>>>(tab, bytes, m_bits, idx, int(n_idx), iters, out);
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
        double lookups = double(sms) * BENCH_NT * iters * BENCH_TM * 4;
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
