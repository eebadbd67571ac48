// Internal declarations shared by the host side (amsim_host.cpp) and the
// kernel side (amsim_dispatch.cuh and the amsim_*.cu entry points) of libamsim.  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/amsim.h"

namespace amsim {

constexpr int kMaxDevices = 64;

// Device copy of a table in the kernels' layout: row k (first operand) is
// 2^m consecutive entries; 8-bit entries hold bits 23..16 of the Alg. 1 entry
// (carry | top 7 mantissa bits) when every entry's low 16 bits are zero,
// 16-bit entries bits 23..8 when every entry's low 8 bits are zero.
struct DeviceTable {
    void *ptr = nullptr;
    size_t bytes = 0;
};

}  // namespace amsim

struct amsim_lut {
    int m = 0;
    std::vector<uint32_t> entries;   // Alg. 1 layout: (carry << 23) | mantissa
    bool symmetric = false;          // entries[k][j] == entries[j][k] for all k, j
    int e_bits = 8;                  // operand exponent casting (1, e, m), reading C23
    int model_id = -1;               // built-in model the table was built from (0 exact, 1 Mitchell, 2 MBM), else -1
    int device_entry_bits = 32;      // 8 if every (e & 0xFFFF) == 0, else 16 if every (e & 0xFF) == 0
    std::mutex mu;
    amsim::DeviceTable dev[amsim::kMaxDevices];        // narrowest layout
    amsim::DeviceTable dev_wide[amsim::kMaxDevices];   // 32-bit layout (policy bit 2, tests)
};

namespace amsim {

amsim_status set_error(amsim_status s, const std::string &msg);
void clear_error();

// Device table for the current device (uploads on first use).
// policy < 0: the process-wide path policy (bit 2 selects the 32-bit layout).
amsim_status device_table(const amsim_lut *lut, const void **ptr, int *entry_bits, int policy = -1);

// Global launch counter (incremented by every kernel launch).
void count_launch(uint64_t n = 1);

int path_policy();
int multiply_mode();

// Stream-ordered scratch (split-K partials, small coefficient buffers) from the
// library's own per-device memory pool, which keeps freed memory (release
// threshold = max) so steady-state calls never return to the OS allocator and
// the host application's default pool is untouched.  Capturable in CUDA graphs.
amsim_status scratch_alloc(void **ptr, size_t bytes, cudaStream_t stream);
void scratch_free(void *ptr, cudaStream_t stream);

}  // namespace amsim
