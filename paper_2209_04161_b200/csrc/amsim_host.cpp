// libamsim host side: error state, built-in multiplier models, LUT build
// (Alg. 1), LUT file I/O and the per-device table upload.
// Citations "PAPER.md:L" are lines of /root/reference/PAPER.md.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "amsim_internal.h"

namespace amsim {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};
// path policy and multiply mode are per calling thread: a test hook on one
// thread never changes the arithmetic of another thread's calls
static thread_local int g_policy = 0;
static thread_local int g_mul_mode = 0;

amsim_status set_error(amsim_status s, const std::string &msg)
{
    g_last_error = msg;
    return s;
}

void clear_error() { g_last_error.clear(); }

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int path_policy() { return g_policy; }

int multiply_mode() { return g_mul_mode; }

static inline uint32_t bits(float f)
{
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}
static inline float flt(uint32_t u)
{
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// Compose sign | E << 23 | mant with FP32 range handling (E is the biased
// exponent of a significand in [1, 2)).
static inline float compose(uint32_t sign, int E, uint32_t mant)
{
    if (E >= 255) return flt(sign | 0x7F800000u);
    if (E <= 0) return flt(sign);  // models are only meaningful on normal products
    return flt(sign | (uint32_t(E) << 23) | (mant & 0x7FFFFFu));
}

static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[kMaxDevices];

amsim_status scratch_alloc(void **ptr, size_t bytes, cudaStream_t stream)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
        return set_error(AMSIM_ERR_UNSUPPORTED, "no CUDA device");
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> g(g_pool_mu);
        if (!g_pools[dev]) {
            cudaMemPoolProps props = {};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            if (cudaMemPoolCreate(&g_pools[dev], &props) != cudaSuccess)
                return set_error(AMSIM_ERR_NOMEM, "cudaMemPoolCreate failed");
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(g_pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = g_pools[dev];
    }
    cudaError_t e = cudaMallocFromPoolAsync(ptr, bytes, pool, stream);
    if (e != cudaSuccess) return set_error(AMSIM_ERR_NOMEM, std::string("scratch allocation: ") + cudaGetErrorString(e));
    return AMSIM_OK;
}

void scratch_free(void *ptr, cudaStream_t stream)
{
    if (ptr) cudaFreeAsync(ptr, stream);
}

// Upload the table for the current device in layout `eb` (8, 16 or 32 bits).
static amsim_status upload(amsim_lut *lut, int dev, int eb, DeviceTable &t)
{
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return set_error(AMSIM_ERR_UNSUPPORTED, "libamsim is built for sm_100a (B200) only; device is sm_" +
                                                    std::to_string(major) + std::to_string(minor));
    size_t n = lut->entries.size();
    size_t bytes = n * (eb / 8);
    std::vector<uint8_t> host(bytes);
    if (eb == 8) {
        for (size_t i = 0; i < n; i++) host[i] = uint8_t(lut->entries[i] >> 16);
    } else if (eb == 16) {
        uint16_t *h16 = reinterpret_cast<uint16_t *>(host.data());
        for (size_t i = 0; i < n; i++) h16[i] = uint16_t(lut->entries[i] >> 8);
    } else {
        std::memcpy(host.data(), lut->entries.data(), bytes);
    }
    // The first call on a device may come inside a CUDA graph capture: allocate
    // and copy in relaxed capture mode on a private non-blocking stream (never
    // the legacy stream, which would join the capture), so the upload is an
    // ordinary synchronous host operation that the captured graph does not see.
    cudaStreamCaptureMode cm = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&cm);
    void *p = nullptr;
    cudaStream_t us = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&us, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p, host.data(), bytes, cudaMemcpyHostToDevice, us);
    if (e == cudaSuccess) e = cudaStreamSynchronize(us);
    if (us) cudaStreamDestroy(us);
    cudaThreadExchangeStreamCaptureMode(&cm);
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        return set_error(AMSIM_ERR_CUDA, std::string("LUT upload: ") + cudaGetErrorString(e));
    }
    t.ptr = p;
    t.bytes = bytes;
    return AMSIM_OK;
}

amsim_status device_table(const amsim_lut *lut_c, const void **ptr, int *entry_bits, int policy)
{
    amsim_lut *lut = const_cast<amsim_lut *>(lut_c);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_error(AMSIM_ERR_UNSUPPORTED, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (dev < 0 || dev >= kMaxDevices) return set_error(AMSIM_ERR_UNSUPPORTED, "device index out of range");
    // policy bit 2: the 32-bit layout whatever the table's width (tests prove the width never changes bits)
    const bool wide = ((policy < 0 ? path_policy() : policy) & 4) != 0 && lut->device_entry_bits != 32;
    int eb = wide ? 32 : lut->device_entry_bits;
    std::lock_guard<std::mutex> g(lut->mu);
    DeviceTable &t = wide ? lut->dev_wide[dev] : lut->dev[dev];
    if (!t.ptr) {
        amsim_status s = upload(lut, dev, eb, t);
        if (s != AMSIM_OK) return s;
    }
    *ptr = t.ptr;
    *entry_bits = eb;
    return AMSIM_OK;
}

static void finalize_lut(amsim_lut *lut)
{
    // Narrowest device layout that holds every entry exactly: 8 bits (carry |
    // 7 mantissa bits, e.g. Mitchell at m <= 7), 16 bits (carry | 15), else 32.
    uint32_t low = 0;
    for (uint32_t e : lut->entries) low |= e;
    // Every table that fits 8 bits gets the 8-bit layout.  (Round 1 kept 16-bit
    // entries up to m = 6, where a 2^m-entry 16-bit row still fits one 128-byte
    // wavefront and LDS.U16 + packed operands measured 5.7 % faster; with the
    // round-2 quad decode and 16 x 8 tiles for 8-bit tables the 8-bit layout is
    // 19 % faster there: 4096^3 Mitchell m = 4..6, 4.92 -> 5.85 T/s,
    // profiles/r02b_ab_min_m8.jsonl.)
    const bool fits8 = (low & 0xFFFFu) == 0, fits16 = (low & 0xFFu) == 0;
    int min_m8 = 1;   // AMSIM_MIN_M8: tuning experiments only
    if (const char *f = std::getenv("AMSIM_MIN_M8"); f && *f) min_m8 = std::atoi(f);
    lut->device_entry_bits = (fits8 && lut->m >= min_m8) ? 8 : (fits16 ? 16 : 32);
    // symmetric tables (model(a, b) == model(b, a) on every probe pair) may be used
    // transposed, which the skinny-N kernel orientation needs
    const size_t n = size_t(1) << lut->m;
    lut->symmetric = true;
    for (size_t k = 0; k < n && lut->symmetric; k++)
        for (size_t j = k + 1; j < n; j++)
            if (lut->entries[k * n + j] != lut->entries[j * n + k]) {
                lut->symmetric = false;
                break;
            }
}

}  // namespace amsim

using namespace amsim;

extern "C" {

const char *amsim_last_error(void) { return g_last_error.c_str(); }

int amsim_abi_version(void) { return AMSIM_ABI_VERSION; }

uint64_t amsim_launch_count(void) { return g_launches.load(); }

amsim_status amsim_set_path_policy(int policy)
{
    if (policy < 0 || policy > 63) return set_error(AMSIM_ERR_INVALID_ARG, "policy must be in [0, 63]");
    g_policy = policy;
    return AMSIM_OK;
}

amsim_status amsim_set_multiply_mode(int mode)
{
    if (mode < AMSIM_MUL_LUT || mode > AMSIM_MUL_DIRECT)
        return set_error(AMSIM_ERR_INVALID_ARG, "multiply mode must be AMSIM_MUL_LUT, _NATIVE or _DIRECT");
    g_mul_mode = mode;
    return AMSIM_OK;
}

// ---------------------------------------------------------------------------
// Built-in functional models (integer fixed point on the 23-bit fraction).

// Exact multiplier: IEEE FP32 product (exact for operands truncated to
// m <= 11 bits; bfloat16 by truncation at m = 7).
float amsim_model_exact(float a, float b) { return a * b; }

// Mitchell (MIT16): log2(1+f) ~ f.  With 23-bit fractions fa,
// fb the log-domain sum fa + fb either stays below 2^23 (significand
// 1 + fa + fb) or carries (significand 1 + (fa + fb - 2^23), exponent + 1).
float amsim_model_mitchell(float a, float b)
{
    uint32_t ua = bits(a), ub = bits(b);
    uint32_t sign = (ua ^ ub) & 0x80000000u;
    int ea = int((ua >> 23) & 0xFF), eb = int((ub >> 23) & 0xFF);
    uint32_t s = (ua & 0x7FFFFFu) + (ub & 0x7FFFFFu);
    int carry = int(s >> 23);
    return compose(sign, ea + eb - 127 + carry, s & 0x7FFFFFu);
}

// MBM / AFM16 stand-in (PAPER.md:782-785 cites Saadat et al. 2018 without
// defining it; fidelity unpinned): Mitchell plus a constant
// bias compensation, 5/64 on the un-carried significand and 5/128 on the
// carried one, the latter saturating below 2 so the carry stays <= 1.
float amsim_model_mbm(float a, float b)
{
    uint32_t ua = bits(a), ub = bits(b);
    uint32_t sign = (ua ^ ub) & 0x80000000u;
    int ea = int((ua >> 23) & 0xFF), eb = int((ub >> 23) & 0xFF);
    uint32_t s = (ua & 0x7FFFFFu) + (ub & 0x7FFFFFu);   // fa + fb in units of 2^-23
    const uint32_t one = 1u << 23;
    if (s < one) {
        uint32_t sig = one + s + (5u << 17);            // 1 + fa + fb + 5/64
        int E = ea + eb - 127;
        if (sig >= 2 * one) {                           // renormalise: halve, round to nearest even
            uint32_t h = sig >> 1;
            if ((sig & 1u) && (h & 1u)) h += 1;
            sig = h;
            E += 1;
        }
        return compose(sign, E, sig - one);
    }
    uint32_t sig = s + (5u << 16);                      // (fa + fb) + 5/128, already in [1, 2)
    const uint32_t sat = 2 * one - (1u << 8);           // 2 - 2^-15
    if (sig > sat) sig = sat;
    return compose(sign, ea + eb - 127 + 1, sig - one);
}

// ---------------------------------------------------------------------------
// Alg. 1

amsim_status amsim_lut_build(amsim_mul_fn model, int m, amsim_lut **out)
{
    clear_error();
    if (!model || !out) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_build: null argument");
    if (m < 1 || m > 11) return set_error(AMSIM_ERR_UNSUPPORTED, "amsim_lut_build: m must be in [1, 11] (PAPER.md:302)");
    amsim_lut *lut = new (std::nothrow) amsim_lut;
    if (!lut) return set_error(AMSIM_ERR_NOMEM, "amsim_lut_build: out of host memory");
    lut->m = m;
    lut->model_id = model == amsim_model_exact ? 0 : model == amsim_model_mitchell ? 1 : model == amsim_model_mbm ? 2 : -1;
    const uint32_t n = 1u << m;
    try {
        lut->entries.resize(size_t(n) * n);
    } catch (...) {
        delete lut;
        return set_error(AMSIM_ERR_NOMEM, "amsim_lut_build: out of host memory");
    }
    // Alg. 1 l.2-4: sign +, exponent field 127 for both probes, so the
    // un-normalised exponent is 127 and the product's exponent must be 127 or
    // 128 (reading C9).
    const int un_normalized_exp = 127 + 127 - 127;
    for (uint32_t k = 0; k < n; k++) {
        for (uint32_t j = 0; j < n; j++) {
            float A = flt((127u << 23) | (k << (23 - m)));   // Mantissa(A) <- k (top m bits)
            float B = flt((127u << 23) | (j << (23 - m)));
            uint32_t C = bits(model(A, B));
            int ec = int((C >> 23) & 0xFF);
            if ((C >> 31) || (ec != un_normalized_exp && ec != un_normalized_exp + 1)) {
                char msg[160];
                std::snprintf(msg, sizeof msg,
                              "model: product of probes (k=%u, j=%u) has sign %u exponent %d; Alg. 1 needs a positive "
                              "product with exponent %d or %d",
                              k, j, C >> 31, ec, un_normalized_exp, un_normalized_exp + 1);
                delete lut;
                return set_error(AMSIM_ERR_MODEL, msg);
            }
            uint32_t carry = ec > un_normalized_exp ? 1u : 0u;            // l.11-13
            lut->entries[size_t(k) * n + j] = (carry << 23) | (C & 0x7FFFFFu);  // l.14
        }
    }
    finalize_lut(lut);
    *out = lut;
    return AMSIM_OK;
}

amsim_status amsim_lut_from_entries(const uint32_t *entries, int m, amsim_lut **out)
{
    clear_error();
    if (!entries || !out) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_from_entries: null argument");
    if (m < 1 || m > 11) return set_error(AMSIM_ERR_UNSUPPORTED, "amsim_lut_from_entries: m must be in [1, 11]");
    size_t n = size_t(1) << (2 * m);
    for (size_t i = 0; i < n; i++)
        if (entries[i] >> 24) {
            char msg[96];
            std::snprintf(msg, sizeof msg, "amsim_lut_from_entries: entry %zu has bits 31..24 set", i);
            return set_error(AMSIM_ERR_INVALID_ARG, msg);
        }
    amsim_lut *lut = new (std::nothrow) amsim_lut;
    if (!lut) return set_error(AMSIM_ERR_NOMEM, "out of host memory");
    lut->m = m;
    lut->entries.assign(entries, entries + n);
    finalize_lut(lut);
    *out = lut;
    return AMSIM_OK;
}

amsim_status amsim_lut_entries(const amsim_lut *lut, const uint32_t **entries, size_t *count)
{
    if (!lut || !entries || !count) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_entries: null argument");
    *entries = lut->entries.data();
    *count = lut->entries.size();
    return AMSIM_OK;
}

amsim_status amsim_lut_info(const amsim_lut *lut, int *m_bits, int *device_entry_bits)
{
    if (!lut) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_info: null lut");
    if (m_bits) *m_bits = lut->m;
    if (device_entry_bits) *device_entry_bits = lut->device_entry_bits;
    return AMSIM_OK;
}

amsim_status amsim_lut_save(const amsim_lut *lut, const char *path)
{
    if (!lut || !path) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_save: null argument");
    FILE *f = std::fopen(path, "wb");
    if (!f) return set_error(AMSIM_ERR_IO, std::string("amsim_lut_save: cannot open ") + path);
    uint8_t hdr[8] = {'A', 'M', 'L', 'T', 1, uint8_t(lut->m), 0, 0};
    bool ok = std::fwrite(hdr, 1, 8, f) == 8;
    for (size_t i = 0; ok && i < lut->entries.size(); i++) {
        uint32_t e = lut->entries[i];
        uint8_t le[4] = {uint8_t(e), uint8_t(e >> 8), uint8_t(e >> 16), uint8_t(e >> 24)};
        ok = std::fwrite(le, 1, 4, f) == 4;
    }
    ok = (std::fclose(f) == 0) && ok;
    return ok ? AMSIM_OK : set_error(AMSIM_ERR_IO, std::string("amsim_lut_save: write failed for ") + path);
}

amsim_status amsim_lut_load(const char *path, amsim_lut **out)
{
    clear_error();
    if (!path || !out) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_load: null argument");
    FILE *f = std::fopen(path, "rb");
    if (!f) return set_error(AMSIM_ERR_IO, std::string("amsim_lut_load: cannot open ") + path);
    uint8_t hdr[8];
    if (std::fread(hdr, 1, 8, f) != 8) {
        std::fclose(f);
        return set_error(AMSIM_ERR_IO, "amsim_lut_load: truncated header");
    }
    if (std::memcmp(hdr, "AMLT", 4) != 0) {
        std::fclose(f);
        return set_error(AMSIM_ERR_IO, "amsim_lut_load: bad magic (expected AMLT)");
    }
    if (hdr[4] != 1) {
        std::fclose(f);
        return set_error(AMSIM_ERR_IO, "amsim_lut_load: unsupported format version");
    }
    int m = hdr[5];
    if (m < 1 || m > 11 || hdr[6] || hdr[7]) {
        std::fclose(f);
        return set_error(AMSIM_ERR_IO, "amsim_lut_load: mantissa bits out of range [1, 11] or reserved bytes set");
    }
    size_t n = size_t(1) << (2 * m);
    std::vector<uint32_t> e(n);
    for (size_t i = 0; i < n; i++) {
        uint8_t le[4];
        if (std::fread(le, 1, 4, f) != 4) {
            std::fclose(f);
            return set_error(AMSIM_ERR_IO, "amsim_lut_load: truncated payload");
        }
        e[i] = uint32_t(le[0]) | uint32_t(le[1]) << 8 | uint32_t(le[2]) << 16 | uint32_t(le[3]) << 24;
    }
    uint8_t extra;
    bool trailing = std::fread(&extra, 1, 1, f) == 1;
    std::fclose(f);
    if (trailing) return set_error(AMSIM_ERR_IO, "amsim_lut_load: trailing bytes after payload");
    amsim_status s = amsim_lut_from_entries(e.data(), m, out);
    if (s != AMSIM_OK) return set_error(AMSIM_ERR_IO, std::string("amsim_lut_load: ") + amsim_last_error());
    return AMSIM_OK;
}

amsim_status amsim_lut_with_exponent_bits(const amsim_lut *src, int e_bits, amsim_lut **out)
{
    clear_error();
    if (!src || !out) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_with_exponent_bits: null argument");
    if (e_bits < 1 || e_bits > 8)
        return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_with_exponent_bits: e must be in [1, 8] (PAPER.md:392)");
    amsim_lut *lut = new (std::nothrow) amsim_lut;
    if (!lut) return set_error(AMSIM_ERR_NOMEM, "out of host memory");
    lut->m = src->m;
    lut->entries = src->entries;
    lut->device_entry_bits = src->device_entry_bits;
    lut->model_id = src->model_id;
    lut->symmetric = src->symmetric;
    lut->e_bits = e_bits;
    *out = lut;
    return AMSIM_OK;
}

amsim_status amsim_lut_exponent_bits(const amsim_lut *lut, int *e_bits)
{
    if (!lut || !e_bits) return set_error(AMSIM_ERR_INVALID_ARG, "amsim_lut_exponent_bits: null argument");
    *e_bits = lut->e_bits;
    return AMSIM_OK;
}

void amsim_lut_destroy(amsim_lut *lut)
{
    if (!lut) return;
    int cur = -1;
    cudaGetDevice(&cur);
    for (int d = 0; d < kMaxDevices; d++) {
        for (amsim::DeviceTable *t : {&lut->dev[d], &lut->dev_wide[d]}) {
            if (t->ptr) {
                cudaSetDevice(d);
                cudaFree(t->ptr);
            }
        }
    }
    if (cur >= 0) cudaSetDevice(cur);
    delete lut;
}

}  // extern "C"
