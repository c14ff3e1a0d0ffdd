// cbrng_host.cpp — host-side pieces of the C ABI: version, thread-local error
// text, launch-geometry cache, and the byte-serial FNV-1a checksum
// (_kernels.py:89-96), which is sequential by definition and stays on the host.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include <cuda_runtime.h>

#include "cbrng_b200.h"
#include "cbrng_internal.cuh"

namespace cbrng {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

void clear_error() { g_err[0] = 0; }

int tuning_knob(const char *name, int dflt, int lo, int hi) {
#if CBRNG_TUNING
    const char *e = getenv(name);
    const int x = e ? atoi(e) : dflt;
    return (x >= lo && x <= hi) ? x : dflt;
#else
    (void)name; (void)lo; (void)hi;
    return dflt;
#endif
}

int grid_mult() {
    static const int v = tuning_knob("CBRNG_GRID_MULT", 8, 0, 64);
    return v;
}

int resident_blocks(const void *kernel, int block, size_t smem) {
    static std::mutex mu;
    static std::unordered_map<uint64_t, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    uint64_t key = reinterpret_cast<uint64_t>(kernel) ^ ((uint64_t)dev << 56) ^ ((uint64_t)block << 40) ^ smem;
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int sms = 0, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, smem);
    if (occ < 1) occ = 1;
    if (sms < 1) sms = 1;
    int g = sms * occ;
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = g;
    return g;
}

}  // namespace cbrng

extern "C" {

const char *cbrng_version(void) { return "cbrng-b200 0.1.0 (sm_100a)"; }

const char *cbrng_last_error(void) { return cbrng::g_err; }

int cbrng_device_sm_count(int device) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return CBRNG_ECUDA;
    return sms;
}

uint64_t cbrng_fnv1a64(const uint8_t *data, uint64_t n, uint64_t h) {
    for (uint64_t i = 0; i < n; i++) h = (h ^ data[i]) * 0x100000001B3ull;
    return h;
}

}  // extern "C"
