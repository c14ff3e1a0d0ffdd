// cbrng_host.cpp — host-side pieces of the C ABI: version, thread-local error
// text, launch-geometry cache, the byte-serial FNV-1a checksum
// (_kernels.py:89-96), which is sequential by definition and stays on the host,
// and the low-latency scalar transport (cbrng_scalar).
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

// Scalar transport (cbrng_scalar): per device, one mapped pinned host buffer
// (outputs at SCALAR_OUT_OFF) and one non-blocking stream. The block functions
// take their arguments by value (scalar_kernel) and every kernel writes its
// output straight through the mapping, so a call is one launch and one stream
// synchronisation, with nothing read over PCIe.
constexpr size_t SCALAR_OUT_OFF = 4096, SCALAR_OUT_WORDS = 1u << 18;
struct ScalarCtx {
    std::mutex mu;
    uint8_t *host = nullptr;
    uint8_t *dev = nullptr;
    cudaStream_t st = nullptr;
};

static ScalarCtx *scalar_ctx(int &rc) {
    static std::mutex mu;
    static ScalarCtx *ctx[64] = {};
    int d = 0;
    rc = check_cuda(cudaGetDevice(&d), "cudaGetDevice");
    if (rc) return nullptr;
    if (d < 0 || d >= 64) {
        set_error("device %d out of range", d);
        rc = CBRNG_EINVAL;
        return nullptr;
    }
    std::lock_guard<std::mutex> g(mu);
    if (!ctx[d]) {
        auto *c = new ScalarCtx;
        void *h = nullptr, *dp = nullptr;
        rc = check_cuda(cudaHostAlloc(&h, SCALAR_OUT_OFF + 4 * SCALAR_OUT_WORDS, cudaHostAllocMapped | cudaHostAllocPortable),
                        "cudaHostAlloc (scalar buffer)");
        if (!rc) rc = check_cuda(cudaHostGetDevicePointer(&dp, h, 0), "cudaHostGetDevicePointer");
        if (!rc) rc = check_cuda(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking), "cudaStreamCreate");
        if (rc) {
            if (h) cudaFreeHost(h);
            delete c;
            return nullptr;
        }
        c->host = static_cast<uint8_t *>(h);
        c->dev = static_cast<uint8_t *>(dp);
        ctx[d] = c;
    }
    return ctx[d];
}

}  // namespace cbrng

extern "C" {

int cbrng_scalar(int op, const uint64_t *args, uint32_t nargs, uint32_t *out, uint64_t nout) {
    using namespace cbrng;
    clear_error();
    static const uint32_t NARGS[9] = {6, 9, 1, 2, 2, 5, 4, 4, 2};
    static const uint64_t NOUT[6] = {4, 4, 2, 1, 4, 4};
    if (op < 0 || op > 8) {
        set_error("unknown scalar op %d", op);
        return CBRNG_EINVAL;
    }
    if (nargs != NARGS[op] || (nargs && !args) || (nout && !out)) {
        set_error("scalar op %d: expects %u args and an output buffer", op, NARGS[op]);
        return CBRNG_EINVAL;
    }
    const uint64_t min_out = op == 7 ? 4 : (op == 8 ? 8 : 0);
    if (op < 6 ? nout != NOUT[op] : (nout < min_out || nout > SCALAR_OUT_WORDS)) {
        set_error("scalar op %d: bad output length %llu", op, (unsigned long long)nout);
        return CBRNG_EINVAL;
    }
    int rc = 0;
    ScalarCtx *c = scalar_ctx(rc);
    if (!c) return rc;
    std::lock_guard<std::mutex> g(c->mu);
    uint32_t *hout = reinterpret_cast<uint32_t *>(c->host + SCALAR_OUT_OFF);
    uint32_t *dout = reinterpret_cast<uint32_t *>(c->dev + SCALAR_OUT_OFF);
    void *st = c->st;
    switch (op) {
        case CBRNG_SCALAR_PHILOX_BLOCK:    // ctr[4], key[2]
        case CBRNG_SCALAR_THREEFRY_BLOCK:  // ctr[4], key[4], rounds
        case CBRNG_SCALAR_SQUARES_KEY:     // seed -> key (lo, hi)
        case CBRNG_SCALAR_SQUARES_ROUND:   // key, ctr
        case CBRNG_SCALAR_TYCHE_INIT:      // seed, stream counter -> state[4]
        case CBRNG_SCALAR_TYCHE_MIX:       // state[4], rounds -> state[4]
            if (op == CBRNG_SCALAR_THREEFRY_BLOCK && args[8] > (1u << 20)) {  // < 0 or absurd: one thread would spin
                set_error("rounds must be in [0, 2^20]");
                return CBRNG_EINVAL;
            }
            rc = launch_scalar(op, args, nargs, dout, c->st);
            break;
        case CBRNG_SCALAR_STREAM_WORDS:  // alg, seed, stream counter, word position -> nout words
            if (args[0] > 2) {
                set_error("scalar stream words: counter-based generators only (alg %llu)", (unsigned long long)args[0]);
                return CBRNG_EALG;
            }
            rc = nout ? cbrng_words((int)args[0], args[1], (uint32_t)args[2], args[3], nullptr, nout, dout, nullptr, st)
                      : CBRNG_OK;
            break;
        case CBRNG_SCALAR_TYCHE_SEED_WORDS:  // seed, stream counter -> init state, nout - 8 words, final state
            rc = launch_tyche_seed_words(args[0], (uint32_t)args[1], nout - 8, dout, c->st);
            break;
        default: {  // CBRNG_SCALAR_TYCHE_WORDS: state[4] -> nout - 4 words, then the state after them
            uint32_t s4[4];
            for (int i = 0; i < 4; i++) s4[i] = (uint32_t)args[i];
            const uint64_t n = nout - 4;
            if (n) {
                rc = cbrng_words(3, 0, 0, 0, s4, n, dout, dout + ((n + 3) & ~3ull), st);
            } else {
                for (int i = 0; i < 4; i++) hout[i] = s4[i];
            }
            break;
        }
    }
    if (rc) return rc;
    rc = check_cuda(cudaStreamSynchronize(c->st), "scalar call");
    if (rc) return rc;
    if (op == CBRNG_SCALAR_TYCHE_WORDS && nout > 4) {
        const uint64_t n = nout - 4;
        std::memcpy(out, hout, 4 * n);
        std::memcpy(out + n, hout + ((n + 3) & ~3ull), 16);
    } else {
        std::memcpy(out, hout, 4 * nout);
    }
    return CBRNG_OK;
}


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
