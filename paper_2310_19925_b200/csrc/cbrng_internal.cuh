// cbrng_internal.cuh — host-side plumbing shared by the C-ABI translation units:
// error reporting, launch geometry (grid = SMs x resident CTAs), stream casts.
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "cbrng_b200.h"
#include "cbrng_cores.cuh"

// Tuning builds. The product library (libcbrng_b200.so) is built with
// CBRNG_TUNING=0: every launch parameter is the compile-time default measured
// on B200, no environment variable is read and only the
// default kernel instantiations exist. tools/ builds libcbrng_b200_tuning.so
// with -DCBRNG_TUNING=1, where tuning_knob() reads CBRNG_* environment knobs
// once per process and the alternative variants are compiled in, for A/B sweeps
// (tests/test_gpu_variants.py keeps every variant bit-exact).
#ifndef CBRNG_TUNING
#define CBRNG_TUNING 0
#endif

namespace cbrng {

constexpr bool TUNING = CBRNG_TUNING != 0;

// CBRNG_CEILING=1 builds the measurement-only libcbrng_ceiling.so that bench.py
// times beside the product: the single-stream fills and the multi-stream rows
// store into a small ring that stays in L2, so the HBM-free rate of the same
// instruction stream can be measured. Never set for the product library.
#ifndef CBRNG_CEILING
#define CBRNG_CEILING 0
#endif

// The value of environment knob `name` in [lo, hi] (tuning build), else dflt.
int tuning_knob(const char *name, int dflt, int lo, int hi);

// Launches go to the device that owns `stream` (the tensor's device in the
// Python layer), not whichever device happens to be current: the guard makes
// it current for the call and restores the caller's device afterwards.
class DeviceGuard {
  public:
    explicit DeviceGuard(void *stream) {
        if (!stream) return;
        int want = -1;
        if (cudaStreamGetDevice(reinterpret_cast<cudaStream_t>(stream), &want) != cudaSuccess) {
            cudaGetLastError();  // not a stream of this context: leave the device alone, the launch reports it
            return;
        }
        if (cudaGetDevice(&prev_) == cudaSuccess && prev_ != want && cudaSetDevice(want) == cudaSuccess) switched_ = true;
    }
    ~DeviceGuard() {
        if (switched_) cudaSetDevice(prev_);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;

  private:
    int prev_ = 0;
    bool switched_ = false;
};

void set_error(const char *fmt, ...);
void clear_error();

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Check the launch that was just enqueued (cudaGetLastError, non-blocking).
inline int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return CBRNG_ECUDA;
    }
    return CBRNG_OK;
}

inline int check_cuda(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return CBRNG_ECUDA;
    }
    return CBRNG_OK;
}

// Resident-grid size for a kernel on the current device: SMs x max resident
// CTAs (cached per kernel x device), capped by the amount of work.
int resident_blocks(const void *kernel, int block, size_t smem);

// cbrng_scalar ops 0-5: one thread, arguments by value (cbrng_multistream.cu).
int launch_scalar(int op, const uint64_t *args, uint32_t nargs, uint32_t *out, cudaStream_t st);
// cbrng_scalar op TYCHE_SEED_WORDS (cbrng_fill.cu).
int launch_tyche_seed_words(uint64_t seed, uint32_t sc, uint64_t n, uint32_t *out, cudaStream_t st);

// Grid policy for the streaming kernels: k x the resident grid (grid-stride),
// k = 8 (tuning build: CBRNG_GRID_MULT = k >= 1, or 0 = one tile per warp). The
// write-only probe (tools/probe_store.py) reaches 6.2 TB/s from a resident
// persistent grid (ncu: warps active ~60 % of theoretical) and 7.18 TB/s from a
// 16x grid; the fills gain 1-2 % and reach 95 % warps active at 8x
// (profiles/r1g_tune.md, profiles/r1h_ncu.md).
int grid_mult();

template <typename K>
inline unsigned grid_for(K kernel, int block, size_t smem, uint64_t work_blocks) {
    const int gm = grid_mult();
    uint64_t g = gm == 0 ? work_blocks : (uint64_t)resident_blocks(reinterpret_cast<const void *>(kernel), block, smem) * gm;
    if (work_blocks < g) g = work_blocks;
    if (g > 0x7FFFFFFFull) g = 0x7FFFFFFFull;
    if (g < 1) g = 1;
    return (unsigned)g;
}

inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

#define CBRNG_CHECK_ALG(alg)                                     \
    do {                                                         \
        if ((alg) < 0 || (alg) > 3) {                            \
            ::cbrng::set_error("unknown algorithm id %d", (alg)); \
            return CBRNG_EALG;                                   \
        }                                                        \
    } while (0)

#define CBRNG_REQUIRE(cond, ...)            \
    do {                                    \
        if (!(cond)) {                      \
            ::cbrng::set_error(__VA_ARGS__); \
            return CBRNG_EINVAL;            \
        }                                   \
    } while (0)

// 64-bit finaliser (SplitMix64) used by the order-free digests.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace cbrng
