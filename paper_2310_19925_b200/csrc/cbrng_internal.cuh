// cbrng_internal.cuh — host-side plumbing shared by the C-ABI translation units:
// error reporting, launch geometry (grid = SMs x resident CTAs), stream casts.
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "cbrng_b200.h"
#include "cbrng_cores.cuh"

namespace cbrng {

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

template <typename K>
inline unsigned grid_for(K kernel, int block, size_t smem, uint64_t work_blocks) {
    uint64_t g = (uint64_t)resident_blocks(reinterpret_cast<const void *>(kernel), block, smem);
    if (work_blocks < g) g = work_blocks;
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
