// cbrng_stats.cu — fused data producers + reductions for the statistical
// battery (reference stats.py:117-306).
//
// The reference battery materialises every byte it tests (stream_words ->
// bytes -> np.bincount). Here the generators feed the reductions directly:
//   * byte histogram of a single stream (monobit, chi_square_bytes;
//     stats.py:117-139 over run_battery's stream, :300-306), words never hit HBM;
//   * byte histogram of interleaved multi-stream micro-streams
//     (iter_interleave_chunks, stats.py:276-286) — same, per stream thread;
//   * byte histogram of an arbitrary device buffer (monobit(data) on user blobs);
//   * avalanche sums (avalanche_stats, stats.py:171-192): first words of
//     (seed, ctr) and (seed ^ flip, ctr), popcount and per-bit flip counts;
//   * Pearson sums of two unit-double arrays (interstream_correlation,
//     stats.py:205-240), deterministic: fixed per-block partials reduced in
//     block order.
// All counts are integers accumulated with atomics on u64, so the results are
// exact and independent of scheduling.
#include "cbrng_internal.cuh"
#include "cbrng_stream.cuh"

namespace cbrng {

constexpr int ST_BLOCK = 256;

// Block-shared byte histogram, flushed to the global u64 counts once per CTA.
struct SmemHist {
    uint32_t *h;
    __device__ __forceinline__ void add_word(uint32_t w) const {
        atomicAdd(&h[w & 0xFF], 1u);
        atomicAdd(&h[(w >> 8) & 0xFF], 1u);
        atomicAdd(&h[(w >> 16) & 0xFF], 1u);
        atomicAdd(&h[w >> 24], 1u);
    }
};

__device__ __forceinline__ void hist_init(uint32_t *h) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
}

__device__ __forceinline__ void hist_flush(const uint32_t *h, unsigned long long *counts) {
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(counts + i, (unsigned long long)h[i]);
}

// ---------------- single stream, counter-based ----------------
template <int ALG>
struct HistArgs {
    typename StreamOf<ALG>::T p;
    uint32_t bc0, skip, tail;  // tail: trailing words after the last full unit
    uint64_t n_units;
    unsigned long long *counts;
};

template <int ALG, bool SKIP>
__global__ void __launch_bounds__(ST_BLOCK) stream_hist_kernel(const __grid_constant__ HistArgs<ALG> a) {
    __shared__ uint32_t h[256];
    hist_init(h);
    const SmemHist H{h};
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < a.n_units;
         u += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 w = unit_words<ALG, SKIP>(a.p, a.bc0, a.skip, u);
        H.add_word(w.x); H.add_word(w.y); H.add_word(w.z); H.add_word(w.w);
    }
    if (a.tail && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint4 w = unit_words<ALG, SKIP>(a.p, a.bc0, a.skip, a.n_units);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        for (uint32_t k = 0; k < a.tail; k++) H.add_word(ws[k]);
    }
    hist_flush(h, a.counts);
}

// Tyche: one thread walks the chain (generators.py:221-224).
__global__ void tyche_hist_kernel(uint4 s, uint64_t n, unsigned long long *counts, uint32_t *state_out) {
    __shared__ uint32_t h[256];
    for (int i = 0; i < 256; i++) h[i] = 0;
    uint32_t A = s.x, B = s.y, C = s.z, D = s.w;
    for (uint64_t i = 0; i < n; i++) {
        tyche_mix(A, B, C, D);
        h[B & 0xFF]++; h[(B >> 8) & 0xFF]++; h[(B >> 16) & 0xFF]++; h[B >> 24]++;
    }
    for (int i = 0; i < 256; i++)
        if (h[i]) counts[i] += h[i];
    if (state_out) { state_out[0] = A; state_out[1] = B; state_out[2] = C; state_out[3] = D; }
}

template <int ALG>
static int launch_stream_hist(uint64_t seed, uint32_t sc, uint64_t word_pos, uint64_t n, unsigned long long *counts,
                              cudaStream_t st) {
    HistArgs<ALG> a;
    a.p = stream_setup<ALG>(seed, sc);
    if constexpr (ALG == SQUARES) { a.bc0 = (uint32_t)word_pos; a.skip = 0; }
    else { a.bc0 = (uint32_t)(word_pos >> 2); a.skip = (uint32_t)(word_pos & 3); }
    a.n_units = n / 4;
    a.tail = (uint32_t)(n % 4);
    a.counts = counts;
    if (ALG != SQUARES && a.skip) {
        auto k = stream_hist_kernel<ALG, true>;
        k<<<grid_for(k, ST_BLOCK, 0, (a.n_units + ST_BLOCK - 1) / ST_BLOCK), ST_BLOCK, 0, st>>>(a);
    } else {
        auto k = stream_hist_kernel<ALG, false>;
        k<<<grid_for(k, ST_BLOCK, 0, (a.n_units + ST_BLOCK - 1) / ST_BLOCK), ST_BLOCK, 0, st>>>(a);
    }
    return check_launch("stream_hist_kernel");
}

// ---------------- many short streams (interleave) ----------------
struct MultiHistArgs {
    uint64_t seed_base;
    uint32_t ctr0;     // iteration t uses counter ctr0 + t
    uint32_t nwords;
    uint64_t n_streams;
    uint64_t n_total;  // n_streams * n_iterations (stream, iteration) pairs
    unsigned long long *counts;
};

// First `nwords` words of stream (seed, ctr), fed to f(word) in stream order.
template <int ALG, typename F>
__device__ __forceinline__ void for_stream_words(uint64_t seed, uint32_t ctr, uint32_t nwords, F &&f) {
    if constexpr (ALG == PHILOX || ALG == THREEFRY) {
        for (uint32_t b = 0; 4 * b < nwords; b++) {
            const uint4 w = ALG == PHILOX
                                ? philox_block(make_uint4(ctr, b, 0, 0), (uint32_t)seed, (uint32_t)(seed >> 32))
                                : threefry_block(make_uint4(b, 0, 0, 0), (uint32_t)seed, (uint32_t)(seed >> 32), ctr, 0);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (4 * b + k < nwords) f(ws[k]);
        }
    } else if constexpr (ALG == SQUARES) {
        const uint64_t key = squares_key(seed);
        const uint64_t base = ((uint64_t)ctr << 32) * key;
        for (uint32_t j = 0; j < nwords; j++) f(squares_from_x((uint64_t)j * key + base, key));
    } else {
        uint4 s = tyche_init(seed, ctr);
        uint32_t A = s.x, B = s.y, C = s.z, D = s.w;
        for (uint32_t j = 0; j < nwords; j++) {
            tyche_mix(A, B, C, D);
            f(B);
        }
    }
}

template <int ALG>
__global__ void __launch_bounds__(ST_BLOCK) multi_hist_kernel(const __grid_constant__ MultiHistArgs a) {
    __shared__ uint32_t h[256];
    hist_init(h);
    const SmemHist H{h};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = i / a.n_streams, p = i - t * a.n_streams;
        for_stream_words<ALG>(a.seed_base + p, a.ctr0 + (uint32_t)t, a.nwords, [&](uint32_t w) { H.add_word(w); });
    }
    hist_flush(h, a.counts);
}

// ---------------- arbitrary device bytes ----------------
__global__ void __launch_bounds__(ST_BLOCK) buffer_hist_kernel(const uint8_t *data, uint64_t n,
                                                              unsigned long long *counts) {
    __shared__ uint32_t h[256];
    hist_init(h);
    const uint64_t nw = n / 4;  // whole 32-bit words (the pointer is 4-byte aligned)
    const uint32_t *w = reinterpret_cast<const uint32_t *>(data);
    const SmemHist H{h};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (uint64_t)gridDim.x * blockDim.x)
        H.add_word(__ldg(w + i));
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) atomicAdd(&h[data[4 * nw + threadIdx.x]], 1u);
    hist_flush(h, counts);
}

// ---------------- avalanche ----------------
// out[0] = sum popcount(w(seed) ^ w(seed ^ flip)); out[1 + b] = trials with bit b flipped.
template <int ALG>
__global__ void __launch_bounds__(ST_BLOCK) avalanche_kernel(const uint64_t *seeds, const uint32_t *ctrs,
                                                             const uint64_t *flips, uint64_t n,
                                                             unsigned long long *out) {
    const uint32_t lane = threadIdx.x & 31;
    uint64_t pop = 0, bitcnt = 0;  // lane b accumulates bit b's count
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const uint64_t i = base + threadIdx.x;
        uint32_t diff = 0;
        if (i < n) {
            uint32_t w0 = 0, w1 = 0;
            for_stream_words<ALG>(seeds[i], ctrs[i], 1, [&](uint32_t w) { w0 = w; });
            for_stream_words<ALG>(seeds[i] ^ flips[i], ctrs[i], 1, [&](uint32_t w) { w1 = w; });
            diff = w0 ^ w1;
            pop += __popc(diff);
        }
#pragma unroll
        for (int b = 0; b < 32; b++) {
            const uint32_t m = __ballot_sync(0xffffffffu, (diff >> b) & 1u);
            if (lane == b) bitcnt += __popc(m);
        }
    }
    for (int o = 16; o; o >>= 1) pop += __shfl_xor_sync(0xffffffffu, pop, o);
    if (lane == 0) atomicAdd(out, (unsigned long long)pop);
    atomicAdd(out + 1 + lane, (unsigned long long)bitcnt);
}

// ---------------- Pearson sums ----------------
// partials[block][5] = (sum a, sum b, sum a^2, sum b^2, sum ab) over the block's
// fixed index set; the host reduces blocks in order -> deterministic.
__global__ void __launch_bounds__(ST_BLOCK) pearson_kernel(const double *a, const double *b, uint64_t n,
                                                           double *partials) {
    double s[5] = {0, 0, 0, 0, 0};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double x = a[i], y = b[i];
        s[0] += x; s[1] += y; s[2] = fma(x, x, s[2]); s[3] = fma(y, y, s[3]); s[4] = fma(x, y, s[4]);
    }
    __shared__ double red[ST_BLOCK / 32][5];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 5; k++) {
        double v = s[k];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[w][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 5) {
        double v = 0;
        for (int j = 0; j < ST_BLOCK / 32; j++) v += red[j][threadIdx.x];
        partials[blockIdx.x * 5 + threadIdx.x] = v;
    }
}

}  // namespace cbrng

using namespace cbrng;

extern "C" {

int cbrng_stream_byte_histogram(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos,
                                const uint32_t *tyche_state, uint64_t n_words, uint64_t *counts,
                                uint32_t *tyche_state_out, void *stream) {
    const DeviceGuard device_guard(stream);
    CBRNG_CHECK_ALG(alg);
    clear_error();
    CBRNG_REQUIRE(counts, "counts is NULL");
    cudaStream_t st = as_stream(stream);
    auto *c = reinterpret_cast<unsigned long long *>(counts);
    if (alg == TYCHE) {
        CBRNG_REQUIRE(tyche_state, "tyche needs the serial state");
        tyche_hist_kernel<<<1, 1, 0, st>>>(make_uint4(tyche_state[0], tyche_state[1], tyche_state[2], tyche_state[3]),
                                           n_words, c, tyche_state_out);
        return check_launch("tyche_hist_kernel");
    }
    if (n_words == 0) return CBRNG_OK;
    if (alg == SQUARES) seed &= 0xFFFFFFFFull;
    switch (alg) {
        case PHILOX: return launch_stream_hist<PHILOX>(seed, stream_ctr, word_pos, n_words, c, st);
        case THREEFRY: return launch_stream_hist<THREEFRY>(seed, stream_ctr, word_pos, n_words, c, st);
        default: return launch_stream_hist<SQUARES>(seed, stream_ctr, word_pos, n_words, c, st);
    }
}

int cbrng_prefix_byte_histogram(int alg, uint64_t seed_base, uint32_t ctr0, uint32_t n_ctrs, uint64_t n_streams,
                                uint32_t nwords, uint64_t *counts, void *stream) {
    const DeviceGuard device_guard(stream);
    CBRNG_CHECK_ALG(alg);
    clear_error();
    CBRNG_REQUIRE(counts, "counts is NULL");
    if (n_streams == 0 || nwords == 0 || n_ctrs == 0) return CBRNG_OK;
    MultiHistArgs a{seed_base, ctr0, nwords, n_streams, n_streams * n_ctrs, reinterpret_cast<unsigned long long *>(counts)};
    cudaStream_t st = as_stream(stream);
    const uint64_t work = (a.n_total + ST_BLOCK - 1) / ST_BLOCK;
    switch (alg) {
        case PHILOX: { auto k = multi_hist_kernel<PHILOX>; k<<<grid_for(k, ST_BLOCK, 0, work), ST_BLOCK, 0, st>>>(a); break; }
        case THREEFRY: { auto k = multi_hist_kernel<THREEFRY>; k<<<grid_for(k, ST_BLOCK, 0, work), ST_BLOCK, 0, st>>>(a); break; }
        case SQUARES: { auto k = multi_hist_kernel<SQUARES>; k<<<grid_for(k, ST_BLOCK, 0, work), ST_BLOCK, 0, st>>>(a); break; }
        default: { auto k = multi_hist_kernel<TYCHE>; k<<<grid_for(k, ST_BLOCK, 0, work), ST_BLOCK, 0, st>>>(a); break; }
    }
    return check_launch("multi_hist_kernel");
}

int cbrng_buffer_byte_histogram(const uint8_t *data, uint64_t n, uint64_t *counts, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    CBRNG_REQUIRE(counts, "counts is NULL");
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(data && aligned(data, 4), "data must be a 4-byte aligned device pointer");
    auto k = buffer_hist_kernel;
    k<<<grid_for(k, ST_BLOCK, 0, (n / 4 + ST_BLOCK - 1) / ST_BLOCK + 1), ST_BLOCK, 0, as_stream(stream)>>>(
        data, n, reinterpret_cast<unsigned long long *>(counts));
    return check_launch("buffer_hist_kernel");
}

int cbrng_avalanche(int alg, const uint64_t *seeds, const uint32_t *ctrs, const uint64_t *flips, uint64_t n,
                    uint64_t *out, void *stream) {
    const DeviceGuard device_guard(stream);
    CBRNG_CHECK_ALG(alg);
    clear_error();
    CBRNG_REQUIRE(seeds && ctrs && flips && out, "NULL pointer");
    if (n == 0) return CBRNG_OK;
    auto *o = reinterpret_cast<unsigned long long *>(out);
    cudaStream_t st = as_stream(stream);
    const uint64_t work = (n + ST_BLOCK - 1) / ST_BLOCK;
    switch (alg) {
        case PHILOX: { auto k = avalanche_kernel<PHILOX>; k<<<grid_for(k, ST_BLOCK, 0, work), ST_BLOCK, 0, st>>>(seeds, ctrs, flips, n, o); break; }
        case THREEFRY: { auto k = avalanche_kernel<THREEFRY>; k<<<grid_for(k, ST_BLOCK, 0, work), ST_BLOCK, 0, st>>>(seeds, ctrs, flips, n, o); break; }
        case SQUARES: { auto k = avalanche_kernel<SQUARES>; k<<<grid_for(k, ST_BLOCK, 0, work), ST_BLOCK, 0, st>>>(seeds, ctrs, flips, n, o); break; }
        default: { auto k = avalanche_kernel<TYCHE>; k<<<grid_for(k, ST_BLOCK, 0, work), ST_BLOCK, 0, st>>>(seeds, ctrs, flips, n, o); break; }
    }
    return check_launch("avalanche_kernel");
}

int cbrng_pearson_partials(const double *a, const double *b, uint64_t n, uint32_t n_blocks, double *partials,
                           void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    CBRNG_REQUIRE(a && b && partials && n_blocks > 0, "bad arguments");
    pearson_kernel<<<n_blocks, ST_BLOCK, 0, as_stream(stream)>>>(a, b, n, partials);
    return check_launch("pearson_kernel");
}

}  // extern "C"
