// curand_baseline.cu — cuRAND comparison arm (timing baseline only, NOT the product).
//
// Built into its own library (libcbrng_curand_baseline.so) so the product
// library never links cuRAND. Two shapes:
//   * host-API fills with CURAND_RNG_PSEUDO_PHILOX4_32_10 (curandGenerate,
//     curandGenerateUniform, curandGenerateNormalDouble);
//   * the paper's cuRAND Brownian kernel: a 64-byte
//     curandStatePhilox4_32_10_t per particle in HBM, an init kernel
//     (curand_init(1984, i, 0, &state[i])), and curand_uniform2_double with the
//     state loaded and stored every step. Same SoA particle layout and update
//     arithmetic as the product kernel, so only the RNG strategy differs.
//   * a stronger cuRAND variant for the time-fused comparison: the state is
//     loaded once, kept in registers for all steps, and stored once;
//   * configs[4]'s many-stream shape through the device API (curand_rows_kernel).
// cuRAND's double map differs from the reference's (curand_uniform.h), so these
// results are not parity-checked — they only time the same work.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <curand.h>
#include <curand_kernel.h>

extern "C" {

static thread_local char g_cr_err[256] = "";
const char *cbrng_curand_last_error(void) { return g_cr_err; }

static int cr_check(curandStatus_t s, const char *what) {
    if (s != CURAND_STATUS_SUCCESS) {
        snprintf(g_cr_err, sizeof g_cr_err, "%s: curand status %d", what, (int)s);
        return -3;
    }
    return 0;
}

// Opaque generator handle: created once, reused for timing.
void *cbrng_curand_create(uint64_t seed, void *stream) {
    curandGenerator_t g;
    if (curandCreateGenerator(&g, CURAND_RNG_PSEUDO_PHILOX4_32_10) != CURAND_STATUS_SUCCESS) return nullptr;
    curandSetPseudoRandomGeneratorSeed(g, seed);
    curandSetStream(g, (cudaStream_t)stream);
    return (void *)g;
}

int cbrng_curand_destroy(void *g) { return cr_check(curandDestroyGenerator((curandGenerator_t)g), "destroy"); }

int cbrng_curand_set_offset(void *g, uint64_t offset) {
    return cr_check(curandSetGeneratorOffset((curandGenerator_t)g, offset), "offset");
}

int cbrng_curand_u32(void *g, uint32_t *out, uint64_t n) {
    return cr_check(curandGenerate((curandGenerator_t)g, out, n), "curandGenerate");
}

int cbrng_curand_uniform_f32(void *g, float *out, uint64_t n) {
    return cr_check(curandGenerateUniform((curandGenerator_t)g, out, n), "curandGenerateUniform");
}

int cbrng_curand_uniform_f64(void *g, double *out, uint64_t n) {
    return cr_check(curandGenerateUniformDouble((curandGenerator_t)g, out, n), "curandGenerateUniformDouble");
}

int cbrng_curand_normal_f64(void *g, double *out, uint64_t n) {
    return cr_check(curandGenerateNormalDouble((curandGenerator_t)g, out, n, 0.0, 1.0), "curandGenerateNormalDouble");
}

}  // extern "C"

__global__ void curand_state_init_kernel(curandStatePhilox4_32_10_t *st, uint64_t n) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    curand_init(1984, i, 0, &st[i]);
}

__global__ void curand_brownian_init_kernel(curandStatePhilox4_32_10_t *st, uint64_t n, double *x, double *y,
                                            double *vx, double *vy) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    curandStatePhilox4_32_10_t s = st[i];
    double2 p = curand_uniform2_double(&s);
    double2 v = curand_uniform2_double(&s);
    x[i] = p.x; y[i] = p.y;
    vx[i] = v.x * 2.0 - 1.0; vy[i] = v.y * 2.0 - 1.0;
    st[i] = s;
}

// state loaded and stored every step.
__global__ void curand_brownian_step_kernel(curandStatePhilox4_32_10_t *st, uint64_t n, double *x, double *y,
                                            double *vx, double *vy, uint64_t nsteps, double gm, double dt,
                                            double sqrt_dt) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double X = x[i], Y = y[i], VX = vx[i], VY = vy[i];
    curandStatePhilox4_32_10_t s = st[i];
    for (uint64_t k = 0; k < nsteps; k++) {
        VX = __dsub_rn(VX, __dmul_rn(__dmul_rn(gm, VX), dt));
        VY = __dsub_rn(VY, __dmul_rn(__dmul_rn(gm, VY), dt));
        double2 r = curand_uniform2_double(&s);
        VX = __dadd_rn(VX, __dmul_rn(__dsub_rn(__dmul_rn(r.x, 2.0), 1.0), sqrt_dt));
        VY = __dadd_rn(VY, __dmul_rn(__dsub_rn(__dmul_rn(r.y, 2.0), 1.0), sqrt_dt));
        X = __dadd_rn(X, __dmul_rn(VX, dt));
        Y = __dadd_rn(Y, __dmul_rn(VY, dt));
    }
    st[i] = s;
    x[i] = X; y[i] = Y; vx[i] = VX; vy[i] = VY;
}

extern "C" {

uint64_t cbrng_curand_state_bytes(void) { return sizeof(curandStatePhilox4_32_10_t); }

// state: [dev] n * cbrng_curand_state_bytes() bytes.
int cbrng_curand_brownian_init(void *state, uint64_t n, double *x, double *y, double *vx, double *vy, void *stream) {
    auto *st = (curandStatePhilox4_32_10_t *)state;
    unsigned grid = (unsigned)((n + 255) / 256);
    curand_state_init_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(st, n);
    curand_brownian_init_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(st, n, x, y, vx, vy);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// fused != 0: one launch keeping the state in registers; else one launch per step.
int cbrng_curand_brownian_steps(void *state, uint64_t n, double *x, double *y, double *vx, double *vy, uint64_t nsteps,
                                double gamma, double mass, double dt, int fused, void *stream) {
    auto *st = (curandStatePhilox4_32_10_t *)state;
    unsigned grid = (unsigned)((n + 255) / 256);
    double gm = gamma / mass, sq = std::sqrt(dt);
    if (fused) {
        curand_brownian_step_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(st, n, x, y, vx, vy, nsteps, gm, dt, sq);
    } else {
        for (uint64_t k = 0; k < nsteps; k++)
            curand_brownian_step_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(st, n, x, y, vx, vy, 1, gm, dt, sq);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // extern "C"

// configs[4] shape with the cuRAND device API: stream s = curand_init(seed = s,
// subsequence 0, offset 0) on a Philox4_32_10 state in registers, 256 words
// drawn with curand4 and written row-major (out[s][j]), one thread per stream,
// 16-byte stores. What a cuRAND user writes for "n independent streams x 256".
__global__ void __launch_bounds__(256) curand_rows_kernel(uint64_t seed_base, uint64_t n_streams, uint32_t nwords,
                                                          uint4 *out) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_streams) return;
    curandStatePhilox4_32_10_t st;
    curand_init(seed_base + s, 0, 0, &st);
    uint4 *row = out + s * (nwords / 4);
    for (uint32_t j = 0; j < nwords / 4; j++) __stcs(row + j, curand4(&st));
}

extern "C" int cbrng_curand_rows(uint64_t seed_base, uint64_t n_streams, uint32_t nwords, uint32_t *out,
                                 void *stream) {
    if (nwords % 4) return -1;
    const uint64_t grid = (n_streams + 255) / 256;
    curand_rows_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(seed_base, n_streams, nwords, (uint4 *)out);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ---------------------------------------------------------------------------
// Store-bandwidth probe (measurement only): the write-only HBM ceiling for the
// fill kernels' exact store pattern (resident grid, 4 x 16-byte streaming stores
// per lane per tile). pattern 0 writes zeros (compressible), 1 writes
// index*golden (incompressible, one IMAD per word) — B200's L2 compresses
// zero-filled lines, so memset overstates what random data can reach.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) probe_store_kernel(uint4 *out, uint64_t n_units, int pattern) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = warp; t * 128 < n_units; t += nwarps) {
        const uint64_t base = t * 128 + lane;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint64_t u = base + 32 * j;
            if (u < n_units) {
                const uint32_t v = (uint32_t)u * 0x9E3779B9u;
                __stcs(out + u, pattern ? make_uint4(v, v ^ 0x5bd1e995u, v + 0x1b873593u, v * 3u)
                                        : make_uint4(0u, 0u, 0u, 0u));
            }
        }
    }
}

extern "C" int cbrng_probe_store(void *out, uint64_t n_bytes, int pattern, int blocks, void *stream) {
    uint64_t n_units = n_bytes / 16;
    if (blocks <= 0) {
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe_store_kernel, 256, 0);
        blocks = sms * occ;
    }
    probe_store_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((uint4 *)out, n_units, pattern);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
