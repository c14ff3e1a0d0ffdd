// cbrng_brownian.cu — the paper's Brownian-dynamics benchmark (PAPER.md:100-139,
// :263) with the reference semantics of brownian.py:107-195.
//
// Particles are SoA float64 (x, y, vx, vy) in HBM; pid is implicit (pid_base + i)
// or an explicit u64 array. Randomness is re-derived every step from the stream
// (seed = pid, counter = init_counter + it): no RNG state exists anywhere, and
// no random buffer is materialised — the 4 words are produced in registers
// and consumed by the update in the same thread.
//
// Two step kernels share one device function:
//   * PER_STEP: one launch per step, 64 B of HBM traffic per particle-step
//     (the paper's kernel shape; HBM-bound);
//   * FUSED: the particle stays in registers for all steps (particles are
//     independent, brownian.py:158-161, so this is a legal reordering); the
//     pid-only part of the key schedule is hoisted out of the step loop.
//     INT/FP64-pipe-bound.
//
// FP64 arithmetic is bit-exact with numpy's evaluation order:
//   vx -= ((gamma/mass) * vx) * dt;  vx += (r * 2.0 - 1.0) * sqrt(dt);  x += vx * dt
// with every operation an explicit round-to-nearest intrinsic (no FMA contraction).
#include <cmath>
#include <cstdlib>

#include "cbrng_internal.cuh"

namespace cbrng {

struct BrownArgs {
    uint64_t n;
    const uint64_t *pid;
    uint64_t pid_base;
    double *x, *y, *vx, *vy;
    uint32_t init_ctr;
    uint64_t first_it;
    uint64_t nsteps;
    double gm, dt, sqrt_dt;
    double kick_scale;  // sqrt_dt * 2^-52 (see kick())
    int fold;           // kick_scale is exact and normal: use the folded kick
    int reverse;        // per-step launches alternate the particle order (L2 reuse)
};

// Per-particle, step-invariant state.
template <int ALG, bool HI0 = false> struct Particle;
template <bool HI0> struct Particle<PHILOX, HI0> {
    PhiloxParticle<HI0> p;
    __device__ __forceinline__ explicit Particle(uint64_t pid) : p(philox_particle_setup<HI0>(pid)) {}
    __device__ __forceinline__ uint4 words(uint32_t ctr) const {
        uint32_t mh, ml;
        mulhilo(PHILOX_M0, ctr, mh, ml);
        return philox_particle_block<HI0>(p, mh, ml);
    }
};
template <bool HI0> struct Particle<THREEFRY, HI0> {
    uint32_t k0, k1;
    __device__ __forceinline__ explicit Particle(uint64_t pid) : k0((uint32_t)pid), k1((uint32_t)(pid >> 32)) {}
    __device__ __forceinline__ uint4 words(uint32_t ctr) const {
        return threefry_block(make_uint4(0, 0, 0, 0), k0, k1, ctr, 0);
    }
};
template <bool HI0> struct Particle<SQUARES, HI0> {
    uint64_t key;
    __device__ __forceinline__ explicit Particle(uint64_t pid) : key(squares_key(pid)) {}
    __device__ __forceinline__ uint4 words(uint32_t ctr) const {
        return squares_x4(((uint64_t)ctr << 32) * key, key);  // counters (ctr << 32) | k, k = 0..3
    }
};
template <bool HI0> struct Particle<TYCHE, HI0> {
    uint64_t pid;
    __device__ __forceinline__ explicit Particle(uint64_t p) : pid(p) {}
    __device__ __forceinline__ uint4 words(uint32_t ctr) const {
        uint4 s = tyche_init(pid, ctr);
        uint32_t a = s.x, b = s.y, c = s.z, d = s.w;
        uint4 w;
        tyche_mix(a, b, c, d); w.x = b;
        tyche_mix(a, b, c, d); w.y = b;
        tyche_mix(a, b, c, d); w.z = b;
        tyche_mix(a, b, c, d); w.w = b;
        return w;
    }
};

// Words 0..7 of stream (pid, ctr) for init_particles.
template <int ALG>
__device__ __forceinline__ void words8(uint64_t pid, uint32_t ctr, uint4 &w0, uint4 &w1) {
    if constexpr (ALG == PHILOX) {
        w0 = philox_block(make_uint4(ctr, 0, 0, 0), (uint32_t)pid, (uint32_t)(pid >> 32));
        w1 = philox_block(make_uint4(ctr, 1, 0, 0), (uint32_t)pid, (uint32_t)(pid >> 32));
    } else if constexpr (ALG == THREEFRY) {
        w0 = threefry_block(make_uint4(0, 0, 0, 0), (uint32_t)pid, (uint32_t)(pid >> 32), ctr, 0);
        w1 = threefry_block(make_uint4(1, 0, 0, 0), (uint32_t)pid, (uint32_t)(pid >> 32), ctr, 0);
    } else if constexpr (ALG == SQUARES) {
        uint64_t key = squares_key(pid), base = ((uint64_t)ctr << 32);
        w0 = make_uint4(squares_round(key, base | 0), squares_round(key, base | 1), squares_round(key, base | 2),
                        squares_round(key, base | 3));
        w1 = make_uint4(squares_round(key, base | 4), squares_round(key, base | 5), squares_round(key, base | 6),
                        squares_round(key, base | 7));
    } else {
        uint4 s = tyche_init(pid, ctr);
        uint32_t a = s.x, b = s.y, c = s.z, d = s.w;
        tyche_mix(a, b, c, d); w0.x = b;
        tyche_mix(a, b, c, d); w0.y = b;
        tyche_mix(a, b, c, d); w0.z = b;
        tyche_mix(a, b, c, d); w0.w = b;
        tyche_mix(a, b, c, d); w1.x = b;
        tyche_mix(a, b, c, d); w1.y = b;
        tyche_mix(a, b, c, d); w1.z = b;
        tyche_mix(a, b, c, d); w1.w = b;
    }
}

template <int ALG>
__global__ void __launch_bounds__(256) brownian_init_kernel(const __grid_constant__ BrownArgs a) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t pid = a.pid ? a.pid[i] : a.pid_base + i;
        uint4 w0, w1;
        words8<ALG>(pid, a.init_ctr, w0, w1);
        a.x[i] = u32x2_to_f64(w0.x, w0.y);
        a.y[i] = u32x2_to_f64(w0.z, w0.w);
        a.vx[i] = __dsub_rn(__dmul_rn(u32x2_to_f64(w1.x, w1.y), 2.0), 1.0);
        a.vy[i] = __dsub_rn(__dmul_rn(u32x2_to_f64(w1.z, w1.w), 2.0), 1.0);
    }
}

// The kick (r * 2.0 - 1.0) * sqrt(dt) of brownian.py:139-140 with r =
// ((lo | hi << 32) >> 11) * 2^-53. r*2 and r*2-1 are exact, and r*2-1 =
// v * 2^-52 with v = (u >> 11) - 2^52 = ((int64)(u ^ 2^63)) >> 11 (a signed
// 53-bit integer, converted exactly). Scaling by a power of two commutes with
// rounding (no subnormals here), so round((v * 2^-52) * s) == round(v * (s *
// 2^-52)): one conversion + one DMUL instead of conversion + 3 DMUL/DADD +
// DMUL, bit-identical (tests/test_gpu_parity.py::TestBrownian).
template <bool FOLD>
__device__ __forceinline__ double kick(uint32_t lo, uint32_t hi, double sqrt_dt, double kick_scale) {
    if constexpr (FOLD) {
        const int64_t v = (int64_t)(((uint64_t)(hi ^ 0x80000000u) << 32) | lo) >> 11;
        return __dmul_rn(__ll2double_rn(v), kick_scale);
    } else {
        return __dmul_rn(__dsub_rn(__dmul_rn(u32x2_to_f64(lo, hi), 2.0), 1.0), sqrt_dt);
    }
}

// One dynamics step of one particle (brownian.py:129-142).
template <bool FOLD>
__device__ __forceinline__ void step_update(double &x, double &y, double &vx, double &vy, uint4 w, const BrownArgs &a) {
    vx = __dsub_rn(vx, __dmul_rn(__dmul_rn(a.gm, vx), a.dt));
    vy = __dsub_rn(vy, __dmul_rn(__dmul_rn(a.gm, vy), a.dt));
    vx = __dadd_rn(vx, kick<FOLD>(w.x, w.y, a.sqrt_dt, a.kick_scale));
    vy = __dadd_rn(vy, kick<FOLD>(w.z, w.w, a.sqrt_dt, a.kick_scale));
    x = __dadd_rn(x, __dmul_rn(vx, a.dt));
    y = __dadd_rn(y, __dmul_rn(vy, a.dt));
}

// MINB: minimum resident CTAs per SM requested from ptxas (register cap). 5 CTAs
// (<= 51 registers) measured 3.40e11 p-steps/s; 6 CTAs (40 registers, small
// spill) 3.27e11 (profiles/r1j_tune.md).
template <int ALG, bool HI0, bool FOLD, int MINB>
__global__ void __launch_bounds__(256, MINB) brownian_steps_kernel(const __grid_constant__ BrownArgs a) {
    // Programmatic dependent launch (per-step mode): once every CTA of this grid
    // has started, the next step's grid may be scheduled onto the SMs this
    // grid's tail leaves idle; it sets up its particles' key schedules and waits
    // (griddepcontrol.wait) for this grid's writes before reading the state.
    // Both are no-ops for a normally launched grid.
    asm volatile("griddepcontrol.launch_dependents;");
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.n; j += (uint64_t)gridDim.x * blockDim.x) {
        // per-step mode walks the arrays in alternating directions, so each step
        // starts on the particles the previous step wrote last — still in L2
        const uint64_t i = a.reverse ? a.n - 1 - j : j;
        // an explicit pid array may have been written by the previous kernel on
        // the stream (load_snapshot's unpack_records): wait before reading it.
        // Implicit pids set up the key schedule under the previous grid's tail.
        if (a.pid) asm volatile("griddepcontrol.wait;" ::: "memory");
        const uint64_t pid = a.pid ? a.pid[i] : a.pid_base + i;
        const Particle<ALG, HI0> P(pid);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        double x = a.x[i], y = a.y[i], vx = a.vx[i], vy = a.vy[i];
        uint32_t ctr = a.init_ctr + (uint32_t)a.first_it;
        const uint32_t nsteps = (uint32_t)a.nsteps;  // host splits launches at 2^32 - 1 steps
        for (uint32_t s = 0; s < nsteps; s++, ctr++) step_update<FOLD>(x, y, vx, vy, P.words(ctr), a);
        a.x[i] = x; a.y[i] = y; a.vx[i] = vx; a.vy[i] = vy;
    }
}

// Fused walk, Philox with pid < 2^32: the two step-uniform multiplies of
// rounds 0-1 (philox_step_uniform) are computed once per step per CTA into a
// shared table of TAB steps (one step per thread), so each particle-step runs
// 16 IMAD.WIDE instead of 18 (the kernel is FMA-heavy-pipe bound). One thread
// per particle; threads past n take part in the table and the barriers only.
constexpr int BR_TAB = 256;

// SPLIT: Philox mulhilo as IMAD.HI + IMAD (mulhilo_c), tuning build only.
template <bool FOLD, int MINB, bool SPLIT = false>
__global__ void __launch_bounds__(256, MINB) brownian_fused_philox_kernel(const __grid_constant__ BrownArgs a) {
    __shared__ uint4 tab[BR_TAB];
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < a.n;
    const uint64_t pid = live ? (a.pid ? a.pid[i] : a.pid_base + i) : 0;
    double x = 0.0, y = 0.0, vx = 0.0, vy = 0.0;
    if (live) { x = a.x[i]; y = a.y[i]; vx = a.vx[i]; vy = a.vy[i]; }
    const PhiloxParticle<true> P = philox_particle_setup<true>(pid);
    const uint32_t ctr0 = a.init_ctr + (uint32_t)a.first_it;
    const uint32_t nsteps = (uint32_t)a.nsteps;
    for (uint32_t base = 0; base < nsteps; base += BR_TAB) {
        __syncthreads();  // the previous chunk's table is no longer read
        for (uint32_t j = threadIdx.x; j < BR_TAB; j += blockDim.x) tab[j] = philox_step_uniform(ctr0 + base + j);
        __syncthreads();
        const uint32_t m = nsteps - base < (uint32_t)BR_TAB ? nsteps - base : (uint32_t)BR_TAB;
#pragma unroll 2  // steps s and s+1 interleave (the cipher of s+1 under the FP64 chain of s): +3.5 %, r1t_tune.md
        for (uint32_t s = 0; s < m; s++) step_update<FOLD>(x, y, vx, vy, philox_particle_block_u<SPLIT>(P, tab[s]), a);
    }
    if (live) { a.x[i] = x; a.y[i] = y; a.vx[i] = vx; a.vy[i] = vy; }
}

// The same walk with one step table per warp instead of per CTA: lane l
// computes the step-uniform products of step base + l, the warp reads entry s
// for step base + s (a broadcast LDS), and __syncwarp is the only
// synchronisation, so warps of a CTA never wait for each other (the CTA-wide
// table costs two __syncthreads per 256 steps: ncu r1zd "barrier" 2.0 cycles per
// instruction, 12 % of the stall time). The table work grows from 1/256 to 1/32
// of a step-uniform evaluation per particle-step (2 IMAD.WIDE / 32). Measured
// 1 % slower than the CTA table (3.657e11 vs 3.691e11 p-steps/s): the barrier
// stalls were not what bounds the walk (the FMA-heavy pipe at 63 %, dispatch
// stalls). Tuning build only (CBRNG_BROWNIAN_TAB=2).
template <bool FOLD, int MINB>
__global__ void __launch_bounds__(256, MINB) brownian_fused_philox_wtab_kernel(const __grid_constant__ BrownArgs a) {
    __shared__ uint4 tab[256 / 32][32];
    uint4 *wt = tab[threadIdx.x >> 5];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < a.n;
    const uint64_t pid = live ? (a.pid ? a.pid[i] : a.pid_base + i) : 0;
    double x = 0.0, y = 0.0, vx = 0.0, vy = 0.0;
    if (live) { x = a.x[i]; y = a.y[i]; vx = a.vx[i]; vy = a.vy[i]; }
    const PhiloxParticle<true> P = philox_particle_setup<true>(pid);
    const uint32_t ctr0 = a.init_ctr + (uint32_t)a.first_it;
    const uint32_t nsteps = (uint32_t)a.nsteps;
    for (uint32_t base = 0; base < nsteps; base += 32) {
        __syncwarp();  // the previous chunk's entries are no longer read
        wt[lane] = philox_step_uniform(ctr0 + base + lane);
        __syncwarp();
        const uint32_t m = nsteps - base < 32u ? nsteps - base : 32u;
#pragma unroll 2
        for (uint32_t s = 0; s < m; s++) step_update<FOLD>(x, y, vx, vy, philox_particle_block_u(P, wt[s]), a);
    }
    if (live) { a.x[i] = x; a.y[i] = y; a.vx[i] = vx; a.vy[i] = vy; }
}

// ---------------- deterministic statistics ----------------
__device__ __forceinline__ int64_t fixq(double v, double scale) { return __double2ll_rn(v * scale); }

__global__ void __launch_bounds__(256) brownian_stats_kernel(uint64_t n, const uint64_t *pid, uint64_t pid_base,
                                                             const double *x, const double *y, const double *vx,
                                                             const double *vy, int64_t *acc) {
    int64_t s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = pid ? pid[i] : pid_base + i;
        const double X = x[i], Y = y[i], VX = vx[i], VY = vy[i];
        s[0] += 1;
        s[1] += fixq(X, 0x1p32);
        s[2] += fixq(Y, 0x1p32);
        s[3] += fixq(VX, 0x1p32);
        s[4] += fixq(VY, 0x1p32);
        s[5] += fixq(__dadd_rn(__dmul_rn(X, X), __dmul_rn(Y, Y)), 0x1p24);
        s[6] += fixq(__dadd_rn(__dmul_rn(VX, VX), __dmul_rn(VY, VY)), 0x1p24);
        uint64_t h = mix64(p ^ 0x5851F42D4C957F2Dull);
        h = mix64(h ^ (uint64_t)__double_as_longlong(X));
        h = mix64(h ^ (uint64_t)__double_as_longlong(Y));
        h = mix64(h ^ (uint64_t)__double_as_longlong(VX));
        h = mix64(h ^ (uint64_t)__double_as_longlong(VY));
        s[7] += (int64_t)h;
    }
    __shared__ int64_t red[8][8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        int64_t v = s[k];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[w][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        int64_t v = 0;
        for (int j = 0; j < (int)(blockDim.x >> 5); j++) v += red[j][threadIdx.x];
        atomicAdd(reinterpret_cast<unsigned long long *>(acc) + threadIdx.x, (unsigned long long)v);
    }
}

__global__ void __launch_bounds__(256) digest_u32_kernel(const uint32_t *w, uint64_t n, uint64_t off, uint64_t *acc) {
    uint64_t s = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        s += mix64(mix64(off + i) ^ (uint64_t)w[i]);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ uint64_t red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t v = 0;
        for (int j = 0; j < (int)(blockDim.x >> 5); j++) v += red[j];
        atomicAdd(reinterpret_cast<unsigned long long *>(acc), (unsigned long long)v);
    }
}

// Per-step launches alternate the particle order (tuning build:
// CBRNG_BROWNIAN_PINGPONG=0 keeps every launch ascending, for A/B runs).
static bool brownian_pingpong() {
    static const bool v = tuning_knob("CBRNG_BROWNIAN_PINGPONG", 1, 0, 1) != 0;
    return v;
}

// Per-step grids use programmatic dependent launch (tuning build:
// CBRNG_BROWNIAN_PDL=0 launches them plainly, for A/B runs).
static bool brownian_pdl() {
    static const bool v = tuning_knob("CBRNG_BROWNIAN_PDL", 1, 0, 1) != 0;
    return v;
}

constexpr int BROWNIAN_TAB_DEFAULT = 1;

// MINB applies to the fused table kernel; the per-step kernel keeps 5 CTAs/SM
// (6 spills there).
template <int ALG, bool HI0, bool FOLD, int MINB>
static int launch_steps_kb(BrownArgs a, int mode, cudaStream_t st) {
    // per-step launches (HBM-bound, one step each) run best at 4 CTAs/SM
    auto k = mode == CBRNG_BROWNIAN_PER_STEP && MINB > 1 ? brownian_steps_kernel<ALG, HI0, FOLD, (MINB > 4 ? 4 : MINB)>
                                                       : brownian_steps_kernel<ALG, HI0, FOLD, (MINB > 5 ? 5 : MINB)>;
    if constexpr (ALG == PHILOX && HI0) {
        // step table: 0 none, 1 per CTA (brownian_fused_philox_kernel), 2 per warp
        static const int tab = tuning_knob("CBRNG_BROWNIAN_TAB", BROWNIAN_TAB_DEFAULT, 0, 2);
        if (mode == CBRNG_BROWNIAN_FUSED && tab == 1) k = brownian_fused_philox_kernel<FOLD, MINB>;
        if constexpr (TUNING) {  // per-warp tables: 1 % slower (profiles/r2c_tune.md), tuning build only
            if (mode == CBRNG_BROWNIAN_FUSED && tab == 2) k = brownian_fused_philox_wtab_kernel<FOLD, MINB>;
            static const int split = tuning_knob("CBRNG_BROWNIAN_SPLIT", 0, 0, 2);
            if (mode == CBRNG_BROWNIAN_FUSED && tab == 1 && split == 1) k = brownian_fused_philox_kernel<FOLD, MINB, true>;
            if (mode == CBRNG_BROWNIAN_FUSED && tab == 1 && split == 2) k = brownian_fused_philox_kernel<FOLD, 4, true>;
        }
    }
    // One thread per particle: the fused kernel needs every particle resident
    // or queued, so the grid covers n (no persistence).
    const unsigned grid = (unsigned)((a.n + 255) / 256);
    const uint64_t total = a.nsteps;
    const uint64_t per_launch = mode == CBRNG_BROWNIAN_FUSED ? 0xFFFFFFFFull : 1;
    for (uint64_t done = 0; done < total;) {
        a.nsteps = total - done < per_launch ? total - done : per_launch;
        a.reverse = mode == CBRNG_BROWNIAN_PER_STEP && brownian_pingpong() ? (int)(a.first_it & 1) : 0;
        if (mode == CBRNG_BROWNIAN_PER_STEP && brownian_pdl()) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(256);
            cfg.stream = st;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            const int rc = check_cuda(cudaLaunchKernelEx(&cfg, k, a), "cudaLaunchKernelEx");
            if (rc) return rc;
        } else {
            k<<<grid, 256, 0, st>>>(a);
        }
        a.first_it += a.nsteps;
        done += a.nsteps;
    }
    return check_launch("brownian_steps_kernel");
}

constexpr int BROWNIAN_MINB = 5;

template <int ALG, bool HI0, bool FOLD>
static int launch_steps_k(BrownArgs a, int mode, cudaStream_t st) {
    if constexpr (!HI0) {
        return launch_steps_kb<ALG, HI0, FOLD, 1>(a, mode, st);  // 64-bit pids: 20 live keys, no cap
    } else {
        // register cap: 5 CTAs/SM (6 measured no better and spills with the
        // unrolled step loop, r1t_tune.md)
        return launch_steps_kb<ALG, HI0, FOLD, BROWNIAN_MINB>(a, mode, st);
    }
}

template <int ALG>
static int launch_steps(BrownArgs a, int mode, cudaStream_t st) {
    // pid < 2^32 everywhere (implicit pids): the high key word is zero.
    const bool hi0 = a.pid == nullptr && a.pid_base + a.n <= (1ull << 32);
    if (a.fold) {
        if (hi0) return launch_steps_k<ALG, true, true>(a, mode, st);
        return launch_steps_k<ALG, false, true>(a, mode, st);
    }
    if (hi0) return launch_steps_k<ALG, true, false>(a, mode, st);
    return launch_steps_k<ALG, false, false>(a, mode, st);
}

}  // namespace cbrng

using namespace cbrng;

// Snapshot / checksum records (brownian.py:198-250): pid-ordered 40-byte
// little-endian `<Qdddd` records, packed from the SoA arrays in HBM so only the
// packed bytes cross PCIe. Each record is five 8-byte words; thread i writes
// record i (a warp's 32 records are 1280 contiguous bytes, merged in L2).
__global__ void __launch_bounds__(256) pack_records_kernel(uint64_t n, const uint64_t *pid, uint64_t pid_base,
                                                           const double *x, const double *y, const double *vx,
                                                           const double *vy, uint64_t *rec) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t *r = rec + 5 * i;
        __stcs(r + 0, (unsigned long long)(pid ? pid[i] : pid_base + i));
        __stcs(r + 1, (unsigned long long)__double_as_longlong(x[i]));
        __stcs(r + 2, (unsigned long long)__double_as_longlong(y[i]));
        __stcs(r + 3, (unsigned long long)__double_as_longlong(vx[i]));
        __stcs(r + 4, (unsigned long long)__double_as_longlong(vy[i]));
    }
}

// Inverse of pack_records_kernel (load_snapshot, brownian.py:233-250); pid may be NULL.
__global__ void __launch_bounds__(256) unpack_records_kernel(uint64_t n, const uint64_t *rec, uint64_t *pid, double *x,
                                                             double *y, double *vx, double *vy) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t *r = rec + 5 * i;
        if (pid) pid[i] = __ldcs((const unsigned long long *)r);
        x[i] = __longlong_as_double((long long)__ldcs((const unsigned long long *)r + 1));
        y[i] = __longlong_as_double((long long)__ldcs((const unsigned long long *)r + 2));
        vx[i] = __longlong_as_double((long long)__ldcs((const unsigned long long *)r + 3));
        vy[i] = __longlong_as_double((long long)__ldcs((const unsigned long long *)r + 4));
    }
}

// Nonzero flag if pid[] is not strictly increasing (checksum precondition, brownian.py:209-212).
__global__ void __launch_bounds__(256) pid_order_kernel(uint64_t n, const uint64_t *pid, uint32_t *bad) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (pid[i] <= pid[i - 1]) *bad = 1u;
}

extern "C" {

int cbrng_brownian_init(int alg, uint64_t n, const uint64_t *pid, uint64_t pid_base, uint32_t init_ctr, double *x,
                        double *y, double *vx, double *vy, void *stream) {
    const DeviceGuard device_guard(stream);
    CBRNG_CHECK_ALG(alg);
    clear_error();
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(x && y && vx && vy, "NULL particle array");
    BrownArgs a{n, pid, pid_base, x, y, vx, vy, init_ctr, 0, 0, 0.0, 0.0, 0.0, 0.0, 0, 0};
    cudaStream_t st = as_stream(stream);
    const unsigned grid = (unsigned)((n + 255) / 256);
    switch (alg) {
        case PHILOX: brownian_init_kernel<PHILOX><<<grid, 256, 0, st>>>(a); break;
        case THREEFRY: brownian_init_kernel<THREEFRY><<<grid, 256, 0, st>>>(a); break;
        case SQUARES: brownian_init_kernel<SQUARES><<<grid, 256, 0, st>>>(a); break;
        default: brownian_init_kernel<TYCHE><<<grid, 256, 0, st>>>(a); break;
    }
    return check_launch("brownian_init_kernel");
}

int cbrng_brownian_steps(int alg, uint64_t n, const uint64_t *pid, uint64_t pid_base, double *x, double *y, double *vx,
                         double *vy, uint32_t init_ctr, uint64_t first_it, uint64_t nsteps, double gamma, double mass,
                         double dt, int mode, void *stream) {
    const DeviceGuard device_guard(stream);
    CBRNG_CHECK_ALG(alg);
    clear_error();
    CBRNG_REQUIRE(first_it >= 1, "iteration must be >= 1; counter 0 is reserved for init");
    CBRNG_REQUIRE(mode == CBRNG_BROWNIAN_PER_STEP || mode == CBRNG_BROWNIAN_FUSED, "bad mode %d", mode);
    CBRNG_REQUIRE(mass > 0.0 && gamma >= 0.0 && dt >= 0.0, "bad physical parameters");
    if (n == 0 || nsteps == 0) return CBRNG_OK;
    CBRNG_REQUIRE(x && y && vx && vy, "NULL particle array");
    // Host-side scalars exactly as the reference forms them (brownian.py:134, :177).
    BrownArgs a{n, pid, pid_base, x, y, vx, vy, init_ctr, first_it, nsteps, gamma / mass, dt, std::sqrt(dt), 0.0, 0, 0};
    a.kick_scale = a.sqrt_dt * 0x1p-52;
    // fold only when the scaled constant is exact (normal, no underflow)
    a.fold = a.sqrt_dt == 0.0 || (a.kick_scale >= 0x1p-1022 && a.kick_scale * 0x1p52 == a.sqrt_dt);
    cudaStream_t st = as_stream(stream);
    switch (alg) {
        case PHILOX: return launch_steps<PHILOX>(a, mode, st);
        case THREEFRY: return launch_steps<THREEFRY>(a, mode, st);
        case SQUARES: return launch_steps<SQUARES>(a, mode, st);
        default: return launch_steps<TYCHE>(a, mode, st);
    }
}

int cbrng_brownian_stats(uint64_t n, const uint64_t *pid, uint64_t pid_base, const double *x, const double *y,
                         const double *vx, const double *vy, int64_t *acc, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    CBRNG_REQUIRE(acc, "acc is NULL");
    if (n == 0) return CBRNG_OK;
    auto k = brownian_stats_kernel;
    k<<<grid_for(k, 256, 0, (n + 255) / 256), 256, 0, as_stream(stream)>>>(n, pid, pid_base, x, y, vx, vy, acc);
    return check_launch("brownian_stats_kernel");
}

int cbrng_digest_u32(const uint32_t *words, uint64_t n, uint64_t global_offset, uint64_t *acc, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    CBRNG_REQUIRE(acc, "acc is NULL");
    if (n == 0) return CBRNG_OK;
    auto k = digest_u32_kernel;
    k<<<grid_for(k, 256, 0, (n + 255) / 256), 256, 0, as_stream(stream)>>>(words, n, global_offset, acc);
    return check_launch("digest_u32_kernel");
}

int cbrng_pack_records(uint64_t n, const uint64_t *pid, uint64_t pid_base, const double *x, const double *y,
                       const double *vx, const double *vy, uint8_t *rec, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(x && y && vx && vy && rec, "NULL particle array or record buffer");
    CBRNG_REQUIRE(((uintptr_t)rec & 7) == 0, "record buffer must be 8-byte aligned");
    auto k = pack_records_kernel;
    k<<<grid_for(k, 256, 0, (n + 255) / 256), 256, 0, as_stream(stream)>>>(n, pid, pid_base, x, y, vx, vy,
                                                                           (uint64_t *)rec);
    return check_launch("pack_records_kernel");
}

int cbrng_unpack_records(uint64_t n, const uint8_t *rec, uint64_t *pid, double *x, double *y, double *vx,
                         double *vy, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(x && y && vx && vy && rec, "NULL particle array or record buffer");
    CBRNG_REQUIRE(((uintptr_t)rec & 7) == 0, "record buffer must be 8-byte aligned");
    auto k = unpack_records_kernel;
    k<<<grid_for(k, 256, 0, (n + 255) / 256), 256, 0, as_stream(stream)>>>(n, (const uint64_t *)rec, pid, x, y,
                                                                           vx, vy);
    return check_launch("unpack_records_kernel");
}

int cbrng_pid_order_check(uint64_t n, const uint64_t *pid, uint32_t *bad, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    CBRNG_REQUIRE(bad, "bad is NULL");
    if (n < 2 || !pid) return CBRNG_OK;
    auto k = pid_order_kernel;
    k<<<grid_for(k, 256, 0, (n + 255) / 256), 256, 0, as_stream(stream)>>>(n, pid, bad);
    return check_launch("pid_order_kernel");
}

}  // extern "C"
