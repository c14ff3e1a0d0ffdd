// cbrng_cores.cuh — register-resident counter-based generator cores for sm_100a.
//
// Bit-exact restatements of the reference algorithms
// (/root/reference/pkg/src/cbrng/generators.py:97-224), written for the GPU:
// every function is a pure function of (key, counter) kept in registers, with
// no global state. Launch-uniform work (round-key schedules, the parts of the
// first rounds that depend only on (seed, stream counter)) is folded on the
// host into kernel parameters, so it costs zero per-element instructions: the
// LOP3s read it straight from the constant bank.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cbrng {

enum Alg : int { PHILOX = 0, THREEFRY = 1, SQUARES = 2, TYCHE = 3 };

// generators.py:35-54
constexpr uint32_t PHILOX_M0 = 0xD2511F53u;
constexpr uint32_t PHILOX_M1 = 0xCD9E8D57u;
constexpr uint32_t PHILOX_W0 = 0x9E3779B9u;
constexpr uint32_t PHILOX_W1 = 0xBB67AE85u;
constexpr uint32_t THREEFRY_PARITY = 0x1BD11BDAu;
constexpr uint32_t TYCHE_INIT_CONST = 0x9E3779B9u;
constexpr uint64_t GOLDEN64 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t SPLITMIX_M1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t SPLITMIX_M2 = 0x94D049BB133111EBull;

__host__ __device__ __forceinline__ uint32_t rotl32(uint32_t x, int r) {
#ifdef __CUDA_ARCH__
    return __funnelshift_l(x, x, r);  // SHF.L.W
#else
    return (x << r) | (x >> (32 - r));
#endif
}

__host__ __device__ __forceinline__ void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#ifdef __CUDA_ARCH__
    // mul.wide.u32 -> IMAD.WIDE.U32 (one FMA-heavy op for both halves)
    uint64_t p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
#else
    uint64_t p = (uint64_t)a * b;
#endif
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
}

// The Philox multipliers in the constant bank: an IMAD can read one directly.
static __constant__ uint32_t c_philox_m[2] = {0xD2511F53u, 0xCD9E8D57u};

// M * b as separate high (IMAD.HI, immediate M) and low (IMAD, constant-bank M,
// so ptxas cannot fuse the pair back into one IMAD.WIDE) halves. In kernels
// that mix the cipher with FP64 work the split form overlaps with DFMA/DMUL,
// while IMAD.WIDE and the FP64 ops all but serialise on B200 (pipe probes,
// profiles/r2f_probe_pipes.json: IMAD.WIDE + 2 DFMA 7.8 cycles per warp and
// set, IMAD.HI + IMAD + 2 DFMA 6.6, for 4 and 6 heavy-pipe cycles alone).
template <uint32_t M, bool SPLIT>
__device__ __forceinline__ void mulhilo_c(uint32_t b, uint32_t &hi, uint32_t &lo) {
    if constexpr (SPLIT) {
        hi = __umulhi(b, M);
        lo = b * c_philox_m[M == 0xD2511F53u ? 0 : 1];
    } else {
        mulhilo(M, b, hi, lo);
    }
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (generators.py:101-122)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                                      uint32_t k0, uint32_t k1) {
    uint32_t h0, l0, h1, l1;
    mulhilo(PHILOX_M0, c0, h0, l0);
    mulhilo(PHILOX_M1, c2, h1, l1);
    c0 = h1 ^ c1 ^ k0;
    c1 = l1;
    c2 = h0 ^ c3 ^ k1;
    c3 = l0;
}

// Generic block: per-element key schedule (used where the key varies per lane).
__host__ __device__ __forceinline__ uint4 philox_block(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        philox_round(c.x, c.y, c.z, c.w, k0, k1);
        k0 += PHILOX_W0;
        k1 += PHILOX_W1;
    }
    return c;
}

// Single stream (key, stream counter sc) with ctr = (sc, bc, 0, 0): rounds 0-3
// partially depend only on (key, sc). The host folds those parts into this
// struct (philox_stream_setup) and the device runs 16 IMAD.WIDE + 18 LOP per
// block instead of 20 + 20 (+18 key adds).
struct PhiloxStream {
    uint32_t k0_0;    // round 0: c0 = bc ^ k0_0
    uint32_t a1;      // round 1: c2 = hi(M0*c0) ^ a1
    uint32_t b2, c2;  // round 2: c0 = hi(M1*c2) ^ b2 ; c2 = c3 ^ c2k
    uint32_t v0, v1;  // round-1 uniform outputs (c0, c1)
    uint32_t k0_3, e3;  // round 3: c0 = hi(M1*c2) ^ c1 ^ k0_3 ; c2 = hi(M0*c0) ^ e3
    uint32_t rk0[6], rk1[6];  // rounds 4..9
};

__host__ __device__ inline PhiloxStream philox_stream_setup(uint64_t seed, uint32_t sc) {
    uint32_t K0[10], K1[10];
    K0[0] = (uint32_t)seed;
    K1[0] = (uint32_t)(seed >> 32);
    for (int r = 1; r < 10; r++) { K0[r] = K0[r - 1] + PHILOX_W0; K1[r] = K1[r - 1] + PHILOX_W1; }
    PhiloxStream p;
    uint32_t h, l;
    // round 0 with c = (sc, bc, 0, 0): p0 = M0*sc, p1 = 0
    mulhilo(PHILOX_M0, sc, h, l);
    uint32_t u2 = h ^ K1[0], u3 = l;  // c2, c3 after round 0; c0 = bc ^ K0[0], c1 = 0
    p.k0_0 = K0[0];
    // round 1: p0 = M0*c0 (varies), p1 = M1*u2 (uniform)
    mulhilo(PHILOX_M1, u2, h, l);
    p.v0 = h ^ 0u ^ K0[1];
    p.v1 = l;
    p.a1 = u3 ^ K1[1];  // c2 = hi(M0*c0) ^ c3(=u3) ^ K1[1]; c3 = lo(M0*c0)
    // round 2: p0 = M0*v0 (uniform), p1 = M1*c2 (varies)
    mulhilo(PHILOX_M0, p.v0, h, l);
    p.b2 = p.v1 ^ K0[2];  // c0 = hi(M1*c2) ^ v1 ^ K0[2]; c1 = lo(M1*c2)
    p.c2 = h ^ K1[2];     // c2 = hi(M0*v0) ^ c3 ^ K1[2]
    uint32_t d = l;       // c3 = lo(M0*v0)
    // round 3: c2 = hi(M0*c0) ^ d ^ K1[3]
    p.k0_3 = K0[3];
    p.e3 = d ^ K1[3];
    for (int r = 4; r < 10; r++) { p.rk0[r - 4] = K0[r]; p.rk1[r - 4] = K1[r]; }
    return p;
}

template <bool SPLIT>
__device__ __forceinline__ void philox_round_d(uint32_t &c0, uint32_t &c1, uint32_t &c2, uint32_t &c3, uint32_t k0,
                                               uint32_t k1) {
    uint32_t h0, l0, h1, l1;
    mulhilo_c<PHILOX_M0, SPLIT>(c0, h0, l0);
    mulhilo_c<PHILOX_M1, SPLIT>(c2, h1, l1);
    c0 = h1 ^ c1 ^ k0;
    c1 = l1;
    c2 = h0 ^ c3 ^ k1;
    c3 = l0;
}

// SPLIT: bit r set = round r's mulhilos as IMAD.HI + IMAD (mulhilo_c), for
// kernels that mix in FP64 (1 = every round).
template <int SPLIT = 0>
__device__ __forceinline__ uint4 philox_stream_block(const PhiloxStream& p, uint32_t bc) {
    constexpr int M = SPLIT == 1 ? 0x3FF : SPLIT;
    uint32_t c0, c1, c2, c3, h, l;
    // round 0
    c0 = bc ^ p.k0_0;
    // round 1
    mulhilo_c<PHILOX_M0, (M >> 1) & 1>(c0, h, l);
    c2 = h ^ p.a1;
    c3 = l;
    // round 2
    mulhilo_c<PHILOX_M1, (M >> 2) & 1>(c2, h, l);
    c0 = h ^ p.b2;
    c1 = l;
    c2 = c3 ^ p.c2;
    // round 3 (c3 of round 2 is uniform and folded into e3)
    {
        uint32_t h0, l0, h1, l1;
        mulhilo_c<PHILOX_M0, (M >> 3) & 1>(c0, h0, l0);
        mulhilo_c<PHILOX_M1, (M >> 3) & 1>(c2, h1, l1);
        c0 = h1 ^ c1 ^ p.k0_3;
        c1 = l1;
        c2 = h0 ^ p.e3;
        c3 = l0;
    }
    philox_round_d<(M >> 4) & 1>(c0, c1, c2, c3, p.rk0[0], p.rk1[0]);
    philox_round_d<(M >> 5) & 1>(c0, c1, c2, c3, p.rk0[1], p.rk1[1]);
    philox_round_d<(M >> 6) & 1>(c0, c1, c2, c3, p.rk0[2], p.rk1[2]);
    philox_round_d<(M >> 7) & 1>(c0, c1, c2, c3, p.rk0[3], p.rk1[3]);
    philox_round_d<(M >> 8) & 1>(c0, c1, c2, c3, p.rk0[4], p.rk1[4]);
    philox_round_d<(M >> 9) & 1>(c0, c1, c2, c3, p.rk0[5], p.rk1[5]);
    return make_uint4(c0, c1, c2, c3);
}

// Per-particle Philox for the Brownian walk: key = pid, ctr = (counter, 0, 0, 0).
// Everything that depends only on pid is hoisted out of the step loop. HI0:
// every pid < 2^32 (the reference's np.arange pids for n <= 2^32), so the
// high key word is 0 and its round keys K1[r] = r*W1 are compile-time
// constants — 10 fewer registers per particle.
template <bool HI0>
struct PhiloxParticle {
    uint32_t k0[10], k1[HI0 ? 1 : 10];
    uint32_t q1;       // round 1: c2 = c3 ^ q1, q1 = hi(M0*pid_lo) ^ K1[1]
    uint32_t r2;       // round 2: c2 = hi(M0*c0) ^ r2, r2 = lo(M0*pid_lo) ^ K1[2]
    __device__ __forceinline__ uint32_t K1(int r) const {
        if constexpr (HI0) return (uint32_t)r * PHILOX_W1;
        else return k1[r];
    }
};

template <bool HI0>
__device__ __forceinline__ PhiloxParticle<HI0> philox_particle_setup(uint64_t pid) {
    PhiloxParticle<HI0> p;
    p.k0[0] = (uint32_t)pid;
#pragma unroll
    for (int r = 1; r < 10; r++) p.k0[r] = p.k0[r - 1] + PHILOX_W0;
    if constexpr (!HI0) {
        p.k1[0] = (uint32_t)(pid >> 32);
#pragma unroll
        for (int r = 1; r < 10; r++) p.k1[r] = p.k1[r - 1] + PHILOX_W1;
    }
    uint32_t h, l;
    mulhilo(PHILOX_M0, p.k0[0], h, l);
    p.q1 = h ^ p.K1(1);
    p.r2 = l ^ p.K1(2);
    // Pin the round keys in registers: without this the compiler re-derives
    // k[r] = k[0] + r*W inside the step loop (18 VIADDs per step on the
    // FMA-heavy pipe, ncu r1a) to save registers.
#pragma unroll
    for (int r = 0; r < 10; r++) asm volatile("" : "+r"(p.k0[r]));
    if constexpr (!HI0) {
#pragma unroll
        for (int r = 0; r < 10; r++) asm volatile("" : "+r"(p.k1[r]));
    }
    return p;
}

// Block 0 of stream (pid, ctr); mh/ml = hi/lo(M0*ctr) are step-uniform.
template <bool HI0>
__device__ __forceinline__ uint4 philox_particle_block(const PhiloxParticle<HI0>& p, uint32_t mh, uint32_t ml) {
    uint32_t c0, c1, c2, c3, h, l;
    // round 0: c = (ctr, 0, 0, 0): c0 = pid_lo ; c1 = 0 ; c2 = hi(M0*ctr) ^ K1 ; c3 = lo(M0*ctr)
    c2 = mh ^ p.K1(0);
    c3 = ml;
    // round 1: p0 = M0*pid_lo (hoisted), p1 = M1*c2
    mulhilo(PHILOX_M1, c2, h, l);
    c0 = h ^ p.k0[1];  // c1 == 0
    c1 = l;
    c2 = c3 ^ p.q1;
    // round 2: c3 == lo(M0*pid_lo) (hoisted) is folded into r2
    {
        uint32_t h0, l0, h1, l1;
        mulhilo(PHILOX_M0, c0, h0, l0);
        mulhilo(PHILOX_M1, c2, h1, l1);
        c0 = h1 ^ c1 ^ p.k0[2];
        c1 = l1;
        c2 = h0 ^ p.r2;
        c3 = l0;
    }
#pragma unroll
    for (int r = 3; r < 10; r++) philox_round(c0, c1, c2, c3, p.k0[r], p.K1(r));
    return make_uint4(c0, c1, c2, c3);
}

// The same block from rounds 0-1's step-uniform products: with pid < 2^32 (HI0)
// round 0's c2 = hi(M0*ctr) does not depend on the particle, so both
// M0*ctr and round 1's M1*c2 are the same for every thread of a step. The
// fused Brownian kernel computes them once per step per CTA (u = {-, lo(M0*ctr),
// hi(M1*c2), lo(M1*c2)}) and each particle starts at round 1's xors.
template <bool SPLIT = false>
__device__ __forceinline__ uint4 philox_particle_block_u(const PhiloxParticle<true>& p, uint4 u) {
    uint32_t c0 = u.z ^ p.k0[1];  // c1 of round 0 == 0
    uint32_t c1 = u.w;
    uint32_t c2 = u.y ^ p.q1;     // c3 of round 0 = lo(M0*ctr)
    uint32_t c3;
    {
        uint32_t h0, l0, h1, l1;
        mulhilo_c<PHILOX_M0, SPLIT>(c0, h0, l0);
        mulhilo_c<PHILOX_M1, SPLIT>(c2, h1, l1);
        c0 = h1 ^ c1 ^ p.k0[2];
        c1 = l1;
        c2 = h0 ^ p.r2;
        c3 = l0;
    }
#pragma unroll
    for (int r = 3; r < 10; r++) philox_round_d<SPLIT>(c0, c1, c2, c3, p.k0[r], p.K1(r));
    return make_uint4(c0, c1, c2, c3);
}

__host__ __device__ __forceinline__ uint4 philox_step_uniform(uint32_t ctr) {
    uint32_t mh, ml, h1, l1;
    mulhilo(PHILOX_M0, ctr, mh, ml);
    mulhilo(PHILOX_M1, mh, h1, l1);  // c2 = mh ^ K1(0), K1(0) = pid_hi = 0
    return make_uint4(mh, ml, h1, l1);
}

// ---------------------------------------------------------------------------
// Threefry4x32-20 (generators.py:125-154)
// ---------------------------------------------------------------------------
// Rotation pairs R[r % 8] (generators.py:44-47) as compile-time constants.
template <int R> struct TfRot;
template <> struct TfRot<0> { static constexpr int a = 10, b = 26; };
template <> struct TfRot<1> { static constexpr int a = 11, b = 21; };
template <> struct TfRot<2> { static constexpr int a = 13, b = 27; };
template <> struct TfRot<3> { static constexpr int a = 23, b = 5; };
template <> struct TfRot<4> { static constexpr int a = 6, b = 20; };
template <> struct TfRot<5> { static constexpr int a = 17, b = 11; };
template <> struct TfRot<6> { static constexpr int a = 25, b = 10; };
template <> struct TfRot<7> { static constexpr int a = 18, b = 20; };

template <int R>
__host__ __device__ __forceinline__ void threefry_round(uint32_t& x0, uint32_t& x1, uint32_t& x2, uint32_t& x3) {
    constexpr int ra = TfRot<R % 8>::a, rb = TfRot<R % 8>::b;
    if (R % 2 == 0) {
        x0 += x1; x1 = rotl32(x1, ra) ^ x0;
        x2 += x3; x3 = rotl32(x3, rb) ^ x2;
    } else {
        x0 += x3; x3 = rotl32(x3, ra) ^ x0;
        x2 += x1; x1 = rotl32(x1, rb) ^ x2;
    }
}

// Key injection j (after round 4j-1): x[i] += ks[(j+i)%5]; x3 += j.
template <int J>
__host__ __device__ __forceinline__ void threefry_inject(uint32_t& x0, uint32_t& x1, uint32_t& x2, uint32_t& x3,
                                                         const uint32_t ks[5]) {
    x0 += ks[(J + 0) % 5];
    x1 += ks[(J + 1) % 5];
    x2 += ks[(J + 2) % 5];
    x3 += ks[(J + 3) % 5] + (uint32_t)J;
}

// Rounds FIRST..19 with injections, starting from state x (already past rounds < FIRST).
template <int FIRST>
__host__ __device__ __forceinline__ void threefry_rounds_from(uint32_t& x0, uint32_t& x1, uint32_t& x2, uint32_t& x3,
                                                              const uint32_t ks[5]) {
#define TF_R(R)                                                         \
    if (R >= FIRST) {                                                   \
        threefry_round<R>(x0, x1, x2, x3);                              \
        if ((R + 1) % 4 == 0) threefry_inject<(R + 1) / 4>(x0, x1, x2, x3, ks); \
    }
    TF_R(0) TF_R(1) TF_R(2) TF_R(3) TF_R(4) TF_R(5) TF_R(6) TF_R(7) TF_R(8) TF_R(9)
    TF_R(10) TF_R(11) TF_R(12) TF_R(13) TF_R(14) TF_R(15) TF_R(16) TF_R(17) TF_R(18) TF_R(19)
#undef TF_R
}

__host__ __device__ __forceinline__ uint4 threefry_block(uint4 c, uint32_t k0, uint32_t k1, uint32_t k2, uint32_t k3) {
    uint32_t ks[5] = {k0, k1, k2, k3, THREEFRY_PARITY ^ k0 ^ k1 ^ k2 ^ k3};
    uint32_t x0 = c.x + ks[0], x1 = c.y + ks[1], x2 = c.z + ks[2], x3 = c.w + ks[3];
    threefry_rounds_from<0>(x0, x1, x2, x3, ks);
    return make_uint4(x0, x1, x2, x3);
}

// Variable round count (the reference's `rounds=` argument, used by the
// 13-round Random123 KAT). Not a hot path.
__host__ __device__ inline uint4 threefry_block_rounds(uint4 c, const uint32_t key[4], int rounds) {
    uint32_t ks[5] = {key[0], key[1], key[2], key[3], THREEFRY_PARITY ^ key[0] ^ key[1] ^ key[2] ^ key[3]};
    uint32_t x[4] = {c.x + ks[0], c.y + ks[1], c.z + ks[2], c.w + ks[3]};
    const int ROT[8][2] = {{10, 26}, {11, 21}, {13, 27}, {23, 5}, {6, 20}, {17, 11}, {25, 10}, {18, 20}};
    for (int r = 0; r < rounds; r++) {
        int ra = ROT[r % 8][0], rb = ROT[r % 8][1];
        int a = (r % 2 == 0) ? 1 : 3, b = (r % 2 == 0) ? 3 : 1;
        x[0] += x[a]; x[a] = rotl32(x[a], ra) ^ x[0];
        x[2] += x[b]; x[b] = rotl32(x[b], rb) ^ x[2];
        if ((r + 1) % 4 == 0) {
            uint32_t j = (uint32_t)((r + 1) / 4);
            for (int i = 0; i < 4; i++) x[i] += ks[(j + i) % 5];
            x[3] += j;
        }
    }
    return make_uint4(x[0], x[1], x[2], x[3]);
}

// Rotate-then-xor, two ways. SHF.L.W + LOP3 puts both ops on the ALU pipe;
// IMAD.WIDE.U32 by 2^r yields (x << r, x >> (32-r)) in one FMA-heavy op and a
// single LOP3 folds (lo | hi) ^ y. Threefry is ALU-bound (ncu: ALU 97 %, heavy
// 40 %), so moving a share of its 40 rotations to the multiplier balances the
// two pipes. The multiplier must be a runtime (parameter) value, or the
// compiler turns the multiply back into shifts.
template <bool MUL>
__device__ __forceinline__ uint32_t rotx(uint32_t v, int r, uint32_t p2, uint32_t y) {
    if constexpr (MUL) {
        const uint64_t w = (uint64_t)v * p2;
        return ((uint32_t)w | (uint32_t)(w >> 32)) ^ y;
    } else {
        return rotl32(v, r) ^ y;
    }
}

// Spread NMUL multiplier-rotations evenly over the 40 rotations of a block.
__host__ __device__ constexpr bool tf_mul(int rot, int nmul) { return nmul > 0 && ((rot * nmul) % 40) < nmul; }

// a + b forced onto the FMA-heavy pipe: mad.lo with a multiplier the compiler
// cannot see is 1 (a kernel parameter), so ptxas must emit IMAD, not IADD3.
template <bool FORCE>
__device__ __forceinline__ uint32_t addp(uint32_t a, uint32_t b, uint32_t one) {
    if constexpr (FORCE) {
        uint32_t r;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(one), "r"(a));
        return r;
    } else {
        return a + b;
    }
}

// Key injection J with the adds forced onto the multiplier (ADDMUL); kj3[j] =
// ks[(j+3)%5] + j precomputed, so each injection is exactly four IMADs.
template <int J, bool ADDMUL>
__device__ __forceinline__ void threefry_inject_m(uint32_t &x0, uint32_t &x1, uint32_t &x2, uint32_t &x3,
                                                  const uint32_t ks[5], const uint32_t *kj3, uint32_t one) {
    if constexpr (ADDMUL) {
        x0 = addp<true>(x0, ks[(J + 0) % 5], one);
        x1 = addp<true>(x1, ks[(J + 1) % 5], one);
        x2 = addp<true>(x2, ks[(J + 2) % 5], one);
        x3 = addp<true>(x3, kj3[J], one);
    } else {
        threefry_inject<J>(x0, x1, x2, x3, ks);
    }
}

template <int R, int NMUL, bool ADDMUL>
__device__ __forceinline__ void threefry_round_m(uint32_t &x0, uint32_t &x1, uint32_t &x2, uint32_t &x3,
                                                 const uint32_t *p2, uint32_t one) {
    constexpr int ra = TfRot<R % 8>::a, rb = TfRot<R % 8>::b;
    constexpr bool ma = tf_mul(2 * R, NMUL), mb = tf_mul(2 * R + 1, NMUL);
    if (R % 2 == 0) {
        x0 = addp<ADDMUL>(x0, x1, one); x1 = rotx<ma>(x1, ra, p2[2 * (R % 8)], x0);
        x2 = addp<ADDMUL>(x2, x3, one); x3 = rotx<mb>(x3, rb, p2[2 * (R % 8) + 1], x2);
    } else {
        x0 = addp<ADDMUL>(x0, x3, one); x3 = rotx<ma>(x3, ra, p2[2 * (R % 8)], x0);
        x2 = addp<ADDMUL>(x2, x1, one); x1 = rotx<mb>(x1, rb, p2[2 * (R % 8) + 1], x2);
    }
}

// INJMUL: the key-injection adds forced onto the multiplier as well.
template <int FIRST, int NMUL, bool ADDMUL = false, bool INJMUL = false>
__device__ __forceinline__ void threefry_rounds_m(uint32_t &x0, uint32_t &x1, uint32_t &x2, uint32_t &x3,
                                                  const uint32_t ks[5], const uint32_t *p2, uint32_t one = 1,
                                                  const uint32_t *kj3 = nullptr) {
#define TF_RM(R)                                                                                     \
    if (R >= FIRST) {                                                                                \
        threefry_round_m<R, NMUL, ADDMUL>(x0, x1, x2, x3, p2, one);                                  \
        if ((R + 1) % 4 == 0) threefry_inject_m<(R + 1) / 4, INJMUL>(x0, x1, x2, x3, ks, kj3, one); \
    }
    TF_RM(0) TF_RM(1) TF_RM(2) TF_RM(3) TF_RM(4) TF_RM(5) TF_RM(6) TF_RM(7) TF_RM(8) TF_RM(9)
    TF_RM(10) TF_RM(11) TF_RM(12) TF_RM(13) TF_RM(14) TF_RM(15) TF_RM(16) TF_RM(17) TF_RM(18) TF_RM(19)
#undef TF_RM
}

// Single stream: key (k0, k1, sc, 0), ctr (bc, 0, 0, 0). Rounds 0-1 are mostly
// launch-uniform; the host folds them.
struct ThreefryStream {
    uint32_t ks[5];
    uint32_t s01;   // ks0 + ks1: round 0 x0 = bc + s01
    uint32_t r1;    // rotl(ks1, 10): round 0 x1 = r1 ^ x0
    uint32_t x2_0;  // ks2 + ks3 (round 0 x2)
    uint32_t x3_0;  // rotl(ks3, 26) ^ x2_0 (round 0 x3)
    uint32_t x3r;   // rotl(x3_0, 11) (round 1)
    uint32_t p2[16];  // 2^R[r%8] multipliers for rotx<true>
    uint32_t one;     // 1, opaque to the compiler (addp<true>)
    uint32_t kj3[6];  // ks[(j+3)%5] + j: the x3 term of key injection j
};

__host__ __device__ inline ThreefryStream threefry_stream_setup(uint64_t seed, uint32_t sc) {
    ThreefryStream p;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32), k2 = sc, k3 = 0;
    p.ks[0] = k0; p.ks[1] = k1; p.ks[2] = k2; p.ks[3] = k3;
    p.ks[4] = THREEFRY_PARITY ^ k0 ^ k1 ^ k2 ^ k3;
    p.s01 = p.ks[0] + p.ks[1];
    p.r1 = rotl32(p.ks[1], 10);
    p.x2_0 = p.ks[2] + p.ks[3];
    p.x3_0 = rotl32(p.ks[3], 26) ^ p.x2_0;
    p.x3r = rotl32(p.x3_0, 11);
    const int ROT[8][2] = {{10, 26}, {11, 21}, {13, 27}, {23, 5}, {6, 20}, {17, 11}, {25, 10}, {18, 20}};
    for (int i = 0; i < 8; i++) { p.p2[2 * i] = 1u << ROT[i][0]; p.p2[2 * i + 1] = 1u << ROT[i][1]; }
    p.one = 1;
    for (int j = 0; j < 6; j++) p.kj3[j] = p.ks[(j + 3) % 5] + (uint32_t)j;
    return p;
}

template <int NMUL = 0, bool ADDMUL = false, bool INJMUL = false>
__device__ __forceinline__ uint4 threefry_stream_block(const ThreefryStream& p, uint32_t bc) {
    // round 0 (even; rot 10, 26): x = (bc+ks0, ks1, ks2, ks3)
    uint32_t x0 = bc + p.s01;
    uint32_t x1 = p.r1 ^ x0;
    // x2 = x2_0, x3 = x3_0 (uniform)
    // round 1 (odd; rot 11, 21)
    x0 += p.x3_0;
    uint32_t x3 = p.x3r ^ x0;
    uint32_t x2 = p.x2_0 + x1;
    x1 = rotl32(x1, 21) ^ x2;
    threefry_rounds_m<2, NMUL, ADDMUL, INJMUL>(x0, x1, x2, x3, p.ks, p.p2, p.one, p.kj3);
    return make_uint4(x0, x1, x2, x3);
}

// ---------------------------------------------------------------------------
// Squares (generators.py:157-187)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t squares_key(uint64_t seed) {
    uint64_t s = seed & 0xFFFFFFFFull;
    uint64_t z = s + GOLDEN64;
    z = (z ^ (z >> 30)) * SPLITMIX_M1;
    z = (z ^ (z >> 27)) * SPLITMIX_M2;
    z ^= z >> 31;
    return (z ^ (s << 32)) | 1ull;
}

__host__ __device__ __forceinline__ uint64_t swap32(uint64_t x) { return (x >> 32) | (x << 32); }

__host__ __device__ __forceinline__ uint32_t squares_round(uint64_t key, uint64_t ctr) {
    uint64_t x = ctr * key, y = x, z = y + key;
    x = swap32(x * x + y);
    x = swap32(x * x + z);
    x = swap32(x * x + y);
    return (uint32_t)((x * x + z) >> 32);
}

// One squaring step on 32-bit halves: (h, l) <- swap32((h:l)^2 + a) mod 2^64.
// (h:l)^2 mod 2^64 = l*l + ((2*h*l) << 32). Pipe budget per squaring (the
// kernel is FMA-heavy-bound): one IMAD.WIDE.U32 with the 64-bit addend folded
// in, one IMAD for l*h, and the doubling folded into a 3-input IADD3
// (hi + t + t) on the ALU pipe. Written naturally, ptxas emits l*(h+h) and puts
// about half of the h+h adds on the heavy pipe (profiles/r1h SASS).
__device__ __forceinline__ uint32_t mul_lo_opaque(uint32_t a, uint32_t b) {
    uint32_t t;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(t) : "r"(a), "r"(b));
    return t;
}

__device__ __forceinline__ void squares_sq_swap(uint32_t &h, uint32_t &l, uint64_t a) {
    const uint64_t p = (uint64_t)l * l + a;
    const uint32_t t = mul_lo_opaque(l, h);
    const uint32_t hi = (uint32_t)(p >> 32) + t + t;
    h = (uint32_t)p;  // swap32: the low half becomes the high half
    l = hi;
}

// squares32 from x = ctr*key (generators.py:173-187) on 32-bit halves.
__device__ __forceinline__ uint32_t squares_from_x(uint64_t x, uint64_t key) {
    const uint64_t y = x, z = x + key;
    uint32_t h = (uint32_t)(x >> 32), l = (uint32_t)x;
    squares_sq_swap(h, l, y);
    squares_sq_swap(h, l, z);
    squares_sq_swap(h, l, y);
    // last round: only the high half of x*x + z
    const uint64_t p = (uint64_t)l * l + z;
    const uint32_t t = mul_lo_opaque(l, h);
    return (uint32_t)(p >> 32) + t + t;
}

// Four consecutive counters c..c+3 of one key: x_{k+1} = x_k + key (64-bit add on
// the ALU pipe) instead of another 64-bit multiply.
__device__ __forceinline__ uint64_t add64_opaque(uint64_t a, uint64_t b) {
    // add.cc/addc in inline PTX: the compiler cannot re-associate x0 + key back
    // into (c+1)*key + base (which costs an IMAD.WIDE + IMAD on the FMA-heavy pipe).
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
        : "=r"(lo), "=r"(hi)
        : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint4 squares_x4(uint64_t x0, uint64_t key) {
    const uint64_t x1 = add64_opaque(x0, key), x2 = add64_opaque(x1, key), x3 = add64_opaque(x2, key);
    return make_uint4(squares_from_x(x0, key), squares_from_x(x1, key), squares_from_x(x2, key),
                      squares_from_x(x3, key));
}

// Single stream: ctr = (sc << 32) | bc, so ctr*key = bc*key + ((sc*key_lo) << 32).
struct SquaresStream {
    uint64_t key;
    uint64_t base;  // (sc << 32) * key mod 2^64
    uint64_t k2x2;  // 2 key^2 (squares_x4_inc)
    uint64_t k2x4;  // 4 key^2
    uint64_t ebase; // ((sc << 33) + 1) key^2 + key: E for counter 0
};

inline SquaresStream squares_stream_setup(uint64_t seed, uint32_t sc) {
    SquaresStream p;
    p.key = squares_key(seed);
    p.base = ((uint64_t)sc << 32) * p.key;
    const uint64_t k2 = p.key * p.key;
    p.k2x2 = 2 * k2;
    p.k2x4 = 4 * k2;
    p.ebase = (((uint64_t)sc << 33) + 1) * k2 + p.key;
    return p;
}

// Round 1 of squares32 as a 64-bit value, r = x^2 + x (before its swap).
__device__ __forceinline__ uint64_t squares_r1(uint64_t x) {
    const uint32_t h = (uint32_t)(x >> 32), l = (uint32_t)x;
    const uint64_t p = (uint64_t)l * l + x;
    const uint32_t t = mul_lo_opaque(l, h);
    return ((uint64_t)((uint32_t)(p >> 32) + t + t) << 32) | (uint32_t)p;
}

// Rounds 2-4 from round 1's r (swapped into (h, l) = (lo r, hi r)), y = x, z = x + key.
__device__ __forceinline__ uint32_t squares_rounds_234(uint64_t r, uint64_t y, uint64_t z) {
    uint32_t h = (uint32_t)r, l = (uint32_t)(r >> 32);
    squares_sq_swap(h, l, z);
    squares_sq_swap(h, l, y);
    const uint64_t p = (uint64_t)l * l + z;
    const uint32_t t = mul_lo_opaque(l, h);
    return (uint32_t)(p >> 32) + t + t;
}

// An opaque zero in the constant bank: ptxas cannot fold it, and IADD3 takes
// it as a c[] operand (no register). Tuning-build variants only (squares_x4_inc<true>).
static __constant__ uint32_t c_zero = 0;
// An opaque one, for addp<true> where the stream is set up on the device
// (multi-stream Threefry rows): IMAD takes it as a c[] operand.
static __constant__ uint32_t c_one = 1;

// 64-bit a + b whose high half is a 3-input add against an opaque zero
// (c_zero): ptxas then emits IADD3.X on the ALU pipe. Left as a
// 2-input addc it picks IMAD.X for about half of them, a slot on the
// FMA-heavy pipe that bounds Squares (1.1 of its 12.1 slots per word, r2d).
__device__ __forceinline__ uint64_t add64_alu(uint64_t a, uint64_t b) {
    uint32_t lo, hi;
    asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;\n\tadd.u32 %1, %1, %6;"
        : "=r"(lo), "=r"(hi)
        : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)), "r"(c_zero));
    return ((uint64_t)hi << 32) | lo;
}

// 64-bit a + b + c: one IADD3 (two carries out) and one IADD3.X, both ALU.
__device__ __forceinline__ uint64_t add64_3(uint64_t a, uint64_t b, uint64_t c) {
    uint32_t lo, hi;
    asm("{.reg .u32 t0, t1;\n\tadd.cc.u32 t0, %2, %4;\n\taddc.u32 t1, %3, %5;\n\t"
        "add.cc.u32 %0, t0, %6;\n\taddc.u32 %1, t1, %7;}"
        : "=r"(lo), "=r"(hi)
        : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)),
          "r"((uint32_t)c), "r"((uint32_t)(c >> 32)));
    return ((uint64_t)hi << 32) | lo;
}

// Four consecutive counters with round 1 stepped by finite differences: for
// x_k = x_0 + k key, r_k = x_k^2 + x_k satisfies r_{k+1} = r_k + E_k with
// E_k = 2 key x_k + key^2 + key and E_{k+1} = E_k + 2 key^2 (all mod 2^64), so
// three of the four round-1 squarings (an IMAD.WIDE + IMAD each on the
// FMA-heavy pipe, which bounds Squares) become 64-bit adds on the ALU pipe.
// z_k = x_k + key = x_{k+1}. k2x2 = 2 key^2, k2x4 = 4 key^2; x4_out <- x_4.
// ALUC (tuning build): every carry add forced onto the ALU pipe (add64_alu /
// add64_3: E_1, E_2 folded into 3-input adds). It removes 9 % of the
// FMA-heavy slots (IMAD.X) and measured 2 % slower (profiles/r2k_tune.md).
template <bool ALUC = false>
__device__ __forceinline__ uint4 squares_x4_inc(uint64_t x0, uint64_t e0, uint64_t key, uint64_t k2x2, uint64_t k2x4,
                                                uint64_t *x4_out = nullptr) {
    uint64_t x1, x2, x3, x4, r1, r2, r3;
    const uint64_t r0 = squares_r1(x0);
    if constexpr (ALUC) {
        x1 = add64_alu(x0, key), x2 = add64_alu(x1, key), x3 = add64_alu(x2, key), x4 = add64_alu(x3, key);
        r1 = add64_alu(r0, e0), r2 = add64_3(r1, e0, k2x2), r3 = add64_3(r2, e0, k2x4);
    } else {
        x1 = add64_opaque(x0, key), x2 = add64_opaque(x1, key), x3 = add64_opaque(x2, key), x4 = add64_opaque(x3, key);
        const uint64_t e1 = add64_opaque(e0, k2x2), e2 = add64_opaque(e1, k2x2);
        r1 = add64_opaque(r0, e0), r2 = add64_opaque(r1, e1), r3 = add64_opaque(r2, e2);
    }
    if (x4_out) *x4_out = x4;
    return make_uint4(squares_rounds_234(r0, x0, x1), squares_rounds_234(r1, x1, x2), squares_rounds_234(r2, x2, x3),
                      squares_rounds_234(r3, x3, x4));
}

__device__ __forceinline__ uint32_t squares_stream_word(const SquaresStream &p, uint32_t bc) {
    return squares_from_x((uint64_t)bc * p.key + p.base, p.key);
}

// Words bc..bc+3 (counters wrap mod 2^32 in the low half only, bulk.py:268): the
// incremental form is exact unless bc+k wraps, which the caller checks.
template <bool NOWRAP = false>
__device__ __forceinline__ uint4 squares_stream_word4(const SquaresStream &p, uint32_t bc) {
    if (!NOWRAP && bc > 0xFFFFFFFCu) {
        return make_uint4(squares_stream_word(p, bc), squares_stream_word(p, bc + 1), squares_stream_word(p, bc + 2),
                          squares_stream_word(p, bc + 3));
    }
    return squares_x4((uint64_t)bc * p.key + p.base, p.key);
}

// ---------------------------------------------------------------------------
// Tyche (generators.py:190-224)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ void tyche_mix(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
    a += b; d = rotl32(d ^ a, 16);
    c += d; b = rotl32(b ^ c, 12);
    a += b; d = rotl32(d ^ a, 8);
    c += d; b = rotl32(b ^ c, 7);
}

// The same mix for a single serial chain (latency-bound): the adds carry an
// opaque zero third operand, so ptxas emits 3-input IADD3 on the ALU pipe
// instead of IMAD.IADD on the FMA pipe, and the 12-op dependency chain never
// pays the cross-pipe latency (+1 cycle per pipe switch, 8 per mix).
__device__ __forceinline__ uint32_t add3z(uint32_t a, uint32_t b, uint32_t z) {
    uint32_t r;
    asm("add.u32 %0, %1, %2;\n\tadd.u32 %0, %0, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(z));
    return r;
}

__device__ __forceinline__ void tyche_mix_alu(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d, uint32_t z) {
    a = add3z(a, b, z); d = rotl32(d ^ a, 16);
    c = add3z(c, d, z); b = rotl32(b ^ c, 12);
    a = add3z(a, b, z); d = rotl32(d ^ a, 8);
    c = add3z(c, d, z); b = rotl32(b ^ c, 7);
}

__host__ __device__ __forceinline__ uint4 tyche_init(uint64_t seed, uint32_t sc) {
    uint32_t a = (uint32_t)(seed >> 32), b = (uint32_t)seed, c = TYCHE_INIT_CONST, d = sc;
#pragma unroll 4
    for (int i = 0; i < 20; i++) tyche_mix(a, b, c, d);
    return make_uint4(a, b, c, d);
}

// ---------------------------------------------------------------------------
// Word -> variate maps (distributions.py:42-120), exact where the reference is.
// ---------------------------------------------------------------------------
// uniform_f32: (w >> 8) * 2^-24 (exact in float; the reference rounds
// (w>>8)*2^-24 in double then casts, which is the same value).
__device__ __forceinline__ float u32_to_f32(uint32_t w) { return (float)(w >> 8) * 0x1p-24f; }

// Same map with no FP multiply: float(m) for m = w >> 8 < 2^24 is exact, and
// scaling by 2^-24 is an exponent decrement (bits - (24 << 23)) for m != 0; the
// signed max with 0 maps m = 0 to +0.0f. Three ALU ops instead of an FMUL on the
// FMA-heavy pipe — used by the heavy-bound Squares fill.
__device__ __forceinline__ float u32_to_f32_alu(uint32_t w) {
    const int b = __float_as_int((float)(w >> 8)) - (24 << 23);
    return __int_as_float(max(b, 0));
}

// Same map with the shift done as hi(w * 2^24) on the FMA-heavy pipe instead of
// SHF on the ALU pipe, for ALU-bound generators (Threefry, Tyche). `m24` must
// be the runtime value 1 << 24 (a kernel parameter), or the compiler folds the
// multiply back into a shift.
__device__ __forceinline__ float u32_to_f32_mul(uint32_t w, uint32_t m24) {
    return (float)__umulhi(w, m24) * 0x1p-24f;
}

// int -> float on the XU pipe. For m < 2^24 every rounding mode gives the
// exact value; ptxas lowers the directed-rounding cvt to the legacy I2F (XU,
// otherwise idle in these kernels) where cvt.rn becomes I2FP on the ALU pipe.
__device__ __forceinline__ float u24_to_f32_xu(uint32_t m) {
    float f;
    asm("cvt.rm.f32.u32 %0, %1;" : "=f"(f) : "r"(m));
    return f;
}

// The exact map (w >> 8) * 2^-24, with its three steps (shift, convert, scale)
// placed on whichever pipes a kernel has spare (profiles/r1r_tune.md):
//   CV 0: SHF (alu)       + I2FP (alu) + FMUL (fma)
//   CV 1: IMAD.HI (heavy) + I2FP (alu) + FMUL (fma)      [u32_to_f32_mul]
//   CV 2: SHF (alu)       + I2FP (alu) + exponent IADD + max (alu)
//   CV 3: IMAD.HI (heavy) + I2F (xu)   + FMUL (fma)
//   CV 4: SHF (alu)       + I2F (xu)   + FMUL (fma)
//   CV 5: SHF (alu)       + I2F (xu)   + exponent IADD + max (alu)
template <int CV>
__device__ __forceinline__ float u32_to_f32_cv(uint32_t w, uint32_t m24) {
    if constexpr (CV == 0) {
        return u32_to_f32(w);
    } else if constexpr (CV == 1) {
        return u32_to_f32_mul(w, m24);
    } else if constexpr (CV == 2) {
        return u32_to_f32_alu(w);
    } else if constexpr (CV == 3) {
        return u24_to_f32_xu(__umulhi(w, m24)) * 0x1p-24f;
    } else if constexpr (CV == 4) {
        return u24_to_f32_xu(w >> 8) * 0x1p-24f;
    } else {
        const int b = __float_as_int(u24_to_f32_xu(w >> 8)) - (24 << 23);
        return __int_as_float(max(b, 0));
    }
}

template <int CV>
__device__ __forceinline__ float4 u32x4_to_f32x4(uint4 w, uint32_t m24) {
    return make_float4(u32_to_f32_cv<CV>(w.x, m24), u32_to_f32_cv<CV>(w.y, m24), u32_to_f32_cv<CV>(w.z, m24),
                       u32_to_f32_cv<CV>(w.w, m24));
}

// uniform_f64: ((lo | hi<<32) >> 11) * 2^-53, low word first.
__device__ __forceinline__ double u32x2_to_f64(uint32_t lo, uint32_t hi) {
    uint64_t u = ((uint64_t)hi << 32) | lo;
    return (double)(u >> 11) * 0x1p-53;
}

// Box-Muller (distributions.py:72-81, :110-120): u1 = 1 - f64(w0,w1), u2 = f64(w2,w3),
// r = sqrt(-2 ln u1), (r cos(2pi u2), r sin(2pi u2)). The argument is the
// ROUNDED product (2*pi)*u2, exactly as the reference forms it.
__device__ __forceinline__ void box_muller(uint4 w, double& z0, double& z1) {
    const double two_pi = 6.283185307179586;  // 2.0 * math.pi, rounded
    double u1 = 1.0 - u32x2_to_f64(w.x, w.y);
    double u2 = u32x2_to_f64(w.z, w.w);
    double r = sqrt(-2.0 * log(u1));
    double t = __dmul_rn(two_pi, u2);
    double s, c;
    sincos(t, &s, &c);
    z0 = __dmul_rn(r, c);
    z1 = __dmul_rn(r, s);
}

}  // namespace cbrng
