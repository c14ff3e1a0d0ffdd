// cbrng_bm.cuh — Box-Muller on the FP64 pipe with domain-restricted math.
//
// distributions.py:72-81/110-120: u1 = 1 - f64(w0,w1) in [2^-53, 1],
// u2 = f64(w2,w3) in [0, 1), r = sqrt(-2 ln u1), t = (2*pi)*u2 (the rounded
// product, as the reference forms it), z = (r cos t, r sin t).
//
// The FP64 pipe bounds this kernel (ncu r1q: math-pipe throttle and
// not-selected are half the stall samples), so the design goal is the fewest
// FP64 instructions per pair at the accuracy the parity tests demand
// (<= 4 ulp(max(|z|,1)) of glibc; 3 is the worst seen over 4e7 random pairs
// in the host prototype of exactly these formulas, fewer 3-ulp cases than
// the r1 libm-style version). About 32 FP64 instructions per pair, from 63:
//   u1:   never formed. f64(w0,w1) = u 2^-53 with u = (w >> 11), so
//         u1 = v 2^-53, v = 2^53 - u an integer in [1, 2^53]: one 64-bit
//         integer subtract and one I2F (XU pipe); the 2^-53 goes into the
//         exponent k of the log.
//   -2 ln u1: table-driven (cbrng_logtab.h, tools/gen_logtab.py): v = 2^k z,
//         z in [0.6875, 1.375), 256 subintervals with (-2 invc, -2 logc), invc
//         chosen so that -2 logc is a multiple of 2^-43 to within 2^-66 (Gal's
//         accurate tables); s = -2 r = fma(z, -2 invc, 2) exact-ish, |s| <= 2^-8,
//         -2 ln(1+r) = s + s^2 (1/4 + s/12 + s^2/32 + s^3/80 + s^4/192)
//         (the series 2 sum (s/2)^n / n, truncation < 2^-56 relative); the
//         sum k(-2 ln2_hi) + (-2 logc) is exact, k(-2 ln2_lo) is added to the
//         small part: 10 FP64 ops instead of ~25 for the fdlibm form with a
//         Newton reciprocal. The two subintervals around 1 use invc = 1, so
//         r = z - 1 is exact, ln u1 keeps full relative accuracy as u1 -> 1
//         and u1 = 1 gives exactly 0.
//   sqrt: MUFU.RSQ64H seed, two Heron corrections with the seed's
//         1/(2 sqrt): 6 ops.
//   t:    (2 pi 2^-64) * f64(u2 2^11): the same rounded value as (2 pi) * u2
//         (scaling by powers of two is exact on both sides), one DMUL.
//   sincos: table point j = round(1024 u2) from the integer u2, reduction by
//         j pi/512, short Taylor sin/cos on |x| <= pi/1024 and the angle sum
//         with a 1025-entry {sin, cos}(j pi/512) table: 12 ops.
#pragma once
#include <cstdint>

#include "cbrng_logtab.h"

namespace cbrng {

struct BmConst {
    double m2ln2_hi, m2ln2_lo;  // -2 ln2 split: ln2_hi a multiple of 2^-43
    double two_pi_2m53;         // (2 pi) * 2^-53, exact scaling of the rounded 2*math.pi
    double two_pi_2m64;         // (2 pi) * 2^-64
};

__constant__ BmConst c_bm = {
    -2.0 * 0x1.62e42fefa3800p-1, -2.0 * 0x1.ef35793c7673p-45,
    6.283185307179586 * 0x1p-53, 6.283185307179586 * 0x1p-64,
};

// {-2 invc, -2 logc} per subinterval, |-2 logc - 2 ln invc| < 2^-66 (Gal's
// accurate tables, tools/gen_logtab.py): 16 bytes, one LDS.128 per lookup.
constexpr int BM_LOGTAB_N = 256;
__constant__ double2 c_logtab[BM_LOGTAB_N] = CBRNG_LOGTAB_INIT;

// {sin, cos}(j pi/512), j = 0..1024 (tools/gen_logtab.py).
constexpr int BM_SCTAB_N = 2 * CBRNG_SINCOS_NSC + 1;
__constant__ double2 c_sctab[BM_SCTAB_N] = CBRNG_SINCOSTAB_INIT;

// Both tables in shared memory (divergent indices would serialise constant-bank
// reads), staged once per CTA. The two random-index LDS.128 per pair bound the
// fused fill when the tables are stored once (ncu r2d: LSU data pipe 94 %,
// 3.8x the conflict-free wavefronts): a 128-bit shared load is served a
// quarter-warp (8 lanes, 128 B) per wavefront, so 8 lanes hitting the same
// 16-byte bank group serialise. LC / SC copies of each table are interleaved
// entry-major (entry e of copy c at index e*C + c) and lane l reads copy
// l mod C: with C = 8 the 8 lanes of every quarter-warp hit 8 distinct bank
// groups, 4 wavefronts per LDS.128 instead of ~10.
template <int LC = 1, int SC = 1>
struct BmTables {
    double2 log[BM_LOGTAB_N * LC];
    double2 sc[BM_SCTAB_N * SC];
};

// A lane's view of its copies (entry e at log[e * LC], sc[e * SC]).
template <int LC = 1, int SC = 1>
struct BmView {
    const double2 *log;
    const double2 *sc;
};

template <int LC, int SC>
__device__ __forceinline__ BmView<LC, SC> bm_stage_table(BmTables<LC, SC> *t) {
    for (uint32_t i = threadIdx.x; i < BM_LOGTAB_N * LC; i += blockDim.x) t->log[i] = c_logtab[i / LC];
    for (uint32_t i = threadIdx.x; i < BM_SCTAB_N * SC; i += blockDim.x) t->sc[i] = c_sctab[i / SC];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    return {t->log + (lane & (LC - 1)), t->sc + (lane & (SC - 1))};
}

__device__ __forceinline__ double rsqrt_approx(double a) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    return y;
}

__device__ __forceinline__ double u64_to_f64_xu(uint64_t v) {
    double d;
    asm("cvt.rn.f64.u64 %0, %1;" : "=d"(d) : "l"(v));
    return d;
}

// -2 ln(dv 2^-E) for dv = v 2^(E-53), v an integer in [1, 2^53] (dv exact).
// w = k (-2 ln2_hi) + (-2 logc) is exact; the table's -2 logc is within 2^-66
// of 2 ln invc, so no low-order table term is added.
template <int E = 53, int LC = 1>
__device__ __forceinline__ double bm_m2log_d(double dv, const double2 *tab) {
    const uint32_t hi = (uint32_t)__double2hiint(dv);
    const uint32_t th = hi - 0x3fe60000u;            // bits(dv) - bits(0.6875); the low word of OFF is 0
    const int k = ((int)th >> 20) - E;               // dv = 2^(k+E) z
    const uint32_t i = (th >> 12) & 255u;            // top 8 mantissa bits of bits(dv) - OFF
    const double z = __hiloint2double((int)(hi - (th & 0xfff00000u)), __double2loint(dv));
    const double2 e = tab[i * LC];
    const double kd = (double)k;
    const double s = fma(z, e.x, 2.0);                 // -2 r
    const double w = fma(kd, c_bm.m2ln2_hi, e.y);      // exact
    double p = fma(s, 1.0 / 192, 1.0 / 80);
    p = fma(s, p, 1.0 / 32);
    p = fma(s, p, 1.0 / 12);
    p = fma(s, p, 1.0 / 4);
    const double q = fma(s * s, p, s);
    return w + fma(kd, c_bm.m2ln2_lo, q);
}

// sqrt(a), a >= 0 finite: two Heron corrections r <- r + (a - r^2) y0/2 from
// t = a y0, both with the seed's half-reciprocal h = y0/2 (its error eps only
// scales the residual: after two steps the relative error is ~1.5 eps^3,
// eps <= 2^-20 for the high-word seed): 6 FP64 ops. a = 0 (u1 == 1) must give
// 0: the rsqrt input is clamped to the smallest normal on the high word (one
// integer max, no FP compare/select), so y0 stays finite and r = 0 exactly.
__device__ __forceinline__ double bm_sqrt(double a) {
    const double ac = __hiloint2double(max(__double2hiint(a), 0x00100000), __double2loint(a));
    const double y0 = rsqrt_approx(ac);
    const double h = 0.5 * y0, t = a * y0;
    const double r1 = fma(h, fma(-t, t, a), t);
    return fma(h, fma(-r1, r1, a), r1);
}

// sin(t), cos(t) for t = (2 pi) u2 in [0, 2 pi), u2 = v 2^-53. The table
// point j = round(1024 u2) comes from the integer v (no FP64 op); x = t - j pi/512
// (2-term Cody-Waite, |x| <= pi/1024 up to t's rounding); sin x = x + x^3 (-1/6 +
// x^2/120) and cos x = 1 + x^2 (-1/2 + x^2/24) (the next terms are below
// 2^-61 relative on that range); then the angle sum with the table's
// {sin, cos}(j pi/512), which are exact zeros and ones at the multiples of
// pi/2, so results next to a zero keep their relative accuracy. 12 FP64 ops
// (a pi/64 table needs a degree higher: 14; the fdlibm-kernel form with a
// pi/2 reduction: 18). Host prototype over 3e7 random pairs against glibc:
// max 3 ulp(max(|z|,1)) and 3 ulp of z, as with the pi/64 table.
template <int SC = 1>
__device__ __forceinline__ void sincos_2pi(double t, uint32_t w3, const double2 *sct, double &sn, double &cs) {
    static_assert(CBRNG_SINCOS_NSC == 512, "table step pi/512");
    // j = round(1024 u2) = (u2 + 2^42) >> 43 with u2 = (w3:w2) >> 11, from the high word alone
    const int j = (int)(((w3 >> 21) + 1u) >> 1);  // 0..1024
    const double jd = (double)j;
    double x = fma(-jd, CBRNG_PIN_HI, t);
    x = fma(-jd, CBRNG_PIN_LO, x);
    const double z = x * x;
    const double s = fma(x * z, fma(z, 1.0 / 120, -1.0 / 6), x);
    const double c = fma(z, fma(z, 1.0 / 24, -0.5), 1.0);
    const double2 a = sct[j * SC];  // {sin, cos}(j pi/512)
    sn = fma(a.x, c, a.y * s);
    cs = fma(a.y, c, -(a.x * s));
}

// One Box-Muller pair from one 4-word block; `v` = the lane's view of the
// tables staged in shared memory (bm_stage_table).
//   With m = (w1:w0) with the low 11 bits cleared = u 2^11 (exact in f64),
//   v 2^11 = (2^53 - u) 2^11 = 2^64 - m, a multiple of 2^11 in [2^11, 2^64]: one
//   exact DADD. One LOP3 + I2F + DADD instead of two 64-bit shifts, a 64-bit
//   subtract and the I2F; the log takes the 2^11 into its exponent.
//   u2 2^11 = (w3:w2) with the low 11 bits cleared converts exactly, and
//   (2 pi 2^-64) (u2 2^11) rounds exactly like (2 pi) (u2 2^-53).
template <int LC, int SC>
__device__ __forceinline__ void box_muller_fast(uint4 w, double &z0, double &z1, const BmView<LC, SC> &v) {
    const uint64_t m1 = ((uint64_t)w.y << 32) | (w.x & 0xFFFFF800u);  // u 2^11
    const uint64_t m2 = ((uint64_t)w.w << 32) | (w.z & 0xFFFFF800u);  // u2 2^11
    const double r = bm_sqrt(bm_m2log_d<64, LC>(__dsub_rn(0x1p64, u64_to_f64_xu(m1)), v.log));
    double s, c;
    sincos_2pi<SC>(c_bm.two_pi_2m64 * u64_to_f64_xu(m2), w.w, v.sc, s, c);
    z0 = __dmul_rn(r, c);
    z1 = __dmul_rn(r, s);
}

}  // namespace cbrng
