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
// the r1 libm-style version). About 35 FP64 instructions per pair, from 63:
//   u1:   never formed. f64(w0,w1) = u 2^-53 with u = (w >> 11), so
//         u1 = v 2^-53, v = 2^53 - u an integer in [1, 2^53]: one 64-bit
//         integer subtract and one I2F (XU pipe); the 2^-53 goes into the
//         exponent k of the log.
//   -2 ln u1: table-driven (cbrng_logtab.h, tools/gen_logtab.py): v = 2^k z,
//         z in [0.6875, 1.375), 256 subintervals with (-2 invc, -2 logc as
//         hi + lo); s = -2 r = fma(z, -2 invc, 2) exact-ish, |s| <= 2^-8,
//         -2 ln(1+r) = s + s^2 (1/4 + s/12 + s^2/32 + s^3/80 + s^4/192)
//         (the series 2 sum (s/2)^n / n, truncation < 2^-56 relative); the
//         sum k(-2 ln2_hi) + hi is exact, lo and k(-2 ln2_lo) are added to the
//         small part: 11 FP64 ops instead of ~25 for the fdlibm form with a
//         Newton reciprocal. The subinterval just below 1 uses invc = 1, so
//         r = z - 1 is exact and ln u1 keeps full relative accuracy as u1 -> 1.
//   sqrt: MUFU.RSQ64H seed, one Newton step for sqrt, one residual
//         correction with the seed's 1/(2 sqrt): 7 ops.
//   t:    (2 pi 2^-64) * f64(u2 2^11): the same rounded value as (2 pi) * u2
//         (scaling by powers of two is exact on both sides), one DMUL.
//   sincos: table point j = round(128 u2) from the integer u2, reduction by
//         j pi/64, short Taylor sin/cos on |x| <= pi/128 and the angle sum with
//         a 129-entry {sin, cos}(j pi/64) table: 14 ops.
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

// {-2 invc, -2 logc hi, -2 logc lo, 0} per subinterval (tools/gen_logtab.py).
constexpr int BM_LOGTAB_N = 256;
__constant__ double4 c_logtab[BM_LOGTAB_N] = CBRNG_LOGTAB_INIT;

// {sin, cos}(j pi/64), j = 0..128 (tools/gen_logtab.py).
constexpr int BM_SCTAB_N = 129;
__constant__ double2 c_sctab[BM_SCTAB_N] = CBRNG_SINCOSTAB_INIT;

// Both tables in shared memory: divergent indices would serialise constant-bank
// reads. A CTA stages them once.
struct BmTables {
    double4 log[BM_LOGTAB_N];
    double2 sc[BM_SCTAB_N];
};

__device__ __forceinline__ void bm_stage_table(BmTables *t) {
    const double2 *src = reinterpret_cast<const double2 *>(c_logtab);
    double2 *dst = reinterpret_cast<double2 *>(t->log);
    for (uint32_t i = threadIdx.x; i < 2 * BM_LOGTAB_N; i += blockDim.x) dst[i] = src[i];
    for (uint32_t i = threadIdx.x; i < BM_SCTAB_N; i += blockDim.x) t->sc[i] = c_sctab[i];
    __syncthreads();
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
template <int E = 53>
__device__ __forceinline__ double bm_m2log_d(double dv, const double4 *tab) {
    const uint32_t hi = (uint32_t)__double2hiint(dv);
    const uint32_t th = hi - 0x3fe60000u;            // bits(dv) - bits(0.6875); the low word of OFF is 0
    const int k = ((int)th >> 20) - E;               // dv = 2^(k+E) z
    const uint32_t i = (th >> 12) & 255u;            // top 8 mantissa bits of bits(dv) - OFF
    const double z = __hiloint2double((int)(hi - (th & 0xfff00000u)), __double2loint(dv));
    const double4 e = tab[i];
    const double kd = (double)k;
    const double s = fma(z, e.x, 2.0);                 // -2 r
    const double w = fma(kd, c_bm.m2ln2_hi, e.y);      // exact
    double p = fma(s, 1.0 / 192, 1.0 / 80);
    p = fma(s, p, 1.0 / 32);
    p = fma(s, p, 1.0 / 12);
    p = fma(s, p, 1.0 / 4);
    const double q = fma(s * s, p, s);
    return w + fma(kd, c_bm.m2ln2_lo, q + e.z);
}


// sqrt(a), a >= 0 finite. a = 0 (u1 == 1) must give 0: the rsqrt input is
// clamped to the smallest normal on the high word (one integer max, no FP
// compare/select), so y stays finite and r = 0 exactly.
__device__ __forceinline__ double bm_sqrt(double a) {
    const double ac = __hiloint2double(max(__double2hiint(a), 0x00100000), __double2loint(a));
    const double y0 = rsqrt_approx(ac);
    const double h0 = 0.5 * y0, t = a * y0, g = a * h0;
    const double e = fma(-t, y0, 1.0);  // 1 - a y0^2
    const double r1 = fma(g, e, t);     // sqrt(a), ~2x the seed's bits
    // residual correction; the seed's 1/(2 sqrt a) suffices: its error only
    // scales the ~2^-46 residual
    return fma(h0, fma(-r1, r1, a), r1);
}

// sin(t), cos(t) for t = (2 pi) u2 in [0, 2 pi), u2 = v 2^-53. The table
// point j = round(128 u2) comes from the integer v (no FP64 op); x = t - j pi/64
// (2-term Cody-Waite, |x| <= pi/128 up to t's rounding); sin x and cos x by
// short Taylor polynomials (truncation < 2^-60 on that range); then the angle
// sum with the table's sin/cos of j pi/64, which are exact zeros and ones at
// the multiples of pi/2, so results next to a zero keep their relative
// accuracy. 14 FP64 ops (the fdlibm-kernel form with a pi/2 reduction: 18).
__device__ __forceinline__ void sincos_2pi(double t, uint32_t w3, const double2 *sct, double &sn, double &cs) {
    // j = round(128 u2) = (u2 + 2^45) >> 46 with u2 = (w3:w2) >> 11, from the high word alone
    const int j = (int)(((w3 >> 24) + 1u) >> 1);  // 0..128
    const double jd = (double)j;
    double x = fma(-jd, CBRNG_PI64_HI, t);
    x = fma(-jd, CBRNG_PI64_LO, x);
    const double z = x * x;
    const double ps = fma(z, fma(z, -1.0 / 5040, 1.0 / 120), -1.0 / 6);
    const double s = fma(x * z, ps, x);
    const double pc = fma(z, fma(z, -1.0 / 720, 1.0 / 24), -0.5);
    const double c = fma(z, pc, 1.0);
    const double2 a = sct[j];  // {sin, cos}(j pi/64)
    sn = fma(a.x, c, a.y * s);
    cs = fma(a.y, c, -(a.x * s));
}

// One Box-Muller pair from one 4-word block; `tab` = the tables staged in shared
// memory (bm_stage_table).
//   With m = (w1:w0) with the low 11 bits cleared = u 2^11 (exact in f64),
//   v 2^11 = (2^53 - u) 2^11 = 2^64 - m, a multiple of 2^11 in [2^11, 2^64]: one
//   exact DADD. One LOP3 + I2F + DADD instead of two 64-bit shifts, a 64-bit
//   subtract and the I2F; the log takes the 2^11 into its exponent.
//   u2 2^11 = (w3:w2) with the low 11 bits cleared converts exactly, and
//   (2 pi 2^-64) (u2 2^11) rounds exactly like (2 pi) (u2 2^-53).
__device__ __forceinline__ void box_muller_fast(uint4 w, double &z0, double &z1, const BmTables *tab) {
    const uint64_t m1 = ((uint64_t)w.y << 32) | (w.x & 0xFFFFF800u);  // u 2^11
    const uint64_t m2 = ((uint64_t)w.w << 32) | (w.z & 0xFFFFF800u);  // u2 2^11
    const double r = bm_sqrt(bm_m2log_d<64>(__dsub_rn(0x1p64, u64_to_f64_xu(m1)), tab->log));
    double s, c;
    sincos_2pi(c_bm.two_pi_2m64 * u64_to_f64_xu(m2), w.w, tab->sc, s, c);
    z0 = __dmul_rn(r, c);
    z1 = __dmul_rn(r, s);
}

}  // namespace cbrng
