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
// the r1 libm-style version). About 39 FP64 instructions per pair, from 63:
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
//   t:    (2 pi 2^-53) * f64(u2 bits): the same rounded value as (2 pi) * u2
//         (scaling by 2^-53 is exact on both sides), one DMUL.
//   sincos: quadrant from the integer u2, 2-term Cody-Waite reduction by
//         pi/2 with DFMA, fdlibm k_sin / k_cos minimax kernels on |x| <= pi/4;
//         cos as fma(x^4, C(x^2), 1 - x^2/2) without fdlibm's extra
//         compensation (the tolerance allows it): 18 ops.
#pragma once
#include <cstdint>

#include "cbrng_logtab.h"

namespace cbrng {

struct BmConst {
    double s[6];
    double c[6];
    double pio2_hi, pio2_lo;
    double m2ln2_hi, m2ln2_lo;  // -2 ln2 split: ln2_hi a multiple of 2^-43
    double two_pi_2m53;         // (2 pi) * 2^-53, exact scaling of the rounded 2*math.pi
};

__constant__ BmConst c_bm = {
    {-1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
     2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10},
    {4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
     -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11},
    1.57079632679489655800e+00, 6.12323399573676603587e-17,
    -2.0 * 0x1.62e42fefa3800p-1, -2.0 * 0x1.ef35793c7673p-45,
    6.283185307179586 * 0x1p-53,
};

// {-2 invc, -2 logc hi, -2 logc lo, 0} per subinterval (tools/gen_logtab.py).
constexpr int BM_LOGTAB_N = 256;
__constant__ double4 c_logtab[BM_LOGTAB_N] = CBRNG_LOGTAB_INIT;

// Fill kernels read the table from shared memory (divergent indices would
// serialise constant-bank reads); a CTA stages it once.
__device__ __forceinline__ void bm_stage_table(double4 *s_tab) {
    const double2 *src = reinterpret_cast<const double2 *>(c_logtab);
    double2 *dst = reinterpret_cast<double2 *>(s_tab);
    for (uint32_t i = threadIdx.x; i < 2 * BM_LOGTAB_N; i += blockDim.x) dst[i] = src[i];
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

// -2 ln(v 2^-53) for an integer v in [1, 2^53].
__device__ __forceinline__ double bm_m2log(uint64_t v, const double4 *tab) {
    const double dv = u64_to_f64_xu(v);  // exact: v < 2^54
    const uint32_t hi = (uint32_t)__double2hiint(dv);
    const uint32_t th = hi - 0x3fe60000u;            // bits(dv) - bits(0.6875); the low word of OFF is 0
    const int k = ((int)th >> 20) - 53;              // dv = 2^(k+53) z
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

// sin(t), cos(t) for t = (2 pi) u2 in [0, 2 pi), u2 = v 2^-53. The quadrant
// q = round(4 u2) comes from the integer v (XU conversion, no FP64 ops); x =
// t - q pi/2 is then within pi/4 of 0 up to t's rounding, where the fdlibm
// kernels are accurate.
__device__ __forceinline__ void sincos_2pi(double t, uint64_t v, double &sn, double &cs) {
    const int qlo = (int)((v + (1ull << 50)) >> 51);  // 0..4
    const double q = (double)qlo;
    double x = fma(-q, c_bm.pio2_hi, t);
    x = fma(-q, c_bm.pio2_lo, x);
    const double z = x * x;
    // fdlibm k_sin: x + x*z*(S1 + z*r)
    const double rs = fma(z, fma(z, fma(z, fma(z, c_bm.s[5], c_bm.s[4]), c_bm.s[3]), c_bm.s[2]), c_bm.s[1]);
    const double sx = fma(x * z, fma(z, rs, c_bm.s[0]), x);
    // cos: 1 - z/2 + z^2 C(z)
    const double rc =
        fma(z, fma(z, fma(z, fma(z, fma(z, c_bm.c[5], c_bm.c[4]), c_bm.c[3]), c_bm.c[2]), c_bm.c[1]), c_bm.c[0]);
    const double cx = fma(z * z, rc, fma(z, -0.5, 1.0));
    // quadrant: odd q swaps sin/cos; the signs are xor-ed into the high words
    const bool odd = qlo & 1;
    const double a = odd ? cx : sx;  // |sin(t)| up to sign
    const double b = odd ? sx : cx;  // |cos(t)| up to sign
    const int ssgn = (qlo << 30) & 0x80000000;        // q & 2
    const int csgn = ((qlo + 1) << 30) & 0x80000000;  // (q + 1) & 2
    sn = __hiloint2double(__double2hiint(a) ^ ssgn, __double2loint(a));
    cs = __hiloint2double(__double2hiint(b) ^ csgn, __double2loint(b));
}

// One Box-Muller pair from one 4-word block; `tab` = c_logtab staged in shared
// memory (fill kernels) or c_logtab itself (single-thread kernels).
__device__ __forceinline__ void box_muller_fast(uint4 w, double &z0, double &z1, const double4 *tab) {
    const uint64_t u = (((uint64_t)w.y << 32) | w.x) >> 11;
    const uint64_t u2 = (((uint64_t)w.w << 32) | w.z) >> 11;
    const double r = bm_sqrt(bm_m2log((1ull << 53) - u, tab));
    double s, c;
    sincos_2pi(c_bm.two_pi_2m53 * u64_to_f64_xu(u2), u2, s, c);
    z0 = __dmul_rn(r, c);
    z1 = __dmul_rn(r, s);
}

}  // namespace cbrng
