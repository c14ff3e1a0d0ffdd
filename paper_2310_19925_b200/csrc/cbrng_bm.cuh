// cbrng_bm.cuh — Box-Muller on the FP64 pipe with domain-restricted math.
//
// distributions.py:72-81/110-120: u1 = 1 - f64(w0,w1) in [2^-53, 1],
// u2 = f64(w2,w3) in [0, 1), r = sqrt(-2 ln u1), t = (2*pi)*u2 (the rounded
// product, as the reference forms it), z = (r cos t, r sin t).
//
// CUDA's libm log/sincos are general-purpose: special-value branches, a
// Payne-Hanek slow path for huge arguments, and 64-bit constants materialised
// through uniform/regular register moves (ncu r1a: ~240 instructions per pair,
// FP64 pipe 40 %). Here the arguments are known to be finite, positive and
// small, so each function is a straight-line polynomial evaluation with
// constants read from the constant bank:
//   log:   x = 2^k m, m in [sqrt(1/2), sqrt(2)); log(m) by the classic
//          s = f/(2+f) atanh-series form (Sun fdlibm e_log.c minimax
//          coefficients Lg1..Lg7, < 1 ulp), reciprocal via MUFU.RCP64H + Newton;
//   sqrt:  MUFU.RSQ64H + Newton, one residual correction;
//   sincos: 2-term Cody-Waite reduction by pi/2 (t < 2*pi, quadrant <= 4) with
//          DFMA, fdlibm k_sin/k_cos minimax kernels on |x| <= pi/4.
// Accuracy vs glibc (bit-identical to the reference's scalar normal2): within
// the 4 ulp(max(|z|,1)) bound the parity tests assert; the measured maximum is
// reported by tests/test_gpu_parity.py::TestDistributions.
#pragma once
#include <cstdint>

namespace cbrng {

struct BmConst {
    double lg[7];
    double ln2_hi, ln2_lo;
    double s[6];
    double c[6];
    double two_over_pi, pio2_hi, pio2_lo;
};

__constant__ BmConst c_bm = {
    {6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01, 2.222219843214978396e-01,
     1.818357216161805012e-01, 1.531383769920937332e-01, 1.479819860511658591e-01},
    6.93147180369123816490e-01, 1.90821492927058770002e-10,
    {-1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
     2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10},
    {4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
     -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11},
    6.36619772367581382433e-01, 1.57079632679489655800e+00, 6.12323399573676603587e-17,
};

__device__ __forceinline__ double rcp_approx(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    return y;
}

__device__ __forceinline__ double rsqrt_approx(double a) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    return y;
}

// ln(x) for x in [2^-53, 1] (positive, normal, finite).
__device__ __forceinline__ double log_unit(double x) {
    int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    int k = (hi >> 20) - 1023;
    int mh = (hi & 0x000FFFFF) | 0x3FF00000;  // m in [1, 2)
    if ((hi & 0x000FFFFF) > 0x6A09E) {        // m > ~sqrt(2): use m/2, k+1
        mh -= 0x00100000;
        k += 1;
    }
    const double f = __hiloint2double(mh, lo) - 1.0;  // exact
    const double d = 2.0 + f;
    double y = rcp_approx(d);
    y = fma(y, fma(-d, y, 1.0), y);
    y = fma(y, fma(-d, y, 1.0), y);
    const double s = f * y;  // f / (2 + f)
    const double z = s * s, w = z * z;
    const double t1 = w * fma(w, fma(w, c_bm.lg[5], c_bm.lg[3]), c_bm.lg[1]);
    const double t2 = z * fma(w, fma(w, fma(w, c_bm.lg[6], c_bm.lg[4]), c_bm.lg[2]), c_bm.lg[0]);
    const double R = t2 + t1;
    const double hfsq = 0.5 * f * f;
    const double dk = (double)k;
    return fma(dk, c_bm.ln2_hi, -((hfsq - fma(s, hfsq + R, dk * c_bm.ln2_lo)) - f));
}

// sqrt(a), a >= 0 finite. a = 0 (u1 == 1) must give 0: the rsqrt input is
// clamped to the smallest normal on the high word (one integer max, no FP
// compare/select), so y stays finite and r = a*y = 0 exactly.
__device__ __forceinline__ double sqrt_fast(double a) {
    const double ac = __hiloint2double(max(__double2hiint(a), 0x00100000), __double2loint(a));
    double y = rsqrt_approx(ac);
    y = y * fma(-0.5 * a * y, y, 1.5);
    y = y * fma(-0.5 * a * y, y, 1.5);
    const double r = a * y;
    return fma(0.5 * y, fma(-r, r, a), r);  // residual correction
}

// sin(t), cos(t) for t in [0, 2*pi).
__device__ __forceinline__ void sincos_2pi(double t, double &sn, double &cs) {
    // quadrant q = nearest integer to t*2/pi via the 1.5*2^52 shifter: the
    // integer lands in the low mantissa bits (no FRND/F2I round trip)
    const double shifter = 0x1.8p52;
    const double qs = fma(t, c_bm.two_over_pi, shifter);
    const int qlo = __double2loint(qs);
    const double q = qs - shifter;
    double x = fma(-q, c_bm.pio2_hi, t);
    x = fma(-q, c_bm.pio2_lo, x);
    const double z = x * x;
    // fdlibm k_sin: x + x*z*(S1 + z*r)
    const double rs = fma(z, fma(z, fma(z, fma(z, c_bm.s[5], c_bm.s[4]), c_bm.s[3]), c_bm.s[2]), c_bm.s[1]);
    const double sx = fma(x * z, fma(z, rs, c_bm.s[0]), x);
    // fdlibm k_cos: w + (((1-w) - hz) + z*r), w = 1 - z/2
    const double rc = z * fma(z, fma(z, fma(z, fma(z, fma(z, c_bm.c[5], c_bm.c[4]), c_bm.c[3]), c_bm.c[2]),
                                     c_bm.c[1]), c_bm.c[0]);
    const double hz = 0.5 * z, wv = 1.0 - hz;
    const double cx = wv + (((1.0 - wv) - hz) + z * rc);
    // quadrant: odd q swaps sin/cos; the signs are xor-ed into the high words
    const bool odd = qlo & 1;
    const double a = odd ? cx : sx;  // |sin(t)| up to sign
    const double b = odd ? sx : cx;  // |cos(t)| up to sign
    const int ssgn = (qlo << 30) & 0x80000000;        // q & 2
    const int csgn = ((qlo + 1) << 30) & 0x80000000;  // (q + 1) & 2
    sn = __hiloint2double(__double2hiint(a) ^ ssgn, __double2loint(a));
    cs = __hiloint2double(__double2hiint(b) ^ csgn, __double2loint(b));
}

__device__ __forceinline__ void box_muller_fast(uint4 w, double &z0, double &z1) {
    const double two_pi = 6.283185307179586;  // 2.0 * math.pi
    const double u1 = 1.0 - (double)((((uint64_t)w.y << 32) | w.x) >> 11) * 0x1p-53;
    const double u2 = (double)((((uint64_t)w.w << 32) | w.z) >> 11) * 0x1p-53;
    const double r = sqrt_fast(-2.0 * log_unit(u1));
    double s, c;
    sincos_2pi(__dmul_rn(two_pi, u2), s, c);
    z0 = __dmul_rn(r, c);
    z1 = __dmul_rn(r, s);
}

}  // namespace cbrng
