// normal.cuh -- device normal transform (rng.cpp:94-130) built for the FP64 pipe.
//
// The reference maps a uniform p to N(0,1) with Acklam's rational seed and one
// Halley step e = 0.5 erfc(-x/sqrt2) - p, u = e sqrt(2 pi) exp(x^2/2),
// x -= u / (1 + x u / 2).  Here:
//   * Acklam's seed is evaluated as the reference does (FP64, same branches,
//     same coefficients) with a reciprocal-Newton divide; the erfc argument
//     -x/sqrt2 is formed as the correctly rounded quotient, as the reference's;
//   * erfc is a branch-free Weideman-map polynomial (tools/fit_erfc.py):
//     erfc(a) = exp(-a^2) P((a-2)/(a+2)) / (1+2a), exp(-a^2) from the exact
//     split a^2 = hi + lo, with all coefficients in constant memory, so the hot
//     loop issues FP64 FMAs instead of rematerialising 64-bit literals;
//   * exp(x^2/2) in u is 1/exp(-a^2), already at hand (u needs ~1e-8 relative,
//     being a ~1e-9 correction);
//   * u / (1 + v) = u (1 - v + v^2) + O(u v^3).
// Agreement with the reference is bounded by the reference's own accuracy of
// Phi(x) - p (ulp(p) or ulp(1) over phi(x)); tests/test_gpu_simulation.py and
// tests/test_gpu_special.py pin both the transform and the special functions.
#pragma once
#include <cstdint>

namespace hcva {

#include "special_coeffs.inc"

__device__ __forceinline__ double rcp_approx(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    return r;
}

// ~0.5-1 ulp reciprocal of a normal, finite d (two Newton steps).
__device__ __forceinline__ double rcp_nr(double d) {
    double r = rcp_approx(d);
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// a / d, correctly rounded in all but rare ties (residual correction).
__device__ __forceinline__ double div_nr(double a, double d) {
    const double r = rcp_nr(d);
    const double q = a * r;
    return fma(fma(-q, d, a), r, q);
}

// exp(z) for z in [-1022 ln2, 0]: Cody-Waite reduction + degree-11 polynomial.
__device__ __forceinline__ double exp_neg(double z) {
    const double magic = 6755399441055744.0;  // 1.5 * 2^52
    const double t = fma(z, 1.4426950408889634, magic);
    const double kf = t - magic;
    const int k = __double2loint(t);
    double r = fma(-kf, 6.93147180559945286e-01, z);
    r = fma(-kf, 2.31904681384629956e-17, r);
    double q = kExpQ[11];
#pragma unroll
    for (int j = 10; j >= 0; --j) q = fma(q, r, kExpQ[j]);
    return __hiloint2double(__double2hiint(q) + (k << 20), __double2loint(q));
}

// erfc(y) for |y| <= 6 and, in E, exp(-y^2).
__device__ __forceinline__ double erfc_fast(double y, double& E) {
    const double a = fabs(y);
    const double t = (a - 2.0) * rcp_nr(a + 2.0);
    double P = kErfcP[21];
#pragma unroll
    for (int j = 20; j >= 0; --j) P = fma(P, t, kErfcP[j]);
    const double hi = a * a;
    const double lo = fma(a, a, -hi);
    E = exp_neg(-hi) * (1.0 - lo);
    const double q = E * P * rcp_nr(fma(2.0, a, 1.0));
    return (y < 0.0) ? 2.0 - q : q;
}

constexpr double kSqrt2 = 1.4142135623730951;      // std::sqrt(2.0)
constexpr double kInvSqrt2 = 0.70710678118654757;  // rounded 1/sqrt(2)
constexpr double kSqrt2Pi = 2.5066282746310002;    // std::sqrt(2.0 * M_PI)

__device__ __forceinline__ bool acklam_tail(double p) {
    return p < 0.02425 || p > 1.0 - 0.02425;
}

// Acklam seed, central region (rng.cpp:103-107).
__device__ __forceinline__ double acklam_central(double p) {
    const double q = p - 0.5;
    const double r = q * q;
    const double num =
        (((((-3.969683028665376e+01 * r + 2.209460984245205e+02) * r + -2.759285104469687e+02) * r +
           1.383577518672690e+02) * r + -3.066479806614716e+01) * r + 2.506628277459239e+00) * q;
    const double den =
        ((((-5.447609879822406e+01 * r + 1.615858368580409e+02) * r + -1.556989798598866e+02) * r +
          6.680131188771972e+01) * r + -1.328068155288572e+01) * r + 1.0;
    return div_nr(num, den);
}

// Acklam seed, tails (rng.cpp:99-102, 108-112); runs on compacted warps.
__device__ __forceinline__ double acklam_tail_seed(double p) {
    const bool upper = p > 0.5;
    const double q = sqrt(-2.0 * log(upper ? 1.0 - p : p));
    const double num =
        ((((-7.784894002430293e-03 * q + -3.223964580411365e-01) * q + -2.400758277161838e+00) * q +
          -2.549732539343734e+00) * q + 4.374664141464968e+00) * q + 2.938163982698783e+00;
    const double den =
        (((7.784695709041462e-03 * q + 3.224671290700398e-01) * q + 2.445134137142996e+00) * q +
         3.754408661907416e+00) * q + 1.0;
    return upper ? -num / den : num / den;
}

// One Halley step against erfc (rng.cpp:120-127).
__device__ __forceinline__ double halley_refine(double x, double p) {
    const double y0 = -x * kInvSqrt2;                   // -x / sqrt2, then
    const double y = fma(fma(-y0, kSqrt2, -x), kInvSqrt2, y0);  // one residual step
    double E;
    const double e = 0.5 * erfc_fast(y, E) - p;
    double ri = rcp_approx(E);                          // exp(x^2/2) = 1 / exp(-y^2)
    ri = fma(ri, fma(-E, ri, 1.0), ri);
    const double u = e * kSqrt2Pi * ri;
    const double v = x * u * 0.5;
    return x - u * (1.0 - v * (1.0 - v));
}

// ---- two independent central-region draws at once (K1's Philox block yields
// a pair): every coefficient is fetched once for both chains and the two
// dependency chains interleave.  Same arithmetic as acklam_central +
// halley_refine on each element except the seed quotient (see below).
__constant__ double kAcklamA[6] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                                   1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
__constant__ double kAcklamB[5] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                                   6.680131188771972e+01,  -1.328068155288572e+01};


// sqrt(2 pi) exp(t) for t = y^2 = x^2/2 (the erf argument squared, already at hand)
// to ~3e-7 in single precision: enough for u, itself a ~1e-9 relative correction
// (its error enters x at < 1e-15 relative).
__device__ __forceinline__ double sqrt2pi_exp_approx(double t) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(static_cast<float>(t) * 1.44269504088896341f));
    return static_cast<double>(r * 2.50662827463100050f);
}

__device__ __forceinline__ void normal_central_x2(const double (&p)[2], double (&x)[2]) {
    // Acklam seed (rng.cpp:103-107)
    double q[2], r[2], num[2], den[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        q[i] = p[i] - 0.5;
        r[i] = q[i] * q[i];
        num[i] = kAcklamA[0];
        den[i] = kAcklamB[0];
    }
#pragma unroll
    for (int j = 1; j < 6; ++j) {
        const double a = kAcklamA[j];
        num[0] = num[0] * r[0] + a;
        num[1] = num[1] * r[1] + a;
    }
#pragma unroll
    for (int j = 1; j < 5; ++j) {
        const double b = kAcklamB[j];
        den[0] = den[0] * r[0] + b;
        den[1] = den[1] * r[1] + b;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        num[i] = num[i] * q[i];
        den[i] = den[i] * r[i] + 1.0;
        // The seed only needs ~1e-12: Halley's step below is insensitive to the
        // seed's low bits (its error enters squared), so one Newton step on the
        // hardware reciprocal replaces the correctly rounded quotient.
        double rd = rcp_approx(den[i]);
        rd = fma(rd, fma(-den[i], rd, 1.0), rd);
        x[i] = num[i] * rd;
    }
    // Halley step (rng.cpp:120-127), central form (halley_central)
    double y[2], t[2], P[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double y0 = -x[i] * kInvSqrt2;
        y[i] = fma(fma(-y0, kSqrt2, -x[i]), kInvSqrt2, y0);
        t[i] = y[i] * y[i];  // x^2 / 2
        P[i] = kErfE[14];
    }
#pragma unroll
    for (int j = 13; j >= 0; --j) {
        const double c = kErfE[j];
        P[0] = fma(P[0], t[0], c);
        P[1] = fma(P[1], t[1], c);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double e = fma(-0.5, y[i] * P[i], 0.5 - p[i]);
        const double u = e * sqrt2pi_exp_approx(t[i]);
        const double v = x[i] * u * 0.5;
        x[i] = x[i] - u * (1.0 - v * (1.0 - v));
    }
}

// Halley step for Acklam's central region (|x| <= 1.973, |x|/sqrt2 <= 1.395):
// Phi(x) - p = (0.5 - p) - 0.5 erf(-x/sqrt2) with erf from one even
// polynomial (kErfE) -- no erfc map, division or double exp -- and the
// correction's exp(x^2/2) in single precision.  Same argument rounding as the
// reference (correctly rounded -x/sqrt2); the result stays within the
// reference's own accuracy bound ulp(p)/phi(x) (tests/test_gpu_simulation.py).
__device__ __forceinline__ double halley_central(double x, double p) {
    const double y0 = -x * kInvSqrt2;
    const double y = fma(fma(-y0, kSqrt2, -x), kInvSqrt2, y0);
    const double t = y * y;  // x^2 / 2
    double P = kErfE[14];
#pragma unroll
    for (int j = 13; j >= 0; --j) P = fma(P, t, kErfE[j]);
    const double e = fma(-0.5, y * P, 0.5 - p);
    const double u = e * sqrt2pi_exp_approx(t);
    const double v = x * u * 0.5;
    return x - u * (1.0 - v * (1.0 - v));
}

__device__ __forceinline__ double normal_from_uniform(double p) {
    return acklam_tail(p) ? halley_refine(acklam_tail_seed(p), p) : halley_central(acklam_central(p), p);
}

}  // namespace hcva
