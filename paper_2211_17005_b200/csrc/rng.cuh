// rng.cuh -- K0: the reference's counter-based stream on the device and host.
//
// Reproduces hiercva::RandomStream (proj/src/rng.cpp:9-130) draw for draw:
//   * key derivation: root = mix64(seed ^ kRootSalt) (rng.cpp:44-46),
//     split(k) = mix64(key ^ (mix64(k + kSplitSalt) + W + (key<<6) + (key>>2)))
//     (rng.cpp:48-55);
//   * draw j of a stream is word (j % 2) of Philox-2x64-10 block
//     (counter = j / 2, 0) under the stream key (rng.cpp:22-40,57-67), so any
//     (path, substep, factor) draw is addressable without replaying the stream;
//   * uniform ((x >> 11) + 0.5) * 2^-53 (rng.cpp:69-72); normal = Acklam
//     rational + one Halley step (rng.cpp:94-130); exponential = -log(u).
// The 64x64->128 multiply is __umul64hi + a 64-bit multiply on the device.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define HCVA_HD __host__ __device__ __forceinline__
#else
#define HCVA_HD inline
#endif

namespace hcva {

constexpr uint64_t kPhiloxM = 0xD2B74407B1CE6E93ULL;
constexpr uint64_t kPhiloxW = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kRootSalt = 0x9FB21C651E98DF25ULL;
constexpr uint64_t kSplitSalt = 0x632BE59BD9B4E019ULL;

HCVA_HD uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

HCVA_HD uint64_t root_key(uint64_t seed) { return mix64(seed ^ kRootSalt); }

HCVA_HD uint64_t split_key(uint64_t key, uint64_t k) {
    return mix64(key ^ (mix64(k + kSplitSalt) + kPhiloxW + (key << 6) + (key >> 2)));
}

HCVA_HD void philox2x64(uint64_t c0, uint64_t key, uint64_t& o0, uint64_t& o1) {
    uint64_t c1 = 0;
#ifdef __CUDA_ARCH__
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t hi = __umul64hi(kPhiloxM, c0);
        const uint64_t lo = kPhiloxM * c0;
        c0 = hi ^ key ^ c1;
        c1 = lo;
        key += kPhiloxW;
    }
#else
    for (int r = 0; r < 10; ++r) {
        const unsigned __int128 p = static_cast<unsigned __int128>(kPhiloxM) * c0;
        c0 = static_cast<uint64_t>(p >> 64) ^ key ^ c1;
        c1 = static_cast<uint64_t>(p);
        key += kPhiloxW;
    }
#endif
    o0 = c0;
    o1 = c1;
}

HCVA_HD uint64_t draw_u64(uint64_t key, uint64_t j) {
    uint64_t o0, o1;
    philox2x64(j >> 1, key, o0, o1);
    return (j & 1) ? o1 : o0;
}

HCVA_HD double u64_to_uniform(uint64_t x) {
#ifdef __CUDA_ARCH__
    // fl(v + 0.5) * 2^-53 == fl(v * 2^-53 + 2^-54): scaling by 2^-53 commutes
    // with rounding (results >= 2^-54 are normal), so one FMA is bit-identical.
    return fma(static_cast<double>(x >> 11), 0x1.0p-53, 0x1.0p-54);
#else
    return (static_cast<double>(x >> 11) + 0.5) * 0x1.0p-53;
#endif
}

// Acklam's rational approximation + one Halley refinement against erfc
// (rng.cpp:94-130), same coefficients and branch points.
HCVA_HD double inverse_normal_cdf(double p) {
    const double p_low = 0.02425;
    double x;
    if (p < p_low || p > 1.0 - p_low) {
        const bool upper = p > 0.5;
        const double q = sqrt(-2.0 * log(upper ? 1.0 - p : p));
        const double num =
            ((((-7.784894002430293e-03 * q + -3.223964580411365e-01) * q + -2.400758277161838e+00) * q +
              -2.549732539343734e+00) * q + 4.374664141464968e+00) * q + 2.938163982698783e+00;
        const double den =
            (((7.784695709041462e-03 * q + 3.224671290700398e-01) * q + 2.445134137142996e+00) * q +
             3.754408661907416e+00) * q + 1.0;
        x = upper ? -num / den : num / den;
    } else {
        const double q = p - 0.5;
        const double r = q * q;
        const double num =
            (((((-3.969683028665376e+01 * r + 2.209460984245205e+02) * r + -2.759285104469687e+02) * r +
               1.383577518672690e+02) * r + -3.066479806614716e+01) * r + 2.506628277459239e+00) * q;
        const double den =
            ((((-5.447609879822406e+01 * r + 1.615858368580409e+02) * r + -1.556989798598866e+02) * r +
              6.680131188771972e+01) * r + -1.328068155288572e+01) * r + 1.0;
        x = num / den;
    }
    const double e = 0.5 * erfc(-x / 1.4142135623730951) - p;   // sqrt(2.0)
    const double u = e * 2.5066282746310002 * exp(x * x / 2.0);  // sqrt(2*pi)
    return x - u / (1.0 + x * u / 2.0);
}

HCVA_HD double draw_normal(uint64_t key, uint64_t j) {
    return inverse_normal_cdf(u64_to_uniform(draw_u64(key, j)));
}


HCVA_HD double draw_exponential(uint64_t key, uint64_t j) {
    return -log(u64_to_uniform(draw_u64(key, j)));
}

}  // namespace hcva
