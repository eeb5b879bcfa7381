// regress_act.cuh -- device helpers shared by the tensor-core regression
// kernels (regress_tc.cu, regress_split.cu): activations and warp reductions.
#pragma once
#include <cuda_runtime.h>

namespace hcva {

// tanh from one exp2 and one reciprocal: (1 - e^{-2|z|}) / (1 + e^{-2|z|}),
// absolute error ~1e-7 (FP32 rounding level of the O(1) activations that
// feed the next layer), a third of tanhf's instruction count.
__device__ __forceinline__ float tanh_fast(float z) {
    float e, r;  // 1 - 2 / (e^{2z} + 1): saturates to +-1 through e^{2z} = inf / 0
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(2.8853900817779268f * z));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
    return fmaf(-2.0f, r, 1.0f);
}

// Activations (regressor.cpp:35-57), derivative from the activation value.
template <int ACT>
__device__ __forceinline__ float act_f(float z) {
    if constexpr (ACT == 0) return tanh_fast(z);
    else if constexpr (ACT == 1) return 1.0f / (1.0f + expf(-z));
    else if constexpr (ACT == 2) return fmaxf(z, 0.0f) + log1pf(expf(-fabsf(z)));
    else return fmaxf(z, 0.0f);
}
template <int ACT>
__device__ __forceinline__ float act_d(float v) {
    if constexpr (ACT == 0) return 1.0f - v * v;
    else if constexpr (ACT == 1) return v * (1.0f - v);
    else if constexpr (ACT == 2) return -expm1f(-v);
    else return v > 0.0f ? 1.0f : 0.0f;
}


__device__ __forceinline__ float warp_sum(float v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Butterfly reduce-scatter of N (8, 16 or 32) per-lane columns over the warp:
// N-1 shuffles, then log2(32/N) more to add the lane groups; the result is
// the warp's sum of column lane % N.
template <int N>
__device__ __forceinline__ float bfly_sum(float* v, int lane) {
#pragma unroll
    for (int off = N / 2; off >= 1; off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            const float send = up ? v[i] : v[i + off];
            const float keep = up ? v[i + off] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    float s = v[0];
#pragma unroll
    for (int off = N; off < 32; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
}

// acc[b] += warp column sum of g[b*32 + lane % NW] (NW = min(U, 32)).
template <int U>
__device__ __forceinline__ void colsum_acc(const float* g, float* acc, int lane) {
    constexpr int NW = U < 32 ? U : 32;
#pragma unroll
    for (int b = 0; b < (U + 31) / 32; ++b) {
        float t[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) t[i] = g[b * 32 + i];
        acc[b] += bfly_sum<NW>(t, lane);
    }
}

}  // namespace hcva
