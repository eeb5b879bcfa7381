// regress_opt.cuh -- the optimizer step of the regression (regressor.cpp:
// 236-261) and the refresh of the tensor-core weight image, shared by k_adam
// (regress.cu) and the persistent SGD kernel (regress_split.cu).
#pragma once
#include <cstdint>

#include "tc.cuh"

namespace hcva {

// Weight image of the tensor-core tile kernel, refreshed by k_adam (img == nullptr: none).
struct ImgArgs {
    uint8_t* img = nullptr;
    int U = 0, d = 0, dp = 0, off0 = 0, off1 = 0, off2 = 0;
};

__device__ __forceinline__ void img_store(const ImgArgs& im, int P, int i, float w) {
    const int U = im.U;
    const uint32_t w0b = U * im.dp * 4, w1b = U * U * 4;
    uint8_t* w0 = im.img;
    uint8_t* w1 = w0 + 2 * w0b;
    uint8_t* w1t = w1 + 2 * w1b;
    float* vec = reinterpret_cast<float*>(w1t + 2 * w1b);
    if (i == P - 1) {
        vec[193] = w;
    } else if (i >= im.off2) {
        const int k = i - im.off2;
        if (k < U) vec[128 + k] = w;
        else vec[192] = w;
    } else if (i >= im.off1) {
        const int k = i - im.off1;
        if (k < U * U) {
            tc::put_split(w1, w1b, k / U, k % U, U, w);
            tc::put_split(w1t, w1b, k % U, k / U, U, w);
        } else {
            vec[64 + k - U * U] = w;
        }
    } else {
        const int k = i - im.off0;
        if (k < U * im.d) tc::put_split(w0, w0b, k / im.d, k % im.d, U, w);
        else vec[k - U * im.d] = w;
    }
}

// Adam / SGD update of parameter i (regressor.cpp:236-261).
__device__ __forceinline__ void optimizer_step(int i, double g, int P, double* p64, float* p32, double* m, double* v,
                                               double c1, double c2, double lr, int adam, const ImgArgs& im) {
    double w = p64[i];
    if (adam) {
        const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
        const double mi = b1 * m[i] + (1.0 - b1) * g;
        const double vi = b2 * v[i] + (1.0 - b2) * g * g;
        m[i] = mi;
        v[i] = vi;
        w -= lr * (mi / c1) / (sqrt(vi / c2) + eps);
    } else {
        w -= lr * g;
    }
    p64[i] = w;
    p32[i] = static_cast<float>(w);
    if (im.img) img_store(im, P, i, static_cast<float>(w));
}

}  // namespace hcva
