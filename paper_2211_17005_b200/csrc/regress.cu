// regress.cu -- K5: the backward MLP regression of the conditional CVA
// (proj/src/regressor.cpp, Alg. 1 train_base :265-347, Alg. 2 backward_learn
// :354-395), device-resident end to end.
//
// Per pricing step i = n..1: the feature rows of every replica (k,l)
// (labels.cpp:142-167) are built on the device and standardised with the
// scaler fitted over all rows (regressor.cpp:84-95); the network starts from
// Glorot init at i = n (host RNG, same stream as the reference) or from step
// i+1's best; train_base runs E epochs of |B| contiguous batches with Adam,
// the closed-form ridge refit and head switch at epoch floor(E/2), full-sample
// evaluation and best tracking each epoch -- all without host round trips.
//
// Kernels:
//   k_sgd       forward + backward of one batch tile (TR rows per CTA):
//               activations in shared memory, FP32 FMA tiles, per-CTA partial
//               gradients (FP32) and loss (FP64)
//   k_adam      fixed-order FP64 reduction of the partials + Adam (:236-261)
//               on the FP64 master parameters, FP32 compute copy
//   k_eval      full-sample forward: loss with the positive head, min of the
//               plain-head fit (head switch), predictions
//   k_gram      Gram matrix and rhs of [z_h, 1] (refit, :191-213), FP64
//   k_refit     one-CTA reduction + ridge + LDL^T solve of the (u+1)^2 system
//   k_switch / k_track   head switch (:299-314) and best tracking (:316-327)
// Reductions are over fixed CTA partitions in fixed order: results are
// deterministic and independent of scheduling.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "common.cuh"
#include "rng.cuh"

namespace hcva {

constexpr int kMaxLayers = 5;  // hidden layers <= 4

}  // namespace hcva
#include <fstream>
#include <functional>

#include "comm.cuh"
#include "regress_opt.cuh"
#include "regress_tc.cuh"
#include "tc.cuh"  // tensor-core tiles for the paper's network shape
namespace hcva {

struct NetDims {
    int d, h, u, act, P;
    int off[kMaxLayers + 1];  // W_l offset; b_l = off[l] + fout*fin
    int fin[kMaxLayers + 1], fout[kMaxLayers + 1];
};

NetDims make_dims(int d, int h, int u, int act) {
    if (h < 1 || h > kMaxLayers - 1) throw config_error("training: hidden_layers must be in 1..4");
    if (u < 1 || u > 128) throw config_error("training: width must be in 1..128");
    NetDims n{};
    n.d = d;
    n.h = h;
    n.u = u;
    n.act = act;
    int off = 0, fin = d;
    for (int l = 0; l <= h; ++l) {
        const int fout = (l == h) ? 1 : u;
        n.off[l] = off;
        n.fin[l] = fin;
        n.fout[l] = fout;
        off += fout * fin + fout;
        fin = fout;
    }
    n.P = off + 1;  // + mu
    return n;
}

// regressor.cpp:35-57.  Derivatives from the activation value: tanh 1-a^2,
// sigmoid a(1-a), softplus sigma(z) = 1 - exp(-a), relu 1{a>0}.
__device__ __forceinline__ float act_fwd(int a, float z) {
    switch (a) {
        case 0: return tanhf(z);
        case 1: return 1.0f / (1.0f + expf(-z));
        case 2: return fmaxf(z, 0.0f) + log1pf(expf(-fabsf(z)));
        default: return fmaxf(z, 0.0f);
    }
}
__device__ __forceinline__ float act_der(int a, float v) {
    switch (a) {
        case 0: return 1.0f - v * v;
        case 1: return v * (1.0f - v);
        case 2: return -expm1f(-v);
        default: return v > 0.0f ? 1.0f : 0.0f;
    }
}

// Shared-memory plan of one tile: params (P floats), x tile [TR][d+1],
// h activation buffers [TR][u+1] (reused in place as gradient buffers).
__host__ __device__ inline size_t tile_smem(const NetDims& n, int TR) {
    return sizeof(float) * (static_cast<size_t>(n.P) + 1 + static_cast<size_t>(TR) * (n.d + 1) +
                            static_cast<size_t>(n.h) * TR * (n.u + 1)) + 64 * sizeof(double);
}

// Forward of the rows of a tile: thread r owns row r.  Returns f (pre-head output).
__device__ float tile_forward(const NetDims& n, const float* W, const float* xs, float* acts, int TR, int r) {
    const int ld_in0 = n.d + 1, ld = n.u + 1;
    for (int l = 0; l < n.h; ++l) {
        const float* in = (l == 0) ? xs + r * ld_in0 : acts + (l - 1) * TR * ld + r * ld;
        float* out = acts + l * TR * ld + r * ld;
        const float* Wl = W + n.off[l];
        const int fin = n.fin[l], fout = n.fout[l];
        const float* bl = Wl + fout * fin;
        for (int o0 = 0; o0 < fout; o0 += 8) {
            float acc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = (o0 + q < fout) ? bl[o0 + q] : 0.0f;
            for (int j = 0; j < fin; ++j) {
                const float v = in[j];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (o0 + q < fout) acc[q] = fmaf(v, Wl[(o0 + q) * fin + j], acc[q]);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (o0 + q < fout) out[o0 + q] = act_fwd(n.act, acc[q]);
        }
    }
    const float* top = acts + (n.h - 1) * TR * ld + r * ld;
    const float* w = W + n.off[n.h];
    float f = w[n.u];
    for (int j = 0; j < n.u; ++j) f = fmaf(top[j], w[j], f);
    return f;
}

// Partial gradient of W_l over the tile rows: sum_r g[r][o] in[r][j], 4x4 blocks per thread.
__device__ void tile_outer(const float* g, int ldg, const float* in, int ldi, int TR, int rows, int fout, int fin,
                           float* gW, float* gb) {
    const int bo = (fout + 3) / 4, bj = (fin + 3) / 4;
    for (int blk = threadIdx.x; blk < bo * bj; blk += blockDim.x) {
        const int o0 = (blk / bj) * 4, j0 = (blk % bj) * 4;
        float acc[4][4] = {};
        for (int r = 0; r < rows; ++r) {
            float gv[4], iv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                gv[q] = (o0 + q < fout) ? g[r * ldg + o0 + q] : 0.0f;
                iv[q] = (j0 + q < fin) ? in[r * ldi + j0 + q] : 0.0f;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(gv[a], iv[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (o0 + a < fout && j0 + b < fin) gW[(o0 + a) * fin + j0 + b] = acc[a][b];
    }
    for (int o = threadIdx.x; o < fout; o += blockDim.x) {
        float s = 0.0f;
        for (int r = 0; r < rows; ++r) s += g[r * ldg + o];
        gb[o] = s;
    }
}

__device__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    return s;  // valid in thread 0
}

// One batch tile: rows [row0 + blockIdx.x*TR, min(+TR, row_end)).  Writes the
// CTA's partial gradient (FP32, parameter layout incl. mu) and partial
// sum of squared residuals (FP64).  nb = batch size (loss normaliser).
__global__ void k_sgd(NetDims n, const float* X, const double* y, long row0, long row_end, const float* params,
                      int head, double nb, float* gpart, double* lpart, int TR) {
    extern __shared__ double smd[];
    float* W = reinterpret_cast<float*>(smd);
    float* xs = W + n.P + 1;
    float* acts = xs + TR * (n.d + 1);
    double* red = reinterpret_cast<double*>(acts + n.h * TR * (n.u + 1) + 1);
    red = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(red) + 15) & ~uintptr_t(15));
    const long base = row0 + static_cast<long>(blockIdx.x) * TR;
    const int rows = static_cast<int>(min(static_cast<long>(TR), row_end - base));
    for (int i = threadIdx.x; i < n.P; i += blockDim.x) W[i] = params[i];
    for (int i = threadIdx.x; i < rows * n.d; i += blockDim.x) {
        const int r = i / n.d, c = i % n.d;
        xs[r * (n.d + 1) + c] = X[(base + r) * n.d + c];
    }
    __syncthreads();
    const int r = threadIdx.x;
    const int ld = n.u + 1;
    const float mu = W[n.P - 1];
    double resid2 = 0.0, dmu = 0.0;
    float dd = 0.0f;
    if (r < rows) {
        const float f = tile_forward(n, W, xs, acts, TR, r);
        const float pred = ((head && f < 0.0f) ? 0.0f : f) + mu;
        const double resid = static_cast<double>(pred) - y[base + r];
        resid2 = resid * resid;
        dmu = 2.0 * resid / nb;
        dd = static_cast<float>(dmu);
        if (head && !(f > 0.0f)) dd = 0.0f;
    }
    const double lsum = block_sum(resid2, red);
    const double msum = block_sum(dmu, red);
    float* gout = gpart + static_cast<size_t>(blockIdx.x) * n.P;
    if (threadIdx.x == 0) {
        lpart[blockIdx.x] = lsum;
        gout[n.P - 1] = static_cast<float>(msum);
    }
    // Output layer: gw[j] = sum_r dd_r z_r[j], gb = sum_r dd_r; stash dd in xs[r][d].
    if (r < rows) xs[r * (n.d + 1) + n.d] = dd;
    __syncthreads();
    {
        const float* top = acts + (n.h - 1) * TR * ld;
        float* gw = gout + n.off[n.h];
        for (int j = threadIdx.x; j <= n.u; j += blockDim.x) {
            float s = 0.0f;
            for (int rr = 0; rr < rows; ++rr) s = fmaf(xs[rr * (n.d + 1) + n.d], (j < n.u) ? top[rr * ld + j] : 1.0f, s);
            gw[j] = s;
        }
    }
    __syncthreads();
    // g = dd w (x) act'(z_{h}) in place of the top activations.
    if (r < rows) {
        float* top = acts + (n.h - 1) * TR * ld + r * ld;
        const float* w = W + n.off[n.h];
        for (int j = 0; j < n.u; ++j) top[j] = dd * w[j] * act_der(n.act, top[j]);
    }
    __syncthreads();
    for (int l = n.h - 1; l >= 0; --l) {
        const float* g = acts + l * TR * ld;
        const float* in = (l == 0) ? xs : acts + (l - 1) * TR * ld;
        const int ldi = (l == 0) ? n.d + 1 : ld;
        float* gW = gout + n.off[l];
        tile_outer(g, ld, in, ldi, TR, rows, n.fout[l], n.fin[l], gW, gW + n.fout[l] * n.fin[l]);
        if (l > 0) {
            // g_prev[j] = sum_o g[o] W_l[o][j], times act'(z_{l}) -- in place of act[l-1].
            __syncthreads();
            if (r < rows) {
                const float* Wl = W + n.off[l];
                float* prev = acts + (l - 1) * TR * ld + r * ld;
                const float* gr = g + r * ld;
                for (int j = 0; j < n.u; ++j) {
                    float s = 0.0f;
                    for (int o = 0; o < n.u; ++o) s = fmaf(gr[o], Wl[o * n.u + j], s);
                    prev[j] = s * act_der(n.act, prev[j]);
                }
            }
            __syncthreads();
        }
    }
}

// Fixed-order reduction of the tile partials + optimiser step (regressor.cpp:236-261).
// Parameters whose gradient partials come from the weight-gradient kernel
// (tensor-core path: W0 and W1) instead of the per-tile kernel.
struct SplitPartials;
__host__ __device__ inline size_t split_index(const SplitPartials& sp, int i);

struct SplitPartials {
    const float* gpartB = nullptr;
    int nB = 0;
    int lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;  // [lo, hi) index ranges served by gpartB
    int stride = 0, U = 0, d = 0, dp = 0;    // gpartB rows: W1 | b1 as [U][U+8], then W0 | b0 as [U][dp]
};

// Block (32, 16): x = parameter, y = partial group c = y (mod 16); the group
// sums combine in a fixed pairwise tree.  Warp 0 of CTA 0 also checks the loss.
__host__ __device__ inline size_t split_index(const SplitPartials& sp, int i) {
    const int U = sp.U;
    if (i >= sp.lo1 && i < sp.hi1) {  // W1 row-major, then b1
        const int k = i - sp.lo1;
        return k < U * U ? static_cast<size_t>(k / U) * (U + 8) + k % U : static_cast<size_t>(k - U * U) * (U + 8) + U;
    }
    const int k = i - sp.lo0;  // W0 row-major, then b0 (pad column d of the feature tile)
    const size_t base = static_cast<size_t>(U) * (U + 8);
    return k < U * sp.d ? base + static_cast<size_t>(k / sp.d) * sp.dp + k % sp.d
                        : base + static_cast<size_t>(k - U * sp.d) * sp.dp + sp.d;
}

#ifndef HCVA_ADAM_G
#define HCVA_ADAM_G 8  // partial groups per parameter (8 measured best of 8, 16, 32)
#endif
__global__ void k_adam(int P, const float* gpart, int nct, SplitPartials sp, const double* lpart, double nb,
                       double* p64, float* p32, double* m, double* v, double c1, double c2, double lr, int adam,
                       int* nonfinite,
                       ImgArgs im) {
    constexpr int G = HCVA_ADAM_G;
    __shared__ double part[G][33];
    const int x = threadIdx.x, grp = threadIdx.y;
    const int i = blockIdx.x * 32 + x;
    pdl_trigger();  // the next tile kernel may run its prologue now (it waits for this grid)
    if (blockIdx.x == 0 && grp == 0) {
        double s = 0.0;
        for (int c = x; c < nct; c += 32) s += lpart[c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (x == 0 && !isfinite(s / nb)) atomicExch(nonfinite, 1);
    }
    double s = 0.0;
    if (i < P) {
        const bool split = sp.nB && ((i >= sp.lo0 && i < sp.hi0) || (i >= sp.lo1 && i < sp.hi1));
        const float* src = split ? sp.gpartB + split_index(sp, i) : gpart + i;
        const size_t stride = split ? sp.stride : P;
        const int cnt = split ? sp.nB : nct;
#pragma unroll 4
        for (int c = grp; c < cnt; c += G) s += static_cast<double>(__ldg(src + static_cast<size_t>(c) * stride));
    }
    part[grp][x] = s;
    __syncthreads();
#pragma unroll
    for (int h = G / 2; h >= 1; h >>= 1) {
        if (grp < h) part[grp][x] += part[grp + h][x];
        __syncthreads();
    }
    if (grp != 0 || i >= P) return;
    optimizer_step(i, part[0][x], P, p64, p32, m, v, c1, c2, lr, adam, im);
}

// Multi-GPU: this rank's gradient (FP64, fixed-order sum of its partials) and
// loss sum -> red[0..P], red[P]; gathered across ranks before k_adam_dist.
__global__ void k_rank_sum(int P, const float* gpart, int nct, SplitPartials sp, const double* lpart, double* red) {
    constexpr int G = 16;
    __shared__ double part[G][33];
    const int x = threadIdx.x, grp = threadIdx.y;
    const int i = blockIdx.x * 32 + x;
    if (blockIdx.x == 0 && grp == 0) {
        double s = 0.0;
        for (int c = x; c < nct; c += 32) s += lpart[c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (x == 0) red[P] = s;
    }
    double s = 0.0;
    if (i < P) {
        const bool split = sp.nB && ((i >= sp.lo0 && i < sp.hi0) || (i >= sp.lo1 && i < sp.hi1));
        const float* src = split ? sp.gpartB + split_index(sp, i) : gpart + i;
        const size_t stride = split ? sp.stride : P;
        const int cnt = split ? sp.nB : nct;
#pragma unroll 4
        for (int c = grp; c < cnt; c += G) s += static_cast<double>(__ldg(src + static_cast<size_t>(c) * stride));
    }
    part[grp][x] = s;
    __syncthreads();
#pragma unroll
    for (int h = G / 2; h >= 1; h >>= 1) {
        if (grp < h) part[grp][x] += part[grp + h][x];
        __syncthreads();
    }
    if (grp == 0 && i < P) red[i] = part[0][x];
}

// Update from the gathered per-rank vectors all[G][stride], summed in rank order.
__global__ void k_adam_dist(int P, const double* all, int G, int stride, double nb, double* p64, float* p32, double* m,
                            double* v, double c1, double c2, double lr, int adam, int* nonfinite, ImgArgs im) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        double s = 0.0;
        for (int r = 0; r < G; ++r) s += all[static_cast<size_t>(r) * stride + P];
        if (!isfinite(s / nb)) atomicExch(nonfinite, 1);
    }
    if (i >= P) return;
    double g = 0.0;
    for (int r = 0; r < G; ++r) g += all[static_cast<size_t>(r) * stride + i];
    optimizer_step(i, g, P, p64, p32, m, v, c1, c2, lr, adam, im);
}

// out[0] = sum (op 0) or min (op 1) of parts[0..n), fixed order (one warp).
__global__ void k_reduce_scalar(const double* parts, int n, int op, double* out) {
    const int x = threadIdx.x;
    double s = op ? INFINITY : 0.0;
    for (int c = x; c < n; c += 32) s = op ? fmin(s, parts[c]) : s + parts[c];
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, s, o);
        s = op ? fmin(s, w) : s + w;
    }
    if (x == 0) out[0] = s;
}

// Full-sample forward over tiles (grid-stride, fixed tile->CTA map).
// mode bit 0: loss with the positive head -> lpart; bit 1: min of the plain
// fit f + mu -> mpart; bit 2: predictions (head on) -> pred.
__global__ void k_eval(NetDims n, const float* X, const double* y, long R, const float* params, int mode,
                       double* lpart, double* mpart, double* pred, int TR) {
    extern __shared__ double smd[];
    float* W = reinterpret_cast<float*>(smd);
    float* xs = W + n.P + 1;
    float* acts = xs + TR * (n.d + 1);
    double* red = reinterpret_cast<double*>(acts + n.h * TR * (n.u + 1) + 1);
    red = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(red) + 15) & ~uintptr_t(15));
    for (int i = threadIdx.x; i < n.P; i += blockDim.x) W[i] = params[i];
    const float mu = params[n.P - 1];
    double lacc = 0.0, macc = INFINITY;
    const long ntiles = (R + TR - 1) / TR;
    for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long base = tile * TR;
        const int rows = static_cast<int>(min(static_cast<long>(TR), R - base));
        __syncthreads();
        for (int i = threadIdx.x; i < rows * n.d; i += blockDim.x) {
            const int r = i / n.d, c = i % n.d;
            xs[r * (n.d + 1) + c] = X[(base + r) * n.d + c];
        }
        __syncthreads();
        const int r = threadIdx.x;
        if (r < rows) {
            const float f = tile_forward(n, W, xs, acts, TR, r);
            const double ph = static_cast<double>((f < 0.0f ? 0.0f : f) + mu);
            if (mode & 1) {
                const double res = ph - y[base + r];
                lacc += res * res;
            }
            if (mode & 2) macc = fmin(macc, static_cast<double>(f + mu));
            if (mode & 4) pred[base + r] = ph;
        }
    }
    if (mode & 1) {
        const double s = block_sum(lacc, red);
        if (threadIdx.x == 0) lpart[blockIdx.x] = s;
    }
    if (mode & 2) {
        for (int o = 16; o > 0; o >>= 1) macc = fmin(macc, __shfl_down_sync(0xffffffffu, macc, o));
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = macc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double mn = INFINITY;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mn = fmin(mn, red[i]);
            mpart[blockIdx.x] = mn;
        }
    }
}

// Gram of [z_h, 1] (upper triangle, row-major) and rhs sum z (y - mu) over the
// CTA's tiles, accumulated in FP64 into the CTA's own partial slot.
// gpart[cta][(u+1)(u+2)/2 + (u+1)].
__global__ void k_gram(NetDims n, const float* X, const double* y, long R, const float* params, double* gpart,
                       int TR) {
    extern __shared__ double smd[];
    float* W = reinterpret_cast<float*>(smd);
    float* xs = W + n.P + 1;
    float* acts = xs + TR * (n.d + 1);
    const int ld = n.u + 1, m = n.u + 1, tri = m * (m + 1) / 2, npair = tri + m;
    for (int i = threadIdx.x; i < n.P; i += blockDim.x) W[i] = params[i];
    const double mu = params[n.P - 1];
    double* out = gpart + static_cast<size_t>(blockIdx.x) * npair;
    for (int idx = threadIdx.x; idx < npair; idx += blockDim.x) out[idx] = 0.0;
    const long ntiles = (R + TR - 1) / TR;
    for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long base = tile * TR;
        const int rows = static_cast<int>(min(static_cast<long>(TR), R - base));
        __syncthreads();
        for (int i = threadIdx.x; i < rows * n.d; i += blockDim.x) {
            const int r = i / n.d, c = i % n.d;
            xs[r * (n.d + 1) + c] = X[(base + r) * n.d + c];
        }
        __syncthreads();
        if (static_cast<int>(threadIdx.x) < rows) {
            const int r = threadIdx.x;
            (void)tile_forward(n, W, xs, acts, TR, r);
            acts[(n.h - 1) * TR * ld + r * ld + n.u] = 1.0f;
        }
        __syncthreads();
        const float* top = acts + (n.h - 1) * TR * ld;
        int a = 0, rem = threadIdx.x;  // idx -> (a, b) walk, advanced by blockDim each step
        for (int idx = threadIdx.x; idx < npair; idx += blockDim.x) {
            double s = 0.0;
            if (idx < tri) {
                while (rem >= m - a) {
                    rem -= m - a;
                    ++a;
                }
                const int b = a + rem;
                for (int rr = 0; rr < rows; ++rr) s += static_cast<double>(top[rr * ld + a]) * top[rr * ld + b];
                rem += blockDim.x;
            } else {
                const int c = idx - tri;
                for (int rr = 0; rr < rows; ++rr) s += static_cast<double>(top[rr * ld + c]) * (y[base + rr] - mu);
            }
            out[idx] += s;
        }
    }
}

// out[idx] = sum over c of parts[c * stride + idx], four interleaved chains
// combined pairwise (fixed order).
// out[i] = sum over the n partial rows of parts[.][i] in a fixed order: block
// (32, 16), x = entry, y = group g summing rows g, g + 16, ... with four chains,
// then the 16 group sums in a fixed pairwise tree.
__global__ void k_sum_parts(const double* parts, int n, int stride, double* out) {
    constexpr int G = 16;
    __shared__ double part[G][33];
    const int x = threadIdx.x, grp = threadIdx.y;
    const int idx = blockIdx.x * 32 + x;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    if (idx < stride) {
        int c = grp, k = 0;
        for (; c < n; c += G, k = (k + 1) & 3) a[k] += parts[static_cast<size_t>(c) * stride + idx];
    }
    part[grp][x] = (a[0] + a[1]) + (a[2] + a[3]);
    __syncthreads();
#pragma unroll
    for (int h = G / 2; h >= 1; h >>= 1) {
        if (grp < h) part[grp][x] += part[grp + h][x];
        __syncthreads();
    }
    if (grp == 0 && idx < stride) out[idx] = part[0][x];
}

// One CTA: reduce the Gram partials (fixed order), ridge lam = max(ridge tr/(u+1), 1e-300),
// LDL^T solve, write the output layer (regressor.cpp:191-213).
__global__ void k_refit(NetDims n, const double* gpart, int nct, double ridge, double* p64, float* p32) {
    extern __shared__ double sm[];
    const int m = n.u + 1, tri = m * (m + 1) / 2, stride = tri + m;
    double* G = sm;           // [m][m]
    double* rhs = G + m * m;  // [m]
    double* D = rhs + m;      // [m]
    for (int idx = threadIdx.x; idx < stride; idx += blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < nct; ++c) s += gpart[static_cast<size_t>(c) * stride + idx];
        if (idx < tri) {
            int a = 0, rem = idx;
            while (rem >= m - a) {
                rem -= m - a;
                ++a;
            }
            const int b = a + rem;
            G[a * m + b] = s;
            G[b * m + a] = s;
        } else {
            rhs[idx - tri] = s;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tr = 0.0;
        for (int a = 0; a < m; ++a) tr += G[a * m + a];
        const double lam = fmax(ridge * tr / m, 1e-300);
        for (int a = 0; a < m; ++a) G[a * m + a] += lam;
    }
    __syncthreads();
    // LDL^T in place (lower part of G holds L), right-looking: per column j, d_j and the
    // column below it are saved, L[i][j] = c_i / d_j, and the trailing lower block takes
    // the rank-1 update G[i][k] -= L[i][j] c_k (j < k <= i) in parallel.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto wsum = [](double v) {
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    double* cj = D + m;    // [m] column j below the diagonal, unscaled
    double* lj = cj + m;   // [m] ... scaled: L[i][j]
    for (int j = 0; j < m; ++j) {
        const double dj = G[j * m + j];
        for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) {
            const double c = G[i * m + j];
            cj[i] = c;
            lj[i] = c / dj;
            G[i * m + j] = c / dj;
        }
        if (threadIdx.x == 0) D[j] = dj;
        __syncthreads();
        const int nn = m - j - 1;
        for (int t = threadIdx.x; t < nn * nn; t += blockDim.x) {
            const int ii = t / nn, kk = t - ii * nn;
            if (kk <= ii) {
                const int i = j + 1 + ii, k = j + 1 + kk;
                G[i * m + k] -= lj[i] * cj[k];
            }
        }
        __syncthreads();
    }
    if (warp == 0) {
        for (int i = 0; i < m; ++i) {  // L z = rhs
            double s = 0.0;
            for (int k = lane; k < i; k += 32) s += G[i * m + k] * rhs[k];
            s = wsum(s);
            if (lane == 0) rhs[i] -= s;
            __syncwarp();
        }
        for (int i = lane; i < m; i += 32) rhs[i] /= D[i];
        __syncwarp();
        for (int i = m - 1; i >= 0; --i) {  // L^T x = z
            double s = 0.0;
            for (int k = i + 1 + lane; k < m; k += 32) s += G[k * m + i] * rhs[k];
            s = wsum(s);
            if (lane == 0) rhs[i] -= s;
            __syncwarp();
        }
    }
    if (threadIdx.x == 0) {
        const int o = n.off[n.h];
        for (int c = 0; c < m; ++c) {
            p64[o + c] = rhs[c];
            p32[o + c] = static_cast<float>(rhs[c]);
        }
    }
}

// The minimum of the fitted values f + mu (regressor.cpp:299-304) of a network whose
// hidden layers produced the kept layer-2 activations H2 [R][64] and whose output layer
// is (w2, b_out): the output sum in k_eval_split's order (four sequential 16-column
// FMA chains, combined pairwise), kept per row in fsum for k_loss_fsum.
__global__ void __launch_bounds__(512) k_min_from_h2(const float* H2, long R, const float* w2, const float* b_out,
                                                     const double* mu, float* fsum, double* mpart) {
    __shared__ float ws[64];
    __shared__ double red[32];
    if (threadIdx.x < 64) ws[threadIdx.x] = w2[threadIdx.x];
    __syncthreads();
    const float b = *b_out;
    const double m = *mu;
    double mn = INFINITY;
    // four lanes per row (lane k: columns 16k..16k+15, 64 contiguous bytes): a warp reads
    // 8 consecutive rows, 2 KB
    const int k = threadIdx.x & 3;
    const float* w = ws + 16 * k;
    const long step = static_cast<long>(gridDim.x) * (blockDim.x / 4);
    for (long r0 = blockIdx.x * static_cast<long>(blockDim.x / 4); r0 < R; r0 += step) {
        const long r = r0 + (threadIdx.x >> 2);
        float acc = 0.0f;
        if (r < R) {
            const float4* h = reinterpret_cast<const float4*>(H2 + r * 64 + 16 * k);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 v = __ldcs(h + q);
                acc = fmaf(v.x, w[4 * q], acc);
                acc = fmaf(v.y, w[4 * q + 1], acc);
                acc = fmaf(v.z, w[4 * q + 2], acc);
                acc = fmaf(v.w, w[4 * q + 3], acc);
            }
        }
        const float a1 = __shfl_xor_sync(0xffffffffu, acc, 1);  // lane pair (g0, g1) / (g2, g3)
        const float s01 = (k & 1) ? a1 + acc : acc + a1;        // g0 + g1 or g2 + g3, in that order
        const float s23 = __shfl_xor_sync(0xffffffffu, s01, 2);
        const float fs = (k & 2) ? s23 + s01 : s01 + s23;       // (g0 + g1) + (g2 + g3)
        if (r < R && k == 0) {
            fsum[r] = fs;
            mn = fmin(mn, static_cast<double>(b + fs) + m);
        }
    }
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = red[0];
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = fmin(t, red[w]);
        mpart[blockIdx.x] = t;
    }
}

// The full-sample loss (head on) of the network whose output bias is b_out and mu
// mu, from each row's kept output-layer sum s (k_eval_split mode 16): f = b_out + s in
// FP32 as the evaluation kernel forms it, pred = max(f, 0) + mu, fixed-order partial
// sums per CTA over contiguous row ranges.
__global__ void __launch_bounds__(256) k_loss_fsum(const float* fsum, const double* y, long R, const float* b_out,
                                                   const double* mu, double* lpart) {
    __shared__ double red[32];
    const long per = (R + gridDim.x - 1) / gridDim.x, r0 = blockIdx.x * per, r1 = min(R, r0 + per);
    const float b = *b_out;
    const double m = *mu;
    double s = 0.0;
    for (long r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const float f = b + fsum[r];
        const double res = ((f < 0.0f) ? 0.0 : static_cast<double>(f)) + m - y[r];
        s += res * res;
    }
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) lpart[blockIdx.x] = t;
}

// Head switch (regressor.cpp:299-314): mu_new = max(0, min fit), output bias += mu - mu_new,
// Adam state reset.
__global__ void k_switch(NetDims n, const double* mpart, int nct, double* p64, float* p32, double* m, double* v) {
    for (int i = threadIdx.x; i < n.P; i += blockDim.x) {
        m[i] = 0.0;
        v[i] = 0.0;
    }
    if (threadIdx.x < 32) {  // the minimum is order-free: lanes take strided partials
        double mn = INFINITY;
        for (int c = threadIdx.x; c < nct; c += 32) mn = fmin(mn, mpart[c]);
        for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        if (threadIdx.x != 0) return;
        const double mu_new = fmax(0.0, mn);
        const int bo = n.off[n.h] + n.u;
        p64[bo] += p64[n.P - 1] - mu_new;
        p64[n.P - 1] = mu_new;
        p32[bo] = static_cast<float>(p64[bo]);
        p32[n.P - 1] = static_cast<float>(mu_new);
    }
}

// Epoch bookkeeping (regressor.cpp:316-327): record the full-sample loss,
// keep the best parameters on a strict improvement.
__global__ void k_track(int P, const double* lpart, int nct, double R, int epoch, const double* __restrict__ p64,
                        double* __restrict__ best, double* losses, double* best_loss, int* best_epoch, int* nonfinite) {
    __shared__ int improved;
    if (threadIdx.x < 32) {  // lanes sum strided partials (loads in flight together), then a fixed butterfly
        double s = 0.0;
        for (int c = threadIdx.x; c < nct; c += 32) s += lpart[c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double ev = s / R;
        if (threadIdx.x == 0) {
            losses[epoch - 1] = ev;
            if (!isfinite(ev)) *nonfinite = 1;
            improved = ev < *best_loss;
            if (improved) {
                *best_loss = ev;
                *best_epoch = epoch;
            }
        }
    }
    __syncthreads();
    if (improved) {
#pragma unroll 4
        for (int i = threadIdx.x; i < P; i += blockDim.x) best[i] = p64[i];
    }
}

__global__ void k_to_f32(const double* a, float* b, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = static_cast<float>(a[i]);
}

__global__ void k_set_mu_mean(const double* y, long R, double* p64, float* p32, int P) {
    __shared__ double red[32];
    double s = 0.0;
    for (long r = threadIdx.x; r < R; r += blockDim.x) s += y[r];
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) {
        p64[P - 1] = t / static_cast<double>(R);
        p32[P - 1] = static_cast<float>(t / static_cast<double>(R));
    }
}

// Label mean over all ranks' rows: mu = sum_r all[r] / R_total.
__global__ void k_set_mu_from(const double* all, int G, double R_total, double* p64, float* p32, int P) {
    double s = 0.0;
    for (int r = 0; r < G; ++r) s += all[r];
    p64[P - 1] = s / R_total;
    p32[P - 1] = static_cast<float>(s / R_total);
}

__global__ void k_sq_err(const double* pred, const double* y, long n, double* out) {
    const long j = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (j < n) {
        const double e = pred[j] - y[j];
        out[j] = e * e;
    }
}

__global__ void k_local_sum(const double* y, long R, double* out) {
    __shared__ double red[32];
    double s = 0.0;
    for (long r = threadIdx.x; r < R; r += blockDim.x) s += y[r];
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) out[0] = t;
}

// ---------------------------------------------------------------- trainer

struct Trainer {
    hcva_ctx* ctx;
    NetDims n;
    int TR = 128, eval_ctas = 0;
    DeviceBuf p64, p32, m, v, best, gpart, lpart, mpart, gram, flag, losses, best_loss, best_epoch;
    // Tensor-core path: weight-gradient partials, transposed activations, packed operand images.
    DeviceBuf gpartB, h1t, g2t, g1t, wimg, ximg, xt, h2, gram_sum, fsumb;
    int max_tiles = 0, last_parts = 0, dp = 0, gram_parts = 0;
    bool use_tc = false, xf32 = false;
    long ld_x = 0, ld_tmax = 0, x_rows = 0;
    bool wimg_valid = false;  // weight image matches p32
    const uint8_t* ximg_over = nullptr;    // evaluation on another feature image (Q/R probe)
    std::function<void(int)> on_epoch;     // after each epoch's bookkeeping (Q/R probe)
    hcva_comm* comm = nullptr;  // multi-GPU: rank-ordered allgather of the FP64 partials
    int world = 1;
    DeviceBuf red, gath;
    // Layer-0 split (regress_split.cu): per-path columns yhat [M][qp] of the
    // current step + the default steps instead of a feature matrix.
    bool split = false;
    SplitArgs sa{};
    DeviceBuf yhat, pg;  // per-path columns of the step; layer-0 path parts (evaluations)
    const SplitArgs* sa_over = nullptr;  // evaluation on other rows of the same paths (Q/R probe)

    void set_comm(hcva_comm* c, size_t max_len) {
        comm = c;  // an explicit comm always takes the gather path (world 1 included)
        world = comm ? comm->world : 1;
        if (!comm) return;
        red.alloc(max_len * 8);
        gath.alloc(max_len * 8 * world);
    }
    // Gather this rank's vector local[0..len) from every rank: [world][len] in rank order.
    const double* gather(const double* local, size_t len) {
        comm->allgather(local, gath.p, len * 8, ctx->stream);
        return gath.as<double>();
    }

    Trainer(hcva_ctx* c, const NetDims& dims, long max_batch, long max_rows = 0, bool split_mode = false)
        : ctx(c), n(dims) {
        use_tc = tc_eligible(n.d, n.h, n.u);
        split = split_mode && use_tc;
        while (TR > 32 && tile_smem(n, TR) > 200 * 1024) TR /= 2;
        if (tile_smem(n, TR) > 227 * 1024) throw config_error("training: network too wide for the tile kernel");
        const size_t smem = tile_smem(n, TR);
        HCVA_CUDA(cudaFuncSetAttribute(k_sgd, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        HCVA_CUDA(cudaFuncSetAttribute(k_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        HCVA_CUDA(cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int per_sm = 1;
        HCVA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eval, TR, smem));
        eval_ctas = std::max(1, per_sm) * ctx->sm_count;
        max_tiles = static_cast<int>((max_batch + TR - 1) / TR);
        const size_t P = n.P;
        long parts = std::max<long>(max_tiles, eval_ctas);
        if (use_tc && split) {
            dp = tc_dp(n.d);
            parts = std::max<long>(parts, std::max(ctx->sm_count, split_max_ctas(ctx->sm_count)));
            wimg.alloc(tc_weight_image_bytes(n.u, dp));
        } else if (use_tc) {
            dp = tc_dp(n.d);
            xf32 = tc_two_cta(n.u, dp);
            parts = std::max<long>(parts, std::max(ctx->sm_count, tc_eval_max_ctas(ctx->sm_count)));
            ld_tmax = ((std::max<long>(max_batch, 1) + 63) / 64) * 64;
            const size_t tsz = static_cast<size_t>(n.u) * ld_tmax * 4;
            h1t.alloc(tsz);
            g2t.alloc(tsz);
            g1t.alloc(tsz);
            gpartB.alloc(static_cast<size_t>(tc_wgrad_max_ctas(ctx->sm_count)) * (n.u * (n.u + 8) + n.u * dp) * 4);
            wimg.alloc(tc_weight_image_bytes(n.u, dp));
            x_rows = std::max(max_rows, max_batch);
            ld_x = ((x_rows + 64 + 3) / 4) * 4;  // slack for the 64-row chunk loads
            ximg.alloc(static_cast<size_t>((x_rows + 127) / 128) * tc_x_tile_bytes(dp));
            xt.alloc(static_cast<size_t>(dp) * ld_x * 4);
        }
        p64.alloc(P * 8);
        p32.alloc(P * 4);
        m.alloc(P * 8);
        v.alloc(P * 8);
        best.alloc(P * 8);
        gpart.alloc(static_cast<size_t>(std::max<long>(parts, 1)) * P * 4);
        lpart.alloc(static_cast<size_t>(parts) * 8);
        mpart.alloc(static_cast<size_t>(parts) * 8);
        const size_t mm = n.u + 1;
        gram_parts = std::max(eval_ctas, 4 * ctx->sm_count);
        gram.alloc(static_cast<size_t>(gram_parts) * (mm * (mm + 1) / 2 + mm) * 8);
        flag.alloc(4);
        HCVA_CUDA(cudaMemsetAsync(flag.p, 0, 4, ctx->stream));  // pool memory is not zeroed
        best_loss.alloc(8);
        best_epoch.alloc(4);
    }

    size_t smem() const { return tile_smem(n, TR); }

    void set_params(const double* host_or_dev) {
        HCVA_CUDA(cudaMemcpyAsync(p64.p, host_or_dev, n.P * 8, cudaMemcpyDefault, ctx->stream));
        k_to_f32<<<grid1(n.P, 256), 256, 0, ctx->stream>>>(p64.as<double>(), p32.as<float>(), n.P);
        check_launch(ctx);
        wimg_valid = false;
    }

    // The split source of a simulated set (paths M, replicas N): the per-path
    // columns are rebuilt for every step by build_yhat.
    void split_source(const hcva_sim* sim) {
        const int Cc = sim->model.Cc, q = n.d - Cc;
        sa = SplitArgs{};
        sa.d = n.d; sa.Cc = Cc; sa.q = q; sa.qp = ((q + 3) / 4) * 4; sa.N = sim->N;
        sa.P = n.P; sa.off0 = n.off[0]; sa.off1 = n.off[1]; sa.off2 = n.off[2]; sa.act = n.act;
        sa.M = sim->M; sa.R = static_cast<long>(sim->M) * sim->N;
        sa.steps = sim->steps.as<uint16_t>();
        yhat.alloc(static_cast<size_t>(sim->M) * sa.qp * 4);
        sa.yhat = yhat.as<float>();
        pg.alloc(static_cast<size_t>(sim->M) * n.u * 4);
    }

    SplitArgs split_args(const SplitArgs& base, const double* y, long b0, long b1, int head, int mode, double nb,
                         double* pred) {
        if (!wimg_valid) {
            launch_pack_w(n.u, n.d, dp, n.off[0], n.off[1], n.off[2], n.P, p32.as<float>(), wimg.as<uint8_t>(),
                          ctx->stream);
            check_launch(ctx);
            wimg_valid = true;
        }
        SplitArgs a = base;
        const size_t w0b = static_cast<size_t>(n.u) * dp * 4, w1b = static_cast<size_t>(n.u) * n.u * 4;
        a.w1img = wimg.as<uint8_t>() + 2 * w0b;
        a.vec = reinterpret_cast<const float*>(wimg.as<uint8_t>() + 2 * w0b + 4 * w1b);
        a.p32 = p32.as<float>();
        a.mu64 = p64.as<double>() + n.P - 1;
        a.y = y; a.b0 = b0; a.b1 = b1; a.head = head; a.mode = mode; a.nb = nb;
        a.gpart = gpart.as<float>(); a.lpart = lpart.as<double>(); a.mpart = mpart.as<double>(); a.pred = pred;
        a.H2 = h2.as<float>();
        a.Pg_out = pg.as<float>();
        return a;
    }

    // Features of the sample (X [R][d], device) -> the tensor-core operand images.
    void prepare_x(const float* X, long R) {
        if (!use_tc) return;
        if (R > x_rows) throw contract_error("training: feature rows exceed the trainer's capacity");
        launch_pack_x(X, R, n.d, dp, ximg.as<uint8_t>(), xt.as<float>(), ld_x, xf32 ? 1 : 0, ctx->stream);
        check_launch(ctx);
    }

    // Launch the persistent tile kernel over rows [b0, b1); returns the partial count.
    int tile_launch(const double* y, long b0, long b1, int head, int mode, double nb, double* pred) {
        if (!wimg_valid) {
            launch_pack_w(n.u, n.d, dp, n.off[0], n.off[1], n.off[2], n.P, p32.as<float>(), wimg.as<uint8_t>(),
                          ctx->stream);
            check_launch(ctx);
            wimg_valid = true;
        }
        TileArgs ta{};
        ta.d = n.d; ta.dp = dp; ta.act = n.act; ta.P = n.P;
        ta.off0 = n.off[0]; ta.off1 = n.off[1]; ta.off2 = n.off[2];
        ta.wimg = wimg.as<uint8_t>(); ta.ximg = ximg_over ? ximg_over : ximg.as<uint8_t>(); ta.y = y; ta.b0 = b0;
        ta.b1 = b1;
        ta.head = head; ta.mode = mode; ta.nb = nb;
        ta.gpart = gpart.as<float>(); ta.lpart = lpart.as<double>(); ta.mpart = mpart.as<double>(); ta.pred = pred;
        ta.H2 = h2.as<float>();
        ta.H1t = h1t.as<float>(); ta.G2t = g2t.as<float>(); ta.G1t = g1t.as<float>();
        ta.ld_t = ((b1 - b0 + 63) / 64) * 64;
        ta.xf32 = xf32 ? 1 : 0;
        const int ctas = launch_tile_tc(n.u, ta, ctx->sm_count, ctx->stream);
        check_launch(ctx);
        return ctas;
    }

    // Gradient partials of rows [b0, b1): per-tile partials (+ weight-gradient
    // partials on the tensor-core path, described by sp); returns the tile count.
    int grad_tiles(const float* X, const double* y, long b0, long b1, int head, double nb, SplitPartials* sp) {
        if (split) {
            const int ctas = launch_sgd_split(split_args(sa, y, b0, b1, head, 0, nb, nullptr), ctx->sm_count,
                                              ctx->stream);
            check_launch(ctx);
            if (sp) *sp = SplitPartials{};
            return ctas;
        }
        if (use_tc) {
            const int ctas = tile_launch(y, b0, b1, head, 0, nb, nullptr);
            WgradArgs wa{};
            wa.d = n.d; wa.dp = dp; wa.P = n.P; wa.off0 = n.off[0]; wa.off1 = n.off[1];
            wa.G2t = g2t.as<float>(); wa.H1t = h1t.as<float>(); wa.G1t = g1t.as<float>();
            wa.ld_t = ((b1 - b0 + 63) / 64) * 64;
            wa.Xt = xt.as<float>(); wa.ld_x = ld_x; wa.row0 = b0; wa.rows = b1 - b0; wa.gpart = gpartB.as<float>();
            static const bool twice = std::getenv("HCVA_WGRAD_TWICE") != nullptr;  // profiling probe
            if (twice) {  // an extra launch with the row loop skipped: the kernel's fixed costs
                WgradArgs wp = wa;
                wp.probe = 1;
                launch_wgrad_tc(n.u, wp, ctx->sm_count, ctx->stream);
            }
            const int nB = launch_wgrad_tc(n.u, wa, ctx->sm_count, ctx->stream);
            check_launch(ctx);
            if (sp) *sp = SplitPartials{gpartB.as<float>(), nB, n.off[0], n.off[0] + n.u * n.d + n.u, n.off[1],
                                        n.off[1] + n.u * n.u + n.u, n.u * (n.u + 8) + n.u * dp, n.u, n.d, dp};
            return ctas;
        }
        const int tiles = static_cast<int>((b1 - b0 + TR - 1) / TR);
        k_sgd<<<tiles, TR, smem(), ctx->stream>>>(n, X, y, b0, b1, p32.as<float>(), head, nb, gpart.as<float>(),
                                                 lpart.as<double>(), TR);
        check_launch(ctx);
        if (sp) *sp = SplitPartials{};
        return tiles;
    }

    cudaEvent_t* phase_ev = nullptr;  // profiling: events after the gradient kernels and after the update
    DeviceBuf gbar, c12;              // persistent SGD: grid-barrier counter, per-step bias corrections

    // The SGD steps of one epoch (batches [0, nb) of bs rows) as one persistent
    // launch with the optimizer fused (split path, one GPU); c12_dev: this
    // epoch's [nb][2] bias corrections.  False when the batch shape does not
    // allow it (the caller then runs sgd_step per batch).
    bool fusable(long bs, int nb) const {
        static const bool on = [] {
            const char* e = std::getenv("HCVA_FUSED_EPOCH");
            return !(e && e[0] == '0');
        }();
        return on && split && !comm && nb >= 1 && nb <= 64 && bs % 128 == 0 && sa.N >= 16;
    }
    bool sgd_epoch(const double* y, long bs, int nb, int head, const double* c12_dev, double lr, int adam) {
        if (!gbar.p) gbar.alloc(16);
        HCVA_CUDA(cudaMemsetAsync(gbar.p, 0, 16, ctx->stream));
        SplitArgs a = split_args(sa, y, 0, bs, head, 0, static_cast<double>(bs), nullptr);
        a.fuse = 1;
        a.nsteps = nb;
        a.bs = bs;
        a.lr = lr;
        a.adam = adam;
        a.dp = dp;
        a.p64w = p64.as<double>();
        a.m = m.as<double>();
        a.v = v.as<double>();
        a.p32w = p32.as<float>();
        a.img = wimg.as<uint8_t>();
        a.gbar = gbar.as<unsigned>();
        a.nonfinite = flag.as<int>();
        a.c12 = c12_dev;
        if (!launch_sgd_split_fused(a, ctx->sm_count, ctx->stream)) return false;
        ctx->launches++;
        check_launch(ctx);
        return true;
    }

    void sgd_step(const float* X, const double* y, long b0, long b1, int head, long t, double lr, int adam) {
        SplitPartials sp;
        const double nb = static_cast<double>(b1 - b0) * world;  // the global batch
        const int tiles = grad_tiles(X, y, b0, b1, head, nb, &sp);
        if (phase_ev) HCVA_CUDA(cudaEventRecord(phase_ev[0], ctx->stream));
        // Adam bias corrections 1 - beta^t on the host with the host libm, as
        // the reference's adam_update (regressor.cpp:236-252).
        const double c1 = 1.0 - std::pow(0.9, static_cast<double>(t)), c2 = 1.0 - std::pow(0.999, static_cast<double>(t));
        if (comm) {
            k_rank_sum<<<(n.P + 31) / 32, dim3(32, 16), 0, ctx->stream>>>(n.P, gpart.as<float>(), tiles, sp,
                                                                           lpart.as<double>(), red.as<double>());
            check_launch(ctx);
            const double* all = gather(red.as<double>(), n.P + 1);
            k_adam_dist<<<grid1(n.P, 128), 128, 0, ctx->stream>>>(n.P, all, world, n.P + 1, nb, p64.as<double>(),
                                                                  p32.as<float>(), m.as<double>(), v.as<double>(), c1,
                                                                  c2, lr, adam, flag.as<int>(), img_args());
            check_launch(ctx);
            return;
        }
        k_adam<<<(n.P + 31) / 32, dim3(32, HCVA_ADAM_G), 0, ctx->stream>>>(n.P, gpart.as<float>(), tiles, sp, lpart.as<double>(),
                                                         static_cast<double>(b1 - b0), p64.as<double>(), p32.as<float>(),
                                                         m.as<double>(), v.as<double>(), c1, c2, lr, adam,
                                                         flag.as<int>(), img_args());
        check_launch(ctx);
        if (phase_ev) HCVA_CUDA(cudaEventRecord(phase_ev[1], ctx->stream));
    }

    ImgArgs img_args() {
        ImgArgs im;
        if (use_tc && wimg_valid) im = ImgArgs{wimg.as<uint8_t>(), n.u, n.d, dp, n.off[0], n.off[1], n.off[2]};
        return im;
    }

    // Full-sample forward; sets last_parts = number of loss / min partials written.
    void eval(const float* X, const double* y, long R, int mode, double* pred) {
        if (split) {
            const SplitArgs& base = sa_over ? *sa_over : sa;
            last_parts = launch_eval_split(split_args(base, y, 0, R, 1, mode, 1.0, pred), ctx->sm_count, ctx->stream);
            check_launch(ctx);
            return;
        }
        if (use_tc) {
            last_parts = tile_launch(y, 0, R, 1, mode, 1.0, pred);
            return;
        }
        k_eval<<<eval_ctas, TR, smem(), ctx->stream>>>(n, X, y, R, p32.as<float>(), mode, lpart.as<double>(),
                                                      mpart.as<double>(), pred, TR);
        check_launch(ctx);
        last_parts = eval_ctas;
    }

    void refit(const float* X, const double* y, long R, double ridge) {
        int nct = eval_ctas;
        if (use_tc) {
            const size_t hbytes = static_cast<size_t>(R) * n.u * 4;
            if (h2.bytes < hbytes) h2.alloc(hbytes);  // layer-2 activations, first refit only
            if (split) {
                launch_eval_split(split_args(sa, y, 0, R, 1, 8, 1.0, nullptr), ctx->sm_count, ctx->stream);
                check_launch(ctx);
            } else {
                tile_launch(y, 0, R, 1, 8, 1.0, nullptr);
            }
            nct = launch_gram_h2(n.u, h2.as<float>(), y, R, p32.as<float>(), n.P, gram.as<double>(), gram_parts,
                                 ctx->sm_count, ctx->stream);
        } else {
            k_gram<<<eval_ctas, TR, smem(), ctx->stream>>>(n, X, y, R, p32.as<float>(), gram.as<double>(), TR);
        }
        check_launch(ctx);
        const int mm = n.u + 1;
        const size_t sm = sizeof(double) * (static_cast<size_t>(mm) * mm + 4 * mm);  // G, rhs, D, column j x2
        HCVA_CUDA(cudaFuncSetAttribute(k_refit, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        const double* gsrc = gram.as<double>();
        if (nct > 8 || comm) {  // pre-reduce the partials across the GPU, k_refit then reads one
            const int stride = mm * (mm + 1) / 2 + mm;
            if (gram_sum.bytes < static_cast<size_t>(stride) * 8) gram_sum.alloc(static_cast<size_t>(stride) * 8);
            k_sum_parts<<<(stride + 31) / 32, dim3(32, 16), 0, ctx->stream>>>(gram.as<double>(), nct, stride,
                                                                         gram_sum.as<double>());
            check_launch(ctx);
            gsrc = gram_sum.as<double>();
            nct = 1;
            if (comm) {  // every rank's Gram + rhs, summed in rank order by k_refit
                gsrc = gather(gsrc, stride);
                nct = world;
            }
        }
        k_refit<<<1, 256, sm, ctx->stream>>>(n, gsrc, nct, ridge, p64.as<double>(), p32.as<float>());
        wimg_valid = false;
        check_launch(ctx);
    }

    // This rank's sum (op 0) / min (op 1) of n partials, gathered from every rank
    // ([world] in rank order); without a comm the partials themselves.
    const double* rank_scalar(const double* parts, int cnt, int op) {
        if (!comm) return parts;
        k_reduce_scalar<<<1, 32, 0, ctx->stream>>>(parts, cnt, op, red.as<double>());
        check_launch(ctx);
        return gather(red.as<double>(), 1);
    }

    // train_base (regressor.cpp:265-347) on device-resident X [R][d] (FP32), y [R] (FP64).
    // losses_dev: [epochs] (device).  Parameters start in p64/p32; the best end in `best`.
    void train_base(const float* X, const double* y, long R, int epochs, int n_batches, double lr, int adam,
                    double ridge, double* losses_dev) {
        if (epochs < 2) throw config_error("training: epochs must be >= 2 (head switch at E/2)");
        if (n_batches < 1 || R % n_batches != 0) throw config_error("make_batches: batch count must divide M*N");
        const long bs = R / n_batches;
        const double inf = INFINITY;
        HCVA_CUDA(cudaMemcpyAsync(best_loss.p, &inf, 8, cudaMemcpyHostToDevice, ctx->stream));
        HCVA_CUDA(cudaMemsetAsync(best_epoch.p, 0, 4, ctx->stream));
        HCVA_CUDA(cudaMemsetAsync(m.p, 0, n.P * 8, ctx->stream));
        HCVA_CUDA(cudaMemsetAsync(v.p, 0, n.P * 8, ctx->stream));
        HCVA_CUDA(cudaMemcpyAsync(best.p, p64.p, n.P * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        HCVA_CUDA(cudaStreamSynchronize(ctx->stream));  // &inf lives on this frame
        int head = 0;
        long t = 0;
        const int sw = epochs / 2;
        // persistent epochs: the Adam bias corrections 1 - beta^t of every step of this
        // train_base (t restarts at the head switch), host libm pow as adam_update
        // (regressor.cpp:247-248), staged once
        const bool fuse = fusable(bs, n_batches);
        if (fuse) {
            std::vector<double> h(2 * static_cast<size_t>(epochs) * n_batches);
            long tt = 0;
            for (int e = 1; e <= epochs; ++e) {
                for (int b = 0; b < n_batches; ++b) {
                    ++tt;
                    h[2 * ((e - 1) * static_cast<size_t>(n_batches) + b)] = 1.0 - std::pow(0.9, static_cast<double>(tt));
                    h[2 * ((e - 1) * static_cast<size_t>(n_batches) + b) + 1] =
                        1.0 - std::pow(0.999, static_cast<double>(tt));
                }
                if (e == sw) tt = 0;
            }
            if (c12.bytes < h.size() * 8) c12.alloc(h.size() * 8);
            HCVA_CUDA(cudaMemcpyAsync(c12.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        for (int e = 1; e <= epochs; ++e) {
            if (fuse && sgd_epoch(y, bs, n_batches, head,
                                  c12.as<double>() + 2 * (e - 1) * static_cast<size_t>(n_batches), lr, adam))
                t += n_batches;
            else
                for (int b = 0; b < n_batches; ++b) sgd_step(X, y, b * bs, (b + 1) * bs, head, ++t, lr, adam);
            bool loss_done = false;
            if (e == sw) {
                refit(X, y, R, ridge);
                // split path: the refit changed only the output layer, so the minimum of the
                // fitted values is one GEMV over the layer-2 activations the refit pass kept
                // (the evaluation kernel's summation order: bit-identical output sums), and
                // the epoch loss after the switch (mu and the output bias change) one pass
                // over those sums -- instead of two full forward evaluations
                const bool keep = split && !sa_over && h2.bytes >= static_cast<size_t>(R) * n.u * 4;
                if (keep) {
                    if (fsumb.bytes < static_cast<size_t>(R) * 4) fsumb.alloc(static_cast<size_t>(R) * 4);
                    last_parts = split_max_ctas(ctx->sm_count);  // rows of mpart the trainer holds
                    k_min_from_h2<<<last_parts, 512, 0, ctx->stream>>>(
                        h2.as<float>(), R, p32.as<float>() + n.off[n.h], p32.as<float>() + n.off[n.h] + n.u,
                        p64.as<double>() + n.P - 1, fsumb.as<float>(), mpart.as<double>());
                    check_launch(ctx);
                } else {
                    eval(X, y, R, 2, nullptr);
                }
                wimg_valid = false;
                const double* mp = rank_scalar(mpart.as<double>(), last_parts, 1);
                k_switch<<<1, 256, 0, ctx->stream>>>(n, mp, comm ? world : last_parts, p64.as<double>(),
                                                      p32.as<float>(), m.as<double>(), v.as<double>());
                check_launch(ctx);
                head = 1;
                t = 0;
                if (keep) {
                    const int bo = n.off[n.h] + n.u;
                    last_parts = ctx->sm_count;
                    k_loss_fsum<<<last_parts, 256, 0, ctx->stream>>>(fsumb.as<float>(), y, R, p32.as<float>() + bo,
                                                                       p64.as<double>() + n.P - 1, lpart.as<double>());
                    check_launch(ctx);
                    loss_done = true;
                }
            }
            if (!loss_done) eval(X, y, R, 1, nullptr);
            const double* lp = rank_scalar(lpart.as<double>(), last_parts, 0);
            k_track<<<1, 1024, 0, ctx->stream>>>(n.P, lp, comm ? world : last_parts, static_cast<double>(R) * world, e,
                                                 p64.as<double>(), best.as<double>(), losses_dev,
                                                 best_loss.as<double>(), best_epoch.as<int>(), flag.as<int>());
            check_launch(ctx);
            if (on_epoch) on_epoch(e);
        }
    }

    void check_finite() {
        int f = 0;
        copy_out(ctx, &f, flag.p, 4);
        if (f) throw numeric_error("training diverged (non-finite loss); try a smaller learning rate");
    }
};

// Features of step i for every replica row, standardised (labels.cpp:142-167,
// regressor.cpp:76-95): [indicators 1{s_c <= i}, rates, fx, client intensities, lagged].
struct FeatArgs {
    int M, N, E, Cn, step;
    const double *rates, *fx, *intens, *lag0;
    const uint16_t* steps;
    const double* mean;
    const double* scale;
    float* X;          // [R][d] row-major (SIMT path), or
    uint8_t* ximg;     // tensor-core path: 128-row operand tiles (hi | lo) ...
    float* Xt;         // ... and the transposed copy [dp][ld_x]
    long ld_x;
    int dp;
    int xf32;          // feature tiles as one FP32 plane (tc_two_cta) instead of hi | lo planes
};

__device__ __forceinline__ double state_col(const FeatArgs& a, int k, int j) {
    const int E = a.E, Cc = a.Cn - 1, M = a.M, i = a.step;
    if (j < E) return a.rates[(static_cast<size_t>(i) * E + j) * M + k];
    j -= E;
    if (j < E - 1) return a.fx[(static_cast<size_t>(i) * (E - 1) + j) * M + k];
    j -= E - 1;
    if (j < Cc) return a.intens[(static_cast<size_t>(i) * a.Cn + j + 1) * M + k];
    j -= Cc;
    return (i == 0) ? a.lag0[j] : a.rates[(static_cast<size_t>(i - 1) * E + j) * M + k];
}

__global__ void k_build_x(FeatArgs a) {
    const size_t R = static_cast<size_t>(a.M) * a.N;
    const size_t row = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const int Cc = a.Cn - 1, q = 3 * a.E - 1 + Cc, d = Cc + q;
    if (a.ximg) {  // grid covers the padded last tile: rows >= R are zero
        const size_t tiles = (R + 127) / 128;
        if (row >= tiles * 128) return;
        const bool in = row < R;
        const int k = in ? static_cast<int>(row / a.N) : 0;
        const uint32_t xb = 128u * a.dp * 4;
        uint8_t* tb = a.ximg + (row / 128) * (a.xf32 ? 1 : 2) * xb;
        for (int c = 0; c < a.dp; c += 4) {
            float v[4];
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                const int col = c + qq;
                float x = 0.0f;
                if (in && col < Cc) x = (a.steps[(col + 1) * R + row] <= a.step) ? 1.0f : 0.0f;
                else if (in && col < d)
                    x = static_cast<float>((state_col(a, k, col - Cc) - a.mean[col]) / a.scale[col]);
                v[qq] = x;
                if (in && a.Xt) a.Xt[col * a.ld_x + row] = x;
            }
            if (a.xf32)
                *reinterpret_cast<float4*>(tb + tc::core_off(static_cast<int>(row % 128), c, 128)) =
                    make_float4(v[0], v[1], v[2], v[3]);
            else
                tc::put_split4(tb, xb, static_cast<int>(row % 128), c, 128, make_float4(v[0], v[1], v[2], v[3]));
        }
        return;
    }
    if (row >= R) return;
    const int k = static_cast<int>(row / a.N);
    float* o = a.X + row * d;
    for (int c = 1; c <= Cc; ++c) o[c - 1] = (a.steps[c * R + row] <= a.step) ? 1.0f : 0.0f;
    for (int j = 0; j < q; ++j)
        o[Cc + j] = static_cast<float>((state_col(a, k, j) - a.mean[Cc + j]) / a.scale[Cc + j]);
}

// Layer-0 split: the standardised per-path columns of step i, yhat [M][qp]
// (FP32 of the FP64 standardisation, the values k_build_x writes; zero pad).
__global__ void k_build_yhat(FeatArgs a, float* yhat, int q, int qp) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<size_t>(a.M) * qp) return;
    const int k = static_cast<int>(i % a.M), j = static_cast<int>(i / a.M);
    const int Cc = a.Cn - 1;
    yhat[static_cast<size_t>(k) * qp + j] =
        j < q ? static_cast<float>((state_col(a, k, j) - a.mean[Cc + j]) / a.scale[Cc + j]) : 0.0f;
}

// Scaler (regressor.cpp:84-95) over the rows: the state columns repeat per path,
// so mean / population variance over rows equal those over paths.  One CTA per
// column, fixed-order FP64 reduction; indicator columns pass through.
__global__ void k_scaler(FeatArgs a, double* mean, double* scale) {
    __shared__ double red[32];
    const int Cc = a.Cn - 1, j = blockIdx.x;
    if (j < Cc) {
        if (threadIdx.x == 0) {
            mean[j] = 0.0;
            scale[j] = 1.0;
        }
        return;
    }
    const int js = j - Cc;
    double s = 0.0;
    for (int k = threadIdx.x; k < a.M; k += blockDim.x) s += state_col(a, k, js);
    const double tot = block_sum(s, red);
    __shared__ double m_sh;
    if (threadIdx.x == 0) m_sh = tot / a.M;
    __syncthreads();
    const double mu = m_sh;
    double v = 0.0;
    for (int k = threadIdx.x; k < a.M; k += blockDim.x) {
        const double dlt = state_col(a, k, js) - mu;
        v += dlt * dlt;
    }
    const double vt = block_sum(v, red);
    if (threadIdx.x == 0) {
        const double sd = sqrt(vt / a.M);
        mean[j] = mu;
        scale[j] = (sd > 1e-12) ? sd : 1.0;
    }
}

// Multi-GPU scaler: this rank's column sums (pass 0) or centred squared sums
// about the global mean (pass 1) over its paths; indicator columns give 0.
__global__ void k_scaler_moment(FeatArgs a, int pass, const double* mean, double* out) {
    __shared__ double red[32];
    const int Cc = a.Cn - 1, j = blockIdx.x;
    if (j < Cc) {
        if (threadIdx.x == 0) out[j] = 0.0;
        return;
    }
    const int js = j - Cc;
    const double mu = pass ? mean[j] : 0.0;
    double s = 0.0;
    for (int k = threadIdx.x; k < a.M; k += blockDim.x) {
        const double x = state_col(a, k, js) - mu;
        s += pass ? x * x : x;
    }
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) out[j] = t;
}

// Gathered moments all[G][d] (rank order) -> mean (pass 0) / scale (pass 1) over Mt paths.
__global__ void k_scaler_fin(const double* all, int G, int d, int Cc, double Mt, int pass, double* mean,
                             double* scale) {
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < G; ++r) s += all[static_cast<size_t>(r) * d + j];
        if (j < Cc) {
            mean[j] = 0.0;
            scale[j] = 1.0;
        } else if (pass == 0) {
            mean[j] = s / Mt;
        } else {
            const double sd = sqrt(s / Mt);
            scale[j] = (sd > 1e-12) ? sd : 1.0;
        }
    }
}

}  // namespace hcva

// Trained model sequence (regressor.hpp:120-131), device resident.
struct hcva_models {
    hcva_ctx* ctx = nullptr;
    hcva::NetDims n{};
    int n_steps = 0, epochs = 0;
    hcva::DeviceBuf params, mean, scale, losses, best_loss, best_epoch;  // [n][...]
};

using namespace hcva;

namespace {

NetDims dims_from(const hcva_train_cfg* cfg, int d) {
    if (!cfg) throw contract_error("training: null config");
    return make_dims(d, cfg->hidden_layers, cfg->width, cfg->activation);
}

// Glorot-uniform init (regressor.cpp:172-189) from stream key, mu = 0.
std::vector<double> init_params(const NetDims& n, uint64_t key) {
    std::vector<double> p(n.P, 0.0);
    uint64_t j = 0;
    for (int l = 0; l <= n.h; ++l) {
        const double limit = std::sqrt(6.0 / (n.fin[l] + n.fout[l]));
        for (int r = 0; r < n.fout[l]; ++r)
            for (int c = 0; c < n.fin[l]; ++c)
                p[n.off[l] + r * n.fin[l] + c] = limit * (2.0 * u64_to_uniform(draw_u64(key, j++)) - 1.0);
    }
    return p;
}

FeatArgs feat_args(hcva_sim* sim, int step) {
    FeatArgs a{};
    a.M = sim->M;
    a.N = sim->N;
    a.E = sim->model.E;
    a.Cn = sim->model.Cn;
    a.step = step;
    a.rates = sim->rates.as<double>();
    a.fx = sim->fx.as<double>();
    a.intens = sim->intens.as<double>();
    a.lag0 = sim->lag0.as<double>();
    a.steps = sim->steps.as<uint16_t>();
    return a;
}

// Stage host features (FP64 [rows][d]) as FP32 X (+ the tensor-core images).
void stage_features(Trainer& tr, const double* x, int rows, int d, DeviceBuf& dX) {
    std::vector<float> xf(static_cast<size_t>(rows) * d);
    for (size_t i = 0; i < xf.size(); ++i) xf[i] = static_cast<float>(x[i]);
    stage(dX, xf);
    tr.prepare_x(dX.as<float>(), rows);
}

// Whether a trainer on this simulated set takes the layer-0 split path (the
// SGD kernel needs N >= 16 replicas per path, the evaluation any N).
bool use_split(const NetDims& n, const hcva_sim* sim, bool sgd = true) {
    const int Cc = sim->model.Cc;
    return tc_eligible(n.d, n.h, n.u) && n.d == 2 * Cc + 3 * sim->model.E - 1 && (!sgd || sim->N >= 16) &&
           split_eligible(n.u, n.h, sim->N, Cc, n.d - Cc);
}

// Loss and gradient of the mean loss from a launch's partials, summed on the
// host in fixed order (FP64).
void reduce_partials(Trainer& tr, int tiles, const SplitPartials& sp, long rows, double* loss, double* grads) {
    hcva_ctx* ctx = tr.ctx;
    const NetDims& n = tr.n;
    std::vector<float> gp(static_cast<size_t>(tiles) * n.P), gb(static_cast<size_t>(sp.nB) * sp.stride);
    std::vector<double> lp(tiles);
    copy_out(ctx, gp.data(), tr.gpart.p, gp.size() * 4);
    if (sp.nB) copy_out(ctx, gb.data(), sp.gpartB, gb.size() * 4);
    copy_out(ctx, lp.data(), tr.lpart.p, lp.size() * 8);
    double l = 0.0;
    for (double v : lp) l += v;
    *loss = l / rows;
    if (grads)
        for (int i = 0; i < n.P; ++i) {
            const bool split = (i >= sp.lo0 && i < sp.hi0) || (i >= sp.lo1 && i < sp.hi1);
            const bool fromB = split && sp.nB;
            const float* src = fromB ? gb.data() + split_index(sp, i) : gp.data() + i;
            const size_t stride = fromB ? sp.stride : n.P;
            const int cnt = fromB ? sp.nB : tiles;
            double g = 0.0;
            for (int c = 0; c < cnt; ++c) g += src[static_cast<size_t>(c) * stride];
            grads[i] = g;
        }
}

// Standardised features of one step (fa with mean / scale set): straight into
// the tensor-core operand images, or into X [R][d] for the SIMT path.
// With `img` (tensor-core path) the features go to that operand image only
// (evaluation rows, e.g. the Q/R probe), not to the trainer's own.
void build_features(Trainer& tr, FeatArgs fa, DeviceBuf& X, long R, DeviceBuf* img = nullptr) {
    hcva_ctx* ctx = tr.ctx;
    if (tr.split) {  // no feature matrix: the per-path columns of this step (shared by other rows of the paths)
        if (!img) {
            k_build_yhat<<<grid1(static_cast<size_t>(fa.M) * tr.sa.qp, 256), 256, 0, ctx->stream>>>(
                fa, tr.yhat.as<float>(), tr.sa.q, tr.sa.qp);
            tr.sa.step = fa.step;
            check_launch(ctx);
        }
        return;
    }
    if (tr.use_tc) {
        if (!img && R > tr.x_rows) throw contract_error("training: feature rows exceed the trainer's capacity");
        fa.ximg = img ? img->as<uint8_t>() : tr.ximg.as<uint8_t>();
        fa.xf32 = tr.xf32 ? 1 : 0;
        fa.Xt = img ? nullptr : tr.xt.as<float>();
        fa.ld_x = tr.ld_x;
        fa.dp = tr.dp;
        k_build_x<<<grid1(((R + 127) / 128) * 128, 256), 256, 0, ctx->stream>>>(fa);
    } else {
        fa.X = X.as<float>();
        k_build_x<<<grid1(R, 256), 256, 0, ctx->stream>>>(fa);
    }
    check_launch(ctx);
}

}  // namespace

extern "C" {

hcva_status hcva_net_size(const hcva_train_cfg* cfg, int input_dim, int* n_params) {
    return guarded([&] { *n_params = dims_from(cfg, input_dim).P; });
}

hcva_status hcva_init_network(const hcva_train_cfg* cfg, int input_dim, uint64_t key, double* params) {
    return guarded([&] {
        const auto p = init_params(dims_from(cfg, input_dim), key);
        std::memcpy(params, p.data(), p.size() * 8);
    });
}

hcva_status hcva_quadratic_loss(hcva_ctx* ctx, const hcva_train_cfg* cfg, int input_dim, const double* params,
                                int head, const double* x, const double* y, int rows, double* loss, double* grads) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const NetDims n = dims_from(cfg, input_dim);
        Trainer tr(ctx, n, rows);
        DeviceBuf dX, dy;
        stage_features(tr, x, rows, input_dim, dX);
        stage(dy, std::vector<double>(y, y + rows));
        tr.set_params(params);
        SplitPartials sp;
        const int tiles =
            tr.grad_tiles(dX.as<float>(), dy.as<double>(), 0, rows, head, static_cast<double>(rows), &sp);
        reduce_partials(tr, tiles, sp, rows, loss, grads);
    });
}

// quadratic_loss (regressor.cpp:115-158) on rows [b0, b1) of the label
// source's data at step i (make_label_source, pipeline.cpp:72-111): features
// of the simulated set standardised with host mean / scale [d], labels of
// label_kind -- through the kernels backward_learn runs on this set (the
// layer-0 split kernel where eligible).
hcva_status hcva_sim_quadratic_loss(hcva_sim* sim, const hcva_train_cfg* cfg, int step, int label_kind,
                                    const double* params, const double* mean, const double* scale, int head,
                                    long b0, long b1, double* loss, double* grads) {
    return guarded([&] {
        hcva_ctx* ctx = sim->ctx;
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (!sim->has_defaults || !sim->has_cube) throw contract_error("quadratic_loss: set has no defaults / cube");
        if (step < 1 || step > sim->n) throw contract_error("label step out of range");
        const long R = static_cast<long>(sim->M) * sim->N;
        if (b0 < 0 || b1 > R || b1 <= b0) throw contract_error("quadratic_loss: bad row range");
        const int d = sim->model.Cc * 2 + 3 * sim->model.E - 1;
        const NetDims n = dims_from(cfg, d);
        if (sim->labels_kind != label_kind) launch_labels_all(sim, label_kind);
        Trainer tr(ctx, n, b1 - b0, R, use_split(n, sim));
        if (tr.split) tr.split_source(sim);
        DeviceBuf dmean, dscale, X;
        stage(dmean, std::vector<double>(mean, mean + d));
        stage(dscale, std::vector<double>(scale, scale + d));
        FeatArgs fa = feat_args(sim, step);
        fa.mean = dmean.as<double>();
        fa.scale = dscale.as<double>();
        if (!tr.use_tc) X.alloc(sizeof(float) * R * d);
        build_features(tr, fa, X, R);
        tr.set_params(params);
        SplitPartials sp;
        const double* y = sim->labels.as<double>() + static_cast<size_t>(step) * R;
        const int tiles = tr.grad_tiles(X.as<float>(), y, b0, b1, head, static_cast<double>(b1 - b0), &sp);
        reduce_partials(tr, tiles, sp, b1 - b0, loss, grads);
    });
}

// forward (regressor.cpp:97-113) with the positive head on, as
// TrainedModelSequence::predict applies it (regressor.cpp:349-352), on host
// rows that are already standardised.
hcva_status hcva_forward(hcva_ctx* ctx, const hcva_train_cfg* cfg, int input_dim, const double* params,
                         const double* x, int rows, double* out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (rows < 1) throw contract_error("forward: no rows");
        const NetDims n = dims_from(cfg, input_dim);
        Trainer tr(ctx, n, 1, rows);
        DeviceBuf dX, pred;
        stage_features(tr, x, rows, input_dim, dX);
        pred.alloc(static_cast<size_t>(rows) * 8);
        tr.set_params(params);
        tr.eval(dX.as<float>(), nullptr, rows, 4, pred.as<double>());
        copy_out(ctx, out, pred.p, static_cast<size_t>(rows) * 8);
    });
}

// refit_output_layer (regressor.cpp:191-213): the output layer of `params`
// (positive head off) replaced by the ridge least-squares fit on [z_h, 1]
// against y - mu: Gram on the device in FP64 from the FP32 activations, LDL^T
// solve in FP64.
hcva_status hcva_refit_output_layer(hcva_ctx* ctx, const hcva_train_cfg* cfg, int input_dim, double* params,
                                    const double* x, const double* y, int rows) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (rows < 1) throw contract_error("refit_output_layer: no rows");
        const NetDims n = dims_from(cfg, input_dim);
        Trainer tr(ctx, n, 1, rows);
        DeviceBuf dX, dy;
        stage_features(tr, x, rows, input_dim, dX);
        stage(dy, std::vector<double>(y, y + rows));
        tr.set_params(params);
        tr.refit(dX.as<float>(), dy.as<double>(), rows, cfg->ridge);
        copy_out(ctx, params, tr.p64.p, static_cast<size_t>(n.P) * 8);
    });
}

// Roofline probe of the SGD step (bench.py): train_base's inner loop at step
// `step` of a simulated set (scaler, features, Glorot init with mu = label
// mean), three untimed SGD steps, then `steps` SGD steps over consecutive
// batches with CUDA events on the engine's stream around every step and after
// its gradient kernels.  out = mean ms of [whole step, gradient kernels,
// optimizer], and the number of gradient partial rows per step.
hcva_status hcva_diag_sgd_timing(hcva_sim* sim, const hcva_train_cfg* cfg, int step, int label_kind, int steps,
                                 double* out) {
    return guarded([&] {
        hcva_ctx* ctx = sim->ctx;
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (steps < 1 || step < 1 || step > sim->n) throw contract_error("sgd timing: bad step / count");
        const long R = static_cast<long>(sim->M) * sim->N;
        if (cfg->n_batches < 1 || R % cfg->n_batches) throw config_error("make_batches: batch count must divide M*N");
        const long bs = R / cfg->n_batches;
        const int d = sim->model.Cc * 2 + 3 * sim->model.E - 1;
        const NetDims n = dims_from(cfg, d);
        if (sim->labels_kind != label_kind) launch_labels_all(sim, label_kind);
        Trainer tr(ctx, n, bs, R, use_split(n, sim));
        if (tr.split) tr.split_source(sim);
        DeviceBuf mean, scale, X;
        mean.alloc(static_cast<size_t>(d) * 8);
        scale.alloc(static_cast<size_t>(d) * 8);
        FeatArgs fa = feat_args(sim, step);
        k_scaler<<<d, 256, 0, ctx->stream>>>(fa, mean.as<double>(), scale.as<double>());
        fa.mean = mean.as<double>();
        fa.scale = scale.as<double>();
        if (!tr.use_tc) X.alloc(sizeof(float) * R * d);
        build_features(tr, fa, X, R);
        const double* y = sim->labels.as<double>() + static_cast<size_t>(step) * R;
        const auto p = init_params(n, split_key(split_key(root_key(cfg->seed), 0xBEEF), step));
        tr.set_params(p.data());
        HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
        k_set_mu_mean<<<1, 1024, 0, ctx->stream>>>(y, R, tr.p64.as<double>(), tr.p32.as<float>(), n.P);
        HCVA_CUDA(cudaMemsetAsync(tr.m.p, 0, n.P * 8, ctx->stream));
        HCVA_CUDA(cudaMemsetAsync(tr.v.p, 0, n.P * 8, ctx->stream));
        tr.wimg_valid = false;
        auto run = [&](long t) {
            const long b = t % cfg->n_batches;
            tr.sgd_step(X.as<float>(), y, b * bs, (b + 1) * bs, 0, t + 1, cfg->learning_rate, cfg->adam);
        };
        for (long w = 0; w < 3; ++w) run(w);
        std::vector<cudaEvent_t> ev(3 * static_cast<size_t>(steps));
        for (auto& e : ev) HCVA_CUDA(cudaEventCreate(&e));
        for (int s = 0; s < steps; ++s) {
            HCVA_CUDA(cudaEventRecord(ev[3 * s], ctx->stream));
            tr.phase_ev = &ev[3 * s + 1];
            run(3 + s);
        }
        tr.phase_ev = nullptr;
        if (tr.split && std::getenv("HCVA_SPLIT_TRACE")) {  // profiling: phase clocks of one more step
            DeviceBuf tb;
            tb.alloc(96 * 8);
            HCVA_CUDA(cudaMemsetAsync(tb.p, 0, 96 * 8, ctx->stream));
            tr.sa.trace = tb.as<long long>();
            run(3 + steps);
            tr.sa.trace = nullptr;
            long long h[80];
            copy_out(ctx, h, tb.p, sizeof h);
            for (int t = 0; t < 4; ++t) {
                std::fprintf(stderr, "tile %d:", t);
                for (int k = 1; k <= 10; ++k) std::fprintf(stderr, " %lld", h[t * 16 + k] - h[t * 16 + k - 1]);
                std::fprintf(stderr, "\n");
            }
            std::fprintf(stderr, "fixed:");
            for (int k = 1; k < 8; ++k) std::fprintf(stderr, " %lld", h[64 + k] - h[64 + k - 1]);
            std::fprintf(stderr, " | tail:");
            for (int k = 8; k < 13; ++k) std::fprintf(stderr, " %lld", h[64 + k] - h[64 + 5]);
            std::fprintf(stderr, "  entry->tile0 %lld, tile3 end->final %lld\n", h[0] - h[64], h[67] - h[3 * 16 + 10]);
        }
        out[4] = 0.0;
        if (tr.fusable(bs, cfg->n_batches)) {  // the persistent epoch: mean ms per SGD step
            const int nb = cfg->n_batches;
            std::vector<double> h(2 * static_cast<size_t>(nb));
            for (int s = 0; s < nb; ++s) {
                h[2 * s] = 1.0 - std::pow(0.9, static_cast<double>(4 + steps + s));
                h[2 * s + 1] = 1.0 - std::pow(0.999, static_cast<double>(4 + steps + s));
            }
            if (tr.c12.bytes < h.size() * 8) tr.c12.alloc(h.size() * 8);
            HCVA_CUDA(cudaMemcpyAsync(tr.c12.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
            tr.sgd_epoch(y, bs, nb, 0, tr.c12.as<double>(), cfg->learning_rate, cfg->adam);  // warm-up
            cudaEvent_t f0, f1;
            HCVA_CUDA(cudaEventCreate(&f0));
            HCVA_CUDA(cudaEventCreate(&f1));
            HCVA_CUDA(cudaEventRecord(f0, ctx->stream));
            const bool ran = tr.sgd_epoch(y, bs, nb, 0, tr.c12.as<double>(), cfg->learning_rate, cfg->adam);
            HCVA_CUDA(cudaEventRecord(f1, ctx->stream));
            HCVA_CUDA(cudaEventSynchronize(f1));
            float ms = 0.f;
            HCVA_CUDA(cudaEventElapsedTime(&ms, f0, f1));
            cudaEventDestroy(f0);
            cudaEventDestroy(f1);
            if (ran) out[4] = ms / nb;
            if (ran && std::getenv("HCVA_SPLIT_TRACE")) {
                DeviceBuf tb;
                tb.alloc(96 * 8);
                HCVA_CUDA(cudaMemsetAsync(tb.p, 0, 96 * 8, ctx->stream));
                tr.sa.trace = tb.as<long long>();
                tr.sgd_epoch(y, bs, nb, 0, tr.c12.as<double>(), cfg->learning_rate, cfg->adam);
                tr.sa.trace = nullptr;
                long long hh[96];
                copy_out(ctx, hh, tb.p, sizeof hh);
                std::fprintf(stderr, "fused last step start (cycles): weights+P %lld | first tile staged %lld | to tile 0 %lld"
                             " | adam: gather %lld, sums %lld\n",
                             hh[81] - hh[80], hh[65] - hh[81], hh[0] - hh[65], hh[82] - hh[77], hh[83] - hh[82]);
                std::fprintf(stderr, "fused last step (cycles): tiles %lld | final wait + readout %lld | partials %lld"
                             " | sync1 %lld | adam %lld | sync2 %lld | step total %.0f\n",
                             hh[67] - hh[66], hh[69] - hh[67], hh[70] - hh[69], hh[77] - hh[70], hh[78] - hh[77],
                             hh[79] - hh[78], ms / nb * 1.965e6);
                std::fprintf(stderr, "per-tile (last step):");
                for (int t = 0; t < 4; ++t) std::fprintf(stderr, " %lld", hh[t * 16 + 10] - hh[t * 16]);
                std::fprintf(stderr, "\n");
            }
        }
        HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
        double tot = 0.0, grad = 0.0, opt = 0.0;
        for (int s = 0; s < steps; ++s) {
            float a = 0.f, b = 0.f;
            HCVA_CUDA(cudaEventElapsedTime(&a, ev[3 * s], ev[3 * s + 1]));
            HCVA_CUDA(cudaEventElapsedTime(&b, ev[3 * s + 1], ev[3 * s + 2]));
            grad += a, opt += b, tot += a + b;
        }
        for (auto e : ev) cudaEventDestroy(e);
        tr.check_finite();
        out[0] = tot / steps, out[1] = grad / steps, out[2] = opt / steps, out[3] = tr.split ? 1.0 : 0.0;
    });
}

hcva_status hcva_train_base(hcva_ctx* ctx, const hcva_train_cfg* cfg, int input_dim, const double* x,
                            const double* y, int rows, const double* init, double* best, double* epoch_losses,
                            double* best_loss, int* best_epoch) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const NetDims n = dims_from(cfg, input_dim);
        if (cfg->n_batches < 1 || rows % cfg->n_batches != 0)
            throw config_error("make_batches: batch count must divide M*N");
        Trainer tr(ctx, n, rows / cfg->n_batches, rows);
        DeviceBuf dX, dy, dl;
        stage_features(tr, x, rows, input_dim, dX);
        stage(dy, std::vector<double>(y, y + rows));
        dl.alloc(sizeof(double) * std::max(cfg->epochs, 1));
        tr.set_params(init);
        tr.train_base(dX.as<float>(), dy.as<double>(), rows, cfg->epochs, cfg->n_batches, cfg->learning_rate,
                      cfg->adam, cfg->ridge, dl.as<double>());
        tr.check_finite();
        copy_out(ctx, best, tr.best.p, n.P * 8);
        copy_out(ctx, epoch_losses, dl.p, cfg->epochs * 8);
        copy_out(ctx, best_loss, tr.best_loss.p, 8);
        copy_out(ctx, best_epoch, tr.best_epoch.p, 4);
    });
}

// backward_learn (regressor.cpp:354-395) over a simulated set with the label
// source of pipeline.cpp:72-111 (features_at + defaults_/intensity_label).
static hcva_status hcva_backward_learn_ex(hcva_sim* sim, const hcva_train_cfg* cfg, int label_kind, hcva_comm* comm,
                                          uint64_t probe_key, double* qr_trace, hcva_models** out);

hcva_status hcva_backward_learn(hcva_sim* sim, const hcva_train_cfg* cfg, int label_kind, hcva_models** out) {
    return hcva_backward_learn_dist(sim, cfg, label_kind, nullptr, out);
}

hcva_status hcva_backward_learn_dist(hcva_sim* sim, const hcva_train_cfg* cfg, int label_kind, hcva_comm* comm,
                                     hcva_models** out) {
    return hcva_backward_learn_ex(sim, cfg, label_kind, comm, 0, nullptr, out);
}

hcva_status hcva_backward_learn_qr(hcva_sim* sim, const hcva_train_cfg* cfg, int label_kind, uint64_t probe_key,
                                   double* trace, hcva_models** out) {
    if (!trace) return hcva_backward_learn_ex(sim, cfg, label_kind, nullptr, 0, nullptr, out);
    return hcva_backward_learn_ex(sim, cfg, label_kind, nullptr, probe_key, trace, out);
}

static hcva_status hcva_backward_learn_ex(hcva_sim* sim, const hcva_train_cfg* cfg, int label_kind, hcva_comm* comm,
                                          uint64_t probe_key, double* qr_trace, hcva_models** out) {
    return guarded([&] {
        hcva_ctx* ctx = sim->ctx;
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (!sim->has_defaults || !sim->has_cube) throw contract_error("backward_learn: simulate a full set first");
        if (sim->start_step != 0) throw contract_error("labels expect an outer (non-rebased) market block");
        if (label_kind != 0 && label_kind != 1) throw config_error("config: label_kind must be 'defaults' or 'intensity'");
        const int Cc = sim->model.Cc, E = sim->model.E, nsteps = sim->n;
        const int d = Cc + 3 * E - 1 + Cc;
        const NetDims n = dims_from(cfg, d);
        const long R = static_cast<long>(sim->M) * sim->N;
        if (cfg->n_batches < 1 || R % cfg->n_batches != 0) throw config_error("make_batches: batch count must divide M*N");
        auto models = std::make_unique<hcva_models>();
        models->ctx = ctx;
        models->n = n;
        models->n_steps = nsteps;
        models->epochs = cfg->epochs;
        models->params.alloc(static_cast<size_t>(nsteps) * n.P * 8);
        models->mean.alloc(static_cast<size_t>(nsteps) * d * 8);
        models->scale.alloc(static_cast<size_t>(nsteps) * d * 8);
        models->losses.alloc(static_cast<size_t>(nsteps) * std::max(cfg->epochs, 1) * 8);
        models->best_loss.alloc(static_cast<size_t>(nsteps) * 8);
        models->best_epoch.alloc(static_cast<size_t>(nsteps) * 4);
        if (sim->labels_kind != label_kind) launch_labels_all(sim, label_kind);
        Trainer tr(ctx, n, R / cfg->n_batches, R, use_split(n, sim));
        if (tr.split) tr.split_source(sim);
        const int mm = n.u + 1;
        tr.set_comm(comm, std::max<size_t>({static_cast<size_t>(n.P) + 1, static_cast<size_t>(mm * (mm + 1) / 2 + mm),
                                            static_cast<size_t>(d)}));
        const int world = tr.world;
        HCVA_CUDA(cudaMemsetAsync(tr.flag.p, 0, 4, ctx->stream));
        DeviceBuf X;
        if (!tr.use_tc) X.alloc(sizeof(float) * R * d);
        // Q/R probe (pipeline.cpp:79-108, regressor.cpp:328-338): two extra
        // replicas per path; after every epoch the current network (positive
        // head) predicts both, g_t = squared errors, estimate_qr on the host.
        const bool probe = qr_trace != nullptr;
        if (probe && comm) throw contract_error("Q/R probe: single-GPU runs only");
        DeviceBuf p_steps, p_labels, p_img, p_X, p_pred, p_g;
        const long R2 = 2L * sim->M;
        const double* p_y = nullptr;  // this step's probe labels (device)
        size_t trace_row = 0;
        int cur_step = 0;
        if (probe) {
            probe_block(sim, probe_key, label_kind, p_steps, p_labels);
            if (tr.split) { /* the probe rows reuse this step's per-path columns */ }
            else if (tr.use_tc) p_img.alloc(static_cast<size_t>((R2 + 127) / 128) * tc_x_tile_bytes(tr.dp));
            else p_X.alloc(sizeof(float) * R2 * d);
            p_pred.alloc(sizeof(double) * R2);
            p_g.alloc(sizeof(double) * R2);
            tr.on_epoch = [&](int epoch) {
                tr.ximg_over = tr.use_tc && !tr.split ? p_img.as<uint8_t>() : nullptr;
                SplitArgs p_sa = tr.sa;  // the probe's two replicas per path
                p_sa.steps = p_steps.as<uint16_t>();
                p_sa.N = 2;
                p_sa.R = R2;
                tr.sa_over = tr.split ? &p_sa : nullptr;
                tr.eval(p_X.as<float>(), nullptr, R2, 4, p_pred.as<double>());
                tr.ximg_over = nullptr;
                tr.sa_over = nullptr;
                // g[k] = (squared error of replica 0, of replica 1): already the pair layout
                k_sq_err<<<grid1(R2, 256), 256, 0, ctx->stream>>>(p_pred.as<double>(), p_y, R2, p_g.as<double>());
                ctx->launches++;
                double qr[6];
                estimate_qr_device(ctx, p_g.as<double>(), sim->M, qr);
                double* row = qr_trace + 4 * trace_row++;
                row[0] = cur_step;
                row[1] = epoch;
                row[2] = qr[0];
                row[3] = qr[1];
            };
        }
        NvtxRange nvtx_all("hcva_backward_learn");
        for (int i = nsteps; i >= 1; --i) {
            NvtxRange nvtx_step("train_base (pricing step)");
            FeatArgs fa = feat_args(sim, i);
            double* mean = models->mean.as<double>() + static_cast<size_t>(i - 1) * d;
            double* scale = models->scale.as<double>() + static_cast<size_t>(i - 1) * d;
            if (!comm) {
                k_scaler<<<d, 256, 0, ctx->stream>>>(fa, mean, scale);
            } else {  // moments over every rank's paths: sums, gathered, then centred sums
                const double Mt = static_cast<double>(sim->M) * world;
                k_scaler_moment<<<d, 256, 0, ctx->stream>>>(fa, 0, mean, tr.red.as<double>());
                k_scaler_fin<<<1, 64, 0, ctx->stream>>>(tr.gather(tr.red.as<double>(), d), world, d, Cc, Mt, 0, mean,
                                                        scale);
                k_scaler_moment<<<d, 256, 0, ctx->stream>>>(fa, 1, mean, tr.red.as<double>());
                k_scaler_fin<<<1, 64, 0, ctx->stream>>>(tr.gather(tr.red.as<double>(), d), world, d, Cc, Mt, 1, mean,
                                                        scale);
            }
            check_launch(ctx);
            fa.mean = mean;
            fa.scale = scale;
            build_features(tr, fa, X, R);
            if (probe) {  // the probe rows, standardised with this step's scaler
                FeatArgs fp = fa;
                fp.N = 2;
                fp.steps = p_steps.as<uint16_t>();
                build_features(tr, fp, p_X, R2, &p_img);
                p_y = p_labels.as<double>() + static_cast<size_t>(i) * R2;
                cur_step = i;
            }
            const double* y = sim->labels.as<double>() + static_cast<size_t>(i) * R;
            if (i == nsteps) {
                const auto p = init_params(n, split_key(split_key(root_key(cfg->seed), 0xBEEF), i));
                tr.set_params(p.data());
                HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
                if (!comm) {
                    k_set_mu_mean<<<1, 1024, 0, ctx->stream>>>(y, R, tr.p64.as<double>(), tr.p32.as<float>(), n.P);
                } else {
                    k_local_sum<<<1, 1024, 0, ctx->stream>>>(y, R, tr.red.as<double>());
                    k_set_mu_from<<<1, 1, 0, ctx->stream>>>(tr.gather(tr.red.as<double>(), 1), world,
                                                            static_cast<double>(R) * world, tr.p64.as<double>(),
                                                            tr.p32.as<float>(), n.P);
                }
                tr.wimg_valid = false;
                check_launch(ctx);
            } else {
                tr.set_params(tr.best.as<double>());  // warm start from step i+1's best
            }
            tr.train_base(X.as<float>(), y, R, cfg->epochs, cfg->n_batches, cfg->learning_rate, cfg->adam, cfg->ridge,
                          models->losses.as<double>() + static_cast<size_t>(i - 1) * cfg->epochs);
            HCVA_CUDA(cudaMemcpyAsync(models->params.as<double>() + static_cast<size_t>(i - 1) * n.P, tr.best.p, n.P * 8,
                                      cudaMemcpyDeviceToDevice, ctx->stream));
            HCVA_CUDA(cudaMemcpyAsync(models->best_loss.as<double>() + (i - 1), tr.best_loss.p, 8,
                                      cudaMemcpyDeviceToDevice, ctx->stream));
            HCVA_CUDA(cudaMemcpyAsync(models->best_epoch.as<int>() + (i - 1), tr.best_epoch.p, 4,
                                      cudaMemcpyDeviceToDevice, ctx->stream));
        }
        tr.check_finite();
        *out = models.release();
    });
}

hcva_status hcva_models_info(const hcva_models* m, int* info) {
    return guarded([&] {
        info[0] = m->n_steps;
        info[1] = m->n.d;
        info[2] = m->n.P;
        info[3] = m->epochs;
    });
}

hcva_status hcva_models_get(const hcva_models* m, int step, double* params, double* mean, double* scale,
                            double* epoch_losses, double* best_loss, int* best_epoch) {
    return guarded([&] {
        StreamScope sc__(m->ctx->stream);
        if (step < 1 || step > m->n_steps) throw contract_error("models: step out of range");
        const size_t s = step - 1;
        if (params) copy_out(m->ctx, params, m->params.as<double>() + s * m->n.P, m->n.P * 8);
        if (mean) copy_out(m->ctx, mean, m->mean.as<double>() + s * m->n.d, m->n.d * 8);
        if (scale) copy_out(m->ctx, scale, m->scale.as<double>() + s * m->n.d, m->n.d * 8);
        if (epoch_losses) copy_out(m->ctx, epoch_losses, m->losses.as<double>() + s * m->epochs, m->epochs * 8);
        if (best_loss) copy_out(m->ctx, best_loss, m->best_loss.as<double>() + s, 8);
        if (best_epoch) copy_out(m->ctx, best_epoch, m->best_epoch.as<int>() + s, 4);
    });
}

// TrainedModelSequence::predict (regressor.cpp:349-352) on a simulated set's
// features at `step` (e.g. the validation set, pipeline.cpp:138-156).
hcva_status hcva_predict(const hcva_models* m, hcva_sim* sim, int step, double* out) {
    return guarded([&] {
        NvtxRange nvtx__("hcva_predict");
        hcva_ctx* ctx = sim->ctx;
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (step < 1 || step > m->n_steps) throw contract_error("models: step out of range");
        if (!sim->has_defaults) throw contract_error("predict: no default block");
        const int d = sim->model.Cc * 2 + 3 * sim->model.E - 1;
        if (d != m->n.d) throw contract_error("forward: feature dimension mismatch");
        const long R = static_cast<long>(sim->M) * sim->N;
        Trainer tr(ctx, m->n, 1, R, use_split(m->n, sim, false));
        if (tr.split) tr.split_source(sim);
        tr.set_params(m->params.as<double>() + static_cast<size_t>(step - 1) * m->n.P);
        FeatArgs fa = feat_args(sim, step);
        fa.mean = m->mean.as<double>() + static_cast<size_t>(step - 1) * d;
        fa.scale = m->scale.as<double>() + static_cast<size_t>(step - 1) * d;
        DeviceBuf X, pred;
        if (!tr.use_tc) X.alloc(sizeof(float) * R * d);
        pred.alloc(sizeof(double) * R);
        build_features(tr, fa, X, R);
        tr.eval(X.as<float>(), nullptr, R, 4, pred.as<double>());
        copy_out(ctx, out, pred.p, R * 8);
    });
}

// percentile_table (pipeline.cpp:138-156): per step i = 1..n the out-of-sample
// predictions on the validation set, sorted on the device; out [n][6] = step,
// mean, p1, p2.5, p97.5, p99 (percentile_sorted's linear interpolation).
hcva_status hcva_percentile_table(const hcva_models* m, hcva_sim* sim, double* out) {
    return guarded([&] {
        NvtxRange nvtx__("hcva_percentile_table");
        hcva_ctx* ctx = sim->ctx;
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (!sim->has_defaults) throw contract_error("predict: no default block");
        const int d = sim->model.Cc * 2 + 3 * sim->model.E - 1;
        if (d != m->n.d) throw contract_error("forward: feature dimension mismatch");
        const long R = static_cast<long>(sim->M) * sim->N;
        Trainer tr(ctx, m->n, 1, R, use_split(m->n, sim, false));
        if (tr.split) tr.split_source(sim);
        DeviceBuf X, pred;
        if (!tr.use_tc) X.alloc(sizeof(float) * R * d);
        pred.alloc(sizeof(double) * R);
        for (int i = 1; i <= m->n_steps; ++i) {
            tr.set_params(m->params.as<double>() + static_cast<size_t>(i - 1) * m->n.P);
            FeatArgs fa = feat_args(sim, i);
            fa.mean = m->mean.as<double>() + static_cast<size_t>(i - 1) * d;
            fa.scale = m->scale.as<double>() + static_cast<size_t>(i - 1) * d;
            build_features(tr, fa, X, R);
            tr.eval(X.as<float>(), nullptr, R, 4, pred.as<double>());
            double* row = out + 6 * static_cast<size_t>(i - 1);
            row[0] = i;
            percentile_bands(ctx, pred.as<double>(), R, row + 1);
        }
    });
}

// ---- HCVAMDL1 model files (TrainedModelSequence::save/load, regressor.cpp:397-481):
// magic, u32 version 1, u64 seed, i32 n_steps, u32 + bytes config hash; per
// step i32 layers (h+1), i32 activation, f64 mu, then every weight, every
// bias, scaler mean and scale as (i64 rows, i64 cols, column-major f64).
}  // extern "C"

namespace {

template <typename T>
void put(std::ofstream& o, T v) {
    o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T get(std::ifstream& in) {
    T v;
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) throw numeric_error("model file truncated");
    return v;
}
constexpr char kModelMagic[8] = {'H', 'C', 'V', 'A', 'M', 'D', 'L', '1'};

}  // namespace

extern "C" {

hcva_status hcva_models_save(const hcva_models* m, const char* path, uint64_t seed, const char* config_hash) {
    return guarded([&] {
        StreamScope sc__(m->ctx->stream);
        const NetDims& n = m->n;
        const int S = m->n_steps, d = n.d;
        std::vector<double> p(static_cast<size_t>(S) * n.P), mean(static_cast<size_t>(S) * d), scale(mean.size());
        copy_out(m->ctx, p.data(), m->params.p, p.size() * 8);
        copy_out(m->ctx, mean.data(), m->mean.p, mean.size() * 8);
        copy_out(m->ctx, scale.data(), m->scale.p, scale.size() * 8);
        std::ofstream o(path, std::ios::binary);
        if (!o) throw config_error(std::string("cannot write model file ") + path);
        const std::string hash = config_hash ? config_hash : "";
        o.write(kModelMagic, 8);
        put<uint32_t>(o, 1u);
        put<uint64_t>(o, seed);
        put<int32_t>(o, S);
        put<uint32_t>(o, static_cast<uint32_t>(hash.size()));
        o.write(hash.data(), static_cast<std::streamsize>(hash.size()));
        for (int s = 0; s < S; ++s) {
            const double* q = p.data() + static_cast<size_t>(s) * n.P;
            put<int32_t>(o, n.h + 1);
            put<int32_t>(o, n.act);
            put<double>(o, q[n.P - 1]);
            for (int l = 0; l <= n.h; ++l) {
                put<int64_t>(o, n.fout[l]);
                put<int64_t>(o, n.fin[l]);
                for (int c = 0; c < n.fin[l]; ++c)
                    for (int r = 0; r < n.fout[l]; ++r) put<double>(o, q[n.off[l] + r * n.fin[l] + c]);
            }
            for (int l = 0; l <= n.h; ++l) {
                put<int64_t>(o, n.fout[l]);
                put<int64_t>(o, 1);
                for (int r = 0; r < n.fout[l]; ++r) put<double>(o, q[n.off[l] + n.fout[l] * n.fin[l] + r]);
            }
            for (const std::vector<double>* v : {&mean, &scale}) {
                put<int64_t>(o, d);
                put<int64_t>(o, 1);
                for (int j = 0; j < d; ++j) put<double>(o, (*v)[static_cast<size_t>(s) * d + j]);
            }
        }
        if (!o) throw config_error(std::string("cannot write model file ") + path);
    });
}

hcva_status hcva_models_load(hcva_ctx* ctx, const char* path, uint64_t* seed, char* config_hash, int hash_capacity,
                             hcva_models** out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        std::ifstream in(path, std::ios::binary);
        if (!in) throw config_error(std::string("cannot open model file ") + path);
        char magic[8];
        in.read(magic, 8);
        if (!in || std::memcmp(magic, kModelMagic, 8) != 0) throw config_error(std::string("not a model file: ") + path);
        if (get<uint32_t>(in) != 1u) throw config_error("unsupported model file version");
        const uint64_t sd = get<uint64_t>(in);
        const int S = get<int32_t>(in);
        const uint32_t hl = get<uint32_t>(in);
        std::string hash(hl, '\0');
        in.read(hash.data(), hl);
        if (!in) throw numeric_error("model file truncated");
        if (S < 1) throw contract_error("model file: no steps");
        auto matrix = [&](int64_t want_r, int64_t want_c, std::vector<double>& v) {
            const int64_t r = get<int64_t>(in), c = get<int64_t>(in);
            if ((want_r >= 0 && r != want_r) || (want_c >= 0 && c != want_c) || r < 0 || c < 0)
                throw contract_error("model file: inconsistent network shapes");
            v.resize(static_cast<size_t>(r * c));
            in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(sizeof(double) * v.size()));
            if (!in) throw numeric_error("model file truncated");
            return std::pair<int64_t, int64_t>(r, c);
        };
        NetDims n{};
        std::vector<double> params, means, scales;
        for (int s = 0; s < S; ++s) {
            const int layers = get<int32_t>(in), act = get<int32_t>(in);
            const double mu = get<double>(in);
            std::vector<std::vector<double>> W(layers), B(layers);
            std::vector<std::pair<int64_t, int64_t>> shape(layers);
            for (int l = 0; l < layers; ++l) shape[l] = matrix(-1, -1, W[l]);
            if (s == 0) {
                if (layers < 2) throw contract_error("model file: inconsistent network shapes");
                n = make_dims(static_cast<int>(shape[0].second), layers - 1, static_cast<int>(shape[0].first), act);
                params.assign(static_cast<size_t>(S) * n.P, 0.0);
                means.assign(static_cast<size_t>(S) * n.d, 0.0);
                scales.assign(means.size(), 0.0);
            }
            if (layers != n.h + 1 || act != n.act) throw contract_error("model file: inconsistent network shapes");
            double* q = params.data() + static_cast<size_t>(s) * n.P;
            for (int l = 0; l < layers; ++l) {
                if (shape[l].first != n.fout[l] || shape[l].second != n.fin[l])
                    throw contract_error("model file: inconsistent network shapes");
                for (int c = 0; c < n.fin[l]; ++c)
                    for (int r = 0; r < n.fout[l]; ++r)
                        q[n.off[l] + r * n.fin[l] + c] = W[l][static_cast<size_t>(c) * n.fout[l] + r];
            }
            for (int l = 0; l < layers; ++l) {
                matrix(n.fout[l], 1, B[l]);
                for (int r = 0; r < n.fout[l]; ++r) q[n.off[l] + n.fout[l] * n.fin[l] + r] = B[l][r];
            }
            q[n.P - 1] = mu;
            std::vector<double> v;
            matrix(n.d, 1, v);
            std::copy(v.begin(), v.end(), means.begin() + static_cast<size_t>(s) * n.d);
            matrix(n.d, 1, v);
            std::copy(v.begin(), v.end(), scales.begin() + static_cast<size_t>(s) * n.d);
        }
        auto models = std::make_unique<hcva_models>();
        models->ctx = ctx;
        models->n = n;
        models->n_steps = S;
        models->epochs = 0;  // reports are not part of the file
        stage(models->params, params);
        stage(models->mean, means);
        stage(models->scale, scales);
        models->losses.alloc(8);
        stage(models->best_loss, std::vector<double>(S, 0.0));
        stage(models->best_epoch, std::vector<int>(S, 0));
        HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
        if (seed) *seed = sd;
        if (config_hash && hash_capacity > 0) {
            const size_t k = std::min<size_t>(hash.size(), static_cast<size_t>(hash_capacity - 1));
            std::memcpy(config_hash, hash.data(), k);
            config_hash[k] = '\0';
        }
        *out = models.release();
    });
}

hcva_status hcva_models_destroy(hcva_models* m) {
    return guarded([&] {
        if (!m) return;
        cudaStreamSynchronize(m->ctx->stream);
        delete m;
    });
}

}  // extern "C"
