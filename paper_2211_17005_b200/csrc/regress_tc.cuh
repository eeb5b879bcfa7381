// regress_tc.cuh -- launch interface of the tensor-core regression kernels (regress_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace hcva {

// Byte sizes of the packed operand images (3xTF32 hi / lo planes in the
// canonical K-major core layout, tc.cuh).
size_t tc_weight_image_bytes(int u, int dp);  // W0 | W1 | W1^T planes + bias vector block
size_t tc_x_tile_bytes(int dp);               // one 128-row feature tile, hi | lo

struct TileArgs {
    int d, dp, act, P, off0, off1, off2;
    const uint8_t* wimg;  // packed weights (k_pack_w)
    const uint8_t* ximg;  // packed feature tiles [R/128][hi | lo] (k_pack_x)
    const double* y;      // labels, absolute row index
    long b0, b1;          // live rows [b0, b1)
    int head, mode;       // mode 0: SGD; else bits 1: loss (head on), 2: min plain fit, 4: predictions,
                          //   8: layer-2 activations -> H2 (refit Gram)
    double nb;
    float* gpart;    // SGD: [cta][P] partials of b0, b1, w2, b2, mu
    double* lpart;   // [cta] sum of squared residuals
    double* mpart;   // [cta] min of f + mu (plain head)
    double* pred;    // predictions (head on), absolute row index
    float* H2;       // [R][U] layer-2 activations (mode bit 8)
    float *H1t, *G2t, *G1t;  // SGD: [U][ld_t] transposed, row index relative to b0
    long ld_t;
    int xf32;                // feature tiles are one FP32 plane (tc_two_cta shapes), else hi | lo planes
};

struct WgradArgs {
    int d, dp, P, off0, off1;
    const float *G2t, *H1t, *G1t;  // [U][ld_t]
    long ld_t;
    const float* Xt;               // [dp][ld_x] transposed features, column = absolute row
    long ld_x, row0, rows;         // rows of the batch (relative index 0..rows-1)
    int rows_per_cta;              // multiple of the chunk (set by the launcher)
    int probe;                     // profiling: skip the row loop
    float* gpart;                  // [cta][U*U + U*dp]: W1 rows, then W0 rows padded to dp
};

// Layer-0 split (regress_split.cu): the feature row of replica (k, l) at
// step i is [1{s_klc <= i} (c = 1..Cc), y_k (q per-path market columns)], so
// W0 x = W0_ind 1{s <= i} + (b0 + W0_y y_k): the per-path part is computed
// once per path per tile, the indicator part from the default steps; the
// feature matrix is never built.
struct SplitArgs {
    int d, Cc, q, qp, N, step, P, off0, off1, off2, act;
    long M, R;                 // paths and rows of the set
    const float* yhat;         // [M][qp] standardised per-path columns of this step
    const uint16_t* steps;     // [Cn][R] default steps (name 0 = bank)
    const uint8_t* w1img;      // W1 hi | lo, W1^T hi | lo planes of the weight image
    const float* vec;          // b0 | b1 | w2 | b2, mu of the weight image
    const float* p32;          // FP32 parameters (W0 columns)
    const double* mu64;        // FP64 master copy of mu
    const double* y;           // labels [R]
    long b0, b1;               // live rows
    int head, mode;            // mode 0: SGD; else TileArgs::mode bits (1 loss, 2 min, 4 pred, 8 H2)
    double nb;
    float* gpart;              // SGD: [cta][P] gradient partials (every parameter)
    double* lpart;             // [cta] sum of squared residuals
    double* mpart;             // [cta] min of f + mu
    double* pred;              // predictions, absolute row
    float* H2;                 // [R][U] layer-2 activations (mode 8)
    long long* trace;          // profiling: phase clocks of CTA 0 (HCVA_SPLIT_TRACE), or null
    const float* Pg;           // evaluation: layer-0 path parts [M][64] (k_path_proj)
    float* Pg_out;             // evaluation: where the launcher writes them
    // Persistent SGD (fuse != 0): nsteps steps over consecutive batches of bs rows
    // from b0, the optimizer fused behind grid barriers (cooperative launch).
    int fuse, nsteps;
    long bs;
    double lr;
    int adam, dp;
    double *p64w, *m, *v;      // FP64 master parameters, Adam moments
    float* p32w;               // FP32 parameters (the same buffer as p32)
    uint8_t* img;              // weight image (W1, W1^T planes and vectors refreshed in place)
    unsigned* gbar;            // grid-barrier counter (zeroed before the launch)
    int* nonfinite;
    const double* c12;         // [nsteps][2] Adam bias corrections 1 - beta^t (host libm pow)
};
// Persistent SGD over a.nsteps batches; false if the grid would not be co-resident.
bool launch_sgd_split_fused(const SplitArgs& a, int sm_count, cudaStream_t s);
// Shapes served by the split kernels: U = 64, two hidden layers, Cc <= 8,
// q <= 48; the SGD kernel also needs N >= 16 replicas per path (<= 9 paths
// per 128-row tile), the evaluation kernel any N.
bool split_eligible(int u, int h, int N, int Cc, int q);
// Returns the number of per-CTA partials written.
int launch_sgd_split(const SplitArgs& a, int sm_count, cudaStream_t s);
int launch_eval_split(const SplitArgs& a, int sm_count, cudaStream_t s);
int split_max_ctas(int sm_count);

bool tc_eligible(int d, int h, int u);
// Shapes served by the two-CTA-per-SM kernels (k_sgd_tc / k_eval_tc): their
// feature tiles are one FP32 plane, split into tensor memory in the kernel.
bool tc_two_cta(int u, int dp);
int tc_dp(int d);  // input dimension padded for the tensor-core tiles
// Pack the FP32 parameters into the weight image.
void launch_pack_w(int u, int d, int dp, int off0, int off1, int off2, int P, const float* params, uint8_t* wimg,
                   cudaStream_t s);
// Pack X [R][d] into 128-row tiles and the transposed copy Xt [dp][ld_x] (pad rows zero).
void launch_pack_x(const float* X, long R, int d, int dp, uint8_t* ximg, float* Xt, long ld_x, int xf32,
                   cudaStream_t s);
// Returns the number of per-CTA partials written (gpart / lpart / mpart rows).
int launch_tile_tc(int u, const TileArgs& a, int sm_count, cudaStream_t s);
int launch_wgrad_tc(int u, WgradArgs a, int sm_count, cudaStream_t s);
int tc_wgrad_max_ctas(int sm_count);
int tc_eval_max_ctas(int sm_count);  // partial rows an evaluation launch may write  // rows of WgradArgs::gpart the launcher may write
// FP64 Gram partials of z = [H2 row, 1] and rhs z (y - mu) in k_refit's packed
// layout (upper triangle, then rhs); returns the partial count (<= max_parts).
int launch_gram_h2(int u, const float* H2, const double* y, long R, const float* params, int P, double* gpart,
                   int max_parts, int sm_count, cudaStream_t s);

}  // namespace hcva
