// regress_tc.cuh -- launch interface of the tensor-core regression kernels (regress_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace hcva {

struct TileArgs {
    int d, dp, act, P, off0, off1, off2;
    const float* X;  // [R][d]
    const double* y;
    long row0, row_end;
    const float* params;
    int head, mode;  // mode 0: SGD; else bits 1: loss (head on), 2: min plain fit, 4: predictions
    double nb;
    float* gpart;    // SGD: [tile][P] partials of b0, b1, w2, b2, mu
    double* lpart;   // [tile] sum of squared residuals
    double* mpart;   // [tile] min of f + mu (plain head)
    double* pred;    // predictions (head on), indexed by absolute row
    float *H1t, *G2t, *G1t;  // SGD: [U][ld_t] transposed, row index relative to row0
    long ld_t;
};

struct WgradArgs {
    int d, dp, P, off0, off1;
    const float *G2t, *H1t, *G1t;  // [U][ld_t]
    long ld_t;
    const float* Xt;               // [dp][ld_x] transposed features, column = absolute row
    long ld_x, row0, rows;         // rows of the batch (relative index 0..rows-1)
    int rows_per_cta;              // multiple of 64 (set by the launcher)
    float* gpart;                  // [cta][P]: W0, W1 entries
};

bool tc_eligible(int d, int h, int u);
int tc_dp(int d);  // input dimension padded for the tensor-core tiles
void launch_tile_tc(int u, const TileArgs& a, cudaStream_t s);
int launch_wgrad_tc(int u, WgradArgs a, int sm_count, cudaStream_t s);

}  // namespace hcva
