// regress_tc.cu -- K5 on the 5th-generation tensor cores: the SGD step and the
// full-sample evaluation of the backward regression (regressor.cpp:97-158) as
// tcgen05 kind::tf32 GEMMs (3xTF32, FP32 accumulation in TMEM) for the paper's
// network shape: two hidden layers of width U in {16, 32, 64}, input d <= 64.
// All operands are K-major (canonical no-swizzle core tiles, tc.cuh).
//
// k_tile_tc<U>   one 128-row tile per CTA, 128 threads (thread r = row r =
//                TMEM lane r); thread 0 issues the MMAs, tcgen05.commit
//                signals an mbarrier, epilogues read TMEM with tcgen05.ld.
//     F0   D0  = X  W0^T   (M=128, N=U, K=dp)  -> H1 = act(D0 + b0)
//     F1   D1  = H1 W1^T   (M=128, N=U, K=U)   -> H2, f, loss, G2
//     B    Dbp = G2 W1     (M=128, N=U, K=U; B operand = W1^T tile)
//                                              -> G1 = Dbp act'(H1)
//   SGD mode also writes H1, G2, G1 transposed ([feature][row]) for the
//   weight-gradient kernel, and per-tile partials of the biases, the output
//   layer and mu; eval mode produces the loss / min fit / predictions.
// k_wgrad_tc<U>  split-K weight gradients over the batch rows: each CTA
//                accumulates  gW1 = G2^T H1 (M=64, N=U)  and
//                gW0 = G1^T X (M=64, N=dp) over its rows in TMEM, 64-row
//                chunks, and writes one partial.
// Reductions of the partials are fixed-order FP64 (k_adam in regress.cu).
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "regress_tc.cuh"
#include "tc.cuh"

namespace hcva {

__device__ __forceinline__ float tc_act(int a, float z) {
    switch (a) {
        case 0: return tanhf(z);
        case 1: return 1.0f / (1.0f + expf(-z));
        case 2: return fmaxf(z, 0.0f) + log1pf(expf(-fabsf(z)));
        default: return fmaxf(z, 0.0f);
    }
}
__device__ __forceinline__ float tc_der(int a, float v) {
    switch (a) {
        case 0: return 1.0f - v * v;
        case 1: return v * (1.0f - v);
        case 2: return -expm1f(-v);
        default: return v > 0.0f ? 1.0f : 0.0f;
    }
}

constexpr uint32_t kRowTile = 128 * 64 * 4;  // 128 x 64 FP32 core tile
constexpr int kTcThreads = 128;

__host__ __device__ constexpr size_t tile_tc_smem(int U) {
    return 4 * static_cast<size_t>(kRowTile) + 6 * static_cast<size_t>(U) * 64 * 4 + 512 * 4 + 64 * 8 + 64;
}

__device__ __forceinline__ float warp_sum(float v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int U>
__global__ void __launch_bounds__(kTcThreads, 1) k_tile_tc(TileArgs a) {
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr uint32_t wbytes = U * 64 * 4;
    uint8_t* bufX = sm;                // X, then G2 (128 x 64 core tile, lo at +kRowTile)
    uint8_t* bufH = sm + 2 * kRowTile; // H1
    uint8_t* w0 = sm + 4 * kRowTile;   // U x 64
    uint8_t* w1 = w0 + 2 * wbytes;     // U x U (row = out, col = in)
    uint8_t* w1t = w1 + 2 * wbytes;    // U x U transposed (row = in, col = out)
    float* vec = reinterpret_cast<float*>(w1t + 2 * wbytes);  // b0 b1 w2 misc [64 each], colsum [4][64]
    float* colsum = vec + 256;
    double* red = reinterpret_cast<double*>(vec + 512);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(red + 64);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);

    const int r = threadIdx.x, warp = r >> 5, lane = r & 31;
    const int d = a.d, dp = a.dp;
    const bool sgd = a.mode == 0;
    const long base = a.row0 + static_cast<long>(blockIdx.x) * 128;
    const int rows = static_cast<int>(min(128L, a.row_end - base));
    const bool live = r < rows;
    const float* P = a.params;

    if (r == 0) tc::mbar_init(mbar, 1);
    if (warp == 0) tc::tmem_alloc(tbase, 256);
    for (int i = r; i < U * dp; i += kTcThreads) {
        const int o = i / dp, j = i % dp;
        tc::put_split(w0, wbytes, o, j, U, (j < d) ? P[a.off0 + o * d + j] : 0.0f);
    }
    for (int i = r; i < U * U; i += kTcThreads) {
        const int o = i / U, j = i % U;
        const float wv = P[a.off1 + o * U + j];
        tc::put_split(w1, wbytes, o, j, U, wv);
        if (sgd) tc::put_split(w1t, wbytes, j, o, U, wv);
    }
    if (r < 64) {
        vec[r] = (r < U) ? P[a.off0 + U * d + r] : 0.0f;       // b0
        vec[64 + r] = (r < U) ? P[a.off1 + U * U + r] : 0.0f;  // b1
        vec[128 + r] = (r < U) ? P[a.off2 + r] : 0.0f;         // w2
    }
    if (r == 0) {
        vec[192] = P[a.off2 + U];  // b2
        vec[193] = P[a.P - 1];     // mu
    }
    for (int i = r; i < 128 * dp; i += kTcThreads) {
        const int rr = i / dp, j = i % dp;
        const float v = (rr < rows && j < d) ? a.X[(base + rr) * d + j] : 0.0f;
        tc::put_split(bufX, kRowTile, rr, j, 128, v);
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    uint32_t phase = 0;
    auto mma_sync = [&]() {
        tc::mbar_wait(mbar, phase);
        phase ^= 1;
        tc::fence_after_sync();
    };
    auto smem_sync = [&]() {
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
    };
    const long trow = base - a.row0 + r;  // row index in the transposed arrays

    // ---- F0: D0 = X W0^T ; H1 = act(D0 + b0)
    if (r == 0) {
        tc::gemm3(tm, tc::kmajor(bufX, kRowTile, 128), tc::kmajor(w0, wbytes, U), dp, tc::idesc_tf32(128, U, 0, 0), 0);
        tc::commit(mbar);
    }
    mma_sync();
#pragma unroll
    for (int c0 = 0; c0 < U; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + c0, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float h = tc_act(a.act, v[q] + vec[c0 + q]);
            tc::put_split(bufH, kRowTile, r, c0 + q, 128, h);
            if (sgd && live) a.H1t[(c0 + q) * a.ld_t + trow] = h;
        }
    }
    smem_sync();
    // ---- F1: D1 = H1 W1^T ; H2, f
    if (r == 0) {
        tc::gemm3(tm + 64, tc::kmajor(bufH, kRowTile, 128), tc::kmajor(w1, wbytes, U), U, tc::idesc_tf32(128, U, 0, 0),
                  0);
        tc::commit(mbar);
    }
    mma_sync();
    float h2[U];
#pragma unroll
    for (int c0 = 0; c0 < U; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + 64 + c0, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) h2[c0 + q] = tc_act(a.act, v[q] + vec[64 + c0 + q]);
    }
    float f = vec[192];
#pragma unroll
    for (int j = 0; j < U; ++j) f = fmaf(h2[j], vec[128 + j], f);
    const float mu = vec[193];

    if (!sgd) {  // ---------------- evaluation
        double l = 0.0, mn = INFINITY;
        if (live) {
            const double ph = static_cast<double>((f < 0.0f ? 0.0f : f) + mu);
            if (a.mode & 1) {
                const double res = ph - a.y[base + r];
                l = res * res;
            }
            if (a.mode & 2) mn = static_cast<double>(f + mu);
            if (a.mode & 4) a.pred[base + r] = ph;
        }
        l = warp_sum(l);
        for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        if (lane == 0) {
            red[warp] = l;
            red[4 + warp] = mn;
        }
        tc::fence_before_sync();
        __syncthreads();
        if (r == 0) {
            if (a.mode & 1) a.lpart[blockIdx.x] = red[0] + red[1] + red[2] + red[3];
            if (a.mode & 2) a.mpart[blockIdx.x] = fmin(fmin(red[4], red[5]), fmin(red[6], red[7]));
        }
        if (warp == 0) tc::tmem_dealloc(tm, 256);
        return;
    }

    // ---------------- SGD: residual, output layer, mu
    double resid2 = 0.0, dmu = 0.0;
    float dd = 0.0f;
    if (live) {
        const float pred = ((a.head && f < 0.0f) ? 0.0f : f) + mu;
        const double res = static_cast<double>(pred) - a.y[base + r];
        resid2 = res * res;
        dmu = 2.0 * res / a.nb;
        dd = static_cast<float>(dmu);
        if (a.head && !(f > 0.0f)) dd = 0.0f;
    }
    float* gout = a.gpart + static_cast<size_t>(blockIdx.x) * a.P;
    {
        const double l = warp_sum(resid2), m = warp_sum(dmu);
        const float gb = warp_sum(dd);
        if (lane == 0) {
            red[warp] = l;
            red[4 + warp] = m;
            red[8 + warp] = gb;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const float s = warp_sum(dd * h2[j]);
            if (lane == 0) colsum[warp * 64 + j] = s;
        }
    }
    __syncthreads();
    if (r == 0) {
        a.lpart[blockIdx.x] = red[0] + red[1] + red[2] + red[3];
        gout[a.P - 1] = static_cast<float>(red[4] + red[5] + red[6] + red[7]);
        gout[a.off2 + U] = static_cast<float>(red[8] + red[9] + red[10] + red[11]);
    }
    if (r < U) gout[a.off2 + r] = colsum[r] + colsum[64 + r] + colsum[128 + r] + colsum[192 + r];
    __syncthreads();
    // G2 = dd w2 act'(H2) -> bufX (K-major), G2t; bias gradient of layer 1.
#pragma unroll
    for (int j = 0; j < U; ++j) {
        const float g = dd * vec[128 + j] * tc_der(a.act, h2[j]);
        tc::put_split(bufX, kRowTile, r, j, 128, g);
        if (live) a.G2t[j * a.ld_t + trow] = g;
        const float s = warp_sum(g);
        if (lane == 0) colsum[warp * 64 + j] = s;
    }
    smem_sync();
    if (r < U) gout[a.off1 + U * U + r] = colsum[r] + colsum[64 + r] + colsum[128 + r] + colsum[192 + r];
    // ---- B: Dbp = G2 W1 (B operand: the W1^T tile, K-major over the outputs of layer 1)
    if (r == 0) {
        tc::gemm3(tm + 128, tc::kmajor(bufX, kRowTile, 128), tc::kmajor(w1t, wbytes, U), U,
                  tc::idesc_tf32(128, U, 0, 0), 0);
        tc::commit(mbar);
    }
    mma_sync();
    __syncthreads();  // colsum reads of layer 1 done
#pragma unroll
    for (int c0 = 0; c0 < U; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + 128 + c0, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float h1 = tc::get_split(bufH, kRowTile, r, c0 + q, 128);
            const float g = live ? v[q] * tc_der(a.act, h1) : 0.0f;
            if (live) a.G1t[(c0 + q) * a.ld_t + trow] = g;
            const float s = warp_sum(g);
            if (lane == 0) colsum[warp * 64 + c0 + q] = s;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (r < U) gout[a.off0 + U * d + r] = colsum[r] + colsum[64 + r] + colsum[128 + r] + colsum[192 + r];
    if (warp == 0) tc::tmem_dealloc(tm, 256);
}

constexpr uint32_t kChunkTile = 64 * 64 * 4;  // 64 x 64 FP32 core tile

template <int U>
__global__ void __launch_bounds__(kTcThreads, 1) k_wgrad_tc(WgradArgs a) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* tA1 = sm;                   // G2t chunk: 64 (o, zero-padded) x 64 (rows)
    uint8_t* tB1 = sm + 2 * kChunkTile;  // H1t chunk: U x 64
    uint8_t* tA0 = sm + 4 * kChunkTile;  // G1t chunk
    uint8_t* tB0 = sm + 6 * kChunkTile;  // Xt chunk: dp x 64
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + 8 * kChunkTile);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int dp = a.dp;
    if (t == 0) tc::mbar_init(mbar, 1);
    if (warp == 0) tc::tmem_alloc(tbase, 128);
    for (int i = t; i < 8 * kChunkTile / 4; i += kTcThreads) reinterpret_cast<float*>(sm)[i] = 0.0f;
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    const long r_begin = static_cast<long>(blockIdx.x) * a.rows_per_cta;
    const long r_end = min(r_begin + a.rows_per_cta, a.rows);
    uint32_t phase = 0;
    int first = 1;
    for (long c0 = r_begin; c0 < r_end; c0 += 64) {
        const int n = static_cast<int>(min(64L, r_end - c0));
        // Coalesced loads: 64 consecutive rows of each feature line.
        for (int i = t; i < U * 64; i += kTcThreads) {
            const int f = i / 64, k = i % 64;
            const bool in = k < n;
            tc::put_split(tA1, kChunkTile, f, k, 64, in ? a.G2t[f * a.ld_t + c0 + k] : 0.0f);
            tc::put_split(tB1, kChunkTile, f, k, 64, in ? a.H1t[f * a.ld_t + c0 + k] : 0.0f);
            tc::put_split(tA0, kChunkTile, f, k, 64, in ? a.G1t[f * a.ld_t + c0 + k] : 0.0f);
        }
        for (int i = t; i < dp * 64; i += kTcThreads) {
            const int f = i / 64, k = i % 64;
            tc::put_split(tB0, kChunkTile, f, k, 64, (k < n) ? a.Xt[f * a.ld_x + a.row0 + c0 + k] : 0.0f);
        }
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        if (t == 0) {
            tc::gemm3(tm, tc::kmajor(tA1, kChunkTile, 64), tc::kmajor(tB1, kChunkTile, 64), 64,
                      tc::idesc_tf32(64, U, 0, 0), !first);
            tc::gemm3(tm + 64, tc::kmajor(tA0, kChunkTile, 64), tc::kmajor(tB0, kChunkTile, 64), 64,
                      tc::idesc_tf32(64, dp, 0, 0), !first);
            tc::commit(mbar);
        }
        tc::mbar_wait(mbar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        first = 0;
        __syncthreads();  // chunk consumed before the next overwrites it
    }
    float* gout = a.gpart + static_cast<size_t>(blockIdx.x) * a.P;
    const int o = warp * 16 + lane;  // M=64 accumulator: row 16w+t in lane 32w+t, t < 16
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
#pragma unroll
    for (int c = 0; c < U; c += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + c, v);
        if (lane < 16 && o < U)
#pragma unroll
            for (int q = 0; q < 16; ++q) gout[a.off1 + o * U + c + q] = first ? 0.0f : v[q];
    }
    for (int c = 0; c < dp; c += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + 64 + c, v);
        if (lane < 16 && o < U)
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (c + q < a.d) gout[a.off0 + o * a.d + c + q] = first ? 0.0f : v[q];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, 128);
}

// Diagnostic GEMM: D (M x N) = A (M x K) B (N x K)^T, K-major no-swizzle
// (variant 0) or 128B-swizzled (variant 2) operand tiles; test hook for the
// descriptor conventions.
__global__ void k_tc_gemm_diag(int M, int N, int K, const float* A, const float* B, float* D, int swz) {
    extern __shared__ __align__(128) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t abytes = M * ((K + 31) / 32) * 32 * 4, bbytes = N * ((K + 31) / 32) * 32 * 4;
    uint8_t* ta = sm;
    uint8_t* tb = sm + 2 * abytes;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(tb + 2 * bbytes);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);
    const int t = threadIdx.x, warp = t >> 5;
    if (t == 0) tc::mbar_init(mbar, 1);
    if (warp == 0) tc::tmem_alloc(tbase, 256);
    for (int i = t; i < 2 * (abytes + bbytes) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.0f;
    __syncthreads();
    for (int i = t; i < M * K; i += blockDim.x) {
        if (swz) tc::put_split_sw(ta, abytes, i / K, i % K, M, A[i]);
        else tc::put_split(ta, abytes, i / K, i % K, M, A[i]);
    }
    for (int i = t; i < N * K; i += blockDim.x) {
        if (swz) tc::put_split_sw(tb, bbytes, i / K, i % K, N, B[i]);
        else tc::put_split(tb, bbytes, i / K, i % K, N, B[i]);
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    if (t == 0) {
        if (swz) {
            tc::gemm3_sw(tm, tc::OperandSW{tc::smem_u32(ta), abytes, static_cast<uint32_t>(M), 0},
                         tc::OperandSW{tc::smem_u32(tb), bbytes, static_cast<uint32_t>(N), 0}, K,
                         tc::idesc_tf32(M, N, 0, 0), 0);
        } else {
            tc::gemm3(tm, tc::kmajor(ta, abytes, M), tc::kmajor(tb, bbytes, N), K, tc::idesc_tf32(M, N, 0, 0), 0);
        }
        tc::commit(mbar);
    }
    tc::mbar_wait(mbar, 0);
    tc::fence_after_sync();
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
        const int lane = t & 31;
        const int row = (M == 128) ? t : ((lane < 16) ? warp * 16 + lane : -1);
        if (row >= 0)
            for (int q = 0; q < 16 && c0 + q < N; ++q) D[row * N + c0 + q] = v[q];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, 256);
}

// ------------------------------------------------------------------ host

bool tc_eligible(int d, int h, int u) {
    if (const char* e = std::getenv("HCVA_REGRESS_SIMT"))
        if (std::atoi(e)) return false;
    return h == 2 && (u == 16 || u == 32 || u == 64) && d >= 1 && d <= 64;
}

int tc_dp(int d) { return ((d + 15) / 16) * 16; }

template <int U>
void launch_tile_u(const TileArgs& a, int tiles, cudaStream_t s) {
    const size_t smem = tile_tc_smem(U);
    HCVA_CUDA(cudaFuncSetAttribute(k_tile_tc<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_tile_tc<U><<<tiles, kTcThreads, smem, s>>>(a);
}

void launch_tile_tc(int u, const TileArgs& a, cudaStream_t s) {
    const int tiles = static_cast<int>((a.row_end - a.row0 + 127) / 128);
    if (u == 16) launch_tile_u<16>(a, tiles, s);
    else if (u == 32) launch_tile_u<32>(a, tiles, s);
    else launch_tile_u<64>(a, tiles, s);
}

template <int U>
void launch_wgrad_u(const WgradArgs& a, int ctas, cudaStream_t s) {
    const size_t smem = 8 * static_cast<size_t>(kChunkTile) + 64;
    HCVA_CUDA(cudaFuncSetAttribute(k_wgrad_tc<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_wgrad_tc<U><<<ctas, kTcThreads, smem, s>>>(a);
}

// Returns the number of weight-gradient partials written.
int launch_wgrad_tc(int u, WgradArgs a, int sm_count, cudaStream_t s) {
    const long chunks = (a.rows + 63) / 64;
    const long per = std::max(1L, (chunks + sm_count - 1) / sm_count);
    a.rows_per_cta = static_cast<int>(per * 64);
    const int ctas = static_cast<int>((a.rows + a.rows_per_cta - 1) / a.rows_per_cta);
    if (u == 16) launch_wgrad_u<16>(a, ctas, s);
    else if (u == 32) launch_wgrad_u<32>(a, ctas, s);
    else launch_wgrad_u<64>(a, ctas, s);
    return ctas;
}

}  // namespace hcva

using namespace hcva;

extern "C" hcva_status hcva_diag_tc_gemm(hcva_ctx* ctx, int M, int N, int K, int swizzle, const float* A,
                                         const float* B, float* D) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if ((M != 64 && M != 128) || N % 16 || N > 128 || K % 8 || K > 128)
            throw contract_error("diag gemm: M in {64,128}, N % 16 == 0 <= 128, K % 8 == 0 <= 128");
        DeviceBuf dA, dB, dD;
        stage(dA, std::vector<float>(A, A + M * K));
        stage(dB, std::vector<float>(B, B + N * K));
        dD.alloc(sizeof(float) * M * N);
        const size_t kp = ((K + 31) / 32) * 32;
        const size_t smem = 2 * 4 * kp * (static_cast<size_t>(M) + N) + 2048;
        HCVA_CUDA(cudaFuncSetAttribute(k_tc_gemm_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_tc_gemm_diag<<<1, 128, smem, ctx->stream>>>(M, N, K, dA.as<float>(), dB.as<float>(), dD.as<float>(),
                                                      swizzle);
        check_launch(ctx);
        copy_out(ctx, D, dD.p, sizeof(float) * M * N);
    });
}
