// regress_tc.cu -- K5 on the 5th-generation tensor cores: the SGD step and the
// full-sample evaluation of the backward regression (regressor.cpp:97-158) as
// tcgen05 kind::tf32 GEMMs (3xTF32, FP32 accumulation in TMEM) for the paper's
// network shape: two hidden layers of width U in {16, 32, 64}, input d <= 255.
// Shared-memory operands are K-major (canonical no-swizzle core tiles, tc.cuh).
//
// k_pack_w      parameters -> weight image (W0, W1, W1^T hi/lo planes + biases),
//               one bulk copy per CTA.
// k_pack_x      features X [R][d] -> 128-row operand tiles + Xt [dp][R]: one
//               FP32 plane for the two-CTA kernels, hi/lo planes otherwise.
// The per-tile GEMM chain (thread r = row r = TMEM lane r; one thread issues
// the MMAs, tcgen05.commit signals an mbarrier, epilogues read TMEM):
//     F0   D0  = X  W0^T   (M=128, N=U, K=dp)  -> H1 = act(D0 + b0); act'(H1) -> D0
//     F1   D1  = H1 W1^T   (M=128, N=U, K=U)   -> H2, f, loss, G2
//     B    Dbp = G2 W1     (M=128, N=U, K=U; B operand = W1^T tile)
//                                              -> G1 = Dbp act'(H1)
//   SGD also writes H1, G2, G1 transposed ([feature][row]) for the weight-
//   gradient kernel; bias / output-layer / mu gradients are column sums
//   (butterfly reduce-scatter across the warp, accumulated per CTA).
// k_sgd_tc<U, ACT>   SGD, two CTAs per SM (tc_two_cta shapes): the A operands
//               X, H1, G2 live in tensor memory (A-in-TMEM MMAs), shared memory
//               holds W0, W1, W1^T and the FP32 feature tile.
// k_eval_tc<U, ACT>  evaluation (loss / min fit / predictions / H2), two CTAs
//               per SM, X and H1 in tensor memory.
// k_tile_tc<U, ACT, CH>  the general one-CTA-per-SM kernel (both modes) with
//               A operands in shared memory; CH streams layer 0's K dimension
//               in 16-column chunks for wide inputs (C5).
// k_wgrad_tc<U, XR>  split-K weight gradients over the batch rows: each CTA
//               accumulates gW1 = G2^T H1 (M=64, N=U) and gW0 = G1^T X
//               (M=64, N=dp) over its rows in TMEM, 32-row chunks with two
//               chunks of loads in flight, one partial per CTA.
// Reductions of the per-CTA partials are fixed-order FP64 (k_adam in regress.cu).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "regress_act.cuh"
#include "regress_tc.cuh"
#include "tc.cuh"

namespace hcva {

__host__ __device__ constexpr uint32_t w_image_bytes(int U, int dp) {
    return 2u * U * dp * 4 + 4u * U * U * 4 + 1024;
}
__host__ __device__ constexpr uint32_t x_plane_bytes(int dp) { return 128u * dp * 4; }
// Wide inputs (the resident layout below exceeds shared memory, e.g. C5's 157
// features): W1, W1^T and the vectors stay resident, layer 0's K dimension is
// streamed in kKc-column chunks of (X tile, W0) through kNst stages.
constexpr int kKc = 16, kNst = 3;
// mbarriers (MMA, weights, features, kNst full + kNst empty) and the TMEM base
// word, after the partial-sum scratch.
constexpr size_t kTileBarBytes = 8 * (3 + 2 * kNst) + 16;
__host__ __device__ constexpr size_t tile_tc_smem(int U, int dp) {
    return w_image_bytes(U, dp) + 2ull * 128 * U * 4 + 2ull * x_plane_bytes(dp) + 8 * 128 * 4 + kTileBarBytes;
}
constexpr int kWgXMax = 256;  // widest padded input of the tensor-core path
__host__ __device__ constexpr uint32_t stage_bytes(int U) { return 2u * 128 * kKc * 4 + 2u * U * kKc * 4; }
__host__ __device__ constexpr size_t tile_tc_smem_ch(int U) {
    return 4ull * U * U * 4 + 1024 + 2ull * 128 * U * 4 + static_cast<size_t>(kNst) * stage_bytes(U) + 8 * 128 * 4 +
           kTileBarBytes;
}
__host__ __device__ constexpr bool tile_chunked(int U, int dp) { return tile_tc_smem(U, dp) > 227 * 1024; }

size_t tc_weight_image_bytes(int u, int dp) { return w_image_bytes(u, dp); }
size_t tc_x_tile_bytes(int dp) { return 2ull * x_plane_bytes(dp); }

__global__ void k_pack_w(int U, int d, int dp, int off0, int off1, int off2, int P, const float* __restrict__ p,
                         uint8_t* __restrict__ img) {
    const uint32_t w0b = U * dp * 4, w1b = U * U * 4;
    uint8_t* w0 = img;
    uint8_t* w1 = w0 + 2 * w0b;
    uint8_t* w1t = w1 + 2 * w1b;
    float* vec = reinterpret_cast<float*>(w1t + 2 * w1b);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < U * dp) {
        const int o = i / dp, j = i % dp;
        tc::put_split(w0, w0b, o, j, U, (j < d) ? p[off0 + o * d + j] : 0.0f);
    }
    if (i < U * U) {
        const int o = i / U, j = i % U;
        const float wv = p[off1 + o * U + j];
        tc::put_split(w1, w1b, o, j, U, wv);
        tc::put_split(w1t, w1b, j, o, U, wv);
    }
    if (i < 256) {
        const int q = i >> 6, k = i & 63;
        float v = 0.0f;
        if (q == 0 && k < U) v = p[off0 + U * d + k];
        else if (q == 1 && k < U) v = p[off1 + U * U + k];
        else if (q == 2 && k < U) v = p[off2 + k];
        else if (q == 3 && k == 0) v = p[off2 + U];
        else if (q == 3 && k == 1) v = p[P - 1];
        vec[i] = v;
    }
}

__global__ void k_pack_x(const float* __restrict__ X, long R, int d, int dp, uint8_t* __restrict__ img,
                         float* __restrict__ Xt, long ld_x, int xf32) {
    const uint32_t xb = x_plane_bytes(dp);
    uint8_t* tile = img + static_cast<size_t>(blockIdx.x) * (xf32 ? 1 : 2) * xb;
    const int r = threadIdx.x;
    const long row = static_cast<long>(blockIdx.x) * 128 + r;
    const bool in = row < R;
    for (int c = 0; c < dp; c += 4) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = (in && c + q < d) ? X[row * d + c + q] : 0.0f;
        if (xf32) *reinterpret_cast<float4*>(tile + tc::core_off(r, c, 128)) = make_float4(v[0], v[1], v[2], v[3]);
        else tc::put_split4(tile, xb, r, c, 128, make_float4(v[0], v[1], v[2], v[3]));
        if (in)
#pragma unroll
            for (int q = 0; q < 4; ++q) Xt[(c + q) * ld_x + row] = v[q];
    }
}

// Column split: U/UH warpgroups share each 128-row tile, warpgroup h owning
// columns [UH h, UH (h+1)) of every layer (TMEM lane quarter = warp % 4).
#ifndef HCVA_TILE_UH
#define HCVA_TILE_UH 16
#endif
template <int U>
struct TileShape {
    static constexpr int UH = HCVA_TILE_UH < U ? HCVA_TILE_UH : U;  // columns per thread
    static constexpr int NS = U / UH;                               // warpgroups
    static constexpr int threads = 128 * NS;
    static constexpr int warps = 4 * NS;
};

template <int U, int ACT, bool CH>
__global__ void __launch_bounds__(TileShape<U>::threads, 1) k_tile_tc(TileArgs a, long t_first, long n_tiles) {
    constexpr int NS = TileShape<U>::NS, UH = TileShape<U>::UH;
    extern __shared__ __align__(128) uint8_t sm[];
    const int dp = a.dp;
    const uint32_t w0b = U * dp * 4, w1b = U * U * 4, hb = 128 * U * 4, xb = x_plane_bytes(dp);
    const uint32_t wbytes = w_image_bytes(U, dp);
    // Resident layout: [W0 | W1 | W1^T | vec][H][X tile]; chunked (CH):
    // [W1 | W1^T | vec][H][kNst stages of (X chunk hi | lo, W0 chunk hi | lo)].
    uint8_t* w0 = sm;
    uint8_t* w1 = CH ? sm : w0 + 2 * w0b;
    uint8_t* w1t = w1 + 2 * w1b;
    const float* vec = reinterpret_cast<const float*>(w1t + 2 * w1b);  // b0 | b1 | w2 | b2, mu
    uint8_t* bufH = CH ? sm + 4 * w1b + 1024 : sm + wbytes;  // H1, then G2 (hi | lo)
    uint8_t* bufX = bufH + 2 * hb;  // feature tile (hi | lo) / the chunk stages
    float* fsh = reinterpret_cast<float*>(bufX + (CH ? kNst * stage_bytes(U) : 2 * xb));  // [NS][128] partial sums
    uint64_t* bar = reinterpret_cast<uint64_t*>(fsh + 8 * 128);  // [0] MMA, [1] weights, [2] features
    uint64_t* full = bar + 3;                                    // CH: stage loaded / consumed
    uint64_t* empty = full + kNst;
    uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 3 + 2 * kNst);
    constexpr uint32_t xcb = 128u * kKc * 4, wcb = static_cast<uint32_t>(U) * kKc * 4;  // chunk plane bytes
    const int nq = dp / kKc;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r = tid & 127, hf = tid >> 7, cb = hf * UH;
    const bool sgd = a.mode == 0;
    if (tid == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        tc::mbar_init(&bar[2], 1);
        if (CH)
            for (int q = 0; q < kNst; ++q) {
                tc::mbar_init(&full[q], 1);
                tc::mbar_init(&empty[q], 1);
            }
        tc::fence_async_smem();
    }
    if (warp == 0) tc::tmem_alloc(tbase, 256);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const long t_end = t_first + n_tiles;
    long tile = t_first + blockIdx.x;
    pdl_wait();  // the optimizer's weight image / the previous weight gradient's reads of H1t, G2t, G1t
    // CH: chunk g of this CTA = chunk g % nq of its (g / nq)-th tile, stage g % kNst.
    const long my_tiles = tile < t_end ? (t_end - tile + gridDim.x - 1) / gridDim.x : 0;
    const long n_chunks = my_tiles * nq;
    auto load_chunk = [&](long g) {  // one thread
        const int st = static_cast<int>(g % kNst), q = static_cast<int>(g % nq);
        const long tl = t_first + blockIdx.x + (g / nq) * gridDim.x;
        uint8_t* sb = bufX + st * stage_bytes(U);
        const uint8_t* xs = a.ximg + tl * 2 * xb + q * xcb;
        const uint8_t* ws = a.wimg + q * wcb;
        tc::mbar_expect_tx(&full[st], 2 * xcb + 2 * wcb);
        tc::bulk_g2s(sb, xs, xcb, &full[st]);
        tc::bulk_g2s(sb + xcb, xs + xb, xcb, &full[st]);
        tc::bulk_g2s(sb + 2 * xcb, ws, wcb, &full[st]);
        tc::bulk_g2s(sb + 2 * xcb + wcb, ws + w0b, wcb, &full[st]);
    };
    if (tid == 0) {
        if (CH) {
            tc::mbar_expect_tx(&bar[1], 4 * w1b + 1024);
            tc::bulk_g2s(w1, a.wimg + 2 * w0b, 4 * w1b + 1024, &bar[1]);
            for (long g = 0; g < kNst && g < n_chunks; ++g) load_chunk(g);
        } else {
            tc::mbar_expect_tx(&bar[1], wbytes);
            tc::bulk_g2s(w0, a.wimg, wbytes, &bar[1]);
            tc::mbar_expect_tx(&bar[2], 2 * xb);
            tc::bulk_g2s(bufX, a.ximg + tile * 2 * xb, 2 * xb, &bar[2]);
        }
    }
    tc::mbar_wait(&bar[1], 0);
    long g_next = 0;  // CH: next chunk to consume
    uint32_t mph = 0, xph = 0;
    auto mma_wait = [&]() {  // one waiting warp, the rest parked at the barrier
        if (warp == 0) tc::mbar_wait(&bar[0], mph);
        mph ^= 1;
        __syncthreads();
        tc::fence_after_sync();
    };
    auto cta_sync = [&]() {
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
    };
    const float b2 = vec[192], mu = vec[193];
    constexpr int NB = (UH + 31) / 32;
    double loss = 0.0, dmu = 0.0, mn = INFINITY;
    float gb2 = 0.0f;
    float acc_w2[NB];  // output-layer gradient; the hidden biases come from the weight-gradient GEMMs
#pragma unroll
    for (int b = 0; b < NB; ++b) acc_w2[b] = 0.0f;

    for (; tile < t_end; tile += gridDim.x) {
        const long row = tile * 128 + r;
        const bool live = row >= a.b0 && row < a.b1;
        const long trow = row - a.b0;
        // the label of this row, loaded under the layer-0 GEMM (SGD and loss evaluation)
        const double yrow = (live && (sgd || ((a.mode & 1) && hf == 0))) ? __ldg(a.y + row) : 0.0;
        // ---- F0: D0 = X W0^T
        if constexpr (CH) {
            if (warp == 0) {
                for (int q = 0; q < nq; ++q, ++g_next) {
                    const int st = static_cast<int>(g_next % kNst);
                    tc::mbar_wait(&full[st], static_cast<uint32_t>((g_next / kNst) & 1));
                    uint8_t* sb = bufX + st * stage_bytes(U);
                    tc::gemm3_warp(tm, tc::kmajor(sb, xcb, 128), tc::kmajor(sb + 2 * xcb, wcb, U), kKc,
                                   tc::idesc_tf32(128, U, 0, 0), q > 0, &empty[st]);
                    if (g_next >= 1) {  // the previous chunk's MMAs done: refill its stage kNst chunks ahead
                        const long gp = g_next - 1;
                        tc::mbar_wait(&empty[gp % kNst], static_cast<uint32_t>((gp / kNst) & 1));
                        if (lane == 0 && gp + kNst < n_chunks) load_chunk(gp + kNst);
                        __syncwarp();
                    }
                }
                tc::commit_if(tc::elect_one(), &bar[0]);  // every F0 MMA of the tile
            }
        } else {
            if (tid == 0) tc::mbar_wait(&bar[2], xph);  // only the issuing thread reads the feature tile
            xph ^= 1;
            if (warp == 0)
                tc::gemm3_warp(tm, tc::kmajor(bufX, xb, 128), tc::kmajor(w0, w0b, U), dp,
                               tc::idesc_tf32(128, U, 0, 0), 0, &bar[0]);
        }
        mma_wait();
        if (!CH && tid == 0 && tile + gridDim.x < t_end) {  // feature tile consumed: stream in the next one
            tc::mbar_expect_tx(&bar[2], 2 * xb);
            tc::bulk_g2s(bufX, a.ximg + (tile + gridDim.x) * 2 * xb, 2 * xb, &bar[2]);
        }
        // H1 = act(D0 + b0) -> bufH (+ H1t); act'(H1) back into D0
        {
            const int c0 = cb;
            float v[UH];
            tc::tmem_ldw<UH>(tm + lb + c0, v);
#pragma unroll
            for (int q = 0; q < UH; ++q) v[q] = act_f<ACT>(v[q] + vec[c0 + q]);
#pragma unroll
            for (int q = 0; q < UH; q += 4)
                tc::put_split4(bufH, hb, r, c0 + q, 128, make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]));
            if (sgd) {
                if (live)
#pragma unroll
                    for (int q = 0; q < UH; ++q) a.H1t[(c0 + q) * a.ld_t + trow] = v[q];
#pragma unroll
                for (int q = 0; q < UH; ++q) v[q] = act_d<ACT>(v[q]);
                tc::tmem_stw<UH>(tm + lb + c0, v);
            }
        }
        if (sgd) tc::tmem_wait_st();
        cta_sync();
        // ---- F1: D1 = H1 W1^T ; H2, f
        if (warp == 0)
            tc::gemm3_warp(tm + 64, tc::kmajor(bufH, hb, 128), tc::kmajor(w1, w1b, U), U,
                           tc::idesc_tf32(128, U, 0, 0), 0, &bar[0]);
        mma_wait();
        float h2[UH];
        tc::tmem_ldw<UH>(tm + lb + 64 + cb, h2);
#pragma unroll
        for (int q = 0; q < UH; ++q) h2[q] = act_f<ACT>(h2[q] + vec[64 + cb + q]);
        float f;
        {
            float fp = 0.0f;
#pragma unroll
            for (int j = 0; j < UH; ++j) fp = fmaf(h2[j], vec[128 + cb + j], fp);
            if (NS > 1) {
                fsh[hf * 128 + r] = fp;
                __syncthreads();
                float fs = fsh[r];
#pragma unroll
                for (int h = 1; h < NS; ++h) fs += fsh[h * 128 + r];
                f = b2 + fs;
            } else {
                f = b2 + fp;
            }
        }

        if (!sgd) {  // ---------------- evaluation
            if ((a.mode & 8) && live)
#pragma unroll
                for (int j = 0; j < UH; j += 4)
                    *reinterpret_cast<float4*>(a.H2 + row * U + cb + j) =
                        make_float4(h2[j], h2[j + 1], h2[j + 2], h2[j + 3]);
            if (live && hf == 0) {
                const double ph = static_cast<double>((f < 0.0f ? 0.0f : f) + mu);
                if (a.mode & 1) {
                    const double res = ph - yrow;
                    loss += res * res;
                }
                if (a.mode & 2) mn = fmin(mn, static_cast<double>(f + mu));
                if (a.mode & 4) a.pred[row] = ph;
            }
            continue;
        }

        // ---------------- SGD: residual, output layer, mu
        float dd = 0.0f;
        if (live) {
            const float pr = ((a.head && f < 0.0f) ? 0.0f : f) + mu;
            const double res = static_cast<double>(pr) - yrow;
            const double dm = 2.0 * res / a.nb;
            if (hf == 0) {
                loss += res * res;
                dmu += dm;
            }
            dd = static_cast<float>(dm);
            if (a.head && !(f > 0.0f)) dd = 0.0f;
        }
        if (hf == 0) gb2 += dd;
        {
            float g[UH];
#pragma unroll
            for (int j = 0; j < UH; ++j) g[j] = dd * h2[j];
            colsum_acc<UH>(g, acc_w2, lane);
        }
        {  // G2 = dd w2 act'(H2) -> bufH (F1 has consumed H1), G2t
            float g[UH];
#pragma unroll
            for (int j = 0; j < UH; ++j) g[j] = dd * vec[128 + cb + j] * act_d<ACT>(h2[j]);
#pragma unroll
            for (int j = 0; j < UH; j += 4)
                tc::put_split4(bufH, hb, r, cb + j, 128, make_float4(g[j], g[j + 1], g[j + 2], g[j + 3]));
            if (live)
#pragma unroll
                for (int j = 0; j < UH; ++j) a.G2t[(cb + j) * a.ld_t + trow] = g[j];
        }
        cta_sync();
        // ---- B: Dbp = G2 W1 (B operand: the W1^T tile, K-major over the outputs of layer 1)
        if (warp == 0)
            tc::gemm3_warp(tm + 128, tc::kmajor(bufH, hb, 128), tc::kmajor(w1t, w1b, U), U,
                           tc::idesc_tf32(128, U, 0, 0), 0, &bar[0]);
        mma_wait();
        {
            float g[UH], dv[UH];
            tc::tmem_ldw<UH>(tm + lb + 128 + cb, g);
            tc::tmem_ldw<UH>(tm + lb + cb, dv);
#pragma unroll
            for (int q = 0; q < UH; ++q) g[q] = live ? g[q] * dv[q] : 0.0f;
            if (live)
#pragma unroll
                for (int j = 0; j < UH; ++j) a.G1t[(cb + j) * a.ld_t + trow] = g[j];
        }
        tc::fence_before_sync();
        __syncthreads();  // TMEM reads of D0 / Dbp done before the next tile's F0
        tc::fence_after_sync();
    }

    // ---- per-CTA partials (fixed order over the warps)
    tc::fence_before_sync();
    __syncthreads();
    constexpr int NWP = TileShape<U>::warps;
    float* part = reinterpret_cast<float*>(bufH);  // [warp][3][64]
    double* red = reinterpret_cast<double*>(part + NWP * 3 * 64);  // [4][warps]
    constexpr int NW = UH < 32 ? UH : 32;
    if (sgd && lane < NW)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int c = cb + b * 32 + lane;
            part[(warp * 3 + 0) * 64 + c] = acc_w2[b];
        }
    loss = warp_sum(loss);
    dmu = warp_sum(dmu);
    gb2 = warp_sum(gb2);
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0) {
        red[warp] = loss;
        red[NWP + warp] = dmu;
        red[2 * NWP + warp] = gb2;
        red[3 * NWP + warp] = mn;
    }
    __syncthreads();
    const int cta = blockIdx.x;
    if (sgd) {
        float* gout = a.gpart + static_cast<size_t>(cta) * a.P;
        if (tid < U) {
            const int w0q = (tid / UH) * 4;  // first warp of the owning warpgroup
            const auto sum4 = [&](int k) {
                return part[((w0q + 0) * 3 + k) * 64 + tid] + part[((w0q + 1) * 3 + k) * 64 + tid] +
                       part[((w0q + 2) * 3 + k) * 64 + tid] + part[((w0q + 3) * 3 + k) * 64 + tid];
            };
            gout[a.off2 + tid] = sum4(0);
        }
        if (tid == 0) {
            a.lpart[cta] = red[0] + red[1] + red[2] + red[3];  // warpgroup 0 holds the per-row terms
            gout[a.P - 1] = static_cast<float>(red[NWP] + red[NWP + 1] + red[NWP + 2] + red[NWP + 3]);
            gout[a.off2 + U] =
                static_cast<float>(red[2 * NWP] + red[2 * NWP + 1] + red[2 * NWP + 2] + red[2 * NWP + 3]);
        }
    } else if (tid == 0) {
        if (a.mode & 1) a.lpart[cta] = red[0] + red[1] + red[2] + red[3];
        if (a.mode & 2)
            a.mpart[cta] = fmin(fmin(red[3 * NWP], red[3 * NWP + 1]), fmin(red[3 * NWP + 2], red[3 * NWP + 3]));
    }
    if (warp == 0) tc::tmem_dealloc(tm, 256);
}

// The FP32 feature tile (core layout, one plane) -> tensor memory as the A
// operand of layer 0: hi at column 128, lo at 128 + dp.  The NS warpgroups
// split the 8-column groups between them; rows = TMEM lanes of each warp.
template <int NS>
__device__ __forceinline__ void x_to_tmem(const uint8_t* bufX, int dp, uint32_t tm, uint32_t lb, int r, int hf) {
    const int groups = dp / 8, per = (groups + NS - 1) / NS;
    for (int gi = hf * per; gi < min(groups, (hf + 1) * per); ++gi) {
        const float4 x0 = *reinterpret_cast<const float4*>(bufX + tc::core_off(r, 8 * gi, 128));
        const float4 x1 = *reinterpret_cast<const float4*>(bufX + tc::core_off(r, 8 * gi + 4, 128));
        float hi[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w}, lo[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float v = hi[q];
            hi[q] = tc::tf32_rna(v);
            lo[q] = v - hi[q];
        }
        tc::tmem_st8(tm + lb + 128 + 8 * gi, hi);
        tc::tmem_st8(tm + lb + 128 + dp + 8 * gi, lo);
    }
}

// Full-sample evaluation (loss / head-switch minimum / predictions / layer-2
// activations) for the resident-input shapes, two CTAs per SM: the layer-1
// operand H1 (hi | lo) goes from the layer-0 epilogue straight into tensor
// memory (tcgen05.st) and layer 1 reads it from there (A-in-TMEM MMA), so a
// CTA needs no H tile in shared memory (W0, W1, vectors and the feature tile:
// ~82 KB), and two CTAs per SM interleave their GEMM -> epilogue chains.
template <int U>
struct EvalShape {
    static constexpr int UH = U < 32 ? U : 32;  // columns per thread
    static constexpr int NS = U / UH;           // warpgroups
    static constexpr int threads = 128 * NS;
};

__host__ __device__ constexpr size_t eval_tc_smem(int U, int dp) {
    return 2ull * U * dp * 4 + 2ull * U * U * 4 + 1024 + 1ull * 128 * dp * 4 + 2 * 128 * 4 + 64;
}

template <int U, int ACT>
__global__ void __launch_bounds__(EvalShape<U>::threads, 2) k_eval_tc(TileArgs a, long t_first, long n_tiles) {
    constexpr int NS = EvalShape<U>::NS, UH = EvalShape<U>::UH;
    extern __shared__ __align__(128) uint8_t sm[];
    const int dp = a.dp;
    const uint32_t w0b = U * dp * 4, w1b = U * U * 4, xb = x_plane_bytes(dp);
    uint8_t* w0 = sm;                                         // W0 hi | lo
    uint8_t* w1 = w0 + 2 * w0b;                               // W1 hi | lo
    float* vec = reinterpret_cast<float*>(w1 + 2 * w1b);      // b0 | b1 | w2 | b2, mu
    uint8_t* bufX = reinterpret_cast<uint8_t*>(vec) + 1024;   // feature tile, FP32
    float* fsh = reinterpret_cast<float*>(bufX + xb);         // [NS][128] partial output sums
    uint64_t* bar = reinterpret_cast<uint64_t*>(fsh + 2 * 128);  // [0] MMA, [1] weights, [2] features
    uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 3);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r = tid & 127, hf = tid >> 7, cb = hf * UH;
    if (tid == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        tc::mbar_init(&bar[2], 1);
        tc::fence_async_smem();
    }
    if (warp == 0) tc::tmem_alloc(tbase, 256);  // D0 | D1 | H1 hi | H1 lo
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const long t_end = t_first + n_tiles;
    long tile = t_first + blockIdx.x;
    pdl_wait();  // the optimizer's weight image
    if (tid == 0) {
        tc::mbar_expect_tx(&bar[1], 2 * w0b + 2 * w1b + 1024);
        tc::bulk_g2s(w0, a.wimg, 2 * w0b + 2 * w1b, &bar[1]);  // W0 | W1 (W1^T not needed)
        tc::bulk_g2s(vec, a.wimg + 2 * w0b + 4 * w1b, 1024, &bar[1]);
        tc::mbar_expect_tx(&bar[2], xb);
        tc::bulk_g2s(bufX, a.ximg + tile * xb, xb, &bar[2]);
    }
    tc::mbar_wait(&bar[1], 0);
    const float b2 = vec[192], mu = vec[193];
    uint32_t mph = 0, xph = 0;
    auto mma_wait = [&]() {
        if (warp == 0) tc::mbar_wait(&bar[0], mph);
        mph ^= 1;
        __syncthreads();
        tc::fence_after_sync();
    };
    double loss = 0.0, mn = INFINITY;
    for (; tile < t_end; tile += gridDim.x) {
        const long row = tile * 128 + r;
        const bool live = row >= a.b0 && row < a.b1;
        const double yrow = (live && (a.mode & 1) && hf == 0) ? __ldg(a.y + row) : 0.0;
        tc::mbar_wait(&bar[2], xph);
        xph ^= 1;
        x_to_tmem<NS>(bufX, dp, tm, lb, r, hf);  // the feature tile, split, into tensor memory
        tc::tmem_wait_st();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        if (tid == 0) {
            if (tile + gridDim.x < t_end) {  // feature tile read: stream in the next one
                tc::mbar_expect_tx(&bar[2], xb);
                tc::bulk_g2s(bufX, a.ximg + (tile + gridDim.x) * xb, xb, &bar[2]);
            }
            // ---- F0: D0 = X W0^T, X from tensor memory
            tc::gemm3_ts(tm, tm + 128, tm + 128 + dp, tc::kmajor(w0, w0b, U), dp, tc::idesc_tf32(128, U, 0, 0), 0);
            tc::commit(&bar[0]);
        }
        mma_wait();
#pragma unroll
        for (int c = 0; c < UH; c += 16) {  // H1 = act(D0 + b0) -> tensor memory, hi | lo
            float v[16], lo[16];
            tc::tmem_ld16(tm + lb + cb + c, v);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const float h = act_f<ACT>(v[q] + vec[cb + c + q]);
                v[q] = tc::tf32_rna(h);
                lo[q] = h - v[q];
            }
            tc::tmem_st16(tm + lb + 128 + cb + c, v);
            tc::tmem_st16(tm + lb + 192 + cb + c, lo);
        }
        tc::tmem_wait_st();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        if (tid == 0) {  // ---- F1: D1 = H1 W1^T, H1 from tensor memory
            tc::gemm3_ts(tm + 64, tm + 128, tm + 192, tc::kmajor(w1, w1b, U), U, tc::idesc_tf32(128, U, 0, 0), 0);
            tc::commit(&bar[0]);
        }
        mma_wait();
        float h2[UH];
#pragma unroll
        for (int c = 0; c < UH; c += 16) tc::tmem_ld16(tm + lb + 64 + cb + c, h2 + c);
#pragma unroll
        for (int q = 0; q < UH; ++q) h2[q] = act_f<ACT>(h2[q] + vec[64 + cb + q]);
        float fp = 0.0f;
#pragma unroll
        for (int j = 0; j < UH; ++j) fp = fmaf(h2[j], vec[128 + cb + j], fp);
        float f = b2 + fp;
        if (NS > 1) {
            fsh[hf * 128 + r] = fp;
            __syncthreads();
            float fs = fsh[r];
#pragma unroll
            for (int h = 1; h < NS; ++h) fs += fsh[h * 128 + r];
            f = b2 + fs;
        }
        if ((a.mode & 8) && live)
#pragma unroll
            for (int j = 0; j < UH; j += 4)
                *reinterpret_cast<float4*>(a.H2 + row * U + cb + j) = make_float4(h2[j], h2[j + 1], h2[j + 2], h2[j + 3]);
        if (live && hf == 0) {
            const double ph = static_cast<double>((f < 0.0f ? 0.0f : f) + mu);
            if (a.mode & 1) {
                const double res = ph - yrow;
                loss += res * res;
            }
            if (a.mode & 2) mn = fmin(mn, static_cast<double>(f + mu));
            if (a.mode & 4) a.pred[row] = ph;
        }
    }
    // per-CTA partials: warpgroup 0 holds the per-row terms (fixed order over its warps)
    tc::fence_before_sync();
    __syncthreads();
    double* red = reinterpret_cast<double*>(bufX);
    loss = warp_sum(loss);
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0 && warp < 4) {
        red[warp] = loss;
        red[4 + warp] = mn;
    }
    __syncthreads();
    if (tid == 0) {
        if (a.mode & 1) a.lpart[blockIdx.x] = red[0] + red[1] + red[2] + red[3];
        if (a.mode & 2) a.mpart[blockIdx.x] = fmin(fmin(red[4], red[5]), fmin(red[6], red[7]));
    }
    if (warp == 0) tc::tmem_dealloc(tm, 256);
}

// SGD tile kernel, two CTAs per SM, for the feature-matrix path (host rows and
// sets the layer-0 split kernels do not serve, regress_split.cu): the A
// operands of layer 1 (H1) and of the backward GEMM (G2) go through tensor
// memory instead of a shared H tile, the vectors are read through L1, and each
// thread covers 32 columns in two 16-column passes; layer 2's activations are
// stored back into D1 and reloaded for the gradient pass.  Admission
// (tc_two_cta): sgd_tc_smem <= 113 KB, i.e. dp <= 48 at U = 64; TMEM: D0 | D1
// in columns 0..127, the feature tile's hi | lo split at 128..128 + 2 dp.
// Same arithmetic and outputs as k_tile_tc's SGD mode.
template <int U>
struct SgdShape {
    static constexpr int UH = U < 32 ? U : 32;  // columns per thread
    static constexpr int NS = U / UH;           // warpgroups
    static constexpr int CP = 16;               // columns per pass
    static constexpr int NP = UH / CP;
    static constexpr int threads = 128 * NS;
    static constexpr int warps = 4 * NS;
};

__host__ __device__ constexpr size_t sgd_tc_smem(int U, int dp) {
    return 2ull * U * dp * 4 + 4ull * U * U * 4 + 1ull * 128 * dp * 4 + 128 * 4 + 64;
}

template <int U, int ACT>
__global__ void __launch_bounds__(SgdShape<U>::threads, 2) k_sgd_tc(TileArgs a, long t_first, long n_tiles) {
    using S = SgdShape<U>;
    constexpr int NS = S::NS, UH = S::UH, CP = S::CP, NP = S::NP;
    extern __shared__ __align__(128) uint8_t sm[];
    const int dp = a.dp;
    const uint32_t w0b = U * dp * 4, w1b = U * U * 4, xb = x_plane_bytes(dp);
    uint8_t* w0 = sm;                                        // W0 hi | lo
    uint8_t* w1 = w0 + 2 * w0b;                              // W1 hi | lo
    uint8_t* w1t = w1 + 2 * w1b;                             // W1^T hi | lo
    uint8_t* bufX = w1t + 2 * w1b;                           // feature tile, FP32
    float* fsh = reinterpret_cast<float*>(bufX + xb);        // [128] output-sum exchange
    uint64_t* bar = reinterpret_cast<uint64_t*>(fsh + 128);  // [0] MMA, [1] weights, [2] features
    uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 3);
    const float* vec = reinterpret_cast<const float*>(a.wimg + 2 * w0b + 4 * w1b);  // b0 | b1 | w2 | b2, mu
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r = tid & 127, hf = tid >> 7, cb = hf * UH;
    if (tid == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        tc::mbar_init(&bar[2], 1);
        tc::fence_async_smem();
    }
    if (warp == 0) tc::tmem_alloc(tbase, 256);  // D0 | D1, then Dbp | A hi | A lo
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const long t_end = t_first + n_tiles;
    long tile = t_first + blockIdx.x;
    pdl_wait();  // the optimizer's weight image, the previous weight gradient's reads of H1t, G2t, G1t
    if (tid == 0) {
        tc::mbar_expect_tx(&bar[1], 2 * w0b + 4 * w1b);
        tc::bulk_g2s(w0, a.wimg, 2 * w0b + 4 * w1b, &bar[1]);  // W0 | W1 | W1^T
        tc::mbar_expect_tx(&bar[2], xb);
        tc::bulk_g2s(bufX, a.ximg + tile * xb, xb, &bar[2]);
    }
    const float b2 = __ldg(vec + 192), mu = __ldg(vec + 193);
    tc::mbar_wait(&bar[1], 0);
    uint32_t mph = 0, xph = 0;
    auto mma_wait = [&]() {
        if (warp == 0) tc::mbar_wait(&bar[0], mph);
        mph ^= 1;
        __syncthreads();
        tc::fence_after_sync();
    };
    auto cta_sync = [&]() {
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
    };
    double loss = 0.0, dmu = 0.0;
    float gb2 = 0.0f;
    float acc_w2[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) acc_w2[p] = 0.0f;

    for (; tile < t_end; tile += gridDim.x) {
        const long row = tile * 128 + r;
        const bool live = row >= a.b0 && row < a.b1;
        const long trow = row - a.b0;
        const double yrow = live ? __ldg(a.y + row) : 0.0;
        tc::mbar_wait(&bar[2], xph);
        xph ^= 1;
        x_to_tmem<NS>(bufX, dp, tm, lb, r, hf);  // the feature tile, split, into tensor memory
        tc::tmem_wait_st();
        cta_sync();
        if (tid == 0) {
            if (tile + gridDim.x < t_end) {  // feature tile read: stream in the next one
                tc::mbar_expect_tx(&bar[2], xb);
                tc::bulk_g2s(bufX, a.ximg + (tile + gridDim.x) * xb, xb, &bar[2]);
            }
            // ---- F0: D0 = X W0^T, X from tensor memory
            tc::gemm3_ts(tm, tm + 128, tm + 128 + dp, tc::kmajor(w0, w0b, U), dp, tc::idesc_tf32(128, U, 0, 0), 0);
            tc::commit(&bar[0]);
        }
        mma_wait();
        // H1 = act(D0 + b0) -> A (hi | lo), H1t; act'(H1) back into D0
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int c0 = cb + p * CP;
            float v[CP], hi[CP];
            tc::tmem_ld16(tm + lb + c0, v);
#pragma unroll
            for (int q = 0; q < CP; ++q) {
                v[q] = act_f<ACT>(v[q] + __ldg(vec + c0 + q));
                hi[q] = tc::tf32_rna(v[q]);
            }
            if (live)
#pragma unroll
                for (int q = 0; q < CP; ++q) a.H1t[(c0 + q) * a.ld_t + trow] = v[q];
            tc::tmem_st16(tm + lb + 128 + c0, hi);
#pragma unroll
            for (int q = 0; q < CP; ++q) {
                hi[q] = v[q] - hi[q];  // lo
                v[q] = act_d<ACT>(v[q]);
            }
            tc::tmem_st16(tm + lb + 192 + c0, hi);
            tc::tmem_st16(tm + lb + c0, v);
        }
        tc::tmem_wait_st();
        cta_sync();
        if (tid == 0) {  // ---- F1: D1 = H1 W1^T, H1 from tensor memory
            tc::gemm3_ts(tm + 64, tm + 128, tm + 192, tc::kmajor(w1, w1b, U), U, tc::idesc_tf32(128, U, 0, 0), 0);
            tc::commit(&bar[0]);
        }
        mma_wait();
        // f = b2 + H2 w2 (warpgroup partials summed in order 0, 1)
        float fp = 0.0f;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int c0 = cb + p * CP;
            float h[CP];
            tc::tmem_ld16(tm + lb + 64 + c0, h);
#pragma unroll
            for (int j = 0; j < CP; ++j) {
                h[j] = act_f<ACT>(h[j] + __ldg(vec + 64 + c0 + j));
                fp = fmaf(h[j], __ldg(vec + 128 + c0 + j), fp);
            }
            tc::tmem_st16(tm + lb + 64 + c0, h);  // H2 back into D1 for the gradient pass
        }
        tc::tmem_wait_st();
        float f = b2 + fp;
        if (NS > 1) {
            if (hf == 1) fsh[r] = fp;
            __syncthreads();
            if (hf == 0) {
                f = b2 + (fp + fsh[r]);
                fsh[r] = f;
            }
            __syncthreads();
            f = fsh[r];
        }
        // residual, output layer, mu
        float dd = 0.0f;
        if (live) {
            const float pr = ((a.head && f < 0.0f) ? 0.0f : f) + mu;
            const double res = static_cast<double>(pr) - yrow;
            const double dm = 2.0 * res / a.nb;
            if (hf == 0) {
                loss += res * res;
                dmu += dm;
            }
            dd = static_cast<float>(dm);
            if (a.head && !(f > 0.0f)) dd = 0.0f;
        }
        if (hf == 0) gb2 += dd;
        // G2 = dd w2 act'(H2) -> A (hi | lo; layer 1 has consumed H1), G2t; output-layer gradient
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const int c0 = cb + p * CP;
            float h[CP], g[CP];
            tc::tmem_ld16(tm + lb + 64 + c0, h);  // H2
#pragma unroll
            for (int j = 0; j < CP; ++j) g[j] = dd * h[j];
            acc_w2[p] += bfly_sum<CP>(g, lane);
#pragma unroll
            for (int j = 0; j < CP; ++j) g[j] = dd * __ldg(vec + 128 + c0 + j) * act_d<ACT>(h[j]);
            if (live)
#pragma unroll
                for (int j = 0; j < CP; ++j) a.G2t[(c0 + j) * a.ld_t + trow] = g[j];
#pragma unroll
            for (int j = 0; j < CP; ++j) h[j] = tc::tf32_rna(g[j]);
            tc::tmem_st16(tm + lb + 128 + c0, h);
#pragma unroll
            for (int j = 0; j < CP; ++j) h[j] = g[j] - h[j];
            tc::tmem_st16(tm + lb + 192 + c0, h);
        }
        tc::tmem_wait_st();
        cta_sync();  // every D1 read done: the backward GEMM reuses its columns
        if (tid == 0) {  // ---- B: Dbp = G2 W1 (B: the W1^T tile), G2 from tensor memory
            tc::gemm3_ts(tm + 64, tm + 128, tm + 192, tc::kmajor(w1t, w1b, U), U, tc::idesc_tf32(128, U, 0, 0), 0);
            tc::commit(&bar[0]);
        }
        mma_wait();
#pragma unroll
        for (int p = 0; p < NP; ++p) {  // G1 = Dbp act'(H1) -> G1t
            const int c0 = cb + p * CP;
            float g[CP], dv[CP];
            tc::tmem_ld16(tm + lb + 64 + c0, g);
            tc::tmem_ld16(tm + lb + c0, dv);
            if (live)
#pragma unroll
                for (int j = 0; j < CP; ++j) a.G1t[(c0 + j) * a.ld_t + trow] = g[j] * dv[j];
        }
        cta_sync();  // TMEM reads of D0 / Dbp done before the next tile's F0
    }

    // ---- per-CTA partials (fixed order over the warps), scratch in the feature tile
    cta_sync();
    constexpr int NWP = S::warps;
    float* part = reinterpret_cast<float*>(bufX);                    // [warp][64]
    double* red = reinterpret_cast<double*>(part + NWP * 64);        // [3][warps]
    if (lane < CP)
#pragma unroll
        for (int p = 0; p < NP; ++p) part[warp * 64 + cb + p * CP + lane] = acc_w2[p];
    loss = warp_sum(loss);
    dmu = warp_sum(dmu);
    gb2 = warp_sum(gb2);
    if (lane == 0) {
        red[warp] = loss;
        red[NWP + warp] = dmu;
        red[2 * NWP + warp] = gb2;
    }
    __syncthreads();
    float* gout = a.gpart + static_cast<size_t>(blockIdx.x) * a.P;
    if (tid < U) {
        const int w0q = (tid / UH) * 4;  // first warp of the owning warpgroup
        gout[a.off2 + tid] = part[(w0q + 0) * 64 + tid] + part[(w0q + 1) * 64 + tid] + part[(w0q + 2) * 64 + tid] +
                             part[(w0q + 3) * 64 + tid];
    }
    if (tid == 0) {
        a.lpart[blockIdx.x] = red[0] + red[1] + red[2] + red[3];  // warpgroup 0 holds the per-row terms
        gout[a.P - 1] = static_cast<float>(red[NWP] + red[NWP + 1] + red[NWP + 2] + red[NWP + 3]);
        gout[a.off2 + U] = static_cast<float>(red[2 * NWP] + red[2 * NWP + 1] + red[2 * NWP + 2] + red[2 * NWP + 3]);
    }
    if (warp == 0) tc::tmem_dealloc(tm, 256);
}

// Refit Gram (regressor.cpp:191-213) in FP64 from the FP32 layer-2
// activations: z = [h2, 1, y - mu] padded to MP = 4 * NBK, one thread per
// 4x4 block (bi <= bj) of z z^T, 64-row chunks staged in shared memory,
// chunk c -> CTA c % gridDim.x (fixed), one partial per CTA.
template <int U>
struct GramShape {
    static constexpr int B = 8;                           // register block edge
    static constexpr int MP = ((U + 2 + B - 1) / B) * B;  // [h2, 1, y - mu] padded
    static constexpr int NBK = MP / B;
    static constexpr int pairs = NBK * (NBK + 1) / 2;
    static constexpr int G = pairs <= 16 ? 8 : 4;        // row groups per CTA (fixed order at the end)
    static constexpr int threads = ((pairs * G + 31) / 32) * 32;
    static constexpr int CH = 64;
    static constexpr int LD = MP + 2;  // padded row (doubles)
};

template <int U>
__global__ void __launch_bounds__(GramShape<U>::threads) k_gram_h2(const float* __restrict__ H2,
                                                                    const double* __restrict__ y, long R,
                                                                    const float* __restrict__ params, int P,
                                                                    double* __restrict__ gpart) {
    using S = GramShape<U>;
    constexpr int B = S::B;
    __shared__ __align__(16) double zs[S::CH * S::LD];
    const int t = threadIdx.x;
    const int grp = t / S::pairs, pt = t % S::pairs;  // row group, block pair
    int bi = 0, rem = pt;  // pt -> (bi, bj), bi <= bj
    while (bi < S::NBK && rem >= S::NBK - bi) {
        rem -= S::NBK - bi;
        ++bi;
    }
    const bool act = grp < S::G;
    const int bj = bi + rem;
    const double mu = static_cast<double>(params[P - 1]);
    double acc[B * B];
#pragma unroll
    for (int k = 0; k < B * B; ++k) acc[k] = 0.0;
    const long nch = (R + S::CH - 1) / S::CH;
    for (long ch = blockIdx.x; ch < nch; ch += gridDim.x) {
        const long base = ch * S::CH;
        const int rows = static_cast<int>(min(static_cast<long>(S::CH), R - base));
        __syncthreads();
        for (int i = t; i < S::CH * (U / 4); i += blockDim.x) {
            const int r = i / (U / 4), c4 = (i % (U / 4)) * 4;
            float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (r < rows) v = __ldg(reinterpret_cast<const float4*>(H2 + (base + r) * U + c4));
            double* z = zs + r * S::LD + c4;
            z[0] = v.x;
            z[1] = v.y;
            z[2] = v.z;
            z[3] = v.w;
        }
        for (int r = t; r < S::CH; r += blockDim.x) {
            double* z = zs + r * S::LD;
            const bool in = r < rows;
            z[U] = in ? 1.0 : 0.0;
            z[U + 1] = in ? y[base + r] - mu : 0.0;
            for (int c = U + 2; c < S::MP; ++c) z[c] = 0.0;
        }
        __syncthreads();
        if (act)
            for (int r = grp; r < rows; r += S::G) {
                const double2* zi = reinterpret_cast<const double2*>(zs + r * S::LD + B * bi);
                const double2* zj = reinterpret_cast<const double2*>(zs + r * S::LD + B * bj);
                double av[B], bv[B];
#pragma unroll
                for (int h = 0; h < B / 2; ++h) {
                    const double2 x = zi[h], w = zj[h];
                    av[2 * h] = x.x;
                    av[2 * h + 1] = x.y;
                    bv[2 * h] = w.x;
                    bv[2 * h + 1] = w.y;
                }
#pragma unroll
                for (int p = 0; p < B; ++p)
#pragma unroll
                    for (int q = 0; q < B; ++q) acc[p * B + q] = fma(av[p], bv[q], acc[p * B + q]);
            }
    }
    // Row groups summed in group order through shared memory (reusing the chunk buffer).
    __syncthreads();
    double* red = zs;  // [G-1][pairs][B*B] would exceed it: accumulate group by group instead
    for (int g = 1; g < S::G; ++g) {
        if (grp == g && act)
#pragma unroll
            for (int k = 0; k < B * B; ++k) red[pt * B * B + k] = acc[k];
        __syncthreads();
        if (grp == 0)
#pragma unroll
            for (int k = 0; k < B * B; ++k) acc[k] += red[pt * B * B + k];
        __syncthreads();
    }
    if (grp != 0) return;
    // Packed output: (a, b) a <= b < m = U+1 -> upper-triangle index; rhs c = (c, U+1).
    constexpr int m = U + 1, tri = m * (m + 1) / 2;
    double* out = gpart + static_cast<size_t>(blockIdx.x) * (tri + m);
#pragma unroll
    for (int p = 0; p < B; ++p)
#pragma unroll
        for (int q = 0; q < B; ++q) {
            const int ra = B * bi + p, cb = B * bj + q;
            if (ra < m && cb < m && ra <= cb) out[ra * m - ra * (ra - 1) / 2 + (cb - ra)] = acc[p * B + q];
            else if (ra < m && cb == m) out[tri + ra] = acc[p * B + q];
        }
}

// Four consecutive floats, zero beyond `valid`; 16-byte load when aligned.
__device__ __forceinline__ float4 ld4(const float* p, bool vec, int valid) {
    float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (valid <= 0) return v;
    if (vec) {
        v = __ldg(reinterpret_cast<const float4*>(p));
    } else {
        v.x = p[0];
        if (valid > 1) v.y = p[1];
        if (valid > 2) v.z = p[2];
        if (valid > 3) v.w = p[3];
    }
    if (valid < 4) {
        if (valid < 2) v.y = 0.0f;
        if (valid < 3) v.z = 0.0f;
        v.w = 0.0f;
    }
    return v;
}

// Chunk tiles are 128B-swizzled K-major (tc.cuh sw_off): 64 feature rows x
// kWgK batch rows (one 128-byte atom column), so the coalesced 16-byte row
// loads land in distinct bank groups.  64 KB of tiles and <= 85 registers keep
// three CTAs per SM, whose load / split / MMA phases interleave.
constexpr int kWgThreads = 256;
constexpr int kWgK = 32;                     // batch rows per chunk (the MMAs' K)
constexpr uint32_t kWgTile = 64 * kWgK * 4;   // one plane of a 64-row chunk tile
constexpr uint32_t kWgTileB1 = 72 * kWgK * 4; // H1t tile: U rows + a row of ones (+ zero rows to 8)
// The Xt tile has XR rows: 64 for dp <= 64, kWgXMax for wide inputs (one CTA
// per SM then: 512 TMEM columns, gW0 at column 128 with N = dp).
__host__ __device__ constexpr size_t wgrad_smem(int XR) {
    return 4 * static_cast<size_t>(kWgTile) + 2ull * XR * kWgK * 4 + 2 * static_cast<size_t>(kWgTileB1) + 64 + 1024;
}

template <int U, int XR>
__global__ void __launch_bounds__(kWgThreads, XR > 64 ? 1 : 2) k_wgrad_tc(WgradArgs a) {
    constexpr uint32_t kWgTileX = XR * kWgK * 4;
    constexpr int kTmemCols = XR > 64 ? 512 : 256;
    extern __shared__ __align__(128) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    // The row of ones in tB1 (row U) and tB0 (row d, a pad column of the
    // features) turns the last output columns into the bias gradients
    // sum_r G2[r][o] (gb1) and sum_r G1[r][o] (gb0).
    uint8_t* tA1 = sm;                                // G2t chunk: 64 (o, zero-padded) x kWgK (rows)
    uint8_t* tA0 = sm + 2 * kWgTile;                  // G1t chunk
    uint8_t* tB0 = sm + 4 * kWgTile;                  // Xt chunk: dp (of XR) x kWgK, row d = 1
    uint8_t* tB1 = tB0 + 2 * kWgTileX;                // H1t chunk: U x kWgK, row U = 1
    uint64_t* mbar = reinterpret_cast<uint64_t*>(tB1 + 2 * kWgTileB1);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int dp = a.dp;
    if (t == 0) tc::mbar_init(mbar, 1);
    if (warp == 0) tc::tmem_alloc(tbase, kTmemCols);
    for (int i = t; i < (4 * kWgTile + 2 * kWgTileX + 2 * kWgTileB1) / 16; i += kWgThreads)
        reinterpret_cast<float4*>(sm)[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    const long r_begin = static_cast<long>(blockIdx.x) * a.rows_per_cta;
    const long r_end = a.probe ? r_begin : min(r_begin + a.rows_per_cta, a.rows);  // probe: fixed costs only
    const bool vt = (a.ld_t % 4) == 0;
    const bool vx = (a.ld_x % 4) == 0 && (a.row0 % 4) == 0;
    constexpr int Q = kWgK / 4;                                 // float4 per feature row of a chunk
    constexpr int NF = (U * Q + kWgThreads - 1) / kWgThreads;   // per thread per activation array
    constexpr int NX = (XR * Q + kWgThreads - 1) / kWgThreads;  // per thread of the Xt chunk (dp <= XR)
    struct Regs {
        float4 g2[NF], h1[NF], g1[NF], x[NX];
    };
    auto load = [&](Regs& q, long c0) {
        const int n = static_cast<int>(min(static_cast<long>(kWgK), r_end - c0));
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const int idx = t + i * kWgThreads, f = idx / Q, k = (idx % Q) * 4;
            if (f < U) {
                const size_t o = static_cast<size_t>(f) * a.ld_t + c0 + k;
                q.g2[i] = ld4(a.G2t + o, vt, n - k);
                q.h1[i] = ld4(a.H1t + o, vt, n - k);
                q.g1[i] = ld4(a.G1t + o, vt, n - k);
            }
        }
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            const int idx = t + i * kWgThreads, f = idx / Q, k = (idx % Q) * 4;
            if (f < dp && f != a.d) q.x[i] = ld4(a.Xt + static_cast<size_t>(f) * a.ld_x + a.row0 + c0 + k, vx, n - k);
        }
    };
    uint32_t phase = 0;
    int first = 1;
    auto consume = [&](const Regs& q, long c0) {
        if (!first) {  // previous chunk's MMAs done reading the tiles
            tc::mbar_wait(mbar, phase);
            phase ^= 1;
        }
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const int idx = t + i * kWgThreads, f = idx / Q, k = (idx % Q) * 4;
            if (f < U) {
                tc::put_split4_sw(tA1, kWgTile, f, k, 64, q.g2[i]);
                tc::put_split4_sw(tB1, kWgTileB1, f, k, 72, q.h1[i]);
                tc::put_split4_sw(tA0, kWgTile, f, k, 64, q.g1[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            const int idx = t + i * kWgThreads, f = idx / Q, k = (idx % Q) * 4;
            if (f < dp && f != a.d) tc::put_split4_sw(tB0, kWgTileX, f, k, XR, q.x[i]);
        }
        if (t < 2 * Q) {  // the rows of ones (1 for the chunk's live rows, 0 past the batch end)
            const int k = (t % Q) * 4, n = static_cast<int>(min(static_cast<long>(kWgK), r_end - c0));
            const float4 one = make_float4(k < n ? 1.0f : 0.0f, k + 1 < n ? 1.0f : 0.0f, k + 2 < n ? 1.0f : 0.0f,
                                           k + 3 < n ? 1.0f : 0.0f);
            if (t < Q) tc::put_split4_sw(tB1, kWgTileB1, U, k, 72, one);
            else tc::put_split4_sw(tB0, kWgTileX, a.d, k, XR, one);
        }
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        if (warp == 0) {
            const uint32_t R64 = 64;
            tc::gemm3_sw_warp(tm, tc::OperandSW{tc::smem_u32(tA1), kWgTile, R64, 0},
                              tc::OperandSW{tc::smem_u32(tB1), kWgTileB1, 72u, 0}, kWgK,
                              tc::idesc_tf32(64, U + 8, 0, 0), !first, nullptr);
            tc::gemm3_sw_warp(tm + 128, tc::OperandSW{tc::smem_u32(tA0), kWgTile, R64, 0},
                              tc::OperandSW{tc::smem_u32(tB0), kWgTileX, static_cast<uint32_t>(XR), 0}, kWgK,
                              tc::idesc_tf32(64, dp, 0, 0), !first, mbar);
        }
        first = 0;
    };
    // Two register sets: chunk c+2's loads are in flight while chunk c is
    // split into shared memory and its MMAs run.
    Regs ra, rb;
    if (r_begin < r_end) load(ra, r_begin);
    if (r_begin + kWgK < r_end) load(rb, r_begin + kWgK);
    for (long c0 = r_begin; c0 < r_end; c0 += 2 * kWgK) {
        consume(ra, c0);
        if (c0 + 2 * kWgK < r_end) load(ra, c0 + 2 * kWgK);
        if (c0 + kWgK < r_end) {
            consume(rb, c0 + kWgK);
            if (c0 + 3 * kWgK < r_end) load(rb, c0 + 3 * kWgK);
        }
    }
    if (!first) {
        tc::mbar_wait(mbar, phase);
        tc::fence_after_sync();
    }
    // Partial row of this CTA: W1 [U][U+8] (column U = gb1) then W0 [U][dp]
    // (column d = gb0), 16-byte stores.
    float* gout = a.gpart + static_cast<size_t>(blockIdx.x) * (U * (U + 8) + U * dp);
    if (warp < 4) {
        const int o = warp * 16 + lane;  // M=64 accumulator: row 16w+t in lane 32w+t, t < 16
        const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
        const bool own = lane < 16 && o < U;
#pragma unroll
        for (int c = 0; c < U + 8; c += 8) {
            float v[8];
            tc::tmem_ld8(tm + lane_base + c, v);
            if (own)
#pragma unroll
                for (int q = 0; q < 8; q += 4)
                    *reinterpret_cast<float4*>(gout + o * (U + 8) + c + q) =
                        first ? make_float4(0.0f, 0.0f, 0.0f, 0.0f) : make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
        for (int c = 0; c < dp; c += 16) {
            float v[16];
            tc::tmem_ld16(tm + lane_base + 128 + c, v);
            if (own)
#pragma unroll
                for (int q = 0; q < 16; q += 4)
                    *reinterpret_cast<float4*>(gout + U * (U + 8) + o * dp + c + q) =
                        first ? make_float4(0.0f, 0.0f, 0.0f, 0.0f) : make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, kTmemCols);
}

// Diagnostic GEMM: D (M x N) = A (M x K) B (N x K)^T; test hook for the
// descriptor conventions.  variant 0: K-major no-swizzle, 1: K-major SW128,
// 2: A MN-major, 3: B MN-major, 4: both MN-major (no swizzle; an MN-major
// operand is stored as the K x MN core tile, SBO = K/8*128, LBO = 128),
// 5 / 6 / 7: A / B / both MN-major with 128B swizzle (K x MN atoms).
__global__ void k_tc_gemm_diag(int M, int N, int K, const float* A, const float* B, float* D, int variant) {
    extern __shared__ __align__(128) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t abytes = M * ((K + 31) / 32) * 32 * 4, bbytes = N * ((K + 31) / 32) * 32 * 4;
    uint8_t* ta = sm;
    uint8_t* tb = sm + 2 * abytes;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(tb + 2 * bbytes);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);
    const int t = threadIdx.x, warp = t >> 5;
    const bool swz = variant == 1 || (variant >= 5 && variant <= 7);
    const bool amn = variant == 2 || variant == 4 || variant == 5 || variant == 7;
    const bool bmn = variant == 3 || variant == 4 || variant == 6 || variant == 7;
    if (t == 0) tc::mbar_init(mbar, 1);
    if (warp == 0) tc::tmem_alloc(tbase, 256);
    for (int i = t; i < 2 * (abytes + bbytes) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.0f;
    __syncthreads();
    for (int i = t; i < M * K; i += blockDim.x) {
        if (swz && amn) tc::put_split_sw(ta, abytes, i % K, i / K, K, A[i]);
        else if (swz) tc::put_split_sw(ta, abytes, i / K, i % K, M, A[i]);
        else if (amn) tc::put_split(ta, abytes, i % K, i / K, K, A[i]);
        else tc::put_split(ta, abytes, i / K, i % K, M, A[i]);
    }
    for (int i = t; i < N * K; i += blockDim.x) {
        if (swz && bmn) tc::put_split_sw(tb, bbytes, i % K, i / K, K, B[i]);
        else if (swz) tc::put_split_sw(tb, bbytes, i / K, i % K, N, B[i]);
        else if (bmn) tc::put_split(tb, bbytes, i % K, i / K, K, B[i]);
        else tc::put_split(tb, bbytes, i / K, i % K, N, B[i]);
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    if (variant == 8) {  // A (hi | lo) from tensor memory at columns 128 / 192 (M = 128, K <= 64)
        const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
        for (int c0 = 0; c0 < K; c0 += 16) {
            float hi[16], lo[16];
            for (int q = 0; q < 16; ++q) {
                const float a = (t < M && c0 + q < K) ? A[t * K + c0 + q] : 0.0f;
                hi[q] = tc::tf32_rna(a);
                lo[q] = a - hi[q];
            }
            tc::tmem_st16(tm + lane_base + 128 + c0, hi);
            tc::tmem_st16(tm + lane_base + 192 + c0, lo);
        }
        tc::tmem_wait_st();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        if (t == 0) {
            tc::gemm3_ts(tm, tm + 128, tm + 192, tc::kmajor(tb, bbytes, N), K, tc::idesc_tf32(M, N, 0, 0), 0);
            tc::commit(mbar);
        }
    } else if (t == 0) {
        if (swz) {
            // MN-major SW128 tiles hold K rows x MN columns (R = K).
            tc::gemm3_sw(tm, tc::OperandSW{tc::smem_u32(ta), abytes, static_cast<uint32_t>(amn ? K : M), amn},
                         tc::OperandSW{tc::smem_u32(tb), bbytes, static_cast<uint32_t>(bmn ? K : N), bmn}, K,
                         tc::idesc_tf32(M, N, amn, bmn), 0);
        } else {
            tc::gemm3(tm, amn ? tc::mnmajor(ta, abytes, K) : tc::kmajor(ta, abytes, M),
                      bmn ? tc::mnmajor(tb, bbytes, K) : tc::kmajor(tb, bbytes, N), K,
                      tc::idesc_tf32(M, N, amn, bmn), 0);
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

// Tensor-core rate probe: every CTA (one per SM) issues `iters` kind::tf32
// MMAs of M x N x 8 back to back on the same K-major tiles into one TMEM
// accumulator (warp-collective issue, one commit at the end).
__global__ void k_tc_rate(int M, int N, int iters, float* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + 2 * 128 * 8 * 4 * 2);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 2 * 128 * 8 * 2; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i % 7);
    if (t == 0) tc::mbar_init(mbar, 1);
    if (warp == 0) tc::tmem_alloc(tbase, 256);
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    if (warp == 0) {
        const uint32_t issue = tc::elect_one();
        const uint64_t da = tc::sdesc(tc::smem_u32(sm), 128u * 16, 128u);
        const uint64_t db = tc::sdesc(tc::smem_u32(sm + 128 * 8 * 4), 256u / 8 * 128, 128u);
        const uint32_t id = tc::idesc_tf32(M, N, 0, 0);
        for (int i = 0; i < iters; ++i) tc::mma_tf32_if(issue, tm, da, db, id, i > 0);
        tc::commit_if(issue, mbar);
    }
    tc::mbar_wait(mbar, 0);
    tc::fence_after_sync();
    if (warp == 0) {
        float v[16];
        tc::tmem_ld16(tm, v);
        if (t == 0) sink[blockIdx.x] = v[0];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, 256);
}

// ------------------------------------------------------------------ host

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("HCVA_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool tc_two_cta(int u, int dp) {
    static const bool on = [] {
        const char* e = std::getenv("HCVA_TWO_CTA");
        return !(e && e[0] == '0');
    }();
    return on && u >= 16 && dp <= 64 && sgd_tc_smem(u, dp) <= 113 * 1024 && eval_tc_smem(u, dp) <= 113 * 1024;
}

bool tc_eligible(int d, int h, int u) {
    if (const char* e = std::getenv("HCVA_REGRESS_SIMT"))
        if (std::atoi(e)) return false;
    const int dp = ((d + 16) / 16) * 16;
    return h == 2 && (u == 16 || u == 32 || u == 64) && d >= 1 && dp <= kWgXMax &&
           (tile_tc_smem(u, dp) <= 227 * 1024 || tile_tc_smem_ch(u) <= 227 * 1024);
}

// Input width padded for the tensor-core tiles, with at least one pad column:
// the weight-gradient kernel puts a row of ones there (bias gradient of layer 0).
int tc_dp(int d) { return ((d + 16) / 16) * 16; }

void launch_pack_w(int u, int d, int dp, int off0, int off1, int off2, int P, const float* params, uint8_t* wimg,
                   cudaStream_t s) {
    const int n = std::max(256, std::max(u * dp, u * u));
    k_pack_w<<<(n + 255) / 256, 256, 0, s>>>(u, d, dp, off0, off1, off2, P, params, wimg);
}

void launch_pack_x(const float* X, long R, int d, int dp, uint8_t* ximg, float* Xt, long ld_x, int xf32,
                   cudaStream_t s) {
    const long tiles = (R + 127) / 128;
    if (tiles > 0) k_pack_x<<<static_cast<unsigned>(tiles), 128, 0, s>>>(X, R, d, dp, ximg, Xt, ld_x, xf32);
}

template <int U, int ACT>
void launch_tile_ua(const TileArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    if (tile_chunked(U, a.dp)) {
        const size_t smem = tile_tc_smem_ch(U);
        HCVA_CUDA(cudaFuncSetAttribute(k_tile_tc<U, ACT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        pdl_launch(k_tile_tc<U, ACT, true>, dim3(ctas), dim3(TileShape<U>::threads), smem, s, a, t_first, n_tiles);
        return;
    }
    const size_t smem = tile_tc_smem(U, a.dp);
    HCVA_CUDA(cudaFuncSetAttribute(k_tile_tc<U, ACT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pdl_launch(k_tile_tc<U, ACT, false>, dim3(ctas), dim3(TileShape<U>::threads), smem, s, a, t_first, n_tiles);
}

template <int U>
void launch_tile_u(const TileArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    switch (a.act) {
        case 0: launch_tile_ua<U, 0>(a, t_first, n_tiles, ctas, s); break;
        case 1: launch_tile_ua<U, 1>(a, t_first, n_tiles, ctas, s); break;
        case 2: launch_tile_ua<U, 2>(a, t_first, n_tiles, ctas, s); break;
        default: launch_tile_ua<U, 3>(a, t_first, n_tiles, ctas, s); break;
    }
}

template <int U, int ACT>
void launch_eval_ua(const TileArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    const size_t smem = eval_tc_smem(U, a.dp);
    HCVA_CUDA(cudaFuncSetAttribute(k_eval_tc<U, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pdl_launch(k_eval_tc<U, ACT>, dim3(ctas), dim3(EvalShape<U>::threads), smem, s, a, t_first, n_tiles);
}

template <int U>
void launch_eval_u(const TileArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    switch (a.act) {
        case 0: launch_eval_ua<U, 0>(a, t_first, n_tiles, ctas, s); break;
        case 1: launch_eval_ua<U, 1>(a, t_first, n_tiles, ctas, s); break;
        case 2: launch_eval_ua<U, 2>(a, t_first, n_tiles, ctas, s); break;
        default: launch_eval_ua<U, 3>(a, t_first, n_tiles, ctas, s); break;
    }
}

int tc_eval_max_ctas(int sm_count) { return 2 * sm_count; }

template <int U, int ACT>
void launch_sgd_ua(const TileArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    const size_t smem = sgd_tc_smem(U, a.dp);
    HCVA_CUDA(cudaFuncSetAttribute(k_sgd_tc<U, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pdl_launch(k_sgd_tc<U, ACT>, dim3(ctas), dim3(SgdShape<U>::threads), smem, s, a, t_first, n_tiles);
}

template <int U>
void launch_sgd_u(const TileArgs& a, long t_first, long n_tiles, int ctas, cudaStream_t s) {
    switch (a.act) {
        case 0: launch_sgd_ua<U, 0>(a, t_first, n_tiles, ctas, s); break;
        case 1: launch_sgd_ua<U, 1>(a, t_first, n_tiles, ctas, s); break;
        case 2: launch_sgd_ua<U, 2>(a, t_first, n_tiles, ctas, s); break;
        default: launch_sgd_ua<U, 3>(a, t_first, n_tiles, ctas, s); break;
    }
}

int launch_tile_tc(int u, const TileArgs& a, int sm_count, cudaStream_t s) {
    if (a.b1 <= a.b0) throw contract_error("regression tile: empty row range");
    const long t_first = a.b0 / 128, n_tiles = (a.b1 - 1) / 128 - t_first + 1;
    if (a.xf32 && a.mode == 0) {  // two CTAs per SM (tc_two_cta shapes)
        const int ctas = static_cast<int>(std::min<long>(n_tiles, tc_eval_max_ctas(sm_count)));
        if (u == 16) launch_sgd_u<16>(a, t_first, n_tiles, ctas, s);
        else if (u == 32) launch_sgd_u<32>(a, t_first, n_tiles, ctas, s);
        else launch_sgd_u<64>(a, t_first, n_tiles, ctas, s);
        return ctas;
    }
    if (a.xf32) {
        const int ctas = static_cast<int>(std::min<long>(n_tiles, tc_eval_max_ctas(sm_count)));
        if (u == 16) launch_eval_u<16>(a, t_first, n_tiles, ctas, s);
        else if (u == 32) launch_eval_u<32>(a, t_first, n_tiles, ctas, s);
        else launch_eval_u<64>(a, t_first, n_tiles, ctas, s);
        return ctas;
    }
    const int ctas = static_cast<int>(std::min<long>(n_tiles, sm_count));
    if (u == 16) launch_tile_u<16>(a, t_first, n_tiles, ctas, s);
    else if (u == 32) launch_tile_u<32>(a, t_first, n_tiles, ctas, s);
    else launch_tile_u<64>(a, t_first, n_tiles, ctas, s);
    return ctas;
}

template <int U>
void launch_wgrad_u(const WgradArgs& a, int ctas, cudaStream_t s) {
    if (a.dp > 64) {
        HCVA_CUDA(cudaFuncSetAttribute(k_wgrad_tc<U, kWgXMax>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)wgrad_smem(kWgXMax)));
        k_wgrad_tc<U, kWgXMax><<<ctas, kWgThreads, wgrad_smem(kWgXMax), s>>>(a);
        return;
    }
    HCVA_CUDA(cudaFuncSetAttribute(k_wgrad_tc<U, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wgrad_smem(64)));
    k_wgrad_tc<U, 64><<<ctas, kWgThreads, wgrad_smem(64), s>>>(a);
}

// Refit Gram for U = 64 on the FP64 tensor cores (mma.sync m8n8k4 .f64, FP64
// accumulation): z = [h2, 1, y - mu, 0...] (72 columns, 9 blocks of 8); the
// 45 upper block pairs (bi <= bj) of z^T z are split over 8 warps, each warp
// walking the CTA's 64-row chunks in 4-row K steps (fixed order: chunk, then
// K step).
constexpr int kGdRows = 64, kGdLD = 76;  // chunk rows, padded row (doubles)
// The 45 upper-triangle 8x8 block pairs (bi <= bj) of the 72-column padded row, grouped
// by block row so that each warp reads few distinct blocks per K step (6, 7, 7, 7, 6,
// 5, 4 and 2 fragment loads for 6 x 7 + 3 MMAs): warp w owns pairs kGdPair[w][0..kGdCnt[w]).
__device__ constexpr int kGdCnt[8] = {6, 6, 6, 6, 6, 6, 6, 3};
__device__ constexpr int kGdPair[8][6][2] = {
    {{0, 0}, {0, 1}, {0, 2}, {0, 3}, {0, 4}, {0, 5}}, {{0, 6}, {0, 7}, {0, 8}, {1, 1}, {1, 2}, {1, 3}},
    {{1, 4}, {1, 5}, {1, 6}, {1, 7}, {1, 8}, {2, 2}}, {{2, 3}, {2, 4}, {2, 5}, {2, 6}, {2, 7}, {2, 8}},
    {{3, 3}, {3, 4}, {3, 5}, {3, 6}, {3, 7}, {3, 8}}, {{4, 4}, {4, 5}, {4, 6}, {4, 7}, {4, 8}, {5, 5}},
    {{5, 6}, {5, 7}, {5, 8}, {6, 6}, {6, 7}, {6, 8}}, {{7, 7}, {7, 8}, {8, 8}, {8, 8}, {8, 8}, {8, 8}}};

// One 64-row chunk for warp W: the fragments of the blocks its pairs touch are loaded
// once per K step (compile-time indices: they stay in registers), then its MMAs.
template <int W>
__device__ __forceinline__ void gram_chunk(const double* zs, int fr, int fc, double (&acc)[6][2]) {
    constexpr int cnt = kGdCnt[W];
    for (int k0 = 0; k0 < kGdRows; k0 += 4) {
        const double* zr = zs + (k0 + fr) * kGdLD + fc;
        double f[9];
#pragma unroll
        for (int b = 0; b < 9; ++b) {
            bool need = false;
#pragma unroll
            for (int q = 0; q < cnt; ++q) need = need || kGdPair[W][q][0] == b || kGdPair[W][q][1] == b;
            f[b] = need ? zr[8 * b] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < cnt; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[q][0]), "+d"(acc[q][1])
                         : "d"(f[kGdPair[W][q][0]]), "d"(f[kGdPair[W][q][1]]));
    }
}

// The kernel: 64-row chunks staged as FP64 in shared memory (row pitch 76 doubles:
// conflict-free fragment loads), the next chunk's rows prefetched into registers; one
// partial per CTA in k_gram_h2's packed layout.
__global__ void __launch_bounds__(256) k_gram_dmma(const float* __restrict__ H2, const double* __restrict__ y,
                                                    long R, const float* __restrict__ params, int P,
                                                    double* __restrict__ gpart) {
    constexpr int U = 64;
    __shared__ __align__(16) double zs[kGdRows * kGdLD];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const double mu = static_cast<double>(params[P - 1]);
    double acc[6][2];
#pragma unroll
    for (int q = 0; q < 6; ++q) acc[q][0] = acc[q][1] = 0.0;
    const int fr = lane & 3, fc = lane >> 2;  // fragment: row (K) and column (M / N) of this lane
    const long nch = (R + kGdRows - 1) / kGdRows;
    constexpr int kPer = kGdRows * (U / 4) / 256;  // float4 per thread per chunk
    float4 v[kPer];
    double yv = 0.0;
    auto fetch = [&](long ch) {
        const long base = ch * kGdRows;
        const int rows = static_cast<int>(min(static_cast<long>(kGdRows), R - base));
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int i = t + 256 * u, r = i / (U / 4), c4 = (i % (U / 4)) * 4;
            v[u] = r < rows ? __ldg(reinterpret_cast<const float4*>(H2 + (base + r) * U + c4))
                            : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
        if (t < kGdRows) yv = t < rows ? y[base + t] - mu : 0.0;
    };
    if (static_cast<long>(blockIdx.x) < nch) fetch(blockIdx.x);
    for (long ch = blockIdx.x; ch < nch; ch += gridDim.x) {
        const int rows = static_cast<int>(min(static_cast<long>(kGdRows), R - ch * kGdRows));
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int i = t + 256 * u, r = i / (U / 4), c4 = (i % (U / 4)) * 4;
            double* z = zs + r * kGdLD + c4;
            z[0] = v[u].x;
            z[1] = v[u].y;
            z[2] = v[u].z;
            z[3] = v[u].w;
        }
        if (t < kGdRows) {
            double* z = zs + t * kGdLD;
            z[U] = t < rows ? 1.0 : 0.0;
            z[U + 1] = yv;
            for (int c = U + 2; c < 72; ++c) z[c] = 0.0;
        }
        __syncthreads();
        if (ch + gridDim.x < nch) fetch(ch + gridDim.x);
        switch (warp) {
            case 0: gram_chunk<0>(zs, fr, fc, acc); break;
            case 1: gram_chunk<1>(zs, fr, fc, acc); break;
            case 2: gram_chunk<2>(zs, fr, fc, acc); break;
            case 3: gram_chunk<3>(zs, fr, fc, acc); break;
            case 4: gram_chunk<4>(zs, fr, fc, acc); break;
            case 5: gram_chunk<5>(zs, fr, fc, acc); break;
            case 6: gram_chunk<6>(zs, fr, fc, acc); break;
            default: gram_chunk<7>(zs, fr, fc, acc); break;
        }
    }
    // Packed output: (a, b) a <= b < m = U+1 -> upper-triangle index; rhs c = (c, U+1).
    constexpr int m = U + 1, tri = m * (m + 1) / 2;
    double* out = gpart + static_cast<size_t>(blockIdx.x) * (tri + m);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        if (q >= kGdCnt[warp]) continue;
        const int bi = kGdPair[warp][q][0], bj = kGdPair[warp][q][1];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int ra = 8 * bi + fc, cb = 8 * bj + 2 * fr + e;  // D[row = lane/4][col = 2 (lane%4) + e]
            if (ra < m && cb < m && ra <= cb) out[ra * m - ra * (ra - 1) / 2 + (cb - ra)] = acc[q][e];
            else if (ra < m && cb == m) out[tri + ra] = acc[q][e];
        }
    }
}

template <int U>
int launch_gram_u(const float* H2, const double* y, long R, const float* params, int P, double* gpart, int ctas,
                  cudaStream_t s) {
    k_gram_h2<U><<<ctas, GramShape<U>::threads, 0, s>>>(H2, y, R, params, P, gpart);
    return ctas;
}

int launch_gram_h2(int u, const float* H2, const double* y, long R, const float* params, int P, double* gpart,
                   int max_parts, int sm_count, cudaStream_t s) {
    const long chunks = (R + 63) / 64;
    const int ctas = static_cast<int>(std::max<long>(1, std::min<long>({chunks, 4L * sm_count, max_parts})));
    if (u == 16) return launch_gram_u<16>(H2, y, R, params, P, gpart, ctas, s);
    if (u == 32) return launch_gram_u<32>(H2, y, R, params, P, gpart, ctas, s);
    static const bool dmma = [] {
        const char* e = std::getenv("HCVA_GRAM_DMMA");
        return !(e && e[0] == '0');
    }();
    if (dmma) {
        k_gram_dmma<<<ctas, 256, 0, s>>>(H2, y, R, params, P, gpart);
        return ctas;
    }
    return launch_gram_u<64>(H2, y, R, params, P, gpart, ctas, s);
}

int tc_wgrad_max_ctas(int sm_count) { return 2 * sm_count; }  // 256 TMEM columns each

// Returns the number of weight-gradient partials written.
int launch_wgrad_tc(int u, WgradArgs a, int sm_count, cudaStream_t s) {
    const long chunks = (a.rows + kWgK - 1) / kWgK;
    static const int per_sm = [] {  // CTAs per SM (profiling override HCVA_WGRAD_SLOTS)
        const char* e = std::getenv("HCVA_WGRAD_SLOTS");
        const int v = e ? std::atoi(e) : 2;  // 2 measured best (partials vs overlap)
        return v < 1 ? 1 : (v > 2 ? 2 : v);
    }();
    const long slots = static_cast<long>(a.dp > 64 ? 1 : per_sm) * sm_count;  // resident CTAs
    const long per = std::max(1L, (chunks + slots - 1) / slots);
    a.rows_per_cta = static_cast<int>(per * kWgK);
    const int ctas = static_cast<int>((a.rows + a.rows_per_cta - 1) / a.rows_per_cta);
    if (u == 16) launch_wgrad_u<16>(a, ctas, s);
    else if (u == 32) launch_wgrad_u<32>(a, ctas, s);
    else launch_wgrad_u<64>(a, ctas, s);
    return ctas;
}

}  // namespace hcva

using namespace hcva;

extern "C" hcva_status hcva_diag_tc_gemm(hcva_ctx* ctx, int M, int N, int K, int variant, const float* A,
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
                                                      variant);
        check_launch(ctx);
        copy_out(ctx, D, dD.p, sizeof(float) * M * N);
    });
}

extern "C" hcva_status hcva_diag_tc_rate(hcva_ctx* ctx, int M, int N, int iters, double* tflops) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if ((M != 64 && M != 128) || N % 16 || N < 16 || N > 256) throw contract_error("tc rate: bad shape");
        DeviceBuf sink;
        sink.alloc(sizeof(float) * ctx->sm_count);
        const size_t smem = 2 * 128 * 8 * 4 * 2 + 64;
        cudaEvent_t e0, e1;
        HCVA_CUDA(cudaEventCreate(&e0));
        HCVA_CUDA(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            HCVA_CUDA(cudaEventRecord(e0, ctx->stream));
            k_tc_rate<<<ctx->sm_count, 128, smem, ctx->stream>>>(M, N, iters, sink.as<float>());
            HCVA_CUDA(cudaEventRecord(e1, ctx->stream));
            HCVA_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            HCVA_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0) best = std::min(best, ms);
        }
        check_launch(ctx);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *tflops = 2.0 * M * N * 8.0 * iters * ctx->sm_count / (best * 1e-3) / 1e12;
    });
}
