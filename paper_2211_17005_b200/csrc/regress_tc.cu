// regress_tc.cu -- K5 on the 5th-generation tensor cores: the SGD tile of the
// backward regression (regressor.cpp:115-158) as tcgen05 kind::tf32 GEMMs
// (3xTF32, FP32 accumulation in TMEM) for the paper's network shape: two
// hidden layers of width U in {16, 32, 64}, input dimension d <= 64.
//
// One CTA = one 128-row tile of a batch, 128 threads (thread r owns row r =
// TMEM lane r).  Thread 0 issues the MMAs; completion is signalled through an
// mbarrier by tcgen05.commit; epilogues read the accumulators with
// tcgen05.ld and write the next operands (split hi/lo) into shared memory.
//   F0   D0  = X  W0^T      (M=128, N=U,  K=dp)   -> H1 = act(D0 + b0)
//   F1   D1  = H1 W1^T      (M=128, N=U,  K=U)    -> H2, f, residual, G2
//   B1   DgW1 = G2^T H1     (M=64,  N=U,  K=128)  weight gradient, layer 1
//        Dbp = G2 W1        (M=128, N=U,  K=U)    -> G1 = Dbp * act'(H1)
//   B0   DgW0 = G1^T X      (M=64,  N=dp, K=128)  weight gradient, layer 0
// The output layer, biases and mu reduce over rows in shared memory.  Two
// 64 KB operand buffers are reused across the phases (X -> G2 -> X,
// H1 -> G1), so the CTA fits in 194 KB of shared memory.
#include <cmath>

#include "common.cuh"
#include "tc.cuh"

namespace hcva {

struct TcArgs {
    int d, dp, act, P;
    int off0, off1, off2;  // W0, W1, w2 offsets in the flat parameter vector
    const float* X;
    const double* y;
    long row0, row_end;
    const float* params;
    int head;
    double nb;
    float* gpart;   // [tiles][P]
    double* lpart;  // [tiles]
};

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

constexpr uint32_t kTileBytes = 128 * 64 * 4;  // one 128 x 64 FP32 core tile
constexpr int kTcThreads = 128;

__host__ __device__ constexpr size_t tc_smem_bytes(int U) {
    return 4 * static_cast<size_t>(kTileBytes) + 4 * static_cast<size_t>(U) * 64 * 4 + 512 * 4 + 64 * 8 + 64;
}

template <int U>
__global__ void __launch_bounds__(kTcThreads, 1) k_sgd_tc(TcArgs a) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* bufA = sm;                            // hi, lo at +kTileBytes
    uint8_t* bufB = sm + 2 * kTileBytes;
    uint8_t* w0 = sm + 4 * kTileBytes;             // U x 64 core tile, lo at +wbytes
    constexpr uint32_t wbytes = U * 64 * 4;
    uint8_t* w1 = w0 + 2 * wbytes;
    float* vec = reinterpret_cast<float*>(w1 + 2 * wbytes);  // b0[64] b1[64] w2[64] misc[64]
    float* wsum = vec + 256;                                 // [4][64] per-warp output-layer sums
    double* red = reinterpret_cast<double*>(vec + 512);      // [64]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(red + 64);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);

    const int r = threadIdx.x, warp = r >> 5;
    const int d = a.d, dp = a.dp;
    const long base = a.row0 + static_cast<long>(blockIdx.x) * 128;
    const int rows = static_cast<int>(min(128L, a.row_end - base));
    const float* P = a.params;

    if (r == 0) tc::mbar_init(mbar, 1);
    if (warp == 0) tc::tmem_alloc(tbase, 256);
    // Weights (hi/lo core tiles), vectors.
    for (int i = r; i < U * 64; i += kTcThreads) {
        const int o = i / 64, j = i % 64;
        tc::put_split(w0, wbytes, o, j, U, (j < d) ? P[a.off0 + o * d + j] : 0.0f);
    }
    for (int i = r; i < U * U; i += kTcThreads) {
        const int o = i / U, j = i % U;
        tc::put_split(w1, wbytes, o, j, U, P[a.off1 + o * U + j]);
    }
    if (r < 64) {
        vec[r] = (r < U) ? P[a.off0 + U * d + r] : 0.0f;        // b0
        vec[64 + r] = (r < U) ? P[a.off1 + U * U + r] : 0.0f;   // b1
        vec[128 + r] = (r < U) ? P[a.off2 + r] : 0.0f;          // w2
    }
    if (r == 0) {
        vec[192] = P[a.off2 + U];  // b2
        vec[193] = P[a.P - 1];     // mu
    }
    auto load_x = [&]() {
        for (int i = r; i < 128 * dp; i += kTcThreads) {
            const int rr = i / dp, j = i % dp;
            const float v = (rr < rows && j < d) ? a.X[(base + rr) * d + j] : 0.0f;
            tc::put_split(bufA, kTileBytes, rr, j, 128, v);
        }
    };
    load_x();
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    uint32_t phase = 0;

    // ---- F0: D0 = X W0^T
    if (r == 0) {
        tc::gemm3(tm + 0, tc::kmajor(bufA, kTileBytes, 128), tc::kmajor(w0, wbytes, U), dp,
                  tc::idesc_tf32(128, U, 0, 0), 0);
        tc::commit(mbar);
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    // ---- epilogue F0: H1 = act(D0 + b0) -> bufB
#pragma unroll
    for (int c0 = 0; c0 < U; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + c0, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) tc::put_split(bufB, kTileBytes, r, c0 + q, 128, tc_act(a.act, v[q] + vec[c0 + q]));
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    // ---- F1: D1 = H1 W1^T
    if (r == 0) {
        tc::gemm3(tm + 64, tc::kmajor(bufB, kTileBytes, 128), tc::kmajor(w1, wbytes, U), U,
                  tc::idesc_tf32(128, U, 0, 0), 0);
        tc::commit(mbar);
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    // ---- epilogue F1: H2, f, residual, output-layer and mu gradients, G2 -> bufA
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
    double resid2 = 0.0, dmu = 0.0;
    float dd = 0.0f;
    if (r < rows) {
        const float pred = ((a.head && f < 0.0f) ? 0.0f : f) + mu;
        const double res = static_cast<double>(pred) - a.y[base + r];
        resid2 = res * res;
        dmu = 2.0 * res / a.nb;
        dd = static_cast<float>(dmu);
        if (a.head && !(f > 0.0f)) dd = 0.0f;
    }
    float* gout = a.gpart + static_cast<size_t>(blockIdx.x) * a.P;
    {
        // Row reductions: loss, mu, output bias, output weights (warp shuffles + smem).
        double l = resid2, m = dmu;
        float g2b = dd;
        for (int o = 16; o > 0; o >>= 1) {
            l += __shfl_xor_sync(0xffffffffu, l, o);
            m += __shfl_xor_sync(0xffffffffu, m, o);
            g2b += __shfl_xor_sync(0xffffffffu, g2b, o);
        }
        if ((r & 31) == 0) {
            red[warp] = l;
            red[4 + warp] = m;
            red[8 + warp] = g2b;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            float s = dd * h2[j];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if ((r & 31) == 0) wsum[warp * U + j] = s;
        }
        __syncthreads();
        if (r == 0) {
            a.lpart[blockIdx.x] = red[0] + red[1] + red[2] + red[3];
            gout[a.P - 1] = static_cast<float>(red[4] + red[5] + red[6] + red[7]);
            gout[a.off2 + U] = static_cast<float>(red[8] + red[9] + red[10] + red[11]);
        }
        if (r < U) gout[a.off2 + r] = wsum[r] + wsum[U + r] + wsum[2 * U + r] + wsum[3 * U + r];
    }
    // G2 = dd w2 act'(H2); columns U..63 zero (M=64 padding of the weight-gradient GEMM).
#pragma unroll
    for (int j = 0; j < 64; ++j) {
        const float g = (j < U) ? dd * vec[128 + j] * tc_der(a.act, h2[j < U ? j : 0]) : 0.0f;
        tc::put_split(bufA, kTileBytes, r, j, 128, g);
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    // ---- B1: DgW1 = G2^T H1 (M=64), Dbp = G2 W1
    if (r == 0) {
        tc::gemm3(tm + 192, tc::mnmajor(bufA, kTileBytes, 128), tc::mnmajor(bufB, kTileBytes, 128), 128,
                  tc::idesc_tf32(64, U, 1, 1), 0);
        tc::gemm3(tm + 128, tc::kmajor(bufA, kTileBytes, 128), tc::mnmajor(w1, wbytes, U), U,
                  tc::idesc_tf32(128, U, 0, 1), 0);
        tc::commit(mbar);
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    // ---- epilogue B1: bias gradient of layer 1 (column sums of G2), G1 = Dbp act'(H1) -> bufB
    if (r < U) {
        float s = 0.0f;
        for (int rr = 0; rr < rows; ++rr) s += tc::get_split(bufA, kTileBytes, rr, r, 128);
        gout[a.off1 + U * U + r] = s;
    }
#pragma unroll
    for (int c0 = 0; c0 < U; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + 128 + c0, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float h1 = tc::get_split(bufB, kTileBytes, r, c0 + q, 128);
            tc::put_split(bufB, kTileBytes, r, c0 + q, 128, (r < rows) ? v[q] * tc_der(a.act, h1) : 0.0f);
        }
    }
    for (int j = U; j < 64; ++j) tc::put_split(bufB, kTileBytes, r, j, 128, 0.0f);
    // Weight gradient of layer 1 out of TMEM (M=64 layout: rows 16w+t in lanes 32w+t, t < 16).
#pragma unroll
    for (int c0 = 0; c0 < U; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + 192 + c0, v);
        const int o = warp * 16 + (r & 31);
        if ((r & 31) < 16 && o < U)
#pragma unroll
            for (int q = 0; q < 16; ++q) gout[a.off1 + o * U + c0 + q] = v[q];
    }
    __syncthreads();  // G2 column sums done before X overwrites bufA
    load_x();
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    // ---- B0: DgW0 = G1^T X (M=64, N=dp)
    if (r == 0) {
        tc::gemm3(tm + 0, tc::mnmajor(bufB, kTileBytes, 128), tc::mnmajor(bufA, kTileBytes, 128), 128,
                  tc::idesc_tf32(64, dp, 1, 1), 0);
        tc::commit(mbar);
    }
    if (r < U) {
        float s = 0.0f;
        for (int rr = 0; rr < rows; ++rr) s += tc::get_split(bufB, kTileBytes, rr, r, 128);
        gout[a.off0 + U * d + r] = s;
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1;
    tc::fence_after_sync();
    for (int c0 = 0; c0 < dp; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tm + lane_base + c0, v);
        const int o = warp * 16 + (r & 31);
        if ((r & 31) < 16 && o < U)
#pragma unroll
            for (int q = 0; q < 16; ++q)
                if (c0 + q < d) gout[a.off0 + o * d + c0 + q] = v[q];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tm, 256);
}

// Diagnostic GEMM: D (M x N) = A (M x K) B (N x K)^T with the operands laid out
// K-major or MN-major in core tiles (test hook for the descriptor conventions).
__global__ void k_tc_gemm_diag(int M, int N, int K, int amn, int bmn, const float* A, const float* B, float* D) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int R_A = amn ? K : M, C_A = amn ? M : K, R_B = bmn ? K : N, C_B = bmn ? N : K;
    const uint32_t abytes = R_A * C_A * 4, bbytes = R_B * C_B * 4;
    uint8_t* ta = sm;
    uint8_t* tb = sm + 2 * abytes;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(tb + 2 * bbytes);
    uint32_t* tbase = reinterpret_cast<uint32_t*>(mbar + 1);
    const int t = threadIdx.x, warp = t >> 5;
    if (t == 0) tc::mbar_init(mbar, 1);
    if (warp == 0) tc::tmem_alloc(tbase, 256);
    for (int i = t; i < M * K; i += blockDim.x) {
        const int m = i / K, k = i % K;
        if (amn) tc::put_split(ta, abytes, k, m, R_A, A[i]); else tc::put_split(ta, abytes, m, k, R_A, A[i]);
    }
    for (int i = t; i < N * K; i += blockDim.x) {
        const int n = i / K, k = i % K;
        if (bmn) tc::put_split(tb, bbytes, k, n, R_B, B[i]); else tc::put_split(tb, bbytes, n, k, R_B, B[i]);
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = *tbase;
    if (t == 0) {
        const tc::Operand oa = amn ? tc::mnmajor(ta, abytes, R_A) : tc::kmajor(ta, abytes, R_A);
        const tc::Operand ob = bmn ? tc::mnmajor(tb, bbytes, R_B) : tc::kmajor(tb, bbytes, R_B);
        tc::gemm3(tm, oa, ob, K, tc::idesc_tf32(M, N, amn, bmn), 0);
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

bool tc_eligible(int d, int h, int u) {
    if (const char* e = std::getenv("HCVA_REGRESS_SIMT"))
        if (std::atoi(e)) return false;
    return h == 2 && (u == 16 || u == 32 || u == 64) && d >= 1 && d <= 64;
}

void launch_sgd_tc(int d, int u, int act, int P, int off0, int off1, int off2, const float* X, const double* y,
                   long row0, long row_end, const float* params, int head, double nb, float* gpart, double* lpart,
                   cudaStream_t s) {
    TcArgs a{};
    a.d = d;
    a.dp = ((d + 15) / 16) * 16;  // K multiple of 8, TMEM loads in 16-column groups
    a.act = act;
    a.P = P;
    a.off0 = off0;
    a.off1 = off1;
    a.off2 = off2;
    a.X = X;
    a.y = y;
    a.row0 = row0;
    a.row_end = row_end;
    a.params = params;
    a.head = head;
    a.nb = nb;
    a.gpart = gpart;
    a.lpart = lpart;
    const int tiles = static_cast<int>((row_end - row0 + 127) / 128);
    const size_t smem = tc_smem_bytes(u);
    switch (u) {
        case 16:
            HCVA_CUDA(cudaFuncSetAttribute(k_sgd_tc<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_sgd_tc<16><<<tiles, kTcThreads, smem, s>>>(a);
            break;
        case 32:
            HCVA_CUDA(cudaFuncSetAttribute(k_sgd_tc<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_sgd_tc<32><<<tiles, kTcThreads, smem, s>>>(a);
            break;
        default:
            HCVA_CUDA(cudaFuncSetAttribute(k_sgd_tc<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_sgd_tc<64><<<tiles, kTcThreads, smem, s>>>(a);
            break;
    }
}

}  // namespace hcva

using namespace hcva;

extern "C" hcva_status hcva_diag_tc_gemm(hcva_ctx* ctx, int M, int N, int K, int a_mn_major, int b_mn_major,
                                         const float* A, const float* B, float* D) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if ((M != 64 && M != 128) || N % 16 || N > 128 || K % 8 || K > 128)
            throw contract_error("diag gemm: M in {64,128}, N % 16 == 0 <= 128, K % 8 == 0 <= 128");
        DeviceBuf dA, dB, dD;
        stage(dA, std::vector<float>(A, A + M * K));
        stage(dB, std::vector<float>(B, B + N * K));
        dD.alloc(sizeof(float) * M * N);
        const size_t smem = 2 * 4 * (static_cast<size_t>(M) * K + static_cast<size_t>(N) * K) + 64;
        HCVA_CUDA(cudaFuncSetAttribute(k_tc_gemm_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_tc_gemm_diag<<<1, 128, smem, ctx->stream>>>(M, N, K, a_mn_major, b_mn_major, dA.as<float>(), dB.as<float>(),
                                                      dD.as<float>());
        check_launch(ctx);
        copy_out(ctx, D, dD.p, sizeof(float) * M * N);
    });
}
