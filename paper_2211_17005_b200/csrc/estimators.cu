// estimators.cu -- the validation statistics of the engine as device
// reductions: the twin-MC L2 estimator and its relative RMSE with a
// delta-method standard error (reference validation.cpp:41-117), the Q/R
// split of the probe losses (planner.cpp:11-70), the nested-MC relative RMSE
// (validation.cpp:181-210) and the percentile bands of percentile_table
// (pipeline.cpp:41-47,138-156).
//
// Every estimator is a mean or a centred second moment of O(M*N) terms that
// already live on the GPU (labels, predictions, probe losses).  They are
// reduced where they are: one pass forms per-cluster sums, one CTA of 1024
// threads folds them in a fixed order (thread t takes entries t, t+1024, ...
// in sequence, then a fixed shuffle tree and a fixed tree over the 32 warp
// partials), so a result depends only on the inputs and never on the grid or
// on scheduling.  Centred moments are taken in a second pass around the
// first pass's mean, as the reference does.  The few scalar formulas on the
// final moments (square roots, the delta method) run on the host.
//
// Parity: these are statistics, summed in a different order from the
// reference's sequential loops, so they agree to rounding (1e-12 relative in
// tests/test_estimators.py), not bit for bit.
#include <cub/device/device_radix_sort.cuh>

#include <cmath>

#include "common.cuh"

namespace hcva {
namespace {

constexpr int kRedThreads = 1024;

// Fixed-order sum of `v` over the CTA; the result is valid in every thread.
template <int K>
__device__ void cta_sum(double (&v)[K], double* smem /* [32*K] */) {
#pragma unroll
    for (int q = 0; q < K; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < K; ++q) smem[q * 32 + warp] = v[q];
    __syncthreads();
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < K; ++q) {
        double x = lane < nw ? smem[q * 32 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        v[q] = x;
    }
}

__device__ __forceinline__ double twin_term(double phi, double x1, double x2) {
    return phi * phi - (x1 + x2) * phi + x1 * x2;
}

// Per-cluster sums of a_j = phi^2 - (xi1 + xi2) phi + xi1 xi2 and
// b_j = xi1 xi2 over clusters of `block` consecutive rows (one outer path and
// its replicas).  A warp per cluster for wide clusters (lanes stride the
// rows, fixed shuffle tree); a thread per cluster otherwise.
__global__ void k_twin_clusters(const double* __restrict__ pred, const double* __restrict__ t1,
                                const double* __restrict__ t2, size_t nb, int block, double* __restrict__ A,
                                double* __restrict__ B) {
    const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (block >= 32) {
        const size_t b = tid >> 5;
        const int lane = threadIdx.x & 31;
        if (b >= nb) return;
        double a = 0.0, s = 0.0;
        for (int j = lane; j < block; j += 32) {
            const size_t r = b * block + j;
            a += twin_term(pred[r], t1[r], t2[r]);
            s += t1[r] * t2[r];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            s += __shfl_xor_sync(0xffffffffu, s, o);
        }
        if (lane == 0) A[b] = a, B[b] = s;
    } else {
        if (tid >= nb) return;
        double a = 0.0, s = 0.0;
        for (int j = 0; j < block; ++j) {
            const size_t r = tid * block + j;
            a += twin_term(pred[r], t1[r], t2[r]);
            s += t1[r] * t2[r];
        }
        A[tid] = a, B[tid] = s;
    }
}

// One CTA: means of the row terms and the centred moments of the cluster
// means.  out = [mean a, mean b, S_aa, S_bb, S_ab] with S the sums over
// clusters of products of (cluster mean - overall mean).
__global__ void __launch_bounds__(kRedThreads) k_twin_moments(const double* __restrict__ A,
                                                               const double* __restrict__ B, size_t nb, int block,
                                                               double* __restrict__ out) {
    __shared__ double sm[32 * 3];
    double s[2] = {0.0, 0.0};
    for (size_t b = threadIdx.x; b < nb; b += blockDim.x) s[0] += A[b], s[1] += B[b];
    cta_sum(s, sm);
    const double rows = static_cast<double>(nb) * block;
    const double ma = s[0] / rows, mb = s[1] / rows;
    double c[3] = {0.0, 0.0, 0.0};
    for (size_t b = threadIdx.x; b < nb; b += blockDim.x) {
        const double da = A[b] / block - ma, db = B[b] / block - mb;
        c[0] += da * da, c[1] += db * db, c[2] += da * db;
    }
    cta_sum(c, sm);
    if (threadIdx.x == 0) out[0] = ma, out[1] = mb, out[2] = c[0], out[3] = c[1], out[4] = c[2];
}

// Q/R moments over segments of the probe pairs g[k] = (g1_k, g2_k): segment 0
// is every pair, segment s >= 1 the s-th batch of `bs` pairs.  One CTA per
// segment; out[s] = (pooled variance about the segment mean, covariance).
__global__ void __launch_bounds__(kRedThreads) k_qr_segments(const double2* __restrict__ g, size_t n, size_t bs,
                                                              double2* __restrict__ out) {
    __shared__ double sm[32 * 2];
    const size_t lo = blockIdx.x == 0 ? 0 : (blockIdx.x - 1) * bs;
    const size_t len = blockIdx.x == 0 ? n : bs;
    double s[1] = {0.0};
    for (size_t k = lo + threadIdx.x; k < lo + len; k += blockDim.x) s[0] += g[k].x + g[k].y;
    cta_sum(s, sm);
    const double mean = s[0] / (2.0 * len);
    double c[2] = {0.0, 0.0};
    for (size_t k = lo + threadIdx.x; k < lo + len; k += blockDim.x) {
        const double d1 = g[k].x - mean, d2 = g[k].y - mean;
        c[0] += d1 * d1 + d2 * d2;
        c[1] += d1 * d2;
    }
    cta_sum(c, sm);
    if (threadIdx.x == 0) out[blockIdx.x] = make_double2(c[0] / (2.0 * len), c[1] / len);
}

// Nested relative RMSE: squared relative errors over the nonzero benchmarks,
// their mean, and the sum of squares about it.  out = [used, mean, S].
__global__ void __launch_bounds__(kRedThreads) k_nested_rmse(const double* __restrict__ pred,
                                                              const double* __restrict__ nested, size_t n,
                                                              double* __restrict__ out) {
    __shared__ double sm[32 * 2];
    double s[2] = {0.0, 0.0};
    for (size_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double v = nested[j];
        if (v == 0.0) continue;
        const double e = (pred[j] - v) / v;
        s[0] += 1.0, s[1] += e * e;
    }
    cta_sum(s, sm);
    const double used = s[0];
    const double m = used > 0.0 ? s[1] / used : 0.0;
    double c[1] = {0.0};
    for (size_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double v = nested[j];
        if (v == 0.0) continue;
        const double e = (pred[j] - v) / v;
        c[0] += (e * e - m) * (e * e - m);
    }
    cta_sum(c, sm);
    if (threadIdx.x == 0) out[0] = used, out[1] = m, out[2] = c[0];
}

// Mean and the four interpolated percentiles of an ascending array
// (percentile_sorted, pipeline.cpp:41-47): out = [mean, p1, p2.5, p97.5, p99].
__global__ void __launch_bounds__(kRedThreads) k_bands(const double* __restrict__ v, size_t n,
                                                        double* __restrict__ out) {
    __shared__ double sm[32];
    double s[1] = {0.0};
    for (size_t j = threadIdx.x; j < n; j += blockDim.x) s[0] += v[j];
    cta_sum(s, sm);
    if (threadIdx.x < 4) {
        const double q[4] = {0.01, 0.025, 0.975, 0.99};
        const double pos = q[threadIdx.x] * (static_cast<double>(n) - 1.0);
        const size_t i = static_cast<size_t>(pos);
        const double f = pos - static_cast<double>(i);
        out[1 + threadIdx.x] = i + 1 < n ? v[i] * (1.0 - f) + v[i + 1] * f : v[i];
    }
    if (threadIdx.x == 0) out[0] = s[0] / static_cast<double>(n);
}

// Standard error of the mean of a short host list (the Q/R batch statistics).
double se_of_mean(const double* x, size_t n) {
    double m = 0.0;
    for (size_t i = 0; i < n; ++i) m += x[i];
    m /= static_cast<double>(n);
    double ss = 0.0;
    for (size_t i = 0; i < n; ++i) ss += (x[i] - m) * (x[i] - m);
    return std::sqrt(ss / static_cast<double>(n - 1) / static_cast<double>(n));
}

struct TwinMoments {
    double ma, mb, saa, sbb, sab;
    size_t clusters;
};

// Inputs may be host or device memory (cudaMemcpyDefault through UVA).
TwinMoments twin_moments(hcva_ctx* ctx, const double* pred, const double* t1, const double* t2, size_t n,
                         int block) {
    if (!pred || !t1 || !t2 || n == 0) throw contract_error("twin estimator: size mismatch or empty input");
    if (block <= 1 || n % static_cast<size_t>(block) != 0) block = 1;
    const size_t nb = n / block;
    DeviceBuf in, part, res;
    in.alloc(3 * n * 8);
    part.alloc(2 * nb * 8);
    res.alloc(5 * 8);
    double* d = in.as<double>();
    HCVA_CUDA(cudaMemcpyAsync(d, pred, n * 8, cudaMemcpyDefault, ctx->stream));
    HCVA_CUDA(cudaMemcpyAsync(d + n, t1, n * 8, cudaMemcpyDefault, ctx->stream));
    HCVA_CUDA(cudaMemcpyAsync(d + 2 * n, t2, n * 8, cudaMemcpyDefault, ctx->stream));
    const size_t threads = block >= 32 ? nb * 32 : nb;
    k_twin_clusters<<<grid1(threads, 256), 256, 0, ctx->stream>>>(d, d + n, d + 2 * n, nb, block,
                                                                   part.as<double>(), part.as<double>() + nb);
    k_twin_moments<<<1, kRedThreads, 0, ctx->stream>>>(part.as<double>(), part.as<double>() + nb, nb, block,
                                                        res.as<double>());
    ctx->launches += 2;
    check_launch(ctx);
    double h[5];
    copy_out(ctx, h, res.p, sizeof h);
    return {h[0], h[1], h[2], h[3], h[4], nb};
}

}  // namespace

// estimate_qr on device pairs g [n][2]; out = Q, R, total, n, Q s.e., R s.e.
void estimate_qr_device(hcva_ctx* ctx, const double* g, size_t n, double* out) {
    if (n < 2) throw numeric_error("estimate_qr: need at least two outer paths");
    const size_t nb = std::min<size_t>(20, n / 2);
    const size_t segs = nb >= 2 ? nb + 1 : 1;
    DeviceBuf res;
    res.alloc(segs * 16);
    k_qr_segments<<<static_cast<unsigned>(segs), kRedThreads, 0, ctx->stream>>>(
        reinterpret_cast<const double2*>(g), n, nb >= 2 ? n / nb : 0, res.as<double2>());
    ctx->launches++;
    check_launch(ctx);
    std::vector<double> h(2 * segs);
    copy_out(ctx, h.data(), res.p, h.size() * 8);
    const double total = h[0], r = h[1];
    out[0] = total - r;
    out[1] = r;
    out[2] = total;
    out[3] = static_cast<double>(n);
    out[4] = out[5] = 0.0;
    if (segs > 1) {
        std::vector<double> q(nb), rr(nb);
        for (size_t b = 0; b < nb; ++b) q[b] = h[2 * (b + 1)] - h[2 * (b + 1) + 1], rr[b] = h[2 * (b + 1) + 1];
        out[4] = se_of_mean(q.data(), nb);
        out[5] = se_of_mean(rr.data(), nb);
    }
}

// Mean and percentile bands of n device values (sorted on the device).
void percentile_bands(hcva_ctx* ctx, const double* dev_values, size_t n, double* out) {
    if (n == 0) throw contract_error("percentile_table: no predictions");
    DeviceBuf sorted, tmp, res;
    sorted.alloc(n * 8);
    res.alloc(5 * 8);
    size_t tmp_bytes = 0;
    HCVA_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, dev_values, sorted.as<double>(),
                                             static_cast<int>(n), 0, 64, ctx->stream));
    tmp.alloc(std::max<size_t>(tmp_bytes, 16));
    HCVA_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, dev_values, sorted.as<double>(),
                                             static_cast<int>(n), 0, 64, ctx->stream));
    k_bands<<<1, kRedThreads, 0, ctx->stream>>>(sorted.as<double>(), n, res.as<double>());
    ctx->launches++;
    check_launch(ctx);
    copy_out(ctx, out, res.p, 5 * 8);
}

}  // namespace hcva

using namespace hcva;

extern "C" {

// twin_l2_error (validation.cpp:41-56): mean of a_j and its standard error
// clustered over blocks of `block` rows.
hcva_status hcva_twin_l2_error(hcva_ctx* ctx, const double* pred, const double* twin1, const double* twin2,
                               size_t n, int block, double* value, double* std_error) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const TwinMoments t = twin_moments(ctx, pred, twin1, twin2, n, block);
        *value = t.ma;
        if (std_error) {
            const double k = static_cast<double>(t.clusters);
            *std_error = t.clusters < 2 ? 0.0 : std::sqrt(t.saa / (k - 1.0) / k);
        }
    });
}

// twin_relative_rmse (validation.cpp:58-69): sqrt(E[a]^+ / E[xi1 xi2]).
hcva_status hcva_twin_relative_rmse(hcva_ctx* ctx, const double* pred, const double* twin1, const double* twin2,
                                    size_t n, double* out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const TwinMoments t = twin_moments(ctx, pred, twin1, twin2, n, 1);
        if (t.mb <= 0.0) throw numeric_error("twin_relative_rmse: E[xi1 xi2] <= 0 (degenerate portfolio)");
        *out = std::sqrt(std::max(t.ma, 0.0) / t.mb);
    });
}

// twin_relative_rmse_std_error (validation.cpp:71-117): delta method for
// sqrt(A/B) with A, B the means above and their clustered (co)variances:
// se = sqrt(A/B)/2 * sqrt(Var A/A^2 + Var B/B^2 - 2 Cov(A,B)/(A B)).
hcva_status hcva_twin_relative_rmse_se(hcva_ctx* ctx, const double* pred, const double* twin1,
                                       const double* twin2, size_t n, int block, double* out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const TwinMoments t = twin_moments(ctx, pred, twin1, twin2, n, block);
        *out = 0.0;
        if (t.ma <= 0.0 || t.mb <= 0.0 || t.clusters < 2) return;
        const double k = static_cast<double>(t.clusters), norm = k * (k - 1.0);
        const double var_a = t.saa / norm, var_b = t.sbb / norm, cov = t.sab / norm;
        const double rel = var_a / (t.ma * t.ma) + var_b / (t.mb * t.mb) - 2.0 * cov / (t.ma * t.mb);
        *out = 0.5 * std::sqrt(t.ma / t.mb) * std::sqrt(std::max(rel, 0.0));
    });
}

// estimate_qr (planner.cpp:11-70) on host or device loss pairs.
hcva_status hcva_estimate_qr(hcva_ctx* ctx, const double* g1, const double* g2, size_t n, double* out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (!g1 || !g2) throw contract_error("estimate_qr: pair length mismatch");
        if (n < 2) throw numeric_error("estimate_qr: need at least two outer paths");
        DeviceBuf g;
        g.alloc(n * 16);
        HCVA_CUDA(cudaMemcpy2DAsync(g.p, 16, g1, 8, 8, n, cudaMemcpyDefault, ctx->stream));
        HCVA_CUDA(cudaMemcpy2DAsync(g.as<char>() + 8, 16, g2, 8, 8, n, cudaMemcpyDefault, ctx->stream));
        estimate_qr_device(ctx, g.as<double>(), n, out);
    });
}

// nested_relative_rmse (validation.cpp:181-210): out = value, std_error,
// excluded_zero, used.
hcva_status hcva_nested_relative_rmse(hcva_ctx* ctx, const double* pred, const double* nested, size_t n,
                                      double* out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (!pred || !nested || n == 0) throw contract_error("nested_relative_rmse: size mismatch or empty input");
        DeviceBuf in, res;
        in.alloc(2 * n * 8);
        res.alloc(3 * 8);
        HCVA_CUDA(cudaMemcpyAsync(in.p, pred, n * 8, cudaMemcpyDefault, ctx->stream));
        HCVA_CUDA(cudaMemcpyAsync(in.as<double>() + n, nested, n * 8, cudaMemcpyDefault, ctx->stream));
        k_nested_rmse<<<1, kRedThreads, 0, ctx->stream>>>(in.as<double>(), in.as<double>() + n, n,
                                                           res.as<double>());
        ctx->launches++;
        check_launch(ctx);
        double h[3];
        copy_out(ctx, h, res.p, sizeof h);
        const double used = h[0], m = h[1];
        if (used == 0.0) throw numeric_error("nested_relative_rmse: all benchmarks are zero");
        out[0] = std::sqrt(m);
        out[1] = used > 1.0 && m > 0.0 ? std::sqrt(h[2] / (used - 1.0) / used) / (2.0 * out[0]) : 0.0;
        out[2] = static_cast<double>(n) - used;
        out[3] = used;
    });
}

}  // extern "C"
