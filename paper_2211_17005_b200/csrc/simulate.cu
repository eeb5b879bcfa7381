// simulate.cu -- the Y / MtM / X engine on sm_100a and its C ABI.
//
// Kernels (see DESIGN.md for the roofline of each):
//   k_draws        K0  raw stream draws (RandomStream::next_* on the device)
//   k_market       K1  Euler diffusion of rates / log-FX / CIR (market.cpp:161-310)
//   k_mtm_linear   K2  closed-form swap MtM cube, coefficient form (portfolio.cpp:58-147)
//   k_mtm_direct   K2' per-swap MtM in the reference's exact summation order
//   k_defaults     K3  hierarchical over-simulation of X (defaults.cpp:20-45)
//   k_labels_all   K4  defaults labels for every step in one pass (labels.cpp:21-48)
//   k_intensity_*  K4' intensity labels (labels.cpp:50-88)
//   k_features     K4" feature rows of one step (labels.cpp:142-167)
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <fstream>
#include <memory>

#include "common.cuh"
#include "rng.cuh"
#include "normal.cuh"

namespace hcva {

// Non-contracting FP64 helpers: the reference is compiled without FMA
// (x86-64, no -march), so the diffusion recursion uses explicitly rounded
// adds and multiplies to stay bit-faithful to it.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// ------------------------------------------------------------------ K0
__global__ void k_draws(uint64_t key, uint64_t start, size_t count, int kind, void* out) {
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (t >= count) return;
    const uint64_t x = draw_u64(key, start + t);
    if (kind == 0) {
        static_cast<uint64_t*>(out)[t] = x;
        return;
    }
    const double u = u64_to_uniform(x);
    double v = u;
    if (kind == 2) v = normal_from_uniform(u);
    if (kind == 3) v = -log(u);
    static_cast<double*>(out)[t] = v;
}

// Global path index of local path k in an interleaved shard: blocks of `blk`
// consecutive global paths every `stride` (blk == 0: identity).  Rank g of G
// owning slice g of every regression batch of P_B paths uses blk = P_B / G,
// stride = P_B and path_offset = g * P_B / G.
__host__ __device__ __forceinline__ uint64_t shard_path(int k, int blk, int stride) {
    return blk ? static_cast<uint64_t>(k / blk) * static_cast<uint64_t>(stride) + static_cast<uint64_t>(k % blk)
               : static_cast<uint64_t>(k);
}

// ------------------------------------------------------------------ K1
struct MarketArgs {
    int E, Cn, D, substeps, n_store, M, T, nnz;
    int mode;    // profiling probe: bit 0 skips normal generation, bit 1 skips the recursion
    int W_econ;  // economy-thread slots per path (E rounded up to whole warps)
    int qcap;    // per-warp tail-queue entries: 64 x the generator iterations of a chunk
    int paths_per_group;
    int shard_blk, shard_stride;  // interleaved shard map (0: identity), see shard_path
    uint64_t local_offset;
    double h, sqh;
    uint64_t key0;               // key of group 0 when group_keys == nullptr
    const uint64_t* group_keys;  // [groups] or nullptr
    const double* init_state;    // [groups][D]
    const FactorCoef* coef;      // [D]
    const int* chol_row;         // [D+1]
    const int* chol_col;         // [nnz]
    const double* chol_val;      // [nnz]
    double *rates, *fx, *intens, *hazard, *disc;
};

// K1: Euler diffusion of the exogenous factors Y (market.cpp:161-310).
//
// CTA = P paths x (threads per path).  The fine grid is processed in chunks of
// T substeps.  Per chunk, every thread first generates Philox blocks of its
// path (the chunk's P*T*D normals are counter-addressable, draw j = (substep,
// factor) of split(k), rng.cpp:57-67) into a double-buffered shared-memory
// tile; after one __syncthreads each thread advances the factors it owns for
// the T substeps with its state in registers:
//   economy thread e < E : r_e, log chi_e (e > 0) and a private copy of r_0
//                          (log-FX reads the pre-step r_0 and r_e,
//                          market.cpp:211-223); thread 0 also carries -ln beta;
//   credit thread        : two CIR intensities and their cumulative hazards.
// Every update is rounded as the reference rounds it (no FMA contraction).
// The correlated increment z = L zraw reads the chunk tile through the CSR of
// the Cholesky factor (exact zeros skipped).  Stores at pricing steps are
// coalesced over the path index.
// HCVA_K1_FMA (default on): the recursion's multiply-adds contract to FMAs.
// The factors then differ from the reference's separately rounded products by
// ~1 ulp per substep (market parity is 1e-11 relative); a default step could
// only flip for a threshold within ~1e-15 of a cumulative hazard, and the
// full C2 comparison (tests/test_gpu_simulation.py) counts 0 mismatches.
#ifndef HCVA_K1_FMA
#define HCVA_K1_FMA 1
#endif
__device__ __forceinline__ double madd(double a, double b, double c) {
#if HCVA_K1_FMA
    return fma(a, b, c);
#else
    return dadd(dmul(a, b), c);
#endif
}

__device__ __forceinline__ double vasicek_step(double r, const FactorCoef& k, double h, double z) {
    // r + (a(b - r) - q) h + (sigma sqrt h) z     (market.cpp:121-124)
#if HCVA_K1_FMA
    return fma(k.c3, z, fma(fma(k.c0, dsub(k.c1, r), -k.c2), h, r));
#else
    return dadd(dadd(r, dmul(dsub(dmul(k.c0, dsub(k.c1, r)), k.c2), h)), dmul(k.c3, z));
#endif
}

constexpr int kMaxGenIters = 16;  // generator iterations per chunk: two tail bits each in a 32-bit mask
// Acklam's branch points 0.02425 and 0.97575 on the top 32 bits of a draw.
constexpr uint32_t kTailLo32 = static_cast<uint32_t>(0.02425 * 4294967296.0);
constexpr uint32_t kTailHi32 = static_cast<uint32_t>((1.0 - 0.02425) * 4294967296.0);

template <int P>
#ifndef HCVA_K1_MAXNREG
#define HCVA_K1_MAXNREG 128  // <= 128 keeps 512-thread CTAs launchable (80: 3 CTAs/SM measured slower)
#endif
__global__ void __maxnreg__(HCVA_K1_MAXNREG) k_market(MarketArgs a) {
    extern __shared__ double smem[];
    const int E = a.E, Cn = a.Cn, D = a.D, T = a.T;
    const int NT = blockDim.x, NW = NT / 32;
    FactorCoef* coef = reinterpret_cast<FactorCoef*>(smem);          // [D] (8 doubles each)
    double* chol_val = smem + 8 * D;
    int* chol_col = reinterpret_cast<int*>(chol_val + a.nnz);
    int* chol_row = chol_col + a.nnz;
    // Philox round keys of the CTA's paths, [10][P]: key + r W (rng.cpp:33-37), one shared
    // load per round instead of a 64-bit add in every generator call
    uint64_t* ksched = reinterpret_cast<uint64_t*>(smem + 8 * D + a.nnz + (a.nnz + D + 2) / 2);
    int* qs_all = reinterpret_cast<int*>(ksched + 10 * P);            // [NW][qcap] tail slots
    double* zs = reinterpret_cast<double*>(ksched + 10 * P) + (NW * a.qcap + 1) / 2;  // [2][T*D][P]

    for (int t = threadIdx.x; t < D; t += NT) coef[t] = a.coef[t];
    for (int t = threadIdx.x; t < a.nnz; t += NT) {
        chol_val[t] = a.chol_val[t];
        chol_col[t] = a.chol_col[t];
    }
    for (int t = threadIdx.x; t <= D; t += NT) chol_row[t] = a.chol_row[t];

    const int p = threadIdx.x % P, w = threadIdx.x / P, TPP = NT / P;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int* qs = qs_all + wid * a.qcap;
    const int M = a.M;
    const int kloc = static_cast<int>(blockIdx.x) * P + p;
    const bool valid = kloc < M;
    const int kk = valid ? kloc : M - 1;
    const int grp = kk / a.paths_per_group;
    const uint64_t within = shard_path(kk - grp * a.paths_per_group, a.shard_blk, a.shard_stride) + a.local_offset;
    const uint64_t pkey = split_key(a.group_keys ? a.group_keys[grp] : a.key0, within);

    // Roles.  Economy threads w < We (We = E rounded up so warps are role-uniform);
    // credit threads own names c0 = 2(w - We), c1 = c0 + 1.
    const int We = a.W_econ;
    const bool econ = w < We;
    const bool econ_real = w < E;
    const int c0 = 2 * (w - We), c1 = c0 + 1;
    const bool cred = !econ && c0 < Cn;
    const bool has_c1 = cred && c1 < Cn;
    const int e = econ_real ? w : 0;
    const int fr = e, fx = (e > 0) ? E + e - 1 : 0;         // own rate / log-FX factor
    const int fg0 = cred ? 2 * E - 1 + c0 : 0, fg1 = has_c1 ? 2 * E - 1 + c1 : fg0;
    const double* init = a.init_state + static_cast<size_t>(grp) * D;
    // Registers: economy (s0 = r_e, s1 = r_0 copy, s2 = log chi_e, s3 = -ln beta);
    //            credit  (s0, s1 = intensities c0, c1; s2, s3 = their hazards).
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (econ) {
        s0 = init[fr];
        s1 = init[0];
        s2 = init[fx];
    } else if (cred) {
        s0 = init[fg0];
        s1 = init[fg1];
    }
    auto store = [&](int i) {
        if (!valid) return;
        if (econ_real) {
            a.rates[(static_cast<size_t>(i) * E + e) * M + kloc] = s0;
            if (e > 0) a.fx[(static_cast<size_t>(i) * (E - 1) + e - 1) * M + kloc] = exp(s2);
            else a.disc[static_cast<size_t>(i) * M + kloc] = exp(-s3);
        } else if (cred) {
            a.intens[(static_cast<size_t>(i) * Cn + c0) * M + kloc] = s0;
            a.hazard[(static_cast<size_t>(i) * Cn + c0) * M + kloc] = s2;
            if (has_c1) {
                a.intens[(static_cast<size_t>(i) * Cn + c1) * M + kloc] = s1;
                a.hazard[(static_cast<size_t>(i) * Cn + c1) * M + kloc] = s3;
            }
        }
    };
    store(0);
    if (w == 0) {
        uint64_t k = pkey;
#pragma unroll
        for (int rr = 0; rr < 10; ++rr, k += kPhiloxW) ksched[rr * P + p] = k;
    }
    const uint64_t* ks = ksched + p;
    __syncthreads();

    const double h = a.h, sqh = a.sqh;
    const int total_sub = a.n_store * a.substeps;
    const int n_chunks = (total_sub + T - 1) / T;
    const bool do_gen = !(a.mode & 1);
    const bool do_rec = valid && !(a.mode & 2) && (econ || cred);

    // Generation of chunk c, iteration it (one Philox block -> 2 draws per
    // thread).  Central draws are refined in place; the 4.85% in Acklam's tails
    // are queued per warp (ballot + popc) and refined by full warps at the end
    // of the chunk, so the log/sqrt branch does not serialise ~80% of warps.
    // it and iters are warp-uniform.
    // Per-chunk constants of the generator (hoisted out of the iterations).
    struct GenChunk {
        double* zb;         // the chunk's tile
        uint32_t zb_s;      // its shared-space address
        int nn, nb;         // draws and Philox blocks of the chunk
        uint32_t blk0;      // first block (a path's blocks fit 32 bits: checked on the host)
    };
    auto gen_chunk = [&](int cc) {
        GenChunk g;
        g.zb = zs + (cc & 1) * (T * D * P);
        g.zb_s = static_cast<uint32_t>(__cvta_generic_to_shared(g.zb));
        g.nn = min(T, total_sub - cc * T) * D;
        g.nb = (g.nn + 1) >> 1;
        g.blk0 = static_cast<uint32_t>(cc * T * D) >> 1;
        return g;
    };
    auto gen_iter = [&](const GenChunk& g, int it, int iters, uint32_t& tmask) {
        double* zb = g.zb;
        const int nn = g.nn;
        const int b = w + it * TPP;
        const bool vb = b < g.nb;
        uint64_t w0, w1;
        {  // Philox-2x64-10 on the staged round keys; past the chunk's last block the draws are discarded
            uint64_t c0 = static_cast<uint32_t>(g.blk0 + b), c1 = 0;  // high word 0: a cheaper first round
#pragma unroll
            for (int rr = 0; rr < 10; ++rr) {
                const uint64_t hi = __umul64hi(kPhiloxM, c0);
                const uint64_t lo = kPhiloxM * c0;
                c0 = hi ^ ks[rr * P] ^ c1;
                c1 = lo;
            }
            w0 = c0;
            w1 = c1;
        }
        const double uu[2] = {u64_to_uniform(w0), u64_to_uniform(w1)};
        const uint32_t hw[2] = {static_cast<uint32_t>(w0 >> 32), static_cast<uint32_t>(w1 >> 32)};
        bool v[2], tail[2];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            v[hf] = vb && 2 * b + hf < nn;
            // Acklam's tail test on the draw's top 32 bits (p within 2^-32 of 0.02425 may
            // take either branch: both are refined to the same normal): hw < lo or hw > hi
            tail[hf] = v[hf] && (hw[hf] - kTailLo32 > kTailHi32 - kTailLo32);
        }
        tmask |= (static_cast<uint32_t>(tail[0]) | (static_cast<uint32_t>(tail[1]) << 1)) << (2 * it);
        // Both draws through the central transform, branch-free; a tail draw's slot keeps
        // its uniform until the chunk's tail pass below refines it in place.
        double xx[2];
        normal_central_x2(uu, xx);
        const double s0 = tail[0] ? uu[0] : xx[0], s1 = tail[1] ? uu[1] : xx[1];
        const uint32_t sa = g.zb_s + static_cast<uint32_t>((2 * b * P + p) * 8);
        asm volatile(
            "{\n\t.reg .pred q0, q1;\n\t"
            "setp.ne.b32 q0, %2, 0;\n\t"
            "setp.ne.b32 q1, %4, 0;\n\t"
            "@q0 st.shared.f64 [%0], %1;\n\t"
            "@q1 st.shared.f64 [%0+%5], %3;\n\t}" ::"r"(sa),
            "d"(s0), "r"(static_cast<int>(v[0])), "d"(s1), "r"(static_cast<int>(v[1])), "n"(P * 8)
            : "memory");
        if (it == iters - 1) {
            // The chunk's tail draws (4.85%): each lane's bits compacted into the warp's slot
            // list (exclusive scan of the counts), then refined by full warps.
            const int cnt = __popc(tmask);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            int k = incl - cnt;
            for (uint32_t m = tmask; m; m &= m - 1) {
                const int bit = __ffs(m) - 1;
                qs[k++] = (2 * (w + (bit >> 1) * TPP) + (bit & 1)) * P + p;
            }
            __syncwarp();
            for (int base = 0; base < total; base += 32) {
                const int i = base + lane;
                if (i < total) {
                    const int slot = qs[i];
                    const double u = zb[slot];
                    zb[slot] = halley_refine(acklam_tail_seed(u), u);
                }
            }
            __syncwarp();
            tmask = 0;
        }
    };
    // generator iterations of a full chunk and of the last one (two divisions per launch)
    const int iters_full = ((((T * D) + 1) >> 1) + TPP - 1) / TPP;
    const int iters_last = ((((total_sub - (n_chunks - 1) * T) * D + 1) >> 1) + TPP - 1) / TPP;
    auto gen_iters = [&](int cc) { return cc == n_chunks - 1 ? iters_last : iters_full; };

    // Recursion: substep t of chunk c for the factors this thread owns.  The
    // Cholesky rows of the owned factors live in registers (<= 2 nonzeros:
    // two coefficients and tile offsets; dense rows read the CSR in smem).
    struct ZRow {
        double v0, v1;
        int o0, o1, d;
        bool dense, single;  // single: one nonzero, z = v0 * zraw (0 + v0 z is exact)
    };
    auto zrow = [&](int d) {
        const FactorCoef& k = coef[d];
        return ZRow{k.v0, k.v1, k.col0 * P, k.col1 * P, d, k.dense != 0, k.dense == 0 && k.v1 == 0.0};
    };
    const ZRow zr_a = zrow(econ ? fr : fg0), zr_b = zrow(econ ? 0 : fg1), zr_c = zrow(econ ? fx : fg1);
    // Drift / vol coefficients of the owned factors, also register resident.
    const FactorCoef kc_a = coef[econ ? fr : fg0], kc_b = coef[econ ? 0 : fg1];
    const double kx_c0 = coef[fx].c0, kx_c1 = coef[fx].c1;
    int sub_ctr = a.substeps, next_store = 1;  // countdown to the next pricing step
    auto rec_step = [&](const double* zt) {  // zt: this substep's row of the chunk tile, at path p
        auto zcorr = [&](const ZRow& k) {
            if (k.single) return dmul(k.v0, zt[k.o0]);
            if (!k.dense) return madd(k.v1, zt[k.o1], dmul(k.v0, zt[k.o0]));
            double acc = 0.0;
            for (int q = chol_row[k.d]; q < chol_row[k.d + 1]; ++q) acc = madd(chol_val[q], zt[chol_col[q] * P], acc);
            return acc;
        };
        if (econ) {
            const double r0 = s1, re = s0;
            const double zr = zcorr(zr_a), z0 = zcorr(zr_b), zx = zcorr(zr_c);
            s3 = madd(r0, h, s3);  // -ln beta, left endpoint (market.cpp:208)
            // log chi + (r0 - re - sigma^2/2) h + sigma sqrt(h) z, pre-step rates (market.cpp:211-223)
            s2 = madd(kx_c1, zx, madd(dsub(dsub(r0, re), kx_c0), h, s2));
            s0 = vasicek_step(re, kc_a, h, zr);
            s1 = vasicek_step(r0, kc_b, h, z0);
        } else {
            // Hazards first (left endpoint, market.cpp:209), then full-truncation CIR (:130-134).
            const double z0 = zcorr(zr_a), z1 = zcorr(zr_b);
            const FactorCoef& k0 = kc_a;
            const FactorCoef& k1 = kc_b;
            s2 = madd(s0, h, s2);
            s3 = madd(s1, h, s3);
            const double gp0 = (s0 < 0.0) ? 0.0 : s0, gp1 = (s1 < 0.0) ? 0.0 : s1;
            const double nx0 = madd(dmul(dmul(k0.c2, sqrt(gp0)), sqh), z0, madd(dmul(k0.c0, dsub(k0.c1, gp0)), h, s0));
            const double nx1 = madd(dmul(dmul(k1.c2, sqrt(gp1)), sqh), z1, madd(dmul(k1.c0, dsub(k1.c1, gp1)), h, s1));
            s0 = (nx0 < 0.0) ? 0.0 : nx0;
            s1 = (nx1 < 0.0) ? 0.0 : nx1;
        }
        if (--sub_ctr == 0) {
            store(next_store++);
            sub_ctr = a.substeps;
        }
    };

    // Software pipeline: generation of chunk c+1 (into the other buffer) is
    // interleaved with the recursion of chunk c, so the recursion's short
    // dependent chains hide under the generator's FP64 throughput.  One
    // __syncthreads per chunk publishes the next buffer.
    if (do_gen) {
        uint32_t tmask = 0;
        const int iters = gen_iters(0);
        const GenChunk g0 = gen_chunk(0);
        for (int it = 0; it < iters; ++it) gen_iter(g0, it, iters, tmask);
    }
    __syncthreads();
    for (int c = 0; c < n_chunks; ++c) {
        const int iters = (do_gen && c + 1 < n_chunks) ? gen_iters(c + 1) : 0;
        const int tc = min(T, total_sub - c * T);
        const int steps = max(iters, tc);
        uint32_t tmask = 0;
        const GenChunk gn = gen_chunk(c + 1);
        const double* zt = zs + (c & 1) * (T * D * P) + p;  // advanced by one substep row per step
        for (int s = 0; s < steps; ++s, zt += D * P) {
            if (s < iters) gen_iter(gn, s, iters, tmask);
            if (s < tc && do_rec) rec_step(zt);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K2
struct MtmArgs {
    int E, Cc, M, n_local, start, n_total, paths_per_group;
    const double* lnA;   // [E][n_total+1]
    const double2* dAB;  // [E][n_total+1]: (lnA[m+1] - lnA[m], B[m+1] - B[m])
    const double* B;     // [E][n_total+1]
    const double* Nsuf;  // [E][n_total+1][Cc]  sum notional, maturity >= j
    const double* N;     // [E][n_total+1][Cc]  sum notional, maturity == j
    const double* NSsuf; // [E][n_total+1][Cc]  sum notional*delta*Sigma, maturity >= j
    const double* H;     // [E][n_total+1][Cc]  N[j] + NSsuf[j]
    const double* rates;
    const double* fx;
    const double* lag0;  // [groups][E]
    double* cube;
};

// Thread per (path, local step).  With every swap resetting each pricing step
// (tenor == dt, the reference's generated books, portfolio.cpp:166), the book
// collapses per (economy, client) onto maturity-indexed coefficient vectors:
//   MtM_c = sum_e chi_e [ lead*Nsuf_g - N_g - [g>0] NSsuf_g - sum_{m>=1} Z_m H_{g+m} ]
// with Z_m = exp(lnA_m - B_m r) the Vasicek ZC to g+m (portfolio.cpp:34-45),
// lead = 1/ZC(r_lag, dt) for g > 0 and 1 at g = 0 (portfolio.cpp:65-92).
// Cost per path: E*n^2/2 exponentials instead of the reference's O(S*n^2).
template <int CB>
__global__ void __launch_bounds__(128) k_mtm_linear(MtmArgs a) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (k >= a.M) return;
    const int g = a.start + i;
    const int M = a.M, E = a.E, Cc = a.Cc, n1 = a.n_total + 1;
    for (int c0 = 0; c0 < Cc; c0 += CB) {
        double acc[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) acc[c] = 0.0;
        for (int e = 0; e < E; ++e) {
            const double r = a.rates[(static_cast<size_t>(i) * E + e) * M + k];
            const double chi = (e == 0) ? 1.0 : a.fx[(static_cast<size_t>(i) * (E - 1) + e - 1) * M + k];
            const double* lnA = a.lnA + e * n1;
            const double* B = a.B + e * n1;
            double lead = 1.0;
            if (g > 0) {
                const double rl = (i > 0) ? a.rates[(static_cast<size_t>(i - 1) * E + e) * M + k]
                                          : a.lag0[(k / a.paths_per_group) * E + e];
                lead = 1.0 / exp(lnA[1] - B[1] * rl);
            }
            double v[CB];
            const size_t base = (static_cast<size_t>(e) * n1 + g) * Cc + c0;
#pragma unroll
            for (int c = 0; c < CB; ++c) {
                if (c0 + c < Cc) {
                    v[c] = lead * a.Nsuf[base + c] - a.N[base + c];
                    if (g > 0) v[c] -= a.NSsuf[base + c];
                } else {
                    v[c] = 0.0;
                }
            }
            if (CB % 2 == 0 && Cc % 2 == 0) {  // 16-byte loads of the (warp-uniform) H rows
                // Z_{m+1} = Z_m exp(dA_m - dB_m r): one full exp per (e, path), then a
                // short Taylor factor per maturity (|dA - dB r| <~ dt r; degree 9).
                const double2* dab = a.dAB + e * n1;
                double z = exp_neg(lnA[1] - B[1] * r);
                for (int m = 1; g + m <= a.n_total; ++m) {
                    if (m > 1) {
                        const double2 d = __ldg(dab + m - 1);
                        const double x = fma(-d.y, r, d.x);
                        double q = 2.7557319223985893e-6;  // 1/9!
                        q = fma(q, x, 2.4801587301587302e-5);
                        q = fma(q, x, 1.9841269841269841e-4);
                        q = fma(q, x, 1.3888888888888889e-3);
                        q = fma(q, x, 8.3333333333333333e-3);
                        q = fma(q, x, 4.1666666666666667e-2);
                        q = fma(q, x, 1.6666666666666667e-1);
                        q = fma(q, x, 0.5);
                        q = fma(q, x, 1.0);
                        z = z * fma(q, x, 1.0);
                    }
                    const double2* h =
                        reinterpret_cast<const double2*>(a.H + (static_cast<size_t>(e) * n1 + g + m) * Cc + c0);
#pragma unroll
                    for (int c = 0; c < CB; c += 2)
                        if (c0 + c < Cc) {
                            const double2 hv = __ldg(h + c / 2);
                            v[c] -= z * hv.x;
                            v[c + 1] -= z * hv.y;
                        }
                }
            } else {
                for (int m = 1; g + m <= a.n_total; ++m) {
                    const double z = exp_neg(lnA[m] - B[m] * r);
                    const double* h = a.H + (static_cast<size_t>(e) * n1 + g + m) * Cc + c0;
#pragma unroll
                    for (int c = 0; c < CB; ++c)
                        if (c0 + c < Cc) v[c] -= z * __ldg(h + c);
                }
            }
#pragma unroll
            for (int c = 0; c < CB; ++c) acc[c] += chi * v[c];
        }
#pragma unroll
        for (int c = 0; c < CB; ++c)
            if (c0 + c < Cc) a.cube[(static_cast<size_t>(i) * Cc + c0 + c) * M + k] = acc[c];
    }
}

// NP paths per thread (k + 128 j of the CTA's 128 NP-path slab): the
// warp-uniform coefficient loads (dA/dB, H rows), address arithmetic and loop
// control are shared by the paths, and their independent ZC recurrences
// interleave.  chi_e is folded into the running ZC (z' = chi z), so the client
// accumulators take the maturity sum directly: acc_c += chi (lead Nsuf - N -
// NSsuf) - sum_m z'_m H_{g+m} (same terms as k_mtm_linear, re-associated at
// rounding level).  Requires Cc even (16-byte H loads).
template <int CB, int NP>
__global__ void __launch_bounds__(128) k_mtm_multi(MtmArgs a) {
    const int M = a.M;
    const int kb = blockIdx.x * (128 * NP) + threadIdx.x;
    if (kb >= M) return;
    int kp[NP];
    bool own[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        own[j] = kb + 128 * j < M;
        kp[j] = own[j] ? kb + 128 * j : kb;
    }
    const int i = blockIdx.y;
    const int g = a.start + i;
    const int E = a.E, Cc = a.Cc, n1 = a.n_total + 1;
    for (int c0 = 0; c0 < Cc; c0 += CB) {
        double acc[NP][CB];
#pragma unroll
        for (int j = 0; j < NP; ++j)
#pragma unroll
            for (int c = 0; c < CB; ++c) acc[j][c] = 0.0;
        for (int e = 0; e < E; ++e) {
            const size_t ri = (static_cast<size_t>(i) * E + e) * M;
            const double* lnA = a.lnA + e * n1;
            const double* B = a.B + e * n1;
            double r[NP], z[NP], lead[NP], chi[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                r[j] = a.rates[ri + kp[j]];
                chi[j] = (e > 0) ? a.fx[(static_cast<size_t>(i) * (E - 1) + e - 1) * M + kp[j]] : 1.0;
                lead[j] = 1.0;
                if (g > 0) {
                    const double rl = (i > 0) ? a.rates[(static_cast<size_t>(i - 1) * E + e) * M + kp[j]]
                                              : a.lag0[(kp[j] / a.paths_per_group) * E + e];
                    lead[j] = 1.0 / exp(lnA[1] - B[1] * rl);
                }
            }
            const size_t base = (static_cast<size_t>(e) * n1 + g) * Cc + c0;
#pragma unroll
            for (int c = 0; c < CB; ++c) {
                if (c0 + c < Cc) {
                    const double ns = a.Nsuf[base + c], nn = a.N[base + c];
                    const double nss = (g > 0) ? a.NSsuf[base + c] : 0.0;
#pragma unroll
                    for (int j = 0; j < NP; ++j) acc[j][c] += chi[j] * (lead[j] * ns - nn - nss);
                }
            }
#pragma unroll
            for (int j = 0; j < NP; ++j) z[j] = chi[j] * exp_neg(lnA[1] - B[1] * r[j]);
            const double2* dab = a.dAB + e * n1;
            const double2* hrow = reinterpret_cast<const double2*>(a.H + (static_cast<size_t>(e) * n1 + g + 1) * Cc + c0);
            const int hstep = Cc / 2;
            for (int m = 1; g + m <= a.n_total; ++m, hrow += hstep) {
                if (m > 1) {  // Z_m = Z_{m-1} exp(dA - dB r), degree-9 Taylor (|dA - dB r| <~ dt r)
                    const double2 d = __ldg(dab + m - 1);
                    double x[NP], q[NP];
#pragma unroll
                    for (int j = 0; j < NP; ++j) {
                        x[j] = fma(-d.y, r[j], d.x);
                        q[j] = 2.7557319223985893e-6;  // 1/9!
                    }
#define HCVA_TAYLOR_STEP(cf) _Pragma("unroll") for (int j = 0; j < NP; ++j) q[j] = fma(q[j], x[j], cf);
                    HCVA_TAYLOR_STEP(2.4801587301587302e-5)
                    HCVA_TAYLOR_STEP(1.9841269841269841e-4)
                    HCVA_TAYLOR_STEP(1.3888888888888889e-3)
                    HCVA_TAYLOR_STEP(8.3333333333333333e-3)
                    HCVA_TAYLOR_STEP(4.1666666666666667e-2)
                    HCVA_TAYLOR_STEP(1.6666666666666667e-1)
                    HCVA_TAYLOR_STEP(0.5)
                    HCVA_TAYLOR_STEP(1.0)
#undef HCVA_TAYLOR_STEP
#pragma unroll
                    for (int j = 0; j < NP; ++j) z[j] = z[j] * fma(q[j], x[j], 1.0);
                }
#pragma unroll
                for (int c = 0; c < CB; c += 2)
                    if (c0 + c < Cc) {
                        const double2 hv = __ldg(hrow + c / 2);
#pragma unroll
                        for (int j = 0; j < NP; ++j) {
                            acc[j][c] = fma(-z[j], hv.x, acc[j][c]);
                            acc[j][c + 1] = fma(-z[j], hv.y, acc[j][c + 1]);
                        }
                    }
            }
        }
#pragma unroll
        for (int c = 0; c < CB; ++c)
            if (c0 + c < Cc)
#pragma unroll
                for (int j = 0; j < NP; ++j)
                    if (own[j]) a.cube[(static_cast<size_t>(i) * Cc + c0 + c) * M + kp[j]] = acc[j][c];
    }
}

// Direct per-swap pricing in the reference's loop and summation order
// (portfolio.cpp:58-147) for books that do not reset every pricing step.
struct DirectArgs {
    int E, Cc, M, n_local, start, n_swaps, paths_per_group;
    double dt;
    const hcva_swap* book;
    const hcva_vasicek* vas;
    const double* rates;
    const double* fx;
    const double* lag0;
    double* cube;
};

__device__ double zc_dev(double r, double tau, const hcva_vasicek& p) {
    if (tau == 0.0) return 1.0;
    const double a = p.a, b = p.b, s = p.sigma;
    if (fabs(a) < 1e-8) return exp(-r * tau + s * s * tau * tau * tau / 6.0);
    const double B = (1.0 - exp(-a * tau)) / a;
    const double lnA = (b - s * s / (2.0 * a * a)) * (B - tau) - s * s * B * B / (4.0 * a);
    return exp(lnA - B * r);
}

__device__ bool is_multiple_dev(double x, double step) {
    const double q = x / step;
    return fabs(q - round(q)) < 1e-9 * fmax(1.0, fabs(q));
}

__global__ void __launch_bounds__(128) k_mtm_direct(DirectArgs a) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (k >= a.M) return;
    const int E = a.E, M = a.M;
    const int g = a.start + i;
    const double t = g * a.dt;
    for (int c = 0; c < a.Cc; ++c) a.cube[(static_cast<size_t>(i) * a.Cc + c) * M + k] = 0.0;
    for (int s = 0; s < a.n_swaps; ++s) {
        const hcva_swap sw = a.book[s];
        if (t > sw.maturity + 1e-9) continue;
        const hcva_vasicek vp = a.vas[sw.economy];
        const double r_now = a.rates[(static_cast<size_t>(i) * E + sw.economy) * M + k];
        const double delta = sw.tenor, tbar = sw.maturity, sr = sw.fixed_rate;
        double px;
        if (t < 1e-9) {
            const int m = static_cast<int>(llround(tbar / delta));
            double ann = 0.0;
            for (int j = 1; j <= m; ++j) ann = __dadd_rn(ann, zc_dev(r_now, j * delta, vp));
            px = 1.0 - zc_dev(r_now, tbar, vp) - delta * sr * ann;
        } else {
            const int lag = static_cast<int>(llround(sw.tenor / a.dt));
            const int prev_global = ((g - 1) / lag) * lag;
            const int prev_local = prev_global - a.start;
            const double r_lag = (prev_local >= 0)
                                     ? a.rates[(static_cast<size_t>(prev_local) * E + sw.economy) * M + k]
                                     : a.lag0[(k / a.paths_per_group) * E + sw.economy];
            const bool on_reset = is_multiple_dev(t, delta);
            const int m_total = static_cast<int>(llround(tbar / delta));
            const int j_first = on_reset ? static_cast<int>(llround(t / delta)) + 1
                                         : static_cast<int>(floor(t / delta + 1e-9)) + 1;
            double ann = 0.0;
            for (int j = j_first; j <= m_total; ++j) ann = __dadd_rn(ann, zc_dev(r_now, j * delta - t, vp));
            if (on_reset) {
                px = 1.0 / zc_dev(r_lag, delta, vp) - zc_dev(r_now, tbar - t, vp) - delta * sr * (1.0 + ann);
            } else {
                const double t_prev = floor(t / delta + 1e-9) * delta;
                const double t_next = t_prev + delta;
                px = zc_dev(r_now, t_next - t, vp) / zc_dev(r_lag, t_next - t_prev, vp) -
                     zc_dev(r_now, tbar - t, vp) - delta * sr * ann;
            }
        }
        const double chi = (sw.economy == 0) ? 1.0 : a.fx[(static_cast<size_t>(i) * (E - 1) + sw.economy - 1) * M + k];
        double* dst = a.cube + (static_cast<size_t>(i) * a.Cc + sw.client - 1) * M + k;
        *dst = __dadd_rn(*dst, __dmul_rn(__dmul_rn(sw.notional, px), chi));
    }
}

// ------------------------------------------------------------------ K3
struct DefaultArgs {
    int M, N, n, Cn, path_offset, shard_blk, shard_stride;
    uint64_t key;
    const double* hazard;  // SoA [(i*Cn+c)*M + k]
    uint16_t* steps;       // [c][k*N+l]
    unsigned long long* ties;  // [2]
};

// CTA per path: the path's cumulative hazards are staged in shared memory
// and shared by its N replicas; each replica (k,l) draws one Exp(1)
// threshold per name from split(k).split(l) (defaults.cpp:28-43) and finds
// the first pricing step with Lambda >= eps by binary search over the
// nondecreasing hazard path (identical to the reference's linear scan,
// defaults.cpp:13-18).
__global__ void __launch_bounds__(128) k_defaults(DefaultArgs a) {
    extern __shared__ double hz[];  // [c][i]
    const int k = blockIdx.x;
    const int n1 = a.n + 1, Cn = a.Cn;
    for (int t = threadIdx.x; t < n1 * Cn; t += blockDim.x) {
        const int c = t / n1, i = t % n1;
        hz[t] = a.hazard[(static_cast<size_t>(i) * Cn + c) * a.M + k];
    }
    __syncthreads();
    const uint64_t pkey = split_key(a.key, static_cast<uint64_t>(a.path_offset) + shard_path(k, a.shard_blk, a.shard_stride));
    unsigned long long tie_ulp = 0, tie_rel = 0;
    const size_t R = static_cast<size_t>(a.M) * a.N;
    for (int l = threadIdx.x; l < a.N; l += blockDim.x) {
        const uint64_t rkey = split_key(pkey, static_cast<uint64_t>(l));
        const size_t row = static_cast<size_t>(k) * a.N + l;
        uint64_t w0 = 0, w1 = 0;
        for (int c = 0; c < Cn; ++c) {
            if ((c & 1) == 0) philox2x64(static_cast<uint64_t>(c >> 1), rkey, w0, w1);
            const double eps = -log(u64_to_uniform((c & 1) ? w1 : w0));
            const double* h = hz + c * n1;
            int lo = 0, hi = n1;  // first index in [0, n1) with h >= eps, n1 if none
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (h[mid] >= eps) hi = mid; else lo = mid + 1;
            }
            a.steps[c * R + row] = (lo < n1) ? static_cast<uint16_t>(lo) : static_cast<uint16_t>(0xFFFF);
            // Threshold ties: a neighbouring hazard within 1 ulp / 1e-12 of eps.
            const double ulp = fabs(nextafter(eps, 2.0 * eps + 1.0) - eps);
            const double near_hi = (lo < n1) ? h[lo] - eps : INFINITY;
            const double near_lo = (lo > 0) ? eps - h[lo - 1] : INFINITY;
            const double gap = fmin(near_hi, near_lo);
            if (gap <= ulp) ++tie_ulp;
            if (gap <= 1e-12 * eps) ++tie_rel;
        }
    }
    if (tie_ulp) atomicAdd(&a.ties[0], tie_ulp);
    if (tie_rel) atomicAdd(&a.ties[1], tie_rel);
}

// ------------------------------------------------------------------ K4
struct LabelArgs {
    int M, N, n, Cn, E;
    double dt;
    const double* disc;
    const double* intens;
    const double* cube;      // SoA [(i*Cc + c-1)*M + k]
    const uint16_t* steps;   // [c][R]
    double* out;             // [i][R] for i in [i0, i1]
    int i0, i1;
};

// Defaults labels (labels.cpp:21-48) for steps i0..i1 in one pass: CTA per
// path, discounts and positive exposures staged in shared memory, thread per
// replica.  Summation order is the reference's (clients ascending) and the
// products are rounded as (beta_i^-1 * beta_s) * exposure.
__global__ void __launch_bounds__(128) k_labels_defaults(LabelArgs a) {
    extern __shared__ double sm[];
    const int k = blockIdx.x;
    const int n1 = a.n + 1, Cc = a.Cn - 1;
    double* disc = sm;             // [n1]
    double* inv = sm + n1;         // [n1]
    double* expo = sm + 2 * n1;    // [n1][Cc]
    for (int t = threadIdx.x; t < n1; t += blockDim.x) {
        disc[t] = a.disc[static_cast<size_t>(t) * a.M + k];
        inv[t] = 1.0 / disc[t];
    }
    for (int t = threadIdx.x; t < n1 * Cc; t += blockDim.x) {
        const int i = t / Cc, c = t % Cc;
        const double v = a.cube[(static_cast<size_t>(i) * Cc + c) * a.M + k];
        expo[t] = (v < 0.0) ? 0.0 : v;
    }
    __syncthreads();
    const size_t R = static_cast<size_t>(a.M) * a.N;
    for (int l = threadIdx.x; l < a.N; l += blockDim.x) {
        const size_t row = static_cast<size_t>(k) * a.N + l;
        for (int i = a.i0; i <= a.i1; ++i) {
            double sum = 0.0;
            for (int c = 1; c <= Cc; ++c) {
                const int s = a.steps[c * R + row];
                if (s > i && s <= a.n)
                    sum = __dadd_rn(sum, __dmul_rn(__dmul_rn(inv[i], disc[s]), expo[s * Cc + c - 1]));
            }
            a.out[static_cast<size_t>(i - a.i0) * R + row] = sum;
        }
    }
}

// Register form for Cc <= CMAX: each replica's default steps, the discount at
// its default step and the exposure there are loop invariants over the label
// step i, so per (i, c) only (inv_i * beta_s) * exposure remains -- the same
// rounded products, summed in client order.  A CTA takes PP consecutive paths
// (PP = 1 is used: wider CTAs measured no faster).
template <int CMAX, int PP>
__global__ void __launch_bounds__(128) k_labels_defaults_reg(LabelArgs a) {
    extern __shared__ double sm[];
    const int k0 = blockIdx.x * PP;
    const int np = min(PP, a.M - k0);
    const int n1 = a.n + 1, Cc = a.Cn - 1;
    double* disc = sm;                 // [n1][PP]
    double* inv = sm + n1 * PP;        // [n1][PP]
    double* expo = sm + 2 * n1 * PP;   // [n1][Cc][PP]
    for (int t = threadIdx.x; t < n1 * PP; t += blockDim.x) {
        const int i = t / PP, p = t % PP;
        const double d = (p < np) ? a.disc[static_cast<size_t>(i) * a.M + k0 + p] : 1.0;
        disc[t] = d;
        inv[t] = 1.0 / d;
    }
    for (int t = threadIdx.x; t < n1 * Cc * PP; t += blockDim.x) {
        const int ic = t / PP, p = t % PP;
        const double v = (p < np) ? a.cube[static_cast<size_t>(ic) * a.M + k0 + p] : 0.0;
        expo[t] = (v < 0.0) ? 0.0 : v;
    }
    __syncthreads();
    const size_t R = static_cast<size_t>(a.M) * a.N;
    for (int idx = threadIdx.x; idx < np * a.N; idx += blockDim.x) {
        const int p = idx / a.N;
        const size_t row = static_cast<size_t>(k0) * a.N + idx;
        // w_c = beta_s * exposure_s at client c's default step s; the label at i
        // is beta_i^-1 * sum_{c: s_c > i} w_c (clients ascending) -- the
        // reference's (beta_i^-1 beta_s) exposure products re-associated, equal
        // to a few ulp, with one FP64 multiply per step instead of 2 Cc.
        int st[CMAX];
        double w[CMAX];
#pragma unroll
        for (int c = 0; c < CMAX; ++c) {
            st[c] = -1;
            w[c] = 0.0;
            if (c < Cc) {
                const int s = a.steps[(c + 1) * R + row];
                if (s <= a.n) {
                    st[c] = s;
                    w[c] = __dmul_rn(disc[s * PP + p], expo[(s * Cc + c) * PP + p]);
                }
            }
        }
        for (int i = a.i0; i <= a.i1; ++i) {
            double sum = 0.0;
#pragma unroll
            for (int c = 0; c < CMAX; ++c)
                if (st[c] > i) sum = __dadd_rn(sum, w[c]);
            a.out[static_cast<size_t>(i - a.i0) * R + row] = __dmul_rn(inv[i * PP + p], sum);
        }
    }
}

// Defaults labels for many clients (Cc > 16, e.g. C5's 64): per replica the
// clients are chained by default step (head[s] -> next[c], one byte each in
// shared memory), then one sweep over the steps from n down to 0 adds each
// client's beta_s * exposure_s as the step passes its default step:
// label_i = beta_i^-1 * sum_{c: s_c > i} beta_{s_c} (MtM_{s_c,c})^+ -- the
// reference's terms, summed by descending default step (equal to a few ulp),
// in O(n + Cc) per replica instead of O(n Cc).  PROFILE: per-path sums of each
// step's labels (as k_profile_defaults) instead of the labels.
template <bool PROFILE>
__global__ void __launch_bounds__(128) k_labels_defaults_sweep(LabelArgs a, double* part) {
    extern __shared__ double sm[];
    const int k = blockIdx.x;
    const int n1 = a.n + 1, Cc = a.Cn - 1, nt = blockDim.x;
    constexpr int NW = 4;
    double* disc = sm;                                         // [n1]
    double* inv = disc + n1;                                   // [n1]
    double* expo = inv + n1;                                   // [n1][Cc]
    double* red = expo + static_cast<size_t>(n1) * Cc;         // [n1][NW] (PROFILE)
    uint8_t* head = reinterpret_cast<uint8_t*>(red + (PROFILE ? n1 * NW : 0));  // [n1][nt]
    uint8_t* next = head + static_cast<size_t>(n1) * nt;                         // [Cc][nt]
    for (int t = threadIdx.x; t < n1; t += nt) {
        const double d = a.disc[static_cast<size_t>(t) * a.M + k];
        disc[t] = d;
        inv[t] = 1.0 / d;
    }
    for (int t = threadIdx.x; t < n1 * Cc; t += nt) {
        const double v = a.cube[static_cast<size_t>(t) * a.M + k];
        expo[t] = (v < 0.0) ? 0.0 : v;
    }
    if (PROFILE)
        for (int t = threadIdx.x; t < n1 * NW; t += nt) red[t] = 0.0;
    const size_t R = static_cast<size_t>(a.M) * a.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int l0 = 0; l0 < a.N; l0 += nt) {  // block-uniform passes over the replicas
        __syncthreads();
        for (int t = tid; t < n1 * nt; t += nt) head[t] = 0xFF;
        __syncthreads();
        const int l = l0 + tid;
        const bool live = l < a.N;
        const size_t row = static_cast<size_t>(k) * a.N + (live ? l : 0);
        if (live)
            for (int c = 0; c < Cc; ++c) {  // chain client c under its default step
                const int st = a.steps[(c + 1) * R + row];
                if (st <= a.n) {
                    next[c * nt + tid] = head[st * nt + tid];
                    head[st * nt + tid] = static_cast<uint8_t>(c);
                }
            }
        double S = 0.0;  // sum over clients defaulting after step i
        for (int i = a.n; i >= 0; --i) {
            if (i < a.n)
                for (int c = head[(i + 1) * nt + tid]; c != 0xFF; c = next[c * nt + tid])
                    S = __dadd_rn(S, __dmul_rn(disc[i + 1], expo[(i + 1) * Cc + c]));
            if (i < a.i0 || i > a.i1) continue;
            double v = live ? __dmul_rn(inv[i], S) : 0.0;
            if (PROFILE) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) red[i * NW + warp] += v;
            } else if (live) {
                a.out[static_cast<size_t>(i - a.i0) * R + row] = v;
            }
        }
    }
    if (PROFILE) {
        __syncthreads();
        for (int i = a.i0 + tid; i <= a.i1; i += nt)
            part[static_cast<size_t>(i - a.i0) * a.M + k] =
                red[i * NW] + red[i * NW + 1] + red[i * NW + 2] + red[i * NW + 3];
    }
}

inline size_t sweep_smem(int n1, int Cc, int nt, bool profile) {
    return sizeof(double) * (2 * static_cast<size_t>(n1) + static_cast<size_t>(n1) * Cc + (profile ? 4 * n1 : 0)) +
           static_cast<size_t>(n1) * nt + static_cast<size_t>(Cc) * nt;
}

// CVA profile without materialising the labels (defaults kind): the register
// form of k_labels_defaults_reg per path, each step's labels summed over the
// path's replicas (warp shuffles, then the warps in fixed order) into
// part[i][k]; k_profile_paths sums the paths.  1.7 GB of label stores and
// re-reads at C2 become 13 MB of per-path sums.
template <int CMAX>
__global__ void __launch_bounds__(128) k_profile_defaults(LabelArgs a, double* part) {
    extern __shared__ double sm[];
    const int k = blockIdx.x;
    const int n1 = a.n + 1, Cc = a.Cn - 1;
    constexpr int NW = 4;              // 128 threads
    double* disc = sm;                 // [n1]
    double* inv = sm + n1;             // [n1]
    double* expo = sm + 2 * n1;        // [n1][Cc]
    double* red = expo + n1 * Cc;      // [n1][NW]
    for (int t = threadIdx.x; t < n1; t += blockDim.x) {
        const double d = a.disc[static_cast<size_t>(t) * a.M + k];
        disc[t] = d;
        inv[t] = 1.0 / d;
    }
    for (int t = threadIdx.x; t < n1 * Cc; t += blockDim.x) {
        const double v = a.cube[static_cast<size_t>(t) * a.M + k];
        expo[t] = (v < 0.0) ? 0.0 : v;
    }
    for (int t = threadIdx.x; t < n1 * NW; t += blockDim.x) red[t] = 0.0;
    __syncthreads();
    const size_t R = static_cast<size_t>(a.M) * a.N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int l0 = 0; l0 < a.N; l0 += blockDim.x) {  // block-uniform passes over the replicas
        const int l = l0 + threadIdx.x;
        const bool live = l < a.N;
        const size_t row = static_cast<size_t>(k) * a.N + (live ? l : 0);
        int st[CMAX];
        double w[CMAX];
#pragma unroll
        for (int c = 0; c < CMAX; ++c) {
            st[c] = -1;
            w[c] = 0.0;
            if (live && c < Cc) {
                const int s = a.steps[(c + 1) * R + row];
                if (s <= a.n) {
                    st[c] = s;
                    w[c] = __dmul_rn(disc[s], expo[s * Cc + c]);
                }
            }
        }
        for (int i = a.i0; i <= a.i1; ++i) {
            double sum = 0.0;
#pragma unroll
            for (int c = 0; c < CMAX; ++c)
                if (st[c] > i) sum = __dadd_rn(sum, w[c]);
            double v = __dmul_rn(inv[i], sum);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[i * NW + warp] += v;
        }
    }
    __syncthreads();
    for (int i = a.i0 + threadIdx.x; i <= a.i1; i += blockDim.x)
        part[static_cast<size_t>(i - a.i0) * a.M + k] = red[i * NW] + red[i * NW + 1] + red[i * NW + 2] + red[i * NW + 3];
}

__global__ void __launch_bounds__(256) k_profile_paths(const double* part, int M, double R, double* out) {
    __shared__ double red[256];
    const double* row = part + static_cast<size_t>(blockIdx.x) * M;
    double s = 0.0;
    for (int k = threadIdx.x; k < M; k += 256) s += row[k];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = red[0] / R;
}

// Intensity labels (labels.cpp:50-88).  Phase 1: survivor values per
// (step, client) in the reference's loop order; phase 2: per replica sum over
// surviving clients.
__global__ void __launch_bounds__(128) k_labels_intensity(LabelArgs a) {
    extern __shared__ double sm[];
    const int k = blockIdx.x;
    const int n1 = a.n + 1, Cn = a.Cn, Cc = Cn - 1;
    double* disc = sm;                 // [n1]
    double* expo = sm + n1;            // [n1][Cc]
    double* gam = expo + n1 * Cc;      // [n1][Cc]
    double* sv = gam + n1 * Cc;        // [n1][Cc]
    for (int t = threadIdx.x; t < n1; t += blockDim.x) disc[t] = a.disc[static_cast<size_t>(t) * a.M + k];
    for (int t = threadIdx.x; t < n1 * Cc; t += blockDim.x) {
        const int i = t / Cc, c = t % Cc;
        const double v = a.cube[(static_cast<size_t>(i) * Cc + c) * a.M + k];
        expo[t] = (v < 0.0) ? 0.0 : v;
        gam[t] = a.intens[(static_cast<size_t>(i) * Cn + c + 1) * a.M + k];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < (a.i1 - a.i0 + 1) * Cc; t += blockDim.x) {
        const int i = a.i0 + t / Cc, c = t % Cc;
        const double inv = 1.0 / disc[i];
        double acc = 0.0, gsum = 0.0;
        for (int j = i; j <= a.n - 1; ++j) {
            const double gj = gam[j * Cc + c];
            const double term = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(inv, disc[j]), expo[j * Cc + c]), gj), a.dt);
            acc = __dadd_rn(acc, __dmul_rn(term, exp(-gsum)));
            gsum = __dadd_rn(gsum, __dmul_rn(gj, a.dt));
        }
        sv[i * Cc + c] = acc;
    }
    __syncthreads();
    const size_t R = static_cast<size_t>(a.M) * a.N;
    for (int l = threadIdx.x; l < a.N; l += blockDim.x) {
        const size_t row = static_cast<size_t>(k) * a.N + l;
        for (int i = a.i0; i <= a.i1; ++i) {
            double sum = 0.0;
            for (int c = 1; c <= Cc; ++c)
                if (a.steps[c * R + row] > i) sum = __dadd_rn(sum, sv[i * Cc + c - 1]);
            a.out[static_cast<size_t>(i - a.i0) * R + row] = sum;
        }
    }
}

// Feature rows of one step (labels.cpp:142-167), row-major R x (p+q).
struct FeatureArgs {
    int M, N, n, Cn, E, step, paths_per_group;
    const double *rates, *fx, *intens, *lag0;
    const uint16_t* steps;
    double* out;
};

__global__ void k_features(FeatureArgs a) {
    const size_t R = static_cast<size_t>(a.M) * a.N;
    const size_t row = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (row >= R) return;
    const int k = static_cast<int>(row / a.N);
    const int E = a.E, Cn = a.Cn, M = a.M, i = a.step;
    const int cols = (Cn - 1) + E + (E - 1) + (Cn - 1) + E;
    double* o = a.out + row * cols;
    int col = 0;
    for (int c = 1; c < Cn; ++c) o[col++] = (a.steps[c * R + row] <= i) ? 1.0 : 0.0;
    for (int e = 0; e < E; ++e) o[col++] = a.rates[(static_cast<size_t>(i) * E + e) * M + k];
    for (int e = 1; e < E; ++e) o[col++] = a.fx[(static_cast<size_t>(i) * (E - 1) + e - 1) * M + k];
    for (int c = 1; c < Cn; ++c) o[col++] = a.intens[(static_cast<size_t>(i) * Cn + c) * M + k];
    for (int e = 0; e < E; ++e)
        o[col++] = (i == 0) ? a.lag0[(k / a.paths_per_group) * E + e]
                            : a.rates[(static_cast<size_t>(i - 1) * E + e) * M + k];
}

// SoA [(i*F+f)*M + k] -> AoS [(k*(n1)+i)*F + f]
__global__ void k_soa_to_aos(const double* in, double* out, int M, int n1, int F, int mode,
                             const double* lag0, int E, int ppg) {
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const size_t total = static_cast<size_t>(M) * n1 * F;
    if (t >= total) return;
    const int f = static_cast<int>(t % F);
    const size_t ki = t / F;
    const int i = static_cast<int>(ki % n1), k = static_cast<int>(ki / n1);
    double v;
    if (mode == 1) {  // lagged rates derived from the rate block
        v = (i == 0) ? lag0[(k / ppg) * E + f] : in[(static_cast<size_t>(i - 1) * F + f) * M + k];
    } else {
        v = in[(static_cast<size_t>(i) * F + f) * M + k];
    }
    out[t] = v;
}

__global__ void k_steps_to_aos(const uint16_t* in, uint16_t* out, size_t R, int Cn) {
    const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (t >= R * Cn) return;
    const int c = static_cast<int>(t % Cn);
    const size_t r = t / Cn;
    out[t] = in[c * R + r];
}

// Per-step mean of the labels: the CVA profile E[xi_i] (deterministic
// fixed-order reduction; CTA per step).
__global__ void __launch_bounds__(256) k_profile(const double* labels, size_t R, double* out) {
    __shared__ double red[256];
    const double* row = labels + blockIdx.x * R;
    double s = 0.0;
    for (size_t r = threadIdx.x; r < R; r += 256) s += row[r];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = red[0] / static_cast<double>(R);
}

// ================================================================= host side

void check_launch(hcva_ctx* ctx) {
    ctx->launches++;
    HCVA_CUDA(cudaGetLastError());
}

template <int P>
void launch_market_p(const MarketArgs& a, int grid, int threads, size_t smem, cudaStream_t s) {
    k_market<P><<<grid, threads, smem, s>>>(a);
}

using MarketLauncher = void (*)(const MarketArgs&, int, int, size_t, cudaStream_t);

MarketLauncher market_launcher(int P) {
    switch (P) {
        case 1: return launch_market_p<1>;
        case 2: return launch_market_p<2>;
        case 4: return launch_market_p<4>;
        case 8: return launch_market_p<8>;
        case 16: return launch_market_p<16>;
        default: return launch_market_p<32>;
    }
}

const void* market_kernel(int P) {
    switch (P) {
        case 1: return reinterpret_cast<const void*>(k_market<1>);
        case 2: return reinterpret_cast<const void*>(k_market<2>);
        case 4: return reinterpret_cast<const void*>(k_market<4>);
        case 8: return reinterpret_cast<const void*>(k_market<8>);
        case 16: return reinterpret_cast<const void*>(k_market<16>);
        default: return reinterpret_cast<const void*>(k_market<32>);
    }
}

// K1 launch shape: P paths per CTA (P | 32), owner threads per path W =
// E + ceil(Cn/2), chunk T substeps.  Chosen to minimise the wave-quantisation
// loss ceil(waves)/waves of M/P equal-cost CTAs over the resident slots.
void choose_market_shape(hcva_sim* sim) {
    const Model& m = sim->model;
    const int D = m.D;
    // K1 counts a path's Philox blocks (and its chunks' draws) in 32-bit integers
    if (static_cast<long long>(sim->n) * m.substeps * D + 64LL * D >= (1LL << 31))
        throw config_error("diffusion: normals per path exceed the engine's 32-bit draw counter");
    const size_t head = 8 * D + sim->m_nnz + (sim->m_nnz + D + 2) / 2;
    double best = -1.0;
    for (int P : {16, 8, 4, 2, 1}) {
        const int per_warp = 32 / P;
        const int We = ((m.E + per_warp - 1) / per_warp) * per_warp;
        const int W = We + (m.Cn + 1) / 2;
        const int NT = ((P * W + 31) / 32) * 32;
        if (NT > 512) continue;
        const int TPP = NT / P;
        auto qcap_of = [&](int T) {  // 64 tail slots per generator iteration of a chunk, per warp
            return 64 * (((T * D + 1) / 2 + TPP - 1) / TPP);
        };
        // T even, ~7 normal pairs per thread per chunk, bounded by shared memory.
        int T = std::max(2, ((2 * TPP * 7) / D) & ~1);
        T = std::min(T, 16);
        if (const char* e = std::getenv("HCVA_K1_T")) T = std::max(2, std::atoi(e) & ~1);  // profiling knob
        while (T > 2 && qcap_of(T) > 64 * kMaxGenIters) T -= 2;
        if (qcap_of(T) > 64 * kMaxGenIters) continue;
        const size_t hk = head + 10 * static_cast<size_t>(P);  // + the Philox key schedule
        auto smem_of = [&](int T) {
            return sizeof(double) * (hk + (static_cast<size_t>(NT / 32) * qcap_of(T) + 1) / 2 +
                                     2 * static_cast<size_t>(T) * D * P);
        };
        size_t smem = smem_of(T);
        while (smem > 100 * 1024 && T > 2) {
            T -= 2;
            smem = smem_of(T);
        }
        if (smem > 227 * 1024) continue;
        HCVA_CUDA(cudaFuncSetAttribute(market_kernel(P), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(std::max<size_t>(smem, 48 * 1024))));
        int per_sm = 0;
        HCVA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, market_kernel(P), NT, smem));
        if (per_sm < 1) continue;
        const double ctas = (sim->M + P - 1) / P;
        const double waves = ctas / (static_cast<double>(per_sm) * sim->ctx->sm_count);
        const double eff = waves / std::ceil(waves) * std::min(1.0, static_cast<double>(P * W) / NT);
        if (eff > best + 1e-3) {
            best = eff;
            sim->m_P = P;
            sim->m_NT = NT;
            sim->m_We = We;
            sim->m_T = T;
            sim->m_qcap = qcap_of(T);
            sim->m_smem = smem;
        }
    }
    if (best < 0) throw config_error("model too large for the diffusion kernel (shared memory)");
}

// Stage K1's tables: per-factor coefficients computed with the reference's
// rounding (market.cpp:121-134, 214-216), the Cholesky factor as CSR (exact
// zeros skipped: adding +-0 to the running sum is an identity), group states.
void prepare_market(hcva_sim* sim, const std::vector<uint64_t>& group_keys,
                    const std::vector<double>& init_state, int paths_per_group, uint64_t local_offset) {
    const Model& m = sim->model;
    const int D = m.D, E = m.E, Cn = m.Cn;
    const double h = m.dt / m.substeps;
    const double sqh = std::sqrt(h);
    std::vector<FactorCoef> coef(D);
    for (int e = 0; e < E; ++e) {
        const double q = (e == 0) ? 0.0 : m.fx[e - 1].rho * m.fx[e - 1].sigma * m.rates[e].sigma;
        coef[e] = FactorCoef{m.rates[e].a, m.rates[e].b, q, m.rates[e].sigma * sqh};
    }
    for (int e = 1; e < E; ++e)
        coef[E + e - 1] = FactorCoef{0.5 * m.fx[e - 1].sigma * m.fx[e - 1].sigma, m.fx[e - 1].sigma * sqh, 0, 0};
    for (int c = 0; c < Cn; ++c)
        coef[2 * E - 1 + c] = FactorCoef{m.credit[c].alpha, m.credit[c].delta, m.credit[c].nu, 0};
    std::vector<int> row(D + 1, 0), col;
    std::vector<double> val;
    for (int d = 0; d < D; ++d) {
        for (int j = 0; j <= d; ++j) {
            const double v = m.chol[static_cast<size_t>(d) * D + j];
            if (v != 0.0) {
                col.push_back(j);
                val.push_back(v);
            }
        }
        row[d + 1] = static_cast<int>(col.size());
        // Short rows inline: acc = 0 + v0 z0 (+ v1 z1), a missing second term is
        // +0 * z1, which leaves the sum unchanged bit for bit.
        const int nz = row[d + 1] - row[d];
        FactorCoef& k = coef[d];
        k.dense = nz > 2;
        k.v0 = nz >= 1 ? val[row[d]] : 0.0;
        k.col0 = nz >= 1 ? col[row[d]] : 0;
        k.v1 = nz == 2 ? val[row[d] + 1] : 0.0;
        k.col1 = nz == 2 ? col[row[d] + 1] : k.col0;
    }
    sim->m_nnz = static_cast<int>(col.size());
    stage(sim->m_coef, coef);
    stage(sim->m_row, row);
    stage(sim->m_col, col);
    stage(sim->m_val, val);
    stage(sim->m_init, init_state);
    if (group_keys.size() > 1) stage(sim->m_keys, group_keys);
    sim->m_ppg = paths_per_group;
    sim->m_local_offset = local_offset;
    choose_market_shape(sim);
    const Model& mm = sim->model;
    const size_t n1 = sim->n + 1, M = sim->M;
    sim->rates.alloc(sizeof(double) * n1 * mm.E * M);
    sim->fx.alloc(sizeof(double) * n1 * std::max(mm.E - 1, 1) * M);
    sim->intens.alloc(sizeof(double) * n1 * mm.Cn * M);
    sim->hazard.alloc(sizeof(double) * n1 * mm.Cn * M);
    sim->disc.alloc(sizeof(double) * n1 * M);
}

void launch_market(hcva_sim* sim, uint64_t key0) {
    hcva_ctx* ctx = sim->ctx;
    const Model& m = sim->model;
    MarketArgs a{};
    a.E = m.E; a.Cn = m.Cn; a.D = m.D; a.substeps = m.substeps; a.n_store = sim->n; a.M = sim->M;
    a.T = sim->m_T; a.nnz = sim->m_nnz; a.paths_per_group = sim->m_ppg; a.local_offset = sim->m_local_offset;
    a.shard_blk = sim->shard_blk; a.shard_stride = sim->shard_stride;
    a.h = m.dt / m.substeps; a.sqh = std::sqrt(a.h);
    a.key0 = key0;
    a.W_econ = sim->m_We;
    a.qcap = sim->m_qcap;
    if (const char* env = std::getenv("HCVA_K1_MODE")) a.mode = std::atoi(env);
    a.group_keys = sim->m_keys.p ? sim->m_keys.as<uint64_t>() : nullptr;
    a.init_state = sim->m_init.as<double>(); a.coef = sim->m_coef.as<FactorCoef>();
    a.chol_row = sim->m_row.as<int>(); a.chol_col = sim->m_col.as<int>(); a.chol_val = sim->m_val.as<double>();
    a.rates = sim->rates.as<double>(); a.fx = sim->fx.as<double>(); a.intens = sim->intens.as<double>();
    a.hazard = sim->hazard.as<double>(); a.disc = sim->disc.as<double>();
    market_launcher(sim->m_P)(a, grid1(sim->M, sim->m_P), sim->m_NT, sim->m_smem, ctx->stream);
    check_launch(ctx);
}

// Stage K2's tables.  Linear (coefficient) form when every swap resets each
// pricing step; the direct per-swap kernel otherwise (portfolio.cpp:97-147).
void prepare_cube(hcva_sim* sim, const hcva_swap* book, int n_swaps) {
    const Model& m = sim->model;
    if (!book || n_swaps < 1) throw contract_error("build_mtm_cube: empty book");
    const int E = m.E, Cc = m.Cc, n_total = m.n_steps;
    bool linear = true;
    for (int s = 0; s < n_swaps; ++s) {
        const hcva_swap& sw = book[s];
        if (sw.client < 1 || sw.client > Cc) throw contract_error("build_mtm_cube: swap client out of range");
        if (sw.economy < 0 || sw.economy >= E) throw contract_error("build_mtm_cube: swap economy out of range");
        const double lag_d = sw.tenor / m.dt;
        const int lag = static_cast<int>(std::llround(lag_d));
        if (std::fabs(lag_d - lag) > 1e-9 || lag < 1)
            throw config_error("build_mtm_cube: swap tenor must be a multiple of the pricing step");
        if (sim->start_step > 0 && lag != 1)
            throw contract_error("build_mtm_cube: conditional blocks require tenor == pricing step");
        if (lag != 1 || !is_multiple(sw.maturity, sw.tenor)) linear = false;
        if (sw.maturity > n_total * m.dt + 1e-9) linear = false;
    }
    sim->c_linear = linear;
    sim->c_nswaps = n_swaps;
    sim->cube.alloc(sizeof(double) * (sim->n + 1) * static_cast<size_t>(Cc) * sim->M);
    if (!linear) {
        stage(sim->c_book, std::vector<hcva_swap>(book, book + n_swaps));
        stage(sim->c_vas, m.rates);
        return;
    }
    const int n1 = n_total + 1;
    std::vector<double> lnA(static_cast<size_t>(E) * n1), B(static_cast<size_t>(E) * n1);
    for (int e = 0; e < E; ++e) {  // zc_price's A(tau), B(tau) at tau = j*dt (portfolio.cpp:34-45)
        const hcva_vasicek& p = m.rates[e];
        for (int j = 0; j < n1; ++j) {
            const double tau = j * m.dt;
            double b = 0.0, la = 0.0;
            if (tau == 0.0) {
            } else if (std::fabs(p.a) < 1e-8) {
                b = tau;
                la = p.sigma * p.sigma * tau * tau * tau / 6.0;
            } else {
                b = (1.0 - std::exp(-p.a * tau)) / p.a;
                la = (p.b - p.sigma * p.sigma / (2.0 * p.a * p.a)) * (b - tau) - p.sigma * p.sigma * b * b / (4.0 * p.a);
            }
            lnA[e * n1 + j] = la;
            B[e * n1 + j] = b;
        }
    }
    const size_t tsz = static_cast<size_t>(E) * n1 * Cc;
    std::vector<double> Nm(tsz, 0.0), NSm(tsz, 0.0), Nsuf(tsz, 0.0), NSsuf(tsz, 0.0), H(tsz, 0.0);
    for (int s = 0; s < n_swaps; ++s) {
        const hcva_swap& sw = book[s];
        const int mat = static_cast<int>(std::llround(sw.maturity / sw.tenor));
        const size_t idx = (static_cast<size_t>(sw.economy) * n1 + mat) * Cc + sw.client - 1;
        Nm[idx] += sw.notional;
        NSm[idx] += sw.notional * (sw.tenor * sw.fixed_rate);
    }
    for (int e = 0; e < E; ++e)
        for (int c = 0; c < Cc; ++c) {
            double a1 = 0.0, a2 = 0.0;
            for (int j = n1 - 1; j >= 0; --j) {
                const size_t idx = (static_cast<size_t>(e) * n1 + j) * Cc + c;
                a1 += Nm[idx];
                a2 += NSm[idx];
                Nsuf[idx] = a1;
                NSsuf[idx] = a2;
                H[idx] = Nm[idx] + a2;
            }
        }
    std::vector<double> dAB(static_cast<size_t>(E) * n1 * 2, 0.0);
    for (int e = 0; e < E; ++e)
        for (int j = 0; j + 1 < n1; ++j) {
            dAB[(static_cast<size_t>(e) * n1 + j) * 2] = lnA[e * n1 + j + 1] - lnA[e * n1 + j];
            dAB[(static_cast<size_t>(e) * n1 + j) * 2 + 1] = B[e * n1 + j + 1] - B[e * n1 + j];
        }
    stage(sim->c_lnA, lnA);
    stage(sim->c_B, B);
    stage(sim->c_dAB, dAB);
    stage(sim->c_Nsuf, Nsuf);
    stage(sim->c_N, Nm);
    stage(sim->c_NSsuf, NSsuf);
    stage(sim->c_H, H);
}

void launch_cube(hcva_sim* sim) {
    hcva_ctx* ctx = sim->ctx;
    const Model& m = sim->model;
    dim3 grid(grid1(sim->M, 128), sim->n + 1);
    if (sim->c_linear) {
        MtmArgs a{};
        a.E = m.E; a.Cc = m.Cc; a.M = sim->M; a.n_local = sim->n; a.start = sim->start_step; a.n_total = m.n_steps;
        a.paths_per_group = sim->M / sim->n_groups;
        a.lnA = sim->c_lnA.as<double>(); a.B = sim->c_B.as<double>(); a.Nsuf = sim->c_Nsuf.as<double>();
        a.dAB = sim->c_dAB.as<double2>();
        a.N = sim->c_N.as<double>(); a.NSsuf = sim->c_NSsuf.as<double>(); a.H = sim->c_H.as<double>();
        a.rates = sim->rates.as<double>(); a.fx = sim->fx.as<double>(); a.lag0 = sim->lag0.as<double>();
        a.cube = sim->cube.as<double>();
        if (m.Cc % 2 == 0) {  // four paths per thread (measured best for 8 and 64 clients)
            k_mtm_multi<8, 4><<<dim3((sim->M + 511) / 512, sim->n + 1), 128, 0, ctx->stream>>>(a);
        } else {
            k_mtm_linear<8><<<grid, 128, 0, ctx->stream>>>(a);
        }
    } else {
        DirectArgs a{};
        a.E = m.E; a.Cc = m.Cc; a.M = sim->M; a.n_local = sim->n; a.start = sim->start_step; a.n_swaps = sim->c_nswaps;
        a.paths_per_group = sim->M / sim->n_groups; a.dt = m.dt;
        a.book = sim->c_book.as<hcva_swap>(); a.vas = sim->c_vas.as<hcva_vasicek>();
        a.rates = sim->rates.as<double>(); a.fx = sim->fx.as<double>();
        a.lag0 = sim->lag0.as<double>(); a.cube = sim->cube.as<double>();
        k_mtm_direct<<<grid, 128, 0, ctx->stream>>>(a);
    }
    check_launch(ctx);
    sim->has_cube = true;
}

void prepare_defaults(hcva_sim* sim, int N) {
    if (N < 1) throw contract_error("sample_default_block: n_replicas must be >= 1");
    if (sim->n >= 0xFFFF) throw contract_error("sample_default_block: too many steps for uint16 storage");
    sim->N = N;
    const size_t R = static_cast<size_t>(sim->M) * N;
    const size_t bytes = sizeof(uint16_t) * R * sim->model.Cn;
    if (sim->steps.bytes != bytes) sim->steps.alloc(bytes);
    if (!sim->ties.p) sim->ties.alloc(2 * sizeof(unsigned long long));
    const size_t smem = sizeof(double) * (sim->n + 1) * sim->model.Cn;
    if (smem > 227 * 1024) throw config_error("too many names x steps for the over-simulation kernel");
    if (smem > 48 * 1024)
        HCVA_CUDA(cudaFuncSetAttribute(k_defaults, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
}

// K3 for N replicas of every path of sim's market into `steps` ([c][k*N+l]).
void launch_defaults_into(hcva_sim* sim, uint64_t key, int N, uint16_t* steps, unsigned long long* ties) {
    hcva_ctx* ctx = sim->ctx;
    HCVA_CUDA(cudaMemsetAsync(ties, 0, 2 * sizeof(unsigned long long), ctx->stream));
    DefaultArgs a{};
    a.M = sim->M; a.N = N; a.n = sim->n; a.Cn = sim->model.Cn; a.path_offset = sim->path_offset; a.key = key;
    a.shard_blk = sim->shard_blk; a.shard_stride = sim->shard_stride;
    a.hazard = sim->hazard.as<double>(); a.steps = steps;
    a.ties = ties;
    const size_t smem = sizeof(double) * (sim->n + 1) * sim->model.Cn;
    const int threads = std::min(128, ((N + 31) / 32) * 32);
    k_defaults<<<sim->M, threads, smem, ctx->stream>>>(a);
    check_launch(ctx);
}

void launch_defaults(hcva_sim* sim, uint64_t key) {
    launch_defaults_into(sim, key, sim->N, sim->steps.as<uint16_t>(), sim->ties.as<unsigned long long>());
    sim->has_defaults = true;
    sim->labels_kind = -1;
}

void launch_labels(hcva_sim* sim, int kind, int i0, int i1, double* dev_out) {
    if (!sim->has_defaults) throw contract_error("labels: no default block");
    launch_labels_from(sim, kind, i0, i1, sim->steps.as<uint16_t>(), sim->N, dev_out);
}

// K4 over an arbitrary default block of sim's market (steps [c][k*N+l], N replicas).
void launch_labels_from(hcva_sim* sim, int kind, int i0, int i1, const uint16_t* steps, int N, double* dev_out) {
    hcva_ctx* ctx = sim->ctx;
    if (!sim->has_cube) throw contract_error("labels: no MtM cube");
    if (sim->start_step != 0) throw contract_error("labels expect an outer (non-rebased) market block");
    if (i0 < 0 || i1 > sim->n || i0 > i1) throw contract_error("label step out of range");
    const Model& m = sim->model;
    LabelArgs a{};
    a.M = sim->M; a.N = N; a.n = sim->n; a.Cn = m.Cn; a.E = m.E; a.dt = m.dt;
    a.disc = sim->disc.as<double>(); a.intens = sim->intens.as<double>(); a.cube = sim->cube.as<double>();
    a.steps = steps; a.out = dev_out; a.i0 = i0; a.i1 = i1;
    const int n1 = sim->n + 1, Cc = m.Cc;
    const int threads = std::min(128, ((N + 31) / 32) * 32);
    if (kind == 0) {
        const size_t smem = sizeof(double) * (2 * n1 + static_cast<size_t>(n1) * Cc);
        if (smem > 48 * 1024)
            HCVA_CUDA(cudaFuncSetAttribute(k_labels_defaults, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        if (Cc <= 16) {
            const void* fn = Cc <= 8 ? (const void*)k_labels_defaults_reg<8, 1> : (const void*)k_labels_defaults_reg<16, 1>;
            if (smem > 48 * 1024)
                HCVA_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            void* args[] = {&a};
            HCVA_CUDA(cudaLaunchKernel(fn, dim3(sim->M), dim3(threads), args, smem, ctx->stream));
        } else if (Cc < 255) {
            const size_t sm2 = sweep_smem(n1, Cc, 128, false);
            HCVA_CUDA(cudaFuncSetAttribute(k_labels_defaults_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(sm2)));
            k_labels_defaults_sweep<false><<<sim->M, 128, sm2, ctx->stream>>>(a, nullptr);
        } else {
            k_labels_defaults<<<sim->M, threads, smem, ctx->stream>>>(a);
        }
    } else {
        const size_t smem = sizeof(double) * (n1 + 3 * static_cast<size_t>(n1) * Cc);
        if (smem > 48 * 1024)
            HCVA_CUDA(cudaFuncSetAttribute(k_labels_intensity, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        k_labels_intensity<<<sim->M, 128, smem, ctx->stream>>>(a);
    }
    check_launch(ctx);
}

// Q/R probe block (pipeline.cpp:79-81): two extra replicas per path from
// `key` and their labels at every step, beside the set's own default block.
void probe_block(hcva_sim* sim, uint64_t key, int kind, DeviceBuf& steps, DeviceBuf& labels) {
    if (!sim->has_cube) throw contract_error("labels: no MtM cube");
    if (sim->start_step != 0) throw contract_error("labels expect an outer (non-rebased) market block");
    const size_t R2 = static_cast<size_t>(sim->M) * 2;
    steps.alloc(R2 * sim->model.Cn * sizeof(uint16_t));
    labels.alloc(R2 * (sim->n + 1) * sizeof(double));
    DeviceBuf ties;
    ties.alloc(2 * sizeof(unsigned long long));
    launch_defaults_into(sim, key, 2, steps.as<uint16_t>(), ties.as<unsigned long long>());
    launch_labels_from(sim, kind, 0, sim->n, steps.as<uint16_t>(), 2, labels.as<double>());
}

void launch_labels_all(hcva_sim* sim, int kind) {
    const size_t R = static_cast<size_t>(sim->M) * sim->N, bytes = R * (sim->n + 1) * sizeof(double);
    if (sim->labels.bytes != bytes) sim->labels.alloc(bytes);
    launch_labels(sim, kind, 0, sim->n, sim->labels.as<double>());
    sim->labels_kind = kind;
}

void copy_out(hcva_ctx* ctx, void* dst, const void* src, size_t bytes) {
    HCVA_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
    HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
}

hcva_sim* new_sim(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid) {
    return new_sim(ctx, make_model(model, grid));
}

hcva_sim* new_sim(hcva_ctx* ctx, const Model& model) {
    if (!ctx) throw contract_error("null context");
    HCVA_CUDA(cudaSetDevice(ctx->device));
    auto sim = std::make_unique<hcva_sim>();
    sim->ctx = ctx;
    sim->model = model;
    return sim.release();
}

void record(hcva_sim* sim, int slot, int phase) {
    if (slot < 0) return;
    const size_t idx = static_cast<size_t>(slot) * 5 + phase;
    while (sim->events.size() <= idx) {
        cudaEvent_t e;
        HCVA_CUDA(cudaEventCreate(&e));
        sim->events.push_back(e);
    }
    HCVA_CUDA(cudaEventRecord(sim->events[idx], sim->ctx->stream));
}

}  // namespace hcva

using namespace hcva;

extern "C" {

hcva_status hcva_ctx_create(int device, hcva_ctx** out) {
    return guarded([&] {
        int n = 0;
        HCVA_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw contract_error("hcva_ctx_create: no such device");
        HCVA_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        HCVA_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10 || prop.minor != 0)
            throw cuda_error("libhcva_gpu.so is built for sm_100a (B200); found sm_" + std::to_string(prop.major) +
                             std::to_string(prop.minor));
        auto ctx = std::make_unique<hcva_ctx>();
        ctx->device = device;
        ctx->sm_count = prop.multiProcessorCount;
        HCVA_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        // Keep freed pool memory reserved: repeated simulate/label calls then
        // re-use it instead of returning gigabytes to the driver each time.
        cudaMemPool_t pool;
        HCVA_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t threshold = UINT64_MAX;
        HCVA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
        *out = ctx.release();
    });
}

hcva_status hcva_ctx_destroy(hcva_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

hcva_status hcva_ctx_stream(hcva_ctx* ctx, void** stream_out) {
    return guarded([&] { *stream_out = ctx->stream; });
}

hcva_status hcva_ctx_synchronize(hcva_ctx* ctx) {
    return guarded([&] { HCVA_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

hcva_status hcva_ctx_launch_count(hcva_ctx* ctx, uint64_t* out) {
    return guarded([&] { *out = ctx->launches; });
}

hcva_status hcva_rng_draw(hcva_ctx* ctx, uint64_t key, uint64_t start, size_t count, int kind, void* out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        if (kind < 0 || kind > 3) throw contract_error("hcva_rng_draw: kind must be 0..3");
        HCVA_CUDA(cudaSetDevice(ctx->device));
        DeviceBuf buf;
        buf.alloc(count * 8);
        if (count) {
            k_draws<<<grid1(count, 256), 256, 0, ctx->stream>>>(key, start, count, kind, buf.p);
            check_launch(ctx);
            copy_out(ctx, out, buf.p, count * 8);
        }
    });
}

hcva_status hcva_simulate_set(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                              const hcva_swap* book, int n_swaps, int n_paths, int path_offset,
                              int n_replicas, uint64_t key_market, uint64_t key_defaults, hcva_sim** out) {
    return hcva_simulate_set_sharded(ctx, model, grid, book, n_swaps, n_paths, path_offset, 0, 0, n_replicas,
                                     key_market, key_defaults, out);
}

hcva_status hcva_simulate_set_sharded(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                                      const hcva_swap* book, int n_swaps, int n_paths, int path_offset,
                                      int shard_blk, int shard_stride, int n_replicas, uint64_t key_market,
                                      uint64_t key_defaults, hcva_sim** out) {
    return guarded([&] {
        NvtxRange nvtx__("hcva_simulate_set");
        StreamScope sc__(ctx->stream);
        if (!grid) throw contract_error("simulate_set: null grid");
        if (n_paths < 1) throw contract_error("simulate_market: n_paths must be >= 1");
        if (path_offset < 0) throw contract_error("simulate_set: negative path offset");
        if (shard_blk < 0 || (shard_blk > 0 && (shard_stride < shard_blk || n_paths % shard_blk != 0)))
            throw contract_error("simulate_set: shard map needs 0 < blk <= stride and blk | n_paths");
        std::unique_ptr<hcva_sim> sim(new_sim(ctx, model, grid));
        const Model& m = sim->model;
        sim->M = n_paths;
        sim->n = m.n_steps;
        sim->path_offset = path_offset;
        sim->shard_blk = shard_blk;
        sim->shard_stride = shard_stride;
        std::vector<double> init(m.D);
        for (int e = 0; e < m.E; ++e) init[e] = m.rates[e].r0;
        for (int e = 1; e < m.E; ++e) init[m.E + e - 1] = std::log(m.fx[e - 1].chi0);
        for (int c = 0; c < m.Cn; ++c) init[2 * m.E - 1 + c] = m.credit[c].gamma0;
        std::vector<double> lag0(m.E);
        for (int e = 0; e < m.E; ++e) lag0[e] = m.rates[e].r0;
        stage(sim->lag0, lag0);
        prepare_market(sim.get(), {key_market}, init, n_paths, static_cast<uint64_t>(path_offset));
        if (n_replicas > 0) prepare_defaults(sim.get(), n_replicas);
        if (book) prepare_cube(sim.get(), book, n_swaps);
        launch_market(sim.get(), key_market);
        if (n_replicas > 0) launch_defaults(sim.get(), key_defaults);
        if (book) launch_cube(sim.get());
        HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = sim.release();
    });
}

hcva_status hcva_sim_rerun(hcva_sim* sim, uint64_t key_market, uint64_t key_defaults, int labels_kind,
                           int event_slot) {
    return guarded([&] {
        NvtxRange nvtx__("hcva_sim_rerun");
        StreamScope sc__(sim->ctx->stream);
        if (sim->start_step != 0 || sim->n_groups != 1) throw contract_error("rerun: outer blocks only");
        if (!sim->m_coef.p) throw contract_error("rerun: the set was loaded, not simulated");
        HCVA_CUDA(cudaSetDevice(sim->ctx->device));
        record(sim, event_slot, 0);
        launch_market(sim, key_market);
        record(sim, event_slot, 1);
        if (sim->N > 0) launch_defaults(sim, key_defaults);
        record(sim, event_slot, 2);
        if (sim->c_nswaps > 0) launch_cube(sim);
        record(sim, event_slot, 3);
        if (labels_kind >= 0) launch_labels_all(sim, labels_kind);
        record(sim, event_slot, 4);
    });
}

hcva_status hcva_sim_phase_times(hcva_sim* sim, int event_slot, float* ms) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        const size_t base = static_cast<size_t>(event_slot) * 5;
        if (event_slot < 0 || base + 4 >= sim->events.size()) throw contract_error("phase times: no such slot");
        for (int p = 0; p < 4; ++p)
            HCVA_CUDA(cudaEventElapsedTime(&ms[p], sim->events[base + p], sim->events[base + p + 1]));
    });
}

hcva_status hcva_simulate_conditional(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                                      const double* st_rates, const double* st_logfx, const double* st_intens,
                                      const double* st_lagged, int start_step, int horizon, int n_inner,
                                      uint64_t key, hcva_sim** out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        if (!grid) throw contract_error("simulate_conditional_market: null grid");
        std::unique_ptr<hcva_sim> sim(new_sim(ctx, model, grid));
        const Model& m = sim->model;
        if (horizon < 0 || start_step < 0 || start_step + horizon > m.n_steps)
            throw contract_error("simulate_conditional_market: horizon out of range");
        if (n_inner < 1) throw contract_error("simulate_conditional_market: n_inner must be >= 1");
        sim->M = n_inner;
        sim->n = horizon;
        sim->start_step = start_step;
        std::vector<double> init(m.D);
        for (int e = 0; e < m.E; ++e) init[e] = st_rates[e];
        for (int e = 1; e < m.E; ++e) init[m.E + e - 1] = st_logfx[e - 1];
        for (int c = 0; c < m.Cn; ++c) init[2 * m.E - 1 + c] = st_intens[c];
        stage(sim->lag0, std::vector<double>(st_lagged, st_lagged + m.E));
        prepare_market(sim.get(), {key}, init, n_inner, 0);
        launch_market(sim.get(), key);
        HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = sim.release();
    });
}

hcva_status hcva_sample_defaults(hcva_sim* sim, int n_replicas, uint64_t key) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        HCVA_CUDA(cudaSetDevice(sim->ctx->device));
        prepare_defaults(sim, n_replicas);
        launch_defaults(sim, key);
        HCVA_CUDA(cudaStreamSynchronize(sim->ctx->stream));
    });
}

hcva_status hcva_probe_block(hcva_sim* sim, uint64_t key, int label_kind, uint16_t* steps_out, double* labels_out) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        HCVA_CUDA(cudaSetDevice(sim->ctx->device));
        if (label_kind != 0 && label_kind != 1) throw config_error("config: label_kind must be 'defaults' or 'intensity'");
        DeviceBuf st, lab;
        probe_block(sim, key, label_kind, st, lab);
        const size_t R2 = static_cast<size_t>(sim->M) * 2, Cn = sim->model.Cn;
        if (steps_out) {
            std::vector<uint16_t> soa(R2 * Cn);
            copy_out(sim->ctx, soa.data(), st.p, soa.size() * 2);
            for (size_t r = 0; r < R2; ++r)
                for (size_t c = 0; c < Cn; ++c) steps_out[r * Cn + c] = soa[c * R2 + r];
        }
        if (labels_out) copy_out(sim->ctx, labels_out, lab.p, R2 * (sim->n + 1) * 8);
    });
}

hcva_status hcva_build_cube(hcva_sim* sim, const hcva_swap* book, int n_swaps) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        HCVA_CUDA(cudaSetDevice(sim->ctx->device));
        prepare_cube(sim, book, n_swaps);
        launch_cube(sim);
        HCVA_CUDA(cudaStreamSynchronize(sim->ctx->stream));
    });
}

hcva_status hcva_sim_destroy(hcva_sim* sim) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        if (!sim) return;
        cudaSetDevice(sim->ctx->device);
        cudaStreamSynchronize(sim->ctx->stream);
        delete sim;
    });
}

hcva_status hcva_sim_dims(const hcva_sim* sim, int* dims) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        dims[0] = sim->M; dims[1] = sim->n; dims[2] = sim->model.E; dims[3] = sim->model.Cn;
        dims[4] = sim->N; dims[5] = sim->start_step; dims[6] = sim->model.D; dims[7] = sim->model.substeps;
    });
}

hcva_status hcva_sim_tie_counts(const hcva_sim* sim, uint64_t* counts) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        if (!sim->has_defaults) throw contract_error("tie counts: no default block");
        unsigned long long h[2];
        copy_out(sim->ctx, h, sim->ties.p, sizeof h);
        counts[0] = h[0];
        counts[1] = h[1];
    });
}

hcva_status hcva_sim_export_market(const hcva_sim* sim, double* rates, double* fx, double* intens,
                                   double* lagged, double* disc, double* hazard) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        hcva_ctx* ctx = sim->ctx;
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const Model& m = sim->model;
        const int n1 = sim->n + 1, M = sim->M, ppg = M / sim->n_groups;
        DeviceBuf tmp;
        auto conv = [&](const double* src, double* dst, int F, int mode) {
            if (!dst || F == 0) return;
            const size_t cnt = static_cast<size_t>(M) * n1 * F;
            tmp.alloc(cnt * sizeof(double));
            k_soa_to_aos<<<grid1(cnt, 256), 256, 0, ctx->stream>>>(src, tmp.as<double>(), M, n1, F, mode,
                                                                   sim->lag0.as<double>(), m.E, ppg);
            check_launch(ctx);
            copy_out(ctx, dst, tmp.p, cnt * sizeof(double));
        };
        conv(sim->rates.as<double>(), rates, m.E, 0);
        conv(sim->fx.as<double>(), fx, m.E - 1, 0);
        conv(sim->intens.as<double>(), intens, m.Cn, 0);
        conv(sim->rates.as<double>(), lagged, m.E, 1);
        conv(sim->disc.as<double>(), disc, 1, 0);
        conv(sim->hazard.as<double>(), hazard, m.Cn, 0);
    });
}

hcva_status hcva_sim_export_defaults(const hcva_sim* sim, uint16_t* steps) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        if (!sim->has_defaults) throw contract_error("export: no default block");
        hcva_ctx* ctx = sim->ctx;
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const size_t R = static_cast<size_t>(sim->M) * sim->N, cnt = R * sim->model.Cn;
        DeviceBuf tmp;
        tmp.alloc(cnt * sizeof(uint16_t));
        k_steps_to_aos<<<grid1(cnt, 256), 256, 0, ctx->stream>>>(sim->steps.as<uint16_t>(), tmp.as<uint16_t>(), R,
                                                                 sim->model.Cn);
        check_launch(ctx);
        copy_out(ctx, steps, tmp.p, cnt * sizeof(uint16_t));
    });
}

hcva_status hcva_sim_export_cube(const hcva_sim* sim, double* cube) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        if (!sim->has_cube) throw contract_error("export: no MtM cube");
        hcva_ctx* ctx = sim->ctx;
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const int n1 = sim->n + 1, M = sim->M, Cc = sim->model.Cc;
        const size_t cnt = static_cast<size_t>(M) * n1 * Cc;
        DeviceBuf tmp;
        tmp.alloc(cnt * sizeof(double));
        k_soa_to_aos<<<grid1(cnt, 256), 256, 0, ctx->stream>>>(sim->cube.as<double>(), tmp.as<double>(), M, n1, Cc, 0,
                                                               nullptr, 0, 1);
        check_launch(ctx);
        copy_out(ctx, cube, tmp.p, cnt * sizeof(double));
    });
}

hcva_status hcva_labels(hcva_sim* sim, int step, int kind, double* out) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        if (kind != 0 && kind != 1) throw config_error("label_kind must be 'defaults' or 'intensity'");
        HCVA_CUDA(cudaSetDevice(sim->ctx->device));
        const size_t R = static_cast<size_t>(sim->M) * sim->N;
        DeviceBuf tmp;
        tmp.alloc(R * sizeof(double));
        launch_labels(sim, kind, step, step, tmp.as<double>());
        copy_out(sim->ctx, out, tmp.p, R * sizeof(double));
    });
}

hcva_status hcva_labels_all(hcva_sim* sim, int kind, double* out) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        if (kind != 0 && kind != 1) throw config_error("label_kind must be 'defaults' or 'intensity'");
        HCVA_CUDA(cudaSetDevice(sim->ctx->device));
        launch_labels_all(sim, kind);
        if (out) copy_out(sim->ctx, out, sim->labels.p, sim->labels.bytes);
    });
}

hcva_status hcva_cva_profile(hcva_sim* sim, int kind, double* out) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        if (kind != 0 && kind != 1) throw config_error("label_kind must be 'defaults' or 'intensity'");
        HCVA_CUDA(cudaSetDevice(sim->ctx->device));
        const size_t R = static_cast<size_t>(sim->M) * sim->N;
        if (!sim->profile.p) sim->profile.alloc(sizeof(double) * (sim->n + 1));
        const int Cc = sim->model.Cc, n1 = sim->n + 1;
        if (kind == 0 && Cc < 255 && sim->labels_kind != kind) {  // fused: no label array
            if (!sim->has_cube) throw contract_error("labels: no MtM cube");
            if (!sim->has_defaults) throw contract_error("labels: no default block");
            if (sim->start_step != 0) throw contract_error("labels expect an outer (non-rebased) market block");
            LabelArgs a{};
            a.M = sim->M; a.N = sim->N; a.n = sim->n; a.Cn = sim->model.Cn; a.E = sim->model.E; a.dt = sim->model.dt;
            a.disc = sim->disc.as<double>(); a.cube = sim->cube.as<double>(); a.steps = sim->steps.as<uint16_t>();
            a.i0 = 0; a.i1 = sim->n;
            DeviceBuf part;
            part.alloc(sizeof(double) * n1 * sim->M);
            const size_t smem = Cc <= 16 ? sizeof(double) * (2 * n1 + static_cast<size_t>(n1) * Cc + 4 * n1)
                                         : sweep_smem(n1, Cc, 128, true);
            const void* fn = Cc <= 8    ? (const void*)k_profile_defaults<8>
                             : Cc <= 16 ? (const void*)k_profile_defaults<16>
                                        : (const void*)k_labels_defaults_sweep<true>;
            if (smem > 48 * 1024)
                HCVA_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            double* pp = part.as<double>();
            void* args[] = {&a, &pp};
            HCVA_CUDA(cudaLaunchKernel(fn, dim3(sim->M), dim3(128), args, smem, sim->ctx->stream));
            check_launch(sim->ctx);
            k_profile_paths<<<n1, 256, 0, sim->ctx->stream>>>(pp, sim->M, static_cast<double>(R),
                                                              sim->profile.as<double>());
            check_launch(sim->ctx);
            copy_out(sim->ctx, out, sim->profile.p, sizeof(double) * n1);
            return;
        }
        if (sim->labels_kind != kind) launch_labels_all(sim, kind);
        k_profile<<<sim->n + 1, 256, 0, sim->ctx->stream>>>(sim->labels.as<double>(), R, sim->profile.as<double>());
        check_launch(sim->ctx);
        copy_out(sim->ctx, out, sim->profile.p, sizeof(double) * (sim->n + 1));
    });
}

hcva_status hcva_features(hcva_sim* sim, int step, double* out) {
    return guarded([&] {
        StreamScope sc__(sim->ctx->stream);
        if (!sim->has_defaults) throw contract_error("features: no default block");
        if (step < 0 || step > sim->n) throw contract_error("label step out of range");
        if (sim->start_step != 0) throw contract_error("labels expect an outer (non-rebased) market block");
        hcva_ctx* ctx = sim->ctx;
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const Model& m = sim->model;
        const size_t R = static_cast<size_t>(sim->M) * sim->N;
        const int cols = (m.Cn - 1) + m.E + (m.E - 1) + (m.Cn - 1) + m.E;
        DeviceBuf tmp;
        tmp.alloc(R * cols * sizeof(double));
        FeatureArgs a{};
        a.M = sim->M; a.N = sim->N; a.n = sim->n; a.Cn = m.Cn; a.E = m.E; a.step = step;
        a.paths_per_group = sim->M / sim->n_groups;
        a.rates = sim->rates.as<double>(); a.fx = sim->fx.as<double>(); a.intens = sim->intens.as<double>();
        a.lag0 = sim->lag0.as<double>(); a.steps = sim->steps.as<uint16_t>(); a.out = tmp.as<double>();
        k_features<<<grid1(R, 128), 128, 0, ctx->stream>>>(a);
        check_launch(ctx);
        copy_out(ctx, out, tmp.p, R * cols * sizeof(double));
    });
}

// ---- HCVAMKT1 market dumps (save_market / load_market, pipeline.cpp:371-442):
// magic, u32 version 1, u64 seed, i32 paths, steps, economies, credit names,
// start step, f64 dt, i32 substeps, then per (k, i): rates[E], fx[E-1],
// intensities[Cn], lagged[E], discount, hazards[Cn] (f64).
}  // extern "C"

namespace {
constexpr char kMarketMagic[8] = {'H', 'C', 'V', 'A', 'M', 'K', 'T', '1'};
template <typename T>
void mput(std::ofstream& o, T v) {
    o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T mget(std::ifstream& in) {
    T v;
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) throw numeric_error("market dump truncated");
    return v;
}
}  // namespace

extern "C" {

hcva_status hcva_sim_save_market(const hcva_sim* sim, const char* path, uint64_t seed) {
    return guarded([&] {
        const Model& m = sim->model;
        const int M = sim->M, n1 = sim->n + 1, E = m.E, Cn = m.Cn;
        const size_t rows = static_cast<size_t>(M) * n1;
        std::vector<double> r(rows * E), f(rows * std::max(E - 1, 1)), g(rows * Cn), lg(rows * E), d(rows),
            hz(rows * Cn);
        const hcva_status st = hcva_sim_export_market(sim, r.data(), E > 1 ? f.data() : nullptr, g.data(), lg.data(),
                                                      d.data(), hz.data());
        if (st != HCVA_OK) throw contract_error(hcva_last_error());
        std::ofstream o(path, std::ios::binary);
        if (!o) throw config_error(std::string("cannot write ") + path);
        o.write(kMarketMagic, 8);
        mput<uint32_t>(o, 1u);
        mput<uint64_t>(o, seed);
        mput<int32_t>(o, M);
        mput<int32_t>(o, sim->n);
        mput<int32_t>(o, E);
        mput<int32_t>(o, Cn);
        mput<int32_t>(o, sim->start_step);
        mput<double>(o, m.dt);
        mput<int32_t>(o, m.substeps);
        for (size_t row = 0; row < rows; ++row) {
            for (int e = 0; e < E; ++e) mput(o, r[row * E + e]);
            for (int e = 1; e < E; ++e) mput(o, f[row * (E - 1) + e - 1]);
            for (int c = 0; c < Cn; ++c) mput(o, g[row * Cn + c]);
            for (int e = 0; e < E; ++e) mput(o, lg[row * E + e]);
            mput(o, d[row]);
            for (int c = 0; c < Cn; ++c) mput(o, hz[row * Cn + c]);
        }
        if (!o) throw config_error(std::string("cannot write ") + path);
    });
}

hcva_status hcva_market_load(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid, const char* path,
                             uint64_t* seed, hcva_sim** out) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        std::unique_ptr<hcva_sim> sim(new_sim(ctx, model, grid));
        const Model& m = sim->model;
        std::ifstream in(path, std::ios::binary);
        if (!in) throw config_error(std::string("cannot open ") + path);
        char magic[8];
        in.read(magic, 8);
        if (!in || std::memcmp(magic, kMarketMagic, 8) != 0) throw config_error(std::string("not a market dump: ") + path);
        if (mget<uint32_t>(in) != 1u) throw config_error("unsupported market dump version");
        const uint64_t sd = mget<uint64_t>(in);
        const int M = mget<int32_t>(in), n = mget<int32_t>(in), E = mget<int32_t>(in), Cn = mget<int32_t>(in);
        const int start = mget<int32_t>(in);
        const double dt = mget<double>(in);
        const int substeps = mget<int32_t>(in);
        if (E != m.E || Cn != m.Cn) throw contract_error("market dump: economies / credit names differ from the model");
        if (n != m.n_steps || dt != m.dt || substeps != m.substeps)
            throw contract_error("market dump: time grid differs from the model's");
        if (start != 0) throw contract_error("market dump: only outer (start step 0) blocks load into a set");
        if (M < 1) throw contract_error("market dump: no paths");
        const int n1 = n + 1;
        const size_t Ms = M;
        std::vector<double> r(static_cast<size_t>(n1) * E * Ms), f(static_cast<size_t>(n1) * std::max(E - 1, 1) * Ms),
            g(static_cast<size_t>(n1) * Cn * Ms), hz(g.size()), d(static_cast<size_t>(n1) * Ms), lag0(E);
        std::vector<double> lg(E);
        for (int k = 0; k < M; ++k)
            for (int i = 0; i < n1; ++i) {
                for (int e = 0; e < E; ++e) r[(static_cast<size_t>(i) * E + e) * Ms + k] = mget<double>(in);
                for (int e = 1; e < E; ++e) f[(static_cast<size_t>(i) * (E - 1) + e - 1) * Ms + k] = mget<double>(in);
                for (int c = 0; c < Cn; ++c) g[(static_cast<size_t>(i) * Cn + c) * Ms + k] = mget<double>(in);
                for (int e = 0; e < E; ++e) lg[e] = mget<double>(in);
                d[static_cast<size_t>(i) * Ms + k] = mget<double>(in);
                for (int c = 0; c < Cn; ++c) hz[(static_cast<size_t>(i) * Cn + c) * Ms + k] = mget<double>(in);
                // Lagged rates are derived here (market.cpp:186-195): the dump's must agree.
                for (int e = 0; e < E; ++e) {
                    const double want = (i == 0) ? ((k == 0) ? (lag0[e] = lg[e]) : lag0[e])
                                                 : r[(static_cast<size_t>(i - 1) * E + e) * Ms + k];
                    if (lg[e] != want)
                        throw contract_error("market dump: lagged rates do not follow the simulated layout");
                }
            }
        sim->M = M;
        sim->n = n;
        sim->start_step = 0;
        stage(sim->rates, r);
        stage(sim->fx, f);
        stage(sim->intens, g);
        stage(sim->hazard, hz);
        stage(sim->disc, d);
        stage(sim->lag0, lag0);
        HCVA_CUDA(cudaStreamSynchronize(ctx->stream));
        if (seed) *seed = sd;
        *out = sim.release();
    });
}

}  // extern "C"
