// nested.cu -- K6: batched nested Monte Carlo CVA benchmark (validation.cpp:123-179).
//
// For S outer states at pricing step i the reference calls nested_cva once per
// state inside a parallel_for (pipeline.cpp:285-292): n_inner conditional
// market continuations from the frozen Y-state (market.cpp:236-310), their MtM
// cube (portfolio.cpp:97-147 with start_step = i), and the intensity-form
// payoff over the clients that survived to i.  Here every (state, inner path)
// pair is one path of a single K1 launch (group = state: its own key
// parent.split(s), initial state and lagged rates), K2 prices the conditional
// cube, and K6 computes the payoff per inner path and the per-state mean and
// standard error in the reference's summation order.  States are processed in
// batches sized to a memory budget.
#include <algorithm>
#include <cmath>
#include <memory>

#include "common.cuh"
#include "rng.cuh"

namespace hcva {

struct NestedArgs {
    int M, h, Cn, L;  // paths in batch, horizon, names, inner paths per state
    double dt;
    const double* disc;    // [j*M + k]
    const double* intens;  // [(j*Cn + c)*M + k]
    const double* cube;    // [(j*Cc + c-1)*M + k]
    const int* survived;   // [state][Cc]
    double* payoff;        // [k]
};

// Payoff of inner path k (validation.cpp:139-160): clients ascending, steps
// ascending, sum_j beta_j (MtM_j)^+ gamma_j dt exp(-sum_{s<j} gamma_s dt).
__global__ void k_nested_payoff(NestedArgs a) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.M) return;
    const int s = k / a.L, Cc = a.Cn - 1, M = a.M;
    double payoff = 0.0;
    for (int c = 1; c <= Cc; ++c) {
        if (!a.survived[s * Cc + c - 1]) continue;
        double gsum = 0.0;
        for (int j = 0; j <= a.h - 1; ++j) {
            const double mtm = a.cube[(static_cast<size_t>(j) * Cc + c - 1) * M + k];
            const double expo = (mtm < 0.0) ? 0.0 : mtm;
            const double g = a.intens[(static_cast<size_t>(j) * a.Cn + c) * M + k];
            const double term = __dmul_rn(__dmul_rn(__dmul_rn(a.disc[static_cast<size_t>(j) * M + k], expo), g), a.dt);
            payoff = __dadd_rn(payoff, __dmul_rn(term, exp(-gsum)));
            gsum = __dadd_rn(gsum, __dmul_rn(g, a.dt));
        }
    }
    a.payoff[k] = payoff;
}

// Per-state mean and standard error over its L inner payoffs, summed in inner
// index order as the reference does (validation.cpp:157-176).
__global__ void k_nested_reduce(const double* payoff, int S, int L, const int* any, double* value, double* se) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    if (!any[s]) {
        value[s] = 0.0;
        se[s] = 0.0;
        return;
    }
    double sum = 0.0, sum_sq = 0.0;
    for (int l = 0; l < L; ++l) {
        const double p = payoff[static_cast<size_t>(s) * L + l];
        sum = __dadd_rn(sum, p);
        sum_sq = __dadd_rn(sum_sq, __dmul_rn(p, p));
    }
    const double m = sum / L;
    value[s] = m;
    double e = 0.0;
    if (L > 1) {
        const double var = (sum_sq - L * m * m) / (L - 1);
        e = sqrt((var > 0.0 ? var : 0.0) / L);
    }
    se[s] = e;
}

// ------------------------------------------------------------------ twin MC
// twin_labels (labels.cpp:90-140): outer path k (batch-local s) has two
// continuation paths 2s, 2s+1 in the conditional block (group s, key
// split(k).split(0)).  Thread per (s, l): for twin t the surviving clients
// redraw their default on continuation t with resample_continuation
// (defaults.cpp:47-57) -- one Exp(1) per survivor, in client order, from
// split(k).split(1).split(l).split(t) -- found by binary search over the
// nondecreasing continuation hazard (the reference's linear scan), and the
// label sums discount x positive exposure at the hit step in client order.
struct TwinArgs {
    int S, N, h, Cn, step, k0, Mc;
    size_t R;               // outer rows M*N
    uint64_t key;
    const uint16_t* steps;  // outer default steps [c][k*N + l]
    const double* hazard;   // continuation [(j*Cn + c)*Mc + kk]
    const double* disc;     // [j*Mc + kk]
    const double* cube;     // [(j*Cc + c-1)*Mc + kk]
    double* t1;             // [s*N + l] (batch rows)
    double* t2;
};

__global__ void k_twin(TwinArgs a) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= a.S * a.N) return;
    const int s = idx / a.N, l = idx % a.N, k = a.k0 + s;
    const int Cc = a.Cn - 1, Mc = a.Mc, h = a.h;
    const uint64_t rkey = split_key(split_key(split_key(a.key, static_cast<uint64_t>(k)), 1), static_cast<uint64_t>(l));
    const size_t orow = static_cast<size_t>(k) * a.N + l;
    for (int t = 0; t < 2; ++t) {
        const uint64_t tkey = split_key(rkey, static_cast<uint64_t>(t));
        const int kk = 2 * s + t;
        uint64_t draw = 0;
        double sum = 0.0;
        for (int c = 1; c <= Cc; ++c) {
            if (a.steps[c * a.R + orow] <= a.step) continue;  // stays defaulted
            const double eps = -log(u64_to_uniform(draw_u64(tkey, draw++)));
            const double base = a.hazard[static_cast<size_t>(c) * Mc + kk];
            int lo = 1, hi = h + 1;  // first j in [1, h] with H_j - base >= eps, h+1 if none
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (a.hazard[(static_cast<size_t>(mid) * a.Cn + c) * Mc + kk] - base >= eps) hi = mid;
                else lo = mid + 1;
            }
            if (lo <= h) {
                const double mtm = a.cube[(static_cast<size_t>(lo) * Cc + c - 1) * Mc + kk];
                const double expo = (mtm < 0.0) ? 0.0 : mtm;
                sum = __dadd_rn(sum, __dmul_rn(a.disc[static_cast<size_t>(lo) * Mc + kk], expo));
            }
        }
        (t == 0 ? a.t1 : a.t2)[static_cast<size_t>(s) * a.N + l] = sum;
    }
}

}  // namespace hcva

using namespace hcva;

extern "C" hcva_status hcva_nested_cva_range(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                                             const hcva_swap* book, int n_swaps, const double* states,
                                             const int* survived, int n_states, int first_state, int step,
                                             int inner, uint64_t parent_key, double* value, double* std_error) {
    return guarded([&] {
        NvtxRange nvtx__("hcva_nested_cva");
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (inner < 1) throw contract_error("nested_cva: inner_count must be >= 1");
        if (first_state < 0) throw contract_error("nested_cva: negative first state");
        if (!grid) throw contract_error("nested_cva: null grid");
        const Model probe = make_model(model, grid);
        const int E = probe.E, Cn = probe.Cn, Cc = probe.Cc, D = probe.D;
        const int h = grid->n_steps - step;
        if (step < 0 || h < 0) throw contract_error("simulate_conditional_market: horizon out of range");
        const int stride = 3 * E - 1 + Cn;  // rates[E], log_fx[E-1], intens[Cn], lagged[E]
        std::vector<double> val(n_states, 0.0), err(n_states, 0.0);
        if (h == 0 || n_states == 0) {
            std::copy(val.begin(), val.end(), value);
            std::copy(err.begin(), err.end(), std_error);
            return;
        }
        // Batch size: per path (h+1) steps x (E + E-1 + 2Cn + 1 + Cc) doubles.
        const double per_state = static_cast<double>(inner) * (h + 1) * (3 * E + 2 * Cn + Cc) * 8.0;
        const int batch = std::max(1, std::min(n_states, static_cast<int>(12e9 / per_state)));
        for (int s0 = 0; s0 < n_states; s0 += batch) {
            const int S = std::min(batch, n_states - s0);
            std::unique_ptr<hcva_sim> sim(new_sim(ctx, model, grid));
            sim->M = S * inner;
            sim->n = h;
            sim->start_step = step;
            sim->n_groups = S;
            std::vector<uint64_t> keys(S);
            std::vector<double> init(static_cast<size_t>(S) * D), lag(static_cast<size_t>(S) * E);
            std::vector<int> surv(static_cast<size_t>(S) * Cc), any(S, 0);
            for (int s = 0; s < S; ++s) {
                const double* st = states + static_cast<size_t>(s0 + s) * stride;
                keys[s] = split_key(parent_key, static_cast<uint64_t>(first_state + s0 + s));
                for (int e = 0; e < E; ++e) init[s * D + e] = st[e];
                for (int e = 1; e < E; ++e) init[s * D + E + e - 1] = st[E + e - 1];
                for (int c = 0; c < Cn; ++c) init[s * D + 2 * E - 1 + c] = st[2 * E - 1 + c];
                for (int e = 0; e < E; ++e) lag[s * E + e] = st[2 * E - 1 + Cn + e];
                for (int c = 0; c < Cc; ++c) {
                    surv[s * Cc + c] = survived[static_cast<size_t>(s0 + s) * Cc + c] != 0;
                    any[s] |= surv[s * Cc + c];
                }
            }
            stage(sim->lag0, lag);
            if (S == 1) {
                prepare_market(sim.get(), {}, init, inner, 0);
                launch_market(sim.get(), keys[0]);
            } else {
                prepare_market(sim.get(), keys, init, inner, 0);
                launch_market(sim.get(), 0);
            }
            prepare_cube(sim.get(), book, n_swaps);
            launch_cube(sim.get());
            DeviceBuf d_surv, d_any, d_pay, d_val, d_se;
            stage(d_surv, surv);
            stage(d_any, any);
            d_pay.alloc(sizeof(double) * sim->M);
            d_val.alloc(sizeof(double) * S);
            d_se.alloc(sizeof(double) * S);
            NestedArgs a{};
            a.M = sim->M; a.h = h; a.Cn = Cn; a.L = inner; a.dt = grid->dt;
            a.disc = sim->disc.as<double>(); a.intens = sim->intens.as<double>(); a.cube = sim->cube.as<double>();
            a.survived = d_surv.as<int>(); a.payoff = d_pay.as<double>();
            k_nested_payoff<<<grid1(sim->M, 128), 128, 0, ctx->stream>>>(a);
            check_launch(ctx);
            k_nested_reduce<<<grid1(S, 128), 128, 0, ctx->stream>>>(d_pay.as<double>(), S, inner, d_any.as<int>(),
                                                                   d_val.as<double>(), d_se.as<double>());
            check_launch(ctx);
            copy_out(ctx, val.data() + s0, d_val.p, sizeof(double) * S);
            copy_out(ctx, err.data() + s0, d_se.p, sizeof(double) * S);
        }
        std::copy(val.begin(), val.end(), value);
        std::copy(err.begin(), err.end(), std_error);
    });
}

extern "C" hcva_status hcva_nested_cva_batch(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                                             const hcva_swap* book, int n_swaps, const double* states,
                                             const int* survived, int n_states, int step, int inner,
                                             uint64_t parent_key, double* value, double* std_error) {
    return hcva_nested_cva_range(ctx, model, grid, book, n_swaps, states, survived, n_states, 0, step, inner,
                                 parent_key, value, std_error);
}

extern "C" hcva_status hcva_twin_labels(hcva_sim* outer, const hcva_swap* book, int n_swaps, int step, uint64_t key,
                                        double* twin1, double* twin2) {
    return guarded([&] {
        NvtxRange nvtx__("hcva_twin_labels");
        hcva_ctx* ctx = outer->ctx;
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (!outer->has_defaults) throw contract_error("twin_labels: simulate a default block first");
        if (outer->start_step != 0) throw contract_error("labels expect an outer (non-rebased) market block");
        const Model& m = outer->model;
        const int E = m.E, Cn = m.Cn, Cc = m.Cc, D = m.D, M = outer->M, N = outer->N, n = outer->n;
        if (step < 0 || step > n) throw contract_error("labels: step outside the simulated grid");
        const size_t R = static_cast<size_t>(M) * N;
        const int h = n - step;
        if (h == 0) {
            std::fill(twin1, twin1 + R, 0.0);
            std::fill(twin2, twin2 + R, 0.0);
            return;
        }
        // state_at(k, step) (market.cpp:100-113) on the host: log of the stored FX
        // with the host libm, as the reference does.
        std::vector<double> r(static_cast<size_t>(E) * M), f(static_cast<size_t>(std::max(E - 1, 1)) * M),
            g(static_cast<size_t>(Cn) * M), lag(static_cast<size_t>(E) * M);
        copy_out(ctx, r.data(), outer->rates.as<double>() + static_cast<size_t>(step) * E * M, sizeof(double) * E * M);
        if (E > 1)
            copy_out(ctx, f.data(), outer->fx.as<double>() + static_cast<size_t>(step) * (E - 1) * M,
                     sizeof(double) * (E - 1) * M);
        copy_out(ctx, g.data(), outer->intens.as<double>() + static_cast<size_t>(step) * Cn * M,
                 sizeof(double) * Cn * M);
        if (step > 0) {
            copy_out(ctx, lag.data(), outer->rates.as<double>() + static_cast<size_t>(step - 1) * E * M,
                     sizeof(double) * E * M);
        } else {
            std::vector<double> l0(E);
            copy_out(ctx, l0.data(), outer->lag0.as<double>(), sizeof(double) * E);
            for (int e = 0; e < E; ++e)
                for (int k = 0; k < M; ++k) lag[static_cast<size_t>(e) * M + k] = l0[e];
        }
        // Batches of outer paths by memory: 2 continuations x (h+1) steps x (3E + 2Cn + Cc) doubles.
        const double per_path = 2.0 * (h + 1) * (3 * E + 2 * Cn + Cc) * 8.0;
        const int batch = std::max(1, std::min(M, static_cast<int>(12e9 / per_path)));
        for (int k0 = 0; k0 < M; k0 += batch) {
            const int S = std::min(batch, M - k0);
            std::unique_ptr<hcva_sim> sim(new_sim(ctx, m));
            sim->M = 2 * S;
            sim->n = h;
            sim->start_step = step;
            sim->n_groups = S;
            std::vector<uint64_t> keys(S);
            std::vector<double> init(static_cast<size_t>(S) * D), lg(static_cast<size_t>(S) * E);
            for (int s = 0; s < S; ++s) {
                const int k = k0 + s;
                keys[s] = split_key(split_key(key, static_cast<uint64_t>(k)), 0);
                for (int e = 0; e < E; ++e) init[s * D + e] = r[static_cast<size_t>(e) * M + k];
                for (int e = 1; e < E; ++e) init[s * D + E + e - 1] = std::log(f[static_cast<size_t>(e - 1) * M + k]);
                for (int c = 0; c < Cn; ++c) init[s * D + 2 * E - 1 + c] = g[static_cast<size_t>(c) * M + k];
                for (int e = 0; e < E; ++e) lg[s * E + e] = lag[static_cast<size_t>(e) * M + k];
            }
            stage(sim->lag0, lg);
            if (S == 1) {
                prepare_market(sim.get(), {}, init, 2, 0);
                launch_market(sim.get(), keys[0]);
            } else {
                prepare_market(sim.get(), keys, init, 2, 0);
                launch_market(sim.get(), 0);
            }
            prepare_cube(sim.get(), book, n_swaps);
            launch_cube(sim.get());
            DeviceBuf d1, d2;
            d1.alloc(sizeof(double) * S * N);
            d2.alloc(sizeof(double) * S * N);
            TwinArgs a{};
            a.S = S; a.N = N; a.h = h; a.Cn = Cn; a.step = step; a.k0 = k0; a.Mc = 2 * S; a.R = R; a.key = key;
            a.steps = outer->steps.as<uint16_t>(); a.hazard = sim->hazard.as<double>();
            a.disc = sim->disc.as<double>(); a.cube = sim->cube.as<double>();
            a.t1 = d1.as<double>(); a.t2 = d2.as<double>();
            k_twin<<<grid1(static_cast<size_t>(S) * N, 128), 128, 0, ctx->stream>>>(a);
            check_launch(ctx);
            copy_out(ctx, twin1 + static_cast<size_t>(k0) * N, d1.p, sizeof(double) * S * N);
            copy_out(ctx, twin2 + static_cast<size_t>(k0) * N, d2.p, sizeof(double) * S * N);
        }
    });
}
