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

}  // namespace hcva

using namespace hcva;

extern "C" hcva_status hcva_nested_cva_batch(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                                             const hcva_swap* book, int n_swaps, const double* states,
                                             const int* survived, int n_states, int step, int inner,
                                             uint64_t parent_key, double* value, double* std_error) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        if (inner < 1) throw contract_error("nested_cva: inner_count must be >= 1");
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
                keys[s] = split_key(parent_key, static_cast<uint64_t>(s0 + s));
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
