// ard.cu -- ARD variance sampling (ard.cpp:56-125) on the GPU, SURVEY §8(f) f4.
//
// n_dgp draws of the DGP parameters from a multiplicative uniform prior
// (perturb, ard.cpp:20-35, drawn on the host from stream.split(0) with
// rejection of draws that fail ModelParams::validate), then per draw the same
// engine as the training set -- K1 / K3 (one replica) / K2 / K4 for every
// pricing step, keys stream.split(1).split(d) -- and the time-averaged
// cross-path variances (1/(n+1)) sum_i Var_k(.) of every default indicator,
// rate, FX rate, client intensity and of the defaults label.  The variance
// kernels sum over paths in path order without contraction, as the
// reference's loops (time_averaged_variance, ard.cpp:37-52).
#include <memory>
#include <vector>

#include "common.cuh"
#include "rng.cuh"

namespace hcva {

// out[i] = sum_k (v(k,i) - m_i)^2 / M, m_i = (sum_k v(k,i)) / M; v(k,i) = base[i*stride + k].
__global__ void k_var_series(const double* base, size_t stride, int M, int n1, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n1) return;
    const double* col = base + static_cast<size_t>(i) * stride;
    double m = 0.0;
    for (int k = 0; k < M; ++k) m = __dadd_rn(m, col[k]);
    m = m / M;
    double v = 0.0;
    for (int k = 0; k < M; ++k) {
        const double d = __dsub_rn(col[k], m);
        v = __dadd_rn(v, __dmul_rn(d, d));
    }
    out[i] = v / M;
}

// The same for the default indicator 1{step(k) <= i} of one name (steps [k], one replica).
__global__ void k_var_indicator(const uint16_t* steps, int M, int n1, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n1) return;
    double m = 0.0;
    for (int k = 0; k < M; ++k) m = __dadd_rn(m, steps[k] <= i ? 1.0 : 0.0);
    m = m / M;
    double v = 0.0;
    for (int k = 0; k < M; ++k) {
        const double d = __dsub_rn(steps[k] <= i ? 1.0 : 0.0, m);
        v = __dadd_rn(v, __dmul_rn(d, d));
    }
    out[i] = v / M;
}

}  // namespace hcva

using namespace hcva;

extern "C" hcva_status hcva_ard_sample_variances(hcva_ctx* ctx, const hcva_model* base, const hcva_grid* grid,
                                                 const hcva_swap* book, int n_swaps, const double* prior, int n_dgp,
                                                 int paths_per_dgp, uint64_t key, double* v_x, double* v_y,
                                                 double* v_xi, int* rejected) {
    return guarded([&] {
        StreamScope sc__(ctx->stream);
        HCVA_CUDA(cudaSetDevice(ctx->device));
        const Model bm = make_model(base, grid);  // base.validate(), grid.validate()
        if (n_dgp < 1 || paths_per_dgp < 2) throw config_error("ard: need n_dgp >= 1 and paths >= 2");
        const int E = bm.E, C = bm.Cc, Cn = bm.Cn, n1 = grid->n_steps + 1, M = paths_per_dgp;
        const int nf = 2 * E - 1 + C;
        // ArdPrior (ard.hpp:23-27): vol_lo, vol_hi, level_lo, level_hi, speed_lo, speed_hi.
        const double vol_lo = prior[0], vol_hi = prior[1], level_lo = prior[2], level_hi = prior[3];
        const double speed_lo = prior[4], speed_hi = prior[5];
        const uint64_t pkey = split_key(key, 0);
        uint64_t draw = 0;
        auto uniform_in = [&](double lo, double hi) { return lo + (hi - lo) * u64_to_uniform(draw_u64(pkey, draw++)); };
        struct Params {
            std::vector<hcva_vasicek> r;
            std::vector<hcva_fx> f;
            std::vector<hcva_cir> c;
        };
        std::vector<Params> draws;
        int rej = 0;
        while (static_cast<int>(draws.size()) < n_dgp) {
            Params p;
            p.r.assign(base->rates, base->rates + E);
            if (E > 1) p.f.assign(base->fx, base->fx + (E - 1));
            p.c.assign(base->credit, base->credit + Cn);
            for (auto& r : p.r) {
                r.a *= uniform_in(speed_lo, speed_hi);
                r.b *= uniform_in(level_lo, level_hi);
                r.sigma *= uniform_in(vol_lo, vol_hi);
            }
            for (auto& f : p.f) f.sigma *= uniform_in(vol_lo, vol_hi);
            for (auto& c : p.c) {
                c.alpha *= uniform_in(speed_lo, speed_hi);
                c.delta *= uniform_in(level_lo, level_hi);
                c.nu *= uniform_in(vol_lo, vol_hi);
                c.gamma0 *= uniform_in(level_lo, level_hi);
            }
            hcva_model nu = *base;
            nu.rates = p.r.data();
            nu.fx = p.f.empty() ? nullptr : p.f.data();
            nu.credit = p.c.data();
            try {
                (void)make_model(&nu, grid);
            } catch (const config_error&) {
                ++rej;
                continue;
            }
            draws.push_back(std::move(p));
        }
        if (rejected) *rejected = rej;
        DeviceBuf part;
        part.alloc(sizeof(double) * n1);
        std::vector<double> host(n1);
        for (int d = 0; d < n_dgp; ++d) {
            hcva_model nu = *base;
            nu.rates = draws[d].r.data();
            nu.fx = draws[d].f.empty() ? nullptr : draws[d].f.data();
            nu.credit = draws[d].c.data();
            const uint64_t skey = split_key(split_key(key, 1), static_cast<uint64_t>(d));
            hcva_sim* raw = nullptr;
            if (hcva_simulate_set(ctx, &nu, grid, book, n_swaps, M, 0, 1, split_key(skey, 0), split_key(skey, 1),
                                  &raw) != HCVA_OK)
                throw contract_error(hcva_last_error());
            std::unique_ptr<hcva_sim> sim(raw);
            launch_labels_all(sim.get(), 0);
            auto tavar = [&](auto launch) {
                launch();
                check_launch(ctx);
                copy_out(ctx, host.data(), part.p, sizeof(double) * n1);
                double acc = 0.0;
                for (int i = 0; i < n1; ++i) acc += host[i];
                return acc / n1;
            };
            const int blocks = (n1 + 127) / 128;
            for (int c = 1; c <= C; ++c)
                v_x[static_cast<size_t>(d) * C + c - 1] = tavar([&] {
                    k_var_indicator<<<blocks, 128, 0, ctx->stream>>>(sim->steps.as<uint16_t>() + static_cast<size_t>(c) * M,
                                                                    M, n1, part.as<double>());
                });
            int col = 0;
            auto series = [&](const double* b, size_t stride) {
                return tavar([&] { k_var_series<<<blocks, 128, 0, ctx->stream>>>(b, stride, M, n1, part.as<double>()); });
            };
            double* vy = v_y + static_cast<size_t>(d) * nf;
            for (int e = 0; e < E; ++e)
                vy[col++] = series(sim->rates.as<double>() + static_cast<size_t>(e) * M, static_cast<size_t>(E) * M);
            for (int e = 1; e < E; ++e)
                vy[col++] = series(sim->fx.as<double>() + static_cast<size_t>(e - 1) * M,
                                   static_cast<size_t>(E - 1) * M);
            for (int c = 1; c <= C; ++c)
                vy[col++] = series(sim->intens.as<double>() + static_cast<size_t>(c) * M, static_cast<size_t>(Cn) * M);
            v_xi[d] = series(sim->labels.as<double>(), static_cast<size_t>(M));
        }
    });
}
