// hiercva_gpu.cpp -- see hiercva_gpu.hpp.  Link with -lhcva_gpu.
#include "hiercva_gpu.hpp"

#include <stdexcept>
#include <string>

#include "hcva_gpu.h"
#include "hiercva/errors.hpp"

namespace hiercva::gpu {
namespace {

void check(hcva_status s) {
    if (s == HCVA_OK) return;
    const std::string msg = hcva_last_error();
    if (s == HCVA_ERR_CONFIG) throw config_error(msg);
    if (s == HCVA_ERR_CONTRACT) throw contract_error(msg);
    if (s == HCVA_ERR_NUMERIC) throw numeric_error(msg);
    throw std::runtime_error("hcva: " + msg);  // device failure: no reference counterpart
}

hcva_ctx* context() {
    static hcva_ctx* c = [] {
        hcva_ctx* p = nullptr;
        check(hcva_ctx_create(0, &p));
        return p;
    }();
    return c;
}

// ModelParams (market.hpp:35-56) -> hcva_model; the views own the arrays.
struct ModelView {
    std::vector<hcva_vasicek> rates;
    std::vector<hcva_fx> fx;
    std::vector<hcva_cir> credit;
    hcva_model m{};
    explicit ModelView(const ModelParams& p) {
        for (const auto& v : p.rates) rates.push_back({v.a, v.b, v.sigma, v.r0});
        for (const auto& v : p.fx) fx.push_back({v.sigma, v.rho, v.chi0});
        for (const auto& v : p.credit) credit.push_back({v.alpha, v.delta, v.nu, v.gamma0});
        m.n_economies = p.n_economies();
        m.n_clients = p.n_clients();
        m.rates = rates.data();
        m.fx = fx.empty() ? nullptr : fx.data();
        m.credit = credit.data();
        m.correlation = p.brownian_correlation.empty() ? nullptr : p.brownian_correlation.data();
    }
};

// The engine's AoS export -> the reference block, through its public accessors.
MarketBlock export_market(const hcva_sim* sim, int M, int n, int E, int C, double dt) {
    const std::size_t rows = static_cast<std::size_t>(M) * (n + 1);
    std::vector<double> r(rows * E), fx(rows * (E > 1 ? E - 1 : 1)), g(rows * C), lag(rows * E), disc(rows),
        haz(rows * C);
    check(hcva_sim_export_market(sim, r.data(), E > 1 ? fx.data() : nullptr, g.data(), lag.data(), disc.data(),
                                 haz.data()));
    MarketBlock b(M, n, E, C, dt);
    for (int k = 0; k < M; ++k)
        for (int i = 0; i <= n; ++i) {
            const std::size_t row = static_cast<std::size_t>(k) * (n + 1) + i;
            for (int e = 0; e < E; ++e) {
                b.rate(k, i, e) = r[row * E + e];
                b.lagged_rate(k, i, e) = lag[row * E + e];
            }
            for (int e = 1; e < E; ++e) b.fx_raw(k, i, e - 1) = fx[row * (E - 1) + e - 1];
            for (int c = 0; c < C; ++c) {
                b.intensity(k, i, c) = g[row * C + c];
                b.hazard(k, i, c) = haz[row * C + c];
            }
            b.discount(k, i) = disc[row];
        }
    return b;
}

}  // namespace

std::uint64_t stream_key(const RandomStream& stream) {
    std::uint64_t key = hcva_rng_root_key(stream.seed());
    for (std::uint64_t k : stream.lineage()) key = hcva_rng_split_key(key, k);
    return key;
}

SimulationBlocks simulate_set_gpu(const ModelParams& params, const TimeGrid& grid,
                                  const std::vector<SwapSpec>& book, int n_paths, int n_replicas,
                                  const RandomStream& stream) {
    const ModelView mv(params);
    const hcva_grid g{grid.n_steps, grid.substeps, grid.dt};
    std::vector<hcva_swap> bk;
    for (const auto& s : book) bk.push_back({s.economy, s.client, s.notional, s.tenor, s.maturity, s.fixed_rate});
    const std::uint64_t key = stream_key(stream);
    hcva_sim* sim = nullptr;
    check(hcva_simulate_set(context(), &mv.m, &g, bk.data(), static_cast<int>(bk.size()), n_paths, 0, n_replicas,
                            hcva_rng_split_key(key, 0), hcva_rng_split_key(key, 1), &sim));
    struct Release {
        hcva_sim* s;
        ~Release() { hcva_sim_destroy(s); }
    } release{sim};
    const int E = params.n_economies(), C = params.n_clients() + 1, n = grid.n_steps;
    MarketBlock market = export_market(sim, n_paths, n, E, C, grid.dt);
    std::vector<std::uint16_t> st(static_cast<std::size_t>(n_paths) * n_replicas * C);
    check(hcva_sim_export_defaults(sim, st.data()));
    DefaultBlock defaults(n_paths, n_replicas, n, C);
    for (int k = 0; k < n_paths; ++k)
        for (int l = 0; l < n_replicas; ++l)
            for (int c = 0; c < C; ++c)
                defaults.default_step(k, l, c) = st[(static_cast<std::size_t>(k) * n_replicas + l) * C + c];
    MtMCube cube{n_paths, n, C - 1, std::vector<double>(static_cast<std::size_t>(n_paths) * (n + 1) * (C - 1))};
    check(hcva_sim_export_cube(sim, cube.values.data()));
    return {std::move(market), std::move(defaults), std::move(cube)};
}

MarketBlock simulate_market_gpu(const ModelParams& params, const TimeGrid& grid, int n_paths,
                                const RandomStream& stream) {
    // The market of a set whose market stream is `stream`: the engine draws the
    // market from key_market directly (no replicas, no book).
    const ModelView mv(params);
    const hcva_grid g{grid.n_steps, grid.substeps, grid.dt};
    hcva_sim* sim = nullptr;
    check(hcva_simulate_set(context(), &mv.m, &g, nullptr, 0, n_paths, 0, 0, stream_key(stream),
                            hcva_rng_split_key(stream_key(stream), 1), &sim));
    struct Release {
        hcva_sim* s;
        ~Release() { hcva_sim_destroy(s); }
    } release{sim};
    return export_market(sim, n_paths, grid.n_steps, params.n_economies(), params.n_clients() + 1, grid.dt);
}

}  // namespace hiercva::gpu
