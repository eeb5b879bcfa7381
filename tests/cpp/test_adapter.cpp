// test_adapter.cpp -- TEST INFRASTRUCTURE: the maintainer-side adapter
// (integration/hiercva_gpu.cpp) compiled against the reference's own headers
// and linked with the reference's own rng / market / defaults / portfolio
// translation units (built by oracle/Makefile into oracle/_ref/).  The GPU
// drop-in simulate_set_gpu must reproduce the reference's simulate_set
// (pipeline.cpp:63-70 = simulate_market + sample_default_block +
// build_mtm_cube) for the same RandomStream: market 1e-11 relative, default
// steps bit for bit, cube 1e-10 of its scale; a non-PSD correlation is the
// same config_error from both.  Exit status 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "hiercva/defaults.hpp"
#include "hiercva/errors.hpp"
#include "hiercva/market.hpp"
#include "hiercva/portfolio.hpp"
#include "hiercva/rng.hpp"
#include "hiercva_gpu.hpp"

using namespace hiercva;

namespace {

int failures = 0;

void expect(bool ok, const std::string& what) {
    if (!ok) {
        ++failures;
        std::printf("FAIL %s\n", what.c_str());
    }
}

bool close(double got, double want, double rtol, double atol) {
    return std::fabs(got - want) <= rtol * std::fabs(want) + atol;
}

ModelParams desk(bool dense) {
    ModelParams p;
    p.rates = {{0.30, 0.030, 0.010, 0.025}, {0.45, 0.020, 0.012, 0.018}, {0.25, 0.040, 0.009, 0.035}};
    p.fx = {{0.10, -0.25, 1.10}, {0.12, 0.30, 0.85}};
    p.credit = {{0.50, 0.010, 0.05, 0.008}, {0.40, 0.030, 0.09, 0.020}, {0.60, 0.050, 0.12, 0.040},
                {0.35, 0.020, 0.07, 0.015}, {0.55, 0.060, 0.10, 0.050}};
    if (dense) {  // D = 2E - 1 + Cn = 10: a dense PSD correlation with the (r_e, chi_e) entries = rho_e
        const int D = p.n_factors();
        p.brownian_correlation.assign(D * D, 0.0);
        for (int i = 0; i < D; ++i)
            for (int j = 0; j < D; ++j)
                p.brownian_correlation[i * D + j] = i == j ? 1.0 : 0.2 * std::cos(0.7 * (i + 1) * (j + 1));
        auto set = [&](int i, int j, double v) {
            p.brownian_correlation[i * D + j] = v;
            p.brownian_correlation[j * D + i] = v;
        };
        set(1, 3, -0.25);  // (r_1, chi_1) = rho_1
        set(2, 4, 0.30);   // (r_2, chi_2) = rho_2
    }
    return p;
}

void compare(const ModelParams& params, const TimeGrid& grid, int M, int N, const char* name) {
    const RandomStream root(20240901);
    const std::vector<SwapSpec> book = generate_book(params, grid, BookGenSpec{12, 1.0, 25.0}, root.split(0));
    const RandomStream sim = root.split(1);
    const MarketBlock market = simulate_market(params, grid, M, sim.split(0));
    const DefaultBlock defaults = sample_default_block(market, N, sim.split(1));
    const MtMCube cube = build_mtm_cube(market, book, params);
    const gpu::SimulationBlocks g = gpu::simulate_set_gpu(params, grid, book, M, N, sim);
    const int E = params.n_economies(), C = params.n_clients() + 1, n = grid.n_steps;
    int bad = 0;
    for (int k = 0; k < M; ++k)
        for (int i = 0; i <= n; ++i) {
            for (int e = 0; e < E; ++e) {
                bad += !close(g.market.rate(k, i, e), market.rate(k, i, e), 1e-11, 1e-15);
                bad += !close(g.market.lagged_rate(k, i, e), market.lagged_rate(k, i, e), 1e-11, 1e-15);
                bad += !close(g.market.fx(k, i, e), market.fx(k, i, e), 1e-11, 0.0);
            }
            for (int c = 0; c < C; ++c) {
                bad += !close(g.market.intensity(k, i, c), market.intensity(k, i, c), 1e-11, 1e-15);
                bad += !close(g.market.hazard(k, i, c), market.hazard(k, i, c), 1e-11, 1e-15);
            }
            bad += !close(g.market.discount(k, i), market.discount(k, i), 1e-11, 0.0);
        }
    expect(bad == 0, std::string(name) + ": market (" + std::to_string(bad) + " entries outside 1e-11)");
    int mism = 0;
    for (int k = 0; k < M; ++k)
        for (int l = 0; l < N; ++l)
            for (int c = 0; c < C; ++c) mism += g.defaults.default_step(k, l, c) != defaults.default_step(k, l, c);
    expect(mism == 0, std::string(name) + ": default steps (" + std::to_string(mism) + " mismatches)");
    double scale = 0.0;
    for (double v : cube.values) scale = std::fmax(scale, std::fabs(v));
    int cbad = 0;
    for (std::size_t i = 0; i < cube.values.size(); ++i)
        cbad += !close(g.cube.values[i], cube.values[i], 1e-10, 1e-10 * scale);
    expect(cbad == 0 && g.cube.values.size() == cube.values.size(),
           std::string(name) + ": cube (" + std::to_string(cbad) + " entries outside 1e-10)");
    const MarketBlock gm = gpu::simulate_market_gpu(params, grid, M, sim.split(0));
    int mbad = 0;
    for (int k = 0; k < M; ++k)
        for (int i = 0; i <= n; ++i) mbad += gm.rate(k, i, 0) != g.market.rate(k, i, 0);
    expect(mbad == 0, std::string(name) + ": simulate_market_gpu == the set's market");
    std::printf("%s: %d paths x %d replicas x %d steps: market ok=%d, default steps compared %d (mismatches %d), "
                "cube ok=%d\n",
                name, M, N, n, bad == 0, M * N * C, mism, cbad == 0);
}

}  // namespace

int main() {
    const TimeGrid grid{12, 5, 0.5};
    compare(desk(false), grid, 64, 16, "desk (block correlation)");
    compare(desk(true), grid, 48, 8, "desk_corr (dense correlation)");
    // error mapping: a non-PSD correlation is config_error from both
    ModelParams bad = desk(true);
    const int D = bad.n_factors();
    bad.brownian_correlation[0 * D + 5] = bad.brownian_correlation[5 * D + 0] = 0.999;
    bad.brownian_correlation[5 * D + 6] = bad.brownian_correlation[6 * D + 5] = 0.999;
    bad.brownian_correlation[0 * D + 6] = bad.brownian_correlation[6 * D + 0] = -0.999;
    std::string ref_msg, gpu_msg;
    try {
        simulate_market(bad, grid, 4, RandomStream(1));
    } catch (const config_error& e) {
        ref_msg = e.what();
    }
    try {
        gpu::simulate_market_gpu(bad, grid, 4, RandomStream(1));
    } catch (const config_error& e) {
        gpu_msg = e.what();
    }
    expect(!ref_msg.empty() && ref_msg == gpu_msg, "non-PSD correlation: config_error '" + ref_msg + "' vs '" +
                                                       gpu_msg + "'");
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "adapter ok", failures);
    return failures ? 1 : 0;
}
