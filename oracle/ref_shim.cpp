// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the compiled reference (/root/reference/proj/src/{rng,market,
// defaults,portfolio,labels,validation}.cpp, built by oracle/Makefile into
// oracle/_ref/libhcva_ref.so) behind the C interface of hcva_oracle.h, so the
// restatement and the reference can be compared call for call.  No reference
// source is copied into this repository; the Makefile compiles it in place.
#include <cmath>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "hiercva/defaults.hpp"
#include "hiercva/errors.hpp"
#include "hiercva/labels.hpp"
#include "hiercva/market.hpp"
#include "hiercva/portfolio.hpp"
#include "hiercva/rng.hpp"
#include "hiercva/planner.hpp"
#include "hiercva/validation.hpp"
#include "hcva_oracle.h"

using namespace hiercva;

namespace {

std::string g_err;

// RandomStream has no public key constructor; rebuild the lineage instead.
// Keys in the shim API are (seed, lineage) pairs encoded by the caller via
// or_stream_*; for or_* entry points taking a raw key we need the stream that
// produced it, so the shim keeps a registry of streams by key.
struct Registry {
    std::unordered_map<std::uint64_t, RandomStream> items;
    const RandomStream* find(std::uint64_t key) const {
        auto it = items.find(key);
        return it == items.end() ? nullptr : &it->second;
    }
    void add(std::uint64_t key, const RandomStream& s) { items.emplace(key, s); }
};
Registry& reg() {
    static Registry r;
    return r;
}

// Keys are computed with the documented formula (rng.cpp:44-55); the pin test
// checks each registered stream's draws against the restatement's draws.
std::uint64_t mix64(std::uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

ModelParams to_params(const or_model* m) {
    ModelParams p;
    for (int e = 0; e < m->n_economies; ++e)
        p.rates.push_back({m->rates[4 * e], m->rates[4 * e + 1], m->rates[4 * e + 2],
                           m->rates[4 * e + 3]});
    for (int e = 0; e + 1 < m->n_economies; ++e)
        p.fx.push_back({m->fx[3 * e], m->fx[3 * e + 1], m->fx[3 * e + 2]});
    for (int c = 0; c <= m->n_clients; ++c)
        p.credit.push_back({m->credit[4 * c], m->credit[4 * c + 1], m->credit[4 * c + 2],
                            m->credit[4 * c + 3]});
    if (m->corr) {
        const int d = p.n_factors();
        p.brownian_correlation.assign(m->corr, m->corr + d * d);
    }
    return p;
}

TimeGrid to_grid(const or_model* m) { return TimeGrid{m->n_steps, m->substeps, m->dt}; }

const RandomStream& stream_for(std::uint64_t key) {
    const RandomStream* s = reg().find(key);
    if (!s) throw contract_error("ref_shim: unknown stream key (derive it via or_root_key/or_split_key)");
    return *s;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const config_error& e) {
        g_err = e.what();
        return 1;
    } catch (const contract_error& e) {
        g_err = e.what();
        return 2;
    } catch (const numeric_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

void export_market(const MarketBlock& b, double* rates, double* fx, double* intens,
                   double* lagged, double* disc, double* hazard) {
    const int M = b.n_paths(), n = b.n_steps(), E = b.n_economies(), Cn = b.n_credit();
    for (int k = 0; k < M; ++k)
        for (int i = 0; i <= n; ++i) {
            const std::size_t row = static_cast<std::size_t>(k) * (n + 1) + i;
            for (int e = 0; e < E; ++e) rates[row * E + e] = b.rate(k, i, e);
            for (int e = 1; e < E; ++e) fx[row * (E - 1) + e - 1] = b.fx(k, i, e);
            for (int c = 0; c < Cn; ++c) intens[row * Cn + c] = b.intensity(k, i, c);
            for (int e = 0; e < E; ++e) lagged[row * E + e] = b.lagged_rate(k, i, e);
            disc[row] = b.discount(k, i);
            for (int c = 0; c < Cn; ++c) hazard[row * Cn + c] = b.hazard(k, i, c);
        }
}

MarketBlock import_market(int M, int n, int E, int Cn, double dt, int start, const double* rates,
                          const double* fx, const double* intens, const double* lagged,
                          const double* disc, const double* hazard) {
    MarketBlock b(M, n, E, Cn, dt, start);
    for (int k = 0; k < M; ++k)
        for (int i = 0; i <= n; ++i) {
            const std::size_t row = static_cast<std::size_t>(k) * (n + 1) + i;
            for (int e = 0; e < E; ++e) b.rate(k, i, e) = rates ? rates[row * E + e] : 0.0;
            for (int e = 1; e < E; ++e) b.fx_raw(k, i, e - 1) = fx ? fx[row * (E - 1) + e - 1] : 1.0;
            for (int c = 0; c < Cn; ++c) b.intensity(k, i, c) = intens ? intens[row * Cn + c] : 0.0;
            for (int e = 0; e < E; ++e) b.lagged_rate(k, i, e) = lagged ? lagged[row * E + e] : 0.0;
            b.discount(k, i) = disc ? disc[row] : 1.0;
            for (int c = 0; c < Cn; ++c) b.hazard(k, i, c) = hazard ? hazard[row * Cn + c] : 0.0;
        }
    return b;
}

DefaultBlock import_defaults(int M, int N, int n, int Cn, const std::uint16_t* steps) {
    DefaultBlock d(M, N, n, Cn);
    for (int k = 0; k < M; ++k)
        for (int l = 0; l < N; ++l)
            for (int c = 0; c < Cn; ++c)
                d.default_step(k, l, c) = steps[(static_cast<std::size_t>(k) * N + l) * Cn + c];
    return d;
}

MtMCube import_cube(int M, int n, int C, const double* cube) {
    MtMCube q;
    q.n_paths = M;
    q.n_steps = n;
    q.n_clients = C;
    q.values.assign(cube, cube + static_cast<std::size_t>(M) * (n + 1) * C);
    return q;
}

std::vector<SwapSpec> to_book(const or_swap* book, int n) {
    std::vector<SwapSpec> out;
    for (int s = 0; s < n; ++s) {
        SwapSpec sw;
        sw.economy = book[s].economy;
        sw.client = book[s].client;
        sw.notional = book[s].notional;
        sw.tenor = book[s].tenor;
        sw.maturity = book[s].maturity;
        sw.fixed_rate = book[s].fixed_rate;
        out.push_back(sw);
    }
    return out;
}

}  // namespace

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }

std::uint64_t or_root_key(std::uint64_t seed) {
    const std::uint64_t key = mix64(seed ^ 0x9FB21C651E98DF25ULL);
    reg().add(key, RandomStream(seed));
    return key;
}

std::uint64_t or_split_key(std::uint64_t key, std::uint64_t k) {
    const std::uint64_t child =
        mix64(key ^ (mix64(k + 0x632BE59BD9B4E019ULL) + 0x9E3779B97F4A7C15ULL + (key << 6) + (key >> 2)));
    if (const RandomStream* parent = reg().find(key)) reg().add(child, parent->split(k));
    return child;
}

static RandomStream positioned(std::uint64_t key, std::uint64_t start) {
    RandomStream s = stream_for(key);
    for (std::uint64_t i = 0; i < start; ++i) s.next_u64();
    return s;
}

void or_draw_u64(std::uint64_t key, std::uint64_t start, std::size_t count, std::uint64_t* out) {
    RandomStream s = positioned(key, start);
    for (std::size_t i = 0; i < count; ++i) out[i] = s.next_u64();
}
void or_uniforms(std::uint64_t key, std::uint64_t start, std::size_t count, double* out) {
    RandomStream s = positioned(key, start);
    for (std::size_t i = 0; i < count; ++i) out[i] = s.next_uniform();
}
void or_normals(std::uint64_t key, std::uint64_t start, std::size_t count, double* out) {
    RandomStream s = positioned(key, start);
    for (std::size_t i = 0; i < count; ++i) out[i] = s.next_normal();
}
void or_exponentials(std::uint64_t key, std::uint64_t start, std::size_t count, double* out) {
    RandomStream s = positioned(key, start);
    for (std::size_t i = 0; i < count; ++i) out[i] = s.next_exponential();
}
double or_inverse_normal_cdf(double p) { return inverse_normal_cdf(p); }

int or_cholesky(const or_model* m, double* chol_out) {
    return guarded([&] {
        ModelParams p = to_params(m);
        auto l = cholesky_lower(p.correlation_matrix(), p.n_factors(), "brownian correlation");
        std::memcpy(chol_out, l.data(), sizeof(double) * l.size());
    });
}

int or_simulate_market(const or_model* m, int n_paths, std::uint64_t key, double* rates,
                       double* fx, double* intens, double* lagged, double* disc, double* hazard) {
    return guarded([&] {
        MarketBlock b = simulate_market(to_params(m), to_grid(m), n_paths, stream_for(key));
        export_market(b, rates, fx, intens, lagged, disc, hazard);
    });
}

int or_simulate_conditional(const or_model* m, const double* st_rates, const double* st_logfx,
                            const double* st_intens, const double* st_lagged, int start_step,
                            int horizon, int n_inner, std::uint64_t key, double* rates,
                            double* fx, double* intens, double* lagged, double* disc,
                            double* hazard) {
    return guarded([&] {
        const int E = m->n_economies, Cn = m->n_clients + 1;
        MarketState st;
        st.rates.assign(st_rates, st_rates + E);
        st.log_fx.assign(st_logfx, st_logfx + (E - 1));
        st.intensities.assign(st_intens, st_intens + Cn);
        st.lagged_rates.assign(st_lagged, st_lagged + E);
        MarketBlock b = simulate_conditional_market(to_params(m), to_grid(m), st, start_step,
                                                    horizon, n_inner, stream_for(key));
        export_market(b, rates, fx, intens, lagged, disc, hazard);
    });
}

int or_sample_defaults(int n_paths, int n_steps, int n_names, const double* hazard,
                       int n_replicas, std::uint64_t key, std::uint16_t* steps) {
    return guarded([&] {
        MarketBlock b = import_market(n_paths, n_steps, 1, n_names, 1.0, 0, nullptr, nullptr,
                                      nullptr, nullptr, nullptr, hazard);
        DefaultBlock d = sample_default_block(b, n_replicas, stream_for(key));
        for (int k = 0; k < n_paths; ++k)
            for (int l = 0; l < n_replicas; ++l)
                for (int c = 0; c < n_names; ++c)
                    steps[(static_cast<std::size_t>(k) * n_replicas + l) * n_names + c] =
                        d.default_step(k, l, c);
    });
}

int or_zc_price(double r, double tau, const double* v, double* out) {
    return guarded([&] { *out = zc_price(r, tau, VasicekParams{v[0], v[1], v[2], v[3]}); });
}

int or_par_rate(double maturity, double tenor, const double* v, double* out) {
    return guarded([&] { *out = par_rate(maturity, tenor, VasicekParams{v[0], v[1], v[2], v[3]}); });
}

int or_generate_book(const or_model* m, int count, double nmin, double nmax, std::uint64_t key,
                     or_swap* out) {
    return guarded([&] {
        BookGenSpec spec;
        spec.count = count;
        spec.notional_min = nmin;
        spec.notional_max = nmax;
        auto book = generate_book(to_params(m), to_grid(m), spec, stream_for(key));
        for (std::size_t s = 0; s < book.size(); ++s)
            out[s] = or_swap{book[s].economy, book[s].client, book[s].notional, book[s].tenor,
                             book[s].maturity, book[s].fixed_rate};
    });
}

int or_build_cube(const or_model* m, int n_paths, int n_steps, int start_step,
                  const double* rates, const double* fx, const double* lagged,
                  const or_swap* book, int n_swaps, double* cube) {
    return guarded([&] {
        MarketBlock b = import_market(n_paths, n_steps, m->n_economies, m->n_clients + 1, m->dt,
                                      start_step, rates, fx, nullptr, lagged, nullptr, nullptr);
        MtMCube q = build_mtm_cube(b, to_book(book, n_swaps), to_params(m));
        std::memcpy(cube, q.values.data(), sizeof(double) * q.values.size());
    });
}

int or_defaults_label(int step, int M, int n, int E, int Cn, int N, double dt, const double* disc,
                      const double* intens, const std::uint16_t* steps, const double* cube,
                      double* out) {
    return guarded([&] {
        MarketBlock b = import_market(M, n, E, Cn, dt, 0, nullptr, nullptr, intens, nullptr, disc,
                                      nullptr);
        LabelSet l = defaults_label(step, b, import_defaults(M, N, n, Cn, steps),
                                    import_cube(M, n, Cn - 1, cube));
        std::memcpy(out, l.values.data(), sizeof(double) * l.values.size());
    });
}

int or_intensity_label(int step, int M, int n, int E, int Cn, int N, double dt,
                       const double* disc, const double* intens, const std::uint16_t* steps,
                       const double* cube, double* out) {
    return guarded([&] {
        MarketBlock b = import_market(M, n, E, Cn, dt, 0, nullptr, nullptr, intens, nullptr, disc,
                                      nullptr);
        LabelSet l = intensity_label(step, b, import_defaults(M, N, n, Cn, steps),
                                     import_cube(M, n, Cn - 1, cube));
        std::memcpy(out, l.values.data(), sizeof(double) * l.values.size());
    });
}

int or_features(int step, int M, int n, int E, int Cn, int N, const double* rates,
                const double* fx, const double* intens, const double* lagged,
                const std::uint16_t* steps, double* out) {
    return guarded([&] {
        MarketBlock b = import_market(M, n, E, Cn, 1.0, 0, rates, fx, intens, lagged, nullptr,
                                      nullptr);
        FeatureMatrix f = features_at(step, b, import_defaults(M, N, n, Cn, steps));
        std::memcpy(out, f.values.data(), sizeof(double) * f.values.size());
    });
}

int or_nested_cva(const or_model* m, const or_swap* book, int n_swaps, const double* st_rates,
                  const double* st_logfx, const double* st_intens, const double* st_lagged,
                  const int* survived, int step, int inner, std::uint64_t key, double* value,
                  double* std_error) {
    return guarded([&] {
        const int E = m->n_economies, Cn = m->n_clients + 1;
        MarketState st;
        st.rates.assign(st_rates, st_rates + E);
        st.log_fx.assign(st_logfx, st_logfx + (E - 1));
        st.intensities.assign(st_intens, st_intens + Cn);
        st.lagged_rates.assign(st_lagged, st_lagged + E);
        std::vector<bool> surv(m->n_clients);
        for (int c = 0; c < m->n_clients; ++c) surv[c] = survived[c] != 0;
        EstimateWithError est = nested_cva(to_params(m), to_grid(m), to_book(book, n_swaps), st,
                                           surv, step, inner, stream_for(key));
        *value = est.value;
        *std_error = est.std_error;
    });
}

int or_twin_labels(const or_model* m, const or_swap* book, int n_swaps, int step, int M, int N,
                   const double* rates, const double* fx, const double* intens, const double* lagged,
                   const std::uint16_t* steps, std::uint64_t key, double* t1, double* t2) {
    return guarded([&] {
        const int n = m->n_steps, E = m->n_economies, Cn = m->n_clients + 1;
        MarketBlock b = import_market(M, n, E, Cn, m->dt, 0, rates, fx, intens, lagged, nullptr, nullptr);
        auto tw = twin_labels(step, to_params(m), to_grid(m), to_book(book, n_swaps), b,
                              import_defaults(M, N, n, Cn, steps), stream_for(key));
        std::memcpy(t1, tw.first.values.data(), sizeof(double) * tw.first.values.size());
        std::memcpy(t2, tw.second.values.data(), sizeof(double) * tw.second.values.size());
    });
}

int or_twin_l2_error(const double* pred, const double* t1, const double* t2, std::size_t n, int block,
                     double* value, double* std_error) {
    return guarded([&] {
        EstimateWithError e = twin_l2_error(std::vector<double>(pred, pred + n), std::vector<double>(t1, t1 + n),
                                            std::vector<double>(t2, t2 + n), block);
        *value = e.value;
        *std_error = e.std_error;
    });
}

int or_twin_relative_rmse(const double* pred, const double* t1, const double* t2, std::size_t n, double* out) {
    return guarded([&] {
        *out = twin_relative_rmse(std::vector<double>(pred, pred + n), std::vector<double>(t1, t1 + n),
                                  std::vector<double>(t2, t2 + n));
    });
}

int or_twin_relative_rmse_se(const double* pred, const double* t1, const double* t2, std::size_t n, int block,
                             double* out) {
    return guarded([&] {
        *out = twin_relative_rmse_std_error(std::vector<double>(pred, pred + n), std::vector<double>(t1, t1 + n),
                                            std::vector<double>(t2, t2 + n), block);
    });
}

int or_nested_relative_rmse(const double* pred, const double* nested, std::size_t n, double* out) {
    return guarded([&] {
        NestedRmse r = nested_relative_rmse(std::vector<double>(pred, pred + n),
                                            std::vector<double>(nested, nested + n));
        out[0] = r.value;
        out[1] = r.std_error;
        out[2] = static_cast<double>(r.excluded_zero);
        out[3] = static_cast<double>(r.used);
    });
}

int or_save_book_csv(const char* path, const or_swap* book, int n_swaps) {
    return guarded([&] { save_book_csv(path, to_book(book, n_swaps)); });
}

int or_estimate_qr(const double* g1, const double* g2, std::size_t n, double* out) {
    return guarded([&] {
        QRDecomposition qr = estimate_qr(std::vector<double>(g1, g1 + n), std::vector<double>(g2, g2 + n));
        out[0] = qr.q;
        out[1] = qr.r;
        out[2] = qr.total;
        out[3] = static_cast<double>(qr.n_pairs);
        out[4] = qr.q_std_error;
        out[5] = qr.r_std_error;
    });
}

}  // extern "C"

// Timed CPU baseline through the reference's own functions, exactly the work
// of simulate_set (pipeline.cpp:63-70) + the labels of the label source for
// i = n..1 (pipeline.cpp:83-90; features_at is not timed, as on the GPU arm);
// parallel_for uses HIERCVA_THREADS workers.
#include <chrono>
extern "C" int or_pipeline_bench(const or_model* m, const or_swap* book, int n_swaps, int M, int N,
                                 std::uint64_t key_sim, int kind, double* seconds, double* checksum) {
    return guarded([&] {
        const ModelParams p = to_params(m);
        const TimeGrid g = to_grid(m);
        const std::vector<SwapSpec> bk = to_book(book, n_swaps);
        const RandomStream& s = stream_for(key_sim);
        const auto t0 = std::chrono::steady_clock::now();
        MarketBlock market = simulate_market(p, g, M, s.split(0));
        DefaultBlock defaults = sample_default_block(market, N, s.split(1));
        MtMCube cube = build_mtm_cube(market, bk, p);
        double sum = 0.0;
        for (int i = g.n_steps; i >= 1; --i) {
            LabelSet l = kind ? intensity_label(i, market, defaults, cube) : defaults_label(i, market, defaults, cube);
            for (double v : l.values) sum += v;
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *checksum = sum;
    });
}
