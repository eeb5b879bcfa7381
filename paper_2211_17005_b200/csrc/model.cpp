// model.cpp -- host-side model utilities of the engine (validation, Cholesky,
// zero-coupon/par arithmetic, book generation).  These run once per call on
// the host and must reproduce the reference's generated book, par rates and
// error texts bit for bit, so is_multiple / cholesky_lower / zc_price /
// par_rate / generate_book are restatements of the reference's own lines
// (portfolio.cpp:16-56,149-174, market.cpp:136-159; SURVEY §8(a) a5, a11,
// a14 allow the reuse); the hot loops live in the kernels.
#include <cmath>
#include <cstring>
#include <mutex>
#include <sstream>

#include "common.cuh"
#include "rng.cuh"

namespace hcva {

namespace {
thread_local std::string g_last_error;
constexpr double kGridTol = 1e-9;  // portfolio.cpp:14
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

cudaStream_t& alloc_stream() {
    static thread_local cudaStream_t s = nullptr;
    return s;
}

bool is_multiple(double x, double step) {  // portfolio.cpp:16-19
    const double q = x / step;
    return std::fabs(q - std::round(q)) < kGridTol * std::max(1.0, std::fabs(q));
}

// market.cpp:136-159
std::vector<double> cholesky_lower(const std::vector<double>& a, int n, const std::string& what) {
    std::vector<double> l(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j <= i; ++j) {
            double sum = a[static_cast<size_t>(i) * n + j];
            for (int k = 0; k < j; ++k) sum -= l[static_cast<size_t>(i) * n + k] * l[static_cast<size_t>(j) * n + k];
            if (i == j) {
                if (sum < -1e-12) {
                    std::ostringstream msg;
                    msg << what << ": not positive semi-definite, leading minor of order " << (i + 1)
                        << " is negative";
                    throw config_error(msg.str());
                }
                l[static_cast<size_t>(i) * n + i] = std::sqrt(std::max(sum, 0.0));
            } else {
                const double d = l[static_cast<size_t>(j) * n + j];
                l[static_cast<size_t>(i) * n + j] = (d > 0.0) ? sum / d : 0.0;
            }
        }
    }
    return l;
}

// ModelParams::validate + correlation_matrix + TimeGrid::validate (market.cpp:12-75)
Model make_model(const hcva_model* m, const hcva_grid* g) {
    if (!m) throw contract_error("model: null pointer");
    Model out;
    out.E = m->n_economies;
    out.Cc = m->n_clients;
    out.Cn = m->n_clients + 1;
    if (out.E < 1) throw config_error("model: at least one economy required");
    if (out.Cc < 0 || !m->credit) throw config_error("model: credit list must include the bank (index 0)");
    if (!m->rates || (out.E > 1 && !m->fx))
        throw config_error("model: need exactly one FX process per non-reference economy");
    out.D = 2 * out.E - 1 + out.Cn;
    out.rates.assign(m->rates, m->rates + out.E);
    if (out.E > 1) out.fx.assign(m->fx, m->fx + out.E - 1);
    out.credit.assign(m->credit, m->credit + out.Cn);
    for (const auto& r : out.rates) {
        if (r.sigma < 0.0) throw config_error("model: rate vol must be >= 0");
        if (r.a < 0.0) throw config_error("model: mean-reversion speed must be >= 0");
    }
    for (const auto& f : out.fx) {
        if (f.sigma < 0.0) throw config_error("model: FX vol must be >= 0");
        if (std::fabs(f.rho) > 1.0) throw config_error("model: |rho| must be <= 1");
        if (f.chi0 <= 0.0) throw config_error("model: initial FX rate must be > 0");
    }
    for (const auto& c : out.credit)
        if (c.delta < 0.0 || c.gamma0 < 0.0 || c.nu < 0.0 || c.alpha < 0.0)
            throw config_error("model: CIR parameters must be >= 0");
    const int d = out.D;
    if (m->correlation) {
        out.corr.assign(m->correlation, m->correlation + static_cast<size_t>(d) * d);
        for (int i = 0; i < d; ++i) {
            if (std::fabs(out.corr[i * d + i] - 1.0) > 1e-12)
                throw config_error("model: correlation matrix must have unit diagonal");
            for (int j = 0; j < d; ++j)
                if (std::fabs(out.corr[i * d + j] - out.corr[j * d + i]) > 1e-12)
                    throw config_error("model: correlation matrix must be symmetric");
        }
        for (int e = 1; e < out.E; ++e)
            if (std::fabs(out.corr[e * d + (out.E + e - 1)] - out.fx[e - 1].rho) > 1e-12)
                throw config_error("model: correlation entry (r_e, chi_e) must equal rho of economy " +
                                   std::to_string(e));
    } else {
        out.corr.assign(static_cast<size_t>(d) * d, 0.0);
        for (int i = 0; i < d; ++i) out.corr[i * d + i] = 1.0;
        for (int e = 1; e < out.E; ++e) {
            out.corr[e * d + (out.E + e - 1)] = out.fx[e - 1].rho;
            out.corr[(out.E + e - 1) * d + e] = out.fx[e - 1].rho;
        }
    }
    if (g) {
        if (g->n_steps <= 0 || g->substeps <= 0 || g->dt <= 0.0)
            throw config_error("grid: steps, substeps and dt must all be positive");
        out.n_steps = g->n_steps;
        out.substeps = g->substeps;
        out.dt = g->dt;
    }
    out.chol = cholesky_lower(out.corr, d, "brownian correlation");
    return out;
}

// portfolio.cpp:34-45
double zc_price(double r, double tau, const hcva_vasicek& p) {
    if (tau < 0.0) throw contract_error("zc_price: negative maturity");
    if (tau == 0.0) return 1.0;
    const double a = p.a, b = p.b, s = p.sigma;
    if (std::fabs(a) < 1e-8) return std::exp(-r * tau + s * s * tau * tau * tau / 6.0);
    const double B = (1.0 - std::exp(-a * tau)) / a;
    const double lnA = (b - s * s / (2.0 * a * a)) * (B - tau) - s * s * B * B / (4.0 * a);
    return std::exp(lnA - B * r);
}

// portfolio.cpp:47-56
double par_rate(double maturity, double tenor, const hcva_vasicek& p) {
    if (tenor <= 0.0 || maturity <= 0.0 || !is_multiple(maturity, tenor))
        throw contract_error("par_rate: invalid schedule");
    const int m = static_cast<int>(std::llround(maturity / tenor));
    double annuity = 0.0;
    for (int j = 1; j <= m; ++j) annuity += zc_price(p.r0, j * tenor, p);
    if (annuity <= 0.0 || !std::isfinite(annuity)) throw numeric_error("par_rate: degenerate annuity");
    return (1.0 - zc_price(p.r0, maturity, p)) / (tenor * annuity);
}

}  // namespace hcva

using namespace hcva;

extern "C" {

const char* hcva_last_error(void) { return g_last_error.c_str(); }
const char* hcva_version(void) { return "hcva-b200 0.1.0 (sm_100a)"; }

uint64_t hcva_rng_root_key(uint64_t seed) { return root_key(seed); }
uint64_t hcva_rng_split_key(uint64_t key, uint64_t k) { return split_key(key, k); }

hcva_status hcva_cholesky(const hcva_model* model, double* chol_out) {
    return guarded([&] {
        Model m = make_model(model, nullptr);
        std::memcpy(chol_out, m.chol.data(), sizeof(double) * m.chol.size());
    });
}

hcva_status hcva_par_rate(double maturity, double tenor, const hcva_vasicek* v, double* out) {
    return guarded([&] { *out = par_rate(maturity, tenor, *v); });
}

hcva_status hcva_zc_price(double r, double tau, const hcva_vasicek* v, double* out) {
    return guarded([&] { *out = zc_price(r, tau, *v); });
}

// portfolio.cpp:149-174: four uniforms per swap, drawn in order from `key`.
hcva_status hcva_generate_book(const hcva_model* model, const hcva_grid* grid, int count,
                               double notional_min, double notional_max, uint64_t key,
                               hcva_swap* out) {
    return guarded([&] {
        if (count < 1) throw config_error("book generator: count must be >= 1");
        if (notional_min <= 0.0 || notional_max < notional_min)
            throw config_error("book generator: invalid notional range");
        Model m = make_model(model, grid);
        uint64_t j = 0;
        auto next_uniform = [&] { return u64_to_uniform(draw_u64(key, j++)); };
        for (int s = 0; s < count; ++s) {
            hcva_swap sw{};
            sw.economy = static_cast<int>(next_uniform() * m.E);
            if (sw.economy >= m.E) sw.economy = m.E - 1;
            sw.client = 1 + static_cast<int>(next_uniform() * m.Cc);
            if (sw.client > m.Cc) sw.client = m.Cc;
            const double u = next_uniform();
            sw.notional = notional_min * std::exp(u * std::log(notional_max / notional_min));
            sw.tenor = m.dt;
            int steps = 1 + static_cast<int>(next_uniform() * m.n_steps);
            if (steps > m.n_steps) steps = m.n_steps;
            sw.maturity = steps * m.dt;
            sw.fixed_rate = par_rate(sw.maturity, sw.tenor, m.rates[sw.economy]);
            out[s] = sw;
        }
    });
}

}  // extern "C"
