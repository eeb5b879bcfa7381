/*
 * hcva_oracle.c -- TEST INFRASTRUCTURE ONLY (see hcva_oracle.h).
 *
 * Plain-C FP64 restatement of the reference hot path.  Every function cites
 * the reference file:line it follows (paths relative to /root/reference/proj).
 * Arithmetic is written in the reference's evaluation order and compiled
 * with -ffp-contract=off so that, on x86-64 with glibc libm, the results are
 * bit-identical to the compiled reference (checked by tests/test_oracle_pin.py).
 */
#include "hcva_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];

const char* or_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ------------------------------------------------------------------ RNG */
/* rng.cpp:11-14 constants */
#define PHILOX_M 0xD2B74407B1CE6E93ULL
#define PHILOX_W 0x9E3779B97F4A7C15ULL
#define ROOT_SALT 0x9FB21C651E98DF25ULL
#define SPLIT_SALT 0x632BE59BD9B4E019ULL

/* rng.cpp:15-20 SplitMix64 finalizer */
static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.cpp:44-46 */
uint64_t or_root_key(uint64_t seed) { return mix64(seed ^ ROOT_SALT); }

/* rng.cpp:48-55 */
uint64_t or_split_key(uint64_t key, uint64_t k) {
    return mix64(key ^ (mix64(k + SPLIT_SALT) + PHILOX_W + (key << 6) + (key >> 2)));
}

/* rng.cpp:22-40 Philox-2x64-10 */
static void philox(uint64_t c0, uint64_t c1, uint64_t k, uint64_t* o0, uint64_t* o1) {
    for (int r = 0; r < 10; ++r) {
        unsigned __int128 p = (unsigned __int128)PHILOX_M * c0;
        uint64_t hi = (uint64_t)(p >> 64), lo = (uint64_t)p;
        c0 = hi ^ k ^ c1;
        c1 = lo;
        k += PHILOX_W;
    }
    *o0 = c0;
    *o1 = c1;
}

/* rng.cpp:57-67: draw j is word (j % 2) of block (counter = j / 2, 0). */
static uint64_t draw_u64(uint64_t key, uint64_t j) {
    uint64_t o0, o1;
    philox(j >> 1, 0, key, &o0, &o1);
    return (j & 1) ? o1 : o0;
}

/* rng.cpp:69-72 */
static double u64_to_uniform(uint64_t x) { return ((double)(x >> 11) + 0.5) * 0x1.0p-53; }

/* rng.cpp:94-130 Acklam + one Halley step */
double or_inverse_normal_cdf(double p) {
    static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                               -2.759285104469687e+02, 1.383577518672690e+02,
                               -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                               -1.556989798598866e+02, 6.680131188771972e+01,
                               -1.328068155288572e+01};
    static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                               -2.400758277161838e+00, -2.549732539343734e+00,
                               4.374664141464968e+00,  2.938163982698783e+00};
    static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                               2.445134137142996e+00, 3.754408661907416e+00};
    const double p_low = 0.02425;
    double x;
    if (p < p_low) {
        double q = sqrt(-2.0 * log(p));
        x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
    } else if (p <= 1.0 - p_low) {
        double q = p - 0.5;
        double r = q * q;
        x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
            (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
    } else {
        double q = sqrt(-2.0 * log(1.0 - p));
        x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
    }
    double e = 0.5 * erfc(-x / sqrt(2.0)) - p;
    double u = e * sqrt(2.0 * M_PI) * exp(x * x / 2.0);
    x = x - u / (1.0 + x * u / 2.0);
    return x;
}

void or_draw_u64(uint64_t key, uint64_t start, size_t count, uint64_t* out) {
    for (size_t i = 0; i < count; ++i) out[i] = draw_u64(key, start + i);
}
void or_uniforms(uint64_t key, uint64_t start, size_t count, double* out) {
    for (size_t i = 0; i < count; ++i) out[i] = u64_to_uniform(draw_u64(key, start + i));
}
void or_normals(uint64_t key, uint64_t start, size_t count, double* out) {
    for (size_t i = 0; i < count; ++i)
        out[i] = or_inverse_normal_cdf(u64_to_uniform(draw_u64(key, start + i)));
}
/* rng.cpp:76 */
void or_exponentials(uint64_t key, uint64_t start, size_t count, double* out) {
    for (size_t i = 0; i < count; ++i) out[i] = -log(u64_to_uniform(draw_u64(key, start + i)));
}

/* --------------------------------------------------------------- market */
#define V_A(m, e) ((m)->rates[4 * (e) + 0])
#define V_B(m, e) ((m)->rates[4 * (e) + 1])
#define V_S(m, e) ((m)->rates[4 * (e) + 2])
#define V_R0(m, e) ((m)->rates[4 * (e) + 3])
#define FX_S(m, e1) ((m)->fx[3 * (e1) + 0])
#define FX_RHO(m, e1) ((m)->fx[3 * (e1) + 1])
#define FX_CHI0(m, e1) ((m)->fx[3 * (e1) + 2])
#define CR_AL(m, c) ((m)->credit[4 * (c) + 0])
#define CR_DE(m, c) ((m)->credit[4 * (c) + 1])
#define CR_NU(m, c) ((m)->credit[4 * (c) + 2])
#define CR_G0(m, c) ((m)->credit[4 * (c) + 3])

static int n_factors(const or_model* m) { return 2 * m->n_economies - 1 + m->n_clients + 1; }

/* market.cpp:12-47 (ModelParams::validate) + market.cpp:71-74 (TimeGrid::validate) */
static int validate_model(const or_model* m) {
    const int E = m->n_economies, Cn = m->n_clients + 1;
    if (E < 1) return fail(1, "model: at least one economy required");
    if (Cn < 1) return fail(1, "model: credit list must include the bank (index 0)");
    for (int e = 0; e < E; ++e) {
        if (V_S(m, e) < 0.0) return fail(1, "model: rate vol must be >= 0");
        if (V_A(m, e) < 0.0) return fail(1, "model: mean-reversion speed must be >= 0");
    }
    for (int e = 0; e + 1 < E; ++e) {
        if (FX_S(m, e) < 0.0) return fail(1, "model: FX vol must be >= 0");
        if (fabs(FX_RHO(m, e)) > 1.0) return fail(1, "model: |rho| must be <= 1");
        if (FX_CHI0(m, e) <= 0.0) return fail(1, "model: initial FX rate must be > 0");
    }
    for (int c = 0; c < Cn; ++c)
        if (CR_DE(m, c) < 0.0 || CR_G0(m, c) < 0.0 || CR_NU(m, c) < 0.0 || CR_AL(m, c) < 0.0)
            return fail(1, "model: CIR parameters must be >= 0");
    if (m->n_steps <= 0 || m->substeps <= 0 || m->dt <= 0.0)
        return fail(1, "grid: steps, substeps and dt must all be positive");
    return 0;
}

/* market.cpp:49-65 correlation_matrix */
static void corr_matrix(const or_model* m, double* corr) {
    const int d = n_factors(m), E = m->n_economies;
    if (m->corr) {
        memcpy(corr, m->corr, sizeof(double) * d * d);
        return;
    }
    for (int i = 0; i < d * d; ++i) corr[i] = 0.0;
    for (int i = 0; i < d; ++i) corr[i * d + i] = 1.0;
    for (int e = 1; e < E; ++e) {
        corr[e * d + (E + e - 1)] = FX_RHO(m, e - 1);
        corr[(E + e - 1) * d + e] = FX_RHO(m, e - 1);
    }
}

/* market.cpp:136-159 cholesky_lower */
static int cholesky(const double* a, int n, double* l) {
    for (int i = 0; i < n * n; ++i) l[i] = 0.0;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j <= i; ++j) {
            double sum = a[i * n + j];
            for (int k = 0; k < j; ++k) sum -= l[i * n + k] * l[j * n + k];
            if (i == j) {
                if (sum < -1e-12) {
                    snprintf(g_err, sizeof g_err,
                             "brownian correlation: not positive semi-definite, leading minor "
                             "of order %d is negative", i + 1);
                    return 1;
                }
                l[i * n + i] = sqrt(sum > 0.0 ? sum : 0.0);
            } else {
                double dd = l[j * n + j];
                l[i * n + j] = (dd > 0.0) ? sum / dd : 0.0;
            }
        }
    }
    return 0;
}

int or_cholesky(const or_model* m, double* chol_out) {
    const int d = n_factors(m);
    double* corr = malloc(sizeof(double) * d * d);
    corr_matrix(m, corr);
    int rc = cholesky(corr, d, chol_out);
    free(corr);
    return rc;
}

/* market.cpp:121-134 elementary Euler steps */
static double step_vasicek(double r, double dt, double a, double b, double sigma, double q,
                           double z) {
    return r + (a * (b - r) - q) * dt + sigma * sqrt(dt) * z;
}
static double step_log_fx(double lc, double r0, double re, double dt, double sigma, double z) {
    return lc + (r0 - re - 0.5 * sigma * sigma) * dt + sigma * sqrt(dt) * z;
}
static double step_cir(double g, double dt, double alpha, double delta, double nu, double z) {
    double gp = (g < 0.0) ? 0.0 : g; /* std::max(g, 0.0) */
    double next = g + alpha * (delta - gp) * dt + nu * sqrt(gp) * sqrt(dt) * z;
    return (next < 0.0) ? 0.0 : next;
}

/* Shared path recursion of market.cpp:173-231 and market.cpp:256-307. */
static void run_path(const or_model* m, const double* chol, uint64_t pkey, int n_store,
                     double* r, double* logchi, double* gamma, const double* lag0, size_t base,
                     double* rates, double* fx, double* intens, double* lagged, double* disc,
                     double* hazard_out) {
    const int E = m->n_economies, Cn = m->n_clients + 1, D = n_factors(m);
    const double h = m->dt / m->substeps;
    double hazard[Cn], zraw[D], z[D], r_now[E];
    for (int c = 0; c < Cn; ++c) hazard[c] = 0.0;
    double log_beta = 0.0;
    uint64_t j = 0;
#define STORE(i)                                                                     \
    do {                                                                             \
        size_t row = base + (size_t)(i);                                             \
        for (int e = 0; e < E; ++e) rates[row * E + e] = r[e];                       \
        for (int e = 1; e < E; ++e) fx[row * (E - 1) + e - 1] = exp(logchi[e - 1]);  \
        for (int c = 0; c < Cn; ++c) intens[row * Cn + c] = gamma[c];                \
        for (int c = 0; c < Cn; ++c) hazard_out[row * Cn + c] = hazard[c];           \
        disc[row] = exp(-log_beta);                                                  \
        for (int e = 0; e < E; ++e)                                                  \
            lagged[row * E + e] = ((i) == 0) ? lag0[e] : rates[(row - 1) * E + e];   \
    } while (0)
    STORE(0);
    for (int i = 1; i <= n_store; ++i) {
        for (int s = 0; s < m->substeps; ++s) {
            for (int d = 0; d < D; ++d)
                zraw[d] = or_inverse_normal_cdf(u64_to_uniform(draw_u64(pkey, j++)));
            for (int d = 0; d < D; ++d) {
                double acc = 0.0;
                for (int q = 0; q <= d; ++q) acc += chol[d * D + q] * zraw[q];
                z[d] = acc;
            }
            log_beta += r[0] * h;
            for (int c = 0; c < Cn; ++c) hazard[c] += gamma[c] * h;
            const double r0_now = r[0];
            for (int e = 0; e < E; ++e) r_now[e] = r[e];
            for (int e = 0; e < E; ++e) {
                const double quanto =
                    (e == 0) ? 0.0 : FX_RHO(m, e - 1) * FX_S(m, e - 1) * V_S(m, e);
                r[e] = step_vasicek(r[e], h, V_A(m, e), V_B(m, e), V_S(m, e), quanto, z[e]);
            }
            for (int e = 1; e < E; ++e)
                logchi[e - 1] = step_log_fx(logchi[e - 1], r0_now, r_now[e], h, FX_S(m, e - 1),
                                            z[E + e - 1]);
            for (int c = 0; c < Cn; ++c)
                gamma[c] = step_cir(gamma[c], h, CR_AL(m, c), CR_DE(m, c), CR_NU(m, c),
                                    z[E + (E - 1) + c]);
        }
        STORE(i);
    }
#undef STORE
}

/* market.cpp:161-234 simulate_market; path k uses split(k). */
int or_simulate_market(const or_model* m, int n_paths, uint64_t key, double* rates, double* fx,
                       double* intens, double* lagged, double* disc, double* hazard) {
    int rc = validate_model(m);
    if (rc) return rc;
    if (n_paths < 1) return fail(2, "simulate_market: n_paths must be >= 1");
    const int E = m->n_economies, Cn = m->n_clients + 1, D = n_factors(m), n = m->n_steps;
    double* chol = malloc(sizeof(double) * D * D);
    if (or_cholesky(m, chol)) {
        free(chol);
        return 1;
    }
    double r[E], logchi[E], gamma[Cn], lag0[E];
    for (int k = 0; k < n_paths; ++k) {
        for (int e = 0; e < E; ++e) r[e] = V_R0(m, e), lag0[e] = V_R0(m, e);
        for (int e = 1; e < E; ++e) logchi[e - 1] = log(FX_CHI0(m, e - 1));
        for (int c = 0; c < Cn; ++c) gamma[c] = CR_G0(m, c);
        run_path(m, chol, or_split_key(key, (uint64_t)k), n, r, logchi, gamma, lag0,
                 (size_t)k * (n + 1), rates, fx, intens, lagged, disc, hazard);
    }
    free(chol);
    return 0;
}

/* market.cpp:236-310 simulate_conditional_market; inner path l uses split(l). */
int or_simulate_conditional(const or_model* m, const double* st_rates, const double* st_logfx,
                            const double* st_intens, const double* st_lagged, int start_step,
                            int horizon, int n_inner, uint64_t key, double* rates, double* fx,
                            double* intens, double* lagged, double* disc, double* hazard) {
    int rc = validate_model(m);
    if (rc) return rc;
    if (horizon < 0 || start_step + horizon > m->n_steps)
        return fail(2, "simulate_conditional_market: horizon out of range");
    const int E = m->n_economies, Cn = m->n_clients + 1, D = n_factors(m);
    double* chol = malloc(sizeof(double) * D * D);
    if (or_cholesky(m, chol)) {
        free(chol);
        return 1;
    }
    double r[E], logchi[E], gamma[Cn];
    for (int l = 0; l < n_inner; ++l) {
        for (int e = 0; e < E; ++e) r[e] = st_rates[e];
        for (int e = 1; e < E; ++e) logchi[e - 1] = st_logfx[e - 1];
        for (int c = 0; c < Cn; ++c) gamma[c] = st_intens[c];
        run_path(m, chol, or_split_key(key, (uint64_t)l), horizon, r, logchi, gamma, st_lagged,
                 (size_t)l * (horizon + 1), rates, fx, intens, lagged, disc, hazard);
    }
    free(chol);
    return 0;
}

/* ------------------------------------------------------------- defaults */
/* defaults.cpp:13-18 + 20-45 */
int or_sample_defaults(int n_paths, int n_steps, int n_names, const double* hazard,
                       int n_replicas, uint64_t key, uint16_t* steps) {
    if (n_replicas < 1) return fail(2, "sample_default_block: n_replicas must be >= 1");
    const int n = n_steps;
    for (int k = 0; k < n_paths; ++k) {
        uint64_t pk = or_split_key(key, (uint64_t)k);
        for (int l = 0; l < n_replicas; ++l) {
            uint64_t rk = or_split_key(pk, (uint64_t)l);
            for (int c = 0; c < n_names; ++c) {
                const double eps = -log(u64_to_uniform(draw_u64(rk, (uint64_t)c)));
                uint16_t hit = 0xFFFF;
                for (int i = 0; i <= n; ++i)
                    if (hazard[((size_t)k * (n + 1) + i) * n_names + c] >= eps) {
                        hit = (uint16_t)i;
                        break;
                    }
                steps[((size_t)k * n_replicas + l) * n_names + c] = hit;
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------ portfolio */
#define GRID_TOL 1e-9

/* portfolio.cpp:16-19 */
static int is_multiple(double x, double step) {
    double q = x / step;
    double aq = fabs(q);
    return fabs(q - round(q)) < GRID_TOL * (aq > 1.0 ? aq : 1.0);
}

/* portfolio.cpp:34-45 zc_price; vasicek = {a, b, sigma, r0} */
static double zc(double r, double tau, const double* v) {
    if (tau == 0.0) return 1.0;
    const double a = v[0], b = v[1], s = v[2];
    if (fabs(a) < 1e-8) return exp(-r * tau + s * s * tau * tau * tau / 6.0);
    const double B = (1.0 - exp(-a * tau)) / a;
    const double lnA = (b - s * s / (2.0 * a * a)) * (B - tau) - s * s * B * B / (4.0 * a);
    return exp(lnA - B * r);
}

int or_zc_price(double r, double tau, const double* vasicek, double* out) {
    if (tau < 0.0) return fail(2, "zc_price: negative maturity");
    *out = zc(r, tau, vasicek);
    return 0;
}

/* portfolio.cpp:47-56 */
int or_par_rate(double maturity, double tenor, const double* v, double* out) {
    if (tenor <= 0.0 || maturity <= 0.0 || !is_multiple(maturity, tenor))
        return fail(2, "par_rate: invalid schedule");
    const int m = (int)llround(maturity / tenor);
    double annuity = 0.0;
    for (int j = 1; j <= m; ++j) annuity += zc(v[3], j * tenor, v);
    if (annuity <= 0.0 || !isfinite(annuity)) return fail(3, "par_rate: degenerate annuity");
    *out = (1.0 - zc(v[3], maturity, v)) / (tenor * annuity);
    return 0;
}

/* portfolio.cpp:58-95 swap_price */
static double swap_price(double t, double r_now, double r_lag, const or_swap* sw,
                         const double* v) {
    const double delta = sw->tenor, tbar = sw->maturity, sr = sw->fixed_rate;
    if (t < GRID_TOL) {
        const int m = (int)llround(tbar / delta);
        double annuity = 0.0;
        for (int j = 1; j <= m; ++j) annuity += zc(r_now, j * delta, v);
        return 1.0 - zc(r_now, tbar, v) - delta * sr * annuity;
    }
    const int on_reset = is_multiple(t, delta);
    const int m_total = (int)llround(tbar / delta);
    const int j_first = on_reset ? (int)llround(t / delta) + 1 : (int)floor(t / delta + GRID_TOL) + 1;
    double annuity = 0.0;
    for (int j = j_first; j <= m_total; ++j) annuity += zc(r_now, j * delta - t, v);
    if (on_reset) {
        const double zc_prev = zc(r_lag, delta, v);
        return 1.0 / zc_prev - zc(r_now, tbar - t, v) - delta * sr * (1.0 + annuity);
    }
    const double t_prev = floor(t / delta + GRID_TOL) * delta;
    const double t_next = t_prev + delta;
    const double zc_prev = zc(r_lag, t_next - t_prev, v);
    return zc(r_now, t_next - t, v) / zc_prev - zc(r_now, tbar - t, v) - delta * sr * annuity;
}

/* portfolio.cpp:149-174 generate_book; stream = key (draws consumed in order) */
int or_generate_book(const or_model* m, int count, double nmin, double nmax, uint64_t key,
                     or_swap* out) {
    if (count < 1) return fail(1, "book generator: count must be >= 1");
    if (nmin <= 0.0 || nmax < nmin) return fail(1, "book generator: invalid notional range");
    const int E = m->n_economies, C = m->n_clients;
    uint64_t j = 0;
    for (int s = 0; s < count; ++s) {
        or_swap sw;
        sw.economy = (int)(u64_to_uniform(draw_u64(key, j++)) * E);
        if (sw.economy >= E) sw.economy = E - 1;
        sw.client = 1 + (int)(u64_to_uniform(draw_u64(key, j++)) * C);
        if (sw.client > C) sw.client = C;
        const double u = u64_to_uniform(draw_u64(key, j++));
        sw.notional = nmin * exp(u * log(nmax / nmin));
        sw.tenor = m->dt;
        int steps = 1 + (int)(u64_to_uniform(draw_u64(key, j++)) * m->n_steps);
        if (steps > m->n_steps) steps = m->n_steps;
        sw.maturity = steps * m->dt;
        int rc = or_par_rate(sw.maturity, sw.tenor, m->rates + 4 * sw.economy, &sw.fixed_rate);
        if (rc) return rc;
        out[s] = sw;
    }
    return 0;
}

/* portfolio.cpp:97-147 build_mtm_cube (market given as AoS arrays; start_step
 * > 0 for conditional blocks, whose lagged[(k*(n+1))*E+e] carries the state lag) */
int or_build_cube(const or_model* m, int n_paths, int n_steps, int start_step,
                  const double* rates, const double* fx, const double* lagged,
                  const or_swap* book, int n_swaps, double* cube) {
    if (n_swaps < 1) return fail(2, "build_mtm_cube: empty book");
    const int E = m->n_economies, C = m->n_clients;
    const double dt = m->dt;
    for (int s = 0; s < n_swaps; ++s) {
        if (book[s].client < 1 || book[s].client > C)
            return fail(2, "build_mtm_cube: swap client out of range");
        const double lag_d = book[s].tenor / dt;
        const int lag = (int)llround(lag_d);
        if (fabs(lag_d - lag) > GRID_TOL || lag < 1)
            return fail(1, "build_mtm_cube: swap tenor must be a multiple of the pricing step");
        if (start_step > 0 && lag != 1)
            return fail(2, "build_mtm_cube: conditional blocks require tenor == pricing step");
    }
    const size_t total = (size_t)n_paths * (n_steps + 1) * C;
    for (size_t i = 0; i < total; ++i) cube[i] = 0.0;
    for (int k = 0; k < n_paths; ++k) {
        for (int s = 0; s < n_swaps; ++s) {
            const or_swap* sw = &book[s];
            const double* vp = m->rates + 4 * sw->economy;
            const int lag = (int)llround(sw->tenor / dt);
            for (int i = 0; i <= n_steps; ++i) {
                const int g = start_step + i;
                const double t = g * dt;
                if (t > sw->maturity + GRID_TOL) break;
                const size_t row = (size_t)k * (n_steps + 1) + i;
                const double r_now = rates[row * E + sw->economy];
                double r_lag;
                if (g == 0) {
                    r_lag = NAN;
                } else {
                    const int prev_global = ((g - 1) / lag) * lag;
                    const int prev_local = prev_global - start_step;
                    r_lag = (prev_local >= 0)
                                ? rates[((size_t)k * (n_steps + 1) + prev_local) * E + sw->economy]
                                : lagged[((size_t)k * (n_steps + 1)) * E + sw->economy];
                }
                const double px = swap_price(t, r_now, r_lag, sw, vp);
                const double chi = (sw->economy == 0) ? 1.0 : fx[row * (E - 1) + sw->economy - 1];
                cube[row * C + sw->client - 1] += sw->notional * px * chi;
            }
        }
    }
    return 0;
}

/* --------------------------------------------------------------- labels */
/* labels.cpp:21-48 defaults_label */
int or_defaults_label(int i, int M, int n, int E, int Cn, int N, double dt, const double* disc,
                      const double* intens, const uint16_t* steps, const double* cube,
                      double* out) {
    (void)E, (void)dt, (void)intens;
    if (i < 0 || i > n) return fail(2, "label step out of range");
    const int C = Cn - 1;
    for (int k = 0; k < M; ++k) {
        const double inv_beta_i = 1.0 / disc[(size_t)k * (n + 1) + i];
        for (int l = 0; l < N; ++l) {
            double sum = 0.0;
            for (int c = 1; c < Cn; ++c) {
                const int s = steps[((size_t)k * N + l) * Cn + c];
                if (s > i && s <= n) {
                    const double mtm = cube[((size_t)k * (n + 1) + s) * C + c - 1];
                    const double exposure = (mtm < 0.0) ? 0.0 : mtm; /* std::max(x, 0.0) */
                    sum += inv_beta_i * disc[(size_t)k * (n + 1) + s] * exposure;
                }
            }
            out[(size_t)k * N + l] = sum;
        }
    }
    return 0;
}

/* labels.cpp:50-88 intensity_label */
int or_intensity_label(int i, int M, int n, int E, int Cn, int N, double dt, const double* disc,
                       const double* intens, const uint16_t* steps, const double* cube,
                       double* out) {
    (void)E;
    if (i < 0 || i > n) return fail(2, "label step out of range");
    const int C = Cn - 1;
    double sv[Cn];
    for (int k = 0; k < M; ++k) {
        const double inv_beta_i = 1.0 / disc[(size_t)k * (n + 1) + i];
        for (int c = 0; c < Cn; ++c) sv[c] = 0.0;
        for (int c = 1; c < Cn; ++c) {
            double acc = 0.0, gsum = 0.0;
            for (int j = i; j <= n - 1; ++j) {
                const size_t row = (size_t)k * (n + 1) + j;
                const double mtm = cube[row * C + c - 1];
                const double exposure = (mtm < 0.0) ? 0.0 : mtm;
                const double g = intens[row * Cn + c];
                acc += inv_beta_i * disc[row] * exposure * g * dt * exp(-gsum);
                gsum += g * dt;
            }
            sv[c] = acc;
        }
        for (int l = 0; l < N; ++l) {
            double sum = 0.0;
            for (int c = 1; c < Cn; ++c)
                if (steps[((size_t)k * N + l) * Cn + c] > i) sum += sv[c];
            out[(size_t)k * N + l] = sum;
        }
    }
    return 0;
}

/* labels.cpp:142-167 features_at */
int or_features(int i, int M, int n, int E, int Cn, int N, const double* rates, const double* fx,
                const double* intens, const double* lagged, const uint16_t* steps, double* out) {
    if (i < 0 || i > n) return fail(2, "label step out of range");
    const int cols = (Cn - 1) + E + (E - 1) + (Cn - 1) + E;
    for (int k = 0; k < M; ++k) {
        const size_t row = (size_t)k * (n + 1) + i;
        for (int l = 0; l < N; ++l) {
            double* o = out + ((size_t)k * N + l) * cols;
            int col = 0;
            for (int c = 1; c < Cn; ++c) o[col++] = (steps[((size_t)k * N + l) * Cn + c] <= i) ? 1.0 : 0.0;
            for (int e = 0; e < E; ++e) o[col++] = rates[row * E + e];
            for (int e = 1; e < E; ++e) o[col++] = fx[row * (E - 1) + e - 1];
            for (int c = 1; c < Cn; ++c) o[col++] = intens[row * Cn + c];
            for (int e = 0; e < E; ++e) o[col++] = lagged[row * E + e];
        }
    }
    return 0;
}

/* ------------------------------------------------------------ nested MC */
/* validation.cpp:123-168 nested_cva (state overload) */
int or_nested_cva(const or_model* m, const or_swap* book, int n_swaps, const double* st_rates,
                  const double* st_logfx, const double* st_intens, const double* st_lagged,
                  const int* survived, int step, int inner, uint64_t key, double* value,
                  double* std_error) {
    if (inner < 1) return fail(2, "nested_cva: inner_count must be >= 1");
    const int n = m->n_steps, horizon = n - step, C = m->n_clients, E = m->n_economies;
    const int Cn = C + 1;
    *value = 0.0;
    *std_error = 0.0;
    int any = 0;
    for (int c = 0; c < C; ++c) any = any || survived[c];
    if (!any || horizon == 0) return 0;
    const size_t rows = (size_t)inner * (horizon + 1);
    double* rates = malloc(sizeof(double) * rows * E);
    double* fx = malloc(sizeof(double) * rows * (E > 1 ? E - 1 : 1));
    double* intens = malloc(sizeof(double) * rows * Cn);
    double* lagged = malloc(sizeof(double) * rows * E);
    double* disc = malloc(sizeof(double) * rows);
    double* hazard = malloc(sizeof(double) * rows * Cn);
    double* cube = malloc(sizeof(double) * rows * C);
    int rc = or_simulate_conditional(m, st_rates, st_logfx, st_intens, st_lagged, step, horizon,
                                     inner, key, rates, fx, intens, lagged, disc, hazard);
    if (!rc) rc = or_build_cube(m, inner, horizon, step, rates, fx, lagged, book, n_swaps, cube);
    if (!rc) {
        const double dt = m->dt;
        double sum = 0.0, sum_sq = 0.0;
        for (int l = 0; l < inner; ++l) {
            double payoff = 0.0;
            for (int c = 1; c <= C; ++c) {
                if (!survived[c - 1]) continue;
                double gsum = 0.0;
                for (int j = 0; j <= horizon - 1; ++j) {
                    const size_t row = (size_t)l * (horizon + 1) + j;
                    const double mtm = cube[row * C + c - 1];
                    const double exposure = (mtm < 0.0) ? 0.0 : mtm;
                    const double g = intens[row * Cn + c];
                    payoff += disc[row] * exposure * g * dt * exp(-gsum);
                    gsum += g * dt;
                }
            }
            sum += payoff;
            sum_sq += payoff * payoff;
        }
        const double mm = sum / inner;
        *value = mm;
        if (inner > 1) {
            const double var = (sum_sq - inner * mm * mm) / (inner - 1);
            *std_error = sqrt((var > 0.0 ? var : 0.0) / inner);
        }
    }
    free(rates), free(fx), free(intens), free(lagged), free(disc), free(hazard), free(cube);
    return rc;
}

/* --------------------------------------------- twin MC validator (f1) */

/* twin_labels (labels.cpp:90-140): per outer path k two fresh market
 * continuations from state_at(k, step) (market.cpp:100-113, log of the stored
 * FX) with inner paths 0 / 1 from split(k).split(0); per replica l and twin t
 * the surviving clients (default_step > step) redraw their default on the
 * continuation with resample_continuation (defaults.cpp:47-57): one
 * exponential per survivor from split(k).split(1).split(l).split(t), first
 * continuation step whose hazard increment reaches it; the label sums the
 * continuation discount times the positive exposure at that step. */
int or_twin_labels(const or_model* m, const or_swap* book, int n_swaps, int step, int M, int N,
                   const double* rates, const double* fx, const double* intens, const double* lagged,
                   const uint16_t* steps, uint64_t key, double* t1, double* t2) {
    const int n = m->n_steps, E = m->n_economies, C = m->n_clients, Cn = C + 1;
    if (step < 0 || step > n) return fail(2, "labels: step outside the simulated grid");
    const int h = n - step;
    for (size_t r = 0; r < (size_t)M * N; ++r) t1[r] = t2[r] = 0.0;
    if (h == 0) return 0;
    const size_t rows = (size_t)2 * (h + 1);
    double* cr = malloc(sizeof(double) * rows * E);
    double* cf = malloc(sizeof(double) * rows * (E > 1 ? E - 1 : 1));
    double* ci = malloc(sizeof(double) * rows * Cn);
    double* cl = malloc(sizeof(double) * rows * E);
    double* cd = malloc(sizeof(double) * rows);
    double* ch = malloc(sizeof(double) * rows * Cn);
    double* cq = malloc(sizeof(double) * rows * (C > 0 ? C : 1));
    double* st_r = malloc(sizeof(double) * E);
    double* st_f = malloc(sizeof(double) * (E > 1 ? E - 1 : 1));
    double* st_i = malloc(sizeof(double) * Cn);
    double* st_l = malloc(sizeof(double) * E);
    int rc = 0;
    for (int k = 0; k < M && !rc; ++k) {
        const size_t row = (size_t)k * (n + 1) + step;
        for (int e = 0; e < E; ++e) {
            st_r[e] = rates[row * E + e];
            st_l[e] = lagged[row * E + e];
        }
        for (int e = 1; e < E; ++e) st_f[e - 1] = log(fx[row * (E - 1) + e - 1]);
        for (int c = 0; c < Cn; ++c) st_i[c] = intens[row * Cn + c];
        const uint64_t pkey = or_split_key(key, (uint64_t)k);
        rc = or_simulate_conditional(m, st_r, st_f, st_i, st_l, step, h, 2, or_split_key(pkey, 0), cr, cf, ci, cl,
                                     cd, ch);
        if (!rc) rc = or_build_cube(m, 2, h, step, cr, cf, cl, book, n_swaps, cq);
        if (rc) break;
        const uint64_t dkey = or_split_key(pkey, 1);
        for (int l = 0; l < N; ++l) {
            const uint64_t rkey = or_split_key(dkey, (uint64_t)l);
            for (int t = 0; t < 2; ++t) {
                const uint64_t tkey = or_split_key(rkey, (uint64_t)t);
                uint64_t draw = 0;
                double sum = 0.0;
                for (int c = 1; c < Cn; ++c) {
                    if (steps[((size_t)k * N + l) * Cn + c] <= step) continue; /* stays defaulted */
                    double eps;
                    or_exponentials(tkey, draw++, 1, &eps);
                    const double base = ch[((size_t)t * (h + 1)) * Cn + c];
                    int hit = -1;
                    for (int j = 1; j <= h; ++j)
                        if (ch[((size_t)t * (h + 1) + j) * Cn + c] - base >= eps) {
                            hit = j;
                            break;
                        }
                    if (hit >= 0) {
                        const double mtm = cq[((size_t)t * (h + 1) + hit) * C + c - 1];
                        const double exposure = (mtm < 0.0) ? 0.0 : mtm;
                        sum += cd[(size_t)t * (h + 1) + hit] * exposure;
                    }
                }
                (t == 0 ? t1 : t2)[(size_t)k * N + l] = sum;
            }
        }
    }
    free(cr), free(cf), free(ci), free(cl), free(cd), free(ch), free(cq);
    free(st_r), free(st_f), free(st_i), free(st_l);
    return rc;
}

/* clustered_std_error (validation.cpp:19-38): blocks of `block` entries. */
static double clustered_se(const double* v, size_t n, int block) {
    if (block <= 1 || n % (size_t)block != 0) block = 1;
    const size_t nb = n / block;
    if (nb < 2) return 0.0;
    double grand = 0.0;
    for (size_t j = 0; j < n; ++j) grand += v[j];
    grand /= (double)n;
    double s = 0.0;
    for (size_t b = 0; b < nb; ++b) {
        double bm = 0.0;
        for (int j = 0; j < block; ++j) bm += v[b * block + j];
        bm /= (double)block;
        s += (bm - grand) * (bm - grand);
    }
    s /= (double)(nb - 1);
    return sqrt(s / (double)nb);
}

/* twin_l2_error (validation.cpp:41-56). */
int or_twin_l2_error(const double* pred, const double* t1, const double* t2, size_t n, int block,
                     double* value, double* std_error) {
    if (n == 0) return fail(2, "twin estimator: size mismatch or empty input");
    double* terms = malloc(sizeof(double) * n);
    double sum = 0.0;
    for (size_t j = 0; j < n; ++j) {
        const double phi = pred[j];
        terms[j] = phi * phi - (t1[j] + t2[j]) * phi + t1[j] * t2[j];
        sum += terms[j];
    }
    *value = sum / (double)n;
    *std_error = clustered_se(terms, n, block);
    free(terms);
    return 0;
}

/* twin_relative_rmse (validation.cpp:58-69). */
int or_twin_relative_rmse(const double* pred, const double* t1, const double* t2, size_t n, double* out) {
    if (n == 0) return fail(2, "twin estimator: size mismatch or empty input");
    double denom = 0.0;
    for (size_t j = 0; j < n; ++j) denom += t1[j] * t2[j];
    denom /= (double)n;
    if (denom <= 0.0) return fail(3, "twin_relative_rmse: E[xi1 xi2] <= 0 (degenerate portfolio)");
    double l2, se;
    or_twin_l2_error(pred, t1, t2, n, 1, &l2, &se);
    *out = sqrt((l2 > 0.0 ? l2 : 0.0) / denom);
    return 0;
}

/* twin_relative_rmse_std_error (validation.cpp:71-117): delta method, clustered. */
int or_twin_relative_rmse_se(const double* pred, const double* t1, const double* t2, size_t n, int block,
                             double* out) {
    if (n == 0) return fail(2, "twin estimator: size mismatch or empty input");
    double* at = malloc(sizeof(double) * n);
    double* bt = malloc(sizeof(double) * n);
    for (size_t j = 0; j < n; ++j) {
        const double phi = pred[j];
        at[j] = phi * phi - (t1[j] + t2[j]) * phi + t1[j] * t2[j];
        bt[j] = t1[j] * t2[j];
    }
    double ma = 0.0, mb = 0.0;
    for (size_t j = 0; j < n; ++j) {
        ma += at[j];
        mb += bt[j];
    }
    ma /= (double)n;
    mb /= (double)n;
    *out = 0.0;
    if (block <= 1 || n % (size_t)block != 0) block = 1;
    const size_t nb = n / block;
    if (ma > 0.0 && mb > 0.0 && nb >= 2) {
        double va = 0.0, vb = 0.0, cab = 0.0;
        for (size_t b = 0; b < nb; ++b) {
            double bma = 0.0, bmb = 0.0;
            for (int j = 0; j < block; ++j) {
                bma += at[b * block + j];
                bmb += bt[b * block + j];
            }
            bma /= (double)block;
            bmb /= (double)block;
            va += (bma - ma) * (bma - ma);
            vb += (bmb - mb) * (bmb - mb);
            cab += (bma - ma) * (bmb - mb);
        }
        const double nbm1 = (double)(nb - 1) * (double)nb;
        va /= nbm1;
        vb /= nbm1;
        cab /= nbm1;
        const double rho = sqrt(ma / mb);
        const double rel = va / (ma * ma) + vb / (mb * mb) - 2.0 * cab / (ma * mb);
        *out = 0.5 * rho * sqrt(rel > 0.0 ? rel : 0.0);
    }
    free(at), free(bt);
    return 0;
}

/* estimate_qr (planner.cpp:11-70): R = Cov(g1, g2), total = pooled variance,
 * Q = total - R; batch-means standard errors over min(20, n/2) batches. */
static double qr_se(const double* v, size_t nb) {
    double mm = 0.0;
    for (size_t b = 0; b < nb; ++b) mm += v[b];
    mm /= (double)nb;
    double s = 0.0;
    for (size_t b = 0; b < nb; ++b) s += (v[b] - mm) * (v[b] - mm);
    s /= (double)(nb - 1);
    return sqrt(s / (double)nb);
}

int or_estimate_qr(const double* g1, const double* g2, size_t n, double* out) {
    if (n < 2) return fail(3, "estimate_qr: need at least two outer paths");
    double grand = 0.0;
    for (size_t k = 0; k < n; ++k) grand += g1[k] + g2[k];
    grand /= (double)(2 * n);
    double total = 0.0, r = 0.0;
    for (size_t k = 0; k < n; ++k) {
        const double d1 = g1[k] - grand, d2 = g2[k] - grand;
        total += d1 * d1 + d2 * d2;
        r += d1 * d2;
    }
    total /= (double)(2 * n);
    r /= (double)n;
    out[0] = total - r;
    out[1] = r;
    out[2] = total;
    out[3] = (double)n;
    out[4] = out[5] = 0.0;
    const size_t nb = (n / 2 < 20) ? n / 2 : 20;
    if (nb >= 2) {
        double qb[20], rb[20];
        const size_t bs = n / nb;
        for (size_t b = 0; b < nb; ++b) {
            double bg = 0.0;
            for (size_t k = b * bs; k < (b + 1) * bs; ++k) bg += g1[k] + g2[k];
            bg /= (double)(2 * bs);
            double bt = 0.0, br = 0.0;
            for (size_t k = b * bs; k < (b + 1) * bs; ++k) {
                const double d1 = g1[k] - bg, d2 = g2[k] - bg;
                bt += d1 * d1 + d2 * d2;
                br += d1 * d2;
            }
            bt /= (double)(2 * bs);
            br /= (double)bs;
            qb[b] = bt - br;
            rb[b] = br;
        }
        out[4] = qr_se(qb, nb);
        out[5] = qr_se(rb, nb);
    }
    return 0;
}

/* -------------------------------------------- ARD sampling (f4) */

/* time_averaged_variance (ard.cpp:37-52): values[k*(n+1)+i]. */
static double ta_var(const double* v, int M, int n) {
    double acc = 0.0;
    for (int i = 0; i <= n; ++i) {
        double mm = 0.0;
        for (int k = 0; k < M; ++k) mm += v[(size_t)k * (n + 1) + i];
        mm /= M;
        double var = 0.0;
        for (int k = 0; k < M; ++k) {
            const double d = v[(size_t)k * (n + 1) + i] - mm;
            var += d * d;
        }
        acc += var / M;
    }
    return acc / (n + 1);
}

/* sample_variances (ard.cpp:56-125): prior = vol_lo, vol_hi, level_lo,
 * level_hi, speed_lo, speed_hi (ArdPrior); draws from key.split(0) with
 * rejection; draw d simulates from key.split(1).split(d) with one replica;
 * v_x [n_dgp][Cc], v_y [n_dgp][2E-1+Cc], v_xi [n_dgp]. */
int or_ard_sample_variances(const or_model* base, const or_swap* book, int n_swaps, const double* prior, int n_dgp,
                            int paths, uint64_t key, double* v_x, double* v_y, double* v_xi, int* rejected) {
    int rc = validate_model(base);
    if (rc) return rc;
    if (n_dgp < 1 || paths < 2) return fail(1, "ard: need n_dgp >= 1 and paths >= 2");
    const int E = base->n_economies, C = base->n_clients, Cn = C + 1, n = base->n_steps, M = paths;
    const int nf = 2 * E - 1 + C;
    const uint64_t pkey = or_split_key(key, 0);
    uint64_t draw = 0;
#define UNIF(lo, hi) ((lo) + ((hi) - (lo)) * u64_to_uniform(draw_u64(pkey, draw++)))
    double* pr = malloc(sizeof(double) * (size_t)n_dgp * 4 * E);
    double* pf = malloc(sizeof(double) * (size_t)n_dgp * 3 * (E > 1 ? E - 1 : 1));
    double* pc = malloc(sizeof(double) * (size_t)n_dgp * 4 * Cn);
    int have = 0, rej = 0;
    while (have < n_dgp) {
        double* r = pr + (size_t)have * 4 * E;
        double* f = pf + (size_t)have * 3 * (E > 1 ? E - 1 : 1);
        double* c = pc + (size_t)have * 4 * Cn;
        memcpy(r, base->rates, sizeof(double) * 4 * E);
        if (E > 1) memcpy(f, base->fx, sizeof(double) * 3 * (E - 1));
        memcpy(c, base->credit, sizeof(double) * 4 * Cn);
        for (int e = 0; e < E; ++e) {
            r[4 * e + 0] *= UNIF(prior[4], prior[5]);
            r[4 * e + 1] *= UNIF(prior[2], prior[3]);
            r[4 * e + 2] *= UNIF(prior[0], prior[1]);
        }
        for (int e = 0; e + 1 < E; ++e) f[3 * e] *= UNIF(prior[0], prior[1]);
        for (int k = 0; k < Cn; ++k) {
            c[4 * k + 0] *= UNIF(prior[4], prior[5]);
            c[4 * k + 1] *= UNIF(prior[2], prior[3]);
            c[4 * k + 2] *= UNIF(prior[0], prior[1]);
            c[4 * k + 3] *= UNIF(prior[2], prior[3]);
        }
        or_model nu = *base;
        nu.rates = r;
        nu.fx = f;
        nu.credit = c;
        if (validate_model(&nu)) {
            ++rej;
            continue;
        }
        ++have;
    }
#undef UNIF
    if (rejected) *rejected = rej;
    const size_t rows = (size_t)M * (n + 1);
    double* rates = malloc(sizeof(double) * rows * E);
    double* fx = malloc(sizeof(double) * rows * (E > 1 ? E - 1 : 1));
    double* intens = malloc(sizeof(double) * rows * Cn);
    double* lagged = malloc(sizeof(double) * rows * E);
    double* disc = malloc(sizeof(double) * rows);
    double* hazard = malloc(sizeof(double) * rows * Cn);
    double* cube = malloc(sizeof(double) * rows * (C > 0 ? C : 1));
    uint16_t* steps = malloc(sizeof(uint16_t) * (size_t)M * Cn);
    double* buf = malloc(sizeof(double) * rows);
    double* lab = malloc(sizeof(double) * M);
    for (int d = 0; d < n_dgp && !rc; ++d) {
        or_model nu = *base;
        nu.rates = pr + (size_t)d * 4 * E;
        nu.fx = pf + (size_t)d * 3 * (E > 1 ? E - 1 : 1);
        nu.credit = pc + (size_t)d * 4 * Cn;
        const uint64_t skey = or_split_key(or_split_key(key, 1), (uint64_t)d);
        rc = or_simulate_market(&nu, M, or_split_key(skey, 0), rates, fx, intens, lagged, disc, hazard);
        if (!rc) rc = or_sample_defaults(M, n, Cn, hazard, 1, or_split_key(skey, 1), steps);
        if (!rc) rc = or_build_cube(&nu, M, n, 0, rates, fx, lagged, book, n_swaps, cube);
        if (rc) break;
        for (int c = 1; c <= C; ++c) {
            for (int k = 0; k < M; ++k)
                for (int i = 0; i <= n; ++i) buf[(size_t)k * (n + 1) + i] = steps[(size_t)k * Cn + c] <= i ? 1.0 : 0.0;
            v_x[(size_t)d * C + c - 1] = ta_var(buf, M, n);
        }
        double* vy = v_y + (size_t)d * nf;
        int col = 0;
        for (int e = 0; e < E; ++e) {
            for (size_t r = 0; r < rows; ++r) buf[r] = rates[r * E + e];
            vy[col++] = ta_var(buf, M, n);
        }
        for (int e = 1; e < E; ++e) {
            for (size_t r = 0; r < rows; ++r) buf[r] = fx[r * (E - 1) + e - 1];
            vy[col++] = ta_var(buf, M, n);
        }
        for (int c = 1; c <= C; ++c) {
            for (size_t r = 0; r < rows; ++r) buf[r] = intens[r * Cn + c];
            vy[col++] = ta_var(buf, M, n);
        }
        for (int i = 0; i <= n && !rc; ++i) {
            rc = or_defaults_label(i, M, n, E, Cn, 1, base->dt, disc, intens, steps, cube, lab);
            for (int k = 0; k < M; ++k) buf[(size_t)k * (n + 1) + i] = lab[k];
        }
        v_xi[d] = ta_var(buf, M, n);
    }
    free(pr), free(pf), free(pc), free(rates), free(fx), free(intens), free(lagged), free(disc), free(hazard);
    free(cube), free(steps), free(buf), free(lab);
    return rc;
}

/* ------------------------------------------------------ timed baseline */
#include <time.h>

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int or_pipeline_bench(const or_model* m, const or_swap* book, int n_swaps, int M, int N,
                      uint64_t key_sim, int kind, double* seconds, double* checksum) {
    const int E = m->n_economies, Cn = m->n_clients + 1, n = m->n_steps, C = m->n_clients;
    const size_t rows = (size_t)M * (n + 1);
    double* rates = malloc(sizeof(double) * rows * E);
    double* fx = malloc(sizeof(double) * rows * (E > 1 ? E - 1 : 1));
    double* intens = malloc(sizeof(double) * rows * Cn);
    double* lagged = malloc(sizeof(double) * rows * E);
    double* disc = malloc(sizeof(double) * rows);
    double* hazard = malloc(sizeof(double) * rows * Cn);
    double* cube = malloc(sizeof(double) * rows * C);
    uint16_t* steps = malloc(sizeof(uint16_t) * (size_t)M * N * Cn);
    double* lab = malloc(sizeof(double) * (size_t)M * N);
    const double t0 = now_s();
    int rc = or_simulate_market(m, M, or_split_key(key_sim, 0), rates, fx, intens, lagged, disc, hazard);
    if (!rc) rc = or_sample_defaults(M, n, Cn, hazard, N, or_split_key(key_sim, 1), steps);
    if (!rc) rc = or_build_cube(m, M, n, 0, rates, fx, lagged, book, n_swaps, cube);
    double sum = 0.0;
    for (int i = n; i >= 1 && !rc; --i) {
        rc = (kind ? or_intensity_label : or_defaults_label)(i, M, n, E, Cn, N, m->dt, disc, intens,
                                                                 steps, cube, lab);
        for (size_t r = 0; r < (size_t)M * N && !rc; ++r) sum += lab[r];
    }
    *seconds = now_s() - t0;
    *checksum = sum;
    free(rates), free(fx), free(intens), free(lagged), free(disc), free(hazard), free(cube);
    free(steps), free(lab);
    return rc;
}

/* nested_relative_rmse (validation.cpp:181-210): squared relative errors over
 * the nonzero benchmarks; out = value, std_error, excluded_zero, used. */
int or_nested_relative_rmse(const double* pred, const double* nested, size_t n, double* out) {
    if (n == 0) return fail(2, "nested_relative_rmse: size mismatch or empty input");
    size_t used = 0;
    double m = 0.0;
    for (size_t j = 0; j < n; ++j) {
        if (nested[j] == 0.0) continue;
        const double e = (pred[j] - nested[j]) / nested[j];
        m += e * e;
        ++used;
    }
    if (used == 0) return fail(3, "nested_relative_rmse: all benchmarks are zero");
    m /= (double)used;
    out[0] = sqrt(m);
    out[1] = 0.0;
    if (used > 1 && m > 0.0) {
        double v = 0.0;
        for (size_t j = 0; j < n; ++j) {
            if (nested[j] == 0.0) continue;
            const double e = (pred[j] - nested[j]) / nested[j];
            v += (e * e - m) * (e * e - m);
        }
        v /= (double)(used - 1);
        out[1] = sqrt(v / (double)used) / (2.0 * out[0]);
    }
    out[2] = (double)(n - used);
    out[3] = (double)used;
    return 0;
}

/* One row of percentile_table (pipeline.cpp:138-156) with percentile_sorted's
 * linear interpolation (pipeline.cpp:41-47): v is sorted in place; out =
 * mean (sequential sum of the sorted values), p1, p2.5, p97.5, p99. */
static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

int or_percentile_bands(double* v, size_t n, double* out) {
    if (n == 0) return fail(2, "percentile_table: no predictions");
    qsort(v, n, sizeof(double), cmp_double);
    double s = 0.0;
    for (size_t j = 0; j < n; ++j) s += v[j];
    out[0] = s / (double)n;
    const double q[4] = {0.01, 0.025, 0.975, 0.99};
    for (int t = 0; t < 4; ++t) {
        const double pos = q[t] * ((double)n - 1.0);
        const size_t i = (size_t)pos;
        const double f = pos - (double)i;
        out[1 + t] = i + 1 < n ? v[i] * (1.0 - f) + v[i + 1] * f : v[i];
    }
    return 0;
}
