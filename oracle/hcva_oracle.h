/*
 * hcva_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference `hiercva` hot path (arXiv 2211.17005,
 * /root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * (paper_2211_17005_b200/) never links or calls it.
 *
 * The same C interface is exported by two libraries:
 *   oracle/liboracle.so          -- this plain-C restatement (hcva_oracle.c)
 *   oracle/_ref/libhcva_ref.so   -- the reference's own sources compiled from
 *                                   /root/reference/proj/src behind ref_shim.cpp
 * tests/test_oracle_pin.py checks the two are bit-identical, which pins the
 * restatement to the reference (the reference ships no golden vectors; see
 * SURVEY.md section 8c).  The regression restatement (or_train_* / or_backward_*)
 * has no compiled counterpart (the reference regressor needs Eigen, absent)
 * and is pinned against the reference's own analytic tests instead.
 *
 * Layouts follow the reference's AoS blocks exactly:
 *   market  (market.hpp:80-123):  rates[(k*(n+1)+i)*E+e], fx[(k*(n+1)+i)*(E-1)+e-1],
 *                                 intens[(k*(n+1)+i)*Cn+c], lagged like rates,
 *                                 disc[k*(n+1)+i], hazard like intens
 *   defaults (defaults.hpp:38-40): steps[(k*N+l)*Cn+c], 0xFFFF = no default
 *   cube    (portfolio.hpp:30-37): cube[(k*(n+1)+i)*Cc+c-1]
 */
#ifndef HCVA_ORACLE_H
#define HCVA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Model: rates E x {a,b,sigma,r0}; fx (E-1) x {sigma,rho,chi0};
 * credit (Cc+1) x {alpha,delta,nu,gamma0} (bank first); corr D*D or NULL. */
typedef struct {
    int n_economies;
    int n_clients;
    const double* rates;
    const double* fx;
    const double* credit;
    const double* corr;
    int n_steps;
    int substeps;
    double dt;
} or_model;

typedef struct {
    int economy;
    int client;
    double notional;
    double tenor;
    double maturity;
    double fixed_rate;
} or_swap;

/* Status: 0 ok, 1 config_error, 2 contract_error, 3 numeric_error. */
const char* or_last_error(void);

/* --- RNG (rng.cpp:9-130) --- */
uint64_t or_root_key(uint64_t seed);
uint64_t or_split_key(uint64_t key, uint64_t k);
void or_draw_u64(uint64_t key, uint64_t start, size_t count, uint64_t* out);
void or_uniforms(uint64_t key, uint64_t start, size_t count, double* out);
void or_normals(uint64_t key, uint64_t start, size_t count, double* out);
void or_exponentials(uint64_t key, uint64_t start, size_t count, double* out);
double or_inverse_normal_cdf(double p);

/* --- market (market.cpp:136-310) --- */
int or_cholesky(const or_model* m, double* chol_out);
int or_simulate_market(const or_model* m, int n_paths, uint64_t key, double* rates, double* fx,
                       double* intens, double* lagged, double* disc, double* hazard);
/* state: rates[E], log_fx[E-1], intens[Cn], lagged[E] */
int or_simulate_conditional(const or_model* m, const double* st_rates, const double* st_logfx,
                            const double* st_intens, const double* st_lagged, int start_step,
                            int horizon, int n_inner, uint64_t key, double* rates, double* fx,
                            double* intens, double* lagged, double* disc, double* hazard);

/* --- defaults (defaults.cpp:13-45) --- */
int or_sample_defaults(int n_paths, int n_steps, int n_names, const double* hazard,
                       int n_replicas, uint64_t key, uint16_t* steps);

/* --- portfolio (portfolio.cpp:34-174) --- */
int or_zc_price(double r, double tau, const double* vasicek, double* out);
int or_par_rate(double maturity, double tenor, const double* vasicek, double* out);
int or_generate_book(const or_model* m, int count, double nmin, double nmax, uint64_t key,
                     or_swap* out);
int or_build_cube(const or_model* m, int n_paths, int n_steps, int start_step,
                  const double* rates, const double* fx, const double* lagged,
                  const or_swap* book, int n_swaps, double* cube);

/* --- labels (labels.cpp:21-167) --- */
int or_defaults_label(int step, int n_paths, int n_steps, int n_economies, int n_names,
                      int n_replicas, double dt, const double* disc, const double* intens,
                      const uint16_t* steps, const double* cube, double* out);
int or_intensity_label(int step, int n_paths, int n_steps, int n_economies, int n_names,
                       int n_replicas, double dt, const double* disc, const double* intens,
                       const uint16_t* steps, const double* cube, double* out);
int or_features(int step, int n_paths, int n_steps, int n_economies, int n_names,
                int n_replicas, const double* rates, const double* fx, const double* intens,
                const double* lagged, const uint16_t* steps, double* out);

/* --- nested MC (validation.cpp:123-179) --- */
int or_nested_cva(const or_model* m, const or_swap* book, int n_swaps, const double* st_rates,
                  const double* st_logfx, const double* st_intens, const double* st_lagged,
                  const int* survived, int step, int inner, uint64_t key, double* value,
                  double* std_error);

/* --- twin MC validator (labels.cpp:90-140, defaults.cpp:47-57, validation.cpp:41-117) ---
 * market / steps: the outer AoS blocks above; t1, t2 [M*N]. */
int or_twin_labels(const or_model* m, const or_swap* book, int n_swaps, int step, int M, int N,
                   const double* rates, const double* fx, const double* intens, const double* lagged,
                   const uint16_t* steps, uint64_t key, double* t1, double* t2);
int or_twin_l2_error(const double* pred, const double* t1, const double* t2, size_t n, int block,
                     double* value, double* std_error);
int or_twin_relative_rmse(const double* pred, const double* t1, const double* t2, size_t n, double* out);
int or_twin_relative_rmse_se(const double* pred, const double* t1, const double* t2, size_t n, int block,
                             double* out);

/* --- ARD sampling (ard.cpp:56-125; the reference's ard.cpp needs Eigen, so
 * this restatement is pinned through its parts: simulate / defaults / cube /
 * labels above, time_averaged_variance and perturb restated) --- */
int or_ard_sample_variances(const or_model* base, const or_swap* book, int n_swaps, const double* prior, int n_dgp,
                            int paths, uint64_t key, double* v_x, double* v_y, double* v_xi, int* rejected);

/* --- book CSV (portfolio.cpp:216-226); compiled reference only --- */
int or_save_book_csv(const char* path, const or_swap* book, int n_swaps);

/* --- Q/R probe (planner.cpp:11-70): out = q, r, total, n_pairs, q_se, r_se --- */
int or_estimate_qr(const double* g1, const double* g2, size_t n, double* out);

/* --- nested_relative_rmse (validation.cpp:181-210): out = value, std_error,
 * excluded_zero, used --- */
int or_nested_relative_rmse(const double* pred, const double* nested, size_t n, double* out);
/* --- percentile_table row (pipeline.cpp:41-47,138-156); restatement only
 * (the reference's pipeline.cpp needs Eigen): v sorted in place, out = mean,
 * p1, p2.5, p97.5, p99 --- */
int or_percentile_bands(double* v, size_t n, double* out);

/* --- regression (regressor.cpp, restated in regress_oracle.c) ---
 * activation: 0 tanh, 1 sigmoid, 2 softplus, 3 relu.  Flat parameters: for
 * l = 0..hidden, W_l [fan_out][fan_in] then b_l [fan_out]; then mu. */
typedef struct {
    int input_dim;
    int hidden;
    int width;
    int activation;
} or_net_shape;

size_t or_net_size(const or_net_shape* s);
void or_init_network(const or_net_shape* s, uint64_t key, double* params);
int or_fit_scaler(const double* x, int rows, int cols, int passthrough, double* mean, double* scale);
void or_forward(const or_net_shape* s, const double* params, int head, const double* x, int rows, double* out);
double or_quadratic_loss(const or_net_shape* s, const double* params, int head, const double* x,
                         const double* y, int rows, double* grads);
int or_refit(const or_net_shape* s, double* params, const double* x, const double* y, int rows, double ridge);
int or_train_base(const or_net_shape* s, const double* x, const double* y, int rows, int n_batches,
                  int epochs, double lr, int adam, double ridge, const double* init, double* best,
                  double* epoch_losses, double* best_loss, int* best_epoch);

/* --- timed CPU baseline of the scenario pipeline ---
 * simulate_set (pipeline.cpp:63-70) with market = split(0), defaults =
 * split(1) of `key_sim`, then for every step i = n..1 the label of the
 * label source (pipeline.cpp:83-90): defaults_label (kind 0) or
 * intensity_label (kind 1).  features_at is not timed: the engine never
 * materialises the feature matrix (it is built inside the regression), so
 * both arms time the same work.  *seconds = wall time of exactly that work;
 * *checksum = sum of all labels (to keep the work observable). */
int or_pipeline_bench(const or_model* m, const or_swap* book, int n_swaps, int n_paths,
                      int n_replicas, uint64_t key_sim, int kind, double* seconds,
                      double* checksum);

#ifdef __cplusplus
}
#endif

#endif
