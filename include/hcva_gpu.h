/*
 * hcva_gpu.h -- C ABI of the B200-native pathwise CVA engine (libhcva_gpu.so).
 *
 * Drop-in boundary for the hot path of the reference `hiercva` library
 * (arXiv 2211.17005; /root/reference/proj).  The reference exposes its hot
 * path as C++ free functions; each entry point below names the reference
 * interface it replaces (file:line under proj/).  A C++ or pybind caller binds
 * these symbols exactly as INTEGRATION.md shows.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "host or device" output pointers may be
 *    pageable/pinned host memory or device memory of the context's GPU
 *    (copied with cudaMemcpyDefault through UVA).
 *  - Every function returns hcva_status; on failure hcva_last_error() holds
 *    the message.  Status codes map one to one onto the reference's exception
 *    types (proj/include/hiercva/errors.hpp:9-25):
 *      HCVA_ERR_CONFIG   -> config_error   (bad parameters, non-PSD correlation)
 *      HCVA_ERR_CONTRACT -> contract_error (precondition / shape violations)
 *      HCVA_ERR_NUMERIC  -> numeric_error  (degenerate annuity, NaN loss)
 *      HCVA_ERR_CUDA     -> (no reference counterpart: device failure)
 *  - Stream keys are the 64-bit Philox keys of the reference's RandomStream
 *    (rng.cpp:44-55): a caller holding a RandomStream passes the key of the
 *    stream it would have handed to the reference function.
 *  - Layouts: exports reproduce the reference's AoS blocks exactly
 *    (market.hpp:80-123, defaults.hpp:38-40, portfolio.hpp:30-37,
 *    labels.hpp:15-37); device-resident data is SoA, path index fastest.
 */
#ifndef HCVA_GPU_H
#define HCVA_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HCVA_OK = 0,
    HCVA_ERR_CONFIG = 1,
    HCVA_ERR_CONTRACT = 2,
    HCVA_ERR_NUMERIC = 3,
    HCVA_ERR_CUDA = 4
} hcva_status;

typedef struct hcva_ctx hcva_ctx; /* one GPU + one CUDA stream + scratch */
typedef struct hcva_sim hcva_sim; /* a simulated set resident on the GPU  */

/* --- model description (market.hpp:13-75, portfolio.hpp:14-22) --------- */
typedef struct { double a, b, sigma, r0; } hcva_vasicek;      /* VasicekParams */
typedef struct { double sigma, rho, chi0; } hcva_fx;          /* FxParams      */
typedef struct { double alpha, delta, nu, gamma0; } hcva_cir; /* CirParams     */

typedef struct {
    int n_economies;            /* E, economy 0 = reference currency             */
    int n_clients;              /* Cc; credit names = Cc + 1 (bank first)         */
    const hcva_vasicek* rates;  /* [E]                                            */
    const hcva_fx* fx;          /* [E-1] (may be NULL when E == 1)                */
    const hcva_cir* credit;     /* [Cc+1]                                         */
    const double* correlation;  /* [D*D] row-major or NULL (block default)        */
} hcva_model;

typedef struct { int n_steps; int substeps; double dt; } hcva_grid; /* TimeGrid */

typedef struct {                 /* SwapSpec, portfolio.hpp:14-22 */
    int economy;
    int client;
    double notional;
    double tenor;
    double maturity;
    double fixed_rate;
} hcva_swap;

/* --- runtime ------------------------------------------------------------ */
const char* hcva_last_error(void);
const char* hcva_version(void);
hcva_status hcva_ctx_create(int device, hcva_ctx** out);
hcva_status hcva_ctx_destroy(hcva_ctx* ctx);
/* cudaStream_t the context launches on (for events / interop). */
hcva_status hcva_ctx_stream(hcva_ctx* ctx, void** stream_out);
hcva_status hcva_ctx_synchronize(hcva_ctx* ctx);
/* Number of kernels this context launched since creation (evidence counter). */
hcva_status hcva_ctx_launch_count(hcva_ctx* ctx, uint64_t* out);

/* Diagnostic: measured FP64 FMA throughput of this GPU in TFLOP/s (the
 * roofline denominator of the FP64-bound simulation kernels). */
hcva_status hcva_diag_fp64_peak(hcva_ctx* ctx, double* tflops);
/* Diagnostic: the device special functions of the normal transform on host
 * arguments (fn 0 erfc, 1 exp(z<=0), 2 uniform->normal, 3 exp(-y^2)). */
hcva_status hcva_diag_special(hcva_ctx* ctx, int fn, const double* x, size_t n, double* out);
/* Diagnostic: one 3xTF32 tcgen05 GEMM D[M][N] = A[M][K] B[N][K]^T in the
 * regression kernels' operand forms (variant 0: A, B in shared memory; 8: A in
 * tensor memory). */
hcva_status hcva_diag_tc_gemm(hcva_ctx* ctx, int M, int N, int K, int variant, const float* A, const float* B,
                              float* D);
/* Diagnostic: measured kind::tf32 tcgen05.mma throughput (TFLOP/s) of an
 * M x N x 8 MMA chain on every SM (the regression's tensor roofline). */
hcva_status hcva_diag_tc_rate(hcva_ctx* ctx, int M, int N, int iters, double* tflops);

/* --- RNG (rng.hpp:16-52, rng.cpp:44-130) --------------------------------- */
uint64_t hcva_rng_root_key(uint64_t seed);               /* RandomStream(seed) */
uint64_t hcva_rng_split_key(uint64_t key, uint64_t k);   /* .split(k)          */
/* Draws j = start .. start+count-1 of stream `key` on the GPU.
 * kind: 0 = next_u64 (out is uint64_t*), 1 = next_uniform, 2 = next_normal,
 * 3 = next_exponential (out is double*).  Replaces RandomStream::next_*. */
hcva_status hcva_rng_draw(hcva_ctx* ctx, uint64_t key, uint64_t start, size_t count, int kind,
                          void* out);

/* --- host-side model utilities ------------------------------------------- */
/* cholesky_lower of the effective correlation (market.cpp:49-65,136-159). */
hcva_status hcva_cholesky(const hcva_model* model, double* chol_out /* [D*D] */);
/* par_rate (portfolio.cpp:47-56) and zc_price (portfolio.cpp:34-45). */
hcva_status hcva_par_rate(double maturity, double tenor, const hcva_vasicek* v, double* out);
hcva_status hcva_zc_price(double r, double tau, const hcva_vasicek* v, double* out);
/* generate_book (portfolio.cpp:149-174); key = root.split(kBook). */
hcva_status hcva_generate_book(const hcva_model* model, const hcva_grid* grid, int count,
                               double notional_min, double notional_max, uint64_t key,
                               hcva_swap* out /* [count] */);

/* --- simulation (the Y / X / MtM engine) ---------------------------------- */
/* simulate_set (pipeline.cpp:63-70): market from key_market (= stream.split(0)),
 * defaults from key_defaults (= stream.split(1)), MtM cube from the book.
 * Paths path_offset .. path_offset+n_paths-1 of the global path index space
 * (shard of a multi-GPU run; 0 for a single GPU).  n_replicas == 0 skips the
 * default block; book == NULL skips the cube. */
hcva_status hcva_simulate_set(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                              const hcva_swap* book, int n_swaps, int n_paths, int path_offset,
                              int n_replicas, uint64_t key_market, uint64_t key_defaults,
                              hcva_sim** out);
/* Interleaved shard of the global path space: local path k is global path
 * path_offset + (k / shard_blk) * shard_stride + k % shard_blk (shard_blk == 0:
 * path_offset + k).  Rank g of G owning slice g of every regression batch of
 * P_B paths: shard_blk = P_B / G, shard_stride = P_B, path_offset = g * P_B / G,
 * n_paths = M / G -- its local batches are then the rank's slices of the
 * global batches (regressor.cpp:160-170), SURVEY §8(e). */
hcva_status hcva_simulate_set_sharded(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                                      const hcva_swap* book, int n_swaps, int n_paths, int path_offset,
                                      int shard_blk, int shard_stride, int n_replicas, uint64_t key_market,
                                      uint64_t key_defaults, hcva_sim** out);
/* simulate_conditional_market (market.cpp:236-310) for ONE outer state:
 * state = rates[E], log_fx[E-1], intensities[Cc+1], lagged_rates[E]. */
hcva_status hcva_simulate_conditional(hcva_ctx* ctx, const hcva_model* model,
                                      const hcva_grid* grid, const double* state_rates,
                                      const double* state_log_fx, const double* state_intens,
                                      const double* state_lagged, int start_step, int horizon,
                                      int n_inner, uint64_t key, hcva_sim** out);
/* sample_default_block (defaults.cpp:20-45) on an existing market block. */
hcva_status hcva_sample_defaults(hcva_sim* sim, int n_replicas, uint64_t key);
/* build_mtm_cube (portfolio.cpp:97-147) on an existing market block. */
hcva_status hcva_build_cube(hcva_sim* sim, const hcva_swap* book, int n_swaps);
hcva_status hcva_sim_destroy(hcva_sim* sim);
/* Re-run an outer set in place with new stream keys: market, defaults, cube
 * and (labels_kind >= 0) the labels of every step, launched asynchronously on
 * the context stream with no host synchronisation (the execution plan staged
 * by hcva_simulate_set is reused).  event_slot >= 0 records CUDA events around
 * the four phases; hcva_sim_phase_times() reads them after a synchronise. */
hcva_status hcva_sim_rerun(hcva_sim* sim, uint64_t key_market, uint64_t key_defaults, int labels_kind,
                           int event_slot);
/* ms[0..3] = market, defaults, cube, labels durations of slot `event_slot`. */
hcva_status hcva_sim_phase_times(hcva_sim* sim, int event_slot, float* ms /* [4] */);

/* dims: [0]=paths [1]=steps [2]=economies [3]=credit names [4]=replicas
 *       [5]=start_step [6]=factors D [7]=substeps */
hcva_status hcva_sim_dims(const hcva_sim* sim, int* dims /* [8] */);
/* Threshold ties of the last default sampling: (k,l,c) whose exponential
 * threshold lies within tol_ulps ulps of a cumulative hazard it was compared
 * against.  counts[0] = within 1 ulp, counts[1] = within 1e-12 relative. */
hcva_status hcva_sim_tie_counts(const hcva_sim* sim, uint64_t* counts /* [2] */);

/* Exports in the reference's AoS layouts (host or device destination). */
hcva_status hcva_sim_export_market(const hcva_sim* sim, double* rates, double* fx,
                                   double* intensities, double* lagged, double* discounts,
                                   double* hazards);
hcva_status hcva_sim_export_defaults(const hcva_sim* sim, uint16_t* steps);
hcva_status hcva_sim_export_cube(const hcva_sim* sim, double* cube);

/* --- labels / features (labels.cpp:21-88,142-167) ------------------------- */
/* kind: 0 = defaults_label, 1 = intensity_label. out[k*N+l]. */
hcva_status hcva_labels(hcva_sim* sim, int step, int kind, double* out);
/* Labels for every step 0..n in one pass, out[i*M*N + k*N + l] (host or
 * device); out == NULL keeps them on the device only (bench / regression). */
hcva_status hcva_labels_all(hcva_sim* sim, int kind, double* out);
/* CVA profile: out[i] = mean over (k,l) of the step-i labels, i = 0..n (the
 * pathwise CVA estimator E[xi_i]; out[0] is the time-0 CVA).  Host or device. */
hcva_status hcva_cva_profile(hcva_sim* sim, int kind, double* out /* [n+1] */);
/* --- nested Monte Carlo benchmark (validation.cpp:123-179) ---------------- */
/* nested_cva for n_states outer states at pricing step `step`, batched:
 * state s = states[s*(3E-1+Cn) ...] laid out as rates[E], log_fx[E-1],
 * intensities[Cn], lagged_rates[E] (MarketState, market.hpp:58-63);
 * survived[s*Cc + c-1] != 0 when client c survived to `step`.  Inner path l of
 * state s draws from split(split(parent_key, s), l) -- parent_key is the key
 * of the reference's nstream (pipeline.cpp:284-288).  value/std_error[s]
 * are EstimateWithError (validation.hpp:17-20). */
hcva_status hcva_nested_cva_batch(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                                  const hcva_swap* book, int n_swaps, const double* states,
                                  const int* survived, int n_states, int step, int inner,
                                  uint64_t parent_key, double* value, double* std_error);
/* The same for states first_state .. first_state+n_states-1 of a larger set
 * (state s draws from split(parent_key, first_state + s)): one rank's
 * contiguous block of outer states in the multi-GPU nested benchmark. */
hcva_status hcva_nested_cva_range(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid,
                                  const hcva_swap* book, int n_swaps, const double* states,
                                  const int* survived, int n_states, int first_state, int step, int inner,
                                  uint64_t parent_key, double* value, double* std_error);

/* save_market / load_market (pipeline.cpp:371-442): the HCVAMKT1 dump of a
 * set's market block; a loaded outer block becomes a set on which defaults,
 * cube, labels and training run (model / grid must match the dump). */
hcva_status hcva_sim_save_market(const hcva_sim* sim, const char* path, uint64_t seed);
hcva_status hcva_market_load(hcva_ctx* ctx, const hcva_model* model, const hcva_grid* grid, const char* path,
                             uint64_t* seed, hcva_sim** out);

/* --- ARD variance sampling (ard.cpp:56-125) -------------- */
/* prior[6] = vol_lo, vol_hi, level_lo, level_hi, speed_lo, speed_hi (ArdPrior);
 * n_dgp parameter draws from key.split(0) (rejected draws redrawn, count in
 * *rejected), draw d simulated from key.split(1).split(d) with one replica;
 * v_x [n_dgp][Cc], v_y [n_dgp][2E-1+Cc], v_xi [n_dgp] (VarianceSample). */
hcva_status hcva_ard_sample_variances(hcva_ctx* ctx, const hcva_model* base, const hcva_grid* grid,
                                      const hcva_swap* book, int n_swaps, const double* prior, int n_dgp,
                                      int paths_per_dgp, uint64_t key, double* v_x, double* v_y, double* v_xi,
                                      int* rejected);

/* --- twin Monte Carlo validator ------------------------- */
/* twin_labels (labels.cpp:90-140) at pricing step `step` of an outer set: per
 * outer path k two market continuations from state_at(k, step) (inner paths
 * 0/1 of split(k).split(0)), per replica l and twin t the surviving clients
 * re-sample their default on the continuation (resample_continuation,
 * defaults.cpp:47-57, draws from split(k).split(1).split(l).split(t)); twin1/2
 * [M*N] row k*N+l.  `key` is the key of the reference's twin stream. */
hcva_status hcva_twin_labels(hcva_sim* sim, const hcva_swap* book, int n_swaps, int step, uint64_t key,
                             double* twin1, double* twin2);
/* twin_l2_error / twin_relative_rmse / twin_relative_rmse_std_error
 * (validation.cpp:41-117); block = paths_per_block of the clustered s.e.
 * Inputs are host or device arrays of n rows, reduced on the context's GPU in
 * a fixed order (estimators.cu).  twin_relative_rmse fails with
 * HCVA_ERR_NUMERIC when E[xi1 xi2] <= 0. */
hcva_status hcva_twin_l2_error(hcva_ctx* ctx, const double* pred, const double* twin1, const double* twin2,
                               size_t n, int block, double* value, double* std_error);
hcva_status hcva_twin_relative_rmse(hcva_ctx* ctx, const double* pred, const double* twin1, const double* twin2,
                                    size_t n, double* out);
hcva_status hcva_twin_relative_rmse_se(hcva_ctx* ctx, const double* pred, const double* twin1,
                                       const double* twin2, size_t n, int block, double* out);
/* nested_relative_rmse (validation.cpp:181-210) over host or device arrays:
 * out = value, std_error, excluded_zero, used.  HCVA_ERR_NUMERIC when every
 * benchmark is zero. */
hcva_status hcva_nested_relative_rmse(hcva_ctx* ctx, const double* pred, const double* nested, size_t n,
                                      double* out /* [4] */);

/* --- regression (regressor.hpp:33-139) ----------------------------------- */
typedef struct {              /* TrainConfig, regressor.hpp:33-44 */
    int epochs;               /* >= 2, head switch at floor(epochs/2)  */
    int n_batches;            /* must divide the row count             */
    int hidden_layers;        /* 1..4                                   */
    int width;                /* 1..128                                 */
    int activation;           /* 0 tanh, 1 sigmoid, 2 softplus, 3 relu  */
    int adam;                 /* 1 Adam, 0 plain SGD                    */
    double learning_rate;
    double ridge;
    uint64_t seed;            /* init stream RandomStream(seed).split(0xBEEF).split(n) */
} hcva_train_cfg;
typedef struct hcva_models hcva_models; /* TrainedModelSequence, device resident */

/* Flat parameter layout: for l = 0..hidden, W_l [fan_out][fan_in] row-major
 * then b_l [fan_out]; then mu (NetworkParams, regressor.hpp:21-31). */
hcva_status hcva_net_size(const hcva_train_cfg* cfg, int input_dim, int* n_params);
/* init_network (regressor.cpp:172-189) from a stream key; mu = 0. */
hcva_status hcva_init_network(const hcva_train_cfg* cfg, int input_dim, uint64_t key, double* params);
/* quadratic_loss (regressor.cpp:115-158) on host rows x [rows][input_dim];
 * grads may be NULL. */
hcva_status hcva_quadratic_loss(hcva_ctx* ctx, const hcva_train_cfg* cfg, int input_dim, const double* params,
                                int head, const double* x, const double* y, int rows, double* loss, double* grads);
/* forward (regressor.cpp:97-113) with the positive head on (as
 * TrainedModelSequence::predict, regressor.cpp:349-352) on standardised host
 * rows x [rows][input_dim]: out [rows]. */
hcva_status hcva_forward(hcva_ctx* ctx, const hcva_train_cfg* cfg, int input_dim, const double* params,
                         const double* x, int rows, double* out);
/* refit_output_layer (regressor.cpp:191-213): params' output layer replaced by
 * the ridge (cfg->ridge) least-squares fit of y - mu on [z_h, 1]. */
hcva_status hcva_refit_output_layer(hcva_ctx* ctx, const hcva_train_cfg* cfg, int input_dim, double* params,
                                    const double* x, const double* y, int rows);
/* Profiling probe (bench.py roofline): train_base's SGD steps at pricing step
 * `step` of a simulated set (scaler, features, init as backward_learn), CUDA
 * events on the context's stream; out = mean ms of [step, gradient kernels,
 * optimizer], 1 if the layer-0 split kernels ran, and the mean ms per step of
 * the persistent epoch kernel (0 when the shape does not take it). */
hcva_status hcva_diag_sgd_timing(hcva_sim* sim, const hcva_train_cfg* cfg, int step, int label_kind, int steps,
                                 double* out /* [5] */);
/* quadratic_loss (regressor.cpp:115-158) on rows [b0, b1) of the label
 * source at pricing step `step` (pipeline.cpp:72-111): the set's features
 * standardised with mean / scale [input_dim], its labels of label_kind,
 * through the kernels backward_learn runs on this set. */
hcva_status hcva_sim_quadratic_loss(hcva_sim* sim, const hcva_train_cfg* cfg, int step, int label_kind,
                                    const double* params, const double* mean, const double* scale, int head,
                                    long b0, long b1, double* loss, double* grads);
/* train_base (regressor.cpp:265-347) on host rows, contiguous batches. */
hcva_status hcva_train_base(hcva_ctx* ctx, const hcva_train_cfg* cfg, int input_dim, const double* x,
                            const double* y, int rows, const double* init, double* best, double* epoch_losses,
                            double* best_loss, int* best_epoch);
/* backward_learn (regressor.cpp:354-395) fed by the label source of
 * make_label_source (pipeline.cpp:72-111) on a simulated set; label_kind 0 =
 * defaults, 1 = intensity.  Everything stays on the GPU. */
hcva_status hcva_backward_learn(hcva_sim* sim, const hcva_train_cfg* cfg, int label_kind, hcva_models** out);

/* backward_learn with the Q/R probe (pipeline.cpp:79-108, regressor.cpp:328-338,
 * collect_qr_trace): two extra replicas per path from probe_key (the
 * reference's root.split(kTrainSim).split(2)); after every epoch of every
 * step the current network predicts them and estimate_qr (planner.cpp:11-70)
 * gives (Q, R).  trace [n_steps*epochs][4] = step, epoch, Q, R in training
 * order (steps n..1, epochs 1..E).  Single GPU. */
hcva_status hcva_backward_learn_qr(hcva_sim* sim, const hcva_train_cfg* cfg, int label_kind, uint64_t probe_key,
                                   double* trace, hcva_models** out);
/* The probe's default block and labels alone (make_label_source's aux block):
 * steps_out [M][2][Cn] (AoS, DefaultBlock layout), labels_out [n+1][M*2];
 * NULL skips either. */
hcva_status hcva_probe_block(hcva_sim* sim, uint64_t probe_key, int label_kind, uint16_t* steps_out,
                             double* labels_out);
/* estimate_qr (planner.cpp:11-70) on host or device loss pairs:
 * out = Q, R, total, n_pairs, Q s.e., R s.e. */
hcva_status hcva_estimate_qr(hcva_ctx* ctx, const double* g1, const double* g2, size_t n, double* out /* [6] */);

/* --- multi-GPU regression -------------------------------------
 * Y-paths shard by hcva_simulate_set_sharded (rank g owns slice g of every
 * batch); each rank trains on its rows and every cross-rank sum (gradient +
 * loss per SGD step, epoch loss, head-switch minimum, refit Gram, scaler
 * moments, label mean) is an allgather of FP64 partials combined in rank
 * order on the device, so all ranks hold identical networks.  Transports:
 * NCCL (one process per GPU; id from rank 0, broadcast by the caller) or an
 * in-process group (one host thread + context per rank). */
typedef struct hcva_comm hcva_comm;
typedef struct hcva_group hcva_group;
hcva_status hcva_comm_nccl_id(uint8_t* id /* [128] */);
hcva_status hcva_comm_create_nccl(hcva_ctx* ctx, int world, int rank, const uint8_t* id /* [128] */,
                                  hcva_comm** out);
hcva_status hcva_group_create(int world, hcva_group** out);
hcva_status hcva_group_destroy(hcva_group* group);
hcva_status hcva_comm_create_local(hcva_ctx* ctx, hcva_group* group, int rank, hcva_comm** out);
hcva_status hcva_comm_info(const hcva_comm* comm, int* rank, int* world);
hcva_status hcva_comm_destroy(hcva_comm* comm);
/* backward_learn over this rank's shard; comm == NULL is hcva_backward_learn. */
hcva_status hcva_backward_learn_dist(hcva_sim* sim, const hcva_train_cfg* cfg, int label_kind, hcva_comm* comm,
                                     hcva_models** out);
/* info: [0] n_steps [1] input_dim [2] n_params [3] epochs */
hcva_status hcva_models_info(const hcva_models* m, int* info /* [4] */);
/* Per-step model (steps[i-1]): params, scaler mean/scale, report.  NULL skips. */
hcva_status hcva_models_get(const hcva_models* m, int step, double* params, double* mean, double* scale,
                            double* epoch_losses, double* best_loss, int* best_epoch);
/* TrainedModelSequence::predict (regressor.cpp:349-352) on sim's features at step. */
hcva_status hcva_predict(const hcva_models* m, hcva_sim* sim, int step, double* out /* [M*N] */);
/* percentile_table (pipeline.cpp:138-156): per step i = 1..n of the models,
 * the predictions on sim (the validation set) reduced on the device to
 * out [n][6] = step, mean, p1, p2.5, p97.5, p99. */
hcva_status hcva_percentile_table(const hcva_models* m, hcva_sim* sim, double* out);
hcva_status hcva_models_destroy(hcva_models* m);
/* TrainedModelSequence::save / load (regressor.cpp:397-481), the HCVAMDL1
 * format byte for byte (weights column-major as Eigen writes them).  Loaded
 * models carry no training reports; config_hash is NUL-terminated into
 * config_hash[hash_capacity] (NULL skips). */
hcva_status hcva_models_save(const hcva_models* m, const char* path, uint64_t seed, const char* config_hash);
hcva_status hcva_models_load(hcva_ctx* ctx, const char* path, uint64_t* seed, char* config_hash, int hash_capacity,
                             hcva_models** out);

/* features_at: row-major (M*N) x (p+q) FP64. */
hcva_status hcva_features(hcva_sim* sim, int step, double* out);

#ifdef __cplusplus
}
#endif

#endif /* HCVA_GPU_H */
