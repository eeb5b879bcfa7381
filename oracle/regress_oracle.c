/*
 * regress_oracle.c -- TEST INFRASTRUCTURE ONLY (see hcva_oracle.h).
 *
 * FP64 restatement of the reference regressor (proj/src/regressor.cpp), which
 * cannot be compiled here (Eigen is absent).  Same algorithm, same parameter
 * init stream, same batch order, same Adam/refit/head-switch/best-tracking
 * logic; plain loops instead of Eigen GEMMs, so results agree with the
 * reference to FP64 rounding (summation order), not bit for bit.  Pinned by
 * tests/test_oracle_regressor.py against the reference's own analytic tests
 * (finite-difference gradients, hand-solved refit, backward_learn(n=1) ==
 * train_base, determinism).
 *
 * Flat parameter layout (shared with the GPU engine): for l = 0..h,
 * W_l [fan_out][fan_in] row-major then b_l [fan_out]; then mu.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "hcva_oracle.h"

uint64_t or_split_key(uint64_t key, uint64_t k);
void or_uniforms(uint64_t key, uint64_t start, size_t count, double* out);

static size_t layer_off(const or_net_shape* s, int l) {
    size_t off = 0;
    int fin = s->input_dim;
    for (int j = 0; j < l; ++j) {
        const int fout = (j == s->hidden) ? 1 : s->width;
        off += (size_t)fout * fin + fout;
        fin = fout;
    }
    return off;
}

size_t or_net_size(const or_net_shape* s) { return layer_off(s, s->hidden + 1) + 1; }

/* regressor.cpp:172-189: Glorot-uniform limit*(2u-1), row-major per layer, biases 0 */
void or_init_network(const or_net_shape* s, uint64_t key, double* p) {
    memset(p, 0, sizeof(double) * or_net_size(s));
    uint64_t j = 0;
    int fin = s->input_dim;
    for (int l = 0; l <= s->hidden; ++l) {
        const int fout = (l == s->hidden) ? 1 : s->width;
        const double limit = sqrt(6.0 / (fin + fout));
        double* W = p + layer_off(s, l);
        for (int r = 0; r < fout; ++r)
            for (int c = 0; c < fin; ++c) {
                double u;
                or_uniforms(key, j++, 1, &u);
                W[(size_t)r * fin + c] = limit * (2.0 * u - 1.0);
            }
        fin = fout;
    }
}

/* regressor.cpp:35-57 */
static double act(int a, double z, double* d) {
    switch (a) {
        case 0: {
            const double t = tanh(z);
            if (d) *d = 1.0 - t * t;
            return t;
        }
        case 1: {
            const double sg = 1.0 / (1.0 + exp(-z));
            if (d) *d = sg * (1.0 - sg);
            return sg;
        }
        case 2: {
            const double sg = 1.0 / (1.0 + exp(-z));
            if (d) *d = sg;
            return (z > 0.0 ? z : 0.0) + log1p(exp(-fabs(z)));
        }
        default:
            if (d) *d = (z > 0.0) ? 1.0 : 0.0;
            return z > 0.0 ? z : 0.0;
    }
}

/* regressor.cpp:84-95 fit_scaler: mean and population sd of columns >= passthrough */
int or_fit_scaler(const double* x, int rows, int cols, int passthrough, double* mean, double* scale) {
    for (int j = 0; j < cols; ++j) {
        mean[j] = 0.0;
        scale[j] = 1.0;
    }
    for (int j = passthrough; j < cols; ++j) {
        double s = 0.0;
        for (int r = 0; r < rows; ++r) s += x[(size_t)r * cols + j];
        const double m = s / rows;
        double v = 0.0;
        for (int r = 0; r < rows; ++r) {
            const double d = x[(size_t)r * cols + j] - m;
            v += d * d;
        }
        const double sd = sqrt(v / rows);
        mean[j] = m;
        scale[j] = (sd > 1e-12) ? sd : 1.0;
    }
    return 0;
}

/* Forward through the hidden layers for one row; z[l] holds layer l+1 activations. */
static void hidden_row(const or_net_shape* s, const double* p, const double* x, double* acts, double* dacts) {
    const double* in = x;
    int fin = s->input_dim;
    for (int l = 0; l < s->hidden; ++l) {
        const double* W = p + layer_off(s, l);
        const double* b = W + (size_t)s->width * fin;
        double* out = acts + (size_t)l * s->width;
        for (int r = 0; r < s->width; ++r) {
            double a = 0.0;
            for (int c = 0; c < fin; ++c) a += in[c] * W[(size_t)r * fin + c];
            out[r] = act(s->activation, a + b[r], dacts ? dacts + (size_t)l * s->width + r : NULL);
        }
        in = out;
        fin = s->width;
    }
}

static double head_value(const or_net_shape* s, const double* p, const double* top) {
    const int fin = s->hidden > 0 ? s->width : s->input_dim;
    const double* w = p + layer_off(s, s->hidden);
    double f = 0.0;
    for (int c = 0; c < fin; ++c) f += top[c] * w[c];
    return f + w[fin];
}

/* regressor.cpp:97-113 forward */
void or_forward(const or_net_shape* s, const double* p, int head, const double* x, int rows, double* out) {
    const size_t P = or_net_size(s);
    double* acts = malloc(sizeof(double) * (size_t)(s->hidden + 1) * s->width + 1);
    for (int r = 0; r < rows; ++r) {
        const double* xr = x + (size_t)r * s->input_dim;
        hidden_row(s, p, xr, acts, NULL);
        double f = head_value(s, p, s->hidden ? acts + (size_t)(s->hidden - 1) * s->width : xr);
        if (head && f < 0.0) f = 0.0;
        out[r] = f + p[P - 1];
    }
    free(acts);
}

/* regressor.cpp:115-158 quadratic_loss (+ gradients in the flat layout) */
double or_quadratic_loss(const or_net_shape* s, const double* p, int head, const double* x, const double* y,
                         int rows, double* g) {
    const size_t P = or_net_size(s);
    const int h = s->hidden, u = s->width, d = s->input_dim;
    double* acts = malloc(sizeof(double) * (size_t)(h + 1) * u + 1);
    double* dacts = malloc(sizeof(double) * (size_t)(h + 1) * u + 1);
    double* gl = malloc(sizeof(double) * (size_t)u + 1);
    double* gn = malloc(sizeof(double) * (size_t)u + 1);
    const double nb = (double)rows;
    if (g) memset(g, 0, sizeof(double) * P);
    double loss = 0.0;
    for (int r = 0; r < rows; ++r) {
        const double* xr = x + (size_t)r * d;
        hidden_row(s, p, xr, acts, dacts);
        const double* top = h ? acts + (size_t)(h - 1) * u : xr;
        const double f = head_value(s, p, top);
        double pred = (head && f < 0.0) ? 0.0 : f;
        pred += p[P - 1];
        const double resid = pred - y[r];
        loss += resid * resid;
        if (!g) continue;
        g[P - 1] += 2.0 * resid / nb;
        double dd = (2.0 / nb) * resid;
        if (head && !(f > 0.0)) dd = 0.0;
        const int fin_top = h ? u : d;
        double* gw = g + layer_off(s, h);
        const double* w = p + layer_off(s, h);
        for (int c = 0; c < fin_top; ++c) gw[c] += dd * top[c];
        gw[fin_top] += dd;
        for (int c = 0; c < u && h; ++c) gl[c] = dd * w[c];
        for (int l = h - 1; l >= 0; --l) {
            const int fin = (l == 0) ? d : u;
            const double* in = (l == 0) ? xr : acts + (size_t)(l - 1) * u;
            const double* W = p + layer_off(s, l);
            double* gW = g + layer_off(s, l);
            for (int c = 0; c < u; ++c) gl[c] *= dacts[(size_t)l * u + c];
            for (int rr = 0; rr < u; ++rr) {
                for (int c = 0; c < fin; ++c) gW[(size_t)rr * fin + c] += gl[rr] * in[c];
                gW[(size_t)u * fin + rr] += gl[rr];
            }
            if (l > 0) {
                for (int c = 0; c < u; ++c) {
                    double a = 0.0;
                    for (int rr = 0; rr < u; ++rr) a += gl[rr] * W[(size_t)rr * u + c];
                    gn[c] = a;
                }
                memcpy(gl, gn, sizeof(double) * u);
            }
        }
    }
    free(acts), free(dacts), free(gl), free(gn);
    return loss / nb;
}

/* regressor.cpp:191-213 refit_output_layer (LDL^T of the SPD ridge system) */
int or_refit(const or_net_shape* s, double* p, const double* x, const double* y, int rows, double ridge) {
    const int u = s->width, h = s->hidden, n = u + 1;
    const size_t P = or_net_size(s);
    double* gram = calloc((size_t)n * n, sizeof(double));
    double* rhs = calloc((size_t)n, sizeof(double));
    double* acts = malloc(sizeof(double) * (size_t)(h + 1) * u + 1);
    double* row = malloc(sizeof(double) * n);
    for (int r = 0; r < rows; ++r) {
        hidden_row(s, p, x + (size_t)r * s->input_dim, acts, NULL);
        for (int c = 0; c < u; ++c) row[c] = acts[(size_t)(h - 1) * u + c];
        row[u] = 1.0;
        const double t = y[r] - p[P - 1];
        for (int a = 0; a < n; ++a) {
            for (int b = 0; b < n; ++b) gram[a * n + b] += row[a] * row[b];
            rhs[a] += row[a] * t;
        }
    }
    double tr = 0.0;
    for (int a = 0; a < n; ++a) tr += gram[a * n + a];
    double lam = ridge * tr / n;
    if (lam < 1e-300) lam = 1e-300;
    for (int a = 0; a < n; ++a) gram[a * n + a] += lam;
    /* LDL^T without pivoting (SPD after the ridge) */
    double* L = calloc((size_t)n * n, sizeof(double));
    double* D = calloc((size_t)n, sizeof(double));
    for (int j = 0; j < n; ++j) {
        double dj = gram[j * n + j];
        for (int k = 0; k < j; ++k) dj -= L[j * n + k] * L[j * n + k] * D[k];
        D[j] = dj;
        L[j * n + j] = 1.0;
        for (int i = j + 1; i < n; ++i) {
            double v = gram[i * n + j];
            for (int k = 0; k < j; ++k) v -= L[i * n + k] * L[j * n + k] * D[k];
            L[i * n + j] = v / dj;
        }
    }
    double* z = malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        double v = rhs[i];
        for (int k = 0; k < i; ++k) v -= L[i * n + k] * z[k];
        z[i] = v;
    }
    for (int i = 0; i < n; ++i) z[i] /= D[i];
    for (int i = n - 1; i >= 0; --i) {
        double v = z[i];
        for (int k = i + 1; k < n; ++k) v -= L[k * n + i] * z[k];
        z[i] = v;
    }
    double* w = p + layer_off(s, h);
    for (int c = 0; c <= u; ++c) w[c] = z[c];
    free(gram), free(rhs), free(acts), free(row), free(L), free(D), free(z);
    return 0;
}

/* regressor.cpp:236-261 Adam (t counted from 1 after reset) */
static void adam(double* p, const double* g, double* m, double* v, long t, size_t P, double lr) {
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    const double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
    for (size_t i = 0; i < P; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        p[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
    }
}

/* regressor.cpp:265-347 train_base (Alg. 1); returns 3 on a non-finite loss */
int or_train_base(const or_net_shape* s, const double* x, const double* y, int rows, int n_batches, int epochs,
                  double lr, int use_adam, double ridge, const double* init, double* best, double* epoch_losses,
                  double* best_loss, int* best_epoch) {
    if (epochs < 2) return 1;
    if (n_batches < 1 || rows % n_batches) return 1;
    const size_t P = or_net_size(s);
    double* p = malloc(sizeof(double) * P);
    double* g = malloc(sizeof(double) * P);
    double* m = calloc(P, sizeof(double));
    double* v = calloc(P, sizeof(double));
    double* fit = malloc(sizeof(double) * rows);
    memcpy(p, init, sizeof(double) * P);
    memcpy(best, p, sizeof(double) * P);
    int head = 0;
    long t = 0;
    double bl = INFINITY;
    int be = 0, rc = 0;
    const int bs = rows / n_batches, sw = epochs / 2;
    for (int e = 1; e <= epochs && !rc; ++e) {
        for (int b = 0; b < n_batches; ++b) {
            const double l = or_quadratic_loss(s, p, head, x + (size_t)b * bs * s->input_dim, y + (size_t)b * bs, bs, g);
            if (!isfinite(l)) {
                rc = 3;
                break;
            }
            if (use_adam) {
                adam(p, g, m, v, ++t, P, lr);
            } else {
                for (size_t i = 0; i < P; ++i) p[i] -= lr * g[i];
            }
        }
        if (rc) break;
        if (e == sw) {
            or_refit(s, p, x, y, rows, ridge);
            or_forward(s, p, 0, x, rows, fit);
            double mn = fit[0];
            for (int r = 1; r < rows; ++r) mn = fit[r] < mn ? fit[r] : mn;
            const double mu_new = mn > 0.0 ? mn : 0.0;
            p[layer_off(s, s->hidden) + (s->hidden ? s->width : s->input_dim)] += p[P - 1] - mu_new;
            p[P - 1] = mu_new;
            head = 1;
            memset(m, 0, sizeof(double) * P);
            memset(v, 0, sizeof(double) * P);
            t = 0;
        }
        const double ev = or_quadratic_loss(s, p, 1, x, y, rows, NULL);
        if (!isfinite(ev)) {
            rc = 3;
            break;
        }
        epoch_losses[e - 1] = ev;
        if (ev < bl) {
            bl = ev;
            be = e;
            memcpy(best, p, sizeof(double) * P);
        }
    }
    *best_loss = bl;
    *best_epoch = be;
    free(p), free(g), free(m), free(v), free(fit);
    return rc;
}
