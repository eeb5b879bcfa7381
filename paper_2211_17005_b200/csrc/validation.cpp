// validation.cpp -- host estimators of the twin-MC validator
// (validation.cpp:19-117 of the reference): O(M*N) scalar reductions over
// the predictions and the two twin labels, in the reference's summation
// order (FP64, no contraction), so the results match it bit for bit.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

using namespace hcva;

namespace {

void check_triplet(const double* pred, const double* t1, const double* t2, size_t n) {
    if (!pred || !t1 || !t2 || n == 0) throw contract_error("twin estimator: size mismatch or empty input");
}

// clustered_std_error (validation.cpp:19-38): blocks of `block` entries.
double clustered_std_error(const std::vector<double>& v, int block) {
    const size_t n = v.size();
    if (block <= 1 || n % static_cast<size_t>(block) != 0) block = 1;
    const size_t nb = n / block;
    if (nb < 2) return 0.0;
    double grand = 0.0;
    for (double x : v) grand += x;
    grand /= static_cast<double>(n);
    double s = 0.0;
    for (size_t b = 0; b < nb; ++b) {
        double bm = 0.0;
        for (int j = 0; j < block; ++j) bm += v[b * block + j];
        bm /= static_cast<double>(block);
        s += (bm - grand) * (bm - grand);
    }
    s /= static_cast<double>(nb - 1);
    return std::sqrt(s / static_cast<double>(nb));
}

// twin_l2_error (validation.cpp:41-56): mean and clustered s.e. of
// phi^2 - (xi1 + xi2) phi + xi1 xi2.
void twin_l2(const double* pred, const double* t1, const double* t2, size_t n, int block, double* value,
             double* se) {
    std::vector<double> terms(n);
    double sum = 0.0;
    for (size_t j = 0; j < n; ++j) {
        const double phi = pred[j];
        terms[j] = phi * phi - (t1[j] + t2[j]) * phi + t1[j] * t2[j];
        sum += terms[j];
    }
    *value = sum / static_cast<double>(n);
    if (se) *se = clustered_std_error(terms, block);
}

}  // namespace

extern "C" {

hcva_status hcva_twin_l2_error(const double* pred, const double* twin1, const double* twin2, size_t n, int block,
                               double* value, double* std_error) {
    return guarded([&] {
        check_triplet(pred, twin1, twin2, n);
        twin_l2(pred, twin1, twin2, n, block, value, std_error);
    });
}

// twin_relative_rmse (validation.cpp:58-69).
hcva_status hcva_twin_relative_rmse(const double* pred, const double* twin1, const double* twin2, size_t n,
                                    double* out) {
    return guarded([&] {
        check_triplet(pred, twin1, twin2, n);
        double denom = 0.0;
        for (size_t j = 0; j < n; ++j) denom += twin1[j] * twin2[j];
        denom /= static_cast<double>(n);
        if (denom <= 0.0) throw numeric_error("twin_relative_rmse: E[xi1 xi2] <= 0 (degenerate portfolio)");
        double l2;
        twin_l2(pred, twin1, twin2, n, 1, &l2, nullptr);
        *out = std::sqrt(std::max(l2, 0.0) / denom);
    });
}

// twin_relative_rmse_std_error (validation.cpp:71-117): delta method on
// rho = sqrt(A/B), covariance pieces clustered over blocks of outer paths.
hcva_status hcva_twin_relative_rmse_se(const double* pred, const double* twin1, const double* twin2, size_t n,
                                       int block, double* out) {
    return guarded([&] {
        check_triplet(pred, twin1, twin2, n);
        std::vector<double> at(n), bt(n);
        for (size_t j = 0; j < n; ++j) {
            const double phi = pred[j];
            at[j] = phi * phi - (twin1[j] + twin2[j]) * phi + twin1[j] * twin2[j];
            bt[j] = twin1[j] * twin2[j];
        }
        double ma = 0.0, mb = 0.0;
        for (size_t j = 0; j < n; ++j) {
            ma += at[j];
            mb += bt[j];
        }
        ma /= static_cast<double>(n);
        mb /= static_cast<double>(n);
        *out = 0.0;
        if (ma <= 0.0 || mb <= 0.0) return;
        if (block <= 1 || n % static_cast<size_t>(block) != 0) block = 1;
        const size_t nb = n / block;
        if (nb < 2) return;
        double va = 0.0, vb = 0.0, cab = 0.0;
        for (size_t b = 0; b < nb; ++b) {
            double bma = 0.0, bmb = 0.0;
            for (int j = 0; j < block; ++j) {
                bma += at[b * block + j];
                bmb += bt[b * block + j];
            }
            bma /= static_cast<double>(block);
            bmb /= static_cast<double>(block);
            va += (bma - ma) * (bma - ma);
            vb += (bmb - mb) * (bmb - mb);
            cab += (bma - ma) * (bmb - mb);
        }
        const double nbm1 = static_cast<double>(nb - 1) * static_cast<double>(nb);
        va /= nbm1;
        vb /= nbm1;
        cab /= nbm1;
        const double rho = std::sqrt(ma / mb);
        const double rel = va / (ma * ma) + vb / (mb * mb) - 2.0 * cab / (ma * mb);
        *out = 0.5 * rho * std::sqrt(std::max(rel, 0.0));
    });
}

// estimate_qr (planner.cpp:11-70): per outer path two conditionally
// independent losses; R = Cov(g1, g2), total = pooled variance, Q = total - R,
// batch-means standard errors over min(20, n/2) batches.
hcva_status hcva_estimate_qr(const double* g1, const double* g2, size_t n, double* out) {
    return guarded([&] {
        if (!g1 || !g2) throw contract_error("estimate_qr: pair length mismatch");
        estimate_qr_host(g1, g2, n, out);
    });
}

}  // extern "C"

void hcva::estimate_qr_host(const double* g1, const double* g2, size_t n, double* out) {
    {
        if (n < 2) throw numeric_error("estimate_qr: need at least two outer paths");
        double grand = 0.0;
        for (size_t k = 0; k < n; ++k) grand += g1[k] + g2[k];
        grand /= static_cast<double>(2 * n);
        double total = 0.0, r = 0.0;
        for (size_t k = 0; k < n; ++k) {
            const double d1 = g1[k] - grand;
            const double d2 = g2[k] - grand;
            total += d1 * d1 + d2 * d2;
            r += d1 * d2;
        }
        total /= static_cast<double>(2 * n);
        r /= static_cast<double>(n);
        out[0] = total - r;
        out[1] = r;
        out[2] = total;
        out[3] = static_cast<double>(n);
        out[4] = out[5] = 0.0;
        const size_t nb = std::min<size_t>(20, n / 2);
        if (nb >= 2) {
            std::vector<double> qb(nb), rb(nb);
            const size_t bs = n / nb;
            for (size_t b = 0; b < nb; ++b) {
                double bgrand = 0.0;
                for (size_t k = b * bs; k < (b + 1) * bs; ++k) bgrand += g1[k] + g2[k];
                bgrand /= static_cast<double>(2 * bs);
                double bt = 0.0, br = 0.0;
                for (size_t k = b * bs; k < (b + 1) * bs; ++k) {
                    const double d1 = g1[k] - bgrand;
                    const double d2 = g2[k] - bgrand;
                    bt += d1 * d1 + d2 * d2;
                    br += d1 * d2;
                }
                bt /= static_cast<double>(2 * bs);
                br /= static_cast<double>(bs);
                qb[b] = bt - br;
                rb[b] = br;
            }
            auto se = [](const std::vector<double>& v) {
                double m = 0.0;
                for (double x : v) m += x;
                m /= static_cast<double>(v.size());
                double s = 0.0;
                for (double x : v) s += (x - m) * (x - m);
                s /= static_cast<double>(v.size() - 1);
                return std::sqrt(s / static_cast<double>(v.size()));
            };
            out[4] = se(qb);
            out[5] = se(rb);
        }
    }
}
