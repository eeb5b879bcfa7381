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

}  // extern "C"
