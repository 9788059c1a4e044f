// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Restatement of the reference's training-data preparation,
// P:src/dataset.cpp: balance_and_split (:212-262; libstdc++ std::mt19937_64
// and std::shuffle, so the split is the reference's) and
// zscore_fit_transform (:264-282; population standard deviation, constant
// columns keep sd = 1).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "ksvm_oracle.h"

namespace {
thread_local std::string t_err = "ok";
}

extern "C" int oracle_balance_and_split(const double* labels, int64_t n, double train_fraction, uint64_t seed,
                                        int64_t* train_idx, int64_t* n_train, int64_t* test_idx, int64_t* n_test) {
    if (!(train_fraction > 0.0 && train_fraction < 1.0)) return 2;
    int64_t npos = 0;
    for (int64_t i = 0; i < n; ++i) npos += labels[i] > 0;
    if (npos == 0 || npos == n) return 2;
    std::mt19937_64 rng(seed);
    std::vector<int64_t> perm(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) perm[static_cast<size_t>(i)] = i;
    std::shuffle(perm.begin(), perm.end(), rng);
    const auto nt = static_cast<int64_t>(std::floor(train_fraction * static_cast<double>(n)));
    std::vector<int64_t> pos, neg;
    for (int64_t r = 0; r < nt; ++r) {
        const int64_t i = perm[static_cast<size_t>(r)];
        (labels[i] > 0 ? pos : neg).push_back(i);
    }
    std::vector<int64_t>& major = pos.size() > neg.size() ? pos : neg;
    const size_t keep = std::min(pos.size(), neg.size());
    std::shuffle(major.begin(), major.end(), rng);
    major.resize(keep);
    if (keep == 0 || pos.size() + neg.size() < 2) return 2;
    std::vector<int64_t> all(pos);
    all.insert(all.end(), neg.begin(), neg.end());
    std::sort(all.begin(), all.end());
    std::copy(all.begin(), all.end(), train_idx);
    *n_train = static_cast<int64_t>(all.size());
    std::copy(perm.begin() + nt, perm.end(), test_idx);
    *n_test = n - nt;
    return 0;
}

extern "C" int oracle_zscore(double* train_cm, int64_t n_train, double* test_cm, int64_t n_test, int d,
                             double* means, double* stddevs) {
    if (n_train == 0) return 2;  // "empty training split"
    for (int j = 0; j < d; ++j) {
        double* col = train_cm + static_cast<int64_t>(j) * n_train;
        double s = 0.0;
        for (int64_t i = 0; i < n_train; ++i) s += col[i];
        const double mean = s / static_cast<double>(n_train);
        double q = 0.0;
        for (int64_t i = 0; i < n_train; ++i) q += (col[i] - mean) * (col[i] - mean);
        double sd = std::sqrt(q / static_cast<double>(n_train));
        if (sd < 1e-300) sd = 1.0;
        means[j] = mean;
        stddevs[j] = sd;
        for (int64_t i = 0; i < n_train; ++i) col[i] = (col[i] - mean) / sd;
        if (n_test > 0) {
            double* tc = test_cm + static_cast<int64_t>(j) * n_test;
            for (int64_t i = 0; i < n_test; ++i) tc[i] = (tc[i] - mean) / sd;
        }
    }
    return 0;
}
