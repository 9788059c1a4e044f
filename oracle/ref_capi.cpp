// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// C wrapper around the reference's OWN hot-path code. oracle/Makefile
// compiles this file together with /root/reference/proj/src/{fastsum,kernel,
// windowing}.cpp — unmodified, by path — against the Eigen/FFTW shims in
// oracle/shim, into oracle/_ref/libref.so (git-ignored; it travels to the
// GPU box with the snapshot). No reference source is copied into this repo.
#include <cstring>
#include <stdexcept>
#include <string>

#include "ksvm/fastsum.hpp"
#include "ksvm/kernel.hpp"
#include "ksvm/windowing.hpp"
#include "ksvm/dataset.hpp"
#include "ksvm_oracle.h"

namespace {
thread_local std::string t_err = "ok";

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ksvm::DomainError& e) {
        t_err = e.what();
        return 2;
    } catch (const ksvm::DataError& e) {
        t_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        t_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        t_err = e.what();
        return 5;
    }
}

Eigen::MatrixXd colmajor(const double* p, int64_t n, int d) {
    Eigen::MatrixXd m(n, d);
    std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(n * d));
    return m;
}

ksvm::FastsumConfig make_cfg(int N, int m, int sigma, double rT) {
    ksvm::FastsumConfig c;
    c.bandwidth = N;
    c.window_cutoff = m;
    c.oversampling = sigma;
    c.torus_radius = rT;
    return c;
}
}  // namespace

struct ref_plan {
    ksvm::FastsumPlan plan;
    int d;
};

struct ref_anova {
    std::unique_ptr<ksvm::KernelOperator> op;
};

extern "C" {

const char* ref_last_error(void) { return t_err.c_str(); }

int ref_plan_create(const double* pts, int64_t n, int d, double ell, int N, int m, int sigma,
                    double rT, double fit, ref_plan** out) {
    return guard([&] {
        auto p = ksvm::plan_fastsum(colmajor(pts, n, d), ksvm::GaussianKernelSpec{ell},
                                    make_cfg(N, m, sigma, rT), fit);
        *out = new ref_plan{std::move(p), d};
    });
}

int ref_plan_apply(const ref_plan* p, const double* v, double* out) {
    return guard([&] {
        Eigen::VectorXd vv(p->plan.num_sources());
        std::memcpy(vv.data(), v, sizeof(double) * static_cast<std::size_t>(vv.size()));
        const Eigen::VectorXd r = ksvm::apply_fastsum(p->plan, vv);
        std::memcpy(out, r.data(), sizeof(double) * static_cast<std::size_t>(r.size()));
    });
}

int ref_plan_apply_cross(const ref_plan* p, const double* targets, int64_t t, const double* v,
                         double* out) {
    return guard([&] {
        Eigen::VectorXd vv(p->plan.num_sources());
        std::memcpy(vv.data(), v, sizeof(double) * static_cast<std::size_t>(vv.size()));
        const Eigen::VectorXd r = ksvm::apply_fastsum_cross(p->plan, colmajor(targets, t, p->d), vv);
        std::memcpy(out, r.data(), sizeof(double) * static_cast<std::size_t>(r.size()));
    });
}

double ref_plan_scaled_length(const ref_plan* p) { return p->plan.scaled_length(); }
double ref_plan_coefficient_sum(const ref_plan* p) { return p->plan.coefficient_sum(); }

int ref_plan_scale_points(const ref_plan* p, const double* pts, int64_t t, double* out) {
    return guard([&] {
        const Eigen::MatrixXd r = p->plan.scale_points(colmajor(pts, t, p->d));
        std::memcpy(out, r.data(), sizeof(double) * static_cast<std::size_t>(t * p->d));
    });
}

void ref_plan_free(ref_plan* p) { delete p; }

int ref_anova_create(const double* pts_rm, int64_t n, int d, const int* feats, const int* sizes,
                     int P, const double* weights, const double* ells, int N, int m, int sigma,
                     double rT, double fit, ref_anova** out) {
    return guard([&] {
        ksvm::Dataset data;
        data.points = Eigen::MatrixXd(n, d);
        for (int64_t i = 0; i < n; ++i)
            for (int j = 0; j < d; ++j) data.points(i, j) = pts_rm[i * d + j];
        data.labels = Eigen::VectorXd(n);
        ksvm::AnovaKernelSpec spec;
        int off = 0;
        for (int l = 0; l < P; ++l) {
            spec.windowing.windows.emplace_back(feats + off, feats + off + sizes[l]);
            off += sizes[l];
            spec.windowing.weights.push_back(weights[l]);
            spec.windowing.length_scales.push_back(ells[l]);
        }
        spec.windowing.mi_scores.assign(static_cast<std::size_t>(d), 0.0);
        *out = new ref_anova{ksvm::anova_fast_operator(data, spec, make_cfg(N, m, sigma, rT), fit)};
    });
}

int ref_anova_apply(const ref_anova* op, const double* v, double* out) {
    return guard([&] {
        Eigen::VectorXd vv(op->op->size());
        std::memcpy(vv.data(), v, sizeof(double) * static_cast<std::size_t>(vv.size()));
        const Eigen::VectorXd r = op->op->apply(vv);
        std::memcpy(out, r.data(), sizeof(double) * static_cast<std::size_t>(r.size()));
    });
}

double ref_anova_entry(const ref_anova* op, int64_t i, int64_t j) { return op->op->entry(i, j); }

void ref_anova_free(ref_anova* op) { delete op; }

}  // extern "C"

// ---- P:src/dataset.cpp: the reference's own split / z-score ---------------
// balance_and_split returns datasets, not indices: the wrapper feeds a 1-column
// dataset whose entries are the row numbers and reads them back.
extern "C" int ref_balance_and_split(const double* labels, int64_t n, double train_fraction, uint64_t seed,
                                     int64_t* train_idx, int64_t* n_train, int64_t* test_idx, int64_t* n_test) {
    return guard([&] {
        ksvm::Dataset d;
        d.points = Eigen::MatrixXd(n, 1);
        d.labels = Eigen::VectorXd(n);
        for (int64_t i = 0; i < n; ++i) {
            d.points(i, 0) = static_cast<double>(i);
            d.labels[i] = labels[i];
        }
        auto [tr, te] = ksvm::balance_and_split(d, train_fraction, seed);
        *n_train = tr.n();
        *n_test = te.n();
        for (int64_t i = 0; i < tr.n(); ++i) train_idx[i] = static_cast<int64_t>(tr.points(i, 0));
        for (int64_t i = 0; i < te.n(); ++i) test_idx[i] = static_cast<int64_t>(te.points(i, 0));
    });
}

extern "C" int ref_zscore(double* train_cm, int64_t n_train, double* test_cm, int64_t n_test, int d, double* means,
                          double* stddevs) {
    return guard([&] {
        ksvm::Dataset tr, te;
        tr.points = colmajor(train_cm, n_train, d);
        te.points = n_test > 0 ? colmajor(test_cm, n_test, d) : Eigen::MatrixXd(0, d);
        ksvm::zscore_fit_transform(tr, te);
        std::memcpy(train_cm, tr.points.data(), sizeof(double) * static_cast<std::size_t>(n_train * d));
        if (n_test > 0) std::memcpy(test_cm, te.points.data(), sizeof(double) * static_cast<std::size_t>(n_test * d));
        for (int j = 0; j < d; ++j) {
            means[j] = (*tr.normalization)[static_cast<std::size_t>(j)].mean;
            stddevs[j] = (*tr.normalization)[static_cast<std::size_t>(j)].stddev;
        }
    });
}
