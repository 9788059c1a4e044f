// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// C entry points into the reference's OWN host driver, compiled unmodified
// by path from /root/reference/proj/src (dataset, windowing, kernel,
// low_rank, saddle, ipm, pipeline) against oracle/shim2 (an Eigen subset;
// Eigen itself is absent from this image). Two libraries are built from this
// file (oracle/driver/Makefile):
//
//   oracle/_ref/libdriver_cpu.so  + the reference's src/fastsum.cpp (FFT on
//                                   oracle/shim/fftw3.h): the reference end
//                                   to end on the CPU;
//   oracle/_ref/libdriver_gpu.so  + paper_2312_00538_b200/cpp/ksvm_fastsum_gpu.cpp
//                                   (the drop-in fastsum.cpp on the B200 C
//                                   ABI), linked to libksvm_nfft.so: the
//                                   reference's IPM / GMRES / Nystrom /
//                                   pipeline code calling the GPU path.
//
// drv_train_pipeline runs ksvm::train_pipeline (P:src/pipeline.cpp:229-265)
// exactly as ksvm_train does (P:capi/ksvm_capi.cpp:264-284), then reports
// the TrainReport, the dual objective D(alpha) = sum(alpha) - 1/2 (y o
// alpha)^T K (y o alpha) (the reference never logs it; K is a
// fresh anova_fast_operator on the training split with fit 1/1.2, the
// operator train_on_prepared used), alpha, the bias and the held-out test
// split's decision values and labels (TrainedModel::decision_values on the
// de-normalised test points, as ksvm_predict_normalized does,
// P:capi/ksvm_capi.cpp:114-140).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "ksvm/fastsum.hpp"
#include "ksvm/pipeline.hpp"

namespace {
thread_local std::string t_err = "ok";

template <typename F>
int guarded(F&& f) {
    try {
        f();
        t_err = "ok";
        return 0;
    } catch (const ksvm::DataError& e) {
        t_err = e.what();
        return 2;
    } catch (const ksvm::DomainError& e) {
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
}  // namespace

extern "C" {

const char* drv_last_error(void) { return t_err.c_str(); }

// X: n x d row-major raw points; labels +-1. precond: 0 none, 1 cholesky-greedy,
// 4 nystrom-gaussian (ksvm::PrecondMethod order). fast: 1 fast backend (the
// path under test), 0 exact. Outputs (capacity n each): alpha, test decision
// values, test labels. scal[12] = {n_train, n_test, ipm_iters, mean_gmres,
// status, rank, xi_alpha, xi_lambda, mu_final, dual_objective, bias,
// dual_feasibility}.
int drv_train_pipeline(const double* X, const double* labels, int64_t n, int d, const char* windows,
                       int precond, int rank, double C, uint64_t seed, int fast, double* scal,
                       double* alpha_out, double* test_dec, double* test_lab) {
    return guarded([&] {
        ksvm::Dataset raw;
        raw.points.resize(n, d);
        raw.labels.resize(n);
        for (int64_t i = 0; i < n; ++i) {
            for (int j = 0; j < d; ++j) raw.points(i, j) = X[i * d + j];
            raw.labels[i] = labels[i];
        }
        ksvm::PipelineConfig cfg;
        cfg.seed = seed;
        cfg.explicit_windows = windows;
        cfg.backend = fast ? ksvm::OperatorBackend::kFast : ksvm::OperatorBackend::kExact;
        cfg.precond = static_cast<ksvm::PrecondMethod>(precond);
        cfg.rank = rank;
        cfg.ipm.C = C;
        ksvm::TrainReport rep;
        auto [model, test] = ksvm::train_pipeline(raw, cfg, rep);

        // dual objective on the training split
        ksvm::Dataset tr;
        tr.points = model.train_points;
        tr.labels = model.y;
        auto op = fast ? ksvm::anova_fast_operator(tr, model.kernel, model.fastsum, 1.0 / 1.2)
                       : ksvm::exact_operator(tr, model.kernel);
        const Eigen::VectorXd ya = model.y.cwiseProduct(model.alpha);
        const Eigen::VectorXd kya = op->apply(ya);
        const double dual = model.alpha.sum() - 0.5 * ya.dot(kya);

        // held-out predictions: decision_values re-applies the normalization
        Eigen::MatrixXd pts = test.points;
        for (Eigen::Index j = 0; j < pts.cols(); ++j) {
            const auto& s = model.normalization[static_cast<std::size_t>(j)];
            pts.col(j) = pts.col(j).array() * s.stddev + s.mean;
        }
        const Eigen::VectorXd f =
            model.decision_values(pts, fast ? ksvm::PredictBackend::kFast : ksvm::PredictBackend::kExact);

        const double s[12] = {static_cast<double>(rep.n_train), static_cast<double>(rep.n_test),
                              static_cast<double>(rep.ipm_iters), rep.mean_gmres, static_cast<double>(rep.status),
                              static_cast<double>(rep.rank), rep.xi_alpha, rep.xi_lambda, rep.mu_final, dual,
                              model.bias, model.dual_feasibility};
        std::memcpy(scal, s, sizeof(s));
        for (Eigen::Index i = 0; i < model.alpha.size(); ++i) alpha_out[i] = model.alpha[i];
        for (Eigen::Index i = 0; i < f.size(); ++i) {
            test_dec[i] = f[i];
            test_lab[i] = f[i] >= 0.0 ? 1.0 : -1.0;
        }
    });
}

// train_on_prepared's sequence (P:src/pipeline.cpp:195-227) called step by
// step on the reference's own functions - balance_and_split, zscore_fit_
// transform, anova_fast_operator (fit 1/1.2), build_precond_factor,
// ipm_train, make_model - in the same order and with the same arguments as
// train_pipeline, so every number equals drv_train_pipeline's bit for bit,
// plus the per-Newton-step log train_pipeline does not return:
// log[it * 6 + {0..5}] = {mu, xi_alpha_rel, xi_lambda_rel, step_alpha,
// gmres iterations, gmres converged} (capacity 6 * max_ip_iters).
int drv_train_steps(const double* X, const double* labels, int64_t n, int d, const char* windows, int precond,
                    int rank, double C, uint64_t seed, double* scal, double* alpha_out, double* test_dec,
                    double* log, int log_cap) {
    return guarded([&] {
        ksvm::Dataset raw;
        raw.points.resize(n, d);
        raw.labels.resize(n);
        for (int64_t i = 0; i < n; ++i) {
            for (int j = 0; j < d; ++j) raw.points(i, j) = X[i * d + j];
            raw.labels[i] = labels[i];
        }
        ksvm::PipelineConfig cfg;
        cfg.seed = seed;
        cfg.explicit_windows = windows;
        cfg.precond = static_cast<ksvm::PrecondMethod>(precond);
        cfg.rank = rank;
        cfg.ipm.C = C;
        auto [train, test] = ksvm::balance_and_split(raw, cfg.train_fraction, cfg.seed);
        ksvm::zscore_fit_transform(train, test);
        ksvm::AnovaKernelSpec spec;
        spec.windowing.windows = ksvm::parse_window_spec(cfg.explicit_windows, static_cast<int>(train.dim()));
        const int P = spec.windowing.num_windows();
        spec.windowing.weights.assign(static_cast<std::size_t>(P), 1.0 / P);
        spec.windowing.length_scales.assign(static_cast<std::size_t>(P), 1.0);
        spec.windowing.mi_scores.assign(static_cast<std::size_t>(train.dim()), 0.0);
        ksvm::check_windowing(spec.windowing, static_cast<int>(train.dim()));
        auto op = ksvm::anova_fast_operator(train, spec, cfg.fastsum, 1.0 / 1.2);
        ksvm::StackedFactor factor;
        const bool pre = cfg.precond != ksvm::PrecondMethod::kNone;
        if (pre) factor = ksvm::build_precond_factor(*op, train, spec, cfg, nullptr);
        ksvm::IpmResult res = ksvm::ipm_train(*op, train.labels, pre ? &factor : nullptr, cfg.ipm);
        ksvm::TrainedModel model = ksvm::make_model(res, train, spec, cfg.fastsum, *op, cfg.ipm.C);
        const Eigen::VectorXd ya = model.y.cwiseProduct(model.alpha);
        const Eigen::VectorXd kya = op->apply(ya);
        const double dual = model.alpha.sum() - 0.5 * ya.dot(kya);
        Eigen::MatrixXd pts = test.points;
        for (Eigen::Index j = 0; j < pts.cols(); ++j) {
            const auto& s = model.normalization[static_cast<std::size_t>(j)];
            pts.col(j) = pts.col(j).array() * s.stddev + s.mean;
        }
        const Eigen::VectorXd f = model.decision_values(pts, ksvm::PredictBackend::kFast);
        const double s[12] = {static_cast<double>(train.n()), static_cast<double>(test.n()),
                              static_cast<double>(res.iterations.size()), res.mean_gmres_iters(),
                              static_cast<double>(res.status), static_cast<double>(factor.rank()),
                              res.xi_alpha_rel, res.xi_lambda_rel, res.mu_final, dual, model.bias, res.lambda};
        std::memcpy(scal, s, sizeof(s));
        for (Eigen::Index i = 0; i < model.alpha.size(); ++i) alpha_out[i] = model.alpha[i];
        for (Eigen::Index i = 0; i < f.size(); ++i) test_dec[i] = f[i];
        int k = 0;
        for (const auto& it : res.iterations) {
            if (k >= log_cap) break;
            const double row[6] = {it.mu, it.xi_alpha_rel, it.xi_lambda_rel, it.step_alpha,
                                   static_cast<double>(it.gmres.iterations), it.gmres.converged ? 1.0 : 0.0};
            std::memcpy(log + 6 * k, row, sizeof(row));
            ++k;
        }
    });
}

// One GMRES solve of the reference (P:src/saddle.cpp:92-178) on the fast
// operator over the given (already normalized) points, with the reference's
// SaddlePreconditioner built from a stacked factor Z (k x n row-major, k = 0:
// identity). Returns iterations / residual; x receives n + 1 entries.
int drv_gmres(const double* X, int64_t n, int d, const char* windows, const double* y, const double* theta,
              const double* Z, int k, const double* rhs, double tol, int max_iter, double* x, double* scal) {
    return guarded([&] {
        ksvm::Dataset ds;
        ds.points.resize(n, d);
        for (int64_t i = 0; i < n; ++i)
            for (int j = 0; j < d; ++j) ds.points(i, j) = X[i * d + j];
        ksvm::AnovaKernelSpec spec;
        spec.windowing.windows = ksvm::parse_window_spec(windows, d);
        const int P = spec.windowing.num_windows();
        spec.windowing.weights.assign(static_cast<std::size_t>(P), 1.0 / P);
        spec.windowing.length_scales.assign(static_cast<std::size_t>(P), 1.0);
        auto op = ksvm::anova_fast_operator(ds, spec, ksvm::FastsumConfig{}, 1.0 / 1.2);
        Eigen::VectorXd yv(n), th(n), r(n + 1);
        for (int64_t i = 0; i < n; ++i) {
            yv[i] = y[i];
            th[i] = theta[i];
        }
        for (int64_t i = 0; i <= n; ++i) r[i] = rhs[i];
        ksvm::StackedFactor f;
        if (k > 0) {
            f.Z.resize(k, n);
            for (int a = 0; a < k; ++a)
                for (int64_t i = 0; i < n; ++i) f.Z(a, i) = Z[a * n + i];
        }
        ksvm::SaddleOperator A(*op, yv, th);
        ksvm::SaddlePreconditioner Pc(k > 0 ? &f : nullptr, yv);
        Pc.refresh(th);
        auto [sol, st] = ksvm::gmres_solve(A, Pc, r, tol, max_iter);
        for (int64_t i = 0; i <= n; ++i) x[i] = sol[i];
        scal[0] = st.iterations;
        scal[1] = st.relative_residual;
        scal[2] = st.converged ? 1.0 : 0.0;
        scal[3] = Pc.diagonal_fallback() ? 1.0 : 0.0;
    });
}

}  // extern "C"
