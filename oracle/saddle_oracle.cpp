// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Eigen-free restatement of the reference's Newton saddle system solver
// (P:src/saddle.cpp, P:include/ksvm/saddle.hpp), the caller of the ANOVA
// matvec that SURVEY.md 8(f) ranks first for a GPU-resident version:
//   * SaddleOperator::apply            P:src/saddle.cpp:22-33
//   * SaddlePreconditioner::refresh    P:src/saddle.cpp:41-63
//   * SaddlePreconditioner::apply      P:src/saddle.cpp:65-90
//   * gmres_solve                      P:src/saddle.cpp:92-178
// with the same arithmetic order (modified Gram-Schmidt with one
// re-orthogonalisation pass, Givens rotations, upper-triangular back
// substitution). The capacitance LU uses row partial pivoting like
// Eigen::PartialPivLU; the reciprocal condition number is computed exactly
// from the inverse's 1-norm (Eigen estimates it), which only matters for the
// rcond < 1e-15 fallback decision.
//
// K is either an oracle ANOVA operator (the NFFT matvec) or a dense
// row-major n x n matrix (the reference tests' DenseOperator,
// P:tests/helpers.hpp).
//
// Also the interior point loop around it (P:src/ipm.cpp): ipm_train
// (:76-155) with assemble_newton_rhs (:31-42), step_lengths (:44-55),
// barrier_diagonal (:59-64), initial_alpha (:66-74, libstdc++ mt19937_64 and
// uniform_real_distribution as in the reference build), and compute_bias
// (:157-185); plus the tests' blobs generator (P:tests/helpers.hpp:41-56).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "ksvm_oracle.h"

namespace {

thread_local std::string t_err;

using Vec = std::vector<double>;

struct KOp {
    const oracle_anova* op;
    const double* dense;
    int64_t n;
    void apply(const Vec& v, Vec& out) const {
        out.assign(static_cast<size_t>(n), 0.0);
        if (dense) {
            for (int64_t i = 0; i < n; ++i) {
                double s = 0.0;
                const double* row = dense + i * n;
                for (int64_t j = 0; j < n; ++j) s += row[j] * v[static_cast<size_t>(j)];
                out[static_cast<size_t>(i)] = s;
            }
        } else if (oracle_anova_apply(op, v.data(), out.data()) != 0) {
            throw std::runtime_error(oracle_last_error());
        }
    }
};

// P:src/saddle.cpp:22-33
void saddle_apply(const KOp& K, const double* y, const double* theta, const Vec& vw, Vec& out) {
    const int64_t n = K.n;
    Vec yv(static_cast<size_t>(n)), kv;
    for (int64_t j = 0; j < n; ++j) yv[static_cast<size_t>(j)] = y[j] * vw[static_cast<size_t>(j)];
    K.apply(yv, kv);
    const double w = vw[static_cast<size_t>(n)];
    out.assign(static_cast<size_t>(n) + 1, 0.0);
    double dot = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        out[static_cast<size_t>(j)] = y[j] * kv[static_cast<size_t>(j)] + theta[j] * vw[static_cast<size_t>(j)] - w * y[j];
        dot += y[j] * vw[static_cast<size_t>(j)];
    }
    out[static_cast<size_t>(n)] = -dot;
}

struct Precond {
    const double* Z = nullptr;  // k x n row-major
    int k = 0;
    int64_t n = 0;
    const double* y = nullptr;
    Vec theta;
    bool identity = false, fallback = false, fresh = false;
    std::vector<double> lu;  // k x k, row-major, L unit lower + U
    std::vector<int> piv;

    // P:src/saddle.cpp:41-63
    void refresh(const double* th) {
        for (int64_t j = 0; j < n; ++j)
            if (!(th[j] > 0.0)) throw std::invalid_argument("SaddlePreconditioner: bad Theta");
        theta.assign(th, th + n);
        fallback = false;
        fresh = true;
        if (identity || k == 0) return;
        std::vector<double> cap(static_cast<size_t>(k) * k, 0.0);
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) {
                double s = 0.0;
                for (int64_t j = 0; j < n; ++j) s += Z[a * n + j] * (1.0 / theta[static_cast<size_t>(j)]) * Z[b * n + j];
                cap[static_cast<size_t>(a) * k + b] = (a == b ? 1.0 : 0.0) + s;
            }
        for (double c : cap)
            if (!std::isfinite(c)) {
                fallback = true;
                return;
            }
        // partial-pivot LU
        lu = cap;
        piv.resize(static_cast<size_t>(k));
        double anorm = 0.0;  // 1-norm of cap
        for (int b = 0; b < k; ++b) {
            double s = 0.0;
            for (int a = 0; a < k; ++a) s += std::fabs(cap[static_cast<size_t>(a) * k + b]);
            anorm = std::max(anorm, s);
        }
        bool singular = false;
        for (int c = 0; c < k; ++c) {
            int p = c;
            for (int r = c + 1; r < k; ++r)
                if (std::fabs(lu[static_cast<size_t>(r) * k + c]) > std::fabs(lu[static_cast<size_t>(p) * k + c])) p = r;
            piv[static_cast<size_t>(c)] = p;
            if (p != c)
                for (int q = 0; q < k; ++q) std::swap(lu[static_cast<size_t>(c) * k + q], lu[static_cast<size_t>(p) * k + q]);
            const double d = lu[static_cast<size_t>(c) * k + c];
            if (d == 0.0) {
                singular = true;
                continue;
            }
            for (int r = c + 1; r < k; ++r) {
                const double f = lu[static_cast<size_t>(r) * k + c] / d;
                lu[static_cast<size_t>(r) * k + c] = f;
                for (int q = c + 1; q < k; ++q) lu[static_cast<size_t>(r) * k + q] -= f * lu[static_cast<size_t>(c) * k + q];
            }
        }
        if (singular) {
            fallback = true;
            return;
        }
        double inorm = 0.0;  // 1-norm of the inverse, column by column
        for (int b = 0; b < k; ++b) {
            Vec e(static_cast<size_t>(k), 0.0);
            e[static_cast<size_t>(b)] = 1.0;
            solve(e);
            double s = 0.0;
            for (double x : e) s += std::fabs(x);
            inorm = std::max(inorm, s);
        }
        const double rcond = 1.0 / (anorm * inorm);
        if (!std::isfinite(rcond) || rcond < 1e-15) fallback = true;
    }

    void solve(Vec& b) const {  // in place, P A = L U
        for (int c = 0; c < k; ++c) std::swap(b[static_cast<size_t>(c)], b[static_cast<size_t>(piv[static_cast<size_t>(c)])]);
        for (int r = 0; r < k; ++r)
            for (int c = 0; c < r; ++c) b[static_cast<size_t>(r)] -= lu[static_cast<size_t>(r) * k + c] * b[static_cast<size_t>(c)];
        for (int r = k - 1; r >= 0; --r) {
            for (int c = r + 1; c < k; ++c) b[static_cast<size_t>(r)] -= lu[static_cast<size_t>(r) * k + c] * b[static_cast<size_t>(c)];
            b[static_cast<size_t>(r)] /= lu[static_cast<size_t>(r) * k + r];
        }
    }

    // P:src/saddle.cpp:65-90
    void apply(const Vec& g, Vec& out) const {
        if (identity) {
            out = g;
            return;
        }
        if (!fresh) throw std::logic_error("SaddlePreconditioner: refresh() before apply()");
        Vec x1(static_cast<size_t>(n));
        if (fallback || k == 0) {
            for (int64_t j = 0; j < n; ++j) x1[static_cast<size_t>(j)] = g[static_cast<size_t>(j)] / theta[static_cast<size_t>(j)];
        } else {
            Vec t(static_cast<size_t>(n)), zt(static_cast<size_t>(k), 0.0);
            for (int64_t j = 0; j < n; ++j) t[static_cast<size_t>(j)] = y[j] * g[static_cast<size_t>(j)] / theta[static_cast<size_t>(j)];
            for (int a = 0; a < k; ++a) {
                double s = 0.0;
                for (int64_t j = 0; j < n; ++j) s += Z[a * n + j] * t[static_cast<size_t>(j)];
                zt[static_cast<size_t>(a)] = s;
            }
            solve(zt);
            for (int64_t j = 0; j < n; ++j) {
                double s = 0.0;
                for (int a = 0; a < k; ++a) s += Z[a * n + j] * zt[static_cast<size_t>(a)];
                x1[static_cast<size_t>(j)] = g[static_cast<size_t>(j)] / theta[static_cast<size_t>(j)] - y[j] * s / theta[static_cast<size_t>(j)];
            }
        }
        out.assign(static_cast<size_t>(n) + 1, 0.0);
        double dot = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            out[static_cast<size_t>(j)] = x1[static_cast<size_t>(j)];
            dot += y[j] * x1[static_cast<size_t>(j)];
        }
        out[static_cast<size_t>(n)] = -dot - g[static_cast<size_t>(n)];
    }
};

double dotv(const Vec& a, const Vec& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        t_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        t_err = e.what();
        return 5;
    }
}

// gmres_solve (P:src/saddle.cpp:92-178) with a refreshed preconditioner
void gmres_core(const KOp& K, const double* y, const double* theta, const Precond& P, const double* rhs, double tol,
                int max_iter, double* x_out, double* stats, double* history) {
    const int64_t n = K.n;
        const size_t N1 = static_cast<size_t>(n) + 1;
    Vec r(rhs, rhs + N1);
    int iterations = 0;
    bool converged = false, breakdown = false;
    const double rhs_norm = std::sqrt(dotv(r, r));
    if (rhs_norm == 0.0) {
        std::memset(x_out, 0, sizeof(double) * N1);
        stats[0] = 0;
        stats[1] = 0.0;
        stats[2] = 1;
        stats[3] = 0;
        return;
    }
    std::vector<Vec> basis;
    basis.push_back(r);
    for (double& e : basis[0]) e /= rhs_norm;
    const size_t MI = static_cast<size_t>(max_iter);
    std::vector<double> H((MI + 1) * MI, 0.0);
    auto h = [&](size_t i, size_t j) -> double& { return H[i * MI + j]; };
    Vec cs(MI, 0.0), sn(MI, 0.0), beta(MI + 1, 0.0);
    beta[0] = rhs_norm;
    int kk = 0;
    Vec z, w;
    for (; kk < max_iter; ++kk) {
        P.apply(basis[static_cast<size_t>(kk)], z);
        saddle_apply(K, y, theta, z, w);
        for (int pass = 0; pass < 2; ++pass)
            for (int i = 0; i <= kk; ++i) {
                const double hv = dotv(w, basis[static_cast<size_t>(i)]);
                h(static_cast<size_t>(i), static_cast<size_t>(kk)) += hv;
                for (size_t q = 0; q < N1; ++q) w[q] -= hv * basis[static_cast<size_t>(i)][q];
            }
        const double hnext = std::sqrt(dotv(w, w));
        h(static_cast<size_t>(kk) + 1, static_cast<size_t>(kk)) = hnext;
        for (int i = 0; i < kk; ++i) {
            const size_t I = static_cast<size_t>(i), KK = static_cast<size_t>(kk);
            const double tmp = cs[I] * h(I, KK) + sn[I] * h(I + 1, KK);
            h(I + 1, KK) = -sn[I] * h(I, KK) + cs[I] * h(I + 1, KK);
            h(I, KK) = tmp;
        }
        const size_t KK = static_cast<size_t>(kk);
        const double denom = std::hypot(h(KK, KK), h(KK + 1, KK));
        if (denom == 0.0) {
            breakdown = true;
            break;
        }
        cs[KK] = h(KK, KK) / denom;
        sn[KK] = h(KK + 1, KK) / denom;
        h(KK, KK) = denom;
        h(KK + 1, KK) = 0.0;
        beta[KK + 1] = -sn[KK] * beta[KK];
        beta[KK] = cs[KK] * beta[KK];
        const double rel = std::fabs(beta[KK + 1]) / rhs_norm;
        if (history) history[iterations] = rel;
        ++iterations;
        if (rel <= tol) {
            ++kk;
            converged = true;
            break;
        }
        if (hnext <= 1e-14 * rhs_norm) {
            breakdown = true;
            converged = true;
            ++kk;
            break;
        }
        Vec nb(w);
        for (double& e : nb) e /= hnext;
        basis.push_back(std::move(nb));
    }
    Vec u(N1, 0.0);
    if (kk > 0) {
        Vec yk(static_cast<size_t>(kk));
        for (int i = kk - 1; i >= 0; --i) {
            double s = beta[static_cast<size_t>(i)];
            for (int j = i + 1; j < kk; ++j) s -= h(static_cast<size_t>(i), static_cast<size_t>(j)) * yk[static_cast<size_t>(j)];
            yk[static_cast<size_t>(i)] = s / h(static_cast<size_t>(i), static_cast<size_t>(i));
        }
        for (int i = 0; i < kk; ++i)
            for (size_t q = 0; q < N1; ++q) u[q] += yk[static_cast<size_t>(i)] * basis[static_cast<size_t>(i)][q];
    }
    Vec x, ax;
    P.apply(u, x);
    saddle_apply(K, y, theta, x, ax);
    double rr = 0.0;
    for (size_t q = 0; q < N1; ++q) rr += (rhs[q] - ax[q]) * (rhs[q] - ax[q]);
    const double rel_res = std::sqrt(rr) / rhs_norm;
    if (rel_res <= tol) converged = true;
    std::memcpy(x_out, x.data(), sizeof(double) * N1);
    stats[0] = iterations;
    stats[1] = rel_res;
    stats[2] = converged ? 1 : 0;
    stats[3] = breakdown ? 1 : 0;
}

}  // namespace

extern "C" {

const char* oracle_saddle_last_error(void) { return t_err.c_str(); }

int oracle_saddle_apply(const oracle_anova* op, const double* dense, int64_t n, const double* y,
                        const double* theta, const double* vw, double* out) {
    return guarded([&] {
        KOp K{op, dense, n};
        Vec v(vw, vw + n + 1), o;
        saddle_apply(K, y, theta, v, o);
        std::memcpy(out, o.data(), sizeof(double) * (n + 1));
    });
}

int oracle_precond_apply(const double* Z, int k, int64_t n, const double* y, const double* theta,
                         const double* g, double* out, int* fallback) {
    return guarded([&] {
        Precond P;
        P.Z = Z;
        P.k = Z ? k : 0;
        P.n = n;
        P.y = y;
        P.identity = Z == nullptr;
        P.refresh(theta);
        Vec gv(g, g + n + 1), o;
        P.apply(gv, o);
        std::memcpy(out, o.data(), sizeof(double) * (n + 1));
        if (fallback) *fallback = P.fallback ? 1 : 0;
    });
}

// stats: [iterations, relative_residual, converged, breakdown]
int oracle_gmres_solve(const oracle_anova* op, const double* dense, int64_t n, const double* y,
                       const double* theta, const double* Z, int k, const double* rhs, double tol,
                       int max_iter, double* x_out, double* stats, double* history) {
    return guarded([&] {
        if (!(tol > 0.0)) throw std::invalid_argument("gmres tol must be positive");
        KOp K{op, dense, n};
        Precond P;
        P.Z = Z;
        P.k = Z ? k : 0;
        P.n = n;
        P.y = y;
        P.identity = Z == nullptr;
        P.refresh(theta);
        gmres_core(K, y, theta, P, rhs, tol, max_iter, x_out, stats, history);
    });
}

// cfg: {C, sigma, gamma0, tol_ip, max_ip_iters, tol_gmres, max_gmres_iters, mu0} (IpmConfig)
// res: {lambda, mu_final, xi_alpha_rel, xi_lambda_rel, status, iterations, mean_gmres_iters}
//      status 0 converged, 1 max iterations, 2 stalled
// log (may be NULL): per iteration {mu, xi_alpha_rel, xi_lambda_rel, step_alpha, gmres_iters, gmres_converged}
int oracle_ipm_train(const oracle_anova* op, const double* dense, int64_t n, const double* y, const double* Z, int k,
                     const double* cfg, double* alpha_out, double* res, double* log) {
    return guarded([&] {
        const double C = cfg[0], sigma = cfg[1], gamma0 = cfg[2], tol_ip = cfg[3], tol_gmres = cfg[5], mu0 = cfg[7];
        const int max_ip = static_cast<int>(cfg[4]), max_gm = static_cast<int>(cfg[6]);
        if (!(C > 0.0)) throw std::invalid_argument("C must be positive");  // P:src/ipm.cpp:10-21
        if (!(sigma > 0.0 && sigma < 1.0)) throw std::invalid_argument("sigma must lie in (0, 1)");
        if (!(gamma0 > 0.0 && gamma0 < 1.0)) throw std::invalid_argument("gamma0 must lie in (0, 1)");
        if (!(tol_ip > 0.0) || !(tol_gmres > 0.0)) throw std::invalid_argument("tolerances must be positive");
        if (max_ip < 1 || max_gm < 1) throw std::invalid_argument("iteration caps must be >= 1");
        if (!(mu0 > 0.0)) throw std::invalid_argument("mu0 must be positive");
        for (int64_t i = 0; i < n; ++i)
            if (y[i] != 1.0 && y[i] != -1.0) throw std::invalid_argument("ipm_train: labels must be +-1");
        const size_t N = static_cast<size_t>(n);
        KOp K{op, dense, n};
        Vec alpha(N);
        {
            std::mt19937_64 rng(0x5EED5EEDull);
            std::uniform_real_distribution<double> unif(0.0, 1.0);
            for (size_t j = 0; j < N; ++j) alpha[j] = C * (0.4 + 0.2 * unif(rng));
        }
        double lambda = 0.0, mu = mu0;
        auto yky = [&](const Vec& a, Vec& out) {
            Vec ya(N), ka;
            for (size_t j = 0; j < N; ++j) ya[j] = y[j] * a[j];
            K.apply(ya, ka);
            out.resize(N);
            for (size_t j = 0; j < N; ++j) out[j] = y[j] * ka[j];
        };
        auto rhs_of = [&](const Vec& a, double lam, const Vec& ykya, double m, Vec& rhs) {
            rhs.assign(N + 1, 0.0);
            double dot = 0.0;
            for (size_t j = 0; j < N; ++j) {
                rhs[j] = 1.0 - ykya[j] + lam * y[j] + m * (1.0 / a[j]) - m * (1.0 / (C - a[j]));
                dot += y[j] * a[j];
            }
            rhs[N] = dot;
        };
        auto head_norm = [&](const Vec& v) {
            double s = 0.0;
            for (size_t j = 0; j < N; ++j) s += v[j] * v[j];
            return std::sqrt(s);
        };
        Vec ykya, rhs;
        yky(alpha, ykya);
        double ya = 0.0;
        for (size_t j = 0; j < N; ++j) ya += y[j] * alpha[j];
        const double xi_alpha0 = std::fabs(ya);
        rhs_of(alpha, lambda, ykya, mu, rhs);
        const double xi_lambda0 = head_norm(rhs);
        if (xi_alpha0 == 0.0 || xi_lambda0 == 0.0)
            throw std::runtime_error("ipm_train: degenerate initial infeasibility");
        Precond P;
        P.Z = Z;
        P.k = Z ? k : 0;
        P.n = n;
        P.y = y;
        P.identity = Z == nullptr;
        double xi_a = 1.0, xi_l = 1.0;
        int it = 0, streak = 0, status = -1;
        double gm_sum = 0.0;
        Vec theta(N), delta(N + 1);
        while ((mu > tol_ip || xi_a > tol_ip || xi_l > tol_ip) && it < max_ip) {
            mu *= sigma;
            for (size_t j = 0; j < N; ++j)
                theta[j] = mu * (1.0 / (alpha[j] * alpha[j]) + 1.0 / ((C - alpha[j]) * (C - alpha[j])));
            P.refresh(theta.data());
            rhs_of(alpha, lambda, ykya, mu, rhs);
            double st[4];
            gmres_core(K, y, theta.data(), P, rhs.data(), tol_gmres, max_gm, delta.data(), st, nullptr);
            double smax = 1.0;  // step_lengths (P:src/ipm.cpp:44-55)
            for (size_t j = 0; j < N; ++j) {
                if (delta[j] < 0.0)
                    smax = std::min(smax, -alpha[j] / delta[j]);
                else if (delta[j] > 0.0)
                    smax = std::min(smax, (C - alpha[j]) / delta[j]);
            }
            const double s_alpha = gamma0 * smax, s_lambda = gamma0;
            for (size_t j = 0; j < N; ++j) alpha[j] += s_alpha * delta[j];
            lambda += s_lambda * delta[N];
            yky(alpha, ykya);
            ya = 0.0;
            for (size_t j = 0; j < N; ++j) ya += y[j] * alpha[j];
            xi_a = std::fabs(ya) / xi_alpha0;
            rhs_of(alpha, lambda, ykya, mu, rhs);
            xi_l = head_norm(rhs) / xi_lambda0;
            if (log) {
                double* L = log + 6 * it;
                L[0] = mu;
                L[1] = xi_a;
                L[2] = xi_l;
                L[3] = s_alpha;
                L[4] = st[0];
                L[5] = st[2];
            }
            gm_sum += st[0];
            ++it;
            streak = st[2] == 0.0 ? streak + 1 : 0;
            if (streak > 3) {
                status = 2;
                break;
            }
        }
        if (status != 2) status = (mu <= tol_ip && xi_a <= tol_ip && xi_l <= tol_ip) ? 0 : 1;
        std::memcpy(alpha_out, alpha.data(), sizeof(double) * N);
        res[0] = lambda;
        res[1] = mu;
        res[2] = xi_a;
        res[3] = xi_l;
        res[4] = status;
        res[5] = it;
        res[6] = it ? gm_sum / it : 0.0;
    });
}

// P:src/ipm.cpp:157-185 (no support vectors: 0, the reference also warns)
int oracle_compute_bias(const oracle_anova* op, const double* dense, int64_t n, const double* alpha, const double* y,
                        double C, double eps_sv, double* bias) {
    return guarded([&] {
        KOp K{op, dense, n};
        Vec ay(static_cast<size_t>(n)), kay;
        for (int64_t j = 0; j < n; ++j) ay[static_cast<size_t>(j)] = alpha[j] * y[j];
        K.apply(ay, kay);
        std::vector<double> free_vals, sv_vals;
        for (int64_t j = 0; j < n; ++j) {
            if (alpha[j] > eps_sv) {
                const double val = y[j] - kay[static_cast<size_t>(j)];
                sv_vals.push_back(val);
                if (alpha[j] < C - eps_sv) free_vals.push_back(val);
            }
        }
        if (!free_vals.empty()) {
            double sum = 0.0;
            for (double v : free_vals) sum += v;
            *bias = sum / static_cast<double>(free_vals.size());
        } else if (!sv_vals.empty()) {
            std::nth_element(sv_vals.begin(), sv_vals.begin() + sv_vals.size() / 2, sv_vals.end());
            double med = sv_vals[sv_vals.size() / 2];
            if (sv_vals.size() % 2 == 0) {
                const double lower = *std::max_element(sv_vals.begin(), sv_vals.begin() + sv_vals.size() / 2);
                med = 0.5 * (med + lower);
            }
            *bias = med;
        } else {
            *bias = 0.0;
        }
    });
}

// helpers::blobs (P:tests/helpers.hpp:41-56): n x d column-major points, labels
void oracle_blobs(int64_t n, int64_t d, double gap, uint64_t seed, double noise, double* pts_cm, double* labels) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> normal(0.0, noise);
    for (int64_t i = 0; i < n; ++i) {
        const double label = i % 2 == 0 ? 1.0 : -1.0;
        const double center = label * gap / 2.0;
        for (int64_t j = 0; j < d; ++j) pts_cm[j * n + i] = center + normal(rng);
        labels[i] = label;
    }
}

}  // extern "C"
