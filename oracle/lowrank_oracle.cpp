// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Eigen-free restatement of the reference's greedy pivoted Cholesky
// (P:src/low_rank.cpp:25-92, pivoted_cholesky_impl + pivoted_cholesky_greedy)
// over the exact kernel entries the IPM preconditioner uses:
//   window >= 0: WindowOperator::entry (P:src/pipeline.cpp:103-105),
//                exp(-||x_i - x_j||^2 / ell^2) on the window's coordinates;
//   window == -1: anova_entry (P:src/kernel.cpp:33-48), sum_l w_l exp(...).
// Points are row-major n x d (the dataset's features). Z is rank x n
// row-major (LowRankFactor::Z). Status 4: rank < 1 (invalid_argument);
// 5: the reference's non-PSD runtime_errors.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string t_err;

struct Entries {
    const double* pts;
    int64_t n;
    int d;
    std::vector<std::vector<int>> wins;
    std::vector<double> w, ell;
    int window;
    double operator()(int64_t i, int64_t j) const {
        double sum = 0.0;
        for (size_t l = 0; l < wins.size(); ++l) {
            if (window >= 0 && static_cast<int>(l) != window) continue;
            double d2 = 0.0;
            for (int f : wins[l]) {
                const double diff = pts[i * d + f] - pts[j * d + f];
                d2 += diff * diff;
            }
            const double e = std::exp(-d2 / (ell[l] * ell[l]));
            if (window >= 0) return e;
            sum += w[l] * e;
        }
        return sum;
    }
};

template <class Entry>
int pivoted_core(const Entry& E, int64_t n, int rank, double err_tol, double* Z_out, int* achieved_rank,
                 double* trace_residual, int64_t* pivots) {
    try {
        if (rank < 1) throw std::invalid_argument("rank must be >= 1");
        rank = static_cast<int>(std::min<int64_t>(rank, n));
        std::vector<double> diag(static_cast<size_t>(n));
        for (int64_t j = 0; j < n; ++j) diag[static_cast<size_t>(j)] = E(j, j);
        double initial_trace = 0.0;
        for (double x : diag) initial_trace += x;
        std::vector<double> Z(static_cast<size_t>(rank) * n, 0.0), row(static_cast<size_t>(n));
        int r = 0;
        while (r < rank) {
            double mx = diag[0], sm = 0.0;
            for (double x : diag) {
                mx = std::max(mx, x);
                sm += x;
            }
            if (mx <= err_tol || sm <= err_tol) break;  // greedy stop (P:src/low_rank.cpp:82-84)
            int64_t p = 0;                               // largest, smallest index on ties (:75-79)
            for (int64_t j = 1; j < n; ++j)
                if (diag[static_cast<size_t>(j)] > diag[static_cast<size_t>(p)]) p = j;
            const double dp = diag[static_cast<size_t>(p)];
            if (dp <= 0.0) {
                if (dp < -1e-10 * std::max(1.0, initial_trace))
                    throw std::runtime_error("pivoted Cholesky: negative pivot, operator not PSD");
                break;
            }
            const double root = std::sqrt(dp);
            for (int64_t j = 0; j < n; ++j) {
                double s = 0.0;
                for (int i = 0; i < r; ++i) s += Z[static_cast<size_t>(i) * n + j] * Z[static_cast<size_t>(i) * n + p];
                row[static_cast<size_t>(j)] = (E(p, j) - s) / root;
            }
            double mn = 0.0;
            for (int64_t j = 0; j < n; ++j) {
                Z[static_cast<size_t>(r) * n + j] = row[static_cast<size_t>(j)];
                diag[static_cast<size_t>(j)] -= row[static_cast<size_t>(j)] * row[static_cast<size_t>(j)];
                mn = j == 0 ? diag[0] : std::min(mn, diag[static_cast<size_t>(j)]);
            }
            if (mn < -1e-10 * std::max(1.0, initial_trace))
                throw std::runtime_error("pivoted Cholesky: negative residual diagonal, operator not PSD");
            for (double& x : diag) x = std::max(x, 0.0);
            diag[static_cast<size_t>(p)] = 0.0;
            if (pivots) pivots[r] = p;
            ++r;
        }
        double tr = 0.0;
        for (double x : diag) tr += x;
        std::memcpy(Z_out, Z.data(), sizeof(double) * static_cast<size_t>(r) * n);
        *achieved_rank = r;
        *trace_residual = std::max(tr, 0.0);
        return 0;
    } catch (const std::invalid_argument& e) {
        t_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        t_err = e.what();
        return 5;
    }
}

struct DenseEntries {
    const double* M;
    int64_t n;
    double operator()(int64_t i, int64_t j) const { return M[i * n + j]; }
};

}  // namespace

extern "C" {

const char* oracle_lowrank_last_error(void) { return t_err.c_str(); }

int oracle_pivoted_cholesky(const double* pts_rm, int64_t n, int d, const int* feats, const int* sizes, int P,
                            const double* weights, const double* ells, int window, int rank, double err_tol,
                            double* Z_out, int* achieved_rank, double* trace_residual, int64_t* pivots) {
    Entries E{pts_rm, n, d, {}, std::vector<double>(weights, weights + P), std::vector<double>(ells, ells + P),
              window};
    int off = 0;
    for (int l = 0; l < P; ++l) {
        E.wins.emplace_back(feats + off, feats + off + sizes[l]);
        off += sizes[l];
    }
    return pivoted_core(E, n, rank, err_tol, Z_out, achieved_rank, trace_residual, pivots);
}

// Same on a dense row-major n x n matrix (the reference tests' DenseOperator).
int oracle_pivoted_cholesky_dense(const double* M, int64_t n, int rank, double err_tol, double* Z_out,
                                  int* achieved_rank, double* trace_residual, int64_t* pivots) {
    return pivoted_core(DenseEntries{M, n}, n, rank, err_tol, Z_out, achieved_rank, trace_residual, pivots);
}

}  // extern "C"
