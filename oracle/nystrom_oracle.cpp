// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Eigen-free restatement of the reference's Nystrom factorization
// (P:src/low_rank.cpp:115-168, nystrom) with its three ingredients stated
// the way Eigen 3 computes them:
//   * the sketch: kColumns draws std::shuffle(iota(n)) with
//     std::mt19937_64(seed) and keeps the first k indices (:124-134);
//     kGaussian fills G(i, c) = N(0, 1) row by row (:137-139), Y = K G,
//     thin Q of a Householder QR of Y (unblocked dgeqr2 with Eigen's
//     makeHouseholder sign rule; Eigen's blocked path only starts above 48
//     columns, and Q is basis-equivalent either way), KQ = K Q, C = Q^T KQ;
//   * C = (C + C^T) / 2 and Eigen's LDLT<Lower>: left-looking, symmetric
//     pivoting on the largest remaining ORIGINAL diagonal magnitude, zero
//     pivots left unscaled (:155-156);
//   * D clamped to max(|d|, ldl_threshold), Z = D^{-1/2} L^{-1} P (KQ)^T
//     (:157-162).
// The operator is a dense row-major matrix (the reference tests'
// DenseOperator), the exact window kernel (WindowOperator, columns mode)
// or an oracle fastsum plan (FastWindowOperator, Gaussian mode).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "ksvm_oracle.h"

namespace {

thread_local std::string t_err = "ok";
using Apply = std::function<void(const double*, double*)>;  // out = K v, length n

// Householder QR of the n x k column-major Y, thin Q (n x k) out.
void householder_thin_q(std::vector<double>& Y, int64_t n, int k, std::vector<double>& Q) {
    std::vector<double> tau(static_cast<size_t>(k), 0.0);
    auto A = [&](int64_t i, int j) -> double& { return Y[static_cast<size_t>(j) * n + i]; };
    for (int j = 0; j < k && j < n; ++j) {
        double tail = 0.0;
        for (int64_t i = j + 1; i < n; ++i) tail += A(i, j) * A(i, j);
        const double c0 = A(j, j);
        double beta, t;
        if (tail <= std::numeric_limits<double>::min()) {
            t = 0.0;
            beta = c0;
            for (int64_t i = j + 1; i < n; ++i) A(i, j) = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            for (int64_t i = j + 1; i < n; ++i) A(i, j) /= (c0 - beta);
            t = (beta - c0) / beta;
        }
        A(j, j) = beta;
        tau[static_cast<size_t>(j)] = t;
        for (int c = j + 1; c < k; ++c) {  // H = I - t v v^T, v = [1; essential]
            double w = A(j, c);
            for (int64_t i = j + 1; i < n; ++i) w += A(i, j) * A(i, c);
            w *= t;
            A(j, c) -= w;
            for (int64_t i = j + 1; i < n; ++i) A(i, c) -= w * A(i, j);
        }
    }
    Q.assign(static_cast<size_t>(n) * k, 0.0);
    for (int c = 0; c < k && c < n; ++c) Q[static_cast<size_t>(c) * n + c] = 1.0;
    for (int j = std::min<int64_t>(k, n) - 1; j >= 0; --j) {  // Q = H_0 ... H_{k-1} [I; 0]
        const double t = tau[static_cast<size_t>(j)];
        if (t == 0.0) continue;
        for (int c = 0; c < k; ++c) {
            double* q = Q.data() + static_cast<size_t>(c) * n;
            double w = q[j];
            for (int64_t i = j + 1; i < n; ++i) w += A(i, j) * q[i];
            w *= t;
            q[j] -= w;
            for (int64_t i = j + 1; i < n; ++i) q[i] -= w * A(i, j);
        }
    }
}

// Eigen's ldlt_inplace<Lower>::unblocked on the k x k row-major C (lower
// part used): returns transpositions, unit-lower L (in C) and D.
void ldlt_eigen(std::vector<double>& C, int k, std::vector<int>& tr, std::vector<double>& D) {
    auto M = [&](int i, int j) -> double& { return C[static_cast<size_t>(i) * k + j]; };
    tr.assign(static_cast<size_t>(k), 0);
    std::vector<double> temp(static_cast<size_t>(k));
    for (int j = 0; j < k; ++j) {
        int big = j;
        double bv = std::fabs(M(j, j));
        for (int i = j + 1; i < k; ++i)
            if (std::fabs(M(i, i)) > bv) {
                bv = std::fabs(M(i, i));
                big = i;
            }
        tr[static_cast<size_t>(j)] = big;
        if (big != j) {  // symmetric swap on the lower triangle
            for (int c = 0; c < j; ++c) std::swap(M(j, c), M(big, c));
            for (int r = big + 1; r < k; ++r) std::swap(M(r, j), M(r, big));
            std::swap(M(j, j), M(big, big));
            for (int i = j + 1; i < big; ++i) std::swap(M(i, j), M(big, i));
        }
        const int rs = k - j - 1;
        if (j > 0) {
            for (int c = 0; c < j; ++c) temp[static_cast<size_t>(c)] = M(c, c) * M(j, c);
            double s = 0.0;
            for (int c = 0; c < j; ++c) s += M(j, c) * temp[static_cast<size_t>(c)];
            M(j, j) -= s;
            for (int r = j + 1; r < k; ++r) {
                double t = 0.0;
                for (int c = 0; c < j; ++c) t += M(r, c) * temp[static_cast<size_t>(c)];
                M(r, j) -= t;
            }
        }
        const double akk = M(j, j);
        if (rs > 0 && std::fabs(akk) > 0.0)
            for (int r = j + 1; r < k; ++r) M(r, j) /= akk;
    }
    D.resize(static_cast<size_t>(k));
    for (int j = 0; j < k; ++j) D[static_cast<size_t>(j)] = M(j, j);
}

int nystrom_core(int64_t n, int rank, int mode, uint64_t seed, double thr, const Apply& apply, double* Z_out) {
    try {
        if (rank < 1 || rank > n) throw std::invalid_argument("nystrom: rank must lie in [1, n]");
        const int k = rank;
        std::mt19937_64 rng(seed);
        std::vector<double> KQ(static_cast<size_t>(n) * k), C(static_cast<size_t>(k) * k);  // KQ col-major
        if (mode == 0) {  // kColumns
            std::vector<int64_t> pool(static_cast<size_t>(n));
            std::iota(pool.begin(), pool.end(), int64_t{0});
            std::shuffle(pool.begin(), pool.end(), rng);
            std::vector<double> e(static_cast<size_t>(n), 0.0);
            for (int c = 0; c < k; ++c) {
                const int64_t idx = pool[static_cast<size_t>(c)];
                e[static_cast<size_t>(idx)] = 1.0;
                apply(e.data(), KQ.data() + static_cast<size_t>(c) * n);
                e[static_cast<size_t>(idx)] = 0.0;
            }
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < k; ++r)
                    C[static_cast<size_t>(r) * k + c] = KQ[static_cast<size_t>(c) * n + pool[static_cast<size_t>(r)]];
        } else {  // kGaussian
            std::normal_distribution<double> normal(0.0, 1.0);
            std::vector<double> G(static_cast<size_t>(n) * k), Y(static_cast<size_t>(n) * k), Q;
            for (int64_t i = 0; i < n; ++i)
                for (int c = 0; c < k; ++c) G[static_cast<size_t>(c) * n + i] = normal(rng);
            for (int c = 0; c < k; ++c) apply(G.data() + static_cast<size_t>(c) * n, Y.data() + static_cast<size_t>(c) * n);
            householder_thin_q(Y, n, k, Q);
            for (int c = 0; c < k; ++c) apply(Q.data() + static_cast<size_t>(c) * n, KQ.data() + static_cast<size_t>(c) * n);
            for (int r = 0; r < k; ++r)
                for (int c = 0; c < k; ++c) {
                    double s = 0.0;
                    for (int64_t i = 0; i < n; ++i) s += Q[static_cast<size_t>(r) * n + i] * KQ[static_cast<size_t>(c) * n + i];
                    C[static_cast<size_t>(r) * k + c] = s;
                }
        }
        std::vector<double> S(C);
        for (int r = 0; r < k; ++r)
            for (int c = 0; c < k; ++c)
                S[static_cast<size_t>(r) * k + c] = 0.5 * (C[static_cast<size_t>(r) * k + c] + C[static_cast<size_t>(c) * k + r]);
        std::vector<int> tr;
        std::vector<double> D;
        ldlt_eigen(S, k, tr, D);
        for (double& d : D) d = std::max(std::fabs(d), thr);
        // rhs = P KQ^T (k x n, row-major), rows swapped in transposition order
        std::vector<double> R(static_cast<size_t>(k) * n);
        for (int c = 0; c < k; ++c) std::memcpy(R.data() + static_cast<size_t>(c) * n, KQ.data() + static_cast<size_t>(c) * n, sizeof(double) * n);
        for (int j = 0; j < k; ++j)
            if (tr[static_cast<size_t>(j)] != j)
                std::swap_ranges(R.begin() + static_cast<std::ptrdiff_t>(j) * n, R.begin() + static_cast<std::ptrdiff_t>(j + 1) * n,
                                 R.begin() + static_cast<std::ptrdiff_t>(tr[static_cast<size_t>(j)]) * n);
        for (int r = 0; r < k; ++r)  // L^{-1} (unit lower, forward substitution)
            for (int c = 0; c < r; ++c) {
                const double l = S[static_cast<size_t>(r) * k + c];
                if (l == 0.0) continue;
                double* dst = R.data() + static_cast<size_t>(r) * n;
                const double* src = R.data() + static_cast<size_t>(c) * n;
                for (int64_t i = 0; i < n; ++i) dst[i] -= l * src[i];
            }
        for (int r = 0; r < k; ++r) {
            const double s = 1.0 / std::sqrt(D[static_cast<size_t>(r)]);
            for (int64_t i = 0; i < n; ++i) Z_out[static_cast<size_t>(r) * n + i] = s * R[static_cast<size_t>(r) * n + i];
        }
        return 0;
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

const char* oracle_nystrom_last_error(void) { return t_err.c_str(); }

// DenseOperator (row-major n x n)
int oracle_nystrom_dense(const double* M, int64_t n, int rank, int mode, uint64_t seed, double thr, double* Z_out) {
    Apply ap = [&](const double* v, double* out) {
        for (int64_t i = 0; i < n; ++i) {
            double s = 0.0;
            for (int64_t j = 0; j < n; ++j) s += M[i * n + j] * v[j];
            out[i] = s;
        }
    };
    return nystrom_core(n, rank, mode, seed, thr, ap, Z_out);
}

// One window of row-major points: mode 0 on the exact WindowOperator
// (P:src/pipeline.cpp:89-111), mode 1 on the FastWindowOperator's plan
// (an oracle plan built with fit 1.0 over the window's columns, :114-133).
int oracle_nystrom_window(const double* pts_rm, int64_t n, int d, const int* feats, int nf, double ell,
                          const oracle_plan* plan, int rank, int mode, uint64_t seed, double thr, double* Z_out) {
    const double ell2 = ell * ell;
    Apply exact = [&](const double* v, double* out) {
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int64_t j = 0; j < n; ++j) {
                if (v[j] == 0.0) continue;  // adds exact zeros in the reference's dense sweep
                double d2 = 0.0;
                for (int t = 0; t < nf; ++t) {
                    const double diff = pts_rm[i * d + feats[t]] - pts_rm[j * d + feats[t]];
                    d2 += diff * diff;
                }
                acc += std::exp(-d2 / ell2) * v[j];
            }
            out[i] = acc;
        }
    };
    Apply fast = [&](const double* v, double* out) {
        if (oracle_plan_apply(plan, v, out) != 0) throw std::runtime_error(oracle_last_error());
    };
    if (mode == 1 && !plan) {
        t_err = "gaussian mode needs the window's plan";
        return 4;
    }
    return nystrom_core(n, rank, mode, seed, thr, mode == 1 ? fast : exact, Z_out);
}

}  // extern "C"
