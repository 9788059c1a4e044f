/* ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * C ABI of the CPU checkers. Two libraries export it with different
 * prefixes and identical argument meaning:
 *   oracle/liboracle.so   prefix "oracle_"  - the Eigen-free restatement of
 *                                             the reference hot path
 *                                             (oracle/fastsum_oracle.cpp)
 *   oracle/_ref/libref.so prefix "ref_"     - the reference's OWN fastsum.cpp /
 *                                             kernel.cpp / windowing.cpp,
 *                                             compiled unmodified by path
 *                                             against oracle/shim
 *                                             (oracle/ref_capi.cpp)
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load these; the product path never does.
 *
 * Point matrices: `pts` is n x d COLUMN-major (Eigen's default storage, as
 * plan_fastsum receives it, P:include/ksvm/fastsum.hpp:60-62) unless a
 * function says row-major. Status: 0 ok, 2 DomainError/DataError,
 * 4 invalid_argument, 5 other (P:capi/ksvm_capi.cpp:31-48).
 */
#ifndef KSVM_ORACLE_H
#define KSVM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KSVM_ORACLE_DECLARE(P)                                                           \
    typedef struct P##plan P##plan;                                                      \
    typedef struct P##anova P##anova;                                                    \
    const char* P##last_error(void);                                                     \
    int P##plan_create(const double* pts, int64_t n, int d, double ell, int N, int m,    \
                       int sigma, double torus_radius, double fit, P##plan** out);       \
    int P##plan_apply(const P##plan* p, const double* v, double* out);                   \
    int P##plan_apply_cross(const P##plan* p, const double* targets, int64_t t,          \
                            const double* v, double* out);                               \
    double P##plan_scaled_length(const P##plan* p);                                      \
    double P##plan_coefficient_sum(const P##plan* p);                                    \
    int P##plan_scale_points(const P##plan* p, const double* pts, int64_t t, double* out); \
    void P##plan_free(P##plan* p);                                                       \
    int P##anova_create(const double* pts_rowmajor, int64_t n, int d,                   \
                        const int* win_features, const int* win_sizes, int P_,           \
                        const double* weights, const double* ells, int N, int m,         \
                        int sigma, double torus_radius, double fit, P##anova** out);     \
    int P##anova_apply(const P##anova* op, const double* v, double* out);               \
    double P##anova_entry(const P##anova* op, int64_t i, int64_t j);                     \
    void P##anova_free(P##anova* op);                                                    \
    int P##balance_and_split(const double* labels, int64_t n, double train_fraction,     \
                             uint64_t seed, int64_t* train_idx, int64_t* n_train,        \
                             int64_t* test_idx, int64_t* n_test);                        \
    int P##zscore(double* train_cm, int64_t n_train, double* test_cm, int64_t n_test,    \
                  int d, double* means, double* stddevs);

KSVM_ORACLE_DECLARE(oracle_)
KSVM_ORACLE_DECLARE(ref_)

/* balance_and_split (P:src/dataset.cpp:212-262) as row indices (train
 * sorted, test in shuffled order; arrays of room n) and
 * zscore_fit_transform (:264-282) in place on column-major n x d matrices
 * (test may be NULL when n_test == 0); means / stddevs receive the d
 * FeatureStats. */

/* Nystrom factor (oracle/nystrom_oracle.cpp, restating P:src/low_rank.cpp:115-168):
 * mode 0 kColumns, 1 kGaussian; Z_out rank x n row-major. _dense: the row-major
 * n x n DenseOperator; _window: the window `feats` (nf of them) of row-major
 * n x d points, exact WindowOperator (mode 0) or the FastWindowOperator plan
 * `plan` (mode 1, built with fit 1.0 over those columns). */
const char* oracle_nystrom_last_error(void);
int oracle_nystrom_dense(const double* M, int64_t n, int rank, int mode, uint64_t seed, double thr, double* Z_out);
int oracle_nystrom_window(const double* pts_rm, int64_t n, int d, const int* feats, int nf, double ell,
                          const oracle_plan* plan, int rank, int mode, uint64_t seed, double thr, double* Z_out);

/* Input generators matching P:tests/helpers.hpp:15-31 (libstdc++
 * std::mt19937_64 + std::normal_distribution, row-by-row fill). Output of
 * random_points is n x d COLUMN-major like the Eigen matrix it mirrors. */
void oracle_random_points(int64_t n, int64_t d, uint64_t seed, double scale, double* out);
void oracle_random_vector(int64_t n, uint64_t seed, double* out);
void oracle_uniform(int64_t n, uint64_t seed, double lo, double hi, double* out);
void oracle_bernoulli(int64_t n, uint64_t seed, double p, double* out);

/* Saddle system (oracle/saddle_oracle.cpp, restating P:src/saddle.cpp). K is
 * the ANOVA operator `op`, or, when `dense` is not NULL, the row-major n x n
 * matrix (P:tests/helpers.hpp DenseOperator). Z: k x n row-major factor
 * (StackedFactor::Z) or NULL for the identity preconditioner. gmres stats:
 * {iterations, relative_residual, converged, breakdown}. */
const char* oracle_saddle_last_error(void);
int oracle_saddle_apply(const oracle_anova* op, const double* dense, int64_t n, const double* y,
                        const double* theta, const double* vw, double* out);
int oracle_precond_apply(const double* Z, int k, int64_t n, const double* y, const double* theta,
                         const double* g, double* out, int* fallback);
int oracle_gmres_solve(const oracle_anova* op, const double* dense, int64_t n, const double* y,
                       const double* theta, const double* Z, int k, const double* rhs, double tol,
                       int max_iter, double* x_out, double* stats, double* history);

/* Interior point loop (P:src/ipm.cpp), compute_bias and helpers::blobs; see
 * oracle/saddle_oracle.cpp for the array layouts. */
int oracle_ipm_train(const oracle_anova* op, const double* dense, int64_t n, const double* y, const double* Z, int k,
                     const double* cfg, double* alpha_out, double* res, double* log);
int oracle_compute_bias(const oracle_anova* op, const double* dense, int64_t n, const double* alpha, const double* y,
                        double C, double eps_sv, double* bias);
void oracle_blobs(int64_t n, int64_t d, double gap, uint64_t seed, double noise, double* pts_cm, double* labels);

/* Greedy pivoted Cholesky (oracle/lowrank_oracle.cpp, restating
 * P:src/low_rank.cpp:25-92) on exact entries: window >= 0 the
 * WindowOperator entry of that window, -1 the weighted ANOVA entry. Z_out
 * holds rank x n (row-major); pivots (may be NULL) the chosen indices. */
const char* oracle_lowrank_last_error(void);
int oracle_pivoted_cholesky(const double* pts_rowmajor, int64_t n, int d, const int* win_features,
                            const int* win_sizes, int P, const double* weights, const double* ells,
                            int window, int rank, double err_tol, double* Z_out, int* achieved_rank,
                            double* trace_residual, int64_t* pivots);
int oracle_pivoted_cholesky_dense(const double* M, int64_t n, int rank, double err_tol, double* Z_out,
                                  int* achieved_rank, double* trace_residual, int64_t* pivots);
void oracle_fft(const double* in, double* out, int rank, const int* dims, int sign);

#ifdef __cplusplus
}
#endif

#endif
