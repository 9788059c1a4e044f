/* Plain-C client of the training entry points of the B200 C ABI
 * (include/ksvm_nfft.h): the reference's train_on_prepared
 * (P:src/pipeline.cpp:198-227) as a C program -- operator (fit 1/1.2),
 * per-window greedy pivoted-Cholesky factors stacked with sqrt(eta),
 * ksvm_nfft_ipm_train, ksvm_nfft_compute_bias, fast decision values.
 * Build: gcc -I include examples/c_train_example.c -L paper_2312_00538_b200 -lksvm_nfft -lm
 * Run (needs a B200): LD_LIBRARY_PATH=paper_2312_00538_b200 ./a.out */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ksvm_nfft.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        int st_ = (call);                                                            \
        if (st_ != KSVM_NFFT_OK) {                                                   \
            fprintf(stderr, "%s failed (%d): %s\n", #call, st_, ksvm_nfft_last_error()); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(void) {
    const int64_t n = 1000, d = 4;
    const int P = 2, rank_per_window = 20;
    double* x = malloc(sizeof(double) * n * d);
    double* y = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) {  /* two shifted clouds, labels +-1 */
        const double lab = (i % 2 == 0) ? 1.0 : -1.0;
        for (int64_t j = 0; j < d; ++j) x[i * d + j] = 0.8 * lab + sin(1.7 * (double)(i * d + j));
        y[i] = lab;
    }
    const int feats[4] = {0, 1, 2, 3};
    const int sizes[2] = {2, 2};
    const double eta[2] = {0.5, 0.5}, ell[2] = {1.0, 1.0};
    ksvm_nfft_config cfg;
    ksvm_nfft_config_default(&cfg);
    ksvm_nfft_op* op = NULL;
    CHECK(ksvm_nfft_op_create(x, n, d, d, KSVM_NFFT_ROW_MAJOR, feats, sizes, P, eta, ell, &cfg, 1.0 / 1.2, NULL, 0,
                              KSVM_NFFT_FP64, &op));
    /* stacked factor: window l's rows scaled by sqrt(eta_l) (P:src/low_rank.cpp:200-222) */
    double* Z = malloc(sizeof(double) * (size_t)(P * rank_per_window) * n);
    int k = 0;
    for (int l = 0; l < P; ++l) {
        int r = 0;
        double trace = 0.0;
        CHECK(ksvm_nfft_pivoted_cholesky(op, l, rank_per_window, 1e-5, Z + (size_t)k * n, &r, &trace, NULL,
                                         KSVM_NFFT_HOST, NULL));
        for (int64_t q = 0; q < (int64_t)r * n; ++q) Z[(size_t)k * n + q] *= sqrt(eta[l]);
        k += r;
    }
    ksvm_nfft_ipm_config icfg;
    ksvm_nfft_ipm_config_default(&icfg);
    icfg.C = 1.0;
    double* alpha = malloc(sizeof(double) * n);
    ksvm_nfft_ipm_result res;
    ksvm_nfft_ipm_log* log = malloc(sizeof(ksvm_nfft_ipm_log) * icfg.max_ip_iters);
    CHECK(ksvm_nfft_ipm_train(op, y, Z, k, KSVM_NFFT_HOST, &icfg, alpha, &res, log));
    double bias = 0.0;
    int64_t nsv = 0;
    CHECK(ksvm_nfft_compute_bias(op, alpha, y, icfg.C, 1e-4 * icfg.C, &bias, &nsv));
    double* coeff = malloc(sizeof(double) * n);
    double* f = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) coeff[i] = alpha[i] * y[i];
    int64_t nexact = 0;
    CHECK(ksvm_nfft_decision_values(x, n, (int)d, d, KSVM_NFFT_ROW_MAJOR, feats, sizes, P, eta, ell, &cfg, coeff,
                                    bias, x, n, d, KSVM_NFFT_PREDICT_FAST, 0, f, &nexact));
    int correct = 0;
    for (int64_t i = 0; i < n; ++i) correct += ((f[i] >= 0.0) ? 1.0 : -1.0) == y[i];
    printf("status %d, %d Newton steps (mean GMRES %.2f), rank %d, bias %.6f, %lld SVs, training accuracy %.3f\n",
           res.status, res.iterations, res.mean_gmres_iters, k, bias, (long long)nsv, (double)correct / (double)n);
    ksvm_nfft_op_free(op);
    free(x); free(y); free(Z); free(alpha); free(log); free(coeff); free(f);
    return 0;
}
