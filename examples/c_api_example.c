/* Plain-C client of the B200 ANOVA-NFFT C ABI (include/ksvm_nfft.h).
 * Build: gcc -I include examples/c_api_example.c -L paper_2312_00538_b200 -lksvm_nfft -lm
 * Run (needs a B200): LD_LIBRARY_PATH=paper_2312_00538_b200 ./a.out */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "ksvm_nfft.h"

int main(void) {
    const int64_t n = 2000, d = 6;
    double* x = malloc(sizeof(double) * n * d);
    double* v = malloc(sizeof(double) * n);
    double* y = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n * d; ++i) x[i] = 0.25 * sin(0.37 * (double)i);
    for (int64_t i = 0; i < n; ++i) v[i] = cos(0.11 * (double)i);
    const int feats[6] = {0, 1, 2, 3, 4, 5};
    const int sizes[2] = {3, 3};
    const double eta[2] = {0.5, 0.5}, ell[2] = {1.0, 1.0};
    ksvm_nfft_config cfg;
    ksvm_nfft_config_default(&cfg);
    ksvm_nfft_op* op = NULL;
    int st = ksvm_nfft_op_create(x, n, d, d, KSVM_NFFT_ROW_MAJOR, feats, sizes, 2, eta, ell, &cfg,
                                 1.0 / 1.2, NULL, 0, KSVM_NFFT_FP64, &op);
    if (st != KSVM_NFFT_OK) {
        fprintf(stderr, "create failed (%d): %s\n", st, ksvm_nfft_last_error());
        return 1;
    }
    st = ksvm_nfft_op_apply(op, v, y, KSVM_NFFT_HOST, NULL);
    if (st != KSVM_NFFT_OK) {
        fprintf(stderr, "apply failed (%d): %s\n", st, ksvm_nfft_last_error());
        return 1;
    }
    printf("y[0] = %.17g, K(0,1) = %.17g\n", y[0], ksvm_nfft_op_entry(op, 0, 1));
    ksvm_nfft_op_free(op);
    free(x);
    free(v);
    free(y);
    return 0;
}
