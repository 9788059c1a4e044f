"""Test helper: train_pipeline (P:src/pipeline.cpp:229-265) restated on the
oracle pieces (split, z-score, low-rank factor, IPM, bias, fast predict)."""
import numpy as np

import oracle

FIT = 1.0 / 1.2


def oracle_pipeline(w, windows, rank, C, seed=0, precond="cholesky-greedy"):
    """train_pipeline restated on the oracle pieces (P:src/pipeline.cpp:229-265)."""
    tr, te = oracle.balance_and_split(w.labels, 0.5, seed)
    Xtr, Xte, mu, sd = oracle.zscore(w.points[tr], w.points[te])
    ytr = w.labels[tr]
    P = len(windows)
    if precond == "cholesky-greedy":
        Zs = [oracle.pivoted_cholesky(Xtr, windows, window=l, rank=max(1, rank // P), err_tol=1e-5)[0]
              for l in range(P)]
    else:
        mode = oracle.NYSTROM_GAUSSIAN if precond == "nystrom-gaussian" else oracle.NYSTROM_COLUMNS
        Zs = [oracle.nystrom_window(Xtr, windows[l], 1.0, max(1, rank // P), mode, seed + l) for l in range(P)]
    Z = np.vstack([np.sqrt(1.0 / P) * z for z in Zs])
    Ko = oracle.Lib("oracle").anova(Xtr, windows, fit=FIT)
    alpha, res, log = oracle.ipm_train(Ko, ytr, Z, C=C)
    b = oracle.compute_bias(Ko, alpha, ytr, C, 1e-4 * C)
    f, _ = oracle.decision_values(Xtr, windows, [1.0 / P] * P, [1.0] * P, alpha * ytr, b, Xte, fast=True)
    return dict(tr=tr, te=te, alpha=alpha, res=res, log=log, bias=b, f=f, Ko=Ko, ytr=ytr, Z=Z)


