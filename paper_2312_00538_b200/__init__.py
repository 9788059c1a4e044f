"""B200-native NFFT-accelerated ANOVA Gaussian-kernel matvec.

The hot path of arXiv 2312.00538's kernel-SVM interior point method
(reference: /root/reference/proj/src/fastsum.cpp), rebuilt as hand-written
sm_100a CUDA behind a C ABI (include/ksvm_nfft.h, libksvm_nfft.so) with this
package as the Python mirror of the reference's operator seam.
"""
from .fastsum import (AnovaFastOperator, AnovaKernelSpec, Dataset, DomainError, FastsumConfig,
                      FastsumPlan, FeatureWindowing, GaussianKernelSpec, KernelOperator,
                      anova_fast_operator, apply_fastsum, apply_fastsum_cross, decision_values,
                      plan_fastsum)
from .lowrank import LowRankFactor, fast_window_operator, nystrom, pivoted_cholesky_greedy, stack_anova_factors
from .saddle import GmresStats, SaddleOperator, SaddlePreconditioner, gmres_solve
from .ipm import (FeatureStats, IpmConfig, IpmResult, IpmStatus, TrainedModel, apply_normalization, compute_bias,
                  dual_objective, ipm_train, make_model)
from .pipeline import (PipelineConfig, TrainReport, balance_and_split, build_precond_factor, parse_window_spec,
                       train_on_prepared, train_pipeline, zscore_fit_transform)

__all__ = [
    "AnovaFastOperator", "AnovaKernelSpec", "Dataset", "DomainError", "FastsumConfig",
    "FastsumPlan", "FeatureWindowing", "GaussianKernelSpec", "KernelOperator",
    "anova_fast_operator", "apply_fastsum", "apply_fastsum_cross", "decision_values", "plan_fastsum",
    "GmresStats", "SaddleOperator", "SaddlePreconditioner", "gmres_solve",
    "LowRankFactor", "fast_window_operator", "nystrom", "pivoted_cholesky_greedy", "stack_anova_factors",
    "FeatureStats", "IpmConfig", "IpmResult", "IpmStatus", "TrainedModel", "apply_normalization", "compute_bias",
    "dual_objective", "ipm_train", "make_model",
    "PipelineConfig", "TrainReport", "balance_and_split", "build_precond_factor", "parse_window_spec",
    "train_on_prepared", "train_pipeline", "zscore_fit_transform",
]
