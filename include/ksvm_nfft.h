/* ksvm_nfft.h — C ABI of the B200 ANOVA-NFFT fast-summation path.
 *
 * Drop-in for the reference's hot path, P:src/fastsum.cpp (P: =
 * /root/reference/proj). It sits beside the reference C API
 * (P:capi/ksvm.h) and uses the same conventions: integer status codes with
 * the same numeric values, and a thread-local message for the last failure.
 *
 * Exported entry point             replaces (reference interface, file:line)
 * -------------------------------  ---------------------------------------------------------
 * ksvm_nfft_config_default         FastsumConfig defaults   P:include/ksvm/fastsum.hpp:13-17
 * ksvm_nfft_config_validate        FastsumConfig::validate  P:src/fastsum.cpp:38-47
 * ksvm_nfft_plan_create            plan_fastsum             P:include/ksvm/fastsum.hpp:60-62, P:src/fastsum.cpp:103-209
 * ksvm_nfft_plan_apply             apply_fastsum            P:include/ksvm/fastsum.hpp:65, P:src/fastsum.cpp:300-305
 * ksvm_nfft_plan_apply_cross       apply_fastsum_cross      P:include/ksvm/fastsum.hpp:70-72, P:src/fastsum.cpp:307-322
 * ksvm_nfft_plan_num_sources/dim/  FastsumPlan accessors    P:include/ksvm/fastsum.hpp:31-40, P:src/fastsum.cpp:94-101
 *   scaled_length/coefficient_sum/
 *   scale_points
 * ksvm_nfft_plan_free              ~FastsumPlan             P:src/fastsum.cpp:80-90
 * ksvm_nfft_op_create              anova_fast_operator      P:include/ksvm/fastsum.hpp:81-84, P:src/fastsum.cpp:326-341,366-371
 * ksvm_nfft_op_size                KernelOperator::size     P:include/ksvm/kernel.hpp:35
 * ksvm_nfft_op_window_points       (diagnostic: work actually executed per window)
 * ksvm_nfft_op_apply               KernelOperator::apply    P:include/ksvm/kernel.hpp:36, P:src/fastsum.cpp:345-352
 * ksvm_nfft_op_apply_batch         k applies (Nystrom sketch Y = K G, P:src/low_rank.cpp:139-150)
 * ksvm_nfft_op_entry               KernelOperator::entry    P:include/ksvm/kernel.hpp:37, P:src/fastsum.cpp:354-356
 * ksvm_nfft_kernel_rows            WindowOperator::entry rows / anova rows for pivoted Cholesky
 *                                                           P:src/pipeline.cpp:103-105, P:src/low_rank.cpp:49-51
 * ksvm_nfft_kernel_diag            diagonal loop            P:src/low_rank.cpp:33-35
 * ksvm_nfft_op_free                ~AnovaFastOperator
 * ksvm_nfft_op_create_sharded/     (multi-GPU point sharding: two-phase apply with a grid exchange;
 *   apply_spread/grids/finish       SURVEY.md 8(e) hybrid, no reference counterpart)
 * ksvm_nfft_saddle_create/         SaddleOperator           P:include/ksvm/saddle.hpp:14-31, P:src/saddle.cpp:7-33
 *   set_theta/apply/free
 * ksvm_nfft_precond_create(_ex)/   SaddlePreconditioner     P:include/ksvm/saddle.hpp:33-58, P:src/saddle.cpp:35-90
 *   refresh/apply/identity/          (_ex: the stacked factor Z already in device memory)
 *   diagonal_fallback/free
 * ksvm_nfft_gmres_solve            gmres_solve              P:include/ksvm/saddle.hpp:60-77, P:src/saddle.cpp:92-178
 * ksvm_nfft_pivoted_cholesky       pivoted_cholesky_greedy  P:include/ksvm/low_rank.hpp, P:src/low_rank.cpp:25-92
 * ksvm_nfft_decision_values        TrainedModel::decision_values  P:include/ksvm/ipm.hpp:51-69, P:src/ipm.cpp:213-288
 * ksvm_nfft_saddle_set_theta_ex/   SaddleOperator(op, y, theta) per IPM step / refresh(theta) on device Theta
 *   precond_refresh_ex                                      P:src/ipm.cpp:105-107, P:src/saddle.cpp:41-63
 * ksvm_nfft_ipm_config_default/    IpmConfig / ipm_train    P:include/ksvm/ipm.hpp:15-49, P:src/ipm.cpp:76-155
 *   ipm_train
 * ksvm_nfft_compute_bias           compute_bias             P:src/ipm.cpp:157-185
 * ksvm_nfft_nystrom                nystrom                  P:include/ksvm/low_rank.hpp:42-47, P:src/low_rank.cpp:115-168
 * ksvm_nfft_balance_and_split      balance_and_split        P:include/ksvm/dataset.hpp, P:src/dataset.cpp:212-262
 *
 * Status values equal ksvm_status (P:capi/ksvm.h:17-23): 0 ok, 2 data/domain
 * error (DomainError, P:src/fastsum.cpp:316-320), 4 invalid argument
 * (std::invalid_argument), 5 internal (CUDA failure, out of memory).
 *
 * Point matrices are n x d doubles addressed as
 *   layout == KSVM_NFFT_ROW_MAJOR: x(i, j) = points[i * ld + j]  (ld >= d)
 *   layout == KSVM_NFFT_COL_MAJOR: x(i, j) = points[j * ld + i]  (ld >= n)
 * Eigen's MatrixXd (what plan_fastsum receives) is COL_MAJOR with ld = n;
 * ksvm_dataset_from_arrays' input (P:capi/ksvm.h:46-47) is ROW_MAJOR, ld = d.
 *
 * Vectors v / y are length-n doubles. ptr_kind says where they live:
 * KSVM_NFFT_HOST (the call copies, runs and synchronises) or
 * KSVM_NFFT_DEVICE (pointers are on the plan's device; work is ordered after
 * `stream` (a cudaStream_t, NULL = legacy default) and the call returns once
 * it is enqueued). Plans and operators are immutable after creation; applies
 * from several threads are safe (they serialise on the object's internal
 * stream) and bit-reproducible run to run (no atomics anywhere on the path).
 */
#ifndef KSVM_NFFT_H
#define KSVM_NFFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    KSVM_NFFT_OK = 0,
    KSVM_NFFT_ERR_DATA = 2,
    KSVM_NFFT_ERR_CONFIG = 4,
    KSVM_NFFT_ERR_INTERNAL = 5
};

enum { KSVM_NFFT_ROW_MAJOR = 0, KSVM_NFFT_COL_MAJOR = 1 };
enum { KSVM_NFFT_HOST = 0, KSVM_NFFT_DEVICE = 1 };
/* precision of ksvm_nfft_op_create / _create_sharded. FP32 (north_star's
 * optional fp32 mode, <= 1e-5 relative l2 against the fp64 reference): the
 * dense d = 3, m = 4 windows spread and gather with fp32 window weights on the
 * tensor cores (3xTF32 split products, fp32 accumulation; 16 B of factors per
 * point; KSVM_NFFT_F32K=ffma in the environment selects the CUDA-core
 * kernels); d <= 2 windows, sparse d = 3 classes, the grid stage and the
 * window sum stay fp64; v and y are fp64 either way. */
enum { KSVM_NFFT_FP64 = 0, KSVM_NFFT_FP32 = 1 };

/* FastsumConfig (P:include/ksvm/fastsum.hpp:13-20). */
typedef struct {
    int bandwidth;       /* N, even, >= 2           (default 32)   */
    int window_cutoff;   /* m, in [2, 8]            (default 4)    */
    int oversampling;    /* sigma, grid edge M = sigma * N (default 2) */
    double torus_radius; /* r_T in (0, 1/4]         (default 0.25) */
} ksvm_nfft_config;

typedef struct ksvm_nfft_plan ksvm_nfft_plan;
typedef struct ksvm_nfft_op ksvm_nfft_op;

const char* ksvm_nfft_last_error(void);
/* Library build string and the number of CUDA kernel launches this process
 * has issued through the library (instrumentation for the benchmark). */
const char* ksvm_nfft_version(void);
int64_t ksvm_nfft_launch_count(void);

void ksvm_nfft_config_default(ksvm_nfft_config* cfg);
int ksvm_nfft_config_validate(const ksvm_nfft_config* cfg);

/* ---- single-window plan (FastsumPlan) -------------------------------- */
int ksvm_nfft_plan_create(const double* points, int64_t n, int d, int64_t ld, int layout,
                          double length_scale, const ksvm_nfft_config* cfg,
                          double fit_fraction, int device, ksvm_nfft_plan** out);
int ksvm_nfft_plan_apply(const ksvm_nfft_plan* plan, const double* v, double* out,
                         int ptr_kind, void* stream);
/* targets: t x d raw window coordinates (host), mapped with the plan's
 * affine map; DomainError (status 2) if any lands outside r_T (1 + 1e-12). */
int ksvm_nfft_plan_apply_cross(const ksvm_nfft_plan* plan, const double* targets, int64_t t,
                               int64_t ld, int layout, const double* v, double* out,
                               int ptr_kind, void* stream);
int64_t ksvm_nfft_plan_num_sources(const ksvm_nfft_plan* plan);
int ksvm_nfft_plan_dim(const ksvm_nfft_plan* plan);
double ksvm_nfft_plan_scaled_length(const ksvm_nfft_plan* plan);
double ksvm_nfft_plan_coefficient_sum(const ksvm_nfft_plan* plan);
/* out: t x d, same layout/ld convention as the input. */
int ksvm_nfft_plan_scale_points(const ksvm_nfft_plan* plan, const double* pts, int64_t t,
                                int64_t ld, int layout, double* out);
void ksvm_nfft_plan_free(ksvm_nfft_plan* plan);

/* ---- ANOVA operator (anova_fast_operator) ------------------------------
 * window_features: concatenation of the P windows' 0-based feature indices;
 * window_sizes[l] in 1..3; weights = eta_l > 0; length_scales = ell_l > 0.
 * window_mask (NULL = all windows) selects the windows this process owns
 * when windows are sharded over GPUs: apply then returns the partial sum
 * over the owned windows, and the caller sums partials across ranks
 * (SURVEY.md 8(e)). Entries (op_entry / kernel_rows / kernel_diag) always use
 * every window. */
int ksvm_nfft_op_create(const double* points, int64_t n, int64_t d, int64_t ld, int layout,
                        const int* window_features, const int* window_sizes,
                        int num_windows, const double* weights,
                        const double* length_scales, const ksvm_nfft_config* cfg,
                        double fit_fraction, const int* window_mask, int device,
                        int precision, ksvm_nfft_op** out);
int64_t ksvm_nfft_op_size(const ksvm_nfft_op* op);
int ksvm_nfft_op_num_windows(const ksvm_nfft_op* op);
/* Points window `window` is evaluated on: n, or the number of distinct scaled
 * points when exact duplicates were merged (binary / low-cardinality
 * features; the merge is exact); 0 for windows outside
 * window_mask or an invalid index. */
int64_t ksvm_nfft_op_window_points(const ksvm_nfft_op* op, int window);
int ksvm_nfft_op_apply(const ksvm_nfft_op* op, const double* v, double* y, int ptr_kind,
                       void* stream);
/* k right-hand sides; column c of V / Y starts at V + c * ld (ld >= n). */
int ksvm_nfft_op_apply_batch(const ksvm_nfft_op* op, const double* V, double* Y, int k,
                             int64_t ld, int ptr_kind, void* stream);
double ksvm_nfft_op_entry(const ksvm_nfft_op* op, int64_t i, int64_t j);
/* Exact kernel rows: out[r * n + j] = K(rows[r], j) with
 *   window >= 0 : exp(-||x_i^W - x_j^W||^2 / ell_W^2) on the op's raw window
 *                 coordinates (P:src/pipeline.cpp:103-105)
 *   window == -1: the ANOVA entry sum_l eta_l exp(...) (P:src/kernel.cpp:15-29)
 * rows is a host array; out follows ptr_kind. */
int ksvm_nfft_kernel_rows(const ksvm_nfft_op* op, int window, const int64_t* rows, int r,
                          double* out, int ptr_kind, void* stream);
int ksvm_nfft_kernel_diag(const ksvm_nfft_op* op, int window, double* out, int ptr_kind,
                          void* stream);
/* Per-launch device timing (CUDA events on the op's stream, off by default;
 * env KSVM_NFFT_STAGE_TIMING=1 also enables it). last_stage_ms fills the
 * device ms of each kernel launch of the last apply (synchronising on it)
 * and returns how many; stage_name(i) names launch i ("spread_d3",
 * "reduce", "conv_0", "gather_d3", "combine", ...). on = 1 times every
 * launch and runs the dimension classes one after another; on = 2 times the
 * main branch (the first class, d = 3 when present, and the window sum) and
 * keeps the other classes concurrent as in an untimed apply. */
int ksvm_nfft_op_set_stage_timing(ksvm_nfft_op* op, int on);
int ksvm_nfft_op_last_stage_ms(const ksvm_nfft_op* op, float* ms, int cap);
const char* ksvm_nfft_op_stage_name(const ksvm_nfft_op* op, int i);
int ksvm_nfft_op_device(const ksvm_nfft_op* op);

/* ---- point-sharded operator (hybrid sharding) -------------
 * Multi-GPU decomposition by points instead of windows: every rank creates
 * the operator from ALL n points (so the affine maps and grids are
 * identical on every rank) plus the ascending indices of the points it owns.
 * One matvec is then
 *   ksvm_nfft_op_apply_spread(op, v)     spread of the owned points' v into
 *                                        each window's grid G (v: length n;
 *                                        entries of other ranks' points ignored)
 *   sum the G buffers over the ranks     (ksvm_nfft_op_grids: device pointers
 *                                        and lengths, in window order; e.g. one
 *                                        NCCL all-reduce per window, in place)
 *   ksvm_nfft_op_apply_finish(op, y)     convolution, gather at the owned
 *                                        points, window sum; y (length n) holds
 *                                        the owned points' entries and 0 elsewhere
 * and a sum (all-reduce) of y over the ranks gives the full product. Spreading
 * is linear in the points, so the summed grids equal the unsharded operator's
 * and the result equals it to rounding. Exact duplicate merging is off for
 * sharded operators; a plain ksvm_nfft_op_apply on one returns the
 * owned-points block product. ksvm_nfft_op_grids returns the number of grids
 * (filling at most max_grids entries), or minus the status on error.
 * Replaces nothing in the reference (its apply is single-process); the
 * window-sharded alternative is window_mask in ksvm_nfft_op_create. */
int ksvm_nfft_op_create_sharded(const double* points, int64_t n, int64_t d, int64_t ld, int layout,
                                const int* window_features, const int* window_sizes, int num_windows,
                                const double* weights, const double* length_scales,
                                const ksvm_nfft_config* cfg, double fit_fraction,
                                const int64_t* own_points, int64_t n_own, int device, int precision,
                                ksvm_nfft_op** out);
int ksvm_nfft_op_apply_spread(ksvm_nfft_op* op, const double* v, int ptr_kind, void* stream);
int ksvm_nfft_op_grids(const ksvm_nfft_op* op, double** grids, int64_t* lengths, int max_grids);
int ksvm_nfft_op_apply_finish(ksvm_nfft_op* op, double* y, int ptr_kind, void* stream);
/* The owned windows' grids G of a point-sharded operator as ONE contiguous
 * device buffer (the concatenation ksvm_nfft_op_grids lists, window order):
 * the ranks sum it with a single all-reduce per matvec. */
int ksvm_nfft_op_grid_pool(const ksvm_nfft_op* op, double** pool, int64_t* length);

/* ---- window-sharded matvec, pipelined with the cross-rank sum -------------
 * with windows sharded over GPUs (window_mask), the length-n
 * partial sums are all-reduced once per matvec. Splitting the apply lets the
 * caller overlap that all-reduce with the window sum:
 *   ksvm_nfft_op_apply_windows(op, v)          spread / grid / gather of every
 *                                              owned window (per-window outputs)
 *   for each row range [lo, hi):
 *     ksvm_nfft_op_combine_range(op, y, lo, hi)  y[lo:hi) = sum_l eta_l out_l
 *     all-reduce y[lo:hi) (async, e.g. NCCL)   overlaps the next range's sum
 * Both take device pointers (ptr_kind KSVM_NFFT_DEVICE) and are ordered on
 * `stream` like ksvm_nfft_op_apply; y[lo:hi) equals ksvm_nfft_op_apply's rows
 * bit for bit. combine_range reads the per-window outputs of the operator's
 * most recent apply_windows (or apply): a caller that shares the operator
 * between threads must not interleave other applies with one pipelined
 * matvec. Replaces nothing in the reference (single process). */
int ksvm_nfft_op_apply_windows(ksvm_nfft_op* op, const double* v, int ptr_kind, void* stream);
int ksvm_nfft_op_combine_range(ksvm_nfft_op* op, double* y, int64_t lo, int64_t hi, int ptr_kind,
                               void* stream);

/* ---- Newton saddle system, GPU resident ----------------
 * The IPM's inner solve, A [v; w] = [Y K Y v + Theta v - w y; -y^T v] with K
 * the ANOVA operator, right-preconditioned by the block-triangular SMW
 * preconditioner of A-hat = Theta + Y Z^T Z Y (Z: k x n row-major, the
 * stacked low-rank factor; NULL or k == 0 gives the identity, like a null
 * StackedFactor). Every vector stays on the operator's GPU; GMRES keeps its
 * Krylov basis in HBM and only the (k+2)-entry Hessenberg column crosses to
 * the host per iteration. Vectors of the saddle system have n + 1 entries.
 * y, theta, Z are host arrays copied at create/refresh time. Theta must be
 * positive (std::invalid_argument, status 4); precond_apply before refresh
 * is std::logic_error (status 5). The rank is limited to k <= 1024. */
typedef struct ksvm_nfft_saddle ksvm_nfft_saddle;
typedef struct ksvm_nfft_precond ksvm_nfft_precond;
typedef struct ksvm_nfft_gmres_stats {
    int iterations;            /* GmresStats::iterations */
    double relative_residual;  /* true relative residual of the returned x */
    int converged;
    int breakdown;
} ksvm_nfft_gmres_stats;

int ksvm_nfft_saddle_create(const ksvm_nfft_op* op, const double* y, const double* theta,
                            ksvm_nfft_saddle** out);
int ksvm_nfft_saddle_set_theta(ksvm_nfft_saddle* s, const double* theta);
int ksvm_nfft_saddle_apply(const ksvm_nfft_saddle* s, const double* vw, double* out, int ptr_kind,
                           void* stream);
void ksvm_nfft_saddle_free(ksvm_nfft_saddle* s);

int ksvm_nfft_precond_create(const double* Z, int k, int64_t n, const double* y, int device,
                             ksvm_nfft_precond** out);
/* Same with Z on the device (z_ptr_kind DEVICE: copied after `stream`). */
int ksvm_nfft_precond_create_ex(const double* Z, int k, int64_t n, const double* y, int device,
                                int z_ptr_kind, void* stream, ksvm_nfft_precond** out);
int ksvm_nfft_precond_refresh(ksvm_nfft_precond* p, const double* theta);
int ksvm_nfft_precond_apply(const ksvm_nfft_precond* p, const double* g, double* out, int ptr_kind,
                            void* stream);
int ksvm_nfft_precond_identity(const ksvm_nfft_precond* p);
int ksvm_nfft_precond_diagonal_fallback(const ksvm_nfft_precond* p);
void ksvm_nfft_precond_free(ksvm_nfft_precond* p);

/* ---- greedy pivoted Cholesky, GPU resident -----------
 * pivoted_cholesky_greedy(op, rank, err_tol) of the exact kernel: window
 * >= 0 factorizes that window's WindowOperator (exp(-||dx||^2/ell^2) on its
 * raw coordinates, P:src/pipeline.cpp:103-105); window == -1 the weighted
 * ANOVA kernel (P:src/kernel.cpp:33-48). Z receives achieved_rank x n rows
 * (row-major; room for min(rank, n) rows), pivots (may be NULL) the chosen
 * indices. rank < 1: status 4; a non-PSD operator: status 5 with the
 * reference's message. */
int ksvm_nfft_pivoted_cholesky(const ksvm_nfft_op* op, int window, int rank, double err_tol, double* Z,
                               int* achieved_rank, double* trace_residual, int64_t* pivots, int ptr_kind,
                               void* stream);

/* ---- Nystrom factor, GPU (P:src/low_rank.cpp:115-168) ----------------------
 * nystrom(op, rank, mode, seed, ldl_threshold) -> Z (rank x n row-major,
 * host or device per ptr_kind). GAUSSIAN sketches op's own applies (window
 * must be -1): the reference builds it on the FastWindowOperator of one
 * window (P:src/pipeline.cpp:172-181), i.e. a one-window operator with
 * weight 1 and fit 1.0; Y = K G and KQ = K Q run as batched applies.
 * COLUMNS takes exact kernel columns of `window` (>= 0: WindowOperator,
 * -1: the ANOVA entries). The draws are the reference's
 * (std::mt19937_64(seed)); Z^T Z equals the reference's to rounding (the
 * orthonormal basis of range(Y) may differ by signs). rank outside
 * [1, n]: status 4. */
#define KSVM_NFFT_NYSTROM_COLUMNS 0
#define KSVM_NFFT_NYSTROM_GAUSSIAN 1
int ksvm_nfft_nystrom(const ksvm_nfft_op* op, int window, int rank, int mode, uint64_t seed,
                      double ldl_threshold, double* Z, int ptr_kind, void* stream);

/* ---- prediction, GPU -----------------------------------
 * TrainedModel::decision_values (P:src/ipm.cpp:213-288): f_j = sum_i coeff_i
 * K(x_i, t_j) + bias for the t test points, coeff = alpha .* y. Backend FAST
 * builds one plan per window over the training points (fit 1/1.2, :258),
 * evaluates the targets whose scaled norm is <= r_T by the cross transform
 * and recomputes the others exactly (:261-284); EXACT sums every target
 * directly (:236-239). Points are already normalized (the reference applies
 * the model's z-score first, :216-218); layout / ld as in plan_create, the
 * same layout for train and test. n_exact (may be NULL) returns how many
 * targets took the exact path. Host arrays. */
#define KSVM_NFFT_PREDICT_EXACT 0
#define KSVM_NFFT_PREDICT_FAST 1
int ksvm_nfft_decision_values(const double* train, int64_t n, int d, int64_t ld_train, int layout,
                              const int* window_features, const int* window_sizes, int P,
                              const double* weights, const double* length_scales,
                              const ksvm_nfft_config* cfg, const double* coeff, double bias,
                              const double* test, int64_t t, int64_t ld_test, int backend, int device,
                              double* f_out, int64_t* n_exact);

/* residual_history: NULL or room for max_iter estimates (host). */
int ksvm_nfft_gmres_solve(const ksvm_nfft_saddle* s, const ksvm_nfft_precond* p, const double* rhs,
                          double tol, int max_iter, double* x, ksvm_nfft_gmres_stats* stats,
                          double* residual_history, int ptr_kind, void* stream);

/* Theta from host (ptr_kind HOST; stream ignored) or device memory (ordered
 * on `stream`), for device-resident drivers such as ksvm_nfft_ipm_train.
 * Replaces constructing a fresh SaddleOperator(op, y, theta)
 * (P:src/ipm.cpp:107) / SaddlePreconditioner::refresh(theta) (P:src/saddle.cpp:41-63). */
int ksvm_nfft_saddle_set_theta_ex(ksvm_nfft_saddle* s, const double* theta, int ptr_kind, void* stream);
int ksvm_nfft_precond_refresh_ex(ksvm_nfft_precond* p, const double* theta, int ptr_kind, void* stream);

/* ---- interior point trainer, GPU resident ---------------------------------
 * ipm_train(op, y, factor, cfg) (P:src/ipm.cpp:76-155; IpmConfig /
 * IpmResult / IpmIterationLog, P:include/ksvm/ipm.hpp:15-53): alpha, Theta,
 * the Newton systems and the Krylov bases stay on op's GPU; every matvec is
 * op's NFFT apply. y: n labels (+-1, host); Z: the stacked low-rank factor
 * (k x n row-major, host or op's GPU per z_ptr_kind) or NULL for the
 * unpreconditioned run (null StackedFactor); alpha: n entries out (host); log: NULL or room for
 * cfg->max_ip_iters entries. Invalid config / labels: status 4 with the
 * reference's messages; degenerate initial infeasibility: status 5. */
typedef struct ksvm_nfft_ipm_config {
    double C;             /* 0.5 */
    double sigma;         /* 0.6, barrier reduction */
    double gamma0;        /* 0.99995, fraction to boundary */
    double tol_ip;        /* 1e-1 */
    int max_ip_iters;     /* 50 */
    double tol_gmres;     /* 1e-3 */
    int max_gmres_iters;  /* 100 */
    double mu0;           /* 1.0 */
} ksvm_nfft_ipm_config;

#define KSVM_NFFT_IPM_CONVERGED 0
#define KSVM_NFFT_IPM_MAX_ITERATIONS 1
#define KSVM_NFFT_IPM_STALLED 2

typedef struct ksvm_nfft_ipm_result {
    double lambda;
    double mu_final;
    double xi_alpha_rel;
    double xi_lambda_rel;
    int status;            /* KSVM_NFFT_IPM_* */
    int iterations;
    double mean_gmres_iters;
} ksvm_nfft_ipm_result;

typedef struct ksvm_nfft_ipm_log {
    int it;
    double mu;
    double xi_alpha_rel;
    double xi_lambda_rel;
    double step_alpha;
    int gmres_iterations;
    double gmres_relative_residual;
    int gmres_converged;
    int gmres_breakdown;
} ksvm_nfft_ipm_log;

void ksvm_nfft_ipm_config_default(ksvm_nfft_ipm_config* cfg);
int ksvm_nfft_ipm_train(const ksvm_nfft_op* op, const double* y, const double* Z, int k, int z_ptr_kind,
                        const ksvm_nfft_ipm_config* cfg, double* alpha, ksvm_nfft_ipm_result* result,
                        ksvm_nfft_ipm_log* log);

/* compute_bias (P:src/ipm.cpp:157-185): mean of y_j - (K(alpha.*y))_j over
 * free support vectors (eps_sv < alpha_j < C - eps_sv), else the median
 * over all support vectors, else 0. Host arrays of op_size entries;
 * n_support (may be NULL) returns #{alpha_j > eps_sv}. */
int ksvm_nfft_compute_bias(const ksvm_nfft_op* op, const double* alpha, const double* y, double C,
                           double eps_sv, double* bias, int64_t* n_support);

/* balance_and_split (P:src/dataset.cpp:212-262) as row indices: the
 * reference's std::mt19937_64(seed) + std::shuffle stream, the training part
 * balanced by down-sampling the majority class and sorted. train_idx and
 * test_idx need room for n entries. Bad fraction / one class / too few
 * points: status 2 (DataError) with the reference's messages. CPU only. */
int ksvm_nfft_balance_and_split(const double* labels, int64_t n, double train_fraction, uint64_t seed,
                                int64_t* train_idx, int64_t* n_train, int64_t* test_idx, int64_t* n_test);
void ksvm_nfft_op_free(ksvm_nfft_op* op);

#ifdef __cplusplus
}
#endif

#endif
