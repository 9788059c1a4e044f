// GPU-resident interior point trainer (north_star: "end-to-end IPM training
// reproducing the reference's dual objective and predicted labels"): the
// reference's ipm_train (P:src/ipm.cpp:76-155) with assemble_newton_rhs
// (:31-42), step_lengths (:44-55), barrier_diagonal (:59-64) and
// initial_alpha (:66-74), plus compute_bias (:157-185).
//
// Every length-n vector (alpha, y, Theta, the Newton right-hand side and
// step, K(y .* alpha)) lives on the operator's GPU; each IPM iteration is
//   theta/rhs kernel -> SaddleOperator / SaddlePreconditioner refresh on the
//   device Theta -> GPU GMRES (saddle.cu) -> step-length min reduction ->
//   alpha update fused with u = y .* alpha -> one ANOVA matvec -> residual
//   reductions,
// with three small host round trips (the capacitance LU inside the refresh,
// the step length, the two infeasibility norms). Scalars (mu, lambda, the
// infeasibilities, step lengths) stay on the host exactly as in the
// reference loop. Reductions use a fixed grid with fixed ownership and
// fixed-order finishers, so training is bit-reproducible run to run;
// against the reference the differences are rounding only (summation
// order), amplified by GMRES's 1e-3 stopping rule (tests compare the dual
// objective, labels and iteration counts).
//
// initial_alpha uses libstdc++'s std::mt19937_64 + uniform_real_distribution
// with the reference's seed, so alpha^0 is bit-identical to the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <vector>

#include "capi_common.cuh"
#include "launch.cuh"
#include "reduce.cuh"

namespace ksvm_nfft {
namespace {

// u = y .* alpha (matvec input), partial of y . alpha
__global__ void __launch_bounds__(kRT) ki_yalpha(double* __restrict__ u, const double* __restrict__ y,
                                                 const double* __restrict__ alpha, long long n,
                                                 double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        u[j] = y[j] * alpha[j];
        acc += y[j] * alpha[j];
    }
    block_partial(acc, partial);
}

// P:src/ipm.cpp:31-42 with yky_alpha = y .* kv; theta (P:src/ipm.cpp:59-64)
// when theta != nullptr; partial of ||rhs_head||^2.
__global__ void __launch_bounds__(kRT) ki_newton(double* __restrict__ rhs, double* __restrict__ theta,
                                                 const double* __restrict__ alpha, const double* __restrict__ y,
                                                 const double* __restrict__ kv, double lambda, double mu, double C,
                                                 long long n, double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        const double a = alpha[j], c = C - a;
        const double r = 1.0 - y[j] * kv[j] + lambda * y[j] + mu * (1.0 / a) - mu * (1.0 / c);
        if (rhs) rhs[j] = r;
        if (theta) theta[j] = mu * (1.0 / (a * a) + 1.0 / (c * c));
        acc += r * r;
    }
    block_partial(acc, partial);
}

// step_lengths ratio test (P:src/ipm.cpp:44-55): block minimum of the
// admissible steps, starting from 1.
__global__ void __launch_bounds__(kRT) ki_step_min(const double* __restrict__ alpha,
                                                   const double* __restrict__ dalpha, double C, long long n,
                                                   double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    double m = 1.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        const double d = dalpha[j];
        if (d < 0.0)
            m = fmin(m, -alpha[j] / d);
        else if (d > 0.0)
            m = fmin(m, (C - alpha[j]) / d);
    }
    block_min(m, partial);
}

// alpha += s dalpha; u = y .* alpha; partial of y . alpha
__global__ void __launch_bounds__(kRT) ki_update(double* __restrict__ alpha, double* __restrict__ u,
                                                 const double* __restrict__ dalpha, const double* __restrict__ y,
                                                 double s, long long n, double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        const double a = alpha[j] + s * dalpha[j];
        alpha[j] = a;
        u[j] = y[j] * a;
        acc += y[j] * a;
    }
    block_partial(acc, partial);
}

// dst[0] = sum(partial_a), dst[1] = sum(partial_b) (fixed order), or the minimum
__global__ void ki_finish2(const double* __restrict__ pa, const double* __restrict__ pb, int nb,
                           double* __restrict__ dst, int min_mode) {
    pdl_trigger();
    pdl_wait();
    if (min_mode) {
        const double m = warp_min_strided(pa, nb);
        if (threadIdx.x == 0) dst[0] = m;
        return;
    }
    const double a = warp_sum_strided(pa, nb, 1);
    const double b = pb ? warp_sum_strided(pb, nb, 1) : 0.0;
    if (threadIdx.x == 0) {
        dst[0] = a;
        dst[1] = b;
    }
}

void validate(const ksvm_nfft_ipm_config& c) {  // P:src/ipm.cpp:10-21
    if (!(c.C > 0.0)) throw std::invalid_argument("C must be positive");
    if (!(c.sigma > 0.0 && c.sigma < 1.0)) throw std::invalid_argument("sigma must lie in (0, 1)");
    if (!(c.gamma0 > 0.0 && c.gamma0 < 1.0)) throw std::invalid_argument("gamma0 must lie in (0, 1)");
    if (!(c.tol_ip > 0.0) || !(c.tol_gmres > 0.0)) throw std::invalid_argument("tolerances must be positive");
    if (c.max_ip_iters < 1 || c.max_gmres_iters < 1) throw std::invalid_argument("iteration caps must be >= 1");
    if (!(c.mu0 > 0.0)) throw std::invalid_argument("mu0 must be positive");
}

struct Handles {  // owns the saddle operator / preconditioner of one training run
    ksvm_nfft_saddle* s = nullptr;
    ksvm_nfft_precond* p = nullptr;
    cudaStream_t st = nullptr;
    ~Handles() {
        if (s) ksvm_nfft_saddle_free(s);
        if (p) ksvm_nfft_precond_free(p);
        if (st) cudaStreamDestroy(st);
    }
};

void ok(int rc, const char* who) {
    if (rc == KSVM_NFFT_OK) return;
    const std::string msg = std::string(who) + ": " + ksvm_nfft_last_error();
    if (rc == KSVM_NFFT_ERR_CONFIG) throw std::invalid_argument(msg);
    if (rc == KSVM_NFFT_ERR_DATA) throw DomainErr(msg);
    throw std::runtime_error(msg);
}

}  // namespace
}  // namespace ksvm_nfft

using namespace ksvm_nfft;

extern "C" {

void ksvm_nfft_ipm_config_default(ksvm_nfft_ipm_config* c) {  // P:include/ksvm/ipm.hpp:15-24
    if (!c) return;
    c->C = 0.5;
    c->sigma = 0.6;
    c->gamma0 = 0.99995;
    c->tol_ip = 1e-1;
    c->max_ip_iters = 50;
    c->tol_gmres = 1e-3;
    c->max_gmres_iters = 100;
    c->mu0 = 1.0;
}

int ksvm_nfft_ipm_train(const ksvm_nfft_op* op, const double* y_h, const double* Z, int k, int z_ptr_kind,
                        const ksvm_nfft_ipm_config* cfg, double* alpha_out, ksvm_nfft_ipm_result* result,
                        ksvm_nfft_ipm_log* log) {
    return guarded([&] {
        if (!op || !y_h || !cfg || !alpha_out || !result) throw std::invalid_argument("ipm_train: null argument");
        validate(*cfg);
        const ksvm_nfft_ipm_config c = *cfg;
        const int64_t n = ksvm_nfft_op_size(op);
        for (int64_t i = 0; i < n; ++i)  // P:src/ipm.cpp:82-85
            if (y_h[i] != 1.0 && y_h[i] != -1.0) throw std::invalid_argument("ipm_train: labels must be +-1");
        const size_t N = static_cast<size_t>(n), N1 = N + 1;
        const double C = c.C;
        // initial_alpha (P:src/ipm.cpp:66-74): the reference's RNG stream
        std::vector<double> alpha0(N);
        {
            std::mt19937_64 rng(0x5EED5EEDull);
            std::uniform_real_distribution<double> unif(0.0, 1.0);
            for (size_t j = 0; j < N; ++j) alpha0[j] = C * (0.4 + 0.2 * unif(rng));
        }
        const int dev = ksvm_nfft_op_device(op);
        DeviceGuard dg(dev);
        Handles H;
        CK(cudaStreamCreateWithFlags(&H.st, cudaStreamNonBlocking));
        cudaStream_t st = H.st;
        DevBuf<double> y, alpha, u, kv, theta, rhs, delta, pa, pb, scal;
        y.upload(y_h, N, st);
        alpha.upload(alpha0.data(), N, st);
        u.alloc(N);
        kv.alloc(N);
        theta.alloc(N);
        rhs.alloc(N1);
        delta.alloc(N1);
        pa.alloc(kRB);
        pb.alloc(kRB);
        scal.alloc(4);
        double* hs = nullptr;
        CK(cudaMallocHost(&hs, 4 * sizeof(double)));
        std::unique_ptr<double, decltype(&cudaFreeHost)> hs_guard(hs, &cudaFreeHost);
        const int nb = reduce_blocks(n);
        auto matvec = [&] {  // kv = K u
            ok(ksvm_nfft_op_apply(op, u.p, kv.p, KSVM_NFFT_DEVICE, st), "ipm_train matvec");
        };
        auto fetch2 = [&](const double* p1, const double* p2, int min_mode) {
            launch_k(ki_finish2, dim3(1), dim3(32), 0, st, p1, p2, nb, scal.p, min_mode);
            ++launch_counter();
            CK(cudaMemcpyAsync(hs, scal.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        };
        // yky(alpha), xi_alpha0, xi_lambda0 (P:src/ipm.cpp:87-99)
        launch_k(ki_yalpha, dim3(nb), dim3(kRT), 0, st, u.p, static_cast<const double*>(y.p),
                 static_cast<const double*>(alpha.p), static_cast<long long>(n), pa.p);
        ++launch_counter();
        matvec();
        double lambda = 0.0, mu = c.mu0;
        launch_k(ki_newton, dim3(nb), dim3(kRT), 0, st, static_cast<double*>(nullptr), static_cast<double*>(nullptr),
                 static_cast<const double*>(alpha.p), static_cast<const double*>(y.p),
                 static_cast<const double*>(kv.p), lambda, mu, C, static_cast<long long>(n), pb.p);
        ++launch_counter();
        CK(cudaGetLastError());
        fetch2(pa.p, pb.p, 0);
        const double xi_alpha0 = std::fabs(hs[0]);
        const double xi_lambda0 = std::sqrt(hs[1]);
        if (xi_alpha0 == 0.0 || xi_lambda0 == 0.0)
            throw std::runtime_error("ipm_train: degenerate initial infeasibility");

        // SaddlePreconditioner(factor, y) (P:src/ipm.cpp:101); the operator is
        // created once and re-pointed at each iteration's Theta.
        std::vector<double> ones(N, 1.0);
        ok(ksvm_nfft_saddle_create(op, y_h, ones.data(), &H.s), "ipm_train");
        ok(ksvm_nfft_precond_create_ex(Z, Z ? k : 0, n, y_h, dev, z_ptr_kind, st, &H.p), "ipm_train");

        double xi_a = 1.0, xi_l = 1.0, gm_sum = 0.0;
        int it = 0, streak = 0, status = -1;
        while ((mu > c.tol_ip || xi_a > c.tol_ip || xi_l > c.tol_ip) && it < c.max_ip_iters) {
            mu *= c.sigma;
            // Theta and the Newton right-hand side (rhs[n] = y . alpha from the last update)
            launch_k(ki_newton, dim3(nb), dim3(kRT), 0, st, rhs.p, theta.p, static_cast<const double*>(alpha.p),
                     static_cast<const double*>(y.p), static_cast<const double*>(kv.p), lambda, mu, C,
                     static_cast<long long>(n), pb.p);
            launch_k(ki_yalpha, dim3(nb), dim3(kRT), 0, st, u.p, static_cast<const double*>(y.p),
                     static_cast<const double*>(alpha.p), static_cast<long long>(n), pa.p);
            launch_k(ki_finish2, dim3(1), dim3(32), 0, st, static_cast<const double*>(pa.p),
                     static_cast<const double*>(nullptr), nb, rhs.p + n, 0);
            launch_counter() += 3;
            CK(cudaGetLastError());
            ok(ksvm_nfft_saddle_set_theta_ex(H.s, theta.p, KSVM_NFFT_DEVICE, st), "ipm_train");
            ok(ksvm_nfft_precond_refresh_ex(H.p, theta.p, KSVM_NFFT_DEVICE, st), "ipm_train");
            ksvm_nfft_gmres_stats gs{};
            ok(ksvm_nfft_gmres_solve(H.s, H.p, rhs.p, c.tol_gmres, c.max_gmres_iters, delta.p, &gs, nullptr,
                                     KSVM_NFFT_DEVICE, st),
               "ipm_train");
            // step_lengths (P:src/ipm.cpp:44-55)
            launch_k(ki_step_min, dim3(nb), dim3(kRT), 0, st, static_cast<const double*>(alpha.p),
                     static_cast<const double*>(delta.p), C, static_cast<long long>(n), pa.p);
            ++launch_counter();
            CK(cudaMemcpyAsync(hs + 2, delta.p + n, sizeof(double), cudaMemcpyDeviceToHost, st));
            fetch2(pa.p, nullptr, 1);  // syncs: hs[0] = min ratio, hs[2] = dlambda
            const double smax = std::min(1.0, hs[0]);
            const double s_alpha = c.gamma0 * smax, s_lambda = c.gamma0;
            lambda += s_lambda * hs[2];
            // alpha update, yky(alpha), infeasibilities (P:src/ipm.cpp:119-128)
            launch_k(ki_update, dim3(nb), dim3(kRT), 0, st, alpha.p, u.p, static_cast<const double*>(delta.p),
                     static_cast<const double*>(y.p), s_alpha, static_cast<long long>(n), pa.p);
            ++launch_counter();
            matvec();
            launch_k(ki_newton, dim3(nb), dim3(kRT), 0, st, static_cast<double*>(nullptr),
                     static_cast<double*>(nullptr), static_cast<const double*>(alpha.p),
                     static_cast<const double*>(y.p), static_cast<const double*>(kv.p), lambda, mu, C,
                     static_cast<long long>(n), pb.p);
            ++launch_counter();
            CK(cudaGetLastError());
            fetch2(pa.p, pb.p, 0);
            xi_a = std::fabs(hs[0]) / xi_alpha0;
            xi_l = std::sqrt(hs[1]) / xi_lambda0;
            if (log) {
                ksvm_nfft_ipm_log& L = log[it];
                L.it = it;
                L.mu = mu;
                L.xi_alpha_rel = xi_a;
                L.xi_lambda_rel = xi_l;
                L.step_alpha = s_alpha;
                L.gmres_iterations = gs.iterations;
                L.gmres_relative_residual = gs.relative_residual;
                L.gmres_converged = gs.converged;
                L.gmres_breakdown = gs.breakdown;
            }
            gm_sum += gs.iterations;
            ++it;
            streak = gs.converged ? 0 : streak + 1;  // P:src/ipm.cpp:138-143
            if (streak > 3) {
                status = KSVM_NFFT_IPM_STALLED;
                break;
            }
        }
        if (status != KSVM_NFFT_IPM_STALLED)
            status = (mu <= c.tol_ip && xi_a <= c.tol_ip && xi_l <= c.tol_ip) ? KSVM_NFFT_IPM_CONVERGED
                                                                             : KSVM_NFFT_IPM_MAX_ITERATIONS;
        CK(cudaMemcpyAsync(alpha_out, alpha.p, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        ksvm_nfft_ipm_result r{};
        r.lambda = lambda;
        r.mu_final = mu;
        r.xi_alpha_rel = xi_a;
        r.xi_lambda_rel = xi_l;
        r.status = status;
        r.iterations = it;
        r.mean_gmres_iters = it ? gm_sum / it : 0.0;
        *result = r;
    });
}

// P:src/ipm.cpp:157-185: the matvec K (alpha .* y) on the GPU, the
// support-vector selection and mean / median on the host in index order
int ksvm_nfft_compute_bias(const ksvm_nfft_op* op, const double* alpha, const double* y, double C, double eps_sv,
                           double* bias, int64_t* n_support) {
    return guarded([&] {
        if (!op || !alpha || !y || !bias) throw std::invalid_argument("compute_bias: null argument");
        const int64_t n = ksvm_nfft_op_size(op);
        std::vector<double> ay(static_cast<size_t>(n)), kay(static_cast<size_t>(n));
        for (int64_t j = 0; j < n; ++j) ay[static_cast<size_t>(j)] = alpha[j] * y[j];
        ok(ksvm_nfft_op_apply(op, ay.data(), kay.data(), KSVM_NFFT_HOST, nullptr), "compute_bias");
        std::vector<double> free_vals, sv_vals;
        for (int64_t j = 0; j < n; ++j) {
            if (alpha[j] > eps_sv) {
                const double val = y[j] - kay[static_cast<size_t>(j)];
                sv_vals.push_back(val);
                if (alpha[j] < C - eps_sv) free_vals.push_back(val);
            }
        }
        if (n_support) *n_support = static_cast<int64_t>(sv_vals.size());
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
            *bias = 0.0;  // the reference also warns on stderr
        }
    });
}

// balance_and_split (P:src/dataset.cpp:212-262), index form: the same
// libstdc++ std::mt19937_64 / std::shuffle stream as the reference, so the
// split is identical. train_idx (sorted) and test_idx need room for n entries.
int ksvm_nfft_balance_and_split(const double* labels, int64_t n, double train_fraction, uint64_t seed,
                                int64_t* train_idx, int64_t* n_train, int64_t* test_idx, int64_t* n_test) {
    return guarded([&] {
        if (!labels || !train_idx || !n_train || !test_idx || !n_test)
            throw std::invalid_argument("balance_and_split: null argument");
        if (!(train_fraction > 0.0 && train_fraction < 1.0)) throw DomainErr("train_fraction must lie in (0, 1)");
        int64_t npos = 0;
        for (int64_t i = 0; i < n; ++i)
            if (labels[i] > 0) ++npos;
        if (npos == 0 || npos == n) throw DomainErr("both classes must be present before splitting");
        std::mt19937_64 rng(seed);
        std::vector<int64_t> perm(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) perm[static_cast<size_t>(i)] = i;
        std::shuffle(perm.begin(), perm.end(), rng);
        const auto nt = static_cast<int64_t>(std::floor(train_fraction * static_cast<double>(n)));
        std::vector<int64_t> pos, neg;
        for (int64_t r = 0; r < nt; ++r) {
            const int64_t i = perm[static_cast<size_t>(r)];
            (labels[i] > 0 ? pos : neg).push_back(i);
        }
        auto& majority = pos.size() > neg.size() ? pos : neg;
        const size_t keep = std::min(pos.size(), neg.size());
        std::shuffle(majority.begin(), majority.end(), rng);
        majority.resize(keep);
        if (keep == 0 || pos.size() + neg.size() < 2) throw DomainErr("balancing leaves fewer than 2 training points");
        std::vector<int64_t> bal(pos);
        bal.insert(bal.end(), neg.begin(), neg.end());
        std::sort(bal.begin(), bal.end());
        std::copy(bal.begin(), bal.end(), train_idx);
        *n_train = static_cast<int64_t>(bal.size());
        std::copy(perm.begin() + nt, perm.end(), test_idx);
        *n_test = n - nt;
    });
}

}  // extern "C"
