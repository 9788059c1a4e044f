// GPU fast prediction: the reference's
// TrainedModel::decision_values (P:src/ipm.cpp:213-288) for both backends.
//   kFast: per window a plan over the training points with fit 1/1.2
//   (:258), the targets whose scaled norm is <= r_T (:261-265) evaluated by
//   apply_fastsum_cross and added with weight eta_l in window order
//   (:266-275); targets outside the ball in any window are recomputed
//   exactly (:278-284);
//   kExact: every target exactly (:236-239).
// f + bias is returned. The exact sums run on the GPU (one CTA per target,
// fixed-order block reduction) with anova_eval's arithmetic
// (P:src/kernel.cpp:15-29); the fast part reuses the plan C ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "capi_common.cuh"

namespace ksvm_nfft {
namespace {

// out[r] = sum_i coeff_i sum_l w_l exp(-||x_i^l - t_r^l||^2 / ell_l^2)
// train: n x d column-major (ld n); targets: m x d column-major (ld m)
__global__ void __launch_bounds__(256) k_exact_anova(const double* __restrict__ train, long long n,
                                                     const int* __restrict__ woff, const int* __restrict__ feat, int P,
                                                     const double* __restrict__ w, const double* __restrict__ ell2,
                                                     const double* __restrict__ coeff, const double* __restrict__ tgt,
                                                     long long m, const long long* __restrict__ rows,
                                                     double* __restrict__ out) {
    const long long rr = blockIdx.x;
    const long long tr = rows[rr];
    double acc = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        double sum = 0.0;
        for (int l = 0; l < P; ++l) {
            double d2 = 0.0;
            for (int q = woff[l]; q < woff[l + 1]; ++q) {
                const int f = feat[q];
                const double diff = train[static_cast<long long>(f) * n + i] - tgt[static_cast<long long>(f) * m + tr];
                d2 += diff * diff;
            }
            sum += w[l] * exp(-d2 / ell2[l]);
        }
        acc += coeff[i] * sum;
    }
    __shared__ double sh[8];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) s += sh[q];
        out[rr] = s;
    }
}

double at(const double* p, int64_t i, int64_t j, int64_t ld, int layout) {
    return layout == KSVM_NFFT_ROW_MAJOR ? p[i * ld + j] : p[j * ld + i];
}

}  // namespace
}  // namespace ksvm_nfft

using namespace ksvm_nfft;

extern "C" int ksvm_nfft_decision_values(const double* train, int64_t n, int d, int64_t ld_train, int layout,
                                         const int* window_features, const int* window_sizes, int P,
                                         const double* weights, const double* length_scales,
                                         const ksvm_nfft_config* cfg, const double* coeff, double bias,
                                         const double* test, int64_t t, int64_t ld_test, int backend, int device,
                                         double* f_out, int64_t* n_exact) {
    return guarded([&] {
        if (!train || !window_features || !window_sizes || !weights || !length_scales || !coeff || !f_out ||
            (t > 0 && !test))
            throw std::invalid_argument("decision_values: null argument");
        if (n < 1 || d < 1 || P < 1 || t < 0) throw std::invalid_argument("decision_values: bad sizes");
        if (backend != KSVM_NFFT_PREDICT_EXACT && backend != KSVM_NFFT_PREDICT_FAST)
            throw std::invalid_argument("decision_values: bad backend");
        const int64_t ldt = layout == KSVM_NFFT_ROW_MAJOR ? d : n, lds = layout == KSVM_NFFT_ROW_MAJOR ? d : t;
        if (ld_train < ldt || (t > 0 && ld_test < lds)) throw std::invalid_argument("decision_values: bad ld");
        ksvm_nfft_config c;
        if (cfg) {
            c = *cfg;
        } else {
            ksvm_nfft_config_default(&c);
        }
        std::vector<int> woff(static_cast<size_t>(P) + 1, 0);
        for (int l = 0; l < P; ++l) {
            if (window_sizes[l] < 1) throw std::invalid_argument("decision_values: empty window");
            woff[static_cast<size_t>(l) + 1] = woff[static_cast<size_t>(l)] + window_sizes[l];
        }
        for (int q = 0; q < woff[static_cast<size_t>(P)]; ++q)
            if (window_features[q] < 0 || window_features[q] >= d)
                throw std::invalid_argument("decision_values: feature index out of range");
        std::vector<double> f(static_cast<size_t>(t), 0.0);
        std::vector<char> offending(static_cast<size_t>(t), backend == KSVM_NFFT_PREDICT_EXACT ? 1 : 0);
        if (backend == KSVM_NFFT_PREDICT_FAST) {
            // P:src/ipm.cpp:247-276. Windows are independent (own plan, own
            // stream), so they run on concurrent host threads; their parts are
            // added to f afterwards in window order (the reference's order).
            struct WinOut {
                std::vector<int64_t> ok;
                std::vector<double> part;
                std::vector<char> off;
                std::string err;
            };
            std::vector<WinOut> outs(static_cast<size_t>(P));
            auto work = [&](int l) {
                WinOut& o = outs[static_cast<size_t>(l)];
                try {
                    const int dl = window_sizes[l];
                    std::vector<double> src(static_cast<size_t>(n) * dl), tgt(static_cast<size_t>(t) * dl);
                    for (int q = 0; q < dl; ++q) {
                        const int fq = window_features[woff[static_cast<size_t>(l)] + q];
                        for (int64_t i = 0; i < n; ++i) src[static_cast<size_t>(q * n + i)] = at(train, i, fq, ld_train, layout);
                        for (int64_t j = 0; j < t; ++j) tgt[static_cast<size_t>(q * t + j)] = at(test, j, fq, ld_test, layout);
                    }
                    ksvm_nfft_plan* plan = nullptr;
                    int rc = ksvm_nfft_plan_create(src.data(), n, dl, n, KSVM_NFFT_COL_MAJOR, length_scales[l], &c,
                                                   1.0 / 1.2, device, &plan);
                    if (rc != KSVM_NFFT_OK) throw std::runtime_error(ksvm_nfft_last_error());
                    std::unique_ptr<ksvm_nfft_plan, void (*)(ksvm_nfft_plan*)> guard(plan, ksvm_nfft_plan_free);
                    std::vector<double> scaled(static_cast<size_t>(t) * dl);
                    if (t > 0) {
                        rc = ksvm_nfft_plan_scale_points(plan, tgt.data(), t, t, KSVM_NFFT_COL_MAJOR, scaled.data());
                        if (rc != KSVM_NFFT_OK) throw std::runtime_error(ksvm_nfft_last_error());
                    }
                    o.off.assign(static_cast<size_t>(t), 0);
                    for (int64_t j = 0; j < t; ++j) {
                        double s2 = 0.0;
                        for (int q = 0; q < dl; ++q) s2 += scaled[static_cast<size_t>(q * t + j)] * scaled[static_cast<size_t>(q * t + j)];
                        if (std::sqrt(s2) <= c.torus_radius)
                            o.ok.push_back(j);
                        else
                            o.off[static_cast<size_t>(j)] = 1;
                    }
                    if (o.ok.empty()) return;
                    const int64_t m = static_cast<int64_t>(o.ok.size());
                    std::vector<double> tok(static_cast<size_t>(m) * dl);
                    o.part.resize(static_cast<size_t>(m));
                    for (int q = 0; q < dl; ++q)
                        for (int64_t r = 0; r < m; ++r)
                            tok[static_cast<size_t>(q * m + r)] = tgt[static_cast<size_t>(q * t + o.ok[static_cast<size_t>(r)])];
                    rc = ksvm_nfft_plan_apply_cross(plan, tok.data(), m, m, KSVM_NFFT_COL_MAJOR, coeff, o.part.data(),
                                                    KSVM_NFFT_HOST, nullptr);
                    if (rc != KSVM_NFFT_OK) throw std::runtime_error(ksvm_nfft_last_error());
                } catch (const std::exception& e) {
                    o.err = e.what();
                }
            };
            const int nthr = std::max(1, std::min<int>(P, static_cast<int>(std::thread::hardware_concurrency())));
            std::atomic<int> next{0};
            std::vector<std::thread> pool;
            for (int k = 0; k < nthr; ++k)
                pool.emplace_back([&] {
                    for (int l = next++; l < P; l = next++) work(l);
                });
            for (auto& th : pool) th.join();
            for (int l = 0; l < P; ++l) {
                const WinOut& o = outs[static_cast<size_t>(l)];
                if (!o.err.empty()) throw std::runtime_error(o.err);
                for (int64_t j = 0; j < t; ++j)
                    if (o.off[static_cast<size_t>(j)]) offending[static_cast<size_t>(j)] = 1;
                for (size_t r = 0; r < o.ok.size(); ++r) f[static_cast<size_t>(o.ok[r])] += weights[l] * o.part[r];
            }
        }
        std::vector<long long> redo;
        for (int64_t j = 0; j < t; ++j)
            if (offending[static_cast<size_t>(j)]) redo.push_back(j);
        if (!redo.empty()) {  // exact sums (P:src/ipm.cpp:222-233, 278-284)
            DeviceGuard dg(device);
            cudaStream_t st;
            CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            std::unique_ptr<CUstream_st, cudaError_t (*)(cudaStream_t)> sguard(st, cudaStreamDestroy);
            std::vector<double> tr_cm(static_cast<size_t>(n) * d), te_cm(static_cast<size_t>(t) * d), ell2(static_cast<size_t>(P));
            for (int q = 0; q < d; ++q) {
                for (int64_t i = 0; i < n; ++i) tr_cm[static_cast<size_t>(q * n + i)] = at(train, i, q, ld_train, layout);
                for (int64_t j = 0; j < t; ++j) te_cm[static_cast<size_t>(q * t + j)] = at(test, j, q, ld_test, layout);
            }
            for (int l = 0; l < P; ++l) ell2[static_cast<size_t>(l)] = length_scales[l] * length_scales[l];
            DevBuf<double> dtr, dte, dw, de, dc, dout;
            DevBuf<int> doff, dfeat;  // per-call buffers: concurrent calls share nothing
            DevBuf<long long> drows;
            dtr.upload(tr_cm.data(), tr_cm.size(), st);
            dte.upload(te_cm.data(), te_cm.size(), st);
            dw.upload(weights, static_cast<size_t>(P), st);
            de.upload(ell2.data(), ell2.size(), st);
            dc.upload(coeff, static_cast<size_t>(n), st);
            doff.upload(woff.data(), woff.size(), st);
            drows.upload(redo.data(), redo.size(), st);
            dout.alloc(redo.size());
            dfeat.upload(window_features, static_cast<size_t>(woff[static_cast<size_t>(P)]), st);
            k_exact_anova<<<static_cast<unsigned>(redo.size()), 256, 0, st>>>(dtr.p, n, doff.p, dfeat.p, P, dw.p, de.p,
                                                                               dc.p, dte.p, t, drows.p, dout.p);
            ++launch_counter();
            CK(cudaGetLastError());
            std::vector<double> vals(redo.size());
            CK(cudaMemcpyAsync(vals.data(), dout.p, sizeof(double) * vals.size(), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            for (size_t r = 0; r < redo.size(); ++r) f[static_cast<size_t>(redo[r])] = vals[r];
        }
        for (int64_t j = 0; j < t; ++j) f_out[j] = f[static_cast<size_t>(j)] + bias;
        if (n_exact) *n_exact = static_cast<int64_t>(redo.size());
    });
}
