// Drop-in replacement for the reference's P:src/fastsum.cpp on the B200 path.
//
// This translation unit implements the reference's own header,
// P:include/ksvm/fastsum.hpp (FastsumConfig::validate, FastsumPlan and its
// accessors, plan_fastsum, apply_fastsum, apply_fastsum_cross,
// anova_fast_operator), on top of the C ABI in include/ksvm_nfft.h
// (libksvm_nfft.so). A maintainer swaps it for src/fastsum.cpp in the ksvm
// library target and every caller of the hot path - the IPM
// (P:src/ipm.cpp:91-93,128,167), GMRES (P:src/saddle.cpp:29,175), the
// Nystrom sketch through FastWindowOperator (P:src/pipeline.cpp:114-133),
// fast prediction (P:src/ipm.cpp:258-274) and train_on_prepared's operator
// (P:src/pipeline.cpp:200-203) - runs on the GPU unchanged. Nothing else in
// the reference is modified; FFTW is no longer needed.
//
// Exceptions follow the reference: std::invalid_argument for configuration
// and shape errors (status 4), DomainError for cross targets outside the
// torus ball (status 2), std::runtime_error for CUDA failures (status 5).
// The device is $KSVM_NFFT_DEVICE (default 0). Plans and operators are
// immutable; concurrent apply() calls are safe (the C ABI serialises them on
// the object's stream), as P:include/ksvm/kernel.hpp:28-31 requires.
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ksvm/fastsum.hpp"
#include "ksvm_nfft.h"

namespace ksvm {

namespace {

int device_id() {
    const char* e = std::getenv("KSVM_NFFT_DEVICE");
    return e ? std::atoi(e) : 0;
}

ksvm_nfft_config to_c(const FastsumConfig& c) {
    ksvm_nfft_config r;
    r.bandwidth = c.bandwidth;
    r.window_cutoff = c.window_cutoff;
    r.oversampling = c.oversampling;
    r.torus_radius = c.torus_radius;
    return r;
}

[[noreturn]] void raise(int status, bool domain = false) {
    const std::string msg = ksvm_nfft_last_error();
    if (status == KSVM_NFFT_ERR_CONFIG) throw std::invalid_argument(msg);
    if (status == KSVM_NFFT_ERR_DATA && domain) throw DomainError(msg);
    throw std::runtime_error(msg);
}

void check(int status, bool domain = false) {
    if (status != KSVM_NFFT_OK) raise(status, domain);
}

}  // namespace

// P:src/fastsum.cpp:38-47
void FastsumConfig::validate() const {
    const ksvm_nfft_config c = to_c(*this);
    check(ksvm_nfft_config_validate(&c));
}

// P:src/fastsum.cpp:49-92: the plan is the device plan handle.
struct FastsumPlan::Impl {
    ksvm_nfft_plan* h = nullptr;
    Eigen::Index n = 0;
    int d = 0;
    ~Impl() { ksvm_nfft_plan_free(h); }
};

FastsumPlan::FastsumPlan() : impl_(std::make_unique<Impl>()) {}
FastsumPlan::~FastsumPlan() = default;
FastsumPlan::FastsumPlan(FastsumPlan&&) noexcept = default;
FastsumPlan& FastsumPlan::operator=(FastsumPlan&&) noexcept = default;

Eigen::Index FastsumPlan::num_sources() const { return impl_->n; }
int FastsumPlan::dim() const { return impl_->d; }
double FastsumPlan::scaled_length() const { return ksvm_nfft_plan_scaled_length(impl_->h); }
double FastsumPlan::coefficient_sum() const { return ksvm_nfft_plan_coefficient_sum(impl_->h); }

// P:src/fastsum.cpp:99-101 (same affine map, computed by the library)
Eigen::MatrixXd FastsumPlan::scale_points(const Eigen::MatrixXd& pts) const {
    if (pts.cols() != impl_->d) throw std::invalid_argument("scale_points: dimension mismatch");
    Eigen::MatrixXd out(pts.rows(), pts.cols());
    if (pts.rows() == 0) return out;
    check(ksvm_nfft_plan_scale_points(impl_->h, pts.data(), pts.rows(), pts.rows(), KSVM_NFFT_COL_MAJOR,
                                      out.data()));
    return out;
}

// P:src/fastsum.cpp:103-209
FastsumPlan plan_fastsum(const Eigen::MatrixXd& points, const GaussianKernelSpec& spec,
                         const FastsumConfig& cfg, double fit_fraction) {
    cfg.validate();
    const ksvm_nfft_config c = to_c(cfg);
    FastsumPlan plan;
    plan.impl_->n = points.rows();
    plan.impl_->d = static_cast<int>(points.cols());
    check(ksvm_nfft_plan_create(points.data(), points.rows(), static_cast<int>(points.cols()), points.rows(),
                                KSVM_NFFT_COL_MAJOR, spec.length_scale, &c, fit_fraction, device_id(),
                                &plan.impl_->h));
    return plan;
}

// P:src/fastsum.cpp:300-305
Eigen::VectorXd apply_fastsum(const FastsumPlan& plan, const Eigen::VectorXd& v) {
    const auto& im = *plan.impl_;
    if (v.size() != im.n) throw std::invalid_argument("apply_fastsum: vector length mismatch");
    Eigen::VectorXd out(im.n);
    check(ksvm_nfft_plan_apply(im.h, v.data(), out.data(), KSVM_NFFT_HOST, nullptr));
    return out;
}

// P:src/fastsum.cpp:307-322
Eigen::VectorXd apply_fastsum_cross(const FastsumPlan& plan, const Eigen::MatrixXd& targets,
                                    const Eigen::VectorXd& v) {
    const auto& im = *plan.impl_;
    if (v.size() != im.n) throw std::invalid_argument("apply_fastsum_cross: vector length mismatch");
    if (targets.cols() != im.d) throw std::invalid_argument("apply_fastsum_cross: target dimension mismatch");
    Eigen::VectorXd out(targets.rows());
    if (targets.rows() == 0) return out;
    check(ksvm_nfft_plan_apply_cross(im.h, targets.data(), targets.rows(), targets.rows(), KSVM_NFFT_COL_MAJOR,
                                     v.data(), out.data(), KSVM_NFFT_HOST, nullptr),
          /*domain=*/true);
    return out;
}

namespace {

// P:src/fastsum.cpp:326-362: the ANOVA operator, window sum on the device.
class GpuAnovaOperator final : public KernelOperator {
public:
    GpuAnovaOperator(const Dataset& data, const AnovaKernelSpec& spec, const FastsumConfig& cfg,
                     double fit_fraction)
        : n_(data.n()) {
        check_windowing(spec.windowing, static_cast<int>(data.dim()));
        cfg.validate();
        const auto& w = spec.windowing;
        std::vector<int> feats, sizes;
        for (const auto& win : w.windows) {
            sizes.push_back(static_cast<int>(win.size()));
            feats.insert(feats.end(), win.begin(), win.end());
        }
        const ksvm_nfft_config c = to_c(cfg);
        check(ksvm_nfft_op_create(data.points.data(), data.n(), data.dim(), data.n(), KSVM_NFFT_COL_MAJOR,
                                  feats.data(), sizes.data(), w.num_windows(), w.weights.data(),
                                  w.length_scales.data(), &c, fit_fraction, nullptr, device_id(), KSVM_NFFT_FP64,
                                  &op_));
    }
    ~GpuAnovaOperator() override { ksvm_nfft_op_free(op_); }
    GpuAnovaOperator(const GpuAnovaOperator&) = delete;
    GpuAnovaOperator& operator=(const GpuAnovaOperator&) = delete;

    Eigen::Index size() const override { return n_; }

    // KernelOperator::apply (P:include/ksvm/kernel.hpp:36): host vectors in
    // and out; the call uploads v, runs the cached apply graph, downloads y.
    Eigen::VectorXd apply(const Eigen::VectorXd& v) const override {
        if (v.size() != n_) throw std::invalid_argument("AnovaFastOperator: vector length mismatch");
        Eigen::VectorXd out(n_);
        check(ksvm_nfft_op_apply(op_, v.data(), out.data(), KSVM_NFFT_HOST, nullptr));
        return out;
    }

    // P:src/fastsum.cpp:354-356 (exact anova_eval entry)
    double entry(Eigen::Index i, Eigen::Index j) const override { return ksvm_nfft_op_entry(op_, i, j); }

private:
    Eigen::Index n_;
    ksvm_nfft_op* op_ = nullptr;
};

}  // namespace

// P:src/fastsum.cpp:366-371
std::unique_ptr<KernelOperator> anova_fast_operator(const Dataset& data, const AnovaKernelSpec& spec,
                                                    const FastsumConfig& cfg, double fit_fraction) {
    return std::make_unique<GpuAnovaOperator>(data, spec, cfg, fit_fraction);
}

}  // namespace ksvm
