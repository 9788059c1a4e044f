// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Exact multi-dimensional complex DFT used by (a) the oracle restatement of
// the reference hot path and (b) the FFTW shim through which the reference's
// own fastsum.cpp is compiled (oracle/shim/fftw3.h). It reproduces the FFTW
// semantics the reference relies on (P:src/fastsum.cpp:161-172, 201-207,
// 273, 282):
//   * unnormalised transform, sign -1 (FFTW_FORWARD) or +1 (FFTW_BACKWARD),
//   * row-major multi-index (dimension 0 slowest),
//   * out-of-place, input preserved.
// Power-of-two lengths use an iterative radix-2 Cooley-Tukey with twiddles
// evaluated in long double; other lengths use a direct DFT whose twiddle
// angle is reduced exactly (k*j mod n). Both agree with FFTW to a few ulp
// relative to the transform's magnitude, which is all the reference's
// arithmetic (and the 1e-10 parity bar) can see.
#ifndef KSVM_ORACLE_OFFT_HPP
#define KSVM_ORACLE_OFFT_HPP

#include <cmath>
#include <complex>
#include <cstddef>
#include <vector>

namespace offt {

using cd = std::complex<double>;

class Plan1D {
public:
    Plan1D() = default;
    Plan1D(int n, int sign) : n_(n), sign_(sign) {
        pow2_ = n > 0 && (n & (n - 1)) == 0;
        tw_.resize(static_cast<std::size_t>(n));
        const long double two_pi = 6.283185307179586476925286766559005768L;
        for (int k = 0; k < n; ++k) {
            const long double ang = sign * two_pi * k / n;
            tw_[static_cast<std::size_t>(k)] =
                cd(static_cast<double>(std::cos(ang)), static_cast<double>(std::sin(ang)));
        }
        if (pow2_) {
            rev_.resize(static_cast<std::size_t>(n));
            int lg = 0;
            while ((1 << lg) < n) ++lg;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int b = 0; b < lg; ++b)
                    if (i & (1 << b)) r |= 1 << (lg - 1 - b);
                rev_[static_cast<std::size_t>(i)] = r;
            }
        }
    }

    // In-place transform of a contiguous line; scratch must hold n entries.
    void run(cd* x, cd* scratch) const {
        const int n = n_;
        if (n == 1) return;
        if (pow2_) {
            for (int i = 0; i < n; ++i) scratch[rev_[static_cast<std::size_t>(i)]] = x[i];
            for (int len = 2; len <= n; len <<= 1) {
                const int half = len >> 1;
                const int step = n / len;
                for (int s = 0; s < n; s += len) {
                    for (int j = 0; j < half; ++j) {
                        const cd w = tw_[static_cast<std::size_t>(j * step)];
                        const cd u = scratch[s + j];
                        const cd t = w * scratch[s + j + half];
                        scratch[s + j] = u + t;
                        scratch[s + j + half] = u - t;
                    }
                }
            }
            for (int i = 0; i < n; ++i) x[i] = scratch[i];
        } else {
            for (int k = 0; k < n; ++k) {
                cd acc(0.0, 0.0);
                for (int j = 0; j < n; ++j)
                    acc += x[j] * tw_[static_cast<std::size_t>((static_cast<long long>(k) * j) % n)];
                scratch[k] = acc;
            }
            for (int i = 0; i < n; ++i) x[i] = scratch[i];
        }
    }

    int size() const { return n_; }

private:
    int n_ = 0;
    int sign_ = -1;
    bool pow2_ = false;
    std::vector<cd> tw_;
    std::vector<int> rev_;
};

// Multi-dimensional plan (row-major). Thread-safe execute: all scratch is
// per call.
class PlanND {
public:
    PlanND() = default;
    PlanND(const std::vector<int>& dims, int sign) : dims_(dims) {
        for (int n : dims) lines_.emplace_back(n, sign);
        total_ = 1;
        for (int n : dims) total_ *= static_cast<std::size_t>(n);
    }

    void execute(const cd* in, cd* out) const {
        if (out != in)
            for (std::size_t i = 0; i < total_; ++i) out[i] = in[i];
        const int d = static_cast<int>(dims_.size());
        int maxn = 1;
        for (int n : dims_) maxn = n > maxn ? n : maxn;
        std::vector<cd> line(static_cast<std::size_t>(maxn)), scratch(static_cast<std::size_t>(maxn));
        for (int ax = 0; ax < d; ++ax) {
            const std::size_t n = static_cast<std::size_t>(dims_[static_cast<std::size_t>(ax)]);
            std::size_t stride = 1;
            for (int t = ax + 1; t < d; ++t) stride *= static_cast<std::size_t>(dims_[static_cast<std::size_t>(t)]);
            const std::size_t outer = total_ / (n * stride);
            for (std::size_t o = 0; o < outer; ++o) {
                for (std::size_t s = 0; s < stride; ++s) {
                    cd* base = out + o * n * stride + s;
                    for (std::size_t k = 0; k < n; ++k) line[k] = base[k * stride];
                    lines_[static_cast<std::size_t>(ax)].run(line.data(), scratch.data());
                    for (std::size_t k = 0; k < n; ++k) base[k * stride] = line[k];
                }
            }
        }
    }

    std::size_t total() const { return total_; }

private:
    std::vector<int> dims_;
    std::vector<Plan1D> lines_;
    std::size_t total_ = 0;
};

}  // namespace offt

#endif
