// ORACLE / TEST INFRASTRUCTURE ONLY — the CPU checker for the B200 path.
// Never linked into paper_2312_00538_b200; only tests/, smoke() and
// bench.py's cpu_baseline leg load it.
//
// Eigen-free restatement of the reference NFFT fast summation
// (/root/reference/proj/src/fastsum.cpp) with the same arithmetic order, so
// that it agrees with the reference compiled by path (oracle/_ref) to the
// last few ulp. Each block cites the reference lines it restates.
// Pinned against oracle/_ref (tests/test_oracle.py) and against the
// reference's own known-answer tests (P:tests/test_fastsum.cpp).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "ksvm_oracle.h"
#include "offt.hpp"

namespace {

thread_local std::string t_err = "ok";

struct DomainErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const DomainErr& e) {
        t_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        t_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        t_err = e.what();
        return 5;
    }
}

// P:src/fastsum.cpp:38-47 (FastsumConfig::validate)
void check_config(int N, int m, int sigma, double rT) {
    if (N < 2 || N % 2 != 0) throw std::invalid_argument("bandwidth must be a positive even integer");
    if (m < 2 || m > 8) throw std::invalid_argument("window_cutoff must lie in [2, 8]");
    if (sigma < 1) throw std::invalid_argument("oversampling must be >= 1");
    if (!(rT > 0.0 && rT <= 0.25)) throw std::invalid_argument("torus_radius must lie in (0, 1/4]");
}

}  // namespace

struct oracle_plan {
    int dim = 0, bw = 0, cut = 0, grid_edge = 0;  // d, N, m, M
    double bwin = 0.0, rT = 0.0, fit = 1.0;
    double ctr[3] = {0, 0, 0};
    double scale = 1.0, ell_s = 0.0, csum = 0.0;
    int64_t n = 0;
    std::vector<double> nodes;           // n x d column-major, scaled
    std::vector<std::size_t> kept_index;  // N^d grid positions
    std::vector<double> kept_mult;        // b_J * dec(J)^2
    offt::PlanND fwd, bwd;

    std::size_t gsize() const {
        std::size_t s = 1;
        for (int t = 0; t < dim; ++t) s *= static_cast<std::size_t>(grid_edge);
        return s;
    }
    // P:src/fastsum.cpp:75-78
    double phi(double t) const {
        const double mt = static_cast<double>(grid_edge) * t;
        return std::exp(-mt * mt / bwin) / std::sqrt(std::numbers::pi * bwin);
    }
};

namespace {

// P:src/fastsum.cpp:99-101 (scale_points): (x - centre) * scale, column-major
void affine(const oracle_plan& p, const double* pts, int64_t t, double* out) {
    for (int c = 0; c < p.dim; ++c)
        for (int64_t i = 0; i < t; ++i)
            out[c * t + i] = (pts[c * t + i] - p.ctr[c]) * p.scale;
}

// P:src/fastsum.cpp:103-209 (plan_fastsum)
oracle_plan* build_plan(const double* pts, int64_t n, int d, double ell, int N, int m,
                        int sigma, double rT, double fit) {
    check_config(N, m, sigma, rT);
    if (d < 1 || d > 3) throw std::invalid_argument("fast summation window dimension must be 1..3");
    if (n < 1) throw std::invalid_argument("empty node set");
    if (!(fit > 0.0 && fit <= 1.0)) throw std::invalid_argument("fit_fraction must lie in (0, 1]");

    auto* p = new oracle_plan;
    p->dim = d;
    p->bw = N;
    p->cut = m;
    p->grid_edge = sigma * N;
    p->rT = rT;
    p->fit = fit;
    p->n = n;
    const double sg = static_cast<double>(sigma);
    p->bwin = (2.0 * sg * m) / ((2.0 * sg - 1.0) * std::numbers::pi);  // :123-124

    // :129 bounding-box midpoint
    for (int c = 0; c < d; ++c) {
        double hi = pts[c * n], lo = pts[c * n];
        for (int64_t i = 1; i < n; ++i) {
            hi = std::max(hi, pts[c * n + i]);
            lo = std::min(lo, pts[c * n + i]);
        }
        p->ctr[c] = 0.5 * (hi + lo);
    }
    // :130-134 max l2 distance, sequential sum of squares
    double radius = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) {
            const double diff = pts[c * n + i] - p->ctr[c];
            s += diff * diff;
        }
        radius = std::max(radius, std::sqrt(s));
    }
    p->scale = radius > 0.0 ? fit * rT / radius : 1.0;
    p->nodes.resize(static_cast<std::size_t>(n) * d);
    affine(*p, pts, n, p->nodes.data());  // :135
    p->ell_s = p->scale * ell;           // :136

    // :142-199 coefficients of the rescaled Gaussian and the kept multipliers
    std::size_t nf = 1;
    for (int t = 0; t < d; ++t) nf *= static_cast<std::size_t>(N);
    std::vector<offt::cd> samp(nf), spec(nf);
    const double inv_l2 = 1.0 / (p->ell_s * p->ell_s);
    for (std::size_t k = 0; k < nf; ++k) {
        std::size_t r = k;
        double r2 = 0.0;
        for (int t = d - 1; t >= 0; --t) {  // last dimension first, as :152-158
            const int kt = static_cast<int>(r % static_cast<std::size_t>(N));
            r /= static_cast<std::size_t>(N);
            const double s = (kt < N / 2 ? kt : kt - N) / static_cast<double>(N);
            r2 += s * s;
        }
        samp[k] = std::exp(-r2 * inv_l2);
    }
    offt::PlanND(std::vector<int>(static_cast<std::size_t>(d), N), -1).execute(samp.data(), spec.data());

    p->kept_index.resize(nf);
    p->kept_mult.resize(nf);
    const double invn = 1.0 / static_cast<double>(nf);
    const int M = p->grid_edge;
    for (std::size_t k = 0; k < nf; ++k) {
        int kd[3] = {0, 0, 0};
        std::size_t r = k;
        for (int t = d - 1; t >= 0; --t) {
            kd[t] = static_cast<int>(r % static_cast<std::size_t>(N));
            r /= static_cast<std::size_t>(N);
        }
        std::size_t gi = 0;
        double dec = 1.0;
        for (int t = 0; t < d; ++t) {
            const int J = kd[t] < N / 2 ? kd[t] : kd[t] - N;  // I_N keeps -N/2, drops +N/2
            gi = gi * static_cast<std::size_t>(M) + static_cast<std::size_t>((J % M + M) % M);
            const double a = std::numbers::pi * J / static_cast<double>(M);
            dec *= std::exp(2.0 * p->bwin * a * a);
        }
        const double bJ = spec[k].real() * invn;
        p->kept_index[k] = gi;
        p->kept_mult[k] = bJ * dec;
        p->csum += bJ;
    }
    // :201-207 grid transforms
    const std::vector<int> gd(static_cast<std::size_t>(d), M);
    p->fwd = offt::PlanND(gd, -1);
    p->bwd = offt::PlanND(gd, +1);
    return p;
}

// P:src/fastsum.cpp:213-255 (for_each_neighbor): base = floor(xM) - m + 1,
// all 2m taps, wrap mod M, loop order dim0 > dim1 > dim2.
template <typename F>
void visit(const oracle_plan& p, const double* x, F&& f) {
    const int M = p.grid_edge, m = p.cut, span = 2 * m;
    int base[3] = {0, 0, 0};
    double w[3][16];
    for (int t = 0; t < p.dim; ++t) {
        base[t] = static_cast<int>(std::floor(x[t] * M)) - m + 1;
        for (int o = 0; o < span; ++o) w[t][o] = p.phi(x[t] - static_cast<double>(base[t] + o) / M);
    }
    auto wrap = [M](int l) { return static_cast<std::size_t>(((l % M) + M) % M); };
    const std::size_t Ms = static_cast<std::size_t>(M);
    if (p.dim == 1) {
        for (int a = 0; a < span; ++a) f(wrap(base[0] + a), w[0][a]);
    } else if (p.dim == 2) {
        for (int a = 0; a < span; ++a)
            for (int b = 0; b < span; ++b) f(wrap(base[0] + a) * Ms + wrap(base[1] + b), w[0][a] * w[1][b]);
    } else {
        for (int a = 0; a < span; ++a)
            for (int b = 0; b < span; ++b) {
                const std::size_t row = (wrap(base[0] + a) * Ms + wrap(base[1] + b)) * Ms;
                const double wab = w[0][a] * w[1][b];
                for (int c = 0; c < span; ++c) f(row + wrap(base[2] + c), wab * w[2][c]);
            }
    }
}

// P:src/fastsum.cpp:257-296 (run_transform); tgt is t x d column-major.
void transform(const oracle_plan& p, const double* tgt, int64_t t, const double* v, double* out) {
    const std::size_t G = p.gsize();
    std::vector<offt::cd> a(G, offt::cd(0.0, 0.0)), b(G);
    double x[3];
    for (int64_t i = 0; i < p.n; ++i) {  // :265-272 spread
        const double vi = v[i];
        if (vi == 0.0) continue;
        for (int c = 0; c < p.dim; ++c) x[c] = p.nodes[static_cast<std::size_t>(c * p.n + i)];
        visit(p, x, [&](std::size_t idx, double w) { a[idx] += vi * w; });
    }
    p.fwd.execute(a.data(), b.data());  // :273
    std::fill(a.begin(), a.end(), offt::cd(0.0, 0.0));  // :277-281 multiply
    for (std::size_t k = 0; k < p.kept_index.size(); ++k) {
        const std::size_t idx = p.kept_index[k];
        a[idx] = b[idx] * p.kept_mult[k];
    }
    p.bwd.execute(a.data(), b.data());  // :282
    for (int64_t j = 0; j < t; ++j) {  // :286-294 gather
        for (int c = 0; c < p.dim; ++c) x[c] = tgt[c * t + j];
        double acc = 0.0;
        visit(p, x, [&](std::size_t idx, double w) { acc += b[idx].real() * w; });
        out[j] = acc;
    }
}

}  // namespace

// P:src/fastsum.cpp:326-362 (AnovaFastOperator)
struct oracle_anova {
    int64_t n = 0;
    int d = 0;
    std::vector<double> pts;  // row-major n x d (entry evaluation)
    std::vector<std::vector<int>> wins;
    std::vector<double> eta, ell;
    std::vector<oracle_plan*> plans;
    ~oracle_anova() {
        for (auto* p : plans) delete p;
    }
};

extern "C" {

const char* oracle_last_error(void) { return t_err.c_str(); }

int oracle_plan_create(const double* pts, int64_t n, int d, double ell, int N, int m, int sigma,
                       double rT, double fit, oracle_plan** out) {
    return guard([&] { *out = build_plan(pts, n, d, ell, N, m, sigma, rT, fit); });
}

// P:src/fastsum.cpp:300-305
int oracle_plan_apply(const oracle_plan* p, const double* v, double* out) {
    return guard([&] { transform(*p, p->nodes.data(), p->n, v, out); });
}

// P:src/fastsum.cpp:307-322
int oracle_plan_apply_cross(const oracle_plan* p, const double* targets, int64_t t, const double* v,
                            double* out) {
    return guard([&] {
        std::vector<double> sc(static_cast<std::size_t>(t) * p->dim);
        affine(*p, targets, t, sc.data());
        for (int64_t j = 0; j < t; ++j) {
            double s = 0.0;
            for (int c = 0; c < p->dim; ++c) s += sc[c * t + j] * sc[c * t + j];
            if (std::sqrt(s) > p->rT * (1.0 + 1e-12))
                throw DomainErr("target " + std::to_string(j) + " falls outside the scaled torus ball");
        }
        transform(*p, sc.data(), t, v, out);
    });
}

double oracle_plan_scaled_length(const oracle_plan* p) { return p->ell_s; }
double oracle_plan_coefficient_sum(const oracle_plan* p) { return p->csum; }
int oracle_plan_scale_points(const oracle_plan* p, const double* pts, int64_t t, double* out) {
    return guard([&] { affine(*p, pts, t, out); });
}
void oracle_plan_free(oracle_plan* p) { delete p; }

int oracle_anova_create(const double* pts_rm, int64_t n, int d, const int* feats, const int* sizes,
                        int P, const double* weights, const double* ells, int N, int m, int sigma,
                        double rT, double fit, oracle_anova** out) {
    return guard([&] {
        // P:src/windowing.cpp:79-103 (check_windowing)
        if (P == 0) throw std::invalid_argument("windowing has no windows");
        std::vector<bool> seen(static_cast<std::size_t>(d), false);
        auto* op = new oracle_anova;
        op->n = n;
        op->d = d;
        op->pts.assign(pts_rm, pts_rm + n * d);
        int off = 0;
        for (int l = 0; l < P; ++l) {
            if (sizes[l] < 1 || sizes[l] > 3) {
                delete op;
                throw std::invalid_argument("window size must be 1..3");
            }
            std::vector<int> w(feats + off, feats + off + sizes[l]);
            off += sizes[l];
            for (int f : w) {
                if (f < 0 || f >= d || seen[static_cast<std::size_t>(f)]) {
                    delete op;
                    throw std::invalid_argument("bad window feature index");
                }
                seen[static_cast<std::size_t>(f)] = true;
            }
            if (!(weights[l] > 0.0) || !(ells[l] > 0.0)) {
                delete op;
                throw std::invalid_argument("window weights and length scales must be positive");
            }
            op->wins.push_back(w);
            op->eta.push_back(weights[l]);
            op->ell.push_back(ells[l]);
        }
        for (int l = 0; l < P; ++l) {  // :333-340 one plan per window
            const auto& w = op->wins[static_cast<std::size_t>(l)];
            std::vector<double> sub(static_cast<std::size_t>(n) * w.size());
            for (std::size_t c = 0; c < w.size(); ++c)
                for (int64_t i = 0; i < n; ++i) sub[c * n + i] = pts_rm[i * d + w[c]];
            try {
                op->plans.push_back(build_plan(sub.data(), n, static_cast<int>(w.size()), ells[l], N, m,
                                               sigma, rT, fit));
            } catch (...) {
                delete op;
                throw;
            }
        }
        *out = op;
    });
}

// P:src/fastsum.cpp:345-352: out = 0; out += eta_l * apply_l, window order
int oracle_anova_apply(const oracle_anova* op, const double* v, double* out) {
    return guard([&] {
        std::vector<double> part(static_cast<std::size_t>(op->n));
        for (int64_t i = 0; i < op->n; ++i) out[i] = 0.0;
        for (std::size_t l = 0; l < op->plans.size(); ++l) {
            const oracle_plan& p = *op->plans[l];
            transform(p, p.nodes.data(), p.n, v, part.data());
            for (int64_t i = 0; i < op->n; ++i) out[i] += op->eta[l] * part[static_cast<std::size_t>(i)];
        }
    });
}

// P:src/kernel.cpp:15-29 (anova_eval) via P:src/fastsum.cpp:354-356
double oracle_anova_entry(const oracle_anova* op, int64_t i, int64_t j) {
    double sum = 0.0;
    for (std::size_t l = 0; l < op->wins.size(); ++l) {
        const double e = op->ell[l];
        double d2 = 0.0;
        for (int f : op->wins[l]) {
            const double diff = op->pts[static_cast<std::size_t>(i * op->d + f)] -
                                op->pts[static_cast<std::size_t>(j * op->d + f)];
            d2 += diff * diff;
        }
        sum += op->eta[l] * std::exp(-d2 / (e * e));
    }
    return sum;
}

void oracle_anova_free(oracle_anova* op) { delete op; }

// The exact DFT behind both the restatement and the FFTW shim (offt.hpp),
// exposed so tests can pin it against numpy.fft. in/out: interleaved complex.
void oracle_fft(const double* in, double* out, int rank, const int* dims, int sign) {
    offt::PlanND(std::vector<int>(dims, dims + rank), sign)
        .execute(reinterpret_cast<const offt::cd*>(in), reinterpret_cast<offt::cd*>(out));
}

// P:tests/helpers.hpp:15-31
void oracle_random_points(int64_t n, int64_t d, uint64_t seed, double scale, double* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> normal(0.0, scale);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < d; ++j) out[j * n + i] = normal(rng);
}

void oracle_random_vector(int64_t n, uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    for (int64_t i = 0; i < n; ++i) out[i] = normal(rng);
}

void oracle_uniform(int64_t n, uint64_t seed, double lo, double hi, double* out) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(lo, hi);
    for (int64_t i = 0; i < n; ++i) out[i] = u(rng);
}

void oracle_bernoulli(int64_t n, uint64_t seed, double p, double* out) {
    std::mt19937_64 rng(seed);
    std::bernoulli_distribution b(p);
    for (int64_t i = 0; i < n; ++i) out[i] = b(rng) ? 1.0 : 0.0;
}

}  // extern "C"
