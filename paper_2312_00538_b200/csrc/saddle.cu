// GPU-resident Newton saddle solver: the reference's
// SaddleOperator, SaddlePreconditioner and gmres_solve (P:src/saddle.cpp,
// P:include/ksvm/saddle.hpp) with every length-(n+1) vector and the Krylov
// basis in HBM. The kernel matvec goes through the public C ABI
// (ksvm_nfft_op_apply on device pointers, same stream).
//
// Differences from the reference are rounding only:
//  * reductions (dots, norms, Z t, Z^T inner) use a fixed grid of kRB
//    blocks with fixed index ownership, fixed warp butterflies and
//    fixed-order finishers, so every solve is bit-reproducible;
//  * Gram-Schmidt is classical with one re-orthogonalisation pass (two
//    block GEMVs per pass over the basis) instead of modified Gram-Schmidt
//    with one re-orthogonalisation pass; H(:,k) = h1 + h2 in both, and the
//    Arnoldi relation is the same;
//  * the capacitance I + Z Theta^{-1} Z^T is formed on the FP64 tensor cores
//    and inverted explicitly after a partial-pivot LU on the host (the
//    reference keeps the LU, P:src/saddle.cpp:57); the rcond < 1e-15
//    fallback (:59-60) uses the exact 1-norm condition number.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "capi_common.cuh"
#include "launch.cuh"

namespace ksvm_nfft {
namespace {

constexpr int kRB = 296;   // reduction blocks: fixed, so partial sums have a fixed order
constexpr int kRT = 256;   // threads per reduction block
constexpr int kRows = 8;   // basis rows per pass of the multi-dot kernel
constexpr int kMaxRank = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block b owns indices b*kRT + t + q*kRB*kRT; its sum is written to
// partial[b] (lane butterfly, then warps in order).
__device__ __forceinline__ void block_partial(double v, double* partial) {
    __shared__ double sh[kRT / 32];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kRT / 32; ++w) s += sh[w];
        partial[blockIdx.x] = s;
    }
}

#define KSVM_FOR_BLOCK_INDEX(i, L) \
    for (long long i = static_cast<long long>(blockIdx.x) * kRT + threadIdx.x; i < (L); i += static_cast<long long>(kRB) * kRT)

__global__ void __launch_bounds__(kRT) k_mul(double* __restrict__ out, const double* __restrict__ a,
                                             const double* __restrict__ b, long long n) {
    pdl_trigger();
    pdl_wait();
    KSVM_FOR_BLOCK_INDEX(j, n) out[j] = a[j] * b[j];
}

// P:src/saddle.cpp:29-31: out_j = y_j (K y v)_j + theta_j v_j - w y_j; partial of y . v
__global__ void __launch_bounds__(kRT) k_saddle_post(double* __restrict__ out, const double* __restrict__ y,
                                                     const double* __restrict__ kv, const double* __restrict__ theta,
                                                     const double* __restrict__ vw, long long n,
                                                     double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    const double w = vw[n];
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        const double v = vw[j];
        out[j] = y[j] * kv[j] + theta[j] * v - w * y[j];
        acc += y[j] * v;
    }
    block_partial(acc, partial);
}

// *dst = coef * sum(partial) - (sub ? *sub : 0), or sqrt(sum) when root.
__global__ void k_finish_scalar(const double* __restrict__ partial, int nb, double* __restrict__ dst, double coef,
                                const double* __restrict__ sub, int root) {
    pdl_trigger();
    pdl_wait();
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += partial[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) *dst = root ? sqrt(s) : coef * s - (sub ? *sub : 0.0);
}

// partial[b * rows + a] = block b's share of sum_i M[a][i] x_i for a < rows,
// x_i = w_i (mode 0) or y_i g_i / theta_i (mode 1, P:src/saddle.cpp:80).
__global__ void __launch_bounds__(kRT) k_mdot(const double* __restrict__ M, long long ld, int rows, long long L,
                                              int mode, const double* __restrict__ w, const double* __restrict__ y,
                                              const double* __restrict__ theta, double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[kRT / 32][kRows];
    for (int a0 = 0; a0 < rows; a0 += kRows) {
        double acc[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = 0.0;
        KSVM_FOR_BLOCK_INDEX(i, L) {
            const double x = mode == 0 ? w[i] : y[i] * w[i] / theta[i];
#pragma unroll
            for (int r = 0; r < kRows; ++r)
                if (a0 + r < rows) acc[r] += M[static_cast<long long>(a0 + r) * ld + i] * x;
        }
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = warp_sum(acc[r]);
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (int r = 0; r < kRows; ++r) sh[threadIdx.x >> 5][r] = acc[r];
        }
        __syncthreads();
        if (threadIdx.x < kRows && a0 + static_cast<int>(threadIdx.x) < rows) {
            double s = 0.0;
            for (int wv = 0; wv < kRT / 32; ++wv) s += sh[wv][threadIdx.x];
            partial[static_cast<long long>(blockIdx.x) * rows + a0 + threadIdx.x] = s;
        }
        __syncthreads();
    }
}

// out[a] = sum_b partial[b * rows + a] (one warp per row).
__global__ void k_rows_finish(const double* __restrict__ partial, int nb, int rows, double* __restrict__ out) {
    pdl_trigger();
    pdl_wait();
    const int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (a >= rows) return;
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += partial[static_cast<long long>(b) * rows + a];
    s = warp_sum(s);
    if (lane == 0) out[a] = s;
}

// inner = Cinv s (k x k, k <= kMaxRank)
__global__ void k_gemv_small(const double* __restrict__ Cinv, int k, const double* __restrict__ s,
                             double* __restrict__ inner) {
    pdl_trigger();
    pdl_wait();
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= k) return;
    double acc = 0.0;
    for (int c = 0; c < k; ++c) acc += Cinv[static_cast<long long>(a) * k + c] * s[c];
    inner[a] = acc;
}

// P:src/saddle.cpp:81-83: x1 = g/theta - y (Z^T inner)/theta; partial of y . x1
__global__ void __launch_bounds__(kRT) k_smw_out(double* __restrict__ out, const double* __restrict__ g,
                                                 const double* __restrict__ y, const double* __restrict__ theta,
                                                 const double* __restrict__ Z, int k, const double* __restrict__ inner,
                                                 long long n, double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    extern __shared__ double s_inner[];
    for (int a = threadIdx.x; a < k; a += blockDim.x) s_inner[a] = inner[a];
    __syncthreads();
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        double s = 0.0;
        for (int a = 0; a < k; ++a) s += Z[static_cast<long long>(a) * n + j] * s_inner[a];
        const double x1 = g[j] / theta[j] - y[j] * s / theta[j];
        out[j] = x1;
        acc += y[j] * x1;
    }
    block_partial(acc, partial);
}

// P:src/saddle.cpp:74-75 (fallback / rank 0): x1 = g / theta
__global__ void __launch_bounds__(kRT) k_diag_out(double* __restrict__ out, const double* __restrict__ g,
                                                  const double* __restrict__ y, const double* __restrict__ theta,
                                                  long long n, double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        const double x1 = g[j] / theta[j];
        out[j] = x1;
        acc += y[j] * x1;
    }
    block_partial(acc, partial);
}

// mode 0: w_i -= sum_a V[a][i] c[a]; mode 1: w_i = sum_a V[a][i] c[a]
__global__ void __launch_bounds__(kRT) k_combine_rows(double* __restrict__ w, const double* __restrict__ V,
                                                      long long ld, int rows, const double* __restrict__ c,
                                                      long long L, int mode) {
    pdl_trigger();
    pdl_wait();
    KSVM_FOR_BLOCK_INDEX(i, L) {
        double s = 0.0;
        for (int a = 0; a < rows; ++a) s += V[static_cast<long long>(a) * ld + i] * c[a];
        w[i] = mode == 0 ? w[i] - s : s;
    }
}

__global__ void __launch_bounds__(kRT) k_scale(double* __restrict__ dst, const double* __restrict__ src, long long L,
                                               const double* __restrict__ denom) {
    pdl_trigger();
    pdl_wait();
    const double d = *denom;
    KSVM_FOR_BLOCK_INDEX(i, L) dst[i] = src[i] / d;
}

__global__ void __launch_bounds__(kRT) k_sq_diff(const double* __restrict__ a, const double* __restrict__ b, long long L,
                                                 double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(i, L) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    block_partial(acc, partial);
}

// Capacitance partials on the FP64 tensor cores: warp (ta, tb, chunk) forms
// the 8x8 tile sum_{j in chunk} (Z[a][j] / theta_j) Z[b][j] with DMMA.8x8x4
// (P:src/saddle.cpp:52-54 computes Z * Theta^{-1} * Z^T).
__global__ void k_cap_partial(const double* __restrict__ Z, const double* __restrict__ theta, int k, long long n,
                              long long chunk, int nt, double* __restrict__ partial) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ta = blockIdx.x / nt, tb = blockIdx.x % nt;
    const long long j0 = static_cast<long long>(blockIdx.y) * chunk, j1 = min(n, j0 + chunk);
    const int a = ta * 8 + g, b = tb * 8 + g;
    double d0 = 0.0, d1 = 0.0;
    for (long long j = j0; j < j1; j += 4) {
        const long long jj = j + t;
        const bool ok = jj < j1;
        const double av = ok && a < k ? Z[static_cast<long long>(a) * n + jj] * (1.0 / theta[jj]) : 0.0;
        const double bv = ok && b < k ? Z[static_cast<long long>(b) * n + jj] : 0.0;
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(d0), "+d"(d1)
            : "d"(av), "d"(bv));
    }
    double* out = partial + (static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x) * 64;
    out[g * 8 + 2 * t] = d0;
    out[g * 8 + 2 * t + 1] = d1;
}

// C[a][b] = (a == b) + sum over chunks (in order) of the tile partials
__global__ void k_cap_finish(const double* __restrict__ partial, int nchunks, int nt, int k, double* __restrict__ C) {
    pdl_trigger();
    pdl_wait();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * k) return;
    const int a = idx / k, b = idx % k;
    const int tile = (a >> 3) * nt + (b >> 3), e = (a & 7) * 8 + (b & 7);
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += partial[(static_cast<long long>(c) * nt * nt + tile) * 64 + e];
    C[idx] = (a == b ? 1.0 : 0.0) + s;
}

int blocks_for(long long L) { return static_cast<int>(std::min<long long>(kRB, (L + kRT - 1) / kRT)); }

}  // namespace
}  // namespace ksvm_nfft

using namespace ksvm_nfft;

struct ksvm_nfft_saddle {
    const ksvm_nfft_op* op = nullptr;
    int64_t n = 0;
    int device = 0;
    DevBuf<double> y, theta, u, kv, partial;
    cudaStream_t stream = nullptr;
    mutable std::mutex mu;
    // GMRES workspace, reused while max_iter does not grow
    int ws_iter = -1;
    DevBuf<double> V, z, w, x, r, ax, h, coef, partial_rows, scal;
    double* pinned = nullptr;
    ~ksvm_nfft_saddle() {
        if (pinned) cudaFreeHost(pinned);
        if (stream) cudaStreamDestroy(stream);
    }
};

struct ksvm_nfft_precond {
    int64_t n = 0;
    int k = 0, device = 0;
    bool identity = false, fallback = false, fresh = false;
    DevBuf<double> Z, y, theta, Cinv, partial, s, inner;
    cudaStream_t stream = nullptr;
    mutable std::mutex mu;
    ~ksvm_nfft_precond() {
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace ksvm_nfft {
namespace {

void check_theta(const double* theta, int64_t n, const char* who) {
    if (!theta) throw std::invalid_argument(std::string(who) + ": null Theta");
    for (int64_t j = 0; j < n; ++j)
        if (!(theta[j] > 0.0)) throw std::invalid_argument(std::string(who) + ": Theta must be positive");
}

// out = A vw (device vectors of length n + 1), P:src/saddle.cpp:22-33
void saddle_apply_dev(const ksvm_nfft_saddle& S, const double* vw, double* out, cudaStream_t st) {
    const long long n = S.n;
    const int nb = blocks_for(n);
    launch_k(k_mul, dim3(nb), dim3(kRT), 0, st, S.u.p, S.y.p, vw, n);
    const int rc = ksvm_nfft_op_apply(S.op, S.u.p, S.kv.p, KSVM_NFFT_DEVICE, st);
    if (rc != KSVM_NFFT_OK) throw std::runtime_error(std::string("saddle apply: ") + ksvm_nfft_last_error());
    launch_k(k_saddle_post, dim3(nb), dim3(kRT), 0, st, out, S.y.p, S.kv.p, S.theta.p, vw, n, S.partial.p);
    launch_k(k_finish_scalar, dim3(1), dim3(32), 0, st, S.partial.p, nb, out + n, -1.0, nullptr, 0);
    launch_counter() += 4;
    CK(cudaGetLastError());
}

// out = P^{-1} g (device vectors of length n + 1), P:src/saddle.cpp:65-90
void precond_apply_dev(const ksvm_nfft_precond& P, const double* g, double* out, cudaStream_t st) {
    const long long n = P.n;
    if (P.identity) {
        CK(cudaMemcpyAsync(out, g, sizeof(double) * (n + 1), cudaMemcpyDeviceToDevice, st));
        return;
    }
    if (!P.fresh) throw std::logic_error("SaddlePreconditioner: refresh() before apply()");
    const int nb = blocks_for(n);
    if (P.fallback || P.k == 0) {
        launch_k(k_diag_out, dim3(nb), dim3(kRT), 0, st, out, g, P.y.p, P.theta.p, n, P.partial.p);
        launch_counter() += 1;
    } else {
        launch_k(k_mdot, dim3(nb), dim3(kRT), 0, st, P.Z.p, n, P.k, n, 1, g, P.y.p, P.theta.p, P.partial.p);
        launch_k(k_rows_finish, dim3((P.k + 7) / 8), dim3(256), 0, st, P.partial.p, nb, P.k, P.s.p);
        launch_k(k_gemv_small, dim3((P.k + 127) / 128), dim3(128), 0, st, P.Cinv.p, P.k, P.s.p, P.inner.p);
        launch_k(k_smw_out, dim3(nb), dim3(kRT), sizeof(double) * P.k, st, out, g, P.y.p, P.theta.p, P.Z.p, P.k, P.inner.p, n, P.partial.p);
        launch_counter() += 4;
    }
    launch_k(k_finish_scalar, dim3(1), dim3(32), 0, st, P.partial.p, nb, out + n, -1.0, g + n, 0);
    launch_counter() += 1;
    CK(cudaGetLastError());
}

// Capacitance I + Z Theta^{-1} Z^T, partial-pivot LU, rcond, inverse.
void precond_refresh(ksvm_nfft_precond& P, const double* theta_h) {
    check_theta(theta_h, P.n, "SaddlePreconditioner");
    const long long n = P.n;
    cudaStream_t st = P.stream;
    P.theta.upload(theta_h, static_cast<size_t>(n), st);
    P.fallback = false;
    P.fresh = true;
    if (P.identity || P.k == 0) {
        CK(cudaStreamSynchronize(st));
        return;
    }
    const int k = P.k, nt = (k + 7) / 8;
    const int nchunks = static_cast<int>(std::min<long long>(64, std::max<long long>(1, n / 1024)));
    const long long chunk = ((n + nchunks - 1) / nchunks + 3) / 4 * 4;
    DevBuf<double> part, C;
    part.alloc(static_cast<size_t>(nchunks) * nt * nt * 64);
    C.alloc(static_cast<size_t>(k) * k);
    launch_k(k_cap_partial, dim3(dim3(nt * nt, nchunks)), dim3(32), 0, st, P.Z.p, P.theta.p, k, n, chunk, nt, part.p);
    launch_k(k_cap_finish, dim3((k * k + 255) / 256), dim3(256), 0, st, part.p, nchunks, nt, k, C.p);
    launch_counter() += 2;
    CK(cudaGetLastError());
    std::vector<double> cap(static_cast<size_t>(k) * k);
    CK(cudaMemcpyAsync(cap.data(), C.p, sizeof(double) * cap.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (double c : cap)
        if (!std::isfinite(c)) {  // P:src/saddle.cpp:55-58
            P.fallback = true;
            return;
        }
    double anorm = 0.0;
    for (int b = 0; b < k; ++b) {
        double s = 0.0;
        for (int a = 0; a < k; ++a) s += std::fabs(cap[static_cast<size_t>(a) * k + b]);
        anorm = std::max(anorm, s);
    }
    std::vector<double> lu = cap;
    std::vector<int> piv(static_cast<size_t>(k));
    for (int c = 0; c < k; ++c) {
        int p = c;
        for (int r = c + 1; r < k; ++r)
            if (std::fabs(lu[static_cast<size_t>(r) * k + c]) > std::fabs(lu[static_cast<size_t>(p) * k + c])) p = r;
        piv[static_cast<size_t>(c)] = p;
        if (p != c)
            for (int q = 0; q < k; ++q) std::swap(lu[static_cast<size_t>(c) * k + q], lu[static_cast<size_t>(p) * k + q]);
        const double d = lu[static_cast<size_t>(c) * k + c];
        if (d == 0.0) {
            P.fallback = true;
            return;
        }
        for (int r = c + 1; r < k; ++r) {
            const double f = lu[static_cast<size_t>(r) * k + c] / d;
            lu[static_cast<size_t>(r) * k + c] = f;
            for (int q = c + 1; q < k; ++q) lu[static_cast<size_t>(r) * k + q] -= f * lu[static_cast<size_t>(c) * k + q];
        }
    }
    std::vector<double> inv(static_cast<size_t>(k) * k);
    double inorm = 0.0;
    std::vector<double> e(static_cast<size_t>(k));
    for (int b = 0; b < k; ++b) {  // column b of the inverse
        std::fill(e.begin(), e.end(), 0.0);
        e[static_cast<size_t>(b)] = 1.0;
        for (int c = 0; c < k; ++c) std::swap(e[static_cast<size_t>(c)], e[static_cast<size_t>(piv[static_cast<size_t>(c)])]);
        for (int r = 0; r < k; ++r)
            for (int c = 0; c < r; ++c) e[static_cast<size_t>(r)] -= lu[static_cast<size_t>(r) * k + c] * e[static_cast<size_t>(c)];
        for (int r = k - 1; r >= 0; --r) {
            for (int c = r + 1; c < k; ++c) e[static_cast<size_t>(r)] -= lu[static_cast<size_t>(r) * k + c] * e[static_cast<size_t>(c)];
            e[static_cast<size_t>(r)] /= lu[static_cast<size_t>(r) * k + r];
        }
        double s = 0.0;
        for (int a = 0; a < k; ++a) {
            inv[static_cast<size_t>(a) * k + b] = e[static_cast<size_t>(a)];
            s += std::fabs(e[static_cast<size_t>(a)]);
        }
        inorm = std::max(inorm, s);
    }
    const double rcond = 1.0 / (anorm * inorm);
    if (!std::isfinite(rcond) || rcond < 1e-15) {  // P:src/saddle.cpp:59-60
        P.fallback = true;
        return;
    }
    P.Cinv.upload(inv.data(), inv.size(), st);
    CK(cudaStreamSynchronize(st));
}

cudaStream_t pick_stream(int ptr_kind, void* stream, cudaStream_t own) {
    if (ptr_kind == KSVM_NFFT_DEVICE) return static_cast<cudaStream_t>(stream);
    if (ptr_kind != KSVM_NFFT_HOST) throw std::invalid_argument("bad ptr_kind");
    return own;
}

}  // namespace
}  // namespace ksvm_nfft

extern "C" {

int ksvm_nfft_saddle_create(const ksvm_nfft_op* op, const double* y, const double* theta, ksvm_nfft_saddle** out) {
    return guarded([&] {
        if (!op || !y || !out) throw std::invalid_argument("SaddleOperator: null argument");
        const int64_t n = ksvm_nfft_op_size(op);
        check_theta(theta, n, "SaddleOperator");
        auto S = std::make_unique<ksvm_nfft_saddle>();
        S->op = op;
        S->n = n;
        S->device = ksvm_nfft_op_device(op);
        DeviceGuard dg(S->device);
        CK(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
        S->y.upload(y, static_cast<size_t>(n), S->stream);
        S->theta.upload(theta, static_cast<size_t>(n), S->stream);
        S->u.alloc(static_cast<size_t>(n));
        S->kv.alloc(static_cast<size_t>(n));
        S->partial.alloc(kRB);
        CK(cudaStreamSynchronize(S->stream));
        *out = S.release();
    });
}

int ksvm_nfft_saddle_set_theta(ksvm_nfft_saddle* s, const double* theta) {
    return guarded([&] {
        if (!s) throw std::invalid_argument("null saddle operator");
        check_theta(theta, s->n, "SaddleOperator");  // P:src/saddle.cpp:16-18
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        CK(cudaMemcpyAsync(s->theta.p, theta, sizeof(double) * s->n, cudaMemcpyHostToDevice, s->stream));
        CK(cudaStreamSynchronize(s->stream));
    });
}

int ksvm_nfft_saddle_apply(const ksvm_nfft_saddle* s, const double* vw, double* out, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!s || !vw || !out) throw std::invalid_argument("SaddleOperator: null argument");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        auto& S = const_cast<ksvm_nfft_saddle&>(*s);
        cudaStream_t st = pick_stream(ptr_kind, stream, S.stream);
        const size_t n1 = static_cast<size_t>(S.n) + 1;
        if (ptr_kind == KSVM_NFFT_DEVICE) {
            saddle_apply_dev(S, vw, out, st);
            return;
        }
        DevBuf<double> din, dout;
        din.upload(vw, n1, st);
        dout.alloc(n1);
        saddle_apply_dev(S, din.p, dout.p, st);
        CK(cudaMemcpyAsync(out, dout.p, sizeof(double) * n1, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

void ksvm_nfft_saddle_free(ksvm_nfft_saddle* s) { delete s; }

int ksvm_nfft_precond_create(const double* Z, int k, int64_t n, const double* y, int device, ksvm_nfft_precond** out) {
    return guarded([&] {
        if (!y || !out || n < 1) throw std::invalid_argument("SaddlePreconditioner: bad argument");
        if (Z && (k < 0 || k > kMaxRank)) throw std::invalid_argument("SaddlePreconditioner: rank must be in [0, 1024]");
        auto P = std::make_unique<ksvm_nfft_precond>();
        P->n = n;
        P->k = Z ? k : 0;
        P->device = device;
        P->identity = Z == nullptr;  // P:src/saddle.cpp:37-38
        DeviceGuard dg(device);
        CK(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
        P->y.upload(y, static_cast<size_t>(n), P->stream);
        if (P->k > 0) P->Z.upload(Z, static_cast<size_t>(P->k) * n, P->stream);
        P->partial.alloc(static_cast<size_t>(kRB) * std::max(P->k, 1));
        P->s.alloc(static_cast<size_t>(std::max(P->k, 1)));
        P->inner.alloc(static_cast<size_t>(std::max(P->k, 1)));
        CK(cudaStreamSynchronize(P->stream));
        *out = P.release();
    });
}

int ksvm_nfft_precond_refresh(ksvm_nfft_precond* p, const double* theta) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("null preconditioner");
        std::lock_guard<std::mutex> lk(p->mu);
        DeviceGuard dg(p->device);
        precond_refresh(*p, theta);
    });
}

int ksvm_nfft_precond_apply(const ksvm_nfft_precond* p, const double* g, double* out, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!p || !g || !out) throw std::invalid_argument("SaddlePreconditioner: null argument");
        std::lock_guard<std::mutex> lk(p->mu);
        DeviceGuard dg(p->device);
        cudaStream_t st = pick_stream(ptr_kind, stream, p->stream);
        const size_t n1 = static_cast<size_t>(p->n) + 1;
        if (ptr_kind == KSVM_NFFT_DEVICE) {
            precond_apply_dev(*p, g, out, st);
            return;
        }
        if (!p->identity && !p->fresh) throw std::logic_error("SaddlePreconditioner: refresh() before apply()");
        DevBuf<double> din, dout;
        din.upload(g, n1, st);
        dout.alloc(n1);
        precond_apply_dev(*p, din.p, dout.p, st);
        CK(cudaMemcpyAsync(out, dout.p, sizeof(double) * n1, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int ksvm_nfft_precond_identity(const ksvm_nfft_precond* p) { return p && p->identity ? 1 : 0; }
int ksvm_nfft_precond_diagonal_fallback(const ksvm_nfft_precond* p) { return p && p->fallback ? 1 : 0; }
void ksvm_nfft_precond_free(ksvm_nfft_precond* p) { delete p; }

// P:src/saddle.cpp:92-178
int ksvm_nfft_gmres_solve(const ksvm_nfft_saddle* s, const ksvm_nfft_precond* p, const double* rhs, double tol,
                          int max_iter, double* x, ksvm_nfft_gmres_stats* stats, double* residual_history,
                          int ptr_kind, void* stream) {
    return guarded([&] {
        if (!s || !p || !rhs || !x || !stats) throw std::invalid_argument("gmres: null argument");
        if (!(tol > 0.0)) throw std::invalid_argument("gmres tol must be positive");
        if (max_iter < 0) throw std::invalid_argument("gmres max_iter must be >= 0");
        if (p->n != s->n) throw std::invalid_argument("gmres: preconditioner size mismatch");
        if (p->device != s->device) throw std::invalid_argument("gmres: operator and preconditioner on different GPUs");
        std::lock_guard<std::mutex> lk(s->mu);
        std::lock_guard<std::mutex> lk2(p->mu);
        auto& S = const_cast<ksvm_nfft_saddle&>(*s);
        const ksvm_nfft_precond& P = *p;
        if (!P.identity && !P.fresh) throw std::logic_error("SaddlePreconditioner: refresh() before apply()");
        DeviceGuard dg(S.device);
        cudaStream_t st = pick_stream(ptr_kind, stream, S.stream);
        const long long n1 = S.n + 1;
        const int MI = max_iter;
        if (S.ws_iter < MI) {
            S.V.alloc(static_cast<size_t>(MI + 1) * n1);
            S.h.alloc(static_cast<size_t>(2 * (MI + 1) + 2));
            S.coef.alloc(static_cast<size_t>(MI + 1));
            S.partial_rows.alloc(static_cast<size_t>(kRB) * (MI + 1));
            if (S.pinned) cudaFreeHost(S.pinned);
            S.pinned = nullptr;
            CK(cudaMallocHost(&S.pinned, sizeof(double) * (2 * (MI + 1) + 4)));
            S.ws_iter = MI;
        }
        if (S.z.n < static_cast<size_t>(n1)) {
            S.z.alloc(n1);
            S.w.alloc(n1);
            S.x.alloc(n1);
            S.r.alloc(n1);
            S.ax.alloc(n1);
            S.scal.alloc(4);
        }
        const int nb = blocks_for(n1);
        double* hp = S.pinned;
        auto norm_into = [&](const double* a, const double* b, double* dst) {  // sqrt(sum (a-b)^2) or |a|
            if (b)
                launch_k(k_sq_diff, dim3(nb), dim3(kRT), 0, st, a, b, n1, S.partial_rows.p);
            else
                launch_k(k_mdot, dim3(nb), dim3(kRT), 0, st, a, n1, 1, n1, 0, a, nullptr, nullptr, S.partial_rows.p);
            launch_k(k_finish_scalar, dim3(1), dim3(32), 0, st, S.partial_rows.p, nb, dst, 1.0, nullptr, 1);
            launch_counter() += 2;
        };
        // right-hand side
        if (ptr_kind == KSVM_NFFT_HOST)
            CK(cudaMemcpyAsync(S.r.p, rhs, sizeof(double) * n1, cudaMemcpyHostToDevice, st));
        else
            CK(cudaMemcpyAsync(S.r.p, rhs, sizeof(double) * n1, cudaMemcpyDeviceToDevice, st));
        norm_into(S.r.p, nullptr, S.scal.p);
        CK(cudaMemcpyAsync(hp, S.scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double rhs_norm = hp[0];
        ksvm_nfft_gmres_stats out{};
        auto put_x = [&](const double* dx) {
            CK(cudaMemcpyAsync(x, dx, sizeof(double) * n1,
                               ptr_kind == KSVM_NFFT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
        };
        if (rhs_norm == 0.0) {  // P:src/saddle.cpp:100-104
            CK(cudaMemsetAsync(S.x.p, 0, sizeof(double) * n1, st));
            put_x(S.x.p);
            CK(cudaStreamSynchronize(st));
            out.converged = 1;
            *stats = out;
            return;
        }
        launch_k(k_scale, dim3(nb), dim3(kRT), 0, st, S.V.p, S.r.p, n1, S.scal.p);
        ++launch_counter();
        std::vector<double> H(static_cast<size_t>(MI + 1) * std::max(MI, 1), 0.0);
        auto Hk = [&](int i, int j) -> double& { return H[static_cast<size_t>(i) * std::max(MI, 1) + j]; };
        std::vector<double> cs(static_cast<size_t>(std::max(MI, 1)), 0.0), sn(cs), beta(static_cast<size_t>(MI) + 1, 0.0);
        beta[0] = rhs_norm;
        int k = 0;
        for (; k < MI; ++k) {
            const double* vk = S.V.p + static_cast<long long>(k) * n1;
            precond_apply_dev(P, vk, S.z.p, st);
            saddle_apply_dev(S, S.z.p, S.w.p, st);
            // classical Gram-Schmidt, two passes: h = V^T w; w -= V h
            for (int pass = 0; pass < 2; ++pass) {
                double* hd = S.h.p + pass * (k + 1);
                launch_k(k_mdot, dim3(nb), dim3(kRT), 0, st, S.V.p, n1, k + 1, n1, 0, S.w.p, nullptr, nullptr, S.partial_rows.p);
                launch_k(k_rows_finish, dim3((k + 1 + 7) / 8), dim3(256), 0, st, S.partial_rows.p, nb, k + 1, hd);
                launch_k(k_combine_rows, dim3(nb), dim3(kRT), 0, st, S.w.p, S.V.p, n1, k + 1, hd, n1, 0);
                launch_counter() += 3;
            }
            norm_into(S.w.p, nullptr, S.scal.p + 1);
            CK(cudaMemcpyAsync(hp, S.h.p, sizeof(double) * 2 * (k + 1), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(hp + 2 * (k + 1), S.scal.p + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            for (int i = 0; i <= k; ++i) Hk(i, k) = hp[i] + hp[k + 1 + i];
            const double hnext = hp[2 * (k + 1)];
            Hk(k + 1, k) = hnext;
            for (int i = 0; i < k; ++i) {  // stored Givens rotations
                const double tmp = cs[static_cast<size_t>(i)] * Hk(i, k) + sn[static_cast<size_t>(i)] * Hk(i + 1, k);
                Hk(i + 1, k) = -sn[static_cast<size_t>(i)] * Hk(i, k) + cs[static_cast<size_t>(i)] * Hk(i + 1, k);
                Hk(i, k) = tmp;
            }
            const double denom = std::hypot(Hk(k, k), Hk(k + 1, k));
            if (denom == 0.0) {
                out.breakdown = 1;
                break;
            }
            const size_t K = static_cast<size_t>(k);
            cs[K] = Hk(k, k) / denom;
            sn[K] = Hk(k + 1, k) / denom;
            Hk(k, k) = denom;
            Hk(k + 1, k) = 0.0;
            beta[K + 1] = -sn[K] * beta[K];
            beta[K] = cs[K] * beta[K];
            const double rel = std::fabs(beta[K + 1]) / rhs_norm;
            if (residual_history) residual_history[out.iterations] = rel;
            ++out.iterations;
            if (rel <= tol) {
                ++k;
                out.converged = 1;
                break;
            }
            if (hnext <= 1e-14 * rhs_norm) {  // happy breakdown
                out.breakdown = 1;
                out.converged = 1;
                ++k;
                break;
            }
            launch_k(k_scale, dim3(nb), dim3(kRT), 0, st, S.V.p + static_cast<long long>(k + 1) * n1, S.w.p, n1, S.scal.p + 1);
            ++launch_counter();
        }
        // u = V_k y_k with the upper-triangular solve, x = P^{-1} u
        if (k > 0) {
            std::vector<double> yk(static_cast<size_t>(k));
            for (int i = k - 1; i >= 0; --i) {
                double sacc = beta[static_cast<size_t>(i)];
                for (int j = i + 1; j < k; ++j) sacc -= Hk(i, j) * yk[static_cast<size_t>(j)];
                yk[static_cast<size_t>(i)] = sacc / Hk(i, i);
            }
            std::memcpy(hp, yk.data(), sizeof(double) * k);
            CK(cudaMemcpyAsync(S.coef.p, hp, sizeof(double) * k, cudaMemcpyHostToDevice, st));
            launch_k(k_combine_rows, dim3(nb), dim3(kRT), 0, st, S.z.p, S.V.p, n1, k, S.coef.p, n1, 1);
            ++launch_counter();
        } else {
            CK(cudaMemsetAsync(S.z.p, 0, sizeof(double) * n1, st));
        }
        precond_apply_dev(P, S.z.p, S.x.p, st);
        saddle_apply_dev(S, S.x.p, S.ax.p, st);
        norm_into(S.r.p, S.ax.p, S.scal.p + 2);
        CK(cudaMemcpyAsync(hp, S.scal.p + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
        put_x(S.x.p);
        CK(cudaStreamSynchronize(st));
        out.relative_residual = hp[0] / rhs_norm;
        if (out.relative_residual <= tol) out.converged = 1;
        *stats = out;
    });
}

}  // extern "C"
