// GPU Nystrom factor (P:src/low_rank.cpp:115-168, nystrom), the
// preconditioner factor the reference builds per window with the
// FastWindowOperator (P:src/pipeline.cpp:114-133,172-181): the Gaussian
// sketch Y = K G and KQ = K Q are batched applies of the NFFT operator
// (ksvm_nfft_op_apply_batch: one upload, concurrent apply lanes), the
// columns sketch takes exact kernel rows (ksvm_nfft_kernel_rows).
//
// Versus the reference (rounding / basis only, ZZ^T-equivalent):
//  * the sketch draws are the reference's: std::mt19937_64(seed) with
//    std::normal_distribution filled row by row, or std::shuffle of iota(n);
//  * the orthonormal basis of range(Y) comes from classical Gram-Schmidt
//    with one re-orthogonalisation pass (fixed-order reductions) instead of
//    a Householder QR: Q differs by column signs and rounding, and
//    Z^T Z = KQ (Q^T K Q)^{-1} KQ^T does not depend on the basis (it is the
//    same Nystrom approximation; only the preconditioner's Z^T Z matters,
//    saddle.cu);
//  * C = Q^T KQ on the FP64 tensor cores (DMMA per 8x8 tile and column
//    chunk, fixed chunk order), symmetrised and factored on the host with
//    Eigen's LDLT<Lower> rule (pivot on the largest remaining original
//    diagonal, first index on ties), D clamped to max(|d|, ldl_threshold);
//    the k x k map M = D^{-1/2} L^{-1} P is applied to KQ on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#include "capi_common.cuh"
#include "launch.cuh"
#include "reduce.cuh"

namespace ksvm_nfft {
namespace {

constexpr int kRowsN = 8;

// partial[b * rows + a] = block b's share of sum_i Q[a][i] y[i], a < rows
__global__ void __launch_bounds__(kRT) kn_mdot(const double* __restrict__ Q, long long n, int rows,
                                               const double* __restrict__ y, double* __restrict__ partial) {
    __shared__ double sh[kRT / 32][kRowsN];
    for (int a0 = 0; a0 < rows; a0 += kRowsN) {
        double acc[kRowsN];
#pragma unroll
        for (int r = 0; r < kRowsN; ++r) acc[r] = 0.0;
        KSVM_FOR_BLOCK_INDEX(i, n) {
            const double x = y[i];
#pragma unroll
            for (int r = 0; r < kRowsN; ++r)
                if (a0 + r < rows) acc[r] += Q[static_cast<long long>(a0 + r) * n + i] * x;
        }
#pragma unroll
        for (int r = 0; r < kRowsN; ++r) acc[r] = warp_sum(acc[r]);
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (int r = 0; r < kRowsN; ++r) sh[threadIdx.x >> 5][r] = acc[r];
        }
        __syncthreads();
        if (threadIdx.x < kRowsN && a0 + static_cast<int>(threadIdx.x) < rows) {
            double s = 0.0;
            for (int w = 0; w < kRT / 32; ++w) s += sh[w][threadIdx.x];
            partial[static_cast<long long>(blockIdx.x) * rows + a0 + threadIdx.x] = s;
        }
        __syncthreads();
    }
}

// h[a] = sum_b partial[b * rows + a] (one warp per row)
__global__ void kn_rows_finish(const double* __restrict__ partial, int nb, int rows, double* __restrict__ h) {
    const int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (a >= rows) return;
    const double s = warp_sum_strided(partial + a, nb, rows);
    if ((threadIdx.x & 31) == 0) h[a] = s;
}

// y_i -= sum_a Q[a][i] h[a]
__global__ void __launch_bounds__(kRT) kn_project(double* __restrict__ y, const double* __restrict__ Q, long long n,
                                                  int rows, const double* __restrict__ h) {
    KSVM_FOR_BLOCK_INDEX(i, n) {
        double s = 0.0;
        for (int a = 0; a < rows; ++a) s += Q[static_cast<long long>(a) * n + i] * h[a];
        y[i] -= s;
    }
}

__global__ void __launch_bounds__(kRT) kn_sumsq(const double* __restrict__ y, long long n,
                                                double* __restrict__ partial) {
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(i, n) acc += y[i] * y[i];
    block_partial(acc, partial);
}

// q = y / ||y|| (partial sums of squares), or 0 for an exactly zero column
__global__ void __launch_bounds__(kRT) kn_normalize(double* __restrict__ q, long long n,
                                                    const double* __restrict__ partial, int nb) {
    __shared__ double s_norm;
    if (threadIdx.x < 32) {
        const double s = warp_sum_strided(partial, nb, 1);
        if (threadIdx.x == 0) s_norm = sqrt(s);
    }
    __syncthreads();
    const double nr = s_norm;
    KSVM_FOR_BLOCK_INDEX(i, n) q[i] = nr > 0.0 ? q[i] / nr : 0.0;
}

// 8x8 tile partials of A B^T (k x n row-major operands) on DMMA.8x8x4, one
// warp per (tile pair, column chunk)
__global__ void kn_gram_partial(const double* __restrict__ A, const double* __restrict__ B, int k, long long n,
                                long long chunk, int nt, double* __restrict__ partial) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ta = blockIdx.x / nt, tb = blockIdx.x % nt;
    const long long j0 = static_cast<long long>(blockIdx.y) * chunk, j1 = min(n, j0 + chunk);
    const int a = ta * 8 + g, b = tb * 8 + g;
    double d0 = 0.0, d1 = 0.0;
    for (long long j = j0; j < j1; j += 4) {
        const long long jj = j + t;
        const bool ok = jj < j1;
        const double av = ok && a < k ? A[static_cast<long long>(a) * n + jj] : 0.0;
        const double bv = ok && b < k ? B[static_cast<long long>(b) * n + jj] : 0.0;
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(d0), "+d"(d1)
            : "d"(av), "d"(bv));
    }
    double* out = partial + (static_cast<long long>(blockIdx.y) * gridDim.x + blockIdx.x) * 64;
    out[g * 8 + 2 * t] = d0;
    out[g * 8 + 2 * t + 1] = d1;
}

__global__ void kn_gram_finish(const double* __restrict__ partial, int nchunks, int nt, int k, double* __restrict__ C) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * k) return;
    const int a = idx / k, b = idx % k;
    const int tile = (a >> 3) * nt + (b >> 3), e = (a & 7) * 8 + (b & 7);
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += partial[(static_cast<long long>(c) * nt * nt + tile) * 64 + e];
    C[idx] = s;
}

// C[r][c] = KQ[c][cols[r]] (columns sketch: the sampled rows of the sampled columns)
__global__ void kn_gather_cols(const double* __restrict__ KQ, long long n, int k, const long long* __restrict__ cols,
                               double* __restrict__ C) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * k) return;
    const int r = idx / k, c = idx % k;
    C[idx] = KQ[static_cast<long long>(c) * n + cols[r]];
}

// Z[a][i] = sum_c M[a][c] KQ[c][i]
__global__ void __launch_bounds__(kRT) kn_apply_small(double* __restrict__ Z, const double* __restrict__ M,
                                                      const double* __restrict__ KQ, int k, long long n) {
    KSVM_FOR_BLOCK_INDEX(i, n) {
        for (int a = 0; a < k; ++a) {
            double s = 0.0;
            for (int c = 0; c < k; ++c) s += M[a * k + c] * KQ[static_cast<long long>(c) * n + i];
            Z[static_cast<long long>(a) * n + i] = s;
        }
    }
}

void okc(int rc, const char* who) {
    if (rc == KSVM_NFFT_OK) return;
    const std::string msg = std::string(who) + ": " + ksvm_nfft_last_error();
    if (rc == KSVM_NFFT_ERR_CONFIG) throw std::invalid_argument(msg);
    if (rc == KSVM_NFFT_ERR_DATA) throw DomainErr(msg);
    throw std::runtime_error(msg);
}

// Eigen's ldlt_inplace<Lower>::unblocked on the row-major k x k S; then
// M = D~^{-1/2} L^{-1} P with D~ = max(|D|, thr) (P:src/low_rank.cpp:152-162).
std::vector<double> ldlt_map(std::vector<double> S, int k, double thr) {
    auto A = [&](int i, int j) -> double& { return S[static_cast<size_t>(i) * k + j]; };
    std::vector<int> tr(static_cast<size_t>(k));
    std::vector<double> temp(static_cast<size_t>(k));
    for (int j = 0; j < k; ++j) {
        int big = j;
        double bv = std::fabs(A(j, j));
        for (int i = j + 1; i < k; ++i)
            if (std::fabs(A(i, i)) > bv) {
                bv = std::fabs(A(i, i));
                big = i;
            }
        tr[static_cast<size_t>(j)] = big;
        if (big != j) {
            for (int c = 0; c < j; ++c) std::swap(A(j, c), A(big, c));
            for (int r = big + 1; r < k; ++r) std::swap(A(r, j), A(r, big));
            std::swap(A(j, j), A(big, big));
            for (int i = j + 1; i < big; ++i) std::swap(A(i, j), A(big, i));
        }
        if (j > 0) {
            for (int c = 0; c < j; ++c) temp[static_cast<size_t>(c)] = A(c, c) * A(j, c);
            double s = 0.0;
            for (int c = 0; c < j; ++c) s += A(j, c) * temp[static_cast<size_t>(c)];
            A(j, j) -= s;
            for (int r = j + 1; r < k; ++r) {
                double t = 0.0;
                for (int c = 0; c < j; ++c) t += A(r, c) * temp[static_cast<size_t>(c)];
                A(r, j) -= t;
            }
        }
        const double akk = A(j, j);
        if (j + 1 < k && std::fabs(akk) > 0.0)
            for (int r = j + 1; r < k; ++r) A(r, j) /= akk;
    }
    std::vector<double> M(static_cast<size_t>(k) * k, 0.0);
    for (int i = 0; i < k; ++i) M[static_cast<size_t>(i) * k + i] = 1.0;
    for (int j = 0; j < k; ++j)  // P: transpositions applied to rows in order
        if (tr[static_cast<size_t>(j)] != j)
            std::swap_ranges(M.begin() + static_cast<std::ptrdiff_t>(j) * k, M.begin() + static_cast<std::ptrdiff_t>(j + 1) * k,
                             M.begin() + static_cast<std::ptrdiff_t>(tr[static_cast<size_t>(j)]) * k);
    for (int r = 0; r < k; ++r)  // L^{-1}
        for (int c = 0; c < r; ++c) {
            const double l = A(r, c);
            if (l == 0.0) continue;
            for (int q = 0; q < k; ++q) M[static_cast<size_t>(r) * k + q] -= l * M[static_cast<size_t>(c) * k + q];
        }
    for (int r = 0; r < k; ++r) {
        const double s = 1.0 / std::sqrt(std::max(std::fabs(A(r, r)), thr));
        for (int q = 0; q < k; ++q) M[static_cast<size_t>(r) * k + q] *= s;
    }
    return M;
}

}  // namespace
}  // namespace ksvm_nfft

using namespace ksvm_nfft;

extern "C" int ksvm_nfft_nystrom(const ksvm_nfft_op* op, int window, int rank, int mode, uint64_t seed,
                                 double ldl_threshold, double* Z, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!op || !Z) throw std::invalid_argument("nystrom: null argument");
        const int64_t n = ksvm_nfft_op_size(op);
        if (rank < 1 || rank > n) throw std::invalid_argument("nystrom: rank must lie in [1, n]");
        if (mode != KSVM_NFFT_NYSTROM_COLUMNS && mode != KSVM_NFFT_NYSTROM_GAUSSIAN)
            throw std::invalid_argument("nystrom: unknown mode");
        if (mode == KSVM_NFFT_NYSTROM_GAUSSIAN && window != -1)
            throw std::invalid_argument("nystrom: the Gaussian sketch applies the whole operator (window -1)");
        if (ptr_kind != KSVM_NFFT_HOST && ptr_kind != KSVM_NFFT_DEVICE) throw std::invalid_argument("bad ptr_kind");
        const int k = rank;
        const size_t N = static_cast<size_t>(n), KN = static_cast<size_t>(k) * N;
        DeviceGuard dg(ksvm_nfft_op_device(op));
        cudaStream_t own = nullptr;
        CK(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{own};
        cudaStream_t st = ptr_kind == KSVM_NFFT_DEVICE ? static_cast<cudaStream_t>(stream) : own;
        std::mt19937_64 rng(seed);
        DevBuf<double> KQ, C, scratch, Md, Zd;
        KQ.alloc(KN);
        C.alloc(static_cast<size_t>(k) * k);
        std::vector<double> Ch(static_cast<size_t>(k) * k);
        if (mode == KSVM_NFFT_NYSTROM_COLUMNS) {  // P:src/low_rank.cpp:124-136
            std::vector<int64_t> pool(N);
            std::iota(pool.begin(), pool.end(), int64_t{0});
            std::shuffle(pool.begin(), pool.end(), rng);
            std::vector<int64_t> cols(pool.begin(), pool.begin() + k);
            DevBuf<long long> cd;
            cd.upload(reinterpret_cast<const long long*>(cols.data()), static_cast<size_t>(k), st);
            okc(ksvm_nfft_kernel_rows(op, window, cols.data(), k, KQ.p, KSVM_NFFT_DEVICE, st), "nystrom");
            kn_gather_cols<<<(k * k + 255) / 256, 256, 0, st>>>(KQ.p, n, k, cd.p, C.p);
            ++launch_counter();
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(Ch.data(), C.p, sizeof(double) * Ch.size(), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else {  // P:src/low_rank.cpp:137-147
            std::normal_distribution<double> normal(0.0, 1.0);
            std::vector<double> G(KN);
            for (int64_t i = 0; i < n; ++i)
                for (int c = 0; c < k; ++c) G[static_cast<size_t>(c) * N + static_cast<size_t>(i)] = normal(rng);
            DevBuf<double> Gd, Q;
            Gd.upload(G.data(), KN, st);
            Q.alloc(KN);
            okc(ksvm_nfft_op_apply_batch(op, Gd.p, Q.p, k, n, KSVM_NFFT_DEVICE, st), "nystrom sketch");
            // orthonormal basis of range(Y), Y in Q: CGS with one re-orthogonalisation
            const int nb = reduce_blocks(n);
            DevBuf<double> part, h;
            part.alloc(static_cast<size_t>(kRB) * std::max(k, 1));
            h.alloc(static_cast<size_t>(std::max(k, 1)));
            for (int j = 0; j < k; ++j) {
                double* yj = Q.p + static_cast<size_t>(j) * N;
                for (int pass = 0; pass < 2 && j > 0; ++pass) {
                    kn_mdot<<<nb, kRT, 0, st>>>(Q.p, n, j, yj, part.p);
                    kn_rows_finish<<<(j + 7) / 8, 256, 0, st>>>(part.p, nb, j, h.p);
                    kn_project<<<nb, kRT, 0, st>>>(yj, Q.p, n, j, h.p);
                    launch_counter() += 3;
                }
                kn_sumsq<<<nb, kRT, 0, st>>>(yj, n, part.p);
                kn_normalize<<<nb, kRT, 0, st>>>(yj, n, part.p, nb);
                launch_counter() += 2;
            }
            CK(cudaGetLastError());
            Gd.reset();
            okc(ksvm_nfft_op_apply_batch(op, Q.p, KQ.p, k, n, KSVM_NFFT_DEVICE, st), "nystrom sketch");
            // C = Q^T KQ (P:src/low_rank.cpp:147)
            const int nt = (k + 7) / 8;
            const int nchunks = static_cast<int>(std::min<long long>(64, std::max<long long>(1, n / 1024)));
            const long long chunk = ((n + nchunks - 1) / nchunks + 3) / 4 * 4;
            scratch.alloc(static_cast<size_t>(nchunks) * nt * nt * 64);
            kn_gram_partial<<<dim3(nt * nt, nchunks), 32, 0, st>>>(Q.p, KQ.p, k, n, chunk, nt, scratch.p);
            kn_gram_finish<<<(k * k + 255) / 256, 256, 0, st>>>(scratch.p, nchunks, nt, k, C.p);
            launch_counter() += 2;
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(Ch.data(), C.p, sizeof(double) * Ch.size(), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
        std::vector<double> S(Ch.size());  // C = (C + C^T) / 2 (P:src/low_rank.cpp:150)
        for (int r = 0; r < k; ++r)
            for (int c = 0; c < k; ++c)
                S[static_cast<size_t>(r) * k + c] = 0.5 * (Ch[static_cast<size_t>(r) * k + c] + Ch[static_cast<size_t>(c) * k + r]);
        const std::vector<double> M = ldlt_map(std::move(S), k, ldl_threshold);
        Md.upload(M.data(), M.size(), st);
        double* zdst = Z;
        if (ptr_kind == KSVM_NFFT_HOST) {
            Zd.alloc(KN);
            zdst = Zd.p;
        }
        kn_apply_small<<<reduce_blocks(n), kRT, 0, st>>>(zdst, Md.p, KQ.p, k, n);
        ++launch_counter();
        CK(cudaGetLastError());
        if (ptr_kind == KSVM_NFFT_HOST)
            CK(cudaMemcpyAsync(Z, Zd.p, sizeof(double) * KN, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}
