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
//    and inverted explicitly on the device by Gauss-Jordan with the same
//    partial-pivoting rule (the reference keeps the LU, P:src/saddle.cpp:57);
//    the rcond < 1e-15 fallback (:59-60) uses the exact 1-norm condition
//    number.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "capi_common.cuh"
#include "launch.cuh"
#include "reduce.cuh"

namespace ksvm_nfft {
namespace {

constexpr int kRows = 32;  // basis rows per pass of the multi-dot kernels
constexpr int kMaxRank = 1024;

// sum_a M[a][i] c[a] for a < rows with four independent accumulators
// (a mod 4), so eight row loads are in flight per thread; fixed order.
__device__ __forceinline__ double rows_dot(const double* __restrict__ M, long long ld, int rows, long long i,
                                          const double* __restrict__ c) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int a = 0;
#pragma unroll 2
    for (; a + 4 <= rows; a += 4) {
        const double m0 = M[static_cast<long long>(a) * ld + i], m1 = M[static_cast<long long>(a + 1) * ld + i];
        const double m2 = M[static_cast<long long>(a + 2) * ld + i], m3 = M[static_cast<long long>(a + 3) * ld + i];
        s0 += m0 * c[a];
        s1 += m1 * c[a + 1];
        s2 += m2 * c[a + 2];
        s3 += m3 * c[a + 3];
    }
    for (; a < rows; ++a) s0 += M[static_cast<long long>(a) * ld + i] * c[a];
    return (s0 + s1) + (s2 + s3);
}

__global__ void __launch_bounds__(kRT) k_mul(double* __restrict__ out, const double* __restrict__ a,
                                             const double* __restrict__ b, long long n,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
    KSVM_FOR_BLOCK_INDEX(j, n) out[j] = a[j] * b[j];
}

// P:src/saddle.cpp:29-31: out_j = y_j (K y v)_j + theta_j v_j - w y_j; partial of y . v
__global__ void __launch_bounds__(kRT) k_saddle_post(double* __restrict__ out, const double* __restrict__ y,
                                                     const double* __restrict__ kv, const double* __restrict__ theta,
                                                     const double* __restrict__ vw, long long n,
                                                     double* __restrict__ partial,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
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
                                const double* __restrict__ sub, int root,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
    const double s = warp_sum_strided(partial, nb, 1);
    if (threadIdx.x == 0) *dst = root ? sqrt(s) : coef * s - (sub ? *sub : 0.0);
}

// partial[b * rows + a] = block b's share of sum_i M[a][i] x_i for a < rows,
// x_i = w_i (mode 0) or y_i g_i / theta_i (mode 1, P:src/saddle.cpp:80).
__global__ void __launch_bounds__(kRT) k_mdot(const double* __restrict__ M, long long ld, int rows, long long L,
                                              int mode, const double* __restrict__ w, const double* __restrict__ y,
                                              const double* __restrict__ theta, double* __restrict__ partial,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
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
__global__ void k_rows_finish(const double* __restrict__ partial, int nb, int rows, double* __restrict__ out,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
    const int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (a >= rows) return;
    const double s = warp_sum_strided(partial + a, nb, rows);
    if (lane == 0) out[a] = s;
}

// inner = Cinv s (k x k, k <= kMaxRank)
__global__ void k_gemv_small(const double* __restrict__ Cinv, int k, const double* __restrict__ s,
                             double* __restrict__ inner,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
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
                                                 long long n, double* __restrict__ partial,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
    extern __shared__ double s_inner[];
    for (int a = threadIdx.x; a < k; a += blockDim.x) s_inner[a] = inner[a];
    __syncthreads();
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        const double s = rows_dot(Z, n, k, j, s_inner);
        const double x1 = g[j] / theta[j] - y[j] * s / theta[j];
        out[j] = x1;
        acc += y[j] * x1;
    }
    block_partial(acc, partial);
}

// P:src/saddle.cpp:74-75 (fallback / rank 0): x1 = g / theta
__global__ void __launch_bounds__(kRT) k_diag_out(double* __restrict__ out, const double* __restrict__ g,
                                                  const double* __restrict__ y, const double* __restrict__ theta,
                                                  long long n, double* __restrict__ partial,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
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
                                                      long long L, int mode,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
    KSVM_FOR_BLOCK_INDEX(i, L) {
        const double s = rows_dot(V, ld, rows, i, c);
        w[i] = mode == 0 ? w[i] - s : s;
    }
}

__global__ void __launch_bounds__(kRT) k_scale(double* __restrict__ dst, const double* __restrict__ src, long long L,
                                               const double* __restrict__ denom,
        const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;  // GMRES look-ahead past convergence
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

// Capacitance partials, SMEM-staged (k <= kGramMaxK): CTA x owns a fixed
// column range and stages 32-column slices of Z (all k rows, one HBM read of
// Z per refresh) in shared memory; each warp owns a contiguous run of the
// upper-triangle 8x8 tiles (ta <= tb; C is symmetric) and accumulates them in
// registers with DMMA.8x8x4 over the whole range. Slices arrive by cp.async
// into two SMEM buffers (the next one in flight during the current MMAs). partial[x][tile][64], tile
// in row-major upper-triangle order; k_cap_finish_sym sums x in order.
constexpr int kGramWarps = 16, kGramTiles = 24, kGramCols = 32, kGramLd = 36;
constexpr int kGramMaxK = 256;
constexpr int kGramCTAs = 148;                                     // one per B200 SM

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0) : "memory");
}

__global__ void __launch_bounds__(kGramWarps * 32, 1)
    k_cap_gram(const double* __restrict__ Z, const double* __restrict__ theta, int k, long long n, int nt, int T,
               long long cols, double* __restrict__ partial) {
    extern __shared__ double s_z[];  // 2 buffers: nt*8 rows x kGramLd, then kGramCols theta values
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int rows = nt * 8, nthr = kGramWarps * 32, bufsz = rows * kGramLd + kGramCols;
    const long long jb = blockIdx.x * cols, je = min(n, jb + cols);
    // this warp's tiles [L0, L1) of the T upper-triangle tiles
    const int L0 = warp * T / kGramWarps, L1 = (warp + 1) * T / kGramWarps, cnt = L1 - L0;
    int ta0 = 0, rs = 0;
    while (ta0 < nt && rs + (nt - ta0) <= L0) {
        rs += nt - ta0;
        ++ta0;
    }
    const int tb0 = ta0 + (L0 - rs);
    double acc[kGramTiles][2];
#pragma unroll
    for (int i = 0; i < kGramTiles; ++i) acc[i][0] = acc[i][1] = 0.0;
    auto issue = [&](long long j0, double* buf) {  // slice [j0, j0 + 32) -> buf (zero-filled outside)
        for (int e = tid; e < rows * kGramCols; e += nthr) {
            const int r = e >> 5, c = e & 31;
            const long long j = j0 + c;
            const bool ok = r < k && j < je;
            cp_async8(buf + r * kGramLd + c, ok ? Z + static_cast<long long>(r) * n + j : Z, ok);
        }
        if (tid < kGramCols) {
            const bool ok = j0 + tid < je;
            cp_async8(buf + rows * kGramLd + tid, ok ? theta + j0 + tid : theta, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    if (jb < je) issue(jb, s_z);
    int it = 0;
    for (long long j0 = jb; j0 < je; j0 += kGramCols, ++it) {
        const double* cur = s_z + (it & 1) * bufsz;
        if (j0 + kGramCols < je)
            issue(j0 + kGramCols, s_z + ((it + 1) & 1) * bufsz);  // in flight during the MMAs
        else
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();  // slice `it` landed for every thread
        if (cnt > 0) {
#pragma unroll 2
            for (int kk = 0; kk < kGramCols / 4; ++kk) {
                const int col = kk * 4 + t;
                const double th = cur[rows * kGramLd + col];
                const double sc = th != 0.0 ? 1.0 / th : 0.0;  // zero-filled columns past the range
                int ta = ta0, tb = tb0;
                double a = cur[(ta * 8 + g) * kGramLd + col] * sc;
#pragma unroll
                for (int i = 0; i < kGramTiles; ++i)
                    if (i < cnt) {
                        const double b = cur[(tb * 8 + g) * kGramLd + col];
                        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                            : "+d"(acc[i][0]), "+d"(acc[i][1])
                            : "d"(a), "d"(b));
                        if (++tb == nt) {
                            ++ta;
                            tb = ta;
                            if (ta < nt) a = cur[(ta * 8 + g) * kGramLd + col] * sc;
                        }
                    }
            }
        }
        __syncthreads();  // slice consumed before its buffer is refilled
    }
    double* out = partial + static_cast<long long>(blockIdx.x) * T * 64;
#pragma unroll
    for (int i = 0; i < kGramTiles; ++i)
        if (i < cnt) {
            out[static_cast<long long>(L0 + i) * 64 + g * 8 + 2 * t] = acc[i][0];
            out[static_cast<long long>(L0 + i) * 64 + g * 8 + 2 * t + 1] = acc[i][1];
        }
}

// C[a][b] = (a == b) + sum over column ranges (in order) of the symmetric tile
__global__ void k_cap_finish_sym(const double* __restrict__ partial, int nparts, int nt, int T, int k,
                                 double* __restrict__ C) {
    pdl_trigger();
    pdl_wait();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= k * k) return;
    int a = idx / k, b = idx % k;
    if ((a >> 3) > (b >> 3)) {
        const int s = a;
        a = b;
        b = s;
    }
    const int ta = a >> 3, tb = b >> 3;
    const int tile = ta * nt - ta * (ta - 1) / 2 + (tb - ta), e = (a & 7) * 8 + (b & 7);
    double s = 0.0;
    for (int c = 0; c < nparts; ++c) s += partial[(static_cast<long long>(c) * T + tile) * 64 + e];
    C[idx] = (idx / k == idx % k ? 1.0 : 0.0) + s;
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

// Capacitance inverse on the device (one CTA, deterministic): Gauss-Jordan
// with partial pivoting (pivot = first row of largest |a|, as getrf / Eigen's
// PartialPivLU choose it) on [C | I] (k x 2k, row-major, in global memory /
// L2), plus the reference's guards (P:src/saddle.cpp:55-60): a non-finite
// capacitance, a zero pivot or rcond = 1 / (|C|_1 |C^-1|_1) < 1e-15 set
// *flag (the diagonal fallback); otherwise Cinv receives C^-1.
__device__ __forceinline__ double block_max_1024(double v, double* sh) {
    for (int o = 16; o >= 1; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double m = sh[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    __syncthreads();
    return m;
}

__global__ void __launch_bounds__(1024) k_cap_invert(double* __restrict__ A, const double* __restrict__ C, int k,
                                                      double* __restrict__ Cinv, int* __restrict__ flag) {
    extern __shared__ double s_f[];  // k multipliers of the current column
    __shared__ double sh[32];
    __shared__ int s_piv;
    __shared__ double s_pval;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int w2 = 2 * k;
    int bad = 0;
    for (int e = tid; e < k * w2; e += nt) {
        const int r = e / w2, j = e - r * w2;
        const double v = j < k ? C[r * k + j] : (j - k == r ? 1.0 : 0.0);
        if (!isfinite(v)) bad = 1;
        A[e] = v;
    }
    double cs = 0.0;  // |C|_1: column abs sums
    for (int j = tid; j < k; j += nt) {
        double s = 0.0;
        for (int r = 0; r < k; ++r) s += fabs(C[r * k + j]);
        cs = fmax(cs, s);
    }
    bad = __syncthreads_or(bad);
    if (bad) {
        if (tid == 0) *flag = 1;
        return;
    }
    const double anorm = block_max_1024(cs, sh);
    for (int c = 0; c < k; ++c) {
        // pivot: first row r >= c with the largest |A[r][c]|
        double best = -1.0;
        int bi = k;
#pragma unroll 4
        for (int r = c + tid; r < k; r += nt) {
            const double a = fabs(A[r * w2 + c]);
            if (a > best) {
                best = a;
                bi = r;
            }
        }
        for (int o = 16; o >= 1; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        if ((tid & 31) == 0) {
            sh[tid >> 5] = best;
            reinterpret_cast<int*>(s_f)[tid >> 5] = bi;  // scratch before s_f is used this step
        }
        __syncthreads();
        if (tid == 0) {
            double b = sh[0];
            int p = reinterpret_cast<int*>(s_f)[0];
            for (int w = 1; w < nt / 32; ++w) {
                const double ob = sh[w];
                const int oi = reinterpret_cast<int*>(s_f)[w];
                if (ob > b || (ob == b && oi < p)) {
                    b = ob;
                    p = oi;
                }
            }
            s_piv = p;
            s_pval = p < k ? A[p * w2 + c] : 0.0;
        }
        __syncthreads();
        const int p = s_piv;
        const double pv = s_pval;
        if (pv == 0.0) {  // singular (P:src/saddle.cpp:59-60 via rcond)
            if (tid == 0) *flag = 1;
            return;
        }
        if (p != c)
            for (int j = tid; j < w2; j += nt) {
                const double t = A[c * w2 + j];
                A[c * w2 + j] = A[p * w2 + j];
                A[p * w2 + j] = t;
            }
        __syncthreads();
        for (int j = tid; j < w2; j += nt) A[c * w2 + j] /= pv;
        for (int r = tid; r < k; r += nt) s_f[r] = r == c ? 0.0 : A[r * w2 + c];
        __syncthreads();
        // row c of the right block and of columns >= c are reread by every row:
        // stage them in registers per thread column j (fixed j per thread when
        // nt is a multiple of w2 is not guaranteed, so read through L1)
#pragma unroll 8
        for (int e = tid; e < k * w2; e += nt) {
            const int r = e / w2, j = e - r * w2;
            if (r != c && j >= c) A[e] -= s_f[r] * __ldcg(A + c * w2 + j);
        }
        __syncthreads();
    }
    double is = 0.0;  // |C^-1|_1
    for (int j = tid; j < k; j += nt) {
        double s = 0.0;
        for (int r = 0; r < k; ++r) s += fabs(A[r * w2 + k + j]);
        is = fmax(is, s);
    }
    const double inorm = block_max_1024(is, sh);
    const double rcond = 1.0 / (anorm * inorm);
    if (!isfinite(rcond) || rcond < 1e-15) {
        if (tid == 0) *flag = 1;
        return;
    }
    for (int e = tid; e < k * k; e += nt) {
        const int r = e / k, j = e - r * k;
        Cinv[e] = A[r * w2 + k + j];
    }
}

// The same inverse with [C | I] resident in the shared memory of a cluster of
// kCapCTAs CTAs (CTA q holds rows [q R, q R + R), R = ceil(k / kCapCTAs)):
// Gauss-Jordan with implicit partial pivoting (no row swaps: the pivot of
// column c is the unused row of largest |a|, lowest row on ties, found from
// one candidate per CTA over DSMEM; every CTA reads the pivot row from its
// owner and eliminates its own rows in SMEM). Row p_c ends as [e_c | row c of
// C^-1]. Two cluster barriers per column instead of the one-CTA kernel's
// passes over an L2-resident k x 2k matrix. All CTAs take the same decisions
// from the same data, so the guards (non-finite C, zero pivot, rcond) exit
// uniformly through the final barrier.
constexpr int kCapCTAs = 8, kCapThreads = 512;

__device__ __forceinline__ void cap_cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

size_t cap_cluster_smem(int k) {
    const size_t R = (k + kCapCTAs - 1) / kCapCTAs, W = 2 * static_cast<size_t>(k);
    return sizeof(double) * (R * W + W + k + R + 8) + sizeof(int) * (2 * R + 8);
}

__global__ void __launch_bounds__(kCapThreads) k_cap_invert_cluster(const double* __restrict__ C, int k,
                                                                      double* __restrict__ Cinv,
                                                                      int* __restrict__ flag) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double s_cap[];
    const int R = (k + kCapCTAs - 1) / kCapCTAs, W = 2 * k;
    const int q = static_cast<int>(cl.block_rank());
    const int r0 = q * R, nr = max(0, min(k, r0 + R) - r0);
    double* A = s_cap;              // nr x W
    double* prow = A + R * W;       // W
    double* s_col = prow + W;       // k column |.| sums of this CTA's rows
    double* s_f = s_col + k;        // R factors of the current column
    double* s_cand = s_f + R;       // [0] |a|, [1] signed a, [2] pivot value, [3] bad flag, [4] norm
    int* s_used = reinterpret_cast<int*>(s_cand + 8);  // R: step at which the row was the pivot, -1
    int* s_ci = s_used + R;         // [0] candidate row, [1] pivot row, [2] status
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kCapThreads / 32;
    int bad = 0;
    for (int e = tid; e < nr * W; e += kCapThreads) {
        const int r = e / W, j = e - r * W;
        const double v = j < k ? C[static_cast<long long>(r0 + r) * k + j] : (j - k == r0 + r ? 1.0 : 0.0);
        if (!isfinite(v)) bad = 1;
        A[e] = v;
    }
    for (int r = tid; r < R; r += kCapThreads) s_used[r] = -1;
    bad = __syncthreads_or(bad);
    for (int j = tid; j < k; j += kCapThreads) {
        double s = 0.0;
        for (int r = 0; r < nr; ++r) s += fabs(A[r * W + j]);
        s_col[j] = s;
    }
    if (tid == 0) s_cand[3] = bad ? 1.0 : 0.0;
    cap_cluster_barrier();
    // identical in every CTA: any non-finite entry, |C|_1
    double anorm = 0.0;
    bool fail = false;
    if (warp == 0) {
        double m = 0.0;
        for (int j = lane; j < k; j += 32) {
            double s = 0.0;
            for (int o = 0; o < kCapCTAs; ++o) s += cl.map_shared_rank(s_col, o)[j];
            m = fmax(m, s);
        }
        for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        int b = lane < kCapCTAs ? cl.map_shared_rank(s_cand, lane)[3] != 0.0 : 0;
        b = __any_sync(0xffffffffu, b);
        if (lane == 0) {
            s_cand[4] = m;
            s_ci[2] = b;
        }
    }
    __syncthreads();
    anorm = s_cand[4];
    fail = s_ci[2] != 0;
    for (int c = 0; c < k && !fail; ++c) {
        // this CTA's candidate and the factors of column c
        if (warp == 0) {
            double best = -1.0, sv = 0.0;
            int bi = k;
            for (int r = lane; r < nr; r += 32) {
                const double a = A[r * W + c];
                s_f[r] = a;
                if (s_used[r] < 0 && fabs(a) > best) {
                    best = fabs(a);
                    sv = a;
                    bi = r0 + r;
                }
            }
            for (int o = 16; o >= 1; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o), os = __shfl_xor_sync(0xffffffffu, sv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    sv = os;
                    bi = oi;
                }
            }
            if (lane == 0) {
                s_cand[0] = best;
                s_cand[1] = sv;
                s_ci[0] = bi;
            }
        }
        cap_cluster_barrier();  // #1: candidates and factors complete
        if (warp == 0) {
            double best = -1.0, sv = 0.0;
            int bi = k;
            if (lane < kCapCTAs) {
                const double* rc = cl.map_shared_rank(s_cand, lane);
                best = rc[0];
                sv = rc[1];
                bi = cl.map_shared_rank(s_ci, lane)[0];
            }
            for (int o = 16; o >= 1; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o), os = __shfl_xor_sync(0xffffffffu, sv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    sv = os;
                    bi = oi;
                }
            }
            if (lane == 0) {
                s_ci[1] = bi;
                s_cand[2] = bi < k ? sv : 0.0;
            }
        }
        __syncthreads();
        const int p = s_ci[1];
        const double pv = s_cand[2];
        if (pv == 0.0) {  // singular (P:src/saddle.cpp:59-60 via rcond); same in every CTA
            fail = true;
            break;
        }
        {
            const int po = p / R, pr = p - po * R;
            const double* src = cl.map_shared_rank(A, po) + static_cast<long long>(pr) * W;
            for (int j = c + tid; j < W; j += kCapThreads) prow[j] = src[j] / pv;
        }
        cap_cluster_barrier();  // #2: every CTA holds the pivot row; the owner may overwrite it
        const int pl = p - r0;  // local index of the pivot row (if this CTA owns it)
        for (int r = warp; r < nr; r += nw) {
            double* row = A + r * W;
            if (r == pl) {
                for (int j = c + lane; j < W; j += 32) row[j] = prow[j];
                if (lane == 0) s_used[r] = c;
            } else {
                const double f = s_f[r];
                if (f != 0.0)
                    for (int j = c + lane; j < W; j += 32) row[j] -= f * prow[j];
            }
        }
        __syncthreads();
    }
    if (!fail) {
        // |C^-1|_1: right halves over all rows (a row permutation of C^-1)
        for (int j = tid; j < k; j += kCapThreads) {
            double s = 0.0;
            for (int r = 0; r < nr; ++r) s += fabs(A[r * W + k + j]);
            s_col[j] = s;
        }
        cap_cluster_barrier();
        if (warp == 0) {
            double m = 0.0;
            for (int j = lane; j < k; j += 32) {
                double s = 0.0;
                for (int o = 0; o < kCapCTAs; ++o) s += cl.map_shared_rank(s_col, o)[j];
                m = fmax(m, s);
            }
            for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) s_cand[4] = m;
        }
        __syncthreads();
        const double rcond = 1.0 / (anorm * s_cand[4]);
        fail = !isfinite(rcond) || rcond < 1e-15;
        if (!fail)
            for (int e = tid; e < nr * k; e += kCapThreads) {
                const int r = e / k, j = e - r * k;
                Cinv[static_cast<long long>(s_used[r]) * k + j] = A[r * W + k + j];
            }
    }
    if (fail && q == 0 && tid == 0) *flag = 1;
    cap_cluster_barrier();  // no CTA leaves while another may read its shared memory
}

// ---- fused GMRES-iteration kernels ----------------------------------------
// The iteration's vector work, fused where the pieces share a block's index
// set (no grid-wide dependency between them): the preconditioner output also
// writes the matvec input u = y .* z; the saddle post-step and the first
// Gram-Schmidt pass finish the scalar entries (z_n, w_n) from the previous
// kernel's block partials themselves; each Gram-Schmidt subtraction is fused
// with the next pass's dot partials (or the norm partial).

// s[a] = sum_b partial[b*k + a] (warp per row), then inner = Cinv s
__global__ void __launch_bounds__(1024) gk_inner(const double* __restrict__ partial, int nb, int k,
                                                 const double* __restrict__ Cinv, double* __restrict__ inner,
                                                 const int* __restrict__ stop) {
    extern __shared__ double s_s[];
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;
    const int lane = threadIdx.x & 31;
    for (int a = threadIdx.x >> 5; a < k; a += blockDim.x >> 5) {
        const double acc = warp_sum_strided(partial + a, nb, k);
        if (lane == 0) s_s[a] = acc;
    }
    __syncthreads();
    for (int a = threadIdx.x; a < k; a += blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < k; ++c) acc += Cinv[static_cast<long long>(a) * k + c] * s_s[c];
        inner[a] = acc;
    }
}

// z = P^{-1} g on [0, n) (mode 0: SMW, 1: diagonal fallback / rank 0,
// 2: identity), u = y .* z, partial of y . z (z_n is finished by gk_post)
__global__ void __launch_bounds__(kRT) gk_precond_out(double* __restrict__ z, double* __restrict__ u,
                                                      const double* __restrict__ y_op,
                                                      const double* __restrict__ g, const double* __restrict__ y,
                                                      const double* __restrict__ theta, const double* __restrict__ Z,
                                                      int k, const double* __restrict__ inner, long long n, int mode,
                                                      double* __restrict__ partial, const int* __restrict__ stop) {
    extern __shared__ double s_inner[];
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;
    if (mode == 0) {
        for (int a = threadIdx.x; a < k; a += blockDim.x) s_inner[a] = inner[a];
        __syncthreads();
    }
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        double x1;
        if (mode == 0) {
            const double s = rows_dot(Z, n, k, j, s_inner);
            x1 = g[j] / theta[j] - y[j] * s / theta[j];
        } else if (mode == 1) {
            x1 = g[j] / theta[j];
        } else {
            x1 = g[j];
        }
        z[j] = x1;
        u[j] = y_op[j] * x1;  // the saddle matvec's input y .* z (P:src/saddle.cpp:29)
        acc += y[j] * x1;
    }
    block_partial(acc, partial);
}

// z_n (P:src/saddle.cpp:88: -y.x1 - g_n; identity: g_n) from the
// preconditioner's partials, then w = A z on [0, n) and partial of y . z
__global__ void __launch_bounds__(kRT) gk_post(double* __restrict__ w, const double* __restrict__ y,
                                               const double* __restrict__ kv, const double* __restrict__ theta,
                                               const double* __restrict__ z, const double* __restrict__ g,
                                               const double* __restrict__ pre_partial, int pre_nb, int identity,
                                               long long n, double* __restrict__ partial, const int* __restrict__ stop) {
    __shared__ double s_zn;
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;
    if (threadIdx.x < 32) {
        const double s = identity ? 0.0 : warp_sum_strided(pre_partial, pre_nb, 1);
        if (threadIdx.x == 0) s_zn = identity ? g[n] : -s - g[n];
    }
    __syncthreads();
    const double zn = s_zn;
    double acc = 0.0;
    KSVM_FOR_BLOCK_INDEX(j, n) {
        const double v = z[j];
        w[j] = y[j] * kv[j] + theta[j] * v - zn * y[j];
        acc += y[j] * v;
    }
    block_partial(acc, partial);
}

// row-tiled partial dots of V[0..rows) with x over this block's indices
__device__ __forceinline__ void mdot_block(const double* __restrict__ V, long long ld, int rows, long long L,
                                           const double* __restrict__ x, double* __restrict__ partial) {
    __shared__ double sh[kRT / 32][kRows];
    for (int a0 = 0; a0 < rows; a0 += kRows) {
        double acc[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) acc[r] = 0.0;
        KSVM_FOR_BLOCK_INDEX(i, L) {
            const double xi = x[i];
#pragma unroll
            for (int r = 0; r < kRows; ++r)
                if (a0 + r < rows) acc[r] += V[static_cast<long long>(a0 + r) * ld + i] * xi;
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

// w_n = -y . z (P:src/saddle.cpp:32) from gk_post's partials (the block that
// owns index n stores it first), then the first Gram-Schmidt pass's partial
// dots h = V^T w
__global__ void __launch_bounds__(kRT) gk_cgs_first(const double* __restrict__ V, long long ld, int rows,
                                                    double* __restrict__ w, long long n1,
                                                    const double* __restrict__ post_partial, int post_nb,
                                                    double* __restrict__ partial, const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;
    const long long nidx = n1 - 1;
    const bool owner = (nidx / kRT) % kRB == blockIdx.x;
    if (owner) {
        if (threadIdx.x < 32) {
            const double s = warp_sum_strided(post_partial, post_nb, 1);
            if (threadIdx.x == 0) w[nidx] = -s;
        }
        __syncthreads();
    }
    mdot_block(V, ld, rows, n1, w, partial);
}

// w -= V h (this block's indices); then either the next pass's partial dots
// (norm == 0) or the partial of |w|^2 (norm == 1)
__global__ void __launch_bounds__(kRT) gk_cgs_combine(const double* __restrict__ V, long long ld, int rows,
                                                      const double* __restrict__ h, double* __restrict__ w,
                                                      long long n1, int norm, double* __restrict__ partial,
                                                      const int* __restrict__ stop) {
    pdl_trigger();
    pdl_wait();
    if (stop && *stop) return;
    double sq = 0.0;
    KSVM_FOR_BLOCK_INDEX(i, n1) {
        const double wi = w[i] - rows_dot(V, ld, rows, i, h);
        w[i] = wi;
        sq += wi * wi;
    }
    if (norm)
        block_partial(sq, partial);
    else
        mdot_block(V, ld, rows, n1, w, partial);
}

// hnext = |w| from gk_cgs_combine's partials, then the Givens step
__global__ void gk_norm_givens(const double* __restrict__ npartial, int nb, double* __restrict__ hnext_out, int k,
                               int MI, const double* __restrict__ h, double rhs_norm, double tol,
                               double* __restrict__ H, double* __restrict__ cs, double* __restrict__ sn,
                               double* __restrict__ beta, double* __restrict__ hist, int* __restrict__ stat);

// One GMRES step's Givens update on the device (P:src/saddle.cpp:127-163),
// so the host can enqueue iterations ahead instead of waiting for each
// Hessenberg column: H(:,k) = h1 + h2, H(k+1,k) = hnext, stored rotations,
// new rotation, beta, the relative residual estimate and the stop rules.
// stat = {stop, iterations, converged, breakdown, kfinal}.


// The new rotation, beta, the residual estimate and the stop rules
// (P:src/saddle.cpp:135-163) on the rotated column col[0..k+1] (col[k+1]
// = hnext on entry); col[k], col[k+1] are updated in place.
__device__ void givens_tail(int k, int MI, double* col, double hnext, double rhs_norm, double tol,
                            double* __restrict__ cs, double* __restrict__ sn, double* __restrict__ beta,
                            double* __restrict__ hist, int* __restrict__ stat) {
    col[k + 1] = hnext;
    const double denom = hypot(col[k], col[k + 1]);
    if (denom == 0.0) {
        stat[3] = 1;
        stat[0] = 1;
        stat[4] = k;
        return;
    }
    cs[k] = col[k] / denom;
    sn[k] = col[k + 1] / denom;
    col[k] = denom;
    col[k + 1] = 0.0;
    beta[k + 1] = -sn[k] * beta[k];
    beta[k] = cs[k] * beta[k];
    const double rel = fabs(beta[k + 1]) / rhs_norm;
    hist[stat[1]] = rel;
    stat[1] += 1;
    if (rel <= tol) {
        stat[2] = 1;
        stat[0] = 1;
        stat[4] = k + 1;
    } else if (hnext <= 1e-14 * rhs_norm) {  // happy breakdown
        stat[3] = 1;
        stat[2] = 1;
        stat[0] = 1;
        stat[4] = k + 1;
    } else if (k + 1 == MI) {
        stat[0] = 1;
        stat[4] = MI;
    }
}


__global__ void gk_norm_givens(const double* __restrict__ npartial, int nb, double* __restrict__ hnext_out, int k,
                               int MI, const double* __restrict__ h, double rhs_norm, double tol,
                               double* __restrict__ H, double* __restrict__ cs, double* __restrict__ sn,
                               double* __restrict__ beta, double* __restrict__ hist, int* __restrict__ stat) {
    extern __shared__ double sg[];  // [0, k+1): H(:,k) = h1 + h2; [k+1, 2k+1): cs; [2k+1, 3k+1): sn
    pdl_trigger();
    pdl_wait();
    if (stat[0] || threadIdx.x >= 32) return;
    const double s = warp_sum_strided(npartial, nb, 1);
    for (int i = threadIdx.x; i <= k; i += 32) sg[i] = h[i] + h[k + 1 + i];
    for (int i = threadIdx.x; i < k; i += 32) {
        sg[k + 1 + i] = cs[i];
        sg[2 * k + 1 + i] = sn[i];
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        const double hnext = sqrt(s);
        *hnext_out = hnext;
        // stored rotations on the new column: carried in a register chain
        // (P:src/saddle.cpp:130-134)
        double x = sg[0];
        for (int i = 0; i < k; ++i) {
            const double c = sg[k + 1 + i], sv = sg[2 * k + 1 + i], yv = sg[i + 1];
            sg[i] = c * x + sv * yv;
            x = -sv * x + c * yv;
        }
        sg[k] = x;
        givens_tail(k, MI, sg, hnext, rhs_norm, tol, cs, sn, beta, hist, stat);
    }
    __syncwarp();
    for (int i = threadIdx.x; i <= k + 1; i += 32) H[static_cast<long long>(i) * MI + k] = sg[i];
}


int blocks_for(long long L) { return reduce_blocks(L); }

constexpr size_t kGivensMaxSmem = 227 * 1024;

// gk_norm_givens past 48 KB of dynamic shared memory (max_iter > 2047):
// per-device opt-in, set the first time each device needs it.
void ensure_givens_attributes() {
    static std::mutex mu;
    static std::vector<bool> done(256, false);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 256 && !done[static_cast<size_t>(dev)]) {
        CK(cudaFuncSetAttribute(gk_norm_givens, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kGivensMaxSmem)));
        done[static_cast<size_t>(dev)] = true;
    }
}

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
    DevBuf<double> gH, gcs, gsn, gbeta, ghist;  // device-side Givens state (gk_norm_givens)
    DevBuf<double> pre_partial, norm_partial;   // fused-iteration block partials
    DevBuf<int> gstat;                          // {stop, iterations, converged, breakdown, kfinal}
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
    DevBuf<double> cap_part, cap_C, cap_aug;  // refresh workspace, kept across refreshes
    DevBuf<int> cap_flag;
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

// count of entries that are not > 0 (NaN included)
__global__ void __launch_bounds__(kRT) k_count_nonpositive(const double* __restrict__ theta, long long n,
                                                           int* __restrict__ bad) {
    int c = 0;
    KSVM_FOR_BLOCK_INDEX(j, n) c += !(theta[j] > 0.0);
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, c);
}

// Device-side check_theta: one small kernel and a 4-byte read back (syncs st).
void check_theta_dev(const double* theta, int64_t n, cudaStream_t st, const char* who) {
    if (!theta) throw std::invalid_argument(std::string(who) + ": null Theta");
    DevBuf<int> bad;
    bad.alloc(1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    k_count_nonpositive<<<blocks_for(n), kRT, 0, st>>>(theta, n, bad.p);
    ++launch_counter();
    CK(cudaGetLastError());
    int h = 0;
    CK(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h) throw std::invalid_argument(std::string(who) + ": Theta must be positive");
}

// out = A vw (device vectors of length n + 1), P:src/saddle.cpp:22-33
void saddle_apply_dev(const ksvm_nfft_saddle& S, const double* vw, double* out, cudaStream_t st,
                      const int* stop = nullptr) {
    const long long n = S.n;
    const int nb = blocks_for(n);
    launch_k(k_mul, dim3(nb), dim3(kRT), 0, st, S.u.p, S.y.p, vw, n, stop);
    const int rc = ksvm_nfft_op_apply(S.op, S.u.p, S.kv.p, KSVM_NFFT_DEVICE, st);
    if (rc != KSVM_NFFT_OK) throw std::runtime_error(std::string("saddle apply: ") + ksvm_nfft_last_error());
    launch_k(k_saddle_post, dim3(nb), dim3(kRT), 0, st, out, S.y.p, S.kv.p, S.theta.p, vw, n, S.partial.p, stop);
    launch_k(k_finish_scalar, dim3(1), dim3(32), 0, st, S.partial.p, nb, out + n, -1.0, nullptr, 0, stop);
    launch_counter() += 4;
    CK(cudaGetLastError());
}

// out = P^{-1} g (device vectors of length n + 1), P:src/saddle.cpp:65-90
void precond_apply_dev(const ksvm_nfft_precond& P, const double* g, double* out, cudaStream_t st,
                       const int* stop = nullptr) {
    const long long n = P.n;
    if (P.identity) {
        CK(cudaMemcpyAsync(out, g, sizeof(double) * (n + 1), cudaMemcpyDeviceToDevice, st));
        return;
    }
    if (!P.fresh) throw std::logic_error("SaddlePreconditioner: refresh() before apply()");
    const int nb = blocks_for(n);
    if (P.fallback || P.k == 0) {
        launch_k(k_diag_out, dim3(nb), dim3(kRT), 0, st, out, g, P.y.p, P.theta.p, n, P.partial.p, stop);
        launch_counter() += 1;
    } else {
        launch_k(k_mdot, dim3(nb), dim3(kRT), 0, st, P.Z.p, n, P.k, n, 1, g, P.y.p, P.theta.p, P.partial.p, stop);
        launch_k(k_rows_finish, dim3((P.k + 7) / 8), dim3(256), 0, st, P.partial.p, nb, P.k, P.s.p, stop);
        launch_k(k_gemv_small, dim3((P.k + 127) / 128), dim3(128), 0, st, P.Cinv.p, P.k, P.s.p, P.inner.p, stop);
        launch_k(k_smw_out, dim3(nb), dim3(kRT), sizeof(double) * P.k, st, out, g, P.y.p, P.theta.p, P.Z.p, P.k, P.inner.p, n, P.partial.p, stop);
        launch_counter() += 4;
    }
    launch_k(k_finish_scalar, dim3(1), dim3(32), 0, st, P.partial.p, nb, out + n, -1.0, g + n, 0, stop);
    launch_counter() += 1;
    CK(cudaGetLastError());
}

// The capacitance kernels' shared-memory opt-in is a per-device function
// attribute: set it the first time each device is seen (like
// ensure_attributes in nfft_capi.cu), on the current device.
void ensure_cap_attributes() {
    static std::mutex mu;
    static std::vector<bool> done(256, false);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 256 && !done[static_cast<size_t>(dev)]) {
        CK(cudaFuncSetAttribute(k_cap_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        CK(cudaFuncSetAttribute(k_cap_invert_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        done[static_cast<size_t>(dev)] = true;
    }
}

// The cluster inverse when [C | I] fits the cluster's shared memory
// (k <= ~330); false: use the one-CTA kernel. KSVM_NFFT_CAP=single forces it.
bool launch_cap_cluster(const double* C, int k, double* Cinv, int* flag, cudaStream_t st) {
    static const bool disabled = [] {
        const char* e = std::getenv("KSVM_NFFT_CAP");
        return e && std::strcmp(e, "single") == 0;
    }();
    const size_t smem = cap_cluster_smem(k);
    if (disabled || smem > 227 * 1024) return false;
    ensure_cap_attributes();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kCapCTAs, 1, 1);
    cfg.blockDim = dim3(kCapThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCapCTAs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_cap_invert_cluster, C, k, Cinv, flag));
    return true;
}

// Capacitance I + Z Theta^{-1} Z^T, partial-pivot LU, rcond, inverse.
// Theta on the host (device == false, P's own stream) or on the device
// (ordered on the caller's stream st).
void precond_refresh(ksvm_nfft_precond& P, const double* theta_in, bool device, cudaStream_t st) {
    const long long n = P.n;
    if (device) {
        check_theta_dev(theta_in, n, st, "SaddlePreconditioner");
        if (P.theta.n < static_cast<size_t>(n)) P.theta.alloc(static_cast<size_t>(n));
        CK(cudaMemcpyAsync(P.theta.p, theta_in, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    } else {
        check_theta(theta_in, P.n, "SaddlePreconditioner");
        st = P.stream;
        P.theta.upload(theta_in, static_cast<size_t>(n), st);
    }
    // Not fresh until every step below succeeded: a throw part-way (launch
    // failure, out of memory) must not leave the new Theta paired with the
    // previous refresh's inverse.
    P.fresh = false;
    if (P.identity || P.k == 0) {
        CK(cudaStreamSynchronize(st));
        P.fallback = false;
        P.fresh = true;
        return;
    }
    const int k = P.k, nt = (k + 7) / 8;
    const int nchunks = static_cast<int>(std::min<long long>(64, std::max<long long>(1, n / 1024)));
    const long long chunk = ((n + nchunks - 1) / nchunks + 3) / 4 * 4;
    auto grow = [](auto& b, size_t count) {
        if (b.n < count) b.alloc(count);
    };
    DevBuf<double>& part = P.cap_part;
    DevBuf<double>& C = P.cap_C;
    grow(C, static_cast<size_t>(k) * k);
    const int T = nt * (nt + 1) / 2;
    if (k <= kGramMaxK && T <= kGramWarps * kGramTiles) {
        ensure_cap_attributes();
        const long long slices = (n + kGramCols - 1) / kGramCols;
        const long long per = (slices + kGramCTAs - 1) / kGramCTAs;  // slices per CTA
        const int nparts = static_cast<int>((slices + per - 1) / per);
        grow(part, static_cast<size_t>(nparts) * T * 64);
        const size_t smem = 2 * sizeof(double) * (static_cast<size_t>(nt) * 8 * kGramLd + kGramCols);
        k_cap_gram<<<nparts, kGramWarps * 32, smem, st>>>(P.Z.p, P.theta.p, k, n, nt, T, per * kGramCols, part.p);
        launch_k(k_cap_finish_sym, dim3((k * k + 255) / 256), dim3(256), 0, st, part.p, nparts, nt, T, k, C.p);
    } else {
        grow(part, static_cast<size_t>(nchunks) * nt * nt * 64);
        launch_k(k_cap_partial, dim3(dim3(nt * nt, nchunks)), dim3(32), 0, st, P.Z.p, P.theta.p, k, n, chunk, nt, part.p);
        launch_k(k_cap_finish, dim3((k * k + 255) / 256), dim3(256), 0, st, part.p, nchunks, nt, k, C.p);
    }
    launch_counter() += 2;
    CK(cudaGetLastError());
    // inverse on the device: Gauss-Jordan with the reference's pivot rule and guards
    DevBuf<double>& aug = P.cap_aug;
    DevBuf<int>& flag = P.cap_flag;
    grow(flag, 1);
    if (P.Cinv.n < static_cast<size_t>(k) * k) P.Cinv.alloc(static_cast<size_t>(k) * k);
    CK(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    if (!launch_cap_cluster(C.p, k, P.Cinv.p, flag.p, st)) {
        grow(aug, static_cast<size_t>(k) * 2 * k);
        k_cap_invert<<<1, 1024, sizeof(double) * std::max(k, 32), st>>>(aug.p, C.p, k, P.Cinv.p, flag.p);
    }
    ++launch_counter();
    CK(cudaGetLastError());
    int hflag = 0;
    CK(cudaMemcpyAsync(&hflag, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    P.fallback = hflag != 0;  // P:src/saddle.cpp:55-60
    P.fresh = true;
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

int ksvm_nfft_saddle_set_theta_ex(ksvm_nfft_saddle* s, const double* theta, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!s) throw std::invalid_argument("null saddle operator");
        if (ptr_kind == KSVM_NFFT_HOST) {
            check_theta(theta, s->n, "SaddleOperator");
            std::lock_guard<std::mutex> lk(s->mu);
            DeviceGuard dg(s->device);
            CK(cudaMemcpyAsync(s->theta.p, theta, sizeof(double) * s->n, cudaMemcpyHostToDevice, s->stream));
            CK(cudaStreamSynchronize(s->stream));
            return;
        }
        if (ptr_kind != KSVM_NFFT_DEVICE) throw std::invalid_argument("bad ptr_kind");
        std::lock_guard<std::mutex> lk(s->mu);
        DeviceGuard dg(s->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        check_theta_dev(theta, s->n, st, "SaddleOperator");
        CK(cudaMemcpyAsync(s->theta.p, theta, sizeof(double) * s->n, cudaMemcpyDeviceToDevice, st));
    });
}

void ksvm_nfft_saddle_free(ksvm_nfft_saddle* s) { delete s; }

int ksvm_nfft_precond_create(const double* Z, int k, int64_t n, const double* y, int device, ksvm_nfft_precond** out) {
    return ksvm_nfft_precond_create_ex(Z, k, n, y, device, KSVM_NFFT_HOST, nullptr, out);
}

int ksvm_nfft_precond_create_ex(const double* Z, int k, int64_t n, const double* y, int device, int z_ptr_kind,
                                void* stream, ksvm_nfft_precond** out) {
    return guarded([&] {
        if (z_ptr_kind != KSVM_NFFT_HOST && z_ptr_kind != KSVM_NFFT_DEVICE) throw std::invalid_argument("bad ptr_kind");
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
        if (P->k > 0 && z_ptr_kind == KSVM_NFFT_DEVICE) {  // Z already on this GPU: ordered after `stream`
            cudaStream_t zs = static_cast<cudaStream_t>(stream);
            P->Z.alloc(static_cast<size_t>(P->k) * n);
            CK(cudaMemcpyAsync(P->Z.p, Z, sizeof(double) * P->k * n, cudaMemcpyDeviceToDevice, zs));
            CK(cudaStreamSynchronize(zs));
        } else if (P->k > 0) {
            P->Z.upload(Z, static_cast<size_t>(P->k) * n, P->stream);
        }
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
        precond_refresh(*p, theta, false, nullptr);
    });
}

int ksvm_nfft_precond_refresh_ex(ksvm_nfft_precond* p, const double* theta, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("null preconditioner");
        if (ptr_kind != KSVM_NFFT_HOST && ptr_kind != KSVM_NFFT_DEVICE) throw std::invalid_argument("bad ptr_kind");
        std::lock_guard<std::mutex> lk(p->mu);
        DeviceGuard dg(p->device);
        precond_refresh(*p, theta, ptr_kind == KSVM_NFFT_DEVICE, static_cast<cudaStream_t>(stream));
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
        // gk_norm_givens stages the new Hessenberg column and the stored
        // rotations, 3 max_iter + 3 doubles, in shared memory
        if (static_cast<size_t>(3) * max_iter + 3 > kGivensMaxSmem / sizeof(double))
            throw std::invalid_argument("gmres max_iter must be <= " +
                                        std::to_string((kGivensMaxSmem / sizeof(double) - 3) / 3));
        if (p->n != s->n) throw std::invalid_argument("gmres: preconditioner size mismatch");
        if (p->device != s->device) throw std::invalid_argument("gmres: operator and preconditioner on different GPUs");
        std::lock_guard<std::mutex> lk(s->mu);
        std::lock_guard<std::mutex> lk2(p->mu);
        auto& S = const_cast<ksvm_nfft_saddle&>(*s);
        const ksvm_nfft_precond& P = *p;
        if (!P.identity && !P.fresh) throw std::logic_error("SaddlePreconditioner: refresh() before apply()");
        DeviceGuard dg(S.device);
        if ((static_cast<size_t>(3) * max_iter + 3) * sizeof(double) > 48 * 1024) ensure_givens_attributes();
        cudaStream_t st = pick_stream(ptr_kind, stream, S.stream);
        const long long n1 = S.n + 1;
        const int MI = max_iter, MIc = std::max(MI, 1);
        if (S.ws_iter < MI) {
            S.V.alloc(static_cast<size_t>(MI + 1) * n1);
            S.h.alloc(static_cast<size_t>(2 * (MI + 1) + 2));
            S.coef.alloc(static_cast<size_t>(MI + 1));
            S.partial_rows.alloc(static_cast<size_t>(kRB) * (MI + 1));
            S.gH.alloc(static_cast<size_t>(MI + 1) * MIc);
            S.gcs.alloc(static_cast<size_t>(MIc));
            S.gsn.alloc(static_cast<size_t>(MIc));
            S.gbeta.alloc(static_cast<size_t>(MI + 1));
            S.ghist.alloc(static_cast<size_t>(MIc));
            S.gstat.alloc(8);
            if (S.pinned) cudaFreeHost(S.pinned);
            S.pinned = nullptr;
            CK(cudaMallocHost(&S.pinned, sizeof(double) * (static_cast<size_t>(MI + 1) * MIc + 2 * MIc + 16)));
            S.ws_iter = MI;
        }
        if (S.z.n < static_cast<size_t>(n1)) {
            S.z.alloc(n1);
            S.w.alloc(n1);
            S.x.alloc(n1);
            S.r.alloc(n1);
            S.ax.alloc(n1);
            S.scal.alloc(4);
            S.pre_partial.alloc(kRB);
            S.norm_partial.alloc(kRB);
        }
        const int nb = blocks_for(n1);
        double* hp = S.pinned;
        const int* nostop = nullptr;
        auto norm_into = [&](const double* a, const double* b, double* dst, const int* stop) {  // |a - b| or |a|
            if (b)
                launch_k(k_sq_diff, dim3(nb), dim3(kRT), 0, st, a, b, n1, S.partial_rows.p);
            else
                launch_k(k_mdot, dim3(nb), dim3(kRT), 0, st, a, n1, 1, n1, 0, a, nullptr, nullptr, S.partial_rows.p,
                         stop);
            launch_k(k_finish_scalar, dim3(1), dim3(32), 0, st, static_cast<const double*>(S.partial_rows.p), nb, dst,
                     1.0, nullptr, 1, stop);
            launch_counter() += 2;
        };
        // right-hand side and its norm
        if (ptr_kind == KSVM_NFFT_HOST)
            CK(cudaMemcpyAsync(S.r.p, rhs, sizeof(double) * n1, cudaMemcpyHostToDevice, st));
        else
            CK(cudaMemcpyAsync(S.r.p, rhs, sizeof(double) * n1, cudaMemcpyDeviceToDevice, st));
        norm_into(S.r.p, nullptr, S.scal.p, nostop);
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
        launch_k(k_scale, dim3(nb), dim3(kRT), 0, st, S.V.p, static_cast<const double*>(S.r.p), n1,
                 static_cast<const double*>(S.scal.p), nostop);
        ++launch_counter();
        // device-side Hessenberg / Givens state
        CK(cudaMemsetAsync(S.gH.p, 0, sizeof(double) * S.gH.n, st));
        CK(cudaMemsetAsync(S.gcs.p, 0, sizeof(double) * S.gcs.n, st));
        CK(cudaMemsetAsync(S.gsn.p, 0, sizeof(double) * S.gsn.n, st));
        CK(cudaMemsetAsync(S.gbeta.p, 0, sizeof(double) * S.gbeta.n, st));
        CK(cudaMemsetAsync(S.gstat.p, 0, sizeof(int) * 8, st));
        CK(cudaMemcpyAsync(S.gbeta.p, &rhs_norm, sizeof(double), cudaMemcpyHostToDevice, st));
        if (MI == 0) {
            const int st0[5] = {1, 0, 0, 0, 0};
            CK(cudaMemcpyAsync(S.gstat.p, st0, sizeof(st0), cudaMemcpyHostToDevice, st));
        }
        // Iterations are enqueued ahead (kLookAhead per host check); once
        // gk_norm_givens sets stop, every later loop kernel returns at once, so
        // the look-ahead only costs the matvec graphs it launched.
        constexpr int kLookAhead = 4;
        const int* stop = S.gstat.p;
        int* hstat = reinterpret_cast<int*>(hp + static_cast<size_t>(MI + 1) * MIc + 2 * MIc);
        const long long n = S.n;
        const int nbn = blocks_for(n);
        const int pmode = P.identity ? 2 : ((P.fallback || P.k == 0) ? 1 : 0);
        for (int k = 0; k < MI; ++k) {
            const double* vk = S.V.p + static_cast<long long>(k) * n1;
            // z = P^{-1} v_k (z_n deferred), u = y .* z
            if (pmode == 0) {
                launch_k(k_mdot, dim3(nbn), dim3(kRT), 0, st, static_cast<const double*>(P.Z.p), n, P.k, n, 1, vk,
                         static_cast<const double*>(P.y.p), static_cast<const double*>(P.theta.p), P.partial.p, stop);
                launch_k(gk_inner, dim3(1), dim3(1024), sizeof(double) * P.k, st,
                         static_cast<const double*>(P.partial.p), nbn, P.k, static_cast<const double*>(P.Cinv.p),
                         P.inner.p, stop);
                launch_counter() += 2;
            }
            launch_k(gk_precond_out, dim3(nbn), dim3(kRT), pmode == 0 ? sizeof(double) * P.k : 0, st, S.z.p, S.u.p,
                     static_cast<const double*>(S.y.p), vk, static_cast<const double*>(P.y.p),
                     static_cast<const double*>(P.theta.p), static_cast<const double*>(P.Z.p), P.k,
                     static_cast<const double*>(P.inner.p), n, pmode, S.pre_partial.p, stop);
            // w = A z (matvec on u, then the saddle rows; z_n from the partials)
            const int rc = ksvm_nfft_op_apply(S.op, S.u.p, S.kv.p, KSVM_NFFT_DEVICE, st);
            if (rc != KSVM_NFFT_OK) throw std::runtime_error(std::string("saddle apply: ") + ksvm_nfft_last_error());
            launch_k(gk_post, dim3(nbn), dim3(kRT), 0, st, S.w.p, static_cast<const double*>(S.y.p),
                     static_cast<const double*>(S.kv.p), static_cast<const double*>(S.theta.p),
                     static_cast<const double*>(S.z.p), vk, static_cast<const double*>(S.pre_partial.p), nbn,
                     pmode == 2 ? 1 : 0, n, S.partial.p, stop);
            // classical Gram-Schmidt, two passes (w_n finished in the first)
            double* h1 = S.h.p;
            double* h2 = S.h.p + (k + 1);
            launch_k(gk_cgs_first, dim3(nb), dim3(kRT), 0, st, static_cast<const double*>(S.V.p), n1, k + 1, S.w.p,
                     n1, static_cast<const double*>(S.partial.p), nbn, S.partial_rows.p, stop);
            launch_k(k_rows_finish, dim3((k + 1 + 7) / 8), dim3(256), 0, st,
                     static_cast<const double*>(S.partial_rows.p), nb, k + 1, h1, stop);
            launch_k(gk_cgs_combine, dim3(nb), dim3(kRT), 0, st, static_cast<const double*>(S.V.p), n1, k + 1,
                     static_cast<const double*>(h1), S.w.p, n1, 0, S.partial_rows.p, stop);
            launch_k(k_rows_finish, dim3((k + 1 + 7) / 8), dim3(256), 0, st,
                     static_cast<const double*>(S.partial_rows.p), nb, k + 1, h2, stop);
            launch_k(gk_cgs_combine, dim3(nb), dim3(kRT), 0, st, static_cast<const double*>(S.V.p), n1, k + 1,
                     static_cast<const double*>(h2), S.w.p, n1, 1, S.norm_partial.p, stop);
            launch_k(gk_norm_givens, dim3(1), dim3(32), sizeof(double) * (3 * k + 3), st,
                     static_cast<const double*>(S.norm_partial.p), nb,
                     S.scal.p + 1, k, MI, static_cast<const double*>(S.h.p), rhs_norm, tol, S.gH.p, S.gcs.p, S.gsn.p,
                     S.gbeta.p, S.ghist.p, S.gstat.p);
            launch_k(k_scale, dim3(nb), dim3(kRT), 0, st, S.V.p + static_cast<long long>(k + 1) * n1,
                     static_cast<const double*>(S.w.p), n1, static_cast<const double*>(S.scal.p + 1), stop);
            launch_counter() += 9;
            if ((k + 1) % kLookAhead == 0 && k + 1 < MI) {
                CK(cudaGetLastError());  // a failed launch must not read as "not converged"
                CK(cudaMemcpyAsync(hstat, S.gstat.p, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (hstat[0]) break;
            }
        }
        // final state: H, beta, history, counters
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hstat, S.gstat.p, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hp, S.gH.p, sizeof(double) * static_cast<size_t>(MI + 1) * MIc, cudaMemcpyDeviceToHost, st));
        double* hbeta = hp + static_cast<size_t>(MI + 1) * MIc;
        double* hhist = hbeta + MIc;
        CK(cudaMemcpyAsync(hbeta, S.gbeta.p, sizeof(double) * std::min(MI + 1, MIc), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hhist, S.ghist.p, sizeof(double) * MIc, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const int k = hstat[4];
        out.iterations = hstat[1];
        out.converged = hstat[2];
        out.breakdown = hstat[3];
        if (residual_history)
            for (int i = 0; i < out.iterations; ++i) residual_history[i] = hhist[i];
        // u = V_k y_k with the upper-triangular solve, x = P^{-1} u
        if (k > 0) {
            std::vector<double> yk(static_cast<size_t>(k));
            for (int i = k - 1; i >= 0; --i) {
                double sacc = hbeta[i];
                for (int j = i + 1; j < k; ++j) sacc -= hp[static_cast<size_t>(i) * MIc + j] * yk[static_cast<size_t>(j)];
                yk[static_cast<size_t>(i)] = sacc / hp[static_cast<size_t>(i) * MIc + i];
            }
            CK(cudaMemcpyAsync(S.coef.p, yk.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
            launch_k(k_combine_rows, dim3(nb), dim3(kRT), 0, st, S.z.p, static_cast<const double*>(S.V.p), n1, k,
                     static_cast<const double*>(S.coef.p), n1, 1, nostop);
            ++launch_counter();
        } else {
            CK(cudaMemsetAsync(S.z.p, 0, sizeof(double) * n1, st));
        }
        precond_apply_dev(P, S.z.p, S.x.p, st);
        saddle_apply_dev(S, S.x.p, S.ax.p, st);
        norm_into(S.r.p, S.ax.p, S.scal.p + 2, nostop);
        double rr = 0.0;
        CK(cudaMemcpyAsync(&rr, S.scal.p + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
        put_x(S.x.p);
        CK(cudaStreamSynchronize(st));
        out.relative_residual = rr / rhs_norm;
        if (out.relative_residual <= tol) out.converged = 1;
        *stats = out;
    });
}

}  // extern "C"
