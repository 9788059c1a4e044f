// GPU greedy pivoted Cholesky: the reference's
// pivoted_cholesky_impl + pivoted_cholesky_greedy (P:src/low_rank.cpp:25-92)
// on the exact kernel entries the IPM preconditioner factorizes
// (WindowOperator::entry, P:src/pipeline.cpp:103-105; or the ANOVA entry,
// P:src/kernel.cpp:33-48), with the diagonal, the factor and every
// reduction on the device. Each pivot is four short kernels (select, its
// finisher, the new row, its finisher) driven by a device-side state
// {done, r, p, err}, so the host enqueues all `rank` pivots without waiting;
// kernels after the stop/failure point return at once.
//
// Same selection rule as the reference (largest residual diagonal, smallest
// index on ties), same stop rule (max <= err_tol or sum <= err_tol), same
// PSD checks (negative pivot / residual diagonal below -1e-10 max(1, trace)
// -> std::runtime_error) and clamping. Rows are
// (entry(p, j) - sum_{i<r} Z[i][j] Z[i][p]) / sqrt(d_p) like :49-52.
// Differences are rounding only (device exp vs libm, fixed-order sums).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "capi_common.cuh"
#include "launch.cuh"

namespace ksvm_nfft {

void op_entry_view(const ksvm_nfft_op* op, int window, EntryView& v);

namespace {

constexpr int kRB = 296;
constexpr int kRT = 256;

struct PivState {
    int done, r, p, err;  // err: 1 negative pivot, 2 negative residual diagonal
    double trace0, root;
};

struct EntryArgs {
    const double* const* cols;
    const int* wdim;
    const double* wgt;
    const double* ell2;
    int nw;
};

// the arithmetic of kernel_rows_kernel (nfft_kernels.cu)
__device__ __forceinline__ double entry(const EntryArgs& a, long long p, long long j) {
    double sum = 0.0;
    int f = 0;
    for (int l = 0; l < a.nw; ++l) {
        double d2 = 0.0;
        for (int t = 0; t < a.wdim[l]; ++t, ++f) {
            const double diff = a.cols[f][p] - a.cols[f][j];
            d2 += diff * diff;
        }
        const double e = exp(-d2 / a.ell2[l]);
        sum = a.wgt[l] < 0.0 ? e : sum + a.wgt[l] * e;
    }
    return sum;
}

#define KSVM_FOR_OWNED(i, L) \
    for (long long i = static_cast<long long>(blockIdx.x) * kRT + threadIdx.x; i < (L); i += static_cast<long long>(kRB) * kRT)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (value, index): larger value wins, smaller index on ties
__device__ __forceinline__ void argmax_merge(double& v, long long& i, double v2, long long i2) {
    if (v2 > v || (v2 == v && i2 < i)) {
        v = v2;
        i = i2;
    }
}

__device__ __forceinline__ void warp_argmax(double& v, long long& i) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
        argmax_merge(v, i, v2, i2);
    }
}

__global__ void __launch_bounds__(kRT) k_diag_init(EntryArgs a, long long n, double* __restrict__ diag,
                                                   double* __restrict__ psum) {
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[kRT / 32];
    double s = 0.0;
    KSVM_FOR_OWNED(j, n) {
        const double d = entry(a, j, j);
        diag[j] = d;
        s += d;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRT / 32; ++w) t += sh[w];
        psum[blockIdx.x] = t;
    }
}

__global__ void k_init_finish(const double* __restrict__ psum, int nb, PivState* __restrict__ st) {
    pdl_trigger();
    pdl_wait();
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += psum[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) {
        st->done = 0;
        st->r = 0;
        st->p = 0;
        st->err = 0;
        st->trace0 = s;
        st->root = 0.0;
    }
}

// per block: max (smallest index) and sum of the residual diagonal
__global__ void __launch_bounds__(kRT) k_select(const double* __restrict__ diag, long long n,
                                                const PivState* __restrict__ st, double* __restrict__ pmax,
                                                long long* __restrict__ pidx, double* __restrict__ psum) {
    pdl_trigger();
    pdl_wait();
    if (st->done) return;
    __shared__ double sv[kRT / 32], ss[kRT / 32];
    __shared__ long long si[kRT / 32];
    double v = -INFINITY, s = 0.0;
    long long i = n;
    KSVM_FOR_OWNED(j, n) {
        const double d = diag[j];
        argmax_merge(v, i, d, j);
        s += d;
    }
    warp_argmax(v, i);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = v;
        si[threadIdx.x >> 5] = i;
        ss[threadIdx.x >> 5] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bv = sv[0], bs = ss[0];
        long long bi = si[0];
        for (int w = 1; w < kRT / 32; ++w) {
            argmax_merge(bv, bi, sv[w], si[w]);
            bs += ss[w];
        }
        pmax[blockIdx.x] = bv;
        pidx[blockIdx.x] = bi;
        psum[blockIdx.x] = bs;
    }
}

// stop rule, pivot, negative-pivot check (P:src/low_rank.cpp:38-47, 82-84)
__global__ void k_select_finish(const double* __restrict__ pmax, const long long* __restrict__ pidx,
                                const double* __restrict__ psum, int nb, double err_tol,
                                PivState* __restrict__ st) {
    pdl_trigger();
    pdl_wait();
    if (st->done) return;
    double v = -INFINITY, s = 0.0;
    long long i = 0x7fffffffffffffffLL;
    for (int b = threadIdx.x; b < nb; b += 32) {
        argmax_merge(v, i, pmax[b], pidx[b]);
        s += psum[b];
    }
    warp_argmax(v, i);
    s = warp_sum(s);
    if (threadIdx.x != 0) return;
    if (v <= err_tol || s <= err_tol) {
        st->done = 1;
        return;
    }
    const double dp = v;
    if (dp <= 0.0) {
        if (dp < -1e-10 * fmax(1.0, st->trace0)) st->err = 1;
        st->done = 1;
        return;
    }
    st->p = static_cast<int>(i);
    st->root = sqrt(dp);
}

// new row r: Z[r][j] = (entry(p, j) - sum_{i<r} Z[i][j] Z[i][p]) / root,
// diag -= row^2 (block minimum before clamping), clamp at 0
__global__ void __launch_bounds__(kRT) k_row(EntryArgs a, long long n, double* __restrict__ Z,
                                             double* __restrict__ diag, const PivState* __restrict__ st,
                                             double* __restrict__ pmin) {
    extern __shared__ double zp[];
    pdl_trigger();
    pdl_wait();
    if (st->done) return;
    const int r = st->r;
    const long long p = st->p;
    const double root = st->root;
    for (int i = threadIdx.x; i < r; i += blockDim.x) zp[i] = Z[static_cast<long long>(i) * n + p];
    __syncthreads();
    __shared__ double sm[kRT / 32];
    double mn = INFINITY;
    KSVM_FOR_OWNED(j, n) {
        double s = 0.0;
        for (int i = 0; i < r; ++i) s += Z[static_cast<long long>(i) * n + j] * zp[i];
        const double row = (entry(a, p, j) - s) / root;
        Z[static_cast<long long>(r) * n + j] = row;
        const double nd = diag[j] - row * row;
        mn = fmin(mn, nd);
        diag[j] = fmax(nd, 0.0);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = sm[0];
        for (int w = 1; w < kRT / 32; ++w) b = fmin(b, sm[w]);
        pmin[blockIdx.x] = b;
    }
}

// residual-diagonal check, diag[p] = 0, record the pivot (:53-64)
__global__ void k_row_finish(const double* __restrict__ pmin, int nb, double* __restrict__ diag,
                             long long* __restrict__ pivots, PivState* __restrict__ st) {
    pdl_trigger();
    pdl_wait();
    if (st->done) return;
    double mn = INFINITY;
    for (int b = threadIdx.x; b < nb; b += 32) mn = fmin(mn, pmin[b]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (threadIdx.x != 0) return;
    if (mn < -1e-10 * fmax(1.0, st->trace0)) {
        st->err = 2;
        st->done = 1;
        return;
    }
    diag[st->p] = 0.0;
    pivots[st->r] = st->p;
    st->r += 1;
}

__global__ void __launch_bounds__(kRT) k_diag_sum(const double* __restrict__ diag, long long n,
                                                  double* __restrict__ psum) {
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[kRT / 32];
    double s = 0.0;
    KSVM_FOR_OWNED(j, n) s += diag[j];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRT / 32; ++w) t += sh[w];
        psum[blockIdx.x] = t;
    }
}

__global__ void k_sum_finish(const double* __restrict__ psum, int nb, double* __restrict__ out) {
    pdl_trigger();
    pdl_wait();
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += psum[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) *out = fmax(s, 0.0);
}

}  // namespace
}  // namespace ksvm_nfft

using namespace ksvm_nfft;

extern "C" int ksvm_nfft_pivoted_cholesky(const ksvm_nfft_op* op, int window, int rank, double err_tol, double* Z,
                                          int* achieved_rank, double* trace_residual, int64_t* pivots, int ptr_kind,
                                          void* stream) {
    return guarded([&] {
        if (!op || !Z || !achieved_rank || !trace_residual) throw std::invalid_argument("null argument");
        if (rank < 1) throw std::invalid_argument("rank must be >= 1");  // P:src/low_rank.cpp:30
        EntryView v;
        op_entry_view(op, window, v);
        const long long n = v.n;
        rank = static_cast<int>(std::min<long long>(rank, n));
        DeviceGuard dg(v.device);
        std::lock_guard<std::mutex> lk(*v.mu);
        cudaStream_t st = v.stream;
        if (ptr_kind == KSVM_NFFT_DEVICE) {
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, static_cast<cudaStream_t>(stream)));
            CK(cudaStreamWaitEvent(st, ev, 0));
            CK(cudaEventDestroy(ev));
        } else if (ptr_kind != KSVM_NFFT_HOST) {
            throw std::invalid_argument("bad ptr_kind");
        }
        DevBuf<double> dwgt, dell2, diag, pmax, psum, pmin, dZ, trace;
        DevBuf<long long> pidx, dpiv;
        DevBuf<PivState> state;
        dwgt.upload(v.wgt.data(), v.wgt.size(), st);
        dell2.upload(v.ell2.data(), v.ell2.size(), st);
        diag.alloc(static_cast<size_t>(n));
        pmax.alloc(kRB);
        psum.alloc(kRB);
        pmin.alloc(kRB);
        pidx.alloc(kRB);
        dpiv.alloc(static_cast<size_t>(rank));
        state.alloc(1);
        trace.alloc(1);
        double* zd = Z;
        if (ptr_kind == KSVM_NFFT_HOST) {
            dZ.alloc(static_cast<size_t>(rank) * n);
            zd = dZ.p;
        }
        const EntryArgs a{v.cols, v.wdim, dwgt.p, dell2.p, v.nw};
        const int nb = static_cast<int>(std::min<long long>(kRB, (n + kRT - 1) / kRT));
        launch_k(k_diag_init, dim3(nb), dim3(kRT), 0, st, a, n, diag.p, psum.p);
        launch_k(k_init_finish, dim3(1), dim3(32), 0, st, static_cast<const double*>(psum.p), nb, state.p);
        for (int r = 0; r < rank; ++r) {
            launch_k(k_select, dim3(nb), dim3(kRT), 0, st, static_cast<const double*>(diag.p), n,
                     static_cast<const PivState*>(state.p), pmax.p, pidx.p, psum.p);
            launch_k(k_select_finish, dim3(1), dim3(32), 0, st, static_cast<const double*>(pmax.p),
                     static_cast<const long long*>(pidx.p), static_cast<const double*>(psum.p), nb, err_tol, state.p);
            launch_k(k_row, dim3(nb), dim3(kRT), sizeof(double) * rank, st, a, n, zd, diag.p,
                     static_cast<const PivState*>(state.p), pmin.p);
            launch_k(k_row_finish, dim3(1), dim3(32), 0, st, static_cast<const double*>(pmin.p), nb, diag.p, dpiv.p,
                     state.p);
        }
        launch_k(k_diag_sum, dim3(nb), dim3(kRT), 0, st, static_cast<const double*>(diag.p), n, psum.p);
        launch_k(k_sum_finish, dim3(1), dim3(32), 0, st, static_cast<const double*>(psum.p), nb, trace.p);
        launch_counter() += 4 + 4LL * rank;
        CK(cudaGetLastError());
        PivState hs{};
        double htr = 0.0;
        CK(cudaMemcpyAsync(&hs, state.p, sizeof(PivState), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&htr, trace.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hs.err == 1) throw std::runtime_error("pivoted Cholesky: negative pivot, operator not PSD");
        if (hs.err == 2)
            throw std::runtime_error("pivoted Cholesky: negative residual diagonal, operator not PSD");
        if (ptr_kind == KSVM_NFFT_HOST && hs.r > 0)
            CK(cudaMemcpyAsync(Z, dZ.p, sizeof(double) * static_cast<size_t>(hs.r) * n, cudaMemcpyDeviceToHost, st));
        if (pivots && hs.r > 0) {
            std::vector<long long> hp(static_cast<size_t>(hs.r));
            CK(cudaMemcpyAsync(hp.data(), dpiv.p, sizeof(long long) * hs.r, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            for (int r = 0; r < hs.r; ++r) pivots[r] = hp[static_cast<size_t>(r)];
        }
        CK(cudaStreamSynchronize(st));
        if (ptr_kind == KSVM_NFFT_DEVICE) {  // later work on the caller's stream sees Z
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, st));
            CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ev, 0));
            CK(cudaEventDestroy(ev));
        }
        *achieved_rank = hs.r;
        *trace_residual = htr;
    });
}
