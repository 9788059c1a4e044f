// Fixed-grid deterministic reductions over length-n vectors (saddle.cu,
// ipm.cu): kRB blocks of kRT threads, block b owns the indices
// b*kRT + t + q*kRB*kRT, lane butterflies then warps in order, and the
// finishers read the kRB block partials in a fixed lane assignment. The
// summation order depends only on n, so every result is bit-reproducible.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>

namespace ksvm_nfft {

constexpr int kRB = 296;  // reduction blocks (2 x 148 SMs): fixed, so partial sums have a fixed order
constexpr int kRT = 256;  // threads per reduction block

inline int reduce_blocks(long long L) { return static_cast<int>(std::min<long long>(kRB, (L + kRT - 1) / kRT)); }

#define KSVM_FOR_BLOCK_INDEX(i, L) \
    for (long long i = static_cast<long long>(blockIdx.x) * kRT + threadIdx.x; i < (L); i += static_cast<long long>(kRB) * kRT)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Warp sum of p[q * stride] for q < count <= kRB (one warp): every load is
// issued before the adds (fixed lane assignment, fixed order), so a finisher
// costs one L2 round trip instead of one per element.
__device__ __forceinline__ double warp_sum_strided(const double* __restrict__ p, int count, long long stride) {
    constexpr int kPer = (kRB + 31) / 32;
    const int lane = threadIdx.x & 31;
    double v[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int q = lane + 32 * j;
        v[j] = q < count ? p[static_cast<long long>(q) * stride] : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) s += v[j];
    return warp_sum(s);
}

__device__ __forceinline__ double warp_min_strided(const double* __restrict__ p, int count) {
    constexpr int kPer = (kRB + 31) / 32;
    const int lane = threadIdx.x & 31;
    double m = __longlong_as_double(0x7ff0000000000000LL);  // +inf
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int q = lane + 32 * j;
        if (q < count) m = fmin(m, p[q]);
    }
    return warp_min(m);
}

// Block sum of v (every thread of a kRT-thread block) into partial[blockIdx.x].
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

// Block minimum of v into partial[blockIdx.x].
__device__ __forceinline__ void block_min(double v, double* partial) {
    __shared__ double shm[kRT / 32];
    v = warp_min(v);
    if ((threadIdx.x & 31) == 0) shm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = shm[0];
        for (int w = 1; w < kRT / 32; ++w) m = fmin(m, shm[w]);
        partial[blockIdx.x] = m;
    }
}

}  // namespace ksvm_nfft
