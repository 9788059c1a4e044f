// sm_100a kernels of the ANOVA-NFFT matvec y = sum_l eta_l K~_l v
// (reference: P:src/fastsum.cpp:257-296 run_transform, :345-352 window sum).
//
// Per apply, for every window (batched over windows in each launch):
//   spread   adjoint NFFT, sources -> per-item grid patches   (:264-272)
//   reduce   patches -> grid G, fixed order (deterministic, no atomics)
//   conv     G -> H: FFT, spectral multiply, inverse FFT, real part
//            (:273-282), evaluated as the equivalent real separable
//            convolution on the touched sub-grid
//   gather   forward NFFT, H -> per-window output           (:284-295)
//   combine  y = sum_l eta_l out_l in window order          (:345-352)
//
// No global atomics anywhere: every reduction has a fixed order, so two
// applies with the same plan and v are bit-identical
// (P:tests/test_fastsum.cpp:208-215).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "nfft_engine.cuh"

namespace ksvm_nfft {

namespace {

__device__ __forceinline__ int pmod(int a, int M) {
    int r = a % M;
    return r < 0 ? r + M : r;
}

// Truncated-Gaussian window weights of one coordinate
// (P:src/fastsum.cpp:75-78, 222-228): taps o = 0..S-1 sit at grid index
// floor(xM) - m + 1 + o and weigh
//   phi = exp(-(xM - floor(xM) + m - 1 - o)^2 / b) / sqrt(pi b)
//       = [Cw exp(-u^2/b)] * exp(2u/b)^o * exp(-o^2/b),   u = xM - floor(xM) + m - 1,
// i.e. two exp() per coordinate instead of 2m. Returns floor(xM).
template <int S>
__device__ __forceinline__ int window_weights(double x, const DWin& w, double* out) {
    const double xm = x * w.Mf;
    const double fl = floor(xm);
    const double u = (xm - fl) + static_cast<double>(w.m - 1);
    double q = w.Cw * exp(-(u * u) * w.invb);
    const double Q = exp((2.0 * u) * w.invb);
#pragma unroll
    for (int o = 0; o < S; ++o) {
        out[o] = q * w.R[o];
        q *= Q;
    }
    return static_cast<int>(fl);
}

__device__ __forceinline__ int window_weights_rt(double x, const DWin& w, double* out) {
    const double xm = x * w.Mf;
    const double fl = floor(xm);
    const double u = (xm - fl) + static_cast<double>(w.m - 1);
    double q = w.Cw * exp(-(u * u) * w.invb);
    const double Q = exp((2.0 * u) * w.invb);
    for (int o = 0; o < w.S; ++o) {
        out[o] = q * w.R[o];
        q *= Q;
    }
    return static_cast<int>(fl);
}

__device__ __forceinline__ void tile_coords(int tile, int d, int nt, int* t) {
    for (int k = d - 1; k >= 0; --k) {
        t[k] = tile % nt;
        tile /= nt;
    }
}

// Split an item's range over the CTA's warps (contiguous, balanced).
__device__ __forceinline__ void warp_range(const Item& it, int warp, int W, int* b, int* e) {
    const int len = it.end - it.begin;
    const int per = (len + W - 1) / W;
    *b = it.begin + warp * per;
    if (*b > it.end) *b = it.end;
    *e = min(*b + per, it.end);
}

// Per-point staging row (doubles): w0[8] w1[8] w2[8] | cell code (int) | pad.
// 26 doubles = 208 B keeps every double2 slot 16-byte aligned.
constexpr int kSt = 26;

__device__ __forceinline__ int cell_of(const double* st) {
    return *reinterpret_cast<const int*>(st + 24);
}

__device__ __forceinline__ double2 ld2(const double* p) {
    return *reinterpret_cast<const double2*>(p);
}

}  // namespace

// ---------------------------------------------------------------------------
// Spread, d = 3, m = 4 (S = 8): register-blocked per cell.
// Lane L owns the 16 taps (a, b0..b0+1, 0..7) of the cell's 8^3 block with
// a = L/4, b0 = 2 (L%4); consecutive points of one cell accumulate in
// registers and are flushed into the warp's private SMEM patch when the
// cell changes. Points are sorted by cell, so a run of 4 with equal first
// and last cell is one cell: that fast path has no branches and 16
// independent FMA chains. The W private patches are summed in warp order
// and written to the item's global patch.
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(W * 32)
spread3_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                  const DWin* __restrict__ wins, const double* __restrict__ v,
                  double* __restrict__ patches) {
    constexpr int S = 8, TC = 4, PE = TC + S - 1, PV = PE * PE * PE;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* wp = smem + warp * PV;
    double* stage = smem + W * PV + warp * 32 * kSt;

    const Item it = items[blockIdx.x];
    const DPSet& ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    for (int k = lane; k < PV; k += 32) wp[k] = 0.0;
    int tc[3];
    tile_coords(it.tile, 3, wn.ntile, tc);
    const int off0 = wn.cmin + tc[0] * TC, off1 = wn.cmin + tc[1] * TC, off2 = wn.cmin + tc[2] * TC;
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    const int a = lane >> 2, b0 = (lane & 3) << 1;

    double acc0[S], acc1[S];
#pragma unroll
    for (int c = 0; c < S; ++c) acc0[c] = acc1[c] = 0.0;
    int cur = -1;
    __syncwarp();

    auto flush = [&](int cell) {
        const int l0 = cell / (TC * TC), l1 = (cell / TC) % TC, l2 = cell % TC;
        double* dst = wp + ((l0 + a) * PE + l1 + b0) * PE + l2;
#pragma unroll
        for (int c = 0; c < S; ++c) {
            dst[c] += acc0[c];
            dst[PE + c] += acc1[c];
            acc0[c] = 0.0;
            acc1[c] = 0.0;
        }
    };
    auto accumulate = [&](const double* st) {
        const double w0a = st[a];
        const double2 w1 = ld2(st + 8 + b0);
        const double u0 = w0a * w1.x, u1 = w0a * w1.y;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 w2 = ld2(st + 16 + 2 * k);
            acc0[2 * k] = fma(u0, w2.x, acc0[2 * k]);
            acc0[2 * k + 1] = fma(u0, w2.y, acc0[2 * k + 1]);
            acc1[2 * k] = fma(u1, w2.x, acc1[2 * k]);
            acc1[2 * k + 1] = fma(u1, w2.y, acc1[2 * k + 1]);
        }
    };

    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) {
            const int i = base + lane;
            double w[S];
            double* st = stage + lane * kSt;
            const double vi = v[ps.perm[i]];
            const int c0 = window_weights<S>(ps.x[0][i], wn, w) - off0;
#pragma unroll
            for (int o = 0; o < S; ++o) st[o] = w[o] * vi;
            const int c1 = window_weights<S>(ps.x[1][i], wn, w) - off1;
#pragma unroll
            for (int o = 0; o < S; ++o) st[8 + o] = w[o];
            const int c2 = window_weights<S>(ps.x[2][i], wn, w) - off2;
#pragma unroll
            for (int o = 0; o < S; ++o) st[16 + o] = w[o];
            *reinterpret_cast<int*>(st + 24) = (c0 * TC + c1) * TC + c2;
        }
        __syncwarp();
        int p = 0;
        while (p < cnt) {
            const double* st = stage + p * kSt;
            const int cp = cell_of(st);
            if (cp != cur) {
                if (cur >= 0) flush(cur);
                cur = cp;
            }
            if (p + 3 < cnt && cell_of(st + 3 * kSt) == cp) {
                accumulate(st);
                accumulate(st + kSt);
                accumulate(st + 2 * kSt);
                accumulate(st + 3 * kSt);
                p += 4;
            } else {
                accumulate(st);
                p += 1;
            }
        }
        __syncwarp();
    }
    if (cur >= 0) flush(cur);
    __syncthreads();
    double* out = patches + it.patch;
    for (int k = threadIdx.x; k < PV; k += W * 32) {
        double s = smem[k];
#pragma unroll
        for (int q = 1; q < W; ++q) s += smem[q * PV + k];
        out[k] = s;
    }
}

// ---------------------------------------------------------------------------
// Gather, d = 3, m = 4: the tile's 11^3 grid halo sits in SMEM; lane L holds
// the 16 grid values of its taps for the current cell in registers and
// computes a partial for each of 32 consecutive points (4-point same-cell
// fast path, 4 independent chains per point); a transposed butterfly
// (reduce-scatter) leaves point p's sum in lane p.
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(W * 32)
gather3_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                  const DWin* __restrict__ wins) {
    constexpr int S = 8, TC = 4, PE = TC + S - 1, PV = PE * PE * PE;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* halo = smem;
    // PV = 1331 doubles is not a multiple of 2: start the staging area at 1332
    double* stage = smem + (PV + 1) + warp * 32 * kSt;

    const Item it = items[blockIdx.x];
    const DPSet& ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    int tc[3];
    tile_coords(it.tile, 3, wn.ntile, tc);
    const int Lg = wn.Lg;
    for (int k = threadIdx.x; k < PV; k += W * 32) {
        const int n0 = k / (PE * PE), n1 = (k / PE) % PE, n2 = k % PE;
        int g[3] = {tc[0] * TC + n0, tc[1] * TC + n1, tc[2] * TC + n2};
        bool ok = true;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            if (wn.wrap) g[t] = pmod(wn.lo + g[t], wn.M);
            else ok = ok && g[t] < Lg;
        }
        halo[k] = ok ? wn.H[(static_cast<long long>(g[0]) * Lg + g[1]) * Lg + g[2]] : 0.0;
    }
    __syncthreads();

    const int off0 = wn.cmin + tc[0] * TC, off1 = wn.cmin + tc[1] * TC, off2 = wn.cmin + tc[2] * TC;
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    const int a = lane >> 2, b0 = (lane & 3) << 1;
    double h0[S], h1[S];
#pragma unroll
    for (int c = 0; c < S; ++c) h0[c] = h1[c] = 0.0;
    int cur = -1;

    auto reload = [&](int cell) {
        const int l0 = cell / (TC * TC), l1 = (cell / TC) % TC, l2 = cell % TC;
        const double* src = halo + ((l0 + a) * PE + l1 + b0) * PE + l2;
#pragma unroll
        for (int c = 0; c < S; ++c) {
            h0[c] = src[c];
            h1[c] = src[PE + c];
        }
    };
    auto partial = [&](const double* st) {
        double e0 = 0.0, o0 = 0.0, e1 = 0.0, o1 = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 w2 = ld2(st + 16 + 2 * k);
            e0 = fma(h0[2 * k], w2.x, e0);
            o0 = fma(h0[2 * k + 1], w2.y, o0);
            e1 = fma(h1[2 * k], w2.x, e1);
            o1 = fma(h1[2 * k + 1], w2.y, o1);
        }
        const double2 w1 = ld2(st + 8 + b0);
        return st[a] * fma(w1.x, e0 + o0, w1.y * (e1 + o1));
    };

    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) {
            const int i = base + lane;
            double w[S];
            double* st = stage + lane * kSt;
            const int c0 = window_weights<S>(ps.x[0][i], wn, w) - off0;
#pragma unroll
            for (int o = 0; o < S; ++o) st[o] = w[o];
            const int c1 = window_weights<S>(ps.x[1][i], wn, w) - off1;
#pragma unroll
            for (int o = 0; o < S; ++o) st[8 + o] = w[o];
            const int c2 = window_weights<S>(ps.x[2][i], wn, w) - off2;
#pragma unroll
            for (int o = 0; o < S; ++o) st[16 + o] = w[o];
            *reinterpret_cast<int*>(st + 24) = (c0 * TC + c1) * TC + c2;
        }
        __syncwarp();
        double pp[32];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int p0 = 4 * g;
            const double* st = stage + p0 * kSt;
            if (p0 + 3 < cnt && cell_of(st) == cell_of(st + 3 * kSt)) {
                const int cp = cell_of(st);
                if (cp != cur) {
                    cur = cp;
                    reload(cp);
                }
                pp[p0] = partial(st);
                pp[p0 + 1] = partial(st + kSt);
                pp[p0 + 2] = partial(st + 2 * kSt);
                pp[p0 + 3] = partial(st + 3 * kSt);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    pp[p0 + q] = 0.0;
                    if (p0 + q < cnt) {
                        const int cp = cell_of(st + q * kSt);
                        if (cp != cur) {
                            cur = cp;
                            reload(cp);
                        }
                        pp[p0 + q] = partial(st + q * kSt);
                    }
                }
            }
        }
        // transposed butterfly: after the 5 stages lane p holds point p's sum
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
            const bool upper = (lane & s) != 0;
#pragma unroll
            for (int k = 0; k < s; ++k) {
                const double send = upper ? pp[k] : pp[k + s];
                const double keep = upper ? pp[k + s] : pp[k];
                pp[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
            }
        }
        if (lane < cnt) ps.out[ps.perm[base + lane]] = pp[0];
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Generic spread / gather for any d in 1..3 and any m (runtime S <= 16):
// lanes stride over the S^d taps of one point at a time; spread accumulates
// straight into the warp's private SMEM patch.
// ---------------------------------------------------------------------------
constexpr int kStageG = 3 * kMaxSpan + 1;

template <int D>
__global__ void spread_generic_kernel(const Item* __restrict__ items,
                                      const DPSet* __restrict__ psets,
                                      const DWin* __restrict__ wins,
                                      const double* __restrict__ v,
                                      double* __restrict__ patches, int W) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Item it = items[blockIdx.x];
    const DPSet& ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    const int S = wn.S, TC = wn.TC, PE = wn.PE;
    int PV = 1, taps = 1;
    for (int t = 0; t < D; ++t) {
        PV *= PE;
        taps *= S;
    }
    double* wp = smem + warp * PV;
    double* stage = smem + W * PV + warp * 32 * kStageG;
    for (int k = lane; k < PV; k += 32) wp[k] = 0.0;
    int tc[3] = {0, 0, 0};
    tile_coords(it.tile, D, wn.ntile, tc);
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    __syncwarp();
    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) {
            const int i = base + lane;
            double* st = stage + lane * kStageG;
            const double vi = v[ps.perm[i]];
            int code = 0;
            for (int t = 0; t < D; ++t) {
                double w[kMaxSpan];
                const int c = window_weights_rt(ps.x[t][i], wn, w) - wn.cmin - tc[t] * TC;
                for (int o = 0; o < S; ++o) st[t * kMaxSpan + o] = t == 0 ? w[o] * vi : w[o];
                code = code * TC + c;
            }
            st[3 * kMaxSpan] = static_cast<double>(code);
        }
        __syncwarp();
        for (int p = 0; p < cnt; ++p) {
            const double* st = stage + p * kStageG;
            int code = static_cast<int>(st[3 * kMaxSpan]);
            int cl[3] = {0, 0, 0};
            for (int t = D - 1; t >= 0; --t) {
                cl[t] = code % TC;
                code /= TC;
            }
            for (int tap = lane; tap < taps; tap += 32) {
                int r = tap, node = 0;
                double wgt = 1.0;
                int o[3] = {0, 0, 0};
                for (int t = D - 1; t >= 0; --t) {
                    o[t] = r % S;
                    r /= S;
                }
                for (int t = 0; t < D; ++t) {
                    wgt = t == 0 ? st[o[0]] : wgt * st[t * kMaxSpan + o[t]];
                    node = node * PE + cl[t] + o[t];
                }
                wp[node] += wgt;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    double* out = patches + it.patch;
    for (int k = threadIdx.x; k < PV; k += W * 32) {
        double s = smem[k];
        for (int q = 1; q < W; ++q) s += smem[q * PV + k];
        out[k] = s;
    }
}

template <int D>
__global__ void gather_generic_kernel(const Item* __restrict__ items,
                                      const DPSet* __restrict__ psets,
                                      const DWin* __restrict__ wins, int W) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Item it = items[blockIdx.x];
    const DPSet& ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    const int S = wn.S, TC = wn.TC, PE = wn.PE, Lg = wn.Lg;
    int PV = 1, taps = 1;
    for (int t = 0; t < D; ++t) {
        PV *= PE;
        taps *= S;
    }
    double* halo = smem;
    double* stage = smem + PV + warp * 32 * kStageG;
    int tc[3] = {0, 0, 0};
    tile_coords(it.tile, D, wn.ntile, tc);
    for (int k = threadIdx.x; k < PV; k += W * 32) {
        int r = k;
        long long gi = 0;
        bool ok = true;
        int n[3];
        for (int t = D - 1; t >= 0; --t) {
            n[t] = r % PE;
            r /= PE;
        }
        for (int t = 0; t < D; ++t) {
            int g = tc[t] * TC + n[t];
            if (wn.wrap) g = pmod(wn.lo + g, wn.M);
            else ok = ok && g < Lg;
            gi = gi * Lg + g;
        }
        halo[k] = ok ? wn.H[gi] : 0.0;
    }
    __syncthreads();
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) {
            const int i = base + lane;
            double* st = stage + lane * kStageG;
            int code = 0;
            for (int t = 0; t < D; ++t) {
                double w[kMaxSpan];
                const int c = window_weights_rt(ps.x[t][i], wn, w) - wn.cmin - tc[t] * TC;
                for (int o = 0; o < S; ++o) st[t * kMaxSpan + o] = w[o];
                code = code * TC + c;
            }
            st[3 * kMaxSpan] = static_cast<double>(code);
        }
        __syncwarp();
        for (int p = 0; p < cnt; ++p) {
            const double* st = stage + p * kStageG;
            int code = static_cast<int>(st[3 * kMaxSpan]);
            int cl[3] = {0, 0, 0};
            for (int t = D - 1; t >= 0; --t) {
                cl[t] = code % TC;
                code /= TC;
            }
            double part = 0.0;
            for (int tap = lane; tap < taps; tap += 32) {
                int r = tap, node = 0;
                double wgt = 1.0;
                int o[3] = {0, 0, 0};
                for (int t = D - 1; t >= 0; --t) {
                    o[t] = r % S;
                    r /= S;
                }
                for (int t = 0; t < D; ++t) {
                    wgt = t == 0 ? st[o[0]] : wgt * st[t * kMaxSpan + o[t]];
                    node = node * PE + cl[t] + o[t];
                }
                part = fma(halo[node], wgt, part);
            }
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) part += __shfl_xor_sync(0xffffffffu, part, s);
            if (lane == 0) ps.out[ps.perm[base + p]] = part;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Patch reduction: grid node <- sum of every covering item's patch value, in
// (e0, T0, e1, T1, e2, T2, item) order. blockIdx.y = window slot.
// ---------------------------------------------------------------------------
__global__ void reduce_patches_kernel(const DWin* __restrict__ wins, const int* __restrict__ slots,
                                      const double* __restrict__ patches) {
    const DWin& wn = wins[slots[blockIdx.y]];
    const int D = wn.d, Lg = wn.Lg, TC = wn.TC, PE = wn.PE, nt = wn.ntile;
    long long nodes = 1;
    int PV = 1;
    for (int t = 0; t < D; ++t) {
        nodes *= Lg;
        PV *= PE;
    }
    const long long node = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (node >= nodes) return;
    int lg[3] = {0, 0, 0};
    long long r = node;
    for (int t = D - 1; t >= 0; --t) {
        lg[t] = static_cast<int>(r % Lg);
        r /= Lg;
    }
    // candidate (extended index, tile) pairs per dimension
    const int Eext = nt * TC + wn.S - 1;
    int ce[3][16], ct[3][16], nc[3] = {0, 0, 0};
    for (int t = 0; t < D; ++t) {
        int e0 = wn.wrap ? pmod(lg[t] - wn.lo, wn.M) : lg[t];
        for (int e = e0; e < Eext; e += (wn.wrap ? wn.M : Eext)) {
            int tlo = (e - PE + 1 + TC - 1) / TC;  // ceil((e - PE + 1) / TC) for e - PE + 1 >= 0
            if (e - PE + 1 < 0) tlo = 0;
            const int thi = min(e / TC, nt - 1);
            for (int T = tlo; T <= thi && nc[t] < 16; ++T) {
                ce[t][nc[t]] = e;
                ct[t][nc[t]] = T;
                ++nc[t];
            }
        }
    }
    double sum = 0.0;
    if (D == 1) {
        for (int i0 = 0; i0 < nc[0]; ++i0) {
            const int T = ct[0][i0];
            const int off = ce[0][i0] - T * TC;
            for (int k = wn.tile_first[T]; k < wn.tile_first[T + 1]; ++k)
                sum += patches[wn.patch_base + static_cast<long long>(k - wn.item_base) * PV + off];
        }
    } else if (D == 2) {
        for (int i0 = 0; i0 < nc[0]; ++i0)
            for (int i1 = 0; i1 < nc[1]; ++i1) {
                const int T = ct[0][i0] * nt + ct[1][i1];
                const int off = (ce[0][i0] - ct[0][i0] * TC) * PE + ce[1][i1] - ct[1][i1] * TC;
                for (int k = wn.tile_first[T]; k < wn.tile_first[T + 1]; ++k)
                    sum += patches[wn.patch_base + static_cast<long long>(k - wn.item_base) * PV + off];
            }
    } else {
        for (int i0 = 0; i0 < nc[0]; ++i0)
            for (int i1 = 0; i1 < nc[1]; ++i1)
                for (int i2 = 0; i2 < nc[2]; ++i2) {
                    const int T = (ct[0][i0] * nt + ct[1][i1]) * nt + ct[2][i2];
                    const int off = ((ce[0][i0] - ct[0][i0] * TC) * PE + ce[1][i1] - ct[1][i1] * TC) * PE +
                                    ce[2][i2] - ct[2][i2] * TC;
                    for (int k = wn.tile_first[T]; k < wn.tile_first[T + 1]; ++k)
                        sum += patches[wn.patch_base + static_cast<long long>(k - wn.item_base) * PV + off];
                }
    }
    wn.G[node] = sum;
}

// ---------------------------------------------------------------------------
// Grid stage as a real separable convolution. With
// z(r) = sum_{J in I_N} m1[J] e^{2 pi i J r / M} = a(r) + i s(r) the
// reference's  Re( IFFT( mult . FFT(g) ) )  equals  sum_k' g(k') Re(prod_t z(k_t - k'_t)),
//   d=1: H = A g
//   d=2: H = A0 (A1 g) - S0 (S1 g)
//   d=3: H = A0 [A1 A2 g - S1 S2 g] - S0 [A1 S2 g + S1 A2 g]
// stage s works along dimension d-1-s. blockIdx.y = window slot.
// ---------------------------------------------------------------------------
__global__ void conv_stage_kernel(const DWin* __restrict__ wins, const int* __restrict__ slots,
                                  int stage) {
    const DWin& wn = wins[slots[blockIdx.y]];
    const int D = wn.d, Lg = wn.Lg;
    if (stage >= D) return;
    long long nodes = 1;
    for (int t = 0; t < D; ++t) nodes *= Lg;
    const long long node = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (node >= nodes) return;
    const int dim = D - 1 - stage;
    long long stride = 1;
    for (int t = dim + 1; t < D; ++t) stride *= Lg;
    const int i = static_cast<int>((node / stride) % Lg);
    const long long fb = node - static_cast<long long>(i) * stride;
    const double* A = wn.tabA + (Lg - 1 + i);  // A[i][j] = A[-j]
    const double* Sg = wn.tabS + (Lg - 1 + i);
    if (stage == 0) {
        const double* g = wn.G;
        double ya = 0.0, ys = 0.0;
        for (int j = 0; j < Lg; ++j) {
            const double x = g[fb + j * stride];
            ya = fma(A[-j], x, ya);
            ys = fma(Sg[-j], x, ys);
        }
        if (D == 1) {
            wn.H[node] = ya;
        } else {
            wn.T[0][node] = ya;
            wn.T[1][node] = ys;
        }
    } else if (stage == 1 && D == 3) {
        const double* ta = wn.T[0];
        const double* ts = wn.T[1];
        double p = 0.0, q = 0.0;
        for (int j = 0; j < Lg; ++j) {
            const double xa = ta[fb + j * stride], xs = ts[fb + j * stride];
            const double aj = A[-j], sj = Sg[-j];
            p = fma(aj, xa, fma(-sj, xs, p));
            q = fma(aj, xs, fma(sj, xa, q));
        }
        wn.T[2][node] = p;
        wn.T[3][node] = q;
    } else {
        const double* xa = D == 3 ? wn.T[2] : wn.T[0];
        const double* xs = D == 3 ? wn.T[3] : wn.T[1];
        double h = 0.0;
        for (int j = 0; j < Lg; ++j) h = fma(A[-j], xa[fb + j * stride], fma(-Sg[-j], xs[fb + j * stride], h));
        wn.H[node] = h;
    }
}

// y[j] = sum over owned windows (ascending) of eta_l * out_l[j]
// (P:src/fastsum.cpp:346-351: out = 0; out += eta_l * apply_l).
__global__ void combine_kernel(double* __restrict__ y, const double* __restrict__ parts,
                               const double* __restrict__ eta, int P, long long n) {
    for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<long long>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int l = 0; l < P; ++l) acc += eta[l] * parts[static_cast<long long>(l) * n + j];
        y[j] = acc;
    }
}

// Exact kernel rows for the preconditioners (P:src/pipeline.cpp:103-105,
// P:src/kernel.cpp:15-29): out[r, j] = sum_l w_l exp(-||x_p^l - x_j^l||^2 / ell_l^2)
// over the listed windows (raw coordinates, SoA per feature).
__global__ void kernel_rows_kernel(double* __restrict__ out, const long long* __restrict__ rows,
                                   const double* const* __restrict__ cols,
                                   const int* __restrict__ wdim, const double* __restrict__ wgt,
                                   const double* __restrict__ ell2, int nw, long long n) {
    const long long p = rows[blockIdx.y];
    for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<long long>(gridDim.x) * blockDim.x) {
        double sum = 0.0;
        int f = 0;
        for (int l = 0; l < nw; ++l) {
            double d2 = 0.0;
            for (int t = 0; t < wdim[l]; ++t, ++f) {
                const double diff = cols[f][p] - cols[f][j];
                d2 += diff * diff;
            }
            const double e = exp(-d2 / ell2[l]);
            sum = wgt[l] < 0.0 ? e : sum + wgt[l] * e;
        }
        out[static_cast<long long>(blockIdx.y) * n + j] = sum;
    }
}

__global__ void fill_kernel(double* __restrict__ out, double val, long long n) {
    for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<long long>(gridDim.x) * blockDim.x)
        out[j] = val;
}

// ---- plan-time helpers ---------------------------------------------------

// Sort key of each point: tile-major, cell-within-tile minor.
__global__ void cell_keys_kernel(const double* __restrict__ x0, const double* __restrict__ x1,
                                 const double* __restrict__ x2, int d, long long n, double Mf,
                                 int cmin, int ncell, int TC, int ntile,
                                 unsigned* __restrict__ keys, int* __restrict__ idx,
                                 int* __restrict__ bad) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double* xs[3] = {x0, x1, x2};
        unsigned tile = 0, cell = 0;
        for (int t = 0; t < d; ++t) {
            int c = static_cast<int>(floor(xs[t][i] * Mf)) - cmin;
            if (c < 0 || c >= ncell) {
                *bad = 1;
                c = c < 0 ? 0 : ncell - 1;
            }
            tile = tile * ntile + c / TC;
            cell = cell * TC + c % TC;
        }
        unsigned tcd = 1;
        for (int t = 0; t < d; ++t) tcd *= TC;
        keys[i] = tile * tcd + cell;
        idx[i] = static_cast<int>(i);
    }
}

__global__ void permute_kernel(double* __restrict__ dst, const double* __restrict__ src,
                               const int* __restrict__ perm, long long n) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[i] = src[perm[i]];
}

// ---- launchers -----------------------------------------------------------

constexpr int kW3 = 4;  // warps per CTA of the d=3, m=4 kernels

size_t spread3_smem() { return sizeof(double) * (kW3 * 1331 + kW3 * 32 * kSt); }
size_t gather3_smem() { return sizeof(double) * (1332 + kW3 * 32 * kSt); }

int generic_warps(int D, int PE, bool spread) {
    int PV = 1;
    for (int t = 0; t < D; ++t) PV *= PE;
    const size_t budget = 200 * 1024;
    const size_t stage = sizeof(double) * 32 * kStageG;
    const size_t patch = sizeof(double) * PV;
    int W = 8;
    while (W > 1 && (spread ? W * (patch + stage) : patch + W * stage) > budget) --W;
    return W;
}

size_t generic_smem(int D, int PE, int W, bool spread) {
    int PV = 1;
    for (int t = 0; t < D; ++t) PV *= PE;
    return sizeof(double) * ((spread ? W : 1) * PV + W * 32 * kStageG);
}

cudaError_t init_kernel_attributes() {
    cudaError_t e = cudaFuncSetAttribute(spread3_s8_kernel<kW3>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(spread3_smem()));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gather3_s8_kernel<kW3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(gather3_smem()));
    if (e != cudaSuccess) return e;
    const int big = 227 * 1024;
    cudaFuncSetAttribute(spread_generic_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(spread_generic_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(spread_generic_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(gather_generic_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(gather_generic_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    return cudaFuncSetAttribute(gather_generic_kernel<3>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, big);
}

// Launch spread over `nitems` items whose windows all have dimension D and
// span S (fast path for D = 3, S = 8).
void launch_spread(int D, int S, int PE, const Item* items, int nitems, const DPSet* ps,
                   const DWin* wins, const double* v, double* patches, cudaStream_t st) {
    if (nitems == 0) return;
    if (D == 3 && S == 8) {
        spread3_s8_kernel<kW3><<<nitems, kW3 * 32, spread3_smem(), st>>>(items, ps, wins, v, patches);
        return;
    }
    const int W = generic_warps(D, PE, true);
    const size_t sm = generic_smem(D, PE, W, true);
    if (D == 1) spread_generic_kernel<1><<<nitems, W * 32, sm, st>>>(items, ps, wins, v, patches, W);
    else if (D == 2) spread_generic_kernel<2><<<nitems, W * 32, sm, st>>>(items, ps, wins, v, patches, W);
    else spread_generic_kernel<3><<<nitems, W * 32, sm, st>>>(items, ps, wins, v, patches, W);
}

void launch_gather(int D, int S, int PE, const Item* items, int nitems, const DPSet* ps,
                   const DWin* wins, cudaStream_t st) {
    if (nitems == 0) return;
    if (D == 3 && S == 8) {
        gather3_s8_kernel<kW3><<<nitems, kW3 * 32, gather3_smem(), st>>>(items, ps, wins);
        return;
    }
    const int W = generic_warps(D, PE, false);
    const size_t sm = generic_smem(D, PE, W, false);
    if (D == 1) gather_generic_kernel<1><<<nitems, W * 32, sm, st>>>(items, ps, wins, W);
    else if (D == 2) gather_generic_kernel<2><<<nitems, W * 32, sm, st>>>(items, ps, wins, W);
    else gather_generic_kernel<3><<<nitems, W * 32, sm, st>>>(items, ps, wins, W);
}

void launch_reduce(const DWin* wins, const int* slots, int nslots, long long max_nodes,
                   const double* patches, cudaStream_t st) {
    if (nslots == 0) return;
    dim3 grid(static_cast<unsigned>((max_nodes + 255) / 256), nslots);
    reduce_patches_kernel<<<grid, 256, 0, st>>>(wins, slots, patches);
}

void launch_conv(const DWin* wins, const int* slots, int nslots, long long max_nodes, int stage,
                 cudaStream_t st) {
    if (nslots == 0) return;
    dim3 grid(static_cast<unsigned>((max_nodes + 255) / 256), nslots);
    conv_stage_kernel<<<grid, 256, 0, st>>>(wins, slots, stage);
}

void launch_combine(double* y, const double* parts, const double* eta, int P, long long n,
                    cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    combine_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(y, parts, eta, P, n);
}

void launch_kernel_rows(double* out, const long long* rows, int r, const double* const* cols,
                        const int* wdim, const double* wgt, const double* ell2, int nw,
                        long long n, cudaStream_t st) {
    dim3 grid(static_cast<unsigned>(std::min<long long>((n + 255) / 256, 1024)), r);
    kernel_rows_kernel<<<grid, 256, 0, st>>>(out, rows, cols, wdim, wgt, ell2, nw, n);
}

void launch_fill(double* out, double val, long long n, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    fill_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(out, val, n);
}

void launch_cell_keys(const double* x0, const double* x1, const double* x2, int d, long long n,
                      double Mf, int cmin, int ncell, int TC, int ntile, unsigned* keys, int* idx,
                      int* bad, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    cell_keys_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(x0, x1, x2, d, n, Mf, cmin, ncell,
                                                               TC, ntile, keys, idx, bad);
}

void launch_permute(double* dst, const double* src, const int* perm, long long n, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    permute_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(dst, src, perm, n);
}

}  // namespace ksvm_nfft
