// sm_100a kernels of the ANOVA-NFFT matvec y = sum_l eta_l K~_l v
// (reference: P:src/fastsum.cpp:257-296 run_transform, :345-352 window sum).
//
// Per apply, for every window (each launch covers all windows of a class):
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
// (P:tests/test_fastsum.cpp:208-215). Window weights come from per-point
// factors precomputed at plan time (nfft_engine.cuh), so no exp() runs here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "launch.cuh"
#include "nfft_engine.cuh"

namespace ksvm_nfft {

namespace {


__device__ __forceinline__ int pmod(int a, int M) {
    int r = a % M;
    return r < 0 ? r + M : r;
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
    *b = min(it.begin + warp * per, it.end);
    *e = min(*b + per, it.end);
}

__device__ __forceinline__ double2 ld2(const double* p) {
    return *reinterpret_cast<const double2*>(p);
}

// Staged per-point row: w_0[S] (times P, and v for spread) | w_1[S] | w_2[S] | code.
template <int D, int S>
struct Row {
    // (D*S + 2) rounded up to a multiple of 4 doubles: double2 slots stay
    // aligned and rows start 16*odd words apart, so the 4 rows a
    // 16-lane phase reads land in disjoint banks.
    static constexpr int kLen = ((D * S + 2) + 3) & ~3;
};

__device__ __forceinline__ int row_code(const double* st, int D, int S) {
    return *reinterpret_cast<const int*>(st + D * S);
}

// Write the tensor-factor weights of one point into its staging row.
template <int D, int S>
__device__ __forceinline__ void stage_row(double* st, const double* R, double P, const double* Q,
                                          int code) {
#pragma unroll
    for (int t = 0; t < D; ++t) {
        double q = t == 0 ? P : 1.0;
#pragma unroll
        for (int o = 0; o < S; ++o) {
            st[t * S + o] = q * R[o];
            q *= Q[t];
        }
    }
    *reinterpret_cast<int*>(st + D * S) = code;
}

// Power-only staging row: w_t[o] = (P for t = 0) * Q_t^o. The constant factor
// R[o] = exp(-o^2/b) of each tap is applied per cell block instead (spread:
// at flush; it is a fixed product R[a] R[b] R[c] per block node), which
// saves 24 FP64 multiplies per point on the datapath DMMA shares.
template <int D, int S>
__device__ __forceinline__ void stage_pow(double* st, double P, const double* Q, int code) {
#pragma unroll
    for (int t = 0; t < D; ++t) {
        double q = t == 0 ? P : 1.0;
#pragma unroll
        for (int o = 0; o < S; ++o) {
            st[t * S + o] = q;
            q *= Q[t];
        }
    }
    *reinterpret_cast<int*>(st + D * S) = code;
}

// Registers of one prefetched point (software pipeline over 32-point batches).
template <int D>
struct Pref {
    double P = 0.0, Q[3] = {0.0, 0.0, 0.0};
    int code = 0, perm = 0;
    __device__ __forceinline__ void load(const DPSet& ps, int i) {
        const double2* f = reinterpret_cast<const double2*>(ps.F + i);
        const double2 a = __ldg(f);
        P = a.x;
        Q[0] = a.y;
        if (D > 1) {
            const double2 b = __ldg(f + 1);
            Q[1] = b.x;
            Q[2] = b.y;
        }
        const int2 c = __ldg(ps.CP + i);
        code = c.x;
        perm = c.y;
    }
    // same, streamed through L2 evict-first (launch.cuh)
    __device__ __forceinline__ void load(const DPSet& ps, int i, unsigned long long pol) {
        const double2* f = reinterpret_cast<const double2*>(ps.F + i);
        const double2 a = ld_plan(f, pol);
        P = a.x;
        Q[0] = a.y;
        if (D > 1) {
            const double2 b = ld_plan(f + 1, pol);
            Q[1] = b.x;
            Q[2] = b.y;
        }
        const int2 c = ld_plan(ps.CP + i, pol);
        code = c.x;
        perm = c.y;
    }
};

}  // namespace

// Load the (TC+S-1)^d grid halo of a tile into SMEM (wrap / bounds aware).
// PEc/TCc > 0: compile-time patch/tile edge (the m = 4 kernels), so the
// per-element index arithmetic has no runtime divisions.
template <int D, int PEc = 0, int TCc = 0, bool kFoldR = false>
__device__ __forceinline__ void load_halo(double* halo, const DWin& wn, const int* tc, int TCr, int PEr,
                                          int PV, const double* sR = nullptr) {
    const int PE = PEc > 0 ? PEc : PEr, TC = TCc > 0 ? TCc : TCr;
    const int Lg = wn.Lg;
    const bool wrap = wn.wrap != 0;
    long long base = 0;
#pragma unroll
    for (int t = 0; t < D; ++t) base = base * Lg + tc[t] * TC;
    for (int k = threadIdx.x; k < PV; k += blockDim.x) {
        int r = k, n[3] = {0, 0, 0};
#pragma unroll
        for (int t = D - 1; t >= 0; --t) {
            n[t] = r % PE;
            r /= PE;
        }
        if (!wrap) {
            bool ok = true;
            long long off = 0;
#pragma unroll
            for (int t = 0; t < D; ++t) {
                ok = ok && tc[t] * TC + n[t] < Lg;
                off = off * Lg + n[t];
            }
            double h = ok ? __ldcg(wn.H + base + off) : 0.0;
            if (kFoldR) {  // tile-relative window factor R[j0] R[j1] R[j2] (factors_kernel)
#pragma unroll
                for (int t = 0; t < D; ++t) h *= sR[n[t]];
            }
            halo[k] = h;
        } else {
            long long gi = 0;
#pragma unroll
            for (int t = 0; t < D; ++t) gi = gi * Lg + pmod(wn.lo + tc[t] * TC + n[t], wn.M);
            double h = __ldcg(wn.H + gi);
            if (kFoldR) {
#pragma unroll
                for (int t = 0; t < D; ++t) h *= sR[n[t]];
            }
            halo[k] = h;
        }
    }
}

// d = 3, m = 4 halo with the tile-relative factor R[n0] R[n1] R[n2]
// (factors_kernel) folded in. Thread k < PE^2 owns the column (n1, n2) and
// walks n0, so the index arithmetic is per column, not per element.
template <int PE, int TC>
__device__ __forceinline__ void load_halo3_r(double* halo, const DWin& wn, const int* tc, const double* sR) {
    const int k = threadIdx.x;
    if (k >= PE * PE) return;
    const int n1 = k / PE, n2 = k - n1 * PE;
    const int Lg = wn.Lg;
    const long long plane = static_cast<long long>(Lg) * Lg;
    const double r12 = sR[n1] * sR[n2];
    if (!wn.wrap) {
        const int i0 = tc[0] * TC, i1 = tc[1] * TC + n1, i2 = tc[2] * TC + n2;
        const bool ok12 = i1 < Lg && i2 < Lg;
        const double* src = wn.H + (static_cast<long long>(i0) * Lg + i1) * Lg + i2;
#pragma unroll
        for (int n0 = 0; n0 < PE; ++n0) {
            const bool ok = ok12 && i0 + n0 < Lg;
            halo[n0 * PE * PE + k] = ok ? __ldcg(src + n0 * plane) * (r12 * sR[n0]) : 0.0;
        }
    } else {
        const long long o12 = static_cast<long long>(pmod(wn.lo + tc[1] * TC + n1, wn.M)) * Lg +
                              pmod(wn.lo + tc[2] * TC + n2, wn.M);
        int i0 = pmod(wn.lo + tc[0] * TC, wn.M);
#pragma unroll
        for (int n0 = 0; n0 < PE; ++n0) {
            halo[n0 * PE * PE + k] = __ldcg(wn.H + i0 * plane + o12) * (r12 * sR[n0]);
            i0 = i0 + 1 == wn.M ? 0 : i0 + 1;
        }
    }
}

// Transposed butterfly over 32 point partials: afterwards lane p holds the
// full sum of point p (each sum in a fixed order).
__device__ __forceinline__ double butterfly32(double (&pp)[32], int lane) {
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
    return pp[0];
}

// One FP64 tensor-core MMA, D(8x8) += A(8x4) B(4x8) (SASS DMMA.8x8x4). Lane
// l = 4g + t holds A[g][t], B[t][g] and D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// Sum the per-warp patches (fixed warp order) and apply the tile-relative
// factor R[j0] R[j1] R[j2] of node (j0, j1, j2) (factors_kernel). Thread
// k < PE^2 owns the column (j1, j2) and walks j0.
template <int W, int PE>
__device__ __forceinline__ void spread3_epilogue(const double* smem, const DWin& wn, double* out) {
    constexpr int PV = PE * PE * PE;
    if (threadIdx.x >= PE * PE) return;
    const int k = threadIdx.x, n1 = k / PE, n2 = k - n1 * PE;
    const double r12 = wn.R[n1] * wn.R[n2];
#pragma unroll
    for (int n0 = 0; n0 < PE; ++n0) {
        const int e = n0 * PE * PE + k;
        double s = smem[e];
#pragma unroll
        for (int q = 1; q < W; ++q) s += smem[q * PV + e];
        out[e] = s * (r12 * wn.R[n0]);
    }
}

// ===========================================================================
// d = 3, m = 4 (S = 8), dense cells, on the FP64 tensor cores (DMMA.8x8x4).
// The tap weights are powers, w_t[o] = Q_t^o (the per-node factor R[o] is
// applied at flush / halo load), so with b = 4 b1 + b0 the 8^3 block of one
// cell is
//   G[(a, b1), (b0, c)] = sum_p (x_p[a] Y4_p^b1) (Q1_p^b0 z_p[c]),
//   x = P v Q0^a, z = Q2^c, Y4 = Q1^4:
// a 16 x 32 tile whose operands hold 16 + 32 entries per point, 32 of them
// products. (The plain form G[(a,b), c] = sum_p (x[a] w1[b]) z[c] needs 64
// products per point; each DMUL costs 4-6 cycles of the FP64 datapath it
// shares with DMMA, scripts/micro/dmma_interleave.cu, and the split form took
// config 5's spread from 3.77 to 3.26 ms.) Per 4 same-cell points: A tiles
// x, x Y4 (1 DMUL), B tiles z, z Q1, z Q1^2, z Q1^3 (3 DMUL), 2 x 4 = 8 DMMA,
// K = the 4 points. Points are sorted by cell; a group is the run of <= 4
// consecutive points in the current cell (the rest of the group is masked to
// zero and handled next round).
// Lane l = 4g + t: A[g][t] = A-tile entry (a = g, point t), B[t][g] = B-tile
// entry (point t, c = g); accumulator (b1, b0) holds G[a = g][b = 4 b1 + b0]
// [c = 2t..2t+1].
//
// Staging rows are kRow3s = 22 doubles (11 16-byte chunks; 11 is odd, so the
// 8 rows a quarter warp stores land in 8 different chunk slots mod 8 and the
// 128-bit staging stores are bank-conflict free):
// x[8] | z[8] | Q1, Q1^2, Q1^3, Q1^4 | {code, perm}. The run structure of a
// 32-point batch (which points continue the cell of their predecessor) is one
// ballot, so the DMMA loop carries no shared-memory loads of cell codes; a
// batch that lies entirely in the current cell (the common case for dense
// data) runs eight unmasked groups with no control flow.
// ===========================================================================
constexpr int kRow3s = 22;

// Length of the run of same-cell points starting at p: bit q of `same` says
// point q continues the cell of point q - 1.
__device__ __forceinline__ int run_len(unsigned same, int p) {
    const unsigned s = p + 1 < 32 ? (same >> (p + 1)) : 0u;
    return __ffs(~s);  // 1 + number of consecutive set bits above p
}

__device__ __forceinline__ void stage_split3(double* st, double P, const double* Q, int code, int perm) {
    double2* s2 = reinterpret_cast<double2*>(st);
#pragma unroll
    for (int t = 0; t < 2; ++t) {  // x = P Q0^a, z = Q2^c
        const double q = Q[t == 0 ? 0 : 2];
        double q0 = t == 0 ? P : 1.0;
#pragma unroll
        for (int o = 0; o < 8; o += 2) {
            const double q1 = q0 * q;
            s2[(t * 8 + o) >> 1] = make_double2(q0, q1);
            if (o + 2 < 8) q0 = q1 * q;
        }
    }
    const double y2 = Q[1] * Q[1];
    s2[8] = make_double2(Q[1], y2);
    s2[9] = make_double2(y2 * Q[1], y2 * y2);
    *reinterpret_cast<int2*>(st + 20) = make_int2(code, perm);
}

template <int W>
__global__ void __launch_bounds__(W * 32)
spread3_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                   const DWin* __restrict__ wins, const double* __restrict__ v,
                   double* __restrict__ patches) {
    constexpr int PE = 11, PV = PE * PE * PE, RL = kRow3s, B = 32;  // B: points per staging batch
    constexpr unsigned kFull = 0xffffffffu;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    double* wp = smem + warp * PV;
    double* stage = smem + ((W * PV + 1) & ~1) + warp * B * RL;

    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    if (ps.vsrc) v = ps.vsrc;  // exact-duplicate window: per-distinct-point sums of v
    const DWin& wn = wins[ps.win];
    for (int k = lane; k < PV; k += 32) wp[k] = 0.0;
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    Pref<3> pa, pb;  // plan data: prefetched before the dependency wait
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    if (wb + lane < we) pa.load(ps, wb + lane, pol_stream);
    if (wb + B + lane < we) pb.load(ps, wb + B + lane, pol_stream);

    double acc[8][2];  // [4 b1 + b0]
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r][0] = acc[r][1] = 0.0;
    int cur = -1;
    auto flush = [&](int cell) {
        const int l0 = cell >> 4, l1 = (cell >> 2) & 3, l2 = cell & 3;
        double* dst = wp + ((l0 + g) * PE + l1) * PE + l2 + 2 * t;
#pragma unroll
        for (int r = 0; r < 8; ++r) {  // b = r
            dst[r * PE] += acc[r][0];
            dst[r * PE + 1] += acc[r][1];
            acc[r][0] = acc[r][1] = 0.0;
        }
    };
    auto mma8 = [&](double xg, double zg, double2 y12, double2 y34) {
        const double a1 = xg * y34.y, b1 = zg * y12.x, b2 = zg * y12.y, b3 = zg * y34.x;
        dmma(acc[0][0], acc[0][1], xg, zg);
        dmma(acc[1][0], acc[1][1], xg, b1);
        dmma(acc[2][0], acc[2][1], xg, b2);
        dmma(acc[3][0], acc[3][1], xg, b3);
        dmma(acc[4][0], acc[4][1], a1, zg);
        dmma(acc[5][0], acc[5][1], a1, b1);
        dmma(acc[6][0], acc[6][1], a1, b2);
        dmma(acc[7][0], acc[7][1], a1, b3);
    };
    // 4 points p0..p0+3 of the current cell; lanes t >= nv contribute zero
    auto group4 = [&](int p0, int nv) {
        const bool valid = t < nv;
        const double* st = stage + (p0 + (valid ? t : 0)) * RL;
        mma8(valid ? st[g] : 0.0, st[8 + g], ld2(st + 16), ld2(st + 18));
    };
    auto group4f = [&](int p0) {  // unmasked
        const double* st = stage + (p0 + t) * RL;
        mma8(st[g], st[8 + g], ld2(st + 16), ld2(st + 18));
    };

    // software pipeline: per-point factors two batches ahead, v one batch ahead
    double va = 0.0;
    {
        const int i0 = wb + lane;
        pdl_wait();  // v may come from the previous kernel (plan factors above did not)
        v = launder(v);
        if (i0 < we) va = ld_keep(v + pa.perm, pol_keep);
    }
    __syncwarp();
    for (int base = wb; base < we; base += B) {
        const int cnt = min(B, we - base);
        const int code = pa.code;
        if (lane < cnt) stage_split3(stage + lane * RL, pa.P * va, pa.Q, code, 0);
        const int prev = __shfl_up_sync(kFull, code, 1);
        const unsigned same = __ballot_sync(kFull, lane < cnt && code == (lane == 0 ? cur : prev));
        pa = pb;
        if (base + B + lane < we) va = ld_keep(v + pa.perm, pol_keep);
        if (base + 2 * B + lane < we) pb.load(ps, base + 2 * B + lane, pol_stream);
        __syncwarp();
        if (same == kFull) {  // the whole batch continues the current cell
#pragma unroll
            for (int q = 0; q < B / 4; ++q) group4f(4 * q);
        } else {
            int p = 0;
            while (p < cnt) {
                if (!((same >> p) & 1u)) {  // a new cell starts at p
                    if (cur >= 0) flush(cur);
                    cur = __shfl_sync(kFull, code, p);
                }
                int L = run_len(same, p);
                for (; L >= 8; L -= 8, p += 8) {
                    group4f(p);
                    group4f(p + 4);
                }
                if (L >= 4) {
                    group4f(p);
                    p += 4;
                    L -= 4;
                }
                if (L > 0) {
                    group4(p, L);
                    p += L;
                }
            }
        }
        __syncwarp();
    }
    if (cur >= 0) flush(cur);
    __syncthreads();
    spread3_epilogue<W, PE>(smem, wn, patches + it.patch);
}

// ===========================================================================
// d = 3, m = 4 spread for sparse cells (few points per cell): one accumulator
// block per cell COLUMN (l0, l1 fixed, l2 = 0..3; consecutive in the sorted
// order), so the SMEM flush happens once per column instead of once per cell
// and 4-point groups rarely need masking. Eleven 8x8 tiles r = c = 0..10;
// tile rows are b = l1 + g, tile columns a = l0 + n:
//   A[g][t] = w1_t[g] w2_t[r - l2_t]   (zero outside the point's 8 taps)
//   B[t][g] = (P v w0)_t[g]
// The staging row holds w2 pre-shifted into 11 slots (w2p).
// Warp w owns the columns 2w, 2w+1 (l0 = w/2, l1 = 2(w%2) + {0,1}; point
// ranges from the plan's colb table), so its private SMEM sub-patch is only
// the 8 x 9 x 11 footprint of those columns, and 8 warps per CTA fit twice
// per SM. The epilogue adds the sub-patches in warp order.
// ===========================================================================
constexpr int kCol3Row = 28;                 // staging row: w0[8] w1[8] w2p[11] code
constexpr int kCol3Sub = 8 * 9 * 11;         // a x b x c footprint of a warp's two columns

__global__ void __launch_bounds__(kColWarps * 32, 2)
spread3c_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                   const DWin* __restrict__ wins, const double* __restrict__ v,
                   double* __restrict__ patches, const int* __restrict__ colb) {
    constexpr int W = kColWarps, S = 8, PE = 11, RL = kCol3Row, SUB = kCol3Sub;
    constexpr int kW2p = 2 * S, kCode = kW2p + PE;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    double* wp = smem + warp * SUB;
    double* stage = smem + W * SUB + warp * 32 * RL;
    const int l1w = 2 * (warp & 1);  // b offset of this warp's footprint

    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    if (ps.vsrc) v = ps.vsrc;  // exact-duplicate window: per-distinct-point sums of v
    const DWin& wn = wins[ps.win];
    for (int k = lane; k < SUB; k += 32) wp[k] = 0.0;
    const int wb = __ldg(colb + blockIdx.x * kColBounds + 2 * warp);
    const int we = __ldg(colb + blockIdx.x * kColBounds + 2 * warp + 2);
    Pref<3> pa, pb;  // plan data: prefetched before the dependency wait
    if (wb + lane < we) pa.load(ps, wb + lane);
    if (wb + 32 + lane < we) pb.load(ps, wb + 32 + lane);

    double acc[PE][2];
#pragma unroll
    for (int r = 0; r < PE; ++r) acc[r][0] = acc[r][1] = 0.0;
    int cur = -1;
    auto col_of = [&](int p) { return *reinterpret_cast<const int*>(stage + p * RL + kCode) >> 2; };
    auto flush = [&](int col) {  // col = l0 * 4 + l1, l0 = warp / 2
        double* dst = wp + (2 * t * 9 + (col & 3) - l1w + g) * PE;
#pragma unroll
        for (int r = 0; r < PE; ++r) {
            dst[r] += acc[r][0];
            dst[9 * PE + r] += acc[r][1];
            acc[r][0] = acc[r][1] = 0.0;
        }
    };
    auto group = [&](const double* st, bool valid) {
        const double bq = valid ? st[g] : 0.0;
        const double w1g = st[S + g];
        const double2 c01 = ld2(st + kW2p), c23 = ld2(st + kW2p + 2), c45 = ld2(st + kW2p + 4),
                      c67 = ld2(st + kW2p + 6), c89 = ld2(st + kW2p + 8);
        const double c10 = st[kW2p + 10];
        dmma(acc[0][0], acc[0][1], c01.x * w1g, bq);
        dmma(acc[1][0], acc[1][1], c01.y * w1g, bq);
        dmma(acc[2][0], acc[2][1], c23.x * w1g, bq);
        dmma(acc[3][0], acc[3][1], c23.y * w1g, bq);
        dmma(acc[4][0], acc[4][1], c45.x * w1g, bq);
        dmma(acc[5][0], acc[5][1], c45.y * w1g, bq);
        dmma(acc[6][0], acc[6][1], c67.x * w1g, bq);
        dmma(acc[7][0], acc[7][1], c67.y * w1g, bq);
        dmma(acc[8][0], acc[8][1], c89.x * w1g, bq);
        dmma(acc[9][0], acc[9][1], c89.y * w1g, bq);
        dmma(acc[10][0], acc[10][1], c10 * w1g, bq);
    };

    double va = 0.0;
    pdl_wait();  // v may come from the previous kernel (plan factors above did not)
    v = launder(v);
    if (wb + lane < we) va = __ldcg(v + pa.perm);
    __syncwarp();
    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) {
            double* st = stage + lane * RL;
            double q0 = pa.P * va, q1 = 1.0;
#pragma unroll
            for (int o = 0; o < S; ++o) {
                st[o] = q0;
                st[S + o] = q1;
                q0 *= pa.Q[0];
                q1 *= pa.Q[1];
            }
            const int l2 = pa.code & 3;
            double q2 = 1.0;
#pragma unroll
            for (int r = 0; r < PE; ++r) {
                const bool in = r >= l2 && r < l2 + S;
                st[kW2p + r] = in ? q2 : 0.0;
                if (in) q2 *= pa.Q[2];
            }
            *reinterpret_cast<int*>(st + kCode) = pa.code;
        }
        pa = pb;
        if (base + 32 + lane < we) va = __ldcg(v + pa.perm);
        if (base + 64 + lane < we) pb.load(ps, base + 64 + lane);
        __syncwarp();
        int p = 0;
        while (p < cnt) {
            const int cp = col_of(p);
            if (cp != cur) {
                if (cur >= 0) flush(cur);
                cur = cp;
            }
            if (p + 7 < cnt && col_of(p + 7) == cur) {
                group(stage + (p + t) * RL, true);  // 8 points of one column: two unmasked rounds
                group(stage + (p + 4 + t) * RL, true);
                p += 8;
                continue;
            }
            const int q = p + t;
            const bool valid = q < cnt && col_of(q) == cur;
            const int nvalid = __popc(__ballot_sync(0xffffffffu, valid) & 0xFu);
            group(stage + (valid ? q : p) * RL, valid);
            p += nvalid;
        }
        __syncwarp();
    }
    if (cur >= 0) flush(cur);
    __syncthreads();
    // node (n0, n1, n2) = sum over warps w (ascending) whose footprint
    // [w/2, w/2 + 8) x [2(w%2), 2(w%2) + 9) x [0, 11) holds it, times the
    // tile-relative factor R[n0] R[n1] R[n2]
    double* out = patches + it.patch;
    if (threadIdx.x < PE * PE) {
        const int k = threadIdx.x, n1 = k / PE, n2 = k - n1 * PE;
        const double r12 = wn.R[n1] * wn.R[n2];
#pragma unroll
        for (int n0 = 0; n0 < PE; ++n0) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const int a = n0 - (w >> 1), b = n1 - 2 * (w & 1);
                if (a >= 0 && a < 8 && b >= 0 && b < 9) s += smem[w * SUB + (a * 9 + b) * PE + n2];
            }
            out[(n0 * PE + n1) * PE + n2] = s * (r12 * wn.R[n0]);
        }
    }
}

// ===========================================================================
// Dense-cell gather, d = 3, m = 4, split-power form (the default). With
// b = 2 b1 + b0 and Y = Q1:
//   Z[p, (b0, c)] = sum_{(a, b1)} (x_p[a] Y_p^{2 b1}) H[a, 2 b1 + b0, c]
//   y_p           = sum_c z_p[c] (Z[p, (0, c)] + Y_p Z[p, (1, c)])
// M = 8 points, K = 32 (a, b1) in 8 k-steps of 4, N = 16 (b0, c) in two
// tiles = 16 DMMA per 8 points as above, but the A operand has 32 entries
// per point (24 products, 6 DMUL per lane) instead of 64, and the epilogue is
// 5 FP64 instructions per lane. Lane l = 4g + t, k-step s: A[g][t] = x_g[4(s%2) + t]
// Y_g^{2(s/2)}, B[t][g] = H[4(s%2) + t, 2(s/2) + b0, c = g] (16 values per
// lane, reloaded per cell), D(b0) holds Z[point g][(b0, 2t..2t+1)].
// Row: x[8] (P folded) | z[8] | Y^2, Y^4, Y^6, Y | {code, perm}.
// ===========================================================================
template <int W>
__global__ void __launch_bounds__(W * 32, 4)
gather3_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                    const DWin* __restrict__ wins) {
    constexpr int S = 8, TC = 4, PE = TC + S - 1, PV = PE * PE * PE, RL = kRow3s;
    constexpr unsigned kFull = 0xffffffffu;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    double* halo = smem;
    double* stage = smem + ((PV + 1) & ~1) + warp * 32 * RL;

    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    int tc[3];
    tile_coords(it.tile, 3, wn.ntile, tc);
    __shared__ double sR[PE];
    if (threadIdx.x < PE) sR[threadIdx.x] = wn.R[threadIdx.x];
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    Pref<3> pa, pb;
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    if (wb + lane < we) pa.load(ps, wb + lane, pol_stream);
    if (wb + 32 + lane < we) pb.load(ps, wb + 32 + lane, pol_stream);
    __syncthreads();
    pdl_wait();
    load_halo3_r<PE, TC>(halo, *launder(&wn), tc, sR);
    __syncthreads();

    double hb[16];  // [2 s + b0]
#pragma unroll
    for (int k = 0; k < 16; ++k) hb[k] = 0.0;
    int cur = -1;
    auto reload = [&](int cell) {
        const int l0 = cell >> 4, l1 = (cell >> 2) & 3, l2 = cell & 3;
        const double* src = halo + ((l0 + t) * PE + l1) * PE + l2 + g;
#pragma unroll
        for (int k = 0; k < 16; ++k) hb[k] = src[4 * ((k >> 1) & 1) * PE * PE + (2 * (k >> 2) + (k & 1)) * PE];
    };
    // one 8-point round; returns lane (g, t)'s share of point g's sum (c = 2t, 2t+1)
    auto round8 = [&](const double* sg, bool vg) {
        const double xa = vg ? sg[t] : 0.0, xb = vg ? sg[4 + t] : 0.0;
        const double2 y24 = ld2(sg + 16), y6y = ld2(sg + 18);
        const double A[8] = {xa, xb, xa * y24.x, xb * y24.x, xa * y24.y, xb * y24.y, xa * y6y.x, xb * y6y.x};
        double z[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            dmma(z[0][0], z[0][1], A[s], hb[2 * s]);
            dmma(z[1][0], z[1][1], A[s], hb[2 * s + 1]);
        }
        const double2 w2 = ld2(sg + 8 + 2 * t);
        const double e0 = fma(z[0][0], w2.x, z[0][1] * w2.y), e1 = fma(z[1][0], w2.x, z[1][1] * w2.y);
        return fma(y6y.y, e1, e0);
    };
    auto group8 = [&](int p0, int nv) {
        const bool vg = g < nv;
        const double* sg = stage + (p0 + (vg ? g : 0)) * RL;
        double part = round8(sg, vg);
        part += __shfl_xor_sync(kFull, part, 1);
        part += __shfl_xor_sync(kFull, part, 2);
        if (t == 0 && vg) st_keep(ps.out + reinterpret_cast<const int*>(sg + 20)[1], part, pol_keep);
    };
    // a full batch in one cell: four rounds, then one transposed butterfly
    // over t (3 adds instead of 8); lane (g, t) ends with the sum of point
    // 8 j + g, j = 2 (t & 1) + (t >> 1), and all 32 lanes store.
    auto batch32 = [&]() {
        double q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) q[j] = round8(stage + (8 * j + g) * RL, true);
        const bool odd = (t & 1) != 0, hi = (t & 2) != 0;
        const double k0 = (odd ? q[2] : q[0]) + __shfl_xor_sync(kFull, odd ? q[0] : q[2], 1);
        const double k1 = (odd ? q[3] : q[1]) + __shfl_xor_sync(kFull, odd ? q[1] : q[3], 1);
        const double sum = (hi ? k1 : k0) + __shfl_xor_sync(kFull, hi ? k0 : k1, 2);
        const int j = 2 * (t & 1) + (t >> 1);
        st_keep(ps.out + reinterpret_cast<const int*>(stage + (8 * j + g) * RL + 20)[1], sum, pol_keep);
    };

    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        const int code = pa.code;
        if (lane < cnt) {
            double2* s2 = reinterpret_cast<double2*>(stage + lane * RL);
#pragma unroll
            for (int d = 0; d < 2; ++d) {
                const double qd = pa.Q[d == 0 ? 0 : 2];
                double q = d == 0 ? pa.P : 1.0;
#pragma unroll
                for (int o = 0; o < 8; o += 2) {
                    const double q1 = q * qd;
                    s2[(d * 8 + o) >> 1] = make_double2(q, q1);
                    if (o + 2 < 8) q = q1 * qd;
                }
            }
            const double y2 = pa.Q[1] * pa.Q[1], y4 = y2 * y2;
            s2[8] = make_double2(y2, y4);
            s2[9] = make_double2(y4 * y2, pa.Q[1]);
            *reinterpret_cast<int2*>(stage + lane * RL + 20) = make_int2(code, pa.perm);
        }
        const int prev = __shfl_up_sync(kFull, code, 1);
        const unsigned same = __ballot_sync(kFull, lane < cnt && code == (lane == 0 ? cur : prev));
        pa = pb;
        if (base + 64 + lane < we) pb.load(ps, base + 64 + lane, pol_stream);
        __syncwarp();
        if (same == kFull) {
            batch32();
        } else {
            int p = 0;
            while (p < cnt) {
                if (!((same >> p) & 1u)) {
                    cur = __shfl_sync(kFull, code, p);
                    reload(cur);
                }
                for (int L = run_len(same, p); L > 0;) {
                    const int nv = min(L, 8);
                    group8(p, nv);
                    p += nv;
                    L -= nv;
                }
            }
        }
        __syncwarp();
    }
}

// ===========================================================================
// Gather, d = 3, m = 4, sparse cells: CTA (item, l0) handles the cell slab l0
// of a tile, warp w the cell column (l0, l1 = w), whose points are
// consecutive (plan colb table), so every 8-point group is full but the last.
// N = a (8 taps), K = (b, c) over the column's 8 x 11 (b, c) block in 22
// k-steps (k-step j: c = j/2, b = 4(j%2) + t):
//   A[g][t] = P w1_g[b] w2_g[c - l2_g]  (w2 pre-shifted into 11 slots, w2p)
//   B[t][g] = H[l0 + g, l1 + b, c]     (22 values per lane, loaded once)
//   y_p     = sum_a Z[p, a] w0_p[a]
// The slab halo (8 x 11 x 11 nodes, tile-relative R folded in) is loaded once
// per CTA.
// ===========================================================================
__global__ void __launch_bounds__(128, 4)
gather3c_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                   const DWin* __restrict__ wins, const int* __restrict__ colb) {
    constexpr int S = 8, TC = 4, PE = TC + S - 1, SL = S * PE * PE, RL = kCol3Row;
    constexpr int kW2p = 2 * S, kCode = kW2p + PE;  // row: P w0[8] w1[8] w2p[11] code perm
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int l0 = blockIdx.y;
    double* halo = smem;
    double* stage = smem + SL + warp * 32 * RL;

    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    int tc[3];
    tile_coords(it.tile, 3, wn.ntile, tc);
    __shared__ double sR[PE];
    if (threadIdx.x < PE) sR[threadIdx.x] = wn.R[threadIdx.x];
    const int col = 4 * l0 + warp;
    const int wb = __ldg(colb + blockIdx.x * kColBounds + col);
    const int we = __ldg(colb + blockIdx.x * kColBounds + col + 1);
    Pref<3> pa, pb;  // plan data: prefetched before the dependency wait
    if (wb + lane < we) pa.load(ps, wb + lane);
    if (wb + 32 + lane < we) pb.load(ps, wb + 32 + lane);
    __syncthreads();
    pdl_wait();
    if (threadIdx.x < PE * PE) {  // column (n1, n2) of the slab, walking n0 = l0 .. l0 + 7
        const double* __restrict__ Hg = launder(wn.H);  // written by the grid kernels
        const int k = threadIdx.x, n1 = k / PE, n2 = k - n1 * PE;
        const int Lg = wn.Lg;
        const long long plane = static_cast<long long>(Lg) * Lg;
        const double r12 = sR[n1] * sR[n2];
        if (!wn.wrap) {
            const int i0 = tc[0] * TC + l0, i1 = tc[1] * TC + n1, i2 = tc[2] * TC + n2;
            const bool ok12 = i1 < Lg && i2 < Lg;
            const double* src = Hg + (static_cast<long long>(i0) * Lg + i1) * Lg + i2;
#pragma unroll
            for (int a = 0; a < S; ++a) {
                const bool ok = ok12 && i0 + a < Lg;
                halo[a * PE * PE + k] = ok ? __ldcg(src + a * plane) * (r12 * sR[l0 + a]) : 0.0;
            }
        } else {
            const long long o12 = static_cast<long long>(pmod(wn.lo + tc[1] * TC + n1, wn.M)) * Lg +
                                  pmod(wn.lo + tc[2] * TC + n2, wn.M);
            int i0 = pmod(wn.lo + tc[0] * TC + l0, wn.M);
#pragma unroll
            for (int a = 0; a < S; ++a) {
                halo[a * PE * PE + k] = __ldcg(Hg + i0 * plane + o12) * (r12 * sR[l0 + a]);
                i0 = i0 + 1 == wn.M ? 0 : i0 + 1;
            }
        }
    }
    __syncthreads();
    if (wb >= we) return;

    double hb[2 * PE];
    {
        const double* src = halo + g * PE * PE + (warp + t) * PE;
#pragma unroll
        for (int j = 0; j < 2 * PE; ++j) hb[j] = src[(j & 1) * 4 * PE + (j >> 1)];
    }
    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) {
            double* st = stage + lane * RL;
            double q0 = pa.P, q1 = 1.0;
#pragma unroll
            for (int o = 0; o < S; ++o) {
                st[o] = q0;
                st[S + o] = q1;
                q0 *= pa.Q[0];
                q1 *= pa.Q[1];
            }
            const int l2 = pa.code & 3;
            double q2 = 1.0;
#pragma unroll
            for (int r = 0; r < PE; ++r) {
                const bool in = r >= l2 && r < l2 + S;
                st[kW2p + r] = in ? q2 : 0.0;
                if (in) q2 *= pa.Q[2];
            }
            reinterpret_cast<int*>(st + kCode)[1] = pa.perm;
        }
        pa = pb;
        if (base + 64 + lane < we) pb.load(ps, base + 64 + lane);
        __syncwarp();
        for (int p = 0; p < cnt; p += 8) {
            const bool vg = p + g < cnt;
            const double* sg = stage + (vg ? p + g : p) * RL;
            const double u0 = vg ? sg[S + t] : 0.0, u1 = vg ? sg[S + 4 + t] : 0.0;
            const double2 c01 = ld2(sg + kW2p), c23 = ld2(sg + kW2p + 2), c45 = ld2(sg + kW2p + 4),
                          c67 = ld2(sg + kW2p + 6), c89 = ld2(sg + kW2p + 8);
            const double c[PE] = {c01.x, c01.y, c23.x, c23.y, c45.x, c45.y, c67.x, c67.y, c89.x, c89.y,
                                  sg[kW2p + 10]};
            const double2 w0 = ld2(sg + 2 * t);
            double z[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
#pragma unroll
            for (int j = 0; j < 2 * PE; ++j) dmma(z[j & 3][0], z[j & 3][1], c[j >> 1] * ((j & 1) ? u1 : u0), hb[j]);
            const double z0 = (z[0][0] + z[1][0]) + (z[2][0] + z[3][0]);
            const double z1 = (z[0][1] + z[1][1]) + (z[2][1] + z[3][1]);
            double part = fma(z0, w0.x, z1 * w0.y);
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            if (t == 0 && vg) ps.out[reinterpret_cast<const int*>(sg + kCode)[1]] = part;
        }
        __syncwarp();
    }
}

// ===========================================================================
// d = 2, m = 4: lane L owns taps (a, b0), (a, b0+1), a = L/4, b0 = 2 (L%4).
// ===========================================================================
template <int W>
__global__ void __launch_bounds__(W * 32)
spread2_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                  const DWin* __restrict__ wins, const double* __restrict__ v,
                  double* __restrict__ patches) {
    constexpr int D = 2, S = 8, TC = 8, PE = TC + S - 1, PV = PE * PE, RL = Row<D, S>::kLen;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* wp = smem + warp * PV;
    double* stage = smem + ((W * PV + 1) & ~1) + warp * 32 * RL;
    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    if (ps.vsrc) v = ps.vsrc;  // exact-duplicate window: per-distinct-point sums of v
    const DWin& wn = wins[ps.win];
    double R[S];
#pragma unroll
    for (int o = 0; o < S; ++o) R[o] = wn.R[o];
    for (int k = lane; k < PV; k += 32) wp[k] = 0.0;
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    Pref<D> pa, pb;  // plan data: prefetched before the dependency wait
    if (wb + lane < we) pa.load(ps, wb + lane);
    if (wb + 32 + lane < we) pb.load(ps, wb + 32 + lane);
    const int a = lane >> 2, b0 = (lane & 3) << 1;
    double acc0 = 0.0, acc1 = 0.0;
    int cur = -1;
    auto flush = [&](int cell) {
        double* dst = wp + ((cell >> 3) + a) * PE + (cell & 7) + b0;
        dst[0] += acc0;
        dst[1] += acc1;
        acc0 = acc1 = 0.0;
    };
    // software pipeline: per-point factors two batches ahead, v one batch ahead
    double va = 0.0;
    {
        const int i0 = wb + lane;
        pdl_wait();  // v may come from the previous kernel (plan factors above did not)
        v = launder(v);
        if (i0 < we) va = __ldcg(v + pa.perm);
    }
    __syncwarp();
    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) stage_row<D, S>(stage + lane * RL, R, pa.P * va, pa.Q, pa.code);
        pa = pb;
        if (base + 32 + lane < we) va = __ldcg(v + pa.perm);
        if (base + 64 + lane < we) pb.load(ps, base + 64 + lane);
        __syncwarp();
        for (int p = 0; p < cnt; ++p) {
            const double* st = stage + p * RL;
            const int cp = row_code(st, D, S);
            if (cp != cur) {
                if (cur >= 0) flush(cur);
                cur = cp;
            }
            const double u = st[a];
            const double2 w1 = ld2(st + S + b0);
            acc0 = fma(u, w1.x, acc0);
            acc1 = fma(u, w1.y, acc1);
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

template <int W>
__global__ void __launch_bounds__(W * 32)
gather2_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                  const DWin* __restrict__ wins) {
    constexpr int D = 2, S = 8, TC = 8, PE = TC + S - 1, PV = PE * PE, RL = Row<D, S>::kLen;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* halo = smem;
    double* stage = smem + ((PV + 1) & ~1) + warp * 32 * RL;
    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    double R[S];
#pragma unroll
    for (int o = 0; o < S; ++o) R[o] = wn.R[o];
    int tc[3];
    tile_coords(it.tile, D, wn.ntile, tc);
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    Pref<D> pa, pb;  // plan data: prefetched before the dependency wait
    if (wb + lane < we) pa.load(ps, wb + lane);
    if (wb + 32 + lane < we) pb.load(ps, wb + 32 + lane);
    pdl_wait();
    load_halo<D, PE, TC>(halo, *launder(&wn), tc, TC, PE, PV);
    int permc = 0;
    __syncthreads();
    const int a = lane >> 2, b0 = (lane & 3) << 1;
    double h0 = 0.0, h1 = 0.0;
    int cur = -1;
    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) stage_row<D, S>(stage + lane * RL, R, pa.P, pa.Q, pa.code);
        permc = pa.perm;
        pa = pb;
        if (base + 64 + lane < we) pb.load(ps, base + 64 + lane);
        __syncwarp();
        double pp[32];
#pragma unroll
        for (int p = 0; p < 32; ++p) {
            pp[p] = 0.0;
            if (p < cnt) {
                const double* st = stage + p * RL;
                const int cp = row_code(st, D, S);
                if (cp != cur) {
                    cur = cp;
                    const double* src = halo + ((cp >> 3) + a) * PE + (cp & 7) + b0;
                    h0 = src[0];
                    h1 = src[1];
                }
                const double2 w1 = ld2(st + S + b0);
                pp[p] = st[a] * fma(w1.x, h0, w1.y * h1);
            }
        }
        const double val = butterfly32(pp, lane);
        if (lane < cnt) ps.out[permc] = val;
        __syncwarp();
    }
}

// ===========================================================================
// d = 1, m = 4: one lane per point. Spread accumulates into a lane-private
// column of the warp's SMEM patch (node-major, lane-minor), reduced in fixed
// (warp, lane) order at the end.
// ===========================================================================
template <int W>
__global__ void __launch_bounds__(W * 32)
spread1_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                  const DWin* __restrict__ wins, const double* __restrict__ v,
                  double* __restrict__ patches) {
    constexpr int S = 8, TC = 32, PE = TC + S - 1;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* lp = smem + warp * PE * 32;
    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    if (ps.vsrc) v = ps.vsrc;  // exact-duplicate window: per-distinct-point sums of v
    const DWin& wn = wins[ps.win];
    double R[S];
#pragma unroll
    for (int o = 0; o < S; ++o) R[o] = wn.R[o];
    for (int k = lane; k < PE * 32; k += 32) lp[k] = 0.0;
    __syncwarp();
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    // four points per lane in flight: plan loads first, then the dependent
    // v[perm] loads, then the SMEM updates in point order (a lane's points
    // may share a column)
    constexpr int U = 4;
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    pdl_wait();
    v = launder(v);
    for (int base = wb + lane; base < we; base += 32 * U) {
        double2 f[U];
        int2 cp[U];
        double vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = base + 32 * u;
            f[u] = i < we ? ld_plan(reinterpret_cast<const double2*>(ps.F + i), pol_stream) : make_double2(0.0, 0.0);
            cp[u] = i < we ? ld_plan(ps.CP + i, pol_stream) : make_int2(0, -1);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) vv[u] = cp[u].y >= 0 ? ld_keep(v + cp[u].y, pol_keep) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (cp[u].y < 0) break;
            double q = f[u].x * vv[u];
            const double Q = f[u].y;
            double* col = lp + cp[u].x * 32 + lane;
#pragma unroll
            for (int o = 0; o < S; ++o) {
                col[o * 32] = fma(q, R[o], col[o * 32]);
                q *= Q;
            }
        }
    }
    __syncthreads();
    double* out = patches + it.patch;
    for (int k = threadIdx.x; k < PE; k += W * 32) {
        double s = 0.0;
        for (int q = 0; q < W; ++q)
            for (int l = 0; l < 32; ++l) s += smem[q * PE * 32 + k * 32 + l];
        out[k] = s;
    }
}

template <int W>
__global__ void __launch_bounds__(W * 32)
gather1_s8_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                  const DWin* __restrict__ wins) {
    constexpr int D = 1, S = 8, TC = 32, PE = TC + S - 1;
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    double R[S];
#pragma unroll
    for (int o = 0; o < S; ++o) R[o] = wn.R[o];
    int tc[3];
    tile_coords(it.tile, D, wn.ntile, tc);
    pdl_wait();
    load_halo<D, PE, TC>(smem, *launder(&wn), tc, TC, PE, PE);
    __syncthreads();
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    constexpr int U = 4;  // four points per lane in flight
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    for (int base = wb + lane; base < we; base += 32 * U) {
        double2 f[U];
        int2 cp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = base + 32 * u;
            f[u] = i < we ? ld_plan(reinterpret_cast<const double2*>(ps.F + i), pol_stream) : make_double2(0.0, 0.0);
            cp[u] = i < we ? ld_plan(ps.CP + i, pol_stream) : make_int2(0, -1);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double q = f[u].x;
            const double Q = f[u].y;
            const double* h = smem + cp[u].x;
            double y = 0.0;
#pragma unroll
            for (int o = 0; o < S; ++o) {
                y = fma(h[o], q * R[o], y);
                q *= Q;
            }
            if (cp[u].y >= 0) st_keep(ps.out + cp[u].y, y, pol_keep);
        }
    }
}

// ===========================================================================
// Generic spread / gather for any d in 1..3 and any m (runtime S <= 16):
// lanes stride over the S^d taps of one point at a time.
// ===========================================================================
constexpr int kRowG = 3 * kMaxSpan + 2;

template <int D>
__global__ void spread_generic_kernel(const Item* __restrict__ items,
                                      const DPSet* __restrict__ psets,
                                      const DWin* __restrict__ wins,
                                      const double* __restrict__ v,
                                      double* __restrict__ patches, int W) {
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    if (ps.vsrc) v = ps.vsrc;  // exact-duplicate window: per-distinct-point sums of v
    const DWin& wn = wins[ps.win];
    const int S = wn.S, TC = wn.TC, PE = wn.PE;
    int PV = 1, taps = 1;
    for (int t = 0; t < D; ++t) {
        PV *= PE;
        taps *= S;
    }
    double* wp = smem + warp * PV;
    double* stage = smem + ((W * PV + 1) & ~1) + warp * 32 * kRowG;
    for (int k = lane; k < PV; k += 32) wp[k] = 0.0;
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    pdl_wait();
    __syncwarp();
    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) {
            const int i = base + lane;
            double* st = stage + lane * kRowG;
            const double4 f = ps.F[i];
            const double Qs[3] = {f.y, f.z, f.w};
            for (int t = 0; t < D; ++t) {
                double q = t == 0 ? f.x * __ldcg(v + ps.CP[i].y) : 1.0;
                const double Q = Qs[t];
                for (int o = 0; o < S; ++o) {
                    st[t * kMaxSpan + o] = q * wn.R[o];
                    q *= Q;
                }
            }
            *reinterpret_cast<int*>(st + 3 * kMaxSpan) = ps.CP[i].x;
        }
        __syncwarp();
        for (int p = 0; p < cnt; ++p) {
            const double* st = stage + p * kRowG;
            int code = *reinterpret_cast<const int*>(st + 3 * kMaxSpan);
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
    extern __shared__ __align__(16) double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    const int S = wn.S, TC = wn.TC, PE = wn.PE;
    int PV = 1, taps = 1;
    for (int t = 0; t < D; ++t) {
        PV *= PE;
        taps *= S;
    }
    double* halo = smem;
    double* stage = smem + ((PV + 1) & ~1) + warp * 32 * kRowG;
    int tc[3] = {0, 0, 0};
    tile_coords(it.tile, D, wn.ntile, tc);
    pdl_wait();
    load_halo<D>(halo, *launder(&wn), tc, TC, PE, PV);
    __syncthreads();
    int wb, we;
    warp_range(it, warp, W, &wb, &we);
    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        if (lane < cnt) {
            const int i = base + lane;
            double* st = stage + lane * kRowG;
            const double4 f = ps.F[i];
            const double Qs[3] = {f.y, f.z, f.w};
            for (int t = 0; t < D; ++t) {
                double q = t == 0 ? f.x : 1.0;
                const double Q = Qs[t];
                for (int o = 0; o < S; ++o) {
                    st[t * kMaxSpan + o] = q * wn.R[o];
                    q *= Q;
                }
            }
            *reinterpret_cast<int*>(st + 3 * kMaxSpan) = ps.CP[i].x;
        }
        __syncwarp();
        for (int p = 0; p < cnt; ++p) {
            const double* st = stage + p * kRowG;
            int code = *reinterpret_cast<const int*>(st + 3 * kMaxSpan);
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
            if (lane == 0) ps.out[ps.CP[base + p].y] = part;
        }
        __syncwarp();
    }
}

// ===========================================================================
// Tile pre-reduction: for every tile split into several items, sum the
// items' patches (ascending item order) into the tile's first patch, so the
// node reduction below reads one patch per covering tile. Work list:
// (window slot, tile) pairs of multi-item tiles; blockIdx.y = pair.
// ===========================================================================
constexpr int kTrSlices = 4;  // tile_reduce: threads per element (patches k = slice, slice + 4, ...)

__global__ void __launch_bounds__(64 * kTrSlices)
tile_reduce_kernel(const DWin* __restrict__ wins, const int2* __restrict__ multi, double* __restrict__ patches) {
    __shared__ double part[kTrSlices][64];
    pdl_trigger();
    const int2 wt = multi[blockIdx.y];
    const DWin& wn = wins[wt.x];
    int PV = 1;
    for (int t = 0; t < wn.d; ++t) PV *= wn.PE;
    const int k0 = wn.tile_first[wt.y], k1 = wn.tile_first[wt.y + 1];
    double* base = patches + wn.patch_base + static_cast<long long>(k0 - wn.item_base) * PV;
    const int nk = k1 - k0, sl = threadIdx.y;
    pdl_wait();
    base = launder(base);  // patches: written by the spread kernels
    for (int e0 = blockIdx.x * 64; e0 < PV; e0 += gridDim.x * 64) {
        const int e = e0 + threadIdx.x;
        // slice sl sums patches sl, sl + 4, ... in four interleaved partial
        // sums (16 loads in flight per element); slices and partials are
        // combined in a fixed order
        double s[4] = {0, 0, 0, 0};
        if (e < PV) {
            int k = sl;
            for (; k + 3 * kTrSlices < nk; k += 4 * kTrSlices) {
#pragma unroll
                for (int j = 0; j < 4; ++j) s[j] += __ldcg(base + static_cast<long long>(k + j * kTrSlices) * PV + e);
            }
            for (int j = 0; k < nk; k += kTrSlices, ++j) s[j] += __ldcg(base + static_cast<long long>(k) * PV + e);
        }
        part[sl][threadIdx.x] = (s[0] + s[1]) + (s[2] + s[3]);
        __syncthreads();
        if (sl == 0 && e < PV)
            base[e] = (part[0][threadIdx.x] + part[1][threadIdx.x]) + (part[2][threadIdx.x] + part[3][threadIdx.x]);
        __syncthreads();
    }
}

// ===========================================================================
// Patch reduction: grid node <- sum over every covering tile's (pre-reduced)
// patch value, in (e0, T0, e1, T1, e2, T2) order. blockIdx.y = window slot.
// ===========================================================================
template <int D, int NC>
__global__ void reduce_patches_kernel(const DWin* __restrict__ wins, const int* __restrict__ slots,
                                      const double* __restrict__ patches) {
    pdl_trigger();
    const DWin& wn = wins[slots[blockIdx.y]];
    pdl_wait();
    patches = launder(patches);
    if (wn.d != D || !wn.wrap) return;  // non-wrapping grids use reduce_owner_kernel
    const int Lg = wn.Lg, TC = wn.TC, PE = wn.PE, nt = wn.ntile;
    int nodes = 1;
#pragma unroll
    for (int t = 0; t < D; ++t) nodes *= Lg;
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= nodes) return;
    int lg[3] = {0, 0, 0};
    {
        int r = node;
#pragma unroll
        for (int t = D - 1; t >= 0; --t) {
            lg[t] = r % Lg;
            r /= Lg;
        }
    }
    const long long* __restrict__ tp = wn.tile_patch;
    double sum = 0.0;
    if (!wn.wrap) {
        // extended index e = lg; covering tiles T = e/TC - a, a < NC, with e - T TC < PE
        int thi[3] = {0, 0, 0};
#pragma unroll
        for (int t = 0; t < D; ++t) thi[t] = min(lg[t] / TC, nt - 1);
#pragma unroll
        for (int a0 = 0; a0 < NC; ++a0) {
            const int T0 = thi[0] - a0, o0 = lg[0] - T0 * TC;
            if (T0 < 0 || o0 >= PE) continue;
            if constexpr (D == 1) {
                const long long off = tp[T0];
                if (off >= 0) sum += __ldcg(patches + off + o0);
            } else {
#pragma unroll
                for (int a1 = 0; a1 < NC; ++a1) {
                    const int T1 = thi[1] - a1, o1 = lg[1] - T1 * TC;
                    if (T1 < 0 || o1 >= PE) continue;
                    if constexpr (D == 2) {
                        const long long off = tp[T0 * nt + T1];
                        if (off >= 0) sum += __ldcg(patches + off + o0 * PE + o1);
                    } else {
#pragma unroll
                        for (int a2 = 0; a2 < NC; ++a2) {
                            const int T2 = thi[2] - a2, o2 = lg[2] - T2 * TC;
                            if (T2 < 0 || o2 >= PE) continue;
                            const long long off = tp[(T0 * nt + T1) * nt + T2];
                            if (off >= 0) sum += __ldcg(patches + off + (o0 * PE + o1) * PE + o2);
                        }
                    }
                }
            }
        }
    } else {
        // wrapped grid: every extended index e = (lg - lo) mod M + k M
        const int Eext = nt * TC + wn.S - 1;
        int e0s[3] = {0, 0, 0};
#pragma unroll
        for (int t = 0; t < D; ++t) e0s[t] = pmod(lg[t] - wn.lo, wn.M);
#define KSVM_TLO(e) ((e) - PE + 1 <= 0 ? 0 : ((e) - PE + TC) / TC)
#define KSVM_THI(e) min((e) / TC, nt - 1)
        for (int e0 = e0s[0]; e0 < Eext; e0 += wn.M)
            for (int T0 = KSVM_TLO(e0); T0 <= KSVM_THI(e0); ++T0) {
                const int o0 = e0 - T0 * TC;
                if constexpr (D == 1) {
                    const long long off = tp[T0];
                    if (off >= 0) sum += __ldcg(patches + off + o0);
                } else {
                    for (int e1 = e0s[1]; e1 < Eext; e1 += wn.M)
                        for (int T1 = KSVM_TLO(e1); T1 <= KSVM_THI(e1); ++T1) {
                            const int o1 = o0 * PE + e1 - T1 * TC;
                            if constexpr (D == 2) {
                                const long long off = tp[T0 * nt + T1];
                                if (off >= 0) sum += __ldcg(patches + off + o1);
                            } else {
                                for (int e2 = e0s[2]; e2 < Eext; e2 += wn.M)
                                    for (int T2 = KSVM_TLO(e2); T2 <= KSVM_THI(e2); ++T2) {
                                        const long long off = tp[(T0 * nt + T1) * nt + T2];
                                        if (off >= 0) sum += __ldcg(patches + off + o1 * PE + e2 - T2 * TC);
                                    }
                            }
                        }
                }
            }
#undef KSVM_TLO
#undef KSVM_THI
    }
    wn.G[node] = sum;
}

// ===========================================================================
// Grid stage as a real separable convolution. With
// z(r) = sum_{J in I_N} m1[J] e^{2 pi i J r / M} = a(r) + i s(r) the
// reference's  Re( IFFT( mult . FFT(g) ) )  equals  sum_k' g(k') Re(prod_t z(k_t - k'_t)):
//   d=1: H = A g
//   d=2: H = A0 (A1 g) - S0 (S1 g)
//   d=3: H = A0 [A1 A2 g - S1 S2 g] - S0 [A1 S2 g + S1 A2 g]
// Stage s works along dimension d-1-s as a Toeplitz GEMM on the FP64 tensor
// cores: Out[i, f] = sum_j T[i - j] X[j, f] over the Lg^(d-1) fibres f.
// Latency-oriented: one warp per 8x8 output tile (8 rows i x 8 fibres f),
// every operand load of its K = Lg reduction issued up front (no SMEM, no
// block barrier), then a short chain of DMMAs (conv_tile_unit below).
// ===========================================================================
constexpr int kConvMaxL = 128;  // Lg bound (M = sigma N <= 128)

// ===========================================================================
// Grid-side work units (reduce and convolution), shared by the kernels below.
// (A single persistent cooperative kernel running all of them with grid-wide
// barriers was measured slower than separate launches: profiles/README.md.)
// ===========================================================================
namespace {

// Owner-tile block reduction of one tile (whole CTA; one unit per CTA).
// soff/sT: SMEM scratch.
template <int D, int NC>
__device__ void reduce_owner_unit(const DWin& wn, int tileT, const double* __restrict__ patches,
                                  long long* soff, int (*sT)[3], int* any) {
    const int TC = wn.TC, PE = wn.PE, nt = wn.ntile, Lg = wn.Lg;
    const int nown = (Lg + TC - 1) / TC;  // owner blocks per dimension (tiles + halo blocks)
    constexpr int NS = D == 1 ? NC : (D == 2 ? NC * NC : NC * NC * NC);
    int T[3] = {0, 0, 0};
    {
        int r = tileT;
#pragma unroll
        for (int t = D - 1; t >= 0; --t) {
            T[t] = r % nown;
            r /= nown;
        }
    }
    if (threadIdx.x == 0) *any = 0;
    __syncthreads();
    if (threadIdx.x < NS) {
        int r = threadIdx.x, Sx[3] = {0, 0, 0};
        bool ok = true;
        int lin = 0;
#pragma unroll
        for (int t = D - 1; t >= 0; --t) {
            Sx[t] = T[t] - (NC - 1) + r % NC;
            r /= NC;
            ok = ok && Sx[t] >= 0 && Sx[t] < nt;
        }
#pragma unroll
        for (int t = 0; t < D; ++t) lin = lin * nt + min(max(Sx[t], 0), nt - 1);
        const long long off = ok ? wn.tile_patch[lin] : -1;
        soff[threadIdx.x] = off;
#pragma unroll
        for (int t = 0; t < 3; ++t) sT[threadIdx.x][t] = Sx[t];
        if (off >= 0) *any = 1;
    }
    __syncthreads();
    int lo[3] = {0, 0, 0}, len[3] = {1, 1, 1}, nodes = 1;
#pragma unroll
    for (int t = 0; t < D; ++t) {
        lo[t] = T[t] * TC;
        len[t] = max(0, min(lo[t] + TC, Lg) - lo[t]);
        nodes *= len[t];
    }
    const bool have = *any != 0;
    pdl_wait();  // patches come from the spread / tile_reduce kernels
    patches = launder(patches);
    for (int k = threadIdx.x; k < nodes; k += blockDim.x) {
        int r = k, e[3] = {0, 0, 0};
#pragma unroll
        for (int t = D - 1; t >= 0; --t) {
            e[t] = lo[t] + r % len[t];
            r /= len[t];
        }
        double sum = 0.0;
        if (have) {
            // per-dimension offsets into the NC candidate source patches
            int od[3][NC];
            bool vd[3][NC];
#pragma unroll
            for (int t = 0; t < D; ++t)
#pragma unroll
                for (int a = 0; a < NC; ++a) {
                    const int o = e[t] - (T[t] - (NC - 1) + a) * TC;
                    vd[t][a] = o >= 0 && o < PE;
                    od[t][a] = o;
                }
#pragma unroll(NS <= 27 ? NS : 1)
            for (int q = 0; q < NS; ++q) {
                int a[3] = {0, 0, 0}, rq = q;
#pragma unroll
                for (int t = D - 1; t >= 0; --t) {
                    a[t] = rq % NC;
                    rq /= NC;
                }
                bool ok = true;
                int o = 0;
#pragma unroll
                for (int t = 0; t < D; ++t) {
                    ok = ok && vd[t][a[t]];
                    o = o * PE + od[t][a[t]];
                }
                const long long off = soff[q];
                if (ok && off >= 0) sum += __ldcg(patches + off + o);
            }
        }
        long long gi = 0;
#pragma unroll
        for (int t = 0; t < D; ++t) gi = gi * Lg + e[t];
        wn.G[gi] = sum;
    }
}

// One 8x8 output tile of a separable-convolution stage (one warp).
__device__ void conv_tile_unit(const DWin& wn, int stage, int tile) {
    const int D = wn.d, Lg = wn.Lg;
    const int dim = D - 1 - stage;
    int nfib = 1;
    for (int t = 0; t < D - 1; ++t) nfib *= Lg;
    const int Mt = (Lg + 7) >> 3;
    const int mt = tile % Mt, ft = tile / Mt;
    int inner = 1;
    for (int t = dim + 1; t < D; ++t) inner *= Lg;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const double* in0 = stage == 0 ? wn.G : (stage == 1 ? wn.T[0] : (D == 3 ? wn.T[2] : wn.T[0]));
    const double* in1 = stage == 0 ? nullptr : (stage == 1 ? wn.T[1] : (D == 3 ? wn.T[3] : wn.T[1]));
    const bool two_in = stage > 0, mid = stage == 1 && D == 3, first = stage == 0 && D > 1;
    auto fbase = [&](int f) -> long long {
        if (dim == D - 1) return static_cast<long long>(f) * Lg;
        const int outer = f / inner, in = f - outer * inner;
        return static_cast<long long>(outer) * Lg * inner + in;
    };
    const long long jstride = dim == D - 1 ? 1 : inner;
    const int fB = ft * 8 + g;
    const bool fok = fB < nfib;
    const long long bb = fok ? fbase(fB) : 0;
    const int i0 = mt * 8;
    const double* __restrict__ tA = wn.tabA;
    const double* __restrict__ tS = wn.tabS;
    const int KS = (Lg + 3) >> 2;
    pdl_wait();  // G / T come from the reduce / previous stage
    in0 = launder(in0);
    if (in1) in1 = launder(in1);
    double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
    double e00 = 0.0, e01 = 0.0, e10 = 0.0, e11 = 0.0;
#pragma unroll 4
    for (int ks = 0; ks < KS; ++ks) {
        const int j = 4 * ks + t;
        const bool jok = j < Lg && fok;
        const double bx = jok ? __ldcg(in0 + bb + j * jstride) : 0.0;
        const double by = (jok && two_in) ? __ldcg(in1 + bb + j * jstride) : 0.0;
        const int r = i0 + g - j;
        const bool rok = r > -Lg && r < Lg;
        const double a = rok ? __ldg(tA + r + Lg - 1) : 0.0;
        const double sv = rok ? __ldg(tS + r + Lg - 1) : 0.0;
        double& p0 = (ks & 1) ? e00 : d00;
        double& p1 = (ks & 1) ? e01 : d01;
        double& q0 = (ks & 1) ? e10 : d10;
        double& q1 = (ks & 1) ? e11 : d11;
        if (!two_in) {
            dmma(p0, p1, a, bx);
            if (first) dmma(q0, q1, sv, bx);
        } else if (mid) {
            dmma(p0, p1, a, bx);
            dmma(p0, p1, -sv, by);
            dmma(q0, q1, a, by);
            dmma(q0, q1, sv, bx);
        } else {
            dmma(p0, p1, a, bx);
            dmma(p0, p1, -sv, by);
        }
    }
    double* o0;
    double* o1 = nullptr;
    if (stage == 0 && D == 1) {
        o0 = wn.H;
    } else if (stage == 0) {
        o0 = wn.T[0];
        o1 = wn.T[1];
    } else if (mid) {
        o0 = wn.T[2];
        o1 = wn.T[3];
    } else {
        o0 = wn.H;
    }
    const int i = i0 + g;
    if (i >= Lg) return;
    const double r0[2] = {d00 + e00, d01 + e01}, r1[2] = {d10 + e10, d11 + e11};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int f = ft * 8 + 2 * t + e;
        if (f >= nfib) continue;
        const long long ad = fbase(f) + i * jstride;
        o0[ad] = r0[e];
        if (o1) o1[ad] = r1[e];
    }
}

__device__ __forceinline__ int conv_tiles(const DWin& wn) {
    int nfib = 1;
    for (int t = 0; t < wn.d - 1; ++t) nfib *= wn.Lg;
    return ((wn.Lg + 7) >> 3) * ((nfib + 7) >> 3);
}

}  // namespace

// Owner-tile reduction (non-wrapping grids): CTA (T, window) produces the
// grid nodes of its own TC^d block (blocks past the last tile own the halo);
// the <= NC^d source tiles whose patches
// reach it are looked up once into SMEM (reduce_owner_unit).
template <int D, int NC>
__global__ void __launch_bounds__(128)
reduce_owner_kernel(const DWin* __restrict__ wins, const int* __restrict__ slots,
                    const double* __restrict__ patches) {
    pdl_trigger();
    const DWin& wn = wins[slots[blockIdx.y]];
    const int nown = (wn.Lg + wn.TC - 1) / wn.TC;
    int ntd = 1;
    for (int t = 0; t < D; ++t) ntd *= nown;
    if (wn.d != D || wn.wrap || static_cast<int>(blockIdx.x) >= ntd) {
        pdl_wait();
        return;
    }
    constexpr int NS = D == 1 ? NC : (D == 2 ? NC * NC : NC * NC * NC);
    __shared__ long long soff[NS];
    __shared__ int sT[NS][3];
    __shared__ int any;
    reduce_owner_unit<D, NC>(wn, blockIdx.x, patches, soff, sT, &any);
}

__global__ void __launch_bounds__(128)
conv_stage_kernel(const DWin* __restrict__ wins, const int* __restrict__ slots, int stage) {
    pdl_trigger();
    const DWin& wn = wins[slots[blockIdx.y]];
    const int tile = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (stage >= wn.d || tile >= conv_tiles(wn)) {
        pdl_wait();
        return;
    }
    conv_tile_unit(wn, stage, tile);
}

// y[j] = sum over owned windows (ascending) of eta_l * out_l[j]
// (P:src/fastsum.cpp:346-351: out = 0; out += eta_l * apply_l).
// Duplicate-merged windows with <= kSmallBins distinct points read their
// distinct-point outputs from an SMEM table (filled after the wait: the
// gathers write them) through one-byte codes (plan data), so no value load
// waits on a code load from memory.
__global__ void __launch_bounds__(256)
combine_kernel(double* __restrict__ y, const double* const* __restrict__ src,
               const int* const* __restrict__ inv, const uint8_t* const* __restrict__ inv8,
               const int* __restrict__ nu8, const double* __restrict__ eta, int P, long long lo, long long n) {
    constexpr int kMaxP = 64;  // window table staged in SMEM (plan data, before the wait)
    __shared__ const double* s_src[kMaxP];
    __shared__ const int* s_inv[kMaxP];
    __shared__ const uint8_t* s_inv8[kMaxP];
    __shared__ double s_eta[kMaxP];
    __shared__ double s_tab[kMaxP][kSmallBins];
    pdl_trigger();
    __shared__ int s_any;
    const int PS = min(P, kMaxP);
    if (threadIdx.x == 0) s_any = P > kMaxP;
    __syncthreads();
    for (int l = threadIdx.x; l < PS; l += blockDim.x) {
        s_src[l] = src[l];
        s_inv[l] = inv[l];
        s_inv8[l] = inv8[l];
        s_eta[l] = eta[l];
        if (inv[l] || inv8[l]) s_any = 1;
    }
    __syncthreads();
    const bool any_map = s_any != 0;
    pdl_wait();
    if (!any_map) {  // no duplicate-merged window: straight window-order sum
        for (long long j = lo + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
             j += static_cast<long long>(gridDim.x) * blockDim.x) {
            double acc = 0.0;
            for (int l = 0; l < P; ++l) acc += s_eta[l] * __ldcg(s_src[l] + j);
            y[j] = acc;
        }
        return;
    }
    for (int k = threadIdx.x; k < PS * kSmallBins; k += blockDim.x) {
        const int l = k / kSmallBins, u = k - l * kSmallBins;
        if (s_inv8[l] && u < nu8[l]) s_tab[l][u] = __ldcg(s_src[l] + u);  // outputs of this apply's gathers
    }
    __syncthreads();
    for (long long j = lo + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<long long>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
#pragma unroll 4
        for (int l = 0; l < P; ++l) {  // window order; the unrolled windows' loads are in flight together
            double val;
            if (l < kMaxP) {
                const uint8_t* i8 = s_inv8[l];
                const int* iv = s_inv[l];
                if (i8) val = s_tab[l][__ldg(i8 + j)];
                else val = __ldcg(s_src[l] + (iv ? static_cast<long long>(__ldg(iv + j)) : j));
                acc += s_eta[l] * val;
            } else {
                const long long k = inv8[l] ? static_cast<long long>(__ldg(inv8[l] + j))
                                            : (inv[l] ? static_cast<long long>(__ldg(inv[l] + j)) : j);
                acc += eta[l] * __ldcg(src[l] + k);
            }
        }
        y[j] = acc;
    }
}

// Exact-duplicate windows, pass 1: one warp per chunk of <= kSegChunk members
// of one distinct point; fixed lane assignment and butterfly, so the sum is
// bit-reproducible.
__global__ void seg_partial_kernel(const double* __restrict__ v, const int* __restrict__ members,
                                   const int2* __restrict__ chunks, double* __restrict__ partial, int C) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= C) return;
    const int2 ch = chunks[c];
    double s = 0.0;
    for (int i = ch.x + lane; i < ch.y; i += 32) s += __ldcg(v + __ldg(members + i));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) partial[c] = s;
}

// Exact-duplicate windows with <= NB distinct points: CTA (b, q) sums v over
// the fixed point range b into lane-private SMEM bins of window q (one per
// distinct point; no two lanes share a cell, so no atomics), then adds each
// bin over the lanes and the warps in a fixed order. v is streamed once per
// range and the codes are one byte, instead of chasing member lists.
template <int NB>
__global__ void __launch_bounds__(256)
bins_partial_kernel(const double* __restrict__ v, const uint8_t* const* __restrict__ codes, int nwl, long long n,
                    double* __restrict__ partial) {
    constexpr int kW = 8;
    __shared__ double bins[kW][NB][33];
    __shared__ double red[NB][kW];
    pdl_trigger();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long per = (n + gridDim.x - 1) / gridDim.x;
    const long long b0 = static_cast<long long>(blockIdx.x) * per, b1 = min(n, b0 + per);
    const int q = blockIdx.y;
    const uint8_t* __restrict__ cq = codes[q];
#pragma unroll
    for (int u = 0; u < NB; ++u) bins[warp][u][lane] = 0.0;
    pdl_wait();
    v = launder(v);
    long long i = b0 + threadIdx.x;
    for (; i + 3 * blockDim.x < b1; i += 4 * blockDim.x) {  // four elements' loads in flight
        const long long s1 = blockDim.x;
        const uint8_t c0 = __ldg(cq + i), c1 = __ldg(cq + i + s1), c2 = __ldg(cq + i + 2 * s1), c3 = __ldg(cq + i + 3 * s1);
        const double x0 = __ldcg(v + i), x1 = __ldcg(v + i + s1), x2 = __ldcg(v + i + 2 * s1), x3 = __ldcg(v + i + 3 * s1);
        bins[warp][c0][lane] += x0;
        bins[warp][c1][lane] += x1;
        bins[warp][c2][lane] += x2;
        bins[warp][c3][lane] += x3;
    }
    for (; i < b1; i += blockDim.x) bins[warp][__ldg(cq + i)][lane] += __ldcg(v + i);
    __syncwarp();
    if (lane < NB) {
        double s = 0.0;
        for (int l = 0; l < 32; ++l) s += bins[warp][lane][l];
        red[lane][warp] = s;
    }
    __syncthreads();
    if (threadIdx.x < NB) {
        double sum = 0.0;
        for (int w = 0; w < kW; ++w) sum += red[threadIdx.x][w];
        partial[(static_cast<long long>(blockIdx.x) * nwl + q) * NB + threadIdx.x] = sum;
    }
}

// Pass 2 of the register-bin sums: vs[q][u] = sum of the block partials,
// one warp per (window q, distinct point u): fixed lane stride + butterfly.
__global__ void bins_sum_kernel(const double* __restrict__ partial, int nblk, int nwl, int NB,
                                const long long* __restrict__ vs_off, const int* __restrict__ nu,
                                double* __restrict__ vs) {
    pdl_trigger();
    pdl_wait();
    const int q = blockIdx.x, u = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (q >= nwl || u >= nu[q]) return;
    double acc = 0.0;
    for (int b = lane; b < nblk; b += 32) acc += __ldcg(partial + (static_cast<long long>(b) * nwl + q) * NB + u);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) vs[vs_off[q] + u] = acc;
}

// Pass 2: per distinct point (one warp each), its chunk partials with a
// fixed lane stride + butterfly.
__global__ void seg_sum_kernel(const double* __restrict__ partial, const int* __restrict__ seg_cb,
                               double* __restrict__ vs, int U) {
    pdl_trigger();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (u >= U) return;
    const int c0 = seg_cb[u], c1 = seg_cb[u + 1];
    if (c0 == c1) return;  // entry of a register-bin window (bins_sum_kernel)
    double acc = 0.0;
    for (int c = c0 + lane; c < c1; c += 32) acc += __ldcg(partial + c);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) vs[u] = acc;
}

// Exact kernel rows for the preconditioners (P:src/pipeline.cpp:103-105,
// P:src/kernel.cpp:15-29): out[r, j] = sum_l w_l exp(-||x_p^l - x_j^l||^2 / ell_l^2)
// over the listed windows (raw coordinates, SoA per feature); w_l < 0 marks
// the single-window WindowOperator entry (plain exp, no weight).
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
    pdl_trigger();
    pdl_wait();
    for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<long long>(gridDim.x) * blockDim.x)
        out[j] = val;
}

// ---- plan-time kernels ----------------------------------------------------

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

// Window factors of each sorted point (nfft_engine.cuh): {P, Q_t}, {code, perm}.
// tile_rel (d = 3, m = 4 kernels): factors relative to the tile origin node
// instead of the cell's first tap: delta_t = u_t + l_t (l_t = cell offset in
// its tile), P = C^d exp(-sum_t (delta_t^2 - 2 l_t delta_t) / b) (this folds
// Q_t^{l_t}), Q_t = exp(2 delta_t / b). Tap o of the point then weighs
// P prod Q_t^{o_t} R[l_t + o_t], and R[j] = exp(-j^2/b) depends only on the
// tile-relative node j, so the kernels apply it per patch / halo node.
__global__ void factors_kernel(const double* __restrict__ x0, const double* __restrict__ x1,
                               const double* __restrict__ x2, const int* __restrict__ perm, int d,
                               long long n, double Mf, int m, double invb, double Cw, int cmin,
                               int TC, int tile_rel, double4* __restrict__ F, int2* __restrict__ CP) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int src = perm[i];
        const double* xs[3] = {x0, x1, x2};
        double Q[3] = {0.0, 0.0, 0.0};
        double ex = 0.0, pre = 1.0;
        int cd = 0;
        for (int t = 0; t < d; ++t) {
            const double xm = xs[t][src] * Mf;
            const double fl = floor(xm);
            const double u = (xm - fl) + static_cast<double>(m - 1);
            const int l = (static_cast<int>(fl) - cmin) % TC;
            const double dl = tile_rel ? u + l : u;
            ex += tile_rel ? dl * dl - 2.0 * l * dl : dl * dl;
            pre *= Cw;
            Q[t] = exp((2.0 * dl) * invb);
            cd = cd * TC + l;
        }
        F[i] = make_double4(pre * exp(-ex * invb), Q[0], Q[1], Q[2]);
        CP[i] = make_int2(cd, src);
    }
}

// ---- launchers ------------------------------------------------------------

constexpr int kW3 = 4;  // warps per CTA of the d=3, m=4 kernels
static_assert(kW3 * 32 >= 11 * 11, "load_halo3_r / spread3 epilogue: one thread per (n1, n2) column");
constexpr int kW2 = 4;
constexpr int kW1 = 8;

size_t gather3c_smem() { return sizeof(double) * (8 * 121 + 4 * 32 * kCol3Row); }
size_t spread3c_smem() { return sizeof(double) * (kColWarps * (kCol3Sub + 32 * kCol3Row)); }
size_t spread3_smem() { return sizeof(double) * (((kW3 * 1331 + 1) & ~1) + kW3 * 32 * kRow3s); }
size_t gather3_smem() { return sizeof(double) * (1332 + kW3 * 32 * kRow3s); }
size_t spread2_smem() { return sizeof(double) * (((kW2 * 225 + 1) & ~1) + kW2 * 32 * Row<2, 8>::kLen); }
size_t gather2_smem() { return sizeof(double) * (226 + kW2 * 32 * Row<2, 8>::kLen); }
size_t spread1_smem() { return sizeof(double) * (kW1 * 39 * 32); }
size_t gather1_smem() { return sizeof(double) * 40; }

int generic_warps(int D, int PE, bool spread) {
    int PV = 1;
    for (int t = 0; t < D; ++t) PV *= PE;
    const size_t budget = 200 * 1024;
    const size_t stage = sizeof(double) * 32 * kRowG;
    const size_t patch = sizeof(double) * (PV + 2);
    int W = 8;
    while (W > 1 && (spread ? W * (patch + stage) : patch + W * stage) > budget) --W;
    return W;
}

size_t generic_smem(int D, int PE, int W, bool spread) {
    int PV = 1;
    for (int t = 0; t < D; ++t) PV *= PE;
    return sizeof(double) * ((((spread ? W : 1) * PV + 1) & ~1) + W * 32 * kRowG);
}



cudaError_t init_kernel_attributes() {
    cudaError_t e = cudaSuccess;
    auto set = [&](const void* f, size_t bytes) {
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    };
    set(reinterpret_cast<const void*>(spread3_s8_kernel<kW3>), spread3_smem());
    set(reinterpret_cast<const void*>(spread3c_s8_kernel), spread3c_smem());
    set(reinterpret_cast<const void*>(gather3c_s8_kernel), gather3c_smem());
    set(reinterpret_cast<const void*>(gather3_s8_kernel<kW3>), gather3_smem());
    set(reinterpret_cast<const void*>(spread2_s8_kernel<kW2>), spread2_smem());
    set(reinterpret_cast<const void*>(gather2_s8_kernel<kW2>), gather2_smem());
    set(reinterpret_cast<const void*>(spread1_s8_kernel<kW1>), spread1_smem());
    const size_t big = 227 * 1024;
    set(reinterpret_cast<const void*>(spread_generic_kernel<1>), big);
    set(reinterpret_cast<const void*>(spread_generic_kernel<2>), big);
    set(reinterpret_cast<const void*>(spread_generic_kernel<3>), big);
    set(reinterpret_cast<const void*>(gather_generic_kernel<1>), big);
    set(reinterpret_cast<const void*>(gather_generic_kernel<2>), big);
    set(reinterpret_cast<const void*>(gather_generic_kernel<3>), big);
    return e;
}

// Launch spread over `nitems` items whose windows all have dimension D and
// span S (specialised kernels for S = 8, i.e. m = 4).
void launch_spread(int D, int S, int PE, const Item* items, int nitems, const DPSet* ps,
                   const DWin* wins, const double* v, double* patches, const int* colb, cudaStream_t st) {
    if (nitems == 0) return;
    if (S == 8) {
        if (D == 3 && colb)
            launch_k(spread3c_s8_kernel, dim3(nitems), dim3(kColWarps * 32), spread3c_smem(), st, items, ps, wins, v,
                     patches, colb);
        else if (D == 3)
            launch_k(spread3_s8_kernel<kW3>, dim3(nitems), dim3(kW3 * 32), spread3_smem(), st, items, ps, wins, v,
                     patches);
        else if (D == 2)
            launch_k(spread2_s8_kernel<kW2>, dim3(nitems), dim3(kW2 * 32), spread2_smem(), st, items, ps, wins, v, patches);
        else
            launch_k(spread1_s8_kernel<kW1>, dim3(nitems), dim3(kW1 * 32), spread1_smem(), st, items, ps, wins, v, patches);
        return;
    }
    const int W = generic_warps(D, PE, true);
    const size_t sm = generic_smem(D, PE, W, true);
    if (D == 1) launch_k(spread_generic_kernel<1>, dim3(nitems), dim3(W * 32), sm, st, items, ps, wins, v, patches, W);
    else if (D == 2) launch_k(spread_generic_kernel<2>, dim3(nitems), dim3(W * 32), sm, st, items, ps, wins, v, patches, W);
    else launch_k(spread_generic_kernel<3>, dim3(nitems), dim3(W * 32), sm, st, items, ps, wins, v, patches, W);
}

// Sparse d = 3 gather over the spread items (whole tiles) and their column
// bounds: CTA (item, l0 slab).
void launch_gather3c(const Item* items, int nitems, const DPSet* ps, const DWin* wins, const int* colb,
                     cudaStream_t st) {
    if (nitems == 0) return;
    launch_k(gather3c_s8_kernel, dim3(nitems, 4), dim3(128), gather3c_smem(), st, items, ps, wins, colb);
}

void launch_gather(int D, int S, int PE, const Item* items, int nitems, const DPSet* ps,
                   const DWin* wins, cudaStream_t st) {
    if (nitems == 0) return;
    if (S == 8) {
        if (D == 3) launch_k(gather3_s8_kernel<kW3>, dim3(nitems), dim3(kW3 * 32), gather3_smem(), st, items, ps, wins);
        else if (D == 2) launch_k(gather2_s8_kernel<kW2>, dim3(nitems), dim3(kW2 * 32), gather2_smem(), st, items, ps, wins);
        else launch_k(gather1_s8_kernel<kW1>, dim3(nitems), dim3(kW1 * 32), gather1_smem(), st, items, ps, wins);
        return;
    }
    const int W = generic_warps(D, PE, false);
    const size_t sm = generic_smem(D, PE, W, false);
    if (D == 1) launch_k(gather_generic_kernel<1>, dim3(nitems), dim3(W * 32), sm, st, items, ps, wins, W);
    else if (D == 2) launch_k(gather_generic_kernel<2>, dim3(nitems), dim3(W * 32), sm, st, items, ps, wins, W);
    else launch_k(gather_generic_kernel<3>, dim3(nitems), dim3(W * 32), sm, st, items, ps, wins, W);
}

void launch_tile_reduce(const DWin* wins, const int2* multi, int nmulti, int max_pv, double* patches,
                        cudaStream_t st) {
    if (nmulti == 0) return;
    // narrow blocks (64 elements x 4 patch slices): one heavy tile's patches are read by ~max_pv/64 SMs
    dim3 grid(static_cast<unsigned>((max_pv + 63) / 64), static_cast<unsigned>(nmulti));
    launch_k(tile_reduce_kernel, dim3(grid), dim3(64, kTrSlices), 0, st, wins, multi, patches);
}

void launch_reduce(const DWin* wins, const int* slots, int nslots, long long max_nodes, int D, int S,
                   const double* patches, bool wrap, int max_tiles, cudaStream_t st) {
    if (nslots == 0) return;
    if (!wrap) {
        // owner-tile blocks; NC = ceil(PE / TC) source tiles per dimension
        dim3 grid(static_cast<unsigned>(max_tiles), nslots);
        if (S == 8) {
            if (D == 1) launch_k(reduce_owner_kernel<1, 2>, dim3(grid), dim3(64), 0, st, wins, slots, patches);
            else if (D == 2) launch_k(reduce_owner_kernel<2, 2>, dim3(grid), dim3(64), 0, st, wins, slots, patches);
            else launch_k(reduce_owner_kernel<3, 3>, dim3(grid), dim3(64), 0, st, wins, slots, patches);
        } else {
            if (D == 1) launch_k(reduce_owner_kernel<1, 5>, dim3(grid), dim3(64), 0, st, wins, slots, patches);
            else if (D == 2) launch_k(reduce_owner_kernel<2, 5>, dim3(grid), dim3(64), 0, st, wins, slots, patches);
            else launch_k(reduce_owner_kernel<3, 5>, dim3(grid), dim3(128), 0, st, wins, slots, patches);
        }
        return;
    }
    dim3 grid(static_cast<unsigned>((max_nodes + 255) / 256), nslots);
    if (D == 1) launch_k(reduce_patches_kernel<1, 5>, dim3(grid), dim3(256), 0, st, wins, slots, patches);
    else if (D == 2) launch_k(reduce_patches_kernel<2, 5>, dim3(grid), dim3(256), 0, st, wins, slots, patches);
    else if (S == 8) launch_k(reduce_patches_kernel<3, 3>, dim3(grid), dim3(256), 0, st, wins, slots, patches);
    else launch_k(reduce_patches_kernel<3, 5>, dim3(grid), dim3(256), 0, st, wins, slots, patches);
}

void launch_conv(const DWin* wins, const int* slots, int nslots, int Lg_max, long long max_fibres,
                 int stage, cudaStream_t st) {
    if (nslots == 0) return;
    const long long tiles = static_cast<long long>((Lg_max + 7) / 8) * ((max_fibres + 7) / 8);
    dim3 grid(static_cast<unsigned>((tiles + 3) / 4), nslots);
    launch_k(conv_stage_kernel, dim3(grid), dim3(128), 0, st, wins, slots, stage);
}

int conv_max_lg() { return kConvMaxL; }

// y[j] = sum_l eta_l out_l[j] for j in [lo, hi) (the whole vector: lo = 0, hi = n)
void launch_combine(double* y, const double* const* src, const int* const* inv, const uint8_t* const* inv8,
                    const int* nu8, const double* eta, int P, long long lo, long long hi, cudaStream_t st) {
    const long long len = hi - lo;
    const int blocks = static_cast<int>(std::min<long long>((len + 255) / 256, 148LL * 16));
    launch_k(combine_kernel, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, st, y, src, inv, inv8, nu8, eta, P, lo,
             hi);
}

void launch_bin_sums(const double* v, const uint8_t* const* codes, int nwl, long long n, double* partial,
                     int nblk, const long long* vs_off, const int* nu, double* vs, cudaStream_t st) {
    if (nwl == 0) return;
    launch_k(bins_partial_kernel<kSmallBins>, dim3(nblk, nwl), dim3(256), 0, st, v, codes, nwl, n, partial);
    launch_k(bins_sum_kernel, dim3(nwl), dim3(32 * kSmallBins), 0, st, static_cast<const double*>(partial), nblk,
             nwl, kSmallBins, vs_off, nu, vs);
}

void launch_seg_sums(const double* v, const int* members, const int2* chunks, double* partial, int C,
                     const int* seg_cb, double* vs, int U, cudaStream_t st) {
    if (C == 0) return;
    launch_k(seg_partial_kernel, dim3((C + 7) / 8), dim3(256), 0, st, v, members, chunks, partial, C);
    launch_k(seg_sum_kernel, dim3((U + 7) / 8), dim3(256), 0, st, static_cast<const double*>(partial), seg_cb, vs, U);
}

void launch_kernel_rows(double* out, const long long* rows, int r, const double* const* cols,
                        const int* wdim, const double* wgt, const double* ell2, int nw,
                        long long n, cudaStream_t st) {
    dim3 grid(static_cast<unsigned>(std::min<long long>((n + 255) / 256, 1024)), r);
    kernel_rows_kernel<<<grid, 256, 0, st>>>(out, rows, cols, wdim, wgt, ell2, nw, n);
}

void launch_fill(double* out, double val, long long n, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    launch_k(fill_kernel, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, st, out, val, n);
}

void launch_cell_keys(const double* x0, const double* x1, const double* x2, int d, long long n,
                      double Mf, int cmin, int ncell, int TC, int ntile, unsigned* keys, int* idx,
                      int* bad, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    cell_keys_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(x0, x1, x2, d, n, Mf, cmin, ncell,
                                                               TC, ntile, keys, idx, bad);
}

void launch_factors(const double* x0, const double* x1, const double* x2, const int* perm, int d,
                    long long n, double Mf, int m, double invb, double Cw, int cmin, int TC,
                    int tile_rel, double4* F, int2* CP, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    factors_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(x0, x1, x2, perm, d, n, Mf, m, invb, Cw,
                                                             cmin, TC, tile_rel, F, CP);
}

}  // namespace ksvm_nfft
