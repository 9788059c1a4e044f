// Optional fp32 mode of the d = 3, m = 4 spread / gather (north_star:
// "<= 1e-5 in an optional fp32 mode"; the same operator as
// P:src/fastsum.cpp:257-296, computed with fp32 window weights and fp32
// FFMA accumulation on the CUDA cores).
//
// Two kernel pairs. The default runs on the warp-level tensor path with
// 3xTF32 splitting (spread3_t32 / gather3_t32 below): tf32 keeps 11
// significant bits, so every operand is split x = hi + lo (hi = x with the
// low 13 mantissa bits cleared, lo = x - hi, exact) and a product is
// lo*hi + hi*lo + hi*hi on HMMA.1688.F32.TF32 with fp32 accumulation
// (mma.sync: 8.6 cycles per m16n8k8 per SM sub-partition on B200, 277
// TFLOP/s, scripts/micro/mma_legacy_rates.cu; there is no tcgen05 route for
// an M = 16, N = 8 tile that changes operands every 8 points). The operands
// use the split-power form of the fp64 kernels (nfft_kernels.cu): 32 operand
// products per point. KSVM_NFFT_F32K=ffma selects the CUDA-core pair
// (spread3_f32 / gather3_f32: fp32 weights, scalar FFMA at 128 FMA/clk/SM).
// The grid side (node reduction, separable convolution) and the window sum
// stay fp64: they are a few percent of the work. Inputs (v) and outputs
// (per-window results, y) stay fp64, so the C ABI does not change.
//
// Window factors (factors32_kernel) are relative to the CELL CENTRE
// (u' = x M - floor(x M) - 1/2 in [-1/2, 1/2), u = u' + m - 1/2):
//   w_t[o] = C e^{-(u_t - o)^2/b} = P_t Q_t^o R[o],
//   P = C^3 e^{-sum_t (u'_t^2 + (2m-1) u'_t)/b},  Q_t = e^{2 u'_t/b},  R[o] = e^{-(o - m + 1/2)^2/b},
// so Q is in [0.55, 1.8] and every power and operand product stays within a
// few decades of 1 (the fp64 kernels' tile-relative factors would leave the
// fp32 range). A plan stores {P, Q0, Q1, Q2} as float4 (16 B per point
// instead of 32 B).
//
// Decomposition (FFMA pair): a CTA is one item (a 4^3-cell tile's point
// range), W warps, and every warp runs two independent half-warp streams in
// lockstep. A half-warp processes one point per step; its lane (a, bq)
// (a = 0..7, bq = 0 or 4) owns the 32 taps (a, bq..bq+3, 0..7) of the
// current cell's 8^3 block: 4 FMUL + 32 FFMA per point per lane. The spread
// keeps the block in registers until the cell changes and then adds it into
// the half-warp's private SMEM patch (11^3 floats; no atomics, fixed order);
// the epilogue adds the 2W half patches in a fixed order in fp64. The gather
// keeps the cell's 32 halo values per lane in registers and reduces the 16
// lane partials of 16 points with one transposed butterfly per batch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "launch.cuh"
#include "nfft_engine.cuh"

namespace ksvm_nfft {

namespace {

constexpr int kW3f = 4;        // warps per CTA
constexpr int kHalfRows = 16;  // points per half-warp per batch
// Staging rows (floats): w0[8] w1[8] w2[8] code perm pad pad. 28 floats =
// 7 16-byte chunks (odd), so the 8 rows a quarter-warp stores hit distinct
// bank groups; +8 floats between the two halves' rows keeps their w0[a]
// reads in disjoint banks.
constexpr int kRowS = 28;
constexpr int kRowG = 28;
constexpr int kPEf = 11, kPVf = kPEf * kPEf * kPEf;
constexpr int kHP = kPVf + 1;  // patch / halo stride (floats), 16-byte multiple

__device__ __forceinline__ int half_stage(int row_len) { return kHalfRows * row_len + 8; }

struct PrefF {
    float4 F = make_float4(0.f, 0.f, 0.f, 0.f);
    int code = 0, perm = 0;
    __device__ __forceinline__ void load(const DPSet& ps, int i, unsigned long long pol) {
        F = ld_plan(ps.F32 + i, pol);  // streamed evict-first (launch.cuh)
        const int2 c = ld_plan(ps.CP + i, pol);
        code = c.x;
        perm = c.y;
    }
};

// R[o] = e^{-(o - m + 1/2)^2/b} of the centred factors (m = 4).
__device__ __forceinline__ float centred_R(const DWin& wn, int o) {
    const double c = static_cast<double>(o) - (static_cast<double>(wn.m) - 0.5);
    return static_cast<float>(exp(-c * c * wn.invb));
}

// Window weights of one point: w[t][o] = (s P for t = 0) Q_t^o R[o].
__device__ __forceinline__ void weights_f32(float (&w)[3][8], float s, const float4& F, const float* sR) {
    const float Q[3] = {F.y, F.z, F.w};
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        float q = t == 0 ? s * F.x : 1.0f;
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            w[t][o] = q * sR[o];
            q *= Q[t];
        }
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Spread, fp32: patches[it.patch + node] (fp64) = sum over the item's points.
// Scalar FFMA: acc[j][c] += u_j w2[c], u_j = w0[a] w1[bq + j] (packed FFMA2
// was measured slower for this operand pattern: 47 vs 65 TFLOP/s,
// scripts/micro/ffma_rates.cu). The warp's two half-warps share one SMEM patch and flush in a fixed order
// (half 0, then half 1) at the same lockstep step, so the summation order is
// a function of the plan alone.
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(W * 32, 5)
spread3_f32_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                   const DWin* __restrict__ wins, const double* __restrict__ v,
                   double* __restrict__ patches) {
    constexpr unsigned kFull = 0xffffffffu;
    extern __shared__ __align__(16) float smf[];
    __shared__ float sR[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane >> 4, hl = lane & 15, a = hl >> 1, bq = (hl & 1) * 4;
    const int HS = half_stage(kRowS);
    float* wp = smf + warp * kHP;
    float* stage_w = smf + W * kHP + warp * (2 * HS);
    const float* st_h = stage_w + h * HS;

    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    if (ps.vsrc) v = ps.vsrc;
    const DWin& wn = wins[ps.win];
    if (threadIdx.x < 8) sR[threadIdx.x] = centred_R(wn, threadIdx.x);
    for (int k = lane; k < kHP; k += 32) wp[k] = 0.f;
    int wb, we;
    {
        const int len = it.end - it.begin, per = (len + W - 1) / W;
        wb = min(it.begin + warp * per, it.end);
        we = min(wb + per, it.end);
    }
    PrefF pa, pb;
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    if (wb + lane < we) pa.load(ps, wb + lane, pol_stream);
    if (wb + 32 + lane < we) pb.load(ps, wb + 32 + lane, pol_stream);
    __syncthreads();
    double va = 0.0;
    pdl_wait();  // v may be produced by the previous kernel (duplicate-merge sums)
    v = launder(v);
    if (wb + lane < we) va = ld_keep(v + pa.perm, pol_keep);

    float acc[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[j][c] = 0.f;
    int cur = -1;  // current cell of this half-warp (uniform within the half)
    auto flush = [&](int cell) {
        const int l0 = cell >> 4, l1 = (cell >> 2) & 3, l2 = cell & 3;
        float* dst = wp + ((l0 + a) * kPEf + l1 + bq) * kPEf + l2;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                dst[j * kPEf + c] += acc[j][c];
                acc[j][c] = 0.f;
            }
    };
    // both halves, half 0 first (fixed order on the shared patch)
    auto flush_halves = [&](bool mine, int cell) {
        if (h == 0 && mine) flush(cell);
        __syncwarp();
        if (h == 1 && mine) flush(cell);
        __syncwarp();
    };
    auto point = [&](int k) {
        const float* r = st_h + k * kRowS;
        const float w0a = r[a];
        const float4 w1 = *reinterpret_cast<const float4*>(r + 8 + bq);
        const float4 x = *reinterpret_cast<const float4*>(r + 16);
        const float4 y = *reinterpret_cast<const float4*>(r + 20);
        const float w2[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
        const float u[4] = {w0a * w1.x, w0a * w1.y, w0a * w1.z, w0a * w1.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[j][c] = fmaf(u[j], w2[c], acc[j][c]);
    };

    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        const bool valid = lane < cnt;
        float* row = stage_w + (lane >> 4) * HS + (lane & 15) * kRowS;
        const int code = valid ? pa.code : -1;
        {
            float w[3][8];
            weights_f32(w, valid ? static_cast<float>(va) : 0.f, pa.F, sR);
            float4* r4 = reinterpret_cast<float4*>(row);
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                r4[2 * t] = make_float4(w[t][0], w[t][1], w[t][2], w[t][3]);
                r4[2 * t + 1] = make_float4(w[t][4], w[t][5], w[t][6], w[t][7]);
            }
        }
        const int prev = __shfl_up_sync(kFull, code, 1);
        // bit q: point q of the batch (half q >> 4, step q & 15) continues its half's cell
        const unsigned same = __ballot_sync(kFull, !valid || code == (hl == 0 ? cur : prev));
        pa = pb;
        if (base + 32 + lane < we) va = ld_keep(v + pa.perm, pol_keep);
        if (base + 64 + lane < we) pb.load(ps, base + 64 + lane, pol_stream);
        __syncwarp();
        if (same == kFull) {
#pragma unroll
            for (int k = 0; k < kHalfRows; ++k) point(k);
        } else {
            const unsigned nb = ~same;
#pragma unroll 1
            for (int k = 0; k < kHalfRows; ++k) {
                if (((nb >> k) | (nb >> (16 + k))) & 1u) {  // a cell starts in either half
                    const int c0 = __shfl_sync(kFull, code, k), c1 = __shfl_sync(kFull, code, 16 + k);
                    const bool mine = ((nb >> (16 * h + k)) & 1u) != 0;
                    flush_halves(mine && cur >= 0, cur);
                    if (mine) cur = h ? c1 : c0;
                }
                point(k);
            }
        }
        __syncwarp();
    }
    flush_halves(cur >= 0, cur);
    __syncthreads();
    // epilogue: the W warp patches in fixed order, in fp64
    if (threadIdx.x < kPEf * kPEf) {
        double* out = patches + it.patch;
        for (int n0 = 0; n0 < kPEf; ++n0) {
            const int e = n0 * kPEf * kPEf + threadIdx.x;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < W; ++q) s += static_cast<double>(smf[q * kHP + e]);
            out[e] = s;
        }
    }
}

// ---------------------------------------------------------------------------
// Gather, fp32: ps.out[perm] (fp64) = sum over the 8^3 taps of the point.
// s_j = sum_c w2[c] H[a, bq+j, c], then y = w0[a] sum_j w1[bq+j] s_j, reduced
// over the 16 lanes of the half-warp by one transposed butterfly per 16 points.
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(W * 32, 4)
gather3_f32_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                   const DWin* __restrict__ wins) {
    constexpr unsigned kFull = 0xffffffffu;
    constexpr int TC = 4;
    extern __shared__ __align__(16) float smf[];
    __shared__ float sR[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane >> 4, hl = lane & 15, a = hl >> 1, bq = (hl & 1) * 4;
    const int HS = half_stage(kRowG);
    float* halo = smf;
    float* stage_w = smf + kHP + warp * (2 * HS);
    const float* st_h = stage_w + h * HS;

    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    int tc[3];
    {
        int tile = it.tile;
        for (int k = 2; k >= 0; --k) {
            tc[k] = tile % wn.ntile;
            tile /= wn.ntile;
        }
    }
    if (threadIdx.x < 8) sR[threadIdx.x] = centred_R(wn, threadIdx.x);
    int wb, we;
    {
        const int len = it.end - it.begin, per = (len + W - 1) / W;
        wb = min(it.begin + warp * per, it.end);
        we = min(wb + per, it.end);
    }
    PrefF pa, pb;
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    if (wb + lane < we) pa.load(ps, wb + lane, pol_stream);
    if (wb + 32 + lane < we) pb.load(ps, wb + 32 + lane, pol_stream);
    pdl_wait();  // H is written by the grid stage
    {
        const DWin& w = *launder(&wn);
        const int Lg = w.Lg, M = w.M;
        const bool wrap = w.wrap != 0;
        const double* H = w.H;
        for (int k = threadIdx.x; k < kPEf * kPEf; k += blockDim.x) {
            const int n1 = k / kPEf, n2 = k - n1 * kPEf;
            const int i1 = tc[1] * TC + n1, i2 = tc[2] * TC + n2;
            for (int n0 = 0; n0 < kPEf; ++n0) {
                const int i0 = tc[0] * TC + n0;
                double hv;
                if (!wrap) {
                    hv = (i0 < Lg && i1 < Lg && i2 < Lg)
                             ? __ldcg(H + (static_cast<long long>(i0) * Lg + i1) * Lg + i2)
                             : 0.0;
                } else {
                    auto pm = [M](int x) { int r = x % M; return r < 0 ? r + M : r; };
                    hv = __ldcg(H + (static_cast<long long>(pm(w.lo + i0)) * Lg + pm(w.lo + i1)) * Lg +
                                pm(w.lo + i2));
                }
                halo[n0 * kPEf * kPEf + k] = static_cast<float>(hv);
            }
        }
    }
    __syncthreads();

    float hreg[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < 8; ++c) hreg[j][c] = 0.f;
    int cur = -1;
    auto reload = [&](int cell) {
        const int l0 = cell >> 4, l1 = (cell >> 2) & 3, l2 = cell & 3;
        const float* src = halo + ((l0 + a) * kPEf + l1 + bq) * kPEf + l2;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int c = 0; c < 8; ++c) hreg[j][c] = src[j * kPEf + c];
    };
    float part[kHalfRows];
    auto point = [&](int k) {
        const float* r = st_h + k * kRowG;
        const float w0a = r[a];
        const float4 w1 = *reinterpret_cast<const float4*>(r + 8 + bq);
        const float4 x = *reinterpret_cast<const float4*>(r + 16);
        const float4 y = *reinterpret_cast<const float4*>(r + 20);
        const float w2[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
        float s[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float t = hreg[j][0] * w2[0];
#pragma unroll
            for (int c = 1; c < 8; ++c) t = fmaf(hreg[j][c], w2[c], t);
            s[j] = t;
        }
        const float t = fmaf(w1.w, s[3], fmaf(w1.z, s[2], fmaf(w1.y, s[1], w1.x * s[0])));
        part[k] = w0a * t;
    };

    for (int base = wb; base < we; base += 32) {
        const int cnt = min(32, we - base);
        const bool valid = lane < cnt;
        float* row = stage_w + (lane >> 4) * HS + (lane & 15) * kRowG;
        const int code = valid ? pa.code : -1;
        const int perm = pa.perm;
        {
            float w[3][8];
            weights_f32(w, valid ? 1.0f : 0.f, pa.F, sR);
            float4* r4 = reinterpret_cast<float4*>(row);
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                r4[2 * t] = make_float4(w[t][0], w[t][1], w[t][2], w[t][3]);
                r4[2 * t + 1] = make_float4(w[t][4], w[t][5], w[t][6], w[t][7]);
            }
        }
        const int prev = __shfl_up_sync(kFull, code, 1);
        const unsigned same = __ballot_sync(kFull, !valid || code == (hl == 0 ? cur : prev));
        pa = pb;
        if (base + 64 + lane < we) pb.load(ps, base + 64 + lane, pol_stream);
        __syncwarp();
        if (same == kFull) {
#pragma unroll
            for (int k = 0; k < kHalfRows; ++k) point(k);
        } else {
            const unsigned nb = ~same;
#pragma unroll
            for (int k = 0; k < kHalfRows; ++k) {
                if (((nb >> k) | (nb >> (16 + k))) & 1u) {
                    const int c0 = __shfl_sync(kFull, code, k), c1 = __shfl_sync(kFull, code, 16 + k);
                    if ((nb >> (16 * h + k)) & 1u) {
                        cur = h ? c1 : c0;
                        reload(cur);
                    }
                }
                point(k);
            }
        }
        // transposed butterfly over the half-warp: lane hl ends with point hl's sum
#pragma unroll
        for (int s = 8; s >= 1; s >>= 1) {
            const bool upper = (hl & s) != 0;
#pragma unroll
            for (int k = 0; k < s; ++k) {
                const float send = upper ? part[k] : part[k + s];
                const float keep = upper ? part[k + s] : part[k];
                part[k] = keep + __shfl_xor_sync(kFull, send, s);
            }
        }
        if (valid) st_keep(ps.out + perm, static_cast<double>(part[0]), pol_keep);
        __syncwarp();
    }
}

// ===========================================================================
// 3xTF32 tensor-core pair (the default fp32 kernels).
// One warp-level HMMA.1688.F32.TF32 is D(16x8) += A(16x8) B(8x8); lane
// l = 4g + t holds A[g][t], A[g+8][t], A[g][t+4], A[g+8][t+4], B[t][g],
// B[t+4][g] and D[g][2t..2t+1], D[g+8][2t..2t+1].
// Staging rows are kRowT = 24 floats: 24 t mod 32 = 0, 24, 16, 8 for the four
// rows a load touches, so 8-word segments of 4 consecutive rows hit disjoint
// banks. Row: x[8] | z[8] | four powers of Q1 | {code, perm}.
// ===========================================================================
constexpr int kRowT = 24;

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// x = hi + lo exactly; hi has the 11 significant bits tf32 keeps
__device__ __forceinline__ void split_tf32(float x, unsigned& hi, unsigned& lo) {
    hi = __float_as_uint(x) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

// Power rows of one point: x[o] = p Q0^o, z[o] = Q2^o, then four powers of Q1.
__device__ __forceinline__ void stage_t32(float* row, float p, const float4& F, float y0, float y1, float y2,
                                          float y3, int code, int perm) {
    float4* r4 = reinterpret_cast<float4*>(row);
    float q[8];
    q[0] = p;
#pragma unroll
    for (int o = 1; o < 8; ++o) q[o] = q[o - 1] * F.y;
    r4[0] = make_float4(q[0], q[1], q[2], q[3]);
    r4[1] = make_float4(q[4], q[5], q[6], q[7]);
    q[0] = 1.0f;
#pragma unroll
    for (int o = 1; o < 8; ++o) q[o] = q[o - 1] * F.w;
    r4[2] = make_float4(q[0], q[1], q[2], q[3]);
    r4[3] = make_float4(q[4], q[5], q[6], q[7]);
    r4[4] = make_float4(y0, y1, y2, y3);
    *reinterpret_cast<int2*>(row + 20) = make_int2(code, perm);
}

__device__ __forceinline__ int run_len32(unsigned same, int p) {
    const unsigned s = p + 1 < 32 ? (same >> (p + 1)) : 0u;
    return __ffs(~s);  // 1 + number of consecutive set bits above p
}

// ---------------------------------------------------------------------------
// Spread, 3xTF32. Per cell the 8^3 block is G[(a, b1), (b0, c)], b = 4 b1 + b0
// (split-power form): A[(a, b1)][p] = x_p[a] (Q1_p^4)^b1, B[p][(b0, c)] =
// Q1_p^b0 z_p[c], K = 8 same-cell points per MMA, four N tiles (b0) -> 12 HMMA
// per 8 points. Accumulator tile b0 holds G[a = g][b = b0 | 4 + b0][c = 2t..2t+1].
// R[a] R[b] R[c] is applied when a cell's block is added into the warp's SMEM
// patch (fp32); the epilogue adds the W patches in fp64 in a fixed order.
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(W * 32, 4)
spread3_t32_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                   const DWin* __restrict__ wins, const double* __restrict__ v,
                   double* __restrict__ patches) {
    constexpr unsigned kFull = 0xffffffffu;
    constexpr int PE = kPEf;
    extern __shared__ __align__(16) float smf[];
    __shared__ float sR[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    float* wp = smf + warp * kHP;
    float* stage = smf + W * kHP + warp * 32 * kRowT;

    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    if (ps.vsrc) v = ps.vsrc;
    const DWin& wn = wins[ps.win];
    if (threadIdx.x < 8) sR[threadIdx.x] = centred_R(wn, threadIdx.x);
    for (int k = lane; k < kHP; k += 32) wp[k] = 0.f;
    int wb, we;
    {
        const int len = it.end - it.begin, per = (len + W - 1) / W;
        wb = min(it.begin + warp * per, it.end);
        we = min(wb + per, it.end);
    }
    // Two point buffers in rotation (the loop is unrolled by two batches, so no
    // buffer is ever copied): a batch's plan data is requested two batches
    // ahead, right after the buffer has been staged, and its v one batch
    // ahead. With a copy `pa = pb` the warp waits for the newest load every
    // iteration, and these kernels consume a batch faster than DRAM answers.
    PrefF p0, p1;
    double v0 = 0.0, v1 = 0.0;
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    // Loads are unconditional with the index clamped into the item (lanes past
    // the range read a valid point they never use): a predicated load lands in
    // a temporary and its predicated copy waits for the data at once.
    const int last = it.end - 1;
    p0.load(ps, min(wb + lane, last), pol_stream);
    p1.load(ps, min(wb + 32 + lane, last), pol_stream);
    __syncthreads();
    pdl_wait();  // v may be produced by the previous kernel (duplicate-merge sums)
    v = launder(v);
    v0 = ld_keep(v + p0.perm, pol_keep);

    // The tensor cores add into an fp32 accumulator with truncation, a bias
    // that grows with the length of the chain (measured 3e-6 relative at 58
    // points per cell), so a chain is at most one 32-point batch plus a
    // partial one: `acc` is drained into `sum` (round-to-nearest adds) after
    // every full batch.
    float acc[4][4], sum[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[j][c] = sum[j][c] = 0.f;
    int cur = -1;
    auto drain = [&]() {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                sum[j][c] += acc[j][c];
                acc[j][c] = 0.f;
            }
    };
    auto flush = [&](int cell) {
        const int l0 = cell >> 4, l1 = (cell >> 2) & 3, l2 = cell & 3;
        float* dst = wp + ((l0 + g) * PE + l1) * PE + l2 + 2 * t;
        const float rg = sR[g], rc0 = sR[2 * t], rc1 = sR[2 * t + 1];
        drain();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float r0 = rg * sR[j], r1 = rg * sR[4 + j];
            dst[j * PE] += (sum[j][0] * r0) * rc0;
            dst[j * PE + 1] += (sum[j][1] * r0) * rc1;
            dst[(4 + j) * PE] += (sum[j][2] * r1) * rc0;
            dst[(4 + j) * PE + 1] += (sum[j][3] * r1) * rc1;
            sum[j][0] = sum[j][1] = sum[j][2] = sum[j][3] = 0.f;
        }
    };
    // 8 points p0..p0+7 of the current cell (K index t -> p0 + t, t + 4 -> p0 + t + 4);
    // points >= nv contribute zero
    auto group8 = [&](int p0, int nv) {
        const bool v0 = t < nv, v1 = t + 4 < nv;
        const float* r0 = stage + (p0 + (v0 ? t : 0)) * kRowT;
        const float* r1 = stage + (p0 + (v1 ? t + 4 : 0)) * kRowT;
        const float x0 = v0 ? r0[g] : 0.f, x1 = v1 ? r1[g] : 0.f;
        const float z0 = r0[8 + g], z1 = r1[8 + g];
        const float4 y0 = *reinterpret_cast<const float4*>(r0 + 16);  // Q1, Q1^2, Q1^3, Q1^4
        const float4 y1 = *reinterpret_cast<const float4*>(r1 + 16);
        unsigned ah[4], al[4];
        split_tf32(x0, ah[0], al[0]);
        split_tf32(x0 * y0.w, ah[1], al[1]);
        split_tf32(x1, ah[2], al[2]);
        split_tf32(x1 * y1.w, ah[3], al[3]);
        const float f0[4] = {1.0f, y0.x, y0.y, y0.z}, f1[4] = {1.0f, y1.x, y1.y, y1.z};
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // small terms first
            unsigned bh[2], bl[2];
            split_tf32(j == 0 ? z0 : z0 * f0[j], bh[0], bl[0]);
            split_tf32(j == 0 ? z1 : z1 * f1[j], bh[1], bl[1]);
            mma_tf32(acc[j], al, bh);
            mma_tf32(acc[j], ah, bl);
            mma_tf32(acc[j], ah, bh);
        }
    };

    // one 32-point batch from buffer (pc, vc); pn / vn is the next batch's buffer
    auto batch = [&](int base, PrefF& pc, double vc, const PrefF& pn, double& vn) {
        const int cnt = min(32, we - base);
        const int code = pc.code;
        if (lane < cnt) {
            const float y1 = pc.F.z, y2 = y1 * y1;
            stage_t32(stage + lane * kRowT, static_cast<float>(vc) * pc.F.x, pc.F, y1, y2, y2 * y1, y2 * y2, code, 0);
        }
        const int prev = __shfl_up_sync(kFull, code, 1);
        const unsigned same = __ballot_sync(kFull, lane < cnt && code == (lane == 0 ? cur : prev));
        vn = ld_keep(v + pn.perm, pol_keep);
        pc.load(ps, min(base + 64 + lane, last), pol_stream);
        __syncwarp();
        if (same == kFull) {  // the whole batch continues the current cell
#pragma unroll
            for (int q = 0; q < 4; ++q) group8(8 * q, 8);
            drain();
        } else {
            int p = 0;
            while (p < cnt) {
                if (!((same >> p) & 1u)) {  // a new cell starts at p
                    if (cur >= 0) flush(cur);
                    cur = __shfl_sync(kFull, code, p);
                }
                for (int L = run_len32(same, p); L > 0;) {
                    const int nv = min(L, 8);
                    group8(p, nv);
                    p += nv;
                    L -= nv;
                }
            }
        }
        __syncwarp();
    };
    for (int base = wb; base < we; base += 64) {
        batch(base, p0, v0, p1, v1);
        if (base + 32 < we) batch(base + 32, p1, v1, p0, v0);
    }
    if (cur >= 0) flush(cur);
    __syncthreads();
    // epilogue: the W warp patches in fixed order, in fp64
    if (threadIdx.x < PE * PE) {
        double* out = patches + it.patch;
        for (int n0 = 0; n0 < PE; ++n0) {
            const int e = n0 * PE * PE + threadIdx.x;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < W; ++q) s += static_cast<double>(smf[q * kHP + e]);
            out[e] = s;
        }
    }
}

// ---------------------------------------------------------------------------
// Gather, 3xTF32. With b = 2 b1 + b0, Y = Q1:
//   Z[p, (b0, c)] = sum_{(a, b1)} (x_p[a] Y_p^{2 b1}) H[a, 2 b1 + b0, c]
//   y_p           = sum_c z_p[c] (Z[p, (0, c)] + Y_p Z[p, (1, c)])
// M = 16 same-cell points per MMA, K = 32 in four k-steps (k-step s: b1 = s,
// column a), N = 16 in two tiles (b0) -> 24 HMMA per 16 points. The cell's
// halo values (times R[a] R[b] R[c]) are kept split in registers and reloaded
// when the cell changes. Row: x[8] (P folded) | z[8] | Y^2, Y^4, Y^6, Y | {code, perm}.
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(W * 32, 4)
gather3_t32_kernel(const Item* __restrict__ items, const DPSet* __restrict__ psets,
                   const DWin* __restrict__ wins) {
    constexpr unsigned kFull = 0xffffffffu;
    constexpr int TC = 4, PE = kPEf;
    extern __shared__ __align__(16) float smf[];
    __shared__ float sR[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    float* halo = smf;
    float* stage = smf + kHP + warp * 32 * kRowT;

    pdl_trigger();
    const Item it = items[blockIdx.x];
    const DPSet ps = psets[it.ps];
    const DWin& wn = wins[ps.win];
    int tc[3];
    {
        int tile = it.tile;
        for (int k = 2; k >= 0; --k) {
            tc[k] = tile % wn.ntile;
            tile /= wn.ntile;
        }
    }
    if (threadIdx.x < 8) sR[threadIdx.x] = centred_R(wn, threadIdx.x);
    int wb, we;
    {
        const int len = it.end - it.begin, per = (len + W - 1) / W;
        wb = min(it.begin + warp * per, it.end);
        we = min(wb + per, it.end);
    }
    PrefF p0, p1;  // two buffers in rotation, see spread3_t32_kernel
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    const int last = it.end - 1;  // unconditional, clamped loads: see spread3_t32_kernel
    p0.load(ps, min(wb + lane, last), pol_stream);
    p1.load(ps, min(wb + 32 + lane, last), pol_stream);
    pdl_wait();  // H is written by the grid stage
    {
        const DWin& w = *launder(&wn);
        const int Lg = w.Lg, M = w.M;
        const bool wrap = w.wrap != 0;
        const double* H = w.H;
        for (int k = threadIdx.x; k < PE * PE; k += blockDim.x) {
            const int n1 = k / PE, n2 = k - n1 * PE;
            const int i1 = tc[1] * TC + n1, i2 = tc[2] * TC + n2;
            for (int n0 = 0; n0 < PE; ++n0) {
                const int i0 = tc[0] * TC + n0;
                double hv;
                if (!wrap) {
                    hv = (i0 < Lg && i1 < Lg && i2 < Lg)
                             ? __ldcg(H + (static_cast<long long>(i0) * Lg + i1) * Lg + i2)
                             : 0.0;
                } else {
                    auto pm = [M](int x) { int r = x % M; return r < 0 ? r + M : r; };
                    hv = __ldcg(H + (static_cast<long long>(pm(w.lo + i0)) * Lg + pm(w.lo + i1)) * Lg +
                                pm(w.lo + i2));
                }
                halo[n0 * PE * PE + k] = static_cast<float>(hv);
            }
        }
    }
    __syncthreads();

    unsigned bh[4][2][2], bl[4][2][2];  // [k-step s][tile b0][a = t | t + 4]
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) bh[s][nt][0] = bh[s][nt][1] = bl[s][nt][0] = bl[s][nt][1] = 0u;
    int cur = -1;
    auto reload = [&](int cell) {
        const int l0 = cell >> 4, l1 = (cell >> 2) & 3, l2 = cell & 3;
        const float* src = halo + ((l0 + t) * PE + l1) * PE + l2 + g;
        const float rc = sR[g], ra0 = sR[t] * rc, ra1 = sR[t + 4] * rc;
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int b = 2 * s + nt;
                split_tf32(src[b * PE] * (ra0 * sR[b]), bh[s][nt][0], bl[s][nt][0]);
                split_tf32(src[4 * PE * PE + b * PE] * (ra1 * sR[b]), bh[s][nt][1], bl[s][nt][1]);
            }
    };
    // 16 points p0..p0+15 of the current cell (row g -> p0 + g, row g + 8 -> p0 + g + 8)
    auto group16 = [&](int p0, int nv) {
        const bool v0 = g < nv, v1 = g + 8 < nv;
        const float* r0 = stage + (p0 + (v0 ? g : 0)) * kRowT;
        const float* r1 = stage + (p0 + (v1 ? g + 8 : 0)) * kRowT;
        const float xa0 = v0 ? r0[t] : 0.f, xb0 = v0 ? r0[t + 4] : 0.f;
        const float xa1 = v1 ? r1[t] : 0.f, xb1 = v1 ? r1[t + 4] : 0.f;
        const float4 Y0 = *reinterpret_cast<const float4*>(r0 + 16);  // Y^2, Y^4, Y^6, Y
        const float4 Y1 = *reinterpret_cast<const float4*>(r1 + 16);
        const float f0[4] = {1.0f, Y0.x, Y0.y, Y0.z}, f1[4] = {1.0f, Y1.x, Y1.y, Y1.z};
        float d[2][2][4];  // [tile b0][k-step parity][fragment]
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int q = 0; q < 2; ++q) d[nt][q][0] = d[nt][q][1] = d[nt][q][2] = d[nt][q][3] = 0.f;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            unsigned ah[4], al[4];
            split_tf32(s == 0 ? xa0 : xa0 * f0[s], ah[0], al[0]);
            split_tf32(s == 0 ? xa1 : xa1 * f1[s], ah[1], al[1]);
            split_tf32(s == 0 ? xb0 : xb0 * f0[s], ah[2], al[2]);
            split_tf32(s == 0 ? xb1 : xb1 * f1[s], ah[3], al[3]);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) mma_tf32(d[nt][s & 1], al, bh[s][nt]);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) mma_tf32(d[nt][s & 1], ah, bl[s][nt]);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) mma_tf32(d[nt][s & 1], ah, bh[s][nt]);
        }
        const float2 z0 = *reinterpret_cast<const float2*>(r0 + 8 + 2 * t);
        const float2 z1 = *reinterpret_cast<const float2*>(r1 + 8 + 2 * t);
        float e[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int c = 0; c < 4; ++c) e[nt][c] = d[nt][0][c] + d[nt][1][c];
        float part0 = fmaf(z0.x, fmaf(Y0.w, e[1][0], e[0][0]), z0.y * fmaf(Y0.w, e[1][1], e[0][1]));
        float part1 = fmaf(z1.x, fmaf(Y1.w, e[1][2], e[0][2]), z1.y * fmaf(Y1.w, e[1][3], e[0][3]));
        part0 += __shfl_xor_sync(kFull, part0, 1);
        part1 += __shfl_xor_sync(kFull, part1, 1);
        part0 += __shfl_xor_sync(kFull, part0, 2);
        part1 += __shfl_xor_sync(kFull, part1, 2);
        if (t == 0 && v0) st_keep(ps.out + reinterpret_cast<const int*>(r0 + 20)[1], static_cast<double>(part0), pol_keep);
        if (t == 1 && v1) st_keep(ps.out + reinterpret_cast<const int*>(r1 + 20)[1], static_cast<double>(part1), pol_keep);
    };

    auto batch = [&](int base, PrefF& pc) {
        const int cnt = min(32, we - base);
        const int code = pc.code;
        if (lane < cnt) {
            const float y1 = pc.F.z, y2 = y1 * y1, y4 = y2 * y2;
            stage_t32(stage + lane * kRowT, pc.F.x, pc.F, y2, y4, y4 * y2, y1, code, pc.perm);
        }
        const int prev = __shfl_up_sync(kFull, code, 1);
        const unsigned same = __ballot_sync(kFull, lane < cnt && code == (lane == 0 ? cur : prev));
        pc.load(ps, min(base + 64 + lane, last), pol_stream);
        __syncwarp();
        if (same == kFull) {
            group16(0, 16);
            group16(16, 16);
        } else {
            int p = 0;
            while (p < cnt) {
                if (!((same >> p) & 1u)) {
                    cur = __shfl_sync(kFull, code, p);
                    reload(cur);
                }
                for (int L = run_len32(same, p); L > 0;) {
                    const int nv = min(L, 16);
                    group16(p, nv);
                    p += nv;
                    L -= nv;
                }
            }
        }
        __syncwarp();
    };
    for (int base = wb; base < we; base += 64) {
        batch(base, p0);
        if (base + 32 < we) batch(base + 32, p1);
    }
}

// Centre-relative fp32 window factors of each sorted point, plus {code, perm}
// (the same tile-local cell code as factors_kernel).
__global__ void factors32_kernel(const double* __restrict__ x0, const double* __restrict__ x1,
                                 const double* __restrict__ x2, const int* __restrict__ perm,
                                 long long n, double Mf, int m, double invb, double Cw, int cmin, int TC,
                                 float4* __restrict__ F, int2* __restrict__ CP) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int src = perm[i];
        const double* xs[3] = {x0, x1, x2};
        double Q[3];
        double ex = 0.0;
        int cd = 0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const double xm = xs[t][src] * Mf;
            const double fl = floor(xm);
            const double u = (xm - fl) - 0.5;  // relative to the cell centre
            ex += u * u + static_cast<double>(2 * m - 1) * u;
            Q[t] = exp((2.0 * u) * invb);
            cd = cd * TC + (static_cast<int>(fl) - cmin) % TC;
        }
        F[i] = make_float4(static_cast<float>(Cw * Cw * Cw * exp(-ex * invb)), static_cast<float>(Q[0]),
                           static_cast<float>(Q[1]), static_cast<float>(Q[2]));
        CP[i] = make_int2(cd, src);
    }
}

size_t spread3_f32_smem() { return sizeof(float) * (kW3f * kHP + kW3f * 2 * (kHalfRows * kRowS + 8)); }
size_t gather3_f32_smem() { return sizeof(float) * (kHP + kW3f * 2 * (kHalfRows * kRowG + 8)); }
size_t spread3_t32_smem() { return sizeof(float) * (kW3f * kHP + kW3f * 32 * kRowT); }
size_t gather3_t32_smem() { return sizeof(float) * (kHP + kW3f * 32 * kRowT); }

// KSVM_NFFT_F32K=ffma: the CUDA-core kernels instead of the 3xTF32 pair
static bool f32_ffma() {  // read per launch (a graph capture fixes it for the operator)
    const char* e = std::getenv("KSVM_NFFT_F32K");
    return e && e[0] == 'f';
}

cudaError_t init_f32_attributes() {
    cudaError_t e = cudaSuccess;
    auto set = [&](const void* f, size_t bytes) {
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    };
    set(reinterpret_cast<const void*>(spread3_f32_kernel<kW3f>), spread3_f32_smem());
    set(reinterpret_cast<const void*>(gather3_f32_kernel<kW3f>), gather3_f32_smem());
    set(reinterpret_cast<const void*>(spread3_t32_kernel<kW3f>), spread3_t32_smem());
    set(reinterpret_cast<const void*>(gather3_t32_kernel<kW3f>), gather3_t32_smem());
    return e;
}

void launch_spread3_f32(const Item* items, int nitems, const DPSet* ps, const DWin* wins, const double* v,
                        double* patches, cudaStream_t st) {
    if (nitems == 0) return;
    if (f32_ffma())
        launch_k(spread3_f32_kernel<kW3f>, dim3(nitems), dim3(kW3f * 32), spread3_f32_smem(), st, items, ps, wins, v,
                 patches);
    else
        launch_k(spread3_t32_kernel<kW3f>, dim3(nitems), dim3(kW3f * 32), spread3_t32_smem(), st, items, ps, wins, v,
                 patches);
}

void launch_gather3_f32(const Item* items, int nitems, const DPSet* ps, const DWin* wins, cudaStream_t st) {
    if (nitems == 0) return;
    if (f32_ffma())
        launch_k(gather3_f32_kernel<kW3f>, dim3(nitems), dim3(kW3f * 32), gather3_f32_smem(), st, items, ps, wins);
    else
        launch_k(gather3_t32_kernel<kW3f>, dim3(nitems), dim3(kW3f * 32), gather3_t32_smem(), st, items, ps, wins);
}

void launch_factors32(const double* x0, const double* x1, const double* x2, const int* perm, long long n,
                      double Mf, int m, double invb, double Cw, int cmin, int TC, float4* F, int2* CP,
                      cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    factors32_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(x0, x1, x2, perm, n, Mf, m, invb, Cw, cmin, TC, F,
                                                               CP);
}

}  // namespace ksvm_nfft
