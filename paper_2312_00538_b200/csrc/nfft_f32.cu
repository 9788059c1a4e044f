// Optional fp32 mode of the d = 3, m = 4 spread / gather (north_star:
// "<= 1e-5 in an optional fp32 mode"; the same operator as
// P:src/fastsum.cpp:257-296, computed with fp32 window weights and fp32
// FFMA accumulation on the CUDA cores).
//
// Why CUDA cores: B200 has no fp32 tensor-core kind that is accurate to
// 1e-5 without splitting (tf32 keeps 10 mantissa bits), and FFMA runs at
// 128 FMA/clk/SM, twice the FP64 datapath the fp64 kernels (DMMA) share.
// The grid side (node reduction, separable convolution) and the window sum
// stay fp64: they are a few percent of the work. Inputs (v) and outputs
// (per-window results, y) stay fp64, so the C ABI does not change.
//
// Window factors (factors32_kernel) are CELL-relative (u_t in [m-1, m)):
//   w_t[o] = C e^{-(u_t - o)^2/b} = P_t Q_t^o R[o],
//   P = C^3 e^{-sum_t u_t^2/b},  Q_t = e^{2 u_t/b},  R[o] = e^{-o^2/b},
// all comfortably inside the fp32 range (the fp64 kernels' tile-relative
// factors would not be). A plan stores {P, Q0, Q1, Q2} as float4 (16 B per
// point instead of 32 B).
//
// Decomposition (both kernels): a CTA is one item (a 4^3-cell tile's point
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
    if (threadIdx.x < 8) sR[threadIdx.x] = static_cast<float>(wn.R[threadIdx.x]);
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
    if (threadIdx.x < 8) sR[threadIdx.x] = static_cast<float>(wn.R[threadIdx.x]);
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

// Cell-relative fp32 window factors of each sorted point, plus {code, perm}
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
            const double u = (xm - fl) + static_cast<double>(m - 1);
            ex += u * u;
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

cudaError_t init_f32_attributes() {
    cudaError_t e = cudaFuncSetAttribute(spread3_f32_kernel<kW3f>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(spread3_f32_smem()));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(gather3_f32_kernel<kW3f>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(gather3_f32_smem()));
    return e;
}

void launch_spread3_f32(const Item* items, int nitems, const DPSet* ps, const DWin* wins, const double* v,
                        double* patches, cudaStream_t st) {
    if (nitems == 0) return;
    launch_k(spread3_f32_kernel<kW3f>, dim3(nitems), dim3(kW3f * 32), spread3_f32_smem(), st, items, ps, wins, v,
             patches);
}

void launch_gather3_f32(const Item* items, int nitems, const DPSet* ps, const DWin* wins, cudaStream_t st) {
    if (nitems == 0) return;
    launch_k(gather3_f32_kernel<kW3f>, dim3(nitems), dim3(kW3f * 32), gather3_f32_smem(), st, items, ps, wins);
}

void launch_factors32(const double* x0, const double* x1, const double* x2, const int* perm, long long n,
                      double Mf, int m, double invb, double Cw, int cmin, int TC, float4* F, int2* CP,
                      cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16));
    factors32_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(x0, x1, x2, perm, n, Mf, m, invb, Cw, cmin, TC, F,
                                                               CP);
}

}  // namespace ksvm_nfft
