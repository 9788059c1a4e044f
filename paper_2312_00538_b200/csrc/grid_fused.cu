// Fused grid side of one dimension class: patch reduction + the d separable
// convolution stages ("grid stage as a real separable
// convolution") in ONE launch, with the whole (data-range) grid of a window
// held on chip.
//
// The staged path (reduce_owner_kernel + d x conv_stage_kernel) is a chain
// of d + 1 short kernels whose cost on the small configs is launch-to-drain
// latency (~5 us each for tiny work, profiles/README.md). Here:
//   d = 3: one thread-block CLUSTER of C <= 16 CTAs per window. CTA r owns
//          the dim-0 planes [r np, (r+1) np) of the grid in shared memory:
//          it reduces their nodes from the tile patches, runs the dim-2 and
//          dim-1 stages locally, then (cluster barrier) gathers the dim-1
//          rows it owns for stage 2 from every CTA's shared memory (DSMEM,
//          an all-to-all transpose of 1/C of the grid per CTA), runs the
//          dim-0 stage and writes H.
//   d = 1, 2: one CTA per window, everything in its shared memory.
// Arithmetic per output is the Toeplitz sum of the staged kernels
// (H = A0 [A1 A2 g - S1 S2 g] - S0 [A1 S2 g + S1 A2 g] for d = 3), each line
// summed in ascending j by one thread on CUDA-core DFMA with a 4-output
// register block and a sliding window of table values; the summation order is
// fixed, so applies stay bit-reproducible. Only non-wrapping grids (the
// operator data-range grids: every node index is its extended index).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "launch.cuh"
#include "nfft_engine.cuh"

namespace cg = cooperative_groups;

namespace ksvm_nfft {

constexpr int kFusedThreads = 512;
constexpr int kFusedMaxCluster = 16;

namespace {

// Table (a or s) staged in SMEM as tab[r + Lg] for r in [-(Lg+1), Lg+3],
// zero outside [-(Lg-1), Lg-1], so 4-output blocks never index out of range.
__device__ __forceinline__ int tab_len(int Lg) { return 2 * Lg + 6; }

__device__ void stage_tables(const DWin& wn, double* sA, double* sS) {
    const int Lg = wn.Lg, TL = tab_len(Lg);
    for (int k = threadIdx.x; k < TL; k += blockDim.x) {
        const int r = k - Lg - 1;  // sA[k] = a(r); index of a(r) is r + Lg + 1
        const bool ok = r > -Lg && r < Lg;
        sA[k] = ok ? wn.tabA[r + Lg - 1] : 0.0;
        sS[k] = ok ? wn.tabS[r + Lg - 1] : 0.0;
    }
}

// 4 outputs i0..i0+3 of out_u = sum_j T[i0 + u - j] x[j] for two tables
// (ta, ts) and one input line x (stride xs, Lg entries).
struct Acc8 {
    double a[4], s[4];
};

__device__ __forceinline__ Acc8 line_conv1(const double* __restrict__ sA, const double* __restrict__ sS,
                                           const double* __restrict__ x, int xs, int Lg, int i0) {
    Acc8 r;
    // window: w_u = T[i0 + u - j], table index (i0 + u - j) + Lg + 1
    double wa[4], ws[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        wa[u] = sA[i0 + u + Lg + 1];
        ws[u] = sS[i0 + u + Lg + 1];
        r.a[u] = 0.0;
        r.s[u] = 0.0;
    }
#pragma unroll 4
    for (int j = 0; j < Lg; ++j) {
        const double xv = x[j * xs];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            r.a[u] = fma(wa[u], xv, r.a[u]);
            r.s[u] = fma(ws[u], xv, r.s[u]);
        }
#pragma unroll
        for (int u = 3; u > 0; --u) {
            wa[u] = wa[u - 1];
            ws[u] = ws[u - 1];
        }
        wa[0] = sA[i0 - j - 1 + Lg + 1];
        ws[0] = sS[i0 - j - 1 + Lg + 1];
    }
    return r;
}

// Two input lines x, y: p_u = sum_j a x - s y,  q_u = sum_j a y + s x
__device__ __forceinline__ Acc8 line_conv2(const double* __restrict__ sA, const double* __restrict__ sS,
                                           const double* __restrict__ x, const double* __restrict__ y, int xs,
                                           int Lg, int i0, bool need_q) {
    Acc8 r;
    double wa[4], ws[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        wa[u] = sA[i0 + u + Lg + 1];
        ws[u] = sS[i0 + u + Lg + 1];
        r.a[u] = 0.0;
        r.s[u] = 0.0;
    }
#pragma unroll 4
    for (int j = 0; j < Lg; ++j) {
        const double xv = x[j * xs], yv = y[j * xs];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            r.a[u] = fma(wa[u], xv, r.a[u]);
            r.a[u] = fma(-ws[u], yv, r.a[u]);
            if (need_q) {
                r.s[u] = fma(wa[u], yv, r.s[u]);
                r.s[u] = fma(ws[u], xv, r.s[u]);
            }
        }
#pragma unroll
        for (int u = 3; u > 0; --u) {
            wa[u] = wa[u - 1];
            ws[u] = ws[u - 1];
        }
        wa[0] = sA[i0 - j - 1 + Lg + 1];
        ws[0] = sS[i0 - j - 1 + Lg + 1];
    }
    return r;
}

// Grid node (e0, e1, e2) of a non-wrapping grid <- sum of the covering
// tiles' (pre-reduced) patch values, in (a0, a1, a2) order. soff: the
// tile_patch offsets of tiles T0 in [t0lo, t0lo + n0), all T1, T2, staged in
// SMEM, so the <= NC^d patch loads of a node are independent (no dependent
// offset load in front of each).
template <int D, int NC>
__device__ __forceinline__ double node_sum(const DWin& wn, const double* __restrict__ patches,
                                           const long long* __restrict__ soff, int t0lo, const int* e) {
    const int TC = wn.TC, PE = wn.PE, nt = wn.ntile;
    int thi[3] = {0, 0, 0};
#pragma unroll
    for (int t = 0; t < D; ++t) thi[t] = min(e[t] / TC, nt - 1);
    // NC^d values loaded first (independent loads), summed in index order;
    // for large NC^d (generic m) the running sum keeps registers bounded
    constexpr int NV = D == 1 ? NC : (D == 2 ? NC * NC : NC * NC * NC);
    constexpr bool kArr = NV <= 27;
    double v[kArr ? NV : 1];
    double run = 0.0;
    auto put = [&](int q, double x) {
        if constexpr (kArr) v[q] = x;
        else run += x;
    };
#pragma unroll
    for (int a0 = 0; a0 < NC; ++a0) {
        const int T0 = thi[0] - a0, o0 = e[0] - T0 * TC;
        const bool ok0 = T0 >= 0 && o0 < PE;
        if constexpr (D == 1) {
            const long long off = ok0 ? soff[T0 - t0lo] : -1;
            put(a0, off >= 0 ? __ldcg(patches + off + o0) : 0.0);
        } else {
#pragma unroll
            for (int a1 = 0; a1 < NC; ++a1) {
                const int T1 = thi[1] - a1, o1 = e[1] - T1 * TC;
                const bool ok1 = ok0 && T1 >= 0 && o1 < PE;
                if constexpr (D == 2) {
                    const long long off = ok1 ? soff[(T0 - t0lo) * nt + T1] : -1;
                    put(a0 * NC + a1, off >= 0 ? __ldcg(patches + off + o0 * PE + o1) : 0.0);
                } else {
#pragma unroll
                    for (int a2 = 0; a2 < NC; ++a2) {
                        const int T2 = thi[2] - a2, o2 = e[2] - T2 * TC;
                        const bool ok2 = ok1 && T2 >= 0 && o2 < PE;
                        const long long off = ok2 ? soff[((T0 - t0lo) * nt + T1) * nt + T2] : -1;
                        put((a0 * NC + a1) * NC + a2, off >= 0 ? __ldcg(patches + off + (o0 * PE + o1) * PE + o2) : 0.0);
                    }
                }
            }
        }
    }
    if constexpr (!kArr) return run;
    double sum = 0.0;  // skipped terms are exact zeros: same value as the staged reduction's skip
#pragma unroll
    for (int q = 0; q < (kArr ? NV : 0); ++q) sum += v[q];
    return sum;
}

// Stage tile_patch offsets for tiles T0 in [t0lo, t0hi] (all T1, T2) into SMEM.
__device__ void stage_offsets(const DWin& wn, int D, int t0lo, int t0hi, long long* soff) {
    int per = 1;
    for (int t = 1; t < D; ++t) per *= wn.ntile;
    const int cnt = max(0, t0hi - t0lo + 1) * per;
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) soff[k] = wn.tile_patch[static_cast<long long>(t0lo) * per + k];
}

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

}  // namespace

// d = 3: grid (C, nslots), cluster (C, 1, 1). Dynamic SMEM: two tables and
// four slabs of np * Lg^2 doubles (G -> T2, T0 -> X2, T1 -> X3, T3).
// kReduce = false: the grid G was produced by the staged node reduction
// (reduce_owner_kernel on every SM) and the cluster only runs the three
// convolution stages (its slab of G is one coalesced read from L2).
template <int NC, bool kReduce = true>
__global__ void __launch_bounds__(kFusedThreads) grid3_fused_kernel(const DWin* __restrict__ wins,
                                                                    const int* __restrict__ slots,
                                                                    const double* __restrict__ patches, int np) {
    pdl_trigger();
    cg::cluster_group cl = cg::this_cluster();
    const int C = static_cast<int>(cl.num_blocks());
    const int rank = static_cast<int>(cl.block_rank());
    const DWin& wn = wins[slots[blockIdx.y]];
    if (wn.d != 3 || wn.wrap) {  // uniform over the cluster (one window per cluster)
        pdl_wait();
        return;
    }
    const int Lg = wn.Lg, L2 = Lg * Lg;
    const int TL = tab_len(Lg);
    extern __shared__ double smem[];
    double* sA = smem;
    double* sS = sA + TL;
    double* slab0 = sS + ((TL + 1) & ~1);  // G, then T2
    const long long SL = static_cast<long long>(np) * L2;
    double* slab1 = slab0 + SL;  // T0, then X2
    double* slab2 = slab1 + SL;  // T1, then X3
    double* slab3 = slab2 + SL;  // T3
    const int p0 = rank * np, p1 = min(Lg, p0 + np), mine = max(0, p1 - p0);
    long long* soff = reinterpret_cast<long long*>(slab3 + SL);
    const int t0lo = max(0, min(p0 / wn.TC, wn.ntile - 1) - (NC - 1));
    const int t0hi = min(wn.ntile - 1, max(p1 - 1, 0) / wn.TC);
    stage_tables(wn, sA, sS);
    if constexpr (kReduce) stage_offsets(wn, 3, t0lo, t0hi, soff);
    __syncthreads();
    pdl_wait();  // patches (G) come from the spread / tile_reduce (reduce) kernels
    patches = launder(patches);
    const DWin& wg = *launder(&wn);  // G: read through a pointer loaded after the wait
    // 1. node reduction of my planes (or my planes of the staged reduction's G)
    if constexpr (kReduce) {
#pragma unroll 3
        for (int k = threadIdx.x; k < mine * L2; k += blockDim.x) {
            const int e[3] = {p0 + k / L2, (k / Lg) % Lg, k % Lg};
            slab0[k] = node_sum<3, NC>(wn, patches, soff, t0lo, e);
        }
    } else {
        const double* __restrict__ G = wg.G + static_cast<long long>(p0) * L2;
#pragma unroll 4
        for (int k = threadIdx.x; k < mine * L2; k += blockDim.x) slab0[k] = __ldcg(G + k);
    }
    __syncthreads();
    // 2. stage 0 along dim 2: T0 = A2 g, T1 = S2 g (lines (p, i1), 4-output blocks)
    const int nb = (Lg + 3) >> 2;
    for (int k = threadIdx.x; k < mine * Lg * nb; k += blockDim.x) {
        const int line = k % (mine * Lg), i0 = (k / (mine * Lg)) * 4;
        const Acc8 r = line_conv1(sA, sS, slab0 + line * Lg, 1, Lg, i0);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u < Lg) {
                slab1[line * Lg + i0 + u] = r.a[u];
                slab2[line * Lg + i0 + u] = r.s[u];
            }
    }
    __syncthreads();
    // 3. stage 1 along dim 1: T2 = A1 T0 - S1 T1 (-> slab0), T3 = A1 T1 + S1 T0 (lines (p, i2))
    for (int k = threadIdx.x; k < mine * Lg * nb; k += blockDim.x) {
        const int i2 = k % Lg, p = (k / Lg) % max(mine, 1), i0 = (k / (mine * Lg)) * 4;
        const int base = p * L2 + i2;
        const Acc8 r = line_conv2(sA, sS, slab1 + base, slab2 + base, Lg, Lg, i0, true);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u < Lg) {
                slab0[base + (i0 + u) * Lg] = r.a[u];
                slab3[base + (i0 + u) * Lg] = r.s[u];
            }
    }
    cluster_barrier();  // every CTA's T2 / T3 slab complete and visible cluster-wide
    // 4. transpose: my dim-1 rows [q0, q1) of T2 / T3 over all planes j, from
    //    the owning CTAs' shared memory: X[(j * qn + qq) * Lg + i2]
    const int q0 = rank * np, q1 = min(Lg, q0 + np), qn = max(0, q1 - q0);
#pragma unroll 4
    for (int k = threadIdx.x; k < Lg * qn * Lg; k += blockDim.x) {
        const int i2 = k % Lg, qq = (k / Lg) % max(qn, 1), j = k / (qn * Lg);
        const int own = j / np, jj = j - own * np;
        const long long src = static_cast<long long>(jj) * L2 + (q0 + qq) * Lg + i2;
        const double* r2 = cl.map_shared_rank(slab0, own);
        const double* r3 = cl.map_shared_rank(slab3, own);
        slab1[k] = r2[src];
        slab2[k] = r3[src];
    }
    cluster_barrier();  // remote reads done: slabs may be released / exited
    // 5. stage 2 along dim 0: H = A0 X2 - S0 X3 (lines (qq, i2)), written to HBM
    double* __restrict__ H = wn.H;
    for (int k = threadIdx.x; k < qn * Lg * nb; k += blockDim.x) {
        const int line = k % (qn * Lg), i0 = (k / (qn * Lg)) * 4;
        const int i2 = line % Lg, qq = line / Lg;
        const Acc8 r = line_conv2(sA, sS, slab1 + line, slab2 + line, qn * Lg, Lg, i0, false);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u < Lg) H[(static_cast<long long>(i0 + u) * Lg + q0 + qq) * Lg + i2] = r.a[u];
    }
}

// d = 1, 2: one CTA per window (grid (1, nslots)). SMEM: tables + G, T0, T1.
template <int D, int NC>
__global__ void __launch_bounds__(kFusedThreads) grid12_fused_kernel(const DWin* __restrict__ wins,
                                                                     const int* __restrict__ slots,
                                                                     const double* __restrict__ patches) {
    pdl_trigger();
    const DWin& wn = wins[slots[blockIdx.y]];
    if (wn.d != D || wn.wrap) {
        pdl_wait();
        return;
    }
    const int Lg = wn.Lg, TL = tab_len(Lg);
    const int nodes = D == 1 ? Lg : Lg * Lg;
    extern __shared__ double smem[];
    double* sA = smem;
    double* sS = sA + TL;
    double* sG = sS + ((TL + 1) & ~1);
    double* sT0 = sG + nodes;
    double* sT1 = sT0 + nodes;
    long long* soff = reinterpret_cast<long long*>(sT1 + nodes);
    stage_tables(wn, sA, sS);
    stage_offsets(wn, D, 0, wn.ntile - 1, soff);
    __syncthreads();
    pdl_wait();
    patches = launder(patches);
    for (int k = threadIdx.x; k < nodes; k += blockDim.x) {
        int e[3] = {0, 0, 0};
        if (D == 1) {
            e[0] = k;
        } else {
            e[0] = k / Lg;
            e[1] = k % Lg;
        }
        sG[k] = node_sum<D, NC>(wn, patches, soff, 0, e);
    }
    __syncthreads();
    const int nb = (Lg + 3) >> 2;
    double* __restrict__ H = wn.H;
    if constexpr (D == 1) {  // H = A g
        for (int k = threadIdx.x; k < nb; k += blockDim.x) {
            const int i0 = 4 * k;
            const Acc8 r = line_conv1(sA, sS, sG, 1, Lg, i0);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u < Lg) H[i0 + u] = r.a[u];
        }
    } else {
    // stage 0 along dim 1: T0 = A1 g, T1 = S1 g (lines i0)
    for (int k = threadIdx.x; k < Lg * nb; k += blockDim.x) {
        const int line = k % Lg, i0 = (k / Lg) * 4;
        const Acc8 r = line_conv1(sA, sS, sG + line * Lg, 1, Lg, i0);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u < Lg) {
                sT0[line * Lg + i0 + u] = r.a[u];
                sT1[line * Lg + i0 + u] = r.s[u];
            }
    }
    __syncthreads();
    // stage 1 along dim 0: H = A0 T0 - S0 T1 (lines i1)
    for (int k = threadIdx.x; k < Lg * nb; k += blockDim.x) {
        const int i1 = k % Lg, i0 = (k / Lg) * 4;
        const Acc8 r = line_conv2(sA, sS, sT0 + i1, sT1 + i1, Lg, Lg, i0, false);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u < Lg) H[(i0 + u) * Lg + i1] = r.a[u];
    }
    }
}

// ---- host side ---------------------------------------------------------------

static size_t tables_doubles(int Lg) { return static_cast<size_t>(((2 * Lg + 6) + 1) & ~1) + (2 * Lg + 6); }

// Planes per CTA for d = 3 (C = ceil(Lg / np) CTAs per cluster, C <= 16).
int fused3_planes(int Lg) { return (Lg + kFusedMaxCluster - 1) / kFusedMaxCluster; }
int fused3_cluster_size(int Lg) {
    const int np = fused3_planes(Lg);
    return (Lg + np - 1) / np;
}

// Tile grid bound: ntile = ceil(ncell / TC) <= ceil(Lg / TC), TC = 4 / 8 / 32 for d = 3 / 2 / 1.
static long long tiles_bound(int D, int Lg) {
    const int TC = D == 3 ? 4 : (D == 2 ? 8 : 32);
    return (Lg + TC - 1) / TC;
}

size_t fused_smem_bytes(int D, int Lg) {
    const long long nt = tiles_bound(D, Lg);
    if (D == 3) {
        const long long np = fused3_planes(Lg);
        const long long n0 = 5 + (np + 3) / 4;  // T0 range of a slab: <= NC - 1 + ceil(np / TC) + 1
        return sizeof(double) * (tables_doubles(Lg) + 4 * np * Lg * Lg) + sizeof(long long) * n0 * nt * nt;
    }
    const long long nodes = D == 1 ? Lg : static_cast<long long>(Lg) * Lg;
    return sizeof(double) * (tables_doubles(Lg) + 3 * nodes) + sizeof(long long) * (D == 1 ? nt : nt * nt);
}

static cudaError_t set_fused_attrs(const void* f, bool cluster) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess && cluster) e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
}

cudaError_t init_fused_attributes() {
    cudaError_t e = cudaSuccess;
    for (const void* f : {reinterpret_cast<const void*>(grid3_fused_kernel<3>),
                          reinterpret_cast<const void*>(grid3_fused_kernel<5>),
                          reinterpret_cast<const void*>(grid3_fused_kernel<3, false>)})
        if (e == cudaSuccess) e = set_fused_attrs(f, true);
    for (const void* f : {reinterpret_cast<const void*>(grid12_fused_kernel<1, 2>),
                          reinterpret_cast<const void*>(grid12_fused_kernel<1, 5>),
                          reinterpret_cast<const void*>(grid12_fused_kernel<2, 2>),
                          reinterpret_cast<const void*>(grid12_fused_kernel<2, 5>)})
        if (e == cudaSuccess) e = set_fused_attrs(f, false);
    return e;
}

// Whether the d = 3 cluster shape for Lg can be resident on this device.
bool fused3_supported(int Lg, int NC) {
    const int np = fused3_planes(Lg);
    const int C = (Lg + np - 1) / np;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C, 1, 1);
    cfg.blockDim = dim3(kFusedThreads, 1, 1);
    cfg.dynamicSmemBytes = fused_smem_bytes(3, Lg);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    const void* f = NC == 3 ? reinterpret_cast<const void*>(grid3_fused_kernel<3>)
                            : reinterpret_cast<const void*>(grid3_fused_kernel<5>);
    if (cudaOccupancyMaxActiveClusters(&nclusters, f, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return nclusters > 0;
}

// One launch for the grid side of a class: D = 3 as clusters of C CTAs
// (one cluster per window slot), D = 1, 2 as one CTA per slot.
void launch_grid_fused(const DWin* wins, const int* slots, int nslots, int D, int NC, int Lg_max,
                       const double* patches, cudaStream_t st, bool conv_only) {
    if (nslots == 0) return;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kFusedThreads, 1, 1);
    cfg.dynamicSmemBytes = fused_smem_bytes(D, Lg_max);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    if (pdl_enabled()) ++na;
    if (D == 3) {
        const int np = fused3_planes(Lg_max);
        const int C = (Lg_max + np - 1) / np;
        cfg.gridDim = dim3(C, nslots, 1);
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = C;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
        cfg.attrs = attr;
        cfg.numAttrs = na;
        if (conv_only)
            (void)cudaLaunchKernelEx(&cfg, grid3_fused_kernel<3, false>, wins, slots, patches, np);
        else if (NC == 3)
            (void)cudaLaunchKernelEx(&cfg, grid3_fused_kernel<3>, wins, slots, patches, np);
        else
            (void)cudaLaunchKernelEx(&cfg, grid3_fused_kernel<5>, wins, slots, patches, np);
        return;
    }
    cfg.gridDim = dim3(1, nslots, 1);
    cfg.attrs = attr;
    cfg.numAttrs = na;
    if (D == 1) {
        if (NC == 2) (void)cudaLaunchKernelEx(&cfg, grid12_fused_kernel<1, 2>, wins, slots, patches);
        else (void)cudaLaunchKernelEx(&cfg, grid12_fused_kernel<1, 5>, wins, slots, patches);
    } else {
        if (NC == 2) (void)cudaLaunchKernelEx(&cfg, grid12_fused_kernel<2, 2>, wins, slots, patches);
        else (void)cudaLaunchKernelEx(&cfg, grid12_fused_kernel<2, 5>, wins, slots, patches);
    }
}

}  // namespace ksvm_nfft
