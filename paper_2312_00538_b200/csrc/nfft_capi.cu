// Host side of the B200 ANOVA-NFFT path and its C ABI (include/ksvm_nfft.h).
//
// Plan construction mirrors P:src/fastsum.cpp:103-209 exactly where it
// defines results (affine map, ell_scaled, the kept Fourier multipliers) and
// departs from it where only the execution strategy changes (points sorted
// into cell tiles on the device; the grid FFT pair replaced by the
// equivalent separable real convolution).
#include <cuda_runtime.h>

#include <algorithm>
#include <exception>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/ksvm_nfft.h"
#include "capi_common.cuh"
#include "nfft_engine.cuh"

namespace ksvm_nfft {

// launchers (nfft_kernels.cu)
cudaError_t init_kernel_attributes();
void launch_spread(int D, int S, int PE, const Item* items, int nitems, const DPSet* ps,
                   const DWin* wins, const double* v, double* patches, const int* colb, cudaStream_t st);
void launch_gather(int D, int S, int PE, const Item* items, int nitems, const DPSet* ps,
                   const DWin* wins, cudaStream_t st);
void launch_gather3c(const Item* items, int nitems, const DPSet* ps, const DWin* wins, const int* colb,
                     cudaStream_t st);
void launch_reduce(const DWin* wins, const int* slots, int nslots, long long max_nodes, int D, int S,
                   const double* patches, bool wrap, int max_tiles, cudaStream_t st);
void launch_tile_reduce(const DWin* wins, const int2* multi, int nmulti, int max_pv, double* patches,
                        cudaStream_t st);
void launch_conv(const DWin* wins, const int* slots, int nslots, int Lg_max, long long max_fibres,
                 int stage, cudaStream_t st);
int conv_max_lg();
// fused grid side (grid_fused.cu)
cudaError_t init_fused_attributes();
size_t fused_smem_bytes(int D, int Lg);
bool fused3_supported(int Lg, int NC);
int fused3_cluster_size(int Lg);
void launch_grid_fused(const DWin* wins, const int* slots, int nslots, int D, int NC, int Lg_max,
                       const double* patches, cudaStream_t st, bool conv_only);

void launch_combine(double* y, const double* const* src, const int* const* inv, const uint8_t* const* inv8,
                    const int* nu8, const double* eta, int P, long long lo, long long hi, cudaStream_t st);
void launch_bin_sums(const double* v, const uint8_t* const* codes, int nwl, long long n, double* partial,
                     int nblk, const long long* vs_off, const int* nu, double* vs, cudaStream_t st);
void launch_seg_sums(const double* v, const int* members, const int2* chunks, double* partial, int C,
                     const int* seg_cb, double* vs, int U, cudaStream_t st);
void launch_kernel_rows(double* out, const long long* rows, int r, const double* const* cols,
                        const int* wdim, const double* wgt, const double* ell2, int nw,
                        long long n, cudaStream_t st);
void launch_fill(double* out, double val, long long n, cudaStream_t st);
void launch_cell_keys(const double* x0, const double* x1, const double* x2, int d, long long n,
                      double Mf, int cmin, int ncell, int TC, int ntile, unsigned* keys, int* idx,
                      int* bad, cudaStream_t st);
void launch_factors(const double* x0, const double* x1, const double* x2, const int* perm, int d,
                    long long n, double Mf, int m, double invb, double Cw, int cmin, int TC,
                    int tile_rel, double4* F, int2* CP, cudaStream_t st);
// fp32 mode of the d = 3, m = 4 spread / gather (nfft_f32.cu)
cudaError_t init_f32_attributes();
void launch_spread3_f32(const Item* items, int nitems, const DPSet* ps, const DWin* wins, const double* v,
                        double* patches, cudaStream_t st);
void launch_gather3_f32(const Item* items, int nitems, const DPSet* ps, const DWin* wins, cudaStream_t st);
void launch_factors32(const double* x0, const double* x1, const double* x2, const int* perm, long long n,
                      double Mf, int m, double invb, double Cw, int cmin, int TC, float4* F, int2* CP,
                      cudaStream_t st);

namespace {

void ensure_attributes(int dev) {
    static std::mutex mu;
    static std::vector<bool> done(256, false);
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 256 && !done[static_cast<size_t>(dev)]) {
        CK(init_kernel_attributes());
        CK(init_fused_attributes());
        CK(init_f32_attributes());
        done[static_cast<size_t>(dev)] = true;
    }
}

// P:src/fastsum.cpp:38-47
void validate_cfg(const ksvm_nfft_config& c) {
    if (c.bandwidth < 2 || c.bandwidth % 2 != 0)
        throw std::invalid_argument("bandwidth must be a positive even integer");
    if (c.window_cutoff < 2 || c.window_cutoff > 8)
        throw std::invalid_argument("window_cutoff must lie in [2, 8]");
    if (c.oversampling < 1) throw std::invalid_argument("oversampling must be >= 1");
    if (!(c.torus_radius > 0.0 && c.torus_radius <= 0.25))
        throw std::invalid_argument("torus_radius must lie in (0, 1/4]");
}

inline double at(const double* p, int64_t i, int64_t j, int64_t ld, int layout) {
    return layout == KSVM_NFFT_COL_MAJOR ? p[j * ld + i] : p[i * ld + j];
}

void check_layout(int64_t n, int64_t d, int64_t ld, int layout) {
    if (layout != KSVM_NFFT_ROW_MAJOR && layout != KSVM_NFFT_COL_MAJOR)
        throw std::invalid_argument("layout must be KSVM_NFFT_ROW_MAJOR or KSVM_NFFT_COL_MAJOR");
    if (layout == KSVM_NFFT_ROW_MAJOR ? ld < d : ld < n)
        throw std::invalid_argument("leading dimension too small");
}

const long double kPi = 3.141592653589793238462643383279502884L;

// Per-dimension Fourier data of the rescaled Gaussian (P:src/fastsum.cpp:142-199).
// The reference's d-dim coefficients are products of these 1-D factors:
// b_J = prod_t b1[J_t] (the N^d samples are a tensor product), and so is the
// multiplier mult[J] = b_J * prod_t exp(2 b (pi J_t / M)^2) = prod_t m1[J_t].
struct Spectral1D {
    std::vector<long double> b1, m1;  // index J + N/2, J in I_N = [-N/2, N/2)
};

Spectral1D spectral_1d(int N, int M, double bwin, double ell_s) {
    Spectral1D s;
    s.b1.assign(static_cast<size_t>(N), 0.0L);
    s.m1.assign(static_cast<size_t>(N), 0.0L);
    const long double inv_l2 = 1.0L / (static_cast<long double>(ell_s) * ell_s);
    std::vector<long double> f(static_cast<size_t>(N));
    for (int k = 0; k < N; ++k) {
        const long double c = static_cast<long double>(k < N / 2 ? k : k - N) / N;
        f[static_cast<size_t>(k)] = std::exp(-c * c * inv_l2);
    }
    for (int J = -N / 2; J < N / 2; ++J) {
        long double acc = 0.0L;
        for (int k = 0; k < N; ++k) {
            const long long ph = ((static_cast<long long>(k) * J) % N + N) % N;  // exact reduction
            acc += f[static_cast<size_t>(k)] * std::cos(2.0L * kPi * ph / N);
        }
        const long double bJ = acc / N;
        const long double arg = kPi * J / M;
        s.b1[static_cast<size_t>(J + N / 2)] = bJ;
        s.m1[static_cast<size_t>(J + N / 2)] = bJ * std::exp(2.0L * bwin * arg * arg);
    }
    return s;
}

struct Geometry {
    int M, S, m, cmin, ncell, TC, ntile, PE, Lext, Lg, lo, wrap;
    double bwin, invb, Cw;
};

struct PointSet {
    int64_t n = 0;
    int d = 0;
    DevBuf<double4> F;  // window factors {P, Q0, Q1, Q2}, sorted order (nfft_engine.cuh)
    DevBuf<float4> F32; // fp32 mode (d = 3, m = 4): cell-relative factors instead of F (nfft_f32.cu)
    DevBuf<int2> CP;    // {tile-local cell code, original index}
    DevBuf<int> perm;
    std::vector<Item> items;      // spread items (one patch each; global numbering later)
    std::vector<int> tile_first;  // local item index of each tile's first spread item
    std::vector<Item> gitems;     // gather items (finer: no patch cost, better balance)
    // d = 3, TC = 4: per spread item, the first point of cell columns
    // 0..16 (column = l0 * 4 + l1; kColBounds entries per item), the warp
    // ranges of spread3c / gather3c
    std::vector<int> colb;
};

struct Window {
    int d = 0;
    int feat[3] = {0, 0, 0};
    double ell = 1.0, eta = 1.0;
    bool owned = true;
    // affine map (P:src/fastsum.cpp:126-140)
    double center[3] = {0, 0, 0};
    double scale = 1.0, ell_s = 0.0, coef_sum = 0.0;
    DWin dw{};
    Geometry geom{};
    DevBuf<double> G, H, T[4], tabA, tabS;
    DevBuf<int> tile_first;
    DevBuf<long long> tile_patch;
    PointSet src;
    // Exact duplicates (operators only): the window runs on its nu distinct
    // scaled points; members (CSR by distinct point, ascending original
    // index) feed the segmented sum of v, inv maps each point to its
    // distinct point for the output broadcast.
    int64_t nu = 0;  // 0: no dedup
    std::vector<int> offs, members;  // nu > kSmallBins only
    DevBuf<int> inv;                 // nu > kSmallBins
    DevBuf<uint8_t> inv8;            // nu <= kSmallBins (register-bin sums)
};

// Distinct points of a window's scaled coordinates (column-major n x d),
// compared bit for bit: identical coordinates give identical kernel rows and
// columns, so K~ v = K~_u (sum of v over each duplicate group) exactly up to
// summation order. Used only when it shrinks the point count at least
// kDedupRatio-fold; a leading sample rejects continuous data cheaply.
constexpr int64_t kDedupRatio = 8;

bool dedup_enabled() {  // KSVM_NFFT_DEDUP=0 turns the duplicate merge off
    const char* e = std::getenv("KSVM_NFFT_DEDUP");
    return !(e && e[0] == '0');
}

struct DedupKey {
    uint64_t x[3];
    bool operator==(const DedupKey& o) const { return x[0] == o.x[0] && x[1] == o.x[1] && x[2] == o.x[2]; }
};
struct DedupHash {
    size_t operator()(const DedupKey& k) const {
        uint64_t h = 1469598103934665603ull;
        for (uint64_t v : k.x) h = (h ^ v) * 1099511628211ull ^ (v >> 29);
        return static_cast<size_t>(h);
    }
};

bool find_duplicates(const std::vector<double>& sc, int64_t n, int d, std::vector<int>& inv, int64_t& nu) {
    auto key = [&](int64_t i) {
        DedupKey k{{0, 0, 0}};
        for (int t = 0; t < d; ++t) std::memcpy(&k.x[t], &sc[static_cast<size_t>(t * n + i)], sizeof(double));
        return k;
    };
    const int64_t sample = std::min<int64_t>(n, 4096);
    {
        std::unordered_map<DedupKey, int, DedupHash> ids;
        for (int64_t i = 0; i < sample; ++i) {
            ids.emplace(key(i), 0);
            if (static_cast<int64_t>(ids.size()) * kDedupRatio > sample) return false;
        }
    }
    std::unordered_map<DedupKey, int, DedupHash> ids;
    ids.reserve(static_cast<size_t>(n / kDedupRatio + 1));
    inv.assign(static_cast<size_t>(n), 0);
    for (int64_t i = 0; i < n; ++i) {
        auto r = ids.emplace(key(i), static_cast<int>(ids.size()));
        inv[static_cast<size_t>(i)] = r.first->second;
        if (static_cast<int64_t>(ids.size()) * kDedupRatio > n) return false;
    }
    nu = static_cast<int64_t>(ids.size());
    return n >= 2 * kDedupRatio;
}

// Grid geometry of one window. Without `range` it covers every admissible
// point (sources: |x| <= fit r_T; cross targets: ||x|| <= r_T (1 + 1e-12),
// P:src/fastsum.cpp:316). With range = {min, max} of the scaled source
// coordinates over all dimensions (ANOVA operators, which only self-apply)
// it covers just the cells the data occupy. The plan-time cell-key kernel
// verifies every point lands in [cmin, cmax].
Geometry geometry(const ksvm_nfft_config& c, int d, const double* range = nullptr) {
    Geometry g{};
    g.M = c.oversampling * c.bandwidth;
    g.m = c.window_cutoff;
    g.S = 2 * g.m;
    const double rx = c.torus_radius * (1.0 + 1e-12) * g.M;
    g.cmin = static_cast<int>(std::floor(-rx));
    int cmax = static_cast<int>(std::floor(rx));
    if (range) {
        g.cmin = std::max(g.cmin, static_cast<int>(std::floor(range[0] * g.M)));
        cmax = std::min(cmax, static_cast<int>(std::floor(range[1] * g.M)));
    }
    g.ncell = std::max(1, cmax - g.cmin + 1);
    g.TC = d == 3 ? 4 : (d == 2 ? 8 : 32);
    g.ntile = (g.ncell + g.TC - 1) / g.TC;
    g.PE = g.TC + g.S - 1;
    g.Lext = g.ncell + g.S - 1;
    g.lo = g.cmin - g.m + 1;
    g.wrap = g.Lext > g.M ? 1 : 0;
    g.Lg = g.wrap ? g.M : g.Lext;
    if (g.Lg > conv_max_lg())
        throw std::invalid_argument("oversampled grid edge too large for this build (local grid edge > " +
                                    std::to_string(conv_max_lg()) + ")");
    const double sg = static_cast<double>(c.oversampling);
    g.bwin = (2.0 * sg * g.m) / ((2.0 * sg - 1.0) * 3.14159265358979323846);  // P:src/fastsum.cpp:123-124
    g.invb = 1.0 / g.bwin;
    g.Cw = 1.0 / std::sqrt(3.14159265358979323846 * g.bwin);
    return g;
}

// Sort a point set by (tile, cell) on the device and split tiles into items.
void build_pointset(PointSet& ps, const std::vector<double>& scaled_cm, int64_t n, int d,
                    const Geometry& g, int64_t chunk_points, int64_t gather_chunk, cudaStream_t st,
                    bool f32 = false) {
    ps.n = n;
    ps.d = d;
    DevBuf<double> raw[3];
    for (int t = 0; t < d; ++t) raw[t].upload(scaled_cm.data() + static_cast<size_t>(t) * n, n, st);
    DevBuf<unsigned> keys_in, keys_out;
    DevBuf<int> idx_in, bad;
    keys_in.alloc(n);
    keys_out.alloc(n);
    idx_in.alloc(n);
    ps.perm.alloc(n);
    bad.alloc(1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    launch_cell_keys(raw[0].p, d > 1 ? raw[1].p : nullptr, d > 2 ? raw[2].p : nullptr, d, n,
                     static_cast<double>(g.M), g.cmin, g.ncell, g.TC, g.ntile, keys_in.p,
                     idx_in.p, bad.p, st);
    CK(cudaGetLastError());
    unsigned maxkey = 1;
    for (int t = 0; t < d; ++t) maxkey *= static_cast<unsigned>(g.ntile * g.TC);
    int bits = 1;
    while ((1u << bits) < maxkey && bits < 32) ++bits;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in.p, keys_out.p, idx_in.p,
                                       ps.perm.p, static_cast<int>(n), 0, bits, st));
    DevBuf<unsigned char> tmp;
    tmp.alloc(tmp_bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys_in.p, keys_out.p, idx_in.p,
                                       ps.perm.p, static_cast<int>(n), 0, bits, st));
    ps.CP.alloc(n);
    ps.F.alloc(n);
    launch_factors(raw[0].p, d > 1 ? raw[1].p : nullptr, d > 2 ? raw[2].p : nullptr, ps.perm.p, d, n,
                   static_cast<double>(g.M), g.m, g.invb, g.Cw, g.cmin, g.TC,
                   /*tile_rel=*/(d == 3 && g.S == 8) ? 1 : 0, ps.F.p, ps.CP.p, st);
    if (f32) {  // fp32 mode (d = 3, m = 4): cell-relative float factors too; the
                // engine keeps one of F / F32 once it knows the class density
        ps.F32.alloc(n);
        launch_factors32(raw[0].p, raw[1].p, raw[2].p, ps.perm.p, n, static_cast<double>(g.M), g.m, g.invb,
                         g.Cw, g.cmin, g.TC, ps.F32.p, ps.CP.p, st);
    }
    CK(cudaGetLastError());
    std::vector<unsigned> hk(static_cast<size_t>(n));
    int hbad = 0;
    CK(cudaMemcpyAsync(hk.data(), keys_out.p, sizeof(unsigned) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hbad) throw std::runtime_error("internal: point outside the planned cell range");

    unsigned tcd = 1;
    int ntiles = 1;
    for (int t = 0; t < d; ++t) {
        tcd *= static_cast<unsigned>(g.TC);
        ntiles *= g.ntile;
    }
    // Items: tiles split into chunks of <= chunk_points points (fixed at plan
    // time, so the summation order -- and hence every bit of the result -- is
    // a function of the plan alone).
    ps.items.clear();
    ps.gitems.clear();
    ps.colb.clear();
    ps.tile_first.assign(static_cast<size_t>(ntiles) + 1, 0);
    auto split = [](std::vector<Item>& out, int T, int64_t i, int64_t cnt, int64_t chunk) {
        const int64_t pieces = (cnt + chunk - 1) / chunk;
        for (int64_t q = 0; q < pieces; ++q) {
            Item it{};
            it.tile = T;
            it.begin = static_cast<int>(i + cnt * q / pieces);
            it.end = static_cast<int>(i + cnt * (q + 1) / pieces);
            out.push_back(it);
        }
    };
    int64_t i = 0;
    for (int T = 0; T < ntiles; ++T) {
        ps.tile_first[static_cast<size_t>(T)] = static_cast<int>(ps.items.size());
        int64_t j = i;
        while (j < n && hk[static_cast<size_t>(j)] / tcd == static_cast<unsigned>(T)) ++j;
        const int64_t cnt = j - i;
        if (cnt > 0) {
            const size_t first = ps.items.size();
            split(ps.items, T, i, cnt, chunk_points);
            split(ps.gitems, T, i, cnt, gather_chunk);
            if (d == 3 && g.TC == 4) {
                for (size_t q = first; q < ps.items.size(); ++q) {
                    const Item& it = ps.items[q];
                    int p = it.begin;
                    for (int b = 0; b < kColBounds; ++b) {  // first point of column b
                        while (p < it.end && static_cast<int>((hk[static_cast<size_t>(p)] % tcd) >> 2) < b) ++p;
                        ps.colb.push_back(p);
                    }
                }
            }
        }
        i = j;
    }
    ps.tile_first[static_cast<size_t>(ntiles)] = static_cast<int>(ps.items.size());
}

// Points per spread item: ~24 items per SM over all windows of the operator
// (load balance) but no more, since each item writes one (TC+2m-1)^d patch
// that must be reduced; d = 3 items hold >= 1024 points (measured: 2048
// left config 3's dense tiles too coarse, 512 cost more patch reduction).
// Gather items carry no patch, so they are finer.
int64_t item_chunk(int64_t total_points, int d) {
    // d = 3: large items (a 4^3-cell tile is rarely split, so no pre-reduce);
    // d <= 2 have few, large tiles and need splitting for parallelism
    int64_t floor_pts = d == 3 ? 1024 : 512;
    if (const char* e = std::getenv(d == 3 ? "KSVM_NFFT_ITEM3" : "KSVM_NFFT_ITEM12")) floor_pts = std::max(32, std::atoi(e));
    static const int64_t div = [] {  // items per SM target (A/B knob)
        const char* e = std::getenv("KSVM_NFFT_ITEMS_PER_SM");
        return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t{24};
    }();
    return std::max<int64_t>(floor_pts, (total_points + 148 * div - 1) / (148 * div));
}
// d = 3 gather items load an 11^3 halo (10.6 KB) each: >= 512 points
// amortise it (config 3: 0.1865 -> 0.1721 ms); d <= 2 halos are small, so
// finer items balance better (config 2's d = 2 gather).
int64_t gather_chunk(int64_t total_points, int d) {
    int64_t floor_pts = d == 3 ? 512 : 128;
    if (const char* e = std::getenv("KSVM_NFFT_GITEM")) floor_pts = std::max(32, std::atoi(e));
    static const int64_t div = [] {
        const char* e = std::getenv("KSVM_NFFT_GITEMS_PER_SM");
        return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t{48};
    }();
    return std::max<int64_t>(floor_pts, (total_points + 148 * div - 1) / (148 * div));
}

// Affine map of P:src/fastsum.cpp:126-140 on a column-major n x d block.
void affine_map(Window& w, const double* cm, int64_t n, double fit, double rT) {
    const int d = w.d;
    for (int t = 0; t < d; ++t) {
        double hi = cm[static_cast<size_t>(t) * n], lo = hi;
        for (int64_t i = 1; i < n; ++i) {
            const double x = cm[static_cast<size_t>(t * n + i)];
            hi = std::max(hi, x);
            lo = std::min(lo, x);
        }
        w.center[t] = 0.5 * (hi + lo);
    }
    double radius = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int t = 0; t < d; ++t) {
            const double diff = cm[static_cast<size_t>(t * n + i)] - w.center[t];
            s += diff * diff;
        }
        radius = std::max(radius, std::sqrt(s));
    }
    w.scale = radius > 0.0 ? fit * rT / radius : 1.0;
    w.ell_s = w.scale * w.ell;
    if (w.ell_s > rT && std::getenv("KSVM_NFFT_QUIET") == nullptr)
        std::fprintf(stderr,
                     "ksvm: warning: scaled length scale %g exceeds torus radius %g; "
                     "periodization error may be large\n",
                     w.ell_s, rT);
}

std::vector<double> scale_cm(const Window& w, const double* pts, int64_t t, int64_t ld, int layout,
                             const int* cols) {
    std::vector<double> out(static_cast<size_t>(t) * w.d);
    for (int c = 0; c < w.d; ++c)
        for (int64_t i = 0; i < t; ++i)
            out[static_cast<size_t>(c * t + i)] =
                (at(pts, i, cols[c], ld, layout) - w.center[c]) * w.scale;
    return out;
}

}  // namespace

// ---------------------------------------------------------------------------
// The engine: every owned window's plan plus the per-apply scratch.
// ---------------------------------------------------------------------------
constexpr long long kColumnDensity = 10;
constexpr int kBatchLanes = 4;  // concurrent applies of a multi-RHS batch  // points per cell below which spread3c runs

struct Engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side[4] = {nullptr, nullptr, nullptr, nullptr};  // class branches (d = 1, 2)
    cudaEvent_t ev_fork = nullptr, ev_join[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    static constexpr int kMaxTicks = 24;
    cudaEvent_t ev_stage[kMaxTicks] = {};
    const char* tick_name[kMaxTicks] = {};
    int nticks = 0, last_nticks = 0;
    int stage_timing = 0;  // 0 off; 1 every launch, classes serialised; 2 main branch only, branches kept
    cudaStream_t tick_stream = nullptr;  // stream of the class being enqueued (mode 2 ticks only there)
    ksvm_nfft_config cfg{};
    double fit = 1.0;
    int precision = KSVM_NFFT_FP64;
    // fp32 mode covers the d = 3, m = 4 windows with dense cells (the
    // FP64-bound part). Sparse-cell classes are latency-bound and keep the
    // fp64 column kernels (faster there; exact, so within the 1e-5 contract);
    // KSVM_NFFT_F32=all forces the fp32 kernels on them too. d <= 2 windows,
    // the grid side and the window sum stay fp64.
    bool f32_want(int D) const { return precision == KSVM_NFFT_FP32 && D == 3 && cfg.window_cutoff == 4; }
    bool f32_dense[4] = {false, false, false, false};  // decided in finalize()
    bool f32_class(int D) const { return f32_dense[D]; }
    int64_t n = 0;
    int64_t dfull = 0;
    std::vector<std::unique_ptr<Window>> wins;  // all windows, window order
    std::vector<int> owned;                     // window indices owned here, ascending
    std::vector<double> raw_rm;                 // row-major window features (entries)
    std::vector<int> raw_cols;                  // feature index of each raw_rm column
    // device state
    DevBuf<DWin> d_wins;    // owned windows (slot = position in `owned`)
    DevBuf<DPSet> d_ps;     // sources of owned windows
    DevBuf<Item> d_items;   // spread items of owned windows, grouped by d
    DevBuf<int> d_colb;     // column bounds of the d = 3 spread items (PointSet::colb)
    DevBuf<Item> d_gitems;  // gather items of owned windows, grouped by d
    int gclass_begin[4] = {0, 0, 0, 0}, gclass_end[4] = {0, 0, 0, 0};
    DevBuf<int> d_slots;    // 0..P_owned-1
    DevBuf<int2> d_multi;   // (slot, tile) of tiles split into several items, grouped by d
    int n_multi = 0, max_pv = 0;
    int multi_begin[4] = {0, 0, 0, 0}, n_multi_cls[4] = {0, 0, 0, 0};
    int slot_begin[4] = {0, 0, 0, 0}, nslots_cls[4] = {0, 0, 0, 0};  // d_slots grouped by d
    // fused grid side per class (grid_fused.cu): reduce + all conv stages in one launch
    bool grid_fused[4] = {false, false, false, false};
    bool grid_conv_only[4] = {false, false, false, false};  // d = 3: staged reduce + fused conv cluster
    int grid_nc[4] = {0, 0, 0, 0}, grid_lg[4] = {0, 0, 0, 0};
    DevBuf<double> d_eta;
    DevBuf<double> patches, parts, vbuf, ybuf;
    DevBuf<double> gpool;  // point-sharded operators: the owned windows' grids G, contiguous
    int64_t gpool_len = 0;
    // exact-duplicate windows (Window::nu): segmented sums of v and output maps
    DevBuf<int> seg_members, seg_cb;
    DevBuf<int2> seg_chunks;
    DevBuf<double> seg_partial, vs_all, uout_all;
    int n_seg_chunks = 0, n_segs = 0;
    DevBuf<const double*> d_src;
    DevBuf<const int*> d_inv;
    DevBuf<const uint8_t*> d_inv8, d_codes;  // combine maps; codes of the register-bin windows
    DevBuf<int> d_nu8;                       // distinct points of each register-bin window (0: other)
    DevBuf<long long> d_small_off;
    DevBuf<int> d_small_nu;
    DevBuf<double> bin_partial;
    int n_small = 0;
    static constexpr int kBinBlocks = 148 * 2;
    DevBuf<double> d_raw;   // SoA raw window features (entries), original order
    DevBuf<const double*> d_rawcols;
    DevBuf<int> d_wdim;
    int class_begin[4] = {0, 0, 0, 0}, class_end[4] = {0, 0, 0, 0};
    int class_PE[4] = {0, 0, 0, 0};
    bool spread_columns[4] = {false, false, false, false};  // d = 3: column-accumulating spread
    bool gather_columns[4] = {false, false, false, false};  // d = 3: column-slab gather
    long long max_nodes = 0, max_fibres = 0;
    int max_lg = 0;
    bool has_dim[4] = {false, false, false, false};
    std::mutex mu;
    float last_ms[kMaxTicks] = {};
    const char* last_name[kMaxTicks] = {};

    ~Engine() {
        if (stream) {
            cudaSetDevice(device);
            cudaStreamSynchronize(stream);
            drop_graphs();
            for (int D = 1; D <= 2; ++D) {
                if (side[D]) {
                    cudaStreamSynchronize(side[D]);
                    cudaStreamDestroy(side[D]);
                }
                if (ev_join[D]) cudaEventDestroy(ev_join[D]);
            }
            if (ev_fork) cudaEventDestroy(ev_fork);
            cudaStreamDestroy(stream);
            cudaEventDestroy(ev_in);
            cudaEventDestroy(ev_out);
            for (auto& ev : ev_stage)
                if (ev) cudaEventDestroy(ev);
        }
    }

    int P_owned() const { return static_cast<int>(owned.size()); }

    // Device SoA copy of the raw window features (entries), built on first use.
    std::mutex raw_mu;
    void ensure_raw_device() {
        std::lock_guard<std::mutex> lk(raw_mu);
        if (d_raw.p) return;
        DeviceGuard dg(device);
        const size_t nc = raw_cols.size();
        std::vector<double> soa(static_cast<size_t>(n) * nc);
        for (int64_t i = 0; i < n; ++i)
            for (size_t c = 0; c < nc; ++c) soa[c * static_cast<size_t>(n) + static_cast<size_t>(i)] = raw_rm[static_cast<size_t>(i) * nc + c];
        DevBuf<double> buf;
        buf.upload(soa.data(), soa.size(), stream);
        std::vector<const double*> cols(nc);
        for (size_t c = 0; c < nc; ++c) cols[c] = buf.p + c * static_cast<size_t>(n);
        d_rawcols.upload(cols.data(), cols.size(), stream);
        CK(cudaStreamSynchronize(stream));
        d_raw = std::move(buf);
    }
    int64_t n_owned_windows = 1;  // set before planning (item sizing)
    bool data_range = false;      // grid range from the data (self-apply only operators)
    // Point sharding (SURVEY.md 8(e) hybrid): this operator spreads / gathers
    // only the points own_idx (ascending global indices) while its grids are
    // planned from all n points, so every rank's grid is the same and the
    // partial grids add up (ksvm_nfft_op_apply_spread / _grids / _finish).
    std::vector<int64_t> own_idx;
    bool sharded() const { return !own_idx.empty(); }
    bool has_wrap[4] = {false, false, false, false}, has_nowrap[4] = {false, false, false, false};
    int max_tiles[4] = {0, 0, 0, 0};

    void init(int dev) {
        device = dev;
        CK(cudaSetDevice(dev));
        ensure_attributes(dev);
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        for (int D = 1; D <= 2; ++D) {
            CK(cudaStreamCreateWithFlags(&side[D], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ev_join[D], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
        stage_timing = std::getenv("KSVM_NFFT_STAGE_TIMING") != nullptr ? 1 : 0;
        for (auto& e : ev_stage) CK(cudaEventCreate(&e));
    }

    // plan_fastsum for one window (P:src/fastsum.cpp:103-209) on the device.
    // Host half of plan_fastsum for one window: affine map, scaled
    // coordinates, data range. Touches only w and `out` (windows run on
    // concurrent host threads).
    struct WinPrep {
        std::vector<double> sc;
        double range[2] = {0.0, 0.0};
    };
    void prep_window(Window& w, const double* cm, WinPrep& out) const {
        const int d = w.d;
        affine_map(w, cm, n, fit, cfg.torus_radius);
        std::vector<double>& sc = out.sc;
        sc.resize(static_cast<size_t>(n) * d);
        for (int t = 0; t < d; ++t)
            for (int64_t i = 0; i < n; ++i)
                sc[static_cast<size_t>(t * n + i)] = (cm[static_cast<size_t>(t * n + i)] - w.center[t]) * w.scale;
        if (data_range) {
            out.range[0] = out.range[1] = sc[0];
            for (double x : sc) {
                out.range[0] = std::min(out.range[0], x);
                out.range[1] = std::max(out.range[1], x);
            }
        }
    }

    void plan_window(Window& w, WinPrep& prep) {
        const int d = w.d;
        std::vector<double>& sc = prep.sc;
        const double* range = prep.range;
        const Geometry g = geometry(cfg, d, data_range ? range : nullptr);
        w.geom = g;
        const double bwin = g.bwin;
        // spectral data and the separable convolution tables
        const Spectral1D sp = spectral_1d(cfg.bandwidth, g.M, bwin, w.ell_s);
        long double csum1 = 0.0L;
        for (long double b : sp.b1) csum1 += b;
        long double cs = 1.0L;
        for (int t = 0; t < d; ++t) cs *= csum1;
        w.coef_sum = static_cast<double>(cs);
        const int Lg = g.Lg, N = cfg.bandwidth;
        std::vector<double> ta(static_cast<size_t>(2 * Lg - 1)), ts(static_cast<size_t>(2 * Lg - 1));
        for (int r = -(Lg - 1); r <= Lg - 1; ++r) {
            long double ca = 0.0L, cs2 = 0.0L;
            for (int J = -N / 2; J < N / 2; ++J) {
                const long long ph = ((static_cast<long long>(J) * r) % g.M + g.M) % g.M;
                const long double ang = 2.0L * kPi * ph / g.M;
                ca += sp.m1[static_cast<size_t>(J + N / 2)] * std::cos(ang);
                cs2 += sp.m1[static_cast<size_t>(J + N / 2)] * std::sin(ang);
            }
            ta[static_cast<size_t>(r + Lg - 1)] = static_cast<double>(ca);
            ts[static_cast<size_t>(r + Lg - 1)] = static_cast<double>(cs2);
        }
        w.tabA.upload(ta.data(), ta.size(), stream);
        w.tabS.upload(ts.data(), ts.size(), stream);
        long long nodes = 1;
        for (int t = 0; t < d; ++t) nodes *= Lg;
        max_nodes = std::max(max_nodes, nodes);
        max_fibres = std::max(max_fibres, nodes / Lg);
        max_lg = std::max(max_lg, Lg);
        has_dim[d] = true;
        (g.wrap ? has_wrap : has_nowrap)[d] = true;
        int tiles = 1;  // owner blocks of the node reduction: ceil(Lg / TC)^d
        for (int t = 0; t < d; ++t) tiles *= (Lg + g.TC - 1) / g.TC;
        max_tiles[d] = std::max(max_tiles[d], tiles);
        w.G.alloc(nodes);
        w.H.alloc(nodes);
        for (int k = 0; k < (d == 1 ? 0 : (d == 2 ? 2 : 4)); ++k) w.T[k].alloc(nodes);
        std::vector<int> inv;
        int64_t nu = 0;
        if (sharded()) {
            w.nu = 0;
            const int64_t no = static_cast<int64_t>(own_idx.size());
            std::vector<double> so(static_cast<size_t>(no) * d);
            for (int t = 0; t < d; ++t)
                for (int64_t r = 0; r < no; ++r)
                    so[static_cast<size_t>(t * no + r)] = sc[static_cast<size_t>(t * n + own_idx[static_cast<size_t>(r)])];
            build_pointset(w.src, so, no, d, g, item_chunk(no * n_owned_windows, d),
                           gather_chunk(no * n_owned_windows, d), stream, f32_want(d));
            // point-set indices are local to the owned rows: map them to global ones
            std::vector<int2> cp(static_cast<size_t>(no));
            CK(cudaMemcpyAsync(cp.data(), w.src.CP.p, sizeof(int2) * cp.size(), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            for (auto& e : cp) e.y = static_cast<int>(own_idx[static_cast<size_t>(e.y)]);
            CK(cudaMemcpyAsync(w.src.CP.p, cp.data(), sizeof(int2) * cp.size(), cudaMemcpyHostToDevice, stream));
            CK(cudaStreamSynchronize(stream));
        } else if (data_range && dedup_enabled() && find_duplicates(sc, n, d, inv, nu)) {
            // distinct points (first occurrence order) and the CSR member lists
            std::vector<double> su(static_cast<size_t>(nu) * d);
            std::vector<int> first(static_cast<size_t>(nu), -1);
            w.offs.assign(static_cast<size_t>(nu) + 1, 0);
            for (int64_t i = 0; i < n; ++i) {
                const int u = inv[static_cast<size_t>(i)];
                if (first[static_cast<size_t>(u)] < 0) first[static_cast<size_t>(u)] = static_cast<int>(i);
                ++w.offs[static_cast<size_t>(u) + 1];
            }
            for (int64_t u = 0; u < nu; ++u) {
                w.offs[static_cast<size_t>(u) + 1] += w.offs[static_cast<size_t>(u)];
                for (int t = 0; t < d; ++t)
                    su[static_cast<size_t>(t * nu + u)] =
                        sc[static_cast<size_t>(t * n + first[static_cast<size_t>(u)])];
            }
            w.nu = nu;
            if (nu <= kSmallBins) {
                std::vector<uint8_t> i8(inv.begin(), inv.end());
                w.inv8.upload(i8.data(), i8.size(), stream);
                w.offs.clear();
            } else {
                w.members.assign(static_cast<size_t>(n), 0);
                std::vector<int> fill(w.offs.begin(), w.offs.end() - 1);
                for (int64_t i = 0; i < n; ++i)
                    w.members[static_cast<size_t>(fill[static_cast<size_t>(inv[static_cast<size_t>(i)])]++)] =
                        static_cast<int>(i);
                w.inv.upload(inv.data(), inv.size(), stream);
            }
            build_pointset(w.src, su, nu, d, g, item_chunk(n * n_owned_windows, d),
                           gather_chunk(n * n_owned_windows, d), stream, f32_want(d));
        } else {
            w.nu = 0;
            build_pointset(w.src, sc, n, d, g, item_chunk(n * n_owned_windows, d),
                           gather_chunk(n * n_owned_windows, d), stream, f32_want(d));
        }

        DWin& dw = w.dw;
        dw.d = d;
        dw.S = g.S;
        dw.m = g.m;
        dw.M = g.M;
        dw.Lg = Lg;
        dw.lo = g.lo;
        dw.wrap = g.wrap;
        dw.cmin = g.cmin;
        dw.ncell = g.ncell;
        dw.TC = g.TC;
        dw.ntile = g.ntile;
        dw.PE = g.PE;
        dw.Lext = g.Lext;
        dw.Mf = static_cast<double>(g.M);
        dw.bwin = bwin;
        dw.invb = g.invb;
        dw.Cw = g.Cw;
        for (int o = 0; o < kMaxSpan; ++o) dw.R[o] = std::exp(-static_cast<double>(o) * o / bwin);
        dw.G = w.G.p;
        dw.H = w.H.p;
        for (int k = 0; k < 4; ++k) dw.T[k] = w.T[k].p;
        dw.tabA = w.tabA.p;
        dw.tabS = w.tabS.p;
    }

    // Sparse cells favour the column kernels for d = 3 (spread: one SMEM
    // flush per cell column; gather: one fragment load per column; both:
    // full point groups); dense cells the per-cell kernels (fewer FP64
    // operations per point).
    // Threshold: mean points per cell of the occupied tiles.
    bool use_columns(int D, const char* env) const {
        if (const char* e = std::getenv(env)) return std::strcmp(e, "column") == 0;
        return sparse_cells(D);
    }
    bool sparse_cells(int D) const {
        long long pts = 0, cells = 0;
        for (size_t s = 0; s < owned.size(); ++s) {
            const Window& w = *wins[static_cast<size_t>(owned[s])];
            if (w.d != D || w.dw.S != 8) continue;
            const std::vector<int>& tf = w.src.tile_first;
            long long occ = 0;
            for (size_t T = 0; T + 1 < tf.size(); ++T) occ += tf[T + 1] > tf[T] ? 1 : 0;
            pts += w.src.n;
            cells += occ * w.dw.TC * w.dw.TC * w.dw.TC;
        }
        return cells > 0 && pts < kColumnDensity * cells;
    }

    // KSVM_NFFT_LPT=0 keeps the items in (window, tile) order (A/B knob).
    static int lpt_items() {  // read per plan (tests compare both orders in one process)
        const char* e = std::getenv("KSVM_NFFT_LPT");
        return e ? std::atoi(e) : 1;
    }

    // Assign global item numbers / patch offsets and upload device tables.
    void finalize() {
        const int P = P_owned();
        std::vector<Item> all, gall;
        std::vector<int> colb;  // kColBounds per item of `all` (zeros unless d = 3, TC = 4)
        std::vector<int2> multi;
        std::vector<DPSet> ps(static_cast<size_t>(P));
        long long patch_total = 0;
        for (int D = 1; D <= 3; ++D) {
            class_begin[D] = static_cast<int>(all.size());
            multi_begin[D] = static_cast<int>(multi.size());
            for (int s = 0; s < P; ++s) {
                Window& w = *wins[static_cast<size_t>(owned[static_cast<size_t>(s)])];
                if (w.d != D) continue;
                int PV = 1;
                for (int t = 0; t < D; ++t) PV *= w.dw.PE;
                class_PE[D] = w.dw.PE;
                w.dw.item_base = static_cast<int>(all.size());
                w.dw.patch_base = patch_total;
                std::vector<int> tf = w.src.tile_first;
                for (size_t T = 0; T + 1 < tf.size(); ++T)
                    if (tf[T + 1] - tf[T] > 1) multi.push_back(make_int2(s, static_cast<int>(T)));
                max_pv = std::max(max_pv, PV);
                for (auto& v : tf) v += w.dw.item_base;
                w.tile_first.upload(tf.data(), tf.size(), stream);
                w.dw.tile_first = w.tile_first.p;
                std::vector<long long> tpo(tf.size() - 1, -1);
                for (size_t T = 0; T + 1 < tf.size(); ++T)
                    if (tf[T + 1] > tf[T])
                        tpo[T] = patch_total + static_cast<long long>(tf[T] - w.dw.item_base) * PV;
                w.tile_patch.upload(tpo.data(), tpo.size(), stream);
                w.dw.tile_patch = w.tile_patch.p;
                const bool has_colb = w.src.colb.size() == w.src.items.size() * kColBounds;
                for (size_t q = 0; q < w.src.items.size(); ++q) {
                    Item it = w.src.items[q];
                    it.ps = s;
                    it.patch = patch_total;
                    patch_total += PV;
                    all.push_back(it);
                    for (int b = 0; b < kColBounds; ++b)
                        colb.push_back(has_colb ? w.src.colb[q * kColBounds + b] : 0);
                }
            }
            class_end[D] = static_cast<int>(all.size());
            // Largest items first: CTAs are dispatched in item order, so the
            // last wave of a launch holds the smallest items (edge tiles)
            // instead of whatever the tile order ends with. Patch offsets
            // travel with the items; the column bounds are permuted alike.
            if (lpt_items()) {
                const size_t b = static_cast<size_t>(class_begin[D]), e = all.size();
                std::vector<size_t> ord(e - b);
                for (size_t q = 0; q < ord.size(); ++q) ord[q] = b + q;
                const bool by_window = lpt_items() == 2;  // A/B: windows kept in order
                std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) {
                    if (by_window && all[x].ps != all[y].ps) return all[x].ps < all[y].ps;
                    return all[x].end - all[x].begin > all[y].end - all[y].begin;
                });
                std::vector<Item> sorted_items(ord.size());
                std::vector<int> sorted_colb(ord.size() * kColBounds);
                for (size_t q = 0; q < ord.size(); ++q) {
                    sorted_items[q] = all[ord[q]];
                    std::copy_n(colb.begin() + static_cast<long long>(ord[q]) * kColBounds, kColBounds,
                                sorted_colb.begin() + static_cast<long long>(q) * kColBounds);
                }
                std::copy(sorted_items.begin(), sorted_items.end(), all.begin() + static_cast<long long>(b));
                std::copy(sorted_colb.begin(), sorted_colb.end(), colb.begin() + static_cast<long long>(b) * kColBounds);
            }
            if (f32_want(D)) {
                const char* fe = std::getenv("KSVM_NFFT_F32");
                f32_dense[D] = (fe && std::strcmp(fe, "all") == 0) || !sparse_cells(D);
                for (int s = 0; s < P; ++s) {  // keep the factors the chosen kernels read
                    Window& w = *wins[static_cast<size_t>(owned[static_cast<size_t>(s)])];
                    if (w.d != D) continue;
                    if (f32_dense[D]) w.src.F.reset();
                    else w.src.F32.reset();
                }
            }
            spread_columns[D] = D == 3 && !f32_class(D) && use_columns(D, "KSVM_NFFT_SPREAD3");
            gather_columns[D] = D == 3 && !f32_class(D) && use_columns(D, "KSVM_NFFT_GATHER3");
            gclass_begin[D] = static_cast<int>(gall.size());
            for (int s = 0; s < P; ++s) {
                Window& w = *wins[static_cast<size_t>(owned[static_cast<size_t>(s)])];
                if (w.d != D) continue;
                for (const Item& it0 : w.src.gitems) {
                    Item it = it0;
                    it.ps = s;
                    gall.push_back(it);
                }
            }
            gclass_end[D] = static_cast<int>(gall.size());
            // Gather items: largest first within each window, windows kept in
            // order. Each window scatters into its own length-n output, which
            // stays in L2 (evict-last) while that window is being gathered;
            // mixing the windows' items made config 5's gather 10 % slower.
            if (lpt_items())
                std::stable_sort(gall.begin() + gclass_begin[D], gall.end(), [](const Item& x, const Item& y) {
                    return x.ps != y.ps ? x.ps < y.ps : x.end - x.begin > y.end - y.begin;
                });
            n_multi_cls[D] = static_cast<int>(multi.size()) - multi_begin[D];
        }
        std::vector<DWin> dws(static_cast<size_t>(P));
        std::vector<double> eta(static_cast<size_t>(P));
        std::vector<int> slots;  // window slots grouped by d (per-class launches)
        for (int D = 1; D <= 3; ++D) {
            slot_begin[D] = static_cast<int>(slots.size());
            for (int s = 0; s < P; ++s)
                if (wins[static_cast<size_t>(owned[static_cast<size_t>(s)])]->d == D) slots.push_back(s);
            nslots_cls[D] = static_cast<int>(slots.size()) - slot_begin[D];
        }
        // Fused grid side: every owned window of the class has a non-wrapping
        // grid whose on-chip working set fits. KSVM_NFFT_GRID = conv3
        // (default: 1-/2-d classes fused; 3-d: staged node reduction on every
        // SM, then the three convolution stages in one cluster launch),
        // fused12 (3-d fully staged), fused (3-d reduction inside the cluster
        // too: measured slower, the patch reads on 14 SMs are L2-latency
        // bound), staged (no fusion).
        {
            const char* ge = std::getenv("KSVM_NFFT_GRID");
            const std::string gm = ge ? ge : "conv3";
            for (int D = 1; D <= 3; ++D) {
                const bool conv3 = gm == "conv3" && D == 3;
                bool allow = gm == "fused" || ((gm == "fused12" || gm == "conv3") && D < 3) || conv3;
                if (sharded()) allow = conv3;  // the node reduction must stay a separate phase
                bool ok = allow && nslots_cls[D] > 0;
                int lg = 0, nc = 0;
                for (int s = 0; s < P && ok; ++s) {
                    const Window& w = *wins[static_cast<size_t>(owned[static_cast<size_t>(s)])];
                    if (w.d != D) continue;
                    const Geometry& g = w.geom;
                    if (g.wrap) ok = false;
                    lg = std::max(lg, g.Lg);
                    const int pe = g.PE;
                    nc = std::max(nc, (pe + g.TC - 1) / g.TC);
                }
                const int ncT = nc <= (D == 3 ? 3 : 2) ? (D == 3 ? 3 : 2) : 5;
                if (ok && nc > 5) ok = false;
                if (ok && fused_smem_bytes(D, lg) > 227 * 1024) ok = false;
                if (ok && D == 3 && !fused3_supported(lg, ncT)) ok = false;
                if (ok && conv3 && ncT != 3) ok = false;
                // one cluster per window: past one wave of SMs (config 4's 18
                // windows x 14 CTAs) the staged convolutions use the GPU better
                if (ok && D == 3 && static_cast<long long>(nslots_cls[D]) * fused3_cluster_size(lg) > 148) ok = false;
                grid_fused[D] = ok;
                grid_conv_only[D] = ok && conv3;
                grid_nc[D] = ncT;
                grid_lg[D] = lg;
            }
        }
        if (sharded()) {
            // the owned windows' spread grids G in one contiguous pool, so the
            // ranks sum them with ONE all-reduce (ksvm_nfft_op_grid_pool)
            size_t total = 0;
            for (int s = 0; s < P; ++s) {
                const Window& w = *wins[static_cast<size_t>(owned[static_cast<size_t>(s)])];
                long long nodes = 1;
                for (int t = 0; t < w.d; ++t) nodes *= w.dw.Lg;
                total += static_cast<size_t>(nodes);
            }
            gpool.alloc(std::max<size_t>(total, 1));
            size_t off = 0;
            for (int s = 0; s < P; ++s) {
                Window& w = *wins[static_cast<size_t>(owned[static_cast<size_t>(s)])];
                long long nodes = 1;
                for (int t = 0; t < w.d; ++t) nodes *= w.dw.Lg;
                w.G.reset();
                w.dw.G = gpool.p + off;
                off += static_cast<size_t>(nodes);
            }
            gpool_len = static_cast<int64_t>(total);
        }
        parts.alloc(static_cast<size_t>(std::max(P, 1)) * n);
        if (sharded())  // gathers write the owned points only; the rest stays 0 for the combine
            CK(cudaMemsetAsync(parts.p, 0, sizeof(double) * parts.n, stream));
        // exact-duplicate windows: member chunks of <= kSegChunk within one
        // distinct point, global distinct-point numbering in slot order
        std::vector<int> segm, segcb(1, 0);
        std::vector<int2> chunks;
        long long utotal = 0;
        for (int s = 0; s < P; ++s) utotal += wins[static_cast<size_t>(owned[static_cast<size_t>(s)])]->nu;
        if (utotal > 0) {
            vs_all.alloc(static_cast<size_t>(utotal));
            uout_all.alloc(static_cast<size_t>(utotal));
        }
        std::vector<const double*> srcs(static_cast<size_t>(P));
        std::vector<const int*> invs(static_cast<size_t>(P), nullptr);
        std::vector<const uint8_t*> inv8s(static_cast<size_t>(P), nullptr), codes;
        std::vector<int> nu8s(static_cast<size_t>(std::max(P, 1)), 0);
        std::vector<long long> small_off;
        std::vector<int> small_nu;
        long long uoff = 0;
        for (int s = 0; s < P; ++s) {
            Window& w = *wins[static_cast<size_t>(owned[static_cast<size_t>(s)])];
            dws[static_cast<size_t>(s)] = w.dw;
            eta[static_cast<size_t>(s)] = w.eta;
            DPSet& p = ps[static_cast<size_t>(s)];
            p.F = w.src.F.p;
            p.F32 = w.src.F32.p;
            p.CP = w.src.CP.p;
            p.win = s;
            if (w.nu > 0 && w.nu <= kSmallBins) {
                codes.push_back(w.inv8.p);
                small_off.push_back(uoff);
                small_nu.push_back(static_cast<int>(w.nu));
                p.n = w.nu;
                p.vsrc = vs_all.p + uoff;
                p.out = uout_all.p + uoff;
                srcs[static_cast<size_t>(s)] = p.out;
                inv8s[static_cast<size_t>(s)] = w.inv8.p;
                nu8s[static_cast<size_t>(s)] = static_cast<int>(w.nu);
                uoff += w.nu;
            } else if (w.nu > 0) {
                // the CSR segments are numbered in vs_all order: pad the
                // register-bin windows' entries with empty segments
                while (static_cast<long long>(segcb.size()) - 1 < uoff) segcb.push_back(static_cast<int>(chunks.size()));
                const int base = static_cast<int>(segm.size());
                segm.insert(segm.end(), w.members.begin(), w.members.end());
                for (int64_t u = 0; u < w.nu; ++u) {
                    for (int b = w.offs[static_cast<size_t>(u)]; b < w.offs[static_cast<size_t>(u) + 1]; b += kSegChunk)
                        chunks.push_back(make_int2(base + b, base + std::min(b + kSegChunk, w.offs[static_cast<size_t>(u) + 1])));
                    segcb.push_back(static_cast<int>(chunks.size()));
                }
                p.n = w.nu;
                p.vsrc = vs_all.p + uoff;
                p.out = uout_all.p + uoff;
                srcs[static_cast<size_t>(s)] = p.out;
                invs[static_cast<size_t>(s)] = w.inv.p;
                uoff += w.nu;
            } else {
                p.n = n;
                p.vsrc = nullptr;
                p.out = parts.p + static_cast<size_t>(s) * n;
                srcs[static_cast<size_t>(s)] = p.out;
            }
        }
        n_seg_chunks = static_cast<int>(chunks.size());
        n_segs = static_cast<int>(segcb.size()) - 1;
        if (n_seg_chunks > 0) {
            seg_members.upload(segm.data(), segm.size(), stream);
            seg_chunks.upload(chunks.data(), chunks.size(), stream);
            seg_cb.upload(segcb.data(), segcb.size(), stream);
            seg_partial.alloc(static_cast<size_t>(n_seg_chunks));
        }
        d_src.upload(srcs.data(), srcs.size(), stream);
        d_inv.upload(invs.data(), invs.size(), stream);
        d_inv8.upload(inv8s.data(), inv8s.size(), stream);
        d_nu8.upload(nu8s.data(), nu8s.size(), stream);
        n_small = static_cast<int>(codes.size());
        if (n_small > 0) {
            d_codes.upload(codes.data(), codes.size(), stream);
            d_small_off.upload(small_off.data(), small_off.size(), stream);
            d_small_nu.upload(small_nu.data(), small_nu.size(), stream);
            bin_partial.alloc(static_cast<size_t>(kBinBlocks) * n_small * kSmallBins);
        }
        d_wins.upload(dws.data(), dws.size(), stream);
        d_ps.upload(ps.data(), ps.size(), stream);
        h_dws = dws;
        h_ps = ps;
        h_srcs = srcs;
        d_items.upload(all.data(), all.size(), stream);
        d_colb.upload(colb.data(), colb.size(), stream);
        d_gitems.upload(gall.data(), gall.size(), stream);
        if (!slots.empty()) d_slots.upload(slots.data(), slots.size(), stream);
        n_multi = static_cast<int>(multi.size());

        if (n_multi) d_multi.upload(multi.data(), multi.size(), stream);
        d_eta.upload(eta.data(), eta.size(), stream);
        patches.alloc(static_cast<size_t>(std::max<long long>(patch_total, 1)));
        vbuf.alloc(n);
        ybuf.alloc(n);
        CK(cudaStreamSynchronize(stream));
    }

    // Per-launch device timing: an event before each launch and one at the end.
    void tick(const char* name) {
        if (!stage_timing || nticks >= kMaxTicks) return;
        if (stage_timing == 2 && tick_stream != S()) return;  // side branches run untimed
        tick_name[nticks] = name;
        // external event node when captured into a graph, so the event stays timeable
        CK(cudaEventRecordWithFlags(ev_stage[nticks], stream, capturing ? cudaEventRecordExternal : 0));
        ++nticks;
    }

    // One dimension class (all owned windows with d_l = D): spread -> patch
    // reduce -> separable convolution -> (gather). Classes are independent
    // until `combine`, so they run on separate streams (graph branches).
    // Phases of one class: spread (spread, tile pre-reduction, node reduction
    // unless fused into the grid kernel), grid (convolution stages), gather.
    enum : int { kPhSpread = 1, kPhGrid = 2, kPhGather = 4, kPhAll = 7 };
    void run_class(int D, const double* v, cudaStream_t st, bool gather) {
        run_class_phases(D, v, st, kPhSpread | kPhGrid | (gather ? kPhGather : 0));
    }
    void run_class_phases(int D, const double* v, cudaStream_t st, int ph) {
        // the fp32-mode kernels carry a "_f32" suffix (bench.py reads it)
        static const char* kSpread[4] = {"", "spread_d1", "spread_d2", "spread_d3"};
        static const char* kGather[4] = {"", "gather_d1", "gather_d2", "gather_d3"};
        static const char* kSpread32 = "spread_d3_f32";
        static const char* kGather32 = "gather_d3_f32";
        static const char* kConv[3] = {"conv_0", "conv_1", "conv_2"};
        const int cnt = class_end[D] - class_begin[D];
        if (cnt == 0) return;
        tick_stream = st;
        if (ph & kPhSpread) {
        NvtxRange nr(f32_class(D) ? kSpread32 : kSpread[D]);
        tick(f32_class(D) ? kSpread32 : kSpread[D]);
        if (f32_class(D))
            launch_spread3_f32(d_items.p + class_begin[D], cnt, PS(), WINS(), v, PATCHES(), st);
        else
            launch_spread(D, 2 * cfg.window_cutoff, class_PE[D], d_items.p + class_begin[D], cnt, PS(),
                          WINS(), v, PATCHES(),
                          spread_columns[D] ? d_colb.p + static_cast<size_t>(class_begin[D]) * kColBounds : nullptr,
                          st);
        ++launch_counter();
        if (n_multi_cls[D]) {
            tick("tile_reduce");
            launch_tile_reduce(WINS(), d_multi.p + multi_begin[D], n_multi_cls[D], max_pv, PATCHES(), st);
            ++launch_counter();
        }
        if (grid_conv_only[D]) {  // staged node reduction, then one cluster launch for the conv stages
            tick("reduce");
            launch_reduce(WINS(), d_slots.p + slot_begin[D], nslots_cls[D], max_nodes, D, 2 * cfg.window_cutoff,
                          PATCHES(), false, max_tiles[D], st);
            ++launch_counter();
        } else if (!grid_fused[D]) {
            tick("reduce");
            for (int wrap = 0; wrap < 2; ++wrap) {
                if (!(wrap ? has_wrap : has_nowrap)[D]) continue;
                launch_reduce(WINS(), d_slots.p + slot_begin[D], nslots_cls[D], max_nodes, D,
                              2 * cfg.window_cutoff, PATCHES(), wrap != 0, max_tiles[D], st);
                ++launch_counter();
            }
        }
        }  // spread phase
        if (ph & kPhGrid) {
        static const char* kGridR[4] = {"", "grid_d1", "grid_d2", "grid_d3"};
        NvtxRange nr(kGridR[D]);
        if (grid_conv_only[D]) {
            tick("conv_d3");
            launch_grid_fused(WINS(), d_slots.p + slot_begin[D], nslots_cls[D], D, grid_nc[D], grid_lg[D],
                              PATCHES(), st, true);
            ++launch_counter();
        } else if (grid_fused[D]) {
            static const char* kGrid[4] = {"", "grid_d1", "grid_d2", "grid_d3"};
            tick(kGrid[D]);
            launch_grid_fused(WINS(), d_slots.p + slot_begin[D], nslots_cls[D], D, grid_nc[D], grid_lg[D],
                              PATCHES(), st, false);
            ++launch_counter();
        } else {
            for (int stg = 0; stg < D; ++stg) {
                tick(kConv[stg]);
                launch_conv(WINS(), d_slots.p + slot_begin[D], nslots_cls[D], max_lg, max_fibres, stg, st);
                ++launch_counter();
            }
        }
        }  // grid phase
        if (ph & kPhGather) {
            NvtxRange nr(f32_class(D) ? kGather32 : kGather[D]);
            const int gcnt = gclass_end[D] - gclass_begin[D];
            tick(f32_class(D) ? kGather32 : kGather[D]);
            if (f32_class(D)) {
                launch_gather3_f32(d_gitems.p + gclass_begin[D], gcnt, PS(), WINS(), st);
            } else if (gather_columns[D]) {
                launch_gather3c(d_items.p + class_begin[D], cnt, PS(), WINS(),
                                d_colb.p + static_cast<size_t>(class_begin[D]) * kColBounds, st);
            } else {
                launch_gather(D, 2 * cfg.window_cutoff, class_PE[D], d_gitems.p + gclass_begin[D], gcnt, PS(),
                              WINS(), st);
            }
            ++launch_counter();
        }
        CK(cudaGetLastError());
    }

    // All classes; concurrent branches unless per-launch timing is on.
    void run_classes(const double* v, bool gather) {
        if (n_small > 0 || n_seg_chunks > 0) tick("dedup_sums");  // per-distinct-point sums of v
        if (n_small > 0) {
            launch_bin_sums(v, d_codes.p, n_small, n, BINP(), kBinBlocks, d_small_off.p, d_small_nu.p,
                            VSALL(), S());
            launch_counter() += 2;
        }
        if (n_seg_chunks > 0) {
            launch_seg_sums(v, seg_members.p, seg_chunks.p, SEGP(), n_seg_chunks, seg_cb.p, VSALL(),
                            n_segs, S());
            launch_counter() += 2;
        }
        int ncls = 0;
        for (int D = 1; D <= 3; ++D) ncls += class_end[D] > class_begin[D] ? 1 : 0;
        if (stage_timing == 1 || ncls < 2) {
            for (int D = 3; D >= 1; --D) run_class(D, v, S(), gather);
            return;
        }
        CK(cudaEventRecord(EVF(), S()));
        bool first = true;
        for (int D = 3; D >= 1; --D) {
            if (class_end[D] == class_begin[D]) continue;
            cudaStream_t st = S();
            if (!first) {
                st = SIDE(D);
                CK(cudaStreamWaitEvent(st, EVF(), 0));
            }
            run_class(D, v, st, gather);
            if (!first) {
                CK(cudaEventRecord(EVJ(D), st));
                CK(cudaStreamWaitEvent(S(), EVJ(D), 0));
            }
            first = false;
        }
    }

    // grid stage only (cross applies gather over their own targets afterwards)
    void run_grid(const double* v) { run_classes(v, false); }

    // Point-sharded two-phase apply (no duplicate merge on sharded operators):
    // spread + node reduction into the windows' grids G, then -- after the
    // caller has summed G over the ranks -- convolution, gather and combine.
    void run_spread_phase(const double* v) {
        nticks = 0;
        for (int D = 3; D >= 1; --D) run_class_phases(D, v, S(), kPhSpread);
        CK(cudaGetLastError());
    }
    void run_finish_phase(double* y) {
        for (int D = 3; D >= 1; --D) run_class_phases(D, nullptr, S(), kPhGrid | kPhGather);
        launch_combine(y, SRC(), d_inv.p, d_inv8.p, d_nu8.p, d_eta.p, P_owned(), 0, n, S());
        ++launch_counter();
        CK(cudaGetLastError());
    }

    // Window-sharded multi-GPU pipeline (ksvm_nfft_op_apply_windows /
    // _combine_range): every owned window's transform into its per-window
    // output, then the window-order sum over row ranges, so the caller can
    // all-reduce range k while range k+1 is being summed.
    void run_windows(const double* v) {
        nticks = 0;
        if (P_owned() > 0) run_classes(v, true);
        CK(cudaGetLastError());
    }
    void run_combine(double* y, int64_t lo, int64_t hi) {
        if (P_owned() == 0) {
            launch_fill(y + lo, 0.0, hi - lo, S());
        } else {
            NvtxRange nr("combine");
            launch_combine(y, SRC(), d_inv.p, d_inv8.p, d_nu8.p, d_eta.p, P_owned(), lo, hi, S());
        }
        ++launch_counter();
        CK(cudaGetLastError());
    }

    void run_apply(const double* v, double* y) {
        const int P = P_owned();
        if (P == 0) {
            launch_fill(y, 0.0, n, S());
            ++launch_counter();
            return;
        }
        nticks = 0;
        run_classes(v, true);
        tick_stream = S();
        NvtxRange nr("combine");
        tick("combine");
        launch_combine(y, SRC(), d_inv.p, d_inv8.p, d_nu8.p, d_eta.p, P, 0, n, S());
        ++launch_counter();
        CK(cudaGetLastError());
        tick("end");
        last_nticks = nticks;
    }

    int collect_stage_times() {
        if (!stage_timing || last_nticks < 2) return 0;
        CK(cudaEventSynchronize(ev_stage[last_nticks - 1]));
        for (int k = 0; k + 1 < last_nticks; ++k) {
            CK(cudaEventElapsedTime(&last_ms[k], ev_stage[k], ev_stage[k + 1]));
            last_name[k] = tick_name[k];
        }
        return last_nticks - 1;
    }

    // ---- CUDA graph of the whole apply, cached per (v, y, timing) ----------
    struct GraphEntry {
        const double* v;
        double* y;
        int timed;
        cudaGraphExec_t exec;
        int nticks;
        int64_t launches;
        const char* names[kMaxTicks];
    };
    std::vector<GraphEntry> graphs;  // most recent last; at most kMaxGraphs
    static constexpr size_t kMaxGraphs = 8;
    bool use_graphs = std::getenv("KSVM_NFFT_NO_GRAPH") == nullptr;

    bool capturing = false;

    // ---- apply lanes: extra scratch sets so independent applies (the
    // columns of a batch) run concurrently. A lane owns everything an
    // in-flight apply writes -- streams, grids G/H/T, patches, per-window
    // outputs, staging, the duplicate-merge sums and the device tables that
    // point at them -- and shares the immutable plan. Lane 0 is the
    // engine's own members (cur == nullptr).
    struct Lane {
        cudaStream_t stream = nullptr, side[4] = {nullptr, nullptr, nullptr, nullptr};
        cudaEvent_t ev_fork = nullptr, ev_join[4] = {nullptr, nullptr, nullptr, nullptr}, ev_done = nullptr;
        DevBuf<double> grids, patches, parts, vbuf, ybuf, seg_partial, vs_all, uout_all, bin_partial;
        DevBuf<DWin> d_wins;
        DevBuf<DPSet> d_ps;
        DevBuf<const double*> d_src;
        std::vector<GraphEntry> graphs;
        ~Lane() {
            for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
            if (stream) cudaStreamSynchronize(stream);
            for (int D = 1; D <= 2; ++D) {
                if (side[D]) cudaStreamDestroy(side[D]);
                if (ev_join[D]) cudaEventDestroy(ev_join[D]);
            }
            if (ev_fork) cudaEventDestroy(ev_fork);
            if (ev_done) cudaEventDestroy(ev_done);
            if (stream) cudaStreamDestroy(stream);
        }
    };
    std::vector<std::unique_ptr<Lane>> lanes;  // lanes 1..
    Lane* cur = nullptr;
    std::vector<DWin> h_dws;        // host copies of the lane-0 tables (finalize)
    std::vector<DPSet> h_ps;
    std::vector<const double*> h_srcs;

    cudaStream_t S() const { return cur ? cur->stream : stream; }
    cudaStream_t SIDE(int D) const { return cur ? cur->side[D] : side[D]; }
    cudaEvent_t EVF() const { return cur ? cur->ev_fork : ev_fork; }
    cudaEvent_t EVJ(int D) const { return cur ? cur->ev_join[D] : ev_join[D]; }
    double* PATCHES() const { return cur ? cur->patches.p : patches.p; }
    DWin* WINS() const { return cur ? cur->d_wins.p : d_wins.p; }
    DPSet* PS() const { return cur ? cur->d_ps.p : d_ps.p; }
    const double* const* SRC() const { return cur ? cur->d_src.p : d_src.p; }
    double* BINP() const { return cur ? cur->bin_partial.p : bin_partial.p; }
    double* SEGP() const { return cur ? cur->seg_partial.p : seg_partial.p; }
    double* VSALL() const { return cur ? cur->vs_all.p : vs_all.p; }
    std::vector<GraphEntry>& GR() { return cur ? cur->graphs : graphs; }

    // map a lane-0 scratch pointer into the same offset of lane L's buffer
    static double* remap(const double* p, const DevBuf<double>& from, DevBuf<double>& to) {
        return const_cast<double*>(p) - from.p + to.p;
    }
    static bool inside(const double* p, const DevBuf<double>& b) { return p && b.p && p >= b.p && p < b.p + b.n; }

    void add_lane() {
        auto L = std::make_unique<Lane>();
        CK(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking));
        for (int D = 1; D <= 2; ++D) {
            CK(cudaStreamCreateWithFlags(&L->side[D], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&L->ev_join[D], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&L->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&L->ev_done, cudaEventDisableTiming));
        std::vector<DWin> dws = h_dws;
        size_t total = 0;
        for (const DWin& w : dws) {
            long long nodes = 1;
            for (int t = 0; t < w.d; ++t) nodes *= w.Lg;
            total += static_cast<size_t>(nodes) * (2 + (w.d == 1 ? 0 : (w.d == 2 ? 2 : 4)));
        }
        L->grids.alloc(total);
        size_t off = 0;
        for (DWin& w : dws) {
            long long nodes = 1;
            for (int t = 0; t < w.d; ++t) nodes *= w.Lg;
            w.G = L->grids.p + off;
            off += static_cast<size_t>(nodes);
            w.H = L->grids.p + off;
            off += static_cast<size_t>(nodes);
            for (int k = 0; k < 4; ++k) {
                if (k < (w.d == 1 ? 0 : (w.d == 2 ? 2 : 4))) {
                    w.T[k] = L->grids.p + off;
                    off += static_cast<size_t>(nodes);
                } else {
                    w.T[k] = nullptr;
                }
            }
        }
        L->patches.alloc(patches.n);
        L->parts.alloc(parts.n);
        if (sharded()) CK(cudaMemsetAsync(L->parts.p, 0, sizeof(double) * parts.n, stream));
        L->vbuf.alloc(vbuf.n);
        L->ybuf.alloc(ybuf.n);
        if (vs_all.p) L->vs_all.alloc(vs_all.n);
        if (uout_all.p) L->uout_all.alloc(uout_all.n);
        if (seg_partial.p) L->seg_partial.alloc(seg_partial.n);
        if (bin_partial.p) L->bin_partial.alloc(bin_partial.n);
        std::vector<DPSet> ps = h_ps;
        std::vector<const double*> srcs = h_srcs;
        auto map_out = [&](const double* q) -> double* {
            if (inside(q, parts)) return remap(q, parts, L->parts);
            if (inside(q, uout_all)) return remap(q, uout_all, L->uout_all);
            throw std::logic_error("add_lane: unmapped output pointer");
        };
        for (size_t i = 0; i < ps.size(); ++i) {
            ps[i].out = map_out(ps[i].out);
            if (ps[i].vsrc) ps[i].vsrc = remap(ps[i].vsrc, vs_all, L->vs_all);
            srcs[i] = map_out(srcs[i]);
        }
        L->d_wins.upload(dws.data(), dws.size(), stream);
        L->d_ps.upload(ps.data(), ps.size(), stream);
        L->d_src.upload(srcs.data(), srcs.size(), stream);
        CK(cudaStreamSynchronize(stream));
        lanes.push_back(std::move(L));
    }

    void drop_graphs() {
        for (auto& gph : graphs) cudaGraphExecDestroy(gph.exec);
        graphs.clear();
    }

    // One apply: replays a captured graph (one launch) or captures it first.
    void apply(const double* v, double* y) {
        NvtxRange nr("ksvm_nfft_apply");
        (void)cudaGetLastError();  // a stale error must not be blamed on this apply
        if (!use_graphs || P_owned() == 0) {
            run_apply(v, y);
            return;
        }
        for (size_t k = 0; k < GR().size(); ++k) {
            GraphEntry& gph = GR()[k];
            if (gph.v == v && gph.y == y && gph.timed == stage_timing) {
                CK(cudaGraphLaunch(gph.exec, S()));
                launch_counter() += gph.launches;
                last_nticks = gph.nticks;
                for (int i = 0; i < gph.nticks; ++i) tick_name[i] = gph.names[i];
                if (k + 1 != GR().size()) std::rotate(GR().begin() + k, GR().begin() + k + 1, GR().end());
                return;
            }
        }
        cudaGraph_t graph = nullptr;
        const int64_t before = launch_counter().load();
        CK(cudaStreamBeginCapture(S(), cudaStreamCaptureModeThreadLocal));
        capturing = true;
        try {
            run_apply(v, y);
            capturing = false;
        } catch (...) {
            capturing = false;
            cudaStreamEndCapture(S(), &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        CK(cudaStreamEndCapture(S(), &graph));
        GraphEntry gph{};
        gph.v = v;
        gph.y = y;
        gph.timed = stage_timing;
        gph.launches = launch_counter().load() - before;
        launch_counter() -= gph.launches;  // counted when launched
        gph.nticks = last_nticks;
        for (int i = 0; i < last_nticks; ++i) gph.names[i] = tick_name[i];
        const cudaError_t e = cudaGraphInstantiate(&gph.exec, graph, 0);
        cudaGraphDestroy(graph);
        CK(e);
        if (GR().size() >= kMaxGraphs) {
            cudaGraphExecDestroy(GR().front().exec);
            GR().erase(GR().begin());
        }
        GR().push_back(gph);
        CK(cudaGraphLaunch(gph.exec, S()));
        launch_counter() += gph.launches;
    }

    // Host/device dispatch shared by every apply-like entry point.
    template <typename F>
    void with_io(const double* v, double* y, int ptr_kind, void* ext_stream, int64_t vin,
                 int64_t yout, F&& body) {
        DeviceGuard dg(device);
        std::lock_guard<std::mutex> lk(mu);
        if (ptr_kind == KSVM_NFFT_HOST) {
            {
                NvtxRange nr("h2d");
                if (vin > 0) CK(cudaMemcpyAsync(vbuf.p, v, sizeof(double) * vin, cudaMemcpyHostToDevice, stream));
            }
            body(vbuf.p, ybuf.p);
            NvtxRange nr("d2h");
            if (yout > 0) CK(cudaMemcpyAsync(y, ybuf.p, sizeof(double) * yout, cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
        } else if (ptr_kind == KSVM_NFFT_DEVICE) {
            cudaStream_t es = static_cast<cudaStream_t>(ext_stream);
            CK(cudaEventRecord(ev_in, es));
            CK(cudaStreamWaitEvent(stream, ev_in, 0));
            body(v, y);
            CK(cudaEventRecord(ev_out, stream));
            CK(cudaStreamWaitEvent(es, ev_out, 0));
        } else {
            throw std::invalid_argument("ptr_kind must be KSVM_NFFT_HOST or KSVM_NFFT_DEVICE");
        }
    }
};

}  // namespace ksvm_nfft

using namespace ksvm_nfft;

struct ksvm_nfft_op {
    Engine e;
};

struct ksvm_nfft_plan {
    Engine e;  // one window, eta = 1
};

namespace {

void build_engine(Engine& E, const double* points, int64_t n, int64_t d, int64_t ld, int layout,
                  const int* feats, const int* sizes, int P, const double* weights,
                  const double* ells, const ksvm_nfft_config* cfg, double fit, const int* mask,
                  int device, int precision, bool data_range, const int64_t* own = nullptr,
                  int64_t n_own = 0) {
    if (!points || !feats || !sizes || !weights || !ells || !cfg)
        throw std::invalid_argument("null argument");
    validate_cfg(*cfg);
    if (precision != KSVM_NFFT_FP64 && precision != KSVM_NFFT_FP32)
        throw std::invalid_argument("precision must be KSVM_NFFT_FP64 or KSVM_NFFT_FP32");
    if (n < 1) throw std::invalid_argument("empty node set");
    if (n > 2147483647LL) throw std::invalid_argument("n must be < 2^31");
    if (!(fit > 0.0 && fit <= 1.0)) throw std::invalid_argument("fit_fraction must lie in (0, 1]");
    check_layout(n, d, ld, layout);
    // P:src/windowing.cpp:79-103 (check_windowing)
    if (P < 1) throw std::invalid_argument("windowing has no windows");
    std::vector<bool> seen(static_cast<size_t>(d), false);
    int off = 0;
    for (int l = 0; l < P; ++l) {
        if (sizes[l] < 1 || sizes[l] > 3) throw std::invalid_argument("window size must be 1..3");
        for (int t = 0; t < sizes[l]; ++t) {
            const int f = feats[off + t];
            if (f < 0 || f >= d) throw std::invalid_argument("window feature index out of range");
            if (seen[static_cast<size_t>(f)]) throw std::invalid_argument("feature appears in two windows");
            seen[static_cast<size_t>(f)] = true;
        }
        off += sizes[l];
    }
    for (int l = 0; l < P; ++l) {
        if (!(weights[l] > 0.0)) throw std::invalid_argument("window weights must be positive");
        if (!(ells[l] > 0.0)) throw std::invalid_argument("length scales must be positive");
    }
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw std::invalid_argument("no such CUDA device");
    DeviceGuard dg(device);
    E.init(device);
    E.cfg = *cfg;
    E.fit = fit;
    E.precision = precision;
    E.data_range = data_range;
    E.n = n;
    if (own) {  // point shard: owned rows, strictly ascending, in [0, n)
        if (n_own < 1) throw std::invalid_argument("a point shard needs at least one point");
        E.own_idx.assign(own, own + n_own);
        for (int64_t r = 0; r < n_own; ++r)
            if (own[r] < 0 || own[r] >= n || (r > 0 && own[r] <= own[r - 1]))
                throw std::invalid_argument("own_points must be strictly ascending indices in [0, n)");
    }
    E.dfull = d;
    off = 0;
    for (int l = 0; l < P; ++l) {
        auto w = std::make_unique<Window>();
        w->d = sizes[l];
        for (int t = 0; t < w->d; ++t) w->feat[t] = feats[off + t];
        off += sizes[l];
        w->eta = weights[l];
        w->ell = ells[l];
        w->owned = mask ? mask[l] != 0 : true;
        E.wins.push_back(std::move(w));
    }
    // raw window features for entries (row-major host copy + device SoA)
    for (auto& w : E.wins)
        for (int t = 0; t < w->d; ++t) E.raw_cols.push_back(w->feat[t]);
    const int nc = static_cast<int>(E.raw_cols.size());
    E.raw_rm.resize(static_cast<size_t>(n) * nc);
    std::vector<double> soa(static_cast<size_t>(n) * nc);
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < nc; ++c) {
            const double x = at(points, i, E.raw_cols[static_cast<size_t>(c)], ld, layout);
            E.raw_rm[static_cast<size_t>(i * nc + c)] = x;
            soa[static_cast<size_t>(c) * n + i] = x;
        }
    // the device SoA copy is uploaded from raw_rm on first use (kernel rows /
    // diagonal / preconditioner entries), so a matvec-only operator -- every
    // rank of a sharded matvec -- holds no device copy of the raw features
    std::vector<int> wdim;
    for (auto& w : E.wins) wdim.push_back(w->d);
    E.d_wdim.upload(wdim.data(), wdim.size(), E.stream);
    // one plan per owned window (P:src/fastsum.cpp:333-340)
    E.n_owned_windows = 0;
    for (auto& w : E.wins) E.n_owned_windows += w->owned ? 1 : 0;
    E.n_owned_windows = std::max<int64_t>(1, E.n_owned_windows);
    // host halves of the owned windows' plans on concurrent threads (a
    // window's feature columns are contiguous in soa), device halves in
    // window order
    std::vector<Engine::WinPrep> prep(static_cast<size_t>(P));
    {
        std::vector<int> col0(static_cast<size_t>(P), 0);
        for (int l = 1; l < P; ++l) col0[static_cast<size_t>(l)] = col0[static_cast<size_t>(l - 1)] + E.wins[static_cast<size_t>(l - 1)]->d;
        // A worker's exception (bad_alloc in the scaled copy, ...) is caught
        // into its window's slot and rethrown here after every started
        // thread joined: nothing may escape a std::thread (std::terminate).
        std::atomic<int> next{0};
        std::vector<std::exception_ptr> err(static_cast<size_t>(P));
        auto work = [&] {
            for (int l; (l = next.fetch_add(1)) < P;) {
                Window& w = *E.wins[static_cast<size_t>(l)];
                if (!w.owned) continue;
                try {
                    E.prep_window(w, soa.data() + static_cast<size_t>(col0[static_cast<size_t>(l)]) * n,
                                  prep[static_cast<size_t>(l)]);
                } catch (...) {
                    err[static_cast<size_t>(l)] = std::current_exception();
                }
            }
        };
        const int nthr = std::max(1, std::min<int>(P, static_cast<int>(std::thread::hardware_concurrency())));
        std::vector<std::thread> pool;
        try {
            for (int t = 1; t < nthr; ++t) pool.emplace_back(work);
        } catch (...) {  // could not start a thread: the ones started (and this one) finish the work
        }
        work();
        for (auto& th : pool) th.join();
        for (auto& e : err)
            if (e) std::rethrow_exception(e);
    }
    for (int l = 0; l < P; ++l) {
        Window& w = *E.wins[static_cast<size_t>(l)];
        if (w.owned) {
            E.plan_window(w, prep[static_cast<size_t>(l)]);
            std::vector<double>().swap(prep[static_cast<size_t>(l)].sc);
            E.owned.push_back(l);
        }
    }
    E.finalize();
}

}  // namespace

extern "C" {

const char* ksvm_nfft_last_error(void) { return last_error_ref().c_str(); }
const char* ksvm_nfft_version(void) { return "ksvm_nfft 0.1 sm_100a fp64"; }
int64_t ksvm_nfft_launch_count(void) { return launch_counter().load(); }

void ksvm_nfft_config_default(ksvm_nfft_config* cfg) {
    if (!cfg) return;
    cfg->bandwidth = 32;
    cfg->window_cutoff = 4;
    cfg->oversampling = 2;
    cfg->torus_radius = 0.25;
}

int ksvm_nfft_config_validate(const ksvm_nfft_config* cfg) {
    return guarded([&] {
        if (!cfg) throw std::invalid_argument("null config");
        validate_cfg(*cfg);
    });
}

int ksvm_nfft_op_create(const double* points, int64_t n, int64_t d, int64_t ld, int layout,
                        const int* window_features, const int* window_sizes, int num_windows,
                        const double* weights, const double* length_scales,
                        const ksvm_nfft_config* cfg, double fit_fraction, const int* window_mask,
                        int device, int precision, ksvm_nfft_op** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("null out");
        auto op = std::make_unique<ksvm_nfft_op>();
        build_engine(op->e, points, n, d, ld, layout, window_features, window_sizes, num_windows,
                     weights, length_scales, cfg, fit_fraction, window_mask, device, precision,
                     /*data_range=*/true);
        *out = op.release();
    });
}

int64_t ksvm_nfft_op_size(const ksvm_nfft_op* op) { return op ? op->e.n : 0; }
int ksvm_nfft_op_num_windows(const ksvm_nfft_op* op) {
    return op ? static_cast<int>(op->e.wins.size()) : 0;
}

int64_t ksvm_nfft_op_window_points(const ksvm_nfft_op* op, int window) {
    if (!op || window < 0 || window >= static_cast<int>(op->e.wins.size())) return 0;
    const Window& w = *op->e.wins[static_cast<size_t>(window)];
    if (!w.owned) return 0;
    return w.nu > 0 ? w.nu : op->e.n;
}

int ksvm_nfft_op_apply(const ksvm_nfft_op* op, const double* v, double* y, int ptr_kind,
                       void* stream) {
    return guarded([&] {
        if (!op || !v || !y) throw std::invalid_argument("null argument");
        Engine& E = const_cast<Engine&>(op->e);
        E.with_io(v, y, ptr_kind, stream, E.n, E.n, [&](const double* dv, double* dy) { E.apply(dv, dy); });
    });
}

int ksvm_nfft_op_create_sharded(const double* points, int64_t n, int64_t d, int64_t ld, int layout,
                                const int* window_features, const int* window_sizes, int num_windows,
                                const double* weights, const double* length_scales, const ksvm_nfft_config* cfg,
                                double fit_fraction, const int64_t* own_points, int64_t n_own, int device,
                                int precision, ksvm_nfft_op** out) {
    return guarded([&] {
        if (!out || !own_points) throw std::invalid_argument("null argument");
        auto op = std::make_unique<ksvm_nfft_op>();
        build_engine(op->e, points, n, d, ld, layout, window_features, window_sizes, num_windows, weights,
                     length_scales, cfg, fit_fraction, nullptr, device, precision, true, own_points, n_own);
        *out = op.release();
    });
}

int ksvm_nfft_op_apply_spread(ksvm_nfft_op* op, const double* v, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!op || !v) throw std::invalid_argument("null argument");
        Engine& E = op->e;
        if (!E.sharded()) throw std::invalid_argument("apply_spread needs a point-sharded operator");
        E.with_io(v, nullptr, ptr_kind, stream, E.n, 0, [&](const double* dv, double*) { E.run_spread_phase(dv); });
    });
}

int ksvm_nfft_op_grids(const ksvm_nfft_op* op, double** grids, int64_t* lengths, int max_grids) {
    int count = 0;
    const int rc = guarded([&] {
        if (!op) throw std::invalid_argument("null argument");
        const Engine& E = op->e;
        if (!E.sharded()) throw std::invalid_argument("grids are exposed by point-sharded operators only");
        for (const auto& w : E.wins) {
            if (!w->owned) continue;
            if (count < max_grids && grids && lengths) {
                long long nodes = 1;
                for (int t = 0; t < w->d; ++t) nodes *= w->dw.Lg;
                grids[count] = w->dw.G;
                lengths[count] = nodes;
            }
            ++count;
        }
    });
    return rc == KSVM_NFFT_OK ? count : -rc;
}

int ksvm_nfft_op_apply_finish(ksvm_nfft_op* op, double* y, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!op || !y) throw std::invalid_argument("null argument");
        Engine& E = op->e;
        if (!E.sharded()) throw std::invalid_argument("apply_finish needs a point-sharded operator");
        E.with_io(nullptr, y, ptr_kind, stream, 0, E.n, [&](const double*, double* dy) { E.run_finish_phase(dy); });
    });
}

int ksvm_nfft_op_grid_pool(const ksvm_nfft_op* op, double** pool, int64_t* length) {
    return guarded([&] {
        if (!op || !pool || !length) throw std::invalid_argument("null argument");
        const Engine& E = op->e;
        if (!E.sharded()) throw std::invalid_argument("the grid pool belongs to point-sharded operators");
        *pool = E.gpool.p;
        *length = E.gpool_len;
    });
}

int ksvm_nfft_op_apply_windows(ksvm_nfft_op* op, const double* v, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!op || !v) throw std::invalid_argument("null argument");
        if (ptr_kind != KSVM_NFFT_DEVICE) throw std::invalid_argument("apply_windows takes device pointers");
        Engine& E = op->e;
        if (E.sharded()) throw std::invalid_argument("apply_windows is for window-sharded operators");
        E.with_io(v, nullptr, ptr_kind, stream, E.n, 0, [&](const double* dv, double*) { E.run_windows(dv); });
    });
}

int ksvm_nfft_op_combine_range(ksvm_nfft_op* op, double* y, int64_t lo, int64_t hi, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!op || !y) throw std::invalid_argument("null argument");
        if (ptr_kind != KSVM_NFFT_DEVICE) throw std::invalid_argument("combine_range takes device pointers");
        Engine& E = op->e;
        if (E.sharded()) throw std::invalid_argument("combine_range is for window-sharded operators");
        if (lo < 0 || hi > E.n || lo > hi) throw std::invalid_argument("row range out of bounds");
        if (lo == hi) return;
        E.with_io(nullptr, y, ptr_kind, stream, 0, 0, [&](const double*, double* dy) { E.run_combine(dy, lo, hi); });
    });
}

int ksvm_nfft_op_apply_batch(const ksvm_nfft_op* op, const double* V, double* Y, int k, int64_t ld,
                             int ptr_kind, void* stream) {
    return guarded([&] {
        if (!op || !V || !Y) throw std::invalid_argument("null argument");
        Engine& E = const_cast<Engine&>(op->e);
        if (ld < E.n) throw std::invalid_argument("ld must be >= n");
        if (k < 0) throw std::invalid_argument("k must be >= 0");
        if (ptr_kind != KSVM_NFFT_HOST && ptr_kind != KSVM_NFFT_DEVICE)
            throw std::invalid_argument("ptr_kind must be KSVM_NFFT_HOST or KSVM_NFFT_DEVICE");
        if (k == 0) return;
        // One upload / download for all columns. Columns are spread over up
        // to kBatchLanes apply lanes (independent scratch, shared plan) that
        // run concurrently; each column replays its lane's cached graph, so
        // every result is bit-identical to a single apply.
        DeviceGuard dg(E.device);
        std::lock_guard<std::mutex> lk(E.mu);
        const int64_t n = E.n;
        const size_t col = sizeof(double) * static_cast<size_t>(n);
        cudaStream_t st = E.stream, es = static_cast<cudaStream_t>(stream);
        DevBuf<double> Vd, Yd;
        const double* vsrc = V;
        double* ydst = Y;
        int64_t vld = ld, yld = ld;
        if (ptr_kind == KSVM_NFFT_HOST) {
            Vd.alloc(static_cast<size_t>(n) * k);
            Yd.alloc(static_cast<size_t>(n) * k);
            CK(cudaMemcpy2DAsync(Vd.p, col, V, sizeof(double) * ld, col, k, cudaMemcpyHostToDevice, st));
            vsrc = Vd.p;
            ydst = Yd.p;
            vld = yld = n;
        } else {
            CK(cudaEventRecord(E.ev_in, es));
            CK(cudaStreamWaitEvent(st, E.ev_in, 0));
        }
        int B = (E.use_graphs && !E.stage_timing && E.P_owned() > 0) ? std::min(k, kBatchLanes) : 1;
        if (const char* e = std::getenv("KSVM_NFFT_LANES")) B = std::max(1, std::min(B, std::atoi(e)));
        while (static_cast<int>(E.lanes.size()) < B - 1) E.add_lane();
        CK(cudaEventRecord(E.ev_in, st));  // inputs staged
        for (int b = 1; b < B; ++b) CK(cudaStreamWaitEvent(E.lanes[static_cast<size_t>(b - 1)]->stream, E.ev_in, 0));
        struct LaneReset {  // the engine is back on lane 0 whatever happens
            Engine& e;
            ~LaneReset() { e.cur = nullptr; }
        } lane_reset{E};
        for (int c = 0; c < k; ++c) {
            const int b = c % B;
            E.cur = b == 0 ? nullptr : E.lanes[static_cast<size_t>(b - 1)].get();
            double* lv = b == 0 ? E.vbuf.p : E.cur->vbuf.p;
            double* ly = b == 0 ? E.ybuf.p : E.cur->ybuf.p;
            CK(cudaMemcpyAsync(lv, vsrc + c * vld, col, cudaMemcpyDeviceToDevice, E.S()));
            E.apply(lv, ly);
            CK(cudaMemcpyAsync(ydst + c * yld, ly, col, cudaMemcpyDeviceToDevice, E.S()));
        }
        E.cur = nullptr;
        for (int b = 1; b < B; ++b) {
            auto& L = *E.lanes[static_cast<size_t>(b - 1)];
            CK(cudaEventRecord(L.ev_done, L.stream));
            CK(cudaStreamWaitEvent(st, L.ev_done, 0));
        }
        if (ptr_kind == KSVM_NFFT_HOST) {
            CK(cudaMemcpy2DAsync(Y, sizeof(double) * ld, Yd.p, col, col, k, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else {
            CK(cudaEventRecord(E.ev_out, st));
            CK(cudaStreamWaitEvent(es, E.ev_out, 0));
        }
    });
}

double ksvm_nfft_op_entry(const ksvm_nfft_op* op, int64_t i, int64_t j) {
    // P:src/kernel.cpp:15-29 on the raw coordinates, every window
    const Engine& E = op->e;
    const size_t nc = E.raw_cols.size();
    double sum = 0.0;
    size_t c = 0;
    for (const auto& w : E.wins) {
        double d2 = 0.0;
        for (int t = 0; t < w->d; ++t, ++c) {
            const double diff = E.raw_rm[static_cast<size_t>(i) * nc + c] - E.raw_rm[static_cast<size_t>(j) * nc + c];
            d2 += diff * diff;
        }
        sum += w->eta * std::exp(-d2 / (w->ell * w->ell));
    }
    return sum;
}

extern "C++" {
namespace ksvm_nfft {
// lowrank.cu: entries of window `window` (-1: the weighted ANOVA kernel),
// the same arithmetic as ksvm_nfft_kernel_rows.
void op_entry_view(const ksvm_nfft_op* op, int window, EntryView& v) {
    if (!op) throw std::invalid_argument("null operator");
    Engine& E = const_cast<Engine&>(op->e);
    const int P = static_cast<int>(E.wins.size());
    if (window < -1 || window >= P) throw std::invalid_argument("window out of range");
    int c0 = 0;
    for (int l = 0; l < (window < 0 ? 0 : window); ++l) c0 += E.wins[static_cast<size_t>(l)]->d;
    v.device = E.device;
    v.stream = E.stream;
    v.mu = &E.mu;
    v.n = E.n;
    v.nw = window < 0 ? P : 1;
    E.ensure_raw_device();
    v.cols = E.d_rawcols.p + c0;
    v.wdim = E.d_wdim.p + (window < 0 ? 0 : window);
    v.wgt.clear();
    v.ell2.clear();
    for (int l = 0; l < P; ++l) {
        if (window >= 0 && l != window) continue;
        const Window& w = *E.wins[static_cast<size_t>(l)];
        v.wgt.push_back(window < 0 ? w.eta : -1.0);
        v.ell2.push_back(w.ell * w.ell);
    }
}
}  // namespace ksvm_nfft
}  // extern "C++"

int ksvm_nfft_kernel_rows(const ksvm_nfft_op* op, int window, const int64_t* rows, int r,
                          double* out, int ptr_kind, void* stream) {
    return guarded([&] {
        if (!op || !rows || !out) throw std::invalid_argument("null argument");
        Engine& E = const_cast<Engine&>(op->e);
        const int P = static_cast<int>(E.wins.size());
        if (window < -1 || window >= P) throw std::invalid_argument("window out of range");
        if (r < 0) throw std::invalid_argument("r must be >= 0");
        for (int q = 0; q < r; ++q)
            if (rows[q] < 0 || rows[q] >= E.n) throw std::invalid_argument("row index out of range");
        if (r == 0) return;
        int c0 = 0;
        for (int l = 0; l < (window < 0 ? 0 : window); ++l) c0 += E.wins[static_cast<size_t>(l)]->d;
        const int nw = window < 0 ? P : 1;
        std::vector<double> wgt, ell2;
        for (int l = 0; l < P; ++l) {
            if (window >= 0 && l != window) continue;
            const Window& w = *E.wins[static_cast<size_t>(l)];
            wgt.push_back(window < 0 ? w.eta : -1.0);  // -1: plain exp (WindowOperator)
            ell2.push_back(w.ell * w.ell);
        }
        E.ensure_raw_device();
        DeviceGuard dg(E.device);
        std::lock_guard<std::mutex> lk(E.mu);
        DevBuf<long long> drows;
        DevBuf<double> dw, de, dout;
        static_assert(sizeof(long long) == sizeof(int64_t), "int64");
        drows.upload(reinterpret_cast<const long long*>(rows), static_cast<size_t>(r), E.stream);
        dw.upload(wgt.data(), wgt.size(), E.stream);
        de.upload(ell2.data(), ell2.size(), E.stream);
        const size_t total = static_cast<size_t>(r) * E.n;
        cudaStream_t es = static_cast<cudaStream_t>(stream);
        double* dst = out;
        if (ptr_kind == KSVM_NFFT_HOST) {
            dout.alloc(total);
            dst = dout.p;
        } else if (ptr_kind == KSVM_NFFT_DEVICE) {
            CK(cudaEventRecord(E.ev_in, es));
            CK(cudaStreamWaitEvent(E.stream, E.ev_in, 0));
        } else {
            throw std::invalid_argument("bad ptr_kind");
        }
        launch_kernel_rows(dst, drows.p, r, E.d_rawcols.p + c0, E.d_wdim.p + (window < 0 ? 0 : window), dw.p, de.p,
                           nw, E.n, E.stream);
        ++launch_counter();
        CK(cudaGetLastError());
        if (ptr_kind == KSVM_NFFT_HOST) {
            CK(cudaMemcpyAsync(out, dst, sizeof(double) * total, cudaMemcpyDeviceToHost, E.stream));
        } else {
            CK(cudaEventRecord(E.ev_out, E.stream));
            CK(cudaStreamWaitEvent(es, E.ev_out, 0));
        }
        CK(cudaStreamSynchronize(E.stream));  // scratch buffers are freed on return
    });
}

int ksvm_nfft_kernel_diag(const ksvm_nfft_op* op, int window, double* out, int ptr_kind,
                          void* stream) {
    return guarded([&] {
        if (!op || !out) throw std::invalid_argument("null argument");
        Engine& E = const_cast<Engine&>(op->e);
        const int P = static_cast<int>(E.wins.size());
        if (window < -1 || window >= P) throw std::invalid_argument("window out of range");
        // exp(-0) = 1 per window: diag = 1 (window) or sum_l eta_l (ANOVA),
        // accumulated in window order like anova_eval.
        double val = 1.0;
        if (window < 0) {
            val = 0.0;
            for (const auto& w : E.wins) val += w->eta * 1.0;
        }
        if (ptr_kind == KSVM_NFFT_HOST) {
            for (int64_t i = 0; i < E.n; ++i) out[i] = val;
            return;
        }
        if (ptr_kind != KSVM_NFFT_DEVICE) throw std::invalid_argument("bad ptr_kind");
        DeviceGuard dg(E.device);
        launch_fill(out, val, E.n, static_cast<cudaStream_t>(stream));
        ++launch_counter();
        CK(cudaGetLastError());
    });
}

int ksvm_nfft_op_device(const ksvm_nfft_op* op) { return op ? op->e.device : -1; }

int ksvm_nfft_op_set_stage_timing(ksvm_nfft_op* op, int on) {
    if (!op) return KSVM_NFFT_ERR_CONFIG;
    std::lock_guard<std::mutex> lk(op->e.mu);
    op->e.stage_timing = on == 2 ? 2 : (on != 0 ? 1 : 0);
    return KSVM_NFFT_OK;
}

int ksvm_nfft_op_last_stage_ms(const ksvm_nfft_op* op, float* ms, int cap) {
    if (!op || !ms || !op->e.stage_timing) return 0;
    Engine& E = const_cast<Engine&>(op->e);
    int k = 0;
    try {
        DeviceGuard dg(E.device);
        std::lock_guard<std::mutex> lk(E.mu);
        k = E.collect_stage_times();
    } catch (const std::exception& e) {
        last_error_ref() = e.what();
        return 0;
    }
    k = std::min(cap, k);
    for (int i = 0; i < k; ++i) ms[i] = E.last_ms[i];
    return k;
}

const char* ksvm_nfft_op_stage_name(const ksvm_nfft_op* op, int i) {
    if (!op || i < 0 || i >= Engine::kMaxTicks || !op->e.last_name[i]) return "";
    return op->e.last_name[i];
}

void ksvm_nfft_op_free(ksvm_nfft_op* op) { delete op; }

// ---- single-window plan --------------------------------------------------

int ksvm_nfft_plan_create(const double* points, int64_t n, int d, int64_t ld, int layout,
                          double length_scale, const ksvm_nfft_config* cfg, double fit_fraction,
                          int device, ksvm_nfft_plan** out) {
    return guarded([&] {
        if (!out || !cfg) throw std::invalid_argument("null argument");
        validate_cfg(*cfg);  // P:src/fastsum.cpp:106 validates before the shape checks
        if (d < 1 || d > 3) throw std::invalid_argument("fast summation window dimension must be 1..3");
        if (n < 1) throw std::invalid_argument("empty node set");
        if (!(fit_fraction > 0.0 && fit_fraction <= 1.0))
            throw std::invalid_argument("fit_fraction must lie in (0, 1]");
        if (!(length_scale > 0.0)) throw std::invalid_argument("length scale must be positive");
        auto p = std::make_unique<ksvm_nfft_plan>();
        const int feats[3] = {0, 1, 2};
        const int sizes[1] = {d};
        const double one = 1.0;
        build_engine(p->e, points, n, d, ld, layout, feats, sizes, 1, &one, &length_scale, cfg,
                     fit_fraction, nullptr, device, KSVM_NFFT_FP64, /*data_range=*/false);
        *out = p.release();
    });
}

int ksvm_nfft_plan_apply(const ksvm_nfft_plan* plan, const double* v, double* out, int ptr_kind,
                         void* stream) {
    return guarded([&] {
        if (!plan || !v || !out) throw std::invalid_argument("null argument");
        Engine& E = const_cast<Engine&>(plan->e);
        E.with_io(v, out, ptr_kind, stream, E.n, E.n, [&](const double* dv, double* dy) { E.apply(dv, dy); });
    });
}

int ksvm_nfft_plan_apply_cross(const ksvm_nfft_plan* plan, const double* targets, int64_t t,
                               int64_t ld, int layout, const double* v, double* out, int ptr_kind,
                               void* stream) {
    return guarded([&] {
        if (!plan || !targets || !v || !out) throw std::invalid_argument("null argument");
        Engine& E = const_cast<Engine&>(plan->e);
        Window& w = *E.wins[0];
        if (t < 0) throw std::invalid_argument("t must be >= 0");
        if (t > 2147483647LL) throw std::invalid_argument("t must be < 2^31");
        check_layout(t, w.d, ld, layout);
        const int cols[3] = {0, 1, 2};
        std::vector<double> sc = scale_cm(w, targets, t, ld, layout, cols);
        // P:src/fastsum.cpp:316-320
        for (int64_t j = 0; j < t; ++j) {
            double s = 0.0;
            for (int c = 0; c < w.d; ++c) s += sc[static_cast<size_t>(c * t + j)] * sc[static_cast<size_t>(c * t + j)];
            if (std::sqrt(s) > E.cfg.torus_radius * (1.0 + 1e-12))
                throw DomainErr("target " + std::to_string(j) + " falls outside the scaled torus ball");
        }
        if (t == 0) return;
        DeviceGuard dg(E.device);
        std::lock_guard<std::mutex> lk(E.mu);
        const Geometry g = w.geom;
        PointSet tp;
        build_pointset(tp, sc, t, w.d, g, item_chunk(t, w.d), gather_chunk(t, w.d), E.stream);
        DevBuf<double> tout;
        tout.alloc(t);
        DPSet dp{};
        dp.F = tp.F.p;
        dp.CP = tp.CP.p;
        dp.n = t;
        dp.win = 0;
        dp.out = ptr_kind == KSVM_NFFT_DEVICE ? out : tout.p;
        DevBuf<DPSet> dps;
        dps.upload(&dp, 1, E.stream);
        std::vector<Item> its = tp.gitems;
        for (auto& it : its) it.ps = 0;
        DevBuf<Item> ditems;
        ditems.upload(its.data(), its.size(), E.stream);
        const double* dv = v;
        cudaStream_t es = static_cast<cudaStream_t>(stream);
        if (ptr_kind == KSVM_NFFT_HOST) {
            CK(cudaMemcpyAsync(E.vbuf.p, v, sizeof(double) * E.n, cudaMemcpyHostToDevice, E.stream));
            dv = E.vbuf.p;
        } else if (ptr_kind == KSVM_NFFT_DEVICE) {
            CK(cudaEventRecord(E.ev_in, es));
            CK(cudaStreamWaitEvent(E.stream, E.ev_in, 0));
        } else {
            throw std::invalid_argument("bad ptr_kind");
        }
        E.run_grid(dv);
        launch_gather(w.d, 2 * E.cfg.window_cutoff, w.dw.PE, ditems.p, static_cast<int>(its.size()), dps.p,
                      E.d_wins.p, E.stream);
        ++launch_counter();
        CK(cudaGetLastError());
        if (ptr_kind == KSVM_NFFT_HOST) {
            CK(cudaMemcpyAsync(out, tout.p, sizeof(double) * t, cudaMemcpyDeviceToHost, E.stream));
        } else {
            CK(cudaEventRecord(E.ev_out, E.stream));
            CK(cudaStreamWaitEvent(es, E.ev_out, 0));
        }
        CK(cudaStreamSynchronize(E.stream));  // target scratch is freed on return
    });
}

int64_t ksvm_nfft_plan_num_sources(const ksvm_nfft_plan* plan) { return plan ? plan->e.n : 0; }
int ksvm_nfft_plan_dim(const ksvm_nfft_plan* plan) { return plan ? plan->e.wins[0]->d : 0; }
double ksvm_nfft_plan_scaled_length(const ksvm_nfft_plan* plan) { return plan->e.wins[0]->ell_s; }
double ksvm_nfft_plan_coefficient_sum(const ksvm_nfft_plan* plan) { return plan->e.wins[0]->coef_sum; }

int ksvm_nfft_plan_scale_points(const ksvm_nfft_plan* plan, const double* pts, int64_t t, int64_t ld,
                                int layout, double* out) {
    return guarded([&] {
        if (!plan || !pts || !out) throw std::invalid_argument("null argument");
        const Window& w = *plan->e.wins[0];
        check_layout(t, w.d, ld, layout);
        for (int64_t i = 0; i < t; ++i)
            for (int c = 0; c < w.d; ++c) {
                const double x = (at(pts, i, c, ld, layout) - w.center[c]) * w.scale;
                if (layout == KSVM_NFFT_COL_MAJOR) out[c * ld + i] = x;
                else out[i * ld + c] = x;
            }
    });
}

void ksvm_nfft_plan_free(ksvm_nfft_plan* plan) { delete plan; }

}  // extern "C"
