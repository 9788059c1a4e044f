// Shared host/device structures of the B200 ANOVA-NFFT engine.
//
// Vocabulary: a *window* is one ANOVA feature group (d_l
// <= 3 features) with its own NFFT plan; its *sources* are the n scaled
// nodes; the *grid* is the sigma-oversampled M^d torus grid restricted to
// the nodes any in-ball point can touch; a *cell* is the unit grid cube a
// point falls in (floor(x M)); a *tile* is TC^d cells whose points one CTA
// processes; an *item* is a tile's point range (heavy tiles are split into
// several items); a *patch* is the (TC+2m-1)^d grid block an item spreads
// into.
//
// Window factors. The reference weight of tap o (0..2m-1) in dimension t is
//   phi = exp(-(u_t - o)^2 / b) / sqrt(pi b),  u_t = x_t M - floor(x_t M) + m - 1
// (P:src/fastsum.cpp:75-78, 222-228). Expanding the square,
//   prod_t phi_t(o_t) = P * prod_t Q_t^{o_t} R[o_t],
//   P = (pi b)^{-d/2} exp(-sum_t u_t^2 / b),  Q_t = exp(2 u_t / b),  R[o] = exp(-o^2 / b),
// so a plan stores (P, Q_0..Q_{d-1}, tile-local cell code) per sorted point
// and the apply evaluates no exp() at all. Layout is AoS so a point costs
// three vector loads: F[i] = {P, Q0, Q1, Q2} (32 B), CP[i] = {code, perm}.
#pragma once

#include <cstdint>

namespace ksvm_nfft {

constexpr int kMaxSpan = 16;  // 2m, m <= 8 (P:src/fastsum.cpp:41-42, w[3][16] at :225)
// d = 3 column kernels (sparse cells): the 16 cell columns (l0, l1) of a
// 4^3-cell tile; per spread item the first sorted point of columns 0..16.
// spread3c: 8 warps, two columns each; gather3c: one CTA per l0 slab, one
// warp per column.
constexpr int kColWarps = 8;
constexpr int kColBounds = 17;

// One tile's (or part of a tile's) sorted point range.
struct Item {
    int ps;           // point-set slot
    int tile;         // linear tile index within the window's tile grid
    int begin;        // sorted point range [begin, end)
    int end;
    long long patch;  // offset of this item's patch in the patch buffer (spread only)
};

// Per-window grid description and device buffers.
struct DWin {
    int d;       // window dimension 1..3
    int S;       // taps per dimension, 2m
    int m;
    int M;       // grid edge sigma*N
    int Lg;      // local grid edge (<= M)
    int lo;      // global index of extended node 0
    int wrap;    // 1: local index = (lo + e) mod M (Lg == M); 0: local index = e
    int cmin;    // smallest cell index floor(xM) any in-ball point can have
    int ncell;   // number of cell indices per dimension
    int TC;      // cells per tile edge
    int ntile;   // tiles per dimension
    int PE;      // patch edge TC + S - 1
    int Lext;    // extended node count ncell + S - 1
    double Mf;   // M as double
    double bwin; // Gaussian window shape b (P:src/fastsum.cpp:124)
    double invb; // 1 / b
    double Cw;   // 1/sqrt(pi b)        (P:src/fastsum.cpp:77)
    double R[kMaxSpan];  // exp(-o^2/b), o = 0..S-1
    double* G;   // spread grid, Lg^d
    double* H;   // filtered grid, Lg^d
    double* T[4];  // separable-convolution temporaries, Lg^d each
    const double* tabA;  // a(r), r = -(Lg-1)..(Lg-1), index r + Lg - 1
    const double* tabS;  // s(r)
    const int* tile_first;  // sources: first item of each tile (ntile^d + 1 entries)
    const long long* tile_patch;  // patch-buffer offset of each tile's (pre-reduced) patch, -1 if empty
    int item_base;          // global index of the window's first source item
    long long patch_base;   // patch-buffer offset of that item
};

// A sorted point set (a window's sources, or cross-apply targets).
struct DPSet {
    const double4* F;    // {P, Q0, Q1, Q2}: P = (pi b)^{-d/2} exp(-sum u^2/b), Q_t = exp(2 u_t/b)
    const float4* F32;   // fp32 mode, d = 3, m = 4: cell-relative {P, Q0, Q1, Q2} (nfft_f32.cu); else null
    const int2* CP;      // {tile-local cell code sum_t (c_t mod TC) TC^{d-1-t}, original index}
    long long n;
    int win;             // owning window slot
    double* out;         // gather output, original order (length n)
    const double* vsrc;  // spread input (length n) if not the apply's v: the per-distinct-point
                         // sums of an exact-duplicate window; nullptr otherwise
};

constexpr int kSegChunk = 256;  // members per warp in the duplicate-group sums of v
constexpr int kSmallBins = 16;  // windows with <= this many distinct points use register bins

}  // namespace ksvm_nfft
