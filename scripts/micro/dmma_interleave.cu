// Does the order in which DMUL and DMMA are issued matter on the shared FP64 datapath?
// Per "group": 8 DMMA.8x8x4 whose A operand is a fresh DMUL product (the d = 3 spread's
// inner loop), issued (0) one DMUL right before each DMMA, (1) 8 DMUL then 8 DMMA,
// (2) 8 DMUL per 16 DMMA (the products repeat and are shared), (3) 8 DMMA only (no DMUL),
// (5) 4 DMUL feeding 8 DMMA at once (the split-power spread), (6) the same with the products
// made one iteration ahead. ptxas interleaves (0) and (1) identically. warps/SM swept.
#include <cstdio>
#include <cuda_runtime.h>
#define DMMA(c0, c1, a, b) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))
#define DMULV(r, x, y) asm volatile("mul.f64 %0, %1, %2;" : "=d"(r) : "d"(x), "d"(y))
template <int MODE>
__global__ void k(double* out, double x, int iters, int one) {
    double w[8], c[8][2], u = x + 1e-9 * threadIdx.x, b = x - 1e-9 * threadIdx.x;
    for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = 0; w[i] = x + 1e-7 * i; }
    double nx[4] = {x, x, x, x};
    for (int it = 0; it < iters; ++it) {
        double a[16];
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) { DMULV(a[i], w[i], u); DMMA(c[i][0], c[i][1], a[i], b); }
        } else if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) DMULV(a[i], w[i], u);
#pragma unroll
            for (int i = 0; i < 8; ++i) DMMA(c[i][0], c[i][1], a[i], b);
        } else if (MODE == 2) {
#pragma unroll
            for (int i = 0; i < 16; ++i) DMULV(a[i], w[i & 7], u);
#pragma unroll
            for (int i = 0; i < 16; ++i) DMMA(c[i & 7][0], c[i & 7][1], a[i], b);
            ++it;
        } else if (MODE == 4) {  // software-pipelined: products of the next group under this group's DMMAs, in two clumps
            double n[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) DMULV(n[i], w[i], u);
#pragma unroll
            for (int i = 0; i < 8; ++i) DMMA(c[i][0], c[i][1], n[i], b);
        } else if (MODE == 7) {  // warp-specialised: of 4 warps, 3 issue only DMMA (8 per step), 1 only DMUL (12 per step)
            if (((threadIdx.x >> 5) + blockIdx.x / 148) % 4 == 3) {  // one DMUL warp per SMSP (CTA k of an SM rotates it)
#pragma unroll
                for (int i = 0; i < 12; ++i) DMULV(nx[i & 3], w[i & 7], u);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) DMMA(c[i][0], c[i][1], w[i], b);
            }
        } else if (MODE == 8) {  // mode 5 with the 4 DMULs fenced into their own basic block (a 1-trip loop ptxas cannot see through)
            double p[4];
#pragma unroll 1
            for (int r = 0; r < one; ++r) {
#pragma unroll
                for (int i = 0; i < 4; ++i) DMULV(p[i], w[i], u);
            }
            DMMA(c[0][0], c[0][1], w[4], p[0]); DMMA(c[1][0], c[1][1], w[4], p[1]);
            DMMA(c[2][0], c[2][1], w[4], p[2]); DMMA(c[3][0], c[3][1], w[4], b);
            DMMA(c[4][0], c[4][1], p[3], p[0]); DMMA(c[5][0], c[5][1], p[3], p[1]);
            DMMA(c[6][0], c[6][1], p[3], p[2]); DMMA(c[7][0], c[7][1], p[3], b);
        } else if (MODE == 5) {  // split-power spread: 4 products feed 8 DMMAs, consumed at once
            double p[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) DMULV(p[i], w[i], u);
            DMMA(c[0][0], c[0][1], w[4], p[0]); DMMA(c[1][0], c[1][1], w[4], p[1]);
            DMMA(c[2][0], c[2][1], w[4], p[2]); DMMA(c[3][0], c[3][1], w[4], b);
            DMMA(c[4][0], c[4][1], p[3], p[0]); DMMA(c[5][0], c[5][1], p[3], p[1]);
            DMMA(c[6][0], c[6][1], p[3], p[2]); DMMA(c[7][0], c[7][1], p[3], b);
        } else if (MODE == 6) {  // same mix, products made one iteration ahead (carried in nx[])
            double p[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) p[i] = nx[i];
#pragma unroll
            for (int i = 0; i < 4; ++i) DMULV(nx[i], w[i], u);
            DMMA(c[0][0], c[0][1], w[4], p[0]); DMMA(c[1][0], c[1][1], w[4], p[1]);
            DMMA(c[2][0], c[2][1], w[4], p[2]); DMMA(c[3][0], c[3][1], w[4], b);
            DMMA(c[4][0], c[4][1], p[3], p[0]); DMMA(c[5][0], c[5][1], p[3], p[1]);
            DMMA(c[6][0], c[6][1], p[3], p[2]); DMMA(c[7][0], c[7][1], p[3], b);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) DMMA(c[i][0], c[i][1], w[i], b);
        }
        u += 1e-12;
    }
    double s = nx[0] + nx[1] + nx[2] + nx[3]; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> void run(double* out, int wpsm) {
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int iters = 4096; dim3 grid(148 * (wpsm / 4)), block(128);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(s); k<MODE><<<grid, block>>>(out, 1.0000001, iters, 1); cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, s, e);
        double warps = grid.x * block.x / 32.0;
        double fma = warps * iters * 8 * 256;
        double cyc = ms * 1e-3 * 1.965e9 / (iters * (wpsm / 4.0));  // pipe cycles per group per SMSP
        if (MODE == 7) { fma *= 0.75; cyc /= 0.75; }
        if (rep) printf("mode %d warps/SM %2d: %.3f ms  DMMA %.2f TF  %.1f cycles per 8-DMMA group per SMSP\n", MODE, wpsm, ms, 2 * fma / ms / 1e9, cyc);
    }
}
int main() {
    double* out; cudaMalloc(&out, 148 * 16 * 128 * sizeof(double));
    for (int w : {4, 8, 12, 16, 24}) { run<3>(out, w); run<0>(out, w); run<1>(out, w); run<2>(out, w); run<5>(out, w); run<6>(out, w); run<8>(out, w); }
    // mode 7: 3 of 4 warps are DMMA warps: a 'group' is one DMMA warp's step, so scale warps/SM by 4/3
    for (int w : {16, 32}) run<7>(out, w);
    return 0;
}
