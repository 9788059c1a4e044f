// Does the order in which DMUL and DMMA are issued matter on the shared FP64 datapath?
// Per "group": 8 DMMA.8x8x4 whose A operand is a fresh DMUL product (the d = 3 spread's
// inner loop), issued (0) one DMUL right before each DMMA, (1) 8 DMUL then 8 DMMA,
// (2) two groups: 16 DMUL then 16 DMMA, (3) 8 DMMA only (no DMUL). warps/SM swept.
#include <cstdio>
#include <cuda_runtime.h>
#define DMMA(c0, c1, a, b) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))
#define DMULV(r, x, y) asm volatile("mul.f64 %0, %1, %2;" : "=d"(r) : "d"(x), "d"(y))
template <int MODE>
__global__ void k(double* out, double x, int iters) {
    double w[8], c[8][2], u = x + 1e-9 * threadIdx.x, b = x - 1e-9 * threadIdx.x;
    for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = 0; w[i] = x + 1e-7 * i; }
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
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) DMMA(c[i][0], c[i][1], w[i], b);
        }
        u += 1e-12;
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> void run(double* out, int wpsm) {
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int iters = 4096; dim3 grid(148 * (wpsm / 4)), block(128);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(s); k<MODE><<<grid, block>>>(out, 1.0000001, iters); cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, s, e);
        double warps = grid.x * block.x / 32.0;
        double fma = warps * iters * 8 * 256;
        double cyc = ms * 1e-3 * 1.965e9 / (iters * (wpsm / 4.0));  // pipe cycles per group per SMSP
        if (rep) printf("mode %d warps/SM %2d: %.3f ms  DMMA %.2f TF  %.1f cycles per 8-DMMA group per SMSP\n", MODE, wpsm, ms, 2 * fma / ms / 1e9, cyc);
    }
}
int main() {
    double* out; cudaMalloc(&out, 148 * 16 * 128 * sizeof(double));
    for (int w : {4, 8, 12, 16, 24}) { run<3>(out, w); run<0>(out, w); run<1>(out, w); run<2>(out, w); }
    return 0;
}
