// Does FP64 vector work (DFMA) run concurrently with DMMA, or share its datapath?
#include <cstdio>
#include <cuda_runtime.h>
template <int NF>
__global__ void mix_k(double* out, double x, int iters) {
    double a = x + threadIdx.x, b = x - threadIdx.x;
    double c[8][2], f[8];
    for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = 0; f[i] = x * i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
        for (int j = 0; j < NF; ++j) f[j & 7] = fma(f[j & 7], x, 1e-3);
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NF> void run(double* out) {
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int iters = 2048; dim3 grid(148 * 4), block(128);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(s); mix_k<NF><<<grid, block>>>(out, 1.0000001, iters); cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, s, e);
        double warps = grid.x * block.x / 32.0;
        double dmma_fma = warps * iters * 8 * 256, dfma = grid.x * (double)block.x * iters * NF;
        if (rep) printf("NF=%2d DFMA per 8 DMMA: %.3f ms  DMMA %.1f TF  DFMA %.1f TF  total %.1f TF\n", NF, ms,
                        2 * dmma_fma / ms / 1e9, 2 * dfma / ms / 1e9, 2 * (dmma_fma + dfma) / ms / 1e9);
    }
}
int main() {
    double* out; cudaMalloc(&out, 148 * 4 * 128 * sizeof(double));
    run<0>(out); run<4>(out); run<8>(out); run<16>(out); run<32>(out); run<64>(out);
    return 0;
}
