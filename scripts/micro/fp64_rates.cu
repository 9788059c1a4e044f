// Microbenchmark: FP64 vector DFMA vs DMMA.8x8x4 throughput on one B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_k(double* out, double x, int iters) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = x + i + threadIdx.x;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], x, 1e-3);
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dmma_k(double* out, double x, int iters) {
    double a = x + threadIdx.x, b = x - threadIdx.x;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* out; cudaMalloc(&out, 148 * 32 * 1024 * sizeof(double));
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        for (int kind = 0; kind < 2; ++kind) {
            dim3 grid(148 * 4), block(32 * warps / 4);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(s);
                if (kind == 0) dfma_k<<<grid, block>>>(out, 1.0000001, iters);
                else dmma_k<<<grid, block>>>(out, 1.0000001, iters);
                cudaEventRecord(e); cudaEventSynchronize(e);
                float ms; cudaEventElapsedTime(&ms, s, e);
                double threads = (double)grid.x * block.x;
                double fma = kind == 0 ? threads * iters * 8 : (threads / 32) * iters * 8 * 256;
                if (rep) printf("%s warps/SM=%d: %.2f TFLOPS (%.3f ms)\n", kind ? "DMMA" : "DFMA", warps, 2 * fma / ms / 1e9, ms);
            }
        }
    }
    return 0;
}
