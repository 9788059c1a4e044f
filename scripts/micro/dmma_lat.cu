// DMMA.8x8x4 / DMUL / LDS latency (one warp, dependent chains) and DMMA
// throughput per SMSP vs warps per SMSP and independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void chain_k(double* out, long long* cyc, double x, int iters) {
    double c[CH][2];
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = x * i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], x, x);
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void dmul_k(double* out, long long* cyc, double x, int iters) {
    double a = x + threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) a = a * x;
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int CH> void run(double* out, long long* cyc, int blocks, int threads) {
    int iters = 4096;
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(s);
        chain_k<CH><<<blocks, threads>>>(out, cyc, 1.0000001, iters);
        cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, s, e);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double warps = blocks * threads / 32.0;
        if (rep) printf("chains=%2d blocks=%4d threads=%4d: %.1f cyc per DMMA-step (warp 0), %.2f TF\n", CH, blocks,
                        threads, (double)c / iters / CH, warps * iters * CH * 512.0 / ms / 1e9);
    }
}
int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 8 * sizeof(double)); cudaMalloc(&cyc, 8);
    run<1>(out, cyc, 1, 32); run<2>(out, cyc, 1, 32); run<4>(out, cyc, 1, 32); run<8>(out, cyc, 1, 32);
    run<16>(out, cyc, 1, 32);
    for (int w : {1, 2, 4, 8, 16}) { run<4>(out, cyc, 148, 128 * w / 4 * 4 / 4 * 1 ); }
    run<1>(out, cyc, 148, 128); run<2>(out, cyc, 148, 128); run<4>(out, cyc, 148, 128); run<8>(out, cyc, 148, 128);
    run<1>(out, cyc, 148, 512); run<2>(out, cyc, 148, 512); run<4>(out, cyc, 148, 512); run<8>(out, cyc, 148, 512);
    run<8>(out, cyc, 148, 1024);
    dmul_k<<<1, 32>>>(out, cyc, 1.0000001, 4096); cudaDeviceSynchronize();
    dmul_k<<<1, 32>>>(out, cyc, 1.0000001, 4096);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMUL dependent latency: %.1f cyc\n", (double)c / 4096);
    return 0;
}
