// FP32 FMA throughput on B200 by instruction form (guides the fp32-mode
// kernels, csrc/nfft_f32.cu): scalar FFMA vs packed FFMA2, with the
// outer-product operand pattern of the spread (acc[j][c] += u[j] * w[c]).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ffma_rates ffma_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, float s, int iters) {
    float u[4], w[8];
    for (int j = 0; j < 4; ++j) u[j] = s * (threadIdx.x + j);
    for (int c = 0; c < 8; ++c) w[c] = s * (c + 1);
    if (MODE == 0) {
        float acc[4][8] = {};
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[j][c] = fmaf(u[j], w[c], acc[j][c]);
            u[it & 3] += 1e-7f;
        }
        float t = 0;
        for (int j = 0; j < 4; ++j)
            for (int c = 0; c < 8; ++c) t += acc[j][c];
        out[blockIdx.x * blockDim.x + threadIdx.x] = t;
    } else {
        float2 acc[4][4] = {};
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    acc[j][c] = __ffma2_rn(make_float2(u[j], u[j]), make_float2(w[2 * c], w[2 * c + 1]), acc[j][c]);
            u[it & 3] += 1e-7f;
        }
        float t = 0;
        for (int j = 0; j < 4; ++j)
            for (int c = 0; c < 4; ++c) t += acc[j][c].x + acc[j][c].y;
        out[blockIdx.x * blockDim.x + threadIdx.x] = t;
    }
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 16 * 256 * sizeof(float));
    const int iters = 20000;
    for (int bpsm : {4, 8, 16}) {
        for (int mode = 0; mode < 2; ++mode) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            auto run = [&] {
                if (mode == 0) k<0><<<148 * bpsm, 128>>>(out, 1e-3f, iters);
                else k<1><<<148 * bpsm, 128>>>(out, 1e-3f, iters);
            };
            run();
            cudaEventRecord(a);
            run();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double fl = 2.0 * 32 * iters * 148.0 * bpsm * 128;
            printf("%s blocks/SM=%2d warps/SM=%2d: %.1f TFLOP/s\n", mode ? "FFMA2" : "FFMA ", bpsm, bpsm * 4,
                   fl / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
