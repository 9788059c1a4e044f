// Throughput of the legacy warp-level tensor path (mma.sync) on B200 for the types an fp32-accurate
// split scheme could use: tf32 m16n8k8 and bf16 / f16 m16n8k16, fp32 accumulate.
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND>
__global__ void k(float* out, int iters) {
    unsigned a[4], b[2];
    float c[8][4];
    for (int i = 0; i < 4; ++i) a[i] = 0x3f800000u + threadIdx.x + i;
    for (int i = 0; i < 2; ++i) b[i] = 0x3f800000u + 2 * threadIdx.x + i;
    for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            else if (KIND == 1)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    float s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int KIND> void run(float* out, int wpsm, const char* name, double macs) {
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int iters = 4096; dim3 grid(148 * (wpsm / 4)), block(128);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(s); k<KIND><<<grid, block>>>(out, iters); cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, s, e);
        double warps = grid.x * block.x / 32.0, n = warps * iters * 8;
        double cyc = ms * 1e-3 * 1.965e9 / (iters * 8.0 * (wpsm / 4.0));
        if (rep) printf("%s warps/SM %2d: %.3f ms  %.1f TFLOP/s  %.2f cycles per mma per SMSP\n", name, wpsm, ms, 2 * n * macs / ms / 1e9, cyc);
    }
}

// tf32 MMAs with the operand work of the 3xTF32 kernels between them: per MMA NF fp32
// instructions (FMUL, LOP, FADD in turn) on values that feed the next MMA's operands.
template <int NF>
__global__ void kmix(float* out, int iters) {
    unsigned a[4], b[2];
    float c[8][4], w[8];
    for (int i = 0; i < 4; ++i) a[i] = 0x3f800000u + threadIdx.x + i;
    for (int i = 0; i < 2; ++i) b[i] = 0x3f800000u + 2 * threadIdx.x + i;
    for (int i = 0; i < 8; ++i) { w[i] = 1.0f + 1e-3f * i + 1e-6f * threadIdx.x; for (int j = 0; j < 4; ++j) c[i][j] = 0.f; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                float& x = w[(i + f) & 7];
                if (f % 3 == 0) asm volatile("mul.f32 %0, %0, %1;" : "+f"(x) : "f"(1.0000001f));
                else if (f % 3 == 1) asm volatile("and.b32 %0, %1, 0xffffe000;" : "=r"(a[f & 3]) : "r"(__float_as_uint(x)));
                else asm volatile("sub.f32 %0, %1, %2;" : "=f"(x) : "f"(x), "f"(__uint_as_float(a[f & 3])));
            }
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    float s = 0; for (int i = 0; i < 8; ++i) { s += w[i]; for (int j = 0; j < 4; ++j) s += c[i][j]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NF> void runmix(float* out, int wpsm) {
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int iters = 4096; dim3 grid(148 * (wpsm / 4)), block(128);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(s); kmix<NF><<<grid, block>>>(out, iters); cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, s, e);
        double cyc = ms * 1e-3 * 1.965e9 / (iters * 8.0 * (wpsm / 4.0));
        if (rep) printf("tf32 m16n8k8 + %d fp32 ops per mma, warps/SM %2d: %.3f ms  %.2f cycles per mma per SMSP\n", NF, wpsm, ms, cyc);
    }
}
int main() {
    float* out; cudaMalloc(&out, 148 * 16 * 128 * sizeof(float));
    for (int w : {4, 8, 16, 32}) {
        run<0>(out, w, "tf32 m16n8k8 ", 16 * 8 * 8);
        run<1>(out, w, "bf16 m16n8k16", 16 * 8 * 16);
        run<2>(out, w, "f16  m16n8k16", 16 * 8 * 16);
    }
    for (int w : {16, 20}) { runmix<0>(out, w); runmix<1>(out, w); runmix<2>(out, w); runmix<3>(out, w); runmix<4>(out, w); }
    return 0;
}
