// Microbenchmark: FP32 FFMA (3-register form) vs packed FFMA2 throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, float a, float b, int iters) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
    float m0 = a + threadIdx.x * 1e-7f, m1 = b - threadIdx.x * 1e-7f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], m0, m1 * x[(i + 1) & 15]);
    }
    float s = 0; for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float2* out, float a, float b, int iters) {
    float2 x[16];
    for (int i = 0; i < 16; ++i) x[i] = make_float2(threadIdx.x + i, i);
    float2 m0 = make_float2(a + threadIdx.x * 1e-7f, a), m1 = make_float2(b, b - threadIdx.x * 1e-7f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = __ffma2_rn(x[i], m0, __fmul2_rn(m1, x[(i + 1) & 15]));
    }
    float2 s = make_float2(0, 0); for (int i = 0; i < 16; ++i) { s.x += x[i].x; s.y += x[i].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* o; cudaMalloc(&o, 1 << 26);
    int blocks = 148 * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0); k_ffma<<<blocks, threads>>>(o, 0.999f, 0.001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 2 * 16 * (double)iters * blocks * threads;  // fma + mul per element
        printf("FFMA/FMUL scalar : %.2f ms  %.1f TFLOP/s  (%.1f Ginstr/s)\n", ms, flops / ms / 1e9, flops / 2 / ms / 1e6 / 1e3);
        cudaEventRecord(e0); k_ffma2<<<blocks, threads>>>((float2*)o, 0.999f, 0.001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 2 * 2 * 16 * (double)iters * blocks * threads;
        printf("FFMA2/FMUL2 packed: %.2f ms  %.1f TFLOP/s  (%.1f Ginstr/s)\n", ms, flops / ms / 1e9, flops / 4 / ms / 1e6 / 1e3);
    }
    return 0;
}
