// Measured CUDA-core peaks on the B200 under sustained load (roofline
// denominators for the compute side of the sweep kernels):
//   FP32 packed FFMA2 (the c64 sweeps' arithmetic), FP32 scalar FFMA, FP64 DFMA
//   (the c128 paths).  Each kernel runs many independent FMA chains per thread
//   (enough ILP for the 4-cycle latency), 148 x 8 CTAs of 256 threads, back to
//   back for >= `seconds`, timed with CUDA events; prints one JSON line.
// Build/run: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/peaks.cu -o /tmp/peaks && /tmp/peaks
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kChains = 16;

__global__ void k_ffma2(float2* out, float a, float b, int iters) {
    float2 x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = make_float2(threadIdx.x + i, i);
    const float2 m = make_float2(a + threadIdx.x * 1e-9f, a), c = make_float2(b, -b);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) x[i] = __ffma2_rn(x[i], m, c);
    }
    float2 s = make_float2(0, 0);
#pragma unroll
    for (int i = 0; i < kChains; ++i) { s.x += x[i].x; s.y += x[i].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// all three operands in per-thread registers (the sweeps' form: amplitudes x matrix entries)
__global__ void k_ffma2r(float2* out, float a, float b, int iters) {
    float2 x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = make_float2(threadIdx.x + i, i);
    const float2 m = make_float2(a + threadIdx.x * 1e-9f, a - threadIdx.x * 1e-9f);
    const float2 c = make_float2(b + threadIdx.x * 1e-9f, -b - threadIdx.x * 1e-9f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) x[i] = __ffma2_rn(x[i], m, c);
    }
    float2 s = make_float2(0, 0);
#pragma unroll
    for (int i = 0; i < kChains; ++i) { s.x += x[i].x; s.y += x[i].y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, float a, float b, int iters) {
    float x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x + i;
    const float m = a + threadIdx.x * 1e-9f, c = b - threadIdx.x * 1e-9f;  // register operands (3-reg form)
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) x[i] = fmaf(x[i], m, c);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double a, double b, int iters) {
    double x[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x + i;
    const double m = a + threadIdx.x * 1e-12, c = b - threadIdx.x * 1e-12;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) x[i] = fma(x[i], m, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
static double time_tflops(F launch, double flops_per_launch, double seconds) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();  // warm-up
    cudaDeviceSynchronize();
    float ms = 0;
    int reps = 1;
    for (;;) {  // grow the repetition count until the timed region lasts >= seconds
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms >= 1000.0 * seconds) break;
        reps *= 2;
    }
    return flops_per_launch * reps / (ms * 1e-3) / 1e12;
}

int main(int argc, char** argv) {
    const double seconds = argc > 1 ? atof(argv[1]) : 1.0;
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    void* o;
    cudaMalloc(&o, 1 << 26);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    const double thr = (double)blocks * threads;
    const double f_ffma2 = 2.0 * 2 * kChains * (double)iters * thr;  // 2 lanes x (mul + add)
    const double f_ffma = 2.0 * kChains * (double)iters * thr;
    const double f_dfma = 2.0 * kChains * (double)iters * thr;
    const double t2 = time_tflops([&] { k_ffma2<<<blocks, threads>>>((float2*)o, 0.9999f, 1e-4f, iters); }, f_ffma2, seconds);
    const double t1 = time_tflops([&] { k_ffma<<<blocks, threads>>>((float*)o, 0.9999f, 1e-4f, iters); }, f_ffma, seconds);
    const double t2r = time_tflops([&] { k_ffma2r<<<blocks, threads>>>((float2*)o, 0.9999f, 1e-4f, iters); }, f_ffma2, seconds);
    // the sweeps' occupancy: 2 CTAs x 256 threads per SM (16 warps)
    const int b2 = sms * 2;
    const double t2r_occ = time_tflops([&] { k_ffma2r<<<b2, threads>>>((float2*)o, 0.9999f, 1e-4f, iters); },
                                       f_ffma2 * b2 / blocks, seconds);
    const double t1_occ = time_tflops([&] { k_ffma<<<b2, threads>>>((float*)o, 0.9999f, 1e-4f, iters); },
                                      f_ffma * b2 / blocks, seconds);
    const double t64 = time_tflops([&] { k_dfma<<<blocks, threads>>>((double*)o, 0.9999, 1e-4, iters); }, f_dfma, seconds);
    const double nominal32 = 2.0 * 128 * sms * (clk * 1e3) / 1e12;
    printf("{\"fp32_ffma2_uniform_operand_tflops\": %.2f, \"fp32_ffma2_register_operands_tflops\": %.2f, "
           "\"fp32_ffma2_register_operands_16warps_tflops\": %.2f, \"fp32_ffma_3reg_16warps_tflops\": %.2f, ",
           t2, t2r, t2r_occ, t1_occ);
    printf("\"fp32_ffma_3reg_tflops\": %.2f, \"fp64_dfma_tflops\": %.2f, "
           "\"sms\": %d, \"max_sm_mhz\": %.0f, \"fp32_nominal_tflops_at_max_clock\": %.2f, "
           "\"how\": \"%d x %d threads, %d independent FMA chains/thread, back to back for >= %.1f s per kernel, CUDA events\"}\n",
           t1, t64, sms, clk / 1e3, nominal32, blocks, threads, kChains, seconds);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
