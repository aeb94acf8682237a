// ffma_peak.cu -- chip-wide fp32 FFMA throughput of this B200 (the roofline denominator of the
// K1 "ffma" / "exact" SIMT paths; not product code).  Every thread runs 8 independent FFMA
// chains (enough ILP to cover the 4-cycle FMA latency), 4 x 148 CTAs of 512 threads, timed
// with CUDA events after a warm-up.  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ffma_peak.cu -o tools/ffma_peak.bin
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) ffma_kernel(float *out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
          x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5f) out[blockIdx.x] = s;  // keeps the chains alive
}

int main() {
    float *out;
    cudaMalloc(&out, 4096 * sizeof(float));
    const int blocks = 148 * 4, threads = 512, iters = 4096;
    ffma_kernel<<<blocks, threads>>>(out, 64, 0.999f, 1e-3f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double flops = 2.0 * blocks * threads * double(iters) * 16 * 8;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"ffma_tflops\": %.2f, \"ms\": %.3f, \"blocks\": %d, \"threads\": %d, \"max_clock_mhz\": %.0f, "
           "\"error\": \"%s\"}\n",
           flops / (best * 1e-3) / 1e12, best, blocks, threads, clk / 1e3, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
