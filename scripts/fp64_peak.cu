// FP64 FMA throughput microbenchmark (the denominator of bench.py's
// fp64_roofline): 8 independent DFMA chains per thread, 4 CTAs x 256
// threads per SM, CUDA-event timed after a warm-up launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
//   ./fp64_peak > fp64_peak.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) k_dfma(double *out, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;   // keep the chains live
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);   // kHz
    double *out;
    cudaMalloc(&out, sizeof(double));
    const int blocks = sms * 4, threads = 256;
    k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double fmas = (double)blocks * threads * ITERS * CHAINS;
    const double tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
    const double per_clk_sm = fmas / (best * 1e-3) / (clk * 1e3) / sms;
    printf("{\"fp64_fma_tflops\": %.3f, \"dfma_per_clk_per_sm\": %.2f, \"sms\": %d, "
           "\"max_sm_khz\": %d, \"ms\": %.4f, \"note\": \"8 independent DFMA chains x 256 "
           "threads x 4 CTAs/SM, best of 5 launches (scripts/fp64_peak.cu)\"}\n",
           tflops, per_clk_sm, sms, clk, best);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
