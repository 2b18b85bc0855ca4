// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput microbenchmark:
// does B200 run FP64 MMA faster than DFMA (scripts/fp64_peak.cu)?  Each warp
// keeps NACC independent 8x8 accumulators, 4 CTAs x 256 threads per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NACC = 8;
constexpr int ITERS = 2048;

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) k_dmma(double *out, double a, double b) {
    double c[NACC][2];
#pragma unroll
    for (int k = 0; k < NACC; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
    double aa = a + threadIdx.x * 1e-9, bb = b;
#pragma unroll 2
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int k = 0; k < NACC; ++k) dmma(c[k][0], c[k][1], aa, bb);
    double s = 0;
#pragma unroll
    for (int k = 0; k < NACC; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double *out;
    cudaMalloc(&out, sizeof(double));
    for (int cps : {1, 2, 4}) {
        const int blocks = sms * cps, threads = 256;
        k_dmma<<<blocks, threads>>>(out, 0.999999, 1e-7);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_dmma<<<blocks, threads>>>(out, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double fmas = (double)blocks * (threads / 32) * ITERS * NACC * 256.0;
        printf("{\"ctas_per_sm\": %d, \"dmma_tflops\": %.3f, \"fma_per_clk_per_sm\": %.2f, \"ms\": %.4f}\n",
               cps, 2.0 * fmas / (best * 1e-3) / 1e12, fmas / (best * 1e-3) / (clk * 1e3) / sms, best);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
