// DFMA throughput microbenchmark (the compositing roofline is
// the fp64 pipe).  Independent FMA chains per thread, enough warps to hide the
// pipe latency; reports TFLOP/s counting an FMA as 2 flops.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void __launch_bounds__(256) k_dfma(double *out, int iters, double a, double b) {
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;  // keep the chains alive
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 8);
    const int iters = 1 << 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int blocksPerSm = 4; blocksPerSm <= 8; blocksPerSm *= 2) {
        const int grid = sms * blocksPerSm;
        k_dfma<8><<<grid, 256>>>(out, 1024, 0.999999, 1e-7);  // warm-up
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            k_dfma<8><<<grid, 256>>>(out, iters, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            const double flops = 2.0 * 8.0 * iters * (double)grid * 256.0;
            const double tf = flops / (ms * 1e-3) / 1e12;
            if (tf > best) best = tf;
        }
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"fp64_fma_tflops\": %.2f, \"sms\": %d, \"clock_khz\": %d, \"what\": \"DFMA, 8 chains/thread, best of 10\"}\n",
           best, sms, clk);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
