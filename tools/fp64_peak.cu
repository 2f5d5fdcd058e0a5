// FP64 FMA throughput probe (not part of the product): the denominator for the
// multi-RHS products' FP64 roofline (C5 is FP64-FMA bound and
// MEASURED_PEAKS.json carries no FP64 figure).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int blocks = nsm * 8, threads = 256, iters = 20000;
    k_fma<<<blocks, threads>>>(out, 100, 0.999999, 1e-9);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double tflops = 2.0 * 8 * double(iters) * blocks * threads / (ms * 1e-3) / 1e12;
        if (tflops > best) best = tflops;
    }
    printf("{\"fp64_fma_tflops\": %.2f, \"sms\": %d, \"kernel\": \"8 independent DFMA chains x %d iters, %d x %d threads\"}\n",
           best, nsm, iters, blocks, threads);
    return 0;
}
