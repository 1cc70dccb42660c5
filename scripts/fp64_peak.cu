// FP64 peak probes on one B200 (denominator for the sup-sup roofline).
//   dfma: 8 independent FMA chains per thread, 148 x 8 CTAs of 256 threads.
//   dmma: mma.sync.m8n8k4.f64 (SASS DMMA), 4 independent accumulators per warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak scripts/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-7 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int pass = 0; pass < 2; ++pass) {
        float best = 1e30f;
        int grid = sms * 8, threads = 256;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            if (pass == 0) k_dfma<<<grid, threads>>>(out, iters, 0.9999999, 1e-9);
            else k_dmma<<<grid, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r && ms < best) best = ms;
        }
        double flops = pass == 0 ? 2.0 * 8 * iters * (double)grid * threads
                                 : 2.0 * 8 * 8 * 4 * 4 * (double)iters * grid * (threads / 32);
        printf("{\"probe\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d}\n",
               pass == 0 ? "dfma" : "dmma_m8n8k4", flops / best / 1e9, best, sms);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
    return 0;
}
