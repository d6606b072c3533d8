// FP64 roofline denominators on this B200: DMMA.8x8x4 (mma.sync f64) and
// DFMA issue peaks from register-only loops, timed with CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double *out, int iters) {
    double acc[8][2];
    double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double *out, int iters) {
    double acc[16];
    double a = threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
    for (int i = 0; i < 16; ++i) acc[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], b, a);
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        dim3 grid(sms), block(32 * warps);
        dmma_loop<<<grid, block>>>(out, 100);
        cudaEventRecord(e0);
        dmma_loop<<<grid, block>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 256 * 8 * iters * (double)grid.x * warps;
        printf("{\"kind\":\"dmma\",\"warps_per_sm\":%d,\"tflops\":%.3f}\n", warps, flops / ms / 1e9);
        dfma_loop<<<grid, block>>>(out, 100);
        cudaEventRecord(e0);
        dfma_loop<<<grid, block>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 16 * iters * (double)grid.x * block.x;
        printf("{\"kind\":\"dfma\",\"warps_per_sm\":%d,\"tflops\":%.3f}\n", warps, flops / ms / 1e9);
    }
    return 0;
}
