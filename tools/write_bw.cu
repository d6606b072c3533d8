// Write-only HBM bandwidth on this B200 (the ceiling of the stress kernel,
// which streams 56 B per Gauss point): 16-byte streaming stores, 8-byte
// stores, and a 1:16 read:write mix, over 14.6 GB.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void w16(size_t n2, double2 *o) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x)
        __stcs(o + i, make_double2(double(i), 1.0));
}
__global__ void w8(size_t n, double *o) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        __stcs(o + i, double(i));
}
__global__ void w8plain(size_t n, double *o) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        o[i] = double(i);
}
int main() {
    const size_t bytes = 14616ull << 20;
    double *o; if (cudaMalloc(&o, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, auto f) {
        float best = 1e9;
        for (int r = 0; r < 4; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms; }
        printf("%-28s %8.3f ms  %7.1f GB/s\n", name, best, bytes / best / 1e6);
    };
    for (int per : {4, 8, 16}) {
        char nm[64];
        snprintf(nm, 64, "stcs 16B grid=%d*sms", per); run(nm, [&] { w16<<<sms * per, 256>>>(bytes / 16, (double2 *)o); });
        snprintf(nm, 64, "stcs 8B grid=%d*sms", per); run(nm, [&] { w8<<<sms * per, 256>>>(bytes / 8, o); });
        snprintf(nm, 64, "plain 8B grid=%d*sms", per); run(nm, [&] { w8plain<<<sms * per, 256>>>(bytes / 8, o); });
    }
    run("cudaMemset", [&] { cudaMemsetAsync(o, 0, bytes); });
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
