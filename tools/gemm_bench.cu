// K1 tile-configuration sweep on config-3 shapes (M = 10112 blocks,
// N = 654 reduced DoFs, K = 656): TFLOP/s per variant, CUDA events.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2411_12690_b200/csrc -o tools/gemm_bench tools/gemm_bench.cu
#include <cstdio>
#include <vector>
#include "kernels.cuh"
using namespace tsvb200;

template <class Cfg>
void run(const char *name, int M, int N, int K, const double *A, const double *B, double *C, unsigned *ctr, int sms) {
    cudaFuncSetAttribute(gemm_nt_f64<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_nt_f64<Cfg>, Cfg::THREADS, Cfg::SMEM);
    GemmParams p{};
    p.A = A; p.lda = K; p.Bt[0] = p.Bt[1] = B; p.ldb = K; p.C = C; p.ldc = K;
    p.m_tiles = M / Cfg::BM; p.n_tiles = (N + Cfg::BN - 1) / Cfg::BN; p.k_chunks = K / Cfg::KC;
    p.n_valid = N; p.n_store = N; p.tile_counter = ctr;
    const int grid = occ * sms;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) gemm_nt_f64<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM>>>(p);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) gemm_nt_f64<Cfg><<<grid, Cfg::THREADS, Cfg::SMEM>>>(p);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    double fl = 2.0 * (double)(M) * N * K;
    printf("{\"variant\":\"%s\",\"occ\":%d,\"smem\":%zu,\"ms\":%.4f,\"tflops\":%.2f,\"err\":\"%s\"}\n", name, occ, Cfg::SMEM, ms,
           fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char **argv) {
    int M = 10112, N = 654, K = 656;
    if (argc > 3) { M = atoi(argv[1]); N = atoi(argv[2]); K = atoi(argv[3]); }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int Npad = (N + 255) / 256 * 256;
    std::vector<double> h((size_t)M * K);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (i % 97) * 0.01;
    double *A, *B, *C; unsigned *ctr;
    cudaMalloc(&A, (size_t)M * K * 8); cudaMalloc(&B, (size_t)Npad * K * 8); cudaMalloc(&C, (size_t)M * K * 8);
    cudaMalloc(&ctr, 8); cudaMemset(ctr, 0, 8);
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(B, 0, (size_t)Npad * K * 8);
    cudaMemcpy(B, h.data(), (size_t)N * K * 8, cudaMemcpyHostToDevice);
    run<GemmCfg<128, 64, 2, 2, 16, 3, 2>>("128x64_w2x2_kc16_s3", M, N, K, A, B, C, ctr, sms);
    run<GemmCfg<128, 64, 2, 2, 16, 2, 3>>("128x64_w2x2_kc16_s2_3cta", M, N, K, A, B, C, ctr, sms);
    run<GemmCfg<128, 64, 2, 2, 8, 4, 3>>("128x64_w2x2_kc8_s4_3cta", M, N, K, A, B, C, ctr, sms);
    run<GemmCfg<64, 128, 2, 2, 16, 3, 2>>("64x128_w2x2_kc16_s3", M, N, K, A, B, C, ctr, sms);
    run<GemmCfg<128, 64, 2, 2, 8, 6, 2>>("128x64_w2x2_kc8_s6", M, N, K, A, B, C, ctr, sms);
    run<GemmCfg<128, 96, 2, 2, 16, 3, 2>>("128x96_w2x2_kc16_s3", M, N, K, A, B, C, ctr, sms);
    run<GemmCfg<96, 64, 2, 2, 16, 3, 2>>("96x64_w2x2_kc16_s3", M, N, K, A, B, C, ctr, sms);
    return 0;
}
