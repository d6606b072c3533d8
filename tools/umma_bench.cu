// tcgen05.mma issue-rate microbenchmark (B200): cycles per MMA instruction
// for kind::i8 / kind::tf32 / kind::f16, A from smem (SS) or TMEM (TS),
// M = 128, N in {16 .. 256}. One CTA per SM, operands are garbage (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_bench tools/umma_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

template <int KIND, bool TS, bool WARP_ISSUE = false>
__global__ void bench(int reps, int n, int nacc, long long *cycles) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
    uint32_t fmt;
    if (KIND == 0) fmt = (2u << 4) | (1u << 7) | (1u << 10);  // i8 -> s32
    else if (KIND == 1) fmt = (1u << 4) | (2u << 7) | (2u << 10);  // tf32 -> f32
    else fmt = (1u << 4) | (1u << 7) | (1u << 10);  // bf16 -> f32
    const uint32_t idesc = fmt | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
    long long t0 = 0, t1 = 0;
    if (WARP_ISSUE && warp == 0) {
        const uint64_t db = desc(base + 32768), da = desc(base);
        t0 = clock64();
        for (int i = 0; i < reps; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t dcol = tmem + static_cast<uint32_t>((j % nacc) * n);
                asm volatile("{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" ::"r"(dcol),
                             "l"(da), "l"(db), "r"(idesc), "r"(1));
            }
        }
        asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        do {
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar))
                         : "memory");
        } while (!ok);
        t1 = clock64();
        if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    } else if (!WARP_ISSUE && threadIdx.x == 0) {
        const uint64_t da = desc(base), db = desc(base + 32768);
        t0 = clock64();
        // 8 MMAs per iteration into 8 accumulators (compile-time offsets: no ALU work per MMA)
        for (int i = 0; i < reps; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t dcol = tmem + static_cast<uint32_t>((j % nacc) * n);
                if (TS) {
                    if (KIND == 0)
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(dcol),
                                     "r"(tmem + 480), "l"(db), "r"(idesc), "r"(1));
                    else
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}" ::"r"(dcol),
                                     "r"(tmem + 480), "l"(db), "r"(idesc), "r"(1));
                } else {
                    if (KIND == 0)
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" ::"r"(dcol),
                                     "l"(da), "l"(db), "r"(idesc), "r"(1));
                    else
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}" ::"r"(dcol),
                                     "l"(da), "l"(db), "r"(idesc), "r"(1));
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        do {
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar))
                         : "memory");
        } while (!ok);
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, bool TS, bool WI = false>
void run(const char *name, int n, int nacc = 1) {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    const int reps = 4096;
    cudaFuncSetAttribute(bench<KIND, TS, WI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    bench<KIND, TS, WI><<<148, 128, 100 * 1024>>>(reps, n, nacc, d);
    bench<KIND, TS, WI><<<148, 128, 100 * 1024>>>(reps, n, nacc, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148.0 * reps;
    const int k = KIND == 0 ? 32 : KIND == 1 ? 8 : 16;
    const double macs_per_clk = 128.0 * n * k / avg;
    std::printf("%s acc=%d %-6s %s N=%3d: %6.1f clk/MMA  %7.0f MAC/clk/SM  (%s)\n", WI ? "warp" : "thr ", nacc, name, TS ? "TS" : "SS", n, avg, macs_per_clk,
                e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    for (int n : {16, 32, 48, 64, 128}) run<0, false, false>("i8", n, 4);
    for (int n : {16, 32, 48, 64, 128}) run<0, false, true>("i8", n, 4);
    return 0;
}
