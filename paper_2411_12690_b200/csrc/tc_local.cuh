// Schwarz local solves on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
//   ZL[row][col] = sum_k XL32[row][k] * Ainv32_type(row)[col][k]
//
// The local inverses are a preconditioner, not the operator: the PCG
// iteration (K1, residuals, dot products) stays FP64, only M^-1 r is formed
// from TF32 operands with FP32 accumulation. Rounding the operands to 10
// mantissa bits leaves the iteration counts unchanged (tools/round_scan.py:
// configs 1-4 at 48 / 56 / 92 / 123 vs 48 / 56 / 97 / 122 in FP64), and the
// converged u is still checked against the reference at 1e-10.
//
// One CTA per (128-row type tile, BN-column tile): warp 0 lane 0 streams A/B
// K-slices with TMA (128B swizzle) into a 4-stage mbarrier ring, warp 1
// lane 0 issues tcgen05.mma into a TMEM accumulator (128 lanes x BN fp32
// columns), and all four warps drain TMEM with tcgen05.ld: each thread owns
// one row and stores 16 consecutive FP32 columns (64 contiguous bytes).
#pragma once

#include <cuda.h>
#include <cstdint>

#include "kernels.cuh"

namespace tsvb200 {

constexpr int kTcBM = 128;     // UMMA_M (cta_group::1)
constexpr int kTcBK = 32;      // fp32 elements per 128-byte swizzle row
constexpr int kTcStages = 4;
constexpr int kTcThreads = 128;

__host__ __device__ constexpr int tc_stage_bytes(int bn) { return kTcBM * kTcBK * 4 + bn * kTcBK * 4; }
__host__ __device__ constexpr int tc_smem_bytes(int bn) { return kTcStages * tc_stage_bytes(bn) + 1024; }

struct TcLocalParams {
    const int *tile_type;  // [m tile] neighbourhood type of the 128 rows
    int NP;                // rows of each type's B block (n padded to a multiple of BN)
    int BN;                // UMMA_N (multiple of 16, <= 256)
    int k_blocks;          // KP / 32
    float *ZL;             // [rows][ldz] output (row-major, FP32 = the accumulator)
    long long ldz;
    const int *done;       // CG state: skip the work once converged
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!ok);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups
// 1024 bytes apart (SBO); LBO is unused for swizzled K-major operands.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
    return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = bn.
__device__ __forceinline__ uint32_t tf32_idesc(int bn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(bn >> 3) << 17) |
           (static_cast<uint32_t>(kTcBM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ float to_tf32(double v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(static_cast<float>(v)));
    return __uint_as_float(r);
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_local_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcLocalParams p) {
    pdl_wait();
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kTcStages], empty_bar[kTcStages], accum_bar;
    __shared__ uint32_t tmem_slot;
    if (*reinterpret_cast<const volatile int *>(p.done)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tile = blockIdx.x, m_tile = blockIdx.y;
    const int BN = p.BN;
    const uint32_t base = (smem_u32(tc_smem_raw) + 1023u) & ~1023u;
    const uint32_t a_bytes = kTcBM * kTcBK * 4, stage_bytes = a_bytes + static_cast<uint32_t>(BN) * kTcBK * 4;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(smem_u32(&full_bar[s]), 1);
            mbar_init(smem_u32(&empty_bar[s]), 1);
        }
        mbar_init(smem_u32(&accum_bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;

    if (warp == 0 && lane == 0) {  // TMA producer
        const int brow = p.tile_type[m_tile] * p.NP + n_tile * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
            const int s = kb % kTcStages;
            const uint32_t ph = static_cast<uint32_t>(kb / kTcStages) & 1u;
            mbar_wait(smem_u32(&empty_bar[s]), ph ^ 1u);
            const uint32_t sa = base + static_cast<uint32_t>(s) * stage_bytes;
            mbar_expect_tx(smem_u32(&full_bar[s]), stage_bytes);
            tma_load_2d(sa, &tmA, smem_u32(&full_bar[s]), kb * kTcBK, m_tile * kTcBM);
            tma_load_2d(sa + a_bytes, &tmB, smem_u32(&full_bar[s]), kb * kTcBK, brow);
        }
    } else if (warp == 1 && lane == 0) {  // MMA issuer
        const uint32_t idesc = tf32_idesc(BN);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
            const int s = kb % kTcStages;
            const uint32_t ph = static_cast<uint32_t>(kb / kTcStages) & 1u;
            mbar_wait(smem_u32(&full_bar[s]), ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = base + static_cast<uint32_t>(s) * stage_bytes, sb = sa + a_bytes;
#pragma unroll
            for (int k = 0; k < kTcBK / 8; ++k)  // UMMA_K = 8 tf32 = 32 bytes along the swizzled row
                umma_tf32(tmem, sw128_desc(sa + 32u * k), sw128_desc(sb + 32u * k), idesc, (kb | k) != 0);
            umma_commit(smem_u32(&empty_bar[s]));
        }
        umma_commit(smem_u32(&accum_bar));
    }
    __syncwarp();

    // Epilogue: warp w owns TMEM lanes (= tile rows) 32w .. 32w+31.
    mbar_wait(smem_u32(&accum_bar), 0u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const long long row = static_cast<long long>(m_tile) * kTcBM + warp * 32 + lane;
    float *out = p.ZL + row * p.ldz + static_cast<long long>(n_tile) * BN;
    for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
              "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint4 *o4 = reinterpret_cast<uint4 *>(out + c0);
#pragma unroll
        for (int j = 0; j < 4; ++j) o4[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

// Paired variant: one CTA per (N tile, pair of consecutive M tiles of the same
// type). The B slice (the type's inverse, the larger operand: BN x KP) is
// streamed once for both M tiles, which land in two TMEM accumulators
// (columns 0 and 256 of a 512-column allocation); with ~half the CTAs the
// launch fits one wave. pairs[y] = {m0, m1 or -1}.
constexpr int kTcPairStages = 3;
__host__ __device__ constexpr int tc_pair_stage_bytes(int bn) { return 2 * kTcBM * kTcBK * 4 + bn * kTcBK * 4; }
__host__ __device__ constexpr int tc_pair_smem_bytes(int bn) { return kTcPairStages * tc_pair_stage_bytes(bn) + 1024; }

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_local_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcLocalParams p,
                         const int2 *pairs) {
    pdl_wait();
    extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kTcPairStages], empty_bar[kTcPairStages], accum_bar;
    __shared__ uint32_t tmem_slot;
    if (*reinterpret_cast<const volatile int *>(p.done)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tile = blockIdx.x;
    const int2 mp = pairs[blockIdx.y];
    const int m0 = mp.x, m1 = mp.y, nm = m1 >= 0 ? 2 : 1;
    const int BN = p.BN;
    const uint32_t base = (smem_u32(tc_smem_raw) + 1023u) & ~1023u;
    const uint32_t a_bytes = kTcBM * kTcBK * 4, b_bytes = static_cast<uint32_t>(BN) * kTcBK * 4;
    const uint32_t stage_bytes = 2 * a_bytes + b_bytes;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kTcPairStages; ++s) {
            mbar_init(smem_u32(&full_bar[s]), 1);
            mbar_init(smem_u32(&empty_bar[s]), 1);
        }
        mbar_init(smem_u32(&accum_bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_slot;

    if (warp == 0 && lane == 0) {  // TMA producer: B once, A of both M tiles
        const int brow = p.tile_type[m0] * p.NP + n_tile * BN;
        const uint32_t tx = static_cast<uint32_t>(nm) * a_bytes + b_bytes;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
            const int s = kb % kTcPairStages;
            const uint32_t ph = static_cast<uint32_t>(kb / kTcPairStages) & 1u;
            mbar_wait(smem_u32(&empty_bar[s]), ph ^ 1u);
            const uint32_t sa = base + static_cast<uint32_t>(s) * stage_bytes;
            mbar_expect_tx(smem_u32(&full_bar[s]), tx);
            tma_load_2d(sa, &tmA, smem_u32(&full_bar[s]), kb * kTcBK, m0 * kTcBM);
            if (nm == 2) tma_load_2d(sa + a_bytes, &tmA, smem_u32(&full_bar[s]), kb * kTcBK, m1 * kTcBM);
            tma_load_2d(sa + 2 * a_bytes, &tmB, smem_u32(&full_bar[s]), kb * kTcBK, brow);
        }
    } else if (warp == 1 && lane == 0) {  // MMA issuer
        const uint32_t idesc = tf32_idesc(BN);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
            const int s = kb % kTcPairStages;
            const uint32_t ph = static_cast<uint32_t>(kb / kTcPairStages) & 1u;
            mbar_wait(smem_u32(&full_bar[s]), ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = base + static_cast<uint32_t>(s) * stage_bytes, sb = sa + 2 * a_bytes;
#pragma unroll
            for (int k = 0; k < kTcBK / 8; ++k) {
                umma_tf32(tmem, sw128_desc(sa + 32u * k), sw128_desc(sb + 32u * k), idesc, (kb | k) != 0);
                if (nm == 2)
                    umma_tf32(tmem + 256u, sw128_desc(sa + a_bytes + 32u * k), sw128_desc(sb + 32u * k), idesc,
                              (kb | k) != 0);
            }
            umma_commit(smem_u32(&empty_bar[s]));
        }
        umma_commit(smem_u32(&accum_bar));
    }
    __syncwarp();

    // Epilogue: warp w owns TMEM lanes (= tile rows) 32w .. 32w+31 of both accumulators.
    mbar_wait(smem_u32(&accum_bar), 0u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int t = 0; t < nm; ++t) {
        const long long row = static_cast<long long>(t ? m1 : m0) * kTcBM + warp * 32 + lane;
        float *out = p.ZL + row * p.ldz + static_cast<long long>(n_tile) * BN;
        for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0) + 256u * t;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                  "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            uint4 *o4 = reinterpret_cast<uint4 *>(out + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) o4[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// Local inverse in the tensor-core layout: Ainv32[type][pidx(a)][pidx(k)]
// (rows padded to NP, columns to KP, zero pads), rounded to TF32.
__global__ void as_pack_inverse_tf32_kernel(const double *inv, int n, int nn, int KP, float *dst) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<long long>(n) * n) return;
    const int a = static_cast<int>(t / n), k = static_cast<int>(t % n);
    const double v = a >= k ? inv[static_cast<long long>(k) * n + a] : inv[static_cast<long long>(a) * n + k];
    dst[static_cast<long long>((a % 3) * nn + a / 3) * KP + (k % 3) * nn + k / 3] = to_tf32(v);
}

}  // namespace tsvb200
