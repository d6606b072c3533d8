// K1 (Y = X K^T, FP64) on the int8 tensor cores: Ozaki splitting with exact
// int32 accumulation (tcgen05.mma kind::i8).
//
// Every row of X (one block's p or x) and every row of K_r is scaled by a
// power of two and cut into S signed 7-bit digits (|d| <= 64):
//
//   X[r][k] = 2^(ex_r - 7) sum_t a_t[r][k] 2^(-7t)      (t = 0 .. S-1)
//   K[j][k] = 2^(ek_j - 7) sum_u b_u[j][k] 2^(-7u)
//
// so  Y[r][j] = 2^(ex_r + ek_j - 14) sum_d 2^(-7d) C_d[r][j],
//     C_d = sum_{t+u=d} A_t B_u^T   (int32, exact: |C_d| <= S * 4096 * k < 2^31)
//
// keeping the S(S+1)/2 digit pairs with t + u < S. The digit split is exact
// in FP64 (power-of-two scaling, rint, exact remainders), the int8 products
// and their int32 sums are exact, and the epilogue combines the S diagonal
// sums in FP64 (Horner from the smallest weight). The only approximation is
// the dropped tail, below 2^(-7S) of max|X_r| max|K_j| per term (S = 9 or 10).
//
// Persistent CTAs over (128-row tile, 48-column tile)s: warp 0 lane 0 streams the S A
// digit planes and S B digit planes of a 64-byte K slice with TMA (64B
// swizzle) into a 2-stage mbarrier ring; warp 1 issues, per A plane t, one
// tcgen05.mma against up to five consecutive B planes (N <= 240), whose
// column blocks land on the diagonal accumulators t + u (S x 48 int32 TMEM
// columns); the four warps then drain TMEM, combine in FP64 and write Y
// through shared memory. Few wide MMAs matter: an MMA costs ~40 cycles
// below N = 64 and N/2 cycles above (tools/umma_bench.cu on B200).
#pragma once

#include <cuda.h>
#include <cstdint>

#include "kernels.cuh"
#include "tc_local.cuh"

namespace tsvb200 {

constexpr int kOzBK = 64;  // bytes (= int8 k values) per slice, one 64B swizzle row
constexpr int kOzStages = 2;
constexpr int kOzMaxPlanes = 5;  // B planes per MMA: N = 5 x 48 = 240 <= 256

// TMEM: S accumulators (diagonals) of BN int32 columns.
template <int S>
struct OzCfg {
    static_assert(S == 9 || S == 10, "digit counts 9 / 10");
    static constexpr int BN = 48;
};

template <int S>
__host__ __device__ constexpr int oz_stage_bytes() {
    return S * (kTcBM * kOzBK) + S * (OzCfg<S>::BN * kOzBK);
}
template <int S>
__host__ __device__ constexpr int oz_smem_bytes() {
    return kOzStages * oz_stage_bytes<S>() + 1024;
}

// Digit planes of the rows of an FP64 matrix: planes[t][row][k] (int8, row
// stride KA bytes, plane stride plane_rows * KA), ex[row] the row exponent.
// One warp per row.
template <int S>
__global__ void __launch_bounds__(256) oz_slice_kernel(const double *__restrict__ M, long long ldm, int rows, int ncols,
                                                       int8_t *__restrict__ planes, long long plane_rows, int KA,
                                                       int *__restrict__ ex, const int *done, const int *run_flag) {
    pdl_wait();
    constexpr int kMaxGroups = 8;  // 4 values per lane per group: rows up to 1024 values
    if (done && *reinterpret_cast<const volatile int *>(done)) return;
    if (run_flag && !*reinterpret_cast<const volatile int *>(run_flag)) return;
    const int lane = threadIdx.x & 31;
    for (int row = blockIdx.x * 8 + (threadIdx.x >> 5); row < rows; row += gridDim.x * 8) {
    const double *m = M + static_cast<long long>(row) * ldm;
    double y[kMaxGroups][4];
    double mx = 0.0;
#pragma unroll
    for (int g = 0; g < kMaxGroups; ++g) {
        const int k0 = 4 * lane + 128 * g;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            y[g][j] = k0 + j < ncols ? m[k0 + j] : 0.0;
            mx = fmax(mx, fabs(y[g][j]));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int e = mx == 0.0 ? 0 : ilogb(mx) + 2;  // |x| < 2^(e-1): first digit in [-64, 64]
    if (lane == 0) ex[row] = e;
    const double sc = scalbn(1.0, 7 - e);
#pragma unroll
    for (int g = 0; g < kMaxGroups; ++g) {
        const int k0 = 4 * lane + 128 * g;
        if (k0 >= KA) break;
        double v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = y[g][j] * sc;  // exact (power of two)
        int8_t *dst = planes + static_cast<long long>(row) * KA + k0;
#pragma unroll
        for (int t = 0; t < S; ++t) {
            char4 c;
            double d;
            d = rint(v[0]); c.x = static_cast<signed char>(d); v[0] = (v[0] - d) * 128.0;
            d = rint(v[1]); c.y = static_cast<signed char>(d); v[1] = (v[1] - d) * 128.0;
            d = rint(v[2]); c.z = static_cast<signed char>(d); v[2] = (v[2] - d) * 128.0;
            d = rint(v[3]); c.w = static_cast<signed char>(d); v[3] = (v[3] - d) * 128.0;
            *reinterpret_cast<char4 *>(dst + t * plane_rows * static_cast<long long>(KA)) = c;
        }
    }
    }  // rows (grid-stride: a fixed grid keeps the early exit of a skipped launch cheap)
}

struct OzParams {
    const uint8_t *tile_kind;  // per 128-row tile
    int m_tiles, n_tiles;
    long long a_plane_rows;    // rows per A plane (panel rows)
    long long b_plane_rows;    // rows per B plane (K rows, padded to the N tiles)
    int k_blocks;              // ceil(KA / 64)
    const int *ex_a;           // [panel rows]
    const int *ex_b[2];        // [K rows] per kind
    double *C;
    long long ldc;
    int n_store;
    const int *done;
    const int *run_flag;  // nullable: run only when *run_flag != 0 (hybrid K1: the A x products)
};

// SWIZZLE_64B K-major: 8-row groups 512 bytes apart.
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(512 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
    d |= static_cast<uint64_t>(4) << 61;  // SWIZZLE_64B
    return d;
}

// Instruction descriptor: D s32, A/B signed int8, K-major, M = 128, N = bn.
__host__ __device__ constexpr uint32_t i8_idesc(int bn) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(bn >> 3) << 17) |
           (static_cast<uint32_t>(kTcBM >> 4) << 24);
}

// Issued from a converged warp: elect.sync picks the one lane that issues
// (uniform predicate; no per-instruction divergence loop in SASS).
__device__ __forceinline__ void umma_i8_elect(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}

template <int S>
__global__ void __launch_bounds__(kTcThreads, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                   const __grid_constant__ CUtensorMap tmB1, OzParams p) {
    pdl_wait();
    constexpr int BN = OzCfg<S>::BN;
    constexpr uint32_t A_TILE = kTcBM * kOzBK, B_TILE = BN * kOzBK;
    constexpr uint32_t STAGE = S * A_TILE + S * B_TILE;
    extern __shared__ __align__(1024) unsigned char oz_smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kOzStages], empty_bar[kOzStages], accum_bar;
    __shared__ uint32_t tmem_slot;
    if (p.done && *reinterpret_cast<const volatile int *>(p.done)) return;
    if (p.run_flag && !*reinterpret_cast<const volatile int *>(p.run_flag)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t base = (smem_u32(oz_smem_raw) + 1023u) & ~1023u;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kOzStages; ++s) {
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

    // Persistent: tiles n-minor (neighbouring CTAs share the A rows in L2);
    // the stage/phase counters run on across tiles.
    const int total = p.n_tiles * p.m_tiles;
    int g = 0;  // k-blocks consumed so far by this CTA
    for (int tile = blockIdx.x, it = 0; tile < total; tile += gridDim.x, ++it, g += p.k_blocks) {
        const int n_tile = tile % p.n_tiles, m_tile = tile / p.n_tiles;
        const int kind = p.tile_kind[m_tile];
        if (warp == 0 && lane == 0) {  // TMA producer
            const CUtensorMap *tmB = kind ? &tmB1 : &tmB0;
            for (int kb = 0; kb < p.k_blocks; ++kb) {
                const int s = (g + kb) % kOzStages;
                const uint32_t ph = static_cast<uint32_t>((g + kb) / kOzStages) & 1u;
                mbar_wait(smem_u32(&empty_bar[s]), ph ^ 1u);
                const uint32_t sa = base + static_cast<uint32_t>(s) * STAGE, sb = sa + S * A_TILE;
                const uint32_t bar = smem_u32(&full_bar[s]);
                mbar_expect_tx(bar, STAGE);
#pragma unroll
                for (int t = 0; t < S; ++t)
                    tma_load_2d(sa + t * A_TILE, &tmA, bar, kb * kOzBK, static_cast<int>(t * p.a_plane_rows) + m_tile * kTcBM);
#pragma unroll
                for (int u = 0; u < S; ++u)
                    tma_load_2d(sb + u * B_TILE, tmB, bar, kb * kOzBK, static_cast<int>(u * p.b_plane_rows) + n_tile * BN);
            }
        } else if (warp == 1) {  // MMA issuer: the whole warp runs the loop, one elected lane issues
            // A_t x [B_u0 .. B_u0+np-1]^T as ONE MMA: the B planes are consecutive
            // 48-row blocks in shared memory, so N = np * 48 columns land in TMEM
            // column blocks t+u0 .. t+u0+np-1 = the diagonals d = t + u.
            for (int kb = 0; kb < p.k_blocks; ++kb) {
                const int s = (g + kb) % kOzStages;
                const uint32_t ph = static_cast<uint32_t>((g + kb) / kOzStages) & 1u;
                mbar_wait(smem_u32(&full_bar[s]), ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t sa = base + static_cast<uint32_t>(s) * STAGE, sb = sa + S * A_TILE;
#pragma unroll
                for (int t = 0; t < S; ++t)
#pragma unroll
                    for (int u0 = 0; u0 < S - t; u0 += kOzMaxPlanes) {
                        const int np = (S - t - u0) < kOzMaxPlanes ? (S - t - u0) : kOzMaxPlanes;
#pragma unroll
                        for (int kk = 0; kk < kOzBK / 32; ++kk)  // UMMA_K = 32 int8 = 32 bytes
                            umma_i8_elect(tmem + static_cast<uint32_t>((t + u0) * BN), sw64_desc(sa + t * A_TILE + 32u * kk),
                                          sw64_desc(sb + u0 * B_TILE + 32u * kk), i8_idesc(np * BN), (kb | kk | t) != 0);
                    }
                umma_commit_elect(smem_u32(&empty_bar[s]));
            }
            umma_commit_elect(smem_u32(&accum_bar));
        }
        __syncwarp();

        // Epilogue: warp w owns TMEM lanes (= tile rows) 32w .. 32w+31.
        mbar_wait(smem_u32(&accum_bar), static_cast<uint32_t>(it) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const long long row0 = static_cast<long long>(m_tile) * kTcBM + warp * 32;
        const int ea = p.ex_a[row0 + lane];
        const int *eb = (kind ? p.ex_b[1] : p.ex_b[0]) + n_tile * BN;
        const uint32_t lane_addr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        // the operand stages are idle until the next tile starts: stage this
        // warp's 32 x BN result rows there
        constexpr int SP = BN + 1;
        double *stg = reinterpret_cast<double *>(oz_smem_raw + (base - smem_u32(oz_smem_raw))) + warp * 32 * SP;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 8) {
            double y[8];
#pragma unroll
            for (int d = S - 1; d >= 0; --d) {
                uint32_t v[8];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                             : "r"(lane_addr + static_cast<uint32_t>(d * BN + c0)));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double c = static_cast<double>(static_cast<int>(v[j]));
                    y[j] = d == S - 1 ? c : y[j] * 0.0078125 + c;  // Horner in 2^-7
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // exact power-of-two scale 2^(ea + eb - 14)
                const int e2 = ea + eb[c0 + j] - 14;
                const double f = __longlong_as_double(static_cast<long long>(min(max(e2 + 1023, 1), 2046)) << 52);
                stg[lane * SP + c0 + j] = y[j] * f;
            }
        }
        __syncwarp();
        const int col0 = n_tile * BN;
        for (int r = 0; r < 32; ++r) {
            double *out = p.C + (row0 + r) * p.ldc + col0;
            for (int c = lane; c < BN; c += 32)
                if (col0 + c < p.n_store) out[c] = stg[r * SP + c];
        }
        // TMEM drained and the staging area free before the next tile
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace tsvb200
