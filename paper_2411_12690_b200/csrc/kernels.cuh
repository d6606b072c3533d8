// sm_100a kernels of the online stage.
//
//   gemm_nt_f64      K1 operator apply  Y = X K_r        (blocks x n x n, DMMA)
//                    K6 block recovery  U = Q Phi^T + dT u_T^T (blocks x n_fine x n)
//   cg_gather_*      K1 scatter half + K2/K5: owner-computes sum of the
//                    per-block products, PCG vector updates, fused dots
//   cg_scatter_*     K1 gather half: write the next operand into the
//                    block-major X panel (one slot per (block, local DoF))
//   stress_gauss     K7 Gauss-point / centroid stress + von Mises
//
// FP64 tensor-core work on sm_100a is warp-level mma.sync m8n8k4 (SASS
// DMMA.8x8x4); tcgen05 has no kind::f64.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tsvb200 {

// ------------------------------------------------------------------ GEMM
// C[m][n] = sum_k A[m][k] * Bt[n][k]  (+ row_scale[m] * col_bias[n]).
// A: block-major operand panel, rows = blocks (GEMM row order), k contiguous.
// Bt: K_r (symmetric, so K_r^T = K_r) or Phi (row-major [fine dof][k]).
// Programmatic dependent launch: kernels of the PCG iteration are launched
// with cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs
// are scheduled while its predecessor drains; griddepcontrol.wait holds them
// until the predecessor's results are visible (a no-op for a normal launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the dependent grid launch once every CTA of this one got here (its CTAs
// then wait in pdl_wait until this grid's memory is visible).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct GemmParams {
    const double *A;
    long long lda;
    const double *Bt[2];  // per block kind
    long long ldb;
    const uint8_t *tile_kind;  // per M tile
    const double *const *Bt_tab;  // nullable: per-tile matrix table indexed by tile_type
    const int *tile_type;         // per M tile (with Bt_tab)
    double *C;
    long long ldc;
    int m_tiles, n_tiles, k_chunks;
    int n_valid;  // columns with data; fragments beyond are skipped
    int n_store;  // columns written
    const double *row_scale;     // nullable: dT per row (K6 epilogue)
    const double *col_bias[2];   // u_T per kind
    const int *done;             // nullable: early exit when *done != 0
    const int *skip_flag;        // nullable: early exit when *skip_flag != 0 (hybrid K1: A x goes to int8)
    const int *run_flag;         // nullable: early exit when *run_flag == 0 (the A x products of a symmetric K1)
    unsigned *tile_counter;      // [2] {next tile, exited CTAs}, zero between launches
    int n_major;                 // tile order: 0 = M major (K1: A streamed once, K_r in L2),
                                 // 1 = N major (K6: Phi streamed once, the Q chunk in L2)
    const int *col_map;          // nullable: output column of GEMM column (K6: dense fine DoF rows)
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int BM_, int BN_, int WM_, int WN_, int KC_, int STAGES_, int MINB_ = 2>
struct GemmCfg {
    static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, KC = KC_, STAGES = STAGES_, MINB = MINB_;
    static constexpr int THREADS = WM * WN * 32;
    static constexpr int TM = BM / WM, TN = BN / WN, FM = TM / 8, FN = TN / 8;
    // Row pitch KC+4 doubles: 8-byte fragment loads of a half-warp (4 rows x
    // 4 k) hit 16 distinct 8-byte bank pairs (pitch mod 16 == 4).
    static constexpr int SP = KC + 4;
    static constexpr int A_STAGE = BM * SP, B_STAGE = BN * SP;
    static constexpr size_t SMEM = size_t(STAGES) * (A_STAGE + B_STAGE) * sizeof(double);
    static_assert(TM % 8 == 0 && TN % 8 == 0 && KC % 4 == 0, "tile shape");
};

template <class Cfg>
__device__ __forceinline__ void gemm_load_stage(double *As, double *Bs, const double *A0, long long lda,
                                                const double *B0, long long ldb, int kc) {
    constexpr int CPR = Cfg::KC / 2;  // 16-byte chunks per row
    const int tid = threadIdx.x;
    const long long k0 = static_cast<long long>(kc) * Cfg::KC;
#pragma unroll
    for (int i = tid; i < Cfg::BM * CPR; i += Cfg::THREADS) {
        const int r = i / CPR, c = i % CPR;
        cp_async16(As + r * Cfg::SP + 2 * c, A0 + r * lda + k0 + 2 * c);
    }
#pragma unroll
    for (int i = tid; i < Cfg::BN * CPR; i += Cfg::THREADS) {
        const int r = i / CPR, c = i % CPR;
        cp_async16(Bs + r * Cfg::SP + 2 * c, B0 + r * ldb + k0 + 2 * c);
    }
}

// One KC-deep chunk of warp-tile DMMAs from shared memory; NJ n-fragments.
template <class Cfg, int NJ>
__device__ __forceinline__ void mma_chunk(double (&acc)[Cfg::FM][Cfg::FN][2], const double *as, const double *bs) {
#pragma unroll
    for (int ks = 0; ks < Cfg::KC / 4; ++ks) {
        double af[Cfg::FM], bf[NJ];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = as[i * 8 * Cfg::SP + ks * 4];
#pragma unroll
        for (int j = 0; j < NJ; ++j) bf[j] = bs[j * 8 * Cfg::SP + ks * 4];
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
}

template <class Cfg>
__device__ __forceinline__ void mma_chunk_partial(double (&acc)[Cfg::FM][Cfg::FN][2], const double *as, const double *bs,
                                               int fn_lim) {
    for (int ks = 0; ks < Cfg::KC / 4; ++ks) {
        double af[Cfg::FM];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = as[i * 8 * Cfg::SP + ks * 4];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
            if (j < fn_lim) {
                const double bf = bs[j * 8 * Cfg::SP + ks * 4];
#pragma unroll
                for (int i = 0; i < Cfg::FM; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf);
            }
        }
    }
}

// Accumulate k-chunks [kc0, kc1) of one tile: A0 / B0 point at the tile's
// first row (k = 0) of the operand panel / the matrix.
template <class Cfg>
__device__ __forceinline__ void gemm_core(double *As, double *Bs, const double *A0, long long lda, const double *B0,
                                          long long ldb, int kc0, int kc1, int fn_lim,
                                          double (&acc)[Cfg::FM][Cfg::FN][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / Cfg::WN, wn = warp % Cfg::WN;
#pragma unroll
    for (int s = 0; s < Cfg::STAGES - 1; ++s) {
        if (kc0 + s < kc1)
            gemm_load_stage<Cfg>(As + s * Cfg::A_STAGE, Bs + s * Cfg::B_STAGE, A0, lda, B0, ldb, kc0 + s);
        cp_async_commit();
    }
    for (int kc = kc0; kc < kc1; ++kc) {
        const int i = kc - kc0;
        cp_async_wait<Cfg::STAGES - 2>();
        __syncthreads();
        const int nk = kc + Cfg::STAGES - 1;
        if (nk < kc1) {
            const int st = (i + Cfg::STAGES - 1) % Cfg::STAGES;
            gemm_load_stage<Cfg>(As + st * Cfg::A_STAGE, Bs + st * Cfg::B_STAGE, A0, lda, B0, ldb, nk);
        }
        cp_async_commit();
        const double *as = As + (i % Cfg::STAGES) * Cfg::A_STAGE + (wm * Cfg::TM + (lane >> 2)) * Cfg::SP + (lane & 3);
        const double *bs = Bs + (i % Cfg::STAGES) * Cfg::B_STAGE + (wn * Cfg::TN + (lane >> 2)) * Cfg::SP + (lane & 3);
        if (fn_lim == Cfg::FN)
            mma_chunk<Cfg, Cfg::FN>(acc, as, bs);
        else if (fn_lim > 0)
            mma_chunk_partial<Cfg>(acc, as, bs, fn_lim);
    }
    cp_async_wait<0>();
    __syncthreads();
}

// One tile segment: accumulate k-chunks [kc0, kc1) of tile (mt, nt).
template <class Cfg>
__device__ __forceinline__ void gemm_segment(const GemmParams &p, double *As, double *Bs, int mt, int nt, int kc0,
                                             int kc1, int fn_lim, double (&acc)[Cfg::FM][Cfg::FN][2]) {
    const int kind = p.tile_kind ? p.tile_kind[mt] : 0;
    const double *A0 = p.A + static_cast<long long>(mt) * Cfg::BM * p.lda;
    const double *Bbase = p.Bt_tab ? p.Bt_tab[p.tile_type[mt]] : (kind ? p.Bt[1] : p.Bt[0]);
    const double *B0 = Bbase + static_cast<long long>(nt) * Cfg::BN * p.ldb;
    gemm_core<Cfg>(As, Bs, A0, p.lda, B0, p.ldb, kc0, kc1, fn_lim, acc);
}

// Epilogue: lane holds C[row][col], C[row][col+1] (+ row_scale * col_bias).
template <class Cfg>
__device__ __forceinline__ void gemm_epilogue(const GemmParams &p, int mt, int nt,
                                              const double (&acc)[Cfg::FM][Cfg::FN][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / Cfg::WN, wn = warp % Cfg::WN;
    const int kind = p.tile_kind ? p.tile_kind[mt] : 0;
    const long long row0 = static_cast<long long>(mt) * Cfg::BM + wm * Cfg::TM + (lane >> 2);
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) {
        const int col = nt * Cfg::BN + wn * Cfg::TN + j * 8 + 2 * (lane & 3);
        if (col >= p.n_store) continue;
        double b0 = 0.0, b1 = 0.0;
        const double *cb = kind ? p.col_bias[1] : p.col_bias[0];
        if (p.row_scale) {
            b0 = cb[col];
            b1 = col + 1 < p.n_store ? cb[col + 1] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) {
            const long long row = row0 + i * 8;
            double v0 = acc[i][j][0], v1 = acc[i][j][1];
            if (p.row_scale) {
                const double s = p.row_scale[row];
                v0 += s * b0;
                v1 += s * b1;
            }
            if (p.col_map) {
                double *rowp = p.C + row * p.ldc;
                rowp[p.col_map[col]] = v0;
                if (col + 1 < p.n_store) rowp[p.col_map[col + 1]] = v1;
                continue;
            }
            double *dst = p.C + row * p.ldc + col;
            if (col + 1 < p.n_store) {
                *reinterpret_cast<double2 *>(dst) = make_double2(v0, v1);
            } else {
                dst[0] = v0;
            }
        }
    }
}

template <class Cfg>
__device__ __forceinline__ int gemm_fn_lim(const GemmParams &p, int nt) {
    const int wn = (threadIdx.x >> 5) % Cfg::WN;
    const int frag0 = nt * (Cfg::BN / 8) + wn * Cfg::FN;
    return min(Cfg::FN, max(0, (p.n_valid + 7) / 8 - frag0));
}

// Persistent DMMA GEMM: grid = resident CTAs, tiles handed out by an atomic
// counter (M tile major, N tile minor, so concurrently running CTAs share
// the streamed A panel in L2).
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) gemm_nt_f64(GemmParams p) {
    pdl_wait();
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_tile;
    double *As = smem;
    double *Bs = smem + Cfg::STAGES * Cfg::A_STAGE;
    const int tid = threadIdx.x;
    const int total = p.m_tiles * p.n_tiles;
    const bool skip = (p.done != nullptr && *reinterpret_cast<const volatile int *>(p.done) != 0) ||
                      (p.skip_flag != nullptr && *reinterpret_cast<const volatile int *>(p.skip_flag) != 0) ||
                      (p.run_flag != nullptr && *reinterpret_cast<const volatile int *>(p.run_flag) == 0);

    while (!skip) {
        if (tid == 0) s_tile = static_cast<int>(atomicAdd(&p.tile_counter[0], 1u));
        __syncthreads();
        const int tile = s_tile;
        __syncthreads();
        if (tile >= total) break;
        const int mt = p.n_major ? tile % p.m_tiles : tile / p.n_tiles;
        const int nt = p.n_major ? tile / p.m_tiles : tile % p.n_tiles;
        double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        gemm_segment<Cfg>(p, As, Bs, mt, nt, 0, p.k_chunks, gemm_fn_lim<Cfg>(p, nt), acc);
        gemm_epilogue<Cfg>(p, mt, nt, acc);
    }
    pdl_trigger();
    // The last CTA out resets the tile counter for the next launch.
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&p.tile_counter[1], 1u) == gridDim.x - 1) {
            p.tile_counter[0] = 0u;
            p.tile_counter[1] = 0u;
            __threadfence();
        }
    }
}

// Split-K DMMA GEMM for arrays with fewer tiles than SM slots (configs
// 0-2: 5-128 tiles of 64 x 64): CTA (tile, s) accumulates the k-chunks
// [s kc / S, (s+1) kc / S), parks its accumulators in work (thread-major,
// coalesced) and takes a per-tile ticket; the last of the S CTAs sums the
// S partials in s order (fixed: bitwise reproducible) and runs the epilogue.
struct SplitK {
    double *work;      // [tiles * S][FM*FN*2][THREADS]
    unsigned *ticket;  // [tiles], zero between launches
    int S;
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) gemm_splitk_f64(GemmParams p, SplitK sk) {
    pdl_wait();
    extern __shared__ __align__(16) double smem[];
    __shared__ bool last;
    double *As = smem;
    double *Bs = smem + Cfg::STAGES * Cfg::A_STAGE;
    constexpr int NACC = Cfg::FM * Cfg::FN * 2;
    const int tid = threadIdx.x;
    if ((p.done != nullptr && *reinterpret_cast<const volatile int *>(p.done) != 0) ||
        (p.skip_flag != nullptr && *reinterpret_cast<const volatile int *>(p.skip_flag) != 0) ||
        (p.run_flag != nullptr && *reinterpret_cast<const volatile int *>(p.run_flag) == 0))
        return;
    const int S = sk.S;
    const int tile = blockIdx.x / S, s = blockIdx.x % S;
    const int mt = tile / p.n_tiles, nt = tile % p.n_tiles;
    const int kc0 = (p.k_chunks * s) / S, kc1 = (p.k_chunks * (s + 1)) / S;
    double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    gemm_segment<Cfg>(p, As, Bs, mt, nt, kc0, kc1, gemm_fn_lim<Cfg>(p, nt), acc);
    double *w = sk.work + static_cast<long long>(blockIdx.x) * NACC * Cfg::THREADS;
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) w[((i * Cfg::FN + j) * 2 + h) * Cfg::THREADS + tid] = acc[i][j][h];
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(&sk.ticket[tile], 1u) == static_cast<unsigned>(S - 1);
    __syncthreads();
    pdl_trigger();
    if (!last) return;
    __threadfence();
    const double *w0 = sk.work + static_cast<long long>(tile) * S * NACC * Cfg::THREADS + tid;
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // s outer, all NACC loads of one partial in flight together
    for (int s2 = 0; s2 < S; ++s2) {
        const double *ws = w0 + static_cast<long long>(s2) * NACC * Cfg::THREADS;
        double v[NACC];
#pragma unroll
        for (int e = 0; e < NACC; ++e) v[e] = __ldcg(ws + e * Cfg::THREADS);
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) acc[i][j][h] += v[(i * Cfg::FN + j) * 2 + h];
    }
    gemm_epilogue<Cfg>(p, mt, nt, acc);
    if (tid == 0) sk.ticket[tile] = 0u;
}

// Stream-K DMMA GEMM: CTA g owns the linear (tile, k-chunk) iterations
// [start[g], start[g+1]) (host-balanced by DMMA work), so every SM finishes
// together instead of idling through a partial last wave. A tile split
// between CTAs g and g+1 is completed by g (its k-chunks start at 0): g+1
// computes the tail segment first, parks the partial accumulators in
// work[g] and raises flag[g]; g adds them after its own segment, in that
// fixed order, so results are bitwise reproducible. Requires every tile to
// span at most two CTAs (host checks >= 2 tiles of work per CTA) and all
// CTAs resident (grid = occupancy x SMs).
struct StreamK {
    const int *start;   // [grid + 1] linear iteration boundaries
    double *work;       // [grid][FM*FN*2][THREADS]
    int *flag;          // [grid], zero between launches
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) gemm_streamk_f64(GemmParams p, StreamK sk) {
    pdl_wait();
    extern __shared__ __align__(16) double smem[];
    double *As = smem;
    double *Bs = smem + Cfg::STAGES * Cfg::A_STAGE;
    constexpr int NACC = Cfg::FM * Cfg::FN * 2;
    const int tid = threadIdx.x, g = blockIdx.x;
    if (p.done != nullptr && *reinterpret_cast<const volatile int *>(p.done) != 0) return;
    if ((p.skip_flag != nullptr && *reinterpret_cast<const volatile int *>(p.skip_flag) != 0) ||
        (p.run_flag != nullptr && *reinterpret_cast<const volatile int *>(p.run_flag) == 0))
        return;
    const int KC = p.k_chunks;
    const int i0 = sk.start[g], i1 = sk.start[g + 1];
    int it = i0;
    while (it < i1) {
        const int tile = it / KC, kc0 = it % KC;
        const int kc1 = min(KC, kc0 + (i1 - it));
        const int mt = tile / p.n_tiles, nt = tile % p.n_tiles;
        double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        gemm_segment<Cfg>(p, As, Bs, mt, nt, kc0, kc1, gemm_fn_lim<Cfg>(p, nt), acc);
        if (kc0 > 0) {
            // tail of a tile owned by CTA g-1: park the partial, raise the flag
            double *w = sk.work + static_cast<long long>(g - 1) * NACC * Cfg::THREADS + tid;
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::FN; ++j) {
                    w[((i * Cfg::FN + j) * 2 + 0) * Cfg::THREADS] = acc[i][j][0];
                    w[((i * Cfg::FN + j) * 2 + 1) * Cfg::THREADS] = acc[i][j][1];
                }
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicExch(&sk.flag[g - 1], 1);
        } else {
            if (kc1 < KC) {
                // head of a split tile: wait for CTA g+1's tail partial
                if (tid == 0)
                    while (atomicAdd(&sk.flag[g], 0) == 0) __nanosleep(64);
                __syncthreads();
                __threadfence();
                const double *w = sk.work + static_cast<long long>(g) * NACC * Cfg::THREADS + tid;
#pragma unroll
                for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
                    for (int j = 0; j < Cfg::FN; ++j) {
                        acc[i][j][0] += __ldcg(w + ((i * Cfg::FN + j) * 2 + 0) * Cfg::THREADS);
                        acc[i][j][1] += __ldcg(w + ((i * Cfg::FN + j) * 2 + 1) * Cfg::THREADS);
                    }
                __syncthreads();
                if (tid == 0) sk.flag[g] = 0;  // ready for the next launch
            }
            gemm_epilogue<Cfg>(p, mt, nt, acc);
        }
        it += kc1 - kc0;
    }
}

// ------------------------------------------------------------------- CG
// Iteration state on the device (cg_solve control flow, linalg.cpp:292-362).
enum : int { CG_RUNNING = 0, CG_CONVERGED = 1, CG_NOCONV = 2, CG_BREAKDOWN = 3 };
enum : int { PH_INIT = 0, PH_NORMAL = 1, PH_RESTART = 2, PH_REPLACE = 3 };  // REPLACE: r := b - A x, p kept (Schwarz loop)

struct CgState {
    int done;       // CG_*
    int y_holds_x;  // 1: the next product is A x (true-residual verification)
    int phase;      // what the B kernel does this iteration
    int p_assign;   // 1: p = z (fresh start), 0: p = z + beta p
    int fresh;      // split Schwarz loop: the next p is z (after init / restart)
    int it, best_it, max_it, breakdown_code, restarts;
    double rho, alpha, beta, res, best_res, norm_b, tol, tol_abs;
    double rz_l, rz_c;  // Schwarz: r.z split into the local part and (P^T r).zc
    double verify_margin;  // Schwarz: the recursive residual asks for the A x check at <= margin * tol |b| (0: 1)
    // Schwarz loop: one residual replacement (r := b - A x, search direction kept) when the
    // recursive residual first drops below replace_at |b| (0: never)
    double replace_at;
    int replacing, replaced;
    unsigned ticket_a, ticket_b, ticket_c;  // c: side-stream kernels
    unsigned bar_gen;                       // software grid barrier generation (fused kernels)
};

// Device vectors are structure-of-arrays per component: DoF (node, c) of
// the internal node order lives at c * n_nodes + node. Block panels (X, Y)
// are component-major within a row: local DoF (rank, c) at c * nn + rank,
// with K_r / Phi permuted to match at upload. slots[node] holds the row
// offsets row * ldk + rank of the node's 1, 2 or 4 block copies.
struct CgParams {
    CgState *st;
    int n_nodes;
    int nn;             // surface nodes per block (panel component stride)
    const int *slots;   // [node][4] panel offsets (-1 = none), ascending block order
    const uint8_t *cmask;  // [3][node] constrained
    const double *b;
    double *x, *r, *p, *ap;
    float *xlo;         // nullable (Schwarz loop): low part of the compensated x = x + xlo (a few ulps of x: FP32 holds it)
    const double *Y;    // block products
    double *X;          // block-major operand panel
    int precond;        // 0 none, 1 diagonal, 2 3x3 node blocks
    const double *pre;  // inv_diag [3][node] or inverse node blocks [9][node]
    double *partial;    // [grid][2]
    const double *zbuf; // precond 3 (two-level Schwarz): z = M r computed by as_z_kernel
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block reduction of up to two values (fixed tree order).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *sh /* [32*NV] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) sh[warp * NV + i] = v[i];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double t = lane < nw ? sh[lane * NV + i] : 0.0;
            v[i] = warp_sum(t);
        }
    }
}

// Sum of per-CTA partials (CTA order, fixed strides and tree): every thread
// of the last CTA takes a strided subset, then a block tree. Deterministic
// for a fixed grid; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void grid_sum(const double *partial, int nblocks, double (&out)[NV], double *sh) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double s = 0.0;
        for (int k = threadIdx.x; k < nblocks; k += blockDim.x) s += partial[k * NV + i];
        out[i] = s;
    }
    block_sum<NV>(out, sh);
}

__device__ __forceinline__ void precond_node(int kind, const double *pre, int node, int n_nodes, const double r[3],
                                             double z[3]) {
    if (kind == 1) {
#pragma unroll
        for (int c = 0; c < 3; ++c) z[c] = pre[c * n_nodes + node] * r[c];
    } else if (kind == 2) {
        double m[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) m[k] = pre[static_cast<long long>(k) * n_nodes + node];
        z[0] = m[0] * r[0] + m[1] * r[1] + m[2] * r[2];
        z[1] = m[3] * r[0] + m[4] * r[1] + m[5] * r[2];
        z[2] = m[6] * r[0] + m[7] * r[1] + m[8] * r[2];
    } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) z[c] = r[c];
    }
}

// Publish this CTA's partials; returns true in every thread of the last CTA.
template <int NV>
__device__ __forceinline__ bool publish_partials(const double (&v)[NV], double *partial, unsigned *ticket) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) partial[blockIdx.x * NV + i] = v[i];
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// A: Y (= A p or A x) summed per owned DoF; p'Ap or the true residual.
// Grid-stride over nodes with a fixed grid (deterministic reduction).
// Node loop of the gather (A): Ap = sum over the node's block copies of Y
// (unit rows on constrained DoFs), p.Ap; or, verifying, r = b - A x, r.r.
__device__ __forceinline__ double cg_gather_nodes(const CgParams &q, int yx) {
    const int N = q.n_nodes;
    double part = 0.0;
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
        const int4 s = reinterpret_cast<const int4 *>(q.slots)[node];
        if (!yx) {
            // the hot path with the loads of all three components ahead of the stores (the compiler cannot
            // hoist them itself: the vectors may alias as far as it knows); same sums in the same order
            double y[3][4], pv[3];
            uint8_t cm[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const long long dof = static_cast<long long>(c) * N + node;
                const int co = c * q.nn;
                cm[c] = q.cmask[dof];
                pv[c] = q.p[dof];
                y[c][0] = s.x >= 0 ? q.Y[s.x + co] : 0.0;
                y[c][1] = s.y >= 0 ? q.Y[s.y + co] : 0.0;
                y[c][2] = s.z >= 0 ? q.Y[s.z + co] : 0.0;
                y[c][3] = s.w >= 0 ? q.Y[s.w + co] : 0.0;
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const long long dof = static_cast<long long>(c) * N + node;
                const double acc = cm[c] ? pv[c] : (((0.0 + y[c][0]) + y[c][1]) + y[c][2]) + y[c][3];
                q.ap[dof] = acc;
                part += pv[c] * acc;
            }
            continue;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            const int co = c * q.nn;
            double acc;
            if (q.cmask[dof]) {
                acc = yx ? q.x[dof] : q.p[dof];  // unit row of the lifted matrix
            } else {
                acc = 0.0;
                if (s.x >= 0) acc += q.Y[s.x + co];
                if (s.y >= 0) acc += q.Y[s.y + co];
                if (s.z >= 0) acc += q.Y[s.z + co];
                if (s.w >= 0) acc += q.Y[s.w + co];
            }
            if (!yx) {
                q.ap[dof] = acc;
                part += q.p[dof] * acc;
            } else {
                const double rt = q.b[dof] - acc;
                q.r[dof] = rt;
                part += rt * rt;
            }
        }
    }
    return part;
}

// Loop bookkeeping after the gather's reduction (one thread): alpha, or the
// verification verdict (converged / restart), linalg.cpp:321-336.
__device__ __forceinline__ void cg_gather_finish(CgState *st, int yx, double tot) {
    if (!yx) {
        const double pap = tot;
        if (!isfinite(pap)) {
            st->done = CG_BREAKDOWN;
            st->breakdown_code = 1;  // NaN/Inf
        } else if (pap <= 0.0) {
            st->done = CG_BREAKDOWN;
            st->breakdown_code = 2;  // p'Ap <= 0
        } else {
            st->alpha = st->rho / pap;
        }
        st->phase = PH_NORMAL;
    } else {
        st->res = sqrt(tot);
        if (st->res <= st->tol_abs) {
            st->done = CG_CONVERGED;
            st->phase = PH_RESTART;
        } else if (st->replacing) {
            st->phase = PH_REPLACE;  // mid-solve residual replacement: not a failed check
        } else {
            st->restarts += 1;
            st->phase = PH_RESTART;
        }
        if (st->replacing) {
            st->replacing = 0;
            st->replaced = 1;
        }
    }
}

__global__ void __launch_bounds__(256) cg_gather_kernel(CgParams q) {
    pdl_wait();
    __shared__ double sh[64];
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int yx = st->y_holds_x;
    double part[1] = {cg_gather_nodes(q, yx)};
    pdl_trigger();
    block_sum<1>(part, sh);
    if (!publish_partials<1>(part, q.partial, &st->ticket_a)) return;
    double tot[1];
    grid_sum<1>(q.partial, gridDim.x, tot, sh);
    if (threadIdx.x == 0) {
        st->ticket_a = 0u;
        cg_gather_finish(st, yx, tot[0]);
        __threadfence();
    }
}

// B: x += alpha p, r -= alpha Ap, z = M r, (r.z, r.r); or the restart /
// initial variants. The last CTA advances the iteration counter and
// decides what the next operator product is (loop head of cg_solve).
__global__ void __launch_bounds__(256) cg_update_kernel(CgParams q) {
    pdl_wait();
    __shared__ double sh[64];
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int phase = st->phase;
    const double alpha = st->alpha;
    const int N = q.n_nodes;
    double part[2] = {0.0, 0.0};
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
        double r3[3], z3[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            double rv;
            if (phase == PH_NORMAL) {
                q.x[dof] += alpha * q.p[dof];
                rv = q.r[dof] - alpha * q.ap[dof];
                q.r[dof] = rv;
            } else if (phase == PH_INIT) {
                q.x[dof] = 0.0;
                rv = q.b[dof];  // r = b - A*0
                q.r[dof] = rv;
            } else {
                rv = q.r[dof];
            }
            r3[c] = rv;
        }
        precond_node(q.precond, q.pre, node, N, r3, z3);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            part[0] += r3[c] * z3[c];
            part[1] += r3[c] * r3[c];
        }
    }
    block_sum<2>(part, sh);
    if (!publish_partials<2>(part, q.partial, &st->ticket_b)) return;
    double tot[2];
    grid_sum<2>(q.partial, gridDim.x, tot, sh);
    if (threadIdx.x != 0) return;
    st->ticket_b = 0u;
    if (phase == PH_INIT) {
        st->norm_b = sqrt(tot[1]);
        st->tol_abs = st->tol * st->norm_b;
        st->rho = tot[0];
        st->res = st->norm_b;
        st->best_res = st->res;
        st->best_it = 0;
        st->it = 0;
        st->p_assign = 1;
        if (!isfinite(st->norm_b)) {
            st->done = CG_BREAKDOWN;
            st->breakdown_code = 1;
        } else if (st->norm_b == 0.0) {
            st->done = CG_CONVERGED;  // x = 0 solves exactly (linalg.cpp:298)
        } else {
            st->y_holds_x = st->res <= st->tol_abs ? 1 : 0;
        }
    } else if (phase == PH_RESTART) {
        st->rho = tot[0];
        st->p_assign = 1;
        st->y_holds_x = 0;
    } else {
        const double rho_next = tot[0];
        st->beta = rho_next / st->rho;
        st->rho = rho_next;
        st->res = sqrt(tot[1]);
        st->p_assign = 0;
        if (!isfinite(st->res)) {
            st->done = CG_BREAKDOWN;
            st->breakdown_code = 1;
        } else {
            st->it += 1;
            if (st->res < st->best_res) {
                st->best_res = st->res;
                st->best_it = st->it;
            }
            if (st->it >= st->max_it) {
                st->done = (st->res / st->norm_b <= st->tol) ? CG_CONVERGED : CG_NOCONV;
            } else {
                st->y_holds_x = st->res <= st->tol_abs ? 1 : 0;
            }
        }
    }
    __threadfence();
}

// C: p = z + beta p (or p = z), then write the next operator operand (p,
// or x for a verification) into the block-major panel, free DoFs only.
__global__ void __launch_bounds__(256) cg_scatter_kernel(CgParams q) {
    pdl_wait();
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int p_assign = st->p_assign, yx = st->y_holds_x;
    const double beta = st->beta;
    const int N = q.n_nodes;
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
        double r3[3], z3[3];
        if (q.precond == 3) {
#pragma unroll
            for (int c = 0; c < 3; ++c) z3[c] = q.zbuf[static_cast<long long>(c) * N + node];
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) r3[c] = q.r[static_cast<long long>(c) * N + node];
            precond_node(q.precond, q.pre, node, N, r3, z3);
        }
        const int4 s = reinterpret_cast<const int4 *>(q.slots)[node];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            const double pn = p_assign ? z3[c] : z3[c] + beta * q.p[dof];
            q.p[dof] = pn;
            if (q.cmask[dof]) continue;
            const double v = yx ? q.x[dof] : pn;
            const int co = c * q.nn;
            if (s.x >= 0) q.X[s.x + co] = v;
            if (s.y >= 0) q.X[s.y + co] = v;
            if (s.z >= 0) q.X[s.z + co] = v;
            if (s.w >= 0) q.X[s.w + co] = v;
        }
    }
}

// Assembled thermal load (assemble_global, global_stage.cpp:135-142):
// b[dof] = sum over the blocks holding dof, in increasing cell order, of
// dT_cell * b_el[kind][a], each product rounded then added from 0.0 (the
// reference's sequential loop; no FMA contraction), so b is bit-identical.
// Constrained DoFs take g (lifting, fem.cpp:223-260; g_int may be NULL = 0).
__global__ void rhs_kernel(int n_nodes, int nn, long long ldk, const int *slots, const int *row_cell,
                           const uint8_t *row_kind, const double *row_dt, const double *bel0, const double *bel1,
                           const uint8_t *cmask, const double *g_int, double *b) {
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= n_nodes) return;
    const int4 s4 = reinterpret_cast<const int4 *>(slots)[node];
    const int sl[4] = {s4.x, s4.y, s4.z, s4.w};
    int cell[4], row[4], rank[4], cnt = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (sl[k] < 0) continue;
        const int rw = static_cast<int>(sl[k] / ldk);
        int c = row_cell[rw], q = cnt++;
        while (q > 0 && cell[q - 1] > c) {  // insertion sort by cell (<= 4 copies)
            cell[q] = cell[q - 1]; row[q] = row[q - 1]; rank[q] = rank[q - 1];
            --q;
        }
        cell[q] = c;
        row[q] = rw;
        rank[q] = static_cast<int>(sl[k] - static_cast<long long>(rw) * ldk);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const long long dof = static_cast<long long>(c) * n_nodes + node;
        double acc = 0.0;
        for (int k = 0; k < cnt; ++k) {
            const double *bel = row_kind[row[k]] ? bel1 : bel0;
            acc = __dadd_rn(acc, __dmul_rn(row_dt[row[k]], bel[3 * rank[k] + c]));
        }
        b[dof] = cmask[dof] ? (g_int ? g_int[dof] : 0.0) : acc;
    }
}

// Internal SoA [component][internal node] -> reference DoF order 3 node + c.
__global__ void to_reference_kernel(int n_nodes, const uint32_t *glob_of_int, const double *v, double *out) {
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= n_nodes) return;
    const long long g = 3ll * glob_of_int[node];
#pragma unroll
    for (int c = 0; c < 3; ++c) out[g + c] = v[static_cast<long long>(c) * n_nodes + node];
}

// Plain gather/scatter helpers (tsv_apply, recovery, RHS lifting).
// mode 0: X[slot] = v (free DoFs only, constrained slots zeroed)
// mode 1: X[slot] = v for every DoF (recovery uses u at all DoFs)
// mode 2: X[slot] = v on constrained DoFs only, 0 elsewhere (A_fc g)
__global__ void scatter_vec_kernel(int n_nodes, int nn, const int *slots, const uint8_t *cmask, const double *v,
                                   double *X, int mode) {
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= n_nodes) return;
    const int4 s = reinterpret_cast<const int4 *>(slots)[node];
    const int sl[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const long long dof = static_cast<long long>(c) * n_nodes + node;
        const bool cm = cmask[dof] != 0;
        double val = v[dof];
        if ((mode == 0 && cm) || (mode == 2 && !cm)) val = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (sl[k] >= 0) X[sl[k] + c * nn] = val;
    }
}

// y = Mf o sum(Y) + Mc o x  (mode 0), or b_f -= sum(Y), b_c = g (mode 1).
__global__ void gather_vec_kernel(int n_nodes, int nn, const int *slots, const uint8_t *cmask, const double *Y,
                                  const double *x, double *y, int mode) {
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= n_nodes) return;
    const int4 s = reinterpret_cast<const int4 *>(slots)[node];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const long long dof = static_cast<long long>(c) * n_nodes + node;
        const int co = c * nn;
        double acc = 0.0;
        if (s.x >= 0) acc += Y[s.x + co];
        if (s.y >= 0) acc += Y[s.y + co];
        if (s.z >= 0) acc += Y[s.z + co];
        if (s.w >= 0) acc += Y[s.w + co];
        if (mode == 0) {
            y[dof] = cmask[dof] ? x[dof] : acc;
        } else {
            y[dof] = cmask[dof] ? x[dof] : y[dof] - acc;
        }
    }
}

// K6s: the fine DoFs whose basis rows are sparse (the block's surface nodes,
// pinned to the Lagrange interpolation of one face, edge or corner: <= q^2
// non-zeros of n) are reconstructed from a CSR copy of those rows instead of
// the dense GEMM: u[dof] = sum_e Phi[dof][col_e] q[col_e] + dT u_T[dof]
// (reconstruct_block_field, global_stage.cpp:215-230, without the exact zeros).
// A CTA takes kK6sRows block rows, staged in shared memory column-major
// (xs[col][row]: one entry's kK6sRows operands are 64 contiguous bytes), and
// one of gridDim.y slices of the sparse DoFs; each CSR entry is read once per
// kK6sRows rows.
constexpr int kK6sRows = 8;
struct K6Sparse {
    const double *X;        // Q panel rows of the chunk (row stride ldk)
    long long ldk;
    int rows;               // rows in the chunk
    const double *row_dt;   // dT per chunk row
    int n_sparse;
    const int *ptr, *dof, *col;
    const double *val, *ut;  // ut: u_T over all fine DoFs
    double *U;
    long long ldu;
};

__global__ void __launch_bounds__(256) k6_sparse_kernel(K6Sparse p) {
    extern __shared__ double xs[];  // [ldk][kK6sRows]
    const int r0 = blockIdx.x * kK6sRows;
    const int nr = min(kK6sRows, p.rows - r0);
    for (int i = threadIdx.x; i < kK6sRows * p.ldk; i += blockDim.x) {
        const int r = static_cast<int>(i / p.ldk), c = static_cast<int>(i % p.ldk);
        xs[c * kK6sRows + r] = r < nr ? p.X[(static_cast<long long>(r0) + r) * p.ldk + c] : 0.0;
    }
    __syncthreads();
    double dt[kK6sRows];
#pragma unroll
    for (int r = 0; r < kK6sRows; ++r) dt[r] = r < nr ? p.row_dt[r0 + r] : 0.0;
    const int per = (p.n_sparse + gridDim.y - 1) / gridDim.y;
    const int j0 = blockIdx.y * per, j1 = min(p.n_sparse, j0 + per);
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
        double acc[kK6sRows];
#pragma unroll
        for (int r = 0; r < kK6sRows; ++r) acc[r] = 0.0;
        const int e1 = p.ptr[j + 1];
        for (int e = p.ptr[j]; e < e1; ++e) {
            const int c = __ldg(p.col + e);
            const double v = __ldg(p.val + e);
            const double2 *xc = reinterpret_cast<const double2 *>(xs + c * kK6sRows);
#pragma unroll
            for (int h = 0; h < kK6sRows / 2; ++h) {
                const double2 x2 = xc[h];
                acc[2 * h] += v * x2.x;
                acc[2 * h + 1] += v * x2.y;
            }
        }
        const int dof = p.dof[j];
        const double ut = p.ut[dof];
#pragma unroll
        for (int r = 0; r < kK6sRows; ++r)
            if (r < nr) p.U[(static_cast<long long>(r0) + r) * p.ldu + dof] = acc[r] + dt[r] * ut;
    }
}

// K6f: the surface rows of Phi grouped by (face, component): every row of a
// group interpolates from the same <= kFaceK reduced DoFs (the face's
// interface nodes, one component), so a group is a small dense GEMM
// U[rows][dof_g] = Q[rows][cols_g] W_g^T + dT u_T. A CTA computes 32 block
// rows x 128 group rows (4 x 4 per thread) with K <= kFaceK staged k-major.
constexpr int kFaceK = 64;
struct K6Face {
    const double *X;          // Q panel rows of the chunk (row stride ldk)
    long long ldk;
    int rows;                 // rows in the chunk
    const double *row_dt;     // dT per chunk row
    const int4 *ginfo;        // per group: {row offset, rows, col offset, K}
    const int *gcol;          // [sum K] panel columns
    const double *gwt;        // per group: W^T [K][rows] at K-offset * ... (wt_off)
    const long long *gwoff;   // per group: offset of its W^T in gwt
    const int *gdof;          // [sum rows] fine DoF of each group row
    const double *ut;         // u_T over all fine DoFs
    double *U;
    long long ldu;
};

constexpr int kFaceSub = 8;  // 32-row sub-tiles per CTA (the W tile is staged once)
__global__ void __launch_bounds__(256) k6_face_kernel(K6Face p) {
    extern __shared__ __align__(16) double k6f_smem[];  // ws [K][128], then qs [K][32]
    const int4 gi4 = p.ginfo[blockIdx.y];
    const int row_off = gi4.x, nrows = gi4.y, col_off = gi4.z, K = gi4.w;
    double (*ws)[128] = reinterpret_cast<double (*)[128]>(k6f_smem);
    double (*qs)[32] = reinterpret_cast<double (*)[32]>(k6f_smem + static_cast<size_t>(K) * 128);
    const int t0 = blockIdx.z * 128;
    if (t0 >= nrows) return;
    const int tid = threadIdx.x;
    const double *wt = p.gwt + p.gwoff[blockIdx.y];
    // staging loads issued in batches of 8 before their stores (one memory
    // round trip per batch instead of one per element)
    for (int i0 = tid; i0 < K * 128; i0 += 256 * 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + 256 * u, k = i >> 7, j = i & 127;
            v[u] = (i < K * 128 && t0 + j < nrows) ? wt[static_cast<long long>(k) * nrows + t0 + j] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + 256 * u;
            if (i < K * 128) ws[i >> 7][i & 127] = v[u];
        }
    }
    const int gq = tid & 31, bq = tid >> 5;  // group rows gq + 32 b (coalesced stores), block rows 4 bq + a
    int dof[4];
    double ut[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int j = t0 + gq + 32 * b;
        dof[b] = j < nrows ? p.gdof[row_off + j] : -1;
        ut[b] = j < nrows ? p.ut[dof[b]] : 0.0;
    }
    // X gathers of the next 32-row sub-tile are issued before the current
    // one is computed (register double buffer)
    static_assert(kFaceK * 32 <= 256 * 8, "one batch of gathers per sub-tile");
    double v[8];
    auto gather = [&](int r0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = tid + 256 * u, k = i >> 5, r = i & 31;
            v[u] = (i < K * 32 && r0 + r < p.rows) ? p.X[(static_cast<long long>(r0) + r) * p.ldk + p.gcol[col_off + k]] : 0.0;
        }
    };
    gather(blockIdx.x * kFaceSub * 32);
    for (int sub = 0; sub < kFaceSub; ++sub) {
        const int r0 = (blockIdx.x * kFaceSub + sub) * 32;
        if (r0 >= p.rows) break;
        __syncthreads();  // ws staged / previous sub-tile's qs consumed
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = tid + 256 * u;
            if (i < K * 32) qs[i >> 5][i & 31] = v[u];
        }
        __syncthreads();
        if (sub + 1 < kFaceSub) gather(r0 + 32);
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        for (int k = 0; k < K; ++k) {
            const double2 q01 = *reinterpret_cast<const double2 *>(&qs[k][bq * 4]);
            const double2 q23 = *reinterpret_cast<const double2 *>(&qs[k][bq * 4 + 2]);
            const double q[4] = {q01.x, q01.y, q23.x, q23.y};
            const double w[4] = {ws[k][gq], ws[k][gq + 32], ws[k][gq + 64], ws[k][gq + 96]};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] += q[a] * w[b];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int r = r0 + bq * 4 + a;
            if (r >= p.rows) continue;
            const double dt = p.row_dt[r];
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (dof[b] >= 0) p.U[static_cast<long long>(r) * p.ldu + dof[b]] = acc[a][b] + dt * ut[b];
        }
    }
}

// ---------------------------------------------------------------- stress
// K7: strain/stress/von Mises at Gauss points (or centroids) of every
// element of a chunk of blocks, from the reconstructed fine field U.
struct StressParams {
    const double *U;
    long long ldu;
    int j0;               // first GEMM row of the chunk
    const int *row_cell;  // GEMM row -> original cell (-1 = padding)
    const uint8_t *row_kind;
    const double *row_dt;
    int cx, cy, cz, P;
    const double *hinv[2];    // [kind][cx + cy + cz]: 1/h per axis cell (x, then y, then z)
    const uint8_t *elem_mat[2];
    double lame[2][3][3];     // [kind][mat] lambda, mu, alpha*(3 lambda + 2 mu)
    double *out;
    long long out_cell0;      // first original cell of the output range
    long long out_cells;      // cells in the output range
};

// One CTA per (element layer, block): the two node layers of u are staged in
// shared memory, one thread evaluates one element at all its P points. The
// gradients of a trilinear box element are separable: du_c/dx depends on
// (eta, zeta) only, du_c/dy on (xi, zeta), du_c/dz on (xi, eta), so the 9
// derivatives take 4 distinct values each over the 8 Gauss points; they are
// formed once per element from the 12 edge differences (fem.cpp:27-58 with a
// diagonal Jacobian) and reused, leaving ~40 FP64 operations per point.
// Output: each warp stages one xi-half of its 32 elements' records (4 points
// x 7 values = 224 B = 7 whole sectors per element) in shared memory with an
// odd per-element stride (conflict-free) and streams them out, so the staging
// area stays small enough for 4 CTAs per SM.
constexpr int kStressThreads = 128;
constexpr int kStressWarps = kStressThreads / 32;

__host__ __device__ constexpr int stress_halves(int P) { return P == 8 ? 2 : 1; }
__host__ __device__ constexpr int stress_stride(int P) { return (P / stress_halves(P) * 7) | 1; }
inline size_t stress_smem_bytes(int P, int cx, int cy) {
    return (static_cast<size_t>(kStressWarps) * 32 * stress_stride(P) + 9 + cx + cy +
            2 * static_cast<size_t>(cx + 1) * (cy + 1) * 3) * sizeof(double);
}

// Bilinear form over two natural coordinates s1, s2 in {-g, +g} of the edge
// differences D[a][b] (a along s1, b along s2), scaled by q:
//   out[(s1 > 0) << 1 | (s2 > 0)] = q sum_ab w_a(s1) w_b(s2) D[a][b],  w_0 = 1 - s, w_1 = 1 + s.
__device__ __forceinline__ void stress_bilinear(double d00, double d10, double d01, double d11, double q,
                                                double out[4]) {
    constexpr double g = 0.57735026918962576451;  // 1/sqrt(3)
    const double A = 1.0 + g, Bm = 1.0 - g;
    const double t0m = fma(A, d00, Bm * d10), t1m = fma(A, d01, Bm * d11);  // s1 = -g
    const double t0p = fma(Bm, d00, A * d10), t1p = fma(Bm, d01, A * d11);  // s1 = +g
    const double qA = q * A, qB = q * Bm;
    out[0] = fma(qA, t0m, qB * t1m);
    out[1] = fma(qB, t0m, qA * t1m);
    out[2] = fma(qA, t0p, qB * t1p);
    out[3] = fma(qB, t0p, qA * t1p);
}

template <int P>
__global__ void __launch_bounds__(kStressThreads, 4) stress_kernel(StressParams sp) {
    static_assert(P == 8 || P == 1, "Gauss 2x2x2 or centroid");
    constexpr int REC = P * 7, HALVES = stress_halves(P), GPH = P / HALVES, RECH = GPH * 7;
    constexpr int STR = stress_stride(P), NV = P == 8 ? 4 : 1;
    extern __shared__ double sm[];
    const int k = blockIdx.x;   // element layer
    const int jr = blockIdx.y;  // row within chunk
    const int j = sp.j0 + jr;
    const int cell = sp.row_cell[j];
    if (cell < 0) return;
    const long long oc = cell - sp.out_cell0;
    if (oc < 0 || oc >= sp.out_cells) return;
    const int kind = sp.row_kind[j];
    const int cx = sp.cx, cy = sp.cy, nx = cx + 1, nxy = nx * (cy + 1);
    double *stg = sm;                                  // [warp][32][STR]
    double *ls = stg + kStressWarps * 32 * STR;        // lambda, mu, alpha(3 lambda + 2 mu) per material
    double *hs = ls + 9;                               // 1/h along x (cx), then y (cy)
    double *su = hs + cx + cy;                         // node layers k, k+1: [2][nxy][3]
    const double *U = sp.U + static_cast<long long>(jr) * sp.ldu + static_cast<long long>(k) * nxy * 3;
    for (int i = threadIdx.x; i < 2 * nxy * 3; i += kStressThreads) su[i] = __ldg(U + i);
    const double *hk = sp.hinv[kind];
    for (int i = threadIdx.x; i < cx + cy; i += kStressThreads) hs[i] = hk[i];
    if (threadIdx.x < 9) ls[threadIdx.x] = sp.lame[kind][threadIdx.x / 3][threadIdx.x % 3];
    __syncthreads();
    const double dt = sp.row_dt[j];
    const double qz = 0.25 * hk[cx + cy + k];
    const int ne = cx * cy;
    const long long E = static_cast<long long>(cx) * cy * sp.cz;
    double *out_layer = sp.out + (oc * E + static_cast<long long>(k) * ne) * REC;
    const uint8_t *emat = sp.elem_mat[kind] + static_cast<long long>(k) * ne;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *wst = stg + warp * 32 * STR;
    for (int base = warp * 32; base < ne; base += kStressThreads) {
        const int e2 = base + lane;
        const bool live = e2 < ne;
        double dux[3][NV], duy[3][NV], duz[3][NV];
        double lambda = 0.0, mu = 0.0, thermal = 0.0;
        if (live) {
            const int i = e2 % cx, jj = e2 / cx;
            const double qx = 0.25 * hs[i], qy = 0.25 * hs[cx + jj];
            const double *u0 = su + (jj * nx + i) * 3;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double v000 = u0[c], v100 = u0[3 + c], v010 = u0[nx * 3 + c], v110 = u0[nx * 3 + 3 + c];
                const double v001 = u0[nxy * 3 + c], v101 = u0[nxy * 3 + 3 + c];
                const double v011 = u0[(nxy + nx) * 3 + c], v111 = u0[(nxy + nx) * 3 + 3 + c];
                // edge differences: x-edges at (y, z), y-edges at (x, z), z-edges at (x, y)
                const double x00 = v100 - v000, x10 = v110 - v010, x01 = v101 - v001, x11 = v111 - v011;
                const double y00 = v010 - v000, y10 = v110 - v100, y01 = v011 - v001, y11 = v111 - v101;
                const double z00 = v001 - v000, z10 = v101 - v100, z01 = v011 - v010, z11 = v111 - v110;
                if constexpr (P == 8) {
                    stress_bilinear(x00, x10, x01, x11, qx, dux[c]);  // (eta, zeta)
                    stress_bilinear(y00, y10, y01, y11, qy, duy[c]);  // (xi, zeta)
                    stress_bilinear(z00, z10, z01, z11, qz, duz[c]);  // (xi, eta)
                } else {
                    dux[c][0] = qx * ((x00 + x10) + (x01 + x11));
                    duy[c][0] = qy * ((y00 + y10) + (y01 + y11));
                    duz[c][0] = qz * ((z00 + z10) + (z01 + z11));
                }
            }
            const int mat = emat[e2];
            lambda = ls[mat * 3];
            mu = ls[mat * 3 + 1];
            thermal = ls[mat * 3 + 2] * dt;
        }
        const double mu2 = 2.0 * mu;
        const int nel = min(32, ne - base);
        double *dst = out_layer + static_cast<long long>(base) * REC;
#pragma unroll
        for (int h = 0; h < HALVES; ++h) {
            if (live) {
                double *o = wst + lane * STR;
#pragma unroll
                for (int gl = 0; gl < GPH; ++gl) {
                    // gp = (xi bit) << 2 | (eta bit) << 1 | (zeta bit), zeta fastest (fem.cpp:87-92)
                    const int gp = h * GPH + gl;
                    const int ix = P == 8 ? (gp & 3) : 0;                        // (eta, zeta)
                    const int iy = P == 8 ? (((gp >> 2) << 1) | (gp & 1)) : 0;  // (xi, zeta)
                    const int iz = P == 8 ? (gp >> 1) : 0;                       // (xi, eta)
                    const double exx = dux[0][ix], eyy = duy[1][iy], ezz = duz[2][iz];
                    const double s0 = fma(lambda, exx + eyy + ezz, -thermal);
                    const double sxx = fma(mu2, exx, s0), syy = fma(mu2, eyy, s0), szz = fma(mu2, ezz, s0);
                    const double sxy = mu * (duy[0][iy] + dux[1][ix]);
                    const double syz = mu * (duz[1][iz] + duy[2][iy]);
                    const double szx = mu * (dux[2][ix] + duz[0][iz]);
                    const double d1 = sxx - syy, d2 = syy - szz, d3 = szz - sxx;
                    const double nrm = fma(d1, d1, fma(d2, d2, d3 * d3));
                    const double shr = fma(sxy, sxy, fma(syz, syz, szx * szx));
                    const double vm2 = fma(0.5, nrm, 3.0 * shr);
                    o[gl * 7 + 0] = sxx; o[gl * 7 + 1] = syy; o[gl * 7 + 2] = szz;
                    o[gl * 7 + 3] = sxy; o[gl * 7 + 4] = syz; o[gl * 7 + 5] = szx;
                    o[gl * 7 + 6] = sqrt(fmax(vm2, 0.0));
                }
            }
            __syncwarp();
            // element el's half-record: dst[el*REC + h*RECH .. + RECH) (whole sectors when P = 8)
            for (int q = lane; q < nel * RECH; q += 32) {
                const int el = q / RECH, off = q - el * RECH;
                __stcs(dst + el * REC + h * RECH + off, wst[el * STR + off]);
            }
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------- cut plane
// cutplane_von_mises (global_stage.cpp:245-274): von Mises at res x res
// cell-centred samples of the plane z = h/2 of every block
// (StressGrid::local_coord, stress_grid.cpp:32-34), the containing element
// found with the reference's tie rule (locate_axis_cell, mesh.cpp:97-104:
// a point on a grid plane belongs to the lower cell).
struct CutParams {
    const double *U;
    long long ldu;
    int j0;
    const int *row_cell;
    const uint8_t *row_kind;
    const double *row_dt;
    const double *grid[2][3];  // [kind][axis] grid lines
    int len[3];                // grid line counts
    const uint8_t *elem_mat[2];
    double lame[2][3][3];
    int res;
    double pitch, z_mid;
    double *out;               // StressGrid::values
    long long out_cell0, out_cells;
};

__device__ __forceinline__ int locate_axis_cell(const double *axis, int len, double v) {
    int lo = 0, hi = len;  // upper_bound: first index with axis[idx] > v
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (axis[mid] <= v) lo = mid + 1;
        else hi = mid;
    }
    int k = lo == 0 ? 0 : lo - 1;  // axis[k] <= v
    if (k > 0 && axis[k] == v) return k - 1;
    return min(k, len - 2);
}

__global__ void cutplane_kernel(CutParams cp) {
    const int jr = blockIdx.x;
    const int j = cp.j0 + jr;
    const int cell = cp.row_cell[j];
    if (cell < 0) return;
    const long long oc = cell - cp.out_cell0;
    if (oc < 0 || oc >= cp.out_cells) return;
    const int t = blockIdx.y * blockDim.x + threadIdx.x;
    if (t >= cp.res * cp.res) return;
    const int py = t / cp.res, px = t % cp.res;
    const int kind = cp.row_kind[j];
    const double *gx = cp.grid[kind][0], *gy = cp.grid[kind][1], *gz = cp.grid[kind][2];
    const double x = (static_cast<double>(px) + 0.5) * cp.pitch / static_cast<double>(cp.res);
    const double y = (static_cast<double>(py) + 0.5) * cp.pitch / static_cast<double>(cp.res);
    const double z = cp.z_mid;
    const int i = locate_axis_cell(gx, cp.len[0], x);
    const int jj = locate_axis_cell(gy, cp.len[1], y);
    const int k = locate_axis_cell(gz, cp.len[2], z);
    const double x0 = gx[i], x1 = gx[i + 1], y0 = gy[jj], y1 = gy[jj + 1], z0 = gz[k], z1 = gz[k + 1];
    const double xi = 2.0 * (x - x0) / (x1 - x0) - 1.0;  // fem.cpp:271-273
    const double eta = 2.0 * (y - y0) / (y1 - y0) - 1.0;
    const double zeta = 2.0 * (z - z0) / (z1 - z0) - 1.0;
    const double hxi = 1.0 / (x1 - x0), hyi = 1.0 / (y1 - y0), hzi = 1.0 / (z1 - z0);
    const int nx = cp.len[0], ny = cp.len[1];
    const double *U = cp.U + static_cast<long long>(jr) * cp.ldu;
    double du[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const int di = (a == 1 || a == 2 || a == 5 || a == 6);
        const int dj = (a == 2 || a == 3 || a == 6 || a == 7);
        const int dk = a >= 4;
        const double sx = di ? 1.0 : -1.0, sy = dj ? 1.0 : -1.0, sz = dk ? 1.0 : -1.0;
        const double gxa = 0.25 * sx * (1.0 + sy * eta) * (1.0 + sz * zeta) * hxi;
        const double gya = 0.25 * sy * (1.0 + sx * xi) * (1.0 + sz * zeta) * hyi;
        const double gza = 0.25 * sz * (1.0 + sx * xi) * (1.0 + sy * eta) * hzi;
        const double *ua = U + 3LL * (((k + dk) * ny + (jj + dj)) * nx + (i + di));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            du[c][0] += ua[c] * gxa;
            du[c][1] += ua[c] * gya;
            du[c][2] += ua[c] * gza;
        }
    }
    const long long e = (static_cast<long long>(k) * (ny - 1) + jj) * (nx - 1) + i;
    const int mat = cp.elem_mat[kind][e];
    const double lambda = cp.lame[kind][mat][0], mu = cp.lame[kind][mat][1];
    const double thermal = cp.lame[kind][mat][2] * cp.row_dt[j];
    const double exx = du[0][0], eyy = du[1][1], ezz = du[2][2];
    const double tr = exx + eyy + ezz;
    const double sxx = lambda * tr + 2.0 * mu * exx - thermal;
    const double syy = lambda * tr + 2.0 * mu * eyy - thermal;
    const double szz = lambda * tr + 2.0 * mu * ezz - thermal;
    const double sxy = mu * (du[0][1] + du[1][0]), syz = mu * (du[1][2] + du[2][1]), szx = mu * (du[2][0] + du[0][2]);
    const double d1 = sxx - syy, d2 = syy - szz, d3 = szz - sxx;
    const double vm2 = 0.5 * (d1 * d1 + d2 * d2 + d3 * d3) + 3.0 * (sxy * sxy + syz * syz + szx * szx);
    cp.out[(oc * cp.res + py) * cp.res + px] = sqrt(fmax(vm2, 0.0));
}

// ------------------------------------------------------------ peaks
__global__ void peak_dmma_kernel(double *sink, int iters) {
    double acc[8][2];
    const double a = threadIdx.x * 1e-9, b = 1.0 + threadIdx.x * 1e-12;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma_8x8x4(acc[i][0], acc[i][1], a, b);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.0) sink[0] = s;
}

__global__ void peak_dfma_kernel(double *sink, int iters) {
    double acc[16];
    const double a = threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], b, a);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 12345.0) sink[0] = s;
}

}  // namespace tsvb200
