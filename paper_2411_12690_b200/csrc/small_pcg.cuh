// Persistent two-level Schwarz PCG for small arrays (configs 0-1).
//
// At 9-100 blocks every pass of the graph-captured loop is a few microseconds
// of work behind a kernel boundary (~11 kernels per iteration, ~50 us). Here
// the whole solve is ONE cooperative kernel: the same passes run back to back
// with grid-wide barriers between them, and the CG scalars live in every CTA
// (each CTA keeps an identical copy of CgState in shared memory, updated from
// the same fixed-order reductions, so no broadcast is needed). The control
// flow is the reference's cg_solve (linalg.cpp:292-362) as on the graph path:
// x0 = 0, recursive-residual test, true-residual verification (K1 on x) with
// restart, p'Ap / NaN breakdown, best iterate, max iterations.
//
// Per iteration (8 grid barriers):
//   U  x += alpha p, r -= alpha Ap, r -> XL panel (FP64), r.r, loop head
//   P  local products ZL = XL Ainv_type (split-K DMMA items)  | restriction
//   R  split-K reduction -> ZL, coarse rhs rc = P^T r
//   C  zc = Ainv_c rc (FP64 dense, warp per row), rc.zc       | z_l, r.z_l
//   S  p = z_l + P zc + beta p -> X panel (x when verifying)
//   K  Y = X K_r (split-K DMMA items) ; K' reduction -> Y
//   G  gather Ap = sum of block copies, p.Ap -> alpha (or r = b - A x)
// Local solves and the coarse inverse are FP64 here (the graph path uses
// TF32 tcgen05 local solves and an FP32 coarse inverse for bandwidth; at
// these sizes bandwidth is irrelevant).
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"
#include "schwarz.cuh"

namespace tsvb200 {

struct SmallPcgParams {
    CgParams q;
    AsParams a;
    GemmParams k1, loc;       // K1 (Y = X K_r) and the local products (ZL = XL Ainv_type)
    SplitK sk1, skl;          // split-K partial buffers (tickets unused here)
    int k1_tiles, loc_tiles;  // tiles of each GEMM (items = tiles x S)
    const double *ainv_c;     // dense symmetric FP64 coarse inverse [Nc][Nc]
    double *gpart;            // [4][gridDim] per-CTA partials: U (1), C (2), G (1) slots
};

// Fixed-order grid reduction of one value per thread: block tree, per-CTA
// partial, barrier, then every CTA sums the partials in CTA order (each CTA
// obtains the identical total). Each call site owns its partial slot: a
// slot is reused only after further grid barriers.
template <int NV>
__device__ __forceinline__ void small_allreduce(cooperative_groups::grid_group &grid, double (&v)[NV], double *gpart,
                                                double *sh, double (&out)[NV]) {
    block_sum<NV>(v, sh);
    if (threadIdx.x == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) gpart[blockIdx.x * NV + i] = v[i];
    grid.sync();
    double s[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        s[i] = 0.0;
        for (int k = threadIdx.x; k < static_cast<int>(gridDim.x); k += blockDim.x) s[i] += __ldcg(gpart + k * NV + i);
    }
    block_sum<NV>(s, sh);
    __shared__ double bc[NV];
    if (threadIdx.x == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) bc[i] = s[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) out[i] = bc[i];
    __syncthreads();
}

// Split-K GEMM items (tile, slice) over the grid: partial accumulators to
// work, thread-major (as gemm_splitk_f64).
template <class Cfg>
__device__ __forceinline__ void small_gemm_items(const GemmParams &p, const SplitK &sk, int tiles, double *As, double *Bs) {
    constexpr int NACC = Cfg::FM * Cfg::FN * 2;
    const int S = sk.S;
    for (int item = blockIdx.x; item < tiles * S; item += gridDim.x) {
        const int tile = item / S, s = item % S;
        const int mt = tile / p.n_tiles, nt = tile % p.n_tiles;
        const int kc0 = (p.k_chunks * s) / S, kc1 = (p.k_chunks * (s + 1)) / S;
        double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        gemm_segment<Cfg>(p, As, Bs, mt, nt, kc0, kc1, gemm_fn_lim<Cfg>(p, nt), acc);
        double *w = sk.work + static_cast<long long>(item) * NACC * Cfg::THREADS + threadIdx.x;
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) w[((i * Cfg::FN + j) * 2 + h) * Cfg::THREADS] = acc[i][j][h];
    }
}

// Sum of the S partials of each tile in slice order, then the epilogue.
template <class Cfg>
__device__ __forceinline__ void small_gemm_finish(const GemmParams &p, const SplitK &sk, int tiles) {
    constexpr int NACC = Cfg::FM * Cfg::FN * 2;
    const int S = sk.S;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int mt = tile / p.n_tiles, nt = tile % p.n_tiles;
        double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
            for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        const double *w0 = sk.work + static_cast<long long>(tile) * S * NACC * Cfg::THREADS + threadIdx.x;
        for (int s2 = 0; s2 < S; ++s2) {
            const double *ws = w0 + static_cast<long long>(s2) * NACC * Cfg::THREADS;
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
                for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) acc[i][j][h] += __ldcg(ws + ((i * Cfg::FN + j) * 2 + h) * Cfg::THREADS);
        }
        gemm_epilogue<Cfg>(p, mt, nt, acc);
    }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS) pcg_small_kernel(SmallPcgParams P) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double smem[];
    __shared__ double sh[64];
    __shared__ CgState S;
    double *As = smem;
    double *Bs = smem + Cfg::STAGES * Cfg::A_STAGE;
    const CgParams &q = P.q;
    const AsParams &a = P.a;
    const int N = q.n_nodes;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int gtid = blockIdx.x * blockDim.x + tid, gthreads = gridDim.x * blockDim.x;
    if (tid == 0) S = *q.st;
    __syncthreads();
    const double rdz = 1.0 / static_cast<double>(a.qm1);

    for (;;) {
        // ---- U: x, r update; r -> XL panel; r.r; loop head
        {
            double v[1] = {as_update_nodes(q, a, S.phase, S.alpha)}, tot[1];
            small_allreduce<1>(grid, v, P.gpart, sh, tot);
            if (tid == 0) as_update_finish(&S, S.phase, tot[0]);
            __syncthreads();
            if (S.done) break;
        }
        if (!S.y_holds_x) {
            // ---- P: local products (split-K items) | restriction (warp per coarse cell)
            small_gemm_items<Cfg>(P.loc, P.skl, P.loc_tiles, As, Bs);
            for (int cell = blockIdx.x * nwarps + warp; cell < a.ncells; cell += gridDim.x * nwarps) {
                const AsCell cc = as_cell(a, cell);
                const int nb = a.cell_ptr[cell], ne = a.cell_ptr[cell + 1];
                double acc[3][8];
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[c][k] = 0.0;
                for (int node = nb + lane; node < ne; node += 32) {
                    double w[8];
                    as_cell_weights(a, cc, node, w);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const long long dof = static_cast<long long>(c) * N + node;
                        const double rv = q.cmask[dof] ? 0.0 : __ldcg(q.r + dof);
#pragma unroll
                        for (int k = 0; k < 8; ++k) acc[c][k] += w[k] * rv;
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double v = warp_sum(acc[c][k]);
                        if (lane == 3 * k + c) a.cellpart[cell * 24 + 3 * k + c] = v;
                    }
            }
            grid.sync();
            // ---- R: local reduction -> ZL; coarse rhs
            small_gemm_finish<Cfg>(P.loc, P.skl, P.loc_tiles);
            for (int j = gtid; j < a.Nc; j += gthreads) {
                const int comp = j % 3, cn = j / 3;
                const int nxn = a.SX + 1, nyn = a.SY + 1;
                const int gx = cn % nxn, gy = (cn / nxn) % nyn, gz = cn / (nxn * nyn);
                double s = 0.0;
                for (int cy = gy - 1; cy <= gy; ++cy) {
                    if (cy < 0 || cy >= a.SY) continue;
                    for (int cx = gx - 1; cx <= gx; ++cx) {
                        if (cx < 0 || cx >= a.SX) continue;
                        const int corner = (gx - cx) | ((gy - cy) << 1) | (gz << 2);
                        s += __ldcg(a.cellpart + (cy * a.SX + cx) * 24 + 3 * corner + comp);
                    }
                }
                a.rc[j] = s;
            }
            grid.sync();
            // ---- C: zc = Ainv_c rc (warp per row) and rc.zc | z_l and r.z_l
            double v2[2] = {0.0, 0.0}, tot2[2];
            for (int i = blockIdx.x * nwarps + warp; i < a.Nc; i += gridDim.x * nwarps) {
                const double *row = P.ainv_c + static_cast<long long>(i) * a.Nc;
                double s = 0.0;
                for (int j = lane; j < a.Nc; j += 32) s += row[j] * __ldcg(a.rc + j);
                s = warp_sum(s);
                if (lane == 0) {
                    a.zc[i] = s;
                    v2[0] += __ldcg(a.rc + i) * s;
                }
            }
            for (int node = gtid; node < N; node += gthreads) {
                const int4 s2 = reinterpret_cast<const int4 *>(a.slots2)[node];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const long long dof = static_cast<long long>(c) * N + node;
                    const double rv = __ldcg(q.r + dof);
                    double zv = rv;  // unit row on constrained DoFs
                    if (!q.cmask[dof]) {
                        const int co = c * q.nn;
                        zv = 0.0;
                        if (s2.x >= 0) zv += __ldcg(a.ZL + s2.x + co);
                        if (s2.y >= 0) zv += __ldcg(a.ZL + s2.y + co);
                        if (s2.z >= 0) zv += __ldcg(a.ZL + s2.z + co);
                        if (s2.w >= 0) zv += __ldcg(a.ZL + s2.w + co);
                    }
                    a.z[dof] = zv;
                    v2[1] += rv * zv;
                }
            }
            small_allreduce<2>(grid, v2, P.gpart + gridDim.x, sh, tot2);
            if (tid == 0) {
                S.rz_c = tot2[0];
                S.rz_l = tot2[1];
            }
            __syncthreads();
        }
        // ---- S: p = z_l + P zc + beta p (or p = z after init / restart) -> X
        // panel; x into the panel when verifying
        {
            const int yx = S.y_holds_x;
            const bool normal = S.phase == PH_NORMAL;
            const double rz = S.rz_l + S.rz_c;
            const double beta = normal ? rz / S.rho : 0.0;
            for (int node = gtid; node < N; node += gthreads) {
                const int4 s = reinterpret_cast<const int4 *>(q.slots)[node];
                if (yx) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const long long dof = static_cast<long long>(c) * N + node;
                        if (q.cmask[dof]) continue;
                        const double v = __ldcg(q.x + dof);
                        const int co = c * q.nn;
                        if (s.x >= 0) q.X[s.x + co] = v;
                        if (s.y >= 0) q.X[s.y + co] = v;
                        if (s.z >= 0) q.X[s.z + co] = v;
                        if (s.w >= 0) q.X[s.w + co] = v;
                    }
                    continue;
                }
                const int cell = a.node_cell[node];
                const double4 ct = a.celltab[cell];
                const short4 L = a.lat[node];
                const double tx = (static_cast<double>(L.x) - ct.x) * ct.z;
                const double ty = (static_cast<double>(L.y) - ct.y) * ct.w;
                const double tz = static_cast<double>(L.z) * rdz;
                const int cx = cell % a.SX, cy = cell / a.SX;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const long long dof = static_cast<long long>(c) * N + node;
                    double zv = __ldcg(a.z + dof);
                    const bool cm = q.cmask[dof] != 0;
                    if (!cm) {
                        double zcoarse = 0.0;
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const double w = ((k & 1) ? tx : 1.0 - tx) * ((k & 2) ? ty : 1.0 - ty) * ((k & 4) ? tz : 1.0 - tz);
                            zcoarse += w * __ldcg(a.zc + 3 * as_corner_node(a, cx, cy, k) + c);
                        }
                        zv += zcoarse;
                    }
                    const double pn = normal ? zv + beta * __ldcg(q.p + dof) : zv;
                    q.p[dof] = pn;
                    if (cm) continue;
                    const int co = c * q.nn;
                    if (s.x >= 0) q.X[s.x + co] = pn;
                    if (s.y >= 0) q.X[s.y + co] = pn;
                    if (s.z >= 0) q.X[s.z + co] = pn;
                    if (s.w >= 0) q.X[s.w + co] = pn;
                }
            }
            if (!yx && tid == 0) {
                if (normal) {
                    S.beta = beta;
                    S.p_assign = 0;
                } else {
                    S.p_assign = 1;
                    S.phase = PH_NORMAL;
                }
                S.rho = rz;
            }
            __syncthreads();
        }
        grid.sync();
        // ---- K: Y = X K_r (split-K items), reduction
        small_gemm_items<Cfg>(P.k1, P.sk1, P.k1_tiles, As, Bs);
        grid.sync();
        small_gemm_finish<Cfg>(P.k1, P.sk1, P.k1_tiles);
        grid.sync();
        // ---- G: gather, p.Ap -> alpha; or the true residual -> converged / restart
        {
            const int yx = S.y_holds_x;
            double v[1] = {cg_gather_nodes(q, yx)}, tot[1];
            small_allreduce<1>(grid, v, P.gpart + 3 * gridDim.x, sh, tot);
            if (tid == 0) cg_gather_finish(&S, yx, tot[0]);
            __syncthreads();
            if (S.done) break;
        }
    }
    if (blockIdx.x == 0 && tid == 0) {
        *q.st = S;
        __threadfence();
    }
}

}  // namespace tsvb200
