// Two-level additive Schwarz preconditioner for the reduced system
// (TSV_PRECOND_SCHWARZ2, new: the reference offers none / Jacobi / 3x3
// blocks, linalg.hpp:117; a stronger preconditioner is allowed when the
// solution parity holds).
//
//   z = sum_b R_b^T A_b^-1 R_b r  +  P A_c^-1 P^T r
//
//   local:  A_b = R_b A R_b^T, the lifted global matrix restricted to block
//           b's interface DoFs. It depends only on the block's neighbourhood
//           (own kind, the 8 neighbours' kinds or absence, constrained
//           pattern), so blocks are grouped into types and the local solves
//           are one batched DMMA GEMM over a type-ordered panel.
//   coarse: trilinear interpolation P from the corner lattice of s x s
//           super-blocks (x, y) and the bottom/top planes (z); A_c = P^T A P
//           is assembled from per-block 24 x 24 Galerkin products and
//           inverted once (dense, <= 8192 DoFs); the coarse solve is a dense
//           GEMV. P is zero on constrained DoFs.
//
// All reductions are fixed-order (deterministic).
#pragma once

#include "kernels.cuh"
#include "tc_local.cuh"

namespace tsvb200 {

struct AsParams {
    const int *slots2;     // [node][4] offsets into XL / ZL (type-ordered panel rows)
    double *XL;            // local-solve operand panel (FP64 path)
    const double *ZL;      // local-solve product panel (FP64 path)
    const float *ZL32;     // local-solve product panel (tensor-core path)
    double *z;             // [3][node] preconditioned residual
    const short4 *lat;     // (gx, gy, gz) lattice position of each internal node
    int step, step_y, SX, SY, lat_x, lat_y, qm1;  // super-cell steps along x / y (lattice units)
    const int *cell_ptr;   // super cell -> its contiguous internal node range
    const int *node_cell;  // internal node -> its super cell
    const double4 *celltab;  // per super cell: x0, y0, 1/dx, 1/dy (lattice units)
    int ncells;
    double *cellpart;      // [ncells][24]
    double *rc, *zc;       // coarse vectors [Nc]
    double *dotpart;       // [sym_nt] partials of rc.zc (symmetric coarse path)
    const double *ainv_c;  // dense [Nc][Nc]
    const float *ainv_c32; // FP32 copy [Nc][ldc32] (default; TSV_AS_COARSE_F64 keeps FP64): halves the
                           // coarse HBM stream. With the FP64 DMMA true-residual check it raised the
                           // restart count at tol 1e-12; with the exact int8 check it does not.
    int ldc32;
    int Nc;
    int round_bits;        // experiment: round the local-solve operand to this many mantissa bits (0 = off)
    // tensor-core local solve (tc_local.cuh): TF32 operand panel (same
    // row stride as ZL, so slots2 addresses both)
    float *XL32;
    // split loop: A P zc as a block panel (same layout as Y), from the
    // per-key products K_b P_b (as_kpzc_kernel)
    double *Yc;
    // early coarse chain: in a NORMAL phase the restriction reads A p and the
    // coarse rhs becomes rc - alpha P^T (A p) (forked before the r update)
    int rc_recur;
};

// as_kpzc_kernel work: per-key K_b P_b ([key][ldk][24], internal row order
// c nn + rank, columns 3 corner + comp), panel rows sorted by key, and
// (key, begin, end) items over that list.
struct KpzcParams {
    const double *kp;
    const int4 *items;
    const int *rows;
    const int *row_cell;
    int cols, sb, n;
    long long ldk;
};
constexpr int kKpzcChunk = 64;

// Round to `bits` explicit mantissa bits (emulates a low-precision operand).
__device__ __forceinline__ double round_mantissa(double v, int bits) {
    if (bits <= 0 || bits >= 52) return v;
    const int drop = 52 - bits;
    long long i = __double_as_longlong(v);
    i += 1LL << (drop - 1);
    i &= ~((1LL << drop) - 1);
    return __longlong_as_double(i);
}

// Per-cell kernels may run kAsSplit CTAs per super cell, each over a
// contiguous part of the cell's node range (partials stay per part). Measured
// on B200 at config 3: splitting by 4 makes both kernels slower (per-CTA
// reductions and the single completion ticket dominate), so 1.
constexpr int kAsSplit = 1;  // as_update_kernel<true> assumes one CTA per cell
__device__ __forceinline__ void as_part_range(const AsParams &a, int cell, int part, int &n0, int &n1) {
    const int b0 = a.cell_ptr[cell], b1 = a.cell_ptr[cell + 1], len = b1 - b0;
    n0 = b0 + static_cast<int>((static_cast<long long>(len) * part) / kAsSplit);
    n1 = b0 + static_cast<int>((static_cast<long long>(len) * (part + 1)) / kAsSplit);
}

// Trilinear weights of a node relative to super cell (cx, cy). Nodes are
// numbered super-cell-major, so a CTA per super cell sees a contiguous node
// range [cell_ptr[c], cell_ptr[c+1]) lying in that (closed) cell.
struct AsCell {
    int cx, cy, x0, y0;
    double rdx, rdy, rdz;  // reciprocal cell extents (lattice units)
};

__device__ __forceinline__ AsCell as_cell(const AsParams &a, int cell) {
    AsCell c;
    c.cx = cell % a.SX;
    c.cy = cell / a.SX;
    c.x0 = c.cx * a.step;
    c.y0 = c.cy * a.step_y;
    c.rdx = 1.0 / static_cast<double>(min(c.x0 + a.step, a.lat_x - 1) - c.x0);
    c.rdy = 1.0 / static_cast<double>(min(c.y0 + a.step_y, a.lat_y - 1) - c.y0);
    c.rdz = 1.0 / static_cast<double>(a.qm1);
    return c;
}

// Restriction (as_restrict_kernel) and prolongation (as_z_kernel) evaluate
// the same weights for the same node (its owner cell), so the two-level
// preconditioner stays symmetric.
__device__ __forceinline__ void as_cell_weights(const AsParams &a, const AsCell &c, int node, double w[8]) {
    const short4 L = a.lat[node];
    const double tx = static_cast<double>(L.x - c.x0) * c.rdx;
    const double ty = static_cast<double>(L.y - c.y0) * c.rdy;
    const double tz = static_cast<double>(L.z) * c.rdz;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        w[k] = ((k & 1) ? tx : 1.0 - tx) * ((k & 2) ? ty : 1.0 - ty) * ((k & 4) ? tz : 1.0 - tz);
}

__device__ __forceinline__ int as_corner_node(const AsParams &a, int cx, int cy, int c) {
    return (((c >> 2) & 1) * (a.SY + 1) + cy + ((c >> 1) & 1)) * (a.SX + 1) + cx + (c & 1);
}

// U': x += alpha p, r -= alpha Ap (NORMAL) | r = b (INIT) | r as is (RESTART);
// r scattered into the local-solve panel; r.r reduced; the last CTA runs
// the loop-head bookkeeping of cg_solve (iteration count, best iterate,
// max-iteration exit, next product = A x when the residual test passes).

// Node loop of U' (grid-stride): returns this thread's r.r partial.
__device__ __forceinline__ double as_update_nodes(const CgParams &q, const AsParams &a, int phase, double alpha) {
    const int N = q.n_nodes;
    double part = 0.0;
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
        const int4 s = reinterpret_cast<const int4 *>(a.slots2)[node];
        if (phase == PH_NORMAL && q.xlo && a.XL32) {
            // the hot path with the loads of all three components ahead of the stores (the compiler cannot
            // hoist them itself: the vectors may alias as far as it knows); same arithmetic as below
            double xh[3], pv[3], rr[3], av[3];
            float xl[3];
            uint8_t cm[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const long long dof = static_cast<long long>(c) * N + node;
                xh[c] = q.x[dof], pv[c] = q.p[dof], rr[c] = q.r[dof], av[c] = q.ap[dof], xl[c] = q.xlo[dof], cm[c] = q.cmask[dof];
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const long long dof = static_cast<long long>(c) * N + node;
                const double inc = __dmul_rn(alpha, pv[c]);
                const double t = __dadd_rn(xh[c], inc), bp = __dsub_rn(t, xh[c]);
                const double err = __dadd_rn(__dsub_rn(xh[c], __dsub_rn(t, bp)), __dsub_rn(inc, bp));
                q.x[dof] = t;
                q.xlo[dof] = static_cast<float>(static_cast<double>(xl[c]) + err);
                const double rv = rr[c] - alpha * av[c];
                q.r[dof] = rv;
                part += rv * rv;
                if (cm[c]) continue;
                const int co = c * q.nn;
                const float f = to_tf32(rv);
                if (s.x >= 0) a.XL32[s.x + co] = f;
                if (s.y >= 0) a.XL32[s.y + co] = f;
                if (s.z >= 0) a.XL32[s.z + co] = f;
                if (s.w >= 0) a.XL32[s.w + co] = f;
            }
            continue;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            double rv;
            if (phase == PH_NORMAL) {
                if (q.xlo) {
                    // x + alpha p by TwoSum: the rounding error of the sum goes to xlo. At
                    // the large configs eps |x| per update, seen through A, is ~0.25 tol |b|;
                    // accumulated over the iterations it is the gap between the recursive
                    // and the true residual that fails the first A x check.
                    const double xh = q.x[dof], inc = __dmul_rn(alpha, q.p[dof]);
                    const double t = __dadd_rn(xh, inc), bp = __dsub_rn(t, xh);
                    const double err = __dadd_rn(__dsub_rn(xh, __dsub_rn(t, bp)), __dsub_rn(inc, bp));
                    q.x[dof] = t;
                    q.xlo[dof] = static_cast<float>(static_cast<double>(q.xlo[dof]) + err);
                } else {
                    q.x[dof] += alpha * q.p[dof];
                }
                rv = q.r[dof] - alpha * q.ap[dof];
                q.r[dof] = rv;
            } else if (phase == PH_INIT) {
                q.x[dof] = 0.0;
                if (q.xlo) q.xlo[dof] = 0.f;
                rv = q.b[dof];
                q.r[dof] = rv;
            } else {
                if (q.xlo) {  // restart from the x the check multiplied: x + xlo rounded once
                    q.x[dof] += static_cast<double>(q.xlo[dof]);
                    q.xlo[dof] = 0.f;
                }
                rv = q.r[dof];
            }
            part += rv * rv;
            if (q.cmask[dof]) continue;
            const int co = c * q.nn;
            if (a.XL32) {
                const float f = to_tf32(rv);
                if (s.x >= 0) a.XL32[s.x + co] = f;
                if (s.y >= 0) a.XL32[s.y + co] = f;
                if (s.z >= 0) a.XL32[s.z + co] = f;
                if (s.w >= 0) a.XL32[s.w + co] = f;
            } else {
                rv = round_mantissa(rv, a.round_bits);
                if (s.x >= 0) a.XL[s.x + co] = rv;
                if (s.y >= 0) a.XL[s.y + co] = rv;
                if (s.z >= 0) a.XL[s.z + co] = rv;
                if (s.w >= 0) a.XL[s.w + co] = rv;
            }
        }
    }
    return part;
}

// Loop-head bookkeeping of cg_solve after r.r (one thread): iteration count,
// best iterate, max-iteration exit, next product = A x when the residual
// test passes (linalg.cpp:310-350).
__device__ __forceinline__ void as_update_finish(CgState *st, int phase, double tot) {
    if (phase != PH_NORMAL) st->fresh = 1;  // split loop: p = z next
    if (phase == PH_INIT) {
        st->norm_b = sqrt(tot);
        st->tol_abs = st->tol * st->norm_b;
        st->res = st->norm_b;
        st->best_res = st->res;
        st->best_it = 0;
        st->it = 0;
        if (!isfinite(st->norm_b)) {
            st->done = CG_BREAKDOWN;
            st->breakdown_code = 1;
        } else if (st->norm_b == 0.0) {
            st->done = CG_CONVERGED;
        } else {
            st->y_holds_x = st->res <= st->tol_abs ? 1 : 0;
        }
        if (!(st->verify_margin > 0.0)) st->verify_margin = 1.0;
        st->replacing = st->replaced = 0;
    } else if (phase == PH_RESTART || phase == PH_REPLACE) {
        st->y_holds_x = 0;
    } else {
        st->res = sqrt(tot);
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
                st->y_holds_x = st->res <= st->verify_margin * st->tol_abs ? 1 : 0;
                // Residual replacement (van der Vorst & Ye): once, while the gap between the
                // recursive and the true residual is still far below the residual itself, r is
                // recomputed as b - A x with the search direction kept. What the gap had
                // accumulated from the large early steps is gone, so the A x check at the end
                // passes at the first try instead of restarting CG.
                if (!st->y_holds_x && st->replace_at > 0.0 && !st->replaced && st->res <= st->replace_at * st->norm_b) {
                    st->y_holds_x = 1;
                    st->replacing = 1;
                }
            }
        }
    }
}

__global__ void __launch_bounds__(256) as_update_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double sh[64];
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int phase = st->phase;
    double part[1] = {as_update_nodes(q, a, phase, st->alpha)};
    pdl_trigger();
    block_sum<1>(part, sh);
    if (!publish_partials<1>(part, q.partial, &st->ticket_b)) return;
    double tot[1];
    grid_sum<1>(q.partial, gridDim.x, tot, sh);
    if (threadIdx.x != 0) return;
    st->ticket_b = 0u;
    as_update_finish(st, phase, tot[0]);
    __threadfence();
}

// Gather (A) and update (U') fused across one software grid barrier: the
// p.Ap reduction that alpha needs is finished by the last CTA to arrive,
// which then releases the others (generation counter). Ap stays in L2
// between the halves; one launch and one kernel boundary less per
// iteration. The grid must be co-resident (host: occupancy x SMs), and
// dependents are released only after the barrier (a PDL-launched successor
// cannot take the slots of CTAs that have not arrived yet).
__global__ void __launch_bounds__(256, 8) as_gather_update_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double sh[64];
    __shared__ bool last;
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const unsigned gen = *reinterpret_cast<volatile unsigned *>(&st->bar_gen);
    const int yx = st->y_holds_x;
    double part[1] = {cg_gather_nodes(q, yx)};
    block_sum<1>(part, sh);
    if (threadIdx.x == 0) {
        q.partial[blockIdx.x] = part[0];
        __threadfence();
        last = atomicAdd(&st->ticket_a, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double tot[1];
        grid_sum<1>(q.partial, gridDim.x, tot, sh);
        if (threadIdx.x == 0) {
            st->ticket_a = 0u;
            cg_gather_finish(st, yx, tot[0]);
            __threadfence();
            atomicExch(&st->bar_gen, gen + 1u);
        }
    } else if (threadIdx.x == 0) {
        while (*reinterpret_cast<volatile unsigned *>(&st->bar_gen) == gen) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();
    pdl_trigger();
    if (*reinterpret_cast<volatile int *>(&st->done)) return;  // breakdown or converged (verification)
    const int phase = *reinterpret_cast<volatile int *>(&st->phase);
    const double alpha = *reinterpret_cast<volatile double *>(&st->alpha);
    part[0] = as_update_nodes(q, a, phase, alpha);
    block_sum<1>(part, sh);
    if (!publish_partials<1>(part, q.partial + gridDim.x, &st->ticket_b)) return;
    double tot[1];
    grid_sum<1>(q.partial + gridDim.x, gridDim.x, tot, sh);
    if (threadIdx.x != 0) return;
    st->ticket_b = 0u;
    as_update_finish(st, phase, tot[0]);
    __threadfence();
}

// Restriction, one CTA per super cell over its contiguous node range: the
// cell's 24 partials of P^T r.
// One CTA per coarse cell, kRestrictGroup threads per displacement component
// (thread group c accumulates the 8 corner sums of component c: 8 registers
// instead of 24, so more warps stay resident in this latency-bound pass).
constexpr int kRestrictGroup = 128;
__global__ void __launch_bounds__(3 * kRestrictGroup) as_restrict_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double sh[3 * kRestrictGroup / 32][8];
    if (*reinterpret_cast<volatile int *>(&q.st->done)) return;
    const int N = q.n_nodes;
    const int cell = blockIdx.x / kAsSplit;
    const AsCell cc = as_cell(a, cell);
    int nb, ne;
    as_part_range(a, cell, blockIdx.x % kAsSplit, nb, ne);
    const int c = threadIdx.x / kRestrictGroup, lt = threadIdx.x % kRestrictGroup;
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0;
    // early coarse chain: A p in a NORMAL phase (rc recurrence), else r
    const double *src = (a.rc_recur && q.st->phase == PH_NORMAL) ? q.ap : q.r;
    for (int node = nb + lt; node < ne; node += kRestrictGroup) {
        const long long dof = static_cast<long long>(c) * N + node;
        const double r0 = __ldg(src + dof);  // loaded unconditionally: no cmask -> r dependency
        const double rv = __ldg(q.cmask + dof) ? 0.0 : r0;
        double w[8];
        as_cell_weights(a, cc, node, w);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += w[k] * rv;
    }
    pdl_trigger();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const double v = warp_sum(acc[k]);
        if (lane == 0) sh[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 24) {  // entry 3 k + c: component c's warps, in order
        const int k = threadIdx.x / 3, cc2 = threadIdx.x % 3;
        constexpr int wpg = kRestrictGroup / 32;
        double t = 0.0;
        for (int w2 = 0; w2 < wpg; ++w2) t += sh[cc2 * wpg + w2][k];
        a.cellpart[blockIdx.x * 24 + threadIdx.x] = t;  // [cell][part][24]
    }
}

// Restriction with one warp per coarse cell (8 cells per CTA): a lane
// walks its cell's contiguous node range with stride 32 and keeps all 24
// weighted sums (3 components x 8 corners); one warp reduction per sum.
// A single wave of short-lived warps instead of thousands of CTAs whose
// block reductions dominate (as_restrict_kernel); TSV_AS_RESTRICT_CTA=1
// keeps the CTA-per-cell kernel.
#ifndef TSV_RESTRICT_WARPS
#define TSV_RESTRICT_WARPS 8
#endif
constexpr int kRestrictWarps = TSV_RESTRICT_WARPS;
__global__ void __launch_bounds__(32 * kRestrictWarps) as_restrict_warp_kernel(CgParams q, AsParams a) {
    pdl_wait();
    if (*reinterpret_cast<volatile int *>(&q.st->done)) return;
    const int N = q.n_nodes;
    const int lane = threadIdx.x & 31;
    const int cell = blockIdx.x * kRestrictWarps + (threadIdx.x >> 5);
    if (cell >= a.ncells) return;
    const AsCell cc = as_cell(a, cell);
    const int nb = a.cell_ptr[cell], ne = a.cell_ptr[cell + 1];
    const double *src = (a.rc_recur && q.st->phase == PH_NORMAL) ? q.ap : q.r;
    double acc[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[c][k] = 0.0;
#pragma unroll 2
    for (int node = nb + lane; node < ne; node += 32) {
        double rv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            const double r0 = __ldg(src + dof);
            rv[c] = __ldg(q.cmask + dof) ? 0.0 : r0;
        }
        double w[8];
        as_cell_weights(a, cc, node, w);
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c][k] += w[k] * rv[c];
    }
    pdl_trigger();
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double v = warp_sum(acc[c][k]);
            if (lane == 3 * k + c) a.cellpart[cell * 24 + 3 * k + c] = v;
        }
}

// Coarse right-hand side: each coarse DoF sums its (up to 4) cells in order.
__global__ void as_coarse_rhs_kernel(CgParams q, AsParams a) {
    pdl_wait();
    if (*reinterpret_cast<volatile int *>(&q.st->done)) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.Nc) return;
    const int comp = j % 3, cn = j / 3;
    const int nxn = a.SX + 1, nyn = a.SY + 1;
    const int gx = cn % nxn, gy = (cn / nxn) % nyn, gz = cn / (nxn * nyn);
    double s = 0.0;
    for (int cy = gy - 1; cy <= gy; ++cy) {
        if (cy < 0 || cy >= a.SY) continue;
        for (int cx = gx - 1; cx <= gx; ++cx) {
            if (cx < 0 || cx >= a.SX) continue;
            const int corner = (gx - cx) | ((gy - cy) << 1) | (gz << 2);
            for (int part = 0; part < kAsSplit; ++part)
                s += a.cellpart[((cy * a.SX + cx) * kAsSplit + part) * 24 + 3 * corner + comp];
        }
    }
    if (a.rc_recur && q.st->phase == PH_NORMAL)
        a.rc[j] -= q.st->alpha * s;  // P^T r' = P^T r - alpha P^T (A p)
    else
        a.rc[j] = s;
}

// Coarse solve zc = A_c^-1 rc (fixed-order reductions): a CTA of 8 warps
// computes 16 rows, 2 per warp, over rc chunks staged in shared memory (the
// rows re-read rc from shared memory, not L2). FP32 matrix by default.
constexpr int kGemvRows = 16;
constexpr int kGemvChunk = 2048;

__global__ void __launch_bounds__(256) as_coarse_gemv_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double rcs[kGemvChunk];
    if (*reinterpret_cast<volatile int *>(&q.st->done)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = blockIdx.x * kGemvRows + 2 * warp;
    const bool v0 = r0 < a.Nc, v1 = r0 + 1 < a.Nc;
    double s0 = 0.0, s1 = 0.0;
    for (int c0 = 0; c0 < a.Nc; c0 += kGemvChunk) {
        const int len = min(kGemvChunk, a.Nc - c0);
        __syncthreads();
        for (int i = threadIdx.x; i < kGemvChunk; i += blockDim.x) rcs[i] = i < len ? a.rc[c0 + i] : 0.0;
        __syncthreads();
        if (a.ainv_c32) {
            const int n4 = (len + 3) >> 2;  // rows are zero-padded to ldc32
            const float4 *m0 = reinterpret_cast<const float4 *>(a.ainv_c32 + static_cast<long long>(v0 ? r0 : 0) * a.ldc32 + c0);
            const float4 *m1 = reinterpret_cast<const float4 *>(a.ainv_c32 + static_cast<long long>(v1 ? r0 + 1 : 0) * a.ldc32 + c0);
            for (int j = lane; j < n4; j += 32) {
                const float4 x0 = __ldcs(m0 + j), x1 = __ldcs(m1 + j);
                const double4 rv = make_double4(rcs[4 * j], rcs[4 * j + 1], rcs[4 * j + 2], rcs[4 * j + 3]);
                s0 += static_cast<double>(x0.x) * rv.x + static_cast<double>(x0.y) * rv.y + static_cast<double>(x0.z) * rv.z +
                      static_cast<double>(x0.w) * rv.w;
                s1 += static_cast<double>(x1.x) * rv.x + static_cast<double>(x1.y) * rv.y + static_cast<double>(x1.z) * rv.z +
                      static_cast<double>(x1.w) * rv.w;
            }
        } else {
            const double *m0 = a.ainv_c + static_cast<long long>(v0 ? r0 : 0) * a.Nc + c0;
            const double *m1 = a.ainv_c + static_cast<long long>(v1 ? r0 + 1 : 0) * a.Nc + c0;
            for (int j = lane; j < len; j += 32) {
                s0 += m0[j] * rcs[j];
                s1 += m1[j] * rcs[j];
            }
        }
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
        if (v0) a.zc[r0] = s0;
        if (v1) a.zc[r0 + 1] = s1;
    }
}

// Coarse solve on the packed lower triangle of the symmetric FP32 inverse
// (half the HBM stream of the dense GEMV). Tile (I, J), I >= J, of
// kSymT x kSymT is stored contiguously; its CTA writes the partial
// A_IJ rc_J to part[I][J] and (I != J) A_IJ^T rc_I to part[J][I]; the
// reduction sums part[I][0..NT) in order (fixed order: deterministic).
constexpr int kSymT = 64;

__device__ __forceinline__ void sym_tile_of(int t, int &I, int &J) {
    // t enumerates lower tiles row by row: t = I (I + 1) / 2 + J
    I = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    J = t - I * (I + 1) / 2;
}

__global__ void __launch_bounds__(128) as_coarse_symv_kernel(CgParams q, AsParams a, const float *tiles, int NT,
                                                             double *part) {
    pdl_wait();
    __shared__ double xi[kSymT], xj[kSymT];
    __shared__ double colp[8][kSymT];
    if (*reinterpret_cast<volatile int *>(&q.st->done)) return;
    int I, J;
    sym_tile_of(blockIdx.x, I, J);
    const int t = threadIdx.x;
    if (t < kSymT) {
        const int gi = I * kSymT + t, gj = J * kSymT + t;
        xi[t] = gi < a.Nc ? a.rc[gi] : 0.0;
        xj[t] = gj < a.Nc ? a.rc[gj] : 0.0;
    }
    // thread t holds rows t/16 + 8k (k = 0..7), columns 4 (t % 16) .. + 3
    const float4 *src = reinterpret_cast<const float4 *>(tiles + static_cast<long long>(blockIdx.x) * kSymT * kSymT);
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(src + t + 128 * k);
    __syncthreads();
    const int c0 = 4 * (t & 15), r0 = t >> 4;
    double cs[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int row = r0 + 8 * k;
        double rs = static_cast<double>(v[k].x) * xj[c0] + static_cast<double>(v[k].y) * xj[c0 + 1] +
                    static_cast<double>(v[k].z) * xj[c0 + 2] + static_cast<double>(v[k].w) * xj[c0 + 3];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);  // 16 lanes share a row
        if ((t & 15) == 0) part[(static_cast<long long>(I) * NT + J) * kSymT + row] = rs;
        const double xr = xi[row];
        cs[0] += static_cast<double>(v[k].x) * xr;
        cs[1] += static_cast<double>(v[k].y) * xr;
        cs[2] += static_cast<double>(v[k].z) * xr;
        cs[3] += static_cast<double>(v[k].w) * xr;
    }
    if (I == J) return;
    // column sums: reduce over the 8 row groups r0 (lanes 16 apart, then warps)
#pragma unroll
    for (int c = 0; c < 4; ++c) cs[c] += __shfl_xor_sync(0xffffffffu, cs[c], 16);
    const int warp = t >> 5;
    if ((t & 16) == 0)
#pragma unroll
        for (int c = 0; c < 4; ++c) colp[warp][c0 + c] = cs[c];
    __syncthreads();
    if (t < kSymT) {
        const double s = (colp[0][t] + colp[1][t]) + (colp[2][t] + colp[3][t]);
        part[(static_cast<long long>(J) * NT + I) * kSymT + t] = s;
    }
}

// zc[I*T + r] = sum_J part[I][J][r], J in order: a CTA of 16 x 64 threads per
// block row I; thread group g sums J = g, g + 16, ... and the 16 group sums
// are added in group order (fixed order: deterministic).
constexpr int kSymRedG = 16;
__global__ void __launch_bounds__(kSymRedG * kSymT) as_coarse_symv_reduce_kernel(CgParams q, AsParams a, int NT,
                                                                               const double *part) {
    pdl_wait();
    __shared__ double sh[kSymRedG][kSymT];
    __shared__ double shd[64];
    if (*reinterpret_cast<volatile int *>(&q.st->done)) return;
    const int I = blockIdx.x, r = threadIdx.x % kSymT, grp = threadIdx.x / kSymT;
    double s = 0.0;
    for (int J = grp; J < NT; J += kSymRedG) s += part[(static_cast<long long>(I) * NT + J) * kSymT + r];
    sh[grp][r] = s;
    __syncthreads();
    // rc.zc folded in: this block row's partial, then the last CTA (ticket_c)
    // sums the partials in CTA order
    double d[1] = {0.0};
    if (grp == 0) {
        double t = 0.0;
#pragma unroll
        for (int g = 0; g < kSymRedG; ++g) t += sh[g][r];
        const int i = I * kSymT + r;
        if (i < a.Nc) {
            a.zc[i] = t;
            d[0] = a.rc[i] * t;
        }
    }
    block_sum<1>(d, shd);
    if (!publish_partials<1>(d, a.dotpart, &q.st->ticket_c)) return;
    double tot[1];
    grid_sum<1>(a.dotpart, gridDim.x, tot, shd);
    if (threadIdx.x == 0) {
        q.st->ticket_c = 0u;
        q.st->rz_c = tot[0];
        __threadfence();
    }
}

// Pack the lower tiles of the full symmetric FP64 inverse (column-major) as FP32.
__global__ void as_pack_sym_tiles_kernel(const double *A, int Nc, float *tiles, long long total) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int t = static_cast<int>(e / (kSymT * kSymT)), w = static_cast<int>(e % (kSymT * kSymT));
    int I, J;
    sym_tile_of(t, I, J);
    const int row = I * kSymT + w / kSymT, col = J * kSymT + w % kSymT;
    tiles[e] = (row < Nc && col < Nc) ? static_cast<float>(A[static_cast<long long>(col) * Nc + row]) : 0.0f;
}

// The preconditioned residual is z = z_l + P zc, with z_l the local part
// (owner gather of the local products; z = r on constrained DoFs) and P zc
// the coarse part (free DoFs). Since P^T r (free DoFs) is the coarse
// right-hand side rc, r.z = r.z_l + rc.zc: the local kernel (as_zl) runs on
// the main stream while the coarse chain finishes on the side stream, and
// the coarse part is added where z is consumed (as_scatter_kernel).

// z_l and r.z_l (grid-stride, fixed grid; the last CTA stores rz_l).
__global__ void __launch_bounds__(256) as_zl_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double sh[64];
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int N = q.n_nodes;
    double part[1] = {0.0};
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
        const int4 s = reinterpret_cast<const int4 *>(a.slots2)[node];
        if (a.ZL32) {
            // the hot path with the loads of all three components ahead of the stores; same sums, same order
            double rr[3];
            float zl[3][4];
            uint8_t cm[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const long long dof = static_cast<long long>(c) * N + node;
                const int co = c * q.nn;
                rr[c] = q.r[dof];
                cm[c] = q.cmask[dof];
                zl[c][0] = s.x >= 0 ? a.ZL32[s.x + co] : 0.f;
                zl[c][1] = s.y >= 0 ? a.ZL32[s.y + co] : 0.f;
                zl[c][2] = s.z >= 0 ? a.ZL32[s.z + co] : 0.f;
                zl[c][3] = s.w >= 0 ? a.ZL32[s.w + co] : 0.f;
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const long long dof = static_cast<long long>(c) * N + node;
                const double zv = cm[c] ? rr[c]
                                        : (((0.0 + static_cast<double>(zl[c][0])) + static_cast<double>(zl[c][1])) +
                                           static_cast<double>(zl[c][2])) + static_cast<double>(zl[c][3]);
                a.z[dof] = zv;
                part[0] += rr[c] * zv;
            }
            continue;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            const double rv = q.r[dof];
            double zv;
            if (q.cmask[dof]) {
                zv = rv;  // unit row of the lifted matrix
            } else {
                const int co = c * q.nn;
                zv = 0.0;
                if (a.ZL32) {
                    if (s.x >= 0) zv += static_cast<double>(a.ZL32[s.x + co]);
                    if (s.y >= 0) zv += static_cast<double>(a.ZL32[s.y + co]);
                    if (s.z >= 0) zv += static_cast<double>(a.ZL32[s.z + co]);
                    if (s.w >= 0) zv += static_cast<double>(a.ZL32[s.w + co]);
                } else {
                    if (s.x >= 0) zv += a.ZL[s.x + co];
                    if (s.y >= 0) zv += a.ZL[s.y + co];
                    if (s.z >= 0) zv += a.ZL[s.z + co];
                    if (s.w >= 0) zv += a.ZL[s.w + co];
                }
            }
            a.z[dof] = zv;
            part[0] += rv * zv;
        }
    }
    pdl_trigger();
    block_sum<1>(part, sh);
    if (!publish_partials<1>(part, q.partial, &st->ticket_a)) return;
    double tot[1];
    grid_sum<1>(q.partial, gridDim.x, tot, sh);
    if (threadIdx.x != 0) return;
    st->ticket_a = 0u;
    st->rz_l = tot[0];
    __threadfence();
}

// rc.zc on the side stream (one CTA, fixed order).
__global__ void __launch_bounds__(1024) as_coarse_dot_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double sh[64];
    if (*reinterpret_cast<volatile int *>(&q.st->done)) return;
    double v[1] = {0.0};
    for (int i = threadIdx.x; i < a.Nc; i += blockDim.x) v[0] += a.rc[i] * a.zc[i];
    block_sum<1>(v, sh);
    if (threadIdx.x == 0) q.st->rz_c = v[0];
}

// p = z + beta p (or p = z after init/restart) with z = z_l + P zc, beta =
// (rz_l + rz_c) / rho; the next operator operand (p, or x for a
// verification) goes into the block-major panel (free DoFs). The last CTA
// advances rho / phase. With write_z (tsv_precond_apply) z is stored too.
__global__ void __launch_bounds__(256) as_scatter_kernel(CgParams q, AsParams a, int write_z) {
    pdl_wait();
    __shared__ bool last;
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int yx = st->y_holds_x;
    // a residual replacement is about to multiply x: p, rho and the phase stay as they are
    // (the direction is updated from the replaced residual in the next pass)
    const bool hold = yx && st->replacing;
    const bool normal = st->phase == PH_NORMAL || st->phase == PH_REPLACE;
    const double rz = st->rz_l + st->rz_c;
    const double beta = normal ? rz / st->rho : 0.0;
    const int N = q.n_nodes;
    const double rdz = 1.0 / static_cast<double>(a.qm1);
    if (hold) {
        for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
            const int4 s = reinterpret_cast<const int4 *>(q.slots)[node];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const long long dof = static_cast<long long>(c) * N + node;
                if (q.cmask[dof]) continue;
                const double v = q.xlo ? q.x[dof] + static_cast<double>(q.xlo[dof]) : q.x[dof];
                const int co = c * q.nn;
                if (s.x >= 0) q.X[s.x + co] = v;
                if (s.y >= 0) q.X[s.y + co] = v;
                if (s.z >= 0) q.X[s.z + co] = v;
                if (s.w >= 0) q.X[s.w + co] = v;
            }
        }
        return;
    }
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
        const int cell = a.node_cell[node];
        const double4 ct = a.celltab[cell];
        const short4 L = a.lat[node];
        const double tx = (static_cast<double>(L.x) - ct.x) * ct.z;
        const double ty = (static_cast<double>(L.y) - ct.y) * ct.w;
        const double tz = static_cast<double>(L.z) * rdz;
        const int cx = cell % a.SX, cy = cell / a.SX;
        const int4 s = reinterpret_cast<const int4 *>(q.slots)[node];
        // loads of all three components ahead of the stores (the compiler cannot hoist them itself)
        double zl3[3], pold[3], xv3[3];
        uint8_t cm3[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            zl3[c] = a.z[dof];
            cm3[c] = q.cmask[dof];
            pold[c] = normal ? q.p[dof] : 0.0;
            xv3[c] = yx ? (q.xlo ? q.x[dof] + static_cast<double>(q.xlo[dof]) : q.x[dof]) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            double zv = zl3[c];
            const bool cm = cm3[c] != 0;
            double zcoarse = 0.0;  // computed whether or not the DoF is constrained (no cmask -> zc dependency)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double w = ((k & 1) ? tx : 1.0 - tx) * ((k & 2) ? ty : 1.0 - ty) * ((k & 4) ? tz : 1.0 - tz);
                zcoarse += w * __ldg(a.zc + 3 * as_corner_node(a, cx, cy, k) + c);
            }
            if (!cm) zv += zcoarse;
            if (write_z) a.z[dof] = zv;
            const double pn = normal ? zv + beta * pold[c] : zv;
            q.p[dof] = pn;
            if (cm) continue;
            const double v = yx ? xv3[c] : pn;
            const int co = c * q.nn;
            if (s.x >= 0) q.X[s.x + co] = v;
            if (s.y >= 0) q.X[s.y + co] = v;
            if (s.z >= 0) q.X[s.z + co] = v;
            if (s.w >= 0) q.X[s.w + co] = v;
        }
    }
    pdl_trigger();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&st->ticket_b, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    st->ticket_b = 0u;
    if (normal) {
        st->beta = beta;
        st->p_assign = 0;
        st->phase = PH_NORMAL;
    } else {
        st->p_assign = 1;
        st->phase = PH_NORMAL;
    }
    st->rho = rz;
    __threadfence();
}

// ------------------------------------------------------------------------
// Split two-level Schwarz loop. With z = z_l + P zc, the next operator
// product is formed as
//     A p = A z_l + A P zc + beta A p_old,   p = z_l + P zc + beta p_old,
// so K1 multiplies the local part z_l (ready right after the tensor-core
// local solves) while the coarse chain (restriction, coarse solve, and
// A P zc = sum_b G_b^T (K_b P_b) zc_b) runs beside it on the side stream
// instead of in front of it. The reference's control flow is unchanged: the
// same stopping test, true-residual verification (K1 on x) and restart.
// Per iteration: GU (gather + p/Ap recurrences | grid barrier | x, r update)
// -> {coarse chain} || {tc local solve -> z_l (+ X panel) -> K1} -> join.

// z_l = sum of the node's local products (r on constrained DoFs), r.z_l,
// and the next K1 operand: z_l (or x when verifying) into the X panel.
__global__ void __launch_bounds__(256) as_zl_split_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double sh[64];
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int yx = st->y_holds_x;
    const int N = q.n_nodes;
    double part[1] = {0.0};
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
        const int4 s2 = reinterpret_cast<const int4 *>(a.slots2)[node];
        const int4 s = reinterpret_cast<const int4 *>(q.slots)[node];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            const double rv = q.r[dof];
            const bool cm = q.cmask[dof] != 0;
            const int co = c * q.nn;
            double zv;
            if (cm) {
                zv = rv;  // unit row of the lifted matrix
            } else if (a.ZL32) {
                zv = 0.0;
                if (s2.x >= 0) zv += static_cast<double>(a.ZL32[s2.x + co]);
                if (s2.y >= 0) zv += static_cast<double>(a.ZL32[s2.y + co]);
                if (s2.z >= 0) zv += static_cast<double>(a.ZL32[s2.z + co]);
                if (s2.w >= 0) zv += static_cast<double>(a.ZL32[s2.w + co]);
            } else {
                zv = 0.0;
                if (s2.x >= 0) zv += a.ZL[s2.x + co];
                if (s2.y >= 0) zv += a.ZL[s2.y + co];
                if (s2.z >= 0) zv += a.ZL[s2.z + co];
                if (s2.w >= 0) zv += a.ZL[s2.w + co];
            }
            a.z[dof] = zv;
            part[0] += rv * zv;
            if (cm) continue;
            const double v = yx ? (q.xlo ? q.x[dof] + static_cast<double>(q.xlo[dof]) : q.x[dof]) : zv;
            if (s.x >= 0) q.X[s.x + co] = v;
            if (s.y >= 0) q.X[s.y + co] = v;
            if (s.z >= 0) q.X[s.z + co] = v;
            if (s.w >= 0) q.X[s.w + co] = v;
        }
    }
    pdl_trigger();
    block_sum<1>(part, sh);
    if (!publish_partials<1>(part, q.partial, &st->ticket_a)) return;
    double tot[1];
    grid_sum<1>(q.partial, gridDim.x, tot, sh);
    if (threadIdx.x != 0) return;
    st->ticket_a = 0u;
    st->rz_l = tot[0];
    __threadfence();
}

// A P zc per block: Yc[row] = (K_b P_b) zc_cell(b). CTA = (key chunk of up
// to kKpzcChunk blocks, slice of kKpzcRows panel columns); each thread keeps
// one row of the key's n x 24 product in registers and walks the chunk's
// blocks (their 24 coarse values broadcast from shared memory); the Yc row
// writes are coalesced. Side stream, after the coarse solve.
constexpr int kKpzcRows = 128;
__global__ void __launch_bounds__(kKpzcRows) as_kpzc_kernel(CgParams q, AsParams a, KpzcParams k) {
    pdl_wait();
    __shared__ double zcs[kKpzcChunk][24];
    __shared__ int rows[kKpzcChunk];
    if (*reinterpret_cast<volatile int *>(&q.st->done)) return;
    const int4 it = k.items[blockIdx.x];
    const int nb = it.z - it.y;
    for (int i = threadIdx.x; i < nb * 24; i += blockDim.x) {
        const int bi = i / 24, j = i % 24;
        const int row = k.rows[it.y + bi];
        const int cell = k.row_cell[row];
        const int cx = (cell % k.cols) / k.sb, cy = (cell / k.cols) / k.sb;
        zcs[bi][j] = a.zc[3 * as_corner_node(a, cx, cy, j / 3) + j % 3];
        if (j == 0) rows[bi] = row;
    }
    const int r = blockIdx.y * kKpzcRows + threadIdx.x;
    double kr[24];
    if (r < k.n) {
        const double2 *src = reinterpret_cast<const double2 *>(k.kp + (static_cast<long long>(it.x) * k.ldk + r) * 24);
#pragma unroll
        for (int j = 0; j < 12; ++j) {
            const double2 v = __ldg(src + j);
            kr[2 * j] = v.x;
            kr[2 * j + 1] = v.y;
        }
    }
    __syncthreads();
    pdl_trigger();
    if (r >= k.n) return;
    for (int bi = 0; bi < nb; ++bi) {
        double y = 0.0;
#pragma unroll
        for (int j = 0; j < 24; ++j) y += kr[j] * zcs[bi][j];
        a.Yc[static_cast<long long>(rows[bi]) * k.ldk + r] = y;
    }
}

// Node loop of GU's first half: p = z_l + P zc + beta p, A p = sum(Y) +
// sum(Yc) + beta A p (unit rows on constrained DoFs), returns p.Ap; or,
// verifying, r = b - A x, returns r.r.
__device__ __forceinline__ double as_gu_nodes(const CgParams &q, const AsParams &a, int yx, bool fresh, double beta) {
    if (yx) return cg_gather_nodes(q, 1);
    const int N = q.n_nodes;
    const double rdz = 1.0 / static_cast<double>(a.qm1);
    double part = 0.0;
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < N; node += gridDim.x * blockDim.x) {
        const int cell = a.node_cell[node];
        const double4 ct = a.celltab[cell];
        const short4 L = a.lat[node];
        const double tx = (static_cast<double>(L.x) - ct.x) * ct.z;
        const double ty = (static_cast<double>(L.y) - ct.y) * ct.w;
        const double tz = static_cast<double>(L.z) * rdz;
        const int cx = cell % a.SX, cy = cell / a.SX;
        const int4 s = reinterpret_cast<const int4 *>(q.slots)[node];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const long long dof = static_cast<long long>(c) * N + node;
            const int co = c * q.nn;
            const double zl = a.z[dof];
            double zv = zl, az;
            if (q.cmask[dof]) {
                az = zl;  // unit row: (A z)_c = z_c
            } else {
                az = 0.0;
                if (s.x >= 0) az += q.Y[s.x + co] + a.Yc[s.x + co];
                if (s.y >= 0) az += q.Y[s.y + co] + a.Yc[s.y + co];
                if (s.z >= 0) az += q.Y[s.z + co] + a.Yc[s.z + co];
                if (s.w >= 0) az += q.Y[s.w + co] + a.Yc[s.w + co];
                double zcoarse = 0.0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double w = ((k & 1) ? tx : 1.0 - tx) * ((k & 2) ? ty : 1.0 - ty) * ((k & 4) ? tz : 1.0 - tz);
                    zcoarse += w * __ldg(a.zc + 3 * as_corner_node(a, cx, cy, k) + c);
                }
                zv += zcoarse;
            }
            const double pn = fresh ? zv : zv + beta * q.p[dof];
            const double apn = fresh ? az : az + beta * q.ap[dof];
            q.p[dof] = pn;
            q.ap[dof] = apn;
            part += pn * apn;
        }
    }
    return part;
}

// G' alone (the update follows as as_update_kernel): p, Ap recurrences and
// p.Ap (or the true residual); the last CTA stores rho, beta and alpha.
__global__ void __launch_bounds__(256, 4) as_g_split_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double sh[64];
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int yx = st->y_holds_x;
    const bool fresh = st->fresh != 0;
    const double rz = st->rz_l + st->rz_c;
    const double beta = fresh ? 0.0 : rz / st->rho;
    double part[1] = {as_gu_nodes(q, a, yx, fresh, beta)};
    pdl_trigger();
    block_sum<1>(part, sh);
    if (!publish_partials<1>(part, q.partial, &st->ticket_a)) return;
    double tot[1];
    grid_sum<1>(q.partial, gridDim.x, tot, sh);
    if (threadIdx.x != 0) return;
    st->ticket_a = 0u;
    if (!yx) {
        st->rho = rz;
        st->fresh = 0;
        st->beta = beta;
    }
    cg_gather_finish(st, yx, tot[0]);
    __threadfence();
}

// GU: the gather half (p, Ap recurrences and p.Ap; or the true residual)
// and the update half (x, r, XL32 panel, r.r, loop head) across one
// software grid barrier. The grid must be co-resident (host: occupancy x
// SMs); dependents are released only after the barrier.
__global__ void __launch_bounds__(256) as_gu_split_kernel(CgParams q, AsParams a) {
    pdl_wait();
    __shared__ double sh[64];
    __shared__ bool last;
    CgState *st = q.st;
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const unsigned gen = *reinterpret_cast<volatile unsigned *>(&st->bar_gen);
    const int yx = st->y_holds_x;
    const bool fresh = st->fresh != 0;
    const double rz = st->rz_l + st->rz_c;
    const double beta = fresh ? 0.0 : rz / st->rho;
    double part[1] = {as_gu_nodes(q, a, yx, fresh, beta)};
    block_sum<1>(part, sh);
    if (threadIdx.x == 0) {
        q.partial[blockIdx.x] = part[0];
        __threadfence();
        last = atomicAdd(&st->ticket_a, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double tot[1];
        grid_sum<1>(q.partial, gridDim.x, tot, sh);
        if (threadIdx.x == 0) {
            st->ticket_a = 0u;
            if (!yx) {
                st->rho = rz;  // r.z of the current residual
                st->fresh = 0;
                st->beta = beta;
            }
            cg_gather_finish(st, yx, tot[0]);
            __threadfence();
            atomicExch(&st->bar_gen, gen + 1u);
        }
    } else if (threadIdx.x == 0) {
        while (*reinterpret_cast<volatile unsigned *>(&st->bar_gen) == gen) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();
    pdl_trigger();
    if (*reinterpret_cast<volatile int *>(&st->done)) return;
    const int phase = *reinterpret_cast<volatile int *>(&st->phase);
    const double alpha = *reinterpret_cast<volatile double *>(&st->alpha);
    part[0] = as_update_nodes(q, a, phase, alpha);
    block_sum<1>(part, sh);
    if (!publish_partials<1>(part, q.partial + gridDim.x, &st->ticket_b)) return;
    double tot[1];
    grid_sum<1>(q.partial + gridDim.x, gridDim.x, tot, sh);
    if (threadIdx.x != 0) return;
    st->ticket_b = 0u;
    as_update_finish(st, phase, tot[0]);
    __threadfence();
}

}  // namespace tsvb200

namespace tsvb200 {

// ---------------------------------------------------------------- setup
// potri leaves the inverse in the lower triangle (column-major); write the
// full symmetric matrix in the permuted, padded GEMM layout
// dst[pidx(a) * ldk + pidx(k)], pidx(3 rank + c) = c nn + rank.
__global__ void as_pack_inverse_kernel(const double *inv, int n, int nn, int ldk, double *dst, int round_bits) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<long long>(n) * n) return;
    const int a = static_cast<int>(t / n), k = static_cast<int>(t % n);
    const double v = a >= k ? inv[static_cast<long long>(k) * n + a] : inv[static_cast<long long>(a) * n + k];
    dst[static_cast<long long>((a % 3) * nn + a / 3) * ldk + (k % 3) * nn + k / 3] = round_mantissa(v, round_bits);
}

// Dense coarse matrix (column-major), one colour of super cells at a time
// (cells of equal (cx, cy) parity share no corner, so no write conflicts).
__global__ void as_coarse_scatter_kernel(const double *kc_cell, int SX, int SY, int px, int py, double *Ac, int Nc) {
    const int ncx = (SX - px + 1) / 2, ncy = (SY - py + 1) / 2;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<long long>(ncx) * ncy * 576) return;
    const int e = static_cast<int>(t % 576);
    const long long cid = t / 576;
    const int cx = px + 2 * static_cast<int>(cid % ncx), cy = py + 2 * static_cast<int>(cid / ncx);
    const int i = e % 24, j = e / 24;
    auto cdof = [&](int k) {
        const int c = k / 3, comp = k % 3;
        const int node = (((c >> 2) & 1) * (SY + 1) + cy + ((c >> 1) & 1)) * (SX + 1) + cx + (c & 1);
        return 3 * node + comp;
    };
    Ac[static_cast<long long>(cdof(j)) * Nc + cdof(i)] += kc_cell[(static_cast<long long>(cy) * SX + cx) * 576 + e];
}

// Coarse DoFs with no free fine support get a unit diagonal (decoupled).
__global__ void as_fix_zero_rows_kernel(double *Ac, int Nc) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= Nc) return;
    bool nz = false;
    for (int j = lane; j < Nc && !nz; j += 32) nz = Ac[static_cast<long long>(row) * Nc + j] != 0.0;
    nz = __any_sync(0xffffffffu, nz);
    if (!nz && lane == 0) Ac[static_cast<long long>(row) * Nc + row] = 1.0;
}

// FP32 copy of the coarse inverse, rows padded to ld.
__global__ void as_coarse_to_f32_kernel(const double *A, int Nc, int ld, float *dst) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<long long>(Nc) * ld) return;
    const int row = static_cast<int>(t / ld), col = static_cast<int>(t % ld);
    dst[t] = col < Nc ? static_cast<float>(A[static_cast<long long>(row) * Nc + col]) : 0.0f;
}

// Lower triangle -> full symmetric (column-major).
__global__ void as_symmetrize_kernel(double *A, int Nc) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<long long>(Nc) * Nc) return;
    const int col = static_cast<int>(t / Nc), row = static_cast<int>(t % Nc);
    if (row < col) A[t] = A[static_cast<long long>(row) * Nc + col];
}

// x += xlo, xlo = 0 (end of a solve with the compensated x).
__global__ void fold_x_kernel(double *x, float *xlo, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        x[i] += static_cast<double>(xlo[i]);
        xlo[i] = 0.f;
    }
}

}  // namespace tsvb200
