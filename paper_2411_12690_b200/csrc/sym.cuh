// Mirror-symmetric macro-elements (symmetry.hpp): the operand panels are taken
// to the symmetry-adapted basis by a Walsh-Hadamard pass over the mirror
// orbits of each row, the dense FP64 contractions run as 8 independent
// (irrep) GEMMs with 1/8 of the FLOPs, and the products are taken back.
//
//   sym_fwd_kernel    X  [rows][ldx]  -> Xs [rows][lds]  (irrep-segmented)
//                     (+ optional TF32 copy of X for the K_r symmetry-defect
//                      correction on the tensor cores, tc_local.cuh)
//   gemm_seg_f64      Ys[:, seg r] = Xs[:, seg r] * K''_r^T   (K1)
//                     Us[:, seg r] = Qs[:, seg r] * Phi''_r^T + dT (H u_T)_r  (K6)
//   sym_bwd_kernel    Ys -> Y  (inverse transform, 1/|orbit|, + correction)
//   sym_fine_kernel   Us -> U  (inverse transform over the fine-DoF orbits)
//
// All butterflies are additions; the scales are powers of two.
#pragma once

#include "kernels.cuh"
#include "symmetry.hpp"

namespace tsvb200 {

constexpr int kSymWarps = 8;

struct SymPanelParams {
    const double *in;   // fwd: plain panel X; bwd: segmented panel Ys
    long long ld_in;
    double *out;        // fwd: segmented panel Xs; bwd: plain panel Y
    long long ld_out;
    int rows;
    int n_plain;        // plain row length processed (ldk, pads zero)
    int n_seg;          // segmented row length (lds)
    const short *src;   // [n_orbits][8] plain columns (-1: absent)
    const short *dst;   // [n_orbits][8] segmented columns
    int n_orbits;
    float *x32;         // fwd, nullable: TF32 copy of the plain row
    const float *c32;   // bwd, nullable: FP32 correction rows (plain layout)
    long long ld32;
    double c_scale;     // bwd: Y += c_scale * c32
    int n_valid;        // plain columns with data (n)
    const int *done;    // nullable CG early exit
};

__device__ __forceinline__ void sym_butterfly(double (&x)[8], int f) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!(f >> a & 1)) continue;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >> a & 1) continue;
            const double lo = x[g], hi = x[g | 1 << a];
            x[g] = lo + hi;
            x[g | 1 << a] = lo - hi;
        }
    }
}

// One warp per row: the row is staged in shared memory (coalesced 16-byte
// loads), each lane transforms whole orbits, the result row is written back
// coalesced. DIR = 0 forward (plain -> segmented), 1 backward.
template <int DIR>
__global__ void __launch_bounds__(32 * kSymWarps) sym_panel_kernel(SymPanelParams p) {
    pdl_wait();
    extern __shared__ __align__(16) double sym_smem[];
    if (p.done != nullptr && *reinterpret_cast<const volatile int *>(p.done) != 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_in = DIR == 0 ? p.n_plain : p.n_seg, n_out = DIR == 0 ? p.n_seg : p.n_plain;
    short *tab = reinterpret_cast<short *>(sym_smem);  // [n_orbits][16]: src[8], dst[8]
    const int tab_doubles = (p.n_orbits * 32 + 15) / 16 * 2;
    double *bin = sym_smem + tab_doubles + static_cast<size_t>(warp) * (n_in + n_out);
    double *bout = bin + n_in;
    for (int i = threadIdx.x; i < p.n_orbits * 8; i += blockDim.x) {
        tab[(i >> 3) * 16 + (i & 7)] = p.src[i];
        tab[(i >> 3) * 16 + 8 + (i & 7)] = p.dst[i];
    }
    for (int i = lane; i < n_out; i += 32) bout[i] = 0.0;  // pads stay zero
    __syncthreads();
    for (int row = blockIdx.x * kSymWarps + warp; row < p.rows; row += gridDim.x * kSymWarps) {
        const double2 *gi = reinterpret_cast<const double2 *>(p.in + static_cast<long long>(row) * p.ld_in);
        for (int i = lane; i < n_in / 2; i += 32) reinterpret_cast<double2 *>(bin)[i] = gi[i];
        __syncwarp();
        if (DIR == 0 && p.x32 != nullptr) {
            float *xr = p.x32 + static_cast<long long>(row) * p.ld32;
            for (int i = lane; i < p.n_valid; i += 32) {
                uint32_t t;
                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(static_cast<float>(bin[i])));
                xr[i] = __uint_as_float(t);
            }
        }
        for (int o = lane; o < p.n_orbits; o += 32) {
            const short *t = tab + o * 16;
            const short *from = DIR == 0 ? t : t + 8, *to = DIR == 0 ? t + 8 : t;
            double x[8];
            int f = 0;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const int c = from[g];
                x[g] = c >= 0 ? bin[c] : 0.0;
                if (c >= 0) f |= g;
            }
            sym_butterfly(x, f);
            double s = 1.0;
            if (DIR == 1) s = f == 7 ? 0.125 : (f == 0 ? 1.0 : ((f & (f - 1)) == 0 ? 0.5 : 0.25));
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const int c = to[g];
                if (c >= 0) bout[c] = DIR == 1 ? s * x[g] : x[g];
            }
        }
        __syncwarp();
        if (DIR == 1 && p.c32 != nullptr) {
            const float *cr = p.c32 + static_cast<long long>(row) * p.ld32;
            for (int i = lane; i < p.n_valid; i += 32) bout[i] += p.c_scale * static_cast<double>(cr[i]);
            __syncwarp();
        }
        double2 *go = reinterpret_cast<double2 *>(p.out + static_cast<long long>(row) * p.ld_out);
        for (int i = lane; i < n_out / 2; i += 32) go[i] = reinterpret_cast<const double2 *>(bout)[i];
        __syncwarp();
    }
    pdl_trigger();
}

inline size_t sym_panel_smem(int n_orbits, int n_plain, int n_seg) {
    const size_t tab_doubles = (static_cast<size_t>(n_orbits) * 32 + 15) / 16 * 2;
    return (tab_doubles + static_cast<size_t>(kSymWarps) * (n_plain + n_seg)) * sizeof(double);
}

// Us -> U over the fine-DoF orbits: thread = (orbit, group of kFineRows rows).
constexpr int kFineRows = 8;
struct SymFineParams {
    const double *Us;
    long long ldus;
    double *U;
    long long ldu;
    int rows;
    const int *src;  // [n_orbits][8] fine DoF (column of U) of member g (-1: absent)
    const int *dst;  // [n_orbits][8] column of Us of combination g
    int n_orbits;
};

__global__ void __launch_bounds__(256) sym_fine_kernel(SymFineParams p) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= p.n_orbits) return;
    int s[8], t[8], f = 0;
    {
        const int4 *sp = reinterpret_cast<const int4 *>(p.src + static_cast<long long>(o) * 8);
        const int4 *tp = reinterpret_cast<const int4 *>(p.dst + static_cast<long long>(o) * 8);
        const int4 a = sp[0], b = sp[1], c = tp[0], d = tp[1];
        s[0] = a.x, s[1] = a.y, s[2] = a.z, s[3] = a.w, s[4] = b.x, s[5] = b.y, s[6] = b.z, s[7] = b.w;
        t[0] = c.x, t[1] = c.y, t[2] = c.z, t[3] = c.w, t[4] = d.x, t[5] = d.y, t[6] = d.z, t[7] = d.w;
    }
#pragma unroll
    for (int g = 0; g < 8; ++g)
        if (s[g] >= 0) f |= g;
    const double sc = f == 7 ? 0.125 : (f == 0 ? 1.0 : ((f & (f - 1)) == 0 ? 0.5 : 0.25));
    const int r0 = blockIdx.y * kFineRows;
#pragma unroll 2
    for (int rr = 0; rr < kFineRows; ++rr) {
        const int row = r0 + rr;
        if (row >= p.rows) break;
        const double *in = p.Us + static_cast<long long>(row) * p.ldus;
        double *out = p.U + static_cast<long long>(row) * p.ldu;
        double x[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) x[g] = t[g] >= 0 ? __ldcs(in + t[g]) : 0.0;
        sym_butterfly(x, f);
#pragma unroll
        for (int g = 0; g < 8; ++g)
            if (s[g] >= 0) out[s[g]] = sc * x[g];
    }
}

// ---------------------------------------------------------- segmented GEMM
// C[m][c_off + j] = sum_k A[m][a_off + k] * B_seg[j][k]  (+ row_scale[m] * bias_seg[j])
// for every segment (irrep). Tiles (M tile, segment, N tile) come from the
// persistent atomic queue of gemm_nt_f64; m_major = 1 walks all tiles of an M
// tile first (K1: the operand panel is streamed once), 0 walks an (segment,
// N tile) over all M tiles (K6: the basis is streamed once per chunk).
struct GemmSegParams {
    const double *A;
    long long lda;
    const double *Bt[2];  // per block kind: packed segment matrices
    const uint8_t *tile_kind;
    double *C;
    long long ldc;
    int m_tiles, tiles_per_m, n_segs;
    const GemmSeg *segs;
    const double *row_scale;    // nullable
    const double *col_bias[2];  // per kind, indexed bias_off + j
    const int *done;
    unsigned *tile_counter;
    int m_major;
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) gemm_seg_f64(GemmSegParams p) {
    pdl_wait();
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_tile;
    double *As = smem;
    double *Bs = smem + Cfg::STAGES * Cfg::A_STAGE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / Cfg::WN, wn = warp % Cfg::WN;
    const int total = p.m_tiles * p.tiles_per_m;
    const bool skip = p.done != nullptr && *reinterpret_cast<const volatile int *>(p.done) != 0;
    while (!skip) {
        if (tid == 0) s_tile = static_cast<int>(atomicAdd(&p.tile_counter[0], 1u));
        __syncthreads();
        const int tile = s_tile;
        __syncthreads();
        if (tile >= total) break;
        const int mt = p.m_major ? tile / p.tiles_per_m : tile % p.m_tiles;
        const int j = p.m_major ? tile % p.tiles_per_m : tile / p.m_tiles;
        int sg = 0;
        while (sg + 1 < p.n_segs && j >= p.segs[sg + 1].tile0) ++sg;
        const GemmSeg seg = p.segs[sg];
        const int nt = j - seg.tile0;
        const int kind = p.tile_kind ? p.tile_kind[mt] : 0;
        const double *A0 = p.A + static_cast<long long>(mt) * Cfg::BM * p.lda + seg.a_off;
        const double *B0 = (kind ? p.Bt[1] : p.Bt[0]) + seg.b_off + static_cast<long long>(nt) * Cfg::BN * seg.ldb;
        const int frag0 = nt * (Cfg::BN / 8) + wn * Cfg::FN;
        const int fn_lim = min(Cfg::FN, max(0, (seg.n_valid + 7) / 8 - frag0));
        double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
            for (int jj = 0; jj < Cfg::FN; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
        gemm_core<Cfg>(As, Bs, A0, p.lda, B0, seg.ldb, 0, seg.k_chunks, fn_lim, acc);
        const long long row0 = static_cast<long long>(mt) * Cfg::BM + wm * Cfg::TM + (lane >> 2);
        const double *cb = (kind ? p.col_bias[1] : p.col_bias[0]);
#pragma unroll
        for (int jj = 0; jj < Cfg::FN; ++jj) {
            const int col = nt * Cfg::BN + wn * Cfg::TN + jj * 8 + 2 * (lane & 3);
            if (col >= seg.n_valid) continue;
            const bool two = col + 1 < seg.n_valid;
            double b0 = 0.0, b1 = 0.0;
            if (p.row_scale) {
                b0 = cb[seg.bias_off + col];
                b1 = two ? cb[seg.bias_off + col + 1] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i) {
                const long long row = row0 + i * 8;
                double v0 = acc[i][jj][0], v1 = acc[i][jj][1];
                if (p.row_scale) {
                    const double s = p.row_scale[row];
                    v0 += s * b0;
                    v1 += s * b1;
                }
                double *dstp = p.C + row * p.ldc + seg.c_off + col;
                if (two) *reinterpret_cast<double2 *>(dstp) = make_double2(v0, v1);
                else dstp[0] = v0;
            }
        }
    }
    pdl_trigger();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&p.tile_counter[1], 1u) == gridDim.x - 1) {
            p.tile_counter[0] = 0u;
            p.tile_counter[1] = 0u;
            __threadfence();
        }
    }
}

}  // namespace tsvb200
