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
#include "tc_local.cuh"

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
#ifndef TSV_FINE_ROWS
#define TSV_FINE_ROWS 8
#endif
#ifndef TSV_FINE_UNROLL
#define TSV_FINE_UNROLL 4
#endif
constexpr int kFineRows = TSV_FINE_ROWS;
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
    // TSV_FINE_UNROLL rows per batch: all loads of the batch first (the compiler cannot move a row's
    // loads above the previous row's stores itself), then the butterflies and the stores
    constexpr int RB = TSV_FINE_UNROLL;
    for (int rr = 0; rr < kFineRows; rr += RB) {
        double x[RB][8];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int row = min(r0 + rr + u, p.rows - 1);
            const double *in = p.Us + static_cast<long long>(row) * p.ldus;
#pragma unroll
            for (int g = 0; g < 8; ++g) x[u][g] = t[g] >= 0 ? __ldcs(in + t[g]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int row = r0 + rr + u;
            if (row >= p.rows) break;
            double *out = p.U + static_cast<long long>(row) * p.ldu;
            sym_butterfly(x[u], f);
#pragma unroll
            for (int g = 0; g < 8; ++g)
                if (s[g] >= 0) out[s[g]] = sc * x[u][g];
        }
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


// ------------------------------------------------ fused K1 (one kernel)
// Y = X K_r for a mirror-symmetric K_r, one pass over the panel: a CTA takes
// R = 8 MF whole rows of X into shared memory (plain panel layout), runs the
// Walsh-Hadamard butterflies over the mirror orbits in place (combination w
// lands on member w), multiplies every irrep block on the DMMA pipe with the
// A fragments gathered from shared memory through the irrep's column list and
// the K''_r fragments streamed from L2 in fragment order, writes the products
// back in place, runs the inverse butterflies and stores the rows. HBM
// traffic is X in + Y out; FLOPs are 1/8 of the dense product.
//
// Work items are (irrep, pair of 8-column fragments); item i runs in round
// i / WARPS on warp i % WARPS. The product of irrep r overwrites its own
// operand columns, so an item's accumulators are parked in registers until
// the round in which the last item of its irrep ran (flush_round; at most
// kSymSlots - 1 rounds later - checked on the host).
//
// Shared-memory access: the row pitch is ldk + 4 doubles, so the A fragment
// loads of a half-warp (4 rows x 4 k) are conflict-free when the four columns
// of a k-step differ mod 4; the host orders each irrep's column list that way
// (SymK1Pack). A lane's columns for four consecutive k-steps are one 8-byte
// load from the transposed list [lane % 4][k-step].
constexpr int kSymSlots = 2;
#ifndef TSV_SYM_KB
#define TSV_SYM_KB 4
#endif
#ifndef TSV_SYM_RING
#define TSV_SYM_RING 3
#endif
#ifndef TSV_SYM_VOLATILE
#define TSV_SYM_VOLATILE 0  // 0: plain loads and DMMAs, 1: volatile K'' loads, 2: volatile loads and DMMAs
#endif
constexpr int kSymKB = TSV_SYM_KB;      // k-steps (of 4) per K'' chunk
constexpr int kSymRing = TSV_SYM_RING;  // K'' chunks in the register ring (prefetch distance kSymRing - 1 chunks)

// volatile: keeps the K'' prefetch loads ahead of the DMMAs they overlap (the compiler otherwise
// sinks them behind the chunk's DMMAs to shorten live ranges, which exposes the L2 latency)
__device__ __forceinline__ double ldg_nc_volatile(const double *p) {
#if TSV_SYM_VOLATILE >= 1
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ void dmma_8x8x4_v(double &d0, double &d1, double a, double b) {
#if TSV_SYM_VOLATILE < 2
    return dmma_8x8x4(d0, d1, a, b);
#endif
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

struct SymK1Item {
    int b_off;          // first double of the item's K'' fragments [ksteps4][2][32]
    short ksteps;       // k-steps of 4 (even); the fragment array is padded to a multiple of kSymKB
    short kcol;         // coltab offset of the irrep's transposed k column list [4][ksteps4]
    short ncol;         // coltab offset of the first fragment's 8 output columns (the second follows)
    short nvalid;       // valid output columns of the pair (1..16)
    short flush_round;  // round after which the irrep's operand columns are dead
    short ksteps4;      // ksteps rounded up to kSymKB
};
static_assert(sizeof(SymK1Item) == 16, "SymK1Item");

struct SymK1Params {
    const double *X;
    double *Y;
    long long ld;                // panel row pitch (ldk)
    int ldk;                     // doubles per row copied in / out
    const int4 *tiles;           // [n_tiles] {row0, rows (<= R, multiple of 8), kind, 0}
    int n_tiles;
    const double *Bf[2];         // per kind: K'' fragment streams [warp][round][cpi chunks][kSymKB][2][32]
    int cpi;                     // chunks (of kSymKB k-steps) per item slot in the stream, a multiple of kSymRing
    const SymK1Item *items;
    int n_items, rounds;
    const short *orb;            // [n_orbits][8] plain columns of the orbit members (-1: absent)
    int n_orbits;
    const short *coltab;
    int n_coltab;
    const int *done;             // nullable
    const int *skip_flag;        // nullable: early exit when != 0 (A x goes to the verification path)
    unsigned *tile_counter;
    int ablate;                  // timing experiments only (TSV_SYM_ABLATE): 1 no K'' prefetch, 2 no butterflies, 4 no products
};

inline size_t sym_k1_smem(int mf, int ldk, int n_orbits, int n_coltab, int n_items) {
    size_t b = static_cast<size_t>(mf) * 8 * (ldk + 4) * sizeof(double);
    b += static_cast<size_t>(n_items) * sizeof(SymK1Item);
    b += (static_cast<size_t>(n_orbits) * 16 + n_coltab) * sizeof(short);
    return (b + 15) / 16 * 16;
}

// In-place butterflies over every (row, orbit) of the tile. A half-warp takes
// 4 consecutive orbits x 4 rows (lane = 4 row + orbit), so with the row pitch
// = 4 mod 16 doubles an 8-byte access to member g of the four orbits is
// conflict-free when their columns differ mod 4 - the orbit order of the host
// tables (SymTables::order_orbits_for_banks). orbL / orbS: the members' columns
// for the loads / stores [n_orbits][8]; an absent member loads the row's zero
// column and stores to its sink column, so the three butterfly stages run
// unconditionally (a stage over an axis the orbit does not move adds zeros to
// the present members and only touches absent ones otherwise). INV: scaled by
// 1 / |orbit|.
#ifndef TSV_SYM_BF_PAIR
#define TSV_SYM_BF_PAIR 0
#endif
#ifndef TSV_SYM_BF_NOINLINE
#define TSV_SYM_BF_NOINLINE 0
#endif
#if TSV_SYM_BF_NOINLINE
#define TSV_SYM_BF_ATTR __noinline__
#else
#define TSV_SYM_BF_ATTR __forceinline__
#endif
template <bool INV, int WARPS>
__device__ TSV_SYM_BF_ATTR void sym_tile_butterflies(double *xs, int P, int rows, const short *orbL, const short *orbS,
                                                     int n_orbits, int zcol) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r0 = lane >> 2;  // 0..7: row within a block of 8
    for (int o = warp * 4 + (lane & 3); o < n_orbits; o += WARPS * 4) {
        const int4 lv = *reinterpret_cast<const int4 *>(orbL + o * 8);
        const int4 sv = *reinterpret_cast<const int4 *>(orbS + o * 8);
        int ml[8], ms[8];
        ml[0] = lv.x & 0xffff, ml[1] = static_cast<unsigned>(lv.x) >> 16, ml[2] = lv.y & 0xffff, ml[3] = static_cast<unsigned>(lv.y) >> 16;
        ml[4] = lv.z & 0xffff, ml[5] = static_cast<unsigned>(lv.z) >> 16, ml[6] = lv.w & 0xffff, ml[7] = static_cast<unsigned>(lv.w) >> 16;
        ms[0] = sv.x & 0xffff, ms[1] = static_cast<unsigned>(sv.x) >> 16, ms[2] = sv.y & 0xffff, ms[3] = static_cast<unsigned>(sv.y) >> 16;
        ms[4] = sv.z & 0xffff, ms[5] = static_cast<unsigned>(sv.z) >> 16, ms[6] = sv.w & 0xffff, ms[7] = static_cast<unsigned>(sv.w) >> 16;
        double s = 1.0;
        if (INV) {
            int members = 0;
#pragma unroll
            for (int g = 0; g < 8; ++g) members += ml[g] != zcol;
            s = 1.0 / static_cast<double>(members);  // 1, 2, 4 or 8 members: exact
        }
#if TSV_SYM_BF_PAIR
        // two rows per pass with all loads ahead of the stores (the compiler cannot reorder them itself)
        int r = r0;
        for (; r + 8 < rows; r += 16) {
            double *row = xs + r * P, *row2 = row + 8 * P;
            double x[8], y[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) x[g] = row[ml[g]], y[g] = row2[ml[g]];
            sym_butterfly(x, 7);
            sym_butterfly(y, 7);
#pragma unroll
            for (int g = 0; g < 8; ++g) row[ms[g]] = INV ? s * x[g] : x[g], row2[ms[g]] = INV ? s * y[g] : y[g];
        }
        if (r < rows) {
            double *row = xs + r * P;
            double x[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) x[g] = row[ml[g]];
            sym_butterfly(x, 7);
#pragma unroll
            for (int g = 0; g < 8; ++g) row[ms[g]] = INV ? s * x[g] : x[g];
        }
#else
#pragma unroll 2
        for (int r = r0; r < rows; r += 8) {
            double *row = xs + r * P;
            double x[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) x[g] = row[ml[g]];
            sym_butterfly(x, 7);
#pragma unroll
            for (int g = 0; g < 8; ++g) row[ms[g]] = INV ? s * x[g] : x[g];
        }
#endif
    }
}

// 1-D bulk copies (TMA unit) of whole panel rows
__device__ __forceinline__ void bulk_load_row(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_store_row(void *dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes) : "memory");
}

// The irrep products of one tile on MF row fragments (the kernel's inner part).
template <int MF, int WARPS, int SLOTS>
__device__ __forceinline__ void sym_tile_products(const SymK1Params &p, double *xs, int P, const SymK1Item *items,
                                                  const short *coltab, double (&b)[kSymRing][kSymKB][2], const double *bw,
                                                  int stream_chunks) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc[SLOTS][MF][2][2];
    int pend_round[SLOTS], pend_ncol[SLOTS], pend_nvalid[SLOTS];
#pragma unroll
    for (int v = 0; v < SLOTS; ++v) pend_round[v] = -1;
    const double *arow = xs + (lane >> 2) * P;
    for (int t0 = 0; t0 < p.rounds; t0 += SLOTS) {
#pragma unroll
        for (int v = 0; v < SLOTS; ++v) {
            const int t = t0 + v;
            const int it = t * WARPS + warp;
            if (t < p.rounds && it < p.n_items && !(p.ablate & 4)) {
                const SymK1Item item = items[it];
#pragma unroll
                for (int i = 0; i < MF; ++i) acc[v][i][0][0] = acc[v][i][0][1] = acc[v][i][1][0] = acc[v][i][1][1] = 0.0;
                const short *kc = coltab + item.kcol + (lane & 3) * item.ksteps4;
                const int ks = item.ksteps;
                for (int c0 = 0; c0 < p.cpi; c0 += kSymRing) {
#pragma unroll
                    for (int u = 0; u < kSymRing; ++u) {
                        const int c = c0 + u, s0 = c * kSymKB, g = t * p.cpi + c;
                        constexpr int kAhead = kSymRing - 1;
                        if (g + kAhead < stream_chunks && !(p.ablate & 1)) {
                            const double *q = bw + static_cast<long long>(g + kAhead) * (kSymKB * 64);
#pragma unroll
                            for (int s = 0; s < kSymKB; ++s) {
                                b[(u + kAhead) % kSymRing][s][0] = ldg_nc_volatile(q + s * 64);
                                b[(u + kAhead) % kSymRing][s][1] = ldg_nc_volatile(q + s * 64 + 32);
                            }
                        }
                        if (s0 < ks) {  // ksteps is even: whole chunks (padding k-steps inside ksteps read a real column; their K'' is zero)
                            int cols[kSymKB];
                            if constexpr (kSymKB == 2) {
                                const short2 cv = *reinterpret_cast<const short2 *>(kc + s0);
                                cols[0] = cv.x, cols[1] = cv.y;
                            } else {
                                static_assert(kSymKB == 2 || kSymKB == 4, "kSymKB");
                                const short4 cv = *reinterpret_cast<const short4 *>(kc + s0);
                                cols[0] = cv.x, cols[1] = cv.y, cols[2] = cv.z, cols[3] = cv.w;
                            }
                            double af[kSymKB][MF];
#pragma unroll
                            for (int s = 0; s < kSymKB; ++s)
#pragma unroll
                                for (int i = 0; i < MF; ++i) af[s][i] = arow[i * 8 * P + cols[s]];
#pragma unroll
                            for (int s = 0; s < kSymKB; ++s)
#pragma unroll
                                for (int i = 0; i < MF; ++i) {
                                    dmma_8x8x4_v(acc[v][i][0][0], acc[v][i][0][1], af[s][i], b[u][s][0]);
                                    dmma_8x8x4_v(acc[v][i][1][0], acc[v][i][1][1], af[s][i], b[u][s][1]);
                                }
                        }
                    }
                }
                pend_round[v] = item.flush_round;
                pend_ncol[v] = item.ncol;
                pend_nvalid[v] = item.nvalid;
            }
            __syncthreads();  // round t done: operands of irreps that ended in it are dead
            if (t < p.rounds) {
#pragma unroll
                for (int w = 0; w < SLOTS; ++w) {
                    if (pend_round[w] >= 0 && pend_round[w] <= t) {
                        double *orow = xs + (lane >> 2) * P;
#pragma unroll
                        for (int fr = 0; fr < 2; ++fr) {
                            const int j = 8 * fr + 2 * (lane & 3);
                            const short *nc = coltab + pend_ncol[w] + j;
                            const int c0 = nc[0], c1 = nc[1];
                            const bool v0 = j < pend_nvalid[w], v1 = j + 1 < pend_nvalid[w];
#pragma unroll
                            for (int i = 0; i < MF; ++i) {
                                if (v0) orow[i * 8 * P + c0] = acc[w][i][fr][0];
                                if (v1) orow[i * 8 * P + c1] = acc[w][i][fr][1];
                            }
                        }
                        pend_round[w] = -1;
                    }
                }
            }
        }
    }
}

template <int MF, int WARPS, int MINB, int SLOTS = kSymSlots>
__global__ void __launch_bounds__(32 * WARPS, MINB) sym_k1_fused_kernel(SymK1Params p) {
    pdl_wait();
    extern __shared__ __align__(16) double sym_smem[];
    __shared__ int s_tile;
    constexpr int R = 8 * MF, THREADS = 32 * WARPS;
    const int P = p.ldk + 4;
    double *xs = sym_smem;
    SymK1Item *items = reinterpret_cast<SymK1Item *>(xs + static_cast<size_t>(R) * P);
    short *orbL = reinterpret_cast<short *>(items + p.n_items);  // load / store columns of the orbit members
    short *orbS = orbL + p.n_orbits * 8;
    short *coltab = orbS + p.n_orbits * 8;
    const int zcol = p.ldk, sink = p.ldk + 2;  // in the row pitch padding: always zero / write-only
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool skip = (p.done != nullptr && *reinterpret_cast<const volatile int *>(p.done) != 0) ||
                      (p.skip_flag != nullptr && *reinterpret_cast<const volatile int *>(p.skip_flag) != 0);
    if (!skip) {
        for (int i = tid; i < p.n_items * 4; i += THREADS)
            reinterpret_cast<int *>(items)[i] = reinterpret_cast<const int *>(p.items)[i];
        for (int i = tid; i < p.n_orbits * 8; i += THREADS) {
            const short c = p.orb[i];
            orbL[i] = c >= 0 ? c : static_cast<short>(zcol);
            orbS[i] = c >= 0 ? c : static_cast<short>(sink);
        }
        for (int r = tid; r < R; r += THREADS) xs[r * P + zcol] = 0.0;
        for (int i = tid; i < p.n_coltab; i += THREADS) coltab[i] = p.coltab[i];
    }
    __shared__ __align__(8) uint64_t row_bar;
    const uint32_t bar = smem_u32(&row_bar);
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    const uint32_t row_bytes = static_cast<uint32_t>(p.ldk) * 8u;
    uint32_t phase = 0;
    while (!skip) {
        if (tid == 0) {
            s_tile = static_cast<int>(atomicAdd(&p.tile_counter[0], 1u));
            // the previous tile's rows have left shared memory before it is overwritten
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncthreads();
        const int tile = s_tile;
        if (tile >= p.n_tiles) break;
        const int4 tl = p.tiles[tile];
        const int rows = tl.y;
        const double *Bf = tl.z ? p.Bf[1] : p.Bf[0];
        // ---- rows in: one bulk copy per row (absent rows of a short tile: zeros)
        if (tid == 0) {
            mbar_expect_tx(bar, row_bytes * static_cast<uint32_t>(rows));
            const double *src = p.X + static_cast<long long>(tl.x) * p.ld;
            for (int r = 0; r < rows; ++r) bulk_load_row(smem_u32(xs + r * P), src + r * p.ld, row_bytes, bar);
        }
        {   // rows of the last active fragment beyond the tile (tiles are whole fragments unless a kind group is not): zeros
            const int rpad = (rows + 7) / 8 * 8;
            for (int i = tid; i < (rpad - rows) * p.ldk; i += THREADS) xs[rows * P + (i / p.ldk) * P + i % p.ldk] = 0.0;
        }
        // K'' register ring: the warp's fragment stream is contiguous over its items,
        // chunk g of the stream lives in b[g % kSymRing] (cpi % kSymRing == 0)
        double b[kSymRing][kSymKB][2];
        const double *bw = Bf + static_cast<long long>(warp) * p.rounds * p.cpi * (kSymKB * 64) + lane;
        const int stream_chunks = p.rounds * p.cpi;
#pragma unroll
        for (int u = 0; u < kSymRing - 1; ++u)
#pragma unroll
            for (int s = 0; s < kSymKB; ++s) {
                b[u][s][0] = ldg_nc_volatile(bw + (u * kSymKB + s) * 64);
                b[u][s][1] = ldg_nc_volatile(bw + (u * kSymKB + s) * 64 + 32);
            }
        mbar_wait(bar, phase);
        phase ^= 1u;
        __syncthreads();
        if (!(p.ablate & 2)) sym_tile_butterflies<false, WARPS>(xs, P, rows, orbL, orbS, p.n_orbits, zcol);
        __syncthreads();
        // ---- irrep products (a short tile of the balanced tail multiplies its present row fragments only)
        if (rows > 8 * (MF - 1)) {
            sym_tile_products<MF, WARPS, SLOTS>(p, xs, P, items, coltab, b, bw, stream_chunks);
        } else if (rows <= 8) {
            sym_tile_products<1, WARPS, SLOTS>(p, xs, P, items, coltab, b, bw, stream_chunks);
        } else {
            if constexpr (MF > 2) {
                if (rows <= 16) sym_tile_products<2, WARPS, SLOTS>(p, xs, P, items, coltab, b, bw, stream_chunks);
                else sym_tile_products<MF - 1, WARPS, SLOTS>(p, xs, P, items, coltab, b, bw, stream_chunks);
            }
        }
        __syncthreads();
        if (!(p.ablate & 2)) sym_tile_butterflies<true, WARPS>(xs, P, rows, orbL, orbS, p.n_orbits, zcol);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes before the bulk stores
        __syncthreads();
        // ---- rows out
        if (tid == 0) {
            double *dst = p.Y + static_cast<long long>(tl.x) * p.ld;
            for (int r = 0; r < rows; ++r) bulk_store_row(dst + r * p.ld, smem_u32(xs + r * P), row_bytes);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

// ------------------------------------------------ fused K1, two row buffers
// The same tile work as sym_k1_fused_kernel with one CTA of WARPS warps per SM
// and two row buffers: the bulk load of the next tile and the bulk store of
// the previous one are in flight while this tile's butterflies and products
// run, so the copies leave the critical path (they are 24 of the ~94 us of
// the single-buffer kernel at config 3).
inline size_t sym_k1_pipe_smem(int mf, int ldk, int n_orbits, int n_coltab, int n_items) {
    return sym_k1_smem(mf, ldk, n_orbits, n_coltab, n_items) + static_cast<size_t>(mf) * 8 * (ldk + 4) * sizeof(double);
}

template <int MF, int WARPS, int SLOTS = kSymSlots>
__global__ void __launch_bounds__(32 * WARPS, 1) sym_k1_pipe_kernel(SymK1Params p) {
    pdl_wait();
    extern __shared__ __align__(16) double sym_smem[];
    __shared__ int s_tile;
    __shared__ __align__(8) uint64_t row_bar[2];
    constexpr int R = 8 * MF, THREADS = 32 * WARPS;
    const int P = p.ldk + 4;
    double *buf[2] = {sym_smem, sym_smem + static_cast<size_t>(R) * P};
    SymK1Item *items = reinterpret_cast<SymK1Item *>(sym_smem + 2 * static_cast<size_t>(R) * P);
    short *orbL = reinterpret_cast<short *>(items + p.n_items);
    short *orbS = orbL + p.n_orbits * 8;
    short *coltab = orbS + p.n_orbits * 8;
    const int zcol = p.ldk, sink = p.ldk + 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool skip = (p.done != nullptr && *reinterpret_cast<const volatile int *>(p.done) != 0) ||
                      (p.skip_flag != nullptr && *reinterpret_cast<const volatile int *>(p.skip_flag) != 0);
    const uint32_t bar[2] = {smem_u32(&row_bar[0]), smem_u32(&row_bar[1])};
    const uint32_t row_bytes = static_cast<uint32_t>(p.ldk) * 8u;
    auto issue_load = [&](int tile, int bi) {  // one thread
        const int4 tl = p.tiles[tile];
        mbar_expect_tx(bar[bi], row_bytes * static_cast<uint32_t>(tl.y));
        const double *src = p.X + static_cast<long long>(tl.x) * p.ld;
        for (int r = 0; r < tl.y; ++r) bulk_load_row(smem_u32(buf[bi] + r * P), src + r * p.ld, row_bytes, bar[bi]);
    };
    int cur = p.n_tiles;
    if (!skip) {
        for (int i = tid; i < p.n_items * 4; i += THREADS)
            reinterpret_cast<int *>(items)[i] = reinterpret_cast<const int *>(p.items)[i];
        for (int i = tid; i < p.n_orbits * 8; i += THREADS) {
            const short c = p.orb[i];
            orbL[i] = c >= 0 ? c : static_cast<short>(zcol);
            orbS[i] = c >= 0 ? c : static_cast<short>(sink);
        }
        for (int r = tid; r < 2 * R; r += THREADS) sym_smem[r * P + zcol] = 0.0;
        for (int i = tid; i < p.n_coltab; i += THREADS) coltab[i] = p.coltab[i];
        if (tid == 0) {
            mbar_init(bar[0], 1);
            mbar_init(bar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            s_tile = static_cast<int>(atomicAdd(&p.tile_counter[0], 1u));
            if (s_tile < p.n_tiles) issue_load(s_tile, 0);
        }
        __syncthreads();
        cur = s_tile;
    }
    uint32_t phase[2] = {0u, 0u};
    for (int it = 0; cur < p.n_tiles; ++it) {
        const int bi = it & 1;
        double *xs = buf[bi];
        __syncthreads();  // everyone has read s_tile (cur)
        if (tid == 0) s_tile = static_cast<int>(atomicAdd(&p.tile_counter[0], 1u));
        const int4 tl = p.tiles[cur];
        const int rows = tl.y;
        const double *Bf = tl.z ? p.Bf[1] : p.Bf[0];
        double b[kSymRing][kSymKB][2];
        const double *bw = Bf + static_cast<long long>(warp) * p.rounds * p.cpi * (kSymKB * 64) + lane;
        const int stream_chunks = p.rounds * p.cpi;
#pragma unroll
        for (int u = 0; u < kSymRing - 1; ++u)
#pragma unroll
            for (int s = 0; s < kSymKB; ++s) {
                b[u][s][0] = ldg_nc_volatile(bw + (u * kSymKB + s) * 64);
                b[u][s][1] = ldg_nc_volatile(bw + (u * kSymKB + s) * 64 + 32);
            }
        mbar_wait(bar[bi], phase[bi]);
        phase[bi] ^= 1u;
        {   // rows of the last active fragment beyond the tile: zeros
            const int rpad = (rows + 7) / 8 * 8;
            for (int i = tid; i < (rpad - rows) * p.ldk; i += THREADS) xs[rows * P + (i / p.ldk) * P + i % p.ldk] = 0.0;
        }
        __syncthreads();
        const int nxt = s_tile;
        sym_tile_butterflies<false, WARPS>(xs, P, rows, orbL, orbS, p.n_orbits, zcol);
        // the next tile's rows into the other buffer: its previous tenant's bulk stores were
        // committed a whole tile ago, their shared-memory reads are long done
        if (tid == 0 && nxt < p.n_tiles) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            issue_load(nxt, bi ^ 1);
        }
        __syncthreads();
        if (rows > 8 * (MF - 1)) {
            sym_tile_products<MF, WARPS, SLOTS>(p, xs, P, items, coltab, b, bw, stream_chunks);
        } else if (rows <= 8) {
            sym_tile_products<1, WARPS, SLOTS>(p, xs, P, items, coltab, b, bw, stream_chunks);
        } else {
            if constexpr (MF > 2) {
                if (rows <= 16) sym_tile_products<2, WARPS, SLOTS>(p, xs, P, items, coltab, b, bw, stream_chunks);
                else sym_tile_products<MF - 1, WARPS, SLOTS>(p, xs, P, items, coltab, b, bw, stream_chunks);
            }
        }
        __syncthreads();
        sym_tile_butterflies<true, WARPS>(xs, P, rows, orbL, orbS, p.n_orbits, zcol);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            double *dst = p.Y + static_cast<long long>(tl.x) * p.ld;
            for (int r = 0; r < rows; ++r) bulk_store_row(dst + r * p.ld, smem_u32(xs + r * P), row_bytes);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        cur = nxt;
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
