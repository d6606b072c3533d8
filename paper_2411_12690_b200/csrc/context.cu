// tsv_ctx: device residency, the PCG driver and the recovery driver behind
// the C ABI of include/tsv_b200.h.
//
// Data layout in HBM:
//   K_r[kind]   [round_up(n, BN) rows][ldk]     zero-padded, symmetric
//   Phi[kind]   [round_up(n_fine, BN)][ldk]     row-major fine DoF x reduced DoF
//   X, Y        [B_pad][ldk]                    block-major operand / product panels
//               (GEMM row j = block, blocks grouped by kind, each kind padded to BM)
//   slots       [nodes][4] int32                offsets j*ldk + 3*rank of every
//               (block, local node) copy of an owned global node; nodes are
//               renumbered block-major (owner = first block in GEMM-row order)
//   x r p ap b  [N] in that internal node order; mapped back to the
//               reference numbering (global_stage.cpp:94-119) at the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <exception>
#include <vector>

#include "../../include/tsv_b200.h"
#include "host_index.hpp"
#include "kernels.cuh"
#include "schwarz.cuh"
#include "ozaki.cuh"
#include "small_pcg.cuh"
#include "sym.cuh"
#include "symmetry.hpp"

#include <cublas_v2.h>
#include <cusolverDn.h>
#include <map>
#include <unordered_map>

using namespace tsvb200;

namespace {

// K1 tile configuration (BM, BN, warps M x N, KC, stages, CTAs per SM). Measured
// at configs 3 / 4 (ms per launch): 2x2 warps 0.289 / 0.254; 4x1 warps 0.285 /
// 0.248 (default); 4 stages 0.395 / 0.351; 2 stages 0.293 / 0.255; 8x1 warps
// (1 CTA/SM) 0.342 / 0.299; 4x2 warps (1 CTA/SM) 0.340 / 0.305.
#ifndef TSV_K1CFG
#define TSV_K1CFG 128, 64, 4, 1, 16, 3, 2
#endif
#ifndef TSV_K6CFG  // K6 (recovery GEMM), same shape family: 4x1 warps 16.33 ms vs 2x2 16.60 ms recovery at config 3
#define TSV_K6CFG 128, 64, 4, 1, 16, 3, 2
#endif
using K1Cfg = GemmCfg<TSV_K1CFG>;
using K6Cfg = GemmCfg<TSV_K6CFG>;
using K1SmallCfg = GemmCfg<64, 64, 2, 2, 16, 3, 3>;  // KC must divide ldk (multiple of 16)
constexpr int kBM = K1Cfg::BM;
constexpr int kBN = K1Cfg::BN;
constexpr int kKC = K1Cfg::KC;
constexpr int kVecThreads = 256;
constexpr int kItersPerGraph = 16;

struct StatusError : std::runtime_error {
    StatusError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
    int code;
};

#define CK(expr)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw StatusError(e_ == cudaErrorMemoryAllocation ? TSV_ENOMEM : TSV_ECUDA,            \
                              std::string(#expr) + ": " + cudaGetErrorString(e_));                 \
    } while (0)

// Stream-ordered device buffers: inside an ABI call (guarded()) allocations
// and frees are queued on the context stream (cudaMallocAsync / cudaFreeAsync
// from the device pool), so dropping a temporary never stalls the host on
// the device (a plain cudaFree synchronises the whole device).
thread_local cudaStream_t tl_alloc_stream = nullptr;

template <typename T>
struct DevBuf {
    T *ptr = nullptr;
    size_t count = 0;
    cudaStream_t s_ = nullptr;  // stream the memory is ordered on (null: synchronous)
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (ptr) {
            if (s_) cudaFreeAsync(ptr, s_);
            else cudaFree(ptr);
        }
        ptr = nullptr;
        count = 0;
    }
    void alloc(size_t n) {
        if (n == count && ptr) return;
        release();
        if (n == 0) return;
        // long-lived large buffers (>= 1 GB: stress, U, recovery staging) come
        // from cudaMalloc: a stream-ordered pool allocation that grows the pool
        // by tens of GB maps its pages lazily inside the first timed use
        s_ = n * sizeof(T) >= (size_t(1) << 30) ? nullptr : tl_alloc_stream;
        if (s_) CK(cudaMallocAsync(reinterpret_cast<void **>(&ptr), n * sizeof(T), s_));
        else CK(cudaMalloc(&ptr, n * sizeof(T)));
        count = n;
    }
    void upload(const T *src, size_t n, cudaStream_t s) {
        alloc(n);
        if (n) CK(cudaMemcpyAsync(ptr, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
};

// TSV_TIMING=1: host wall time of the set-up phases on stderr (no syncs added).
struct PhaseTimer {
    const char *name;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit PhaseTimer(const char *n) : name(n) {}
    void report() const {
        static const bool on = [] { const char *v = std::getenv("TSV_TIMING"); return v && *v && *v != '0'; }();
        if (on)
            std::fprintf(stderr, "[tsv timing] %-22s %8.2f ms\n", name,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    void lap(const char *next) {  // report this phase, start the next
        report();
        name = next;
        t0 = std::chrono::steady_clock::now();
    }
    ~PhaseTimer() { report(); }
};

// Owns a stream; declared first in tsv_ctx so it is destroyed after every
// DevBuf member has queued its free on it.
struct StreamOwner {
    cudaStream_t s = nullptr;
    ~StreamOwner() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

// Device -> host copy ordered after everything queued on `s` (the context
// stream is non-blocking, so a plain cudaMemcpy would not wait for it).
void d2h(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
}

// Panel column of local reduced DoF a = 3 rank + c (rom.cpp:26-31 order):
// component-major within a block row.
inline size_t pidx(size_t a, size_t nn) { return (a % 3) * nn + a / 3; }

struct RomHost {
    bool set = false;
    uint32_t q[3] = {0, 0, 0};
    double geom[4] = {0, 0, 0, 0};
    std::vector<double> grid[3];
    double mats[3][3] = {};
    double lame[3][3] = {};  // lambda, mu, alpha*(3 lambda + 2 mu)
    std::vector<uint8_t> elem_mat;
    std::vector<double> k_r, b_el, u_t;  // host copies used for assembly of b / preconditioners
    size_t n = 0, n_fine = 0, cells[3] = {0, 0, 0};
    uint8_t fingerprint[32] = {};
    DevBuf<double> d_k, d_phi, d_ut, d_hinv, d_grid[3], d_bel;
    // K6 split: d_phi / d_ut hold the dense basis rows only (n_dense, in fine
    // DoF order, d_dmap = their fine DoFs); the sparse (surface) rows are CSR
    size_t n_dense = 0, n_sparse = 0;
    DevBuf<int> d_dmap, d_sp_ptr, d_sp_dof, d_sp_col;
    DevBuf<double> d_sp_val, d_ut_full;
    // surface rows grouped by (face, component): small dense GEMMs (k6_face_kernel)
    int n_groups = 0, max_group_rows = 0, max_group_k = 0;
    DevBuf<int4> d_ginfo;
    DevBuf<int> d_gcol, d_gdof;
    DevBuf<double> d_gwt;
    DevBuf<long long> d_gwoff;
    DevBuf<uint8_t> d_em;
    // Ozaki digit planes of K_r (int8 K1): [S][rows][KA], row exponents
    int oz_s = 0;
    DevBuf<int8_t> oz_b;
    DevBuf<int> oz_eb;
    // Mirror symmetry (symmetry.hpp, sym.cuh): set when K_r and the dense basis
    // rows are block diagonal over the 8 irreps to rounding.
    bool sym = false;
    SymTables sred, sfine;           // reduced DoFs (panel order) / dense fine DoFs
    double sym_defect_k = 0.0, sym_defect_phi = 0.0;
    std::vector<GemmSeg> k1_segs, k6_segs;
    int k1_tiles_per_m = 0, k6_tiles_per_m = 0;
    DevBuf<double> d_ks, d_phis, d_uts;   // packed K''_r / Phi''_r blocks, H u_T (fine segmented layout)
    DevBuf<short> d_ssrc, d_sdst;         // reduced orbit tables
    DevBuf<int> d_fsrc, d_fdst;           // fine orbit tables (U column / Us column)
    DevBuf<GemmSeg> d_k1_segs, d_k6_segs;
    SymK1Pack k1f;                        // fused K1 (sym_k1_fused_kernel): items, column lists
    // K_r - K_sym (the rounding-level symmetry defect of K_r), TF32, times 2^d_exp:
    // added back on the tensor cores so the operator stays the reference's K_r
    std::vector<float> d32_host;          // [n][n] panel order, scaled
    int d_exp = 0;
    bool d_nonzero = false;
};

// Symmetry-adapted packing of one ROM (tsv_set_rom): host tables from
// SymRomPack (symmetry.hpp), uploaded here.
void build_rom_symmetry(RomHost &m, const std::vector<double> &kp, const double *basis, const double *thermal,
                        const std::vector<int> &dmap, cudaStream_t stream, int bn, int kc) {
    m.sym = false;
    const char *env = std::getenv("TSV_SYM");
    if (env && *env == '0') return;
    SymRomPack pk;
    const int cells[3] = {static_cast<int>(m.cells[0]), static_cast<int>(m.cells[1]), static_cast<int>(m.cells[2])};
    const bool ok = pk.build(m.q, cells, m.n, kp, basis, thermal, dmap, bn, kc);
    m.sym_defect_k = pk.defect_k;
    m.sym_defect_phi = pk.defect_phi;
    if (!ok) return;
    m.k1f.build(pk.red, pk.k1_segs, pk.ks, kSymKB);
    m.sred = std::move(pk.red);
    m.sfine = std::move(pk.fine);
    m.k1_segs = std::move(pk.k1_segs);
    m.k6_segs = std::move(pk.k6_segs);
    m.k1_tiles_per_m = pk.k1_tiles_per_m;
    m.k6_tiles_per_m = pk.k6_tiles_per_m;
    m.d32_host = std::move(pk.d32);
    m.d_exp = pk.d_exp;
    m.d_nonzero = pk.d_nonzero;
    m.d_ks.upload(pk.ks.data(), pk.ks.size(), stream);
    m.d_phis.upload(pk.ps.data(), pk.ps.size(), stream);
    m.d_uts.upload(pk.uts.data(), pk.uts.size(), stream);
    m.d_ssrc.upload(pk.ssrc.data(), pk.ssrc.size(), stream);
    m.d_sdst.upload(pk.sdst.data(), pk.sdst.size(), stream);
    m.d_fsrc.upload(pk.fsrc.data(), pk.fsrc.size(), stream);
    m.d_fdst.upload(m.sfine.dst.data(), m.sfine.dst.size(), stream);
    m.d_k1_segs.upload(m.k1_segs.data(), m.k1_segs.size(), stream);
    m.d_k6_segs.upload(m.k6_segs.data(), m.k6_segs.size(), stream);
    CK(cudaStreamSynchronize(stream));
    m.sym = true;
}

}  // namespace

struct tsv_ctx {
    StreamOwner own_stream, own_side, own_copy;  // first: destroyed last
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    int sm_count = 148;
    uint64_t launches = 0;

    RomHost rom[2];

    // layout
    bool layout_set = false;
    ArrayLayout layout;
    NodeLayout nl;
    GlobalIndex index;
    std::vector<uint32_t> dofmap;  // [B][n]
    size_t n = 0, ldk = 0, B = 0, B_pad = 0, m_tiles = 0, nodes = 0, N = 0;
    std::vector<int> row_cell, cell_row;
    std::vector<double> dt_host;  // per panel row dT (set_delta_t staging)
    std::vector<uint8_t> row_kind, tile_kind;
    std::vector<double> row_dt;
    std::vector<uint32_t> node_glob_of_int, node_int_of_glob;
    std::vector<int> node_super_ptr;
    bool rhs_dirty = true;  // [super cell + 1] internal node ranges (super-cell-major numbering)

    // boundary conditions (reference numbering)
    bool bc_set = false;
    std::vector<uint8_t> constrained;
    std::vector<double> g;
    bool any_g = false;

    // device
    DevBuf<double> X, Y, b, x, r, p, ap, pre, partial, row_dt_d, U, stress;
    DevBuf<int> slots, row_cell_d;
    DevBuf<uint32_t> glob_of_int_d;  // internal node -> reference node
    DevBuf<double> uref;             // reference-ordered staging for D2H
    DevBuf<uint8_t> cmask, row_kind_d, tile_kind_d, tile_kind_small_d;
    DevBuf<unsigned> tile_counter;
    DevBuf<CgState> state;
    DevBuf<int> zero_flag;  // a device int that stays 0 (kernels with a mandatory done flag, outside a solve)
    int pre_kind = -1;
    bool solution_valid = false;
    int stress_points = 0;
    CgState *h_state = nullptr;  // pinned

    cudaGraphExec_t iter_graph = nullptr;
    int k1_grid = 0, k6_grid = 0;
    int k1s_grid = 0;
    bool k1_small = false;  // small arrays: 64 x 64 tiles keep every SM busy
    bool k1_streamk = false;  // large arrays: stream-K balanced K1
    // two-level additive Schwarz (precond 3)
    struct As2 {
        int s = 0, SX = 0, SY = 0, Nc = 0, ncells = 0, ntypes = 0, step = 0, step_y = 0;
        size_t BL_pad = 0, mtiles = 0;
        DevBuf<int> slots2, tile_type, cell_ptr;
        DevBuf<double> XL, ZL, z, cellpart, rc, zc, ainv_c, ainv_store;
        DevBuf<const double *> ainv_tab;
        DevBuf<short4> lat;
        DevBuf<int> node_cell;
        DevBuf<double4> celltab;
        double setup_ms = 0.0;
        // tensor-core (TF32) local solves
        bool tc = false;
        int KP = 0, NP = 0, BN = 0, ntn = 0, LD = 0;  // LD: row stride of XL32 and ZL
        DevBuf<float> XL32, ainv32, ZL32;
        DevBuf<int2> tc_pairs;  // consecutive same-type M tiles for tc_local_pair_kernel
        int npairs = 0;
        CUtensorMap tmA{}, tmB{};
        DevBuf<float> ainv_c32;
        int ldc32 = 0;
        // packed lower tiles of the FP32 inverse (symmetric GEMV, default)
        DevBuf<float> sym_tiles;
        DevBuf<double> sym_part, dotpart, kcell_d, cwork;
        int sym_nt = 0;
        // split loop: A P zc panel and its per-key products
        DevBuf<double> Yc, kp;
        DevBuf<int4> kp_items;
        DevBuf<int> kp_rows;
        int kp_nitems = 0;
    } as2;
    // mirror-symmetric ROMs (sym.cuh): irrep-segmented operand / product panels
    struct SymCtx {
        bool on = false;   // every ROM of the layout is mirror-symmetric (K6 path)
        bool k1 = false;   // K1 on the symmetric path too
        int tab_kind = 0;  // ROM whose (shared) reduced tables are used
        int lds = 0;       // row length of the segmented reduced panel
        size_t panel_smem = 0;
        DevBuf<double> Xs, Ys, Us;
        // fused K1 (one kernel, sym_k1_fused_kernel)
        bool fused = false;
        bool pipe = false;  // two row buffers, one CTA per SM (sym_k1_pipe_kernel)
        int f_mf = 2, f_items = 0, f_rounds = 0, f_tiles = 0, f_coltab = 0, f_grid = 0, f_max_grid = 0;
        size_t f_smem = 0;
        DevBuf<int4> f_tile_tab;
        DevBuf<SymK1Item> f_item_tab;
        DevBuf<short> f_col_tab;
        DevBuf<double> f_stream[2];  // per kind: K'' fragment streams in warp order
        int f_cpi = 0;
        // K_r symmetry-defect correction on tcgen05 (TF32): Yc32 = X32 D32^T
        bool corr = false;
        int KP = 0, NP = 0, BN = 0, ntn = 0, LD = 0, npairs = 0;
        double c_scale = 0.0;
        DevBuf<float> X32, Yc32, d32;
        DevBuf<int> tile_type;
        DevBuf<int2> pairs;
        CUtensorMap tmA{}, tmB{};
    } sym;
    // int8 (Ozaki) K1: digit planes of the X panel
    int oz_s = 0;            // digits per value (0 = DMMA K1)
    int graph_oz_s = 0;      // K1 variant baked into the captured graph
    const float *graph_xlo = nullptr;  // compensated-x vector baked into the captured graph
    long long oz_brows = 0;  // K rows padded to the N tiles
    DevBuf<int8_t> oz_a;
    DevBuf<int> oz_ea;
    CUtensorMap oz_tmA{}, oz_tmB[2]{};
    bool sk_resident = false;
    DevBuf<int> sk_start, sk_flag;
    DevBuf<double> sk_work;

    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaStream_t side = nullptr;                       // Schwarz coarse chain (forked in the graph)
    cudaStream_t copy = nullptr;                       // recovery D2H (overlaps the next chunk)
    cudaEvent_t rec_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // [computed, copied] x 2 staging buffers
    cudaEvent_t k67_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // [K6 done, K7 done] x 2 U buffers (recover_range)
    DevBuf<double> U2;                                             // second U chunk buffer
    DevBuf<double> rstage[2];
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    double last_solve_ms = 0, last_recover_ms = 0, last_apply_ms = 0;
    // K7 launch times of the last recovery (CUDA events around every stress kernel launch)
    double last_stress_ms = 0;
    int last_stress_launches = 0;
    std::vector<cudaEvent_t> k7_ev;  // [2 * launches] start / stop
    int k7_used = 0;
    cudaEvent_t k7_event() {
        if (k7_used == static_cast<int>(k7_ev.size())) {
            cudaEvent_t e = nullptr;
            CK(cudaEventCreate(&e));
            k7_ev.push_back(e);
        }
        return k7_ev[k7_used++];
    }
    void collect_stress_times() {  // after the recovery's final synchronize
        last_stress_ms = 0;
        last_stress_launches = k7_used / 2;
        for (int i = 0; i + 1 < k7_used; i += 2) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, k7_ev[i], k7_ev[i + 1]) == cudaSuccess) last_stress_ms += ms;
            else cudaGetLastError();
        }
        k7_used = 0;
    }

    ~tsv_ctx() {
        if (iter_graph) cudaGraphExecDestroy(iter_graph);
        if (h_state) cudaFreeHost(h_state);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (stream) cudaStreamSynchronize(stream);
        if (copy) cudaStreamSynchronize(copy);
        tl_alloc_stream = nullptr;
        for (auto &e : k67_ev)
            if (e) cudaEventDestroy(e);
        for (auto &e : k7_ev)
            if (e) cudaEventDestroy(e);
        for (auto &e : rec_ev)
            if (e) cudaEventDestroy(e);
        // streams: own_stream / own_side / own_copy, after the DevBuf members
    }

    void drop_graph() {
        if (iter_graph) cudaGraphExecDestroy(iter_graph);
        iter_graph = nullptr;
    }

    const RomHost &rom_of(int kind) const { return rom[kind]; }

    // ------------------------------------------------------------ layout
    void build_layout(uint32_t rows, uint32_t cols, const uint8_t *kinds, const double *dt, size_t ndt,
                      double pitch, double height) {
        PhaseTimer pt("set_layout");
        ArrayLayout L;
        L.rows = rows;
        L.cols = cols;
        if (kinds) L.kinds.assign(kinds, kinds + static_cast<size_t>(rows) * cols);
        if (!dt && ndt) throw StatusError(TSV_EINVAL, "layout: delta_t pointer is NULL");
        L.delta_t.assign(dt, dt + ndt);
        L.pitch = pitch;
        L.height = height;
        L.validate();
        // RomSet::check_consistency (global_stage.cpp:52-80)
        bool need[2] = {false, false};
        for (size_t c = 0; c < L.cell_count(); ++c) need[L.kind_at(c)] = true;
        if (need[0] && !rom[0].set) throw StatusError(TSV_EINVAL, "layout contains tsv blocks but no tsv model is loaded");
        if (need[1] && !rom[1].set)
            throw StatusError(TSV_EINVAL, "layout contains dummy blocks but no dummy model is loaded");
        if (rom[0].set && rom[1].set && std::memcmp(rom[0].fingerprint, rom[1].fingerprint, 32) != 0)
            throw StatusError(TSV_EINVAL, "tsv and dummy models come from different parameter sets (fingerprint mismatch)");
        const RomHost &m = rom[0].set ? rom[0] : rom[1];
        if (!m.set) throw StatusError(TSV_EINVAL, "RomSet: no models loaded");
        if (m.geom[3] != pitch || m.geom[1] != height)
            throw StatusError(TSV_EINVAL, "model geometry does not match the layout pitch/height (fingerprint mismatch)");

        layout = L;
        nl = NodeLayout::create(m.q[0], m.q[1], m.q[2]);
        {
            PhaseTimer pt1("  index_global_nodes");
            index = index_global_nodes(layout, nl);
        }
        {
            PhaseTimer pt1("  dof_map");
            dofmap = tsvb200::dof_map(layout, index, nl);
        }
        n = nl.reduced_dofs();
        ldk = round_up(n, kKC);
        B = layout.cell_count();
        N = index.dof_count();
        nodes = index.node_count();

        // GEMM row order: blocks grouped by kind, each group padded to BM rows.
        row_cell.clear();
        row_kind.clear();
        row_dt.clear();
        tile_kind.clear();
        for (int kind = 0; kind < 2; ++kind) {
            size_t cnt = 0;
            for (size_t c = 0; c < B; ++c)
                if (layout.kind_at(c) == kind) {
                    row_cell.push_back(static_cast<int>(c));
                    row_kind.push_back(static_cast<uint8_t>(kind));
                    row_dt.push_back(layout.delta_t_at(c));
                    ++cnt;
                }
            while (row_cell.size() % kBM) {
                row_cell.push_back(-1);
                row_kind.push_back(static_cast<uint8_t>(kind));
                row_dt.push_back(0.0);
            }
            for (size_t t = 0; t < round_up(cnt, kBM) / kBM; ++t) tile_kind.push_back(static_cast<uint8_t>(kind));
        }
        B_pad = row_cell.size();
        m_tiles = B_pad / kBM;
        if (B_pad * ldk >= 0x7fffffffULL) throw StatusError(TSV_EINVAL, "array too large for 32-bit panel offsets");
        cell_row.assign(B, -1);
        for (size_t j = 0; j < B_pad; ++j)
            if (row_cell[j] >= 0) cell_row[row_cell[j]] = static_cast<int>(j);

        // Few 128 x 64 tiles (small arrays): switch K1 to 64 x 64 tiles.
        k1_small = m_tiles * (round_up(n, kBN) / kBN) < static_cast<size_t>(k1_grid);  // fewer tiles than CTA slots
        setup_streamk();
        prepare_k1_splitk();

        PhaseTimer pt_ren("  renumber+slots");
        // Node renumbering (first visit, blocks in super-cell-major order:
        // the nodes of each Schwarz super cell form one contiguous range)
        // + slot table.
        const size_t nn = nl.node_count();
        node_int_of_glob.assign(nodes, 0xffffffffu);
        node_glob_of_int.clear();
        node_glob_of_int.reserve(nodes);
        std::vector<int> slot_tab(nodes * 4, -1);
        const uint32_t sbn = static_cast<uint32_t>(schwarz_super_block(rows, cols));
        std::vector<int> visit;
        visit.reserve(B);
        node_super_ptr.assign(1, 0);
        for (uint32_t cy = 0; cy < (rows + sbn - 1) / sbn; ++cy)
            for (uint32_t cx = 0; cx < (cols + sbn - 1) / sbn; ++cx) {
                for (uint32_t r = cy * sbn; r < std::min(rows, (cy + 1) * sbn); ++r)
                    for (uint32_t c = cx * sbn; c < std::min(cols, (cx + 1) * sbn); ++c)
                        visit.push_back(static_cast<int>(static_cast<size_t>(r) * cols + c));
                node_super_ptr.push_back(static_cast<int>(visit.size()));  // block counts for now
            }
        const std::vector<int> super_blocks = node_super_ptr;
        for (size_t sc = 0; sc + 1 < super_blocks.size(); ++sc) {
            for (int v = super_blocks[sc]; v < super_blocks[sc + 1]; ++v) {
                const int cell = visit[v];
                const size_t j = static_cast<size_t>(cell_row[cell]);
                const uint32_t *dm = dofmap.data() + static_cast<size_t>(cell) * n;
                for (size_t rank = 0; rank < nn; ++rank) {
                    const uint32_t gnode = dm[3 * rank] / 3;
                    uint32_t &in = node_int_of_glob[gnode];
                    if (in == 0xffffffffu) {
                        in = static_cast<uint32_t>(node_glob_of_int.size());
                        node_glob_of_int.push_back(gnode);
                    }
                    int *s = slot_tab.data() + static_cast<size_t>(in) * 4;
                    int k = 0;
                    while (k < 4 && s[k] >= 0) ++k;
                    if (k == 4) throw StatusError(TSV_EINVAL, "index: a reduced node is shared by more than 4 blocks");
                    s[k] = static_cast<int>(j * ldk + rank);  // + c * nn per component
                }
            }
            node_super_ptr[sc + 1] = static_cast<int>(node_glob_of_int.size());
        }
        if (node_glob_of_int.size() != nodes) throw StatusError(TSV_EINVAL, "index: unreferenced global node");

        pt_ren.lap("  uploads");
        drop_graph();
        solution_valid = false;
        pre_kind = -1;
        oz_s = 0;
        stress.release();
        cudaStream_t s = stream;
        slots.upload(slot_tab.data(), slot_tab.size(), s);
        glob_of_int_d.upload(node_glob_of_int.data(), node_glob_of_int.size(), s);
        row_cell_d.upload(row_cell.data(), row_cell.size(), s);
        row_kind_d.upload(row_kind.data(), row_kind.size(), s);
        tile_kind_d.upload(tile_kind.data(), tile_kind.size(), s);
        {
            std::vector<uint8_t> tks;
            for (uint8_t k : tile_kind)
                for (int i = 0; i < kBM / K1SmallCfg::BM; ++i) tks.push_back(k);
            tile_kind_small_d.upload(tks.data(), tks.size(), s);
        }
        row_dt_d.upload(row_dt.data(), row_dt.size(), s);
        X.alloc(B_pad * ldk);
        Y.alloc(B_pad * ldk);
        CK(cudaMemsetAsync(X.ptr, 0, X.count * sizeof(double), s));
        CK(cudaMemsetAsync(Y.ptr, 0, Y.count * sizeof(double), s));
        for (DevBuf<double> *v : {&b, &x, &r, &p, &ap}) {
            v->alloc(N);
            CK(cudaMemsetAsync(v->ptr, 0, N * sizeof(double), s));
        }
        const size_t vec_blocks = (nodes + kVecThreads - 1) / kVecThreads;
        partial.alloc(2 * std::max<size_t>(vec_blocks, 1));
        setup_symmetry(need);
        layout_set = true;
        bc_set = false;
        set_bc_mask(std::vector<uint8_t>(N, 0), {});
        bc_set = false;
        CK(cudaStreamSynchronize(s));
    }

    // Mirror-symmetric path (sym.cuh): on when every ROM the layout uses passed
    // the symmetry check in tsv_set_rom and the kinds share the reduced tables.
    void setup_symmetry(const bool need[2]) {
        sym.on = sym.k1 = sym.corr = sym.fused = false;
        const RomHost *first = nullptr;
        for (int k = 0; k < 2; ++k) {
            if (!need[k]) continue;
            if (!rom[k].sym) return;
            if (first && (first->sred.src != rom[k].sred.src || first->sred.dst != rom[k].sred.dst)) return;
            if (!first) first = &rom[k];
        }
        if (!first || static_cast<size_t>(first->sred.n) != n) return;
        sym.on = true;
        sym.tab_kind = static_cast<int>(first - rom);
        sym.lds = first->sred.ld;
        sym.panel_smem = sym_panel_smem(first->sred.n_orbits, static_cast<int>(ldk), sym.lds);
        if (sym.panel_smem > 227 * 1024) {
            sym.on = false;
            return;
        }
        CK(cudaFuncSetAttribute(sym_panel_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sym.panel_smem)));
        CK(cudaFuncSetAttribute(sym_panel_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sym.panel_smem)));
        CK(cudaFuncSetAttribute(gemm_seg_f64<K1Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(K1Cfg::SMEM)));
        CK(cudaFuncSetAttribute(gemm_seg_f64<K6Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(K6Cfg::SMEM)));
        sym.Xs.alloc(B_pad * static_cast<size_t>(sym.lds));
        CK(cudaMemsetAsync(sym.Xs.ptr, 0, sym.Xs.count * sizeof(double), stream));
        const char *env = std::getenv("TSV_SYM_K1");
        // Large arrays, and mid-size ones whose 8-row tiles still fill three quarters of the SMs (config 2:
        // 128 tiles, 19 -> 13 us against 26.5 us for the split-K DMMA K1); TSV_SYM_K1=1 forces it (tests)
        sym.k1 = env ? *env == '1' : (!k1_small || (B_pad / 8) * 4 >= static_cast<size_t>(sm_count) * 3);
        if (!sym.k1) return;
        setup_sym_fused(*first);
        if (sym.fused) return;
        {   // the multi-kernel irrep K1 only on request: its true-residual check runs through the irrep
            // product in FP64, which does not pass at the large configs (section 3 of DESIGN.md)
            const char *ef = std::getenv("TSV_SYM_K1_FUSED");
            if (!(ef && *ef == '0')) {
                sym.k1 = false;
                return;
            }
        }
        sym.Ys.alloc(B_pad * static_cast<size_t>(sym.lds));
        CK(cudaMemsetAsync(sym.Ys.ptr, 0, sym.Ys.count * sizeof(double), stream));
        // correction operand: D32[kind][NP][KP] (the tc_local layout), one common scale
        bool any = false;
        int e = 0;
        for (int k = 0; k < 2; ++k)
            if (need[k] && rom[k].d_nonzero) {
                e = any ? std::min(e, rom[k].d_exp) : rom[k].d_exp;
                any = true;
            }
        const char *envc = std::getenv("TSV_SYM_CORR");
        if (!any || (envc && *envc == '0')) return;
        sym.corr = true;
        sym.c_scale = std::ldexp(1.0, -e);
        sym.KP = static_cast<int>(round_up(n, kTcBK));
        sym.ntn = static_cast<int>((n + 255) / 256);
        sym.BN = static_cast<int>(round_up((n + sym.ntn - 1) / sym.ntn, 16));
        sym.NP = sym.ntn * sym.BN;
        sym.LD = std::max(sym.KP, sym.NP);
        std::vector<float> d32(static_cast<size_t>(2) * sym.NP * sym.KP, 0.f);
        for (int k = 0; k < 2; ++k) {
            const RomHost &m = need[k] ? rom[k] : *first;
            if (!m.d_nonzero) continue;
            const float sc = std::ldexp(1.0f, e - m.d_exp);
            for (size_t a = 0; a < n; ++a)
                for (size_t b = 0; b < n; ++b) {
                    uint32_t u;
                    const float v = m.d32_host[a * n + b] * sc;
                    std::memcpy(&u, &v, 4);
                    u = (u + 0x1000u) & 0xffffe000u;  // round to TF32 (10 mantissa bits)
                    float w;
                    std::memcpy(&w, &u, 4);
                    d32[(static_cast<size_t>(k) * sym.NP + a) * sym.KP + b] = w;
                }
        }
        sym.d32.upload(d32.data(), d32.size(), stream);
        if (B_pad * static_cast<size_t>(sym.LD) >= 0x7fffffffULL) {
            sym.corr = sym.k1 = false;
            return;
        }
        sym.X32.alloc(B_pad * static_cast<size_t>(sym.LD));
        sym.Yc32.alloc(B_pad * static_cast<size_t>(sym.LD));
        CK(cudaMemsetAsync(sym.X32.ptr, 0, sym.X32.count * sizeof(float), stream));
        CK(cudaMemsetAsync(sym.Yc32.ptr, 0, sym.Yc32.count * sizeof(float), stream));
        std::vector<int> tt(tile_kind.begin(), tile_kind.end());
        sym.tile_type.upload(tt.data(), tt.size(), stream);
        std::vector<int2> pr;
        for (size_t i = 0; i < tt.size();) {
            if (i + 1 < tt.size() && tt[i + 1] == tt[i]) {
                pr.push_back(make_int2(static_cast<int>(i), static_cast<int>(i + 1)));
                i += 2;
            } else {
                pr.push_back(make_int2(static_cast<int>(i), -1));
                i += 1;
            }
        }
        const bool use_pairs = sym.BN <= 256 && tc_pair_smem_bytes(sym.BN) <= 227 * 1024;
        sym.npairs = use_pairs ? static_cast<int>(pr.size()) : 0;
        if (use_pairs) sym.pairs.upload(pr.data(), pr.size(), stream);
        encode_f32_map(&sym.tmA, sym.X32.ptr, sym.KP, B_pad, static_cast<uint32_t>(kTcBM), sym.LD);
        encode_f32_map(&sym.tmB, sym.d32.ptr, sym.KP, static_cast<uint64_t>(2) * sym.NP, static_cast<uint32_t>(sym.BN), sym.KP);
        CK(cudaFuncSetAttribute(tc_local_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes(256)));
        CK(cudaFuncSetAttribute(tc_local_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_pair_smem_bytes(256)));
    }

    // Fused K1 on mirror-symmetric ROMs (sym_k1_fused_kernel): item / column /
    // tile tables. TSV_SYM_K1_FUSED=0 keeps the multi-kernel path (panel
    // passes + segmented GEMM); TSV_SYM_K1_MF=2|3|4 picks 16 / 24 / 32 rows per CTA.
    template <int MF, int WARPS, int MINB, int SLOTS = kSymSlots>
    bool sym_fused_config() {
        auto kern = sym_k1_fused_kernel<MF, WARPS, MINB, SLOTS>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sym.f_smem)) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * WARPS, sym.f_smem));
        if (occ < 1) return false;
        sym.f_max_grid = occ * sm_count;
        if (const char *gr = std::getenv("TSV_SYM_GRID")) sym.f_max_grid = std::max(1, std::min(sym.f_max_grid, std::atoi(gr)));
        sym.f_grid = std::min(sym.f_tiles, sym.f_max_grid);
        return true;
    }

    bool sym_pipe_config() {
        auto kern = sym_k1_pipe_kernel<2, 16>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sym.f_smem)) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, sym.f_smem));
        if (occ < 1) return false;
        sym.f_max_grid = occ * sm_count;
        sym.f_grid = std::min(sym.f_tiles, sym.f_max_grid);
        return true;
    }

    void setup_sym_fused(const RomHost &first) {
        sym.fused = false;
        const char *env = std::getenv("TSV_SYM_K1_FUSED");
        if (env && *env == '0') return;
        const char *emf = std::getenv("TSV_SYM_K1_MF");
        const int mf = emf ? std::atoi(emf) : 2;
        if (mf < 1 || mf > 4) return;
        const char *ep = std::getenv("TSV_SYM_K1_PIPE");
        sym.pipe = mf == 2 && ep && *ep == '1';
        const int warps = sym.pipe ? 16 : mf == 1 ? 4 : mf == 2 ? 8 : 16;  // mf = 1: 8 rows, 4 warps, 4 CTAs per SM (experiment)
        const SymK1Pack &pk = first.k1f;
        std::vector<short> flush;
        if (pk.items.empty() || pk.flush_rounds(warps, flush) > (mf == 1 ? 3 : kSymSlots) - 1) return;
        std::vector<SymK1Item> items(pk.items.size());
        for (size_t i = 0; i < items.size(); ++i) {
            SymK1Item it{};
            it.b_off = pk.items[i].b_off;
            it.ksteps = pk.items[i].ksteps;
            it.ksteps4 = pk.items[i].ksteps4;
            it.kcol = pk.items[i].kcol;
            it.ncol = pk.items[i].ncol;
            it.nvalid = pk.items[i].nvalid;
            it.flush_round = flush[i];
            items[i] = it;
        }
        sym.f_mf = mf;
        sym.f_items = static_cast<int>(items.size());
        sym.f_rounds = (sym.f_items + warps - 1) / warps;
        sym.f_coltab = static_cast<int>(pk.coltab.size());
        sym.f_smem = (sym.pipe ? sym_k1_pipe_smem : sym_k1_smem)(mf, static_cast<int>(ldk), first.sred.n_orbits, sym.f_coltab, sym.f_items);
        if (sym.f_smem > 227 * 1024) return;
        // row tiles: runs of same-kind M tiles cut into 8 MF rows
        std::vector<int4> tiles;
        const int R = 8 * mf;
        for (size_t t = 0; t < tile_kind.size();) {
            size_t e = t;
            while (e < tile_kind.size() && tile_kind[e] == tile_kind[t]) ++e;
            const int r0 = static_cast<int>(t * kBM), r1 = static_cast<int>(e * kBM);
            for (int r = r0; r < r1; r += R) tiles.push_back(make_int4(r, std::min(R, r1 - r), tile_kind[t], 0));
            t = e;
        }
        sym.f_tiles = static_cast<int>(tiles.size());
        const bool ok = sym.pipe ? sym_pipe_config() : mf == 1 ? sym_fused_config<1, 4, 4, 3>() : mf == 2 ? sym_fused_config<2, 8, 2>()
                        : mf == 3 ? sym_fused_config<3, 16, 1>() : sym_fused_config<4, 16, 1>();
        if (!ok) return;
        // Balanced tail: the tiles past the last full wave of the grid are cut into single row
        // fragments (8 rows: half the butterflies and products of a 16-row tile), so the last
        // wave is short instead of leaving most CTAs idle for a whole tile
        {
            // (an array with fewer tiles than CTA slots is all tail: every tile is cut)
            const int T = static_cast<int>(tiles.size()), rem = T % sym.f_max_grid;
            const char *bt = std::getenv("TSV_SYM_K1_TAIL");
            if (rem > 0 && rem * mf <= sym.f_max_grid && !(bt && *bt == '0')) {
                std::vector<int4> cut(tiles.begin(), tiles.end() - rem);
                for (int i = T - rem; i < T; ++i)
                    for (int r = 0; r < tiles[i].y; r += 8)
                        cut.push_back(make_int4(tiles[i].x + r, std::min(8, tiles[i].y - r), tiles[i].z, 0));
                tiles.swap(cut);
                sym.f_tiles = static_cast<int>(tiles.size());
                sym.f_grid = std::min(sym.f_tiles, sym.f_max_grid);
            }
        }
        // K'' fragment streams: warp w reads its items (w, w + warps, ...) back to back, every
        // item slot padded to cpi chunks of kSymKB k-steps (cpi % kSymRing == 0: the kernel's register ring)
        int max_chunks = 1;
        for (const auto &it : pk.items) max_chunks = std::max(max_chunks, it.ksteps4 / kSymKB);
        sym.f_cpi = (max_chunks + kSymRing - 1) / kSymRing * kSymRing;
        const size_t slot = static_cast<size_t>(sym.f_cpi) * kSymKB * 64;
        for (int k = 0; k < 2; ++k) {
            const RomHost &m = rom[k].set && rom[k].sym ? rom[k] : first;
            std::vector<double> st(static_cast<size_t>(warps) * sym.f_rounds * slot, 0.0);
            for (size_t i = 0; i < m.k1f.items.size() && i < pk.items.size(); ++i) {
                const auto &it = m.k1f.items[i];
                const size_t w = i % warps, t = i / warps;
                std::memcpy(st.data() + (w * sym.f_rounds + t) * slot, m.k1f.bf.data() + it.b_off,
                            static_cast<size_t>(it.ksteps4) * 64 * sizeof(double));
            }
            sym.f_stream[k].upload(st.data(), st.size(), stream);
        }
        sym.f_tile_tab.upload(tiles.data(), tiles.size(), stream);
        sym.f_item_tab.upload(items.data(), items.size(), stream);
        sym.f_col_tab.upload(pk.coltab.data(), pk.coltab.size(), stream);
        CK(cudaStreamSynchronize(stream));
        sym.fused = true;
    }

    void launch_k1_sym_fused(const int *done, const int *skip) {
        const RomHost &mt = rom[sym.tab_kind];
        SymK1Params sp{};
        sp.X = X.ptr;
        sp.Y = Y.ptr;
        sp.ld = static_cast<long long>(ldk);
        sp.ldk = static_cast<int>(ldk);
        sp.tiles = sym.f_tile_tab.ptr;
        sp.n_tiles = sym.f_tiles;
        sp.Bf[0] = sym.f_stream[0].ptr;
        sp.Bf[1] = sym.f_stream[1].ptr;
        sp.cpi = sym.f_cpi;
        sp.items = sym.f_item_tab.ptr;
        sp.n_items = sym.f_items;
        sp.rounds = sym.f_rounds;
        sp.orb = mt.d_ssrc.ptr;
        sp.n_orbits = mt.sred.n_orbits;
        sp.coltab = sym.f_col_tab.ptr;
        sp.n_coltab = sym.f_coltab;
        sp.done = done;
        sp.skip_flag = skip;
        sp.tile_counter = tile_counter.ptr;
        if (const char *ab = std::getenv("TSV_SYM_ABLATE")) sp.ablate = std::atoi(ab);
        if (sym.pipe) launch_pdl(sym_k1_pipe_kernel<2, 16>, sym.f_grid, 512, sym.f_smem, stream, sp);
        else if (sym.f_mf == 1) launch_pdl(sym_k1_fused_kernel<1, 4, 4, 3>, sym.f_grid, 128, sym.f_smem, stream, sp);
        else if (sym.f_mf == 2) launch_pdl(sym_k1_fused_kernel<2, 8, 2>, sym.f_grid, 256, sym.f_smem, stream, sp);
        else if (sym.f_mf == 3) launch_pdl(sym_k1_fused_kernel<3, 16, 1>, sym.f_grid, 512, sym.f_smem, stream, sp);
        else launch_pdl(sym_k1_fused_kernel<4, 16, 1>, sym.f_grid, 512, sym.f_smem, stream, sp);
        ++launches;
        CK(cudaGetLastError());
    }

    // fp32 2-D tensor map: [rows][cols] with a row stride, {32 x box_rows} boxes, 128-byte swizzle
    static void encode_f32_map(CUtensorMap *m, void *ptr, int cols, uint64_t rows_, uint32_t box_rows, int row_stride) {
        using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                      const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        static EncodeFn encode = [] {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q{};
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                fn = nullptr;
            return reinterpret_cast<EncodeFn>(fn);
        }();
        if (!encode) throw StatusError(TSV_ECUDA, "cuTensorMapEncodeTiled unavailable");
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), rows_};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride) * sizeof(float)};
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(kTcBK), box_rows};
        const cuuint32_t estr[2] = {1, 1};
        if (encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            throw StatusError(TSV_ECUDA, "tensor map encoding failed");
    }

    // Stream-K boundaries for K1: split the linear (tile, k-chunk) space into
    // k1_grid ranges of equal DMMA work (a chunk of a tile costs its number
    // of valid 8-column fragments). Requires >= one full tile per range.
    void setup_streamk() {
        k1_streamk = false;
        if (k1_small || !sk_resident || getenv_flag("TSV_NO_STREAMK")) return;
        const size_t nt = round_up(n, kBN) / kBN, T = m_tiles * nt, KC = ldk / kKC, G = static_cast<size_t>(k1_grid);
        const size_t nf = (n + 7) / 8, fpt = kBN / 8;
        std::vector<double> w(nt);
        for (size_t t = 0; t < nt; ++t) w[t] = static_cast<double>(std::min(fpt, nf - t * fpt));
        double per_m = 0.0;
        for (double v : w) per_m += v;
        const double C = per_m * static_cast<double>(m_tiles) * static_cast<double>(KC);
        // Wave efficiency of the dynamic tile queue: work / (tile rounds x slots).
        // Stream-K pays extra segment prologues and partial fix-ups, so it is
        // used only when the queue would waste > 12% in its last wave
        // (deterministic choice: results stay bitwise reproducible).
        const double rounds = std::ceil(static_cast<double>(T) / static_cast<double>(G));
        const double eff = (C / (static_cast<double>(KC) * static_cast<double>(fpt))) / (rounds * static_cast<double>(G));
        if (eff > 0.88 && !getenv_flag("TSV_STREAMK")) return;
        std::vector<int> start(G + 1, 0);
        size_t it = 0;
        double cum = 0.0;
        for (size_t g = 1; g < G; ++g) {
            const double target = C * static_cast<double>(g) / static_cast<double>(G);
            while (it < T * KC && cum + w[(it / KC) % nt] <= target) {
                cum += w[(it / KC) % nt];
                ++it;
            }
            start[g] = static_cast<int>(it);
        }
        start[G] = static_cast<int>(T * KC);
        for (size_t g = 0; g < G; ++g)
            if (static_cast<size_t>(start[g + 1] - start[g]) < KC) return;  // a tile could span 3 CTAs
        sk_start.upload(start.data(), start.size(), stream);
        sk_flag.alloc(G);
        CK(cudaMemsetAsync(sk_flag.ptr, 0, G * sizeof(int), stream));
        sk_work.alloc(G * static_cast<size_t>(K1Cfg::FM * K1Cfg::FN * 2 * K1Cfg::THREADS));
        k1_streamk = true;
    }

    // Super-block side s of the Schwarz coarse space: the smallest s whose
    // corner lattice has <= TSV_AS_COARSE_MAX (16384) coarse DoFs, or TSV_AS_S.
    // It also fixes the node numbering (set_layout), so it depends only on
    // the array shape. Measured at config 3 (B200): s = 3 (7350 coarse DoFs)
    // 75 iterations x 0.537 ms; s = 2 (15606) 57 x 0.628 ms; s = 1 does not
    // cut iterations further (60 in the FP64 oracle, tools/coarse_quant_scan.py).
    static int schwarz_super_block(uint32_t rows, uint32_t cols) {
        if (getenv("TSV_AS_S")) return std::max(1, std::atoi(getenv("TSV_AS_S")));
        const size_t cap = getenv("TSV_AS_COARSE_MAX") ? std::strtoul(getenv("TSV_AS_COARSE_MAX"), nullptr, 10) : 16384;
        for (int sb = 1;; ++sb) {
            const size_t SX = (cols + sb - 1) / sb, SY = (rows + sb - 1) / sb;
            if ((SX + 1) * (SY + 1) * 6 <= cap || (SX == 1 && SY == 1)) return sb;
        }
    }

    // f(r) for r in [0, rows) on the host threads (rows are independent).
    template <typename F>
    static void parallel_rows(uint32_t rows, F &&f) {
        const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), rows));
        if (nt == 1) {
            for (uint32_t r = 0; r < rows; ++r) f(r);
            return;
        }
        std::vector<std::thread> pool;
        for (unsigned w = 0; w < nt; ++w)
            pool.emplace_back([&, w] {
                for (uint32_t r = w; r < rows; r += nt) f(r);
            });
        for (auto &t : pool) t.join();
    }

    static bool getenv_flag(const char *name) {
        const char *v = std::getenv(name);
        return v && *v && *v != '0';
    }

    // Online dT update (ArrayLayout::delta_t, global.hpp:16-32): the
    // thermal load is the only input that changes per call in the reference's
    // online stage. Index, dof map, slots, masks, BCs and the preconditioner
    // (a function of kinds and BCs only) stay; the RHS is re-assembled on the
    // device on next use and recovery reads the new per-row dT.
    void set_delta_t(const double *dt, size_t ndt) {
        PhaseTimer pt("set_delta_t");
        if (!layout_set) throw StatusError(TSV_ESTATE, "set_delta_t: no layout set");
        if (!dt && ndt) throw StatusError(TSV_EINVAL, "layout: delta_t pointer is NULL");
        if (ndt != 1 && ndt != B) throw StatusError(TSV_EINVAL, "layout: delta_t must have one entry or rows*cols entries");
        layout.delta_t.assign(dt, dt + ndt);
        dt_host.resize(B_pad);
        for (size_t j = 0; j < B_pad; ++j) dt_host[j] = row_cell[j] >= 0 ? layout.delta_t_at(row_cell[j]) : 0.0;
        row_dt_d.upload(dt_host.data(), dt_host.size(), stream);
        rhs_dirty = true;
        solution_valid = false;
        CK(cudaStreamSynchronize(stream));  // dt_host is reused by the next call
    }

    // ------------------------------------------------------------------ BC
    // mask: constrained DoFs (reference numbering); vals: the prescribed
    // (dof, value) pairs, sorted (only the non-zero values matter for lifting).
    void set_bc_mask(std::vector<uint8_t> mask, const std::vector<std::pair<uint32_t, double>> &vals) {
        PhaseTimer pt("set_bc_mask");
        constrained = std::move(mask);
        any_g = false;
        for (const auto &e : vals)
            if (e.second != 0.0) any_g = true;
        g.clear();
        if (any_g) {
            g.assign(N, 0.0);
            for (const auto &e : vals) g[e.first] = e.second;
        }
        std::vector<uint8_t> cm_int(N);
        for (size_t in = 0; in < nodes; ++in)
            for (int c = 0; c < 3; ++c) cm_int[c * nodes + in] = constrained[3 * node_glob_of_int[in] + c];
        cmask.upload(cm_int.data(), N, stream);
        bc_set = true;
        pre_kind = -1;
        solution_valid = false;
        rhs_dirty = true;  // assembled on first use (set_layout + set_bc assemble it once)
    }

    void ensure_rhs() {
        if (!rhs_dirty) return;
        build_rhs();
        rhs_dirty = false;
    }

    // Device vector (internal order) -> host array in reference DoF order.
    void copy_to_reference(const double *v_int, double *out) {
        uref.alloc(N);
        to_reference_kernel<<<vec_grid(), kVecThreads, 0, stream>>>(static_cast<int>(nodes), glob_of_int_d.ptr, v_int,
                                                                    uref.ptr);
        ++launches;
        CK(cudaGetLastError());
        d2h(out, uref.ptr, N * sizeof(double), stream);
    }

    template <typename T>
    std::vector<T> to_internal(const T *v) const {
        std::vector<T> out(N);
        for (size_t in = 0; in < nodes; ++in)
            for (int c = 0; c < 3; ++c) out[c * nodes + in] = v[3 * node_glob_of_int[in] + c];
        return out;
    }
    template <typename T>
    void to_reference(const T *v_int, T *out) const {
        for (size_t in = 0; in < nodes; ++in)
            for (int c = 0; c < 3; ++c) out[3 * node_glob_of_int[in] + c] = v_int[c * nodes + in];
    }

    // Assembled load (global_stage.cpp:135-142, cell order, bit-exact) and
    // symmetric lifting (fem.cpp:223-260): b_c = g, b_f -= A_fc g.
    void build_rhs() {
        PhaseTimer pt("build_rhs");
        const RomHost &m0 = rom[0].set ? rom[0] : rom[1];
        const RomHost &m1 = rom[1].set ? rom[1] : rom[0];
        DevBuf<double> gd;
        if (any_g) {
            std::vector<double> gi = to_internal(g.data());
            gd.upload(gi.data(), N, stream);
        }
        rhs_kernel<<<vec_grid(), kVecThreads, 0, stream>>>(static_cast<int>(nodes), static_cast<int>(n / 3),
                                                           static_cast<long long>(ldk), slots.ptr, row_cell_d.ptr,
                                                           row_kind_d.ptr, row_dt_d.ptr, m0.d_bel.ptr, m1.d_bel.ptr,
                                                           cmask.ptr, any_g ? gd.ptr : nullptr, b.ptr);
        ++launches;
        CK(cudaGetLastError());
        if (any_g) {  // b_f -= A_fc g on the device
            CK(cudaMemcpyAsync(r.ptr, gd.ptr, N * sizeof(double), cudaMemcpyDeviceToDevice, stream));
            launch_scatter(r.ptr, 2);
            launch_k1(nullptr);
            gather_vec_kernel<<<vec_grid(), kVecThreads, 0, stream>>>(static_cast<int>(nodes), static_cast<int>(n / 3), slots.ptr, cmask.ptr,
                                                                    Y.ptr, b.ptr, b.ptr, 1);
            ++launches;
            CK(cudaGetLastError());
        }
        CK(cudaStreamSynchronize(stream));
    }

    // Jacobi / 3x3 block-Jacobi of the lifted matrix, built on the host in
    // the reference's summation order (linalg.cpp:223-262).
    void build_precond(int kind) {
        if (pre_kind == kind) return;
        if (kind == TSV_PRECOND_DIAGONAL) {
            std::vector<double> d(N, 0.0);
            for (size_t c = 0; c < B; ++c) {
                const RomHost &m = rom[layout.kind_at(c)];
                const uint32_t *dm = dofmap.data() + c * n;
                for (size_t a = 0; a < n; ++a) d[dm[a]] += m.k_r[a * n + a];
            }
            for (size_t i = 0; i < N; ++i) {
                if (constrained[i]) d[i] = 1.0;
                d[i] = d[i] != 0.0 ? 1.0 / d[i] : 1.0;
            }
            std::vector<double> di = to_internal(d.data());
            pre.upload(di.data(), N, stream);
        } else if (kind == TSV_PRECOND_BLOCK_DIAGONAL) {
            std::vector<double> mb(nodes * 9, 0.0);
            const size_t nn = nl.node_count();
            for (size_t c = 0; c < B; ++c) {
                const RomHost &m = rom[layout.kind_at(c)];
                const uint32_t *dm = dofmap.data() + c * n;
                for (size_t rank = 0; rank < nn; ++rank) {
                    const size_t node = dm[3 * rank] / 3;
                    for (int i = 0; i < 3; ++i)
                        for (int j = 0; j < 3; ++j) mb[node * 9 + i * 3 + j] += m.k_r[(3 * rank + i) * n + 3 * rank + j];
                }
            }
            std::vector<double> inv_int(nodes * 9);
            for (size_t node = 0; node < nodes; ++node) {
                double mm[9];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) {
                        double v = mb[node * 9 + i * 3 + j];
                        if (constrained[3 * node + i]) v = (i == j) ? 1.0 : 0.0;
                        else if (constrained[3 * node + j]) v = 0.0;
                        mm[i * 3 + j] = v;
                    }
                const double *m = mm;
                double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                             m[2] * (m[3] * m[7] - m[4] * m[6]);
                double inv[9];
                if (std::abs(det) < 1e-300) {
                    for (int i = 0; i < 9; ++i) inv[i] = 0.0;
                    for (int i = 0; i < 3; ++i) {
                        double dd = m[i * 3 + i];
                        inv[i * 3 + i] = dd != 0.0 ? 1.0 / dd : 1.0;
                    }
                } else {
                    inv[0] = (m[4] * m[8] - m[5] * m[7]) / det;
                    inv[1] = (m[2] * m[7] - m[1] * m[8]) / det;
                    inv[2] = (m[1] * m[5] - m[2] * m[4]) / det;
                    inv[3] = (m[5] * m[6] - m[3] * m[8]) / det;
                    inv[4] = (m[0] * m[8] - m[2] * m[6]) / det;
                    inv[5] = (m[2] * m[3] - m[0] * m[5]) / det;
                    inv[6] = (m[3] * m[7] - m[4] * m[6]) / det;
                    inv[7] = (m[1] * m[6] - m[0] * m[7]) / det;
                    inv[8] = (m[0] * m[4] - m[1] * m[3]) / det;
                }
                const size_t in = node_int_of_glob[node];
                for (int k = 0; k < 9; ++k) inv_int[k * nodes + in] = inv[k];
            }
            pre.upload(inv_int.data(), inv_int.size(), stream);
        } else if (kind == TSV_PRECOND_SCHWARZ2) {
            pre.alloc(1);
            build_schwarz2();
        } else {
            pre.alloc(1);
        }
        pre_kind = kind;
        drop_graph();
    }

    // --------------------------------------------------- two-level Schwarz
    struct SolverHandles {
        cusolverDnHandle_t sol = nullptr;
        cublasHandle_t blas = nullptr;
        ~SolverHandles() {
            if (sol) cusolverDnDestroy(sol);
            if (blas) cublasDestroy(blas);
        }
    };

    // In-place SPD inverse on the device (column-major, lower triangle
    // valid on return): potrf + potri, no host synchronisation. `info`
    // collects the factorisation status, checked once at the end.
    void spd_inverse_inplace(SolverHandles &h, double *dA, int nn, DevBuf<double> &work, int *info) {
        int lwork = 0, lwork2 = 0;
        if (cusolverDnDpotrf_bufferSize(h.sol, CUBLAS_FILL_MODE_LOWER, nn, dA, nn, &lwork) != CUSOLVER_STATUS_SUCCESS ||
            cusolverDnDpotri_bufferSize(h.sol, CUBLAS_FILL_MODE_LOWER, nn, dA, nn, &lwork2) != CUSOLVER_STATUS_SUCCESS)
            throw StatusError(TSV_ECUDA, "schwarz2: cuSOLVER buffer query failed");
        const size_t need = static_cast<size_t>(std::max(std::max(lwork, lwork2), 1));
        if (work.count < need) work.alloc(need);
        if (cusolverDnDpotrf(h.sol, CUBLAS_FILL_MODE_LOWER, nn, dA, nn, work.ptr, lwork, info) != CUSOLVER_STATUS_SUCCESS ||
            cusolverDnDpotri(h.sol, CUBLAS_FILL_MODE_LOWER, nn, dA, nn, work.ptr, lwork2, info + 1) !=
                CUSOLVER_STATUS_SUCCESS)
            throw StatusError(TSV_ECUDA, "schwarz2: potrf/potri failed");
    }

    // Launch with programmatic stream serialisation (PDL) unless TSV_NO_PDL:
    // the PCG iteration kernels (each starts with griddepcontrol.wait).
    template <typename... KArgs, typename... Args>
    void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
        const bool off = getenv_flag("TSV_NO_PDL");  // read per launch (graph capture, run_cg prologue)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        int na = 0;
        if (!off) {
            attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[na].val.programmaticStreamSerializationAllowed = 1;
            ++na;
        }
        // CTA scheduling priority (captured into the graph nodes): the split
        // Schwarz loop keeps the main chain (K1) ahead of the side chain's
        // many small CTAs; the serial loop prefers the coarse chain, its
        // longer branch.
        const int prio = st == side ? prio_side : prio_main;
        if (prio != 0) {
            attr[na].id = cudaLaunchAttributePriority;
            attr[na].val.priority = prio;
            ++na;
        }
        cfg.attrs = attr;
        cfg.numAttrs = na;
        CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
    }

    // Split-K factor of the small-array K1 (TSV_K1_SPLITK=0 disables): as many
    // k-slices as fill the resident CTA slots once, at most one per k-chunk.
    DevBuf<double> sk1_work;
    DevBuf<unsigned> sk1_ticket;
    int k1_split_k(int tiles, int k_chunks) const {
        const char *v = getenv("TSV_K1_SPLITK");
        if (v && *v == '0') return 1;
        return std::min(std::min(k_chunks, kSplitKMax), std::max(1, k1s_grid / std::max(1, tiles)));
    }
    static constexpr int kSplitKMax = 8;
    // buffers sized at set_layout (never inside a graph capture)
    void prepare_k1_splitk() {
        if (!k1_small) return;
        const int tiles = static_cast<int>(B_pad / K1SmallCfg::BM) * static_cast<int>(round_up(n, K1SmallCfg::BN) / K1SmallCfg::BN);
        const int S = k1_split_k(tiles, static_cast<int>(ldk / K1SmallCfg::KC));
        if (S <= 1) return;
        const size_t need = static_cast<size_t>(tiles) * S * K1SmallCfg::FM * K1SmallCfg::FN * 2 * K1SmallCfg::THREADS;
        if (sk1_work.count < need) sk1_work.alloc(need);
        if (sk1_ticket.count < static_cast<size_t>(tiles)) sk1_ticket.alloc(static_cast<size_t>(tiles));
        CK(cudaMemsetAsync(sk1_ticket.ptr, 0, sk1_ticket.count * sizeof(unsigned), stream));
    }

    int prio_main = 0, prio_side = 0;  // launch priorities (set per loop variant in ensure_graph)
    void set_launch_priorities() {
        int least = 0, greatest = 0;
        CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        // Opt-in (TSV_PRIO=1): measured on B200 at config 3, no change either
        // way (0.6796 vs 0.6793 ms split, 0.6284 vs 0.6282 ms serial).
        if (!getenv_flag("TSV_PRIO")) {
            prio_main = prio_side = 0;
        } else if (pre_kind == TSV_PRECOND_SCHWARZ2 && as_split()) {
            prio_main = greatest;
            prio_side = least;
        } else {
            prio_main = 0;
            prio_side = greatest;
        }
    }

    SolverHandles solver;   // created on first use, kept for the context's lifetime
    SolverHandles solver2;  // the coarse inverse's (worker thread, side stream)

    void build_schwarz2() {
        PhaseTimer pt("build_schwarz2");
        const auto t0 = std::chrono::steady_clock::now();
        if (!solver.sol && (cusolverDnCreate(&solver.sol) != CUSOLVER_STATUS_SUCCESS ||
                            cublasCreate(&solver.blas) != CUBLAS_STATUS_SUCCESS))
            throw StatusError(TSV_ECUDA, "schwarz2: cuSOLVER/cuBLAS init failed");
        SolverHandles &h = solver;
        cusolverDnSetStream(h.sol, stream);
        cublasSetStream(h.blas, stream);
        const uint32_t rows = layout.rows, cols = layout.cols;
        const size_t nn = n / 3;
        const bool dbg = getenv_flag("TSV_DEBUG"), timing = getenv_flag("TSV_TIMING");
        auto tick = [&](const char *what) {  // TSV_DEBUG: device-synchronised; TSV_TIMING: host time only
            if (dbg) cudaStreamSynchronize(stream);
            if (dbg || timing)
                std::fprintf(stderr, "[schwarz2] %-28s %8.1f ms\n", what,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        };
        DevBuf<double> work;
        DevBuf<int> cinfo;
        cinfo.alloc(2);
        CK(cudaMemsetAsync(cinfo.ptr, 0, 2 * sizeof(int), stream));
        // --- 1. coarse space (first: its dense inverse runs on the device while
        // the host builds the local stage): corners of s x s super-blocks, bottom/top planes
        // per-axis lattice steps: x uses n_x, y uses n_y, z uses n_z
        // (NodeLayout axes, config.cpp:293-295; lat_y = rows*(n_y-1)+1)
        const uint32_t q = nl.n_x, qy = nl.n_y, qz = nl.n_z;
        const int sb = schwarz_super_block(rows, cols);
        if (node_super_ptr.size() != static_cast<size_t>(((cols + sb - 1) / sb) * ((rows + sb - 1) / sb)) + 1)
            throw StatusError(TSV_ESTATE, "schwarz2: super-block size changed since set_layout");
        as2.s = sb;
        as2.SX = static_cast<int>((cols + sb - 1) / sb);
        as2.SY = static_cast<int>((rows + sb - 1) / sb);
        as2.step = sb * static_cast<int>(q - 1);
        as2.step_y = sb * static_cast<int>(qy - 1);
        as2.Nc = (as2.SX + 1) * (as2.SY + 1) * 6;
        as2.ncells = as2.SX * as2.SY;
        std::vector<short4> lat(nodes);
        for (size_t in = 0; in < nodes; ++in) {
            const auto &L = index.lattice_of_node[node_glob_of_int[in]];
            lat[in] = make_short4(static_cast<short>(L[0]), static_cast<short>(L[1]), static_cast<short>(L[2]), 0);
        }
        as2.lat.upload(lat.data(), lat.size(), stream);
        as2.cell_ptr.upload(node_super_ptr.data(), node_super_ptr.size(), stream);
        {
            std::vector<int> nc(nodes);
            std::vector<double4> ct(static_cast<size_t>(as2.ncells));
            for (int c = 0; c < as2.ncells; ++c) {
                for (int v = node_super_ptr[c]; v < node_super_ptr[c + 1]; ++v) nc[v] = c;
                const int x0 = (c % as2.SX) * as2.step, y0 = (c / as2.SX) * as2.step_y;
                const int x1 = std::min<int>(x0 + as2.step, static_cast<int>(index.lat_x) - 1);
                const int y1 = std::min<int>(y0 + as2.step_y, static_cast<int>(index.lat_y) - 1);
                ct[c] = make_double4(x0, y0, 1.0 / static_cast<double>(x1 - x0), 1.0 / static_cast<double>(y1 - y0));
            }
            as2.node_cell.upload(nc.data(), nc.size(), stream);
            as2.celltab.upload(ct.data(), ct.size(), stream);
        }
        if (partial.count < 2 * static_cast<size_t>(as2.ncells) * kAsSplit)
            partial.alloc(2 * static_cast<size_t>(as2.ncells) * kAsSplit);
        as2.cellpart.alloc(static_cast<size_t>(as2.ncells) * kAsSplit * 24);
        as2.rc.alloc(as2.Nc);
        as2.zc.alloc(as2.Nc);
        // Galerkin A_c = sum_b P_b^T K_b P_b (P_b relative to b's super cell,
        // zero on constrained DoFs). Blocks with identical P_b (kind, offsets
        // in the cell, cell extents, constrained pattern) share one 24 x 24
        // product; the products are batched per kind on cuBLAS.
        std::map<std::vector<long>, int> key_id;
        std::vector<int> key_of(B), key_kind, key_local;
        std::vector<double> Pall[2];  // per kind, column-major n x 24 each
        int nkind_keys[2] = {0, 0};
        const auto &snodes = nl.surface_nodes;
        // per-cell keys on host threads (the constrained scan is B x n random
        // reads), then numbered serially in cell order (deterministic ids)
        std::vector<std::vector<long>> keys(B);
        parallel_rows(rows, [&](uint32_t r) {
            for (uint32_t c = 0; c < cols; ++c) {
                const size_t cell = static_cast<size_t>(r) * cols + c;
                const uint32_t *dm = dofmap.data() + cell * n;
                const int cx = static_cast<int>(c) / sb, cy = static_cast<int>(r) / sb;
                const long x0 = static_cast<long>(cx) * as2.step, y0 = static_cast<long>(cy) * as2.step_y;
                const long x1 = std::min<long>(x0 + as2.step, index.lat_x - 1), y1 = std::min<long>(y0 + as2.step_y, index.lat_y - 1);
                const long bx = static_cast<long>(c) * (q - 1), by = static_cast<long>(r) * (qy - 1);
                std::vector<long> &key = keys[cell];
                key = {layout.kind_at(cell), bx - x0, x1 - x0, by - y0, y1 - y0};
                for (size_t a = 0; a < n; ++a)
                    if (constrained[dm[a]]) key.push_back(static_cast<long>(a));
            }
        });
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t c = 0; c < cols; ++c) {
                const size_t cell = static_cast<size_t>(r) * cols + c;
                const uint32_t *dm = dofmap.data() + cell * n;
                const int cx = static_cast<int>(c) / sb, cy = static_cast<int>(r) / sb;
                const long x0 = static_cast<long>(cx) * as2.step, y0 = static_cast<long>(cy) * as2.step_y;
                const long x1 = std::min<long>(x0 + as2.step, index.lat_x - 1), y1 = std::min<long>(y0 + as2.step_y, index.lat_y - 1);
                const long bx = static_cast<long>(c) * (q - 1), by = static_cast<long>(r) * (qy - 1);
                const std::vector<long> &key = keys[cell];
                auto it = key_id.find(key);
                if (it == key_id.end()) {
                    it = key_id.emplace(key, static_cast<int>(key_kind.size())).first;
                    const int kd = layout.kind_at(cell);
                    key_kind.push_back(kd);
                    key_local.push_back(nkind_keys[kd]++);
                    const size_t off = Pall[kd].size();
                    Pall[kd].resize(off + n * 24, 0.0);
                    double *Pb = Pall[kd].data() + off;
                    for (size_t rank = 0; rank < nn; ++rank) {
                        const double tx = static_cast<double>(bx + snodes[rank][0] - x0) / static_cast<double>(x1 - x0);
                        const double ty = static_cast<double>(by + snodes[rank][1] - y0) / static_cast<double>(y1 - y0);
                        const double tz = static_cast<double>(snodes[rank][2]) / static_cast<double>(qz - 1);
                        for (int k = 0; k < 8; ++k) {
                            const double w = ((k & 1) ? tx : 1.0 - tx) * ((k & 2) ? ty : 1.0 - ty) * ((k & 4) ? tz : 1.0 - tz);
                            for (int comp = 0; comp < 3; ++comp) {
                                const size_t a = 3 * rank + comp;
                                if (!constrained[dm[a]]) Pb[(3 * k + comp) * n + a] = w;
                            }
                        }
                    }
                }
                key_of[cell] = it->second;
            }
        const int nkeys = static_cast<int>(key_kind.size());
        tick("coarse keys");
        if (dbg) std::fprintf(stderr, "[schwarz2] keys %d s %d Nc %d n %zu\n", nkeys, sb, as2.Nc, n);
        std::vector<double> Kcall[2], KPall[2];
        {
            DevBuf<double> dP, dKP, dKc, dK;
            const double one = 1.0, zero = 0.0;
            const int ni = static_cast<int>(n);
            const long long sP = static_cast<long long>(n) * 24;
            for (int kind = 0; kind < 2; ++kind) {
                const int cnt = nkind_keys[kind];
                if (!cnt) continue;
                dK.upload(rom[kind].k_r.data(), n * n, stream);  // row-major K == column-major K^T == K
                dP.upload(Pall[kind].data(), Pall[kind].size(), stream);
                dKP.alloc(Pall[kind].size());
                dKc.alloc(static_cast<size_t>(cnt) * 576);
                if (cublasDgemmStridedBatched(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, ni, 24, ni, &one, dK.ptr, ni, 0, dP.ptr,
                                              ni, sP, &zero, dKP.ptr, ni, sP, cnt) != CUBLAS_STATUS_SUCCESS ||
                    cublasDgemmStridedBatched(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, 24, 24, ni, &one, dP.ptr, ni, sP,
                                              dKP.ptr, ni, sP, &zero, dKc.ptr, 24, 576, cnt) != CUBLAS_STATUS_SUCCESS)
                    throw StatusError(TSV_ECUDA, "schwarz2: coarse Galerkin products failed");
                Kcall[kind].resize(static_cast<size_t>(cnt) * 576);
                d2h(Kcall[kind].data(), dKc.ptr, Kcall[kind].size() * sizeof(double), stream);
                KPall[kind].resize(Pall[kind].size());
                d2h(KPall[kind].data(), dKP.ptr, KPall[kind].size() * sizeof(double), stream);
            }
        }
        tick("coarse products (device)");
        {
            // split loop: K_b P_b per key in the internal panel row order
            // (c nn + rank) x 24, and the panel rows grouped by key in chunks
            const size_t nnl = n / 3;
            std::vector<double> kph(static_cast<size_t>(nkeys) * ldk * 24, 0.0);
            for (int key = 0; key < nkeys; ++key) {
                const double *src = KPall[key_kind[key]].data() + static_cast<size_t>(key_local[key]) * n * 24;
                double *dst = kph.data() + static_cast<size_t>(key) * ldk * 24;
                for (size_t ai = 0; ai < n; ++ai) {
                    const size_t a_ref = 3 * (ai % nnl) + ai / nnl;
                    for (int j = 0; j < 24; ++j) dst[ai * 24 + j] = src[static_cast<size_t>(j) * n + a_ref];
                }
            }
            as2.kp.upload(kph.data(), kph.size(), stream);
            std::vector<std::vector<int>> rows_of(static_cast<size_t>(nkeys));
            for (size_t j = 0; j < B_pad; ++j)
                if (row_cell[j] >= 0) rows_of[static_cast<size_t>(key_of[static_cast<size_t>(row_cell[j])])].push_back(static_cast<int>(j));
            std::vector<int> krows;
            std::vector<int4> items;
            for (int key = 0; key < nkeys; ++key) {
                const auto &v = rows_of[static_cast<size_t>(key)];
                for (size_t i0 = 0; i0 < v.size(); i0 += kKpzcChunk) {
                    const int b0 = static_cast<int>(krows.size() + i0);
                    const int b1 = static_cast<int>(krows.size() + std::min(v.size(), i0 + kKpzcChunk));
                    items.push_back(make_int4(key, b0, b1, 0));
                }
                krows.insert(krows.end(), v.begin(), v.end());
            }
            as2.kp_rows.upload(krows.data(), krows.size(), stream);
            as2.kp_items.upload(items.data(), items.size(), stream);
            as2.kp_nitems = static_cast<int>(items.size());
            as2.Yc.alloc(B_pad * ldk);
            CK(cudaMemsetAsync(as2.Yc.ptr, 0, B_pad * ldk * sizeof(double), stream));
            CK(cudaStreamSynchronize(stream));  // host staging vectors go out of scope
        }
        // per super cell: sum of its blocks' products in block order
        std::vector<double> kcell(static_cast<size_t>(as2.ncells) * 576, 0.0);
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t c = 0; c < cols; ++c) {
                const size_t cell = static_cast<size_t>(r) * cols + c;
                const int cx = static_cast<int>(c) / sb, cy = static_cast<int>(r) / sb;
                const int key = key_of[cell];
                const double *src = Kcall[key_kind[key]].data() + static_cast<size_t>(key_local[key]) * 576;
                double *dst = kcell.data() + (static_cast<size_t>(cy) * as2.SX + cx) * 576;
                for (int e = 0; e < 576; ++e) dst[e] += src[e];
            }
        tick("coarse Galerkin products");
        const size_t Ncs = static_cast<size_t>(as2.Nc);
        // The dense coarse inverse (cuSOLVER potrf + potri on Nc ~ 7e3, whose
        // host-side enqueue alone blocks for ~30 ms) runs on a worker thread
        // on the side stream while this thread builds the local stage. Device
        // buffers are allocated here, on the context stream, before the fork.
        const bool coarse_f64 = getenv_flag("TSV_AS_COARSE_F64"), coarse_dense = getenv_flag("TSV_AS_COARSE_DENSE");
        as2.ainv_c.alloc(Ncs * Ncs);
        CK(cudaMemsetAsync(as2.ainv_c.ptr, 0, Ncs * Ncs * sizeof(double), stream));
        as2.kcell_d.upload(kcell.data(), kcell.size(), stream);
        if (!coarse_f64 && coarse_dense) {
            as2.ldc32 = static_cast<int>(round_up(Ncs, 32));
            as2.ainv_c32.alloc(Ncs * as2.ldc32);
        } else {
            as2.ainv_c32.release();
        }
        long long sym_total = 0;
        if (!coarse_f64 && !coarse_dense) {
            as2.sym_nt = static_cast<int>((Ncs + kSymT - 1) / kSymT);
            sym_total = static_cast<long long>(as2.sym_nt) * (as2.sym_nt + 1) / 2 * kSymT * kSymT;
            as2.sym_tiles.alloc(static_cast<size_t>(sym_total));
            as2.sym_part.alloc(static_cast<size_t>(as2.sym_nt) * as2.sym_nt * kSymT);
            as2.dotpart.alloc(static_cast<size_t>(as2.sym_nt));
        } else {
            as2.sym_nt = 0;
            as2.sym_tiles.release();
            as2.sym_part.release();
        }
        if (!solver2.sol && (cusolverDnCreate(&solver2.sol) != CUSOLVER_STATUS_SUCCESS ||
                             cublasCreate(&solver2.blas) != CUBLAS_STATUS_SUCCESS))
            throw StatusError(TSV_ECUDA, "schwarz2: cuSOLVER/cuBLAS init failed");
        cusolverDnSetStream(solver2.sol, side);
        {
            int lw1 = 0, lw2 = 0;
            if (cusolverDnDpotrf_bufferSize(solver2.sol, CUBLAS_FILL_MODE_LOWER, as2.Nc, as2.ainv_c.ptr, as2.Nc, &lw1) !=
                    CUSOLVER_STATUS_SUCCESS ||
                cusolverDnDpotri_bufferSize(solver2.sol, CUBLAS_FILL_MODE_LOWER, as2.Nc, as2.ainv_c.ptr, as2.Nc, &lw2) !=
                    CUSOLVER_STATUS_SUCCESS)
                throw StatusError(TSV_ECUDA, "schwarz2: cuSOLVER buffer query failed");
            as2.cwork.alloc(static_cast<size_t>(std::max(std::max(lw1, lw2), 1)));
        }
        CK(cudaEventRecord(ev_fork, stream));
        CK(cudaStreamWaitEvent(side, ev_fork, 0));
        std::exception_ptr coarse_err;
        std::thread coarse_worker([&, Ncs, sym_total] {
            try {
                cudaSetDevice(device);
                const cudaStream_t cs = side;
                for (int py = 0; py < 2; ++py)
                    for (int px = 0; px < 2; ++px) {
                        const long long cnt = static_cast<long long>((as2.SX - px + 1) / 2) * ((as2.SY - py + 1) / 2) * 576;
                        if (cnt <= 0) continue;
                        as_coarse_scatter_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, cs>>>(
                            as2.kcell_d.ptr, as2.SX, as2.SY, px, py, as2.ainv_c.ptr, as2.Nc);
                    }
                as_fix_zero_rows_kernel<<<static_cast<unsigned>((Ncs + 7) / 8), 256, 0, cs>>>(as2.ainv_c.ptr, as2.Nc);
                spd_inverse_inplace(solver2, as2.ainv_c.ptr, as2.Nc, as2.cwork, cinfo.ptr);
                as_symmetrize_kernel<<<static_cast<unsigned>((Ncs * Ncs + 255) / 256), 256, 0, cs>>>(as2.ainv_c.ptr,
                                                                                                   as2.Nc);
                if (as2.ainv_c32.ptr) {
                    const size_t tot = Ncs * as2.ldc32;
                    as_coarse_to_f32_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, cs>>>(
                        as2.ainv_c.ptr, as2.Nc, as2.ldc32, as2.ainv_c32.ptr);
                }
                if (as2.sym_nt)
                    as_pack_sym_tiles_kernel<<<static_cast<unsigned>((sym_total + 255) / 256), 256, 0, cs>>>(
                        as2.ainv_c.ptr, as2.Nc, as2.sym_tiles.ptr, sym_total);
                CK(cudaGetLastError());
            } catch (...) {
                coarse_err = std::current_exception();
            }
        });
        struct Joiner {
            std::thread &t;
            ~Joiner() {
                if (t.joinable()) t.join();
            }
        } joiner{coarse_worker};
        tick("coarse inverse (enqueued)");
        // --- 2. neighbourhood types: own kind, the 4 edge neighbours' kinds
        // (or absence), corner neighbours' presence, constrained pattern.
        // Blocks of one type share the representative's local matrix
        // (exact except for corner-neighbour kinds; TSV_AS_EXACT_TYPES=1
        // makes corner kinds part of the type too).
        tick("handles");
        const bool exact_types = getenv_flag("TSV_AS_EXACT_TYPES");
        std::map<std::vector<int>, int> sig_type;
        std::vector<int> type_of(B), rep_of;
        std::vector<std::vector<int>> sigs(B);
        parallel_rows(rows, [&](uint32_t r) {
            for (uint32_t c = 0; c < cols; ++c) {
                const size_t cell = static_cast<size_t>(r) * cols + c;
                std::vector<int> &sig = sigs[cell];
                sig.push_back(layout.kind_at(cell));
                for (int dr = -1; dr <= 1; ++dr)
                    for (int dc = -1; dc <= 1; ++dc) {
                        if (!dr && !dc) continue;
                        const long rr = static_cast<long>(r) + dr, cc = static_cast<long>(c) + dc;
                        const bool in = rr >= 0 && cc >= 0 && rr < rows && cc < cols;
                        const int kd = in ? layout.kind_at(static_cast<size_t>(rr) * cols + static_cast<size_t>(cc)) : -1;
                        sig.push_back((dr && dc && !exact_types) ? (in ? 0 : -1) : kd);
                    }
                const uint32_t *dm = dofmap.data() + cell * n;
                for (size_t a = 0; a < n; ++a)
                    if (constrained[dm[a]]) sig.push_back(1000 + static_cast<int>(a));
            }
        });
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t c = 0; c < cols; ++c) {
                const size_t cell = static_cast<size_t>(r) * cols + c;
                const std::vector<int> &sig = sigs[cell];
                auto it = sig_type.find(sig);
                if (it == sig_type.end()) {
                    it = sig_type.emplace(sig, static_cast<int>(rep_of.size())).first;
                    rep_of.push_back(static_cast<int>(cell));
                }
                type_of[cell] = it->second;
            }
        const int T = static_cast<int>(rep_of.size());
        as2.ntypes = T;
        tick("types");
        // --- 3. local matrices A_b = R_b A R_b^T (lifted), assembled on host
        // threads, inverted in place on the device, packed by a kernel.
        std::vector<double> Aall(static_cast<size_t>(T) * n * n, 0.0);
        {
            const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), static_cast<unsigned>(T)));
            std::vector<std::thread> pool;
            for (unsigned w = 0; w < nt; ++w)
                pool.emplace_back([&, w] {
                    std::vector<int> idx(n);
                    for (int t = static_cast<int>(w); t < T; t += static_cast<int>(nt)) {
                        double *A = Aall.data() + static_cast<size_t>(t) * n * n;  // column-major
                        const size_t cell = static_cast<size_t>(rep_of[t]);
                        const uint32_t r = static_cast<uint32_t>(cell / cols), c = static_cast<uint32_t>(cell % cols);
                        const uint32_t *dm = dofmap.data() + cell * n;
                        std::unordered_map<uint32_t, int> loc;
                        loc.reserve(2 * n);
                        for (size_t a = 0; a < n; ++a) loc[dm[a]] = static_cast<int>(a);
                        for (int dr = -1; dr <= 1; ++dr)
                            for (int dc = -1; dc <= 1; ++dc) {
                                const long rr = static_cast<long>(r) + dr, cc = static_cast<long>(c) + dc;
                                if (rr < 0 || cc < 0 || rr >= rows || cc >= cols) continue;
                                const size_t b2 = static_cast<size_t>(rr) * cols + static_cast<size_t>(cc);
                                const uint32_t *dm2 = dofmap.data() + b2 * n;
                                const std::vector<double> &K2 = rom[layout.kind_at(b2)].k_r;
                                for (size_t a = 0; a < n; ++a) {
                                    auto f = loc.find(dm2[a]);
                                    idx[a] = f == loc.end() ? -1 : f->second;
                                }
                                for (size_t a = 0; a < n; ++a) {
                                    if (idx[a] < 0) continue;
                                    for (size_t q2 = 0; q2 < n; ++q2)
                                        if (idx[q2] >= 0) A[static_cast<size_t>(idx[q2]) * n + idx[a]] += K2[a * n + q2];
                                }
                            }
                        for (size_t a = 0; a < n; ++a)
                            if (constrained[dm[a]]) {
                                for (size_t k = 0; k < n; ++k) A[a * n + k] = A[k * n + a] = 0.0;
                                A[a * n + a] = 1.0;
                            }
                    }
                });
            for (auto &th : pool) th.join();
        }
        tick("local assembly (host)");
        as2.tc = !getenv_flag("TSV_AS_LOCAL_F64") && as_round_bits() == 0 && !small_pcg_candidate();
        const size_t rowsK = round_up(n, kBN);
        if (as2.tc) {
            as2.KP = static_cast<int>(round_up(n, kTcBK));
            as2.ntn = static_cast<int>((n + 255) / 256);
            as2.BN = static_cast<int>(round_up((n + as2.ntn - 1) / as2.ntn, 16));
            as2.NP = as2.ntn * as2.BN;
            as2.LD = std::max(as2.KP, as2.NP);
            as2.ainv32.alloc(static_cast<size_t>(T) * as2.NP * as2.KP);
            CK(cudaMemsetAsync(as2.ainv32.ptr, 0, as2.ainv32.count * sizeof(float), stream));
            as2.ainv_store.release();
        } else {
            as2.ainv_store.alloc(static_cast<size_t>(T) * rowsK * ldk);
            CK(cudaMemsetAsync(as2.ainv_store.ptr, 0, as2.ainv_store.count * sizeof(double), stream));
            as2.ainv32.release();
        }
        DevBuf<double> dAll;
        DevBuf<int> infos;
        dAll.upload(Aall.data(), Aall.size(), stream);
        infos.alloc(static_cast<size_t>(2 * T + 2));
        CK(cudaMemsetAsync(infos.ptr, 0, infos.count * sizeof(int), stream));
        std::vector<const double *> tab(T);
        for (int t = 0; t < T; ++t) {
            double *dA = dAll.ptr + static_cast<size_t>(t) * n * n;
            spd_inverse_inplace(h, dA, static_cast<int>(n), work, infos.ptr + 2 * t);
            if (as2.tc) {
                as_pack_inverse_tf32_kernel<<<static_cast<unsigned>((n * n + 255) / 256), 256, 0, stream>>>(
                    dA, static_cast<int>(n), static_cast<int>(nn), as2.KP,
                    as2.ainv32.ptr + static_cast<size_t>(t) * as2.NP * as2.KP);
                tab[t] = nullptr;
                continue;
            }
            double *dst = as2.ainv_store.ptr + static_cast<size_t>(t) * rowsK * ldk;
            as_pack_inverse_kernel<<<static_cast<unsigned>((n * n + 255) / 256), 256, 0, stream>>>(
                dA, static_cast<int>(n), static_cast<int>(nn), static_cast<int>(ldk), dst, as_round_bits());
            tab[t] = dst;
        }
        CK(cudaGetLastError());
        as2.ainv_tab.upload(tab.data(), tab.size(), stream);
        tick("local inverses (device)");
        // --- 4. type-ordered panel rows (types padded to the small-GEMM tile height)
        const size_t BML = as2.tc ? static_cast<size_t>(kTcBM) : K1SmallCfg::BM;
        const size_t lstride = as2.tc ? static_cast<size_t>(as2.LD) : ldk;
        std::vector<int> rowL(B, -1), tiles;
        size_t row = 0;
        {
            std::vector<std::vector<int>> members(T);
            for (size_t cell = 0; cell < B; ++cell) members[type_of[cell]].push_back(static_cast<int>(cell));
            for (int t = 0; t < T; ++t) {
                const size_t first = row;
                for (int cell : members[t]) rowL[cell] = static_cast<int>(row++);
                row = first + round_up(row - first, BML);
                for (size_t k = first / BML; k < row / BML; ++k) tiles.push_back(t);
            }
        }
        as2.BL_pad = row;
        as2.mtiles = row / BML;
        if (as2.BL_pad * ldk >= 0x7fffffffULL) throw StatusError(TSV_EINVAL, "schwarz2: panel too large");
        as2.tile_type.upload(tiles.data(), tiles.size(), stream);
        {
            std::vector<int2> pr;
            for (size_t i = 0; i < tiles.size();) {
                if (i + 1 < tiles.size() && tiles[i + 1] == tiles[i]) {
                    pr.push_back(make_int2(static_cast<int>(i), static_cast<int>(i + 1)));
                    i += 2;
                } else {
                    pr.push_back(make_int2(static_cast<int>(i), -1));
                    i += 1;
                }
            }
            const bool use_pairs = as2.tc && as2.BN <= 256 && !getenv_flag("TSV_TC_SINGLE") &&
                                   tc_pair_smem_bytes(as2.BN) <= 227 * 1024;
            as2.npairs = use_pairs ? static_cast<int>(pr.size()) : 0;
            if (use_pairs) as2.tc_pairs.upload(pr.data(), pr.size(), stream);
        }
        std::vector<int> s2(nodes * 4, -1);
        for (size_t cell = 0; cell < B; ++cell) {
            const uint32_t *dm = dofmap.data() + cell * n;
            for (size_t rank = 0; rank < nn; ++rank) {
                const size_t in = node_int_of_glob[dm[3 * rank] / 3];
                int *sl = s2.data() + in * 4;
                int k = 0;
                while (sl[k] >= 0) ++k;
                sl[k] = static_cast<int>(static_cast<size_t>(rowL[cell]) * lstride + rank);
            }
        }
        as2.slots2.upload(s2.data(), s2.size(), stream);
        if (as2.tc) {
            if (as2.BL_pad * as2.LD >= 0x7fffffffULL) throw StatusError(TSV_EINVAL, "schwarz2: panel too large");
            as2.XL32.alloc(as2.BL_pad * as2.LD);
            CK(cudaMemsetAsync(as2.XL32.ptr, 0, as2.XL32.count * sizeof(float), stream));
            as2.ZL32.alloc(as2.BL_pad * as2.LD);
            as2.XL.release();
            as2.ZL.release();
            encode_tc_maps(T);
        } else {
            as2.XL.alloc(as2.BL_pad * ldk);
            as2.ZL.alloc(as2.BL_pad * ldk);
            CK(cudaMemsetAsync(as2.XL.ptr, 0, as2.XL.count * sizeof(double), stream));
            as2.XL32.release();
            as2.ZL32.release();
        }
        as2.z.alloc(N);
        tick("panel tables");
        coarse_worker.join();
        if (coarse_err) std::rethrow_exception(coarse_err);
        CK(cudaEventRecord(ev_join, side));
        CK(cudaStreamWaitEvent(stream, ev_join, 0));
        tick("coarse inverse joined");
        {
            std::vector<int> hinfo(infos.count), hc(2);
            d2h(hinfo.data(), infos.ptr, hinfo.size() * sizeof(int), stream);
            d2h(hc.data(), cinfo.ptr, hc.size() * sizeof(int), stream);
            hinfo.insert(hinfo.end(), hc.begin(), hc.end());
            for (int v : hinfo)
                if (v != 0) throw StatusError(TSV_EINVAL, "schwarz2: local/coarse matrix not positive definite");
        }
        tick("done");
        as2.setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }

    GemmParams local_gemm_params() {
        GemmParams gp{};
        gp.A = as2.XL.ptr;
        gp.lda = static_cast<long long>(ldk);
        gp.Bt_tab = as2.ainv_tab.ptr;
        gp.tile_type = as2.tile_type.ptr;
        gp.ldb = static_cast<long long>(ldk);
        gp.C = as2.ZL.ptr;
        gp.ldc = static_cast<long long>(ldk);
        gp.m_tiles = static_cast<int>(as2.mtiles);
        gp.n_tiles = static_cast<int>(round_up(n, K1SmallCfg::BN) / K1SmallCfg::BN);
        gp.k_chunks = static_cast<int>(ldk / K1SmallCfg::KC);
        gp.n_valid = gp.n_store = static_cast<int>(n);
        gp.done = &state.ptr->done;
        gp.tile_counter = tile_counter.ptr;
        return gp;
    }

    // TMA descriptors of the tensor-core local solve: A = XL32 [rows][KP],
    // B = Ainv32 [T * NP][KP], fp32, 32 x {128 | BN} boxes, 128-byte swizzle.
    void encode_tc_maps(int T) {
        using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                      const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        static EncodeFn encode = [] {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q{};
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                fn = nullptr;
            return reinterpret_cast<EncodeFn>(fn);
        }();
        if (!encode) throw StatusError(TSV_ECUDA, "schwarz2: cuTensorMapEncodeTiled unavailable");
        auto make = [&](CUtensorMap *m, void *ptr, uint64_t rows_, uint32_t box_rows, int row_stride) {
            const cuuint64_t dims[2] = {static_cast<cuuint64_t>(as2.KP), rows_};
            const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride) * sizeof(float)};
            const cuuint32_t box[2] = {static_cast<cuuint32_t>(kTcBK), box_rows};
            const cuuint32_t estr[2] = {1, 1};
            if (encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                throw StatusError(TSV_ECUDA, "schwarz2: tensor map encoding failed");
        };
        make(&as2.tmA, as2.XL32.ptr, as2.BL_pad, static_cast<uint32_t>(kTcBM), as2.LD);
        make(&as2.tmB, as2.ainv32.ptr, static_cast<uint64_t>(T) * as2.NP, static_cast<uint32_t>(as2.BN), as2.KP);
        // per-device function attributes: set on this context's device every
        // build (a process-wide flag would skip a second device)
        CK(cudaFuncSetAttribute(tc_local_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes(256)));
        CK(cudaFuncSetAttribute(tc_local_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                tc_pair_smem_bytes(256)));
    }

    void launch_tc_local() {
        TcLocalParams tp{};
        tp.tile_type = as2.tile_type.ptr;
        tp.NP = as2.NP;
        tp.BN = as2.BN;
        tp.k_blocks = as2.KP / kTcBK;
        tp.ZL = as2.ZL32.ptr;
        tp.ldz = static_cast<long long>(as2.LD);
        tp.done = &state.ptr->done;
        if (as2.npairs) {
            launch_pdl(tc_local_pair_kernel, dim3(static_cast<unsigned>(as2.ntn), static_cast<unsigned>(as2.npairs)),
                       kTcThreads, tc_pair_smem_bytes(as2.BN), stream, as2.tmA, as2.tmB, tp,
                       static_cast<const int2 *>(as2.tc_pairs.ptr));
        } else {
            launch_pdl(tc_local_tf32_kernel, dim3(static_cast<unsigned>(as2.ntn), static_cast<unsigned>(as2.mtiles)),
                       kTcThreads, tc_smem_bytes(as2.BN), stream, as2.tmA, as2.tmB, tp);
        }
    }

    size_t nn_count() const { return n / 3; }

    static int as_round_bits() { return getenv("TSV_AS_ROUND_BITS") ? std::atoi(getenv("TSV_AS_ROUND_BITS")) : 0; }

    AsParams as_params() {
        AsParams a{};
        a.slots2 = as2.slots2.ptr;
        a.XL = as2.XL.ptr;
        a.ZL = as2.ZL.ptr;
        a.z = as2.z.ptr;
        a.lat = as2.lat.ptr;
        a.step = as2.step;
        a.step_y = as2.step_y;
        a.Yc = as2.Yc.ptr;
        a.SX = as2.SX;
        a.SY = as2.SY;
        a.lat_x = static_cast<int>(index.lat_x);
        a.lat_y = static_cast<int>(index.lat_y);
        a.qm1 = static_cast<int>(nl.n_z - 1);
        a.cell_ptr = as2.cell_ptr.ptr;
        a.node_cell = as2.node_cell.ptr;
        a.celltab = as2.celltab.ptr;
        a.ncells = as2.ncells;
        a.cellpart = as2.cellpart.ptr;
        a.rc = as2.rc.ptr;
        a.dotpart = as2.dotpart.ptr;
        a.zc = as2.zc.ptr;
        a.ainv_c = as2.ainv_c.ptr;
        a.ainv_c32 = as2.ainv_c32.ptr;
        a.ldc32 = as2.ldc32;
        a.Nc = as2.Nc;
        a.round_bits = as_round_bits();
        if (as2.tc) {
            a.XL32 = as2.XL32.ptr;
            a.ZL32 = as2.ZL32.ptr;
        }
        return a;
    }

    // r update + two-level Schwarz z = M r (U', local GEMM, restriction,
    // coarse solve, prolongation + r.z).
    // Early coarse chain (default; TSV_AS_EARLY_COARSE=0 forks after the
    // update instead): the restriction of the new residual is formed as
    // P^T r' = P^T r - alpha P^T (A p), so the coarse chain forks right after
    // the gather (alpha known) and runs beside the update as well as the
    // local solves. Restarts and the initial residual restrict r itself.
    static bool early_coarse() {
        const char *v = getenv("TSV_AS_EARLY_COARSE");
        return !(v && *v == '0');
    }

    void launch_coarse_chain(const CgParams &q, const AsParams &a, cudaStream_t cs = nullptr) {
        if (!cs) cs = side;
        if (getenv_flag("TSV_AS_RESTRICT_CTA"))
            launch_pdl(as_restrict_kernel, as2.ncells * kAsSplit, 3 * kRestrictGroup, 0, cs, q, a);
        else
            launch_pdl(as_restrict_warp_kernel, (as2.ncells + kRestrictWarps - 1) / kRestrictWarps, 32 * kRestrictWarps, 0,
                       cs, q, a);
        launch_pdl(as_coarse_rhs_kernel, (as2.Nc + 255) / 256, 256, 0, cs, q, a);
        if (as2.sym_nt) {
            const int ntiles = as2.sym_nt * (as2.sym_nt + 1) / 2;
            // one 64 x 64 tile per CTA (a fixed grid walking tiles with a
            // register prefetch of the next tile measured slower: 0.655 vs
            // 0.620 ms per iteration at config 3)
            launch_pdl(as_coarse_symv_kernel, ntiles, 128, 0, cs, q, a, static_cast<const float *>(as2.sym_tiles.ptr),
                       as2.sym_nt, as2.sym_part.ptr);
            launch_pdl(as_coarse_symv_reduce_kernel, as2.sym_nt, kSymRedG * kSymT, 0, cs, q, a, as2.sym_nt,
                       static_cast<const double *>(as2.sym_part.ptr));
        } else {
            as_coarse_gemv_kernel<<<(as2.Nc + kGemvRows - 1) / kGemvRows, 256, 0, cs>>>(q, a);
            as_coarse_dot_kernel<<<1, 1024, 0, cs>>>(q, a);
        }
    }

    void launch_local_solve() {
        if (as2.tc) {
            launch_tc_local();
        } else {
            GemmParams gp = local_gemm_params();
            gemm_nt_f64<K1SmallCfg><<<std::min(k1s_grid, gp.m_tiles * gp.n_tiles), K1SmallCfg::THREADS, K1SmallCfg::SMEM,
                                      stream>>>(gp);
        }
    }

    void launch_as_update_precond(const CgParams &q, bool with_gather) {
        AsParams a = as_params();
        if (with_gather && !fused_gu() && early_coarse()) {
            // gather -> fork {coarse chain on P^T r - alpha P^T Ap} || {update
            // -> local solves -> z_l} -> join
            launch_pdl(cg_gather_kernel, wave_grid(cg_gather_kernel), kVecThreads, 0, stream, q);
            AsParams ae = a;
            ae.rc_recur = 1;
            if (getenv_flag("TSV_AS_SERIAL")) {
                // experiment: the coarse chain in line on the context stream (no fork / join)
                launch_coarse_chain(q, ae, stream);
                launch_pdl(as_update_kernel, wave_grid(as_update_kernel), kVecThreads, 0, stream, q, a);
                launch_local_solve();
                launch_pdl(as_zl_kernel, wave_grid(as_zl_kernel), kVecThreads, 0, stream, q, a);
                launches += 7;
                return;
            }
            CK(cudaEventRecord(ev_fork, stream));
            CK(cudaStreamWaitEvent(side, ev_fork, 0));
            launch_coarse_chain(q, ae);
            CK(cudaEventRecord(ev_join, side));
            launch_pdl(as_update_kernel, wave_grid(as_update_kernel), kVecThreads, 0, stream, q, a);
            launch_local_solve();
            launch_pdl(as_zl_kernel, wave_grid(as_zl_kernel), kVecThreads, 0, stream, q, a);
            CK(cudaStreamWaitEvent(stream, ev_join, 0));
            launches += 7;
            return;
        }
        // r update (grid-stride). Fusing the coarse restriction in (warp-level
        // per-cell partials) measured slower at config 3: 80 us vs 47 + 34 us
        // with the restriction off the critical path on the side stream.
        if (!with_gather) {
            launch_pdl(as_update_kernel, wave_grid(as_update_kernel), kVecThreads, 0, stream, q, a);
        } else if (fused_gu()) {
            launch_pdl(as_gather_update_kernel, gu_grid(), kVecThreads, 0, stream, q, a);
        } else {
            launch_pdl(cg_gather_kernel, wave_grid(cg_gather_kernel), kVecThreads, 0, stream, q);
            launch_pdl(as_update_kernel, wave_grid(as_update_kernel), kVecThreads, 0, stream, q, a);
        }
        // fork: the coarse chain (cell sums of the restriction -> coarse rhs
        // -> coarse solve, HBM and latency bound) runs on a side stream beside
        // the local solves (tensor cores); both join before z. Captured as a
        // forked graph.
        CK(cudaEventRecord(ev_fork, stream));
        CK(cudaStreamWaitEvent(side, ev_fork, 0));
        launch_coarse_chain(q, a);
        CK(cudaEventRecord(ev_join, side));
        launch_local_solve();
        // the local part of z (and r.z_l) while the coarse chain finishes
        launch_pdl(as_zl_kernel, wave_grid(as_zl_kernel), kVecThreads, 0, stream, q, a);
        CK(cudaStreamWaitEvent(stream, ev_join, 0));
        launches += 7;
    }

    // C: p update + next operand panel (Schwarz: adds the coarse part of z).
    void launch_scatter_p(const CgParams &q, int write_z = 0) {
        if (pre_kind == TSV_PRECOND_SCHWARZ2) {
            AsParams a = as_params();
            // node-parallel (a warp-per-coarse-cell variant that loads the
            // cell's 24 coarse values once measured slower: 68.8 vs 54 us at
            // config 3, too few threads in flight for an HBM-bound pass)
            launch_pdl(as_scatter_kernel, wave_grid(as_scatter_kernel), kVecThreads, 0, stream, q, a, write_z);
        } else {
            launch_pdl(cg_scatter_kernel, cg_grid(), kVecThreads, 0, stream, q);
        }
        ++launches;
    }

    // ------------------------------------------------------------ kernels
    unsigned vec_grid() const { return static_cast<unsigned>(std::max<size_t>(1, (nodes + kVecThreads - 1) / kVecThreads)); }
    // CG vector kernels: fixed grid (grid-stride), so the per-CTA partials
    // and their fixed-order sum stay small and deterministic.
    unsigned cg_grid() const { return std::min<unsigned>(vec_grid(), static_cast<unsigned>(sm_count) * 8u); }
    // One resident wave of a grid-stride vector kernel: its occupancy x SMs (capped by cg_grid()). With the
    // three components' loads hoisted the kernels use 40-74 registers, so 8 CTAs per SM no longer fit and the
    // fixed grid of 8 per SM ran 1.3-2.7 waves with a partly filled last one. TSV_VEC_WAVE=0: the old grid.
    template <class K>
    unsigned wave_grid(K kern) {
        static const bool off = [] { const char *e = std::getenv("TSV_VEC_WAVE"); return e && *e == '0'; }();
        if (off) return cg_grid();
        const void *key = reinterpret_cast<const void *>(kern);
        for (const auto &kv : wave_cache)
            if (kv.first == key) return std::min(kv.second, cg_grid());
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kVecThreads, 0));
        const unsigned g = static_cast<unsigned>(std::max(1, occ) * sm_count);
        wave_cache.emplace_back(key, g);
        return std::min(g, cg_grid());
    }
    std::vector<std::pair<const void *, unsigned>> wave_cache;

    void launch_scatter(const double *v, int mode) {
        scatter_vec_kernel<<<vec_grid(), kVecThreads, 0, stream>>>(static_cast<int>(nodes), static_cast<int>(n / 3), slots.ptr, cmask.ptr, v,
                                                                    X.ptr, mode);
        ++launches;
        CK(cudaGetLastError());
    }

    GemmParams k1_params(const int *done) {
        GemmParams gp{};
        gp.A = X.ptr;
        gp.lda = static_cast<long long>(ldk);
        gp.Bt[0] = rom[0].set ? rom[0].d_k.ptr : rom[1].d_k.ptr;
        gp.Bt[1] = rom[1].set ? rom[1].d_k.ptr : rom[0].d_k.ptr;
        gp.ldb = static_cast<long long>(ldk);
        gp.tile_kind = tile_kind_d.ptr;
        gp.C = Y.ptr;
        gp.ldc = static_cast<long long>(ldk);
        gp.m_tiles = static_cast<int>(m_tiles);
        gp.n_tiles = static_cast<int>(round_up(n, kBN) / kBN);
        gp.k_chunks = static_cast<int>(ldk / kKC);
        gp.n_valid = static_cast<int>(n);
        gp.n_store = static_cast<int>(n);
        gp.row_scale = nullptr;
        gp.done = done;
        gp.tile_counter = tile_counter.ptr;
        return gp;
    }

    // ------------------------------------------------ int8 (Ozaki) K1
    // K1 variants. Default: FP64 DMMA for every product. Opt-in: the A x of the
    // true-residual check on the int8 tensor cores with 10 Ozaki digits (exact
    // int32 accumulation: a more accurate residual; in round 1, with the s = 3
    // coarse space, 72 iterations / 1 restart instead of 84 / 5 at config 3).
    //   TSV_K1_VERIFY=0|9|10  hybrid off / digits (any preconditioner)
    //   TSV_K1_OZAKI=9|10     every K1 on the int8 tensor cores
    int oz_verify_digits() const {
        if (const char *v = getenv("TSV_K1_VERIFY")) {
            const int s = std::atoi(v);
            return (s == 9 || s == 10) ? s : 0;
        }
        // With the irrep K1 (mirror-symmetric ROMs) the A x of the check runs on the
        // exact int8 path: the irrep products round differently from the plain
        // DMMA product, and at config 3 the FP64 rounding of A x on the smooth
        // solution is already ~tol |b| (sym vs plain: 1.1e-12 |b|), so an FP64
        // check on that path never passes (B200: 84 restarts in 400 iterations).
        if (sym.k1 && sym.fused && ldk <= 1024 && !k1_small) return 10;  // small arrays: the FP64 DMMA check passes there
        // Default off since round 2: with the s = 2 coarse space the FP64 DMMA
        // check restarts no more often than the exact int8 one (config 3: 57
        // iterations / 1 restart either way; configs 0-4 unchanged), and the two
        // early-exit int8 launches per iteration cost 3-8% (B200: config 3
        // 195.7 k vs 190.0 k blocks/s, config 1 38.3 k vs 35.6 k).
        return 0;
    }

    int oz_digits_env() const {
        if (const int v = oz_verify_digits()) return v;
        const char *v = getenv("TSV_K1_OZAKI");
        if (!v) return 0;
        const int s = std::atoi(v);
        return (s == 9 || s == 10) ? s : 0;
    }

    template <int S>
    void oz_prepare() {
        constexpr int BN = OzCfg<S>::BN;
        const int KA = static_cast<int>(ldk);
        oz_brows = static_cast<long long>(round_up(n, BN));
        for (int k = 0; k < 2; ++k) {
            RomHost &m = rom[k];
            if (!m.set || m.oz_s == S) continue;
            m.oz_b.alloc(static_cast<size_t>(S) * oz_brows * KA);
            m.oz_eb.alloc(static_cast<size_t>(oz_brows));
            CK(cudaMemsetAsync(m.oz_b.ptr, 0, m.oz_b.count, stream));
            CK(cudaMemsetAsync(m.oz_eb.ptr, 0, m.oz_eb.count * sizeof(int), stream));
            oz_slice_kernel<S><<<static_cast<unsigned>((n + 7) / 8), 256, 0, stream>>>(
                m.d_k.ptr, static_cast<long long>(ldk), static_cast<int>(n), static_cast<int>(ldk), m.oz_b.ptr, oz_brows, KA,
                m.oz_eb.ptr, nullptr, nullptr);
            CK(cudaGetLastError());
            m.oz_s = S;
        }
        oz_a.alloc(static_cast<size_t>(S) * B_pad * KA);
        oz_ea.alloc(B_pad);
        using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                      const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            throw StatusError(TSV_ECUDA, "ozaki: cuTensorMapEncodeTiled unavailable");
        EncodeFn encode = reinterpret_cast<EncodeFn>(fn);
        auto make = [&](CUtensorMap *map, void *ptr, uint64_t rows_, uint32_t box_rows) {
            const cuuint64_t dims[2] = {static_cast<cuuint64_t>(KA), rows_};
            const cuuint64_t strides[1] = {static_cast<cuuint64_t>(KA)};
            const cuuint32_t box[2] = {static_cast<cuuint32_t>(kOzBK), box_rows};
            const cuuint32_t estr[2] = {1, 1};
            if (encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                throw StatusError(TSV_ECUDA, "ozaki: tensor map encoding failed");
        };
        make(&oz_tmA, oz_a.ptr, static_cast<uint64_t>(S) * B_pad, static_cast<uint32_t>(kTcBM));
        for (int k = 0; k < 2; ++k) {
            const RomHost &m = rom[k].set ? rom[k] : rom[1 - k];
            make(&oz_tmB[k], m.oz_b.ptr, static_cast<uint64_t>(S) * oz_brows, static_cast<uint32_t>(BN));
        }
        CK(cudaFuncSetAttribute(oz_gemm_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, oz_smem_bytes<S>()));
        oz_s = S;
    }

    void oz_ensure() {
        const int S = ldk <= 1024 ? oz_digits_env() : 0;  // the digit split keeps a row in registers
        if (S == oz_s && (S == 0 || oz_a.ptr)) return;
        if (S == 0) {
            oz_s = 0;
            return;
        }
        if (S == 10) oz_prepare<10>();
        else oz_prepare<9>();
    }

    template <int S>
    void launch_k1_oz(const int *done, const int *run_flag = nullptr) {
        constexpr int BN = OzCfg<S>::BN;
        const int KA = static_cast<int>(ldk);
        // with a run flag (the true-residual check) the launch is usually an
        // early exit: one CTA per SM keeps that cheap
        const size_t slice_ctas = static_cast<size_t>(sm_count) * (run_flag ? 1 : 8);
        launch_pdl(oz_slice_kernel<S>, static_cast<unsigned>(std::min<size_t>((B_pad + 7) / 8, slice_ctas)),
                   256, 0, stream, static_cast<const double *>(X.ptr), static_cast<long long>(ldk), static_cast<int>(B_pad),
                   static_cast<int>(ldk), oz_a.ptr, static_cast<long long>(B_pad), KA, oz_ea.ptr, done, run_flag);
        OzParams op{};
        op.tile_kind = tile_kind_d.ptr;
        op.a_plane_rows = static_cast<long long>(B_pad);
        op.b_plane_rows = oz_brows;
        op.k_blocks = (KA + kOzBK - 1) / kOzBK;
        op.ex_a = oz_ea.ptr;
        op.ex_b[0] = (rom[0].set ? rom[0] : rom[1]).oz_eb.ptr;
        op.ex_b[1] = (rom[1].set ? rom[1] : rom[0]).oz_eb.ptr;
        op.C = Y.ptr;
        op.ldc = static_cast<long long>(ldk);
        op.n_store = static_cast<int>(n);
        op.done = done;
        op.run_flag = run_flag;
        op.m_tiles = static_cast<int>(m_tiles);
        op.n_tiles = static_cast<int>(oz_brows / BN);
        const int tiles = op.m_tiles * op.n_tiles;
        launch_pdl(oz_gemm_kernel<S>, static_cast<unsigned>(std::min(tiles, sm_count)), kTcThreads,
                   static_cast<size_t>(oz_smem_bytes<S>()), stream, oz_tmA, oz_tmB[0], oz_tmB[1], op);
        launches += 2;
        CK(cudaGetLastError());
    }

    // Forward / backward Walsh-Hadamard pass over a whole operand panel.
    void launch_sym_panel(int dir, const double *in, double *out, bool with32, const int *done) {
        const RomHost &mt = rom[sym.tab_kind];
        SymPanelParams sp{};
        sp.in = in;
        sp.out = out;
        sp.ld_in = static_cast<long long>(dir == 0 ? ldk : static_cast<size_t>(sym.lds));
        sp.ld_out = static_cast<long long>(dir == 0 ? static_cast<size_t>(sym.lds) : ldk);
        sp.rows = static_cast<int>(B_pad);
        sp.n_plain = static_cast<int>(ldk);
        sp.n_seg = sym.lds;
        sp.src = mt.d_ssrc.ptr;
        sp.dst = mt.d_sdst.ptr;
        sp.n_orbits = mt.sred.n_orbits;
        sp.n_valid = static_cast<int>(n);
        sp.ld32 = static_cast<long long>(sym.LD);
        sp.done = done;
        if (with32) {
            if (dir == 0) sp.x32 = sym.X32.ptr;
            else sp.c32 = sym.Yc32.ptr;
            sp.c_scale = sym.c_scale;
        }
        const unsigned grid = static_cast<unsigned>(std::min<size_t>((B_pad + kSymWarps - 1) / kSymWarps, static_cast<size_t>(sm_count) * 2));
        if (dir == 0) launch_pdl(sym_panel_kernel<0>, grid, 32 * kSymWarps, sym.panel_smem, stream, sp);
        else launch_pdl(sym_panel_kernel<1>, grid, 32 * kSymWarps, sym.panel_smem, stream, sp);
        ++launches;
    }

    // K1 on mirror-symmetric ROMs: X -> Xs (Walsh-Hadamard over the mirror
    // orbits), 8 irrep GEMMs Ys_r = Xs_r K''_r^T (1/8 of the DMMA FLOPs), the
    // rounding-level defect K_r - K_sym on tcgen05 (TF32), Ys -> Y.
    void launch_k1_sym(const int *done) {
        const RomHost &mt = rom[sym.tab_kind];
        launch_sym_panel(0, X.ptr, sym.Xs.ptr, sym.corr, done);
        GemmSegParams gp{};
        gp.A = sym.Xs.ptr;
        gp.lda = sym.lds;
        gp.Bt[0] = (rom[0].set && rom[0].sym ? rom[0] : rom[1]).d_ks.ptr;
        gp.Bt[1] = (rom[1].set && rom[1].sym ? rom[1] : rom[0]).d_ks.ptr;
        gp.tile_kind = tile_kind_d.ptr;
        gp.C = sym.Ys.ptr;
        gp.ldc = sym.lds;
        gp.m_tiles = static_cast<int>(m_tiles);
        gp.tiles_per_m = mt.k1_tiles_per_m;
        gp.n_segs = static_cast<int>(mt.k1_segs.size());
        gp.segs = mt.d_k1_segs.ptr;
        gp.done = done;
        gp.tile_counter = tile_counter.ptr;
        gp.m_major = 1;
        launch_pdl(gemm_seg_f64<K1Cfg>, std::min(k1_grid, gp.m_tiles * gp.tiles_per_m), K1Cfg::THREADS, K1Cfg::SMEM, stream, gp);
        ++launches;
        if (sym.corr) {
            TcLocalParams tp{};
            tp.tile_type = sym.tile_type.ptr;
            tp.NP = sym.NP;
            tp.BN = sym.BN;
            tp.k_blocks = sym.KP / kTcBK;
            tp.ZL = sym.Yc32.ptr;
            tp.ldz = static_cast<long long>(sym.LD);
            tp.done = done ? done : zero_flag.ptr;
            if (sym.npairs)
                launch_pdl(tc_local_pair_kernel, dim3(static_cast<unsigned>(sym.ntn), static_cast<unsigned>(sym.npairs)),
                           kTcThreads, tc_pair_smem_bytes(sym.BN), stream, sym.tmA, sym.tmB, tp,
                           static_cast<const int2 *>(sym.pairs.ptr));
            else
                launch_pdl(tc_local_tf32_kernel, dim3(static_cast<unsigned>(sym.ntn), static_cast<unsigned>(m_tiles)),
                           kTcThreads, tc_smem_bytes(sym.BN), stream, sym.tmA, sym.tmB, tp);
            ++launches;
        }
        launch_sym_panel(1, sym.Ys.ptr, Y.ptr, sym.corr, done);
        CK(cudaGetLastError());
    }

    // The fused irrep K1 carries this product? On mid-size arrays (k1_small) only for the Schwarz loop and
    // for stand-alone applies: the reference's preconditioners take thousands of iterations there, and
    // the irrep products' larger rounding on smooth vectors costs them accuracy against the reference's
    // own Jacobi solution (config 2: 1.4e-10 instead of 8.8e-13), while Schwarz stays at 3e-12.
    bool k1_irrep(bool in_loop) const {
        return sym.k1 && sym.fused && (!k1_small || !in_loop || pre_kind == TSV_PRECOND_SCHWARZ2);
    }

    void launch_k1(const int *done) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CK(cudaStreamIsCapturing(stream, &cs));
        if (cs == cudaStreamCaptureStatusNone) oz_ensure();
        const int *yx = done ? &state.ptr->y_holds_x : nullptr;
        const bool verify_mode = oz_s && oz_verify_digits();
        const bool hybrid = verify_mode && done;
        if (oz_s && !verify_mode) return oz_s == 9 ? launch_k1_oz<9>(done) : launch_k1_oz<10>(done);
        if (sym.k1 && !sym.fused && !oz_s) return launch_k1_sym(done);
        GemmParams gp = k1_params(done);
        if (k1_irrep(done != nullptr)) {
            // The irrep products carry the iteration; inside the PCG loop the A x of
            // the true-residual check goes to the exact int8 path (hybrid) or, when
            // that is off, to the plain DMMA K1 below (run only when y_holds_x).
            launch_k1_sym_fused(done, yx);
            if (!done) return;
            if (hybrid) {
                if (oz_s == 9) launch_k1_oz<9>(done, yx);
                else launch_k1_oz<10>(done, yx);
                return;
            }
            gp.run_flag = yx;
        }
        if (hybrid) gp.skip_flag = yx;
        if (k1_small) {
            gp.m_tiles = static_cast<int>(B_pad / K1SmallCfg::BM);
            gp.n_tiles = static_cast<int>(round_up(n, K1SmallCfg::BN) / K1SmallCfg::BN);
            gp.k_chunks = static_cast<int>(ldk / K1SmallCfg::KC);
            gp.tile_kind = tile_kind_small_d.ptr;
            const int tiles = gp.m_tiles * gp.n_tiles;
            const int S = k1_split_k(tiles, gp.k_chunks);
            if (S > 1) {
                // split-K: tiles x S CTAs fill the resident slots (one wave)
                SplitK sk{sk1_work.ptr, sk1_ticket.ptr, S};
                launch_pdl(gemm_splitk_f64<K1SmallCfg>, tiles * S, K1SmallCfg::THREADS, K1SmallCfg::SMEM, stream, gp, sk);
            } else {
                // no more CTAs than tiles: idle CTAs would only contend on the tile counter
                const int g = std::min(k1s_grid, tiles);
                launch_pdl(gemm_nt_f64<K1SmallCfg>, g, K1SmallCfg::THREADS, K1SmallCfg::SMEM, stream, gp);
            }
        } else if (k1_streamk) {
            StreamK sk{sk_start.ptr, sk_work.ptr, sk_flag.ptr};
            launch_pdl(gemm_streamk_f64<K1Cfg>, k1_grid, K1Cfg::THREADS, K1Cfg::SMEM, stream, gp, sk);
        } else {
            launch_pdl(gemm_nt_f64<K1Cfg>, std::min(k1_grid, gp.m_tiles * gp.n_tiles), K1Cfg::THREADS, K1Cfg::SMEM,
                       stream, gp);
        }
        ++launches;
        CK(cudaGetLastError());
        if (hybrid) {
            if (oz_s == 9) launch_k1_oz<9>(done, yx);
            else launch_k1_oz<10>(done, yx);
        }
    }

    // Compensated x (x + xlo, TwoSum in the update kernel) for the Schwarz loop; TSV_COMP_X=0: plain x.
    bool comp_x_active() {
        if (pre_kind != TSV_PRECOND_SCHWARZ2 || small_pcg_active()) return false;
        const char *e = std::getenv("TSV_COMP_X");
        if (e && *e == '0') return false;
        if (xlo.count != x.count) {
            xlo.alloc(x.count);
            CK(cudaMemsetAsync(xlo.ptr, 0, xlo.count * sizeof(float), stream));
        }
        return true;
    }
    DevBuf<float> xlo;

    CgParams cg_params() {
        CgParams q{};
        q.st = state.ptr;
        q.n_nodes = static_cast<int>(nodes);
        q.nn = static_cast<int>(n / 3);
        q.slots = slots.ptr;
        q.cmask = cmask.ptr;
        q.b = b.ptr;
        q.x = x.ptr;
        q.r = r.ptr;
        q.p = p.ptr;
        q.ap = ap.ptr;
        q.xlo = comp_x_active() ? xlo.ptr : nullptr;
        q.Y = Y.ptr;
        q.X = X.ptr;
        q.precond = pre_kind;
        q.pre = pre.ptr;
        q.partial = partial.ptr;
        q.zbuf = as2.z.ptr;
        return q;
    }

    void launch_iteration(const CgParams &q) {
        if (pre_kind == TSV_PRECOND_SCHWARZ2 && as_split()) {
            if (fused_gu()) {
                launch_pdl(as_gu_split_kernel, gu_split_grid(), kVecThreads, 0, stream, q, as_params());
            } else {
                launch_pdl(as_g_split_kernel, cg_grid(), kVecThreads, 0, stream, q, as_params());
                launch_pdl(as_update_kernel, cg_grid(), kVecThreads, 0, stream, q, as_params());
                ++launches;
            }
            ++launches;
            launch_split_tail(q);
            return;
        }
        launch_k1(&state.ptr->done);
        if (pre_kind == TSV_PRECOND_SCHWARZ2) {
            launch_as_update_precond(q, true);
        } else {
            launch_pdl(cg_gather_kernel, cg_grid(), kVecThreads, 0, stream, q);
            launch_pdl(cg_update_kernel, cg_grid(), kVecThreads, 0, stream, q);
            ++launches;
        }
        launch_scatter_p(q);
        ++launches;
    }

    int graph_kernels_per_iteration() const {
        const int schwarz = as_split() ? (fused_gu() ? 10 : 11) : (fused_gu() ? 9 : 10);
        const bool oz_verify = oz_s && oz_verify_digits();
        int symk = 0;  // extra launches of the irrep K1
        if (sym.k1 && !(oz_s && !oz_verify)) symk = sym.fused ? (k1_irrep(true) && !oz_verify ? 1 : 0) : (sym.corr ? 3 : 2);
        return (pre_kind == TSV_PRECOND_SCHWARZ2 ? schwarz : 4) + (oz_s ? (oz_verify ? 2 : 1) : 0) + symk;
    }

    // Split Schwarz loop (opt-in, TSV_AS_SPLIT=1): after r is updated, the
    // coarse chain runs on the side stream beside the local solve, z_l and K1
    // (A z_l); A P zc enters through the Yc panel. Correct (same iterations
    // +-6, parity tests) but measured slower on B200 at config 3 (0.583 vs
    // 0.537 ms per iteration at s = 3; 0.680 vs 0.628 at s = 2): K1 holds
    // every SM's register file (2 x 128 x 240 regs), so the side chain only
    // runs between kernels, and every other kernel is HBM-bound like it.
    static bool as_split() { return getenv_flag("TSV_AS_SPLIT"); }
    unsigned gu_split_grid() {
        if (!gu_split_grid_) {
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, as_gu_split_kernel, kVecThreads, 0));
            if (per_sm < 1) throw StatusError(TSV_ECUDA, "as_gu_split_kernel: no resident CTA");
            gu_split_grid_ = static_cast<unsigned>(per_sm * sm_count);
        }
        return std::min<unsigned>(vec_grid(), gu_split_grid_);
    }
    unsigned gu_split_grid_ = 0;

    KpzcParams kpzc_params() const {
        KpzcParams k{};
        k.kp = as2.kp.ptr;
        k.items = as2.kp_items.ptr;
        k.rows = as2.kp_rows.ptr;
        k.row_cell = row_cell_d.ptr;
        k.cols = static_cast<int>(layout.cols);
        k.sb = as2.s;
        k.n = static_cast<int>(n);
        k.ldk = static_cast<long long>(ldk);
        return k;
    }

    // After r is updated (prologue U or GU): fork the coarse chain (+ A P zc)
    // to the side stream; local solve, z_l / X panel and K1 on the main
    // stream; join.
    void launch_split_tail(const CgParams &q) {
        AsParams a = as_params();
        CK(cudaEventRecord(ev_fork, stream));
        CK(cudaStreamWaitEvent(side, ev_fork, 0));
        launch_pdl(as_restrict_kernel, as2.ncells * kAsSplit, 3 * kRestrictGroup, 0, side, q, a);
        launch_pdl(as_coarse_rhs_kernel, (as2.Nc + 255) / 256, 256, 0, side, q, a);
        if (as2.sym_nt) {
            const int ntiles = as2.sym_nt * (as2.sym_nt + 1) / 2;
            launch_pdl(as_coarse_symv_kernel, ntiles, 128, 0, side, q, a, static_cast<const float *>(as2.sym_tiles.ptr),
                       as2.sym_nt, as2.sym_part.ptr);
            launch_pdl(as_coarse_symv_reduce_kernel, as2.sym_nt, kSymRedG * kSymT, 0, side, q, a, as2.sym_nt,
                       static_cast<const double *>(as2.sym_part.ptr));
        } else {
            as_coarse_gemv_kernel<<<(as2.Nc + kGemvRows - 1) / kGemvRows, 256, 0, side>>>(q, a);
            as_coarse_dot_kernel<<<1, 1024, 0, side>>>(q, a);
        }
        launch_pdl(as_kpzc_kernel, dim3(static_cast<unsigned>(as2.kp_nitems), static_cast<unsigned>((n + kKpzcRows - 1) / kKpzcRows)),
                   kKpzcRows, 0, side, q, a, kpzc_params());
        CK(cudaEventRecord(ev_join, side));
        if (as2.tc) {
            launch_tc_local();
        } else {
            GemmParams gp = local_gemm_params();
            gemm_nt_f64<K1SmallCfg><<<std::min(k1s_grid, gp.m_tiles * gp.n_tiles), K1SmallCfg::THREADS, K1SmallCfg::SMEM,
                                      stream>>>(gp);
        }
        launch_pdl(as_zl_split_kernel, cg_grid(), kVecThreads, 0, stream, q, a);
        launches += 7;
        launch_k1(&state.ptr->done);
        CK(cudaStreamWaitEvent(stream, ev_join, 0));
    }

    // Gather + update as one kernel across a software grid barrier (Schwarz
    // path; TSV_NO_FUSED_GU=1 keeps the two kernels).
    // Measured at config 3 (B200): the barrier-fused kernels are slower than
    // the two kernels with PDL between them (92 vs 35 + 50 us serial; 141 us
    // split), so they are opt-in (TSV_FUSED_GU=1).
    static bool fused_gu() { return getenv_flag("TSV_FUSED_GU"); }
    unsigned gu_grid() {
        if (!gu_grid_) {
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, as_gather_update_kernel, kVecThreads, 0));
            if (per_sm < 1) throw StatusError(TSV_ECUDA, "as_gather_update_kernel: no resident CTA");
            gu_grid_ = static_cast<unsigned>(per_sm * sm_count);
        }
        return std::min<unsigned>(vec_grid(), gu_grid_);
    }
    unsigned gu_grid_ = 0;

    void ensure_graph() {
        oz_ensure();
        const float *want_xlo = comp_x_active() ? xlo.ptr : nullptr;
        if (iter_graph && graph_oz_s == oz_s && graph_xlo == want_xlo) return;
        PhaseTimer pt("graph capture");
        drop_graph();
        set_launch_priorities();
        graph_oz_s = oz_s;
        graph_xlo = want_xlo;
        CgParams q = cg_params();
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        const uint64_t before = launches;
        for (int i = 0; i < kItersPerGraph; ++i) launch_iteration(q);
        launches = before;
        CK(cudaStreamEndCapture(stream, &graph));
        CK(cudaGraphInstantiate(&iter_graph, graph, 0));
        cudaGraphDestroy(graph);
    }

    // ------------------------------------------------------------- solve
    int solve(const tsv_iter_options &o, double *u_out, tsv_solve_info *info) {
        if (!layout_set) throw StatusError(TSV_ESTATE, "solve: no layout set");
        if (!(o.tolerance > 0.0)) throw StatusError(TSV_EINVAL, "IterOptions: tolerance must be > 0");
        if (o.max_iterations < 1) throw StatusError(TSV_EINVAL, "IterOptions: max_iterations must be >= 1");
        if (o.precond < 0 || o.precond > 3) throw StatusError(TSV_EINVAL, "IterOptions: unknown preconditioner");
        PhaseTimer pt("solve");
        build_precond(o.precond);
        const uint64_t l0 = launches;
        CK(cudaEventRecord(ev0, stream));
        CgState st = run_cg(o.tolerance, o.max_iterations);
        float loop_ms = 0.f;
        CK(cudaEventRecord(ev1, stream));
        CK(cudaEventSynchronize(ev1));
        CK(cudaEventElapsedTime(&loop_ms, ev0, ev1));
        int status = TSV_OK;
        int best_it = st.it;
        double relres = st.norm_b > 0.0 ? st.res / st.norm_b : 0.0;
        if (st.done == CG_NOCONV) {
            status = TSV_ENOCONV;
            best_it = st.best_it;
            relres = st.best_res / st.norm_b;
            if (st.best_it == 0) {
                // no iterate beat the initial residual: the reference returns
                // best_x = x0 = 0 (linalg.cpp:316-317, 354-355); a replay
                // would still run one update (max_it is checked after it += 1)
                CK(cudaMemsetAsync(x.ptr, 0, x.count * sizeof(double), stream));
            } else if (st.best_it < st.it) {
                // Bitwise-deterministic replay up to the best iterate
                // (the reference keeps a copy of it, linalg.cpp:346-349).
                CgState st2 = run_cg(o.tolerance, st.best_it);
                (void)st2;
            }
        } else if (st.done == CG_BREAKDOWN) {
            CK(cudaEventRecord(ev1, stream));
            CK(cudaEventSynchronize(ev1));
            solution_valid = false;
            throw StatusError(TSV_EBREAKDOWN, st.breakdown_code == 2
                                                  ? "iterative_solve: matrix not positive definite for CG (p'Ap <= 0)"
                                                  : "iterative_solve: NaN/Inf breakdown");
        }
        CK(cudaEventRecord(ev1, stream));
        CK(cudaEventSynchronize(ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev0, ev1));
        last_solve_ms = ms;
        solution_valid = true;
        if (u_out) {
            PhaseTimer pt2("u -> host");
            copy_to_reference(x.ptr, u_out);
        }
        if (info) {
            info->iterations = st.it;
            info->relative_residual = relres;
            info->direct_fallback = 0;
            info->best_iterations = best_it;
            info->solve_ms = ms;
            info->loop_ms = loop_ms;
            info->restarts = st.restarts;
            info->replacements = st.replaced;
            info->kernel_launches = launches - l0;
        }
        if (status == TSV_ENOCONV) {
            char buf[256];
            std::snprintf(buf, sizeof buf,
                          "iterative_solve: CG did not reach tolerance %f in %d iterations (best residual %f)",
                          o.tolerance, st.it, relres);
            err = buf;
        }
        return status;
    }

    // ------------------------------------------- persistent small-array PCG
    // Opt-in (TSV_SMALL_PCG=1, small-tile arrays): the whole Schwarz PCG as
    // one cooperative kernel (small_pcg.cuh) with FP64 local solves. Correct
    // (parity suites pass, same iteration counts) but measured slower than the
    // graph path on B200: config 0 54.5 vs 47.6 us per iteration, config 1
    // 59.3 vs 55.6 (148 CTAs; 296 / 74 / 32 / 16 CTAs slower still): the
    // split-K GEMM items inside the kernel are latency-bound and each of the
    // ~10 grid barriers per iteration costs more than a PDL kernel boundary.
    bool small_pcg_candidate() const {
        const char *v = getenv("TSV_SMALL_PCG");
        return v && *v == '1' && k1_small && coop_launch;
    }
    bool small_pcg_active() const { return pre_kind == TSV_PRECOND_SCHWARZ2 && !as2.tc && small_pcg_candidate(); }
    int coop_launch = 0;
    unsigned small_grid = 0;
    DevBuf<double> small_w1, small_wl, small_gpart;

    CgState run_small_pcg(double tol, int max_it) {
        CgState s{};
        s.done = CG_RUNNING;
        s.phase = PH_INIT;
        s.tol = tol;
        s.max_it = max_it;
        *h_state = s;
        CK(cudaMemcpyAsync(state.ptr, h_state, sizeof(CgState), cudaMemcpyHostToDevice, stream));
        CK(cudaMemsetAsync(X.ptr, 0, X.count * sizeof(double), stream));
        using Cfg = K1SmallCfg;
        auto kern = pcg_small_kernel<Cfg>;
        if (!small_grid) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::SMEM)));
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::THREADS, Cfg::SMEM));
            if (per_sm < 1) throw StatusError(TSV_ECUDA, "pcg_small_kernel: no resident CTA");
            const char *cv = getenv("TSV_SMALL_PCG_CTAS");  // grid barriers: fewer CTAs, cheaper
            const int cap = cv ? std::max(1, std::atoi(cv)) : sm_count;
            small_grid = static_cast<unsigned>(std::min(per_sm * sm_count, cap));
        }
        SmallPcgParams P{};
        P.q = cg_params();
        P.a = as_params();
        P.k1 = k1_params(nullptr);
        P.k1.m_tiles = static_cast<int>(B_pad / Cfg::BM);
        P.k1.n_tiles = static_cast<int>(round_up(n, Cfg::BN) / Cfg::BN);
        P.k1.k_chunks = static_cast<int>(ldk / Cfg::KC);
        P.k1.tile_kind = tile_kind_small_d.ptr;
        P.loc = local_gemm_params();
        P.k1_tiles = P.k1.m_tiles * P.k1.n_tiles;
        P.loc_tiles = P.loc.m_tiles * P.loc.n_tiles;
        auto slices = [&](int tiles, int kc) {
            return std::max(1, std::min(std::min(kc, kSplitKMax), static_cast<int>(small_grid) / std::max(1, tiles)));
        };
        P.sk1.S = slices(P.k1_tiles, P.k1.k_chunks);
        P.skl.S = slices(P.loc_tiles, P.loc.k_chunks);
        constexpr size_t per = static_cast<size_t>(Cfg::FM) * Cfg::FN * 2 * Cfg::THREADS;
        const size_t n1 = static_cast<size_t>(P.k1_tiles) * P.sk1.S * per, nl = static_cast<size_t>(P.loc_tiles) * P.skl.S * per;
        if (small_w1.count < n1) small_w1.alloc(n1);
        if (small_wl.count < nl) small_wl.alloc(nl);
        if (small_gpart.count < 4 * static_cast<size_t>(small_grid)) small_gpart.alloc(4 * static_cast<size_t>(small_grid));
        P.sk1.work = small_w1.ptr;
        P.skl.work = small_wl.ptr;
        P.ainv_c = as2.ainv_c.ptr;
        P.gpart = small_gpart.ptr;
        void *args[] = {&P};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(kern), dim3(small_grid), dim3(Cfg::THREADS), args, Cfg::SMEM,
                                       stream));
        ++launches;
        CK(cudaMemcpyAsync(h_state, state.ptr, sizeof(CgState), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return *h_state;
    }

    CgState run_cg(double tol, int max_it) {
        if (small_pcg_active()) return run_small_pcg(tol, max_it);
        ensure_graph();
        CgState s{};
        s.done = CG_RUNNING;
        s.phase = PH_INIT;
        s.tol = tol;
        s.max_it = max_it;
        if (const char *vm = std::getenv("TSV_VERIFY_MARGIN")) s.verify_margin = std::atof(vm);
        if (pre_kind == TSV_PRECOND_SCHWARZ2 && !as_split() && !fused_gu() && comp_x_active()) {
            s.replace_at = 1e-6;
            if (const char *ra = std::getenv("TSV_REPLACE_AT")) s.replace_at = std::atof(ra);
        }
        *h_state = s;
        CK(cudaMemcpyAsync(state.ptr, h_state, sizeof(CgState), cudaMemcpyHostToDevice, stream));
        CK(cudaMemsetAsync(X.ptr, 0, X.count * sizeof(double), stream));
        CgParams q = cg_params();
        if (pre_kind == TSV_PRECOND_SCHWARZ2 && as_split()) {
            launch_pdl(as_update_kernel, cg_grid(), kVecThreads, 0, stream, q, as_params());
            ++launches;
            launch_split_tail(q);
        } else {
            if (pre_kind == TSV_PRECOND_SCHWARZ2) {
                launch_as_update_precond(q, false);
            } else {
                cg_update_kernel<<<cg_grid(), kVecThreads, 0, stream>>>(q);
                ++launches;
            }
            launch_scatter_p(q);
        }
        CK(cudaGetLastError());
        // Host-polled batches of graph-captured iterations; a finished
        // solve turns the remaining launches into early exits.
        const int graph_nodes = graph_kernels_per_iteration() * kItersPerGraph;
        for (;;) {
            CK(cudaGraphLaunch(iter_graph, stream));
            launches += graph_nodes;
            CK(cudaMemcpyAsync(h_state, state.ptr, sizeof(CgState), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            if (h_state->done != CG_RUNNING) break;
        }
        if (q.xlo) {
            fold_x_kernel<<<static_cast<unsigned>(sm_count) * 4, 256, 0, stream>>>(x.ptr, xlo.ptr, static_cast<long long>(x.count));
            ++launches;
            CK(cudaGetLastError());
        }
        return *h_state;
    }

    // ----------------------------------------------------------- recovery
    void check_recovery(int points) {
        if (!layout_set) throw StatusError(TSV_ESTATE, "recover: no layout set");
        if (!solution_valid) throw StatusError(TSV_ESTATE, "recover: no solution (call tsv_solve or tsv_set_solution)");
        if (points != 1 && points != 8) throw StatusError(TSV_EINVAL, "recover: points must be 1 (centroid) or 8 (Gauss)");
        const RomHost &m = rom[0].set ? rom[0] : rom[1];
        if (rom[0].set && rom[1].set)
            for (int a = 0; a < 3; ++a)
                if (rom[0].cells[a] != rom[1].cells[a]) throw StatusError(TSV_EINVAL, "recover: tsv/dummy meshes differ");
        (void)m;
    }

    size_t elems() const {
        const RomHost &m = rom[0].set ? rom[0] : rom[1];
        return m.cells[0] * m.cells[1] * m.cells[2];
    }

    // K6: U rows of GEMM tiles [t, t1) (U row = GEMM row - t kBM) =
    // Q Phi^T + dT u_T^T: the dense basis rows on the DMMA GEMM (scattered to
    // their fine DoFs through d_dmap), the sparse surface rows on k6_sparse_kernel.
    void launch_k6(const RomHost &mk, size_t t, size_t t1, double *Uout, size_t ldu) {
        GemmParams gp{};
        gp.A = X.ptr + t * kBM * ldk;
        gp.lda = static_cast<long long>(ldk);
        gp.Bt[0] = gp.Bt[1] = mk.d_phi.ptr;
        gp.ldb = static_cast<long long>(ldk);
        gp.tile_kind = nullptr;
        gp.C = Uout;
        gp.ldc = static_cast<long long>(ldu);
        gp.m_tiles = static_cast<int>(t1 - t);
        gp.n_tiles = static_cast<int>(round_up(std::max<size_t>(mk.n_dense, 1), kBN) / kBN);
        gp.k_chunks = static_cast<int>(ldk / kKC);
        gp.n_valid = static_cast<int>(mk.n_dense);
        gp.n_store = static_cast<int>(mk.n_dense);
        gp.row_scale = row_dt_d.ptr + t * kBM;
        gp.col_bias[0] = gp.col_bias[1] = mk.d_ut.ptr;
        gp.done = nullptr;
        gp.tile_counter = tile_counter.ptr;
        gp.n_major = 1;
        gp.col_map = mk.n_dense < mk.n_fine ? mk.d_dmap.ptr : nullptr;
        if (mk.n_dense && sym.on && mk.sym) {
            // mirror-symmetric ROM: 8 irrep GEMMs on the segmented Q panel
            // (recover_range built it), then the inverse transform over the
            // fine-DoF orbits scatters the dense rows into U
            GemmSegParams sg{};
            sg.A = sym.Xs.ptr + t * kBM * static_cast<size_t>(sym.lds);
            sg.lda = sym.lds;
            sg.Bt[0] = sg.Bt[1] = mk.d_phis.ptr;
            sg.tile_kind = nullptr;
            sg.C = sym.Us.ptr;
            sg.ldc = mk.sfine.ld;
            sg.m_tiles = static_cast<int>(t1 - t);
            sg.tiles_per_m = mk.k6_tiles_per_m;
            sg.n_segs = static_cast<int>(mk.k6_segs.size());
            sg.segs = mk.d_k6_segs.ptr;
            sg.row_scale = row_dt_d.ptr + t * kBM;
            sg.col_bias[0] = sg.col_bias[1] = mk.d_uts.ptr;
            sg.done = nullptr;
            sg.tile_counter = tile_counter.ptr;
            sg.m_major = 0;
            gemm_seg_f64<K6Cfg><<<std::min(k6_grid, sg.m_tiles * sg.tiles_per_m), K6Cfg::THREADS, K6Cfg::SMEM, stream>>>(sg);
            SymFineParams fp{};
            fp.Us = sym.Us.ptr;
            fp.ldus = mk.sfine.ld;
            fp.U = Uout;
            fp.ldu = static_cast<long long>(ldu);
            fp.rows = static_cast<int>((t1 - t) * kBM);
            fp.src = mk.d_fsrc.ptr;
            fp.dst = mk.d_fdst.ptr;
            fp.n_orbits = mk.sfine.n_orbits;
            dim3 fgrid(static_cast<unsigned>((fp.n_orbits + 255) / 256), static_cast<unsigned>((fp.rows + kFineRows - 1) / kFineRows));
            sym_fine_kernel<<<fgrid, 256, 0, stream>>>(fp);
            launches += 2;
        } else if (mk.n_dense) {
            gemm_nt_f64<K6Cfg><<<std::min(k6_grid, gp.m_tiles * gp.n_tiles), K6Cfg::THREADS, K6Cfg::SMEM, stream>>>(gp);
            ++launches;
        }
        if (mk.n_groups) {
            K6Face fp{};
            fp.X = X.ptr + t * kBM * ldk;
            fp.ldk = static_cast<long long>(ldk);
            fp.rows = static_cast<int>((t1 - t) * kBM);
            fp.row_dt = row_dt_d.ptr + t * kBM;
            fp.ginfo = mk.d_ginfo.ptr;
            fp.gcol = mk.d_gcol.ptr;
            fp.gwt = mk.d_gwt.ptr;
            fp.gwoff = mk.d_gwoff.ptr;
            fp.gdof = mk.d_gdof.ptr;
            fp.ut = mk.d_ut_full.ptr;
            fp.U = Uout;
            fp.ldu = static_cast<long long>(ldu);
            dim3 grid(static_cast<unsigned>((fp.rows + 32 * kFaceSub - 1) / (32 * kFaceSub)), static_cast<unsigned>(mk.n_groups),
                      static_cast<unsigned>((mk.max_group_rows + 127) / 128));
            const size_t smem = static_cast<size_t>(mk.max_group_k) * (32 + 128) * sizeof(double);
            CK(cudaFuncSetAttribute(k6_face_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            k6_face_kernel<<<grid, 256, smem, stream>>>(fp);
            ++launches;
        }
        if (mk.n_sparse) {
            K6Sparse sp{};
            sp.X = X.ptr + t * kBM * ldk;
            sp.ldk = static_cast<long long>(ldk);
            sp.rows = static_cast<int>((t1 - t) * kBM);
            sp.row_dt = row_dt_d.ptr + t * kBM;
            sp.n_sparse = static_cast<int>(mk.n_sparse);
            sp.ptr = mk.d_sp_ptr.ptr;
            sp.dof = mk.d_sp_dof.ptr;
            sp.col = mk.d_sp_col.ptr;
            sp.val = mk.d_sp_val.ptr;
            sp.ut = mk.d_ut_full.ptr;
            sp.U = Uout;
            sp.ldu = static_cast<long long>(ldu);
            const size_t smem = static_cast<size_t>(kK6sRows) * ldk * sizeof(double);
            CK(cudaFuncSetAttribute(k6_sparse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            dim3 grid(static_cast<unsigned>((sp.rows + kK6sRows - 1) / kK6sRows), 1);
            k6_sparse_kernel<<<grid, 256, smem, stream>>>(sp);
            ++launches;
        }
        CK(cudaGetLastError());
    }

    // Recover cells [c0, c1) into device buffer `out` (cells-relative).
    // Recover cells [c0, c1) into device buffer `out` (cells-relative):
    // points = 8 / 1 -> stress_kernel; points = -res -> cut-plane samples.
    void recover_range(int points, size_t c0, size_t c1, double *out) {
        const RomHost &m = rom[0].set ? rom[0] : rom[1];
        const size_t ldu = round_up(m.n_fine, 8);
        // Q panel: u at every DoF of every block (gather_cell_values does not mask).
        launch_scatter(x.ptr, 1);
        // M tiles holding the requested cells.
        std::vector<char> need(m_tiles, 0);
        for (size_t c = c0; c < c1; ++c) need[cell_row[c] / kBM] = 1;
        const size_t chunk_tiles = std::max<size_t>(1, std::min<size_t>(32, (size_t(1) << 30) / (ldu * 8 * kBM)));
        U.alloc(chunk_tiles * kBM * ldu);
        if (sym.on) {
            size_t ldus = 0;
            for (int k = 0; k < 2; ++k)
                if (rom[k].set && rom[k].sym) ldus = std::max<size_t>(ldus, static_cast<size_t>(rom[k].sfine.ld));
            sym.Us.alloc(chunk_tiles * kBM * ldus);
            launch_sym_panel(0, X.ptr, sym.Xs.ptr, false, nullptr);
        }
        StressParams sp{};
        sp.ldu = static_cast<long long>(ldu);
        sp.row_cell = row_cell_d.ptr;
        sp.row_kind = row_kind_d.ptr;
        sp.row_dt = row_dt_d.ptr;
        sp.cx = static_cast<int>(m.cells[0]);
        sp.cy = static_cast<int>(m.cells[1]);
        sp.cz = static_cast<int>(m.cells[2]);
        sp.P = points;
        for (int k = 0; k < 2; ++k) {
            const RomHost &mk = rom[k].set ? rom[k] : m;
            sp.hinv[k] = mk.d_hinv.ptr;
            sp.elem_mat[k] = mk.d_em.ptr;
            for (int a = 0; a < 3; ++a)
                for (int b2 = 0; b2 < 3; ++b2) sp.lame[k][a][b2] = mk.lame[a][b2];
        }
        sp.out = out;
        sp.out_cell0 = static_cast<long long>(c0);
        sp.out_cells = static_cast<long long>(c1 - c0);
        const size_t smem = stress_smem_bytes(points > 0 ? points : 1, static_cast<int>(m.cells[0]), static_cast<int>(m.cells[1]));
        if (points > 0) {
            if (smem > 227 * 1024) throw StatusError(TSV_EINVAL, "recover: element layer too large for shared memory");
            if (points == 8) CK(cudaFuncSetAttribute(stress_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            else CK(cudaFuncSetAttribute(stress_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        }
        // Opt-in (TSV_REC_OVERLAP=1): stress evaluation of chunk i on the side stream beside the reconstruction
        // of chunk i + 1 (two U buffers). Measured on B200 with the irrep K6: no gain (config 3 10.5 vs 10.4 ms,
        // config 4 10.05 vs 10.08 ms) - the persistent K6 grid and K7 take turns on the SMs.
        const char *eo = std::getenv("TSV_REC_OVERLAP");
        const bool overlap = points > 0 && eo && *eo == '1';
        if (overlap) U2.alloc(chunk_tiles * kBM * ldu);
        int chunk = 0;
        size_t t = 0;
        while (t < m_tiles) {
            if (!need[t]) { ++t; continue; }
            size_t t1 = t;
            while (t1 < m_tiles && need[t1] && t1 - t < chunk_tiles && tile_kind[t1] == tile_kind[t]) ++t1;
            const int kind = tile_kind[t];
            const RomHost &mk = rom[kind];
            const int ub = overlap ? (chunk & 1) : 0;
            double *Uc = ub ? U2.ptr : U.ptr;
            if (overlap && chunk >= 2) CK(cudaStreamWaitEvent(stream, k67_ev[2 + ub], 0));  // K7 of chunk - 2 has read this buffer
            launch_k6(mk, t, t1, Uc, ldu);
            if (points > 0) {
                cudaStream_t ks = stream;
                if (overlap) {
                    CK(cudaEventRecord(k67_ev[ub], stream));
                    CK(cudaStreamWaitEvent(side, k67_ev[ub], 0));
                    ks = side;
                }
                sp.U = Uc;
                sp.j0 = static_cast<int>(t * kBM);
                dim3 grid(static_cast<unsigned>(m.cells[2]), static_cast<unsigned>((t1 - t) * kBM));
                CK(cudaEventRecord(k7_event(), ks));
                if (points == 8) stress_kernel<8><<<grid, kStressThreads, smem, ks>>>(sp);
                else stress_kernel<1><<<grid, kStressThreads, smem, ks>>>(sp);
                CK(cudaEventRecord(k7_event(), ks));
                if (overlap) CK(cudaEventRecord(k67_ev[2 + ub], side));
                ++chunk;
            } else {
                const int res = -points;
                CutParams cp{};
                cp.U = U.ptr;
                cp.ldu = static_cast<long long>(ldu);
                cp.j0 = static_cast<int>(t * kBM);
                cp.row_cell = row_cell_d.ptr;
                cp.row_kind = row_kind_d.ptr;
                cp.row_dt = row_dt_d.ptr;
                for (int kk = 0; kk < 2; ++kk) {
                    const RomHost &mk2 = rom[kk].set ? rom[kk] : m;
                    for (int a = 0; a < 3; ++a) cp.grid[kk][a] = mk2.d_grid[a].ptr;
                    cp.elem_mat[kk] = mk2.d_em.ptr;
                    for (int a = 0; a < 3; ++a)
                        for (int b2 = 0; b2 < 3; ++b2) cp.lame[kk][a][b2] = mk2.lame[a][b2];
                }
                for (int a = 0; a < 3; ++a) cp.len[a] = static_cast<int>(m.grid[a].size());
                cp.res = res;
                cp.pitch = layout.pitch;
                cp.z_mid = 0.5 * layout.height;
                cp.out = out;
                cp.out_cell0 = static_cast<long long>(c0);
                cp.out_cells = static_cast<long long>(c1 - c0);
                dim3 grid(static_cast<unsigned>((t1 - t) * kBM), static_cast<unsigned>((res * res + 255) / 256));
                cutplane_kernel<<<grid, 256, 0, stream>>>(cp);
            }
            ++launches;  // stress or cut plane (launch_k6 counts its own)
            CK(cudaGetLastError());
            t = t1;
        }
        if (overlap) {  // join: the context stream continues after the last stress kernels
            for (int b2 = 0; b2 < std::min(chunk, 2); ++b2) CK(cudaStreamWaitEvent(stream, k67_ev[2 + b2], 0));
        }
    }
};

namespace {

template <typename F>
int guarded(tsv_ctx *ctx, F &&f) {
    if (!ctx) return TSV_EINVAL;
    struct AllocScope {
        cudaStream_t prev;
        explicit AllocScope(cudaStream_t s) : prev(tl_alloc_stream) { tl_alloc_stream = s; }
        ~AllocScope() { tl_alloc_stream = prev; }
    } scope(ctx->stream);
    try {
        int rc = f();
        if (rc == TSV_OK) ctx->err.clear();
        return rc;
    } catch (const StatusError &e) {
        ctx->err = e.what();
        return e.code;
    } catch (const tsvb200::Error &e) {
        ctx->err = e.what();
        return TSV_EINVAL;
    } catch (const std::bad_alloc &) {
        ctx->err = "host allocation failed";
        return TSV_ENOMEM;
    } catch (const std::exception &e) {
        ctx->err = e.what();
        return TSV_EINVAL;
    }
}

}  // namespace

extern "C" {

int tsv_abi_version(void) { return TSV_B200_ABI_VERSION; }

int tsv_host_register(void *ptr, size_t bytes) {
    return cudaHostRegister(ptr, bytes, cudaHostRegisterDefault) == cudaSuccess ? TSV_OK : TSV_ECUDA;
}

int tsv_host_unregister(void *ptr) { return cudaHostUnregister(ptr) == cudaSuccess ? TSV_OK : TSV_ECUDA; }

int tsv_host_alloc(size_t bytes, void **ptr) {
    if (!ptr) return TSV_EINVAL;
    *ptr = nullptr;
    const cudaError_t e = cudaHostAlloc(ptr, bytes, cudaHostAllocDefault);
    return e == cudaSuccess ? TSV_OK : (e == cudaErrorMemoryAllocation ? TSV_ENOMEM : TSV_ECUDA);
}

int tsv_host_free(void *ptr) { return cudaFreeHost(ptr) == cudaSuccess ? TSV_OK : TSV_ECUDA; }

int tsv_fp64_peak(int device, double *dmma_tflops, double *dfma_tflops) {
    if (cudaSetDevice(device) != cudaSuccess) return TSV_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double *sink = nullptr;
    if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return TSV_ENOMEM;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4000, warps = 16;
    float ms = 0.f;
    peak_dmma_kernel<<<sms, 32 * warps>>>(sink, 64);
    cudaEventRecord(e0);
    peak_dmma_kernel<<<sms, 32 * warps>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (dmma_tflops) *dmma_tflops = 2.0 * 256 * 8 * iters * double(sms) * warps / ms / 1e9;
    peak_dfma_kernel<<<sms, 32 * warps>>>(sink, 64);
    cudaEventRecord(e0);
    peak_dfma_kernel<<<sms, 32 * warps>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (dfma_tflops) *dfma_tflops = 2.0 * 16 * iters * double(sms) * 32 * warps / ms / 1e9;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? TSV_OK : TSV_ECUDA;
}

int tsv_index_global_nodes(uint32_t rows, uint32_t cols, const uint32_t q[3], uint64_t *n_dofs, uint32_t lattice[3],
                           int32_t *nol, uint32_t *lon, uint32_t *dm) {
    try {
        if (!q) return TSV_EINVAL;
        ArrayLayout L;
        L.rows = rows;
        L.cols = cols;
        L.delta_t = {0.0};
        L.pitch = 1.0;
        L.height = 1.0;
        NodeLayout nl = NodeLayout::create(q[0], q[1], q[2]);
        GlobalIndex idx = index_global_nodes(L, nl);
        if (n_dofs) *n_dofs = idx.dof_count();
        if (lattice) {
            lattice[0] = idx.lat_x;
            lattice[1] = idx.lat_y;
            lattice[2] = idx.lat_z;
        }
        if (nol) std::memcpy(nol, idx.node_of_lattice.data(), idx.node_of_lattice.size() * sizeof(int32_t));
        if (lon)
            for (size_t i = 0; i < idx.node_count(); ++i)
                for (int c = 0; c < 3; ++c) lon[3 * i + c] = idx.lattice_of_node[i][c];
        if (dm) {
            std::vector<uint32_t> m = tsvb200::dof_map(L, idx, nl);
            std::memcpy(dm, m.data(), m.size() * sizeof(uint32_t));
        }
        return TSV_OK;
    } catch (...) {
        return TSV_EINVAL;
    }
}

int tsv_ctx_create(int device, tsv_ctx **out) {
    if (!out) return TSV_EINVAL;
    *out = nullptr;
    auto ctx = std::make_unique<tsv_ctx>();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return TSV_ECUDA;
    int rc = guarded(ctx.get(), [&] {
        CK(cudaStreamCreateWithFlags(&ctx->own_stream.s, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->own_side.s, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->own_copy.s, cudaStreamNonBlocking));
        ctx->stream = ctx->own_stream.s;
        ctx->side = ctx->own_side.s;
        ctx->copy = ctx->own_copy.s;
        for (auto &e : ctx->rec_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto &e : ctx->k67_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        {
            // freed temporaries stay in the pool up to 16 GB (no OS round trip per set-up)
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, device));
            uint64_t thr = 16ull << 30;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        }
        CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
        CK(cudaEventCreate(&ctx->ev0));
        CK(cudaEventCreate(&ctx->ev1));
        CK(cudaMallocHost(&ctx->h_state, sizeof(CgState)));
        CK(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
        CK(cudaDeviceGetAttribute(&ctx->coop_launch, cudaDevAttrCooperativeLaunch, device));
        CK(cudaFuncSetAttribute(gemm_nt_f64<K1Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(K1Cfg::SMEM)));
        CK(cudaFuncSetAttribute(gemm_nt_f64<K6Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(K6Cfg::SMEM)));
        CK(cudaFuncSetAttribute(gemm_streamk_f64<K1Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(K1Cfg::SMEM)));
        CK(cudaFuncSetAttribute(gemm_nt_f64<K1SmallCfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(K1SmallCfg::SMEM)));
        CK(cudaFuncSetAttribute(gemm_splitk_f64<K1SmallCfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(K1SmallCfg::SMEM)));
        int occ_s = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, gemm_nt_f64<K1SmallCfg>, K1SmallCfg::THREADS,
                                                         K1SmallCfg::SMEM));
        ctx->k1s_grid = std::max(1, occ_s) * ctx->sm_count;
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_nt_f64<K1Cfg>, K1Cfg::THREADS, K1Cfg::SMEM));
        ctx->k1_grid = std::max(1, occ) * ctx->sm_count;
        int occ6 = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ6, gemm_nt_f64<K6Cfg>, K6Cfg::THREADS, K6Cfg::SMEM));
        ctx->k6_grid = std::max(1, occ6) * ctx->sm_count;
        int occ_sk = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_sk, gemm_streamk_f64<K1Cfg>, K1Cfg::THREADS, K1Cfg::SMEM));
        ctx->sk_resident = occ_sk * ctx->sm_count >= ctx->k1_grid;  // stream-K waits need every CTA resident
        ctx->tile_counter.alloc(2);
        CK(cudaMemset(ctx->tile_counter.ptr, 0, 2 * sizeof(unsigned)));
        ctx->state.alloc(1);
        CK(cudaMemset(ctx->state.ptr, 0, sizeof(CgState)));
        ctx->zero_flag.alloc(1);
        CK(cudaMemset(ctx->zero_flag.ptr, 0, sizeof(int)));
        return TSV_OK;
    });
    if (rc != TSV_OK) return rc;
    *out = ctx.release();
    return TSV_OK;
}

void tsv_ctx_destroy(tsv_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    delete ctx;
}

const char *tsv_last_error(const tsv_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int tsv_set_rom(tsv_ctx *ctx, int kind, const tsv_rom_desc *d) {
    return guarded(ctx, [&] {
        if (kind != 0 && kind != 1) throw StatusError(TSV_EINVAL, "set_rom: kind must be 0 (tsv) or 1 (dummy)");
        if (!d || !d->a_element || !d->b_element || !d->basis || !d->thermal)
            throw StatusError(TSV_EINVAL, "set_rom: missing ROM arrays");
        for (int a = 0; a < 3; ++a) {
            if (d->q[a] < 2) throw StatusError(TSV_EINVAL, "NodeLayout: need at least 2 interpolation nodes per axis");
            if (d->grid_len[a] < 2 || !d->grid[a]) throw StatusError(TSV_EINVAL, "grid: axis needs at least 2 lines");
        }
        cudaSetDevice(ctx->device);
        RomHost &m = ctx->rom[kind];
        m.set = false;
        std::copy(d->q, d->q + 3, m.q);
        std::copy(d->geometry, d->geometry + 4, m.geom);
        for (int a = 0; a < 3; ++a) {
            m.grid[a].assign(d->grid[a], d->grid[a] + d->grid_len[a]);
            for (size_t i = 1; i < m.grid[a].size(); ++i)
                if (!(m.grid[a][i] > m.grid[a][i - 1])) throw StatusError(TSV_EINVAL, "grid: axis must be strictly increasing");
            m.cells[a] = d->grid_len[a] - 1;
        }
        for (int i = 0; i < 3; ++i) {
            const double E = d->materials[i][0], nu = d->materials[i][1], alpha = d->materials[i][2];
            if (!(E > 0.0)) throw StatusError(TSV_EINVAL, "material: Young modulus must be > 0");
            if (!(nu > -1.0) || !(nu < 0.5)) throw StatusError(TSV_EINVAL, "material: Poisson ratio must lie in (-1, 0.5)");
            // lame_parameters, material.cpp:7-15
            const double lambda = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
            const double mu = E / (2.0 * (1.0 + nu));
            m.mats[i][0] = E;
            m.mats[i][1] = nu;
            m.mats[i][2] = alpha;
            m.lame[i][0] = lambda;
            m.lame[i][1] = mu;
            m.lame[i][2] = alpha * (3.0 * lambda + 2.0 * mu);
        }
        const size_t E = m.cells[0] * m.cells[1] * m.cells[2];
        m.elem_mat.assign(E, 2);
        if (d->element_material) {
            m.elem_mat.assign(d->element_material, d->element_material + E);
        } else if (kind == 0) {  // classify_tsv by centroid radius, mesh.cpp:182-190
            const double dd = d->geometry[0], t = d->geometry[2], p = d->geometry[3];
            for (size_t k = 0; k < m.cells[2]; ++k)
                for (size_t j = 0; j < m.cells[1]; ++j)
                    for (size_t i = 0; i < m.cells[0]; ++i) {
                        const double xc = 0.5 * (m.grid[0][i] + m.grid[0][i + 1]);
                        const double yc = 0.5 * (m.grid[1][j] + m.grid[1][j + 1]);
                        const double rr = std::hypot(xc - 0.5 * p, yc - 0.5 * p);
                        m.elem_mat[(k * m.cells[1] + j) * m.cells[0] + i] =
                            rr < 0.5 * dd ? 0 : (rr < 0.5 * dd + t ? 1 : 2);
                    }
        }
        for (uint8_t v : m.elem_mat)
            if (v > 2) throw StatusError(TSV_EINVAL, "set_rom: element material id out of range");
        const size_t n = num_element_dofs(d->q[0], d->q[1], d->q[2]);
        const size_t n_fine = (m.cells[0] + 1) * (m.cells[1] + 1) * (m.cells[2] + 1) * 3;
        m.n = n;
        m.n_fine = n_fine;
        std::memcpy(m.fingerprint, d->fingerprint, 32);
        m.k_r.assign(d->a_element, d->a_element + n * n);
        m.b_el.assign(d->b_element, d->b_element + n);
        m.d_bel.upload(m.b_el.data(), n, ctx->stream);
        m.u_t.assign(d->thermal, d->thermal + n_fine);
        const size_t ldk = round_up(n, kKC);
        {
            std::vector<double> kp(round_up(n, kBN) * ldk, 0.0);
            // component-major permutation a = 3 rank + c -> c nn + rank on both sides
            const size_t nn = n / 3;
            for (size_t a = 0; a < n; ++a)
                for (size_t k = 0; k < n; ++k) kp[pidx(a, nn) * ldk + pidx(k, nn)] = d->a_element[a * n + k];
            m.d_k.upload(kp.data(), kp.size(), ctx->stream);
            CK(cudaStreamSynchronize(ctx->stream));
            m.oz_s = 0;  // int8 digit planes are rebuilt on next use
        }
        {
            // Basis rows with at most n/4 non-zeros (surface nodes: q^2, q or 1
            // interpolation weights) go to the CSR path (k6_sparse_kernel), the
            // rest to the dense GEMM.
            const size_t kSparseRowMax = n / 4;
            const bool split = !tsv_ctx::getenv_flag("TSV_K6_DENSE");
            const size_t nn = n / 3;
            std::vector<int> dmap, sp_ptr(1, 0), sp_dof, sp_col;
            std::vector<double> sp_val;
            // (face, component) groups of the surface rows; a row whose group's
            // column union exceeds kFaceK stays on the CSR path
            const size_t nx = m.cells[0] + 1, ny = m.cells[1] + 1;
            std::vector<std::vector<int>> grows(18);
            std::vector<std::vector<char>> gmask(18, std::vector<char>(n, 0));
            std::vector<int> sparse_rows;
            for (size_t f = 0; f < n_fine; ++f) {
                const double *row = d->basis + f * n;
                size_t nz = 0;
                for (size_t a = 0; a < n; ++a) nz += row[a] != 0.0;
                if (!(split && nz <= kSparseRowMax)) {
                    dmap.push_back(static_cast<int>(f));
                    continue;
                }
                const size_t node = f / 3, comp = f % 3;
                const size_t i = node % nx, j = (node / nx) % ny, k = node / (nx * ny);
                const int face = k == 0 ? 0 : k == m.cells[2] ? 1 : j == 0 ? 2 : j == m.cells[1] ? 3 : i == 0 ? 4 : i == m.cells[0] ? 5 : -1;
                if (face < 0 || tsv_ctx::getenv_flag("TSV_K6_CSR")) {
                    sparse_rows.push_back(static_cast<int>(f));
                    continue;
                }
                grows[face * 3 + comp].push_back(static_cast<int>(f));
                for (size_t a = 0; a < n; ++a)
                    if (row[a] != 0.0) gmask[face * 3 + comp][a] = 1;
            }
            std::vector<int4> ginfo;
            std::vector<int> gcol, gdof;
            std::vector<double> gwt;
            std::vector<long long> gwoff;
            m.max_group_rows = 0;
            m.max_group_k = 0;
            for (int g = 0; g < 18; ++g) {
                if (grows[g].empty()) continue;
                std::vector<int> cols;  // reduced DoFs a (reference order)
                for (size_t a = 0; a < n; ++a)
                    if (gmask[g][a]) cols.push_back(static_cast<int>(a));
                if (cols.size() > static_cast<size_t>(kFaceK)) {
                    sparse_rows.insert(sparse_rows.end(), grows[g].begin(), grows[g].end());
                    continue;
                }
                const int nr = static_cast<int>(grows[g].size()), K = static_cast<int>(cols.size());
                ginfo.push_back(make_int4(static_cast<int>(gdof.size()), nr, static_cast<int>(gcol.size()), K));
                gwoff.push_back(static_cast<long long>(gwt.size()));
                for (int a : cols) gcol.push_back(static_cast<int>(pidx(static_cast<size_t>(a), nn)));
                gdof.insert(gdof.end(), grows[g].begin(), grows[g].end());
                for (int kk = 0; kk < K; ++kk)  // W^T [K][rows]
                    for (int r = 0; r < nr; ++r) gwt.push_back(d->basis[static_cast<size_t>(grows[g][r]) * n + cols[kk]]);
                m.max_group_rows = std::max(m.max_group_rows, nr);
                m.max_group_k = std::max(m.max_group_k, K);
            }
            m.n_groups = static_cast<int>(ginfo.size());
            std::sort(sparse_rows.begin(), sparse_rows.end());
            for (int f : sparse_rows) {
                const double *row = d->basis + static_cast<size_t>(f) * n;
                sp_dof.push_back(f);
                for (size_t a = 0; a < n; ++a)
                    if (row[a] != 0.0) {
                        sp_col.push_back(static_cast<int>(pidx(a, nn)));
                        sp_val.push_back(row[a]);
                    }
                sp_ptr.push_back(static_cast<int>(sp_col.size()));
            }
            if (m.n_groups) {
                m.d_ginfo.upload(ginfo.data(), ginfo.size(), ctx->stream);
                m.d_gcol.upload(gcol.data(), gcol.size(), ctx->stream);
                m.d_gdof.upload(gdof.data(), gdof.size(), ctx->stream);
                m.d_gwt.upload(gwt.data(), gwt.size(), ctx->stream);
                m.d_gwoff.upload(gwoff.data(), gwoff.size(), ctx->stream);
            }
            m.n_dense = dmap.size();
            m.n_sparse = sp_dof.size();
            const size_t rows = round_up(std::max<size_t>(m.n_dense, 1), kBN);
            std::vector<double> pp(rows * ldk, 0.0), ut(rows, 0.0);
            for (size_t i = 0; i < m.n_dense; ++i) {
                const size_t f = static_cast<size_t>(dmap[i]);
                for (size_t a = 0; a < n; ++a) pp[i * ldk + pidx(a, nn)] = d->basis[f * n + a];
                ut[i] = d->thermal[f];
            }
            m.d_phi.upload(pp.data(), pp.size(), ctx->stream);
            m.d_ut.upload(ut.data(), ut.size(), ctx->stream);
            m.d_ut_full.upload(d->thermal, n_fine, ctx->stream);
            if (m.n_dense < n_fine) m.d_dmap.upload(dmap.data(), dmap.size(), ctx->stream);
            if (m.n_sparse) {
                m.d_sp_ptr.upload(sp_ptr.data(), sp_ptr.size(), ctx->stream);
                m.d_sp_dof.upload(sp_dof.data(), sp_dof.size(), ctx->stream);
                m.d_sp_col.upload(sp_col.data(), std::max<size_t>(sp_col.size(), 1), ctx->stream);
                m.d_sp_val.upload(sp_val.data(), std::max<size_t>(sp_val.size(), 1), ctx->stream);
            }
            if (m.n_dense == n_fine) m.d_dmap.release();
            CK(cudaStreamSynchronize(ctx->stream));
            {
                PhaseTimer pts("  rom symmetry");
                std::vector<double> kpu(n * n);
                for (size_t a = 0; a < n; ++a)
                    for (size_t k = 0; k < n; ++k) kpu[pidx(a, nn) * n + pidx(k, nn)] = d->a_element[a * n + k];
                build_rom_symmetry(m, kpu, d->basis, d->thermal, dmap, ctx->stream, kBN, kKC);
                if (tsv_ctx::getenv_flag("TSV_TIMING"))
                    std::fprintf(stderr, "[tsv] rom kind %d: mirror symmetry %s (defect K %.2e, Phi %.2e)\n", kind,
                                 m.sym ? "on" : "off", m.sym_defect_k, m.sym_defect_phi);
            }
        }
        std::vector<double> hinv;
        for (int a = 0; a < 3; ++a)
            for (size_t i = 0; i < m.cells[a]; ++i) hinv.push_back(1.0 / (m.grid[a][i + 1] - m.grid[a][i]));
        m.d_hinv.upload(hinv.data(), hinv.size(), ctx->stream);
        for (int a = 0; a < 3; ++a) m.d_grid[a].upload(m.grid[a].data(), m.grid[a].size(), ctx->stream);
        m.d_em.upload(m.elem_mat.data(), E, ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
        m.set = true;
        ctx->layout_set = false;  // layout tables depend on the RomSet
        ctx->drop_graph();
        ctx->solution_valid = false;
        return TSV_OK;
    });
}

int tsv_set_layout(tsv_ctx *ctx, uint32_t rows, uint32_t cols, const uint8_t *kinds, const double *delta_t,
                   size_t n_delta_t, double pitch, double height) {
    return guarded(ctx, [&] {
        cudaSetDevice(ctx->device);
        ctx->build_layout(rows, cols, kinds, delta_t, n_delta_t, pitch, height);
        return TSV_OK;
    });
}

int tsv_set_delta_t(tsv_ctx *ctx, const double *delta_t, size_t n_delta_t) {
    return guarded(ctx, [&] {
        cudaSetDevice(ctx->device);
        ctx->set_delta_t(delta_t, n_delta_t);
        return TSV_OK;
    });
}

int tsv_set_dirichlet(tsv_ctx *ctx, size_t count, const uint32_t *dofs, const double *values) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "set_dirichlet: no layout set");
        if (count && (!dofs || !values)) throw StatusError(TSV_EINVAL, "set_dirichlet: NULL arrays");
        DirichletSet set;
        for (size_t i = 0; i < count; ++i) set.set(dofs[i], values[i]);
        std::vector<uint8_t> mask(ctx->N, 0);
        for (const auto &e : set.entries()) {
            if (e.first >= ctx->N)
                throw StatusError(TSV_EINVAL, "apply_dirichlet_lifting: dof " + std::to_string(e.first) + " out of range");
            mask[e.first] = 1;
        }
        cudaSetDevice(ctx->device);
        ctx->drop_graph();
        ctx->set_bc_mask(std::move(mask), set.entries());
        return TSV_OK;
    });
}

int tsv_set_bc(tsv_ctx *ctx, int bc_kind) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "set_bc: no layout set");
        if (bc_kind < 0 || bc_kind > 3) throw StatusError(TSV_EINVAL, "set_bc: unknown boundary condition");
        PhaseTimer pt("  reduced_dirichlet");
        DirichletSet set = reduced_dirichlet(static_cast<BcKind>(bc_kind), ctx->index);
        pt.lap("  bc mask");
        std::vector<uint8_t> mask(ctx->N, 0);
        for (const auto &e : set.entries()) mask[e.first] = 1;
        cudaSetDevice(ctx->device);
        ctx->drop_graph();
        pt.lap("  set_bc_mask");
        ctx->set_bc_mask(std::move(mask), set.entries());
        return TSV_OK;
    });
}

int tsv_get_index(tsv_ctx *ctx, uint64_t *n_dofs, uint64_t *n_nodes, uint32_t lattice[3], uint32_t *n_reduced) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "get_index: no layout set");
        if (n_dofs) *n_dofs = ctx->N;
        if (n_nodes) *n_nodes = ctx->nodes;
        if (lattice) {
            lattice[0] = ctx->index.lat_x;
            lattice[1] = ctx->index.lat_y;
            lattice[2] = ctx->index.lat_z;
        }
        if (n_reduced) *n_reduced = static_cast<uint32_t>(ctx->n);
        return TSV_OK;
    });
}

int tsv_get_dof_map(tsv_ctx *ctx, uint32_t *out) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "get_dof_map: no layout set");
        std::memcpy(out, ctx->dofmap.data(), ctx->dofmap.size() * sizeof(uint32_t));
        return TSV_OK;
    });
}

int tsv_get_lattice(tsv_ctx *ctx, int32_t *nol, uint32_t *lon) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "get_lattice: no layout set");
        if (nol) std::memcpy(nol, ctx->index.node_of_lattice.data(), ctx->index.node_of_lattice.size() * 4);
        if (lon)
            for (size_t i = 0; i < ctx->nodes; ++i)
                for (int c = 0; c < 3; ++c) lon[3 * i + c] = ctx->index.lattice_of_node[i][c];
        return TSV_OK;
    });
}

int tsv_get_constrained(tsv_ctx *ctx, uint8_t *mask) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "get_constrained: no layout set");
        std::memcpy(mask, ctx->constrained.data(), ctx->N);
        return TSV_OK;
    });
}

int tsv_get_load(tsv_ctx *ctx, double *bout) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "get_load: no layout set");
        cudaSetDevice(ctx->device);
        std::vector<double> bi(ctx->N);
        ctx->ensure_rhs();
        d2h(bi.data(), ctx->b.ptr, ctx->N * sizeof(double), ctx->stream);
        ctx->to_reference(bi.data(), bout);
        return TSV_OK;
    });
}

int tsv_apply(tsv_ctx *ctx, const double *xin, double *yout) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "apply: no layout set");
        cudaSetDevice(ctx->device);
        std::vector<double> xi = ctx->to_internal(xin);
        ctx->r.upload(xi.data(), ctx->N, ctx->stream);
        ctx->launch_scatter(ctx->r.ptr, 0);
        ctx->launch_k1(nullptr);
        gather_vec_kernel<<<ctx->vec_grid(), kVecThreads, 0, ctx->stream>>>(
            static_cast<int>(ctx->nodes), static_cast<int>(ctx->n / 3), ctx->slots.ptr, ctx->cmask.ptr, ctx->Y.ptr, ctx->r.ptr,
            ctx->ap.ptr, 0);
        ++ctx->launches;
        CK(cudaGetLastError());
        std::vector<double> yi(ctx->N);
        CK(cudaMemcpyAsync(yi.data(), ctx->ap.ptr, ctx->N * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->to_reference(yi.data(), yout);
        return TSV_OK;
    });
}

int tsv_precond_apply(tsv_ctx *ctx, int precond, const double *r_in, double *z_out) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "precond_apply: no layout set");
        if (precond != TSV_PRECOND_SCHWARZ2) throw StatusError(TSV_EINVAL, "precond_apply: only the Schwarz preconditioner");
        cudaSetDevice(ctx->device);
        ctx->build_precond(precond);
        std::vector<double> ri = ctx->to_internal(r_in);
        ctx->r.upload(ri.data(), ctx->N, ctx->stream);
        CgState st{};
        st.done = CG_RUNNING;
        st.phase = PH_RESTART;  // use r as is
        st.tol = 1.0;
        st.max_it = 1;
        *ctx->h_state = st;
        CK(cudaMemcpyAsync(ctx->state.ptr, ctx->h_state, sizeof(CgState), cudaMemcpyHostToDevice, ctx->stream));
        CgParams q = ctx->cg_params();
        ctx->launch_as_update_precond(q, false);
        ctx->launch_scatter_p(q, 1);  // z = z_l + P zc (p / panel updates are discarded)
        CK(cudaGetLastError());
        std::vector<double> zi(ctx->N);
        CK(cudaMemcpyAsync(zi.data(), ctx->as2.z.ptr, ctx->N * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->to_reference(zi.data(), z_out);
        ctx->solution_valid = false;
        return TSV_OK;
    });
}

int tsv_precond_setup(tsv_ctx *ctx, int precond, tsv_precond_info *out) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "precond_setup: no layout set");
        if (precond < TSV_PRECOND_NONE || precond > TSV_PRECOND_SCHWARZ2)
            throw StatusError(TSV_EINVAL, "precond_setup: unknown preconditioner");
        cudaSetDevice(ctx->device);
        const auto t0 = std::chrono::steady_clock::now();
        const bool had = ctx->pre_kind == precond;
        ctx->build_precond(precond);
        CK(cudaStreamSynchronize(ctx->stream));
        if (out) {
            *out = tsv_precond_info{};
            out->setup_ms = had ? 0.0 : std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (precond == TSV_PRECOND_SCHWARZ2) {
                out->ntypes = ctx->as2.ntypes;
                out->coarse_dofs = ctx->as2.Nc;
                out->super_block = ctx->as2.s;
                out->local_rows = static_cast<int>(ctx->as2.BL_pad);
            }
        }
        return TSV_OK;
    });
}

// Test hook: the coarse level of the last tsv_precond_apply (rc, zc) and A_c^-1.
int tsv_debug_coarse(tsv_ctx *ctx, int *nc, double *rc, double *zc, double *ainv) {
    return guarded(ctx, [&] {
        if (!ctx->as2.rc.ptr) throw StatusError(TSV_ESTATE, "debug_coarse: no Schwarz preconditioner built");
        const size_t Nc = static_cast<size_t>(ctx->as2.Nc);
        if (nc) *nc = static_cast<int>(Nc);
        if (rc) d2h(rc, ctx->as2.rc.ptr, Nc * sizeof(double), ctx->stream);
        if (zc) d2h(zc, ctx->as2.zc.ptr, Nc * sizeof(double), ctx->stream);
        if (ainv) d2h(ainv, ctx->as2.ainv_c.ptr, Nc * Nc * sizeof(double), ctx->stream);
        return TSV_OK;
    });
}

int tsv_solve(tsv_ctx *ctx, const tsv_iter_options *opts, double *u_out, tsv_solve_info *info) {
    return guarded(ctx, [&] {
        if (!opts) throw StatusError(TSV_EINVAL, "solve: NULL options");
        cudaSetDevice(ctx->device);
        ctx->ensure_rhs();
        return ctx->solve(*opts, u_out, info);
    });
}

int tsv_set_solution(tsv_ctx *ctx, const double *u) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "set_solution: no layout set");
        cudaSetDevice(ctx->device);
        std::vector<double> ui = ctx->to_internal(u);
        ctx->x.upload(ui.data(), ctx->N, ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->solution_valid = true;
        return TSV_OK;
    });
}

int tsv_recover(tsv_ctx *ctx, int points, uint64_t c0, uint64_t c1, double *out) {
    return guarded(ctx, [&] {
        cudaSetDevice(ctx->device);
        ctx->check_recovery(points);
        if (c0 > c1 || c1 > ctx->B) throw StatusError(TSV_EINVAL, "recover: cell range out of bounds");
        if (c0 == c1) return TSV_OK;
        const size_t per_cell = ctx->elems() * static_cast<size_t>(points) * 7;
        // Chunks of whole 128-block GEMM tiles (~1 GB), double-buffered: chunk
        // i+1 is computed on the context stream while chunk i is copied to the
        // host on the copy stream (the D2H over PCIe is the bound).
        size_t max_cells = std::max<size_t>(1, (size_t(1) << 30) / (per_cell * sizeof(double)));
        if (max_cells >= kBM) max_cells = max_cells / kBM * kBM;
        const size_t stage = std::min(max_cells, static_cast<size_t>(c1 - c0)) * per_cell;
        for (auto &sb : ctx->rstage)
            if (sb.count < stage) sb.alloc(stage);
        cudaEvent_t *computed = ctx->rec_ev, *copied = ctx->rec_ev + 2;
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        int i = 0;
        for (size_t a = c0; a < c1; a += max_cells, ++i) {
            const size_t b2 = std::min<size_t>(c1, a + max_cells);
            const int k = i & 1;
            if (i >= 2) CK(cudaStreamWaitEvent(ctx->stream, copied[k], 0));
            ctx->recover_range(points, a, b2, ctx->rstage[k].ptr);
            CK(cudaEventRecord(computed[k], ctx->stream));
            CK(cudaStreamWaitEvent(ctx->copy, computed[k], 0));
            CK(cudaMemcpyAsync(out + (a - c0) * per_cell, ctx->rstage[k].ptr, (b2 - a) * per_cell * sizeof(double),
                               cudaMemcpyDeviceToHost, ctx->copy));
            CK(cudaEventRecord(copied[k], ctx->copy));
        }
        CK(cudaStreamWaitEvent(ctx->stream, copied[(i - 1) & 1], 0));
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        CK(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->last_recover_ms = ms;
        ctx->collect_stress_times();
        return TSV_OK;
    });
}

int tsv_recover_resident(tsv_ctx *ctx, int points) {
    return guarded(ctx, [&] {
        cudaSetDevice(ctx->device);
        ctx->check_recovery(points);
        const size_t per_cell = ctx->elems() * static_cast<size_t>(points) * 7;
        ctx->stress.alloc(ctx->B * per_cell);
        ctx->stress_points = points;
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        ctx->recover_range(points, 0, ctx->B, ctx->stress.ptr);
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        CK(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->last_recover_ms = ms;
        ctx->collect_stress_times();
        return TSV_OK;
    });
}

int tsv_copy_stress(tsv_ctx *ctx, uint64_t c0, uint64_t c1, double *out) {
    return guarded(ctx, [&] {
        if (!ctx->stress.ptr) throw StatusError(TSV_ESTATE, "copy_stress: call tsv_recover_resident first");
        if (c0 > c1 || c1 > ctx->B) throw StatusError(TSV_EINVAL, "copy_stress: cell range out of bounds");
        cudaSetDevice(ctx->device);
        const size_t per_cell = ctx->elems() * static_cast<size_t>(ctx->stress_points) * 7;
        d2h(out, ctx->stress.ptr + c0 * per_cell, (c1 - c0) * per_cell * sizeof(double), ctx->stream);
        return TSV_OK;
    });
}

int tsv_cutplane(tsv_ctx *ctx, uint32_t res, double *out) {
    return guarded(ctx, [&] {
        cudaSetDevice(ctx->device);
        ctx->check_recovery(8);
        if (res < 1) throw StatusError(TSV_EINVAL, "StressGrid: rows, cols, res must be >= 1");
        const size_t per_cell = static_cast<size_t>(res) * res;
        const size_t max_cells = std::max<size_t>(1, (size_t(1) << 30) / (per_cell * sizeof(double)));
        DevBuf<double> dout;
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        for (size_t a = 0; a < ctx->B; a += max_cells) {
            const size_t b2 = std::min<size_t>(ctx->B, a + max_cells);
            dout.alloc((b2 - a) * per_cell);
            ctx->recover_range(-static_cast<int>(res), a, b2, dout.ptr);
            CK(cudaMemcpyAsync(out + a * per_cell, dout.ptr, (b2 - a) * per_cell * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        CK(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->last_recover_ms = ms;
        ctx->collect_stress_times();
        return TSV_OK;
    });
}

int tsv_block_field(tsv_ctx *ctx, uint64_t cell, double *out) {
    return guarded(ctx, [&] {
        cudaSetDevice(ctx->device);
        ctx->check_recovery(8);
        if (cell >= ctx->B) throw StatusError(TSV_EINVAL, "block_field: cell out of range");
        const int j = ctx->cell_row[cell];
        const size_t t = j / kBM;
        const RomHost &mk = ctx->rom[ctx->tile_kind[t]];
        const size_t ldu = round_up(mk.n_fine, 8);
        ctx->launch_scatter(ctx->x.ptr, 1);
        ctx->U.alloc(std::max(ctx->U.count, kBM * ldu));
        if (ctx->sym.on) {
            ctx->sym.Us.alloc(std::max(ctx->sym.Us.count, kBM * static_cast<size_t>(mk.sfine.ld)));
            ctx->launch_sym_panel(0, ctx->X.ptr, ctx->sym.Xs.ptr, false, nullptr);
        }
        ctx->launch_k6(mk, t, t + 1, ctx->U.ptr, ldu);
        CK(cudaMemcpyAsync(out, ctx->U.ptr + (j - t * kBM) * ldu, mk.n_fine * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        return TSV_OK;
    });
}

int tsv_profile_apply(tsv_ctx *ctx, int reps, double *ms_per_launch) {
    return guarded(ctx, [&] {
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "profile_apply: no layout set");
        if (reps < 1) throw StatusError(TSV_EINVAL, "profile_apply: reps must be >= 1");
        cudaSetDevice(ctx->device);
        ctx->launch_k1(nullptr);  // warm-up
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        for (int i = 0; i < reps; ++i) ctx->launch_k1(nullptr);
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        CK(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->last_apply_ms = ms / reps;
        if (ms_per_launch) *ms_per_launch = ctx->last_apply_ms;
        return TSV_OK;
    });
}

int tsv_get_symmetry(tsv_ctx *ctx, tsv_symmetry_info *out) {
    return guarded(ctx, [&] {
        if (!out) throw StatusError(TSV_EINVAL, "get_symmetry: null output");
        if (!ctx->layout_set) throw StatusError(TSV_ESTATE, "get_symmetry: no layout set");
        std::memset(out, 0, sizeof *out);
        out->recovery_symmetric = ctx->sym.on;
        out->operator_symmetric = ctx->sym.k1;
        out->defect_correction = ctx->sym.corr;
        out->operator_fused = ctx->sym.k1 && ctx->sym.fused;
        for (int k = 0; k < 2; ++k) {
            out->defect_k[k] = ctx->rom[k].set ? ctx->rom[k].sym_defect_k : 0.0;
            out->defect_phi[k] = ctx->rom[k].set ? ctx->rom[k].sym_defect_phi : 0.0;
        }
        if (ctx->sym.on)
            for (int r = 0; r < 8; ++r) out->irrep_dofs[r] = ctx->rom[ctx->sym.tab_kind].sred.count[r];
        return TSV_OK;
    });
}

int tsv_get_timing(tsv_ctx *ctx, tsv_timing *out) {
    return guarded(ctx, [&] {
        out->solve_ms = ctx->last_solve_ms;
        out->recover_ms = ctx->last_recover_ms;
        out->apply_ms_avg = ctx->last_apply_ms;
        out->kernel_launches = ctx->launches;
        out->stress_ms = ctx->last_stress_ms;
        out->stress_launches = ctx->last_stress_launches;
        return TSV_OK;
    });
}

}  // extern "C"
