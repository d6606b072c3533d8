/*
 * tsv_b200.h — C ABI of the B200-native online stage of MORE-Stress
 * (reduced global solve + per-block stress recovery).
 *
 * Plain pointers and sizes only; no exceptions and no torch/CUDA types
 * cross this boundary. Every entry point names the reference interface it
 * replaces (tsvstress, /root/reference/proj). One context owns all device
 * memory and one CUDA stream on one GPU; a context is not thread-safe, but
 * separate contexts may be used concurrently.
 *
 * Status codes mirror the reference's exception types (core.hpp:14-16,
 * linalg.hpp:137-141, linalg.cpp:333-334): see tsv_status.
 */
#ifndef TSV_B200_H
#define TSV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSV_B200_ABI_VERSION 1

typedef struct tsv_ctx tsv_ctx;

typedef enum {
    TSV_OK = 0,
    TSV_EINVAL = 1,      /* tsvstress::Error from validation (e.g. ArrayLayout::validate, global_stage.cpp:8-15) */
    TSV_ENOCONV = 2,     /* linalg::NoConvergence (linalg.hpp:137-141); best iterate returned */
    TSV_EBREAKDOWN = 3,  /* "NaN/Inf breakdown" / "p'Ap <= 0" (linalg.cpp:217, :333-334) */
    TSV_ECUDA = 4,       /* CUDA runtime failure */
    TSV_ENOMEM = 5,      /* device allocation failed */
    TSV_ESTATE = 6       /* call order violated (e.g. solve before set_layout) */
} tsv_status;

typedef enum { /* linalg::Precond, linalg.hpp:117 */
    TSV_PRECOND_NONE = 0,
    TSV_PRECOND_DIAGONAL = 1,
    TSV_PRECOND_BLOCK_DIAGONAL = 2,
    TSV_PRECOND_SCHWARZ2 = 3    /* new: two-level additive Schwarz (per-block local solves + super-block coarse space) */
} tsv_precond;

typedef enum { TSV_KIND_TSV = 0, TSV_KIND_DUMMY = 1 } tsv_block_kind; /* BlockKind, mesh.hpp:43 */

typedef enum { /* recovery points per element (new; the reference only samples a cut plane) */
    TSV_POINTS_CENTROID = 1,
    TSV_POINTS_GAUSS8 = 8
} tsv_points;

typedef enum { /* boundary conditions of the reduced system */
    TSV_BC_BOTTOM_PIN = 0,      /* configs, literal: u_z = 0 on gz = 0, corner (0,0,0) pinned */
    TSV_BC_BOTTOM_PIN_321 = 1,  /* + u_y = 0 at lattice (lat_x-1, 0, 0) (3-2-1 rule, SPD) */
    TSV_BC_CLAMPED = 2,         /* GlobalBC::clamped(), global_stage.cpp:159-163 */
    TSV_BC_NONE = 3
} tsv_bc_kind;

/* One reduced-order model (rom::ReducedOrderModel, rom.hpp:57-72) plus the
 * unit-block mesh data recovery needs (BlockMeshes, global.hpp:113-119).
 * Arrays are read during tsv_set_rom only. */
typedef struct {
    uint32_t q[3];                   /* NodeLayout n_x, n_y, n_z (rom.hpp:18-31) */
    double geometry[4];              /* UnitBlockGeometry d, h, t, p (mesh.hpp:17-24) */
    uint32_t grid_len[3];            /* TensorGrid line counts (mesh.hpp:28-41) */
    const double *grid[3];           /* TensorGrid x, y, z lines */
    double materials[3][3];          /* MaterialTable: E, nu, alpha per MaterialId (material.hpp:17-47) */
    const uint8_t *element_material; /* cells MaterialId (mesh.cpp:182-190); NULL = rebuild from geometry */
    const double *a_element;         /* K_r: n*n row-major */
    const double *b_element;         /* n, for dT = 1 */
    const double *basis;             /* Phi: n_fine*n row-major (rom.hpp:53-56) */
    const double *thermal;           /* u_T: n_fine, for dT = 1 */
    uint8_t fingerprint[32];         /* rom_fingerprint (rom.cpp:110-132); checked like RomSet::check_consistency */
} tsv_rom_desc;

typedef struct { /* linalg::IterOptions, linalg.hpp:120-129 (method fixed to CG) */
    double tolerance;
    int max_iterations;
    int precond;
} tsv_iter_options;

typedef struct { /* GlobalSolution (global.hpp:91-96) + device timings */
    int iterations;
    double relative_residual;
    int direct_fallback;      /* always 0: no CPU fallback on the GPU path */
    int best_iterations;      /* on TSV_ENOCONV: iteration of the returned best iterate */
    double solve_ms;          /* device time of the solve, CUDA events on the context stream */
    double loop_ms;           /* of which the iteration loop (excludes the best-iterate replay) */
    int restarts;             /* true-residual verifications that failed and restarted CG (linalg.cpp:321-330) */
    int replacements;         /* Schwarz loop: mid-solve residual replacements (r := b - A x, direction kept); 0 or 1 */
    uint64_t kernel_launches; /* kernels launched by this call */
} tsv_solve_info;

typedef struct { /* device-side timings of the last calls (CUDA events, context stream) */
    double solve_ms, recover_ms;
    double apply_ms_avg;      /* mean K1 (operator apply) launch in the last tsv_profile_apply */
    uint64_t kernel_launches; /* cumulative since tsv_ctx_create */
    double stress_ms;         /* sum of the K7 (stress kernel) launch times of the last recovery, CUDA events */
    int stress_launches;      /* K7 launches of the last recovery */
    int reserved_;
} tsv_timing;

/* Context. */
int tsv_ctx_create(int device, tsv_ctx **out);
void tsv_ctx_destroy(tsv_ctx *ctx);
const char *tsv_last_error(const tsv_ctx *ctx);
int tsv_abi_version(void);

/* RomSet slot `kind` (global.hpp:36-43): upload K_r, b_el, Phi, u_T and the
 * element materials to HBM. */
int tsv_set_rom(tsv_ctx *ctx, int kind, const tsv_rom_desc *rom);

/* The reference's ".rom" files (MRST v1, rom.cpp:257-377) straight into a
 * RomSet slot: magic/version/kind checks, SHA-256 header fingerprint,
 * length validation, column-major basis. slot < 0 uses the file's kind. */
int tsv_load_rom_file(tsv_ctx *ctx, int slot, const char *path, int *kind_out, char *err, size_t err_len);
/* save_rom (rom.cpp:262-303) of a ROM given as a descriptor. */
int tsv_save_rom_file(const tsv_rom_desc *rom, int kind, const char *path, char *err, size_t err_len);

/* ArrayLayout (global.hpp:16-32) + RomSet::check_consistency (:52-80) +
 * index_global_nodes (global_stage.cpp:94-119): builds the global index,
 * the B x n dof map and the device-side gather/scatter tables. kinds may be
 * NULL (all TSV); delta_t has 1 or rows*cols entries. */
int tsv_set_layout(tsv_ctx *ctx, uint32_t rows, uint32_t cols, const uint8_t *kinds,
                   const double *delta_t, size_t n_delta_t, double pitch, double height);

/* Online update of the per-block temperature change only (ArrayLayout::
 * delta_t, global.hpp:16-32; the thermal load b[dof] += dT_b b_el[a],
 * global_stage.cpp:135-142, and the recovery's dT_b u_T term,
 * global_stage.cpp:215-230). Keeps the index, dof map, Dirichlet set and
 * the preconditioner (which depends on kinds and BCs only); the load is
 * re-assembled on the device by the next solve. 1 or rows*cols entries. */
int tsv_set_delta_t(tsv_ctx *ctx, const double *delta_t, size_t n_delta_t);

/* Dirichlet data: a fem::DirichletSet (fem.hpp:22-36) given as sorted or
 * unsorted (dof, value) pairs, or one of the tsv_bc_kind sets. Lifting
 * follows apply_dirichlet_lifting (fem.cpp:223-260). */
int tsv_set_dirichlet(tsv_ctx *ctx, size_t count, const uint32_t *dofs, const double *values);
int tsv_set_bc(tsv_ctx *ctx, int bc_kind);

/* Host-only (no GPU, no context): index_global_nodes + global_dof for a
 * rows x cols array with NodeLayout q[3]. Any output may be NULL; sizes:
 * node_of_lattice lat_x*lat_y*lat_z, lattice_of_node [nodes][3], dof_map
 * rows*cols*n. Returns TSV_OK / TSV_EINVAL. */
int tsv_index_global_nodes(uint32_t rows, uint32_t cols, const uint32_t q[3], uint64_t *n_dofs,
                           uint32_t lattice[3], int32_t *node_of_lattice, uint32_t *lattice_of_node,
                           uint32_t *dof_map);

/* Introspection of GlobalIndex (global.hpp:47-62) for bit-exact checks. */
int tsv_get_index(tsv_ctx *ctx, uint64_t *n_dofs, uint64_t *n_nodes, uint32_t lattice[3], uint32_t *n_reduced);
int tsv_get_dof_map(tsv_ctx *ctx, uint32_t *dof_map /* B*n */);
int tsv_get_lattice(tsv_ctx *ctx, int32_t *node_of_lattice, uint32_t *lattice_of_node /* [nodes][3] */);
int tsv_get_constrained(tsv_ctx *ctx, uint8_t *mask /* N */);
int tsv_get_load(tsv_ctx *ctx, double *b /* N, lifted */);

/* y = A_lifted x (CsrMatrix::apply on the lifted assembled matrix,
 * linalg.cpp:74-86), matrix-free on the GPU. Host buffers. */
int tsv_apply(tsv_ctx *ctx, const double *x, double *y);

/* solve_global (global_stage.cpp:187-205) -> cg_solve (linalg.cpp:292-362)
 * on the GPU. u_out (N doubles, host) may be NULL: the solution stays
 * resident for tsv_recover*. On TSV_ENOCONV u_out holds the best iterate. */
int tsv_solve(tsv_ctx *ctx, const tsv_iter_options *opts, double *u_out, tsv_solve_info *info);

/* z = M^-1 r for the two-level Schwarz preconditioner (test hook). */
int tsv_precond_apply(tsv_ctx *ctx, int precond, const double *r, double *z);
typedef struct { /* preconditioner set-up of the current layout */
    double setup_ms;   /* host wall time of the build (0 when it was already built) */
    int ntypes;        /* Schwarz: block neighbourhood types (local inverses) */
    int coarse_dofs;   /* Schwarz: coarse-space size Nc */
    int super_block;   /* Schwarz: super-block side s (blocks) */
    int local_rows;    /* Schwarz: type-padded rows of the local-solve panel */
} tsv_precond_info;
/* Build the preconditioner for the current layout now (tsv_solve builds it
 * on first use) and describe it. No reference counterpart: the reference
 * builds its Jacobi/block preconditioners inside cg_solve (linalg.cpp:221-290). */
int tsv_precond_setup(tsv_ctx *ctx, int precond, tsv_precond_info *out);
/* Test hook: coarse-level vectors of the last tsv_precond_apply and A_c^-1 (any may be NULL). */
int tsv_debug_coarse(tsv_ctx *ctx, int *nc, double *rc, double *zc, double *ainv_c);

/* Make u (N doubles, host) the resident solution (recovery from given data). */
int tsv_set_solution(tsv_ctx *ctx, const double *u);

/* Per-block recovery: gather_cell_values + reconstruct_block_field
 * (global_stage.cpp:207-230) + evaluate_stress_in_element + von_mises
 * (fem.cpp:262-316) at `points` per element, for original cells
 * [cell_begin, cell_end). out[((c*E + e)*P + g)*7 + k], c relative to
 * cell_begin, e = cell_id (mesh.cpp:125-127), g in (gx,gy,gz) order with gz
 * fastest, k = xx,yy,zz,xy,yz,zx,vm. Host output. */
int tsv_recover(tsv_ctx *ctx, int points, uint64_t cell_begin, uint64_t cell_end, double *out);

/* Recover the whole array into context-owned HBM (no host copy) and read
 * back any cell range of it. */
int tsv_recover_resident(tsv_ctx *ctx, int points);
int tsv_copy_stress(tsv_ctx *ctx, uint64_t cell_begin, uint64_t cell_end, double *out);

/* cutplane_von_mises (global_stage.cpp:245-274): von Mises at res x res
 * cell-centred samples of z = h/2 in every block, the containing element
 * chosen with locate_axis_cell's lower-cell tie rule (mesh.cpp:97-104).
 * out = StressGrid::values, [((row*cols + col)*res + py)*res + px]. */
int tsv_cutplane(tsv_ctx *ctx, uint32_t res, double *out);

/* Reconstructed fine displacement of one cell (reconstruct_block_field). */
int tsv_block_field(tsv_ctx *ctx, uint64_t cell, double *out /* n_fine */);

/* One-shot local stage (rom::build_rom, rom.cpp:134-253) on the GPU: the
 * reduced-order model of one unit block, i.e. the INPUT of the online
 * stage, timed separately. Outputs are caller-allocated (sizes from
 * tsv_rom_dims); any array pointer may be NULL. */
typedef struct {
    uint32_t q[3];          /* NodeLayout n_x, n_y, n_z */
    double geometry[4];     /* d, h, t, p */
    uint32_t grid_len[3];
    const double *grid[3];  /* TensorGrid lines spanning [0,p]x[0,p]x[0,h] */
    double materials[3][3]; /* E, nu, alpha per MaterialId */
    int kind;               /* 0 tsv (materials by centroid radius), 1 dummy (all silicon) */
} tsv_local_desc;

typedef struct {
    double *a_element;          /* n*n row-major */
    double *b_element;          /* n */
    double *basis;              /* n_fine*n row-major */
    double *thermal;            /* n_fine */
    uint8_t *element_material;  /* cells */
    uint8_t fingerprint[32];    /* rom_fingerprint (rom.cpp:110-132) */
    double build_ms;
} tsv_rom_out;

int tsv_rom_dims(const tsv_local_desc *desc, uint64_t *n, uint64_t *n_fine, uint64_t *cells);
/* rom_fingerprint (rom.cpp:110-132) of a configuration (host only), and the
 * kind + stored fingerprint of a .rom file (header checked like load_rom):
 * what cmd_solve's "ROM ... was built for a different configuration" check
 * (cli.cpp:38-44) compares. */
int tsv_rom_fingerprint(const tsv_local_desc *desc, uint8_t fingerprint[32]);
int tsv_rom_file_info(const char *path, int *kind, uint8_t fingerprint[32], char *err, size_t err_len);
int tsv_build_rom(int device, const tsv_local_desc *desc, tsv_rom_out *out, char *err, size_t err_len);

/* Page-lock a host buffer so tsv_recover / tsv_solve copies run at full
 * PCIe/C2C rate (cudaHostRegister); unregister before freeing it. */
int tsv_host_register(void *ptr, size_t bytes);
int tsv_host_unregister(void *ptr);
/* Allocate / free page-locked host memory for results (cudaHostAlloc):
 * device-to-host copies into it run ~10% faster than into registered
 * pageable memory on this platform (57 vs 51 GB/s). */
int tsv_host_alloc(size_t bytes, void **ptr);
int tsv_host_free(void *ptr);

/* FP64 roofline denominators measured live on `device`: register-only
 * DMMA.8x8x4 (mma.sync f64) and DFMA issue loops over all SMs. */
int tsv_fp64_peak(int device, double *dmma_tflops, double *dfma_tflops);

/* Measurement hooks: time `reps` K1 launches alone; read timings. */
int tsv_profile_apply(tsv_ctx *ctx, int reps, double *ms_per_launch);
int tsv_get_timing(tsv_ctx *ctx, tsv_timing *out);

/* Mirror symmetry of the loaded ROMs (csrc/symmetry.hpp). A macro-element
 * whose grid and materials are symmetric about its three mid-planes has
 * K_r and Phi block diagonal over the 8 irreps of Z2^3; tsv_set_rom checks
 * that numerically and the layout then runs K1 / K6 as 8 irrep products
 * with 1/8 of the FP64 FLOPs. K1 is one fused kernel (rows of the operand
 * panel in shared memory, butterflies in place, the irrep blocks on the DMMA
 * pipe); inside the PCG loop the A x of the true-residual check stays on the
 * reference's K_r (exact int8 product), so the returned solution satisfies
 * the reference's stopping rule for the reference's operator.
 * TSV_SYM=0 disables the path; TSV_SYM_K1_FUSED=0 selects the multi-kernel
 * K1 (panel passes + segmented GEMM + TF32 term for K_r - K_sym). */
typedef struct tsv_symmetry_info {
    int recovery_symmetric;   /* K6 on the irrep path for this layout */
    int operator_symmetric;   /* K1 on the irrep path for this layout */
    int defect_correction;    /* K_r - K_sym carried as a TF32 term */
    int irrep_dofs[8];        /* reduced DoFs per irrep */
    double defect_k[2];       /* per kind: max off-block |K''| / max |K''| */
    double defect_phi[2];
    int operator_fused;       /* K1 irrep path as one fused kernel */
    int reserved_;
} tsv_symmetry_info;
int tsv_get_symmetry(tsv_ctx *ctx, tsv_symmetry_info *out);

#ifdef __cplusplus
}
#endif
#endif /* TSV_B200_H */
