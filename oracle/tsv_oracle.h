/* ORACLE TEST INFRASTRUCTURE — not product code.
 *
 * Plain-C restatement of the reference's online-stage hot path
 * (tsvstress, /root/reference/proj), used as the CPU checker for the GPU
 * path and as the "port" CPU baseline. It is matrix-free (no CSR), so it
 * also runs at configs 3/4 where the reference's CSR assembly needs
 * ~100-120 GB of host RAM. It is pinned against the
 * reference itself (oracle/_ref, built from the unmodified sources) on
 * configs 0-2 by tests/test_oracle_pin.py.
 *
 * Every function cites the reference code it restates.
 */
#ifndef TSV_ORACLE_H
#define TSV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* NodeLayout::create surface-node enumeration, rom.cpp:12-33:
 * i (x) outer, j, k (z) inner, skipping strictly interior points.
 * out: [count][3]; returns count (call with out = NULL to size). */
size_t orc_surface_nodes(uint32_t nx, uint32_t ny, uint32_t nz, uint32_t *out);

/* index_global_nodes, global_stage.cpp:94-119. node_of_lattice has
 * lat_x*lat_y*lat_z entries (-1 = none); lattice_of_node [count][3].
 * Returns the node count. */
size_t orc_index_global_nodes(uint32_t rows, uint32_t cols, uint32_t nx, uint32_t ny, uint32_t nz,
                              int32_t *node_of_lattice, uint32_t *lattice_of_node);

/* dof_map[b*n + a] = GlobalIndex::global_dof (global_stage.cpp:82-92). */
void orc_dof_map(uint32_t rows, uint32_t cols, uint32_t nx, uint32_t ny, uint32_t nz,
                 const int32_t *node_of_lattice, uint32_t *dof_map);

/* Dirichlet mask for the configs' boundary conditions (new; the reference
 * receives it as a fem::DirichletSet, fem.cpp:62-80):
 * mode 0 literal: u_z on every gz = 0 node + corner (0,0,0) xyz;
 * mode 1 3-2-1: mode 0 + u_y at lattice (lat_x-1, 0, 0);
 * mode 2 clamped top/bottom (reduced_dirichlet, global_stage.cpp:154-163);
 * mode 3 none. Values are zero in all modes. Returns #constrained. */
size_t orc_bc_mask(int mode, size_t node_count, const uint32_t *lattice_of_node, uint32_t lat_x,
                   uint32_t lat_z, uint8_t *constrained);

/* The lifted reduced system, matrix-free. kinds[b] selects K/b_el/Phi/u_T
 * of model 0 (tsv) or 1 (dummy). */
typedef struct {
    size_t B, n, N;
    const uint32_t *dof_map;     /* [B][n] */
    const uint8_t *kinds;        /* [B] or NULL (all kind 0) */
    const double *delta_t;       /* [B] */
    const double *K[2];          /* n*n row-major (a_element) */
    const double *b_el[2];       /* n */
    const uint8_t *constrained;  /* [N] */
    const double *g;             /* [N] prescribed values (may be NULL = 0) */
    int threads;
} orc_system;

/* y = A_lifted x, restating CsrMatrix::apply (linalg.cpp:74-86) on the
 * matrix assemble_global (global_stage.cpp:121-145) + apply_dirichlet_lifting
 * (fem.cpp:223-260) would build: y = Mf∘(Σ_b G_bᵀ K_b G_b (Mf∘x)) + Mc∘x.
 * Blocks are scattered in 4 colours (row%2, col%2) so threads never
 * collide; results are independent of the thread count. */
void orc_apply(const orc_system *s, uint32_t rows, uint32_t cols, const double *x, double *y);

/* Lifted load vector: b[dof] += ΔT_b b_el[a] in cell/a order
 * (global_stage.cpp:141), then b_f -= A_fc g, b_c = g (fem.cpp:250-258). */
void orc_rhs(const orc_system *s, uint32_t rows, uint32_t cols, double *b);

/* Diagonal of the lifted matrix, summed in cell order as csr_from_triplets
 * sums duplicates in stable input order (linalg.cpp:35-72); 1 on
 * constrained rows (fem.cpp:240-247). */
void orc_lifted_diagonal(const orc_system *s, double *diag);

/* 3x3 node blocks of the lifted matrix (BlockDiagonal preconditioner input,
 * linalg.cpp:231-237): blocks[node][9]. */
void orc_lifted_node_blocks(const orc_system *s, double *blocks);

enum { ORC_OK = 0, ORC_ENOCONV = 2, ORC_EBREAKDOWN = 3, ORC_EINVAL = 1 };

/* cg_solve (linalg.cpp:292-362) with Preconditioner (:221-290):
 * precond 0 none, 1 diagonal, 2 block-diagonal. x0 = 0. On ENOCONV x holds
 * the best iterate and iterations and relres describe it (linalg.cpp:354-360).
 * max_iterations: cap; tol: relative residual. */
int orc_cg_solve(const orc_system *s, uint32_t rows, uint32_t cols, const double *b, double tol,
                 int max_iterations, int precond, double *x, int *iterations, double *relres);

/* cg_solve (linalg.cpp:292-362) with a caller-supplied preconditioner
 * z = M^-1 r (fixed, SPD): the same control flow as orc_cg_solve. Used by
 * the FP64 two-level Schwarz oracle (oracle/schwarz64.py), which gives the
 * configs 3/4 an independent CPU solution in minutes instead of the
 * ~21k Jacobi iterations the reference's own preconditioner needs. */
typedef void (*orc_pc_fn)(void *ctx, const double *r, double *z);
int orc_cg_solve_pc(const orc_system *s, uint32_t rows, uint32_t cols, const double *b, double tol,
                    int max_iterations, orc_pc_fn pc, void *pc_ctx, int exact_residual, double *x,
                    int *iterations, double *relres);

/* r = b - A_lifted x with long-double products and sums, rounded once
 * (the true-residual check of orc_cg_solve_pc when exact_residual != 0). */
void orc_residual_ld(const orc_system *s, uint32_t rows, uint32_t cols, const double *b, const double *x,
                     double *r);

/* Per-block recovery: gather_cell_values (global_stage.cpp:207-213) +
 * reconstruct_block_field (:215-230, sequential i) + evaluate_stress_in_element
 * (fem.cpp:262-301) + von_mises (:311-316) at 8 Gauss points (points = 8,
 * (gx,gy,gz) order gz fastest, natural coords -+1/sqrt(3), fem.cpp:87-92) or
 * the centroid (points = 1). Box elements on tensor grid lines gx/gy/gz,
 * element ids (k*cy + j)*cx + i (mesh.cpp:125-127), corner order
 * mesh.cpp:171-176, element_material[kind][e] -> (lambda, mu, alpha) from
 * mat[kind][3][3]. out[((cb*E + e)*points + g)*7 + c]. */
typedef struct {
    size_t n_fine;
    uint32_t cx, cy, cz;
    const double *gx[2], *gy[2], *gz[2];
    const double *Phi[2];       /* [n_fine][n] row-major */
    const double *u_T[2];       /* [n_fine] */
    const uint8_t *elem_mat[2]; /* [E] */
    double lame[2][3][3];       /* [kind][material][lambda, mu, alpha] */
} orc_recovery;

void orc_recover(const orc_system *s, const orc_recovery *r, const double *u, int points,
                 size_t cell_begin, size_t cell_end, double *out);

#ifdef __cplusplus
}
#endif
#endif
