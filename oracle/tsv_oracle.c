/* ORACLE TEST INFRASTRUCTURE — not product code. See tsv_oracle.h.
 * Restates the reference's hot path (tsvstress) in plain C, function by
 * function; the reference file:line is cited at each definition. */
#include "tsv_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ threading */
/* Static contiguous partition, as parallel_for_ranges (core.cpp:24-43). */
typedef void (*orc_range_fn)(void *ctx, size_t begin, size_t end);
typedef struct {
    orc_range_fn fn;
    void *ctx;
    size_t begin, end;
} orc_task;

static void *orc_task_main(void *p) {
    orc_task *t = (orc_task *)p;
    t->fn(t->ctx, t->begin, t->end);
    return NULL;
}

static void orc_parallel(size_t n, int threads, orc_range_fn fn, void *ctx) {
    if (n == 0) return;
    size_t nt = threads < 1 ? 1 : (size_t)threads;
    if (nt > n) nt = n;
    if (nt == 1) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t *th = malloc(nt * sizeof(pthread_t));
    orc_task *tasks = malloc(nt * sizeof(orc_task));
    size_t chunk = (n + nt - 1) / nt, used = 0;
    for (size_t t = 0; t < nt; ++t) {
        size_t b = t * chunk, e = b + chunk < n ? b + chunk : n;
        if (b >= e) break;
        tasks[t] = (orc_task){fn, ctx, b, e};
        pthread_create(&th[t], NULL, orc_task_main, &tasks[t]);
        ++used;
    }
    for (size_t t = 0; t < used; ++t) pthread_join(th[t], NULL);
    free(th);
    free(tasks);
}

/* ------------------------------------------------------------- indexing */
size_t orc_surface_nodes(uint32_t nx, uint32_t ny, uint32_t nz, uint32_t *out) {
    /* rom.cpp:26-31 */
    size_t count = 0;
    for (uint32_t i = 0; i < nx; ++i)
        for (uint32_t j = 0; j < ny; ++j)
            for (uint32_t k = 0; k < nz; ++k) {
                int interior = i > 0 && i < nx - 1 && j > 0 && j < ny - 1 && k > 0 && k < nz - 1;
                if (interior) continue;
                if (out) {
                    out[3 * count + 0] = i;
                    out[3 * count + 1] = j;
                    out[3 * count + 2] = k;
                }
                ++count;
            }
    return count;
}

size_t orc_index_global_nodes(uint32_t rows, uint32_t cols, uint32_t nx, uint32_t ny, uint32_t nz,
                              int32_t *node_of_lattice, uint32_t *lattice_of_node) {
    /* global_stage.cpp:94-119 */
    uint32_t lat_x = cols * (nx - 1) + 1, lat_y = rows * (ny - 1) + 1, lat_z = nz;
    size_t count = 0;
    for (uint32_t gz = 0; gz < lat_z; ++gz)
        for (uint32_t gy = 0; gy < lat_y; ++gy)
            for (uint32_t gx = 0; gx < lat_x; ++gx) {
                size_t slot = ((size_t)gz * lat_y + gy) * lat_x + gx;
                int x_int = (gx % (nx - 1)) != 0;
                int y_int = (gy % (ny - 1)) != 0;
                int z_int = gz > 0 && gz < lat_z - 1;
                if (x_int && y_int && z_int) {
                    if (node_of_lattice) node_of_lattice[slot] = -1;
                    continue;
                }
                if (node_of_lattice) node_of_lattice[slot] = (int32_t)count;
                if (lattice_of_node) {
                    lattice_of_node[3 * count + 0] = gx;
                    lattice_of_node[3 * count + 1] = gy;
                    lattice_of_node[3 * count + 2] = gz;
                }
                ++count;
            }
    return count;
}

void orc_dof_map(uint32_t rows, uint32_t cols, uint32_t nx, uint32_t ny, uint32_t nz,
                 const int32_t *node_of_lattice, uint32_t *dof_map) {
    /* GlobalIndex::global_dof, global_stage.cpp:82-92 */
    size_t nn = orc_surface_nodes(nx, ny, nz, NULL);
    uint32_t *sn = malloc(nn * 3 * sizeof(uint32_t));
    orc_surface_nodes(nx, ny, nz, sn);
    uint32_t lat_x = cols * (nx - 1) + 1, lat_y = rows * (ny - 1) + 1;
    size_t n = 3 * nn;
    for (uint32_t r = 0; r < rows; ++r)
        for (uint32_t c = 0; c < cols; ++c) {
            size_t b = (size_t)r * cols + c;
            for (size_t a = 0; a < n; ++a) {
                size_t rank = a / 3;
                uint32_t comp = (uint32_t)(a % 3);
                uint32_t gx = c * (nx - 1) + sn[3 * rank + 0];
                uint32_t gy = r * (ny - 1) + sn[3 * rank + 1];
                uint32_t gz = sn[3 * rank + 2];
                int32_t id = node_of_lattice[((size_t)gz * lat_y + gy) * lat_x + gx];
                dof_map[b * n + a] = (uint32_t)id * 3u + comp;
            }
        }
    free(sn);
}

size_t orc_bc_mask(int mode, size_t node_count, const uint32_t *lat, uint32_t lat_x, uint32_t lat_z,
                   uint8_t *constrained) {
    memset(constrained, 0, node_count * 3);
    size_t count = 0;
    for (size_t id = 0; id < node_count; ++id) {
        uint32_t gx = lat[3 * id], gy = lat[3 * id + 1], gz = lat[3 * id + 2];
        if (mode == 2) { /* reduced_dirichlet ClampedTopBottom, global_stage.cpp:159-163 */
            if (gz == 0 || gz == lat_z - 1)
                for (int c = 0; c < 3; ++c) constrained[3 * id + c] = 1;
        } else if (mode == 0 || mode == 1) {
            if (gz != 0) continue;
            constrained[3 * id + 2] = 1;
            if (gx == 0 && gy == 0) constrained[3 * id] = constrained[3 * id + 1] = 1;
            if (mode == 1 && gx == lat_x - 1 && gy == 0) constrained[3 * id + 1] = 1;
        }
    }
    for (size_t i = 0; i < node_count * 3; ++i) count += constrained[i];
    return count;
}

/* --------------------------------------------------------------- apply */
static inline double orc_dot(const double *a, const double *b, size_t n) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    size_t k = 0;
    for (; k + 4 <= n; k += 4) {
        s0 += a[k] * b[k];
        s1 += a[k + 1] * b[k + 1];
        s2 += a[k + 2] * b[k + 2];
        s3 += a[k + 3] * b[k + 3];
    }
    for (; k < n; ++k) s0 += a[k] * b[k];
    return (s0 + s1) + (s2 + s3);
}

typedef struct {
    const orc_system *s;
    const size_t *blocks; /* block ids of the current colour */
    const double *x;
    double *y;
    int mask_out; /* 1: free rows only (apply); 0: all */
} orc_apply_ctx;

static void orc_apply_range(void *p, size_t begin, size_t end) {
    orc_apply_ctx *c = (orc_apply_ctx *)p;
    const orc_system *s = c->s;
    const size_t n = s->n;
    double *xb = malloc(n * sizeof(double));
    for (size_t t = begin; t < end; ++t) {
        size_t b = c->blocks[t];
        const uint32_t *dm = s->dof_map + b * n;
        int kind = s->kinds ? s->kinds[b] : 0;
        const double *K = s->K[kind];
        for (size_t a = 0; a < n; ++a) xb[a] = s->constrained[dm[a]] ? 0.0 : c->x[dm[a]];
        for (size_t a = 0; a < n; ++a) {
            if (c->mask_out && s->constrained[dm[a]]) continue;
            c->y[dm[a]] += orc_dot(K + a * n, xb, n);
        }
    }
    free(xb);
}

/* Σ_b G_bᵀ K_b G_b (Mf∘x) restricted to free rows, coloured scatter. */
static void orc_block_sum(const orc_system *s, uint32_t rows, uint32_t cols, const double *x, double *y) {
    size_t *blocks = malloc(s->B * sizeof(size_t));
    for (int colour = 0; colour < 4; ++colour) {
        size_t nb = 0;
        for (uint32_t r = (uint32_t)(colour >> 1); r < rows; r += 2)
            for (uint32_t c = (uint32_t)(colour & 1); c < cols; c += 2) blocks[nb++] = (size_t)r * cols + c;
        orc_apply_ctx ctx = {s, blocks, x, y, 1};
        orc_parallel(nb, s->threads, orc_apply_range, &ctx);
    }
    free(blocks);
}

void orc_apply(const orc_system *s, uint32_t rows, uint32_t cols, const double *x, double *y) {
    memset(y, 0, s->N * sizeof(double));
    orc_block_sum(s, rows, cols, x, y);
    for (size_t i = 0; i < s->N; ++i)
        if (s->constrained[i]) y[i] = x[i]; /* unit row, fem.cpp:240-245 */
}

/* r = b - A x with the block products and the sums in long double (x87,
 * 64-bit mantissa), rounded once at the end. Only the oracle's
 * true-residual check uses it (orc_cg_solve_pc with exact_residual): at
 * configs 3/4 the FP64 rounding of A x alone is ~1e-12 relative to |b|,
 * the solver tolerance, so an FP64 check restarts forever. */
typedef struct {
    const orc_system *s;
    const size_t *blocks;
    const double *x;
    long double *y;
} orc_apply_ld_ctx;

static void orc_apply_ld_range(void *p, size_t begin, size_t end) {
    orc_apply_ld_ctx *c = (orc_apply_ld_ctx *)p;
    const orc_system *s = c->s;
    const size_t n = s->n;
    double *xb = malloc(n * sizeof(double));
    for (size_t t = begin; t < end; ++t) {
        size_t b = c->blocks[t];
        const uint32_t *dm = s->dof_map + b * n;
        const double *K = s->K[s->kinds ? s->kinds[b] : 0];
        for (size_t a = 0; a < n; ++a) xb[a] = s->constrained[dm[a]] ? 0.0 : c->x[dm[a]];
        for (size_t a = 0; a < n; ++a) {
            if (s->constrained[dm[a]]) continue;
            const double *row = K + a * n;
            long double acc = 0.0L;
            for (size_t k = 0; k < n; ++k) acc += (long double)row[k] * (long double)xb[k];
            c->y[dm[a]] += acc;
        }
    }
    free(xb);
}

void orc_residual_ld(const orc_system *s, uint32_t rows, uint32_t cols, const double *b, const double *x,
                     double *r) {
    long double *y = calloc(s->N, sizeof(long double));
    size_t *blocks = malloc(s->B * sizeof(size_t));
    for (int colour = 0; colour < 4; ++colour) {
        size_t nb = 0;
        for (uint32_t rr = (uint32_t)(colour >> 1); rr < rows; rr += 2)
            for (uint32_t cc = (uint32_t)(colour & 1); cc < cols; cc += 2) blocks[nb++] = (size_t)rr * cols + cc;
        orc_apply_ld_ctx ctx = {s, blocks, x, y};
        orc_parallel(nb, s->threads, orc_apply_ld_range, &ctx);
    }
    for (size_t i = 0; i < s->N; ++i)
        r[i] = s->constrained[i] ? b[i] - x[i] : (double)((long double)b[i] - y[i]);
    free(blocks);
    free(y);
}

void orc_rhs(const orc_system *s, uint32_t rows, uint32_t cols, double *b) {
    (void)rows;
    (void)cols;
    memset(b, 0, s->N * sizeof(double));
    for (size_t blk = 0; blk < s->B; ++blk) { /* global_stage.cpp:135-142 */
        int kind = s->kinds ? s->kinds[blk] : 0;
        double dt = s->delta_t[blk];
        const uint32_t *dm = s->dof_map + blk * s->n;
        for (size_t a = 0; a < s->n; ++a) b[dm[a]] += dt * s->b_el[kind][a];
    }
    if (s->g) { /* b_f -= A_fc g, fem.cpp:250-256 */
        double *gc = calloc(s->N, sizeof(double));
        double *t = calloc(s->N, sizeof(double));
        for (size_t i = 0; i < s->N; ++i) gc[i] = s->constrained[i] ? s->g[i] : 0.0;
        /* A_fc g: constrained columns scattered into free rows */
        for (size_t blk = 0; blk < s->B; ++blk) {
            int kind = s->kinds ? s->kinds[blk] : 0;
            const double *K = s->K[kind];
            const uint32_t *dm = s->dof_map + blk * s->n;
            for (size_t a = 0; a < s->n; ++a) {
                if (s->constrained[dm[a]]) continue;
                double acc = 0.0;
                for (size_t q = 0; q < s->n; ++q) acc += K[a * s->n + q] * gc[dm[q]];
                t[dm[a]] += acc;
            }
        }
        for (size_t i = 0; i < s->N; ++i) b[i] = s->constrained[i] ? s->g[i] : b[i] - t[i];
        free(gc);
        free(t);
    } else {
        for (size_t i = 0; i < s->N; ++i)
            if (s->constrained[i]) b[i] = 0.0; /* b_c = g = 0, fem.cpp:247 */
    }
}

void orc_lifted_diagonal(const orc_system *s, double *diag) {
    memset(diag, 0, s->N * sizeof(double));
    for (size_t blk = 0; blk < s->B; ++blk) {
        int kind = s->kinds ? s->kinds[blk] : 0;
        const double *K = s->K[kind];
        const uint32_t *dm = s->dof_map + blk * s->n;
        for (size_t a = 0; a < s->n; ++a) diag[dm[a]] += K[a * s->n + a];
    }
    for (size_t i = 0; i < s->N; ++i)
        if (s->constrained[i]) diag[i] = 1.0;
}

void orc_lifted_node_blocks(const orc_system *s, double *blocks) {
    size_t nodes = s->N / 3;
    memset(blocks, 0, nodes * 9 * sizeof(double));
    for (size_t blk = 0; blk < s->B; ++blk) {
        int kind = s->kinds ? s->kinds[blk] : 0;
        const double *K = s->K[kind];
        const uint32_t *dm = s->dof_map + blk * s->n;
        for (size_t rank = 0; rank < s->n / 3; ++rank) {
            size_t node = dm[3 * rank] / 3;
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                    blocks[node * 9 + r * 3 + c] += K[(3 * rank + r) * s->n + 3 * rank + c];
        }
    }
    for (size_t node = 0; node < nodes; ++node)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                int cr = s->constrained[3 * node + r], cc = s->constrained[3 * node + c];
                if (cr) blocks[node * 9 + r * 3 + c] = (r == c) ? 1.0 : 0.0;
                else if (cc) blocks[node * 9 + r * 3 + c] = 0.0;
            }
}

/* ------------------------------------------------------------------ CG */
static double orc_sdot(const double *a, const double *b, size_t n) { /* linalg.cpp:205-209, serial */
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

typedef struct {
    int kind;
    size_t n;
    double *inv_diag;
    double *blocks;
} orc_precond;

static void orc_precond_init(orc_precond *p, const orc_system *s, int kind) {
    /* Preconditioner ctor, linalg.cpp:223-262 */
    p->kind = kind;
    p->n = s->N;
    p->inv_diag = NULL;
    p->blocks = NULL;
    size_t n = s->N;
    if (kind == 1) {
        p->inv_diag = malloc(n * sizeof(double));
        orc_lifted_diagonal(s, p->inv_diag);
        for (size_t i = 0; i < n; ++i) {
            double d = p->inv_diag[i];
            p->inv_diag[i] = d != 0.0 ? 1.0 / d : 1.0;
        }
    } else if (kind == 2) {
        p->blocks = malloc(n / 3 * 9 * sizeof(double));
        double *m_all = malloc(n / 3 * 9 * sizeof(double));
        orc_lifted_node_blocks(s, m_all);
        for (size_t nb = 0; nb < n / 3; ++nb) {
            const double *m = m_all + nb * 9;
            double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                         m[2] * (m[3] * m[7] - m[4] * m[6]);
            double *inv = p->blocks + nb * 9;
            if (fabs(det) < 1e-300) {
                for (int i = 0; i < 9; ++i) inv[i] = 0.0;
                for (int i = 0; i < 3; ++i) {
                    double d = m[i * 3 + i];
                    inv[i * 3 + i] = d != 0.0 ? 1.0 / d : 1.0;
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
        }
        free(m_all);
    }
}

static void orc_precond_apply(const orc_precond *p, const double *r, double *z, size_t n) {
    /* linalg.cpp:265-284 */
    if (p->kind == 0) {
        memcpy(z, r, n * sizeof(double));
    } else if (p->kind == 1) {
        for (size_t i = 0; i < n; ++i) z[i] = p->inv_diag[i] * r[i];
    } else {
        for (size_t nb = 0; nb < n / 3; ++nb) {
            const double *m = p->blocks + nb * 9;
            const double *ri = r + nb * 3;
            double *zi = z + nb * 3;
            zi[0] = m[0] * ri[0] + m[1] * ri[1] + m[2] * ri[2];
            zi[1] = m[3] * ri[0] + m[4] * ri[1] + m[5] * ri[2];
            zi[2] = m[6] * ri[0] + m[7] * ri[1] + m[8] * ri[2];
        }
    }
}

static void orc_builtin_pc(void *ctx, const double *r, double *z) {
    const orc_precond *p = (const orc_precond *)ctx;
    orc_precond_apply(p, r, z, p->n);
}

static int orc_cg_core(const orc_system *s, uint32_t rows, uint32_t cols, const double *b, double tol,
                       int max_iterations, orc_pc_fn pc_fn, void *pc_ctx, int exact_residual, double *x,
                       int *iterations, double *relres);

int orc_cg_solve(const orc_system *s, uint32_t rows, uint32_t cols, const double *b, double tol,
                 int max_iterations, int precond, double *x, int *iterations, double *relres) {
    orc_precond pc;
    pc.kind = precond;
    pc.n = s->N;
    pc.inv_diag = NULL;
    pc.blocks = NULL;
    orc_precond_init(&pc, s, precond);
    int st = orc_cg_core(s, rows, cols, b, tol, max_iterations, orc_builtin_pc, &pc, 0, x, iterations, relres);
    free(pc.inv_diag);
    free(pc.blocks);
    return st;
}

int orc_cg_solve_pc(const orc_system *s, uint32_t rows, uint32_t cols, const double *b, double tol,
                    int max_iterations, orc_pc_fn pc, void *pc_ctx, int exact_residual, double *x, int *iterations,
                    double *relres) {
    return orc_cg_core(s, rows, cols, b, tol, max_iterations, pc, pc_ctx, exact_residual, x, iterations, relres);
}

static int orc_cg_core(const orc_system *s, uint32_t rows, uint32_t cols, const double *b, double tol,
                       int max_iterations, orc_pc_fn pc_fn, void *pc_ctx, int exact_residual, double *x,
                       int *iterations, double *relres) {
    /* cg_solve, linalg.cpp:292-362 */
    const size_t n = s->N;
    const double norm_b = sqrt(orc_sdot(b, b, n));
    memset(x, 0, n * sizeof(double));
    *iterations = 0;
    *relres = 0.0;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(b[i])) return ORC_EBREAKDOWN; /* check_finite, linalg.cpp:215-218 */
    if (norm_b == 0.0) return ORC_OK;

    double *r = malloc(n * sizeof(double)), *z = malloc(n * sizeof(double));
    double *p = malloc(n * sizeof(double)), *ap = malloc(n * sizeof(double));
    double *best_x = malloc(n * sizeof(double));
    int status = ORC_OK;

    orc_apply(s, rows, cols, x, r);
    for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    pc_fn(pc_ctx, r, z);
    memcpy(p, z, n * sizeof(double));
    double rho = orc_sdot(r, z, n);
    double res_norm = sqrt(orc_sdot(r, r, n));
    memcpy(best_x, x, n * sizeof(double));
    double best_res = res_norm;
    int it = 0;

    while (it < max_iterations) {
        if (res_norm <= tol * norm_b) {
            if (exact_residual) {
                orc_residual_ld(s, rows, cols, b, x, r);
            } else {
                orc_apply(s, rows, cols, x, r);
                for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
            }
            res_norm = sqrt(orc_sdot(r, r, n));
            if (res_norm <= tol * norm_b) break;
            pc_fn(pc_ctx, r, z);
            memcpy(p, z, n * sizeof(double));
            rho = orc_sdot(r, z, n);
        }
        orc_apply(s, rows, cols, p, ap);
        double pap = orc_sdot(p, ap, n);
        if (!isfinite(pap) || pap <= 0.0) {
            status = ORC_EBREAKDOWN;
            goto done;
        }
        double alpha = rho / pap;
        for (size_t i = 0; i < n; ++i) x[i] += alpha * p[i];
        for (size_t i = 0; i < n; ++i) r[i] -= alpha * ap[i];
        pc_fn(pc_ctx, r, z);
        double rho_next = orc_sdot(r, z, n);
        double beta = rho_next / rho;
        rho = rho_next;
        for (size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        res_norm = sqrt(orc_sdot(r, r, n));
        if (!isfinite(res_norm)) {
            status = ORC_EBREAKDOWN;
            goto done;
        }
        ++it;
        if (res_norm < best_res) {
            best_res = res_norm;
            memcpy(best_x, x, n * sizeof(double));
        }
    }
    *iterations = it;
    *relres = res_norm / norm_b;
    if (*relres > tol) {
        memcpy(x, best_x, n * sizeof(double));
        *relres = best_res / norm_b;
        status = ORC_ENOCONV;
    }
done:
    free(r); free(z); free(p); free(ap); free(best_x);
    return status;
}

/* ------------------------------------------------------------ recovery */
static const double kXi[8] = {-1, 1, 1, -1, -1, 1, 1, -1};   /* fem.cpp:11-13 */
static const double kEta[8] = {-1, -1, 1, 1, -1, -1, 1, 1};
static const double kZeta[8] = {-1, -1, -1, -1, 1, 1, 1, 1};

static void orc_physical_gradients(const double corners[8][3], double xi, double eta, double zeta,
                                   double grad[8][3]) {
    /* shape_gradients_natural fem.cpp:17-23 + physical_gradients :27-58 */
    double dn[8][3];
    for (int a = 0; a < 8; ++a) {
        dn[a][0] = 0.125 * kXi[a] * (1.0 + kEta[a] * eta) * (1.0 + kZeta[a] * zeta);
        dn[a][1] = 0.125 * kEta[a] * (1.0 + kXi[a] * xi) * (1.0 + kZeta[a] * zeta);
        dn[a][2] = 0.125 * kZeta[a] * (1.0 + kXi[a] * xi) * (1.0 + kEta[a] * eta);
    }
    double jac[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int a = 0; a < 8; ++a)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) jac[r][c] += dn[a][r] * corners[a][c];
    double det = jac[0][0] * (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) -
                 jac[0][1] * (jac[1][0] * jac[2][2] - jac[1][2] * jac[2][0]) +
                 jac[0][2] * (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]);
    double inv[3][3];
    inv[0][0] = (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) / det;
    inv[0][1] = (jac[0][2] * jac[2][1] - jac[0][1] * jac[2][2]) / det;
    inv[0][2] = (jac[0][1] * jac[1][2] - jac[0][2] * jac[1][1]) / det;
    inv[1][0] = (jac[1][2] * jac[2][0] - jac[1][0] * jac[2][2]) / det;
    inv[1][1] = (jac[0][0] * jac[2][2] - jac[0][2] * jac[2][0]) / det;
    inv[1][2] = (jac[0][2] * jac[1][0] - jac[0][0] * jac[1][2]) / det;
    inv[2][0] = (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]) / det;
    inv[2][1] = (jac[0][1] * jac[2][0] - jac[0][0] * jac[2][1]) / det;
    inv[2][2] = (jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0]) / det;
    for (int a = 0; a < 8; ++a)
        for (int i = 0; i < 3; ++i)
            grad[a][i] = inv[0][i] * dn[a][0] + inv[1][i] * dn[a][1] + inv[2][i] * dn[a][2];
}

typedef struct {
    const orc_system *s;
    const orc_recovery *r;
    const double *u;
    int points;
    size_t cell_begin;
    double *out;
} orc_recover_ctx;

static void orc_recover_range(void *p, size_t begin, size_t end) {
    orc_recover_ctx *c = (orc_recover_ctx *)p;
    const orc_system *s = c->s;
    const orc_recovery *rc = c->r;
    const size_t n = s->n, nf = rc->n_fine;
    const uint32_t cx = rc->cx, cy = rc->cy, cz = rc->cz;
    const size_t E = (size_t)cx * cy * cz;
    const uint32_t nx = cx + 1, ny = cy + 1;
    const double g = 1.0 / sqrt(3.0);
    const int P = c->points;
    double *q = malloc(n * sizeof(double));
    double *field = malloc(nf * sizeof(double));
    for (size_t ci = begin; ci < end; ++ci) {
        size_t blk = c->cell_begin + ci;
        int kind = s->kinds ? s->kinds[blk] : 0;
        double dt = s->delta_t[blk];
        const uint32_t *dm = s->dof_map + blk * n;
        for (size_t a = 0; a < n; ++a) q[a] = c->u[dm[a]]; /* global_stage.cpp:207-213 */
        const double *Phi = rc->Phi[kind], *uT = rc->u_T[kind];
        for (size_t dof = 0; dof < nf; ++dof) { /* global_stage.cpp:222-228 */
            const double *row = Phi + dof * n;
            double acc = dt * uT[dof];
            for (size_t i = 0; i < n; ++i) acc += row[i] * q[i];
            field[dof] = acc;
        }
        const double *GX = rc->gx[kind], *GY = rc->gy[kind], *GZ = rc->gz[kind];
        for (uint32_t k = 0; k < cz; ++k)
            for (uint32_t j = 0; j < cy; ++j)
                for (uint32_t i = 0; i < cx; ++i) {
                    size_t e = ((size_t)k * cy + j) * cx + i; /* mesh.cpp:125-127 */
                    uint32_t nodes[8];
                    double corners[8][3];
                    for (int a = 0; a < 8; ++a) { /* corner order mesh.cpp:171-176 */
                        uint32_t di = (a == 1 || a == 2 || a == 5 || a == 6);
                        uint32_t dj = (a == 2 || a == 3 || a == 6 || a == 7);
                        uint32_t dk = a >= 4;
                        nodes[a] = ((k + dk) * ny + (j + dj)) * nx + (i + di);
                        corners[a][0] = GX[i + di];
                        corners[a][1] = GY[j + dj];
                        corners[a][2] = GZ[k + dk];
                    }
                    int mat = rc->elem_mat[kind][e];
                    double lambda = rc->lame[kind][mat][0], mu = rc->lame[kind][mat][1];
                    double alpha = rc->lame[kind][mat][2];
                    double x0 = corners[0][0], x1 = corners[1][0];
                    double y0 = corners[0][1], y1 = corners[2][1];
                    double z0 = corners[0][2], z1 = corners[4][2];
                    for (int gp = 0; gp < P; ++gp) {
                        double xi0 = 0, eta0 = 0, zeta0 = 0;
                        if (P == 8) {
                            xi0 = (gp >> 2) ? g : -g;
                            eta0 = ((gp >> 1) & 1) ? g : -g;
                            zeta0 = (gp & 1) ? g : -g;
                        }
                        double pt[3] = {x0 + 0.5 * (1.0 + xi0) * (x1 - x0), y0 + 0.5 * (1.0 + eta0) * (y1 - y0),
                                        z0 + 0.5 * (1.0 + zeta0) * (z1 - z0)};
                        /* fem.cpp:271-273 */
                        double xi = 2.0 * (pt[0] - corners[0][0]) / (corners[1][0] - corners[0][0]) - 1.0;
                        double eta = 2.0 * (pt[1] - corners[0][1]) / (corners[2][1] - corners[0][1]) - 1.0;
                        double zeta = 2.0 * (pt[2] - corners[0][2]) / (corners[4][2] - corners[0][2]) - 1.0;
                        double grad[8][3];
                        orc_physical_gradients((const double(*)[3])corners, xi, eta, zeta, grad);
                        double du[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
                        for (int a = 0; a < 8; ++a)
                            for (int ii = 0; ii < 3; ++ii)
                                for (int jj = 0; jj < 3; ++jj) du[ii][jj] += field[3 * nodes[a] + ii] * grad[a][jj];
                        double exx = du[0][0], eyy = du[1][1], ezz = du[2][2];
                        double exy = 0.5 * (du[0][1] + du[1][0]);
                        double eyz = 0.5 * (du[1][2] + du[2][1]);
                        double ezx = 0.5 * (du[2][0] + du[0][2]);
                        double trace = exx + eyy + ezz;
                        double thermal = alpha * (3.0 * lambda + 2.0 * mu) * dt;
                        double sxx = lambda * trace + 2.0 * mu * exx - thermal;
                        double syy = lambda * trace + 2.0 * mu * eyy - thermal;
                        double szz = lambda * trace + 2.0 * mu * ezz - thermal;
                        double sxy = 2.0 * mu * exy, syz = 2.0 * mu * eyz, szx = 2.0 * mu * ezx;
                        double d1 = sxx - syy, d2 = syy - szz, d3 = szz - sxx; /* fem.cpp:311-316 */
                        double v = 0.5 * (d1 * d1 + d2 * d2 + d3 * d3) + 3.0 * (sxy * sxy + syz * syz + szx * szx);
                        double *o = c->out + ((ci * E + e) * (size_t)P + (size_t)gp) * 7;
                        o[0] = sxx; o[1] = syy; o[2] = szz; o[3] = sxy; o[4] = syz; o[5] = szx;
                        o[6] = sqrt(v > 0.0 ? v : 0.0);
                    }
                }
    }
    free(q);
    free(field);
}

void orc_recover(const orc_system *s, const orc_recovery *r, const double *u, int points,
                 size_t cell_begin, size_t cell_end, double *out) {
    orc_recover_ctx ctx = {s, r, u, points, cell_begin, out};
    orc_parallel(cell_end - cell_begin, s->threads, orc_recover_range, &ctx);
}
