// ORACLE TEST INFRASTRUCTURE — not product code. Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
//
// extern "C" shim over the reference's OWN sources (compiled unmodified
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It
// drives the reference library the way its test drivers do
// (tests/acceptance.cpp:108-128 PitchArtifacts::solve_mor):
//   index_global_nodes -> assemble_global -> Dirichlet lifting ->
//   solve_global -> per-cell gather + reconstruct_block_field +
//   evaluate_stress_in_element + von_mises.
// The configs' boundary condition (bottom u_z = 0 + pinned corner [+ 3-2-1
// pin]) and Gauss-point / centroid recovery are not expressible through
// RunConfig (config.cpp:297-303), so, as SURVEY.md §3.2 prescribes, this
// shim builds the fem::DirichletSet by hand and passes it to
// fem::apply_dirichlet_lifting (the call apply_global_bcs makes at
// global_stage.cpp:182-183), and loops over cells as cutplane_von_mises
// does (global_stage.cpp:253-271) with Gauss-point coordinates.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "tsvstress/core.hpp"
#include "tsvstress/fem.hpp"
#include "tsvstress/global.hpp"
#include "tsvstress/linalg.hpp"
#include "tsvstress/material.hpp"
#include "tsvstress/mesh.hpp"
#include "tsvstress/rom.hpp"

using namespace tsvstress;

namespace {
thread_local std::string g_err;

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Rom {
    rom::ReducedOrderModel model;
};

struct Session {
    global::RomSet roms;
    global::ArrayLayout layout;
    global::GlobalIndex index;
    global::GlobalSystem sys;        // lifted
    fem::DirichletSet bc;
    global::BlockMeshes meshes;
    double t_index = 0, t_assemble = 0, t_lift = 0;
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const linalg::NoConvergence& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

/// build_rom (rom.cpp:134-253) on a uniform TensorGrid (linspace, as the
/// reference fixtures do, test_global.cpp:22-28) with the default materials
/// (material.cpp:37-43) except the liner Young modulus.
void* ref_rom_build3(double d, double h, double t, double p, int m_xy, int m_z, int qx, int qy, int qz,
                     int kind, double liner_e, int threads);

void* ref_rom_build(double d, double h, double t, double p, int m_xy, int m_z, int q, int kind,
                    double liner_e, int threads) {
    return ref_rom_build3(d, h, t, p, m_xy, m_z, q, q, q, kind, liner_e, threads);
}

// NodeLayout with separate node counts per axis (rom::NodeLayout::create(nx, ny, nz, ...)).
void* ref_rom_build3(double d, double h, double t, double p, int m_xy, int m_z, int qx, int qy, int qz,
                     int kind, double liner_e, int threads) {
    Rom* out = nullptr;
    int st = guarded([&] {
        UnitBlockGeometry g;
        g.d = d; g.h = h; g.t = t; g.p = p;
        TensorGrid grid;
        grid.x = linspace(0.0, p, static_cast<std::size_t>(m_xy));
        grid.y = grid.x;
        grid.z = linspace(0.0, h, static_cast<std::size_t>(m_z));
        MaterialTable mats = MaterialTable::defaults();
        const Material& l = mats[MaterialId::Liner];
        mats[MaterialId::Liner] = Material::make(liner_e, l.poisson_ratio, l.thermal_expansion);
        rom::NodeLayout nl = rom::NodeLayout::create(qx, qy, qz, p, p, h);
        BlockKind k = kind == 0 ? BlockKind::Tsv : BlockKind::Dummy;
        HexMesh mesh = k == BlockKind::Tsv ? build_unit_block_mesh(g, grid) : build_dummy_block_mesh(g, grid);
        out = new Rom{rom::build_rom(g, mesh, mats, nl, k, threads)};
    });
    return st == 0 ? out : nullptr;
}

void* ref_rom_load(const char* path) {
    Rom* out = nullptr;
    int st = guarded([&] { out = new Rom{rom::load_rom(path)}; });
    return st == 0 ? out : nullptr;
}

int ref_rom_save(void* h, const char* path) {
    return guarded([&] { rom::save_rom(static_cast<Rom*>(h)->model, path); });
}

void ref_rom_free(void* h) { delete static_cast<Rom*>(h); }

/// dims[0..] = n, n_fine, n_elem, cells_x, cells_y, cells_z, q_x, q_y, q_z, kind
void ref_rom_dims(void* h, int64_t* dims) {
    const auto& m = static_cast<Rom*>(h)->model;
    dims[0] = static_cast<int64_t>(m.reduced_dofs());
    dims[1] = static_cast<int64_t>(m.fine_dofs());
    dims[2] = static_cast<int64_t>(m.grid.cell_count());
    dims[3] = static_cast<int64_t>(m.grid.cells_x());
    dims[4] = static_cast<int64_t>(m.grid.cells_y());
    dims[5] = static_cast<int64_t>(m.grid.cells_z());
    dims[6] = m.layout.n_x;
    dims[7] = m.layout.n_y;
    dims[8] = m.layout.n_z;
    dims[9] = static_cast<int64_t>(m.kind);
}

/// Copies K_r (n*n row-major), b_el (n), Phi (n_fine*n row-major), u_T
/// (n_fine), grid lines, element materials (MaterialId of the rebuilt
/// mesh, BlockMeshes::from global_stage.cpp:232-237), material constants
/// [E, nu, alpha, lambda, mu] x 3, geometry [d,h,t,p], fingerprint (32 B).
int ref_rom_copy(void* h, double* k_r, double* b_el, double* phi, double* u_t, double* gx,
                 double* gy, double* gz, uint8_t* elem_mat, double* mats, double* geom,
                 uint8_t* fingerprint) {
    return guarded([&] {
        const auto& m = static_cast<Rom*>(h)->model;
        if (k_r) std::memcpy(k_r, m.a_element.values().data(), m.a_element.values().size() * 8);
        if (b_el) std::memcpy(b_el, m.b_element.data(), m.b_element.size() * 8);
        if (phi) std::memcpy(phi, m.basis.values().data(), m.basis.values().size() * 8);
        if (u_t) std::memcpy(u_t, m.thermal.data(), m.thermal.size() * 8);
        if (gx) std::memcpy(gx, m.grid.x.data(), m.grid.x.size() * 8);
        if (gy) std::memcpy(gy, m.grid.y.data(), m.grid.y.size() * 8);
        if (gz) std::memcpy(gz, m.grid.z.data(), m.grid.z.size() * 8);
        if (elem_mat) {
            HexMesh mesh = m.kind == BlockKind::Tsv ? build_unit_block_mesh(m.geometry, m.grid)
                                                    : build_dummy_block_mesh(m.geometry, m.grid);
            for (std::size_t e = 0; e < mesh.element_count(); ++e)
                elem_mat[e] = static_cast<uint8_t>(mesh.element_material[e]);
        }
        if (mats)
            for (int i = 0; i < 3; ++i) {
                const Material& mt = m.materials.entries[i];
                mats[5 * i + 0] = mt.youngs_modulus;
                mats[5 * i + 1] = mt.poisson_ratio;
                mats[5 * i + 2] = mt.thermal_expansion;
                mats[5 * i + 3] = mt.lame_lambda;
                mats[5 * i + 4] = mt.lame_mu;
            }
        if (geom) {
            geom[0] = m.geometry.d; geom[1] = m.geometry.h; geom[2] = m.geometry.t; geom[3] = m.geometry.p;
        }
        if (fingerprint) std::memcpy(fingerprint, m.fingerprint.data(), 32);
    });
}

/// bc_mode: 0 = literal config BC (u_z = 0 on every bottom-lattice node,
/// corner (0,0,0) fully pinned); 1 = 3-2-1 (literal + u_y = 0 at
/// (lat_x-1,0,0)); 2 = reference GlobalBC::clamped()
/// (global_stage.cpp:154-163); 3 = no Dirichlet set.
void* ref_session_create(void* tsv, void* dummy, uint32_t rows, uint32_t cols, const uint8_t* kinds,
                         const double* delta_t, uint64_t n_dt, double pitch, double height, int bc_mode) {
    Session* s = new Session();
    int st = guarded([&] {
        if (tsv) s->roms.tsv = static_cast<Rom*>(tsv)->model;
        if (dummy) s->roms.dummy = static_cast<Rom*>(dummy)->model;
        s->layout.rows = rows;
        s->layout.cols = cols;
        if (kinds) {
            s->layout.kinds.resize(static_cast<std::size_t>(rows) * cols);
            for (std::size_t i = 0; i < s->layout.kinds.size(); ++i)
                s->layout.kinds[i] = kinds[i] ? BlockKind::Dummy : BlockKind::Tsv;
        }
        s->layout.delta_t.assign(delta_t, delta_t + n_dt);
        s->layout.pitch = pitch;
        s->layout.height = height;
        const rom::NodeLayout& nl = s->roms.any().layout;

        double t0 = now_s();
        s->index = global::index_global_nodes(s->layout, nl);
        double t1 = now_s();
        s->sys = global::assemble_global(s->roms, s->layout, s->index);
        double t2 = now_s();
        if (bc_mode == 2) {
            s->bc = global::reduced_dirichlet(global::GlobalBC::clamped(), s->index, s->layout);
        } else if (bc_mode == 0 || bc_mode == 1) {
            const auto& idx = s->index;
            for (std::size_t id = 0; id < idx.node_count(); ++id) {
                const auto& lat = idx.lattice_of_node[id];
                if (lat[2] != 0) continue;
                std::uint32_t base = static_cast<std::uint32_t>(3 * id);
                s->bc.set(base + 2, 0.0);
                if (lat[0] == 0 && lat[1] == 0) {
                    s->bc.set(base + 0, 0.0);
                    s->bc.set(base + 1, 0.0);
                }
                if (bc_mode == 1 && lat[0] == idx.lat_x - 1 && lat[1] == 0) s->bc.set(base + 1, 0.0);
            }
        }
        fem::apply_dirichlet_lifting(s->sys.stiffness, s->sys.load, s->bc);
        double t3 = now_s();
        s->meshes = global::BlockMeshes::from(s->roms);
        s->t_index = t1 - t0;
        s->t_assemble = t2 - t1;
        s->t_lift = t3 - t2;
    });
    if (st != 0) {
        delete s;
        return nullptr;
    }
    return s;
}

void ref_session_free(void* h) { delete static_cast<Session*>(h); }

/// info[0..] = N, nnz, lat_x, lat_y, lat_z, node_count, n (reduced/block), n_constrained
void ref_session_info(void* h, int64_t* info, double* timings) {
    auto* s = static_cast<Session*>(h);
    info[0] = static_cast<int64_t>(s->index.dof_count());
    info[1] = static_cast<int64_t>(s->sys.stiffness.nnz());
    info[2] = s->index.lat_x;
    info[3] = s->index.lat_y;
    info[4] = s->index.lat_z;
    info[5] = static_cast<int64_t>(s->index.node_count());
    info[6] = static_cast<int64_t>(s->roms.any().reduced_dofs());
    info[7] = static_cast<int64_t>(s->bc.size());
    if (timings) {
        timings[0] = s->t_index;
        timings[1] = s->t_assemble;
        timings[2] = s->t_lift;
    }
}

/// dof_map[b*n + a] = GlobalIndex::global_dof(row, col, layout, a)
/// (global_stage.cpp:82-92), b = row*cols + col.
void ref_session_dof_map(void* h, uint32_t* out) {
    auto* s = static_cast<Session*>(h);
    const auto& nl = s->roms.any().layout;
    const std::size_t n = nl.reduced_dofs();
    for (std::uint32_t r = 0; r < s->layout.rows; ++r)
        for (std::uint32_t c = 0; c < s->layout.cols; ++c) {
            std::size_t b = static_cast<std::size_t>(r) * s->layout.cols + c;
            for (std::size_t a = 0; a < n; ++a) out[b * n + a] = s->index.global_dof(r, c, nl, a);
        }
}

void ref_session_lattice(void* h, int32_t* node_of_lattice, uint32_t* lattice_of_node) {
    auto* s = static_cast<Session*>(h);
    if (node_of_lattice)
        std::memcpy(node_of_lattice, s->index.node_of_lattice.data(), s->index.node_of_lattice.size() * 4);
    if (lattice_of_node)
        for (std::size_t i = 0; i < s->index.node_count(); ++i)
            for (int c = 0; c < 3; ++c) lattice_of_node[3 * i + c] = s->index.lattice_of_node[i][c];
}

/// Lifted right-hand side and the constrained-DoF mask / values.
void ref_session_rhs(void* h, double* b, uint8_t* constrained, double* values) {
    auto* s = static_cast<Session*>(h);
    if (b) std::memcpy(b, s->sys.load.data(), s->sys.load.size() * 8);
    if (constrained || values) {
        for (const auto& [dof, g] : s->bc.entries()) {
            if (constrained) constrained[dof] = 1;
            if (values) values[dof] = g;
        }
    }
}

/// y = A_lifted x via CsrMatrix::apply (linalg.cpp:74-86).
int ref_session_apply(void* h, const double* x, double* y, int threads) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        const std::size_t n = s->sys.stiffness.n_rows();
        s->sys.stiffness.apply(std::span<const double>(x, n), std::span<double>(y, n), threads);
    });
}

/// solve_global (global_stage.cpp:187-205). precond: 0 none, 1 diagonal,
/// 2 block-diagonal. Returns 0 ok, 1 Error (message in ref_last_error).
int ref_session_solve(void* h, double tol, int max_it, int precond, int threads, double* u,
                      int* iterations, double* relres, int* direct_fallback, double* wall_s) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        linalg::IterOptions o;
        o.tolerance = tol;
        o.max_iterations = max_it;
        o.precond = precond == 0 ? linalg::Precond::None
                  : precond == 1 ? linalg::Precond::Diagonal
                                 : linalg::Precond::BlockDiagonal;
        o.threads = threads;
        double t0 = now_s();
        global::GlobalSolution sol = global::solve_global(s->sys, o);
        if (wall_s) *wall_s = now_s() - t0;
        std::memcpy(u, sol.u.data(), sol.u.size() * 8);
        *iterations = sol.iterations;
        *relres = sol.relative_residual;
        *direct_fallback = sol.direct_fallback ? 1 : 0;
    });
}

/// Iterative solve without the direct fallback (linalg::iterative_solve,
/// linalg.cpp:485-493): returns 2 on NoConvergence with the best iterate in
/// u (linalg.hpp:137-141).
int ref_session_iterate(void* h, double tol, int max_it, int precond, int threads, double* u,
                        int* iterations, double* relres) {
    auto* s = static_cast<Session*>(h);
    try {
        linalg::IterOptions o;
        o.tolerance = tol;
        o.max_iterations = max_it;
        o.precond = precond == 0 ? linalg::Precond::None
                  : precond == 1 ? linalg::Precond::Diagonal
                                 : linalg::Precond::BlockDiagonal;
        o.threads = threads;
        linalg::IterResult r = linalg::iterative_solve(s->sys.stiffness, s->sys.load, o);
        std::memcpy(u, r.x.data(), r.x.size() * 8);
        *iterations = r.iterations;
        *relres = r.relative_residual;
        return 0;
    } catch (const linalg::NoConvergence& nc) {
        std::memcpy(u, nc.best.x.data(), nc.best.x.size() * 8);
        *iterations = nc.best.iterations;
        *relres = nc.best.relative_residual;
        g_err = nc.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

/// Gauss-point (points = 8) or centroid (points = 1) stress recovery for
/// cells [cell_begin, cell_end). out[((c - cell_begin)*E + e)*P + g)*7 + k],
/// k = xx,yy,zz,xy,yz,zx,VM; GP order (gx, gy, gz) with gz fastest and
/// natural coordinate -+1/sqrt(3) as in fem.cpp:87-92.
int ref_session_recover(void* h, const double* u, int points, uint64_t cell_begin, uint64_t cell_end,
                        double* out, int threads) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        const rom::NodeLayout& nl = s->roms.any().layout;
        const std::size_t n_global = s->index.dof_count();
        std::span<const double> us(u, n_global);
        const double g = 1.0 / std::sqrt(3.0);
        const int P = points;
        parallel_for_ranges(cell_end - cell_begin, threads, [&](std::size_t begin, std::size_t end) {
            for (std::size_t ci = begin; ci < end; ++ci) {
                std::size_t cell = cell_begin + ci;
                std::uint32_t r = static_cast<std::uint32_t>(cell / s->layout.cols);
                std::uint32_t c = static_cast<std::uint32_t>(cell % s->layout.cols);
                BlockKind kind = s->layout.kind_at(r, c);
                const rom::ReducedOrderModel& model = s->roms.at(kind);
                const HexMesh& mesh = s->meshes.at(kind);
                double dt = s->layout.delta_t_at(r, c);
                std::vector<double> v = global::gather_cell_values(us, r, c, s->index, nl);
                fem::DisplacementField field = global::reconstruct_block_field(model, v, dt);
                const std::size_t E = mesh.element_count();
                for (std::size_t e = 0; e < E; ++e) {
                    auto corners = mesh.element_corners(e);
                    double x0 = corners[0][0], x1 = corners[1][0];
                    double y0 = corners[0][1], y1 = corners[2][1];
                    double z0 = corners[0][2], z1 = corners[4][2];
                    for (int gp = 0; gp < P; ++gp) {
                        double xi = 0, eta = 0, zeta = 0;
                        if (P == 8) {
                            int gx = gp >> 2, gy = (gp >> 1) & 1, gz = gp & 1;
                            xi = gx ? g : -g;
                            eta = gy ? g : -g;
                            zeta = gz ? g : -g;
                        }
                        std::array<double, 3> pt = {x0 + 0.5 * (1.0 + xi) * (x1 - x0),
                                                    y0 + 0.5 * (1.0 + eta) * (y1 - y0),
                                                    z0 + 0.5 * (1.0 + zeta) * (z1 - z0)};
                        fem::StressTensor st =
                            fem::evaluate_stress_in_element(field, mesh, e, pt, model.materials, dt);
                        double* o = out + ((ci * E + e) * P + gp) * 7;
                        o[0] = st.xx; o[1] = st.yy; o[2] = st.zz;
                        o[3] = st.xy; o[4] = st.yz; o[5] = st.zx;
                        o[6] = fem::von_mises(st);
                    }
                }
            }
        });
    });
}

/// The reference's own cut-plane driver (global_stage.cpp:245-274) on a
/// given solution; out = StressGrid::values (stress_grid.hpp:18).
int ref_session_cutplane(void* h, const double* u, uint32_t res, double* out, int threads) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        global::GlobalSolution sol;
        sol.u.assign(u, u + s->index.dof_count());
        StressGrid grid = global::cutplane_von_mises(sol, s->layout, s->roms, s->index, s->meshes, res, threads);
        std::memcpy(out, grid.values.data(), grid.values.size() * 8);
    });
}

/// Reconstructed fine displacement of one cell (reconstruct_block_field).
int ref_session_block_field(void* h, const double* u, uint64_t cell, double* out) {
    auto* s = static_cast<Session*>(h);
    return guarded([&] {
        const rom::NodeLayout& nl = s->roms.any().layout;
        std::uint32_t r = static_cast<std::uint32_t>(cell / s->layout.cols);
        std::uint32_t c = static_cast<std::uint32_t>(cell % s->layout.cols);
        const auto& model = s->roms.at(s->layout.kind_at(r, c));
        std::vector<double> v = global::gather_cell_values(
            std::span<const double>(u, s->index.dof_count()), r, c, s->index, nl);
        auto f = global::reconstruct_block_field(model, v, s->layout.delta_t_at(r, c));
        std::memcpy(out, f.data(), f.size() * 8);
    });
}

}  // extern "C"

extern "C" {

/// index_global_nodes + GlobalIndex::global_dof alone (no assembly), for
/// bit-exact index checks at sizes where assemble_global would need ~100 GB.
/// Returns the dof count; dof_map [rows*cols][n] may be NULL.
int64_t ref_index(uint32_t rows, uint32_t cols, uint32_t q, uint32_t *dof_map) {
    int64_t n_dofs = -1;
    guarded([&] {
        global::ArrayLayout layout;
        layout.rows = rows;
        layout.cols = cols;
        layout.delta_t = {0.0};
        layout.pitch = 1.0;
        layout.height = 1.0;
        rom::NodeLayout nl = rom::NodeLayout::create(q, q, q, 1.0, 1.0, 1.0);
        global::GlobalIndex idx = global::index_global_nodes(layout, nl);
        n_dofs = static_cast<int64_t>(idx.dof_count());
        if (dof_map) {
            const std::size_t n = nl.reduced_dofs();
            for (std::uint32_t r = 0; r < rows; ++r)
                for (std::uint32_t c = 0; c < cols; ++c) {
                    std::size_t b = static_cast<std::size_t>(r) * cols + c;
                    for (std::size_t a = 0; a < n; ++a) dof_map[b * n + a] = idx.global_dof(r, c, nl, a);
                }
        }
    });
    return n_dofs;
}

}  // extern "C"

extern "C" {

/// StressGrid::save_csv (stress_grid.cpp:36-50) of given values, for the
/// byte-format check of the product's CSV writer.
int ref_stress_grid_save_csv(const double *values, uint32_t rows, uint32_t cols, uint32_t res, double pitch,
                             const char *path) {
    return guarded([&] {
        StressGrid g = StressGrid::make(rows, cols, res, pitch);
        std::memcpy(g.values.data(), values, g.values.size() * sizeof(double));
        g.save_csv(path);
    });
}

// default_grading (mesh.cpp:106-119) and rom_fingerprint (rom.cpp:110-132)
// of a geometry with the default materials and a q^3 node layout: pins the
// product CLI's restatement (tests/test_cli.py). Axis lengths in len[3];
// x/y/z must hold cap values each.
int ref_default_grading(double d, double h, double t, double p, double target, uint32_t q, uint32_t cap, double* x,
                        double* y, double* z, uint32_t* len, uint8_t* fingerprint) {
    return guarded([&] {
        UnitBlockGeometry geom;
        geom.d = d;
        geom.h = h;
        geom.t = t;
        geom.p = p;
        TensorGrid g = default_grading(geom, target);
        const std::vector<double>* axes[3] = {&g.x, &g.y, &g.z};
        double* outs[3] = {x, y, z};
        for (int a = 0; a < 3; ++a) {
            if (axes[a]->size() > cap) throw Error("ref_default_grading: axis longer than cap");
            len[a] = static_cast<uint32_t>(axes[a]->size());
            std::memcpy(outs[a], axes[a]->data(), axes[a]->size() * sizeof(double));
        }
        rom::NodeLayout nl = rom::NodeLayout::create(q, q, q, p, p, h);
        Hash256 fp = rom::rom_fingerprint(geom, g, MaterialTable::defaults(), nl);
        std::memcpy(fingerprint, fp.data(), 32);
    });
}

}  // extern "C"
