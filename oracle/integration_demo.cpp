// ORACLE TEST INFRASTRUCTURE — the drop-in demonstration of INTEGRATION.md.
//
// Compiled against the reference's own headers and objects (oracle/_ref)
// and linked with the product library. It runs the reference's online
// stage (index_global_nodes -> assemble_global -> apply_dirichlet_lifting
// -> solve_global -> evaluate_stress_in_element) and the GPU stage fed with
// the SAME reference objects (RomSet, ArrayLayout, DirichletSet,
// IterOptions) through include/tsvstress_b200/global_gpu.hpp, then compares.
// Exit code 0 = parity within the north_star tolerances.
#include <cmath>
#include <cstdio>
#include <random>

#include "tsvstress/fem.hpp"
#include "tsvstress/global.hpp"
#include "tsvstress/linalg.hpp"
#include "tsvstress/mesh.hpp"
#include "tsvstress/rom.hpp"
#include "tsvstress/stress_grid.hpp"
#include "tsvstress_b200/global_gpu.hpp"

using namespace tsvstress;

int main() {
    UnitBlockGeometry geom;  // defaults: d 5 um, h 50 um, t 0.5 um, p 15 um
    TensorGrid grid;
    grid.x = linspace(0.0, geom.p, 8);
    grid.y = grid.x;
    grid.z = linspace(0.0, geom.h, 8);
    MaterialTable mats = MaterialTable::defaults();
    rom::NodeLayout nl = rom::NodeLayout::create(4, 4, 4, geom.p, geom.p, geom.h);
    global::RomSet roms;
    roms.tsv = rom::build_rom(geom, build_unit_block_mesh(geom, grid), mats, nl, BlockKind::Tsv, 4);
    roms.dummy = rom::build_rom(geom, build_dummy_block_mesh(geom, grid), mats, nl, BlockKind::Dummy, 4);

    global::ArrayLayout layout;
    layout.rows = 4;
    layout.cols = 5;
    layout.pitch = geom.p;
    layout.height = geom.h;
    std::mt19937_64 rng(42);
    for (std::size_t c = 0; c < layout.cell_count(); ++c) {
        layout.kinds.push_back((rng() >> 11) * 0x1.0p-53 < 0.3 ? BlockKind::Dummy : BlockKind::Tsv);
        layout.delta_t.push_back(-270.0 + 40.0 * ((rng() >> 11) * 0x1.0p-53));
    }

    // reference path
    global::GlobalIndex index = global::index_global_nodes(layout, nl);
    global::GlobalSystem sys = global::assemble_global(roms, layout, index);
    fem::DirichletSet bc;  // the configs' bottom pin + 3-2-1 rule
    for (std::size_t id = 0; id < index.node_count(); ++id) {
        const auto &lat = index.lattice_of_node[id];
        if (lat[2] != 0) continue;
        const auto base = static_cast<std::uint32_t>(3 * id);
        bc.set(base + 2, 0.0);
        if (lat[0] == 0 && lat[1] == 0) {
            bc.set(base, 0.0);
            bc.set(base + 1, 0.0);
        }
        if (lat[0] == index.lat_x - 1 && lat[1] == 0) bc.set(base + 1, 0.0);
    }
    fem::apply_dirichlet_lifting(sys.stiffness, sys.load, bc);
    linalg::IterOptions opts;
    opts.tolerance = 1e-12;
    global::GlobalSolution ref = global::solve_global(sys, opts);

    // GPU path, fed the same reference objects
    b200::GpuGlobalStage gpu(0);
    gpu.set_roms(roms);
    gpu.set_layout(layout);
    gpu.set_dirichlet(bc);
    b200::GlobalSolution sol = gpu.solve_global(opts);

    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < ref.u.size(); ++i) {
        num += (sol.u[i] - ref.u[i]) * (sol.u[i] - ref.u[i]);
        den += ref.u[i] * ref.u[i];
    }
    const double du = std::sqrt(num / den);

    // Gauss-point stresses of two cells from the reference solution
    gpu.set_solution(ref.u);
    global::BlockMeshes meshes = global::BlockMeshes::from(roms);
    const std::size_t E = grid.cell_count();
    double worst = 0.0;
    for (std::size_t cell : {std::size_t(0), layout.cell_count() - 1}) {
        const auto r = static_cast<std::uint32_t>(cell / layout.cols), c = static_cast<std::uint32_t>(cell % layout.cols);
        const BlockKind kind = layout.kind_at(r, c);
        const auto &model = roms.at(kind);
        const HexMesh &mesh = meshes.at(kind);
        const double dt = layout.delta_t_at(r, c);
        auto field = global::reconstruct_block_field(model, global::gather_cell_values(ref.u, r, c, index, nl), dt);
        std::vector<double> g = gpu.recover(8, E, cell, cell + 1);
        double vmax = 0.0, dmax = 0.0;
        const double gp = 1.0 / std::sqrt(3.0);
        for (std::size_t e = 0; e < E; ++e) {
            auto cr = mesh.element_corners(e);
            for (int k = 0; k < 8; ++k) {
                const double xi = (k >> 2) ? gp : -gp, eta = ((k >> 1) & 1) ? gp : -gp, ze = (k & 1) ? gp : -gp;
                std::array<double, 3> pt = {cr[0][0] + 0.5 * (1 + xi) * (cr[1][0] - cr[0][0]),
                                            cr[0][1] + 0.5 * (1 + eta) * (cr[2][1] - cr[0][1]),
                                            cr[0][2] + 0.5 * (1 + ze) * (cr[4][2] - cr[0][2])};
                fem::StressTensor s = fem::evaluate_stress_in_element(field, mesh, e, pt, model.materials, dt);
                const double vm = fem::von_mises(s);
                vmax = std::max(vmax, std::abs(vm));
                dmax = std::max(dmax, std::abs(vm - g[(e * 8 + k) * 7 + 6]));
            }
        }
        worst = std::max(worst, dmax / vmax);
    }
    // cut plane (cutplane_von_mises, global_stage.cpp:245-274) from the same u
    const std::uint32_t res = 20;
    StressGrid cut_ref = global::cutplane_von_mises(ref, layout, roms, index, meshes, res, 4);
    std::vector<double> cut_gpu = gpu.cutplane_von_mises(res);
    double cmax = 0.0, cdiff = 0.0;
    for (std::size_t i = 0; i < cut_gpu.size(); ++i) {
        cmax = std::max(cmax, std::abs(cut_ref.values[i]));
        cdiff = std::max(cdiff, std::abs(cut_ref.values[i] - cut_gpu[i]));
    }

    // the same objects with the two-level Schwarz preconditioner (TSV_PRECOND_SCHWARZ2)
    b200::GlobalSolution sw = gpu.solve_global(opts, TSV_PRECOND_SCHWARZ2);
    double num2 = 0.0;
    for (std::size_t i = 0; i < ref.u.size(); ++i) num2 += (sw.u[i] - ref.u[i]) * (sw.u[i] - ref.u[i]);
    const double du_sw = std::sqrt(num2 / den);

    std::printf(
        "{\"du_rel_l2\": %.3e, \"iterations_ref\": %d, \"iterations_gpu\": %d, \"vm_rel_err\": %.3e, "
        "\"cutplane_rel_err\": %.3e, \"du_rel_l2_schwarz2\": %.3e, \"iterations_schwarz2\": %d}\n",
        du, ref.iterations, sol.iterations, worst, cdiff / cmax, du_sw, sw.iterations);
    return (du <= 1e-10 && worst <= 1e-8 && cut_gpu.size() == cut_ref.values.size() && cdiff <= 1e-8 * cmax &&
            du_sw <= 1e-10)
               ? 0
               : 1;
}
