// tsvstress_b200/global_gpu.hpp — C++ host API of the B200 online stage.
//
// Header-only layer over the C ABI (tsv_b200.h) that keeps the reference's
// solver and array-config API surface (proj/include/tsvstress/global.hpp,
// linalg.hpp): same names, argument meaning and exception behaviour. The
// set_* members are templates over the reference's own types, so a
// tsvstress build can hand its RomSet / ArrayLayout / DirichletSet /
// IterOptions straight in without this header including the reference:
//
//   RomSet        (global.hpp:36-43)   optional<ReducedOrderModel> tsv, dummy
//   ArrayLayout   (global.hpp:16-32)   rows, cols, kinds, delta_t, pitch, height
//   DirichletSet  (fem.hpp:22-36)      entries() -> (dof, value) pairs
//   IterOptions   (linalg.hpp:120-129) tolerance, max_iterations, precond
//
// Exceptions mirror the reference: Error (core.hpp:14-16), NoConvergence
// carrying the best iterate (linalg.hpp:137-141). There is no direct-LDLT
// fallback on the GPU path: solve_global throws
// NoConvergence where the reference would fall back to factorize_spd.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../tsv_b200.h"

namespace tsvstress::b200 {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class Precond { None = 0, Diagonal = 1, BlockDiagonal = 2 };

struct IterOptions {
    double tolerance = 1e-10;
    int max_iterations = 10000;
    Precond precond = Precond::Diagonal;
};

struct GlobalSolution {
    std::vector<double> u;
    int iterations = 0;
    double relative_residual = 0.0;
    bool direct_fallback = false;
    double device_ms = 0.0;
};

struct NoConvergence : Error {
    NoConvergence(GlobalSolution b, const std::string &what) : Error(what), best(std::move(b)) {}
    GlobalSolution best;
};

struct BreakdownError : Error {
    using Error::Error;
};

/// Field-by-field view of a reference ReducedOrderModel (rom.hpp:57-72).
/// Element materials are rebuilt from the geometry (BlockMeshes::from).
template <class Model>
tsv_rom_desc describe_rom(const Model &m) {
    tsv_rom_desc d{};
    d.q[0] = m.layout.n_x;
    d.q[1] = m.layout.n_y;
    d.q[2] = m.layout.n_z;
    d.geometry[0] = m.geometry.d;
    d.geometry[1] = m.geometry.h;
    d.geometry[2] = m.geometry.t;
    d.geometry[3] = m.geometry.p;
    d.grid_len[0] = static_cast<uint32_t>(m.grid.x.size());
    d.grid_len[1] = static_cast<uint32_t>(m.grid.y.size());
    d.grid_len[2] = static_cast<uint32_t>(m.grid.z.size());
    d.grid[0] = m.grid.x.data();
    d.grid[1] = m.grid.y.data();
    d.grid[2] = m.grid.z.data();
    for (int i = 0; i < 3; ++i) {
        d.materials[i][0] = m.materials.entries[i].youngs_modulus;
        d.materials[i][1] = m.materials.entries[i].poisson_ratio;
        d.materials[i][2] = m.materials.entries[i].thermal_expansion;
    }
    d.element_material = nullptr;
    d.a_element = m.a_element.values().data();
    d.b_element = m.b_element.data();
    d.basis = m.basis.values().data();
    d.thermal = m.thermal.data();
    std::memcpy(d.fingerprint, m.fingerprint.data(), 32);
    return d;
}

/// One GPU context holding the ROMs and the array in HBM.
class GpuGlobalStage {
public:
    explicit GpuGlobalStage(int device = 0) {
        if (tsv_ctx_create(device, &ctx_) != TSV_OK) throw Error("tsv_ctx_create failed (no CUDA device?)");
    }
    ~GpuGlobalStage() { tsv_ctx_destroy(ctx_); }
    GpuGlobalStage(const GpuGlobalStage &) = delete;
    GpuGlobalStage &operator=(const GpuGlobalStage &) = delete;

    /// RomSet::check_consistency runs in set_layout (fingerprints, geometry).
    template <class RomSet>
    void set_roms(const RomSet &roms) {
        if (roms.tsv) set_rom(0, *roms.tsv);
        if (roms.dummy) set_rom(1, *roms.dummy);
    }

    template <class Model>
    void set_rom(int kind, const Model &m) {
        tsv_rom_desc d = describe_rom(m);
        check(tsv_set_rom(ctx_, kind, &d));
    }

    /// ArrayLayout + index_global_nodes (global_stage.cpp:94-119).
    template <class Layout>
    void set_layout(const Layout &l) {
        std::vector<uint8_t> kinds;
        for (const auto &k : l.kinds) kinds.push_back(static_cast<uint8_t>(k));
        rows_ = l.rows;
        cols_ = l.cols;
        check(tsv_set_layout(ctx_, l.rows, l.cols, kinds.empty() ? nullptr : kinds.data(), l.delta_t.data(),
                             l.delta_t.size(), l.pitch, l.height));
    }

    /// fem::DirichletSet (apply_dirichlet_lifting semantics, fem.cpp:223-260).
    template <class Set>
    void set_dirichlet(const Set &set) {
        std::vector<uint32_t> dofs;
        std::vector<double> vals;
        for (const auto &e : set.entries()) {
            dofs.push_back(e.first);
            vals.push_back(e.second);
        }
        check(tsv_set_dirichlet(ctx_, dofs.size(), dofs.data(), vals.data()));
    }

    void set_bc(tsv_bc_kind kind) { check(tsv_set_bc(ctx_, kind)); }

    size_t dof_count() {
        uint64_t n = 0;
        check(tsv_get_index(ctx_, &n, nullptr, nullptr, nullptr));
        return n;
    }

    /// solve_global (global_stage.cpp:187-205) with a linalg::IterOptions-like
    /// argument (tolerance, max_iterations, precond).
    template <class Opts = IterOptions>
    GlobalSolution solve_global(const Opts &o = Opts{}) {
        return solve_with(o, static_cast<int>(o.precond));
    }

    /// The same solve with a preconditioner outside linalg::Precond, e.g.
    /// TSV_PRECOND_SCHWARZ2 (two-level additive Schwarz; same u within the
    /// parity bar, far fewer iterations).
    template <class Opts = IterOptions>
    GlobalSolution solve_global(const Opts &o, int precond_override) {
        return solve_with(o, precond_override);
    }

    /// Online stage with a new temperature field only (ArrayLayout::delta_t,
    /// global.hpp:16-32): index, BCs and the preconditioner are kept.
    void set_delta_t(const std::vector<double> &delta_t) {
        check(tsv_set_delta_t(ctx_, delta_t.data(), delta_t.size()));
    }

    /// rom::load_rom (rom.cpp:305-377) straight into a RomSet slot (-1 = the
    /// file's kind); returns the kind stored in the file.
    int load_rom_file(const std::string &path, int slot = -1) {
        int kind = -1;
        char err[512];
        const int rc = tsv_load_rom_file(ctx_, slot, path.c_str(), &kind, err, sizeof err);
        if (rc != TSV_OK) throw Error(err);
        return kind;
    }

    /// cutplane_von_mises (global_stage.cpp:245-274) on the GPU: the
    /// StressGrid values, [((row * cols + col) * res + py) * res + px].
    std::vector<double> cutplane_von_mises(uint32_t res) {
        std::vector<double> v(static_cast<size_t>(rows_) * cols_ * res * res);
        check(tsv_cutplane(ctx_, res, v.data()));
        return v;
    }

    void set_solution(const std::vector<double> &u) { check(tsv_set_solution(ctx_, u.data())); }

    /// Stress + von Mises at Gauss points (points = 8) or centroids (1) of
    /// every element of cells [c0, c1): [cell][element][point][xx,yy,zz,xy,yz,zx,vm].
    std::vector<double> recover(int points, size_t elements_per_cell, size_t c0, size_t c1) {
        std::vector<double> out((c1 - c0) * elements_per_cell * points * 7);
        check(tsv_recover(ctx_, points, c0, c1, out.data()));
        return out;
    }

    /// y = A_lifted x.
    std::vector<double> apply(const std::vector<double> &x) {
        std::vector<double> y(x.size());
        check(tsv_apply(ctx_, x.data(), y.data()));
        return y;
    }

    tsv_ctx *handle() { return ctx_; }

private:
    template <class Opts>
    GlobalSolution solve_with(const Opts &o, int precond) {
        tsv_iter_options c{o.tolerance, o.max_iterations, precond};
        GlobalSolution sol;
        sol.u.resize(dof_count());
        tsv_solve_info info{};
        const int rc = tsv_solve(ctx_, &c, sol.u.data(), &info);
        sol.iterations = info.iterations;
        sol.relative_residual = info.relative_residual;
        sol.device_ms = info.solve_ms;
        if (rc == TSV_ENOCONV) throw NoConvergence(std::move(sol), tsv_last_error(ctx_));
        check(rc);
        return sol;
    }

    void check(int rc) {
        if (rc == TSV_OK) return;
        const std::string msg = tsv_last_error(ctx_);
        if (rc == TSV_EBREAKDOWN) throw BreakdownError(msg);
        throw Error(msg);
    }
    tsv_ctx *ctx_ = nullptr;
    uint32_t rows_ = 0, cols_ = 0;
};

}  // namespace tsvstress::b200
