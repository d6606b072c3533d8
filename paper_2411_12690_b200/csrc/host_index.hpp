// Host-side array configuration and global indexing of the reduced system.
//
// New C++ that keeps the reference's API surface and numbering, bit for
// bit:
//   NodeLayout::create        rom.cpp:12-33   (i outer, j, k inner; strict interior skipped)
//   num_element_dofs          rom.cpp:40-46
//   ArrayLayout::validate     global_stage.cpp:8-15
//   index_global_nodes        global_stage.cpp:94-119 (gz, gy, gx scan)
//   GlobalIndex::global_dof   global_stage.cpp:82-92
//   reduced_dirichlet         global_stage.cpp:154-178 (clamped) + the configs' bottom-pin sets
//   DirichletSet              fem.cpp:62-80 (sorted, duplicates must agree)
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tsvb200 {

/// tsvstress::Error (core.hpp:14-16).
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct NodeLayout {
    std::uint32_t n_x = 4, n_y = 4, n_z = 4;
    std::vector<std::array<std::uint32_t, 3>> surface_nodes;  // lexicographic (i, j, k), k fastest

    static NodeLayout create(std::uint32_t n_x, std::uint32_t n_y, std::uint32_t n_z);
    std::size_t node_count() const { return surface_nodes.size(); }
    std::size_t reduced_dofs() const { return surface_nodes.size() * 3; }
};

std::size_t num_element_dofs(std::uint32_t n_x, std::uint32_t n_y, std::uint32_t n_z);

struct ArrayLayout {
    std::uint32_t rows = 1, cols = 1;
    std::vector<std::uint8_t> kinds;  // empty = all tsv (0), 1 = dummy
    std::vector<double> delta_t;      // 1 or rows*cols entries
    double pitch = 0.0, height = 0.0;

    void validate() const;
    std::size_t cell_count() const { return static_cast<std::size_t>(rows) * cols; }
    std::uint8_t kind_at(std::size_t cell) const { return kinds.empty() ? 0 : kinds[cell]; }
    double delta_t_at(std::size_t cell) const { return delta_t.size() == 1 ? delta_t[0] : delta_t[cell]; }
};

struct GlobalIndex {
    std::uint32_t lat_x = 0, lat_y = 0, lat_z = 0;
    std::vector<std::int32_t> node_of_lattice;  // -1 where no block surface passes
    std::vector<std::array<std::uint32_t, 3>> lattice_of_node;
    std::uint32_t nx = 0, ny = 0, nz = 0;

    std::size_t node_count() const { return lattice_of_node.size(); }
    std::size_t dof_count() const { return lattice_of_node.size() * 3; }
    std::size_t lattice_slot(std::uint32_t gx, std::uint32_t gy, std::uint32_t gz) const {
        return (static_cast<std::size_t>(gz) * lat_y + gy) * lat_x + gx;
    }
    std::uint32_t global_dof(std::uint32_t row, std::uint32_t col, const NodeLayout& layout,
                             std::size_t local_dof) const;
};

GlobalIndex index_global_nodes(const ArrayLayout& layout, const NodeLayout& node_layout);

/// B x n table dof_map[b*n + a] = global_dof(row(b), col(b), a).
std::vector<std::uint32_t> dof_map(const ArrayLayout& layout, const GlobalIndex& index,
                                   const NodeLayout& node_layout);

/// fem::DirichletSet: prescribed values keyed by reduced global DoF.
class DirichletSet {
public:
    void set(std::uint32_t dof, double value) {
        entries_.emplace_back(dof, value);
        sorted_ = false;
    }
    const std::vector<std::pair<std::uint32_t, double>>& entries() const;
    std::size_t size() const { return entries().size(); }

private:
    mutable std::vector<std::pair<std::uint32_t, double>> entries_;
    mutable bool sorted_ = true;
};

enum class BcKind { BottomPin = 0, BottomPin321 = 1, Clamped = 2, None = 3 };

/// Dirichlet set of the reduced system for one of the built-in boundary
/// conditions (all values zero).
DirichletSet reduced_dirichlet(BcKind kind, const GlobalIndex& index);

}  // namespace tsvb200
