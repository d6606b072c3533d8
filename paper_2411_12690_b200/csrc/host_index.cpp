#include "host_index.hpp"

#include <algorithm>
#include <thread>
#include <vector>

namespace tsvb200 {

NodeLayout NodeLayout::create(std::uint32_t n_x, std::uint32_t n_y, std::uint32_t n_z) {
    if (n_x < 2 || n_y < 2 || n_z < 2) throw Error("NodeLayout: need at least 2 interpolation nodes per axis");
    NodeLayout l;
    l.n_x = n_x;
    l.n_y = n_y;
    l.n_z = n_z;
    for (std::uint32_t i = 0; i < n_x; ++i)
        for (std::uint32_t j = 0; j < n_y; ++j)
            for (std::uint32_t k = 0; k < n_z; ++k) {
                const bool strictly_inside =
                    i > 0 && i + 1 < n_x && j > 0 && j + 1 < n_y && k > 0 && k + 1 < n_z;
                if (!strictly_inside) l.surface_nodes.push_back({i, j, k});
            }
    return l;
}

std::size_t num_element_dofs(std::uint32_t n_x, std::uint32_t n_y, std::uint32_t n_z) {
    if (n_x < 2 || n_y < 2 || n_z < 2) throw Error("num_element_dofs: need at least 2 nodes per axis");
    const std::size_t all = static_cast<std::size_t>(n_x) * n_y * n_z;
    const std::size_t inner = static_cast<std::size_t>(n_x - 2) * (n_y - 2) * (n_z - 2);
    return 3 * (all - inner);
}

void ArrayLayout::validate() const {
    if (rows < 1 || cols < 1) throw Error("layout: rows and cols must be >= 1");
    if (!kinds.empty() && kinds.size() != cell_count())
        throw Error("layout: kinds must be empty or have rows*cols entries");
    for (std::uint8_t k : kinds)
        if (k > 1) throw Error("layout: block kind must be 0 (tsv) or 1 (dummy)");
    if (delta_t.size() != 1 && delta_t.size() != cell_count())
        throw Error("layout: delta_t must have one entry or rows*cols entries");
    if (!(pitch > 0.0) || !(height > 0.0)) throw Error("layout: pitch and height must be > 0");
}

std::uint32_t GlobalIndex::global_dof(std::uint32_t row, std::uint32_t col, const NodeLayout& layout,
                                      std::size_t local_dof) const {
    const auto& p = layout.surface_nodes[local_dof / 3];
    const std::uint32_t comp = static_cast<std::uint32_t>(local_dof % 3);
    const std::uint32_t gx = col * (nx - 1) + p[0];
    const std::uint32_t gy = row * (ny - 1) + p[1];
    const std::int32_t id = node_of_lattice[lattice_slot(gx, gy, p[2])];
    return static_cast<std::uint32_t>(id) * 3u + comp;
}

GlobalIndex index_global_nodes(const ArrayLayout& layout, const NodeLayout& node_layout) {
    layout.validate();
    GlobalIndex idx;
    idx.nx = node_layout.n_x;
    idx.ny = node_layout.n_y;
    idx.nz = node_layout.n_z;
    idx.lat_x = layout.cols * (idx.nx - 1) + 1;
    idx.lat_y = layout.rows * (idx.ny - 1) + 1;
    idx.lat_z = idx.nz;
    const std::size_t slots = static_cast<std::size_t>(idx.lat_x) * idx.lat_y * idx.lat_z;
    if (slots >= 0x7fffffffULL) throw Error("index_global_nodes: lattice too large for 32-bit node ids");
    idx.node_of_lattice.assign(slots, -1);
    // A lattice point is skipped only when it is off every block face plane
    // in x and in y and off the top/bottom planes. Nodes are numbered in scan
    // order gz -> gy -> gx: count the kept points per (gz, gy) line, prefix-sum,
    // then number the lines independently on the host threads (same ids).
    const std::size_t lines = static_cast<std::size_t>(idx.lat_z) * idx.lat_y;
    auto keep = [&](std::uint32_t gx, std::uint32_t gy, std::uint32_t gz) {
        const bool on_z_face = gz == 0 || gz + 1 == idx.lat_z;
        const bool on_y_face = gy % (idx.ny - 1) == 0;
        const bool on_x_face = gx % (idx.nx - 1) == 0;
        return on_x_face || on_y_face || on_z_face;
    };
    std::vector<std::size_t> first(lines + 1, 0);
    const std::size_t x_faces = layout.cols + 1;  // kept points of a line off every y/z face plane
    for (std::size_t l = 0; l < lines; ++l) {
        const std::uint32_t gz = static_cast<std::uint32_t>(l / idx.lat_y), gy = static_cast<std::uint32_t>(l % idx.lat_y);
        const bool full = gz == 0 || gz + 1 == idx.lat_z || gy % (idx.ny - 1) == 0;
        first[l + 1] = first[l] + (full ? idx.lat_x : x_faces);
    }
    idx.lattice_of_node.resize(first[lines]);
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 16u));
    auto work = [&](unsigned w) {
        for (std::size_t l = w; l < lines; l += nt) {
            const std::uint32_t gz = static_cast<std::uint32_t>(l / idx.lat_y), gy = static_cast<std::uint32_t>(l % idx.lat_y);
            std::size_t id = first[l];
            for (std::uint32_t gx = 0; gx < idx.lat_x; ++gx) {
                if (!keep(gx, gy, gz)) continue;
                idx.node_of_lattice[idx.lattice_slot(gx, gy, gz)] = static_cast<std::int32_t>(id);
                idx.lattice_of_node[id] = {gx, gy, gz};
                ++id;
            }
        }
    };
    if (nt == 1 || slots < (1u << 16)) {
        for (unsigned w = 0; w < nt; ++w) work(w);
    } else {
        std::vector<std::thread> pool;
        for (unsigned w = 0; w < nt; ++w) pool.emplace_back(work, w);
        for (auto& t : pool) t.join();
    }
    if (idx.dof_count() >= 0xffffffffULL) throw Error("index_global_nodes: more than 2^32 reduced dofs");
    return idx;
}

std::vector<std::uint32_t> dof_map(const ArrayLayout& layout, const GlobalIndex& index,
                                   const NodeLayout& node_layout) {
    const std::size_t n = node_layout.reduced_dofs();
    std::vector<std::uint32_t> out(layout.cell_count() * n);
    // rows are independent: split them over the host threads (same values)
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), layout.rows));
    auto work = [&](unsigned w) {
        for (std::uint32_t r = w; r < layout.rows; r += nt)
            for (std::uint32_t c = 0; c < layout.cols; ++c) {
                const std::size_t b = static_cast<std::size_t>(r) * layout.cols + c;
                for (std::size_t a = 0; a < n; ++a) out[b * n + a] = index.global_dof(r, c, node_layout, a);
            }
    };
    if (nt == 1 || layout.cell_count() * n < (1u << 16)) {
        for (unsigned w = 0; w < nt; ++w) work(w);
        return out;
    }
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nt; ++w) pool.emplace_back(work, w);
    for (auto& t : pool) t.join();
    return out;
}

const std::vector<std::pair<std::uint32_t, double>>& DirichletSet::entries() const {
    if (!sorted_) {
        std::sort(entries_.begin(), entries_.end());
        for (std::size_t i = 1; i < entries_.size(); ++i)
            if (entries_[i].first == entries_[i - 1].first && entries_[i].second != entries_[i - 1].second)
                throw Error("DirichletSet: dof " + std::to_string(entries_[i].first) +
                            " prescribed twice with different values");
        entries_.erase(std::unique(entries_.begin(), entries_.end()), entries_.end());
        sorted_ = true;
    }
    return entries_;
}

DirichletSet reduced_dirichlet(BcKind kind, const GlobalIndex& index) {
    DirichletSet set;
    for (std::size_t id = 0; id < index.node_count(); ++id) {
        const auto& lat = index.lattice_of_node[id];
        const std::uint32_t base = static_cast<std::uint32_t>(3 * id);
        switch (kind) {
            case BcKind::Clamped:
                if (lat[2] == 0 || lat[2] + 1 == index.lat_z)
                    for (std::uint32_t c = 0; c < 3; ++c) set.set(base + c, 0.0);
                break;
            case BcKind::BottomPin:
            case BcKind::BottomPin321:
                if (lat[2] != 0) break;
                set.set(base + 2, 0.0);  // bottom face u_z = 0
                if (lat[0] == 0 && lat[1] == 0) {  // corner (0,0,0) pinned
                    set.set(base + 0, 0.0);
                    set.set(base + 1, 0.0);
                }
                if (kind == BcKind::BottomPin321 && lat[0] + 1 == index.lat_x && lat[1] == 0)
                    set.set(base + 1, 0.0);  // removes the rotation about z
                break;
            case BcKind::None:
                break;
        }
    }
    return set;
}

}  // namespace tsvb200
