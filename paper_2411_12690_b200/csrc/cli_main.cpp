// tsvstress_b200: the reference's `local` and `solve` commands (cli.cpp:62-113)
// on the GPU, reading the reference's run configuration (config.cpp) and
// writing its outputs: .rom files (rom.cpp:262-303), the cut-plane
// StressGrid CSV (stress_grid.cpp:36-50) and the JSON-lines run log
// (runlog.cpp:9-19).
//
//   tsvstress_b200 local --config FILE [--threads N] [--device D]
//   tsvstress_b200 solve --config FILE [--out CSV] [--threads N] [--device D] [--precond schwarz2]
//
// Differences from the reference, by design: the global solve is the GPU
// matrix-free PCG (no direct-LDLT fallback: NoConvergence is an error,
// exit 1); `solver.precond` also accepts `schwarz2`; `solver.method = gmres`,
// `bc.type = submodel` and `output.vtk` are outside this path and rejected
// with a message. Everything else -- keys, defaults, validation messages,
// printed lines, file formats -- follows config.cpp / cli.cpp.
#include <sys/resource.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/tsv_b200.h"

namespace {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::string trim(const std::string &s) {
    const size_t a = s.find_first_not_of(" \t\r");
    if (a == std::string::npos) return "";
    const size_t b = s.find_last_not_of(" \t\r");
    return s.substr(a, b - a + 1);
}

[[noreturn]] void bad_key(const std::string &key, const std::string &why) { throw Error("config: " + key + ": " + why); }

// KeyValues (config.cpp:25-140): '#' comments, "key = value", last one wins.
class KeyValues {
public:
    static KeyValues parse_file(const std::string &path) {
        std::ifstream in(path);
        if (!in) throw Error("config: cannot open " + path);
        KeyValues kv;
        std::string line;
        size_t line_no = 0;
        while (std::getline(in, line)) {
            ++line_no;
            const size_t hash = line.find('#');
            if (hash != std::string::npos) line.erase(hash);
            const std::string t = trim(line);
            if (t.empty()) continue;
            const size_t eq = t.find('=');
            if (eq == std::string::npos) throw Error("config: line " + std::to_string(line_no) + " is not 'key = value'");
            const std::string key = trim(t.substr(0, eq));
            if (key.empty()) throw Error("config: empty key on line " + std::to_string(line_no));
            kv.set(key, trim(t.substr(eq + 1)));
        }
        return kv;
    }
    const std::string *find(const std::string &key) const {
        for (const auto &kv : items_)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
    bool has(const std::string &key) const { return find(key) != nullptr; }
    const std::vector<std::pair<std::string, std::string>> &items() const { return items_; }
    double get_double(const std::string &key, std::optional<double> fallback) const {
        const std::string *v = find(key);
        if (!v) {
            if (fallback) return *fallback;
            bad_key(key, "missing required value");
        }
        try {
            size_t pos = 0;
            const double d = std::stod(*v, &pos);
            if (pos == v->size()) return d;
        } catch (const std::exception &) {
        }
        bad_key(key, "'" + *v + "' is not a number");
    }
    long get_int(const std::string &key, std::optional<long> fallback) const {
        const std::string *v = find(key);
        if (!v) {
            if (fallback) return *fallback;
            bad_key(key, "missing required value");
        }
        try {
            size_t pos = 0;
            const long n = std::stol(*v, &pos);
            if (pos == v->size()) return n;
        } catch (const std::exception &) {
        }
        bad_key(key, "'" + *v + "' is not an integer");
    }
    std::string get_string(const std::string &key, const std::string &fallback) const {
        const std::string *v = find(key);
        return v ? *v : fallback;
    }
    std::vector<double> get_double_list(const std::string &key) const {
        const std::string *v = find(key);
        if (!v) bad_key(key, "missing required value");
        std::vector<double> out;
        std::istringstream iss(*v);
        std::string item;
        while (std::getline(iss, item, ',')) {
            item = trim(item);
            if (item.empty()) bad_key(key, "empty list entry");
            try {
                size_t pos = 0;
                out.push_back(std::stod(item, &pos));
                if (pos != item.size()) throw std::invalid_argument("");
            } catch (const std::exception &) {
                bad_key(key, "'" + item + "' is not a number");
            }
        }
        if (out.empty()) bad_key(key, "empty list");
        return out;
    }

private:
    void set(const std::string &key, std::string value) {
        for (auto &kv : items_)
            if (kv.first == key) {
                kv.second = std::move(value);
                return;
            }
        items_.emplace_back(key, std::move(value));
    }
    std::vector<std::pair<std::string, std::string>> items_;
};

const char *const kKnownKeys[] = {
    "geometry.d", "geometry.h", "geometry.t", "geometry.p", "material.copper.e", "material.copper.nu",
    "material.copper.alpha", "material.liner.e", "material.liner.nu", "material.liner.alpha", "material.silicon.e",
    "material.silicon.nu", "material.silicon.alpha", "grid.target", "grid.x", "grid.y", "grid.z", "grid.res",
    "layout.rows", "layout.cols", "layout.kinds", "layout.delta_t", "interpolation.nx", "interpolation.ny",
    "interpolation.nz", "bc.type", "bc.submodel_file", "bc.dummy_rings", "solver.tolerance", "solver.max_iterations",
    "solver.precond", "solver.method", "reference.dof_cap", "superposition.halo", "superposition.cache", "rom.tsv",
    "rom.dummy", "output.grid_csv", "output.vtk", "output.run_log", "threads",
};

// linspace (core.cpp:14-22): n cells, exact end points.
std::vector<double> linspace(double a, double b, size_t n) {
    if (n == 0) throw Error("linspace: need at least one cell");
    std::vector<double> p(n + 1);
    p.front() = a;
    for (size_t i = 1; i < n; ++i) p[i] = a + (b - a) * static_cast<double>(i) / static_cast<double>(n);
    p.back() = b;
    return p;
}

// default_grading (mesh.cpp:31-119): geometric silicon span, uniform liner
// and copper core on the half axis, mirrored; uniform z.
std::vector<double> default_axis_xy(double d, double t, double p, double target) {
    constexpr double kGrowth = 1.5;
    const double c = 0.5 * p, r_in = 0.5 * d, r_out = r_in + t;
    const double a1 = c - r_out, a2 = c - r_in;
    const size_t n_liner = std::max<size_t>(1, static_cast<size_t>(std::ceil(t / target - 1e-12)));
    const double h_liner = t / static_cast<double>(n_liner);
    const double core_h = std::min(target, 0.5 * r_in);
    const size_t n_core = std::max<size_t>(1, static_cast<size_t>(std::ceil(r_in / core_h - 1e-12)));
    const double h0 = std::min(target, kGrowth * h_liner);
    std::vector<double> outer;
    if (a1 <= h0) {
        outer = {a1};
    } else {
        double s = h0, sum = 0.0;
        while (sum < a1) {
            outer.push_back(s);
            sum += s;
            s = std::min(s * kGrowth, target);
        }
        const double scale = a1 / sum;
        for (double &v : outer) v *= scale;
    }
    std::vector<double> half{0.0};
    double pos = 0.0;
    for (size_t i = outer.size(); i > 1; --i) {
        pos += outer[i - 1];
        half.push_back(pos);
    }
    half.push_back(a1);
    for (size_t i = 1; i < n_liner; ++i) half.push_back(a1 + t * static_cast<double>(i) / static_cast<double>(n_liner));
    half.push_back(a2);
    for (size_t i = 1; i < n_core; ++i) half.push_back(a2 + r_in * static_cast<double>(i) / static_cast<double>(n_core));
    half.push_back(c);
    std::vector<double> axis = half;
    for (size_t i = half.size() - 1; i > 0; --i) axis.push_back(p - half[i - 1]);
    return axis;
}

struct RunConfig {  // config.hpp:37-80, the keys local/solve read
    double geom[4] = {5e-6, 50e-6, 0.5e-6, 15e-6};  // d, h, t, p
    double mats[3][3] = {{110e9, 0.35, 17e-6}, {71e9, 0.16, 0.5e-6}, {130e9, 0.28, 2.8e-6}};
    std::vector<double> grid[3];
    uint32_t grid_res = 100, rows = 1, cols = 1, q[3] = {4, 4, 4};
    std::vector<uint8_t> kinds;  // empty = all TSV
    std::vector<double> delta_t{-250.0};
    double tol = 1e-10;
    int max_it = 10000;
    int precond = TSV_PRECOND_DIAGONAL;
    std::string rom_tsv = "tsv.rom", rom_dummy = "dummy.rom", out_csv = "stress_grid.csv", run_log = "run_log.jsonl";
    int threads = 1;

    static RunConfig from_file(const std::string &path) {
        const KeyValues kv = KeyValues::parse_file(path);
        for (const auto &item : kv.items()) {
            bool known = false;
            for (const char *k : kKnownKeys) known |= item.first == k;
            if (!known) bad_key(item.first, "unknown key");
        }
        RunConfig c;
        const char *gk[4] = {"geometry.d", "geometry.h", "geometry.t", "geometry.p"};
        for (int i = 0; i < 4; ++i) c.geom[i] = kv.get_double(gk[i], c.geom[i]);
        if (!(c.geom[0] > 0.0)) bad_key("geometry.d", "must be > 0");
        if (!(c.geom[1] > 0.0)) bad_key("geometry.h", "must be > 0");
        if (!(c.geom[2] > 0.0)) bad_key("geometry.t", "must be > 0");
        if (!(c.geom[0] + 2.0 * c.geom[2] < c.geom[3])) bad_key("geometry.p", "pitch must exceed d + 2t");
        const char *mn[3] = {"material.copper", "material.liner", "material.silicon"};
        for (int m = 0; m < 3; ++m) {
            const std::string pre = mn[m];
            c.mats[m][0] = kv.get_double(pre + ".e", c.mats[m][0]);
            c.mats[m][1] = kv.get_double(pre + ".nu", c.mats[m][1]);
            c.mats[m][2] = kv.get_double(pre + ".alpha", c.mats[m][2]);
            if (!(c.mats[m][0] > 0.0)) bad_key(pre + ".e", "must be > 0");
            if (!(c.mats[m][1] > -1.0 && c.mats[m][1] < 0.5)) bad_key(pre + ".nu", "must lie in (-1, 0.5)");
        }
        const double target = kv.get_double("grid.target", 2e-6);
        if (!(target > 0.0)) bad_key("grid.target", "must be > 0");
        if (kv.has("grid.x") || kv.has("grid.y") || kv.has("grid.z")) {
            if (!(kv.has("grid.x") && kv.has("grid.y") && kv.has("grid.z")))
                bad_key("grid.x", "explicit grids need all of grid.x, grid.y, grid.z");
            const char *ak[3] = {"grid.x", "grid.y", "grid.z"};
            const double ext[3] = {c.geom[3], c.geom[3], c.geom[1]};
            for (int a = 0; a < 3; ++a) {
                std::vector<double> axis = kv.get_double_list(ak[a]);
                if (axis.size() < 2) bad_key(ak[a], "needs at least 2 coordinates");
                if (axis.front() != 0.0 || axis.back() != ext[a])
                    bad_key(ak[a], "must span [0, " + std::to_string(ext[a]) + "] exactly");
                for (size_t i = 1; i < axis.size(); ++i)
                    if (!(axis[i] > axis[i - 1])) bad_key(ak[a], "must be strictly increasing");
                c.grid[a] = std::move(axis);
            }
        } else {
            c.grid[0] = default_axis_xy(c.geom[0], c.geom[2], c.geom[3], target);
            c.grid[1] = c.grid[0];
            c.grid[2] = linspace(0.0, c.geom[1],
                                 std::max<size_t>(1, static_cast<size_t>(std::ceil(c.geom[1] / target - 1e-12))));
        }
        const long res = kv.get_int("grid.res", 100);
        if (res < 1 || res > 4096) bad_key("grid.res", "must lie in [1, 4096]");
        c.grid_res = static_cast<uint32_t>(res);
        const long rows = kv.get_int("layout.rows", 1), cols = kv.get_int("layout.cols", 1);
        if (rows < 1) bad_key("layout.rows", "must be >= 1");
        if (cols < 1) bad_key("layout.cols", "must be >= 1");
        c.rows = static_cast<uint32_t>(rows);
        c.cols = static_cast<uint32_t>(cols);
        c.parse_kinds(kv.get_string("layout.kinds", "tsv"));
        c.parse_delta_t(kv);
        const char *qk[3] = {"interpolation.nx", "interpolation.ny", "interpolation.nz"};
        for (int a = 0; a < 3; ++a) {
            const long n = kv.get_int(qk[a], 4);
            if (n < 2 || n > 64) bad_key(qk[a], "must lie in [2, 64]");
            c.q[a] = static_cast<uint32_t>(n);
        }
        const std::string bc = kv.get_string("bc.type", "clamped");
        if (bc == "submodel") bad_key("bc.type", "submodel boundary fields are outside the GPU online stage (use clamped)");
        if (bc != "clamped") bad_key("bc.type", "'" + bc + "' is not one of clamped|submodel");
        c.tol = kv.get_double("solver.tolerance", 1e-10);
        if (!(c.tol > 0.0)) bad_key("solver.tolerance", "must be > 0");
        const long max_it = kv.get_int("solver.max_iterations", 10000);
        if (max_it < 1) bad_key("solver.max_iterations", "must be >= 1");
        c.max_it = static_cast<int>(max_it);
        c.precond = parse_precond(kv.get_string("solver.precond", "diagonal"));
        const std::string method = kv.get_string("solver.method", "cg");
        if (method == "gmres") bad_key("solver.method", "gmres is outside the GPU online stage (use cg)");
        if (method != "cg") bad_key("solver.method", "'" + method + "' is not one of cg|gmres");
        c.rom_tsv = kv.get_string("rom.tsv", c.rom_tsv);
        c.rom_dummy = kv.get_string("rom.dummy", c.rom_dummy);
        c.out_csv = kv.get_string("output.grid_csv", c.out_csv);
        if (!kv.get_string("output.vtk", "").empty()) bad_key("output.vtk", "VTK output is not produced by tsvstress_b200");
        c.run_log = kv.get_string("output.run_log", c.run_log);
        const long threads = kv.get_int("threads", 1);
        if (threads < 1 || threads > 256) bad_key("threads", "must lie in [1, 256]");
        c.threads = static_cast<int>(threads);
        return c;
    }

    static int parse_precond(const std::string &p) {
        if (p == "none") return TSV_PRECOND_NONE;
        if (p == "diagonal") return TSV_PRECOND_DIAGONAL;
        if (p == "block") return TSV_PRECOND_BLOCK_DIAGONAL;
        if (p == "schwarz2") return TSV_PRECOND_SCHWARZ2;
        bad_key("solver.precond", "'" + p + "' is not one of none|diagonal|block|schwarz2");
    }

    void parse_kinds(const std::string &text) {  // config.cpp:164-193
        const std::string key = "layout.kinds";
        if (text == "tsv") return;
        if (text == "dummy") {
            kinds.assign(static_cast<size_t>(rows) * cols, 1);
            return;
        }
        std::vector<std::string> rs;
        std::istringstream iss(text);
        std::string r;
        while (std::getline(iss, r, ';')) rs.push_back(trim(r));
        if (rs.size() != rows)
            bad_key(key, "pattern has " + std::to_string(rs.size()) + " rows, layout has " + std::to_string(rows));
        for (const std::string &row : rs) {
            if (row.size() != cols) bad_key(key, "pattern row '" + row + "' does not have " + std::to_string(cols) + " cells");
            for (char ch : row) {
                if (ch == 't') kinds.push_back(0);
                else if (ch == 'd') kinds.push_back(1);
                else bad_key(key, std::string("unknown cell kind '") + ch + "' (use 't' or 'd')");
            }
        }
    }

    void parse_delta_t(const KeyValues &kv) {  // config.cpp:195-222
        const std::string key = "layout.delta_t";
        const std::string *v = kv.find(key);
        if (!v) return;
        if (v->find(';') == std::string::npos && v->find(',') == std::string::npos) {
            delta_t = {kv.get_double(key, std::nullopt)};
            return;
        }
        delta_t.clear();
        std::istringstream iss(*v);
        std::string row;
        size_t n_rows = 0;
        while (std::getline(iss, row, ';')) {
            ++n_rows;
            std::istringstream riss(row);
            std::string item;
            size_t n_cols = 0;
            while (std::getline(riss, item, ',')) {
                ++n_cols;
                try {
                    delta_t.push_back(std::stod(trim(item)));
                } catch (const std::exception &) {
                    bad_key(key, "'" + trim(item) + "' is not a number");
                }
            }
            if (n_cols != cols) bad_key(key, "each row needs " + std::to_string(cols) + " values");
        }
        if (n_rows != rows) bad_key(key, "needs " + std::to_string(rows) + " rows");
    }

    bool any_kind(uint8_t k) const {
        if (kinds.empty()) return k == 0;
        return std::find(kinds.begin(), kinds.end(), k) != kinds.end();
    }

    tsv_local_desc local_desc(int kind) const {
        tsv_local_desc d{};
        for (int a = 0; a < 3; ++a) {
            d.q[a] = q[a];
            d.grid_len[a] = static_cast<uint32_t>(grid[a].size());
            d.grid[a] = grid[a].data();
        }
        for (int i = 0; i < 4; ++i) d.geometry[i] = geom[i];
        for (int m = 0; m < 3; ++m)
            for (int k = 0; k < 3; ++k) d.materials[m][k] = mats[m][k];
        d.kind = kind;
        return d;
    }
};

std::string hash_hex(const uint8_t *h) {
    static const char *digits = "0123456789abcdef";
    std::string s;
    for (int i = 0; i < 32; ++i) {
        s.push_back(digits[h[i] >> 4]);
        s.push_back(digits[h[i] & 0xf]);
    }
    return s;
}

size_t peak_rss_bytes() {  // core.cpp:127-145
    size_t peak = 0;
    rusage ru{};
    if (getrusage(RUSAGE_SELF, &ru) == 0) peak = static_cast<size_t>(ru.ru_maxrss) * 1024;
    std::ifstream status("/proc/self/status");
    std::string line;
    while (std::getline(status, line))
        if (line.rfind("VmHWM:", 0) == 0) {
            std::istringstream iss(line.substr(6));
            size_t kb = 0;
            if (iss >> kb) peak = std::max(peak, kb * 1024);
        }
    return peak;
}

std::string json_number(double v) {  // shortest round trip, as nlohmann::json::dump
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

// append_run_log (runlog.cpp:9-19); keys in nlohmann's (sorted) order.
void append_run_log(const std::string &path, const std::string &command, double wall_s, size_t peak, size_t dofs,
                    int iterations) {
    std::ofstream out(path, std::ios::app);
    if (!out) throw Error("run log: cannot open " + path);
    out << "{\"command\":\"" << command << "\",\"dofs\":" << dofs << ",\"iterations\":" << iterations
        << ",\"peak_mem_bytes\":" << peak << ",\"wall_s\":" << json_number(wall_s) << "}\n";
    if (!out) throw Error("run log: write failed for " + path);
}

// StressGrid::save_csv (stress_grid.cpp:36-50).
void save_csv(const std::string &path, uint32_t rows, uint32_t cols, uint32_t res, double pitch,
              const std::vector<double> &values) {
    std::FILE *f = std::fopen(path.c_str(), "wb");
    if (!f) throw Error("StressGrid: cannot open " + path);
    std::fputs("block_row,block_col,px,py,x,y,von_mises\n", f);
    auto local = [&](uint32_t q) { return (static_cast<double>(q) + 0.5) * pitch / static_cast<double>(res); };
    for (uint32_t r = 0; r < rows; ++r)
        for (uint32_t c = 0; c < cols; ++c)
            for (uint32_t py = 0; py < res; ++py)
                for (uint32_t px = 0; px < res; ++px) {
                    const double x = static_cast<double>(c) * pitch + local(px);
                    const double y = static_cast<double>(r) * pitch + local(py);
                    std::fprintf(f, "%" PRIu32 ",%" PRIu32 ",%" PRIu32 ",%" PRIu32 ",%.17g,%.17g,%.17g\n", r, c, px, py, x,
                                 y, values[((static_cast<size_t>(r) * cols + c) * res + py) * res + px]);
                }
    if (std::fclose(f) != 0) throw Error("StressGrid: write failed for " + path);
}

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

void check(tsv_ctx *ctx, int rc) {
    if (rc != TSV_OK) throw Error(ctx ? tsv_last_error(ctx) : "device error");
}

int cmd_local(const RunConfig &cfg, int device) {  // cli.cpp:62-88
    const auto t0 = Clock::now();
    uint64_t n = 0, n_fine = 0, cells = 0;
    tsv_local_desc d0 = cfg.local_desc(0);
    if (tsv_rom_dims(&d0, &n, &n_fine, &cells) != TSV_OK) throw Error("local: invalid grid / interpolation layout");
    std::printf("n = %" PRIu64 "\n", n);
    for (int kind = 0; kind < 2; ++kind) {
        if (kind == 1 && !cfg.any_kind(1)) continue;
        tsv_local_desc d = cfg.local_desc(kind);
        std::vector<double> K(n * n), b(n), phi(n_fine * n), ut(n_fine);
        std::vector<uint8_t> em(cells);
        tsv_rom_out out{};
        out.a_element = K.data();
        out.b_element = b.data();
        out.basis = phi.data();
        out.thermal = ut.data();
        out.element_material = em.data();
        char err[512];
        if (tsv_build_rom(device, &d, &out, err, sizeof err) != TSV_OK) throw Error(err);
        tsv_rom_desc rd{};
        for (int a = 0; a < 3; ++a) {
            rd.q[a] = d.q[a];
            rd.grid_len[a] = d.grid_len[a];
            rd.grid[a] = d.grid[a];
        }
        for (int i = 0; i < 4; ++i) rd.geometry[i] = d.geometry[i];
        std::memcpy(rd.materials, d.materials, sizeof rd.materials);
        rd.element_material = em.data();
        rd.a_element = K.data();
        rd.b_element = b.data();
        rd.basis = phi.data();
        rd.thermal = ut.data();
        std::memcpy(rd.fingerprint, out.fingerprint, 32);
        const std::string &path = kind ? cfg.rom_dummy : cfg.rom_tsv;
        if (tsv_save_rom_file(&rd, kind, path.c_str(), err, sizeof err) != TSV_OK) throw Error(err);
        std::printf("wrote %s\n", path.c_str());
    }
    const double wall = seconds_since(t0);
    std::printf("local stage: %.3f s\n", wall);
    append_run_log(cfg.run_log, "local", wall, peak_rss_bytes(), n_fine, 0);
    return 0;
}

int cmd_solve(const RunConfig &cfg, int device) {  // cli.cpp:90-113
    tsv_local_desc d0 = cfg.local_desc(0);
    uint8_t expected[32];
    check(nullptr, tsv_rom_fingerprint(&d0, expected));
    // load_roms (cli.cpp:31-53): the kinds the layout uses, fingerprints checked against the config
    for (int kind = 0; kind < 2; ++kind) {
        if (!cfg.any_kind(static_cast<uint8_t>(kind))) continue;
        const std::string &path = kind ? cfg.rom_dummy : cfg.rom_tsv;
        char err[512];
        int file_kind = -1;
        uint8_t fp[32];
        if (tsv_rom_file_info(path.c_str(), &file_kind, fp, err, sizeof err) != TSV_OK) throw Error(err);
        if (std::memcmp(fp, expected, 32) != 0)
            throw Error("ROM " + path + " was built for a different configuration (fingerprint " + hash_hex(fp) +
                        ", config expects " + hash_hex(expected) + ")");
    }
    tsv_ctx *ctx = nullptr;
    if (tsv_ctx_create(device, &ctx) != TSV_OK) throw Error("cannot create a GPU context on device " + std::to_string(device));
    struct Guard {
        tsv_ctx *c;
        ~Guard() { tsv_ctx_destroy(c); }
    } guard{ctx};
    for (int kind = 0; kind < 2; ++kind) {
        if (!cfg.any_kind(static_cast<uint8_t>(kind))) continue;
        const std::string &path = kind ? cfg.rom_dummy : cfg.rom_tsv;
        char err[512];
        int file_kind = -1;
        if (tsv_load_rom_file(ctx, kind, path.c_str(), &file_kind, err, sizeof err) != TSV_OK) throw Error(err);
    }
    const auto t0 = Clock::now();
    const size_t B = static_cast<size_t>(cfg.rows) * cfg.cols;
    check(ctx, tsv_set_layout(ctx, cfg.rows, cfg.cols, cfg.kinds.empty() ? nullptr : cfg.kinds.data(), cfg.delta_t.data(),
                              cfg.delta_t.size(), cfg.geom[3], cfg.geom[1]));
    check(ctx, tsv_set_bc(ctx, TSV_BC_CLAMPED));
    uint64_t dofs = 0;
    check(ctx, tsv_get_index(ctx, &dofs, nullptr, nullptr, nullptr));
    tsv_iter_options opts{cfg.tol, cfg.max_it, cfg.precond};
    tsv_solve_info info{};
    const int rc = tsv_solve(ctx, &opts, nullptr, &info);
    if (rc == TSV_ENOCONV)
        throw Error(std::string(tsv_last_error(ctx)) + " (no direct fallback on the GPU path; raise solver.max_iterations or use schwarz2)");
    check(ctx, rc);
    std::vector<double> grid(B * cfg.grid_res * cfg.grid_res);
    check(ctx, tsv_cutplane(ctx, cfg.grid_res, grid.data()));
    const double wall = seconds_since(t0);
    save_csv(cfg.out_csv, cfg.rows, cfg.cols, cfg.grid_res, cfg.geom[3], grid);
    std::printf("reduced dofs = %" PRIu64 ", iterations = %d, residual = %.3e%s\n", dofs, info.iterations,
                info.relative_residual, info.direct_fallback ? " (direct fallback)" : "");
    std::printf("global stage: %.3f s, wrote %s\n", wall, cfg.out_csv.c_str());
    append_run_log(cfg.run_log, "solve", wall, peak_rss_bytes(), dofs, info.iterations);
    return 0;
}

int cmd_grid(const RunConfig &cfg) {  // prints the configured TensorGrid (test hook)
    const char *names[3] = {"x", "y", "z"};
    for (int a = 0; a < 3; ++a) {
        std::printf("%s", names[a]);
        for (double v : cfg.grid[a]) std::printf(" %.17g", v);
        std::printf("\n");
    }
    uint8_t fp[32];
    tsv_local_desc d = cfg.local_desc(0);
    if (tsv_rom_fingerprint(&d, fp) == TSV_OK) std::printf("fingerprint %s\n", hash_hex(fp).c_str());
    return 0;
}

int usage() {
    std::fprintf(stderr,
                 "usage: tsvstress_b200 local --config FILE [--threads N] [--device D]\n"
                 "       tsvstress_b200 solve --config FILE [--out CSV] [--threads N] [--device D] [--precond P]\n");
    return 1;
}

}  // namespace

int main(int argc, char **argv) {
    if (argc < 2) return usage();
    const std::string sub = argv[1];
    if (sub != "local" && sub != "solve" && sub != "grid") return usage();
    std::string config_path, out_override, precond_override;
    int threads_override = 0, device = 0;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto value = [&]() -> std::string {
            if (i + 1 >= argc) throw Error(a + " needs a value");
            return argv[++i];
        };
        try {
            if (a == "--config") config_path = value();
            else if (a == "--out") out_override = value();
            else if (a == "--threads") threads_override = std::stoi(value());
            else if (a == "--device") device = std::stoi(value());
            else if (a == "--precond") precond_override = value();
            else return usage();
        } catch (const std::exception &e) {
            std::fprintf(stderr, "error: %s\n", e.what());
            return 1;
        }
    }
    if (config_path.empty()) return usage();
    try {
        RunConfig cfg = RunConfig::from_file(config_path);
        if (!out_override.empty()) cfg.out_csv = out_override;
        if (threads_override > 0) cfg.threads = threads_override;
        if (!precond_override.empty()) cfg.precond = RunConfig::parse_precond(precond_override);
        if (sub == "grid") return cmd_grid(cfg);
        return sub == "local" ? cmd_local(cfg, device) : cmd_solve(cfg, device);
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
