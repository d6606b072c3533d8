// Direct ingest of the reference's ".rom" files (MRST v1, little endian,
// rom.cpp:257-377) into a GPU context, and the matching writer: the
// one-shot local stage and the online stage exchange ROMs through files
// exactly as tsvstress's `local` / `solve` commands do (cli.cpp:31-54).
//
//   magic "MRST" | u32 version = 1 | u8 kind | header | sha256(header) | body
//   header: f64 d,h,t,p | 3 x (u32 len, f64[len]) grid | 3 x (u8 id, f64 E, nu, alpha) | u32 nx, ny, nz
//   body:   basis column-major [n][n_fine] | thermal [n_fine] | a_element [n*n] | b_element [n]
#include <openssl/sha.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tsv_b200.h"

namespace {

struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class Reader {
public:
    Reader(const std::string &data, std::string origin) : d_(data), origin_(std::move(origin)) {}
    template <typename T>
    T get() {
        need(sizeof(T));
        T v;
        std::memcpy(&v, d_.data() + pos_, sizeof(T));
        pos_ += sizeof(T);
        return v;
    }
    void bytes(void *out, size_t n) {
        need(n);
        std::memcpy(out, d_.data() + pos_, n);
        pos_ += n;
    }
    size_t pos() const { return pos_; }
    size_t remaining() const { return d_.size() - pos_; }

private:
    void need(size_t n) {
        if (d_.size() - pos_ < n) throw IoError(origin_ + ": truncated file");
    }
    const std::string &d_;
    std::string origin_;
    size_t pos_ = 0;
};

struct LoadedRom {
    int kind = 0;
    tsv_rom_desc desc{};
    std::vector<double> grid[3], basis, thermal, a_element, b_element;
};

LoadedRom parse(const std::string &path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("load_rom: cannot open " + path);
    const std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    Reader r(data, "load_rom(" + path + ")");
    char magic[4];
    r.bytes(magic, 4);
    if (std::memcmp(magic, "MRST", 4) != 0) throw IoError("load_rom: " + path + " is not a ROM file (bad magic)");
    const uint32_t version = r.get<uint32_t>();
    if (version != 1)
        throw IoError("load_rom: " + path + " has unsupported format version " + std::to_string(version));
    LoadedRom m;
    const uint8_t kind = r.get<uint8_t>();
    if (kind > 1) throw IoError("load_rom: invalid block kind byte");
    m.kind = kind;
    const size_t header_begin = r.pos();
    for (int i = 0; i < 4; ++i) m.desc.geometry[i] = r.get<double>();
    for (int a = 0; a < 3; ++a) {
        const uint32_t len = r.get<uint32_t>();
        if (len < 2 || len > 100000000u) throw IoError("load_rom: corrupt grid axis length");
        m.grid[a].resize(len);
        r.bytes(m.grid[a].data(), len * sizeof(double));
    }
    for (uint8_t id = 0; id < 3; ++id) {
        if (r.get<uint8_t>() != id) throw IoError("load_rom: material table out of order");
        for (int k = 0; k < 3; ++k) m.desc.materials[id][k] = r.get<double>();
    }
    for (int a = 0; a < 3; ++a) m.desc.q[a] = r.get<uint32_t>();
    const size_t header_end = r.pos();
    unsigned char stored[32], computed[32];
    r.bytes(stored, 32);
    SHA256(reinterpret_cast<const unsigned char *>(data.data()) + header_begin, header_end - header_begin, computed);
    if (std::memcmp(stored, computed, 32) != 0)
        throw IoError("load_rom: " + path + " fingerprint does not match its header (corrupt file)");
    std::memcpy(m.desc.fingerprint, stored, 32);
    for (int a = 0; a < 3; ++a)
        if (m.desc.q[a] < 2) throw IoError("NodeLayout: need at least 2 interpolation nodes per axis");
    const size_t nf = 3 * m.grid[0].size() * m.grid[1].size() * m.grid[2].size();
    const size_t all = static_cast<size_t>(m.desc.q[0]) * m.desc.q[1] * m.desc.q[2];
    const size_t inner = static_cast<size_t>(m.desc.q[0] - 2) * (m.desc.q[1] - 2) * (m.desc.q[2] - 2);
    const size_t n = 3 * (all - inner);
    const size_t body = (nf * n + nf + n * n + n) * sizeof(double);
    if (r.remaining() != body)
        throw IoError("load_rom: " + path + ": corrupt length (body is " + std::to_string(r.remaining()) +
                      " bytes, expected " + std::to_string(body) + ")");
    m.basis.resize(nf * n);
    std::vector<double> col(nf);
    for (size_t i = 0; i < n; ++i) {  // column-major on disk -> row-major
        r.bytes(col.data(), nf * sizeof(double));
        for (size_t f = 0; f < nf; ++f) m.basis[f * n + i] = col[f];
    }
    m.thermal.resize(nf);
    r.bytes(m.thermal.data(), nf * sizeof(double));
    m.a_element.resize(n * n);
    r.bytes(m.a_element.data(), n * n * sizeof(double));
    m.b_element.resize(n);
    r.bytes(m.b_element.data(), n * sizeof(double));
    for (int a = 0; a < 3; ++a) {
        m.desc.grid_len[a] = static_cast<uint32_t>(m.grid[a].size());
        m.desc.grid[a] = m.grid[a].data();
    }
    m.desc.element_material = nullptr;  // rebuilt from the geometry (BlockMeshes::from)
    m.desc.basis = m.basis.data();
    m.desc.thermal = m.thermal.data();
    m.desc.a_element = m.a_element.data();
    m.desc.b_element = m.b_element.data();
    return m;
}

template <typename T>
void put(std::string &s, T v) {
    s.append(reinterpret_cast<const char *>(&v), sizeof(T));
}

// rom_fingerprint's byte stream (rom.cpp:110-132), also the .rom header.
std::string header_bytes(const double geometry[4], const uint32_t grid_len[3], const double *const grid[3],
                         const double materials[3][3], const uint32_t q[3]) {
    std::string header;
    for (int i = 0; i < 4; ++i) put(header, geometry[i]);
    for (int a = 0; a < 3; ++a) {
        put(header, grid_len[a]);
        header.append(reinterpret_cast<const char *>(grid[a]), grid_len[a] * sizeof(double));
    }
    for (uint8_t id = 0; id < 3; ++id) {
        put(header, id);
        for (int k = 0; k < 3; ++k) put(header, materials[id][k]);
    }
    for (int a = 0; a < 3; ++a) put(header, q[a]);
    return header;
}

}  // namespace

extern "C" {

int tsv_load_rom_file(tsv_ctx *ctx, int slot, const char *path, int *kind_out, char *err, size_t err_len) {
    try {
        LoadedRom m = parse(path ? path : "");
        if (kind_out) *kind_out = m.kind;
        const int rc = tsv_set_rom(ctx, slot < 0 ? m.kind : slot, &m.desc);
        if (rc != TSV_OK && err && err_len) std::snprintf(err, err_len, "%s", tsv_last_error(ctx));
        else if (err && err_len) err[0] = 0;
        return rc;
    } catch (const std::exception &e) {
        if (err && err_len) std::snprintf(err, err_len, "%s", e.what());
        return TSV_EINVAL;
    }
}

int tsv_rom_fingerprint(const tsv_local_desc *d, uint8_t out[32]) {
    if (!d || !out) return TSV_EINVAL;
    for (int a = 0; a < 3; ++a)
        if (!d->grid[a] || d->grid_len[a] < 2) return TSV_EINVAL;
    const std::string h = header_bytes(d->geometry, d->grid_len, d->grid, d->materials, d->q);
    SHA256(reinterpret_cast<const unsigned char *>(h.data()), h.size(), out);
    return TSV_OK;
}

int tsv_rom_file_info(const char *path, int *kind_out, uint8_t fingerprint[32], char *err, size_t err_len) {
    try {
        LoadedRom m = parse(path ? path : "");
        if (kind_out) *kind_out = m.kind;
        if (fingerprint) std::memcpy(fingerprint, m.desc.fingerprint, 32);
        if (err && err_len) err[0] = 0;
        return TSV_OK;
    } catch (const std::exception &e) {
        if (err && err_len) std::snprintf(err, err_len, "%s", e.what());
        return TSV_EINVAL;
    }
}

int tsv_save_rom_file(const tsv_rom_desc *d, int kind, const char *path, char *err, size_t err_len) {
    try {
        if (!d || !path) throw IoError("save_rom: NULL argument");
        const std::string header = header_bytes(d->geometry, d->grid_len, d->grid, d->materials, d->q);
        unsigned char fp[32];
        SHA256(reinterpret_cast<const unsigned char *>(header.data()), header.size(), fp);
        const size_t nf = 3ull * d->grid_len[0] * d->grid_len[1] * d->grid_len[2];
        const size_t all = static_cast<size_t>(d->q[0]) * d->q[1] * d->q[2];
        const size_t inner = static_cast<size_t>(d->q[0] - 2) * (d->q[1] - 2) * (d->q[2] - 2);
        const size_t n = 3 * (all - inner);
        std::FILE *f = std::fopen(path, "wb");
        if (!f) throw IoError(std::string("save_rom: cannot open ") + path);
        std::string head = "MRST";
        put(head, uint32_t{1});
        put(head, static_cast<uint8_t>(kind));
        head += header;
        head.append(reinterpret_cast<const char *>(fp), 32);
        bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size();
        std::vector<double> col(nf);
        for (size_t i = 0; i < n && ok; ++i) {  // basis column-major
            for (size_t fi = 0; fi < nf; ++fi) col[fi] = d->basis[fi * n + i];
            ok = std::fwrite(col.data(), sizeof(double), nf, f) == nf;
        }
        ok = ok && std::fwrite(d->thermal, sizeof(double), nf, f) == nf;
        ok = ok && std::fwrite(d->a_element, sizeof(double), n * n, f) == n * n;
        ok = ok && std::fwrite(d->b_element, sizeof(double), n, f) == n;
        if (std::fclose(f) != 0 || !ok) throw IoError(std::string("save_rom: write failed for ") + path);
        if (err && err_len) err[0] = 0;
        return TSV_OK;
    } catch (const std::exception &e) {
        if (err && err_len) std::snprintf(err, err_len, "%s", e.what());
        return TSV_EINVAL;
    }
}

}  // extern "C"
