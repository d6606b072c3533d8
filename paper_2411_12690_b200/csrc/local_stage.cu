// One-shot local stage on the GPU: the reduced-order model of one unit
// block (rom::build_rom, rom.cpp:134-253), restated for B200. It produces
// the hot path's INPUTS (K_r, b_el, Phi, u_T); it is timed separately and
// is not part of the online-stage metric (BASELINE.json north_star).
//
//   element matrices    fem.cpp:82-126 (2x2x2 Gauss, generic Jacobian)     host
//   interpolation W     rom.cpp:67-108 (tensor Lagrange on surface nodes)  host
//   A_ii assembly       dense, 8-colour conflict-free element scatter      GPU
//   A_ii X = rhs        Cholesky of the interior block (cuSOLVER potrf/s)  GPU
//   Phi, u_T            interior rows from X, boundary rows = W exactly     GPU
//   K_r = Phi^T A Phi   element-wise A*Phi (colour scatter) + DGEMM         GPU
//   b_el = Phi^T b      DGEMV                                              GPU
//
// The reference factors the full lifted matrix with unit rows on the
// boundary (rom.cpp:186-193); eliminating those rows first gives the same
// interior system, so only the interior block is factored here.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <openssl/sha.h>

#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tsv_b200.h"

namespace {

struct LsError : std::runtime_error {
    LsError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
    int code;
};

#define LCK(expr)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw LsError(e_ == cudaErrorMemoryAllocation ? TSV_ENOMEM : TSV_ECUDA,                \
                          std::string(#expr) + ": " + cudaGetErrorString(e_));                     \
    } while (0)
#define LCS(expr)                                                                                  \
    do {                                                                                           \
        int s_ = static_cast<int>(expr);                                                           \
        if (s_ != 0) throw LsError(TSV_ECUDA, std::string(#expr) + " failed with status " + std::to_string(s_)); \
    } while (0)

template <typename T>
struct Dev {
    T *p = nullptr;
    explicit Dev(size_t n) { LCK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev &) = delete;
    Dev &operator=(const Dev &) = delete;
};

constexpr double kXi[8] = {-1, 1, 1, -1, -1, 1, 1, -1};
constexpr double kEta[8] = {-1, -1, 1, 1, -1, -1, 1, 1};
constexpr double kZeta[8] = {-1, -1, -1, -1, 1, 1, 1, 1};

// physical_gradients (fem.cpp:27-58): returns det J.
double phys_grad(const double c[8][3], double xi, double eta, double zeta, double g[8][3]) {
    double dn[8][3];
    for (int a = 0; a < 8; ++a) {
        dn[a][0] = 0.125 * kXi[a] * (1.0 + kEta[a] * eta) * (1.0 + kZeta[a] * zeta);
        dn[a][1] = 0.125 * kEta[a] * (1.0 + kXi[a] * xi) * (1.0 + kZeta[a] * zeta);
        dn[a][2] = 0.125 * kZeta[a] * (1.0 + kXi[a] * xi) * (1.0 + kEta[a] * eta);
    }
    double j[3][3] = {};
    for (int a = 0; a < 8; ++a)
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) j[r][k] += dn[a][r] * c[a][k];
    const double det = j[0][0] * (j[1][1] * j[2][2] - j[1][2] * j[2][1]) -
                       j[0][1] * (j[1][0] * j[2][2] - j[1][2] * j[2][0]) +
                       j[0][2] * (j[1][0] * j[2][1] - j[1][1] * j[2][0]);
    if (!(det > 0.0)) throw LsError(TSV_EINVAL, "element: degenerate hexahedron (non-positive Jacobian)");
    double inv[3][3];
    inv[0][0] = (j[1][1] * j[2][2] - j[1][2] * j[2][1]) / det;
    inv[0][1] = (j[0][2] * j[2][1] - j[0][1] * j[2][2]) / det;
    inv[0][2] = (j[0][1] * j[1][2] - j[0][2] * j[1][1]) / det;
    inv[1][0] = (j[1][2] * j[2][0] - j[1][0] * j[2][2]) / det;
    inv[1][1] = (j[0][0] * j[2][2] - j[0][2] * j[2][0]) / det;
    inv[1][2] = (j[0][2] * j[1][0] - j[0][0] * j[1][2]) / det;
    inv[2][0] = (j[1][0] * j[2][1] - j[1][1] * j[2][0]) / det;
    inv[2][1] = (j[0][1] * j[2][0] - j[0][0] * j[2][1]) / det;
    inv[2][2] = (j[0][0] * j[1][1] - j[0][1] * j[1][0]) / det;
    for (int a = 0; a < 8; ++a)
        for (int i = 0; i < 3; ++i) g[a][i] = inv[0][i] * dn[a][0] + inv[1][i] * dn[a][1] + inv[2][i] * dn[a][2];
    return det;
}

// element_stiffness + element_thermal_load (fem.cpp:82-126).
void element_matrices(const double c[8][3], double lambda, double mu, double alpha, double *k, double *f) {
    std::memset(k, 0, 576 * sizeof(double));
    std::memset(f, 0, 24 * sizeof(double));
    const double gp = 1.0 / std::sqrt(3.0);
    const double coef = alpha * (3.0 * lambda + 2.0 * mu);
    double g[8][3];
    for (int gx = 0; gx < 2; ++gx)
        for (int gy = 0; gy < 2; ++gy)
            for (int gz = 0; gz < 2; ++gz) {
                const double w = phys_grad(c, gx ? gp : -gp, gy ? gp : -gp, gz ? gp : -gp, g);
                for (int a = 0; a < 8; ++a) {
                    for (int b = 0; b < 8; ++b) {
                        const double gg = g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2];
                        for (int i = 0; i < 3; ++i)
                            for (int j = 0; j < 3; ++j) {
                                double v = lambda * g[a][i] * g[b][j] + mu * g[a][j] * g[b][i];
                                if (i == j) v += mu * gg;
                                k[(3 * a + i) * 24 + 3 * b + j] += w * v;
                            }
                    }
                    for (int i = 0; i < 3; ++i) f[3 * a + i] += w * coef * g[a][i];
                }
            }
}

double lagrange_1d(const std::vector<double> &nodes, size_t i, double x) {  // rom.cpp:48-58
    double w = 1.0;
    for (size_t m = 0; m < nodes.size(); ++m) {
        if (m == i) continue;
        w *= (x - nodes[m]) / (nodes[i] - nodes[m]);
    }
    return w;
}

std::vector<double> linspace(double a, double b, size_t cells) {  // core.cpp:14-22
    std::vector<double> p(cells + 1);
    p.front() = a;
    for (size_t i = 1; i < cells; ++i) p[i] = a + (b - a) * static_cast<double>(i) / static_cast<double>(cells);
    p.back() = b;
    return p;
}

// ------------------------------------------------------------- kernels
// Dense interior block, column-major: A[is * ni + ir] += K_e[r][s].
__global__ void assemble_interior_kernel(int n_elems, const int *elems, const double *ke, const int *int_of_dof,
                                         const int *elem_dofs, double *A, long long ni) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int el = t / 576, rs = t % 576;
    if (el >= n_elems) return;
    const int e = elems[el];
    const int r = rs / 24, s = rs % 24;
    const int ir = int_of_dof[elem_dofs[e * 24 + r]];
    const int is = int_of_dof[elem_dofs[e * 24 + s]];
    if (ir < 0 || is < 0) return;
    A[static_cast<long long>(is) * ni + ir] += ke[static_cast<long long>(e) * 576 + rs];
}

// A*Phi (unlifted) by elements of one colour: APhi[dof_r][a] += sum_s K_e[r][s] Phi[dof_s][a].
__global__ void element_aphi_kernel(int n_elems, const int *elems, const double *ke, const int *elem_dofs,
                                    const double *phi, double *aphi, int n) {
    const int el = blockIdx.y;
    if (el >= n_elems) return;
    const int e = elems[el];
    __shared__ double k[576];
    __shared__ int dofs[24];
    for (int i = threadIdx.x; i < 576; i += blockDim.x) k[i] = ke[static_cast<long long>(e) * 576 + i];
    if (threadIdx.x < 24) dofs[threadIdx.x] = elem_dofs[e * 24 + threadIdx.x];
    __syncthreads();
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    double col[24];
#pragma unroll
    for (int s = 0; s < 24; ++s) col[s] = phi[static_cast<long long>(dofs[s]) * n + a];
#pragma unroll 4
    for (int r = 0; r < 24; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < 24; ++s) acc += k[r * 24 + s] * col[s];
        aphi[static_cast<long long>(dofs[r]) * n + a] += acc;
    }
}

// Phi rows of interior DoFs from the column-major solution X (ni x (n+1)).
__global__ void scatter_solution_kernel(int ni, int n, const int *dof_of_int, const double *X, double *phi,
                                        double *thermal) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<long long>(ni) * (n + 1)) return;
    const int a = static_cast<int>(t / ni), ir = static_cast<int>(t % ni);
    const int dof = dof_of_int[ir];
    const double v = X[t];
    if (a < n) phi[static_cast<long long>(dof) * n + a] = v;
    else thermal[dof] = v;
}

void sha256_fingerprint(const tsv_local_desc *d, uint8_t out[32]) {  // rom_fingerprint, rom.cpp:110-132
    std::string buf;
    auto f64 = [&](double v) {
        uint64_t u;
        std::memcpy(&u, &v, 8);
        for (int i = 0; i < 8; ++i) buf.push_back(static_cast<char>((u >> (8 * i)) & 0xff));
    };
    auto u32 = [&](uint32_t v) {
        for (int i = 0; i < 4; ++i) buf.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
    };
    for (int i = 0; i < 4; ++i) f64(d->geometry[i]);
    for (int a = 0; a < 3; ++a) {
        u32(d->grid_len[a]);
        for (uint32_t i = 0; i < d->grid_len[a]; ++i) f64(d->grid[a][i]);
    }
    for (uint8_t id = 0; id < 3; ++id) {
        buf.push_back(static_cast<char>(id));
        for (int k = 0; k < 3; ++k) f64(d->materials[id][k]);
    }
    for (int a = 0; a < 3; ++a) u32(d->q[a]);
    SHA256(reinterpret_cast<const unsigned char *>(buf.data()), buf.size(), out);
}

struct Dims {
    size_t n, n_fine, cells, nx, ny, nz;
};

Dims dims_of(const tsv_local_desc *d) {
    if (!d) throw LsError(TSV_EINVAL, "build_rom: NULL descriptor");
    for (int a = 0; a < 3; ++a) {
        if (d->q[a] < 2) throw LsError(TSV_EINVAL, "NodeLayout: need at least 2 interpolation nodes per axis");
        if (d->grid_len[a] < 2 || !d->grid[a]) throw LsError(TSV_EINVAL, "grid: axis needs at least 2 lines");
    }
    Dims r{};
    r.nx = d->grid_len[0];
    r.ny = d->grid_len[1];
    r.nz = d->grid_len[2];
    const size_t all = static_cast<size_t>(d->q[0]) * d->q[1] * d->q[2];
    const size_t inner = static_cast<size_t>(d->q[0] - 2) * (d->q[1] - 2) * (d->q[2] - 2);
    r.n = 3 * (all - inner);
    r.n_fine = 3 * r.nx * r.ny * r.nz;
    r.cells = (r.nx - 1) * (r.ny - 1) * (r.nz - 1);
    return r;
}

void build(int device, const tsv_local_desc *d, tsv_rom_out *out) {
    const auto t0 = std::chrono::steady_clock::now();
    const Dims D = dims_of(d);
    const double dd = d->geometry[0], hh = d->geometry[1], tt = d->geometry[2], pp = d->geometry[3];
    // UnitBlockGeometry::validate (mesh.cpp:8-15) and TensorGrid::validate (:16-28)
    if (!(dd > 0.0) || !(tt > 0.0) || !(hh > 0.0) || !(dd + 2.0 * tt < pp))
        throw LsError(TSV_EINVAL, "geometry: invalid d/t/h/p");
    const double ext[3] = {pp, pp, hh};
    std::vector<double> grid[3];
    for (int a = 0; a < 3; ++a) {
        grid[a].assign(d->grid[a], d->grid[a] + d->grid_len[a]);
        if (grid[a].front() != 0.0 || grid[a].back() != ext[a])
            throw LsError(TSV_EINVAL, "grid: axis must span [0, extent] exactly");
        for (size_t i = 1; i < grid[a].size(); ++i)
            if (!(grid[a][i] > grid[a][i - 1])) throw LsError(TSV_EINVAL, "grid: axis must be strictly increasing");
    }
    double lame[3][3];
    for (int i = 0; i < 3; ++i) {
        const double E = d->materials[i][0], nu = d->materials[i][1];
        if (!(E > 0.0) || !(nu > -1.0) || !(nu < 0.5)) throw LsError(TSV_EINVAL, "material: invalid E or nu");
        lame[i][0] = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
        lame[i][1] = E / (2.0 * (1.0 + nu));
        lame[i][2] = d->materials[i][2];
    }
    const size_t nx = D.nx, ny = D.ny, nz = D.nz, cx = nx - 1, cy = ny - 1, cz = nz - 1;
    const size_t n = D.n, nf = D.n_fine, E = D.cells;

    // Element materials (classify_tsv by centroid radius, mesh.cpp:182-190; dummy = silicon).
    std::vector<uint8_t> mat(E, 2);
    if (d->kind == 0)
        for (size_t k = 0; k < cz; ++k)
            for (size_t j = 0; j < cy; ++j)
                for (size_t i = 0; i < cx; ++i) {
                    const double xc = 0.5 * (grid[0][i] + grid[0][i + 1]);
                    const double yc = 0.5 * (grid[1][j] + grid[1][j + 1]);
                    const double r = std::hypot(xc - 0.5 * pp, yc - 0.5 * pp);
                    mat[(k * cy + j) * cx + i] = r < 0.5 * dd ? 0 : (r < 0.5 * dd + tt ? 1 : 2);
                }

    // Element matrices, DoF maps, colours.
    std::vector<double> ke(E * 576), fe(E * 24);
    std::vector<int> edofs(E * 24);
    std::vector<int> colour_elems[8];
    for (size_t k = 0; k < cz; ++k)
        for (size_t j = 0; j < cy; ++j)
            for (size_t i = 0; i < cx; ++i) {
                const size_t e = (k * cy + j) * cx + i;
                double c[8][3];
                for (int a = 0; a < 8; ++a) {
                    const size_t di = (a == 1 || a == 2 || a == 5 || a == 6);
                    const size_t dj = (a == 2 || a == 3 || a == 6 || a == 7);
                    const size_t dk = a >= 4;
                    const size_t node = ((k + dk) * ny + (j + dj)) * nx + (i + di);
                    c[a][0] = grid[0][i + di];
                    c[a][1] = grid[1][j + dj];
                    c[a][2] = grid[2][k + dk];
                    for (int q = 0; q < 3; ++q) edofs[e * 24 + 3 * a + q] = static_cast<int>(3 * node + q);
                }
                const double *L = lame[mat[e]];
                element_matrices(c, L[0], L[1], L[2], ke.data() + e * 576, fe.data() + e * 24);
                colour_elems[(i & 1) | ((j & 1) << 1) | ((k & 1) << 2)].push_back(static_cast<int>(e));
            }

    // Boundary / interior DoFs.
    std::vector<int> int_of_dof(nf, -1), dof_of_int;
    std::vector<uint8_t> on_bnd(nf / 3, 0);
    for (size_t k = 0; k < nz; ++k)
        for (size_t j = 0; j < ny; ++j)
            for (size_t i = 0; i < nx; ++i) {
                const size_t node = (k * ny + j) * nx + i;
                const bool b = i == 0 || i == nx - 1 || j == 0 || j == ny - 1 || k == 0 || k == nz - 1;
                on_bnd[node] = b;
                if (!b)
                    for (int q = 0; q < 3; ++q) {
                        int_of_dof[3 * node + q] = static_cast<int>(dof_of_int.size());
                        dof_of_int.push_back(static_cast<int>(3 * node + q));
                    }
            }
    const size_t ni = dof_of_int.size();

    // Interpolation operator rows of boundary fine DoFs (rom.cpp:67-108).
    std::vector<std::array<uint32_t, 3>> sn;
    for (uint32_t i = 0; i < d->q[0]; ++i)
        for (uint32_t j = 0; j < d->q[1]; ++j)
            for (uint32_t k = 0; k < d->q[2]; ++k)
                if (!(i > 0 && i + 1 < d->q[0] && j > 0 && j + 1 < d->q[1] && k > 0 && k + 1 < d->q[2]))
                    sn.push_back({i, j, k});
    std::vector<double> lc[3];
    for (int a = 0; a < 3; ++a) lc[a] = linspace(0.0, ext[a], d->q[a] - 1);
    std::vector<double> tab[3];  // tab[a][f * q + i]
    for (int a = 0; a < 3; ++a) {
        tab[a].resize(grid[a].size() * d->q[a]);
        for (size_t f = 0; f < grid[a].size(); ++f)
            for (size_t i = 0; i < d->q[a]; ++i) tab[a][f * d->q[a] + i] = lagrange_1d(lc[a], i, grid[a][f]);
    }
    // W rows (per boundary node): sparse list of (rank, weight), same for the 3 components.
    std::vector<std::vector<std::pair<int, double>>> wrow(nf / 3);
    for (size_t node = 0; node < nf / 3; ++node) {
        if (!on_bnd[node]) continue;
        const size_t fi = node % nx, fj = (node / nx) % ny, fk = node / (nx * ny);
        for (size_t rank = 0; rank < sn.size(); ++rank) {
            const double w = tab[0][fi * d->q[0] + sn[rank][0]] * tab[1][fj * d->q[1] + sn[rank][1]] *
                             tab[2][fk * d->q[2] + sn[rank][2]];
            if (w != 0.0) wrow[node].push_back({static_cast<int>(rank), w});
        }
    }

    // Right-hand sides, column-major ni x (n+1): -A_ib W (basis) and b_i (thermal, dT = 1).
    std::vector<double> rhs(ni * (n + 1), 0.0), b_unit(nf, 0.0);
    for (size_t e = 0; e < E; ++e) {
        const int *dofs = edofs.data() + e * 24;
        for (int r = 0; r < 24; ++r) b_unit[dofs[r]] += fe[e * 24 + r];
        for (int r = 0; r < 24; ++r) {
            const int ir = int_of_dof[dofs[r]];
            if (ir < 0) continue;
            for (int s = 0; s < 24; ++s) {
                if (int_of_dof[dofs[s]] >= 0) continue;
                const double v = ke[e * 576 + r * 24 + s];
                const int comp = dofs[s] % 3;
                for (const auto &[rank, w] : wrow[dofs[s] / 3]) rhs[static_cast<size_t>(3 * rank + comp) * ni + ir] -= v * w;
            }
        }
    }
    for (size_t ir = 0; ir < ni; ++ir) rhs[n * ni + ir] = b_unit[dof_of_int[ir]];

    // ----------------------------------------------------------- GPU part
    LCK(cudaSetDevice(device));
    cudaStream_t s;
    LCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    cusolverDnHandle_t sol;
    cublasHandle_t blas;
    LCS(cusolverDnCreate(&sol));
    struct SolGuard {
        cusolverDnHandle_t h;
        ~SolGuard() { cusolverDnDestroy(h); }
    } solg{sol};
    LCS(cublasCreate(&blas));
    struct BlasGuard {
        cublasHandle_t h;
        ~BlasGuard() { cublasDestroy(h); }
    } blasg{blas};
    LCS(cusolverDnSetStream(sol, s));
    LCS(cublasSetStream(blas, s));

    Dev<double> d_ke(E * 576), d_A(ni * ni), d_X(ni * (n + 1)), d_phi(nf * n), d_aphi(nf * n), d_ut(nf),
        d_b(nf), d_kr(n * n), d_bel(n);
    Dev<int> d_edofs(E * 24), d_iod(nf), d_doi(ni), d_elems(E);
    LCK(cudaMemcpyAsync(d_ke.p, ke.data(), E * 576 * 8, cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(d_edofs.p, edofs.data(), E * 24 * 4, cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(d_iod.p, int_of_dof.data(), nf * 4, cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(d_doi.p, dof_of_int.data(), ni * 4, cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(d_X.p, rhs.data(), rhs.size() * 8, cudaMemcpyHostToDevice, s));
    LCK(cudaMemcpyAsync(d_b.p, b_unit.data(), nf * 8, cudaMemcpyHostToDevice, s));
    LCK(cudaMemsetAsync(d_A.p, 0, ni * ni * 8, s));
    // colour-ordered element lists back to back
    std::vector<int> elems_cat;
    std::vector<size_t> col_off(9, 0);
    for (int c = 0; c < 8; ++c) {
        col_off[c] = elems_cat.size();
        elems_cat.insert(elems_cat.end(), colour_elems[c].begin(), colour_elems[c].end());
    }
    col_off[8] = elems_cat.size();
    LCK(cudaMemcpyAsync(d_elems.p, elems_cat.data(), E * 4, cudaMemcpyHostToDevice, s));
    for (int c = 0; c < 8; ++c) {
        const int ne = static_cast<int>(col_off[c + 1] - col_off[c]);
        if (!ne) continue;
        const long long th = static_cast<long long>(ne) * 576;
        assemble_interior_kernel<<<static_cast<unsigned>((th + 255) / 256), 256, 0, s>>>(
            ne, d_elems.p + col_off[c], d_ke.p, d_iod.p, d_edofs.p, d_A.p, static_cast<long long>(ni));
        LCK(cudaGetLastError());
    }
    // Cholesky of the interior block and n+1 solves.
    Dev<int> d_info(1);
    int lwork = 0;
    LCS(cusolverDnDpotrf_bufferSize(sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(ni), d_A.p, static_cast<int>(ni), &lwork));
    Dev<double> d_work(static_cast<size_t>(lwork));
    LCS(cusolverDnDpotrf(sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(ni), d_A.p, static_cast<int>(ni), d_work.p, lwork,
                         d_info.p));
    int info = 0;
    LCK(cudaMemcpyAsync(&info, d_info.p, 4, cudaMemcpyDeviceToHost, s));
    LCK(cudaStreamSynchronize(s));
    if (info != 0) throw LsError(TSV_EINVAL, "factorize_spd: interior block is not positive definite (pivot " + std::to_string(info) + ")");
    LCS(cusolverDnDpotrs(sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(ni), static_cast<int>(n + 1), d_A.p,
                         static_cast<int>(ni), d_X.p, static_cast<int>(ni), d_info.p));
    // Phi: boundary rows pinned to the interpolation weights (rom.cpp:215-219).
    std::vector<double> phi_b(nf * n, 0.0);
    for (size_t node = 0; node < nf / 3; ++node)
        for (const auto &[rank, w] : wrow[node])
            for (int q = 0; q < 3; ++q) phi_b[(3 * node + q) * n + 3 * rank + q] = w;
    LCK(cudaMemcpyAsync(d_phi.p, phi_b.data(), nf * n * 8, cudaMemcpyHostToDevice, s));
    LCK(cudaMemsetAsync(d_ut.p, 0, nf * 8, s));
    {
        const long long th = static_cast<long long>(ni) * (n + 1);
        scatter_solution_kernel<<<static_cast<unsigned>((th + 255) / 256), 256, 0, s>>>(
            static_cast<int>(ni), static_cast<int>(n), d_doi.p, d_X.p, d_phi.p, d_ut.p);
        LCK(cudaGetLastError());
    }
    // A*Phi element by element (colour order, deterministic), then K_r = Phi^T (A Phi).
    LCK(cudaMemsetAsync(d_aphi.p, 0, nf * n * 8, s));
    for (int c = 0; c < 8; ++c) {
        const int ne = static_cast<int>(col_off[c + 1] - col_off[c]);
        if (!ne) continue;
        dim3 grid(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>(ne));
        element_aphi_kernel<<<grid, 128, 0, s>>>(ne, d_elems.p + col_off[c], d_ke.p, d_edofs.p, d_phi.p, d_aphi.p,
                                                 static_cast<int>(n));
        LCK(cudaGetLastError());
    }
    const double one = 1.0, zero = 0.0;
    const int in = static_cast<int>(n), inf = static_cast<int>(nf);
    LCS(cublasDgemm(blas, CUBLAS_OP_N, CUBLAS_OP_T, in, in, inf, &one, d_aphi.p, in, d_phi.p, in, &zero, d_kr.p, in));
    LCS(cublasDgemv(blas, CUBLAS_OP_N, in, inf, &one, d_phi.p, in, d_b.p, 1, &zero, d_bel.p, 1));
    if (out->a_element) LCK(cudaMemcpyAsync(out->a_element, d_kr.p, n * n * 8, cudaMemcpyDeviceToHost, s));
    if (out->b_element) LCK(cudaMemcpyAsync(out->b_element, d_bel.p, n * 8, cudaMemcpyDeviceToHost, s));
    if (out->basis) LCK(cudaMemcpyAsync(out->basis, d_phi.p, nf * n * 8, cudaMemcpyDeviceToHost, s));
    if (out->thermal) LCK(cudaMemcpyAsync(out->thermal, d_ut.p, nf * 8, cudaMemcpyDeviceToHost, s));
    LCK(cudaStreamSynchronize(s));
    if (out->element_material) std::memcpy(out->element_material, mat.data(), E);
    sha256_fingerprint(d, out->fingerprint);
    out->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

int tsv_rom_dims(const tsv_local_desc *d, uint64_t *n, uint64_t *n_fine, uint64_t *cells) {
    try {
        const Dims D = dims_of(d);
        if (n) *n = D.n;
        if (n_fine) *n_fine = D.n_fine;
        if (cells) *cells = D.cells;
        return TSV_OK;
    } catch (const LsError &e) {
        return e.code;
    }
}

int tsv_build_rom(int device, const tsv_local_desc *d, tsv_rom_out *out, char *err, size_t err_len) {
    auto report = [&](const char *m) {
        if (err && err_len) {
            std::strncpy(err, m, err_len - 1);
            err[err_len - 1] = 0;
        }
    };
    try {
        if (!out) throw LsError(TSV_EINVAL, "build_rom: NULL output");
        build(device, d, out);
        report("");
        return TSV_OK;
    } catch (const LsError &e) {
        report(e.what());
        return e.code;
    } catch (const std::bad_alloc &) {
        report("host allocation failed");
        return TSV_ENOMEM;
    } catch (const std::exception &e) {
        report(e.what());
        return TSV_EINVAL;
    }
}

}  // extern "C"
