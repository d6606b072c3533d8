// CPU emulation of the mirror-symmetric K1 / K6 data path (csrc/sym.cuh) on
// the host tables of csrc/symmetry.hpp: forward Walsh-Hadamard pass, the 8
// irrep GEMMs on the packed blocks, the TF32 defect correction, the inverse
// passes. Compiled by tests/test_symmetry_host.py (g++, no GPU).
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../paper_2411_12690_b200/csrc/symmetry.hpp"

using namespace tsvb200;

static void butterfly(double x[8], int f) {
    for (int a = 0; a < 3; ++a) {
        if (!(f >> a & 1)) continue;
        for (int g = 0; g < 8; ++g) {
            if (g >> a & 1) continue;
            const double lo = x[g], hi = x[g | 1 << a];
            x[g] = lo + hi;
            x[g | 1 << a] = lo - hi;
        }
    }
}

static double scale_of(int f) { return f == 7 ? 0.125 : (f == 0 ? 1.0 : ((f & (f - 1)) == 0 ? 0.5 : 0.25)); }

extern "C" int sym_host_check(const uint32_t *q, const int *cells, int n, int n_fine, const double *K, const double *Phi,
                              const double *uT, int bn, int kc, const double *x_ref, double dT, double *out) {
    // out: [0] defect K, [1] defect Phi, [2] rel err of K1 path, [3] rel err of K6 path (dense rows),
    //      [4] dense rows, [5] sum of irrep sizes, [6] K1 err without the correction,
    //      [7] rel err of the fused K1 data path (sym_k1_fused_kernel: in-place butterflies, fragment-ordered K'',
    //          round-wise flush with 8 warps); -1 when its flush span exceeds the kernel's slots,
    //      [8] / [9] k-steps with colliding columns / all k-steps of the fused path
    const size_t nn = n / 3;
    auto pidx = [&](size_t a) { return (a % 3) * nn + a / 3; };
    std::vector<double> kp(static_cast<size_t>(n) * n);
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) kp[pidx(a) * n + pidx(b)] = K[static_cast<size_t>(a) * n + b];
    std::vector<int> dmap;
    for (int f = 0; f < n_fine; ++f) {
        int nz = 0;
        for (int a = 0; a < n; ++a) nz += Phi[static_cast<size_t>(f) * n + a] != 0.0;
        if (nz > n / 4) dmap.push_back(f);
    }
    SymRomPack pk;
    const bool ok = pk.build(q, cells, n, kp, Phi, uT, dmap, bn, kc);
    out[0] = pk.defect_k;
    out[1] = pk.defect_phi;
    out[4] = static_cast<double>(dmap.size());
    if (!ok) return 1;
    const SymTables &R = pk.red, &F = pk.fine;
    int tot = 0;
    for (int r = 0; r < 8; ++r) tot += R.count[r];
    out[5] = tot;
    // panel row
    std::vector<double> X(n), Xs(R.ld, 0.0), Ys(R.ld, 0.0), Y(n, 0.0);
    for (int a = 0; a < n; ++a) X[pidx(a)] = x_ref[a];
    for (int o = 0; o < R.n_orbits; ++o) {
        double v[8];
        int f = 0;
        for (int g = 0; g < 8; ++g) {
            const int c = pk.ssrc[o * 8 + g];
            v[g] = c >= 0 ? X[c] : 0.0;
            if (c >= 0) f |= g;
        }
        butterfly(v, f);
        for (int g = 0; g < 8; ++g)
            if (pk.sdst[o * 8 + g] >= 0) Xs[pk.sdst[o * 8 + g]] = v[g];
    }
    for (const GemmSeg &s : pk.k1_segs)
        for (int j = 0; j < s.n_valid; ++j) {
            double acc = 0.0;
            for (int k = 0; k < s.k_chunks * kc; ++k) acc += Xs[s.a_off + k] * pk.ks[s.b_off + static_cast<long long>(j) * s.ldb + k];
            Ys[s.c_off + j] = acc;
        }
    for (int o = 0; o < R.n_orbits; ++o) {
        double v[8];
        int f = 0;
        for (int g = 0; g < 8; ++g) {
            const int c = pk.sdst[o * 8 + g];
            v[g] = c >= 0 ? Ys[c] : 0.0;
            if (c >= 0) f |= g;
        }
        butterfly(v, f);
        for (int g = 0; g < 8; ++g)
            if (pk.ssrc[o * 8 + g] >= 0) Y[pk.ssrc[o * 8 + g]] = scale_of(f) * v[g];
    }
    std::vector<double> Yref(n, 0.0);
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) Yref[a] += kp[static_cast<size_t>(a) * n + b] * X[b];
    double num = 0.0, den = 0.0, num0 = 0.0;
    for (int a = 0; a < n; ++a) {
        double c = 0.0;
        for (int b = 0; b < n; ++b) c += static_cast<double>(static_cast<float>(X[b])) * pk.d32[static_cast<size_t>(a) * n + b];
        const double y = Y[a] + std::ldexp(c, -pk.d_exp);
        num += (y - Yref[a]) * (y - Yref[a]);
        num0 += (Y[a] - Yref[a]) * (Y[a] - Yref[a]);
        den += Yref[a] * Yref[a];
    }
    out[2] = std::sqrt(num / den);
    out[6] = std::sqrt(num0 / den);
    {
        SymK1Pack fk;
        fk.build(R, pk.k1_segs, pk.ks);
        std::vector<short> flush;
        const int warps = 8, span = fk.flush_rounds(warps, flush);
        std::vector<double> xs(X);
        for (int o = 0; o < R.n_orbits; ++o) {
            double v[8];
            int f = 0;
            for (int g = 0; g < 8; ++g) {
                const int c = pk.ssrc[o * 8 + g];
                v[g] = c >= 0 ? xs[c] : 0.0;
                if (c >= 0) f |= g;
            }
            butterfly(v, f);
            for (int g = 0; g < 8; ++g)
                if (pk.ssrc[o * 8 + g] >= 0) xs[pk.ssrc[o * 8 + g]] = v[g];
        }
        const int ni = static_cast<int>(fk.items.size()), rounds = (ni + warps - 1) / warps;
        std::vector<std::array<double, 16>> res(ni);
        std::vector<char> flushed(ni, 0);
        for (int t = 0; t < rounds; ++t) {
            for (int i = t * warps; i < std::min(ni, (t + 1) * warps); ++i) {
                const SymK1Pack::Item &it = fk.items[i];
                for (int nn2 = 0; nn2 < 16; ++nn2) {
                    double acc = 0.0;
                    for (int s = 0; s < it.ksteps; ++s)
                        for (int kk = 0; kk < 4; ++kk)  // lane = (nn2 % 8) * 4 + kk of fragment nn2 / 8
                            acc += xs[fk.coltab[it.kcol + kk * it.ksteps4 + s]] *
                                   fk.bf[it.b_off + (s * 2 + nn2 / 8) * 32 + (nn2 % 8) * 4 + kk];
                    res[i][nn2] = acc;
                }
            }
            for (int i = 0; i < std::min(ni, (t + 1) * warps); ++i)
                if (!flushed[i] && flush[i] <= t) {
                    for (int nn2 = 0; nn2 < fk.items[i].nvalid; ++nn2) xs[fk.coltab[fk.items[i].ncol + nn2]] = res[i][nn2];
                    flushed[i] = 1;
                }
        }
        for (int o = 0; o < R.n_orbits; ++o) {
            double v[8];
            int f = 0;
            for (int g = 0; g < 8; ++g) {
                const int c = pk.ssrc[o * 8 + g];
                v[g] = c >= 0 ? xs[c] : 0.0;
                if (c >= 0) f |= g;
            }
            butterfly(v, f);
            for (int g = 0; g < 8; ++g)
                if (pk.ssrc[o * 8 + g] >= 0) xs[pk.ssrc[o * 8 + g]] = scale_of(f) * v[g];
        }
        double nf = 0.0;
        for (int a = 0; a < n; ++a) nf += (xs[a] - Yref[a]) * (xs[a] - Yref[a]);
        out[7] = span <= 1 ? std::sqrt(nf / den) : -1.0;
        out[8] = fk.conflict_quads;  // k-steps whose four columns collide mod 4 (shared-memory bank conflicts)
        out[9] = fk.quads;
        out[10] = pk.bank_conflicts_before;  // same-bank pairs of the butterflies' orbit order, natural / reordered
        out[11] = R.bank_conflicts();
    }
    // K6
    std::vector<double> Us(F.ld, 0.0), U(n_fine, 0.0);
    for (const GemmSeg &s : pk.k6_segs)
        for (int j = 0; j < s.n_valid; ++j) {
            double acc = 0.0;
            for (int k = 0; k < s.k_chunks * kc; ++k) acc += Xs[s.a_off + k] * pk.ps[s.b_off + static_cast<long long>(j) * s.ldb + k];
            Us[s.c_off + j] = acc + dT * pk.uts[s.bias_off + j];
        }
    for (int o = 0; o < F.n_orbits; ++o) {
        double v[8];
        int f = 0;
        for (int g = 0; g < 8; ++g) {
            const int c = F.dst[o * 8 + g];
            v[g] = c >= 0 ? Us[c] : 0.0;
            if (pk.fsrc[o * 8 + g] >= 0) f |= g;
        }
        butterfly(v, f);
        for (int g = 0; g < 8; ++g)
            if (pk.fsrc[o * 8 + g] >= 0) U[pk.fsrc[o * 8 + g]] = scale_of(f) * v[g];
    }
    num = den = 0.0;
    for (int f : dmap) {
        double u = dT * uT[f];
        for (int a = 0; a < n; ++a) u += Phi[static_cast<size_t>(f) * n + a] * x_ref[a];
        num += (U[f] - u) * (U[f] - u);
        den += u * u;
    }
    out[3] = den > 0.0 ? std::sqrt(num / den) : 0.0;
    return 0;
}
