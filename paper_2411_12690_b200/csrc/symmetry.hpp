// Mirror symmetry of the macro-element (host tables).
//
// A TSV block on a grid that is symmetric about its three mid-planes maps to
// itself under the axis mirrors m_x, m_y, m_z (the abelian group Z2^3). The
// reduced stiffness K_r and the basis Phi commute with that action, so in a
// symmetry-adapted basis they are block diagonal with 8 blocks, one per
// irreducible representation r in 0..7 (bit a of r = parity under m_a): the
// dense contractions K1 (Y = X K_r) and K6 (U = Q Phi^T) need 1/8 of the FP64
// FLOPs. Whether a given ROM has the symmetry is decided numerically when it
// is set (tsv_set_rom): the off-diagonal blocks must vanish to rounding.
//
// The adapted basis is a Walsh-Hadamard transform over each mirror orbit of a
// DoF (node orbit x component). For the orbit of DoF d with free axes F (the
// axes whose mirror moves the node) and members g (g subset of F: which axes
// are mirrored relative to the representative),
//     x'_w = sum_g (-1)^{popcount(w & g)} x_g,   w subset of F,
// unnormalised (adds only; H H = |orbit| I, the power-of-two scale is folded
// into the packed matrices and the inverse transform). Mirror a flips the sign
// of displacement component a, so combination w of component c belongs to
// irrep r = w xor e_c. Combination w is stored at the position of member g = w.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace tsvb200 {

struct SymDof {
    int ijk[3];
    int comp;
};

// Orbit/segment tables of a DoF set in a "plain" layout (index = position in
// the dofs vector) and its irrep-segmented layout.
struct SymTables {
    bool closed = false;         // the set maps to itself under the three mirrors
    int n = 0;                   // DoFs
    int count[8] = {}, off[8] = {};  // DoFs per irrep, segment offsets (aligned)
    int ld = 0;                  // row length of the segmented layout (aligned)
    std::vector<int8_t> label;   // [n] irrep of the combination stored at DoF d
    std::vector<int> pos;        // [n] column of that combination in the segmented layout
    std::vector<uint8_t> size;   // [n] orbit size (1, 2, 4, 8)
    int n_orbits = 0;
    std::vector<int> src;        // [n_orbits][8] plain index of member g (-1: not a member)
    std::vector<int> dst;        // [n_orbits][8] segmented column of combination g (-1)

    // len: nodes per axis; seg_align: segment offsets/lengths padded to this
    void build(const int len[3], const std::vector<SymDof> &dofs, int seg_align) {
        n = static_cast<int>(dofs.size());
        closed = true;
        const size_t cells = static_cast<size_t>(len[0]) * len[1] * len[2] * 3;
        std::vector<int> where(cells, -1);
        auto key = [&](const int ijk[3], int c) {
            return ((static_cast<size_t>(ijk[2]) * len[1] + ijk[1]) * len[0] + ijk[0]) * 3 + c;
        };
        for (int d = 0; d < n; ++d) where[key(dofs[d].ijk, dofs[d].comp)] = d;
        label.assign(n, -1);
        pos.assign(n, -1);
        size.assign(n, 0);
        src.clear();
        dst.clear();
        for (int r = 0; r < 8; ++r) count[r] = 0;
        for (int d = 0; d < n; ++d) {
            int g = 0;
            for (int a = 0; a < 3; ++a)
                if (2 * dofs[d].ijk[a] > len[a] - 1) g |= 1 << a;
            label[d] = static_cast<int8_t>(g ^ (1 << dofs[d].comp));
            ++count[label[d]];
        }
        int o = 0;
        for (int r = 0; r < 8; ++r) {
            off[r] = o;
            o += (count[r] + seg_align - 1) / seg_align * seg_align;
        }
        ld = o;
        int fill[8] = {};
        for (int d = 0; d < n; ++d) pos[d] = off[label[d]] + fill[label[d]]++;
        for (int d = 0; d < n; ++d) {
            int f = 0, g0 = 0;
            for (int a = 0; a < 3; ++a) {
                if (2 * dofs[d].ijk[a] != len[a] - 1) f |= 1 << a;
                if (2 * dofs[d].ijk[a] > len[a] - 1) g0 |= 1 << a;
            }
            if (g0) continue;  // not the representative
            std::array<int, 8> s, t;
            s.fill(-1);
            t.fill(-1);
            int members = 0;
            for (int g = 0; g < 8; ++g) {
                if (g & ~f) continue;
                int m[3];
                for (int a = 0; a < 3; ++a) m[a] = (g >> a & 1) ? len[a] - 1 - dofs[d].ijk[a] : dofs[d].ijk[a];
                const int e = where[key(m, dofs[d].comp)];
                if (e < 0) {
                    closed = false;
                    return;
                }
                s[g] = e;
                t[g] = pos[e];
                ++members;
            }
            for (int g = 0; g < 8; ++g)
                if (s[g] >= 0) size[s[g]] = static_cast<uint8_t>(members);
            src.insert(src.end(), s.begin(), s.end());
            dst.insert(dst.end(), t.begin(), t.end());
        }
        n_orbits = static_cast<int>(src.size() / 8);
        for (int d = 0; d < n; ++d)
            if (!size[d]) {
                closed = false;  // a DoF whose representative is missing
                return;
            }
    }

    // Orbit order for the shared-memory butterflies of the fused K1 kernel (sym.cuh): a
    // half-warp handles `group` consecutive orbits of 16 / group rows, member g of each in
    // one 8-byte access; with the row pitch = 4 mod 16 doubles and group = 4 that is
    // conflict-free when the 4 columns differ mod 4 (`mod`). Greedy: every group is filled
    // with the orbit that adds the fewest same-bank pairs over the 8 members. (The orbit
    // order is free: src / dst rows move together.)
    void order_orbits_for_banks(int group = 4, int mod = 4) {
        if (n_orbits < 2) return;
        std::vector<int> order, left(n_orbits);
        for (int o = 0; o < n_orbits; ++o) left[o] = o;
        int used[8][16];
        while (!left.empty()) {
            for (auto &u : used)
                for (int &v : u) v = 0;
            for (int slot = 0; slot < group && !left.empty(); ++slot) {
                size_t best = 0;
                int best_cost = 1 << 30;
                for (size_t c = 0; c < left.size(); ++c) {
                    int cost = 0;
                    for (int g = 0; g < 8; ++g) {
                        const int col = src[static_cast<size_t>(left[c]) * 8 + g];
                        if (col >= 0) cost += used[g][col % mod];
                    }
                    if (cost < best_cost) {
                        best_cost = cost;
                        best = c;
                        if (cost == 0) break;
                    }
                }
                const int o = left[best];
                left.erase(left.begin() + static_cast<long>(best));
                order.push_back(o);
                for (int g = 0; g < 8; ++g) {
                    const int col = src[static_cast<size_t>(o) * 8 + g];
                    if (col >= 0) ++used[g][col % mod];
                }
            }
        }
        std::vector<int> s2(src.size()), d2(dst.size());
        for (int i = 0; i < n_orbits; ++i)
            for (int g = 0; g < 8; ++g) {
                s2[static_cast<size_t>(i) * 8 + g] = src[static_cast<size_t>(order[i]) * 8 + g];
                d2[static_cast<size_t>(i) * 8 + g] = dst[static_cast<size_t>(order[i]) * 8 + g];
            }
        src.swap(s2);
        dst.swap(d2);
    }

    // Same-bank pairs left per group of orbits, summed over groups and members (0 = conflict-free).
    int bank_conflicts(int group = 4, int mod = 4) const {
        int total = 0;
        for (int o0 = 0; o0 < n_orbits; o0 += group)
            for (int g = 0; g < 8; ++g) {
                int cnt[16] = {};
                for (int o = o0; o < std::min(n_orbits, o0 + group); ++o) {
                    const int col = src[static_cast<size_t>(o) * 8 + g];
                    if (col >= 0) total += cnt[col % mod]++;
                }
            }
        return total;
    }

    // In-place unnormalised transform of v[index * stride] over every orbit
    // (plain layout: combination g lands on member g).
    void transform(double *v, size_t stride) const {
        for (int o = 0; o < n_orbits; ++o) {
            const int *s = src.data() + static_cast<size_t>(o) * 8;
            double x[8];
            int f = 0;
            for (int g = 0; g < 8; ++g) {
                x[g] = s[g] >= 0 ? v[static_cast<size_t>(s[g]) * stride] : 0.0;
                if (s[g] >= 0) f |= g;
            }
            for (int a = 0; a < 3; ++a) {
                if (!(f >> a & 1)) continue;
                for (int g = 0; g < 8; ++g) {
                    if ((g >> a & 1) || (g & ~f)) continue;
                    const double lo = x[g], hi = x[g | 1 << a];
                    x[g] = lo + hi;
                    x[g | 1 << a] = lo - hi;
                }
            }
            for (int g = 0; g < 8; ++g)
                if (s[g] >= 0) v[static_cast<size_t>(s[g]) * stride] = x[g];
        }
    }

    // The same transform applied to the rows of a row-major matrix M[index][cols]
    // (orbits [o0, o1): callers split the range over threads).
    void transform_rows(double *M, size_t cols, int o0, int o1) const {
        for (int o = o0; o < o1; ++o) {
            const int *s = src.data() + static_cast<size_t>(o) * 8;
            int f = 0;
            for (int g = 0; g < 8; ++g)
                if (s[g] >= 0) f |= g;
            for (int a = 0; a < 3; ++a) {
                if (!(f >> a & 1)) continue;
                for (int g = 0; g < 8; ++g) {
                    if ((g >> a & 1) || (g & ~f)) continue;
                    double *lo = M + static_cast<size_t>(s[g]) * cols, *hi = M + static_cast<size_t>(s[g | 1 << a]) * cols;
                    for (size_t j = 0; j < cols; ++j) {
                        const double l = lo[j], h = hi[j];
                        lo[j] = l + h;
                        hi[j] = l - h;
                    }
                }
            }
        }
    }
};

// One irrep block of a segmented GEMM (sym.cuh: gemm_seg_f64).
struct GemmSeg {
    long long a_off, c_off, b_off, bias_off;
    int ldb, k_chunks, n_valid, n_tiles, tile0;
};

// Symmetry-adapted packing of one ROM.
//   kp      K_r in panel order [n][n] (panel column of reference DoF a = 3 rank + c: c * n/3 + rank)
//   basis   Phi [n_fine][n], thermal u_T [n_fine], reference order
//   dmap    the dense basis rows (fine DoFs, ascending)
//   bn, kc  N tile and k-chunk of the GEMM (segment matrices are padded to them)
// build() returns false (and leaves the defects measured so far) when the
// ROM does not have the mirror symmetry to `tol`.
struct SymRomPack {
    SymTables red, fine;
    double defect_k = 0.0, defect_phi = 0.0;
    std::vector<GemmSeg> k1_segs, k6_segs;
    int k1_tiles_per_m = 0, k6_tiles_per_m = 0;
    int bank_conflicts_before = 0;  // of the reduced orbit order before order_orbits_for_banks()
    std::vector<double> ks, ps, uts;  // packed K''_r, Phi''_r blocks; H u_T in the fine segmented layout
    std::vector<short> ssrc, sdst;    // reduced orbit tables
    std::vector<int> fsrc;            // fine orbit table: U columns (fine DoFs); Us columns are fine.dst
    std::vector<float> d32;           // (K_r - K_sym) * 2^d_exp, [n][n] panel order
    int d_exp = 0;
    bool d_nonzero = false;

    bool build(const uint32_t q[3], const int cells[3], size_t n, const std::vector<double> &kp, const double *basis,
               const double *thermal, const std::vector<int> &dmap, int bn, int kc, double tol = 1e-12) {
        const size_t nn = n / 3;
        if (n == 0 || n > 32000 || dmap.empty()) return false;
        std::vector<SymDof> rd(n);
        {
            size_t rank = 0;  // NodeLayout order (rom.cpp:26-31): i, j, k lexicographic, surface nodes only
            for (uint32_t i = 0; i < q[0]; ++i)
                for (uint32_t j = 0; j < q[1]; ++j)
                    for (uint32_t k = 0; k < q[2]; ++k) {
                        if (i > 0 && i + 1 < q[0] && j > 0 && j + 1 < q[1] && k > 0 && k + 1 < q[2]) continue;
                        for (int c = 0; c < 3; ++c)
                            rd[c * nn + rank] = SymDof{{static_cast<int>(i), static_cast<int>(j), static_cast<int>(k)}, c};
                        ++rank;
                    }
            if (rank != nn) return false;
        }
        const int qlen[3] = {static_cast<int>(q[0]), static_cast<int>(q[1]), static_cast<int>(q[2])};
        red.build(qlen, rd, kc);
        if (!red.closed) return false;
        bank_conflicts_before = red.bank_conflicts();
        red.order_orbits_for_banks();
        const SymTables &R = red;
        // K'' = H K H S^-1
        std::vector<double> k2 = kp;
        for (size_t b = 0; b < n; ++b) R.transform(k2.data() + b, n);
        for (size_t a = 0; a < n; ++a) R.transform(k2.data() + a * n, 1);
        double kmax = 0.0, koff = 0.0;
        for (size_t a = 0; a < n; ++a)
            for (size_t b = 0; b < n; ++b) {
                k2[a * n + b] /= static_cast<double>(R.size[b]);
                const double v = std::fabs(k2[a * n + b]);
                kmax = std::max(kmax, v);
                if (R.label[a] != R.label[b]) koff = std::max(koff, v);
            }
        defect_k = kmax > 0.0 ? koff / kmax : 0.0;
        if (!(defect_k <= tol)) return false;
        // dense fine DoFs (x fastest, mesh.cpp node order)
        const int flen[3] = {cells[0] + 1, cells[1] + 1, cells[2] + 1};
        std::vector<SymDof> fd(dmap.size());
        for (size_t i = 0; i < dmap.size(); ++i) {
            const int node = dmap[i] / 3;
            fd[i] = SymDof{{node % flen[0], (node / flen[0]) % flen[1], node / (flen[0] * flen[1])}, dmap[i] % 3};
        }
        fine.build(flen, fd, 8);
        if (!fine.closed) return false;
        const SymTables &F = fine;
        const size_t nd = dmap.size();
        // Phi'' = H_f Phi H S_r^-1 on the dense rows (columns in panel order)
        std::vector<double> ph(nd * n);
        {
            const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
            std::vector<std::thread> pool;
            for (unsigned w = 0; w < nt; ++w)
                pool.emplace_back([&, w] {
                    for (size_t i = w; i < nd; i += nt) {
                        const double *row = basis + static_cast<size_t>(dmap[i]) * n;
                        double *dst = ph.data() + i * n;
                        for (size_t a = 0; a < n; ++a) dst[(a % 3) * nn + a / 3] = row[a];
                        R.transform(dst, 1);
                    }
                });
            for (auto &t : pool) t.join();
            pool.clear();
            for (unsigned w = 0; w < nt; ++w)
                pool.emplace_back([&, w] {
                    const int per = (F.n_orbits + static_cast<int>(nt) - 1) / static_cast<int>(nt);
                    F.transform_rows(ph.data(), n, std::min(F.n_orbits, static_cast<int>(w) * per),
                                     std::min(F.n_orbits, static_cast<int>(w + 1) * per));
                });
            for (auto &t : pool) t.join();
        }
        double pmax = 0.0, poff = 0.0;
        for (size_t i = 0; i < nd; ++i)
            for (size_t b = 0; b < n; ++b) {
                ph[i * n + b] /= static_cast<double>(R.size[b]);
                const double v = std::fabs(ph[i * n + b]);
                pmax = std::max(pmax, v);
                if (F.label[i] != R.label[b]) poff = std::max(poff, v);
            }
        defect_phi = pmax > 0.0 ? poff / pmax : 0.0;
        if (!(defect_phi <= tol)) return false;
        if (R.ld > 32767 || n > 32767) return false;

        // ---- pack the irrep blocks
        auto pad = [](size_t v, size_t a) { return (v + a - 1) / a * a; };
        std::vector<size_t> cols_of[8], rows_of[8];
        for (size_t b = 0; b < n; ++b) cols_of[R.label[b]].push_back(b);  // ascending = ascending pos
        for (size_t i = 0; i < nd; ++i) rows_of[F.label[i]].push_back(i);
        int t1 = 0, t6 = 0;
        for (int r = 0; r < 8; ++r) {
            const size_t nr = cols_of[r].size(), kpad = pad(nr, kc);
            if (nr) {
                GemmSeg g{};
                g.a_off = g.c_off = R.off[r];
                g.b_off = static_cast<long long>(ks.size());
                g.bias_off = 0;
                g.ldb = static_cast<int>(kpad);
                g.k_chunks = static_cast<int>(kpad / kc);
                g.n_valid = static_cast<int>(nr);
                g.n_tiles = static_cast<int>(pad(nr, bn) / bn);
                g.tile0 = t1;
                t1 += g.n_tiles;
                k1_segs.push_back(g);
                ks.resize(ks.size() + pad(nr, bn) * kpad, 0.0);
                double *blk = ks.data() + g.b_off;
                for (size_t ia = 0; ia < nr; ++ia)
                    for (size_t ib = 0; ib < nr; ++ib) blk[ia * kpad + ib] = k2[cols_of[r][ia] * n + cols_of[r][ib]];
            }
            const size_t nf = rows_of[r].size();
            if (nf) {
                GemmSeg g{};
                g.a_off = R.off[r];
                g.c_off = g.bias_off = F.off[r];
                g.b_off = static_cast<long long>(ps.size());
                g.ldb = static_cast<int>(std::max<size_t>(kpad, kc));
                g.k_chunks = static_cast<int>(kpad / kc);
                g.n_valid = static_cast<int>(nf);
                g.n_tiles = static_cast<int>(pad(nf, bn) / bn);
                g.tile0 = t6;
                t6 += g.n_tiles;
                k6_segs.push_back(g);
                ps.resize(ps.size() + pad(nf, bn) * g.ldb, 0.0);
                double *blk = ps.data() + g.b_off;
                for (size_t i = 0; i < nf; ++i)
                    for (size_t ib = 0; ib < nr; ++ib) blk[i * g.ldb + ib] = ph[rows_of[r][i] * n + cols_of[r][ib]];
            }
        }
        k1_tiles_per_m = t1;
        k6_tiles_per_m = t6;
        // H_f u_T in the fine segmented layout
        std::vector<double> ut(nd);
        uts.assign(static_cast<size_t>(F.ld), 0.0);
        for (size_t i = 0; i < nd; ++i) ut[i] = thermal[dmap[i]];
        F.transform(ut.data(), 1);
        for (size_t i = 0; i < nd; ++i) uts[F.pos[i]] = ut[i];
        // orbit tables
        ssrc.resize(R.src.size());
        sdst.resize(R.dst.size());
        for (size_t i = 0; i < R.src.size(); ++i) {
            ssrc[i] = static_cast<short>(R.src[i]);
            sdst[i] = static_cast<short>(R.dst[i]);
        }
        fsrc.resize(F.src.size());
        for (size_t i = 0; i < F.src.size(); ++i) fsrc[i] = F.src[i] >= 0 ? dmap[F.src[i]] : -1;
        // D = K - K_sym, K_sym = S^-1 H K''_bd H (K''_bd: the diagonal blocks of K'')
        std::vector<double> kb(n * n, 0.0);
        for (size_t a = 0; a < n; ++a)
            for (size_t b = 0; b < n; ++b)
                if (R.label[a] == R.label[b]) kb[a * n + b] = k2[a * n + b];
        for (size_t b = 0; b < n; ++b) R.transform(kb.data() + b, n);
        for (size_t a = 0; a < n; ++a) R.transform(kb.data() + a * n, 1);
        double dmax = 0.0;
        for (size_t a = 0; a < n; ++a)
            for (size_t b = 0; b < n; ++b) {
                kb[a * n + b] = kp[a * n + b] - kb[a * n + b] / static_cast<double>(R.size[a]);
                dmax = std::max(dmax, std::fabs(kb[a * n + b]));
            }
        d_nonzero = dmax > 0.0;
        int e = 0;
        if (d_nonzero) {
            std::frexp(dmax, &e);  // dmax = f * 2^e, f in [0.5, 1)
            e = -e;
        }
        d_exp = e;
        d32.resize(n * n);
        for (size_t i = 0; i < n * n; ++i) d32[i] = static_cast<float>(std::ldexp(kb[i], e));
        return true;
    }
};


// Host tables of the fused K1 kernel (sym.cuh: sym_k1_fused_kernel): work
// items (irrep, pair of 8-column fragments) in irrep order, the irreps' column
// lists in the plain panel layout, and K''_r in DMMA fragment order per item
// ([k-step][fragment][lane]: B[n = 16 j + 8 f + lane / 4][k = 4 s + lane % 4],
// zero padded to whole chunks of `kb` k-steps).
//
// The k order of an irrep is free (a permutation of its columns applied to
// both operands): columns are dealt into k-steps so that the four columns of
// a k-step differ mod 4 wherever the residue classes allow it, which makes
// the kernel's A fragment loads (row pitch = 4 mod 16 doubles) conflict-free.
struct SymK1Pack {
    struct Item {
        int b_off;
        short ksteps, ksteps4, kcol, ncol, nvalid, irrep;
    };
    std::vector<Item> items;
    std::vector<short> coltab;
    std::vector<double> bf;
    int conflict_quads = 0, quads = 0;  // k-steps whose columns collide mod 4 / all k-steps

    // segs / ks: SymRomPack::k1_segs and ::ks of the same ROM (one segment per non-empty irrep, in irrep order)
    void build(const SymTables &R, const std::vector<GemmSeg> &segs, const std::vector<double> &ks, int kb = 4) {
        items.clear();
        coltab.clear();
        bf.clear();
        conflict_quads = quads = 0;
        size_t si = 0;
        for (int r = 0; r < 8; ++r) {
            std::vector<int> cols;  // ascending plain column = ascending index in the packed block
            for (int d = 0; d < R.n; ++d)
                if (R.label[d] == r) cols.push_back(d);
            if (cols.empty()) continue;
            const GemmSeg &g = segs[si++];
            const int nr = static_cast<int>(cols.size());
            const double *blk = ks.data() + g.b_off;
            const int ksteps = (nr + 7) / 8 * 2;  // even
            const int ksteps4 = (ksteps + kb - 1) / kb * kb;
            // k order: korder[k] = index into cols (or -1: padding)
            std::vector<int> korder(static_cast<size_t>(ksteps) * 4, -1);
            {
                std::vector<int> cls[4];
                for (int i = nr - 1; i >= 0; --i) cls[cols[i] & 3].push_back(i);  // pop_back yields ascending
                for (int s = 0; s < ksteps; ++s) {
                    // one column from each of the (up to four) fullest classes
                    int order[4] = {0, 1, 2, 3};
                    std::sort(order, order + 4, [&](int a, int b) { return cls[a].size() > cls[b].size(); });
                    int filled = 0;
                    for (int c = 0; c < 4 && filled < 4; ++c)
                        if (!cls[order[c]].empty()) {
                            korder[s * 4 + filled++] = cls[order[c]].back();
                            cls[order[c]].pop_back();
                        }
                    // classes exhausted unevenly: fill the k-step from the fullest remaining class
                    while (filled < 4) {
                        int best = 0;
                        for (int c = 1; c < 4; ++c)
                            if (cls[c].size() > cls[best].size()) best = c;
                        if (cls[best].empty()) break;
                        korder[s * 4 + filled++] = cls[best].back();
                        cls[best].pop_back();
                    }
                }
                for (int s = 0; s < ksteps; ++s) {
                    bool clash = false;
                    for (int a = 0; a < 4; ++a)
                        for (int b = a + 1; b < 4; ++b)
                            if (korder[s * 4 + a] >= 0 && korder[s * 4 + b] >= 0 &&
                                ((cols[korder[s * 4 + a]] ^ cols[korder[s * 4 + b]]) & 3) == 0)
                                clash = true;
                    conflict_quads += clash;
                    ++quads;
                }
            }
            while (coltab.size() % 4) coltab.push_back(0);
            const int koff = static_cast<int>(coltab.size());
            // transposed k column list [4][ksteps4]; padding points at a real column (its K'' entries are zero)
            for (int q = 0; q < 4; ++q)
                for (int s = 0; s < ksteps4; ++s) {
                    const int ki = s < ksteps ? korder[s * 4 + q] : -1;
                    coltab.push_back(static_cast<short>(cols[ki >= 0 ? ki : 0]));
                }
            const int npairs = (nr + 15) / 16;
            const int noff = static_cast<int>(coltab.size());
            for (int i = 0; i < npairs * 16; ++i) coltab.push_back(static_cast<short>(cols[i < nr ? i : 0]));
            for (int j = 0; j < npairs; ++j) {
                Item it{};
                it.b_off = static_cast<int>(bf.size());
                it.ksteps = static_cast<short>(ksteps);
                it.ksteps4 = static_cast<short>(ksteps4);
                it.kcol = static_cast<short>(koff);
                it.ncol = static_cast<short>(noff + 16 * j);
                it.nvalid = static_cast<short>(std::min(16, nr - 16 * j));
                it.irrep = static_cast<short>(r);
                items.push_back(it);
                for (int s = 0; s < ksteps4; ++s)
                    for (int f = 0; f < 2; ++f)
                        for (int l = 0; l < 32; ++l) {
                            const int nidx = 16 * j + 8 * f + (l >> 2);
                            const int ki = s < ksteps ? korder[s * 4 + (l & 3)] : -1;
                            bf.push_back(nidx < nr && ki >= 0 ? blk[static_cast<size_t>(nidx) * g.ldb + ki] : 0.0);
                        }
            }
        }
    }

    // Round in which the last item of each item's irrep runs when item i runs in
    // round i / warps; returns the largest distance to it.
    int flush_rounds(int warps, std::vector<short> &flush) const {
        int last[8];
        for (int r = 0; r < 8; ++r) last[r] = -1;
        for (size_t i = 0; i < items.size(); ++i) last[items[i].irrep] = static_cast<int>(i) / warps;
        flush.resize(items.size());
        int span = 0;
        for (size_t i = 0; i < items.size(); ++i) {
            flush[i] = static_cast<short>(last[items[i].irrep]);
            span = std::max(span, last[items[i].irrep] - static_cast<int>(i) / warps);
        }
        return span;
    }
};

}  // namespace tsvb200
