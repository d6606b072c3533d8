// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal stand-in for the subset of the Eigen 3 API that the reference's
// own sources use (/root/reference/proj/src/linalg.cpp:3-4,141-191 and
// /root/reference/proj/src/rom.cpp:3,232-242). Eigen is a system dependency
// of the reference (proj/CMakeLists.txt:34) that is absent from this image;
// this file lets linalg.cpp and rom.cpp compile UNMODIFIED so the
// reference's build_rom / factorize_spd / cg_solve can run as the parity
// oracle (oracle/_ref). It is written from the API shape only; no Eigen
// source is reproduced.
//
// Numerics: SimplicialLDLT is an envelope (skyline) LDL^T in natural
// ordering, identity permutation. Real Eigen uses AMD ordering, so factors
// differ at round-off level; this only affects the ROM (an input fed
// byte-identically to the CPU oracle and the GPU path), never the hot path.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <thread>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum StorageOptions { ColMajor = 0, RowMajor = 1 };
constexpr int Dynamic = -1;
enum ComputationInfo { Success = 0, NumericalIssue = 1, InvalidInput = 3 };
enum UpLoType { Lower = 1, Upper = 2 };

template <typename T> class Map;

// ---------------------------------------------------------------- dense
template <typename Scalar, int Rows, int Cols, int Options = ColMajor>
class Matrix;

template <typename Scalar, int Options>
class Matrix<Scalar, Dynamic, 1, Options> {  // column vector
public:
    Matrix() = default;
    explicit Matrix(Index n) : v_(static_cast<std::size_t>(n), Scalar(0)) {}
    Index size() const { return static_cast<Index>(v_.size()); }
    Index rows() const { return size(); }
    Scalar* data() { return v_.data(); }
    const Scalar* data() const { return v_.data(); }
    Scalar& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
    const Scalar& operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
    Scalar& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
    const Scalar& operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
    void resize(Index n) { v_.assign(static_cast<std::size_t>(n), Scalar(0)); }

private:
    std::vector<Scalar> v_;
};

using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXi = Matrix<int, Dynamic, 1>;

template <typename Scalar, int Options>
class Map<const Matrix<Scalar, Dynamic, 1, Options>> {
public:
    Map(const Scalar* p, Index n) : p_(p), n_(n) {}
    Index size() const { return n_; }
    const Scalar* data() const { return p_; }
    const Scalar& operator[](Index i) const { return p_[i]; }

private:
    const Scalar* p_;
    Index n_;
};

// Row-major dynamic matrix views used by the condensation product in
// rom.cpp:232-242 (C = A^T * B, all row-major).
template <typename Scalar>
class Matrix<Scalar, Dynamic, Dynamic, RowMajor> {
public:
    Matrix() = default;
};

template <typename Scalar>
struct RowMajorTransposeExpr {
    const Scalar* p;
    Index rows, cols;  // of the un-transposed operand
};

template <typename Scalar>
struct TransposeTimesExpr {
    RowMajorTransposeExpr<Scalar> a;  // A (rows x cols); product uses A^T
    const Scalar* b;
    Index b_rows, b_cols;
};

template <typename Scalar>
class Map<const Matrix<Scalar, Dynamic, Dynamic, RowMajor>> {
public:
    Map(const Scalar* p, Index r, Index c) : p_(p), r_(r), c_(c) {}
    RowMajorTransposeExpr<Scalar> transpose() const { return {p_, r_, c_}; }
    const Scalar* data() const { return p_; }
    Index rows() const { return r_; }
    Index cols() const { return c_; }

private:
    const Scalar* p_;
    Index r_, c_;
};

template <typename Scalar>
TransposeTimesExpr<Scalar> operator*(const RowMajorTransposeExpr<Scalar>& a,
                                     const Map<const Matrix<Scalar, Dynamic, Dynamic, RowMajor>>& b) {
    return {a, b.data(), b.rows(), b.cols()};
}

namespace standin {
inline unsigned worker_count(std::size_t work_items) {
    unsigned hw = std::thread::hardware_concurrency();
    if (hw == 0) hw = 1;
    if (hw > work_items) hw = static_cast<unsigned>(std::max<std::size_t>(work_items, 1));
    return hw;
}

template <typename F>
void parallel_rows(std::size_t n, F&& f) {
    unsigned nt = worker_count(n);
    std::vector<std::thread> pool;
    std::size_t chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        std::size_t b = t * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& th : pool) th.join();
}
}  // namespace standin

template <typename Scalar>
class NoAliasProxy {
public:
    NoAliasProxy(Scalar* p, Index r, Index c) : p_(p), r_(r), c_(c) {}
    // C (r x c) = A^T B, A: (K x r) row-major, B: (K x c) row-major.
    void operator=(const TransposeTimesExpr<Scalar>& e) {
        const Index K = e.a.rows;
        const Index R = e.a.cols, C = e.b_cols;
        standin::parallel_rows(static_cast<std::size_t>(R), [&](std::size_t rb, std::size_t re) {
            for (std::size_t i = rb; i < re; ++i)
                std::fill(p_ + i * C, p_ + (i + 1) * C, Scalar(0));
            constexpr Index kBlk = 64;
            for (Index k0 = 0; k0 < K; k0 += kBlk) {
                Index k1 = std::min(K, k0 + kBlk);
                for (std::size_t i = rb; i < re; ++i) {
                    Scalar* crow = p_ + i * C;
                    for (Index k = k0; k < k1; ++k) {
                        Scalar a = e.a.p[k * R + static_cast<Index>(i)];
                        if (a == Scalar(0)) continue;
                        const Scalar* brow = e.b + k * C;
                        for (Index j = 0; j < C; ++j) crow[j] += a * brow[j];
                    }
                }
            }
        });
        (void)r_;
        (void)c_;
    }

private:
    Scalar* p_;
    Index r_, c_;
};

template <typename Scalar>
class Map<Matrix<Scalar, Dynamic, Dynamic, RowMajor>> {
public:
    Map(Scalar* p, Index r, Index c) : p_(p), r_(r), c_(c) {}
    NoAliasProxy<Scalar> noalias() { return {p_, r_, c_}; }

private:
    Scalar* p_;
    Index r_, c_;
};

// --------------------------------------------------------------- sparse
template <typename Scalar, int Options = ColMajor, typename StorageIndex = int>
class SparseMatrix;

template <typename Scalar, typename StorageIndex>
class Map<const SparseMatrix<Scalar, RowMajor, StorageIndex>> {
public:
    Map(Index rows, Index cols, Index nnz, const StorageIndex* outer, const StorageIndex* inner,
        const Scalar* values)
        : rows_(rows), cols_(cols), nnz_(nnz), outer_(outer), inner_(inner), values_(values) {}
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index nonZeros() const { return nnz_; }
    const StorageIndex* outerIndexPtr() const { return outer_; }
    const StorageIndex* innerIndexPtr() const { return inner_; }
    const Scalar* valuePtr() const { return values_; }

private:
    Index rows_, cols_, nnz_;
    const StorageIndex* outer_;
    const StorageIndex* inner_;
    const Scalar* values_;
};

/// Column-major compressed sparse matrix (the solver input type).
template <typename Scalar, int Options, typename StorageIndex>
class SparseMatrix {
public:
    SparseMatrix() = default;
    // Conversion from a row-major CSR view: transpose the storage order.
    template <typename SI>
    SparseMatrix(const Map<const SparseMatrix<Scalar, RowMajor, SI>>& m)  // NOLINT(implicit)
        : rows_(m.rows()), cols_(m.cols()) {
        const Index nnz = m.nonZeros();
        outer_.assign(static_cast<std::size_t>(cols_) + 1, 0);
        inner_.resize(static_cast<std::size_t>(nnz));
        values_.resize(static_cast<std::size_t>(nnz));
        const SI* ro = m.outerIndexPtr();
        const SI* ci = m.innerIndexPtr();
        const Scalar* v = m.valuePtr();
        for (Index k = 0; k < nnz; ++k) ++outer_[static_cast<std::size_t>(ci[k]) + 1];
        for (Index c = 0; c < cols_; ++c) outer_[c + 1] += outer_[c];
        std::vector<StorageIndex> fill(outer_.begin(), outer_.end() - 1);
        for (Index r = 0; r < rows_; ++r)
            for (SI k = ro[r]; k < ro[r + 1]; ++k) {
                StorageIndex dst = fill[static_cast<std::size_t>(ci[k])]++;
                inner_[dst] = static_cast<StorageIndex>(r);
                values_[dst] = v[k];
            }
    }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    const std::vector<StorageIndex>& outer() const { return outer_; }
    const std::vector<StorageIndex>& inner() const { return inner_; }
    const std::vector<Scalar>& values() const { return values_; }

private:
    Index rows_ = 0, cols_ = 0;
    std::vector<StorageIndex> outer_, inner_;
    std::vector<Scalar> values_;
};

template <typename StorageIndex>
class PermutationMatrix {
public:
    const VectorXi& indices() const { return idx_; }
    VectorXi& indices() { return idx_; }

private:
    VectorXi idx_;
};

/// Envelope LDL^T (natural ordering) of a symmetric matrix given in full
/// column-major storage; only the lower triangle is read.
template <typename MatrixType>
class SimplicialLDLT {
public:
    SimplicialLDLT() = default;

    SimplicialLDLT& compute(const MatrixType& a) {
        n_ = a.rows();
        info_ = Success;
        const auto& outer = a.outer();
        const auto& inner = a.inner();
        const auto& vals = a.values();
        // Lower triangle of column c == upper triangle of row c (symmetry):
        // row i of L spans [first_[i], i). Entries of column i with row
        // index r <= i give A(i, r).
        first_.assign(static_cast<std::size_t>(n_), 0);
        for (Index i = 0; i < n_; ++i) {
            Index f = i;
            for (auto k = outer[i]; k < outer[i + 1]; ++k)
                if (inner[k] < f && vals[k] != 0.0) f = inner[k];
            first_[i] = f;
        }
        ptr_.assign(static_cast<std::size_t>(n_) + 1, 0);
        for (Index i = 0; i < n_; ++i) ptr_[i + 1] = ptr_[i] + (i - first_[i]);
        env_.assign(static_cast<std::size_t>(ptr_[n_]), 0.0);
        d_.resize(n_);
        std::vector<double> diag(static_cast<std::size_t>(n_), 0.0);
        for (Index i = 0; i < n_; ++i)
            for (auto k = outer[i]; k < outer[i + 1]; ++k) {
                Index r = inner[k];
                if (r == i) diag[i] += vals[k];
                else if (r < i && r >= first_[i]) env_[ptr_[i] + (r - first_[i])] = vals[k];
            }
        // Row-oriented Crout: g_j = A(i,j) - sum_k g_k L(j,k); L(i,j) = g_j / d_j.
        for (Index i = 0; i < n_; ++i) {
            const Index fi = first_[i];
            double* gi = env_.data() + ptr_[i];  // holds g, then L(i, .)
            for (Index j = fi; j < i; ++j) {
                const Index fj = first_[j];
                const Index k0 = std::max(fi, fj);
                const double* lj = env_.data() + ptr_[j] + (k0 - fj);
                const double* gk = gi + (k0 - fi);
                const Index len = j - k0;
                double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
                Index k = 0;
                for (; k + 4 <= len; k += 4) {
                    s0 += gk[k] * lj[k];
                    s1 += gk[k + 1] * lj[k + 1];
                    s2 += gk[k + 2] * lj[k + 2];
                    s3 += gk[k + 3] * lj[k + 3];
                }
                for (; k < len; ++k) s0 += gk[k] * lj[k];
                gi[j - fi] -= (s0 + s1) + (s2 + s3);
            }
            double di = diag[i];
            for (Index j = fi; j < i; ++j) {
                double g = gi[j - fi];
                double l = g / d_[j];
                di -= g * l;
                gi[j - fi] = l;
            }
            d_[i] = di;
            if (!std::isfinite(di) || di == 0.0) info_ = NumericalIssue;
        }
        perm_.indices().resize(n_);
        for (Index i = 0; i < n_; ++i) perm_.indices()[i] = static_cast<int>(i);
        return *this;
    }

    ComputationInfo info() const { return info_; }
    const VectorXd& vectorD() const { return d_; }
    const PermutationMatrix<int>& permutationPinv() const { return perm_; }

    template <typename Rhs>
    VectorXd solve(const Rhs& b) const {
        VectorXd x(n_);
        for (Index i = 0; i < n_; ++i) x[i] = b[i];
        // L y = b
        for (Index i = 0; i < n_; ++i) {
            const Index fi = first_[i];
            const double* li = env_.data() + ptr_[i];
            const double* xk = x.data() + fi;
            double s = 0.0;
            for (Index k = 0; k < i - fi; ++k) s += li[k] * xk[k];
            x[i] -= s;
        }
        for (Index i = 0; i < n_; ++i) x[i] /= d_[i];
        // L^T x = z
        for (Index i = n_ - 1; i >= 0; --i) {
            const Index fi = first_[i];
            const double* li = env_.data() + ptr_[i];
            double xi = x[i];
            double* xk = x.data() + fi;
            for (Index k = 0; k < i - fi; ++k) xk[k] -= li[k] * xi;
        }
        return x;
    }

private:
    Index n_ = 0;
    ComputationInfo info_ = Success;
    std::vector<Index> first_;
    std::vector<std::size_t> ptr_;
    std::vector<double> env_;
    VectorXd d_;
    PermutationMatrix<int> perm_;
};

}  // namespace Eigen
