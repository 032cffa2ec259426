// TEST INFRASTRUCTURE ONLY (oracle/).  A stand-in for the subset of Eigen
// 3.4 the reference library uses (/root/reference/proj), so
// that the reference's own sources compile here, unmodified, into
// oracle/_ref/ and pin the oracle restatement (oracle/octen_oracle.py) and
// the device path against the reference itself.  Eigen is a third-party
// dependency absent from the container; this header restates the published
// semantics of the pieces the reference calls:
//
//   * MatrixXd / VectorXd: column-major fp64, block views that write through
//     (col, row, topRows, middleRows, leftCols, segment, ...), comma
//     initializer, Map / Ref views.  Every expression is evaluated eagerly
//     into a temporary, so aliasing (v = v.cwiseProduct(g)) is safe.
//   * products: OpenBLAS dgemm (scipy's bundled libscipy_openblas), a plain
//     k-ordered loop for tiny products.  Rounding differs from Eigen's own
//     GEMM at the 1e-16 relative level.
//   * ColPivHouseholderQR: dgeqp3; rank() = #{i : |r_ii| > thr * max|r_kk|}
//     with thr = setThreshold() or eps * min(m, n) (Eigen's default);
//     solve() is Eigen's basic solution over the nonzero pivots (Eigen's
//     eps-level pivot cut-off), zeros elsewhere.
//   * CompleteOrthogonalDecomposition: the same pivoted QR and rank rule,
//     then the minimum-norm solution of the leading rank rows.
//   * FullPivLU: full pivoting with Eigen's rank rule (|u_ii| > eps * n *
//     max pivot), inverse() from the factors.
//   * LLT: dpotrf (the same "pivot <= 0 or NaN" failure test as Eigen),
//     matrixL().solve() by dtrsm.
//   * JacobiSVD / BDCSVD: dgesvd / dgesdd (thin U, V); singular vectors may
//     differ from Eigen's by a sign per pair, which the reference's uses
//     (rank-1 peel, subspace bases) are invariant to up to column signs.
//   * EigenSolver: dgeev; real eigenvectors normalised to unit 2-norm like
//     Eigen's; a complex pair's vectors come out with LAPACK's phase, and
//     the Schur-order of the eigenvalues can differ from Eigen's.
// Where a convention can differ (eigen/singular vector signs, column order
// of the GEVD init) the parity tests compare permutation- and
// sign-invariant quantities (fits, congruence, residuals).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <concepts>
#include <cstddef>
#include <cstring>
#include <initializer_list>
#include <limits>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

extern "C" {
void scipy_dgemm_(const char*, const char*, const int*, const int*, const int*, const double*, const double*,
                  const int*, const double*, const int*, const double*, double*, const int*, std::size_t,
                  std::size_t);
void scipy_dgeqp3_(const int*, const int*, double*, const int*, int*, double*, double*, const int*, int*);
void scipy_dgeqrf_(const int*, const int*, double*, const int*, double*, double*, const int*, int*);
void scipy_dormqr_(const char*, const char*, const int*, const int*, const int*, const double*, const int*,
                   const double*, double*, const int*, double*, const int*, int*, std::size_t, std::size_t);
void scipy_dtrsm_(const char*, const char*, const char*, const char*, const int*, const int*, const double*,
                  const double*, const int*, double*, const int*, std::size_t, std::size_t, std::size_t,
                  std::size_t);
void scipy_dgesdd_(const char*, const int*, const int*, double*, const int*, double*, double*, const int*, double*,
                   const int*, double*, const int*, int*, int*, std::size_t);
void scipy_dgesvd_(const char*, const char*, const int*, const int*, double*, const int*, double*, double*,
                   const int*, double*, const int*, double*, const int*, int*, std::size_t, std::size_t);
void scipy_dgeev_(const char*, const char*, const int*, double*, const int*, double*, double*, double*, const int*,
                  double*, const int*, double*, const int*, int*, std::size_t, std::size_t);
void scipy_dpotrf_(const char*, const int*, double*, const int*, int*, std::size_t);
}

namespace Eigen {

using Index = std::ptrdiff_t;

enum DecompositionOptions { ComputeFullU = 0x04, ComputeThinU = 0x08, ComputeFullV = 0x10, ComputeThinV = 0x20 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

namespace shim {
struct CV {  // read-only strided view
    const double* p;
    Index r, c, ld;
    double at(Index i, Index j) const { return p[i + ld * j]; }
};
struct MV {  // writable strided view
    double* p;
    Index r, c, ld;
    double& at(Index i, Index j) const { return p[i + ld * j]; }
};
inline void fail(const char* what) { throw std::logic_error(std::string("eigen shim: ") + what); }
inline int to_int(Index v) {
    if (v < 0 || v > std::numeric_limits<int>::max()) fail("extent exceeds LAPACK int range");
    return static_cast<int>(v);
}
}  // namespace shim

struct DenseTag {};
template <class T>
concept Dense = std::is_base_of_v<DenseTag, std::remove_cvref_t<T>>;

class MatrixXd;
class VectorXd;
class Block;
class ConstBlock;
class DiagonalWrapper;

template <class D>
struct DenseBase : DenseTag {
    shim::CV cv() const { return static_cast<const D&>(*this).cview(); }
    Index rows() const { return cv().r; }
    Index cols() const { return cv().c; }
    Index size() const { return cv().r * cv().c; }
    double operator()(Index i, Index j) const { return cv().at(i, j); }
    double operator()(Index i) const {
        const shim::CV v = cv();
        return v.c == 1 ? v.p[i] : v.p[v.ld * i];
    }
    double operator[](Index i) const { return (*this)(i); }
    double coeff(Index i, Index j) const { return cv().at(i, j); }
    double coeff(Index i) const { return (*this)(i); }
    double value() const { return cv().at(0, 0); }

    template <class F>
    void each(F&& f) const {
        const shim::CV v = cv();
        for (Index j = 0; j < v.c; ++j)
            for (Index i = 0; i < v.r; ++i) f(v.at(i, j));
    }
    double sum() const {
        double s = 0.0;
        each([&](double x) { s += x; });
        return s;
    }
    double prod() const {
        double s = 1.0;
        each([&](double x) { s *= x; });
        return s;
    }
    double mean() const { return sum() / static_cast<double>(size()); }
    double squaredNorm() const {
        double s = 0.0;
        each([&](double x) { s += x * x; });
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    double maxCoeff() const {
        if (size() == 0) shim::fail("maxCoeff of an empty matrix");
        double m = -std::numeric_limits<double>::infinity();
        bool first = true;
        each([&](double x) {
            if (first || x > m) m = x;
            first = false;
        });
        return m;
    }
    double minCoeff() const {
        if (size() == 0) shim::fail("minCoeff of an empty matrix");
        double m = std::numeric_limits<double>::infinity();
        bool first = true;
        each([&](double x) {
            if (first || x < m) m = x;
            first = false;
        });
        return m;
    }
    // first occurrence in column-major order (Eigen's visitor)
    double maxCoeff(Index* row, Index* col) const {
        const shim::CV v = cv();
        double m = v.at(0, 0);
        Index bi = 0, bj = 0;
        for (Index j = 0; j < v.c; ++j)
            for (Index i = 0; i < v.r; ++i)
                if (v.at(i, j) > m) {
                    m = v.at(i, j);
                    bi = i;
                    bj = j;
                }
        if (row) *row = bi;
        if (col) *col = bj;
        return m;
    }
    double minCoeff(Index* row, Index* col) const {
        const shim::CV v = cv();
        double m = v.at(0, 0);
        Index bi = 0, bj = 0;
        for (Index j = 0; j < v.c; ++j)
            for (Index i = 0; i < v.r; ++i)
                if (v.at(i, j) < m) {
                    m = v.at(i, j);
                    bi = i;
                    bj = j;
                }
        if (row) *row = bi;
        if (col) *col = bj;
        return m;
    }
    double maxCoeff(Index* idx) const {
        Index i = 0, j = 0;
        const double m = maxCoeff(&i, &j);
        if (idx) *idx = cv().c == 1 ? i : j;
        return m;
    }
    double minCoeff(Index* idx) const {
        Index i = 0, j = 0;
        const double m = minCoeff(&i, &j);
        if (idx) *idx = cv().c == 1 ? i : j;
        return m;
    }
    bool allFinite() const {
        bool ok = true;
        each([&](double x) { ok = ok && std::isfinite(x); });
        return ok;
    }
    bool hasNaN() const {
        bool n = false;
        each([&](double x) { n = n || std::isnan(x); });
        return n;
    }
    template <Dense O>
    double dot(const O& o) const {
        const shim::CV a = cv(), b = o.cv();
        if (a.r * a.c != b.r * b.c) shim::fail("dot: size mismatch");
        double s = 0.0;
        Index k = 0;
        for (Index j = 0; j < a.c; ++j)
            for (Index i = 0; i < a.r; ++i, ++k) {
                const Index bi = b.c == 1 ? k : 0, bj = b.c == 1 ? 0 : k;
                s += a.at(i, j) * b.at(bi, bj);
            }
        return s;
    }
    MatrixXd transpose() const;
    MatrixXd cwiseAbs() const;
    MatrixXd cwiseAbs2() const;
    MatrixXd cwiseSqrt() const;
    template <Dense O>
    MatrixXd cwiseProduct(const O& o) const;
    template <Dense O>
    MatrixXd cwiseQuotient(const O& o) const;
    template <Dense O>
    MatrixXd cwiseMax(const O& o) const;
    template <Dense O>
    MatrixXd cwiseMin(const O& o) const;
    MatrixXd normalized() const;
    MatrixXd eval() const;
    DiagonalWrapper asDiagonal() const;
    MatrixXd diagonal() const;
    template <Dense O>
    bool isApprox(const O& o, double prec = 1e-12) const;

    ConstBlock block(Index i, Index j, Index r, Index c) const;
    ConstBlock col(Index j) const;
    ConstBlock row(Index i) const;
    ConstBlock topRows(Index n) const;
    ConstBlock bottomRows(Index n) const;
    ConstBlock middleRows(Index s, Index n) const;
    ConstBlock leftCols(Index n) const;
    ConstBlock rightCols(Index n) const;
    ConstBlock middleCols(Index s, Index n) const;
    ConstBlock topLeftCorner(Index r, Index c) const;
    ConstBlock head(Index n) const;
    ConstBlock tail(Index n) const;
    ConstBlock segment(Index s, Index n) const;
};

// Comma initializer (row-major fill of scalars and blocks, Eigen's rules).
class CommaInit {
public:
    CommaInit(shim::MV t) : t_(t) {}
    CommaInit& operator,(double v) {
        if (col_ == t_.c) {
            row_ += cur_rows_;
            col_ = 0;
            cur_rows_ = 1;
        }
        if (row_ >= t_.r || col_ >= t_.c) shim::fail("comma initializer: too many coefficients");
        t_.at(row_, col_) = v;
        ++col_;
        if (cur_rows_ == 0) cur_rows_ = 1;
        return *this;
    }
    template <Dense O>
    CommaInit& operator,(const O& o) {
        const shim::CV b = o.cv();
        if (col_ == t_.c && (b.c != 0 || b.r != cur_rows_)) {
            row_ += cur_rows_;
            col_ = 0;
            cur_rows_ = b.r;
        }
        if (col_ == 0) cur_rows_ = b.r;
        if (row_ + b.r > t_.r || col_ + b.c > t_.c) shim::fail("comma initializer: block does not fit");
        for (Index j = 0; j < b.c; ++j)
            for (Index i = 0; i < b.r; ++i) t_.at(row_ + i, col_ + j) = b.at(i, j);
        col_ += b.c;
        return *this;
    }

private:
    shim::MV t_;
    Index row_ = 0, col_ = 0, cur_rows_ = 0;
};

template <class D>
struct MutableBase : DenseBase<D> {
    using DenseBase<D>::operator();
    using DenseBase<D>::block;
    using DenseBase<D>::col;
    using DenseBase<D>::row;
    using DenseBase<D>::topRows;
    using DenseBase<D>::bottomRows;
    using DenseBase<D>::middleRows;
    using DenseBase<D>::leftCols;
    using DenseBase<D>::rightCols;
    using DenseBase<D>::middleCols;
    using DenseBase<D>::topLeftCorner;
    using DenseBase<D>::head;
    using DenseBase<D>::tail;
    using DenseBase<D>::segment;
    shim::MV mv() { return static_cast<D&>(*this).mview(); }
    double& operator()(Index i, Index j) { return mv().at(i, j); }
    double& operator()(Index i) {
        const shim::MV v = mv();
        return v.c == 1 ? v.p[i] : v.p[v.ld * i];
    }
    double& operator[](Index i) { return (*this)(i); }
    double& coeffRef(Index i, Index j) { return mv().at(i, j); }
    double& coeffRef(Index i) { return (*this)(i); }
    double* data() { return mv().p; }
    const double* data() const { return this->cv().p; }

    template <class F>
    void apply(F&& f) {
        const shim::MV v = mv();
        for (Index j = 0; j < v.c; ++j)
            for (Index i = 0; i < v.r; ++i) f(v.at(i, j));
    }
    D& setConstant(double x) {
        apply([&](double& e) { e = x; });
        return static_cast<D&>(*this);
    }
    D& setZero() { return setConstant(0.0); }
    D& setOnes() { return setConstant(1.0); }
    D& fill(double x) { return setConstant(x); }
    D& setIdentity() {
        const shim::MV v = mv();
        for (Index j = 0; j < v.c; ++j)
            for (Index i = 0; i < v.r; ++i) v.at(i, j) = (i == j) ? 1.0 : 0.0;
        return static_cast<D&>(*this);
    }
    void normalize() {
        const double n = this->norm();
        if (n > 0.0) apply([&](double& e) { e /= n; });
    }
    D& operator*=(double s) {
        apply([&](double& e) { e *= s; });
        return static_cast<D&>(*this);
    }
    D& operator/=(double s) {
        apply([&](double& e) { e /= s; });
        return static_cast<D&>(*this);
    }
    template <Dense O>
    D& operator+=(const O& o);
    template <Dense O>
    D& operator-=(const O& o);
    template <Dense O>
    D& operator*=(const O& o);
    CommaInit operator<<(double v) {
        CommaInit ci(mv());
        ci, v;
        return ci;
    }
    template <Dense O>
    CommaInit operator<<(const O& o) {
        CommaInit ci(mv());
        ci, o;
        return ci;
    }

    Block block(Index i, Index j, Index r, Index c);
    Block col(Index j);
    Block row(Index i);
    Block topRows(Index n);
    Block bottomRows(Index n);
    Block middleRows(Index s, Index n);
    Block leftCols(Index n);
    Block rightCols(Index n);
    Block middleCols(Index s, Index n);
    Block topLeftCorner(Index r, Index c);
    Block head(Index n);
    Block tail(Index n);
    Block segment(Index s, Index n);

protected:
    void copy_in(const shim::CV& src) {
        const shim::MV d = mv();
        if (src.r != d.r || src.c != d.c) shim::fail("block assignment: size mismatch");
        for (Index j = 0; j < d.c; ++j)
            for (Index i = 0; i < d.r; ++i) d.at(i, j) = src.at(i, j);
    }
};

class MatrixXd : public MutableBase<MatrixXd> {
public:
    MatrixXd() = default;
    MatrixXd(Index r, Index c) : r_(r), c_(c), v_(static_cast<std::size_t>(r * c), 0.0) {
        if (r < 0 || c < 0) shim::fail("negative extent");
    }
    MatrixXd(const MatrixXd&) = default;
    MatrixXd(MatrixXd&&) noexcept = default;
    template <Dense O>
        requires(!std::is_base_of_v<MatrixXd, std::remove_cvref_t<O>>)
    MatrixXd(const O& o) {
        from(o.cv());
    }
    MatrixXd& operator=(const MatrixXd&) = default;
    MatrixXd& operator=(MatrixXd&&) noexcept = default;
    template <Dense O>
        requires(!std::is_base_of_v<MatrixXd, std::remove_cvref_t<O>>)
    MatrixXd& operator=(const O& o) {
        MatrixXd t;
        t.from(o.cv());
        swap(t);
        return *this;
    }
    shim::CV cview() const { return {v_.data(), r_, c_, r_}; }
    shim::MV mview() { return {v_.data(), r_, c_, r_}; }
    void resize(Index r, Index c) {
        if (r * c != r_ * c_) v_.assign(static_cast<std::size_t>(r * c), 0.0);
        r_ = r;
        c_ = c;
    }
    void conservativeResize(Index r, Index c) {
        MatrixXd t(r, c);
        for (Index j = 0; j < std::min(c, c_); ++j)
            for (Index i = 0; i < std::min(r, r_); ++i) t(i, j) = (*this)(i, j);
        swap(t);
    }
    void swap(MatrixXd& o) noexcept {
        std::swap(r_, o.r_);
        std::swap(c_, o.c_);
        v_.swap(o.v_);
    }
    static MatrixXd Constant(Index r, Index c, double x) {
        MatrixXd m(r, c);
        m.setConstant(x);
        return m;
    }
    static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
    static MatrixXd Ones(Index r, Index c) { return Constant(r, c, 1.0); }
    static MatrixXd Identity(Index r, Index c) {
        MatrixXd m(r, c);
        m.setIdentity();
        return m;
    }

protected:
    void from(const shim::CV& s) {
        r_ = s.r;
        c_ = s.c;
        v_.assign(static_cast<std::size_t>(s.r * s.c), 0.0);
        for (Index j = 0; j < s.c; ++j)
            for (Index i = 0; i < s.r; ++i) v_[static_cast<std::size_t>(i + r_ * j)] = s.at(i, j);
    }
    Index r_ = 0, c_ = 0;
    std::vector<double> v_;
};

class VectorXd : public MatrixXd {
public:
    VectorXd() : MatrixXd(0, 1) {}
    explicit VectorXd(Index n) : MatrixXd(n, 1) {}
    VectorXd(const VectorXd&) = default;
    VectorXd(VectorXd&&) noexcept = default;
    template <Dense O>
        requires(!std::is_same_v<std::remove_cvref_t<O>, VectorXd>)
    VectorXd(const O& o) {
        from(o.cv());
        as_column();
    }
    VectorXd& operator=(const VectorXd&) = default;
    VectorXd& operator=(VectorXd&&) noexcept = default;
    template <Dense O>
        requires(!std::is_same_v<std::remove_cvref_t<O>, VectorXd>)
    VectorXd& operator=(const O& o) {
        VectorXd t(o);
        swap(t);
        return *this;
    }
    void resize(Index n) { MatrixXd::resize(n, 1); }
    void resize(Index r, Index c) {
        if (c != 1) shim::fail("VectorXd::resize with cols != 1");
        MatrixXd::resize(r, 1);
    }
    static VectorXd Constant(Index n, double x) {
        VectorXd v(n);
        v.setConstant(x);
        return v;
    }
    static VectorXd Zero(Index n) { return VectorXd(n); }
    static VectorXd Ones(Index n) { return Constant(n, 1.0); }
    static VectorXd LinSpaced(Index n, double lo, double hi) {
        VectorXd v(n);
        for (Index i = 0; i < n; ++i) v(i) = n > 1 ? lo + (hi - lo) * double(i) / double(n - 1) : hi;
        return v;
    }

private:
    void as_column() {
        if (c_ == 1) return;
        if (r_ == 1 || r_ * c_ == 0) {
            r_ = r_ * c_;
            c_ = 1;
            return;
        }
        shim::fail("VectorXd from a matrix with several columns");
    }
};

class Block : public MutableBase<Block> {
public:
    Block(double* p, Index r, Index c, Index ld) : p_(p), r_(r), c_(c), ld_(ld) {}
    Block(const Block&) = default;  // a view of the same coefficients
    Block& operator=(const Block& o) {
        const MatrixXd t(o);
        copy_in(t.cview());
        return *this;
    }
    template <Dense O>
    Block& operator=(const O& o) {
        const MatrixXd t(o);
        copy_in(t.cview());
        return *this;
    }
    shim::CV cview() const { return {p_, r_, c_, ld_}; }
    shim::MV mview() { return {p_, r_, c_, ld_}; }

private:
    double* p_;
    Index r_, c_, ld_;
};

class ConstBlock : public DenseBase<ConstBlock> {
public:
    ConstBlock(const double* p, Index r, Index c, Index ld) : p_(p), r_(r), c_(c), ld_(ld) {}
    shim::CV cview() const { return {p_, r_, c_, ld_}; }
    const double* data() const { return p_; }

private:
    const double* p_;
    Index r_, c_, ld_;
};

template <class T>
class Map;
template <>
class Map<const MatrixXd> : public ConstBlock {
public:
    Map(const double* p, Index r, Index c) : ConstBlock(p, r, c, r > 0 ? r : 1) {}
};
template <>
class Map<MatrixXd> : public Block {
public:
    Map(double* p, Index r, Index c) : Block(p, r, c, r > 0 ? r : 1) {}
    using Block::operator=;
};
template <>
class Map<const VectorXd> : public ConstBlock {
public:
    Map(const double* p, Index n) : ConstBlock(p, n, 1, n > 0 ? n : 1) {}
};
template <>
class Map<VectorXd> : public Block {
public:
    Map(double* p, Index n) : Block(p, n, 1, n > 0 ? n : 1) {}
    using Block::operator=;
};

template <class T>
class Ref;
template <>
class Ref<MatrixXd> : public Block {
public:
    Ref(MatrixXd& m) : Block(m.data(), m.rows(), m.cols(), m.rows() > 0 ? m.rows() : 1) {}
    Ref(const Block& b) : Block(b) {}
    using Block::operator=;
};
template <>
class Ref<const MatrixXd> : public ConstBlock {
public:
    template <Dense O>
    Ref(const O& o) : ConstBlock(o.cv().p, o.cv().r, o.cv().c, o.cv().ld) {}
};

// ---- block accessors
namespace shim {
inline void check_range(Index s, Index n, Index ext) {
    if (s < 0 || n < 0 || s + n > ext) fail("block out of range");
}
}  // namespace shim
template <class D>
ConstBlock DenseBase<D>::block(Index i, Index j, Index r, Index c) const {
    const shim::CV v = cv();
    shim::check_range(i, r, v.r);
    shim::check_range(j, c, v.c);
    return ConstBlock(v.p + i + v.ld * j, r, c, v.ld);
}
template <class D>
ConstBlock DenseBase<D>::col(Index j) const {
    return block(0, j, rows(), 1);
}
template <class D>
ConstBlock DenseBase<D>::row(Index i) const {
    return block(i, 0, 1, cols());
}
template <class D>
ConstBlock DenseBase<D>::topRows(Index n) const {
    return block(0, 0, n, cols());
}
template <class D>
ConstBlock DenseBase<D>::bottomRows(Index n) const {
    return block(rows() - n, 0, n, cols());
}
template <class D>
ConstBlock DenseBase<D>::middleRows(Index s, Index n) const {
    return block(s, 0, n, cols());
}
template <class D>
ConstBlock DenseBase<D>::leftCols(Index n) const {
    return block(0, 0, rows(), n);
}
template <class D>
ConstBlock DenseBase<D>::rightCols(Index n) const {
    return block(0, cols() - n, rows(), n);
}
template <class D>
ConstBlock DenseBase<D>::middleCols(Index s, Index n) const {
    return block(0, s, rows(), n);
}
template <class D>
ConstBlock DenseBase<D>::topLeftCorner(Index r, Index c) const {
    return block(0, 0, r, c);
}
template <class D>
ConstBlock DenseBase<D>::segment(Index s, Index n) const {
    return cols() == 1 ? block(s, 0, n, 1) : block(0, s, 1, n);
}
template <class D>
ConstBlock DenseBase<D>::head(Index n) const {
    return segment(0, n);
}
template <class D>
ConstBlock DenseBase<D>::tail(Index n) const {
    return segment(size() - n, n);
}

template <class D>
Block MutableBase<D>::block(Index i, Index j, Index r, Index c) {
    const shim::MV v = mv();
    shim::check_range(i, r, v.r);
    shim::check_range(j, c, v.c);
    return Block(v.p + i + v.ld * j, r, c, v.ld > 0 ? v.ld : 1);
}
template <class D>
Block MutableBase<D>::col(Index j) {
    return block(0, j, this->rows(), 1);
}
template <class D>
Block MutableBase<D>::row(Index i) {
    return block(i, 0, 1, this->cols());
}
template <class D>
Block MutableBase<D>::topRows(Index n) {
    return block(0, 0, n, this->cols());
}
template <class D>
Block MutableBase<D>::bottomRows(Index n) {
    return block(this->rows() - n, 0, n, this->cols());
}
template <class D>
Block MutableBase<D>::middleRows(Index s, Index n) {
    return block(s, 0, n, this->cols());
}
template <class D>
Block MutableBase<D>::leftCols(Index n) {
    return block(0, 0, this->rows(), n);
}
template <class D>
Block MutableBase<D>::rightCols(Index n) {
    return block(0, this->cols() - n, this->rows(), n);
}
template <class D>
Block MutableBase<D>::middleCols(Index s, Index n) {
    return block(0, s, this->rows(), n);
}
template <class D>
Block MutableBase<D>::topLeftCorner(Index r, Index c) {
    return block(0, 0, r, c);
}
template <class D>
Block MutableBase<D>::segment(Index s, Index n) {
    return this->cols() == 1 ? block(s, 0, n, 1) : block(0, s, 1, n);
}
template <class D>
Block MutableBase<D>::head(Index n) {
    return segment(0, n);
}
template <class D>
Block MutableBase<D>::tail(Index n) {
    return segment(this->size() - n, n);
}

// ---- element-wise results
namespace shim {
template <class F>
MatrixXd map1(const CV& a, F&& f) {
    MatrixXd out(a.r, a.c);
    for (Index j = 0; j < a.c; ++j)
        for (Index i = 0; i < a.r; ++i) out(i, j) = f(a.at(i, j));
    return out;
}
template <class F>
MatrixXd map2(const CV& a, const CV& b, F&& f) {
    if (a.r != b.r || a.c != b.c) fail("element-wise operation: size mismatch");
    MatrixXd out(a.r, a.c);
    for (Index j = 0; j < a.c; ++j)
        for (Index i = 0; i < a.r; ++i) out(i, j) = f(a.at(i, j), b.at(i, j));
    return out;
}
}  // namespace shim

template <class D>
MatrixXd DenseBase<D>::transpose() const {
    const shim::CV a = cv();
    MatrixXd out(a.c, a.r);
    for (Index j = 0; j < a.c; ++j)
        for (Index i = 0; i < a.r; ++i) out(j, i) = a.at(i, j);
    return out;
}
template <class D>
MatrixXd DenseBase<D>::cwiseAbs() const {
    return shim::map1(cv(), [](double x) { return std::abs(x); });
}
template <class D>
MatrixXd DenseBase<D>::cwiseAbs2() const {
    return shim::map1(cv(), [](double x) { return x * x; });
}
template <class D>
MatrixXd DenseBase<D>::cwiseSqrt() const {
    return shim::map1(cv(), [](double x) { return std::sqrt(x); });
}
template <class D>
template <Dense O>
MatrixXd DenseBase<D>::cwiseProduct(const O& o) const {
    return shim::map2(cv(), o.cv(), [](double x, double y) { return x * y; });
}
template <class D>
template <Dense O>
MatrixXd DenseBase<D>::cwiseQuotient(const O& o) const {
    return shim::map2(cv(), o.cv(), [](double x, double y) { return x / y; });
}
template <class D>
template <Dense O>
MatrixXd DenseBase<D>::cwiseMax(const O& o) const {
    return shim::map2(cv(), o.cv(), [](double x, double y) { return std::max(x, y); });
}
template <class D>
template <Dense O>
MatrixXd DenseBase<D>::cwiseMin(const O& o) const {
    return shim::map2(cv(), o.cv(), [](double x, double y) { return std::min(x, y); });
}
template <class D>
MatrixXd DenseBase<D>::normalized() const {
    const double n = norm();
    return shim::map1(cv(), [n](double x) { return n > 0.0 ? x / n : x; });
}
template <class D>
MatrixXd DenseBase<D>::eval() const {
    return MatrixXd(static_cast<const D&>(*this));
}
template <class D>
MatrixXd DenseBase<D>::diagonal() const {
    const shim::CV a = cv();
    const Index n = std::min(a.r, a.c);
    MatrixXd out(n, 1);
    for (Index i = 0; i < n; ++i) out(i, 0) = a.at(i, i);
    return out;
}
template <class D>
template <Dense O>
bool DenseBase<D>::isApprox(const O& o, double prec) const {
    const MatrixXd d = shim::map2(cv(), o.cv(), [](double x, double y) { return x - y; });
    return d.norm() <= prec * std::min(norm(), MatrixXd(o).norm());
}

template <class D>
template <Dense O>
D& MutableBase<D>::operator+=(const O& o) {
    const MatrixXd t(o);
    const shim::MV d = mv();
    if (t.rows() != d.r || t.cols() != d.c) shim::fail("+=: size mismatch");
    for (Index j = 0; j < d.c; ++j)
        for (Index i = 0; i < d.r; ++i) d.at(i, j) += t(i, j);
    return static_cast<D&>(*this);
}
template <class D>
template <Dense O>
D& MutableBase<D>::operator-=(const O& o) {
    const MatrixXd t(o);
    const shim::MV d = mv();
    if (t.rows() != d.r || t.cols() != d.c) shim::fail("-=: size mismatch");
    for (Index j = 0; j < d.c; ++j)
        for (Index i = 0; i < d.r; ++i) d.at(i, j) -= t(i, j);
    return static_cast<D&>(*this);
}

// ---- diagonal wrapper
class DiagonalWrapper {
public:
    explicit DiagonalWrapper(MatrixXd d) : d_(std::move(d)) {}
    const MatrixXd& values() const { return d_; }
    Index size() const { return d_.size(); }

private:
    MatrixXd d_;
};
template <class D>
DiagonalWrapper DenseBase<D>::asDiagonal() const {
    MatrixXd v(static_cast<const D&>(*this));
    return DiagonalWrapper(std::move(v));
}

// ---- products and arithmetic
namespace shim {
inline MatrixXd product(const CV& a, const CV& b) {
    if (a.c != b.r) fail("product: inner dimensions differ");
    MatrixXd out(a.r, b.c);
    if (a.r == 0 || b.c == 0 || a.c == 0) return out;
    const double work = double(a.r) * double(a.c) * double(b.c);
    if (work < 32768.0) {
        for (Index j = 0; j < b.c; ++j)
            for (Index k = 0; k < a.c; ++k) {
                const double bk = b.at(k, j);
                for (Index i = 0; i < a.r; ++i) out(i, j) += a.at(i, k) * bk;
            }
        return out;
    }
    const int m = to_int(a.r), n = to_int(b.c), k = to_int(a.c);
    const int lda = to_int(std::max<Index>(a.ld, std::max<Index>(1, a.r)));
    const int ldb = to_int(std::max<Index>(b.ld, std::max<Index>(1, b.r)));
    const int ldc = m;
    const double one = 1.0, zero = 0.0;
    scipy_dgemm_("N", "N", &m, &n, &k, &one, a.p, &lda, b.p, &ldb, &zero, out.data(), &ldc, 1, 1);
    return out;
}
}  // namespace shim

template <Dense A, Dense B>
MatrixXd operator*(const A& a, const B& b) {
    return shim::product(a.cv(), b.cv());
}
template <Dense A>
MatrixXd operator*(const A& a, double s) {
    return shim::map1(a.cv(), [s](double x) { return x * s; });
}
template <Dense A>
MatrixXd operator*(double s, const A& a) {
    return shim::map1(a.cv(), [s](double x) { return s * x; });
}
template <Dense A>
MatrixXd operator/(const A& a, double s) {
    return shim::map1(a.cv(), [s](double x) { return x / s; });
}
template <Dense A, Dense B>
MatrixXd operator+(const A& a, const B& b) {
    return shim::map2(a.cv(), b.cv(), [](double x, double y) { return x + y; });
}
template <Dense A, Dense B>
MatrixXd operator-(const A& a, const B& b) {
    return shim::map2(a.cv(), b.cv(), [](double x, double y) { return x - y; });
}
template <Dense A>
MatrixXd operator-(const A& a) {
    return shim::map1(a.cv(), [](double x) { return -x; });
}
template <Dense A>
MatrixXd operator*(const A& a, const DiagonalWrapper& d) {
    const shim::CV m = a.cv();
    if (m.c != d.size()) shim::fail("matrix * diagonal: size mismatch");
    MatrixXd out(m.r, m.c);
    for (Index j = 0; j < m.c; ++j) {
        const double s = d.values()(j);
        for (Index i = 0; i < m.r; ++i) out(i, j) = m.at(i, j) * s;
    }
    return out;
}
template <Dense A>
MatrixXd operator*(const DiagonalWrapper& d, const A& a) {
    const shim::CV m = a.cv();
    if (m.r != d.size()) shim::fail("diagonal * matrix: size mismatch");
    MatrixXd out(m.r, m.c);
    for (Index j = 0; j < m.c; ++j)
        for (Index i = 0; i < m.r; ++i) out(i, j) = d.values()(i) * m.at(i, j);
    return out;
}
template <class D>
template <Dense O>
D& MutableBase<D>::operator*=(const O& o) {
    const MatrixXd t = *this * o;
    static_cast<D&>(*this) = t;
    return static_cast<D&>(*this);
}
template <Dense A, Dense B>
bool operator==(const A& a, const B& b) {
    const shim::CV x = a.cv(), y = b.cv();
    if (x.r != y.r || x.c != y.c) return false;
    for (Index j = 0; j < x.c; ++j)
        for (Index i = 0; i < x.r; ++i)
            if (!(x.at(i, j) == y.at(i, j))) return false;
    return true;
}
template <Dense A, Dense B>
bool operator!=(const A& a, const B& b) {
    return !(a == b);
}
template <Dense A>
std::ostream& operator<<(std::ostream& os, const A& a) {
    const shim::CV x = a.cv();
    for (Index i = 0; i < x.r; ++i) {
        for (Index j = 0; j < x.c; ++j) os << (j ? " " : "") << x.at(i, j);
        if (i + 1 < x.r) os << "\n";
    }
    return os;
}

// ---------------------------------------------------------------------------
// Decompositions
// ---------------------------------------------------------------------------
namespace shim {
constexpr double kEps = std::numeric_limits<double>::epsilon();

// dgeqp3: A P = Q R.  Returns the packed factors, tau, the 0-based column
// permutation (perm[k] = original column of pivot k) and max |r_kk|.
struct PivQR {
    MatrixXd qr;
    std::vector<double> tau;
    std::vector<Index> perm;
    double maxpivot = 0.0;
    Index m = 0, n = 0;
    void compute(const CV& a) {
        qr = MatrixXd(ConstBlock(a.p, a.r, a.c, a.ld));
        m = a.r;
        n = a.c;
        const Index k = std::min(m, n);
        tau.assign(static_cast<std::size_t>(std::max<Index>(k, 1)), 0.0);
        perm.assign(static_cast<std::size_t>(n), 0);
        maxpivot = 0.0;
        if (m == 0 || n == 0) {
            for (Index j = 0; j < n; ++j) perm[static_cast<std::size_t>(j)] = j;
            return;
        }
        const int mi = to_int(m), ni = to_int(n), lda = mi;
        std::vector<int> jpvt(static_cast<std::size_t>(n), 0);
        int info = 0, lwork = -1;
        double wq = 0.0;
        scipy_dgeqp3_(&mi, &ni, qr.data(), &lda, jpvt.data(), tau.data(), &wq, &lwork, &info);
        lwork = std::max(1, static_cast<int>(wq));
        std::vector<double> work(static_cast<std::size_t>(lwork));
        scipy_dgeqp3_(&mi, &ni, qr.data(), &lda, jpvt.data(), tau.data(), work.data(), &lwork, &info);
        if (info != 0) fail("dgeqp3 failed");
        for (Index j = 0; j < n; ++j) perm[static_cast<std::size_t>(j)] = jpvt[static_cast<std::size_t>(j)] - 1;
        for (Index i = 0; i < k; ++i) maxpivot = std::max(maxpivot, std::abs(qr(i, i)));
    }
    // Eigen ColPivHouseholderQR::rank(): |r_ii| > threshold * maxpivot
    Index rank(double thr) const {
        const double pre = std::abs(maxpivot) * thr;
        Index r = 0;
        for (Index i = 0; i < std::min(m, n); ++i)
            if (std::abs(qr(i, i)) > pre) ++r;
        return r;
    }
    // Eigen's m_nonzero_pivots: the first k whose remaining column norm^2
    // drops below (max initial column norm * eps)^2 * (m - k) / m; the pivot
    // column's remaining norm is |r_kk|.
    Index nonzero_pivots() const {
        const Index k = std::min(m, n);
        if (k == 0) return 0;
        const double helper = (maxpivot * kEps) * (maxpivot * kEps) / double(m);
        for (Index i = 0; i < k; ++i)
            if (qr(i, i) * qr(i, i) < helper * double(m - i)) return i;
        return k;
    }
    // c <- Q^T c (all m rows)
    void apply_qt(MatrixXd& c) const {
        const Index k = std::min(m, n);
        if (k == 0 || c.cols() == 0) return;
        const int mi = to_int(m), ni = to_int(c.cols()), ki = to_int(k), lda = to_int(m), ldc = to_int(m);
        int info = 0, lwork = -1;
        double wq = 0.0;
        scipy_dormqr_("L", "T", &mi, &ni, &ki, qr.data(), &lda, tau.data(), c.data(), &ldc, &wq, &lwork, &info, 1, 1);
        lwork = std::max(1, static_cast<int>(wq));
        std::vector<double> work(static_cast<std::size_t>(lwork));
        scipy_dormqr_("L", "T", &mi, &ni, &ki, qr.data(), &lda, tau.data(), c.data(), &ldc, work.data(), &lwork,
                      &info, 1, 1);
        if (info != 0) fail("dormqr failed");
    }
};
inline void upper_solve(const MatrixXd& r, Index k, MatrixXd& x) {  // R[0:k,0:k] x[0:k,:] = x[0:k,:]
    for (Index c = 0; c < x.cols(); ++c)
        for (Index i = k - 1; i >= 0; --i) {
            double s = x(i, c);
            for (Index j = i + 1; j < k; ++j) s -= r(i, j) * x(j, c);
            x(i, c) = s / r(i, i);
        }
}
}  // namespace shim

template <class M>
class ColPivHouseholderQR {
public:
    ColPivHouseholderQR() = default;
    template <Dense A>
    explicit ColPivHouseholderQR(const A& a) {
        compute(a);
    }
    template <Dense A>
    ColPivHouseholderQR& compute(const A& a) {
        f_.compute(a.cv());
        return *this;
    }
    ColPivHouseholderQR& setThreshold(double t) {
        thr_ = t;
        user_thr_ = true;
        return *this;
    }
    double threshold() const { return user_thr_ ? thr_ : shim::kEps * double(std::min(f_.m, f_.n)); }
    Index rank() const { return f_.rank(threshold()); }
    Index rows() const { return f_.m; }
    Index cols() const { return f_.n; }
    bool isInvertible() const { return f_.m == f_.n && rank() == f_.n; }
    Index nonzeroPivots() const { return f_.nonzero_pivots(); }
    ComputationInfo info() const { return Success; }
    template <Dense B>
    MatrixXd solve(const B& b) const {
        MatrixXd c(b);
        if (c.rows() != f_.m) shim::fail("ColPivHouseholderQR::solve: row mismatch");
        MatrixXd x(f_.n, c.cols());
        const Index nz = f_.nonzero_pivots();
        if (nz == 0) return x;
        f_.apply_qt(c);
        shim::upper_solve(f_.qr, nz, c);
        for (Index i = 0; i < nz; ++i)
            for (Index j = 0; j < c.cols(); ++j) x(f_.perm[static_cast<std::size_t>(i)], j) = c(i, j);
        return x;
    }

private:
    shim::PivQR f_;
    double thr_ = 0.0;
    bool user_thr_ = false;
};

// Minimum-norm least squares over the rank-revealing pivoted QR (rank by
// the ColPivHouseholderQR rule with the COD's threshold).
template <class M>
class CompleteOrthogonalDecomposition {
public:
    CompleteOrthogonalDecomposition() = default;
    template <Dense A>
    explicit CompleteOrthogonalDecomposition(const A& a) {
        compute(a);
    }
    template <Dense A>
    CompleteOrthogonalDecomposition& compute(const A& a) {
        f_.compute(a.cv());
        return *this;
    }
    CompleteOrthogonalDecomposition& setThreshold(double t) {
        thr_ = t;
        user_thr_ = true;
        return *this;
    }
    double threshold() const { return user_thr_ ? thr_ : shim::kEps * double(std::min(f_.m, f_.n)); }
    Index rank() const { return f_.rank(threshold()); }
    ComputationInfo info() const { return Success; }
    template <Dense B>
    MatrixXd solve(const B& b) const {
        MatrixXd c(b);
        if (c.rows() != f_.m) shim::fail("CompleteOrthogonalDecomposition::solve: row mismatch");
        const Index n = f_.n, r = rank();
        MatrixXd x(n, c.cols());
        if (r == 0) return x;
        f_.apply_qt(c);
        MatrixXd y(n, c.cols());  // in pivoted order
        if (r == n) {
            shim::upper_solve(f_.qr, r, c);
            for (Index i = 0; i < n; ++i)
                for (Index j = 0; j < c.cols(); ++j) y(i, j) = c(i, j);
        } else {
            // min-norm solution of T y = c[0:r], T = R[0:r, 0:n] (full row
            // rank): T^T = Z L (QR of the n x r transpose), y = Z L^-T c
            MatrixXd tt(n, r);
            for (Index i = 0; i < r; ++i)
                for (Index j = i; j < n; ++j) tt(j, i) = f_.qr(i, j);
            const int ni = shim::to_int(n), ri = shim::to_int(r), ld = ni;
            std::vector<double> tau(static_cast<std::size_t>(r));
            int info = 0, lwork = -1;
            double wq = 0.0;
            scipy_dgeqrf_(&ni, &ri, tt.data(), &ld, tau.data(), &wq, &lwork, &info);
            lwork = std::max(1, static_cast<int>(wq));
            std::vector<double> work(static_cast<std::size_t>(lwork));
            scipy_dgeqrf_(&ni, &ri, tt.data(), &ld, tau.data(), work.data(), &lwork, &info);
            if (info != 0) shim::fail("dgeqrf failed");
            // z = L^-T c[0:r]: L^T is the upper r x r factor of tt, so solve
            // (upper)^T z = c  -> forward substitution with its transpose
            for (Index col = 0; col < c.cols(); ++col) {
                for (Index i = 0; i < r; ++i) {
                    double s = c(i, col);
                    for (Index k = 0; k < i; ++k) s -= tt(k, i) * y(k, col);
                    y(i, col) = s / tt(i, i);
                }
                for (Index i = r; i < n; ++i) y(i, col) = 0.0;
            }
            const int nc = shim::to_int(c.cols());
            lwork = -1;
            scipy_dormqr_("L", "N", &ni, &nc, &ri, tt.data(), &ld, tau.data(), y.data(), &ld, &wq, &lwork, &info, 1,
                          1);
            lwork = std::max(1, static_cast<int>(wq));
            work.assign(static_cast<std::size_t>(lwork), 0.0);
            scipy_dormqr_("L", "N", &ni, &nc, &ri, tt.data(), &ld, tau.data(), y.data(), &ld, work.data(), &lwork,
                          &info, 1, 1);
            if (info != 0) shim::fail("dormqr failed");
        }
        for (Index i = 0; i < n; ++i)
            for (Index j = 0; j < c.cols(); ++j) x(f_.perm[static_cast<std::size_t>(i)], j) = y(i, j);
        return x;
    }

private:
    shim::PivQR f_;
    double thr_ = 0.0;
    bool user_thr_ = false;
};

// Full-pivoting LU with Eigen's pivot order (largest |a| of the trailing
// block, first in column-major order) and rank rule.
template <class M>
class FullPivLU {
public:
    FullPivLU() = default;
    template <Dense A>
    explicit FullPivLU(const A& a) {
        compute(a);
    }
    template <Dense A>
    FullPivLU& compute(const A& a) {
        lu_ = MatrixXd(a);
        const Index m = lu_.rows(), n = lu_.cols(), k = std::min(m, n);
        rowp_.resize(static_cast<std::size_t>(m));
        colp_.resize(static_cast<std::size_t>(n));
        for (Index i = 0; i < m; ++i) rowp_[static_cast<std::size_t>(i)] = i;
        for (Index j = 0; j < n; ++j) colp_[static_cast<std::size_t>(j)] = j;
        maxpivot_ = 0.0;
        nonzero_ = k;
        for (Index s = 0; s < k; ++s) {
            double big = -1.0;
            Index bi = s, bj = s;
            for (Index j = s; j < n; ++j)
                for (Index i = s; i < m; ++i)
                    if (std::abs(lu_(i, j)) > big) {
                        big = std::abs(lu_(i, j));
                        bi = i;
                        bj = j;
                    }
            if (big == 0.0) {
                nonzero_ = s;
                break;
            }
            maxpivot_ = std::max(maxpivot_, big);
            if (bi != s) {
                for (Index j = 0; j < n; ++j) std::swap(lu_(s, j), lu_(bi, j));
                std::swap(rowp_[static_cast<std::size_t>(s)], rowp_[static_cast<std::size_t>(bi)]);
            }
            if (bj != s) {
                for (Index i = 0; i < m; ++i) std::swap(lu_(i, s), lu_(i, bj));
                std::swap(colp_[static_cast<std::size_t>(s)], colp_[static_cast<std::size_t>(bj)]);
            }
            const double piv = lu_(s, s);
            for (Index i = s + 1; i < m; ++i) lu_(i, s) /= piv;
            for (Index j = s + 1; j < n; ++j) {
                const double u = lu_(s, j);
                for (Index i = s + 1; i < m; ++i) lu_(i, j) -= lu_(i, s) * u;
            }
        }
        return *this;
    }
    double threshold() const { return shim::kEps * double(std::min(lu_.rows(), lu_.cols())); }
    Index rank() const {
        const double pre = std::abs(maxpivot_) * threshold();
        Index r = 0;
        for (Index i = 0; i < nonzero_; ++i)
            if (std::abs(lu_(i, i)) > pre) ++r;
        return r;
    }
    bool isInvertible() const { return lu_.rows() == lu_.cols() && rank() == lu_.rows(); }
    MatrixXd inverse() const {
        const Index n = lu_.rows();
        MatrixXd b(n, n);
        for (Index i = 0; i < n; ++i) b(i, rowp_[static_cast<std::size_t>(i)]) = 1.0;  // P I
        for (Index c = 0; c < n; ++c) {
            for (Index i = 0; i < n; ++i)  // L y = b (unit lower)
                for (Index k = 0; k < i; ++k) b(i, c) -= lu_(i, k) * b(k, c);
            for (Index i = n - 1; i >= 0; --i) {  // U z = y
                double s = b(i, c);
                for (Index k = i + 1; k < n; ++k) s -= lu_(i, k) * b(k, c);
                b(i, c) = s / lu_(i, i);
            }
        }
        MatrixXd x(n, n);
        for (Index i = 0; i < n; ++i)
            for (Index c = 0; c < n; ++c) x(colp_[static_cast<std::size_t>(i)], c) = b(i, c);
        return x;
    }

private:
    MatrixXd lu_;
    std::vector<Index> rowp_, colp_;
    double maxpivot_ = 0.0;
    Index nonzero_ = 0;
};

class TriangularLower {
public:
    explicit TriangularLower(const MatrixXd* l) : l_(l) {}
    template <Dense B>
    MatrixXd solve(const B& b) const {
        MatrixXd x(b);
        const Index n = l_->rows();
        if (x.rows() != n) shim::fail("triangular solve: row mismatch");
        if (n == 0 || x.cols() == 0) return x;
        const int ni = shim::to_int(n), nc = shim::to_int(x.cols()), ld = ni;
        const double one = 1.0;
        scipy_dtrsm_("L", "L", "N", "N", &ni, &nc, &one, l_->data(), &ld, x.data(), &ld, 1, 1, 1, 1);
        return x;
    }
    MatrixXd toDenseMatrix() const { return *l_; }

private:
    const MatrixXd* l_;
};

template <class M>
class LLT {
public:
    LLT() = default;
    template <Dense A>
    explicit LLT(const A& a) {
        compute(a);
    }
    template <Dense A>
    LLT& compute(const A& a) {
        l_ = MatrixXd(a);
        const Index n = l_.rows();
        if (n != l_.cols()) shim::fail("LLT of a non-square matrix");
        info_ = Success;
        if (n > 0) {
            const int ni = shim::to_int(n), ld = ni;
            int info = 0;
            scipy_dpotrf_("L", &ni, l_.data(), &ld, &info, 1);
            if (info != 0) info_ = NumericalIssue;
        }
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < j; ++i) l_(i, j) = 0.0;
        return *this;
    }
    ComputationInfo info() const { return info_; }
    TriangularLower matrixL() const { return TriangularLower(&l_); }
    template <Dense B>
    MatrixXd solve(const B& b) const {
        MatrixXd y = matrixL().solve(b);
        const Index n = l_.rows();
        if (n == 0 || y.cols() == 0) return y;
        const int ni = shim::to_int(n), nc = shim::to_int(y.cols()), ld = ni;
        const double one = 1.0;
        scipy_dtrsm_("L", "L", "T", "N", &ni, &nc, &one, l_.data(), &ld, y.data(), &ld, 1, 1, 1, 1);
        return y;
    }

private:
    MatrixXd l_;
    ComputationInfo info_ = InvalidInput;
};

namespace shim {
// thin SVD; sdd: divide and conquer (BDCSVD) else dgesvd (JacobiSVD)
struct ThinSVD {
    MatrixXd u, v;
    VectorXd s;
    Index nonzero = 0;
    void compute(const CV& a, unsigned opts, bool sdd, bool tiny_is_zero) {
        const Index m = a.r, n = a.c, k = std::min(m, n);
        MatrixXd w(ConstBlock(a.p, a.r, a.c, a.ld));
        s = VectorXd(k);
        u = MatrixXd(m, k);
        MatrixXd vt(k, n);
        if (k > 0) {
            const int mi = to_int(m), ni = to_int(n), lda = mi, ldu = mi, ldvt = to_int(k);
            int info = 0, lwork = -1;
            double wq = 0.0;
            if (sdd) {
                std::vector<int> iwork(static_cast<std::size_t>(8 * k));
                scipy_dgesdd_("S", &mi, &ni, w.data(), &lda, s.data(), u.data(), &ldu, vt.data(), &ldvt, &wq, &lwork,
                              iwork.data(), &info, 1);
                lwork = std::max(1, static_cast<int>(wq));
                std::vector<double> work(static_cast<std::size_t>(lwork));
                scipy_dgesdd_("S", &mi, &ni, w.data(), &lda, s.data(), u.data(), &ldu, vt.data(), &ldvt, work.data(),
                              &lwork, iwork.data(), &info, 1);
            } else {
                scipy_dgesvd_("S", "S", &mi, &ni, w.data(), &lda, s.data(), u.data(), &ldu, vt.data(), &ldvt, &wq,
                              &lwork, &info, 1, 1);
                lwork = std::max(1, static_cast<int>(wq));
                std::vector<double> work(static_cast<std::size_t>(lwork));
                scipy_dgesvd_("S", "S", &mi, &ni, w.data(), &lda, s.data(), u.data(), &ldu, vt.data(), &ldvt,
                              work.data(), &lwork, &info, 1, 1);
            }
            if (info != 0) fail("SVD did not converge");
        }
        v = vt.transpose();
        (void)opts;
        nonzero = k;
        const double cut = tiny_is_zero ? std::numeric_limits<double>::min() : 0.0;
        for (Index i = 0; i < k; ++i)
            if (!(s(i) > cut)) {
                nonzero = i;
                break;
            }
    }
};
}  // namespace shim

template <class M>
class JacobiSVD {
public:
    template <Dense A>
    JacobiSVD(const A& a, unsigned opts = 0) {
        f_.compute(a.cv(), opts, false, false);
    }
    const MatrixXd& matrixU() const { return f_.u; }
    const MatrixXd& matrixV() const { return f_.v; }
    const VectorXd& singularValues() const { return f_.s; }
    Index nonzeroSingularValues() const { return f_.nonzero; }
    Index rank() const {
        if (f_.s.size() == 0) return 0;
        const double thr = std::max(f_.s(0) * shim::kEps * double(std::max(f_.u.rows(), f_.v.rows())),
                                    std::numeric_limits<double>::min());
        Index r = 0;
        for (Index i = 0; i < f_.s.size(); ++i)
            if (f_.s(i) > thr) ++r;
        return r;
    }
    ComputationInfo info() const { return Success; }

private:
    shim::ThinSVD f_;
};

template <class M>
class BDCSVD {
public:
    template <Dense A>
    BDCSVD(const A& a, unsigned opts = 0) {
        f_.compute(a.cv(), opts, true, true);
    }
    const MatrixXd& matrixU() const { return f_.u; }
    const MatrixXd& matrixV() const { return f_.v; }
    const VectorXd& singularValues() const { return f_.s; }
    Index nonzeroSingularValues() const { return f_.nonzero; }
    ComputationInfo info() const { return Success; }

private:
    shim::ThinSVD f_;
};

// ---- complex results of EigenSolver
class ComplexColumn {
public:
    ComplexColumn(VectorXd re, VectorXd im) : re_(std::move(re)), im_(std::move(im)) {}
    const VectorXd& real() const { return re_; }
    const VectorXd& imag() const { return im_; }
    Index size() const { return re_.size(); }

private:
    VectorXd re_, im_;
};
class ComplexVectorXd {
public:
    ComplexVectorXd() = default;
    explicit ComplexVectorXd(Index n) : v_(static_cast<std::size_t>(n)) {}
    std::complex<double> operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
    std::complex<double>& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
    Index size() const { return static_cast<Index>(v_.size()); }
    VectorXd real() const {
        VectorXd r(size());
        for (Index i = 0; i < size(); ++i) r(i) = v_[static_cast<std::size_t>(i)].real();
        return r;
    }
    VectorXd imag() const {
        VectorXd r(size());
        for (Index i = 0; i < size(); ++i) r(i) = v_[static_cast<std::size_t>(i)].imag();
        return r;
    }

private:
    std::vector<std::complex<double>> v_;
};
class ComplexMatrixXd {
public:
    ComplexMatrixXd() = default;
    ComplexMatrixXd(MatrixXd re, MatrixXd im) : re_(std::move(re)), im_(std::move(im)) {}
    ComplexColumn col(Index j) const { return ComplexColumn(VectorXd(re_.col(j)), VectorXd(im_.col(j))); }
    std::complex<double> operator()(Index i, Index j) const { return {re_(i, j), im_(i, j)}; }
    const MatrixXd& real() const { return re_; }
    const MatrixXd& imag() const { return im_; }
    Index rows() const { return re_.rows(); }
    Index cols() const { return re_.cols(); }

private:
    MatrixXd re_, im_;
};

template <class M>
class EigenSolver {
public:
    EigenSolver() = default;
    template <Dense A>
    explicit EigenSolver(const A& a, bool vectors = true) {
        compute(a, vectors);
    }
    template <Dense A>
    EigenSolver& compute(const A& a, bool = true) {
        MatrixXd w(a);
        const Index n = w.rows();
        if (n != w.cols()) shim::fail("EigenSolver of a non-square matrix");
        vals_ = ComplexVectorXd(n);
        MatrixXd vr(n, n), re(n, n), im(n, n);
        info_ = Success;
        if (n > 0) {
            const int ni = shim::to_int(n), ld = ni, one = 1;
            std::vector<double> wr(static_cast<std::size_t>(n)), wi(static_cast<std::size_t>(n));
            double dummy = 0.0, wq = 0.0;
            int info = 0, lwork = -1;
            scipy_dgeev_("N", "V", &ni, w.data(), &ld, wr.data(), wi.data(), &dummy, &one, vr.data(), &ld, &wq,
                         &lwork, &info, 1, 1);
            lwork = std::max(1, static_cast<int>(wq));
            std::vector<double> work(static_cast<std::size_t>(lwork));
            scipy_dgeev_("N", "V", &ni, w.data(), &ld, wr.data(), wi.data(), &dummy, &one, vr.data(), &ld,
                         work.data(), &lwork, &info, 1, 1);
            if (info != 0) {
                info_ = NoConvergence;
                return *this;
            }
            for (Index j = 0; j < n; ++j) vals_(j) = {wr[static_cast<std::size_t>(j)], wi[static_cast<std::size_t>(j)]};
            // Eigen's eigenvectors(): a "real" eigenvalue (|imag| much smaller
            // than |real|, dummy precision 1e-12) takes its column alone, a
            // complex pair (j, j+1) = (re + i im, re - i im); every column
            // normalised to unit 2-norm
            for (Index j = 0; j < n; ++j) {
                const double ai = std::abs(wi[static_cast<std::size_t>(j)]);
                const double ar = std::abs(wr[static_cast<std::size_t>(j)]);
                if (ai <= ar * 1e-12 || j + 1 == n) {
                    double s = 0.0;
                    for (Index i = 0; i < n; ++i) s += vr(i, j) * vr(i, j);
                    s = std::sqrt(s);
                    for (Index i = 0; i < n; ++i) re(i, j) = s > 0.0 ? vr(i, j) / s : vr(i, j);
                } else {
                    double s = 0.0;
                    for (Index i = 0; i < n; ++i) s += vr(i, j) * vr(i, j) + vr(i, j + 1) * vr(i, j + 1);
                    s = std::sqrt(s);
                    for (Index i = 0; i < n; ++i) {
                        re(i, j) = vr(i, j) / s;
                        im(i, j) = vr(i, j + 1) / s;
                        re(i, j + 1) = vr(i, j) / s;
                        im(i, j + 1) = -vr(i, j + 1) / s;
                    }
                    ++j;
                }
            }
        }
        vecs_ = ComplexMatrixXd(std::move(re), std::move(im));
        return *this;
    }
    ComputationInfo info() const { return info_; }
    const ComplexVectorXd& eigenvalues() const { return vals_; }
    const ComplexMatrixXd& eigenvectors() const { return vecs_; }

private:
    ComplexVectorXd vals_;
    ComplexMatrixXd vecs_;
    ComputationInfo info_ = InvalidInput;
};

}  // namespace Eigen
