// TEST INFRASTRUCTURE — a from-scratch, eager subset of the Eigen 3 dense API, written for
// one purpose: compiling the reference's own sources (/root/reference/proj/src, unmodified)
// into oracle/_ref so the oracle restatement can be checked against — and the bench's
// reference arm can run — the reference code itself ("recommended oracle").
// Not used by the product.  It implements only what those sources call:
//   MatrixXd / VectorXd (column-major, double), Index, blocks (col, row, middleCols, block,
//   corners, head / tail) as views, transpose() as a view that products hand to BLAS,
//   +, −, scalar ·, /, products (OpenBLAS dgemm, ILP64, loaded at run time from numpy's
//   bundled library), asDiagonal, diagonal, norms, reductions, cwise ops, LLT (LAPACKE
//   dpotrf / dpotrs), PartialPivLU (dgetrf / dgetri), FullPivLU (complete pivoting, here).
// Expression templates are not reproduced: every operation evaluates eagerly.  Products
// go through multi-threaded dgemm and the element-wise passes and reductions run on all
// host threads (OpenMP) — the reference's Eigen is single-threaded — so timings taken with
// this shim favour the reference.
#pragma once
#include <dlfcn.h>
#include <glob.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
constexpr int Dynamic = -1;

namespace shim {
struct Blas {
    using dgemm_t = void (*)(int, int, int, int64_t, int64_t, int64_t, double, const double*, int64_t, const double*,
                             int64_t, double, double*, int64_t);
    using potrf_t = int64_t (*)(int, char, int64_t, double*, int64_t);
    using potrs_t = int64_t (*)(int, char, int64_t, int64_t, const double*, int64_t, double*, int64_t);
    using getrf_t = int64_t (*)(int, int64_t, int64_t, double*, int64_t, int64_t*);
    using getri_t = int64_t (*)(int, int64_t, double*, int64_t, const int64_t*);
    dgemm_t dgemm = nullptr;
    potrf_t potrf = nullptr;
    potrs_t potrs = nullptr;
    getrf_t getrf = nullptr;
    getri_t getri = nullptr;
    static const Blas& get() {
        static const Blas b = [] {
            Blas r;
            std::vector<std::string> cand;
            if (const char* p = std::getenv("SI_ORACLE_BLAS")) cand.emplace_back(p);
            glob_t g;
            const char* pats[] = {"/opt/prime-rl/.venv/lib/python3.12/site-packages/numpy.libs/libscipy_openblas64_*.so"};
            for (const char* pat : pats) {
                if (glob(pat, 0, nullptr, &g) == 0)
                    for (size_t i = 0; i < g.gl_pathc; ++i) cand.emplace_back(g.gl_pathv[i]);
                globfree(&g);
            }
            for (const auto& path : cand) {
                void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
                if (!h) continue;
                r.dgemm = reinterpret_cast<dgemm_t>(dlsym(h, "scipy_cblas_dgemm64_"));
                r.potrf = reinterpret_cast<potrf_t>(dlsym(h, "scipy_LAPACKE_dpotrf64_"));
                r.potrs = reinterpret_cast<potrs_t>(dlsym(h, "scipy_LAPACKE_dpotrs64_"));
                r.getrf = reinterpret_cast<getrf_t>(dlsym(h, "scipy_LAPACKE_dgetrf64_"));
                r.getri = reinterpret_cast<getri_t>(dlsym(h, "scipy_LAPACKE_dgetri64_"));
                if (r.dgemm && r.potrf && r.potrs && r.getrf && r.getri) return r;
            }
            throw std::runtime_error("eigen shim: OpenBLAS (numpy's bundled ILP64 build) not found");
        }();
        return b;
    }
};
}  // namespace shim

#if defined(_OPENMP)
#define SI_SHIM_PAR _Pragma("omp parallel for schedule(static) if (count > 65536)")
#define SI_SHIM_PAR_SUM _Pragma("omp parallel for schedule(static) reduction(+ : s) if (count > 65536)")
#else
#define SI_SHIM_PAR
#define SI_SHIM_PAR_SUM
#endif

class MatrixXd;
class VectorXd;
class Block;
class ConstBlock;
class Transpose;
class DiagonalWrapper;

// ------------------------------------------------------------------ MatrixXd --
class MatrixXd {
public:
    using Scalar = double;
    MatrixXd() = default;
    MatrixXd(Index r, Index c) : r_(r), c_(c), d_(size_t(r) * size_t(c), 0.0) {}
    MatrixXd(const MatrixXd&) = default;
    MatrixXd(MatrixXd&&) noexcept = default;
    MatrixXd& operator=(const MatrixXd&) = default;
    MatrixXd& operator=(MatrixXd&&) noexcept = default;
    MatrixXd(const Block& b);
    MatrixXd(const ConstBlock& b);
    MatrixXd(const Transpose& t);
    MatrixXd(const DiagonalWrapper& d);
    MatrixXd& operator=(const Block& b);
    MatrixXd& operator=(const ConstBlock& b);
    MatrixXd& operator=(const Transpose& t);

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }
    double& operator()(Index i, Index j) { return d_[size_t(i + j * r_)]; }
    double operator()(Index i, Index j) const { return d_[size_t(i + j * r_)]; }
    double& operator()(Index i) { return d_[size_t(i)]; }
    double operator()(Index i) const { return d_[size_t(i)]; }
    double& operator[](Index i) { return d_[size_t(i)]; }
    double operator[](Index i) const { return d_[size_t(i)]; }
    void resize(Index r, Index c) {
        r_ = r;
        c_ = c;
        d_.assign(size_t(r) * size_t(c), 0.0);
    }

    static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
    static MatrixXd Identity(Index r, Index c) {
        MatrixXd m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    static MatrixXd Constant(Index r, Index c, double v) {
        MatrixXd m(r, c);
        std::fill(m.d_.begin(), m.d_.end(), v);
        return m;
    }
    static MatrixXd Ones(Index r, Index c) { return Constant(r, c, 1.0); }
    MatrixXd& setZero() {
        std::fill(d_.begin(), d_.end(), 0.0);
        return *this;
    }
    MatrixXd& setOnes() {
        std::fill(d_.begin(), d_.end(), 1.0);
        return *this;
    }
    MatrixXd& setIdentity() {
        *this = Identity(r_, c_);
        return *this;
    }

    Block col(Index j);
    ConstBlock col(Index j) const;
    Block row(Index i);
    ConstBlock row(Index i) const;
    Block block(Index i, Index j, Index r, Index c);
    ConstBlock block(Index i, Index j, Index r, Index c) const;
    Block middleCols(Index j, Index c);
    ConstBlock middleCols(Index j, Index c) const;
    Block middleRows(Index i, Index r);
    ConstBlock middleRows(Index i, Index r) const;
    Block leftCols(Index c);
    ConstBlock leftCols(Index c) const;
    Block rightCols(Index c);
    ConstBlock rightCols(Index c) const;
    Block topRows(Index r);
    ConstBlock topRows(Index r) const;
    Block bottomRows(Index r);
    ConstBlock bottomRows(Index r) const;
    Block topLeftCorner(Index r, Index c);
    ConstBlock topLeftCorner(Index r, Index c) const;
    Block topRightCorner(Index r, Index c);
    ConstBlock topRightCorner(Index r, Index c) const;
    Block bottomLeftCorner(Index r, Index c);
    ConstBlock bottomLeftCorner(Index r, Index c) const;
    Block bottomRightCorner(Index r, Index c);
    ConstBlock bottomRightCorner(Index r, Index c) const;
    Block head(Index n);
    ConstBlock head(Index n) const;
    Block tail(Index n);
    ConstBlock tail(Index n) const;
    Block segment(Index i, Index n);
    ConstBlock segment(Index i, Index n) const;

    Transpose transpose() const&;
    Transpose transpose() &&;
    DiagonalWrapper asDiagonal() const;
    VectorXd diagonal() const;
    MatrixXd eval() const { return *this; }
    MatrixXd& noalias() { return *this; }

    double squaredNorm() const {
        double s = 0.0;
        const int64_t count = int64_t(d_.size());
        const double* d = d_.data();
        SI_SHIM_PAR_SUM
        for (int64_t i = 0; i < count; ++i) s += d[i] * d[i];
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    double sum() const {
        double s = 0.0;
        const int64_t count = int64_t(d_.size());
        const double* d = d_.data();
        SI_SHIM_PAR_SUM
        for (int64_t i = 0; i < count; ++i) s += d[i];
        return s;
    }
    double trace() const {
        double s = 0.0;
        for (Index i = 0; i < std::min(r_, c_); ++i) s += (*this)(i, i);
        return s;
    }
    double maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
    double minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
    double dot(const MatrixXd& o) const {
        double s = 0.0;
        for (size_t i = 0; i < d_.size(); ++i) s += d_[i] * o.d_[i];
        return s;
    }
    bool allFinite() const {
        for (double v : d_)
            if (!std::isfinite(v)) return false;
        return true;
    }
    bool isIdentity(double prec = 1e-12) const {
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i)
                if (std::abs((*this)(i, j) - (i == j ? 1.0 : 0.0)) > prec) return false;
        return true;
    }
    MatrixXd cwiseAbs() const { return map([](double v) { return std::abs(v); }); }
    MatrixXd cwiseSqrt() const { return map([](double v) { return std::sqrt(v); }); }
    MatrixXd cwiseInverse() const { return map([](double v) { return 1.0 / v; }); }
    MatrixXd cwiseProduct(const MatrixXd& o) const {
        MatrixXd m(r_, c_);
        for (size_t i = 0; i < d_.size(); ++i) m.d_[i] = d_[i] * o.d_[i];
        return m;
    }
    void normalize() {
        const double n = norm();
        if (n > 0.0)
            for (double& v : d_) v /= n;
    }
    MatrixXd normalized() const {
        MatrixXd m = *this;
        m.normalize();
        return m;
    }
    template <class F>
    MatrixXd map(F f) const {
        MatrixXd m(r_, c_);
        const int64_t count = int64_t(d_.size());
        SI_SHIM_PAR
        for (int64_t i = 0; i < count; ++i) m.d_[size_t(i)] = f(d_[size_t(i)]);
        return m;
    }
    MatrixXd& operator+=(const MatrixXd& o) {
        check_same(o);
        const int64_t count = int64_t(d_.size());
        SI_SHIM_PAR
        for (int64_t i = 0; i < count; ++i) d_[size_t(i)] += o.d_[size_t(i)];
        return *this;
    }
    MatrixXd& operator-=(const MatrixXd& o) {
        check_same(o);
        const int64_t count = int64_t(d_.size());
        SI_SHIM_PAR
        for (int64_t i = 0; i < count; ++i) d_[size_t(i)] -= o.d_[size_t(i)];
        return *this;
    }
    MatrixXd& operator*=(double s) {
        for (double& v : d_) v *= s;
        return *this;
    }
    MatrixXd& operator/=(double s) {
        for (double& v : d_) v /= s;
        return *this;
    }
    void check_same(const MatrixXd& o) const {
        if (o.r_ != r_ || o.c_ != c_) throw std::invalid_argument("eigen shim: dimension mismatch");
    }

protected:
    Index r_ = 0, c_ = 0;
    std::vector<double> d_;
};

class VectorXd : public MatrixXd {
public:
    VectorXd() = default;
    explicit VectorXd(Index n) : MatrixXd(n, 1) {}
    VectorXd(const MatrixXd& m) : MatrixXd(m) { check(); }
    VectorXd(MatrixXd&& m) : MatrixXd(std::move(m)) { check(); }
    VectorXd(const Block& b);
    VectorXd(const ConstBlock& b);
    VectorXd& operator=(const MatrixXd& m) {
        MatrixXd::operator=(m);
        check();
        return *this;
    }
    VectorXd& operator=(const ConstBlock& b);
    VectorXd& operator=(const Block& b);
    static VectorXd Zero(Index n) { return VectorXd(n); }
    static VectorXd Constant(Index n, double v) { return VectorXd(MatrixXd::Constant(n, 1, v)); }
    static VectorXd Ones(Index n) { return Constant(n, 1.0); }
    void resize(Index n) { MatrixXd::resize(n, 1); }
    VectorXd& setOnes() {
        MatrixXd::setOnes();
        return *this;
    }
    VectorXd cwiseAbs() const { return VectorXd(MatrixXd::cwiseAbs()); }
    VectorXd cwiseSqrt() const { return VectorXd(MatrixXd::cwiseSqrt()); }

private:
    void check() {
        if (c_ != 1 && !(r_ == 0 && c_ == 0)) {
            if (r_ == 1) {  // a row converted to a vector: Eigen would transpose implicitly
                r_ = c_;
                c_ = 1;
            } else {
                throw std::invalid_argument("eigen shim: VectorXd from a matrix with several columns");
            }
        }
    }
};

// ------------------------------------------------------------------ views --
class ConstBlock {
public:
    ConstBlock(const double* p, Index r, Index c, Index ld) : p_(p), r_(r), c_(c), ld_(ld) {}
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double operator()(Index i, Index j) const { return p_[i + j * ld_]; }
    double operator()(Index i) const { return c_ == 1 ? p_[i] : p_[i * ld_]; }
    double operator[](Index i) const { return (*this)(i); }
    MatrixXd eval() const { return MatrixXd(*this); }
    Transpose transpose() const;
    double dot(const ConstBlock& o) const {
        double s = 0.0;
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) s += (*this)(i, j) * o(i, j);
        return s;
    }
    double squaredNorm() const { return dot(*this); }
    double norm() const { return std::sqrt(squaredNorm()); }
    double sum() const { return eval().sum(); }
    double maxCoeff() const { return eval().maxCoeff(); }
    double minCoeff() const { return eval().minCoeff(); }
    MatrixXd cwiseProduct(const MatrixXd& o) const { return eval().cwiseProduct(o); }
    MatrixXd cwiseAbs() const { return eval().cwiseAbs(); }
    bool allFinite() const { return eval().allFinite(); }
    const double* p_;
    Index r_, c_, ld_;
};

class Block : public ConstBlock {
public:
    Block(double* p, Index r, Index c, Index ld) : ConstBlock(p, r, c, ld) {}
    double& operator()(Index i, Index j) { return const_cast<double*>(p_)[i + j * ld_]; }
    double& operator()(Index i) { return const_cast<double*>(p_)[c_ == 1 ? i : i * ld_]; }
    double& operator[](Index i) { return (*this)(i); }
    using ConstBlock::operator();
    Block& operator=(const ConstBlock& o) {
        if (o.rows() != r_ || o.cols() != c_) throw std::invalid_argument("eigen shim: block assignment mismatch");
        MatrixXd tmp(o);  // source may alias the destination
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) = tmp(i, j);
        return *this;
    }
    Block& operator=(const Block& o) { return *this = static_cast<const ConstBlock&>(o); }
    Block& operator=(const MatrixXd& m) {
        return *this = ConstBlock(m.data(), m.rows(), m.cols(), std::max<Index>(m.rows(), 1));
    }
    Block& operator+=(const MatrixXd& m) {
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) += m(i, j);
        return *this;
    }
    Block& operator-=(const MatrixXd& m) {
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) -= m(i, j);
        return *this;
    }
    Block& operator*=(double s) {
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) *= s;
        return *this;
    }
    void setZero() {
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) (*this)(i, j) = 0.0;
    }
    void normalize() {
        const double n = norm();
        if (n > 0.0) *this *= 1.0 / n;
    }
};

inline MatrixXd::MatrixXd(const ConstBlock& b) : MatrixXd(b.rows(), b.cols()) {
    for (Index j = 0; j < c_; ++j)
        for (Index i = 0; i < r_; ++i) (*this)(i, j) = b(i, j);
}
inline MatrixXd::MatrixXd(const Block& b) : MatrixXd(static_cast<const ConstBlock&>(b)) {}
inline MatrixXd& MatrixXd::operator=(const ConstBlock& b) { return *this = MatrixXd(b); }
inline MatrixXd& MatrixXd::operator=(const Block& b) { return *this = MatrixXd(b); }
inline VectorXd::VectorXd(const ConstBlock& b) : VectorXd(MatrixXd(b)) {}
inline VectorXd::VectorXd(const Block& b) : VectorXd(MatrixXd(b)) {}
inline VectorXd& VectorXd::operator=(const ConstBlock& b) { return *this = MatrixXd(b); }
inline VectorXd& VectorXd::operator=(const Block& b) { return *this = MatrixXd(b); }

#define SI_SHIM_BLOCKS(CV, BT)                                                                                  \
    inline BT MatrixXd::col(Index j) CV { return BT(const_cast<double*>(data()) + j * r_, r_, 1, r_); }        \
    inline BT MatrixXd::row(Index i) CV { return BT(const_cast<double*>(data()) + i, 1, c_, r_); }             \
    inline BT MatrixXd::block(Index i, Index j, Index r, Index c) CV {                                          \
        return BT(const_cast<double*>(data()) + i + j * r_, r, c, r_);                                          \
    }                                                                                                           \
    inline BT MatrixXd::middleCols(Index j, Index c) CV { return block(0, j, r_, c); }                          \
    inline BT MatrixXd::middleRows(Index i, Index r) CV { return block(i, 0, r, c_); }                          \
    inline BT MatrixXd::leftCols(Index c) CV { return block(0, 0, r_, c); }                                     \
    inline BT MatrixXd::rightCols(Index c) CV { return block(0, c_ - c, r_, c); }                               \
    inline BT MatrixXd::topRows(Index r) CV { return block(0, 0, r, c_); }                                      \
    inline BT MatrixXd::bottomRows(Index r) CV { return block(r_ - r, 0, r, c_); }                              \
    inline BT MatrixXd::topLeftCorner(Index r, Index c) CV { return block(0, 0, r, c); }                        \
    inline BT MatrixXd::topRightCorner(Index r, Index c) CV { return block(0, c_ - c, r, c); }                  \
    inline BT MatrixXd::bottomLeftCorner(Index r, Index c) CV { return block(r_ - r, 0, r, c); }                \
    inline BT MatrixXd::bottomRightCorner(Index r, Index c) CV { return block(r_ - r, c_ - c, r, c); }          \
    inline BT MatrixXd::head(Index n) CV { return c_ == 1 ? block(0, 0, n, 1) : block(0, 0, 1, n); }            \
    inline BT MatrixXd::tail(Index n) CV { return c_ == 1 ? block(r_ - n, 0, n, 1) : block(0, c_ - n, 1, n); }  \
    inline BT MatrixXd::segment(Index i, Index n) CV { return c_ == 1 ? block(i, 0, n, 1) : block(0, i, 1, n); }
SI_SHIM_BLOCKS(, Block)
SI_SHIM_BLOCKS(const, ConstBlock)
#undef SI_SHIM_BLOCKS

// transpose(): a view whose products go to dgemm with the transpose flag; an rvalue's
// storage is kept alive inside the view
class Transpose {
public:
    Transpose(const MatrixXd* m) : m_(m) {}
    explicit Transpose(MatrixXd&& own) : own_(std::make_shared<MatrixXd>(std::move(own))), m_(own_.get()) {}
    const MatrixXd& base() const { return *m_; }
    Index rows() const { return m_->cols(); }
    Index cols() const { return m_->rows(); }
    double operator()(Index i, Index j) const { return (*m_)(j, i); }
    MatrixXd eval() const { return MatrixXd(*this); }
    double norm() const { return m_->norm(); }
    double squaredNorm() const { return m_->squaredNorm(); }
    double trace() const { return m_->trace(); }

private:
    std::shared_ptr<MatrixXd> own_;
    const MatrixXd* m_;
};
inline Transpose MatrixXd::transpose() const& { return Transpose(this); }
inline Transpose MatrixXd::transpose() && { return Transpose(std::move(*this)); }
inline Transpose ConstBlock::transpose() const { return Transpose(MatrixXd(*this)); }
inline MatrixXd::MatrixXd(const Transpose& t) : MatrixXd(t.rows(), t.cols()) {
    const MatrixXd& b = t.base();
    const int64_t count = int64_t(c_) * int64_t(r_);
    const Index cols = c_, rows = r_;
    SI_SHIM_PAR
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) (*this)(i, j) = b(j, i);
    (void)count;
}
inline MatrixXd& MatrixXd::operator=(const Transpose& t) { return *this = MatrixXd(t); }

class DiagonalWrapper {
public:
    explicit DiagonalWrapper(const MatrixXd& v) : v_(v) {}
    const MatrixXd& v() const { return v_; }

private:
    MatrixXd v_;
};
inline DiagonalWrapper MatrixXd::asDiagonal() const { return DiagonalWrapper(*this); }
inline MatrixXd::MatrixXd(const DiagonalWrapper& d) : MatrixXd(d.v().size(), d.v().size()) {
    for (Index i = 0; i < r_; ++i) (*this)(i, i) = d.v()(i);
}
inline VectorXd MatrixXd::diagonal() const {
    VectorXd v(std::min(r_, c_));
    for (Index i = 0; i < v.size(); ++i) v(i) = (*this)(i, i);
    return v;
}

// ------------------------------------------------------------- arithmetic --
namespace shim {
inline MatrixXd gemm(const MatrixXd& a, bool ta, const MatrixXd& b, bool tb) {
    const Index m = ta ? a.cols() : a.rows(), k = ta ? a.rows() : a.cols();
    const Index kb = tb ? b.cols() : b.rows(), n = tb ? b.rows() : b.cols();
    if (k != kb) throw std::invalid_argument("eigen shim: product dimension mismatch");
    MatrixXd out(m, n);
    if (m == 0 || n == 0 || k == 0) return out;
    Blas::get().dgemm(102, ta ? 112 : 111, tb ? 112 : 111, m, n, k, 1.0, a.data(), std::max<Index>(1, a.rows()),
                      b.data(), std::max<Index>(1, b.rows()), 0.0, out.data(), std::max<Index>(1, m));
    return out;
}
template <class F>
inline MatrixXd zip(const MatrixXd& a, const MatrixXd& b, F f) {
    a.check_same(b);
    MatrixXd m(a.rows(), a.cols());
    const int64_t count = int64_t(a.size());
    SI_SHIM_PAR
    for (Index i = 0; i < count; ++i) m(i) = f(a(i), b(i));
    return m;
}
template <class F>
inline MatrixXd zip_t(const MatrixXd& a, const Transpose& b, F f) {  // a ∘ bᵀ without materialising bᵀ
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::invalid_argument("eigen shim: dimension mismatch");
    MatrixXd m(a.rows(), a.cols());
    const MatrixXd& bb = b.base();
    const int64_t count = int64_t(a.size());
    const Index cols = a.cols(), rows = a.rows();
    SI_SHIM_PAR
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) m(i, j) = f(a(i, j), bb(j, i));
    (void)count;
    return m;
}
}  // namespace shim

inline MatrixXd operator*(const MatrixXd& a, const MatrixXd& b) { return shim::gemm(a, false, b, false); }
inline MatrixXd operator*(const Transpose& a, const MatrixXd& b) { return shim::gemm(a.base(), true, b, false); }
inline MatrixXd operator*(const MatrixXd& a, const Transpose& b) { return shim::gemm(a, false, b.base(), true); }
inline MatrixXd operator*(const Transpose& a, const Transpose& b) { return shim::gemm(a.base(), true, b.base(), true); }
inline MatrixXd operator*(const ConstBlock& a, const MatrixXd& b) { return MatrixXd(a) * b; }
inline MatrixXd operator*(const MatrixXd& a, const ConstBlock& b) { return a * MatrixXd(b); }
inline MatrixXd operator*(const ConstBlock& a, const ConstBlock& b) { return MatrixXd(a) * MatrixXd(b); }
inline MatrixXd operator*(const Transpose& a, const ConstBlock& b) { return a * MatrixXd(b); }
inline MatrixXd operator*(const ConstBlock& a, const Transpose& b) { return MatrixXd(a) * b; }
inline MatrixXd operator*(const MatrixXd& a, const DiagonalWrapper& d) {  // column scaling
    MatrixXd m = a;
    for (Index j = 0; j < m.cols(); ++j)
        for (Index i = 0; i < m.rows(); ++i) m(i, j) *= d.v()(j);
    return m;
}
inline MatrixXd operator*(const DiagonalWrapper& d, const MatrixXd& a) {  // row scaling
    MatrixXd m = a;
    for (Index j = 0; j < m.cols(); ++j)
        for (Index i = 0; i < m.rows(); ++i) m(i, j) *= d.v()(i);
    return m;
}
inline MatrixXd operator*(double s, const MatrixXd& a) { return a.map([s](double v) { return s * v; }); }
inline MatrixXd operator*(const MatrixXd& a, double s) { return s * a; }
inline MatrixXd operator*(double s, const ConstBlock& a) { return s * MatrixXd(a); }
inline MatrixXd operator*(double s, const Transpose& a) { return s * MatrixXd(a); }
inline MatrixXd operator/(const MatrixXd& a, double s) { return a.map([s](double v) { return v / s; }); }
inline MatrixXd operator/(const ConstBlock& a, double s) { return MatrixXd(a) / s; }
inline MatrixXd operator-(const MatrixXd& a) { return a.map([](double v) { return -v; }); }

inline MatrixXd operator+(const MatrixXd& a, const MatrixXd& b) { return shim::zip(a, b, [](double x, double y) { return x + y; }); }
inline MatrixXd operator-(const MatrixXd& a, const MatrixXd& b) { return shim::zip(a, b, [](double x, double y) { return x - y; }); }
inline MatrixXd operator+(const MatrixXd& a, const Transpose& b) { return shim::zip_t(a, b, [](double x, double y) { return x + y; }); }
inline MatrixXd operator-(const MatrixXd& a, const Transpose& b) { return shim::zip_t(a, b, [](double x, double y) { return x - y; }); }
inline MatrixXd operator+(const Transpose& a, const MatrixXd& b) { return b + a; }
inline MatrixXd operator-(const Transpose& a, const MatrixXd& b) { return -(b - a); }
inline MatrixXd operator+(const Transpose& a, const Transpose& b) { return MatrixXd(a) + b; }
inline MatrixXd operator-(const Transpose& a, const Transpose& b) { return MatrixXd(a) - b; }
inline MatrixXd operator+(const MatrixXd& a, const ConstBlock& b) { return a + MatrixXd(b); }
inline MatrixXd operator-(const MatrixXd& a, const ConstBlock& b) { return a - MatrixXd(b); }
inline MatrixXd operator+(const ConstBlock& a, const MatrixXd& b) { return MatrixXd(a) + b; }
inline MatrixXd operator-(const ConstBlock& a, const MatrixXd& b) { return MatrixXd(a) - b; }
inline MatrixXd operator+(const ConstBlock& a, const ConstBlock& b) { return MatrixXd(a) + MatrixXd(b); }
inline MatrixXd operator-(const ConstBlock& a, const ConstBlock& b) { return MatrixXd(a) - MatrixXd(b); }
inline MatrixXd operator+(const MatrixXd& a, const DiagonalWrapper& d) { return a + MatrixXd(d); }
inline MatrixXd operator-(const MatrixXd& a, const DiagonalWrapper& d) { return a - MatrixXd(d); }
// rvalue overloads reuse the left operand's storage
inline MatrixXd operator+(MatrixXd&& a, const MatrixXd& b) {
    a += b;
    return std::move(a);
}
inline MatrixXd operator-(MatrixXd&& a, const MatrixXd& b) {
    a -= b;
    return std::move(a);
}
inline MatrixXd operator+(MatrixXd&& a, const Transpose& b) { return static_cast<const MatrixXd&>(a) + b; }
inline MatrixXd operator-(MatrixXd&& a, const Transpose& b) { return static_cast<const MatrixXd&>(a) - b; }

// ----------------------------------------------------------- decompositions --
template <class M>
class LLT {
public:
    LLT() = default;
    explicit LLT(const MatrixXd& a) { compute(a); }
    LLT& compute(const MatrixXd& a) {  // lower factor; info = NumericalIssue when a pivot is not > 0
        l_ = a;
        const Index n = a.rows();
        info_ = Success;
        if (n == 0) return *this;
        const int64_t rc = shim::Blas::get().potrf(102, 'L', n, l_.data(), n);
        if (rc != 0) info_ = NumericalIssue;
        return *this;
    }
    ComputationInfo info() const { return info_; }
    MatrixXd solve(const MatrixXd& b) const {
        MatrixXd x = b;
        const Index n = l_.rows();
        if (n == 0 || b.cols() == 0) return x;
        shim::Blas::get().potrs(102, 'L', n, b.cols(), l_.data(), n, x.data(), std::max<Index>(1, x.rows()));
        return x;
    }
    MatrixXd solve(const Transpose& b) const { return solve(MatrixXd(b)); }
    MatrixXd solve(const ConstBlock& b) const { return solve(MatrixXd(b)); }
    MatrixXd matrixL() const {
        MatrixXd m = l_;
        for (Index j = 0; j < m.cols(); ++j)
            for (Index i = 0; i < j; ++i) m(i, j) = 0.0;
        return m;
    }

private:
    MatrixXd l_;
    ComputationInfo info_ = InvalidInput;
};

template <class M>
class PartialPivLU {
public:
    explicit PartialPivLU(const MatrixXd& a) : lu_(a), piv_(size_t(std::max<Index>(a.rows(), 1))) {
        if (a.rows() != a.cols()) throw std::invalid_argument("PartialPivLU: square matrix required");
        if (a.rows()) shim::Blas::get().getrf(102, a.rows(), a.cols(), lu_.data(), a.rows(), piv_.data());
    }
    MatrixXd inverse() const {
        MatrixXd inv = lu_;
        if (inv.rows()) shim::Blas::get().getri(102, inv.rows(), inv.data(), inv.rows(), piv_.data());
        return inv;
    }

private:
    MatrixXd lu_;
    std::vector<int64_t> piv_;
};

// complete pivoting (Eigen's FullPivLU): rank by the default threshold
// eps·size·max|pivot|, isInvertible ⇔ full rank
template <class M>
class FullPivLU {
public:
    explicit FullPivLU(const MatrixXd& a) : lu_(a), n_(a.rows()), p_(size_t(a.rows())), q_(size_t(a.cols())) {
        if (a.rows() != a.cols()) throw std::invalid_argument("FullPivLU: square matrix required (shim)");
        for (Index i = 0; i < n_; ++i) p_[size_t(i)] = q_[size_t(i)] = i;
        double maxpiv = 0.0;
        rank_ = 0;
        for (Index k = 0; k < n_; ++k) {
            Index bi = k, bj = k;
            double best = -1.0;
            for (Index j = k; j < n_; ++j)
                for (Index i = k; i < n_; ++i)
                    if (std::abs(lu_(i, j)) > best) {
                        best = std::abs(lu_(i, j));
                        bi = i;
                        bj = j;
                    }
            if (k == 0) maxpiv = best;
            if (best <= 0.0) break;
            for (Index j = 0; j < n_; ++j) std::swap(lu_(k, j), lu_(bi, j));
            for (Index i = 0; i < n_; ++i) std::swap(lu_(i, k), lu_(i, bj));
            std::swap(p_[size_t(k)], p_[size_t(bi)]);
            std::swap(q_[size_t(k)], q_[size_t(bj)]);
            for (Index i = k + 1; i < n_; ++i) {
                lu_(i, k) /= lu_(k, k);
                const double f = lu_(i, k);
                for (Index j = k + 1; j < n_; ++j) lu_(i, j) -= f * lu_(k, j);
            }
        }
        const double thr = std::numeric_limits<double>::epsilon() * double(n_) * maxpiv;
        for (Index k = 0; k < n_; ++k)
            if (std::abs(lu_(k, k)) > thr) ++rank_;
    }
    Index rank() const { return rank_; }
    bool isInvertible() const { return rank_ == n_; }
    MatrixXd inverse() const {  // P A Q = L U  →  A⁻¹ = Q U⁻¹ L⁻¹ P
        MatrixXd inv(n_, n_);
        for (Index c = 0; c < n_; ++c) {
            std::vector<double> y(size_t(n_), 0.0);
            for (Index i = 0; i < n_; ++i) y[size_t(i)] = (p_[size_t(i)] == c) ? 1.0 : 0.0;
            for (Index i = 0; i < n_; ++i)
                for (Index k = 0; k < i; ++k) y[size_t(i)] -= lu_(i, k) * y[size_t(k)];
            for (Index i = n_ - 1; i >= 0; --i) {
                for (Index k = i + 1; k < n_; ++k) y[size_t(i)] -= lu_(i, k) * y[size_t(k)];
                y[size_t(i)] /= lu_(i, i);
            }
            for (Index i = 0; i < n_; ++i) inv(q_[size_t(i)], c) = y[size_t(i)];
        }
        return inv;
    }

private:
    MatrixXd lu_;
    Index n_, rank_ = 0;
    std::vector<Index> p_, q_;
};

}  // namespace Eigen
