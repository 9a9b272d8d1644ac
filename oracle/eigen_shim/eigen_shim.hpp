// oracle/eigen_shim/eigen_shim.hpp — TEST INFRASTRUCTURE ONLY.
//
// A minimal, eagerly evaluated stand-in for the subset of Eigen3 that the reference's
// proj/core sources use (Eigen is absent from this image; the reference requires
// "Eigen3 >= 3.3", proj/core/CMakeLists.txt:1). It exists so that the reference's own
// hot-path code compiles unmodified, where it lies, into oracle/_ref/libref_latham.so
// (Oracle-R), which pins the clean-room restatement (Oracle-X).
//
// Design: one dynamic column-major Matrix<T> serves as MatrixXd/VectorXd/MatrixXcd/
// VectorXcd; block views (col, segment, block, middleRows, ...) are Block<T> objects
// that hold a copy of the viewed entries (so every Matrix operation applies to them)
// and write the copy back to the parent on assignment. Expressions are evaluated
// immediately. Decompositions delegate to oracle/linalg.hpp (Cholesky, Jacobi,
// Householder+QL, FFT), i.e. the same published algorithms Eigen implements; results
// agree with Eigen to round-off.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "../linalg.hpp"

namespace Eigen {

using Index = std::ptrdiff_t;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum DecompositionOptions { EigenvaluesOnly = 0x40, ComputeEigenvectors = 0x80 };

template <class T>
struct real_of {
    using type = T;
};
template <class T>
struct real_of<std::complex<T>> {
    using type = T;
};

template <class T>
class Block;

template <class T>
class Matrix {
public:
    using Scalar = T;
    using RealScalar = typename real_of<T>::type;

    Matrix() = default;
    explicit Matrix(Index n) : r_(n), c_(1), a_(static_cast<size_t>(n)) {}
    Matrix(Index r, Index c) : r_(r), c_(c), a_(static_cast<size_t>(r * c)) {}
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) noexcept = default;
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) noexcept = default;
    virtual ~Matrix() = default;

    static Matrix Zero(Index n) { return Zero(n, 1); }
    static Matrix Zero(Index r, Index c) {
        Matrix m(r, c);
        std::fill(m.a_.begin(), m.a_.end(), T(0));
        return m;
    }
    static Matrix Ones(Index n) { return Constant(n, 1, T(1)); }
    static Matrix Ones(Index r, Index c) { return Constant(r, c, T(1)); }
    static Matrix Constant(Index r, Index c, T v) {
        Matrix m(r, c);
        std::fill(m.a_.begin(), m.a_.end(), v);
        return m;
    }
    static Matrix Identity(Index r, Index c) {
        Matrix m = Zero(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = T(1);
        return m;
    }

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    T* data() { return a_.data(); }
    const T* data() const { return a_.data(); }
    void resize(Index n) { resize(n, 1); }
    void resize(Index r, Index c) {
        r_ = r;
        c_ = c;
        a_.assign(static_cast<size_t>(r * c), T(0));
    }
    void setZero() { std::fill(a_.begin(), a_.end(), T(0)); }

    T& operator()(Index i, Index j) { return a_[static_cast<size_t>(i + j * r_)]; }
    const T& operator()(Index i, Index j) const { return a_[static_cast<size_t>(i + j * r_)]; }
    T& operator[](Index i) { return a_[static_cast<size_t>(i)]; }
    const T& operator[](Index i) const { return a_[static_cast<size_t>(i)]; }
    T& operator()(Index i) { return a_[static_cast<size_t>(i)]; }
    const T& operator()(Index i) const { return a_[static_cast<size_t>(i)]; }

    // ---- views (copy + write-back) ----
    Block<T> block(Index i, Index j, Index r, Index c);
    Block<T> block(Index i, Index j, Index r, Index c) const;
    Block<T> col(Index j) { return block(0, j, r_, 1); }
    Block<T> col(Index j) const { return block(0, j, r_, 1); }
    Block<T> row(Index i) { return block(i, 0, 1, c_); }
    Block<T> row(Index i) const { return block(i, 0, 1, c_); }
    Block<T> middleRows(Index i, Index n) { return block(i, 0, n, c_); }
    Block<T> middleRows(Index i, Index n) const { return block(i, 0, n, c_); }
    Block<T> middleCols(Index j, Index n) { return block(0, j, r_, n); }
    Block<T> middleCols(Index j, Index n) const { return block(0, j, r_, n); }
    Block<T> segment(Index i, Index n) { return block(i, 0, n, 1); }
    Block<T> segment(Index i, Index n) const { return block(i, 0, n, 1); }
    Block<T> head(Index n) { return block(0, 0, n, 1); }
    Block<T> head(Index n) const { return block(0, 0, n, 1); }
    Block<T> tail(Index n) { return block(r_ - n, 0, n, 1); }
    Block<T> tail(Index n) const { return block(r_ - n, 0, n, 1); }

    // ---- element-wise and reductions ----
    Matrix transpose() const {
        Matrix m(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) m(j, i) = (*this)(i, j);
        return m;
    }
    Matrix conjugate() const {
        Matrix m = *this;
        if constexpr (!std::is_same_v<T, RealScalar>)
            for (auto& x : m.a_) x = std::conj(x);
        return m;
    }
    Matrix adjoint() const { return transpose().conjugate(); }
    Matrix<RealScalar> real() const {
        Matrix<RealScalar> m(r_, c_);
        for (Index i = 0; i < size(); ++i) m[i] = std::real(a_[i]);
        return m;
    }
    Matrix<RealScalar> imag() const {
        Matrix<RealScalar> m(r_, c_);
        for (Index i = 0; i < size(); ++i) m[i] = std::imag(a_[i]);
        return m;
    }
    Matrix<RealScalar> cwiseAbs() const {
        Matrix<RealScalar> m(r_, c_);
        for (Index i = 0; i < size(); ++i) m[i] = std::abs(a_[i]);
        return m;
    }
    Matrix cwiseProduct(const Matrix& o) const {
        check_same(o);
        Matrix m(r_, c_);
        for (Index i = 0; i < size(); ++i) m[i] = a_[i] * o.a_[i];
        return m;
    }
    Matrix cwiseInverse() const {
        Matrix m(r_, c_);
        for (Index i = 0; i < size(); ++i) m[i] = T(1) / a_[i];
        return m;
    }
    Matrix cwiseSqrt() const {
        Matrix m(r_, c_);
        for (Index i = 0; i < size(); ++i) m[i] = std::sqrt(a_[i]);
        return m;
    }
    template <class U>
    Matrix<U> cast() const {
        Matrix<U> m(r_, c_);
        for (Index i = 0; i < size(); ++i) m[i] = U(a_[i]);
        return m;
    }
    T maxCoeff() const {
        T v = a_.at(0);
        for (const T& x : a_) v = std::max(v, x);
        return v;
    }
    T minCoeff() const {
        T v = a_.at(0);
        for (const T& x : a_) v = std::min(v, x);
        return v;
    }
    T sum() const {
        T s(0);
        for (const T& x : a_) s += x;
        return s;
    }
    T dot(const Matrix& o) const {  // Eigen: conjugate-linear in the first argument
        check_same(o);
        T s(0);
        for (Index i = 0; i < size(); ++i) {
            if constexpr (std::is_same_v<T, RealScalar>) s += a_[i] * o.a_[i];
            else s += std::conj(a_[i]) * o.a_[i];
        }
        return s;
    }
    RealScalar squaredNorm() const {
        RealScalar s(0);
        for (const T& x : a_) s += std::norm(x);
        return s;
    }
    RealScalar norm() const { return std::sqrt(squaredNorm()); }

    Matrix& operator+=(const Matrix& o) {
        check_same(o);
        for (Index i = 0; i < size(); ++i) a_[i] += o.a_[i];
        return *this;
    }
    Matrix& operator-=(const Matrix& o) {
        check_same(o);
        for (Index i = 0; i < size(); ++i) a_[i] -= o.a_[i];
        return *this;
    }
    template <class S>
    Matrix& operator*=(const S& s) {
        for (auto& x : a_) x *= s;
        return *this;
    }
    template <class S>
    Matrix& operator/=(const S& s) {
        for (auto& x : a_) x /= s;
        return *this;
    }

    friend Matrix operator+(const Matrix& a, const Matrix& b) {
        Matrix m = a;
        m += b;
        return m;
    }
    friend Matrix operator-(const Matrix& a, const Matrix& b) {
        Matrix m = a;
        m -= b;
        return m;
    }
    friend Matrix operator-(const Matrix& a) {
        Matrix m = a;
        for (auto& x : m.a_) x = -x;
        return m;
    }
    friend Matrix operator*(const Matrix& a, const Matrix& b) {
        if (a.c_ != b.r_) throw std::runtime_error("eigen_shim: product shape mismatch");
        Matrix m = Zero(a.r_, b.c_);
        for (Index j = 0; j < b.c_; ++j)
            for (Index k = 0; k < a.c_; ++k) {
                const T bkj = b(k, j);
                for (Index i = 0; i < a.r_; ++i) m(i, j) += a(i, k) * bkj;
            }
        return m;
    }
    friend Matrix operator*(const T& s, const Matrix& a) {
        Matrix m = a;
        for (auto& x : m.a_) x = s * x;
        return m;
    }
    friend Matrix operator*(const Matrix& a, const T& s) {
        Matrix m = a;
        for (auto& x : m.a_) x = x * s;
        return m;
    }
    friend Matrix operator/(const Matrix& a, const T& s) {
        Matrix m = a;
        for (auto& x : m.a_) x = x / s;
        return m;
    }
    friend bool operator==(const Matrix& a, const Matrix& b) {
        return a.r_ == b.r_ && a.c_ == b.c_ && a.a_ == b.a_;
    }

protected:
    void check_same(const Matrix& o) const {
        if (o.r_ != r_ || o.c_ != c_) throw std::runtime_error("eigen_shim: shape mismatch");
    }
    Index r_ = 0, c_ = 0;
    std::vector<T> a_;
    template <class U>
    friend class Matrix;
};

// real scalar times complex matrix (e.g. 0.5 * (A + A.adjoint()))
inline Matrix<std::complex<double>> operator*(double s, const Matrix<std::complex<double>>& a) {
    return std::complex<double>(s, 0.0) * a;
}

template <class T>
class Block : public Matrix<T> {
public:
    Block(Matrix<T>* parent, Index i, Index j, Index r, Index c) : Matrix<T>(r, c), p_(parent), i_(i), j_(j) {}
    Block(const Block&) = default;
    Block& operator=(const Matrix<T>& m) {
        if (!p_) throw std::runtime_error("eigen_shim: assignment to a const view");
        if (m.rows() != this->rows() || m.cols() != this->cols())
            throw std::runtime_error("eigen_shim: view assignment shape mismatch");
        for (Index c = 0; c < this->cols(); ++c)
            for (Index r = 0; r < this->rows(); ++r) {
                (*this)(r, c) = m(r, c);
                (*p_)(i_ + r, j_ + c) = m(r, c);
            }
        return *this;
    }
    Block& operator=(const Block& o) { return *this = static_cast<const Matrix<T>&>(o); }
    Block& operator+=(const Matrix<T>& m) { return *this = static_cast<const Matrix<T>&>(*this) + m; }
    Block& operator-=(const Matrix<T>& m) { return *this = static_cast<const Matrix<T>&>(*this) - m; }

private:
    Matrix<T>* p_;
    Index i_, j_;
};

template <class T>
Block<T> Matrix<T>::block(Index i, Index j, Index r, Index c) {
    if (i < 0 || j < 0 || i + r > r_ || j + c > c_) throw std::runtime_error("eigen_shim: view out of range");
    Block<T> b(this, i, j, r, c);
    for (Index cc = 0; cc < c; ++cc)
        for (Index rr = 0; rr < r; ++rr) b(rr, cc) = (*this)(i + rr, j + cc);
    return b;
}

template <class T>
Block<T> Matrix<T>::block(Index i, Index j, Index r, Index c) const {
    if (i < 0 || j < 0 || i + r > r_ || j + c > c_) throw std::runtime_error("eigen_shim: view out of range");
    Block<T> b(nullptr, i, j, r, c);
    for (Index cc = 0; cc < c; ++cc)
        for (Index rr = 0; rr < r; ++rr) b(rr, cc) = (*this)(i + rr, j + cc);
    return b;
}

using MatrixXd = Matrix<double>;
using VectorXd = Matrix<double>;
using MatrixXcd = Matrix<std::complex<double>>;
using VectorXcd = Matrix<std::complex<double>>;

// ---------------------------------------------------------------------------
// decompositions
// ---------------------------------------------------------------------------
template <class MatrixType>
class LLT {
public:
    using T = typename MatrixType::Scalar;
    explicit LLT(const MatrixType& a) : l_(a) {
        const Index n = a.rows();
        // Eigen's LLT reads the lower triangle only
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < j; ++i) l_(i, j) = T(0);
        ok_ = orla::cholesky_lower<T>(n, l_.data());
    }
    ComputationInfo info() const { return ok_ ? Success : NumericalIssue; }

    struct Lower {
        const MatrixType* l;
        MatrixType solve(const MatrixType& b) const {
            MatrixType x = b;
            orla::lower_solve<T>(l->rows(), l->data(), b.cols(), x.data());
            return x;
        }
    };
    struct Upper {  // U = L^H
        const MatrixType* l;
        MatrixType solve(const MatrixType& b) const {
            const Index n = l->rows();
            MatrixType x = b;
            for (Index c = 0; c < x.cols(); ++c)
                for (Index i = n - 1; i >= 0; --i) {
                    T s = x(i, c);
                    for (Index j = i + 1; j < n; ++j) s -= orla::conj_of((*l)(j, i)) * x(j, c);
                    x(i, c) = s / (*l)(i, i);
                }
            return x;
        }
    };
    Lower matrixL() const { return Lower{&l_}; }
    Upper matrixU() const { return Upper{&l_}; }

private:
    MatrixType l_;
    bool ok_ = false;
};

template <class MatrixType>
class SelfAdjointEigenSolver {
public:
    using T = typename MatrixType::Scalar;
    SelfAdjointEigenSolver() = default;
    explicit SelfAdjointEigenSolver(const MatrixType& a, int opts = ComputeEigenvectors) { compute(a, opts); }
    SelfAdjointEigenSolver& compute(const MatrixType& a, int opts = ComputeEigenvectors) {
        const Index n = a.rows();
        evals_.resize(n);
        if (opts & ComputeEigenvectors) {
            vecs_ = MatrixType::Identity(n, n);
            MatrixType w = a;
            jacobi_with_vectors(w);
        } else {
            MatrixType w = a;
            if constexpr (std::is_same_v<T, double>) orla::symmetric_eigenvalues(n, w.data(), evals_.data());
            else orla::jacobi_eigenvalues<T>(n, w.data(), evals_.data());
        }
        return *this;
    }
    const VectorXd& eigenvalues() const { return evals_; }
    const MatrixType& eigenvectors() const { return vecs_; }
    ComputationInfo info() const { return Success; }

private:
    // cyclic Jacobi with accumulated rotations (columns = eigenvectors, ascending)
    void jacobi_with_vectors(MatrixType& A) {
        const Index n = A.rows();
        double fro = A.squaredNorm();
        const double floor_abs = 1e-17 * std::sqrt(fro);
        for (int sweep = 0; sweep < 60; ++sweep) {
            bool rotated = false;
            for (Index p = 0; p < n - 1; ++p)
                for (Index q = p + 1; q < n; ++q) {
                    const T apq = A(p, q);
                    const double r = std::abs(apq);
                    const double app = std::real(A(p, p)), aqq = std::real(A(q, q));
                    if (!(r > floor_abs) || r <= 1.1102230246251565e-16 * std::sqrt(std::abs(app * aqq))) continue;
                    rotated = true;
                    const T ph = apq / r;
                    const T cph = orla::conj_of(ph);
                    for (Index k = 0; k < n; ++k) A(k, q) *= cph;
                    for (Index k = 0; k < n; ++k) A(q, k) *= ph;
                    for (Index k = 0; k < n; ++k) vecs_(k, q) *= cph;
                    const double tau = (aqq - app) / (2.0 * r);
                    const double t = (tau >= 0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
                    const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
                    for (Index k = 0; k < n; ++k) {
                        const T akp = A(k, p), akq = A(k, q);
                        A(k, p) = c * akp - s * akq;
                        A(k, q) = s * akp + c * akq;
                        const T vkp = vecs_(k, p), vkq = vecs_(k, q);
                        vecs_(k, p) = c * vkp - s * vkq;
                        vecs_(k, q) = s * vkp + c * vkq;
                    }
                    for (Index k = 0; k < n; ++k) {
                        const T apk = A(p, k), aqk = A(q, k);
                        A(p, k) = c * apk - s * aqk;
                        A(q, k) = s * apk + c * aqk;
                    }
                    A(p, q) = T(0);
                    A(q, p) = T(0);
                    A(p, p) = T(app - t * r);
                    A(q, q) = T(aqq + t * r);
                }
            if (!rotated) break;
        }
        std::vector<Index> perm(n);
        for (Index i = 0; i < n; ++i) perm[i] = i;
        std::sort(perm.begin(), perm.end(), [&](Index a, Index b) { return std::real(A(a, a)) < std::real(A(b, b)); });
        MatrixType v2(n, n);
        for (Index j = 0; j < n; ++j) {
            evals_[j] = std::real(A(perm[j], perm[j]));
            for (Index i = 0; i < n; ++i) v2(i, j) = vecs_(i, perm[j]);
        }
        vecs_ = v2;
    }
    VectorXd evals_;
    MatrixType vecs_;
};

// Non-Hermitian eigensolver: used only by bc_eigensolve(symmetric = false), which is off
// the hot path; not provided by the shim.
template <class MatrixType>
class ComplexEigenSolver {
public:
    ComplexEigenSolver(const MatrixType&, bool) {
        throw std::runtime_error("eigen_shim: ComplexEigenSolver is not part of the shim");
    }
    VectorXcd eigenvalues() const { return VectorXcd(); }
    MatrixXcd eigenvectors() const { return MatrixXcd(); }
};

template <class T>
class FFT {
public:
    void fwd(std::vector<std::complex<T>>& out, const std::vector<std::complex<T>>& in) {
        out = in;
        orla::fft_forward(out);
    }
};

}  // namespace Eigen
