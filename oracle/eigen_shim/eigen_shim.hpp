// eigen_shim.hpp — the subset of Eigen 3.4 the reference's render path uses, written
// from scratch so /root/reference/proj/src/{math,avatar,lod,crowd,renderer,synthetic,
// bench,metrics}.cpp compile UNMODIFIED into oracle/_ref (Eigen is not installed on
// this box or the GPU box, and there is no network).
//
// TEST INFRASTRUCTURE ONLY (oracle/): never linked into the product.
//
// The shim is eager (no expression templates) and reproduces Eigen 3.4's floating-point
// evaluation order on x86-64 SSE2 without FMA (the reference's Release build,
// CMakeLists.txt:1-8):
//   * coefficient-based ("lazy") products: a column-major LHS with 4 rows (Matrix4f,
//     the SSE packet width) is evaluated column by column as the packet chain
//     ((c0*r0 + c1*r1) + c2*r2) + c3*r3 (etor_product_packet_impl, pmadd = mul then
//     add); every other product coefficient is a reduction of lhs(i,k)*rhs(k,j) over k
//     with redux_novec_unroller's half split (3 terms: a0 + (a1 + a2));
//   * reductions (sum, dot, squaredNorm) of fixed size 4 (Vector4f, quaternion coeffs)
//     use the SSE predux order (a0 + a2) + (a1 + a3); other sizes the half split;
//   * a nested product (A*B*C) is evaluated into a temporary first, as Eigen does for
//     product operands;
//   * Quaternion: toRotationMatrix, the rotation-matrix constructor
//     (quaternionbase_assign_impl), AngleAxis conversion, normalize = coeffs / sqrt(sq)
//     and setFromTwoVectors, whose near-antiparallel branch (a JacobiSVD of the 2x3
//     matrix [a; b] in Eigen) is restated through the path Eigen takes: the more-cols
//     ColPivHouseholderQR preconditioner, V.col(2) = (H0 H1).col(2) (the 2x2 Jacobi
//     sweeps only rotate V's first two columns).
// These orders are Eigen's templates read, not an Eigen build run: this file is where
// that assumption lives (DESIGN.md §2 "parity pin").
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <type_traits>

namespace Eigen {

using Index = std::ptrdiff_t;

namespace shim {

// redux_novec_unroller: split [start, start+n) at n/2, left + right.
template <typename S, typename F>
inline S half_split(F term, int start, int n) {
    if (n == 1) return term(start);
    const int h = n / 2;
    return half_split<S>(term, start, h) + half_split<S>(term, start + h, n - h);
}

// Fixed-size reduction in Eigen's order: SSE predux for a 4-float packet, else half split.
template <typename S, typename F>
inline S redux_sum(F term, int n) {
    if (n == 4 && std::is_same<S, float>::value) return (term(0) + term(2)) + (term(1) + term(3));
    return half_split<S>(term, 0, n);
}

}  // namespace shim

template <typename S, int R, int C, int Options = 0, int MaxR = R, int MaxC = C>
class Matrix;

template <typename M, int BR, int BC>
class BlockRef;

template <typename S, int N>
class DiagonalWrapper {
public:
    explicit DiagonalWrapper(const Matrix<S, N, 1>& d) : d_(d) {}
    const Matrix<S, N, 1>& diagonal() const { return d_; }

private:
    Matrix<S, N, 1> d_;
};

template <typename M>
class CommaInitializer {
public:
    CommaInitializer(M& m, typename M::Scalar first) : m_(m), i_(0) { put(first); }
    template <int R2, int C2>
    CommaInitializer(M& m, const Matrix<typename M::Scalar, R2, C2>& first) : m_(m), i_(0) { put(first); }
    CommaInitializer& operator,(typename M::Scalar v) {
        put(v);
        return *this;
    }
    template <int R2, int C2>
    CommaInitializer& operator,(const Matrix<typename M::Scalar, R2, C2>& v) {
        put(v);
        return *this;
    }

private:
    void put(typename M::Scalar v) {  // row-major fill order, as Eigen's operator<<
        const int r = i_ / M::ColsAtCompileTime, c = i_ % M::ColsAtCompileTime;
        m_(r, c) = v;
        ++i_;
    }
    template <int R2, int C2>
    void put(const Matrix<typename M::Scalar, R2, C2>& v) {  // a row block (R2 == 1)
        static_assert(R2 == 1, "comma initializer: row vectors only");
        for (int c = 0; c < C2; ++c) put(v(0, c));
    }
    M& m_;
    int i_;
};

template <typename S, int R, int C, int Options, int MaxR, int MaxC>
class Matrix {
public:
    using Scalar = S;
    static constexpr int RowsAtCompileTime = R;
    static constexpr int ColsAtCompileTime = C;
    static constexpr int SizeAtCompileTime = R * C;

    Matrix() = default;
    Matrix(S x, S y) {
        static_assert(R * C == 2, "2-vector constructor");
        d_[0] = x;
        d_[1] = y;
    }
    Matrix(S x, S y, S z) {
        static_assert(R * C == 3, "3-vector constructor");
        d_[0] = x;
        d_[1] = y;
        d_[2] = z;
    }
    Matrix(S x, S y, S z, S w) {
        static_assert(R * C == 4 && (R == 1 || C == 1), "4-vector constructor");
        d_[0] = x;
        d_[1] = y;
        d_[2] = z;
        d_[3] = w;
    }
    template <typename M, int BR, int BC>
    Matrix(const BlockRef<M, BR, BC>& b) {  // NOLINT: implicit like Eigen's block -> plain
        *this = b.eval();
    }

    static Matrix Zero() { return Constant(S(0)); }
    static Matrix Ones() { return Constant(S(1)); }
    static Matrix Constant(S v) {
        Matrix m;
        for (int i = 0; i < R * C; ++i) m.d_[i] = v;
        return m;
    }
    static Matrix Identity() {
        Matrix m = Zero();
        for (int i = 0; i < (R < C ? R : C); ++i) m(i, i) = S(1);
        return m;
    }
    static Matrix Unit(int i) {
        Matrix m = Zero();
        m.d_[i] = S(1);
        return m;
    }
    static Matrix UnitX() { return Unit(0); }
    static Matrix UnitY() { return Unit(1); }
    static Matrix UnitZ() { return Unit(2); }
    static Matrix UnitW() { return Unit(3); }

    Index rows() const { return R; }
    Index cols() const { return C; }
    Index size() const { return R * C; }
    S* data() { return d_; }
    const S* data() const { return d_; }

    S& operator()(Index r, Index c) { return d_[c * R + r]; }
    const S& operator()(Index r, Index c) const { return d_[c * R + r]; }
    S& operator()(Index i) { return d_[i]; }
    const S& operator()(Index i) const { return d_[i]; }
    S& operator[](Index i) { return d_[i]; }
    const S& operator[](Index i) const { return d_[i]; }
    S coeff(Index r, Index c) const { return (*this)(r, c); }
    S coeff(Index i) const { return d_[i]; }
    S& coeffRef(Index r, Index c) { return (*this)(r, c); }
    S& coeffRef(Index i) { return d_[i]; }
    S& x() { return d_[0]; }
    S& y() { return d_[1]; }
    S& z() { return d_[2]; }
    S& w() { return d_[3]; }
    S x() const { return d_[0]; }
    S y() const { return d_[1]; }
    S z() const { return d_[2]; }
    S w() const { return d_[3]; }

    CommaInitializer<Matrix> operator<<(S v) { return CommaInitializer<Matrix>(*this, v); }
    template <int R2, int C2>
    CommaInitializer<Matrix> operator<<(const Matrix<S, R2, C2>& v) {
        return CommaInitializer<Matrix>(*this, v);
    }

    Matrix<S, C, R> transpose() const {
        Matrix<S, C, R> t;
        for (int r = 0; r < R; ++r)
            for (int c = 0; c < C; ++c) t(c, r) = (*this)(r, c);
        return t;
    }
    Matrix<S, C, R> adjoint() const { return transpose(); }

    // ---- blocks: const forms return copies, mutable forms a write-through proxy ----
    template <int BR, int BC>
    Matrix<S, BR, BC> block(Index r0, Index c0) const {
        Matrix<S, BR, BC> b;
        for (int r = 0; r < BR; ++r)
            for (int c = 0; c < BC; ++c) b(r, c) = (*this)(r0 + r, c0 + c);
        return b;
    }
    template <int BR, int BC>
    Matrix<S, BR, BC> topLeftCorner() const { return block<BR, BC>(0, 0); }
    template <int BR, int BC>
    Matrix<S, BR, BC> topRightCorner() const { return block<BR, BC>(0, C - BC); }
    template <int BR, int BC>
    BlockRef<Matrix, BR, BC> topLeftCorner() { return BlockRef<Matrix, BR, BC>(*this, 0, 0); }
    template <int BR, int BC>
    BlockRef<Matrix, BR, BC> topRightCorner() { return BlockRef<Matrix, BR, BC>(*this, 0, C - BC); }
    Matrix<S, R, 1> col(Index c) const { return block<R, 1>(0, c); }
    BlockRef<Matrix, R, 1> col(Index c) { return BlockRef<Matrix, R, 1>(*this, 0, c); }
    Matrix<S, 1, C> row(Index r) const { return block<1, C>(r, 0); }
    BlockRef<Matrix, 1, C> row(Index r) { return BlockRef<Matrix, 1, C>(*this, r, 0); }
    template <int N>
    Matrix<S, N, 1> head() const {
        static_assert(C == 1, "head<N> on column vectors");
        return block<N, 1>(0, 0);
    }

    // ---- coefficient-wise ----
    template <typename F>
    Matrix map(F f) const {
        Matrix out;
        for (int i = 0; i < R * C; ++i) out.d_[i] = f(d_[i]);
        return out;
    }
    Matrix cwiseAbs() const { return map([](S v) { return std::abs(v); }); }
    Matrix cwiseMax(S s) const { return map([s](S v) { return std::max(v, s); }); }
    Matrix cwiseMin(S s) const { return map([s](S v) { return std::min(v, s); }); }
    Matrix cwiseMax(const Matrix& o) const {
        Matrix out;
        for (int i = 0; i < R * C; ++i) out.d_[i] = std::max(d_[i], o.d_[i]);
        return out;
    }
    Matrix cwiseMin(const Matrix& o) const {
        Matrix out;
        for (int i = 0; i < R * C; ++i) out.d_[i] = std::min(d_[i], o.d_[i]);
        return out;
    }
    Matrix cwiseProduct(const Matrix& o) const {
        Matrix out;
        for (int i = 0; i < R * C; ++i) out.d_[i] = d_[i] * o.d_[i];
        return out;
    }
    S maxCoeff() const {
        S m = d_[0];
        for (int i = 1; i < R * C; ++i) m = std::max(m, d_[i]);
        return m;
    }
    S minCoeff() const {
        S m = d_[0];
        for (int i = 1; i < R * C; ++i) m = std::min(m, d_[i]);
        return m;
    }
    bool allFinite() const {
        for (int i = 0; i < R * C; ++i)
            if (!std::isfinite(d_[i])) return false;
        return true;
    }
    S sum() const {
        return shim::redux_sum<S>([this](int i) { return d_[i]; }, R * C);
    }
    S dot(const Matrix& o) const {
        return shim::redux_sum<S>([this, &o](int i) { return d_[i] * o.d_[i]; }, R * C);
    }
    S squaredNorm() const { return dot(*this); }
    S norm() const { return std::sqrt(squaredNorm()); }
    Matrix normalized() const {  // MatrixBase::normalized: n / sqrt(squaredNorm)
        const S z = squaredNorm();
        if (z > S(0)) return *this / std::sqrt(z);
        return *this;
    }
    void normalize() {
        const S z = squaredNorm();
        if (z > S(0)) *this /= std::sqrt(z);
    }
    Matrix cross(const Matrix& o) const {  // MatrixBase::cross (scalar path)
        static_assert(R * C == 3, "cross of 3-vectors");
        return Matrix(d_[1] * o.d_[2] - d_[2] * o.d_[1], d_[2] * o.d_[0] - d_[0] * o.d_[2],
                      d_[0] * o.d_[1] - d_[1] * o.d_[0]);
    }
    S determinant() const {  // bruteforce_det3_helper order (3x3 only)
        static_assert(R == 3 && C == 3, "determinant: 3x3 only");
        const auto h = [this](int a, int b, int c) {
            return (*this)(0, a) * ((*this)(1, b) * (*this)(2, c) - (*this)(1, c) * (*this)(2, b));
        };
        return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
    }
    S trace() const {
        return shim::half_split<S>([this](int i) { return (*this)(i, i); }, 0, R < C ? R : C);
    }
    DiagonalWrapper<S, R * C> asDiagonal() const {
        static_assert(C == 1, "asDiagonal of a column vector");
        return DiagonalWrapper<S, R * C>(*this);
    }
    void setZero() { *this = Zero(); }
    void setIdentity() { *this = Identity(); }
    void swap(Matrix& o) { std::swap(*this, o); }

    Matrix& operator+=(const Matrix& o) {
        for (int i = 0; i < R * C; ++i) d_[i] = d_[i] + o.d_[i];
        return *this;
    }
    Matrix& operator-=(const Matrix& o) {
        for (int i = 0; i < R * C; ++i) d_[i] = d_[i] - o.d_[i];
        return *this;
    }
    Matrix& operator*=(S s) {
        for (int i = 0; i < R * C; ++i) d_[i] = d_[i] * s;
        return *this;
    }
    Matrix& operator/=(S s) {
        for (int i = 0; i < R * C; ++i) d_[i] = d_[i] / s;
        return *this;
    }
    Matrix operator-() const { return map([](S v) { return -v; }); }
    friend Matrix operator+(const Matrix& a, const Matrix& b) {
        Matrix out;
        for (int i = 0; i < R * C; ++i) out.d_[i] = a.d_[i] + b.d_[i];
        return out;
    }
    friend Matrix operator-(const Matrix& a, const Matrix& b) {
        Matrix out;
        for (int i = 0; i < R * C; ++i) out.d_[i] = a.d_[i] - b.d_[i];
        return out;
    }
    friend Matrix operator*(S s, const Matrix& a) { return a.map([s](S v) { return s * v; }); }
    friend Matrix operator*(const Matrix& a, S s) { return a.map([s](S v) { return v * s; }); }
    friend Matrix operator/(const Matrix& a, S s) { return a.map([s](S v) { return v / s; }); }
    friend bool operator==(const Matrix& a, const Matrix& b) {
        for (int i = 0; i < R * C; ++i)
            if (!(a.d_[i] == b.d_[i])) return false;
        return true;
    }
    friend bool operator!=(const Matrix& a, const Matrix& b) { return !(a == b); }

private:
    S d_[R * C] = {};
};

// Write-through view of a fixed block of a plain matrix (assignment targets only).
template <typename M, int BR, int BC>
class BlockRef {
public:
    using S = typename M::Scalar;
    BlockRef(M& m, Index r0, Index c0) : m_(m), r0_(r0), c0_(c0) {}
    Matrix<S, BR, BC> eval() const { return static_cast<const M&>(m_).template block<BR, BC>(r0_, c0_); }
    BlockRef& operator=(const Matrix<S, BR, BC>& v) {
        for (int r = 0; r < BR; ++r)
            for (int c = 0; c < BC; ++c) m_(r0_ + r, c0_ + c) = v(r, c);
        return *this;
    }
    BlockRef& operator=(const BlockRef& o) { return *this = o.eval(); }
    BlockRef& operator+=(const Matrix<S, BR, BC>& v) { return *this = eval() + v; }
    BlockRef& operator-=(const Matrix<S, BR, BC>& v) { return *this = eval() - v; }
    S& operator()(Index r, Index c) { return m_(r0_ + r, c0_ + c); }
    S& operator()(Index i) { return BC == 1 ? m_(r0_ + i, c0_) : m_(r0_, c0_ + i); }
    S squaredNorm() const { return eval().squaredNorm(); }
    S norm() const { return eval().norm(); }
    friend bool operator==(const BlockRef& a, const Matrix<S, BR, BC>& b) { return a.eval() == b; }
    friend bool operator!=(const BlockRef& a, const Matrix<S, BR, BC>& b) { return a.eval() != b; }

private:
    M& m_;
    Index r0_, c0_;
};

// Products (see the header comment for the two orders).
template <typename S, int R, int K, int C>
Matrix<S, R, C> operator*(const Matrix<S, R, K>& a, const Matrix<S, K, C>& b) {
    Matrix<S, R, C> out;
    for (int c = 0; c < C; ++c) {
        for (int r = 0; r < R; ++r) {
            if (R == 4 && std::is_same<S, float>::value) {  // column packet chain
                S acc = a(r, 0) * b(0, c);
                for (int k = 1; k < K; ++k) acc = acc + a(r, k) * b(k, c);
                out(r, c) = acc;
            } else {
                out(r, c) = shim::half_split<S>([&](int k) { return a(r, k) * b(k, c); }, 0, K);
            }
        }
    }
    return out;
}
template <typename M, int BR, int BC, typename S, int C>
Matrix<S, BR, C> operator*(const BlockRef<M, BR, BC>& a, const Matrix<S, BC, C>& b) {
    return a.eval() * b;
}

// Matrix * diagonal (DiagonalProduct, OnTheRight): column j scaled by d(j).
template <typename S, int R, int N>
Matrix<S, R, N> operator*(const Matrix<S, R, N>& a, const DiagonalWrapper<S, N>& d) {
    Matrix<S, R, N> out;
    for (int c = 0; c < N; ++c)
        for (int r = 0; r < R; ++r) out(r, c) = d.diagonal()(c) * a(r, c);
    return out;
}

using Matrix2f = Matrix<float, 2, 2>;
using Matrix3f = Matrix<float, 3, 3>;
using Matrix4f = Matrix<float, 4, 4>;
using Vector2f = Matrix<float, 2, 1>;
using Vector3f = Matrix<float, 3, 1>;
using Vector4f = Matrix<float, 4, 1>;
using RowVector4f = Matrix<float, 1, 4>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;

}  // namespace Eigen
