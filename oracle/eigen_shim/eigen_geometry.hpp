// eigen_geometry.hpp — Quaternion / AngleAxis subset of Eigen 3.4 for the reference
// build in oracle/_ref (see eigen_shim.hpp for the contract). TEST INFRASTRUCTURE ONLY.
#pragma once

#include "eigen_shim.hpp"

namespace Eigen {

template <typename S>
class AngleAxis {
public:
    AngleAxis() = default;
    AngleAxis(S angle, const Matrix<S, 3, 1>& axis) : angle_(angle), axis_(axis) {}
    S angle() const { return angle_; }
    const Matrix<S, 3, 1>& axis() const { return axis_; }

private:
    S angle_ = S(0);
    Matrix<S, 3, 1> axis_ = Matrix<S, 3, 1>::UnitX();
};

namespace shim {

// V.col(2) of JacobiSVD<Matrix<S,2,3>>(m, ComputeFullV), m = [v0^T; v1^T]: Eigen takes
// the more-columns-than-rows R-SVD path (JacobiSVD::compute): m is divided by its
// largest |coefficient|, ColPivHouseholderQR factors the 3x2 adjoint (column pivoting by
// norm, first column wins ties; makeHouseholder per column; applyHouseholderOnTheLeft),
// and V is householderQ() evaluated into the identity from the last reflector to the
// first. The 2x2 Jacobi sweeps and the singular-value sort only touch V's first two
// columns, so column 2 is Q's.
template <typename S>
Matrix<S, 3, 1> svd_null_axis(const Matrix<S, 3, 1>& v0, const Matrix<S, 3, 1>& v1) {
    S scale = S(0);
    for (int i = 0; i < 3; ++i) scale = std::max(scale, std::max(std::abs(v0[i]), std::abs(v1[i])));
    if (scale == S(0)) scale = S(1);
    S a[2][3];  // the adjoint's columns
    for (int i = 0; i < 3; ++i) {
        a[0][i] = v0[i] / scale;
        a[1][i] = v1[i] / scale;
    }
    const auto norm3 = [](const S* x) { return std::sqrt(x[0] * x[0] + (x[1] * x[1] + x[2] * x[2])); };
    if (norm3(a[1]) > norm3(a[0])) std::swap(a[0], a[1]);  // pivot: the larger-norm column first
    // makeHouseholder of column 0 (3 entries)
    S e0[2], tau0, beta0;
    {
        const S c0 = a[0][0];
        const S tail = a[0][1] * a[0][1] + a[0][2] * a[0][2];
        if (tail <= std::numeric_limits<S>::min()) {
            tau0 = S(0);
            beta0 = c0;
            e0[0] = e0[1] = S(0);
        } else {
            beta0 = std::sqrt(c0 * c0 + tail);
            if (c0 >= S(0)) beta0 = -beta0;
            e0[0] = a[0][1] / (c0 - beta0);
            e0[1] = a[0][2] / (c0 - beta0);
            tau0 = (beta0 - c0) / beta0;
        }
    }
    // H0 applied to column 1 (applyHouseholderOnTheLeft on a 3x1 block)
    S b[3] = {a[1][0], a[1][1], a[1][2]};
    if (tau0 != S(0)) {
        S tmp = e0[0] * b[1] + e0[1] * b[2];
        tmp = tmp + b[0];
        b[0] = b[0] - tau0 * tmp;
        b[1] = b[1] - tmp * (tau0 * e0[0]);
        b[2] = b[2] - tmp * (tau0 * e0[1]);
    }
    // makeHouseholder of column 1, rows 1..2 (2 entries)
    S e1, tau1;
    {
        const S c0 = b[1];
        const S tail = b[2] * b[2];
        if (tail <= std::numeric_limits<S>::min()) {
            tau1 = S(0);
            e1 = S(0);
        } else {
            S beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= S(0)) beta = -beta;
            e1 = b[2] / (c0 - beta);
            tau1 = (beta - c0) / beta;
        }
    }
    // householderQ().evalTo: identity, then H1 on the bottom-right 2x2, then H0 on the
    // whole 3x3. Only column 2 is needed.
    S q[3] = {S(0), S(0), S(1)};
    if (tau1 != S(0)) {  // block rows 1..2, column 2 of the 2x2 block is (0, 1)
        S tmp = e1 * q[2];
        tmp = tmp + q[1];
        q[1] = q[1] - tau1 * tmp;
        q[2] = q[2] - tmp * (tau1 * e1);
    }
    if (tau0 != S(0)) {
        S tmp = e0[0] * q[1] + e0[1] * q[2];
        tmp = tmp + q[0];
        q[0] = q[0] - tau0 * tmp;
        q[1] = q[1] - tmp * (tau0 * e0[0]);
        q[2] = q[2] - tmp * (tau0 * e0[1]);
    }
    return Matrix<S, 3, 1>(q[0], q[1], q[2]);
}

}  // namespace shim

template <typename S>
class Quaternion {
public:
    using Scalar = S;
    Quaternion() = default;
    Quaternion(S w, S x, S y, S z) : c_(x, y, z, w) {}
    explicit Quaternion(const Matrix<S, 4, 1>& coeffs) : c_(coeffs) {}
    explicit Quaternion(const Matrix<S, 3, 3>& m) { *this = from_rotation(m); }
    explicit Quaternion(const AngleAxis<S>& aa) {  // w = cos(a/2), vec = sin(a/2) * axis
        const S ha = S(0.5) * aa.angle();
        c_[3] = std::cos(ha);
        const Matrix<S, 3, 1> v = std::sin(ha) * aa.axis();
        c_[0] = v[0];
        c_[1] = v[1];
        c_[2] = v[2];
    }
    static Quaternion Identity() { return Quaternion(S(1), S(0), S(0), S(0)); }

    S& x() { return c_[0]; }
    S& y() { return c_[1]; }
    S& z() { return c_[2]; }
    S& w() { return c_[3]; }
    S x() const { return c_[0]; }
    S y() const { return c_[1]; }
    S z() const { return c_[2]; }
    S w() const { return c_[3]; }
    Matrix<S, 4, 1>& coeffs() { return c_; }
    const Matrix<S, 4, 1>& coeffs() const { return c_; }
    Matrix<S, 3, 1> vec() const { return Matrix<S, 3, 1>(c_[0], c_[1], c_[2]); }

    S dot(const Quaternion& o) const { return c_.dot(o.c_); }
    S squaredNorm() const { return c_.squaredNorm(); }
    S norm() const { return c_.norm(); }
    void normalize() { c_.normalize(); }
    Quaternion normalized() const { return Quaternion(c_.normalized()); }

    Matrix<S, 3, 3> toRotationMatrix() const {  // QuaternionBase::toRotationMatrix
        Matrix<S, 3, 3> r;
        const S tx = S(2) * x(), ty = S(2) * y(), tz = S(2) * z();
        const S twx = tx * w(), twy = ty * w(), twz = tz * w();
        const S txx = tx * x(), txy = ty * x(), txz = tz * x();
        const S tyy = ty * y(), tyz = tz * y(), tzz = tz * z();
        r(0, 0) = S(1) - (tyy + tzz);
        r(0, 1) = txy - twz;
        r(0, 2) = txz + twy;
        r(1, 0) = txy + twz;
        r(1, 1) = S(1) - (txx + tzz);
        r(1, 2) = tyz - twx;
        r(2, 0) = txz - twy;
        r(2, 1) = tyz + twx;
        r(2, 2) = S(1) - (txx + tyy);
        return r;
    }

    // Generic (non-SSE) quat_product; only skin_rotations uses it, which render_frame
    // never enables (renderer.cpp:257-261).
    friend Quaternion operator*(const Quaternion& a, const Quaternion& b) {
        return Quaternion(a.w() * b.w() - a.x() * b.x() - a.y() * b.y() - a.z() * b.z(),
                          a.w() * b.x() + a.x() * b.w() + a.y() * b.z() - a.z() * b.y(),
                          a.w() * b.y() + a.y() * b.w() + a.z() * b.x() - a.x() * b.z(),
                          a.w() * b.z() + a.z() * b.w() + a.x() * b.y() - a.y() * b.x());
    }

    // QuaternionBase::setFromTwoVectors (dummy_precision<float> = 1e-5).
    static Quaternion FromTwoVectors(const Matrix<S, 3, 1>& a, const Matrix<S, 3, 1>& b) {
        const Matrix<S, 3, 1> v0 = a.normalized();
        const Matrix<S, 3, 1> v1 = b.normalized();
        S c = v1.dot(v0);
        Quaternion q;
        if (c < S(-1) + S(1e-5)) {
            c = std::max(c, S(-1));
            const Matrix<S, 3, 1> axis = shim::svd_null_axis(v0, v1);
            const S w2 = (S(1) + c) * S(0.5);
            q.c_[3] = std::sqrt(w2);
            const S s = std::sqrt(S(1) - w2);
            q.c_[0] = axis[0] * s;
            q.c_[1] = axis[1] * s;
            q.c_[2] = axis[2] * s;
            return q;
        }
        const Matrix<S, 3, 1> axis = v0.cross(v1);
        const S s = std::sqrt((S(1) + c) * S(2));
        const S invs = S(1) / s;
        q.c_[0] = axis[0] * invs;
        q.c_[1] = axis[1] * invs;
        q.c_[2] = axis[2] * invs;
        q.c_[3] = s * S(0.5);
        return q;
    }

private:
    static Quaternion from_rotation(const Matrix<S, 3, 3>& m) {  // quaternionbase_assign_impl
        Quaternion q;
        S t = m.trace();
        if (t > S(0)) {
            t = std::sqrt(t + S(1));
            q.c_[3] = S(0.5) * t;
            t = S(0.5) / t;
            q.c_[0] = (m(2, 1) - m(1, 2)) * t;
            q.c_[1] = (m(0, 2) - m(2, 0)) * t;
            q.c_[2] = (m(1, 0) - m(0, 1)) * t;
        } else {
            int i = 0;
            if (m(1, 1) > m(0, 0)) i = 1;
            if (m(2, 2) > m(i, i)) i = 2;
            const int j = (i + 1) % 3, k = (j + 1) % 3;
            t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + S(1));
            q.c_[i] = S(0.5) * t;
            t = S(0.5) / t;
            q.c_[3] = (m(k, j) - m(j, k)) * t;
            q.c_[j] = (m(j, i) + m(i, j)) * t;
            q.c_[k] = (m(k, i) + m(i, k)) * t;
        }
        return q;
    }

    Matrix<S, 4, 1> c_ = Matrix<S, 4, 1>(S(0), S(0), S(0), S(1));
};

using Quaternionf = Quaternion<float>;
using AngleAxisf = AngleAxis<float>;

}  // namespace Eigen
