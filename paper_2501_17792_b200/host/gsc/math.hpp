// Fixed-size float math for the host side of the B200 crowd renderer.
//
// The reference builds on Eigen 3.4 (/root/reference/proj/include/gsc/math.hpp:5-19),
// which is not available here. These types keep Eigen's storage (column-major
// matrices, quaternion coeffs x,y,z,w) and its floating-point evaluation order for
// the operations the render path uses, so that host-side results (camera basis,
// covariance cache, sampled poses) are reproducible bit for bit by the GPU kernels and
// by the CPU oracle. The orders:
//   * length-3 reductions (dot, norm, Mat3 products): a0 + (a1 + a2)
//   * Mat4 * Mat4 / Mat4 * Vec4 (SSE packet path): ((c0*r0 + c1*r1) + c2*r2) + c3*r3
//   * length-4 reductions (quaternion dot / norm, SSE predux): (a0 + a2) + (a1 + a3)
// Build with -ffp-contract=off: the reference's Release build has no -march, so x86-64
// SSE2 code without FMA contraction.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>

namespace gsc {

inline constexpr float kAlphaMax = 0.99f;
inline constexpr float kAlphaCutoff = 1.0f / 255.0f;
inline constexpr float kCovDilation = 0.3f;
inline constexpr float kPsnrCap = 99.0f;

// v.cast<T>() / m.cast<T>() as Eigen spells them: a proxy converting to any caller type
// with Eigen-style element access (the reference's tests cast to Eigen's double types).
template <typename T, int N>
struct CastVector {
    T v[N];
    template <typename M>
    operator M() const {  // NOLINT: implicit, as Eigen's cast expression
        M out;
        for (int i = 0; i < N; ++i) out(i) = v[i];
        return out;
    }
};
template <typename T, int R, int C>
struct CastMatrix {
    T m[R * C];  // column-major
    template <typename M>
    operator M() const {  // NOLINT
        M out;
        for (int c = 0; c < C; ++c)
            for (int r = 0; r < R; ++r) out(r, c) = m[c * R + r];
        return out;
    }
};

struct Vec2 {
    float v[2] = {0.0f, 0.0f};
    Vec2() = default;
    Vec2(float x, float y) : v{x, y} {}
    float x() const { return v[0]; }
    float y() const { return v[1]; }
    float& operator[](int i) { return v[i]; }
    float operator[](int i) const { return v[i]; }
    template <typename T>
    CastVector<T, 2> cast() const { return {{static_cast<T>(v[0]), static_cast<T>(v[1])}}; }
};

struct Vec3 {
    float v[3] = {0.0f, 0.0f, 0.0f};
    Vec3() = default;
    Vec3(float x, float y, float z) : v{x, y, z} {}
    static Vec3 Zero() { return Vec3(); }
    static Vec3 Ones() { return Vec3(1.0f, 1.0f, 1.0f); }
    static Vec3 Constant(float c) { return Vec3(c, c, c); }
    float x() const { return v[0]; }
    float y() const { return v[1]; }
    float z() const { return v[2]; }
    float& operator[](int i) { return v[i]; }
    float operator[](int i) const { return v[i]; }

    float dot(const Vec3& o) const { return v[0] * o.v[0] + (v[1] * o.v[1] + v[2] * o.v[2]); }
    float squaredNorm() const { return dot(*this); }
    float norm() const { return std::sqrt(squaredNorm()); }
    Vec3 normalized() const {
        const float n = norm();
        return n > 0.0f ? Vec3(v[0] / n, v[1] / n, v[2] / n) : *this;
    }
    void normalize() { *this = normalized(); }
    Vec3 cross(const Vec3& o) const {
        return Vec3(v[1] * o.v[2] - v[2] * o.v[1], v[2] * o.v[0] - v[0] * o.v[2],
                    v[0] * o.v[1] - v[1] * o.v[0]);
    }
    Vec3 cwiseMax(float c) const {
        return Vec3(std::fmax(v[0], c), std::fmax(v[1], c), std::fmax(v[2], c));
    }
    Vec3 cwiseMin(float c) const {
        return Vec3(std::fmin(v[0], c), std::fmin(v[1], c), std::fmin(v[2], c));
    }
    Vec3 cwiseAbs() const { return Vec3(std::fabs(v[0]), std::fabs(v[1]), std::fabs(v[2])); }
    float maxCoeff() const { return std::fmax(v[0], std::fmax(v[1], v[2])); }
    template <typename T>
    CastVector<T, 3> cast() const { return {{static_cast<T>(v[0]), static_cast<T>(v[1]), static_cast<T>(v[2])}}; }
};

inline Vec3 operator+(const Vec3& a, const Vec3& b) {
    return Vec3(a[0] + b[0], a[1] + b[1], a[2] + b[2]);
}
inline Vec3 operator-(const Vec3& a, const Vec3& b) {
    return Vec3(a[0] - b[0], a[1] - b[1], a[2] - b[2]);
}
inline Vec3 operator-(const Vec3& a) { return Vec3(-a[0], -a[1], -a[2]); }
inline Vec3 operator*(float s, const Vec3& a) { return Vec3(s * a[0], s * a[1], s * a[2]); }
inline Vec3 operator*(const Vec3& a, float s) { return Vec3(a[0] * s, a[1] * s, a[2] * s); }
inline Vec3 operator/(const Vec3& a, float s) { return Vec3(a[0] / s, a[1] / s, a[2] / s); }

struct Vec4 {
    float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    Vec4() = default;
    Vec4(float x, float y, float z, float w) : v{x, y, z, w} {}
    float& operator[](int i) { return v[i]; }
    float operator[](int i) const { return v[i]; }
    template <int N>
    Vec3 head() const {
        static_assert(N == 3, "head<3>() only");
        return Vec3(v[0], v[1], v[2]);
    }
};

// Column-major 3x3: m[c*3 + r].
struct Mat3 {
    float m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    static Mat3 Identity() { return Mat3(); }
    float& operator()(int r, int c) { return m[c * 3 + r]; }
    float operator()(int r, int c) const { return m[c * 3 + r]; }
    Mat3 transpose() const {
        Mat3 t;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) t(r, c) = (*this)(c, r);
        return t;
    }
    float trace() const { return m[0] + (m[4] + m[8]); }
    template <typename T>
    CastMatrix<T, 3, 3> cast() const {
        CastMatrix<T, 3, 3> out;
        for (int i = 0; i < 9; ++i) out.m[i] = static_cast<T>(m[i]);
        return out;
    }
};

// Coefficient-based 3x3 product: inner reduction a0 + (a1 + a2).
inline Mat3 operator*(const Mat3& a, const Mat3& b) {
    Mat3 out;
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r)
            out(r, c) = a(r, 0) * b(0, c) + (a(r, 1) * b(1, c) + a(r, 2) * b(2, c));
    return out;
}
inline Vec3 operator*(const Mat3& a, const Vec3& v) {
    Vec3 out;
    for (int r = 0; r < 3; ++r) out[r] = a(r, 0) * v[0] + (a(r, 1) * v[1] + a(r, 2) * v[2]);
    return out;
}

// Column-major 4x4: m[c*4 + r] (Eigen::Matrix4f storage).
struct Mat4 {
    float m[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
    static Mat4 Identity() { return Mat4(); }
    float& operator()(int r, int c) { return m[c * 4 + r]; }
    float operator()(int r, int c) const { return m[c * 4 + r]; }
    Mat3 topLeft3() const {
        Mat3 out;
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) out(r, c) = (*this)(r, c);
        return out;
    }
    Vec3 translation() const { return Vec3(m[12], m[13], m[14]); }
    void setTopLeft3(const Mat3& a) {
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) (*this)(r, c) = a(r, c);
    }
    void setTranslation(const Vec3& t) {
        m[12] = t[0];
        m[13] = t[1];
        m[14] = t[2];
    }
    template <int R, int C>
    auto topRightCorner() const {  // Eigen's block of the translation column / rotation
        static_assert(R == 3 && C == 1, "topRightCorner<3, 1>() only");
        return translation();
    }
    template <int R, int C>
    Mat3 topLeftCorner() const {
        static_assert(R == 3 && C == 3, "topLeftCorner<3, 3>() only");
        return topLeft3();
    }
    template <typename T>
    CastMatrix<T, 4, 4> cast() const {
        CastMatrix<T, 4, 4> out;
        for (int i = 0; i < 16; ++i) out.m[i] = static_cast<T>(m[i]);
        return out;
    }
};

// SSE packet product (etor_product_packet_impl, ColMajor): res column c accumulated
// over k = 0..3 in order, multiply then add (no FMA).
inline Mat4 operator*(const Mat4& a, const Mat4& b) {
    Mat4 out;
    for (int c = 0; c < 4; ++c) {
        for (int r = 0; r < 4; ++r) {
            float acc = a(r, 0) * b(0, c);
            acc = acc + a(r, 1) * b(1, c);
            acc = acc + a(r, 2) * b(2, c);
            acc = acc + a(r, 3) * b(3, c);
            out(r, c) = acc;
        }
    }
    return out;
}
inline Vec4 operator*(const Mat4& a, const Vec4& v) {
    Vec4 out;
    for (int r = 0; r < 4; ++r) {
        float acc = a(r, 0) * v[0];
        acc = acc + a(r, 1) * v[1];
        acc = acc + a(r, 2) * v[2];
        acc = acc + a(r, 3) * v[3];
        out[r] = acc;
    }
    return out;
}

// Quaternion, coefficient storage (x, y, z, w) as in Eigen.
struct Quat {
    float c[4] = {0.0f, 0.0f, 0.0f, 1.0f};  // x, y, z, w
    Quat() = default;
    Quat(float w, float x, float y, float z) : c{x, y, z, w} {}
    static Quat Identity() { return Quat(); }
    static Quat FromCoeffs(const float* xyzw) {
        Quat q;
        for (int i = 0; i < 4; ++i) q.c[i] = xyzw[i];
        return q;
    }
    float x() const { return c[0]; }
    float y() const { return c[1]; }
    float z() const { return c[2]; }
    float w() const { return c[3]; }
    // SSE predux of a 4-packet: (c0 + c2) + (c1 + c3).
    float dot(const Quat& o) const {
        const float p0 = c[0] * o.c[0], p1 = c[1] * o.c[1], p2 = c[2] * o.c[2],
                    p3 = c[3] * o.c[3];
        return (p0 + p2) + (p1 + p3);
    }
    float squaredNorm() const { return dot(*this); }
    float norm() const { return std::sqrt(squaredNorm()); }
    void normalize() {
        const float z = squaredNorm();
        if (z > 0.0f) {
            const float n = std::sqrt(z);
            for (float& v : c) v = v / n;
        }
    }
    Quat normalized() const {
        Quat q = *this;
        q.normalize();
        return q;
    }
    Mat3 toRotationMatrix() const {
        const float tx = 2.0f * c[0], ty = 2.0f * c[1], tz = 2.0f * c[2];
        const float twx = tx * c[3], twy = ty * c[3], twz = tz * c[3];
        const float txx = tx * c[0], txy = ty * c[0], txz = tz * c[0];
        const float tyy = ty * c[1], tyz = tz * c[1], tzz = tz * c[2];
        Mat3 r;
        r(0, 0) = 1.0f - (tyy + tzz);
        r(0, 1) = txy - twz;
        r(0, 2) = txz + twy;
        r(1, 0) = txy + twz;
        r(1, 1) = 1.0f - (txx + tzz);
        r(1, 2) = tyz - twx;
        r(2, 0) = txz - twy;
        r(2, 1) = tyz + twx;
        r(2, 2) = 1.0f - (txx + tyy);
        return r;
    }
    // Quaternion(AngleAxis): w = cos(a/2), vec = sin(a/2) * axis.
    static Quat FromAngleAxis(float angle, const Vec3& axis) {
        const float ha = 0.5f * angle;
        const float s = std::sin(ha);
        return Quat(std::cos(ha), s * axis[0], s * axis[1], s * axis[2]);
    }
    static Quat FromRotationMatrix(const Mat3& m);
    static Quat FromTwoVectors(const Vec3& a, const Vec3& b);
};

inline Quat Quat::FromRotationMatrix(const Mat3& m) {
    Quat q;
    float t = m.trace();
    if (t > 0.0f) {
        t = std::sqrt(t + 1.0f);
        q.c[3] = 0.5f * t;
        t = 0.5f / t;
        q.c[0] = (m(2, 1) - m(1, 2)) * t;
        q.c[1] = (m(0, 2) - m(2, 0)) * t;
        q.c[2] = (m(1, 0) - m(0, 1)) * t;
    } else {
        int i = 0;
        if (m(1, 1) > m(0, 0)) i = 1;
        if (m(2, 2) > m(i, i)) i = 2;
        const int j = (i + 1) % 3;
        const int k = (j + 1) % 3;
        t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + 1.0f);
        q.c[i] = 0.5f * t;
        t = 0.5f / t;
        q.c[3] = (m(k, j) - m(j, k)) * t;
        q.c[j] = (m(j, i) + m(i, j)) * t;
        q.c[k] = (m(k, i) + m(i, k)) * t;
    }
    return q;
}

// V.col(2) of Eigen's JacobiSVD<Matrix<float,2,3>>(m, ComputeFullV), m = [v0^T; v1^T], the
// axis setFromTwoVectors takes for nearly opposite vectors. Eigen reaches it through the
// R-SVD preconditioner: m is divided by its largest |coefficient|, ColPivHouseholderQR
// factors the 3x2 adjoint (the larger-norm column first, ties keep the first;
// makeHouseholder per column; the reflector applied to the other column), and V =
// householderQ() is evaluated into the identity from the last reflector to the first; the
// 2x2 Jacobi sweeps and the singular-value sort only rotate V's first two columns. The
// synthetic generator hits this branch for about 3 Gaussians per 218 K-Gaussian template.
inline Vec3 svd_null_axis(const Vec3& v0, const Vec3& v1) {
    float scale = 0.0f;
    for (int i = 0; i < 3; ++i) scale = std::fmax(scale, std::fmax(std::fabs(v0[i]), std::fabs(v1[i])));
    if (scale == 0.0f) scale = 1.0f;
    float a[2][3];
    for (int i = 0; i < 3; ++i) {
        a[0][i] = v0[i] / scale;
        a[1][i] = v1[i] / scale;
    }
    const auto norm3 = [](const float* x) { return std::sqrt(x[0] * x[0] + (x[1] * x[1] + x[2] * x[2])); };
    if (norm3(a[1]) > norm3(a[0])) {
        for (int i = 0; i < 3; ++i) {
            const float t = a[0][i];
            a[0][i] = a[1][i];
            a[1][i] = t;
        }
    }
    float e0[2] = {0.0f, 0.0f}, tau0 = 0.0f;
    {
        const float c0 = a[0][0];
        const float tail = a[0][1] * a[0][1] + a[0][2] * a[0][2];
        if (tail > 1.17549435e-38f) {  // numeric_limits<float>::min()
            float beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0f) beta = -beta;
            e0[0] = a[0][1] / (c0 - beta);
            e0[1] = a[0][2] / (c0 - beta);
            tau0 = (beta - c0) / beta;
        }
    }
    float b[3] = {a[1][0], a[1][1], a[1][2]};
    if (tau0 != 0.0f) {
        float tmp = e0[0] * b[1] + e0[1] * b[2];
        tmp = tmp + b[0];
        b[0] = b[0] - tau0 * tmp;
        b[1] = b[1] - tmp * (tau0 * e0[0]);
        b[2] = b[2] - tmp * (tau0 * e0[1]);
    }
    float e1 = 0.0f, tau1 = 0.0f;
    {
        const float c0 = b[1];
        const float tail = b[2] * b[2];
        if (tail > 1.17549435e-38f) {
            float beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0f) beta = -beta;
            e1 = b[2] / (c0 - beta);
            tau1 = (beta - c0) / beta;
        }
    }
    float q[3] = {0.0f, 0.0f, 1.0f};
    if (tau1 != 0.0f) {
        float tmp = e1 * q[2];
        tmp = tmp + q[1];
        q[1] = q[1] - tau1 * tmp;
        q[2] = q[2] - tmp * (tau1 * e1);
    }
    if (tau0 != 0.0f) {
        float tmp = e0[0] * q[1] + e0[1] * q[2];
        tmp = tmp + q[0];
        q[0] = q[0] - tau0 * tmp;
        q[1] = q[1] - tmp * (tau0 * e0[0]);
        q[2] = q[2] - tmp * (tau0 * e0[1]);
    }
    return Vec3(q[0], q[1], q[2]);
}

// Eigen's setFromTwoVectors (dummy_precision<float> = 1e-5).
inline Quat Quat::FromTwoVectors(const Vec3& a, const Vec3& b) {
    const Vec3 v0 = a.normalized();
    const Vec3 v1 = b.normalized();
    float c = v1.dot(v0);
    if (c < -1.0f + 1e-5f) {
        c = std::fmax(c, -1.0f);
        const Vec3 axis = svd_null_axis(v0, v1);
        const float w2 = (1.0f + c) * 0.5f;
        const float s = std::sqrt(1.0f - w2);
        return Quat(std::sqrt(w2), axis[0] * s, axis[1] * s, axis[2] * s);
    }
    const Vec3 axis = v0.cross(v1);
    const float s = std::sqrt((1.0f + c) * 2.0f);
    const float invs = 1.0f / s;
    return Quat(s * 0.5f, axis[0] * invs, axis[1] * invs, axis[2] * invs);
}

// Pinhole camera, camera space x-right, y-down, z-forward (math.hpp:40-57).
struct Camera {
    Vec3 position = Vec3::Zero();
    Quat orientation = Quat::Identity();  // camera-to-world
    float fov_y_deg = 50.0f;
    int width = 1280;
    int height = 720;
    float near_m = 0.1f;

    static Camera look_at(const Vec3& eye, const Vec3& target, float fov_y_deg, int width,
                          int height, float near_m = 0.1f,
                          const Vec3& up = Vec3(0.0f, 1.0f, 0.0f));
    float focal_px() const;
    Mat3 view_rotation() const { return orientation.toRotationMatrix().transpose(); }
};

void validate(const Camera& cam);

struct PixelRect {
    int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
    bool empty() const { return x0 >= x1 || y0 >= y1; }
};

// Integer 3-sigma rectangle clipped to [0, w) x [0, h) (math.cpp:106-116); k_project
// computes the same rect per splat on the GPU.
inline PixelRect splat_bounds(const Vec2& mean_px, float cov_xx, float cov_yy, int width, int height) {
    const float rx = 3.0f * std::sqrt(cov_xx);
    const float ry = 3.0f * std::sqrt(cov_yy);
    PixelRect r;
    r.x0 = std::max(0, static_cast<int>(std::floor(mean_px.x() - rx)));
    r.y0 = std::max(0, static_cast<int>(std::floor(mean_px.y() - ry)));
    r.x1 = std::min(width, static_cast<int>(std::floor(mean_px.x() + rx)) + 1);
    r.y1 = std::min(height, static_cast<int>(std::floor(mean_px.y() + ry)) + 1);
    return r;
}

// Sigma = R S S^T R^T (math.cpp:94-104); used at template load (LodLevel::finalize).
Mat3 build_covariance(const Quat& rotation, const Vec3& scale);

}  // namespace gsc
