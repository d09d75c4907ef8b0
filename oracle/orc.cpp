// CPU ORACLE — test infrastructure only (see orc.h). A literal, Eigen-free restatement
// of the reference renderer's per-frame path. Build: oracle/Makefile
// (g++ -O2 -ffp-contract=off, no -march: x86-64 SSE2 without FMA, as the reference's
// Release build). Each function cites the reference lines it restates; paths are
// relative to /root/reference/proj.
#include "orc.h"

#include <algorithm>
#include <array>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

using M4 = std::array<float, 16>;  // column-major, element (r, c) at [c * 4 + r]
using M3 = std::array<float, 9>;   // column-major, element (r, c) at [c * 3 + r]
using V3 = std::array<float, 3>;
using Q4 = std::array<float, 4>;   // x, y, z, w

M4 ident4() {
    M4 m{};
    m[0] = m[5] = m[10] = m[15] = 1.0f;
    return m;
}

// Eigen lazy 4x4 product, SSE packet path: column c = ((A.c0*B(0,c) + A.c1*B(1,c)) +
// A.c2*B(2,c)) + A.c3*B(3,c), multiply and add rounded separately (no FMA).
M4 mul44(const M4& a, const M4& b) {
    M4 o{};
    for (int c = 0; c < 4; ++c) {
        for (int r = 0; r < 4; ++r) {
            float s = a[0 * 4 + r] * b[c * 4 + 0];
            s = s + a[1 * 4 + r] * b[c * 4 + 1];
            s = s + a[2 * 4 + r] * b[c * 4 + 2];
            s = s + a[3 * 4 + r] * b[c * 4 + 3];
            o[c * 4 + r] = s;
        }
    }
    return o;
}

// Eigen Quaternion::toRotationMatrix.
M3 quat_to_m3(const Q4& q) {
    const float x = q[0], y = q[1], z = q[2], w = q[3];
    const float tx = 2.0f * x, ty = 2.0f * y, tz = 2.0f * z;
    const float twx = tx * w, twy = ty * w, twz = tz * w;
    const float txx = tx * x, txy = ty * x, txz = tz * x;
    const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
    M3 m{};
    m[0 * 3 + 0] = 1.0f - (tyy + tzz);
    m[1 * 3 + 0] = txy - twz;
    m[2 * 3 + 0] = txz + twy;
    m[0 * 3 + 1] = txy + twz;
    m[1 * 3 + 1] = 1.0f - (txx + tzz);
    m[2 * 3 + 1] = tyz - twx;
    m[0 * 3 + 2] = txz - twy;
    m[1 * 3 + 2] = tyz + twx;
    m[2 * 3 + 2] = 1.0f - (txx + tyy);
    return m;
}

inline float at3(const M3& m, int r, int c) { return m[c * 3 + r]; }

// length-3 reductions (Eigen redux_novec_unroller): a0 + (a1 + a2)
inline float dot3(const V3& a, const V3& b) { return a[0] * b[0] + (a[1] * b[1] + a[2] * b[2]); }
inline float norm3(const V3& a) { return std::sqrt(dot3(a, a)); }
inline V3 sub3(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline V3 cross3(const V3& a, const V3& b) {
    return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline V3 normalized3(const V3& a) {
    const float n = norm3(a);
    return {a[0] / n, a[1] / n, a[2] / n};
}
// Quaternion dot / squaredNorm: SSE predux (c0 + c2) + (c1 + c3).
inline float qdot(const Q4& a, const Q4& b) {
    const float p0 = a[0] * b[0], p1 = a[1] * b[1], p2 = a[2] * b[2], p3 = a[3] * b[3];
    return (p0 + p2) + (p1 + p3);
}
inline Q4 qnormalized(const Q4& q) {
    const float z = qdot(q, q);
    if (!(z > 0.0f)) return q;
    const float n = std::sqrt(z);
    return {q[0] / n, q[1] / n, q[2] / n, q[3] / n};
}

// ---------------------------------------------------------------- camera (math.cpp)

struct Basis {
    float W[3][3];  // world -> view, row-major
    V3 pos;
    float focal, cx, cy, near_m;
    int width, height;
};

// Eigen Quaternion(Matrix3) (quaternion_assign_impl<3x3>).
Q4 quat_from_m3(const M3& m) {
    Q4 q{};
    float t = at3(m, 0, 0) + (at3(m, 1, 1) + at3(m, 2, 2));
    if (t > 0.0f) {
        t = std::sqrt(t + 1.0f);
        q[3] = 0.5f * t;
        t = 0.5f / t;
        q[0] = (at3(m, 2, 1) - at3(m, 1, 2)) * t;
        q[1] = (at3(m, 0, 2) - at3(m, 2, 0)) * t;
        q[2] = (at3(m, 1, 0) - at3(m, 0, 1)) * t;
    } else {
        int i = 0;
        if (at3(m, 1, 1) > at3(m, 0, 0)) i = 1;
        if (at3(m, 2, 2) > at3(m, i, i)) i = 2;
        const int j = (i + 1) % 3, k = (j + 1) % 3;
        t = std::sqrt(at3(m, i, i) - at3(m, j, j) - at3(m, k, k) + 1.0f);
        q[i] = 0.5f * t;
        t = 0.5f / t;
        q[3] = (at3(m, k, j) - at3(m, j, k)) * t;
        q[j] = (at3(m, j, i) + at3(m, i, j)) * t;
        q[k] = (at3(m, k, i) + at3(m, i, k)) * t;
    }
    return q;
}

// Camera::look_at (math.cpp:42-64) + view_rotation (:71-73) + focal_px (:66-69) +
// CameraBasis::from (:118-129).
Basis make_basis(const V3& eye, const V3& target, float fov, int w, int h, float near_m, Q4* orient_out) {
    const V3 forward = normalized3(sub3(target, eye));
    V3 axis{0.0f, 1.0f, 0.0f};
    {
        const V3 c = cross3(forward, axis);
        if (dot3(c, c) < 1e-12f) axis = {0.0f, 0.0f, 1.0f};
    }
    const V3 right = normalized3(cross3(forward, axis));
    const V3 down = cross3(forward, right);
    M3 bm{};
    for (int r = 0; r < 3; ++r) {
        bm[0 * 3 + r] = right[r];
        bm[1 * 3 + r] = down[r];
        bm[2 * 3 + r] = forward[r];
    }
    const Q4 orient = qnormalized(quat_from_m3(bm));
    if (orient_out) *orient_out = orient;
    const M3 R = quat_to_m3(orient);
    Basis b{};
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) b.W[r][c] = at3(R, c, r);  // transpose
    b.pos = eye;
    const float half_fov = 0.5f * fov * (3.14159265358979323846f / 180.0f);
    b.focal = 0.5f * static_cast<float>(h) / std::tan(half_fov);
    b.cx = 0.5f * static_cast<float>(w);
    b.cy = 0.5f * static_cast<float>(h);
    b.near_m = near_m;
    b.width = w;
    b.height = h;
    return b;
}

// build_covariance (math.cpp:94-104): M = R diag(s); Sigma = M M^T.
M3 covariance(const Q4& q, const V3& s) {
    const M3 R = quat_to_m3(q);
    M3 M{};
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) M[c * 3 + r] = at3(R, r, c) * s[c];
    M3 S{};
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r)
            S[c * 3 + r] = at3(M, r, 0) * at3(M, c, 0) + (at3(M, r, 1) * at3(M, c, 1) + at3(M, r, 2) * at3(M, c, 2));
    return S;
}

struct Rect {
    int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
    bool empty() const { return x0 >= x1 || y0 >= y1; }
};

// splat_bounds (math.cpp:106-116).
Rect bounds(float mx, float my, float cxx, float cyy, int w, int h) {
    const float rx = 3.0f * std::sqrt(cxx);
    const float ry = 3.0f * std::sqrt(cyy);
    Rect r;
    r.x0 = std::max(0, static_cast<int>(std::floor(mx - rx)));
    r.y0 = std::max(0, static_cast<int>(std::floor(my - ry)));
    r.x1 = std::min(w, static_cast<int>(std::floor(mx + rx)) + 1);
    r.y1 = std::min(h, static_cast<int>(std::floor(my + ry)) + 1);
    return r;
}

bool finite3(const V3& v) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }

// project_covariance (math.cpp:131-170).
bool project(const V3& mean, const M3& cov, const V3& color, float opacity, const Basis& b, orc_splat& out) {
    if (!finite3(mean)) return false;
    for (float v : cov)
        if (!std::isfinite(v)) return false;
    const V3 d = sub3(mean, b.pos);
    float t[3];
    for (int i = 0; i < 3; ++i) t[i] = b.W[i][0] * d[0] + (b.W[i][1] * d[1] + b.W[i][2] * d[2]);
    if (!(t[2] > b.near_m)) return false;
    const float f = b.focal;
    const float inv_z = 1.0f / t[2];
    const float mx = f * t[0] * inv_z + b.cx;
    const float my = f * t[1] * inv_z + b.cy;
    const float J[2][3] = {{f * inv_z, 0.0f, -f * t[0] * inv_z * inv_z},
                           {0.0f, f * inv_z, -f * t[1] * inv_z * inv_z}};
    float m[2][3];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) m[r][c] = J[r][0] * b.W[0][c] + (J[r][1] * b.W[1][c] + J[r][2] * b.W[2][c]);
    float A[2][3];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            A[r][c] = m[r][0] * at3(cov, 0, c) + (m[r][1] * at3(cov, 1, c) + m[r][2] * at3(cov, 2, c));
    float C[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) C[i][j] = A[i][0] * m[j][0] + (A[i][1] * m[j][1] + A[i][2] * m[j][2]);
    C[0][0] += 0.3f;
    C[1][1] += 0.3f;
    const Rect rc = bounds(mx, my, C[0][0], C[1][1], b.width, b.height);
    if (rc.empty()) return false;
    out.mean_px[0] = mx;
    out.mean_px[1] = my;
    out.cov_xx = C[0][0];
    out.cov_xy = 0.5f * (C[0][1] + C[1][0]);
    out.cov_yy = C[1][1];
    out.depth = t[2];
    out.color[0] = color[0];
    out.color[1] = color[1];
    out.color[2] = color[2];
    out.opacity = opacity;
    return true;
}

// SH residual extension, same basis and summation order as the GPU.
void sh_colour(const V3& posed, const V3& cam, const float* sh, float* col) {
    const float vx = posed[0] - cam[0], vy = posed[1] - cam[1], vz = posed[2] - cam[2];
    const float nrm = std::sqrt(vx * vx + (vy * vy + vz * vz));
    const float x = vx / nrm, y = vy / nrm, z = vz / nrm;
    const float C1 = 0.4886025119029199f;
    const float C20 = 1.0925484305920792f, C21 = -1.0925484305920792f, C22 = 0.31539156525252005f,
                C23 = -1.0925484305920792f, C24 = 0.5462742152960396f;
    const float C30 = -0.5900435899266435f, C31 = 2.890611442640554f, C32 = -0.4570457994644658f,
                C33 = 0.3731763325901154f, C34 = -0.4570457994644658f, C35 = 1.445305721320277f,
                C36 = -0.5900435899266435f;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    float Y[15];
    Y[0] = -C1 * y;
    Y[1] = C1 * z;
    Y[2] = -C1 * x;
    Y[3] = C20 * xy;
    Y[4] = C21 * yz;
    Y[5] = C22 * ((2.0f * zz - xx) - yy);
    Y[6] = C23 * xz;
    Y[7] = C24 * (xx - yy);
    Y[8] = (C30 * y) * (3.0f * xx - yy);
    Y[9] = (C31 * xy) * z;
    Y[10] = (C32 * y) * ((4.0f * zz - xx) - yy);
    Y[11] = (C33 * z) * ((2.0f * zz - 3.0f * xx) - 3.0f * yy);
    Y[12] = (C34 * x) * ((4.0f * zz - xx) - yy);
    Y[13] = (C35 * z) * (xx - yy);
    Y[14] = (C36 * x) * (xx - 3.0f * yy);
    for (int c = 0; c < 3; ++c) {
        float v = col[c];
        for (int k = 0; k < 15; ++k) v = v + Y[k] * sh[3 * k + c];
        col[c] = std::fmax(v, 0.0f);
    }
}

// ------------------------------------------------------------- threads (parallel.hpp)

unsigned thread_count(int hint) {
    if (hint > 0) return static_cast<unsigned>(hint);
    if (const char* env = std::getenv("GSCROWD_THREADS")) {
        const long v = std::strtol(env, nullptr, 10);
        if (v > 0) return static_cast<unsigned>(v);
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw > 0 ? hw : 1;
}

template <typename Fn>
void for_ranges(size_t count, int hint, Fn&& fn) {
    const unsigned threads = static_cast<unsigned>(std::min<size_t>(thread_count(hint), count));
    if (threads <= 1) {
        if (count > 0) fn(size_t{0}, count);
        return;
    }
    std::vector<std::thread> pool;
    const size_t chunk = (count + threads - 1) / threads;
    for (unsigned w = 0; w < threads; ++w) {
        const size_t b = w * chunk, e = std::min(count, b + chunk);
        if (b >= e) break;
        pool.emplace_back([b, e, &fn] { fn(b, e); });
    }
    for (auto& t : pool) t.join();
}

// ------------------------------------------------------------------ scene model

struct Level {
    uint32_t n = 0;
    std::vector<V3> means, scales, colors;
    std::vector<Q4> rot;
    std::vector<float> opacity;
    std::vector<std::array<uint16_t, 4>> idx;
    std::vector<std::array<float, 4>> w;
    std::vector<float> sh;
    std::vector<std::array<float, 6>> cov;  // finalize (avatar.cpp:99-105)
};

struct Template {
    uint32_t J = 0;
    std::vector<int16_t> parents;
    std::vector<M4> inverse_bind, bind, local_bind;
    std::vector<Level> levels;
};

struct Motion {
    float fps = 30.0f;
    uint32_t frames = 0, joints = 0;
    std::vector<float> data;  // frames x (4 + 4J)
};

// Skeleton::make (avatar.cpp:40-72) with rigid_inverse (:10-17).
void derive_skeleton(Template& t) {
    t.bind.resize(t.J);
    t.local_bind.resize(t.J);
    for (uint32_t j = 0; j < t.J; ++j) {
        const M4& ib = t.inverse_bind[j];
        M4 b = ident4();
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) b[c * 4 + r] = ib[r * 4 + c];  // R^T
        const float tt[3] = {ib[12], ib[13], ib[14]};
        for (int r = 0; r < 3; ++r) {
            // (R^T t)_r = R^T(r,0) t0 + (R^T(r,1) t1 + R^T(r,2) t2), then negated
            const float v = b[0 * 4 + r] * tt[0] + (b[1 * 4 + r] * tt[1] + b[2 * 4 + r] * tt[2]);
            b[12 + r] = -v;
        }
        t.bind[j] = b;
        t.local_bind[j] = t.parents[j] < 0 ? b : mul44(t.inverse_bind[t.parents[j]], b);
    }
}

// slerp_shortest (avatar.cpp:226-245).
Q4 slerp(const Q4& a, const Q4& b, float t) {
    float d = qdot(a, b);
    Q4 bf = b;
    if (d < 0.0f) {
        d = -d;
        for (float& v : bf) v = -v;
    }
    Q4 o{};
    if (d > 0.9995f) {
        for (int i = 0; i < 4; ++i) o[i] = a[i] + t * (bf[i] - a[i]);
    } else {
        const float theta = std::acos(std::min(d, 1.0f));
        const float s = std::sin(theta);
        const float wa = std::sin((1.0f - t) * theta) / s;
        const float wb = std::sin(t * theta) / s;
        for (int i = 0; i < 4; ++i) o[i] = wa * a[i] + wb * bf[i];
    }
    return qnormalized(o);
}

// sample_pose (avatar.cpp:247-283) into a (4 + 4J) record.
void sample(const float* clip, uint32_t frames, uint32_t J, float fps, float time_s, bool wrap, float* out) {
    const size_t n = frames;
    float fpos = time_s * fps;
    size_t i0, i1;
    float t;
    if (wrap) {
        fpos = std::fmod(fpos, static_cast<float>(n));
        if (fpos < 0.0f) fpos += static_cast<float>(n);
        i0 = static_cast<size_t>(fpos) % n;
        i1 = (i0 + 1) % n;
        t = fpos - std::floor(fpos);
    } else {
        if (fpos <= 0.0f) fpos = 0.0f;
        const float last = static_cast<float>(n - 1);
        if (fpos >= last) {
            i0 = i1 = n - 1;
            t = 0.0f;
        } else {
            i0 = static_cast<size_t>(fpos);
            i1 = i0 + 1;
            t = fpos - static_cast<float>(i0);
        }
    }
    const size_t rec = 4 + 4 * static_cast<size_t>(J);
    const float* a = clip + i0 * rec;
    const float* b = clip + i1 * rec;
    for (int k = 0; k < 3; ++k) out[k] = (1.0f - t) * a[k] + t * b[k];
    out[3] = 0.0f;
    for (uint32_t j = 0; j < J; ++j) {
        const Q4 qa{a[4 + 4 * j], a[5 + 4 * j], a[6 + 4 * j], a[7 + 4 * j]};
        const Q4 qb{b[4 + 4 * j], b[5 + 4 * j], b[6 + 4 * j], b[7 + 4 * j]};
        const Q4 q = slerp(qa, qb, t);
        for (int k = 0; k < 4; ++k) out[4 + 4 * j + k] = q[k];
    }
}

// forward_kinematics (avatar.cpp:149-164).
void fk(const Template& tp, const float* pose, const M4& root, std::vector<M4>& world) {
    world.resize(tp.J);
    M4 off = ident4();
    off[12] = pose[0];
    off[13] = pose[1];
    off[14] = pose[2];
    const M4 root_off = mul44(root, off);
    for (uint32_t j = 0; j < tp.J; ++j) {
        const Q4 q{pose[4 + 4 * j], pose[5 + 4 * j], pose[6 + 4 * j], pose[7 + 4 * j]};
        const M3 r3 = quat_to_m3(q);
        M4 rot = ident4();
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) rot[c * 4 + r] = at3(r3, r, c);
        const M4 local = mul44(tp.local_bind[j], rot);
        world[j] = j == 0 ? mul44(root_off, local) : mul44(world[tp.parents[j]], local);
    }
}

// skin_means (avatar.cpp:178-192) given world transforms; skin = world * inverse_bind.
void skin(const Template& tp, const Level& lv, const std::vector<M4>& world, V3* out) {
    std::vector<M4> S(tp.J);
    for (uint32_t j = 0; j < tp.J; ++j) S[j] = mul44(world[j], tp.inverse_bind[j]);
    for (uint32_t i = 0; i < lv.n; ++i) {
        const float p[4] = {lv.means[i][0], lv.means[i][1], lv.means[i][2], 1.0f};
        float acc[3] = {0.0f, 0.0f, 0.0f};
        for (int k = 0; k < 4; ++k) {
            const float wk = lv.w[i][k];
            if (wk == 0.0f) continue;
            const M4& m = S[lv.idx[i][k]];
            for (int r = 0; r < 3; ++r) {
                float v = m[0 * 4 + r] * p[0];
                v = v + m[1 * 4 + r] * p[1];
                v = v + m[2 * 4 + r] * p[2];
                v = v + m[3 * 4 + r] * p[3];
                acc[r] = acc[r] + wk * v;
            }
        }
        out[i] = {acc[0], acc[1], acc[2]};
    }
}

// CrowdInstance::root_transform (crowd.cpp:20-30).
M4 root_of(const orc_instance& in) {
    M4 m = ident4();
    const float c = std::cos(in.yaw), s = std::sin(in.yaw);
    m[0 * 4 + 0] = c;
    m[2 * 4 + 0] = s;
    m[0 * 4 + 2] = -s;
    m[2 * 4 + 2] = c;
    m[3 * 4 + 0] = in.x;
    m[3 * 4 + 2] = in.z;
    return m;
}

uint32_t lod_select(const std::vector<float>& th, float band, float dist, bool has_prev, uint32_t prev) {
    for (size_t k = 0; k < th.size(); ++k) {
        float t = th[k];
        if (has_prev && band > 0.0f) t += (k >= prev ? 0.5f : -0.5f) * band;
        if (dist < t) return static_cast<uint32_t>(k);
    }
    return static_cast<uint32_t>(th.size());
}

// Bin + blend (renderer.cpp:121-232): conic prep, tile bins in sorted order, per-tile
// splat-major blend with live-pixel early exit.
void raster(const std::vector<orc_splat>& sp, const orc_settings& st, int W, int H, int threads,
            float* rgb_out, float* T_out, std::vector<std::vector<uint32_t>>* bins_out) {
    struct Prep { float a, b, c, pf; };
    std::vector<Prep> prep(sp.size());
    for (size_t i = 0; i < sp.size(); ++i) {
        const orc_splat& s = sp[i];
        const float det = s.cov_xx * s.cov_yy - s.cov_xy * s.cov_xy;
        const float inv_det = 1.0f / det;
        prep[i] = {s.cov_yy * inv_det, -s.cov_xy * inv_det, s.cov_xx * inv_det,
                   std::log(st.alpha_cutoff / s.opacity)};
    }
    const int ts = st.tile_size;
    const int tiles_x = (W + ts - 1) / ts, tiles_y = (H + ts - 1) / ts;
    std::vector<std::vector<uint32_t>> local_bins;
    std::vector<std::vector<uint32_t>>& bins = bins_out ? *bins_out : local_bins;
    bins.assign(static_cast<size_t>(tiles_x) * tiles_y, {});
    for (size_t i = 0; i < sp.size(); ++i) {
        const int* r = sp[i].rect;
        if (r[0] >= r[2] || r[1] >= r[3]) continue;
        const int tx0 = r[0] / ts, tx1 = (r[2] - 1) / ts, ty0 = r[1] / ts, ty1 = (r[3] - 1) / ts;
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) bins[static_cast<size_t>(ty) * tiles_x + tx].push_back(static_cast<uint32_t>(i));
    }
    for_ranges(bins.size(), threads, [&](size_t tb, size_t te) {
        std::vector<float> tbuf(static_cast<size_t>(ts) * ts), cbuf(static_cast<size_t>(ts) * ts * 3);
        for (size_t tile = tb; tile < te; ++tile) {
            const int tx = static_cast<int>(tile) % tiles_x, ty = static_cast<int>(tile) / tiles_x;
            const int px0 = tx * ts, px1 = std::min(W, px0 + ts), py0 = ty * ts, py1 = std::min(H, py0 + ts);
            const int tw = px1 - px0, th = py1 - py0;
            std::fill(tbuf.begin(), tbuf.begin() + tw * th, 1.0f);
            std::fill(cbuf.begin(), cbuf.begin() + tw * th * 3, 0.0f);
            int live = tw * th;
            for (uint32_t idx : bins[tile]) {
                if (live == 0) break;
                const orc_splat& s = sp[idx];
                const Prep& co = prep[idx];
                const int sx0 = std::max(px0, s.rect[0]), sx1 = std::min(px1, s.rect[2]);
                const int sy0 = std::max(py0, s.rect[1]), sy1 = std::min(py1, s.rect[3]);
                for (int py = sy0; py < sy1; ++py) {
                    const size_t row = static_cast<size_t>(py - py0) * tw;
                    for (int px = sx0; px < sx1; ++px) {
                        float& t = tbuf[row + (px - px0)];
                        if (t < st.transmittance_floor) continue;
                        const float dx = (static_cast<float>(px) + 0.5f) - s.mean_px[0];
                        const float dy = (static_cast<float>(py) + 0.5f) - s.mean_px[1];
                        const float power = -0.5f * (co.a * dx * dx + co.c * dy * dy) - co.b * dx * dy;
                        if (power < co.pf) continue;
                        float alpha = s.opacity * std::exp(power);
                        if (alpha > st.alpha_max) alpha = st.alpha_max;
                        const float wgt = t * alpha;
                        float* c = &cbuf[(row + (px - px0)) * 3];
                        c[0] += wgt * s.color[0];
                        c[1] += wgt * s.color[1];
                        c[2] += wgt * s.color[2];
                        t *= 1.0f - alpha;
                        if (t < st.transmittance_floor) --live;
                    }
                }
            }
            for (int py = py0; py < py1; ++py) {
                const size_t row = static_cast<size_t>(py - py0) * tw;
                for (int px = px0; px < px1; ++px) {
                    const float t = tbuf[row + (px - px0)];
                    const float* c = &cbuf[(row + (px - px0)) * 3];
                    const size_t o = static_cast<size_t>(py) * W + px;
                    rgb_out[3 * o + 0] = c[0] + t * st.background[0];
                    rgb_out[3 * o + 1] = c[1] + t * st.background[1];
                    rgb_out[3 * o + 2] = c[2] + t * st.background[2];
                    T_out[o] = t;
                }
            }
        }
    });
}

// sort_splats_impl (renderer.cpp:85-107).
void sort_frame(std::vector<orc_splat>& sp) {
    struct Key { uint64_t p, s; };
    std::vector<Key> keys(sp.size());
    for (size_t i = 0; i < sp.size(); ++i) {
        keys[i].p = (static_cast<uint64_t>(std::bit_cast<uint32_t>(sp[i].depth)) << 32) | sp[i].instance_id;
        keys[i].s = (static_cast<uint64_t>(sp[i].gaussian_index) << 32) | static_cast<uint32_t>(i);
    }
    std::sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
        if (a.p != b.p) return a.p < b.p;
        return a.s < b.s;
    });
    std::vector<orc_splat> tmp(sp.size());
    for (size_t i = 0; i < sp.size(); ++i) tmp[i] = sp[static_cast<uint32_t>(keys[i].s)];
    sp.swap(tmp);
}

}  // namespace

struct orc_scene {
    std::vector<Template> templates;
    std::vector<Motion> motions;
    std::vector<orc_instance> inst;
    std::vector<float> lod_th{5.0f, 10.0f};
    float band = 0.0f;
    Basis basis{};
    bool has_camera = false;
    // last frame
    std::vector<uint32_t> lods;
    std::vector<std::vector<V3>> posed;
    std::vector<orc_splat> splats;
    std::vector<std::vector<uint32_t>> bins;
};

namespace {

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

orc_scene* orc_scene_new(void) { return new orc_scene(); }
void orc_scene_free(orc_scene* s) { delete s; }

int orc_add_template(orc_scene* s, uint32_t J, const int16_t* parents, const float* ib) {
    return guard([&] {
        Template t;
        t.J = J;
        t.parents.assign(parents, parents + J);
        t.inverse_bind.resize(J);
        for (uint32_t j = 0; j < J; ++j) std::memcpy(t.inverse_bind[j].data(), ib + 16 * j, 64);
        derive_skeleton(t);
        s->templates.push_back(std::move(t));
    });
}

int orc_add_level(orc_scene* s, uint32_t tid, uint32_t n, const float* means, const float* rot,
                  const float* scales, const float* op, const float* col, const uint16_t* idx,
                  const float* w, const float* sh) {
    return guard([&] {
        if (tid >= s->templates.size()) throw std::invalid_argument("no such template");
        Level lv;
        lv.n = n;
        lv.means.resize(n);
        lv.scales.resize(n);
        lv.colors.resize(n);
        lv.rot.resize(n);
        lv.opacity.assign(op, op + n);
        lv.idx.resize(n);
        lv.w.resize(n);
        lv.cov.resize(n);
        for (uint32_t i = 0; i < n; ++i) {
            lv.means[i] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
            lv.scales[i] = {scales[3 * i], scales[3 * i + 1], scales[3 * i + 2]};
            lv.colors[i] = {col[3 * i], col[3 * i + 1], col[3 * i + 2]};
            lv.rot[i] = {rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]};
            for (int k = 0; k < 4; ++k) {
                lv.idx[i][k] = idx[4 * i + k];
                lv.w[i][k] = w[4 * i + k];
            }
            const M3 c = covariance(lv.rot[i], lv.scales[i]);
            lv.cov[i] = {at3(c, 0, 0), at3(c, 0, 1), at3(c, 0, 2), at3(c, 1, 1), at3(c, 1, 2), at3(c, 2, 2)};
        }
        if (sh) lv.sh.assign(sh, sh + static_cast<size_t>(n) * 45);
        s->templates[tid].levels.push_back(std::move(lv));
    });
}

int orc_add_motion(orc_scene* s, float fps, uint32_t frames, uint32_t joints, const float* data) {
    return guard([&] {
        Motion m;
        m.fps = fps;
        m.frames = frames;
        m.joints = joints;
        m.data.assign(data, data + static_cast<size_t>(frames) * (4 + 4 * joints));
        s->motions.push_back(std::move(m));
    });
}

int orc_set_instances(orc_scene* s, uint32_t n, const orc_instance* in) {
    return guard([&] { s->inst.assign(in, in + n); });
}

int orc_get_instances(orc_scene* s, uint32_t n, orc_instance* out) {
    return guard([&] {
        if (n > s->inst.size()) throw std::invalid_argument("too many instances");
        std::copy(s->inst.begin(), s->inst.begin() + n, out);
    });
}

int orc_set_camera(orc_scene* s, const float* eye, const float* target, float fov, int32_t w, int32_t h,
                   float near_m) {
    return guard([&] {
        s->basis = make_basis({eye[0], eye[1], eye[2]}, {target[0], target[1], target[2]}, fov, w, h, near_m, nullptr);
        s->has_camera = true;
    });
}

int orc_set_lod(orc_scene* s, const float* th, uint32_t n, float band) {
    return guard([&] {
        s->lod_th.assign(th, th + n);
        s->band = band;
    });
}

int orc_render(orc_scene* s, float time_s, int32_t static_pose, int32_t forced_lod, const orc_settings* st,
               int32_t threads, float* out_rgb, float* out_T, orc_times* times) {
    return guard([&] {
        if (!s->has_camera) throw std::invalid_argument("camera not set");
        using clock = std::chrono::steady_clock;
        const auto ms = [](clock::time_point a, clock::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        const size_t n = s->inst.size();
        s->lods.assign(n, 0);
        s->posed.resize(n);
        const Basis& B = s->basis;

        // update_crowd (crowd.cpp:86-140)
        const auto t0 = clock::now();
        for_ranges(n, threads, [&](size_t b, size_t e) {
            std::vector<float> pose;
            std::vector<M4> world;
            for (size_t i = b; i < e; ++i) {
                orc_instance& in = s->inst[i];
                const Template& tp = s->templates[in.template_id];
                const uint32_t levels = static_cast<uint32_t>(tp.levels.size());
                uint32_t lod;
                if (forced_lod >= 0) {
                    lod = std::min(static_cast<uint32_t>(forced_lod), levels - 1);
                } else {
                    const V3 root{in.x, tp.bind[0][13], in.z};
                    const float dist = norm3(sub3(root, B.pos));
                    lod = std::min(lod_select(s->lod_th, s->band, dist, in.active_lod != 0xffffffffu, in.active_lod), levels - 1);
                }
                in.active_lod = lod;
                s->lods[i] = lod;
                const Level& lv = tp.levels[lod];
                pose.assign(4 + 4 * tp.J, 0.0f);
                if (static_pose) {
                    for (uint32_t j = 0; j < tp.J; ++j) pose[7 + 4 * j] = 1.0f;
                } else {
                    const Motion& m = s->motions[in.motion_id];
                    sample(m.data.data(), m.frames, m.joints, m.fps, time_s + in.phase_offset_s, true, pose.data());
                }
                fk(tp, pose.data(), root_of(in), world);
                s->posed[i].resize(lv.n);
                skin(tp, lv, world, s->posed[i].data());
            }
        });

        // gather_splats (renderer.cpp:25-73)
        const auto t1 = clock::now();
        std::vector<std::vector<orc_splat>> locals(n);
        for_ranges(n, threads, [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) {
                const orc_instance& in = s->inst[i];
                const Template& tp = s->templates[in.template_id];
                const Level& lv = tp.levels[s->lods[i]];
                auto& out = locals[i];
                out.clear();
                for (uint32_t g = 0; g < lv.n; ++g) {
                    const auto& c = lv.cov[g];
                    const M3 cov{c[0], c[1], c[2], c[1], c[3], c[4], c[2], c[4], c[5]};
                    orc_splat sp{};
                    if (!project(s->posed[i][g], cov, lv.colors[g], lv.opacity[g], B, sp)) continue;
                    if (st->sh_colour && !lv.sh.empty()) sh_colour(s->posed[i][g], B.pos, &lv.sh[45ull * g], sp.color);
                    sp.instance_id = in.instance_id;
                    sp.gaussian_index = g;
                    const Rect r = bounds(sp.mean_px[0], sp.mean_px[1], sp.cov_xx, sp.cov_yy, B.width, B.height);
                    sp.rect[0] = r.x0;
                    sp.rect[1] = r.y0;
                    sp.rect[2] = r.x1;
                    sp.rect[3] = r.y1;
                    out.push_back(sp);
                }
            }
        });
        s->splats.clear();
        size_t total = 0;
        for (auto& v : locals) total += v.size();
        s->splats.reserve(total);
        for (auto& v : locals) s->splats.insert(s->splats.end(), v.begin(), v.end());

        // sort_splats (renderer.cpp:85-107)
        const auto t2 = clock::now();
        sort_frame(s->splats);
        const auto t3 = clock::now();
        raster(s->splats, *st, B.width, B.height, threads, out_rgb, out_T, &s->bins);
        const auto t4 = clock::now();
        if (times) {
            times->update_ms = ms(t0, t1);
            times->gather_ms = ms(t1, t2);
            times->sort_ms = ms(t2, t3);
            times->rasterize_ms = ms(t3, t4);
            times->splat_count = s->splats.size();
            uint64_t K = 0, G = 0;
            for (auto& b : s->bins) K += b.size();
            for (auto& p : s->posed) G += p.size();
            times->pair_count = K;
            times->gaussian_count = G;
        }
    });
}

int orc_get_lods(orc_scene* s, uint32_t* out) {
    std::copy(s->lods.begin(), s->lods.end(), out);
    return 0;
}

uint64_t orc_gaussian_count(orc_scene* s) {
    uint64_t g = 0;
    for (auto& p : s->posed) g += p.size();
    return g;
}

int orc_get_posed(orc_scene* s, float* out) {
    size_t o = 0;
    for (auto& p : s->posed)
        for (auto& v : p) {
            out[o++] = v[0];
            out[o++] = v[1];
            out[o++] = v[2];
        }
    return 0;
}

uint64_t orc_splat_count(orc_scene* s) { return s->splats.size(); }

int orc_get_splats(orc_scene* s, orc_splat* out) {
    std::copy(s->splats.begin(), s->splats.end(), out);
    return 0;
}

uint64_t orc_pair_count(orc_scene* s) {
    uint64_t k = 0;
    for (auto& b : s->bins) k += b.size();
    return k;
}

int orc_get_bins(orc_scene* s, uint32_t* counts, uint32_t* items) {
    size_t o = 0;
    for (size_t t = 0; t < s->bins.size(); ++t) {
        counts[t] = static_cast<uint32_t>(s->bins[t].size());
        for (uint32_t v : s->bins[t]) items[o++] = v;
    }
    return 0;
}

int orc_get_level_cov(orc_scene* s, uint32_t t, uint32_t l, float* out) {
    return guard([&] {
        const Level& lv = s->templates.at(t).levels.at(l);
        for (uint32_t i = 0; i < lv.n; ++i) std::memcpy(out + 6 * i, lv.cov[i].data(), 24);
    });
}

int orc_build_covariance(const float* q, const float* sc, float* out9) {
    const M3 c = covariance({q[0], q[1], q[2], q[3]}, {sc[0], sc[1], sc[2]});
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) out9[r * 3 + k] = at3(c, r, k);
    return 0;
}

int orc_camera(const float* eye, const float* target, float fov, int32_t w, int32_t h, float near_m,
               float* w9, float* focal, float* quat) {
    Q4 q{};
    const Basis b = make_basis({eye[0], eye[1], eye[2]}, {target[0], target[1], target[2]}, fov, w, h, near_m, &q);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) w9[r * 3 + c] = b.W[r][c];
    if (focal) *focal = b.focal;
    if (quat) std::memcpy(quat, q.data(), 16);
    return 0;
}

int orc_project(const float* mean, const float* cov9, const float* color, float opacity, const float* eye,
                const float* target, float fov, int32_t w, int32_t h, float near_m, orc_splat* out) {
    const Basis b = make_basis({eye[0], eye[1], eye[2]}, {target[0], target[1], target[2]}, fov, w, h, near_m, nullptr);
    M3 cov{};
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) cov[c * 3 + r] = cov9[r * 3 + c];
    orc_splat sp{};
    if (!project({mean[0], mean[1], mean[2]}, cov, {color[0], color[1], color[2]}, opacity, b, sp)) return 0;
    const Rect r = bounds(sp.mean_px[0], sp.mean_px[1], sp.cov_xx, sp.cov_yy, w, h);
    sp.rect[0] = r.x0;
    sp.rect[1] = r.y0;
    sp.rect[2] = r.x1;
    sp.rect[3] = r.y1;
    *out = sp;
    return 1;
}

uint32_t orc_select_lod(const float* th, uint32_t n, float band, float dist, int64_t prev) {
    return lod_select(std::vector<float>(th, th + n), band, dist, prev >= 0, static_cast<uint32_t>(prev < 0 ? 0 : prev));
}

int orc_sort_splats(orc_splat* sp, uint32_t n) {
    std::vector<orc_splat> v(sp, sp + n);
    sort_frame(v);
    std::copy(v.begin(), v.end(), sp);
    return 0;
}

int orc_rasterize(const orc_splat* sp, uint32_t n, int32_t w, int32_t h, const orc_settings* st, int32_t threads,
                  float* rgb, float* T) {
    return guard([&] { raster(std::vector<orc_splat>(sp, sp + n), *st, w, h, threads, rgb, T, nullptr); });
}

// naive_rasterize (tests/oracles.hpp:179-223): every splat per pixel, no tiles.
int orc_naive_rasterize(const orc_splat* sp, uint32_t n, int32_t W, int32_t H, const orc_settings* st, float* rgb,
                        float* T) {
    for (int py = 0; py < H; ++py) {
        for (int px = 0; px < W; ++px) {
            float t = 1.0f, r = 0.0f, g = 0.0f, b = 0.0f;
            for (uint32_t i = 0; i < n; ++i) {
                const orc_splat& s = sp[i];
                if (px < s.rect[0] || px >= s.rect[2] || py < s.rect[1] || py >= s.rect[3]) continue;
                const float det = s.cov_xx * s.cov_yy - s.cov_xy * s.cov_xy;
                const float inv_det = 1.0f / det;
                const float ca = s.cov_yy * inv_det, cb = -s.cov_xy * inv_det, cc = s.cov_xx * inv_det;
                const float pf = std::log(st->alpha_cutoff / s.opacity);
                const float dx = (static_cast<float>(px) + 0.5f) - s.mean_px[0];
                const float dy = (static_cast<float>(py) + 0.5f) - s.mean_px[1];
                const float power = -0.5f * (ca * dx * dx + cc * dy * dy) - cb * dx * dy;
                if (power < pf) continue;
                float alpha = s.opacity * std::exp(power);
                if (alpha > st->alpha_max) alpha = st->alpha_max;
                const float wgt = t * alpha;
                r += wgt * s.color[0];
                g += wgt * s.color[1];
                b += wgt * s.color[2];
                t *= 1.0f - alpha;
                if (t < st->transmittance_floor) break;
            }
            const size_t o = static_cast<size_t>(py) * W + px;
            rgb[3 * o + 0] = r + t * st->background[0];
            rgb[3 * o + 1] = g + t * st->background[1];
            rgb[3 * o + 2] = b + t * st->background[2];
            T[o] = t;
        }
    }
    return 0;
}

int orc_sample_pose(const float* clip, uint32_t frames, uint32_t joints, float fps, float time_s, int32_t wrap,
                    float* out) {
    if (frames == 0) {
        g_err = "sample_pose: empty clip";
        return -1;
    }
    sample(clip, frames, joints, fps, time_s, wrap != 0, out);
    return 0;
}

int orc_forward_kinematics(orc_scene* s, uint32_t tid, const float* pose, const float* root16, float* world_out) {
    return guard([&] {
        const Template& tp = s->templates.at(tid);
        M4 root;
        std::memcpy(root.data(), root16, 64);
        std::vector<M4> world;
        fk(tp, pose, root, world);
        for (uint32_t j = 0; j < tp.J; ++j) std::memcpy(world_out + 16 * j, world[j].data(), 64);
    });
}

int orc_skin_means(orc_scene* s, uint32_t tid, uint32_t level, const float* world16, float* posed_out) {
    return guard([&] {
        const Template& tp = s->templates.at(tid);
        const Level& lv = tp.levels.at(level);
        std::vector<M4> world(tp.J);
        for (uint32_t j = 0; j < tp.J; ++j) std::memcpy(world[j].data(), world16 + 16 * j, 64);
        std::vector<V3> out(lv.n);
        skin(tp, lv, world, out.data());
        for (uint32_t i = 0; i < lv.n; ++i) std::memcpy(posed_out + 3 * i, out[i].data(), 12);
    });
}

}  // extern "C"

extern "C" void orc_libm_sinf(const float* in, float* out, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) out[i] = std::sin(in[i]);
}

// The host libm's expf over consecutive float bit patterns [first_bits, first_bits + n):
// what the reference's raster calls (renderer.cpp:205); the checker for the device replica.
extern "C" void orc_libm_expf_range(uint32_t first_bits, uint64_t n, float* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t b = first_bits + static_cast<uint32_t>(i);
        float x;
        std::memcpy(&x, &b, 4);
        out[i] = std::exp(x);
    }
}
