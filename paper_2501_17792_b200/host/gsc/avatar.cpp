// Host-side skeleton / pose / template logic. Behaviour follows
// /root/reference/proj/src/avatar.cpp (Skeleton::make :40-72, finalize :99-105,
// validators :107-147, slerp_shortest :226-245, sample_pose :247-283) and
// /root/reference/proj/src/math.cpp (look_at :42-64, focal_px :66-69,
// build_covariance :94-104). Floating-point order per SURVEY.md Appendix A.
#include "gsc/avatar.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

namespace gsc {

namespace {

bool all_finite(const Vec3& v) {
    return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]);
}
bool all_finite(const Quat& q) {
    return std::isfinite(q.c[0]) && std::isfinite(q.c[1]) && std::isfinite(q.c[2]) &&
           std::isfinite(q.c[3]);
}

// Inverse of a rigid transform: [R^T | -(R^T t)].
Mat4 invert_rigid(const Mat4& m) {
    const Mat3 rt = m.topLeft3().transpose();
    const Vec3 t = m.translation();
    Mat4 out = Mat4::Identity();
    out.setTopLeft3(rt);
    out.setTranslation(-(rt * t));
    return out;
}

float det3(const Mat3& m) {
    return m(0, 0) * (m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2)) -
           m(1, 0) * (m(0, 1) * m(2, 2) - m(2, 1) * m(0, 2)) +
           m(2, 0) * (m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2));
}

void require_rigid(const Mat4& m, const char* what) {
    const Mat3 r = m.topLeft3();
    const Mat3 rrt = r * r.transpose();
    float err = 0.0f;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            err = std::max(err, std::fabs(rrt(i, j) - (i == j ? 1.0f : 0.0f)));
    if (err > 1e-4f) throw std::invalid_argument(std::string(what) + ": rotation not orthonormal");
    if (std::fabs(det3(r) - 1.0f) > 1e-4f)
        throw std::invalid_argument(std::string(what) + ": determinant not +1");
    if (m(3, 0) != 0.0f || m(3, 1) != 0.0f || m(3, 2) != 0.0f || m(3, 3) != 1.0f)
        throw std::invalid_argument(std::string(what) + ": bottom row not (0,0,0,1)");
}

}  // namespace

Camera Camera::look_at(const Vec3& eye, const Vec3& target, float fov_y_deg, int width,
                       int height, float near_m, const Vec3& up) {
    const Vec3 forward = (target - eye).normalized();
    Vec3 axis = up;
    if (forward.cross(axis).squaredNorm() < 1e-12f) axis = Vec3(0.0f, 0.0f, 1.0f);
    const Vec3 right = forward.cross(axis).normalized();
    const Vec3 down = forward.cross(right);
    Mat3 basis;
    for (int r = 0; r < 3; ++r) {
        basis(r, 0) = right[r];
        basis(r, 1) = down[r];
        basis(r, 2) = forward[r];
    }
    Camera cam;
    cam.position = eye;
    cam.orientation = Quat::FromRotationMatrix(basis).normalized();
    cam.fov_y_deg = fov_y_deg;
    cam.width = width;
    cam.height = height;
    cam.near_m = near_m;
    return cam;
}

float Camera::focal_px() const {
    const float half_fov = 0.5f * fov_y_deg * (3.14159265358979323846f / 180.0f);
    return 0.5f * static_cast<float>(height) / std::tan(half_fov);
}

void validate(const Camera& cam) {
    if (cam.width < 1 || cam.height < 1)
        throw std::invalid_argument("Camera: width and height must be >= 1");
    if (!(cam.near_m > 0.0f)) throw std::invalid_argument("Camera: near plane must be > 0");
    if (!(cam.fov_y_deg > 0.0f && cam.fov_y_deg < 180.0f))
        throw std::invalid_argument("Camera: fov_y outside (0,180)");
    if (!all_finite(cam.position) || !all_finite(cam.orientation))
        throw std::invalid_argument("Camera: non-finite pose");
}

Mat3 build_covariance(const Quat& rotation, const Vec3& scale) {
    if (!all_finite(rotation) || !all_finite(scale))
        throw std::invalid_argument("build_covariance: non-finite input");
    if (!(scale[0] > 0.0f && scale[1] > 0.0f && scale[2] > 0.0f))
        throw std::invalid_argument("build_covariance: scale components must be positive");
    const Mat3 r = rotation.toRotationMatrix();
    Mat3 m;
    for (int c = 0; c < 3; ++c)
        for (int rr = 0; rr < 3; ++rr) m(rr, c) = r(rr, c) * scale[c];
    return m * m.transpose();
}

Skeleton Skeleton::make(std::vector<int16_t> parents, std::vector<Mat4> inverse_bind) {
    if (parents.empty()) throw std::invalid_argument("Skeleton: no joints");
    if (parents.size() != inverse_bind.size())
        throw std::invalid_argument("Skeleton: parent/inverse_bind size mismatch");
    int roots = 0;
    for (size_t j = 0; j < parents.size(); ++j) {
        if (parents[j] < 0)
            ++roots;
        else if (static_cast<size_t>(parents[j]) >= j)
            throw std::invalid_argument("Skeleton: parent index must precede child");
    }
    if (roots != 1 || parents[0] >= 0)
        throw std::invalid_argument("Skeleton: exactly one root at index 0 required");
    Skeleton s;
    s.parents = std::move(parents);
    s.inverse_bind = std::move(inverse_bind);
    const size_t n = s.inverse_bind.size();
    s.bind.resize(n);
    s.local_bind.resize(n);
    for (size_t j = 0; j < n; ++j) {
        require_rigid(s.inverse_bind[j], "Skeleton inverse_bind");
        s.bind[j] = invert_rigid(s.inverse_bind[j]);
        s.local_bind[j] =
            s.parents[j] < 0 ? s.bind[j] : s.inverse_bind[s.parents[j]] * s.bind[j];
    }
    return s;
}

Pose bind_pose(uint32_t joint_count) {
    Pose p;
    p.local_rotations.assign(joint_count, Quat::Identity());
    return p;
}

void validate(const MotionClip& clip) {
    if (clip.frames.empty()) throw std::invalid_argument("MotionClip: no frames");
    if (!(clip.fps > 0.0f)) throw std::invalid_argument("MotionClip: fps must be > 0");
    for (const Pose& f : clip.frames) {
        if (f.local_rotations.size() != clip.joint_count)
            throw std::invalid_argument("MotionClip: frame joint count mismatch");
        for (const Quat& q : f.local_rotations)
            if (std::fabs(q.norm() - 1.0f) > 1e-5f)
                throw std::invalid_argument("MotionClip: rotation not normalized");
    }
}

void LodLevel::finalize() {
    cov_cache.resize(means.size());
    for (size_t i = 0; i < means.size(); ++i) {
        const Mat3 c = build_covariance(rotations[i], scales[i]);
        cov_cache[i] = {c(0, 0), c(0, 1), c(0, 2), c(1, 1), c(1, 2), c(2, 2)};
    }
}

void validate(const LodLevel& level, uint32_t joint_count) {
    const size_t n = level.means.size();
    if (n == 0) throw std::invalid_argument("LodLevel: empty");
    if (level.rotations.size() != n || level.scales.size() != n ||
        level.opacities.size() != n || level.colors.size() != n ||
        level.skin_indices.size() != n || level.skin_weights.size() != n)
        throw std::invalid_argument("LodLevel: attribute array length mismatch");
    if (!level.sh.empty() && level.sh.size() != n * kShFloats)
        throw std::invalid_argument("LodLevel: SH array length mismatch");
    for (size_t i = 0; i < n; ++i) {
        if (!all_finite(level.means[i]) || !all_finite(level.rotations[i]) ||
            !all_finite(level.scales[i]) || !std::isfinite(level.opacities[i]) ||
            !all_finite(level.colors[i]))
            throw std::invalid_argument("LodLevel: non-finite field");
        if (std::fabs(level.rotations[i].norm() - 1.0f) > 1e-6f)
            throw std::invalid_argument("LodLevel: rotation quaternion not normalized");
        const Vec3& s = level.scales[i];
        if (!(s[0] > 0.0f && s[1] > 0.0f && s[2] > 0.0f))
            throw std::invalid_argument("LodLevel: scale components must be positive");
        if (!(level.opacities[i] > 0.0f && level.opacities[i] <= 1.0f))
            throw std::invalid_argument("LodLevel: opacity outside (0,1]");
        for (int k = 0; k < 3; ++k)
            if (level.colors[i][k] < 0.0f || level.colors[i][k] > 1.0f)
                throw std::invalid_argument("LodLevel: color component outside [0,1]");
        float wsum = 0.0f;
        for (int k = 0; k < 4; ++k) {
            if (level.skin_indices[i][k] >= joint_count)
                throw std::invalid_argument("LodLevel: skin index out of range");
            if (level.skin_weights[i][k] < 0.0f)
                throw std::invalid_argument("LodLevel: negative skin weight");
            wsum += level.skin_weights[i][k];
        }
        if (std::fabs(wsum - 1.0f) > 1e-5f)
            throw std::invalid_argument("LodLevel: skin weights do not sum to 1");
    }
}

void validate(const AvatarTemplate& tpl) {
    if (tpl.levels.empty()) throw std::invalid_argument("AvatarTemplate: no LoD levels");
    for (size_t l = 0; l < tpl.levels.size(); ++l) {
        validate(tpl.levels[l], tpl.skeleton.joint_count());
        if (l > 0 && tpl.levels[l].gaussian_count() >= tpl.levels[l - 1].gaussian_count())
            throw std::invalid_argument("AvatarTemplate: level counts must strictly decrease");
    }
}

Quat slerp_shortest(const Quat& a, const Quat& b, float t) {
    float d = a.dot(b);
    Quat bf = b;
    if (d < 0.0f) {
        d = -d;
        for (float& v : bf.c) v = -v;
    }
    Quat out;
    if (d > 0.9995f) {
        for (int i = 0; i < 4; ++i) out.c[i] = a.c[i] + t * (bf.c[i] - a.c[i]);
    } else {
        const float theta = std::acos(std::min(d, 1.0f));
        const float s = std::sin(theta);
        const float wa = std::sin((1.0f - t) * theta) / s;
        const float wb = std::sin(t * theta) / s;
        for (int i = 0; i < 4; ++i) out.c[i] = wa * a.c[i] + wb * bf.c[i];
    }
    out.normalize();
    return out;
}

namespace {

// Frame pair + blend weight for a clip time (avatar.cpp:253-276).
void locate(const MotionClip& clip, float time_s, bool wrap, size_t& i0, size_t& i1, float& t) {
    if (clip.frames.empty()) throw std::invalid_argument("sample_pose: empty clip");
    const size_t n = clip.frames.size();
    float fpos = time_s * clip.fps;
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
}

}  // namespace

Pose sample_pose(const MotionClip& clip, float time_s, bool wrap) {
    size_t i0, i1;
    float t;
    locate(clip, time_s, wrap, i0, i1, t);
    const Pose& a = clip.frames[i0];
    const Pose& b = clip.frames[i1];
    Pose out;
    out.root_translation = (1.0f - t) * a.root_translation + t * b.root_translation;
    out.local_rotations.resize(a.local_rotations.size());
    for (size_t j = 0; j < a.local_rotations.size(); ++j)
        out.local_rotations[j] = slerp_shortest(a.local_rotations[j], b.local_rotations[j], t);
    return out;
}

void sample_pose_into(const MotionClip& clip, float time_s, bool wrap, float* out,
                      uint32_t joint_stride) {
    size_t i0, i1;
    float t;
    locate(clip, time_s, wrap, i0, i1, t);
    const Pose& a = clip.frames[i0];
    const Pose& b = clip.frames[i1];
    const Vec3 root = (1.0f - t) * a.root_translation + t * b.root_translation;
    out[0] = root[0];
    out[1] = root[1];
    out[2] = root[2];
    out[3] = 0.0f;
    const size_t joints = std::min<size_t>(a.local_rotations.size(), joint_stride);
    for (size_t j = 0; j < joints; ++j) {
        const Quat q = slerp_shortest(a.local_rotations[j], b.local_rotations[j], t);
        for (int k = 0; k < 4; ++k) out[4 + 4 * j + k] = q.c[k];
    }
}

}  // namespace gsc
