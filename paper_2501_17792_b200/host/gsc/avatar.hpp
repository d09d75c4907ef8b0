// Avatar templates, skeletons, motion clips and pose sampling — the host-side data model
// of the B200 crowd renderer. Mirrors /root/reference/proj/include/gsc/avatar.hpp
// (Skeleton :16-31, Pose :33-36, MotionClip :40-48, LodLevel :50-65, AvatarTemplate
// :69-73). Forward kinematics, skin matrices and LBS run on the GPU
// (paper_2501_17792_b200/csrc/gscg_update.cu); pose sampling (acos/sin) stays on host
// so poses are bit-identical to the reference's glibc evaluation.
#pragma once

#include "gsc/math.hpp"

#include <array>
#include <cstdint>
#include <span>
#include <vector>

namespace gsc {

struct Skeleton {
    std::vector<int16_t> parents;
    std::vector<Mat4> inverse_bind;
    std::vector<Mat4> bind;        // inverse_bind^-1
    std::vector<Mat4> local_bind;  // bind[parent]^-1 * bind[j]

    uint32_t joint_count() const { return static_cast<uint32_t>(parents.size()); }
    static Skeleton make(std::vector<int16_t> parents, std::vector<Mat4> inverse_bind);
};

struct Pose {
    Vec3 root_translation = Vec3::Zero();
    std::vector<Quat> local_rotations;
};

Pose bind_pose(uint32_t joint_count);

struct MotionClip {
    float fps = 30.0f;
    uint16_t joint_count = 0;
    std::vector<Pose> frames;
    float duration_s() const { return static_cast<float>(frames.size()) / fps; }
};

void validate(const MotionClip& clip);

// Number of SH residual floats per Gaussian (degrees 1..3, RGB): the BASELINE "SH
// colour" extension. Empty `sh` = reference RGB only.
inline constexpr uint32_t kShFloats = 45;

struct LodLevel {
    std::vector<Vec3> means;
    std::vector<Quat> rotations;
    std::vector<Vec3> scales;
    std::vector<float> opacities;
    std::vector<Vec3> colors;
    std::vector<std::array<uint16_t, 4>> skin_indices;
    std::vector<std::array<float, 4>> skin_weights;
    std::vector<float> sh;  // gaussian_count * kShFloats, or empty

    std::vector<std::array<float, 6>> cov_cache;  // xx,xy,xz,yy,yz,zz (finalize)

    uint32_t gaussian_count() const { return static_cast<uint32_t>(means.size()); }
    void finalize();
};

void validate(const LodLevel& level, uint32_t joint_count);

struct AvatarTemplate {
    uint32_t template_id = 0;
    Skeleton skeleton;
    std::vector<LodLevel> levels;
};

void validate(const AvatarTemplate& tpl);

Quat slerp_shortest(const Quat& a, const Quat& b, float t);
Pose sample_pose(const MotionClip& clip, float time_s, bool wrap);
// Allocation-free form writing the GPU pose record: root xyz, pad, then J quats (xyzw).
void sample_pose_into(const MotionClip& clip, float time_s, bool wrap, float* out,
                      uint32_t joint_stride);

AvatarTemplate generate_synthetic_template(uint64_t seed, std::span<const uint32_t> level_counts,
                                           uint32_t joint_count = 24, bool with_sh = false);
MotionClip generate_synthetic_motion(uint64_t seed, uint32_t joint_count = 24,
                                     float fps = 30.0f, uint32_t frame_count = 60);

}  // namespace gsc
