// Asset files of the crowd renderer: GSAT avatar templates and GSMO motion clips.
// Mirrors the reference's asset API and byte layout (/root/reference/proj/include/gsc/io.hpp
// :18-43, src/io_assets.cpp) so files written by either side load in the other:
//   GSAT v1: "GSAT" u32 version, u16 joints, u8 levels, joints x i16 parent,
//            joints x 16 f32 inverse bind (row-major), then per level u32 count and the
//            SoA blocks means (3 f32), rotations (w,x,y,z f32), scales (3 f32),
//            opacities (f32), colors (3 f32), skin indices (4 u16), skin weights (4 f32).
//   GSAT v2: v1 plus, after each level's skin weights, a u8 SH flag and, when set,
//            count x 45 f32 SH residuals (the SH-3 colour extension).
//            Templates without SH are always written as v1.
//   GSMO v1: "GSMO" u32 version, f32 fps, u32 frames, u16 joints, then per frame the
//            root translation (3 f32) and joints x (w,x,y,z f32).
// All integers and floats are little-endian. Failures are typed (FormatErrorKind), and a
// truncated file names the section it ended in.
#pragma once

#include "gsc/avatar.hpp"

#include <cstdint>
#include <filesystem>
#include <stdexcept>
#include <string>

namespace gsc {

enum class FormatErrorKind { IoError, BadMagic, VersionMismatch, Truncated, InvariantViolation };

const char* to_string(FormatErrorKind kind);

class FormatError : public std::runtime_error {
public:
    FormatError(FormatErrorKind kind, const std::string& message) : std::runtime_error(message), kind_(kind) {}
    FormatErrorKind kind() const { return kind_; }

private:
    FormatErrorKind kind_;
};

inline constexpr uint32_t kGsatVersion = 1;    // reference layout
inline constexpr uint32_t kGsatVersionSh = 2;  // + SH residual blocks
inline constexpr uint32_t kGsmoVersion = 1;

void save_template(const AvatarTemplate& tpl, const std::filesystem::path& path);
AvatarTemplate load_template(const std::filesystem::path& path);  // v1 or v2; levels finalized

void save_motion(const MotionClip& clip, const std::filesystem::path& path);
MotionClip load_motion(const std::filesystem::path& path);

}  // namespace gsc
