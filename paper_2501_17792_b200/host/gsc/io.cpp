// GSAT / GSMO asset files (layout in io.hpp; reference io_assets.cpp:137-330). Files are
// assembled in memory and written with one call, and read whole into memory and decoded
// from a bounds-checked cursor, so block decodes are straight copies on little-endian hosts.
#include "gsc/io.hpp"

#include <algorithm>
#include <bit>
#include <type_traits>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

namespace gsc {

const char* to_string(FormatErrorKind kind) {
    switch (kind) {
        case FormatErrorKind::IoError: return "IoError";
        case FormatErrorKind::BadMagic: return "BadMagic";
        case FormatErrorKind::VersionMismatch: return "VersionMismatch";
        case FormatErrorKind::Truncated: return "Truncated";
        case FormatErrorKind::InvariantViolation: return "InvariantViolation";
    }
    return "?";
}

namespace {

constexpr bool kLittle = std::endian::native == std::endian::little;

// Little-endian encoder into a growing byte buffer.
struct Encoder {
    std::vector<uint8_t> buf;

    void raw(const void* p, size_t n) {
        const auto* b = static_cast<const uint8_t*>(p);
        buf.insert(buf.end(), b, b + n);
    }
    template <typename T>
    void put(T v) {
        static_assert(std::is_trivially_copyable_v<T>);
        uint8_t b[sizeof(T)];
        std::memcpy(b, &v, sizeof(T));
        if constexpr (!kLittle) std::reverse(b, b + sizeof(T));
        raw(b, sizeof(T));
    }
    void floats(const float* p, size_t n) {
        if constexpr (kLittle) {
            raw(p, n * sizeof(float));
        } else {
            for (size_t i = 0; i < n; ++i) put(p[i]);
        }
    }
    void write_file(const std::filesystem::path& path) const {
        std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "wb"), &std::fclose);
        if (!f) throw FormatError(FormatErrorKind::IoError, "cannot open for writing: " + path.string());
        if (!buf.empty() && std::fwrite(buf.data(), 1, buf.size(), f.get()) != buf.size())
            throw FormatError(FormatErrorKind::IoError, "write failed: " + path.string());
        if (std::fflush(f.get()) != 0) throw FormatError(FormatErrorKind::IoError, "write failed: " + path.string());
    }
};

// Bounds-checked little-endian decoder over a whole file; `section` names the part
// being read for truncation errors.
struct Decoder {
    std::vector<uint8_t> buf;
    size_t at = 0;
    std::string section = "magic";

    explicit Decoder(const std::filesystem::path& path) {
        std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
        if (!f) throw FormatError(FormatErrorKind::IoError, "cannot open for reading: " + path.string());
        if (std::fseek(f.get(), 0, SEEK_END) != 0) throw FormatError(FormatErrorKind::IoError, "read failed: " + path.string());
        const long size = std::ftell(f.get());
        if (size < 0) throw FormatError(FormatErrorKind::IoError, "read failed: " + path.string());
        std::rewind(f.get());
        buf.resize(static_cast<size_t>(size));
        if (size > 0 && std::fread(buf.data(), 1, buf.size(), f.get()) != buf.size())
            throw FormatError(FormatErrorKind::IoError, "read failed: " + path.string());
    }
    const uint8_t* take(size_t n) {
        if (n > buf.size() - at)
            throw FormatError(FormatErrorKind::Truncated, "file truncated in section '" + section + "'");
        const uint8_t* p = buf.data() + at;
        at += n;
        return p;
    }
    template <typename T>
    T get() {
        uint8_t b[sizeof(T)];
        std::memcpy(b, take(sizeof(T)), sizeof(T));
        if constexpr (!kLittle) std::reverse(b, b + sizeof(T));
        T v;
        std::memcpy(&v, b, sizeof(T));
        return v;
    }
    void floats(float* out, size_t n) {
        const uint8_t* p = take(n * sizeof(float));
        if constexpr (kLittle) {
            std::memcpy(out, p, n * sizeof(float));
        } else {
            for (size_t i = 0; i < n; ++i) {
                uint8_t b[4] = {p[4 * i + 3], p[4 * i + 2], p[4 * i + 1], p[4 * i]};
                std::memcpy(out + i, b, 4);
            }
        }
    }
    bool done() const { return at == buf.size(); }
};

// Reads magic + version; returns the version (one of `accepted`).
uint32_t open_asset(Decoder& d, const char magic[4], const char* what, std::initializer_list<uint32_t> accepted) {
    d.section = "magic";
    if (std::memcmp(d.take(4), magic, 4) != 0)
        throw FormatError(FormatErrorKind::BadMagic, std::string("bad magic, not a ") + what + " file");
    d.section = "version";
    const uint32_t v = d.get<uint32_t>();
    for (uint32_t a : accepted)
        if (v == a) return v;
    throw FormatError(FormatErrorKind::VersionMismatch, std::string("unsupported ") + what + " version " + std::to_string(v));
}

// std::invalid_argument from the data-model validators becomes an invariant violation.
template <typename F>
auto as_invariant(F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        throw FormatError(FormatErrorKind::InvariantViolation, e.what());
    }
}

}  // namespace

void save_template(const AvatarTemplate& tpl, const std::filesystem::path& path) {
    validate(tpl);
    bool any_sh = false;
    for (const LodLevel& l : tpl.levels) any_sh |= !l.sh.empty();
    Encoder e;
    e.raw("GSAT", 4);
    e.put<uint32_t>(any_sh ? kGsatVersionSh : kGsatVersion);
    const uint32_t J = tpl.skeleton.joint_count();
    e.put<uint16_t>(static_cast<uint16_t>(J));
    e.put<uint8_t>(static_cast<uint8_t>(tpl.levels.size()));
    for (int16_t p : tpl.skeleton.parents) e.put<int16_t>(p);
    for (const Mat4& m : tpl.skeleton.inverse_bind)
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) e.put<float>(m(r, c));
    for (const LodLevel& l : tpl.levels) {
        const uint32_t n = l.gaussian_count();
        e.put<uint32_t>(n);
        for (const Vec3& v : l.means) e.floats(v.v, 3);
        for (const Quat& q : l.rotations) {
            const float wxyz[4] = {q.w(), q.x(), q.y(), q.z()};
            e.floats(wxyz, 4);
        }
        for (const Vec3& v : l.scales) e.floats(v.v, 3);
        e.floats(l.opacities.data(), n);
        for (const Vec3& v : l.colors) e.floats(v.v, 3);
        for (const auto& idx : l.skin_indices)
            for (uint16_t i : idx) e.put<uint16_t>(i);
        for (const auto& w : l.skin_weights) e.floats(w.data(), 4);
        if (any_sh) {
            e.put<uint8_t>(l.sh.empty() ? 0 : 1);
            if (!l.sh.empty()) e.floats(l.sh.data(), l.sh.size());
        }
    }
    e.write_file(path);
}

AvatarTemplate load_template(const std::filesystem::path& path) {
    Decoder d(path);
    const uint32_t version = open_asset(d, "GSAT", "GSAT template", {kGsatVersion, kGsatVersionSh});
    d.section = "header";
    const uint16_t J = d.get<uint16_t>();
    const uint8_t levels = d.get<uint8_t>();
    if (J < 1 || levels < 1)
        throw FormatError(FormatErrorKind::InvariantViolation, "GSAT header: joint and level counts must be >= 1");
    d.section = "parents";
    std::vector<int16_t> parents(J);
    for (int16_t& p : parents) p = d.get<int16_t>();
    d.section = "inverse_bind";
    std::vector<Mat4> inv(J);
    for (Mat4& m : inv)
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) m(r, c) = d.get<float>();
    AvatarTemplate tpl;
    tpl.skeleton = as_invariant([&] { return Skeleton::make(std::move(parents), std::move(inv)); });
    tpl.levels.resize(levels);
    for (uint32_t li = 0; li < levels; ++li) {
        LodLevel& l = tpl.levels[li];
        const std::string lv = "level " + std::to_string(li);
        d.section = lv + " count";
        const uint32_t n = d.get<uint32_t>();
        d.section = lv + " means";
        l.means.resize(n);
        for (Vec3& v : l.means) d.floats(v.v, 3);
        d.section = lv + " rotations";
        l.rotations.resize(n);
        for (Quat& q : l.rotations) {
            float wxyz[4];
            d.floats(wxyz, 4);
            q = Quat(wxyz[0], wxyz[1], wxyz[2], wxyz[3]);
        }
        d.section = lv + " scales";
        l.scales.resize(n);
        for (Vec3& v : l.scales) d.floats(v.v, 3);
        d.section = lv + " opacities";
        l.opacities.resize(n);
        d.floats(l.opacities.data(), n);
        d.section = lv + " colors";
        l.colors.resize(n);
        for (Vec3& v : l.colors) d.floats(v.v, 3);
        d.section = lv + " skin_indices";
        l.skin_indices.resize(n);
        for (auto& idx : l.skin_indices)
            for (uint16_t& i : idx) i = d.get<uint16_t>();
        d.section = lv + " skin_weights";
        l.skin_weights.resize(n);
        for (auto& w : l.skin_weights) d.floats(w.data(), 4);
        if (version == kGsatVersionSh) {
            d.section = lv + " sh";
            const uint8_t has = d.get<uint8_t>();
            if (has > 1) throw FormatError(FormatErrorKind::InvariantViolation, "GSAT " + lv + ": bad SH flag");
            if (has) {
                l.sh.resize(static_cast<size_t>(n) * kShFloats);
                d.floats(l.sh.data(), l.sh.size());
            }
        }
        as_invariant([&] {
            l.finalize();
            return 0;
        });
    }
    if (!d.done()) throw FormatError(FormatErrorKind::InvariantViolation, "GSAT file has trailing bytes");
    as_invariant([&] {
        validate(tpl);
        return 0;
    });
    return tpl;
}

void save_motion(const MotionClip& clip, const std::filesystem::path& path) {
    validate(clip);
    Encoder e;
    e.raw("GSMO", 4);
    e.put<uint32_t>(kGsmoVersion);
    e.put<float>(clip.fps);
    e.put<uint32_t>(static_cast<uint32_t>(clip.frames.size()));
    e.put<uint16_t>(clip.joint_count);
    for (const Pose& p : clip.frames) {
        e.floats(p.root_translation.v, 3);
        for (const Quat& q : p.local_rotations) {
            const float wxyz[4] = {q.w(), q.x(), q.y(), q.z()};
            e.floats(wxyz, 4);
        }
    }
    e.write_file(path);
}

MotionClip load_motion(const std::filesystem::path& path) {
    Decoder d(path);
    open_asset(d, "GSMO", "GSMO motion", {kGsmoVersion});
    d.section = "header";
    MotionClip clip;
    clip.fps = d.get<float>();
    const uint32_t frames = d.get<uint32_t>();
    clip.joint_count = d.get<uint16_t>();
    if (!(clip.fps > 0.0f)) throw FormatError(FormatErrorKind::InvariantViolation, "GSMO header: fps must be > 0");
    if (frames < 1) throw FormatError(FormatErrorKind::InvariantViolation, "GSMO header: frame count must be >= 1");
    clip.frames.resize(frames);
    for (uint32_t f = 0; f < frames; ++f) {
        d.section = "frame " + std::to_string(f);
        Pose& p = clip.frames[f];
        d.floats(p.root_translation.v, 3);
        p.local_rotations.resize(clip.joint_count);
        for (Quat& q : p.local_rotations) {
            float wxyz[4];
            d.floats(wxyz, 4);
            q = Quat(wxyz[0], wxyz[1], wxyz[2], wxyz[3]);
        }
    }
    if (!d.done()) throw FormatError(FormatErrorKind::InvariantViolation, "GSMO file has trailing bytes");
    as_invariant([&] {
        validate(clip);
        return 0;
    });
    return clip;
}

}  // namespace gsc
