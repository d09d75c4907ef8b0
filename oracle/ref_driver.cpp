// ref_driver.cpp — C entry points over the REFERENCE's own render path, compiled from its
// unmodified sources (/root/reference/proj/src/{math,avatar,synthetic,lod,crowd,renderer,
// metrics,bench}.cpp) against the from-scratch Eigen subset in oracle/eigen_shim/
// (oracle/Makefile, target _ref). TEST INFRASTRUCTURE ONLY: tests/, tests/golden/ and the
// bench's reference arm load oracle/_ref/libgsc_ref.so; the product never does.
//
// What it pins: the oracle restatement (oracle/orc.cpp) and the GPU path are compared
// against the reference's own synthetic generator (synthetic.cpp), crowd builder
// (crowd.cpp:46-84), update_crowd (crowd.cpp:86-140), gather/sort/bin/raster
// (renderer.cpp:25-288) and camera math (math.cpp), bit for bit. What it cannot pin is
// Eigen itself: the shim restates Eigen 3.4's evaluation order (eigen_shim.hpp).
#include "gsc/bench.hpp"
#include "gsc/crowd.hpp"
#include "gsc/metrics.hpp"
#include "gsc/renderer.hpp"

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

extern "C" {

typedef struct {
    uint32_t template_count, template_seed_base, level_count, level_counts[8], joint_count;
    uint32_t motion_count, motion_seed_base, motion_frames;
    float motion_fps;
    uint32_t grid_rows, grid_cols;
    float grid_spacing;
    uint32_t crowd_count;
    uint64_t crowd_seed;
    float cam_pos[3], cam_look[3], fov_y_deg;
    int32_t width, height;
    float near_m;
    uint32_t threshold_count;
    float thresholds[8];
    float hysteresis;
} ref_scene_desc;

typedef struct {
    uint32_t instance_id, template_id, motion_id;
    float x, z, yaw, phase_offset_s;
    uint32_t active_lod;
} ref_instance;

typedef struct {
    float mean_px[2];
    float cov_xx, cov_xy, cov_yy;
    float depth;
    float color[3];
    float opacity;
    uint32_t instance_id, gaussian_index;
    int32_t rect[4];
} ref_splat;

typedef struct {
    int32_t tile_size;
    float background[3];
    float alpha_max, alpha_cutoff, transmittance_floor;
    int32_t pad;
} ref_settings;

typedef struct {
    double update_ms, gather_ms, sort_ms, rasterize_ms;
    uint64_t splat_count, pair_count, gaussian_count;
} ref_times;

}  // extern "C"

struct ref_scene {
    gsc::SceneConfig cfg;
    std::shared_ptr<gsc::TemplateStore> templates;
    std::shared_ptr<gsc::MotionStore> motions;
    gsc::Crowd crowd;
    gsc::Camera camera;
    gsc::FrameContext ctx;
};

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_error = e.what();
        return -1;
    }
}

}  // namespace

#define REF_API __attribute__((visibility("default")))

extern "C" {

REF_API const char* ref_last_error(void) { return g_error.c_str(); }

REF_API ref_scene* ref_scene_new(const ref_scene_desc* d) {
    auto s = std::make_unique<ref_scene>();
    const int rc = guarded([&] {
        if (d->level_count < 1 || d->level_count > 8 || d->threshold_count > 8)
            throw std::invalid_argument("ref_scene_new: bad level/threshold count");
        s->templates = std::make_shared<gsc::TemplateStore>();
        s->motions = std::make_shared<gsc::MotionStore>();
        std::vector<uint32_t> counts(d->level_counts, d->level_counts + d->level_count);
        for (uint32_t t = 0; t < d->template_count; ++t) {
            gsc::AvatarTemplate tpl = gsc::generate_synthetic_template(d->template_seed_base + t, counts, d->joint_count);
            tpl.template_id = t;
            s->templates->push_back(std::move(tpl));
        }
        for (uint32_t m = 0; m < d->motion_count; ++m)
            s->motions->push_back(gsc::generate_synthetic_motion(d->motion_seed_base + m, d->joint_count, d->motion_fps,
                                                                 d->motion_frames));
        gsc::SceneConfig& c = s->cfg;
        c.grid.rows = d->grid_rows;
        c.grid.cols = d->grid_cols;
        c.grid.spacing_m = d->grid_spacing;
        c.crowd_count = d->crowd_count;
        c.seed = d->crowd_seed;
        c.camera.position = gsc::Vec3(d->cam_pos[0], d->cam_pos[1], d->cam_pos[2]);
        c.camera.look_at = gsc::Vec3(d->cam_look[0], d->cam_look[1], d->cam_look[2]);
        c.camera.fov_y_deg = d->fov_y_deg;
        c.camera.width = static_cast<uint32_t>(d->width);
        c.camera.height = static_cast<uint32_t>(d->height);
        c.camera.near_m = d->near_m;
        c.lod.thresholds_m.assign(d->thresholds, d->thresholds + d->threshold_count);
        c.lod.hysteresis_band_m = d->hysteresis;
        s->crowd = gsc::build_crowd(c, s->templates, s->motions, d->crowd_seed);
        s->camera = c.camera.to_camera();
    });
    return rc == 0 ? s.release() : nullptr;
}

REF_API void ref_scene_free(ref_scene* s) { delete s; }

REF_API int ref_scene_counts(ref_scene* s, uint32_t* templates, uint32_t* motions, uint32_t* instances) {
    *templates = static_cast<uint32_t>(s->templates->size());
    *motions = static_cast<uint32_t>(s->motions->size());
    *instances = static_cast<uint32_t>(s->crowd.instances.size());
    return 0;
}

REF_API int ref_get_instances(ref_scene* s, ref_instance* out) {
    for (size_t i = 0; i < s->crowd.instances.size(); ++i) {
        const gsc::CrowdInstance& c = s->crowd.instances[i];
        out[i] = {c.instance_id, c.template_id, c.motion_id, c.x, c.z, c.yaw, c.phase_offset_s, c.active_lod};
    }
    return 0;
}

REF_API int ref_set_instances(ref_scene* s, uint32_t n, const ref_instance* in) {
    return guarded([&] {
        s->crowd.instances.assign(n, gsc::CrowdInstance{});
        for (uint32_t i = 0; i < n; ++i) {
            gsc::CrowdInstance& c = s->crowd.instances[i];
            c.instance_id = in[i].instance_id;
            c.template_id = in[i].template_id;
            c.motion_id = in[i].motion_id;
            c.x = in[i].x;
            c.z = in[i].z;
            c.yaw = in[i].yaw;
            c.phase_offset_s = in[i].phase_offset_s;
            c.active_lod = in[i].active_lod;
        }
    });
}

REF_API uint32_t ref_level_size(ref_scene* s, uint32_t t, uint32_t l) {
    return (*s->templates)[t].levels[l].gaussian_count();
}

REF_API int ref_get_level(ref_scene* s, uint32_t t, uint32_t l, float* means, float* rot_xyzw, float* scales, float* opacities,
                  float* colors, uint16_t* skin_idx, float* skin_w, float* cov6) {
    return guarded([&] {
        const gsc::LodLevel& lv = s->templates->at(t).levels.at(l);
        for (size_t i = 0; i < lv.means.size(); ++i) {
            for (int k = 0; k < 3; ++k) {
                means[3 * i + k] = lv.means[i][k];
                scales[3 * i + k] = lv.scales[i][k];
                colors[3 * i + k] = lv.colors[i][k];
            }
            for (int k = 0; k < 4; ++k) {
                rot_xyzw[4 * i + k] = lv.rotations[i].coeffs()[k];
                skin_idx[4 * i + k] = lv.skin_indices[i][k];
                skin_w[4 * i + k] = lv.skin_weights[i][k];
            }
            opacities[i] = lv.opacities[i];
            for (int k = 0; k < 6; ++k) cov6[6 * i + k] = lv.cov_cache[i][k];
        }
    });
}

REF_API int ref_get_skeleton(ref_scene* s, uint32_t t, uint32_t* joints, int16_t* parents, float* inverse_bind) {
    const gsc::Skeleton& sk = s->templates->at(t).skeleton;
    *joints = sk.joint_count();
    if (parents) std::memcpy(parents, sk.parents.data(), sk.parents.size() * 2);
    if (inverse_bind)
        for (size_t j = 0; j < sk.inverse_bind.size(); ++j) std::memcpy(inverse_bind + 16 * j, sk.inverse_bind[j].data(), 64);
    return 0;
}

// Frame records as the product stores clips: root xyz, pad, then per joint (x, y, z, w).
REF_API int ref_get_motion(ref_scene* s, uint32_t m, float* fps, uint32_t* frames, uint32_t* joints, float* data) {
    const gsc::MotionClip& c = s->motions->at(m);
    if (fps) *fps = c.fps;
    if (frames) *frames = static_cast<uint32_t>(c.frames.size());
    if (joints) *joints = c.joint_count;
    if (data) {
        const size_t stride = 4 + 4 * static_cast<size_t>(c.joint_count);
        for (size_t f = 0; f < c.frames.size(); ++f) {
            float* row = data + f * stride;
            for (int k = 0; k < 3; ++k) row[k] = c.frames[f].root_translation[k];
            row[3] = 0.0f;
            for (size_t j = 0; j < c.frames[f].local_rotations.size(); ++j)
                for (int k = 0; k < 4; ++k) row[4 + 4 * j + k] = c.frames[f].local_rotations[j].coeffs()[k];
        }
    }
    return 0;
}

// The reference's render_frame (renderer.cpp:249-280) with its own threading
// (RenderSettings.thread_count, parallel.hpp:14-22; 0 = GSCROWD_THREADS / hardware).
REF_API int ref_render(ref_scene* s, float time_s, int32_t static_pose, int32_t forced_lod, const ref_settings* st,
               int32_t threads, float* rgb, float* T, ref_times* times) {
    return guarded([&] {
        gsc::RenderSettings rs;
        rs.tile_size = st->tile_size;
        rs.background = gsc::Vec3(st->background[0], st->background[1], st->background[2]);
        rs.alpha_max = st->alpha_max;
        rs.alpha_cutoff = st->alpha_cutoff;
        rs.transmittance_floor = st->transmittance_floor;
        rs.thread_count = threads;
        std::optional<uint32_t> forced;
        if (forced_lod >= 0) forced = static_cast<uint32_t>(forced_lod);
        gsc::StageTimes tm;
        gsc::render_frame(s->crowd, s->camera, time_s, rs, static_pose != 0, forced, &tm, s->ctx);
        const size_t px = static_cast<size_t>(s->camera.width) * s->camera.height;
        if (rgb) std::memcpy(rgb, s->ctx.out.color.rgb.data(), px * 12);
        if (T) std::memcpy(T, s->ctx.out.transmittance.data(), px * 4);
        if (times) {
            uint64_t pairs = 0, g = 0;
            for (const auto& b : s->ctx.bins) pairs += b.size();
            for (const auto& inst : s->crowd.instances) g += inst.posed_means.size();
            *times = {tm.update_ms, tm.gather_ms, tm.sort_ms, tm.rasterize_ms, tm.splat_count, pairs, g};
        }
    });
}

REF_API int ref_get_lods(ref_scene* s, uint32_t* out) {
    for (size_t i = 0; i < s->crowd.instances.size(); ++i) out[i] = s->crowd.instances[i].active_lod;
    return 0;
}

REF_API uint64_t ref_gaussian_count(ref_scene* s) {
    uint64_t g = 0;
    for (const auto& inst : s->crowd.instances) g += inst.posed_means.size();
    return g;
}

REF_API int ref_get_posed(ref_scene* s, float* out) {
    size_t o = 0;
    for (const auto& inst : s->crowd.instances)
        for (const auto& p : inst.posed_means) {
            out[o++] = p[0];
            out[o++] = p[1];
            out[o++] = p[2];
        }
    return 0;
}

REF_API uint64_t ref_splat_count(ref_scene* s) { return s->ctx.frame.splats.size(); }

REF_API int ref_get_splats(ref_scene* s, ref_splat* out) {
    for (size_t i = 0; i < s->ctx.frame.splats.size(); ++i) {
        const gsc::FrameSplat& f = s->ctx.frame.splats[i];
        ref_splat& o = out[i];
        o.mean_px[0] = f.splat.mean_px.x();
        o.mean_px[1] = f.splat.mean_px.y();
        o.cov_xx = f.splat.cov_xx;
        o.cov_xy = f.splat.cov_xy;
        o.cov_yy = f.splat.cov_yy;
        o.depth = f.splat.depth;
        for (int k = 0; k < 3; ++k) o.color[k] = f.splat.color[k];
        o.opacity = f.splat.opacity;
        o.instance_id = f.instance_id;
        o.gaussian_index = f.gaussian_index;
        o.rect[0] = f.bounds.x0;
        o.rect[1] = f.bounds.y0;
        o.rect[2] = f.bounds.x1;
        o.rect[3] = f.bounds.y1;
    }
    return 0;
}

REF_API uint64_t ref_pair_count(ref_scene* s) {
    uint64_t k = 0;
    for (const auto& b : s->ctx.bins) k += b.size();
    return k;
}

REF_API int ref_get_bins(ref_scene* s, uint32_t* tile_counts, uint32_t* items) {
    size_t o = 0;
    for (size_t t = 0; t < s->ctx.bins.size(); ++t) {
        tile_counts[t] = static_cast<uint32_t>(s->ctx.bins[t].size());
        for (uint32_t v : s->ctx.bins[t]) items[o++] = v;
    }
    return 0;
}

// The reference's psnr (metrics.cpp:8-23) over two float images.
REF_API float ref_psnr(const float* a, const float* b, int32_t width, int32_t height) {
    gsc::Framebuffer fa(width, height), fb(width, height);
    std::memcpy(fa.rgb.data(), a, fa.rgb.size() * 4);
    std::memcpy(fb.rgb.data(), b, fb.rgb.size() * 4);
    return gsc::psnr(fa, fb);
}

}  // extern "C"
