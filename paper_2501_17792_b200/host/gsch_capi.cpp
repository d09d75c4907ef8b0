// C-ABI of the host scene layer (include/gsch.h) over the gsc host API.
#include "gsch.h"
#include "gsc/io.hpp"
#include "gsc/metrics.hpp"

#include <cstring>
#include <string>
#include <thread>

#include "gsc/renderer.hpp"

using namespace gsc;

struct gsch_scene {
    std::shared_ptr<TemplateStore> templates;
    std::shared_ptr<MotionStore> motions;
    Crowd crowd;
    CameraConfig camera_cfg;
    Camera camera;
    std::vector<std::vector<float>> rot_cache;  // per (template, level) flattened quats
};

struct gsch_renderer {
    gsch_scene* scene;
    std::unique_ptr<FrameContext> ctx;
};

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return GSCG_ERR_INVALID_ARGUMENT;
    } catch (const GpuError& e) {
        g_error = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_error = "out of memory";
        return GSCG_ERR_OOM;
    } catch (const FormatError& e) {
        g_error = std::string("[") + to_string(e.kind()) + "] " + e.what();
        return GSCH_ERR_FORMAT;
    } catch (const std::exception& e) {
        g_error = e.what();
        return GSCG_ERR_STATE;
    }
}

Vec3 v3(const float* p) { return Vec3(p[0], p[1], p[2]); }

}  // namespace

extern "C" {

const char* gsch_last_error(void) { return g_error.c_str(); }

int gsch_scene_create(const gsch_scene_config* cfg, int threads, gsch_scene** out) {
    return guarded([&] {
        if (!cfg || !out) throw std::invalid_argument("null argument");
        if (cfg->level_count < 1 || cfg->level_count > 4) throw std::invalid_argument("level_count must be in [1,4]");
        if (cfg->template_count < 1 || cfg->motion_count < 1) throw std::invalid_argument("need templates and motions");
        auto scene = std::make_unique<gsch_scene>();
        scene->templates = std::make_shared<TemplateStore>(cfg->template_count);
        std::vector<uint32_t> counts(cfg->level_counts, cfg->level_counts + cfg->level_count);
        const unsigned nt = std::max(1u, std::min<unsigned>(resolve_thread_count(threads), cfg->template_count));
        std::vector<std::thread> pool;
        std::vector<std::string> errors(nt);
        for (unsigned w = 0; w < nt; ++w) {
            pool.emplace_back([&, w] {
                try {
                    for (uint32_t i = w; i < cfg->template_count; i += nt) {
                        AvatarTemplate tpl = generate_synthetic_template(
                            cfg->template_seed_base + i, counts, cfg->joint_count, cfg->with_sh != 0);
                        tpl.template_id = i;
                        (*scene->templates)[i] = std::move(tpl);
                    }
                } catch (const std::exception& e) {
                    errors[w] = e.what();
                }
            });
        }
        for (auto& t : pool) t.join();
        for (const auto& e : errors)
            if (!e.empty()) throw std::invalid_argument(e);
        scene->motions = std::make_shared<MotionStore>();
        for (uint32_t m = 0; m < cfg->motion_count; ++m)
            scene->motions->push_back(generate_synthetic_motion(cfg->motion_seed_base + m, cfg->joint_count,
                                                                cfg->motion_fps, cfg->motion_frames));
        SceneConfig sc;
        sc.grid.rows = cfg->grid_rows;
        sc.grid.cols = cfg->grid_cols;
        sc.grid.spacing_m = cfg->grid_spacing;
        sc.crowd_count = cfg->crowd_count;
        sc.seed = cfg->crowd_seed;
        sc.camera.position = v3(cfg->cam_pos);
        sc.camera.look_at = v3(cfg->cam_look);
        sc.camera.fov_y_deg = cfg->fov_y_deg;
        sc.camera.width = cfg->width;
        sc.camera.height = cfg->height;
        sc.camera.near_m = cfg->near_m;
        sc.lod.thresholds_m.assign(cfg->lod_thresholds, cfg->lod_thresholds + cfg->lod_threshold_count);
        sc.lod.hysteresis_band_m = cfg->lod_hysteresis;
        scene->crowd = build_crowd(sc, scene->templates, scene->motions, cfg->crowd_seed);
        scene->camera_cfg = sc.camera;
        scene->camera = sc.camera.to_camera();
        *out = scene.release();
    });
}

int gsch_scene_destroy(gsch_scene* scene) {
    delete scene;
    return 0;
}

int gsch_scene_counts(const gsch_scene* s, uint32_t* t, uint32_t* m, uint32_t* n) {
    if (!s) return GSCG_ERR_INVALID_ARGUMENT;
    if (t) *t = static_cast<uint32_t>(s->templates->size());
    if (m) *m = static_cast<uint32_t>(s->motions->size());
    if (n) *n = static_cast<uint32_t>(s->crowd.instances.size());
    return 0;
}

int gsch_scene_get_instances(const gsch_scene* s, gsch_instance* out, uint32_t n) {
    return guarded([&] {
        if (!s || !out || n > s->crowd.instances.size()) throw std::invalid_argument("bad instance query");
        for (uint32_t i = 0; i < n; ++i) {
            const CrowdInstance& c = s->crowd.instances[i];
            out[i] = {c.instance_id, c.template_id, c.motion_id, c.x, c.z, c.yaw, c.phase_offset_s, c.active_lod};
        }
    });
}

int gsch_scene_set_instances(gsch_scene* s, const gsch_instance* in, uint32_t n) {
    return guarded([&] {
        if (!s || (!in && n)) throw std::invalid_argument("bad instance update");
        s->crowd.instances.resize(n);
        for (uint32_t i = 0; i < n; ++i) {
            if (in[i].template_id >= s->templates->size() || in[i].motion_id >= s->motions->size())
                throw std::invalid_argument("instance references a missing asset");
            CrowdInstance& c = s->crowd.instances[i];
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

int gsch_scene_set_camera(gsch_scene* s, const float* pos, const float* look, float fov,
                          uint32_t w, uint32_t h, float near_m) {
    return guarded([&] {
        if (!s || !pos || !look) throw std::invalid_argument("null camera argument");
        s->camera_cfg.position = v3(pos);
        s->camera_cfg.look_at = v3(look);
        s->camera_cfg.fov_y_deg = fov;
        s->camera_cfg.width = w;
        s->camera_cfg.height = h;
        s->camera_cfg.near_m = near_m;
        s->camera = s->camera_cfg.to_camera();
        validate(s->camera);
    });
}

int gsch_scene_camera_basis(const gsch_scene* s, gscg_camera* out) {
    if (!s || !out) return GSCG_ERR_INVALID_ARGUMENT;
    *out = camera_basis(s->camera);
    return 0;
}

int gsch_scene_set_lod_policy(gsch_scene* s, const float* th, uint32_t count, float band) {
    return guarded([&] {
        if (!s || (count && !th)) throw std::invalid_argument("bad lod policy");
        LodPolicy p;
        p.thresholds_m.assign(th, th + count);
        p.hysteresis_band_m = band;
        validate(p);
        s->crowd.lod = p;
    });
}

int gsch_scene_level_count(const gsch_scene* s, uint32_t t, uint32_t* out) {
    if (!s || !out || t >= s->templates->size()) return GSCG_ERR_INVALID_ARGUMENT;
    *out = static_cast<uint32_t>((*s->templates)[t].levels.size());
    return 0;
}

int gsch_scene_level_view(const gsch_scene* s, uint32_t t, uint32_t l, gsch_level_view* out) {
    if (!s || !out || t >= s->templates->size() || l >= (*s->templates)[t].levels.size())
        return GSCG_ERR_INVALID_ARGUMENT;
    const LodLevel& lv = (*s->templates)[t].levels[l];
    out->count = lv.gaussian_count();
    out->means = lv.means[0].v;
    out->rotations = lv.rotations[0].c;
    out->scales = lv.scales[0].v;
    out->opacities = lv.opacities.data();
    out->colors = lv.colors[0].v;
    out->skin_indices = lv.skin_indices[0].data();
    out->skin_weights = lv.skin_weights[0].data();
    out->sh = lv.sh.empty() ? nullptr : lv.sh.data();
    out->cov6 = lv.cov_cache[0].data();
    return 0;
}

int gsch_scene_skeleton(const gsch_scene* s, uint32_t t, uint32_t* joints, const int16_t** parents,
                        const float** inverse_bind) {
    if (!s || t >= s->templates->size()) return GSCG_ERR_INVALID_ARGUMENT;
    const Skeleton& sk = (*s->templates)[t].skeleton;
    if (joints) *joints = sk.joint_count();
    if (parents) *parents = sk.parents.data();
    if (inverse_bind) *inverse_bind = sk.inverse_bind[0].m;
    return 0;
}

int gsch_scene_motion(const gsch_scene* s, uint32_t m, float* fps, uint32_t* frames, uint32_t* joints,
                      float* out) {
    if (!s || m >= s->motions->size()) return GSCG_ERR_INVALID_ARGUMENT;
    const MotionClip& c = (*s->motions)[m];
    if (fps) *fps = c.fps;
    if (frames) *frames = static_cast<uint32_t>(c.frames.size());
    if (joints) *joints = c.joint_count;
    if (out) {
        const size_t rec = 4 + 4 * static_cast<size_t>(c.joint_count);
        for (size_t f = 0; f < c.frames.size(); ++f) {
            float* o = out + f * rec;
            const Pose& p = c.frames[f];
            o[0] = p.root_translation[0];
            o[1] = p.root_translation[1];
            o[2] = p.root_translation[2];
            o[3] = 0.0f;
            for (size_t j = 0; j < p.local_rotations.size(); ++j)
                std::memcpy(o + 4 + 4 * j, p.local_rotations[j].c, 16);
        }
    }
    return 0;
}

int gsch_scene_sample_crowd(gsch_scene* s, float time_s, int32_t static_pose, int32_t threads,
                            uint32_t joint_stride, uint32_t* template_ids, float* placement, float* poses) {
    return guarded([&] {
        if (!s || !template_ids || !placement || !poses) throw std::invalid_argument("null argument");
        HostPool pool(resolve_thread_count(threads));
        sample_crowd_records(s->crowd, time_s, static_pose != 0, joint_stride, pool, template_ids, placement,
                             poses, nullptr);
    });
}

int gsch_scene_set_motion(gsch_scene* s, uint32_t m, float fps, uint32_t frames, uint32_t joints,
                          const float* data) {
    return guarded([&] {
        if (!s || (frames && !data)) throw std::invalid_argument("bad motion");
        if (m > s->motions->size()) throw std::invalid_argument("motion id beyond the store");
        MotionClip clip;
        clip.fps = fps;
        clip.joint_count = static_cast<uint16_t>(joints);
        clip.frames.resize(frames);
        const size_t rec = 4 + 4 * static_cast<size_t>(joints);
        for (uint32_t f = 0; f < frames; ++f) {
            const float* d = data + f * rec;
            clip.frames[f].root_translation = Vec3(d[0], d[1], d[2]);
            clip.frames[f].local_rotations.resize(joints);
            for (uint32_t j = 0; j < joints; ++j)
                clip.frames[f].local_rotations[j] = Quat::FromCoeffs(d + 4 + 4 * j);
        }
        validate(clip);
        // Copy-on-write: renderers keep the old store alive; motions are read per frame.
        auto next = std::make_shared<MotionStore>(*s->motions);
        if (m == next->size()) next->push_back(std::move(clip));
        else (*next)[m] = std::move(clip);
        s->motions = next;
        s->crowd.motions = next;
    });
}

int gsch_scene_update_crowd(gsch_scene* s, int32_t forced_lod) {
    return guarded([&] {
        if (!s) throw std::invalid_argument("null scene");
        std::optional<uint32_t> forced;
        if (forced_lod >= 0) forced = static_cast<uint32_t>(forced_lod);
        update_crowd_lod(s->crowd, s->camera, forced);  // the LoD step (no GPU)
    });
}

int gsch_scene_save_template(const gsch_scene* s, uint32_t t, const char* path) {
    return guarded([&] {
        if (!s || !path) throw std::invalid_argument("null argument");
        if (t >= s->templates->size()) throw std::invalid_argument("template id beyond the store");
        save_template((*s->templates)[t], path);
    });
}

int gsch_scene_load_template(gsch_scene* s, uint32_t t, const char* path) {
    return guarded([&] {
        if (!s || !path) throw std::invalid_argument("null argument");
        if (t > s->templates->size()) throw std::invalid_argument("template id beyond the store");
        AvatarTemplate tpl = load_template(path);
        tpl.template_id = t;
        // Copy-on-write: a renderer re-uploads when it sees a new store (FrameContext).
        auto next = std::make_shared<TemplateStore>(*s->templates);
        if (t == next->size()) next->push_back(std::move(tpl));
        else (*next)[t] = std::move(tpl);
        s->templates = next;
        s->crowd.templates = next;
    });
}

int gsch_scene_save_motion(const gsch_scene* s, uint32_t m, const char* path) {
    return guarded([&] {
        if (!s || !path) throw std::invalid_argument("null argument");
        if (m >= s->motions->size()) throw std::invalid_argument("motion id beyond the store");
        save_motion((*s->motions)[m], path);
    });
}

int gsch_scene_load_motion(gsch_scene* s, uint32_t m, const char* path) {
    return guarded([&] {
        if (!s || !path) throw std::invalid_argument("null argument");
        if (m > s->motions->size()) throw std::invalid_argument("motion id beyond the store");
        MotionClip clip = load_motion(path);
        auto next = std::make_shared<MotionStore>(*s->motions);
        if (m == next->size()) next->push_back(std::move(clip));
        else (*next)[m] = std::move(clip);
        s->motions = next;
        s->crowd.motions = next;
    });
}

static void fill_report(const MemoryReport& r, gsch_memory_report* out) {
    out->naive_bytes = r.naive_bytes;
    out->shared_bytes = r.shared_bytes;
    out->savings_fraction = r.savings_fraction;
    out->naive_marginal_bytes_per_instance = r.naive_marginal_bytes_per_instance;
    out->shared_marginal_bytes_per_instance = r.shared_marginal_bytes_per_instance;
    out->resident_template_bytes = r.resident_template_bytes;
    out->posed_mean_bytes = r.posed_mean_bytes;
    out->instance_count = r.instance_count;
}

int gsch_memory_report_cell(uint64_t instances, uint64_t gaussians, uint64_t fixed_overhead,
                            gsch_memory_report* out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("null output");
        MemoryLayoutModel model;
        model.fixed_overhead_bytes = fixed_overhead;
        fill_report(memory_report_cell(instances, gaussians, model), out);
    });
}

int gsch_scene_memory_report(const gsch_scene* s, gsch_memory_report* out) {
    return guarded([&] {
        if (!s || !out) throw std::invalid_argument("null argument");
        fill_report(memory_report(s->crowd, MemoryLayoutModel{}), out);
    });
}

int gsch_renderer_create(gsch_scene* scene, int device, gsch_renderer** out) {
    return guarded([&] {
        if (!scene || !out) throw std::invalid_argument("null argument");
        auto r = std::make_unique<gsch_renderer>();
        r->scene = scene;
        r->ctx = std::make_unique<FrameContext>(device);
        r->ctx->ensure_templates(scene->templates);
        *out = r.release();
    });
}

int gsch_renderer_destroy(gsch_renderer* r) {
    delete r;
    return 0;
}

gscg_ctx* gsch_renderer_gpu(gsch_renderer* r) { return r ? r->ctx->gpu() : nullptr; }

uint32_t gsch_renderer_joint_stride(gsch_renderer* r) { return r ? r->ctx->joint_stride : 0; }

int gsch_fill_instances(gsch_renderer* r, int32_t static_pose, uint32_t* template_ids, float* placement,
                        uint32_t* motion_ids, float* phase_offsets, uint32_t* lods) {
    return guarded([&] {
        if (!r) throw std::invalid_argument("null renderer");
        FrameContext& c = *r->ctx;
        c.fill_instances(r->scene->crowd, static_pose != 0);
        const size_t n = r->scene->crowd.instances.size();
        if (template_ids) std::memcpy(template_ids, c.template_ids.data(), n * 4);
        if (placement) std::memcpy(placement, c.placement.data(), n * 16);
        if (motion_ids) std::memcpy(motion_ids, c.motion_ids.data(), n * 4);
        if (phase_offsets) std::memcpy(phase_offsets, c.phases.data(), n * 4);
        if (lods) std::memcpy(lods, c.lods.data(), n * 4);
    });
}

int gsch_renderer_prepare(gsch_renderer* r) {
    return guarded([&] {
        if (!r) throw std::invalid_argument("null renderer");
        r->ctx->ensure_templates(r->scene->crowd.templates);
        r->ctx->ensure_motions(r->scene->crowd.motions);
    });
}

int gsch_renderer_set_device_poses(gsch_renderer* r, int32_t enabled) {
    return guarded([&] {
        if (!r) throw std::invalid_argument("null renderer");
        r->ctx->device_poses = enabled != 0;
    });
}

static RenderSettings to_settings(const gsch_render_settings* st) {
    RenderSettings rs;
    rs.tile_size = st->tile_size;
    rs.background = v3(st->background);
    rs.alpha_max = st->alpha_max;
    rs.alpha_cutoff = st->alpha_cutoff;
    rs.transmittance_floor = st->transmittance_floor;
    rs.thread_count = st->thread_count;
    rs.sh_colour = st->sh_colour != 0;
    return rs;
}

int gsch_psnr(const float* a, const float* b, uint32_t width, uint32_t height, float* out_db) {
    return guarded([&] {
        if (!a || !b || !out_db) throw std::invalid_argument("null argument");
        Framebuffer fa(static_cast<int>(width), static_cast<int>(height)), fb(static_cast<int>(width), static_cast<int>(height));
        std::memcpy(fa.rgb.data(), a, fa.rgb.size() * 4);
        std::memcpy(fb.rgb.data(), b, fb.rgb.size() * 4);
        *out_db = psnr(fa, fb);
    });
}

int gsch_lod_quality_sweep(gsch_scene* s, uint32_t template_id, const float* distances, uint32_t count,
                           const gsch_render_settings* st, int device, gsch_quality_row* rows, uint32_t capacity,
                           uint32_t* row_count) {
    return guarded([&] {
        if (!s || !st || (count && !distances) || !row_count) throw std::invalid_argument("null argument");
        if (template_id >= s->templates->size()) throw std::invalid_argument("template id beyond the store");
        const AvatarTemplate& tpl = (*s->templates)[template_id];
        *row_count = count * static_cast<uint32_t>(tpl.levels.size());
        if (!rows) return;  // size query
        if (capacity < *row_count) throw std::invalid_argument("row buffer too small");
        const QualityTable t = lod_quality_sweep(tpl, std::span<const float>(distances, count), s->camera,
                                                 to_settings(st), device);
        for (size_t i = 0; i < t.size(); ++i) {
            rows[i].distance_m = t[i].distance_m;
            rows[i].level = t[i].level;
            rows[i].gaussian_count = t[i].gaussian_count;
            rows[i].psnr_db = t[i].psnr_db;
        }
    });
}

int gsch_gather_splats(gsch_renderer* r, float time_s, int32_t static_pose, int32_t forced_lod,
                       const gsch_render_settings* st, gscg_frame_splat* out, uint64_t capacity, uint64_t* count) {
    return guarded([&] {
        if (!r || !st || !count) throw std::invalid_argument("null argument");
        std::optional<uint32_t> forced;
        if (forced_lod >= 0) forced = static_cast<uint32_t>(forced_lod);
        const SplatFrame f = gather_splats(r->scene->crowd, r->scene->camera, time_s, to_settings(st), static_pose != 0,
                                           forced, *r->ctx);
        *count = f.splats.size();
        if (out) {
            if (capacity < f.splats.size()) throw std::invalid_argument("splat buffer too small");
            std::memcpy(out, f.splats.data(), f.splats.size() * sizeof(gscg_frame_splat));
        }
    });
}

int gsch_sort_splats(gsch_renderer* r, gscg_frame_splat* splats, uint64_t n) {
    return guarded([&] {
        if (!r || (n && !splats)) throw std::invalid_argument("null argument");
        check_gscg(gscg_sort_splats(r->ctx->gpu(), splats, n), r->ctx->gpu());
    });
}

int gsch_rasterize_splats(gsch_renderer* r, const gscg_frame_splat* splats, uint64_t n, int32_t width, int32_t height,
                          const gsch_render_settings* st, float* out_rgb, float* out_T) {
    return guarded([&] {
        if (!r || !st || (n && !splats)) throw std::invalid_argument("null argument");
        const gscg_render_settings rs = [&] {
            gscg_render_settings x{};
            x.tile_size = st->tile_size;
            for (int i = 0; i < 3; ++i) x.background[i] = st->background[i];
            x.alpha_max = st->alpha_max;
            x.alpha_cutoff = st->alpha_cutoff;
            x.transmittance_floor = st->transmittance_floor;
            x.sh_enabled = st->sh_colour;
            return x;
        }();
        if (!(rs.alpha_max > 0.0f && rs.alpha_max <= 1.0f)) throw std::invalid_argument("RenderSettings: alpha_max outside (0,1]");
        check_gscg(gscg_rasterize_splats(r->ctx->gpu(), splats, n, width, height, &rs, out_rgb, out_T), r->ctx->gpu());
    });
}

static int render_host(gsch_renderer* r, float time_s, int32_t static_pose, int32_t forced_lod,
                       const gsch_render_settings* st, float* out_rgb, float* out_T, gsch_stage_times* times,
                       bool pipelined) {
    return guarded([&] {
        if (!r || !st) throw std::invalid_argument("null argument");
        RenderSettings rs;
        rs.tile_size = st->tile_size;
        rs.background = v3(st->background);
        rs.alpha_max = st->alpha_max;
        rs.alpha_cutoff = st->alpha_cutoff;
        rs.transmittance_floor = st->transmittance_floor;
        rs.thread_count = st->thread_count;
        rs.sh_colour = st->sh_colour != 0;
        StageTimes t;
        std::optional<uint32_t> forced;
        if (forced_lod >= 0) forced = static_cast<uint32_t>(forced_lod);
        (pipelined ? render_frame_async : render_frame_into)(r->scene->crowd, r->scene->camera, time_s, rs,
                                                             static_pose != 0, forced, &t, *r->ctx, out_rgb, out_T);
        if (times) {
            times->update_ms = t.update_ms;
            times->gather_ms = t.gather_ms;
            times->sort_ms = t.sort_ms;
            times->rasterize_ms = t.rasterize_ms;
            times->pose_ms = t.pose_ms;
            times->total_ms = t.total_ms();
            times->splat_count = t.splat_count;
            times->pair_count = t.pair_count;
            times->gaussian_count = t.gaussian_count;
            times->tile_pair_count = t.tile_pair_count;
        }
    });
}

int gsch_render(gsch_renderer* r, float time_s, int32_t static_pose, int32_t forced_lod,
                const gsch_render_settings* st, float* out_rgb, float* out_T, gsch_stage_times* times) {
    return render_host(r, time_s, static_pose, forced_lod, st, out_rgb, out_T, times, false);
}

int gsch_render_async(gsch_renderer* r, float time_s, int32_t static_pose, int32_t forced_lod,
                      const gsch_render_settings* st, float* out_rgb, float* out_T, gsch_stage_times* times) {
    return render_host(r, time_s, static_pose, forced_lod, st, out_rgb, out_T, times, true);
}

int gsch_wait_readback(gsch_renderer* r, uint32_t frames_back) {
    return guarded([&] {
        if (!r) throw std::invalid_argument("null argument");
        wait_readback(*r->ctx, frames_back);
    });
}

int gsch_sample_crowd(gsch_renderer* r, float time_s, int32_t static_pose, int32_t threads,
                      uint32_t* template_ids, float* placement, float* poses) {
    return guarded([&] {
        if (!r) throw std::invalid_argument("null renderer");
        FrameContext& c = *r->ctx;
        c.sample_crowd(r->scene->crowd, time_s, static_pose != 0, threads);
        const size_t n = r->scene->crowd.instances.size();
        if (template_ids) std::memcpy(template_ids, c.template_ids.data(), n * 4);
        if (placement) std::memcpy(placement, c.placement.data(), n * 16);
        if (poses) std::memcpy(poses, c.poses.data(), c.poses.size() * 4);
    });
}

}  // extern "C"
