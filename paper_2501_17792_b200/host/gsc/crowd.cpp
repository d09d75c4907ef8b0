// Crowd construction, LoD policy and memory accounting on the host. Follows
// /root/reference/proj/src/crowd.cpp (uniform01 :14-16, root_transform :20-30,
// validate(SceneConfig) :32-44, build_crowd :46-84, memory model :142-210) and
// /root/reference/proj/src/lod.cpp (validate :6-20, select_lod :22-37,
// instance_distance :39-41). update_crowd (its skinning runs on the GPU) is in renderer.cpp.
#include "gsc/crowd.hpp"

#include <cmath>
#include <random>
#include <set>
#include <stdexcept>

namespace gsc {

namespace {

float unit_draw(std::mt19937& gen) { return static_cast<float>(gen() >> 8) * 0x1.0p-24f; }

MemoryReport make_report(const MemoryLayoutModel& model, uint64_t resident,
                         uint64_t instance_gaussians, uint64_t instances) {
    MemoryReport r;
    r.instance_count = instances;
    r.fixed_overhead_bytes = model.fixed_overhead_bytes;
    r.resident_template_bytes = resident * model.template_bytes_per_gaussian();
    r.resident_channels = {resident * model.mean_bytes,    resident * model.rotation_bytes,
                           resident * model.scale_bytes,   resident * model.opacity_bytes,
                           resident * model.color_bytes,   resident * model.skin_index_bytes,
                           resident * model.skin_weight_bytes};
    const uint64_t base = model.fixed_overhead_bytes + r.resident_template_bytes;
    r.posed_mean_bytes = instance_gaussians * model.posed_bytes_per_gaussian();
    r.naive_bytes = base + instance_gaussians * model.template_bytes_per_gaussian();
    r.shared_bytes = base + r.posed_mean_bytes;
    r.savings_fraction = r.naive_bytes == 0
                             ? 0.0
                             : 1.0 - static_cast<double>(r.shared_bytes) /
                                         static_cast<double>(r.naive_bytes);
    if (instances > 0) {
        r.naive_marginal_bytes_per_instance =
            static_cast<double>(instance_gaussians * model.template_bytes_per_gaussian()) /
            static_cast<double>(instances);
        r.shared_marginal_bytes_per_instance =
            static_cast<double>(r.posed_mean_bytes) / static_cast<double>(instances);
    }
    return r;
}

void validate(const MemoryLayoutModel& model) {
    if (model.mean_bytes == 0 || model.rotation_bytes == 0 || model.scale_bytes == 0 ||
        model.opacity_bytes == 0 || model.color_bytes == 0 || model.skin_index_bytes == 0 ||
        model.skin_weight_bytes == 0)
        throw std::invalid_argument("MemoryLayoutModel: channel sizes must be > 0");
}

}  // namespace

void validate(const LodPolicy& policy) {
    for (size_t i = 0; i < policy.thresholds_m.size(); ++i) {
        const float t = policy.thresholds_m[i];
        if (!std::isfinite(t) || t <= 0.0f)
            throw std::invalid_argument("LodPolicy: thresholds must be positive and finite");
        if (i > 0 && t <= policy.thresholds_m[i - 1])
            throw std::invalid_argument("LodPolicy: thresholds must be strictly ascending");
    }
    if (!(policy.hysteresis_band_m >= 0.0f))
        throw std::invalid_argument("LodPolicy: hysteresis band must be >= 0");
}

uint32_t select_lod(const LodPolicy& policy, float distance_m,
                    std::optional<uint32_t> previous_level) {
    const size_t n = policy.thresholds_m.size();
    for (size_t k = 0; k < n; ++k) {
        float t = policy.thresholds_m[k];
        if (previous_level && policy.hysteresis_band_m > 0.0f)
            t += (k >= *previous_level ? 0.5f : -0.5f) * policy.hysteresis_band_m;
        if (distance_m < t) return static_cast<uint32_t>(k);
    }
    return static_cast<uint32_t>(n);
}

float instance_distance(const Vec3& p, const Vec3& cam) { return (p - cam).norm(); }

Mat4 CrowdInstance::root_transform() const {
    Mat4 m = Mat4::Identity();
    const float c = std::cos(yaw), s = std::sin(yaw);
    m(0, 0) = c;
    m(0, 2) = s;
    m(2, 0) = -s;
    m(2, 2) = c;
    m(0, 3) = x;
    m(2, 3) = z;
    return m;
}

void validate(const SceneConfig& cfg) {
    if (static_cast<uint64_t>(cfg.grid.rows) * cfg.grid.cols < cfg.crowd_count)
        throw std::invalid_argument("SceneConfig: grid capacity below crowd count");
    if (!(cfg.grid.spacing_m >= 0.0f))
        throw std::invalid_argument("SceneConfig: negative grid spacing");
    if (cfg.tile_size < 1) throw std::invalid_argument("SceneConfig: tile size must be >= 1");
    validate(cfg.lod);
    validate(cfg.camera.to_camera());
}

Crowd build_crowd(const SceneConfig& cfg, std::shared_ptr<const TemplateStore> templates,
                  std::shared_ptr<const MotionStore> motions, uint64_t seed) {
    validate(cfg);
    if (!templates || templates->empty()) throw std::invalid_argument("build_crowd: no templates");
    if (!motions || motions->empty()) throw std::invalid_argument("build_crowd: no motions");

    Crowd crowd;
    crowd.templates = std::move(templates);
    crowd.motions = std::move(motions);
    crowd.lod = cfg.lod;
    crowd.instances.resize(cfg.crowd_count);

    std::mt19937 gen(static_cast<uint32_t>(seed ^ (seed >> 32)));
    const float jitter = 0.25f * cfg.grid.spacing_m;
    const auto n_tpl = static_cast<uint32_t>(crowd.templates->size());
    const auto n_mot = static_cast<uint32_t>(crowd.motions->size());
    for (uint32_t i = 0; i < cfg.crowd_count; ++i) {
        CrowdInstance& inst = crowd.instances[i];
        inst.instance_id = i;
        inst.template_id = static_cast<uint32_t>(unit_draw(gen) * n_tpl);
        inst.motion_id = static_cast<uint32_t>(unit_draw(gen) * n_mot);
        inst.phase_offset_s = unit_draw(gen) * (*crowd.motions)[inst.motion_id].duration_s();
        const uint32_t row = i / cfg.grid.cols, col = i % cfg.grid.cols;
        inst.x = static_cast<float>(col) * cfg.grid.spacing_m + (2.0f * unit_draw(gen) - 1.0f) * jitter;
        inst.z = static_cast<float>(row) * cfg.grid.spacing_m + (2.0f * unit_draw(gen) - 1.0f) * jitter;
        inst.yaw = unit_draw(gen) * 6.28318530718f;
    }
    return crowd;
}

MemoryReport memory_report(const Crowd& crowd, const MemoryLayoutModel& model) {
    validate(model);
    std::set<std::pair<uint32_t, uint32_t>> residents;
    uint64_t instance_gaussians = 0;
    for (const CrowdInstance& inst : crowd.instances) {
        const AvatarTemplate& tpl = (*crowd.templates)[inst.template_id];
        const uint32_t lod = inst.active_lod == kLodUnset ? 0 : inst.active_lod;
        residents.emplace(inst.template_id, lod);
        instance_gaussians += tpl.levels[lod].gaussian_count();
    }
    uint64_t resident = 0;
    for (const auto& [tid, lod] : residents)
        resident += (*crowd.templates)[tid].levels[lod].gaussian_count();
    return make_report(model, resident, instance_gaussians, crowd.instances.size());
}

MemoryReport memory_report_cell(uint64_t instances, uint64_t gaussians,
                                const MemoryLayoutModel& model) {
    validate(model);
    return make_report(model, instances > 0 ? gaussians : 0, instances * gaussians, instances);
}

void update_crowd_lod(Crowd& crowd, const Camera& camera, std::optional<uint32_t> forced_lod) {
    const TemplateStore& templates = *crowd.templates;
    for (CrowdInstance& inst : crowd.instances) {
        if (inst.template_id >= templates.size()) throw std::invalid_argument("update_crowd: missing template");
        const AvatarTemplate& tpl = templates[inst.template_id];
        const uint32_t last = static_cast<uint32_t>(tpl.levels.size()) - 1;
        uint32_t lod;
        if (forced_lod) {
            lod = std::min(*forced_lod, last);
        } else {
            const Vec3 root_pos(inst.x, tpl.skeleton.bind[0].translation()[1], inst.z);
            const float dist = instance_distance(root_pos, camera.position);
            std::optional<uint32_t> prev;
            if (inst.active_lod != kLodUnset) prev = inst.active_lod;
            lod = std::min(select_lod(crowd.lod, dist, prev), last);
        }
        if (lod != inst.active_lod) {
            inst.active_lod = lod;
            inst.posed_valid = false;
        }
    }
}

}  // namespace gsc
