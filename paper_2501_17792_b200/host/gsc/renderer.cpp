// Host side of render_frame on the B200 (see renderer.hpp). Stage structure follows
// /root/reference/proj/src/renderer.cpp:249-280; the per-instance update follows
// /root/reference/proj/src/crowd.cpp:86-140 up to the pose (LoD, FK, skinning run on
// the GPU).
#include "gsc/renderer.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <string>

namespace gsc {

void validate(const RenderSettings& s) {
    if (s.tile_size < 1) throw std::invalid_argument("RenderSettings: tile_size must be >= 1");
    if (!(s.alpha_cutoff > 0.0f && s.alpha_cutoff < 1.0f))
        throw std::invalid_argument("RenderSettings: alpha_cutoff outside (0,1)");
    if (!(s.transmittance_floor > 0.0f && s.transmittance_floor < 1.0f))
        throw std::invalid_argument("RenderSettings: transmittance_floor outside (0,1)");
}

void check_gscg(int status, const gscg_ctx* ctx) {
    if (status == GSCG_OK) return;
    const std::string msg = ctx ? gscg_last_error(ctx) : "gscg call failed";
    if (status == GSCG_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (status == GSCG_ERR_OOM) throw std::bad_alloc();
    throw GpuError(status, msg);
}

HostPool::HostPool(unsigned threads) {
    for (unsigned i = 1; i < threads; ++i) workers_.emplace_back([this, i] { worker(i); });
}

HostPool::~HostPool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
        ++generation_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}

void HostPool::worker(unsigned index) {
    uint64_t seen = 0;
    for (;;) {
        const std::function<void(size_t, size_t)>* job;
        size_t count;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return generation_ != seen; });
            seen = generation_;
            if (stop_) return;
            job = job_;
            count = count_;
        }
        const size_t parts = size();
        const size_t chunk = (count + parts - 1) / parts;
        const size_t b = index * chunk, e = std::min(count, b + chunk);
        if (b < e) (*job)(b, e);
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
}

void HostPool::parallel_for(size_t count, const std::function<void(size_t, size_t)>& fn) {
    if (count == 0) return;
    if (workers_.empty() || count < 2) {
        fn(0, count);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(mu_);
        job_ = &fn;
        count_ = count;
        pending_ = static_cast<unsigned>(workers_.size());
        ++generation_;
    }
    cv_.notify_all();
    const size_t chunk = (count + size() - 1) / size();
    fn(0, std::min(count, chunk));
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
}

FrameContext::FrameContext(int device) {
    gscg_ctx* c = nullptr;
    const int st = gscg_create(device, &c);
    if (st != GSCG_OK) {
        std::string msg = c ? gscg_last_error(c) : "gscg_create failed";
        if (c) gscg_destroy(c);
        throw GpuError(st, msg);
    }
    gpu_ = c;
}

FrameContext::~FrameContext() {
    if (gpu_) gscg_destroy(gpu_);
}

void FrameContext::ensure_templates(const std::shared_ptr<const TemplateStore>& store) {
    if (store.get() == uploaded_) return;
    joint_stride = 0;
    for (uint32_t t = 0; t < store->size(); ++t) {
        const AvatarTemplate& tpl = (*store)[t];
        const Skeleton& sk = tpl.skeleton;
        const uint32_t J = sk.joint_count();
        joint_stride = std::max(joint_stride, J);
        std::vector<float> lb(J * 16), ib(J * 16);
        for (uint32_t j = 0; j < J; ++j) {
            std::copy(sk.local_bind[j].m, sk.local_bind[j].m + 16, lb.begin() + j * 16);
            std::copy(sk.inverse_bind[j].m, sk.inverse_bind[j].m + 16, ib.begin() + j * 16);
        }
        gscg_skeleton_desc sd{J, sk.parents.data(), lb.data(), ib.data(), sk.bind[0](1, 3)};
        check_gscg(gscg_upload_skeleton(gpu_, t, &sd), gpu_);
        for (uint32_t l = 0; l < tpl.levels.size(); ++l) {
            const LodLevel& lv = tpl.levels[l];
            if (lv.cov_cache.size() != lv.means.size())
                throw std::invalid_argument("LodLevel: finalize() not called");
            gscg_level_desc d{};
            d.gaussian_count = lv.gaussian_count();
            d.means = lv.means.empty() ? nullptr : lv.means[0].v;
            d.cov6 = lv.cov_cache[0].data();
            d.opacities = lv.opacities.data();
            d.colors = lv.colors[0].v;
            d.skin_indices = lv.skin_indices[0].data();
            d.skin_weights = lv.skin_weights[0].data();
            d.sh = lv.sh.empty() ? nullptr : lv.sh.data();
            check_gscg(gscg_upload_level(gpu_, t, l, &d), gpu_);
        }
    }
    uploaded_ = store.get();
    keep_ = store;
}

void sample_crowd_records(const Crowd& crowd, float time_s, bool static_pose, uint32_t joint_stride,
                          HostPool& pool, uint32_t* template_ids, float* placement, float* poses,
                          uint32_t* lods) {
    const size_t n = crowd.instances.size();
    const uint32_t rec = 4 + 4 * joint_stride;
    const TemplateStore& templates = *crowd.templates;
    const MotionStore& motions = *crowd.motions;
    for (const CrowdInstance& inst : crowd.instances) {
        if (inst.template_id >= templates.size() || inst.motion_id >= motions.size())
            throw std::invalid_argument("render_frame: instance references a missing asset");
        const uint32_t J = templates[inst.template_id].skeleton.joint_count();
        if (J > joint_stride) throw std::invalid_argument("joint_stride below the skeleton's joint count");
        if (!static_pose && motions[inst.motion_id].joint_count != J)
            throw std::invalid_argument("forward_kinematics: pose joint count mismatch");
        if (!static_pose && motions[inst.motion_id].frames.empty())
            throw std::invalid_argument("sample_pose: empty clip");
    }
    pool.parallel_for(n, [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i) {
            const CrowdInstance& inst = crowd.instances[i];
            template_ids[i] = inst.template_id;
            placement[i * 4 + 0] = inst.x;
            placement[i * 4 + 1] = inst.z;
            placement[i * 4 + 2] = std::cos(inst.yaw);
            placement[i * 4 + 3] = std::sin(inst.yaw);
            if (lods) lods[i] = inst.active_lod;
            float* rec_out = poses + i * rec;
            const uint32_t J = templates[inst.template_id].skeleton.joint_count();
            if (static_pose) {
                rec_out[0] = rec_out[1] = rec_out[2] = rec_out[3] = 0.0f;
                for (uint32_t j = 0; j < J; ++j) {
                    rec_out[4 + 4 * j + 0] = 0.0f;
                    rec_out[4 + 4 * j + 1] = 0.0f;
                    rec_out[4 + 4 * j + 2] = 0.0f;
                    rec_out[4 + 4 * j + 3] = 1.0f;
                }
            } else {
                sample_pose_into(motions[inst.motion_id], time_s + inst.phase_offset_s, true, rec_out,
                                 joint_stride);
            }
        }
    });
}

void FrameContext::ensure_motions(const std::shared_ptr<const MotionStore>& store) {
    if (!store || store.get() == motions_uploaded_) return;
    for (uint32_t m = 0; m < store->size(); ++m) {
        const MotionClip& clip = (*store)[m];
        if (clip.frames.empty()) continue;  // rejected per instance when sampled
        const uint32_t J = clip.joint_count;
        const size_t rec = 4 + 4 * static_cast<size_t>(J);
        std::vector<float> frames(clip.frames.size() * rec);
        for (size_t f = 0; f < clip.frames.size(); ++f) {
            float* r = frames.data() + f * rec;
            const Pose& p = clip.frames[f];
            r[0] = p.root_translation[0];
            r[1] = p.root_translation[1];
            r[2] = p.root_translation[2];
            r[3] = 0.0f;
            for (uint32_t j = 0; j < J; ++j)
                for (int k = 0; k < 4; ++k) r[4 + 4 * j + k] = p.local_rotations[j].c[k];
        }
        gscg_motion_desc d{};
        d.fps = clip.fps;
        d.frame_count = static_cast<uint32_t>(clip.frames.size());
        d.joint_count = J;
        d.frames = frames.data();
        check_gscg(gscg_upload_motion(gpu_, m, &d), gpu_);
    }
    motions_uploaded_ = store.get();
    keep_motions_ = store;
}

void FrameContext::fill_instances(const Crowd& crowd, bool static_pose) {
    const size_t n = crowd.instances.size();
    const TemplateStore& templates = *crowd.templates;
    const MotionStore& motions = *crowd.motions;
    template_ids.resize(n);
    placement.resize(n * 4);
    lods.resize(n);
    motion_ids.resize(n);
    phases.resize(n);
    for (size_t i = 0; i < n; ++i) {
        const CrowdInstance& inst = crowd.instances[i];
        if (inst.template_id >= templates.size() || inst.motion_id >= motions.size())
            throw std::invalid_argument("render_frame: instance references a missing asset");
        const uint32_t J = templates[inst.template_id].skeleton.joint_count();
        if (J > joint_stride) throw std::invalid_argument("joint_stride below the skeleton's joint count");
        if (!static_pose && motions[inst.motion_id].joint_count != J)
            throw std::invalid_argument("forward_kinematics: pose joint count mismatch");
        if (!static_pose && motions[inst.motion_id].frames.empty())
            throw std::invalid_argument("sample_pose: empty clip");
        template_ids[i] = inst.template_id;
        placement[i * 4 + 0] = inst.x;
        placement[i * 4 + 1] = inst.z;
        placement[i * 4 + 2] = std::cos(inst.yaw);
        placement[i * 4 + 3] = std::sin(inst.yaw);
        lods[i] = inst.active_lod;
        motion_ids[i] = inst.motion_id;
        phases[i] = inst.phase_offset_s;
    }
}

void FrameContext::sample_crowd(const Crowd& crowd, float time_s, bool static_pose,
                                int thread_hint) {
    const size_t n = crowd.instances.size();
    const uint32_t rec = 4 + 4 * joint_stride;
    template_ids.resize(n);
    placement.resize(n * 4);
    poses.resize(n * rec);
    lods.resize(n);
    const unsigned want = resolve_thread_count(thread_hint);
    if (!pool_ || pool_->size() != want) pool_ = std::make_unique<HostPool>(want);
    sample_crowd_records(crowd, time_s, static_pose, joint_stride, *pool_, template_ids.data(),
                         placement.data(), poses.data(), lods.data());
}

gscg_camera camera_basis(const Camera& cam) {
    gscg_camera c{};
    const Mat3 w = cam.view_rotation();
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) c.world_to_view[r * 3 + k] = w(r, k);
    for (int i = 0; i < 3; ++i) c.position[i] = cam.position[i];
    c.focal = cam.focal_px();
    c.cx = 0.5f * static_cast<float>(cam.width);
    c.cy = 0.5f * static_cast<float>(cam.height);
    c.near_m = cam.near_m;
    c.width = cam.width;
    c.height = cam.height;
    return c;
}

void render_frame(Crowd& crowd, const Camera& camera, float time_s,
                  const RenderSettings& settings, bool static_pose,
                  std::optional<uint32_t> forced_lod, StageTimes* times, FrameContext& ctx) {
    if (ctx.out.color.width != camera.width || ctx.out.color.height != camera.height) {
        ctx.out.color = Framebuffer(camera.width, camera.height);
        ctx.out.transmittance.assign(static_cast<size_t>(camera.width) * camera.height, 0.0f);
    }
    render_frame_into(crowd, camera, time_s, settings, static_pose, forced_lod, times, ctx,
                      ctx.out.color.rgb.data(), ctx.out.transmittance.data());
}

namespace {
void render_frame_host(Crowd& crowd, const Camera& camera, float time_s, const RenderSettings& settings,
                       bool static_pose, std::optional<uint32_t> forced_lod, StageTimes* times,
                       FrameContext& ctx, float* out_rgb, float* out_T, bool pipelined) {
    validate(settings);
    validate(camera);
    validate(crowd.lod);
    if (crowd.lod.thresholds_m.size() > GSCG_MAX_LOD_THRESHOLDS)
        throw std::invalid_argument("LodPolicy: too many thresholds for the GPU path");
    ctx.ensure_templates(crowd.templates);

    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    gscg_frame_desc fd{};
    if (ctx.device_poses) {
        ctx.ensure_motions(crowd.motions);
        ctx.fill_instances(crowd, static_pose);
        fd.pose_source = GSCG_POSES_SAMPLED;
        fd.time_s = time_s;
        fd.static_pose = static_pose ? 1 : 0;
        fd.motion_ids = ctx.motion_ids.data();
        fd.phase_offsets = ctx.phases.data();
    } else {
        ctx.sample_crowd(crowd, time_s, static_pose, settings.thread_count);
        fd.pose_source = GSCG_POSES_GIVEN;
        fd.poses = ctx.poses.data();
    }
    const auto t1 = clock::now();

    fd.instance_count = static_cast<uint32_t>(crowd.instances.size());
    fd.joint_stride = ctx.joint_stride;
    fd.template_ids = ctx.template_ids.data();
    fd.placement = ctx.placement.data();
    fd.active_lod = ctx.lods.data();
    fd.forced_lod = forced_lod ? static_cast<int32_t>(*forced_lod) : -1;
    fd.memory = GSCG_MEM_HOST;

    const gscg_camera cam = camera_basis(camera);
    gscg_render_settings rs{};
    rs.tile_size = settings.tile_size;
    for (int i = 0; i < 3; ++i) rs.background[i] = settings.background[i];
    rs.alpha_max = settings.alpha_max;
    rs.alpha_cutoff = settings.alpha_cutoff;
    rs.transmittance_floor = settings.transmittance_floor;
    rs.sh_enabled = settings.sh_colour ? 1 : 0;
    gscg_lod_policy lp{};
    lp.threshold_count = static_cast<uint32_t>(crowd.lod.thresholds_m.size());
    for (uint32_t i = 0; i < lp.threshold_count; ++i) lp.thresholds_m[i] = crowd.lod.thresholds_m[i];
    lp.hysteresis_band_m = crowd.lod.hysteresis_band_m;

    gscg_stage_times st{};
    check_gscg(pipelined ? gscg_render_frame_async(ctx.gpu(), &fd, &cam, &rs, &lp, out_rgb, out_T, &st)
                         : gscg_render_frame(ctx.gpu(), &fd, &cam, &rs, &lp, out_rgb, out_T, &st),
               ctx.gpu());
    for (size_t i = 0; i < crowd.instances.size(); ++i) {
        CrowdInstance& inst = crowd.instances[i];
        inst.active_lod = ctx.lods[i];
        // The frame's posed means live on the GPU: host copies from an earlier update_crowd
        // are stale now; gather_splats re-derives this frame's from the stamp.
        if (!inst.posed_means.empty()) inst.posed_means.clear();
        inst.posed_valid = false;
    }
    crowd.gpu_pose = Crowd::GpuPoseStamp{time_s, static_pose};

    if (times) {
        times->pose_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        times->update_ms = times->pose_ms + st.h2d_ms + st.update_ms;
        times->gather_ms = st.gather_ms;
        times->sort_ms = st.sort_ms;
        times->rasterize_ms = st.rasterize_ms + st.d2h_ms;
        times->splat_count = st.splat_count;
        times->pair_count = st.pair_count;
        times->gaussian_count = st.gaussian_count;
        times->tile_pair_count = st.tile_pair_count;
    }
}
}  // namespace

void render_frame_into(Crowd& crowd, const Camera& camera, float time_s, const RenderSettings& settings,
                       bool static_pose, std::optional<uint32_t> forced_lod, StageTimes* times,
                       FrameContext& ctx, float* out_rgb, float* out_T) {
    render_frame_host(crowd, camera, time_s, settings, static_pose, forced_lod, times, ctx, out_rgb, out_T, false);
}

void render_frame_async(Crowd& crowd, const Camera& camera, float time_s, const RenderSettings& settings,
                        bool static_pose, std::optional<uint32_t> forced_lod, StageTimes* times,
                        FrameContext& ctx, float* out_rgb, float* out_T) {
    render_frame_host(crowd, camera, time_s, settings, static_pose, forced_lod, times, ctx, out_rgb, out_T, true);
}

void wait_readback(FrameContext& ctx, uint32_t frames_back) {
    check_gscg(gscg_wait_readback(ctx.gpu(), frames_back), ctx.gpu());
}

static_assert(sizeof(FrameSplat) == sizeof(gscg_frame_splat), "FrameSplat mirrors gscg_frame_splat");

namespace {
gscg_render_settings to_gscg(const RenderSettings& settings) {
    gscg_render_settings rs{};
    rs.tile_size = settings.tile_size;
    for (int i = 0; i < 3; ++i) rs.background[i] = settings.background[i];
    rs.alpha_max = settings.alpha_max;
    rs.alpha_cutoff = settings.alpha_cutoff;
    rs.transmittance_floor = settings.transmittance_floor;
    rs.sh_enabled = settings.sh_colour ? 1 : 0;
    return rs;
}
}  // namespace

SplatFrame gather_splats(Crowd& crowd, const Camera& camera, float time_s, const RenderSettings& settings,
                         bool static_pose, std::optional<uint32_t> forced_lod, FrameContext& ctx) {
    validate(settings);
    validate(camera);
    validate(crowd.lod);
    ctx.ensure_templates(crowd.templates);
    ctx.sample_crowd(crowd, time_s, static_pose, settings.thread_count);
    gscg_frame_desc fd{};
    fd.instance_count = static_cast<uint32_t>(crowd.instances.size());
    fd.joint_stride = ctx.joint_stride;
    fd.template_ids = ctx.template_ids.data();
    fd.placement = ctx.placement.data();
    fd.poses = ctx.poses.data();
    fd.active_lod = ctx.lods.data();
    fd.forced_lod = forced_lod ? static_cast<int32_t>(*forced_lod) : -1;
    fd.memory = GSCG_MEM_HOST;
    const gscg_camera cam = camera_basis(camera);
    const gscg_render_settings rs = to_gscg(settings);
    gscg_lod_policy lp{};
    lp.threshold_count = static_cast<uint32_t>(crowd.lod.thresholds_m.size());
    for (uint32_t i = 0; i < lp.threshold_count; ++i) lp.thresholds_m[i] = crowd.lod.thresholds_m[i];
    lp.hysteresis_band_m = crowd.lod.hysteresis_band_m;
    uint64_t count = 0;
    const std::vector<uint32_t> prev_lods = ctx.lods;  // both calls see the same LoD history
    check_gscg(gscg_gather_splats(ctx.gpu(), &fd, &cam, &rs, &lp, nullptr, 0, &count), ctx.gpu());
    ctx.lods = prev_lods;
    fd.active_lod = ctx.lods.data();
    SplatFrame frame;
    frame.width = camera.width;
    frame.height = camera.height;
    frame.splats.resize(count);
    // second call returns the records of the same projection (deterministic)
    check_gscg(gscg_gather_splats(ctx.gpu(), &fd, &cam, &rs, &lp,
                                  reinterpret_cast<gscg_frame_splat*>(frame.splats.data()), count, &count),
               ctx.gpu());
    for (size_t i = 0; i < crowd.instances.size(); ++i) crowd.instances[i].active_lod = ctx.lods[i];
    return frame;
}

void sort_splats(SplatFrame& frame, FrameContext& ctx) {
    check_gscg(gscg_sort_splats(ctx.gpu(), reinterpret_cast<gscg_frame_splat*>(frame.splats.data()),
                                frame.splats.size()),
               ctx.gpu());
}

FrameContext& default_frame_context() {
    // One context per host thread (a gscg context is not thread-safe), never destroyed:
    // process teardown may already have unloaded the CUDA runtime.
    thread_local FrameContext* ctx = [] {
        const char* env = std::getenv("GSCG_DEVICE");
        return new FrameContext(env ? std::atoi(env) : 0);
    }();
    return *ctx;
}

void update_crowd(Crowd& crowd, const Camera& camera, const UpdateOptions& opts) {
    update_crowd(crowd, camera, opts, default_frame_context());
}

void update_crowd(Crowd& crowd, const Camera& camera, const UpdateOptions& opts, FrameContext& ctx) {
    if (opts.skin_rotations)
        throw std::invalid_argument("update_crowd: rotation skinning is not supported by the B200 path");
    const TemplateStore& templates = *crowd.templates;
    update_crowd_lod(crowd, camera, opts.forced_lod);
    bool stale = false;
    for (const CrowdInstance& inst : crowd.instances) {
        // crowd.cpp:112-116: a static instance with valid posed means is left alone.
        if (!(opts.static_pose && inst.posed_valid &&
              inst.posed_means.size() == templates[inst.template_id].levels[inst.active_lod].gaussian_count()))
            stale = true;
    }
    crowd.gpu_pose.reset();
    if (!stale) return;
    // Pose + FK + skin matrices + LBS of every instance's active level on the GPU.
    ctx.ensure_templates(crowd.templates);
    ctx.sample_crowd(crowd, opts.time_s, opts.static_pose, opts.thread_count);
    const uint32_t n = static_cast<uint32_t>(crowd.instances.size());
    gscg_frame_desc fd{};
    fd.instance_count = n;
    fd.joint_stride = ctx.joint_stride;
    fd.template_ids = ctx.template_ids.data();
    fd.placement = ctx.placement.data();
    fd.poses = ctx.poses.data();
    fd.active_lod = ctx.lods.data();
    fd.forced_lod = GSCG_LOD_GIVEN;
    fd.memory = GSCG_MEM_HOST;
    const gscg_camera cam = camera_basis(camera);
    gscg_lod_policy lp{};
    uint64_t G = 0;
    for (const CrowdInstance& inst : crowd.instances)
        G += templates[inst.template_id].levels[inst.active_lod].gaussian_count();
    std::vector<float> posed(std::max<uint64_t>(G, 1) * 3);
    uint64_t got = 0;
    check_gscg(gscg_skin_means(ctx.gpu(), &fd, &cam, &lp, posed.data(), G, &got), ctx.gpu());
    if (got != G) throw GpuError(GSCG_ERR_STATE, "update_crowd: instance-Gaussian count mismatch");
    size_t off = 0;
    for (CrowdInstance& inst : crowd.instances) {
        const size_t cnt = templates[inst.template_id].levels[inst.active_lod].gaussian_count();
        inst.posed_means.resize(cnt);
        for (size_t g = 0; g < cnt; ++g)
            inst.posed_means[g] = Vec3(posed[3 * (off + g)], posed[3 * (off + g) + 1], posed[3 * (off + g) + 2]);
        off += cnt;
        inst.posed_rotations.clear();
        inst.posed_valid = opts.static_pose;
    }
}

void gather_splats(const Crowd& crowd, const Camera& camera, int thread_count, FrameContext& ctx) {
    ctx.frame.width = camera.width;
    ctx.frame.height = camera.height;
    ctx.frame.splats.clear();
    ctx.ensure_templates(crowd.templates);
    const bool none_posed = std::all_of(crowd.instances.begin(), crowd.instances.end(),
                                        [](const CrowdInstance& i) { return i.posed_means.empty(); });
    if (crowd.gpu_pose && none_posed && !crowd.instances.empty()) {
        // After render_frame: the posed means of that frame (its time, its levels) are
        // re-derived on the GPU; identical to what update_crowd would have left behind.
        ctx.sample_crowd(crowd, crowd.gpu_pose->time_s, crowd.gpu_pose->static_pose, thread_count);
        gscg_frame_desc fd{};
        fd.instance_count = static_cast<uint32_t>(crowd.instances.size());
        fd.joint_stride = ctx.joint_stride;
        fd.template_ids = ctx.template_ids.data();
        fd.placement = ctx.placement.data();
        fd.poses = ctx.poses.data();
        fd.active_lod = ctx.lods.data();
        fd.forced_lod = GSCG_LOD_GIVEN;
        fd.memory = GSCG_MEM_HOST;
        const gscg_camera cam = camera_basis(camera);
        const gscg_render_settings rs = to_gscg(RenderSettings{});
        gscg_lod_policy lp{};
        uint64_t count = 0;
        check_gscg(gscg_gather_splats(ctx.gpu(), &fd, &cam, &rs, &lp, nullptr, 0, &count), ctx.gpu());
        ctx.frame.splats.resize(count);
        check_gscg(gscg_gather_splats(ctx.gpu(), &fd, &cam, &rs, &lp,
                                      reinterpret_cast<gscg_frame_splat*>(ctx.frame.splats.data()), count, &count),
                   ctx.gpu());
        return;
    }
    const TemplateStore& templates = *crowd.templates;
    const uint32_t n = static_cast<uint32_t>(crowd.instances.size());
    std::vector<uint32_t> tids(std::max<uint32_t>(n, 1)), lods(std::max<uint32_t>(n, 1)), mask(std::max<uint32_t>(n, 1));
    std::vector<float> place(std::max<uint32_t>(n, 1) * 4, 0.0f);
    uint64_t G = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const CrowdInstance& inst = crowd.instances[i];
        if (inst.template_id >= templates.size()) throw std::invalid_argument("gather_splats: missing template");
        const AvatarTemplate& tpl = templates[inst.template_id];
        const uint32_t lod = std::min<uint32_t>(inst.active_lod == kLodUnset ? 0 : inst.active_lod,
                                                static_cast<uint32_t>(tpl.levels.size()) - 1);
        const uint32_t cnt = tpl.levels[lod].gaussian_count();
        if (!inst.posed_means.empty() && inst.posed_means.size() != cnt)
            throw std::invalid_argument("gather_splats: posed_means do not match the active level (run update_crowd)");
        tids[i] = inst.template_id;
        lods[i] = inst.active_lod;
        mask[i] = inst.posed_means.empty() ? 0u : 1u;  // renderer.cpp:41: n = posed_means.size()
        G += cnt;
    }
    std::vector<float> posed(std::max<uint64_t>(G, 1) * 3, 0.0f);
    size_t off = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const CrowdInstance& inst = crowd.instances[i];
        const AvatarTemplate& tpl = templates[inst.template_id];
        const uint32_t lod = std::min<uint32_t>(inst.active_lod == kLodUnset ? 0 : inst.active_lod,
                                                static_cast<uint32_t>(tpl.levels.size()) - 1);
        for (size_t g = 0; g < inst.posed_means.size(); ++g)
            for (int k = 0; k < 3; ++k) posed[3 * (off + g) + k] = inst.posed_means[g][k];
        off += tpl.levels[lod].gaussian_count();
    }
    gscg_frame_desc fd{};
    fd.instance_count = n;
    fd.joint_stride = ctx.joint_stride;
    fd.template_ids = tids.data();
    fd.placement = place.data();
    fd.active_lod = lods.data();
    fd.forced_lod = GSCG_LOD_GIVEN;
    fd.memory = GSCG_MEM_HOST;
    const gscg_camera cam = camera_basis(camera);
    const gscg_render_settings rs = to_gscg(RenderSettings{});  // colour as render_frame's defaults
    uint64_t count = 0;
    check_gscg(gscg_gather_posed(ctx.gpu(), &fd, posed.data(), G, mask.data(), &cam, &rs, nullptr, 0, &count),
               ctx.gpu());
    ctx.frame.splats.resize(count);
    check_gscg(gscg_gather_posed(ctx.gpu(), &fd, posed.data(), G, mask.data(), &cam, &rs,
                                 reinterpret_cast<gscg_frame_splat*>(ctx.frame.splats.data()), count, &count),
               ctx.gpu());
}

SplatFrame gather_splats(const Crowd& crowd, const Camera& camera, int thread_count) {
    FrameContext& ctx = default_frame_context();
    gather_splats(crowd, camera, thread_count, ctx);
    return std::move(ctx.frame);
}

void sort_splats(SplatFrame& frame) { sort_splats(frame, default_frame_context()); }

void sort_splats(FrameContext& ctx) { sort_splats(ctx.frame, ctx); }

void rasterize_full(const SplatFrame& frame, const RenderSettings& settings, int width, int height,
                    FrameContext& ctx) {
    validate(settings);
    if (width != frame.width || height != frame.height)
        throw std::invalid_argument("rasterize: splat frame was gathered for another size");
    if (ctx.out.color.width != width || ctx.out.color.height != height) {
        ctx.out.color = Framebuffer(width, height);
        ctx.out.transmittance.assign(static_cast<size_t>(width) * height, 0.0f);
    }
    const gscg_render_settings rs = to_gscg(settings);
    check_gscg(gscg_rasterize_splats(ctx.gpu(), reinterpret_cast<const gscg_frame_splat*>(frame.splats.data()),
                                     frame.splats.size(), width, height, &rs, ctx.out.color.rgb.data(),
                                     ctx.out.transmittance.data()),
               ctx.gpu());
}

RasterOutput rasterize_full(const SplatFrame& frame, const RenderSettings& settings, int width, int height) {
    FrameContext& ctx = default_frame_context();
    rasterize_full(frame, settings, width, height, ctx);
    RasterOutput out;
    out.color = std::move(ctx.out.color);
    out.transmittance = std::move(ctx.out.transmittance);
    ctx.out = RasterOutput{};
    return out;
}

Framebuffer rasterize(const SplatFrame& frame, const RenderSettings& settings, int width, int height,
                      FrameContext& ctx) {
    rasterize_full(frame, settings, width, height, ctx);
    Framebuffer fb = std::move(ctx.out.color);
    ctx.out = RasterOutput{};
    return fb;
}

Framebuffer rasterize(const SplatFrame& frame, const RenderSettings& settings, int width, int height) {
    return rasterize(frame, settings, width, height, default_frame_context());
}

Framebuffer render_frame(Crowd& crowd, const Camera& camera, float time_s,
                         const RenderSettings& settings, bool static_pose,
                         std::optional<uint32_t> forced_lod, StageTimes* times) {
    FrameContext ctx;
    render_frame(crowd, camera, time_s, settings, static_pose, forced_lod, times, ctx);
    return std::move(ctx.out.color);
}

}  // namespace gsc
