// render_frame on the B200: host mirror of /root/reference/proj/include/gsc/renderer.hpp
// (RenderSettings :15-22, Framebuffer :26-37, RasterOutput :52-55, FrameContext :57-79,
// StageTimes :105-112, render_frame :114-123). The host samples poses (the only
// transcendental-heavy step, kept on glibc for bit-exact parity) on a persistent
// thread pool and hands everything else to the GPU through the gscg C-ABI
// (include/gscg.h). There is no CPU fallback: construction fails without a GPU.
#pragma once

#include "gsc/crowd.hpp"
#include "gsc/parallel.hpp"
#include "gscg.h"

#include <condition_variable>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <thread>

namespace gsc {

struct RenderSettings {
    int tile_size = 16;
    Vec3 background = Vec3::Zero();
    float alpha_max = kAlphaMax;
    float alpha_cutoff = kAlphaCutoff;
    float transmittance_floor = 1e-4f;
    int thread_count = 0;  // host pose-sampling threads; 0 = GSCROWD_THREADS / hardware
    bool sh_colour = true; // evaluate the SH residual when templates carry it
};

void validate(const RenderSettings& s);

struct Framebuffer {
    int width = 0;
    int height = 0;
    std::vector<float> rgb;
    Framebuffer() = default;
    Framebuffer(int w, int h) : width(w), height(h), rgb(static_cast<size_t>(w) * h * 3, 0.0f) {}
    float* pixel(int x, int y) { return rgb.data() + 3 * (static_cast<size_t>(y) * width + x); }
    const float* pixel(int x, int y) const {
        return rgb.data() + 3 * (static_cast<size_t>(y) * width + x);
    }
};

// Projected splats (reference math.hpp:64-79, renderer.hpp:39-50). FrameSplat is laid
// out exactly as gscg_frame_splat (64 bytes).
struct Splat2D {
    Vec2 mean_px;
    float cov_xx = 1.0f;
    float cov_xy = 0.0f;
    float cov_yy = 1.0f;
    float depth = 0.0f;  // view-space z, meters
    Vec3 color = Vec3::Ones();
    float opacity = 1.0f;
};

struct FrameSplat {
    Splat2D splat;
    uint32_t instance_id = 0;
    uint32_t gaussian_index = 0;
    PixelRect bounds;  // 3-sigma rectangle clipped to the image
};

struct SplatFrame {
    int width = 0;
    int height = 0;
    std::vector<FrameSplat> splats;
};

struct RasterOutput {
    Framebuffer color;
    std::vector<float> transmittance;
};

struct StageTimes {
    double update_ms = 0.0;     // host pose sampling + H2D + LoD/FK kernels
    double gather_ms = 0.0;     // LBS + projection + pair emission
    double sort_ms = 0.0;       // radix sort + tile ranges
    double rasterize_ms = 0.0;  // tile blend + D2H
    double pose_ms = 0.0;       // host part of update
    double total_ms() const { return update_ms + gather_ms + sort_ms + rasterize_ms; }
    uint64_t splat_count = 0;
    uint64_t pair_count = 0;
    uint64_t gaussian_count = 0;
    uint64_t tile_pair_count = 0;  // the reference's per-tile bin entries (renderer.cpp:147-161)
};

// Error from the C-ABI, rethrown as the reference's exception types.
struct GpuError : std::runtime_error {
    int status;
    GpuError(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
void check_gscg(int status, const gscg_ctx* ctx);

// Static-partition fork/join over persistent threads (the reference spawns threads per
// call, parallel.hpp:26-42; the partition is the same contiguous chunking).
class HostPool {
public:
    explicit HostPool(unsigned threads);
    ~HostPool();
    unsigned size() const { return static_cast<unsigned>(workers_.size()) + 1; }
    void parallel_for(size_t count, const std::function<void(size_t, size_t)>& fn);

private:
    void worker(unsigned index);
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(size_t, size_t)>* job_ = nullptr;
    size_t count_ = 0;
    uint64_t generation_ = 0;
    unsigned pending_ = 0;
    bool stop_ = false;
};

// Per-instance pose records for the GPU (update_crowd up to the pose, crowd.cpp:118-124):
// template ids, placement (x, z, cos yaw, sin yaw) and sampled poses, on the pool.
void sample_crowd_records(const Crowd& crowd, float time_s, bool static_pose, uint32_t joint_stride,
                          HostPool& pool, uint32_t* template_ids, float* placement, float* poses,
                          uint32_t* lods);

class FrameContext {
public:
    explicit FrameContext(int device = 0);
    ~FrameContext();
    FrameContext(const FrameContext&) = delete;
    FrameContext& operator=(const FrameContext&) = delete;

    gscg_ctx* gpu() { return gpu_; }
    // Uploads the store once per pointer identity (shared-attribute residency).
    void ensure_templates(const std::shared_ptr<const TemplateStore>& store);
    // Uploads every clip once per store identity (device pose sampling tables).
    void ensure_motions(const std::shared_ptr<const MotionStore>& store);
    // Fills the per-frame pose / placement records for the whole crowd on the pool.
    void sample_crowd(const Crowd& crowd, float time_s, bool static_pose, int thread_hint);
    // Device pose sampling mode: per frame only placement, motion ids and phase offsets
    // go to the GPU, which samples every clip itself (bit-identical to the host path).
    void fill_instances(const Crowd& crowd, bool static_pose);

    // The reference's FrameContext members a caller reads (renderer.hpp:57-79): the
    // gathered / sorted splat frame of the stage functions and the framebuffer + T.
    SplatFrame frame;
    RasterOutput out;
    std::vector<uint32_t> template_ids;
    std::vector<float> placement;  // n x 4
    std::vector<float> poses;      // n x (4 + 4 * joint_stride)
    std::vector<uint32_t> lods;
    std::vector<uint32_t> motion_ids;
    std::vector<float> phases;
    uint32_t joint_stride = 0;
    bool device_poses = false;  // sample poses on the GPU (GSCG_POSES_SAMPLED)

private:
    gscg_ctx* gpu_ = nullptr;
    const TemplateStore* uploaded_ = nullptr;
    std::shared_ptr<const TemplateStore> keep_;
    const MotionStore* motions_uploaded_ = nullptr;
    std::shared_ptr<const MotionStore> keep_motions_;
    std::unique_ptr<HostPool> pool_;
};

gscg_camera camera_basis(const Camera& cam);

void render_frame(Crowd& crowd, const Camera& camera, float time_s,
                  const RenderSettings& settings, bool static_pose,
                  std::optional<uint32_t> forced_lod, StageTimes* times, FrameContext& ctx);

// Same frame, written straight into caller buffers (width*height*3 RGB and width*height
// transmittance; either may be null). Pinned (page-locked) buffers get a direct DMA.
void render_frame_into(Crowd& crowd, const Camera& camera, float time_s, const RenderSettings& settings,
                       bool static_pose, std::optional<uint32_t> forced_lod, StageTimes* times,
                       FrameContext& ctx, float* out_rgb, float* out_T);
// Streaming form of render_frame_into (gscg_render_frame_async): returns once the frame is
// rendered; out_rgb / out_T fill in the background while the next frame renders and are
// valid after wait_readback(ctx, frames_back) (0 = the last submitted frame).
void render_frame_async(Crowd& crowd, const Camera& camera, float time_s, const RenderSettings& settings,
                        bool static_pose, std::optional<uint32_t> forced_lod, StageTimes* times,
                        FrameContext& ctx, float* out_rgb, float* out_T);
void wait_readback(FrameContext& ctx, uint32_t frames_back);

// The calling thread's GPU context (device 0, or GSCG_DEVICE), created on first use: the
// reference's stage functions below take no FrameContext, or a reference-shaped one.
FrameContext& default_frame_context();

// update_crowd on an explicit context (the crowd.hpp form uses default_frame_context()).
void update_crowd(Crowd& crowd, const Camera& camera, const UpdateOptions& opts, FrameContext& ctx);

// ---- Stage functions, reference signatures (renderer.hpp:81-103), on the GPU ----
// gather_splats projects every instance's posed_means (filled by update_crowd) with its
// active level's covariance, colour and opacity; survivors in (instance, gaussian) order.
SplatFrame gather_splats(const Crowd& crowd, const Camera& camera, int thread_count = 0);
void gather_splats(const Crowd& crowd, const Camera& camera, int thread_count, FrameContext& ctx);  // -> ctx.frame
// Ascending depth bits, ties by (instance_id, gaussian_index): a stable GPU radix sort.
void sort_splats(SplatFrame& frame);
void sort_splats(FrameContext& ctx);  // ctx.frame in place
// Conic prep, tile binning in the given splat order, per-tile front-to-back blending.
Framebuffer rasterize(const SplatFrame& frame, const RenderSettings& settings, int width, int height);
RasterOutput rasterize_full(const SplatFrame& frame, const RenderSettings& settings, int width, int height);
void rasterize_full(const SplatFrame& frame, const RenderSettings& settings, int width, int height,
                    FrameContext& ctx);  // -> ctx.out

// Explicit-context variants: the fused update + gather of one time step (the reference's
// update_crowd then gather_splats, without host posed means), and sort / raster on ctx.
SplatFrame gather_splats(Crowd& crowd, const Camera& camera, float time_s, const RenderSettings& settings,
                         bool static_pose, std::optional<uint32_t> forced_lod, FrameContext& ctx);
void sort_splats(SplatFrame& frame, FrameContext& ctx);
Framebuffer rasterize(const SplatFrame& frame, const RenderSettings& settings, int width, int height,
                      FrameContext& ctx);

Framebuffer render_frame(Crowd& crowd, const Camera& camera, float time_s,
                         const RenderSettings& settings, bool static_pose = false,
                         std::optional<uint32_t> forced_lod = std::nullopt,
                         StageTimes* times = nullptr);

}  // namespace gsc
