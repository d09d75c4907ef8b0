// C-ABI of the B200 crowd-render path (include/gscg.h): context, shared attribute store
// upload, per-frame orchestration and parity exports.
//
// Frame schedule on the context stream (render_frame, renderer.cpp:249-280):
//   H2D of the frame records (pinned staging, one copy)
//   update:    k_fk_skin -> k_inst_cull -> k_lod_plan (1 CTA)
//   gather:    k_project (persistent, template-major)       -> counters readback (sync)
//   sort:      splats by the top <= 25 varying depth bits (k_sort_{upsweep,rows,downsweep} x P) ->
//              spans in sorted order (k_sorted_spans) ->
//              pairs scattered in first-cell-pass order, keys tagged with the truncated depth
//              (k_emit_scatter count, k_sort_rows, k_emit_scatter scatter) ->
//              pairs stably by cell (radix x P') -> cell ranges + per-cell (depth, ordinal)
//              order of tied runs (k_cell_fixup, k_pair_long_runs)
//   rasterize: k_raster16q (or k_raster_generic for other tile sizes)
//   D2H of framebuffer / transmittance / active LoDs (host mode)
// The one mid-frame synchronisation reads S, K and the depth-bit range: it sizes the
// sort and detects capacity overflow (buffers grow to the high-water mark and the
// gather is replayed, as the reference's buffers grow, crowd.hpp:26-28).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gscg_common.cuh"
#include "gscg_kernels.h"

using namespace gscg;

// PDL is used for frames of up to kPdlMaxSplats splats (the previous frame's count). With
// the bucket depth sort it pays on every BASELINE config (config 3: 546 vs 539 FPS device,
// 548 vs 528 e2e); the cut stays as a knob for A/B runs.
constexpr uint64_t kPdlMaxSplats = ~0ull;
uint64_t pdl_max_splats() {  // GSCG_PDL_MAX_SPLATS overrides the cut (A/B measurements)
    static const uint64_t v = [] {
        const char* e = std::getenv("GSCG_PDL_MAX_SPLATS");
        return e ? std::strtoull(e, nullptr, 10) : kPdlMaxSplats;
    }();
    return v;
}
thread_local bool t_pdl_frame = true;
// Frame pipelining of render_frame (see gscg_ctx::upd_stream); GSCG_OVERLAP_UPDATE=0 keeps
// every frame on one stream (A/B).
constexpr uint64_t kPipelineMaxSplats = 64000000;
bool overlap_update() {
    static const bool on = [] {
        const char* e = std::getenv("GSCG_OVERLAP_UPDATE");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool gscg::pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("GSCG_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on && t_pdl_frame;
}

namespace {

// Device buffer owned by the context: grow-only, freed on release() or destruction (so
// every buffer a context ever grew goes with gscg_destroy).
struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), cap(o.cap) {
        o.ptr = nullptr;
        o.cap = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            ptr = o.ptr;
            cap = o.cap;
            o.ptr = nullptr;
            o.cap = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
    // Grow-only; contents are not preserved.
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && ptr) return cudaSuccess;
        release();
        const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e != cudaSuccess) {
            ptr = nullptr;
            return e;
        }
        cap = want;
        return cudaSuccess;
    }
    // Exactly `bytes` (the shared template store is sized once, without growth slack).
    cudaError_t ensure_exact(size_t bytes) {
        if (ptr && cap == bytes) return cudaSuccess;
        release();
        cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(bytes, 16));
        if (e != cudaSuccess) {
            ptr = nullptr;
            return e;
        }
        cap = bytes;
        return cudaSuccess;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
};

// Varying depth bits the splat sort orders (LSD passes of <= 5 bits); the lower bits and
// the ordinal tie-break are settled per cell by k_cell_fixup.
constexpr uint32_t kDepthSortBits = 25;
// Frames past this many splats take the LSD depth passes: the average bucket outgrows the
// coalesced local sort. Measured sort stage: config 3 (10.9 M) 0.99 -> 0.82 ms, config 4
// (25.7 M, 2^15 buckets) 2.59 -> 2.40 ms, config 5 (519 M) 51 vs 85 ms in favour of LSD.
constexpr uint64_t kBucketMaxSplats = 40000000;
constexpr uint32_t kBucketWideSplats = 16000000;  // frames past this use 2^15 top-level buckets

struct LevelStore {
    uint32_t count = 0;
    DevBuf core, weights, sh;
    bool has_sh = false;
    std::vector<float> opacities;  // host copy for the power-floor table
    float pf_cutoff = -1.0f;
    // Instance-cull bounds (k_inst_cull): max |mean|, max sqrt of the Gershgorin bound of
    // the covariance, max sum |w|, max |sum w - 1|; +inf when any input is non-finite.
    float mean_r = 0.0f, sigma = 0.0f, wabs = 0.0f, wdev = 0.0f;
};

// A clip as device slerp tables (gscg_pose.cu): roots per frame, key pairs per
// (frame, joint) with the host-libm acos/sin of the pair angle.
struct MotionStore {
    float fps = 0.0f;
    uint32_t frames = 0, joints = 0;
    std::vector<float4> roots;
    std::vector<KeyPairDev> keys;
};

struct TemplateStore {
    bool present = false;
    uint32_t joint_count = 0;
    std::vector<int16_t> parents;
    std::vector<float> local_bind, inverse_bind;
    float pelvis_y = 0.0f;
    std::vector<LevelStore> levels;
};

struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            throw Status(_e == cudaErrorMemoryAllocation ? GSCG_ERR_OOM : GSCG_ERR_CUDA,   \
                         std::string(#expr) + ": " + cudaGetErrorString(_e));             \
    } while (0)

}  // namespace

struct FrameGeom {
    int W = 0, H = 0, ts = 16, tiles_x = 0, tiles_y = 0, cell = 8;
    uint32_t cells_per_tile = 1;
    // The region rendered: the frame, or gscg_set_region's rectangle (tile-aligned).
    int band_x0 = 0, band_y0 = 0, band_x1 = 0, band_y1 = 0;
    int band_tile_col0 = 0, band_tiles_x = 0, band_tile_row0 = 0, band_tile_rows = 0;
};

struct gscg_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    std::string error;
    uint32_t debug = 0;
    // gscg_set_region request: rows [band_req0, band_req1) (empty: every row) x columns
    // [col_req0, col_req1) (col_req1 <= 0: every column).
    int32_t band_req0 = 0, band_req1 = 0, col_req0 = 0, col_req1 = 0;

    std::vector<TemplateStore> templates;
    std::vector<MotionStore> motions;
    bool motions_dirty = false;
    DevBuf d_motions, d_roots, d_keys, motion_ids, phases;
    bool tables_dirty = true;
    DevBuf d_templates, d_groups, d_mats, d_parents;
    uint32_t group_count = 0;
    uint32_t joint_stride = 0;

    // frame inputs
    DevBuf template_ids, placement, poses, lod_prev, lod_out;
    // plan outputs
    DevBuf inst_group, inst_base, members, group_inst_start, group_inst_count, group_item_start, visible;
    DevBuf skin, counters;
    // gather outputs
    // Per-splat outputs of the projection, one set per frame slot: with frame pipelining the
    // next frame's projection writes one slot while this frame's sort and raster read the other.
    DevBuf records_s[2], splat_meta_s[2], splat_depth_s[2];
    int slot = 0;
    DevBuf& rec() { return records_s[slot]; }
    DevBuf& meta() { return splat_meta_s[slot]; }
    DevBuf& depth() { return splat_depth_s[slot]; }
    uint64_t splat_capacity = 0, pair_capacity = 0;
    uint32_t culled = 0;  // instances dropped by k_inst_cull in the last frame
    uint32_t depth_sort_bits = kDepthSortBits;  // top varying depth bits the splat sort orders
    uint64_t bucket_max_splats = kBucketMaxSplats;  // largest frame the bucket depth sort takes
    uint32_t dbits_prev = kDepthSortBits;       // varying depth bits of the last settled frame
    uint32_t deferred_depth_top = 32;           // key bits a deferred frame's depth plan covers
    cudaEvent_t counters_ev = nullptr;          // the frame's counters are in h_counters
    // Frame pipelining (render_frame): a frame's front half (H2D, poses, FK, cull, plan,
    // projection, counters, LoD write-back) runs on upd_stream, its back half (sort, raster,
    // read-back) on `stream`, so the next frame's front half runs under this frame's back
    // half. The projection writes the frame's slot (records / meta / depth), which the back
    // half of the frame two back read: slot_free[slot] marks that raster's end. upd_done
    // marks the end of the last front half (later work on `stream` waits for it); upd_ok the
    // tail of `stream` a first front half waits for.
    cudaStream_t upd_stream = nullptr, sort_stream = nullptr;  // front halves; a pipelined frame's sort
    cudaEvent_t upd_ok = nullptr, upd_done = nullptr, sort_done = nullptr, slot_free[2] = {nullptr, nullptr};
    bool front_active = false;     // the last update_gather ran as a front half
    bool slot_free_rec[2] = {false, false};
    // sort: splat keys/records (ping-pong), pair cells/records (ping-pong), scan scratch
    DevBuf skeys[2], srecs[2], span_sorted, block_sums, hist, status, sorted_ordinals;
    // The sort's outputs the raster reads (cell-sorted pair keys / records, cell ranges), one
    // set per frame slot: with frame pipelining the next frame's sort writes one slot while
    // this frame's raster reads the other.
    DevBuf pcell_s[2][2], precs_s[2][2], ranges_s[2];
    DevBuf* pcell() { return pcell_s[slot]; }
    DevBuf* precs() { return precs_s[slot]; }
    DevBuf& ranges() { return ranges_s[slot]; }
    DevBuf long_runs;  // long runs of equal pair keys found by k_cell_fixup (+ their count)
    DevBuf buckets, bucket_staged;  // depth bucket sort: counts/starts/cursors, staged splats
    const uint32_t* final_recs = nullptr;  // cell-sorted pair records of the last frame
    // output
    DevBuf fb_rgb, fb_T;
    // Pipelined host frames alternate two framebuffers: one is read back on the copy
    // stream while the next frame renders into the other. rb_ev marks the end of the
    // read-back of fb_rgb/fb_T (the _alt members travel with their buffer).
    DevBuf fb_rgb_alt, fb_T_alt;
    cudaEvent_t rb_ev = nullptr, rb_ev_alt = nullptr;
    // A pipelined frame's read-back is enqueued by the next call once that frame's
    // mid-frame read-back of its counters is done (flush_readback): the 25 MB copy then
    // runs under the next frame's sort and raster instead of delaying, on the same PCIe
    // link, the next frame's input staging and counter read-back.
    struct PendingReadback {
        bool active = false;
        float *dst_rgb = nullptr, *dst_T = nullptr;
        const float *src_rgb = nullptr, *src_T = nullptr;
        size_t rgb_bytes = 0, T_bytes = 0;
        cudaEvent_t done = nullptr;  // the frame's raster finished (on the context stream)
        cudaEvent_t rb = nullptr;    // recorded when the read-back has landed
    } pending;
    cudaEvent_t pend_ev = nullptr;
    // debug
    DevBuf posed_dbg, rec_dbg;

    void* pinned = nullptr;
    size_t pinned_cap = 0;
    FrameCounters* h_counters = nullptr;
    uint32_t* h_lod = nullptr;  // page-locked LoD read-back (host frames)
    size_t h_lod_cap = 0;
    cudaEvent_t ev[8] = {};
    cudaStream_t copy_stream = nullptr;  // framebuffer read-back overlapped with the raster bands
    cudaEvent_t band_ev[kReadbackBands] = {};

    // last frame
    uint32_t n = 0, tiles = 0, cells_per_tile = 1;
    uint64_t G = 0, S = 0, K = 0, TP = 0;  // TP: the reference's (tile, splat) bin entries
    uint32_t dmin = 0, dmax = 0;  // depth-bit range of the frame's splats
    FrameGeom geom;
    gscg_render_settings settings{};
    uint32_t launches = 0;
    // screen-band exchange: 0 none, 1 routed, 2 packed, 3 band rendered
    int band_state = 0;
    // Stage-function modes of update_gather (gscg_skin_means / gscg_gather_posed).
    enum class Mode { Frame, SkinOnly, PosedIn } mode = Mode::Frame;
    // Attribute layout (gscg_set_layout): the shared store, or the naive per-instance copies
    // of the config-5 ablation, refilled when the instances' levels change.
    int32_t layout = GSCG_LAYOUT_SHARED;
    DevBuf naive_core, naive_w, naive_key;
    uint64_t naive_G = 0;
    bool naive_valid = false;
    DevBuf posed_in, project_mask, posed_out;
    BandParams band{};
    DevBuf band_scratch;
    unsigned long long* h_band_counts = nullptr;
    uint64_t band_total = 0;
    uint32_t band_row0 = 0;

    void ensure_pinned(size_t bytes) {
        if (bytes <= pinned_cap) return;
        if (pinned) cudaFreeHost(pinned);
        pinned = nullptr;
        const size_t want = bytes + bytes / 4;
        CUDA_TRY(cudaMallocHost(&pinned, want));
        pinned_cap = want;
    }
};

namespace {

int fail(gscg_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->error = msg;
    return code;
}

template <typename F>
int guarded(gscg_ctx* ctx, F&& f) {
    try {
        f();
        return GSCG_OK;
    } catch (const Status& s) {
        return fail(ctx, s.code, s.what());
    } catch (const std::bad_alloc&) {
        return fail(ctx, GSCG_ERR_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(ctx, GSCG_ERR_STATE, e.what());
    }
}

void invalid(const std::string& msg) { throw Status(GSCG_ERR_INVALID_ARGUMENT, msg); }

void upload_tables(gscg_ctx* ctx) {
    if (!ctx->tables_dirty) return;
    std::vector<TemplateDev> tdev(ctx->templates.size());
    std::vector<GroupDev> gdev;
    std::vector<float> mats;
    std::vector<int32_t> parents;
    uint32_t stride = 0;
    for (size_t t = 0; t < ctx->templates.size(); ++t) {
        const TemplateStore& ts = ctx->templates[t];
        TemplateDev& d = tdev[t];
        std::memset(&d, 0, sizeof(d));
        if (!ts.present) continue;
        d.joint_count = static_cast<int32_t>(ts.joint_count);
        d.level_count = static_cast<int32_t>(ts.levels.size());
        d.group_base = static_cast<int32_t>(gdev.size());
        d.mat_offset = static_cast<int32_t>(mats.size() / 16);
        d.parent_offset = static_cast<int32_t>(parents.size());
        d.pelvis_y = ts.pelvis_y;
        d.cull_mean_r = d.cull_sigma = d.cull_wabs = d.cull_wdev = 0.0f;
        for (const LevelStore& ls : ts.levels) {
            d.cull_mean_r = std::max(d.cull_mean_r, ls.mean_r);
            d.cull_sigma = std::max(d.cull_sigma, ls.sigma);
            d.cull_wabs = std::max(d.cull_wabs, ls.wabs);
            d.cull_wdev = std::max(d.cull_wdev, ls.wdev);
        }
        mats.insert(mats.end(), ts.local_bind.begin(), ts.local_bind.end());
        mats.insert(mats.end(), ts.inverse_bind.begin(), ts.inverse_bind.end());
        for (int16_t p : ts.parents) parents.push_back(p);
        stride = std::max(stride, ts.joint_count);
        for (size_t l = 0; l < ts.levels.size(); ++l) {
            const LevelStore& ls = ts.levels[l];
            if (ls.count == 0) invalid("template " + std::to_string(t) + " level " + std::to_string(l) + " missing");
            GroupDev g{};
            g.core = ls.core.as<float4>();
            g.weights = ls.weights.as<float4>();
            g.sh = ls.has_sh ? ls.sh.as<float>() : nullptr;
            g.count = ls.count;
            g.template_id = static_cast<uint32_t>(t);
            g.level = static_cast<uint32_t>(l);
            gdev.push_back(g);
        }
    }
    if (gdev.size() > static_cast<size_t>(kMaxGroups)) invalid("too many (template, level) groups");
    ctx->group_count = static_cast<uint32_t>(gdev.size());
    ctx->joint_stride = stride;
    CUDA_TRY(ctx->d_templates.ensure(std::max<size_t>(1, tdev.size()) * sizeof(TemplateDev)));
    CUDA_TRY(ctx->d_groups.ensure(std::max<size_t>(1, gdev.size()) * sizeof(GroupDev)));
    CUDA_TRY(ctx->d_mats.ensure(std::max<size_t>(1, mats.size()) * sizeof(float)));
    CUDA_TRY(ctx->d_parents.ensure(std::max<size_t>(1, parents.size()) * sizeof(int32_t)));
    if (!tdev.empty())
        CUDA_TRY(cudaMemcpyAsync(ctx->d_templates.ptr, tdev.data(), tdev.size() * sizeof(TemplateDev), cudaMemcpyHostToDevice, ctx->stream));
    if (!gdev.empty())
        CUDA_TRY(cudaMemcpyAsync(ctx->d_groups.ptr, gdev.data(), gdev.size() * sizeof(GroupDev), cudaMemcpyHostToDevice, ctx->stream));
    if (!mats.empty())
        CUDA_TRY(cudaMemcpyAsync(ctx->d_mats.ptr, mats.data(), mats.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    if (!parents.empty())
        CUDA_TRY(cudaMemcpyAsync(ctx->d_parents.ptr, parents.data(), parents.size() * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->tables_dirty = false;
}

void upload_motions(gscg_ctx* ctx) {
    if (!ctx->motions_dirty) return;
    std::vector<MotionDev> md(ctx->motions.size());
    std::vector<float4> roots;
    std::vector<KeyPairDev> keys;
    for (size_t i = 0; i < ctx->motions.size(); ++i) {
        const MotionStore& m = ctx->motions[i];
        md[i].fps = m.fps;
        md[i].frames = m.frames;
        md[i].joints = m.joints;
        md[i].root_offset = static_cast<uint32_t>(roots.size());
        md[i].key_offset = keys.size();
        roots.insert(roots.end(), m.roots.begin(), m.roots.end());
        keys.insert(keys.end(), m.keys.begin(), m.keys.end());
    }
    CUDA_TRY(ctx->d_motions.ensure_exact(std::max<size_t>(md.size(), 1) * sizeof(MotionDev)));
    CUDA_TRY(ctx->d_roots.ensure_exact(std::max<size_t>(roots.size(), 1) * sizeof(float4)));
    CUDA_TRY(ctx->d_keys.ensure_exact(std::max<size_t>(keys.size(), 1) * sizeof(KeyPairDev)));
    if (!md.empty())
        CUDA_TRY(cudaMemcpyAsync(ctx->d_motions.ptr, md.data(), md.size() * sizeof(MotionDev), cudaMemcpyHostToDevice, ctx->stream));
    if (!roots.empty())
        CUDA_TRY(cudaMemcpyAsync(ctx->d_roots.ptr, roots.data(), roots.size() * sizeof(float4), cudaMemcpyHostToDevice, ctx->stream));
    if (!keys.empty())
        CUDA_TRY(cudaMemcpyAsync(ctx->d_keys.ptr, keys.data(), keys.size() * sizeof(KeyPairDev), cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->motions_dirty = false;
}

// power_floor = logf(alpha_cutoff / opacity) with the host libm (renderer.cpp:140).
void refresh_power_floor(gscg_ctx* ctx, float cutoff) {
    std::vector<float> pf;
    DevBuf tmp;
    for (TemplateStore& ts : ctx->templates) {
        if (!ts.present) continue;
        for (LevelStore& ls : ts.levels) {
            if (ls.pf_cutoff == cutoff) continue;
            pf.resize(ls.count);
            for (uint32_t i = 0; i < ls.count; ++i) pf[i] = std::log(cutoff / ls.opacities[i]);
            CUDA_TRY(tmp.ensure(ls.count * sizeof(float)));
            CUDA_TRY(cudaMemcpyAsync(tmp.ptr, pf.data(), ls.count * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
            k_set_power_floor<<<(ls.count + 255) / 256, 256, 0, ctx->stream>>>(ls.core.as<float4>(), tmp.as<float>(), ls.count);
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaStreamSynchronize(ctx->stream));
            ls.pf_cutoff = cutoff;
        }
    }
    tmp.release();
}

// Digit layout of one LSD sort: pass q sorts bits [shift[q], shift[q] + bits[q]).
struct RadixPlan {
    uint32_t wide = 0;  // bit q: pass q uses the 7-bit digit kernels (k_sort_*_wide), else 5-bit
    uint32_t passes = 0;
    uint32_t shift[kMaxSortPasses] = {};
    uint32_t bits[kMaxSortPasses] = {};
};

int bits_for(uint32_t v) { return v == 0 ? 0 : 32 - __builtin_clz(v); }

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

}  // namespace

namespace {

void full_region(FrameGeom& g) {
    g.band_x0 = g.band_y0 = 0;
    g.band_x1 = g.W;
    g.band_y1 = g.H;
    g.band_tile_col0 = g.band_tile_row0 = 0;
    g.band_tiles_x = g.tiles_x;
    g.band_tile_rows = g.tiles_y;
}

void validate_frame(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                    const gscg_render_settings* settings, const gscg_lod_policy* lod) {
    if (!frame || !cam || !settings || !lod) invalid("null argument");
    if (settings->tile_size < 1 || settings->tile_size > 64) invalid("RenderSettings: tile_size must be in [1, 64]");
    if (!(settings->alpha_cutoff > 0.0f && settings->alpha_cutoff < 1.0f))
        invalid("RenderSettings: alpha_cutoff outside (0,1)");
    if (!(settings->transmittance_floor > 0.0f && settings->transmittance_floor < 1.0f))
        invalid("RenderSettings: transmittance_floor outside (0,1)");
    if (cam->width < 1 || cam->height < 1 || cam->width > 65535 || cam->height > 65535)
        invalid("Camera: width and height must be in [1, 65535]");
    if (!(cam->near_m > 0.0f)) invalid("Camera: near plane must be > 0");
    if (lod->threshold_count > GSCG_MAX_LOD_THRESHOLDS) invalid("LodPolicy: too many thresholds");
    const uint32_t n = frame->instance_count;
    const bool sampled = frame->pose_source == GSCG_POSES_SAMPLED;
    if (frame->pose_source != GSCG_POSES_GIVEN && !sampled) invalid("unknown pose_source");
    if (n > 0 && (!frame->template_ids || !frame->placement || !frame->active_lod || (!sampled && !frame->poses)))
        invalid("null frame array");
    if (n > 0 && sampled && !frame->static_pose && (!frame->motion_ids || !frame->phase_offsets))
        invalid("sampled poses need motion_ids and phase_offsets");
    upload_tables(ctx);
    if (sampled) upload_motions(ctx);
    if (n > 0 && frame->joint_stride < ctx->joint_stride) invalid("joint_stride below the largest skeleton");
    if (frame->memory == GSCG_MEM_HOST) {
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t t = frame->template_ids[i];
            if (t >= ctx->templates.size() || !ctx->templates[t].present || ctx->templates[t].levels.empty())
                invalid("instance " + std::to_string(i) + " references a missing template");
            if (sampled && !frame->static_pose) {
                const uint32_t m = frame->motion_ids[i];
                if (m >= ctx->motions.size()) invalid("instance " + std::to_string(i) + " references a missing motion");
                if (ctx->motions[m].joints != ctx->templates[t].joint_count)
                    invalid("forward_kinematics: pose joint count mismatch");
            }
        }
    }
    refresh_power_floor(ctx, settings->alpha_cutoff);
    FrameGeom& g = ctx->geom;
    g.W = cam->width;
    g.H = cam->height;
    g.ts = settings->tile_size;
    g.tiles_x = (g.W + g.ts - 1) / g.ts;
    g.tiles_y = (g.H + g.ts - 1) / g.ts;
    g.cells_per_tile = g.ts == 16 ? 4u : 1u;  // 8x8 quadrant binning for tile 16
    g.cell = g.ts == 16 ? 8 : g.ts;
    full_region(g);  // the whole frame; gscg_render_frame applies gscg_set_region's (apply_band)
    ctx->settings = *settings;
}

// gscg_set_band's rows for a render: the frame keeps only the splats whose rect meets
// rows [band_y0, band_y1) and rasterises those rows (the multi-GPU band frame).
void apply_band(gscg_ctx* ctx) {
    FrameGeom& g = ctx->geom;
    const bool rows = ctx->band_req1 > ctx->band_req0, cols = ctx->col_req1 > ctx->col_req0;
    if (!rows && !cols) return;
    auto aligned = [&](int32_t a, int32_t b, int32_t limit) {
        return a >= 0 && a % g.ts == 0 && (b % g.ts == 0 || b == limit) && b <= limit;
    };
    if (rows) {
        if (!aligned(ctx->band_req0, ctx->band_req1, g.H))
            invalid("gscg_set_region: rows must be tile-aligned and inside the frame");
        g.band_y0 = ctx->band_req0;
        g.band_y1 = ctx->band_req1;
    }
    if (cols) {
        if (!aligned(ctx->col_req0, ctx->col_req1, g.W))
            invalid("gscg_set_region: columns must be tile-aligned and inside the frame");
        g.band_x0 = ctx->col_req0;
        g.band_x1 = ctx->col_req1;
    }
    g.band_tile_row0 = g.band_y0 / g.ts;
    g.band_tile_rows = (g.band_y1 - g.band_y0 + g.ts - 1) / g.ts;
    g.band_tile_col0 = g.band_x0 / g.ts;
    g.band_tiles_x = (g.band_x1 - g.band_x0 + g.ts - 1) / g.ts;
}

// H2D of the frame records, update (LoD plan + FK) and gather (projection) for the
// instances [shard_begin, shard_end); sets S, K, G and the depth-bit range. Events 0..3.
// lod_back: host frames get active_lod back with the mid-frame counter read-back (the LoD
// is final after k_lod_plan), so the frame's end needs no host synchronisation for it.
void flush_readback(gscg_ctx* ctx);

bool settle_counts(gscg_ctx* ctx, const gscg_frame_desc* frame, uint32_t n, bool lod_back, bool flush = true,
                   bool deferred_check = false);

// deferred: return right after enqueueing (no host read of the counters); the caller
// enqueues the sort on device counts and then calls settle_counts.
void update_gather(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                   const gscg_lod_policy* lod, uint32_t shard_begin, uint32_t shard_end, uint32_t& launches,
                   bool lod_back = false, bool deferred = false, bool overlap_update = false) {
    // A front half (overlap_update, frame pipelining) runs whole on the update stream.
    cudaStream_t s = overlap_update ? ctx->upd_stream : ctx->stream;
    cudaStream_t su = s;
    if (overlap_update) {
        // Following other work: wait for everything on the render stream. Following a front
        // half: only for the raster that last read this frame's slot.
        if (!ctx->front_active) {
            CUDA_TRY(cudaEventRecord(ctx->upd_ok, ctx->stream));
            CUDA_TRY(cudaStreamWaitEvent(s, ctx->upd_ok, 0));
        }
        if (ctx->slot_free_rec[ctx->slot]) CUDA_TRY(cudaStreamWaitEvent(s, ctx->slot_free[ctx->slot], 0));
    } else if (ctx->front_active) {
        CUDA_TRY(cudaStreamWaitEvent(s, ctx->upd_done, 0));  // the last front half's tail
    }
    ctx->front_active = overlap_update;
    const FrameGeom& geo = ctx->geom;
    const gscg_render_settings* settings = &ctx->settings;
    const bool host = frame->memory == GSCG_MEM_HOST;
    const uint32_t n = frame->instance_count;
    const uint32_t js = std::max<uint32_t>(ctx->joint_stride, 1);
    const uint32_t pose_stride = 4 + 4 * frame->joint_stride;
    const bool posed_mode = ctx->mode == gscg_ctx::Mode::PosedIn;  // posed means given: no pose / FK / cull
    const bool skin_only = ctx->mode == gscg_ctx::Mode::SkinOnly;   // update_crowd: posed means out, no projection

    CUDA_TRY(ctx->template_ids.ensure(std::max<size_t>(n, 1) * 4));
    CUDA_TRY(ctx->placement.ensure(std::max<size_t>(n, 1) * 16));
    CUDA_TRY(ctx->poses.ensure(std::max<size_t>(n, 1) * pose_stride * 4));
    CUDA_TRY(ctx->lod_prev.ensure(std::max<size_t>(n, 1) * 4));
    CUDA_TRY(ctx->lod_out.ensure(std::max<size_t>(n, 1) * 4));
    CUDA_TRY(ctx->inst_group.ensure(std::max<size_t>(n, 1) * 4));
    CUDA_TRY(ctx->inst_base.ensure(std::max<size_t>(n, 1) * 4));
    CUDA_TRY(ctx->members.ensure(std::max<size_t>(n, 1) * 4));
    CUDA_TRY(ctx->visible.ensure(std::max<size_t>(n, 1) * 4));
    CUDA_TRY(ctx->group_inst_start.ensure((kMaxGroups + 1) * 4));
    CUDA_TRY(ctx->group_inst_count.ensure((kMaxGroups + 1) * 4));
    CUDA_TRY(ctx->group_item_start.ensure((kMaxGroups + 1) * 4));
    CUDA_TRY(ctx->skin.ensure(std::max<size_t>(n, 1) * js * 12 * 4));

    // ---- H2D ----
    CUDA_TRY(cudaEventRecord(ctx->ev[0], su));
    const uint32_t *d_tid, *d_lodprev;
    const float *d_place, *d_poses;
    const bool sampled = frame->pose_source == GSCG_POSES_SAMPLED;
    const bool need_motion = sampled && !frame->static_pose && n > 0;
    const uint32_t *d_mid = nullptr;
    const float* d_phase = nullptr;
    if (sampled) {
        CUDA_TRY(ctx->motion_ids.ensure(std::max<size_t>(n, 1) * 4));
        CUDA_TRY(ctx->phases.ensure(std::max<size_t>(n, 1) * 4));
    }
    if (host) {
        // One pinned staging block; the arrays are pulled into HBM by one k_copy_segments
        // launch (mapped page-locked memory, no copy-engine queueing behind a read-back).
        const size_t b_tid = n * 4ull, b_place = n * 16ull, b_pose = sampled ? 0 : n * 4ull * pose_stride,
                     b_lod = n * 4ull, b_mid = need_motion ? n * 4ull : 0, b_ph = need_motion ? n * 4ull : 0;
        ctx->ensure_pinned(b_tid + b_place + b_pose + b_lod + b_mid + b_ph + 6 * 16 + 64);
        char* h = static_cast<char*>(ctx->pinned);
        size_t off = 0;
        CopySegs segs{};
        uint32_t nseg = 0, max_words = 0;
        auto stage = [&](const void* src, size_t bytes, void* dst) {
            if (!bytes) return;
            std::memcpy(h + off, src, bytes);
            segs.src[nseg] = reinterpret_cast<const uint32_t*>(h + off);
            segs.dst[nseg] = static_cast<uint32_t*>(dst);
            segs.words[nseg] = static_cast<uint32_t>(bytes / 4);
            max_words = std::max(max_words, segs.words[nseg]);
            ++nseg;
            off += (bytes + 15) & ~size_t(15);
        };
        stage(frame->template_ids, b_tid, ctx->template_ids.ptr);
        stage(frame->placement, b_place, ctx->placement.ptr);
        if (!sampled) stage(frame->poses, b_pose, ctx->poses.ptr);
        stage(frame->active_lod, b_lod, ctx->lod_prev.ptr);
        if (need_motion) {
            stage(frame->motion_ids, b_mid, ctx->motion_ids.ptr);
            stage(frame->phase_offsets, b_ph, ctx->phases.ptr);
        }
        if (nseg) {
            const uint32_t bx = std::min<uint32_t>((max_words + 255) / 256, 4u * ctx->sm_count);
            CUDA_TRY(pdl_launch(k_copy_segments, dim3(bx, nseg), 256, 0, su, segs));
            ++launches;
            CUDA_TRY(cudaGetLastError());
        }
        d_tid = ctx->template_ids.as<uint32_t>();
        d_place = ctx->placement.as<float>();
        d_poses = ctx->poses.as<float>();
        d_lodprev = ctx->lod_prev.as<uint32_t>();
        d_mid = ctx->motion_ids.as<uint32_t>();
        d_phase = ctx->phases.as<float>();
    } else {
        d_tid = frame->template_ids;
        d_place = frame->placement;
        d_poses = sampled ? ctx->poses.as<float>() : frame->poses;
        d_lodprev = frame->active_lod;
        d_mid = frame->motion_ids;
        d_phase = frame->phase_offsets;
    }
    CUDA_TRY(cudaEventRecord(ctx->ev[1], su));
    if (sampled && shard_end > shard_begin && !posed_mode) {
        // update_crowd's pose sampling on the device (gscg_pose.cu); FK reads ctx->poses.
        PoseParams pp{};
        pp.n = n;
        pp.joint_stride = frame->joint_stride;
        pp.time_s = frame->time_s;
        pp.static_pose = frame->static_pose ? 1 : 0;
        pp.motion_ids = d_mid;
        pp.phase = d_phase;
        pp.motions = ctx->d_motions.as<MotionDev>();
        pp.roots = ctx->d_roots.as<float4>();
        pp.keys = ctx->d_keys.as<KeyPairDev>();
        pp.poses = ctx->poses.as<float>();
        const uint64_t threads = static_cast<uint64_t>(n) * (frame->joint_stride + 1);
        CUDA_TRY(pdl_launch(k_sample_poses, static_cast<uint32_t>((threads + 255) / 256), 256, 0, su, pp));
        ++launches;
        CUDA_TRY(cudaGetLastError());
    }

    const int project_smem = (settings->sh_enabled ? kProjectThreads * kShFloats * 4 : 0) + kBatch * static_cast<int>(js) * 12 * 4;
    int project_blocks_per_sm = 1;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&project_blocks_per_sm, k_project<false, false>, kProjectThreads,
                                                           project_smem));
    project_blocks_per_sm = std::max(project_blocks_per_sm, 1);

    CameraDev camdev{};
    std::memcpy(camdev.w, cam->world_to_view, sizeof(camdev.w));
    std::memcpy(camdev.pos, cam->position, sizeof(camdev.pos));
    camdev.focal = cam->focal;
    camdev.cx = cam->cx;
    camdev.cy = cam->cy;
    camdev.near_m = cam->near_m;
    camdev.width = geo.W;
    camdev.height = geo.H;
    camdev.band_x0 = geo.band_x0;
    camdev.band_y0 = geo.band_y0;
    camdev.band_x1 = geo.band_x1;
    camdev.band_y1 = geo.band_y1;
    auto* counters = ctx->counters.as<FrameCounters>();
    for (int attempt = 0;; ++attempt) {
        if (lod_back && n && ctx->h_lod_cap < n) {
            if (ctx->h_lod) CUDA_TRY(cudaFreeHost(ctx->h_lod));
            ctx->h_lod = nullptr;
            ctx->h_lod_cap = 0;
            CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_lod), n * 4ull));
            ctx->h_lod_cap = n;
        }
        // ---- update ---- (FK first: the cull reads the skin matrices, the plan the cull)
        if (shard_end > shard_begin && !posed_mode) {
            FkParams fp{};
            fp.n = shard_end;
            fp.first = shard_begin;
            fp.joint_stride = js;
            fp.pose_stride = pose_stride;
            fp.template_ids = d_tid;
            fp.placement = d_place;
            fp.poses = d_poses;
            fp.templates = ctx->d_templates.as<TemplateDev>();
            fp.mats = ctx->d_mats.as<float>();
            fp.parents = ctx->d_parents.as<int32_t>();
            fp.skin = ctx->skin.as<float>();
            const int per_block = kFkThreads / 16;
            const uint32_t m = shard_end - shard_begin;
            CUDA_TRY(pdl_launch(k_fk_skin, (m + per_block - 1) / per_block, kFkThreads, per_block * kFkSmemPerInstance(js), su, fp));
            ++launches;
            CUDA_TRY(cudaGetLastError());
        }
        // Instance frustum cull (off with GSCG_DEBUG_POSED, which keeps every posed mean,
        // and GSCG_DEBUG_NO_CULL).
        const bool cull = shard_end > shard_begin && !posed_mode && !skin_only &&
                          !(ctx->debug & (GSCG_DEBUG_POSED | GSCG_DEBUG_NO_CULL));
        if (cull) {
            CullParams cp{};
            cp.n = shard_end;
            cp.first = shard_begin;
            cp.joint_stride = js;
            cp.template_ids = d_tid;
            cp.templates = ctx->d_templates.as<TemplateDev>();
            cp.skin = ctx->skin.as<float>();
            cp.cam = camdev;
            cp.visible = ctx->visible.as<uint32_t>();
            const uint32_t m = shard_end - shard_begin;
            CUDA_TRY(pdl_launch(k_inst_cull, (m + 7) / 8, 256, 0, su, cp));
            ++launches;
            CUDA_TRY(cudaGetLastError());
        }
        PlanParams pp{};
        pp.n = n;
        pp.shard_begin = shard_begin;
        pp.shard_end = shard_end;
        pp.template_ids = d_tid;
        pp.placement = d_place;
        pp.lod_prev = d_lodprev;
        pp.forced_lod = frame->forced_lod;
        pp.threshold_count = lod->threshold_count;
        for (uint32_t i = 0; i < lod->threshold_count; ++i) pp.thresholds[i] = lod->thresholds_m[i];
        pp.hysteresis = lod->hysteresis_band_m;
        for (int i = 0; i < 3; ++i) pp.cam_pos[i] = cam->position[i];
        pp.templates = ctx->d_templates.as<TemplateDev>();
        pp.groups = ctx->d_groups.as<GroupDev>();
        pp.group_count = ctx->group_count;
        pp.lod_out = ctx->lod_out.as<uint32_t>();
        pp.inst_group = ctx->inst_group.as<uint32_t>();
        pp.inst_base = ctx->inst_base.as<uint32_t>();
        pp.group_inst_start = ctx->group_inst_start.as<uint32_t>();
        pp.group_inst_count = ctx->group_inst_count.as<uint32_t>();
        pp.group_item_start = ctx->group_item_start.as<uint32_t>();
        pp.members = ctx->members.as<uint32_t>();
        pp.visible = cull ? ctx->visible.as<uint32_t>() : posed_mode ? ctx->project_mask.as<uint32_t>() : nullptr;
        pp.counters = counters;
        CUDA_TRY(pdl_launch(k_lod_plan, 1, 1024, 0, su, pp));
        ++launches;
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaEventRecord(ctx->ev[2], su));

        const bool naive = ctx->layout == GSCG_LAYOUT_NAIVE && !posed_mode && !skin_only;
        if (naive) {
            // Per-instance copies sized by this frame's instance-Gaussians (a host read of the
            // plan's counter); refilled only when the level assignment changes.
            if (settings->sh_enabled) invalid("the naive layout ablation renders RGB colour (sh_enabled = 0)");
            CUDA_TRY(cudaMemcpyAsync(ctx->h_counters, counters, sizeof(FrameCounters), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            const uint64_t G = ctx->h_counters->gaussians;
            std::vector<uint32_t> key(n * 2ull + 1);
            if (n) {
                CUDA_TRY(cudaMemcpy(key.data(), ctx->inst_group.ptr, n * 4ull, cudaMemcpyDeviceToHost));
                CUDA_TRY(cudaMemcpy(key.data() + n, ctx->inst_base.ptr, n * 4ull, cudaMemcpyDeviceToHost));
            }
            key[2ull * n] = n;
            const bool same = ctx->naive_valid && G == ctx->naive_G && ctx->naive_key.cap >= key.size() * 4 &&
                              [&] {
                                  std::vector<uint32_t> old(key.size());
                                  return cudaMemcpy(old.data(), ctx->naive_key.ptr, key.size() * 4, cudaMemcpyDeviceToHost) ==
                                             cudaSuccess && old == key;
                              }();
            if (!same) {
                CUDA_TRY(ctx->naive_core.ensure_exact(std::max<uint64_t>(G, 1) * 64));
                CUDA_TRY(ctx->naive_w.ensure_exact(std::max<uint64_t>(G, 1) * 16));
                if (n) {
                    k_naive_fill<<<dim3(64, std::min<uint32_t>(n, 65535u)), 256, 0, s>>>(
                        ctx->inst_group.as<uint32_t>(), ctx->inst_base.as<uint32_t>(), ctx->d_groups.as<GroupDev>(), n,
                        ctx->naive_core.as<float4>(), ctx->naive_w.as<float4>());
                    ++launches;
                    CUDA_TRY(cudaGetLastError());
                }
                CUDA_TRY(ctx->naive_key.ensure(key.size() * 4));
                CUDA_TRY(cudaMemcpyAsync(ctx->naive_key.ptr, key.data(), key.size() * 4, cudaMemcpyHostToDevice, s));
                CUDA_TRY(cudaStreamSynchronize(s));
                ctx->naive_G = G;
                ctx->naive_valid = true;
            }
        }
        if ((ctx->debug & GSCG_DEBUG_POSED) || skin_only) {
            CUDA_TRY(cudaMemcpyAsync(ctx->h_counters, counters, sizeof(FrameCounters), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (ctx->h_counters->gaussians > 0xffffffffull)
                throw Status(GSCG_ERR_OOM, "instance-Gaussian count exceeds 32-bit ordinals");
            CUDA_TRY((skin_only ? ctx->posed_out : ctx->posed_dbg).ensure(std::max<uint64_t>(ctx->h_counters->gaussians, 1) * 12));
        }
        if (skin_only) {  // update_crowd: the posed means of every instance, then stop
            SkinParams sp{};
            sp.n = n;
            sp.joint_stride = js;
            sp.inst_group = ctx->inst_group.as<uint32_t>();
            sp.inst_base = ctx->inst_base.as<uint32_t>();
            sp.groups = ctx->d_groups.as<GroupDev>();
            sp.skin = ctx->skin.as<float>();
            sp.posed = ctx->posed_out.as<float>();
            uint32_t max_count = 0;
            for (const TemplateStore& t : ctx->templates)
                for (const LevelStore& l : t.levels) max_count = std::max(max_count, l.count);
            if (n && max_count) {
                k_skin_means<<<dim3((max_count + 255) / 256, std::min<uint32_t>(n, 65535u)), 256, 0, s>>>(sp);
                ++launches;
                CUDA_TRY(cudaGetLastError());
            }
            ctx->G = ctx->h_counters->gaussians;
            ctx->n = n;
            return;
        }
        if (ctx->splat_capacity == 0) {
            ctx->splat_capacity = 1u << 20;
            ctx->pair_capacity = 1u << 21;
        }
        CUDA_TRY(ctx->rec().ensure(ctx->splat_capacity * 48));
        CUDA_TRY(ctx->meta().ensure(ctx->splat_capacity * 16));
        CUDA_TRY(ctx->depth().ensure(ctx->splat_capacity * 4));
        if (ctx->debug & GSCG_DEBUG_RECORDS)
            CUDA_TRY(ctx->rec_dbg.ensure(ctx->splat_capacity * sizeof(gscg_splat_record)));

        // ---- gather ----
        ProjectParams pj{};
        pj.cam = camdev;
        pj.tile_size = geo.ts;
        pj.tiles_x = geo.tiles_x;
        pj.sh_enabled = settings->sh_enabled ? 1 : 0;
        pj.joint_stride = js;
        pj.group_count = ctx->group_count;
        pj.groups = ctx->d_groups.as<GroupDev>();
        pj.group_item_start = ctx->group_item_start.as<uint32_t>();
        pj.group_inst_start = ctx->group_inst_start.as<uint32_t>();
        pj.group_inst_count = ctx->group_inst_count.as<uint32_t>();
        pj.members = ctx->members.as<uint32_t>();
        pj.inst_base = ctx->inst_base.as<uint32_t>();
        pj.skin = ctx->skin.as<float>();
        pj.counters = counters;
        pj.records = ctx->rec().as<float4>();
        pj.splat_depth = ctx->depth().as<uint32_t>();
        pj.splat_meta = ctx->meta().as<uint4>();
        pj.splat_capacity = ctx->splat_capacity;
        pj.pair_capacity = ctx->pair_capacity;
        pj.posed_in = posed_mode ? ctx->posed_in.as<float>() : nullptr;
        pj.naive_core = naive ? ctx->naive_core.as<float4>() : nullptr;
        pj.naive_weights = naive ? ctx->naive_w.as<float4>() : nullptr;
        pj.posed_debug = (ctx->debug & GSCG_DEBUG_POSED) ? ctx->posed_dbg.as<float>() : nullptr;
        pj.record_debug = (ctx->debug & GSCG_DEBUG_RECORDS) ? ctx->rec_dbg.as<gscg_splat_record>() : nullptr;
        if (shard_end > shard_begin && ctx->group_count > 0) {
            const dim3 grid(ctx->sm_count * project_blocks_per_sm);
            if (posed_mode)
                CUDA_TRY(pdl_launch(k_project<true, false>, grid, kProjectThreads, project_smem, s, pj));
            else if (naive)
                CUDA_TRY(pdl_launch(k_project<false, true>, grid, kProjectThreads, project_smem, s, pj));
            else
                CUDA_TRY(pdl_launch(k_project<false, false>, grid, kProjectThreads, project_smem, s, pj));
            ++launches;
            CUDA_TRY(cudaGetLastError());
        }
        CUDA_TRY(cudaEventRecord(ctx->ev[3], s));
        {  // counters (+ the final LoD for host frames) into page-locked memory by a kernel
            CopySegs segs{};
            segs.src[0] = reinterpret_cast<const uint32_t*>(counters);
            segs.dst[0] = reinterpret_cast<uint32_t*>(ctx->h_counters);
            segs.words[0] = sizeof(FrameCounters) / 4;
            uint32_t nseg = 1;
            if (lod_back && n) {
                segs.src[1] = ctx->lod_out.as<uint32_t>();
                segs.dst[1] = ctx->h_lod;
                segs.words[1] = n;
                nseg = 2;
            }
            CUDA_TRY(pdl_launch(k_copy_segments, dim3(std::min<uint32_t>((n + 255) / 256 + 1, 64u), nseg), 256, 0, s, segs));
            ++launches;
            CUDA_TRY(cudaGetLastError());
        }
        CUDA_TRY(cudaEventRecord(ctx->counters_ev, s));
        ctx->n = n;
        if (deferred) return;  // the caller enqueues the sort on device counts, then settle_counts
        if (settle_counts(ctx, frame, n, lod_back)) return;
        if (attempt > 2) throw Status(GSCG_ERR_STATE, "splat/pair capacity did not converge");
    }
}

// Host read of a frame's counters (after update_gather's counter copy): the 32-bit limits,
// the frame's S / K / G / depth range, the LoD write-back of host frames. Returns false,
// with the capacities grown, when the frame's splats or pairs did not fit (its records were
// clamped and it must be rendered again).
bool settle_counts(gscg_ctx* ctx, const gscg_frame_desc* frame, uint32_t n, bool lod_back, bool flush,
                   bool deferred_check) {
    CUDA_TRY(cudaEventSynchronize(ctx->counters_ev));
    if (flush) flush_readback(ctx);  // the previous pipelined frame's read-back overlaps this frame's sort
    const FrameCounters& c = *ctx->h_counters;
    const uint64_t S = c.splats, K = c.pairs;
    // Global ordinals (instance base + gaussian index) and record / pair indices are 32-bit:
    // a frame past that is reported as out of memory (bench.cpp:94-97 skips it) instead of
    // aliasing.
    if (c.gaussians > 0xffffffffull) throw Status(GSCG_ERR_OOM, "instance-Gaussian count exceeds 32-bit ordinals");
    if (S > 0xF0000000ull) throw Status(GSCG_ERR_OOM, "splat count exceeds 32-bit indexing");
    if (K > 0xF0000000ull) throw Status(GSCG_ERR_OOM, "tile-splat pair count exceeds 32-bit indexing");
    const uint32_t dbits = static_cast<uint32_t>(bits_for(c.depth_min_bits ^ c.depth_max_bits));
    ctx->dbits_prev = dbits;
    if (deferred_check && dbits > ctx->deferred_depth_top) return false;  // the plan missed high key bits
    if (S > ctx->splat_capacity || K > ctx->pair_capacity) {
        ctx->splat_capacity = std::max<uint64_t>(ctx->splat_capacity, S + S / 4 + 1024);
        ctx->pair_capacity = std::max<uint64_t>(ctx->pair_capacity, K + K / 4 + 1024);
        return false;
    }
    if (lod_back && n) std::memcpy(frame->active_lod, ctx->h_lod, n * 4ull);
    ctx->S = S;
    ctx->K = K;
    ctx->G = c.gaussians;
    ctx->TP = c.tile_pairs;
    ctx->dmin = c.depth_min_bits;
    ctx->dmax = c.depth_max_bits;
    ctx->culled = c.instances_culled;
    return true;
}

// Sort (splats by depth + ordinal, pairs in that order, pairs stably by cell) and
// rasterise tile rows [tile_row0, tile_row0 + tile_rows) from the context's records
// (ctx->S splats, ctx->K pairs whose spans are relative to tile_row0). Events 3..5.
// Stable LSD radix sort of (keys, vals) over the plan (reduce-then-scan passes) into the
// ping-pong buffers kb/vb; returns the buffer index holding the result. in_keys/in_vals
// feed pass 0 (vals may be null = identity). ctx->status / ctx->hist must fit `count`.
// count_dev (may be null): the pass count is min(count, *count_dev) on the device, count
// then being the capacity the grid covers (deferred frames).
int run_radix(gscg_ctx* ctx, const uint32_t* in_keys, const uint32_t* in_vals, DevBuf* kb, DevBuf* vb,
              uint32_t count, const RadixPlan& plan, uint32_t& launches, const unsigned long long* count_dev = nullptr,
              cudaStream_t stream = nullptr) {
    cudaStream_t s = stream ? stream : ctx->stream;
    const uint32_t tiles = (count + kSortTile - 1) / kSortTile;
    int out = 0;
    for (uint32_t q = 0; q < plan.passes; ++q) {
        SortPassParams sp{};
        sp.keys_in = q == 0 ? in_keys : kb[out ^ 1].as<uint32_t>();
        sp.vals_in = q == 0 ? in_vals : vb[out ^ 1].as<uint32_t>();
        sp.keys_out = kb[out].as<uint32_t>();
        sp.vals_out = vb[out].as<uint32_t>();
        sp.count = count;
        sp.shift = plan.shift[q];
        sp.bits = plan.bits[q];
        sp.tiles = tiles;
        sp.counts = ctx->status.as<uint32_t>();
        sp.digit_base = ctx->hist.as<uint32_t>();
        sp.count_dev = count_dev;
        const bool wide = (plan.wide >> q) & 1u;
        if (wide) CUDA_TRY(pdl_launch(k_sort_upsweep_wide, tiles, kSortThreads, 0, s, sp));
        else CUDA_TRY(pdl_launch(k_sort_upsweep, tiles, kSortThreads, 0, s, sp));
        CUDA_TRY(pdl_launch(k_sort_rows, 1u << plan.bits[q], 1024, 0, s, sp));
        if (wide) CUDA_TRY(pdl_launch(k_sort_downsweep_wide, tiles, kSortThreads, 0, s, sp));
        else CUDA_TRY(pdl_launch(k_sort_downsweep, tiles, kSortThreads, 0, s, sp));
        launches += 3;
        out ^= 1;
    }
    CUDA_TRY(cudaGetLastError());
    return out ^ 1;
}

// The cheapest LSD plan for `bits` key bits: w wide passes (<= 7 bits) then n 5-bit
// passes, minimising cost(wide) w + n. A wide pass measures 2.16x a 5-bit pass on the
// 61.7 M cell pairs of config 4 (529 vs 245 us: its upsweep ranks with shared counters),
// more than the two 5-bit passes it would replace, so plans use 5-bit passes only (12 cell
// bits -> 4, 4, 4); GSCG_WIDE_PASSES=1 restores the round-1 cost model (1.36) for A/B.
// 8-bit digits ranked with warp match (CUB onesweep style) measured slower still:
// __match_any_sync is slow on sm_100 (upsweep 74 vs 31 us, downsweep 126 vs 77 us per pass).
uint32_t wide_cost() {  // per 100 of a 5-bit pass
    static const uint32_t c = [] {
        const char* e = std::getenv("GSCG_WIDE_PASSES");
        return e && e[0] == '1' ? 136u : 216u;
    }();
    return c;
}
RadixPlan make_plan(uint32_t bits) {
    RadixPlan pl{};
    bits = std::max(bits, 1u);
    uint32_t best_w = 0, best_n = (bits + kRadixBits - 1) / kRadixBits;
    for (uint32_t w = 1; w * kWideBits < bits + kWideBits; ++w) {
        const uint32_t rest = bits > w * kWideBits ? bits - w * kWideBits : 0u;
        const uint32_t n = (rest + kRadixBits - 1) / kRadixBits;
        if (wide_cost() * w + 100 * n < wide_cost() * best_w + 100 * best_n) {
            best_w = w;
            best_n = n;
        }
    }
    pl.passes = best_w + best_n;
    const uint32_t wide_bits = std::min(bits, best_w * static_cast<uint32_t>(kWideBits));
    uint32_t sh = 0;
    for (uint32_t q = 0; q < pl.passes; ++q) {
        const bool wq = q < best_w;
        const uint32_t left = wq ? wide_bits - sh : bits - sh;
        const uint32_t k = wq ? best_w - q : pl.passes - q;
        const uint32_t width = left / k + (left % k ? 1u : 0u);
        pl.shift[q] = sh;
        pl.bits[q] = width;
        if (wq) pl.wide |= 1u << q;
        sh += width;
    }
    return pl;
}

void ensure_sort_buffers(gscg_ctx* ctx, uint32_t splats, uint32_t pairs) {
    const uint32_t max_elems = std::max(splats, pairs);
    const uint32_t max_tiles = (max_elems + kSortTile - 1) / kSortTile;
    CUDA_TRY(ctx->status.ensure(std::max<size_t>(max_tiles, 1) * kWideRadix * 4));  // tile digit counts
    CUDA_TRY(ctx->hist.ensure(kWideRadix * 4));                                        // digit bases
    for (int b = 0; b < 2; ++b) {
        CUDA_TRY(ctx->skeys[b].ensure(std::max<size_t>(splats, 1) * 4));
        CUDA_TRY(ctx->srecs[b].ensure(std::max<size_t>(splats, 1) * 4));
        CUDA_TRY(ctx->pcell()[b].ensure(std::max<size_t>(pairs, 1) * 4));
        CUDA_TRY(ctx->precs()[b].ensure(std::max<size_t>(pairs, 1) * 4));
    }
}

void copy_out(gscg_ctx* ctx, int rows, float* fb_rgb, float* fb_T, bool host);

bool is_host_pointer(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;  // unregistered host memory
    }
    return at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged;
}

// presorted: the caller put the splat order in skeys[0] / srecs[0] (distinct keys), so the
// depth sort is skipped (rasterize_splats: bins follow the given order).
// pipelined: render into the other framebuffer and leave its read-back running on the
// copy stream (gscg_render_frame_async).
// Enqueues a deferred pipelined read-back (see gscg_ctx::pending) on the copy stream.
void flush_readback(gscg_ctx* ctx) {
    auto& p = ctx->pending;
    if (!p.active) return;
    p.active = false;
    CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, p.done, 0));
    if (p.dst_rgb) CUDA_TRY(cudaMemcpyAsync(p.dst_rgb, p.src_rgb, p.rgb_bytes, cudaMemcpyDefault, ctx->copy_stream));
    if (p.dst_T) CUDA_TRY(cudaMemcpyAsync(p.dst_T, p.src_T, p.T_bytes, cudaMemcpyDefault, ctx->copy_stream));
    CUDA_TRY(cudaEventRecord(p.rb, ctx->copy_stream));
}

uint32_t sort_raster(gscg_ctx* ctx, int tile_row0, int tile_rows, uint32_t& launches, float* read_rgb = nullptr,
                     float* read_T = nullptr, bool presorted = false, bool pipelined = false,
                     bool device_counts = false) {
    // A pipelined frame's sort runs on the sort stream (after its front half, and after the
    // raster that last read this slot's pair buffers), its raster on the render stream after
    // the sort: the next frame's sort may run under this frame's raster.
    cudaStream_t rs_ = ctx->stream;
    static const bool split_on = [] {  // GSCG_SPLIT_SORT=0: the sort stays on the render stream (A/B)
        const char* e = std::getenv("GSCG_SPLIT_SORT");
        return !(e && e[0] == '0');
    }();
    const bool split = split_on && ctx->front_active && !presorted && !device_counts;
    cudaStream_t s = split ? ctx->sort_stream : rs_;
    if (split) {
        CUDA_TRY(cudaStreamWaitEvent(s, ctx->upd_done, 0));
        if (ctx->slot_free_rec[ctx->slot]) CUDA_TRY(cudaStreamWaitEvent(s, ctx->slot_free[ctx->slot], 0));
    }
    const FrameGeom& geo = ctx->geom;
    // The region's tile columns (the whole frame's unless gscg_set_region narrowed them).
    const int rtx = geo.band_tiles_x;
    const uint32_t tiles = static_cast<uint32_t>(rtx) * static_cast<uint32_t>(tile_rows);
    const uint32_t cells = tiles * geo.cells_per_tile;
    flush_readback(ctx);
    if (pipelined) {
        std::swap(ctx->fb_rgb, ctx->fb_rgb_alt);
        std::swap(ctx->fb_T, ctx->fb_T_alt);
        std::swap(ctx->rb_ev, ctx->rb_ev_alt);
    }
    CUDA_TRY(ctx->fb_rgb.ensure(static_cast<size_t>(geo.W) * geo.H * 12));
    CUDA_TRY(ctx->fb_T.ensure(static_cast<size_t>(geo.W) * geo.H * 4));
    // An earlier pipelined frame may still be reading this framebuffer back.
    CUDA_TRY(cudaStreamWaitEvent(rs_, ctx->rb_ev, 0));
    CUDA_TRY(ctx->ranges().ensure(std::max<size_t>(cells, 1) * 8));

    // Deferred frames (device_counts): the host has not read this frame's counters yet, so
    // grids and buffers cover the capacities and every kernel takes its count (and the depth
    // plan its drop) from the device counters.
    auto* dcnt = ctx->counters.as<FrameCounters>();
    const uint32_t K = device_counts ? static_cast<uint32_t>(ctx->pair_capacity) : static_cast<uint32_t>(ctx->K);
    const uint32_t S32 = device_counts ? static_cast<uint32_t>(ctx->splat_capacity) : static_cast<uint32_t>(ctx->S);
    const unsigned long long* s_dev = device_counts ? &dcnt->splats : nullptr;
    const unsigned long long* k_dev = device_counts ? &dcnt->pairs : nullptr;
    uint32_t passes = 0;
    if (cells) CUDA_TRY(cudaMemsetAsync(ctx->ranges().ptr, 0, static_cast<size_t>(cells) * 8, s));
    ctx->final_recs = nullptr;
    if (S32 > 0 && K > 0) {
        ensure_sort_buffers(ctx, S32, K);
        // 1. splats by the top (at most kDepthSortBits) varying bits of their depth keys;
        //    the dropped low bits and the ordinal tie-break are settled per cell in step 4.
        // Deferred frames plan on the last settled frame's depth range plus one bit of
        // headroom (settle_counts re-renders a frame whose range outgrew it): the plan covers
        // key bits [drop, top); any drop is exact, the fix-up orders what it leaves tied.
        const uint32_t dbits = device_counts ? std::min(ctx->dbits_prev + 1u, 32u)
                                             : static_cast<uint32_t>(bits_for(ctx->dmin ^ ctx->dmax));
        const uint32_t drop = dbits > ctx->depth_sort_bits ? dbits - ctx->depth_sort_bits : 0u;
        if (device_counts) ctx->deferred_depth_top = dbits;
        // Host-settled frames take the bucket sort (gscg_depth.cu, spans gathered on the way);
        // deferred frames (counts and depth range still on the device) the LSD passes.
        const uint32_t tag_min = ctx->dmin >> drop, tag_range = (ctx->dmax >> drop) - tag_min;
        const uint32_t range_bits = static_cast<uint32_t>(bits_for(tag_range));
        // Top-level buckets: 2^14 up to 16 M splats, 2^15 above (config 3: 14 bits 0.82 vs 15 bits
        // 0.86 ms sort; config 4: 15 bits 2.40 ms vs the LSD passes' 2.59).
        const uint32_t top_bits = S32 > kBucketWideSplats ? static_cast<uint32_t>(kBucketTopBits) : 14u;
        const uint32_t local_bits = range_bits > top_bits ? range_bits - top_bits : 0u;
        const bool buckets = !presorted && !device_counts && (1u << local_bits) <= kBucketLocalBins &&
                             S32 <= ctx->bucket_max_splats;
        RadixPlan dplan{};
        if (!presorted && !buckets) {
            dplan = make_plan(dbits - drop);
            for (uint32_t q = 0; q < dplan.passes; ++q) dplan.shift[q] += drop;
        }
        CUDA_TRY(ctx->span_sorted.ensure(static_cast<size_t>(S32) * 8));
        int sb = 0;
        if (buckets) {
            DepthBucketParams bp{};
            bp.depth = ctx->depth().as<uint32_t>();
            bp.meta = ctx->meta().as<uint4>();
            bp.count = S32;
            bp.drop = drop;
            bp.tag_min = tag_min;
            bp.local_bits = local_bits;
            bp.buckets = (tag_range >> local_bits) + 1u;
            CUDA_TRY(ctx->buckets.ensure((3ull * kMaxDepthBuckets + 1) * 4));
            CUDA_TRY(ctx->bucket_staged.ensure(static_cast<size_t>(S32) * 16));
            bp.bucket_count = ctx->buckets.as<uint32_t>();
            bp.bucket_start = bp.bucket_count + kMaxDepthBuckets;
            bp.bucket_cursor = bp.bucket_start + kMaxDepthBuckets + 1;
            bp.staged = ctx->bucket_staged.as<uint4>();
            bp.keys_out = ctx->skeys[0].as<uint32_t>();
            bp.recs_out = ctx->srecs[0].as<uint32_t>();
            bp.spans_out = ctx->span_sorted.as<uint2>();
            CUDA_TRY(cudaMemsetAsync(bp.bucket_count, 0, bp.buckets * 4ull, s));
            const uint32_t grid = (S32 + kBucketTile - 1) / kBucketTile;
            CUDA_TRY(pdl_launch(k_depth_bucket_count, grid, kBucketThreads, bp.buckets * 4ull, s, bp));
            CUDA_TRY(pdl_launch(k_depth_bucket_scan, 1, 1024, 0, s, bp));
            CUDA_TRY(pdl_launch(k_depth_bucket_scatter, (S32 + kBucketScatterTile - 1) / kBucketScatterTile, kBucketThreads,
                                bp.buckets * 4ull, s, bp));
            CUDA_TRY(pdl_launch(k_depth_bucket_local, bp.buckets, kBucketLocalThreads, kBucketLocalCap * 16ull, s, bp));
            launches += 4;
            dplan.passes = 2;  // reported sort passes: the two bucket levels
        } else if (!presorted) {
            sb = run_radix(ctx, ctx->depth().as<uint32_t>(), nullptr, ctx->skeys, ctx->srecs, S32, dplan, launches,
                           s_dev, s);
        }
        const EmitCounts ec{s_dev};
        // 2. cell spans in sorted order; the first cell-sort digit histogram per emission
        //    block; digit offsets; pairs emitted straight into the order of the first stable
        //    cell-sort pass, each key word tagged with its splat's truncated depth.
        const uint32_t cell_bits = std::max(1, bits_for(cells - 1));
        const uint32_t cell_mask = cell_bits >= 32 ? 0xffffffffu : (1u << cell_bits) - 1u;
        const uint32_t emit_bits = std::min<uint32_t>(cell_bits, kRadixBits);  // the first pass, folded into emission
        const uint32_t dmask = (1u << emit_bits) - 1u;
        const uint32_t eblocks = (S32 + kEmitSplats - 1) / kEmitSplats;  // emission blocks
        CUDA_TRY(ctx->block_sums.ensure(static_cast<size_t>(eblocks) * kRadix * 4));
        const int quads = geo.cells_per_tile == 4 ? 1 : 0;
        const uint32_t* tag_keys = presorted ? nullptr : ctx->skeys[sb].as<uint32_t>();
        if (!buckets) {
            CUDA_TRY(pdl_launch(k_sorted_spans, (S32 + 1023) / 1024, kMetaThreads, 0, s, ctx->srecs[sb].as<uint32_t>(),
                                ctx->meta().as<uint4>(), S32, s_dev, ctx->span_sorted.as<uint2>()));
            ++launches;
        }
        launch_emit(true, eblocks, s, ctx->srecs[sb].as<uint32_t>(), tag_keys, S32, ctx->span_sorted.as<uint2>(),
                    ctx->block_sums.as<uint32_t>(), nullptr, rtx, quads, dmask, drop, cell_bits, nullptr, nullptr, ec);
        SortPassParams bp{};
        bp.counts = ctx->block_sums.as<uint32_t>();
        bp.digit_base = ctx->hist.as<uint32_t>();
        bp.tiles = eblocks;
        bp.bits = emit_bits;
        CUDA_TRY(pdl_launch(k_sort_rows, dmask + 1, 1024, 0, s, bp));
        launch_emit(false, eblocks, s, ctx->srecs[sb].as<uint32_t>(), tag_keys, S32, ctx->span_sorted.as<uint2>(),
                    ctx->block_sums.as<uint32_t>(), ctx->hist.as<uint32_t>(), rtx, quads, dmask, drop, cell_bits,
                    ctx->pcell()[1].as<uint32_t>(), ctx->precs()[1].as<uint32_t>(), ec);
        launches += 3;
        CUDA_TRY(cudaGetLastError());
        // 3. the remaining stable cell-sort passes (cell bits only; the tags ride along).
        RadixPlan rest{};
        if (cell_bits > emit_bits) {
            rest = make_plan(cell_bits - emit_bits);
            for (uint32_t q = 0; q < rest.passes; ++q) rest.shift[q] += emit_bits;
        }
        const int cb = rest.passes ? run_radix(ctx, ctx->pcell()[1].as<uint32_t>(), ctx->precs()[1].as<uint32_t>(),
                                               ctx->pcell(), ctx->precs(), K, rest, launches, k_dev, s)
                                   : 1;
        // 4. cell ranges + every run of equal (cell, tag) ordered by (depth bits, ordinal).
        const uint32_t long_cap = K / kLongRun + K / 2048 + 2;  // see k_cell_fixup
        CUDA_TRY(ctx->long_runs.ensure(static_cast<size_t>(long_cap) * 8 + 16));
        uint32_t* long_count = reinterpret_cast<uint32_t*>(ctx->long_runs.as<uint2>() + long_cap);
        CUDA_TRY(cudaMemsetAsync(long_count, 0, 4, s));
        const uint32_t kblocks = (K + 256 * kStreamItems - 1) / (256 * kStreamItems);  // 2048 pairs per CTA
        CUDA_TRY(pdl_launch(k_cell_fixup, kblocks, 256, 0, s, ctx->pcell()[cb].as<uint32_t>(), ctx->precs()[cb].as<uint32_t>(),
                                             ctx->meta().as<uint4>(), K, k_dev, cell_mask, presorted ? 0 : 1,
                                             ctx->ranges().as<uint2>(), ctx->long_runs.as<uint2>(), long_count, long_cap));
        ++launches;
        if (!presorted) {
            CUDA_TRY(pdl_launch(k_pair_long_runs, ctx->sm_count * 2, 256, 0, s, ctx->pcell()[cb].as<uint32_t>(), K, k_dev,
                                                              ctx->precs()[cb].as<uint32_t>(), ctx->meta().as<uint4>(),
                                                              ctx->long_runs.as<uint2>(), long_count));
            ++launches;
        }
        CUDA_TRY(cudaGetLastError());
        ctx->final_recs = ctx->precs()[cb].as<uint32_t>();
        passes = dplan.passes + 1 + rest.passes;
    }
    CUDA_TRY(cudaEventRecord(ctx->ev[4], s));
    if (split) {
        CUDA_TRY(cudaEventRecord(ctx->sort_done, s));
        CUDA_TRY(cudaStreamWaitEvent(rs_, ctx->sort_done, 0));
    }
    s = rs_;  // the raster and read-back on the render stream

    // ---- rasterize ----
    if (tiles) {
        RasterParams rp{};
        rp.ranges = ctx->ranges().as<uint2>();
        rp.recs = ctx->final_recs;
        rp.records = ctx->rec().as<float4>();
        rp.width = geo.W;
        rp.height = geo.H;
        rp.tile_size = geo.ts;
        rp.tiles_x = rtx;
        rp.tile_col0 = geo.band_tile_col0;
        rp.out_col0 = geo.band_x0;
        rp.out_stride = geo.band_x1 - geo.band_x0;
        rp.tile_row0 = tile_row0;
        rp.out_row0 = tile_row0 * geo.ts;
        for (int i = 0; i < 3; ++i) rp.bg[i] = ctx->settings.background[i];
        rp.alpha_max = ctx->settings.alpha_max;
        rp.t_floor = ctx->settings.transmittance_floor;
        rp.out_rgb = ctx->fb_rgb.as<float>();
        rp.out_T = ctx->fb_T.as<float>();
        if (!read_rgb && !read_T) {
            launch_raster(rp, tiles, s);
            ++launches;
        } else {
            // Host read-back overlapped with the raster: tile-row bands are rasterised in
            // order and each band's rows are copied out on the copy stream while the next
            // band renders. Pipelined frames overlap the read-back with the next frame
            // instead, so their raster stays one launch (no per-band tail).
            const int bands = pipelined ? 1 : std::min(kReadbackBands, tile_rows);
            const size_t row_floats = static_cast<size_t>(geo.band_x1 - geo.band_x0);
            for (int b = 0; b < bands; ++b) {
                const int r0 = tile_rows * b / bands, r1 = tile_rows * (b + 1) / bands;
                if (r1 <= r0) continue;
                RasterParams bp = rp;
                bp.ranges = rp.ranges + static_cast<size_t>(r0) * rtx * geo.cells_per_tile;
                bp.tile_row0 = tile_row0 + r0;
                launch_raster(bp, static_cast<uint32_t>((r1 - r0) * rtx), s);
                ++launches;
                const int y0 = r0 * geo.ts, y1 = std::min(r1 * geo.ts, geo.H - tile_row0 * geo.ts);
                const size_t off = static_cast<size_t>(y0) * row_floats, n = static_cast<size_t>(y1 - y0) * row_floats;
                if (pipelined) {  // deferred to the next call (flush_readback)
                    CUDA_TRY(cudaEventRecord(ctx->pend_ev, s));
                    auto& pr = ctx->pending;
                    pr.active = true;
                    pr.dst_rgb = read_rgb ? read_rgb + 3 * off : nullptr;
                    pr.dst_T = read_T ? read_T + off : nullptr;
                    pr.src_rgb = ctx->fb_rgb.as<float>() + 3 * off;
                    pr.src_T = ctx->fb_T.as<float>() + off;
                    pr.rgb_bytes = n * 12;
                    pr.T_bytes = n * 4;
                    pr.done = ctx->pend_ev;
                    pr.rb = ctx->rb_ev;  // gscg_wait_readback waits on rb_ev
                    continue;
                }
                CUDA_TRY(cudaEventRecord(ctx->band_ev[b], s));
                CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, ctx->band_ev[b], 0));
                if (read_rgb)
                    CUDA_TRY(cudaMemcpyAsync(read_rgb + 3 * off, ctx->fb_rgb.as<float>() + 3 * off, n * 12,
                                             cudaMemcpyDefault, ctx->copy_stream));
                if (read_T)
                    CUDA_TRY(cudaMemcpyAsync(read_T + off, ctx->fb_T.as<float>() + off, n * 4, cudaMemcpyDefault,
                                             ctx->copy_stream));
            }
            if (!pipelined) {
                // The frame's stream resumes only after the read-back (ordering for the caller).
                CUDA_TRY(cudaEventRecord(ctx->band_ev[kReadbackBands - 1], ctx->copy_stream));
                CUDA_TRY(cudaStreamWaitEvent(s, ctx->band_ev[kReadbackBands - 1], 0));
            }
        }
        CUDA_TRY(cudaGetLastError());
    } else if (read_rgb || read_T) {
        copy_out(ctx, geo.H - tile_row0 * geo.ts, read_rgb, read_T, true);
    }
    CUDA_TRY(cudaEventRecord(ctx->ev[5], s));
    ctx->tiles = tiles;
    ctx->cells_per_tile = geo.cells_per_tile;
    return passes;
}

// D2H (host mode) or D2D of `rows` framebuffer rows starting at the context's row 0.
void copy_out(gscg_ctx* ctx, int rows, float* fb_rgb, float* fb_T, bool host) {
    cudaStream_t s = ctx->stream;
    const size_t px = static_cast<size_t>(ctx->geom.band_x1 - ctx->geom.band_x0) * rows;  // region width
    // Destinations may be host (pinned or pageable) or device memory in either mode: the
    // direction comes from unified addressing.
    (void)host;
    if (fb_rgb && px) CUDA_TRY(cudaMemcpyAsync(fb_rgb, ctx->fb_rgb.ptr, px * 12, cudaMemcpyDefault, s));
    if (fb_T && px) CUDA_TRY(cudaMemcpyAsync(fb_T, ctx->fb_T.ptr, px * 4, cudaMemcpyDefault, s));
}

void fill_times(gscg_ctx* ctx, gscg_stage_times* times, uint32_t passes, uint32_t launches) {
    times->h2d_ms = elapsed(ctx->ev[0], ctx->ev[1]);
    times->update_ms = elapsed(ctx->ev[1], ctx->ev[2]);
    times->gather_ms = elapsed(ctx->ev[2], ctx->ev[3]);
    times->sort_ms = elapsed(ctx->ev[3], ctx->ev[4]);
    times->rasterize_ms = elapsed(ctx->ev[4], ctx->ev[5]);
    times->d2h_ms = elapsed(ctx->ev[5], ctx->ev[6]);
    times->splat_count = ctx->S;
    times->pair_count = ctx->K;
    times->gaussian_count = ctx->G;
    times->tile_pair_count = ctx->TP;
    times->sort_passes = passes;
    times->kernel_launches = launches;
}

}  // namespace

extern "C" {

int gscg_device_count(int* out) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    if (out) *out = n;
    return GSCG_OK;
}

int gscg_create(int device, gscg_ctx** out) {
    if (!out) return GSCG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    auto* ctx = new gscg_ctx();
    ctx->device = device;
    const int st = guarded(ctx, [&] {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            throw Status(GSCG_ERR_CUDA, "no CUDA device: the B200 render path has no CPU fallback");
        if (device < 0 || device >= count) invalid("device index out of range");
        CUDA_TRY(cudaSetDevice(device));
        cudaDeviceProp prop{};
        CUDA_TRY(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            throw Status(GSCG_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 (Blackwell)");
        ctx->sm_count = prop.multiProcessorCount;
        if (const char* e = std::getenv("GSCG_DEPTH_SORT_BITS")) {  // tuning knob (see kDepthSortBits)
            const int v = std::atoi(e);
            if (v >= 1 && v <= 32) ctx->depth_sort_bits = static_cast<uint32_t>(v);
        }
        if (const char* e = std::getenv("GSCG_BUCKET_MAX_SPLATS"))  // A/B knob: 0 = LSD depth passes always
            ctx->bucket_max_splats = std::strtoull(e, nullptr, 10);
        for (auto& e : ctx->ev) CUDA_TRY(cudaEventCreate(&e));
        for (auto& e : ctx->band_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->rb_ev, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->rb_ev_alt, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->pend_ev, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->counters_ev, cudaEventDisableTiming));
        {
            // Stream priorities, oldest work first: a pipelined frame's raster (render
            // stream) above the next frame's sort, the sort above the front half. Measured
            // at config 3 (device / e2e FPS): 628 / 606 against 627 / 604 with equal
            // priorities; the front half first (GSCG_STREAM_PRIO=1) 619 / 608, with the sort
            // above the raster as well (=2) 590 / 581. GSCG_STREAM_PRIO=0..5 is the A/B knob.
            static const int mode = [] {
                const char* e = std::getenv("GSCG_STREAM_PRIO");
                return e ? std::atoi(e) : 3;
            }();
            int least = 0, greatest = 0;
            CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            const int mid = (least + greatest) / 2;
            int p_upd = least, p_sort = least, p_rs = least;
            if (mode == 1) p_upd = greatest;
            if (mode == 2) p_upd = greatest, p_sort = mid;
            if (mode == 3) p_rs = greatest, p_sort = mid;
            if (mode == 4) p_rs = greatest;
            if (mode == 5) p_upd = greatest, p_rs = mid;
            CUDA_TRY(cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, p_rs));
            CUDA_TRY(cudaStreamCreateWithPriority(&ctx->upd_stream, cudaStreamNonBlocking, p_upd));
            CUDA_TRY(cudaStreamCreateWithPriority(&ctx->sort_stream, cudaStreamNonBlocking, p_sort));
        }
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->sort_done, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->upd_ok, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->upd_done, cudaEventDisableTiming));
        for (auto& e : ctx->slot_free) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_counters), sizeof(FrameCounters)));
        CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_band_counts), GSCG_MAX_BANDS * sizeof(unsigned long long)));
        CUDA_TRY(ctx->counters.ensure(sizeof(FrameCounters)));
        CUDA_TRY(cudaFuncSetAttribute(k_fk_skin, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (kFkThreads / 16) * kFkSmemPerInstance(kMaxJoints)));
        CUDA_TRY(cudaFuncSetAttribute(k_project<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kProjectThreads * kShFloats * 4 + kBatch * kMaxJoints * 12 * 4));
        CUDA_TRY(cudaFuncSetAttribute(k_project<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kProjectThreads * kShFloats * 4 + kBatch * kMaxJoints * 12 * 4));
        CUDA_TRY(cudaFuncSetAttribute(k_project<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kProjectThreads * kShFloats * 4 + kBatch * kMaxJoints * 12 * 4));
        CUDA_TRY(cudaFuncSetAttribute(k_depth_bucket_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kMaxDepthBuckets * 4));
        CUDA_TRY(cudaFuncSetAttribute(k_depth_bucket_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kMaxDepthBuckets * 4));
        CUDA_TRY(cudaFuncSetAttribute(k_depth_bucket_local, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kBucketLocalCap * 16));
    });
    *out = ctx;
    return st;
}

int gscg_destroy(gscg_ctx* ctx) {
    if (!ctx) return GSCG_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_stream) {
        try {
            flush_readback(ctx);  // a deferred pipelined read-back still lands
        } catch (...) {
        }
        cudaStreamSynchronize(ctx->copy_stream);  // pipelined read-backs
    }
    for (TemplateStore& t : ctx->templates)
        for (LevelStore& l : t.levels) {
            l.core.release();
            l.weights.release();
            l.sh.release();
        }
    DevBuf* bufs[] = {&ctx->d_templates, &ctx->d_groups, &ctx->d_mats, &ctx->d_parents,
                      &ctx->template_ids, &ctx->placement, &ctx->poses, &ctx->lod_prev,
                      &ctx->lod_out, &ctx->inst_group, &ctx->inst_base, &ctx->members, &ctx->visible,
                      &ctx->group_inst_start, &ctx->group_inst_count, &ctx->group_item_start,
                      &ctx->skin, &ctx->counters, &ctx->records_s[0], &ctx->records_s[1], &ctx->splat_meta_s[0], &ctx->splat_meta_s[1],
                      &ctx->splat_depth_s[0], &ctx->splat_depth_s[1], &ctx->skeys[0], &ctx->skeys[1], &ctx->srecs[0], &ctx->srecs[1],
                      &ctx->pcell_s[0][0], &ctx->pcell_s[0][1], &ctx->precs_s[0][0], &ctx->precs_s[0][1],
                      &ctx->pcell_s[1][0], &ctx->pcell_s[1][1], &ctx->precs_s[1][0], &ctx->precs_s[1][1], &ctx->span_sorted,
                      &ctx->block_sums, &ctx->hist, &ctx->status, &ctx->ranges_s[0], &ctx->ranges_s[1], &ctx->sorted_ordinals, &ctx->fb_rgb,
                      &ctx->fb_T, &ctx->posed_dbg, &ctx->rec_dbg, &ctx->band_scratch, &ctx->d_motions, &ctx->d_roots,
                      &ctx->d_keys, &ctx->motion_ids, &ctx->phases, &ctx->long_runs, &ctx->fb_rgb_alt,
                      &ctx->fb_T_alt};
    for (DevBuf* b : bufs) b->release();
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->h_counters) cudaFreeHost(ctx->h_counters);
    if (ctx->h_lod) cudaFreeHost(ctx->h_lod);
    if (ctx->h_band_counts) cudaFreeHost(ctx->h_band_counts);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->band_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->rb_ev) cudaEventDestroy(ctx->rb_ev);
    if (ctx->rb_ev_alt) cudaEventDestroy(ctx->rb_ev_alt);
    if (ctx->pend_ev) cudaEventDestroy(ctx->pend_ev);
    if (ctx->counters_ev) cudaEventDestroy(ctx->counters_ev);
    if (ctx->upd_stream) {
        cudaStreamSynchronize(ctx->upd_stream);
        cudaStreamDestroy(ctx->upd_stream);
    }
    if (ctx->sort_stream) {
        cudaStreamSynchronize(ctx->sort_stream);
        cudaStreamDestroy(ctx->sort_stream);
    }
    if (ctx->sort_done) cudaEventDestroy(ctx->sort_done);
    if (ctx->upd_ok) cudaEventDestroy(ctx->upd_ok);
    if (ctx->upd_done) cudaEventDestroy(ctx->upd_done);
    for (auto& e : ctx->slot_free)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return GSCG_OK;
}

const char* gscg_last_error(const gscg_ctx* ctx) { return ctx ? ctx->error.c_str() : "null context"; }

int gscg_set_region(gscg_ctx* ctx, int32_t x0, int32_t y0, int32_t x1, int32_t y1) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (x0 < 0 || y0 < 0 || x1 < x0 || y1 < y0) invalid("gscg_set_region: bad rectangle");
        ctx->col_req0 = x0;
        ctx->col_req1 = x1;
        ctx->band_req0 = y0;
        ctx->band_req1 = y1;
    });
}

int gscg_set_band(gscg_ctx* ctx, int32_t row_begin, int32_t row_end) {
    return gscg_set_region(ctx, 0, row_begin, 0, row_end);
}

int gscg_set_layout(gscg_ctx* ctx, int32_t layout) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (layout != GSCG_LAYOUT_SHARED && layout != GSCG_LAYOUT_NAIVE) invalid("gscg_set_layout: unknown layout");
        ctx->layout = layout;
        if (layout == GSCG_LAYOUT_SHARED) {  // the per-instance copies go away with the mode
            CUDA_TRY(cudaStreamSynchronize(ctx->stream));
            ctx->naive_core.release();
            ctx->naive_w.release();
            ctx->naive_valid = false;
        }
    });
}

int gscg_set_debug(gscg_ctx* ctx, uint32_t flags) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    ctx->debug = flags;
    return GSCG_OK;
}

int gscg_upload_skeleton(gscg_ctx* ctx, uint32_t template_id, const gscg_skeleton_desc* d) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (!d || !d->parents || !d->local_bind || !d->inverse_bind) invalid("null skeleton field");
        if (d->joint_count < 1 || d->joint_count > GSCG_MAX_JOINTS) invalid("joint_count outside [1, 64]");
        if (d->parents[0] >= 0) invalid("Skeleton: exactly one root at index 0 required");
        for (uint32_t j = 1; j < d->joint_count; ++j)
            if (d->parents[j] < 0 || static_cast<uint32_t>(d->parents[j]) >= j)
                invalid("Skeleton: parent index must precede child");
        if (template_id >= ctx->templates.size()) ctx->templates.resize(template_id + 1);
        TemplateStore& t = ctx->templates[template_id];
        t.present = true;
        t.joint_count = d->joint_count;
        t.parents.assign(d->parents, d->parents + d->joint_count);
        t.local_bind.assign(d->local_bind, d->local_bind + 16 * d->joint_count);
        t.inverse_bind.assign(d->inverse_bind, d->inverse_bind + 16 * d->joint_count);
        t.pelvis_y = d->pelvis_y;
        ctx->tables_dirty = true;
    });
}

int gscg_upload_template(gscg_ctx* ctx, uint32_t template_id, uint32_t level, const gscg_level_desc* desc) {
    return gscg_upload_level(ctx, template_id, level, desc);
}

int gscg_upload_level(gscg_ctx* ctx, uint32_t template_id, uint32_t level, const gscg_level_desc* d) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        if (template_id >= ctx->templates.size() || !ctx->templates[template_id].present)
            invalid("upload the skeleton before its levels");
        if (!d || !d->means || !d->cov6 || !d->opacities || !d->colors || !d->skin_indices || !d->skin_weights)
            invalid("null level field");
        const uint32_t n = d->gaussian_count;
        if (n == 0) invalid("LodLevel: empty");
        TemplateStore& t = ctx->templates[template_id];
        if (level > t.levels.size()) invalid("levels must be uploaded in order");
        if (level == t.levels.size()) t.levels.emplace_back();
        LevelStore& ls = t.levels[level];
        for (uint32_t i = 0; i < n; ++i)
            for (int k = 0; k < 4; ++k)
                if (d->skin_indices[4 * i + k] >= t.joint_count) invalid("LodLevel: skin index out of range");
        std::vector<float> core(static_cast<size_t>(n) * 16);
        for (uint32_t i = 0; i < n; ++i) {
            float* c = core.data() + 16 * static_cast<size_t>(i);
            c[0] = d->means[3 * i + 0];
            c[1] = d->means[3 * i + 1];
            c[2] = d->means[3 * i + 2];
            c[3] = d->opacities[i];
            for (int k = 0; k < 6; ++k) (k < 4 ? c[4 + k] : c[8 + (k - 4)]) = d->cov6[6 * i + k];
            c[10] = d->colors[3 * i + 0];
            c[11] = d->colors[3 * i + 1];
            c[12] = d->colors[3 * i + 2];
            c[13] = 0.0f;  // power floor, filled per alpha_cutoff
            const uint32_t i01 = d->skin_indices[4 * i + 0] | (static_cast<uint32_t>(d->skin_indices[4 * i + 1]) << 16);
            const uint32_t i23 = d->skin_indices[4 * i + 2] | (static_cast<uint32_t>(d->skin_indices[4 * i + 3]) << 16);
            std::memcpy(&c[14], &i01, 4);
            std::memcpy(&c[15], &i23, 4);
        }
        ls.count = n;
        CUDA_TRY(ls.core.ensure_exact(core.size() * sizeof(float)));
        CUDA_TRY(cudaMemcpyAsync(ls.core.ptr, core.data(), core.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_TRY(ls.weights.ensure_exact(static_cast<size_t>(n) * 16));
        CUDA_TRY(cudaMemcpyAsync(ls.weights.ptr, d->skin_weights, static_cast<size_t>(n) * 16, cudaMemcpyHostToDevice, ctx->stream));
        ls.has_sh = d->sh != nullptr;
        if (ls.has_sh) {
            // Pad to a whole 256-Gaussian chunk so chunk copies stay in bounds.
            const size_t chunks = (n + kProjectThreads - 1) / kProjectThreads;
            const size_t bytes = chunks * kProjectThreads * kShFloats * sizeof(float);
            CUDA_TRY(ls.sh.ensure_exact(bytes));
            CUDA_TRY(cudaMemsetAsync(ls.sh.ptr, 0, bytes, ctx->stream));
            CUDA_TRY(cudaMemcpyAsync(ls.sh.ptr, d->sh, static_cast<size_t>(n) * kShFloats * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        } else {
            ls.sh.release();
        }
        ls.opacities.assign(d->opacities, d->opacities + n);
        ls.pf_cutoff = -1.0f;
        {  // instance-cull bounds, rounded up; non-finite input disables the cull
            double mr = 0.0, s2 = 0.0, wa = 0.0, wd = 0.0;
            bool finite = true;
            for (uint32_t i = 0; i < n; ++i) {
                const float* m = d->means + 3ull * i;
                const float* cv = d->cov6 + 6ull * i;
                const float* w = d->skin_weights + 4ull * i;
                const double r2 = double(m[0]) * m[0] + double(m[1]) * m[1] + double(m[2]) * m[2];
                const double g0 = std::fabs(double(cv[0])) + std::fabs(double(cv[1])) + std::fabs(double(cv[2]));
                const double g1 = std::fabs(double(cv[1])) + std::fabs(double(cv[3])) + std::fabs(double(cv[4]));
                const double g2 = std::fabs(double(cv[2])) + std::fabs(double(cv[4])) + std::fabs(double(cv[5]));
                double sa = 0.0, sw = 0.0;
                for (int k = 0; k < 4; ++k) {
                    sa += std::fabs(double(w[k]));
                    sw += double(w[k]);
                }
                finite = finite && std::isfinite(r2) && std::isfinite(g0) && std::isfinite(g1) && std::isfinite(g2) &&
                         std::isfinite(sa);
                mr = std::max(mr, r2);
                s2 = std::max(s2, std::max(g0, std::max(g1, g2)));
                wa = std::max(wa, sa);
                wd = std::max(wd, std::fabs(sw - 1.0));
            }
            auto up = [](double v) { return static_cast<float>(v * (1.0 + 1e-6) + 1e-12); };
            ls.mean_r = finite ? up(std::sqrt(mr)) : INFINITY;
            ls.sigma = finite ? up(std::sqrt(s2)) : INFINITY;
            ls.wabs = finite ? up(wa) : INFINITY;
            ls.wdev = finite ? up(wd) : INFINITY;
        }
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        ctx->tables_dirty = true;
    });
}

int gscg_upload_motion(gscg_ctx* ctx, uint32_t motion_id, const gscg_motion_desc* d) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (!d || !d->frames) invalid("null motion");
        if (!(d->fps > 0.0f)) invalid("MotionClip: fps must be > 0");
        if (d->frame_count < 1) invalid("sample_pose: empty clip");
        if (d->joint_count < 1 || d->joint_count > GSCG_MAX_JOINTS) invalid("MotionClip: joint count outside [1, 64]");
        if (motion_id > ctx->motions.size()) invalid("motion id beyond the store");
        MotionStore m;
        m.fps = d->fps;
        m.frames = d->frame_count;
        m.joints = d->joint_count;
        const size_t rec = 4 + 4 * static_cast<size_t>(m.joints);
        m.roots.resize(m.frames);
        m.keys.resize(static_cast<size_t>(m.frames) * m.joints);
        for (uint32_t f = 0; f < m.frames; ++f) {
            const float* a = d->frames + f * rec;
            const float* b = d->frames + ((f + 1) % m.frames) * rec;
            m.roots[f] = make_float4(a[0], a[1], a[2], 0.0f);
            for (uint32_t j = 0; j < m.joints; ++j) {
                const float* qa = a + 4 + 4 * j;
                const float* qb = b + 4 + 4 * j;
                // slerp_shortest's angle terms (avatar.cpp:226-245) with the host libm.
                float dot = (qa[0] * qb[0] + qa[2] * qb[2]) + (qa[1] * qb[1] + qa[3] * qb[3]);
                float sgn = 1.0f;
                if (dot < 0.0f) {
                    dot = -dot;
                    sgn = -1.0f;
                }
                KeyPairDev& k = m.keys[static_cast<size_t>(f) * m.joints + j];
                k.a = make_float4(qa[0], qa[1], qa[2], qa[3]);
                k.b = sgn < 0.0f ? make_float4(-qb[0], -qb[1], -qb[2], -qb[3]) : make_float4(qb[0], qb[1], qb[2], qb[3]);
                k.lerp = dot > 0.9995f ? 1u : 0u;
                k.theta = k.lerp ? 0.0f : std::acos(std::min(dot, 1.0f));
                k.sin_theta = k.lerp ? 1.0f : std::sin(k.theta);
                k.pad = 0;
            }
        }
        if (motion_id == ctx->motions.size()) ctx->motions.push_back(std::move(m));
        else ctx->motions[motion_id] = std::move(m);
        ctx->motions_dirty = true;
    });
}

int gscg_template_bytes(const gscg_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    uint64_t b = 0;
    for (const TemplateStore& t : ctx->templates)
        for (const LevelStore& l : t.levels) b += l.core.cap + l.weights.cap + l.sh.cap;
    *out = b;
    return GSCG_OK;
}

namespace {
int render_frame_impl(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                      const gscg_render_settings* settings, const gscg_lod_policy* lod, float* fb_rgb,
                      float* fb_T, gscg_stage_times* times, bool pipelined) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        validate_frame(ctx, frame, cam, settings, lod);
        apply_band(ctx);
        const bool host = frame->memory == GSCG_MEM_HOST;
        const uint32_t n = frame->instance_count;
        uint32_t launches = 0;
        ctx->band_state = 0;
        // The frame is enqueued whole before the host reads its counters: update + gather,
        // then the sort and raster sized by the capacities and counted on the device
        // (deferred), then the host waits for the counters (mid-frame, while the GPU runs
        // on). A frame whose splats or pairs outgrew the capacities is rendered again with
        // them grown (settle_counts); the first frame of a context usually is.
        // Host destinations: read-back overlapped with the raster bands (sort_raster).
        // Device destinations: one device-to-device copy after the frame.
        const bool overlap = is_host_pointer(fb_rgb) || is_host_pointer(fb_T);
        pipelined = pipelined && overlap;
        const FrameGeom& g = ctx->geom;  // a region frame renders its tiles only
        auto enqueue_sort = [&](bool device_counts) {
            return overlap ? sort_raster(ctx, g.band_tile_row0, g.band_tile_rows, launches, fb_rgb, fb_T, false,
                                         pipelined, device_counts)
                           : sort_raster(ctx, g.band_tile_row0, g.band_tile_rows, launches, nullptr, nullptr, false,
                                         false, device_counts);
        };
        // Deferred frames are opt-in (GSCG_DEFER=1): measured neutral on the device and 6-10%
        // slower end to end at configs 1-3 (capacity-sized grids).
        static const bool defer = [] {
            const char* e = std::getenv("GSCG_DEFER");
            return e && e[0] == '1';
        }();
        const bool deferred = defer && ctx->splat_capacity > 0 && ctx->pair_capacity > 0 &&
                              !(ctx->debug & GSCG_DEBUG_POSED);
        t_pdl_frame = ctx->S < pdl_max_splats();
        uint32_t passes;
        nvtxRangePushA("gscg_render_frame");  // host-side ranges for nsys / ncu --nvtx
        if (deferred) {
            update_gather(ctx, frame, cam, lod, 0, n, launches, host, true);
            passes = enqueue_sort(true);
            nvtxRangePushA("settle_counts");
            const bool fits = settle_counts(ctx, frame, n, host, false, true);
            nvtxRangePop();
            if (!fits) {
                nvtxRangePushA("re-render (capacity grown)");
                update_gather(ctx, frame, cam, lod, 0, n, launches, host);  // host: active_lod written back here
                passes = enqueue_sort(false);
                nvtxRangePop();
            }
        } else {
            // Frame pipelining: the front half on the update stream into the other slot (frames
            // past kPipelineMaxSplats keep one slot: the second would not fit with them).
            const bool front = overlap_update() && ctx->S <= kPipelineMaxSplats;
            if (front) ctx->slot ^= 1;
            update_gather(ctx, frame, cam, lod, 0, n, launches, host, false, front);
            if (front) {
                if (n && !host)  // the LoD write-back (lod_out is final) ends the front half
                    CUDA_TRY(cudaMemcpyAsync(frame->active_lod, ctx->lod_out.ptr, n * 4ull, cudaMemcpyDeviceToDevice,
                                             ctx->upd_stream));
                CUDA_TRY(cudaEventRecord(ctx->upd_done, ctx->upd_stream));
                CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->upd_done, 0));  // the back half follows
            }
            passes = enqueue_sort(false);
            if (front) {
                CUDA_TRY(cudaEventRecord(ctx->slot_free[ctx->slot], ctx->stream));
                ctx->slot_free_rec[ctx->slot] = true;
            }
        }
        nvtxRangePop();
        if (!overlap) copy_out(ctx, g.band_y1 - g.band_y0, fb_rgb, fb_T, host);  // region rows x region width
        if (n && !host && !ctx->front_active)
            CUDA_TRY(cudaMemcpyAsync(frame->active_lod, ctx->lod_out.ptr, n * 4ull, cudaMemcpyDeviceToDevice,
                                     ctx->stream));
        CUDA_TRY(cudaEventRecord(ctx->ev[6], ctx->stream));
        if (pipelined) {
            // No host synchronisation: the next frame's inputs go in while this one's raster
            // and read-back finish. Counts are known (mid-frame read-back); stage times are not.
            if (times) {
                *times = gscg_stage_times{};
                times->splat_count = ctx->S;
                times->pair_count = ctx->K;
                times->gaussian_count = ctx->G;
                times->tile_pair_count = ctx->TP;
                times->kernel_launches = launches;
            }
            return;
        }
        if (host || times) CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        if (times) fill_times(ctx, times, passes, launches);
    });
}
}  // namespace

int gscg_render_frame(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                      const gscg_render_settings* settings, const gscg_lod_policy* lod,
                      float* fb_rgb, float* fb_T, gscg_stage_times* times) {
    return render_frame_impl(ctx, frame, cam, settings, lod, fb_rgb, fb_T, times, false);
}

int gscg_render_frame_async(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                            const gscg_render_settings* settings, const gscg_lod_policy* lod,
                            float* fb_rgb, float* fb_T, gscg_stage_times* times) {
    return render_frame_impl(ctx, frame, cam, settings, lod, fb_rgb, fb_T, times, true);
}

int gscg_wait_readback(gscg_ctx* ctx, uint32_t frames_back) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        flush_readback(ctx);
        if (frames_back == 0) CUDA_TRY(cudaEventSynchronize(ctx->rb_ev));
        else if (frames_back == 1) CUDA_TRY(cudaEventSynchronize(ctx->rb_ev_alt));
    });
}

int gscg_project_shard(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                       const gscg_render_settings* settings, const gscg_lod_policy* lod,
                       uint32_t shard_begin, uint32_t shard_end, uint32_t bands, const uint32_t* band_rows,
                       uint64_t* band_counts, gscg_stage_times* times) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        validate_frame(ctx, frame, cam, settings, lod);
        const uint32_t n = frame->instance_count;
        if (shard_begin > shard_end || shard_end > n) invalid("instance shard outside [0, instance_count]");
        if (bands < 1 || bands > GSCG_MAX_BANDS || !band_rows || !band_counts) invalid("bad screen band table");
        const FrameGeom& geo = ctx->geom;
        if (band_rows[0] != 0 || band_rows[bands] != static_cast<uint32_t>(geo.H))
            invalid("screen bands must cover rows [0, height)");
        for (uint32_t b = 0; b < bands; ++b) {
            if (band_rows[b + 1] < band_rows[b]) invalid("screen band rows must be non-decreasing");
            if (band_rows[b] % static_cast<uint32_t>(geo.ts) != 0) invalid("screen bands must start on a tile row");
        }
        ctx->band_state = 0;
        uint32_t launches = 0;
        update_gather(ctx, frame, cam, lod, shard_begin, shard_end, launches);
        if (frame->memory == GSCG_MEM_HOST) {
            if (n) CUDA_TRY(cudaMemcpyAsync(frame->active_lod, ctx->lod_out.ptr, n * 4ull, cudaMemcpyDeviceToHost, ctx->stream));
        } else if (n) {
            CUDA_TRY(cudaMemcpyAsync(frame->active_lod, ctx->lod_out.ptr, n * 4ull, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        // Route: splats per destination band.
        BandParams& bp = ctx->band;
        bp = BandParams{};
        bp.records = ctx->rec().as<float4>();
        bp.meta = ctx->meta().as<uint4>();
        bp.depth = ctx->depth().as<uint32_t>();
        bp.count = static_cast<uint32_t>(ctx->S);
        bp.bands = bands;
        for (uint32_t b = 0; b <= bands; ++b) bp.rows[b] = band_rows[b];
        CUDA_TRY(ctx->band_scratch.ensure(2 * kMaxBands * sizeof(unsigned long long)));
        bp.band_counts = ctx->band_scratch.as<unsigned long long>();
        bp.band_cursor = bp.band_counts + kMaxBands;
        CUDA_TRY(cudaMemsetAsync(ctx->band_scratch.ptr, 0, 2 * kMaxBands * sizeof(unsigned long long), ctx->stream));
        const uint32_t grid = (bp.count + 256 * kStreamItems - 1) / (256 * kStreamItems);
        if (grid) {
            k_band_count<<<grid, 256, 0, ctx->stream>>>(bp);
            ++launches;
            CUDA_TRY(cudaGetLastError());
        }
        CUDA_TRY(cudaMemcpyAsync(ctx->h_band_counts, bp.band_counts, bands * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaEventRecord(ctx->ev[4], ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        unsigned long long off = 0;
        for (uint32_t b = 0; b < bands; ++b) {
            band_counts[b] = ctx->h_band_counts[b];
            bp.band_offsets[b] = off;
            off += ctx->h_band_counts[b];
        }
        ctx->band_total = off;
        ctx->band_state = 1;
        ctx->launches = launches;
        if (times) {
            *times = gscg_stage_times{};
            times->h2d_ms = elapsed(ctx->ev[0], ctx->ev[1]);
            times->update_ms = elapsed(ctx->ev[1], ctx->ev[2]);
            times->gather_ms = elapsed(ctx->ev[2], ctx->ev[3]);
            times->sort_ms = elapsed(ctx->ev[3], ctx->ev[4]);  // routing
            times->splat_count = ctx->S;
            times->gaussian_count = ctx->G;
            times->kernel_launches = launches;
        }
    });
}

int gscg_pack_bands(gscg_ctx* ctx, void* send_dev) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        if (ctx->band_state != 1) throw Status(GSCG_ERR_STATE, "gscg_pack_bands needs gscg_project_shard first");
        if (!send_dev && ctx->band_total) invalid("null send buffer");
        BandParams bp = ctx->band;
        bp.packed = static_cast<uint4*>(send_dev);
        const uint32_t grid = (bp.count + 256 * kStreamItems - 1) / (256 * kStreamItems);
        if (grid && ctx->band_total) {
            k_band_pack<<<grid, 256, 0, ctx->stream>>>(bp);
            CUDA_TRY(cudaGetLastError());
        }
        ctx->band_state = 2;
    });
}

int gscg_render_band(gscg_ctx* ctx, const void* recv_dev, uint64_t recv_count, uint32_t row_begin, uint32_t row_end,
                     float* fb_rgb, float* fb_T, int32_t memory, gscg_stage_times* times) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        if (ctx->band_state < 1) throw Status(GSCG_ERR_STATE, "gscg_render_band needs gscg_project_shard first");
        const FrameGeom& geo = ctx->geom;
        if (row_begin > row_end || row_end > static_cast<uint32_t>(geo.H) || row_begin % geo.ts != 0 ||
            (row_end % geo.ts != 0 && row_end != static_cast<uint32_t>(geo.H)))
            invalid("band rows must be tile-aligned and inside the frame");
        if (recv_count && !recv_dev) invalid("null receive buffer");
        if (recv_count > 0xF0000000ull) throw Status(GSCG_ERR_OOM, "band splat count exceeds 32-bit indexing");
        cudaStream_t s = ctx->stream;
        uint32_t launches = 0;
        CUDA_TRY(cudaEventRecord(ctx->ev[0], s));
        // The band's splats replace the context's records (the shard's were packed already).
        const uint64_t cap = std::max<uint64_t>(recv_count, 1);
        if (cap > ctx->splat_capacity) ctx->splat_capacity = cap + cap / 4;
        CUDA_TRY(ctx->rec().ensure(ctx->splat_capacity * 48));
        CUDA_TRY(ctx->meta().ensure(ctx->splat_capacity * 16));
        CUDA_TRY(ctx->depth().ensure(ctx->splat_capacity * 4));
        FrameCounters init{};
        init.depth_min_bits = 0xffffffffu;
        *ctx->h_counters = init;
        auto* counters = ctx->counters.as<FrameCounters>();
        CUDA_TRY(cudaMemcpyAsync(counters, ctx->h_counters, sizeof(FrameCounters), cudaMemcpyHostToDevice, s));
        BandUnpackParams up{};
        up.packed = static_cast<const uint4*>(recv_dev);
        up.count = static_cast<uint32_t>(recv_count);
        up.row_begin = static_cast<int32_t>(row_begin);
        up.row_end = static_cast<int32_t>(row_end);
        up.cell = geo.cell;
        up.records = ctx->rec().as<float4>();
        up.depth = ctx->depth().as<uint32_t>();
        up.meta = ctx->meta().as<uint4>();
        up.counters = counters;
        const uint32_t grid = (up.count + 256 * kStreamItems - 1) / (256 * kStreamItems);
        if (grid) {
            k_band_unpack<<<grid, 256, 0, s>>>(up);
            ++launches;
            CUDA_TRY(cudaGetLastError());
        }
        CUDA_TRY(cudaMemcpyAsync(ctx->h_counters, counters, sizeof(FrameCounters), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaEventRecord(ctx->ev[3], s));
        CUDA_TRY(cudaStreamSynchronize(s));
        ctx->S = recv_count;
        ctx->K = ctx->h_counters->pairs;
        if (ctx->K > 0xF0000000ull) throw Status(GSCG_ERR_OOM, "band pair count exceeds 32-bit indexing");
        ctx->dmin = ctx->h_counters->depth_min_bits;
        ctx->dmax = ctx->h_counters->depth_max_bits;
        const int tile_row0 = static_cast<int>(row_begin) / geo.ts;
        const int tile_rows = (static_cast<int>(row_end) - static_cast<int>(row_begin) + geo.ts - 1) / geo.ts;
        const uint32_t passes = sort_raster(ctx, tile_row0, tile_rows, launches);
        const bool host = memory == GSCG_MEM_HOST;
        copy_out(ctx, static_cast<int>(row_end - row_begin), fb_rgb, fb_T, host);
        CUDA_TRY(cudaEventRecord(ctx->ev[6], s));
        if (host || times) CUDA_TRY(cudaStreamSynchronize(s));
        ctx->band_row0 = row_begin;
        ctx->band_state = 3;
        if (times) {
            fill_times(ctx, times, passes, launches);
            times->h2d_ms = 0.0f;
            times->update_ms = 0.0f;
            times->gather_ms = elapsed(ctx->ev[0], ctx->ev[3]);  // unpack
        }
    });
}

int gscg_memory_usage(gscg_ctx* ctx, gscg_memory_info* out) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        *out = gscg_memory_info{};
        for (const TemplateStore& t : ctx->templates)
            for (const LevelStore& l : t.levels) out->template_bytes += l.core.cap + l.weights.cap + l.sh.cap;
        const DevBuf* bufs[] = {&ctx->d_templates, &ctx->d_groups, &ctx->d_mats, &ctx->d_parents,
                                &ctx->template_ids, &ctx->placement, &ctx->poses, &ctx->lod_prev,
                                &ctx->lod_out, &ctx->inst_group, &ctx->inst_base, &ctx->members, &ctx->visible,
                                &ctx->group_inst_start, &ctx->group_inst_count, &ctx->group_item_start,
                                &ctx->skin, &ctx->counters, &ctx->records_s[0], &ctx->records_s[1], &ctx->splat_meta_s[0], &ctx->splat_meta_s[1],
                                &ctx->splat_depth_s[0], &ctx->splat_depth_s[1], &ctx->skeys[0], &ctx->skeys[1], &ctx->srecs[0], &ctx->srecs[1],
                                &ctx->pcell_s[0][0], &ctx->pcell_s[0][1], &ctx->precs_s[0][0], &ctx->precs_s[0][1],
                      &ctx->pcell_s[1][0], &ctx->pcell_s[1][1], &ctx->precs_s[1][0], &ctx->precs_s[1][1], &ctx->span_sorted,
                                &ctx->block_sums, &ctx->hist, &ctx->status, &ctx->ranges_s[0], &ctx->ranges_s[1], &ctx->sorted_ordinals,
                                &ctx->fb_rgb, &ctx->fb_T, &ctx->posed_dbg, &ctx->rec_dbg, &ctx->band_scratch,
                                &ctx->long_runs};
        for (const DevBuf* b : bufs) out->frame_bytes += b->cap;
        out->pinned_bytes = ctx->pinned_cap + sizeof(FrameCounters) + GSCG_MAX_BANDS * 8;
        out->naive_attribute_bytes = ctx->naive_core.cap + ctx->naive_w.cap;
        size_t fr = 0, tot = 0;
        CUDA_TRY(cudaMemGetInfo(&fr, &tot));
        out->device_free_bytes = fr;
        out->device_total_bytes = tot;
    });
}

int gscg_eval_sinf(gscg_ctx* ctx, const float* in, float* out, uint32_t n) {
    if (!ctx || (n && (!in || !out))) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        if (!n) return;
        DevBuf a, b;
        CUDA_TRY(a.ensure_exact(n * 4ull));
        CUDA_TRY(b.ensure_exact(n * 4ull));
        CUDA_TRY(cudaMemcpyAsync(a.ptr, in, n * 4ull, cudaMemcpyHostToDevice, ctx->stream));
        k_eval_sinf<<<std::min<uint32_t>((n + 255) / 256, 4096), 256, 0, ctx->stream>>>(a.as<float>(), b.as<float>(), n);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(out, b.ptr, n * 4ull, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        a.release();
        b.release();
    });
}

int gscg_eval_expf(gscg_ctx* ctx, uint32_t first_bits, uint32_t n, float* out) {
    if (!ctx || (n && !out)) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        if (!n) return;
        DevBuf b;
        CUDA_TRY(b.ensure_exact(n * 4ull));
        k_eval_expf<<<std::min<uint32_t>((n + 255) / 256, 8192), 256, 0, ctx->stream>>>(first_bits, n, b.as<float>());
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(out, b.ptr, n * 4ull, cudaMemcpyDefault, ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        b.release();
    });
}

int gscg_device_alloc(gscg_ctx* ctx, uint64_t bytes, void** out) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        CUDA_TRY(cudaMalloc(out, std::max<uint64_t>(bytes, 1)));
    });
}

int gscg_device_free(gscg_ctx* ctx, void* ptr) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        if (ptr) CUDA_TRY(cudaFree(ptr));
    });
}

int gscg_psnr(gscg_ctx* ctx, const float* a, const float* b, uint64_t floats, float* out_db) {
    if (!ctx || !out_db || (floats && (!a || !b))) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        if (floats == 0) invalid("psnr: empty images");
        // Host inputs are staged to the device; device inputs are read in place.
        DevBuf ta, tb, part;
        auto on_device = [&](const float* p, DevBuf& tmp) -> const float* {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice) return p;
            cudaGetLastError();
            CUDA_TRY(tmp.ensure_exact(floats * 4));
            CUDA_TRY(cudaMemcpyAsync(tmp.ptr, p, floats * 4, cudaMemcpyDefault, s));
            return tmp.as<float>();
        };
        const float* da = on_device(a, ta);
        const float* db = on_device(b, tb);
        CUDA_TRY(part.ensure_exact((kSseBlocks + 1) * sizeof(double)));
        k_sse_partial<<<kSseBlocks, kSseThreads, 0, s>>>(da, db, floats, part.as<double>());
        k_sse_final<<<1, kSseThreads, 0, s>>>(part.as<double>(), kSseBlocks, part.as<double>() + kSseBlocks);
        CUDA_TRY(cudaGetLastError());
        double sse = 0.0;
        CUDA_TRY(cudaMemcpyAsync(&sse, part.as<double>() + kSseBlocks, sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        // PSNR as the reference (metrics.cpp:8-23): 99 dB cap for identical images.
        constexpr float kCap = 99.0f;
        if (sse == 0.0) {
            *out_db = kCap;
        } else {
            const double mse = sse / static_cast<double>(floats);
            *out_db = std::min(static_cast<float>(10.0 * std::log10(1.0 / mse)), kCap);
        }
        ta.release();
        tb.release();
        part.release();
    });
}

int gscg_host_alloc(uint64_t bytes, void** out) {
    if (!out) return GSCG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    const cudaError_t e = cudaMallocHost(out, std::max<uint64_t>(bytes, 1));
    if (e != cudaSuccess) {
        *out = nullptr;
        return e == cudaErrorMemoryAllocation ? GSCG_ERR_OOM : GSCG_ERR_CUDA;
    }
    return GSCG_OK;
}

int gscg_host_free(void* ptr) {
    if (ptr) cudaFreeHost(ptr);
    return GSCG_OK;
}

int gscg_gather_splats(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                       const gscg_render_settings* settings, const gscg_lod_policy* lod, gscg_frame_splat* out,
                       uint64_t capacity, uint64_t* count) {
    if (!ctx || !count) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        validate_frame(ctx, frame, cam, settings, lod);
        const uint32_t n = frame->instance_count;
        const uint32_t saved = ctx->debug;
        ctx->debug |= GSCG_DEBUG_RECORDS;
        uint32_t launches = 0;
        ctx->band_state = 0;
        try {
            update_gather(ctx, frame, cam, lod, 0, n, launches);
        } catch (...) {
            ctx->debug = saved;
            throw;
        }
        ctx->debug = saved;
        if (n) CUDA_TRY(cudaMemcpyAsync(frame->active_lod, ctx->lod_out.ptr, n * 4ull, cudaMemcpyDefault, ctx->stream));
        *count = ctx->S;
        if (out) {
            if (capacity < ctx->S) invalid("splat buffer smaller than the frame's splat count");
            std::vector<gscg_splat_record> rec(ctx->S);
            if (ctx->S)
                CUDA_TRY(cudaMemcpyAsync(rec.data(), ctx->rec_dbg.ptr, ctx->S * sizeof(gscg_splat_record),
                                         cudaMemcpyDeviceToHost, ctx->stream));
            CUDA_TRY(cudaStreamSynchronize(ctx->stream));
            std::sort(rec.begin(), rec.end(), [](const gscg_splat_record& a, const gscg_splat_record& b) {
                return a.ordinal < b.ordinal;  // = (instance, gaussian) order
            });
            for (size_t i = 0; i < rec.size(); ++i) {
                const gscg_splat_record& r = rec[i];
                gscg_frame_splat& o = out[i];
                o.mean_px[0] = r.mean_px[0];
                o.mean_px[1] = r.mean_px[1];
                o.cov_xx = r.cov_xx;
                o.cov_xy = r.cov_xy;
                o.cov_yy = r.cov_yy;
                o.depth = r.depth;
                for (int c = 0; c < 3; ++c) o.color[c] = r.color[c];
                o.opacity = r.opacity;
                o.instance_id = r.instance_id;
                o.gaussian_index = r.gaussian_index;
                for (int c = 0; c < 4; ++c) o.rect[c] = r.rect[c];
            }
        } else {
            CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        }
    });
}

}  // extern "C"

namespace {
// Runs update_gather in a stage-function mode and restores the frame mode afterwards.
template <typename F>
void with_mode(gscg_ctx* ctx, gscg_ctx::Mode mode, F&& f) {
    ctx->mode = mode;
    try {
        f();
    } catch (...) {
        ctx->mode = gscg_ctx::Mode::Frame;
        throw;
    }
    ctx->mode = gscg_ctx::Mode::Frame;
}

void records_to_splats(gscg_ctx* ctx, gscg_frame_splat* out, uint64_t capacity) {
    if (capacity < ctx->S) invalid("splat buffer smaller than the frame's splat count");
    std::vector<gscg_splat_record> rec(ctx->S);
    if (ctx->S)
        CUDA_TRY(cudaMemcpyAsync(rec.data(), ctx->rec_dbg.ptr, ctx->S * sizeof(gscg_splat_record),
                                 cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    std::sort(rec.begin(), rec.end(), [](const gscg_splat_record& a, const gscg_splat_record& b) {
        return a.ordinal < b.ordinal;  // = (instance, gaussian) order, the reference's concatenation
    });
    for (size_t i = 0; i < rec.size(); ++i) {
        const gscg_splat_record& r = rec[i];
        gscg_frame_splat& o = out[i];
        o.mean_px[0] = r.mean_px[0];
        o.mean_px[1] = r.mean_px[1];
        o.cov_xx = r.cov_xx;
        o.cov_xy = r.cov_xy;
        o.cov_yy = r.cov_yy;
        o.depth = r.depth;
        for (int c = 0; c < 3; ++c) o.color[c] = r.color[c];
        o.opacity = r.opacity;
        o.instance_id = r.instance_id;
        o.gaussian_index = r.gaussian_index;
        for (int c = 0; c < 4; ++c) o.rect[c] = r.rect[c];
    }
}
}  // namespace

extern "C" {

int gscg_skin_means(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam, const gscg_lod_policy* lod,
                    float* posed_out, uint64_t capacity, uint64_t* gaussians) {
    if (!ctx || !gaussians) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        gscg_render_settings rs = ctx->settings;
        if (rs.tile_size < 1) {  // no frame rendered yet: any valid settings (they do not enter skinning)
            rs = gscg_render_settings{16, {0, 0, 0}, 0.99f, 1.0f / 255.0f, 1e-4f, 0};
        }
        validate_frame(ctx, frame, cam, &rs, lod);
        const uint32_t n = frame->instance_count;
        uint32_t launches = 0;
        ctx->band_state = 0;
        with_mode(ctx, gscg_ctx::Mode::SkinOnly, [&] { update_gather(ctx, frame, cam, lod, 0, n, launches); });
        if (n) CUDA_TRY(cudaMemcpyAsync(frame->active_lod, ctx->lod_out.ptr, n * 4ull, cudaMemcpyDefault, ctx->stream));
        *gaussians = ctx->G;
        if (posed_out) {
            if (capacity < ctx->G) invalid("posed buffer smaller than the crowd's instance-Gaussian count");
            if (ctx->G) CUDA_TRY(cudaMemcpyAsync(posed_out, ctx->posed_out.ptr, ctx->G * 12, cudaMemcpyDefault, ctx->stream));
        }
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    });
}

int gscg_gather_posed(gscg_ctx* ctx, const gscg_frame_desc* frame, const float* posed_means, uint64_t gaussians,
                      const uint32_t* project_mask, const gscg_camera* cam, const gscg_render_settings* settings,
                      gscg_frame_splat* out, uint64_t capacity, uint64_t* count) {
    if (!ctx || !count || !frame) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        if (frame->forced_lod != GSCG_LOD_GIVEN) invalid("gscg_gather_posed: forced_lod must be GSCG_LOD_GIVEN");
        gscg_frame_desc fd = *frame;  // no poses: the means are given
        fd.pose_source = GSCG_POSES_SAMPLED;
        fd.static_pose = 1;
        fd.poses = nullptr;
        gscg_lod_policy lp{};
        validate_frame(ctx, &fd, cam, settings, &lp);
        const uint32_t n = fd.instance_count;
        if (gaussians && !posed_means) invalid("null posed means");
        CUDA_TRY(ctx->posed_in.ensure(std::max<uint64_t>(gaussians, 1) * 12));
        CUDA_TRY(ctx->project_mask.ensure(std::max<size_t>(n, 1) * 4));
        if (gaussians)
            CUDA_TRY(cudaMemcpyAsync(ctx->posed_in.ptr, posed_means, gaussians * 12, cudaMemcpyDefault, ctx->stream));
        std::vector<uint32_t> all;
        if (!project_mask) {
            all.assign(std::max<uint32_t>(n, 1), 1u);
            project_mask = all.data();
        }
        if (n) CUDA_TRY(cudaMemcpyAsync(ctx->project_mask.ptr, project_mask, n * 4ull, cudaMemcpyDefault, ctx->stream));
        const uint32_t saved = ctx->debug;
        ctx->debug = (saved | GSCG_DEBUG_RECORDS) & ~GSCG_DEBUG_POSED;
        uint32_t launches = 0;
        ctx->band_state = 0;
        try {
            with_mode(ctx, gscg_ctx::Mode::PosedIn, [&] { update_gather(ctx, &fd, cam, &lp, 0, n, launches); });
        } catch (...) {
            ctx->debug = saved;
            throw;
        }
        ctx->debug = saved;
        if (ctx->G != gaussians) invalid("posed means: " + std::to_string(gaussians) + " given, the levels hold " +
                                         std::to_string(ctx->G));
        *count = ctx->S;
        if (out) records_to_splats(ctx, out, capacity);
        else CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    });
}

int gscg_sort_splats(gscg_ctx* ctx, gscg_frame_splat* splats, uint64_t n) {
    if (!ctx || (n && !splats)) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        if (n > 0xF0000000ull) invalid("too many splats");
        if (n < 2) return;
        const uint32_t n32 = static_cast<uint32_t>(n);
        cudaStream_t s = ctx->stream;
        // Key columns; stable LSD over gaussian, then instance, then depth bits, the
        // permutation as value: the reference's (depth bits, instance, gaussian) order with
        // the original position breaking exact duplicates (renderer.cpp:85-107).
        std::vector<uint32_t> col[3];
        uint32_t lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
            col[k].resize(n32);
            lo[k] = 0xffffffffu;
            hi[k] = 0u;
        }
        for (uint32_t i = 0; i < n32; ++i) {
            uint32_t d;  // the depth's bit pattern, compared as an unsigned integer (renderer.cpp:89)
            std::memcpy(&d, &splats[i].depth, 4);
            const uint32_t v[3] = {splats[i].gaussian_index, splats[i].instance_id, d};
            for (int k = 0; k < 3; ++k) {
                col[k][i] = v[k];
                lo[k] = std::min(lo[k], v[k]);
                hi[k] = std::max(hi[k], v[k]);
            }
        }
        ensure_sort_buffers(ctx, n32, 0);
        DevBuf keys, perm_in;
        CUDA_TRY(keys.ensure_exact(n * 4));
        CUDA_TRY(perm_in.ensure_exact(n * 4));
        uint32_t launches = 0;
        int cur = -1;  // buffer index holding the current permutation (srecs), -1: identity
        for (int k = 0; k < 3; ++k) {
            if (lo[k] == hi[k]) continue;  // constant column: order unchanged
            CUDA_TRY(cudaMemcpyAsync(keys.ptr, col[k].data(), n * 4, cudaMemcpyHostToDevice, s));
            const uint32_t* in_keys = keys.as<uint32_t>();
            const uint32_t* in_vals = nullptr;
            if (cur >= 0) {  // this column in the current order
                k_gather_u32<<<std::min<uint32_t>((n32 + 255) / 256, 4096), 256, 0, s>>>(
                    keys.as<uint32_t>(), ctx->srecs[cur].as<uint32_t>(), ctx->skeys[cur].as<uint32_t>(), n32);
                CUDA_TRY(cudaMemcpyAsync(perm_in.ptr, ctx->srecs[cur].ptr, n * 4, cudaMemcpyDeviceToDevice, s));
                in_keys = ctx->skeys[cur].as<uint32_t>();
                in_vals = perm_in.as<uint32_t>();
                // run_radix reads pass-0 input from in_keys while writing kb[0]: stage the
                // gathered keys outside the ping-pong pair
                CUDA_TRY(cudaMemcpyAsync(keys.ptr, ctx->skeys[cur].ptr, n * 4, cudaMemcpyDeviceToDevice, s));
                in_keys = keys.as<uint32_t>();
            }
            const RadixPlan plan = make_plan(static_cast<uint32_t>(bits_for(lo[k] ^ hi[k])));
            cur = run_radix(ctx, in_keys, in_vals, ctx->skeys, ctx->srecs, n32, plan, launches);
        }
        if (cur < 0) return;  // all keys equal: already in order
        std::vector<uint32_t> perm(n32);
        CUDA_TRY(cudaMemcpyAsync(perm.data(), ctx->srecs[cur].ptr, n * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        std::vector<gscg_frame_splat> tmp(splats, splats + n32);
        for (uint32_t i = 0; i < n32; ++i) splats[i] = tmp[perm[i]];
        keys.release();
        perm_in.release();
    });
}

int gscg_rasterize_splats(gscg_ctx* ctx, const gscg_frame_splat* splats, uint64_t n, int32_t width, int32_t height,
                          const gscg_render_settings* settings, float* fb_rgb, float* fb_T) {
    if (!ctx || !settings || (n && !splats)) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        if (settings->tile_size < 1 || settings->tile_size > 64) invalid("RenderSettings: tile_size must be in [1, 64]");
        if (!(settings->alpha_cutoff > 0.0f && settings->alpha_cutoff < 1.0f))
            invalid("RenderSettings: alpha_cutoff outside (0,1)");
        if (!(settings->transmittance_floor > 0.0f && settings->transmittance_floor < 1.0f))
            invalid("RenderSettings: transmittance_floor outside (0,1)");
        if (width < 1 || height < 1 || width > 65535 || height > 65535) invalid("rasterize: width and height must be in [1, 65535]");
        if (n > 0xF0000000ull) invalid("too many splats");
        FrameGeom& g = ctx->geom;
        g.W = width;
        g.H = height;
        g.ts = settings->tile_size;
        g.tiles_x = (g.W + g.ts - 1) / g.ts;
        g.tiles_y = (g.H + g.ts - 1) / g.ts;
        g.cells_per_tile = g.ts == 16 ? 4u : 1u;
        g.cell = g.ts == 16 ? 8 : g.ts;
        full_region(g);
        ctx->settings = *settings;
        ctx->band_state = 0;
        const uint32_t n32 = static_cast<uint32_t>(n);
        // Conic prep (renderer.cpp:133-141) on the host: the power floor takes the host libm's
        // logf, as the reference; records in the device layout (gscg_project.cu).
        std::vector<float4> rec(static_cast<size_t>(n32) * 3);
        std::vector<uint4> meta(n32);
        uint64_t pairs = 0;
        for (uint32_t i = 0; i < n32; ++i) {
            const gscg_frame_splat& sp = splats[i];
            int x0 = std::max(0, sp.rect[0]), y0 = std::max(0, sp.rect[1]);
            int x1 = std::min(width, sp.rect[2]), y1 = std::min(height, sp.rect[3]);
            const float det = sp.cov_xx * sp.cov_yy - sp.cov_xy * sp.cov_xy;
            const float inv_det = 1.0f / det;
            const float a = sp.cov_yy * inv_det, b = -sp.cov_xy * inv_det, c = sp.cov_xx * inv_det;
            const float pf = std::log(settings->alpha_cutoff / sp.opacity);
            uint32_t span_lo = 0, span_hi = 0;
            if (x0 < x1 && y0 < y1) {
                const int cx0 = x0 / g.cell, cx1 = (x1 - 1) / g.cell, cy0 = y0 / g.cell, cy1 = (y1 - 1) / g.cell;
                span_lo = static_cast<uint32_t>(cx0) | (static_cast<uint32_t>(cy0) << 16);
                span_hi = static_cast<uint32_t>(cx1 - cx0 + 1) | (static_cast<uint32_t>(cy1 - cy0 + 1) << 16);
                pairs += static_cast<uint64_t>(cx1 - cx0 + 1) * static_cast<uint64_t>(cy1 - cy0 + 1);
            } else {
                x0 = y0 = x1 = y1 = 0;  // empty rect: no cells
            }
            float4* r = rec.data() + 3ull * i;
            r[0] = make_float4(sp.mean_px[0], sp.mean_px[1], a, b);
            r[1] = make_float4(c, sp.opacity, pf, sp.color[0]);
            uint32_t xy0 = static_cast<uint32_t>(x0) | (static_cast<uint32_t>(y0) << 16);
            uint32_t xy1 = static_cast<uint32_t>(x1) | (static_cast<uint32_t>(y1) << 16);
            float fx0, fx1;
            std::memcpy(&fx0, &xy0, 4);
            std::memcpy(&fx1, &xy1, 4);
            r[2] = make_float4(sp.color[1], sp.color[2], fx0, fx1);
            meta[i] = make_uint4(i, span_lo, span_hi, 0u);
        }
        if (pairs > 0xF0000000ull) throw Status(GSCG_ERR_OOM, "tile-splat pair count exceeds 32-bit indexing");
        cudaStream_t s = ctx->stream;
        const uint64_t cap = std::max<uint64_t>(n32, 1);
        if (cap > ctx->splat_capacity) ctx->splat_capacity = cap + cap / 4;
        CUDA_TRY(ctx->rec().ensure(ctx->splat_capacity * 48));
        CUDA_TRY(ctx->meta().ensure(ctx->splat_capacity * 16));
        if (n32) {
            CUDA_TRY(cudaMemcpyAsync(ctx->rec().ptr, rec.data(), rec.size() * sizeof(float4), cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(ctx->meta().ptr, meta.data(), meta.size() * sizeof(uint4), cudaMemcpyHostToDevice, s));
        }
        ctx->S = n32;
        ctx->K = pairs;
        ctx->G = n32;
        ensure_sort_buffers(ctx, n32, static_cast<uint32_t>(pairs));
        if (n32) {  // the given order: distinct keys (no tie fix-up), identity records
            k_iota2<<<std::min<uint32_t>((n32 + 255) / 256, 4096), 256, 0, s>>>(ctx->skeys[0].as<uint32_t>(),
                                                                               ctx->srecs[0].as<uint32_t>(), n32);
            CUDA_TRY(cudaGetLastError());
        }
        uint32_t launches = 0;
        CUDA_TRY(cudaEventRecord(ctx->ev[3], s));
        sort_raster(ctx, 0, g.tiles_y, launches, nullptr, nullptr, /*presorted=*/true);
        copy_out(ctx, g.H, fb_rgb, fb_T, true);
        CUDA_TRY(cudaStreamSynchronize(s));
    });
}

int gscg_framebuffer_device(gscg_ctx* ctx, float** rgb, float** T) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    if (rgb) *rgb = ctx->fb_rgb.as<float>();
    if (T) *T = ctx->fb_T.as<float>();
    return GSCG_OK;
}

int gscg_synchronize(gscg_ctx* ctx) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        flush_readback(ctx);
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->copy_stream));
    });
}

int gscg_stream(gscg_ctx* ctx, void** stream) {
    if (!ctx || !stream) return GSCG_ERR_INVALID_ARGUMENT;
    *stream = ctx->stream;
    return GSCG_OK;
}

int gscg_get_counts(gscg_ctx* ctx, uint64_t* gaussians, uint64_t* splats, uint64_t* pairs) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    if (gaussians) *gaussians = ctx->G;
    if (splats) *splats = ctx->S;
    if (pairs) *pairs = ctx->K;
    return GSCG_OK;
}

int gscg_get_instances_culled(gscg_ctx* ctx, uint32_t* out) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    *out = ctx->culled;
    return GSCG_OK;
}

int gscg_get_lod(gscg_ctx* ctx, uint32_t* out, uint32_t n) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (n > ctx->n) invalid("more instances requested than rendered");
        CUDA_TRY(cudaMemcpyAsync(out, ctx->lod_out.ptr, n * 4ull, cudaMemcpyDeviceToHost, ctx->stream)); CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    });
}

int gscg_get_instance_base(gscg_ctx* ctx, uint32_t* out, uint32_t n) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (n > ctx->n) invalid("more instances requested than rendered");
        CUDA_TRY(cudaMemcpyAsync(out, ctx->inst_base.ptr, n * 4ull, cudaMemcpyDeviceToHost, ctx->stream)); CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    });
}

int gscg_get_posed_means(gscg_ctx* ctx, float* out, uint64_t gaussians) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (!(ctx->debug & GSCG_DEBUG_POSED)) invalid("enable GSCG_DEBUG_POSED before rendering");
        if (gaussians > ctx->G) invalid("more Gaussians requested than rendered");
        CUDA_TRY(cudaMemcpyAsync(out, ctx->posed_dbg.ptr, gaussians * 12, cudaMemcpyDeviceToHost, ctx->stream)); CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    });
}

int gscg_get_splat_records(gscg_ctx* ctx, gscg_splat_record* out, uint64_t splats) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (!(ctx->debug & GSCG_DEBUG_RECORDS)) invalid("enable GSCG_DEBUG_RECORDS before rendering");
        if (splats > ctx->S) invalid("more splats requested than rendered");
        CUDA_TRY(cudaMemcpyAsync(out, ctx->rec_dbg.ptr, splats * sizeof(gscg_splat_record), cudaMemcpyDeviceToHost, ctx->stream)); CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        std::sort(out, out + splats, [](const gscg_splat_record& a, const gscg_splat_record& b) {
            return a.ordinal < b.ordinal;
        });
    });
}

int gscg_get_cell_layout(gscg_ctx* ctx, uint32_t* tiles, uint32_t* cells_per_tile) {
    if (!ctx) return GSCG_ERR_INVALID_ARGUMENT;
    if (tiles) *tiles = ctx->tiles;
    if (cells_per_tile) *cells_per_tile = ctx->cells_per_tile;
    return GSCG_OK;
}

int gscg_get_tile_ranges(gscg_ctx* ctx, uint32_t* out, uint32_t cells) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (cells > ctx->tiles * ctx->cells_per_tile) invalid("more cells requested than rendered");
        CUDA_TRY(cudaMemcpyAsync(out, ctx->ranges().ptr, cells * 8ull, cudaMemcpyDeviceToHost, ctx->stream)); CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    });
}

int gscg_get_sorted_ordinals(gscg_ctx* ctx, uint32_t* out, uint64_t pairs) {
    if (!ctx || !out) return GSCG_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (pairs > ctx->K) invalid("more pairs requested than rendered");
        if (pairs == 0) return;
        CUDA_TRY(ctx->sorted_ordinals.ensure(pairs * 4));
        k_sorted_ordinals<<<std::min<uint64_t>((pairs + 255) / 256, 4096), 256, 0, ctx->stream>>>(
            ctx->final_recs, ctx->meta().as<uint4>(), static_cast<uint32_t>(pairs),
            ctx->sorted_ordinals.as<uint32_t>());
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(out, ctx->sorted_ordinals.ptr, pairs * 4, cudaMemcpyDeviceToHost, ctx->stream)); CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    });
}

int gscg_get_sorted_values(gscg_ctx* ctx, uint32_t* out, uint64_t pairs) {
    return gscg_get_sorted_ordinals(ctx, out, pairs);
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// Multi-GPU frame: one process per GPU, each rank owns a
// gscg_ctx and renders one horizontal screen band of the SAME frame (gscg_set_band: its
// own instance cull + projection keep the splats that meet its rows; sort + raster cover
// its tiles), then the bands are gathered into rank 0's framebuffer with grouped
// ncclSend / ncclRecv on the context stream (NVLink / NVSwitch). The only exchange is the
// gather of finished rows: a splat that meets several bands is projected by each of those
// ranks, which costs less here than routing every projected splat through an all-to-all
// (DESIGN.md §5 has the measurement). NCCL is this library's own communicator; the
// caller's process-group plumbing (torch.distributed) only ships the 128-byte unique id.
struct gscg_group {
    gscg_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    DevBuf full_rgb, full_T, stage_rgb, stage_T, row_costs, all_costs;
    // Async frames (gscg_group_render_frame_async): rank 0 alternates two whole-frame
    // buffers; rb_ev[i] marks the end of buffer i's host read-back on the copy stream.
    DevBuf full_rgb_alt, full_T_alt;
    cudaEvent_t rb_ev[2] = {nullptr, nullptr}, done_ev = nullptr;
    bool rb_rec[2] = {false, false};
    int cur = 0;
};

namespace {

// NCCL is bound at run time (dlopen of libnccl.so.2): a process that already holds one
// (torch's bundled NCCL) keeps it — linking at build time would pin the system copy first
// and break torch's own symbol versions.
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    bool ok = false;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return a;
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send && a.Recv &&
               a.AllReduce && a.GetErrorString;
        return a;
    }();
    if (!api.ok) throw Status(GSCG_ERR_NCCL, "libnccl.so.2 not found (multi-GPU groups need NCCL)");
    return api;
}

#define NCCL_TRY(expr)                                                                                \
    do {                                                                                              \
        ncclResult_t _r = (expr);                                                                     \
        if (_r != ncclSuccess) throw Status(GSCG_ERR_NCCL, std::string(#expr) + ": " + nccl().GetErrorString(_r)); \
    } while (0)

}  // namespace

extern "C" {

int gscg_group_unique_id(uint8_t* out) {
    if (!out) return GSCG_ERR_INVALID_ARGUMENT;
    ncclUniqueId id;
    try {
        if (nccl().GetUniqueId(&id) != ncclSuccess) return GSCG_ERR_NCCL;
    } catch (const Status&) {
        return GSCG_ERR_NCCL;
    }
    static_assert(sizeof(id) == GSCG_UNIQUE_ID_BYTES, "NCCL unique id size");
    std::memcpy(out, &id, sizeof(id));
    return GSCG_OK;
}

int gscg_group_create(gscg_ctx* ctx, const uint8_t* unique_id, int32_t nranks, int32_t rank, gscg_group** out) {
    if (!ctx || !unique_id || !out || nranks < 1 || rank < 0 || rank >= nranks) return GSCG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        auto g = std::make_unique<gscg_group>();
        g->ctx = ctx;
        g->nranks = nranks;
        g->rank = rank;
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        NCCL_TRY(nccl().CommInitRank(&g->comm, nranks, id, rank));
        *out = g.release();
    });
}

int gscg_create_group(gscg_ctx* ctx, const uint8_t* unique_id, int32_t nranks, int32_t rank, gscg_group** out) {
    return gscg_group_create(ctx, unique_id, nranks, rank, out);
}

int gscg_group_destroy(gscg_group* g) {
    if (!g) return GSCG_OK;
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
    cudaStreamSynchronize(g->ctx->copy_stream);
    if (g->comm) nccl().CommDestroy(g->comm);
    for (auto& e : g->rb_ev)
        if (e) cudaEventDestroy(e);
    if (g->done_ev) cudaEventDestroy(g->done_ev);
    g->full_rgb.release();
    g->full_T.release();
    g->full_rgb_alt.release();
    g->full_T_alt.release();
    g->stage_rgb.release();
    g->stage_T.release();
    g->row_costs.release();
    g->all_costs.release();
    delete g;
    return GSCG_OK;
}

namespace {
int group_render_impl(gscg_group* g, const gscg_frame_desc* frame, const gscg_camera* cam,
                      const gscg_render_settings* settings, const gscg_lod_policy* lod, int32_t axis,
                      const uint32_t* cuts, float* fb_rgb, float* fb_T, gscg_stage_times* times, bool async) {
    if (!g || !cuts || !cam || (axis != GSCG_SPLIT_ROWS && axis != GSCG_SPLIT_COLS)) return GSCG_ERR_INVALID_ARGUMENT;
    gscg_ctx* ctx = g->ctx;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        const int W = cam->width, H = cam->height, P = g->nranks;
        const bool by_cols = axis == GSCG_SPLIT_COLS;
        const uint32_t extent = static_cast<uint32_t>(by_cols ? W : H);
        if (cuts[0] != 0 || cuts[P] != extent) invalid("cuts must cover the frame along the split axis");
        for (int r = 0; r < P; ++r)
            if (cuts[r + 1] < cuts[r]) invalid("cuts must be ascending");
        const uint32_t a0 = cuts[g->rank], a1 = cuts[g->rank + 1];
        // This rank's region, rendered into the context's framebuffer (region-major, from 0).
        const int32_t s0 = ctx->band_req0, s1 = ctx->band_req1, s2 = ctx->col_req0, s3 = ctx->col_req1;
        if (by_cols) {
            ctx->band_req0 = ctx->band_req1 = 0;
            ctx->col_req0 = static_cast<int32_t>(a0);
            ctx->col_req1 = static_cast<int32_t>(a1);
        } else {
            ctx->band_req0 = static_cast<int32_t>(a0);
            ctx->band_req1 = static_cast<int32_t>(a1);
            ctx->col_req0 = ctx->col_req1 = 0;
        }
        gscg_frame_desc fd = *frame;
        int rc = GSCG_OK;
        if (a1 > a0) rc = render_frame_impl(ctx, &fd, cam, settings, lod, nullptr, nullptr, times, false);
        ctx->band_req0 = s0;
        ctx->band_req1 = s1;
        ctx->col_req0 = s2;
        ctx->col_req1 = s3;
        if (rc != GSCG_OK) throw Status(rc, ctx->error);
        cudaStream_t s = ctx->stream;
        // Region r holds (rows x width) pixels: full-width bands, or full-height columns.
        auto region_px = [&](int r) -> size_t {
            const size_t len = cuts[r + 1] - cuts[r];
            return by_cols ? len * static_cast<size_t>(H) : len * static_cast<size_t>(W);
        };
        if (g->rank == 0) {
            if (async) {  // the other whole-frame buffer, once its last read-back has landed
                std::swap(g->full_rgb, g->full_rgb_alt);
                std::swap(g->full_T, g->full_T_alt);
                g->cur ^= 1;
            }
            // A buffer may still be read back from an async frame (also when a blocking
            // call follows async ones).
            if (g->rb_rec[g->cur]) CUDA_TRY(cudaStreamWaitEvent(s, g->rb_ev[g->cur], 0));
            CUDA_TRY(g->full_rgb.ensure(static_cast<size_t>(W) * H * 12));
            CUDA_TRY(g->full_T.ensure(static_cast<size_t>(W) * H * 4));
            if (by_cols) {
                CUDA_TRY(g->stage_rgb.ensure(static_cast<size_t>(W) * H * 12));
                CUDA_TRY(g->stage_T.ensure(static_cast<size_t>(W) * H * 4));
            }
        }
        // Rank 0's own region, then every other rank's, gathered with grouped send/recv.
        // Row bands land in place; column regions land packed in a staging buffer and are
        // placed with one strided copy each.
        size_t off = 0;  // pixels before region r in the packed layout
        std::vector<size_t> offs(P + 1, 0);
        for (int r = 0; r < P; ++r) {
            offs[r] = off;
            off += region_px(r);
        }
        auto dst_rgb = [&](int r) {
            return by_cols ? g->stage_rgb.as<float>() + 3 * offs[r] : g->full_rgb.as<float>() + 3 * offs[r];
        };
        auto dst_T = [&](int r) { return by_cols ? g->stage_T.as<float>() + offs[r] : g->full_T.as<float>() + offs[r]; };
        if (g->rank == 0 && a1 > a0 && !by_cols) {  // rank 0's own column region is placed from its framebuffer below
            CUDA_TRY(cudaMemcpyAsync(dst_rgb(0), ctx->fb_rgb.ptr, region_px(0) * 12, cudaMemcpyDeviceToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(dst_T(0), ctx->fb_T.ptr, region_px(0) * 4, cudaMemcpyDeviceToDevice, s));
        }
        if (P > 1) {
            NCCL_TRY(nccl().GroupStart());
            if (g->rank == 0) {
                for (int r = 1; r < P; ++r) {
                    if (!region_px(r)) continue;
                    NCCL_TRY(nccl().Recv(dst_rgb(r), region_px(r) * 3, ncclFloat32, r, g->comm, s));
                    NCCL_TRY(nccl().Recv(dst_T(r), region_px(r), ncclFloat32, r, g->comm, s));
                }
            } else if (a1 > a0) {
                NCCL_TRY(nccl().Send(ctx->fb_rgb.ptr, region_px(g->rank) * 3, ncclFloat32, 0, g->comm, s));
                NCCL_TRY(nccl().Send(ctx->fb_T.ptr, region_px(g->rank), ncclFloat32, 0, g->comm, s));
            }
            NCCL_TRY(nccl().GroupEnd());
        }
        if (g->rank == 0 && by_cols) {
            for (int r = 0; r < P; ++r) {
                const size_t wr = cuts[r + 1] - cuts[r];
                if (!wr) continue;
                const float* src_rgb = r == 0 ? ctx->fb_rgb.as<float>() : dst_rgb(r);
                const float* src_T = r == 0 ? ctx->fb_T.as<float>() : dst_T(r);
                CUDA_TRY(cudaMemcpy2DAsync(g->full_rgb.as<float>() + 3 * cuts[r], static_cast<size_t>(W) * 12, src_rgb,
                                           wr * 12, wr * 12, H, cudaMemcpyDeviceToDevice, s));
                CUDA_TRY(cudaMemcpy2DAsync(g->full_T.as<float>() + cuts[r], static_cast<size_t>(W) * 4, src_T, wr * 4,
                                           wr * 4, H, cudaMemcpyDeviceToDevice, s));
            }
        }
        if (g->rank == 0 && (fb_rgb || fb_T)) {
            const size_t px = static_cast<size_t>(W) * H;
            if (async) {  // read-back on the copy stream, under the next frame
                if (!g->done_ev) {
                    CUDA_TRY(cudaEventCreateWithFlags(&g->done_ev, cudaEventDisableTiming));
                    for (auto& e : g->rb_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                }
                CUDA_TRY(cudaEventRecord(g->done_ev, s));
                CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, g->done_ev, 0));
                if (fb_rgb) CUDA_TRY(cudaMemcpyAsync(fb_rgb, g->full_rgb.ptr, px * 12, cudaMemcpyDefault, ctx->copy_stream));
                if (fb_T) CUDA_TRY(cudaMemcpyAsync(fb_T, g->full_T.ptr, px * 4, cudaMemcpyDefault, ctx->copy_stream));
                CUDA_TRY(cudaEventRecord(g->rb_ev[g->cur], ctx->copy_stream));
                g->rb_rec[g->cur] = true;
            } else {
                if (fb_rgb) CUDA_TRY(cudaMemcpyAsync(fb_rgb, g->full_rgb.ptr, px * 12, cudaMemcpyDefault, s));
                if (fb_T) CUDA_TRY(cudaMemcpyAsync(fb_T, g->full_T.ptr, px * 4, cudaMemcpyDefault, s));
                if (is_host_pointer(fb_rgb) || is_host_pointer(fb_T)) CUDA_TRY(cudaStreamSynchronize(s));
            }
        }
    });
}
}  // namespace

int gscg_group_render_frame(gscg_group* g, const gscg_frame_desc* frame, const gscg_camera* cam,
                            const gscg_render_settings* settings, const gscg_lod_policy* lod, int32_t axis,
                            const uint32_t* cuts, float* fb_rgb, float* fb_T, gscg_stage_times* times) {
    return group_render_impl(g, frame, cam, settings, lod, axis, cuts, fb_rgb, fb_T, times, false);
}

int gscg_group_render_frame_async(gscg_group* g, const gscg_frame_desc* frame, const gscg_camera* cam,
                                  const gscg_render_settings* settings, const gscg_lod_policy* lod, int32_t axis,
                                  const uint32_t* cuts, float* fb_rgb, float* fb_T, gscg_stage_times* times) {
    return group_render_impl(g, frame, cam, settings, lod, axis, cuts, fb_rgb, fb_T, times, true);
}

int gscg_group_wait_readback(gscg_group* g) {
    if (!g) return GSCG_ERR_INVALID_ARGUMENT;
    gscg_ctx* ctx = g->ctx;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        CUDA_TRY(cudaStreamSynchronize(ctx->copy_stream));
    });
}

int gscg_group_framebuffer_device(gscg_group* g, float** rgb, float** T) {
    if (!g || g->rank != 0) return GSCG_ERR_INVALID_ARGUMENT;
    if (rgb) *rgb = g->full_rgb.as<float>();
    if (T) *T = g->full_T.as<float>();
    return GSCG_OK;
}

int gscg_group_tile_costs(gscg_group* g, uint32_t tiles_x, uint32_t tiles_y, uint64_t* out) {
    if (!g || !out) return GSCG_ERR_INVALID_ARGUMENT;
    gscg_ctx* ctx = g->ctx;
    return guarded(ctx, [&] {
        CUDA_TRY(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        const FrameGeom& geo = ctx->geom;
        const size_t n = static_cast<size_t>(tiles_x) * tiles_y;
        CUDA_TRY(g->row_costs.ensure(n * 8));
        CUDA_TRY(g->all_costs.ensure(n * 8));
        CUDA_TRY(cudaMemsetAsync(g->row_costs.ptr, 0, n * 8, s));
        // This rank's last region: tiles [band_tile_col0, +band_tiles_x) x [band_tile_row0, +band_tile_rows).
        const uint32_t rtx = static_cast<uint32_t>(geo.band_tiles_x), rows = static_cast<uint32_t>(geo.band_tile_rows);
        if (ctx->tiles && rtx && rows && static_cast<uint32_t>(geo.band_tile_row0) + rows <= tiles_y &&
            static_cast<uint32_t>(geo.band_tile_col0) + rtx <= tiles_x) {
            k_tile_costs<<<(rtx * rows + 255) / 256, 256, 0, s>>>(ctx->ranges().as<uint2>(), rtx, rows, geo.cells_per_tile,
                                                                 geo.band_tile_col0, geo.band_tile_row0, tiles_x,
                                                                 g->row_costs.as<unsigned long long>());
            CUDA_TRY(cudaGetLastError());
        }
        // Every rank's tiles (disjoint regions) summed: all-reduce of the tile map.
        if (g->nranks > 1)
            NCCL_TRY(nccl().AllReduce(g->row_costs.ptr, g->all_costs.ptr, n, ncclUint64, ncclSum, g->comm, s));
        else
            CUDA_TRY(cudaMemcpyAsync(g->all_costs.ptr, g->row_costs.ptr, n * 8, cudaMemcpyDeviceToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(out, g->all_costs.ptr, n * 8, cudaMemcpyDefault, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
