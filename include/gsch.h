/*
 * gsch.h — C-ABI of the host scene layer (paper_2501_17792_b200/host, namespace gsc).
 *
 * It exposes the reference's host-side API to Python (ctypes) without torch types:
 * synthetic assets (generate_synthetic_template / generate_synthetic_motion,
 * /root/reference/proj/src/synthetic.cpp), build_crowd (crowd.cpp:46-84), the camera
 * (Camera::look_at, math.cpp:42-64) and render_frame (renderer.hpp:114-123) running on
 * the B200 path through gscg.h. Array views expose the host asset store so parity tests
 * can feed the identical inputs to the CPU oracle.
 */
#ifndef GSCH_H_
#define GSCH_H_

#include <stdint.h>

#include "gscg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gsch_scene gsch_scene;
typedef struct gsch_renderer gsch_renderer;

typedef struct {
  uint32_t template_count;
  uint64_t template_seed_base; /* template i uses seed base + i, template_id = i */
  uint32_t level_count;
  uint32_t level_counts[4];
  uint32_t joint_count;
  int32_t with_sh;
  uint32_t motion_count;
  uint64_t motion_seed_base;
  float motion_fps;
  uint32_t motion_frames;
  uint32_t grid_rows, grid_cols;
  float grid_spacing;
  uint32_t crowd_count;
  uint64_t crowd_seed;
  float cam_pos[3];
  float cam_look[3];
  float fov_y_deg;
  uint32_t width, height;
  float near_m;
  uint32_t lod_threshold_count;
  float lod_thresholds[8];
  float lod_hysteresis;
} gsch_scene_config;

typedef struct {
  uint32_t instance_id, template_id, motion_id;
  float x, z, yaw, phase_offset_s;
  uint32_t active_lod;
} gsch_instance;

typedef struct {
  uint32_t count;
  const float* means;         /* N x 3 */
  const float* rotations;     /* N x 4 (x, y, z, w) */
  const float* scales;        /* N x 3 */
  const float* opacities;     /* N */
  const float* colors;        /* N x 3 */
  const uint16_t* skin_indices; /* N x 4 */
  const float* skin_weights;  /* N x 4 */
  const float* sh;            /* N x 45 or NULL */
  const float* cov6;          /* N x 6 */
} gsch_level_view;

typedef struct {
  int32_t tile_size;
  float background[3];
  float alpha_max, alpha_cutoff, transmittance_floor;
  int32_t thread_count;
  int32_t sh_colour;
} gsch_render_settings;

typedef struct {
  double update_ms, gather_ms, sort_ms, rasterize_ms, pose_ms, total_ms;
  uint64_t splat_count, pair_count, gaussian_count;
  uint64_t tile_pair_count; /* the reference's per-tile bin entries (gscg_stage_times) */
} gsch_stage_times;

const char* gsch_last_error(void);

int gsch_scene_create(const gsch_scene_config* cfg, int threads, gsch_scene** out);
int gsch_scene_destroy(gsch_scene* scene);
int gsch_scene_counts(const gsch_scene* scene, uint32_t* templates, uint32_t* motions,
                      uint32_t* instances);
int gsch_scene_get_instances(const gsch_scene* scene, gsch_instance* out, uint32_t n);
int gsch_scene_set_instances(gsch_scene* scene, const gsch_instance* in, uint32_t n);
int gsch_scene_set_camera(gsch_scene* scene, const float* pos, const float* look, float fov_y_deg,
                          uint32_t width, uint32_t height, float near_m);
int gsch_scene_camera_basis(const gsch_scene* scene, gscg_camera* out);
int gsch_scene_set_lod_policy(gsch_scene* scene, const float* thresholds, uint32_t count,
                              float hysteresis);
int gsch_scene_level_count(const gsch_scene* scene, uint32_t template_id, uint32_t* out);
int gsch_scene_level_view(const gsch_scene* scene, uint32_t template_id, uint32_t level,
                          gsch_level_view* out);
int gsch_scene_skeleton(const gsch_scene* scene, uint32_t template_id, uint32_t* joint_count,
                        const int16_t** parents, const float** inverse_bind);
/* frames x (4 + 4*J): root xyz, pad, J quaternions (x, y, z, w); call with out = NULL to query */
int gsch_scene_motion(const gsch_scene* scene, uint32_t motion_id, float* fps, uint32_t* frames,
                      uint32_t* joints, float* out);

/* Host pose sampling without a GPU: same records as gsch_sample_crowd. */
int gsch_scene_sample_crowd(gsch_scene* scene, float time_s, int32_t static_pose, int32_t threads,
                            uint32_t joint_stride, uint32_t* template_ids, float* placement, float* poses);

/* Replace (motion_id < count) or append (motion_id == count) a clip; same layout as above. */
int gsch_scene_set_motion(gsch_scene* scene, uint32_t motion_id, float fps, uint32_t frames,
                          uint32_t joints, const float* data);

/* Asset files (reference io.hpp:38-43, io_assets.cpp): GSAT templates (v1 = the
 * reference's layout; v2 adds SH residual blocks) and GSMO motion clips. load_* replace
 * id < count or append id == count; renderers re-upload the changed store on their next
 * frame. Format failures return GSCH_ERR_FORMAT with "[Kind] message" in gsch_last_error
 * (Kind: IoError, BadMagic, VersionMismatch, Truncated, InvariantViolation). */
#define GSCH_ERR_FORMAT (-6)
/* update_crowd's LoD step (crowd.cpp:86-110) on the host: sets every instance's active
 * level for the scene camera (forced_lod < 0: distance LoD with hysteresis). */
int gsch_scene_update_crowd(gsch_scene* scene, int32_t forced_lod);
int gsch_scene_save_template(const gsch_scene* scene, uint32_t template_id, const char* path);
int gsch_scene_load_template(gsch_scene* scene, uint32_t template_id, const char* path);
int gsch_scene_save_motion(const gsch_scene* scene, uint32_t motion_id, const char* path);
int gsch_scene_load_motion(gsch_scene* scene, uint32_t motion_id, const char* path);

/* Metrics (reference metrics.hpp:13-31). gsch_psnr is the reference's CPU psnr over two
 * width x height x 3 images. gsch_lod_quality_sweep renders one bind-posed character of
 * the template per (distance, level) on GPU `device` with the scene camera's fov, size and
 * near plane, and scores each level against level 0 with the on-device PSNR (gscg_psnr);
 * rows = count x levels (query with rows = NULL). */
typedef struct {
  float distance_m;
  uint32_t level;
  uint32_t gaussian_count;
  float psnr_db;
} gsch_quality_row;
int gsch_psnr(const float* a, const float* b, uint32_t width, uint32_t height, float* out_db);
int gsch_lod_quality_sweep(gsch_scene* scene, uint32_t template_id, const float* distances, uint32_t count,
                           const gsch_render_settings* settings, int device, gsch_quality_row* rows,
                           uint32_t capacity, uint32_t* row_count);

/* Shared-attribute memory accounting (crowd.cpp:142-210, MemoryLayoutModel defaults). */
typedef struct {
  uint64_t naive_bytes, shared_bytes;
  double savings_fraction;
  double naive_marginal_bytes_per_instance, shared_marginal_bytes_per_instance;
  uint64_t resident_template_bytes, posed_mean_bytes, instance_count;
} gsch_memory_report;
int gsch_memory_report_cell(uint64_t instances, uint64_t gaussians, uint64_t fixed_overhead,
                            gsch_memory_report* out);
int gsch_scene_memory_report(const gsch_scene* scene, gsch_memory_report* out);

int gsch_renderer_create(gsch_scene* scene, int device, gsch_renderer** out);
int gsch_renderer_destroy(gsch_renderer* r);
gscg_ctx* gsch_renderer_gpu(gsch_renderer* r);
uint32_t gsch_renderer_joint_stride(gsch_renderer* r);
/* Pose sampling on the GPU (GSCG_POSES_SAMPLED, bit-identical to host sampling): per frame
 * only placements, motion ids and phase offsets are uploaded. Default off (host sampling). */
int gsch_renderer_set_device_poses(gsch_renderer* r, int32_t enabled);
/* Uploads the scene's templates and motion clips to the renderer's context now (they are
 * otherwise uploaded by the first render). */
int gsch_renderer_prepare(gsch_renderer* r);
/* Per-instance frame records for device pose sampling (any pointer may be NULL):
 * template ids, placement (x, z, cos yaw, sin yaw; host libm), motion ids, phase offsets
 * and active LoDs, n each (n x 4 for placement). */
int gsch_fill_instances(gsch_renderer* r, int32_t static_pose, uint32_t* template_ids, float* placement,
                        uint32_t* motion_ids, float* phase_offsets, uint32_t* lods);
/* Stage functions over host splat arrays (reference renderer.hpp:81-103): gather (update +
 * projection at time_s; survivors in (instance, gaussian) order; out = NULL queries the
 * count), sort by (depth bits, instance, gaussian), rasterize in the given order. */
int gsch_gather_splats(gsch_renderer* r, float time_s, int32_t static_pose, int32_t forced_lod,
                       const gsch_render_settings* settings, gscg_frame_splat* out, uint64_t capacity,
                       uint64_t* count);
int gsch_sort_splats(gsch_renderer* r, gscg_frame_splat* splats, uint64_t n);
int gsch_rasterize_splats(gsch_renderer* r, const gscg_frame_splat* splats, uint64_t n, int32_t width,
                          int32_t height, const gsch_render_settings* settings, float* out_rgb, float* out_T);
/* render_frame(crowd, camera, time_s, settings, static_pose, forced_lod, times, ctx) */
int gsch_render(gsch_renderer* r, float time_s, int32_t static_pose, int32_t forced_lod,
                const gsch_render_settings* settings, float* out_rgb, float* out_T,
                gsch_stage_times* times);
/* Streaming render (render_frame_async / gscg_render_frame_async): out_rgb / out_T are
 * filled in the background while the next frame renders; valid after
 * gsch_wait_readback(r, frames_back) (0 = the last submitted frame). */
int gsch_render_async(gsch_renderer* r, float time_s, int32_t static_pose, int32_t forced_lod,
                      const gsch_render_settings* settings, float* out_rgb, float* out_T,
                      gsch_stage_times* times);
int gsch_wait_readback(gsch_renderer* r, uint32_t frames_back);
/* Host pose sampling only (the "update" host part) into caller buffers:
 * template_ids n, placement n x 4, poses n x (4 + 4*joint_stride). */
int gsch_sample_crowd(gsch_renderer* r, float time_s, int32_t static_pose, int32_t threads,
                      uint32_t* template_ids, float* placement, float* poses);

#ifdef __cplusplus
}
#endif

#endif /* GSCH_H_ */
