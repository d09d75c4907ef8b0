/*
 * orc.h — CPU ORACLE (test infrastructure only; never on the product path).
 *
 * An Eigen-free C++ restatement of the reference's per-frame render path
 * (/root/reference/proj: src/lod.cpp:22-41, src/avatar.cpp:10-23,40-72,99-105,149-192,
 * 226-283, src/crowd.cpp:20-30,86-140, src/math.cpp:42-170, src/renderer.cpp:25-280,
 * include/gsc/parallel.hpp:14-49), plus the SH-deg-3 residual colour extension
 * (SURVEY.md Appendix B). Only tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline leg may load it.
 *
 * Parity pinning: the reference cannot be compiled here (Eigen 3.4, libpng and the
 * vendored doctest/json/CLI11 are absent), and it ships no golden vectors. The oracle is
 * pinned by the reference's own known-answer and property tests restated in
 * tests/test_oracle.py; Eigen's floating-point evaluation order is restated from its
 * templates and is "parity unpinned" against a real Eigen build.
 */
#ifndef ORC_H_
#define ORC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_scene orc_scene;

typedef struct {
  uint32_t instance_id, template_id, motion_id;
  float x, z, yaw, phase_offset_s;
  uint32_t active_lod;
} orc_instance;

typedef struct {
  float mean_px[2];
  float cov_xx, cov_xy, cov_yy;
  float depth;
  float color[3];
  float opacity;
  uint32_t instance_id, gaussian_index;
  int32_t rect[4]; /* x0, y0, x1, y1 */
} orc_splat;

typedef struct {
  int32_t tile_size;
  float background[3];
  float alpha_max, alpha_cutoff, transmittance_floor;
  int32_t sh_colour;
} orc_settings;

typedef struct {
  double update_ms, gather_ms, sort_ms, rasterize_ms;
  uint64_t splat_count, pair_count, gaussian_count;
} orc_times;

orc_scene* orc_scene_new(void);
void orc_scene_free(orc_scene* s);
const char* orc_last_error(void);

int orc_add_template(orc_scene* s, uint32_t joint_count, const int16_t* parents,
                     const float* inverse_bind);
int orc_add_level(orc_scene* s, uint32_t template_id, uint32_t count, const float* means,
                  const float* rotations_xyzw, const float* scales, const float* opacities,
                  const float* colors, const uint16_t* skin_indices, const float* skin_weights,
                  const float* sh);
int orc_add_motion(orc_scene* s, float fps, uint32_t frames, uint32_t joints, const float* data);
int orc_set_instances(orc_scene* s, uint32_t n, const orc_instance* inst);
int orc_get_instances(orc_scene* s, uint32_t n, orc_instance* out);
int orc_set_camera(orc_scene* s, const float* eye, const float* target, float fov_y_deg,
                   int32_t width, int32_t height, float near_m);
int orc_set_lod(orc_scene* s, const float* thresholds, uint32_t count, float hysteresis);

int orc_render(orc_scene* s, float time_s, int32_t static_pose, int32_t forced_lod,
               const orc_settings* settings, int32_t threads, float* out_rgb, float* out_T,
               orc_times* times);

/* parity dumps of the last orc_render */
int orc_get_lods(orc_scene* s, uint32_t* out);
uint64_t orc_gaussian_count(orc_scene* s);
int orc_get_posed(orc_scene* s, float* out); /* G x 3, instance order then gaussian index */
uint64_t orc_splat_count(orc_scene* s);
int orc_get_splats(orc_scene* s, orc_splat* out); /* sorted frame order */
uint64_t orc_pair_count(orc_scene* s);
int orc_get_bins(orc_scene* s, uint32_t* tile_counts, uint32_t* items);
int orc_get_level_cov(orc_scene* s, uint32_t template_id, uint32_t level, float* out);

/* math / stage entry points for the reference's unit tests */
int orc_build_covariance(const float* q_xyzw, const float* scale, float* out9);
int orc_camera(const float* eye, const float* target, float fov_y_deg, int32_t width,
               int32_t height, float near_m, float* w9_rowmajor, float* focal, float* quat_xyzw);
int orc_project(const float* mean, const float* cov9, const float* color, float opacity,
                const float* eye, const float* target, float fov_y_deg, int32_t width,
                int32_t height, float near_m, orc_splat* out);
uint32_t orc_select_lod(const float* thresholds, uint32_t count, float hysteresis, float distance,
                        int64_t previous);
int orc_sort_splats(orc_splat* splats, uint32_t n);
int orc_rasterize(const orc_splat* splats, uint32_t n, int32_t width, int32_t height,
                  const orc_settings* settings, int32_t threads, float* rgb, float* T);
int orc_naive_rasterize(const orc_splat* splats, uint32_t n, int32_t width, int32_t height,
                        const orc_settings* settings, float* rgb, float* T);
int orc_sample_pose(const float* clip, uint32_t frames, uint32_t joints, float fps, float time_s,
                    int32_t wrap, float* out);
int orc_forward_kinematics(orc_scene* s, uint32_t template_id, const float* pose,
                           const float* root16, float* world_out);
int orc_skin_means(orc_scene* s, uint32_t template_id, uint32_t level, const float* world,
                   float* posed_out);
/* The host libm's sinf (what slerp_shortest calls, avatar.cpp:240-241) over an array: the
 * checker for the device pose sampler's replica. */
void orc_libm_sinf(const float* in, float* out, uint64_t n);
void orc_libm_expf_range(uint32_t first_bits, uint64_t n, float* out);

#ifdef __cplusplus
}
#endif

#endif /* ORC_H_ */
