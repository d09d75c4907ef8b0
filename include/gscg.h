/*
 * gscg.h — C-ABI of the B200 crowd-render hot path (CrowdSplat, arXiv 2501.17792).
 *
 * This is the drop-in boundary the C++ host API (paper_2501_17792_b200/host, namespace
 * gsc) calls. The reference renderer has no FFI of its own; the entry points below
 * replace, one for one, the reference's public renderer / crowd calls
 * (paths relative to /root/reference/proj):
 *
 *   gscg_create / gscg_destroy        FrameContext lifetime          include/gsc/renderer.hpp:57-79
 *   gscg_upload_skeleton              Skeleton (bind/local/inverse)  include/gsc/avatar.hpp:16-31, src/avatar.cpp:40-72
 *   gscg_upload_level                 LodLevel (+ finalize cov_cache) include/gsc/avatar.hpp:50-65, src/avatar.cpp:99-105
 *   gscg_render_frame                 render_frame(Crowd&, Camera, time, settings,
 *                                       static_pose, forced_lod, StageTimes*, FrameContext&)
 *                                                                    include/gsc/renderer.hpp:121-123, src/renderer.cpp:249-280
 *       - stage "update"   = update_crowd: LoD + FK + skin matrices  src/crowd.cpp:86-140
 *       - stage "gather"   = gather_splats: LBS + EWA projection     src/renderer.cpp:25-73
 *       - stage "sort"     = sort_splats + binning                   src/renderer.cpp:85-161
 *       - stage "rasterize"= per-tile front-to-back blend            src/renderer.cpp:163-232
 *   gscg_get_*                        parity / debug exports (no reference equivalent;
 *                                     they expose FrameContext internals: frame.splats, bins)
 *
 * Conventions: one CUDA stream per context; a context is not thread-safe; every
 * function returns GSCG_OK (0) or a negative status and records a message readable
 * through gscg_last_error. Host buffers are caller-owned; device buffers are owned by
 * the context and grow to a high-water mark. Matrices are column-major float[16]
 * (Eigen's Mat4 storage order). There is no CPU fallback: without a CUDA device
 * gscg_create fails with GSCG_ERR_CUDA.
 */
#ifndef GSCG_H_
#define GSCG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSCG_OK 0
#define GSCG_ERR_INVALID_ARGUMENT (-1) /* std::invalid_argument in the reference */
#define GSCG_ERR_CUDA (-2)
#define GSCG_ERR_NCCL (-3)
#define GSCG_ERR_OOM (-4) /* std::bad_alloc in the reference (bench.cpp:94-97) */
#define GSCG_ERR_STATE (-5)

#define GSCG_MAX_JOINTS 64
#define GSCG_MAX_LOD_THRESHOLDS 8
#define GSCG_SH_FLOATS 45 /* SH degree 1..3 residual: 15 coefficients x RGB */
#define GSCG_MAX_BANDS 64
#define GSCG_BAND_SPLAT_BYTES 64 /* one routed splat: 48 B record + ordinal + depth bits + pad */

typedef struct gscg_ctx gscg_ctx;

/* Skeleton of one template (avatar.hpp:16-31). Derived transforms are passed in,
 * computed by the host exactly as Skeleton::make does (avatar.cpp:40-72). */
typedef struct {
  uint32_t joint_count;      /* <= GSCG_MAX_JOINTS */
  const int16_t* parents;    /* joint_count; parents[0] == -1 */
  const float* local_bind;   /* joint_count x 16, column-major */
  const float* inverse_bind; /* joint_count x 16, column-major */
  float pelvis_y;            /* bind[0](1,3): the LoD root height (crowd.cpp:98-100) */
} gscg_skeleton_desc;

/* One LoD level of one template (avatar.hpp:50-65), structure-of-arrays. */
typedef struct {
  uint32_t gaussian_count;
  const float* means;           /* N x 3 */
  const float* cov6;            /* N x 6: cov_cache xx,xy,xz,yy,yz,zz (avatar.cpp:99-105) */
  const float* opacities;       /* N */
  const float* colors;          /* N x 3 linear RGB */
  const uint16_t* skin_indices; /* N x 4 */
  const float* skin_weights;    /* N x 4 */
  const float* sh;              /* N x 45 SH residual coefficients, or NULL (RGB only) */
} gscg_level_desc;

/* Flattened camera (CameraBasis, math.hpp:85-96 / math.cpp:118-129). */
typedef struct {
  float world_to_view[9]; /* row-major W(i,j) */
  float position[3];
  float focal, cx, cy, near_m;
  int32_t width, height;
} gscg_camera;

/* RenderSettings (renderer.hpp:15-22). */
typedef struct {
  int32_t tile_size;
  float background[3];
  float alpha_max;
  float alpha_cutoff;
  float transmittance_floor;
  int32_t sh_enabled; /* 1: evaluate the SH-deg-3 residual colour extension */
} gscg_render_settings;

/* LodPolicy (lod.hpp:16-21). */
typedef struct {
  uint32_t threshold_count; /* <= GSCG_MAX_LOD_THRESHOLDS */
  float thresholds_m[GSCG_MAX_LOD_THRESHOLDS];
  float hysteresis_band_m;
} gscg_lod_policy;

#define GSCG_MEM_HOST 0
#define GSCG_MEM_DEVICE 1

/* Per-frame crowd state: what update_crowd reads from Crowd (crowd.hpp:18-45) after
 * the host has sampled each instance's pose (avatar.cpp:247-283). */
typedef struct {
  uint32_t instance_count;
  uint32_t joint_stride;        /* joints per pose record (max joint count over templates) */
  const uint32_t* template_ids; /* n */
  const float* placement;       /* n x 4: x, z, cos(yaw), sin(yaw) (crowd.cpp:20-30) */
  const float* poses;           /* n x (4 + 4*joint_stride): root_translation xyz, pad,
                                   then per joint quaternion (x, y, z, w) */
  uint32_t* active_lod;         /* n, in/out: previous level (0xffffffff = unset) -> new level */
  int32_t forced_lod;           /* -1: distance LoD; else pinned level (crowd.cpp:94-96) */
  int32_t memory;               /* GSCG_MEM_HOST or GSCG_MEM_DEVICE for the pointers above */
  /* Pose source. GSCG_POSES_GIVEN: `poses` holds the sampled poses. GSCG_POSES_SAMPLED:
   * the device samples each instance's clip (gscg_upload_motion) at time_s + its phase
   * offset (sample_pose with wrap, avatar.cpp:247-283; crowd.cpp:118-128), bit-identical
   * to the host: the per-keyframe-pair acos/sin come from the host libm at upload and the
   * per-instance sinf is an exact replica of glibc's; `poses` may be NULL. */
  int32_t pose_source;
  float time_s;
  int32_t static_pose;          /* sampled mode: 1 = every instance in bind pose */
  const uint32_t* motion_ids;   /* n (sampled mode) */
  const float* phase_offsets;   /* n (sampled mode) */
} gscg_frame_desc;

#define GSCG_POSES_GIVEN 0
#define GSCG_POSES_SAMPLED 1

/* forced_lod value: every instance keeps the level in active_lod (unset = level 0), as
 * the reference's gather_splats reads inst.active_lod (renderer.cpp:38-40). */
#define GSCG_LOD_GIVEN (-2)

/* A motion clip for device pose sampling: frame_count x (4 + 4*joint_count) floats, the
 * frame pose record layout above (MotionClip, avatar.hpp:40-48). */
typedef struct {
  float fps;
  uint32_t frame_count;
  uint32_t joint_count;
  const float* frames;
} gscg_motion_desc;

/* StageTimes (renderer.hpp:105-112), measured with CUDA events on the context stream. */
typedef struct {
  double update_ms;
  double gather_ms;
  double sort_ms;
  double rasterize_ms;
  double h2d_ms;
  double d2h_ms;
  uint64_t splat_count;    /* surviving splats S */
  uint64_t pair_count;     /* tile-splat pairs K */
  uint64_t gaussian_count; /* instance-Gaussians G */
  uint32_t sort_passes;
  uint32_t kernel_launches;
  uint64_t tile_pair_count; /* the reference's per-tile bin entries (renderer.cpp:147-161): K
                               counts tile_size x tile_size tiles; pair_count counts the GPU's
                               binning cells (8x8 quadrants for tile size 16) */
} gscg_stage_times;

/* One surviving splat as gather_splats produces it (FrameSplat, renderer.hpp:39-44),
 * plus the prepared conic (renderer.hpp:72-75). Exported only in debug mode. */
typedef struct {
  uint32_t ordinal; /* instance base + gaussian_index */
  uint32_t instance_id;
  uint32_t gaussian_index;
  float depth;
  float mean_px[2];
  float cov_xx, cov_xy, cov_yy;
  float conic[3];
  float power_floor;
  float opacity;
  float color[3];
  int32_t rect[4]; /* x0, y0, x1, y1 */
} gscg_splat_record;

#define GSCG_DEBUG_POSED 1u   /* keep posed means (G x 3) */
#define GSCG_DEBUG_RECORDS 2u /* keep gscg_splat_record per survivor */
#define GSCG_DEBUG_NO_CULL 4u /* project every instance (no instance frustum cull; A/B runs) */

int gscg_create(int device, gscg_ctx** out);
int gscg_destroy(gscg_ctx* ctx);
const char* gscg_last_error(const gscg_ctx* ctx);
int gscg_device_count(int* out);

int gscg_upload_skeleton(gscg_ctx* ctx, uint32_t template_id, const gscg_skeleton_desc* desc);
int gscg_upload_level(gscg_ctx* ctx, uint32_t template_id, uint32_t level,
                      const gscg_level_desc* desc);
/* SURVEY.md §8(b)'s proposed name for gscg_upload_level (same arguments and behaviour). */
int gscg_upload_template(gscg_ctx* ctx, uint32_t template_id, uint32_t level, const gscg_level_desc* desc);
/* Device bytes held by uploaded templates (shared attribute store). */
int gscg_template_bytes(const gscg_ctx* ctx, uint64_t* out);
/* Replaces (id < count) or appends (id == count) a motion clip. */
int gscg_upload_motion(gscg_ctx* ctx, uint32_t motion_id, const gscg_motion_desc* desc);

/* Device memory of the context (config-5 ablation: shared-attribute store vs the
 * reference's analytic MemoryLayoutModel, crowd.cpp:142-210). */
typedef struct {
  uint64_t template_bytes; /* shared template store: core + skin weights + SH, all levels */
  uint64_t frame_bytes;    /* per-frame device buffers at their high-water mark */
  uint64_t pinned_bytes;   /* page-locked staging */
  uint64_t device_free_bytes, device_total_bytes; /* cudaMemGetInfo */
  uint64_t naive_attribute_bytes; /* per-instance attribute copies (GSCG_LAYOUT_NAIVE) */
} gscg_memory_info;
int gscg_memory_usage(gscg_ctx* ctx, gscg_memory_info* out);

/* Attribute layout of the projection (the config-5 / PAPER.md Table 1-2 ablation):
 * GSCG_LAYOUT_SHARED (default) reads every instance's Gaussians from the one shared
 * (template, level) store; GSCG_LAYOUT_NAIVE gives every instance its own copy of its
 * level's 80 B attributes (the reference MemoryLayoutModel's naive mode, crowd.cpp:142-210),
 * held in HBM and read per instance; RGB colour only. Same pixels either way. */
#define GSCG_LAYOUT_SHARED 0
#define GSCG_LAYOUT_NAIVE 1
int gscg_set_layout(gscg_ctx* ctx, int32_t layout);

int gscg_set_debug(gscg_ctx* ctx, uint32_t flags);

/* Band frames (the multi-GPU frame): gscg_render_frame / _async render
 * only screen rows [row_begin, row_end) (tile-aligned; row_end may be the frame height):
 * the instance cull and the projection keep the splats whose pixel rect meets those rows,
 * the sort and the raster cover the band's tiles, and fb_rgb / fb_T receive the band's
 * rows only ((row_end - row_begin) x width). Every band pixel is bit-identical to the same
 * pixel of the whole frame: a tile's list is the reference's bin (renderer.cpp:147-161),
 * ordinals and LoD are computed over the whole crowd. row_end <= row_begin (0, 0): the
 * whole frame. Persistent per context. */
int gscg_set_band(gscg_ctx* ctx, int32_t row_begin, int32_t row_end);
/* The general form: the region [x0, x1) x [y0, y1) (tile-aligned, or ending at the
 * frame's width / height); fb_rgb / fb_T receive (y1 - y0) rows of (x1 - x0) pixels. An
 * empty column range (x1 <= x0) means every column, an empty row range every row. */
int gscg_set_region(gscg_ctx* ctx, int32_t x0, int32_t y0, int32_t x1, int32_t y1);

/* Renders one frame. fb_rgb (W*H*3) and fb_T (W*H) receive the framebuffer and the
 * final transmittance; with memory == GSCG_MEM_HOST they are host pointers (copied back
 * before return), with GSCG_MEM_DEVICE they may be NULL (result stays in the context,
 * see gscg_framebuffer_device) and the call does not synchronise the host. */
int gscg_render_frame(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                      const gscg_render_settings* settings, const gscg_lod_policy* lod,
                      float* fb_rgb, float* fb_T, gscg_stage_times* times);

/* Pipelined gscg_render_frame for streaming callers (same arguments and errors; the
 * reference's render_frame, renderer.cpp:249-280, called once per frame). With host
 * destinations it returns once the frame is rendered and the LoD state written back;
 * the framebuffer read-back into fb_rgb / fb_T keeps running on a copy stream,
 * overlapped with the next frame, which renders into a second device framebuffer.
 * fb_rgb / fb_T of a frame are valid after gscg_wait_readback, and must stay allocated
 * until then (the copy lands after this call returns); a caller alternating two
 * host buffers submits frame k, then waits for frame k-1 (frames_back = 1). */
int gscg_render_frame_async(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                            const gscg_render_settings* settings, const gscg_lod_policy* lod,
                            float* fb_rgb, float* fb_T, gscg_stage_times* times);
/* Blocks until the host read-back of the frame submitted `frames_back` submissions ago
 * (0 = the last one) has landed. Frames further back than 1 are always complete. */
int gscg_wait_readback(gscg_ctx* ctx, uint32_t frames_back);

/* Page-locked host memory (cudaMallocHost) for frame inputs/outputs: device <-> host copies
 * to and from it run at full DMA speed (gscg_render_frame's host-mode framebuffer read-back
 * goes straight into it). */
int gscg_host_alloc(uint64_t bytes, void** out);
int gscg_host_free(void* ptr);

/* Device memory on the context's GPU (e.g. framebuffers gscg_render_frame writes into:
 * its fb_rgb / fb_T may be host or device pointers in either memory mode). */
int gscg_device_alloc(gscg_ctx* ctx, uint64_t bytes, void** out);
int gscg_device_free(gscg_ctx* ctx, void* ptr);

/* PSNR of two images of `floats` floats (host or device pointers) as the reference's
 * psnr (metrics.cpp:8-23): 10 log10(1 / MSE) over all channels, squared error summed in
 * double on the device (deterministic order), 99 dB for identical images. */
int gscg_psnr(gscg_ctx* ctx, const float* a, const float* b, uint64_t floats, float* out_db);

/* Device pointers of the context's framebuffer (valid until the next render). */
int gscg_framebuffer_device(gscg_ctx* ctx, float** rgb, float** T);
int gscg_synchronize(gscg_ctx* ctx);
/* The context's render stream (cudaStream_t), for event timing by the caller. A frame's
 * work spans three context streams (front half: update + projection; sort; raster +
 * read-back; each waiting for the previous part of the same frame, so the next frame's
 * front half and sort overlap this frame's raster); a frame's output is ready on the
 * render stream, and work the caller orders on it runs after the frame. */
int gscg_stream(gscg_ctx* ctx, void** stream);

/* Parity / debug exports of the last frame. */
int gscg_get_counts(gscg_ctx* ctx, uint64_t* gaussians, uint64_t* splats, uint64_t* pairs);
/* Instances of the last frame the conservative instance frustum cull left out of the
 * projection (none of their splats can survive gather_splats' cull, renderer.cpp:38-50). */
int gscg_get_instances_culled(gscg_ctx* ctx, uint32_t* out);
int gscg_get_lod(gscg_ctx* ctx, uint32_t* out, uint32_t n);
int gscg_get_instance_base(gscg_ctx* ctx, uint32_t* out, uint32_t n);
int gscg_get_posed_means(gscg_ctx* ctx, float* out, uint64_t gaussians);
int gscg_get_splat_records(gscg_ctx* ctx, gscg_splat_record* out, uint64_t splats);
/* Binning layout of the last frame: pairs are binned per cell; a cell is the whole tile,
 * or for tile size 16 one 8x8 quadrant (cell = tile * 4 + (y & 1) * 2 + (x & 1) over
 * quadrant coordinates), so every tile owns cells_per_tile consecutive cells and one
 * contiguous range of the sorted pairs. The reference's per-tile list (bins,
 * renderer.cpp:147-161) is the order-preserving merge of its cells' lists. */
int gscg_get_cell_layout(gscg_ctx* ctx, uint32_t* tiles, uint32_t* cells_per_tile);
int gscg_get_tile_ranges(gscg_ctx* ctx, uint32_t* out, uint32_t cells); /* cells x 2: [start, end) */
int gscg_get_sorted_ordinals(gscg_ctx* ctx, uint32_t* out, uint64_t pairs);
/* SURVEY.md §8(b)'s proposed name: the sorted pair values, reported as splat ordinals
 * (instance base + gaussian index, a frame-independent identity). Same as above. */
int gscg_get_sorted_values(gscg_ctx* ctx, uint32_t* out, uint64_t pairs);
/* ---- Stage functions (reference renderer.hpp:85-103) over host splat arrays ----
 * FrameSplat (renderer.hpp:39-44): the projected Splat2D, its instance and gaussian
 * index, and its pixel rect; 64 bytes. */
typedef struct {
  float mean_px[2];
  float cov_xx, cov_xy, cov_yy;
  float depth;
  float color[3];
  float opacity;
  uint32_t instance_id;
  uint32_t gaussian_index;
  int32_t rect[4]; /* x0, y0, x1, y1 */
} gscg_frame_splat;

/* gather_splats (renderer.cpp:25-73): update + projection of the frame, the surviving
 * splats in (instance, gaussian) order, as the reference concatenates them. out may be
 * NULL to query the count; otherwise capacity >= count. */
int gscg_gather_splats(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                       const gscg_render_settings* settings, const gscg_lod_policy* lod,
                       gscg_frame_splat* out, uint64_t capacity, uint64_t* count);
/* update_crowd (crowd.cpp:86-140) up to the posed means: pose sampling (or the given
 * poses), FK, skin matrices and LBS of every instance's level (forced_lod, or distance
 * LoD, or GSCG_LOD_GIVEN) on the device; posed_out (host or device) receives the
 * instance-Gaussians' posed means, G x 3 floats in instance order then gaussian index
 * (the concatenation of every CrowdInstance::posed_means). out may be NULL to query G;
 * otherwise capacity >= G. active_lod receives the levels used. */
int gscg_skin_means(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                    const gscg_lod_policy* lod, float* posed_out, uint64_t capacity, uint64_t* gaussians);
/* gather_splats (renderer.cpp:25-73) from posed means the caller holds (CrowdInstance::
 * posed_means after update_crowd): frame->forced_lod must be GSCG_LOD_GIVEN (each
 * instance projects its active_lod level); posed_means is G x 3 floats in the
 * gscg_skin_means layout; project_mask (n, may be NULL = all) skips instances whose
 * posed means are empty. Survivors come back in (instance, gaussian) order as
 * gscg_gather_splats returns them. */
int gscg_gather_posed(gscg_ctx* ctx, const gscg_frame_desc* frame, const float* posed_means, uint64_t gaussians,
                      const uint32_t* project_mask, const gscg_camera* cam, const gscg_render_settings* settings,
                      gscg_frame_splat* out, uint64_t capacity, uint64_t* count);
/* sort_splats (renderer.cpp:85-107): in place, by (depth bits, instance_id, gaussian_index),
 * on the GPU (stable LSD passes: gaussian, then instance, then depth). */
int gscg_sort_splats(gscg_ctx* ctx, gscg_frame_splat* splats, uint64_t n);
/* rasterize / rasterize_full (renderer.cpp:133-231): conic prep, tile binning in the given
 * splat order, per-tile blending; fb_rgb (width*height*3) and fb_T (width*height) may be
 * NULL. Power floors use the host libm as the reference. */
int gscg_rasterize_splats(gscg_ctx* ctx, const gscg_frame_splat* splats, uint64_t n, int32_t width,
                          int32_t height, const gscg_render_settings* settings, float* fb_rgb, float* fb_T);

/* The device pose sampler's sinf (glibc replica) over host arguments. */
int gscg_eval_sinf(gscg_ctx* ctx, const float* in, float* out, uint32_t n);
/* The rasteriser's expf (bit-exact replica of the host libm's, gscg_expf.cuh) over the n
 * consecutive float bit patterns starting at first_bits. */
int gscg_eval_expf(gscg_ctx* ctx, uint32_t first_bits, uint32_t n, float* out);

/* ---- Multi-GPU frame: instance shards -> screen bands ----
 * The reference renders one frame in one process (renderer.cpp:249-280); these three
 * calls split it at its only coupling, the splat -> tile routing (renderer.cpp:143-161),
 * so P ranks can each project an instance shard and rasterise a screen band:
 *   1. gscg_project_shard: update + gather for instances [shard_begin, shard_end) (LoD and
 *      global ordinals are computed over the whole crowd, so every rank numbers splats
 *      identically), then counts the surviving splats per screen band. band_rows holds
 *      bands + 1 screen rows (band b = [band_rows[b], band_rows[b+1]), starting on tile
 *      rows, covering [0, height)); band_counts receives the per-band splat counts (the
 *      all-to-all send counts). Synchronises the host.
 *   2. gscg_pack_bands: writes the routed splats, GSCG_BAND_SPLAT_BYTES each, grouped by
 *      band at the exclusive prefix of band_counts, into a caller device buffer.
 *      Asynchronous on gscg_stream.
 *   3. after the caller's exchange (e.g. NCCL all-to-all ordered on gscg_stream),
 *      gscg_render_band sorts the received splats by the reference's total order
 *      (depth, instance, gaussian) and rasterises rows [row_begin, row_end) into fb_rgb
 *      (rows x width x 3) / fb_T. The result is identical to the same rows of
 *      gscg_render_frame. Chunk order inside the receive buffer does not matter. */
int gscg_project_shard(gscg_ctx* ctx, const gscg_frame_desc* frame, const gscg_camera* cam,
                       const gscg_render_settings* settings, const gscg_lod_policy* lod,
                       uint32_t shard_begin, uint32_t shard_end, uint32_t bands, const uint32_t* band_rows,
                       uint64_t* band_counts, gscg_stage_times* times);
int gscg_pack_bands(gscg_ctx* ctx, void* send_dev);
int gscg_render_band(gscg_ctx* ctx, const void* recv_dev, uint64_t recv_count, uint32_t row_begin,
                     uint32_t row_end, float* fb_rgb, float* fb_T, int32_t memory, gscg_stage_times* times);

/* ---- Multi-GPU frame as one group call per frame ----
 * One process per GPU. Rank 0 makes a unique id (gscg_group_unique_id), the caller's
 * plumbing (e.g. torch.distributed) broadcasts the 128 bytes, every rank calls
 * gscg_group_create on its own context (ncclCommInitRank: the group owns the NCCL
 * communicator). gscg_group_render_frame renders rank r's screen region of the frame:
 * columns [cuts[r], cuts[r+1]) x every row (axis GSCG_SPLIT_COLS) or rows [cuts[r],
 * cuts[r+1]) x every column (GSCG_SPLIT_ROWS); cuts: nranks + 1 ascending tile-aligned
 * positions from 0 to the width / height (see gscg_set_region). Every region is then
 * gathered into rank 0's framebuffer with grouped ncclSend/ncclRecv on the context stream;
 * on rank 0 fb_rgb / fb_T (host or device, may be NULL) receive the whole frame, identical
 * to gscg_render_frame's. The call does not synchronise the host unless rank 0 is given
 * host destinations. gscg_group_tile_costs: the binned pairs of every tile of the last
 * frame (tiles_y x tiles_x, row-major) over all ranks (an all-reduce), for re-balancing
 * the cuts. */
#define GSCG_SPLIT_ROWS 0
#define GSCG_SPLIT_COLS 1
#define GSCG_UNIQUE_ID_BYTES 128
typedef struct gscg_group gscg_group;
int gscg_group_unique_id(uint8_t* out /* GSCG_UNIQUE_ID_BYTES */);
int gscg_group_create(gscg_ctx* ctx, const uint8_t* unique_id, int32_t nranks, int32_t rank, gscg_group** out);
/* SURVEY.md §8(b)'s proposed name for gscg_group_create (same arguments and behaviour). */
int gscg_create_group(gscg_ctx* ctx, const uint8_t* unique_id, int32_t nranks, int32_t rank, gscg_group** out);
int gscg_group_destroy(gscg_group* group);
int gscg_group_render_frame(gscg_group* group, const gscg_frame_desc* frame, const gscg_camera* cam,
                            const gscg_render_settings* settings, const gscg_lod_policy* lod, int32_t axis,
                            const uint32_t* cuts, float* fb_rgb, float* fb_T, gscg_stage_times* times);
/* The same frame with rank 0's read-back into host fb_rgb / fb_T left running on the
 * context's copy stream under the next frame (two whole-frame device buffers alternate):
 * the destinations must stay valid until gscg_group_wait_readback. */
int gscg_group_render_frame_async(gscg_group* group, const gscg_frame_desc* frame, const gscg_camera* cam,
                                  const gscg_render_settings* settings, const gscg_lod_policy* lod, int32_t axis,
                                  const uint32_t* cuts, float* fb_rgb, float* fb_T, gscg_stage_times* times);
int gscg_group_wait_readback(gscg_group* group);
int gscg_group_framebuffer_device(gscg_group* group, float** rgb, float** T); /* rank 0 */
int gscg_group_tile_costs(gscg_group* group, uint32_t tiles_x, uint32_t tiles_y, uint64_t* out /* tiles_y x tiles_x */);

#ifdef __cplusplus
}
#endif

#endif /* GSCG_H_ */
