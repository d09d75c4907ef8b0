// Kernel parameter blocks and declarations shared by the gscg translation units.
#pragma once

#include "gscg_common.cuh"

namespace gscg {

struct PlanParams {
    uint32_t n;
    uint32_t shard_begin, shard_end;  // instances projected by this context (all: 0, n)
    const uint32_t* template_ids;
    const float* placement;
    const uint32_t* lod_prev;
    int32_t forced_lod;
    uint32_t threshold_count;
    float thresholds[GSCG_MAX_LOD_THRESHOLDS];
    float hysteresis;
    float cam_pos[3];
    const TemplateDev* templates;
    const GroupDev* groups;
    uint32_t group_count;
    uint32_t* lod_out;
    uint32_t* inst_group;
    uint32_t* inst_base;
    uint32_t* group_inst_start;  // group_count + 1
    uint32_t* group_inst_count;
    uint32_t* group_item_start;  // group_count + 1
    uint32_t* members;
    const uint32_t* visible;  // k_inst_cull flags (null: every instance is projected)
    FrameCounters* counters;
};

// Instance frustum cull: one warp per instance bounds its posed means by a ball from its
// skin matrices and the template bounds, and proves every splat off-screen (see k_inst_cull).
struct CullParams {
    uint32_t n;      // end of the instance range
    uint32_t first;  // first instance (shard begin)
    uint32_t joint_stride;
    const uint32_t* template_ids;
    const TemplateDev* templates;
    const float* skin;
    CameraDev cam;
    uint32_t* visible;  // 1 = project, 0 = culled
};

struct FkParams {
    uint32_t n;      // end of the launch's instance range (bounds check)
    uint32_t first;  // first instance of the launch (shard begin)
    uint32_t joint_stride;
    uint32_t pose_stride;
    const uint32_t* template_ids;
    const float* placement;
    const float* poses;
    const TemplateDev* templates;
    const float* mats;
    const int32_t* parents;
    float* skin;  // n x joint_stride x 12 (rows 0..2 of each skin matrix, row-major)
};

struct ProjectParams {
    CameraDev cam;
    int32_t tile_size;
    int32_t tiles_x;
    int32_t sh_enabled;
    uint32_t joint_stride;
    uint32_t group_count;
    const GroupDev* groups;
    const uint32_t* group_item_start;
    const uint32_t* group_inst_start;
    const uint32_t* group_inst_count;
    const uint32_t* members;
    const uint32_t* inst_base;
    const float* skin;
    FrameCounters* counters;
    // outputs (capacity-checked)
    float4* records;  // 3 float4 per splat
    uint32_t* splat_depth;  // depth bits of every record (the splat sort keys)
    uint4* splat_meta;      // per record: ordinal, cx0 | cy0 << 16, across | down << 16, depth bits
    uint64_t splat_capacity;
    uint64_t pair_capacity;
    const float* posed_in;           // k_project<true, *>: posed means G x 3 by ordinal (no skinning)
    const float4* naive_core;        // k_project<*, true>: per-instance attribute copies by ordinal
    const float4* naive_weights;
    // debug outputs (may be null)
    float* posed_debug;              // G x 3 by ordinal
    gscg_splat_record* record_debug; // per splat
};

struct RasterParams {
    const uint2* ranges;
    const uint32_t* recs;  // record index of every cell-sorted pair
    const float4* records;
    int32_t width, height, tile_size, tiles_x;
    int32_t tile_row0;  // first tile row of the launch (screen band), 0 for a full frame
    int32_t out_row0;   // screen row stored in row 0 of out_rgb / out_T
    int32_t tile_col0;  // first tile column of the region (tiles_x counts the region's columns)
    int32_t out_col0;   // screen column stored in column 0 of out_rgb / out_T
    int32_t out_stride; // pixels per output row (the region's width)
    float bg[3];
    float alpha_max;
    float t_floor;
    float* out_rgb;
    float* out_T;
};

// Device pose sampling (gscg_pose.cu): uploaded clips as per-keyframe-pair slerp tables.
struct MotionDev {
    float fps;
    uint32_t frames, joints;
    uint32_t root_offset;  // into PoseParams::roots (one float4 per frame)
    uint64_t key_offset;   // into PoseParams::keys (frames x joints pairs (i, (i+1) % frames))
};

struct KeyPairDev {
    float4 a, b;           // keyframe i and keyframe i+1 (negated when dot < 0), x y z w
    float theta, sin_theta;  // acos(min(|dot|, 1)), sin(theta): host libm
    uint32_t lerp;         // |dot| > 0.9995: normalized lerp instead of slerp
    uint32_t pad;
};

struct PoseParams {
    uint32_t n;
    uint32_t joint_stride;
    float time_s;
    int32_t static_pose;
    const uint32_t* motion_ids;
    const float* phase;
    const MotionDev* motions;
    const float4* roots;
    const KeyPairDev* keys;
    float* poses;  // n x (4 + 4 * joint_stride)
};

__global__ void k_sample_poses(PoseParams p);
__global__ void k_eval_sinf(const float* in, float* out, uint32_t n);
__global__ void k_eval_expf(uint32_t first_bits, uint32_t n, float* out);

__global__ void k_lod_plan(PlanParams p);

// Small host <-> device transfers through mapped page-locked memory, done by a kernel so
// they never queue behind a framebuffer read-back on the copy engines (pipelined frames):
// segment y copies words[y] 32-bit words src[y] -> dst[y].
constexpr int kMaxCopySegs = 8;
struct CopySegs {
    const uint32_t* src[kMaxCopySegs];
    uint32_t* dst[kMaxCopySegs];
    uint32_t words[kMaxCopySegs];
};
__global__ void k_copy_segments(CopySegs c);
constexpr int kFkThreads = 128;  // k_fk_skin: 8 instances (half-warps) per block
constexpr int kFkSmemPerInstance(int joint_stride) { return joint_stride * 52 * 4; }  // world, bind, inverse, pose
__global__ void k_fk_skin(FkParams p);
__global__ void k_inst_cull(CullParams p);
// <false, false>: the frame (LBS from skin matrices, shared attribute store);
// <true, false>: given posed means; <false, true>: the naive per-instance layout.
template <bool kPosedIn, bool kNaive>
__global__ void k_project(ProjectParams p);
__global__ void k_naive_fill(const uint32_t* inst_group, const uint32_t* inst_base, const GroupDev* groups, uint32_t n,
                             float4* core, float4* weights);

// update_crowd's skin_means for every instance (gscg_skin_means): posed[ordinal] =
// LBS of the instance's level (avatar.cpp:178-192), the arithmetic k_project uses.
struct SkinParams {
    uint32_t n;
    uint32_t joint_stride;
    const uint32_t* inst_group;
    const uint32_t* inst_base;
    const GroupDev* groups;
    const float* skin;
    float* posed;  // G x 3
};
__global__ void k_skin_means(SkinParams p);
__global__ void k_set_power_floor(float4* core, const float* pf, uint32_t n);

// sort: splats by depth, pairs emitted in that order, pairs stably by cell
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kRadixBits = 5;  // widest digit of one LSD pass
constexpr int kRadix = 1 << kRadixBits;
constexpr uint32_t kSortTile = kSortThreads * kSortItems;
constexpr uint32_t kMaxSortPasses = 8;

// One stable LSD pass (reduce-then-scan): digit = (key >> shift) & (2^bits - 1).
struct SortPassParams {
    const uint32_t* keys_in;
    const uint32_t* vals_in;  // null: value = index (first pass of the splat sort)
    uint32_t* keys_out;
    uint32_t* vals_out;
    uint32_t count;
    uint32_t shift;
    uint32_t bits;
    uint32_t tiles;      // ceil(count / kSortTile)
    uint32_t* counts;      // kRadix x tiles, digit-major: tile digit counts -> exclusive offsets
    uint32_t* digit_base;  // kRadix: row totals (scanned by each downsweep CTA)
    // Deferred frames (enqueued before the host reads the counters): the pass count is
    // min(count, *count_dev), count and tiles then being the capacity the grid covers.
    const unsigned long long* count_dev;
};

__device__ __forceinline__ uint32_t resolve_count(uint32_t cap, const unsigned long long* count_dev) {
    if (!count_dev) return cap;
    const unsigned long long c = *count_dev;
    return c < cap ? static_cast<uint32_t>(c) : cap;
}

__global__ void k_sort_upsweep(SortPassParams p);
__global__ void k_sort_rows(SortPassParams p);
__global__ void k_sort_downsweep(SortPassParams p);
constexpr int kWideBits = 7;  // digit bits of the wide passes
constexpr int kWideRadix = 1 << kWideBits;
__global__ void k_sort_upsweep_wide(SortPassParams p);
__global__ void k_sort_downsweep_wide(SortPassParams p);

// Depth bucket sort (gscg_depth.cu): the splats in non-decreasing T = dbits >> drop.
constexpr int kBucketThreads = 1024;
constexpr int kBucketItems = 16;
constexpr uint32_t kBucketTile = kBucketThreads * kBucketItems;  // splats per count CTA
constexpr int kBucketScatterItems = 8;
constexpr uint32_t kBucketScatterTile = kBucketThreads * kBucketScatterItems;  // splats per scatter CTA (ranks < 2^16)
constexpr int kBucketTopBits = 15;
constexpr uint32_t kMaxDepthBuckets = 1u << kBucketTopBits;       // top bits of T (<= 128 KB shared histogram)
constexpr int kBucketLocalThreads = 256;
constexpr uint32_t kBucketLocalBins = 2048;                        // low bits of T per bucket (T <= 25 bits)
constexpr uint32_t kBucketLocalCap = 2048;                         // splats per bulk-copied chunk (32 KB)
constexpr uint32_t kBucketLocalChunks = 3;                         // buckets up to this many chunks write coalesced
struct DepthBucketParams {
    const uint32_t* depth;  // S depth key bits, record order
    const uint4* meta;      // S (ordinal, span lo, span hi, dbits), record order
    uint32_t count;         // S
    uint32_t drop;          // T = dbits >> drop
    uint32_t tag_min;       // min T of the frame
    uint32_t local_bits;    // bucket = (T - tag_min) >> local_bits; local bins = 2^local_bits
    uint32_t buckets;
    uint32_t* bucket_count;   // [buckets], zeroed
    uint32_t* bucket_start;   // [buckets + 1]
    uint32_t* bucket_cursor;  // [buckets]
    uint4* staged;            // [S] (dbits, record, span lo, span hi) grouped by bucket
    uint32_t* keys_out;       // [S] dbits, depth order
    uint32_t* recs_out;       // [S] record index
    uint2* spans_out;         // [S] binning span
};
__global__ void k_depth_bucket_count(DepthBucketParams p);
__global__ void k_depth_bucket_scan(DepthBucketParams p);
__global__ void k_depth_bucket_scatter(DepthBucketParams p);
__global__ void k_depth_bucket_local(DepthBucketParams p);

constexpr int kMetaThreads = 128;  // k_sorted_spans: 128 threads x kStreamItems = one 1024-splat block
__global__ void k_sorted_spans(const uint32_t* recs, const uint4* meta, uint32_t count, const unsigned long long* count_dev,
                               uint2* span_sorted);
constexpr uint32_t kLongRun = 32;       // runs of equal pair keys longer than this go to k_pair_long_runs
constexpr uint32_t kPairRunCap = 2048;  // k_pair_long_runs sorts runs up to this size in shared memory
// long_runs must hold count / kLongRun + count / 2048 + 2 entries (runs longer than
// kLongRun, plus at most one run leaving each 2048-pair fix-up tile).
__global__ void k_cell_fixup(const uint32_t* keys, uint32_t* recs, const uint4* meta, uint32_t count,
                             const unsigned long long* count_dev, uint32_t cell_mask, int fix, uint2* ranges,
                             uint2* long_runs, uint32_t* long_count, uint32_t long_cap);
__global__ void k_pair_long_runs(const uint32_t* keys, uint32_t count, const unsigned long long* count_dev,
                                 uint32_t* recs, const uint4* meta, const uint2* long_runs, const uint32_t* long_count);
constexpr int kEmitThreads = 128;  // k_emit_scatter: 4 sorted splats per thread
constexpr uint32_t kEmitSplats = 4 * kEmitThreads;  // sorted splats per emission block
constexpr uint32_t kEmitStage = 2048;  // pairs per block staged in shared memory for coalesced writes
constexpr int kEmitSmem = (32 * kEmitThreads + 2 * kEmitStage) * 4;  // dynamic shared bytes
struct EmitCounts {  // deferred frames: the splat count from the device counter (null: the host's)
    const unsigned long long* count_dev;
};
template <bool kCount, bool kQuads>
__global__ void k_emit_scatter(const uint32_t* rec_sorted, const uint32_t* key_sorted, uint32_t count,
                               const uint2* span_sorted, uint32_t* block_digit, const uint32_t* digit_total,
                               uint32_t blocks, int tiles_x, int quads, uint32_t dmask, uint32_t tag_drop,
                               uint32_t tag_shift, uint32_t* pair_cell, uint32_t* pair_rec, EmitCounts dc);
// Launches count (true) or scatter (false); defined in the sort TU (template instantiation).
// key_sorted (may be null: no tags) are the depth-sorted keys; a pair's key word is
// cell | ((key >> tag_drop) << tag_shift) (see k_cell_fixup).
void launch_emit(bool count_only, uint32_t blocks, cudaStream_t s, const uint32_t* rec_sorted, const uint32_t* key_sorted,
                 uint32_t count, const uint2* span_sorted, uint32_t* block_digit, const uint32_t* digit_total,
                 int tiles_x, int quads, uint32_t dmask, uint32_t tag_drop, uint32_t tag_shift, uint32_t* pair_cell,
                 uint32_t* pair_rec, EmitCounts dc);
constexpr int kStreamItems = 8;  // elements per thread in the streaming sort kernels

// screen-band exchange (multi-GPU frame)
constexpr int kMaxBands = GSCG_MAX_BANDS;

struct BandParams {
    const float4* records;
    const uint4* meta;
    const uint32_t* depth;
    uint32_t count;
    uint32_t bands;
    uint32_t rows[kMaxBands + 1];  // band b = screen rows [rows[b], rows[b+1])
    unsigned long long* band_counts;  // count pass
    unsigned long long* band_cursor;  // pack pass (zeroed)
    unsigned long long band_offsets[kMaxBands];
    uint4* packed;  // 4 x uint4 per BandSplat: r0, r1, r2, (ordinal, depth, 0, 0)
};

struct BandUnpackParams {
    const uint4* packed;
    uint32_t count;
    int32_t row_begin, row_end;  // the band's screen rows
    int32_t cell;                // binning cell edge in pixels
    float4* records;
    uint32_t* depth;
    uint4* meta;
    FrameCounters* counters;
};

__global__ void k_band_count(BandParams p);
__global__ void k_band_pack(BandParams p);
__global__ void k_band_unpack(BandUnpackParams p);
__global__ void k_tile_costs(const uint2* ranges, uint32_t region_tiles_x, uint32_t region_rows, uint32_t cells_per_tile,
                             int32_t tile_col0, int32_t tile_row0, uint32_t tiles_x, unsigned long long* out);

// metrics
constexpr int kSseThreads = 256;
constexpr uint32_t kSseBlocks = 1024;
__global__ void k_sse_partial(const float* a, const float* b, uint64_t n, double* partial);
__global__ void k_sse_final(const double* partial, uint32_t blocks, double* out);

// raster
constexpr int kReadbackBands = 4;  // tile-row bands of a frame whose host read-back overlaps the raster
// Picks the tile-size specialisation (16: 8x8 quadrant CTAs; else 1/4/16 pixels per thread).
void launch_raster(const RasterParams& p, uint32_t tiles, cudaStream_t stream);

// stage functions
__global__ void k_iota2(uint32_t* a, uint32_t* b, uint32_t n);  // a[i] = b[i] = i
__global__ void k_gather_u32(const uint32_t* src, const uint32_t* idx, uint32_t* dst, uint32_t n);

// debug
__global__ void k_sorted_ordinals(const uint32_t* recs, const uint4* meta, uint32_t count, uint32_t* out);

}  // namespace gscg
