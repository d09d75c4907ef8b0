// Shared device definitions for the B200 crowd-render kernels (sm_100a).
//
// Parity-critical arithmetic (skin matrices, LBS, LoD distance, EWA projection, conic,
// per-pixel power) reproduces the reference's single-rounded SSE evaluation order
// (SURVEY.md Appendix A). The translation units that hold it are compiled with
// --fmad=false, and the expressions below are parenthesised in exactly the reference
// order, so no FMA contraction or reassociation can change a bit.
#pragma once

#include <cstdio>

#include <cstdint>
#include <cuda_runtime.h>
#include <utility>

#include "gscg.h"

namespace gscg {

constexpr int kMaxJoints = GSCG_MAX_JOINTS;
constexpr int kMaxGroups = 256;      // (template, level) pairs resident at once
constexpr int kProjectThreads = 256; // Gaussians per work-item chunk
constexpr int kBatch = 8;           // instances per template-major work item
constexpr int kShFloats = GSCG_SH_FLOATS;

// One (template, level) group of the shared attribute store in HBM.
//   core[4*g+0] = mean.x, mean.y, mean.z, opacity
//   core[4*g+1] = cov xx, xy, xz, yy
//   core[4*g+2] = cov yz, zz, red, green
//   core[4*g+3] = blue, power_floor, idx0|idx1<<16, idx2|idx3<<16
//   weights[g]  = skin weights w0..w3
//   sh[45*g+3*k+c] = SH residual coefficient k (degree 1..3) of channel c (optional)
struct GroupDev {
    const float4* core;
    const float4* weights;
    const float* sh;
    uint32_t count;
    uint32_t template_id;
    uint32_t level;
    uint32_t pad;
};

struct TemplateDev {
    int32_t joint_count;
    int32_t level_count;
    int32_t group_base;  // group id of level 0
    int32_t mat_offset;  // first matrix in the skeleton matrix table (local_bind then inverse_bind)
    int32_t parent_offset;
    float pelvis_y;
    // Conservative bounds over all levels for the instance frustum cull (k_inst_cull):
    // max |mean|, max sqrt(Gershgorin bound of the covariance), max sum |w_k|,
    // max |sum w_k - 1|. +inf disables the cull for the template.
    float cull_mean_r, cull_sigma, cull_wabs, cull_wdev;
    int32_t pad[2];
};

struct CameraDev {
    float w[9];  // world_to_view row-major
    float pos[3];
    float focal, cx, cy, near_m;
    int32_t width, height;
    // The screen region this context renders (gscg_set_region; the whole frame: 0, 0, width, height).
    int32_t band_x0, band_y0, band_x1, band_y1;
};

// Frame-level counters written by the kernels and read back once per frame.
struct FrameCounters {
    unsigned long long splats;     // S of the frame (record slots handed out), block aggregates
    unsigned long long pairs;      // K of the frame (cell-splat pairs), warp aggregates
    unsigned long long gaussians;  // G of the frame (global ordinals must stay below 2^32)
    unsigned long long tile_pairs; // the reference's (tile, splat) bin entries (renderer.cpp:147-161)
    uint32_t depth_min_bits;
    uint32_t depth_max_bits;
    uint32_t items_total;
    uint32_t item_cursor;
    uint32_t sort_ticket[8];  // onesweep tile tickets, one per pass of the frame
    uint32_t instances_culled;  // instances whose every splat is provably off-screen (k_inst_cull)
};

// float -> int as x86 cvttss2si (the reference's static_cast<int>): truncation, with
// the "integer indefinite" INT_MIN for NaN and out-of-range values (SURVEY A8 note).
__device__ __forceinline__ int x86_float_to_int(float v) {
    // |v| < 2^31 is exactly the in-range set: -2^31 itself converts to INT_MIN either way.
    return fabsf(v) < 2147483648.0f ? __float2int_rz(v) : INT32_MIN;
}

// Device bounds checks of the checked build (lib_checked/, -DGSCG_DEVICE_CHECKS; the pool
// has no compute-sanitizer): a failed check prints its site and traps, so the API call
// returns a CUDA error. Compiled out of the product build.
#ifdef GSCG_DEVICE_CHECKS
#define GSCG_DCHECK(cond)                                                                          \
    do {                                                                                           \
        if (!(cond)) {                                                                             \
            printf("GSCG_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,          \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x), #cond);            \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define GSCG_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch (PDL): the frame's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so kernel N+1's CTAs are scheduled
// while kernel N's last wave runs instead of after it drains. Every such kernel starts with
// pdl_entry(): griddepcontrol.wait blocks until the predecessor grid has completed and its
// memory is visible (so no kernel ever reads a predecessor's output early, and completion
// stays transitive down the chain); launch_dependents then lets the successor launch once
// every CTA of this grid has passed that point. A kernel launched without the attribute
// passes straight through both.
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Bulk (TMA) copies global -> shared completing on an mbarrier: one instruction per
// contiguous block instead of a 16-byte cp.async per thread and iteration.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(phase)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}


bool pdl_enabled();  // GSCG_NO_PDL=1 turns the attribute off (A/B measurements)

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace gscg
