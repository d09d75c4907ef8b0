// Screen-band exchange of the multi-GPU frame (the reference is
// single-process — this is the scale-out of renderer.cpp:143-231 across GPUs).
//
// Every rank projects its contiguous instance shard (global ordinals, k_lod_plan over the
// whole crowd), then routes each surviving splat to every horizontal screen band its
// pixel rect overlaps:
//   k_band_count — splats per destination band (the send counts of the all-to-all)
//   k_band_pack  — 64-byte BandSplat records grouped by band at the caller's offsets
// After the exchange the band owner unpacks the received splats into its own record
// arrays and re-derives each splat's binning span clipped to the band:
//   k_band_unpack — records / ordinal / depth / span, pair count and depth-bit range
// Order inside a band's chunk does not matter: the band sorts by (depth, ordinal), the
// reference's total order (renderer.cpp:85-107), so band pixels equal the 1-GPU frame's.
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

// Inclusive band range [b0, b1] a pixel-row interval [y0, y1) overlaps (b1 < b0: none).
__device__ __forceinline__ void band_range(const BandParams& p, uint32_t y0, uint32_t y1, int& b0, int& b1) {
    b0 = 0;
    b1 = -1;
    if (y1 <= y0) return;
    int b = 0;
    while (b < static_cast<int>(p.bands) && p.rows[b + 1] <= y0) ++b;
    b0 = b;
    while (b < static_cast<int>(p.bands) && p.rows[b] < y1) ++b;
    b1 = b - 1;
}

__device__ __forceinline__ void splat_rows(const float4* records, uint32_t i, uint32_t& y0, uint32_t& y1) {
    const float4 r2 = records[3ull * i + 2];
    y0 = __float_as_uint(r2.z) >> 16;
    y1 = __float_as_uint(r2.w) >> 16;
}

}  // namespace

__global__ void __launch_bounds__(256)
k_band_count(BandParams p) {
    __shared__ uint32_t s_cnt[kMaxBands];
    for (int b = threadIdx.x; b < kMaxBands; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    const uint32_t base = blockIdx.x * (256u * kStreamItems);
#pragma unroll
    for (int k = 0; k < kStreamItems; ++k) {
        const uint32_t i = base + k * 256u + threadIdx.x;
        if (i >= p.count) break;
        uint32_t y0, y1;
        splat_rows(p.records, i, y0, y1);
        int b0, b1;
        band_range(p, y0, y1, b0, b1);
        for (int b = b0; b <= b1; ++b) atomicAdd(&s_cnt[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < static_cast<int>(p.bands); b += blockDim.x)
        if (s_cnt[b]) atomicAdd(&p.band_counts[b], static_cast<unsigned long long>(s_cnt[b]));
}

__global__ void __launch_bounds__(256)
k_band_pack(BandParams p) {
    __shared__ uint32_t s_cnt[kMaxBands];
    __shared__ unsigned long long s_base[kMaxBands];
    for (int b = threadIdx.x; b < kMaxBands; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    const uint32_t base = blockIdx.x * (256u * kStreamItems);
    int b0s[kStreamItems], b1s[kStreamItems];
#pragma unroll
    for (int k = 0; k < kStreamItems; ++k) {
        const uint32_t i = base + k * 256u + threadIdx.x;
        b0s[k] = 0;
        b1s[k] = -1;
        if (i < p.count) {
            uint32_t y0, y1;
            splat_rows(p.records, i, y0, y1);
            band_range(p, y0, y1, b0s[k], b1s[k]);
            for (int b = b0s[k]; b <= b1s[k]; ++b) atomicAdd(&s_cnt[b], 1u);
        }
    }
    __syncthreads();
    // One reservation per (block, band) in the band's chunk of the send buffer.
    for (int b = threadIdx.x; b < static_cast<int>(p.bands); b += blockDim.x) {
        s_base[b] = s_cnt[b] ? p.band_offsets[b] + atomicAdd(&p.band_cursor[b], static_cast<unsigned long long>(s_cnt[b]))
                             : 0ull;
        s_cnt[b] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kStreamItems; ++k) {
        const uint32_t i = base + k * 256u + threadIdx.x;
        if (b1s[k] < b0s[k]) continue;
        const float4* src = p.records + 3ull * i;
        const float4 r0 = src[0], r1 = src[1], r2 = src[2];
        const uint4 meta = make_uint4(p.meta[i].x, p.depth[i], 0u, 0u);
        for (int b = b0s[k]; b <= b1s[k]; ++b) {
            const unsigned long long slot = s_base[b] + atomicAdd(&s_cnt[b], 1u);
            float4* dst = reinterpret_cast<float4*>(p.packed + 4ull * slot);
            dst[0] = r0;
            dst[1] = r1;
            dst[2] = r2;
            p.packed[4ull * slot + 3] = meta;
        }
    }
}

__global__ void __launch_bounds__(256)
k_band_unpack(BandUnpackParams p) {
    __shared__ unsigned long long s_pairs;
    __shared__ uint32_t s_dmin, s_dmax;
    if (threadIdx.x == 0) {
        s_pairs = 0ull;
        s_dmin = 0xffffffffu;
        s_dmax = 0u;
    }
    __syncthreads();
    const uint32_t base = blockIdx.x * (256u * kStreamItems);
    const int lane = threadIdx.x & 31;
    uint32_t pairs = 0, dmin = 0xffffffffu, dmax = 0u;
#pragma unroll
    for (int k = 0; k < kStreamItems; ++k) {
        const uint32_t i = base + k * 256u + threadIdx.x;
        if (i >= p.count) break;
        const float4* src = reinterpret_cast<const float4*>(p.packed + 4ull * i);
        const float4 r0 = src[0], r1 = src[1], r2 = src[2];
        const uint4 meta = p.packed[4ull * i + 3];
        float4* dst = p.records + 3ull * i;
        dst[0] = r0;
        dst[1] = r1;
        dst[2] = r2;
        p.depth[i] = meta.y;
        const uint32_t xy0 = __float_as_uint(r2.z), xy1 = __float_as_uint(r2.w);
        const int x0 = static_cast<int>(xy0 & 0xffffu), y0 = static_cast<int>(xy0 >> 16);
        const int x1 = static_cast<int>(xy1 & 0xffffu), y1 = static_cast<int>(xy1 >> 16);
        // Binning span of the rect clipped to the band, cell rows relative to the band.
        const int yc0 = max(y0, p.row_begin), yc1 = min(y1, p.row_end);
        const int cx0 = x0 / p.cell, cy0 = yc0 / p.cell;
        const uint32_t across = static_cast<uint32_t>((x1 - 1) / p.cell - cx0 + 1);
        const uint32_t down = static_cast<uint32_t>((yc1 - 1) / p.cell - cy0 + 1);
        p.meta[i] = make_uint4(meta.x, static_cast<uint32_t>(cx0) | (static_cast<uint32_t>(cy0 - p.row_begin / p.cell) << 16),
                               across | (down << 16), meta.y);
        pairs += across * down;
        dmin = min(dmin, meta.y);
        dmax = max(dmax, meta.y);
    }
    pairs = __reduce_add_sync(0xffffffffu, pairs);
    dmin = __reduce_min_sync(0xffffffffu, dmin);
    dmax = __reduce_max_sync(0xffffffffu, dmax);
    if (lane == 0) {
        atomicAdd(&s_pairs, static_cast<unsigned long long>(pairs));
        atomicMin(&s_dmin, dmin);
        atomicMax(&s_dmax, dmax);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_pairs) atomicAdd(&p.counters->pairs, s_pairs);
        if (s_dmin != 0xffffffffu) atomicMin(&p.counters->depth_min_bits, s_dmin);
        atomicMax(&p.counters->depth_max_bits, s_dmax);
    }
}

// Pairs per tile of a frame region (the region balance of the multi-GPU frame): one
// thread per region tile sums its cells' range lengths into the frame's tile map.
__global__ void k_tile_costs(const uint2* ranges, uint32_t region_tiles_x, uint32_t region_rows, uint32_t cells_per_tile,
                             int32_t tile_col0, int32_t tile_row0, uint32_t tiles_x, unsigned long long* out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= region_tiles_x * region_rows) return;
    unsigned long long sum = 0;
    for (uint32_t c = 0; c < cells_per_tile; ++c) {
        const uint2 r = ranges[static_cast<size_t>(t) * cells_per_tile + c];
        sum += r.y - r.x;
    }
    const uint32_t tx = t % region_tiles_x + tile_col0, ty = t / region_tiles_x + tile_row0;
    out[static_cast<size_t>(ty) * tiles_x + tx] = sum;
}

}  // namespace gscg
