// Stage "sort", last step for 16-px tiles: the per-tile lists split into the rasteriser's
// four 8x8 quadrant lists (reference binning renderer.cpp:143-161 bins by tile; the
// quadrant lists are the tile's list restricted to each quadrant, in the tile's order).
//
// On this path emission, the stable cell passes and k_cell_fixup run over TILE pairs (the
// reference's own pairs: ~30% fewer than quadrant pairs at config 3), each record word
// carrying the tile's quadrants its splat covers in bits 28..31. The split then writes
// every tile pair into the lists of its quadrants:
//
//   k_quad_split_count  per 2,048-pair chunk, the pairs of each quadrant bit
//   k_sort_rows         (4 rows) chunk offsets P_q(chunk) = pairs with bit q before it
//   k_quad_split        quadrant q of tile t is stored at 4 x_t + q len_t (tile t's pairs
//                       being [x_t, x_t + len_t)), a pair at P_q(i) - P_q(x_t) in it; the
//                       chunk holding a tile's last pair writes its four quadrant ranges
//
// Quadrant lists keep gaps (4 x len_t slots per tile), so no global scan of the quadrant
// counts is needed.
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

constexpr uint32_t kSplitThreads = 256;
constexpr uint32_t kSplitItems = 8;

__device__ __forceinline__ uint32_t split_warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Exclusive scan over the CTA of two packed words (each two 16-bit counters, <= 2,048).
__device__ __forceinline__ void split_excl_scan2(uint32_t& a, uint32_t& b, uint32_t (*s_warp)[2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int nw = kSplitThreads / 32;
    const uint32_t xa = split_warp_incl_scan(a, lane), xb = split_warp_incl_scan(b, lane);
    if (lane == 31) {
        s_warp[warp][0] = xa;
        s_warp[warp][1] = xb;
    }
    __syncthreads();
    uint32_t pa = 0, pb = 0;
    for (int w = 0; w < warp; ++w) {
        pa += s_warp[w][0];
        pb += s_warp[w][1];
    }
    a = pa + xa - a;
    b = pb + xb - b;
    (void)nw;
}

__device__ __forceinline__ uint32_t field(uint32_t lo, uint32_t hi, int q) {  // counter q of the packed pair
    const uint32_t w = q < 2 ? lo : hi;
    return (q & 1) ? w >> 16 : w & 0xffffu;
}

__device__ __forceinline__ void add_mask(uint32_t& lo, uint32_t& hi, uint32_t m) {
    lo += (m & 1u) | ((m & 2u) << 15);
    hi += ((m >> 2) & 1u) | ((m & 8u) << 13);
}

}  // namespace

__global__ void __launch_bounds__(kSplitThreads)
k_quad_split_count(QuadSplitParams p) {
    pdl_entry();
    __shared__ uint32_t s_cnt[4];
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    const uint32_t c0 = blockIdx.x * kQuadSplitChunk;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (uint32_t j = 0; j < kSplitItems; ++j) {
        const uint32_t i = c0 + j * kSplitThreads + threadIdx.x;
        if (i < p.count) add_mask(lo, hi, p.recs[i] >> kRecMaskShift);
    }
    lo = __reduce_add_sync(0xffffffffu, lo);
    hi = __reduce_add_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_cnt[0], lo & 0xffffu);
        atomicAdd(&s_cnt[1], lo >> 16);
        atomicAdd(&s_cnt[2], hi & 0xffffu);
        atomicAdd(&s_cnt[3], hi >> 16);
    }
    __syncthreads();
    if (threadIdx.x < 4) p.chunk_counts[threadIdx.x * p.chunks + blockIdx.x] = s_cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kSplitThreads)
k_quad_split(QuadSplitParams p) {
    pdl_entry();
    __shared__ uint32_t s_pref[2][kQuadSplitChunk];  // exclusive in-chunk prefix at every position
    __shared__ uint32_t s_warp[kSplitThreads / 32][2];
    __shared__ uint32_t s_off[4];    // P_q at the chunk start
    __shared__ uint32_t s_enter[4];  // P_q at the first pair of a tile entering from earlier chunks
    const uint32_t c0 = blockIdx.x * kQuadSplitChunk;
    const uint32_t tid = threadIdx.x, t0 = tid * kSplitItems;
    uint32_t r[kSplitItems], k[kSplitItems];
    const uint32_t n_here = min(kQuadSplitChunk, p.count - c0);
    if (n_here == kQuadSplitChunk) {
        const uint4 rlo = *reinterpret_cast<const uint4*>(p.recs + c0 + t0);
        const uint4 rhi = *reinterpret_cast<const uint4*>(p.recs + c0 + t0 + 4);
        const uint4 klo = *reinterpret_cast<const uint4*>(p.keys + c0 + t0);
        const uint4 khi = *reinterpret_cast<const uint4*>(p.keys + c0 + t0 + 4);
        r[0] = rlo.x; r[1] = rlo.y; r[2] = rlo.z; r[3] = rlo.w; r[4] = rhi.x; r[5] = rhi.y; r[6] = rhi.z; r[7] = rhi.w;
        k[0] = klo.x; k[1] = klo.y; k[2] = klo.z; k[3] = klo.w; k[4] = khi.x; k[5] = khi.y; k[6] = khi.z; k[7] = khi.w;
    } else {
#pragma unroll
        for (uint32_t j = 0; j < kSplitItems; ++j) {
            const bool in = t0 + j < n_here;
            r[j] = in ? p.recs[c0 + t0 + j] : 0u;
            k[j] = in ? p.keys[c0 + t0 + j] : 0u;
        }
    }
    if (tid < 4) s_off[tid] = p.chunk_counts[tid * p.chunks + blockIdx.x];
    // The tile entering from an earlier chunk: P_q at its first pair = the offsets of the
    // chunk holding that pair + that chunk's pairs before it.
    const uint32_t first_tile = p.keys[c0] & p.cell_mask;
    const uint32_t xe = p.tile_ranges[first_tile].x;
    if (xe < c0) {
        const uint32_t ce = xe / kQuadSplitChunk, b0 = ce * kQuadSplitChunk;
        uint32_t lo = 0, hi = 0;
        for (uint32_t i = b0 + tid; i < xe; i += kSplitThreads) add_mask(lo, hi, p.recs[i] >> kRecMaskShift);
        lo = __reduce_add_sync(0xffffffffu, lo);
        hi = __reduce_add_sync(0xffffffffu, hi);
        if (tid < 4) s_enter[tid] = p.chunk_counts[tid * p.chunks + ce];
        __syncthreads();
        if ((tid & 31) == 0) {
            atomicAdd(&s_enter[0], lo & 0xffffu);
            atomicAdd(&s_enter[1], lo >> 16);
            atomicAdd(&s_enter[2], hi & 0xffffu);
            atomicAdd(&s_enter[3], hi >> 16);
        }
    }
    // In-chunk exclusive prefixes, packed two 16-bit counters per word.
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (uint32_t j = 0; j < kSplitItems; ++j) add_mask(lo, hi, r[j] >> kRecMaskShift);
    split_excl_scan2(lo, hi, s_warp);
#pragma unroll
    for (uint32_t j = 0; j < kSplitItems; ++j) {
        s_pref[0][t0 + j] = lo;
        s_pref[1][t0 + j] = hi;
        add_mask(lo, hi, r[j] >> kRecMaskShift);
    }
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kSplitItems; ++j) {
        const uint32_t pos = t0 + j;
        if (pos >= n_here) break;
        const uint32_t i = c0 + pos;
        const uint32_t t = k[j] & p.cell_mask;
        const uint2 tr = p.tile_ranges[t];
        const uint32_t len = tr.y - tr.x, m = r[j] >> kRecMaskShift, rec = r[j] & kRecIndexMask;
        const uint32_t plo = s_pref[0][pos], phi = s_pref[1][pos];
        const bool inside = tr.x >= c0;
        const uint32_t xlo = inside ? s_pref[0][tr.x - c0] : 0u, xhi = inside ? s_pref[1][tr.x - c0] : 0u;
        const bool last = i + 1 == tr.y;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t at = s_off[q] + field(plo, phi, q);                          // P_q(i)
            const uint32_t base = inside ? s_off[q] + field(xlo, xhi, q) : s_enter[q];  // P_q(x_t)
            const uint32_t slot0 = 4u * tr.x + static_cast<uint32_t>(q) * len;
            const bool has = (m >> q) & 1u;
            if (has) p.out[slot0 + (at - base)] = rec;
            if (last) p.quad_ranges[4u * t + q] = make_uint2(slot0, slot0 + (at + (has ? 1u : 0u) - base));
        }
    }
}

}  // namespace gscg
