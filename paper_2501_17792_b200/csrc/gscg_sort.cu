// Stage "sort" on the B200: the reference's own two-step order — sort the splats by
// depth, then bin them into tiles in that order (sort_splats_impl renderer.cpp:85-107,
// binning renderer.cpp:143-161) — restated as three device passes:
//
//   1. k_onesweep over the S splat depth keys (32-bit, only the bits that vary in the
//      frame), values = record index; k_tie_fixup orders equal-depth runs by splat
//      ordinal (instance base + gaussian index) = the reference's (instance, gaussian)
//      tie-break. The splats are now in the reference's total order.
//   2. k_splat_cells + k_scan_sums + k_emit_pairs: every sorted splat emits one pair per
//      overlapped binning cell (tile, or 8x8 quadrant of a 16-px tile), in sorted order.
//   3. k_onesweep (stable) over the pairs' cell ids; k_cell_ranges marks each cell's
//      [start, end). Stability keeps the depth order inside every cell, so each cell
//      list is exactly the reference's bin restricted to the cell.
//
// Onesweep pass: a CTA takes a 4096-key tile by atomic ticket (forward progress for the
// look-back), ranks keys stably per warp with __match_any_sync, publishes its digit
// counts, resolves its global digit offsets by decoupled look-back over the preceding
// tiles, stages the tile in shared memory in digit order and writes it out coalesced.
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;

__device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, uint32_t epoch, uint32_t value) {
    return flag | (static_cast<unsigned long long>(epoch & 0x3fffffffu) << 32) | value;
}

__device__ __forceinline__ unsigned long long load_status(const unsigned long long* addr) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void store_status(unsigned long long* addr, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(addr), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Exclusive block scan (blockDim.x multiple of 32); s_warp holds 32 words.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t x = warp_incl_scan(v, lane);
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = warp_incl_scan(lane < nw ? s_warp[lane] : 0u, lane);
        if (lane < nw) s_warp[lane] = w;
    }
    __syncthreads();
    total = s_warp[nw - 1];
    const uint32_t r = (warp ? s_warp[warp - 1] : 0u) + x - v;
    __syncthreads();
    return r;
}

}  // namespace

__global__ void __launch_bounds__(256)
k_digit_histogram(const uint32_t* keys, uint32_t count, SortPlan plan, uint32_t* hist) {
    __shared__ uint32_t s_hist[kMaxSortPasses][256];
    for (int i = threadIdx.x; i < kMaxSortPasses * 256; i += blockDim.x) (&s_hist[0][0])[i] = 0u;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const uint32_t key = keys[i];
        for (uint32_t q = 0; q < plan.passes; ++q)
            atomicAdd(&s_hist[q][(key >> plan.shift[q]) & ((1u << plan.bits[q]) - 1u)], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < plan.passes * 256; i += blockDim.x) {
        const uint32_t c = (&s_hist[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// In-place exclusive scan of each pass's 256-bin histogram (one CTA per pass).
__global__ void __launch_bounds__(256) k_digit_scan(uint32_t* hist) {
    __shared__ uint32_t s_warp[32];
    uint32_t* h = hist + blockIdx.x * 256;
    const uint32_t v = h[threadIdx.x];
    uint32_t total;
    h[threadIdx.x] = block_excl_scan(v, s_warp, total);
}

__global__ void __launch_bounds__(kSortThreads)
k_onesweep(SortPassParams p) {
    __shared__ uint32_t s_keys[kSortTile];
    __shared__ uint32_t s_vals[kSortTile];
    __shared__ uint32_t s_wcount[kSortThreads / 32][256];
    __shared__ uint32_t s_block_excl[256];
    __shared__ uint32_t s_global[256];
    __shared__ uint32_t s_scan[32];
    __shared__ uint32_t s_block;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_block = atomicAdd(p.ticket, 1u);
    for (int i = tid; i < (kSortThreads / 32) * 256; i += kSortThreads) (&s_wcount[0][0])[i] = 0u;
    __syncthreads();
    const uint32_t b = s_block;
    const uint32_t base = b * kSortTile;
    const uint32_t mask = (1u << p.bits) - 1u;

    uint32_t k[kSortItems], v[kSortItems], d[kSortItems], rank[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const bool valid = idx < p.count;
        k[j] = valid ? p.keys_in[idx] : 0u;
        v[j] = valid ? (p.vals_in ? p.vals_in[idx] : idx) : 0u;
        d[j] = valid ? ((k[j] >> p.shift) & mask) : 256u;
    }
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t peers = __match_any_sync(0xffffffffu, d[j]);
        const int leader = __ffs(peers) - 1;
        uint32_t prior = 0;
        if (lane == leader && d[j] < 256u) {
            prior = s_wcount[warp][d[j]];
            s_wcount[warp][d[j]] = prior + __popc(peers);
        }
        prior = __shfl_sync(0xffffffffu, prior, leader);
        rank[j] = prior + __popc(peers & lt_mask);
        __syncwarp();  // the next item's leaders read counters this item's leaders wrote
    }
    __syncthreads();

    // Thread tid owns digit tid: exclusive prefix over warps, block total.
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) {
        const uint32_t c = s_wcount[w][tid];
        s_wcount[w][tid] = total;
        total += c;
    }
    uint32_t all;
    s_block_excl[tid] = block_excl_scan(total, s_scan, all);

    // Decoupled look-back for this digit over preceding tiles.
    unsigned long long* my = p.status + static_cast<size_t>(b) * 256 + tid;
    uint32_t excl = 0;
    if (b == 0) {
        store_status(my, pack_status(kFlagIncl, p.epoch, total));
    } else {
        store_status(my, pack_status(kFlagAgg, p.epoch, total));
        int pb = static_cast<int>(b) - 1;
        for (;;) {
            const unsigned long long w = load_status(p.status + static_cast<size_t>(pb) * 256 + tid);
            const uint32_t ep = static_cast<uint32_t>(w >> 32) & 0x3fffffffu;
            const unsigned long long flag = w & (3ull << 62);
            if (flag == 0ull || ep != (p.epoch & 0x3fffffffu)) continue;
            excl += static_cast<uint32_t>(w);
            if (flag == kFlagIncl) break;
            --pb;
        }
        store_status(my, pack_status(kFlagIncl, p.epoch, excl + total));
    }
    s_global[tid] = p.digit_offsets[tid] + excl;
    __syncthreads();

#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        if (d[j] < 256u) {
            const uint32_t pos = s_block_excl[d[j]] + s_wcount[warp][d[j]] + rank[j];
            s_keys[pos] = k[j];
            s_vals[pos] = v[j];
        }
    }
    __syncthreads();
    const uint32_t n_here = p.count > base ? min(static_cast<uint32_t>(kSortTile), p.count - base) : 0u;
    for (uint32_t e = tid; e < n_here; e += kSortThreads) {
        const uint32_t key = s_keys[e];
        const uint32_t dd = (key >> p.shift) & mask;
        const uint32_t pos = s_global[dd] + (e - s_block_excl[dd]);
        p.keys_out[pos] = key;
        p.vals_out[pos] = s_vals[e];
    }
}

// Equal-depth runs of the sorted splats: order by ordinal (renderer.cpp:91-96).
__global__ void k_tie_fixup(const uint32_t* keys, uint32_t* vals, const uint32_t* ordinal, uint32_t count) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < count; i += gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        if (keys[i + 1] != k) continue;
        if (i > 0 && keys[i - 1] == k) continue;  // not the run start
        uint32_t end = i + 1;
        while (end < count && keys[end] == k) ++end;
        for (uint32_t a = i + 1; a < end; ++a) {
            const uint32_t va = vals[a];
            const uint32_t oa = ordinal[va];
            uint32_t b = a;
            while (b > i && ordinal[vals[b - 1]] > oa) {
                vals[b] = vals[b - 1];
                --b;
            }
            vals[b] = va;
        }
    }
}

// Cell spans gathered into sorted order + per-block pair sums (level 1 of the scan).
__global__ void __launch_bounds__(1024)
k_splat_cells(const uint32_t* sorted_rec, uint32_t count, const uint2* span, uint2* span_sorted,
              uint32_t* block_sums) {
    __shared__ uint32_t s_warp[32];
    const uint32_t i = blockIdx.x * 1024 + threadIdx.x;
    uint32_t n = 0;
    if (i < count) {
        const uint2 sp = span[sorted_rec[i]];
        span_sorted[i] = sp;
        n = (sp.y & 0xffffu) * (sp.y >> 16);
    }
    uint32_t total;
    block_excl_scan(n, s_warp, total);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// Exclusive scan of the block sums in place (one CTA).
__global__ void __launch_bounds__(1024) k_scan_sums(uint32_t* sums, uint32_t n) {
    __shared__ uint32_t s_warp[32];
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < n ? sums[i] : 0u;
        uint32_t total;
        const uint32_t e = block_excl_scan(v, s_warp, total);
        if (i < n) sums[i] = carry + e;
        carry += total;
    }
}

// Emit (cell, record) pairs in the sorted splat order.
__global__ void __launch_bounds__(1024)
k_emit_pairs(const uint32_t* sorted_rec, uint32_t count, const uint2* span_sorted, const uint32_t* block_offsets,
             int tiles_x, int quads, uint32_t* pair_cell, uint32_t* pair_rec) {
    __shared__ uint32_t s_warp[32];
    const uint32_t i = blockIdx.x * 1024 + threadIdx.x;
    const uint2 sp = i < count ? span_sorted[i] : make_uint2(0u, 0u);
    const int ncw = static_cast<int>(sp.y & 0xffffu);
    const uint32_t n = static_cast<uint32_t>(ncw) * (sp.y >> 16);
    uint32_t total;
    const uint32_t off = block_offsets[blockIdx.x] + block_excl_scan(n, s_warp, total);
    if (i >= count) return;
    const uint32_t rec = sorted_rec[i];
    const int cx0 = static_cast<int>(sp.x & 0xffffu), cy0 = static_cast<int>(sp.x >> 16);
    for (int k = 0; k < static_cast<int>(n); ++k) {
        const int cx = cx0 + k % ncw, cy = cy0 + k / ncw;
        pair_cell[off + k] = quads ? static_cast<uint32_t>(((cy >> 1) * tiles_x + (cx >> 1)) * 4 + (cy & 1) * 2 + (cx & 1))
                                   : static_cast<uint32_t>(cy * tiles_x + cx);
        pair_rec[off + k] = rec;
    }
}

// [start, end) of every cell in the cell-sorted pairs (the reference's bins).
__global__ void k_cell_ranges(const uint32_t* cells, uint32_t count, uint2* ranges) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const uint32_t c = cells[i];
        if (i == 0 || cells[i - 1] != c) ranges[c].x = i;
        if (i + 1 == count || cells[i + 1] != c) ranges[c].y = i + 1;
    }
}

__global__ void k_sorted_ordinals(const uint32_t* recs, const uint32_t* ordinal, uint32_t count, uint32_t* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        out[i] = ordinal[recs[i]];
}

}  // namespace gscg
