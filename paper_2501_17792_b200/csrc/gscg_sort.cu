// Stage "sort" on the B200: the reference's own two-step order — sort the splats by
// depth, then bin them into tiles in that order (sort_splats_impl renderer.cpp:85-107,
// binning renderer.cpp:143-161) — restated as three device passes:
//
//   1. LSD radix sort of the S splat depth keys (32-bit, only the bits that vary in the
//      frame), values = record index; k_tie_fixup orders equal-depth runs by splat
//      ordinal (instance base + gaussian index) = the reference's (instance, gaussian)
//      tie-break. The splats are now in the reference's total order.
//   2. k_splat_cells + k_scan_sums + k_emit_pairs: every sorted splat emits one pair per
//      overlapped binning cell (tile, or 8x8 quadrant of a 16-px tile), in sorted order.
//   3. stable LSD radix sort of the pairs' cell ids; k_cell_ranges marks each cell's
//      [start, end). Stability keeps the depth order inside every cell, so each cell
//      list is exactly the reference's bin restricted to the cell.
//
// Each LSD pass (digits of up to 5 bits; a b-bit key takes ceil(b/5) passes with the bits
// spread evenly) is reduce-then-scan: k_sort_upsweep counts digits per 4096-key tile,
// k_sort_rows / k_sort_bases turn the counts into global offsets, k_sort_downsweep ranks
// keys stably inside the tile with a register-only warp multisplit (ballots + shuffles,
// lane d keeps the warp's count of digit d), stages the tile in digit order and writes it
// out coalesced. 8-bit digits with shared-memory counters were measured no faster overall
// (fewer passes, but each ~1.6x slower). No tile waits on another: a decoupled look-back onesweep and
// 8-bit shared-atomic ranking were both measured slower here (serial look-back chains,
// ATOMS throughput).
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

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

// Upsweep: per-tile digit counts, written digit-major (counts[d * tiles + t]).
__global__ void __launch_bounds__(kSortThreads)
k_sort_upsweep(SortPassParams p) {
    __shared__ uint32_t s_hist[kSortWarps][kRadix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = blockIdx.x * kSortTile;
    const uint32_t mask = (1u << p.bits) - 1u;
    uint32_t k[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {  // all loads in flight first
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        k[j] = idx < p.count ? p.keys_in[idx] : 0u;
    }
    // Lane d counts digit d of the warp's keys: per item, five ballots select the lanes
    // holding digit d.
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const uint32_t d = (k[j] >> p.shift) & mask;
        uint32_t mine = __ballot_sync(0xffffffffu, idx < p.count);
#pragma unroll
        for (int b = 0; b < kRadixBits; ++b) {
            const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            mine &= ((lane >> b) & 1) ? bb : ~bb;
        }
        cnt += __popc(mine);
    }
    s_hist[warp][lane] = cnt;
    __syncthreads();
    if (threadIdx.x < kRadix) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) t += s_hist[w][threadIdx.x];
        p.counts[threadIdx.x * p.tiles + blockIdx.x] = t;
    }
}

// Row scans: CTA d turns digit d's tile counts into exclusive offsets; row total ->
// digit_base[d].
__global__ void __launch_bounds__(1024)
k_sort_rows(SortPassParams p) {
    __shared__ uint32_t s_warp[32];
    uint32_t* row = p.counts + static_cast<size_t>(blockIdx.x) * p.tiles;
    uint32_t carry = 0;
    for (uint32_t b = 0; b < p.tiles; b += 1024) {
        const uint32_t i = b + threadIdx.x;
        const uint32_t v = i < p.tiles ? row[i] : 0u;
        uint32_t total;
        const uint32_t e = block_excl_scan(v, s_warp, total);
        if (i < p.tiles) row[i] = carry + e;
        carry += total;
    }
    if (threadIdx.x == 0) p.digit_base[blockIdx.x] = carry;
}

// Exclusive scan of the kRadix digit totals (one warp).
__global__ void __launch_bounds__(32) k_sort_bases(SortPassParams p) {
    const uint32_t v = p.digit_base[threadIdx.x];
    p.digit_base[threadIdx.x] = warp_incl_scan(v, threadIdx.x) - v;
}

// Downsweep: stable rank inside the tile with a register-only warp multisplit (five
// ballots give each key the lanes sharing its digit; lane d keeps the warp's running
// count of digit d), stage the tile in shared memory in digit order, write it out
// coalesced at digit_base[d] + counts[d][tile] + rank-within-digit.
__global__ void __launch_bounds__(kSortThreads, 3)
k_sort_downsweep(SortPassParams p) {
    __shared__ uint32_t s_keys[kSortTile];
    __shared__ uint16_t s_perm[kSortTile];  // tile-local source index of each staged key
    __shared__ uint32_t s_woff[kSortWarps][kRadix];
    __shared__ uint32_t s_block_excl[kRadix];
    __shared__ uint32_t s_global[kRadix];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid < kRadix) s_global[tid] = p.digit_base[tid] + p.counts[tid * p.tiles + blockIdx.x];
    const uint32_t base = blockIdx.x * kSortTile;
    const uint32_t mask = (1u << p.bits) - 1u;
    const uint32_t lt = (1u << lane) - 1u;

    uint32_t k[kSortItems], rank[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        k[j] = idx < p.count ? p.keys_in[idx] : 0u;
    }
    uint32_t cnt = 0;  // lane d: keys of digit d so far in this warp's segment
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const uint32_t d = (k[j] >> p.shift) & mask;
        const uint32_t vm = __ballot_sync(0xffffffffu, idx < p.count);
        uint32_t peers = vm, mine = vm;
#pragma unroll
        for (int b = 0; b < kRadixBits; ++b) {
            const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bb : ~bb;
            mine &= ((lane >> b) & 1) ? bb : ~bb;
        }
        rank[j] = __shfl_sync(0xffffffffu, cnt, static_cast<int>(d)) + __popc(peers & lt);
        cnt += __popc(mine);
    }
    s_woff[warp][lane] = cnt;
    __syncthreads();
    if (tid < 32) {  // digit tid: exclusive over warps, then over digits
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = s_woff[w][tid];
            s_woff[w][tid] = run;
            run += c;
        }
        s_block_excl[tid] = warp_incl_scan(run, tid) - run;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t local = warp * (32 * kSortItems) + j * 32 + lane;
        if (base + local < p.count) {
            const uint32_t d = (k[j] >> p.shift) & mask;
            const uint32_t pos = s_block_excl[d] + s_woff[warp][d] + rank[j];
            s_keys[pos] = k[j];
            s_perm[pos] = static_cast<uint16_t>(local);
        }
    }
    __syncthreads();
    // Write-out: every gather of the thread issued before any store (the value gathers
    // stay inside this tile's 16 KB input window, so they hit L2).
    const uint32_t n_here = p.count > base ? min(kSortTile, p.count - base) : 0u;
    const uint32_t* __restrict__ vals_in = p.vals_in;
    uint32_t okey[kSortItems], opos[kSortItems], oval[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t e = tid + j * kSortThreads;
        if (e < n_here) {
            okey[j] = s_keys[e];
            const uint32_t dd = (okey[j] >> p.shift) & mask;
            opos[j] = s_global[dd] + (e - s_block_excl[dd]);
            const uint32_t src = base + s_perm[e];
            oval[j] = vals_in ? __ldg(vals_in + src) : src;
        }
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t e = tid + j * kSortThreads;
        if (e < n_here) {
            p.keys_out[opos[j]] = okey[j];
            p.vals_out[opos[j]] = oval[j];
        }
    }
}

// Equal-depth runs of the sorted splats: order by ordinal (renderer.cpp:91-96). Each
// thread scans kStreamItems positions and fixes the runs that start there (ties are
// common: far crowd depths share float bit patterns).
__global__ void __launch_bounds__(256)
k_tie_fixup(const uint32_t* keys, uint32_t* recs, const uint32_t* ordinal, uint32_t count) {
    static_assert(kStreamItems == 8, "two uint4 loads per thread");
    const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) * kStreamItems;
    if (b >= count) return;
    uint32_t s = b;  // first position left to the scalar path below
    if (b + kStreamItems < count) {
        uint32_t k[kStreamItems + 1];
        const uint4 lo = *reinterpret_cast<const uint4*>(keys + b);
        const uint4 hi = *reinterpret_cast<const uint4*>(keys + b + 4);
        k[0] = lo.x; k[1] = lo.y; k[2] = lo.z; k[3] = lo.w;
        k[4] = hi.x; k[5] = hi.y; k[6] = hi.z; k[7] = hi.w;
        k[8] = keys[b + kStreamItems];
        bool tie = false;
#pragma unroll
        for (int j = 0; j < kStreamItems; ++j) tie |= k[j] == k[j + 1];
        if (!tie) return;
        const uint32_t prev = b > 0 ? keys[b - 1] : ~0u;
        // [w0, w1): the runs that start and end inside the window, sorted in registers.
        // A run entering from the left belongs to the thread where it starts; a run
        // leaving on the right is finished by the scalar path from its start.
        int w0 = 0;
        if (b > 0 && k[0] == prev) {
            w0 = 1;
#pragma unroll
            for (int j = 1; j < kStreamItems; ++j)
                if (w0 == j && k[j] == k[j - 1]) w0 = j + 1;
        }
        int w1 = kStreamItems;
        if (k[kStreamItems - 1] == k[kStreamItems]) {
            w1 = kStreamItems - 1;
#pragma unroll
            for (int j = kStreamItems - 2; j >= 0; --j)
                if (w1 == j + 1 && k[j] == k[j + 1]) w1 = j;
            w1 = max(w1, w0);
        }
        uint32_t r[kStreamItems], o[kStreamItems];
        const uint4 rlo = *reinterpret_cast<const uint4*>(recs + b);
        const uint4 rhi = *reinterpret_cast<const uint4*>(recs + b + 4);
        r[0] = rlo.x; r[1] = rlo.y; r[2] = rlo.z; r[3] = rlo.w;
        r[4] = rhi.x; r[5] = rhi.y; r[6] = rhi.z; r[7] = rhi.w;
#pragma unroll
        for (int j = 0; j < kStreamItems; ++j) {
            const bool in = j >= w0 && j < w1;
            const bool tied = (j > 0 && k[j] == k[j - 1]) || k[j] == k[j + 1];
            o[j] = in && tied ? ordinal[r[j]] : 0u;  // independent gathers, all in flight
        }
        // Odd-even transposition: equal keys are contiguous, so only runs reorder.
        bool moved = false;
#pragma unroll
        for (int round = 0; round < kStreamItems; ++round) {
#pragma unroll
            for (int j = round & 1; j + 1 < kStreamItems; j += 2) {
                if (j >= w0 && j + 1 < w1 && k[j] == k[j + 1] && o[j] > o[j + 1]) {
                    const uint32_t t0 = o[j]; o[j] = o[j + 1]; o[j + 1] = t0;
                    const uint32_t t1 = r[j]; r[j] = r[j + 1]; r[j + 1] = t1;
                    moved = true;
                }
            }
        }
        if (moved) {
            // Only [w0, w1) is this thread's: the runs crossing the window edges are being
            // reordered by the threads where they start.
#pragma unroll
            for (int j = 0; j < kStreamItems; ++j)
                if (j >= w0 && j < w1) recs[b + j] = r[j];
        }
        if (w1 == kStreamItems) return;
        s = b + static_cast<uint32_t>(w1);  // start of the run leaving the window
    }
    // Scalar path: the window tail of the last thread, and runs that leave a window.
    const uint32_t e = min(count, b + kStreamItems);
    uint32_t prev = s > 0 ? keys[s - 1] : ~0u;
    for (uint32_t i = s; i < e; ++i) {
        const uint32_t k = keys[i];
        if ((i == 0 || k != prev) && i + 1 < count && keys[i + 1] == k) {
            uint32_t end = i + 1;
            while (end < count && keys[end] == k) ++end;
            for (uint32_t a = i + 1; a < end; ++a) {
                const uint32_t ra = recs[a];
                const uint32_t oa = ordinal[ra];
                uint32_t j = a;
                while (j > i && ordinal[recs[j - 1]] > oa) {
                    recs[j] = recs[j - 1];
                    --j;
                }
                recs[j] = ra;
            }
        }
        prev = k;
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

// Emit (cell, record) pairs in sorted splat order. Warp-cooperative: the warp's pairs are
// numbered 0..total-1 and lane L writes pairs L, L+32, ... (coalesced), finding each
// pair's splat by a 5-step search over the warp's exclusive prefix.
__global__ void __launch_bounds__(1024)
k_emit_pairs(const uint32_t* rec_sorted, uint32_t count, const uint2* span_sorted, const uint32_t* block_offsets,
             int tiles_x, int quads, uint32_t* pair_cell, uint32_t* pair_rec) {
    __shared__ uint32_t s_warp[32];
    const int lane = threadIdx.x & 31;
    const uint32_t i = blockIdx.x * 1024 + threadIdx.x;
    const uint2 sp = i < count ? span_sorted[i] : make_uint2(0u, 0u);
    const uint32_t rec = i < count ? rec_sorted[i] : 0u;
    const uint32_t n = (sp.y & 0xffffu) * (sp.y >> 16);
    uint32_t total;
    const uint32_t off = block_offsets[blockIdx.x] + block_excl_scan(n, s_warp, total);
    uint32_t incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - n;
    const uint32_t warp_total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t warp_base = __shfl_sync(0xffffffffu, off, 0);
    for (uint32_t t0 = 0; t0 < warp_total; t0 += 32) {
        const uint32_t t = t0 + lane;
        // owner: the last lane whose exclusive prefix is <= t
        int owner = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t e = __shfl_sync(0xffffffffu, excl, owner + step);
            if (owner + step < 32 && e <= t) owner += step;
        }
        const uint32_t e_own = __shfl_sync(0xffffffffu, excl, owner);
        const uint2 s2 = make_uint2(__shfl_sync(0xffffffffu, sp.x, owner), __shfl_sync(0xffffffffu, sp.y, owner));
        const uint32_t r = __shfl_sync(0xffffffffu, rec, owner);
        if (t < warp_total) {
            const int k = static_cast<int>(t - e_own);
            const int ncw = static_cast<int>(s2.y & 0xffffu);
            const int cx = static_cast<int>(s2.x & 0xffffu) + k % ncw, cy = static_cast<int>(s2.x >> 16) + k / ncw;
            pair_cell[warp_base + t] = quads ? static_cast<uint32_t>(((cy >> 1) * tiles_x + (cx >> 1)) * 4 + (cy & 1) * 2 + (cx & 1))
                                             : static_cast<uint32_t>(cy * tiles_x + cx);
            pair_rec[warp_base + t] = r;
        }
    }
}

// [start, end) of every cell in the cell-sorted pairs (the reference's bins).
__global__ void __launch_bounds__(256)
k_cell_ranges(const uint32_t* cells, uint32_t count, uint2* ranges) {
    const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) * kStreamItems;
    if (b >= count) return;
    const uint32_t e = min(count, b + kStreamItems);
    uint32_t prev = b > 0 ? cells[b - 1] : ~0u;
    for (uint32_t i = b; i < e; ++i) {
        const uint32_t c = cells[i];
        if (c != prev) {
            ranges[c].x = i;
            if (i > 0) ranges[prev].y = i;
        }
        prev = c;
    }
    if (e == count) ranges[prev].y = count;
}

__global__ void k_sorted_ordinals(const uint32_t* recs, const uint32_t* ordinal, uint32_t count, uint32_t* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        out[i] = ordinal[recs[i]];
}

}  // namespace gscg
