// Stage "sort" on the B200: the reference's own two-step order — sort the splats by
// depth, then bin them into tiles in that order (sort_splats_impl renderer.cpp:85-107,
// binning renderer.cpp:143-161) — restated as three device passes:
//
//   1. LSD radix sort of the S splat depth keys (32-bit, only the bits that vary in the
//      frame), values = record index; k_sorted_spans orders equal-depth runs by splat
//      ordinal (instance base + gaussian index) = the reference's (instance, gaussian)
//      tie-break. The splats are now in the reference's total order.
//   2. k_sorted_spans + k_scan_sums + k_emit_pairs: every sorted splat emits one pair per
//      overlapped binning cell (tile, or 8x8 quadrant of a 16-px tile), in sorted order.
//   3. stable LSD radix sort of the pairs' cell ids; k_cell_ranges marks each cell's
//      [start, end). Stability keeps the depth order inside every cell, so each cell
//      list is exactly the reference's bin restricted to the cell.
//
// Each LSD pass (digits of up to 5 bits; a b-bit key takes ceil(b/5) passes with the bits
// spread evenly) is reduce-then-scan: k_sort_upsweep counts digits per 4096-key tile,
// k_sort_rows turns the counts into per-tile offsets and digit totals, k_sort_downsweep ranks
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
    uint32_t lane_mask[kRadixBits];  // all-ones where lane's bit b is set
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) lane_mask[b] = 0u - ((static_cast<uint32_t>(lane) >> b) & 1u);
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const uint32_t d = (k[j] >> p.shift) & mask;
        // Lanes whose digit differs from lane's index in some bit: OR of (ballot ^ lane mask).
        uint32_t differ = 0u;
#pragma unroll
        for (int b = 0; b < kRadixBits; ++b) differ |= __ballot_sync(0xffffffffu, (d >> b) & 1u) ^ lane_mask[b];
        cnt += __popc(__ballot_sync(0xffffffffu, idx < p.count) & ~differ);
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
// digit_base[d] (the downsweep scans the row totals itself). Each thread owns up to
// kRowItems consecutive entries of a 1024 * kRowItems window, so a row of up to 8192 tiles
// takes one block scan.
constexpr int kRowItems = 8;
__global__ void __launch_bounds__(1024)
k_sort_rows(SortPassParams p) {
    __shared__ uint32_t s_warp[32];
    uint32_t* row = p.counts + static_cast<size_t>(blockIdx.x) * p.tiles;
    uint32_t carry = 0;
    for (uint32_t b = 0; b < p.tiles; b += 1024 * kRowItems) {
        const uint32_t i0 = b + threadIdx.x * kRowItems;
        uint32_t v[kRowItems], sum = 0;
#pragma unroll
        for (int k = 0; k < kRowItems; ++k) {
            v[k] = i0 + k < p.tiles ? row[i0 + k] : 0u;
            sum += v[k];
        }
        uint32_t total;
        uint32_t run = carry + block_excl_scan(sum, s_warp, total);
#pragma unroll
        for (int k = 0; k < kRowItems; ++k) {
            if (i0 + k < p.tiles) row[i0 + k] = run;
            run += v[k];
        }
        carry += total;
    }
    if (threadIdx.x == 0) p.digit_base[blockIdx.x] = carry;
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
    const uint32_t mask = (1u << p.bits) - 1u;
    if (tid < kRadix) {  // global digit base (exclusive scan of the row totals) + this tile's offset
        const uint32_t total = static_cast<uint32_t>(tid) <= mask ? p.digit_base[tid] : 0u;
        s_global[tid] = warp_incl_scan(total, lane) - total + p.counts[tid * p.tiles + blockIdx.x];
    }
    const uint32_t base = blockIdx.x * kSortTile;
    const uint32_t lt = (1u << lane) - 1u;

    uint32_t k[kSortItems], rank[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        k[j] = idx < p.count ? p.keys_in[idx] : 0u;
    }
    uint32_t lane_mask[kRadixBits];  // all-ones where lane's bit b is set
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) lane_mask[b] = 0u - ((static_cast<uint32_t>(lane) >> b) & 1u);
    uint32_t cnt = 0;  // lane d: keys of digit d so far in this warp's segment
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const uint32_t d = (k[j] >> p.shift) & mask;
        const uint32_t vm = __ballot_sync(0xffffffffu, idx < p.count);
        uint32_t peers_differ = 0u, mine_differ = 0u;
#pragma unroll
        for (int b = 0; b < kRadixBits; ++b) {
            const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers_differ |= bb ^ (0u - ((d >> b) & 1u));
            mine_differ |= bb ^ lane_mask[b];
        }
        rank[j] = __shfl_sync(0xffffffffu, cnt, static_cast<int>(d)) + __popc(vm & ~peers_differ & lt);
        cnt += __popc(vm & ~mine_differ);
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

namespace {

__device__ __forceinline__ uint32_t cell_id(int cx, int cy, int tiles_x, int quads) {
    return quads ? static_cast<uint32_t>(((cy >> 1) * tiles_x + (cx >> 1)) * 4 + (cy & 1) * 2 + (cx & 1))
                 : static_cast<uint32_t>(cy * tiles_x + cx);
}

// Calls f(cell) for every binning cell of a packed span, row by row (the emission order);
// along a row the cell id advances without recomputing it (quadrant cells: +1 inside a
// tile, +3 into the next tile).
template <typename F>
__device__ __forceinline__ void for_each_cell(uint2 sp, int tiles_x, int quads, F&& f) {
    const int cx0 = static_cast<int>(sp.x & 0xffffu), cy0 = static_cast<int>(sp.x >> 16);
    const int w = static_cast<int>(sp.y & 0xffffu), h = static_cast<int>(sp.y >> 16);
    for (int cy = cy0; cy < cy0 + h; ++cy) {
        uint32_t c = cell_id(cx0, cy, tiles_x, quads);
        for (int cx = cx0; cx < cx0 + w; ++cx) {
            f(c);
            c += quads ? ((cx & 1) ? 3u : 1u) : 1u;
        }
    }
}

}  // namespace

// After the depth sort: every sorted splat's binning span, gathered into sorted order
// (one 16-byte meta gather per splat, all eight of a thread in flight).
__global__ void __launch_bounds__(kMetaThreads)
k_sorted_spans(const uint32_t* recs, const uint4* meta, uint32_t count, uint2* span_sorted) {
    static_assert(kStreamItems == 8, "two uint4 loads per thread");
    const uint32_t b = (blockIdx.x * kMetaThreads + threadIdx.x) * kStreamItems;
    if (b + kStreamItems <= count) {
        const uint4 rlo = *reinterpret_cast<const uint4*>(recs + b);
        const uint4 rhi = *reinterpret_cast<const uint4*>(recs + b + 4);
        const uint32_t r[kStreamItems] = {rlo.x, rlo.y, rlo.z, rlo.w, rhi.x, rhi.y, rhi.z, rhi.w};
        uint4 m[kStreamItems];
#pragma unroll
        for (int j = 0; j < kStreamItems; ++j) m[j] = meta[r[j]];
        uint4* dst = reinterpret_cast<uint4*>(span_sorted + b);
#pragma unroll
        for (int j = 0; j < kStreamItems; j += 2) dst[j / 2] = make_uint4(m[j].y, m[j].z, m[j + 1].y, m[j + 1].z);
    } else {
        for (uint32_t i = b; i < count; ++i) {
            const uint4 m = meta[recs[i]];
            span_sorted[i] = make_uint2(m.y, m.z);
        }
    }
}

// Per-cell order fix-up and cell ranges, over the cell-sorted pairs.
//
// The depth sort orders splats by the top bits of their depth keys only (at most 20
// varying bits: 4 LSD passes); splats whose truncated keys tie keep an arbitrary order.
// Emission tags every pair's key word with the low bits of its splat's truncated key above
// the cell id, and the stable cell passes keep the truncated-depth order inside every
// cell. Inside a cell, a run of equal key words (same cell, same tag) holds pairs of equal
// truncated depth, or, when tags alias, of increasing truncated depth; sorting every such
// run by the full (depth bits, ordinal) key (renderer.cpp:85-107) therefore yields exactly
// the reference's bin order. Runs are short (a few pairs; ties inside one 8x8 cell), so a
// thread orders the runs inside its 8-pair window in registers (odd-even transposition),
// finishes a run leaving its window in global memory, and hands runs longer than kLongRun
// to k_pair_long_runs. Pairs outside runs are never gathered.
namespace {

__device__ __forceinline__ unsigned long long pair_order_key(const uint4& m) {  // (depth bits, ordinal)
    return (static_cast<unsigned long long>(m.w) << 32) | m.x;
}

// Orders the run of equal key words starting at s (insertion sort in global memory).
__device__ void finish_pair_run(const uint32_t* keys, uint32_t* recs, const uint4* meta, uint32_t count, uint32_t s,
                                uint2* long_runs, uint32_t* long_count, uint32_t long_cap) {
    const uint32_t k = keys[s];
    uint32_t end = s + 1;
    while (end < count && keys[end] == k) ++end;
    if (end - s > kLongRun) {
        const uint32_t slot = atomicAdd(long_count, 1u);
        if (slot < long_cap) {
            long_runs[slot] = make_uint2(s, end - s);
            return;
        }
    }
    for (uint32_t a = s + 1; a < end; ++a) {
        const uint32_t ra = recs[a];
        const unsigned long long oa = pair_order_key(meta[ra]);
        uint32_t j = a;
        while (j > s && pair_order_key(meta[recs[j - 1]]) > oa) {
            recs[j] = recs[j - 1];
            --j;
        }
        recs[j] = ra;
    }
}

}  // namespace

__global__ void __launch_bounds__(256)
k_cell_fixup(const uint32_t* keys, uint32_t* recs, const uint4* meta, uint32_t count, uint32_t cell_mask, int fix,
             uint2* ranges, uint2* long_runs, uint32_t* long_count, uint32_t long_cap) {
    static_assert(kStreamItems == 8, "two uint4 loads per thread");
    const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) * kStreamItems;
    if (b >= count) return;
    const uint32_t prev_key = b > 0 ? keys[b - 1] : 0u;
    if (b + kStreamItems <= count) {
        const uint4 lo = *reinterpret_cast<const uint4*>(keys + b);
        const uint4 hi = *reinterpret_cast<const uint4*>(keys + b + 4);
        const uint32_t k[kStreamItems] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        const bool has_next = b + kStreamItems < count;
        const uint32_t next_key = has_next ? keys[b + kStreamItems] : 0u;
        // Cell ranges (the reference's bins).
        uint32_t pc = b > 0 ? (prev_key & cell_mask) : ~0u;
#pragma unroll
        for (int j = 0; j < kStreamItems; ++j) {
            const uint32_t c = k[j] & cell_mask;
            if (c != pc) {
                ranges[c].x = b + j;
                if (b + j > 0) ranges[pc].y = b + j;
            }
            pc = c;
        }
        if (!has_next) ranges[pc].y = count;
        if (!fix) return;
        // [w0, w1): positions whose runs start and end inside the window.
        int w0 = 0;
        if (b > 0 && k[0] == prev_key) {
            w0 = 1;
#pragma unroll
            for (int j = 1; j < kStreamItems; ++j)
                if (w0 == j && k[j] == k[j - 1]) w0 = j + 1;
        }
        int w1 = kStreamItems;
        if (has_next && k[kStreamItems - 1] == next_key) {
            w1 = kStreamItems - 1;
#pragma unroll
            for (int j = kStreamItems - 2; j >= 0; --j)
                if (w1 == j + 1 && k[j] == k[j + 1]) w1 = j;
            w1 = max(w1, w0);
        }
        bool tie[kStreamItems];
        bool any = false;
#pragma unroll
        for (int j = 0; j < kStreamItems; ++j) {
            const bool l = j > 0 && k[j] == k[j - 1];
            const bool r = j + 1 < kStreamItems && k[j] == k[j + 1];
            tie[j] = j >= w0 && j < w1 && ((l && j - 1 >= w0) || (r && j + 1 < w1));
            any |= tie[j];
        }
        if (any) {
            const uint4 rlo = *reinterpret_cast<const uint4*>(recs + b);
            const uint4 rhi = *reinterpret_cast<const uint4*>(recs + b + 4);
            uint32_t r[kStreamItems] = {rlo.x, rlo.y, rlo.z, rlo.w, rhi.x, rhi.y, rhi.z, rhi.w};
            unsigned long long o[kStreamItems];
#pragma unroll
            for (int j = 0; j < kStreamItems; ++j) o[j] = tie[j] ? pair_order_key(meta[r[j]]) : 0ull;
            bool moved = false;
#pragma unroll
            for (int round = 0; round < kStreamItems; ++round) {
#pragma unroll
                for (int j = round & 1; j + 1 < kStreamItems; j += 2) {
                    if (tie[j] && tie[j + 1] && k[j] == k[j + 1] && o[j] > o[j + 1]) {
                        const unsigned long long to = o[j]; o[j] = o[j + 1]; o[j + 1] = to;
                        const uint32_t tr = r[j]; r[j] = r[j + 1]; r[j + 1] = tr;
                        moved = true;
                    }
                }
            }
            if (moved) {
#pragma unroll
                for (int j = 0; j < kStreamItems; ++j)
                    if (tie[j]) recs[b + j] = r[j];
            }
        }
        if (w1 < kStreamItems) finish_pair_run(keys, recs, meta, count, b + static_cast<uint32_t>(w1), long_runs, long_count, long_cap);
        return;
    }
    // Last window: positions one by one.
    uint32_t pc = b > 0 ? (prev_key & cell_mask) : ~0u;
    for (uint32_t i = b; i < count; ++i) {
        const uint32_t c = keys[i] & cell_mask;
        if (c != pc) {
            ranges[c].x = i;
            if (i > 0) ranges[pc].y = i;
        }
        pc = c;
    }
    ranges[pc].y = count;
    if (!fix) return;
    uint32_t i = b;
    if (b > 0)
        while (i < count && keys[i] == prev_key) ++i;  // a run entering from the left
    while (i < count) {
        if (i + 1 < count && keys[i + 1] == keys[i]) {
            finish_pair_run(keys, recs, meta, count, i, long_runs, long_count, long_cap);
            const uint32_t k = keys[i];
            while (i < count && keys[i] == k) ++i;
        } else {
            ++i;
        }
    }
}

// Runs of more than kLongRun equal key words recorded by k_cell_fixup (many pairs of one
// truncated depth in one cell, e.g. characters stacked on one spot): one CTA per run sorts
// ((depth bits, ordinal), record) in shared memory (bitonic, up to kPairRunCap); longer
// runs are sorted in place in global memory.
__global__ void __launch_bounds__(256)
k_pair_long_runs(uint32_t* recs, const uint4* meta, const uint2* long_runs, const uint32_t* long_count, uint32_t long_cap) {
    __shared__ unsigned long long s_key[kPairRunCap];
    __shared__ uint32_t s_rec[kPairRunCap];
    const uint32_t runs = min(*long_count, long_cap);
    for (uint32_t q = blockIdx.x; q < runs; q += gridDim.x) {
        const uint2 run = long_runs[q];
        const uint32_t s = run.x, n = run.y;
        uint32_t P = 1;
        while (P < n) P <<= 1;
        if (n <= kPairRunCap) {
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                unsigned long long key = ~0ull;
                uint32_t rec = 0u;
                if (i < n) {
                    rec = recs[s + i];
                    key = pair_order_key(meta[rec]);
                }
                s_key[i] = key;
                s_rec[i] = rec;
            }
            __syncthreads();
            for (uint32_t k = 2; k <= P; k <<= 1) {
                for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                        const uint32_t l = i ^ j;
                        if (l > i) {
                            const unsigned long long a = s_key[i], c = s_key[l];
                            if ((a > c) == ((i & k) == 0)) {
                                s_key[i] = c;
                                s_key[l] = a;
                                const uint32_t t = s_rec[i]; s_rec[i] = s_rec[l]; s_rec[l] = t;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) recs[s + i] = s_rec[i];
            __syncthreads();
        } else {
            // All-ascending bitonic in place (each merge opens with the mirror comparison),
            // so positions >= n act as +inf and are skipped. Keys are unique per pair.
            uint32_t* r = recs + s;
            for (uint32_t k = 2; k <= P; k <<= 1) {
                for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                    for (uint32_t t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
                        const uint32_t blk = t / j, off = t % j;
                        uint32_t i, l;
                        if (j == (k >> 1)) {
                            i = blk * k + off;
                            l = blk * k + k - 1u - off;
                        } else {
                            i = blk * 2u * j + off;
                            l = i + j;
                        }
                        if (l < n) {
                            const uint32_t ra = r[i], rb = r[l];
                            if (pair_order_key(meta[ra]) > pair_order_key(meta[rb])) {
                                r[i] = rb;
                                r[l] = ra;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
        }
    }
}

// Emit the (cell, record) pairs of every sorted splat directly in the order of the first
// stable cell-sort pass (LSD digit = cell & dmask): a pair's position is the digit's
// global base + this block's offset for the digit (k_sort_rows over k_sorted_spans'
// block histograms) + the pairs of that digit from earlier threads of the block + its
// rank among this thread's pairs of the digit. Threads own 4 consecutive sorted splats and
// enumerate each splat's cells row by row, so pairs of one digit keep the splat order: the
// output equals emitting in sorted order and running the first LSD pass on it.
// kCount: only count the block's pairs per digit (block_digit[d][block], the input of
// k_sort_rows); else scatter them.
template <bool kCount>
__global__ void __launch_bounds__(kEmitThreads)
k_emit_scatter(const uint32_t* rec_sorted, const uint32_t* key_sorted, uint32_t count, const uint2* span_sorted,
               uint32_t* block_digit, const uint32_t* digit_total, uint32_t blocks, int tiles_x, int quads,
               uint32_t dmask, uint32_t tag_drop, uint32_t tag_shift, uint32_t* pair_cell, uint32_t* pair_rec) {
    constexpr int kWarps = kEmitThreads / 32, kDigitsPerWarp = kRadix / kWarps, kPerLane = kEmitThreads / 32;
    static_assert(kRadix % kWarps == 0, "digits split evenly over the warps");
    constexpr uint32_t kStage = kEmitStage;            // pairs staged for coalesced writes
    extern __shared__ uint32_t s_dyn_emit[];
    auto s_cnt = reinterpret_cast<uint32_t (*)[kEmitThreads]>(s_dyn_emit);  // [digit][thread]: count, then start
    uint32_t* s_stage_cell = s_dyn_emit + kRadix * kEmitThreads;
    uint32_t* s_stage_rec = s_stage_cell + kStage;
    __shared__ uint32_t s_base[kRadix];   // global position of the block's first pair of each digit
    __shared__ uint32_t s_local[kRadix];  // block-local start of each digit
    __shared__ uint32_t s_total;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t i0 = blockIdx.x * kEmitSplats + 4u * tid;
    uint2 sp[4];
    uint32_t rc[4], tg[4] = {0u, 0u, 0u, 0u};
    if (i0 + 4 <= count) {
        const uint4 a = *reinterpret_cast<const uint4*>(span_sorted + i0);
        const uint4 b = *reinterpret_cast<const uint4*>(span_sorted + i0 + 2);
        const uint4 r = *reinterpret_cast<const uint4*>(rec_sorted + i0);
        sp[0] = make_uint2(a.x, a.y); sp[1] = make_uint2(a.z, a.w);
        sp[2] = make_uint2(b.x, b.y); sp[3] = make_uint2(b.z, b.w);
        rc[0] = r.x; rc[1] = r.y; rc[2] = r.z; rc[3] = r.w;
        if (!kCount && key_sorted) {
            const uint4 t = *reinterpret_cast<const uint4*>(key_sorted + i0);
            tg[0] = t.x; tg[1] = t.y; tg[2] = t.z; tg[3] = t.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            sp[q] = i0 + q < count ? span_sorted[i0 + q] : make_uint2(0u, 0u);
            rc[q] = i0 + q < count ? rec_sorted[i0 + q] : 0u;
            if (!kCount && key_sorted) tg[q] = i0 + q < count ? key_sorted[i0 + q] : 0u;
        }
    }
    // Tag above the cell id: the low bits of the splat's truncated depth key (k_cell_fixup).
#pragma unroll
    for (int q = 0; q < 4; ++q) tg[q] = key_sorted && tag_shift < 32 ? (tg[q] >> tag_drop) << tag_shift : 0u;
#pragma unroll
    for (int d = 0; d < kRadix; ++d) s_cnt[d][tid] = 0u;
    if (!kCount && tid < kRadix) {  // global base of digit tid: scanned digit totals + this block's offset
        const uint32_t t = static_cast<uint32_t>(tid) <= dmask ? digit_total[tid] : 0u;
        s_base[tid] = warp_incl_scan(t, lane) - t + (static_cast<uint32_t>(tid) <= dmask ? block_digit[tid * blocks + blockIdx.x] : 0u);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) for_each_cell(sp[q], tiles_x, quads, [&](uint32_t c) { ++s_cnt[c & dmask][tid]; });
    __syncthreads();
    if (kCount) {  // digit d's pairs in this block: warp w sums its digits over all threads
#pragma unroll
        for (int dd = 0; dd < kDigitsPerWarp; ++dd) {
            const int d = warp * kDigitsPerWarp + dd;
            uint32_t v = 0;
#pragma unroll
            for (int k = 0; k < kPerLane; ++k) v += s_cnt[d][lane * kPerLane + k];
            v = __reduce_add_sync(0xffffffffu, v);
            if (lane == 0 && static_cast<uint32_t>(d) <= dmask) block_digit[d * blocks + blockIdx.x] = v;
        }
        return;
    }
    // Exclusive scan over threads for each digit (warp w: kDigitsPerWarp digits, lane l:
    // kPerLane consecutive threads), then over digits: s_cnt becomes each thread's start.
#pragma unroll
    for (int dd = 0; dd < kDigitsPerWarp; ++dd) {
        const int d = warp * kDigitsPerWarp + dd;
        uint32_t v[kPerLane], sum = 0;
#pragma unroll
        for (int k = 0; k < kPerLane; ++k) {
            v[k] = s_cnt[d][lane * kPerLane + k];
            sum += v[k];
        }
        const uint32_t incl = warp_incl_scan(sum, lane);
        uint32_t run = incl - sum;
#pragma unroll
        for (int k = 0; k < kPerLane; ++k) {
            s_cnt[d][lane * kPerLane + k] = run;
            run += v[k];
        }
        if (lane == 31) s_local[d] = incl;  // digit total for now
    }
    __syncthreads();
    if (tid < kRadix) {
        const uint32_t t = s_local[tid];
        const uint32_t incl = warp_incl_scan(t, lane);
        s_local[tid] = incl - t;
        if (tid == kRadix - 1) s_total = incl;
    }
    __syncthreads();
    const uint32_t total = s_total;
    const bool staged = total <= kStage;  // else every pair goes straight to its global slot
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t rec = rc[q], tag = tg[q];
        for_each_cell(sp[q], tiles_x, quads, [&](uint32_t c) {
            const uint32_t d = c & dmask;
            const uint32_t r = s_cnt[d][tid]++;  // rank among the block's pairs of digit d
            if (staged) {
                s_stage_cell[s_local[d] + r] = c | tag;
                s_stage_rec[s_local[d] + r] = rec;
            } else {
                pair_cell[s_base[d] + r] = c | tag;
                pair_rec[s_base[d] + r] = rec;
            }
        });
    }
    if (!staged) return;
    __syncthreads();
    // Staged pairs are in digit order: each digit's run goes to consecutive global slots.
    for (uint32_t e = tid; e < total; e += kEmitThreads) {
        const uint32_t c = s_stage_cell[e];
        const uint32_t d = c & dmask;
        const uint32_t pos = s_base[d] + (e - s_local[d]);
        pair_cell[pos] = c;
        pair_rec[pos] = s_stage_rec[e];
    }
}

void launch_emit(bool count_only, uint32_t blocks, cudaStream_t s, const uint32_t* rec_sorted, const uint32_t* key_sorted,
                 uint32_t count, const uint2* span_sorted, uint32_t* block_digit, const uint32_t* digit_total,
                 int tiles_x, int quads, uint32_t dmask, uint32_t tag_drop, uint32_t tag_shift, uint32_t* pair_cell,
                 uint32_t* pair_rec) {
    static bool attr = [] {
        cudaFuncSetAttribute(k_emit_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmem);
        cudaFuncSetAttribute(k_emit_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmem);
        return true;
    }();
    (void)attr;
    if (count_only)
        k_emit_scatter<true><<<blocks, kEmitThreads, kRadix * kEmitThreads * 4, s>>>(rec_sorted, key_sorted, count, span_sorted, block_digit,
                                                                    digit_total, blocks, tiles_x, quads, dmask,
                                                                    tag_drop, tag_shift, pair_cell, pair_rec);
    else
        k_emit_scatter<false><<<blocks, kEmitThreads, kEmitSmem, s>>>(rec_sorted, key_sorted, count, span_sorted, block_digit,
                                                                     digit_total, blocks, tiles_x, quads, dmask,
                                                                     tag_drop, tag_shift, pair_cell, pair_rec);
}

__global__ void k_iota2(uint32_t* a, uint32_t* b, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = b[i] = i;
}

__global__ void k_gather_u32(const uint32_t* src, const uint32_t* idx, uint32_t* dst, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[idx[i]];
}

__global__ void k_sorted_ordinals(const uint32_t* recs, const uint4* meta, uint32_t count, uint32_t* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        out[i] = meta[recs[i]].x;
}

}  // namespace gscg
