// Stage "sort" on the B200: the reference's own two-step order — sort the splats by
// depth, then bin them into tiles in that order (sort_splats_impl renderer.cpp:85-107,
// binning renderer.cpp:143-161) — restated as four device steps:
//
//   1. LSD radix sort of the S splat depth keys over their top (at most 25) varying bits,
//      values = record index.
//   2. k_sorted_spans gathers the spans in sorted order; k_emit_scatter (count: per-block
//      digit counts; k_sort_rows; scatter): every sorted splat emits one pair per
//      overlapped binning cell (tile, or 8x8 quadrant of a 16-px tile) straight into the
//      order of the first stable cell pass; each pair's key word carries its splat's
//      truncated depth above the cell id.
//   3. the remaining stable LSD passes over the cell bits.
//   4. k_cell_fixup: cell ranges, and every run of pairs with equal (cell, truncated
//      depth) ordered by (depth bits, ordinal) — the dropped low bits and the reference's
//      (instance, gaussian) tie-break (ordinal = instance base + gaussian index). Each
//      cell list is then exactly the reference's bin restricted to the cell.
//
// Each LSD pass (digits of up to 5 bits, or 7 in the wide passes a plan takes where they
// save a pass) is reduce-then-scan: k_sort_upsweep counts digits per 4096-key tile,
// k_sort_rows turns the counts into per-tile offsets and digit totals, k_sort_downsweep
// ranks keys stably inside the tile with a register-only warp multisplit (ballots +
// shuffles, lane d keeps the warp's count of digit d), stages the tile in digit order and
// writes it out coalesced. No tile waits on another: a decoupled look-back onesweep and
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

// Upsweep: per-tile digit counts, written digit-major (p.counts[d * tiles + t]). kFull: the
// tile holds kSortTile keys (every tile but the last), so no bounds predicates.
template <bool kFull>
__device__ __forceinline__ void upsweep_tile(const SortPassParams& p, uint32_t (*s_hist)[kRadix][32], uint32_t count) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = blockIdx.x * kSortTile;
    const uint32_t mask = (1u << p.bits) - 1u;
    uint32_t k[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {  // all loads in flight first
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        k[j] = (kFull || idx < count) ? p.keys_in[idx] : 0u;
    }
    // Lane-private digit counters s_hist[warp][d][lane] (lane L's column sits in bank L:
    // no conflicts), then lane d sums row d along a rotated walk (conflict-free too).
    uint32_t(*h)[32] = s_hist[warp];
#pragma unroll
    for (int d = 0; d < kRadix; ++d) h[d][lane] = 0u;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        if (kFull || idx < count) ++h[(k[j] >> p.shift) & mask][lane];
    }
    __syncwarp();
    uint32_t cnt = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) cnt += h[lane][(c + lane) & 31];
    __syncwarp();
    h[0][lane] = cnt;  // warp's count of digit `lane`
    __syncthreads();
    if (threadIdx.x < kRadix) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) t += s_hist[w][0][threadIdx.x];
        p.counts[threadIdx.x * p.tiles + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kSortThreads)
k_sort_upsweep(SortPassParams p) {
    pdl_entry();
    __shared__ uint32_t s_hist[kSortWarps][kRadix][32];
    // count: the host's, or the device counter clamped to it (deferred frames); only the
    // partial (last) tile needs it, so the full-tile path keeps its registers.
    const uint32_t count = resolve_count(p.count, p.count_dev);
    if (blockIdx.x * kSortTile >= count) {  // past the device count (deferred frames): zero counts only
        if (threadIdx.x < kRadix) p.counts[threadIdx.x * p.tiles + blockIdx.x] = 0u;
        return;
    }
    if ((blockIdx.x + 1) * kSortTile <= count) upsweep_tile<true>(p, s_hist, kSortTile);
    else upsweep_tile<false>(p, s_hist, count);
}

// Row scans: CTA d turns digit d's tile counts into exclusive offsets; row total ->
// digit_base[d] (the downsweep scans the row totals itself). A 1024 * kRowItems window per
// step: warp w owns kRowItems lane-contiguous chunks of 32 entries (coalesced loads and
// stores), warp totals are scanned across the CTA, then each chunk with a warp scan.
constexpr int kRowItems = 8;
__global__ void __launch_bounds__(1024)
k_sort_rows(SortPassParams p) {
    pdl_entry();
    __shared__ uint32_t s_warp[32];
    uint32_t* row = p.counts + static_cast<size_t>(blockIdx.x) * p.tiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t carry = 0;
    for (uint32_t b = 0; b < p.tiles; b += 1024 * kRowItems) {
        const uint32_t w0 = b + static_cast<uint32_t>(warp) * (32 * kRowItems) + lane;
        uint32_t v[kRowItems], sum = 0;
#pragma unroll
        for (int k = 0; k < kRowItems; ++k) {
            const uint32_t i = w0 + 32 * k;
            v[k] = i < p.tiles ? row[i] : 0u;
            sum += v[k];
        }
        sum = __reduce_add_sync(0xffffffffu, sum);  // the warp's window total
        uint32_t total;
        const uint32_t before = block_excl_scan(lane == 0 ? sum : 0u, s_warp, total);  // lane 0: earlier warps
        uint32_t run = carry + __shfl_sync(0xffffffffu, before, 0);
#pragma unroll
        for (int k = 0; k < kRowItems; ++k) {
            const uint32_t incl = warp_incl_scan(v[k], lane);
            const uint32_t i = w0 + 32 * k;
            if (i < p.tiles) row[i] = run + incl - v[k];
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        carry += total;
    }
    if (threadIdx.x == 0) p.digit_base[blockIdx.x] = carry;
}

// Downsweep: stable rank inside the tile with a register-only warp multisplit (five
// ballots give each key the lanes sharing its digit; lane d keeps the warp's running
// count of digit d), stage the tile in shared memory in digit order, write it out
// coalesced at digit_base[d] + p.counts[d][tile] + rank-within-digit.
struct DownsweepSmem {
    uint32_t keys[kSortTile];
    uint16_t perm[kSortTile];  // tile-local source index of each staged key
    uint32_t woff[kSortWarps][kRadix];
    uint32_t block_excl[kRadix];
    uint32_t global[kRadix];
};

template <bool kFull>
__device__ __forceinline__ void downsweep_tile(const SortPassParams& p, DownsweepSmem& sm, uint32_t count) {
    uint32_t* s_keys = sm.keys;
    uint16_t* s_perm = sm.perm;
    auto s_woff = sm.woff;
    uint32_t* s_block_excl = sm.block_excl;
    uint32_t* s_global = sm.global;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t mask = (1u << p.bits) - 1u;
    if (tid < kRadix) {  // global digit base (exclusive scan of the row totals) + this tile's offset
        const uint32_t total = static_cast<uint32_t>(tid) <= mask ? p.digit_base[tid] : 0u;
        s_global[tid] = warp_incl_scan(total, lane) - total + p.counts[tid * p.tiles + blockIdx.x];
    }
    const uint32_t base = blockIdx.x * kSortTile;
    const uint32_t lt = (1u << lane) - 1u;

    uint32_t k[kSortItems], rank2[kSortItems / 2];  // ranks (< 512) packed in pairs
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        k[j] = (kFull || idx < count) ? p.keys_in[idx] : 0u;
    }
    uint32_t lane_mask[kRadixBits];  // all-ones where lane's bit b is set
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) lane_mask[b] = 0u - ((static_cast<uint32_t>(lane) >> b) & 1u);
    uint32_t cnt = 0;  // lane d: keys of digit d so far in this warp's segment
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const uint32_t d = (k[j] >> p.shift) & mask;
        const uint32_t vm = kFull ? 0xffffffffu : __ballot_sync(0xffffffffu, idx < count);
        // Lane L's ballots give the lanes holding digit L; a key's own digit group is that
        // mask fetched from lane d (one shuffle instead of five more mask chains).
        uint32_t mine_differ = 0u;
#pragma unroll
        for (int b = 0; b < kRadixBits; ++b) mine_differ |= __ballot_sync(0xffffffffu, (d >> b) & 1u) ^ lane_mask[b];
        const uint32_t mine = vm & ~mine_differ;
        const uint32_t peers = __shfl_sync(0xffffffffu, mine, static_cast<int>(d));
        const uint32_t r = __shfl_sync(0xffffffffu, cnt, static_cast<int>(d)) + __popc(peers & lt);
        rank2[j / 2] = (j & 1) ? (rank2[j / 2] | (r << 16)) : r;
        cnt += __popc(mine);
    }
    s_woff[warp][lane] = cnt;
    __syncthreads();
    if (tid < 32) {  // digit tid: exclusive over warps, then over digits
        uint32_t run = 0, wrun[kSortWarps];
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            wrun[w] = run;
            run += s_woff[w][tid];
        }
        const uint32_t bex = warp_incl_scan(run, tid) - run;
        s_block_excl[tid] = bex;
        s_global[tid] -= bex;  // staged position e of digit d goes to s_global[d] + e
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) s_woff[w][tid] = bex + wrun[w];  // warp w's first slot of digit tid
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t local = warp * (32 * kSortItems) + j * 32 + lane;
        if (kFull || base + local < count) {
            const uint32_t d = (k[j] >> p.shift) & mask;
            const uint32_t pos = s_woff[warp][d] + ((j & 1) ? (rank2[j / 2] >> 16) : (rank2[j / 2] & 0xffffu));
            s_keys[pos] = k[j];
            s_perm[pos] = static_cast<uint16_t>(local);
        }
    }
    __syncthreads();
    // Write-out: every gather of the thread issued before any store (the value gathers
    // stay inside this tile's 16 KB input window, so they hit L2).
    const uint32_t n_here = kFull ? kSortTile : (count > base ? min(kSortTile, count - base) : 0u);
    const uint32_t* __restrict__ vals_in = p.vals_in;
    constexpr int kHalf = kSortItems / 2;  // two rounds: half the live registers
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t okey[kHalf], opos[kHalf], oval[kHalf];
#pragma unroll
        for (int j = 0; j < kHalf; ++j) {
            const uint32_t e = tid + (h * kHalf + j) * kSortThreads;
            if (kFull || e < n_here) {
                okey[j] = s_keys[e];
                opos[j] = s_global[(okey[j] >> p.shift) & mask] + e;
                const uint32_t src = base + s_perm[e];
                oval[j] = vals_in ? __ldg(vals_in + src) : src;
            }
        }
#pragma unroll
        for (int j = 0; j < kHalf; ++j) {
            const uint32_t e = tid + (h * kHalf + j) * kSortThreads;
            if (kFull || e < n_here) {
                GSCG_DCHECK(opos[j] < p.count);
                p.keys_out[opos[j]] = okey[j];
                p.vals_out[opos[j]] = oval[j];
            }
        }
    }
}

__global__ void __launch_bounds__(kSortThreads, 4)
k_sort_downsweep(SortPassParams p) {
    pdl_entry();
    __shared__ DownsweepSmem sm;
    // count: the host's, or the device counter clamped to it (deferred frames); only the
    // partial (last) tile needs it, so the full-tile path keeps its registers.
    const uint32_t count = resolve_count(p.count, p.count_dev);
    if (blockIdx.x * kSortTile >= count) return;  // past the device count (deferred frames)
    if ((blockIdx.x + 1) * kSortTile <= count) downsweep_tile<true>(p, sm, kSortTile);
    else downsweep_tile<false>(p, sm, count);
}

namespace {

template <bool kQuads>
__device__ __forceinline__ uint32_t cell_id(int cx, int cy, int tiles_x) {
    return kQuads ? static_cast<uint32_t>(((cy >> 1) * tiles_x + (cx >> 1)) * 4 + (cy & 1) * 2 + (cx & 1))
                  : static_cast<uint32_t>(cy * tiles_x + cx);
}

// Calls f(cell) for every binning cell of a packed span, row by row (the emission order);
// along a row the cell id advances without recomputing it (quadrant cells: +1 inside a
// tile, +3 into the next tile).
template <bool kQuads, typename F>
__device__ __forceinline__ void for_each_cell_t(uint2 sp, int tiles_x, F&& f) {
    const int cx0 = static_cast<int>(sp.x & 0xffffu), cy0 = static_cast<int>(sp.x >> 16);
    const int w = static_cast<int>(sp.y & 0xffffu), h = static_cast<int>(sp.y >> 16);
    for (int cy = cy0; cy < cy0 + h; ++cy) {
        uint32_t c = cell_id<kQuads>(cx0, cy, tiles_x);
        for (int cx = cx0; cx < cx0 + w; ++cx) {
            f(c);
            c += kQuads ? 1u + 2u * static_cast<uint32_t>(cx & 1) : 1u;
        }
    }
}

}  // namespace

// Wide-digit passes (up to kWideBits = 7 bits, 128 digits): the LSD plans use one where it
// saves a pass (a wide pass costs ~1.36x a 5-bit pass), e.g. the 12 cell bits left after
// emission at 3840x2160 take 7 + 5 instead of 4 + 4 + 4. Ranking keeps the ballot
// multisplit (one ballot per digit bit gives each key the lanes sharing its digit); the
// warp's running count per digit lives in shared memory (128 counters per warp, read by
// every lane of a digit group, advanced by the group's highest lane) instead of in lane
// registers.
namespace {

__device__ __forceinline__ uint32_t peers_of(uint32_t d, int bits, uint32_t valid) {
    uint32_t peers = valid;
#pragma unroll
    for (int b = 0; b < kWideBits; ++b) {
        if (b < bits) {
            const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bb : ~bb;
        }
    }
    return peers;
}

// Exclusive scan of v over the first 128 threads (4 warps); s_tmp holds 4 words.
__device__ __forceinline__ uint32_t scan128(uint32_t v, uint32_t* s_tmp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t x = warp_incl_scan(v, lane);
    if (threadIdx.x < kWideRadix && lane == 31) s_tmp[warp] = x;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp && w < kWideRadix / 32; ++w) off += s_tmp[w];
    __syncthreads();
    return off + x - v;
}

}  // namespace

template <bool kFull>
__device__ __forceinline__ void upsweep_wide_tile(const SortPassParams& p, uint32_t (*s_hist)[kWideRadix], uint32_t count) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * kWideRadix; i += blockDim.x) (&s_hist[0][0])[i] = 0u;
    const uint32_t base = blockIdx.x * kSortTile;
    const uint32_t mask = (1u << p.bits) - 1u;
    const int bits = static_cast<int>(p.bits);
    uint32_t k[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        k[j] = (kFull || idx < count) ? p.keys_in[idx] : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const uint32_t d = (k[j] >> p.shift) & mask;
        const uint32_t peers = peers_of(d, bits, kFull ? 0xffffffffu : __ballot_sync(0xffffffffu, idx < count));
        if ((kFull || idx < count) && lane == 31 - __clz(peers)) s_hist[warp][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x < kWideRadix) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) t += s_hist[w][threadIdx.x];
        if (static_cast<uint32_t>(threadIdx.x) <= mask) p.counts[threadIdx.x * p.tiles + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kSortThreads)
k_sort_upsweep_wide(SortPassParams p) {
    pdl_entry();
    __shared__ uint32_t s_hist[kSortWarps][kWideRadix];
    // count: the host's, or the device counter clamped to it (deferred frames); only the
    // partial (last) tile needs it, so the full-tile path keeps its registers.
    const uint32_t count = resolve_count(p.count, p.count_dev);
    if (blockIdx.x * kSortTile >= count) {  // past the device count (deferred frames): zero counts only
        if (threadIdx.x < kWideRadix) p.counts[threadIdx.x * p.tiles + blockIdx.x] = 0u;
        return;
    }
    if ((blockIdx.x + 1) * kSortTile <= count) upsweep_wide_tile<true>(p, s_hist, kSortTile);
    else upsweep_wide_tile<false>(p, s_hist, count);
}

struct DownsweepWideSmem {
    uint32_t keys[kSortTile];
    uint16_t perm[kSortTile];  // tile-local source index of each staged key
    uint32_t woff[kSortWarps][kWideRadix];
    uint32_t block_excl[kWideRadix];
    uint32_t global[kWideRadix];
    uint32_t tmp[kWideRadix / 32];
};

template <bool kFull>
__device__ __forceinline__ void downsweep_wide_tile(const SortPassParams& p, DownsweepWideSmem& sm, uint32_t count) {
    uint32_t* s_keys = sm.keys;
    uint16_t* s_perm = sm.perm;
    auto s_woff = sm.woff;
    uint32_t* s_block_excl = sm.block_excl;
    uint32_t* s_global = sm.global;
    uint32_t* s_tmp = sm.tmp;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t mask = (1u << p.bits) - 1u;
    const int bits = static_cast<int>(p.bits);
    for (int i = tid; i < kSortWarps * kWideRadix; i += blockDim.x) (&s_woff[0][0])[i] = 0u;
    const uint32_t base = blockIdx.x * kSortTile;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t k[kSortItems], rank2[kSortItems / 2];  // ranks (< 512) packed in pairs
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        k[j] = (kFull || idx < count) ? p.keys_in[idx] : 0u;
    }
    {  // global digit base (exclusive scan of the row totals) + this tile's offset
        const uint32_t total = tid < kWideRadix && static_cast<uint32_t>(tid) <= mask ? p.digit_base[tid] : 0u;
        const uint32_t excl = scan128(total, s_tmp);  // contains the block barrier for s_woff
        if (tid < kWideRadix)
            s_global[tid] = excl + (static_cast<uint32_t>(tid) <= mask ? p.counts[tid * p.tiles + blockIdx.x] : 0u);
    }
    uint32_t* wcnt = s_woff[warp];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const uint32_t d = (k[j] >> p.shift) & mask;
        const uint32_t peers = peers_of(d, bits, kFull ? 0xffffffffu : __ballot_sync(0xffffffffu, idx < count));
        const uint32_t before = wcnt[d];
        const uint32_t r = before + __popc(peers & lt);
        rank2[j / 2] = (j & 1) ? (rank2[j / 2] | (r << 16)) : r;
        __syncwarp();
        if ((kFull || idx < count) && lane == 31 - __clz(peers)) wcnt[d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    uint32_t run = 0;
    if (tid < kWideRadix) {  // digit tid: exclusive over warps
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = s_woff[w][tid];
            s_woff[w][tid] = run;
            run += c;
        }
    }
    const uint32_t bex = scan128(tid < kWideRadix ? run : 0u, s_tmp);  // over digits
    if (tid < kWideRadix) s_block_excl[tid] = bex;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t local = warp * (32 * kSortItems) + j * 32 + lane;
        if (kFull || base + local < count) {
            const uint32_t d = (k[j] >> p.shift) & mask;
            const uint32_t pos = s_block_excl[d] + s_woff[warp][d] + ((j & 1) ? (rank2[j / 2] >> 16) : (rank2[j / 2] & 0xffffu));
            s_keys[pos] = k[j];
            s_perm[pos] = static_cast<uint16_t>(local);
        }
    }
    __syncthreads();
    const uint32_t n_here = kFull ? kSortTile : (count > base ? min(kSortTile, count - base) : 0u);
    const uint32_t* __restrict__ vals_in = p.vals_in;
    constexpr int kHalf = kSortItems / 2;  // two rounds: half the live registers
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t okey[kHalf], opos[kHalf], oval[kHalf];
#pragma unroll
        for (int j = 0; j < kHalf; ++j) {
            const uint32_t e = tid + (h * kHalf + j) * kSortThreads;
            if (kFull || e < n_here) {
                okey[j] = s_keys[e];
                const uint32_t dd = (okey[j] >> p.shift) & mask;
                opos[j] = s_global[dd] + (e - s_block_excl[dd]);
                const uint32_t src = base + s_perm[e];
                oval[j] = vals_in ? __ldg(vals_in + src) : src;
            }
        }
#pragma unroll
        for (int j = 0; j < kHalf; ++j) {
            const uint32_t e = tid + (h * kHalf + j) * kSortThreads;
            if (kFull || e < n_here) {
                GSCG_DCHECK(opos[j] < p.count);
                p.keys_out[opos[j]] = okey[j];
                p.vals_out[opos[j]] = oval[j];
            }
        }
    }
}

__global__ void __launch_bounds__(kSortThreads, 4)
k_sort_downsweep_wide(SortPassParams p) {
    pdl_entry();
    __shared__ DownsweepWideSmem sm;
    // count: the host's, or the device counter clamped to it (deferred frames); only the
    // partial (last) tile needs it, so the full-tile path keeps its registers.
    const uint32_t count = resolve_count(p.count, p.count_dev);
    if (blockIdx.x * kSortTile >= count) return;  // past the device count (deferred frames)
    if ((blockIdx.x + 1) * kSortTile <= count) downsweep_wide_tile<true>(p, sm, kSortTile);
    else downsweep_wide_tile<false>(p, sm, count);
}

// After the depth sort: every sorted splat's binning span, gathered into sorted order
// (one 16-byte meta gather per splat, all eight of a thread in flight).
__global__ void __launch_bounds__(kMetaThreads)
k_sorted_spans(const uint32_t* recs, const uint4* meta, uint32_t count, const unsigned long long* count_dev,
               uint2* span_sorted) {
    pdl_entry();
    count = resolve_count(count, count_dev);
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
// the reference's bin order. Runs are short (a few pairs; ties inside one 8x8 cell): a CTA
// stages 2048 pairs in shared memory, gathers (depth, ordinal) for the tied pairs only,
// and the thread where a run starts insertion-sorts it there; a run leaving the tile is
// finished in global memory, and runs longer than kLongRun go to k_pair_long_runs.
namespace {

__device__ __forceinline__ unsigned long long pair_order_key(const uint4& m) {  // (depth bits, ordinal)
    return (static_cast<unsigned long long>(m.w) << 32) | m.x;
}

}  // namespace

__global__ void __launch_bounds__(256)
k_cell_fixup(const uint32_t* keys, uint32_t* recs, const uint4* meta, uint32_t count,
             const unsigned long long* count_dev, uint32_t cell_mask, int fix, uint2* ranges, uint2* long_runs,
             uint32_t* long_count, uint32_t long_cap) {
    pdl_entry();
    count = resolve_count(count, count_dev);
    static_assert(kStreamItems == 8, "two uint4 loads per thread");
    constexpr uint32_t kThreads = 256, kTile = kThreads * kStreamItems;
    constexpr uint32_t kHalo = 32;  // pairs past the tile: room for a run leaving the tile
    // Tile position p lives at slot (p % 8) * 256 + p / 8: a thread's item j of all lanes
    // is one contiguous row (conflict-free); the halo follows the tile.
    __shared__ uint32_t s_key[kTile + kHalo];
    __shared__ uint32_t s_rec[kTile + kHalo];
    __shared__ unsigned long long s_ord[kTile + kHalo];  // (depth bits, ordinal) of the tied pairs
    __shared__ uint16_t s_runs[kThreads / 32][32 * kStreamItems];  // run starts per warp
    __shared__ uint32_t s_enter_end;
    __shared__ uint32_t s_dirty[kThreads / 32];  // bit t % 32 of word t / 32: window of thread t moved
    auto slot = [](uint32_t p) { return p < kTile ? (p & 7u) * kThreads + (p >> 3) : p; };
    const uint32_t cta0 = blockIdx.x * kTile;
    if (cta0 >= count) return;
    const uint32_t tid = threadIdx.x;
    const uint32_t n_here = min(kTile, count - cta0);
    const uint32_t n_ext = min(kTile + kHalo, count - cta0);
    const bool has_prev = cta0 > 0;
    const uint32_t prev_key = has_prev ? keys[cta0 - 1] : 0u;
    const bool has_beyond = cta0 + n_ext < count;
    const uint32_t beyond_key = fix && has_beyond ? keys[cta0 + n_ext] : 0u;
    const uint32_t t0 = tid * kStreamItems;
    uint32_t k[kStreamItems], r[kStreamItems];
    if (n_here == kTile) {
        const uint4 klo = *reinterpret_cast<const uint4*>(keys + cta0 + t0);
        const uint4 khi = *reinterpret_cast<const uint4*>(keys + cta0 + t0 + 4);
        k[0] = klo.x; k[1] = klo.y; k[2] = klo.z; k[3] = klo.w; k[4] = khi.x; k[5] = khi.y; k[6] = khi.z; k[7] = khi.w;
        if (fix) {
            const uint4 rlo = *reinterpret_cast<const uint4*>(recs + cta0 + t0);
            const uint4 rhi = *reinterpret_cast<const uint4*>(recs + cta0 + t0 + 4);
            r[0] = rlo.x; r[1] = rlo.y; r[2] = rlo.z; r[3] = rlo.w; r[4] = rhi.x; r[5] = rhi.y; r[6] = rhi.z; r[7] = rhi.w;
        }
    } else {
#pragma unroll
        for (uint32_t j = 0; j < kStreamItems; ++j) {
            const bool in = t0 + j < n_here;
            k[j] = in ? keys[cta0 + t0 + j] : 0u;
            r[j] = in && fix ? recs[cta0 + t0 + j] : 0u;
        }
    }
#pragma unroll
    for (uint32_t j = 0; j < kStreamItems; ++j) {
        s_key[j * kThreads + tid] = k[j];
        if (fix) s_rec[j * kThreads + tid] = r[j];
    }
    if (fix && tid < kHalo && kTile + tid < n_ext) {
        s_key[kTile + tid] = keys[cta0 + kTile + tid];
        s_rec[kTile + tid] = recs[cta0 + kTile + tid];
    }
    __syncthreads();
    // Neighbours of the thread's window.
    const bool has_left = t0 > 0 || has_prev;
    const uint32_t left_key = t0 > 0 ? s_key[slot(t0 - 1)] : prev_key;
    const bool has_right = t0 + kStreamItems < n_ext;
    const uint32_t right_key = has_right ? s_key[slot(t0 + kStreamItems)] : 0u;
    // Cell ranges (the reference's bins).
#pragma unroll
    for (uint32_t j = 0; j < kStreamItems; ++j) {
        const uint32_t pos = t0 + j;
        if (pos >= n_here) break;
        const uint32_t c = k[j] & cell_mask;
        const bool first = j == 0 && !has_left;
        const uint32_t pc = (j > 0 ? k[j - 1] : left_key) & cell_mask;
        if (first || c != pc) {
            ranges[c].x = cta0 + pos;
            if (!first) ranges[pc].y = cta0 + pos;
        }
        if (cta0 + pos + 1 == count) ranges[c].y = count;
    }
    if (!fix) return;
    // Tied pairs: equal key word on either side. All their gathers in flight at once.
    bool tie[kStreamItems], left[kStreamItems];
    uint4 m[kStreamItems];
#pragma unroll
    for (uint32_t j = 0; j < kStreamItems; ++j) {
        const uint32_t pos = t0 + j;
        const bool in = pos < n_here;
        left[j] = in && (j > 0 ? k[j - 1] == k[j] : (has_left && left_key == k[j]));
        const bool right = j + 1 < kStreamItems ? (pos + 1 < n_here && k[j + 1] == k[j]) : (has_right && right_key == k[j]);
        tie[j] = in && (left[j] || right);
        m[j] = tie[j] ? meta[r[j]] : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (uint32_t j = 0; j < kStreamItems; ++j)
        if (tie[j]) s_ord[j * kThreads + tid] = pair_order_key(m[j]);
    if (tid < kHalo && n_here == kTile) {  // the run leaving the tile, into the halo
        const uint32_t p = kTile + tid;
        const bool eq = p < n_ext && s_key[p] == s_key[slot(kTile - 1)];
        const uint32_t in_run = __ffs(~__ballot_sync(0xffffffffu, eq)) - 1u;  // leading equal pairs (32: all)
        if (tid < in_run) s_ord[p] = pair_order_key(meta[s_rec[p]]);
    }
    // Run starts of the warp, compacted (a run entering from the previous tile is that
    // tile's): lanes then take one run each instead of walking their own windows.
    const uint32_t lane = tid & 31u, warp = tid >> 5;
    uint32_t starts = 0u;
#pragma unroll
    for (uint32_t j = 0; j < kStreamItems; ++j) starts |= (tie[j] && !left[j]) ? (1u << j) : 0u;
    uint32_t n_starts = __popc(starts), before = n_starts;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, before, o);
        if (lane >= static_cast<uint32_t>(o)) before += y;
    }
    const uint32_t warp_runs = __shfl_sync(0xffffffffu, before, 31);
    before -= n_starts;
    uint16_t* runs = s_runs[warp];
    for (uint32_t bits = starts; bits; bits &= bits - 1u) runs[before++] = static_cast<uint16_t>(t0 + __ffs(bits) - 1);
    // First position of the tile not in the run entering from the previous tile.
    if (tid == 0) s_enter_end = n_here;
    if (tid < kThreads / 32) s_dirty[tid] = 0u;
    __syncthreads();
    if (has_prev) {
        uint32_t first_diff = kStreamItems;
#pragma unroll
        for (int j = kStreamItems - 1; j >= 0; --j)
            if (t0 + j < n_here && k[j] != prev_key) first_diff = j;
        if (first_diff < kStreamItems) atomicMin(&s_enter_end, t0 + first_diff);
    } else if (tid == 0) {
        s_enter_end = 0u;
    }
    // Each lane sorts whole runs by (depth bits, ordinal) in shared memory (insertion sort;
    // the halo holds a run leaving the tile, whose halo part the lane stores itself). Runs
    // longer than kLongRun or leaving the halo are deferred to k_pair_long_runs.
    for (uint32_t q = lane; q < warp_runs; q += 32) {
        const uint32_t pos = runs[q];
        const uint32_t key = s_key[slot(pos)];
        uint32_t end = pos + 1;
        while (end < n_ext && s_key[slot(end)] == key) ++end;
        if ((end == n_ext && has_beyond && beyond_key == key) || end - pos > kLongRun) {
            const uint32_t at = atomicAdd(long_count, 1u);
            if (at < long_cap) long_runs[at] = make_uint2(cta0 + pos, end - pos);  // true end: k_pair_long_runs
            continue;
        }
        bool moved = false;
        for (uint32_t a = pos + 1; a < end; ++a) {
            const unsigned long long oa = s_ord[slot(a)];
            const uint32_t ra = s_rec[slot(a)];
            uint32_t i = a;
            while (i > pos && s_ord[slot(i - 1)] > oa) {
                s_ord[slot(i)] = s_ord[slot(i - 1)];
                s_rec[slot(i)] = s_rec[slot(i - 1)];
                --i;
            }
            if (i != a) {
                s_ord[slot(i)] = oa;
                s_rec[slot(i)] = ra;
                moved = true;
            }
        }
        if (!moved) continue;
        for (uint32_t w = pos / kStreamItems; w <= (min(end, n_here) - 1) / kStreamItems; ++w)
            atomicOr(&s_dirty[w / 32], 1u << (w % 32));
        for (uint32_t i = max(pos, n_here); i < end; ++i) recs[cta0 + i] = s_rec[i];  // halo part
    }
    __syncthreads();
    // The windows holding a reordered run back to memory (coalesced per thread), except
    // the run entering from the previous tile (stored by that tile, or deferred).
    const uint32_t e0 = s_enter_end;
    if (!((s_dirty[warp] >> lane) & 1u)) return;
    if (n_here == kTile && t0 >= e0) {
        uint32_t o[kStreamItems];
#pragma unroll
        for (uint32_t j = 0; j < kStreamItems; ++j) o[j] = s_rec[j * kThreads + tid];
        *reinterpret_cast<uint4*>(recs + cta0 + t0) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(recs + cta0 + t0 + 4) = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
        for (uint32_t j = 0; j < kStreamItems; ++j) {
            const uint32_t pos = t0 + j;
            if (pos >= e0 && pos < n_here) recs[cta0 + pos] = s_rec[j * kThreads + tid];
        }
    }
}

// Runs of more than kLongRun equal key words recorded by k_cell_fixup (many pairs of one
// truncated depth in one cell, e.g. characters stacked on one spot), and runs leaving a
// fix-up tile's halo: one CTA per run sorts
// ((depth bits, ordinal), record) in shared memory (bitonic, up to kPairRunCap); longer
// runs are sorted in place in global memory.
__global__ void __launch_bounds__(256)
k_pair_long_runs(const uint32_t* keys, uint32_t count, const unsigned long long* count_dev, uint32_t* recs,
                 const uint4* meta, const uint2* long_runs, const uint32_t* long_count) {
    pdl_entry();
    count = resolve_count(count, count_dev);
    __shared__ unsigned long long s_key[kPairRunCap];
    __shared__ uint32_t s_rec[kPairRunCap];
    __shared__ uint32_t s_n;
    const uint32_t runs = *long_count;  // <= the capacity sized in k_cell_fixup's contract
    for (uint32_t q = blockIdx.x; q < runs; q += gridDim.x) {
        const uint2 run = long_runs[q];
        const uint32_t s = run.x;
        if (threadIdx.x == 0) {  // a run recorded at a tile's halo may continue further
            const uint32_t k = keys[s];
            uint32_t n = run.y;
            while (s + n < count && keys[s + n] == k) ++n;
            s_n = n;
        }
        __syncthreads();
        const uint32_t n = s_n;
        __syncthreads();
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
// global base + this block's offset for the digit (k_sort_rows over the count pass's
// block histograms) + the pairs of that digit from earlier threads of the block + its
// rank among this thread's pairs of the digit. Threads own 4 consecutive sorted splats and
// enumerate each splat's cells row by row, so pairs of one digit keep the splat order: the
// output equals emitting in sorted order and running the first LSD pass on it.
// kCount: only count the block's pairs per digit (block_digit[d][block], the input of
// k_sort_rows); else scatter them.
template <bool kCount, bool kQuads>
__global__ void __launch_bounds__(kEmitThreads)
k_emit_scatter(const uint32_t* rec_sorted, const uint32_t* key_sorted, uint32_t count, const uint2* span_sorted,
               uint32_t* block_digit, const uint32_t* digit_total, uint32_t blocks, int tiles_x, int quads,
               uint32_t dmask, uint32_t tag_drop, uint32_t tag_shift, uint32_t* pair_cell, uint32_t* pair_rec,
               EmitCounts dc) {
    pdl_entry();
    count = resolve_count(count, dc.count_dev);
    if (blockIdx.x * kEmitSplats >= count) {  // past the device count (deferred frames)
        if (kCount && static_cast<uint32_t>(threadIdx.x) <= dmask && threadIdx.x < kRadix)
            block_digit[threadIdx.x * blocks + blockIdx.x] = 0u;
        return;
    }
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
    if (kCount) {  // block totals only: one shared atomic per pair on the block's 32 counters
        uint32_t* s_tot = &s_cnt[0][0];
        if (tid < kRadix) s_tot[tid] = 0u;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) for_each_cell_t<kQuads>(sp[q], tiles_x, [&](uint32_t c) { atomicAdd(&s_tot[c & dmask], 1u); });
        __syncthreads();
        if (static_cast<uint32_t>(tid) <= dmask && tid < kRadix) block_digit[tid * blocks + blockIdx.x] = s_tot[tid];
        return;
    }
#pragma unroll
    for (int d = 0; d < kRadix; ++d) s_cnt[d][tid] = 0u;
    if (tid < kRadix) {  // global base of digit tid: scanned digit totals + this block's offset
        const uint32_t t = static_cast<uint32_t>(tid) <= dmask ? digit_total[tid] : 0u;
        s_base[tid] = warp_incl_scan(t, lane) - t + (static_cast<uint32_t>(tid) <= dmask ? block_digit[tid * blocks + blockIdx.x] : 0u);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) for_each_cell_t<kQuads>(sp[q], tiles_x, [&](uint32_t c) { ++s_cnt[c & dmask][tid]; });
    __syncthreads();
    // Exclusive scan over threads for each digit (warp w: kDigitsPerWarp digits, lane l:
    // kPerLane consecutive threads), then over digits: s_cnt becomes each thread's start.
#pragma unroll
    for (int dd = 0; dd < kDigitsPerWarp; ++dd) {
        const int d = warp * kDigitsPerWarp + dd;
        static_assert(kPerLane == 4, "one 16-byte shared access per lane");
        uint4* row = reinterpret_cast<uint4*>(&s_cnt[d][lane * kPerLane]);  // conflict-free LDS.128
        const uint4 v = *row;
        const uint32_t sum = v.x + v.y + v.z + v.w;
        const uint32_t incl = warp_incl_scan(sum, lane);
        const uint32_t r0 = incl - sum;
        *row = make_uint4(r0, r0 + v.x, r0 + v.x + v.y, r0 + v.x + v.y + v.z);
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
        for_each_cell_t<kQuads>(sp[q], tiles_x, [&](uint32_t c) {
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
                 uint32_t* pair_rec, EmitCounts dc) {
    static bool attr = [] {
        cudaFuncSetAttribute(k_emit_scatter<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmem);
        cudaFuncSetAttribute(k_emit_scatter<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmem);
        cudaFuncSetAttribute(k_emit_scatter<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmem);
        cudaFuncSetAttribute(k_emit_scatter<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmem);
        return true;
    }();
    (void)attr;
    const int smem = count_only ? kRadix * 4 : kEmitSmem;  // the count pass keeps 32 block counters
    auto kernel = count_only ? (quads ? k_emit_scatter<true, true> : k_emit_scatter<true, false>)
                             : (quads ? k_emit_scatter<false, true> : k_emit_scatter<false, false>);
    pdl_launch(kernel, blocks, kEmitThreads, smem, s, rec_sorted, key_sorted, count, span_sorted, block_digit, digit_total,
               blocks, tiles_x, quads, dmask, tag_drop, tag_shift, pair_cell, pair_rec, dc);
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
