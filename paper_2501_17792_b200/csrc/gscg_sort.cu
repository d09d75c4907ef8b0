// Stage "sort" on the B200: stable LSD radix sort of the 64-bit tile|depth pair keys
// (reference: sort_splats_impl renderer.cpp:85-107 + binning renderer.cpp:143-161).
//
// The reference sorts splats globally by (depth bits, instance_id, gaussian_index) and
// then bins them into tiles in sorted order, so each tile's list is ordered by that
// triple. Here pairs carry key = tile << 32 | depth_bits and value = splat record index;
// an 8-bit-digit onesweep radix sort over the exact significant key bits (depth bits
// above the frame's common prefix are skipped) orders them by (tile, depth), and
// k_tie_fixup orders the rare equal-key runs by the splat ordinal
// (instance base + gaussian index), which is the reference's (instance, gaussian)
// tie-break. Result: per-tile lists identical to the reference's bins.
//
// Onesweep pass: each CTA takes a 4096-key tile by atomic ticket (forward progress for
// the look-back), ranks keys stably per warp with __match_any_sync, publishes its digit
// counts, resolves its global digit offsets with a decoupled look-back over preceding
// tiles, stages the tile in shared memory in digit order and writes it out coalesced.
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

__device__ __forceinline__ uint32_t digit_of(unsigned long long key, uint32_t dbits,
                                             unsigned long long dmask, uint32_t shift) {
    const unsigned long long vkey = ((key >> 32) << dbits) | (key & dmask);
    return static_cast<uint32_t>(vkey >> shift) & 0xffu;
}

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;

__device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, uint32_t epoch,
                                                          uint32_t value) {
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

}  // namespace

__global__ void __launch_bounds__(256)
k_digit_histogram(const unsigned long long* keys, uint32_t count, uint32_t dbits,
                  unsigned long long dmask, uint32_t passes, uint32_t* hist) {
    __shared__ uint32_t s_hist[kMaxSortPasses][256];
    for (int i = threadIdx.x; i < kMaxSortPasses * 256; i += blockDim.x) (&s_hist[0][0])[i] = 0u;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const unsigned long long key = keys[i];
        const unsigned long long vkey = ((key >> 32) << dbits) | (key & dmask);
        for (uint32_t q = 0; q < passes; ++q)
            atomicAdd(&s_hist[q][static_cast<uint32_t>(vkey >> (8 * q)) & 0xffu], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < passes * 256; i += blockDim.x) {
        const uint32_t c = (&s_hist[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// In-place exclusive scan of each pass's 256-bin histogram (one CTA per pass).
__global__ void __launch_bounds__(256) k_digit_scan(uint32_t* hist, uint32_t passes) {
    __shared__ uint32_t s[256];
    uint32_t* h = hist + blockIdx.x * 256;
    const uint32_t v = h[threadIdx.x];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
        const uint32_t y = threadIdx.x >= o ? s[threadIdx.x - o] : 0u;
        __syncthreads();
        s[threadIdx.x] += y;
        __syncthreads();
    }
    h[threadIdx.x] = s[threadIdx.x] - v;
}

__global__ void __launch_bounds__(kSortThreads)
k_onesweep(SortPassParams p) {
    extern __shared__ unsigned long long s_keys[];            // kSortTile keys
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + kSortTile);
    __shared__ uint32_t s_wcount[kSortThreads / 32][256];
    __shared__ uint32_t s_block_excl[256];
    __shared__ uint32_t s_global[256];
    __shared__ uint32_t s_scan[kSortThreads / 32];
    __shared__ uint32_t s_block;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_block = atomicAdd(p.ticket, 1u);
    for (int i = tid; i < (kSortThreads / 32) * 256; i += kSortThreads) (&s_wcount[0][0])[i] = 0u;
    __syncthreads();
    const uint32_t b = s_block;
    const uint32_t base = b * kSortTile;

    unsigned long long k[kSortItems];
    uint32_t v[kSortItems], d[kSortItems], rank[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t idx = base + warp * (32 * kSortItems) + j * 32 + lane;
        const bool valid = idx < p.count;
        k[j] = valid ? p.keys_in[idx] : 0ull;
        v[j] = valid ? p.vals_in[idx] : 0u;
        d[j] = valid ? digit_of(k[j], p.dbits, p.dmask, p.shift) : 256u;
    }
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint32_t peers = __match_any_sync(0xffffffffu, d[j]);
        const uint32_t prior = d[j] < 256u ? s_wcount[warp][d[j] & 0xffu] : 0u;
        rank[j] = prior + __popc(peers & lt_mask);
        __syncwarp();
        if (d[j] < 256u && lane == __ffs(peers) - 1) s_wcount[warp][d[j]] = prior + __popc(peers);
        __syncwarp();
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
    // Digit-major exclusive offsets inside the block (staging layout).
    {
        uint32_t x = total;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_scan[warp] = x;
        __syncthreads();
        uint32_t before = 0;
#pragma unroll
        for (int w = 0; w < kSortThreads / 32; ++w)
            if (w < warp) before += s_scan[w];
        s_block_excl[tid] = before + x - total;
    }

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
        const unsigned long long key = s_keys[e];
        const uint32_t dd = digit_of(key, p.dbits, p.dmask, p.shift);
        const uint32_t pos = s_global[dd] + (e - s_block_excl[dd]);
        p.keys_out[pos] = key;
        p.vals_out[pos] = s_vals[e];
    }
}

// Equal (tile, depth) keys: order the run by splat ordinal = (instance, gaussian) order
// (renderer.cpp:91-96 tie-break). Runs are rare and short.
__global__ void k_tie_fixup(const unsigned long long* keys, uint32_t* vals,
                            const uint32_t* ordinal, uint32_t count) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < count; i += gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
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

// [start, end) of every tile in the sorted pair array (the reference's bins).
__global__ void k_tile_ranges(const unsigned long long* keys, uint32_t count, uint2* ranges) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const uint32_t tile = static_cast<uint32_t>(keys[i] >> 32);
        if (i == 0 || static_cast<uint32_t>(keys[i - 1] >> 32) != tile) ranges[tile].x = i;
        if (i + 1 == count || static_cast<uint32_t>(keys[i + 1] >> 32) != tile) ranges[tile].y = i + 1;
    }
}

__global__ void k_sorted_ordinals(const uint32_t* vals, const uint32_t* ordinal, uint32_t count,
                                  uint32_t* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        out[i] = ordinal[vals[i]];
}

}  // namespace gscg
