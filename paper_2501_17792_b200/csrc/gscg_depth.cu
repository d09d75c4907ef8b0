// Stage "sort", step 1 on the B200: the frame's splats in depth order by a two-level
// bucket sort (reference: sort_splats_impl renderer.cpp:85-107 orders by (depth bits,
// instance, gaussian); the depth bits are settled here, the tie-break per cell by
// k_cell_fixup).
//
// The splat order only has to be non-decreasing in the truncated key T = dbits >> drop
// (the top <= 25 varying bits): emission keeps it stable inside every cell and
// k_cell_fixup orders each run of equal (cell, T-tag) pairs by the full (depth bits,
// ordinal). Splats with equal T may therefore come out in any order, which lets both
// levels rank with shared-memory atomics instead of a stable multisplit:
//
//   k_depth_bucket_count   histogram of the top 14 bits of T (15 past 16 M splats) per CTA
//                          of 16,384 splats, flushed with one global atomic per non-empty bin
//   k_depth_bucket_scan    bucket starts (one CTA)
//   k_depth_bucket_scatter every splat reserves its slot in its bucket (a shared atomic for
//                          the rank inside the CTA, one global atomic per (CTA, bucket)) and
//                          writes (dbits, record, binning span) there — the span rides along,
//                          so no random meta gather follows the sort
//   k_depth_bucket_local   one CTA per bucket: counting sort over the low bits of T (<= 2,048
//                          bins) into the final keys / records / spans
//
// Two streaming passes over the S keys plus one over the staged buckets (L2-resident),
// instead of five reduce-then-scan LSD passes and the span gather.
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

__device__ __forceinline__ uint32_t depth_bucket(const DepthBucketParams& p, uint32_t dbits) {
    return ((dbits >> p.drop) - p.tag_min) >> p.local_bits;
}

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Exclusive scan of one value per thread over the CTA (blockDim.x = 32 * warps).
__device__ __forceinline__ uint32_t cta_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t x = warp_incl_scan_u32(v, lane);
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = warp_incl_scan_u32(lane < nw ? s_warp[lane] : 0u, lane);
        if (lane < nw) s_warp[lane] = w;
    }
    __syncthreads();
    total = s_warp[nw - 1];
    const uint32_t r = (warp ? s_warp[warp - 1] : 0u) + x - v;
    __syncthreads();
    return r;
}

}  // namespace

__global__ void __launch_bounds__(kBucketThreads)
k_depth_bucket_count(DepthBucketParams p) {
    pdl_entry();
    extern __shared__ uint32_t s_hist[];  // p.buckets bins
    for (uint32_t b = threadIdx.x; b < p.buckets; b += kBucketThreads) s_hist[b] = 0u;
    __syncthreads();
    const uint32_t base = blockIdx.x * kBucketTile;
    uint32_t k[kBucketItems];
#pragma unroll
    for (int j = 0; j < kBucketItems; ++j) {  // all loads in flight first
        const uint32_t i = base + j * kBucketThreads + threadIdx.x;
        k[j] = i < p.count ? p.depth[i] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kBucketItems; ++j) {
        const uint32_t i = base + j * kBucketThreads + threadIdx.x;
        if (i < p.count) {
            GSCG_DCHECK(depth_bucket(p, k[j]) < p.buckets);
            atomicAdd(&s_hist[depth_bucket(p, k[j])], 1u);
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < p.buckets; b += kBucketThreads) {
        const uint32_t h = s_hist[b];
        if (h) atomicAdd(&p.bucket_count[b], h);
    }
}

// Bucket starts: warp w scans buckets [w * 32 c, (w + 1) * 32 c), c = ceil(buckets / 1024)
// lane-contiguous chunks of 32 (coalesced loads and stores), then the warp totals.
__global__ void __launch_bounds__(1024)
k_depth_bucket_scan(DepthBucketParams p) {
    pdl_entry();
    __shared__ uint32_t s_warp[32];
    constexpr uint32_t kChunks = kMaxDepthBuckets / 1024;  // most 32-bucket chunks per warp
    const uint32_t nch = (p.buckets + 1023) / 1024;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t v[kChunks], wsum = 0;
#pragma unroll
    for (uint32_t c = 0; c < kChunks; ++c) {
        const uint32_t bk = (warp * nch + c) * 32u + lane;
        v[c] = c < nch && bk < p.buckets ? p.bucket_count[bk] : 0u;
        wsum += v[c];
    }
    wsum = __reduce_add_sync(0xffffffffu, wsum);
    if (lane == 0) s_warp[warp] = wsum;
    __syncthreads();
    uint32_t carry = 0;
    for (uint32_t w = 0; w < warp; ++w) carry += s_warp[w];
#pragma unroll
    for (uint32_t c = 0; c < kChunks; ++c) {
        if (c >= nch) break;
        const uint32_t bk = (warp * nch + c) * 32u + lane;
        const uint32_t incl = warp_incl_scan_u32(v[c], static_cast<int>(lane));
        if (bk < p.buckets) {
            p.bucket_start[bk] = carry + incl - v[c];
            p.bucket_cursor[bk] = carry + incl - v[c];
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (threadIdx.x == 1023) p.bucket_start[p.buckets] = carry;
}

__global__ void __launch_bounds__(kBucketThreads)
k_depth_bucket_scatter(DepthBucketParams p) {
    pdl_entry();
    extern __shared__ uint32_t s_hist[];  // counts, then each bin's global slot base
    const uint32_t base = blockIdx.x * kBucketScatterTile;
    // Every load of the thread in flight at once (the splat meta carries the depth bits),
    // so the CTA pays one memory latency, then the reservations' one.
    uint4 m[kBucketScatterItems];
#pragma unroll
    for (int j = 0; j < kBucketScatterItems; ++j) {
        const uint32_t i = base + j * kBucketThreads + threadIdx.x;
        if (i < p.count) m[j] = p.meta[i];  // (ordinal, span lo, span hi, dbits), coalesced
    }
    for (uint32_t b = threadIdx.x; b < p.buckets; b += kBucketThreads) s_hist[b] = 0u;
    __syncthreads();
    // (bucket << 16 | rank in the CTA's share of the bucket); ranks < kBucketScatterTile.
    uint32_t br[kBucketScatterItems];
#pragma unroll
    for (int j = 0; j < kBucketScatterItems; ++j) {
        const uint32_t i = base + j * kBucketThreads + threadIdx.x;
        if (i < p.count) {
            const uint32_t b = depth_bucket(p, m[j].w);
            GSCG_DCHECK(b < p.buckets);
            br[j] = (b << 16) | atomicAdd(&s_hist[b], 1u);
        }
    }
    __syncthreads();
    {  // one global reservation per non-empty bin, a batch of the thread's bins in flight at once
        constexpr uint32_t kPer = 8;  // bins per batch (registers)
        for (uint32_t half = 0; half * kPer * kBucketThreads < p.buckets; ++half) {
            uint32_t h[kPer];
#pragma unroll
            for (uint32_t q = 0; q < kPer; ++q) {
                const uint32_t b = (half * kPer + q) * kBucketThreads + threadIdx.x;
                h[q] = b < p.buckets ? s_hist[b] : 0u;
            }
#pragma unroll
            for (uint32_t q = 0; q < kPer; ++q)
                if (h[q]) h[q] = atomicAdd(&p.bucket_cursor[(half * kPer + q) * kBucketThreads + threadIdx.x], h[q]);
#pragma unroll
            for (uint32_t q = 0; q < kPer; ++q) {
                const uint32_t b = (half * kPer + q) * kBucketThreads + threadIdx.x;
                if (b < p.buckets) s_hist[b] = h[q];
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kBucketScatterItems; ++j) {
        const uint32_t i = base + j * kBucketThreads + threadIdx.x;
        if (i < p.count) {
            GSCG_DCHECK(s_hist[br[j] >> 16] + (br[j] & 0xffffu) < p.count);
            p.staged[s_hist[br[j] >> 16] + (br[j] & 0xffffu)] = make_uint4(m[j].w, i, m[j].y, m[j].z);
        }
    }
}

// One CTA per bucket: counting sort over the bucket's low T bits (bins in shared memory;
// ranks by shared atomics, so equal T land in any order — see the file comment). The
// bucket (contiguous in the staged array) arrives in chunks of kBucketLocalCap splats, one
// bulk copy each into shared memory completing on an mbarrier. A bucket of up to
// kBucketLocalChunks chunks is ranked into an inverse permutation (sorted position ->
// bucket index) and written out coalesced, chunk by chunk (scattered 16-byte stores cost
// ~2 clocks per sector here: the scattered writes were this kernel's whole cost). Larger
// buckets stream through twice with scattered writes.
__global__ void __launch_bounds__(kBucketLocalThreads)
k_depth_bucket_local(DepthBucketParams p) {
    pdl_entry();
    extern __shared__ uint4 s_el[];  // one chunk of staged splats
    __shared__ uint32_t s_bin[kBucketLocalBins];
    __shared__ uint16_t s_inv[kBucketLocalCap * kBucketLocalChunks];  // sorted position -> bucket index
    __shared__ uint32_t s_warp[32];
    __shared__ __align__(8) uint64_t s_bar;
    const uint32_t b = blockIdx.x;
    const uint32_t s0 = p.bucket_start[b], n = p.bucket_start[b + 1] - s0;
    GSCG_DCHECK(s0 <= p.count && n <= p.count - s0);
    if (n == 0) return;
    const uint4* src = p.staged + s0;
    const uint32_t tid = threadIdx.x;
    auto put = [&](uint32_t o, const uint4& e) {
        GSCG_DCHECK(o >= s0 && o < s0 + n && e.y < p.count);
        p.keys_out[o] = e.x;
        p.recs_out[o] = e.y;
        p.spans_out[o] = make_uint2(e.z, e.w);
    };
    if (n == 1) {
        if (tid == 0) put(s0, src[0]);
        return;
    }
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint32_t bins = 1u << p.local_bits, lmask = bins - 1u;
    const uint32_t zbins = max(bins, 32u);  // whole 32-bin scan chunks
    for (uint32_t d = tid; d < zbins; d += kBucketLocalThreads) s_bin[d] = 0u;
    __syncthreads();
    auto bin = [&](uint32_t key) { return ((key >> p.drop) - p.tag_min) & lmask; };
    const uint32_t chunks = (n + kBucketLocalCap - 1) / kBucketLocalCap;
    uint32_t phase = 0, resident = 0xffffffffu;
    auto load = [&](uint32_t c) {  // chunk c into s_el (callers sync before a reload); returns its size
        const uint32_t c0 = c * kBucketLocalCap, m = min(kBucketLocalCap, n - c0);
        if (c != resident) {
            if (tid == 0) {
                mbar_arrive_expect_tx(&s_bar, m * 16u);
                bulk_g2s(s_el, src + c0, m * 16u, &s_bar);
            }
            mbar_wait(&s_bar, phase);
            phase ^= 1u;
            resident = c;
        }
        return m;
    };
    for (uint32_t c = 0; c < chunks; ++c) {
        const uint32_t m = load(c);
        for (uint32_t i = tid; i < m; i += kBucketLocalThreads) atomicAdd(&s_bin[bin(s_el[i].x)], 1u);
        __syncthreads();  // the chunk buffer may be refilled
    }
    // Exclusive scan of the bins, warp w over chunks [w * C / W, (w + 1) * C / W) of 32
    // consecutive bins (lane-contiguous: no bank conflicts), then the warp totals.
    {
        const int lane = tid & 31, warp = tid >> 5;
        constexpr int kWarps = kBucketLocalThreads / 32;
        const uint32_t bc = zbins / 32, c0 = warp * bc / kWarps, c1 = (warp + 1) * bc / kWarps;
        uint32_t wsum = 0;
        for (uint32_t c = c0; c < c1; ++c) wsum += __reduce_add_sync(0xffffffffu, s_bin[c * 32 + lane]);
        if (lane == 0) s_warp[warp] = wsum;
        __syncthreads();
        uint32_t carry = 0;
        for (int w = 0; w < warp; ++w) carry += s_warp[w];
        for (uint32_t c = c0; c < c1; ++c) {
            const uint32_t v = s_bin[c * 32 + lane];
            const uint32_t incl = warp_incl_scan_u32(v, lane);
            s_bin[c * 32 + lane] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncthreads();
    if (chunks <= kBucketLocalChunks) {
        // Ranks into the inverse permutation (the resident chunk first), then each output
        // row once, coalesced, from whichever chunk is resident.
        for (uint32_t q = 0; q < chunks; ++q) {
            const uint32_t c = chunks - 1 - q;
            const uint32_t m = load(c);
            for (uint32_t i = tid; i < m; i += kBucketLocalThreads)
            {
                const uint32_t slot = atomicAdd(&s_bin[bin(s_el[i].x)], 1u);
                GSCG_DCHECK(slot < n);
                s_inv[slot] = static_cast<uint16_t>(c * kBucketLocalCap + i);
            }
            __syncthreads();
        }
        for (uint32_t q = 0; q < chunks; ++q) {  // chunk 0 is resident now
            const uint32_t c0 = q * kBucketLocalCap;
            load(q);
            for (uint32_t j = tid; j < n; j += kBucketLocalThreads) {
                const uint32_t i = s_inv[j];
                if (chunks == 1 || i - c0 < kBucketLocalCap) put(s0 + j, s_el[i - c0]);
            }
            __syncthreads();
        }
        return;
    }
    for (uint32_t c = 0; c < chunks; ++c) {
        const uint32_t m = load(c);
        for (uint32_t i = tid; i < m; i += kBucketLocalThreads) {
            const uint4 e = s_el[i];
            put(s0 + atomicAdd(&s_bin[bin(e.x)], 1u), e);
        }
        __syncthreads();
    }
}

}  // namespace gscg
