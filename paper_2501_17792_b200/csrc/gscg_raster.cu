// Stage "rasterize" on the B200: per-tile front-to-back alpha blending
// (reference: rasterize_full renderer.cpp:121-232).
//
// One CTA per tile. The tile's sorted splat indices are consumed in batches of 256: each
// thread gathers one 48-byte record into shared memory (3 x float4, coalesced per
// record), then every pixel thread walks the batch in order. Semantics kept from the
// reference (SURVEY.md §7 "reference raster semantics"):
//   * a pixel is touched only inside the splat's clipped 3-sigma rectangle;
//   * the cutoff test is power < power_floor with power_floor = logf(cutoff/opacity)
//     precomputed by the host (glibc, bit-identical to the reference);
//   * the splat that pushes T below the floor is blended, then the pixel stops;
//   * output = rgb + T * background, and T itself.
// The per-pixel power is computed with round-to-nearest intrinsics in the reference
// order (renderer.cpp:197-204) so the set of contributing (pixel, splat) pairs is the
// reference's; alpha uses the hardware exp2 path (tolerance-checked).
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

struct SplatView {
    float mx, my, a, b, c, o, pf, r, g, bl;
    int x0, y0, x1, y1;
};

__device__ __forceinline__ SplatView unpack(const float4* s, int k) {
    const float4 r0 = s[3 * k + 0], r1 = s[3 * k + 1], r2 = s[3 * k + 2];
    SplatView v;
    v.mx = r0.x;
    v.my = r0.y;
    v.a = r0.z;
    v.b = r0.w;
    v.c = r1.x;
    v.o = r1.y;
    v.pf = r1.z;
    v.r = r1.w;
    v.g = r2.x;
    v.bl = r2.y;
    const uint32_t lo = __float_as_uint(r2.z), hi = __float_as_uint(r2.w);
    v.x0 = static_cast<int>(lo & 0xffffu);
    v.y0 = static_cast<int>(lo >> 16);
    v.x1 = static_cast<int>(hi & 0xffffu);
    v.y1 = static_cast<int>(hi >> 16);
    return v;
}

// power = -0.5f * (a*dx*dx + c*dy*dy) - b*dx*dy, single rounding per operation.
__device__ __forceinline__ float pixel_power(const SplatView& s, float fx, float fy) {
    const float dx = __fsub_rn(fx, s.mx);
    const float dy = __fsub_rn(fy, s.my);
    const float q = __fadd_rn(__fmul_rn(__fmul_rn(s.a, dx), dx), __fmul_rn(__fmul_rn(s.c, dy), dy));
    return __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(s.b, dx), dy));
}

// Blend one splat into one pixel; returns true when the pixel reaches the floor.
__device__ __forceinline__ bool blend(const SplatView& s, int px, int py, float& T, float& cr,
                                      float& cg, float& cb, float amax, float tfloor) {
    if (px < s.x0 || px >= s.x1 || py < s.y0 || py >= s.y1) return false;
    const float power = pixel_power(s, static_cast<float>(px) + 0.5f, static_cast<float>(py) + 0.5f);
    if (power < s.pf) return false;
    const float alpha = fminf(s.o * __expf(power), amax);
    const float w = T * alpha;
    cr = fmaf(w, s.r, cr);
    cg = fmaf(w, s.g, cg);
    cb = fmaf(w, s.bl, cb);
    T = T * (1.0f - alpha);
    return T < tfloor;
}

}  // namespace

// Tile size 16, quadrant form: one 64-thread CTA per 8x8 quadrant of a tile (grid =
// 4 x tiles). Crowd frames are extremely skewed — horizon tiles carry tens of thousands
// of pairs and mix saturated crowd pixels with never-saturating sky — so splitting a tile
// four ways cuts the serial list walk of the heaviest tiles by 4x and lets each quadrant
// stop on its own saturation. Warp w covers the 8x4 block at rows 4w..4w+3 and walks the
// quadrant's list on its own (no CTA barrier: a saturated warp never waits for the
// other), staging 32 records at a time with the next 32 already in flight. Each pixel
// still walks the tile's list in order, so results are identical to the whole-tile form.
__global__ void __launch_bounds__(64)
k_raster16q(RasterParams p) {
    __shared__ float4 s_geo[2][32];
    __shared__ float4 s_col[2][32];
    __shared__ float2 s_col2[2][32];
    __shared__ uint2 s_rect[2][32];
    const int tile = blockIdx.x >> 2, quad = blockIdx.x & 3;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x + p.tile_row0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int bx0 = tx * 16 + (quad & 1) * 8;
    const int by0 = ty * 16 + (quad >> 1) * 8 + warp * 4;  // warp block origin (8 x 4)
    const int px = bx0 + (lane & 7);
    const int py = by0 + (lane >> 3);
    const bool inside = px < p.width && py < p.height;
    const uint2 range = p.ranges[blockIdx.x];  // this quadrant's cell: tile * 4 + quad
    const float fx = static_cast<float>(px) + 0.5f, fy = static_cast<float>(py) + 0.5f;
    float4* geo = s_geo[warp];
    float4* col = s_col[warp];
    float2* col2 = s_col2[warp];
    uint2* rect = s_rect[warp];
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    bool done = !inside;
    // Records of the chunk after the current one, loaded while the current one is walked.
    float4 n0 = make_float4(0, 0, 0, 0), n1 = n0, n2 = n0;
    if (range.x + lane < range.y) {
        const float4* src = p.records + 3ull * p.recs[range.x + lane];
        n0 = src[0];
        n1 = src[1];
        n2 = src[2];
    }
    for (uint32_t start = range.x; start < range.y; start += 32) {
        if (__all_sync(0xffffffffu, done)) break;
        __syncwarp();
        geo[lane] = n0;
        col[lane] = n1;
        col2[lane] = make_float2(n2.x, n2.y);
        rect[lane] = make_uint2(__float_as_uint(n2.z), __float_as_uint(n2.w));
        __syncwarp();
        if (start + 32 + lane < range.y) {
            const float4* src = p.records + 3ull * p.recs[start + 32 + lane];
            n0 = src[0];
            n1 = src[1];
            n2 = src[2];
        }
        const int n = min(32u, range.y - start);
        // Lane L: which of this warp's 32 pixels splat L's rect covers (bit = lane).
        uint32_t cover = 0;
        if (lane < n) {
            const uint2 r = rect[lane];
            const int cx0 = max(static_cast<int>(r.x & 0xffff) - bx0, 0);
            const int cx1 = min(static_cast<int>(r.y & 0xffff) - bx0, 8);
            const int cy0 = max(static_cast<int>(r.x >> 16) - by0, 0);
            const int cy1 = min(static_cast<int>(r.y >> 16) - by0, 4);
            if (cx0 < cx1 && cy0 < cy1) {
                const uint32_t row = ((1u << cx1) - 1u) & ~((1u << cx0) - 1u);
                const uint32_t rows = static_cast<uint32_t>(((1ull << (8 * cy1)) - 1ull) & ~((1ull << (8 * cy0)) - 1ull));
                cover = (row * 0x01010101u) & rows;
            }
        }
        // Bit-matrix transpose across the warp: lane L now holds, in list order, the
        // chunk's splats that cover pixel L.
        uint32_t todo = cover;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
            const uint32_t m = s == 16 ? 0x0000ffffu : s == 8 ? 0x00ff00ffu : s == 4 ? 0x0f0f0f0fu
                                                     : s == 2 ? 0x33333333u : 0x55555555u;
            const uint32_t y = __shfl_xor_sync(0xffffffffu, todo, s);
            todo = (lane & s) ? ((todo & ~m) | ((y & ~m) >> s)) : ((todo & m) | ((y & m) << s));
        }
        if (done) todo = 0u;
        // Every lane walks its own splats in order; lanes with disjoint splats work
        // concurrently instead of idling through each other's splats.
        while (__any_sync(0xffffffffu, todo != 0u)) {
            if (todo == 0u) continue;
            const int k = __ffs(todo) - 1;
            todo &= todo - 1u;
            const float4 g = geo[k];
            const float dx = __fsub_rn(fx, g.x);
            const float dy = __fsub_rn(fy, g.y);
            const float4 c = col[k];
            const float q = __fadd_rn(__fmul_rn(__fmul_rn(g.z, dx), dx), __fmul_rn(__fmul_rn(c.x, dy), dy));
            const float power = __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(g.w, dx), dy));
            if (power < c.z) continue;
            const float alpha = fminf(c.y * __expf(power), p.alpha_max);
            const float w = T * alpha;
            const float2 c2 = col2[k];
            cr = fmaf(w, c.w, cr);
            cg = fmaf(w, c2.x, cg);
            cb = fmaf(w, c2.y, cb);
            T = T * (1.0f - alpha);
            if (T < p.t_floor) {
                done = true;
                todo = 0u;
            }
        }
    }
    if (inside) {
        const size_t o = static_cast<size_t>(py - p.out_row0) * p.width + px;
        p.out_rgb[3 * o + 0] = cr + T * p.bg[0];
        p.out_rgb[3 * o + 1] = cg + T * p.bg[1];
        p.out_rgb[3 * o + 2] = cb + T * p.bg[2];
        p.out_T[o] = T;
    }
}

// Any tile size up to 16*sqrt(PPT): PPT pixels per thread, pixel p = tid + k*256.
template <int PPT>
__global__ void __launch_bounds__(256)
k_raster_generic(RasterParams p) {
    __shared__ float4 s_rec[256 * 3];
    const int ts = p.tile_size;
    const int tile = blockIdx.x;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x + p.tile_row0;
    float T[PPT], cr[PPT], cg[PPT], cb[PPT];
    int pxs[PPT], pys[PPT];
    bool live[PPT];
    int live_count = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int lp = threadIdx.x + k * 256;
        pxs[k] = tx * ts + lp % ts;
        pys[k] = ty * ts + lp / ts;
        live[k] = lp < ts * ts && pxs[k] < p.width && pys[k] < p.height;
        T[k] = 1.0f;
        cr[k] = cg[k] = cb[k] = 0.0f;
        live_count += live[k] ? 1 : 0;
    }
    const uint2 range = p.ranges[tile];
    for (uint32_t start = range.x; start < range.y; start += 256) {
        if (__syncthreads_or(live_count > 0) == 0) break;
        const uint32_t i = start + threadIdx.x;
        if (i < range.y) {
            const float4* src = p.records + 3ull * p.recs[i];
            s_rec[3 * threadIdx.x + 0] = src[0];
            s_rec[3 * threadIdx.x + 1] = src[1];
            s_rec[3 * threadIdx.x + 2] = src[2];
        }
        __syncthreads();
        const int n = min(256u, range.y - start);
        for (int s = 0; s < n && live_count > 0; ++s) {
            const SplatView v = unpack(s_rec, s);
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                if (!live[k]) continue;
                if (blend(v, pxs[k], pys[k], T[k], cr[k], cg[k], cb[k], p.alpha_max, p.t_floor)) {
                    live[k] = false;
                    --live_count;
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const int lp = threadIdx.x + k * 256;
        if (lp < ts * ts && pxs[k] < p.width && pys[k] < p.height) {
            const size_t o = static_cast<size_t>(pys[k] - p.out_row0) * p.width + pxs[k];
            p.out_rgb[3 * o + 0] = cr[k] + T[k] * p.bg[0];
            p.out_rgb[3 * o + 1] = cg[k] + T[k] * p.bg[1];
            p.out_rgb[3 * o + 2] = cb[k] + T[k] * p.bg[2];
            p.out_T[o] = T[k];
        }
    }
}

void launch_raster(const RasterParams& p, uint32_t tiles, cudaStream_t stream) {
    if (p.tile_size == 16) k_raster16q<<<tiles * 4, 64, 0, stream>>>(p);
    else if (p.tile_size <= 16) k_raster_generic<1><<<tiles, 256, 0, stream>>>(p);
    else if (p.tile_size <= 32) k_raster_generic<4><<<tiles, 256, 0, stream>>>(p);
    else k_raster_generic<16><<<tiles, 256, 0, stream>>>(p);
}

}  // namespace gscg
