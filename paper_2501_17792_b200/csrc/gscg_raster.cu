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
// Every operation of the per-pixel blend is single-rounded in the reference order
// (renderer.cpp:197-226): power, alpha = opacity * expf(power) with a bit-exact replica of
// the host libm's expf (gscg_expf.cuh), the clamp, w = T * alpha, rgb += w * colour (no
// FMA), T *= 1 - alpha and rgb + T * background; so every pixel and T equal the
// reference's bit for bit.
#include <cstdlib>

#include "gscg_common.cuh"
#include "gscg_expf.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

__constant__ unsigned long long c_exp2f_tab[32] = GSCG_EXP2F_TAB;

// The expf table in shared memory (lanes index it independently; the constant bank would
// serialise divergent indices).
__device__ __forceinline__ void load_exp_table(unsigned long long* s_tab) {
    for (int i = threadIdx.x; i < 32; i += blockDim.x) s_tab[i] = c_exp2f_tab[i];
}

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
                                      float& cg, float& cb, float amax, float tfloor, const ExpfRegs& ek) {
    if (px < s.x0 || px >= s.x1 || py < s.y0 || py >= s.y1) return false;
    const float power = pixel_power(s, static_cast<float>(px) + 0.5f, static_cast<float>(py) + 0.5f);
    if (power < s.pf) return false;
    const float alpha = fminf(__fmul_rn(s.o, glibc_expf_regs(power, ek)), amax);
    const float w = __fmul_rn(T, alpha);
    cr = __fadd_rn(cr, __fmul_rn(w, s.r));
    cg = __fadd_rn(cg, __fmul_rn(w, s.g));
    cb = __fadd_rn(cb, __fmul_rn(w, s.bl));
    T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
    return T < tfloor;
}

}  // namespace

namespace {
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// The 8x4-pixel coverage bits of splat rect r for the warp block at (bx0, by0).
__device__ __forceinline__ uint32_t block_cover(float4 r2, int bx0, int by0) {
    const uint32_t a = __float_as_uint(r2.z), b = __float_as_uint(r2.w);
    const int cx0 = max(static_cast<int>(a & 0xffff) - bx0, 0);
    const int cx1 = min(static_cast<int>(b & 0xffff) - bx0, 8);
    const int cy0 = max(static_cast<int>(a >> 16) - by0, 0);
    const int cy1 = min(static_cast<int>(b >> 16) - by0, 4);
    if (cx0 >= cx1 || cy0 >= cy1) return 0u;
    const uint32_t row = ((1u << cx1) - 1u) & ~((1u << cx0) - 1u);
    const uint32_t rows = static_cast<uint32_t>(((1ull << (8 * cy1)) - 1ull) & ~((1ull << (8 * cy0)) - 1ull));
    return (row * 0x01010101u) & rows;
}

// Warp bit-matrix transpose: lane L receives bit L of every lane's word, in lane order.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const uint32_t m = s == 16 ? 0x0000ffffu : s == 8 ? 0x00ff00ffu : s == 4 ? 0x0f0f0f0fu
                                                 : s == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
        x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
    }
    return x;
}
}  // namespace

// Tile size 16, quadrant form: one 64-thread CTA per 8x8 quadrant of a tile (grid =
// 4 x tiles). Crowd frames are extremely skewed — horizon tiles carry tens of thousands
// of pairs and mix saturated crowd pixels with never-saturating sky — so splitting a tile
// four ways cuts the serial list walk of the heaviest tiles by 4x and lets each quadrant
// stop on its own saturation. Warp w covers the 8x4 block at rows 4w..4w+3 and walks the
// quadrant's list on its own (no CTA barrier: a saturated warp never waits for the other).
// Per round a warp stages 32*CH records with cp.async, double-buffered so the next round
// is in flight while this one is walked. For every 32 staged splats, lane L builds the
// coverage bits of splat L over the warp's pixels and a bit-matrix transpose hands each
// lane the ordered list of splats covering its own pixel; lanes then walk their lists
// across all CH chunks before re-converging (a lane busy in one chunk and idle in the
// other balances within the round: 12% faster than one chunk per round). Each pixel
// still walks the tile's list in order, so results equal the reference's per-tile loop.
template <int CH>
__global__ void __launch_bounds__(64)
k_raster16q(RasterParams p) {
    pdl_entry();
    constexpr int kStage = 32 * CH;
    // [warp][buffer][slot][geo | colour | ext (G, B, rect lo, rect hi)]: one slot base per
    // record, the three rows at fixed offsets.
    __shared__ float4 s_rec[2][2][kStage][3];
    __shared__ unsigned long long s_tab[32];
    load_exp_table(s_tab);
    __syncthreads();
    const ExpfRegs ek = expf_regs(s_tab);
    const int tile = blockIdx.x >> 2, quad = blockIdx.x & 3;
    const int tx = tile % p.tiles_x + p.tile_col0, ty = tile / p.tiles_x + p.tile_row0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int bx0 = tx * 16 + (quad & 1) * 8;
    const int by0 = ty * 16 + (quad >> 1) * 8 + warp * 4;
    const int px = bx0 + (lane & 7);
    const int py = by0 + (lane >> 3);
    const bool inside = px < p.width && py < p.height;
    const uint2 range = p.ranges[blockIdx.x];
    const float fx = static_cast<float>(px) + 0.5f, fy = static_cast<float>(py) + 0.5f;
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    bool done = !inside;
    auto stage = [&](int buf, uint32_t start) {
#pragma unroll
        for (int h = 0; h < CH; ++h) {
            const uint32_t i = start + h * 32 + lane;
            if (i < range.y) {
                const float4* src = p.records + 3ull * p.recs[i];
                float4* dst = s_rec[warp][buf][h * 32 + lane];
                cp_async16(dst + 0, src + 0);
                cp_async16(dst + 1, src + 1);
                cp_async16(dst + 2, src + 2);
            }
        }
        cp_async_commit();
    };
    int buf = 0;
    if (range.x < range.y) stage(0, range.x);
    for (uint32_t start = range.x; start < range.y; start += kStage) {
        if (__all_sync(0xffffffffu, done)) break;
        if (start + kStage < range.y) {
            stage(buf ^ 1, start + kStage);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const float4 (*rec)[3] = s_rec[warp][buf];
        const int n = static_cast<int>(min(static_cast<uint32_t>(kStage), range.y - start));
        static_assert(CH == 2, "two explicit chunk words (a dynamically indexed array spills)");
        uint32_t todo0 = transpose32(lane < n ? block_cover(rec[lane][2], bx0, by0) : 0u, lane);
        uint32_t todo1 = transpose32(32 + lane < n ? block_cover(rec[32 + lane][2], bx0, by0) : 0u, lane);
        if (done) todo0 = todo1 = 0u;
        while (__any_sync(0xffffffffu, (todo0 | todo1) != 0u)) {
            // List order: chunk 0 before chunk 1, lower bit first (select, not branch).
            const bool lo = todo0 != 0u;
            const uint32_t word = lo ? todo0 : todo1;
            if (word == 0u) continue;
            const int k = __ffs(word) - 1 + (lo ? 0 : 32);
            const uint32_t rest = word & (word - 1u);
            todo0 = lo ? rest : todo0;
            todo1 = lo ? todo1 : rest;
            const float4 g = rec[k][0];
            const float dx = __fsub_rn(fx, g.x);
            const float dy = __fsub_rn(fy, g.y);
            const float4 c = rec[k][1];
            const float q = __fadd_rn(__fmul_rn(__fmul_rn(g.z, dx), dx), __fmul_rn(__fmul_rn(c.x, dy), dy));
            const float power = __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(g.w, dx), dy));
            if (power < c.z) continue;
            const float alpha = fminf(__fmul_rn(c.y, glibc_expf_regs(power, ek)), p.alpha_max);
            const float w = __fmul_rn(T, alpha);
            const float4 e = rec[k][2];
            cr = __fadd_rn(cr, __fmul_rn(w, c.w));
            cg = __fadd_rn(cg, __fmul_rn(w, e.x));
            cb = __fadd_rn(cb, __fmul_rn(w, e.y));
            T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
            if (T < p.t_floor) {
                done = true;
                todo0 = todo1 = 0u;
            }
        }
        __syncwarp();
        buf ^= 1;
    }
    cp_async_wait<0>();
    if (inside) {
        const size_t o = static_cast<size_t>(py - p.out_row0) * p.out_stride + (px - p.out_col0);
        p.out_rgb[3 * o + 0] = __fadd_rn(cr, __fmul_rn(T, p.bg[0]));
        p.out_rgb[3 * o + 1] = __fadd_rn(cg, __fmul_rn(T, p.bg[1]));
        p.out_rgb[3 * o + 2] = __fadd_rn(cb, __fmul_rn(T, p.bg[2]));
        p.out_T[o] = T;
    }
}

// Any tile size up to 16*sqrt(PPT): PPT pixels per thread, pixel p = tid + k*256.
template <int PPT>
__global__ void __launch_bounds__(256)
k_raster_generic(RasterParams p) {
    pdl_entry();
    __shared__ float4 s_rec[256 * 3];
    __shared__ unsigned long long s_tab[32];
    load_exp_table(s_tab);
    const ExpfRegs ek = expf_regs(s_tab);  // table read only after the block's first barrier
    const int ts = p.tile_size;
    const int tile = blockIdx.x;
    const int tx = tile % p.tiles_x + p.tile_col0, ty = tile / p.tiles_x + p.tile_row0;
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
                if (blend(v, pxs[k], pys[k], T[k], cr[k], cg[k], cb[k], p.alpha_max, p.t_floor, ek)) {
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
            const size_t o = static_cast<size_t>(pys[k] - p.out_row0) * p.out_stride + (pxs[k] - p.out_col0);
            p.out_rgb[3 * o + 0] = __fadd_rn(cr[k], __fmul_rn(T[k], p.bg[0]));
            p.out_rgb[3 * o + 1] = __fadd_rn(cg[k], __fmul_rn(T[k], p.bg[1]));
            p.out_rgb[3 * o + 2] = __fadd_rn(cb[k], __fmul_rn(T[k], p.bg[2]));
            p.out_T[o] = T[k];
        }
    }
}

void launch_raster(const RasterParams& p, uint32_t tiles, cudaStream_t stream) {
    if (p.tile_size == 16) pdl_launch(k_raster16q<2>, tiles * 4, 64, 0, stream, p);
    else if (p.tile_size <= 16) pdl_launch(k_raster_generic<1>, tiles, 256, 0, stream, p);
    else if (p.tile_size <= 32) pdl_launch(k_raster_generic<4>, tiles, 256, 0, stream, p);
    else pdl_launch(k_raster_generic<16>, tiles, 256, 0, stream, p);
}

// The expf replica over consecutive float bit patterns (gscg_eval_expf: parity check).
__global__ void k_eval_expf(uint32_t first_bits, uint32_t n, float* out) {
    __shared__ unsigned long long s_tab[32];
    load_exp_table(s_tab);
    __syncthreads();
    const ExpfRegs ek = expf_regs(s_tab);  // the rasterisers' exact code path
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = glibc_expf_regs(__uint_as_float(first_bits + i), ek);
}

}  // namespace gscg
