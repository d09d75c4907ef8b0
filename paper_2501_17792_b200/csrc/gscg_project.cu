// Stage "gather" on the B200: fused LBS skinning + EWA projection + cull + conic + SH
// colour + tile-pair emission (reference: skin_means avatar.cpp:178-192 driven by
// crowd.cpp:126-131; gather_splats renderer.cpp:25-73 -> project_covariance
// math.cpp:131-170 and splat_bounds math.cpp:106-116; conic prep renderer.cpp:133-141;
// tile range renderer.cpp:153-157). Compiled with --fmad=false (parity-critical).
//
// Template-major schedule: a work item is (template-level group, chunk of 256
// Gaussians, batch of up to kBatch instances). A CTA loads the chunk's shared attributes
// once (registers + SH in shared memory) and re-uses them for every instance of the
// batch, so the shared store streams from HBM once per batch instead of once per
// instance (CrowdSplat's attribute sharing, moved on-chip). Survivors are compacted with
// a block scan and one 64-bit atomic per (CTA, instance); placement order is therefore
// schedule-dependent, but the sort's key order plus the ordinal tie fix-up make the
// per-tile lists and pixels deterministic.
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

// Real SH basis, degrees 1..3 (same constants and expression order as the oracle).
__device__ __forceinline__ void sh_basis(float x, float y, float z, float Y[15]) {
    const float C1 = 0.4886025119029199f;
    const float C20 = 1.0925484305920792f, C21 = -1.0925484305920792f,
                C22 = 0.31539156525252005f, C23 = -1.0925484305920792f,
                C24 = 0.5462742152960396f;
    const float C30 = -0.5900435899266435f, C31 = 2.890611442640554f,
                C32 = -0.4570457994644658f, C33 = 0.3731763325901154f,
                C34 = -0.4570457994644658f, C35 = 1.445305721320277f,
                C36 = -0.5900435899266435f;
    const float xx = x * x, yy = y * y, zz = z * z;
    const float xy = x * y, yz = y * z, xz = x * z;
    Y[0] = -C1 * y;
    Y[1] = C1 * z;
    Y[2] = -C1 * x;
    Y[3] = C20 * xy;
    Y[4] = C21 * yz;
    Y[5] = C22 * ((2.0f * zz - xx) - yy);
    Y[6] = C23 * xz;
    Y[7] = C24 * (xx - yy);
    Y[8] = (C30 * y) * (3.0f * xx - yy);
    Y[9] = (C31 * xy) * z;
    Y[10] = (C32 * y) * ((4.0f * zz - xx) - yy);
    Y[11] = (C33 * z) * ((2.0f * zz - 3.0f * xx) - 3.0f * yy);
    Y[12] = (C34 * x) * ((4.0f * zz - xx) - yy);
    Y[13] = (C35 * z) * (xx - yy);
    Y[14] = (C36 * x) * (xx - 3.0f * yy);
}

}  // namespace

template <bool kPosedIn, bool kNaive>
__global__ void __launch_bounds__(kProjectThreads, 4)
k_project(ProjectParams p) {
    pdl_entry();
    extern __shared__ float4 s_dyn[];
    float* s_sh = reinterpret_cast<float*>(s_dyn);
    float* s_mats = s_sh + (p.sh_enabled ? kProjectThreads * kShFloats : 0);
    __shared__ uint32_t s_item_start[kMaxGroups + 1];
    __shared__ uint32_t s_member[kBatch], s_member_base[kBatch];  // batch instance ids, ordinal bases
    __shared__ uint32_t s_wcnt[kProjectThreads / 32];
    __shared__ unsigned long long s_base;
    __shared__ uint32_t s_item;
    __shared__ uint32_t s_tile_pairs;  // the reference's (tile, splat) bin entries of this CTA
    __shared__ __align__(8) uint64_t s_bar;  // the work item's bulk copies (SH + skin matrices)

    const int tid = threadIdx.x;
    for (uint32_t g = tid; g <= p.group_count; g += blockDim.x) s_item_start[g] = p.group_item_start[g];
    const uint32_t items_total = p.counters->items_total;
    const CameraDev& cam = p.cam;
    // Binning cell (pairs per splat are counted here; emitted after the depth sort):
    // the tile, or for 16-px tiles each 8x8 quadrant.
    const int cell = p.tile_size == 16 ? 8 : p.tile_size;
    const int cshift = (cell & (cell - 1)) == 0 ? __ffs(cell) - 1 : -1;
    auto cdiv = [&](int v) { return cshift >= 0 ? v >> cshift : v / cell; };  // v >= 0
    uint32_t dmin = 0xffffffffu, dmax = 0u;
    uint32_t pairs = 0;  // binning cells of this thread's splats (summed once at the end)
    const int lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        s_tile_pairs = 0u;
    }
    uint32_t phase = 0;

    for (;;) {
        __syncthreads();
        if (tid == 0) s_item = atomicAdd(&p.counters->item_cursor, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        if (item >= items_total) break;

        // Group: last g with item_start[g] <= item.
        uint32_t lo = 0, hi = p.group_count;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_item_start[mid] <= item) lo = mid; else hi = mid;
        }
        const uint32_t g = lo;
        const GroupDev grp = p.groups[g];
        const uint32_t local = item - s_item_start[g];
        const uint32_t chunks = (grp.count + kProjectThreads - 1) / kProjectThreads;
        const uint32_t chunk = local % chunks, batch = local / chunks;
        const uint32_t gi = chunk * kProjectThreads + tid;
        const bool gvalid = gi < grp.count;

        float4 c0 = make_float4(0, 0, 0, 0), c1 = c0, c2 = c0, c3 = c0, wv = c0;
        if (gvalid && !kNaive) {
            c0 = grp.core[4 * gi + 0];
            c1 = grp.core[4 * gi + 1];
            c2 = grp.core[4 * gi + 2];
            c3 = grp.core[4 * gi + 3];
            wv = grp.weights[gi];
        }
        const bool use_sh = p.sh_enabled && grp.sh != nullptr;
        // Stage the chunk's SH coefficients and every batch instance's skin matrices with
        // bulk copies (TMA engine), once per work item: thread 0 the SH block, thread k
        // instance k's matrices, all completing on s_bar.
        const uint32_t inst_begin = p.group_inst_start[g] + batch * kBatch;
        const uint32_t inst_count = min(static_cast<uint32_t>(kBatch),
                                        p.group_inst_count[g] - batch * kBatch);
        const uint32_t mat_bytes = p.joint_stride * 48u;  // 3 x 4 floats per joint
        if (tid == 0) {
            // Earlier generic-proxy reads of this shared memory precede the async writes.
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            uint32_t bytes = inst_count * mat_bytes;
            if (use_sh) {
                const uint32_t n_here = min(static_cast<uint32_t>(kProjectThreads),
                                            grp.count - chunk * kProjectThreads);
                const uint32_t sh_bytes = (n_here * kShFloats * 4u + 15u) & ~15u;  // chunks are padded
                bytes += sh_bytes;
                mbar_arrive_expect_tx(&s_bar, bytes);
                bulk_g2s(s_sh, grp.sh + static_cast<size_t>(chunk) * kProjectThreads * kShFloats, sh_bytes, &s_bar);
            } else {
                mbar_arrive_expect_tx(&s_bar, bytes);
            }
        }
        if (tid < static_cast<int>(inst_count)) {
            const uint32_t m = p.members[inst_begin + tid];
            s_member[tid] = m;
            s_member_base[tid] = p.inst_base[m];
            if (tid != 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_g2s(s_mats + tid * p.joint_stride * 12, p.skin + static_cast<size_t>(m) * p.joint_stride * 12,
                     mat_bytes, &s_bar);
        }
        __syncthreads();
        mbar_wait(&s_bar, phase);
        phase ^= 1u;
        uint32_t i01 = __float_as_uint(c3.z), i23 = __float_as_uint(c3.w);
        float wk[4] = {wv.x, wv.y, wv.z, wv.w};

        for (uint32_t k = 0; k < inst_count; ++k) {
            if (kNaive && gvalid) {
                // Naive layout (the config-5 ablation): every instance reads its own copy of
                // the level's attributes, stored at its ordinals (instance base + index).
                const size_t o = static_cast<size_t>(s_member_base[k]) + gi;
                c0 = p.naive_core[4 * o + 0];
                c1 = p.naive_core[4 * o + 1];
                c2 = p.naive_core[4 * o + 2];
                c3 = p.naive_core[4 * o + 3];
                wv = p.naive_weights[o];
                i01 = __float_as_uint(c3.z);
                i23 = __float_as_uint(c3.w);
                wk[0] = wv.x;
                wk[1] = wv.y;
                wk[2] = wv.z;
                wk[3] = wv.w;
            }
            const uint32_t jidx[4] = {i01 & 0xffffu, i01 >> 16, i23 & 0xffffu, i23 >> 16};
            const uint32_t inst = s_member[k];
            const float* s_inst = s_mats + k * p.joint_stride * 12;

            bool survive = false;
            uint32_t n_tiles = 0, n_bins = 0;
            float mx = 0, my = 0, depth = 0, cxx = 0, cxy = 0, cyy = 0, ca = 0, cb = 0, cc = 0;
            float col0 = 0, col1 = 0, col2 = 0;
            int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
            uint32_t span_lo = 0, span_hi = 0;
            float ax = 0.0f, ay = 0.0f, az = 0.0f;
            if (gvalid && kPosedIn) {  // posed means given (gather_splats after update_crowd)
                const size_t o = 3ull * (s_member_base[k] + gi);
                ax = p.posed_in[o + 0];
                ay = p.posed_in[o + 1];
                az = p.posed_in[o + 2];
            }
            if (gvalid) {
                // Linear blend skinning (avatar.cpp:182-190), accumulator starts at +0.
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (kPosedIn) break;
                    if (wk[q] == 0.0f) continue;
                    const float4* S = reinterpret_cast<const float4*>(s_inst + jidx[q] * 12);  // 3 rows, 48-B aligned
                    const float4 r0 = S[0], r1 = S[1], r2 = S[2];
                    const float vx = ((r0.x * c0.x + r0.y * c0.y) + r0.z * c0.z) + r0.w * 1.0f;
                    const float vy = ((r1.x * c0.x + r1.y * c0.y) + r1.z * c0.z) + r1.w * 1.0f;
                    const float vz = ((r2.x * c0.x + r2.y * c0.y) + r2.z * c0.z) + r2.w * 1.0f;
                    ax = ax + wk[q] * vx;
                    ay = ay + wk[q] * vy;
                    az = az + wk[q] * vz;
                }
                // EWA projection (math.cpp:131-170).
                const bool finite_in = isfinite(ax) && isfinite(ay) && isfinite(az) &&
                                       isfinite(c1.x) && isfinite(c1.y) && isfinite(c1.z) &&
                                       isfinite(c1.w) && isfinite(c2.x) && isfinite(c2.y);
                const float dx = ax - cam.pos[0], dy = ay - cam.pos[1], dz = az - cam.pos[2];
                const float tx = cam.w[0] * dx + (cam.w[1] * dy + cam.w[2] * dz);
                const float ty = cam.w[3] * dx + (cam.w[4] * dy + cam.w[5] * dz);
                const float tz = cam.w[6] * dx + (cam.w[7] * dy + cam.w[8] * dz);
                if (finite_in && tz > cam.near_m) {
                    const float f = cam.focal;
                    const float iz = 1.0f / tz;
                    mx = (f * tx) * iz + cam.cx;
                    my = (f * ty) * iz + cam.cy;
                    const float j00 = f * iz, j01 = 0.0f, j02 = ((-f * tx) * iz) * iz;
                    const float j10 = 0.0f, j11 = f * iz, j12 = ((-f * ty) * iz) * iz;
                    // m = J * W (2x3)
                    float m[2][3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        m[0][c] = j00 * cam.w[0 * 3 + c] + (j01 * cam.w[1 * 3 + c] + j02 * cam.w[2 * 3 + c]);
                        m[1][c] = j10 * cam.w[0 * 3 + c] + (j11 * cam.w[1 * 3 + c] + j12 * cam.w[2 * 3 + c]);
                    }
                    const float S3[3][3] = {{c1.x, c1.y, c1.z}, {c1.y, c1.w, c2.x}, {c1.z, c2.x, c2.y}};
                    float A[2][3];
#pragma unroll
                    for (int r = 0; r < 2; ++r)
#pragma unroll
                        for (int c = 0; c < 3; ++c)
                            A[r][c] = m[r][0] * S3[0][c] + (m[r][1] * S3[1][c] + m[r][2] * S3[2][c]);
                    float C[2][2];
#pragma unroll
                    for (int i = 0; i < 2; ++i)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            C[i][j] = A[i][0] * m[j][0] + (A[i][1] * m[j][1] + A[i][2] * m[j][2]);
                    C[0][0] = C[0][0] + 0.3f;
                    C[1][1] = C[1][1] + 0.3f;
                    const float rx = 3.0f * sqrtf(C[0][0]);
                    const float ry = 3.0f * sqrtf(C[1][1]);
                    x0 = max(0, x86_float_to_int(floorf(mx - rx)));
                    y0 = max(0, x86_float_to_int(floorf(my - ry)));
                    x1 = min(cam.width, x86_float_to_int(floorf(mx + rx)) + 1);
                    y1 = min(cam.height, x86_float_to_int(floorf(my + ry)) + 1);
                    // A band frame keeps the splats whose rect meets its rows (renderer.cpp
                    // bins by rect, :147-161); the whole frame is the band [0, height).
                    if (x0 < x1 && y0 < y1 && y0 < cam.band_y1 && y1 > cam.band_y0 && x0 < cam.band_x1 &&
                        x1 > cam.band_x0) {
                        survive = true;
                        cxx = C[0][0];
                        cxy = 0.5f * (C[0][1] + C[1][0]);
                        cyy = C[1][1];
                        depth = tz;
                        // Conic (renderer.cpp:136-140).
                        const float det = cxx * cyy - cxy * cxy;
                        const float inv_det = 1.0f / det;
                        ca = cyy * inv_det;
                        cb = -cxy * inv_det;
                        cc = cxx * inv_det;
                        // Binning cells of the rect: first cell, cells across, cells down.
                        const int cxb = cdiv(cam.band_x0), cyb = cdiv(cam.band_y0);  // region's first cell
                        const int cx0 = cdiv(max(x0, cam.band_x0)) - cxb, cx1 = cdiv(min(x1, cam.band_x1) - 1) - cxb;
                        const int cy0 = cdiv(max(y0, cam.band_y0)) - cyb, cy1 = cdiv(min(y1, cam.band_y1) - 1) - cyb;
                        n_tiles = static_cast<uint32_t>((cx1 - cx0 + 1) * (cy1 - cy0 + 1));
                        span_lo = static_cast<uint32_t>(cx0) | (static_cast<uint32_t>(cy0) << 16);
                        span_hi = static_cast<uint32_t>(cx1 - cx0 + 1) | (static_cast<uint32_t>(cy1 - cy0 + 1) << 16);
                        n_bins = cell == p.tile_size ? n_tiles
                                                     : static_cast<uint32_t>(((cx1 >> 1) - (cx0 >> 1) + 1) *
                                                                             ((cy1 >> 1) - (cy0 >> 1) + 1));
                        col0 = c2.z;
                        col1 = c2.w;
                        col2 = c3.x;
                        if (use_sh) {
                            // SH residual colour: dir = normalize(mean - cam).
                            const float vx = ax - cam.pos[0], vy = ay - cam.pos[1], vz = az - cam.pos[2];
                            // One MUFU.RSQ instead of an IEEE sqrt and three IEEE
                            // divisions (colour tolerance, see below).
                            const float inrm = rsqrtf(vx * vx + (vy * vy + vz * vz));
                            float Y[15];
                            sh_basis(vx * inrm, vy * inrm, vz * inrm, Y);
                            const float* sh = s_sh + tid * kShFloats;
                            // Colour only reaches pixels (1e-3 tolerance), never the
                            // bit-exact geometry: fused multiply-adds here (colours agree
                            // with the oracle to ~1e-7).
#pragma unroll
                            for (int q = 0; q < 15; ++q) {
                                col0 = fmaf(Y[q], sh[3 * q + 0], col0);
                                col1 = fmaf(Y[q], sh[3 * q + 1], col1);
                                col2 = fmaf(Y[q], sh[3 * q + 2], col2);
                            }
                            col0 = fmaxf(col0, 0.0f);
                            col1 = fmaxf(col1, 0.0f);
                            col2 = fmaxf(col2, 0.0f);
                        }
                    }
                }
            }

            // Record slots: ballot ranks inside the warp, warp counts across the CTA, one
            // atomic per (CTA, instance) on the frame's splat counter.
            pairs += n_tiles;
            // Tile pairs (= pairs unless quadrant cells) are warp-reduced into shared memory
            // here rather than carried in a register (the kernel sits at its 64-register cap).
            const uint32_t wbins = __reduce_add_sync(0xffffffffu, n_bins);
            if (lane == 0 && wbins) atomicAdd(&s_tile_pairs, wbins);
            const uint32_t bal = __ballot_sync(0xffffffffu, survive);
            if (lane == 0) s_wcnt[warp] = __popc(bal);
            __syncthreads();
            uint32_t before = 0, total = 0;
#pragma unroll
            for (int w = 0; w < kProjectThreads / 32; ++w) {
                const uint32_t t = s_wcnt[w];
                before += w < warp ? t : 0u;
                total += t;
            }
            if (tid == 0) s_base = atomicAdd(&p.counters->splats, static_cast<unsigned long long>(total));
            __syncthreads();
            const unsigned long long base = s_base;
            const uint32_t ordinal = gvalid ? s_member_base[k] + gi : 0u;
            if (p.posed_debug && gvalid) {
                p.posed_debug[3ull * ordinal + 0] = ax;
                p.posed_debug[3ull * ordinal + 1] = ay;
                p.posed_debug[3ull * ordinal + 2] = az;
            }
            const uint64_t ridx = base + before + __popc(bal & lt);
            const uint32_t dbits = __float_as_uint(depth);
            const bool stored = survive && ridx < p.splat_capacity;
            if (survive) {
                dmin = min(dmin, dbits);
                dmax = max(dmax, dbits);
                if (stored) {
                    float4* rec = p.records + 3 * ridx;
                    rec[0] = make_float4(mx, my, ca, cb);
                    rec[1] = make_float4(cc, c0.w, c3.y, col0);
                    rec[2] = make_float4(col1, col2,
                                         __uint_as_float(static_cast<uint32_t>(x0) | (static_cast<uint32_t>(y0) << 16)),
                                         __uint_as_float(static_cast<uint32_t>(x1) | (static_cast<uint32_t>(y1) << 16)));
                    if (p.record_debug) {
                        gscg_splat_record d;
                        d.ordinal = ordinal;
                        d.instance_id = inst;
                        d.gaussian_index = gi;
                        d.depth = depth;
                        d.mean_px[0] = mx;
                        d.mean_px[1] = my;
                        d.cov_xx = cxx;
                        d.cov_xy = cxy;
                        d.cov_yy = cyy;
                        d.conic[0] = ca;
                        d.conic[1] = cb;
                        d.conic[2] = cc;
                        d.power_floor = c3.y;
                        d.opacity = c0.w;
                        d.color[0] = col0;
                        d.color[1] = col1;
                        d.color[2] = col2;
                        d.rect[0] = x0;
                        d.rect[1] = y0;
                        d.rect[2] = x1;
                        d.rect[3] = y1;
                        p.record_debug[ridx] = d;
                    }
                }
            }
            if (stored) {
                p.splat_depth[ridx] = dbits;  // splat sort key (pairs are emitted after it)
                p.splat_meta[ridx] = make_uint4(ordinal, span_lo, span_hi, dbits);
            }
        }
    }

    // Depth-bit range of the frame (sort pass planning).
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    pairs = __reduce_add_sync(0xffffffffu, pairs);
    if (tid == 0 && s_tile_pairs) atomicAdd(&p.counters->tile_pairs, static_cast<unsigned long long>(s_tile_pairs));
    if ((tid & 31) == 0) {
        if (dmin != 0xffffffffu) atomicMin(&p.counters->depth_min_bits, dmin);
        if (dmax != 0u) atomicMax(&p.counters->depth_max_bits, dmax);
        if (pairs) atomicAdd(&p.counters->pairs, static_cast<unsigned long long>(pairs));
    }
}

// Power floor column (core[4g+3].y) = logf(alpha_cutoff / opacity), computed on the host
// with glibc exactly as the reference's conic prep does (renderer.cpp:140).
__global__ void k_set_power_floor(float4* core, const float* pf, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) core[4 * i + 3].y = pf[i];
}

template __global__ void k_project<false, false>(ProjectParams p);
template __global__ void k_project<true, false>(ProjectParams p);
template __global__ void k_project<false, true>(ProjectParams p);

// Naive-layout copies (config-5 ablation): instance i's level attributes at its ordinals.
__global__ void k_naive_fill(const uint32_t* inst_group, const uint32_t* inst_base, const GroupDev* groups, uint32_t n,
                             float4* core, float4* weights) {
    for (uint32_t inst = blockIdx.y; inst < n; inst += gridDim.y) {
        const GroupDev g = groups[inst_group[inst]];
        const size_t base = inst_base[inst];
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < g.count; i += gridDim.x * blockDim.x) {
#pragma unroll
            for (int j = 0; j < 4; ++j) core[4 * (base + i) + j] = g.core[4 * i + j];
            weights[base + i] = g.weights[i];
        }
    }
}

}  // namespace gscg
