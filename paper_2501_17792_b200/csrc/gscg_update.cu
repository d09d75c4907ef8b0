// Stage "update" of render_frame on the B200 (reference: update_crowd,
// /root/reference/proj/src/crowd.cpp:86-140). Compiled with --fmad=false.
//
//  k_lod_plan  — one CTA: per-instance LoD (lod.cpp:22-41, crowd.cpp:93-110), the
//                instance-Gaussian ordinal base of every instance (exclusive scan in
//                instance order), the stable (template, level) grouping of instances
//                and the template-major work-item table the projection kernel consumes.
//  k_fk_skin   — half a warp per instance: forward kinematics and skin matrices
//                (avatar.cpp:149-176, crowd.cpp:20-30, 126-128), one matrix element
//                per lane, Eigen's packet product order.
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

constexpr int kPlanThreads = 1024;

template <typename T>
__device__ T block_exclusive_scan(T v, T* s_warp, T& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nwarps ? s_warp[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nwarps) s_warp[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    const T warp_excl = warp == 0 ? T(0) : s_warp[warp - 1];
    total = s_warp[nwarps - 1];
    __syncthreads();
    return warp_excl + x - v;
}

}  // namespace

__global__ void __launch_bounds__(kPlanThreads)
k_lod_plan(PlanParams p) {
    pdl_entry();
    __shared__ unsigned long long s_scan64[32];
    __shared__ uint32_t s_scan32[32];
    __shared__ uint32_t s_gcount[kMaxGroups];
    __shared__ uint32_t s_gstart[kMaxGroups];
    __shared__ uint32_t s_carry[kMaxGroups];
    __shared__ uint32_t s_tile_total[kMaxGroups];
    __shared__ uint32_t s_wcount[32][kMaxGroups];

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    for (int g = tid; g < kMaxGroups; g += blockDim.x) {
        s_gcount[g] = 0;
        s_carry[g] = 0;
    }
    if (tid == 0) {
        p.counters->splats = 0ull;
        p.counters->pairs = 0ull;
        p.counters->tile_pairs = 0ull;
        p.counters->depth_min_bits = 0xffffffffu;
        p.counters->depth_max_bits = 0u;
        p.counters->item_cursor = 0u;
        p.counters->instances_culled = 0u;
        for (int q = 0; q < 8; ++q) p.counters->sort_ticket[q] = 0u;
    }
    __syncthreads();

    // Pass 1: LoD, group, per-instance Gaussian count; ordinal bases by block scan.
    unsigned long long carry = 0ull;
    for (uint32_t tile = 0; tile < p.n; tile += kPlanThreads) {
        const uint32_t i = tile + tid;
        uint32_t count = 0;
        if (i < p.n) {
            const uint32_t t = p.template_ids[i];
            const TemplateDev tpl = p.templates[t];
            const uint32_t levels = static_cast<uint32_t>(tpl.level_count);
            uint32_t lod;
            if (p.forced_lod >= 0) {
                lod = min(static_cast<uint32_t>(p.forced_lod), levels - 1u);
            } else if (p.forced_lod == GSCG_LOD_GIVEN) {  // the caller's active_lod (renderer.cpp:38-40)
                const uint32_t given = p.lod_prev[i];
                lod = min(given == 0xffffffffu ? 0u : given, levels - 1u);
            } else {
                // instance_distance((x, pelvis.y, z), camera.position): Eigen half-split norm.
                const float dx = p.placement[4 * i + 0] - p.cam_pos[0];
                const float dy = tpl.pelvis_y - p.cam_pos[1];
                const float dz = p.placement[4 * i + 1] - p.cam_pos[2];
                const float sq = dx * dx + (dy * dy + dz * dz);
                const float dist = sqrtf(sq);
                const uint32_t prev = p.lod_prev[i];
                uint32_t sel = p.threshold_count;
                for (uint32_t k = 0; k < p.threshold_count; ++k) {
                    float th = p.thresholds[k];
                    if (prev != 0xffffffffu && p.hysteresis > 0.0f)
                        th = th + (k >= prev ? 0.5f : -0.5f) * p.hysteresis;
                    if (dist < th) {
                        sel = k;
                        break;
                    }
                }
                lod = min(sel, levels - 1u);
            }
            const uint32_t g = static_cast<uint32_t>(tpl.group_base) + lod;
            p.lod_out[i] = lod;
            p.inst_group[i] = g;
            count = p.groups[g].count;
            // Every rank numbers the whole crowd (ordinals are global); only its own
            // instance shard is projected.
            if (i >= p.shard_begin && i < p.shard_end) {
                if (!p.visible || p.visible[i]) atomicAdd(&s_gcount[g], 1u);
                else atomicAdd(&p.counters->instances_culled, 1u);
            }
        }
        unsigned long long total;
        const unsigned long long excl =
            block_exclusive_scan<unsigned long long>(count, s_scan64, total);
        if (i < p.n) p.inst_base[i] = static_cast<uint32_t>(carry + excl);
        carry += total;
    }
    if (tid == 0) p.counters->gaussians = carry;
    __syncthreads();

    // Group starts and work items (template-major: chunks of 256 Gaussians x batches).
    {
        uint32_t cnt = 0, items = 0;
        if (tid < static_cast<int>(p.group_count)) {
            cnt = s_gcount[tid];
            const uint32_t N = p.groups[tid].count;
            const uint32_t chunks = (N + kProjectThreads - 1) / kProjectThreads;
            const uint32_t batches = (cnt + kBatch - 1) / kBatch;
            items = cnt ? chunks * batches : 0u;
        }
        uint32_t tot_c, tot_i;
        const uint32_t ex_c = block_exclusive_scan<uint32_t>(cnt, s_scan32, tot_c);
        const uint32_t ex_i = block_exclusive_scan<uint32_t>(items, s_scan32, tot_i);
        if (tid < static_cast<int>(p.group_count)) {
            s_gstart[tid] = ex_c;
            p.group_inst_start[tid] = ex_c;
            p.group_inst_count[tid] = cnt;
            p.group_item_start[tid] = ex_i;
        }
        if (tid == 0) {
            p.group_inst_start[p.group_count] = tot_c;
            p.group_item_start[p.group_count] = tot_i;
            p.counters->items_total = tot_i;
        }
    }
    __syncthreads();

    // Pass 2: stable counting scatter of instance ids into their groups.
    for (uint32_t tile = 0; tile < p.n; tile += kPlanThreads) {
        for (int k = tid; k < 32 * kMaxGroups; k += blockDim.x) (&s_wcount[0][0])[k] = 0u;
        __syncthreads();
        const uint32_t i = tile + tid;
        const bool valid = i < p.n && i >= p.shard_begin && i < p.shard_end && (!p.visible || p.visible[i]);
        const uint32_t g = valid ? p.inst_group[i] : 0xffffffffu;
        const uint32_t peers = __match_any_sync(0xffffffffu, g);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        if (valid && lane == __ffs(peers) - 1) s_wcount[warp][g] = __popc(peers);
        __syncthreads();
        if (tid < static_cast<int>(p.group_count)) {
            uint32_t run = 0;
            for (int w = 0; w < 32; ++w) {
                const uint32_t c = s_wcount[w][tid];
                s_wcount[w][tid] = run;
                run += c;
            }
            s_tile_total[tid] = run;
        }
        __syncthreads();
        if (valid) p.members[s_gstart[g] + s_carry[g] + s_wcount[warp][g] + rank] = i;
        __syncthreads();
        if (tid < static_cast<int>(p.group_count)) s_carry[tid] += s_tile_total[tid];
        __syncthreads();
    }
}

// Element (r, c) of a column-major 4x4 product A*B given A's row r and B's column c:
// Eigen's packet chain ((a0*b0 + a1*b1) + a2*b2) + a3*b3, no FMA.
__device__ __forceinline__ float chain4(float a0, float a1, float a2, float a3, float b0, float b1,
                                        float b2, float b3) {
    float acc = a0 * b0;
    acc = acc + a1 * b1;
    acc = acc + a2 * b2;
    acc = acc + a3 * b3;
    return acc;
}

// Element (r, c) of rotation_matrix(q) (avatar.cpp:19-23): Eigen toRotationMatrix in the
// top-left 3x3 block, identity elsewhere.
__device__ __forceinline__ float rot_elem(const float4 q, int r, int c) {
    if (r == 3 || c == 3) return (r == c) ? 1.0f : 0.0f;
    const float tx = 2.0f * q.x, ty = 2.0f * q.y, tz = 2.0f * q.z;
    const float twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
    const float txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
    const float tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
    const int k = r * 3 + c;
    switch (k) {
        case 0: return 1.0f - (tyy + tzz);
        case 1: return txy - twz;
        case 2: return txz + twy;
        case 3: return txy + twz;
        case 4: return 1.0f - (txx + tzz);
        case 5: return tyz - twx;
        case 6: return txz - twy;
        case 7: return tyz + twx;
        default: return 1.0f - (txx + tyy);
    }
}

__global__ void __launch_bounds__(kFkThreads)
k_fk_skin(FkParams p) {
    pdl_entry();
    // Per half-warp (one instance): world[J][16], then the instance's local_bind and
    // inverse_bind matrices and pose quaternions, staged once so the joint chain below
    // runs from shared memory instead of paying a global-memory latency per joint.
    extern __shared__ __align__(16) float s_world[];
    const int half = threadIdx.x >> 4;        // half-warp within the block
    const int l = threadIdx.x & 15;           // matrix element, column-major
    const int r = l & 3, c = l >> 2;
    const uint32_t inst = p.first + blockIdx.x * (blockDim.x >> 4) + half;
    const unsigned hmask = 0xffffu << ((threadIdx.x & 31) & 16);
    if (inst >= p.n) return;
    const int js = static_cast<int>(p.joint_stride);
    float* world = s_world + static_cast<size_t>(half) * js * 52;
    float* slb = world + js * 16;
    float* sib = slb + js * 16;
    float* sq = sib + js * 16;

    const TemplateDev tpl = p.templates[p.template_ids[inst]];
    const int J = tpl.joint_count;
    const float4* lb = reinterpret_cast<const float4*>(p.mats + static_cast<size_t>(tpl.mat_offset) * 16);
    const float4* ib = lb + static_cast<size_t>(J) * 4;
    const int32_t* parents = p.parents + tpl.parent_offset;
    const float* pose = p.poses + static_cast<size_t>(inst) * p.pose_stride;
    for (int k = l; k < J * 4; k += 16) {  // all loads in flight at once
        reinterpret_cast<float4*>(slb)[k] = lb[k];
        reinterpret_cast<float4*>(sib)[k] = ib[k];
    }
    for (int k = l; k < J * 4; k += 16) sq[k] = pose[4 + k];
    __syncwarp(hmask);

    // Root transform (crowd.cpp:20-30) and root offset T(root_translation).
    const float x = p.placement[4 * inst + 0], z = p.placement[4 * inst + 1];
    const float cs = p.placement[4 * inst + 2], sn = p.placement[4 * inst + 3];
    auto root_elem = [&](int rr, int cc) -> float {
        if (rr == 0 && cc == 0) return cs;
        if (rr == 0 && cc == 2) return sn;
        if (rr == 2 && cc == 0) return -sn;
        if (rr == 2 && cc == 2) return cs;
        if (rr == 0 && cc == 3) return x;
        if (rr == 2 && cc == 3) return z;
        return rr == cc ? 1.0f : 0.0f;
    };
    auto offset_elem = [&](int rr, int cc) -> float {
        if (cc == 3 && rr < 3) return pose[rr];
        return rr == cc ? 1.0f : 0.0f;
    };
    const float m0 = chain4(root_elem(r, 0), root_elem(r, 1), root_elem(r, 2), root_elem(r, 3),
                            offset_elem(0, c), offset_elem(1, c), offset_elem(2, c),
                            offset_elem(3, c));

    float* out = p.skin + static_cast<size_t>(inst) * p.joint_stride * 12;
    for (int j = 0; j < J; ++j) {
        const float4 q = reinterpret_cast<const float4*>(sq)[j];
        const float* LB = slb + j * 16;
        // local = local_bind[j] * rotation_matrix(q)
        const float local = chain4(LB[0 * 4 + r], LB[1 * 4 + r], LB[2 * 4 + r], LB[3 * 4 + r],
                                   rot_elem(q, 0, c), rot_elem(q, 1, c), rot_elem(q, 2, c),
                                   rot_elem(q, 3, c));
        // local(k, c) lives in lane c*4 + k of this half-warp.
        const float lk0 = __shfl_sync(hmask, local, c * 4 + 0, 16);
        const float lk1 = __shfl_sync(hmask, local, c * 4 + 1, 16);
        const float lk2 = __shfl_sync(hmask, local, c * 4 + 2, 16);
        const float lk3 = __shfl_sync(hmask, local, c * 4 + 3, 16);
        float pr0, pr1, pr2, pr3;  // parent row r
        if (j == 0) {
            pr0 = __shfl_sync(hmask, m0, 0 * 4 + r, 16);
            pr1 = __shfl_sync(hmask, m0, 1 * 4 + r, 16);
            pr2 = __shfl_sync(hmask, m0, 2 * 4 + r, 16);
            pr3 = __shfl_sync(hmask, m0, 3 * 4 + r, 16);
        } else {
            const float* P = world + parents[j] * 16;
            pr0 = P[0 * 4 + r];
            pr1 = P[1 * 4 + r];
            pr2 = P[2 * 4 + r];
            pr3 = P[3 * 4 + r];
        }
        const float wv = chain4(pr0, pr1, pr2, pr3, lk0, lk1, lk2, lk3);
        world[j * 16 + l] = wv;
        __syncwarp(hmask);
        // skin = world[j] * inverse_bind[j]
        const float* IB = sib + j * 16;
        const float* W = world + j * 16;
        const float sv = chain4(W[0 * 4 + r], W[1 * 4 + r], W[2 * 4 + r], W[3 * 4 + r],
                                IB[c * 4 + 0], IB[c * 4 + 1], IB[c * 4 + 2], IB[c * 4 + 3]);
        if (r < 3) out[j * 12 + r * 4 + c] = sv;
    }
}

// Instance frustum cull. An instance is dropped from the projection work table only when
// no Gaussian of it can survive gather_splats' cull (renderer.cpp:38-50: t.z > near and a
// non-empty clipped 3-sigma rect), so the splat set, and everything after it, is unchanged.
//
// Ball of the posed means. posed = sum_k w_k (A_k m + t_k) over the nonzero weights
// (avatar.cpp:182-190), with S_k = [A_k | t_k] the skin matrix. For any centre c:
//   |posed - c| <= sum|w_k| (|A_k|_2 |m| + |t_k - c|) + |sum w_k - 1| |c|
//               <= wabs (Amax mean_r + Tmax) + wdev |c|
// with c the centre of the box of the joint translations, Tmax = max_j |t_j - c|,
// |A_j|_2^2 <= max row sum of |A_j^T A_j| and the template bounds (TemplateDev).
//
// Rect of a splat at camera-space t (math.cpp:131-170): rx = 3 sqrt(C00) with
// C00 = m0 S m0^T + 0.3 and m0 = (f/tz)(W0 - (tx/tz) W2), so
//   rx <= 3 (f/tz) |W0 - (tx/tz) W2| sigma + 3 sqrt(0.3)
// (sigma^2 >= lambda_max of every covariance). The rect is empty on the left when
// mx + rx < 0, on the right when mx - rx >= width (same for y). The test bounds tx/tz over
// the ball in double precision with relative and pixel margins far above the float
// rounding of the projection itself. Non-finite bounds never cull.
__global__ void __launch_bounds__(256)
k_inst_cull(CullParams p) {
    pdl_entry();
    const int lane = threadIdx.x & 31;
    const uint32_t inst = p.first + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (inst >= p.n) return;
    const TemplateDev tpl = p.templates[p.template_ids[inst]];
    const int J = tpl.joint_count;
    const float4* S = reinterpret_cast<const float4*>(p.skin + static_cast<size_t>(inst) * p.joint_stride * 12);
    float tmin[3] = {INFINITY, INFINITY, INFINITY}, tmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    float a2 = 0.0f;
    float tj[2][3];
    for (int r = 0; r < 2; ++r) for (int k = 0; k < 3; ++k) tj[r][k] = 0.0f;
    bool bad = false;  // a non-finite matrix entry: never cull
    for (int j = lane, r = 0; r < 2; j += 32, ++r) {  // joint_count <= 64 (GSCG_MAX_JOINTS)
        if (j >= J) break;
        const float4 r0 = S[3 * j + 0], r1 = S[3 * j + 1], r2 = S[3 * j + 2];
        const float t[3] = {r0.w, r1.w, r2.w};
        for (int k = 0; k < 3; ++k) {
            tj[r][k] = t[k];
            tmin[k] = fminf(tmin[k], t[k]);
            tmax[k] = fmaxf(tmax[k], t[k]);
            bad |= !isfinite(t[k]);
        }
        // G = A^T A; |A|_2^2 = lambda_max(G) <= max row sum of |G|.
        const double a[3][3] = {{r0.x, r0.y, r0.z}, {r1.x, r1.y, r1.z}, {r2.x, r2.y, r2.z}};
        double rowmax = 0.0;
        for (int u = 0; u < 3; ++u) {
            double row = 0.0;
            for (int v = 0; v < 3; ++v) row += fabs(a[0][u] * a[0][v] + a[1][u] * a[1][v] + a[2][u] * a[2][v]);
            rowmax = fmax(rowmax, row);
        }
        bad |= !(rowmax <= 1e30);
        a2 = fmaxf(a2, static_cast<float>(rowmax * (1.0 + 1e-6)));
    }
    bad = __any_sync(0xffffffffu, bad);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        for (int k = 0; k < 3; ++k) {
            tmin[k] = fminf(tmin[k], __shfl_xor_sync(0xffffffffu, tmin[k], o));
            tmax[k] = fmaxf(tmax[k], __shfl_xor_sync(0xffffffffu, tmax[k], o));
        }
        a2 = fmaxf(a2, __shfl_xor_sync(0xffffffffu, a2, o));
    }
    double c[3];
    for (int k = 0; k < 3; ++k) c[k] = 0.5 * (static_cast<double>(tmin[k]) + static_cast<double>(tmax[k]));
    double T = 0.0;
    for (int j = lane, r = 0; r < 2; j += 32, ++r) {
        if (j >= J) break;
        const double d0 = tj[r][0] - c[0], d1 = tj[r][1] - c[1], d2 = tj[r][2] - c[2];
        T = fmax(T, sqrt(d0 * d0 + d1 * d1 + d2 * d2));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) T = fmax(T, __shfl_xor_sync(0xffffffffu, T, o));
    if (lane != 0) return;

    const double cn = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    const double amax = sqrt(static_cast<double>(a2));
    double rho = static_cast<double>(tpl.cull_wabs) * (amax * tpl.cull_mean_r + T) + static_cast<double>(tpl.cull_wdev) * cn;
    rho = rho * 1.001 + 1e-3 * (1.0 + cn);
    const CameraDev& cam = p.cam;
    const double d[3] = {c[0] - cam.pos[0], c[1] - cam.pos[1], c[2] - cam.pos[2]};
    double W[3][3], tc[3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) W[i][j] = cam.w[3 * i + j];
    for (int i = 0; i < 3; ++i) tc[i] = W[i][0] * d[0] + W[i][1] * d[1] + W[i][2] * d[2];
    // The ball in camera space: radius rho |W|_2 (|W|_2^2 <= max row sum of |W W^T|; 1 for
    // the rotation CameraBasis builds, but the C-ABI takes any matrix).
    double dot[3][3], wmax = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dot[i][j] = W[i][0] * W[j][0] + W[i][1] * W[j][1] + W[i][2] * W[j][2];
    for (int i = 0; i < 3; ++i) wmax = fmax(wmax, fabs(dot[i][0]) + fabs(dot[i][1]) + fabs(dot[i][2]));
    const double rc = rho * sqrt(wmax) * (1.0 + 1e-9);
    const double near_m = cam.near_m;
    bool cull = false;
    if (tc[2] + rc < near_m) {
        cull = true;  // every point behind the near plane
    } else {
        const double zmin = fmax(near_m, tc[2] - rc), zmax = tc[2] + rc;
        const double f = cam.focal, sigma = static_cast<double>(tpl.cull_sigma) * 1.001;
        const double margin = 2.0;                             // pixels
        const double pad = 3.0 * 0.5477225575051661 + 0.01;   // 3 sqrt(0.3)
        // tx/tz and ty/tz over the ball: numerator bound over the tz that extremises it.
        auto ratio_hi = [&](double num) { return num >= 0.0 ? num / zmin : num / zmax; };
        auto ratio_lo = [&](double num) { return num >= 0.0 ? num / zmax : num / zmin; };
        const double ux_hi = ratio_hi(tc[0] + rc), ux_lo = ratio_lo(tc[0] - rc);
        const double uy_hi = ratio_hi(tc[1] + rc), uy_lo = ratio_lo(tc[1] - rc);
        const double ux = fmax(fabs(ux_hi), fabs(ux_lo)), uy = fmax(fabs(uy_hi), fabs(uy_lo));
        // |W0 - u W2|^2 <= |W0|^2 + 2 |u| |W0.W2| + u^2 |W2|^2 (= 1 + u^2 for a rotation).
        const double gx = dot[0][0] + 2.0 * ux * fabs(dot[0][2]) + ux * ux * dot[2][2];
        const double gy = dot[1][1] + 2.0 * uy * fabs(dot[1][2]) + uy * uy * dot[2][2];
        const double rx = 3.0 * (f / zmin) * sqrt(gx) * sigma * 1.001 + pad;
        const double ry = 3.0 * (f / zmin) * sqrt(gy) * sigma * 1.001 + pad;
        const double mx_hi = f * ux_hi + cam.cx, mx_lo = f * ux_lo + cam.cx;
        const double my_hi = f * uy_hi + cam.cy, my_lo = f * uy_lo + cam.cy;
        cull = (mx_hi + rx < cam.band_x0 - margin) || (mx_lo - rx > cam.band_x1 + margin) ||
               (my_hi + ry < cam.band_y0 - margin) || (my_lo - ry > cam.band_y1 + margin);
    }
    // NaN anywhere makes the comparisons false; non-finite input never culls.
    if (bad || !(rho < 1e30)) cull = false;
    p.visible[inst] = cull ? 0u : 1u;
}

__global__ void k_copy_segments(CopySegs c) {
    pdl_entry();
    const uint32_t seg = blockIdx.y;
    const uint32_t* __restrict__ src = c.src[seg];
    uint32_t* __restrict__ dst = c.dst[seg];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c.words[seg]; i += gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// skin_means (avatar.cpp:178-192) of every instance's level into posed[ordinal]: a 2-D
// grid of (256-Gaussian chunk, instance) blocks; the LBS expression is k_project's.
__global__ void __launch_bounds__(256) k_skin_means(SkinParams p) {
    for (uint32_t inst = blockIdx.y; inst < p.n; inst += gridDim.y) {
        const GroupDev grp = p.groups[p.inst_group[inst]];
        const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
        if (gi >= grp.count) continue;
        const float4 c0 = grp.core[4 * gi + 0], c3 = grp.core[4 * gi + 3], wv = grp.weights[gi];
        const uint32_t i01 = __float_as_uint(c3.z), i23 = __float_as_uint(c3.w);
        const uint32_t jidx[4] = {i01 & 0xffffu, i01 >> 16, i23 & 0xffffu, i23 >> 16};
        const float wk[4] = {wv.x, wv.y, wv.z, wv.w};
        const float* s_inst = p.skin + static_cast<size_t>(inst) * p.joint_stride * 12;
        float ax = 0.0f, ay = 0.0f, az = 0.0f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (wk[q] == 0.0f) continue;
            const float4* S = reinterpret_cast<const float4*>(s_inst + jidx[q] * 12);
            const float4 r0 = S[0], r1 = S[1], r2 = S[2];
            const float vx = ((r0.x * c0.x + r0.y * c0.y) + r0.z * c0.z) + r0.w * 1.0f;
            const float vy = ((r1.x * c0.x + r1.y * c0.y) + r1.z * c0.z) + r1.w * 1.0f;
            const float vz = ((r2.x * c0.x + r2.y * c0.y) + r2.z * c0.z) + r2.w * 1.0f;
            ax = ax + wk[q] * vx;
            ay = ay + wk[q] * vy;
            az = az + wk[q] * vz;
        }
        const size_t o = 3ull * (p.inst_base[inst] + gi);
        p.posed[o + 0] = ax;
        p.posed[o + 1] = ay;
        p.posed[o + 2] = az;
    }
}

}  // namespace gscg
