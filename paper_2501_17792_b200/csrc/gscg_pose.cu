// Device pose sampling: every instance's clip sampled at
// time_s + phase (sample_pose with wrap, avatar.cpp:247-283, driven by crowd.cpp:118-128),
// bit-identical to the host path so LoD, sort order and pixels are unchanged.
//
// Exactness: the slerp's transcendentals split into per-keyframe-pair values (theta =
// acos(min(|dot|, 1)), s = sin(theta); computed by the host libm when the clip is uploaded)
// and the two per-instance sines sin((1-t) theta), sin(t theta) with arguments in
// [0, pi/2]. Those use glibc_sinf below, a replica of glibc's sinf (the double-precision
// polynomial of sysdeps/ieee754/flt-32/s_sinf.c). It was checked equal to the host's sinf
// on every float in [0, pi/2]; tests/test_gpu_parity.py checks this device copy against
// the host libm through gscg_eval_sinf. This TU is built with --fmad=false: every float
// and double operation rounds exactly as the host's does.
#include "gscg_common.cuh"
#include "gscg_kernels.h"

namespace gscg {

namespace {

// glibc sinf for |x| < 120 (and the tiny-argument shortcut). The polynomial and the
// reduction constants are glibc's __sincosf_table entries.
__device__ __forceinline__ float glibc_sinf(float y) {
    constexpr double S1 = -0x1.555545995a603p-3, S2 = 0x1.1107605230bc4p-7, S3 = -0x1.994eb3774cf24p-13;
    constexpr double C0 = -0x1.ffffffd0c621cp-2, C1 = 0x1.55553e1068f19p-5, C2 = -0x1.6c087e89a359dp-10,
                     C3 = 0x1.99343027bf8c3p-16;
    constexpr double kHpiInv = 0x1.45F306DC9C883p+23, kHpi = 0x1.921FB54442D18p0;
    const uint32_t top = (__float_as_uint(y) >> 20) & 0x7ffu;
    double x = static_cast<double>(y);
    int n = 0;
    if (top < ((__float_as_uint(0x1.921fb6p-1f) >> 20) & 0x7ffu)) {
        if (top < ((__float_as_uint(0x1p-12f) >> 20) & 0x7ffu)) return y;
    } else {
        const double r = x * kHpiInv;
        n = (static_cast<int32_t>(r) + 0x800000) >> 24;
        x = x - static_cast<double>(n) * kHpi;
        if (n & 1) {  // cosine polynomial, sign from the quadrant (n & 2)
            const double neg = (n & 2) ? -1.0 : 1.0;
            const double x2 = x * x;
            const double x4 = x2 * x2;
            const double c2 = neg * C2 + x2 * (neg * C3);
            const double c1 = neg + x2 * (neg * C0);
            const double x6 = x4 * x2;
            const double c = c1 + x4 * (neg * C1);
            return static_cast<float>(c + x6 * c2);
        }
        if (n & 2) x = -x;
    }
    const double x2 = x * x;
    const double x3 = x * x2;
    const double s1 = S2 + x2 * S3;
    const double x7 = x3 * x2;
    const double s = x + x3 * S1;
    return static_cast<float>(s + x7 * s1);
}

}  // namespace

// One thread per (instance, slot): slot 0 = root translation, slot 1 + j = joint j.
__global__ void __launch_bounds__(256)
k_sample_poses(PoseParams p) {
    pdl_entry();
    const uint32_t slots = p.joint_stride + 1;
    const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= static_cast<uint64_t>(p.n) * slots) return;
    const uint32_t i = static_cast<uint32_t>(g / slots), k = static_cast<uint32_t>(g % slots);
    float* rec = p.poses + static_cast<size_t>(i) * (4 + 4 * p.joint_stride);
    if (p.static_pose) {
        if (k == 0) *reinterpret_cast<float4*>(rec) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        else *reinterpret_cast<float4*>(rec + 4 * k) = make_float4(0.0f, 0.0f, 0.0f, 1.0f);
        return;
    }
    const MotionDev M = p.motions[p.motion_ids[i]];
    if (k > M.joints) return;  // beyond the clip's skeleton: FK never reads it
    // locate (wrap): frame pair and blend weight (avatar.cpp:253-276).
    const float time = p.time_s + p.phase[i];
    float fpos = time * M.fps;
    const float nf = static_cast<float>(M.frames);
    fpos = fmodf(fpos, nf);
    if (fpos < 0.0f) fpos += nf;
    const uint32_t i0 = static_cast<uint32_t>(static_cast<unsigned long long>(fpos) % M.frames);
    const uint32_t i1 = (i0 + 1) % M.frames;
    const float t = fpos - floorf(fpos);
    if (k == 0) {
        const float4 a = p.roots[M.root_offset + i0], b = p.roots[M.root_offset + i1];
        const float u = 1.0f - t;
        *reinterpret_cast<float4*>(rec) = make_float4(u * a.x + t * b.x, u * a.y + t * b.y, u * a.z + t * b.z, 0.0f);
        return;
    }
    const KeyPairDev kp = p.keys[M.key_offset + static_cast<size_t>(i0) * M.joints + (k - 1)];
    float c[4];
    const float a[4] = {kp.a.x, kp.a.y, kp.a.z, kp.a.w}, bf[4] = {kp.b.x, kp.b.y, kp.b.z, kp.b.w};
    if (kp.lerp) {
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = a[q] + t * (bf[q] - a[q]);
    } else {
        const float wa = glibc_sinf((1.0f - t) * kp.theta) / kp.sin_theta;
        const float wb = glibc_sinf(t * kp.theta) / kp.sin_theta;
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = wa * a[q] + wb * bf[q];
    }
    // normalize (Eigen: squaredNorm as the SSE packet reduction, then divide by the norm)
    const float z = (c[0] * c[0] + c[2] * c[2]) + (c[1] * c[1] + c[3] * c[3]);
    if (z > 0.0f) {
        const float nrm = sqrtf(z);
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = c[q] / nrm;
    }
    *reinterpret_cast<float4*>(rec + 4 * k) = make_float4(c[0], c[1], c[2], c[3]);
}

// Parity hook: glibc_sinf over a host-chosen argument list (tests compare with the host libm).
__global__ void k_eval_sinf(const float* in, float* out, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = glibc_sinf(in[i]);
}

}  // namespace gscg
