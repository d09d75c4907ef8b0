// Device replica of the host libm's expf, bit for bit, so the rasteriser's alpha =
// opacity * exp(power) (renderer.cpp:205) equals the reference's on every pixel.
//
// glibc 2.28+ expf (sysdeps/ieee754/flt-32/e_expf.c, EXP2F_TABLE_BITS = 5, polynomial
// order 3) evaluated in double: x*32/ln2 = k + r, exp(x) = 2^(k/32) * 2^(r/32) with
// 2^(r/32) ~ C0 r^3 + C1 r^2 + C2 r + 1, then rounded to float. On x86-64 CPUs with FMA
// (the build and GPU boxes) glibc dispatches to its -mfma build, whose contraction puts
// r = fma(InvLn2N, x, -kd) and the polynomial on FMAs; that variant is restated here.
// Checked equal to the host expf on every float in [-103.97, 88.72] (2,239,754,678
// floats, 0 differences; tests/test_gpu_parity.py re-checks the device copy against the
// host libm on every float the rasteriser can see). Table entry i is the double nearest
// 2^(i/32) minus i << 47, as glibc stores it.
#pragma once

#include <cstdint>

namespace gscg {

// For the rasterisers' hot loops: the table's 32-bit shared-memory address is held in a
// register and the polynomial constants come from the constant bank (the compiler would
// otherwise rebuild both, and the shared window base, on every call). k_eval_expf runs this
// same function for the exhaustive check.
struct ExpfRegs {
    double inv_ln2n, c0, c1, c2;
    uint32_t tab;
};
// Constants read from the constant bank (DMUL/DFMA take them as c[][] operands: no moves
// in the loop).
__constant__ double c_expf_k[4] = {0x1.71547652b82fep+0 * 32, 0x1.c6af84b912394p-5 / 32 / 32 / 32,
                                   0x1.ebfce50fac4f3p-3 / 32 / 32, 0x1.62e42ff0c52d6p-1 / 32};
__device__ __forceinline__ ExpfRegs expf_regs(const unsigned long long* s_tab) {
    ExpfRegs k;
    k.inv_ln2n = c_expf_k[0];
    k.c0 = c_expf_k[1];
    k.c1 = c_expf_k[2];
    k.c2 = c_expf_k[3];
    uint32_t t = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
    asm volatile("mov.b32 %0, %0;" : "+r"(t));  // kept in a register, not rebuilt per call
    k.tab = t;
    return k;
}
__device__ __forceinline__ float glibc_expf_regs(float x, const ExpfRegs& k) {
    constexpr double kShift = 0x1.8p+52;
    const double xd = static_cast<double>(x);
    const double z = __dmul_rn(k.inv_ln2n, xd);
    double kd = __dadd_rn(z, kShift);
    const uint32_t ki = static_cast<uint32_t>(__double2loint(kd));  // k's low bits (ki << 47 uses 17 of them)
    kd = __dsub_rn(kd, kShift);
    const double r = __fma_rn(k.inv_ln2n, xd, -kd);
    uint32_t tlo, thi;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(tlo), "=r"(thi) : "r"(k.tab + (ki & 31u) * 8u));
    const double s = __hiloint2double(static_cast<int>(thi + (ki << 15)), static_cast<int>(tlo));  // tab + (ki << 47)
    const double zp = __fma_rn(k.c0, r, k.c1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(k.c2, r, 1.0);
    y = __fma_rn(zp, r2, y);
    return __double2float_rn(__dmul_rn(y, s));
}

// The 32-entry table (glibc __exp2f_data.tab).
#define GSCG_EXP2F_TAB                                                                                  \
    {0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,        \
     0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,        \
     0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,        \
     0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,        \
     0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,        \
     0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,        \
     0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,        \
     0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL}

}  // namespace gscg
