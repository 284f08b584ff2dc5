// Bit-compatible port of glibc's expf (glibc >= 2.28, sysdeps/ieee754/flt-32/e_expf.c;
// algorithm from ARM optimized-routines): exp(x) = 2^(k/32) * 2^(r/32) with a
// 32-entry table and a cubic polynomial, evaluated in double and rounded once.
//
// Why: the reference computes router softmax probabilities with host expf
// (proj/include/spes/kernels.hpp:163-167 via std::exp on float); CUDA's expf
// differs on ~1e5 inputs of [-104, 0], which would flip top-k
// ties. The table/constants are the published algorithm's values (verified
// against this container's libm image). glibc picks an FMA-compiled variant
// (ifunc __expf_fma) on CPUs with FMA+AVX2, so both evaluation orders are
// provided and the host's is detected at runtime; tests check the device port
// exhaustively against host expf over [-104, 0].
//
// Attribution: the 2^(i/32) table, the polynomial coefficients and the evaluation scheme
// are those of ARM optimized-routines' expf (Copyright (c) 2017-2018, Arm Limited; MIT /
// Apache-2.0 WITH LLVM-exception) as shipped in the GNU C Library (LGPL-2.1-or-later).
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SPES_HD __host__ __device__ __forceinline__
#else
#define SPES_HD static inline
#include <math.h>
#endif

#define SPES_EXPF_TAB                                                                          \
    {0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL, \
     0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL, \
     0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL, \
     0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL, \
     0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL, \
     0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL, \
     0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL, \
     0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL}

namespace spes_expf {

#if defined(__CUDACC__)
__device__ const uint64_t k_tab_dev[32] = SPES_EXPF_TAB;
#endif
static const uint64_t k_tab_host[32] = SPES_EXPF_TAB;

SPES_HD uint64_t tab(uint32_t i) {
#if defined(__CUDA_ARCH__)
    return __ldg(&k_tab_dev[i]);
#else
    return k_tab_host[i];
#endif
}

SPES_HD double as_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(u));
#else
    double d;
    memcpy(&d, &u, 8);
    return d;
#endif
}
SPES_HD uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(d));
#else
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
#endif
}
SPES_HD float as_float(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}
SPES_HD uint32_t as_u32(float f) {
#if defined(__CUDA_ARCH__)
    return __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
#endif
}

// Explicitly rounded double ops (no contraction on either side).
SPES_HD double dmul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    volatile double r = a * b;
    return r;
#endif
}
SPES_HD double dadd(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    volatile double r = a + b;
    return r;
#endif
}
SPES_HD double dsub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    volatile double r = a - b;
    return r;
#endif
}
SPES_HD double dfma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

// variant 0: plain double arithmetic (generic e_expf.c build, no FMA)
// variant 1: FMA-contracted build (e_expf-fma.c, -mfma -mavx2), selected by glibc's
//            ifunc on FMA+AVX2 hosts
template <int VARIANT>
SPES_HD float expf_glibc(float x) {
    const double kInvLn2N = 0x1.71547652b82fep+0 * 32;
    const double kShift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32;
    const double C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32;
    const double C2 = 0x1.62e42ff0c52d6p-1 / 32;
    const uint32_t ux = as_u32(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= (0x42b00000u >> 20)) {  // |x| >= 88 or nan
        if (ux == 0xff800000u) return 0.0f;                   // -inf
        if (abstop >= (0x7f800000u >> 20)) return x + x;      // inf / nan
        if (x > 0x1.62e42ep6f) return as_float(0x7f800000u);  // overflow -> inf
        if (x < -0x1.9fe368p6f) return 0.0f;                  // underflow -> 0
    }
    const double xd = static_cast<double>(x);
    double z, kd, r, s, y, r2, zz;
    (void)z;
    uint64_t ki, t;
    if (VARIANT == 0) {
        z = dmul(kInvLn2N, xd);
        kd = dadd(z, kShift);
        ki = as_u64(kd);
        kd = dsub(kd, kShift);
        r = dsub(z, kd);
        t = tab(static_cast<uint32_t>(ki % 32));
        t += ki << (52 - 5);
        s = as_double(t);
        zz = dadd(dmul(C0, r), C1);
        r2 = dmul(r, r);
        y = dadd(dmul(C2, r), 1.0);
        y = dadd(dmul(zz, r2), y);
        y = dmul(y, s);
    } else {
        // e_expf-fma.c: the compiler contracts z = InvLn2N*xd into both of its uses
        kd = dfma(kInvLn2N, xd, kShift);
        ki = as_u64(kd);
        kd = dsub(kd, kShift);
        r = dfma(kInvLn2N, xd, -kd);
        t = tab(static_cast<uint32_t>(ki % 32));
        t += ki << (52 - 5);
        s = as_double(t);
        zz = dfma(C0, r, C1);
        r2 = dmul(r, r);
        y = dfma(C2, r, 1.0);
        y = dfma(zz, r2, y);
        y = dmul(y, s);
    }
    return static_cast<float>(y);
}

}  // namespace spes_expf

namespace spes_expf {
// Which evaluation order does this host's libm use? Two inputs separate the
// variants (found by an exhaustive sweep of all 2^32 floats against glibc 2.39).
static inline int host_variant_from(float (*host_expf)(float)) {
    const uint32_t probes[2] = {0x4202422fu, 0xc27c65d9u};
    int v1 = 1;
    for (uint32_t u : probes) {
        float x = as_float(u);
        if (as_u32(host_expf(x)) != as_u32(expf_glibc<1>(x))) v1 = 0;
    }
    return v1;
}
}  // namespace spes_expf
