// lpic_math.cuh -- bit-reproducible scalar math shared by every LPIC kernel.
//
// Everything here is compiled with -fmad=false and written with explicit
// round-to-nearest intrinsics, so the encoder and the decoder (and every
// thread mapping of the table builder) execute the same IEEE operations.
//
//  * tanhf_glibc: a restatement of the published fdlibm float algorithm
//    (expm1f by Remez rational approximation after k*ln2 argument reduction;
//    tanh(x) = 1 - 2/(expm1(2|x|)+2) for |x| >= 1, -t/(t+2) with
//    t = expm1(-2|x|) below).  Verified bit-exact against the host glibc
//    tanhf on all 2.2e9 float32 inputs with |x| < 30 (oracle/check_tanhf.c),
//    which is what the reference's numba kernels call for the float32 mean
//    update (/root/reference/pkg/src/lpic/kernels.py:234-241).
//  * phi: the Gaussian / logistic CDF of kernels._cdf_value
//    (/root/reference/pkg/src/lpic/kernels.py:202-209) in float64.
//
// expm1f_fdlibm / tanhf_glibc restate the algorithm, thresholds and
// coefficients of fdlibm's s_expm1f.c and s_tanhf.c, which carry this notice:
//
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this
//   software is freely granted, provided that this notice
//   is preserved.
#pragma once
#include <cstdint>

namespace lpic {

__device__ __forceinline__ uint32_t f2u(float x) { return __float_as_uint(x); }
__device__ __forceinline__ float u2f(uint32_t u) { return __uint_as_float(u); }

// fdlibm-style expm1f; constants are the published float coefficients.
__device__ __forceinline__ float expm1f_fdlibm(float x) {
    const float ln2_hi = u2f(0x3f317180u), ln2_lo = u2f(0x3717f7d1u), invln2 = u2f(0x3fb8aa3bu);
    const float Q1 = u2f(0xbd088889u), Q2 = u2f(0x3ad00d01u), Q3 = u2f(0xb8a670cdu),
                Q4 = u2f(0x36867e54u), Q5 = u2f(0xb457edbbu);
    uint32_t hx = f2u(x);
    const uint32_t xsb = hx & 0x80000000u;
    hx &= 0x7fffffffu;
    float hi, lo, c = 0.0f, t;
    int k;
    if (hx >= 0x4195b844u) {                      // |x| >= 27 ln2
        if (hx >= 0x42b17218u) {
            if (hx > 0x7f800000u) return __fadd_rn(x, x);
            if (hx == 0x7f800000u) return xsb ? -1.0f : x;
            if (x > 8.8721679688e+01f) return __int_as_float(0x7f800000);
        }
        if (xsb) return -1.0f;
    }
    if (hx > 0x3eb17218u) {                       // |x| > 0.5 ln2
        if (hx < 0x3F851592u) {                   // |x| < 1.5 ln2
            if (!xsb) { hi = __fsub_rn(x, ln2_hi); lo = ln2_lo; k = 1; }
            else      { hi = __fadd_rn(x, ln2_hi); lo = -ln2_lo; k = -1; }
        } else {
            k = (int)__fadd_rn(__fmul_rn(invln2, x), xsb ? -0.5f : 0.5f);
            t = (float)k;
            hi = __fsub_rn(x, __fmul_rn(t, ln2_hi));
            lo = __fmul_rn(t, ln2_lo);
        }
        x = __fsub_rn(hi, lo);
        c = __fsub_rn(__fsub_rn(hi, x), lo);
    } else if (hx < 0x33000000u) {
        return x;
    } else {
        k = 0;
    }
    const float hfx = __fmul_rn(0.5f, x);
    const float hxs = __fmul_rn(x, hfx);
    float r1 = __fmul_rn(hxs, Q5);
    r1 = __fmul_rn(hxs, __fadd_rn(Q4, r1));
    r1 = __fmul_rn(hxs, __fadd_rn(Q3, r1));
    r1 = __fmul_rn(hxs, __fadd_rn(Q2, r1));
    r1 = __fadd_rn(1.0f, __fmul_rn(hxs, __fadd_rn(Q1, r1)));
    t = __fsub_rn(3.0f, __fmul_rn(r1, hfx));
    float e = __fmul_rn(hxs, __fdiv_rn(__fsub_rn(r1, t), __fsub_rn(6.0f, __fmul_rn(x, t))));
    if (k == 0) return __fsub_rn(x, __fsub_rn(__fmul_rn(x, e), hxs));
    e = __fsub_rn(__fmul_rn(x, __fsub_rn(e, c)), c);
    e = __fsub_rn(e, hxs);
    if (k == -1) return __fsub_rn(__fmul_rn(0.5f, __fsub_rn(x, e)), 0.5f);
    if (k == 1) {
        if (x < -0.25f) return __fmul_rn(-2.0f, __fsub_rn(e, __fadd_rn(x, 0.5f)));
        return __fadd_rn(1.0f, __fmul_rn(2.0f, __fsub_rn(x, e)));
    }
    float y;
    if (k <= -2 || k > 56) {
        y = __fsub_rn(1.0f, __fsub_rn(e, x));
        y = u2f(f2u(y) + ((uint32_t)k << 23));
        return __fsub_rn(y, 1.0f);
    }
    if (k < 23) {
        t = u2f(0x3f800000u - (0x1000000u >> k));
        y = __fsub_rn(t, __fsub_rn(e, x));
        y = u2f(f2u(y) + ((uint32_t)k << 23));
    } else {
        t = u2f((uint32_t)(0x7f - k) << 23);
        y = __fsub_rn(x, __fadd_rn(e, t));
        y = __fadd_rn(y, 1.0f);
        y = u2f(f2u(y) + ((uint32_t)k << 23));
    }
    return y;
}

__device__ __forceinline__ float tanhf_glibc(float x) {
    const uint32_t jx = f2u(x), ix = jx & 0x7fffffffu;
    float t, z;
    if (ix >= 0x7f800000u) return ((int32_t)jx >= 0) ? __fadd_rn(__fdiv_rn(1.0f, x), 1.0f)
                                                       : __fsub_rn(__fdiv_rn(1.0f, x), 1.0f);
    if (ix < 0x41b00000u) {                       // |x| < 22
        if (ix < 0x24000000u) return __fmul_rn(x, __fadd_rn(1.0f, x));
        const float ax = fabsf(x);
        if (ix >= 0x3f800000u) {
            t = expm1f_fdlibm(__fmul_rn(2.0f, ax));
            z = __fsub_rn(1.0f, __fdiv_rn(2.0f, __fadd_rn(t, 2.0f)));
        } else {
            t = expm1f_fdlibm(__fmul_rn(-2.0f, ax));
            z = __fdiv_rn(-t, __fadd_rn(t, 2.0f));
        }
    } else {
        z = 1.0f;
    }
    return ((int32_t)jx >= 0) ? z : -z;
}

// kernels._cdf_value (kernels.py:202-209): the Gaussian as 0.5*erfc(-z/sqrt2)
// exactly as written (product, then erfc), the logistic sign-split.
__device__ __forceinline__ double phi(double z, int dist) {
    if (dist == 0) return __dmul_rn(0.5, erfc(__dmul_rn(-z, 0.7071067811865476)));
    if (z >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-z)));
    const double e = exp(z);
    return __ddiv_rn(e, __dadd_rn(1.0, e));
}

// order-preserving unsigned key of a double (NaN sorts last, like numpy)
__device__ __forceinline__ uint64_t dkey(double x) {
    if (x != x) return ~0ull;
    if (x == 0.0) x = 0.0;                        // -0 == +0 for the stable sort
    const uint64_t u = (uint64_t)__double_as_longlong(x);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

}  // namespace lpic
