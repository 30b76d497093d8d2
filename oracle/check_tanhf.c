/* check_tanhf.c -- test infrastructure for the tanhf replica (see lpic_math.cuh). */
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
static inline uint32_t fbits(float x){uint32_t u; memcpy(&u,&x,4); return u;}
static inline float bitsf(uint32_t u){float x; memcpy(&x,&u,4); return x;}

/* candidate restatement of the fdlibm-style float expm1 */
static float my_expm1f(float x, int variant){
    const float ln2_hi = bitsf(0x3f317180), ln2_lo = bitsf(0x3717f7d1), invln2 = bitsf(0x3fb8aa3b);
    float Q1,Q2,Q3,Q4,Q5;
    if (variant==0){ Q1=bitsf(0xbd088889);Q2=bitsf(0x3ad00d01);Q3=bitsf(0xb8a670cd);Q4=bitsf(0x36867e54);Q5=bitsf(0xb457edbb);}
    else { Q1=bitsf(0xbd088868);Q2=bitsf(0x3acf3010);Q3=0;Q4=0;Q5=0;}
    uint32_t hx = fbits(x); uint32_t xsb = hx & 0x80000000u; hx &= 0x7fffffffu;
    float hi, lo, c = 0.0f, t; int k;
    if (hx >= 0x4195b844u) {
        if (hx >= 0x42b17218u) { if (hx > 0x7f800000u) return x + x; if (hx == 0x7f800000u) return xsb ? -1.0f : x; if (x > 8.8721679688e+01f) return INFINITY; }
        if (xsb) return -1.0f;
    }
    if (hx > 0x3eb17218u) {
        if (hx < 0x3F851592u) {
            if (!xsb) { hi = x - ln2_hi; lo = ln2_lo; k = 1; } else { hi = x + ln2_hi; lo = -ln2_lo; k = -1; }
        } else {
            k = (int)(invln2 * x + (xsb ? -0.5f : 0.5f));
            t = (float)k; hi = x - t * ln2_hi; lo = t * ln2_lo;
        }
        x = hi - lo; c = (hi - x) - lo;
    } else if (hx < 0x33000000u) { return x; }
    else k = 0;
    float hfx = 0.5f * x, hxs = x * hfx;
    float r1;
    if (variant==0) r1 = 1.0f + hxs * (Q1 + hxs * (Q2 + hxs * (Q3 + hxs * (Q4 + hxs * Q5))));
    else r1 = 1.0f + hxs * (Q1 + hxs * Q2);
    t = 3.0f - r1 * hfx;
    float e = hxs * ((r1 - t) / (6.0f - x * t));
    if (k == 0) return x - (x * e - hxs);
    e = (x * (e - c) - c); e -= hxs;
    if (k == -1) return 0.5f * (x - e) - 0.5f;
    if (k == 1) { if (x < -0.25f) return -2.0f * (e - (x + 0.5f)); else return 1.0f + 2.0f * (x - e); }
    float y;
    if (k <= -2 || k > 56) { y = 1.0f - (e - x); y = bitsf(fbits(y) + ((uint32_t)k << 23)); return y - 1.0f; }
    if (k < 23) { t = bitsf(0x3f800000u - (0x1000000u >> k)); y = t - (e - x); y = bitsf(fbits(y) + ((uint32_t)k << 23)); }
    else { t = bitsf((uint32_t)(0x7f - k) << 23); y = x - (e + t); y += 1.0f; y = bitsf(fbits(y) + ((uint32_t)k << 23)); }
    return y;
}
static float my_tanhf(float x, int variant){
    uint32_t jx = fbits(x), ix = jx & 0x7fffffffu; float t, z;
    if (ix >= 0x7f800000u) { if ((int32_t)jx >= 0) return 1.0f / x + 1.0f; else return 1.0f / x - 1.0f; }
    if (ix < 0x41b00000u) {
        if (ix < 0x24000000u) return x * (1.0f + x);
        if (ix >= 0x3f800000u) { t = my_expm1f(2.0f * fabsf(x), variant); z = 1.0f - 2.0f / (t + 2.0f); }
        else { t = my_expm1f(-2.0f * fabsf(x), variant); z = -t / (t + 2.0f); }
    } else z = 1.0f;
    return ((int32_t)jx >= 0) ? z : -z;
}
/* Exhaustive (stride 1) or sampled check that the fdlibm-style float tanh
 * replica used on the GPU (paper_2212_01185_b200/csrc/lpic_math.cuh) equals
 * the host glibc tanhf bit for bit on |x| < 30.  Usage: check_tanhf [stride] */
#include <stdlib.h>
int main(int argc, char** argv){
    uint64_t stride = argc > 1 ? strtoull(argv[1], 0, 10) : 1;
    { int variant = 0;
    long long bad=0, badexp=0, n=0;
    for (uint64_t u = 0; u < 0x100000000ull; u += stride) {
        float x = bitsf((uint32_t)u);
        if (!(fabsf(x) < 30.0f)) continue;
        n++;
        float a = tanhf(x), b = my_tanhf(x, variant);
        if (fbits(a) != fbits(b)) { if (bad < 5) printf("v%d tanh mismatch x=%a glibc=%a mine=%a\n", variant, x, a, b); bad++; }
        if (stride > 1 || (u & 0xff) == 0) { float c = expm1f(x), d = my_expm1f(x, variant); if (fbits(c)!=fbits(d)) badexp++; }
    }
    printf("variant %d: n=%lld tanh mismatches=%lld expm1 sample mismatches=%lld\n", variant, n, bad, badexp);
    }
    return 0;
}
