// lpic_net.cuh -- the causal-neighbourhood network on CUDA cores in the
// reference's canonical float32 order ("compat" precision).
//
// Restates kernels.forward_taps_f32 / _dense_stack
// (/root/reference/pkg/src/lpic/kernels.py:63-136): for each output unit the
// products are added in input order with separate multiply and add (no FMA),
// the bias is added last, then LeakyReLU x>=0 ? x : 0.01f*x.  The result is
// bit-identical to the CPU reference.  One thread evaluates one pixel; the
// activations live in registers, weights are read as warp-uniform float4
// broadcasts through L1.
//
// Padding: C is padded to CP (a multiple of 16) and M to MP (multiple of 4)
// with zero weights.  A padded unit contributes w*a = +-0 after every real
// term; the accumulator is never -0 (it starts at +0 and only a sum of
// non-zero terms can cancel to +0), so padding is bit-exact.
#pragma once
#include <cstdint>

namespace lpic {

struct NetDev {                 // device-resident, padded weights
    const float* mwT;           // (CP, TC) masked weights, filter-major
    const float* mb;            // (CP)
    const float* hw;            // (NH, CP, CP)  [l][out][in]
    const float* hb;            // (NH, CP)
    const float* ow;            // (MP, CP)
    const float* ob;            // (MP)
    int C, CP, M, MP, NH, T, TC;
};

__device__ __forceinline__ float leaky(float x) { return x >= 0.0f ? x : __fmul_rn(0.01f, x); }

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// x[TC] -> raw[M] (written to raw_out with stride 1).  zbuf: per-thread
// column in shared memory, element o at zbuf[o * zstride].
template <int CP, int TC>
__device__ __forceinline__ void net_forward(const NetDev& w, const float (&x)[TC], float* raw_out,
                                            float* zbuf, int zstride) {
    float a[CP];
    // masked layer (kernels.py:98-113)
#pragma unroll 1
    for (int f = 0; f < CP; f += 2) {
        float acc0 = 0.0f, acc1 = 0.0f;
        const float* w0 = w.mwT + (int64_t)f * TC;
        const float* w1 = w0 + TC;
#pragma unroll
        for (int t = 0; t < TC; t += 4) {
            const float4 u = ldg4(w0 + t), v = ldg4(w1 + t);
            acc0 = __fadd_rn(acc0, __fmul_rn(u.x, x[t + 0])); acc1 = __fadd_rn(acc1, __fmul_rn(v.x, x[t + 0]));
            acc0 = __fadd_rn(acc0, __fmul_rn(u.y, x[t + 1])); acc1 = __fadd_rn(acc1, __fmul_rn(v.y, x[t + 1]));
            acc0 = __fadd_rn(acc0, __fmul_rn(u.z, x[t + 2])); acc1 = __fadd_rn(acc1, __fmul_rn(v.z, x[t + 2]));
            acc0 = __fadd_rn(acc0, __fmul_rn(u.w, x[t + 3])); acc1 = __fadd_rn(acc1, __fmul_rn(v.w, x[t + 3]));
        }
        zbuf[f * zstride] = leaky(__fadd_rn(acc0, __ldg(w.mb + f)));
        zbuf[(f + 1) * zstride] = leaky(__fadd_rn(acc1, __ldg(w.mb + f + 1)));
    }
#pragma unroll
    for (int i = 0; i < CP; i++) a[i] = zbuf[i * zstride];
    // hidden 1x1 layers (kernels.py:69-80)
    for (int l = 0; l < w.NH; l++) {
        const float* W = w.hw + (int64_t)l * CP * CP;
        const float* B = w.hb + (int64_t)l * CP;
#pragma unroll 1
        for (int o = 0; o < CP; o += 4) {
            float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
            const float* r0 = W + (int64_t)o * CP;
#pragma unroll
            for (int i = 0; i < CP; i += 4) {
                const float4 p = ldg4(r0 + i), q = ldg4(r0 + CP + i), s = ldg4(r0 + 2 * CP + i),
                             u = ldg4(r0 + 3 * CP + i);
                c0 = __fadd_rn(c0, __fmul_rn(p.x, a[i])); c1 = __fadd_rn(c1, __fmul_rn(q.x, a[i]));
                c2 = __fadd_rn(c2, __fmul_rn(s.x, a[i])); c3 = __fadd_rn(c3, __fmul_rn(u.x, a[i]));
                c0 = __fadd_rn(c0, __fmul_rn(p.y, a[i + 1])); c1 = __fadd_rn(c1, __fmul_rn(q.y, a[i + 1]));
                c2 = __fadd_rn(c2, __fmul_rn(s.y, a[i + 1])); c3 = __fadd_rn(c3, __fmul_rn(u.y, a[i + 1]));
                c0 = __fadd_rn(c0, __fmul_rn(p.z, a[i + 2])); c1 = __fadd_rn(c1, __fmul_rn(q.z, a[i + 2]));
                c2 = __fadd_rn(c2, __fmul_rn(s.z, a[i + 2])); c3 = __fadd_rn(c3, __fmul_rn(u.z, a[i + 2]));
                c0 = __fadd_rn(c0, __fmul_rn(p.w, a[i + 3])); c1 = __fadd_rn(c1, __fmul_rn(q.w, a[i + 3]));
                c2 = __fadd_rn(c2, __fmul_rn(s.w, a[i + 3])); c3 = __fadd_rn(c3, __fmul_rn(u.w, a[i + 3]));
            }
            zbuf[(o + 0) * zstride] = leaky(__fadd_rn(c0, __ldg(B + o + 0)));
            zbuf[(o + 1) * zstride] = leaky(__fadd_rn(c1, __ldg(B + o + 1)));
            zbuf[(o + 2) * zstride] = leaky(__fadd_rn(c2, __ldg(B + o + 2)));
            zbuf[(o + 3) * zstride] = leaky(__fadd_rn(c3, __ldg(B + o + 3)));
        }
#pragma unroll
        for (int i = 0; i < CP; i++) a[i] = zbuf[i * zstride];
    }
    // output layer, no activation (kernels.py:81-85)
#pragma unroll 1
    for (int m = 0; m < w.MP; m += 4) {
        float c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
        const float* r0 = w.ow + (int64_t)m * CP;
#pragma unroll
        for (int i = 0; i < CP; i += 4) {
            const float4 p = ldg4(r0 + i), q = ldg4(r0 + CP + i), s = ldg4(r0 + 2 * CP + i),
                         u = ldg4(r0 + 3 * CP + i);
            c0 = __fadd_rn(c0, __fmul_rn(p.x, a[i])); c1 = __fadd_rn(c1, __fmul_rn(q.x, a[i]));
            c2 = __fadd_rn(c2, __fmul_rn(s.x, a[i])); c3 = __fadd_rn(c3, __fmul_rn(u.x, a[i]));
            c0 = __fadd_rn(c0, __fmul_rn(p.y, a[i + 1])); c1 = __fadd_rn(c1, __fmul_rn(q.y, a[i + 1]));
            c2 = __fadd_rn(c2, __fmul_rn(s.y, a[i + 1])); c3 = __fadd_rn(c3, __fmul_rn(u.y, a[i + 1]));
            c0 = __fadd_rn(c0, __fmul_rn(p.z, a[i + 2])); c1 = __fadd_rn(c1, __fmul_rn(q.z, a[i + 2]));
            c2 = __fadd_rn(c2, __fmul_rn(s.z, a[i + 2])); c3 = __fadd_rn(c3, __fmul_rn(u.z, a[i + 2]));
            c0 = __fadd_rn(c0, __fmul_rn(p.w, a[i + 3])); c1 = __fadd_rn(c1, __fmul_rn(q.w, a[i + 3]));
            c2 = __fadd_rn(c2, __fmul_rn(s.w, a[i + 3])); c3 = __fadd_rn(c3, __fmul_rn(u.w, a[i + 3]));
        }
        if (m + 0 < w.M) raw_out[m + 0] = __fadd_rn(c0, __ldg(w.ob + m + 0));
        if (m + 1 < w.M) raw_out[m + 1] = __fadd_rn(c1, __ldg(w.ob + m + 1));
        if (m + 2 < w.M) raw_out[m + 2] = __fadd_rn(c2, __ldg(w.ob + m + 2));
        if (m + 3 < w.M) raw_out[m + 3] = __fadd_rn(c3, __ldg(w.ob + m + 3));
    }
}

}  // namespace lpic
