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
    // input-major copies for the tiled kernel (net_tile)
    const float* mwI;           // (TC, CP)   [tc][f]  (the reference's own masked_w layout)
    const float* hwI;           // (NH, CP, CP) [l][in][out]
    const float* owI;           // (CP, MT)   [in][m], MT = M padded to 16
    int C, CP, M, MP, NH, T, TC, MT;
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

// ---------------------------------------------------------------------------
// CTA-cooperative tiled network: 256 threads evaluate a tile of NT_TP = 64
// pixels as register-tiled CUDA-core GEMMs with the current layer's weights
// and both activation buffers in shared memory.  Thread t owns pixels
// 4*(t&15) .. +3 and outputs (t>>4)*F .. +F-1 of every layer; each of its
// accumulators runs over the layer input index in increasing order with a
// separate multiply and add, so the result is bit-identical to net_forward
// and to the reference.  (A thread-per-pixel network streams 236 KB of
// weights per pixel through a 25 KB L1 and is L2-latency bound.)
// ---------------------------------------------------------------------------
constexpr int NT_THREADS = 256;
constexpr int NT_TP = 64;

struct NetTileBufs {
    float* act0;     // [max(CP, TC)][NT_TP]; holds the gathered taps on entry
    float* act1;     // [CP][NT_TP]
    float* wbuf;     // max(TC*CP, CP*CP, CP*MT) floats
    float* raw;      // [NT_TP][MP] output
};

__host__ __device__ constexpr size_t net_tile_floats(int CP, int TC, int MT, int MP) {
    return (size_t)(CP > TC ? CP : TC) * NT_TP + (size_t)CP * NT_TP +
           (size_t)((TC * CP > CP * CP ? TC * CP : CP * CP) > CP * MT ? (TC * CP > CP * CP ? TC * CP : CP * CP)
                                                                       : CP * MT) +
           (size_t)NT_TP * MP;
}

__device__ __forceinline__ void tile_copy(float* dst, const float* __restrict__ src, int n) {
    if (threadIdx.x >= NT_THREADS) return;
    for (int k = threadIdx.x * 4; k < n; k += NT_THREADS * 4)
        *reinterpret_cast<float4*>(dst + k) = __ldg(reinterpret_cast<const float4*>(src + k));
}

template <int F>
__device__ __forceinline__ void load_w(const float* p, float (&wv)[F]) {
    if constexpr (F % 4 == 0) {
#pragma unroll
        for (int f = 0; f < F; f += 4) {
            const float4 v = *reinterpret_cast<const float4*>(p + f);
            wv[f] = v.x; wv[f + 1] = v.y; wv[f + 2] = v.z; wv[f + 3] = v.w;
        }
    } else if constexpr (F % 2 == 0) {
#pragma unroll
        for (int f = 0; f < F; f += 2) {
            const float2 v = *reinterpret_cast<const float2*>(p + f);
            wv[f] = v.x; wv[f + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int f = 0; f < F; f++) wv[f] = p[f];
    }
}

// acc[p][f] = sum_{i<KD} W[i][og*F+f] * in[i][4pg+p], i ascending
template <int KD, int F>
__device__ __forceinline__ void tile_layer(const float* in, const float* W, int nout, int og, int pg,
                                           float (&acc)[4][F]) {
#pragma unroll
    for (int p = 0; p < 4; p++)
#pragma unroll
        for (int f = 0; f < F; f++) acc[p][f] = 0.0f;
#pragma unroll 4
    for (int i = 0; i < KD; i++) {
        const float4 a = *reinterpret_cast<const float4*>(in + i * NT_TP + 4 * pg);
        float wv[F];
        load_w<F>(W + i * nout + og * F, wv);
#pragma unroll
        for (int f = 0; f < F; f++) {
            acc[0][f] = __fadd_rn(acc[0][f], __fmul_rn(wv[f], a.x));
            acc[1][f] = __fadd_rn(acc[1][f], __fmul_rn(wv[f], a.y));
            acc[2][f] = __fadd_rn(acc[2][f], __fmul_rn(wv[f], a.z));
            acc[3][f] = __fadd_rn(acc[3][f], __fmul_rn(wv[f], a.w));
        }
    }
}

template <int F>
__device__ __forceinline__ void tile_store_act(const float (&acc)[4][F], const float* __restrict__ bias, int og, int pg,
                                               float* out) {
#pragma unroll
    for (int f = 0; f < F; f++) {
        const float b = __ldg(bias + og * F + f);
        float4 v;
        v.x = leaky(__fadd_rn(acc[0][f], b)); v.y = leaky(__fadd_rn(acc[1][f], b));
        v.z = leaky(__fadd_rn(acc[2][f], b)); v.w = leaky(__fadd_rn(acc[3][f], b));
        *reinterpret_cast<float4*>(out + (og * F + f) * NT_TP + 4 * pg) = v;
    }
}

// Network of one tile.  On entry b.act0 holds the taps as [tc][p]; on exit
// b.raw[p*MP + m] holds the raw parameters.  Five __syncthreads.
template <int CP, int TC>
__device__ void net_tile(const NetDev& w, const NetTileBufs& b) {
    constexpr int F = CP / 16;
    const int t = threadIdx.x, pg = t & 15, og = t >> 4;
    const bool worker = t < NT_THREADS;                  // extra warps only join the barriers
    float acc[4][F];
    tile_copy(b.wbuf, w.mwI, TC * CP);                   // masked layer (kernels.py:98-113)
    __syncthreads();
    if (worker) {
        tile_layer<TC, F>(b.act0, b.wbuf, CP, og, pg, acc);
        tile_store_act<F>(acc, w.mb, og, pg, b.act1);
    }
    __syncthreads();
    float* in = b.act1;
    float* out = b.act0;
    for (int l = 0; l < w.NH; l++) {                     // hidden 1x1 layers (kernels.py:69-80)
        tile_copy(b.wbuf, w.hwI + (int64_t)l * CP * CP, CP * CP);
        __syncthreads();
        if (worker) {
            tile_layer<CP, F>(in, b.wbuf, CP, og, pg, acc);
            tile_store_act<F>(acc, w.hb + l * CP, og, pg, out);
        }
        __syncthreads();
        float* tmp = in; in = out; out = tmp;
    }
    tile_copy(b.wbuf, w.owI, CP * w.MT);                  // output layer (kernels.py:81-85)
    __syncthreads();
    const int FO = worker ? w.MT / 16 : 0;                // outputs per thread (<= 12)
    float oacc[4][12];
#pragma unroll
    for (int p = 0; p < 4; p++)
#pragma unroll
        for (int f = 0; f < 12; f++) oacc[p][f] = 0.0f;
#pragma unroll 2
    for (int i = 0; i < (worker ? CP : 0); i++) {
        const float4 a = *reinterpret_cast<const float4*>(in + i * NT_TP + 4 * pg);
        const float* wr = b.wbuf + i * w.MT + og * FO;
#pragma unroll
        for (int f = 0; f < 12; f++) {
            if (f < FO) {
                const float wv = wr[f];
                oacc[0][f] = __fadd_rn(oacc[0][f], __fmul_rn(wv, a.x));
                oacc[1][f] = __fadd_rn(oacc[1][f], __fmul_rn(wv, a.y));
                oacc[2][f] = __fadd_rn(oacc[2][f], __fmul_rn(wv, a.z));
                oacc[3][f] = __fadd_rn(oacc[3][f], __fmul_rn(wv, a.w));
            }
        }
    }
#pragma unroll
    for (int f = 0; f < 12; f++) {
        const int m = og * FO + f;
        if (f < FO && m < w.M) {
            const float bb = __ldg(w.ob + m);
#pragma unroll
            for (int p = 0; p < 4; p++) b.raw[(4 * pg + p) * w.MP + m] = __fadd_rn(oacc[p][f], bb);
        }
    }
    __syncthreads();
}

}  // namespace lpic
