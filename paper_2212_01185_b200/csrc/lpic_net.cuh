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
    float one;                  // 1.0f at run time (tile_layer's packed FFMA2 must not fold it)
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
    float* wbuf;     // layer weight double buffer: 2 x wstride floats
    int wstride;     // net_wbuf_floats = max(TC*CP, CP*CP, CP*MT)
    float* raw;      // [NT_TP][MP] output
    uint64_t* wbar;  // 2 mbarriers: weights of buffer b landed
    uint32_t wuse0, wuse1;   // completed waits per buffer (every thread keeps the same count)
};

__host__ __device__ constexpr size_t net_wbuf_floats(int CP, int TC, int MT) {
    return (size_t)((TC * CP > CP * CP ? TC * CP : CP * CP) > CP * MT ? (TC * CP > CP * CP ? TC * CP : CP * CP)
                                                                       : CP * MT);
}
__host__ __device__ constexpr size_t net_tile_floats(int CP, int TC, int MT, int MP) {
    return (size_t)(CP > TC ? CP : TC) * NT_TP + (size_t)CP * NT_TP + 2 * net_wbuf_floats(CP, TC, MT) +
           (size_t)NT_TP * MP + 8;   // + 2 mbarriers (4 floats each, 16-byte aligned)
}
// carve the buffers out of `base` (16-byte aligned, net_tile_floats floats)
__device__ __forceinline__ void net_tile_carve(float* base, int CP, int TC, int MT, int MP, NetTileBufs& nb) {
    nb.act0 = base;
    nb.act1 = nb.act0 + (CP > TC ? CP : TC) * NT_TP;
    nb.wbuf = nb.act1 + CP * NT_TP;
    nb.wstride = (int)net_wbuf_floats(CP, TC, MT);
    nb.raw = nb.wbuf + 2 * nb.wstride;
    nb.wbar = reinterpret_cast<uint64_t*>(nb.raw + NT_TP * MP);   // 16-byte aligned (NT_TP * MP % 4 == 0)
    nb.wuse0 = nb.wuse1 = 0;
}
__device__ __forceinline__ uint32_t nt_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// thread 0, once per CTA (callers fence + __syncthreads afterwards)
__device__ __forceinline__ void net_tile_init(const NetTileBufs& nb) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(nt_smem(&nb.wbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(nt_smem(&nb.wbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// thread 0: bulk-copy layer l's input-major weights into buffer b
__device__ __forceinline__ void net_tile_load(const NetDev& w, const NetTileBufs& nb, int l, int b) {
    const int nl = w.NH + 2;
    const float* src = l == 0 ? w.mwI : (l < nl - 1 ? w.hwI + (int64_t)(l - 1) * w.CP * w.CP : w.owI);
    const uint32_t bytes = (uint32_t)(4 * (l == 0 ? w.TC * w.CP : (l < nl - 1 ? w.CP * w.CP : w.CP * w.MT)));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(nt_smem(&nb.wbar[b])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(nt_smem(nb.wbuf + (b ? nb.wstride : 0))), "l"(src), "r"(bytes), "r"(nt_smem(&nb.wbar[b])) : "memory");
}
// thread 0: request the first layer of the next tile (buffer 0 must be idle)
__device__ __forceinline__ void net_tile_prefetch(const NetDev& w, const NetTileBufs& nb) {
    if (threadIdx.x == 0) net_tile_load(w, nb, 0, 0);
}
__device__ __forceinline__ void net_tile_wait(NetTileBufs& nb, int b) {
    const uint32_t parity = (b ? nb.wuse1 : nb.wuse0) & 1u;
    if (b) nb.wuse1++; else nb.wuse0++;
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(nt_smem(&nb.wbar[b])), "r"(parity) : "memory");
    }
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

// Packed fp32 pairs (sm_100 FMUL2 / FFMA2): two pixels' products in one
// instruction.  acc = fl(acc + fl(w * a)) stays two roundings: the product
// is an FMUL2 and the sum an FFMA2 of that product times ONE, a runtime 1.0f
// (NetDev::one) ptxas cannot fold -- with a literal 1.0 it contracts the
// pair into a single fused FFMA2, which would change the result.  Both
// IEEE-exact per lane (checked in scripts/ubench_phi_peak.cu on 2^23 pairs
// and end to end by the bitwise network tests); the FP32 pipe rate is the
// same, but half the issue slots leave room for the operand loads.
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long f2_mac(unsigned long long acc, unsigned long long w2, unsigned long long a2,
                                                     unsigned long long one2) {
    unsigned long long p, r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(w2), "l"(a2));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(p), "l"(one2), "l"(acc));
    return r;
}

// acc[p][f] = sum_{i<KD} W[i][og*F+f] * in[i][4pg+p], i ascending.  The
// operands of row i+1 are loaded while row i is multiplied (register double
// buffer), so the shared-memory latency hides behind the 8F products.
template <int KD, int F>
__device__ __forceinline__ void tile_layer(const float* in, const float* W, int nout, int og, int pg,
                                           float (&acc)[4][F], float one) {
    unsigned long long a01[F], a23[F];                  // pixel pairs (0,1), (2,3)
    const unsigned long long one2 = f2_pack(one, one);
#pragma unroll
    for (int f = 0; f < F; f++) { a01[f] = 0ull; a23[f] = 0ull; }
    const float* ap = in + 4 * pg;
    const float* wp = W + og * F;
    float4 an = *reinterpret_cast<const float4*>(ap);
    float wn[F];
    load_w<F>(wp, wn);
#pragma unroll 2
    for (int i = 0; i < KD; i++) {
        const float4 a = an;
        float wv[F];
#pragma unroll
        for (int f = 0; f < F; f++) wv[f] = wn[f];
        const int inext = i + 1 < KD ? i + 1 : i;       // the last row reloads itself (no branch)
        an = *reinterpret_cast<const float4*>(ap + inext * NT_TP);
        load_w<F>(wp + inext * nout, wn);
        const unsigned long long x01 = f2_pack(a.x, a.y), x23 = f2_pack(a.z, a.w);
#pragma unroll
        for (int f = 0; f < F; f++) {
            const unsigned long long w2 = f2_pack(wv[f], wv[f]);
            a01[f] = f2_mac(a01[f], w2, x01, one2);
            a23[f] = f2_mac(a23[f], w2, x23, one2);
        }
    }
#pragma unroll
    for (int f = 0; f < F; f++) {
        f2_unpack(a01[f], acc[0][f], acc[1][f]);
        f2_unpack(a23[f], acc[2][f], acc[3][f]);
    }
}

// output layer with FO outputs per thread known at compile time
template <int CP, int FO>
__device__ __forceinline__ void tile_out(const NetDev& w, const float* in, const float* wo, int og, int pg, float* raw) {
    float acc[4][FO];
    tile_layer<CP, FO>(in, wo, w.MT, og, pg, acc, w.one);
#pragma unroll
    for (int f = 0; f < FO; f++) {
        const int m = og * FO + f;
        if (m < w.M) {
            const float bb = __ldg(w.ob + m);
#pragma unroll
            for (int p = 0; p < 4; p++) raw[(4 * pg + p) * w.MP + m] = __fadd_rn(acc[p][f], bb);
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

// Network of one tile.  On entry b.act0 holds the taps as [tc][p] and layer
// 0's weights were requested (net_tile_prefetch); on exit b.raw[p*MP + m]
// holds the raw parameters.  Layer l+1's weights stream into the other
// buffer (cp.async.bulk) while layer l computes.
template <int CP, int TC>
__device__ void net_tile(const NetDev& w, NetTileBufs& b) {
    constexpr int F = CP / 16;
    const int t = threadIdx.x, pg = t & 15, og = t >> 4;
    const bool worker = t < NT_THREADS;                  // extra warps only join the barriers
    const int nl = w.NH + 2;
    float acc[4][F];
    // masked layer (kernels.py:98-113)
    net_tile_wait(b, 0);
    if (t == 0) net_tile_load(w, b, 1, 1);
    if (worker) {
        tile_layer<TC, F>(b.act0, b.wbuf, CP, og, pg, acc, w.one);
        tile_store_act<F>(acc, w.mb, og, pg, b.act1);
    }
    __syncthreads();
    float* in = b.act1;
    float* out = b.act0;
    for (int l = 0; l < w.NH; l++) {                     // hidden 1x1 layers (kernels.py:69-80)
        const int L = l + 1, buf = L & 1;
        net_tile_wait(b, buf);
        if (t == 0 && L + 1 < nl) net_tile_load(w, b, L + 1, buf ^ 1);
        if (worker) {
            tile_layer<CP, F>(in, b.wbuf + (buf ? b.wstride : 0), CP, og, pg, acc, w.one);
            tile_store_act<F>(acc, w.hb + l * CP, og, pg, out);
        }
        __syncthreads();
        float* tmp = in; in = out; out = tmp;
    }
    const int ob = (nl - 1) & 1;                         // output layer (kernels.py:81-85)
    net_tile_wait(b, ob);
    const float* wo = b.wbuf + (ob ? b.wstride : 0);
    const int FO = worker ? w.MT / 16 : 0;                // outputs per thread (<= 12)
    if (FO == 3) {                                        // K = 3, 4 (the reference default)
        tile_out<CP, 3>(w, in, wo, og, pg, b.raw);
    } else if (FO == 2) {
        tile_out<CP, 2>(w, in, wo, og, pg, b.raw);
    } else if (FO == 4) {
        tile_out<CP, 4>(w, in, wo, og, pg, b.raw);
    } else if (FO > 0) {
    float oacc[4][12];
#pragma unroll
    for (int p = 0; p < 4; p++)
#pragma unroll
        for (int f = 0; f < 12; f++) oacc[p][f] = 0.0f;
#pragma unroll 2
    for (int i = 0; i < CP; i++) {
        const float4 a = *reinterpret_cast<const float4*>(in + i * NT_TP + 4 * pg);
        const float* wr = wo + i * w.MT + og * FO;
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
    }
    __syncthreads();
}

}  // namespace lpic
