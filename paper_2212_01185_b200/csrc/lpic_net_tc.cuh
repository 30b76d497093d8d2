// lpic_net_tc.cuh -- the causal-neighbourhood network on the 5th-gen tensor
// cores (tcgen05 + TMEM): LPIC_PREC_FAST.
//
// Same network as kernels._dense_stack / forward_taps_f32
// (/root/reference/pkg/src/lpic/kernels.py:63-136), evaluated as a chain of
// 128-row GEMMs with the fp16x3 split that SURVEY App. B.5 measured to meet
// the 1e-4 parameter budget (bf16x3 does not): every fp32 operand x becomes
// hi = fp16(x), lo = fp16((x - hi) * 2^11); per layer
//     D0 = A_hi . W_hi^T            (TMEM columns [0, N))
//     D1 = A_hi . W_lo^T + A_lo . W_hi^T   (columns [N, 2N), scaled by 2^11;
//          the first term shares one N = 2N MMA with D0, the layer blob's
//          W_hi and W_lo rows forming a single 2N-row B operand)
//     y  = D0 + D1 * 2^-11 + bias, LeakyReLU (not on the output layer)
// and y is re-split into the next layer's A operand in shared memory.
// One thread issues the MMAs; the 4 warps of the tile run the epilogue
// (tcgen05.ld of their 32 TMEM lanes = their 32 rows).  Weights (fp16 hi|lo
// blobs, pre-laid-out by the host in the canonical K-major layout) stream
// from L2 into a double buffer with cp.async.bulk, one layer ahead.
//
// The encoder (k_enc_net_tc) and the decoder's producer call the same
// function, so they execute the identical MMA sequence and epilogue: FAST
// streams round-trip bit-exactly on this library (they are not decodable by
// the CPU reference, whose network runs in canonical fp32 order).
#pragma once
#include <cuda_fp16.h>

#include "lpic_umma.cuh"

namespace lpic {

constexpr int TC_M = 128;             // rows (pixels) per tile
constexpr int TC_MAXL = 8;            // layers (masked + hidden + output)
constexpr int TC_KMAX = 128;          // max padded K of any layer
constexpr int TC_NMAX = 128;          // max N
constexpr int TC_WBUF = 2 * TC_NMAX * TC_KMAX * 2;   // bytes of one layer blob (hi | lo), 64 KB

struct TcNetDev {
    const unsigned char* blob[TC_MAXL];   // per layer: W_hi (N x K) | W_lo (N x K), canonical layout
    const float* bias[TC_MAXL];           // TC_NMAX floats each (zero padded)
    int N[TC_MAXL], K[TC_MAXL];           // padded sizes (N % 16 == 0, K % 16 == 0)
    int nl;                               // layers
    int M;                                // real outputs of the last layer (12K)
    int K0;                               // real inputs of the first layer (3T)
};

struct TcSmem {
    alignas(128) unsigned char a_hi[TC_M * TC_KMAX * 2];    // A operand (canonical layout)
    alignas(128) unsigned char a_lo[TC_M * TC_KMAX * 2];
    alignas(128) unsigned char w[2][TC_WBUF];               // weight double buffer
    alignas(8) uint64_t wbar[2];                            // weight copy landed
    alignas(8) uint64_t mbar;                               // MMAs of a layer complete
    uint32_t tmem;                                          // TMEM base (256 columns)
    uint32_t wphase[2], mphase;                             // (thread-0 bookkeeping mirrors)
};

__device__ __forceinline__ void tc_mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(umma::smem_addr(b)), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void tc_load_layer(TcSmem* s, const TcNetDev& w, int l, int buf) {
    const uint32_t bytes = (uint32_t)(2 * w.N[l] * w.K[l] * 2);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(umma::smem_addr(&s->wbar[buf])), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(umma::smem_addr(s->w[buf])), "l"(w.blob[l]), "r"(bytes), "r"(umma::smem_addr(&s->wbar[buf]))
                 : "memory");
}

// One-time setup by the tile's 128 threads (warp 0 allocates TMEM).
__device__ __forceinline__ void tc_init(TcSmem* s) {
    const int tid = threadIdx.x & 127, warp = tid >> 5;
    if (warp == 0) umma::tmem_alloc(&s->tmem, 256);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(umma::smem_addr(&s->wbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(umma::smem_addr(&s->wbar[1])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(umma::smem_addr(&s->mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s->wphase[0] = s->wphase[1] = 0; s->mphase = 0;
    }
}
__device__ __forceinline__ void tc_finish(TcSmem* s) {
    if (((threadIdx.x & 127) >> 5) == 0) umma::tmem_dealloc(s->tmem, 256);
}

// Store a fp32 row chunk (columns c0 .. c0+8*ng-1 of row r, ng <= 4) as the
// split A operand of a K-column layer.
__device__ __forceinline__ void tc_store_split(TcSmem* s, int r, int c0, int K, const float (&y)[32], int ng) {
#pragma unroll
    for (int g = 0; g < 4; g++) {                        // up to 4 core-matrix rows of 8 values
        if (g >= ng) break;
        __half2 h[4], l[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float a = y[8 * g + 2 * i], b = y[8 * g + 2 * i + 1];
            const __half ha = __float2half_rn(a), hb = __float2half_rn(b);
            h[i] = __halves2half2(ha, hb);
            l[i] = __halves2half2(__float2half_rn((a - __half2float(ha)) * 2048.0f),
                                  __float2half_rn((b - __half2float(hb)) * 2048.0f));
        }
        const uint32_t off = umma::op_offset(r, c0 + 8 * g, K);
        *reinterpret_cast<uint4*>(s->a_hi + off) = *reinterpret_cast<uint4*>(h);
        *reinterpret_cast<uint4*>(s->a_lo + off) = *reinterpret_cast<uint4*>(l);
    }
}

// First-layer operand of row r from its K0 gathered taps (zero padded to K).
template <int TC>
__device__ __forceinline__ void tc_store_input(TcSmem* s, int r, const float (&x)[TC], int K) {
#pragma unroll
    for (int c0 = 0; c0 < TC_KMAX; c0 += 32) {
        if (c0 >= K) break;
        float y[32];
#pragma unroll
        for (int i = 0; i < 32; i++) y[i] = (c0 + i < TC) ? x[(c0 + i < TC) ? c0 + i : 0] : 0.0f;
        tc_store_split(s, r, c0, K, y, (K - c0) >= 32 ? 4 : (K - c0) >> 3);
    }
}

// The network of one 128-row tile.  On entry the A operand holds the first
// layer's inputs (K[0] columns, split); `first_loaded` says whether layers 0
// and 1 were already requested (tc_prefetch).  On exit raw_row[0 .. M) of
// this thread's row holds the output (thread t <-> row t).  All 128 threads
// must call it; thread 0 issues the MMAs and copies.
__device__ __forceinline__ void tc_prefetch(TcSmem* s, const TcNetDev& w) {
    if ((threadIdx.x & 127) == 0) {
        tc_load_layer(s, w, 0, 0);
        if (w.nl > 1) tc_load_layer(s, w, 1, 1);
    }
}
// mcnt: MMA-completion count of this CTA's mbar so far (every thread keeps
// the same copy; advanced by w.nl per call).
__device__ __forceinline__ void tc_network(TcSmem* s, const TcNetDev& w, float* raw_row, int raw_stride,
                                           uint32_t& mcnt) {
    const int tid = threadIdx.x & 127, warp = tid >> 5;
    const uint32_t tbase = s->tmem;
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    for (int l = 0; l < w.nl; l++) {
        const int N = w.N[l], K = w.K[l], buf = l & 1;
        // the A operand written by the generic proxy must be visible to the tensor core
        umma::fence_async_smem();
        umma::fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(15) : "memory");
        umma::fence_after();
        if (tid == 0) {
            tc_mbar_wait(&s->wbar[buf], s->wphase[buf]);
            s->wphase[buf] ^= 1u;
            umma::fence_after();
            const uint32_t idesc = umma::idesc_f16(TC_M, N);
            const uint32_t idesc2 = umma::idesc_f16(TC_M, 2 * N);     // [W_hi; W_lo] as one 2N-row operand
            const uint32_t a_hi = umma::smem_addr(s->a_hi), a_lo = umma::smem_addr(s->a_lo);
            const uint32_t w_hi = umma::smem_addr(s->w[buf]);
            const uint32_t sbo = (uint32_t)(K * 16);
            for (int ks = 0; ks < K / 16; ks++) {
                const uint32_t o = (uint32_t)ks * 256u;
                // D0 (columns [0, N)) and the hi.lo half of D1 (columns [N, 2N)) in one MMA
                umma::mma_f16(tbase, umma::smem_desc(a_hi + o, 128, sbo), umma::smem_desc(w_hi + o, 128, sbo), idesc2,
                              ks > 0);
                umma::mma_f16(tbase + (uint32_t)N, umma::smem_desc(a_lo + o, 128, sbo),
                              umma::smem_desc(w_hi + o, 128, sbo), idesc, true);
            }
            umma::commit(&s->mbar);
        }
        // every thread waits for this layer's MMAs (the A buffer is then free)
        tc_mbar_wait(&s->mbar, mcnt & 1u);
        mcnt++;
        umma::fence_after();
        if (tid == 0 && l + 2 < w.nl) tc_load_layer(s, w, l + 2, buf);   // buffer `buf` is free now
        const bool last = (l == w.nl - 1);
        const int Knext = last ? 0 : w.K[l + 1];
        for (int c0 = 0; c0 < N; c0 += 32) {
            float d0[32], d1[32];
            umma::tmem_ld32(tbase + lane_off + (uint32_t)c0, d0);
            umma::tmem_ld32(tbase + lane_off + (uint32_t)(N + c0), d1);
            float y[32];
#pragma unroll
            for (int i = 0; i < 32; i++) {
                const float v = __fadd_rn(__fadd_rn(d0[i], __fmul_rn(d1[i], 4.8828125e-4f)), __ldg(w.bias[l] + c0 + i));
                y[i] = last ? v : (v >= 0.0f ? v : __fmul_rn(0.01f, v));
            }
            if (last) {
#pragma unroll
                for (int i = 0; i < 32; i++)
                    if (raw_row && c0 + i < w.M) raw_row[(c0 + i) * raw_stride] = y[i];
            } else if (c0 < Knext) {
                tc_store_split(s, tid, c0, Knext, y, (Knext - c0) >= 32 ? 4 : (Knext - c0) >> 3);
            }
        }
        // zero the padded K columns of the next A operand (N < Knext never
        // happens: hidden K = N; the first layer's padding is written by the caller)
    }
    umma::fence_before();
}

}  // namespace lpic
