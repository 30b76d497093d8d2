// lpic_net_tc2.cuh -- the FAST encoder network as a warp-specialised,
// two-tile tcgen05 pipeline (k_enc_net_tc2).
//
// Same arithmetic as tc_network (lpic_net_tc.cuh): per layer and 128-row
// tile, D0 = A_hi.W_hi^T and D1 = A_hi.W_lo^T + A_lo.W_hi^T over the K
// slices in ascending order, y = D0 + D1 * 2^-11 + bias, LeakyReLU, re-split
// into fp16 hi/lo -- so its raw outputs are bit-identical to the decoder
// producer's tc_network and FAST streams keep round-tripping.  What changes
// is the schedule.  tc_network runs MMA -> wait -> epilogue -> barrier per
// layer, one tile at a time (tensor pipe active ~9%, ncu r1).  Here a CTA
// owns TWO tiles and four roles:
//
//   warps 0-3, 8-11   epilogue of tile 0 (thread = row = TMEM lane; warps
//                     0-3 output columns 0-63, 8-11 columns 64-127)
//   warps 4-7, 12-15  epilogue of tile 1 (TMEM columns 256..511)
//   warp 16           MMA issue: layer l of tile 0, then of tile 1, then l+1
//   warp 17           weight loader: 64-column K blocks (hi|lo, <= 32 KB)
//                     through a 3-slot ring, each used by both tiles
//
// so the epilogue of one tile (TMEM -> registers -> split -> smem) runs while
// the tensor core works on the other tile's layer.  Hand-offs are mbarriers:
// aready[t] (256 epilogue threads -> MMA: the tile's A operand for the next
// layer is in shared memory), dfull[t] (tcgen05.commit -> epilogue: the
// layer's accumulators are in TMEM), wfull[s] (bulk copy landed), wfree[s]
// (commit after tile 1's last MMA on the block).  Shared memory: 2 x 64 KB A
// operands (in place: a layer's epilogue overwrites its own input only after
// the layer's MMAs completed) + 3 x 32 KB weight slots = 224 KB, one CTA per
// SM, all 512 TMEM columns.
#pragma once
#include "lpic_net_tc.cuh"

namespace lpic {

constexpr int TC2_KB = 64;                                  // K columns per weight block
constexpr int TC2_WBLK = 2 * TC_NMAX * TC2_KB * 2;          // bytes of one block (hi | lo), 32 KB
constexpr int TC2_SLOTS = 3;                                // weight ring slots (96 KB; 6 x 16 KB measured 9% slower, r3e)
constexpr int TC2_MAXB = 2 * TC_MAXL;                       // blocks per network pass
constexpr int TC2_MAXL = 5;                                 // layers (L <= 5: the reference configs; else k_enc_net_tc)
constexpr int TC2_MMA_WARP = 16, TC2_LOAD_WARP = 17;
constexpr int TC2_THREADS = 32 * 18;           // 16 epilogue warps, MMA issue, weight loader

struct TcNet2Dev {
    const unsigned char* blk[TC2_MAXB];   // per block: W_hi (N x Kb) | W_lo (N x Kb), canonical K-major, K = Kb
    int blk_bytes[TC2_MAXB], blk_kb[TC2_MAXB], blk_k0[TC2_MAXB], blk_layer[TC2_MAXB];
    int nb;                               // blocks per pass
    int first_blk[TC_MAXL], n_blk[TC_MAXL];
    const float* bias[TC_MAXL];
    int N[TC_MAXL], K[TC_MAXL];
    int nl, M, K0;
};

struct Tc2Smem {
    alignas(128) unsigned char a_hi[2][TC_M * TC_KMAX * 2];
    alignas(128) unsigned char a_lo[2][TC_M * TC_KMAX * 2];
    alignas(128) unsigned char w[TC2_SLOTS][TC2_WBLK];
    float bias[TC2_MAXL][TC_NMAX];                          // the layers' biases (broadcast reads)
    alignas(8) uint64_t wfull[TC2_SLOTS], wfree[TC2_SLOTS], aready[2], dfull[2];
    uint32_t tmem;
};

__device__ __forceinline__ void tc2_mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(umma::smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void tc2_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_addr(b)) : "memory");
}

// Split-store a chunk of 32 fp32 values (columns c0.. of row r, ng groups of
// 8) into an A operand of K columns (the tc_store_split arithmetic).
__device__ __forceinline__ void tc2_store_split(unsigned char* a_hi, unsigned char* a_lo, int r, int c0, int K,
                                                const float (&y)[32], int ng) {
#pragma unroll
    for (int g = 0; g < 4; g++) {
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
        *reinterpret_cast<uint4*>(a_hi + off) = *reinterpret_cast<uint4*>(h);
        *reinterpret_cast<uint4*>(a_lo + off) = *reinterpret_cast<uint4*>(l);
    }
}

// the same for a 16-column chunk (two groups of 8)
__device__ __forceinline__ void tc2_store_split16(unsigned char* a_hi, unsigned char* a_lo, int r, int c0, int K,
                                                  const float (&y)[16]) {
#pragma unroll
    for (int g = 0; g < 2; g++) {
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
        *reinterpret_cast<uint4*>(a_hi + off) = *reinterpret_cast<uint4*>(h);
        *reinterpret_cast<uint4*>(a_lo + off) = *reinterpret_cast<uint4*>(l);
    }
}

template <int TC>
__device__ __forceinline__ void tc2_store_input(unsigned char* a_hi, unsigned char* a_lo, int r, const float (&x)[TC],
                                                int K) {
#pragma unroll
    for (int c0 = 0; c0 < TC_KMAX; c0 += 32) {
        if (c0 >= K) break;
        float y[32];
#pragma unroll
        for (int i = 0; i < 32; i++) y[i] = (c0 + i < TC) ? x[(c0 + i < TC) ? c0 + i : 0] : 0.0f;
        tc2_store_split(a_hi, a_lo, r, c0, K, y, (K - c0) >= 32 ? 4 : (K - c0) >> 3);
    }
}

__device__ __forceinline__ bool tc2_elect_one() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(p));
    return p != 0;
}

// MMA issue for one (tile, layer): every K block of the layer, in order.
// Executed by the whole MMA warp (so the descriptors stay warp-uniform, in
// uniform registers); one elected lane issues each tcgen05 instruction.
// gbase: global index (over the CTA's whole block stream) of the layer's
// first block; the block's ring slot is its global index mod TC2_SLOTS.  wcnt: uses
// of each slot so far (tile 0 waits for the copy, tile 1 then releases it).
// Descriptors are formed once per block: advancing a K=16 slice adds
// (offset >> 4) to the 14-bit start-address field.
__device__ __forceinline__ void tc2_issue_layer(Tc2Smem* s, const TcNet2Dev& w, int t, int l, uint32_t tbase,
                                                int64_t gbase, uint32_t (&wcnt)[TC2_SLOTS]) {
    const int N = w.N[l], K = w.K[l];
    const uint32_t idesc = umma::idesc_f16(TC_M, N);
    // W_hi (N rows) and W_lo (N rows) sit back to back in the block with the
    // canonical 8-row group stride, so together they are ONE 2N-row B
    // operand: a single N = 2N MMA writes A_hi.W_hi^T to columns [0, N) (D0)
    // and A_hi.W_lo^T to [N, 2N) (D1), then A_lo.W_hi^T accumulates into D1
    // -- two MMAs per K slice instead of three, 20 instead of 24 KB of
    // operand reads, each element accumulated in the same order as before
    const uint32_t idesc2 = umma::idesc_f16(TC_M, 2 * N);
    const uint32_t dcol = tbase + (uint32_t)(256 * t);
    const uint64_t dah = umma::smem_desc(umma::smem_addr(s->a_hi[t]), 128, (uint32_t)(K * 16));
    const uint64_t dal = umma::smem_desc(umma::smem_addr(s->a_lo[t]), 128, (uint32_t)(K * 16));
    for (int j = 0; j < w.n_blk[l]; j++) {
        const int b = w.first_blk[l] + j;
        const int slot = (int)((gbase + j) % TC2_SLOTS);
        if (t == 0) {                                       // first use of the block: wait for its copy
            tc_mbar_wait(&s->wfull[slot], wcnt[slot] & 1u);
            wcnt[slot]++;
            umma::fence_after();
        }
        const int Kb = w.blk_kb[b], k0 = w.blk_k0[b];
        const uint32_t w_hi = umma::smem_addr(s->w[slot]);
        const uint64_t dwh = umma::smem_desc(w_hi, 128, (uint32_t)(Kb * 16));
        const uint64_t oa0 = (uint64_t)(k0 >> 3) * 8u;       // (k0 / 8) * 128 bytes, >> 4
        for (int kk = 0; kk < Kb; kk += 16) {
            const bool acc = (k0 + kk) > 0;
            const uint64_t oa = oa0 + (uint64_t)(kk >> 3) * 8u, ow = (uint64_t)(kk >> 3) * 8u;
            if (tc2_elect_one()) {
                umma::mma_f16(dcol, dah + oa, dwh + ow, idesc2, acc);
                umma::mma_f16(dcol + (uint32_t)N, dal + oa, dwh + ow, idesc, true);
            }
            __syncwarp();
        }
        if (t == 1 && tc2_elect_one()) umma::commit(&s->wfree[slot]);   // both tiles done with the block
        __syncwarp();
    }
    if (tc2_elect_one()) umma::commit(&s->dfull[t]);
    __syncwarp();
}

}  // namespace lpic
