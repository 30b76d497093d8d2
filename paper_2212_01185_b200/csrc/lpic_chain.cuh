// lpic_chain.cuh -- the decoder's on-chain table builder + symbol search.
//
// One quantised CDF table (kernels._quantized_cdf, kernels.py:250-293, fed
// by the g/b branch of kernels._channel_mixture, kernels.py:212-247) and the
// range-decoder symbol lookup (coder.py:98-106) per call, built by the 4
// chain warps of the consumer CTA (128 threads).  This is the critical path
// of the whole decoder (two calls per pixel, SURVEY §7 hard part 3); it is
// laid out for latency and instruction count, with three barriers:
//
//   P  thread t: CDF at the upper edges of bins 2t, 2t+1 for every component
//      (2K interleaved Phi chains, phi_gauss_vec); lane 31 -> edge slot;
//      barrier E; PMF with the reference's per-component order and d > 0
//      rule; exact fixed-point warp partial of the total; barrier T
//   Q  scale, floor, m = f + 1, remainder fr = v - f, 8-bit remainder
//      digit d = floor(256 fr) into a shared histogram (red.shared.add;
//      digit 0 -- the tails -- counted per warp with one REDUX; the
//      histogram is zeroed between E and T); per warp: exclusive prefix of
//      m; barrier A
//   S  every warp redundantly (so no further barrier), lane l owning bins
//      and digits 8l..8l+7: deficit; the digit bucket B holding the
//      deficit-th largest remainder (suffix sums by a warp scan); if B is
//      split (it holds ~1-2 bins), its members are ranked exactly
//      (remainder desc, index asc == the reference's stable argsort of
//      f - v, kernels.py:286-290; warp_rank_pick, or warp_crowded_pick's
//      radix levels first for > 32 members); cdf = prefix of m + prefix of
//      the +1s; symbol search against the target.
//
// The arithmetic is bin-for-bin identical to the warp builder (lpic_cdf.cuh
// warp_table), so encoder and decoder agree (scripts/ubench_chain.cu checks
// it on 288k random tables; tests/test_gpu_parity.py end to end).
#pragma once
#include "lpic_cdf.cuh"

namespace lpic {

constexpr int CH_THREADS = 128;
constexpr int CH_WARPS = 4;

// barrier of the 128 threads of one chain (named barrier `id`; loader and
// publisher warps never join; a CTA may run several chains, each on its own id)
__device__ __forceinline__ void chain_sync(int id = 1) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

struct ChainSmem {
    alignas(16) double frac[256];                 // remainders v - f (selection keys)
    alignas(16) uint32_t mpk[CH_THREADS];         // m of bins 2t | 2t+1 << 16
    alignas(16) uint8_t dig[256];                 // remainder digits floor(256 fr)
    alignas(16) unsigned long long wq[CH_WARPS];  // per-warp fixed-point PMF sums
    alignas(16) int wm[CH_WARPS];                 // per-warp sums of m
    alignas(16) double wedge[CH_WARPS][KMAX];     // each warp's last upper-edge CDF value per component
    alignas(16) uint32_t hist[256];               // 8-bit remainder-digit histogram (digits 1..255)
    alignas(16) int wz[CH_WARPS];                 // per-warp count of digit-0 bins
    float wedgeq[CH_WARPS][KMAX];                 // (FAST) last upper edge as (Q, above-zero)
    int wedgep[CH_WARPS][KMAX];
    alignas(16) uint32_t whist[CH_WARPS][256];    // per-warp histograms of a crowded threshold bucket
};

// key order of the reference's deficit selection: larger remainder first,
// ties to the lower bin index
__device__ __forceinline__ bool beats(double fa, int ja, double fb, int jb) {
    return fa > fb || (fa == fb && ja < jb);
}

// optional phase timestamps (microbenchmarks only): define LPIC_CHAIN_PROF to
// a __shared__ long long accumulator array before including this header
#ifdef LPIC_CHAIN_PROF
#define CHP(i) do { if (threadIdx.x == 0) { long long _c = clock64(); LPIC_CHAIN_PROF[i] += _c - _chp; _chp = _c; } } while (0)
#define CHP0 long long _chp = clock64()
#else
#define CHP(i) do {} while (0)
#define CHP0 do {} while (0)
#endif

// sum over the lanes selected by `mask` of a small per-lane count, via
// bit-sliced ballots (BITS bits of the count)
template <int BITS>
__device__ __forceinline__ int lanes_sum_masked(int c, uint32_t mask) {
    int s = 0;
#pragma unroll
    for (int j = 0; j < BITS; j++) s += __popc(__ballot_sync(0xffffffffu, (c >> j) & 1) & mask) << j;
    return s;
}

// 0x00/0xFF bytes of two words -> 8 bits
__device__ __forceinline__ uint32_t bits8(uint32_t lo, uint32_t hi) {
    return ((lo & 0x01010101u) * 0x01020408u >> 24) | (((hi & 0x01010101u) * 0x01020408u >> 24) << 4);
}


// KU > 0: compile-time component count; KU == 0: runtime K (<= KMAX)
// want_sym < 0: decoder -- find the symbol whose interval holds `target`;
// want_sym >= 0: encoder -- return that symbol's (start, mass).
// F32: FAST-precision tables (float32 Phi/PMF/quantisation, lpic_cdf.cuh),
// bin-for-bin identical to warp_pmf32 / warp_quantize32.
// tgt: the range-decoder target, or a callable producing it -- called in the
// shadow of the Phi phase, so the decoder's advance/target arithmetic for
// this symbol is off the critical path.
// (Testing cdf_k * r <= code instead of cdf_k <= target in the search, so
// no quotient is formed, measured 1.3% slower: the quotient is hidden in
// the Phi phase, the products are not -- r2s A/B.)
__device__ __forceinline__ uint32_t chain_target(uint32_t v) { return v; }
template <class F>
__device__ __forceinline__ uint32_t chain_target(F& f) { return f(); }

template <int KU, bool BLUE, bool F32 = false, class Tgt = uint32_t>
__device__ __forceinline__ void chain_table(const double* __restrict__ pi, const double* __restrict__ inv,
                                            const float* __restrict__ mu0, const float* __restrict__ t1,
                                            const float* __restrict__ t2, float rn, float gn, int Kr, int dist,
                                            const CdfConsts* __restrict__ cc, ChainSmem* __restrict__ cs,
                                            Tgt&& tgt, int& sym, uint32_t& start, uint32_t& mass,
                                            int32_t* trace_row, int want_sym = -1, int bar = 1) {
    constexpr int KC = KU > 0 ? KU : KMAX;
    const int K = KU > 0 ? KU : Kr;
    const int t = threadIdx.x & (CH_THREADS - 1), lane = t & 31, w = t >> 5;   // chain-local thread
    const int k0 = 2 * t;                                   // bins k0, k0 + 1
    uint32_t target = 0;
    CHP0;
#ifdef LPIC_TGT_EARLY
    target = chain_target(tgt);          // (A/B: issued ahead of the Phi phase)
#endif

    double p0 = 0.0, p1 = 0.0;
    if constexpr (F32) {
    // ---- P (float32): Q = Phi(-|z|) and the sign at the upper edges of both bins
    const float e0 = cc->edges32[k0 + 1], e1 = cc->edges32[k0 + 2];
    float qa[KC], qb[KC];
    bool pa[KC], pb[KC];
#pragma unroll
    for (int q = 0; q < KC; q++) {
        if (KU == 0 && q >= K) break;
        const float m32 = BLUE ? __fadd_rn(__fadd_rn(mu0[q], __fmul_rn(t1[q], rn)), __fmul_rn(t2[q], gn))
                               : __fadd_rn(mu0[q], __fmul_rn(t1[q], rn));
        const float iv = __double2float_rn(inv[q]);
        const float z0 = __fmul_rn(__fsub_rn(e0, m32), iv), z1 = __fmul_rn(__fsub_rn(e1, m32), iv);
        qa[q] = phiq32(z0, cc->phic32); pa[q] = z0 > 0.0f;
        qb[q] = phiq32(z1, cc->phic32); pb[q] = z1 > 0.0f;
        if (k0 + 1 == 255) { qb[q] = 0.0f; pb[q] = true; }             // +inf
    }
    if (lane == 31) {
#pragma unroll
        for (int q = 0; q < KC; q++) {
            if (KU == 0 && q >= K) break;
            cs->wedgeq[w][q] = qb[q]; cs->wedgep[w][q] = pb[q];
        }
    }
#ifndef LPIC_TGT_EARLY
    target = chain_target(tgt);
#endif
    CHP(0);
    chain_sync(bar);                                                                        // E
    CHP(1);
    reinterpret_cast<uint2*>(cs->hist)[t] = make_uint2(0u, 0u);    // (read by every warp until its E)
    float f0 = 0.0f, f1 = 0.0f;
#pragma unroll
    for (int q = 0; q < KC; q++) {
        if (KU == 0 && q >= K) break;
        float qp = __shfl_up_sync(0xffffffffu, qb[q], 1);
        bool pp = __shfl_up_sync(0xffffffffu, (int)pb[q], 1) != 0;
        if (lane == 0) {
            if (w == 0) { qp = 0.0f; pp = false; }                           // -inf
            else { qp = cs->wedgeq[w - 1][q]; pp = cs->wedgep[w - 1][q] != 0; }
        }
        const float d0 = bin_prob32(qp, pp, qa[q], pa[q]), d1 = bin_prob32(qa[q], pa[q], qb[q], pb[q]);
        const float piq = __double2float_rn(pi[q]);
        const float n0 = __fadd_rn(f0, __fmul_rn(piq, d0)), n1 = __fadd_rn(f1, __fmul_rn(piq, d1));
        f0 = d0 > 0.0f ? n0 : f0;
        f1 = d1 > 0.0f ? n1 : f1;
    }
    p0 = (double)f0; p1 = (double)f1;                  // exact; used only through fx_bin and the fp32 quantiser
    {
        const unsigned long long wsum = fx_warp_sum(fx_bin(p0) + fx_bin(p1));
        if (lane == 0) cs->wq[w] = wsum;
    }
    CHP(2);
    chain_sync(bar);                                                                        // T
    CHP(3);
    } else {
    // ---- P: CDF at the upper edges of both bins, every component
    const double e0 = cc->edges[k0 + 1], e1 = cc->edges[k0 + 2];
    double cur[2 * KC];
    {
        double z[2 * KC];
#pragma unroll
        for (int q = 0; q < KC; q++) {
            if (KU == 0 && q >= K) { z[2 * q] = 0.0; z[2 * q + 1] = 0.0; continue; }
            const float m32 = BLUE ? __fadd_rn(__fadd_rn(mu0[q], __fmul_rn(t1[q], rn)), __fmul_rn(t2[q], gn))
                                   : __fadd_rn(mu0[q], __fmul_rn(t1[q], rn));      // kernels.py:236-240
            const double mu = (double)m32, iv = inv[q];
            z[2 * q] = __dmul_rn(__dsub_rn(e0, mu), iv);
            z[2 * q + 1] = __dmul_rn(__dsub_rn(e1, mu), iv);
        }
        CHP(11);
        if (KU > 0 && dist == 0) {
#ifdef ABL_NOPHI
#pragma unroll
            for (int i = 0; i < 2 * KC; i++) cur[i] = (double)__frcp_rn(1.0f + __expf(-1.702f * (float)z[i]));   // logistic stub: Kaiming-like shapes, no fp64 polynomial
#else
            phi_gauss_vec<2 * KC>(z, cur, cc->phic);
#endif
        } else {
#pragma unroll
            for (int i = 0; i < 2 * KC; i++) {
                if (KU == 0 && i >= 2 * K) break;
                cur[i] = cdf_value(z[i], dist, cc->phic);
            }
        }
        CHP(12);
        if (k0 + 1 == 255) {
#pragma unroll
            for (int q = 0; q < KC; q++) cur[2 * q + 1] = 1.0;          // kernels.py:263
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int q = 0; q < KC; q++) {
            if (KU == 0 && q >= K) break;
            cs->wedge[w][q] = cur[2 * q + 1];
        }
    }
#ifndef LPIC_TGT_EARLY
    target = chain_target(tgt);
#endif
    CHP(0);
    chain_sync(bar);                                                                        // E
    CHP(1);
    reinterpret_cast<uint2*>(cs->hist)[t] = make_uint2(0u, 0u);    // (read by every warp until its E)
    // PMF (kernels.py:264-271): pmf[k] += pi_i * d for d > 0, components in order
    p0 = 0.0; p1 = 0.0;
#pragma unroll
    for (int q = 0; q < KC; q++) {
        if (KU == 0 && q >= K) break;
        double prev = __shfl_up_sync(0xffffffffu, cur[2 * q + 1], 1);
        if (lane == 0) prev = (w == 0) ? 0.0 : cs->wedge[w - 1][q];
        const double d0 = __dsub_rn(cur[2 * q], prev), d1 = __dsub_rn(cur[2 * q + 1], cur[2 * q]);
        const double piq = pi[q];
        const double n0 = __dadd_rn(p0, __dmul_rn(piq, d0)), n1 = __dadd_rn(p1, __dmul_rn(piq, d1));
        p0 = d0 > 0.0 ? n0 : p0;
        p1 = d1 > 0.0 ? n1 : p1;
    }
    {
        const unsigned long long wsum = fx_warp_sum(fx_bin(p0) + fx_bin(p1));
        if (lane == 0) cs->wq[w] = wsum;
    }
    CHP(2);
    chain_sync(bar);                                                                        // T
    CHP(3);

    }
    // ---- Q: floors, remainders, digits (kernels.py:272-285)
    {
        const ulonglong2 q01 = reinterpret_cast<const ulonglong2*>(cs->wq)[0];
        const ulonglong2 q23 = reinterpret_cast<const ulonglong2*>(cs->wq)[1];
        int m0, m1;
        double fr0, fr1;
        if constexpr (F32) {
            const float scale = __fdiv_rn(CDF_FLOOR_F, __double2float_rn(fx_total((q01.x + q01.y) + (q23.x + q23.y))));
            const float v0 = __fmul_rn((float)p0, scale), v1 = __fmul_rn((float)p1, scale);
            float f0 = floorf(v0), f1 = floorf(v1);
            f0 = f0 > CDF_FLOOR_F ? CDF_FLOOR_F : f0;
            f1 = f1 > CDF_FLOOR_F ? CDF_FLOOR_F : f1;
            m0 = (int)f0 + 1; m1 = (int)f1 + 1;
            fr0 = (double)__fsub_rn(v0, f0); fr1 = (double)__fsub_rn(v1, f1);
        } else {
            const double scale = cdf_scale(fx_total((q01.x + q01.y) + (q23.x + q23.y)));
            CHP(10);
            const double v0 = __dmul_rn(p0, scale), v1 = __dmul_rn(p1, scale);
            double f0 = floor(v0), f1 = floor(v1);
            f0 = f0 > CDF_FLOOR ? CDF_FLOOR : f0;
            f1 = f1 > CDF_FLOOR ? CDF_FLOOR : f1;
            m0 = (int)f0 + 1; m1 = (int)f1 + 1;
            fr0 = __dsub_rn(v0, f0); fr1 = __dsub_rn(v1, f1);     // == -(f - v) exactly
        }
        // 8-bit remainder digit; histogram in shared memory (digit 0 -- the
        // tails, where most bins would collide -- counted per warp instead;
        // counting digit 255 the same way (near-uniform PMFs) cost 100 cycles
        // per table isolated with no gain in situ, r2o)
        const int d0 = min(__double2int_rz(__dmul_rn(fr0, 256.0)), 255);
        const int d1 = min(__double2int_rz(__dmul_rn(fr1, 256.0)), 255);
        if (d0) atomicAdd(cs->hist + d0, 1u);
        if (d1) atomicAdd(cs->hist + d1, 1u);
        const int zc = __reduce_add_sync(0xffffffffu, (d0 == 0) + (d1 == 0));
        if (lane == 0) cs->wz[w] = zc;
        reinterpret_cast<double2*>(cs->frac)[t] = make_double2(fr0, fr1);
        reinterpret_cast<uint16_t*>(cs->dig)[t] = (uint16_t)(d0 | (d1 << 8));
        cs->mpk[t] = (uint32_t)m0 | ((uint32_t)m1 << 16);
        const int ms = __reduce_add_sync(0xffffffffu, m0 + m1);
        if (lane == 0) cs->wm[w] = ms;
    }
    CHP(4);
    chain_sync(bar);                                                                        // A
    CHP(5);

    // ---- S: lane l owns bins 8l..8l+7 (all in warp l >> 3)
    const int4 wm4 = *reinterpret_cast<const int4*>(cs->wm);
    const int deficit = 65536 - ((wm4.x + wm4.y) + (wm4.z + wm4.w));
    const uint2 dg = reinterpret_cast<const uint2*>(cs->dig)[lane];
    // m of this lane's bins, and the digit counts of digits 8l..8l+7
    const uint4 mk = reinterpret_cast<const uint4*>(cs->mpk)[lane];
    const uint32_t mv[4] = {mk.x, mk.y, mk.z, mk.w};
    int c[8];
    {
        const uint4 ha = reinterpret_cast<const uint4*>(cs->hist)[2 * lane];
        const uint4 hb = reinterpret_cast<const uint4*>(cs->hist)[2 * lane + 1];
        c[0] = (int)ha.x; c[1] = (int)ha.y; c[2] = (int)ha.z; c[3] = (int)ha.w;
        c[4] = (int)hb.x; c[5] = (int)hb.y; c[6] = (int)hb.z; c[7] = (int)hb.w;
        if (lane == 0) {
            const int4 z4 = *reinterpret_cast<const int4*>(cs->wz);
            c[0] = (z4.x + z4.y) + (z4.z + z4.w);
        }
    }
    // ONE warp scan for both prefixes over lanes: m (<= 65536, 17 bits) and
    // the digit counts (<= 256, 9 bits) packed as m << 9 | count
    uint32_t mpl[8], cpl[8];                                // in-lane exclusive prefixes
    mpl[0] = 0; cpl[0] = 0;
#pragma unroll
    for (int q = 1; q < 8; q++) {
        mpl[q] = mpl[q - 1] + ((mv[(q - 1) >> 1] >> (16 * ((q - 1) & 1))) & 0xFFFFu);
        cpl[q] = cpl[q - 1] + (uint32_t)c[q - 1];
    }
    const uint32_t packed = ((mpl[7] + (mv[3] >> 16)) << 9) | (cpl[7] + (uint32_t)c[7]);
    uint32_t incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    const uint32_t excl = incl - packed;
    const uint32_t mbase = excl >> 9, hbase = excl & 511u;   // m and digit counts of lower lanes
    uint32_t bm = 0;                                        // bit q: bin 8l+q gets the +1
#ifdef ABL_NOSEL
    if (deficit > 100000) {
#else
    if (deficit > 0) {
#endif
        // 8-bit digit bucket B holding the deficit-th largest remainder:
        // #digits >= b is 256 - (#digits < b), so B is the last digit whose
        // lower count is <= 256 - deficit
        {
            const uint32_t lim = 256u - (uint32_t)deficit;
            int qb = -1, nb_l = 0, sb_l = 0;
#pragma unroll
            for (int q = 0; q < 8; q++)
                if (hbase + cpl[q] <= lim) { qb = q; nb_l = c[q]; sb_l = 256 - (int)(hbase + cpl[q]); }
            const int L = 31 - __clz(__ballot_sync(0xffffffffu, qb >= 0));
            const int B = 8 * L + __shfl_sync(0xffffffffu, qb, L);
            const int nB = __shfl_sync(0xffffffffu, nb_l, L);
            const int need = deficit - (__shfl_sync(0xffffffffu, sb_l, L) - nB);   // 1 <= need <= nB
            CHP(13);
            const uint32_t Bx4 = (uint32_t)B * 0x01010101u;
            bm = bits8(__vcmpgtu4(dg.x, Bx4), __vcmpgtu4(dg.y, Bx4));
            const uint32_t mem = bits8(__vcmpeq4(dg.x, Bx4), __vcmpeq4(dg.y, Bx4));
            if (need == nB) {
                bm |= mem;
            } else {
                double fr8[8];
                const double2* f2 = reinterpret_cast<const double2*>(cs->frac) + 4 * lane;
#pragma unroll
                for (int u = 0; u < 4; u++) { const double2 v = f2[u]; fr8[2 * u] = v.x; fr8[2 * u + 1] = v.y; }
                if (nB > 32) {
                    // Crowded bucket (near-flat mixtures put most remainders in
                    // one digit): radix select on the members' remainder bits
                    // in the warp's own histogram (warp_crowded_pick, lpic_cdf.cuh)
                    bm |= warp_crowded_pick(fr8, mem, need, nB, cs->whist[w]);
                } else {
                    // exact ranks among the members of B (frac desc / index asc)
                    bm |= warp_rank_pick(fr8, mem, need, nB, cs->whist[w]);
                }
            }
        }
    }
    CHP(6);
    // ---- cdf (kernels.py:291-293) = prefix of m + prefix of the +1s; search (coder.py:104)
    const uint32_t bpre = (uint32_t)lanes_sum_masked<4>(__popc(bm), (1u << lane) - 1u);
    uint32_t cdf[8];
#pragma unroll
    for (int q = 0; q < 8; q++) cdf[q] = mbase + mpl[q] + bpre + __popc(bm & ((1u << q) - 1u));
    CHP(7);
    int L, qs = 0;
    if (want_sym >= 0) {
        L = want_sym >> 3;
        qs = want_sym & 7;
    } else {
        L = 31 - __clz(__ballot_sync(0xffffffffu, cdf[0] <= target));   // lane 0: cdf = 0
#pragma unroll
        for (int q = 1; q < 8; q++) qs += (cdf[q] <= target);
    }
    uint32_t st_mine = cdf[0], ms_mine = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) {
        if (q == qs) {
            st_mine = cdf[q];
            ms_mine = ((mv[q >> 1] >> (16 * (q & 1))) & 0xFFFFu) + ((bm >> q) & 1u);
        }
    }
    sym = 8 * L + __shfl_sync(0xffffffffu, qs, L);
    start = __shfl_sync(0xffffffffu, st_mine, L);
    mass = __shfl_sync(0xffffffffu, ms_mine, L);
    if (trace_row && w == 0) {
#pragma unroll
        for (int q = 0; q < 8; q++) trace_row[8 * lane + q] = (int32_t)cdf[q];
        if (lane == 31) trace_row[256] = 65536;
    }
    CHP(9);
}

}  // namespace lpic
