// lpic_sched.cuh -- decoding schedules and causal-context gathers on device.
//
// All three reference schedules (/root/reference/pkg/src/lpic/schedules.py:72-133)
// are linear: pixel (i,j) is decoded at step a*i + j with a = W (sequential),
// h+1 (wavefront) or 1 (diagonal); inside a step pixels go in ascending i
// (raster) order, which is the bitstream order (schedules.py:1-9).
#pragma once
#include <cstdint>

namespace lpic {

__host__ __device__ __forceinline__ int sched_a(int mode, int W, int h) {
    return mode == 0 ? W : (mode == 1 ? h + 1 : 1);
}
__host__ __device__ __forceinline__ int64_t sched_steps(int mode, int H, int W, int h) {
    return (int64_t)sched_a(mode, W, h) * (H - 1) + W;
}
// rows of step t: [i_lo, i_hi] (empty if i_lo > i_hi)
__host__ __device__ __forceinline__ void sched_rows(int64_t t, int a, int H, int W, int& i_lo, int& i_hi) {
    const int64_t lo_num = t - W + 1;
    const int64_t lo = lo_num <= 0 ? 0 : (lo_num + a - 1) / a;
    const int64_t hi = t / a;
    i_lo = (int)lo;
    i_hi = (int)(hi < H - 1 ? hi : H - 1);
}

// byte loaders for gather_u8: read-only path (encoder) / L2, bypassing L1
// (decoder producer, which reads pixels another SM has just written)
struct LdgU8 { __device__ uint8_t operator()(const uint8_t* p) const { return __ldg(p); } };
// normalize_value computed in place of a table lookup (network.py:172-177):
// v / 127.5 - 1 with the quotient formed as q0 = v * rcp, one residual
// correction q0 + (v - q0 * 127.5) * rcp (two FMAs) -- equal to the correctly
// rounded division __fdiv_rn(v, 127.5f) for every byte v (checked with exact
// rational arithmetic on all 256), so bit-identical to the tables built with
// __fdiv_rn, without the division subroutine on the gather path
struct NormU8 {
    __device__ float operator[](uint32_t v) const {
        constexpr float rcp = 1.0f / 127.5f;
        const float x = (float)v;
        const float q0 = __fmul_rn(x, rcp);
        const float q = __fmaf_rn(__fmaf_rn(-q0, 127.5f, x), rcp, q0);
        return __fsub_rn(q, 1.0f);
    }
};
struct LdcgU8 { __device__ uint8_t operator()(const uint8_t* p) const { return __ldcg(p); } };

template <int HH> struct Taps {
    static constexpr int T = (2 * HH + 1) * HH + HH;
    static constexpr int TC = 3 * T;
    __host__ __device__ static constexpr int di(int k) { return k < (2 * HH + 1) * HH ? -HH + k / (2 * HH + 1) : 0; }
    __host__ __device__ static constexpr int dj(int k) {
        return k < (2 * HH + 1) * HH ? -HH + k % (2 * HH + 1) : -HH + (k - (2 * HH + 1) * HH);
    }
};

// NB consecutive bytes from p through aligned 32-bit read-only loads (may read
// up to 3 bytes past p + NB; callers guarantee those lie inside the image)
template <int NB>
__device__ __forceinline__ void load_run_u8(const uint8_t* p, uint32_t (&b)[NB]) {
    constexpr int NW = (NB + 3) / 4 + 1;
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
    const uint32_t sh = (uint32_t)(a & 3) * 8u;
    uint32_t v[NW];
#pragma unroll
    for (int k = 0; k < NW; k++) v[k] = (4 * k < NB + (int)(a & 3)) ? __ldg(w + k) : 0u;
#pragma unroll
    for (int k = 0; k < NW - 1; k++) {
        const uint32_t u = __funnelshift_r(v[k], v[k + 1], sh);   // bytes 4k .. 4k+3 of the run
#pragma unroll
        for (int q = 0; q < 4; q++)
            if (4 * k + q < NB) b[4 * k + q] = (u >> (8 * q)) & 0xFFu;
    }
}

// Causal taps of pixel (i,j) from a u8 image (zero padding outside;
// kernels.py:101-108 / codec.py:93-96), normalised through `lut`.  In
// diagonal mode the taps (-1,1), (-1,2), (-2,2) are redirected to (i-2,j+1)
// or the first decoded in-bounds tap (schedules.py:114-131; h = 2 only).
// LOAD(ptr) abstracts the load (L1-bypassing in the decoder).
template <int HH, typename Load, typename Lut>
__device__ __forceinline__ void gather_u8(const uint8_t* im, int H, int W, int i, int j, int mode,
                                          const Lut& lut, float (&x)[Taps<HH>::TC], Load load) {
    constexpr int T = Taps<HH>::T;
#pragma unroll
    for (int k = 0; k < T; k++) {
        const int ii = i + Taps<HH>::di(k), jj = j + Taps<HH>::dj(k);
        if (ii >= 0 && ii < H && jj >= 0 && jj < W) {
            const uint8_t* p = im + ((int64_t)ii * W + jj) * 3;
            x[3 * k + 0] = lut[load(p + 0)];
            x[3 * k + 1] = lut[load(p + 1)];
            x[3 * k + 2] = lut[load(p + 2)];
        } else {
            x[3 * k + 0] = 0.0f; x[3 * k + 1] = 0.0f; x[3 * k + 2] = 0.0f;
        }
    }
    if constexpr (HH == 2) {
        if (mode == 2) {
            // source pixel: (i-2, j+1) if inside, else the first in-bounds tap on an
            // earlier anti-diagonal in canonical order, else padding (None -> 0.0)
            int si = i - 2, sj = j + 1;
            bool found = (si >= 0 && si < H && sj >= 0 && sj < W);
            if (!found) {
#pragma unroll
                for (int k = 0; k < T; k++) {
                    const int ci = i + Taps<HH>::di(k), cj = j + Taps<HH>::dj(k);
                    if (!found && ci >= 0 && ci < H && cj >= 0 && cj < W && Taps<HH>::di(k) + Taps<HH>::dj(k) < 0) {
                        si = ci; sj = cj; found = true;
                    }
                }
            }
            float v0 = 0.0f, v1 = 0.0f, v2 = 0.0f;
            if (found) {
                const uint8_t* p = im + ((int64_t)si * W + sj) * 3;
                v0 = lut[load(p + 0)]; v1 = lut[load(p + 1)]; v2 = lut[load(p + 2)];
            }
            // tap indices of (-1,1)=8, (-1,2)=9, (-2,2)=4 in the h=2 canonical order
            const int kk[3] = {8, 9, 4};
#pragma unroll
            for (int u = 0; u < 3; u++) {
                const int k = kk[u];
                const int ti = i + Taps<HH>::di(k), tj = j + Taps<HH>::dj(k);
                if (ti >= 0 && ti < H && tj >= 0 && tj < W) {
                    x[3 * k + 0] = v0; x[3 * k + 1] = v1; x[3 * k + 2] = v2;
                }
            }
        }
    }
}

// gather_u8 for the compat encoder network (read-only images): interior
// pixels load each tap row as one byte run through aligned word loads (12
// taps = 36 bytes in 12 loads instead of 36); edge pixels and the diagonal
// substitution take gather_u8.  Same values as gather_u8.  (-0.45% compat
// encode; in the FAST network, whose gather normalises in registers, the
// funnel shifts cost more than the byte loads: 5.45 -> 5.64 ms, r4l.)
template <int HH, typename Lut>
__device__ __forceinline__ void gather_u8_runs(const uint8_t* im, int H, int W, int i, int j, int mode,
                                               const Lut& lut, float (&x)[Taps<HH>::TC]) {
    constexpr int RW = 2 * HH + 1;                         // taps per upper row
    if (i >= HH && j >= HH && j + HH < W && !(HH == 2 && mode == 2)) {
#pragma unroll
        for (int r = 0; r < HH; r++) {                     // rows i-HH .. i-1, columns j-HH .. j+HH
            uint32_t b[3 * RW];
            // (the run ends before pixel (i-HH+r, j+HH+1), which is inside the
            // image or the first pixel of the next row: the word over-read stays in bounds)
            load_run_u8<3 * RW>(im + ((int64_t)(i - HH + r) * W + (j - HH)) * 3, b);
#pragma unroll
            for (int q = 0; q < 3 * RW; q++) x[3 * RW * r + q] = lut[b[q]];
        }
        uint32_t b[3 * HH];                                // row i, columns j-HH .. j-1 (over-read: pixel (i,j))
        load_run_u8<3 * HH>(im + ((int64_t)i * W + (j - HH)) * 3, b);
#pragma unroll
        for (int q = 0; q < 3 * HH; q++) x[3 * RW * HH + q] = lut[b[q]];
        return;
    }
    gather_u8<HH>(im, H, W, i, j, mode, lut, x, LdgU8());
}

}  // namespace lpic
