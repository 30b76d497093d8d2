// lpic_kernels.cu -- B200 (sm_100a) kernels and the C-ABI of liblpic_b200.so.
//
// Kernels (see DESIGN.md for rooflines):
//   k_enc_net / k_enc_net_tc   encoder network over 64/128-pixel tiles in
//                              coding order (compat CUDA cores / FAST tcgen05)
//                              (codec.py:116-145, kernels.py:88-114)
//   k_enc_tables<VAR,BIG>      three quantised CDF tables per pixel -> the
//                              coded symbols' (start, width) (kernels.py:296-313)
//   k_rc_plan / k_rc_chunks / k_rc_merge
//                              parallel byte-exact range coder (coder.py:30-73);
//                              the plan is fused into the table kernel's
//                              cooperative launch (it chases the symbols)
//   k_decode2                  wavefront decoder, one 2-CTA cluster per stream
//                              (producer + serial chain, lpic_decode.cuh;
//                              codec.py:193-247)
//   k_forward_taps / k_channel_cdfs / k_rc_decode_tables / k_true_*   parity seams
#include "../../include/lpic_b200.h"

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "lpic_cdf.cuh"
#include "lpic_chain.cuh"
#include "lpic_decode.cuh"
#include "lpic_math.cuh"
#include "lpic_net.cuh"
#include "lpic_net_tc.cuh"
#include "lpic_net_tc2.cuh"
#include "lpic_rc.cuh"
#include "lpic_sched.cuh"
#include "lpic_decode_launch.h"

namespace lpic {
cudaError_t launch_decode2(int CP, int HH, int S, int n, size_t smem, cudaStream_t st, const DecParams& P) {
    switch (CP) {
        case 16: return launch_decode2_cp16(HH, S, n, smem, st, P);
        case 32: return launch_decode2_cp32(HH, S, n, smem, st, P);
        case 64: return launch_decode2_cp64(HH, S, n, smem, st, P);
        case 128: return launch_decode2_cp128(HH, S, n, smem, st, P);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace lpic

using namespace lpic;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            return fail(LPIC_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
    } while (0)

constexpr int NET_THREADS = 128;   // pixels per CTA tile (encoder) / per decoder chunk



template <int CP>
__host__ __device__ constexpr size_t net_smem_bytes(int MP) {
    return (size_t)NET_THREADS * MP * sizeof(float) + (size_t)CP * NET_THREADS * sizeof(float);
}

// write the warp-held table as an int32 cdf[257] row
__device__ __forceinline__ void store_cdf_row(int32_t* row, const uint32_t start[8], const uint32_t mass[8]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < 8; q++) row[8 * lane + q] = (int32_t)start[q];
    if (lane == 31) row[256] = (int32_t)(start[7] + mass[7]);
}

// ---------------------------------------------------------------------------
// encoder, stage 1: the network over 64-pixel RASTER runs (codec.py:116-145 +
// kernels.py:88-114): gather -> net_tile -> raw plane rows in coding order
// (inv: raster index -> coding index).  Adjacent lanes gather adjacent
// pixels, so each tap load is one short run of bytes.
// ---------------------------------------------------------------------------
template <int CP, int HH>
__global__ void __launch_bounds__(NT_THREADS)
k_enc_net(NetDev w, const uint8_t* __restrict__ images, int H, int W, int mode, const int32_t* __restrict__ inv,
          int64_t N, float* __restrict__ raw_out, int32_t* status, float* trace_raw) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int TC = Taps<HH>::TC;
    __shared__ float lut[256];
    __shared__ int32_t cidx[NT_TP];
    float* fb = reinterpret_cast<float*>(smem);
    NetTileBufs nb;
    net_tile_carve(fb, CP, TC, w.MT, w.MP, nb);
    if (threadIdx.x == 0) {
        net_tile_init(nb);
        net_tile_load(w, nb, 0, 0);                       // layer 0 streams in during the gather
    }
    for (int v = threadIdx.x; v < 256; v += blockDim.x) lut[v] = __fsub_rn(__fdiv_rn((float)v, 127.5f), 1.0f);
    __syncthreads();
    const int img = blockIdx.y, tid = threadIdx.x;
    const int64_t n0 = (int64_t)blockIdx.x * NT_TP;
    const uint8_t* im = images + (int64_t)img * N * 3;
    if (tid < NT_TP) {
        float x[TC];
        const int64_t n = n0 + tid;
        if (n < N) {
            const int i = (int)(n / W), j = (int)(n - (int64_t)i * W);
            gather_u8_runs<HH>(im, H, W, i, j, mode, lut, x);
            cidx[tid] = __ldg(inv + n);
        } else {
#pragma unroll
            for (int q = 0; q < TC; q++) x[q] = 0.0f;
        }
#pragma unroll
        for (int q = 0; q < TC; q++) nb.act0[q * NT_TP + tid] = x[q];
    }
    __syncthreads();
    net_tile<CP, TC>(w, nb);
    const int np = (int)((N - n0) < NT_TP ? (N - n0) : NT_TP);
    bool finite = true;
    for (int e = tid; e < np * w.M; e += NT_THREADS) {
        const int p = e / w.M, m = e - p * w.M;
        const float v = nb.raw[p * w.MP + m];
        finite &= isfinite(v);
        raw_out[((int64_t)img * N + cidx[p]) * w.M + m] = v;
        if (trace_raw) trace_raw[((int64_t)img * N + cidx[p]) * w.M + m] = v;
    }
    if (!finite) atomicOr(status + img, LPIC_S_NONFINITE);
}

// ---------------------------------------------------------------------------
// encoder, stage 1 in FAST precision: the network on the tensor cores
// (lpic_net_tc.cuh), persistent CTAs of 128 threads over 128-pixel tiles in
// coding order; the next tile's first two weight layers stream in while the
// current tile's last layers run.
// ---------------------------------------------------------------------------
template <int HH>
__global__ void __launch_bounds__(128, 1)
k_enc_net_tc(const __grid_constant__ TcNetDev w, const uint8_t* __restrict__ images, int H, int W, int mode,
             const int32_t* __restrict__ order, int64_t N, int n_img, float* __restrict__ raw_out, int32_t* status,
             float* trace_raw) {
    extern __shared__ __align__(128) unsigned char smem[];
    TcSmem* s = reinterpret_cast<TcSmem*>(smem);
    __shared__ float lut[256];
    constexpr int TC = Taps<HH>::TC;
    const int tid = threadIdx.x;
    for (int v = tid; v < 256; v += 128) lut[v] = __fsub_rn(__fdiv_rn((float)v, 127.5f), 1.0f);
    tc_init(s);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const int64_t tiles_per = (N + TC_M - 1) / TC_M, total = tiles_per * n_img;
    uint32_t mcnt = 0;
    if ((int64_t)blockIdx.x < total) tc_prefetch(s, w);
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int64_t img = tile / tiles_per, n = (tile - img * tiles_per) * TC_M + tid;
        float x[TC];
        if (n < N) {
            const int32_t ij = __ldg(order + n);
            gather_u8<HH>(images + img * N * 3, H, W, ij >> 16, ij & 0xFFFF, mode, lut, x, LdgU8());
        } else {
#pragma unroll
            for (int q = 0; q < TC; q++) x[q] = 0.0f;
        }
        tc_store_input<TC>(s, tid, x, w.K[0]);
        float* row = (n < N) ? raw_out + (img * N + n) * w.M : nullptr;
        tc_network(s, w, row, 1, mcnt);
        if (tile + gridDim.x < total) tc_prefetch(s, w);
        if (row) {
            bool finite = true;
            for (int m = 0; m < w.M; m++) {
                const float v = row[m];
                finite &= isfinite(v);
                if (trace_raw) trace_raw[(img * N + n) * w.M + m] = v;
            }
            if (!finite) atomicOr(status + img, LPIC_S_NONFINITE);
        }
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    tc_finish(s);
}

constexpr int RC_CH = 1024;
constexpr int RC_CHUNK = 256;
static_assert(RC_CH % RC_CHUNK == 0 && (RC_CH & (RC_CH - 1)) == 0, "chunk boundaries on block starts");

constexpr uint32_t RC_PENDING = 0xFFFFFFFFu;    // sw sentinel: start 65535 + width 65536 cannot occur
constexpr unsigned long long RC_STALL_NS = 4000000000ull;   // chase: no new symbol for 4 s -> give up
__device__ __forceinline__ uint32_t ld_relaxed_sw(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sw(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long rc_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// chase: the symbols are still being produced (by the table warps of the same
// cooperative launch); wait for each until it is no longer RC_PENDING.  The
// wait is bounded by wall time without progress; once it trips, every later
// load is a plain load (no further waiting).
__device__ __forceinline__ void rc_sym_load(const uint32_t* __restrict__ p, int64_t n, int64_t c, int lane,
                                            uint32_t (&nxt)[RC_CHUNK / 32], bool chase, bool& timed_out) {
#pragma unroll
    for (int q = 0; q < RC_CHUNK / 32; q++) {
        const int64_t k = c + 32 * q + lane;
        nxt[q] = (k < n) ? (chase ? ld_relaxed_sw(p + k) : __ldg(p + k)) : 0u;
    }
    if (chase) {
        bool pend = false;
#pragma unroll
        for (int q = 0; q < RC_CHUNK / 32; q++) pend |= (c + 32 * q + lane < n) && nxt[q] == RC_PENDING;
        if (!__any_sync(0xffffffffu, pend)) return;
        unsigned long long t0 = rc_gtimer();
#pragma unroll
        for (int q = 0; q < RC_CHUNK / 32; q++) {
            const int64_t k = c + 32 * q + lane;
            while (k < n && nxt[q] == RC_PENDING && !timed_out) {
                __nanosleep(128);
                nxt[q] = ld_relaxed_sw(p + k);
                if (nxt[q] != RC_PENDING) t0 = rc_gtimer();
                else if (rc_gtimer() - t0 > RC_STALL_NS) timed_out = true;
            }
        }
        timed_out = __any_sync(0xffffffffu, timed_out);
    }
}

// The serial part of the parallel range coder for one stream, run by one
// warp: the range sequence range_{i+1} = norm((range_i >> 16) * width_i)
// (coder.py:37-57, widths only), recording range and byte position at every
// RC_CH-symbol chunk boundary.  sbuf: RC_CHUNK words of warp-private shared
// memory.  Returns false if a chased symbol never arrived.
__device__ __forceinline__ bool rc_plan_stream(const uint32_t* __restrict__ p, int64_t n, uint32_t* sbuf,
                                               unsigned long long* __restrict__ R_out, int64_t* __restrict__ P_out,
                                               bool chase) {
    const int lane = threadIdx.x & 31;
    uint32_t nxt[RC_CHUNK / 32];
    bool timed_out = false;
    rc_sym_load(p, n, 0, lane, nxt, chase, timed_out);
    uint64_t R = RC_TOP - 1;
    int64_t S = 0;
    for (int64_t c = 0; c < n; c += RC_CHUNK) {
        __syncwarp();
#pragma unroll
        for (int q = 0; q < RC_CHUNK / 32; q++) sbuf[32 * q + lane] = nxt[q];
        __syncwarp();
        rc_sym_load(p, n, c + RC_CHUNK, lane, nxt, chase && !timed_out, timed_out);
        if (lane == 0) {
            if ((c & (RC_CH - 1)) == 0) { R_out[c / RC_CH] = R; P_out[c / RC_CH] = S; }   // RC_CH % RC_CHUNK == 0
            const int m = (int)((n - c) < RC_CHUNK ? (n - c) : RC_CHUNK);
            uint32_t r = (uint32_t)(R >> 16);
            uint32_t x = sbuf[0];
            uint32_t sb = 0;                                   // shifts in this block
#pragma unroll 4
            for (int k = 0; k < m; k++) {
                const uint32_t y = sbuf[(k + 1) & (RC_CHUNK - 1)];
                // range' = r * width; renormalise by whole bytes (sh <= 2 as
                // r >= 2^24): next r = (range' << 8sh) >> 16.  The three
                // candidate shifts are formed in parallel and selected, so the
                // serial chain is multiply -> shift -> two selects.
                const uint32_t wq = (x & 0xFFFFu) + 1u;
                const uint32_t hi = __umulhi(r, wq), lo = r * wq;     // 32-bit halves: 32-bit compares
                const uint32_t r16 = __funnelshift_r(lo, hi, 16), r8 = __funnelshift_r(lo, hi, 8);
                sb += (hi < 0x100u) + (hi == 0u);
                r = hi >= 0x100u ? r16 : (hi != 0u ? r8 : lo);
                x = y;
            }
            S += sb;
            R = (uint64_t)r << 16;      // only r = R >> 16 matters to the next symbol
        }
    }
    if (lane == 0) P_out[(n + RC_CH - 1) / RC_CH] = S;
    return !timed_out;
}

// Stand-alone plan (after the tables, or over explicit streams): one warp
// per stream, RC_PLAN_WARPS streams per block.
constexpr int RC_PLAN_WARPS = 4;
__global__ void __launch_bounds__(32 * RC_PLAN_WARPS)
k_rc_plan(const uint32_t* __restrict__ sw, const int64_t* __restrict__ off, const int64_t* __restrict__ cnt,
          int64_t fixed_cnt, int max_chunks, unsigned long long* __restrict__ Rc, int64_t* __restrict__ posc,
          int n_streams) {
    __shared__ uint32_t sbuf_all[RC_PLAN_WARPS][RC_CHUNK];
    const int s = blockIdx.x * RC_PLAN_WARPS + (threadIdx.x >> 5);
    if (s >= n_streams) return;
    const int64_t base = off ? off[s] : (int64_t)s * fixed_cnt;
    const int64_t n = cnt ? cnt[s] : fixed_cnt;
    rc_plan_stream(sw + base, n, sbuf_all[threadIdx.x >> 5], Rc + (int64_t)s * max_chunks,
                   posc + (int64_t)s * (max_chunks + 1), false);
}

// The plan run INSIDE the table kernel (fused encoder): warp 0 of blocks
// [0, n_plan) follows streams blockIdx.x, blockIdx.x + n_plan, ... while the
// other warps of the same cooperative launch produce the symbols.  A
// cooperative launch guarantees every block is resident, so the chase cannot
// wait on a block that never runs (whatever else shares the GPU, and under
// tools that serialise kernels).
struct RcPlanArgs {
    int n_plan;                        // blocks whose warp 0 runs the plan (0 = none)
    int n_streams;
    int max_chunks;
    int64_t count;                     // symbols per stream
    unsigned long long* Rc;
    int64_t* posc;
    int32_t* status;
};

// ---------------------------------------------------------------------------
// encoder, stage 1 in FAST precision, pipelined (lpic_net_tc2.cuh): a
// persistent CTA per SM owns pairs of 128-pixel tiles; warps 0-7 gather the
// taps and run the epilogues of their tile, warp 8 issues the MMAs, warp 9
// streams the weight blocks.  Bit-identical raw to k_enc_net_tc.
// ---------------------------------------------------------------------------
template <int HH>
__global__ void __launch_bounds__(TC2_THREADS, 1)
k_enc_net_tc2(const __grid_constant__ TcNet2Dev w, const uint8_t* __restrict__ images, int H, int W, int mode,
              const int32_t* __restrict__ inv, int64_t N, int n_img, float* __restrict__ raw_out, int32_t* status,
              float* trace_raw) {
    extern __shared__ __align__(128) unsigned char smem[];
    Tc2Smem* s = reinterpret_cast<Tc2Smem*>(smem);
    constexpr int TC = Taps<HH>::TC;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int l = 0; l < w.nl; l++)
        for (int c = tid; c < TC_NMAX; c += blockDim.x) s->bias[l][c] = c < w.N[l] ? w.bias[l][c] : 0.0f;
    if (warp == TC2_MMA_WARP) umma::tmem_alloc(&s->tmem, 512);
    if (tid == 0) {
        for (int i = 0; i < TC2_SLOTS; i++) { tc2_mbar_init(&s->wfull[i], 1); tc2_mbar_init(&s->wfree[i], 1); }
        for (int t = 0; t < 2; t++) { tc2_mbar_init(&s->aready[t], 256); tc2_mbar_init(&s->dfull[t], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = s->tmem;
    const int64_t tiles_per = (N + TC_M - 1) / TC_M, total = tiles_per * n_img, pairs = (total + 1) / 2;
    const int64_t my_pairs = (int64_t)blockIdx.x < pairs ? (pairs - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (warp == TC2_LOAD_WARP) {                              // weight loader
        if (lane == 0) {
            const int64_t nblocks = my_pairs * w.nb;
            for (int64_t g = 0; g < nblocks; g++) {
                const int slot = (int)(g % TC2_SLOTS), b = (int)(g % w.nb);
                if (g >= TC2_SLOTS) tc_mbar_wait(&s->wfree[slot], (uint32_t)(((g / TC2_SLOTS) - 1) & 1));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(umma::smem_addr(&s->wfull[slot])), "r"((uint32_t)w.blk_bytes[b]) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(umma::smem_addr(s->w[slot])), "l"(w.blk[b]), "r"((uint32_t)w.blk_bytes[b]),
                             "r"(umma::smem_addr(&s->wfull[slot])) : "memory");
            }
        }
    } else if (warp == TC2_MMA_WARP) {                        // MMA issue (whole warp, elected lane)
        uint32_t acnt[2] = {0u, 0u}, wcnt[TC2_SLOTS] = {};
        int64_t g = 0;
        for (int64_t p = 0; p < my_pairs; p++) {
            for (int l = 0; l < w.nl; l++) {
                for (int t = 0; t < 2; t++) {
                    tc_mbar_wait(&s->aready[t], acnt[t] & 1u);
                    acnt[t]++;
                    umma::fence_after();
                    tc2_issue_layer(s, w, t, l, tbase, g, wcnt);
                }
                g += w.n_blk[l];
            }
        }
    } else {
        // epilogue / gather: warps 0-15 -> tile t = (warp >> 2) & 1, row r
        // (TMEM lane quadrant warp % 4), column half hf = warp >> 3: each
        // thread handles 64 of a layer's (<= 128) output columns
        const int t = (warp >> 2) & 1, hf = warp >> 3, r = 32 * (warp & 3) + lane;
        const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
        const uint32_t dcol = tbase + (uint32_t)(256 * t);
        unsigned char* a_hi = s->a_hi[t];
        unsigned char* a_lo = s->a_lo[t];
        uint32_t dcnt = 0;
        // the first layer's operand (all of K0) of row r of `tile`.  Tiles are
        // RASTER runs of 128 pixels (the network is per pixel; only the raw
        // plane is in coding order, row inv[pixel]): a warp's 32 lanes gather
        // 32 adjacent pixels, so every tap load is one 96-byte run instead of
        // 32 rows apart (a coding-order run steps one row down per pixel)
        auto gather = [&](int64_t tile, float (&x)[TC]) {
            const int64_t img = tile / tiles_per, n = (tile - img * tiles_per) * TC_M + r;
            if (tile < total && n < N) {
                const int i = (int)(n / W), j = (int)(n - (int64_t)i * W);
                gather_u8<HH>(images + img * N * 3, H, W, i, j, mode, NormU8(), x, LdgU8());
            } else {
#pragma unroll
                for (int q = 0; q < TC; q++) x[q] = 0.0f;
            }
        };
        for (int64_t p = blockIdx.x; p < pairs; p += gridDim.x) {
            const int64_t tile = 2 * p + t;
            const int64_t img = tile / tiles_per, n = (tile - img * tiles_per) * TC_M + r;
            const bool valid = tile < total && n < N;
            if (hf == 0 && p == (int64_t)blockIdx.x) {        // the CTA's first pair: gathered here
                float x[TC];
                gather(tile, x);
                tc2_store_input<TC>(a_hi, a_lo, r, x, w.K[0]);
                umma::fence_async_smem();
            }
            // (later pairs: the column-half-1 warps gathered this operand during
            // the previous pair's last layer, where they have no columns --
            // the taps' global-load latency overlaps that layer's MMAs)
            umma::fence_before();
            tc2_arrive(&s->aready[t]);
            const int64_t cn = valid ? (int64_t)__ldg(inv + n) : 0;     // coding index of the row
            float* row = valid ? raw_out + (img * N + cn) * w.M : nullptr;
            bool finite = true;
            const bool pre = hf == 1 && p + gridDim.x < pairs;  // this warp prepares the next pair's operand
            for (int l = 0; l < w.nl; l++) {
                const bool last = l == w.nl - 1;
                const int Nl = w.N[l], Knext = last ? 0 : w.K[l + 1];
                const float* bias = s->bias[l];
                float xn[TC];
                if (last && pre) gather(2 * (p + gridDim.x) + t, xn);   // loads in flight during the MMAs
                tc_mbar_wait(&s->dfull[t], dcnt & 1u);
                dcnt++;
                umma::fence_after();
                for (int c0 = 64 * hf; c0 < Nl && c0 < 64 * hf + 64; c0 += 16) {
                    float d0[16], d1[16];
                    umma::tmem_ld16x2(dcol + lane_off + (uint32_t)c0, dcol + lane_off + (uint32_t)(Nl + c0), d0, d1);
                    float y[16];
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const float v = __fadd_rn(__fadd_rn(d0[i], __fmul_rn(d1[i], 4.8828125e-4f)), bias[c0 + i]);
                        y[i] = last ? v : (v >= 0.0f ? v : __fmul_rn(0.01f, v));
                    }
                    if (last) {
                        if (row) {
#pragma unroll
                            for (int i = 0; i < 16; i++)
                                if (c0 + i < w.M) {
                                    row[c0 + i] = y[i];
                                    finite &= isfinite(y[i]);
                                    if (trace_raw) trace_raw[(img * N + cn) * w.M + c0 + i] = y[i];
                                }
                        }
                    } else if (c0 < Knext) {
                        tc2_store_split16(a_hi, a_lo, r, c0, Knext, y);
                    }
                }
                if (last && pre) {
                    // this tile's last MMAs have completed (dfull): its A operand is free
                    tc2_store_input<TC>(a_hi, a_lo, r, xn, w.K[0]);
                    umma::fence_async_smem();
                }
                umma::fence_before();
                if (!last) {
                    umma::fence_async_smem();
                    tc2_arrive(&s->aready[t]);
                }
            }
            if (!finite) atomicOr(status + img, LPIC_S_NONFINITE);
        }
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    if (warp == TC2_MMA_WARP) umma::tmem_dealloc(tbase, 512);
}

// ---------------------------------------------------------------------------
// encoder, stage 2: three quantised CDF tables per pixel (warp builder) and
// the coded symbol's (start, width) in coding order (codec.py:168-182)
// ---------------------------------------------------------------------------
// VAR: 0 float64 Gaussian, 1 float64 logistic, 2 FAST float32 Gaussian; BIG:
// 3K > 32 (one channel's mixture at a time).  One variant per kernel keeps
// the code within the instruction caches.
constexpr int TAB_WARPS = 8;
constexpr int TAB_BATCH = 4;
#ifndef LPIC_TAB_QC
#define LPIC_TAB_QC 2                  // Phi chains per warp step in the table kernel (r4h A/B: 2 > 4 = 8 at 3 blocks/SM)
#endif
#ifndef LPIC_TAB_MINB_F32
#define LPIC_TAB_MINB_F32 4            // the FAST float32 tables: 4 blocks/SM (64 registers; r4p A/B: FAST encode 80.8 -> 78.7 ms)
#endif
#ifndef LPIC_TAB_MINB
#define LPIC_TAB_MINB 3                // blocks per SM the register budget must allow (80 registers; 2: 128)
#endif
template <int VAR, bool BIG>
__global__ void __launch_bounds__(TAB_WARPS * 32, VAR == 2 ? LPIC_TAB_MINB_F32 : LPIC_TAB_MINB)
k_enc_tables(const float* __restrict__ raw, int M, int K, const uint8_t* __restrict__ images, int W,
             const int32_t* __restrict__ order, int64_t N, int64_t total, uint32_t* __restrict__ sw,
             int32_t* trace_cdf, unsigned long long* __restrict__ ctr, const RcPlanArgs plan) {
    constexpr bool f32 = VAR == 2;
    constexpr int dist = VAR == 1 ? 1 : 0;
    __shared__ __align__(16) CdfConsts cc;
    __shared__ WarpCdfScratch sc[TAB_WARPS];
    __shared__ float rbuf[TAB_WARPS][12 * KMAX];
    load_consts(&cc);
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wid == 0 && (int)blockIdx.x < plan.n_plan) {
        // range-coder plan warp: chase this block's streams (warp 0's
        // histogram scratch is its symbol buffer)
        bool ok = true;
        for (int s = blockIdx.x; s < plan.n_streams; s += plan.n_plan) {
            ok = rc_plan_stream(sw + (int64_t)s * plan.count, plan.count, sc[0].hist,
                                plan.Rc + (int64_t)s * plan.max_chunks, plan.posc + (int64_t)s * (plan.max_chunks + 1),
                                ok) && ok;
            if (!ok && lane == 0) atomicOr(plan.status + s, LPIC_S_INTERNAL);
        }
        return;
    }
    // work item t -> pixel nn = t / nimg of image t % nimg: every image's
    // symbols complete front to back at the same rate, which the chasing
    // range-coder plan (k_rc_plan, chase mode) follows
    // Work is handed out in TAB_BATCH-item grabs from a global counter, so
    // production is front to back whatever the block residency.
    const int64_t nimg = total / N;
    int64_t tw = 0, tw_end = 0;
    for (;;) {
        if (tw >= tw_end) {
            unsigned long long b0 = 0;
            if (lane == 0) b0 = atomicAdd(ctr, (unsigned long long)TAB_BATCH);
            b0 = __shfl_sync(0xffffffffu, b0, 0);
            if ((int64_t)b0 >= total) break;
            tw = (int64_t)b0;
            tw_end = tw + TAB_BATCH < total ? tw + TAB_BATCH : total;
        }
        const int64_t t = tw++;
        const int64_t nn = t / nimg, img = t - nn * nimg;
        const int64_t g = img * N + nn;
        for (int m = lane; m < M; m += 32) rbuf[wid][m] = __ldg(raw + g * M + m);
        const int32_t ij = __ldg(order + nn);
        const uint8_t* px = images + ((int64_t)img * N + (int64_t)(ij >> 16) * W + (ij & 0xFFFF)) * 3;
        const int s0 = __ldg(px), s1 = __ldg(px + 1), s2 = __ldg(px + 2);
        const float rn = cc.lut[s0], gn = cc.lut[s1];
        __syncwarp();
        // mixture parameters of all three channels at once: lane ch*K + i
        // holds component i of channel ch (kernels.py:212-247)
        double pi_l = 0.0, mu_l = 0.0, inv_l = 1.0;
        if constexpr (BIG) {                               // (K > 10: one channel at a time)
#pragma unroll 1
            for (int ch = 0; ch < 3; ch++) {
                uint32_t start[8], mass[8];
                if constexpr (f32) warp_table32(rbuf[wid], K, ch, ch >= 1 ? rn : 0.0f, ch == 2 ? gn : 0.0f, &cc, sc + wid, start, mass);
                else warp_table(rbuf[wid], K, dist, ch, ch >= 1 ? rn : 0.0f, ch == 2 ? gn : 0.0f, &cc, sc + wid, start, mass);
                const int sym = ch == 0 ? s0 : (ch == 1 ? s1 : s2);
                if (lane == (sym >> 3)) {
                    uint32_t st = 0, ms = 1;
#pragma unroll
                    for (int q = 0; q < 8; q++) if (q == (sym & 7)) { st = start[q]; ms = mass[q]; }
                    st_relaxed_sw(sw + g * 3 + ch, (st << 16) | (ms - 1));
                }
                if (trace_cdf) store_cdf_row(trace_cdf + (g * 3 + ch) * 257, start, mass);
            }
            __syncwarp();
            continue;
        } else {
        if (lane < 3 * K) {
            const int ch = lane / K, i = lane - ch * K;
            pi_l = mix_pi(rbuf[wid], K, ch, i);
            inv_l = mix_inv(rbuf[wid], K, ch, i);
            mu_l = (double)mix_mu(rbuf[wid], K, ch, i, ch >= 1 ? rn : 0.0f, ch == 2 ? gn : 0.0f);
        }
#pragma unroll 1
        for (int ch = 0; ch < 3; ch++) {
            uint32_t start[8], mass[8];
            if constexpr (f32) {                            // FAST float32 tables (Gaussian)
                float pmf[8];
                warp_pmf32(__double2float_rn(pi_l), (float)mu_l, __double2float_rn(inv_l), K, &cc, pmf, ch * K, sc + wid);
                warp_quantize32(pmf, sc + wid, start, mass);
            } else {
                double pmf[8];
                warp_pmf_t<dist, LPIC_TAB_QC>(pi_l, mu_l, inv_l, K, &cc, pmf, ch * K, sc + wid);
                warp_quantize(pmf, sc + wid, start, mass);
            }
            const int sym = ch == 0 ? s0 : (ch == 1 ? s1 : s2);
            if (lane == (sym >> 3)) {
                uint32_t st = 0, ms = 1;
#pragma unroll
                for (int q = 0; q < 8; q++) if (q == (sym & 7)) { st = start[q]; ms = mass[q]; }
                st_relaxed_sw(sw + g * 3 + ch, (st << 16) | (ms - 1));
            }
            if (trace_cdf) store_cdf_row(trace_cdf + (g * 3 + ch) * 257, start, mass);
        }
        __syncwarp();
        }
    }
}

template <int VAR, bool BIG>
cudaError_t launch_enc_tables_vb(int64_t blocks, int sms, const float* raw, int M, int K, const uint8_t* images,
                                 int W, const int32_t* order, int64_t N, int64_t total, uint32_t* sw, int32_t* tc,
                                 unsigned long long* ctr, RcPlanArgs plan, cudaStream_t st) {
    auto kern = k_enc_tables<VAR, BIG>;
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TAB_WARPS * 32, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    // persistent grid (work is grabbed from a global counter): every block resident
    int64_t g = (int64_t)occ * sms;
    if (plan.n_plan > 0) {
        if (plan.n_plan > g / 2) plan.n_plan = (int)(g / 2);
        if (plan.n_plan < 1) plan.n_plan = 0;
        g = g < blocks + plan.n_plan ? g : blocks + plan.n_plan;
    } else {
        g = g < blocks ? g : blocks;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(TAB_WARPS * 32);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = plan.n_plan > 0 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, raw, M, K, images, W, order, N, total, sw, tc, ctr, plan);
}
// Launch the table kernel; with plan.n_plan > 0 as ONE cooperative launch
// whose plan warps chase the symbols.  Returns the error of the launch (a
// cooperative launch can be refused, e.g. when the GPU is partitioned).
cudaError_t launch_enc_tables(int var, int64_t blocks, int sms, const float* raw, int M, int K, const uint8_t* images,
                              int W, const int32_t* order, int64_t N, int64_t total, uint32_t* sw, int32_t* tc,
                              unsigned long long* ctr, const RcPlanArgs& plan, cudaStream_t st) {
    const bool big = 3 * K > 32;
#define LPIC_TAB(v)                                                                                                  \
    return big ? launch_enc_tables_vb<v, true>(blocks, sms, raw, M, K, images, W, order, N, total, sw, tc, ctr, plan, \
                                               st)                                                                   \
               : launch_enc_tables_vb<v, false>(blocks, sms, raw, M, K, images, W, order, N, total, sw, tc, ctr,    \
                                                plan, st);
    if (var == 2) { LPIC_TAB(2) }
    if (var == 1) { LPIC_TAB(1) }
    LPIC_TAB(0)
#undef LPIC_TAB
}


// ---------------------------------------------------------------------------
// range coder (coder.py:30-73 + the encoder loop, codec.py:178-183), in
// parallel and byte-identical to the sequential coder.
//
// The coder's output is the big integer L = sum_i r_i*start_i * 256^(S-S_i)
// (r_i = range_i >> 16, S_i = byte shifts before symbol i, S = all shifts),
// rounded up to a multiple of 2^24 by finish() and written big-endian; the
// reference's carry propagation is exactly the carries of that sum.  Only
// the range sequence is inherently serial, and it depends on the widths
// alone:
//   1. k_rc_plan   one lane per stream runs range_{i+1} = norm((range_i >> 16)
//                  * w_i) -- three dependent integer ops per symbol -- and
//                  records range and byte position at every RC_CH-symbol chunk;
//   2. k_rc_chunks one thread per chunk codes its symbols from that range with
//                  low = 0, writing its bytes at their final position (carries
//                  ripple inside the chunk; a carry out of its first byte is
//                  counted), and keeps its pending 48-bit low window;
//   3. k_rc_merge  one lane per stream adds every chunk's window and carry-outs
//                  (rare ripples through 0xFF runs) and applies finish().
// ---------------------------------------------------------------------------
// carry of +1 into byte j, rippling back over 0xFF down to `floor`; returns 1
// if it ran past `floor` (a carry out of the region)
__device__ __forceinline__ int rc_carry_into(uint8_t* out, int64_t j, int64_t floor) {
    while (j >= floor && out[j] == 0xFF) { out[j] = 0; j--; }
    if (j < floor) return 1;
    out[j] += 1;
    return 0;
}

__global__ void __launch_bounds__(128)
k_rc_chunks(const uint32_t* __restrict__ sw, const int64_t* __restrict__ off, const int64_t* __restrict__ cnt,
            int64_t fixed_cnt, int n_streams, int max_chunks, const unsigned long long* __restrict__ Rc,
            const int64_t* __restrict__ posc, uint8_t* out, int64_t cap_each, unsigned long long* __restrict__ Wc,
            int32_t* __restrict__ cout, int32_t* status) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = (int)(gid / max_chunks), c = (int)(gid % max_chunks);
    if (s >= n_streams) return;
    const int64_t n = cnt ? cnt[s] : fixed_cnt;
    const int64_t i0 = (int64_t)c * RC_CH;
    if (i0 >= n) return;
    const int64_t i1 = (i0 + RC_CH < n) ? i0 + RC_CH : n;
    const uint32_t* p = sw + (off ? off[s] : (int64_t)s * fixed_cnt);
    uint8_t* o = out + (int64_t)s * cap_each;
    const int64_t* P = posc + (int64_t)s * (max_chunks + 1);
    const int64_t first = P[c];
    int64_t e = first;
    uint64_t low = 0, range = Rc[(int64_t)s * max_chunks + c];
    int carries = 0;
    for (int64_t i = i0; i < i1; i++) {
        const uint32_t x = __ldg(p + i);
        const uint64_t r = range >> 16;
        low += r * (x >> 16);
        range = r * ((x & 0xFFFFu) + 1u);
        if (low >= RC_TOP) { low -= RC_TOP; carries += rc_carry_into(o, e - 1, first); }
        while (range < RC_BOTTOM) {
            if (e < cap_each) o[e] = (uint8_t)(low >> 40);
            e++;
            low = (low << 8) & RC_MASK;
            range <<= 8;
        }
    }
    if (e + 6 > cap_each) atomicOr(status + s, ST_CAPACITY);
    Wc[(int64_t)s * max_chunks + c] = low;
    cout[(int64_t)s * max_chunks + c] = carries;
}

__global__ void __launch_bounds__(32)
k_rc_merge(const int64_t* __restrict__ off, const int64_t* __restrict__ cnt, int64_t fixed_cnt, int n_streams,
           int max_chunks, const int64_t* __restrict__ posc, const unsigned long long* __restrict__ Wc,
           const int32_t* __restrict__ cout, uint8_t* out, int64_t cap_each, int64_t* lens, int32_t* status) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_streams) return;
    const int64_t n = cnt ? cnt[s] : fixed_cnt;
    const int nch = (int)((n + RC_CH - 1) / RC_CH);
    const int64_t* P = posc + (int64_t)s * (max_chunks + 1);
    uint8_t* o = out + (int64_t)s * cap_each;
    const int64_t S = P[nch];
    if (S + 6 > cap_each) { atomicOr(status + s, ST_CAPACITY); lens[s] = S + 3; return; }
    // the final window region starts zeroed
    for (int q = 0; q < 6; q++) o[S + q] = 0;
    for (int c = 0; c < nch; c++) {
        const int32_t co = cout[(int64_t)s * max_chunks + c];
        for (int q = 0; q < co; q++) rc_carry_into(o, P[c] - 1, 0);
        // chunk c's pending window at bytes [P[c+1], P[c+1]+6), big-endian
        const uint64_t W = Wc[(int64_t)s * max_chunks + c];
        const int64_t at = P[c + 1];
        int carry = 0;
        for (int q = 5; q >= 0; q--) {
            const int v = (int)o[at + q] + (int)((W >> (8 * (5 - q))) & 0xFFu) + carry;
            o[at + q] = (uint8_t)v;
            carry = v >> 8;
        }
        if (carry) rc_carry_into(o, at - 1, 0);
    }
    // finish (coder.py:59-73): round the final window up to a multiple of 2^24
    if (o[S + 3] | o[S + 4] | o[S + 5]) {
        int carry = 1;
        for (int q = 2; q >= 0 && carry; q--) {
            const int v = (int)o[S + q] + 1;
            o[S + q] = (uint8_t)v;
            carry = v >> 8;
        }
        if (carry) rc_carry_into(o, S - 1, 0);
    }
    lens[s] = S + 3;
}


// ---------------------------------------------------------------------------
// unquantised probability of the realised bin (kernels.true_symbol_probs,
// kernels.py:316-346) -> theoretical_bpsp (codec.py:255-274).  Same mixture
// and CDF arithmetic as the tables, evaluated only at the coded bin's edges.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double true_prob(const float* raw, int K, int dist, int ch, float rn, float gn, int x,
                                            const CdfConsts* cc) {
    double p = 0.0;
    for (int i = 0; i < K; i++) {
        const double pi = mix_pi(raw, K, ch, i);
        const double inv = mix_inv(raw, K, ch, i);
        const double mu = (double)mix_mu(raw, K, ch, i, rn, gn);
        const double lo = (x == 0) ? 0.0 : cdf_value(__dmul_rn(__dsub_rn(cc->edges[x], mu), inv), dist, cc->phic);
        const double hi = (x == 255) ? 1.0 : cdf_value(__dmul_rn(__dsub_rn(cc->edges[x + 1], mu), inv), dist, cc->phic);
        const double d = __dsub_rn(hi, lo);
        if (d > 0.0) p = __dadd_rn(p, __dmul_rn(pi, d));
    }
    return p;
}

// explicit seam: raw (N,M), syms (N,3) int64, rn/gn (N) -> out (N,3) f64
__global__ void __launch_bounds__(128)
k_true_probs(const float* __restrict__ raw, int64_t N, int M, int K, int dist, const int64_t* __restrict__ syms,
             const float* __restrict__ rn, const float* __restrict__ gn, double* __restrict__ out) {
    __shared__ __align__(16) CdfConsts cc;
    load_consts(&cc);
    __syncthreads();
    for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x) {
        float r[12 * KMAX];
        for (int m = 0; m < M; m++) r[m] = raw[n * M + m];
        for (int ch = 0; ch < 3; ch++)
            out[n * 3 + ch] = true_prob(r, K, dist, ch, ch >= 1 ? rn[n] : 0.0f, ch == 2 ? gn[n] : 0.0f,
                                        (int)syms[n * 3 + ch], &cc);
    }
}

// codec path: raw plane in coding order (k_enc_net) + images -> -log2 p per sub-pixel
__global__ void __launch_bounds__(128)
k_true_bits(const float* __restrict__ raw, int M, int K, int dist, const uint8_t* __restrict__ images, int W,
            const int32_t* __restrict__ order, int64_t N, int64_t total, double* __restrict__ bits) {
    __shared__ __align__(16) CdfConsts cc;
    load_consts(&cc);
    __syncthreads();
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t img = g / N, nn = g - img * N;
        float r[12 * KMAX];
        for (int m = 0; m < M; m++) r[m] = raw[g * M + m];
        const int32_t ij = __ldg(order + nn);
        const uint8_t* px = images + ((int64_t)img * N + (int64_t)(ij >> 16) * W + (ij & 0xFFFF)) * 3;
        const int s0 = px[0], s1 = px[1], s2 = px[2];
        const float rn = cc.lut[s0], gn = cc.lut[s1];
        bits[g * 3 + 0] = -log2(true_prob(r, K, dist, 0, 0.0f, 0.0f, s0, &cc));
        bits[g * 3 + 1] = -log2(true_prob(r, K, dist, 1, rn, 0.0f, s1, &cc));
        bits[g * 3 + 2] = -log2(true_prob(r, K, dist, 2, rn, gn, s2, &cc));
    }
}

// ---------------------------------------------------------------------------
// parity seams
// ---------------------------------------------------------------------------
template <int CP, int HH>
__global__ void __launch_bounds__(NET_THREADS)
k_forward_taps(NetDev w, const float* __restrict__ taps, int64_t N, float* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem[];
    float* raw = reinterpret_cast<float*>(smem);
    float* zbuf = raw + NET_THREADS * w.MP;
    const int64_t n = (int64_t)blockIdx.x * NET_THREADS + threadIdx.x;
    if (n >= N) return;
    float x[Taps<HH>::TC];
#pragma unroll
    for (int k = 0; k < Taps<HH>::TC; k++) x[k] = taps[n * Taps<HH>::TC + k];
    float* r = raw + threadIdx.x * w.MP;
    net_forward<CP, Taps<HH>::TC>(w, x, r, zbuf + threadIdx.x, NET_THREADS);
    for (int m = 0; m < w.M; m++) out[n * w.M + m] = r[m];
}

template <int CP, int HH>
__global__ void __launch_bounds__(NET_THREADS)
k_forward_full(NetDev w, const float* __restrict__ plane, int H, int W, float* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem[];
    float* raw = reinterpret_cast<float*>(smem);
    float* zbuf = raw + NET_THREADS * w.MP;
    const int64_t n = (int64_t)blockIdx.x * NET_THREADS + threadIdx.x;
    if (n >= (int64_t)H * W) return;
    const int i = (int)(n / W), j = (int)(n % W);
    float x[Taps<HH>::TC];
#pragma unroll
    for (int k = 0; k < Taps<HH>::T; k++) {
        const int ii = i + Taps<HH>::di(k), jj = j + Taps<HH>::dj(k);
        const bool in = ii >= 0 && ii < H && jj >= 0 && jj < W;
        for (int c = 0; c < 3; c++) x[3 * k + c] = in ? plane[((int64_t)ii * W + jj) * 3 + c] : 0.0f;
    }
    float* r = raw + threadIdx.x * w.MP;
    net_forward<CP, Taps<HH>::TC>(w, x, r, zbuf + threadIdx.x, NET_THREADS);
    for (int m = 0; m < w.M; m++) out[n * w.M + m] = r[m];
}

__global__ void __launch_bounds__(128)
k_channel_cdfs(const float* __restrict__ raw, int64_t N, int M, int K, int dist, int ch,
               const float* __restrict__ rn, const float* __restrict__ gn, int32_t* __restrict__ out) {
    __shared__ __align__(16) CdfConsts cc;
    __shared__ WarpCdfScratch sc[4];
    load_consts(&cc);
    __syncthreads();
    const int wid = threadIdx.x >> 5;
    const int64_t n = (int64_t)blockIdx.x * 4 + wid;
    if (n >= N) return;
    uint32_t start[8], mass[8];
    warp_table(raw + n * M, K, dist, ch, rn[n], gn[n], &cc, sc + wid, start, mass);
    store_cdf_row(out + n * 257, start, mass);
}

// kernels._quantized_cdf (kernels.py:250-293) from explicit mixture
// parameters: pi/mu/s (N, K) float64 -> cdf (N, 257) int32; one warp per
// row, the same warp builder as the codec (z = (edge - mu) * (1/s)).
__global__ void __launch_bounds__(128)
k_quantized_cdf(const double* __restrict__ pi, const double* __restrict__ mu, const double* __restrict__ s, int64_t N,
                int K, int dist, int32_t* __restrict__ out, double* __restrict__ pmf_out, double* __restrict__ negrem_out) {
    __shared__ __align__(16) CdfConsts cc;
    __shared__ WarpCdfScratch sc[4];
    load_consts(&cc);
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n = (int64_t)blockIdx.x * 4 + wid;
    if (n >= N) return;
    double pi_l = 0.0, mu_l = 0.0, inv_l = 1.0;
    if (lane < K) {
        pi_l = pi[n * K + lane];
        mu_l = mu[n * K + lane];
        inv_l = __ddiv_rn(1.0, s[n * K + lane]);
    }
    double pmf[8];
    warp_pmf(pi_l, mu_l, inv_l, K, dist, &cc, pmf, 0, sc + wid);
    if (pmf_out || negrem_out) {                  // the reference kernel's scratch outputs (pmf, f - v)
        unsigned long long qs = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) qs += fx_bin(pmf[q]);
        const double scale = cdf_scale(fx_total(fx_warp_sum(qs)));
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const double v = __dmul_rn(pmf[q], scale);
            double f = floor(v);
            if (f > CDF_FLOOR) f = CDF_FLOOR;
            if (pmf_out) pmf_out[n * 256 + 8 * lane + q] = pmf[q];
            if (negrem_out) negrem_out[n * 256 + 8 * lane + q] = __dsub_rn(f, v);
        }
    }
    uint32_t start[8], mass[8];
    warp_quantize(pmf, sc + wid, start, mass);
    store_cdf_row(out + n * 257, start, mass);
}

__global__ void k_rc_decode_tables(const uint8_t* data, int64_t len, const int32_t* cdf, int64_t N,
                                   int32_t* syms, int32_t* status) {
    RcDecoder d;
    d.init(data, len);
    for (int64_t n = 0; n < N && !d.status; n++) {
        const int32_t* c = cdf + n * 257;
        uint64_t r;
        const uint32_t target = d.target(r);
        int lo = 0, hi = 256;
        while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if ((uint32_t)c[mid] <= target) lo = mid; else hi = mid; }
        d.advance(r, (uint32_t)c[lo], (uint32_t)(c[lo + 1] - c[lo]));
        syms[n] = lo;
    }
    *status = d.status;
}

// pack payloads of n streams (fixed stride) into one buffer at offs
__global__ void k_pack(const uint8_t* src, int64_t cap_each, const int64_t* offs, const int64_t* lens,
                       uint8_t* dst) {
    const int s = blockIdx.y;
    const int64_t L = lens[s];
    const uint8_t* a = src + (int64_t)s * cap_each;
    uint8_t* b = dst + offs[s];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < L; k += (int64_t)gridDim.x * blockDim.x)
        b[k] = a[k];
}

}  // namespace

// ===========================================================================
// host side: the model handle and the C-ABI
// ===========================================================================
struct lpic_model {
    int K, C, L, h, dist, M, T, TC, CP, MP, MT, NH;
    int device;
    int precision;
    uint64_t fingerprint;
    float* d_w;          // one allocation for all padded tensors
    NetDev net;
    // FAST precision: fp16 hi|lo weight blobs + padded biases (lpic_net_tc.cuh)
    unsigned char* d_tc = nullptr;
    TcNetDev tcnet{};
    bool tc_ok = false;
    unsigned char* d_tc2 = nullptr;        // K-blocked copy for k_enc_net_tc2
    TcNet2Dev tcnet2{};
    bool tc2_ok = false;
    // cached coding order per geometry
    int32_t* d_order = nullptr;
    int32_t* d_inv = nullptr;          // raster index -> coding index (the FAST network's raster tiles)
    int ord_H = -1, ord_W = -1, ord_mode = -1;
    // workspace
    uint32_t* d_sw = nullptr; size_t sw_cap = 0;
    // parallel range-coder workspace (k_rc_plan / k_rc_chunks / k_rc_merge)
    unsigned long long* d_rcR = nullptr; size_t rcR_cap = 0;
    unsigned long long* d_rcW = nullptr; size_t rcW_cap = 0;
    int64_t* d_rcP = nullptr; size_t rcP_cap = 0;
    int32_t* d_rcC = nullptr; size_t rcC_cap = 0;
    float* d_raw = nullptr; size_t raw_cap = 0;
    uint8_t* d_img = nullptr; size_t img_cap = 0;
    uint8_t* d_pay = nullptr; size_t pay_cap = 0;
    uint8_t* d_pack = nullptr; size_t pack_cap = 0;
    int64_t* d_meta = nullptr; size_t meta_cap = 0;   // lens | offs
    int32_t* d_status = nullptr; size_t status_cap = 0;
    // decoder geometry tables (step offsets, producer chunks) per (H, W, mode)
    int64_t* d_step_off = nullptr;
    int32_t* d_chunks = nullptr;
    int n_chunks = 0, ring_size = 0;
    int dg_H = -1, dg_W = -1, dg_mode = -1;
    // decoder ring workspace
    uint8_t* d_ring = nullptr; size_t ring_cap = 0;
    uint32_t* d_flags = nullptr; size_t flags_cap = 0;
    uint32_t* d_progress = nullptr; size_t progress_cap = 0;
    unsigned long long* d_dbg = nullptr;   // optional decoder timeline (lpic_decode_debug)
    unsigned long long* d_ctr = nullptr;   // k_enc_tables work counter
    int launches = 0;
    std::mutex mu;
};

namespace {

template <typename T>
int ensure(T*& p, size_t& cap, size_t need) {
    if (need <= cap && p) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t n = need < 64 ? 64 : need;
    if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return fail(LPIC_E_NOMEM, "cudaMalloc workspace failed");
    cap = n;
    return 0;
}

struct RcWork {
    unsigned long long *R, *W;
    int64_t* P;
    int32_t* C;
};
// the three-phase parallel range coder over n streams (fixed count or
// per-stream off/cnt); max_count bounds every stream's symbol count
int rc_max_chunks(int64_t max_count) {
    return (int)((max_count + RC_CH - 1) / RC_CH) > 0 ? (int)((max_count + RC_CH - 1) / RC_CH) : 1;
}
int rc_plan(const RcWork& wk, const uint32_t* d_sw, const int64_t* d_off, const int64_t* d_cnt, int64_t fixed_cnt,
            int n, int64_t max_count, cudaStream_t st) {
    k_rc_plan<<<(n + RC_PLAN_WARPS - 1) / RC_PLAN_WARPS, 32 * RC_PLAN_WARPS, 0, st>>>(
        d_sw, d_off, d_cnt, fixed_cnt, rc_max_chunks(max_count), wk.R, wk.P, n);
    CUDA_TRY(cudaGetLastError());
    return 0;
}
// phases 2-3 (after the plan)
int rc_encode_finish(const RcWork& wk, const uint32_t* d_sw, const int64_t* d_off, const int64_t* d_cnt,
                     int64_t fixed_cnt, int n, int64_t max_count, uint8_t* d_out, int64_t cap_each,
                     int64_t* d_lens, int32_t* d_status, cudaStream_t st) {
    const int max_chunks = rc_max_chunks(max_count);
    const int64_t threads = (int64_t)n * max_chunks;
    k_rc_chunks<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(d_sw, d_off, d_cnt, fixed_cnt, n, max_chunks, wk.R,
                                                                   wk.P, d_out, cap_each, wk.W, wk.C, d_status);
    CUDA_TRY(cudaGetLastError());
    k_rc_merge<<<(unsigned)((n + 31) / 32), 32, 0, st>>>(d_off, d_cnt, fixed_cnt, n, max_chunks, wk.P, wk.W, wk.C,
                                                           d_out, cap_each, d_lens, d_status);
    CUDA_TRY(cudaGetLastError());
    return 0;
}
int rc_encode_parallel(const RcWork& wk, const uint32_t* d_sw, const int64_t* d_off, const int64_t* d_cnt,
                       int64_t fixed_cnt, int n, int64_t max_count, uint8_t* d_out, int64_t cap_each,
                       int64_t* d_lens, int32_t* d_status, cudaStream_t st) {
    if (int r = rc_plan(wk, d_sw, d_off, d_cnt, fixed_cnt, n, max_count, st)) return r;
    return rc_encode_finish(wk, d_sw, d_off, d_cnt, fixed_cnt, n, max_count, d_out, cap_each, d_lens, d_status, st);
}

template <typename Kern>
int set_smem(Kern k, size_t bytes) {
    CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return 0;
}


int coding_order(lpic_model* m, int H, int W, int mode, cudaStream_t st) {
    if (m->d_order && m->ord_H == H && m->ord_W == W && m->ord_mode == mode) return 0;
    const int64_t N = (int64_t)H * W;
    std::vector<int32_t> ord((size_t)N);
    const int a = sched_a(mode, W, m->h);
    const int64_t steps = sched_steps(mode, H, W, m->h);
    int64_t n = 0;
    for (int64_t t = 0; t < steps; t++) {
        int lo, hi;
        sched_rows(t, a, H, W, lo, hi);
        for (int i = lo; i <= hi; i++) ord[(size_t)n++] = (i << 16) | (int)(t - (int64_t)a * i);
    }
    std::vector<int32_t> inv((size_t)N);
    for (int64_t k = 0; k < N; k++) inv[(size_t)((int64_t)(ord[(size_t)k] >> 16) * W + (ord[(size_t)k] & 0xFFFF))] = (int32_t)k;
    if (m->d_order) cudaFree(m->d_order);
    if (m->d_inv) cudaFree(m->d_inv);
    m->d_order = nullptr;
    m->d_inv = nullptr;
    CUDA_TRY(cudaMalloc(&m->d_order, sizeof(int32_t) * N));
    CUDA_TRY(cudaMalloc(&m->d_inv, sizeof(int32_t) * N));
    CUDA_TRY(cudaMemcpyAsync(m->d_order, ord.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(m->d_inv, inv.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    m->ord_H = H; m->ord_W = W; m->ord_mode = mode;
    return 0;
}

// template dispatch on (CP, HH)
template <template <int, int> class F, typename... A>
int dispatch(int CP, int HH, A&&... args) {
#define LPIC_CASE(cp, hh) if (CP == cp && HH == hh) return F<cp, hh>::run(args...);
    LPIC_CASE(16, 1) LPIC_CASE(32, 1) LPIC_CASE(64, 1) LPIC_CASE(128, 1)
    LPIC_CASE(16, 2) LPIC_CASE(32, 2) LPIC_CASE(64, 2) LPIC_CASE(128, 2)
    LPIC_CASE(16, 3) LPIC_CASE(32, 3) LPIC_CASE(64, 3) LPIC_CASE(128, 3)
#undef LPIC_CASE
    return fail(LPIC_E_UNSUPPORTED, "unsupported (C, kernel_half) instantiation");
}

template <int HH>
int launch_enc_net_tc(lpic_model* m, const uint8_t* d_images, int n, int H, int W, int mode, float* raw,
                      int32_t* d_status, float* tr, cudaStream_t st) {
    static const bool v1 = std::getenv("LPIC_TC_V1") != nullptr;      // (A/B: the serial tile kernel)
    if (m->tc2_ok && !v1) {
        const size_t smem2 = sizeof(Tc2Smem);
        if (set_smem(k_enc_net_tc2<HH>, smem2)) return LPIC_E_CUDA;
        const int64_t N2 = (int64_t)H * W, tiles2 = ((N2 + TC_M - 1) / TC_M) * n, pairs = (tiles2 + 1) / 2;
        int sms2 = 148;
        cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, m->device);
        const unsigned grid2 = (unsigned)(pairs < sms2 ? pairs : sms2);
        k_enc_net_tc2<HH><<<grid2, TC2_THREADS, smem2, st>>>(m->tcnet2, d_images, H, W, mode, m->d_inv, N2, n, raw,
                                                             d_status, tr);
        CUDA_TRY(cudaGetLastError());
        return 0;
    }
    const size_t smem = sizeof(TcSmem);
    if (set_smem(k_enc_net_tc<HH>, smem)) return LPIC_E_CUDA;
    const int64_t N = (int64_t)H * W, tiles = ((N + TC_M - 1) / TC_M) * n;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
    const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
    k_enc_net_tc<HH><<<grid, 128, smem, st>>>(m->tcnet, d_images, H, W, mode, m->d_order, N, n, raw, d_status, tr);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

// Encoder pipeline: network -> tables (+ the range-coder plan fused into the
// same cooperative launch for <= RC_FUSED_MAX streams) -> chunks -> merge.
// The plan's serial width chain then hides under the table work instead of
// following it.  With more streams, or if the cooperative launch is refused,
// the plan runs after the tables (k_rc_plan; it is then short next to them).
constexpr int RC_FUSED_MAX = 64;
struct RcPlanWork {
    RcWork wk;
    int64_t count;               // symbols per stream (3N)
};

template <int CP, int HH> struct EncodeRun {
    // *fused_out: 1 if the plan ran inside the table launch
    static int run(lpic_model* m, const uint8_t* d_images, int n, int H, int W, int mode, float* raw, uint32_t* sw,
                   int32_t* d_status, float* tr, int32_t* tc, const RcPlanWork& pw, int* fused_out, cudaStream_t st) {
        constexpr int TC = Taps<HH>::TC;
        const int64_t N = (int64_t)H * W;
        if (!m->d_ctr && cudaMalloc(&m->d_ctr, sizeof(unsigned long long)) != cudaSuccess)
            return fail(LPIC_E_NOMEM, "cudaMalloc work counter failed");
        if (m->precision == LPIC_PREC_FAST) {
            if (int r = launch_enc_net_tc<HH>(m, d_images, n, H, W, mode, raw, d_status, tr, st)) return r;
        } else {
            const size_t smem = net_tile_floats(CP, TC, m->MT, m->MP) * 4;
            if (set_smem(k_enc_net<CP, HH>, smem)) return LPIC_E_CUDA;
            dim3 grid((unsigned)((N + NT_TP - 1) / NT_TP), (unsigned)n);
            k_enc_net<CP, HH><<<grid, NT_THREADS, smem, st>>>(m->net, d_images, H, W, mode, m->d_inv, N, raw, d_status, tr);
            CUDA_TRY(cudaGetLastError());
        }
        const int64_t total = N * n;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device);
        const int64_t blocks = (total + TAB_WARPS - 1) / TAB_WARPS;
        const int var = (m->precision == LPIC_PREC_FAST && m->dist == 0) ? 2 : m->dist;
        CUDA_TRY(cudaMemsetAsync(m->d_ctr, 0, sizeof(unsigned long long), st));
        RcPlanArgs plan{};
        static const bool fuse_env = std::getenv("LPIC_RC_UNFUSED") == nullptr;   // (A/B timing only)
        if (fuse_env && n <= RC_FUSED_MAX) {
            CUDA_TRY(cudaMemsetAsync(sw, 0xFF, sizeof(uint32_t) * (size_t)N * n * 3, st));   // RC_PENDING
            plan.n_plan = n;
            plan.n_streams = n;
            plan.max_chunks = rc_max_chunks(pw.count);
            plan.count = pw.count;
            plan.Rc = pw.wk.R;
            plan.posc = pw.wk.P;
            plan.status = d_status;
            cudaError_t e = launch_enc_tables(var, blocks, sms, raw, m->M, m->K, d_images, W, m->d_order, N, total, sw,
                                              tc, m->d_ctr, plan, st);
            if (e == cudaSuccess) { *fused_out = 1; return 0; }
            (void)cudaGetLastError();           // refused (e.g. partitioned GPU): unfused below
            plan = RcPlanArgs{};
        }
        *fused_out = 0;
        cudaError_t e = launch_enc_tables(var, blocks, sms, raw, m->M, m->K, d_images, W, m->d_order, N, total, sw, tc,
                                          m->d_ctr, plan, st);
        if (e != cudaSuccess) return fail(LPIC_E_CUDA, std::string("k_enc_tables: ") + cudaGetErrorString(e));
        return 0;
    }
};

template <int CP, int HH> struct NetRun {
    static int run(lpic_model* m, const uint8_t* d_images, int n, int H, int W, int mode, float* raw, int32_t* d_status,
                   cudaStream_t st) {
        constexpr int TC = Taps<HH>::TC;
        const size_t smem = net_tile_floats(CP, TC, m->MT, m->MP) * 4;
        if (set_smem(k_enc_net<CP, HH>, smem)) return LPIC_E_CUDA;
        const int64_t N = (int64_t)H * W;
        dim3 grid((unsigned)((N + NT_TP - 1) / NT_TP), (unsigned)n);
        k_enc_net<CP, HH><<<grid, NT_THREADS, smem, st>>>(m->net, d_images, H, W, mode, m->d_inv, N, raw, d_status,
                                                          nullptr);
        CUDA_TRY(cudaGetLastError());
        return 0;
    }
};

int decode_geometry(lpic_model* m, int H, int W, int mode, cudaStream_t st) {
    if (m->d_step_off && m->dg_H == H && m->dg_W == W && m->dg_mode == mode) return 0;
    const int a = sched_a(mode, W, m->h);
    const int64_t steps = sched_steps(mode, H, W, m->h);
    std::vector<int64_t> off((size_t)steps + 1);
    std::vector<int32_t> chunks;
    int64_t n = 0;
    int maxc = 1;
    for (int64_t t = 0; t < steps; t++) {
        int lo, hi;
        sched_rows(t, a, H, W, lo, hi);
        off[(size_t)t] = n;
        const int cnt = hi - lo + 1;
        if (cnt <= 0) continue;
        maxc = cnt > maxc ? cnt : maxc;
        for (int c0 = 0; c0 < cnt; c0 += NT_TP) {
            chunks.push_back((int32_t)(n + c0));
            chunks.push_back(cnt - c0 < NT_TP ? cnt - c0 : NT_TP);
        }
        n += cnt;
    }
    off[(size_t)steps] = n;
    int ring = 64;
    while (ring < 2 * maxc + 64) ring <<= 1;
    cudaFree(m->d_step_off); cudaFree(m->d_chunks);
    m->d_step_off = nullptr; m->d_chunks = nullptr;
    CUDA_TRY(cudaMalloc(&m->d_step_off, sizeof(int64_t) * off.size()));
    CUDA_TRY(cudaMalloc(&m->d_chunks, sizeof(int32_t) * chunks.size()));
    CUDA_TRY(cudaMemcpyAsync(m->d_step_off, off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(m->d_chunks, chunks.data(), sizeof(int32_t) * chunks.size(), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    m->n_chunks = (int)(chunks.size() / 2);
    m->ring_size = ring;
    m->dg_H = H; m->dg_W = W; m->dg_mode = mode;
    return 0;
}

size_t dec_smem_bytes(int CP, int TC, int MT, int MP, int rec_bytes, int S, bool fast) {
    const size_t prod = fast ? dec_fbase_off() +
                                   sizeof(TcSmem)
                             : dec_fbase_off() + net_tile_floats(CP, TC, MT, MP) * 4;
    const size_t grp = ((sizeof(ConsumerSmem) + 127) & ~(size_t)127) + (size_t)DEC_SLOTS * rec_bytes;
    const size_t cons = ((sizeof(CdfConsts) + 127) & ~(size_t)127) + (size_t)S * grp;
    return prod > cons ? prod : cons;
}

// streams per cluster: one (latency) until the streams outnumber the
// co-resident clusters, then two (throughput: a stream holds a 2-SM cluster
// at ~20-30% utilisation).  LPIC_DEC_STREAMS_PER_CLUSTER overrides.
int dec_streams_per_cluster(int n, int device) {
    if (const char* e = getenv("LPIC_DEC_STREAMS_PER_CLUSTER")) {
        const int v = atoi(e);
        if (v >= 1 && v <= DEC_MAXS) return v;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return n > sms / 2 ? 2 : 1;
}

template <int CP, int HH> struct DecodeRun {
    static int run(lpic_model* m, const uint8_t* d_payload, const int64_t* d_offs, const int64_t* d_lens, int n,
                   int H, int W, int mode, uint8_t* d_images, int32_t* d_status, float* tr, int32_t* tc,
                   cudaStream_t st) {
        if (int r = coding_order(m, H, W, mode, st)) return r;
        if (int r = decode_geometry(m, H, W, mode, st)) return r;
        const int rec = rec_bytes_for(m->K);
        if (int r = ensure(m->d_ring, m->ring_cap, (size_t)n * m->ring_size * rec)) return r;
        if (int r = ensure(m->d_flags, m->flags_cap, (size_t)n * m->ring_size)) return r;
        if (int r = ensure(m->d_progress, m->progress_cap, (size_t)n)) return r;
        CUDA_TRY(cudaMemsetAsync(m->d_flags, 0, sizeof(uint32_t) * n * m->ring_size, st));
        CUDA_TRY(cudaMemsetAsync(m->d_progress, 0, sizeof(uint32_t) * n, st));
        const int S = dec_streams_per_cluster(n, m->device);
        const bool fast = m->precision == LPIC_PREC_FAST;
        const size_t smem = dec_smem_bytes(CP, m->TC, m->MT, m->MP, rec, S, fast);
        DecParams P;
        P.w = m->net; P.K = m->K; P.dist = m->dist; P.H = H; P.W = W; P.mode = mode; P.a = sched_a(mode, W, m->h);
        P.N = (int64_t)H * W; P.payload = d_payload; P.offs = d_offs; P.lens = d_lens; P.images = d_images;
        P.status = d_status; P.order = m->d_order; P.step_off = m->d_step_off; P.chunks = m->d_chunks;
        P.n_chunks = m->n_chunks; P.ring = m->d_ring; P.flags = m->d_flags; P.progress = m->d_progress;
        P.ring_size = m->ring_size; P.rec_bytes = rec; P.trace_raw = tr; P.trace_cdf = tc;
        P.dbg = m->d_dbg;
        P.S = S; P.n = n;
        P.fast = fast ? 1 : 0; P.tc = m->tcnet;
        P.f32 = (fast && m->dist == 0) ? 1 : 0;
        // the k_decode2 instantiations live in lpic_decode_cp*.cu (compiled in parallel)
        cudaError_t e = launch_decode2(CP, HH, S, n, smem, st, P);
        if (e != cudaSuccess) return fail(LPIC_E_CUDA, std::string("k_decode2: ") + cudaGetErrorString(e));
        return 0;
    }
};

template <int CP, int HH> struct TapsRun {
    static int run(lpic_model* m, const float* taps, int64_t N, float* out, cudaStream_t st) {
        const size_t smem = net_smem_bytes<CP>(m->MP);
        if (set_smem(k_forward_taps<CP, HH>, smem)) return LPIC_E_CUDA;
        k_forward_taps<CP, HH><<<(unsigned)((N + NET_THREADS - 1) / NET_THREADS), NET_THREADS, smem, st>>>(
            m->net, taps, N, out);
        CUDA_TRY(cudaGetLastError());
        return 0;
    }
};

template <int CP, int HH> struct FullRun {
    static int run(lpic_model* m, const float* plane, int H, int W, float* out, cudaStream_t st) {
        const size_t smem = net_smem_bytes<CP>(m->MP);
        if (set_smem(k_forward_full<CP, HH>, smem)) return LPIC_E_CUDA;
        const int64_t N = (int64_t)H * W;
        k_forward_full<CP, HH><<<(unsigned)((N + NET_THREADS - 1) / NET_THREADS), NET_THREADS, smem, st>>>(
            m->net, plane, H, W, out);
        CUDA_TRY(cudaGetLastError());
        return 0;
    }
};

// Every entry point that takes a model runs on the model's device and
// restores the caller's current device (multi-device use from one thread).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != d && cudaSetDevice(d) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

int check_geom(const lpic_model* m, int n, int H, int W, int mode) {
    if (!m) return fail(LPIC_E_ARG, "null model");
    if (n < 0 || H < 1 || W < 1 || H > 32767 || W > 65535) return fail(LPIC_E_ARG, "bad image geometry");
    if (mode < 0 || mode > 2) return fail(LPIC_E_ARG, "bad schedule mode");
    if (mode == 2 && m->h != 2) return fail(LPIC_E_ARG, "diagonal schedule is only defined for kernel_half=2");
    return 0;
}

}  // namespace

extern "C" {

int lpic_version(void) { return 1; }
const char* lpic_last_error(void) { return g_last_error.c_str(); }

uint64_t lpic_fnv1a64(const uint8_t* data, int64_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int64_t i = 0; i < n; i++) { h ^= data[i]; h *= 0x100000001b3ull; }
    return h;
}

int lpic_model_create(const float* masked_w, const float* masked_b, const float* hidden_w, const float* hidden_b,
                      const float* out_w, const float* out_b, int K, int C, int L, int h, int dist,
                      lpic_model_t** out) {
    if (!out || !masked_w || !masked_b || !out_w || !out_b || (L > 2 && (!hidden_w || !hidden_b)))
        return fail(LPIC_E_ARG, "null argument");
    if (K < 1 || K > KMAX) return fail(LPIC_E_UNSUPPORTED, "mixtures must be in [1, 16] on the GPU");
    if (C < 1 || C > 128) return fail(LPIC_E_UNSUPPORTED, "filters must be in [1, 128] on the GPU");
    if (L < 3) return fail(LPIC_E_ARG, "need at least 3 layers");
    if (h < 1 || h > 3) return fail(LPIC_E_UNSUPPORTED, "kernel_half must be 1, 2 or 3 on the GPU");
    if (dist != 0 && dist != 1) return fail(LPIC_E_ARG, "unknown distribution");
    lpic_model* m = new lpic_model();
    m->K = K; m->C = C; m->L = L; m->h = h; m->dist = dist;
    m->M = 12 * K; m->T = (2 * h + 1) * h + h; m->TC = 3 * m->T;
    m->CP = C <= 16 ? 16 : C <= 32 ? 32 : C <= 64 ? 64 : 128;
    m->MP = (m->M + 3) & ~3;
    m->MT = (m->M + 15) & ~15;
    m->NH = L - 2;
    m->precision = LPIC_PREC_COMPAT;
    cudaGetDevice(&m->device);
    const int CP = m->CP, MP = m->MP, MT = m->MT, NH = m->NH, T = m->T, TC = m->TC, M = m->M;
    // padded host layouts
    std::vector<float> mwT((size_t)CP * TC, 0.f), mb(CP, 0.f), hw((size_t)NH * CP * CP, 0.f), hb((size_t)NH * CP, 0.f),
        ow((size_t)MP * CP, 0.f), ob(MT, 0.f), mwI((size_t)TC * CP, 0.f), hwI((size_t)NH * CP * CP, 0.f),
        owI((size_t)CP * MT, 0.f);
    for (int t = 0; t < T; t++)
        for (int c = 0; c < 3; c++)
            for (int f = 0; f < C; f++) {
                mwT[(size_t)f * TC + t * 3 + c] = masked_w[(t * 3 + c) * C + f];
                mwI[(size_t)(t * 3 + c) * CP + f] = masked_w[(t * 3 + c) * C + f];
            }
    for (int f = 0; f < C; f++) mb[f] = masked_b[f];
    for (int l = 0; l < NH; l++)
        for (int o = 0; o < C; o++) {
            for (int i = 0; i < C; i++) {
                hw[((size_t)l * CP + o) * CP + i] = hidden_w[((size_t)l * C + o) * C + i];
                hwI[((size_t)l * CP + i) * CP + o] = hidden_w[((size_t)l * C + o) * C + i];
            }
            hb[(size_t)l * CP + o] = hidden_b[(size_t)l * C + o];
        }
    for (int mm = 0; mm < M; mm++) {
        for (int i = 0; i < C; i++) {
            ow[(size_t)mm * CP + i] = out_w[(size_t)mm * C + i];
            owI[(size_t)i * MT + mm] = out_w[(size_t)mm * C + i];
        }
        ob[mm] = out_b[mm];
    }
    const size_t total = mwT.size() + mb.size() + hw.size() + hb.size() + ow.size() + ob.size() + mwI.size() +
                         hwI.size() + owI.size() + 64;
    if (cudaMalloc(&m->d_w, total * sizeof(float)) != cudaSuccess) { delete m; return fail(LPIC_E_NOMEM, "cudaMalloc weights"); }
    float* p = m->d_w;
    auto put = [&](const std::vector<float>& v) -> const float* {
        cudaMemcpy(p, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice);
        const float* r = p;
        p += (v.size() + 3) & ~(size_t)3;                 // keep every tensor 16-byte aligned
        return r;
    };
    m->net.mwT = put(mwT); m->net.mb = put(mb); m->net.hw = put(hw); m->net.hb = put(hb);
    m->net.ow = put(ow); m->net.ob = put(ob); m->net.mwI = put(mwI); m->net.hwI = put(hwI); m->net.owI = put(owI);
    m->net.C = C; m->net.CP = CP; m->net.M = M; m->net.MP = MP; m->net.NH = NH; m->net.T = T; m->net.TC = TC;
    m->net.MT = MT;
    m->net.one = 1.0f;
    // fingerprint of the LPWT serialisation (network.py:255-281)
    std::vector<uint8_t> ser;
    const char magic[4] = {'L', 'P', 'W', 'T'};
    ser.insert(ser.end(), magic, magic + 4);
    const uint8_t hdr[6] = {1, (uint8_t)K, (uint8_t)C, (uint8_t)L, (uint8_t)h, (uint8_t)dist};
    ser.insert(ser.end(), hdr, hdr + 6);
    auto app = [&](const float* src, size_t count) {
        const uint8_t* b = reinterpret_cast<const uint8_t*>(src);
        ser.insert(ser.end(), b, b + count * 4);
    };
    app(masked_w, (size_t)T * 3 * C); app(masked_b, C);
    app(hidden_w, (size_t)NH * C * C); app(hidden_b, (size_t)NH * C);
    app(out_w, (size_t)M * C); app(out_b, M);
    m->fingerprint = lpic_fnv1a64(ser.data(), (int64_t)ser.size());
    // FAST precision operands: per layer W_hi | W_lo (fp16, canonical K-major
    // layout of lpic_umma.cuh) and biases padded to TC_NMAX
    {
        const int K0p = (TC + 15) & ~15;
        const int nl = NH + 2;
        if (CP <= TC_NMAX && MT <= TC_NMAX && K0p <= TC_KMAX && nl <= TC_MAXL) {
            std::vector<int> Ns(nl), Ks(nl);
            for (int l = 0; l < nl; l++) {
                Ns[l] = (l == nl - 1) ? MT : CP;
                Ks[l] = (l == 0) ? K0p : CP;
            }
            size_t total_b = 0;
            std::vector<size_t> boff(nl), bias_off(nl);
            for (int l = 0; l < nl; l++) { boff[l] = total_b; total_b += (size_t)2 * Ns[l] * Ks[l] * 2; }
            for (int l = 0; l < nl; l++) { bias_off[l] = total_b; total_b += TC_NMAX * sizeof(float); }
            std::vector<unsigned char> hb(total_b, 0);
            auto put_w = [&](int l, int n, int k, float v) {
                const __half hi = __float2half_rn(v);
                const __half lo = __float2half_rn((v - __half2float(hi)) * 2048.0f);
                const size_t o = umma::op_offset(n, k, Ks[l]);
                memcpy(&hb[boff[l] + o], &hi, 2);
                memcpy(&hb[boff[l] + (size_t)Ns[l] * Ks[l] * 2 + o], &lo, 2);
            };
            for (int t = 0; t < T; t++)
                for (int c = 0; c < 3; c++)
                    for (int f = 0; f < C; f++) put_w(0, f, t * 3 + c, masked_w[(t * 3 + c) * C + f]);
            for (int l = 0; l < NH; l++)
                for (int o = 0; o < C; o++)
                    for (int i = 0; i < C; i++) put_w(1 + l, o, i, hidden_w[((size_t)l * C + o) * C + i]);
            for (int mm = 0; mm < M; mm++)
                for (int i = 0; i < C; i++) put_w(nl - 1, mm, i, out_w[(size_t)mm * C + i]);
            auto put_b = [&](int l, const float* b, int count) { memcpy(&hb[bias_off[l]], b, count * sizeof(float)); };
            put_b(0, masked_b, C);
            for (int l = 0; l < NH; l++) put_b(1 + l, hidden_b + (size_t)l * C, C);
            put_b(nl - 1, out_b, M);
            if (cudaMalloc(&m->d_tc, total_b) == cudaSuccess &&
                cudaMemcpy(m->d_tc, hb.data(), total_b, cudaMemcpyHostToDevice) == cudaSuccess) {
                m->tcnet.nl = nl; m->tcnet.M = M; m->tcnet.K0 = TC;
                for (int l = 0; l < nl; l++) {
                    m->tcnet.blob[l] = m->d_tc + boff[l];
                    m->tcnet.bias[l] = reinterpret_cast<const float*>(m->d_tc + bias_off[l]);
                    m->tcnet.N[l] = Ns[l]; m->tcnet.K[l] = Ks[l];
                }
                m->tc_ok = true;
            }
            // the same weights as TC2_KB-column K blocks for the pipelined encoder
            // network (k_enc_net_tc2): per block W_hi (N x Kb) | W_lo (N x Kb)
            std::vector<int> bl, bk0, bkb;
            for (int l = 0; l < nl; l++)
                for (int k0 = 0; k0 < Ks[l]; k0 += TC2_KB) {
                    bl.push_back(l); bk0.push_back(k0); bkb.push_back(Ks[l] - k0 < TC2_KB ? Ks[l] - k0 : TC2_KB);
                }
            if ((int)bl.size() <= TC2_MAXB && nl <= TC2_MAXL && m->tc_ok) {
                std::vector<size_t> boff2(bl.size());
                size_t tot2 = 0;
                for (size_t b = 0; b < bl.size(); b++) { boff2[b] = tot2; tot2 += (size_t)2 * Ns[bl[b]] * bkb[b] * 2; }
                std::vector<unsigned char> hb2(tot2, 0);
                for (size_t b = 0; b < bl.size(); b++) {
                    const int l = bl[b], Nl = Ns[l], Kb = bkb[b], k0 = bk0[b];
                    for (int n = 0; n < Nl; n++)
                        for (int k = 0; k < Kb; k++) {
                            // copy from the full-K canonical blob of layer l
                            const size_t src = umma::op_offset(n, k0 + k, Ks[l]), dst = umma::op_offset(n, k, Kb);
                            memcpy(&hb2[boff2[b] + dst], &hb[boff[l] + src], 2);
                            memcpy(&hb2[boff2[b] + (size_t)Nl * Kb * 2 + dst], &hb[boff[l] + (size_t)Nl * Ks[l] * 2 + src], 2);
                        }
                }
                if (cudaMalloc(&m->d_tc2, tot2) == cudaSuccess &&
                    cudaMemcpy(m->d_tc2, hb2.data(), tot2, cudaMemcpyHostToDevice) == cudaSuccess) {
                    TcNet2Dev& t2 = m->tcnet2;
                    t2.nb = (int)bl.size(); t2.nl = nl; t2.M = M; t2.K0 = TC;
                    for (int l = 0; l < nl; l++) {
                        t2.N[l] = Ns[l]; t2.K[l] = Ks[l]; t2.bias[l] = m->tcnet.bias[l];
                        t2.first_blk[l] = -1; t2.n_blk[l] = 0;
                    }
                    for (size_t b = 0; b < bl.size(); b++) {
                        const int l = bl[b];
                        t2.blk[b] = m->d_tc2 + boff2[b];
                        t2.blk_bytes[b] = (int)(2 * Ns[l] * bkb[b] * 2);
                        t2.blk_kb[b] = bkb[b]; t2.blk_k0[b] = bk0[b]; t2.blk_layer[b] = l;
                        if (t2.first_blk[l] < 0) t2.first_blk[l] = (int)b;
                        t2.n_blk[l]++;
                    }
                    m->tc2_ok = true;
                }
            }
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { cudaFree(m->d_w); delete m; return fail(LPIC_E_CUDA, cudaGetErrorString(e)); }
    *out = m;
    return 0;
}

int lpic_model_destroy(lpic_model_t* m) {
    if (!m) return 0;
    DeviceGuard dg_(m->device);
    cudaFree(m->d_w);
    cudaFree(m->d_order); cudaFree(m->d_inv); cudaFree(m->d_sw); cudaFree(m->d_raw); cudaFree(m->d_img); cudaFree(m->d_pay);
    cudaFree(m->d_pack); cudaFree(m->d_meta); cudaFree(m->d_status);
    cudaFree(m->d_step_off); cudaFree(m->d_chunks); cudaFree(m->d_ring); cudaFree(m->d_flags);
    cudaFree(m->d_progress);
    cudaFree(m->d_rcR); cudaFree(m->d_rcW); cudaFree(m->d_rcP); cudaFree(m->d_rcC);
    cudaFree(m->d_tc);
    cudaFree(m->d_tc2);
    cudaFree(m->d_ctr);
    delete m;
    return 0;
}

int lpic_model_set_precision(lpic_model_t* m, int precision) {
    if (!m) return fail(LPIC_E_ARG, "null model");
    if (precision != LPIC_PREC_COMPAT && precision != LPIC_PREC_FAST) return fail(LPIC_E_ARG, "unknown precision");
    if (precision == LPIC_PREC_FAST && !m->tc_ok)
        return fail(LPIC_E_UNSUPPORTED, "FAST precision needs filters <= 128, 12*mixtures <= 128, kernel_half <= 3");
    m->precision = precision;
    return 0;
}

uint64_t lpic_model_fingerprint(const lpic_model_t* m) { return m ? m->fingerprint : 0; }
int lpic_last_launch_count(const lpic_model_t* m) { return m ? m->launches : 0; }

/* Diagnostics (not part of include/lpic_b200.h): record a globaltimer
 * timeline of stream 0 of the next decode into d_buf (4 stamps per producer
 * chunk followed by 12 per pixel; the per-pixel stamps only in builds with
 * -DLPIC_DEC_TIMELINE, scripts/ab_build.py); pass NULL to disable.  Returns
 * the number of producer chunks of the last decode geometry. */
int lpic_decode_debug(lpic_model_t* m, unsigned long long* d_buf) {
    if (!m) return -1;
    m->d_dbg = d_buf;
    return m->n_chunks;
}

int lpic_forward_taps(lpic_model_t* m, const float* d_taps, int64_t N, float* d_raw, void* stream) {
    if (!m || N < 0) return fail(LPIC_E_ARG, "bad argument");
    DeviceGuard dg_(m->device);
    if (N == 0) return 0;
    return dispatch<TapsRun>(m->CP, m->h, m, d_taps, N, d_raw, (cudaStream_t)stream);
}

int lpic_forward_full(lpic_model_t* m, const float* d_plane, int H, int W, float* d_raw, void* stream) {
    if (!m || H < 1 || W < 1) return fail(LPIC_E_ARG, "bad argument");
    DeviceGuard dg_(m->device);
    return dispatch<FullRun>(m->CP, m->h, m, d_plane, H, W, d_raw, (cudaStream_t)stream);
}

int lpic_channel_cdfs(const float* d_raw, int64_t N, int M, int K, int dist, int channel, const float* d_rn,
                      const float* d_gn, int32_t* d_cdf, void* stream) {
    if (N < 0 || K < 1 || K > KMAX || M < 12 * K || channel < 0 || channel > 2) return fail(LPIC_E_ARG, "bad argument");
    if (N == 0) return 0;
    k_channel_cdfs<<<(unsigned)((N + 3) / 4), 128, 0, (cudaStream_t)stream>>>(d_raw, N, M, K, dist, channel, d_rn, d_gn,
                                                                             d_cdf);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int lpic_rc_encode_streams(const uint32_t* d_sw, const int64_t* d_off, const int64_t* d_cnt, int n_streams,
                           uint8_t* d_out, int64_t cap_each, int64_t* d_len, int32_t* d_status, void* stream) {
    if (n_streams < 0 || !d_off || !d_cnt) return fail(LPIC_E_ARG, "bad argument");
    if (n_streams == 0) return 0;
    // parity entry: size the workspace from the largest stream (one host sync)
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<int64_t> hc((size_t)n_streams);
    CUDA_TRY(cudaMemcpyAsync(hc.data(), d_cnt, sizeof(int64_t) * n_streams, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    int64_t mx = 1;
    for (int64_t c : hc) mx = c > mx ? c : mx;
    const int64_t mc = (mx + RC_CH - 1) / RC_CH;
    // grow-only workspace shared by all calls (this entry point has no model handle)
    static std::mutex ws_mu;
    static RcWork ws_dev[64] = {};
    static size_t ws_cap_dev[64] = {};     // chunk slots, per device
    std::lock_guard<std::mutex> lk(ws_mu);
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(LPIC_E_UNSUPPORTED, "device index");
    RcWork& ws = ws_dev[dev];
    size_t& ws_cap = ws_cap_dev[dev];
    const size_t need = (size_t)n_streams * (mc + 1);
    if (need > ws_cap) {
        cudaFree(ws.R); cudaFree(ws.W); cudaFree(ws.P); cudaFree(ws.C);
        ws = RcWork{};
        ws_cap = 0;
        CUDA_TRY(cudaMalloc(&ws.R, sizeof(unsigned long long) * need));
        CUDA_TRY(cudaMalloc(&ws.W, sizeof(unsigned long long) * need));
        CUDA_TRY(cudaMalloc(&ws.P, sizeof(int64_t) * need));
        CUDA_TRY(cudaMalloc(&ws.C, sizeof(int32_t) * need));
        ws_cap = need;
    }
    const int r = rc_encode_parallel(ws, d_sw, d_off, d_cnt, 0, n_streams, mx, d_out, cap_each, d_len, d_status, st);
    CUDA_TRY(cudaStreamSynchronize(st));      // (the workspace is reused by the next call)
    return r;
}

int lpic_quantized_cdf(const double* d_pi, const double* d_mu, const double* d_s, int64_t N, int K, int dist,
                       int32_t* d_cdf, double* d_pmf, double* d_neg_rem, void* stream) {
    if (N < 0 || K < 1 || K > 32 || (dist != 0 && dist != 1)) return fail(LPIC_E_ARG, "bad argument");
    if (N == 0) return 0;
    k_quantized_cdf<<<(unsigned)((N + 3) / 4), 128, 0, (cudaStream_t)stream>>>(d_pi, d_mu, d_s, N, K, dist, d_cdf,
                                                                             d_pmf, d_neg_rem);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int lpic_rc_decode_tables(const uint8_t* d_data, int64_t len, const int32_t* d_cdf, int64_t N, int32_t* d_syms,
                          int32_t* d_status, void* stream) {
    if (N < 0 || len < 0) return fail(LPIC_E_ARG, "bad argument");
    k_rc_decode_tables<<<1, 1, 0, (cudaStream_t)stream>>>(d_data, len, d_cdf, N, d_syms, d_status);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int lpic_true_symbol_probs(const float* d_raw, int64_t N, int M, int K, int dist, const int64_t* d_syms,
                           const float* d_rn, const float* d_gn, double* d_out, void* stream) {
    if (N < 0 || K < 1 || K > KMAX || M < 12 * K || M > 12 * KMAX || (dist != 0 && dist != 1))
        return fail(LPIC_E_ARG, "bad argument");
    if (N == 0) return 0;
    const int64_t blocks = (N + 127) / 128;
    k_true_probs<<<(unsigned)(blocks < 4096 ? blocks : 4096), 128, 0, (cudaStream_t)stream>>>(d_raw, N, M, K, dist,
                                                                                            d_syms, d_rn, d_gn, d_out);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int lpic_network_coding_order(lpic_model_t* m, const uint8_t* d_images, int n, int H, int W, int mode, float* d_raw,
                              void* stream) {
    if (int r = check_geom(m, n, H, W, mode)) return r;
    DeviceGuard dg_(m->device);
    if (n == 0) return 0;
    std::lock_guard<std::mutex> lk(m->mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (int r = coding_order(m, H, W, mode, st)) return r;
    if (int r = ensure(m->d_status, m->status_cap, (size_t)n)) return r;
    CUDA_TRY(cudaMemsetAsync(m->d_status, 0, sizeof(int32_t) * n, st));
    if (m->precision == LPIC_PREC_FAST) {
        int r = LPIC_E_UNSUPPORTED;
        if (m->h == 1) r = launch_enc_net_tc<1>(m, d_images, n, H, W, mode, d_raw, m->d_status, nullptr, st);
        else if (m->h == 2) r = launch_enc_net_tc<2>(m, d_images, n, H, W, mode, d_raw, m->d_status, nullptr, st);
        else if (m->h == 3) r = launch_enc_net_tc<3>(m, d_images, n, H, W, mode, d_raw, m->d_status, nullptr, st);
        if (r) return r;
    } else if (int r = dispatch<NetRun>(m->CP, m->h, m, d_images, n, H, W, mode, d_raw, m->d_status, st)) {
        return r;
    }
    m->launches = 1;
    return 0;
}

int lpic_theoretical_bits(lpic_model_t* m, const uint8_t* d_images, int n, int H, int W, int mode, double* d_bits,
                          void* stream) {
    if (int r = check_geom(m, n, H, W, mode)) return r;
    DeviceGuard dg_(m->device);
    if (n == 0) return 0;
    std::lock_guard<std::mutex> lk(m->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = (int64_t)H * W;
    if (int r = coding_order(m, H, W, mode, st)) return r;
    if (int r = ensure(m->d_raw, m->raw_cap, (size_t)n * N * m->M)) return r;
    if (int r = ensure(m->d_status, m->status_cap, (size_t)n)) return r;
    CUDA_TRY(cudaMemsetAsync(m->d_status, 0, sizeof(int32_t) * n, st));
    if (int r = dispatch<NetRun>(m->CP, m->h, m, d_images, n, H, W, mode, m->d_raw, m->d_status, st)) return r;
    const int64_t total = N * n, blocks = (total + 127) / 128;
    k_true_bits<<<(unsigned)(blocks < 8192 ? blocks : 8192), 128, 0, st>>>(m->d_raw, m->M, m->K, m->dist, d_images, W,
                                                                          m->d_order, N, total, d_bits);
    CUDA_TRY(cudaGetLastError());
    m->launches = 2;
    return 0;
}

int lpic_encode_batch_device(lpic_model_t* m, const uint8_t* d_images, int n, int H, int W, int mode,
                             uint8_t* d_payload, int64_t cap_each, int64_t* d_lens, int32_t* d_status,
                             float* d_trace_raw, int32_t* d_trace_cdf, void* stream) {
    if (int r = check_geom(m, n, H, W, mode)) return r;
    DeviceGuard dg_(m->device);
    if (n == 0) return 0;
    std::lock_guard<std::mutex> lk(m->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = (int64_t)H * W;
    if (int r = coding_order(m, H, W, mode, st)) return r;
    // The raw plane and the symbols are per-batch workspace: batches larger
    // than the budget (LPIC_ENC_WORKSPACE_MB, default 4096) are encoded in
    // image chunks, so any batch fits (BASELINE C3: 256 x 2048x1536 on one
    // GPU would otherwise need ~116 GB of raw plane).
    static const int64_t budget = [] {
        const char* e = std::getenv("LPIC_ENC_WORKSPACE_MB");
        const long long v = e ? atoll(e) : 4096;
        return (int64_t)(v > 0 ? v : 4096) << 20;
    }();
    const int64_t per_img = N * ((int64_t)m->M * 4 + 3 * 4);
    int chunk = n;
    if ((int64_t)n * per_img > budget) chunk = (int)(budget / per_img > 1 ? budget / per_img : 1);
    if (d_trace_raw || d_trace_cdf) chunk = n;                 // (traces index the whole batch)
    if (int r = ensure(m->d_sw, m->sw_cap, (size_t)chunk * N * 3)) return r;
    if (int r = ensure(m->d_raw, m->raw_cap, (size_t)chunk * N * m->M)) return r;
    CUDA_TRY(cudaMemsetAsync(d_status, 0, sizeof(int32_t) * n, st));
    const int64_t mc = (3 * N + RC_CH - 1) / RC_CH;
    if (int r = ensure(m->d_rcR, m->rcR_cap, (size_t)chunk * mc)) return r;
    if (int r = ensure(m->d_rcW, m->rcW_cap, (size_t)chunk * mc)) return r;
    if (int r = ensure(m->d_rcP, m->rcP_cap, (size_t)chunk * (mc + 1))) return r;
    if (int r = ensure(m->d_rcC, m->rcC_cap, (size_t)chunk * mc)) return r;
    const RcPlanWork pw{RcWork{m->d_rcR, m->d_rcW, m->d_rcP, m->d_rcC}, 3 * N};
    int launches = 0;
    for (int b0 = 0; b0 < n; b0 += chunk) {
        const int nb = n - b0 < chunk ? n - b0 : chunk;
        int fused = 0;
        if (int r = dispatch<EncodeRun>(m->CP, m->h, m, d_images + (size_t)b0 * N * 3, nb, H, W, mode, m->d_raw,
                                        m->d_sw, d_status + b0, d_trace_raw, d_trace_cdf, pw, &fused, st))
            return r;
        if (!fused && (rc_plan(pw.wk, m->d_sw, nullptr, nullptr, 3 * N, nb, 3 * N, st))) return LPIC_E_CUDA;
        if (int r = rc_encode_finish(pw.wk, m->d_sw, nullptr, nullptr, 3 * N, nb, 3 * N,
                                     d_payload + (size_t)b0 * cap_each, cap_each, d_lens + b0, d_status + b0, st))
            return r;
        launches += fused ? 4 : 5;
    }
    m->launches = launches;
    return 0;
}

int lpic_decode_batch_device(lpic_model_t* m, const uint8_t* d_payload, const int64_t* d_offs, const int64_t* d_lens,
                             int n, int H, int W, int mode, uint8_t* d_images, int32_t* d_status, float* d_trace_raw,
                             int32_t* d_trace_cdf, void* stream) {
    if (int r = check_geom(m, n, H, W, mode)) return r;
    DeviceGuard dg_(m->device);
    if (n == 0) return 0;
    std::lock_guard<std::mutex> lk(m->mu);
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(d_status, 0, sizeof(int32_t) * n, st));
    CUDA_TRY(cudaMemsetAsync(d_images, 0, (size_t)n * H * W * 3, st));
    if (int r = dispatch<DecodeRun>(m->CP, m->h, m, d_payload, d_offs, d_lens, n, H, W, mode, d_images, d_status,
                                    d_trace_raw, d_trace_cdf, st))
        return r;
    m->launches = 1;
    return 0;
}

int lpic_encode_batch(lpic_model_t* m, const uint8_t* h_images, int n, int H, int W, int mode, uint8_t* h_payload,
                      int64_t payload_cap, int64_t* h_offs, int64_t* h_lens, int32_t* h_status, void* stream) {
    if (int r = check_geom(m, n, H, W, mode)) return r;
    DeviceGuard dg_(m->device);
    if (n == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = (int64_t)H * W;
    const int64_t cap_each = 6 * N + 64;
    {
        std::lock_guard<std::mutex> lk(m->mu);
        if (int r = ensure(m->d_img, m->img_cap, (size_t)n * N * 3)) return r;
        if (int r = ensure(m->d_pay, m->pay_cap, (size_t)n * cap_each)) return r;
        if (int r = ensure(m->d_meta, m->meta_cap, (size_t)2 * n)) return r;
        if (int r = ensure(m->d_status, m->status_cap, (size_t)n)) return r;
        CUDA_TRY(cudaMemcpyAsync(m->d_img, h_images, (size_t)n * N * 3, cudaMemcpyHostToDevice, st));
    }
    if (int r = lpic_encode_batch_device(m, m->d_img, n, H, W, mode, m->d_pay, cap_each, m->d_meta, m->d_status,
                                         nullptr, nullptr, stream))
        return r;
    std::lock_guard<std::mutex> lk(m->mu);
    CUDA_TRY(cudaMemcpyAsync(h_lens, m->d_meta, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_status, m->d_status, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    int64_t total = 0;
    for (int b = 0; b < n; b++) { h_offs[b] = total; total += h_lens[b] > cap_each ? cap_each : h_lens[b]; }
    if (total > payload_cap) return fail(LPIC_E_ARG, "h_payload capacity too small (lens filled)");
    if (int r = ensure(m->d_pack, m->pack_cap, (size_t)total)) return r;
    CUDA_TRY(cudaMemcpyAsync(m->d_meta + n, h_offs, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    k_pack<<<dim3(64, n), 256, 0, st>>>(m->d_pay, cap_each, m->d_meta + n, m->d_meta, m->d_pack);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(h_payload, m->d_pack, (size_t)total, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    m->launches = 6;
    return 0;
}

int lpic_decode_batch(lpic_model_t* m, const uint8_t* h_payload, const int64_t* h_offs, const int64_t* h_lens, int n,
                      int H, int W, int mode, uint8_t* h_images, int32_t* h_status, void* stream) {
    if (int r = check_geom(m, n, H, W, mode)) return r;
    DeviceGuard dg_(m->device);
    if (n == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = (int64_t)H * W;
    int64_t total = 0;
    for (int b = 0; b < n; b++) total = h_offs[b] + h_lens[b] > total ? h_offs[b] + h_lens[b] : total;
    {
        std::lock_guard<std::mutex> lk(m->mu);
        if (int r = ensure(m->d_img, m->img_cap, (size_t)n * N * 3)) return r;
        if (int r = ensure(m->d_pack, m->pack_cap, (size_t)total + 8)) return r;
        if (int r = ensure(m->d_meta, m->meta_cap, (size_t)2 * n)) return r;
        if (int r = ensure(m->d_status, m->status_cap, (size_t)n)) return r;
        CUDA_TRY(cudaMemcpyAsync(m->d_pack, h_payload, (size_t)total, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(m->d_meta, h_offs, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(m->d_meta + n, h_lens, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
    }
    if (int r = lpic_decode_batch_device(m, m->d_pack, m->d_meta, m->d_meta + n, n, H, W, mode, m->d_img, m->d_status,
                                         nullptr, nullptr, stream))
        return r;
    std::lock_guard<std::mutex> lk(m->mu);
    CUDA_TRY(cudaMemcpyAsync(h_images, m->d_img, (size_t)n * N * 3, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_status, m->d_status, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return 0;
}

}  // extern "C"
