// lpic_decode.cuh -- the wavefront decoder: one 2-CTA cluster per stream.
//
// Replaces codec.decode (/root/reference/pkg/src/lpic/codec.py:193-247) and
// RangeDecoder (coder.py:76-112).  The per-stream work splits into
//
//   producer (cluster rank 1, 8 warps): for every pixel, in coding order, as
//     soon as its causal taps are decoded: gather -> network (compat float32)
//     -> red CDF table (warp builder) + the g/b mixture record (softmax
//     weights, 1/s, base means, tanh coefficients).  Records go to a
//     per-stream ring in global memory (L2-resident) with a ready flag each.
//   consumer (cluster rank 0, 4 chain warps + loader + publisher warps): the
//     serial chain.  The loader bulk-copies record n (cp.async.bulk +
//     mbarrier) into a 4-slot shared-memory ring; the chain decodes r from
//     the red table, builds the green table (chain builder, lpic_chain.cuh),
//     decodes g, builds blue, decodes b; the publisher writes the pixel and
//     publishes the stream's progress.
//
// Pixel (i,j) of step t is computable once pixel (i, j-1) -- the latest of
// its taps in coding order, in step t-1 -- is decoded (all earlier steps
// for j = 0), so the producer trails the chain by about one wavefront step
// and its work is off the critical path.  The cluster guarantees both CTAs
// are co-resident, so the cross-CTA spin-waits cannot deadlock.
#pragma once
// In-situ chain phase profile (A/B builds only: -DLPIC_DEC_PROF): the chain
// builder's CHP timestamps (lpic_chain.cuh) accumulate into s_chp and stream
// 0's consumer appends them to the decoder timeline buffer.
#ifdef LPIC_DEC_PROF
__shared__ long long s_chp[16];
#define LPIC_CHAIN_PROF s_chp
#endif
#include "lpic_cdf.cuh"
#include "lpic_chain.cuh"
#include "lpic_net.cuh"
#include "lpic_net_tc.cuh"
#include "lpic_rc.cuh"
#include "lpic_sched.cuh"

namespace lpic {

constexpr int DEC_MAXS = 2;             // streams per cluster (throughput mode)
constexpr int DEC_THREADS = 384;        // (S = 2) consumer: S x (4 chain warps) + S loaders + S publishers;
                                        // producer: net_tile on 256, the rest only join its barriers
constexpr int DEC_SLOTS = 8;
constexpr int DEC_PUBQ = 32;            // decoded pixels queued for the publisher warp
#ifndef LPIC_AUX_SLEEP
#define LPIC_AUX_SLEEP 256               // loader / publisher poll interval (ns): they share schedulers with chain warps
#endif

struct DecParams {
    NetDev w;
    TcNetDev tc;                 // FAST precision network (lpic_net_tc.cuh)
    int fast;
    int f32;                     // FAST float32 tables (fast && Gaussian)
    int S;                       // streams per cluster (chains per consumer CTA)
    int n;                       // streams in the launch
    int K, dist, H, W, mode, a;
    int64_t N;
    const uint8_t* payload;
    const int64_t* offs;
    const int64_t* lens;
    uint8_t* images;
    int32_t* status;
    const int32_t* order;        // coding index -> (i<<16)|j
    const int64_t* step_off;     // steps+1 coding offsets
    const int32_t* chunks;       // (n0, npx) pairs, each inside one step
    int n_chunks;
    uint8_t* ring;               // [n][ring][rec_bytes]
    uint32_t* flags;             // [n][ring]
    uint32_t* progress;          // [n]
    int ring_size;               // power of two
    int rec_bytes;
    float* trace_raw;
    int32_t* trace_cdf;
    unsigned long long* dbg;     // optional timeline (globaltimer ns), see lpic_decode_debug
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// record layout
__host__ __device__ __forceinline__ int rec_mix_off() { return 512; }
__host__ __device__ __forceinline__ int rec_bytes_for(int K) { return (512 + 32 * K + 20 * K + 4 + 15) & ~15; }
struct RecView {
    const uint16_t* red;   // cdf[0..255]
    const double* pi_g; const double* inv_g; const double* pi_b; const double* inv_b;
    const float* mu_g; const float* mu_b; const float* ta; const float* tb; const float* tc;
    int32_t ij;            // pixel (i<<16)|j
    __device__ RecView(const unsigned char* r, int K) {
        red = reinterpret_cast<const uint16_t*>(r);
        const double* d = reinterpret_cast<const double*>(r + 512);
        pi_g = d; inv_g = d + K; pi_b = d + 2 * K; inv_b = d + 3 * K;
        const float* f = reinterpret_cast<const float*>(d + 4 * K);
        mu_g = f; mu_b = f + K; ta = f + 2 * K; tb = f + 3 * K; tc = f + 4 * K;
        ij = *reinterpret_cast<const int32_t*>(f + 5 * K);
    }
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Polling load: relaxed, L1-bypassing.  (ld.acquire.gpu compiles to
// LDG.STRONG + CCTL.IVALL, i.e. it invalidates the whole L1 of the SM on
// every poll; readers here only use L2 loads or TMA after the poll.)
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// one acquire after a relaxed poll succeeded (instead of an acquiring poll)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_volatile_smem(const volatile uint32_t* p) { return *p; }
__device__ __forceinline__ unsigned long long ld_volatile_smem64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ uint32_t ld_acquire_cta_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    return done != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// ---------------------------------------------------------------------------
// producer
// ---------------------------------------------------------------------------
__host__ __device__ constexpr size_t dec_fbase_off() {
    return (sizeof(CdfConsts) + 127) & ~(size_t)127;
}
template <int CP, int HH>
__device__ void dec_producer(const DecParams& P, int img, unsigned char* smem) {
    CdfConsts* cc = reinterpret_cast<CdfConsts*>(smem);

    float* fbase = reinterpret_cast<float*>(smem + dec_fbase_off());
    constexpr int TC = Taps<HH>::TC;
    NetTileBufs nb;
    net_tile_carve(fbase, CP, TC, P.w.MT, P.w.MP, nb);
    __shared__ long long s_need;
    // FAST precision: the tensor-core tile state and a raw buffer replace the fp32 tile buffers
    const size_t tc_off = dec_fbase_off();
    TcSmem* tcs = reinterpret_cast<TcSmem*>(smem + tc_off);
    // (the raw outputs reuse the A-operand buffer: the last layer's epilogue
    // writes them after its MMAs completed, and the next tile's input is
    // stored only after this chunk's records and tables have read them;
    // 64 x MP floats <= 32 KB since FAST needs 12K <= 128)
    float* fraw = reinterpret_cast<float*>(tcs->a_hi);
    uint32_t mcnt = 0;
    load_consts(cc);
    if (P.fast && threadIdx.x < 128) tc_init(tcs);
    if (!P.fast && threadIdx.x == 0) net_tile_init(nb);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    if (P.fast && threadIdx.x < 128) tc_prefetch(tcs, P.tc);
    float* rawbuf = P.fast ? fraw : nb.raw;
    // the red tables' selection histograms (8 warps x 1 KB) live in a buffer
    // that is idle between the network and the next chunk's gather
    WarpCdfScratch* sc = P.fast ? reinterpret_cast<WarpCdfScratch*>(tcs->a_lo) : reinterpret_cast<WarpCdfScratch*>(nb.act0);
    // red-table warps: all of the CTA's warps when the scratch region holds
    // one histogram per warp (act0 + act1 span >= 64 KB... i.e. CP >= 32; FAST: a_lo, 32 KB)
    const int tab_warps = (int)(blockDim.x >> 5) > 8 &&
                                  (P.fast || (size_t)((CP > Taps<HH>::TC ? CP : Taps<HH>::TC) + CP) * NT_TP * 4 >=
                                                 (blockDim.x >> 5) * sizeof(WarpCdfScratch))
                              ? (int)(blockDim.x >> 5) : 8;
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    const int K = P.K;
    const int64_t N = P.N;
    const int img0 = img;
    // chunk-major over the cluster's S streams (same geometry, so the
    // chains progress at similar rates and neither starves the other)
    for (int cs_ = 0; cs_ < P.n_chunks * P.S; cs_++) {
        const int c = cs_ / P.S;
        img = img0 + cs_ % P.S;
        if (img >= P.n) continue;
        if (!P.fast) net_tile_prefetch(P.w, nb);          // layer 0 lands during the wait + gather
        const uint8_t* im = P.images + (int64_t)img * N * 3;
        uint8_t* ring = P.ring + (int64_t)img * P.ring_size * P.rec_bytes;
        uint32_t* flags = P.flags + (int64_t)img * P.ring_size;
        const uint32_t* progress = P.progress + img;
        const int n0 = P.chunks[2 * c], npx = P.chunks[2 * c + 1];
        const int64_t n = n0 + tid;
        const bool act = tid < npx && tid < NT_TP;
        int i = 0, j = 0;
        if (tid == 0) s_need = (int64_t)n0 + npx - P.ring_size;      // ring back-pressure
        __syncthreads();
        if (act) {
            // latest tap in coding order: (i, j-1) in step t-1, else all of step t-1
            const int32_t ij = __ldg(P.order + n);
            i = ij >> 16; j = ij & 0xFFFF;
            const int64_t t = (int64_t)P.a * i + j;
            int64_t req;
            if (j >= 1) {
                int lo, hi;
                sched_rows(t - 1, P.a, P.H, P.W, lo, hi);
                req = __ldg(P.step_off + t - 1) + (i - lo) + 1;
            } else {
                req = __ldg(P.step_off + t);
            }
            atomicMax(&s_need, (long long)req);
        }
        __syncthreads();
        unsigned long long* dbg = (P.dbg && img == 0) ? P.dbg + 4 * (int64_t)c : nullptr;
        if (tid == 0) {
            if (dbg) dbg[0] = gtimer();
            const int64_t need = s_need;
            uint32_t ns = 32;
            while ((int64_t)ld_relaxed_u32(progress) < need) { __nanosleep(ns); ns = ns < 256 ? ns * 2 : 256; }
            // acquire: the publisher's st.release of `progress` now happens-before
            // this thread's later operations, and the barrier below extends that
            // to every thread's gather of the decoded pixels
            fence_acq_rel_gpu();
            if (dbg) dbg[1] = gtimer();
        }
        __syncthreads();
        if (P.fast) {
            if (tid < TC_M) {                                  // warps 0-3: the tensor-core tile
                float x[TC];
                if (act) {
                    gather_u8<HH>(im, P.H, P.W, i, j, P.mode, cc->lut, x, LdcgU8());
                } else {
#pragma unroll
                    for (int q = 0; q < TC; q++) x[q] = 0.0f;
                }
                tc_store_input<TC>(tcs, tid, x, P.tc.K[0]);
                tc_network(tcs, P.tc, act ? fraw + tid * P.w.MP : nullptr, 1, mcnt);
                if (cs_ + 1 < P.n_chunks * P.S) tc_prefetch(tcs, P.tc);
            }
            __syncthreads();
        } else {
            if (act) {
                float x[TC];
                gather_u8<HH>(im, P.H, P.W, i, j, P.mode, cc->lut, x, LdcgU8());
#pragma unroll
                for (int q = 0; q < TC; q++) nb.act0[q * NT_TP + tid] = x[q];
            }
            __syncthreads();
            net_tile<CP, TC>(P.w, nb);
        }
        if (dbg && tid == 0) dbg[2] = gtimer();
        if (act) {
            const float* myraw = rawbuf + tid * P.w.MP;
            if (P.trace_raw)
                for (int m = 0; m < P.w.M; m++) P.trace_raw[((int64_t)img * N + n) * P.w.M + m] = myraw[m];
            // g/b mixture record (kernels.py:212-247 minus the rn/gn-dependent update)
            unsigned char* rec = ring + (int64_t)(n & (P.ring_size - 1)) * P.rec_bytes;
            double* d = reinterpret_cast<double*>(rec + 512);
            float* f = reinterpret_cast<float*>(d + 4 * K);
            for (int q = 0; q < K; q++) {
                d[q] = mix_pi(myraw, K, 1, q);
                d[K + q] = mix_inv(myraw, K, 1, q);
                d[2 * K + q] = mix_pi(myraw, K, 2, q);
                d[3 * K + q] = mix_inv(myraw, K, 2, q);
                f[q] = myraw[3 * K + 1 * K + q];
                f[K + q] = myraw[3 * K + 2 * K + q];
                f[2 * K + q] = tanhf_glibc(myraw[9 * K + q]);
                f[3 * K + q] = tanhf_glibc(myraw[10 * K + q]);
                f[4 * K + q] = tanhf_glibc(myraw[11 * K + q]);
            }
            *reinterpret_cast<int32_t*>(f + 5 * K) = (i << 16) | j;
            __threadfence();
        }
        __syncthreads();
        // red tables, one warp per pixel (pixels w, w+8, ...); each record is
        // published as soon as its table is written, so the consumer can start
        // on the first pixels of a chunk before its last table is built
        for (int p = wid; wid < tab_warps && p < npx; p += tab_warps) {   // (other warps only join the barriers)
            const float* myraw = rawbuf + p * P.w.MP;
            const int64_t np_ = (int64_t)n0 + p;
            unsigned char* rec = ring + (int64_t)(np_ & (P.ring_size - 1)) * P.rec_bytes;
            uint32_t start[8], mass[8];
            if (P.f32) warp_table32(myraw, K, 0, 0.0f, 0.0f, cc, sc + wid, start, mass);
            else warp_table(myraw, K, P.dist, 0, 0.0f, 0.0f, cc, sc + wid, start, mass);
            uint4 v;
            v.x = (start[0] & 0xFFFFu) | (start[1] << 16); v.y = (start[2] & 0xFFFFu) | (start[3] << 16);
            v.z = (start[4] & 0xFFFFu) | (start[5] << 16); v.w = (start[6] & 0xFFFFu) | (start[7] << 16);
            reinterpret_cast<uint4*>(rec)[lane] = v;
            __threadfence();                                  // this lane's record bytes, device-wide
            __syncwarp();
            if (lane == 0) st_release_u32(flags + (np_ & (P.ring_size - 1)), (uint32_t)(np_ + 1));
        }
        __syncthreads();                                      // (raw / activation buffers are reused next chunk)
        if (dbg && tid == 0) dbg[3] = gtimer();
    }
    if (P.fast) {
        umma::fence_before();
        __syncthreads();
        umma::fence_after();
        if (tid < TC_M) tc_finish(tcs);
    }
}

// ---------------------------------------------------------------------------
// consumer: the serial chain
// ---------------------------------------------------------------------------
struct ConsumerSmem {
    uint64_t full[DEC_SLOTS];
    uint64_t empty[DEC_SLOTS];
    unsigned long long pubq[DEC_PUBQ];   // tag(8) | r g b (24) | i<<16|j (32), one store per pixel
    uint32_t ready;                      // records [0, ready) are in their slots (loader -> chain)
    uint32_t pub_done;
    ChainSmem ch;
};

template <int KU, int NT, bool F32>
__device__ __forceinline__ void dec_consumer(const DecParams& P, int img0, unsigned char* smem) {
    CdfConsts* cc = reinterpret_cast<CdfConsts*>(smem);
    const size_t grp = ((sizeof(ConsumerSmem) + 127) & ~(size_t)127) + (size_t)DEC_SLOTS * P.rec_bytes;
    unsigned char* gbase = smem + ((sizeof(CdfConsts) + 127) & ~(size_t)127);
    load_consts(cc);
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    const int S = P.S;
    if (tid < S) {
        ConsumerSmem* c0 = reinterpret_cast<ConsumerSmem*>(gbase + tid * grp);
        for (int s = 0; s < DEC_SLOTS; s++) { mbar_init(&c0->full[s], 1); mbar_init(&c0->empty[s], 1); }
        c0->ready = 0; c0->pub_done = 0;
        for (int q = 0; q < DEC_PUBQ; q++) c0->pubq[q] = ~0ull;      // tag 0xFF never matches pixel 0
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    // roles: warps [0, 4S) chains (group g = wid / 4), [4S, 5S) loaders, [5S, 6S) publishers
    int g, role;
    if (wid < 4 * S) { g = wid >> 2; role = 0; }
    else if (wid < 5 * S) { g = wid - 4 * S; role = 1; }
    else if (wid < 6 * S) { g = wid - 5 * S; role = 2; }
    else return;
    const int img = img0 + g;
    if (img >= P.n) return;
    ConsumerSmem* cs = reinterpret_cast<ConsumerSmem*>(gbase + g * grp);
    unsigned char* slots = gbase + g * grp + ((sizeof(ConsumerSmem) + 127) & ~(size_t)127);
    const int bar = 1 + g;
    const int K = P.K;
    const int64_t N = P.N;
    const uint8_t* ring = P.ring + (int64_t)img * P.ring_size * P.rec_bytes;
    const uint32_t* flags = P.flags + (int64_t)img * P.ring_size;
    if (role == 1) {                                  // loader warp
        if (lane == 0) {
            int64_t done = 0;                         // records published to the chain via `ready`
            // publish the copies (issued for records < issued) that have completed
            auto publish = [&](int64_t issued) {
                while (done < issued && mbar_test(&cs->full[done % DEC_SLOTS], (uint32_t)((done / DEC_SLOTS) & 1))) {
                    done++;
                    st_release_cta_u32(&cs->ready, (uint32_t)done);
                }
            };
            for (int64_t n = 0; n < N; n++) {
                const int s = (int)(n % DEC_SLOTS);
                if (n >= DEC_SLOTS) {
                    while (!mbar_test(&cs->empty[s], (uint32_t)(((n / DEC_SLOTS) - 1) & 1))) { publish(n); __nanosleep(LPIC_AUX_SLEEP); }
                }
                const uint32_t* fl = flags + (n & (P.ring_size - 1));
                uint32_t ns = 32;
                while (ld_relaxed_u32(fl) != (uint32_t)(n + 1)) { publish(n); __nanosleep(ns); ns = ns < LPIC_AUX_SLEEP ? ns * 2 : LPIC_AUX_SLEEP; }
                // acquire (pairs with the producer's st.release of the flag), then
                // order the generic-proxy view before the bulk copy's async proxy
                fence_acq_rel_gpu();
                asm volatile("fence.proxy.async.global;" ::: "memory");
                mbar_arrive_tx(&cs->full[s], (uint32_t)P.rec_bytes);
                bulk_g2s(slots + s * P.rec_bytes, ring + (int64_t)(n & (P.ring_size - 1)) * P.rec_bytes,
                         (uint32_t)P.rec_bytes, &cs->full[s]);
                publish(n + 1);
            }
            while (done < N) { publish(N); __nanosleep(LPIC_AUX_SLEEP); }
        }
        return;
    }
    uint8_t* im = P.images + (int64_t)img * N * 3;
    if (role == 2) {                                  // publisher warp: pixels -> global, progress
        if (lane == 0) {
            for (int64_t pub = 0; pub < N;) {
                // drain every slot whose tag says it holds pixel `pub`
                int64_t got = pub;
                while (got < N) {
                    const unsigned long long v = ld_volatile_smem64(&cs->pubq[got % DEC_PUBQ]);
                    if ((uint32_t)(v >> 56) != (uint32_t)(got & 0xFF)) break;
                    const uint32_t ij = (uint32_t)v, rgb = (uint32_t)(v >> 32) & 0xFFFFFFu;
                    uint8_t* px = im + ((int64_t)(ij >> 16) * P.W + (ij & 0xFFFF)) * 3;
                    px[0] = (uint8_t)rgb; px[1] = (uint8_t)(rgb >> 8); px[2] = (uint8_t)(rgb >> 16);
                    got++;
                }
                if (got == pub) { __nanosleep(LPIC_AUX_SLEEP); continue; }
                pub = got;
                *(volatile uint32_t*)&cs->pub_done = (uint32_t)pub;
                st_release_u32(P.progress + img, (uint32_t)pub);
            }
        }
        return;
    }
    const int ct = tid & (CH_THREADS - 1);            // chain-local thread
#ifdef LPIC_DEC_PROF
    if (ct < 16) s_chp[ct] = 0;
    chain_sync(bar);
#endif
    RcDecoder dec;
    dec.init(P.payload + P.offs[img], P.lens[img]);
    ChainSmem* ch = &cs->ch;
    uint32_t avail = 0;                               // records known to be in their slots
    for (int64_t n = 0; n < N; n++) {
        const int s = (int)(n % DEC_SLOTS);
#ifdef LPIC_DEC_TIMELINE
        unsigned long long* dbg = (P.dbg && img == 0) ? P.dbg + 4 * (int64_t)P.n_chunks + 12 * n : nullptr;
#else
        constexpr unsigned long long* dbg = nullptr;  // (per-pixel stamps: timeline builds only)
#endif
        if (dbg && ct == 0) dbg[0] = gtimer();
        if ((int64_t)avail <= n) {
            // the loader publishes completed copies lazily; if it has not yet
            // confirmed record n, wait on the copy's own mbarrier
            avail = ld_acquire_cta_u32(&cs->ready);
            if ((int64_t)avail <= n) {
                mbar_wait(&cs->full[s], (uint32_t)((n / DEC_SLOTS) & 1));
                avail = (uint32_t)(n + 1);
            }
        }
        if (dbg && ct == 0) { dbg[1] = gtimer(); dbg[3] = clock64(); }
        const RecView rv(slots + s * P.rec_bytes, K);
        int32_t* trow = P.trace_cdf ? P.trace_cdf + ((int64_t)img * N + n) * 3 * 257 : nullptr;
        // ---- red: table precomputed by the producer; every warp searches it
        uint64_t r;
#ifdef LPIC_RED_QUOTIENT
        const uint32_t target = dec.target(r);
        auto le = [&](uint32_t c) { return c <= target; };
#else
        // (no quotient on this serial step: cdf_k <= min(code // r, 65535)
        // <=> cdf_k * r <= code, as every cdf_k < 65536 -- coder.py:100-104)
        r = dec.range >> 16;
        const uint64_t code = dec.code;
        auto le = [&](uint32_t c) { return (uint64_t)c * r <= code; };
#endif
        int sr;
        uint32_t red_start, red_width;
        {
            const uint4 v = reinterpret_cast<const uint4*>(rv.red)[lane];
            const uint32_t e[4] = {v.x, v.y, v.z, v.w};
            int c = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) c += le(e[q] & 0xFFFFu) + le(e[q] >> 16);
            sr = __reduce_add_sync(0xffffffffu, c) - 1;
            const uint32_t rs = rv.red[sr];
            const uint32_t re = sr == 255 ? 65536u : (uint32_t)rv.red[sr + 1];
            red_start = rs; red_width = re - rs;          // (advanced inside the green table's Phi phase)
            if (trow) {
                trow[2 * ct] = rv.red[2 * ct];
                trow[2 * ct + 1] = rv.red[2 * ct + 1];
                if (ct == CH_THREADS - 1) trow[256] = 65536;
            }
        }
        const float rn = cc->lut[sr];
        if (dbg && ct == 0) dbg[4] = clock64();
        // ---- green: mu_g += tanh(alpha)*rn (kernels.py:236-237)
        // (the decoder's advance past the previous symbol and the next target
        // are computed inside each table's Phi phase, off the critical path)
        int sg;
        uint32_t st, ms;
        auto tgt_g = [&]() { dec.advance_bf(r, red_start, red_width); return dec.target(r); };
        chain_table<KU, false, F32>(rv.pi_g, rv.inv_g, rv.mu_g, rv.ta, nullptr, rn, 0.0f, K, P.dist, cc, ch, tgt_g, sg,
                               st, ms, trow ? trow + 257 : nullptr, -1, bar);
        const float gn = cc->lut[sg];
        if (dbg && ct == 0) dbg[6] = clock64();
        // ---- blue: mu_b += tanh(beta)*rn + tanh(gamma)*gn (kernels.py:238-240)
        int sb;
        const uint32_t g_start = st, g_width = ms;
        auto tgt_b = [&]() { dec.advance_bf(r, g_start, g_width); return dec.target(r); };
        chain_table<KU, true, F32>(rv.pi_b, rv.inv_b, rv.mu_b, rv.tb, rv.tc, rn, gn, K, P.dist, cc, ch, tgt_b, sb, st,
                              ms, trow ? trow + 514 : nullptr, -1, bar);
        dec.advance_bf(r, st, ms);
        if (dbg && ct == 0) dbg[8] = clock64();
        if (ct == 0) {                                // (slot s was last read before the blue table's barrier A)
            mbar_arrive(&cs->empty[s]);
            // publisher back-pressure: the queue holds DEC_PUBQ pixels, so
            // checking every DEC_PUBQ / 2 pixels for half a queue of room
            // keeps the load off most pixels' critical path
            if ((n & (DEC_PUBQ / 2 - 1)) == 0)
                while ((int64_t)ld_volatile_smem(&cs->pub_done) + DEC_PUBQ / 2 <= n) __nanosleep(20);
            const unsigned long long v = ((unsigned long long)(n & 0xFF) << 56) |
                                         ((unsigned long long)((uint32_t)sr | ((uint32_t)sg << 8) | ((uint32_t)sb << 16)) << 32) |
                                         (uint32_t)rv.ij;
            *(volatile unsigned long long*)&cs->pubq[n % DEC_PUBQ] = v;
            if (dbg) { dbg[2] = gtimer(); dbg[5] = dbg[4]; dbg[7] = dbg[6]; dbg[9] = clock64(); }
        }
    }
    if (ct == 0 && dec.status) atomicOr(P.status + img, dec.status);
#ifdef LPIC_DEC_PROF
    if (P.dbg && img == 0 && ct < 16) P.dbg[4 * (int64_t)P.n_chunks + 12 * N + ct] = (unsigned long long)s_chp[ct];
#endif
}

// NT = 256: one stream per cluster (latency; up to 255 registers per
// thread); NT = 384: DEC_MAXS = 2 streams per cluster (throughput)
template <int CP, int HH, int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1) k_decode2(const __grid_constant__ DecParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int img0 = (blockIdx.x >> 1) * P.S;
    if (cluster_rank() == 0) {
        if (P.f32) {
            if (P.K == 3) dec_consumer<3, NT, true>(P, img0, smem);
            else if (P.K == 2) dec_consumer<2, NT, true>(P, img0, smem);
            else dec_consumer<0, NT, true>(P, img0, smem);
        } else {
            if (P.K == 3) dec_consumer<3, NT, false>(P, img0, smem);
            else if (P.K == 2) dec_consumer<2, NT, false>(P, img0, smem);
            else dec_consumer<0, NT, false>(P, img0, smem);
        }
    } else {
        dec_producer<CP, HH>(P, img0, smem);
    }
}

}  // namespace lpic
