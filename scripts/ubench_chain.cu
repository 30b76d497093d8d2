// Chain builder microbenchmark + correctness check against the warp builder.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I paper_2212_01185_b200/csrc \
//      scripts/ubench_chain.cu -o scripts/ubench_chain
//
// k_check: for random mixtures / rn / gn / targets, the chain builder's
// table (trace row) and decoded symbol must equal warp_table's table and the
// symbol searchsorted on it.  k_time: cycles per chain_table call (K = 3).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#ifdef PROF
__device__ long long g_prof[16];
__shared__ long long s_prof[16];     // shared accumulator: no global latency inside the timed phases
#define LPIC_CHAIN_PROF s_prof
#endif
#include "lpic_chain.cuh"
#include "lpic_rc.cuh"
using namespace lpic;
#define CT chain_table
#define CSM ChainSmem
#define NTH 128

struct Case { float raw[36]; float rn, gn; uint32_t target; int ch; };

__device__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ float urand(uint32_t& s, float lo, float hi) { s = hash32(s + 0x9e3779b9u); return lo + (hi - lo) * (s >> 8) * (1.0f / 16777216.0f); }

// one CTA per case: warp 0 builds the reference table with warp_table, then
// the 4 chain warps run chain_table on the same mixture record
template <bool F32>
__global__ void __launch_bounds__(NTH) k_check(int ncases, int K, int dist, float scale, int* bad, int32_t* rows) {
    __shared__ __align__(16) CdfConsts cc;
    __shared__ __align__(16) CSM cs;
    __shared__ WarpCdfScratch ws;
    __shared__ float raw[12 * KMAX];
    __shared__ double pi[KMAX], inv[KMAX];
    __shared__ float mu0[KMAX], ta[KMAX], tb[KMAX];
    __shared__ int32_t ref[257];
    __shared__ int32_t got[257];
    load_consts(&cc);
    __syncthreads();
    for (int c = blockIdx.x; c < ncases; c += gridDim.x) {
        uint32_t s = 12345u + 7919u * c;
        const int ch = 1 + (c & 1);
        for (int m = threadIdx.x; m < 12 * K; m += blockDim.x) {
            uint32_t ss = s + 101 * m;
            raw[m] = urand(ss, -fabsf(scale), fabsf(scale));
            // scale < 0: near-flat mixtures (log-scales ~7: most remainders in one digit bucket)
            if (scale < 0.0f && m >= 6 * K && m < 9 * K) raw[m] = urand(ss, 6.0f, 7.5f);
        }
        uint32_t s2 = s ^ 0xabcdefu;
        const float rn = urand(s2, -1.0f, 1.0f), gn = urand(s2, -1.0f, 1.0f);
        __syncthreads();
        if (threadIdx.x < K) {
            const int i = threadIdx.x;
            pi[i] = mix_pi(raw, K, ch, i);
            inv[i] = mix_inv(raw, K, ch, i);
            mu0[i] = raw[3 * K + ch * K + i];
            ta[i] = tanhf_glibc(raw[(ch == 1 ? 9 : 10) * K + i]);
            tb[i] = tanhf_glibc(raw[11 * K + i]);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t st[8], ms[8];
            if (F32) warp_table32(raw, K, ch, rn, ch == 2 ? gn : 0.0f, &cc, &ws, st, ms);
            else warp_table(raw, K, dist, ch, rn, ch == 2 ? gn : 0.0f, &cc, &ws, st, ms);
            for (int q = 0; q < 8; q++) ref[8 * threadIdx.x + q] = (int32_t)st[q];
            if (threadIdx.x == 31) ref[256] = (int32_t)(st[7] + ms[7]);
        }
        __syncthreads();
        for (int rep = 0; rep < 3; rep++) {
            uint32_t s3 = s ^ (0x55aa + rep);
            s3 = hash32(s3);
            const uint32_t target = s3 & 0xFFFFu;
            int sym; uint32_t start, mass;
            if (K == 3) {
                if (ch == 1) CT<3, false, F32>(pi, inv, mu0, ta, nullptr, rn, 0.0f, K, dist, &cc, &cs, target, sym, start, mass, got);
                else CT<3, true, F32>(pi, inv, mu0, ta, tb, rn, gn, K, dist, &cc, &cs, target, sym, start, mass, got);
            } else if (K == 2) {
                if (ch == 1) CT<2, false, F32>(pi, inv, mu0, ta, nullptr, rn, 0.0f, K, dist, &cc, &cs, target, sym, start, mass, got);
                else CT<2, true, F32>(pi, inv, mu0, ta, tb, rn, gn, K, dist, &cc, &cs, target, sym, start, mass, got);
            } else {
                if (ch == 1) CT<0, false, F32>(pi, inv, mu0, ta, nullptr, rn, 0.0f, K, dist, &cc, &cs, target, sym, start, mass, got);
                else CT<0, true, F32>(pi, inv, mu0, ta, tb, rn, gn, K, dist, &cc, &cs, target, sym, start, mass, got);
            }
            __syncthreads();
            // expected symbol from the reference table
            int es = 0;
            for (int k = 0; k < 256; k++) if ((uint32_t)ref[k] <= target) es = k;
            const uint32_t est = ref[es], ems = ref[es + 1] - ref[es];
            bool ok = sym == es && start == est && mass == ems;
            for (int k = threadIdx.x; k < 257; k += blockDim.x) ok &= got[k] == ref[k];
            if (!ok) {
                atomicAdd(bad, 1);
                if (rows && atomicCAS(bad + 1, 0, 1) == 0 && threadIdx.x == 0) {
                    for (int k = 0; k < 257; k++) { rows[k] = ref[k]; rows[257 + k] = got[k]; }
                    rows[514] = sym; rows[515] = es; rows[516] = target; rows[517] = c;
                }
            }
            __syncthreads();
        }
    }
}

// spin_warps > 0: that many extra warps poll shared memory with nanosleep
// while the chain runs (the decoder's loader and publisher warps do that)
template <bool F32, bool DEC = false>
__global__ void __launch_bounds__(NTH + 64, 1) k_time(int tables, long long* out, double inv_scale = 1.0,
                                                      int spin_ns = 0, const uint8_t* payload = nullptr,
                                                      int64_t plen = 0) {
    __shared__ volatile int stop;
    __shared__ volatile unsigned long long sink;
    __shared__ __align__(16) CdfConsts cc;
    __shared__ __align__(16) CSM cs;
    __shared__ double pi[4], inv[4];
    __shared__ float mu0[4], ta[4], tb[4];
    load_consts(&cc);
#ifdef PROF
    if (threadIdx.x < 16) s_prof[threadIdx.x] = 0;
#endif
    if (threadIdx.x < 3) {
        pi[threadIdx.x] = 0.3 + 0.05 * threadIdx.x; inv[threadIdx.x] = (1.1 + 0.2 * threadIdx.x) * inv_scale;
        mu0[threadIdx.x] = 0.1f * threadIdx.x - 0.1f; ta[threadIdx.x] = 0.5f; tb[threadIdx.x] = -0.3f;
    }
    if (threadIdx.x == 0) { stop = 0; sink = 0; }
    __syncthreads();
    if (threadIdx.x >= NTH) {                        // spinner warps
        if ((threadIdx.x & 31) == 0) {
            unsigned long long x = 0;
            while (!stop) { __nanosleep(spin_ns); x += sink + 1; }
            sink = x;
        }
        return;
    }
    long long t0 = clock64();
    uint32_t acc = 0;
    uint32_t target = 1234;
    RcDecoder dec;
    if (DEC) dec.init(payload, plen);
    uint64_t r = 0;
    uint32_t p_st = 0, p_ms = 1;
    for (int it = 0; it < tables; it++) {
        const float rn = -1.0f + 0.001f * (it & 1023);
        int sym; uint32_t st, ms;
        if constexpr (DEC) {        // the decoder's deferred advance + target, as in dec_consumer
            auto tgt = [&]() { dec.advance_bf(r, p_st, p_ms); return dec.target(r); };
            CT<3, true, F32>(pi, inv, mu0, ta, tb, rn, 0.25f, 3, 0, &cc, &cs, tgt, sym, st, ms, nullptr);
            p_st = st; p_ms = ms;
        } else {
            CT<3, true, F32>(pi, inv, mu0, ta, tb, rn, 0.25f, 3, 0, &cc, &cs, target, sym, st, ms, nullptr);
        }
        acc += st + ms;
        target = (target * 2654435761u + st) & 0xFFFFu;     // dependency on the previous result
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / tables; out[1] = acc; stop = 1; }
#ifdef PROF
    if (threadIdx.x < 16) g_prof[threadIdx.x] = s_prof[threadIdx.x];
#endif
}

int main() {
    int* bad; int32_t* rows; long long* d;
    cudaMalloc(&bad, 8); cudaMalloc(&rows, 4 * 600); cudaMalloc(&d, 64);
    const int Ks[4] = {3, 2, 5, 1};
    const float scales[4] = {1.0f, 3.0f, 8.0f, -1.0f};
    int total_bad = 0;
    for (int dist = 0; dist < 3; dist++)                 // 2: FAST float32 tables (Gaussian)
        for (int ki = 0; ki < 4; ki++)
            for (int si = 0; si < 4; si++) {
                cudaMemset(bad, 0, 8);
                const int n = 4000;
                if (dist == 2) k_check<true><<<296, NTH>>>(n, Ks[ki], 0, scales[si], bad, rows);
                else k_check<false><<<296, NTH>>>(n, Ks[ki], dist, scales[si], bad, rows);
                int hb[2]; cudaMemcpy(hb, bad, 8, cudaMemcpyDeviceToHost);
                printf("check K=%d dist=%d scale=%.0f: %d / %d mismatches\n", Ks[ki], dist, scales[si], hb[0], 3 * n);
                total_bad += hb[0];
                if (hb[0]) {
                    int32_t h[600]; cudaMemcpy(h, rows, 4 * 600, cudaMemcpyDeviceToHost);
                    printf("  case %d target %d sym got %d exp %d\n", h[517], h[516], h[514], h[515]);
                    int shown = 0;
                    for (int k = 0; k < 257 && shown < 8; k++)
                        if (h[k] != h[257 + k]) { printf("  k=%d ref %d got %d\n", k, h[k], h[257 + k]); shown++; }
                }
            }
    k_time<false><<<1, NTH>>>(20, d); cudaDeviceSynchronize();
    k_time<true><<<1, NTH>>>(4000, d);
    {
        long long h32[2]; cudaMemcpy(h32, d, 16, cudaMemcpyDeviceToHost);
        printf("chain_table K=3 FAST(f32): %lld cycles per table\n", h32[0]);
#ifdef PROF
        long long hp[16]; cudaMemcpyFromSymbol(hp, g_prof, sizeof(hp));
        const char* nm[14] = {"P cdf", "bar E", "pmf+fx", "bar T", "Q rest", "bar A", "S level2+", "prefix", "-",
                              "D search", "Q scale", "P z", "P phi", "S level1"};
        for (int i = 0; i < 14; i++) printf("  f32 %-10s %6lld cycles/table\n", nm[i], hp[i] / 4000);
#endif
    }
    k_time<false><<<1, NTH>>>(4000, d);
    long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("chain_table K=3: %lld cycles per table (%s)\n", h[0], cudaGetErrorString(cudaGetLastError()));
#ifndef PROF
    {   // with the range decoder's deferred advance/target inside the table (as in the decoder)
        uint8_t* pl; cudaMalloc(&pl, 1 << 20);
        cudaMemset(pl, 0x5A, 1 << 20);
        k_time<false, true><<<1, NTH>>>(4000, d, 1.0, 0, pl, 1 << 20);
        long long hs[2]; cudaMemcpy(hs, d, 16, cudaMemcpyDeviceToHost);
        printf("chain_table K=3 with decoder advance/target: %lld cycles per table (%s)\n", hs[0],
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(pl);
    }
    for (int ns : {32, 256}) {   // with two polling warps beside the chain (as in the decoder)
        k_time<false><<<1, NTH + 64>>>(4000, d, 1.0, ns);
        long long hs[2]; cudaMemcpy(hs, d, 16, cudaMemcpyDeviceToHost);
        printf("chain_table K=3 with 2 polling warps (nanosleep %d): %lld cycles per table\n", ns, hs[0]);
    }
    {   // near-flat mixtures (s ~ e^7): most remainders share the first digit
        k_time<false><<<1, NTH>>>(2000, d, 0.001);
        long long hf[2]; cudaMemcpy(hf, d, 16, cudaMemcpyDeviceToHost);
        printf("chain_table K=3 flat: %lld cycles per table\n", hf[0]);
        k_time<false><<<1, NTH>>>(2000, d, 0.02);
        cudaMemcpy(hf, d, 16, cudaMemcpyDeviceToHost);
        printf("chain_table K=3 wide: %lld cycles per table\n", hf[0]);
    }
#endif
#ifdef PROF
    long long hp[16]; cudaMemcpyFromSymbol(hp, g_prof, sizeof(hp));
    const char* nm[14] = {"P cdf", "bar E", "pmf+fx", "bar T", "Q rest", "bar A", "S level2+", "prefix", "-", "D search",
                          "Q scale", "P z", "P phi", "S level1"};
    for (int i = 0; i < 14; i++) printf("  %-10s %6lld cycles/table\n", nm[i], hp[i] / 4000);
    {   // the same phases on near-flat mixtures (crowded threshold bucket)
        k_time<false><<<1, NTH>>>(2000, d, 0.001);
        long long hf[2]; cudaMemcpy(hf, d, 16, cudaMemcpyDeviceToHost);
        printf("chain_table K=3 flat: %lld cycles per table\n", hf[0]);
        cudaMemcpyFromSymbol(hp, g_prof, sizeof(hp));
        for (int i = 0; i < 14; i++) printf("  flat %-10s %6lld cycles/table\n", nm[i], hp[i] / 2000);
    }
#endif
    printf("TOTAL mismatches %d\n", total_bad);
    return total_bad != 0;
}
