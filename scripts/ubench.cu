// Microbenchmarks of the primitives the LPIC kernels are built from (B200).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I paper_2212_01185_b200/csrc scripts/ubench.cu -o ubench
#include <cstdio>
#include <cuda_runtime.h>
#include "lpic_cdf.cuh"

using namespace lpic;

__global__ void k_dfma_lat(double* out, int iters) {
    double a = out[0], b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; i++) a = __fma_rn(a, b, c);
    if (a == 12345.0) out[1] = a;
}
__global__ void k_dfma_tput(double* out, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; i++) {
        a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c); a3 = __fma_rn(a3, b, c);
        a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c); a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c);
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.0) out[1] = a0;
}
__global__ void k_fp32_tput(float* out, int iters) {
    float a[8], acc[8];
    for (int k = 0; k < 8; k++) { a[k] = threadIdx.x + k; acc[k] = 0.f; }
    const float b = 1.0001f;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) acc[k] = __fadd_rn(acc[k], __fmul_rn(a[k], b));
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = __fadd_rn(a[k], 1e-7f);
    }
    float s = 0; for (int k = 0; k < 8; k++) s += acc[k];
    if (s == 12345.f) out[1] = s;
}
__global__ void k_phi_tput(double* out, int iters) {
    __shared__ __align__(16) CdfConsts cc;
    load_consts(&cc);
    __syncthreads();
    double z = -8.0 + (threadIdx.x % 256) * 0.06, s = 0;
    for (int i = 0; i < iters; i++) { s = __dadd_rn(s, phi_gauss(z, cc.phic)); z = __dadd_rn(z, 1e-6); }
    if (s == 12345.0) out[1] = s;
}
__global__ void k_phi_lat(double* out, int iters) {
    __shared__ __align__(16) CdfConsts cc;
    load_consts(&cc);
    __syncthreads();
    if (threadIdx.x) return;
    double z = -1.5;
    for (int i = 0; i < iters; i++) z = __dsub_rn(phi_gauss(z, cc.phic), 1.5);
    out[1] = z;
}
__global__ void k_block_table(double* out, int tables, long long* cyc) {
    __shared__ __align__(16) CdfConsts cc;
    __shared__ BlockCdfScratch sc;
    load_consts(&cc);
    __syncthreads();
    const int k = threadIdx.x, lane = k & 31;
    double mu0 = 0.1, inv = 1.3, pi = 1.0;
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int it = 0; it < tables; it++) {
        double pmf = 0.0;
        for (int q = 0; q < 3; q++) {
            const double mu = mu0 + 0.01 * q + 1e-5 * it;
            const double cur = (k == 255) ? 1.0 : phi_gauss(__dmul_rn(__dsub_rn(cc.edges[k + 1], mu), inv), cc.phic);
            double prev = __shfl_up_sync(0xffffffffu, cur, 1);
            if (lane == 0) prev = (k == 0) ? 0.0 : phi_gauss(__dmul_rn(__dsub_rn(cc.edges[k], mu), inv), cc.phic);
            const double d = __dsub_rn(cur, prev);
            if (d > 0.0) pmf = __dadd_rn(pmf, __dmul_rn(pi / 3, d));
        }
        uint32_t st, ms;
        block_quantize(pmf, &sc, st, ms);
        acc += st;
    }
    long long t1 = clock64();
    if (k == 0) { cyc[0] = t1 - t0; out[1] = acc; }
}
__global__ void k_block_quant_only(double* out, int tables, long long* cyc) {
    __shared__ BlockCdfScratch sc;
    const int k = threadIdx.x;
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int it = 0; it < tables; it++) {
        double pmf = 1.0 / 256 + 1e-4 * ((k * 7 + it) % 13);
        uint32_t st, ms;
        block_quantize(pmf, &sc, st, ms);
        acc += st;
    }
    long long t1 = clock64();
    if (k == 0) { cyc[0] = t1 - t0; out[1] = acc; }
}
__global__ void k_warp_table(double* out, int tables, long long* cyc, int nwarps_timed) {
    __shared__ __align__(16) CdfConsts cc;
    __shared__ WarpCdfScratch sc[8];
    load_consts(&cc);
    __syncthreads();
    const int wid = threadIdx.x >> 5;
    float raw[36];
    for (int m = 0; m < 36; m++) raw[m] = 0.1f * ((m * 7 + wid) % 11) - 0.5f;
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int it = 0; it < tables; it++) {
        raw[9] += 1e-3f;
        uint32_t st[8], ms[8];
        warp_table(raw, 3, 0, 1, 0.3f, 0.0f, &cc, sc + wid, st, ms);
        acc += st[3];
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && wid == 0) { cyc[0] = t1 - t0; out[1] = acc; }
}

__global__ void k_div_check(unsigned long long* bad, unsigned long long seed, int iters) {
    unsigned long long x = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
    unsigned long long nb = 0;
    for (int i = 0; i < iters; i++) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        // tot in [2^-8, 2^4): random mantissa and exponent
        const double tot = __longlong_as_double((long long)((x & 0x000FFFFFFFFFFFFFull) | ((unsigned long long)(1023 - 8 + (x >> 60) % 12) << 52)));
        if (div_rn_fast(65280.0, tot) != __ddiv_rn(65280.0, tot)) nb++;
    }
    atomicAdd(bad, nb);
}
int main() {
    double* d; long long* c; float* f;
    cudaMalloc(&d, 64); cudaMalloc(&c, 64); cudaMalloc(&f, 64);
    cudaMemset(d, 0, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs %d clock %d kHz\n", sms, clk);
    const double ghz = clk / 1e6;
    // DFMA latency
    k_dfma_lat<<<1, 1>>>(d, 1000); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dfma_lat<<<1, 1>>>(d, 1 << 20); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA dependent latency: %.2f cycles\n", ms * 1e-3 * ghz * 1e9 / (1 << 20));
    // DFMA throughput
    int it = 1 << 14;
    k_dfma_tput<<<sms * 8, 256>>>(d, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dfma_tput<<<sms * 8, 256>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double dfma = (double)sms * 8 * 256 * it * 8;
    printf("DFMA throughput: %.1f TFLOP/s  (%.1f DFMA/clk/SM)\n", dfma * 2 / (ms * 1e-3) / 1e12, dfma / (ms * 1e-3) / (ghz * 1e9) / sms);
    // FP32 mul+add throughput (separate ops)
    k_fp32_tput<<<sms * 8, 256>>>(f, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_fp32_tput<<<sms * 8, 256>>>(f, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double f32 = (double)sms * 8 * 256 * it * 24;
    printf("FP32 FMUL/FADD: %.1f lane-ops/clk/SM\n", f32 / (ms * 1e-3) / (ghz * 1e9) / sms);
    // phi throughput
    k_phi_tput<<<sms * 4, 256>>>(d, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_phi_tput<<<sms * 4, 256>>>(d, 4096); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double nphi = (double)sms * 4 * 256 * 4096;
    printf("phi throughput: %.2f Gphi/s (%.1f cycles per phi per SM)\n", nphi / (ms * 1e-3) / 1e9, (ms * 1e-3) * ghz * 1e9 * sms / nphi);
    k_phi_lat<<<1, 32>>>(d, 1000); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_phi_lat<<<1, 32>>>(d, 1 << 16); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("phi latency: %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / (1 << 16));
    long long cy;
    k_block_table<<<1, 256>>>(d, 10, c); cudaDeviceSynchronize();
    k_block_table<<<1, 256>>>(d, 2000, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("block table (256 thr, K=3): %.0f cycles per table\n", cy / 2000.0);
    k_block_quant_only<<<1, 256>>>(d, 2000, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("block quantize only: %.0f cycles per table\n", cy / 2000.0);
    for (int nw : {1, 4, 8}) {
        k_warp_table<<<1, 32 * nw>>>(d, 500, c, nw); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("warp table, %d warps/CTA: %.0f cycles per table (latency)\n", nw, cy / 500.0);
    }
    cudaEventRecord(e0); k_warp_table<<<sms * 4, 256>>>(d, 200, c, 8); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("warp table throughput: %.1f Mtables/s (%.0f cycles/table/SM)\n", sms * 4 * 8 * 200 / (ms * 1e-3) / 1e6,
           (ms * 1e-3) * ghz * 1e9 * sms / (sms * 4 * 8 * 200.0));
    unsigned long long* bad; cudaMalloc(&bad, 8); cudaMemset(bad, 0, 8);
    k_div_check<<<sms * 8, 256>>>(bad, 12345, 4096);
    unsigned long long hb; cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    printf("div_rn_fast vs __ddiv_rn: %llu mismatches in %.3g random totals\n", hb, (double)sms * 8 * 256 * 4096);
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
