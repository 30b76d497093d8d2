// Phi-evaluation throughput peak of this B200: the fp64 Gaussian CDF the
// table builders use (phi_gauss_vec, lpic_cdf.cuh), every SM busy, many warps,
// independent arguments (ILP 4).  The bench's "phi" roofline divides the
// achieved Phi evaluations per second (765 per sub-pixel) by this.
// Also the fp32 (FAST) variant and FFMA vs FMUL2/FFMA2 issue rates for the
// compat network (scripts note in DESIGN.md).
#include <cstdio>
#include <cuda_runtime.h>
#include "lpic_cdf.cuh"
using namespace lpic;

__global__ void __launch_bounds__(256) k_phi_peak(int iters, double* sink) {
    __shared__ __align__(16) CdfConsts cc;
    load_consts(&cc);
    __syncthreads();
    double z[4];
    for (int i = 0; i < 4; i++) z[i] = -4.0 + 0.031 * (threadIdx.x & 255) + 0.7 * i + 1e-3 * blockIdx.x;
    double acc = 0;
    for (int it = 0; it < iters; it++) {
        double o[4];
        phi_gauss_vec<4>(z, o, cc.phic);
#pragma unroll
        for (int i = 0; i < 4; i++) { acc = __dadd_rn(acc, o[i]); z[i] = __dadd_rn(z[i], 1.0e-3); }
    }
    if (acc == 12345.0) sink[0] = acc;
}
__global__ void __launch_bounds__(256) k_phi32_peak(int iters, float* sink) {
    __shared__ __align__(16) CdfConsts cc;
    load_consts(&cc);
    __syncthreads();
    float z[4];
    for (int i = 0; i < 4; i++) z[i] = -4.0f + 0.031f * (threadIdx.x & 255) + 0.7f * i + 1e-3f * blockIdx.x;
    float acc = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 4; i++) { acc = __fadd_rn(acc, phiq32(z[i], cc.phic32)); z[i] = __fadd_rn(z[i], 1.0e-3f); }
    }
    if (acc == 12345.0f) sink[0] = acc;
}
// fp32 multiply-add issue: separate FMUL+FADD (the compat network's
// canonical order) vs packed FMUL2 + FFMA2(x, 1, acc) (the same IEEE
// operations, two lanes per instruction)
__global__ void __launch_bounds__(256) k_fmul_fadd(int iters, float* sink, float wv) {
    float a[8], w[8];
    for (int i = 0; i < 8; i++) { a[i] = 1.0f + 1e-3f * i + 1e-6f * threadIdx.x; w[i] = wv + 1e-4f * i; }
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] = __fadd_rn(a[i], __fmul_rn(w[i], a[(i + 1) & 7]));
    float s = 0;
    for (int i = 0; i < 8; i++) s += a[i];
    if (s == 12345.0f) sink[0] = s;
}
__device__ __forceinline__ unsigned long long f2pack(float x, float y) {
    return (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(y) << 32);
}
__global__ void __launch_bounds__(256) k_fmul2_ffma2(int iters, float* sink, float wv, float one) {
    unsigned long long a[4], w[4];
    const unsigned long long o2 = f2pack(one, one);
    for (int i = 0; i < 4; i++) {
        a[i] = f2pack(1.0f + 1e-3f * i + 1e-6f * threadIdx.x, 1.0f + 1e-3f * (i + 4));
        w[i] = f2pack(wv + 1e-4f * i, wv + 1e-4f * (i + 4));
    }
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 4; i++) {
            unsigned long long p;
            asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(w[i]), "l"(a[(i + 1) & 3]));
            asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(a[i]) : "l"(p), "l"(o2), "l"(a[i]));
        }
    float s = 0;
    for (int i = 0; i < 4; i++) s += __uint_as_float((unsigned)a[i]) + __uint_as_float((unsigned)(a[i] >> 32));
    if (s == 12345.0f) sink[0] = s;
}
// correctness of the packed pair against the scalar pair on random data
__global__ void k_pack_check(const float* x, const float* y, const float* z, int n, float one, int* bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    const float r0 = __fadd_rn(z[2 * i], __fmul_rn(x[2 * i], y[2 * i]));
    const float r1 = __fadd_rn(z[2 * i + 1], __fmul_rn(x[2 * i + 1], y[2 * i + 1]));
    unsigned long long p, q;
    asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(f2pack(x[2 * i], x[2 * i + 1])), "l"(f2pack(y[2 * i], y[2 * i + 1])));
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(q) : "l"(p), "l"(f2pack(one, one)), "l"(f2pack(z[2 * i], z[2 * i + 1])));
    if (__float_as_uint(r0) != (unsigned)q || __float_as_uint(r1) != (unsigned)(q >> 32)) atomicAdd(bad, 1);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sd; float* sf;
    cudaMalloc(&sd, 64); cudaMalloc(&sf, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = sms * 8, thr = 256, iters = 4000;
    float ms;
    k_phi_peak<<<blocks, thr>>>(10, sd);
    cudaEventRecord(e0); k_phi_peak<<<blocks, thr>>>(iters, sd); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double phi64 = (double)blocks * thr * iters * 4 / (ms * 1e-3);
    k_phi32_peak<<<blocks, thr>>>(10, sf);
    cudaEventRecord(e0); k_phi32_peak<<<blocks, thr>>>(iters, sf); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double phi32 = (double)blocks * thr * iters * 4 / (ms * 1e-3);
    k_fmul_fadd<<<blocks, thr>>>(10, sf, 0.999f);
    cudaEventRecord(e0); k_fmul_fadd<<<blocks, thr>>>(iters, sf, 0.999f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mac1 = (double)blocks * thr * iters * 8 / (ms * 1e-3);
    k_fmul2_ffma2<<<blocks, thr>>>(10, sf, 0.999f, 1.0f);
    cudaEventRecord(e0); k_fmul2_ffma2<<<blocks, thr>>>(iters, sf, 0.999f, 1.0f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double mac2 = (double)blocks * thr * iters * 8 / (ms * 1e-3);
    // packed-pair correctness on 2^24 random triples
    const int n = 1 << 24;
    float *x, *y, *z; int* bad;
    cudaMallocManaged(&x, n * 4); cudaMallocManaged(&y, n * 4); cudaMallocManaged(&z, n * 4); cudaMallocManaged(&bad, 4);
    unsigned s = 12345;
    for (int i = 0; i < n; i++) {
        s = s * 1664525u + 1013904223u; x[i] = ((s >> 8) * (1.0f / 16777216.0f) - 0.5f) * 8.0f;
        s = s * 1664525u + 1013904223u; y[i] = ((s >> 8) * (1.0f / 16777216.0f) - 0.5f) * 3.0f;
        s = s * 1664525u + 1013904223u; z[i] = ((s >> 8) * (1.0f / 16777216.0f) - 0.5f) * 5.0f;
    }
    *bad = 0;
    k_pack_check<<<(n / 2 + 255) / 256, 256>>>(x, y, z, n, 1.0f, bad);
    cudaDeviceSynchronize();
    printf("{\"sms\": %d, \"phi64_evals_per_s\": %.4e, \"phi32_evals_per_s\": %.4e, "
           "\"fp32_mac_fmul_fadd_per_s\": %.4e, \"fp32_mac_fmul2_ffma2_per_s\": %.4e, \"packed_pair_mismatches\": %d, "
           "\"packed_pair_cases\": %d, \"err\": \"%s\"}\n",
           sms, phi64, phi32, mac1, mac2, *bad, n / 2, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
