// cdf_scale (lpic_cdf.cuh) against IEEE division 65280 / total for totals
// around 1: every double within +-2^26 ulps of 1 on both sides (the
// reciprocal-free near-one path) plus random totals across the guard band.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -I paper_2212_01185_b200/csrc \
//      scripts/check_scale.cu -o scripts/check_scale
#include <cstdio>
#include <cuda_runtime.h>
#include "lpic_cdf.cuh"
using namespace lpic;

__global__ void k_near_one(long long span, unsigned long long* bad) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * span) return;
    const long long k = i - span;                     // ulp offset from 1.0 (below: ulp 2^-53, above: 2^-52)
    const double tot = k < 0 ? 1.0 + (double)k * 1.1102230246251565e-16 : 1.0 + (double)k * 2.220446049250313e-16;
    if (cdf_scale(tot) != __ddiv_rn(CDF_FLOOR, tot)) atomicAdd(bad, 1ull);
}
__global__ void k_random(unsigned long long n, unsigned long long* bad) {
    unsigned long long x = 0x9E3779B97F4A7C15ull * ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x + 1);
    for (unsigned long long i = 0; i < n; i++) {
        x ^= x >> 12; x ^= x << 25; x ^= x >> 27;
        const unsigned long long r = x * 2685821657736338717ull;
        // e uniform in log scale over [2^-60, 2^-20], either sign
        const double mag = ldexp(1.0 + (double)(r >> 11) * 0x1p-53, -20 - (int)((r >> 3) % 41));
        const double tot = (r & 1) ? 1.0 + mag : 1.0 - mag;
        if (cdf_scale(tot) != __ddiv_rn(CDF_FLOOR, tot)) atomicAdd(bad, 1ull);
    }
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
    const long long span = 1ll << 26;
    k_near_one<<<(unsigned)((2 * span + 255) / 256), 256>>>(span, d);
    unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cdf_scale vs IEEE division, totals 1 +- 2^26 ulps (%lld values): %llu mismatches\n", 2 * span, h);
    cudaMemset(d, 0, 8);
    k_random<<<148 * 8, 256>>>(4096, d);
    unsigned long long h2 = 0; cudaMemcpy(&h2, d, 8, cudaMemcpyDeviceToHost);
    printf("cdf_scale vs IEEE division, %.3g random totals 1 +- [2^-60, 2^-20]: %llu mismatches (%s)\n",
           148.0 * 8 * 256 * 4096, h2, cudaGetErrorString(cudaGetLastError()));
    return (h || h2) ? 1 : 0;
}
