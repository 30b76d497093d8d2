// Latency of phi_gauss_vec<6> per call, one CTA of 128 threads (the chain's P phase core).
#include <cstdio>
#include <cuda_runtime.h>
#include "lpic_cdf.cuh"
using namespace lpic;
template <int N>
__global__ void __launch_bounds__(128, 1) k_phi(int iters, long long* out, double* sink) {
    __shared__ __align__(16) CdfConsts cc;
    load_consts(&cc);
    __syncthreads();
    double z[N];
    for (int i = 0; i < N; i++) z[i] = -3.0 + 0.02 * threadIdx.x + 0.3 * i;
    double acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        double o[N];
        phi_gauss_vec<N>(z, o, cc.phic);
        for (int i = 0; i < N; i++) { acc += o[i]; z[i] = __dadd_rn(z[i], o[i] * 1e-3); }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    if (acc == 12345.0) sink[0] = acc;
}
int main() {
    long long* d; double* s; cudaMalloc(&d, 64); cudaMalloc(&s, 64);
    long long h;
    k_phi<6><<<1, 128>>>(10, d, s); cudaDeviceSynchronize();
    k_phi<6><<<1, 128>>>(2000, d, s); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("phi_gauss_vec<6>, 128 thr: %lld cycles/call\n", h);
    k_phi<2><<<1, 128>>>(2000, d, s); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("phi_gauss_vec<2>, 128 thr: %lld cycles/call\n", h);
    k_phi<6><<<1, 32>>>(2000, d, s); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("phi_gauss_vec<6>, 32 thr: %lld cycles/call\n", h);
    k_phi<6><<<1, 256>>>(2000, d, s); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("phi_gauss_vec<6>, 256 thr: %lld cycles/call\n", h);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
