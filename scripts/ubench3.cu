// The decoder chain's table build (chain_pmf + block_quantize) in a loop on one CTA.
#include <cstdio>
#include <cuda_runtime.h>
#include "lpic_decode.cuh"
using namespace lpic;
__global__ void __launch_bounds__(256, 1) k_chain(long long* out, int tables) {
    __shared__ __align__(16) CdfConsts cc;
    __shared__ __align__(16) ConsumerSmem cs;
    __shared__ double pi[4], inv[4];
    __shared__ float mu0[4], ta[4];
    load_consts(&cc);
    if (threadIdx.x < 4) { pi[threadIdx.x] = 0.3 + 0.05 * threadIdx.x; inv[threadIdx.x] = 1.1 + 0.2 * threadIdx.x;
                           mu0[threadIdx.x] = 0.1f * threadIdx.x - 0.1f; ta[threadIdx.x] = 0.5f; }
    __syncthreads();
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int it = 0; it < tables; it++) {
        const float rn = -1.0f + 0.001f * (it & 1023);
        double pmf = chain_pmf<false>(pi, inv, mu0, ta, nullptr, rn, 0.0f, 3, 0, &cc, cs.wedge);
        uint32_t st, ms;
        block_quantize(pmf, &cs.sc, st, ms);
        acc += st;
        team_sync();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / tables; out[1] = acc; }
}
int main() {
    long long* d; cudaMalloc(&d, 64);
    k_chain<<<1, 256>>>(d, 20); cudaDeviceSynchronize();
    k_chain<<<1, 256>>>(d, 2000);
    long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("chain table: %lld cycles per table (%s)\n", h[0], cudaGetErrorString(cudaGetLastError()));
}
