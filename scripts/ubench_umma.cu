// tcgen05 sanity test: D[128 x N] = A[128 x K] . B[N x K]^T in fp16 -> fp32 TMEM,
// operands in the K-major SWIZZLE_NONE layout of lpic_umma.cuh; compared with
// a CPU double-precision product of the same fp16 values.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2212_01185_b200/csrc scripts/ubench_umma.cu -o scripts/ubench_umma
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "lpic_umma.cuh"
using namespace lpic;

constexpr int M = 128, N = 128, K = 128;

__global__ void __launch_bounds__(128) k_test(const __half* A, const __half* B, float* D) {
    extern __shared__ __align__(128) unsigned char sm[];
    __half* sA = reinterpret_cast<__half*>(sm);
    __half* sB = reinterpret_cast<__half*>(sm + M * K * 2);
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5;
    // load operands into the canonical layout
    for (int e = tid; e < M * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<__half*>(sm + umma::op_offset(r, k, K)) = A[e];
    }
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<__half*>(sm + M * K * 2 + umma::op_offset(r, k, K)) = B[e];
    }
    if (warp == 0) umma::tmem_alloc(&tmem_base, 128);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(umma::smem_addr(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = umma::idesc_f16(M, N);
        for (int ks = 0; ks < K / 16; ks++) {
            const uint64_t ad = umma::smem_desc(umma::smem_addr(sm) + ks * 256, 128, K * 16);
            const uint64_t bd = umma::smem_desc(umma::smem_addr(sm + M * K * 2) + ks * 256, 128, K * 16);
            umma::mma_f16(tbase, ad, bd, idesc, ks > 0);
        }
        umma::commit(&mbar);
    }
    // wait for the MMAs
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(umma::smem_addr(&mbar)) : "memory");
        }
    }
    umma::fence_after();
    const int row = 32 * (warp & 3) + (tid & 31);
    for (int c = 0; c < N; c += 32) {
        float v[32];
        umma::tmem_ld32(tbase + ((uint32_t)(32 * (warp & 3)) << 16) + c, v);
        for (int i = 0; i < 32; i++) D[row * N + c + i] = v[i];
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tbase, 128);
}

int main() {
    std::vector<__half> hA(M * K), hB(N * K);
    std::vector<float> fA(M * K), fB(N * K);
    srand(1);
    for (int i = 0; i < M * K; i++) { float x = (rand() % 2001 - 1000) / 512.0f; hA[i] = __float2half(x); fA[i] = __half2float(hA[i]); }
    for (int i = 0; i < N * K; i++) { float x = (rand() % 2001 - 1000) / 1024.0f; hB[i] = __float2half(x); fB[i] = __half2float(hB[i]); }
    __half *dA, *dB; float* dD;
    cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
    const size_t smem = (M + N) * K * 2;
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_test<<<1, 128, smem>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> hD(M * N);
    cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; m++)
        for (int n = 0; n < N; n++) {
            double ref = 0;
            for (int k = 0; k < K; k++) ref += (double)fA[m * K + k] * fB[n * K + k];
            maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
            maxref = fmax(maxref, fabs(ref));
        }
    printf("max |err| %.3e (max |ref| %.3f) D[0]=%f D[1]=%f D[N]=%f\n", maxerr, maxref, hD[0], hD[1], hD[N]);
    printf("%s\n", maxerr < 1e-3 * maxref ? "UMMA OK" : "UMMA MISMATCH");
    return 0;
}
