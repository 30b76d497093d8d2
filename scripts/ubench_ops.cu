// Dependent-chain latency of warp primitives on B200 (one warp, clock64).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/ubench_ops.cu -o scripts/ubench_ops
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 512
__global__ void k_ops(long long* out, int seed) {
    __shared__ uint32_t sm[1024];
    __shared__ double smd[256];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + seed) & 1023;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) smd[i] = 0.001 * i;
    __syncthreads();
    uint32_t x = lane + seed;
    double d = 0.5 + lane * 1e-3;
    long long t0, t1;
    int r = 0;
#define TIME(name, body)                                                   \
    __syncwarp(); t0 = clock64();                                          \
    for (int i = 0; i < ITERS; i++) { body; }                              \
    __syncwarp(); t1 = clock64();                                          \
    if (threadIdx.x == 0) out[r] = (t1 - t0) / ITERS; r++;
    TIME("redux", x = __reduce_add_sync(0xffffffffu, x) & 31)
    TIME("vote", x = __popc(__ballot_sync(0xffffffffu, x & 1)) + lane)
    TIME("vote_only", x = __ballot_sync(0xffffffffu, x & 1) ^ lane)
    TIME("shfl", x = __shfl_sync(0xffffffffu, x, (x + 1) & 31))
    TIME("shfl_up", x = __shfl_up_sync(0xffffffffu, x, 1) + 1)
    TIME("match", x = __match_any_sync(0xffffffffu, x & 7) & 31)
    TIME("lds", x = sm[x & 1023])
    TIME("iadd", x = x * 3 + 1)
    TIME("dfma", d = __fma_rn(d, 1.0000001, 1e-9))
    TIME("f2i.f64", d = (double)__double2int_rz(d * 3.0) + 0.25)
    TIME("frnd.floor", d = floor(d * 1.5) + 0.25)
    TIME("i2f.f64", x = (uint32_t)(__uint2double_rn(x) * 0.5))
    TIME("f2f.f64.f32", d = (double)(float)(d + 1.0))
    TIME("dsetp+sel", d = (d > 0.7) ? d * 0.5 : d * 1.5)
    TIME("bar128", __syncthreads())
    TIME("lds.f64", d = smd[((int)d) & 255] + 0.5)
    if (threadIdx.x == 0) out[r] = x + (long long)d;
}

int main() {
    long long* d; cudaMalloc(&d, 8 * 64);
    const char* nm[] = {"redux", "vote+popc", "vote", "shfl.idx", "shfl.up", "match.any", "lds (dep)", "imad",
                        "dfma", "f2i.f64+i2f", "frnd.floor+dfma", "i2f.f64+f2i", "f2f roundtrip", "dsetp+dmul", "bar.sync(128)",
                        "lds.f64 (dep)"};
    for (int nt : {32, 128}) {
        k_ops<<<1, nt>>>(d, 1); cudaDeviceSynchronize();
        k_ops<<<1, nt>>>(d, 2);
        long long h[17]; cudaMemcpy(h, d, 8 * 17, cudaMemcpyDeviceToHost);
        printf("--- %d threads\n", nt);
        for (int i = 0; i < 16; i++) printf("  %-18s %4lld cycles/iter\n", nm[i], h[i]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
