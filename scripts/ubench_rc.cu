// Range encoder cycles/symbol on one thread (diagnostics for k_rc_encode).
#include <cstdio>
#include <cuda_runtime.h>
#include "lpic_rc.cuh"
using namespace lpic;
template <bool WRITE>
__global__ void k_rc(const uint32_t* sw, int n, uint8_t* out, long long* res) {
    if (threadIdx.x) return;
    RcEncoder e; e.init(out, 8 * n);
    long long t0 = clock64();
    for (int k = 0; k < n; k++) { const uint32_t x = sw[k]; e.encode(x >> 16, (x & 0xFFFFu) + 1u, WRITE); }
    long long t1 = clock64();
    res[0] = (t1 - t0) / n; res[1] = e.finish(WRITE);
}
__global__ void k_arith(const uint32_t* sw, int n, long long* res) {   // coder arithmetic only
    if (threadIdx.x) return;
    uint64_t low = 0, range = RC_TOP - 1; int emitted = 0;
    long long t0 = clock64();
    for (int k = 0; k < n; k++) {
        const uint32_t x = sw[k];
        const uint64_t r = range >> 16;
        low += r * (x >> 16); range = r * ((x & 0xFFFFu) + 1u);
        if (low >= RC_TOP) low -= RC_TOP;
        while (range < RC_BOTTOM) { emitted += (int)((low >> 40) & 0xFF); low = (low << 8) & RC_MASK; range <<= 8; }
    }
    long long t1 = clock64();
    res[0] = (t1 - t0) / n; res[1] = emitted;
}
int main() {
    const int n = 1 << 20;
    uint32_t* h = new uint32_t[n];
    unsigned s = 1;
    for (int k = 0; k < n; k++) { s = s * 1103515245u + 12345u; unsigned w = 200 + (s >> 16) % 100; unsigned st = (s >> 8) % (65536 - w); h[k] = (st << 16) | (w - 1); }
    uint32_t* d; uint8_t* o; long long* r; cudaMalloc(&d, 4 * n); cudaMalloc(&o, 8 * n); cudaMalloc(&r, 16);
    cudaMemcpy(d, h, 4 * n, cudaMemcpyHostToDevice);
    long long hr[2];
    k_rc<true><<<1, 32>>>(d, n, o, r); cudaMemcpy(hr, r, 16, cudaMemcpyDeviceToHost); printf("encode+write: %lld cycles/sym (%lld B)\n", hr[0], hr[1]);
    k_rc<false><<<1, 32>>>(d, n, o, r); cudaMemcpy(hr, r, 16, cudaMemcpyDeviceToHost); printf("encode no-write: %lld cycles/sym\n", hr[0]);
    k_arith<<<1, 32>>>(d, n, r); cudaMemcpy(hr, r, 16, cudaMemcpyDeviceToHost); printf("arith only: %lld cycles/sym\n", hr[0]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
