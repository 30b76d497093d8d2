// lpic_decode_launch.h -- host launcher of the wavefront decoder kernel.
// The k_decode2<CP, HH, NT> instantiations are spread over one translation
// unit per padded filter count (lpic_decode_cp*.cu) so the library builds in
// parallel; lpic_kernels.cu calls them through this function.
#pragma once
#include <cuda_runtime.h>

#include "lpic_decode.cuh"

namespace lpic {
// S == 1: 256-thread clusters, one stream each; S == 2: 384-thread clusters
cudaError_t launch_decode2(int CP, int HH, int S, int n, size_t smem, cudaStream_t st, const DecParams& P);
cudaError_t launch_decode2_cp16(int HH, int S, int n, size_t smem, cudaStream_t st, const DecParams& P);
cudaError_t launch_decode2_cp32(int HH, int S, int n, size_t smem, cudaStream_t st, const DecParams& P);
cudaError_t launch_decode2_cp64(int HH, int S, int n, size_t smem, cudaStream_t st, const DecParams& P);
cudaError_t launch_decode2_cp128(int HH, int S, int n, size_t smem, cudaStream_t st, const DecParams& P);

template <int CP, int HH>
cudaError_t launch_decode2_t(int S, int n, size_t smem, cudaStream_t st, const DecParams& P) {
    cudaError_t e;
    if (S == 1) {
        e = cudaFuncSetAttribute(k_decode2<CP, HH, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_decode2<CP, HH, 256><<<2 * n, 256, smem, st>>>(P);
    } else {
        e = cudaFuncSetAttribute(k_decode2<CP, HH, DEC_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_decode2<CP, HH, DEC_THREADS><<<2 * ((n + S - 1) / S), DEC_THREADS, smem, st>>>(P);
    }
    return cudaGetLastError();
}
}  // namespace lpic
