// lpic_decode_cp32.cu -- k_decode2 instantiations for CP = 32 (see lpic_decode_launch.h)
#include "lpic_decode_launch.h"

namespace lpic {
cudaError_t launch_decode2_cp32(int HH, int S, int n, size_t smem, cudaStream_t st, const DecParams& P) {
    if (HH == 1) return launch_decode2_t<32, 1>(S, n, smem, st, P);
    if (HH == 2) return launch_decode2_t<32, 2>(S, n, smem, st, P);
    if (HH == 3) return launch_decode2_t<32, 3>(S, n, smem, st, P);
    return cudaErrorInvalidValue;
}
}  // namespace lpic
