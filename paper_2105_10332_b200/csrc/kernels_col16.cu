// Register-tile heat phase kernels for block 16 (colkernel.cuh).
#include "colkernel.cuh"

namespace sg {
cudaError_t launch_heat_col16(const SweptArgs& a, cudaStream_t s) { return launch_heat_col<16>(a, s); }
}  // namespace sg
