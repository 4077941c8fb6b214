// Register-tile heat phase kernels for block 32 (colkernel.cuh).
#include "colkernel.cuh"

namespace sg {
cudaError_t launch_heat_col32(const SweptArgs& a, cudaStream_t s) { return launch_heat_col<32>(a, s); }
}  // namespace sg
