// Register-tile heat phase kernels for block 24 (colkernel.cuh).
#include "colkernel.cuh"

namespace sg {
cudaError_t launch_heat_col24(const SweptArgs& a, cudaStream_t s) { return launch_heat_col<24>(a, s); }
}  // namespace sg
