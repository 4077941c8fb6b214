// Register-tile heat phase kernels for block 12 (colkernel.cuh).
#include "colkernel.cuh"

namespace sg {
cudaError_t launch_heat_col12(const SweptArgs& a, cudaStream_t s) { return launch_heat_col<12>(a, s); }
}  // namespace sg
