// Register-tile heat phase kernels for block 8 (colkernel.cuh).
#include "colkernel.cuh"

namespace sg {
cudaError_t launch_heat_col8(const SweptArgs& a, cudaStream_t s) { return launch_heat_col<8>(a, s); }
}  // namespace sg
