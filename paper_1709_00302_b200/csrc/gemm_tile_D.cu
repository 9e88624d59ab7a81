// DMMA GEMM tile configuration D: 64x64, BK=16, warps 2x2, 4 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_D, 64, 64, 16, 2, 2, 4, 3)
}  // namespace br
