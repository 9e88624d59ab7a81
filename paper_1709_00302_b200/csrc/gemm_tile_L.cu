// DMMA GEMM tile configuration L: 128x128, BK=16, warps 4x2, 3 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_L, 128, 128, 16, 4, 2, 3, 1)
}  // namespace br
