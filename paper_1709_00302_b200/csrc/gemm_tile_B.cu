// DMMA GEMM tile configuration B: 128x64, BK=16, warps 4x2, 3 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_B, 128, 64, 16, 4, 2, 3, 2)
}  // namespace br
