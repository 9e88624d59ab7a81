// DMMA GEMM tile configuration A: 128x64, BK=16, warps 4x1, 3 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_A, 128, 64, 16, 4, 1, 3, 2)
}  // namespace br
