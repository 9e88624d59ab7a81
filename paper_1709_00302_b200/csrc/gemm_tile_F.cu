// DMMA GEMM tile configuration F: 128x64, BK=32, warps 4x2, 2 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_F, 128, 64, 32, 4, 2, 2, 2)
}  // namespace br
