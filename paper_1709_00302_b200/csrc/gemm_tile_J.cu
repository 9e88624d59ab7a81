// DMMA GEMM tile configuration J: 64x64, BK=32, warps 2x2, 2 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_J, 64, 64, 32, 2, 2, 2, 3)
}  // namespace br
