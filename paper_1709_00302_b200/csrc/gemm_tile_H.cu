// DMMA GEMM tile configuration H: 128x64, BK=16, warps 2x2 (warp 64x32), 3 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_H, 128, 64, 16, 2, 2, 3, 2)
}  // namespace br
