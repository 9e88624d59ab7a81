// DMMA GEMM tile configuration G: 64x128, BK=16, warps 2x2 (warp 32x64), 3 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_G, 64, 128, 16, 2, 2, 3, 2)
}  // namespace br
