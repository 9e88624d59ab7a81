// DMMA GEMM tile configuration K: 64x128, BK=32, warps 2x2 (warp 32x64), 2 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_K, 64, 128, 32, 2, 2, 2, 2)
}  // namespace br
