// DMMA GEMM tile configuration MS: 32x128, BK=16, warps 1x4, 4 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_MS, 32, 128, 16, 1, 4, 4, 2)
}  // namespace br
