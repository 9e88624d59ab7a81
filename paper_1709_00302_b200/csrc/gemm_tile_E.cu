// DMMA GEMM tile configuration E: 64x128, BK=32, warps 2x4, 2 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_E, 64, 128, 32, 2, 4, 2, 2)
}  // namespace br
