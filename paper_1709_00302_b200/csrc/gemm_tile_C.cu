// DMMA GEMM tile configuration C: 64x128, BK=16, warps 2x4, 3 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_C, 64, 128, 16, 2, 4, 3, 2)
}  // namespace br
