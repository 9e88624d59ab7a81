// DMMA GEMM tile configuration NS: 128x32, BK=16, warps 4x1, 4 stages.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {
BR_DEFINE_TILE(launch_tile_NS, 128, 32, 16, 4, 1, 4, 2)
}  // namespace br
