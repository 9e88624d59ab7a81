// Block-cyclic (GF_CYC) instantiations of the DMMA GEMM for the distributed
// SEVP's slab kernels (symm_cyclic / syr2k_cyclic in gemm.cu): the 64x128
// tile (config G) for the staircase products L Wown (A_N) and L^T W (A_T),
// and the square tiles of the SYR2K's LOWER epilogue (configs J and L).
// Kept out of the per-config units so the hot-path kernels compile without
// the map.
#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {

int launch_tile_cyc(int cfg, int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid) {
  if (epi == EPI_LOWER) {
    if (am != A_N || bmd != B_T) return set_error("cyclic LOWER needs A_N, B_T"), -1;
    if (cfg == CFG_J) return launch<64, 64, 32, 2, 2, 2, 3, A_N, B_T, EPI_LOWER, GF_CYC>(st, g, grid);
    if (cfg == CFG_L) return launch<128, 128, 16, 4, 2, 3, 1, A_N, B_T, EPI_LOWER, GF_CYC>(st, g, grid);
    return set_error("cyclic LOWER: tile config %d not instantiated", cfg), -1;
  }
  if (cfg != CFG_G || bmd != B_N || (am != A_N && am != A_T))
    return set_error("cyclic GEMM: config %d / modes %d %d not instantiated", cfg, am, bmd), -1;
  if (am == A_N) {
    if (epi == EPI_GEN) return launch<64, 128, 16, 2, 2, 3, 2, A_N, B_N, EPI_GEN, GF_CYC>(st, g, grid);
    return launch<64, 128, 16, 2, 2, 3, 2, A_N, B_N, EPI_SPLIT, GF_CYC>(st, g, grid);
  }
  if (epi == EPI_GEN) return launch<64, 128, 16, 2, 2, 3, 2, A_T, B_N, EPI_GEN, GF_CYC>(st, g, grid);
  return launch<64, 128, 16, 2, 2, 3, 2, A_T, B_N, EPI_SPLIT, GF_CYC>(st, g, grid);
}

}  // namespace br
