// Tile configurations of the DMMA GEMM and their launchers (one translation
// unit per configuration so they compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include "gemm.cuh"

namespace br {

enum TileCfg { CFG_L = 0, CFG_NS, CFG_MS, CFG_A, CFG_B, CFG_C, CFG_D, CFG_E, CFG_F, CFG_G, CFG_H,
               CFG_J, CFG_K, CFG_COUNT };

struct TileInfo {
  const char* name;
  int bm, bn;
  int ctas_per_sm;  // resident CTAs per SM (registers / shared memory)
};

//                 name   BM   BN  CTAs/SM
constexpr TileInfo kTiles[CFG_COUNT] = {
    {"L", 128, 128, 1},  // 8 warps 4x2, warp 32x64, 3 stages
    {"NS", 128, 32, 2},  // 4 warps 4x1, warp 32x32, 4 stages (N <= 32)
    {"MS", 32, 128, 2},  // 4 warps 1x4, warp 32x32, 4 stages (M <= 32)
    {"A", 128, 64, 2},   // 4 warps 4x1, warp 32x64, 3 stages
    {"B", 128, 64, 2},   // 8 warps 4x2, warp 32x32, 3 stages
    {"C", 64, 128, 2},   // 8 warps 2x4, warp 32x32, 3 stages
    {"D", 64, 64, 3},    // 4 warps 2x2, warp 32x32, 4 stages
    {"E", 64, 128, 2},   // 8 warps 2x4, warp 32x32, BK=32, 2 stages
    {"F", 128, 64, 2},   // 8 warps 4x2, warp 32x32, BK=32, 2 stages
    {"G", 64, 128, 2},   // 4 warps 2x2, warp 32x64, 3 stages
    {"H", 128, 64, 2},   // 4 warps 2x2, warp 64x32, 3 stages
    {"J", 64, 64, 3},    // 4 warps 2x2, warp 32x32, BK=32, 2 stages
    {"K", 64, 128, 2},   // 4 warps 2x2, warp 32x64, BK=32, 2 stages
};
// K depth of one pipeline stage per configuration (split-K granularity)
constexpr int kTileBK[CFG_COUNT] = {16, 16, 16, 16, 16, 16, 16, 32, 32, 16, 16, 32, 32};

int launch_tile_L(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_NS(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_MS(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_A(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_B(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_C(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_D(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_E(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_F(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_G(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_H(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_J(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
int launch_tile_K(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);
// block-cyclic (GF_CYC) instantiations: config G (A_N / A_T, B_N, GEN /
// SPLIT) and the LOWER epilogue on configs J / L (gemm_tile_CYC.cu)
int launch_tile_cyc(int cfg, int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid);

inline int launch_tile(int cfg, int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g,
                       dim3 grid) {
  switch (cfg) {
    case CFG_L: return launch_tile_L(am, bmd, epi, st, g, grid);
    case CFG_NS: return launch_tile_NS(am, bmd, epi, st, g, grid);
    case CFG_MS: return launch_tile_MS(am, bmd, epi, st, g, grid);
    case CFG_A: return launch_tile_A(am, bmd, epi, st, g, grid);
    case CFG_B: return launch_tile_B(am, bmd, epi, st, g, grid);
    case CFG_C: return launch_tile_C(am, bmd, epi, st, g, grid);
    case CFG_D: return launch_tile_D(am, bmd, epi, st, g, grid);
    case CFG_E: return launch_tile_E(am, bmd, epi, st, g, grid);
    case CFG_F: return launch_tile_F(am, bmd, epi, st, g, grid);
    case CFG_G: return launch_tile_G(am, bmd, epi, st, g, grid);
    case CFG_H: return launch_tile_H(am, bmd, epi, st, g, grid);
    case CFG_J: return launch_tile_J(am, bmd, epi, st, g, grid);
    default: return launch_tile_K(am, bmd, epi, st, g, grid);
  }
}

}  // namespace br
