// The SEVP X products in one persistent launch (ref sevp.py:156-176,
// kernels.py:312-341):
//     X1 = sym(A2) W,   X2 = X1^T W / 2,   X3 = X1 + Y X2.
// On the narrow-panel configurations (b <= 64: c1) these three products are
// a chain of small launches on the critical path of every iteration (SYMM
// split-K + its reduction, X2 split-K + its reduction, X3): about 40 us of
// serialized kernels per iteration against a 54 us panel. Here one grid
// (every CTA resident: num_sms x CTAs/SM of the tile configuration) runs
//   1. the SYMM's split-K tiles (the DMMA tile of gemm_kernel.cuh, A_SYM),
//   2. per CTA a block of rows: X1 rows = sum of the partials (fixed order),
//      and that block's partial X1_rows^T W_rows,
//   3. X2 = 1/2 sum of the block partials (fixed order), entries split over
//      the CTAs,
//   4. X3 rows = X1 rows + Y rows X2,
// with a self-resetting grid barrier between the phases (graph replay safe).
// Deterministic; the same kernel serves look-ahead depth 0 and 1, so they
// stay bitwise equal.
#include <algorithm>

#include "gemm_kernel.cuh"
#include "gemm_tiles.cuh"

namespace br {

struct XArgs {
  GemmArgs g;          // the SYMM (A_SYM, EPI_SPLIT into ws, S splits)
  int64_t j, b;
  int S, tiles_m, tiles_n;
  double* X1;
  int64_t ldx1;
  double* X2;
  int64_t ldx2;
  double* X3;
  int64_t ldx3;
  const double* W;
  int64_t ldw;
  const double* Y;
  int64_t ldy;
  double* part;        // [G][b][b] block partials of X1^T W
  unsigned* bar;       // [count, generation]
};

// All CTAs of the grid are resident (the grid is sized to the device), so a
// spin barrier is safe; the last arriver resets the count before releasing
// the others (self-resetting across launches and graph replays).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB>
__global__ void __launch_bounds__(WM* WN * 32, MINB) xchain_kernel(const XArgs x) {
  constexpr int NT = WM * WN * 32;
  extern __shared__ __align__(16) double smem[];
  const unsigned G = gridDim.x;
  const int tid = threadIdx.x;
  const int64_t j = x.j, b = x.b;
  pdl_wait();  // every CTA reads the predecessor's outputs (W, Y, A2)
  // ---- 1. SYMM split-K tiles ----
  const int nwork = x.tiles_m * x.tiles_n * x.S;
  for (int wi = blockIdx.x; wi < nwork; wi += G) {
    const int bx = wi % x.tiles_m, rest = wi / x.tiles_m;
    const int by = rest % x.tiles_n, bz = rest / x.tiles_n;
    dgemm_tile<BM, BN, BK, WM, WN, STAGES, MINB, A_SYM, B_N, EPI_SPLIT, GF_NOTRIG>(x.g, bx, by, bz);
    __syncthreads();  // shared memory reused by the next tile
  }
  grid_barrier(x.bar, G);
  // ---- 2. X1 rows of this block, and the block's X1^T W partial ----
  const int64_t R = cdiv(j, (int64_t)G);
  const int64_t r0 = (int64_t)blockIdx.x * R, r1 = min(j, r0 + R), nr = max((int64_t)0, r1 - r0);
  double* X1s = smem;            // [b][R]
  double* X2s = smem + b * R;    // [b][b]
  const int64_t tot = (int64_t)x.S * b * j;
  for (int64_t e = tid; e < nr * b; e += NT) {
    const int64_t r = r0 + e % nr, c = e / nr;
    const double* p = x.g.ws + c * j + r;
    double s = 0.0;
    for (int z = 0; z < x.S; ++z) s += p[(int64_t)z * b * j];
    X1s[c * R + (e % nr)] = s;
    x.X1[r + c * x.ldx1] = s;
  }
  (void)tot;
  __syncthreads();
  double* part = x.part + (int64_t)blockIdx.x * b * b;
  for (int64_t e = tid; e < b * b; e += NT) {
    const int64_t c1 = e % b, c2 = e / b;
    double s0 = 0.0, s1 = 0.0;
    int64_t q = 0;
    for (; q + 1 < nr; q += 2) {
      s0 = fma(X1s[c1 * R + q], x.W[(r0 + q) + c2 * x.ldw], s0);
      s1 = fma(X1s[c1 * R + q + 1], x.W[(r0 + q + 1) + c2 * x.ldw], s1);
    }
    if (q < nr) s0 = fma(X1s[c1 * R + q], x.W[(r0 + q) + c2 * x.ldw], s0);
    part[c1 + c2 * b] = s0 + s1;
  }
  grid_barrier(x.bar, G);
  // ---- 3. X2 = 1/2 sum of the block partials (entries split over CTAs) ----
  const int64_t E = cdiv(b * b, (int64_t)G);
  for (int64_t e = (int64_t)blockIdx.x * E + tid; e < min(b * b, ((int64_t)blockIdx.x + 1) * E); e += NT) {
    double s = 0.0;
    for (unsigned q = 0; q < G; ++q) s += x.part[(int64_t)q * b * b + e];
    x.X2[(e % b) + (e / b) * x.ldx2] = 0.5 * s;
  }
  grid_barrier(x.bar, G);
  // ---- 4. X3 rows = X1 rows + Y rows X2 ----
  for (int64_t e = tid; e < b * b; e += NT) X2s[e] = __ldcg(&x.X2[(e % b) + (e / b) * x.ldx2]);
  __syncthreads();
  pdl_trigger();
  for (int64_t e = tid; e < nr * b; e += NT) {
    const int64_t q = e % nr, c = e / nr, r = r0 + q;
    double s0 = X1s[c * R + q], s1 = 0.0;
    int64_t k = 0;
    for (; k + 1 < b; k += 2) {
      s0 = fma(x.Y[r + k * x.ldy], X2s[k + c * b], s0);
      s1 = fma(x.Y[r + (k + 1) * x.ldy], X2s[k + 1 + c * b], s1);
    }
    if (k < b) s0 = fma(x.Y[r + k * x.ldy], X2s[k + c * b], s0);
    x.X3[r + c * x.ldx3] = s0 + s1;
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB>
static int launch_xchain(cudaStream_t st, XArgs x, int ctas_per_sm, int num_sms) {
  auto kern = xchain_kernel<BM, BN, BK, WM, WN, STAGES, MINB>;
  const int tile_smem = smem_bytes<BM, BN, BK, STAGES, A_SYM, B_N>();
  static std::atomic<int> attr_dev_mask{0};
  int dev = 0;
  BR_CUDA(cudaGetDevice(&dev));
  if (!(attr_dev_mask.load() & (1 << dev))) {
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_dev_mask.fetch_or(1 << dev);
  }
  int occ = 0;
  const int G0 = num_sms * ctas_per_sm;
  const int64_t R = cdiv(x.j, (int64_t)G0);
  const size_t smem = std::max<size_t>(tile_smem, (size_t)(x.b * R + x.b * x.b) * sizeof(double));
  BR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WM * WN * 32, smem));
  if (occ < 1) {
    set_error("xchain: no residency");
    return -1;
  }
  const int G = num_sms * std::min(occ, ctas_per_sm);
  // splits: about one wave of tiles
  const int64_t tiles = (int64_t)x.tiles_m * x.tiles_n;
  const int64_t nkt = cdiv(x.g.K, BK);
  int64_t S = std::max<int64_t>(1, std::min<int64_t>(G / std::max<int64_t>(tiles, 1), nkt / 2));
  const int64_t kps = cdiv(nkt, S) * BK;
  S = cdiv(x.g.K, kps);
  x.S = (int)S;
  x.g.k_per_split = kps;
  const size_t smem2 = std::max<size_t>(tile_smem, (size_t)(x.b * cdiv(x.j, (int64_t)G) + x.b * x.b) * sizeof(double));
  if (g_preload_only) return 0;
  count_launch();
  BR_CUDA(launch_pdl(kern, dim3(G), dim3(WM * WN * 32), smem2, st, x));
  return 0;
}

int xchain(cudaStream_t st, Scratch& ws, MatView X1, MatView X2, MatView X3, MatView A2, MatView W,
           MatView Y, unsigned* bar) {
  const int64_t j = A2.rows, b = W.cols;
  if (b > 64 || b < 1 || j < 1 || !bar || A2.trans || W.trans || Y.trans || X1.trans || X2.trans ||
      X3.trans)
    return 1;
  const int cfg = b <= 32 ? CFG_NS : CFG_D;
  const int bm = kTiles[cfg].bm, bn = kTiles[cfg].bn, cps = kTiles[cfg].ctas_per_sm;
  const int G = ws.num_sms * cps;
  // workspace: S partials (S <= G) of j x b, plus G b x b block partials
  const int64_t tiles = cdiv(j, bm) * cdiv(b, bn);
  const int64_t smax = std::max<int64_t>(1, G / std::max<int64_t>(tiles, 1));
  if (smax * j * b + (int64_t)G * b * b > ws.cap) return 1;
  XArgs x{};
  GemmArgs& g = x.g;
  g.M = j;
  g.N = b;
  g.K = j;
  g.A = A2.p;
  g.lda = A2.ld;
  g.A2 = A2.p;
  g.lda2 = A2.ld;
  g.ksplitA = INT64_MAX;
  g.B = W.p;
  g.ldb = W.ld;
  g.B2 = W.p;
  g.ldb2 = W.ld;
  g.ksplitB = INT64_MAX;
  g.alpha = 1.0;
  g.beta = 0.0;
  g.vecA = (reinterpret_cast<uintptr_t>(A2.p) % 16 == 0) && (A2.ld % 2 == 0);
  g.vecB = (reinterpret_cast<uintptr_t>(W.p) % 16 == 0) && (W.ld % 2 == 0);
  g.ws = ws.p;
  x.j = j;
  x.b = b;
  x.tiles_m = (int)cdiv(j, bm);
  x.tiles_n = (int)cdiv(b, bn);
  x.X1 = X1.p;
  x.ldx1 = X1.ld;
  x.X2 = X2.p;
  x.ldx2 = X2.ld;
  x.X3 = X3.p;
  x.ldx3 = X3.ld;
  x.W = W.p;
  x.ldw = W.ld;
  x.Y = Y.p;
  x.ldy = Y.ld;
  x.part = ws.p + smax * j * b;
  x.bar = bar;
  if (cfg == CFG_NS) return launch_xchain<128, 32, 16, 4, 1, 4, 2>(st, x, cps, ws.num_sms);
  return launch_xchain<64, 64, 16, 2, 2, 4, 3>(st, x, cps, ws.num_sms);
}

int preload_xchain_kernels() {
  cudaFuncAttributes fa;
  BR_CUDA(cudaFuncGetAttributes(&fa, xchain_kernel<128, 32, 16, 4, 1, 4, 2>));
  BR_CUDA(cudaFuncGetAttributes(&fa, xchain_kernel<64, 64, 16, 2, 2, 4, 3>));
  return 0;
}

}  // namespace br
