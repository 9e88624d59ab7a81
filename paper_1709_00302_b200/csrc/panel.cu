// Householder panel factorization (QR, and LQ through a transposed view).
//
// Reference semantics (ref kernels.py:86-110, 152-208, 211-255):
//   * reflector per column with beta = -sign(x0)*||x||, x0 == 0 counted as
//     positive, applied even when the tail is zero (tau = 2); the zero
//     column gives tau = beta = 0 and v = e_i (identity, no update);
//   * compact WY with Q = H_0 ... H_{b-1} = I + W Y^T, W = Y T, T = -T_larft.
//
// B200 design. A "leaf" is an L x nb (nb <= 32) block held in the REGISTERS
// of one thread-block cluster (<= 16 CTAs; each thread owns R rows x NB
// columns, R*NB = 64 doubles). Each column step needs exactly one
// cluster-wide reduction of an NB-slot vector (see leaf_reg_kernel), one
// barrier.cluster, and a rank-1 update of the owned rows:
//     v^T P_c = (x^T P_c - beta P_ic) / (x0 - beta)
// so the Householder coefficient of column c is simply
//     alpha_c = tau v^T P_c = P_ic - (x^T P_c) / beta.
// Every CTA sums the C partial vectors in the same fixed order, so all CTAs
// hold bit-identical scalars. T follows the reference recurrence from Gram
// columns folded into the same reductions; W = Y T is formed on chip.
// Panels wider than the leaf are processed right-looking: leaf, then the
// block reflector of that leaf is applied to the rest of the panel with
// DMMA GEMMs, and the full T is assembled from the Gram matrix.
#include <algorithm>
#include <cstdlib>
#include <functional>

#include <cuda.h>

#include "driver.cuh"
#include "gemm.cuh"

namespace br {

constexpr int LEAF_NB = 64;    // max leaf width (64 only for the 2D-layout leaf)
constexpr int LEAF_MAXC = 16;  // max cluster size (non-portable)
static long long* g_leaf_prof = nullptr;  // BR_LEAF_PROF phase counters

struct LeafArgs {
  MatView P;  // L x nb leaf (a transposed view gives the LQ rows)
  double* Y;
  int64_t ldy;
  double* tau;
  double* T;  // nb x nb (may be null)
  int64_t ldt;
  double* W;  // L x nb (may be null)
  int64_t ldw;
  int64_t L;
  int nb;
  int wt;           // W output: 0 -> Y T, 1 -> Y T^T (block reflector Q^T = I + Y T^T Y^T)
  long long* prof;  // optional per-phase cycle counters (BR_LEAF_PROF=1)
  // persistent mode: nleaves leaves of width lw over a btot-wide panel P
  int nleaves, lw, btot;
  unsigned* flags;  // [0, 64): leaf done, [64, 128): next leaf's columns ready
  unsigned epoch;
};

}  // namespace br
#include "panel_leaf.cuh"   // leaf_reg_kernel<NB, R, LT>
#include "panel_leaf2.cuh"  // leaf2_kernel<NB, NW>
namespace br {

// Rows one cluster holds at leaf width nb: 16 CTAs x 256 threads x R rows
// with R * NB = 64 register doubles per thread. The 4- and 2-wide leaves
// exist for panels taller than 32768 rows (SEVP n > 32768 + w, SVD m > 32768:
// 65536 / 131072 rows per cluster; an n = 131072 fp64 matrix is 137 GB).
static int leaf_rows_per_thread(int nb) {
  return nb > 32 ? 1 : (nb > 16 ? 2 : (nb > 8 ? 4 : (nb > 4 ? 8 : (nb > 2 ? 16 : 32))));
}
// 64-wide leaves (8 column-group warps, <= 4096 rows): opt-in with
// BR_LEAF64=1. Measured slower than two 32-wide leaves plus their block update
// (4096 x 256 panel 760 vs 686 us): two warps per SM sub-partition lengthen
// every column step more than the saved launches and epilogues win back.
static bool leaf64_enabled() {
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("BR_LEAF64");
    const char* l2 = std::getenv("BR_LEAF2");
    m = (e && std::atoi(e) == 1 && !(l2 && std::atoi(l2) == 0)) ? 1 : 0;
  }
  return m == 1;
}
// Threads per leaf CTA at most (BR_LEAF_LT=128: half-SM CTAs only; tuning aid).
static int leaf_max_lt() {
  static int lt = 0;
  if (!lt) {
    const char* e = std::getenv("BR_LEAF_LT");
    lt = (e && std::atoi(e) == 128) ? 128 : 256;
  }
  return lt;
}
static int64_t leaf_capacity(int nb) {
  return (int64_t)LEAF_MAXC * leaf_max_lt() * leaf_rows_per_thread(nb);
}

// Leaf width for a j x b panel: the widest of {32, 16, 8} (or b if narrower)
// whose L rows fit one cluster.
static int leaf_width(int64_t L, int64_t b) {
  const int cand[6] = {64, 32, 16, 8, 4, 2};
  for (int nb : cand) {
    if (nb == 64 && (b <= 32 || !leaf64_enabled())) continue;
    const int use = (int)std::min<int64_t>(nb, b);
    if (L <= leaf_capacity(use)) return use;
  }
  return -1;
}

template <int NB, int R, int LT>
static int launch_leaf_t(cudaStream_t st, const LeafArgs& a) {
  auto kern = leaf_reg_kernel<NB, R, LT>;
  constexpr int ROWS = LT * R;
  int C = 1;
  while (C < cdiv(a.L, ROWS)) C *= 2;
  const size_t smem = (size_t)NB * ROWS * sizeof(double);
  static std::atomic<int> attr_dev_mask{0};
  int dev = 0;
  BR_CUDA(cudaGetDevice(&dev));
  if (!(attr_dev_mask.load() & (1 << dev))) {
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_dev_mask.fetch_or(1 << dev);
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[3];
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(LT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  at[2].id = cudaLaunchAttributePriority;
  at[2].val.priority = stream_priority(st);
  cfg.attrs = at;
  cfg.numAttrs = 3;
  if (g_preload_only) {
    cudaFuncAttributes fa;
    BR_CUDA(cudaFuncGetAttributes(&fa, kern));
    return 0;
  }
  count_launch();
  BR_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return 0;
}

static bool leaf_pow2() {
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("BR_LEAF_POW2");
    m = (e && std::atoi(e) == 1) ? 1 : 0;
  }
  return m == 1;
}

// 2D-layout leaf (leaf2_kernel): NW warps of 8 columns x 32 RPT rows each.
template <int NB, int NW, int RPT = 8, bool PAIR = false>
static int launch_leaf2_t(cudaStream_t st, const LeafArgs& a) {
  auto kern = leaf2_kernel<NB, NW, RPT, PAIR>;
  constexpr int ROWS = (NW / (NB / 8)) * 32 * RPT;
  // as many CTAs as the rows need (the 2D leaf's source sums take any
  // count): fewer pushes and sources per column step than a power-of-two
  // cluster (1100 x 32 58.7 -> 54.9 us, 5000 x 32 80.7 -> 75.3; c1 5.29 ->
  // 5.15 ms, c2 8.12 -> 7.88, c3 46.75 -> 46.09, c4 444.2 -> 441.1).
  // BR_LEAF_POW2=1 rounds the cluster up to a power of two (A/B aid).
  int C = (int)cdiv(a.L, ROWS);
  if (leaf_pow2()) {
    C = 1;
    while (C < cdiv(a.L, ROWS)) C *= 2;
  }
  const size_t smem = ((size_t)NB * (ROWS + 8) + 2 * (size_t)NB * (NB + 1)) * sizeof(double);
  static std::atomic<int> attr_dev_mask{0};
  int dev = 0;
  BR_CUDA(cudaGetDevice(&dev));
  if (!(attr_dev_mask.load() & (1 << dev))) {
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_dev_mask.fetch_or(1 << dev);
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[3];
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(NW * 32 + ((PAIR && NW <= 4) ? 32 : 0));  // + the T warp
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  at[2].id = cudaLaunchAttributePriority;
  at[2].val.priority = stream_priority(st);
  cfg.attrs = at;
  cfg.numAttrs = 3;
  if (g_preload_only) {
    cudaFuncAttributes fa;
    BR_CUDA(cudaFuncGetAttributes(&fa, kern));
    return 0;
  }
  count_launch();
  BR_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return 0;
}

// BR_LEAF2=0 selects the 1D-layout leaf_reg_kernel everywhere (A/B aid);
// BR_LEAF2_WIDE=1 prefers 8-warp CTAs (fewer CTAs per cluster).
static int leaf2_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("BR_LEAF2");
    const char* w = std::getenv("BR_LEAF2_WIDE");
    m = (e && std::atoi(e) == 0) ? 0 : ((w && std::atoi(w) == 1) ? 2 : 1);
  }
  return m;
}

// Rows per thread of the 2D leaf. Default (44): leaves of 257..2048 rows
// run 4 rows x 8 columns per thread with the same 1 warp per SM
// sub-partition and twice the CTAs of the 8-row layout (half the partial
// sums and update per column step; the cluster exchange exists either way):
// 2016 x 32 60.8 -> 57.6 us, 1024 x 32 59.3 -> 54.4, 2048 x 16 38.6 -> 35.0;
// c1 5.36 -> 5.26 ms, c2 8.96 -> 8.44 ms. At <= 256 rows the 8-row layout
// keeps the leaf in one CTA (no exchange) and stays. BR_LEAF_RPT=8: the
// 8-row layout everywhere; BR_LEAF_RPT=4: 4 rows per thread with twice the
// warps over the same rows (measured slower everywhere).
static int leaf_rpt() {
  static int r = -1;
  if (r < 0) {
    const char* e = std::getenv("BR_LEAF_RPT");
    r = e ? std::atoi(e) : 44;
    if (r != 4 && r != 8) r = 44;
  }
  return r;
}

// Pair steps (two columns per cluster exchange, leaf2_kernel<..., PAIR = true>)
// for every leaf that has an exchange; BR_LEAF_PAIR=0: one column per
// exchange everywhere (A/B aid).
static bool leaf_pair() {
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("BR_LEAF_PAIR");
    m = (e && std::atoi(e) == 0) ? 0 : 1;
  }
  return m == 1;
}

// Launch the 2D-layout leaf when it covers (nb, L) (sets *done).
static int launch_leaf2(cudaStream_t st, const LeafArgs& a, bool* done) {
  const int mode = leaf2_mode();
  *done = true;
  if (mode == 0 || a.nleaves != 1) return *done = false, 0;
  const int64_t L = a.L;
  const bool wide = mode == 2;
  if (leaf_pair() && mode == 1 && leaf_rpt() == 44 && a.nb > 1) {
    if (L <= 256) {  // one CTA, no exchange: single steps, T on the T warp
      if (a.nb > 16 && a.nb <= 32) return launch_leaf2_t<32, 4, 8, true>(st, a);
      if (a.nb > 8 && a.nb <= 16) return launch_leaf2_t<16, 2, 8, true>(st, a);
    }
    if (L > 256 && L <= (int64_t)LEAF_MAXC * 128) {
      if (a.nb > 16 && a.nb <= 32) return launch_leaf2_t<32, 4, 4, true>(st, a);
      if (a.nb > 8 && a.nb <= 16) return launch_leaf2_t<16, 2, 4, true>(st, a);
    }
    if (a.nb > 16 && a.nb <= 32 && L > 256) {
      if (L <= (int64_t)LEAF_MAXC * 256) return launch_leaf2_t<32, 4, 8, true>(st, a);
      if (L <= (int64_t)LEAF_MAXC * 512) return launch_leaf2_t<32, 8, 8, true>(st, a);
    }
    if (a.nb <= 16 && L > 256 && !(a.nb <= 8 && L > (int64_t)LEAF_MAXC * 1024)) {
      if (L <= (int64_t)LEAF_MAXC * 512) return launch_leaf2_t<16, 4, 8, true>(st, a);
      if (L <= (int64_t)LEAF_MAXC * 1024) return launch_leaf2_t<16, 8, 8, true>(st, a);
    }
  }
  if (leaf_rpt() == 44 && !wide && L > 256 && L <= (int64_t)LEAF_MAXC * 128) {
    if (a.nb > 16 && a.nb <= 32) return launch_leaf2_t<32, 4, 4>(st, a);
    if (a.nb > 8 && a.nb <= 16) return launch_leaf2_t<16, 2, 4>(st, a);
  }
  if (leaf_rpt() == 4 && !wide) {
    if (a.nb > 16 && a.nb <= 32) {
      if (L <= (int64_t)LEAF_MAXC * 256) return launch_leaf2_t<32, 8, 4>(st, a);
      if (L <= (int64_t)LEAF_MAXC * 512) return launch_leaf2_t<32, 16, 4>(st, a);
    } else if (a.nb > 8 && a.nb <= 16) {
      if (L <= 256) return launch_leaf2_t<16, 4, 4>(st, a);
      if (L <= (int64_t)LEAF_MAXC * 512) return launch_leaf2_t<16, 8, 4>(st, a);
    }
  }
  if (a.nb > 32) {
    if (a.nb <= 64 && L <= (int64_t)LEAF_MAXC * 256) return launch_leaf2_t<64, 8>(st, a);
    return *done = false, 0;
  }
  if (a.nb > 16) {
    if (!wide && L <= (int64_t)LEAF_MAXC * 256) return launch_leaf2_t<32, 4>(st, a);
    if (L <= (int64_t)LEAF_MAXC * 512) return launch_leaf2_t<32, 8>(st, a);
    return *done = false, 0;
  }
  if (a.nb <= 8 && L > (int64_t)LEAF_MAXC * 1024) {
    // 8-wide leaves of the tallest panels (c5): 16 x 2048-row CTAs, 8 row groups
    if (L <= (int64_t)LEAF_MAXC * 2048) return launch_leaf2_t<8, 8>(st, a);
    return *done = false, 0;
  }
  if (L <= 256) return launch_leaf2_t<16, 2>(st, a);
  if (!wide && L <= (int64_t)LEAF_MAXC * 512) return launch_leaf2_t<16, 4>(st, a);
  // 16 x 1024-row CTAs (4 row groups, combined in shared memory before the
  // cluster exchange): 16384 x 16 51.9 us vs 53-57 us for the 1D layout
  if (L <= (int64_t)LEAF_MAXC * 1024) return launch_leaf2_t<16, 8>(st, a);
  return *done = false, 0;
}

static int launch_leaf(cudaStream_t st, MatView P, MatView Y, double* tau, double* T, int64_t ldt,
                       MatView* W, int wt = 0, int nleaves = 1, int lw = 0,
                       unsigned* flags = nullptr, unsigned epoch = 0) {
  const int64_t L = P.rows;
  const int nb = nleaves > 1 ? lw : (int)P.cols;
  if (nb < 1 || nb > LEAF_NB || L > leaf_capacity(nb)) {
    set_error("panel leaf %lld x %d does not fit one cluster", (long long)L, nb);
    return -1;
  }
  LeafArgs a;
  a.P = P;
  a.Y = Y.p;
  a.ldy = Y.ld;
  a.tau = tau;
  a.T = T;
  a.ldt = ldt;
  a.W = W ? W->p : nullptr;
  a.ldw = W ? W->ld : 0;
  a.L = L;
  a.nb = nb;
  a.wt = wt;
  a.prof = nullptr;
  a.nleaves = nleaves;
  a.lw = nb;
  a.btot = (int)P.cols;
  a.flags = flags;
  a.epoch = epoch;
  static const bool prof_on = std::getenv("BR_LEAF_PROF") != nullptr;
  if (prof_on) {
    if (!g_leaf_prof) {
      BR_CUDA(cudaMalloc(&g_leaf_prof, 16 * sizeof(long long)));
      BR_CUDA(cudaMemset(g_leaf_prof, 0, 16 * sizeof(long long)));
    }
    a.prof = g_leaf_prof;
  }
  {
    bool done = false;
    const int r = launch_leaf2(st, a, &done);
    if (done || r != 0) return r;
  }
  // 128-thread CTAs (one warp per SM sub-partition: the per-step reduction is
  // issue-bound per warp) while one cluster of them holds the leaf; 256
  // threads for the tallest leaves.
  if (nb > 16) {
    if (L <= (int64_t)LEAF_MAXC * 128 * 2) return launch_leaf_t<32, 2, 128>(st, a);
    return launch_leaf_t<32, 2, 256>(st, a);
  }
  if (nb > 8) {
    if (L <= (int64_t)LEAF_MAXC * 128 * 4) return launch_leaf_t<16, 4, 128>(st, a);
    return launch_leaf_t<16, 4, 256>(st, a);
  }
  if (nb > 4 || L <= (int64_t)LEAF_MAXC * 256 * 8) {
    if (L <= (int64_t)LEAF_MAXC * 128 * 8) return launch_leaf_t<8, 8, 128>(st, a);
    return launch_leaf_t<8, 8, 256>(st, a);
  }
  // panels taller than 32768 rows: narrower leaves, more rows per thread (the
  // W epilogue of these leaves is not formed in the kernel: panel_qr builds W)
  if (a.W) {
    set_error("narrow leaf (nb = %d) cannot form W", nb);
    return -1;
  }
  if (nb > 2) return launch_leaf_t<4, 16, 256>(st, a);
  return launch_leaf_t<2, 32, 256>(st, a);
}

}  // namespace br

// Can `st` (a stream of the 16-SM green context) place the leaf clusters a
// confined panel launches? The partition is asked for with the
// max-potential-cluster-size split, but boards differ in their GPC layout: the
// strict split is only enabled when every tall-panel leaf shape fits.
namespace br {
template <class K>
static bool cluster_fits(K kern, int threads, size_t smem, cudaStream_t st) {
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(LEAF_MAXC);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = LEAF_MAXC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  const bool ok = cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n >= 1;
  cudaGetLastError();
  return ok;
}
template <int NB, int NW, int RPT, bool PAIR>
static bool leaf2_fits(cudaStream_t st) {
  constexpr int ROWS = (NW / (NB / 8)) * 32 * RPT;
  const size_t smem = ((size_t)NB * (ROWS + 8) + 2 * (size_t)NB * (NB + 1)) * sizeof(double);
  return cluster_fits(leaf2_kernel<NB, NW, RPT, PAIR>, NW * 32 + ((PAIR && NW <= 4) ? 32 : 0), smem, st);
}
bool panel_clusters_fit(cudaStream_t st) {
  return leaf2_fits<16, 8, 8, true>(st) && leaf2_fits<32, 8, 8, true>(st) && leaf2_fits<16, 4, 8, true>(st) &&
         leaf2_fits<8, 8, 8, false>(st) &&
         cluster_fits(leaf_reg_kernel<4, 16, 256>, 256, (size_t)4 * 256 * 16 * sizeof(double), st) &&
         cluster_fits(leaf_reg_kernel<2, 32, 256>, 256, (size_t)2 * 256 * 32 * sizeof(double), st);
}
}  // namespace br

// Print and reset the leaf phase counters (collected when BR_LEAF_PROF is set;
// development aid, not part of include/bandred_b200.h).
extern "C" int br_leaf_prof_dump() {
  if (!br::g_leaf_prof) return 0;
  long long h[16];
  if (cudaMemcpy(h, br::g_leaf_prof, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  const double st = h[11] ? (double)h[11] : 1.0, nl = h[12] ? (double)h[12] : 1.0;
  printf("leaf phases (cycles/step over %lld steps): reduce %.0f sync1 %.0f push %.0f cbar %.0f "
         "scalars %.0f sync2 %.0f update %.0f | per leaf (%lld): prologue %.0f tail %.0f "
         "cbar-exit+Y/R (2D: tau+sync) %.0f W %.0f | 2D: store_y %.0f T %.0f\n",
         h[11], h[0] / st, h[1] / st, h[2] / st, h[3] / st, h[4] / st, h[5] / st, h[6] / st,
         h[12], h[7] / nl, h[8] / nl, h[9] / nl, h[10] / nl, h[13] / nl, h[14] / nl);
  cudaMemset(br::g_leaf_prof, 0, sizeof(h));
  return 0;
}

namespace br {

// T (b x b, upper triangular, T = -T_larft) from the Gram matrix G = Y^T Y and
// tau, by the reference recurrence T[r][i] = -tau_i sum_{c<i} T[r][c] G[c][i]
// (ref kernels.py:152-162), blocked by 32 columns:
//   T[q, e] = T[q, q:e] G[q:e, e] T_ee            (block rows q < e),
// the blocked form of the same recurrence. CTA q owns row block q of T, so a
// CTA only ever reads its own earlier results: its warps first form the
// diagonal blocks T_ee (e >= q) in parallel (lane r = row r, registers),
// then it walks the later block columns e in order. One launch replaces the
// diagonal kernel and the 2 (nblk-1) small GEMMs of the GEMM formulation.
constexpr int TAB = 32;      // block size
constexpr int TAB_MAXB = 256;  // widest panel handled (smem: row block + diagonal blocks + G stage)
static size_t t_assemble_smem(int b) {
  const int nblk = (b + TAB - 1) / TAB;
  return sizeof(double) * ((size_t)TAB * (b + 1) + (size_t)nblk * TAB * (TAB + 1) + (size_t)b * TAB +
                           TAB * (TAB + 1));
}

// diag_given: the diagonal blocks T_ee are already in T (written by the
// leaves, which form them from the same reflectors); otherwise the CTA forms
// them from G first. G is the symmetric Gram matrix: the G[q-rows, e-cols]
// stage is read as G[e-rows, q-cols] so that consecutive threads read
// consecutive addresses.
__global__ void __launch_bounds__(256) t_assemble_kernel(const double* __restrict__ G, int64_t ldg,
                                                         const double* __restrict__ tau, int b,
                                                         double* __restrict__ T, int64_t ldt,
                                                         int diag_given) {
  extern __shared__ double sm[];
  pdl_wait();
  pdl_trigger();
  const int nblk = (b + TAB - 1) / TAB;
  const int q = blockIdx.x, q0 = q * TAB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int LDR = b + 1;                   // padded row stride of Trow
  double* Trow = sm;                       // [TAB][b + 1]  row block q of T
  double* Td = Trow + TAB * LDR;           // [nblk][TAB][TAB+1] diagonal blocks
  double* Gs = Td + nblk * TAB * (TAB + 1);  // [b][TAB]  G[q0:e0, e-block]
  double* Xs = Gs + b * TAB;               // [TAB][TAB+1]
  for (int i = tid; i < TAB * LDR; i += 256) Trow[i] = 0.0;
  for (int e = q; e < nblk; ++e) {
    const int e0 = e * TAB;
    for (int i = tid; i < TAB * TAB; i += 256) {
      const int r = i % TAB, c = i / TAB;
      const bool ok = e0 + r < b && e0 + c < b;
      Td[(e * TAB + r) * (TAB + 1) + c] =
          !ok ? 0.0 : (diag_given ? T[(e0 + r) + (int64_t)(e0 + c) * ldt] : G[(e0 + r) + (int64_t)(e0 + c) * ldg]);
    }
  }
  __syncthreads();
  if (!diag_given) {
    for (int e = q + warp; e < nblk; e += 8) {  // T_ee: lane r = row r
      const int e0 = e * TAB, r = lane;
      double* D = Td + e * TAB * (TAB + 1);
      double tr[TAB];
#pragma unroll
      for (int c = 0; c < TAB; ++c) tr[c] = (c == r && e0 + r < b) ? -tau[e0 + r] : 0.0;
#pragma unroll
      for (int i = 1; i < TAB; ++i) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int c = 0; c + 1 < i; c += 2) {
          s0 = fma(tr[c], D[c * (TAB + 1) + i], s0);
          s1 = fma(tr[c + 1], D[(c + 1) * (TAB + 1) + i], s1);
        }
        if (i & 1) s0 = fma(tr[i - 1], D[(i - 1) * (TAB + 1) + i], s0);
        if (i > r && e0 + i < b) tr[i] = -tau[e0 + i] * (s0 + s1);
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < TAB; ++c) D[r * (TAB + 1) + c] = tr[c];
    }
    __syncthreads();
  }
  for (int i = tid; i < TAB * TAB; i += 256) {
    const int r = i / TAB, c = i % TAB;
    if (q0 + c < b) Trow[r * LDR + q0 + c] = Td[(q * TAB + r) * (TAB + 1) + c];
  }
  __syncthreads();
  const int cc = tid % TAB, r0 = (tid / TAB) * 4;  // 4 rows x 1 column per thread
  for (int e = q + 1; e < nblk; ++e) {
    const int e0 = e * TAB, kk = e0 - q0;  // K range [q0, e0)
    for (int i = tid; i < kk * TAB; i += 256) {
      const int c = i % TAB, k = i / TAB;  // G[q0 + k][e0 + c] == G[e0 + c][q0 + k]
      Gs[k * TAB + c] = (e0 + c < b) ? G[(e0 + c) + (int64_t)(q0 + k) * ldg] : 0.0;
    }
    __syncthreads();
    double x[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int k = 0; k < kk; k += 2) {  // kk is a multiple of TAB
      const double g0 = Gs[k * TAB + cc], g1 = Gs[(k + 1) * TAB + cc];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u][0] = fma(Trow[(r0 + u) * LDR + q0 + k], g0, x[u][0]);
        x[u][1] = fma(Trow[(r0 + u) * LDR + q0 + k + 1], g1, x[u][1]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) Xs[(r0 + u) * (TAB + 1) + cc] = x[u][0] + x[u][1];
    __syncthreads();
    const double* D = Td + e * TAB * (TAB + 1);
    double y[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 8
    for (int k = 0; k < TAB; k += 2) {
      const double d0 = D[k * (TAB + 1) + cc], d1 = D[(k + 1) * (TAB + 1) + cc];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        y[u][0] = fma(Xs[(r0 + u) * (TAB + 1) + k], d0, y[u][0]);
        y[u][1] = fma(Xs[(r0 + u) * (TAB + 1) + k + 1], d1, y[u][1]);
      }
    }
    if (e0 + cc < b) {
#pragma unroll
      for (int u = 0; u < 4; ++u) Trow[(r0 + u) * LDR + e0 + cc] = y[u][0] + y[u][1];
    }
    __syncthreads();
  }
  for (int i = tid; i < TAB * b; i += 256) {
    const int r = i % TAB, c = i / TAB;
    if (q0 + r < b) T[(q0 + r) + (int64_t)c * ldt] = Trow[r * LDR + c];
  }
}

int t_from_gram(cudaStream_t st, const double* G, int64_t ldg, const double* tau, int64_t b,
                double* T, int64_t ldt, bool diag_given) {
  if (b < 1 || b > TAB_MAXB) {
    set_error("t_from_gram: b = %lld outside [1, %d]", (long long)b, TAB_MAXB);
    return -1;
  }
  const int nblk = (int)cdiv(b, TAB);
  const size_t smem = t_assemble_smem((int)b);
  static std::atomic<int> attr_dev_mask{0};
  int dev = 0;
  BR_CUDA(cudaGetDevice(&dev));
  if (!(attr_dev_mask.load() & (1 << dev))) {
    BR_CUDA(cudaFuncSetAttribute(t_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)t_assemble_smem(TAB_MAXB)));
    attr_dev_mask.fetch_or(1 << dev);
  }
  count_launch();
  BR_CUDA(launch_pdl(t_assemble_kernel, dim3(nblk), dim3(256), smem, st, G, ldg, tau, (int)b, T,
                     ldt, diag_given ? 1 : 0));
  return 0;
}

// Persistent panels for panels of at most this many rows (BR_PERSIST_ROWS,
// default 0 = off). One cluster launch per panel instead of one per leaf:
// under a concurrent rank-b update it cuts the panel's time 3x in isolation
// (tools/overlap_bench.py), but it holds the cluster's SMs for the whole
// panel, and on c3-c5 the net effect measured flat to -2 %, so it is off.
static bool persistent_panel_enabled(int64_t rows) {
  static const int64_t lim = [] {
    const char* e = std::getenv("BR_PERSIST_ROWS");
    return e ? (int64_t)std::atoll(e) : (int64_t)0;  // measured: no gain on c3-c5
  }();
  static const int64_t lo = [] {  // BR_PERSIST_MIN_ROWS: only panels at least this tall
    const char* e = std::getenv("BR_PERSIST_MIN_ROWS");
    return e ? (int64_t)std::atoll(e) : (int64_t)0;
  }();
  return rows <= lim && rows >= lo;
}

// Stream-ordered 32-bit flag wait / release write (driver stream memory
// operations: no SM is held while waiting). Resolved through the runtime's
// driver entry point so the library does not link libcuda directly.
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_waitValue32 g_wait32 = nullptr;
static PFN_writeValue32 g_write32 = nullptr;
static int stream_ops_init() {
  if (g_wait32 && g_write32) return 0;
  cudaDriverEntryPointQueryResult q1, q2;
  void* f1 = nullptr;
  void* f2 = nullptr;
  // the CUDA 12 (_v2) entry points; the unversioned lookup can return the
  // legacy ABI, whose calls succeed without taking effect
  BR_CUDA(cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f1, 12000, cudaEnableDefault, &q1));
  BR_CUDA(cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &f2, 12000, cudaEnableDefault, &q2));
  if (!f1 || !f2 || q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess) {
    set_error("driver stream memory operations unavailable");
    return 1;
  }
  g_wait32 = (PFN_waitValue32)f1;
  g_write32 = (PFN_writeValue32)f2;
  return 0;
}
static int stream_wait_flag(cudaStream_t st, unsigned* f, unsigned v) {
  BR_CHECK(stream_ops_init());
  const CUresult r = g_wait32((CUstream)st, (CUdeviceptr)f, v, CU_STREAM_WAIT_VALUE_EQ);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue32 failed (CUresult %d)", (int)r);
    return 1000 + (int)r;
  }
  return 0;
}
static int stream_set_flag(cudaStream_t st, unsigned* f, unsigned v) {
  BR_CHECK(stream_ops_init());
  const CUresult r = g_write32((CUstream)st, (CUdeviceptr)f, v, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWriteValue32 failed (CUresult %d)", (int)r);
    return 1000 + (int)r;
  }
  return 0;
}

// Multi-leaf panels: the leaf forms Y T^T on DMMA for the block update
// (default), or the update applies T^T inside the split-K reduction and the
// leaf skips W (BR_LEAF_W=0; measured flat to slower: c4 447.2 vs 445.4 ms,
// the reduction pass is then always launched).
static bool leaf_w_mode() {
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("BR_LEAF_W");
    m = (e && std::atoi(e) == 0) ? 0 : 1;
  }
  return m == 1;
}

int64_t panel_scratch_doubles(int64_t b) {
  // + 3 b^2: Gram / product buffers of the recursive split (panel_qr)
  return b * b + LEAF_NB * LEAF_NB + 2 * LEAF_NB * b + (b > TAB_MAXB ? b * TAB_MAXB : 0) + 3 * b * b;
}

// Recursive splitting of wide, tall panels (panel_qr). A panel of at least
// rec_min_rows() rows whose column range is wider than rec_width() is split
// in two halves: the left half is factored, its block reflector
// (I + Y1 T1 Y1^T)^T is applied to the right half with three GEMMs
// (Z = Y1^T P2, Z' = T1^T Z, P2 += Y1 Z'), then the right half is factored.
// Narrower ranges run the right-looking leaf loop. Same reflectors, fewer
// passes over the panel: the right-looking rank-nb updates re-read and
// re-write the whole rest of the panel after every leaf (j x b^2 / (2 nb)
// doubles each way), the recursion moves j x b per level.
static int64_t rec_width() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = std::getenv("BR_REC_WIDTH");
    v = e ? std::atoll(e) : 1 << 30;
  }
  return v;
}
static int64_t rec_min_rows() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = std::getenv("BR_REC_MIN_ROWS");
    v = e ? std::atoll(e) : 0;
  }
  return v;
}

// phase: 0 = the whole panel; 1 = leaves and block updates only (Y, tau, the
// leaves' diagonal T blocks); 2 = the rest of a multi-leaf panel (Gram matrix,
// T, W = Y T) - the strict SM split runs phase 1 on the confined stream and
// phase 2 on the full device. Single-leaf panels finish in phase 1.
int panel_qr(cudaStream_t st, Scratch& ws, DevBuf& pscratch, MatView P, MatView Y, double* tau,
             MatView T, MatView* W, int max_ctas, Workspace* pws, LeafMarks* marks, int phase) {
  const int64_t j = P.rows, b = P.cols;
  if (marks) marks->n = 0;
  auto mark = [&](int64_t c0, int64_t c1) -> int {  // Y[:, c0:c1) final on st
    if (!marks || !pws) return 0;
    if (marks->n >= LeafMarks::kMax) {
      set_error("panel_qr: more than %d leaf marks", LeafMarks::kMax);
      return -1;
    }
    cudaEvent_t ev = ws_event(*pws);
    BR_CUDA(cudaEventRecord(ev, st));
    marks->c0[marks->n] = c0;
    marks->c1[marks->n] = c1;
    marks->ev[marks->n] = ev;
    ++marks->n;
    return 0;
  };
  if (j < b || b < 1) {
    set_error("panel_qr needs j >= b >= 1, got %lld x %lld", (long long)j, (long long)b);
    return -1;
  }
  const int nbl = leaf_width(j, b);
  if (nbl < 1) {
    set_error("panel_qr: %lld rows exceed one cluster's register capacity (%lld)", (long long)j,
              (long long)leaf_capacity(2));
    return -1;
  }
  if (b <= nbl) {
    if (phase == 2) return 0;
    // single leaf: Y, tau, T and W in one kernel (narrow leaves: W by a GEMM)
    if (nbl < 8) {
      BR_CHECK(zero_fill(st, T));
      BR_CHECK(launch_leaf(st, P, Y, tau, T.p, T.ld, nullptr));
      if (W) BR_CHECK(gemm(st, ws, *W, Y, T, 1.0, 0.0, nullptr, max_ctas, 0, true));
      return mark(0, b);
    }
    BR_CHECK(launch_leaf(st, P, Y, tau, T.p, T.ld, W));
    return mark(0, b);
  }
  // multi-leaf, right-looking
  if (phase != 2) {
    BR_CHECK(zero_fill(st, Y));
    BR_CHECK(zero_fill(st, T));
  }
  if (pscratch.cap < panel_scratch_doubles(b)) {
    set_error("panel_qr: panel scratch too small");
    return -1;
  }
  double* scratch = pscratch.p;  // [G b x b][Tblk 32x32][Z 32 x b][Z2 32 x b]
  MatView G(scratch, b, b, b);
  double* tblk = scratch + b * b;
  MatView Z(tblk + LEAF_NB * LEAF_NB, LEAF_NB, LEAF_NB, b);
  MatView Z2(Z.p + LEAF_NB * b, LEAF_NB, LEAF_NB, b);
  const int nleaves = (int)cdiv(b, nbl);
  const bool persist = pws && W && nleaves <= 64 && nbl <= 32 && persistent_panel_enabled(j);
  if (persist && phase != 2) {
    // Persistent panel: one cluster launch factors every leaf; the block
    // update of leaf s is applied on the aux stream, first to the next
    // leaf's columns (then the leaf may proceed), then to the rest of the
    // panel while the next leaf runs.
    Workspace& w = *pws;
    if (++w.epoch == 0) ++w.epoch;
    const unsigned ep = w.epoch;
    BR_CUDA(cudaEventRecord(w.ev_aux0, st));
    BR_CUDA(cudaStreamWaitEvent(w.aux, w.ev_aux0, 0));
    BR_CHECK(launch_leaf(st, P, Y, tau, nullptr, 0, W, 1, nleaves, nbl, w.flags, ep));
    for (int s = 0; s + 1 < nleaves; ++s) {
      const int64_t c0 = (int64_t)s * nbl, e = std::min<int64_t>(c0 + nbl, b), wc = e - c0;
      const int64_t h1 = std::min<int64_t>(e + nbl, b);
      BR_CHECK(stream_wait_flag(w.aux, &w.flags[s], ep));
      MatView leafY = Y.sub(c0, c0, j - c0, wc), What = W->sub(c0, c0, j - c0, wc);
      MatView head = P.sub(c0, e, j - c0, h1 - e), Zh = Z.sub(0, 0, wc, h1 - e);
      BR_CHECK(gemm(w.aux, w.sk_aux, Zh, leafY.T(), head, 1.0, 0.0, nullptr, max_ctas));
      BR_CHECK(gemm(w.aux, w.sk_aux, head, What, Zh, 1.0, 1.0, nullptr, max_ctas));
      BR_CHECK(stream_set_flag(w.aux, &w.flags[64 + s + 1], ep));
      if (h1 < b) {
        MatView rest = P.sub(c0, h1, j - c0, b - h1), Zr = Z.sub(0, h1 - e, wc, b - h1);
        BR_CHECK(gemm(w.aux, w.sk_aux, Zr, leafY.T(), rest, 1.0, 0.0, nullptr, max_ctas));
        BR_CHECK(gemm(w.aux, w.sk_aux, rest, What, Zr, 1.0, 1.0, nullptr, max_ctas));
      }
    }
    BR_CUDA(cudaEventRecord(w.ev_aux1, w.aux));
    BR_CUDA(cudaStreamWaitEvent(st, w.ev_aux1, 0));
    BR_CHECK(mark(0, b));
  }
  // right-looking leaves over columns [c0, c1): every update stops at c1
  auto right_looking = [&](int64_t c0, int64_t c1) -> int {
    for (int64_t s = c0; s < c1; s += nbl) {
      const int64_t e = std::min<int64_t>(s + nbl, c1);
      const int64_t w = e - s;
      MatView leafP = P.sub(s, s, j - s, w);
      MatView leafY = Y.sub(s, s, j - s, w);
      if (e < c1 && W && leaf_w_mode() && nbl >= 8) {
        // P[s:, e:c1] += (Y_blk T_blk^T)(Y_blk^T P[s:, e:c1]); the leaf writes
        // Y_blk T_blk^T into W's columns (W itself is formed at the end)
        MatView What = W->sub(s, s, j - s, w);
        BR_CHECK(launch_leaf(st, leafP, leafY, tau + s, T.p + s + s * T.ld, T.ld, &What, 1));
        BR_CHECK(mark(s, e));
        MatView rest = P.sub(s, e, j - s, c1 - e);
        MatView Zs = Z.sub(0, 0, w, c1 - e);
        BR_CHECK(gemm(st, ws, Zs, leafY.T(), rest, 1.0, 0.0, nullptr, max_ctas));
        BR_CHECK(gemm(st, ws, rest, What, Zs, 1.0, 1.0, nullptr, max_ctas));
        continue;
      }
      BR_CHECK(launch_leaf(st, leafP, leafY, tau + s, T.p + s + s * T.ld, T.ld, nullptr));
      BR_CHECK(mark(s, e));
      if (e < c1) {
        // P[s:, e:c1] += Y_blk (T_blk^T (Y_blk^T P[s:, e:c1])): the T_blk^T product
        // rides on the split-K reduction, so the leaf needs no W
        MatView rest = P.sub(s, e, j - s, c1 - e);
        MatView Z2s = Z2.sub(0, 0, w, c1 - e);
        MatView Tb(T.p + s + s * T.ld, T.ld, w, w);  // the leaf's T block
        BR_CHECK(gemm_tt(st, ws, Z2s, leafY.T(), rest, Tb));
        BR_CHECK(gemm(st, ws, rest, leafY, Z2s, 1.0, 1.0, nullptr, max_ctas));
      }
    }
    return 0;
  };
  double* rbuf = scratch + panel_scratch_doubles(b) - 3 * b * b;  // G1 | Z | Z'
  std::function<int(int64_t, int64_t)> rec = [&](int64_t c0, int64_t c1) -> int {
    const int64_t w = c1 - c0;
    // halves on leaf (and 32-row T block) boundaries: the final T assembly
    // reads the leaves' diagonal blocks at multiples of 32
    const int64_t al = std::max<int64_t>(nbl, TAB);
    const int64_t h = std::max<int64_t>(al, cdiv(w / 2, al) * al);
    // confined panels (phase 1 of the strict SM split) split once at 128 columns:
    // on 16 SMs one K = 128 update of the right half beats the leaf-by-leaf
    // updates it replaces (c4 panel class 215 -> 201 ms, tools/exp_env.sh)
    const int64_t rw = (phase == 1) ? std::min<int64_t>(rec_width(), 128) : rec_width();
    const int64_t rmin = (phase == 1) ? 0 : rec_min_rows();
    if (w <= rw || h >= w || j < rmin) return right_looking(c0, c1);
    BR_CHECK(rec(c0, c0 + h));
    // T1 of the left half from its Gram matrix (leaves wrote the diagonal blocks)
    MatView Y1 = Y.sub(c0, c0, j - c0, h), T1 = T.sub(c0, c0, h, h);
    MatView G1(rbuf, h, h, h), Zr(rbuf + b * b, h, h, w - h), Zr2(rbuf + 2 * b * b, h, h, w - h);
    BR_CHECK(gemm(st, ws, G1, Y1.T(), Y1, 1.0, 0.0, nullptr, max_ctas));
    BR_CHECK(t_from_gram(st, G1.p, G1.ld, tau + c0, h, T1.p, T1.ld, nbl % TAB == 0));
    // P2 := (I + Y1 T1 Y1^T)^T P2
    MatView P2 = P.sub(c0, c0 + h, j - c0, w - h);
    BR_CHECK(gemm(st, ws, Zr, Y1.T(), P2, 1.0, 0.0, nullptr, max_ctas));
    BR_CHECK(gemm(st, ws, Zr2, T1.T(), Zr, 1.0, 0.0, nullptr, max_ctas));
    BR_CHECK(gemm(st, ws, P2, Y1, Zr2, 1.0, 1.0, nullptr, max_ctas));
    return rec(c0 + h, c1);
  };
  if (!persist && phase != 2) BR_CHECK(rec(0, b));
  if (phase == 1) return 0;
  // full T: Gram, then the blocked recurrence in one kernel (T is written whole,
  // zeros below the diagonal). 32-wide leaves already wrote the 32 x 32
  // diagonal blocks of T.
  const bool diag_given = !persist && nbl % TAB == 0;
  BR_CHECK(gemm(st, ws, G, Y.T(), Y, 1.0, 0.0, nullptr, max_ctas));
  if (b <= TAB_MAXB) {
    BR_CHECK(t_from_gram(st, G.p, G.ld, tau, b, T.p, T.ld, diag_given));
  } else {
    // wider than one assembly kernel: diagonal super-blocks by the kernel,
    // T[0:s, s:e] = T[0:s,0:s] (G[0:s,s:e] T[s:e,s:e]) by GEMMs
    double* tmpp = scratch + b * b + LEAF_NB * LEAF_NB + 2 * LEAF_NB * b;
    for (int64_t s = 0; s < b; s += TAB_MAXB) {
      const int64_t e = std::min<int64_t>(s + TAB_MAXB, b);
      BR_CHECK(t_from_gram(st, G.p + s + s * G.ld, G.ld, tau + s, e - s, T.p + s + s * T.ld, T.ld,
                           diag_given));
      if (s == 0) continue;
      MatView tmp(tmpp, s, s, e - s);
      BR_CHECK(gemm(st, ws, tmp, G.sub(0, s, s, e - s), T.sub(s, s, e - s, e - s), 1.0, 0.0, nullptr, max_ctas));
      BR_CHECK(gemm(st, ws, T.sub(0, s, s, e - s), T.sub(0, 0, s, s), tmp, 1.0, 0.0, nullptr, max_ctas));
    }
  }
  if (W) BR_CHECK(gemm(st, ws, *W, Y, T, 1.0, 0.0, nullptr, max_ctas, 0, true));  // T upper
  return 0;
}

// house_gen on a single device vector (ref kernels.py:86-110): writes v and
// (tau, beta). Used by the C-ABI br_house_gen and its parity tests.
__global__ void house_gen_kernel(int64_t L, const double* x, double* v, double* tb) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t r = threadIdx.x; r < L; r += blockDim.x) acc = fma(x[r], x[r], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double nrm2 = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) nrm2 += red[w];
  const double nrm = sqrt(nrm2), x0 = x[0];
  double tau = 0.0, beta = 0.0, v0 = 1.0;
  if (nrm != 0.0) {
    const double sign = x0 < 0.0 ? -1.0 : 1.0;
    beta = -sign * nrm;
    v0 = x0 - beta;
    tau = (beta - x0) / beta;
  }
  for (int64_t r = threadIdx.x; r < L; r += blockDim.x)
    v[r] = (r == 0) ? 1.0 : (nrm != 0.0 ? x[r] / v0 : 0.0);
  if (threadIdx.x == 0) { tb[0] = tau; tb[1] = beta; }
}

int house_gen_dev(cudaStream_t st, int64_t L, const double* x, double* v, double* tb) {
  count_launch();
  house_gen_kernel<<<1, 256, 0, st>>>(L, x, v, tb);
  BR_CUDA(cudaGetLastError());
  return 0;
}

// Load every panel kernel (see g_preload_only).
int preload_panel_kernels() {
  LeafArgs a{};
  a.nleaves = 1;
  BR_CHECK((launch_leaf_t<32, 2, 128>(0, a)));
  BR_CHECK((launch_leaf_t<32, 2, 256>(0, a)));
  BR_CHECK((launch_leaf_t<16, 4, 128>(0, a)));
  BR_CHECK((launch_leaf_t<16, 4, 256>(0, a)));
  BR_CHECK((launch_leaf_t<8, 8, 128>(0, a)));
  BR_CHECK((launch_leaf_t<8, 8, 256>(0, a)));
  BR_CHECK((launch_leaf_t<4, 16, 256>(0, a)));
  BR_CHECK((launch_leaf_t<2, 32, 256>(0, a)));
  BR_CHECK((launch_leaf2_t<64, 8>(0, a)));
  BR_CHECK((launch_leaf2_t<8, 8>(0, a)));
  BR_CHECK((launch_leaf2_t<32, 4>(0, a)));
  BR_CHECK((launch_leaf2_t<32, 8>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 2>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 4>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 8>(0, a)));
  BR_CHECK((launch_leaf2_t<32, 8, 4>(0, a)));
  BR_CHECK((launch_leaf2_t<32, 4, 4>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 2, 4>(0, a)));
  BR_CHECK((launch_leaf2_t<32, 16, 4>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 4, 4>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 8, 4>(0, a)));
  BR_CHECK((launch_leaf2_t<32, 4, 4, true>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 2, 4, true>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 2, 8, true>(0, a)));
  BR_CHECK((launch_leaf2_t<32, 4, 8, true>(0, a)));
  BR_CHECK((launch_leaf2_t<32, 8, 8, true>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 4, 8, true>(0, a)));
  BR_CHECK((launch_leaf2_t<16, 8, 8, true>(0, a)));
  cudaFuncAttributes fa;
  BR_CUDA(cudaFuncGetAttributes(&fa, t_assemble_kernel));
  BR_CUDA(cudaFuncGetAttributes(&fa, house_gen_kernel));
  return 0;
}

}  // namespace br
