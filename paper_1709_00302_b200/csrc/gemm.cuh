// FP64 tensor-core (DMMA, mma.sync m8n8k4) GEMM engine for sm_100a.
//
// One templated CTA-tile kernel serves every dense contraction of the
// band reduction:
//   * general C = alpha*op(A)*op(B) + beta*Cin  (apply_wy_left/right pairs,
//     X2, X3, W = Y*T, Gram Y^T*Y, block-reflector steps inside panels);
//   * SYMM   X1 = sym(A2)*W reading only A2's lower triangle
//     (ref kernels.py:312-341);
//   * SYR2K  A2[:, c0:c1] += X3*Y^T + Y*X3^T on lower tiles only
//     (ref kernels.py:344-378).
// Operands are staged global->shared with cp.async (16 B when aligned, else
// 8 B, zero-filled at the edges) in a STAGES-deep pipeline; fragments are read
// with conflict-free padded layouts and fed to DMMA.8x8x4. There are no
// floating-point atomics: split-K partials go to a workspace and are summed
// in a fixed order, so every result is run-to-run deterministic and
// independent of how the output is split into launches (the look-ahead
// relies on that to stay bitwise equal to the non-look-ahead schedule).
#pragma once
#include "common.cuh"

namespace br {

// Device scratch owned by one stream (split-K partials).
struct Scratch {
  double* p = nullptr;
  int64_t cap = 0;  // doubles
  int num_sms = 148;
};

enum AMode { A_N = 0, A_T = 1, A_SYM = 2 };
enum BMode { B_N = 0, B_T = 1 };
enum EpiMode { EPI_GEN = 0, EPI_SPLIT = 1, EPI_LOWER = 2 };

struct GemmArgs {
  int64_t M, N, K;
  const double* A;
  int64_t lda;
  const double* A2;  // optional second K-source for A_N (k >= ksplitA)
  int64_t lda2, ksplitA;
  const double* B;
  int64_t ldb;
  const double* B2;  // optional second K-source for B_T (k >= ksplitB)
  int64_t ldb2, ksplitB;
  double* C;
  int64_t ldc;
  const double* Cin;  // beta term source (may alias C); unused when beta == 0
  int64_t ldcin;
  double alpha, beta;
  int64_t k_per_split;  // EPI_SPLIT: K range per blockIdx.z
  double* ws;           // EPI_SPLIT: partials [z][N][M]
  int64_t c0, c1;       // EPI_LOWER: rows [c0, M) x cols [c0, c1)
  int vecA, vecB;       // 16-byte cp.async allowed for A / B
  int b_upper;          // B_N with B upper triangular: K range of a tile ends at its last column
  // Block-cyclic staircase (the distributed SEVP, dist.py): local column c of
  // a rank's owned block columns is column cyc_r0 + (c / cyc_bs) * cyc_stride
  // + c % cyc_bs of the j x j trailing matrix, stored from that row down
  // (zeros above). A_N: the K range of a tile ends at the last local column
  // that starts at or above its last row; A_T: it starts at the first row of
  // the tile's first column. EPI_LOWER: C columns are local columns (c0 = 0),
  // rows run from cyc_r0, and element (r, c) is written iff r >= column c's
  // global index. cyc_bs == 0: off.
  int64_t cyc_r0;
  int cyc_bs, cyc_stride;
};

// Global column (= first stored row) of local column c under the map.
__host__ __device__ __forceinline__ int64_t cyc_map(const GemmArgs& g, int64_t c) {
  const int64_t q = c / g.cyc_bs;
  return g.cyc_r0 + q * g.cyc_stride + (c - q * g.cyc_bs);
}
// Number of local columns whose first stored row is <= r.
__host__ __device__ __forceinline__ int64_t cyc_count(const GemmArgs& g, int64_t r) {
  if (r < g.cyc_r0) return 0;
  const int64_t d = r - g.cyc_r0, q = d / g.cyc_stride, rem = d - q * g.cyc_stride;
  return q * g.cyc_bs + (rem + 1 < g.cyc_bs ? rem + 1 : g.cyc_bs);
}

// Host-side launch helpers (gemm.cu). All return 0 or a positive CUDA error.
// C = alpha*op(A)*op(B) + beta*Cin (Cin defaults to C). Views carry the
// transposition; a transposed C is handled by transposing the product.
// kps > 0 pins the split-K chunk (see gemm_plan_kps).
int gemm(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, double alpha,
         double beta, const MatView* Cin = nullptr, int max_ctas = 0, int64_t kps = 0,
         bool b_upper = false);
// C = T^T * op(A) * op(B) for a small C (at most 64 rows; T upper triangular,
// C.rows x C.rows): split-K partials reduced and multiplied by T^T in one pass.
int gemm_tt(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, MatView T);
// The split-K chunk gemm() would choose for this whole product. Updating the
// product in row/column pieces with this kps sums every element in the same
// order as the whole call, so the result is bitwise independent of the pieces.
int64_t gemm_plan_kps(const Scratch& ws, MatView C, MatView A, MatView B, double beta);
// X1 = sym(A2) * W, A2 lower-stored j x j (non-transposed view).
int symm_lower(cudaStream_t st, Scratch& ws, MatView X1, MatView A2, MatView W,
               double alpha = 1.0, double beta = 0.0);
// A2[:, c0:c1] += X3*Y^T + Y*X3^T, lower triangle only.
int syr2k_lower(cudaStream_t st, MatView A2, MatView X3, MatView Y, int64_t c0, int64_t c1,
                int max_ctas = 0);

// C = op(A) op(B) through split-K partials, and in the same reduction pass
// D += P C (left; C at most 64 rows, P at most 64 x C.rows) or D += C Q^T
// (right; C at most 64 columns, Q at most 64 x C.cols). Deterministic.
int gemm_left_update(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, MatView D,
                     MatView P);
int gemm_right_update(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, MatView D,
                      MatView Q);

// Block-cyclic column slab of a j x j lower-stored trailing matrix (the
// distributed SEVP): L is j x ncols, local column c being trailing column
// r0 + (c / bs) * stride + c % bs, stored from that row down with zeros above.
struct CycCols {
  int64_t r0;
  int bs, stride;
};
// Rows [p0, p1) of this slab's share of X1 = sym(A2) W into X1 ((p1 - p0) x
// b; all other entries of A2 belong to other ranks): X1 = L Wown +
// fold(L^T W - diag(L) Wown), Wown the rows of W at the slab's columns, fold
// placing column c's row at row map(c); summed over a partition of A2's
// columns it is sym(A2) W. [p0, p1) must not split an owned block.
// tmp: 2 * ncols * b doubles.
int symm_cyclic(cudaStream_t st, Scratch& ws, MatView X1, MatView L, MatView W, CycCols m,
                double* tmp, int64_t p0, int64_t p1);
// L += lower part of X3 Y^T + Y X3^T at the slab's columns (tmp: 2 * ncols * b).
int syr2k_cyclic(cudaStream_t st, MatView L, MatView X3, MatView Y, CycCols m, double* tmp);

// The SEVP X products in ONE persistent launch (b <= 64, ref sevp.py:156-176):
// X1 = sym(A2) W, X2 = X1^T W / 2, X3 = X1 + Y X2, phases separated by a
// grid barrier (bar: 2 zeroed words, self-resetting). Returns 1 (nothing
// launched) when the shape is not covered; the caller then runs the
// separate kernels.
int xchain(cudaStream_t st, Scratch& ws, MatView X1, MatView X2, MatView X3, MatView A2,
           MatView W, MatView Y, unsigned* bar);

}  // namespace br
