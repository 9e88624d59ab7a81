// DMMA GEMM host dispatch: tile configuration, split-K, fixed-order reduction
// (kernel template in gemm_kernel.cuh, contract in gemm.cuh).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "driver.cuh"
#include "gemm.cuh"
#include "gemm_tiles.cuh"

namespace br {

// Fixed-order split-K reduction: C = alpha * sum_z ws[z] + beta * Cin.
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int S, const double* __restrict__ ws,
                                     double alpha, double beta, const double* Cin, int64_t ldcin,
                                     double* C, int64_t ldc) {
  const int64_t total = M * N;
  pdl_wait();
  pdl_trigger();
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % M, c = idx / M;
    double s = 0.0;
    for (int z = 0; z < S; ++z) s += ws[(int64_t)z * total + idx];
    double out = alpha * s;
    if (beta != 0.0) out += beta * Cin[r + c * ldcin];
    C[r + c * ldc] = out;
  }
}

// Fixed-order split-K reduction followed by a small triangular product:
// C (M x N, M <= 64) = T^T * sum_z ws[z], T upper triangular M x M. CTA per 16
// output columns; the block reflector step of a panel (Z = T^T (Y^T P)) in
// one pass over the partials.
constexpr int TT_MAXM = 64, TT_COLS = 16;
__global__ void __launch_bounds__(256) splitk_reduce_tt_kernel(int64_t M, int64_t N, int S,
                                                               const double* __restrict__ ws,
                                                               const double* __restrict__ T,
                                                               int64_t ldt, double* C, int64_t ldc) {
  __shared__ double Ts[TT_MAXM][TT_MAXM + 1];
  __shared__ double Zs[TT_MAXM][TT_COLS + 1];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * TT_COLS;
  const int m = (int)M;
  for (int i = tid; i < m * m; i += 256) {
    const int r = i % m, c = i / m;
    Ts[r][c] = (r <= c) ? T[r + (int64_t)c * ldt] : 0.0;
  }
  const int64_t total = M * N;
  for (int i = tid; i < m * TT_COLS; i += 256) {
    const int r = i % m, c = i / m;
    double s = 0.0;
    if (c0 + c < N) {
      const double* src = ws + (c0 + c) * M + r;
      for (int z = 0; z < S; ++z) s += src[(int64_t)z * total];
    }
    Zs[r][c] = s;
  }
  __syncthreads();
  for (int i = tid; i < m * TT_COLS; i += 256) {
    const int r = i % m, c = i / m;
    if (c0 + c >= N) continue;
    double s = 0.0;
    for (int k = 0; k <= r; ++k) s = fma(Ts[k][r], Zs[k][c], s);
    C[r + (c0 + c) * ldc] = s;
  }
}

static inline bool al16(const void* p, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 2 == 0);
}

// Tile configuration choices, measured on B200 (tools/gemm_cfg_sweep.sh):
// 2-CTA/SM tiles win because one CTA's prologue/epilogue overlaps the other's
// main loop. Environment overrides (tuning aid): BR_GEMM_BIG, BR_GEMM_SYMM,
// BR_GEMM_LOWER = L|A|B|C|D.
static int env_cfg(const char* var, int dflt) {
  if (const char* e = std::getenv(var)) {
    for (int c = 0; c < CFG_COUNT; ++c)
      if (std::strcmp(e, kTiles[c].name) == 0) return c;
  }
  return dflt;
}
static int big_cfg(int am, bool rank_update) {
  static int gen = -1, sym = -1, rku = -1;
  if (gen < 0) {
    gen = env_cfg("BR_GEMM_BIG", CFG_G);
    // SYMM: 64x128 tiles with BK = 16, 3 stages (G) against BK = 32, 2 stages (K,
    // round 1's choice): SYMM class c3 13.9 -> 13.2 ms, c5 711 -> 703 ms
    // (tools/exp_symm.sh; whole step c3 42.2 -> 41.4 ms, c5 1566 -> 1558 ms)
    sym = env_cfg("BR_GEMM_SYMM", CFG_G);
    rku = env_cfg("BR_GEMM_RANKB", CFG_J);
  }
  if (am == A_SYM) return sym;
  return rank_update ? rku : gen;
}
static int lower_cfg(int64_t j) {
  // 64x64 tiles with BK=32 (3 CTAs/SM) at every size: against 128x128 for
  // j < 4096 (round 1's choice) the SYR2K class went c1 2.17 -> 1.69 ms,
  // c3 18.1 -> 16.1 ms (whole step 46.1 -> 45.2), c5 1582 -> 1577 ms
  static int cfg = -2;
  if (cfg == -2) {
    cfg = -1;
    if (std::getenv("BR_GEMM_LOWER")) cfg = env_cfg("BR_GEMM_LOWER", CFG_L);
    if (cfg >= 0 && kTiles[cfg].bm != kTiles[cfg].bn) cfg = CFG_L;
  }
  if (cfg >= 0) return cfg;
  (void)j;
  return CFG_J;
}

// Tile configuration of a general/symm GEMM of shape (M, N, K).
static int pick_cfg(int am, const GemmArgs& g) {
  // rank-b updates: short K (the band width) accumulated onto a large C
  const bool rank_update = g.beta != 0.0 && g.K <= 512 && g.M * g.N >= (int64_t)1 << 20;
  int cfg = big_cfg(am, rank_update);
  if (g.N <= 32) cfg = CFG_NS;
  else if (g.M <= 32) cfg = CFG_MS;
  return cfg;
}

// Split-K chunk (k_per_split; == K means no split) from a small cost model:
// waves of resident CTAs times the k-tiles each CTA runs, plus the
// fixed-order reduction pass. This keeps the last wave from idling most SMs
// (wave quantization) on the tall-skinny reductions (W^T E, D W_V, X1^T W,
// Y^T Y).
static int64_t pick_kps(int cfg, const Scratch& ws, const GemmArgs& g, int max_ctas) {
  const int bm = kTiles[cfg].bm, bn = kTiles[cfg].bn, cps = kTiles[cfg].ctas_per_sm;
  const int64_t tiles = cdiv(g.M, bm) * cdiv(g.N, bn);
  const int bk = kTileBK[cfg];
  const int64_t nkt = cdiv(g.K, bk);
  const int64_t slots = (max_ctas > 0) ? std::max(1, max_ctas) : (int64_t)ws.num_sms * cps;
  const double kt_time = (double)cps * bm * bn * bk * 2 / 251e9;  // one k-tile, one CTA
  int64_t S = 1;
  double best = 1e30;
  const int64_t smax = std::min<int64_t>(64, std::max<int64_t>(1, nkt / 2));
  for (int64_t s = 1; s <= smax; ++s) {
    if (s > 1 && s * g.M * g.N > ws.cap) break;
    const double waves = (double)cdiv(tiles * s, slots);
    double t = waves * (double)cdiv(nkt, s) * kt_time;
    if (s > 1) t += (double)(s + 1) * g.M * g.N * 8.0 / 5e12 + 3e-6;
    if (t < best * 0.995) {
      best = t;
      S = s;
    }
  }
  return S > 1 ? cdiv(nkt, S) * bk : g.K;
}

// Dispatch a general/symm GEMM: chooses tile config and split-K. A caller
// that updates one logical product in pieces passes the k_per_split planned
// for the whole product (gemm_plan_kps), so every element is summed in the
// same order whatever the pieces are (bitwise split invariance).
static int run_gemm(int am, cudaStream_t st, Scratch& ws, GemmArgs g, bool btrans, int max_ctas,
                    int64_t fixed_kps, const double* tt = nullptr, int64_t ldtt = 0,
                    bool cyc = false) {
  if (g.M <= 0 || g.N <= 0) return 0;
  if (g.K <= 0) {  // C = beta*Cin
    const int64_t total = g.M * g.N;
    int blocks = (int)std::min<int64_t>(cdiv(total, 256), 4096);
    count_launch();
    BR_CUDA(launch_pdl(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st, g.M, g.N, 0,
                       (const double*)nullptr, g.alpha, g.beta, g.Cin, g.ldcin, g.C, g.ldc));
    return 0;
  }
  // block-cyclic staircase products run the GF_CYC instantiations (config G)
  const int cfg = cyc ? CFG_G : pick_cfg(am, g);
  auto lt = [&](int c, int a, int bm_, int e, cudaStream_t s_, const GemmArgs& g_, dim3 gr) {
    return cyc ? launch_tile_cyc(c, a, bm_, e, s_, g_, gr) : launch_tile(c, a, bm_, e, s_, g_, gr);
  };
  const int bm = kTiles[cfg].bm, bn = kTiles[cfg].bn;
  const int sms = ws.num_sms;
  int64_t kps = fixed_kps > 0 ? std::min(fixed_kps, g.K) : pick_kps(cfg, ws, g, max_ctas);
  int64_t S = cdiv(g.K, kps);
  if (S > 1 && S * g.M * g.N > ws.cap) {
    set_error("gemm: split-K scratch too small (%lld x %lld x %lld)", (long long)S,
              (long long)g.M, (long long)g.N);
    return -1;
  }
  g.k_per_split = S > 1 ? kps : g.K;
  dim3 grid((unsigned)cdiv(g.M, bm), (unsigned)cdiv(g.N, bn), (unsigned)S);
  const int bmd = btrans ? B_T : B_N;
  if (tt) {  // C = T^T (sum of partials): always through the workspace
    if (S * g.M * g.N > ws.cap) {
      set_error("gemm_tt: split-K scratch too small");
      return -1;
    }
    g.ws = ws.p;
    BR_CHECK(lt(cfg, am, bmd, EPI_SPLIT, st, g, grid));
    count_launch();
    BR_CUDA(launch_pdl(splitk_reduce_tt_kernel, dim3((unsigned)cdiv(g.N, TT_COLS)), dim3(256), 0, st, g.M,
                       g.N, (int)S, (const double*)ws.p, tt, ldtt, g.C, g.ldc));
    return 0;
  }
  if (S == 1) {
    BR_CHECK(lt(cfg, am, bmd, EPI_GEN, st, g, grid));
  } else {
    g.ws = ws.p;
    BR_CHECK(lt(cfg, am, bmd, EPI_SPLIT, st, g, grid));
    const int64_t total = g.M * g.N;
    int blocks = (int)std::min<int64_t>(cdiv(total, 256), (int64_t)sms * 8);
    count_launch();
    BR_CUDA(launch_pdl(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st, g.M, g.N, (int)S,
                       (const double*)ws.p, g.alpha, g.beta, g.Cin, g.ldcin, g.C, g.ldc));
  }
  return 0;
}

// Normalizes orientation (C^T = op(B)^T op(A)^T) and fills GemmArgs.
static int make_args(MatView C, MatView A, MatView B, double alpha, double beta,
                     const MatView* Cin_, GemmArgs& g, int& am, bool& btrans) {
  MatView Cin = Cin_ ? *Cin_ : C;
  if (C.trans) {
    MatView t = A.T();
    A = B.T();
    B = t;
    C = C.T();
    Cin = Cin.T();
  }
  if (Cin.trans) {
    set_error("gemm: Cin orientation must match C");
    return -1;
  }
  if (A.rows != C.rows || B.cols != C.cols || A.cols != B.rows) {
    set_error("gemm: shape mismatch (%lld x %lld) = (%lld x %lld)(%lld x %lld)", (long long)C.rows,
              (long long)C.cols, (long long)A.rows, (long long)A.cols, (long long)B.rows,
              (long long)B.cols);
    return -1;
  }
  g = GemmArgs{};
  g.M = C.rows;
  g.N = C.cols;
  g.K = A.cols;
  g.A = A.p;
  g.lda = A.ld;
  g.A2 = A.p;
  g.lda2 = A.ld;
  g.ksplitA = INT64_MAX;
  g.B = B.p;
  g.ldb = B.ld;
  g.B2 = B.p;
  g.ldb2 = B.ld;
  g.ksplitB = INT64_MAX;
  g.C = C.p;
  g.ldc = C.ld;
  g.Cin = Cin.p;
  g.ldcin = Cin.ld;
  g.alpha = alpha;
  g.beta = beta;
  g.vecA = al16(A.p, A.ld);
  g.vecB = al16(B.p, B.ld);
  am = A.trans ? A_T : A_N;
  btrans = B.trans;
  return 0;
}

int gemm(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, double alpha,
         double beta, const MatView* Cin, int max_ctas, int64_t kps, bool b_upper) {
  GemmArgs g;
  int am = 0;
  bool bt = false;
  if (b_upper && (B.trans || C.trans)) {
    set_error("gemm: b_upper needs a non-transposed B and C");
    return -1;
  }
  BR_CHECK(make_args(C, A, B, alpha, beta, Cin, g, am, bt));
  g.b_upper = b_upper ? 1 : 0;
  return run_gemm(am, st, ws, g, bt, max_ctas, kps);
}

int gemm_tt(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, MatView T) {
  GemmArgs g;
  int am = 0;
  bool bt = false;
  if (C.trans || T.trans || C.rows > TT_MAXM || T.rows != C.rows || T.cols != C.rows) {
    set_error("gemm_tt: C must be a plain view with at most %d rows and T square", TT_MAXM);
    return -1;
  }
  BR_CHECK(make_args(C, A, B, 1.0, 0.0, nullptr, g, am, bt));
  return run_gemm(am, st, ws, g, bt, 0, 0, T.p, T.ld);
}

// ---------------------------------------------------------------------------
// Split-K products with a small update fused into their reduction pass (the
// narrow-panel chains of the triangular band: Z_L then the LQ panel's rows,
// Z_R then the next QR panel's columns). One launch instead of the split-K
// reduction plus a small GEMM on the critical path of every iteration.
// ---------------------------------------------------------------------------
constexpr int FU_MAX = 64;   // max bp / bq / update width
constexpr int FU_COLS = 16;  // columns of C per CTA (left form)
constexpr int FU_ROWS = 16;  // rows of C per CTA (right form)

// C (M x N, M <= 64) = sum_z ws[z] (fixed order), and D (pr x N) += P (pr x M) C.
__global__ void __launch_bounds__(256) reduce_left_update_kernel(
    int64_t M, int64_t N, int S, const double* __restrict__ ws, double* C, int64_t ldc,
    const double* __restrict__ P, int64_t ldp, int pr, double* D, int64_t ldd) {
  __shared__ double Ps[FU_MAX][FU_MAX + 1];
  __shared__ double Cs[FU_MAX][FU_COLS + 1];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * FU_COLS;
  const int m = (int)M, nc = (int)min((int64_t)FU_COLS, N - c0);
  for (int e = tid; e < pr * m; e += 256) {
    const int r = e % pr, k = e / pr;
    Ps[r][k] = P[r + (int64_t)k * ldp];
  }
  const int64_t tot = M * N;
  for (int e = tid; e < m * nc; e += 256) {
    const int k = e % m, c = e / m;
    const double* src = ws + (c0 + c) * M + k;
    double sacc = 0.0;
    for (int z = 0; z < S; ++z) sacc += src[(int64_t)z * tot];
    Cs[k][c] = sacc;
    C[k + (c0 + c) * ldc] = sacc;
  }
  __syncthreads();
  for (int e = tid; e < pr * nc; e += 256) {
    const int r = e % pr, c = e / pr;
    double* d = D + r + (c0 + c) * ldd;
    double acc = *d;
    for (int k = 0; k < m; ++k) acc = fma(Ps[r][k], Cs[k][c], acc);
    *d = acc;
  }
}

// C (M x N, N <= 64) = sum_z ws[z] (fixed order), and D (M x qc) += C Q^T
// (Q qc x N).
__global__ void __launch_bounds__(256) reduce_right_update_kernel(
    int64_t M, int64_t N, int S, const double* __restrict__ ws, double* C, int64_t ldc,
    const double* __restrict__ Q, int64_t ldq, int qc, double* D, int64_t ldd) {
  __shared__ double Qs[FU_MAX][FU_MAX + 1];
  __shared__ double Cs[FU_ROWS][FU_MAX + 1];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * FU_ROWS;
  const int n = (int)N, nr = (int)min((int64_t)FU_ROWS, M - r0);
  for (int e = tid; e < qc * n; e += 256) {
    const int q = e % qc, k = e / qc;
    Qs[q][k] = Q[q + (int64_t)k * ldq];
  }
  const int64_t tot = M * N;
  for (int e = tid; e < nr * n; e += 256) {
    const int r = e % nr, k = e / nr;
    const double* src = ws + (int64_t)k * M + r0 + r;
    double sacc = 0.0;
    for (int z = 0; z < S; ++z) sacc += src[(int64_t)z * tot];
    Cs[r][k] = sacc;
    C[(r0 + r) + (int64_t)k * ldc] = sacc;
  }
  __syncthreads();
  for (int e = tid; e < nr * qc; e += 256) {
    const int r = e % nr, q = e / nr;
    double* d = D + (r0 + r) + (int64_t)q * ldd;
    double acc = *d;
    for (int k = 0; k < n; ++k) acc = fma(Cs[r][k], Qs[q][k], acc);
    *d = acc;
  }
}

// The split-K partials of C = op(A) op(B) (always through the workspace),
// for the fused reductions below. Returns the number of splits in *S.
static int splitk_partials(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, int* S) {
  GemmArgs g;
  int am = 0;
  bool bt = false;
  BR_CHECK(make_args(C, A, B, 1.0, 0.0, nullptr, g, am, bt));
  if (g.K <= 0) {
    set_error("fused split-K reduction needs K > 0");
    return -1;
  }
  const int cfg = pick_cfg(am, g);
  const int64_t kps = pick_kps(cfg, ws, g, 0);
  const int64_t s = cdiv(g.K, kps);
  if (s * g.M * g.N > ws.cap) {
    set_error("fused split-K reduction: scratch too small");
    return -1;
  }
  g.k_per_split = kps;
  g.ws = ws.p;
  dim3 grid((unsigned)cdiv(g.M, kTiles[cfg].bm), (unsigned)cdiv(g.N, kTiles[cfg].bn), (unsigned)s);
  BR_CHECK(launch_tile(cfg, am, bt ? B_T : B_N, EPI_SPLIT, st, g, grid));
  *S = (int)s;
  return 0;
}

int gemm_left_update(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, MatView D,
                     MatView P) {
  if (C.trans || D.trans || P.trans || C.rows > FU_MAX || P.rows > FU_MAX || P.cols != C.rows ||
      D.rows != P.rows || D.cols != C.cols) {
    set_error("gemm_left_update: bad views");
    return -1;
  }
  if (C.rows == 0 || C.cols == 0) return 0;
  int S = 0;
  BR_CHECK(splitk_partials(st, ws, C, A, B, &S));
  count_launch();
  BR_CUDA(launch_pdl(reduce_left_update_kernel, dim3((unsigned)cdiv(C.cols, FU_COLS)), dim3(256), 0,
                     st, C.rows, C.cols, S, (const double*)ws.p, C.p, C.ld, (const double*)P.p, P.ld,
                     (int)P.rows, D.p, D.ld));
  return 0;
}

int gemm_right_update(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, MatView D,
                      MatView Q) {
  if (C.trans || D.trans || Q.trans || C.cols > FU_MAX || Q.rows > FU_MAX || Q.cols != C.cols ||
      D.rows != C.rows || D.cols != Q.rows) {
    set_error("gemm_right_update: bad views");
    return -1;
  }
  if (C.rows == 0 || C.cols == 0) return 0;
  int S = 0;
  BR_CHECK(splitk_partials(st, ws, C, A, B, &S));
  count_launch();
  BR_CUDA(launch_pdl(reduce_right_update_kernel, dim3((unsigned)cdiv(C.rows, FU_ROWS)), dim3(256), 0,
                     st, C.rows, C.cols, S, (const double*)ws.p, C.p, C.ld, (const double*)Q.p, Q.ld,
                     (int)Q.rows, D.p, D.ld));
  return 0;
}

int64_t gemm_plan_kps(const Scratch& ws, MatView C, MatView A, MatView B, double beta) {
  GemmArgs g;
  int am = 0;
  bool bt = false;
  if (make_args(C, A, B, 1.0, beta, nullptr, g, am, bt) || g.M <= 0 || g.N <= 0 || g.K <= 0)
    return 0;
  return pick_kps(pick_cfg(am, g), ws, g, 0);
}

int symm_lower(cudaStream_t st, Scratch& ws, MatView X1, MatView A2, MatView W, double alpha,
               double beta) {
  if (A2.trans || X1.trans || W.trans || A2.rows != A2.cols || X1.rows != A2.rows ||
      W.rows != A2.rows || X1.cols != W.cols) {
    set_error("symm_lower: bad views");
    return -1;
  }
  GemmArgs g{};
  g.M = A2.rows;
  g.N = W.cols;
  g.K = A2.rows;
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
  g.C = X1.p;
  g.ldc = X1.ld;
  g.Cin = X1.p;
  g.ldcin = X1.ld;
  g.alpha = alpha;
  g.beta = beta;
  g.vecA = al16(A2.p, A2.ld);
  g.vecB = al16(W.p, W.ld);
  return run_gemm(A_SYM, st, ws, g, false, 0, 0);
}

int syr2k_lower(cudaStream_t st, MatView A2, MatView X3, MatView Y, int64_t c0, int64_t c1,
                int max_ctas) {
  const int64_t j = A2.rows;
  if (A2.trans || X3.trans || Y.trans || A2.cols != j || X3.rows != j || Y.rows != j ||
      X3.cols != Y.cols || c0 < 0 || c1 > j || c0 > c1) {
    set_error("syr2k_lower: bad views/range");
    return -1;
  }
  if (c0 == c1 || X3.cols == 0) return 0;
  const int64_t b = X3.cols;
  GemmArgs g{};
  g.M = j;
  g.N = j;
  g.K = 2 * b;
  // A_op = [X3 | Y] (rows), B_op(k, n) = [Y | X3](n, k)
  g.A = X3.p;
  g.lda = X3.ld;
  g.A2 = Y.p;
  g.lda2 = Y.ld;
  g.ksplitA = b;
  g.B = Y.p;
  g.ldb = Y.ld;
  g.B2 = X3.p;
  g.ldb2 = X3.ld;
  g.ksplitB = b;
  g.C = A2.p;
  g.ldc = A2.ld;
  g.Cin = A2.p;
  g.ldcin = A2.ld;
  g.alpha = 1.0;
  g.beta = 1.0;
  g.c0 = c0;
  g.c1 = c1;
  // tile origins are offset by c0: 16-byte chunks need an even c0
  g.vecA = al16(X3.p, X3.ld) && al16(Y.p, Y.ld) && (c0 % 2 == 0);
  g.vecB = g.vecA;
  (void)max_ctas;
  // narrow column ranges (the look-ahead's lead strip) on 64x64 tiles: more
  // CTAs for a latency-bound launch; the per-element K order is the same
  const int cfg = (c1 - c0 <= 64) ? CFG_J : lower_cfg(j);
  dim3 grid((unsigned)cdiv(j - c0, kTiles[cfg].bm), (unsigned)cdiv(c1 - c0, kTiles[cfg].bn), 1);
  return launch_tile(cfg, A_N, B_T, EPI_LOWER, st, g, grid);
}

// ---------------------------------------------------------------------------
// Block-cyclic column slabs (the distributed SEVP, dist.py)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t cyc_col(const CycCols& m, int64_t c) {
  const int64_t q = c / m.bs;
  return m.r0 + q * m.stride + (c - q * m.bs);
}

// Rows of s0 / s1 (j x b) at the slab's columns -> d0 / d1 (ncols x b).
__global__ void cyc_gather_kernel(int64_t ncols, int64_t b, CycCols m, const double* s0,
                                  int64_t lds0, double* d0, int64_t ldd0, const double* s1,
                                  int64_t lds1, double* d1, int64_t ldd1) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = ncols * b;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx % ncols, q = idx / ncols, r = cyc_col(m, c);
    d0[c + q * ldd0] = s0[r + q * lds0];
    if (s1) d1[c + q * ldd1] = s1[r + q * lds1];
  }
}

// X1[map(c), q] += Xo[c, q] - L[map(c), c] Wown[c, q]: the slab's transposed
// contributions land on its own rows (the map is one-to-one), without the
// diagonal the first product already counted.
__global__ void cyc_fold_kernel(int64_t ncols, int64_t b, CycCols m, const double* Xo, int64_t ldxo,
                                const double* L, int64_t ldl, const double* Wown, int64_t ldwo,
                                double* X1, int64_t ldx1, int64_t roff) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = ncols * b;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx % ncols, q = idx / ncols, r = cyc_col(m, c);
    X1[r - roff + q * ldx1] += Xo[c + q * ldxo] - L[r + c * ldl] * Wown[c + q * ldwo];
  }
}

static int cyc_check(const char* who, MatView L, int64_t b, CycCols m) {
  const int64_t j = L.rows, nc = L.cols;
  if (L.trans || m.bs < 1 || m.stride < m.bs || m.r0 < 0 || nc % m.bs != 0 ||
      (nc > 0 && cyc_col(m, nc - 1) >= j) || b < 1) {
    set_error("%s: bad block-cyclic slab (j %lld, ncols %lld, r0 %lld, bs %d, stride %d)", who,
              (long long)j, (long long)nc, (long long)m.r0, m.bs, m.stride);
    return -1;
  }
  return 0;
}

static int cyc_gather(cudaStream_t st, int64_t ncols, int64_t b, CycCols m, MatView s0, double* d0,
                      const MatView* s1, double* d1) {
  const int64_t total = ncols * b;
  const int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 8);
  count_launch();
  BR_CUDA(launch_pdl(cyc_gather_kernel, dim3(blocks), dim3(256), 0, st, ncols, b, m,
                     (const double*)s0.p, s0.ld, d0, ncols, s1 ? (const double*)s1->p : nullptr,
                     s1 ? s1->ld : (int64_t)0, d1, ncols));
  return 0;
}

int symm_cyclic(cudaStream_t st, Scratch& ws, MatView X1, MatView L, MatView W, CycCols m,
                double* tmp, int64_t p0, int64_t p1) {
  const int64_t j = L.rows, nc = L.cols, b = W.cols;
  BR_CHECK(cyc_check("symm_cyclic", L, b, m));
  if (X1.trans || W.trans || p0 < 0 || p1 > j || p0 > p1 || X1.rows != p1 - p0 || W.rows != j ||
      X1.cols != b) {
    set_error("symm_cyclic: bad views / row range");
    return -1;
  }
  if (p0 == p1) return 0;
  MatView Xr = X1;
  if (nc == 0) return gemm(st, ws, Xr, MatView(nullptr, 1, p1 - p0, 0), MatView(nullptr, 1, 0, b), 1.0, 0.0);
  GemmArgs cg{};
  cg.cyc_r0 = m.r0;
  cg.cyc_bs = m.bs;
  cg.cyc_stride = m.stride;
  // columns whose first stored row lies in [p0, p1): their transposed
  // contributions belong to these rows; whole owned blocks only
  const int64_t ca = cyc_count(cg, p0 - 1), cb = cyc_count(cg, p1 - 1);
  if (ca % m.bs || cb % m.bs) {
    set_error("symm_cyclic: row range [%lld, %lld) splits an owned block", (long long)p0, (long long)p1);
    return -1;
  }
  MatView Wown(tmp, nc, nc, b), Xo(tmp + nc * b, nc, nc, b);
  BR_CHECK(cyc_gather(st, nc, b, m, W, Wown.p, nullptr, nullptr));
  GemmArgs g;
  int am = 0;
  bool bt = false;
  // X1[p0:p1] = L[p0:p1] Wown (K clipped to the columns that reach a tile's rows)
  BR_CHECK(make_args(Xr, L.sub(p0, 0, p1 - p0, nc), Wown, 1.0, 0.0, nullptr, g, am, bt));
  g.cyc_r0 = m.r0 - p0;
  g.cyc_bs = m.bs;
  g.cyc_stride = m.stride;
  BR_CHECK(run_gemm(am, st, ws, g, bt, 0, 0, nullptr, 0, true));
  if (cb == ca) return 0;
  // Xo = L[:, ca:cb]^T W (K from each column's first stored row)
  const CycCols ms{cyc_map(cg, ca), m.bs, m.stride};
  MatView Ls = L.sub(0, ca, j, cb - ca), Xos = Xo.sub(ca, 0, cb - ca, b);
  BR_CHECK(make_args(Xos, Ls.T(), W, 1.0, 0.0, nullptr, g, am, bt));
  g.cyc_r0 = ms.r0;
  g.cyc_bs = ms.bs;
  g.cyc_stride = ms.stride;
  BR_CHECK(run_gemm(am, st, ws, g, bt, 0, 0, nullptr, 0, true));
  const int64_t total = (cb - ca) * b;
  const int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 8);
  count_launch();
  BR_CUDA(launch_pdl(cyc_fold_kernel, dim3(blocks), dim3(256), 0, st, cb - ca, b, ms,
                     (const double*)Xos.p, Xos.ld, (const double*)Ls.p, Ls.ld,
                     (const double*)(Wown.p + ca), Wown.ld, X1.p, X1.ld, p0));
  return 0;
}

int syr2k_cyclic(cudaStream_t st, MatView L, MatView X3, MatView Y, CycCols m, double* tmp) {
  const int64_t j = L.rows, nc = L.cols, b = X3.cols;
  BR_CHECK(cyc_check("syr2k_cyclic", L, b, m));
  if (X3.trans || Y.trans || X3.rows != j || Y.rows != j || Y.cols != b) {
    set_error("syr2k_cyclic: bad views");
    return -1;
  }
  if (nc == 0) return 0;
  double* Yo = tmp;
  double* Xo = tmp + nc * b;
  BR_CHECK(cyc_gather(st, nc, b, m, Y, Yo, &X3, Xo));
  GemmArgs g{};
  g.M = j;
  g.N = nc;
  g.K = 2 * b;
  // A_op = [X3 | Y] (trailing rows), B_op(k, c) = [Y | X3](map(c), k) gathered
  g.A = X3.p;
  g.lda = X3.ld;
  g.A2 = Y.p;
  g.lda2 = Y.ld;
  g.ksplitA = b;
  g.B = Yo;
  g.ldb = nc;
  g.B2 = Xo;
  g.ldb2 = nc;
  g.ksplitB = b;
  g.C = L.p;
  g.ldc = L.ld;
  g.Cin = L.p;
  g.ldcin = L.ld;
  g.alpha = 1.0;
  g.beta = 1.0;
  g.c0 = 0;
  g.c1 = nc;
  g.cyc_r0 = m.r0;
  g.cyc_bs = m.bs;
  g.cyc_stride = m.stride;
  g.vecA = al16(X3.p, X3.ld) && al16(Y.p, Y.ld) && (m.r0 % 2 == 0);
  g.vecB = al16(Yo, nc) && al16(Xo, nc);
  const int cfg = CFG_J;  // as lower_cfg; GF_CYC instantiation
  dim3 grid((unsigned)cdiv(j - m.r0, kTiles[cfg].bm), (unsigned)cdiv(nc, kTiles[cfg].bn), 1);
  return launch_tile_cyc(cfg, A_N, B_T, EPI_LOWER, st, g, grid);
}

// Load every GEMM instantiation and the split-K reduction (see g_preload_only).
int preload_gemm_kernels() {
  GemmArgs g{};
  const dim3 grid(1, 1, 1);
  for (int cfg = 0; cfg < CFG_COUNT; ++cfg) {
    for (int am : {A_N, A_T, A_SYM})
      for (int bmd : {B_N, B_T})
        for (int epi : {EPI_GEN, EPI_SPLIT}) {
          if (am == A_SYM && bmd == B_T) continue;
          BR_CHECK(launch_tile(cfg, am, bmd, epi, 0, g, grid));
        }
    if (kTiles[cfg].bm == kTiles[cfg].bn) BR_CHECK(launch_tile(cfg, A_N, B_T, EPI_LOWER, 0, g, grid));
  }
  cudaFuncAttributes fa;
  BR_CUDA(cudaFuncGetAttributes(&fa, splitk_reduce_kernel));
  BR_CUDA(cudaFuncGetAttributes(&fa, splitk_reduce_tt_kernel));
  for (int am : {A_N, A_T})
    for (int epi : {EPI_GEN, EPI_SPLIT}) BR_CHECK(launch_tile_cyc(CFG_G, am, B_N, epi, 0, g, grid));
  BR_CHECK(launch_tile_cyc(CFG_J, A_N, B_T, EPI_LOWER, 0, g, grid));
  BR_CHECK(launch_tile_cyc(CFG_L, A_N, B_T, EPI_LOWER, 0, g, grid));
  BR_CUDA(cudaFuncGetAttributes(&fa, cyc_gather_kernel));
  BR_CUDA(cudaFuncGetAttributes(&fa, reduce_left_update_kernel));
  BR_CUDA(cudaFuncGetAttributes(&fa, reduce_right_update_kernel));
  BR_CUDA(cudaFuncGetAttributes(&fa, cyc_fold_kernel));
  return 0;
}

}  // namespace br
