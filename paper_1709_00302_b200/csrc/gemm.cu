// DMMA GEMM / SYMM / SYR2K kernels (see gemm.cuh for the contract).
#include <algorithm>

#include "driver.cuh"
#include "gemm.cuh"

namespace br {

// Load a TX x TY tile of a column-major region into shared memory:
// element (x, y) lives at src + x + y*ld (or src2 + x + (y-ysplit)*ld2 for
// y >= ysplit) and goes to dst[y*LD + x]. Out-of-range elements read as 0.
template <int TX, int TY, int LD, int NT>
__device__ __forceinline__ void load_tile(double* dst, const double* src, int64_t ld,
                                          const double* src2, int64_t ld2, int64_t ysplit,
                                          int64_t x0, int64_t xmax, int64_t y0, int64_t ymax,
                                          bool vec2, int tid) {
  if (vec2) {
    constexpr int CX = TX / 2;
#pragma unroll 4
    for (int idx = tid; idx < CX * TY; idx += NT) {
      const int y = idx / CX, x = (idx % CX) * 2;
      const int64_t gx = x0 + x, gy = y0 + y;
      const double* s = src;
      int bytes = 0;
      if (gy < ymax && gx < xmax) {
        s = gy < ysplit ? src + gx + gy * ld : src2 + gx + (gy - ysplit) * ld2;
        bytes = (gx + 1 < xmax) ? 16 : 8;
      }
      cp_async16(dst + y * LD + x, s, bytes);
    }
  } else {
#pragma unroll 4
    for (int idx = tid; idx < TX * TY; idx += NT) {
      const int y = idx / TX, x = idx % TX;
      const int64_t gx = x0 + x, gy = y0 + y;
      const double* s = src;
      int bytes = 0;
      if (gy < ymax && gx < xmax) {
        s = gy < ysplit ? src + gx + gy * ld : src2 + gx + (gy - ysplit) * ld2;
        bytes = 8;
      }
      cp_async8(dst + y * LD + x, s, bytes);
    }
  }
}

// Which layout a SYMM K-tile uses: 0 = strictly lower (direct, [k][m]),
// 1 = strictly upper (transposed read of the lower triangle, [m][k]),
// 2 = straddles the diagonal (element-wise select, [k][m]).
__device__ __forceinline__ int sym_case(int64_t k0, int64_t m0, int BK, int BM) {
  if (k0 + BK <= m0) return 0;
  if (k0 >= m0 + BM) return 1;
  return 2;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int AM, int BMD, int EPI>
__global__ void __launch_bounds__(WM* WN * 32) dgemm_kernel(const GemmArgs g) {
  constexpr int NT = WM * WN * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN, MI = WTM / 8, NI = WTN / 8;
  constexpr int LDA_KM = BM + 4, LDA_MK = BK + 4;
  constexpr int A_STAGE = (AM == A_N)   ? BK * LDA_KM
                          : (AM == A_T) ? BM * LDA_MK
                                        : (BK * LDA_KM > BM * LDA_MK ? BK * LDA_KM : BM * LDA_MK);
  constexpr int LDB_NK = BK + 4, LDB_KN = BN + 4;
  constexpr int B_STAGE = (BMD == B_N) ? BN * LDB_NK : BK * LDB_KN;
  static_assert(MI * 8 == WTM && NI * 8 == WTN, "warp tile must be a multiple of 8");

  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = (warp % WM) * WTM, wn = (warp / WM) * WTN;

  int64_t m0, n0, kbeg, kend;
  if (EPI == EPI_LOWER) {
    if (blockIdx.x < blockIdx.y) return;
    m0 = g.c0 + (int64_t)blockIdx.x * BM;
    n0 = g.c0 + (int64_t)blockIdx.y * BN;
    kbeg = 0;
    kend = g.K;
  } else {
    m0 = (int64_t)blockIdx.x * BM;
    n0 = (int64_t)blockIdx.y * BN;
    kbeg = (int64_t)blockIdx.z * g.k_per_split;
    kend = min(g.K, kbeg + g.k_per_split);
  }
  const int64_t nmax = (EPI == EPI_LOWER) ? g.c1 : g.N;

  // Accumulators start from beta*C when alpha == 1 (every rank-b update and
  // the SYR2K): the C tile is fetched in one batch before the main loop
  // instead of load->store pairs in the epilogue, which serialize on the
  // possible C/Cin aliasing and leave the tensor pipe idle.
  const bool cpre = (EPI == EPI_LOWER) || (EPI == EPI_GEN && g.alpha == 1.0 && g.beta != 0.0);
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (cpre) {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = m0 + wm + i * 8 + gq;
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t c = n0 + wn + j * 8 + 2 * tq + h;
          const bool ok = r < g.M && c < nmax && (EPI != EPI_LOWER || r >= c);
          if (ok) acc[i][j][h] = (EPI == EPI_LOWER) ? g.Cin[r + c * g.ldcin]
                                                    : g.beta * g.Cin[r + c * g.ldcin];
        }
    }
  }

  const bool vA = g.vecA != 0, vB = g.vecB != 0;
  auto load_stage = [&](int s, int64_t k0) {
    double* as = As + s * A_STAGE;
    double* bs = Bs + s * B_STAGE;
    if (AM == A_N) {
      load_tile<BM, BK, LDA_KM, NT>(as, g.A, g.lda, g.A2, g.lda2, g.ksplitA, m0, g.M, k0, kend, vA,
                                    tid);
    } else if (AM == A_T) {
      load_tile<BK, BM, LDA_MK, NT>(as, g.A, g.lda, g.A, g.lda, INT64_MAX, k0, kend, m0, g.M, vA,
                                    tid);
    } else {
      const int c = sym_case(k0, m0, BK, BM);
      if (c == 0) {
        load_tile<BM, BK, LDA_KM, NT>(as, g.A, g.lda, g.A, g.lda, INT64_MAX, m0, g.M, k0, kend, vA,
                                      tid);
      } else if (c == 1) {
        load_tile<BK, BM, LDA_MK, NT>(as, g.A, g.lda, g.A, g.lda, INT64_MAX, k0, kend, m0, g.M, vA,
                                      tid);
      } else {
        for (int idx = tid; idx < BK * BM; idx += NT) {
          const int k = idx / BM, m = idx % BM;
          const int64_t r = m0 + m, cc = k0 + k;
          double v = 0.0;
          if (r < g.M && cc < kend) v = (r >= cc) ? g.A[r + cc * g.lda] : g.A[cc + r * g.lda];
          as[k * LDA_KM + m] = v;
        }
      }
    }
    if (BMD == B_N) {
      load_tile<BK, BN, LDB_NK, NT>(bs, g.B, g.ldb, g.B, g.ldb, INT64_MAX, k0, kend, n0, g.N, vB,
                                    tid);
    } else {
      load_tile<BN, BK, LDB_KN, NT>(bs, g.B, g.ldb, g.B2, g.ldb2, g.ksplitB, n0, g.N, k0, kend, vB,
                                    tid);
    }
  };

  auto compute_stage = [&](int s, bool amk) {
    const double* as = As + s * A_STAGE;
    const double* bs = Bs + s * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NI];
      if (amk) {
#pragma unroll
        for (int i = 0; i < MI; ++i) af[i] = as[(wm + i * 8 + gq) * LDA_MK + kk + tq];
      } else {
#pragma unroll
        for (int i = 0; i < MI; ++i) af[i] = as[(kk + tq) * LDA_KM + wm + i * 8 + gq];
      }
#pragma unroll
      for (int j = 0; j < NI; ++j)
        bf[j] = (BMD == B_N) ? bs[(wn + j * 8 + gq) * LDB_NK + kk + tq]
                             : bs[(kk + tq) * LDB_KN + wn + j * 8 + gq];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  };

  const int nkt = (int)cdiv(kend - kbeg, BK);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) load_stage(s, kbeg + (int64_t)s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < nkt) load_stage(nk % STAGES, kbeg + (int64_t)nk * BK);
    cp_async_commit();
    const int64_t k0 = kbeg + (int64_t)kt * BK;
    bool amk = (AM == A_T);
    if (AM == A_SYM) amk = (sym_case(k0, m0, BK, BM) == 1);
    if (AM == A_SYM) {
      if (amk)
        compute_stage(kt % STAGES, true);
      else
        compute_stage(kt % STAGES, false);
    } else {
      compute_stage(kt % STAGES, AM == A_T);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue ----
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int64_t r = m0 + wm + i * 8 + gq;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = n0 + wn + j * 8 + 2 * tq + h;
        if (r >= g.M || c >= nmax) continue;
        const double v = acc[i][j][h];
        if (EPI == EPI_GEN) {
          double out;
          if (cpre) {
            out = v;
          } else {
            out = g.alpha * v;
            if (g.beta != 0.0) out += g.beta * g.Cin[r + c * g.ldcin];
          }
          g.C[r + c * g.ldc] = out;
        } else if (EPI == EPI_SPLIT) {
          g.ws[((int64_t)blockIdx.z * g.N + c) * g.M + r] = v;
        } else {
          if (r >= c) g.C[r + c * g.ldc] = v;
        }
      }
    }
  }
}

// Fixed-order split-K reduction: C = alpha * sum_z ws[z] + beta * Cin.
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int S, const double* __restrict__ ws,
                                     double alpha, double beta, const double* Cin, int64_t ldcin,
                                     double* C, int64_t ldc) {
  const int64_t total = M * N;
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

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int AM, int BMD>
constexpr int smem_bytes() {
  constexpr int LDA_KM = BM + 4, LDA_MK = BK + 4;
  constexpr int A_STAGE = (AM == A_N)   ? BK * LDA_KM
                          : (AM == A_T) ? BM * LDA_MK
                                        : (BK * LDA_KM > BM * LDA_MK ? BK * LDA_KM : BM * LDA_MK);
  constexpr int B_STAGE = (BMD == B_N) ? BN * (BK + 4) : BK * (BN + 4);
  return STAGES * (A_STAGE + B_STAGE) * 8;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int AM, int BMD, int EPI>
static int launch(cudaStream_t st, const GemmArgs& g, dim3 grid) {
  constexpr int smem = smem_bytes<BM, BN, BK, WM, WN, STAGES, AM, BMD>();
  auto kern = dgemm_kernel<BM, BN, BK, WM, WN, STAGES, AM, BMD, EPI>;
  static int attr_dev_mask = 0;  // per-instantiation, per-device
  int dev = 0;
  BR_CUDA(cudaGetDevice(&dev));
  if (!(attr_dev_mask & (1 << dev))) {
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_dev_mask |= 1 << dev;
  }
  count_launch();
  kern<<<grid, WM * WN * 32, smem, st>>>(g);
  BR_CUDA(cudaGetLastError());
  return 0;
}

enum TileCfg { CFG_L = 0, CFG_NS = 1, CFG_MS = 2 };

template <int AM, int BMD, int EPI>
static int launch_cfg(cudaStream_t st, const GemmArgs& g, dim3 grid, int cfg) {
  switch (cfg) {
    case CFG_L: return launch<128, 128, 16, 4, 2, 3, AM, BMD, EPI>(st, g, grid);
    case CFG_NS: return launch<128, 32, 16, 4, 1, 4, AM, BMD, EPI>(st, g, grid);
    default: return launch<32, 128, 16, 1, 4, 4, AM, BMD, EPI>(st, g, grid);
  }
}
static void cfg_tile(int cfg, int& bm, int& bn, int& ctas_per_sm) {
  if (cfg == CFG_L) { bm = 128; bn = 128; ctas_per_sm = 1; }
  else if (cfg == CFG_NS) { bm = 128; bn = 32; ctas_per_sm = 2; }
  else { bm = 32; bn = 128; ctas_per_sm = 2; }
}

static inline bool al16(const void* p, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 2 == 0);
}

// Dispatch a general/symm GEMM: chooses tile config and split-K.
template <int AM>
static int run_gemm(cudaStream_t st, Scratch& ws, GemmArgs g, bool btrans, int max_ctas) {
  if (g.M <= 0 || g.N <= 0) return 0;
  if (g.K <= 0) {  // C = beta*Cin
    g.k_per_split = 1;
    const int64_t total = g.M * g.N;
    int blocks = (int)std::min<int64_t>(cdiv(total, 256), 4096);
    // reuse the reduce kernel with S = 0 partials
    count_launch();
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(g.M, g.N, 0, nullptr, g.alpha, g.beta, g.Cin,
                                                 g.ldcin, g.C, g.ldc);
    BR_CUDA(cudaGetLastError());
    return 0;
  }
  int cfg = CFG_L;
  if (g.N <= 32) cfg = CFG_NS;
  else if (g.M <= 32) cfg = CFG_MS;
  int bm, bn, cps;
  cfg_tile(cfg, bm, bn, cps);
  const int64_t tiles = cdiv(g.M, bm) * cdiv(g.N, bn);
  const int64_t nkt = cdiv(g.K, 16);
  const int sms = ws.num_sms;
  // Split-K factor from a small cost model: waves of resident CTAs times the
  // k-tiles each CTA runs, plus the fixed-order reduction pass. This keeps
  // the last wave from idling most SMs (wave quantization) on the tall-skinny
  // reductions (W^T E, D W_V, X1^T W, Y^T Y).
  const int64_t slots = (max_ctas > 0) ? std::max(1, max_ctas) : (int64_t)sms * cps;
  const double kt_time = (double)cps * bm * bn * 16 * 2 / 251e9;  // one k-tile, one CTA
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
  if (S > 1) {
    const int64_t kps = cdiv(nkt, S) * 16;
    S = cdiv(g.K, kps);
    g.k_per_split = kps;
  } else {
    g.k_per_split = g.K;
  }
  if (max_ctas > 0 && tiles * S > max_ctas) {
    // caller asked to leave SMs free; the grid is still launched in full, the
    // hardware scheduler interleaves (persistent scheduling is a later step)
  }
  dim3 grid((unsigned)cdiv(g.M, bm), (unsigned)cdiv(g.N, bn), (unsigned)S);
  if (S == 1) {
    if (btrans) BR_CHECK((launch_cfg<AM, B_T, EPI_GEN>(st, g, grid, cfg)));
    else BR_CHECK((launch_cfg<AM, B_N, EPI_GEN>(st, g, grid, cfg)));
  } else {
    g.ws = ws.p;
    if (btrans) BR_CHECK((launch_cfg<AM, B_T, EPI_SPLIT>(st, g, grid, cfg)));
    else BR_CHECK((launch_cfg<AM, B_N, EPI_SPLIT>(st, g, grid, cfg)));
    const int64_t total = g.M * g.N;
    int blocks = (int)std::min<int64_t>(cdiv(total, 256), (int64_t)sms * 8);
    count_launch();
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(g.M, g.N, (int)S, ws.p, g.alpha, g.beta,
                                                 g.Cin, g.ldcin, g.C, g.ldc);
    BR_CUDA(cudaGetLastError());
  }
  return 0;
}

int gemm(cudaStream_t st, Scratch& ws, MatView C, MatView A, MatView B, double alpha,
         double beta, const MatView* Cin_, int max_ctas) {
  MatView Cin = Cin_ ? *Cin_ : C;
  if (C.trans) {  // C^T = op(B)^T op(A)^T
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
  GemmArgs g{};
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
  if (A.trans) return run_gemm<A_T>(st, ws, g, B.trans, max_ctas);
  return run_gemm<A_N>(st, ws, g, B.trans, max_ctas);
}

int symm_lower(cudaStream_t st, Scratch& ws, MatView X1, MatView A2, MatView W) {
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
  g.alpha = 1.0;
  g.beta = 0.0;
  g.vecA = al16(A2.p, A2.ld);
  g.vecB = al16(W.p, W.ld);
  return run_gemm<A_SYM>(st, ws, g, false, 0);
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
  dim3 grid((unsigned)cdiv(j - c0, 128), (unsigned)cdiv(c1 - c0, 128), 1);
  return launch<128, 128, 16, 4, 2, 3, A_N, B_T, EPI_LOWER>(st, g, grid);
}

}  // namespace br
