// DMMA GEMM kernel template (shared by the per-tile-config instantiation units).
// See gemm.cuh for the contract.
#pragma once
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

// Per-thread cp.async plan for one operand tile, set up once per CTA
// (CUTLASS-style iterator): each thread owns IT 16-byte chunks at a fixed
// shared-memory offset whose global pointers advance by a constant per
// k-tile, so the main loop issues cp.async with no per-chunk index math.
// The tile is TX (contiguous, 2 doubles per chunk) x TY (stride ld); KX says
// whether K runs along x (A^T, B) or along y (A, B^T). Bounds of the fixed
// dimension are folded into per-chunk byte counts once; the K bound is only
// checked on a partial last k-tile. A second K source (src2 from ksplit on,
// the [X3 | Y] operand of SYR2K) is switched to at its k-tile boundary.
template <int TX, int TY, int LD, int NT, bool KX>
struct TileIter {
  static constexpr int CX = TX / 2;     // chunks per y line
  static constexpr int YS = NT / CX;    // y distance between a thread's chunks
  static constexpr int IT = CX * TY / NT;
  static_assert(NT % CX == 0 && (CX * TY) % NT == 0, "tile / thread count mismatch");
  const double* p[IT];
  uint32_t bytes;  // 2 bits per chunk: 0, 1 (8 B) or 2 (16 B) for the fixed dimension
  int xt, yt;      // this thread's first chunk (x, y) in the tile
  int64_t step;    // pointer advance per k-tile

  __device__ __forceinline__ void init(const double* src, int64_t ld, int64_t x0, int64_t xmax,
                                       int64_t y0, int64_t ymax, int tid) {
    xt = (tid % CX) * 2;
    yt = tid / CX;
    bytes = 0;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int64_t gx = x0 + xt, gy = y0 + yt + it * YS;
      p[it] = src + gx + gy * ld;
      uint32_t bc;
      if (KX) bc = gy < ymax ? 2u : 0u;  // K (x) bound checked per k-tile
      else bc = gx < xmax ? (gx + 1 < xmax ? 2u : 1u) : 0u;
      bytes |= bc << (2 * it);
    }
    step = KX ? (int64_t)TX : (int64_t)TY * ld;
  }
  // Re-base on a second K source (y-K only): y coordinate k0 of the tile is
  // row k0 - ksplit of src2.
  __device__ __forceinline__ void rebase(const double* src2, int64_t ld2, int64_t x0,
                                         int64_t krow) {
#pragma unroll
    for (int it = 0; it < IT; ++it) p[it] = src2 + (x0 + xt) + (krow + yt + it * YS) * ld2;
    step = (int64_t)TY * ld2;
  }
  __device__ __forceinline__ void advance() {
#pragma unroll
    for (int it = 0; it < IT; ++it) p[it] += step;
  }
  // Issue the tile at K offset k0 (the pointers are already there) into
  // shared memory at dst; `kend` bounds K when the tile is partial.
  __device__ __forceinline__ void load(uint32_t dst, int64_t k0, int64_t kend, bool full) {
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      int nb = (int)((bytes >> (2 * it)) & 3u) * 8;
      if (!full) {
        if (KX) {
          const int64_t kx = k0 + xt;
          nb = kx >= kend ? 0 : (kx + 1 >= kend ? min(nb, 8) : nb);
        } else {
          if (k0 + yt + it * YS >= kend) nb = 0;
        }
      }
      cp_async16_u32(dst + (uint32_t)(((yt + it * YS) * LD + xt) * 8), p[it], nb);
      p[it] += step;
    }
  }
};

// Which layout a SYMM K-tile uses: 0 = strictly lower (direct, [k][m]),
// 1 = strictly upper (transposed read of the lower triangle, [m][k]),
// 2 = straddles the diagonal (element-wise select, [k][m]).
__device__ __forceinline__ int sym_case(int64_t k0, int64_t m0, int BK, int BM) {
  if (k0 + BK <= m0) return 0;
  if (k0 >= m0 + BM) return 1;
  return 2;
}

// Compile-time variants of a tile (FL bit mask; 0 for every hot-path
// instantiation, so those compile exactly as without the variants):
//   GF_CYC: the block-cyclic staircase map of GemmArgs.cyc_* (dist.py),
//   GF_NOTRIG: no early PDL trigger (persistent callers, xchain.cu).
enum GemmFlags { GF_CYC = 1, GF_NOTRIG = 2 };

// One output tile (bx, by) of K-split bz.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, int AM, int BMD, int EPI,
          int FL = 0>
__device__ __forceinline__ void dgemm_tile(const GemmArgs& g, const unsigned bx, const unsigned by,
                                           const unsigned bz) {
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
  constexpr bool cyc = (FL & GF_CYC) != 0;
  if (EPI == EPI_LOWER) {
    if constexpr (cyc) {
      m0 = g.cyc_r0 + (int64_t)bx * BM;
      n0 = g.c0 + (int64_t)by * BN;
      if (m0 + BM <= cyc_map(g, n0)) return;  // tile above the staircase
    } else {
      if (bx < by) return;
      m0 = g.c0 + (int64_t)bx * BM;
      n0 = g.c0 + (int64_t)by * BN;
    }
    kbeg = 0;
    kend = g.K;
  } else {
    m0 = (int64_t)bx * BM;
    n0 = (int64_t)by * BN;
    kbeg = (int64_t)bz * g.k_per_split;
    kend = min(g.K, kbeg + g.k_per_split);
    if (BMD == B_N && g.b_upper) kend = max(kbeg, min(kend, n0 + BN));  // rows > n of B are 0
    if constexpr (cyc) {  // block-cyclic staircase operand: skip its all-zero K range
      if (AM == A_N) kend = max(kbeg, min(kend, cyc_count(g, m0 + BM - 1)));
      else if (AM == A_T) kbeg = min(kend, max(kbeg, cyc_map(g, m0) & ~(int64_t)1));
    }
  }
  const int64_t nmax = (EPI == EPI_LOWER) ? g.c1 : g.N;
  pdl_wait();  // inputs written by the previous kernel in the stream

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
  // EPI_LOWER with the block-cyclic map: first row written in each of this
  // thread's columns (the column's global index), formed once per thread;
  // without the map the test is r >= c, as before the map existed
  int64_t cthr[cyc ? NI : 1][2];
  if constexpr (EPI == EPI_LOWER && cyc) {
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) cthr[j][h] = cyc_map(g, n0 + wn + j * 8 + 2 * tq + h);
  }
#define BR_LOWER_OK(r, c, j, h) (cyc ? ((r) >= cthr[cyc ? (j) : 0][h]) : ((r) >= (c)))
  if (cpre) {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int64_t r = m0 + wm + i * 8 + gq;
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t c = n0 + wn + j * 8 + 2 * tq + h;
          const bool ok = r < g.M && c < nmax && (EPI != EPI_LOWER || BR_LOWER_OK(r, c, j, h));
          if (ok) acc[i][j][h] = (EPI == EPI_LOWER || g.beta == 1.0)
                                     ? g.Cin[r + c * g.ldcin]
                                     : g.beta * g.Cin[r + c * g.ldcin];
        }
    }
  }

  const bool vA = g.vecA != 0, vB = g.vecB != 0;
  // fast iterators (16-byte aligned operands; a second K source only at a
  // k-tile boundary)
  using ItA = TileIter<(AM == A_T ? BK : BM), (AM == A_T ? BM : BK),
                       (AM == A_T ? LDA_MK : LDA_KM), NT, AM == A_T>;
  using ItB = TileIter<(BMD == B_N ? BK : BN), (BMD == B_N ? BN : BK),
                       (BMD == B_N ? LDB_NK : LDB_KN), NT, BMD == B_N>;
  const bool fastA = AM != A_SYM && vA && (g.ksplitA == INT64_MAX || (g.ksplitA - kbeg) % BK == 0);
  const bool fastB = vB && (g.ksplitB == INT64_MAX || (g.ksplitB - kbeg) % BK == 0);
  ItA ia;
  ItB ib;
  if (AM != A_SYM && fastA) {
    if (AM == A_T) ia.init(g.A, g.lda, kbeg, kend, m0, g.M, tid);
    else if (kbeg >= g.ksplitA) {
      ia.init(g.A2, g.lda2, m0, g.M, kbeg - g.ksplitA, INT64_MAX, tid);
    } else {
      ia.init(g.A, g.lda, m0, g.M, kbeg, INT64_MAX, tid);
    }
  }
  if (fastB) {
    if (BMD == B_N) ib.init(g.B, g.ldb, kbeg, kend, n0, g.N, tid);
    else if (kbeg >= g.ksplitB) {
      ib.init(g.B2, g.ldb2, n0, g.N, kbeg - g.ksplitB, INT64_MAX, tid);
    } else {
      ib.init(g.B, g.ldb, n0, g.N, kbeg, INT64_MAX, tid);
    }
  }
  // SYMM: a direct iterator for k-tiles below the diagonal block and a
  // transposed one (reading the stored lower triangle) for k-tiles above it
  using ItSN = TileIter<BM, BK, LDA_KM, NT, false>;
  using ItST = TileIter<BK, BM, LDA_MK, NT, true>;
  const bool fastS = AM == A_SYM && vA;
  ItSN isn;
  ItST ist;
  if (AM == A_SYM && fastS) {
    isn.init(g.A, g.lda, m0, g.M, kbeg, INT64_MAX, tid);
    ist.init(g.A, g.lda, kbeg, kend, m0, g.M, tid);
  }
  const uint32_t as_u32 = smem_u32(As), bs_u32 = smem_u32(Bs);
  auto load_stage = [&](int s, int64_t k0) {
    double* as = As + s * A_STAGE;
    double* bs = Bs + s * B_STAGE;
    const bool full = k0 + BK <= kend;
    if (AM != A_SYM && fastA) {
      if (AM == A_N && k0 == g.ksplitA && k0 != kbeg) ia.rebase(g.A2, g.lda2, m0, 0);
      ia.load(as_u32 + (uint32_t)(s * A_STAGE * 8), k0, kend, full);
    } else if (AM == A_N) {
      load_tile<BM, BK, LDA_KM, NT>(as, g.A, g.lda, g.A2, g.lda2, g.ksplitA, m0, g.M, k0, kend, vA,
                                    tid);
    } else if (AM == A_T) {
      load_tile<BK, BM, LDA_MK, NT>(as, g.A, g.lda, g.A, g.lda, INT64_MAX, k0, kend, m0, g.M, vA,
                                    tid);
    } else if (fastS && sym_case(k0, m0, BK, BM) != 2) {
      const uint32_t dst = as_u32 + (uint32_t)(s * A_STAGE * 8);
      if (sym_case(k0, m0, BK, BM) == 0) {
        isn.load(dst, k0, kend, full);
        ist.advance();
      } else {
        ist.load(dst, k0, kend, full);
        isn.advance();
      }
    } else {
      if (fastS) {
        isn.advance();
        ist.advance();
      }
      const int c = sym_case(k0, m0, BK, BM);
      if (c == 0) {
        load_tile<BM, BK, LDA_KM, NT>(as, g.A, g.lda, g.A, g.lda, INT64_MAX, m0, g.M, k0, kend, vA,
                                      tid);
      } else if (c == 1) {
        load_tile<BK, BM, LDA_MK, NT>(as, g.A, g.lda, g.A, g.lda, INT64_MAX, k0, kend, m0, g.M, vA,
                                      tid);
      } else {
        // diagonal k-tile: element (m, k) from the stored lower triangle; the
        // loads are issued in batches (independent) before the shared stores
        constexpr int PER = BK * BM / NT;
        double v[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int idx = tid + u * NT;
          const int k = idx / BM, m = idx % BM;
          const int64_t r = m0 + m, cc = k0 + k;
          v[u] = (r < g.M && cc < kend) ? __ldg((r >= cc) ? &g.A[r + cc * g.lda]
                                                          : &g.A[cc + r * g.lda])
                                        : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int idx = tid + u * NT;
          as[(idx / BM) * LDA_KM + idx % BM] = v[u];
        }
      }
    }
    if (fastB) {
      if (BMD == B_T && k0 == g.ksplitB && k0 != kbeg) ib.rebase(g.B2, g.ldb2, n0, 0);
      ib.load(bs_u32 + (uint32_t)(s * B_STAGE * 8), k0, kend, full);
    } else if (BMD == B_N) {
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
  if constexpr (!(FL & GF_NOTRIG)) pdl_trigger();  // the next kernel may start launching during the epilogue

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
          g.ws[((int64_t)bz * g.N + c) * g.M + r] = v;
        } else {
          if (BR_LOWER_OK(r, c, j, h)) g.C[r + c * g.ldc] = v;
        }
      }
    }
  }
#undef BR_LOWER_OK
}



// One CTA per tile.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, int AM, int BMD, int EPI,
          int FL = 0>
__global__ void __launch_bounds__(WM* WN * 32, MINB) dgemm_kernel(const GemmArgs g) {
  dgemm_tile<BM, BN, BK, WM, WN, STAGES, MINB, AM, BMD, EPI, FL>(g, blockIdx.x, blockIdx.y, blockIdx.z);
}

template <int BM, int BN, int BK, int STAGES, int AM, int BMD>
constexpr int smem_bytes() {
  constexpr int LDA_KM = BM + 4, LDA_MK = BK + 4;
  constexpr int A_STAGE = (AM == A_N)   ? BK * LDA_KM
                          : (AM == A_T) ? BM * LDA_MK
                                        : (BK * LDA_KM > BM * LDA_MK ? BK * LDA_KM : BM * LDA_MK);
  constexpr int B_STAGE = (BMD == B_N) ? BN * (BK + 4) : BK * (BN + 4);
  return STAGES * (A_STAGE + B_STAGE) * 8;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, int AM, int BMD, int EPI,
          int FL = 0>
static int launch(cudaStream_t st, const GemmArgs& g, dim3 grid) {
  constexpr int smem = smem_bytes<BM, BN, BK, STAGES, AM, BMD>();
  auto kern = dgemm_kernel<BM, BN, BK, WM, WN, STAGES, MINB, AM, BMD, EPI, FL>;
  static std::atomic<int> attr_dev_mask{0};  // per-instantiation, per-device
  int dev = 0;
  BR_CUDA(cudaGetDevice(&dev));
  if (!(attr_dev_mask.load() & (1 << dev))) {
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_dev_mask.fetch_or(1 << dev);
  }
  if (g_preload_only) return (int)launch_pdl(kern, grid, dim3(WM * WN * 32), smem, st, g);
  count_launch();
  BR_CUDA(launch_pdl(kern, grid, dim3(WM * WN * 32), smem, st, g));
  return 0;
}

// Instantiates one tile configuration for every (A mode, B mode, epilogue)
// the dispatcher uses; LOWER (SYR2K) only for square tiles.
#define BR_DEFINE_TILE(NAME, BM, BN, BK, WM, WN, STAGES, MINB)                                  \
  int NAME(int am, int bmd, int epi, cudaStream_t st, const GemmArgs& g, dim3 grid) {          \
    if (epi == EPI_LOWER) {                                                                     \
      if constexpr (BM == BN) return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_N, B_T, EPI_LOWER>(st, g, grid); \
      set_error("LOWER epilogue needs a square tile");                                         \
      return -1;                                                                               \
    }                                                                                          \
    if (am == A_SYM) {                                                                         \
      if (epi == EPI_GEN) return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_SYM, B_N, EPI_GEN>(st, g, grid); \
      return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_SYM, B_N, EPI_SPLIT>(st, g, grid);    \
    }                                                                                          \
    if (am == A_N) {                                                                           \
      if (bmd == B_N) {                                                                        \
        if (epi == EPI_GEN) return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_N, B_N, EPI_GEN>(st, g, grid); \
        return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_N, B_N, EPI_SPLIT>(st, g, grid);    \
      }                                                                                        \
      if (epi == EPI_GEN) return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_N, B_T, EPI_GEN>(st, g, grid); \
      return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_N, B_T, EPI_SPLIT>(st, g, grid);      \
    }                                                                                          \
    if (bmd == B_N) {                                                                          \
      if (epi == EPI_GEN) return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_T, B_N, EPI_GEN>(st, g, grid); \
      return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_T, B_N, EPI_SPLIT>(st, g, grid);      \
    }                                                                                          \
    if (epi == EPI_GEN) return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_T, B_T, EPI_GEN>(st, g, grid); \
    return launch<BM, BN, BK, WM, WN, STAGES, MINB, A_T, B_T, EPI_SPLIT>(st, g, grid);        \
  }

}  // namespace br
