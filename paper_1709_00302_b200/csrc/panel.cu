// Householder panel factorization (QR, and LQ through a transposed view).
//
// Reference semantics (ref kernels.py:86-110, 152-208, 211-255):
//   * reflector per column with beta = -sign(x0)*||x||, x0 == 0 counted as
//     positive, applied even when the tail is zero (tau = 2); the zero
//     column gives tau = beta = 0 and v = e_i (identity, no update);
//   * compact WY with Q = H_0 ... H_{b-1} = I + W Y^T, W = Y T, T = -T_larft.
//
// B200 design. A "leaf" is an L x nb (nb <= 32) block held in the REGISTERS
// of one thread-block cluster (<= 16 CTAs x 256 threads, each thread owning
// R rows x NB columns, R*NB = 64 doubles). Each column step needs exactly one
// cluster-wide reduction of an NB-slot vector:
//   slots c >= i   : x^T P_c   (c == i gives ||x||^2)        -> Householder
//   slots c <  i-1 : Y_c^T v_{i-1}  (Gram column of the last reflector) -> T
// computed per thread with FMAs on registers, reduced across the warp with a
// transpose-reduction (each lane ends with one slot; 31 shuffles for 32 slots),
// across warps in shared memory, and across the cluster through DSMEM after
// one barrier.cluster (buffers double-buffered). Every CTA sums the partials in
// the same fixed order, so all CTAs hold bit-identical scalars; then
//     v^T P_c = (x^T P_c - beta * P_ic) / (x0 - beta)
// gives the rank-1 update of every owned row without a second reduction.
// Rows above the diagonal are moved out of the registers as soon as they are
// final (R entries), so the registers always hold Y with an explicit unit
// diagonal and zeros above it and no per-element masking is needed.
// T follows the reference recurrence from the Gram columns; W = Y T is formed
// from the registers. Panels wider than the leaf are processed right-looking:
// leaf, then the block reflector of that leaf is applied to the rest of the
// panel with DMMA GEMMs, and the full T is assembled from the Gram matrix.
#include <algorithm>

#include "driver.cuh"
#include "gemm.cuh"

namespace br {

constexpr int LEAF_NB = 32;   // max leaf width
constexpr int LT = 256;       // threads per CTA
constexpr int LW = LT / 32;   // warps per CTA
constexpr int LEAF_MAXC = 16; // max cluster size (non-portable)

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
};

// Transpose-reduce RC values across a warp: afterwards v[0] of lane l holds
// the warp total of slot (l / (32/RC)). Fixed summation tree (deterministic).
template <int RC>
__device__ __forceinline__ void warp_transpose_reduce(double (&v)[RC], int lane) {
  int n = RC;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (n > 1) {
      const bool up = (lane & o) != 0;
      const int h = n / 2;
#pragma unroll
      for (int q = 0; q < RC / 2; ++q) {
        if (q < h) {
          const double send = up ? v[q] : v[q + h];
          const double keep = up ? v[q + h] : v[q];
          v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      n = h;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}

// One leaf. Thread t of CTA q owns rows q*LT*R + t + k*LT (k < R). Registers
// hold the active columns ROTATED: p[k][0] is always the current column i,
// p[k][c'] is column i + c'. The rank-1 update writes p[k][c'] from
// p[k][c'+1], so the rotation costs no extra instructions and x = p[k][0]
// needs no select. Finished Y columns go to shared memory (Ys), finished R
// rows to Rrow. Slots of the reduced vector:
//   c' <  NB - i      : x^T P_{i+c'}            (c' = 0 gives ||x||^2)
//   c' >= NB - i      : Gram entry (c' - NB + i, i - 1) = Y_c^T v_{i-1}
// Partials are pushed into every CTA's receive buffer with DSMEM stores
// before the cluster barrier, so the reads after it are local.
template <int NB, int R>
__global__ void __launch_bounds__(LT, 1) leaf_reg_kernel(const LeafArgs a) {
  constexpr int RC = NB < 16 ? NB : 16;  // slots per transpose-reduce chunk
  constexpr int NCH = NB / RC;
  constexpr int SH = 32 / RC;  // lanes holding the same reduced slot
  constexpr int ROWS = LT * R;  // rows per CTA
  extern __shared__ __align__(16) double Ys[];  // [NB][ROWS]
  __shared__ double wred[LW][NB];
  __shared__ double recv[2][LEAF_MAXC][NB][2];
  __shared__ double rowi[NB];
  __shared__ double alpha_s[NB];
  __shared__ double scal[NB][3];  // tau, beta, rinv
  __shared__ double G[NB][NB + 1];
  __shared__ double Ts[NB][NB + 1];
  __shared__ double Rrow[NB][NB + 1];

  const uint32_t rank = cluster_ctarank(), ncta = cluster_nctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = a.nb;
  const int64_t base = (int64_t)rank * ROWS;

  int64_t gr[R];
  double p[R][NB];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    gr[k] = base + tid + (int64_t)k * LT;
    const bool valid = gr[k] < a.L;
#pragma unroll
    for (int c = 0; c < NB; ++c) p[k][c] = (valid && c < nb) ? *a.P.at(gr[k], c) : 0.0;
  }
  if (tid < NB) rowi[tid] = 0.0;
  __syncthreads();

  double vprev[R];
#pragma unroll
  for (int k = 0; k < R; ++k) vprev[k] = 0.0;

  for (int i = 0; i <= nb; ++i) {
    const bool hh = i < nb;  // i == nb: final round, Gram column nb-1 only
    const int buf = i & 1;
    const int g0 = NB - i;   // first Gram slot
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (hh && gr[k] == i) {
#pragma unroll
        for (int c = 0; c < NB; ++c) rowi[c] = p[k][c];
      }
    // ---- per-thread partials, transpose-reduced per warp ----
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      double v[RC];
#pragma unroll
      for (int cc = 0; cc < RC; ++cc) {
        const int c = ch * RC + cc;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) s = fma(p[k][0], p[k][c], s);
        if (c >= g0 && c < NB - 1) {  // Gram entry (c - g0, i - 1)
#pragma unroll
          for (int k = 0; k < R; ++k) s = fma(vprev[k], Ys[(c - g0) * ROWS + tid + k * LT], s);
        }
        v[cc] = s;
      }
      warp_transpose_reduce<RC>(v, lane);
      if ((lane & (SH - 1)) == 0) wred[warp][ch * RC + lane / SH] = v[0];
    }
    __syncthreads();
    if (warp == 0 && lane < NB) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < LW; ++w) s += wred[w][lane];
      const double rv = rowi[lane];
      rowi[lane] = 0.0;
      for (uint32_t q = 0; q < ncta; ++q) {
        const uint32_t ad = map_cluster(&recv[buf][rank][lane][0], q);
        st_cluster_f64(ad, s);
        st_cluster_f64(ad + 8, rv);
      }
    }
    cluster_sync_all();
    if (warp == 0) {
      double g = 0.0, pic = 0.0;
      if (lane < NB) {
        for (uint32_t q = 0; q < ncta; ++q) {
          g += recv[buf][q][lane][0];
          pic += recv[buf][q][lane][1];
        }
      }
      if (i > 0 && lane >= g0 && lane < NB - 1) G[lane - g0][i - 1] = g;
      if (hh) {
        const double nrm2 = __shfl_sync(0xffffffffu, g, 0);
        const double x0 = __shfl_sync(0xffffffffu, pic, 0);
        const double nrm = sqrt(nrm2);
        double tau = 0.0, beta = 0.0, rinv = 0.0;
        if (nrm != 0.0) {
          const double sign = (x0 < 0.0) ? -1.0 : 1.0;
          beta = -sign * nrm;
          const double v0 = x0 - beta;
          tau = (beta - x0) / beta;
          rinv = 1.0 / v0;
        }
        if (lane < NB)
          alpha_s[lane] = (lane >= 1 && lane < nb - i) ? tau * ((g - beta * pic) * rinv) : 0.0;
        if (lane == 0) {
          scal[i][0] = tau;
          scal[i][1] = beta;
          scal[i][2] = rinv;
        }
      }
    }
    __syncthreads();
    if (hh) {
      const double rinv = scal[i][2];
      double al[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) al[c] = alpha_s[c];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const double vk = (gr[k] == i) ? 1.0 : p[k][0] * rinv;
        Ys[i * ROWS + tid + k * LT] = vk;  // Y column i (unit diagonal, zeros above)
        vprev[k] = vk;
#pragma unroll
        for (int c = 0; c < NB - 1; ++c) p[k][c] = fma(-vk, al[c + 1], p[k][c + 1]);
        p[k][NB - 1] = 0.0;
        if (gr[k] == i) {  // row i is final: move its R entries (columns i+1..) out
#pragma unroll
          for (int c = 0; c < NB - 1; ++c) {
            if (c < nb - 1 - i) Rrow[i][i + 1 + c] = p[k][c];
            p[k][c] = 0.0;
          }
        }
      }
    }
  }
  cluster_sync_all();  // all DSMEM traffic done before any CTA may exit

  // ---- T by the reference recurrence (ref kernels.py:152-162), one row per lane ----
  if (warp == 0 && lane < nb) {
    const int r = lane;
    for (int c = 0; c < NB; ++c) Ts[r][c] = 0.0;
    Ts[r][r] = -scal[r][0];
    for (int i = r + 1; i < nb; ++i) {
      double s0 = 0.0, s1 = 0.0;
      int c = r;
      for (; c + 1 < i; c += 2) {
        s0 = fma(Ts[r][c], G[c][i], s0);
        s1 = fma(Ts[r][c + 1], G[c + 1][i], s1);
      }
      if (c < i) s0 = fma(Ts[r][c], G[c][i], s0);
      Ts[r][i] = -scal[i][0] * (s0 + s1);
    }
  }
  __syncthreads();

  // ---- outputs: Y, R, W = Y T, tau, T ----
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (gr[k] >= a.L) continue;
    const int lr = tid + k * LT;
    for (int c = 0; c < nb; ++c) a.Y[gr[k] + (int64_t)c * a.ldy] = Ys[c * ROWS + lr];
    if (gr[k] < nb) {
      const int r = (int)gr[k];
      for (int c = r; c < nb; ++c) *a.P.at(r, c) = (c == r) ? scal[r][1] : Rrow[r][c];
    }
    if (a.W) {
      double y[NB];
#pragma unroll
      for (int m = 0; m < NB; ++m) y[m] = (m < nb) ? Ys[m * ROWS + lr] : 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        if (c >= nb) continue;
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < NB; ++m)
          if (m <= c) s = fma(y[m], Ts[m][c], s);
        a.W[gr[k] + (int64_t)c * a.ldw] = s;
      }
    }
  }
  if (rank == 0) {
    if (tid < nb) a.tau[tid] = scal[tid][0];
    if (a.T)
      for (int q = tid; q < nb * nb; q += LT) {
        const int r = q % nb, c = q / nb;
        a.T[r + (int64_t)c * a.ldt] = Ts[r][c];
      }
  }
}

// rows one cluster holds at leaf width nb: 16 CTAs x 256 threads x R rows
static int leaf_rows_per_thread(int nb) { return nb > 16 ? 2 : (nb > 8 ? 4 : 8); }
static int64_t leaf_capacity(int nb) { return (int64_t)LEAF_MAXC * LT * leaf_rows_per_thread(nb); }

// Leaf width for a j x b panel: the widest of {32, 16, 8} (or b if narrower)
// whose L rows fit one cluster.
static int leaf_width(int64_t L, int64_t b) {
  const int cand[3] = {32, 16, 8};
  for (int nb : cand) {
    const int use = (int)std::min<int64_t>(nb, b);
    if (L <= leaf_capacity(use)) return use;
  }
  return -1;
}

template <int NB, int R>
static int launch_leaf_t(cudaStream_t st, const LeafArgs& a, int C) {
  auto kern = leaf_reg_kernel<NB, R>;
  const size_t smem = (size_t)NB * LT * R * sizeof(double);
  static int attr_dev_mask = 0;
  int dev = 0;
  BR_CUDA(cudaGetDevice(&dev));
  if (!(attr_dev_mask & (1 << dev))) {
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_dev_mask |= (1 << dev);
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(LT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  count_launch();
  BR_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return 0;
}

static int launch_leaf(cudaStream_t st, MatView P, MatView Y, double* tau, double* T, int64_t ldt,
                       MatView* W) {
  const int64_t L = P.rows;
  const int nb = (int)P.cols;
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
  auto csize = [&](int64_t rows_per_cta) {
    int C = 1;
    while (C < cdiv(L, rows_per_cta)) C *= 2;
    return C;
  };
  if (nb > 16) {
    if (L <= (int64_t)LEAF_MAXC * LT) return launch_leaf_t<32, 1>(st, a, csize(LT));
    return launch_leaf_t<32, 2>(st, a, csize(2 * LT));
  }
  if (nb > 8) {
    if (L <= (int64_t)LEAF_MAXC * LT) return launch_leaf_t<16, 1>(st, a, csize(LT));
    return launch_leaf_t<16, 4>(st, a, csize(4 * LT));
  }
  if (L <= (int64_t)LEAF_MAXC * LT) return launch_leaf_t<8, 1>(st, a, csize(LT));
  return launch_leaf_t<8, 8>(st, a, csize(8 * LT));
}

// T from the Gram matrix, blocked: diagonal 32x32 blocks by the reference
// recurrence, then T[0:s, s:e] = T[0:s,0:s] * G[0:s, s:e] * T[s:e, s:e].
// One CTA; b <= 256 keeps everything in L2-resident global scratch.
__global__ void t_diag_kernel(const double* G, int64_t ldg, const double* tau, int64_t b,
                              double* T, int64_t ldt) {
  // one warp per 32-column diagonal block
  const int lane = threadIdx.x & 31, blk = threadIdx.x >> 5;
  const int64_t s = (int64_t)blk * 32;
  if (s >= b) return;
  const int nb = (int)std::min<int64_t>(32, b - s);
  for (int i = 0; i < nb; ++i) {
    const double ti = tau[s + i];
    if (lane < i) {
      double acc = 0.0;
      for (int c = lane; c < i; ++c) acc = fma(T[(s + lane) + (s + c) * ldt], G[(s + c) + (s + i) * ldg], acc);
      T[(s + lane) + (s + i) * ldt] = -ti * acc;
    }
    if (lane == i) T[(s + i) + (s + i) * ldt] = -ti;
    __syncwarp();
  }
}

int t_from_gram(cudaStream_t st, const double* G, int64_t ldg, const double* tau, int64_t b,
                double* T, int64_t ldt) {
  // caller zero-fills T
  const int nblk = (int)cdiv(b, 32);
  count_launch();
  t_diag_kernel<<<1, 32 * nblk, 0, st>>>(G, ldg, tau, b, T, ldt);
  BR_CUDA(cudaGetLastError());
  return 0;
}

int64_t panel_scratch_doubles(int64_t b) { return b * b + LEAF_NB * LEAF_NB + 2 * LEAF_NB * b; }

int panel_qr(cudaStream_t st, Scratch& ws, DevBuf& pscratch, MatView P, MatView Y, double* tau,
             MatView T, MatView* W) {
  const int64_t j = P.rows, b = P.cols;
  if (j < b || b < 1) {
    set_error("panel_qr needs j >= b >= 1, got %lld x %lld", (long long)j, (long long)b);
    return -1;
  }
  const int nbl = leaf_width(j, b);
  if (nbl < 1) {
    set_error("panel_qr: %lld rows exceed one cluster's register capacity (%lld)", (long long)j,
              (long long)leaf_capacity(8));
    return -1;
  }
  if (b <= nbl) {
    // single leaf: Y, tau, T and W in one kernel
    return launch_leaf(st, P, Y, tau, T.p, T.ld, W);
  }
  // multi-leaf, right-looking
  BR_CHECK(zero_fill(st, Y));
  BR_CHECK(zero_fill(st, T));
  if (pscratch.cap < panel_scratch_doubles(b)) {
    set_error("panel_qr: panel scratch too small");
    return -1;
  }
  double* scratch = pscratch.p;  // [G b x b][Tblk 32x32][Z 32 x b][Z2 32 x b]
  MatView G(scratch, b, b, b);
  double* tblk = scratch + b * b;
  MatView Z(tblk + LEAF_NB * LEAF_NB, LEAF_NB, LEAF_NB, b);
  MatView Z2(Z.p + LEAF_NB * b, LEAF_NB, LEAF_NB, b);
  for (int64_t s = 0; s < b; s += nbl) {
    const int64_t e = std::min<int64_t>(s + nbl, b);
    const int64_t w = e - s;
    const int64_t Ls = j - std::max<int64_t>(s, 0);
    MatView leafP = P.sub(s, s, j - s, w);
    MatView leafY = Y.sub(s, s, j - s, w);
    // leaf width may need re-evaluation as rows shrink
    BR_CHECK(launch_leaf(st, leafP, leafY, tau + s, tblk, LEAF_NB, nullptr));
    (void)Ls;
    if (e < b) {
      // P[s:, e:b] += Y_blk (T_blk^T (Y_blk^T P[s:, e:b]))
      MatView rest = P.sub(s, e, j - s, b - e);
      MatView Zs = Z.sub(0, 0, w, b - e), Z2s = Z2.sub(0, 0, w, b - e);
      MatView Tb(tblk, LEAF_NB, w, w);
      BR_CHECK(gemm(st, ws, Zs, leafY.T(), rest, 1.0, 0.0));
      BR_CHECK(gemm(st, ws, Z2s, Tb.T(), Zs, 1.0, 0.0));
      BR_CHECK(gemm(st, ws, rest, leafY, Z2s, 1.0, 1.0));
    }
  }
  // full T: Gram, blocked recurrence
  BR_CHECK(gemm(st, ws, G, Y.T(), Y, 1.0, 0.0));
  BR_CHECK(t_from_gram(st, G.p, G.ld, tau, b, T.p, T.ld));
  for (int64_t s = 32; s < b; s += 32) {
    const int64_t e = std::min<int64_t>(s + 32, b);
    // T[0:s, s:e] = T[0:s,0:s] * (G[0:s, s:e] * T[s:e, s:e])
    MatView tmp(Z.p, s, s, e - s);  // s x (e-s) scratch (fits: 32*b >= s*32)
    BR_CHECK(gemm(st, ws, tmp, G.sub(0, s, s, e - s), T.sub(s, s, e - s, e - s), 1.0, 0.0));
    BR_CHECK(gemm(st, ws, T.sub(0, s, s, e - s), T.sub(0, 0, s, s), tmp, 1.0, 0.0));
  }
  if (W) BR_CHECK(gemm(st, ws, *W, Y, T, 1.0, 0.0));
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

}  // namespace br
