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

template <int NB, int R>
__global__ void __launch_bounds__(LT, 1) leaf_reg_kernel(const LeafArgs a) {
  constexpr int RC = NB < 16 ? NB : 16;  // slots per transpose-reduce chunk
  constexpr int NCH = NB / RC;
  constexpr int SH = 32 / RC;  // lanes holding the same reduced slot
  __shared__ double wred[LW][NB];
  __shared__ double red[2][NB][2];
  __shared__ double rowi[NB];
  __shared__ double alpha_s[NB];
  __shared__ double scal[NB][3];  // tau, beta, rinv
  __shared__ double G[NB][NB + 1];
  __shared__ double Ts[NB][NB + 1];
  __shared__ double Rrow[NB][NB + 1];

  const uint32_t rank = cluster_ctarank(), ncta = cluster_nctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = a.nb;
  const int64_t base = (int64_t)rank * (LT * R);

  int64_t gr[R];
  bool valid[R];
  double p[R][NB];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    gr[k] = base + tid + (int64_t)k * LT;
    valid[k] = gr[k] < a.L;
#pragma unroll
    for (int c = 0; c < NB; ++c) p[k][c] = (valid[k] && c < nb) ? *a.P.at(gr[k], c) : 0.0;
  }
  if (tid < NB) rowi[tid] = 0.0;
  __syncthreads();

  double vprev[R];
#pragma unroll
  for (int k = 0; k < R; ++k) vprev[k] = 0.0;

  for (int i = 0; i <= nb; ++i) {
    const bool hh = i < nb;  // i == nb: final round, Gram column nb-1 only
    const int buf = i & 1;
    double x[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      double xv = 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c == i) xv = p[k][c];
      x[k] = xv;  // rows above i hold 0 in column i already
      if (hh && gr[k] == i) {
#pragma unroll
        for (int c = 0; c < NB; ++c) rowi[c] = p[k][c];
      }
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
        for (int k = 0; k < R; ++k) s = fma((c >= i) ? x[k] : vprev[k], p[k][c], s);
        v[cc] = (c >= i || c < i - 1) ? s : 0.0;
      }
      warp_transpose_reduce<RC>(v, lane);
      if ((lane & (SH - 1)) == 0) wred[warp][ch * RC + lane / SH] = v[0];
    }
    __syncthreads();
    if (warp == 0 && lane < NB) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < LW; ++w) s += wred[w][lane];
      red[buf][lane][0] = s;
      red[buf][lane][1] = rowi[lane];
      rowi[lane] = 0.0;
    }
    cluster_sync_all();
    if (warp == 0) {
      double g = 0.0, pic = 0.0;
      if (lane < NB) {
        for (uint32_t q = 0; q < ncta; ++q) {
          const uint32_t ad = map_cluster(&red[buf][lane][0], q);
          g += ld_cluster_f64(ad);
          pic += ld_cluster_f64(ad + 8);
        }
      }
      if (i > 0 && lane < i - 1) G[lane][i - 1] = g;
      if (hh) {
        const double nrm2 = __shfl_sync(0xffffffffu, g, i);
        const double x0 = __shfl_sync(0xffffffffu, pic, i);
        const double nrm = sqrt(nrm2);
        double tau = 0.0, beta = 0.0, rinv = 0.0;
        if (nrm != 0.0) {
          const double sign = (x0 < 0.0) ? -1.0 : 1.0;
          beta = -sign * nrm;
          const double v0 = x0 - beta;
          tau = (beta - x0) / beta;
          rinv = 1.0 / v0;
        }
        if (lane < NB) alpha_s[lane] = (lane > i && lane < nb) ? tau * ((g - beta * pic) * rinv) : 0.0;
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
        const double vk = (gr[k] == i) ? 1.0 : x[k] * rinv;
#pragma unroll
        for (int c = 0; c < NB; ++c) p[k][c] = fma(-vk, al[c], p[k][c]);
#pragma unroll
        for (int c = 0; c < NB; ++c)
          if (c == i) p[k][c] = vk;  // Y column: unit diagonal, tail v
        vprev[k] = vk;
        if (gr[k] == i) {  // row i is final: move its R entries out
#pragma unroll
          for (int c = 0; c < NB; ++c)
            if (c > i) {
              Rrow[i][c] = p[k][c];
              p[k][c] = 0.0;
            }
        }
      }
    }
  }
  cluster_sync_all();  // peers finished reading our partial buffers

  // ---- T by the reference recurrence (ref kernels.py:152-162) ----
  if (warp == 0) {
    if (lane < NB)
      for (int c = 0; c < NB; ++c) Ts[lane][c] = 0.0;
    __syncwarp();
    for (int i = 0; i < nb; ++i) {
      const double ti = scal[i][0];
      if (lane < i) {
        double s = 0.0;
        for (int c = lane; c < i; ++c) s = fma(Ts[lane][c], G[c][i], s);
        Ts[lane][i] = -ti * s;
      }
      if (lane == i) Ts[i][i] = -ti;
      __syncwarp();
    }
  }
  __syncthreads();

  // ---- outputs ----
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (!valid[k]) continue;
#pragma unroll
    for (int c = 0; c < NB; ++c)
      if (c < nb) a.Y[gr[k] + (int64_t)c * a.ldy] = p[k][c];
    if (gr[k] < nb) {  // R row: diagonal beta, then the moved-out entries
      const int r = (int)gr[k];
      for (int c = r; c < nb; ++c) *a.P.at(r, c) = (c == r) ? scal[r][1] : Rrow[r][c];
    }
    if (a.W) {
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        if (c >= nb) continue;
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < NB; ++m)
          if (m <= c) s = fma(p[k][m], Ts[m][c], s);
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
  static int attr_dev_mask = 0;
  int dev = 0;
  BR_CUDA(cudaGetDevice(&dev));
  if (!(attr_dev_mask & (1 << dev))) {
    BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_dev_mask |= (1 << dev);
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(LT);
  cfg.dynamicSmemBytes = 0;
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
  // choose the template (rows per thread) and the cluster size
  if (nb > 16) {
    const int C1 = (int)cdiv(L, LT * 1);
    if (C1 <= LEAF_MAXC) {
      int C = 1;
      while (C < C1) C *= 2;
      return launch_leaf_t<32, 1>(st, a, C);
    }
    int C = 1;
    while (C < cdiv(L, LT * 2)) C *= 2;
    return launch_leaf_t<32, 2>(st, a, C);
  }
  if (nb > 8) {
    int C = 1;
    while (C < cdiv(L, LT * 4)) C *= 2;
    return launch_leaf_t<16, 4>(st, a, C);
  }
  int C = 1;
  while (C < cdiv(L, LT * 8)) C *= 2;
  return launch_leaf_t<8, 8>(st, a, C);
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
