// Register-resident cluster leaf, 2D thread layout (included by panel.cu).
#pragma once
#include "common.cuh"

namespace br {

__device__ __forceinline__ void st_async_f64(uint32_t raddr, double a, uint32_t rmbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr),
      "d"(a), "r"(rmbar)
      : "memory");
}

// Two transpose-reductions in lockstep (the shuffles of a level are issued
// back to back, so a pair step pays one dependent chain of five levels, not
// two): afterwards v[0] / w[0] of lane l hold the warp totals of slot l / 4.
template <int RC>
__device__ __forceinline__ void warp_transpose_reduce2(double (&v)[RC], double (&w)[RC], int lane) {
  int n = RC;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (n > 1) {
      const bool up = (lane & o) != 0;
      const int h = n / 2;
#pragma unroll
      for (int q = 0; q < RC / 2; ++q) {
        if (q < h) {
          const double sv = up ? v[q] : v[q + h], kv = up ? v[q + h] : v[q];
          const double sw = up ? w[q] : w[q + h], kw = up ? w[q + h] : w[q];
          const double rv = __shfl_xor_sync(0xffffffffu, sv, o), rw = __shfl_xor_sync(0xffffffffu, sw, o);
          v[q] = kv + rv;
          w[q] = kw + rw;
        }
      }
      n = h;
    } else {
      const double rv = __shfl_xor_sync(0xffffffffu, v[0], o), rw = __shfl_xor_sync(0xffffffffu, w[0], o);
      v[0] += rv;
      w[0] += rw;
    }
  }
}

// One leaf (L x nb, nb <= NB, NB in {8, 16, 32, 64}) of a Householder panel, same
// outputs and arithmetic contract as leaf_reg_kernel (Y, tau, T, W, R rows of
// P), with a 2D layout: warp w owns the 8 columns 8*(w % CG) .. +8 (CG = NB/8
// column groups) of the 32 RPT rows of its row group rg = w / CG, and lane l
// of it rows rg*32*RPT + 32 r + l (r < RPT) of the CTA's block: RPT x 8
// doubles per thread (RPT = 8, or 4 with twice the warps per row span). The warps owning the current column rotate their 8 register
// columns by one per step, so every register index is compile-time in a
// non-unrolled step loop (see below).
//
// Step i (column i lives in column group cg = i / 8, register column ci):
//   1. the owner warps publish x = column i (rows >= i, zero above) to shared
//      memory; CTA 0's lane i publishes row i; one __syncthreads;
//   2. every warp forms its 8 partial sums x^T p[.][c] over its rows plus
//      ||x||^2 and transpose-reduces them (9 + 5 shuffles instead of the 32
//      slots per warp of the 1D layout); the slot of a finished column is the
//      Gram entry x^T Y_y, as in leaf_reg_kernel;
//   3. exchange (several CTAs or row groups): the row groups of a column
//      group combine their partials in shared memory, then one warp per
//      column group pushes its 8 slot totals (st.async, completing bytes on
//      the receiver's mbarrier) to every CTA; with one CTA and one row group
//      the warp already has the totals;
//   4. every warp forms the same scalars from the same data in the same
//      order: beta = -sign(x0)||x||, alpha_c = P_ic - (x^T P_c)/beta,
//      v = x / (x0 - beta), and updates its columns.
// Deterministic: all CTAs sum the same received vectors in the same order.
template <int NB, int NW, int RPT = 8, bool PAIR = false>
__global__ void __launch_bounds__(NW * 32 + ((PAIR && NW <= 4) ? 32 : 0), 1) leaf2_kernel(const LeafArgs a) {
  // TW: one extra warp forms T column by column behind the step loop (it
  // joins the loop's CTA barriers and reads the columns finished so far from
  // prog[]), so the epilogue no longer pays for T (4.8 k cycles of a 32-wide
  // leaf). Only where the register file has room for a fifth warp.
  constexpr bool TW = PAIR && NW <= 4;
  // PAIR: two columns per exchange where possible (see the pair step below);
  // PR = exchange sets (x / row / slot buffers) per step
  constexpr int PR = PAIR ? 2 : 1;
  static_assert(!PAIR || NB <= 32, "pair steps: the pivot rows live in register row 0");
  constexpr int CG = NB / 8;           // column groups
  constexpr int RG = NW / CG;          // row groups (32 RPT rows each)
  constexpr int RGR = 32 * RPT;        // rows per row group
  constexpr int ROWS = RG * RGR;       // rows per CTA
  static_assert(RPT % 2 == 0 && RPT >= (NB + 31) / 32, "rows per thread");
  constexpr int NT = NW * 32 + (TW ? 32 : 0);
  // PRE: the RG row-group warps of a column group first combine their slot
  // partials through shared memory (named barrier), so each CTA pushes one
  // partial vector instead of RG (fewer st.async, 4x shorter receive sums at RG = 4)
  constexpr bool PRE = RG > 1;
  constexpr int MAXSRC = PRE ? LEAF_MAXC : LEAF_MAXC * RG;
  constexpr int RB = (NB + 31) / 32;  // register rows that can hold rows < NB
  static_assert(CG * RG == NW && RG >= 1, "warp layout");
  // dynamic: Ys [NB][ROWS] (epilogue), G [NB][NB+1] (Gram), Ts [NB][NB+1] (T)
  extern __shared__ __align__(16) double Ys[];
  __shared__ __align__(16) double xs[2][PR][ROWS];
  __shared__ __align__(16) double rowl[2][PR][NB];          // row i (and i + 1), CTA 0 local
  __shared__ __align__(16) double recv[2][PR][MAXSRC][NB];  // slot partials per source
  __shared__ __align__(16) double recvn[2][MAXSRC];         // ||x||^2 partials per source
  __shared__ __align__(16) double recvr[2][PR][NB];         // row i (and i + 1) from CTA 0
  __shared__ double pre[PR][RG][NB];                        // PRE: row-group slot partials
  __shared__ double pren[RG];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double scal[NB][3];  // x0 -> tau, beta, rinv
  __shared__ int prog[2];         // TW: columns finished before the step loop's barrier (by parity)
  // Ys column stride padded by 8 doubles: the W fragment loads
  // Ys[(k0 + tq) * YLD + r] of tq = 0,1 (and 2,3) then fill distinct banks
  constexpr int YLD = ROWS + 8;
  // Gram entries are written every column step: a static array (NB <= 32)
  // keeps those stores shared-space (a pointer carved from the dynamic array
  // was generic and cost a shared-window base read, S2R SR_CgaCtaId, per step)
  __shared__ double Gst[NB <= 32 ? NB : 1][NB <= 32 ? NB + 1 : 1];
  double(*G)[NB + 1] = (NB <= 32) ? reinterpret_cast<double(*)[NB + 1]>(&Gst[0][0])
                                  : reinterpret_cast<double(*)[NB + 1]>(Ys + NB * YLD);
  double(*Ts)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(Ys + NB * YLD + NB * (NB + 1));

  const uint32_t rank = cluster_ctarank(), ncta = cluster_nctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wcg = warp % CG, rg = warp / CG;
  const int64_t base = (int64_t)rank * ROWS;
  const int lrow0 = rg * RGR + lane;  // local row of register row r: lrow0 + 32 r
  const int64_t gr0 = base + lrow0;
  const bool xch = (ncta > 1) || (RG > 1);
  const int nsrc = PRE ? (int)ncta : (int)ncta * RG;
  const int nb = a.nb;
  const int64_t Lr = a.L;
  const MatView P = a.P;
  constexpr unsigned FULL = 0xffffffffu;

#ifdef BR_LEAF_PROF  // phase counters: build with BR_BUILD_PROF=1, run with BR_LEAF_PROF=1
  const bool pr = a.prof != nullptr && rank == 0 && tid == 0;
  long long tp[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tc = pr ? clock64() : 0;
#define BR_PHASE2(k)                \
  if (pr) {                         \
    const long long t_ = clock64(); \
    tp[k] += t_ - tc;               \
    tc = t_;                        \
  }
#else
#define BR_PHASE2(k)
#endif
  pdl_wait();  // the panel columns were written by the previous kernel
  if (xch && tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double p[RPT][8];
  {
    // branch-free addressing of the (possibly transposed) view
    const int64_t rs = P.trans ? P.ld : 1, cs = P.trans ? 1 : P.ld;
    const double* pb = P.p + gr0 * rs + (int64_t)(wcg * 8) * cs;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const bool rok = gr0 + 32 * r < Lr && warp < NW;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        p[r][c] = (rok && wcg * 8 + c < nb) ? __ldcg(pb + (32 * r) * rs + c * cs) : 0.0;
    }
  }
  if (xch) cluster_sync_all();  // mbarriers initialized cluster-wide before any st.async
  BR_PHASE2(7);
  if (TW && warp == NW) {
    // ---- T warp: T[r][i] = -tau_i sum_{c<i} T[r][c] G[c][i] (ref kernels.py:152-162),
    // lane r = row r, in shared memory (Ts), the sum in ascending c as the
    // epilogue version formed it. One CTA barrier per step-loop iteration plus
    // the one after the loop, like the main warps.
    if (lane < NB) {
#pragma unroll
      for (int c = 0; c < NB; ++c) Ts[lane][c] = 0.0;
    }
    int done = 0;
    for (unsigned it = 0;; ++it) {
      __syncthreads();
      const int pi = *reinterpret_cast<volatile int*>(&prog[it & 1]);
      for (; done < pi; ++done) {
        const double be = scal[done][1];
        const double mtau = (be != 0.0) ? -((be - scal[done][0]) / be) : 0.0;
        double acc = 0.0;
        for (int c = 0; c < done; ++c) acc = fma(Ts[lane < NB ? lane : 0][c], G[c][done], acc);
        if (lane < NB && lane <= done) Ts[lane][done] = (lane == done) ? mtau : mtau * acc;
      }
      if (pi >= nb) break;
    }
    __syncthreads();  // Ts complete (the main warps have staged Y)
  } else {

  // The owner warps of column group cg rotate their 8 register columns left
  // by one per step (the finished Y column moves to the end), so the current
  // column is always p[r][0] and every register index stays compile-time with
  // a non-unrolled step loop (the unrolled 8-step sweep overflowed the
  // instruction cache). Register slot s of an owner warp holds column
  // (ci + s) & 7 of its group; slot-ordered exchange buffers need no remap.
  // rows < 32 (the only ones that can lie above the pivot) are register row 0
  // of row group 0 in CTA 0
  const bool top = (rank == 0 && rg == 0);
  // remote addresses of this lane's pushes (buffer 0; buffer 1 at a fixed offset)
  const int src = PRE ? (int)rank : (int)rank * RG + rg;
  const bool pusher = !PRE || rg == 0;  // warps whose slot totals leave the CTA
  const int pu = lane & 7, ppair = lane >> 3;
  uint32_t ra_s[2] = {0, 0}, ra_sm[2] = {0, 0}, ra_n = 0, ra_nm = 0, ra_r[2] = {0, 0},
           ra_rm[2] = {0, 0};
  unsigned vmask = 0;  // bit k: slot push k, bit 2 + k: row-i push k, bit 4: norm push
  if (xch) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int q = pu + 8 * k;
      if (q < (int)ncta && pusher) {
        vmask |= 1u << k;
        ra_s[k] = map_cluster(&recv[0][0][src][wcg * 8 + 2 * ppair], (uint32_t)q);
        ra_sm[k] = map_cluster(&mbar[0], (uint32_t)q);
      }
      const int t = lane + 32 * k;  // row-i pushes (CTA 0, row group 0): pair t & 3 -> CTA t >> 2
      if (top && t < 4 * (int)ncta) {
        vmask |= 4u << k;
        ra_r[k] = map_cluster(&recvr[0][0][wcg * 8 + 2 * (t & 3)], (uint32_t)(t >> 2));
        ra_rm[k] = map_cluster(&mbar[0], (uint32_t)(t >> 2));
      }
    }
    if (lane < (int)ncta && wcg == 0 && pusher) {
      vmask |= 16u;
      ra_n = map_cluster(&recvn[0][src], (uint32_t)lane);
      ra_nm = map_cluster(&mbar[0], (uint32_t)lane);
    }
  }
  constexpr uint32_t RECV_B = PR * MAXSRC * NB * 8, RECVN_B = MAXSRC * 8, RECVR_B = PR * NB * 8;
  constexpr uint32_t RECV_S = MAXSRC * NB * 8, RECVR_S = NB * 8;  // second set of a pair step
  constexpr int SPL = MAXSRC / 4;  // sources summed per lane (4 lanes per slot)

  // stp counts exchange rounds (buffer / mbarrier phase); a pair step advances
  // i by two, and a pair that fails its safeguard is redone as a single step
  int i = 0;
  unsigned stp = 0;
  bool single = false;
#pragma unroll 1
  while (i < nb) {
    const int cg = i >> 3, ci = i & 7;
    const bool own = (wcg == cg);
    const int buf = stp & 1;
    const uint32_t par = (stp >> 1) & 1;
    ++stp;
    if (TW && tid == 0) prog[buf] = i;
    if constexpr (PAIR) {
      if (xch && !single && !(i & 1) && i + 1 < nb) {
        // ---- pair step: columns i and i + 1 (same column group, owner slots 0
        // and 1) in ONE exchange. Besides x = column i's sums d1_c = x^T P_c,
        // the exchange carries d2_c = y^T P_c for y = column i + 1 BEFORE
        // H_i is applied (rows > i). H_i is orthogonal on rows >= i, so after
        // it the sums of the updated column y' over rows > i follow without
        // touching the data again:
        //   y'^T P'_c = (d2_c + y_i P_ic) - R_{i,i+1} R_ic,  R_ic = P_ic - alpha_c
        //   ||y'||^2  = ||y||^2 + alpha_y (2 y_i - alpha_y)   (rows > i)
        // (norm downdating; a pair whose ||y'||^2 cancels below THETA of
        // ||y||^2 is redone as two single steps, so the reflector of column
        // i + 1 keeps the accuracy of a directly summed norm up to 1/THETA).
        // ||x||^2, x^T y and ||y||^2 are the owner slots 0 / 1 themselves.
        constexpr double THETA = 0.25;
        const bool above = top && lane < i, piv = top && lane == i, piv2 = top && lane == i + 1;
        if (tid == 0) mbar_arrive_expect_tx(&mbar[buf], (uint32_t)(nsrc * 2 * NB * 8 + 2 * NB * 8));
        if (own) {
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            xs[buf][0][lrow0 + 32 * r] = (r == 0 && above) ? 0.0 : p[r][0];
            xs[buf][1][lrow0 + 32 * r] = (r == 0 && (above || piv)) ? 0.0 : p[r][1];
          }
        }
        if (piv || piv2) {
#pragma unroll
          for (int c = 0; c < 8; c += 2)
            *reinterpret_cast<double2*>(&rowl[buf][piv ? 0 : 1][wcg * 8 + c]) = make_double2(p[0][c], p[0][c + 1]);
        }
        __syncthreads();
        BR_PHASE2(1);
        if (top) {  // rows i and i + 1 to every CTA
#pragma unroll
          for (int k = 0; k < 2; ++k)
            if (vmask & (4u << k)) {
              const int c = wcg * 8 + 2 * (lane & 3);
              st_async_v2(ra_r[k] + buf * RECVR_B, rowl[buf][0][c], rowl[buf][0][c + 1], ra_rm[k] + buf * 8u);
              st_async_v2(ra_r[k] + buf * RECVR_B + RECVR_S, rowl[buf][1][c], rowl[buf][1][c + 1],
                          ra_rm[k] + buf * 8u);
            }
        }
        double s1[8], s2[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) s1[c] = s2[c] = 0.0;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const double x1 = xs[buf][0][lrow0 + 32 * r], x2 = xs[buf][1][lrow0 + 32 * r];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            s1[c] = fma(x1, p[r][c], s1[c]);
            s2[c] = fma(x2, p[r][c], s2[c]);
          }
        }
        const int sl = lane >> 2;
        warp_transpose_reduce2<8>(s1, s2, lane);  // s1[0], s2[0]: warp totals of register slot lane / 4
        BR_PHASE2(0);
        if (PRE) {
          if ((lane & 3) == 0) {
            pre[0][rg][wcg * 8 + sl] = s1[0];
            pre[1][rg][wcg * 8 + sl] = s2[0];
          }
          asm volatile("bar.sync %0, %1;" ::"r"(1 + wcg), "r"(RG * 32) : "memory");
          if (rg == 0) {
            double t = 0.0, u = 0.0;
#pragma unroll
            for (int g = 0; g < RG; ++g) {
              t += pre[0][g][wcg * 8 + sl];
              u += pre[1][g][wcg * 8 + sl];
            }
            s1[0] = t;
            s2[0] = u;
          }
        }
        {
          const double o1 = __shfl_xor_sync(FULL, s1[0], 4), o2 = __shfl_xor_sync(FULL, s2[0], 4);
          const double v0 = (pu < 4) ? s1[0] : o1, v1 = (pu < 4) ? o1 : s1[0];
          const double w0 = (pu < 4) ? s2[0] : o2, w1 = (pu < 4) ? o2 : s2[0];
#pragma unroll
          for (int k = 0; k < 2; ++k)
            if (vmask & (1u << k)) {
              st_async_v2(ra_s[k] + buf * RECV_B, v0, v1, ra_sm[k] + buf * 8u);
              st_async_v2(ra_s[k] + buf * RECV_B + RECV_S, w0, w1, ra_sm[k] + buf * 8u);
            }
        }
        BR_PHASE2(2);
        while (!mbar_try_wait_cta(&mbar[buf], par)) {
        }
        BR_PHASE2(3);
        double tot1, tot2, nrm2, dxy, ny2;
        {
          const int c = wcg * 8 + sl, q4 = lane & 3, c0 = cg * 8;
          double ta[SPL], tb[SPL], tc_[SPL], td[SPL], te[SPL];
#pragma unroll
          for (int k = 0; k < SPL; ++k) {
            const int sidx = q4 + 4 * k;
            const bool ok = sidx < nsrc;
            ta[k] = ok ? recv[buf][0][sidx][c] : 0.0;
            tb[k] = ok ? recv[buf][1][sidx][c] : 0.0;
            tc_[k] = ok ? recv[buf][0][sidx][c0] : 0.0;      // ||x||^2 (rows >= i)
            td[k] = ok ? recv[buf][0][sidx][c0 + 1] : 0.0;  // x^T y (rows >= i)
            te[k] = ok ? recv[buf][1][sidx][c0 + 1] : 0.0;  // ||y||^2 (rows > i)
          }
#pragma unroll
          for (int h = SPL / 2; h >= 1; h >>= 1)
#pragma unroll
            for (int k = 0; k < h; ++k) {
              ta[k] += ta[k + h];
              tb[k] += tb[k + h];
              tc_[k] += tc_[k + h];
              td[k] += td[k + h];
              te[k] += te[k + h];
            }
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) {
            ta[0] += __shfl_xor_sync(FULL, ta[0], o);
            tb[0] += __shfl_xor_sync(FULL, tb[0], o);
            tc_[0] += __shfl_xor_sync(FULL, tc_[0], o);
            td[0] += __shfl_xor_sync(FULL, td[0], o);
            te[0] += __shfl_xor_sync(FULL, te[0], o);
          }
          tot1 = ta[0];
          tot2 = tb[0];
          nrm2 = tc_[0];
          dxy = td[0];
          ny2 = te[0];
        }
        // ---- scalars of both columns (identical in every warp and CTA) ----
        const double x0 = recvr[buf][0][cg * 8], yi = recvr[buf][0][cg * 8 + 1];   // row i: x_i, y_i
        const double xn = recvr[buf][1][cg * 8], yn = recvr[buf][1][cg * 8 + 1];   // row i + 1
        const double pic1 = recvr[buf][0][wcg * 8 + sl], pic2 = recvr[buf][1][wcg * 8 + sl];
        const int cs = wcg * 8 + (own ? ((ci + sl) & 7) : sl);
        double beta = 0.0, rb = 0.0, rinv = 0.0;
        if (nrm2 != 0.0) {
          const double rs = rsqrt(nrm2), nrm = nrm2 * rs;
          beta = (x0 < 0.0) ? nrm : -nrm;
          rb = (x0 < 0.0) ? rs : -rs;
          rinv = __drcp_rn(x0 - beta);
        }
        const double alpha1 = (nrm2 != 0.0 && cs > i && cs < nb) ? fma(-tot1, rb, pic1) : 0.0;
        const double alphay = (nrm2 != 0.0) ? fma(-dxy, rb, yi) : 0.0;  // alpha of column i + 1
        const double ry = yi - alphay;                                    // R[i][i + 1]
        const double nrm2p = fma(alphay, 2.0 * yi - alphay, ny2);        // ||y'||^2 over rows > i
        if (!(nrm2p >= THETA * fma(yi, yi, ny2))) {  // cancellation (or NaN): two single steps
          single = true;
          continue;
        }
        const double vn = xn * rinv;                  // v_i at row i + 1
        const double x0p = fma(-vn, alphay, yn);      // pivot of y'
        double beta2 = 0.0, rb2 = 0.0, rinv2 = 0.0;
        if (nrm2p != 0.0) {
          const double rs = rsqrt(nrm2p), nrm = nrm2p * rs;
          beta2 = (x0p < 0.0) ? nrm : -nrm;
          rb2 = (x0p < 0.0) ? rs : -rs;
          rinv2 = __drcp_rn(x0p - beta2);
        }
        const double pic2p = fma(-vn, alpha1, pic2);  // row i + 1 of this slot after H_i
        const double tot2p = fma(yi, pic1, tot2) - ry * (pic1 - alpha1);
        const double alpha2 = (nrm2p != 0.0 && cs > i + 1 && cs < nb) ? fma(-tot2p, rb2, pic2p) : 0.0;
        if (rg == 0 && (lane & 3) == 0) {  // Gram entries Y_c^T v_i, Y_c^T v_{i+1} for T
          if (cs < i) {
            const double g1 = fma(fma(-pic1, x0, tot1), rinv, pic1);
            G[cs][i] = g1;
            const double ty = fma(-alphay, g1 - pic1, tot2);  // Y_c^T y' over rows > i
            G[cs][i + 1] = fma(fma(-pic2, x0p, ty), rinv2, pic2);
          } else if (cs == i) {
            // v_i^T y' over rows > i = rinv (x^T y - alpha_y rinv ||x||^2), both over rows > i
            const double xy = fma(-x0, yi, dxy);
            const double sv = rinv * fma(-alphay * rinv, fma(-x0, x0, nrm2), xy);
            G[i][i + 1] = fma(fma(-vn, x0p, sv), rinv2, vn);
          }
        }
        if (tid == 0) {
          scal[i][0] = x0;
          scal[i][1] = beta;
          scal[i][2] = rinv;
          scal[i + 1][0] = x0p;
          scal[i + 1][1] = beta2;
          scal[i + 1][2] = rinv2;
        }
        BR_PHASE2(4);
        if (wcg >= cg) {
          double al1[8], al2[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            al1[c] = __shfl_sync(FULL, alpha1, 4 * c);
            al2[c] = __shfl_sync(FULL, alpha2, 4 * c);
          }
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const double x1 = xs[buf][0][lrow0 + 32 * r], x2 = xs[buf][1][lrow0 + 32 * r];
            double v1 = x1 * rinv;                    // 0 above row i
            if (r == 0 && piv) v1 = 1.0;
            double v2 = fma(-v1, alphay, x2) * rinv2;  // y' / (x0' - beta'); 0 above row i
            if (r == 0 && piv) v2 = 0.0;
            if (r == 0 && piv2) v2 = 1.0;
            if (own) {  // rotate by two: Y columns i, i + 1 (R kept above) to slots 6, 7
              const double y0 = p[r][0], y1 = p[r][1];
#pragma unroll
              for (int c = 0; c < 6; ++c) p[r][c] = fma(-v2, al2[c + 2], fma(-v1, al1[c + 2], p[r][c + 2]));
              p[r][6] = (r == 0 && above) ? y0 : v1;
              p[r][7] = (r == 0 && above) ? y1 : ((r == 0 && piv) ? y1 - alphay : v2);
            } else {
#pragma unroll
              for (int c = 0; c < 8; ++c) p[r][c] = fma(-v2, al2[c], fma(-v1, al1[c], p[r][c]));
            }
          }
        }
        BR_PHASE2(6);
        i += 2;
        continue;
      }
      single = false;
    }
    // register rows r < RB of CTA 0's row group 0 hold rows 32 r + lane < NB,
    // the only rows that can lie above (or be) the pivot row i
    bool above[RB], piv[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      above[r] = top && lane + 32 * r < i;
      piv[r] = top && lane + 32 * r == i;
    }
    if (xch && tid == 0) mbar_arrive_expect_tx(&mbar[buf], (uint32_t)(nsrc * (NB + 1) * 8 + NB * 8));
    // ---- 1. publish x (owner warps) and row i (CTA 0, row group 0, lane i) ----
    if (own) {
#pragma unroll
      for (int r = 0; r < RPT; ++r) xs[buf][0][lrow0 + 32 * r] = (r < RB && above[r]) ? 0.0 : p[r][0];
    }
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (piv[r]) {
#pragma unroll
        for (int c = 0; c < 8; c += 2)
          *reinterpret_cast<double2*>(&rowl[buf][0][wcg * 8 + c]) = make_double2(p[r][c], p[r][c + 1]);
      }
    __syncthreads();
    BR_PHASE2(1);
    if (xch && top) {  // row i to every CTA: 4 slot pairs x ncta
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if (vmask & (4u << k)) {
          const int c = wcg * 8 + 2 * (lane & 3);
          st_async_v2(ra_r[k] + buf * RECVR_B, rowl[buf][0][c], rowl[buf][0][c + 1], ra_rm[k] + buf * 8u);
        }
    }
    // ---- 2. partial sums over this warp's rows ----
    double xv[RPT], s[8];
#pragma unroll
    for (int r = 0; r < RPT; ++r) xv[r] = xs[buf][0][lrow0 + 32 * r];
    double nr0 = 0.0, nr1 = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; r += 2) {
      nr0 = fma(xv[r], xv[r], nr0);
      nr1 = fma(xv[r + 1], xv[r + 1], nr1);
    }
    double nr = warp_sum(nr0 + nr1);  // independent of the slots: overlaps them
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int r = 0; r < RPT; r += 2) {
        t0 = fma(xv[r], p[r][c], t0);
        t1 = fma(xv[r + 1], p[r + 1][c], t1);
      }
      s[c] = t0 + t1;
    }
    warp_transpose_reduce<8>(s, lane);  // s[0]: warp total of register slot lane / 4
    const int sl = lane >> 2;
    BR_PHASE2(0);
    double tot, nrm2;
    if (!xch) {
      tot = s[0];
      nrm2 = nr;
    } else {
      // ---- 3. push slot pairs (and the norm from column group 0) to every CTA ----
      if (PRE) {  // combine the row groups of this column group first (fixed order)
        if ((lane & 3) == 0) pre[0][rg][wcg * 8 + sl] = s[0];
        if (wcg == 0 && lane == 0) pren[rg] = nr;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + wcg), "r"(RG * 32) : "memory");
        if (rg == 0) {
          double t = 0.0;
#pragma unroll
          for (int g = 0; g < RG; ++g) t += pre[0][g][wcg * 8 + sl];
          s[0] = t;
          if (wcg == 0) {
            double u = 0.0;
#pragma unroll
            for (int g = 0; g < RG; ++g) u += pren[g];
            nr = u;
          }
        }
      }
      const double oth = __shfl_xor_sync(FULL, s[0], 4);
      const double v0 = (pu < 4) ? s[0] : oth, v1 = (pu < 4) ? oth : s[0];
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if (vmask & (1u << k)) st_async_v2(ra_s[k] + buf * RECV_B, v0, v1, ra_sm[k] + buf * 8u);
      if (vmask & 16u) st_async_f64(ra_n + buf * RECVN_B, nr, ra_nm + buf * 8u);
      BR_PHASE2(2);
      while (!mbar_try_wait_cta(&mbar[buf], par)) {
      }
      BR_PHASE2(3);
      // slot sl and the norm: the 4 lanes of a slot split the sources (all
      // loads issued at once), then a fixed two-level tree
      const int c = wcg * 8 + sl, q4 = lane & 3;
      double ts[SPL], tn[SPL];
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        const int sidx = q4 + 4 * k;
        ts[k] = (sidx < nsrc) ? recv[buf][0][sidx][c] : 0.0;
        tn[k] = (sidx < nsrc) ? recvn[buf][sidx] : 0.0;
      }
#pragma unroll
      for (int h = SPL / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int k = 0; k < h; ++k) {
          ts[k] += ts[k + h];
          tn[k] += tn[k + h];
        }
      ts[0] += __shfl_xor_sync(FULL, ts[0], 1);
      tn[0] += __shfl_xor_sync(FULL, tn[0], 1);
      ts[0] += __shfl_xor_sync(FULL, ts[0], 2);
      tn[0] += __shfl_xor_sync(FULL, tn[0], 2);
      tot = ts[0];
      nrm2 = tn[0];
    }
    // ---- 4. scalars (identical in every warp and CTA) ----
    // (two direct shared loads: a pointer selected between the arrays would be
    // generic and cost a shared-window base computation every step)
    const double x0 = xch ? recvr[buf][0][cg * 8] : rowl[buf][0][cg * 8];  // owner slot 0 = column i
    const double pic = xch ? recvr[buf][0][wcg * 8 + sl] : rowl[buf][0][wcg * 8 + sl];  // row i, this slot
    const int cs = wcg * 8 + (own ? ((ci + sl) & 7) : sl);  // its column
    double beta = 0.0, rb = 0.0, rinv = 0.0;
    if (nrm2 != 0.0) {
      // ||x|| and 1/||x|| from one rsqrt, 1/(x0 - beta) by rcp (as leaf_reg_kernel)
      const double rs = rsqrt(nrm2), nrm = nrm2 * rs;
      beta = (x0 < 0.0) ? nrm : -nrm;
      rb = (x0 < 0.0) ? rs : -rs;
      rinv = __drcp_rn(x0 - beta);
    }
    const double alpha = (nrm2 != 0.0 && cs > i && cs < nb) ? fma(-tot, rb, pic) : 0.0;
    if (cs < i && rg == 0 && (lane & 3) == 0) G[cs][i] = fma(fma(-pic, x0, tot), rinv, pic);
    if (tid == 0) {
      scal[i][0] = x0;
      scal[i][1] = beta;
      scal[i][2] = rinv;
    }
    BR_PHASE2(4);
    if (wcg >= cg) {  // earlier groups hold finished Y columns only
      double al[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) al[c] = __shfl_sync(FULL, alpha, 4 * c);
      double vk[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) vk[r] = (r < RB && piv[r]) ? 1.0 : xv[r] * rinv;  // 0 above row i
      if (own) {  // rotate: slot s <- slot s+1 updated; Y column i (R kept above) to slot 7
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const double x = p[r][0];
#pragma unroll
          for (int c = 0; c < 7; ++c) p[r][c] = fma(-vk[r], al[c + 1], p[r][c + 1]);
          p[r][7] = (r < RB && above[r]) ? x : vk[r];
        }
      } else {
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) p[r][c] = fma(-vk[r], al[c], p[r][c]);
      }
    }
    BR_PHASE2(6);
    ++i;
  }
  // a partial last group leaves its owners rotated by nb & 7: finish the turn
  if (nb & 7) {
    if (wcg == ((nb - 1) >> 3)) {
#pragma unroll 1
      for (int t = nb & 7; t < 8; ++t) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const double x = p[r][0];
#pragma unroll
          for (int c = 0; c < 7; ++c) p[r][c] = p[r][c + 1];
          p[r][7] = x;
        }
      }
    }
  }
  pdl_trigger();
  if (TW && tid == 0) prog[stp & 1] = nb;
  __syncthreads();  // scal / G complete
  BR_PHASE2(5);
  // ---- T by the reference recurrence (ref kernels.py:152-162), warp 0, while
  // the other warps store Y; then warp 0 stores its own Y ----
  auto store_y = [&]() {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int lrow = lrow0 + 32 * r;
      const int64_t row = base + lrow;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int col = wcg * 8 + c;
        const double y = (col < nb && row >= col) ? p[r][c] : 0.0;
        if (a.W) Ys[col * YLD + lrow] = y;  // staged for W = Y T only
        if (col < nb && row < Lr) a.Y[row + (int64_t)col * a.ldy] = y;
      }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int row = lane + 32 * r;
      if (top && row < nb) {  // R rows
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int col = wcg * 8 + c;
          if (col >= row && col < nb) *P.at(row, col) = (col == row) ? scal[row][1] : p[r][c];
        }
      }
    }
  };
  if constexpr (TW) {
    store_y();
    BR_PHASE2(13);
  } else {
  if (tid < nb) {  // tau = (beta - x0) / beta (ref kernels.py:109); x0 is read by its owner only
    const double be = scal[tid][1];
    scal[tid][0] = (be != 0.0) ? (be - scal[tid][0]) / be : 0.0;
  }
  __syncthreads();
  BR_PHASE2(9);
  if constexpr (NB <= 32) {
    // Warp 0 stores its Y first (its register columns are then dead), then
    // forms T row r = lane by the reference recurrence
    //   T[r][i] = -tau_i sum_{c<i} T[r][c] G[c][i]   (ref kernels.py:152-162)
    // in right-looking order: once T[r][c] is known it is folded into every
    // later column's sum, so the dependent chain is one FMA + one multiply
    // per column instead of a dot product per column.
    store_y();
    BR_PHASE2(13);
    if (warp == 0) {
      const int r = lane;
      double acc[NB], tr[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) acc[i] = 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const double tc = (c < r || c >= nb) ? 0.0 : ((c == r) ? -scal[c][0] : -scal[c][0] * acc[c]);
        tr[c] = tc;
#pragma unroll
        for (int i = c + 1; i < NB; ++i) acc[i] = fma(tc, G[c][i], acc[i]);
      }
      if (r < NB) {
#pragma unroll
        for (int c = 0; c < NB; ++c) Ts[r][c] = tr[c];
      }
    }
    BR_PHASE2(14);
  } else if (warp < NB / 32) {
    // T rows 32 warp + lane by the reference recurrence
    // T[r][i] = -tau_i sum_{c<i} T[r][c] G[c][i] (ref kernels.py:152-162)
    const int r = warp * 32 + lane;
    double tr[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) tr[c] = (c == r && r < nb) ? -scal[c][0] : 0.0;
#pragma unroll
    for (int i = 1; i < NB; ++i) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int c = 0; c + 1 < i; c += 2) {
        s0 = fma(tr[c], G[c][i], s0);
        s1 = fma(tr[c + 1], G[c + 1][i], s1);
      }
      if (i & 1) s0 = fma(tr[i - 1], G[i - 1][i], s0);
      if (i > r && i < nb) tr[i] = -scal[i][0] * (s0 + s1);
    }
    if (r < NB) {
#pragma unroll
      for (int c = 0; c < NB; ++c) Ts[r][c] = tr[c];
    }
    __syncwarp();
    store_y();
  } else {
    store_y();
  }
  }
  __syncthreads();
  BR_PHASE2(8);
  // ---- W = Y T (or Y T^T) on the tensor cores ----
  if (a.W) {
    const int gq = lane >> 2, tq = lane & 3;
    constexpr int U = 4;
    for (int rb = warp * 8; rb < ROWS; rb += NW * 8 * U) {
      if (base + rb >= Lr) break;
      double acc[U][NB / 8][2];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int n = 0; n < NB / 8; ++n) acc[u][n][0] = acc[u][n][1] = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < NB; k0 += 4) {
        double bt[NB / 8];
#pragma unroll
        for (int n = 0; n < NB / 8; ++n)
          bt[n] = a.wt ? Ts[n * 8 + gq][k0 + tq] : Ts[k0 + tq][n * 8 + gq];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r0 = rb + u * NW * 8;
          const double av = (r0 < ROWS) ? Ys[(k0 + tq) * YLD + r0 + gq] : 0.0;
#pragma unroll
          for (int n = 0; n < NB / 8; ++n) {
            if (!a.wt && k0 >= n * 8 + 8) continue;  // zero blocks of the triangular T
            if (a.wt && k0 + 4 <= n * 8) continue;
            dmma884(acc[u][n][0], acc[u][n][1], av, bt[n]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r0 = rb + u * NW * 8;
        const int64_t row = base + r0 + gq;
        if (r0 < ROWS && row < Lr) {
#pragma unroll
          for (int n = 0; n < NB / 8; ++n)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = n * 8 + 2 * tq + h;
              if (c < nb) a.W[row + (int64_t)c * a.ldw] = acc[u][n][h];
            }
        }
      }
    }
  }
  }  // main warps
  BR_PHASE2(10);
#ifdef BR_LEAF_PROF
  if (pr) {
    for (int k = 0; k < 11; ++k) atomicAdd((unsigned long long*)&a.prof[k], (unsigned long long)tp[k]);
    for (int k = 13; k < 15; ++k) atomicAdd((unsigned long long*)&a.prof[k], (unsigned long long)tp[k]);
    atomicAdd((unsigned long long*)&a.prof[11], (unsigned long long)nb);
    atomicAdd((unsigned long long*)&a.prof[12], 1ull);
  }
#endif
#undef BR_PHASE2
  if (rank == 0) {
    if (tid < nb) {
      const double be = scal[tid][1];  // TW: scal[.][0] still holds x0 (ref kernels.py:109)
      a.tau[tid] = !TW ? scal[tid][0] : ((be != 0.0) ? (be - scal[tid][0]) / be : 0.0);
    }
    if (a.T)
      for (int q = tid; q < nb * nb; q += NT) {
        const int r = q % nb, c = q / nb;
        a.T[r + (int64_t)c * a.ldt] = Ts[r][c];
      }
  }
  if (xch) cluster_sync_all();  // no remote traffic is in flight when any CTA exits
}

}  // namespace br
