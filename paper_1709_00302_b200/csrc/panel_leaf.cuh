// Register-resident cluster leaf of the Householder panel (included by panel.cu).
#pragma once
#include "common.cuh"

namespace br {

__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(m)),
               "r"(bytes)
               : "memory");
}
// CTA-scope acquire: the st.async bytes land in this CTA's shared memory and
// are complete when the phase flips; a cluster-scope acquire would also
// invalidate L1 (CCTL.IVALL) on every poll, which measured as the largest
// single stall of the leaf's step loop.
__device__ __forceinline__ bool mbar_try_wait_cta(uint64_t* m, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
      "selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_u32(m)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* m, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
      "selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_u32(m)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Stores into another CTA's shared memory that complete their bytes on that
// CTA's mbarrier transaction count (no cluster barrier, no fence).
__device__ __forceinline__ void st_async_v2(uint32_t raddr, double a, double b, uint32_t rmbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
          raddr),
      "d"(a), "d"(b), "r"(rmbar)
      : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

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

// One leaf (L x nb, nb <= NB) of a Householder panel.
//
// Thread t of CTA q owns rows q*LT*R + t + k*LT (k < R). Its registers p[k][]
// hold, ROTATED, the active columns followed by the finished Y columns:
// at step i, p[k][0..nb-i) are columns i..nb-1 (p[k][0] = current column),
// and p[k][NB-i..NB) are Y_0..Y_{i-1} (explicit unit diagonal, zeros above).
// The rank-1 update writes p[k][c] from p[k][c+1] and appends the new Y
// column at NB-1, so the rotation is free and no element ever needs a mask.
// Slots of the per-step reduced vector S_c = x^T p[.][c] (x = current
// column masked to rows >= i, one multiplier for every slot):
//   c <  NB - i : x^T P_{i+c}                  (c = 0 gives ||x||^2)
//   c >= NB - i : x^T Y_y, y = c-NB+i          -> Gram column i for T:
//       Y_y^T v_i = Y_y[i] + (x^T Y_y - Y_y[i] x0) / (x0 - beta)
//     (v_i = e_i + (x - x0 e_i)/(x0 - beta); Y_y[i] arrives with row i).
// Per step: FMAs on registers, a warp transpose-reduction (shuffles), the
// per-warp partials through shared memory, then warp w pushes its slots with
// st.async into every CTA of the cluster, completing bytes on that CTA's
// mbarrier (double-buffered). The CTA owning row i also pushes row i. Every
// thread waits on its own mbarrier - no cluster barrier, no fence - and every
// warp forms the same scalars from the received vectors in the same order:
//   beta = -sign(x0)||x||,  alpha_c = tau v^T P_c = P_ic - (x^T P_c)/beta,
//   v = x / (x0 - beta)
// so all CTAs hold bit-identical reflectors.
template <int NB, int R, int LT>
__global__ void __launch_bounds__(LT, 1) leaf_reg_kernel(const LeafArgs a) {
  constexpr int LW = LT / 32;
  constexpr int RC = NB < 16 ? NB : 16;  // slots per transpose-reduce chunk
  constexpr int NCH = NB / RC;
  constexpr int SH = 32 / RC;    // lanes holding the same reduced slot
  constexpr int SPW = (NB / LW >= 2) ? NB / LW : 2;  // slots pushed by each pushing warp
  constexpr int NPW = NB / SPW;                       // pushing warps
  constexpr int ROWS = LT * R;                        // rows per CTA
  static_assert(SPW * NPW == NB && NPW <= LW, "slot split");
  extern __shared__ __align__(16) double Ys[];  // [NB][ROWS], epilogue only
  __shared__ double wred[LW][NB];
  __shared__ __align__(16) double recv[2][LEAF_MAXC][NB];
  __shared__ __align__(16) double recv_row[2][NB];
  __shared__ __align__(16) double rowi[NB];
  __shared__ __align__(16) double alw[LW][NB];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double scal[NB][3];  // tau, beta, rinv
  __shared__ double G[NB][NB + 1];
  __shared__ double Ts[NB][NB + 1];
  __shared__ double Rrow[NB][NB + 1];

  const uint32_t rank = cluster_ctarank(), ncta = cluster_nctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)rank * ROWS;
  const bool owner_cta = (base == 0);  // row i < nb <= 32 always lives in CTA 0

#ifdef BR_LEAF_PROF  // phase counters: build with BR_BUILD_PROF=1, run with BR_LEAF_PROF=1
  const bool pr = a.prof != nullptr && rank == 0 && tid == 0;
  long long tp[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tc = pr ? clock64() : 0;
#define BR_PHASE(k)                 \
  if (pr) {                         \
    const long long t_ = clock64(); \
    tp[k] += t_ - tc;               \
    tc = t_;                        \
  }
#else
#define BR_PHASE(k)
#endif
  pdl_wait();  // the panel columns were written by the previous kernel
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned gstep = 0;  // exchange rounds so far (mbarrier buffer / phase)
  // this lane's push targets (slot pair c of this CTA -> CTA q), mapped once
  // (only for the 32-wide leaves: for the narrow ones the extra registers
  // cost more than the per-step index math they save, measured)
  constexpr bool PRE = NB >= 32;
  constexpr int NPP = SPW / 2;  // slot pairs per pushing warp
  constexpr int MAXT = PRE ? (NPP * LEAF_MAXC + 31) / 32 : 1;
  uint32_t ra_recv[MAXT], ra_row[MAXT], ra_mbar[MAXT];
  int tc_[MAXT];
#pragma unroll
  for (int tt = 0; tt < MAXT && PRE; ++tt) {
    const int t = tt * 32 + lane;
    tc_[tt] = -1;
    ra_recv[tt] = ra_row[tt] = ra_mbar[tt] = 0;
    if (warp < NPW && t < NPP * (int)ncta) {
      const int pp = t / (int)ncta;
      const uint32_t q = (uint32_t)(t % (int)ncta);
      const int c = warp * SPW + 2 * pp;
      tc_[tt] = c;
      ra_recv[tt] = map_cluster(&recv[0][rank][c], q);
      ra_row[tt] = map_cluster(&recv_row[0][c], q);
      ra_mbar[tt] = map_cluster(&mbar[0], q);
    }
  }
  // Persistent mode (a.nleaves > 1): the cluster factors the panel's leaves
  // one after another; between leaves the block update of the next leaf's
  // columns runs on the auxiliary stream (flags: done[s] -> aux, aux ->
  // ready[s+1]), so the cluster is launched (and its SMs drained) once per panel.
  for (int leaf = 0; leaf < a.nleaves; ++leaf) {
    const int64_t off = (int64_t)leaf * a.lw;
    const int nb = (a.nleaves == 1) ? a.nb : (int)min((int64_t)a.lw, (int64_t)a.btot - off);
    const int64_t Lr = a.L - off;  // rows of this leaf
    const MatView P = a.P.sub(off, off, Lr, nb);
    double* const Yo = a.Y + off + off * a.ldy;
    double* const Wo = a.W ? a.W + off + off * a.ldw : nullptr;
    double* const tauo = a.tau + off;
    if (leaf > 0) {
      if (tid == 0) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_u32(&a.flags[64 + leaf]) != a.epoch) {
          __nanosleep(64);
          if (globaltimer_ns() - t0 > 10000000000ull) __trap();  // 10 s: fail loudly, never hang
        }
      }
      __syncthreads();
    }
    int64_t gr[R];
    double p[R][NB];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      gr[k] = base + tid + (int64_t)k * LT;
      const bool valid = gr[k] < Lr;
#pragma unroll
      for (int c = 0; c < NB; ++c) p[k][c] = (valid && c < nb) ? __ldcg(P.at(gr[k], c)) : 0.0;
    }
    if (leaf == 0) cluster_sync_all();  // mbarriers initialized cluster-wide before any st.async
    BR_PHASE(7);
    for (int i = 0; i < nb; ++i, ++gstep) {
      const int buf = gstep & 1;
      const int g0 = NB - i;  // first Gram slot
      if (tid == 0) mbar_arrive_expect_tx(&mbar[buf], ncta * NB * 8 + NB * 8);
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (gr[k] == i) {
#pragma unroll
          for (int c = 0; c < NB; c += 2)
            *reinterpret_cast<double2*>(&rowi[c]) = make_double2(p[k][c], p[k][c + 1]);
        }
      // rows above i keep their final R entries in the registers (captured into
      // Rrow when they reach column 0); masking x removes them from every sum
      double xk[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        xk[k] = (gr[k] >= i) ? p[k][0] : 0.0;
        if (gr[k] < i) Rrow[gr[k]][i] = p[k][0];
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
          for (int k = 0; k < R; ++k) s = fma(xk[k], p[k][c], s);
          v[cc] = s;
        }
        warp_transpose_reduce<RC>(v, lane);
        if ((lane & (SH - 1)) == 0) wred[warp][ch * RC + lane / SH] = v[0];
      }
      BR_PHASE(0);
      __syncthreads();
      BR_PHASE(1);
      // ---- warp w sums and pushes slots [w*SPW, (w+1)*SPW) to every CTA ----
      if (PRE && warp < NPW) {
        const bool push_row = owner_cta;
#pragma unroll
        for (int tt = 0; tt < MAXT; ++tt) {
          const int c = tc_[tt];
          if (c >= 0) {
            double u0[LW], u1[LW];  // fixed pairwise tree over the warps
#pragma unroll
            for (int w = 0; w < LW; ++w) {
              u0[w] = wred[w][c];
              u1[w] = wred[w][c + 1];
            }
#pragma unroll
            for (int h = LW / 2; h >= 1; h >>= 1)
#pragma unroll
              for (int w = 0; w < h; ++w) {
                u0[w] += u0[w + h];
                u1[w] += u1[w + h];
              }
            const uint32_t rm = ra_mbar[tt] + buf * 8u;
            st_async_v2(ra_recv[tt] + buf * (uint32_t)(LEAF_MAXC * NB * 8), u0[0], u1[0], rm);
            if (push_row)
              st_async_v2(ra_row[tt] + buf * (uint32_t)(NB * 8), rowi[c], rowi[c + 1], rm);
          }
        }
      } else if (!PRE && warp < NPW) {
        constexpr int NP = SPW / 2;  // slot pairs per warp
        const int ntask = NP * (int)ncta;
        const bool push_row = owner_cta;
        for (int t0 = 0; t0 < ntask; t0 += 32) {
          const int t = t0 + lane;
          if (t < ntask) {
            const int pp = t / (int)ncta;
            const uint32_t q = (uint32_t)(t % (int)ncta);
            const int c = warp * SPW + 2 * pp;
            double u0[LW], u1[LW];  // fixed pairwise tree over the warps
#pragma unroll
            for (int w = 0; w < LW; ++w) {
              u0[w] = wred[w][c];
              u1[w] = wred[w][c + 1];
            }
#pragma unroll
            for (int h = LW / 2; h >= 1; h >>= 1)
#pragma unroll
              for (int w = 0; w < h; ++w) {
                u0[w] += u0[w + h];
                u1[w] += u1[w + h];
              }
            const uint32_t rm = map_cluster(&mbar[buf], q);
            st_async_v2(map_cluster(&recv[buf][rank][c], q), u0[0], u1[0], rm);
            if (push_row) st_async_v2(map_cluster(&recv_row[buf][c], q), rowi[c], rowi[c + 1], rm);
          }
        }
      }
      BR_PHASE(2);
      while (!mbar_try_wait_cta(&mbar[buf], (gstep >> 1) & 1)) {
      }
      BR_PHASE(3);
      // ---- every warp: the same scalars from the same received vectors ----
      double rinv = 0.0;
      {
        const double pic = (lane < NB) ? recv_row[buf][lane] : 0.0;
        double gq[LEAF_MAXC];  // fixed pairwise tree over the (power-of-two) CTAs
#pragma unroll
        for (int q = 0; q < LEAF_MAXC; ++q)
          gq[q] = (lane < NB && q < (int)ncta) ? recv[buf][q][lane] : 0.0;
#pragma unroll
        for (int h = LEAF_MAXC / 2; h >= 1; h >>= 1)
#pragma unroll
          for (int q = 0; q < h; ++q) gq[q] += gq[q + h];
        const double g = gq[0];
        {
          const double nrm2 = __shfl_sync(0xffffffffu, g, 0);
          const double x0 = __shfl_sync(0xffffffffu, pic, 0);
          // ||x|| and 1/||x|| from one rsqrt; 1/(x0 - beta) by rcp (~1 ulp
          // each, far inside the parity tolerance) to keep the chain short
          double beta = 0.0, rb = 0.0;
          if (nrm2 != 0.0) {
            const double rs = rsqrt(nrm2), nrm = nrm2 * rs;
            beta = (x0 < 0.0) ? nrm : -nrm;
            rb = (x0 < 0.0) ? rs : -rs;
            rinv = __drcp_rn(x0 - beta);
          }
          if (lane < NB)  // tau == 0 (zero column): identity reflector, no update
            alw[warp][lane] = (nrm2 != 0.0 && lane >= 1 && lane < nb - i) ? fma(-g, rb, pic) : 0.0;
          if (warp == 0 && lane == 0) {  // tau = (beta - x0) / beta later, off the critical path
            scal[i][0] = x0;
            scal[i][1] = beta;
            scal[i][2] = rinv;
          }
          if (warp == 0 && lane >= g0 && lane < NB) G[lane - g0][i] = fma(fma(-pic, x0, g), rinv, pic);
          __syncwarp();
        }
      }
      BR_PHASE(4);
      {
        double al[NB];
#pragma unroll
        for (int c = 0; c < NB; c += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(&alw[warp][c]);
          al[c] = t2.x;
          al[c + 1] = t2.y;
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const double vk = (gr[k] == i) ? 1.0 : xk[k] * rinv;  // 0 above row i
#pragma unroll
          for (int c = 0; c < NB - 1; ++c) p[k][c] = fma(-vk, al[c + 1], p[k][c + 1]);
          p[k][NB - 1] = vk;  // Y column i (unit diagonal, zeros above)
        }
      }
      BR_PHASE(6);
    }

    // dependents may start launching once the last leaf's steps are done (an
    // earlier trigger could park them on SMs the aux-stream updates need)
    if (leaf == a.nleaves - 1) pdl_trigger();
    // ---- Y from the register tail (column c at p[k][NB - nb + c]): to shared
    // memory for W and straight to global ----
    if (nb == NB) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const bool ok = gr[k] < Lr;
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          Ys[c * ROWS + tid + k * LT] = p[k][c];
          if (ok) Yo[gr[k] + (int64_t)c * a.ldy] = p[k][c];
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) {
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          const int src = NB - nb + c;  // runtime-dependent: select from the array
          double y = 0.0;
#pragma unroll
          for (int m = 0; m < NB; ++m)
            if (m == src) y = p[k][m];
          y = (c < nb) ? y : 0.0;
          Ys[c * ROWS + tid + k * LT] = y;
          if (c < nb && gr[k] < Lr) Yo[gr[k] + (int64_t)c * a.ldy] = y;
        }
      }
    }
    // ---- R rows (owner CTA) ----
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (gr[k] < nb) {
        const int r = (int)gr[k];
        for (int c = r; c < nb; ++c) *P.at(r, c) = (c == r) ? scal[r][1] : Rrow[r][c];
      }
    }
    // ---- tau = (beta - x0) / beta (ref kernels.py:109) ----
    if (tid < nb) {
      const double be = scal[tid][1];
      scal[tid][0] = (be != 0.0) ? (be - scal[tid][0]) / be : 0.0;
    }
    __syncthreads();
    // ---- T by the reference recurrence (ref kernels.py:152-162): lane r owns
    // row r in registers, T[r][i] = -tau_i sum_{c<i} T[r][c] G[c][i]
    // (T[r][c] = 0 for c < r) ----
    if (warp == 0 && lane < NB) {
      const int r = lane;
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
#pragma unroll
      for (int c = 0; c < NB; ++c) Ts[r][c] = tr[c];
    }
    __syncthreads();
    BR_PHASE(8);
    BR_PHASE(9);
    // ---- W = Y T on the tensor cores: each warp 4 independent 8-row slabs
    // at a time x NB columns ----
    if constexpr (NB >= 8) if (Wo) {  // (the narrow tall-panel leaves never form W)
      const int gq = lane >> 2, tq = lane & 3;
      constexpr int U = 4;
      for (int rb = warp * 8; rb < ROWS; rb += LW * 8 * U) {
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
          for (int n = 0; n < NB / 8; ++n)  // B = T, or T^T for the block-reflector form Y T^T
            bt[n] = a.wt ? Ts[n * 8 + gq][k0 + tq] : Ts[k0 + tq][n * 8 + gq];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int r0 = rb + u * LW * 8;
            const double av = (r0 < ROWS) ? Ys[(k0 + tq) * ROWS + r0 + gq] : 0.0;  // A = Y (8 x 4)
#pragma unroll
            for (int n = 0; n < NB / 8; ++n) {
              // T is upper triangular: the 4 x 8 block (k0.., n*8..) is zero when
              // k0 >= n*8 + 8 (B = T) or k0 + 4 <= n*8 (B = T^T); skip those DMMAs
              if (!a.wt && k0 >= n * 8 + 8) continue;
              if (a.wt && k0 + 4 <= n * 8) continue;
              dmma884(acc[u][n][0], acc[u][n][1], av, bt[n]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r0 = rb + u * LW * 8;
          const int64_t row = base + r0 + gq;
          if (r0 < ROWS && row < Lr) {
#pragma unroll
            for (int n = 0; n < NB / 8; ++n)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c = n * 8 + 2 * tq + h;
                if (c < nb) Wo[row + (int64_t)c * a.ldw] = acc[u][n][h];
              }
          }
        }
      }
    }
    BR_PHASE(10);
#undef BR_PHASE
#ifdef BR_LEAF_PROF
    if (pr) {
      for (int k = 0; k < 11; ++k) atomicAdd((unsigned long long*)&a.prof[k], (unsigned long long)tp[k]);
      atomicAdd((unsigned long long*)&a.prof[11], (unsigned long long)(nb + 1));
      atomicAdd((unsigned long long*)&a.prof[12], 1ull);
    }
#endif
    if (rank == 0) {
      if (tid < nb) tauo[tid] = scal[tid][0];
      if (a.T && a.nleaves == 1)
        for (int q = tid; q < nb * nb; q += LT) {
          const int r = q % nb, c = q / nb;
          a.T[r + (int64_t)c * a.ldt] = Ts[r][c];
        }
    }
    if (a.nleaves > 1) {
      // leaf outputs (Y, W, R, tau) visible, then hand the block update to the
      // aux stream; the cluster barrier also protects the smem reused next leaf
      __threadfence();
      cluster_sync_all();
      if (rank == 0 && tid == 0) st_release_u32(&a.flags[leaf], a.epoch);
    }
  }  // leaf
  cluster_sync_all();  // no remote traffic is in flight when any CTA exits
}

}  // namespace br
