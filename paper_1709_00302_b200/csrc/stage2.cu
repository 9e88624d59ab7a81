// Second stage of the two-stage reductions (the reference
// stops at the band):
//   SEVP: symmetric band (bandwidth w, lower triangle) -> tridiagonal (d, e)
//   SVD : upper triangular band (bandwidth w)          -> upper bidiagonal (d, e)
// by Householder bulge chasing, one column (row) per sweep, the task
// sequence of oracle/stage2_oracle.py (reflectors in the reference's
// house_gen convention, ref kernels.py:86-110).
//
// B200 design. The work is latency-bound (each task is O(w^2) flops on a
// w x w block, strictly ordered within a sweep), so the parallelism is the
// pipeline of sweeps: one persistent grid, every CTA resident (sized by the
// occupancy query), CTA q running sweeps q, q + G, q + 2G, ... in order.
// Sweep s publishes the number of tasks it has completed in prog[s]
// (release); task j of sweep s waits (acquire) until sweep s - 1 has
// completed every task that shares a matrix element with it (LAG_SB = 2:
// tasks <= j+1 for the symmetric chase, LAG_BD = 3: tasks <= j+2 for the
// bidiagonal one; the element sets are in the comments below; conflicts
// with older sweeps follow by transitivity). Tasks that do not overlap commute, so the result equals
// the sequential task order to the last bit, whatever the grid size (tested).
// Each task stages its block (at most w x w, w <= 128) in shared memory; all
// matrix loads bypass L1 (ld.global.cg), since other CTAs wrote the data.
#include <algorithm>

#include "driver.cuh"

namespace br {

constexpr int S2_WMAX = 128;
constexpr int LAG_SB = 2, LAG_BD = 3;

struct Stage2Args {
  int64_t n;
  int w;
  double* A;
  int64_t lda;
  int* prog;  // per sweep: tasks completed (1 << 30 when the sweep is done)
  double* d;
  double* e;
};

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i32(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }
// Element loops over an R x C block (R <= LDB - 1, a power of two): the
// row / column split is a mask and a shift, not a division by a runtime R.
#define S2_FOR(R, C, body)                                                      \
  {                                                                             \
    constexpr int WMc = LDB - 1, SHc = ilog2c(LDB - 1);                         \
    static_assert((WMc & (WMc - 1)) == 0, "block height a power of two");      \
    for (int e = threadIdx.x; e < WMc * (C); e += NT) {                         \
      const int i = e & (WMc - 1), c = e >> SHc;                                \
      if (i < (R)) { body; }                                                    \
    }                                                                           \
  }

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // red reused
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < NT / 32; ++q) s += red[q];  // fixed order: identical in every thread
  return s;
}

// Reflector of x (length L, in smem `v`, overwritten by v with v0 = 1):
// beta = -sign(x0)||x||, tau = (beta - x0)/beta, v = x/(x0 - beta); the zero
// vector gives tau = beta = 0, v = e0 (ref kernels.py:86-110).
template <int NT>
__device__ void house_smem(double* v, int L, double* red, double& tau, double& beta) {
  double p = 0.0;
  for (int i = threadIdx.x; i < L; i += NT) p = fma(v[i], v[i], p);
  const double nrm2 = block_sum<NT>(p, red);
  const double x0 = v[0];
  tau = 0.0;
  beta = 0.0;
  double scale = 0.0;
  if (nrm2 != 0.0) {
    const double nrm = sqrt(nrm2);
    beta = (x0 < 0.0) ? nrm : -nrm;
    tau = (beta - x0) / beta;
    scale = 1.0 / (x0 - beta);
  }
  __syncthreads();  // x0 read by everyone
  for (int i = threadIdx.x; i < L; i += NT) v[i] = (i == 0) ? 1.0 : v[i] * scale;
  __syncthreads();
}

// D (L x L, symmetric, full in smem, ld LDB) := H D H, H = I - tau v v^T.
// The rank-2 update is formed without FMA so that D stays exactly symmetric.
template <int NT, int LDB>
__device__ void two_sided_smem(double* D, int L, const double* v, double tau, double* y, double* red) {
  for (int i = threadIdx.x; i < L; i += NT) {
    double s = 0.0;
    for (int c = 0; c < L; ++c) s = fma(D[c * LDB + i], v[c], s);
    y[i] = tau * s;
  }
  __syncthreads();
  double p = 0.0;
  for (int i = threadIdx.x; i < L; i += NT) p = fma(v[i], y[i], p);
  const double a = 0.5 * tau * block_sum<NT>(p, red);
  for (int i = threadIdx.x; i < L; i += NT) y[i] = fma(-a, v[i], y[i]);  // y := w
  __syncthreads();
  S2_FOR(L, L, D[c * LDB + i] -= __dadd_rn(__dmul_rn(v[i], y[c]), __dmul_rn(y[i], v[c])));
  __syncthreads();
}

// Symmetric block A[r0 : r0+L]^2 from its lower triangle into smem (full).
template <int NT, int LDB>
__device__ void load_sym(double* D, const Stage2Args& a, int64_t r0, int L) {
  S2_FOR(L, L, D[c * LDB + i] = __ldcg(&a.A[(r0 + max(i, c)) + (r0 + min(i, c)) * a.lda]));
  __syncthreads();
}
template <int NT, int LDB>
__device__ void store_lower(const double* D, const Stage2Args& a, int64_t r0, int L) {
  S2_FOR(L, L, if (i >= c) a.A[(r0 + i) + (r0 + c) * a.lda] = D[c * LDB + i]);
}
template <int NT, int LDB>
__device__ void load_blk(double* O, const Stage2Args& a, int64_t r0, int64_t c0, int R, int Cn) {
  S2_FOR(R, Cn, O[c * LDB + i] = __ldcg(&a.A[(r0 + i) + (c0 + c) * a.lda]));
  __syncthreads();
}
template <int NT, int LDB>
__device__ void store_blk(const double* O, const Stage2Args& a, int64_t r0, int64_t c0, int R, int Cn) {
  S2_FOR(R, Cn, a.A[(r0 + i) + (c0 + c) * a.lda] = O[c * LDB + i]);
}

// `seen` (thread 0's register): the last progress value read for sweep
// s - 1; the acquire load is skipped while it already covers the need.
__device__ __forceinline__ void wait_prev(const Stage2Args& a, int64_t s, int need, int& seen) {
  if (threadIdx.x == 0 && s > 0) {
    while (seen < need) seen = ld_acquire_i32(&a.prog[s - 1]);
  }
  __syncthreads();
}
// The CTA barrier orders every thread's stores of the task before thread
// 0's release store (st.release carries the gpu-scope fence).
__device__ __forceinline__ void publish(const Stage2Args& a, int64_t s, int done) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_i32(&a.prog[s], done);
}

// ---------------------------------------------------------------------------
// SEVP: band -> tridiagonal. With r_j = s + 1 + j w, sweep s task 0 writes
// column s (rows [r_0, r_0+w)) and D_0 = [r_0, r_0+w)^2 (lower); task j >= 1
// writes O_j = rows [r_j, r_j+w) x cols [r_{j-1}, r_j) and D_j. Sweep s+1
// (all indices + 1) task j shares elements with sweep s tasks j (D_j, O_j)
// and j+1 (row r_{j+1} = r_j + w of O_{j+1} and D_{j+1}), none with j+2
// (its rows start at r_j + 2w): wait until sweep s - 1 has done j + 2 tasks.
// ---------------------------------------------------------------------------
template <int NT, int WM>
__global__ void __launch_bounds__(NT) sb2st_kernel(const Stage2Args a) {
  constexpr int LDB = WM + 1;
  extern __shared__ __align__(16) double sm[];
  double* B = sm;                 // [WM][LDB] the task's block
  double* v = B + WM * LDB;       // current reflector (H of the previous task)
  double* v2 = v + WM;            // new reflector
  double* y = v2 + WM;            // work vector
  double* red = y + WM;           // [32]
  pdl_wait();
  const int64_t n = a.n;
  const int w = a.w;
  for (int64_t s = blockIdx.x; s + 2 < n; s += gridDim.x) {
    int64_t r = s + 1;
    int L = (int)min((int64_t)w, n - r);
    int task = 0, seen = 0;
    wait_prev(a, s, LAG_SB, seen);
    if (L >= 2) {
      // ---- task 0: annihilate column s below the subdiagonal ----
      for (int i = threadIdx.x; i < L; i += NT) v[i] = __ldcg(&a.A[(r + i) + s * a.lda]);
      __syncthreads();
      double tau, beta;
      house_smem<NT>(v, L, red, tau, beta);
      for (int i = threadIdx.x; i < L; i += NT) a.A[(r + i) + s * a.lda] = (i == 0) ? beta : 0.0;
      load_sym<NT, LDB>(B, a, r, L);
      two_sided_smem<NT, LDB>(B, L, v, tau, y, red);
      store_lower<NT, LDB>(B, a, r, L);
      publish(a, s, ++task);
      // ---- chase ----
      while (true) {
        const int64_t rb = r + L;
        const int L2 = (int)min((int64_t)w, n - rb);
        if (L2 <= 0) break;
        wait_prev(a, s, task + LAG_SB, seen);
        load_blk<NT, LDB>(B, a, rb, r, L2, L);
        // O := O H
        for (int i = threadIdx.x; i < L2; i += NT) {
          double t = 0.0;
          for (int c = 0; c < L; ++c) t = fma(B[c * LDB + i], v[c], t);
          y[i] = tau * t;
        }
        __syncthreads();
        S2_FOR(L2, L, B[c * LDB + i] = fma(-y[i], v[c], B[c * LDB + i]));
        __syncthreads();
        double tau2 = 0.0, beta2 = 0.0;
        if (L2 >= 2) {
          // H2 annihilates O[1:, 0]; O[:, 1:] := H2 O[:, 1:]
          for (int i = threadIdx.x; i < L2; i += NT) v2[i] = B[i];
          __syncthreads();
          house_smem<NT>(v2, L2, red, tau2, beta2);
          for (int c = 1 + threadIdx.x; c < L; c += NT) {
            double t = 0.0;
            for (int i = 0; i < L2; ++i) t = fma(v2[i], B[c * LDB + i], t);
            y[c] = tau2 * t;
          }
          __syncthreads();
          S2_FOR(L2, L, if (c == 0) B[i] = (i == 0) ? beta2 : 0.0;
                 else B[c * LDB + i] = fma(-v2[i], y[c], B[c * LDB + i]));
          __syncthreads();
        }
        store_blk<NT, LDB>(B, a, rb, r, L2, L);
        if (L2 < 2) {
          publish(a, s, ++task);
          break;
        }
        __syncthreads();
        load_sym<NT, LDB>(B, a, rb, L2);
        two_sided_smem<NT, LDB>(B, L2, v2, tau2, y, red);
        store_lower<NT, LDB>(B, a, rb, L2);
        for (int i = threadIdx.x; i < L2; i += NT) v[i] = v2[i];
        tau = tau2;
        publish(a, s, ++task);
        __syncthreads();
        r = rb;
        L = L2;
      }
    }
    publish(a, s, 1 << 30);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// SVD: upper triangular band -> upper bidiagonal. Sweep s task j >= 1
// (r = s+1+(j-1)w, c0 = r+w) writes rows [r, c0+w) x cols [c0, c0+w) (the
// right reflector of row r) and rows [c0, c0+w) x cols [c0, c0+2w) (the left
// reflector of column c0); task 0 the same shape from row s / column s+1.
// Sweep s+1 task j shares elements with sweep s tasks up to j+2 (the single
// element (c0+w, c0+2w) of task j+2), none with j+3 (its rows start at
// c0 + 2w): wait until sweep s - 1 has done j + 3 tasks.
// ---------------------------------------------------------------------------
template <int NT, int WM>
__global__ void __launch_bounds__(NT) tb2bd_kernel(const Stage2Args a) {
  constexpr int LDB = WM + 1;
  extern __shared__ __align__(16) double sm[];
  double* B = sm;             // [WM][LDB]: one chunk of a block (<= w x w)
  double* v = B + WM * LDB;
  double* y = v + WM;
  double* red = y + WM;
  pdl_wait();
  const int64_t n = a.n;
  const int w = a.w;
  // right reflector (v, length L) on columns [c0, c0+L), applied to rows
  // [r0, r1) in chunks of WM rows: A[r0:r1, c0:c0+L] -= (A v) tau v^T
  auto apply_right = [&](int64_t r0, int64_t r1, int64_t c0, int L, double tau) {
    for (int64_t rr = r0; rr < r1; rr += WM) {
      const int Rb = (int)min((int64_t)WM, r1 - rr);
      load_blk<NT, LDB>(B, a, rr, c0, Rb, L);
      for (int i = threadIdx.x; i < Rb; i += NT) {
        double t = 0.0;
        for (int c = 0; c < L; ++c) t = fma(B[c * LDB + i], v[c], t);
        y[i] = tau * t;
      }
      __syncthreads();
      S2_FOR(Rb, L, B[c * LDB + i] = fma(-y[i], v[c], B[c * LDB + i]));
      __syncthreads();
      store_blk<NT, LDB>(B, a, rr, c0, Rb, L);
      __syncthreads();
    }
  };
  // left reflector (v, length L) on rows [r0, r0+L), applied to columns
  // [c0, c1) in chunks of WM columns: A[r0:r0+L, c0:c1] -= v tau (v^T A)
  auto apply_left = [&](int64_t r0, int L, int64_t c0, int64_t c1, double tau) {
    for (int64_t cc = c0; cc < c1; cc += WM) {
      const int Cb = (int)min((int64_t)WM, c1 - cc);
      load_blk<NT, LDB>(B, a, r0, cc, L, Cb);
      for (int c = threadIdx.x; c < Cb; c += NT) {
        double t = 0.0;
        for (int i = 0; i < L; ++i) t = fma(v[i], B[c * LDB + i], t);
        y[c] = tau * t;
      }
      __syncthreads();
      S2_FOR(L, Cb, B[c * LDB + i] = fma(-v[i], y[c], B[c * LDB + i]));
      __syncthreads();
      store_blk<NT, LDB>(B, a, r0, cc, L, Cb);
      __syncthreads();
    }
  };
  for (int64_t s = blockIdx.x; s + 1 < n; s += gridDim.x) {
    int task = 0, seen = 0;
    wait_prev(a, s, LAG_BD, seen);
    // ---- task 0 ----
    const int L = (int)min((int64_t)w, n - s - 1);
    if (L >= 2) {  // right reflector on row s
      for (int c = threadIdx.x; c < L; c += NT) v[c] = __ldcg(&a.A[s + (s + 1 + c) * a.lda]);
      __syncthreads();
      double tau, beta;
      house_smem<NT>(v, L, red, tau, beta);
      for (int c = threadIdx.x; c < L; c += NT) a.A[s + (s + 1 + c) * a.lda] = (c == 0) ? beta : 0.0;
      apply_right(s + 1, s + 1 + L, s + 1, L, tau);
    }
    int64_t r = s + 1;
    int Lr = (int)min((int64_t)w, n - r);
    if (L >= 1 && Lr >= 2) {
      // left reflector on column r, rows [r, r+Lr)
      for (int i = threadIdx.x; i < Lr; i += NT) v[i] = __ldcg(&a.A[(r + i) + r * a.lda]);
      __syncthreads();
      double tau, beta;
      house_smem<NT>(v, Lr, red, tau, beta);
      for (int i = threadIdx.x; i < Lr; i += NT) a.A[(r + i) + r * a.lda] = (i == 0) ? beta : 0.0;
      apply_left(r, Lr, r + 1, min(n, r + Lr + w), tau);
      publish(a, s, ++task);
      // ---- chase ----
      while (true) {
        const int64_t c0 = r + Lr;
        const int L2 = (int)min((int64_t)w, n - c0);
        if (L2 <= 0) break;
        wait_prev(a, s, task + LAG_BD, seen);
        if (L2 >= 2) {  // right reflector on row r, columns [c0, c0+L2)
          for (int c = threadIdx.x; c < L2; c += NT) v[c] = __ldcg(&a.A[r + (c0 + c) * a.lda]);
          __syncthreads();
          double tau2, beta2;
          house_smem<NT>(v, L2, red, tau2, beta2);
          for (int c = threadIdx.x; c < L2; c += NT) a.A[r + (c0 + c) * a.lda] = (c == 0) ? beta2 : 0.0;
          apply_right(r + 1, c0 + L2, c0, L2, tau2);
        } else {
          publish(a, s, ++task);
          break;
        }
        // left reflector on column c0, rows [c0, c0+L2)
        for (int i = threadIdx.x; i < L2; i += NT) v[i] = __ldcg(&a.A[(c0 + i) + c0 * a.lda]);
        __syncthreads();
        double tau3, beta3;
        house_smem<NT>(v, L2, red, tau3, beta3);
        for (int i = threadIdx.x; i < L2; i += NT) a.A[(c0 + i) + c0 * a.lda] = (i == 0) ? beta3 : 0.0;
        apply_left(c0, L2, c0 + 1, min(n, c0 + L2 + w), tau3);
        publish(a, s, ++task);
        r = c0;
        Lr = L2;
      }
    }
    publish(a, s, 1 << 30);
    __syncthreads();
  }
}

__global__ void diag_pair_kernel(int64_t n, const double* A, int64_t lda, int sub, double* d,
                                 double* e) {
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    d[i] = A[i + i * lda];
    if (i + 1 < n) e[i] = sub ? A[(i + 1) + i * lda] : A[i + (i + 1) * lda];
  }
}

static size_t s2_smem(int wm) { return sizeof(double) * ((size_t)wm * (wm + 1) + 3 * wm + 32); }

template <int NT, int WM>
static int launch_stage2(bool bd, cudaStream_t st, const Stage2Args& a, int num_sms, int max_ctas) {
  auto kern = bd ? tb2bd_kernel<NT, WM> : sb2st_kernel<NT, WM>;
  const size_t smem = s2_smem(WM);
  BR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (g_preload_only) return 0;
  int occ = 0;
  BR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
  if (occ < 1) {
    set_error("stage2: kernel does not fit an SM");
    return -1;
  }
  // every CTA resident (the sweeps wait on each other): at most one wave
  int64_t G = (int64_t)num_sms * occ;
  G = std::min<int64_t>(G, std::max<int64_t>(1, a.n - (bd ? 1 : 2)));
  if (max_ctas > 0) G = std::min<int64_t>(G, max_ctas);
  BR_CUDA(cudaMemsetAsync(a.prog, 0, sizeof(int) * std::max<int64_t>(a.n, 1), st));
  count_launch();
  BR_CUDA(launch_pdl(kern, dim3((unsigned)G), dim3(NT), smem, st, a));
  return 0;
}

// Grid cap for the stage-2 kernels (BR_S2_CTAS; 0 = the whole device). A cap
// of 1 runs the sweeps one after another in one CTA (the sequential order):
// the tests compare it bitwise with the pipelined grid.
static int s2_max_ctas() {
  const char* e = std::getenv("BR_S2_CTAS");
  return e ? std::atoi(e) : 0;
}

// Threads per CTA (BR_S2_THREADS = 128 / 256 / 512 / 1024 overrides; 0 =
// per-width default). The per-task element loops dominate: tridiagonal
// n = 2048, w = 32 with 128 / 256 / 512 / 1024 threads 32.4 / 24.9 / 24.0 /
// 24.9 ms; n = 8192, w = 64 350 / 241 / 175 ms (128 / 256 / 512); w = 128
// 666 / 460 / 431 ms (256 / 512 / 1024). Defaults: 512, 512, 1024.
static int s2_threads() {
  const char* e = std::getenv("BR_S2_THREADS");
  const int t = e ? std::atoi(e) : 0;
  return (t == 128 || t == 256 || t == 512 || t == 1024) ? t : 0;
}

int band_to_condensed(cudaStream_t st, bool bd, int64_t n, int64_t w, double* A, int64_t lda,
                      double* d, double* e, int* prog, int num_sms) {
  if (n < 1) return 0;
  if (w > S2_WMAX) {
    set_error("band_to_%s: bandwidth %lld > %d (second stage handles w <= %d)",
              bd ? "bidiag" : "tridiag", (long long)w, S2_WMAX, S2_WMAX);
    return -2;
  }
  Stage2Args a{n, (int)w, A, lda, prog, d, e};
  const int cap = s2_max_ctas();
  if (n > 2 || (bd && n > 1)) {
    const int nt = s2_threads();
    if (w <= 32) {
      if (nt == 128) BR_CHECK((launch_stage2<128, 32>(bd, st, a, num_sms, cap)));
      else if (nt == 256) BR_CHECK((launch_stage2<256, 32>(bd, st, a, num_sms, cap)));
      else BR_CHECK((launch_stage2<512, 32>(bd, st, a, num_sms, cap)));
    } else if (w <= 64) {
      if (nt == 128) BR_CHECK((launch_stage2<128, 64>(bd, st, a, num_sms, cap)));
      else if (nt == 256) BR_CHECK((launch_stage2<256, 64>(bd, st, a, num_sms, cap)));
      else BR_CHECK((launch_stage2<512, 64>(bd, st, a, num_sms, cap)));
    } else {
      if (nt == 256) BR_CHECK((launch_stage2<256, 128>(bd, st, a, num_sms, cap)));
      else if (nt == 512) BR_CHECK((launch_stage2<512, 128>(bd, st, a, num_sms, cap)));
      else BR_CHECK((launch_stage2<1024, 128>(bd, st, a, num_sms, cap)));
    }
  }
  const int blocks = (int)std::min<int64_t>(cdiv(n, 256), 1024);
  count_launch();
  BR_CUDA(launch_pdl(diag_pair_kernel, dim3(blocks), dim3(256), 0, st, n, (const double*)A, lda,
                     bd ? 0 : 1, d, e));
  return 0;
}

int preload_stage2_kernels() {
  Stage2Args a{};
  for (bool bd : {false, true}) {
    BR_CHECK((launch_stage2<128, 32>(bd, 0, a, 148, 0)));
    BR_CHECK((launch_stage2<256, 32>(bd, 0, a, 148, 0)));
    BR_CHECK((launch_stage2<512, 32>(bd, 0, a, 148, 0)));
    BR_CHECK((launch_stage2<128, 64>(bd, 0, a, 148, 0)));
    BR_CHECK((launch_stage2<256, 64>(bd, 0, a, 148, 0)));
    BR_CHECK((launch_stage2<512, 64>(bd, 0, a, 148, 0)));
    BR_CHECK((launch_stage2<256, 128>(bd, 0, a, 148, 0)));
    BR_CHECK((launch_stage2<512, 128>(bd, 0, a, 148, 0)));
    BR_CHECK((launch_stage2<1024, 128>(bd, 0, a, 148, 0)));
  }
  cudaFuncAttributes fa;
  BR_CUDA(cudaFuncGetAttributes(&fa, diag_pair_kernel));
  return 0;
}

}  // namespace br
