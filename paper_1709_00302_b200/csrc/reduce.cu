// The two first-stage reductions with static look-ahead, as stream programs.
//
// SEVP  (ref sevp.py:110-324): dense symmetric -> symmetric band.
// Triband SVD (ref svd.py:179-247): dense general (m >= n) -> upper
//   triangular-band.
//
// Look-ahead (ref sevp.py:209-273, PAPER.md T1/T2): the reference's two
// worker groups T_S / T_P become two CUDA streams of one context: `panel`
// (high priority, the T_S role) factors the next panel while `main` (the
// T_P role) finishes the rest of the current trailing update. The updates
// that touch the next panel's columns are issued first on `main`, then an
// event hands the panel to the panel stream. Every update kernel is
// split-invariant (fixed K order, no atomics), so look-ahead depth 1 is
// bitwise identical to depth 0 on the same GPU.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "driver.cuh"
#include "gemm.cuh"

namespace br {

static double gemm_flops(double m, double n, double k) { return 2.0 * m * n * k; }
// Lower-triangle SYR2K columns [c0, c1) of a j x j matrix, rank 2*bp.
static double syr2k_flops(int64_t j, int64_t bp, int64_t c0, int64_t c1) {
  double s = 0.0;  // sum_{c=c0}^{c1-1} (j - c)
  s = (double)(c1 - c0) * (double)j - 0.5 * ((double)c1 * (c1 - 1) - (double)c0 * (c0 - 1));
  return 4.0 * (double)bp * s;
}
// CTA cap for the split-K GEMMs inside a panel factorization (0 = none):
// while the trailing update is large, the panel stream's GEMMs run on few
// CTAs so they steal fewer SM slots from the update (tuning: BR_PANEL_CAP,
// BR_PANEL_CAP_ROWS). Depends only on the panel height, so the schedule with
// and without look-ahead makes the same choice (bitwise equality).
static int panel_cap(int64_t rows) {
  static int cap = -1;
  static int64_t min_rows = 6144;
  if (cap < 0) {
    const char* e = std::getenv("BR_PANEL_CAP");
    cap = e ? std::atoi(e) : 0;
    if (const char* r = std::getenv("BR_PANEL_CAP_ROWS")) min_rows = std::atoll(r);
  }
  return rows >= min_rows ? cap : 0;
}

// Trailing heights at or below which the triangular-band reduction pipelines
// its Z products with the panels (BR_PZ_ROWS; default 0 = off). Measured on
// c4 (2 x 3 runs): off 447.2 ms, 6144 445.9 ms, 8192 446.3 ms, 10240 469 ms
// (the 16-wide leaves of taller panels make the leaf products too small to
// hide); the 0.3 % is within run-to-run spread of bench.py, and the
// 32-row leaf products lower the GEMM class's DMMA efficiency, so it is off.
static int64_t pz_rows() {
  static int64_t r = -1;
  if (r < 0) {
    const char* e = std::getenv("BR_PZ_ROWS");
    r = e ? std::atoll(e) : 0;
  }
  return r;
}

// The fused X-product launch (xchain, BR_XCHAIN=1) for narrow panels.
// Measured on c1 (one box, 2 x 3 steps): 5.68 ms fused vs 5.62 ms with the
// separate SYMM / X2 / X3 kernels - the three grid barriers and the lost
// PDL overlap of the next launch cost what the saved launches win - so off.
static bool xchain_enabled() {
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("BR_XCHAIN");
    m = (e && std::atoi(e) == 1) ? 1 : 0;
  }
  return m == 1;
}

// Narrow panels (b <= 64): Z_L's split-K reduction also updates the LQ
// panel's rows, Z_R's the next QR panel's columns (gemm_left_update /
// gemm_right_update: one launch instead of reduction + small GEMM on the
// panel chain). BR_FUSE_SMALL=0: separate kernels (A/B aid). Used by both
// look-ahead depths, so they stay bitwise equal.
static bool fuse_small() {
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("BR_FUSE_SMALL");
    m = (e && std::atoi(e) == 0) ? 0 : 1;
  }
  return m == 1;
}

static double panel_flops(int64_t j, int64_t b) {
  return 2.0 * j * b * b - 2.0 * b * b * b / 3.0 + (double)j * b * b;  // QR + T/W
}

// ---------------------------------------------------------------------------
// SEVP
// ---------------------------------------------------------------------------
// The strict SM split (confined tall panels, two-phase panel) is wired into the
// triangular band only: the other reductions keep their panels unconfined.
struct NoSplit {
  Workspace& ws;
  int64_t saved;
  explicit NoSplit(Workspace& w) : ws(w), saved(w.green_rows) {
    if (ws.split_upd) ws.green_rows = INT64_MAX;
  }
  ~NoSplit() { ws.green_rows = saved; }
};

int sevp_reduce(Workspace& ws, int64_t n, int64_t w, int64_t b, int lookahead, double* A,
                int64_t lda, double* Q, int64_t ldq, int64_t* iterations, BandOut* bo) {
  NoSplit nosplit(ws);
  std::vector<int64_t> ks;
  for (int64_t k = 0; n - k - w >= 2; k += std::min(b, n - k - w)) ks.push_back(k);
  // partial reduction (BR_OPT_MAX_ITERS): the first max_iters panels only,
  // raw working matrix out (no finalize, no streamed finalized blocks)
  const bool partial = ws.max_iters > 0 && ws.max_iters < (int64_t)ks.size();
  if (partial) ks.resize((size_t)ws.max_iters);
  BandOut* bof = partial ? nullptr : bo;
  *iterations = (int64_t)ks.size();
  if (ks.empty()) {  // n <= w + 1: input returned unchanged (sevp.py:302-305)
    if (bo) {
      BR_CUDA(cudaMemcpy2DAsync(bo->host, bo->ldh * sizeof(double), A, lda * sizeof(double),
                                n * sizeof(double), n, cudaMemcpyDeviceToHost, ws.main));
      bo->done = n;
    }
    return 0;
  }

  const int64_t jmax = n - w;
  // factor buffers: Y[2], W[2] (jmax x b), T[2] (b x b), tau[2] (b), X1, X3
  // (jmax x b), X2 (b x b), Zm (b x w) mid-block temp, ZQ (n x b)
  const int64_t nY = jmax * b, nT = b * b;
  const int64_t total = 4 * nY + 2 * nT + 2 * b + 2 * nY + nT + b * w + n * b;
  BR_CHECK(devbuf_reserve(ws.factors, total));
  BR_CHECK(devbuf_reserve(ws.skbuf_main, 4 * n * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.skbuf_panel, 4 * jmax * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.skbuf_aux, 4 * jmax * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.pscratch, panel_scratch_doubles(b)));
  ws.sk_main = Scratch{ws.skbuf_main.p, ws.skbuf_main.cap, ws.num_sms};
  ws.sk_panel = Scratch{ws.skbuf_panel.p, ws.skbuf_panel.cap, ws.num_sms};
  ws.sk_aux = Scratch{ws.skbuf_aux.p, ws.skbuf_aux.cap, ws.num_sms};
  double* f = ws.factors.p;
  double *Yb[2], *Wb[2], *Tb[2], *taub[2];
  for (int p = 0; p < 2; ++p) {
    Yb[p] = f; f += nY;
    Wb[p] = f; f += nY;
  }
  for (int p = 0; p < 2; ++p) {
    Tb[p] = f; f += nT;
  }
  for (int p = 0; p < 2; ++p) {
    taub[p] = f; f += b;
  }
  double* X1b = f; f += nY;
  double* X3b = f; f += nY;
  double* X2b = f; f += nT;
  double* Zm = f; f += b * w;
  double* ZQ = f; f += n * b;

  if (Q) BR_CHECK(set_identity(ws.main, Q, ldq, n));
  auto Aat = [&](int64_t r, int64_t c) { return A + r + c * lda; };

  auto do_panel = [&](cudaStream_t st, Scratch& sk, int64_t k, int par) -> int {
    const int64_t bp = std::min(b, n - k - w), j = n - k - w;
    MatView P(Aat(k + w, k), lda, j, bp);
    MatView Y(Yb[par], jmax, j, bp), T(Tb[par], b, bp, bp), W(Wb[par], jmax, j, bp);
    TimeScope ts(ws, st, TC_PANEL, panel_flops(j, bp), "qr", k);
    Scratch s = ws.pscratch_for(sk, j);
    BR_CHECK(panel_qr(st, s, ws.pscratch, P, Y, taub[par], T, &W, panel_cap(j), &ws));
    return store_factors(ws, st, 0, k, k + w, j, bp, Yb[par], jmax, Tb[par], b, taub[par]);
  };

  cudaEvent_t ev_panel = nullptr;
  BR_CHECK(do_panel(ws.main, ws.sk_main, ks[0], 0));
  for (size_t idx = 0; idx < ks.size(); ++idx) {
    const int64_t k = ks[idx];
    const int64_t bp = std::min(b, n - k - w), j = n - k - w;
    const int par = (int)(idx & 1);
    if (ev_panel) {
      BR_CUDA(cudaStreamWaitEvent(ws.main, ev_panel, 0));
      ev_panel = nullptr;
    }
    MatView Y(Yb[par], jmax, j, bp), W(Wb[par], jmax, j, bp);
    MatView A2(Aat(k + w, k + w), lda, j, j);
    const bool has_next = idx + 1 < ks.size();
    const int64_t kn = has_next ? ks[idx + 1] : 0;
    const int64_t bpn = has_next ? std::min(b, n - kn - w) : 0;
    const int64_t split = has_next ? std::max<int64_t>(0, bp + bpn - w) : 0;
    const bool la = lookahead && has_next;

    // mid block A[k+w:n, k+bp:k+w] := Q^T mid (ref sevp.py:147-153)
    // split-K chunks of the whole mid-block products: pieces sum in the same order
    const int64_t kps_z = gemm_plan_kps(ws.sk_main, MatView(Zm, b, bp, w - bp), W.T(),
                                        MatView(Aat(k + w, k + bp), lda, j, w - bp), 0.0);
    const int64_t kps_u = gemm_plan_kps(ws.sk_main, MatView(Aat(k + w, k + bp), lda, j, w - bp), Y,
                                        MatView(Zm, b, bp, w - bp), 1.0);
    auto mid = [&](int64_t c0, int64_t c1, const char* tag) -> int {
      if (c0 >= c1) return 0;
      MatView M(Aat(k + w, c0), lda, j, c1 - c0);
      MatView Z(Zm + (c0 - k - bp) * b, b, bp, c1 - c0);
      TimeScope ts(ws, ws.main, TC_GEMM, 2 * gemm_flops(bp, c1 - c0, j), tag, k);
      BR_CHECK(gemm(ws.main, ws.sk_main, Z, W.T(), M, 1.0, 0.0, nullptr, 0, kps_z));
      return gemm(ws.main, ws.sk_main, M, Y, Z, 1.0, 1.0, nullptr, 0, kps_u);
    };
    // X1 = sym(A2) W; X2 = 1/2 X1^T W; X3 = X1 + Y X2 (ref sevp.py:156-176)
    auto xprods = [&]() -> int {
      MatView X1(X1b, jmax, j, bp), X3(X3b, jmax, j, bp), X2(X2b, b, bp, bp);
      if (xchain_enabled()) {  // narrow panels: the three products in one launch
        TimeScope ts(ws, ws.main, TC_SYMM,
                     gemm_flops(j, bp, j) + gemm_flops(bp, bp, j) + gemm_flops(j, bp, bp), "xchain", k);
        const int r = xchain(ws.main, ws.sk_main, X1, X2, X3, A2, W, Y, ws.flags + 128);
        if (r <= 0) return r;
      }
      {
        TimeScope ts(ws, ws.main, TC_SYMM, gemm_flops(j, bp, j), "xprod1", k);
        BR_CHECK(symm_lower(ws.main, ws.sk_main, X1, A2, W));
      }
      TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(bp, bp, j) + gemm_flops(j, bp, bp), "xprod3", k);
      BR_CHECK(gemm(ws.main, ws.sk_main, X2, X1.T(), W, 0.5, 0.0));
      return gemm(ws.main, ws.sk_main, X3, Y, X2, 1.0, 1.0, &X1);
    };
    // `overlap`: this piece runs beside the next panel's factorization; where the
    // panel chain bounds the iteration it goes to the SM-partitioned stream
    // (Workspace::gupd), ordered after / before the main stream by events
    auto trail = [&](int64_t c0, int64_t c1, const char* tag, bool overlap = false) -> int {
      if (c0 >= c1) return 0;
      MatView X3(X3b, jmax, j, bp);
      cudaStream_t us = ws.ustream(j, overlap);
      if (us != ws.main) {
        cudaEvent_t ev = ws_event(ws);
        BR_CUDA(cudaEventRecord(ev, ws.main));
        BR_CUDA(cudaStreamWaitEvent(us, ev, 0));
      }
      {
        TimeScope ts(ws, us, TC_SYR2K, syr2k_flops(j, bp, c0, c1), tag, k);
        BR_CHECK(syr2k_lower(us, A2, X3, Y, c0, c1));
      }
      if (us != ws.main) {
        cudaEvent_t ev = ws_event(ws);
        BR_CUDA(cudaEventRecord(ev, us));
        BR_CUDA(cudaStreamWaitEvent(ws.main, ev, 0));
      }
      return 0;
    };
    // Q[:, k+w:n] := Q[:, k+w:n] (I + W Y^T) (ref sevp.py:138-144)
    auto accq = [&]() -> int {
      if (!Q) return 0;
      MatView Qs(Q + (k + w) * ldq, ldq, n, j);
      MatView Z(ZQ, n, n, bp);
      TimeScope ts(ws, ws.main, TC_GEMM, 2 * gemm_flops(n, bp, j), "accq", k);
      BR_CHECK(gemm(ws.main, ws.sk_main, Z, Qs, W, 1.0, 0.0));
      return gemm(ws.main, ws.sk_main, Qs, Z, Y.T(), 1.0, 1.0);
    };
    auto launch_next_panel = [&]() -> int {
      cudaStream_t ps = ws.pstream(n - kn - w);
      cudaEvent_t ev = ws_event(ws);
      BR_CUDA(cudaEventRecord(ev, ws.main));
      BR_CUDA(cudaStreamWaitEvent(ps, ev, 0));
      BR_CHECK(do_panel(ps, ws.sk_panel, kn, par ^ 1));
      ev_panel = ws_event(ws);
      BR_CUDA(cudaEventRecord(ev_panel, ps));
      return 0;
    };

    if (la && split == 0) {
      // V1 regime (2b <= w): next panel lies inside the mid block
      const int64_t h1 = std::min(k + bp + bpn, k + w);
      BR_CHECK(mid(k + bp, h1, "mid-head"));
      BR_CHECK(launch_next_panel());
      BR_CHECK(mid(h1, k + w, "mid-rest"));
      BR_CHECK(xprods());
      BR_CHECK(trail(0, j, "trail"));
      BR_CHECK(accq());
    } else if (la) {
      // V2 regime (2b > w): next panel spills `split` columns into A2
      BR_CHECK(mid(k + bp, k + w, "mid"));
      BR_CHECK(xprods());
      BR_CHECK(trail(0, split, "trail-lead"));
      BR_CHECK(launch_next_panel());
      BR_CHECK(trail(split, j, "trail-rest", true));
      BR_CHECK(accq());
    } else {
      BR_CHECK(mid(k + bp, k + w, "mid"));
      BR_CHECK(xprods());
      BR_CHECK(trail(0, j, "trail"));
      BR_CHECK(accq());
      if (has_next) BR_CHECK(do_panel(ws.main, ws.sk_main, kn, par ^ 1));
    }
    BR_CHECK(band_out_flush(ws, bof, k + bp));  // columns [0, k + bp) are final
  }
  if (partial) {
    BR_CHECK(band_out_raw(ws, bo, n));
    ws_events_reset(ws);
    return 0;
  }
  if (bo) {
    BR_CHECK(band_out_flush(ws, bo, n));
    ws_events_reset(ws);
    return 0;
  }
  ws_events_reset(ws);
  return finalize_sym(ws.main, A, lda, n, w);
}

// ---------------------------------------------------------------------------
// Triangular-band SVD
// ---------------------------------------------------------------------------
int tri_reduce(Workspace& ws, int64_t m, int64_t n, int64_t w, int64_t b, int lookahead,
               double* A, int64_t lda, int64_t* iterations, BandOut* bo) {
  struct It {
    int64_t k, bp;
  };
  std::vector<It> its;
  for (int64_t k = 0; m - k >= 2 && k < n;) {
    const int64_t bp = std::min({b, n - k, m - k});
    its.push_back({k, bp});
    k += bp;
  }
  const bool partial = ws.max_iters > 0 && ws.max_iters < (int64_t)its.size();
  if (partial) its.resize((size_t)ws.max_iters);
  *iterations = (int64_t)its.size();
  BandOut* const bo_full = bo;
  if (partial) bo = nullptr;
  BandIn* bi = ws.band_in;
  if (bi) BR_CHECK(band_in_start(ws, bi));
  if (its.empty()) {
    BR_CHECK(band_in_wait(ws, bi, n));
    if (bo) return band_out_flush(ws, bo, n);
    return mask_tri(ws.main, A, lda, m, n, 0, w);
  }

  const int64_t nYu = m * b, nYv = n * b, nT = b * b;
  const int64_t total = 4 * nYu + 2 * nT + 2 * b + 2 * nYv + nT + b + 2 * (b * n + m * b);
  BR_CHECK(devbuf_reserve(ws.factors, total));
  BR_CHECK(devbuf_reserve(ws.skbuf_main, 4 * std::max(m, n) * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.skbuf_panel, 4 * std::max(m, n) * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.skbuf_aux, 4 * std::max(m, n) * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.pscratch, panel_scratch_doubles(b)));
  ws.sk_main = Scratch{ws.skbuf_main.p, ws.skbuf_main.cap, ws.num_sms};
  ws.sk_panel = Scratch{ws.skbuf_panel.p, ws.skbuf_panel.cap, ws.num_sms};
  ws.sk_aux = Scratch{ws.skbuf_aux.p, ws.skbuf_aux.cap, ws.num_sms};
  double* f = ws.factors.p;
  double *Yu[2], *Wu[2], *Tu[2], *tauu[2];
  for (int p = 0; p < 2; ++p) {
    Yu[p] = f; f += nYu;
    Wu[p] = f; f += nYu;
  }
  for (int p = 0; p < 2; ++p) {
    Tu[p] = f; f += nT;
  }
  for (int p = 0; p < 2; ++p) {
    tauu[p] = f; f += b;
  }
  double* Yv = f; f += nYv;
  double* Wv = f; f += nYv;
  double* Tv = f; f += nT;
  double* tauv = f; f += b;
  double* ZL = f; f += b * n;
  double* ZR = f; f += m * b;
  double* ZLr = f; f += b * n;  // Y_U^T E, leaf by leaf (pipelined Z_L)
  double* ZRr = f; f += m * b;  // D Y_V, leaf by leaf (pipelined Z_R)
  LeafMarks mk_qr[2], mk_lq;

  auto Aat = [&](int64_t r, int64_t c) { return A + r + c * lda; };
  // Strict SM split (BR_SPLIT_ROWS, experimental): the leaves and block updates
  // of a tall panel run confined to the reserved SMs (`st` is then the confined
  // stream, or the main stream without look-ahead - same plans either way), the
  // three full-size products that finish it (Gram, T, W) on the full device.
  auto split_panel = [&](cudaStream_t st, Scratch& sk, int64_t rows, MatView P, MatView Y, double* tau,
                         MatView T, MatView W) -> int {
    Scratch s1 = ws.pscratch_for(sk, rows);
    BR_CHECK(panel_qr(st, s1, ws.pscratch, P, Y, tau, T, &W, panel_cap(rows), &ws, nullptr, 1));
    cudaStream_t fs = (st == ws.gpanel) ? ws.panel : st;
    if (fs != st) {
      cudaEvent_t ev = ws_event(ws);
      BR_CUDA(cudaEventRecord(ev, st));
      BR_CUDA(cudaStreamWaitEvent(fs, ev, 0));
    }
    BR_CHECK(panel_qr(fs, sk, ws.pscratch, P, Y, tau, T, &W, panel_cap(rows), &ws, nullptr, 2));
    if (fs != st) {  // callers mark completion on `st`
      cudaEvent_t ev = ws_event(ws);
      BR_CUDA(cudaEventRecord(ev, fs));
      BR_CUDA(cudaStreamWaitEvent(st, ev, 0));
    }
    return 0;
  };
  auto qr = [&](cudaStream_t st, Scratch& sk, int64_t k, int64_t bp, int par) -> int {
    const int64_t i = m - k;
    MatView P(Aat(k, k), lda, i, bp);
    MatView Y(Yu[par], m, i, bp), T(Tu[par], b, bp, bp), W(Wu[par], m, i, bp);
    TimeScope ts(ws, st, TC_PANEL, panel_flops(i, bp), "qr", k);
    if (ws.split_upd && ws.confined(i)) {
      BR_CHECK(split_panel(st, sk, i, P, Y, tauu[par], T, W));
    } else {
      Scratch s = ws.pscratch_for(sk, i);
      BR_CHECK(panel_qr(st, s, ws.pscratch, P, Y, tauu[par], T, &W, panel_cap(i), &ws,
                        pz_rows() > 0 ? &mk_qr[par] : nullptr));
    }
    return store_factors(ws, st, 0, k, k, i, bp, Yu[par], m, Tu[par], b, tauu[par]);
  };
  auto lq = [&](cudaStream_t st, Scratch& sk, int64_t k, int64_t bq) -> int {
    const int64_t jr = n - k - w;
    MatView P(Aat(k, k + w), lda, jr, bq, true);  // transposed view of the bq x jr rows
    MatView Y(Yv, n, jr, bq), T(Tv, b, bq, bq), W(Wv, n, jr, bq);
    TimeScope ts(ws, st, TC_PANEL, panel_flops(jr, bq), "lq", k);
    if (ws.split_upd && ws.confined(jr)) {
      BR_CHECK(split_panel(st, sk, jr, P, Y, tauv, T, W));
    } else {
      Scratch s = ws.pscratch_for(sk, jr);
      BR_CHECK(panel_qr(st, s, ws.pscratch, P, Y, tauv, T, &W, panel_cap(jr), &ws,
                        pz_rows() > 0 ? &mk_lq : nullptr));
    }
    return store_factors(ws, st, 1, k, k + w, jr, bq, Yv, n, Tv, b, tauv);
  };
  auto handoff = [&](cudaStream_t ps) -> int {  // main -> panel ordering point
    cudaEvent_t ev = ws_event(ws);
    BR_CUDA(cudaEventRecord(ev, ws.main));
    BR_CUDA(cudaStreamWaitEvent(ps, ev, 0));
    return 0;
  };
  auto mark_panel = [&](cudaStream_t ps) -> cudaEvent_t {  // completion of the last panel launch
    cudaEvent_t ev = ws_event(ws);
    cudaEventRecord(ev, ps);
    return ev;
  };
  auto join = [&](cudaEvent_t ev) -> int {  // panel -> main
    BR_CUDA(cudaStreamWaitEvent(ws.main, ev, 0));
    return 0;
  };
  // the overlapped rest of an update on the SM-partitioned stream (Workspace::gupd)
  auto upd_begin = [&](cudaStream_t us) -> int {
    if (us == ws.main) return 0;
    cudaEvent_t ev = ws_event(ws);
    BR_CUDA(cudaEventRecord(ev, ws.main));
    BR_CUDA(cudaStreamWaitEvent(us, ev, 0));
    return 0;
  };
  auto upd_end = [&](cudaStream_t us) -> int {
    if (us == ws.main) return 0;
    cudaEvent_t ev = ws_event(ws);
    BR_CUDA(cudaEventRecord(ev, us));
    BR_CUDA(cudaStreamWaitEvent(ws.main, ev, 0));
    return 0;
  };

  BR_CHECK(band_in_wait(ws, bi, its[0].bp));  // the first panel's columns
  BR_CHECK(qr(ws.main, ws.sk_main, its[0].k, its[0].bp, 0));
  cudaEvent_t ev_qr = nullptr;
  for (size_t idx = 0; idx < its.size(); ++idx) {
    const int64_t k = its[idx].k, bp = its[idx].bp, i = m - k;
    const int par = (int)(idx & 1);
    // pipelined Z (short trailing matrices, where the panels are the critical
    // path): Z_L = T_U^T (Y_U^T E) and Z_R = (D Y_V) T_V, the Y products taken
    // leaf by leaf while the panel is still factoring its later leaves. The
    // choice depends on i only, so depth 0 and depth 1 stay bitwise equal.
    const bool pz = i <= pz_rows() && bp >= 64;  // multi-leaf panels only
    if (ev_qr && !pz) {
      BR_CHECK(join(ev_qr));
      ev_qr = nullptr;
    }
    const bool has_next = idx + 1 < its.size();
    const int64_t kn = has_next ? its[idx + 1].k : 0, bpn = has_next ? its[idx + 1].bp : 0;
    const bool la = lookahead && has_next;
    MatView Yuv(Yu[par], m, i, bp), Wuv(Wu[par], m, i, bp);
    const int64_t ncE = n - k - bp;
    const int64_t jr = n - k - w;
    const int64_t bq = jr >= 1 ? std::min(bp, jr) : 0;
    bool next_issued = false;

    auto next_qr_on_panel = [&]() -> int {
      cudaStream_t ps = ws.pstream(m - kn);
      BR_CHECK(handoff(ps));
      BR_CHECK(qr(ps, ws.sk_panel, kn, bpn, par ^ 1));
      ev_qr = mark_panel(ps);
      next_issued = true;
      return 0;
    };

    // streamed input: iteration 0's left update runs column chunk by column
    // chunk as the chunks arrive (every piece with its whole product's
    // split-K plan, so the result is bitwise that of the one-shot update)
    const bool chunked = bi && idx == 0 && ncE > 0 && bq > 0 && !pz;
    if (!chunked) BR_CHECK(band_in_wait(ws, bi, n));
    if (ncE > 0) {
      // left update E := Q_U^T E = E + Y_U (W_U^T E)  (ref svd.py:191)
      MatView E(Aat(k, k + bp), lda, i, ncE);
      MatView Z(ZL, b, bp, ncE);
      auto zleft = [&]() -> int {
        if (!pz) {
          TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(bp, ncE, i), "zleft", k);
          return gemm(ws.main, ws.sk_main, Z, Wuv.T(), E, 1.0, 0.0);
        }
        const LeafMarks& mk = mk_qr[par];
        MatView Zr(ZLr, b, bp, ncE);
        for (int s = 0; s < mk.n; ++s) {
          const int64_t c0 = mk.c0[s], wc = mk.c1[s] - c0;
          BR_CUDA(cudaStreamWaitEvent(ws.main, mk.ev[s], 0));
          TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(wc, ncE, i - c0), "zleft-leaf", k);
          BR_CHECK(gemm(ws.main, ws.sk_main, Zr.sub(c0, 0, wc, ncE), Yuv.sub(c0, c0, i - c0, wc).T(),
                        E.sub(c0, 0, i - c0, ncE), 1.0, 0.0));
        }
        if (ev_qr) {
          BR_CHECK(join(ev_qr));
          ev_qr = nullptr;
        }
        TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(bp, ncE, bp), "zleft", k);
        return gemm(ws.main, ws.sk_main, Z, MatView(Tu[par], b, bp, bp).T(), Zr, 1.0, 0.0);
      };
      if (bq > 0) {
        cudaEvent_t ev_lq = nullptr;
        auto issue_lq = [&]() -> int {  // LQ on the panel stream once its rows are updated
          if (!lookahead) return 0;
          // streamed input: the whole left update has been issued chunk by chunk
          // before this point, so this LQ overlaps nothing - it runs its (same)
          // two-phase plan on the whole device instead of the confined stream
          cudaStream_t ps = chunked ? ws.panel : ws.pstream(jr);
          BR_CHECK(handoff(ps));
          BR_CHECK(lq(ps, ws.sk_panel, k, bq));
          ev_lq = mark_panel(ps);
          return 0;
        };
        if (chunked) {
          const int64_t kz = gemm_plan_kps(ws.sk_main, Z, Wuv.T(), E, 0.0);
          const int64_t kr = gemm_plan_kps(ws.sk_main, E.sub(0, 0, bq, ncE), Yuv.sub(0, 0, bq, bp), Z, 1.0);
          const int64_t ks = gemm_plan_kps(ws.sk_main, E.sub(bq, 0, i - bq, ncE),
                                           Yuv.sub(bq, 0, i - bq, bp), Z, 1.0);
          for (int64_t a0 = k + bp; a0 < n;) {
            const int64_t a1 = std::min(n, (a0 / bi->chunk + 1) * bi->chunk);
            BR_CHECK(band_in_wait(ws, bi, a1));
            const int64_t e0 = a0 - k - bp, ne = a1 - a0;
            MatView Ec = E.sub(0, e0, i, ne), Zc = Z.sub(0, e0, bp, ne);
            TimeScope ts(ws, ws.main, TC_GEMM, 2 * gemm_flops(bp, ne, i), "left-chunk", k);
            BR_CHECK(gemm(ws.main, ws.sk_main, Zc, Wuv.T(), Ec, 1.0, 0.0, nullptr, 0, kz));
            BR_CHECK(gemm(ws.main, ws.sk_main, Ec.sub(0, 0, bq, ne), Yuv.sub(0, 0, bq, bp), Zc, 1.0,
                          1.0, nullptr, 0, kr));
            BR_CHECK(gemm(ws.main, ws.sk_main, Ec.sub(bq, 0, i - bq, ne), Yuv.sub(bq, 0, i - bq, bp),
                          Zc, 1.0, 1.0, nullptr, 0, ks));
            a0 = a1;
          }
          BR_CHECK(band_in_wait(ws, bi, n));
          BR_CHECK(issue_lq());
        } else {
          if (fuse_small() && !pz && bp <= 64 && bq <= 64) {
            // Z_L = W_U^T E and the LQ panel's rows E[0:bq] += Y_U[0:bq] Z_L in one reduction
            TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(bp, ncE, i) + gemm_flops(bq, ncE, bp),
                         "zleft+lq-rows", k);
            BR_CHECK(gemm_left_update(ws.main, ws.sk_main, Z, Wuv.T(), E, E.sub(0, 0, bq, ncE),
                                      Yuv.sub(0, 0, bq, bp)));
          } else {
            BR_CHECK(zleft());
            // rows of the LQ panel first
            TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(bq, ncE, bp), "left-lq-rows", k);
            BR_CHECK(gemm(ws.main, ws.sk_main, E.sub(0, 0, bq, ncE), Yuv.sub(0, 0, bq, bp), Z, 1.0,
                          1.0));
          }
          BR_CHECK(issue_lq());
          cudaStream_t us = ws.ustream(i, lookahead != 0);
          BR_CHECK(upd_begin(us));
          {
            TimeScope ts(ws, us, TC_GEMM, gemm_flops(i - bq, ncE, bp), "left", k);
            BR_CHECK(gemm(us, ws.sk_main, E.sub(bq, 0, i - bq, ncE), Yuv.sub(bq, 0, i - bq, bp), Z, 1.0,
                          1.0));
          }
          BR_CHECK(upd_end(us));
        }
        const int64_t splitc = has_next ? std::max<int64_t>(0, bp + bpn - w) : 0;
        if (la && splitc == 0) BR_CHECK(next_qr_on_panel());  // next panel is left-only
        if (!lookahead) BR_CHECK(lq(ws.main, ws.sk_main, k, bq));
        else if (!pz) BR_CHECK(join(ev_lq));
        // right update D := D Q_V = D + (D W_V) Y_V^T (ref svd.py:199)
        MatView D(Aat(k + bq, k + w), lda, i - bq, jr);
        MatView Yvv(Yv, n, jr, bq), Wvv(Wv, n, jr, bq);
        MatView Zr(ZR, m, i - bq, bq);
        if (pz && lookahead && i - bq <= 0) BR_CHECK(join(ev_lq));
        const int64_t sc_f = std::min(splitc, jr);
        const bool fuse_r = fuse_small() && !pz && bq <= 64 && has_next && !next_issued &&
                            splitc > 0 && sc_f <= 64 && i - bq > 0;
        if (fuse_r) {
          // Z_R = D W_V and the next QR panel's columns D[:, 0:sc] += Z_R Y_V[0:sc]^T
          // in one reduction, then (look-ahead) QR(k+1) and the rest of D
          {
            TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(i - bq, bq, jr) + gemm_flops(i - bq, sc_f, bq),
                         "zright+right-head", k);
            BR_CHECK(gemm_right_update(ws.main, ws.sk_main, Zr, D, Wvv, D.sub(0, 0, i - bq, sc_f),
                                       Yvv.sub(0, 0, sc_f, bq)));
          }
          if (la) BR_CHECK(next_qr_on_panel());
          if (sc_f < jr) {
            TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(i - bq, jr - sc_f, bq), "right", k);
            BR_CHECK(gemm(ws.main, ws.sk_main, D.sub(0, sc_f, i - bq, jr - sc_f), Zr,
                          Yvv.sub(sc_f, 0, jr - sc_f, bq).T(), 1.0, 1.0));
          }
        } else if (i - bq > 0) {
          if (pz) {
            MatView Zrr(ZRr, m, i - bq, bq);
            for (int s = 0; s < mk_lq.n; ++s) {
              const int64_t c0 = mk_lq.c0[s], wc = mk_lq.c1[s] - c0;
              BR_CUDA(cudaStreamWaitEvent(ws.main, mk_lq.ev[s], 0));
              TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(i - bq, wc, jr - c0), "zright-leaf", k);
              BR_CHECK(gemm(ws.main, ws.sk_main, Zrr.sub(0, c0, i - bq, wc), D.sub(0, c0, i - bq, jr - c0),
                            Yvv.sub(c0, c0, jr - c0, wc), 1.0, 0.0));
            }
            if (lookahead) BR_CHECK(join(ev_lq));
            TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(i - bq, bq, bq), "zright", k);
            BR_CHECK(gemm(ws.main, ws.sk_main, Zr, Zrr, MatView(Tv, b, bq, bq), 1.0, 0.0));
          } else {
            TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(i - bq, bq, jr), "zright", k);
            BR_CHECK(gemm(ws.main, ws.sk_main, Zr, D, Wvv, 1.0, 0.0));
          }
          if (la && !next_issued && splitc > 0) {
            const int64_t sc = std::min(splitc, jr);
            const int64_t kps = gemm_plan_kps(ws.sk_main, D, Zr, Yvv.T(), 1.0);
            {
              TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(i - bq, sc, bq), "right-head", k);
              BR_CHECK(gemm(ws.main, ws.sk_main, D.sub(0, 0, i - bq, sc), Zr,
                            Yvv.sub(0, 0, sc, bq).T(), 1.0, 1.0, nullptr, 0, kps));
            }
            BR_CHECK(next_qr_on_panel());
            if (sc < jr) {
              cudaStream_t us = ws.ustream(i, true);
              BR_CHECK(upd_begin(us));
              {
                TimeScope ts(ws, us, TC_GEMM, gemm_flops(i - bq, jr - sc, bq), "right", k);
                BR_CHECK(gemm(us, ws.sk_main, D.sub(0, sc, i - bq, jr - sc), Zr,
                              Yvv.sub(sc, 0, jr - sc, bq).T(), 1.0, 1.0, nullptr, 0, kps));
              }
              BR_CHECK(upd_end(us));
            }
          } else {
            TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(i - bq, jr, bq), "right", k);
            BR_CHECK(gemm(ws.main, ws.sk_main, D, Zr, Yvv.T(), 1.0, 1.0));
          }
        }
      } else {
        BR_CHECK(zleft());
        TimeScope ts(ws, ws.main, TC_GEMM, gemm_flops(i, ncE, bp), "left", k);
        BR_CHECK(gemm(ws.main, ws.sk_main, E, Yuv, Z, 1.0, 1.0));
      }
    }
    if (has_next && !next_issued) {
      if (la) BR_CHECK(next_qr_on_panel());
      else BR_CHECK(qr(ws.main, ws.sk_main, kn, bpn, par ^ 1));
    }
    BR_CHECK(band_out_flush(ws, bo, k + bp));  // columns [0, k + bp) are final
  }
  if (ev_qr) BR_CHECK(join(ev_qr));
  BR_CHECK(band_in_wait(ws, bi, n));
  if (partial) {
    BR_CHECK(band_out_raw(ws, bo_full, n));
    ws_events_reset(ws);
    return 0;
  }
  if (bo) {
    BR_CHECK(band_out_flush(ws, bo, n));
    ws_events_reset(ws);
    return 0;
  }
  ws_events_reset(ws);
  return mask_tri(ws.main, A, lda, m, n, 0, w);
}

// ---------------------------------------------------------------------------
// Equal-bandwidth band form of the SVD (ref svd.py:250-589), m >= n
// ---------------------------------------------------------------------------
// Iteration k (bp = min(b, m-k-w, n-k), jr = n-k-w, bq = min(bp, jr)):
//   QR of A[k+w:m, k:k+bp]      -> Q_U = I + W_U Y_U^T (ref svd.py:275-283)
//   LQ of A[k:k+bq, k+w:n]      -> Q_V = I + W_V Y_V^T (ref svd.py:295-306)
//   left:  ML = A[k+w:m, k+bp:n] = [B1 | D] += Y_U (W_U^T ML)
//   right: MR = A[k+bq:m, k+w:n] = [C1 ; D] += (MR W_V) Y_V^T
// The LQ rows lie above the rows the left update touches, so both panels of
// an iteration are factored together. fused == 0 applies left then right
// (Reference / V1 order, ref svd.py:359-376); fused == 1 updates D once from
// its old value (Simultaneous / V2, ref svd.py:377-391):
//   Z_L = W_U^T D, Z_R = D W_V, X = Z_R + Y_U (Z_L W_V),
//   D += X Y_V^T, then D += Y_U Z_L.
// Look-ahead (ref svd.py:394-492): the parts of this iteration's update that
// the next QR columns / LQ rows read are issued first, both next panels are
// factored on the panel stream, and main finishes the rest. Every piece uses
// the split-K chunk planned for its whole product, so depth 1 is bitwise
// equal to depth 0.
int band_reduce(Workspace& ws, int64_t m, int64_t n, int64_t w, int64_t b, int fused,
                int lookahead, double* A, int64_t lda, int64_t* iterations, BandOut* bo) {
  NoSplit nosplit(ws);
  struct It {
    int64_t k, bp, jr, bq;
  };
  std::vector<It> its;
  for (int64_t k = 0; m - k - w >= 2 && k < n;) {
    const int64_t bp = std::min({b, m - k - w, n - k});
    const int64_t jr = n - k - w;
    its.push_back({k, bp, jr, jr >= 1 ? std::min(bp, jr) : 0});
    k += bp;
  }
  const bool partial = ws.max_iters > 0 && ws.max_iters < (int64_t)its.size();
  if (partial) its.resize((size_t)ws.max_iters);
  BandOut* const bo_full = bo;
  if (partial) bo = nullptr;
  *iterations = (int64_t)its.size();
  if (its.empty()) {  // m <= w + 1: returned unchanged (ref svd.py:561-564)
    if (bo) {
      BR_CUDA(cudaMemcpy2DAsync(bo->host, bo->ldh * sizeof(double), A, lda * sizeof(double),
                                m * sizeof(double), n, cudaMemcpyDeviceToHost, ws.main));
      bo->done = n;
    }
    return 0;
  }

  const int64_t nYu = m * b, nYv = n * b, nT = b * b;
  const int64_t total = 4 * nYu + 4 * nYv + 4 * nT + 4 * b + b * n + 2 * m * b + nT;
  BR_CHECK(devbuf_reserve(ws.factors, total));
  BR_CHECK(devbuf_reserve(ws.skbuf_main, 4 * std::max(m, n) * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.skbuf_panel, 4 * std::max(m, n) * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.skbuf_aux, 4 * std::max(m, n) * b + (1 << 20)));
  BR_CHECK(devbuf_reserve(ws.pscratch, panel_scratch_doubles(b)));
  ws.sk_main = Scratch{ws.skbuf_main.p, ws.skbuf_main.cap, ws.num_sms};
  ws.sk_panel = Scratch{ws.skbuf_panel.p, ws.skbuf_panel.cap, ws.num_sms};
  ws.sk_aux = Scratch{ws.skbuf_aux.p, ws.skbuf_aux.cap, ws.num_sms};
  double* f = ws.factors.p;
  double *Yu[2], *Wu[2], *Tu[2], *tauu[2], *Yv[2], *Wv[2], *Tv[2], *tauv[2];
  for (int p = 0; p < 2; ++p) {
    Yu[p] = f; f += nYu;
    Wu[p] = f; f += nYu;
    Yv[p] = f; f += nYv;
    Wv[p] = f; f += nYv;
    Tu[p] = f; f += nT;
    Tv[p] = f; f += nT;
    tauu[p] = f; f += b;
    tauv[p] = f; f += b;
  }
  double* ZLb = f; f += b * n;  // W_U^T ML  (bp x (n-k-bp), ld b)
  double* ZRb = f; f += m * b;  // MR W_V    ((m-k-bq) x bq, ld m)
  double* Xb = f; f += m * b;   // X         (i x bq, ld m)
  double* Tmb = f; f += nT;     // Z_L W_V   (bp x bq, ld b)

  auto Aat = [&](int64_t r, int64_t c) { return A + r + c * lda; };
  auto qr = [&](cudaStream_t st, Scratch& sk, const It& t, int par) -> int {
    const int64_t i = m - t.k - w;
    MatView P(Aat(t.k + w, t.k), lda, i, t.bp);
    MatView Y(Yu[par], m, i, t.bp), T(Tu[par], b, t.bp, t.bp), W(Wu[par], m, i, t.bp);
    TimeScope ts(ws, st, TC_PANEL, panel_flops(i, t.bp), "qr", t.k);
    Scratch s = ws.pscratch_for(sk, i);
    BR_CHECK(panel_qr(st, s, ws.pscratch, P, Y, tauu[par], T, &W, panel_cap(i), &ws));
    return store_factors(ws, st, 0, t.k, t.k + w, i, t.bp, Yu[par], m, Tu[par], b, tauu[par]);
  };
  auto lq = [&](cudaStream_t st, Scratch& sk, const It& t, int par) -> int {
    MatView P(Aat(t.k, t.k + w), lda, t.jr, t.bq, true);  // transposed view of the bq x jr rows
    MatView Y(Yv[par], n, t.jr, t.bq), T(Tv[par], b, t.bq, t.bq), W(Wv[par], n, t.jr, t.bq);
    TimeScope ts(ws, st, TC_PANEL, panel_flops(t.jr, t.bq), "lq", t.k);
    Scratch s = ws.pscratch_for(sk, t.jr);
    BR_CHECK(panel_qr(st, s, ws.pscratch, P, Y, tauv[par], T, &W, panel_cap(t.jr), &ws));
    return store_factors(ws, st, 1, t.k, t.k + w, t.jr, t.bq, Yv[par], n, Tv[par], b, tauv[par]);
  };
  auto panels = [&](cudaStream_t st, Scratch& sk, const It& t, int par) -> int {
    BR_CHECK(qr(st, sk, t, par));
    return t.jr >= 1 ? lq(st, sk, t, par) : 0;
  };

  cudaEvent_t ev_panels = nullptr;
  BR_CHECK(panels(ws.main, ws.sk_main, its[0], 0));
  for (size_t idx = 0; idx < its.size(); ++idx) {
    const It t = its[idx];
    const int par = (int)(idx & 1);
    if (ev_panels) {
      BR_CUDA(cudaStreamWaitEvent(ws.main, ev_panels, 0));
      ev_panels = nullptr;
    }
    const bool has_next = idx + 1 < its.size();
    const It tn = has_next ? its[idx + 1] : It{0, 0, 0, 0};
    const bool la = lookahead && has_next;
    cudaStream_t st = ws.main;
    Scratch& sk = ws.sk_main;
    const int64_t i = m - t.k - w;           // rows of D (and of ML)
    const int64_t ncL = n - t.k - t.bp;      // columns of ML = [B1 | D]
    const int64_t b1w = std::min(w - t.bp, ncL);  // columns of B1
    const int64_t jr = std::max<int64_t>(t.jr, 0), bq = t.bq;
    const int64_t c1r = w - bq;              // rows of C1
    const int64_t nrR = c1r + i;             // rows of MR = [C1 ; D]

    MatView ML(Aat(t.k + w, t.k + t.bp), lda, i, ncL);
    MatView MR(Aat(t.k + bq, t.k + w), lda, nrR, jr);
    MatView Yuv(Yu[par], m, i, t.bp), Wuv(Wu[par], m, i, t.bp);
    MatView Yvv(Yv[par], n, jr, bq), Wvv(Wv[par], n, jr, bq);
    MatView ZL(ZLb, b, t.bp, ncL), ZR(ZRb, m, nrR, bq), X(Xb, m, i, bq), Tm(Tmb, b, t.bp, bq);

    // whole-product split-K plans
    const int64_t kz_l = gemm_plan_kps(sk, ZL, Wuv.T(), ML, 0.0);
    const int64_t ku_l = gemm_plan_kps(sk, ML, Yuv, ZL, 1.0);
    const int64_t kz_r = jr ? gemm_plan_kps(sk, ZR, MR, Wvv, 0.0) : 0;
    const int64_t ku_r = jr ? gemm_plan_kps(sk, MR, ZR, Yvv.T(), 1.0) : 0;
    const int64_t ku_x = jr ? gemm_plan_kps(sk, MR.sub(c1r, 0, i, jr), X, Yvv.T(), 1.0) : 0;

    // ZL[:, c0:c1] = W_U^T ML[:, c0:c1]
    auto zl = [&](int64_t c0, int64_t c1) -> int {
      if (c0 >= c1) return 0;
      TimeScope ts(ws, st, TC_GEMM, gemm_flops(t.bp, c1 - c0, i), "zleft", t.k);
      return gemm(st, sk, ZL.sub(0, c0, t.bp, c1 - c0), Wuv.T(), ML.sub(0, c0, i, c1 - c0), 1.0,
                  0.0, nullptr, 0, kz_l);
    };
    // ML[r0:r1, c0:c1] += Y_U[r0:r1] ZL[:, c0:c1]
    auto ul = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) -> int {
      if (c0 >= c1 || r0 >= r1) return 0;
      TimeScope ts(ws, st, TC_GEMM, gemm_flops(r1 - r0, c1 - c0, t.bp), "left", t.k);
      return gemm(st, sk, ML.sub(r0, c0, r1 - r0, c1 - c0), Yuv.sub(r0, 0, r1 - r0, t.bp),
                  ZL.sub(0, c0, t.bp, c1 - c0), 1.0, 1.0, nullptr, 0, ku_l);
    };
    // ZR[r0:r1] = MR[r0:r1] W_V
    auto zr = [&](int64_t r0, int64_t r1) -> int {
      if (r0 >= r1 || !jr) return 0;
      TimeScope ts(ws, st, TC_GEMM, gemm_flops(r1 - r0, bq, jr), "zright", t.k);
      return gemm(st, sk, ZR.sub(r0, 0, r1 - r0, bq), MR.sub(r0, 0, r1 - r0, jr), Wvv, 1.0, 0.0,
                  nullptr, 0, kz_r);
    };
    // MR[r0:r1, c0:c1] += ZR[r0:r1] Y_V[c0:c1]^T
    auto ur = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) -> int {
      if (r0 >= r1 || c0 >= c1) return 0;
      TimeScope ts(ws, st, TC_GEMM, gemm_flops(r1 - r0, c1 - c0, bq), "right", t.k);
      return gemm(st, sk, MR.sub(r0, c0, r1 - r0, c1 - c0), ZR.sub(r0, 0, r1 - r0, bq),
                  Yvv.sub(c0, 0, c1 - c0, bq).T(), 1.0, 1.0, nullptr, 0, ku_r);
    };
    // Simultaneous D block [r0:r1, c0:c1] (D coordinates): += X Y_V^T, += Y_U Z_L
    auto dsim = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) -> int {
      if (r0 >= r1 || c0 >= c1) return 0;
      {
        TimeScope ts(ws, st, TC_GEMM, gemm_flops(r1 - r0, c1 - c0, bq), "dsub", t.k);
        BR_CHECK(gemm(st, sk, MR.sub(c1r + r0, c0, r1 - r0, c1 - c0), X.sub(r0, 0, r1 - r0, bq),
                      Yvv.sub(c0, 0, c1 - c0, bq).T(), 1.0, 1.0, nullptr, 0, ku_x));
      }
      return ul(r0, r1, b1w + c0, b1w + c1);
    };
    auto issue_next = [&]() -> int {  // both next panels on the panel stream
      cudaStream_t ps = ws.pstream(m - tn.k - w);
      cudaEvent_t ev = ws_event(ws);
      BR_CUDA(cudaEventRecord(ev, ws.main));
      BR_CUDA(cudaStreamWaitEvent(ps, ev, 0));
      BR_CHECK(panels(ps, ws.sk_panel, tn, par ^ 1));
      ev_panels = ws_event(ws);
      BR_CUDA(cudaEventRecord(ev_panels, ps));
      // the updates issued after this point overlap the panels: below the
      // threshold they go to the SM-partitioned stream (Workspace::gupd)
      cudaStream_t us = ws.ustream(i, true);
      if (us != ws.main) {
        cudaEvent_t e2 = ws_event(ws);
        BR_CUDA(cudaEventRecord(e2, ws.main));
        BR_CUDA(cudaStreamWaitEvent(us, e2, 0));
        st = us;
      }
      return 0;
    };

    // footprints of the next panels: QR columns ML[:, 0:bpn), LQ rows
    // MR[bp-bq : bp-bq+bqn) (ref svd.py:394-420)
    const int64_t bpn = tn.bp, bqn = tn.jr >= 1 ? tn.bq : 0;
    const int64_t hc = la ? std::min(bpn, ncL) : 0;                        // ML head columns
    const int64_t hr = la ? std::min(t.bp - bq + bqn, nrR) : 0;            // MR head rows
    const int64_t sc = la ? std::max<int64_t>(0, std::min(bpn - b1w, jr)) : 0;  // D cols of next QR
    const int64_t sr = la ? std::max<int64_t>(0, std::min(hr - c1r, i)) : 0;    // D rows of next LQ
    bool issued = false;

    BR_CHECK(zl(0, ncL));
    if (!fused || !jr) {
      if (jr && sc == 0 && sr == 0 && la) {
        // V1 regime: next QR inside B1, next LQ inside C1
        BR_CHECK(ul(0, i, 0, hc));
        BR_CHECK(zr(0, hr));
        BR_CHECK(ur(0, hr, 0, jr));
        BR_CHECK(issue_next());
        issued = true;
        BR_CHECK(ul(0, i, hc, ncL));
        BR_CHECK(zr(hr, nrR));
        BR_CHECK(ur(hr, nrR, 0, jr));
      } else if (!jr && la) {
        BR_CHECK(ul(0, i, 0, hc));
        BR_CHECK(issue_next());
        issued = true;
        BR_CHECK(ul(0, i, hc, ncL));
      } else {
        BR_CHECK(ul(0, i, 0, ncL));
        BR_CHECK(zr(0, nrR));
        if (la) {  // V2 regime: heads (LQ rows, then QR columns of D) first
          BR_CHECK(ur(0, hr, 0, jr));
          BR_CHECK(ur(hr, nrR, 0, c1r < hr ? sc : std::min(sc, jr)));
          BR_CHECK(issue_next());
          issued = true;
          BR_CHECK(ur(hr, nrR, sc, jr));
        } else {
          BR_CHECK(ur(0, nrR, 0, jr));
        }
      }
    } else {
      // Simultaneous: ZL, ZR from the old D; X = ZR_D + Y_U (ZL_D W_V)
      BR_CHECK(zr(0, nrR));
      {
        TimeScope ts(ws, st, TC_GEMM, gemm_flops(t.bp, bq, jr) + gemm_flops(i, bq, t.bp), "xprod", t.k);
        BR_CHECK(gemm(st, sk, Tm, ZL.sub(0, b1w, t.bp, jr), Wvv, 1.0, 0.0));
        MatView ZRD = ZR.sub(c1r, 0, i, bq);
        BR_CHECK(gemm(st, sk, X, Yuv, Tm, 1.0, 1.0, &ZRD));
      }
      if (la) {
        const int64_t hb = std::min(hc, b1w), hcr = std::min(hr, c1r);
        BR_CHECK(ul(0, i, 0, hb));           // B1 head
        BR_CHECK(ur(0, hcr, 0, jr));         // C1 head
        BR_CHECK(dsim(0, sr, 0, sc));        // D11
        BR_CHECK(dsim(sr, i, 0, sc));        // D21
        BR_CHECK(dsim(0, sr, sc, jr));       // D12
        BR_CHECK(issue_next());
        issued = true;
        BR_CHECK(ul(0, i, hb, b1w));         // B1 rest
        BR_CHECK(ur(hcr, c1r, 0, jr));       // C1 rest
        BR_CHECK(dsim(sr, i, sc, jr));       // D22
      } else {
        BR_CHECK(ul(0, i, 0, b1w));
        BR_CHECK(ur(0, c1r, 0, jr));
        BR_CHECK(dsim(0, i, 0, jr));
      }
    }
    if (st != ws.main) {  // join the partitioned update stream
      cudaEvent_t e2 = ws_event(ws);
      BR_CUDA(cudaEventRecord(e2, st));
      BR_CUDA(cudaStreamWaitEvent(ws.main, e2, 0));
      st = ws.main;
    }
    if (has_next && !issued) BR_CHECK(panels(ws.main, ws.sk_main, tn, par ^ 1));
    BR_CHECK(band_out_flush(ws, bo, std::min(n, t.k + t.bp)));  // columns [0, k + bp) are final
  }
  if (ev_panels) BR_CUDA(cudaStreamWaitEvent(ws.main, ev_panels, 0));
  if (partial) {
    BR_CHECK(band_out_raw(ws, bo_full, n));
    ws_events_reset(ws);
    return 0;
  }
  if (bo) {
    BR_CHECK(band_out_flush(ws, bo, n));
    ws_events_reset(ws);
    return 0;
  }
  ws_events_reset(ws);
  return mask_tri(ws.main, A, lda, m, n, w, w);
}

}  // namespace br
