// Host-side handle, workspace and driver entry points (internal header).
#pragma once
#include <vector>

#include "../../include/bandred_b200.h"
#include "common.cuh"
#include "gemm.cuh"

namespace br {

// Growable device buffer (cudaMalloc'd; grows only between synchronized calls).
struct DevBuf {
  double* p = nullptr;
  int64_t cap = 0;  // doubles
};
int devbuf_reserve(DevBuf& b, int64_t n);
int64_t alloc_generation();  // bumped whenever a DevBuf is (re)allocated
void devbuf_free(DevBuf& b);

enum TimeClass { TC_PANEL = 0, TC_SYMM = 1, TC_SYR2K = 2, TC_GEMM = 3, TC_COUNT = 4 };

// Per-device execution context: the two streams of the look-ahead (main =
// trailing update, panel = next panel's factorization; the T_P / T_S groups
// of the reference runtime, ref runtime.py:142-180), events, and reusable
// device workspace.
struct Workspace {
  int device = 0;
  int num_sms = 148;
  // SM-partitioned panel stream (green context, BR_GREEN_SMS): panels taller
  // than green_rows run on gpanel, confined to green_sms SMs, so they take
  // SMs only from that partition while the trailing update (whole device)
  // runs; shorter panels (the critical path near the end) use `panel`.
  cudaStream_t gpanel = nullptr;
  int green_sms = 0;
  int64_t green_rows = 8192;
  bool confined(int64_t rows) const { return gpanel != nullptr && rows > green_rows; }
  cudaStream_t pstream(int64_t rows) const { return confined(rows) ? gpanel : panel; }
  // split-K plan of a panel's GEMMs: depends on the panel height only, so the
  // schedules with and without look-ahead plan (and round) identically
  Scratch pscratch_for(const Scratch& s, int64_t rows) const {
    Scratch r = s;
    if (confined(rows)) r.num_sms = green_sms;
    return r;
  }
  // SM-partitioned update stream (green context over all but BR_UPD_SMS SMs):
  // where the panel chain bounds an iteration (trailing rows <= upd_rows) the
  // overlapped rest of the trailing update runs there, so the SMs left out
  // never hold a long-running update CTA and the high-priority panel kernels
  // (16-CTA leaf clusters, small GEMMs) start on them at once instead of
  // waiting for update tiles to drain. Results do not depend on the stream.
  cudaStream_t gupd = nullptr;
  void *gctx_upd = nullptr, *gctx_panel = nullptr;  // the partition's green contexts (br_destroy)
  int upd_sms = 0;
  int64_t upd_rows = 0;
  cudaStream_t ustream(int64_t rows, bool overlap) const {
    return (gupd && overlap && !no_partition && (rows <= upd_rows || (split_upd && confined(rows)))) ? gupd
                                                                                                   : main;
  }
  bool split_upd = false;  // BR_SPLIT_ROWS: confined panels, their update on the other SMs
  bool no_partition = false;  // set while a graphable (small) reduction runs or is captured
  cudaStream_t main = nullptr, panel = nullptr;
  cudaStream_t own_main = nullptr, own_panel = nullptr;
  Scratch sk_main, sk_panel;  // split-K partials, one per stream
  DevBuf skbuf_main, skbuf_panel;
  DevBuf pscratch;  // panel_qr internal scratch (reductions; kernel-level calls on main)
  DevBuf pscratch_panel;  // panel_qr scratch of kernel-level calls on the panel stream
  DevBuf factors;   // reduction buffers
  DevBuf s2prog;    // second stage: per-sweep progress counters
  DevBuf tmp, tmp_panel;  // kernel-level API temporaries, one per stream
  DevBuf stageA, stageQ;  // host-buffer entry points
  DevBuf stageF;          // host-buffer entry points: device copy of the factor output
  // auxiliary stream of the persistent panel: the block updates between
  // leaves run there while the leaf cluster stays resident
  cudaStream_t aux = nullptr;
  Scratch sk_aux;
  DevBuf skbuf_aux;
  unsigned* flags = nullptr;  // 128 leaf handshake words
  unsigned epoch = 0;
  cudaEvent_t ev_aux0 = nullptr, ev_aux1 = nullptr;
  // CUDA graph of the last reduction's stream program, replayed when the
  // same reduction (sizes, pointers, streams, workspace generation) repeats
  struct GraphKey {
    int kind = -1, fused = 0, la = 0, timing = 0;
    int64_t m = 0, n = 0, w = 0, b = 0, lda = 0, ldq = 0, gen = -1, max_iters = 0;
    const void* A = nullptr;
    const void* Q = nullptr;
    br_factors fo{};  // factor output pointers (all NULL when none)
    cudaStream_t main = nullptr, panel = nullptr;
    bool operator==(const GraphKey& o) const {
      return kind == o.kind && fused == o.fused && la == o.la && timing == o.timing && m == o.m &&
             n == o.n && w == o.w && b == o.b && lda == o.lda && ldq == o.ldq && gen == o.gen &&
             max_iters == o.max_iters && A == o.A && Q == o.Q && main == o.main &&
             panel == o.panel && fo.yl == o.fo.yl && fo.ldyl == o.fo.ldyl && fo.tl == o.fo.tl &&
             fo.ldtl == o.fo.ldtl && fo.taul == o.fo.taul && fo.yr == o.fo.yr &&
             fo.ldyr == o.fo.ldyr && fo.tr == o.fo.tr && fo.ldtr == o.fo.ldtr &&
             fo.taur == o.fo.taur;
    }
  };
  GraphKey gkey;
  struct BandOut* band_out = nullptr;  // set by the host entry points while streaming out
  cudaStream_t copy = nullptr;         // D2H stream of the streamed band
  struct BandIn* band_in = nullptr;    // set by the host entry points while streaming in
  cudaStream_t copy_in = nullptr;      // H2D stream of the streamed input
  int gseen = 0;  // eager runs of gkey so far
  cudaGraphExec_t gexec = nullptr;
  int64_t g_iters = 0, g_launches = 0;
  // events
  std::vector<cudaEvent_t> events;
  size_t event_next = 0;
  // optional per-class timing (timing >= 1) and per-task event trace (2)
  int timing = 0;
  struct Timed {
    int cls;
    cudaEvent_t a, b;
    double flops;
    const char* tag;  // task name ("qr", "left", ...) or nullptr
    int64_t k;        // iteration's leading column
    int stream;       // 0 main (T_P role), 1 panel (T_S role)
  };
  struct TraceRec {
    char id[40];
    int stream;
    double t0_us, t1_us;
  };
  std::vector<TraceRec> trace;
  cudaEvent_t trace_base = nullptr;  // start of the current reduction call
  std::vector<Timed> timed;
  std::vector<cudaEvent_t> tevents;
  size_t tevent_next = 0;
  double t_ms[TC_COUNT] = {0, 0, 0, 0};
  double t_flops[TC_COUNT] = {0, 0, 0, 0};
  int64_t t_launches[TC_COUNT] = {0, 0, 0, 0};
  int64_t launches = 0;
  int active = 0;  // stream used by kernel-level C-ABI calls: 0 main, 1 panel
  // factor output of the reduction in progress (device pointers; nullable)
  const br_factors* fo = nullptr;
  int64_t max_iters = 0;  // BR_OPT_MAX_ITERS: partial reduction (0 = full)
};

// Store one panel's factors into the reduction's factor output (on the
// panel's stream, right after it was factored). chain 0 = left (QR), 1 =
// right (LQ); r0 = first row of Y_k in the packed layout (br_factors).
int store_factors(Workspace& ws, cudaStream_t st, int chain, int64_t k, int64_t r0, int64_t j,
                  int64_t bp, const double* Y, int64_t ldy, const double* T, int64_t ldt,
                  const double* tau);
// Copy the raw working matrix of a partial reduction (BR_OPT_MAX_ITERS) to a
// streamed host destination.
int band_out_raw(Workspace& ws, BandOut* bo, int64_t cols);

// Kernels launched by this library in this process (stats / bench evidence).
int64_t launch_count();
void count_launch(int64_t n = 1);
void g_launches_adjust(int64_t d);

cudaEvent_t ws_event(Workspace& ws);  // recycled sync-only event
void ws_events_reset(Workspace& ws);
// Timing scope: records CUDA events around the enclosed launches on `st`
// (only when ws.timing), attributing `flops` algorithmic flops to `cls`.
// With ws.timing == 2 the scope is also a trace record "tag@k" on its stream.
struct TimeScope {
  Workspace& ws;
  cudaStream_t st;
  int cls;
  double flops;
  const char* tag;
  int64_t k;
  cudaEvent_t a = nullptr;
  TimeScope(Workspace& w, cudaStream_t s, int c, double f, const char* tag = nullptr,
            int64_t k = -1);
  ~TimeScope();
};
int ws_collect_timing(Workspace& ws);  // after a sync: fold events into t_ms

// Panel factorization (panel.cu). P is the j x b panel view (a transposed
// view gives the LQ of the underlying b x j rows). Outputs: Y (j x b, unit
// lower trapezoidal with explicit zeros/ones), tau (b), T (b x b, T =
// -T_larft), W = Y*T (j x b, optional). R (or L) is written into P's top
// b x b triangle; the strictly-lower part of P is left unspecified (the
// reductions zero it in their final band mask).
// Completion points of a panel's leaves: Y columns [c0[s], c1[s]) are final
// once ev[s] (recorded on the panel's stream) has completed.
struct LeafMarks {
  static constexpr int kMax = 256;
  int n = 0;
  int64_t c0[kMax], c1[kMax];
  cudaEvent_t ev[kMax];
};
int panel_qr(cudaStream_t st, Scratch& sk, DevBuf& pscratch, MatView P, MatView Y, double* tau,
             MatView T, MatView* W, int max_ctas = 0, Workspace* pws = nullptr,
             LeafMarks* marks = nullptr, int phase = 0);
int64_t panel_scratch_doubles(int64_t b);
bool panel_clusters_fit(cudaStream_t st);  // every tall-panel leaf cluster can be placed on st's SMs
int t_from_gram(cudaStream_t st, const double* G, int64_t ldg, const double* tau, int64_t b,
                double* T, int64_t ldt, bool diag_given = false);
int house_gen_dev(cudaStream_t st, int64_t L, const double* x, double* v, double* tau_beta);

// Force-load every kernel of the library (gemm.cu, panel.cu, driver.cu).
int preload_gemm_kernels();
int preload_xchain_kernels();
int preload_stage2_kernels();
// Second stage (stage2.cu): band (bandwidth w) -> tridiagonal (bd = false,
// symmetric band in the lower triangle) or upper bidiagonal (bd = true,
// upper triangular band, n x n) by bulge chasing, in place on A; d (n) and
// e (n - 1) receive the diagonals. prog: n ints of scratch.
int band_to_condensed(cudaStream_t st, bool bd, int64_t n, int64_t w, double* A, int64_t lda,
                      double* d, double* e, int* prog, int num_sms);
int preload_panel_kernels();

// Elementwise helpers (driver.cu)
int finalize_sym(cudaStream_t st, double* A, int64_t lda, int64_t n, int64_t w, int64_t c0 = 0,
                 int64_t c1 = -1);
int mask_tri(cudaStream_t st, double* A, int64_t lda, int64_t m, int64_t n, int64_t lower_bw,
             int64_t upper_bw, int64_t c0 = 0, int64_t c1 = -1);

// Host entry points with a pinned destination: finished column blocks are
// finalized and copied out on a copy stream while the reduction continues
// (after iteration k, columns [0, k + bp) are final in all three reductions).
struct BandOut {
  cudaStream_t st = nullptr;
  double* host = nullptr;
  int64_t ldh = 0;
  double* A = nullptr;
  int64_t lda = 0, rows = 0;
  bool sym = false;  // SEVP finalize (mirror + zero) instead of the band mask
  int64_t w = 0, lo = 0, up = 0;
  int64_t done = 0;  // columns already queued
};
int band_out_flush(Workspace& ws, BandOut* bo, int64_t upto);
// Input streamed in by column chunks (pinned host source): the reduction
// starts on the first chunks while the rest are still in flight.
struct BandIn {
  const double* host = nullptr;
  int64_t ldh = 0;
  double* A = nullptr;
  int64_t lda = 0, rows = 0, cols = 0;
  int64_t chunk = 0;   // columns per chunk
  int nchunks = 0;
  int waited = 0;      // chunks the main stream already waits for
  cudaEvent_t ev[256];
};
int band_in_start(Workspace& ws, BandIn* bi);
// Main stream waits until columns [0, upto) have arrived.
int band_in_wait(Workspace& ws, BandIn* bi, int64_t upto);
int zero_fill(cudaStream_t st, MatView V);
int set_identity(cudaStream_t st, double* Q, int64_t ldq, int64_t n);

// Reductions (reduce.cu)
int sevp_reduce(Workspace& ws, int64_t n, int64_t w, int64_t b, int lookahead, double* A,
                int64_t lda, double* Q, int64_t ldq, int64_t* iterations, BandOut* bo = nullptr);
int tri_reduce(Workspace& ws, int64_t m, int64_t n, int64_t w, int64_t b, int lookahead,
               double* A, int64_t lda, int64_t* iterations, BandOut* bo = nullptr);
int band_reduce(Workspace& ws, int64_t m, int64_t n, int64_t w, int64_t b, int fused,
                int lookahead, double* A, int64_t lda, int64_t* iterations,
                BandOut* bo = nullptr);

}  // namespace br
