// Context, workspace, elementwise kernels and the C ABI (include/bandred_b200.h).
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <new>

#include <cuda.h>

#include "../../include/bandred_b200.h"
#include "driver.cuh"
#include "gemm.cuh"

namespace br {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};
int64_t launch_count() { return g_launches.load(); }
void count_launch(int64_t n) { g_launches += n; }
void g_launches_adjust(int64_t d) { g_launches += d; }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<int64_t> g_alloc_gen{0};
int64_t alloc_generation() { return g_alloc_gen.load(); }

int devbuf_reserve(DevBuf& b, int64_t n) {
  if (n <= b.cap) return 0;
  ++g_alloc_gen;
  if (b.p) {
    BR_CUDA(cudaDeviceSynchronize());
    BR_CUDA(cudaFree(b.p));
    b.p = nullptr;
    b.cap = 0;
  }
  BR_CUDA(cudaMalloc(&b.p, (size_t)n * sizeof(double)));
  b.cap = n;
  return 0;
}
void devbuf_free(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

thread_local bool g_preload_only = false;

int stream_priority(cudaStream_t st) {
  thread_local cudaStream_t last = nullptr;
  thread_local int prio = 0;
  if (st != last || st == nullptr) {
    int p = 0;
    if (cudaStreamGetPriority(st, &p) != cudaSuccess) {
      cudaGetLastError();
      p = 0;
    }
    last = st;
    prio = p;
  }
  return prio;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BR_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaEvent_t ws_event(Workspace& ws) {
  if (ws.event_next == ws.events.size()) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    ws.events.push_back(e);
  }
  return ws.events[ws.event_next++];
}
void ws_events_reset(Workspace& ws) { ws.event_next = 0; }

static cudaEvent_t ws_tevent(Workspace& ws) {
  if (ws.tevent_next == ws.tevents.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ws.tevents.push_back(e);
  }
  return ws.tevents[ws.tevent_next++];
}

TimeScope::TimeScope(Workspace& w, cudaStream_t s, int c, double f, const char* tg, int64_t kk)
    : ws(w), st(s), cls(c), flops(f), tag(tg), k(kk) {
  if (ws.timing) {
    a = ws_tevent(ws);
    cudaEventRecord(a, st);
  }
}
TimeScope::~TimeScope() {
  if (ws.timing) {
    cudaEvent_t b = ws_tevent(ws);
    cudaEventRecord(b, st);
    ws.timed.push_back({cls, a, b, flops, tag, k, (st == ws.panel || st == ws.gpanel) ? 1 : 0});
  }
}

static const char* kClassName[TC_COUNT] = {"panel", "symm", "syr2k", "gemm"};

int ws_collect_timing(Workspace& ws) {
  for (auto& t : ws.timed) {
    float ms = 0.f;
    BR_CUDA(cudaEventElapsedTime(&ms, t.a, t.b));
    ws.t_ms[t.cls] += ms;
    ws.t_flops[t.cls] += t.flops;
    ws.t_launches[t.cls] += 1;
    if (ws.timing >= 2 && ws.trace_base) {
      Workspace::TraceRec r{};
      const char* tg = t.tag ? t.tag : kClassName[t.cls];
      if (t.k >= 0) snprintf(r.id, sizeof(r.id), "%s@%lld", tg, (long long)t.k);
      else snprintf(r.id, sizeof(r.id), "%s", tg);
      r.stream = t.stream;
      float t0 = 0.f, t1 = 0.f;
      BR_CUDA(cudaEventElapsedTime(&t0, ws.trace_base, t.a));
      BR_CUDA(cudaEventElapsedTime(&t1, ws.trace_base, t.b));
      r.t0_us = 1e3 * t0;
      r.t1_us = 1e3 * t1;
      ws.trace.push_back(r);
    }
  }
  ws.timed.clear();
  ws.tevent_next = 0;
  return 0;
}

// ---------------------------------------------------------------------------
// elementwise kernels
// ---------------------------------------------------------------------------

// In-place finalize of the SEVP band (ref sevp.py:276-284): lower in-band
// entries kept, upper in-band entries mirrored from the lower triangle,
// everything with |i-j| > w set to exactly 0. Upper entries are only
// written, never read, so the input's upper triangle is never observed.
// Columns [c0, c0 + nc) only (the host entry points finalize and stream out
// finished column blocks while the reduction continues).
__global__ void finalize_sym_kernel(double* A, int64_t lda, int64_t n, int64_t c0, int64_t nc,
                                    int64_t w) {
  const int64_t total = n * nc;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % n, c = c0 + idx / n;
    const int64_t d = r - c;
    if (d > w || -d > w) A[r + c * lda] = 0.0;
    else if (d < 0) A[r + c * lda] = A[c + r * lda];
  }
}

// Exact off-band zeroing (ref svd.py:237-239 / oracles.py band pattern).
__global__ void mask_band_kernel(double* A, int64_t lda, int64_t m, int64_t c0, int64_t nc,
                                 int64_t lo, int64_t up) {
  const int64_t total = m * nc;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % m, c = c0 + idx / m;
    if (r - c > lo || c - r > up) A[r + c * lda] = 0.0;
  }
}

__global__ void identity_kernel(double* Q, int64_t ldq, int64_t n) {
  const int64_t total = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % n, c = idx / n;
    Q[r + c * ldq] = (r == c) ? 1.0 : 0.0;
  }
}

static int grid_for(int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 148 * 16));
}

int finalize_sym(cudaStream_t st, double* A, int64_t lda, int64_t n, int64_t w, int64_t c0,
                 int64_t c1) {
  if (c1 < 0) c1 = n;
  if (n <= 0 || c1 <= c0) return 0;
  count_launch();
  finalize_sym_kernel<<<grid_for(n * (c1 - c0)), 256, 0, st>>>(A, lda, n, c0, c1 - c0, w);
  BR_CUDA(cudaGetLastError());
  return 0;
}
int mask_tri(cudaStream_t st, double* A, int64_t lda, int64_t m, int64_t n, int64_t lo,
             int64_t up, int64_t c0, int64_t c1) {
  if (c1 < 0) c1 = n;
  if (m <= 0 || c1 <= c0) return 0;
  count_launch();
  mask_band_kernel<<<grid_for(m * (c1 - c0)), 256, 0, st>>>(A, lda, m, c0, c1 - c0, lo, up);
  BR_CUDA(cudaGetLastError());
  return 0;
}
int set_identity(cudaStream_t st, double* Q, int64_t ldq, int64_t n) {
  if (n <= 0) return 0;
  count_launch();
  identity_kernel<<<grid_for(n * n), 256, 0, st>>>(Q, ldq, n);
  BR_CUDA(cudaGetLastError());
  return 0;
}

// Finish columns [done, upto) of the band on the copy stream (after the main
// stream's work so far) and queue their D2H copy into the pinned host buffer.
int band_out_flush(Workspace& ws, BandOut* bo, int64_t upto) {
  if (!bo || upto <= bo->done) return 0;
  cudaEvent_t ev = ws_event(ws);
  BR_CUDA(cudaEventRecord(ev, ws.main));
  BR_CUDA(cudaStreamWaitEvent(bo->st, ev, 0));
  if (bo->sym) BR_CHECK(finalize_sym(bo->st, bo->A, bo->lda, bo->rows, bo->w, bo->done, upto));
  else BR_CHECK(mask_tri(bo->st, bo->A, bo->lda, bo->rows, upto, bo->lo, bo->up, bo->done, upto));
  BR_CUDA(cudaMemcpy2DAsync(bo->host + bo->done * bo->ldh, bo->ldh * sizeof(double),
                            bo->A + bo->done * bo->lda, bo->lda * sizeof(double),
                            bo->rows * sizeof(double), upto - bo->done, cudaMemcpyDeviceToHost,
                            bo->st));
  bo->done = upto;
  return 0;
}
int store_factors(Workspace& ws, cudaStream_t st, int chain, int64_t k, int64_t r0, int64_t j,
                  int64_t bp, const double* Y, int64_t ldy, const double* T, int64_t ldt,
                  const double* tau) {
  const br_factors* f = ws.fo;
  if (!f || j <= 0 || bp <= 0) return 0;
  double* y = chain ? f->yr : f->yl;
  double* t = chain ? f->tr : f->tl;
  double* ta = chain ? f->taur : f->taul;
  const int64_t ldyo = chain ? f->ldyr : f->ldyl, ldto = chain ? f->ldtr : f->ldtl;
  const size_t D = sizeof(double);
  if (y)
    BR_CUDA(cudaMemcpy2DAsync(y + r0 + k * ldyo, ldyo * D, Y, ldy * D, j * D, bp,
                              cudaMemcpyDeviceToDevice, st));
  if (t)
    BR_CUDA(cudaMemcpy2DAsync(t + k * ldto, ldto * D, T, ldt * D, bp * D, bp,
                              cudaMemcpyDeviceToDevice, st));
  if (ta) BR_CUDA(cudaMemcpyAsync(ta + k, tau, bp * D, cudaMemcpyDeviceToDevice, st));
  return 0;
}

int band_out_raw(Workspace& ws, BandOut* bo, int64_t cols) {
  if (!bo) return 0;
  cudaEvent_t ev = ws_event(ws);
  BR_CUDA(cudaEventRecord(ev, ws.main));
  BR_CUDA(cudaStreamWaitEvent(bo->st, ev, 0));
  BR_CUDA(cudaMemcpy2DAsync(bo->host, bo->ldh * sizeof(double), bo->A, bo->lda * sizeof(double),
                            bo->rows * sizeof(double), cols, cudaMemcpyDeviceToHost, bo->st));
  bo->done = cols;
  return 0;
}

int zero_fill(cudaStream_t st, MatView V) {
  if (V.rows <= 0 || V.cols <= 0) return 0;
  const int64_t r = V.trans ? V.cols : V.rows, c = V.trans ? V.rows : V.cols;
  BR_CUDA(cudaMemset2DAsync(V.p, V.ld * sizeof(double), 0, r * sizeof(double), c, st));
  return 0;
}

// Graph replay pays off while launch latency is a visible share of the run
// (c1/c2: -6 % / -5 %); for the large reductions the graph's replay of the
// two-stream program measured 10 % slower than the stream program itself, so
// only reductions below BR_GRAPH_MAX_FLOPS nominal flops (default 2e11) are
// graphed; BR_GRAPHS=0 disables graphs.
static bool graphs_enabled(double nominal) {
  static const bool on = [] {
    const char* e = std::getenv("BR_GRAPHS");
    return !(e && e[0] == '0');
  }();
  static const double lim = [] {
    const char* e = std::getenv("BR_GRAPH_MAX_FLOPS");
    return e ? std::atof(e) : 2e11;
  }();
  return on && nominal <= lim;
}

// Runs one reduction on the handle's streams, timed by events on `main`
// around the whole stream program (both streams joined at the end). Without
// timing, the stream program of a reduction that repeats with identical
// arguments is captured once into a CUDA graph (on its second call; the
// first call sizes the workspace) and replayed afterwards: one launch per
// reduction instead of hundreds, with the programmatic (PDL) edges kept.
template <class F>
int timed_reduction(Workspace& ws, br_stats* stats, double nominal, Workspace::GraphKey key,
                    F&& body) {
  cudaEvent_t e0, e1;
  BR_CUDA(cudaEventCreate(&e0));
  BR_CUDA(cudaEventCreate(&e1));
  const int64_t l0 = launch_count();
  auto cu = [](cudaError_t e) -> int {
    if (e == cudaSuccess) return 0;
    set_error("CUDA: %s", cudaGetErrorString(e));
    return 1000 + (int)e;
  };
  key.gen = alloc_generation();
  key.max_iters = ws.max_iters;
  if (ws.fo) key.fo = *ws.fo;
  key.main = ws.main;
  key.panel = ws.panel;
  key.timing = ws.timing;
  // events recorded by captured graph nodes cannot be timed, so the timing /
  // trace modes stay eager
  const bool graphable =
      graphs_enabled(nominal) && ws.timing == 0 && ws.main != nullptr && ws.band_out == nullptr &&
      ws.band_in == nullptr;
  const bool same = graphable && key == ws.gkey;
  ws.no_partition = graphable;  // green-context streams stay out of captured programs
  int rc = 0;
  int64_t iters = 0;
  float ms = 0.f;
  if (same && !ws.gexec && ws.gseen >= 1) {
    // capture the stream program (workspace already sized by the eager run)
    const int64_t c0 = launch_count();
    ws.timed.clear();
    ws.tevent_next = 0;
    rc = cu(cudaStreamBeginCapture(ws.main, cudaStreamCaptureModeRelaxed));
    if (!rc) {
      const int brc = body(&iters);
      cudaGraph_t g = nullptr;
      const cudaError_t ee = cudaStreamEndCapture(ws.main, &g);
      if (brc == 0 && ee == cudaSuccess && g) {
        if (cudaGraphInstantiate(&ws.gexec, g, 0) != cudaSuccess) ws.gexec = nullptr;
      }
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();  // a failed capture leaves no sticky error
      ws_events_reset(ws);
      if (brc != 0 && brc < 0) rc = brc;  // argument errors are real
      ws.g_iters = iters;
      ws.g_launches = launch_count() - c0;
      ws.timed.clear();
      g_launches_adjust(-(launch_count() - c0));  // the capture itself launched nothing
    }
    if (!ws.gexec) ws.gseen = -1000000;  // capture failed: stay eager for this key
  }
  rc = rc ? rc : cu(cudaEventRecord(e0, ws.main));
  ws.trace_base = e0;
  if (ws.timing >= 2) ws.trace.clear();
  if (!rc) {
    if (same && ws.gexec) {
      rc = cu(cudaGraphLaunch(ws.gexec, ws.main));
      iters = ws.g_iters;
      count_launch(ws.g_launches);
    } else {
      rc = body(&iters);
      if (graphable) {
        if (!same) {
          if (ws.gexec) cudaGraphExecDestroy(ws.gexec);
          ws.gexec = nullptr;
          ws.gkey = key;
          ws.gseen = 0;
        }
        ++ws.gseen;
      }
    }
  }
  if (!rc) rc = cu(cudaEventRecord(e1, ws.main));
  if (!rc) rc = cu(cudaEventSynchronize(e1));
  if (!rc) rc = cu(cudaStreamSynchronize(ws.panel));
  if (!rc && ws.gpanel) rc = cu(cudaStreamSynchronize(ws.gpanel));
  if (!rc && ws.gupd) rc = cu(cudaStreamSynchronize(ws.gupd));
  if (!rc) rc = cu(cudaGetLastError());
  if (!rc) rc = cu(cudaEventElapsedTime(&ms, e0, e1));
  if (!rc && ws.timing) rc = ws_collect_timing(ws);
  ws.trace_base = nullptr;
  if (rc) {
    ws.timed.clear();
    ws.tevent_next = 0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc) return rc;
  if (stats) {
    stats->iterations = iters;
    stats->device_ms = ms;
    stats->nominal_flops = nominal;
    stats->launches = launch_count() - l0;
  }
  return 0;
}

int band_in_start(Workspace& ws, BandIn* bi) {
  // the device buffer may still be read by work queued on main (none between
  // synchronous calls, but order the copies after it anyway)
  cudaEvent_t ev0 = ws_event(ws);
  BR_CUDA(cudaEventRecord(ev0, ws.main));
  BR_CUDA(cudaStreamWaitEvent(ws.copy_in, ev0, 0));
  for (int c = 0; c < bi->nchunks; ++c) {
    const int64_t c0 = (int64_t)c * bi->chunk, nc = std::min(bi->chunk, bi->cols - c0);
    BR_CUDA(cudaMemcpy2DAsync(bi->A + c0 * bi->lda, bi->lda * sizeof(double), bi->host + c0 * bi->ldh,
                              bi->ldh * sizeof(double), bi->rows * sizeof(double), nc,
                              cudaMemcpyHostToDevice, ws.copy_in));
    bi->ev[c] = ws_event(ws);
    BR_CUDA(cudaEventRecord(bi->ev[c], ws.copy_in));
  }
  bi->waited = 0;
  return 0;
}

int band_in_wait(Workspace& ws, BandIn* bi, int64_t upto) {
  if (!bi) return 0;
  const int need = (int)std::min<int64_t>(bi->nchunks, cdiv(std::max<int64_t>(upto, 0), bi->chunk));
  for (; bi->waited < need; ++bi->waited)
    BR_CUDA(cudaStreamWaitEvent(ws.main, bi->ev[bi->waited], 0));
  return 0;
}

}  // namespace br

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using namespace br;

struct br_handle_s {
  Workspace ws;
};

// Stream (and its split-K scratch) used by kernel-level calls: br_stream_select.
static cudaStream_t cur_stream(Workspace& ws) { return ws.active ? ws.panel : ws.main; }
static Scratch& cur_sk(Workspace& ws) { return ws.active ? ws.sk_panel : ws.sk_main; }
// Temporaries and panel scratch of kernel-level calls are per stream too, so
// calls issued concurrently on the two streams never share a buffer.
static DevBuf& cur_tmp(Workspace& ws) { return ws.active ? ws.tmp_panel : ws.tmp; }
static DevBuf& cur_pscr(Workspace& ws) { return ws.active ? ws.pscratch_panel : ws.pscratch; }

#define ARG(cond, i)                                   \
  do {                                                 \
    if (!(cond)) {                                     \
      set_error("invalid argument %d (%s)", i, #cond); \
      return -(i);                                     \
    }                                                  \
  } while (0)

#define DEV(h)                                  \
  do {                                          \
    BR_CUDA(cudaSetDevice((h)->ws.device));     \
  } while (0)

static int ensure_scratch(Workspace& ws, int64_t main_doubles, int64_t panel_doubles,
                          int64_t pscr) {
  const int64_t both = std::max(main_doubles, panel_doubles);
  BR_CHECK(devbuf_reserve(ws.skbuf_main, both));
  BR_CHECK(devbuf_reserve(ws.skbuf_panel, both));
  BR_CHECK(devbuf_reserve(ws.skbuf_aux, both));
  BR_CHECK(devbuf_reserve(cur_pscr(ws), pscr));
  ws.sk_main.p = ws.skbuf_main.p;
  ws.sk_main.cap = ws.skbuf_main.cap;
  ws.sk_panel.p = ws.skbuf_panel.p;
  ws.sk_panel.cap = ws.skbuf_panel.cap;
  ws.sk_aux.p = ws.skbuf_aux.p;
  ws.sk_aux.cap = ws.skbuf_aux.cap;
  ws.sk_main.num_sms = ws.sk_panel.num_sms = ws.sk_aux.num_sms = ws.num_sms;
  return 0;
}

// Optional SM partition for the panel stream (BR_GREEN_SMS = N): a green
// context holding N SMs; the panel stream is created on it, so panel
// kernels (leaf clusters, panel GEMMs) are confined to those SMs while the
// main stream's kernels keep the whole device. Driver entry points are
// resolved through the runtime (no libcuda link).
typedef CUresult (*PFN_getDevRes)(CUdevice, CUdevResource*, CUdevResourceType);
typedef CUresult (*PFN_split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned,
                              unsigned);
typedef CUresult (*PFN_genDesc)(CUdevResourceDesc*, CUdevResource*, unsigned);
typedef CUresult (*PFN_gcCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
typedef CUresult (*PFN_gcStream)(CUstream*, CUgreenCtx, unsigned, int);
template <class F>
static int drv_sym(const char* name, F* f) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  BR_CUDA(cudaGetDriverEntryPointByVersion(name, &p, 12090, cudaEnableDefault, &q));
  if (!p || q != cudaDriverEntryPointSuccess) {
    set_error("driver entry point %s unavailable", name);
    return 1;
  }
  *f = (F)p;
  return 0;
}
// Stream on the complement of an nsm-SM partition (see Workspace::gupd).
typedef CUresult (*PFN_gcDestroy)(CUgreenCtx);
static int green_update_stream(int device, int nsm, int prio, cudaStream_t* upd, int* got_sms,
                               cudaStream_t* panel, int panel_prio, int* panel_sms, void** ctx_upd,
                               void** ctx_panel) {
  PFN_getDevRes getres;
  PFN_split split;
  PFN_genDesc gen;
  PFN_gcCreate create;
  PFN_gcStream mkstream;
  BR_CHECK(drv_sym("cuDeviceGetDevResource", &getres));
  BR_CHECK(drv_sym("cuDevSmResourceSplitByCount", &split));
  BR_CHECK(drv_sym("cuDevResourceGenerateDesc", &gen));
  BR_CHECK(drv_sym("cuGreenCtxCreate", &create));
  BR_CHECK(drv_sym("cuGreenCtxStreamCreate", &mkstream));
  CUdevResource sm, part, rest;
  unsigned n = 1;
  if (getres((CUdevice)device, &sm, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
      split(&part, &n, &sm, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, (unsigned)nsm) !=
          CUDA_SUCCESS ||
      n != 1 || rest.sm.smCount == 0) {
    set_error("green context: SM split of %d failed", nsm);
    return 1;
  }
  CUdevResourceDesc desc;
  CUgreenCtx g;
  if (gen(&desc, &rest, 1) != CUDA_SUCCESS ||
      create(&g, desc, (CUdevice)device, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    set_error("green context creation failed");
    return 1;
  }
  CUstream s1;
  if (mkstream(&s1, g, CU_STREAM_NON_BLOCKING, prio) != CUDA_SUCCESS) {
    set_error("green context stream creation failed");
    return 1;
  }
  *upd = (cudaStream_t)s1;
  *got_sms = (int)rest.sm.smCount;
  *ctx_upd = (void*)g;
  if (panel) {  // experimental: a panel stream on the nsm SMs themselves (strict split)
    CUdevResourceDesc pdesc;
    CUgreenCtx pg;
    CUstream s2;
    if (gen(&pdesc, &part, 1) != CUDA_SUCCESS ||
        create(&pg, pdesc, (CUdevice)device, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        mkstream(&s2, pg, CU_STREAM_NON_BLOCKING, panel_prio) != CUDA_SUCCESS) {
      set_error("green context (panel side) creation failed");
      return 1;
    }
    *panel = (cudaStream_t)s2;
    *panel_sms = (int)part.sm.smCount;
    *ctx_panel = (void*)pg;
  }
  return 0;
}

static int green_panel_streams(int device, int nsm, int prio, cudaStream_t* panel, cudaStream_t* aux,
                               int* got_sms) {
  PFN_getDevRes getres;
  PFN_split split;
  PFN_genDesc gen;
  PFN_gcCreate create;
  PFN_gcStream mkstream;
  BR_CHECK(drv_sym("cuDeviceGetDevResource", &getres));
  BR_CHECK(drv_sym("cuDevSmResourceSplitByCount", &split));
  BR_CHECK(drv_sym("cuDevResourceGenerateDesc", &gen));
  BR_CHECK(drv_sym("cuGreenCtxCreate", &create));
  BR_CHECK(drv_sym("cuGreenCtxStreamCreate", &mkstream));
  CUdevResource sm, part, rest;
  unsigned n = 1;
  if (getres((CUdevice)device, &sm, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
      split(&part, &n, &sm, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, (unsigned)nsm) !=
          CUDA_SUCCESS ||
      n != 1) {
    set_error("green context: SM split of %d failed", nsm);
    return 1;
  }
  CUdevResourceDesc desc;
  CUgreenCtx g;
  if (gen(&desc, &part, 1) != CUDA_SUCCESS || create(&g, desc, (CUdevice)device, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
    set_error("green context creation failed");
    return 1;
  }
  CUstream s1, s2;
  if (mkstream(&s1, g, CU_STREAM_NON_BLOCKING, prio) != CUDA_SUCCESS ||
      mkstream(&s2, g, CU_STREAM_NON_BLOCKING, prio) != CUDA_SUCCESS) {
    set_error("green context stream creation failed");
    return 1;
  }
  *panel = (cudaStream_t)s1;
  *aux = (cudaStream_t)s2;
  *got_sms = (int)part.sm.smCount;
  return 0;
}

extern "C" {

int br_version(void) { return 100; }
int64_t br_launch_count(void) { return launch_count(); }
const char* br_last_error(void) { return g_err; }

int br_create(int device, br_handle_t* out) {
  ARG(out != nullptr, 2);
  int ndev = 0;
  BR_CUDA(cudaGetDeviceCount(&ndev));
  ARG(device >= 0 && device < ndev, 1);
  BR_CUDA(cudaSetDevice(device));
  auto* h = new (std::nothrow) br_handle_s();
  if (!h) {
    set_error("out of host memory");
    return 1;
  }
  h->ws.device = device;
  BR_CUDA(cudaDeviceGetAttribute(&h->ws.num_sms, cudaDevAttrMultiProcessorCount, device));
  int lo = 0, hi = 0;
  BR_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  BR_CUDA(cudaStreamCreateWithPriority(&h->ws.own_main, cudaStreamNonBlocking, lo));
  // BR_PANEL_PRIO=lo (tuning aid): panel stream at the main stream's priority
  const char* pp = std::getenv("BR_PANEL_PRIO");
  BR_CUDA(cudaStreamCreateWithPriority(&h->ws.own_panel, cudaStreamNonBlocking,
                                       (pp && pp[0] == 'l') ? lo : hi));
  h->ws.main = h->ws.own_main;
  h->ws.panel = h->ws.own_panel;
  BR_CUDA(cudaStreamCreateWithPriority(&h->ws.aux, cudaStreamNonBlocking, hi));
  if (const char* g = std::getenv("BR_GREEN_SMS")) {  // experimental SM partition (see above)
    cudaStream_t gp = nullptr, ga = nullptr;
    int got = 0;
    const int rc = green_panel_streams(device, std::atoi(g), hi, &gp, &ga, &got);
    if (rc) return rc;
    h->ws.gpanel = gp;
    h->ws.green_sms = got;
    if (const char* r = std::getenv("BR_GREEN_ROWS")) h->ws.green_rows = std::atoll(r);
  }
  {
    // SMs kept free of overlapped update CTAs (Workspace::gupd): 16 = one leaf
    // cluster; BR_UPD_SMS=0 disables the partition, BR_UPD_ROWS moves the
    // trailing-rows threshold. Measured (tools/exp_upd.sh): c4 441.5 -> 433.8 ms,
    // c3 44.4 -> 42.0 ms, c5 1572 -> 1568 ms; 8 SMs do nothing, 24-48 lose more
    // update throughput than the panels gain. A driver without green contexts
    // just runs without the partition.
    const char* g = std::getenv("BR_UPD_SMS");
    // Nsight Compute cannot prepare kernels launched on green-context streams
    // ("Failed to prepare kernel for profiling"): under its injection the
    // partition stays off unless BR_UPD_SMS asks for it, so `ncu python
    // bench.py` and the launch lists in profiles/ work (they then show the
    // two-stream program without the partition)
    const bool profiled = std::getenv("NV_NSIGHT_INJECTION_PORT_BASE") != nullptr ||
                          std::getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") != nullptr;
    const int nres = g ? std::atoi(g) : (profiled ? 0 : 16);
    if (nres > 0) {
      cudaStream_t gu = nullptr;
      int got = 0;
      // Strict split for the triangular band's tall panels (BR_SPLIT_ROWS = R,
      // default 10240, 0 disables): above R rows the update has slack over the
      // panels, and what it loses beside them are dispatch pauses around the
      // panel's ~70 launches. There the leaves and block updates of a panel run
      // confined to the nres SMs (panel_qr phase 1), only the three full-size
      // products that finish it (Gram, T, W) on the whole device, and the
      // overlapped update on the other SMs: update class 411 -> 404 ms, c4
      // 433.8 -> 430.2 ms (tools/exp_upd.sh). Without the two-phase panel the
      // confined panels became the bottleneck (447 ms).
      const char* sre = std::getenv("BR_SPLIT_ROWS");
      const int64_t srows = sre ? std::atoll(sre) : 10240;
      const bool sr = srows > 0;
      cudaStream_t gp = nullptr;
      int gps = 0;
      if (green_update_stream(device, nres, lo, &gu, &got, sr ? &gp : nullptr, hi, &gps, &h->ws.gctx_upd,
                              &h->ws.gctx_panel) == 0) {
        h->ws.gupd = gu;
        h->ws.upd_sms = got;
        h->ws.upd_rows = 10240;
        if (const char* r = std::getenv("BR_UPD_ROWS")) h->ws.upd_rows = std::atoll(r);
        if (sr && gp && !panel_clusters_fit(gp)) {  // this board's partition cannot hold a leaf cluster
          cudaStreamDestroy(gp);
          gp = nullptr;
        }
        if (std::getenv("BR_DEBUG_PARTITION"))
          fprintf(stderr, "bandred: update partition %d SMs, panel partition %d SMs, strict split %s\n", got,
                  gps, (sr && gp) ? "on" : "off");
        if (sr && gp) {
          h->ws.gpanel = gp;
          h->ws.green_sms = gps;
          h->ws.green_rows = srows;
          h->ws.split_upd = true;
        }
      } else {
        cudaGetLastError();
        set_error("%s", "");
      }
    }
  }
  BR_CUDA(cudaStreamCreateWithFlags(&h->ws.copy, cudaStreamNonBlocking));
  BR_CUDA(cudaStreamCreateWithFlags(&h->ws.copy_in, cudaStreamNonBlocking));
  // [0, 128): persistent-panel handshakes; [128, 130): xchain grid barrier
  BR_CUDA(cudaMalloc(&h->ws.flags, 256 * sizeof(unsigned)));
  BR_CUDA(cudaMemset(h->ws.flags, 0, 256 * sizeof(unsigned)));
  BR_CUDA(cudaEventCreateWithFlags(&h->ws.ev_aux0, cudaEventDisableTiming));
  BR_CUDA(cudaEventCreateWithFlags(&h->ws.ev_aux1, cudaEventDisableTiming));
  // load every kernel now: under lazy loading a first launch inside the
  // persistent panel's handshake would wait for the spinning panel kernel
  g_preload_only = true;
  int prc = preload_gemm_kernels();
  if (!prc) prc = preload_panel_kernels();
  if (!prc) prc = preload_xchain_kernels();
  if (!prc) prc = preload_stage2_kernels();
  g_preload_only = false;
  if (prc) return prc;
  {
    cudaFuncAttributes fa;
    BR_CUDA(cudaFuncGetAttributes(&fa, finalize_sym_kernel));
    BR_CUDA(cudaFuncGetAttributes(&fa, mask_band_kernel));
    BR_CUDA(cudaFuncGetAttributes(&fa, identity_kernel));
  }
  *out = h;
  return 0;
}

int br_destroy(br_handle_t h) {
  if (!h) return 0;
  cudaSetDevice(h->ws.device);
  cudaDeviceSynchronize();
  Workspace& ws = h->ws;
  devbuf_free(ws.skbuf_main);
  devbuf_free(ws.skbuf_panel);
  devbuf_free(ws.pscratch);
  devbuf_free(ws.factors);
  devbuf_free(ws.tmp);
  devbuf_free(ws.tmp_panel);
  devbuf_free(ws.s2prog);
  devbuf_free(ws.pscratch_panel);
  devbuf_free(ws.stageA);
  devbuf_free(ws.stageQ);
  devbuf_free(ws.stageF);
  devbuf_free(ws.skbuf_aux);
  if (ws.flags) cudaFree(ws.flags);
  if (ws.ev_aux0) cudaEventDestroy(ws.ev_aux0);
  if (ws.ev_aux1) cudaEventDestroy(ws.ev_aux1);
  if (ws.aux) cudaStreamDestroy(ws.aux);
  if (ws.copy) cudaStreamDestroy(ws.copy);
  if (ws.copy_in) cudaStreamDestroy(ws.copy_in);
  for (auto e : ws.events) cudaEventDestroy(e);
  for (auto e : ws.tevents) cudaEventDestroy(e);
  if (ws.gexec) cudaGraphExecDestroy(ws.gexec);
  if (ws.gupd) cudaStreamDestroy(ws.gupd);
  if (ws.split_upd && ws.gpanel) cudaStreamDestroy(ws.gpanel);
  {
    PFN_gcDestroy gdestroy = nullptr;
    if ((ws.gctx_upd || ws.gctx_panel) && drv_sym("cuGreenCtxDestroy", &gdestroy) == 0) {
      if (ws.gctx_upd) gdestroy((CUgreenCtx)ws.gctx_upd);
      if (ws.gctx_panel) gdestroy((CUgreenCtx)ws.gctx_panel);
    }
  }
  if (ws.own_main) cudaStreamDestroy(ws.own_main);
  if (ws.own_panel) cudaStreamDestroy(ws.own_panel);
  delete h;
  return 0;
}

int br_set_streams(br_handle_t h, void* main_stream, void* panel_stream) {
  ARG(h != nullptr, 1);
  h->ws.main = main_stream ? (cudaStream_t)main_stream : h->ws.own_main;
  h->ws.panel = panel_stream ? (cudaStream_t)panel_stream : h->ws.own_panel;
  return 0;
}

int br_sync(br_handle_t h) {
  ARG(h != nullptr, 1);
  DEV(h);
  BR_CUDA(cudaStreamSynchronize(h->ws.main));
  BR_CUDA(cudaStreamSynchronize(h->ws.panel));
  if (h->ws.gpanel) BR_CUDA(cudaStreamSynchronize(h->ws.gpanel));
  if (h->ws.gupd) BR_CUDA(cudaStreamSynchronize(h->ws.gupd));
  return 0;
}

int br_set_timing(br_handle_t h, int enable) {
  ARG(h != nullptr, 1);
  ARG(enable >= 0 && enable <= 2, 2);
  h->ws.timing = enable;
  h->ws.trace.clear();
  for (int c = 0; c < TC_COUNT; ++c) {
    h->ws.t_ms[c] = 0;
    h->ws.t_flops[c] = 0;
    h->ws.t_launches[c] = 0;
  }
  h->ws.timed.clear();
  h->ws.tevent_next = 0;
  return 0;
}

int br_get_timing(br_handle_t h, int cls, double* ms, double* flops, int64_t* launches) {
  ARG(h != nullptr, 1);
  ARG(cls >= 0 && cls < TC_COUNT, 2);
  if (ms) *ms = h->ws.t_ms[cls];
  if (flops) *flops = h->ws.t_flops[cls];
  if (launches) *launches = h->ws.t_launches[cls];
  return 0;
}

int64_t br_trace_count(br_handle_t h) { return h ? (int64_t)h->ws.trace.size() : -1; }

int br_trace_get(br_handle_t h, int64_t idx, char* id, int64_t idlen, int* stream, double* t0_us,
                 double* t1_us) {
  ARG(h != nullptr, 1);
  ARG(idx >= 0 && idx < (int64_t)h->ws.trace.size(), 2);
  const auto& r = h->ws.trace[idx];
  if (id && idlen > 0) snprintf(id, (size_t)idlen, "%s", r.id);
  if (stream) *stream = r.stream;
  if (t0_us) *t0_us = r.t0_us;
  if (t1_us) *t1_us = r.t1_us;
  return 0;
}

int br_house_gen(br_handle_t h, int64_t L, const double* x, double* v, double* tau_beta) {
  ARG(h != nullptr, 1);
  ARG(L >= 1, 2);
  ARG(x && v && tau_beta, 3);
  DEV(h);
  return house_gen_dev(cur_stream(h->ws), L, x, v, tau_beta);
}

static int qr_common(br_handle_t h, MatView P, double* Y, int64_t ldy, double* T, int64_t ldt,
                     double* W, int64_t ldw, double* tau) {
  Workspace& ws = h->ws;
  const int64_t j = P.rows, b = P.cols;
  BR_CHECK(ensure_scratch(ws, 4 * std::max<int64_t>(j, 1) * b + (1 << 20), (1 << 20) + 4 * j * b,
                          panel_scratch_doubles(b)));
  MatView Yv(Y, ldy, j, b), Tv(T, ldt, b, b), Wv(W, ldw, j, b);
  return panel_qr(cur_stream(ws), cur_sk(ws), cur_pscr(ws), P, Yv, tau, Tv, W ? &Wv : nullptr, 0,
                  &ws);
}

int br_qr_panel(br_handle_t h, int64_t j, int64_t b, double* P, int64_t ldp, double* Y,
                int64_t ldy, double* T, int64_t ldt, double* W, int64_t ldw, double* tau) {
  ARG(h != nullptr, 1);
  ARG(b >= 1 && j >= b, 2);
  ARG(P != nullptr && ldp >= j, 4);
  ARG(Y != nullptr && ldy >= j, 6);
  ARG(T != nullptr && ldt >= b, 8);
  ARG(W == nullptr || ldw >= j, 11);
  ARG(tau != nullptr, 12);
  DEV(h);
  return qr_common(h, MatView(P, ldp, j, b), Y, ldy, T, ldt, W, ldw, tau);
}

int br_lq_panel(br_handle_t h, int64_t b, int64_t j, double* P, int64_t ldp, double* Y,
                int64_t ldy, double* T, int64_t ldt, double* W, int64_t ldw, double* tau) {
  ARG(h != nullptr, 1);
  ARG(b >= 1 && j >= b, 3);
  ARG(P != nullptr && ldp >= b, 4);
  ARG(Y != nullptr && ldy >= j, 6);
  ARG(T != nullptr && ldt >= b, 8);
  ARG(W == nullptr || ldw >= j, 11);
  ARG(tau != nullptr, 12);
  DEV(h);
  // LQ of the b x j rows == QR of the transposed (j x b) view
  return qr_common(h, MatView(P, ldp, j, b, true), Y, ldy, T, ldt, W, ldw, tau);
}

int br_build_w(br_handle_t h, int64_t j, int64_t b, const double* Y, int64_t ldy,
               const double* T, int64_t ldt, double* W, int64_t ldw) {
  ARG(h != nullptr, 1);
  ARG(j >= 0 && b >= 0, 2);
  ARG(Y && ldy >= std::max<int64_t>(j, 1), 4);
  ARG(T && ldt >= std::max<int64_t>(b, 1), 6);
  ARG(W && ldw >= std::max<int64_t>(j, 1), 8);
  DEV(h);
  Workspace& ws = h->ws;
  BR_CHECK(ensure_scratch(ws, 4 * std::max<int64_t>(j, 1) * std::max<int64_t>(b, 1) + (1 << 20),
                          1 << 20, panel_scratch_doubles(1)));
  // W[:, i] = Y[:, :i+1] T[:i+1, i] (ref kernels.py:139-149): only T's upper
  // triangle is read
  return gemm(cur_stream(ws), cur_sk(ws), MatView(W, ldw, j, b), MatView((double*)Y, ldy, j, b),
              MatView((double*)T, ldt, b, b), 1.0, 0.0, nullptr, 0, 0, true);
}

int br_apply_wy_left(br_handle_t h, int64_t rows, int64_t cols, double* A, int64_t lda,
                     const double* Y, int64_t ldy, const double* W, int64_t ldw, int64_t b) {
  ARG(h != nullptr, 1);
  ARG(rows >= 0, 2);
  ARG(cols >= 0, 3);
  ARG(A && lda >= std::max<int64_t>(rows, 1), 4);
  ARG(Y && ldy >= std::max<int64_t>(rows, 1), 6);
  ARG(W && ldw >= std::max<int64_t>(rows, 1), 8);
  ARG(b >= 0, 10);
  DEV(h);
  if (rows == 0 || cols == 0 || b == 0) return 0;
  Workspace& ws = h->ws;
  BR_CHECK(ensure_scratch(ws, 4 * std::max(rows, cols) * b + (1 << 20), 1 << 20,
                          panel_scratch_doubles(1)));
  DevBuf& tmp = cur_tmp(ws);
  BR_CHECK(devbuf_reserve(tmp, b * cols));
  MatView Z(tmp.p, b, b, cols), Av(A, lda, rows, cols);
  BR_CHECK(gemm(cur_stream(ws), cur_sk(ws), Z, MatView((double*)W, ldw, rows, b).T(), Av, 1.0, 0.0));
  return gemm(cur_stream(ws), cur_sk(ws), Av, MatView((double*)Y, ldy, rows, b), Z, 1.0, 1.0);
}

int br_apply_wy_right(br_handle_t h, int64_t rows, int64_t cols, double* A, int64_t lda,
                      const double* Y, int64_t ldy, const double* W, int64_t ldw, int64_t b) {
  ARG(h != nullptr, 1);
  ARG(rows >= 0, 2);
  ARG(cols >= 0, 3);
  ARG(A && lda >= std::max<int64_t>(rows, 1), 4);
  ARG(Y && ldy >= std::max<int64_t>(cols, 1), 6);
  ARG(W && ldw >= std::max<int64_t>(cols, 1), 8);
  ARG(b >= 0, 10);
  DEV(h);
  if (rows == 0 || cols == 0 || b == 0) return 0;
  Workspace& ws = h->ws;
  BR_CHECK(ensure_scratch(ws, 4 * std::max(rows, cols) * b + (1 << 20), 1 << 20,
                          panel_scratch_doubles(1)));
  DevBuf& tmp = cur_tmp(ws);
  BR_CHECK(devbuf_reserve(tmp, rows * b));
  MatView Z(tmp.p, rows, rows, b), Av(A, lda, rows, cols);
  BR_CHECK(gemm(cur_stream(ws), cur_sk(ws), Z, Av, MatView((double*)W, ldw, cols, b), 1.0, 0.0));
  return gemm(cur_stream(ws), cur_sk(ws), Av, Z, MatView((double*)Y, ldy, cols, b).T(), 1.0, 1.0);
}

int br_symm_lower(br_handle_t h, int64_t j, int64_t b, const double* A2, int64_t lda,
                  const double* W, int64_t ldw, double* X1, int64_t ldx) {
  ARG(h != nullptr, 1);
  ARG(j >= 0, 2);
  ARG(b >= 0, 3);
  ARG(A2 && lda >= std::max<int64_t>(j, 1), 4);
  ARG(W && ldw >= std::max<int64_t>(j, 1), 6);
  ARG(X1 && ldx >= std::max<int64_t>(j, 1), 8);
  DEV(h);
  if (j == 0 || b == 0) return 0;
  Workspace& ws = h->ws;
  BR_CHECK(ensure_scratch(ws, 4 * j * b + (1 << 20), 1 << 20, panel_scratch_doubles(1)));
  return symm_lower(cur_stream(ws), cur_sk(ws), MatView(X1, ldx, j, b), MatView((double*)A2, lda, j, j),
                    MatView((double*)W, ldw, j, b));
}

int br_syr2k_lower(br_handle_t h, int64_t j, int64_t b, double* A2, int64_t lda,
                   const double* X3, int64_t ldx, const double* Y, int64_t ldy, int64_t c0,
                   int64_t c1) {
  ARG(h != nullptr, 1);
  ARG(j >= 0, 2);
  ARG(b >= 0, 3);
  ARG(A2 && lda >= std::max<int64_t>(j, 1), 4);
  ARG(X3 && ldx >= std::max<int64_t>(j, 1), 6);
  ARG(Y && ldy >= std::max<int64_t>(j, 1), 8);
  ARG(0 <= c0 && c0 <= c1 && c1 <= j, 10);
  DEV(h);
  if (j == 0 || b == 0 || c0 == c1) return 0;
  return syr2k_lower(cur_stream(h->ws), MatView(A2, lda, j, j), MatView((double*)X3, ldx, j, b),
                     MatView((double*)Y, ldy, j, b), c0, c1);
}

// Block-cyclic slab kernels of the distributed SEVP (dist.py):
// the rank's owned trailing block columns as ONE j x ncols slab, local column
// c = trailing column r0 + (c / bs) * stride + c % bs, zeros above it.
int br_symm_lower_cyclic(br_handle_t h, int64_t j, int64_t ncols, int64_t b, const double* L,
                         int64_t ldl, const double* W, int64_t ldw, double* X1, int64_t ldx,
                         int64_t r0, int64_t bs, int64_t stride, int64_t p0, int64_t p1) {
  ARG(h != nullptr, 1);
  ARG(j >= 0, 2);
  ARG(ncols >= 0, 3);
  ARG(b >= 0, 4);
  ARG(L || ncols == 0, 5);
  ARG(ldl >= std::max<int64_t>(j, 1), 6);
  ARG(W && ldw >= std::max<int64_t>(j, 1), 8);
  ARG(0 <= p0 && p0 <= p1 && p1 <= j, 14);
  ARG(X1 && ldx >= std::max<int64_t>(p1 - p0, 1), 10);
  ARG(r0 >= 0, 11);
  ARG(bs >= 1 && (ncols % bs) == 0, 12);
  ARG(stride >= bs, 13);
  DEV(h);
  if (j == 0 || b == 0) return 0;
  Workspace& ws = h->ws;
  BR_CHECK(ensure_scratch(ws, 4 * std::max(j, ncols) * b + (1 << 20), 1 << 20, panel_scratch_doubles(1)));
  DevBuf& tmp = cur_tmp(ws);
  BR_CHECK(devbuf_reserve(tmp, 2 * std::max<int64_t>(ncols, 1) * b));
  return symm_cyclic(cur_stream(ws), cur_sk(ws), MatView(X1, ldx, p1 - p0, b),
                     MatView((double*)L, ldl, j, ncols), MatView((double*)W, ldw, j, b),
                     CycCols{r0, (int)bs, (int)stride}, tmp.p, p0, p1);
}

int br_syr2k_lower_cyclic(br_handle_t h, int64_t j, int64_t ncols, int64_t b, double* L,
                          int64_t ldl, const double* X3, int64_t ldx, const double* Y, int64_t ldy,
                          int64_t r0, int64_t bs, int64_t stride) {
  ARG(h != nullptr, 1);
  ARG(j >= 0, 2);
  ARG(ncols >= 0, 3);
  ARG(b >= 0, 4);
  ARG(L || ncols == 0, 5);
  ARG(ldl >= std::max<int64_t>(j, 1), 6);
  ARG(X3 && ldx >= std::max<int64_t>(j, 1), 8);
  ARG(Y && ldy >= std::max<int64_t>(j, 1), 10);
  ARG(r0 >= 0, 11);
  ARG(bs >= 1 && (ncols % bs) == 0, 12);
  ARG(stride >= bs, 13);
  DEV(h);
  if (j == 0 || b == 0 || ncols == 0) return 0;
  Workspace& ws = h->ws;
  DevBuf& tmp = cur_tmp(ws);
  BR_CHECK(devbuf_reserve(tmp, 2 * ncols * b));
  return syr2k_cyclic(cur_stream(ws), MatView(L, ldl, j, ncols), MatView((double*)X3, ldx, j, b),
                      MatView((double*)Y, ldy, j, b), CycCols{r0, (int)bs, (int)stride}, tmp.p);
}

// ---- second stage (no reference counterpart) ----------------
int br_band_to_tridiag(br_handle_t h, int64_t n, int64_t w, double* A, int64_t lda, double* d,
                       double* e) {
  ARG(h != nullptr, 1);
  ARG(n >= 0, 2);
  ARG(w >= 1 && w <= 128, 3);
  ARG(A || n == 0, 4);
  ARG(lda >= std::max<int64_t>(n, 1), 5);
  ARG(d || n == 0, 6);
  ARG(e || n <= 1, 7);
  DEV(h);
  if (n == 0) return 0;
  Workspace& ws = h->ws;
  BR_CHECK(devbuf_reserve(ws.s2prog, n / 2 + 1));
  return band_to_condensed(cur_stream(ws), false, n, w, A, lda, d, e, (int*)ws.s2prog.p, ws.num_sms);
}

int br_band_to_bidiag(br_handle_t h, int64_t m, int64_t n, int64_t w, double* A, int64_t lda,
                      double* d, double* e) {
  ARG(h != nullptr, 1);
  ARG(m >= 0, 2);
  ARG(n >= 0 && n <= m, 3);
  ARG(w >= 1 && w <= 128, 4);
  ARG(A || n == 0, 5);
  ARG(lda >= std::max<int64_t>(m, 1), 6);
  ARG(d || n == 0, 7);
  ARG(e || n <= 1, 8);
  DEV(h);
  if (n == 0) return 0;
  Workspace& ws = h->ws;
  BR_CHECK(devbuf_reserve(ws.s2prog, n / 2 + 1));
  return band_to_condensed(cur_stream(ws), true, n, w, A, lda, d, e, (int*)ws.s2prog.p, ws.num_sms);
}

int br_stream_select(br_handle_t h, int which) {
  ARG(h != nullptr, 1);
  ARG(which == 0 || which == 1, 2);
  h->ws.active = which;
  return 0;
}

int br_stream_join(br_handle_t h, int waiter) {
  ARG(h != nullptr, 1);
  ARG(waiter == 0 || waiter == 1, 2);
  DEV(h);
  Workspace& ws = h->ws;
  cudaStream_t w = waiter ? ws.panel : ws.main, o = waiter ? ws.main : ws.panel;
  cudaEvent_t ev = ws_event(ws);
  BR_CUDA(cudaEventRecord(ev, o));
  BR_CUDA(cudaStreamWaitEvent(w, ev, 0));
  if (ws.event_next > 4096) ws_events_reset(ws);
  return 0;
}

int br_gemm(br_handle_t h, int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha,
            const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
            int64_t ldc) {
  ARG(h != nullptr, 1);
  ARG(m >= 0, 4);
  ARG(n >= 0, 5);
  ARG(k >= 0, 6);
  ARG(A != nullptr || m == 0 || k == 0, 8);
  ARG(lda >= std::max<int64_t>(1, transa ? k : m), 9);
  ARG(B != nullptr || n == 0 || k == 0, 10);
  ARG(ldb >= std::max<int64_t>(1, transb ? n : k), 11);
  ARG(C != nullptr || m == 0 || n == 0, 13);
  ARG(ldc >= std::max<int64_t>(1, m), 14);
  DEV(h);
  if (m == 0 || n == 0) return 0;
  Workspace& ws = h->ws;
  // split-K partials: S * m * n doubles for S splits; pick_kps only splits
  // products whose partials fit, so a large C is simply not split (the
  // budget stays <= 4 m n and <= 64 Mi doubles instead of growing with C)
  BR_CHECK(ensure_scratch(ws, std::min<int64_t>(4 * m * n, (int64_t)1 << 26) + (1 << 20), 1 << 20,
                          panel_scratch_doubles(1)));
  MatView Av = transa ? MatView((double*)A, lda, k, m).T() : MatView((double*)A, lda, m, k);
  MatView Bv = transb ? MatView((double*)B, ldb, n, k).T() : MatView((double*)B, ldb, k, n);
  return gemm(cur_stream(ws), cur_sk(ws), MatView(C, ldc, m, n), Av, Bv, alpha, beta);
}

int br_symm_lower_ex(br_handle_t h, int64_t j, int64_t b, double alpha, const double* A2,
                     int64_t lda, const double* W, int64_t ldw, double beta, double* X1,
                     int64_t ldx) {
  ARG(h != nullptr, 1);
  ARG(j >= 0, 2);
  ARG(b >= 0, 3);
  ARG(A2 && lda >= std::max<int64_t>(j, 1), 5);
  ARG(W && ldw >= std::max<int64_t>(j, 1), 7);
  ARG(X1 && ldx >= std::max<int64_t>(j, 1), 10);
  DEV(h);
  if (j == 0 || b == 0) return 0;
  Workspace& ws = h->ws;
  BR_CHECK(ensure_scratch(ws, 4 * j * b + (1 << 20), 1 << 20, panel_scratch_doubles(1)));
  return symm_lower(cur_stream(ws), cur_sk(ws), MatView(X1, ldx, j, b),
                    MatView((double*)A2, lda, j, j), MatView((double*)W, ldw, j, b), alpha, beta);
}

int br_sym_two_sided_update(br_handle_t h, int64_t j, int64_t b, double* A2, int64_t lda,
                            const double* Y, int64_t ldy, const double* W, int64_t ldw) {
  ARG(h != nullptr, 1);
  ARG(j >= 0, 2);
  ARG(b >= 0, 3);
  ARG(A2 && lda >= std::max<int64_t>(j, 1), 4);
  ARG(Y && ldy >= std::max<int64_t>(j, 1), 6);
  ARG(W && ldw >= std::max<int64_t>(j, 1), 8);
  DEV(h);
  if (j == 0 || b == 0) return 0;
  Workspace& ws = h->ws;
  BR_CHECK(ensure_scratch(ws, 4 * j * b + (1 << 20), 1 << 20, panel_scratch_doubles(1)));
  DevBuf& tmp = cur_tmp(ws);
  BR_CHECK(devbuf_reserve(tmp, 2 * j * b + b * b));
  MatView X1(tmp.p, j, j, b), X3(tmp.p + j * b, j, j, b), X2(tmp.p + 2 * j * b, b, b, b);
  MatView A2v(A2, lda, j, j), Yv((double*)Y, ldy, j, b), Wv((double*)W, ldw, j, b);
  BR_CHECK(symm_lower(cur_stream(ws), cur_sk(ws), X1, A2v, Wv));
  BR_CHECK(gemm(cur_stream(ws), cur_sk(ws), X2, X1.T(), Wv, 0.5, 0.0));
  BR_CHECK(gemm(cur_stream(ws), cur_sk(ws), X3, Yv, X2, 1.0, 1.0, &X1));
  return syr2k_lower(cur_stream(ws), A2v, X3, Yv, 0, j);
}

static double sevp_nominal(int64_t n) { return 4.0 * (double)n * n * n / 3.0; }
static double svd_nominal(int64_t m, int64_t n) {
  return 4.0 * ((double)m * n * n - (double)n * n * n / 3.0);
}

// Factor output checks: leading dimensions cover the packed layout.
static bool factors_ok(const br_factors* f, int64_t m, int64_t n, int64_t b, bool right) {
  if (!f) return true;
  if (f->yl && f->ldyl < std::max<int64_t>(m, 1)) return false;
  if (f->tl && f->ldtl < b) return false;
  if (right && f->yr && f->ldyr < std::max<int64_t>(n, 1)) return false;
  if (right && f->tr && f->ldtr < b) return false;
  return true;
}

// Sets the handle's per-call state (factor output) for the duration of one
// reduction call.
struct CallState {
  Workspace& ws;
  CallState(Workspace& w, const br_factors* f) : ws(w) {
    ws.fo = (f && (f->yl || f->tl || f->taul || f->yr || f->tr || f->taur)) ? f : nullptr;
  }
  ~CallState() { ws.fo = nullptr; }
};

int br_set_option(br_handle_t h, int key, int64_t value) {
  ARG(h != nullptr, 1);
  ARG(key == BR_OPT_MAX_ITERS, 2);
  ARG(value >= 0, 3);
  h->ws.max_iters = value;
  return 0;
}

int br_reduce_sym_band(br_handle_t h, int64_t n, int64_t w, int64_t b, int lookahead, double* A,
                       int64_t lda, double* Q, int64_t ldq, const br_factors* factors,
                       br_stats* stats) {
  ARG(h != nullptr, 1);
  ARG(n >= 1, 2);
  ARG(w >= 1, 3);
  ARG(b >= 1 && b <= w, 4);
  ARG(lookahead == 0 || lookahead == 1, 5);
  ARG(A != nullptr && lda >= n, 6);
  ARG(Q == nullptr || ldq >= n, 9);
  ARG(factors_ok(factors, n, n, b, false), 10);
  DEV(h);
  CallState cs(h->ws, factors);
  Workspace::GraphKey key;
  key.kind = 0;
  key.n = n;
  key.w = w;
  key.b = b;
  key.la = lookahead;
  key.A = A;
  key.lda = lda;
  key.Q = Q;
  key.ldq = ldq;
  return timed_reduction(h->ws, stats, sevp_nominal(n), key,
                         [&](int64_t* it) {
                           return sevp_reduce(h->ws, n, w, b, lookahead, A, lda, Q, ldq, it,
                                              h->ws.band_out);
                         });
}

int br_reduce_tri_band(br_handle_t h, int64_t m, int64_t n, int64_t w, int64_t b, int lookahead,
                       double* A, int64_t lda, const br_factors* factors, br_stats* stats) {
  ARG(h != nullptr, 1);
  ARG(m >= 1 && m >= n, 2);
  ARG(n >= 1, 3);
  ARG(w >= 1, 4);
  ARG(b >= 1 && b <= w, 5);
  ARG(lookahead == 0 || lookahead == 1, 6);
  ARG(A != nullptr && lda >= m, 7);
  ARG(factors_ok(factors, m, n, b, true), 9);
  DEV(h);
  CallState cs(h->ws, factors);
  Workspace::GraphKey key;
  key.kind = 1;
  key.m = m;
  key.n = n;
  key.w = w;
  key.b = b;
  key.la = lookahead;
  key.A = A;
  key.lda = lda;
  return timed_reduction(h->ws, stats, svd_nominal(m, n), key,
                         [&](int64_t* it) {
                           return tri_reduce(h->ws, m, n, w, b, lookahead, A, lda, it,
                                             h->ws.band_out);
                         });
}

int br_reduce_band(br_handle_t h, int64_t m, int64_t n, int64_t w, int64_t b, int simultaneous,
                   int lookahead, double* A, int64_t lda, const br_factors* factors,
                   br_stats* stats) {
  ARG(h != nullptr, 1);
  ARG(m >= 1 && m >= n, 2);
  ARG(n >= 1, 3);
  ARG(w >= 1, 4);
  ARG(b >= 1 && b <= w, 5);
  ARG(simultaneous == 0 || simultaneous == 1, 6);
  ARG(lookahead == 0 || lookahead == 1, 7);
  ARG(A != nullptr && lda >= m, 8);
  ARG(factors_ok(factors, m, n, b, true), 10);
  DEV(h);
  CallState cs(h->ws, factors);
  Workspace::GraphKey key;
  key.kind = 2;
  key.m = m;
  key.n = n;
  key.w = w;
  key.b = b;
  key.fused = simultaneous;
  key.la = lookahead;
  key.A = A;
  key.lda = lda;
  return timed_reduction(h->ws, stats, svd_nominal(m, n), key,
                         [&](int64_t* it) {
                           return band_reduce(h->ws, m, n, w, b, simultaneous, lookahead, A,
                                              lda, it, h->ws.band_out);
                         });
}

// BR_STREAM_IN=0 turns the streamed input off (A/B aid).
static bool stream_in_enabled() {
  static int m = -1;
  if (m < 0) {
    const char* e = std::getenv("BR_STREAM_IN");
    m = (e && std::atoi(e) == 0) ? 0 : 1;
  }
  return m == 1;
}

// Stream the band out while reducing when the destination is pinned host
// memory and the matrix is large (pageable D2H copies block the host thread).
static bool setup_band_out(Workspace& ws, BandOut& bo, double* band, int64_t ldb, double* dA,
                           int64_t ldd, int64_t m, int64_t n) {
  cudaPointerAttributes pa;
  const bool pinned = cudaPointerGetAttributes(&pa, band) == cudaSuccess &&
                      pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  // streamed output from BR_STREAM_MIN_MB MiB (default 16; 64 until late in
  // round 2): at c1 / c2's 32 MiB the overlapped copy-out is worth more end to
  // end than the graph replay it displaces (e2e c1 1964 -> 2059 GFLOP/s, c2
  // 2676 -> 2789)
  static const int64_t min_mb = [] {
    const char* e = std::getenv("BR_STREAM_MIN_MB");
    return e ? (int64_t)std::atoll(e) : (int64_t)16;
  }();
  if (!pinned || m * n * (int64_t)sizeof(double) < (min_mb << 20)) return false;
  bo.st = ws.copy;
  bo.host = band;
  bo.ldh = ldb;
  bo.A = dA;
  bo.lda = ldd;
  bo.rows = m;
  bo.done = 0;
  ws.band_out = &bo;
  return true;
}

// Host factor output: device staging buffers (zeroed; the packed layout with
// leading dimensions m / b / n) and the copy back into the caller's arrays.
struct FactorStage {
  br_factors dev{};
  const br_factors* host = nullptr;
  int64_t m = 0, n = 0, b = 0;
};
static int factors_stage(Workspace& ws, const br_factors* hf, int64_t m, int64_t n, int64_t b,
                         bool right, FactorStage& fs) {
  fs.host = nullptr;
  if (!hf || !(hf->yl || hf->tl || hf->taul || (right && (hf->yr || hf->tr || hf->taur))))
    return 0;
  fs.host = hf;
  fs.m = m;
  fs.n = n;
  fs.b = b;
  // only the requested members are staged (a tau-only request is n doubles)
  const int64_t ny = hf->yl ? m * n : 0, nt = hf->tl ? b * n : 0, na = hf->taul ? n : 0;
  const int64_t nyr = right && hf->yr ? n * n : 0, ntr = right && hf->tr ? b * n : 0,
                nar = right && hf->taur ? n : 0;
  const int64_t need = ny + nt + na + nyr + ntr + nar;
  BR_CHECK(devbuf_reserve(ws.stageF, need));
  BR_CUDA(cudaMemsetAsync(ws.stageF.p, 0, need * sizeof(double), ws.main));
  double* p = ws.stageF.p;
  br_factors& d = fs.dev;
  d = br_factors{};
  d.yl = ny ? p : nullptr, d.ldyl = m;
  p += ny;
  d.tl = nt ? p : nullptr, d.ldtl = b;
  p += nt;
  d.taul = na ? p : nullptr;
  p += na;
  if (right) {
    d.yr = nyr ? p : nullptr, d.ldyr = n;
    p += nyr;
    d.tr = ntr ? p : nullptr, d.ldtr = b;
    p += ntr;
    d.taur = nar ? p : nullptr;
  }
  return 0;
}
static int factors_unstage(Workspace& ws, const FactorStage& fs) {
  if (!fs.host) return 0;
  const br_factors &h = *fs.host, &d = fs.dev;
  const size_t D = sizeof(double);
  auto mat = [&](double* dst, int64_t ldd, const double* src, int64_t lds, int64_t r, int64_t c) {
    if (!dst || !src) return cudaSuccess;
    return cudaMemcpy2DAsync(dst, ldd * D, src, lds * D, r * D, c, cudaMemcpyDeviceToHost, ws.main);
  };
  BR_CUDA(mat(h.yl, h.ldyl, d.yl, d.ldyl, fs.m, fs.n));
  BR_CUDA(mat(h.tl, h.ldtl, d.tl, d.ldtl, fs.b, fs.n));
  BR_CUDA(mat(h.taul, 1, d.taul, 1, 1, fs.n));
  BR_CUDA(mat(h.yr, h.ldyr, d.yr, d.ldyr, fs.n, fs.n));
  BR_CUDA(mat(h.tr, h.ldtr, d.tr, d.ldtr, fs.b, fs.n));
  BR_CUDA(mat(h.taur, 1, d.taur, 1, 1, fs.n));
  return 0;
}

static int host_stage_in(Workspace& ws, int64_t m, int64_t n, const double* A, int64_t lda,
                         DevBuf& dev, int64_t& ldd) {
  ldd = (m + 31) / 32 * 32;
  BR_CHECK(devbuf_reserve(dev, ldd * n));
  BR_CUDA(cudaMemcpy2DAsync(dev.p, ldd * sizeof(double), A, lda * sizeof(double),
                            m * sizeof(double), n, cudaMemcpyHostToDevice, ws.main));
  return 0;
}

// Bytes the symmetric stage-in copies for an n x n input (br_sym_stage_bytes in
// the header): column blocks of the lower triangle, from each block's first
// row down. The reduction reads the lower triangle only (ref sevp.py reads
// A's lower part; the upper triangle of the device copy is first written by
// the finalize pass), so half of the input never crosses PCIe.
static int64_t sym_stage_block(int64_t n) { return std::max<int64_t>(256, (n / 32 + 31) / 32 * 32); }
static int host_stage_in_lower(Workspace& ws, int64_t n, const double* A, int64_t lda, DevBuf& dev,
                               int64_t& ldd) {
  ldd = (n + 31) / 32 * 32;
  BR_CHECK(devbuf_reserve(dev, ldd * n));
  const int64_t blk = sym_stage_block(n);
  for (int64_t c0 = 0; c0 < n; c0 += blk) {
    const int64_t nc = std::min(blk, n - c0);
    BR_CUDA(cudaMemcpy2DAsync(dev.p + c0 + c0 * ldd, ldd * sizeof(double), A + c0 + c0 * lda,
                              lda * sizeof(double), (n - c0) * sizeof(double), nc,
                              cudaMemcpyHostToDevice, ws.main));
  }
  return 0;
}
extern "C" int64_t br_sym_stage_bytes(int64_t n) {
  int64_t bytes = 0;
  const int64_t blk = sym_stage_block(n);
  for (int64_t c0 = 0; c0 < n; c0 += blk) bytes += (n - c0) * std::min(blk, n - c0) * (int64_t)sizeof(double);
  return bytes;
}

int br_reduce_sym_band_host(br_handle_t h, int64_t n, int64_t w, int64_t b, int lookahead,
                            const double* A, int64_t lda, double* band, int64_t ldb, double* Q,
                            int64_t ldq, const br_factors* factors, br_stats* stats) {
  ARG(h != nullptr, 1);
  ARG(n >= 1, 2);
  ARG(w >= 1, 3);
  ARG(b >= 1 && b <= w, 4);
  ARG(A != nullptr && lda >= n, 6);
  ARG(band != nullptr && ldb >= n, 8);
  ARG(Q == nullptr || ldq >= n, 11);
  ARG(factors_ok(factors, n, n, b, false), 12);
  DEV(h);
  FactorStage fs;
  BR_CHECK(factors_stage(h->ws, factors, n, n, b, false, fs));
  Workspace& ws = h->ws;
  DevBuf& dA = ws.stageA;
  DevBuf& dQ = ws.stageQ;
  int64_t ldd = 0;
  // the unchanged-input case (n <= w + 1) and partial runs hand the raw matrix back
  if (n <= w + 1 || ws.max_iters > 0) BR_CHECK(host_stage_in(ws, n, n, A, lda, dA, ldd));
  else BR_CHECK(host_stage_in_lower(ws, n, A, lda, dA, ldd));
  double* qd = nullptr;
  if (Q) {
    BR_CHECK(devbuf_reserve(dQ, ldd * n));
    qd = dQ.p;
  }
  BandOut bo;
  bo.sym = true;
  bo.w = w;
  const bool streamed = setup_band_out(ws, bo, band, ldb, dA.p, ldd, n, n);
  const int rc = br_reduce_sym_band(h, n, w, b, lookahead, dA.p, ldd, qd, ldd,
                                    fs.host ? &fs.dev : nullptr, stats);
  ws.band_out = nullptr;
  if (streamed) BR_CUDA(cudaStreamSynchronize(ws.copy));
  BR_CHECK(rc);
  BR_CHECK(factors_unstage(ws, fs));
  if (!streamed)
    BR_CUDA(cudaMemcpy2DAsync(band, ldb * sizeof(double), dA.p, ldd * sizeof(double),
                              n * sizeof(double), n, cudaMemcpyDeviceToHost, ws.main));
  if (Q)
    BR_CUDA(cudaMemcpy2DAsync(Q, ldq * sizeof(double), dQ.p, ldd * sizeof(double),
                              n * sizeof(double), n, cudaMemcpyDeviceToHost, ws.main));
  BR_CUDA(cudaStreamSynchronize(ws.main));
  return 0;
}

int br_reduce_tri_band_host(br_handle_t h, int64_t m, int64_t n, int64_t w, int64_t b,
                            int lookahead, const double* A, int64_t lda, double* band,
                            int64_t ldb, const br_factors* factors, br_stats* stats) {
  ARG(h != nullptr, 1);
  ARG(m >= 1 && m >= n, 2);
  ARG(n >= 1, 3);
  ARG(w >= 1, 4);
  ARG(b >= 1 && b <= w, 5);
  ARG(A != nullptr && lda >= m, 7);
  ARG(band != nullptr && ldb >= m, 9);
  ARG(factors_ok(factors, m, n, b, true), 10);
  DEV(h);
  FactorStage fs;
  BR_CHECK(factors_stage(h->ws, factors, m, n, b, true, fs));
  Workspace& ws = h->ws;
  DevBuf& dA = ws.stageA;
  int64_t ldd = 0;
  // pinned, large input: stream it in by column chunks while the first
  // iteration's panel and left update start on the columns already there
  cudaPointerAttributes pa;
  const bool pinned_in = cudaPointerGetAttributes(&pa, A) == cudaSuccess &&
                         pa.type == cudaMemoryTypeHost && stream_in_enabled();
  cudaGetLastError();
  BandIn bi;
  static const int64_t in_min_mb = [] {  // BR_STREAM_IN_MIN_MB (default 64)
    const char* e = std::getenv("BR_STREAM_IN_MIN_MB");
    return e ? (int64_t)std::atoll(e) : (int64_t)64;
  }();
  const bool stream_in = pinned_in && m * n * (int64_t)sizeof(double) >= (in_min_mb << 20);
  if (stream_in) {
    ldd = (m + 31) / 32 * 32;
    BR_CHECK(devbuf_reserve(dA, ldd * n));
    bi.host = A;
    bi.ldh = lda;
    bi.A = dA.p;
    bi.lda = ldd;
    bi.rows = m;
    bi.cols = n;
    bi.chunk = std::max<int64_t>(b, cdiv(std::max<int64_t>(n / 16, 1), b) * b);
    bi.nchunks = (int)cdiv(n, bi.chunk);
    if (bi.nchunks > 256) {
      bi.chunk = cdiv(cdiv(n, 256), b) * b;
      bi.nchunks = (int)cdiv(n, bi.chunk);
    }
    ws.band_in = &bi;
  } else {
    BR_CHECK(host_stage_in(ws, m, n, A, lda, dA, ldd));
  }
  BandOut bo;
  bo.lo = 0;
  bo.up = w;
  const bool streamed = setup_band_out(ws, bo, band, ldb, dA.p, ldd, m, n);
  const int rc = br_reduce_tri_band(h, m, n, w, b, lookahead, dA.p, ldd,
                                    fs.host ? &fs.dev : nullptr, stats);
  ws.band_out = nullptr;
  ws.band_in = nullptr;
  if (stream_in) BR_CUDA(cudaStreamSynchronize(ws.copy_in));
  if (streamed) BR_CUDA(cudaStreamSynchronize(ws.copy));
  BR_CHECK(rc);
  BR_CHECK(factors_unstage(ws, fs));
  if (!streamed)
    BR_CUDA(cudaMemcpy2DAsync(band, ldb * sizeof(double), dA.p, ldd * sizeof(double),
                              m * sizeof(double), n, cudaMemcpyDeviceToHost, ws.main));
  BR_CUDA(cudaStreamSynchronize(ws.main));
  return 0;
}

int br_reduce_band_host(br_handle_t h, int64_t m, int64_t n, int64_t w, int64_t b,
                        int simultaneous, int lookahead, const double* A, int64_t lda,
                        double* band, int64_t ldb, const br_factors* factors, br_stats* stats) {
  ARG(h != nullptr, 1);
  ARG(m >= 1 && m >= n, 2);
  ARG(n >= 1, 3);
  ARG(w >= 1, 4);
  ARG(b >= 1 && b <= w, 5);
  ARG(A != nullptr && lda >= m, 8);
  ARG(band != nullptr && ldb >= m, 10);
  ARG(factors_ok(factors, m, n, b, true), 11);
  DEV(h);
  FactorStage fs;
  BR_CHECK(factors_stage(h->ws, factors, m, n, b, true, fs));
  Workspace& ws = h->ws;
  DevBuf& dA = ws.stageA;
  int64_t ldd = 0;
  BR_CHECK(host_stage_in(ws, m, n, A, lda, dA, ldd));
  BandOut bo;
  bo.lo = w;
  bo.up = w;
  const bool streamed = setup_band_out(ws, bo, band, ldb, dA.p, ldd, m, n);
  const int rc = br_reduce_band(h, m, n, w, b, simultaneous, lookahead, dA.p, ldd,
                                fs.host ? &fs.dev : nullptr, stats);
  ws.band_out = nullptr;
  if (streamed) BR_CUDA(cudaStreamSynchronize(ws.copy));
  BR_CHECK(rc);
  BR_CHECK(factors_unstage(ws, fs));
  if (!streamed)
    BR_CUDA(cudaMemcpy2DAsync(band, ldb * sizeof(double), dA.p, ldd * sizeof(double),
                              m * sizeof(double), n, cudaMemcpyDeviceToHost, ws.main));
  BR_CUDA(cudaStreamSynchronize(ws.main));
  return 0;
}

}  // extern "C"
