/*
 * bandred_b200 — C ABI of the B200-native (sm_100a) first-stage band
 * reduction: dense symmetric -> symmetric band (SEVP) and dense general ->
 * upper triangular-band (SVD), arXiv 1709.00302, with static look-ahead.
 *
 * Every entry point replaces one function of the reference package
 * `bandred` (paths relative to the reference's pkg/src/bandred/); the
 * reference-side binding a maintainer would add is in INTEGRATION.md.
 *
 * Conventions (all functions):
 *   - fp64, column-major, leading dimensions in elements, sizes int64_t;
 *   - device pointers unless the name ends in _host;
 *   - work is enqueued on the handle's streams; kernel-level calls run on
 *     the handle's main stream and are asynchronous (call br_sync), the
 *     reductions return after the device work completed;
 *   - return 0 on success, -i when argument i is invalid (LAPACK style,
 *     Python raises ValueError), >0 on a CUDA/NCCL failure (RuntimeError);
 *     br_last_error() gives the message. No exception crosses the ABI.
 *   - Reflector conventions follow the reference exactly: beta =
 *     -sign(x0)*||x|| with x0 == 0 counted positive, tau = 2 for a zero
 *     tail, tau = beta = 0 for a zero vector; Q = I + W*Y^T with W = Y*T
 *     (T = -T_larft).
 */
#ifndef BANDRED_B200_H
#define BANDRED_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct br_handle_s* br_handle_t;

/* Statistics filled by the reductions (nullable). */
typedef struct br_stats {
  int64_t iterations;   /* panels factored (ref SevpResult/SvdResult.iterations) */
  double device_ms;     /* device time of the reduction proper (CUDA events) */
  double nominal_flops; /* 4n^3/3 (SEVP) or 4(mn^2 - n^3/3) (SVD) */
  int64_t launches;     /* kernels launched by the reduction */
} br_stats;

/* Householder factors of a reduction (extension: the reference keeps them
 * only in private state, ref sevp.py:106,128-134 state.factors[k] and
 * svd.py:185,195 fu/fv; SURVEY 8(b) `return_factors` / `factors_out`).
 * Every panel's compact-WY factors Q_k = I + W_k Y_k^T, W_k = Y_k T_k
 * (T = -T_larft), are stored packed, panel by panel, like LAPACK's
 * sytrd_sy2sb / gebrd keep their reflectors below/right of the band:
 *   left chain (QR panels: SEVP, the SVD's U side), panel at leading column k
 *   with bp columns and j rows starting at row r0 (SEVP and band form
 *   r0 = k + w, triangular band r0 = k):
 *     Y_k  -> yl[r0 + r + (k + c) * ldyl], r < j, c < bp (unit lower
 *             trapezoidal, explicit zeros above the unit diagonal)
 *     T_k  -> tl[r + (k + c) * ldtl],       r, c < bp (upper triangular)
 *     tau  -> taul[k + c]
 *   right chain (LQ panels, SVD only, ignored for SEVP), panel at leading
 *   column k with bq reflectors acting on columns k + w .. n:
 *     Y_k  -> yr[(k + w) + r + (k + c) * ldyr], r < n - k - w, c < bq
 *     T_k  -> tr[r + (k + c) * ldtr];  tau -> taur[k + c]
 * Sizes: yl m x n (SEVP n x n), tl b x n, taul n, yr n x n, tr b x n, taur
 * n. Entries outside the panels are not written. The reduced matrix A then
 * equals Q_L B Q_R^T with Q_L = Q_0 Q_1 ... (left chain) and Q_R likewise
 * (SEVP: A = Q B Q^T). Device pointers for the device entry points, host
 * pointers for the _host ones. Any chain pointer may be NULL (not stored). */
typedef struct br_factors {
  double* yl;
  int64_t ldyl;
  double* tl;
  int64_t ldtl;
  double* taul;
  double* yr;
  int64_t ldyr;
  double* tr;
  int64_t ldtr;
  double* taur;
} br_factors;

/* ---- context ---------------------------------------------------------- */
int br_version(void);
const char* br_last_error(void);
/* Kernels this library has launched in this process (bench evidence). */
int64_t br_launch_count(void);
/* Create a context on `device` with its own main/panel streams (the panel
 * stream has the higher priority: look-ahead factorizations win SMs). */
int br_create(int device, br_handle_t* out);
int br_destroy(br_handle_t h);
/* Use caller-owned streams (cudaStream_t passed as void*); NULL keeps the
 * handle's own. */
int br_set_streams(br_handle_t h, void* main_stream, void* panel_stream);
int br_sync(br_handle_t h);
/* Per-kernel-class CUDA-event timing of subsequent reductions (bench).
 * enable: 0 off, 1 per-class totals, 2 totals + per-task event trace. */
int br_set_timing(br_handle_t h, int enable);
/* Class: 0 = panel, 1 = symm, 2 = syr2k, 3 = gemm (other updates).
 * Accumulated since br_set_timing(h, 1 or 2). */
int br_get_timing(br_handle_t h, int cls, double* ms, double* flops, int64_t* launches);
/* Event trace of the last reduction run with br_set_timing(h, 2): one record
 * per task ("qr@k", "lq@k", "left@k", "trail@k", ...; the task ids of the
 * reference's EventTrace, ref runtime.py:76-104), its stream (0 = main, the
 * T_P group; 1 = panel, the T_S group) and its device start/end time in
 * microseconds since the call began. Overlap of the two streams is the
 * look-ahead. br_trace_count returns the record count (-1 for a NULL h). */
int64_t br_trace_count(br_handle_t h);
/* Handle options (extension). BR_OPT_MAX_ITERS = k > 0: the reductions stop
 * after their first k panels and return the raw working matrix (no
 * finalize / band mask; the panels' own columns below the band hold R/L and
 * scratch) - a partial reduction used to compare the trailing matrix with
 * the reference after k iterations at sizes where a full CPU reference run
 * is too slow; 0 (default) = full reduction. */
#define BR_OPT_MAX_ITERS 1
int br_set_option(br_handle_t h, int key, int64_t value);
int br_trace_get(br_handle_t h, int64_t idx, char* id, int64_t idlen, int* stream, double* t0_us,
                 double* t1_us);

/* Kernel-level calls below run on the main stream (which = 0, default) or the
 * panel stream (which = 1) - the two worker groups of the reference runtime
 * (runtime.py:142-180). br_stream_join(h, w) makes stream w wait for all work
 * enqueued so far on the other one. */
int br_stream_select(br_handle_t h, int which);
int br_stream_join(br_handle_t h, int waiter);

/* ---- kernel level (ref kernels.py) ------------------------------------ */
/* matmul (kernels.py:39-83): C = alpha op(A) op(B) + beta C on the FP64
 * tensor cores (fixed K order per element, deterministic). */
int br_gemm(br_handle_t h, int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha,
            const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
            int64_t ldc);
/* symm_lower with scaling: X1 = alpha sym(A2) W + beta X1, A2 lower-only. */
int br_symm_lower_ex(br_handle_t h, int64_t j, int64_t b, double alpha, const double* A2,
                     int64_t lda, const double* W, int64_t ldw, double beta, double* X1,
                     int64_t ldx);
/* house_gen (kernels.py:86-110): v (L) and tau_beta = {tau, beta}. */
int br_house_gen(br_handle_t h, int64_t L, const double* x, double* v, double* tau_beta);
/* qr_panel (kernels.py:165-208): in-place QR of the j x b panel P; R into
 * P's top triangle; Y (j x b), T (b x b), W (j x b, nullable), tau (b). */
int br_qr_panel(br_handle_t h, int64_t j, int64_t b, double* P, int64_t ldp, double* Y,
                int64_t ldy, double* T, int64_t ldt, double* W, int64_t ldw, double* tau);
/* lq_panel (kernels.py:211-255): in-place LQ of the b x j panel P; L into
 * P's left triangle; Y (j x b), T, W, tau as for QR. */
int br_lq_panel(br_handle_t h, int64_t b, int64_t j, double* P, int64_t ldp, double* Y,
                int64_t ldy, double* T, int64_t ldt, double* W, int64_t ldw, double* tau);
/* build_w (kernels.py:139-149): W = Y T. */
int br_build_w(br_handle_t h, int64_t j, int64_t b, const double* Y, int64_t ldy,
               const double* T, int64_t ldt, double* W, int64_t ldw);
/* apply_wy_left (kernels.py:258-284): A (rows x cols) += Y (W^T A). */
int br_apply_wy_left(br_handle_t h, int64_t rows, int64_t cols, double* A, int64_t lda,
                     const double* Y, int64_t ldy, const double* W, int64_t ldw, int64_t b);
/* apply_wy_right (kernels.py:287-309): A (rows x cols) += (A W) Y^T. */
int br_apply_wy_right(br_handle_t h, int64_t rows, int64_t cols, double* A, int64_t lda,
                      const double* Y, int64_t ldy, const double* W, int64_t ldw, int64_t b);
/* symm_lower (kernels.py:312-341): X1 = sym(A2) W, A2 lower-only. */
int br_symm_lower(br_handle_t h, int64_t j, int64_t b, const double* A2, int64_t lda,
                  const double* W, int64_t ldw, double* X1, int64_t ldx);
/* syr2k_lower (kernels.py:344-378): A2[:, c0:c1] += X3 Y^T + Y X3^T, lower. */
int br_syr2k_lower(br_handle_t h, int64_t j, int64_t b, double* A2, int64_t lda,
                   const double* X3, int64_t ldx, const double* Y, int64_t ldy, int64_t c0,
                   int64_t c1);
/* Distributed SEVP (SURVEY 8(e), 1D block-cyclic columns; the multi-rank
 * form of symm_lower / syr2k_lower, kernels.py:312-378). L is one rank's
 * owned trailing block columns as a j x ncols slab: local column c is column
 * r0 + (c / bs) * stride + c % bs of the j x j trailing matrix A2 (stride =
 * world * bs), stored from that row down with ZEROS above (the rank keeps
 * its strict upper triangle zero). */
/* Rows [p0, p1) of this slab's share of X1 = sym(A2) W into X1 ((p1 - p0) x
 * b, overwritten): the sum over the ranks' slabs (an all-reduce) is
 * sym(A2) W. The range must not split an owned block (chunked all-reduce:
 * compute a row chunk, reduce it while the next chunk computes). */
int br_symm_lower_cyclic(br_handle_t h, int64_t j, int64_t ncols, int64_t b, const double* L,
                         int64_t ldl, const double* W, int64_t ldw, double* X1, int64_t ldx,
                         int64_t r0, int64_t bs, int64_t stride, int64_t p0, int64_t p1);
/* L += X3 Y^T + Y X3^T at the slab's columns, lower triangle of A2 only. */
int br_syr2k_lower_cyclic(br_handle_t h, int64_t j, int64_t ncols, int64_t b, double* L,
                          int64_t ldl, const double* X3, int64_t ldx, const double* Y, int64_t ldy,
                          int64_t r0, int64_t bs, int64_t stride);
/* sym_two_sided_update (kernels.py:381-401): A2 := Q^T A2 Q, lower only. */
int br_sym_two_sided_update(br_handle_t h, int64_t j, int64_t b, double* A2, int64_t lda,
                            const double* Y, int64_t ldy, const double* W, int64_t ldw);

/* ---- second stage (beyond the reference, which stops at
 * the band) ------------------------------------------------------ */
/* Symmetric band (bandwidth w <= 128, lower triangle of the n x n device
 * matrix A) -> symmetric tridiagonal by Householder bulge chasing, in place;
 * d (n) = diagonal, e (n - 1) = subdiagonal (device). The eigenvalues are
 * those of the band. */
int br_band_to_tridiag(br_handle_t h, int64_t n, int64_t w, double* A, int64_t lda, double* d,
                       double* e);
/* Upper triangular band (bandwidth w <= 128; m x n device matrix, m >= n,
 * rows >= n zero) -> upper bidiagonal, in place; d (n), e (n - 1) =
 * superdiagonal. The singular values are those of the band. */
int br_band_to_bidiag(br_handle_t h, int64_t m, int64_t n, int64_t w, double* A, int64_t lda,
                      double* d, double* e);

/* ---- reductions --------------------------------------------------------- */
/* Every reduction takes `factors` (nullable, see br_factors): when given,
 * each panel's Y, T and tau are stored there as the panel is factored. */
/* reduce_sym_band (sevp.py:287-324) on a device matrix, in place. Reads
 * only the lower triangle; on return A holds the finalized band (mirrored,
 * off-band exactly zero). lookahead: 0 = reference schedule, 1 = next panel
 * factored on the panel stream while the trailing update finishes (V1/V2).
 * Q (nullable, n x n) receives the accumulated orthogonal factor
 * (accumulate_q, sevp.py:138-144). If n <= w+1 nothing is done. */
int br_reduce_sym_band(br_handle_t h, int64_t n, int64_t w, int64_t b, int lookahead, double* A,
                       int64_t lda, double* Q, int64_t ldq, const br_factors* factors,
                       br_stats* stats);
/* reduce_tri_band (svd.py:179-247) on a device m x n matrix, m >= n, in
 * place: upper triangular-band with bandwidth w, everything else exactly 0.
 * lookahead 1 overlaps the LQ / next QR panels with the rank-b updates
 * (extension: the reference schedule is sequential, results identical). */
int br_reduce_tri_band(br_handle_t h, int64_t m, int64_t n, int64_t w, int64_t b, int lookahead,
                       double* A, int64_t lda, const br_factors* factors, br_stats* stats);
/* Host-buffer variants: copy A (host, lda) to the device, reduce, copy the
 * band back to `band` (host, ldb). Host buffers may be pageable or pinned.
 * Pinned buffers of 16 MiB and more are streamed: finished band column
 * blocks are copied out while the reduction runs, and (triangular band) the
 * input is copied in by column chunks while iteration 0's panel and left
 * update start on the chunks already there. Results are bitwise those of
 * the staged copies. */
int br_reduce_sym_band_host(br_handle_t h, int64_t n, int64_t w, int64_t b, int lookahead,
                            const double* A, int64_t lda, double* band, int64_t ldb, double* Q,
                            int64_t ldq, const br_factors* factors, br_stats* stats);
int br_reduce_tri_band_host(br_handle_t h, int64_t m, int64_t n, int64_t w, int64_t b,
                            int lookahead, const double* A, int64_t lda, double* band,
                            int64_t ldb, const br_factors* factors, br_stats* stats);
/* Bytes br_reduce_sym_band_host copies to the device for an n x n input with
 * n > w + 1: the reduction reads the lower triangle only (as the reference
 * does, sevp.py:287-324 / kernels.py:312-341), so the stage-in copies the
 * lower triangle by column blocks and the upper triangle of A is never
 * touched. */
int64_t br_sym_stage_bytes(int64_t n);

/* Equal-bandwidth band form of the SVD (replaces the band branch of
 * reduce_band_svd, ref pkg/src/bandred/svd.py:515-589, task bodies
 * svd.py:250-391). Column-major device A (m x n, m >= n, lda >= m) is
 * reduced in place to band form: A[i,j] = 0 exactly for |i-j| > w; m <= w+1
 * returns A unchanged. simultaneous 0 = reference order (left then right
 * update of the trailing block, SvdVariant.REFERENCE / V1), 1 = fused
 * two-sided trailing update (SvdVariant.SIMULTANEOUS / V2). lookahead 1 =
 * static look-ahead (V1 / V2 schedules, svd.py:394-492): bitwise equal to
 * lookahead 0 with the same `simultaneous`. Needs 1 <= b <= w. */
int br_reduce_band(br_handle_t h, int64_t m, int64_t n, int64_t w, int64_t b, int simultaneous,
                   int lookahead, double* A, int64_t lda, const br_factors* factors,
                   br_stats* stats);
int br_reduce_band_host(br_handle_t h, int64_t m, int64_t n, int64_t w, int64_t b,
                        int simultaneous, int lookahead, const double* A, int64_t lda,
                        double* band, int64_t ldb, const br_factors* factors, br_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* BANDRED_B200_H */
