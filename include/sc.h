/* sc.h — C ABI of libsc, the B200 (sm_100a) software-context evaluator.
 *
 * What it computes (ChameleonAPI drafts bundled in arXiv 2310.07240; PAPER.md
 * under /root/reference, see SURVEY.md §0 and DESIGN.md):
 *   an application turns a multi-label API output into a decision,
 *   z = Decision(API(x)), by walking the output labels in
 *   descending confidence and returning the branch of the first
 *   label found in one of its lists, checked in code order (the Heapsortcypher
 *   listing).  For a batch of B inputs with logits [B, C] and
 *   ground-truth label sets ŷ_i, libsc produces in one read of the logits:
 *     - the decision of every input,
 *     - the incorrect-decision count of Eq. goal,
 *     - the histogram of ground-truth category masks G_i used for the
 *       rebalancing weights M/N_i and the histogram of
 *       predicted decisions,
 *     - the forward and backward of the Multi-Choice API-output-order loss,
 *       Eq. api_output, weighted by M/N_i.
 *
 * Notation.  D' = number of lists of an application (0..8); decision ids
 * 0..D'-1 are the lists in code order and D' is the default (no label matched,
 * reading A6).  cat[c] = first list containing label c (reading A5).  G_i =
 * bit set of the lists the ground truth of input i intersects;
 * y_i = [G_i != 0].  tau = threshold on logits: label c is an
 * API output iff z_c > tau (reading A3); theta = sigma(tau).
 *
 * Conventions for every call below.
 *   - Device pointers are caller-owned and must stay valid until the work
 *     enqueued on `stream` completes.  Calls are stream-ordered and
 *     asynchronous; hot calls never allocate and never synchronise.
 *   - Every uint64_t / double output ACCUMULATES (+=): zero it once, then the
 *     batch may be split into chunks, shards or resumed passes.  Per-row
 *     outputs are overwritten.  Any output pointer may be NULL (= not wanted).
 *   - Host-side validation failures return SC_ERR_INVALID_ARG before anything
 *     is enqueued; CUDA launch failures return SC_ERR_CUDA.  sc_last_error()
 *     gives a thread-local message for the last non-OK status.  No call aborts
 *     or exits; no C++ exception crosses the ABI.
 *   - Device-side preconditions (finite logits, GT ids in [0,C), app ids <
 *     n_apps) are not checked on the device: violating them gives unspecified
 *     (but memory-safe within the documented buffers) results.
 */
#ifndef SC_H
#define SC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SC_OK = 0,
  SC_ERR_INVALID_ARG = 1,
  SC_ERR_OOM = 2,
  SC_ERR_CUDA = 3,
  SC_ERR_UNSUPPORTED = 4
} sc_status;

typedef enum { SC_F32 = 0, SC_BF16 = 1 } sc_dtype;

/* The application's decision pattern ("type of decision" and examination order of the
 * extracted summary).  A True-False application is any
 * of them with a single list: all three reduce to Eq. loss there. */
typedef enum {
  SC_ORDER_API_OUTPUT = 0,  /* Multi-Choice, API-output order: the hot path      */
  SC_ORDER_APP_CHOICE = 1,  /* Multi-Choice, application-choice order            */
  SC_ORDER_MULTI_SELECT = 2 /* Multi-Select: decision = mask of selected lists   */
} sc_order;

/* cudaStream_t without pulling in CUDA headers: pass a cudaStream_t (or 0). */
typedef void* sc_stream;

typedef struct sc_context_s* sc_context; /* library-owned; immutable after load */

/* sc_context_load — upload the applications' extracted software contexts
 * ("summary of the software decision process": target classes, decision type,
 * examination order) once, before any batch.
 *   C            number of API labels, 1 <= C < 2^23.
 *   n_apps       number of applications, 1..65535; batch rows pick one via sc_batch.app.
 *   n_lists      host [n_apps]: D'_a, the number of lists of app a, 0..8.
 *   list_off     host: for each app, n_lists[a]+1 offsets into list_labels,
 *                concatenated app after app (list j of app a is
 *                list_labels[list_off[b+j] .. list_off[b+j+1]), b = sum_{a'<a}(n_lists[a']+1)).
 *   list_labels  host: label ids in [0, C), lists in code order.  A label may
 *                appear in several lists; it belongs to the first (reading A5).
 *   tau          logit threshold (finite); theta = sigma(tau) is computed in double.
 *   k            steepness of S(x) = 1/(1+e^{-kx}), finite, > 0.
 *   order        decision pattern (sc_order).  For the two Multi-Choice orders a label in
 *                several lists belongs to the first (the if-chain returns, reading A5); for
 *                Multi-Select it belongs to every list containing it (all are acted on).
 *   out          receives the handle.
 * The host arrays are copied; the context allocates its device tables on the
 * current CUDA device (synchronously) and is usable from any stream/thread on it.
 * Errors: SC_ERR_INVALID_ARG (bad sizes, ids, tau, k), SC_ERR_UNSUPPORTED,
 * SC_ERR_OOM (device allocation), SC_ERR_CUDA. */
sc_status sc_context_load(int32_t C, int32_t n_apps, const int32_t* n_lists, const int64_t* list_off,
                          const int32_t* list_labels, float tau, float k, sc_order order,
                          sc_context* out);

/* sc_context_load_compact — the same context for COLUMN-COMPACTED logit rows (SURVEY.md
 * §8(f)3, sparse contexts such as the OpenImages-shaped one: "applications
 * heavily cluster on a small subset of labels").  Unmapped labels never affect a decision,
 * a count or the loss, and their gradient is exactly 0 (Eq. api_output), so a
 * producer that emits only the mapped columns (e.g. a classifier head restricted to those
 * rows of W) hands over everything the path needs.  Batch rows then hold n_cols columns:
 * column j is the logit of label cols[j], the union of the applications' mapped labels in
 * ascending order (sc_context_columns); sc_batch.ld >= n_cols.  Ground truth (gt_off/gt_lab)
 * stays in label ids [0, C).  Decisions, counters, loss and sparse gradient indices (label
 * ids) are those of sc_context_load on the dense rows; grad_dense is laid out like the
 * compacted rows.  Not accepted by sc_decide_all_apps (dense rows only). */
sc_status sc_context_load_compact(int32_t C, int32_t n_apps, const int32_t* n_lists, const int64_t* list_off,
                                  const int32_t* list_labels, float tau, float k, sc_order order,
                                  sc_context* out);

/* sc_context_columns — the logit columns a batch row of this context holds: *n_cols (C for
 * a dense context) and, if cols != NULL (host [n_cols]), the label of each column. */
sc_status sc_context_columns(sc_context ctx, int32_t* cols, int32_t* n_cols);

/* sc_context_free — release the context's device tables (synchronises the device). NULL is a no-op. */
sc_status sc_context_free(sc_context ctx);

/* sc_context_info — D'_a of app a (n_lists), and the number of mapped labels |𝕎_a|. */
sc_status sc_context_info(sc_context ctx, int32_t app, int32_t* n_lists, int32_t* n_mapped);

/* sc_context_order — the context's pattern and S, the sparse-gradient slots per row
 * (2 for the Multi-Choice orders, 8 for Multi-Select: one per list). */
sc_status sc_context_order(sc_context ctx, sc_order* order, int32_t* grad_slots);

/* A batch of inputs (rows).  All pointers are device pointers.
 *   logits   [rows, ld] row-major, dtype elements; base 16-B aligned and
 *            ld*sizeof(elt) % 16 == 0; ld >= C; columns C..ld-1 are never read
 *            as values (they may hold anything).  May be NULL only for sc_decision_hist.
 *   gt_off   [rows+1] int64 CSR offsets into gt_lab (any base, non-decreasing) —
 *   gt_lab   ... the ground-truth label ids ŷ_i of row i, in [0,C), duplicates allowed.
 *   gt_mask  [rows] uint8, optional: the precomputed G_i of each row, as written by
 *            sc_decision_hist.  When non-NULL it replaces gt_off/gt_lab.  Any alignment;
 *            only bytes of rows [0, rows) are read.
 *   app      [rows] uint16 application ids < n_apps, or NULL (every row is app 0);
 *            2-B aligned; only rows [0, rows) are read.
 * A batch "has GT" iff gt_mask != NULL or gt_off != NULL. */
typedef struct {
  const void*     logits;
  sc_dtype        dtype;
  int64_t         rows;
  int64_t         ld;
  const int64_t*  gt_off;
  const int32_t*  gt_lab;
  const uint8_t*  gt_mask;
  const uint16_t* app;
} sc_batch;

/* sc_decide — decisions and counters, no loss.
 *   decision     [rows] uint8: API-output / application-choice order: 0..D'-1 or D'
 *                (default); Multi-Select: the mask of selected lists.
 *   n_incorrect  [n_apps] += #{i : decision_i ≠ Decision(ŷ_i)} (Eq. goal).  API-output
 *                order: Decision(ŷ) is set-valued (reading A7); application-choice order:
 *                the lowest list ŷ hits; Multi-Select: the mask of lists
 *                ŷ hits (exact match).  Needs GT.
 *   hist_pred    [n_apps*256] += #{i : decision_i = d} at [app*256 + d] (a Multi-Select
 *                decision is a list mask, hence 256 bins).
 *   hist_gt      [n_apps*256] += #{i : G_i = m} at [app*256 + m].  Needs GT. */
sc_status sc_decide(sc_context ctx, const sc_batch* batch, uint8_t* decision, uint64_t* n_incorrect,
                    uint64_t* hist_pred, uint64_t* hist_gt, sc_stream stream);

/* sc_decision_hist — ground-truth-only pre-pass (reads ~18 B/row, never the logits):
 *   hist_gt      [n_apps*256] += mask histogram H (the per-class
 *                marginals are h[d] = sum_{m ∋ d} H[m], h[default] = H[0]).
 *   gt_mask_out  [rows] uint8, optional: G_i per row, for sc_batch.gt_mask.
 * batch->logits is ignored; batch needs gt_off/gt_lab. */
sc_status sc_decision_hist(sc_context ctx, const sc_batch* batch, uint64_t* hist_gt, uint8_t* gt_mask_out,
                           sc_stream stream);

/* sc_decision_hist_weights — sc_decision_hist followed, in the same launch, by
 * sc_weights_from_hist on the histogram it produced (the last CTA to finish computes
 * w).  For a batch that is the whole dataset (one GPU): hist_gt must be zero on entry.
 * Safe across streams and host threads: the context keeps one completion counter per
 * stream that has called it (64 preallocated; beyond that the call falls back to two
 * launches, hist then weights, with identical results).  rows == 0: only w is computed.
 *   w  device [n_apps*256] float, overwritten. */
sc_status sc_decision_hist_weights(sc_context ctx, const sc_batch* batch, uint64_t* hist_gt, uint8_t* gt_mask_out,
                                   float* w, sc_stream stream);

/* sc_weights_from_hist — rebalancing weights from the GLOBAL mask histogram
 * (PAPER.md:2014, :2020, :2029): per app, M = sum_m H[m]; N(m) = #inputs whose
 * ground truth intersects m's lists = M - sum_{m' ∩ m = ∅} H[m'] for m != 0,
 * N(0) = H[0] (non-target inputs); w[m] = M/N(m) in double rounded to float,
 * 0 when N(m) = 0 (reading A13).
 *   hist_gt  device [n_apps*256] uint64 (all ranks' counts, e.g. after an allreduce)
 *   w        device [n_apps*256] float, overwritten. */
sc_status sc_weights_from_hist(sc_context ctx, const uint64_t* hist_gt, float* w, sc_stream stream);

/* sc_loss_fwd_bwd — the fused hot path: one read of each logit row gives the
 * decision, the counters, and the pattern's decision-aware loss with its gradient.
 * API-output order, Eq. api_output:
 *   L_i = w[G_i] ( y_i S(max(P⁻,θ) − P⁺) + (1−y_i) S(P⁻ − θ) ),
 *   P⁺ = σ(max_{c: cat[c] ∈ G_i} z_c), P⁻ = σ(max_{c ∈ 𝕎, cat[c] ∉ G_i} z_c), max ∅ = −∞.
 * Application-choice order, Eq. app_choice, k = lowest list in G_i:
 *   L_i = w[G_i] ( y_i S(max(θ, P_{k⁻}) − P_k) + (1−y_i) S(P − θ) ),
 *   P_k over list k, P_{k⁻} over lists j < k (reading A21), P over 𝕎.
 * Multi-Select, Eq. multi-select, y_ij = bit j of G_i:
 *   L_i = w[G_i] Σ_j ( y_ij S(θ − P_j) + (1 − y_ij) S(P_j − θ) ).
 * The arg maxima are exact (ties to the smaller label id, A8); a competitor inside
 * max(·, θ) gets gradient only when its logit is > tau (A10).
 *   w           device [n_apps*256] float (from sc_weights_from_hist) or NULL (all 1).
 *   grad_scale  multiplies every gradient entry (e.g. 1/B_global, reading A14).
 *   loss_sum    [n_apps] double += sum_i L_i (unscaled).
 *   loss_row    [rows] float, L_i.
 *   grad_idx    [rows*S] int32: S = sc_context_order's grad_slots.  Multi-Choice:
 *   grad_val    [rows*S] float   slot 0 = the label the loss pushes up (c⁺ / the arg max
 *                                of list k), slot 1 = the competitor (c⁻ / of lists < k,
 *                                or of 𝕎 when y_i = 0); Multi-Select: slot j = the arg
 *                                max of list j.  -1 / 0.0f when absent; every other
 *                                dL_i/dz_c is exactly 0.
 *   grad_dense  [rows*ld] float: the full gradient (zeros + at most 2 entries),
 *               every element written, including the padding columns.
 *   decision, n_incorrect, hist_pred, hist_gt: as in sc_decide (same pass).
 * Needs GT.  Computes in fp32, accumulates loss_sum in fp64.
 * Accuracy (the parity bar): decisions / counters / indices exact; loss_row
 * and each gradient entry within 1e-5 of the fp64 value relative to max(|value|, 1e-30) —
 * below 1e-30 the bound is absolute (σ'(z) of |z| > ~87 is subnormal in fp32, SURVEY.md
 * §8(c)9).  Holds for k·|S argument| <= ~40 (k <= 40 with probabilities as arguments);
 * larger k amplifies the fp32 rounding of the argument by k. */
sc_status sc_loss_fwd_bwd(sc_context ctx, const sc_batch* batch, const float* w, float grad_scale,
                          double* loss_sum, float* loss_row, int32_t* grad_idx, float* grad_val,
                          float* grad_dense, uint8_t* decision, uint64_t* n_incorrect, uint64_t* hist_pred,
                          uint64_t* hist_gt, sc_stream stream);

/* ---- Host-resident batches ----------------------------------------------------------------
 * The logits of a training set often live in host memory (a data loader's pinned buffers).
 * sc_stager owns the device side of moving them: chunk_bytes of device staging twice over,
 * a copy stream and its events, allocated once (hot calls never allocate).  One stager serves
 * one call at a time (calls on different streams need different stagers).
 *   chunk_bytes  bytes of logits per chunk (>= one row; e.g. 256 MiB); rounded up to 256.
 * Errors: SC_ERR_INVALID_ARG (chunk_bytes < 1), SC_ERR_OOM, SC_ERR_CUDA. */
typedef struct sc_stager_s* sc_stager;
sc_status sc_stager_create(int64_t chunk_bytes, sc_stager* out);
/* Waits for the stager's copies; NULL is a no-op. */
sc_status sc_stager_free(sc_stager stager);

typedef enum {
  SC_HOST_AUTO = 0,       /* ZERO_COPY when the rows are page-locked and the context reads few
                             128-B lines of a row (the sparse gather kernel's regime), else COPY */
  SC_HOST_COPY = 1,       /* chunked host->device copies on the stager's copy stream, double-
                             buffered: chunk i's pass overlaps chunk i+1's copy */
  SC_HOST_ZERO_COPY = 2   /* the kernels read the page-locked host rows in place: only the lines
                             holding mapped labels cross the host link */
} sc_host_mode;

/* sc_loss_fwd_bwd_host — sc_loss_fwd_bwd (the same pass, outputs and accumulation, Eq.
 * api_output PAPER.md:2035 and the other patterns) over logits in HOST memory:
 * batch->logits is a host pointer ([rows, ld] row-major, 16-B aligned, ld*elt % 16 == 0;
 * page-locked — cudaHostAlloc / cudaHostRegister — for COPY to overlap and for ZERO_COPY at
 * all).  Every other pointer (gt_mask / gt_off / gt_lab / app, w, all outputs) is a DEVICE
 * pointer exactly as in sc_loss_fwd_bwd; per-row outputs are written for all `rows`.
 * Asynchronous with respect to the host, stream-ordered on `stream` (the host rows must stay
 * valid until it completes).
 *   mode     sc_host_mode; *mode_used (may be NULL) receives the mode taken.
 * Errors: as sc_loss_fwd_bwd; SC_ERR_INVALID_ARG for a NULL stager in COPY mode, a row wider
 * than the stager's chunk, or ZERO_COPY on pageable memory. */
sc_status sc_loss_fwd_bwd_host(sc_context ctx, sc_stager stager, const sc_batch* batch, int32_t mode,
                               const float* w, float grad_scale, double* loss_sum, float* loss_row,
                               int32_t* grad_idx, float* grad_val, float* grad_dense, uint8_t* decision,
                               uint64_t* n_incorrect, uint64_t* hist_pred, uint64_t* hist_gt,
                               int32_t* mode_used, sc_stream stream);

/* ---- One read, many contexts (NEXT f3) ------------------------------------------------
 * sc_decide_all_apps — every row is evaluated under EVERY application of the context
 * (the provider's what-if: which applications would these outputs mislead), reading the
 * logits once.  API-output order only; batch->app and batch->gt_mask are ignored, the
 * ground truth comes from gt_off/gt_lab (G differs per application).
 *   n_incorrect  [n_apps] += per application, rows whose decision is incorrect (Eq. goal)
 *   hist_pred    [n_apps*256] += per application decision histogram
 *   decision     [rows*n_apps] uint8 (row-major) or NULL
 * All applications' mapped labels must fit in shared memory (about 50K entries). */
sc_status sc_decide_all_apps(sc_context ctx, const sc_batch* batch, uint64_t* n_incorrect, uint64_t* hist_pred,
                             uint8_t* decision, sc_stream stream);

/* ---- Value-ranges applications, NEXT f1 -------------------------
 * The API returns a score O_i per input; the application checks, in code order, whether
 * it lies in each of its ranges [lo_j, hi_j] (reading A22: closed ranges, the first
 * containing range wins, none -> default m).  Loss:
 *   L_i = w[r_i] ( S(lo_{r_i} − O_i) + S(O_i − hi_{r_i}) ),  r_i = the range the
 * ground-truth score lies in (no range -> L_i = 0), w[r] = M / N_r (rebalancing). */
typedef struct sc_ranges_s* sc_ranges;

/* m in [1, 255] ranges; lo/hi host arrays (copied), lo_j <= hi_j finite; k > 0. */
sc_status sc_ranges_load(int32_t m, const float* lo, const float* hi, float k, sc_ranges* out);
sc_status sc_ranges_free(sc_ranges r);
/* Ground-truth pre-pass: hist_gt [m+1] += #{i : r_i = r}; gt_range_out [rows] = r_i (optional). */
sc_status sc_ranges_hist(sc_ranges r, const float* gt_score, int64_t rows, uint64_t* hist_gt,
                         uint8_t* gt_range_out, sc_stream stream);
/* w [m+1] = M / hist_gt[r] (0 for empty bins), M = sum of hist_gt (the GLOBAL histogram). */
sc_status sc_ranges_weights(sc_ranges r, const uint64_t* hist_gt, float* w, sc_stream stream);
/* One pass over the scores: decision [rows] (range id, m = none), n_incorrect [1] += #{d_i ≠ r_i},
 * hist_pred [m+1] += decision histogram, loss_sum [1] += Σ L_i, loss_row [rows] = L_i,
 * grad [rows] = dL_i/dO_i · grad_scale.  w NULL = all 1.  Outputs may be NULL. */
sc_status sc_ranges_loss_fwd_bwd(sc_ranges r, const float* score, const uint8_t* gt_range, int64_t rows,
                                 const float* w, float grad_scale, double* loss_sum, float* loss_row, float* grad,
                                 uint8_t* decision, uint64_t* n_incorrect, uint64_t* hist_pred,
                                 sc_stream stream);
const char* sc_ranges_last_error(void);

/* ---- Rebalanced training-data sampler (NEXT f2) --------------------
 * Draws n row indices i.i.d. with probability q_i = w[G_i] / Σ_j w[G_j] (w = M/N from
 * sc_weights_from_hist: the balance of PAPER.md:2020/2029), one application's rows.
 * Mapping of uniforms to rows (reading A24): rows grouped by G (ascending mask, row order
 * inside), bucket weights count_m·w[m] summed in double in ascending m; bucket = first m
 * with u1·ΣW < cumulative W; row = number min(count_m − 1, floor(u2·count_m)) of the bucket.
 *   gt_mask    device [rows] G_i (from sc_decision_hist)
 *   w          device [256] float per-mask weights
 *   u          device [2n] double uniforms in [0,1), interleaved (u1, u2) per draw
 *   out        device [n] int64 row indices (-1 for every draw if all weights are 0)
 *   workspace  device scratch of at least sc_sample_workspace_bytes(rows) bytes
 *   rows       1 .. 2^31 - 1 (SC_ERR_INVALID_ARG otherwise)
 * Five launches (mask counts per 1024-row chunk, per-mask scans, bucket starts + CDF, a stable
 * scatter, the draws), stream-ordered; no allocation. */
size_t sc_sample_workspace_bytes(int64_t rows);
sc_status sc_rebalance_sample(const uint8_t* gt_mask, int64_t rows, const float* w, const double* u, int64_t n,
                              int64_t* out, void* workspace, size_t workspace_bytes, sc_stream stream);
const char* sc_sample_last_error(void);

/* ---- Classifier head fused with the evaluation (NEXT f4) ------------------------------
 * The step upstream of the path: the API's logits are a linear head over features,
 * z_i = x_i Wᵀ + b (x_i ∈ R^d, W ∈ R^{C×d}).  Labels outside 𝕎 are in no list, so they
 * never pick a decision (the if-chain) and Eq. api_output
 * only reads maxima over 𝕎: the head is compiled down to the |𝕎|
 * mapped rows of W, computed on the tensor cores (tcgen05, bf16 operands, fp32
 * accumulation in TMEM), and the decision, counters, loss and gradient are produced in the
 * GEMM's epilogue.  The logits never reach HBM.  Every decision pattern (the context's
 * order: API-output, application-choice, Multi-Select — PAPER.md:2022-2055), one application.
 *
 * sc_head_load — compile the head for ctx: copies the mapped rows of W (in label order),
 * their bias and keys into a device buffer the head owns (W and bias are not referenced
 * afterwards).
 *   weight  device bf16 (uint16 bit patterns) [C][ldw], ldw >= d;  d >= 1.
 *   bias    device float [C] or NULL (0).
 * SC_ERR_UNSUPPORTED: n_apps != 1, or more than 4096 head columns (see sc_head_info).
 * The head is compiled for the context's pattern (Multi-Select: a label in several lists has
 * a column in each) and may only be used with contexts of that pattern (SC_ERR_INVALID_ARG).
 * The copy is enqueued on `stream`; the head is usable on that stream when this returns. */
typedef struct sc_head_s* sc_head;
sc_status sc_head_load(sc_context ctx, const uint16_t* weight, int64_t ldw, int64_t d, const float* bias,
                       sc_stream stream, sc_head* out);
sc_status sc_head_free(sc_head head);
/* d, and the number of head columns computed per row: the mapped labels grouped by list
 * (code order, ascending label id inside a list), each list padded to a multiple of 16,
 * the total to a multiple of 32.  Up to 512 columns live in tensor memory at once; wider
 * heads (e.g. the OpenImages-shaped 1000 mapped labels) run in equal
 * column passes of <= 256 columns (padded to a multiple of the pass width), the features
 * re-read from L2 per pass.  SC_ERR_UNSUPPORTED from sc_head_load above 4096. */
sc_status sc_head_info(sc_head head, int64_t* d, int32_t* n_cols);

typedef struct {
  const uint16_t* x;       /* device bf16 [rows][ldx] features, ldx >= d, ldx % 8 == 0, 16-B aligned */
  int64_t rows;
  int64_t ldx;             /* elements */
  const int64_t* gt_off;   /* ground truth as in sc_batch (CSR, rows+1) or NULL */
  const int32_t* gt_lab;
  const uint8_t* gt_mask;  /* or precomputed G_i (sc_decision_hist's gt_mask_out); wins over CSR */
} sc_head_batch;

/* sc_head_loss_fwd_bwd — z_i = x_i W_𝕎ᵀ + b_𝕎 (fp32 accumulation of bf16 products, then
 * + bias in fp32), then exactly sc_loss_fwd_bwd's outputs for those logits (S =
 * sc_context_order's grad_slots; grad_idx holds label ids in [0, C), grad_val = dL_i/dz_c).  Every output may be NULL;
 * the loss is computed when loss_sum, loss_row, grad_idx or grad_val is given, which needs
 * the ground truth, as do n_incorrect and hist_gt.  The gradient w.r.t. x and W follows
 * from grad_idx/grad_val (at most two rows of W per sample) and is the caller's. */
sc_status sc_head_loss_fwd_bwd(sc_context ctx, sc_head head, const sc_head_batch* batch, const float* w,
                               float grad_scale, double* loss_sum, float* loss_row, int32_t* grad_idx,
                               float* grad_val, uint8_t* decision, uint64_t* n_incorrect, uint64_t* hist_pred,
                               uint64_t* hist_gt, sc_stream stream);

/* Thread-local text for the last non-OK status of this thread ("" if none). */
const char* sc_last_error(void);

/* Number of kernel launches enqueued by this process (for bench accounting). */
uint64_t sc_launch_count(void);

/* Name of the evaluation kernel the last sc_decide / sc_loss_fwd_bwd call of this
 * thread launched: "tma_ring" (dense rows staged through shared memory) or
 * "gather_epl<N>" (sector-sparse loads of the mapped labels only). */
const char* sc_last_kernel(void);

#ifdef __cplusplus
}
#endif
#endif /* SC_H */
