/* sc_oracle.c — plain, slow, obviously-correct CPU oracle for the
 * software-context hot path (ChameleonAPI drafts bundled in arXiv 2310.07240's
 * source).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may link, import or
 * execute this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg use it.  It shares no code, header,
 * table or constant with paper_2310_07240_b200/ (the CUDA path).
 *
 * Every function follows the paper's text in its order and notation, in
 * double precision (the paper fixes no precision).  Citations are
 * PAPER.md:<line> (Section / Equation) under /root/reference; the readings
 * A1..A19 taken where the paper is silent are listed in DESIGN.md §3.
 *
 * Pins (tests/test_oracle_*.py): the paper's worked example,
 * the non-critical-error example, the paper's Python listing
 * executed verbatim, brute force over every label subset for
 * C <= 12 against the argmax characterisation, step-function limit of the loss
 * vs the incorrect-decision indicator, central finite
 * differences for the gradient, the True-False special case of the weights
 * and an O(M^2) literal recount of N_i.
 * "Parity unpinned": the absolute loss scale depends on k, theta and the batch
 * reduction, which the paper leaves open (readings A3, A11, A14).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t C;                  /* number of API labels                                */
  int32_t n_apps;             /* number of applications (software contexts)          */
  const int32_t* n_lists;     /* [n_apps] number of target classes W_1..W_m per app  */
  const int64_t* list_off;    /* per app n_lists[a]+1 offsets, concatenated          */
  const int32_t* list_labels; /* label ids of every list, in code order              */
  double tau;                 /* label c is in the API output iff z_c > tau          */
  double k;                   /* steepness of S(x) = 1/(1+e^{-kx})                   */
  int32_t order;              /* decision pattern: 0 Multi-Choice API-output order,
                                 1 Multi-Choice application-choice order, 2 Multi-Select */
} orc_ctx;

/* ---------------------------------------------------------------- context */

static int64_t app_base(const orc_ctx* x, int32_t app) {
  int64_t b = 0;
  for (int32_t a = 0; a < app; ++a) b += x->n_lists[a] + 1;
  return b;
}

/* The listing's "if obj.name in Recycle: ... if obj.name in Compost: ..."
 * (PAPER.md:128-134): the first list, in code order, that contains label c;
 * -1 if none.  Reading A5: a label in several lists belongs to the first. */
int32_t orc_first_list(const orc_ctx* x, int32_t app, int32_t c) {
  const int64_t b = app_base(x, app);
  for (int32_t j = 0; j < x->n_lists[app]; ++j)
    for (int64_t t = x->list_off[b + j]; t < x->list_off[b + j + 1]; ++t)
      if (x->list_labels[t] == c) return j;
  return -1;
}

/* a1: per-label result of that scan for every label (done once per app). */
void orc_compile(const orc_ctx* x, int32_t app, int8_t* cat) {
  for (int32_t c = 0; c < x->C; ++c) cat[c] = (int8_t)orc_first_list(x, app, c);
}

/* ---------------------------------------------------------------- decision */

static _Thread_local const double* t_sort_z; /* qsort has no context argument */
static int cmp_confidence(const void* pa, const void* pb) {
  const int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  const double za = t_sort_z[a], zb = t_sort_z[b];
  if (za > zb) return -1;          /* descending confidence */
  if (za < zb) return 1;
  return (a < b) ? -1 : (a > b);   /* reading A4: equal confidence -> smaller label id first */
}

/* Decision(API(x)) for one input, simulated literally:
 * API output = labels with z_c > tau (reading A3), ranked by
 * descending confidence; the app walks them and returns the
 * branch of the first label found in a list.  Falling off
 * the loop is the default decision D' = n_lists (reading A6). */
int32_t orc_decide(const orc_ctx* x, int32_t app, const int8_t* cat, const double* z, int32_t* scratch) {
  int32_t n = 0;
  for (int32_t c = 0; c < x->C; ++c)
    if (z[c] > x->tau) scratch[n++] = c;
  t_sort_z = z;
  qsort(scratch, (size_t)n, sizeof(int32_t), cmp_confidence);
  for (int32_t t = 0; t < n; ++t)
    if (cat[scratch[t]] >= 0) return cat[scratch[t]];
  return x->n_lists[app];
}

/* G_i: the target classes the ground truth intersects, {j : W_j ∩ ŷ_i ≠ ∅}
 * (PAPER.md:2028 for 𝒲_i, :2038 for y_i), as a bit set over j. */
uint32_t orc_gt_set(const int8_t* cat, const int32_t* labels, int64_t n) {
  uint32_t G = 0;
  for (int64_t t = 0; t < n; ++t)
    if (cat[labels[t]] >= 0) G |= 1u << cat[labels[t]];
  return G;
}

/* Eq. goal counts Decision(API(x_i)) ≠ Decision(ŷ_i).
 * Reading A7: with the ground truth as API output the app reaches any j in G_i
 * (depending on order), and the default iff G_i = ∅. */
int32_t orc_correct(uint32_t G, int32_t d, int32_t n_lists) {
  if (G == 0) return d == n_lists;
  return d < n_lists && ((G >> d) & 1u);
}

/* ---------------------------------------------------------------- loss */

static double sigma(double z) {               /* p_c = σ(z_c), reading A2 */
  if (z >= 0) return 1.0 / (1.0 + exp(-z));
  const double e = exp(z);
  return e / (1.0 + e);
}
static double S(double k, double x) { return sigma(k * x); }
static double dS(double k, double x) { return k * sigma(k * x) * sigma(-k * x); }
static double dsigma(double z) { return sigma(z) * sigma(-z); }

/* Multi-Choice API-output-order loss, Eq. api_output:
 *   L = (M/N_i) ( y_i S(max(P⁻, θ) − P⁺) + (1 − y_i) S(P⁻ − θ) )
 * P⁺ = max_{c ∈ 𝒲_i} p_c, P⁻ = max_{c ∈ 𝕎∖𝒲_i} p_c, θ = σ(τ) (reading A3),
 * max over ∅ = −∞ (A9).  w = M/N_i is passed in.  σ is increasing, so
 * max_c σ(z_c) = σ(max_c z_c): the arg max is taken over z (smallest id on
 * ties, A8) and σ applied after, which keeps the arg max exact where σ
 * saturates in floating point.  Gradient: chain rule with the whole
 * subgradient on the arg max (A10); P⁻ receives gradient through max(P⁻, θ)
 * only when P⁻ > θ, i.e. z⁻ > τ.
 * Outputs: ell (unweighted), L = w·ell, and up to two gradient entries. */
void orc_loss_row(const orc_ctx* x, const int8_t* cat, const double* z, uint32_t G, double w,
                  double* ell_out, double* L_out,
                  int32_t* c_plus, double* g_plus, int32_t* c_minus, double* g_minus) {
  const double theta = sigma(x->tau);
  const int y = G != 0;
  int32_t cp = -1, cm = -1;
  for (int32_t c = 0; c < x->C; ++c) {
    if (cat[c] < 0) continue;                                       /* c ∉ 𝕎 */
    if ((G >> cat[c]) & 1u) { if (cp < 0 || z[c] > z[cp]) cp = c; } /* c ∈ 𝒲_i      */
    else                     { if (cm < 0 || z[c] > z[cm]) cm = c; } /* c ∈ 𝕎 ∖ 𝒲_i */
  }
  const double Pp = cp >= 0 ? sigma(z[cp]) : -INFINITY;
  const double Pm = cm >= 0 ? sigma(z[cm]) : -INFINITY;
  const int m_over = cm >= 0 && z[cm] > x->tau;                     /* P⁻ > θ */
  double ell = 0.0, gp = 0.0, gm = 0.0;
  int32_t op = -1, om = -1;
  if (y) {
    const double a = m_over ? Pm : theta;                           /* max(P⁻, θ) */
    ell = S(x->k, a - Pp);
    const double d = dS(x->k, a - Pp);
    gp = -w * d * dsigma(z[cp]); op = cp;
    if (m_over) { gm = w * d * dsigma(z[cm]); om = cm; }
  } else if (cm >= 0) {
    ell = S(x->k, Pm - theta);
    gm = w * dS(x->k, Pm - theta) * dsigma(z[cm]); om = cm;
  }
  *ell_out = ell;
  *L_out = w * ell;
  *c_plus = op; *g_plus = gp; *c_minus = om; *g_minus = gm;
}

/* ---------------------------------------------------------------- weights */

/* N_i and M/N_i by the literal definitions: for a
 * target input N_i = Σ_j 1[ŷ_j ∩ 𝒲_i ≠ ∅]; for a non-target input N_i =
 * Σ_j 1[ŷ_j ∩ 𝕎 = ∅] (reading A12: ŷ_j).  O(M²) — small M only.
 * Rows are one app's inputs; cat is that app's compiled map. */
void orc_weights_literal(const int8_t* cat, int64_t M, const int64_t* gt_off, const int32_t* gt_lab,
                         double* w_row) {
  for (int64_t i = 0; i < M; ++i) {
    const uint32_t Gi = orc_gt_set(cat, gt_lab + gt_off[i], gt_off[i + 1] - gt_off[i]);
    int64_t N = 0;
    for (int64_t j = 0; j < M; ++j) {
      int hit = 0, any_mapped = 0;
      for (int64_t t = gt_off[j]; t < gt_off[j + 1]; ++t) {
        const int8_t cj = cat[gt_lab[t]];
        if (cj >= 0) { any_mapped = 1; if ((Gi >> cj) & 1u) hit = 1; }
      }
      N += Gi ? hit : !any_mapped;
    }
    w_row[i] = (double)M / (double)N;   /* N >= 1: row i counts itself */
  }
}

/* The same definition evaluated once per distinct G (rows with equal G_i have
 * equal N_i): H[m] = #{j : G_j = m};  N(m) = Σ_{m'} H[m']·1[m' ∩ m ≠ ∅] for
 * m ≠ ∅, N(∅) = H[∅].  w[m] = M/N(m), and 0 for masks no input has (A13). */
void orc_weights_by_mask(int32_t n_apps, const uint64_t* H, double* w) {
  for (int32_t a = 0; a < n_apps; ++a) {
    const uint64_t* h = H + (int64_t)a * 256;
    uint64_t M = 0;
    for (int m = 0; m < 256; ++m) M += h[m];
    for (int m = 0; m < 256; ++m) {
      uint64_t N = 0;
      if (m == 0) N = h[0];
      else for (int q = 0; q < 256; ++q) if (q & m) N += h[q];
      w[(int64_t)a * 256 + m] = N ? (double)M / (double)N : 0.0;
    }
  }
}

/* ---------------------------------------------------------------- other decision patterns */

/* Lists (bit j) containing label c, by scanning every list: a Multi-Select
 * application acts on every list an output label belongs to,
 * so for that pattern a label shared by two lists counts for both. */
uint32_t orc_label_lists(const orc_ctx* x, int32_t app, int32_t c) {
  const int64_t b = app_base(x, app);
  uint32_t m = 0;
  for (int32_t j = 0; j < x->n_lists[app]; ++j)
    for (int64_t t = x->list_off[b + j]; t < x->list_off[b + j + 1]; ++t)
      if (x->list_labels[t] == c) { m |= 1u << j; break; }
  return m;
}

/* {j : W_j ∩ ŷ ≠ ∅} with every list scanned (Multi-Select's ground-truth decision). */
uint32_t orc_gt_set_raw(const orc_ctx* x, int32_t app, const int32_t* labels, int64_t n) {
  uint32_t G = 0;
  for (int64_t t = 0; t < n; ++t) G |= orc_label_lists(x, app, labels[t]);
  return G;
}

/* Multi-Choice, application-choice order (loop nesting PAPER.md:2154-2156):
 * "checking if the first target class matches with any output label before moving to
 * the next class" — lists in code order, the first with any output label wins. */
int32_t orc_decide_app_choice(const orc_ctx* x, int32_t app, const double* z) {
  const int64_t b = app_base(x, app);
  for (int32_t j = 0; j < x->n_lists[app]; ++j)
    for (int64_t t = x->list_off[b + j]; t < x->list_off[b + j + 1]; ++t)
      if (z[x->list_labels[t]] > x->tau) return j;
  return x->n_lists[app];
}

/* k = min{j | W_j ∩ ŷ_i ≠ ∅}: the application-choice decision the
 * ground truth leads to (unique, whatever the output order); D' if none. */
int32_t orc_gt_decision_app_choice(const orc_ctx* x, int32_t app, const int32_t* labels, int64_t n) {
  const int64_t b = app_base(x, app);
  for (int32_t j = 0; j < x->n_lists[app]; ++j)
    for (int64_t t = x->list_off[b + j]; t < x->list_off[b + j + 1]; ++t)
      for (int64_t q = 0; q < n; ++q)
        if (labels[q] == x->list_labels[t]) return j;
  return x->n_lists[app];
}

/* Multi-Select: every list with an output label is selected. */
uint32_t orc_decide_multi_select(const orc_ctx* x, int32_t app, const double* z) {
  const int64_t b = app_base(x, app);
  uint32_t m = 0;
  for (int32_t j = 0; j < x->n_lists[app]; ++j)
    for (int64_t t = x->list_off[b + j]; t < x->list_off[b + j + 1]; ++t)
      if (z[x->list_labels[t]] > x->tau) { m |= 1u << j; break; }
  return m;
}

/* Eq. app_choice:
 *   L = (M/N_i) ( y_i S(max(θ, P_{k⁻}) − P_k) + (1 − y_i) S(P − θ) ),
 * P_k = max over W_k, P_{k⁻} = max over the higher-priority lists W_j, j < k (the
 * printed condition "ŷ ∩ W_j ≠ ∅ and j < k" is empty by the definition of k; reading
 * A21: j < k), P = max over 𝕎.  Lists are the compiled first-list sets (A5): a label
 * shared with an earlier list can only ever trigger the earlier one.  Arg maxima over
 * z, smallest id on ties (A8); P_{k⁻} gets gradient only when it exceeds θ (A10). */
void orc_loss_row_app_choice(const orc_ctx* x, const int8_t* cat, const double* z, uint32_t G, double w,
                             double* ell_out, double* L_out, int32_t* c_a, double* g_a, int32_t* c_b,
                             double* g_b) {
  const double theta = sigma(x->tau);
  const int y = G != 0;
  int32_t kk = -1;
  for (int32_t j = 0; j < 32 && y; ++j) if ((G >> j) & 1u) { kk = j; break; }
  int32_t ck = -1, ckm = -1, cP = -1;
  for (int32_t c = 0; c < x->C; ++c) {
    if (cat[c] < 0) continue;
    if (cP < 0 || z[c] > z[cP]) cP = c;
    if (y && cat[c] == kk && (ck < 0 || z[c] > z[ck])) ck = c;
    if (y && cat[c] < kk && (ckm < 0 || z[c] > z[ckm])) ckm = c;
  }
  double ell = 0.0, ga = 0.0, gb = 0.0;
  int32_t oa = -1, ob = -1;
  if (y) {
    const int km_over = ckm >= 0 && z[ckm] > x->tau;            /* P_{k⁻} > θ */
    const double a = km_over ? sigma(z[ckm]) : theta;           /* max(θ, P_{k⁻}) */
    const double arg = a - sigma(z[ck]);
    ell = S(x->k, arg);
    const double d = dS(x->k, arg);
    ga = -w * d * dsigma(z[ck]); oa = ck;
    if (km_over) { gb = w * d * dsigma(z[ckm]); ob = ckm; }
  } else if (cP >= 0) {
    const double arg = sigma(z[cP]) - theta;
    ell = S(x->k, arg);
    gb = w * dS(x->k, arg) * dsigma(z[cP]); ob = cP;
  }
  *ell_out = ell;
  *L_out = w * ell;
  *c_a = oa; *g_a = ga; *c_b = ob; *g_b = gb;
}

/* Eq. multi-select, reading the printed y_i inside the sum as y_ij
 * (= bit j of G):
 *   L = (M/N_i) Σ_j ( y_ij S(θ − P_j) + (1 − y_ij) S(P_j − θ) ),  P_j = max over W_j.
 * Lists are scanned as written (a shared label belongs to every list containing it).
 * An empty list contributes nothing (P_j = −∞, and y_ij = 0 for it).  c[j], g[j]: the
 * gradient entry of list j (−1 / 0 when the list is empty). */
void orc_loss_row_multi_select(const orc_ctx* x, int32_t app, const double* z, uint32_t G, double w,
                               double* ell_out, double* L_out, int32_t* c, double* g) {
  const double theta = sigma(x->tau);
  const int64_t b = app_base(x, app);
  double ell = 0.0;
  for (int32_t j = 0; j < 8; ++j) { c[j] = -1; g[j] = 0.0; }
  for (int32_t j = 0; j < x->n_lists[app]; ++j) {
    int32_t cj = -1;
    for (int64_t t = x->list_off[b + j]; t < x->list_off[b + j + 1]; ++t) {
      const int32_t q = x->list_labels[t];
      if (cj < 0 || z[q] > z[cj] || (z[q] == z[cj] && q < cj)) cj = q;
    }
    if (cj < 0) continue;
    const double Pj = sigma(z[cj]);
    if ((G >> j) & 1u) {
      ell += S(x->k, theta - Pj);
      g[j] = -w * dS(x->k, theta - Pj) * dsigma(z[cj]);
    } else {
      ell += S(x->k, Pj - theta);
      g[j] = w * dS(x->k, Pj - theta) * dsigma(z[cj]);
    }
    c[j] = cj;
  }
  *ell_out = ell;
  *L_out = w * ell;
}

/* N_i by the literal definition for any pattern: lm[c] = the lists label
 * c counts for (first list for the choice orders, every list for Multi-Select);
 * 𝒲_i = labels whose lists meet G_i. */
void orc_weights_literal_masks(const uint8_t* lm, int64_t M, const int64_t* gt_off, const int32_t* gt_lab,
                               double* w_row) {
  for (int64_t i = 0; i < M; ++i) {
    uint32_t Gi = 0;
    for (int64_t t = gt_off[i]; t < gt_off[i + 1]; ++t) Gi |= lm[gt_lab[t]];
    int64_t N = 0;
    for (int64_t j = 0; j < M; ++j) {
      int hit = 0, any_mapped = 0;
      for (int64_t t = gt_off[j]; t < gt_off[j + 1]; ++t) {
        const uint32_t mj = lm[gt_lab[t]];
        if (mj) { any_mapped = 1; if (mj & Gi) hit = 1; }
      }
      N += Gi ? hit : !any_mapped;
    }
    w_row[i] = (double)M / (double)N;
  }
}

/* ---------------------------------------------------------------- batch */

static double load_z(const void* logits, int32_t dtype, int64_t idx) {
  if (dtype == 0) return (double)((const float*)logits)[idx];
  uint32_t u = (uint32_t)((const uint16_t*)logits)[idx] << 16;   /* bf16 -> f32 bits */
  float f; memcpy(&f, &u, 4);
  return (double)f;
}

/* Every output of the hot path for `rows` inputs, for the context's decision pattern.
 * Any output may be NULL; counters ACCUMULATE (+=).  w: [n_apps*256] per-mask weights,
 * NULL = 1.  hist_pred: [n_apps*256] (a Multi-Select decision is a list mask).
 * grad_idx/grad_val: [rows*S], S = 2 for the choice orders (slot 0: the class the loss
 * pushes up, slot 1: the competitor), S = 8 for Multi-Select (slot j = list j); −1 / 0
 * when absent; values multiplied by grad_scale.  Returns 0, or −1 on a non-finite logit
 * (reading A18) or an out-of-range id. */
int orc_eval(const orc_ctx* x, int64_t rows, int64_t ld, int32_t dtype, const void* logits,
             const int64_t* gt_off, const int32_t* gt_lab, const uint16_t* app,
             const double* w, double grad_scale,
             uint8_t* decision, uint8_t* gt_mask, uint8_t* correct,
             uint64_t* n_incorrect, uint64_t* hist_pred, uint64_t* hist_gt,
             double* loss_sum, double* loss_row, int32_t* grad_idx, double* grad_val) {
  const int32_t C = x->C;
  const int S_ = x->order == 2 ? 8 : 2;
  int8_t* cat = (int8_t*)malloc((size_t)x->n_apps * (size_t)(C > 0 ? C : 1));
  double* z = (double*)malloc(sizeof(double) * (size_t)(C > 0 ? C : 1));
  int32_t* scratch = (int32_t*)malloc(sizeof(int32_t) * (size_t)(C > 0 ? C : 1));
  int rc = 0;
  for (int32_t a = 0; a < x->n_apps; ++a) orc_compile(x, a, cat + (int64_t)a * C);
  for (int64_t i = 0; i < rows && rc == 0; ++i) {
    const int32_t a = app ? (int32_t)app[i] : 0;
    if (a >= x->n_apps) { rc = -1; break; }
    const int8_t* ca = cat + (int64_t)a * C;
    for (int32_t c = 0; c < C; ++c) {
      z[c] = load_z(logits, dtype, i * ld + c);
      if (!isfinite(z[c])) rc = -1;
    }
    if (rc) break;
    const int32_t D = x->n_lists[a];
    int32_t d;
    if (x->order == 0) d = orc_decide(x, a, ca, z, scratch);
    else if (x->order == 1) d = orc_decide_app_choice(x, a, z);
    else d = (int32_t)orc_decide_multi_select(x, a, z);
    if (decision) decision[i] = (uint8_t)d;
    if (hist_pred) hist_pred[(int64_t)a * 256 + d] += 1;
    if (!gt_off) continue;
    for (int64_t t = gt_off[i]; t < gt_off[i + 1]; ++t)
      if (gt_lab[t] < 0 || gt_lab[t] >= C) rc = -1;
    if (rc) break;
    const int32_t* gl = gt_lab + gt_off[i];
    const int64_t gn = gt_off[i + 1] - gt_off[i];
    uint32_t G;
    int32_t ok;
    if (x->order == 0) {
      G = orc_gt_set(ca, gl, gn);
      ok = orc_correct(G, d, D);
    } else if (x->order == 1) {
      G = orc_gt_set(ca, gl, gn);
      ok = d == orc_gt_decision_app_choice(x, a, gl, gn);
    } else {
      G = orc_gt_set_raw(x, a, gl, gn);
      ok = (uint32_t)d == G;   /* "exactly match with the ground-truth decisions" */
    }
    if (gt_mask) gt_mask[i] = (uint8_t)G;
    if (correct) correct[i] = (uint8_t)ok;
    if (n_incorrect) n_incorrect[a] += (uint64_t)!ok;
    if (hist_gt) hist_gt[(int64_t)a * 256 + G] += 1;
    if (loss_sum || loss_row || grad_idx || grad_val) {
      const double wi = w ? w[(int64_t)a * 256 + G] : 1.0;
      double ell, L;
      int32_t cs[8];
      double gs[8];
      for (int q = 0; q < 8; ++q) { cs[q] = -1; gs[q] = 0.0; }
      if (x->order == 0) orc_loss_row(x, ca, z, G, wi, &ell, &L, &cs[0], &gs[0], &cs[1], &gs[1]);
      else if (x->order == 1) orc_loss_row_app_choice(x, ca, z, G, wi, &ell, &L, &cs[0], &gs[0], &cs[1], &gs[1]);
      else orc_loss_row_multi_select(x, a, z, G, wi, &ell, &L, cs, gs);
      if (loss_sum) loss_sum[a] += L;
      if (loss_row) loss_row[i] = L;
      for (int q = 0; q < S_; ++q) {
        if (grad_idx) grad_idx[S_ * i + q] = cs[q];
        if (grad_val) grad_val[S_ * i + q] = gs[q] * grad_scale;
      }
    }
  }
  free(cat); free(z); free(scratch);
  return rc;
}

/* The ground-truth-only pass (rows a2 + a6 of SURVEY.md §8(a)): G_i = the lists the
 * ground-truth labels of input i hit (Multi-Select: the raw list set,
 * PAPER.md:2031) and the mask histogram hist_gt[a][G_i] += 1 whose entries give the N_i
 * counts.  The same per-row definitions orc_eval uses, without logits,
 * so full-size tests can build the weights before the full pass.  Any output may be NULL;
 * hist_gt ACCUMULATES.  Returns 0, or -1 on an out-of-range id. */
int orc_gt_hist(const orc_ctx* x, int64_t rows, const int64_t* gt_off, const int32_t* gt_lab,
                const uint16_t* app, uint8_t* gt_mask, uint64_t* hist_gt) {
  const int32_t C = x->C;
  int8_t* cat = (int8_t*)malloc((size_t)x->n_apps * (size_t)(C > 0 ? C : 1));
  int rc = 0;
  for (int32_t a = 0; a < x->n_apps; ++a) orc_compile(x, a, cat + (int64_t)a * C);
  for (int64_t i = 0; i < rows && rc == 0; ++i) {
    const int32_t a = app ? (int32_t)app[i] : 0;
    if (a >= x->n_apps) { rc = -1; break; }
    for (int64_t t = gt_off[i]; t < gt_off[i + 1]; ++t)
      if (gt_lab[t] < 0 || gt_lab[t] >= C) rc = -1;
    if (rc) break;
    const int32_t* gl = gt_lab + gt_off[i];
    const int64_t gn = gt_off[i + 1] - gt_off[i];
    const uint32_t G = x->order == 2 ? orc_gt_set_raw(x, a, gl, gn) : orc_gt_set(cat + (int64_t)a * C, gl, gn);
    if (gt_mask) gt_mask[i] = (uint8_t)G;
    if (hist_gt) hist_gt[(int64_t)a * 256 + G] += 1;
  }
  free(cat);
  return rc;
}

/* ---------------------------------------------------------------- value ranges */

/* Value-ranges applications: the API returns a score O_i (e.g. a
 * sentiment score) and the application checks, in code order, whether it lies in each
 * of its ranges [l_j, h_j] (reading A22: closed ranges, the first containing range
 * wins, none -> default m).  The ground-truth range r_i is the one the true score lies in. */
int32_t orc_range_of(int32_t m, const double* lo, const double* hi, double score) {
  for (int32_t j = 0; j < m; ++j)
    if (score >= lo[j] && score <= hi[j]) return j;
  return m;
}

/* L = (M/N_i) ( S(l_i − O_i) + S(O_i − h_i) ) with [l_i, h_i] the ground-truth range
 * (PAPER.md:2061); rows whose ground truth lies in no range have no target range and
 * contribute nothing (reading A22).  dL/dO = w ( −S'(l − O) + S'(O − h) ). */
void orc_range_loss(int32_t m, const double* lo, const double* hi, double k, int32_t r, double score, double w,
                    double* L, double* dL) {
  if (r < 0 || r >= m) { *L = 0.0; *dL = 0.0; return; }
  const double a = lo[r] - score, b = score - hi[r];
  *L = w * (S(k, a) + S(k, b));
  *dL = w * (-dS(k, a) + dS(k, b));
}

/* Batch: decisions, counters (hist over ranges, [m+1] bins), loss and gradient. */
void orc_ranges_eval(int32_t m, const double* lo, const double* hi, double k, int64_t rows, const float* score,
                     const float* gt_score, const double* w, double grad_scale, uint8_t* decision, uint8_t* gt_range,
                     uint64_t* n_incorrect, uint64_t* hist_pred, uint64_t* hist_gt, double* loss_sum,
                     double* loss_row, double* grad) {
  for (int64_t i = 0; i < rows; ++i) {
    const int32_t d = orc_range_of(m, lo, hi, (double)score[i]);
    const int32_t r = orc_range_of(m, lo, hi, (double)gt_score[i]);
    if (decision) decision[i] = (uint8_t)d;
    if (gt_range) gt_range[i] = (uint8_t)r;
    if (n_incorrect) n_incorrect[0] += (uint64_t)(d != r);
    if (hist_pred) hist_pred[d] += 1;
    if (hist_gt) hist_gt[r] += 1;
    double L, dL;
    orc_range_loss(m, lo, hi, k, r, (double)score[i], w ? w[r] : 1.0, &L, &dL);
    if (loss_sum) loss_sum[0] += L;
    if (loss_row) loss_row[i] = L;
    if (grad) grad[i] = dL * grad_scale;
  }
}

/* Rebalancing over ranges: N_i = #inputs with the same ground-truth range (PAPER.md:2063
 * "N_i is defined similarly"); w[r] = M / N_r, 0 for an empty bin. */
void orc_ranges_weights(int32_t m, const uint64_t* H, double* w) {
  uint64_t M = 0;
  for (int32_t r = 0; r <= m; ++r) M += H[r];
  for (int32_t r = 0; r <= m; ++r) w[r] = H[r] ? (double)M / (double)H[r] : 0.0;
}

/* ---------------------------------------------------------------- rebalanced sampler */

/* The strawman of PAPER.md:1989-1990 (abstract PAPER.md:19-20): re-train on a re-sampled
 * training set that rebalances the application's target classes.  Inputs are drawn
 * i.i.d. with probability q_i = w_i / Σ_j w_j, w_i = M/N_i, the balance
 * the loss weights express ("the number of target-inputs and non-target-inputs are
 * effectively balanced").  Mapping of the two uniforms to an input
 * (reading A24): group rows by G (ascending mask, rows in row order), bucket weight
 * W_m = count_m · w[m] summed in double in ascending m; the bucket is the first m with
 * u1 · ΣW < cumulative W, the row is number min(count_m − 1, floor(u2 · count_m)) of it.
 * w: the per-mask weights as the caller has them (the kernel's f32 values, widened).
 * Returns 0, or −1 when every weight is 0. */
int orc_sample(const uint8_t* gt_mask, int64_t rows, const double* w, int64_t n, const double* u1, const double* u2,
               int64_t* out) {
  int64_t count[256] = {0};
  for (int64_t i = 0; i < rows; ++i) count[gt_mask[i]] += 1;
  int64_t start[256];
  int64_t acc = 0;
  for (int m = 0; m < 256; ++m) { start[m] = acc; acc += count[m]; }
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rows > 0 ? rows : 1));
  int64_t fill[256];
  for (int m = 0; m < 256; ++m) fill[m] = start[m];
  for (int64_t i = 0; i < rows; ++i) order[fill[gt_mask[i]]++] = i;   /* stable: row order within a mask */
  double cum[256];
  double total = 0.0;
  for (int m = 0; m < 256; ++m) { total += (double)count[m] * w[m]; cum[m] = total; }
  if (!(total > 0.0)) { free(order); return -1; }
  for (int64_t i = 0; i < n; ++i) {
    const double t = u1[i] * total;
    int m = 0;
    while (m < 255 && !(t < cum[m])) ++m;
    const int64_t c = count[m];
    int64_t pos = (int64_t)floor(u2[i] * (double)c);
    if (pos > c - 1) pos = c - 1;
    out[i] = order[start[m] + pos];
  }
  free(order);
  return 0;
}
