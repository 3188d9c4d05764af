// sc_api.cu — host side of libsc: the C ABI declared in include/sc.h.
// Validation, the context compile (a1), launch configuration and dispatch.
#include "sc.h"
#include "sc_host.h"
#include "sc_internal.cuh"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>


namespace {

thread_local std::string g_err;
thread_local std::string g_last_kernel;
std::atomic<uint64_t> g_launches{0};

sc_status fail(sc_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

sc_status cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? SC_ERR_OOM : SC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

constexpr size_t kSmemMax = 227 * 1024;

struct DeviceInfo {
  int sms = 0;
  bool eval_attr = false;
};

DeviceInfo& device_info(int dev) {
  static std::mutex mu;
  static DeviceInfo infos[64];
  std::lock_guard<std::mutex> lock(mu);
  DeviceInfo& d = infos[dev & 63];
  if (d.sms == 0) {
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    if (d.sms <= 0) d.sms = 148;
  }
  if (!d.eval_attr) {
    if (sc::set_eval_smem_limit(kSmemMax) == cudaSuccess) d.eval_attr = true;
  }
  return d;
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

sc::DevContext dev_ctx(const sc_context_s* c) {
  sc::DevContext d;
  d.cat = c->d_cat;
  d.ent = c->d_ent;
  d.ent_off = c->d_ent_off;
  d.nlists = c->d_nlists;
  d.lent = c->d_lent;
  d.lent_off = c->d_lent_off;
  d.lslot = c->d_lslot;
  d.col_label = c->d_col_label;
  d.C = c->C;
  d.n_apps = c->n_apps;
  d.max_ent = c->max_ent;
  d.tau = c->tau;
  d.theta = c->theta;
  d.k = c->k;
  d.order = c->order;
  return d;
}

sc_status check_batch_common(const sc_context_s* ctx, const sc_batch* b) {
  if (!ctx) return fail(SC_ERR_INVALID_ARG, "ctx is NULL");
  if (!b) return fail(SC_ERR_INVALID_ARG, "batch is NULL");
  if (b->rows < 0) return fail(SC_ERR_INVALID_ARG, "rows < 0");
  if (b->gt_off && !b->gt_lab && !b->gt_mask) return fail(SC_ERR_INVALID_ARG, "gt_off without gt_lab");
  return SC_OK;
}

// Largest fraction of touched 128-B lines at which the sector-sparse gather is chosen.
// Measured crossovers on B200: cfg3 f32 (0.81 touched) gather 5.41 ms vs TMA 5.80 ms; cfg4
// f32 (256 apps, 0.875 touched on average) gather 3.02 ms vs blocked TMA 2.38 ms.
double gather_threshold(int n_apps) {
  const char* s = std::getenv("SC_GATHER_MAX_FRAC");
  return s ? std::atof(s) : (n_apps > 1 ? 0.7 : 0.85);
}

int stage_kb_override() {
  const char* s = std::getenv("SC_STAGE_KB");
  if (!s) return 0;
  const int v = std::atoi(s);
  return (v >= 8 && v <= 200) ? v : 0;
}

// The fused pass behind sc_decide and sc_loss_fwd_bwd.
sc_status run_eval(const sc_context_s* ctx, const sc_batch* b, const float* w, float grad_scale, double* loss_sum,
                   float* loss_row, int32_t* grad_idx, float* grad_val, float* grad_dense, uint8_t* decision,
                   uint64_t* n_incorrect, uint64_t* hist_pred, uint64_t* hist_gt, bool loss_call, cudaStream_t st) {
  if (sc_status s = check_batch_common(ctx, b)) return s;
  if (b->dtype != SC_F32 && b->dtype != SC_BF16) return fail(SC_ERR_INVALID_ARG, "unknown dtype %d", (int)b->dtype);
  const bool has_gt = b->gt_mask || b->gt_off;
  const bool want_loss = loss_call && (loss_sum || loss_row || grad_idx || grad_val || grad_dense);
  if ((n_incorrect || hist_gt || loss_call) && !has_gt)
    return fail(SC_ERR_INVALID_ARG, "n_incorrect / hist_gt / loss need ground truth (gt_mask or gt_off+gt_lab)");
  if (b->rows == 0) return SC_OK;
  if (!b->logits) return fail(SC_ERR_INVALID_ARG, "logits is NULL");
  const int64_t elt = b->dtype == SC_F32 ? 4 : 2;
  if (b->ld < ctx->ncols)
    return fail(SC_ERR_INVALID_ARG, "ld (%lld) < logit columns (%d)", (long long)b->ld, ctx->ncols);
  if ((b->ld * elt) % 16) return fail(SC_ERR_INVALID_ARG, "ld*sizeof(elt) must be a multiple of 16");
  if (reinterpret_cast<uintptr_t>(b->logits) % 16) return fail(SC_ERR_INVALID_ARG, "logits not 16-B aligned");
  if (grad_dense && reinterpret_cast<uintptr_t>(grad_dense) % 16)
    return fail(SC_ERR_INVALID_ARG, "grad_dense not 16-B aligned");
  if (b->app && reinterpret_cast<uintptr_t>(b->app) % 2) return fail(SC_ERR_INVALID_ARG, "app not 2-B aligned");

  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_fail(e, "cudaGetDevice");
  if (dev != ctx->device) return fail(SC_ERR_INVALID_ARG, "context belongs to device %d, current is %d", ctx->device, dev);
  DeviceInfo& di = device_info(dev);
  if (!di.eval_attr) return fail(SC_ERR_CUDA, "cannot raise the kernel's shared-memory limit");

  sc::EvalParams p{};
  p.pend_off = -1;
  p.hdr_off = -1;
  p.ctx = dev_ctx(ctx);
  p.logits = static_cast<const uint8_t*>(b->logits);
  p.rows = b->rows;
  p.ld = b->ld;
  p.ld_bytes = b->ld * elt;
  p.bf16 = b->dtype == SC_BF16;
  p.gt_off = b->gt_mask ? nullptr : b->gt_off;
  p.gt_lab = b->gt_mask ? nullptr : b->gt_lab;
  p.gt_mask = b->gt_mask;
  p.app = b->app;
  p.has_gt = has_gt;
  p.w = want_loss ? w : nullptr;
  p.grad_scale = grad_scale;
  p.want_loss = want_loss;
  p.loss_sum = loss_call ? loss_sum : nullptr;
  p.loss_row = loss_call ? loss_row : nullptr;
  p.grad_idx = loss_call ? grad_idx : nullptr;
  p.grad_val = loss_call ? grad_val : nullptr;
  p.grad_dense = loss_call ? grad_dense : nullptr;
  p.decision = decision;
  p.n_incorrect = reinterpret_cast<unsigned long long*>(n_incorrect);
  p.hist_pred = reinterpret_cast<unsigned long long*>(hist_pred);
  p.hist_gt = reinterpret_cast<unsigned long long*>(hist_gt);

  // per-list patterns (application-choice order, Multi-Select) need every list's arg max
  const int pat = ctx->order == SC_ORDER_API_OUTPUT ? 0 : 1;
  const char* epl_env = std::getenv("SC_EPL");
  const bool want_epl = epl_env ? std::atoi(epl_env) != 0 : true;
  const int64_t force_chunk = std::getenv("SC_FORCE_CHUNK") ? std::atoll(std::getenv("SC_FORCE_CHUNK")) : 0;
  const bool whole_rows = sc::kConsumerWarps * p.ld_bytes <= 64 * 1024 && force_chunk == 0;
  // lane-resident entries on the TMA ring: whole rows per stage and |W| <= 1024
  // (per-list patterns: <= 8 list-major slots per app, one per register slot)
  const bool lane_ok = whole_rows && ctx->max_ent <= 1024 && want_epl &&
                       (pat ? ctx->max_slots <= 8 : sc::eval_epl_for(ctx->max_ent) > 0);
  // dense-mapped rows: every column of a row is a mapped label of the one application (column-
  // compacted rows): 16-B vector loads per lane, winners tracked by slot index (pat 2).
  const int dm_vec = elt == 4 ? 4 : 8;
  const int dm_nv = static_cast<int>((static_cast<int64_t>(ctx->ncols) + 32 * dm_vec - 1) / (32 * dm_vec));
  const char* dm_env = std::getenv("SC_DM");
  // Taken above 256 entries (EPL > 8, where the lane-resident path stops caching offsets in
  // registers): B200, cfg3 compacted (1000 columns) 0.392 vs 0.695 ms; cfg2 compacted (180
  // columns) the lane-resident path is faster, 0.330 vs 0.386 ms.
  // SC_DM=0 disables it, SC_DM=2 takes it at any width (tests)
  const int dm_mode = dm_env ? std::atoi(dm_env) : 1;
  const bool dm = pat == 0 && ctx->n_apps == 1 && whole_rows && (ctx->ncols > 256 || dm_mode == 2) &&
                  ctx->ncols >= 1 && ctx->max_ent == ctx->ncols && dm_nv * dm_vec <= 32 && dm_mode != 0 &&
                  !(std::getenv("SC_KERNEL") && std::string(std::getenv("SC_KERNEL")) == "gather");
  // application-choice order with <= 256 mapped labels: two arg maxima per row (list k and the
  // lists before it) plus a warp OR of the output lists, on lane-resident entries (pat 3),
  // instead of one arg max per 32-label slot (SC_AC2=0 keeps the slots)
  const char* ac2_env = std::getenv("SC_AC2");
  const bool ac2 = ctx->order == SC_ORDER_APP_CHOICE && whole_rows && ctx->max_ent <= 256 && want_epl &&
                   !(ac2_env && std::atoi(ac2_env) == 0) &&
                   !(std::getenv("SC_KERNEL") && std::string(std::getenv("SC_KERNEL")) == "gather");
  // ---- kernel choice: sector-sparse gather when the mapped labels leave enough row sectors untouched
  if (!dm && !ac2) {
    const char* kenv = std::getenv("SC_KERNEL");
    const int dt = b->dtype == SC_BF16 ? 1 : 0;
    // HBM is read in 128-B lines here (measured: sector-sparse loads still move whole lines),
    // so the sparse gather only pays when whole lines of the row stay untouched.  Multi-app
    // batches stream on the TMA ring with a blocked schedule (cfg4, B200: f32 2.38 ms vs
    // 2.96 ms gather, bf16 1.42 ms vs 5.17 ms).
    const int64_t lines_row = (static_cast<int64_t>(std::max(ctx->ncols, 1)) * elt + 127) / 128;
    const double frac = static_cast<double>(ctx->touched_lines[dt]) / (static_cast<double>(lines_row) * ctx->n_apps);
    bool gather = ctx->max_ent <= 1024 && frac <= gather_threshold(ctx->n_apps);
    if (kenv && std::string(kenv) == "tma") gather = false;
    if (kenv && std::string(kenv) == "gather" && ctx->max_ent <= 1024) gather = true;
    if (pat) {
      // per-list maxima: on the TMA ring with lane-resident entries, or on the gather kernel
      // (always when rows are wider than a stage allows)
      if (ctx->max_ent > 1024)
        return fail(SC_ERR_UNSUPPORTED, "this decision pattern supports at most 1024 mapped labels per app");
      // B200 cfg2: application-choice f32 0.77 ms (TMA slots) vs 0.83 ms (gather), bf16 0.55 ms;
      // Multi-Select f32 0.89 vs 0.86 ms; cfg4 f32 application-choice 2.98 vs 3.34 ms
      gather = !lane_ok;
      if (kenv && std::string(kenv) == "tma" && lane_ok) gather = false;
      if (kenv && std::string(kenv) == "gather") gather = true;
    }
    if (gather) {
      p.ld_flavor = std::getenv("SC_LD_FLAVOR") ? std::atoi(std::getenv("SC_LD_FLAVOR")) : 0;
      if (const char* g = std::getenv("SC_L2_FETCH")) {  // experiment: L2 fetch granularity hint (bytes)
        static int applied = -1;
        const int v = std::atoi(g);
        if (v != applied) {
          cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(v));
          applied = v;
        }
      }
      int epl = 1;
      while (epl * 32 < ctx->max_ent) epl *= 2;
      p.wtab_off = (want_loss && w && ctx->n_apps == 1) ? 0 : -1;
      const int pat = ctx->order == SC_ORDER_API_OUTPUT ? 0 : 1;
      if (cudaError_t e = sc::launch_gather(p, epl, pat, di.sms, st)) return cuda_fail(e, "gather kernel launch");
      g_last_kernel = (pat ? "gather_lists_epl" : "gather_epl") + std::to_string(epl);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return SC_OK;
    }
  }
  // ---- schedule: stage = R rows (or R row-chunks) in shared memory
  const int W = sc::kConsumerWarps;
  const int64_t stage_cap = 64 * 1024;
  p.copy_row_bytes = static_cast<int32_t>(round_up(static_cast<int64_t>(std::max(ctx->ncols, 1)) * elt, 16));
  // mapped labels in registers when whole rows fit a stage and |W| <= 1024
  int epl = 0;
  // Lane-resident entries cut the per-row instruction count (bf16 cfg2: 1.6x faster than the
  // shared list); with the batch epilogue moved after the stage release they also stream
  // f32 cfg2 fastest (0.592 vs 0.625 ms, 7.09 TB/s), so they are the default wherever whole
  // rows fit a stage.  SC_EPL=0 forces the shared-list path.
  if (lane_ok) epl = pat ? std::max(1, ctx->max_slots) : sc::eval_epl_for(ctx->max_ent);
  int launch_pat = pat;
  if (ac2) {
    epl = sc::eval_epl_for(ctx->max_ent);
    launch_pat = 3;
  }
  if (dm) {
    epl = dm_nv;
    launch_pat = 2;
    p.dm_full = 1;  // nv = ceil(n / (32 kVec)): every group but the last lies inside the row
  }
  int64_t logits_region;
  p.ng = 1;
  if (epl > 0) {
    // ~16 rows per stage: rpw rows per warp (about 4 KB of logits per warp), NG = min(4, rpw)
    // groups of W/NG warps; a group releases its stage as soon as its own warps are done.
    int64_t rpw = 1;
    while (rpw < 32 && 2 * rpw * p.ld_bytes <= 4096) rpw *= 2;
    p.ng = static_cast<int32_t>(std::min<int64_t>(4, rpw));
    // the per-list slot path (Multi-Select): two groups of 8 warps on 8-row stages — a warp's
    // long batch epilogue then holds back only its group's stages (same box: 0.680 -> 0.663 ms
    // on cfg2, profiles/r5k_*; the split-maxima paths are best with one group)
    if (launch_pat == 1 && p.ng == 1) p.ng = 2;
    if (const char* ng_env = std::getenv("SC_NG")) p.ng = std::atoi(ng_env);
    if (p.ng != 1 && p.ng != 2 && p.ng != 4 && p.ng != 8 && p.ng != 16) p.ng = 1;
    const int wg = W / p.ng;
    if (stage_kb_override()) rpw = std::max<int64_t>(1, std::min<int64_t>(32, stage_kb_override() * 1024 / (wg * p.ld_bytes)));
    p.R = static_cast<int32_t>(wg * rpw);
    p.nchunks = 1;
    p.chunk_bytes = static_cast<int32_t>(p.ld_bytes);
    p.chunk_elems = static_cast<int32_t>(b->ld);
    logits_region = p.R * p.ld_bytes;
  } else if (whole_rows) {
    const int64_t cap = (stage_kb_override() ? stage_kb_override() : 64) * 1024;
    const int64_t rpw = std::max<int64_t>(1, std::min<int64_t>(16, cap / (W * p.ld_bytes)));
    p.R = static_cast<int32_t>(W * rpw);
    p.nchunks = 1;
    p.chunk_bytes = static_cast<int32_t>(p.ld_bytes);
    p.chunk_elems = static_cast<int32_t>(b->ld);
    logits_region = p.R * p.ld_bytes;
  } else {
    p.R = W;
    p.chunk_bytes = static_cast<int32_t>((force_chunk ? force_chunk : stage_cap / W) / 16 * 16);
    p.chunk_elems = static_cast<int32_t>(p.chunk_bytes / elt);
    p.nchunks = static_cast<int32_t>((p.copy_row_bytes + p.chunk_bytes - 1) / p.chunk_bytes);
    logits_region = static_cast<int64_t>(p.R) * p.chunk_bytes;
  }
  p.nunits = (b->rows + p.R - 1) / p.R;
  p.mask_off = static_cast<int32_t>(round_up(logits_region, 128));
  p.app_off = static_cast<int32_t>(p.mask_off + round_up(p.R + 32, 16));
  p.stage_bytes = static_cast<int32_t>(round_up(p.app_off + round_up(2 * p.R + 32, 16), 128));

  // entries: in registers (epl > 0), else one shared list (1 app), per-warp slots
  // (several apps), or straight from global
  int64_t ent_bytes = 0;
  p.pmtab_off = -1;
  p.pmtab_bits = 0;
  int64_t pmtab_bytes = 0;
  if (epl > 0) {
    p.ent_mode = 3;  // lane registers
    if (ctx->n_apps == 1 && launch_pat != 1) {
      p.pmtab_bits = ctx->nlists[0];
      // pat 3: two masks per k = 0..D' (list k, lists before k); else one per G value
      pmtab_bytes = launch_pat == 3 ? static_cast<int64_t>(p.pmtab_bits + 1) * 2 * 32 * 4
                                    : (int64_t(1) << p.pmtab_bits) * 32 * 4;
    }
  } else if (ctx->n_apps == 1 && static_cast<int64_t>(ctx->max_ent) * 4 <= 64 * 1024) {
    p.ent_mode = 0;
    ent_bytes = round_up(static_cast<int64_t>(ctx->max_ent) * 4, 128);
  } else if (ctx->n_apps > 1 && static_cast<int64_t>(W) * ctx->max_ent * 4 <= 48 * 1024) {
    p.ent_mode = 1;
    p.ent_slot = ctx->max_ent;
    ent_bytes = round_up(static_cast<int64_t>(W) * ctx->max_ent * 4, 128);
  } else {
    p.ent_mode = 2;
  }
  const bool wtab = want_loss && w && ctx->n_apps == 1;
  const int64_t max_stages = epl > 0 ? 32 : 8;
  // dense-mapped rows read whole 512-B groups: up to 511 B past a row's last column
  const int64_t dm_slack = launch_pat == 2 ? 512 : 0;
  // dense gradient on the whole-row paths with two arg maxima per row: per-warp slabs where the
  // batch's gradient rows wait to be written between stages (sc_device.cuh dense_pair_rows)
  const int64_t pend_bytes = (grad_dense && epl > 0 && epl <= 8 && (launch_pat == 0 || launch_pat == 3))
                                 ? static_cast<int64_t>(W) * sc::kPendSlab : 0;  // eval_kernel<..., DEFER>
  const int64_t other = ent_bytes + pmtab_bytes + (wtab ? 1024 : 0) + pend_bytes + (2 * 8 + 32) * max_stages + 256 + dm_slack;
  int64_t S = (static_cast<int64_t>(kSmemMax) - other) / p.stage_bytes;
  if (S > max_stages) S = max_stages;
  S -= S % p.ng;  // stage s always belongs to group s % ng
  if (S < 2 * p.ng) return fail(SC_ERR_UNSUPPORTED, "row too large for the shared-memory pipeline");
  p.stages = static_cast<int32_t>(S);
  int64_t off = S * p.stage_bytes;
  p.ent_smem_off = static_cast<int32_t>(off);
  off += ent_bytes;
  if (pmtab_bytes) {
    p.pmtab_off = static_cast<int32_t>(off);
    off += pmtab_bytes;
  }
  p.wtab_off = wtab ? static_cast<int32_t>(off) : -1;
  off += wtab ? 1024 : 0;
  p.pend_off = pend_bytes ? static_cast<int32_t>(round_up(off, 16)) : -1;
  if (pend_bytes) off = p.pend_off + pend_bytes;
  p.bar_off = static_cast<int32_t>(round_up(off, 16));
  p.hdr_off = static_cast<int32_t>(p.bar_off + 2 * 8 * S);  // unit headers, 32 B per stage (16-B aligned)
  off = p.hdr_off + 32 * S + dm_slack;
  const size_t smem = static_cast<size_t>(off);

  p.split_copy = std::getenv("SC_SPLIT_COPY") ? 1 : 0;
  p.no_evict_first = std::getenv("SC_NO_EVICT_FIRST") ? 1 : 0;
  // Unit schedule: round-robin for one application; one contiguous block of units per CTA
  // when rows carry application ids.  With round-robin every CTA works inside the same
  // application at once and cfg4 (contiguous 2^18-row blocks per app) ran at half the
  // bandwidth (bf16 2.90 ms vs 1.42 ms blocked, f32 3.56 vs 2.38 ms, B200).
  p.blocked = std::getenv("SC_BLOCKED") ? std::atoi(std::getenv("SC_BLOCKED")) : (b->app ? 1 : 0);
  const int grid = static_cast<int>(std::min<int64_t>(p.nunits, di.sms));
  if (cudaError_t e = sc::launch_eval(p, epl, launch_pat, grid, smem, st)) return cuda_fail(e, "eval kernel launch");
  g_last_kernel = epl ? (launch_pat == 3   ? "tma_ring_appchoice_epl"
                         : launch_pat == 2 ? "tma_ring_dense_nv"
                         : launch_pat      ? "tma_ring_lists_epl"
                                           : "tma_ring_epl") +
                            std::to_string(epl)
                      : "tma_ring_list";
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return SC_OK;
}

}  // namespace

namespace sc {
sc_status set_error(sc_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}
void note_launch(const char* kernel) {
  g_last_kernel = kernel;
  g_launches.fetch_add(1, std::memory_order_relaxed);
}
int device_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  return device_info(dev).sms;
}
}  // namespace sc

extern "C" {

static sc_status load_context(int32_t C, int32_t n_apps, const int32_t* n_lists, const int64_t* list_off,
                              const int32_t* list_labels, float tau, float k, sc_order order, bool compact,
                              sc_context* out) {
  if (!out) return fail(SC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (order != SC_ORDER_API_OUTPUT && order != SC_ORDER_APP_CHOICE && order != SC_ORDER_MULTI_SELECT)
    return fail(SC_ERR_INVALID_ARG, "unknown order %d", (int)order);
  if (C < 1 || C >= (1 << 23)) return fail(SC_ERR_INVALID_ARG, "C must be in [1, 2^23)");
  if (n_apps < 1 || n_apps > 65535) return fail(SC_ERR_INVALID_ARG, "n_apps must be in [1, 65535]");
  if (!n_lists || !list_off) return fail(SC_ERR_INVALID_ARG, "n_lists / list_off is NULL");
  if (!std::isfinite(tau)) return fail(SC_ERR_INVALID_ARG, "tau must be finite");
  if (!(k > 0.f) || !std::isfinite(k)) return fail(SC_ERR_INVALID_ARG, "k must be finite and > 0");
  // validate the CSR
  int64_t base = 0, total = 0;
  for (int32_t a = 0; a < n_apps; ++a) {
    if (n_lists[a] < 0 || n_lists[a] > 8) return fail(SC_ERR_INVALID_ARG, "n_lists[%d] = %d not in [0, 8]", a, n_lists[a]);
    for (int32_t j = 0; j < n_lists[a]; ++j) {
      if (list_off[base + j + 1] < list_off[base + j]) return fail(SC_ERR_INVALID_ARG, "list_off not non-decreasing (app %d)", a);
    }
    if (n_lists[a] > 0 && list_off[base] < 0) return fail(SC_ERR_INVALID_ARG, "negative list_off");
    total = std::max<int64_t>(total, list_off[base + n_lists[a]]);
    base += n_lists[a] + 1;
  }
  if (total > 0 && !list_labels) return fail(SC_ERR_INVALID_ARG, "list_labels is NULL");

  auto* ctx = new sc_context_s();
  ctx->C = C;
  ctx->n_apps = n_apps;
  ctx->tau = tau;
  ctx->k = k;
  ctx->theta = static_cast<float>(1.0 / (1.0 + std::exp(-static_cast<double>(tau))));
  ctx->nlists.assign(n_lists, n_lists + n_apps);
  ctx->order = static_cast<int32_t>(order);
  const bool ms = order == SC_ORDER_MULTI_SELECT;
  // a1: Multi-Choice: cat[app][c] = first list, in code order, containing c (the listing's
  // if-chain); Multi-Select: the mask of every list containing c.
  std::vector<uint8_t> cat(static_cast<size_t>(n_apps) * C, ms ? uint8_t(0) : sc::kCatNone);
  std::vector<uint32_t> ent;
  std::vector<int32_t> ent_off(n_apps + 1, 0);
  base = 0;
  for (int32_t a = 0; a < n_apps; ++a) {
    uint8_t* ca = cat.data() + static_cast<size_t>(a) * C;
    for (int32_t j = 0; j < n_lists[a]; ++j) {
      for (int64_t t = list_off[base + j]; t < list_off[base + j + 1]; ++t) {
        const int32_t c = list_labels[t];
        if (c < 0 || c >= C) {
          delete ctx;
          return fail(SC_ERR_INVALID_ARG, "label %d of app %d list %d not in [0, C)", c, a, j);
        }
        if (ms) ca[c] |= static_cast<uint8_t>(1u << j);
        else if (ca[c] == sc::kCatNone) ca[c] = static_cast<uint8_t>(j);
      }
    }
    base += n_lists[a] + 1;
    const uint8_t none = ms ? uint8_t(0) : sc::kCatNone;
    for (int32_t c = 0; c < C; ++c)
      if (ca[c] != none) ent.push_back(static_cast<uint32_t>(c) << 8 | ca[c]);
    ent_off[a + 1] = static_cast<int32_t>(ent.size());
    for (int dt = 0; dt < 2; ++dt) {
      const int per_sector = dt == 0 ? 8 : 16;
      int64_t last = -1, last_line = -1;
      for (int32_t c = 0; c < C; ++c)
        if (ca[c] != none) {
          if (c / per_sector != last) {
            last = c / per_sector;
            ++ctx->touched_sectors[dt];
          }
          if (c / (4 * per_sector) != last_line) {
            last_line = c / (4 * per_sector);
            ++ctx->touched_lines[dt];
          }
        }
    }
    ctx->n_mapped.push_back(ent_off[a + 1] - ent_off[a]);
    ctx->max_ent = std::max(ctx->max_ent, ent_off[a + 1] - ent_off[a]);
  }
  ctx->ncols = C;
  if (compact) {
    // column-compacted rows: the union of the apps' mapped labels,
    // ascending, one logit column each; entry keys hold the column, so the arg max ties
    // (smaller key first) still break toward the smaller label
    std::vector<int32_t> pos(C, -1);
    for (uint32_t e : ent) pos[e >> 8] = 0;
    for (int32_t c = 0; c < C; ++c)
      if (pos[c] == 0) {
        pos[c] = static_cast<int32_t>(ctx->cols.size());
        ctx->cols.push_back(c);
      }
    for (uint32_t& e : ent) e = static_cast<uint32_t>(pos[e >> 8]) << 8 | (e & 0xFFu);
    ctx->ncols = static_cast<int32_t>(ctx->cols.size());
    ctx->compact = true;
    for (int dt = 0; dt < 2; ++dt) {  // touched sectors / lines of the compacted rows
      const int per_sector = dt == 0 ? 8 : 16;
      ctx->touched_sectors[dt] = ctx->touched_lines[dt] = 0;
      for (int32_t a = 0; a < n_apps; ++a) {
        int64_t last = -1, last_line = -1;
        for (int32_t e = ent_off[a]; e < ent_off[a + 1]; ++e) {
          const int64_t col = ent[e] >> 8;
          if (col / per_sector != last) {
            last = col / per_sector;
            ++ctx->touched_sectors[dt];
          }
          if (col / (4 * per_sector) != last_line) {
            last_line = col / (4 * per_sector);
            ++ctx->touched_lines[dt];
          }
        }
      }
    }
  }
  if (ent.empty()) ent.push_back(0);
  // per-list patterns: list-major slots (DevContext::lent) — list j's members in ascending
  // label order, padded to 32 entries per slot, so a warp reduces one list per slot
  std::vector<uint32_t> lent;
  std::vector<int32_t> lent_off(n_apps + 1, 0);
  std::vector<uint32_t> lslot(n_apps, 0);
  if (order != SC_ORDER_API_OUTPUT) {
    for (int32_t a = 0; a < n_apps; ++a) {
      int slots = 0;
      for (int32_t j = 0; j < n_lists[a]; ++j) {
        const size_t before = lent.size();
        for (int32_t e = ent_off[a]; e < ent_off[a + 1]; ++e)
          if (sc::label_lists(static_cast<uint8_t>(ent[e] & 0xFFu), order) >> j & 1u) lent.push_back(ent[e]);
        while ((lent.size() - before) % 32) lent.push_back(sc::kNone);
        for (size_t q = before; q < lent.size(); q += 32, ++slots)
          if (slots < 8) lslot[a] |= static_cast<uint32_t>(j) << (4 * slots);
      }
      lent_off[a + 1] = static_cast<int32_t>(lent.size());
      ctx->max_slots = std::max(ctx->max_slots, slots);
    }
  }
  if (lent.empty()) lent.push_back(sc::kNone);
  std::vector<uint8_t> nl(n_apps);
  for (int32_t a = 0; a < n_apps; ++a) nl[a] = static_cast<uint8_t>(n_lists[a]);

  cudaError_t e = cudaGetDevice(&ctx->device);
  if (!e) e = cudaMalloc(&ctx->d_cat, cat.size());
  if (!e) e = cudaMalloc(&ctx->d_ent, ent.size() * 4);
  if (!e) e = cudaMalloc(&ctx->d_ent_off, ent_off.size() * 4);
  if (!e) e = cudaMalloc(&ctx->d_nlists, nl.size());
  if (!e) e = cudaMalloc(&ctx->d_lent, lent.size() * 4);
  if (!e) e = cudaMalloc(&ctx->d_lent_off, lent_off.size() * 4);
  if (!e) e = cudaMalloc(&ctx->d_lslot, lslot.size() * 4);
  if (!e) e = cudaMemcpy(ctx->d_lent, lent.data(), lent.size() * 4, cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(ctx->d_lent_off, lent_off.data(), lent_off.size() * 4, cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(ctx->d_lslot, lslot.data(), lslot.size() * 4, cudaMemcpyHostToDevice);
  if (!e) e = cudaMalloc(&ctx->d_done, sizeof(unsigned int) * sc_context_s::kDonePool);
  std::vector<uint8_t> catT(static_cast<size_t>(n_apps) * C);
  for (int32_t a = 0; a < n_apps; ++a)
    for (int32_t c = 0; c < C; ++c) catT[static_cast<size_t>(c) * n_apps + a] = cat[static_cast<size_t>(a) * C + c];
  ctx->n_ent_total = ent_off[n_apps];
  if (!e) e = cudaMalloc(&ctx->d_catT, catT.size());
  if (!e) e = cudaMemcpy(ctx->d_catT, catT.data(), catT.size(), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemset(ctx->d_done, 0, sizeof(unsigned int) * sc_context_s::kDonePool);
  {  // all-apps, lane per application: applications by |W_a| descending, 32 per group,
     // each group's entries transposed and padded to its largest application
    std::vector<int32_t> perm(n_apps);
    for (int32_t a = 0; a < n_apps; ++a) perm[a] = a;
    std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) {
      return ent_off[x + 1] - ent_off[x] > ent_off[y + 1] - ent_off[y];
    });
    const int32_t ng = (n_apps + 31) / 32;
    std::vector<int32_t> goff(ng + 1, 0);
    std::vector<uint16_t> aperm(static_cast<size_t>(ng) * 32, 0xFFFF);
    for (int32_t g = 0; g < ng; ++g) {
      const int32_t a0 = perm[32 * g];
      goff[g + 1] = goff[g] + 32 * (ent_off[a0 + 1] - ent_off[a0]);
      for (int l = 0; l < 32 && 32 * g + l < n_apps; ++l) aperm[32 * g + l] = static_cast<uint16_t>(perm[32 * g + l]);
    }
    // keys column << 8 | (1 << list) (the kernel's class test is one AND with G); padding
    // entries: the row buffer's -inf slot (column round_up(C, 8), past the bytes a row copy
    // writes for f32 and bf16) and no list bit
    const uint32_t dummy = static_cast<uint32_t>((C + 7) / 8 * 8) << 8;
    std::vector<uint32_t> aent(std::max<int32_t>(goff[ng], 1), dummy);
    for (int32_t g = 0; g < ng; ++g)
      for (int l = 0; l < 32 && 32 * g + l < n_apps; ++l) {
        const int32_t a = perm[32 * g + l];
        for (int32_t t = ent_off[a]; t < ent_off[a + 1]; ++t)
          aent[goff[g] + 32 * (t - ent_off[a]) + l] = (ent[t] & ~0xFFu) | (1u << (ent[t] & 0xFFu));
      }
    ctx->aa_groups = ng;
    ctx->aa_ent_total = goff[ng];
    if (!e) e = cudaMalloc(&ctx->d_aa_ent, aent.size() * 4);
    if (!e) e = cudaMalloc(&ctx->d_aa_goff, goff.size() * 4);
    if (!e) e = cudaMalloc(&ctx->d_aa_perm, aperm.size() * 2);
    if (!e) e = cudaMemcpy(ctx->d_aa_ent, aent.data(), aent.size() * 4, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(ctx->d_aa_goff, goff.data(), goff.size() * 4, cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(ctx->d_aa_perm, aperm.data(), aperm.size() * 2, cudaMemcpyHostToDevice);
    if (C <= sc::kTRMaxC) {  // lane per row: word offsets of the columns in the transposed unit
      std::vector<int32_t> toff(n_apps + 1, 0);
      for (int32_t a = 0; a < n_apps; ++a) toff[a + 1] = toff[a] + (ent_off[a + 1] - ent_off[a] + 3) / 4 * 4;
      const uint16_t pad = static_cast<uint16_t>(sc::kTRStride * C);
      std::vector<uint16_t> tkey(std::max<int32_t>(toff[n_apps], 4), pad);
      for (int32_t a = 0; a < n_apps; ++a)
        for (int32_t t = ent_off[a]; t < ent_off[a + 1]; ++t) {
          tkey[toff[a] + t - ent_off[a]] = static_cast<uint16_t>(sc::kTRStride * (ent[t] >> 8));
        }
      ctx->tr_total = static_cast<int32_t>(tkey.size());
      if (!e) e = cudaMalloc(&ctx->d_tr_key, tkey.size() * 2);
      if (!e) e = cudaMalloc(&ctx->d_tr_off, toff.size() * 4);
      if (!e) e = cudaMemcpy(ctx->d_tr_key, tkey.data(), tkey.size() * 2, cudaMemcpyHostToDevice);
      if (!e) e = cudaMemcpy(ctx->d_tr_off, toff.data(), toff.size() * 4, cudaMemcpyHostToDevice);
    }
  }
  if (!e) e = cudaMemcpy(ctx->d_cat, cat.data(), cat.size(), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(ctx->d_ent, ent.data(), ent.size() * 4, cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(ctx->d_ent_off, ent_off.data(), ent_off.size() * 4, cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(ctx->d_nlists, nl.data(), nl.size(), cudaMemcpyHostToDevice);
  if (!e && compact && !ctx->cols.empty()) {
    e = cudaMalloc(&ctx->d_col_label, ctx->cols.size() * 4);
    if (!e) e = cudaMemcpy(ctx->d_col_label, ctx->cols.data(), ctx->cols.size() * 4, cudaMemcpyHostToDevice);
  }
  if (e) {
    sc_context_free(ctx);
    return cuda_fail(e, "context upload");
  }
  *out = ctx;
  return SC_OK;
}

sc_status sc_context_free(sc_context ctx) {
  if (!ctx) return SC_OK;
  cudaFree(ctx->d_cat);
  cudaFree(ctx->d_ent);
  cudaFree(ctx->d_ent_off);
  cudaFree(ctx->d_lent);
  cudaFree(ctx->d_lent_off);
  cudaFree(ctx->d_lslot);
  cudaFree(ctx->d_nlists);
  cudaFree(ctx->d_done);
  cudaFree(ctx->d_catT);
  cudaFree(ctx->d_aa_ent);
  cudaFree(ctx->d_aa_goff);
  cudaFree(ctx->d_aa_perm);
  cudaFree(ctx->d_tr_key);
  cudaFree(ctx->d_tr_off);
  cudaFree(ctx->d_col_label);
  delete ctx;
  return SC_OK;
}

sc_status sc_context_load(int32_t C, int32_t n_apps, const int32_t* n_lists, const int64_t* list_off,
                          const int32_t* list_labels, float tau, float k, sc_order order, sc_context* out) {
  return load_context(C, n_apps, n_lists, list_off, list_labels, tau, k, order, false, out);
}

sc_status sc_context_load_compact(int32_t C, int32_t n_apps, const int32_t* n_lists, const int64_t* list_off,
                                  const int32_t* list_labels, float tau, float k, sc_order order, sc_context* out) {
  return load_context(C, n_apps, n_lists, list_off, list_labels, tau, k, order, true, out);
}

sc_status sc_context_columns(sc_context ctx, int32_t* cols, int32_t* n_cols) {
  if (!ctx) return fail(SC_ERR_INVALID_ARG, "ctx is NULL");
  if (n_cols) *n_cols = ctx->ncols;
  if (cols)
    for (int32_t j = 0; j < ctx->ncols; ++j) cols[j] = ctx->compact ? ctx->cols[j] : j;
  return SC_OK;
}

sc_status sc_context_info(sc_context ctx, int32_t app, int32_t* n_lists, int32_t* n_mapped) {
  if (!ctx) return fail(SC_ERR_INVALID_ARG, "ctx is NULL");
  if (app < 0 || app >= ctx->n_apps) return fail(SC_ERR_INVALID_ARG, "app out of range");
  if (n_lists) *n_lists = ctx->nlists[app];
  if (n_mapped) *n_mapped = ctx->n_mapped[app];
  return SC_OK;
}

sc_status sc_context_order(sc_context ctx, sc_order* order, int32_t* grad_slots) {
  if (!ctx) return fail(SC_ERR_INVALID_ARG, "ctx is NULL");
  if (order) *order = static_cast<sc_order>(ctx->order);
  if (grad_slots) *grad_slots = ctx->order == SC_ORDER_MULTI_SELECT ? 8 : 2;
  return SC_OK;
}

sc_status sc_decide(sc_context ctx, const sc_batch* batch, uint8_t* decision, uint64_t* n_incorrect,
                    uint64_t* hist_pred, uint64_t* hist_gt, sc_stream stream) {
  return run_eval(ctx, batch, nullptr, 1.f, nullptr, nullptr, nullptr, nullptr, nullptr, decision, n_incorrect,
                  hist_pred, hist_gt, false, static_cast<cudaStream_t>(stream));
}

sc_status sc_loss_fwd_bwd(sc_context ctx, const sc_batch* batch, const float* w, float grad_scale, double* loss_sum,
                          float* loss_row, int32_t* grad_idx, float* grad_val, float* grad_dense, uint8_t* decision,
                          uint64_t* n_incorrect, uint64_t* hist_pred, uint64_t* hist_gt, sc_stream stream) {
  return run_eval(ctx, batch, w, grad_scale, loss_sum, loss_row, grad_idx, grad_val, grad_dense, decision,
                  n_incorrect, hist_pred, hist_gt, true, static_cast<cudaStream_t>(stream));
}

// The fused pre-pass's completion counter for `stream`: a slot of the context's pool owned
// by that stream from its first use on (nullptr once the pool is exhausted).
static unsigned int* done_counter_for(sc_context ctx, sc_stream stream) {
  std::lock_guard<std::mutex> lock(ctx->done_mu);
  auto& v = ctx->done_streams;
  for (size_t i = 0; i < v.size(); ++i)
    if (v[i] == stream) return ctx->d_done + i;
  if (static_cast<int>(v.size()) == sc_context_s::kDonePool) return nullptr;
  v.push_back(stream);
  return ctx->d_done + (v.size() - 1);
}

static sc_status run_hist(sc_context ctx, const sc_batch* b, uint64_t* hist_gt, uint8_t* gt_mask_out, float* w_out,
                          sc_stream stream) {
  if (sc_status s = check_batch_common(ctx, b)) return s;
  if (!b->gt_off || !b->gt_lab) return fail(SC_ERR_INVALID_ARG, "sc_decision_hist needs gt_off and gt_lab");
  if (w_out && !hist_gt) return fail(SC_ERR_INVALID_ARG, "weights need hist_gt");
  if (b->rows == 0 && w_out) return sc_weights_from_hist(ctx, hist_gt, w_out, stream);  // w of the histogram as is
  if (b->rows == 0 || (!hist_gt && !gt_mask_out)) return SC_OK;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_fail(e, "cudaGetDevice");
  if (dev != ctx->device) return fail(SC_ERR_INVALID_ARG, "context belongs to device %d, current is %d", ctx->device, dev);
  DeviceInfo& di = device_info(dev);
  sc::HistParams p{};
  p.ctx = dev_ctx(ctx);
  p.rows = b->rows;
  p.gt_off = b->gt_off;
  p.gt_lab = b->gt_lab;
  p.app = b->app;
  p.hist_gt = reinterpret_cast<unsigned long long*>(hist_gt);
  p.gt_mask_out = gt_mask_out;
  p.w_out = w_out;
  p.done_counter = w_out ? done_counter_for(ctx, stream) : nullptr;
  if (w_out && !p.done_counter) {  // more streams than counters: two launches (hist, then weights)
    if (sc_status s = run_hist(ctx, b, hist_gt, gt_mask_out, nullptr, stream)) return s;
    return sc_weights_from_hist(ctx, hist_gt, w_out, stream);
  }
  const size_t hbytes = static_cast<size_t>(ctx->n_apps) * 256 * 8;
  p.smem_hist = hbytes <= 32 * 1024;
  // single application: one row per thread, the category table in shared memory
  const char* hk = std::getenv("SC_HIST");
  const bool rows_kernel = ctx->n_apps == 1 && ctx->C <= 128 * 1024 && !(hk && std::string(hk) == "warp");
  if (rows_kernel) {
    const char* gps = std::getenv("SC_HIST_CTAS_PER_SM");  // experiment knob (default 8)
    const int64_t per_sm = gps ? std::max(1, std::atoi(gps)) : 8;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((b->rows + 255) / 256, static_cast<int64_t>(di.sms) * per_sm));
    if (cudaError_t e = sc::launch_hist_rows(p, static_cast<int>(blocks), static_cast<cudaStream_t>(stream)))
      return cuda_fail(e, "hist kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SC_OK;
  }
  const int64_t per_block = 8 * 32 * 2;  // 8 warps x kHB blocks of 32 rows
  // persistent: one wave (3 CTAs/SM at <= 85 registers), warps loop with a prefetch pipeline
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((b->rows + per_block - 1) / per_block,
                                                                static_cast<int64_t>(di.sms) * 3));
  if (cudaError_t e = sc::launch_hist(p, static_cast<int>(blocks), p.smem_hist ? hbytes : 0,
                                      static_cast<cudaStream_t>(stream)))
    return cuda_fail(e, "hist kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return SC_OK;
}

sc_status sc_decision_hist(sc_context ctx, const sc_batch* b, uint64_t* hist_gt, uint8_t* gt_mask_out,
                           sc_stream stream) {
  return run_hist(ctx, b, hist_gt, gt_mask_out, nullptr, stream);
}

sc_status sc_decision_hist_weights(sc_context ctx, const sc_batch* b, uint64_t* hist_gt, uint8_t* gt_mask_out,
                                   float* w, sc_stream stream) {
  if (!w) return fail(SC_ERR_INVALID_ARG, "w is NULL");
  return run_hist(ctx, b, hist_gt, gt_mask_out, w, stream);
}

sc_status sc_decide_all_apps(sc_context ctx, const sc_batch* b, uint64_t* n_incorrect, uint64_t* hist_pred,
                             uint8_t* decision, sc_stream stream) {
  if (sc_status s = check_batch_common(ctx, b)) return s;
  if (ctx->order != SC_ORDER_API_OUTPUT)
    return fail(SC_ERR_UNSUPPORTED, "sc_decide_all_apps supports the API-output order");
  if (ctx->compact) return fail(SC_ERR_UNSUPPORTED, "sc_decide_all_apps reads dense rows (column c = label c)");
  if (!b->gt_off || !b->gt_lab) return fail(SC_ERR_INVALID_ARG, "sc_decide_all_apps needs gt_off and gt_lab");
  if (b->dtype != SC_F32 && b->dtype != SC_BF16) return fail(SC_ERR_INVALID_ARG, "unknown dtype");
  if (b->rows == 0) return SC_OK;
  if (!b->logits) return fail(SC_ERR_INVALID_ARG, "logits is NULL");
  const int64_t elt = b->dtype == SC_F32 ? 4 : 2;
  if (b->ld < ctx->C || (b->ld * elt) % 16 || reinterpret_cast<uintptr_t>(b->logits) % 16)
    return fail(SC_ERR_INVALID_ARG, "bad logits layout (ld >= C, ld*elt %% 16 == 0, 16-B aligned)");
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return cuda_fail(e, "cudaGetDevice");
  if (dev != ctx->device) return fail(SC_ERR_INVALID_ARG, "context belongs to another device");
  DeviceInfo& di = device_info(dev);
  sc::AllAppsParams p{};
  p.ctx = dev_ctx(ctx);
  p.catT = ctx->d_catT;
  p.logits = static_cast<const uint8_t*>(b->logits);
  p.rows = b->rows;
  p.ld_bytes = b->ld * elt;
  p.bf16 = b->dtype == SC_BF16;
  p.copy_bytes = static_cast<uint32_t>(round_up(static_cast<int64_t>(ctx->C) * elt, 16));
  p.n_ent_total = ctx->n_ent_total;
  p.gt_off = b->gt_off;
  p.gt_lab = b->gt_lab;
  p.n_incorrect = reinterpret_cast<unsigned long long*>(n_incorrect);
  p.hist_pred = reinterpret_cast<unsigned long long*>(hist_pred);
  p.decision = decision;
  const int64_t A = ctx->n_apps;
  const char* aa_env = std::getenv("SC_ALLAPPS");
  const std::string aa_mode = aa_env ? aa_env : "";
  if (aa_mode.empty() && ctx->d_tr_key) {
    // lane per row: the unit transposed in shared memory ([C+1] columns of kTRStride words),
    // G / decision tile [A][kTRRows], counters [A] + [A][16], D' [A]
    p.tr_key = ctx->d_tr_key;
    p.tr_off = ctx->d_tr_off;
    p.aa_perm = ctx->d_aa_perm;
    p.tr_total = ctx->tr_total;
    const int64_t o = round_up(4 * static_cast<int64_t>(sc::kTRStride) * (ctx->C + 1) + sc::kTRRows * A + 4 * A + 64 * A + A, 16) +
                      2 * static_cast<int64_t>(ctx->tr_total) + 4 * (A + 1) + 2 * A;  // + entries, offsets, order
    const size_t sm = static_cast<size_t>(round_up(o, 16));
    if (sm <= kSmemMax) {
      const int grid = static_cast<int>(std::min<int64_t>((b->rows + sc::kTRRows - 1) / sc::kTRRows, di.sms));
      if (cudaError_t e = sc::launch_all_apps_rows(p, grid, sm, static_cast<cudaStream_t>(stream)))
        return cuda_fail(e, "all-apps kernel launch");
      g_last_kernel = "all_apps_rows";
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return SC_OK;
    }
  }
  if (aa_mode != "warp") {
    // lane per application: [2 units x R] row buffers (each with a -inf slot at column C),
    // transposed entries, group offsets, perm, counters, G [2][R][A], D'
    p.aa_ent = ctx->d_aa_ent;
    p.aa_goff = ctx->d_aa_goff;
    p.aa_perm = ctx->d_aa_perm;
    p.n_groups = ctx->aa_groups;
    p.aa_ent_total = ctx->aa_ent_total;
    p.dummy_key = static_cast<uint32_t>((ctx->C + 7) / 8 * 8) << 8;
    p.row_bytes_pad = static_cast<int32_t>(round_up(static_cast<int64_t>((ctx->C + 7) / 8 * 8 + 1) * elt, 128));
    const int64_t ng = ctx->aa_groups;
    for (int R = 8; R >= 1; R /= 2) {
      int64_t o = 2 * R * static_cast<int64_t>(p.row_bytes_pad) + 4 * static_cast<int64_t>(p.aa_ent_total) +
                  4 * (ng + 1) + 64 * ng + 4 * A + 64 * A + 2 * R * A + A;
      o = round_up(o, 8);
      const size_t sm = static_cast<size_t>(o + 16);
      if (sm <= kSmemMax) {
        p.rows_per_unit = R;
        p.bar_off = static_cast<int32_t>(o);
        const int grid = static_cast<int>(std::min<int64_t>((b->rows + R - 1) / R, di.sms));
        if (cudaError_t e = sc::launch_all_apps_lane(p, grid, sm, static_cast<cudaStream_t>(stream)))
          return cuda_fail(e, "all-apps kernel launch");
        g_last_kernel = "all_apps_lane";
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return SC_OK;
      }
    }
    // contexts too large for the lane layout: the warp-per-application kernel below
  }
  p.row_bytes_pad = static_cast<int32_t>(round_up(p.copy_bytes, 128));
  // [2 units x kAARows] row buffers, entries, offsets, counters, G [2 units x kAARows][A], D'
  const int64_t ur = sc::kAllAppsRows;
  int64_t off = 2 * ur * static_cast<int64_t>(p.row_bytes_pad) + 4 * p.n_ent_total + 4 * (A + 1) + 4 * A + 64 * A +
                (2 * ur + 1) * A;
  p.bar_off = static_cast<int32_t>(round_up(off, 8));
  const size_t smem = static_cast<size_t>(p.bar_off + 16);
  if (smem > kSmemMax) return fail(SC_ERR_UNSUPPORTED, "contexts too large for the all-apps pass (shared memory)");
  const int grid = static_cast<int>(std::min<int64_t>((b->rows + ur - 1) / ur, di.sms));  // kAARows-row units
  if (cudaError_t e = sc::launch_all_apps(p, grid, smem, static_cast<cudaStream_t>(stream)))
    return cuda_fail(e, "all-apps kernel launch");
  g_last_kernel = "all_apps_warp";
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return SC_OK;
}

sc_status sc_weights_from_hist(sc_context ctx, const uint64_t* hist_gt, float* w, sc_stream stream) {
  if (!ctx) return fail(SC_ERR_INVALID_ARG, "ctx is NULL");
  if (!hist_gt || !w) return fail(SC_ERR_INVALID_ARG, "hist_gt / w is NULL");
  if (cudaError_t e = sc::launch_weights(reinterpret_cast<const unsigned long long*>(hist_gt), w, ctx->n_apps,
                                         static_cast<cudaStream_t>(stream)))
    return cuda_fail(e, "weights kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return SC_OK;
}

}  // extern "C"

struct sc_stager_s {
  int device = 0;
  int64_t chunk_bytes = 0;
  void* buf[2] = {nullptr, nullptr};
  cudaStream_t copy = nullptr;
  cudaEvent_t ready[2] = {nullptr, nullptr};  // chunk copied (copy stream)
  cudaEvent_t free_[2] = {nullptr, nullptr};  // the pass that read the buffer is done (caller's stream)
};

extern "C" {

sc_status sc_stager_create(int64_t chunk_bytes, sc_stager* out) {
  if (!out) return fail(SC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (chunk_bytes < 1) return fail(SC_ERR_INVALID_ARG, "chunk_bytes < 1");
  sc_stager s = new sc_stager_s;
  s->chunk_bytes = round_up(chunk_bytes, 256);
  cudaError_t e = cudaGetDevice(&s->device);
  for (int i = 0; i < 2 && !e; ++i) e = cudaMalloc(&s->buf[i], static_cast<size_t>(s->chunk_bytes));
  if (!e) e = cudaStreamCreateWithFlags(&s->copy, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && !e; ++i) e = cudaEventCreateWithFlags(&s->ready[i], cudaEventDisableTiming);
  for (int i = 0; i < 2 && !e; ++i) e = cudaEventCreateWithFlags(&s->free_[i], cudaEventDisableTiming);
  if (e) {
    sc_stager_free(s);
    return cuda_fail(e, "sc_stager_create");
  }
  *out = s;
  return SC_OK;
}

sc_status sc_stager_free(sc_stager s) {
  if (!s) return SC_OK;
  if (s->copy) cudaStreamSynchronize(s->copy);
  for (int i = 0; i < 2; ++i) {
    if (s->free_[i]) cudaEventSynchronize(s->free_[i]);
    cudaFree(s->buf[i]);
    if (s->ready[i]) cudaEventDestroy(s->ready[i]);
    if (s->free_[i]) cudaEventDestroy(s->free_[i]);
  }
  if (s->copy) cudaStreamDestroy(s->copy);
  delete s;
  return SC_OK;
}

sc_status sc_loss_fwd_bwd_host(sc_context ctx, sc_stager stg, const sc_batch* batch, int32_t mode, const float* w,
                               float grad_scale, double* loss_sum, float* loss_row, int32_t* grad_idx,
                               float* grad_val, float* grad_dense, uint8_t* decision, uint64_t* n_incorrect,
                               uint64_t* hist_pred, uint64_t* hist_gt, int32_t* mode_used, sc_stream stream) {
  if (sc_status s = check_batch_common(ctx, batch)) return s;
  if (mode < SC_HOST_AUTO || mode > SC_HOST_ZERO_COPY) return fail(SC_ERR_INVALID_ARG, "unknown host mode %d", mode);
  if (batch->dtype != SC_F32 && batch->dtype != SC_BF16) return fail(SC_ERR_INVALID_ARG, "unknown dtype");
  const int64_t elt = batch->dtype == SC_F32 ? 4 : 2;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  // page-locked host rows have a device address (UVA): the kernels can read them in place
  void* dev_alias = nullptr;
  if (batch->logits) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, batch->logits) == cudaSuccess && pa.type == cudaMemoryTypeHost)
      dev_alias = pa.devicePointer;
    cudaGetLastError();  // pageable memory reports an error on some drivers: not sticky
  }
  int32_t m = mode;
  if (m == SC_HOST_AUTO) {
    // zero copy pays where the gather kernel runs: whole 128-B lines of a row stay untouched
    // (B200, cfg3 f32: 1.46x over copy-then-compute); dense contexts copy
    const int dt = batch->dtype == SC_BF16 ? 1 : 0;
    const int64_t lines_row = (static_cast<int64_t>(std::max(ctx->ncols, 1)) * elt + 127) / 128;
    const double frac = static_cast<double>(ctx->touched_lines[dt]) / (static_cast<double>(lines_row) * ctx->n_apps);
    const bool sparse = ctx->max_ent <= 1024 && ctx->order == SC_ORDER_API_OUTPUT && frac <= gather_threshold(ctx->n_apps);
    m = (dev_alias && sparse) ? SC_HOST_ZERO_COPY : SC_HOST_COPY;
  }
  if (mode_used) *mode_used = m;
  if (m == SC_HOST_ZERO_COPY) {
    if (batch->rows > 0 && !dev_alias)
      return fail(SC_ERR_INVALID_ARG, "SC_HOST_ZERO_COPY needs page-locked host logits");
    sc_batch b = *batch;
    b.logits = dev_alias;
    return run_eval(ctx, &b, w, grad_scale, loss_sum, loss_row, grad_idx, grad_val, grad_dense, decision,
                    n_incorrect, hist_pred, hist_gt, true, st);
  }
  if (!stg) return fail(SC_ERR_INVALID_ARG, "SC_HOST_COPY needs a stager");
  if (batch->rows == 0) return run_eval(ctx, batch, w, grad_scale, loss_sum, loss_row, grad_idx, grad_val,
                                        grad_dense, decision, n_incorrect, hist_pred, hist_gt, true, st);
  if (!batch->logits) return fail(SC_ERR_INVALID_ARG, "logits is NULL");
  const int64_t row_bytes = batch->ld * elt;
  if (row_bytes <= 0 || row_bytes > stg->chunk_bytes)
    return fail(SC_ERR_INVALID_ARG, "a row (%lld B) is wider than the stager's chunk (%lld B)",
                (long long)row_bytes, (long long)stg->chunk_bytes);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != stg->device) return fail(SC_ERR_INVALID_ARG, "the stager belongs to device %d", stg->device);
  const int S = ctx->order == SC_ORDER_MULTI_SELECT ? 8 : 2;
  const int64_t chunk_rows = stg->chunk_bytes / row_bytes;
  // buffers are free once every earlier use on `stream` is done
  for (int i = 0; i < 2; ++i)
    if (cudaError_t e = cudaEventRecord(stg->free_[i], st)) return cuda_fail(e, "cudaEventRecord");
  const uint8_t* host = static_cast<const uint8_t*>(batch->logits);
  for (int64_t lo = 0, ci = 0; lo < batch->rows; lo += chunk_rows, ++ci) {
    const int64_t nr = std::min<int64_t>(chunk_rows, batch->rows - lo);
    const int k = static_cast<int>(ci & 1);
    cudaError_t e = cudaStreamWaitEvent(stg->copy, stg->free_[k], 0);
    if (!e) e = cudaMemcpyAsync(stg->buf[k], host + lo * row_bytes, static_cast<size_t>(nr * row_bytes),
                                cudaMemcpyHostToDevice, stg->copy);
    if (!e) e = cudaEventRecord(stg->ready[k], stg->copy);
    if (!e) e = cudaStreamWaitEvent(st, stg->ready[k], 0);
    if (e) return cuda_fail(e, "sc_loss_fwd_bwd_host: staging copy");
    sc_batch b = *batch;
    b.logits = stg->buf[k];
    b.rows = nr;
    b.gt_mask = batch->gt_mask ? batch->gt_mask + lo : nullptr;
    b.gt_off = batch->gt_mask ? nullptr : (batch->gt_off ? batch->gt_off + lo : nullptr);
    b.app = batch->app ? batch->app + lo : nullptr;
    if (sc_status s = run_eval(ctx, &b, w, grad_scale, loss_sum, loss_row ? loss_row + lo : nullptr,
                               grad_idx ? grad_idx + S * lo : nullptr, grad_val ? grad_val + S * lo : nullptr,
                               grad_dense ? grad_dense + lo * batch->ld : nullptr, decision ? decision + lo : nullptr,
                               n_incorrect, hist_pred, hist_gt, true, st))
      return s;
    if (cudaError_t e2 = cudaEventRecord(stg->free_[k], st)) return cuda_fail(e2, "cudaEventRecord");
  }
  return SC_OK;
}

const char* sc_last_error(void) { return g_err.c_str(); }

const char* sc_last_kernel(void) { return g_last_kernel.c_str(); }

uint64_t sc_launch_count(void) { return g_launches.load(); }

}  // extern "C"
