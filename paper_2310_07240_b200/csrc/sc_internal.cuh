// sc_internal.cuh — shared between the libsc host code and its sm_100a kernels.
// Not part of the ABI (include/sc.h is).  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sc {

constexpr int kConsumerWarps = 16;                 // W: consumer warps per CTA
constexpr int kThreads = 32 * (1 + kConsumerWarps);  // + 1 TMA producer warp
constexpr uint32_t kPendSlab = 16 + 32 * 8 + 32 * 16;  // per-warp parked dense-gradient rows (sc_device.cuh)
constexpr uint32_t kNone = 0xFFFFFFFFu;            // "no label" key
constexpr uint8_t kCatNone = 0xFF;                 // label in no list (Multi-Choice tables)

// Device-side context tables (built once by sc_context_load).
// Decision patterns (sc_order).
constexpr int kApiOutput = 0, kAppChoice = 1, kMultiSelect = 2;

struct DevContext {
  const uint8_t* cat;       // [n_apps*C]  Multi-Choice: first list containing label c, or kCatNone (a1);
                            //             Multi-Select: mask of every list containing c (0 = none)
  const uint32_t* ent;      // per app, mapped labels sorted by id: key = c << 8 | cat[c]
  const int32_t* ent_off;   // [n_apps+1]
  const uint8_t* nlists;    // [n_apps]  D'
  // per-list patterns (application-choice order, Multi-Select), list-major slots: per app,
  // list j's member labels (ascending keys) padded with kNone to a multiple of 32 — one
  // 32-entry slot per lane position, every slot inside one list
  const uint32_t* lent = nullptr;     // slot entries
  const int32_t* lent_off = nullptr;  // [n_apps+1]  (multiples of 32)
  const uint32_t* lslot = nullptr;    // [n_apps]  list of slot s in bits 4s..4s+3 (<= 8 slots)
  // column-compacted contexts (sc_context_load_compact): entry keys hold column positions,
  // col_label maps a position back to its label for the gradient indices; nullptr = dense
  const int32_t* col_label = nullptr;
  int32_t C, n_apps, max_ent;
  float tau, theta, k;
  int32_t order;            // kApiOutput / kAppChoice / kMultiSelect
};

// Label id reported for the logit column `pos` of an entry key (identity for dense rows).
__device__ __forceinline__ int32_t out_label(const DevContext& c, int32_t pos) {
  return (c.col_label != nullptr && pos >= 0) ? __ldg(c.col_label + pos) : pos;
}

// Lists (bit set) label-table value v stands for.
__host__ __device__ __forceinline__ uint32_t label_lists(uint8_t v, int order) {
  return order == kMultiSelect ? static_cast<uint32_t>(v) : (v == kCatNone ? 0u : (1u << v));
}

// Parameters of the fused evaluation kernel (decide + counters + loss fwd/bwd).
struct EvalParams {
  DevContext ctx;
  // batch
  const uint8_t* logits;    // byte pointer, rows of ld_bytes
  int64_t rows;
  int64_t ld;               // elements
  int64_t ld_bytes;
  int32_t bf16;             // 0: f32, 1: bf16
  const int64_t* gt_off;
  const int32_t* gt_lab;
  const uint8_t* gt_mask;
  const uint16_t* app;
  int32_t has_gt;
  // loss
  const float* w;
  float grad_scale;
  int32_t want_loss;
  // outputs (NULL = not wanted)
  double* loss_sum;
  float* loss_row;
  int32_t* grad_idx;
  float* grad_val;
  float* grad_dense;
  uint8_t* decision;
  unsigned long long* n_incorrect;
  unsigned long long* hist_pred;
  unsigned long long* hist_gt;
  // schedule (host-computed)
  int32_t R;                // rows per unit (multiple of kConsumerWarps)
  int32_t nchunks;          // column chunks per row (1: whole rows, R rows copied at once)
  int32_t chunk_bytes;      // bytes per row-chunk in smem (nchunks > 1)
  int32_t chunk_elems;
  int32_t copy_row_bytes;   // bytes of a row that carry labels 0..C-1, rounded up to 16
  int64_t nunits;
  int32_t stages;
  int32_t stage_bytes;
  int32_t mask_off;         // sideband offsets inside a stage
  int32_t app_off;
  int32_t ent_mode;         // 0: one shared smem list (n_apps==1), 1: per-warp smem slot, 2: global
  int32_t ent_smem_off;     // byte offset of entry storage
  int32_t ent_slot;         // entries per warp slot (mode 1)
  int32_t wtab_off;         // byte offset of smem weight table (n_apps==1 && w), or -1
  int32_t bar_off;          // byte offset of the mbarriers
  int32_t ng;               // consumer groups (stage i is consumed by group i % ng); 1 on the generic path
  int32_t pmtab_off;        // byte offset of the plus-mask table [2^pmtab_bits][32] (single app), or -1
  int32_t pmtab_bits;       // D' of the single app
  int32_t split_copy;       // experiment: one bulk copy per row instead of one per stage
  int32_t no_evict_first;   // experiment: L2 evict_normal instead of evict_first for the stream
  int32_t blocked;          // units: one contiguous block per CTA (1) or round-robin over CTAs (0)
  int32_t ld_flavor;        // gather kernel global-load cache flavour (see ldg_stream_f32)
  int32_t dm_full;          // dense-mapped rows (pat 2): groups 0..NV-2 fully inside the row's n columns
  int32_t pend_off;         // byte offset of the per-warp parked dense-gradient slabs (sc_device.cuh), or -1
  int32_t hdr_off;          // byte offset of the per-stage unit headers (32 B: r0, nr, side-band windows), or -1
};

struct HistParams {
  DevContext ctx;
  int64_t rows;
  const int64_t* gt_off;
  const int32_t* gt_lab;
  const uint16_t* app;
  unsigned long long* hist_gt;
  uint8_t* gt_mask_out;
  int32_t smem_hist;        // 1: CTA-private shared histogram (n_apps*256 counters)
  float* w_out;             // optional: weights from the finished histogram (last CTA)
  unsigned int* done_counter;  // zero between calls (reset by the last CTA)
};

// "One read, many contexts" (sc_allapps.cu).
struct AllAppsParams {
  DevContext ctx;
  const uint8_t* catT;      // [C][n_apps] label-major copy of the category table
  const uint8_t* logits;
  int64_t rows, ld_bytes;
  int32_t bf16;
  uint32_t copy_bytes;      // bytes of a row holding labels 0..C-1, rounded up to 16
  int32_t row_bytes_pad;    // row buffer stride in shared memory
  int32_t n_ent_total;      // entries of all applications
  int32_t bar_off;
  const int64_t* gt_off;
  const int32_t* gt_lab;
  unsigned long long* n_incorrect;
  unsigned long long* hist_pred;
  uint8_t* decision;        // [rows][n_apps] or NULL
  // lane-per-application layout (all_apps_lane_kernel): applications sorted by |𝕎_a| in
  // groups of 32 (lane l of group g = application perm[32 g + l]); group g's entries
  // transposed, entry e of lane l at aa_ent[aa_goff[g] + 32 e + l] as column << 8 | (1 << list)
  // (a dummy key past the application's own entries), so a lane scans its application with no
  // cross-lane reduction
  const uint32_t* aa_ent;
  const int32_t* aa_goff;   // [n_groups + 1]
  const uint16_t* aa_perm;  // [n_groups * 32], 0xFFFF = no application
  int32_t n_groups, aa_ent_total;
  int32_t rows_per_unit;    // R
  uint32_t dummy_key;       // key of a padding entry: column = the row buffer's -inf slot, no list bit
  // lane-per-row layout (all_apps_rows_kernel, C <= kTRMaxC): a unit of kTRRows rows is held
  // transposed in shared memory, element (row r, column c) at word kTRStride * c + r (every
  // lane of a warp reads the same column of its own row: 32 distinct banks), column C = -inf.
  // Application a's entries tr_key[tr_off[a] .. tr_off[a+1]) = kTRStride * c (the word
  // offset of column c, < 2^16), ascending, padded to a multiple of 4 with column C (a winner's
  // list is read from catT).  Applications are dealt in aa_perm order (|W_a| descending).
  const uint16_t* tr_key;
  int32_t tr_total;         // entries of all applications (padded)
  const int32_t* tr_off;    // [n_apps + 1]
};
constexpr int kTRRows = 32;               // rows per unit of the lane-per-row kernel (one per lane)
constexpr int kTRStride = kTRRows + 1;    // words between columns of the transposed unit
constexpr int kTRWarps = 32;              // warps per CTA of the lane-per-row kernel (one staged row each)
constexpr int kTRMaxC = 1024;             // columns a unit's rows may have (staged in registers)
constexpr int kAllAppsRows = 4;  // rows per barrier interval of the warp-per-application kernel
cudaError_t launch_all_apps_lane(const AllAppsParams& p, int grid, size_t smem, cudaStream_t st);
cudaError_t launch_all_apps_rows(const AllAppsParams& p, int grid, size_t smem, cudaStream_t st);
cudaError_t launch_all_apps(const AllAppsParams& p, int grid, size_t smem, cudaStream_t st);

// Launchers (sc_kernels.cu).  Return cudaError_t of the launch.
// epl > 0: lane-resident entries (|W| <= 32*epl, whole rows per stage); 0: generic list path.
// pat 0: split maxima; 1: per-list slots; 2: dense-mapped rows (epl = 16-B groups per lane, 1..8).
cudaError_t launch_eval(const EvalParams& p, int epl, int pat, int grid, size_t smem, cudaStream_t st);
// Sector-sparse variant: epl = entries per lane capacity (1,2,4,8,16,32 -> |W| <= 32*epl).
// pat 0: split maxima (API-output order); pat 1: per-list maxima (application-choice, Multi-Select).
cudaError_t launch_gather(const EvalParams& p, int epl, int pat, int sms, cudaStream_t st);
cudaError_t launch_hist(const HistParams& p, int grid, size_t smem, cudaStream_t st);
cudaError_t launch_hist_rows(const HistParams& p, int grid, cudaStream_t st);  // single app, C <= 128K
cudaError_t launch_weights(const unsigned long long* hist, float* w, int n_apps, cudaStream_t st);
cudaError_t set_eval_smem_limit(size_t smem);
// Smallest compiled lane-resident entry capacity for max_ent mapped labels (-1: none fits).
int eval_epl_for(int max_ent, int pat = 0);

}  // namespace sc
