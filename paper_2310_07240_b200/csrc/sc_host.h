// sc_host.h — host-side state shared by the libsc translation units (not part of the ABI).
#pragma once
#include "sc.h"

#include <cstdint>
#include <mutex>
#include <vector>

struct sc_context_s {
  int32_t C = 0, n_apps = 0, max_ent = 0;
  // logit columns a batch row holds: C (dense: column c = label c), or |union of the apps'
  // mapped labels| for a column-compacted context (column j = label cols[j], ascending)
  int32_t ncols = 0;
  bool compact = false;
  std::vector<int32_t> cols;        // compact: label of each column
  int32_t* d_col_label = nullptr;   // compact: device copy of cols (gradient indices -> labels)
  int32_t order = 0;
  float tau = 0.f, theta = 0.5f, k = 1.f;
  int device = 0;
  std::vector<int32_t> nlists, n_mapped;
  int64_t touched_sectors[2] = {0, 0};  // sum over apps of 32-B sectors holding mapped labels (f32, bf16)
  int64_t touched_lines[2] = {0, 0};    // same for 128-B lines (the granularity HBM is read at, measured)
  uint8_t* d_cat = nullptr;
  uint32_t* d_ent = nullptr;
  int32_t* d_ent_off = nullptr;
  uint8_t* d_nlists = nullptr;
  // completion counters of the fused hist+weights pre-pass: one per stream that has used
  // this context (kDonePool preallocated at load, so calls on different streams never share
  // one; each returns to 0 when its launch completes, so calls on one stream reuse it)
  static constexpr int kDonePool = 64;
  unsigned int* d_done = nullptr;  // [kDonePool]
  std::mutex done_mu;
  std::vector<void*> done_streams;  // stream handle of each slot in use
  uint8_t* d_catT = nullptr;       // [C][n_apps] label-major category table (all-apps pass)
  int32_t n_ent_total = 0;
  int32_t max_slots = 0;           // per-list patterns: most list-major 32-entry slots of an app
  uint32_t* d_lent = nullptr;
  int32_t* d_lent_off = nullptr;
  uint32_t* d_lslot = nullptr;
  // all-apps pass, lane per application (see AllAppsParams)
  uint32_t* d_aa_ent = nullptr;
  int32_t* d_aa_goff = nullptr;
  uint16_t* d_aa_perm = nullptr;
  int32_t aa_groups = 0, aa_ent_total = 0;
  // all-apps pass, lane per row (C <= kTRMaxC; see AllAppsParams::tr_*)
  uint16_t* d_tr_key = nullptr;
  int32_t tr_total = 0;
  int32_t* d_tr_off = nullptr;
};

namespace sc {
// Record the message returned by sc_last_error(); returns st.
sc_status set_error(sc_status st, const char* fmt, ...);
// Count one kernel launch of libsc (sc_launch_count) and name it (sc_last_kernel).
void note_launch(const char* kernel);
// Streaming multiprocessors of the current device.
int device_sms();
}  // namespace sc
