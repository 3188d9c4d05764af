// sc_allapps.cu — "one read, many contexts".
//
// The provider's what-if: every row's logits are read from HBM once and evaluated under
// EVERY application of the context (Multi-Choice, API-output order, PAPER.md:862,
// :128-134, Eq. goal): per application, the decision, its correctness and
// the decision histogram.  Reading the batch once per application would cost n_apps full
// passes; here the bound moves from HBM to the shared-memory / issue rate.
//
// A persistent CTA per SM holds every application's mapped labels (sorted per app,
// key = c << 8 | cat) in shared memory, double-buffers rows with TMA bulk copies, builds
// G for all applications from the row's ground-truth labels and a label-major copy of
// the category table (one coalesced 256-B read per label for 256 apps), then its 32 warps
// take the applications round-robin: split maxima over the app's labels, two REDUX pairs,
// the app's maxima parked in one lane so decision, correctness and the shared-memory
// counters run lane-parallel once per row; the next row's G is built while this row is
// evaluated; counters flushed once per CTA.
#include "sc_internal.cuh"

#include <cuda_runtime.h>
#include <math_constants.h>

namespace sc {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kAAWarps = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nAA_WAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra AA_WAIT_%=;\n}\n" ::
          "r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                   "r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ uint32_t ord_key(float z) {
  const uint32_t u = __float_as_uint(z + 0.0f);
  return u ^ (static_cast<uint32_t>(static_cast<int32_t>(u) >> 31) | 0x80000000u);
}

__device__ __forceinline__ void argmax_warp(float& z, uint32_t& k) {
  const uint32_t o = (k == kNone) ? 0u : ord_key(z);
  const uint32_t om = __reduce_max_sync(kFull, o);
  k = __reduce_min_sync(kFull, (o == om) ? k : kNone);
  z = om ? __uint_as_float((om & 0x80000000u) ? (om ^ 0x80000000u) : ~om) : -CUDART_INF_F;
}

// Split maxima of one app over one row, both classes (P⁺ over 𝒲_i, P⁻ over the rest).
struct Split {
  float zp, zm;
  uint32_t kp, km;
};

// Decision and correctness of one (row, app) from its reduced split maxima.
__device__ __forceinline__ void aa_decide(const Split& m, uint32_t G, uint32_t D, float tau, uint32_t& dec, bool& ok) {
  const bool hp = m.kp != kNone, hm = m.km != kNone;
  const bool take_p = hp && (!hm || m.zp > m.zm || (m.zp == m.zm && m.kp < m.km));
  const float zs = take_p ? m.zp : m.zm;
  const uint32_t ks = take_p ? m.kp : m.km;
  dec = ((hp || hm) && zs > tau) ? (ks & 0xFFu) : D;
  ok = G ? (dec < D && ((G >> dec) & 1u)) : (dec == D);
}

// Units of kAARows consecutive rows: one barrier interval evaluates every app on all of
// them (the app's keys are read once per unit, kAARows rows' loads in flight per entry).
constexpr int kAARows = kAllAppsRows;

__global__ void __launch_bounds__(kAAWarps * 32, 1) all_apps_kernel(const AllAppsParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int A = p.ctx.n_apps;
  // carve shared memory: [2 units][kAARows rows] row buffers
  uint8_t* rowbuf = sm;
  uint32_t* ents = reinterpret_cast<uint32_t*>(sm + 2 * kAARows * p.row_bytes_pad);
  int32_t* eoff = reinterpret_cast<int32_t*>(ents + p.n_ent_total);
  unsigned* cnt_inc = reinterpret_cast<unsigned*>(eoff + A + 1);
  unsigned* cnt_pred = cnt_inc + A;                                   // [A][16]
  uint8_t* gs2 = reinterpret_cast<uint8_t*>(cnt_pred + A * 16);      // [2 units][kAARows][A] G per app
  uint8_t* nl = gs2 + 2 * kAARows * A;                                // [A] D'
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + p.bar_off);      // [2]
  for (int i = tid; i < p.n_ent_total; i += blockDim.x) ents[i] = __ldg(p.ctx.ent + i);
  for (int i = tid; i <= A; i += blockDim.x) eoff[i] = __ldg(p.ctx.ent_off + i);
  for (int i = tid; i < A; i += blockDim.x) { cnt_inc[i] = 0; nl[i] = __ldg(p.ctx.nlists + i); }
  for (int i = tid; i < A * 16; i += blockDim.x) cnt_pred[i] = 0;
  if (tid == 0) { mbar_init1(bar); mbar_init1(bar + 1); }
  __syncthreads();

  const int64_t n_units = (p.rows + kAARows - 1) / kAARows;
  const int64_t first = blockIdx.x, step = gridDim.x;
  auto unit_rows = [&](int64_t u) {
    const int64_t r0 = u * kAARows;
    return static_cast<int>(p.rows - r0 < kAARows ? p.rows - r0 : kAARows);
  };
  // issue a unit's row copies (one barrier for all of them)
  auto load_unit = [&](int64_t u, int b) {
    const int nr = unit_rows(u);
    mbar_expect(bar + b, p.copy_bytes * nr);
    for (int r = 0; r < nr; ++r)
      bulk_copy(rowbuf + (b * kAARows + r) * p.row_bytes_pad, p.logits + (u * kAARows + r) * p.ld_bytes,
                p.copy_bytes, bar + b);
  };
  // G for every app from each row's ground truth (label-major category table)
  auto build_g = [&](int64_t u, uint8_t* gs) {
    if (u >= n_units) return;
    const int nr = unit_rows(u);
    for (int r = 0; r < nr; ++r) {
      const int64_t row = u * kAARows + r;
      const int64_t g0 = __ldg(p.gt_off + row), g1 = __ldg(p.gt_off + row + 1);
      for (int a = tid; a < A; a += blockDim.x) {
        uint32_t G = 0;
        for (int64_t t = g0; t < g1; ++t) {
          const int32_t c = __ldg(p.gt_lab + t);
          G |= label_lists(__ldg(p.catT + static_cast<int64_t>(c) * A + a), kApiOutput);
        }
        gs[r * A + a] = static_cast<uint8_t>(G);
      }
    }
  };
  if (tid == 0 && first < n_units) load_unit(first, 0);
  build_g(first, gs2);
  __syncthreads();
  uint32_t phase[2] = {0, 0};
  int buf = 0;
  for (int64_t u = first; u < n_units; u += step, buf ^= 1) {
    // the next unit's rows into the other buffers (consumed: barrier below), and its G
    const int64_t nxt = u + step;
    if (tid == 0 && nxt < n_units) load_unit(nxt, buf ^ 1);
    build_g(nxt, gs2 + (buf ^ 1) * kAARows * A);
    mbar_wait_parity(bar + buf, phase[buf]);
    phase[buf] ^= 1u;
    const int nr = unit_rows(u);
    const uint8_t* rb = rowbuf + (buf * kAARows) * p.row_bytes_pad;
    const uint8_t* gs = gs2 + buf * kAARows * A;
    // this warp's apps a = warp + 32 j: app j's maxima park in lane j; the decisions and
    // counters run lane-parallel once per unit
    Split pk[kAARows];
    int pa = -1, j = 0;
    for (int a = warp; a < A; a += kAAWarps, ++j) {
      uint32_t G[kAARows];
      Split m[kAARows];
#pragma unroll
      for (int r = 0; r < kAARows; ++r) {
        G[r] = gs[r * A + a];
        m[r] = Split{-CUDART_INF_F, -CUDART_INF_F, kNone, kNone};
      }
      for (int e = eoff[a] + lane; e < eoff[a + 1]; e += 32) {
        const uint32_t key = ents[e];
        const uint32_t cat = key & 0xFFu;
        float z[kAARows];
#pragma unroll
        for (int r = 0; r < kAARows; ++r)
          z[r] = p.bf16 ? __uint_as_float(static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(
                              rb + r * p.row_bytes_pad + 2u * (key >> 8))) << 16)
                        : *reinterpret_cast<const float*>(rb + r * p.row_bytes_pad + 4u * (key >> 8));
#pragma unroll
        for (int r = 0; r < kAARows; ++r) {
          if ((G[r] >> cat) & 1u) {
            if (z[r] > m[r].zp) { m[r].zp = z[r]; m[r].kp = key; }
          } else {
            if (z[r] > m[r].zm) { m[r].zm = z[r]; m[r].km = key; }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < kAARows; ++r) {
        if (r < nr) {  // warp-uniform
          argmax_warp(m[r].zp, m[r].kp);
          argmax_warp(m[r].zm, m[r].km);
        }
      }
      if (lane == (j & 31)) {
#pragma unroll
        for (int r = 0; r < kAARows; ++r) pk[r] = m[r];
        pa = a;
      }
      if ((j & 31) == 31 || a + kAAWarps >= A) {  // warp-uniform: flush the parked apps
        if (pa >= 0) {
          const uint32_t D = nl[pa];
#pragma unroll
          for (int r = 0; r < kAARows; ++r) {
            if (r >= nr) break;
            uint32_t dec;
            bool ok;
            aa_decide(pk[r], gs[r * A + pa], D, p.ctx.tau, dec, ok);
            if (!ok) atomicAdd(cnt_inc + pa, 1u);
            atomicAdd(cnt_pred + pa * 16 + dec, 1u);
            if (p.decision) p.decision[(u * kAARows + r) * A + pa] = static_cast<uint8_t>(dec);
          }
        }
        pa = -1;
      }
    }
    __syncthreads();  // row buffers, gs and the next unit's G are reused / complete
  }
  for (int i = tid; i < A; i += blockDim.x)
    if (cnt_inc[i] && p.n_incorrect) atomicAdd(p.n_incorrect + i, static_cast<unsigned long long>(cnt_inc[i]));
  for (int i = tid; i < A * 16; i += blockDim.x)
    if (cnt_pred[i] && p.hist_pred)
      atomicAdd(p.hist_pred + (i >> 4) * 256 + (i & 15), static_cast<unsigned long long>(cnt_pred[i]));
}

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}

// One entry of a lane's arg max (strict '>': the earlier, smaller label keeps ties).
__device__ __forceinline__ void aa_max(float z, uint32_t key, float& zb, uint32_t& kb) {
  asm("{\n\t"
      ".reg .pred g;\n\t"
      "setp.gt.f32 g, %2, %0;\n\t"
      "@g mov.f32 %0, %2;\n\t"
      "@g mov.b32 %1, %3;\n\t"
      "}"
      : "+f"(zb), "+r"(kb)
      : "f"(z), "r"(key));
}

// Lane per application (the default): the 32 lanes of a warp scan 32 different applications
// of one row, each its own entries in ascending label order (strict '>' keeps the smaller
// label on ties, A4), so no warp reduction is needed at all; decision, correctness and the
// counters are per lane.  Applications are grouped 32 at a time by size (largest first) so a
// warp's lanes run similar trip counts; work items (group, row of the unit) are dealt to the
// warps in a snake order over the size-sorted items, pairing large groups with small ones.
// Padding entries point at a -inf slot past the row's copied columns and carry no list bit.
__global__ void __launch_bounds__(kAAWarps * 32, 1) all_apps_lane_kernel(const AllAppsParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int A = p.ctx.n_apps, R = p.rows_per_unit, NG = p.n_groups;
  uint8_t* rowbuf = sm;                                                     // [2][R][row_bytes_pad]
  uint32_t* ents = reinterpret_cast<uint32_t*>(sm + 2 * R * p.row_bytes_pad);  // [aa_ent_total]
  int32_t* goff = reinterpret_cast<int32_t*>(ents + p.aa_ent_total);        // [NG + 1]
  uint16_t* perm = reinterpret_cast<uint16_t*>(goff + NG + 1);             // [NG * 32]
  unsigned* cnt_inc = reinterpret_cast<unsigned*>(perm + NG * 32);          // [A]
  unsigned* cnt_pred = cnt_inc + A;                                         // [A][16]
  uint8_t* gs2 = reinterpret_cast<uint8_t*>(cnt_pred + A * 16);            // [2][R][A]
  uint8_t* nl = gs2 + 2 * R * A;                                            // [A]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + p.bar_off);            // [2]
  for (int i = tid; i < p.aa_ent_total; i += blockDim.x) ents[i] = __ldg(p.aa_ent + i);
  for (int i = tid; i <= NG; i += blockDim.x) goff[i] = __ldg(p.aa_goff + i);
  for (int i = tid; i < NG * 32; i += blockDim.x) perm[i] = __ldg(p.aa_perm + i);
  for (int i = tid; i < A; i += blockDim.x) { cnt_inc[i] = 0; nl[i] = __ldg(p.ctx.nlists + i); }
  for (int i = tid; i < A * 16; i += blockDim.x) cnt_pred[i] = 0;
  // the -inf slot of every row buffer (column round_up(C, 8), past what the bulk copies write)
  const uint32_t elt = p.bf16 ? 2u : 4u;
  for (int i = tid; i < 2 * R; i += blockDim.x) {
    uint8_t* slot = rowbuf + i * p.row_bytes_pad + (p.dummy_key >> 8) * elt;
    if (p.bf16) *reinterpret_cast<uint16_t*>(slot) = 0xFF80u;
    else *reinterpret_cast<uint32_t*>(slot) = 0xFF800000u;
  }
  if (tid == 0) { mbar_init1(bar); mbar_init1(bar + 1); }
  __syncthreads();

  const int64_t n_units = (p.rows + R - 1) / R;
  const int64_t first = blockIdx.x, step = gridDim.x;
  auto unit_rows = [&](int64_t u) {
    const int64_t r0 = u * R;
    return static_cast<int>(p.rows - r0 < R ? p.rows - r0 : R);
  };
  auto load_unit = [&](int64_t u, int b) {
    const int nr = unit_rows(u);
    mbar_expect(bar + b, p.copy_bytes * nr);
    for (int r = 0; r < nr; ++r)
      bulk_copy(rowbuf + (b * R + r) * p.row_bytes_pad, p.logits + (u * R + r) * p.ld_bytes, p.copy_bytes, bar + b);
  };
  auto build_g = [&](int64_t u, uint8_t* gs) {
    if (u >= n_units) return;
    const int nr = unit_rows(u);
    for (int r = 0; r < nr; ++r) {
      const int64_t row = u * R + r;
      const int64_t g0 = __ldg(p.gt_off + row), g1 = __ldg(p.gt_off + row + 1);
      for (int a = tid; a < A; a += blockDim.x) {
        uint32_t G = 0;
        for (int64_t t = g0; t < g1; ++t) {
          const int32_t c = __ldg(p.gt_lab + t);
          G |= label_lists(__ldg(p.catT + static_cast<int64_t>(c) * A + a), kApiOutput);
        }
        gs[r * A + a] = static_cast<uint8_t>(G);
      }
    }
  };
  if (tid == 0 && first < n_units) load_unit(first, 0);
  build_g(first, gs2);
  __syncthreads();
  uint32_t phase[2] = {0, 0};
  int buf = 0;
  const int n_items = NG * R;
  for (int64_t u = first; u < n_units; u += step, buf ^= 1) {
    const int64_t nxt = u + step;
    if (tid == 0 && nxt < n_units) load_unit(nxt, buf ^ 1);
    build_g(nxt, gs2 + (buf ^ 1) * R * A);
    mbar_wait_parity(bar + buf, phase[buf]);
    phase[buf] ^= 1u;
    const int nr = unit_rows(u);
    const uint8_t* gs = gs2 + buf * R * A;
    // items i = g * R + r in descending cost; warp w takes w, 2*32-1-w, 2*32+w, 4*32-1-w, ...
    for (int k = 0;; ++k) {
      const int blk = k >> 1;
      const int i = blk * 2 * kAAWarps + ((k & 1) ? 2 * kAAWarps - 1 - warp : warp);
      if (i >= n_items) {
        if (k & 1) continue;  // the mirrored item of this round is past the end; the next may not be
        break;
      }
      const int g = i / R, r = i - g * R;
      if (r >= nr) continue;
      const int slot = 32 * g + lane;
      const uint32_t a = perm[slot];
      const bool live = a != 0xFFFFu;
      const uint32_t G = live ? gs[r * A + a] : 0u;
      const uint32_t rb = smem_u32(rowbuf + (buf * R + r) * p.row_bytes_pad);
      const uint32_t e0 = smem_u32(ents + goff[g] + lane);
      const int n = (goff[g + 1] - goff[g]) >> 5;
      // The decision needs only the arg max over the application's 𝕎 (a3: the first mapped
      // label in confidence order, then z > tau), not the split into 𝒲_i / 𝕎∖𝒲_i: one
      // compare-select per entry.  Keys are column << 8 | (1 << list), ascending in the lane,
      // so the strict '>' keeps the smaller label on ties (A4); padding entries point at
      // z = -inf, which never wins.
      float zb = -CUDART_INF_F;
      uint32_t kb = kNone;
      if (p.bf16) {
#pragma unroll 4
        for (int t = 0; t < n; ++t) {
          const uint32_t key = lds32(e0 + 128u * t);
          const float z = __uint_as_float(lds16(rb + 2u * (key >> 8)) << 16);
          aa_max(z, key, zb, kb);
        }
      } else {
#pragma unroll 4
        for (int t = 0; t < n; ++t) {
          const uint32_t key = lds32(e0 + 128u * t);
          const float z = __uint_as_float(lds32(rb + 4u * (key >> 8)));
          aa_max(z, key, zb, kb);
        }
      }
      // back to column << 8 | list for the decision
      if (kb != kNone) kb = (kb & ~0xFFu) | static_cast<uint32_t>(__ffs(kb & 0xFFu) - 1);
      if (live) {
        uint32_t dec;
        bool ok;
        aa_decide(Split{zb, -CUDART_INF_F, kb, kNone}, G, nl[a], p.ctx.tau, dec, ok);
        if (!ok) atomicAdd(cnt_inc + a, 1u);
        atomicAdd(cnt_pred + a * 16 + dec, 1u);
        if (p.decision) p.decision[(u * R + r) * A + a] = static_cast<uint8_t>(dec);
      }
    }
    __syncthreads();  // row buffers, gs and the next unit's G are reused / complete
  }
  for (int i = tid; i < A; i += blockDim.x)
    if (cnt_inc[i] && p.n_incorrect) atomicAdd(p.n_incorrect + i, static_cast<unsigned long long>(cnt_inc[i]));
  for (int i = tid; i < A * 16; i += blockDim.x)
    if (cnt_pred[i] && p.hist_pred)
      atomicAdd(p.hist_pred + (i >> 4) * 256 + (i & 15), static_cast<unsigned long long>(cnt_pred[i]));
}

// Lane per ROW (the default when C <= kTRMaxC): a unit of kTRRows = 32 rows is held
// transposed in shared memory — element (r, c) at word kTRStride·c + r — so when the 32 lanes
// of a warp (one row each) read the same column of their own rows they hit 32 distinct banks
// (the lane-per-application kernel above reads 32 random columns of one row: ~3.5-way bank
// conflicts per load, and shared-memory wavefronts bounded it).  A warp evaluates one
// application on all 32 rows of the unit: its entries (16-bit word offsets of the columns,
// ascending, every application's in shared memory) are warp-uniform 8-B broadcast loads of 4
// entries, and per entry a lane does one address computation, one conflict-free shared load
// and one compare-select — the arg max over 𝕎_a (a3; the strict '>' keeps the smaller label
// on ties, A4), tracked by its shared address, from which the column and then its list
// (catT) are recovered once per (row, application).  The next
// unit's rows are loaded into registers (one row per warp) while the current unit is
// evaluated, then stored transposed; G per (row, application) comes from the row's ground
// truth and the label-major category table (Eq. goal's correctness).
template <bool BF16>
__global__ void __launch_bounds__(kTRWarps * 32, 1) all_apps_rows_kernel(const AllAppsParams p) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int A = p.ctx.n_apps, C = p.ctx.C;
  float* tr = reinterpret_cast<float*>(sm);                                        // [C + 1][kTRStride]
  uint8_t* gtile = sm + 4 * static_cast<size_t>(kTRStride) * (C + 1);                // [A][kTRRows]
  unsigned* cnt_inc = reinterpret_cast<unsigned*>(gtile + kTRRows * A + 3 - (kTRRows * A + 3) % 4);  // [A]
  unsigned* cnt_pred = cnt_inc + A;                                                  // [A][16]
  uint8_t* nl = reinterpret_cast<uint8_t*>(cnt_pred + 16 * A);                       // [A]
  const size_t kofs = (4 * static_cast<size_t>(kTRStride) * (C + 1) + kTRRows * A + 4 * A + 64 * A + A + 15) / 16 * 16;
  uint16_t* keys = reinterpret_cast<uint16_t*>(sm + kofs);                           // [tr_total]
  int32_t* toff = reinterpret_cast<int32_t*>(keys + p.tr_total);                     // [A + 1] (tr_total % 4 == 0)
  uint16_t* order = reinterpret_cast<uint16_t*>(toff + A + 1);                        // [A] applications, |W_a| descending
  for (int i = tid; i < p.tr_total / 8; i += blockDim.x)
    reinterpret_cast<uint4*>(keys)[i] = __ldg(reinterpret_cast<const uint4*>(p.tr_key) + i);
  for (int i = p.tr_total / 8 * 8 + tid; i < p.tr_total; i += blockDim.x) keys[i] = __ldg(p.tr_key + i);
  for (int i = tid; i <= A; i += blockDim.x) toff[i] = __ldg(p.tr_off + i);
  for (int i = tid; i < A; i += blockDim.x) order[i] = __ldg(p.aa_perm + i);
  for (int i = tid; i < kTRRows; i += blockDim.x) tr[kTRStride * C + i] = -CUDART_INF_F;  // padding column
  for (int i = tid; i < A; i += blockDim.x) { cnt_inc[i] = 0; nl[i] = __ldg(p.ctx.nlists + i); }
  for (int i = tid; i < 16 * A; i += blockDim.x) cnt_pred[i] = 0;

  const int64_t n_units = (p.rows + kTRRows - 1) / kTRRows;
  constexpr int kJ = BF16 ? kTRMaxC / 64 : kTRMaxC / 32;  // staged words per lane and row
  constexpr int kRW = kTRRows / kTRWarps;  // rows staged per warp
  uint32_t v[kRW][kJ];
  // stage row u*32 + w of unit u in registers (f32: column 32 j + lane; bf16: the
  // column pair 64 j + 2 lane, +1)
  auto stage = [&](int64_t u) {
#pragma unroll
    for (int h = 0; h < kRW; ++h) {
      const int64_t row = u * kTRRows + kRW * warp + h;
      const uint8_t* src = p.logits + row * p.ld_bytes;
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int c = BF16 ? 64 * j + 2 * lane : 32 * j + lane;
        v[h][j] = (u < n_units && row < p.rows && c < C) ? __ldg(reinterpret_cast<const uint32_t*>(src) + (BF16 ? c / 2 : c)) : 0u;
      }
    }
  };
  const int64_t first = blockIdx.x, step = gridDim.x;
  stage(first);
  __syncthreads();
  const uint32_t lb = smem_u32(tr) + 4u * static_cast<uint32_t>(lane);
  const float tau = p.ctx.tau;
  for (int64_t u = first; u < n_units; u += step) {
    const int64_t row0 = u * kTRRows;
    const int nr = static_cast<int>(p.rows - row0 < kTRRows ? p.rows - row0 : kTRRows);
    // the staged rows, transposed
#pragma unroll
    for (int h = 0; h < kRW; ++h) {
      const int r = kRW * warp + h;
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        if constexpr (BF16) {
          const int c = 64 * j + 2 * lane;
          if (c < C) tr[kTRStride * c + r] = __uint_as_float(v[h][j] << 16);
          if (c + 1 < C) tr[kTRStride * (c + 1) + r] = __uint_as_float(v[h][j] & 0xFFFF0000u);
        } else {
          const int c = 32 * j + lane;
          if (c < C) tr[kTRStride * c + r] = __uint_as_float(v[h][j]);
        }
      }
    }
    // G of every (row, application), a2: warp w builds row w; the row's ground-truth
    // labels are warp-uniform loads, each lane ORs the lists of applications lane + 32 k
    // (independent, coalesced 32-B reads of the label-major category table)
#pragma unroll 1
    for (int h = 0; h < kRW; ++h) {
      const int r = kRW * warp + h;
      const int64_t g0 = r < nr ? __ldg(p.gt_off + row0 + r) : 0, g1 = r < nr ? __ldg(p.gt_off + row0 + r + 1) : 0;
      for (int a0 = 0; a0 < A; a0 += 256) {
        uint32_t G[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t t = g0; t < g1; ++t) {
          const uint8_t* crow = p.catT + static_cast<int64_t>(__ldg(p.gt_lab + t)) * A;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int a = a0 + 32 * k + lane;
            if (a < A) G[k] |= label_lists(__ldg(crow + a), kApiOutput);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int a = a0 + 32 * k + lane;
          if (a < A) gtile[a * kTRRows + r] = static_cast<uint8_t>(G[k]);
        }
      }
    }
    __syncthreads();
    stage(u + step);  // in flight while this unit is evaluated
    const bool live_row = lane < nr;
    const unsigned act = __ballot_sync(kFull, live_row);
    // One application on the unit's 32 rows per item; applications in |W_a|-descending order,
    // dealt in a snake over the warps.  The epilogue of an item (its list from catT, a global
    // load) runs after the NEXT item's scan, so the load's latency hides behind that scan.
    int pa = -1;          // the pending item's application
    uint32_t pcat = 0;    // its winner's list (load in flight), 0xFF: default
    auto finish = [&](int a, uint32_t cat) {
      const uint32_t D = nl[a];
      const uint32_t dec = cat != 0xFFu ? cat : D;
      const uint32_t G = gtile[a * kTRRows + lane];
      const bool ok = G ? (dec < D && ((G >> dec) & 1u)) : (dec == D);
      const unsigned inc = __ballot_sync(kFull, live_row && !ok);
      if (lane == 0 && inc) cnt_inc[a] += __popc(inc);  // application a: this warp only, this unit
      if (live_row) {
        const unsigned peers = __match_any_sync(act, dec);
        if (lane == __ffs(peers) - 1) cnt_pred[a * 16 + dec] += __popc(peers);
        gtile[a * kTRRows + lane] = static_cast<uint8_t>(dec);  // G is read; the tile now holds decisions
      }
    };
    for (int k = 0;; ++k) {
      const int i = (k >> 1) * 2 * kTRWarps + ((k & 1) ? 2 * kTRWarps - 1 - warp : warp);
      if (i >= A) {
        if (k & 1) continue;
        break;
      }
      const int a = order[i];
      const int32_t e0 = toff[a], n = toff[a + 1] - e0;
      const uint32_t kb0 = smem_u32(keys + e0);
      float zb = -CUDART_INF_F;
      uint32_t ab = 0;  // shared address of the winner (0: none)
#pragma unroll 2
      for (int q = 0; q < n; q += 4) {
        uint32_t k01, k23;  // four entries (16-bit word offsets of their columns), warp-uniform
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(k01), "=r"(k23) : "r"(kb0 + 2u * q));
        // per entry: the address (extract + one multiply-add), a conflict-free load, and the
        // strict '>' update of the running maximum and its address (A4: earlier entries win ties)
        asm volatile(
            "{\n\t"
            ".reg .u32 a0, a1, a2, a3;\n\t"
            ".reg .f32 z0, z1, z2, z3;\n\t"
            ".reg .pred p;\n\t"
            "and.b32 a0, %2, 65535;\n\t"
            "shr.u32 a1, %2, 16;\n\t"
            "and.b32 a2, %3, 65535;\n\t"
            "shr.u32 a3, %3, 16;\n\t"
            "mad.lo.u32 a0, a0, 4, %4;\n\t"
            "mad.lo.u32 a1, a1, 4, %4;\n\t"
            "mad.lo.u32 a2, a2, 4, %4;\n\t"
            "mad.lo.u32 a3, a3, 4, %4;\n\t"
            "ld.shared.f32 z0, [a0];\n\t"
            "ld.shared.f32 z1, [a1];\n\t"
            "ld.shared.f32 z2, [a2];\n\t"
            "ld.shared.f32 z3, [a3];\n\t"
            "setp.gt.f32 p, z0, %0;\n\t"
            "@p mov.f32 %0, z0;\n\t"
            "@p mov.u32 %1, a0;\n\t"
            "setp.gt.f32 p, z1, %0;\n\t"
            "@p mov.f32 %0, z1;\n\t"
            "@p mov.u32 %1, a1;\n\t"
            "setp.gt.f32 p, z2, %0;\n\t"
            "@p mov.f32 %0, z2;\n\t"
            "@p mov.u32 %1, a2;\n\t"
            "setp.gt.f32 p, z3, %0;\n\t"
            "@p mov.f32 %0, z3;\n\t"
            "@p mov.u32 %1, a3;\n\t"
            "}"
            : "+f"(zb), "+r"(ab)
            : "r"(k01), "r"(k23), "r"(lb));
      }
      // a3: the first mapped label in confidence order is an output iff z > tau; its list
      // from catT (column recovered from the winner's address), loaded now, used next item
      uint32_t cat = 0xFFu;
      if (ab != 0 && zb > tau) {
        const uint32_t c = (ab - lb) / (4u * kTRStride);
        cat = __ldg(p.catT + static_cast<int64_t>(c) * A + a);
      }
      if (pa >= 0) finish(pa, pcat);
      pa = a;
      pcat = cat;
    }
    if (pa >= 0) finish(pa, pcat);
    __syncthreads();
    if (p.decision) {
      for (int i = tid; i < nr * A; i += blockDim.x) {
        const int r = i / A, a = i - r * A;
        p.decision[(row0 + r) * A + a] = gtile[a * kTRRows + r];
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < A; i += blockDim.x)
    if (cnt_inc[i] && p.n_incorrect) atomicAdd(p.n_incorrect + i, static_cast<unsigned long long>(cnt_inc[i]));
  for (int i = tid; i < A * 16; i += blockDim.x)
    if (cnt_pred[i] && p.hist_pred)
      atomicAdd(p.hist_pred + (i >> 4) * 256 + (i & 15), static_cast<unsigned long long>(cnt_pred[i]));
}

}  // namespace

cudaError_t launch_all_apps_lane(const AllAppsParams& p, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(all_apps_lane_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e) return e;
  all_apps_lane_kernel<<<grid, kAAWarps * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_all_apps_rows(const AllAppsParams& p, int grid, size_t smem, cudaStream_t st) {
  auto k = p.bf16 ? all_apps_rows_kernel<true> : all_apps_rows_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e) return e;
  k<<<grid, kTRWarps * 32, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_all_apps(const AllAppsParams& p, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(all_apps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e) return e;
  all_apps_kernel<<<grid, kAAWarps * 32, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace sc
