// sc_kernels.cu — sm_100a kernels of libsc.
//
// eval_kernel: the fused hot path — one read of
// every logit row yields the decision, the
// incorrect-decision count (Eq. goal), the decision/GT-mask
// histograms and Eq. api_output with its gradient
// (PAPER.md:2033-2040).  It is an HBM-bound row reduction, so there are no
// tensor cores: a persistent CTA per SM streams row blocks HBM -> shared memory
// with TMA bulk copies (cp.async.bulk + mbarrier ring, one producer lane) and
// 16 consumer warps scan only the context's mapped labels out of shared memory
// (the compact list: |W| entries instead of C), reduce with warp shuffles and
// run the per-row epilogue 32 rows at a time (one row per lane).
//
// hist_kernel: the ground-truth-only pre-pass (a2 + a6 for the mask histogram).
// weights_kernel: a7, M/N from the mask histogram via a subset-sum (zeta) transform.
#include "sc_device.cuh"

#include <cuda_runtime.h>
#include <math_constants.h>

namespace sc {
namespace {

// ------------------------------------------------------------------ warp arg max (REDUX)

// Order-preserving map float -> uint32 (negative: ~bits, positive: bits | sign).
// -0.0 is first canonicalised to +0.0: the two compare equal, so they must tie (A4).
__device__ __forceinline__ uint32_t ord_f32(float z) {
  const uint32_t u = __float_as_uint(z + 0.0f);
  return u ^ (static_cast<uint32_t>(static_cast<int32_t>(u) >> 31) | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o ^ 0x80000000u) : ~o);
}

// Warp-wide lexicographic max of (z, -label) with two redux.sync instructions: the max of
// the ordered logits, then the min key among the lanes holding it.  Keys are
// label << 8 | cat (ordered like the label); kNone marks an empty lane.
__device__ __forceinline__ void warp_argmax(float& z, uint32_t& k) {
  const uint32_t o = (k == kNone) ? 0u : ord_f32(z);
  const uint32_t om = __reduce_max_sync(kFull, o);
  k = __reduce_min_sync(kFull, (o == om) ? k : kNone);
  z = om ? unord_f32(om) : -CUDART_INF_F;
}

// ------------------------------------------------------------------ lane-resident context entries

// The mapped labels of one application, spread over the warp: entry t of lane l is
// mapped label number t*32 + l (ascending label ids within a lane, so a strict '>'
// keeps the smaller id on ties).  Kept in registers across rows.
template <int EPL>
struct LaneEnt {
  static constexpr bool kKeepOff = EPL <= 8;  // byte offsets cached in registers only when they fit
  uint32_t key[EPL];   // label << 8 | cat
  uint32_t off_[kKeepOff ? EPL : 1];  // byte offset of the label in a row (0 for absent entries)
  __device__ __forceinline__ uint32_t off(int t, uint32_t elt) const {
    if constexpr (kKeepOff) return off_[t];
    else return key[t] == kNone ? 0u : (key[t] >> 8) * elt;
  }
  uint32_t catm[8];    // bit t set iff entry t is in list j (several bits for Multi-Select)
  uint32_t valid;      // bit t set iff entry t exists
  int32_t app;
  int tc;              // warp-uniform: entry slots in use, ceil(n / 32)
};

template <int EPL>
__device__ __forceinline__ void lane_ent_load(LaneEnt<EPL>& le, const uint32_t* ents, int n, int32_t app, int lane,
                                              uint32_t elt, int order = kApiOutput) {
  le.valid = 0;
  le.app = app;
  le.tc = (n + 31) >> 5;
#pragma unroll
  for (int j = 0; j < 8; ++j) le.catm[j] = 0;
#pragma unroll
  for (int t = 0; t < EPL; ++t) {
    const int e = t * 32 + lane;
    const uint32_t k = e < n ? ents[e] : kNone;
    le.key[t] = k;
    if constexpr (LaneEnt<EPL>::kKeepOff) le.off_[t] = e < n ? (k >> 8) * elt : 0u;
    if (e < n) {
      le.valid |= 1u << t;
      const uint32_t lists = label_lists(static_cast<uint8_t>(k & 0xFFu), order);
#pragma unroll
      for (int j = 0; j < 8; ++j) le.catm[j] |= ((lists >> j) & 1u) << t;
    }
  }
}

// Bit t of the result: entry t of this lane belongs to a list in G (i.e. to 𝒲_i).
template <int EPL>
__device__ __forceinline__ uint32_t plus_mask(const LaneEnt<EPL>& le, uint32_t G) {
  uint32_t pm = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) pm |= (G & (1u << j)) ? le.catm[j] : 0u;
  return pm;
}

// a3/a4 for one row, branch-free: zs[t] = the row's logit of the lane's entry t (all
// loads issued before this is called); pm = plus_mask(G); tc = warp-uniform number of
// entry slots in use.  Split maxima over 𝒲_i and 𝕎∖𝒲_i, reduced over the warp.
// One entry of the split-maxima scan, in PTX so it stays at ~6 instructions:
// the plus/minus class comes from one mask bit, each class keeps (max, key) with a
// strict '>' (ascending ids within a lane keep the smaller id on ties).
template <uint32_t BIT>
__device__ __forceinline__ void scan_entry(float z, uint32_t key, uint32_t pm, float& zp, uint32_t& kp, float& zm,
                                           uint32_t& km) {
  asm("{\n\t"
      ".reg .pred bp, gp, gm;\n\t"
      ".reg .b32 t;\n\t"
      "and.b32 t, %6, %7;\n\t"
      "setp.ne.u32 bp, t, 0;\n\t"
      "setp.gt.and.f32 gp, %4, %0, bp;\n\t"
      "setp.gt.and.f32 gm, %4, %2, !bp;\n\t"
      "@gp mov.f32 %0, %4;\n\t"
      "@gp mov.b32 %1, %5;\n\t"
      "@gm mov.f32 %2, %4;\n\t"
      "@gm mov.b32 %3, %5;\n\t"
      "}"
      : "+f"(zp), "+r"(kp), "+f"(zm), "+r"(km)
      : "f"(z), "r"(key), "r"(pm), "n"(BIT));
}

// The lane's last slot may be empty (lanes >= n mod 32): separate plus / minus masks.
template <uint32_t BIT>
__device__ __forceinline__ void scan_entry_masked(float z, uint32_t key, uint32_t vp, uint32_t vm, float& zp,
                                                  uint32_t& kp, float& zm, uint32_t& km) {
  asm("{\n\t"
      ".reg .pred bp, bm, gp, gm;\n\t"
      ".reg .b32 t, u;\n\t"
      "and.b32 t, %6, %8;\n\t"
      "and.b32 u, %7, %8;\n\t"
      "setp.ne.u32 bp, t, 0;\n\t"
      "setp.ne.u32 bm, u, 0;\n\t"
      "setp.gt.and.f32 gp, %4, %0, bp;\n\t"
      "setp.gt.and.f32 gm, %4, %2, bm;\n\t"
      "@gp mov.f32 %0, %4;\n\t"
      "@gp mov.b32 %1, %5;\n\t"
      "@gm mov.f32 %2, %4;\n\t"
      "@gm mov.b32 %3, %5;\n\t"
      "}"
      : "+f"(zp), "+r"(kp), "+f"(zm), "+r"(km)
      : "f"(z), "r"(key), "r"(vp), "r"(vm), "n"(BIT));
}

// FULL: every slot before the last is populated in every lane (n > (EPL-1)*32), so
// only the last slot needs the validity mask.
template <int EPL, bool FULL, int T = 0>
__device__ __forceinline__ void scan_all(const LaneEnt<EPL>& le, uint32_t pm, uint32_t vp, uint32_t vm,
                                         const float (&zs)[EPL], float& zp, uint32_t& kp, float& zm, uint32_t& km) {
  if constexpr (T < EPL - 1 && FULL) {
    scan_entry<(1u << T)>(zs[T], le.key[T], pm, zp, kp, zm, km);
  } else {
    scan_entry_masked<(1u << T)>(zs[T], le.key[T], vp, vm, zp, kp, zm, km);
  }
  if constexpr (T + 1 < EPL) scan_all<EPL, FULL, T + 1>(le, pm, vp, vm, zs, zp, kp, zm, km);
}

// a3/a4 for one row: zs[t] = the row's logit of the lane's entry t (all loads issued
// before this is called); pm = plus_mask(G).  Split maxima over 𝒲_i and 𝕎∖𝒲_i,
// reduced over the warp.
template <int EPL>
__device__ __forceinline__ void scan_vals(const LaneEnt<EPL>& le, uint32_t pm, const float (&zs)[EPL], float& zp,
                                          uint32_t& kp, float& zm, uint32_t& km) {
  zp = zm = -CUDART_INF_F;
  kp = km = kNone;
  if (le.tc == EPL)  // warp-uniform
    scan_all<EPL, true>(le, pm, le.valid & pm, le.valid & ~pm, zs, zp, kp, zm, km);
  else
    scan_all<EPL, false>(le, pm, le.valid & pm, le.valid & ~pm, zs, zp, kp, zm, km);
  warp_argmax(zp, kp);
  warp_argmax(zm, km);
}

// ------------------------------------------------------------------ per-list maxima (NEXT f1)

// The application-choice order and Multi-Select need the arg max of every list (P_j,
// PAPER.md:2026, :2050), not just the split into 𝒲_i / 𝕎∖𝒲_i.  One predicated update per
// (entry, list): the entry belongs to list j iff bit t of catm[j] is set.
template <uint32_t BIT>
__device__ __forceinline__ void list_entry(float z, uint32_t key, uint32_t cm, float& az, uint32_t& ak) {
  asm("{\n\t"
      ".reg .pred b, g;\n\t"
      ".reg .b32 t;\n\t"
      "and.b32 t, %4, %5;\n\t"
      "setp.ne.u32 b, t, 0;\n\t"
      "setp.gt.and.f32 g, %2, %0, b;\n\t"
      "@g mov.f32 %0, %2;\n\t"
      "@g mov.b32 %1, %3;\n\t"
      "}"
      : "+f"(az), "+r"(ak)
      : "f"(z), "r"(key), "r"(cm), "n"(BIT));
}

template <int EPL, int T = 0>
__device__ __forceinline__ void list_scan(const LaneEnt<EPL>& le, uint32_t cm, const float (&zs)[EPL], float& az,
                                          uint32_t& ak) {
  list_entry<(1u << T)>(zs[T], le.key[T], cm, az, ak);
  if constexpr (T + 1 < EPL) list_scan<EPL, T + 1>(le, cm, zs, az, ak);
}

constexpr int kListPad = 9;  // row stride (floats) of the per-warp list-maxima batch: conflict-free reads

// Per-warp batch of 32 rows' per-list arg maxima, in shared memory.
struct ListBatch {
  float* z;      // [32][kListPad]
  uint32_t* k;   // [32][kListPad]
};

// a3/a4 for one row, every list: the warp-reduced arg max of list j lands in batch row `slot`.
template <int EPL>
__device__ __forceinline__ void scan_lists(const LaneEnt<EPL>& le, int D, const float (&zs)[EPL], ListBatch lb,
                                           int slot, int lane) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j < D) {  // warp-uniform
      float az = -CUDART_INF_F;
      uint32_t ak = kNone;
      list_scan<EPL>(le, le.catm[j], zs, az, ak);
      warp_argmax(az, ak);
      if (lane == j) {
        lb.z[slot * kListPad + j] = az;
        lb.k[slot * kListPad + j] = ak;
      }
    }
  }
}

// Epilogue of the application-choice order (Eq. app_choice) and Multi-Select (Eq.
// multi-select) for the batch's rows, one row per lane; counters as in finish_batch.
__device__ __forceinline__ void finish_lists(const EvalParams& p, RowBatch& b, ListBatch lb, const float* wtab_smem,
                                             int lane) {
  __syncwarp();
  float zj[8];
  uint32_t kj[8];
  const int D = lane < b.n ? __ldg(p.ctx.nlists + b.app) : 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    zj[j] = j < D ? lb.z[lane * kListPad + j] : -CUDART_INF_F;
    kj[j] = j < D ? lb.k[lane * kListPad + j] : kNone;
  }
  finish_lists_core(p, b, zj, kj, wtab_smem, lane);
}

// The per-list patterns on the TMA ring use list-major slots (DevContext::lent): slot t of
// an application holds 32 labels of ONE list (lane l: entry t*32 + l), so a row needs one
// warp arg max per slot — not one masked scan of every entry per list — and the list
// maxima are assembled per lane (one row each) in the batch epilogue.
template <int EPL>
struct SlotEnt {
  uint32_t key[EPL];  // c << 8 | cat[c]; padding 0xFF (column 0, never a winner)
  int ns;             // slots of the application (warp-uniform)
  uint32_t lastm;     // bit t: slot t is the last slot of its list (warp-uniform)
  int32_t app;
};

// Bit t set iff slot t (< ns) ends its list: the next slot holds another list, or none.
__device__ __forceinline__ uint32_t slot_lastm(uint32_t lists, int ns) {
  uint32_t m = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (t < ns && (t + 1 == ns || ((lists >> (4 * t)) & 15u) != ((lists >> (4 * t + 4)) & 15u))) m |= 1u << t;
  return m;
}

template <int EPL>
__device__ __forceinline__ void slot_ent_load(SlotEnt<EPL>& se, const DevContext& c, int32_t app, int lane,
                                              uint32_t elt) {
  const int32_t e0 = __ldg(c.lent_off + app), e1 = __ldg(c.lent_off + app + 1);
  se.ns = (e1 - e0) >> 5;
  se.lastm = slot_lastm(__ldg(c.lslot + app), se.ns);
  se.app = app;
#pragma unroll
  for (int t = 0; t < EPL; ++t) {
    const uint32_t k = t < se.ns ? __ldg(c.lent + e0 + t * 32 + lane) : kNone;
    se.key[t] = k == kNone ? 0xFFu : k;  // the byte offset (key >> 8) * elt is 0 for padding
  }
}

// One entry of a list's fold: padding (key 0xFF) never wins; strict '>' keeps the smaller,
// earlier label on ties (A4).
__device__ __forceinline__ void slot_fold(float z, uint32_t key, float& fz, uint32_t& fk) {
  asm("{\n\t"
      ".reg .pred v, g;\n\t"
      "setp.ne.u32 v, %3, 255;\n\t"
      "setp.gt.and.f32 g, %2, %0, v;\n\t"
      "@g mov.f32 %0, %2;\n\t"
      "@g mov.b32 %1, %3;\n\t"
      "}"
      : "+f"(fz), "+r"(fk)
      : "f"(z), "r"(key));
}

// a3 for one row: the arg max of every list; lane `slot` keeps them (sz, sk), at the
// position of the list's last slot (se.lastm; the other slots' sz / sk are left stale).  A
// list's slots are consecutive and a lane's entries in them ascend, so each lane first folds
// its slots of one list, then one warp arg max per list — not one per 32-label slot.
template <int EPL>
__device__ __forceinline__ void scan_slots(const SlotEnt<EPL>& se, const float (&zs)[EPL], float (&sz)[EPL],
                                           uint32_t (&sk)[EPL], int slot, int lane) {
  float fz = -CUDART_INF_F;
  uint32_t fk = kNone;
#pragma unroll
  for (int t = 0; t < EPL; ++t) {  // slots >= ns hold padding keys only and end no list
    slot_fold(zs[t], se.key[t], fz, fk);
    if ((se.lastm >> t) & 1u) {  // warp-uniform: list of slot t ends here
      float z = fz;
      uint32_t kk = fk;
      warp_argmax(z, kk);
      if (lane == slot) {
        sz[t] = z;
        sk[t] = kk;
      }
      fz = -CUDART_INF_F;
      fk = kNone;
    }
  }
}

// Batch epilogue: each lane folds its row's slot maxima into list maxima (P_j, PAPER.md:2026,
// :2050), then the shared per-list epilogue.
template <int EPL>
__device__ __forceinline__ void finish_slots(const EvalParams& p, RowBatch& b, const float (&sz)[EPL],
                                             const uint32_t (&sk)[EPL], const float* wtab_smem, int lane) {
  float zj[8];
  uint32_t kj[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    zj[j] = -CUDART_INF_F;
    kj[j] = kNone;
  }
  if (lane < b.n) {
    const uint32_t lists = __ldg(p.ctx.lslot + b.app);
    const int ns = (__ldg(p.ctx.lent_off + b.app + 1) - __ldg(p.ctx.lent_off + b.app)) >> 5;
    const uint32_t lastm = slot_lastm(lists, ns);
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
      if (((lastm >> t) & 1u) && sk[t] != kNone) {
        const uint32_t j = (lists >> (4 * t)) & 15u;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q == static_cast<int>(j) && beats(sz[t], sk[t], zj[q], kj[q])) {
            zj[q] = sz[t];
            kj[q] = sk[t];
          }
      }
    }
  }
  finish_lists_core(p, b, zj, kj, wtab_smem, lane);
}

// ------------------------------------------------------------------ dense-mapped rows (PAT 2)

// Every column 0..n-1 of a row is a mapped label of the single application (column-compacted
// rows; or a context that maps every label).  Lane l reads 16-B vectors at
// byte 512 g + 16 l of the row: entry (g, q) = column g·32·kVec + l·kVec + q (kVec = 4 f32 /
// 8 bf16), ascending within the lane, so the strict '>' keeps the smaller label on ties.  No
// per-entry key or offset registers (the EPL = 32 path of a 1000-label row spilled at the
// 96-register cap and was ALU-bound): a winner is tracked by its slot index (an immediate)
// and its key rebuilt once per row.
template <int NV, bool BF16>
struct DmEnt {
  static constexpr int kVec = BF16 ? 8 : 4;
  static constexpr bool kOk = NV * kVec <= 32;  // slot bits fit one register
  uint32_t catm[8];  // bit g*kVec+q set iff entry (g, q) belongs to list j
  uint32_t valid;    // bit set iff the entry's column is < n
};

template <int NV, bool BF16>
__device__ __forceinline__ void dm_ent_load(DmEnt<NV, BF16>& de, const uint32_t* ents, int n, int lane) {
  constexpr int V = DmEnt<NV, BF16>::kVec;
  de.valid = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) de.catm[j] = 0;
#pragma unroll
  for (int g = 0; g < NV; ++g)
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int col = g * 32 * V + lane * V + q, bit = g * V + q;
      if (bit < 32 && col < n) {
        de.valid |= 1u << bit;
        const uint32_t lists = label_lists(static_cast<uint8_t>(__ldg(ents + col) & 0xFFu), kApiOutput);
#pragma unroll
        for (int j = 0; j < 8; ++j) de.catm[j] |= ((lists >> j) & 1u) << bit;
      }
    }
}

// One entry of the split-maxima scan with its slot index as an immediate.
template <uint32_t IDX>
__device__ __forceinline__ void dm_entry(float z, uint32_t pm, float& zp, uint32_t& ip, float& zm, uint32_t& im) {
  asm("{\n\t"
      ".reg .pred bp, gp, gm;\n\t"
      ".reg .b32 t;\n\t"
      "and.b32 t, %5, %6;\n\t"
      "setp.ne.u32 bp, t, 0;\n\t"
      "setp.gt.and.f32 gp, %4, %0, bp;\n\t"
      "setp.gt.and.f32 gm, %4, %2, !bp;\n\t"
      "@gp mov.f32 %0, %4;\n\t"
      "@gp mov.b32 %1, %7;\n\t"
      "@gm mov.f32 %2, %4;\n\t"
      "@gm mov.b32 %3, %7;\n\t"
      "}"
      : "+f"(zp), "+r"(ip), "+f"(zm), "+r"(im)
      : "f"(z), "r"(pm), "n"(1u << IDX), "n"(IDX));
}

// The same for a slot that may lie past column n (separate plus / minus validity masks).
template <uint32_t IDX>
__device__ __forceinline__ void dm_entry_masked(float z, uint32_t vp, uint32_t vm, float& zp, uint32_t& ip, float& zm,
                                                uint32_t& im) {
  asm("{\n\t"
      ".reg .pred bp, bm, gp, gm;\n\t"
      ".reg .b32 t, u;\n\t"
      "and.b32 t, %5, %7;\n\t"
      "and.b32 u, %6, %7;\n\t"
      "setp.ne.u32 bp, t, 0;\n\t"
      "setp.ne.u32 bm, u, 0;\n\t"
      "setp.gt.and.f32 gp, %4, %0, bp;\n\t"
      "setp.gt.and.f32 gm, %4, %2, bm;\n\t"
      "@gp mov.f32 %0, %4;\n\t"
      "@gp mov.b32 %1, %8;\n\t"
      "@gm mov.f32 %2, %4;\n\t"
      "@gm mov.b32 %3, %8;\n\t"
      "}"
      : "+f"(zp), "+r"(ip), "+f"(zm), "+r"(im)
      : "f"(z), "r"(vp), "r"(vm), "n"(1u << IDX), "n"(IDX));
}

__device__ __forceinline__ void lds_v4(uint32_t a, uint32_t (&w)[4]) {
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(a));
}

// Element q of a 16-B vector: f32 word q, or bf16 half q (little-endian: even q in the low half).
template <bool BF16, int Q>
__device__ __forceinline__ float dm_elem(const uint32_t (&w)[4]) {
  if constexpr (BF16) return __uint_as_float((Q & 1) ? (w[Q >> 1] & 0xFFFF0000u) : (w[Q >> 1] << 16));
  else return __uint_as_float(w[Q]);
}

template <int NV, bool BF16, bool MASKED, int G, int Q = 0>
__device__ __forceinline__ void dm_vec(const uint32_t (&w)[4], uint32_t pm, uint32_t vp, uint32_t vm, float& zp,
                                       uint32_t& ip, float& zm, uint32_t& im) {
  constexpr int V = BF16 ? 8 : 4;
  const float z = dm_elem<BF16, Q>(w);
  if constexpr (MASKED) dm_entry_masked<G * V + Q>(z, vp, vm, zp, ip, zm, im);
  else dm_entry<G * V + Q>(z, pm, zp, ip, zm, im);
  if constexpr (Q + 1 < V) dm_vec<NV, BF16, MASKED, G, Q + 1>(w, pm, vp, vm, zp, ip, zm, im);
}

// FULL: every slot of groups 0..NV-2 is valid in every lane (n > (NV-1)·32·kVec).
template <int NV, bool BF16, bool FULL, int G = 0>
__device__ __forceinline__ void dm_scan(const uint32_t (&w)[NV][4], uint32_t pm, uint32_t vp, uint32_t vm, float& zp,
                                        uint32_t& ip, float& zm, uint32_t& im) {
  if constexpr (FULL && G < NV - 1) dm_vec<NV, BF16, false, G>(w[G], pm, vp, vm, zp, ip, zm, im);
  else dm_vec<NV, BF16, true, G>(w[G], pm, vp, vm, zp, ip, zm, im);
  if constexpr (G + 1 < NV) dm_scan<NV, BF16, FULL, G + 1>(w, pm, vp, vm, zp, ip, zm, im);
}

// Ordering key (column << 8) of this lane's slot `idx`, kNone if none; the winner's list is
// looked up once, after the warp reduction (dm_cat).
template <bool BF16>
__device__ __forceinline__ uint32_t dm_colkey(uint32_t idx, int lane) {
  constexpr uint32_t LV = BF16 ? 3 : 2;  // log2 kVec
  const uint32_t col = ((idx >> LV) << (5 + LV)) | (static_cast<uint32_t>(lane) << LV) | (idx & ((1u << LV) - 1));
  return idx == kNone ? kNone : col << 8;
}
// Full key of a reduced winner: entry `column` of the application's sorted entry list IS the
// column's key (every column is mapped, so entry e = column e).
__device__ __forceinline__ uint32_t dm_cat(const EvalParams& p, uint32_t k) {
  return k == kNone ? kNone : __ldg(p.ctx.ent + (k >> 8));
}

// ------------------------------------------------------------------ fused evaluation kernel

// The CTA's units: round-robin (u = blockIdx + i*grid) or one contiguous block per CTA.
struct UnitSched {
  int64_t base, stride, count;
  __device__ __forceinline__ UnitSched(const EvalParams& p) {
    if (p.blocked) {
      const int64_t per = (p.nunits + gridDim.x - 1) / gridDim.x;
      base = static_cast<int64_t>(blockIdx.x) * per;
      stride = 1;
      count = p.nunits - base < per ? p.nunits - base : per;
      if (count < 0) count = 0;
    } else {
      base = blockIdx.x;
      stride = gridDim.x;
      count = (p.nunits - blockIdx.x + gridDim.x - 1) / gridDim.x;
    }
  }
  __device__ __forceinline__ int64_t unit(int64_t i) const { return base + i * stride; }
};

// EPL > 0: whole rows per stage, mapped labels held in registers (|𝕎| <= 32*EPL).
// EPL == 0: generic path — entries read from a shared/global list, rows may be split
// into column chunks across stages (large C).
// PAT = 1: the per-list patterns (application-choice order, Multi-Select) on the same
// ring — EPL = list-major slots per app, one warp arg max per slot (scan_slots), list
// maxima assembled in the batch epilogue (finish_slots).
// DEFER: dense gradient rows parked per warp and written between stages (dense_pair_rows); a
// separate instantiation, so the register allocation of the sparse-gradient kernels is the
// one without it (the shared code cost bf16 5.8 % on the same box, profiles/r4p_*).
template <int EPL, bool BF16, int PAT, bool DEFER = false>
__global__ void __launch_bounds__(kThreads, 1) eval_kernel(const EvalParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- prologue: barriers, context entries and weights into shared memory
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps / p.ng);
    }
    fence_mbar_init();
  }
  uint32_t* ent_smem = reinterpret_cast<uint32_t*>(smem + p.ent_smem_off);
  if (EPL == 0 && p.ent_mode == 0) {
    const int n = p.ctx.ent_off[1];
    for (int e = threadIdx.x; e < n; e += blockDim.x) ent_smem[e] = __ldg(p.ctx.ent + e);
  }
  float* wtab = p.wtab_off >= 0 ? reinterpret_cast<float*>(smem + p.wtab_off) : nullptr;
  if (wtab)
    for (int m = threadIdx.x; m < 256; m += blockDim.x) wtab[m] = __ldg(p.w + m);
  __syncthreads();

  if (warp == 0) {
    // ================= TMA producer (one lane) =================
    if (lane == 0) {
      uint64_t pol = evict_first_policy();
      if (p.no_evict_first) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      uint32_t phase = 0;
      const UnitSched us(p);
      for (int64_t i = 0; i < us.count; ++i) {
        const int64_t u = us.unit(i);
        const int64_t r0 = u * p.R;
        const int nr = static_cast<int>((p.rows - r0 < p.R ? p.rows - r0 : (int64_t)p.R));
        for (int kc = 0; kc < p.nchunks; ++kc) {
          mbar_wait(empty + s, phase ^ 1u);
          uint8_t* st = smem + static_cast<size_t>(s) * p.stage_bytes;
          uint32_t bytes = 0;
          const uint8_t* src_m = nullptr;
          const uint8_t* src_a = nullptr;
          uint32_t nb_m = 0, nb_a = 0;
          if (kc == 0) {
            // side bands: only the 16-B-aligned interior of each window is bulk-copied (no
            // byte outside the caller's array is touched); rows outside it read global memory
            if (p.gt_mask) {
              const SideBand w = sb_window(p.gt_mask, r0, nr, 1);
              src_m = reinterpret_cast<const uint8_t*>(p.gt_mask + r0) + w.head;
              nb_m = w.nb;
            }
            if (p.app) {
              const SideBand w = sb_window(p.app, r0, nr, 2);
              src_a = reinterpret_cast<const uint8_t*>(p.app + r0) + w.head;
              nb_a = w.nb;
            }
          }
          if (p.nchunks == 1) {
            bytes = static_cast<uint32_t>(nr * p.ld_bytes);
          } else {
            const int rem = p.copy_row_bytes - kc * p.chunk_bytes;
            const uint32_t cb = static_cast<uint32_t>(rem < p.chunk_bytes ? rem : p.chunk_bytes);
            bytes = cb * nr;
          }
          if (kc == 0 && p.hdr_off >= 0) {
            // the unit's header for the consumers (visible after their full-barrier wait: the
            // arrive below releases it): r0, nr and the side-band windows, so a consumer warp
            // reads 32 B instead of redoing the 64-bit unit and window arithmetic per stage
            const SideBand wm = p.gt_mask ? sb_window(p.gt_mask, r0, nr, 1) : SideBand{0u, 0u};
            const SideBand wa = p.app ? sb_window(p.app, r0, nr, 2) : SideBand{0u, 0u};
            const uint32_t h = smem_addr(smem) + static_cast<uint32_t>(p.hdr_off) + 32u * static_cast<uint32_t>(s);
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(h), "r"(static_cast<uint32_t>(r0)),
                         "r"(static_cast<uint32_t>(r0 >> 32)) : "memory");
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(h + 8u), "r"(static_cast<uint32_t>(nr)) : "memory");
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(h + 16u), "r"(wm.head), "r"(wm.nb), "r"(wa.head),
                         "r"(wa.nb) : "memory");
          }
          mbar_arrive_expect_tx(full + s, bytes + nb_m + nb_a);
          if (p.nchunks == 1 && !p.split_copy) {
            bulk_g2s(st, p.logits + r0 * p.ld_bytes, bytes, full + s, pol);
          } else if (p.nchunks == 1) {
            const uint32_t rb = static_cast<uint32_t>(p.ld_bytes);
            for (int j = 0; j < nr; ++j) bulk_g2s(st + static_cast<size_t>(j) * rb, p.logits + (r0 + j) * p.ld_bytes, rb, full + s, pol);
          } else {
            const uint32_t cb = bytes / nr;
            for (int j = 0; j < nr; ++j)
              bulk_g2s(st + static_cast<size_t>(j) * p.chunk_bytes,
                       p.logits + (r0 + j) * p.ld_bytes + static_cast<int64_t>(kc) * p.chunk_bytes, cb, full + s,
                       pol);
          }
          if (nb_m) bulk_g2s(st + p.mask_off, src_m, nb_m, full + s, pol);
          if (nb_a) bulk_g2s(st + p.app_off, src_a, nb_a, full + s, pol);
          if (++s == p.stages) { s = 0; phase ^= 1u; }
        }
      }
    }
    return;
  }

  // ================= consumer warps =================
  const int cw = warp - 1;
  RowBatch b;
  b.n = 0; b.zp = b.zm = 0.f; b.kp = b.km = kNone; b.G = 0; b.app = 0; b.row = 0;

  auto row_app_mask = [&](const uint8_t* st, int64_t r0, int nr, int64_t row, uint32_t& a, uint32_t& G) {
    const uint32_t j = static_cast<uint32_t>(row - r0);
    a = 0;
    if (p.app) {
      const SideBand w = sb_window(p.app, r0, nr, 2);
      a = 2u * j - w.head < w.nb ? *reinterpret_cast<const uint16_t*>(st + p.app_off + (2u * j - w.head))
                                 : static_cast<uint32_t>(__ldg(p.app + row));
    }
    G = 0;
    if (p.gt_mask) {
      const SideBand w = sb_window(p.gt_mask, r0, nr, 1);
      G = j - w.head < w.nb ? st[p.mask_off + (j - w.head)] : static_cast<uint32_t>(__ldg(p.gt_mask + row));
    } else if (p.has_gt) {
      G = warp_gt_mask(p, row, a, lane);
    }
  };

  int s = 0;
  uint32_t phase = 0;
  if constexpr (EPL > 0) {
    // ---- whole rows, lane-resident entries.  Consumer warps form NG groups of WG warps;
    // CTA-local unit i lives in stage i % S and is consumed by group i % NG only, so a
    // stage is released as soon as its WG warps are done (no CTA-wide stage barrier).
    constexpr uint32_t kElt = BF16 ? 2u : 4u;
    constexpr bool kSplit = PAT != 1;  // two arg maxima per row: PAT 0, 2 (finish_batch), 3 (finish_app_choice)
    LaneEnt<(PAT == 0 || PAT == 3) ? EPL : 1> le;  // lane-resident entries (PAT 0, 3)
    SlotEnt<PAT == 1 ? EPL : 1> se;    // list-major slots (PAT 1)
    DmEnt<PAT == 2 ? EPL : 1, BF16> de;  // dense-mapped rows (PAT 2)
    float sz[PAT == 1 ? EPL : 1];      // this lane's batch row: arg max of every slot (PAT 1)
    uint32_t sk[PAT == 1 ? EPL : 1];
    if constexpr (PAT == 0 || PAT == 3)
      lane_ent_load(le, p.ctx.ent + __ldg(p.ctx.ent_off), __ldg(p.ctx.ent_off + 1) - __ldg(p.ctx.ent_off), 0, lane,
                    kElt, PAT == 3 ? kAppChoice : kApiOutput);
    else if constexpr (PAT == 1)
      slot_ent_load(se, p.ctx, 0, lane, kElt);
    else
      dm_ent_load(de, p.ctx.ent, __ldg(p.ctx.ent_off + 1), lane);
    // single app: table of plus-masks per G value (one LDS per row instead of 8 selects)
    uint32_t* pmtab = p.pmtab_off >= 0 ? reinterpret_cast<uint32_t*>(smem + p.pmtab_off) : nullptr;
    if (PAT == 3 && pmtab) {
      // application-choice order, single app: per k (the lowest list of G; k = D' for G = ∅)
      // the lane's entries of list k (P_k side) and of lists j < k (P_{k⁻}; all of 𝕎 for k = D')
      for (int kq = cw; kq <= p.pmtab_bits; kq += kConsumerWarps) {
        uint32_t vp = 0, vm = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j == kq) vp = le.catm[j];
          if (j < kq) vm |= le.catm[j];
        }
        pmtab[(2 * kq) * 32 + lane] = vp & le.valid;
        pmtab[(2 * kq + 1) * 32 + lane] = vm & le.valid;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kConsumerWarps * 32) : "memory");
    } else if (kSplit && pmtab) {
      for (int g = cw; g < (1 << p.pmtab_bits); g += kConsumerWarps) {
        uint32_t pmv;
        if constexpr (PAT == 2) {
          pmv = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) pmv |= (g & (1 << j)) ? de.catm[j] : 0u;
        } else {
          pmv = plus_mask(le, g);
        }
        pmtab[g * 32 + lane] = pmv;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kConsumerWarps * 32) : "memory");
    }
    const int ng = p.ng, wg = kConsumerWarps / p.ng;
    const int grp = cw / wg, wi = cw % wg;
    const uint32_t sbase = smem_addr(smem);
    if (DEFER) {  // this warp's parked dense-gradient slab: none parked
      if (lane == 0) asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(pend_slab(p)), "r"(0u) : "memory");
      __syncwarp();
    }
    // this group's units are the CTA-local indices grp, grp+ng, ...: stage and phase advance by ng
    int st_idx = grp;
    uint32_t ph = 0;
    const UnitSched us(p);
    // A warp scans at most rpw rows per stage, and its batch epilogue runs only after it has
    // released the stage (never inside the row loop): a batch ends at the first stage boundary
    // where it holds >= lim rows, so lim <= 33 - rpw keeps it within 32 rows; the first batch
    // sizes are staggered over the warps so they do not all hold the ring in the same stage.
    // (The f32 split-maxima path, HBM-bound, keeps the in-loop epilogue of rounds 1-2 and
    // 32-row batches: same-box A/B, the stage-boundary-only epilogue ran 1.2 % slower there
    // while bf16 gained 6 % and Multi-Select 12 %, profiles/r4s_*, r4t_*.)
    constexpr bool kEpiInLoop = !BF16 && PAT == 0;
    const int rpw = p.R / wg;
    const int lim_max = kEpiInLoop ? 32 : 33 - rpw;
    int lim = 32 - 2 * (cw % 16);
    if (lim > lim_max) lim = lim_max;
    if (lim < 1) lim = 1;
    for (int64_t i = grp; i < us.count; i += ng) {
      mbar_wait(full + st_idx, ph);
      const uint32_t st_off = static_cast<uint32_t>(st_idx) * p.stage_bytes;
      // the unit's header (written by the producer): r0, nr and the side-band windows (the
      // aligned interior of rows [r0, r0 + nr) is in the stage)
      int64_t r0;
      int nr;
      SideBand wm, wa;
      {
        const uint32_t h = sbase + static_cast<uint32_t>(p.hdr_off) + 32u * static_cast<uint32_t>(st_idx);
        uint32_t lo, hi, n;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(h));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(n) : "r"(h + 8u));
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(wm.head), "=r"(wm.nb), "=r"(wa.head), "=r"(wa.nb)
                     : "r"(h + 16u));
        r0 = static_cast<int64_t>((static_cast<uint64_t>(hi) << 32) | lo);
        nr = static_cast<int>(n);
      }
      const uint32_t m_base = sbase + st_off + p.mask_off - wm.head;
      const uint32_t a_base = sbase + st_off + p.app_off - wa.head;
      [[maybe_unused]] int nscan = 0;  // rows this warp scans in this stage (DEFER)
      for (int j = wi; j < nr; j += wg) {
        ++nscan;
        const int64_t row = r0 + j;
        const uint32_t a = !p.app ? 0u
                           : (2u * j - wa.head < wa.nb ? lds_u16(a_base + 2u * j) : static_cast<uint32_t>(__ldg(p.app + row)));
        uint32_t G = 0;
        if (p.gt_mask) G = static_cast<uint32_t>(j) - wm.head < wm.nb ? lds_u8(m_base + j) : static_cast<uint32_t>(__ldg(p.gt_mask + row));
        else if (p.has_gt) G = warp_gt_mask(p, row, a, lane);
        const uint32_t srow = sbase + st_off + static_cast<uint32_t>(j) * static_cast<uint32_t>(p.ld_bytes);
        float zs[PAT == 2 ? 1 : EPL];
        if constexpr (PAT == 2) {
          if constexpr (DmEnt<EPL, BF16>::kOk) {
            uint32_t w[EPL][4];
            const uint32_t lrow = srow + 16u * static_cast<uint32_t>(lane);
#pragma unroll
            for (int g = 0; g < EPL; ++g) lds_v4(lrow + 512u * g, w[g]);
            const uint32_t pm = pmtab ? lds_u32(sbase + p.pmtab_off + (G * 32 + lane) * 4) : 0u;
            float zp = -CUDART_INF_F, zm = -CUDART_INF_F;
            uint32_t ip = kNone, im = kNone;
            if (p.dm_full)  // warp-uniform
              dm_scan<EPL, BF16, true>(w, pm, de.valid & pm, de.valid & ~pm, zp, ip, zm, im);
            else
              dm_scan<EPL, BF16, false>(w, pm, de.valid & pm, de.valid & ~pm, zp, ip, zm, im);
            uint32_t kp = dm_colkey<BF16>(ip, lane), km = dm_colkey<BF16>(im, lane);
            warp_argmax(zp, kp);
            warp_argmax(zm, km);
            kp = dm_cat(p, kp);
            km = dm_cat(p, km);
            deposit(b, lane, zp, kp, zm, km, G, a, row);
          }
        } else if constexpr (PAT == 3) {
          // application-choice order by two arg maxima (finish_app_choice) + the lists holding
          // an output label (one warp OR)
          if (static_cast<int32_t>(a) != le.app) {
            const int32_t e0 = __ldg(p.ctx.ent_off + a);
            lane_ent_load(le, p.ctx.ent + e0, __ldg(p.ctx.ent_off + a + 1) - e0, static_cast<int32_t>(a), lane, kElt,
                          kAppChoice);
          }
#pragma unroll
          for (int t = 0; t < EPL; ++t) zs[t] = lds_z<BF16>(srow + le.off(t, kElt));
          const uint32_t D = pmtab ? static_cast<uint32_t>(p.pmtab_bits) : __ldg(p.ctx.nlists + a);
          const uint32_t kq = G ? static_cast<uint32_t>(__ffs(G) - 1) : D;
          uint32_t vp, vm;
          if (pmtab) {
            vp = lds_u32(sbase + p.pmtab_off + ((2 * kq) * 32 + lane) * 4);
            vm = lds_u32(sbase + p.pmtab_off + ((2 * kq + 1) * 32 + lane) * 4);
          } else {
            vp = 0;
            vm = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (q == static_cast<int>(kq)) vp = le.catm[q];
              if (q < static_cast<int>(kq)) vm |= le.catm[q];
            }
            vp &= le.valid;
            vm &= le.valid;
          }
          float zp = -CUDART_INF_F, zm = -CUDART_INF_F;
          uint32_t kp = kNone, km = kNone;
          scan_all<EPL, false>(le, 0u, vp, vm, zs, zp, kp, zm, km);
          // output lists: entries above tau, folded by list
          uint32_t ob = 0;
#pragma unroll
          for (int t = 0; t < EPL; ++t) ob |= (zs[t] > p.ctx.tau ? 1u : 0u) << t;
          ob &= le.valid;
          uint32_t lo = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) lo |= (ob & le.catm[q]) ? (1u << q) : 0u;
          lo = __reduce_or_sync(kFull, lo);
          warp_argmax(zp, kp);
          warp_argmax(zm, km);
          deposit(b, lane, zp, kp, zm, km, G, a, row, lo);
        } else if constexpr (PAT == 0) {
          if (static_cast<int32_t>(a) != le.app) {
            const int32_t e0 = __ldg(p.ctx.ent_off + a);
            lane_ent_load(le, p.ctx.ent + e0, __ldg(p.ctx.ent_off + a + 1) - e0, static_cast<int32_t>(a), lane, kElt);
          }
#pragma unroll
          for (int t = 0; t < EPL; ++t) zs[t] = lds_z<BF16>(srow + le.off(t, kElt));
          const uint32_t pm = pmtab ? lds_u32(sbase + p.pmtab_off + (G * 32 + lane) * 4) : plus_mask(le, G);
          float zp, zm;
          uint32_t kp, km;
          scan_vals<EPL>(le, pm, zs, zp, kp, zm, km);
          if constexpr (kEpiInLoop) {
            if (b.n == lim) {  // several rows per warp in this stage
              finish_batch<DEFER>(p, b, wtab, lane);
              lim = 32;
            }
          }
          deposit(b, lane, zp, kp, zm, km, G, a, row);
        } else {
          if (static_cast<int32_t>(a) != se.app) slot_ent_load(se, p.ctx, static_cast<int32_t>(a), lane, kElt);
#pragma unroll
          for (int t = 0; t < EPL; ++t) zs[t] = lds_z<BF16>(srow + (se.key[t] >> 8) * kElt);  // slots >= ns: key 0xFF, column 0
          scan_slots<EPL>(se, zs, sz, sk, b.n, lane);
          deposit(b, lane, 0.f, kNone, 0.f, kNone, G, a, row);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st_idx);
      // dense gradient: the previous batch's rows, as many as rows were scanned, so the writes
      // interleave with the reads instead of bursting at the batch boundary
      if constexpr (DEFER) dense_drain(p, lane, nscan);
      // the batch epilogue runs after the stage is released, and the warps' batch boundaries
      // are staggered (lim) so they do not all hold the pipeline in the same stage
      if (kEpiInLoop ? b.n == lim : b.n >= lim) {
        if constexpr (PAT == 3) finish_app_choice<DEFER>(p, b, wtab, lane);
        else if constexpr (kSplit) finish_batch<DEFER>(p, b, wtab, lane);
        else finish_slots<EPL>(p, b, sz, sk, wtab, lane);
        lim = lim_max;
      }
      st_idx += ng;
      if (st_idx >= p.stages) { st_idx -= p.stages; ph ^= 1u; }
    }
    if (b.n > 0) {
      if constexpr (PAT == 3) finish_app_choice<DEFER>(p, b, wtab, lane);
      else if constexpr (kSplit) finish_batch<DEFER>(p, b, wtab, lane);
      else finish_slots<EPL>(p, b, sz, sk, wtab, lane);
    }
    if constexpr (DEFER) dense_drain(p, lane, 32);
    return;
  } else {
    // ---- generic: entries from a list, rows possibly split into column chunks
    uint32_t* slot = p.ent_mode == 1 ? ent_smem + static_cast<size_t>(cw) * p.ent_slot : nullptr;
    int32_t cur_app = -1;
    const uint32_t* ents = p.ent_mode == 0 ? ent_smem : nullptr;
    int32_t n_ent = p.ent_mode == 0 ? p.ctx.ent_off[1] : 0;
    auto select_app = [&](uint32_t a) {
      if (p.ent_mode == 0 || static_cast<int32_t>(a) == cur_app) return;
      const int32_t e0 = __ldg(p.ctx.ent_off + a), e1 = __ldg(p.ctx.ent_off + a + 1);
      n_ent = e1 - e0;
      if (p.ent_mode == 1) {
        __syncwarp();
        for (int e = lane; e < n_ent; e += 32) slot[e] = __ldg(p.ctx.ent + e0 + e);
        __syncwarp();
        ents = slot;
      } else {
        ents = p.ctx.ent + e0;
      }
      cur_app = static_cast<int32_t>(a);
    };
    const UnitSched us(p);
    int lim = 32 - 2 * (cw % 16);  // first batch size of this warp (staggered), then 32
    for (int64_t i = 0; i < us.count; ++i) {
      const int64_t u = us.unit(i);
      const int64_t r0 = u * p.R;
      const int nr = static_cast<int>((p.rows - r0 < p.R ? p.rows - r0 : (int64_t)p.R));
      // rows of this warp: one per stage pass when chunked (R == W), else j = cw + W*t
      const int rows_here = p.nchunks == 1 ? (nr > cw ? (nr - cw + kConsumerWarps - 1) / kConsumerWarps : 0)
                                           : (cw < nr ? 1 : 0);
      if (p.nchunks == 1) {
        mbar_wait(full + s, phase);
        const uint8_t* st = smem + static_cast<size_t>(s) * p.stage_bytes;
        for (int j = cw; j < nr; j += kConsumerWarps) {
          const int64_t row = r0 + j;
          uint32_t a, G;
          row_app_mask(st, r0, nr, row, a, G);
          select_app(a);
          const uint8_t* rowp = st + static_cast<int64_t>(j) * p.ld_bytes;
          float zp = -CUDART_INF_F, zm = -CUDART_INF_F;
          uint32_t kp = kNone, km = kNone;
          for (int e = lane; e < n_ent; e += 32) {
            const uint32_t key = ents[e];
            const float z = load_logit(rowp, key >> 8, BF16);
            if ((G >> (key & 0xFFu)) & 1u) {
              if (z > zp) { zp = z; kp = key; }
            } else {
              if (z > zm) { zm = z; km = key; }
            }
          }
          warp_argmax(zp, kp);
          warp_argmax(zm, km);
          if (b.n == lim) {  // several rows per warp in this stage
            finish_batch(p, b, wtab, lane);
            lim = 32;
          }
          deposit(b, lane, zp, kp, zm, km, G, a, row);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
        if (++s == p.stages) { s = 0; phase ^= 1u; }
        if (b.n == lim) {  // after the release; staggered over the warps (see the EPL path)
          finish_batch(p, b, wtab, lane);
          lim = 32;
        }
      } else {
        const bool mine = rows_here > 0;
        const int64_t row = r0 + cw;
        uint32_t a = 0, G = 0;
        float zp = -CUDART_INF_F, zm = -CUDART_INF_F;
        uint32_t kp = kNone, km = kNone;
        int pos = 0;
        for (int kc = 0; kc < p.nchunks; ++kc) {
          mbar_wait(full + s, phase);
          const uint8_t* st = smem + static_cast<size_t>(s) * p.stage_bytes;
          if (mine) {
            if (kc == 0) {
              row_app_mask(st, r0, nr, row, a, G);
              select_app(a);
            }
            const uint8_t* rowp = st + static_cast<int64_t>(cw) * p.chunk_bytes;
            const uint32_t c_lo = static_cast<uint32_t>(kc) * p.chunk_elems;
            const uint32_t c_hi = c_lo + p.chunk_elems;
            int stop = n_ent;
            for (int e = pos + lane; e < n_ent; e += 32) {
              const uint32_t key = ents[e];
              const uint32_t col = key >> 8;
              if (col >= c_hi) { stop = e; break; }
              const float z = load_logit(rowp, col - c_lo, BF16);
              if ((G >> (key & 0xFFu)) & 1u) {
                if (z > zp) { zp = z; kp = key; }
              } else {
                if (z > zm) { zm = z; km = key; }
              }
            }
            pos = static_cast<int>(__reduce_min_sync(kFull, static_cast<uint32_t>(stop)));
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + s);
          if (++s == p.stages) { s = 0; phase ^= 1u; }
        }
        if (mine) {
          warp_argmax(zp, kp);
          warp_argmax(zm, km);
          deposit(b, lane, zp, kp, zm, km, G, a, row);
          if (b.n == lim) {
            finish_batch(p, b, wtab, lane);
            lim = 32;
          }
        }
      }
    }
  }
  if (b.n > 0) finish_batch(p, b, wtab, lane);
}

// ------------------------------------------------------------------ sector-sparse gather kernel

// Load flavours (experiment, EvalParams::ld_flavor): 0 nc+L1::no_allocate, 1 .cg, 2 default, 3 .cs
__device__ __forceinline__ float ldg_stream_f32(const float* p, int fl) {
  float v;
  if (fl == 1) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if (fl == 2) asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if (fl == 3) asm volatile("ld.global.cs.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ float ldg_stream_bf16(const uint16_t* p, int fl) {
  unsigned short v;
  if (fl == 1) asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(v) : "l"(p));
  else if (fl == 2) asm volatile("ld.global.u16 %0, [%1];" : "=h"(v) : "l"(p));
  else if (fl == 3) asm volatile("ld.global.cs.u16 %0, [%1];" : "=h"(v) : "l"(p));
  else asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return __uint_as_float(static_cast<uint32_t>(v) << 16);
}

// The same computation as eval_kernel, but each lane loads only its mapped labels'
// logits straight from HBM (no shared-memory staging), so DRAM traffic is the 32-B
// sectors that hold mapped labels instead of whole rows.  A warp issues the loads of
// G rows (EPL per lane per row) before reducing any of them.
template <int EPL, int G, bool BF16, int PAT>
__global__ void __launch_bounds__(256) gather_kernel(const EvalParams p) {
  __shared__ float wtab_s[256];
  constexpr int kLB = PAT ? 8 * 32 * kListPad : 1;  // per-warp list-maxima batches (PAT 1)
  __shared__ float lbz_s[kLB];
  __shared__ uint32_t lbk_s[kLB];
  const int lane = threadIdx.x & 31;
  const bool wtab = p.wtab_off >= 0;
  if (wtab)
    for (int m = threadIdx.x; m < 256; m += blockDim.x) wtab_s[m] = __ldg(p.w + m);
  __syncthreads();
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t ngroups = (p.rows + G - 1) / G;

  LaneEnt<EPL> le;
  le.app = -1;
  RowBatch b;
  b.n = 0; b.zp = b.zm = 0.f; b.kp = b.km = kNone; b.G = 0; b.app = 0; b.row = 0;
  ListBatch lb;
  lb.z = lbz_s + (PAT ? (threadIdx.x >> 5) * 32 * kListPad : 0);
  lb.k = lbk_s + (PAT ? (threadIdx.x >> 5) * 32 * kListPad : 0);
  for (int64_t grp = gw; grp < ngroups; grp += nw) {
    const int64_t r0 = grp * G;
    const int nr = static_cast<int>(p.rows - r0 < G ? p.rows - r0 : G);
    int j = 0;
    while (j < nr) {
      // a run of rows [j, j+run) sharing one application
      const uint32_t a = p.app ? static_cast<uint32_t>(__ldg(p.app + r0 + j)) : 0u;
      int run = 1;
      if (p.app) {
        while (j + run < nr && __ldg(p.app + r0 + j + run) == a) ++run;
      } else {
        run = nr - j;
      }
      if (static_cast<int32_t>(a) != le.app) {
        const int32_t e0 = __ldg(p.ctx.ent_off + a);
        lane_ent_load(le, p.ctx.ent + e0, __ldg(p.ctx.ent_off + a + 1) - e0, static_cast<int32_t>(a), lane,
                      BF16 ? 2u : 4u, p.ctx.order);
      }
      // issue every load of the run first (memory-level parallelism), then reduce
      float z[G][EPL];
      uint32_t gm[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int64_t row = r0 + j + g;
        const uint8_t* rowp = p.logits + row * p.ld_bytes;
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          const bool ok = g < run && ((le.valid >> t) & 1u);
          if (BF16) z[g][t] = ok ? ldg_stream_bf16(reinterpret_cast<const uint16_t*>(rowp + le.off(t, 2u)), p.ld_flavor) : -CUDART_INF_F;
          else      z[g][t] = ok ? ldg_stream_f32(reinterpret_cast<const float*>(rowp + le.off(t, 4u)), p.ld_flavor) : -CUDART_INF_F;
        }
        gm[g] = (g < run && p.gt_mask) ? static_cast<uint32_t>(__ldg(p.gt_mask + row)) : 0u;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (g < run) {  // warp-uniform
          const int64_t row = r0 + j + g;
          uint32_t Gi = gm[g];
          if (!p.gt_mask && p.has_gt) Gi = warp_gt_mask(p, row, a, lane);
          if constexpr (PAT == 0) {
            float zp, zm;
            uint32_t kp, km;
            scan_vals<EPL>(le, plus_mask(le, Gi), z[g], zp, kp, zm, km);
            deposit(b, lane, zp, kp, zm, km, Gi, a, row);
            if (b.n == 32) finish_batch(p, b, wtab ? wtab_s : nullptr, lane);
          } else {
            scan_lists<EPL>(le, __ldg(p.ctx.nlists + a), z[g], lb, b.n, lane);
            deposit(b, lane, 0.f, kNone, 0.f, kNone, Gi, a, row);
            if (b.n == 32) finish_lists(p, b, lb, wtab ? wtab_s : nullptr, lane);
          }
        }
      }
      j += run;
    }
  }
  if (b.n > 0) {
    if constexpr (PAT == 0) finish_batch(p, b, wtab ? wtab_s : nullptr, lane);
    else finish_lists(p, b, lb, wtab ? wtab_s : nullptr, lane);
  }
}

// ------------------------------------------------------------------ GT-only pre-pass

// Warp-cooperative: a warp takes kHB blocks of 32 consecutive rows at once.  The rows'
// offsets are coalesced loads, their labels one contiguous span per block (the CSR keeps a
// row's labels adjacent) loaded coalesced; every load of all kHB blocks is issued before
// any is used, so a warp pays ~3 dependent latencies per 32·kHB rows.  Each label finds
// its row through a per-warp owner table and ORs its lists into that row's G with a
// shared atomic.  Optionally (w_out) the last CTA to finish turns the histogram into the
// weights (a7), saving a launch when the batch is the whole dataset (one GPU).
constexpr int kHB = 2;         // 32-row blocks in flight per warp
constexpr int kSpanCap = 128;  // labels per block handled by the owner table (4 per row)
constexpr int kSpanLd = kSpanCap / 32;

__device__ void weights_from_hist_block(const unsigned long long* hist, float* w, int n_apps);

__global__ void __launch_bounds__(256, 3) hist_kernel(const HistParams p) {
  extern __shared__ unsigned long long sh_hist[];
  __shared__ uint8_t owner_s[8][kHB][kSpanCap];
  __shared__ uint32_t g_s[8][kHB][32];
  __shared__ uint32_t app_s[8][kHB][32];
  __shared__ bool last_block;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nbins = p.ctx.n_apps * 256;
  if (p.smem_hist)
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) sh_hist[i] = 0;
  __syncthreads();
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  // software pipeline: the next group's offsets are in flight while this group is processed
  int64_t n_lo[kHB], n_hi[kHB];
  uint32_t n_a[kHB];
  auto prefetch = [&](int64_t r00) {
#pragma unroll
    for (int b = 0; b < kHB; ++b) {
      const int64_t row = r00 + b * 32 + lane;
      const bool act = row < p.rows;
      n_lo[b] = act ? __ldg(p.gt_off + row) : 0;
      n_hi[b] = act ? __ldg(p.gt_off + row + 1) : 0;
      n_a[b] = (act && p.app) ? static_cast<uint32_t>(__ldg(p.app + row)) : 0u;
    }
  };
  prefetch(gw * 32 * kHB);
  for (int64_t r00 = gw * 32 * kHB; r00 < p.rows; r00 += nw * 32 * kHB) {
    int64_t o_lo[kHB], o_hi[kHB], base[kHB], span[kHB];
    uint32_t a[kHB];
    unsigned amask[kHB];
#pragma unroll
    for (int b = 0; b < kHB; ++b) {
      o_lo[b] = n_lo[b];
      o_hi[b] = n_hi[b];
      a[b] = n_a[b];
    }
    prefetch(r00 + nw * 32 * kHB);
#pragma unroll
    for (int b = 0; b < kHB; ++b) {
      amask[b] = __ballot_sync(kFull, r00 + b * 32 + lane < p.rows);
      const int last = amask[b] ? 31 - __clz(amask[b]) : 0;
      base[b] = __shfl_sync(kFull, o_lo[b], 0);
      span[b] = amask[b] ? __shfl_sync(kFull, o_hi[b], last) - base[b] : 0;
    }
    int32_t lab[kHB][kSpanLd];
#pragma unroll
    for (int b = 0; b < kHB; ++b)
#pragma unroll
      for (int q = 0; q < kSpanLd; ++q) {
        const int pos = q * 32 + lane;
        lab[b][q] = (pos < span[b] && span[b] <= kSpanCap) ? __ldg(p.gt_lab + base[b] + pos) : -1;
      }
#pragma unroll
    for (int b = 0; b < kHB; ++b) {
      for (int64_t t = o_lo[b]; t < o_hi[b] && span[b] <= kSpanCap; ++t)
        owner_s[wib][b][t - base[b]] = static_cast<uint8_t>(lane);
      g_s[wib][b][lane] = 0;
      app_s[wib][b][lane] = a[b];
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < kHB; ++b)
#pragma unroll
      for (int q = 0; q < kSpanLd; ++q)
        if (lab[b][q] >= 0) {
          const int own = owner_s[wib][b][q * 32 + lane];
          const uint8_t* cat = p.ctx.cat + static_cast<int64_t>(app_s[wib][b][own]) * p.ctx.C;
          const uint32_t lists = label_lists(__ldg(cat + lab[b][q]), p.ctx.order);
          if (lists) atomicOr(&g_s[wib][b][own], lists);
        }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < kHB; ++b) {
      const int64_t row = r00 + b * 32 + lane;
      const bool act = row < p.rows;
      uint32_t G = g_s[wib][b][lane];
      if (span[b] > kSpanCap) {  // very long label lists (warp-uniform): one row per lane
        G = 0;
        const uint8_t* cat = p.ctx.cat + static_cast<int64_t>(a[b]) * p.ctx.C;
        for (int64_t t = o_lo[b]; t < o_hi[b]; ++t) G |= label_lists(__ldg(cat + __ldg(p.gt_lab + t)), p.ctx.order);
      }
      if (act && p.gt_mask_out) p.gt_mask_out[row] = static_cast<uint8_t>(G);
      if (p.hist_gt && act) {
        const uint32_t key = a[b] * 256u + G;
        const unsigned peers = __match_any_sync(amask[b], key);
        if (lane == __ffs(peers) - 1) {
          if (p.smem_hist) atomicAdd(sh_hist + key, static_cast<unsigned long long>(__popc(peers)));
          else atomicAdd(p.hist_gt + key, static_cast<unsigned long long>(__popc(peers)));
        }
      }
    }
    __syncwarp();
  }
  if (p.smem_hist && p.hist_gt) {
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x)
      if (sh_hist[i]) atomicAdd(p.hist_gt + i, sh_hist[i]);
  }
  if (p.w_out) {  // last CTA done: weights from the finished histogram
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last_block = atomicAdd(p.done_counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last_block) {
      __threadfence();
      weights_from_hist_block(p.hist_gt, p.w_out, p.ctx.n_apps);
      if (threadIdx.x == 0) *p.done_counter = 0;  // ready for the next call
    }
  }
}

// One row per thread for single-application contexts (the one-GPU step's pre-pass): the
// category table sits in shared memory, so a row is two coalesced offset loads, its labels
// (adjacent rows' labels are adjacent in the CSR) and shared-memory lookups; occupancy, not a
// software pipeline, hides the dependent loads.  Same outputs as hist_kernel.
__global__ void __launch_bounds__(256) hist_rows_kernel(const HistParams p) {
  extern __shared__ __align__(16) uint8_t hsm[];
  unsigned long long* sh_hist = reinterpret_cast<unsigned long long*>(hsm);  // [256]
  uint8_t* cat_s = hsm + 256 * 8;                                          // [C]
  __shared__ bool last_block;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sh_hist[i] = 0;
  // the table holds each label's list bits (label_lists), so a label costs one shared load and an OR
  for (int c = threadIdx.x; c < p.ctx.C; c += blockDim.x)
    cat_s[c] = static_cast<uint8_t>(label_lists(__ldg(p.ctx.cat + c), p.ctx.order));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * blockDim.x; r0 < p.rows; r0 += stride) {
    const int64_t row = r0 + threadIdx.x;
    const bool act = row < p.rows;
    uint32_t G = 0;
    if (act) {
      const int64_t lo = __ldg(p.gt_off + row);
      const int n = static_cast<int>(__ldg(p.gt_off + row + 1) - lo);
      const int32_t* lab = p.gt_lab + lo;
      for (int t = 0; t < n; ++t) G |= cat_s[__ldg(lab + t)];
      if (p.gt_mask_out) p.gt_mask_out[row] = static_cast<uint8_t>(G);
    }
    const unsigned am = __ballot_sync(kFull, act);
    if (p.hist_gt && act) {
      const unsigned peers = __match_any_sync(am, G);
      if (lane == __ffs(peers) - 1) atomicAdd(sh_hist + G, static_cast<unsigned long long>(__popc(peers)));
    }
  }
  __syncthreads();
  if (p.hist_gt)
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      if (sh_hist[i]) atomicAdd(p.hist_gt + i, sh_hist[i]);
  if (p.w_out) {  // last CTA done: weights from the finished histogram
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last_block = atomicAdd(p.done_counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last_block) {
      __threadfence();
      weights_from_hist_block(p.hist_gt, p.w_out, 1);
      if (threadIdx.x == 0) *p.done_counter = 0;  // ready for the next call
    }
  }
}

// ------------------------------------------------------------------ weights (a7)

// One CTA per app.  F = subset-sum (zeta) transform of H over 8 bits, so
// F[s] = #inputs whose G ⊆ s.  N(m) = M − F[~m] counts the inputs whose G
// intersects m; N(0) = H[0] counts non-target inputs (:2014).
__device__ void weights_one_app(const unsigned long long* H, float* w_app);

__global__ void __launch_bounds__(256) weights_kernel(const unsigned long long* hist, float* w) {
  weights_one_app(hist + static_cast<int64_t>(blockIdx.x) * 256, w + static_cast<int64_t>(blockIdx.x) * 256);
}

// All apps by one CTA (the hist kernel's last block).
__device__ void weights_from_hist_block(const unsigned long long* hist, float* w, int n_apps) {
  for (int a = 0; a < n_apps; ++a) {
    weights_one_app(hist + static_cast<int64_t>(a) * 256, w + static_cast<int64_t>(a) * 256);
    __syncthreads();
  }
}

// One app, 256 threads (a thread per mask).
__device__ void weights_one_app(const unsigned long long* H, float* w_app) {
  __shared__ unsigned long long F[256];
  const int m = threadIdx.x;
  const unsigned long long h = __ldcg(H + m);  // L2: the histogram was built by atomics
  F[m] = h;
#pragma unroll
  for (int bit = 0; bit < 8; ++bit) {
    __syncthreads();
    unsigned long long add = 0;
    if (m & (1 << bit)) add = F[m ^ (1 << bit)];
    __syncthreads();
    F[m] += add;
  }
  __syncthreads();
  const unsigned long long M = F[255];
  const unsigned long long N = m == 0 ? h : M - F[(~m) & 255];
  w_app[m] = N ? static_cast<float>(static_cast<double>(M) / static_cast<double>(N)) : 0.f;
  __syncthreads();
}

}  // namespace

template <int EPL, int PAT = 0, bool DEFER = false>
static cudaError_t set_limit_t(size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(eval_kernel<EPL, false, PAT, DEFER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e) return e;
  return cudaFuncSetAttribute(eval_kernel<EPL, true, PAT, DEFER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem));
}

#define SC_EVAL_EPLS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(12) X(16) X(24) X(32)
#define SC_EVAL_EPLS_PAT(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)  // per-list patterns: slots (PAT = 1)
#define SC_EVAL_NV_DM(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)     // dense-mapped rows: 16-B groups (PAT = 2)
#define SC_EVAL_EPLS_AC(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)   // application-choice, two maxima (PAT = 3)
#define SC_EVAL_EPLS_DEFER(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) // dense gradient parked (PAT 0 / 3, DEFER)

cudaError_t set_eval_smem_limit(size_t smem) {
  cudaError_t e = set_limit_t<0>(smem);
#define SC_SET(N) if (!e) e = set_limit_t<N>(smem);
  SC_EVAL_EPLS(SC_SET)
#undef SC_SET
#define SC_SET(N) if (!e) e = set_limit_t<N, 1>(smem);
  SC_EVAL_EPLS_PAT(SC_SET)
#undef SC_SET
#define SC_SET(N) if (!e) e = set_limit_t<N, 2>(smem);
  SC_EVAL_NV_DM(SC_SET)
#undef SC_SET
#define SC_SET(N) if (!e) e = set_limit_t<N, 3>(smem);
  SC_EVAL_EPLS_AC(SC_SET)
#undef SC_SET
#define SC_SET(N) if (!e) e = set_limit_t<N, 0, true>(smem); if (!e) e = set_limit_t<N, 3, true>(smem);
  SC_EVAL_EPLS_DEFER(SC_SET)
#undef SC_SET
  return e;
}

int eval_epl_for(int max_ent, int pat) {
  const int need = (max_ent + 31) / 32;
#define SC_PICK(N) if (need <= N) return N;
  if (pat) {
    SC_EVAL_EPLS_PAT(SC_PICK)
  } else {
    SC_EVAL_EPLS(SC_PICK)
  }
#undef SC_PICK
  return -1;
}

template <bool BF16>
static void launch_eval_dt(const EvalParams& p, int epl, int pat, int grid, size_t smem, cudaStream_t st) {
  if (p.pend_off >= 0) {  // dense gradient parked (host: PAT 0 / 3, epl <= 8)
    switch (epl) {
#define SC_CASE(N)                                                                \
  case N:                                                                         \
    if (pat == 3) eval_kernel<N, BF16, 3, true><<<grid, kThreads, smem, st>>>(p); \
    else eval_kernel<N, BF16, 0, true><<<grid, kThreads, smem, st>>>(p);          \
    break;
      SC_EVAL_EPLS_DEFER(SC_CASE)
#undef SC_CASE
      default: break;
    }
    return;
  }
  if (pat == 3) {
    switch (epl) {
#define SC_CASE(N) case N: eval_kernel<N, BF16, 3><<<grid, kThreads, smem, st>>>(p); break;
      SC_EVAL_EPLS_AC(SC_CASE)
#undef SC_CASE
      default: break;
    }
    return;
  }
  if (pat == 2) {
    switch (epl) {
#define SC_CASE(N) case N: eval_kernel<N, BF16, 2><<<grid, kThreads, smem, st>>>(p); break;
      SC_EVAL_NV_DM(SC_CASE)
#undef SC_CASE
      default: break;
    }
    return;
  }
  if (pat) {
    switch (epl) {
#define SC_CASE(N) case N: eval_kernel<N, BF16, 1><<<grid, kThreads, smem, st>>>(p); break;
      SC_EVAL_EPLS_PAT(SC_CASE)
#undef SC_CASE
      default: break;
    }
    return;
  }
  switch (epl) {
    case 0: eval_kernel<0, BF16, 0><<<grid, kThreads, smem, st>>>(p); break;
#define SC_CASE(N) case N: eval_kernel<N, BF16, 0><<<grid, kThreads, smem, st>>>(p); break;
    SC_EVAL_EPLS(SC_CASE)
#undef SC_CASE
    default: break;
  }
}

cudaError_t launch_eval(const EvalParams& p, int epl, int pat, int grid, size_t smem, cudaStream_t st) {
  if (pat && epl <= 0) return cudaErrorInvalidValue;  // the per-list patterns need lane-resident entries
  if (p.bf16) launch_eval_dt<true>(p, epl, pat, grid, smem, st);
  else launch_eval_dt<false>(p, epl, pat, grid, smem, st);
  return cudaGetLastError();
}

template <int EPL, int G, bool BF16, int PAT>
static cudaError_t launch_gather_t(const EvalParams& p, int sms, cudaStream_t st) {
  static const int blocks_per_sm = [] {  // thread-safe one-time occupancy query
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gather_kernel<EPL, G, BF16, PAT>, 256, 0);
    return n < 1 ? 1 : n;
  }();
  const int64_t warps_needed = (p.rows + G - 1) / G;
  int64_t grid = static_cast<int64_t>(sms) * blocks_per_sm;
  const int64_t max_grid = (warps_needed + 7) / 8;
  if (grid > max_grid) grid = max_grid;
  if (grid < 1) grid = 1;
  gather_kernel<EPL, G, BF16, PAT><<<static_cast<int>(grid), 256, 0, st>>>(p);
  return cudaGetLastError();
}

template <bool BF16, int PAT>
static cudaError_t launch_gather_dt(const EvalParams& p, int epl, int sms, cudaStream_t st) {
  switch (epl) {
    case 1: return launch_gather_t<1, 8, BF16, PAT>(p, sms, st);
    case 2: return launch_gather_t<2, 8, BF16, PAT>(p, sms, st);
    case 4: return launch_gather_t<4, 4, BF16, PAT>(p, sms, st);
    case 8: return launch_gather_t<8, 4, BF16, PAT>(p, sms, st);
    case 16: return launch_gather_t<16, 2, BF16, PAT>(p, sms, st);
    default: return launch_gather_t<32, 1, BF16, PAT>(p, sms, st);
  }
}

cudaError_t launch_gather(const EvalParams& p, int epl, int pat, int sms, cudaStream_t st) {
  if (pat) return p.bf16 ? launch_gather_dt<true, 1>(p, epl, sms, st) : launch_gather_dt<false, 1>(p, epl, sms, st);
  return p.bf16 ? launch_gather_dt<true, 0>(p, epl, sms, st) : launch_gather_dt<false, 0>(p, epl, sms, st);
}

cudaError_t launch_hist(const HistParams& p, int grid, size_t smem, cudaStream_t st) {
  hist_kernel<<<grid, 256, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_hist_rows(const HistParams& p, int grid, cudaStream_t st) {
  const size_t smem = 256 * 8 + static_cast<size_t>(p.ctx.C);
  if (smem > 48 * 1024) {
    // thread-safe one-time opt-in to large dynamic shared memory (C > ~46K labels)
    static const cudaError_t attr =
        cudaFuncSetAttribute(hist_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (attr) return attr;
  }
  hist_rows_kernel<<<grid, 256, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_weights(const unsigned long long* hist, float* w, int n_apps, cudaStream_t st) {
  weights_kernel<<<n_apps, 256, 0, st>>>(hist, w);
  return cudaGetLastError();
}

}  // namespace sc
