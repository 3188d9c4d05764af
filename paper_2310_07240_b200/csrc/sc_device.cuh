// sc_device.cuh — device helpers shared by the libsc kernels (sc_kernels.cu, sc_head.cu):
// PTX wrappers (mbarrier, bulk copies, streaming stores), the fp32 math of the loss
// (reading A2), and the per-row epilogue of the API-output order (rows a3-a9 of
// SURVEY.md §8(a)).  Internal; nothing here is shared with oracle/.
#pragma once
#include "sc_internal.cuh"

#include <cuda_runtime.h>
#include <math_constants.h>

namespace sc {
namespace {


constexpr unsigned kFull = 0xFFFFFFFFu;

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SC_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SC_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void st_cs_f4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// Side band of rows [r0, r0 + nr) of a per-row array (elt bytes per row): the 16-B-aligned
// interior [r0·elt + head, r0·elt + head + nb) is what a bulk copy may move (its source and
// size must be 16-B multiples); the ragged head and tail rows are read from global memory,
// so nothing outside the caller's array is ever read.  Byte offset o = j·elt of row r0 + j
// lies in the window iff (o − head) < nb as unsigned.
struct SideBand {
  uint32_t head, nb;
};
__device__ __forceinline__ SideBand sb_window(const void* base, int64_t r0, int nr, uint32_t elt) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(base) + static_cast<uintptr_t>(r0) * elt;
  const uintptr_t a1 = a0 + static_cast<uintptr_t>(nr) * elt;
  const uintptr_t lo = (a0 + 15) & ~uintptr_t(15), hi = a1 & ~uintptr_t(15);
  return SideBand{static_cast<uint32_t>(lo - a0), hi > lo ? static_cast<uint32_t>(hi - lo) : 0u};
}

// ------------------------------------------------------------------ math (fp32, no fast-math)

// σ(z) = 1/(1+e^{-z}) without overflow (reading A2).
__device__ __forceinline__ float sigmoid_f(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

// σ'(z) = t/(1+t)^2, t = e^{-|z|}: no cancellation (σ(1-σ) in fp32 loses digits for |z| > 8).
__device__ __forceinline__ float dsigmoid_f(float z) {
  const float t = expf(-fabsf(z));
  const float d = 1.f + t;
  return t / (d * d);
}

// σ(z) and σ'(z) from one exponential and one division: t = e^{-|z|}, r = 1/(1+t); σ = r
// (z >= 0) or t·r, σ' = t·r² (sigmoid_f / dsigmoid_f's forms, one or two more roundings).
// Used by the Multi-Select epilogue, which needs both at every list's maximum and at every
// S argument: 0.749 -> 0.68-0.70 ms on cfg2.  (Used in every epilogue it made the others
// slower on the same box — f32 0.592 -> 0.615 ms, bf16, the head — so they keep the separate
// calls; profiles/r5e_*.)
__device__ __forceinline__ void sig_dsig_f(float z, float& s, float& ds) {
  const float t = expf(-fabsf(z));
  const float r = 1.f / (1.f + t);
  s = z >= 0.f ? r : t * r;
  ds = t * r * r;
}

// Lexicographic max over (z, -label): keys are c << 8 | cat, ordered like c.
__device__ __forceinline__ bool beats(float zo, uint32_t ko, float z, uint32_t k) {
  return zo > z || (zo == z && ko < k);
}

__device__ __forceinline__ float load_logit(const uint8_t* rowp, uint32_t col, int bf16) {
  if (bf16) return __uint_as_float(static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(rowp + 2u * col)) << 16);
  return *reinterpret_cast<const float*>(rowp + 4u * col);
}

// G_i from the CSR ground truth (a2): OR of 1 << cat[c] over ŷ_i.
__device__ __forceinline__ uint32_t warp_gt_mask(const EvalParams& p, int64_t row, uint32_t a, int lane) {
  const int64_t b = __ldg(p.gt_off + row), e = __ldg(p.gt_off + row + 1);
  uint32_t G = 0;
  const uint8_t* cat = p.ctx.cat + static_cast<int64_t>(a) * p.ctx.C;
  for (int64_t t = b + lane; t < e; t += 32) G |= label_lists(__ldg(cat + __ldg(p.gt_lab + t)), p.ctx.order);
  return __reduce_or_sync(kFull, G);
}

// ------------------------------------------------------------------ per-warp row batch

// Results of up to 32 reduced rows, one row per lane, finished together.
struct RowBatch {
  float zp, zm;      // max logit over 𝒲_i (P⁺ side) and over 𝕎∖𝒲_i (P⁻ side)
  uint32_t kp, km;   // their keys (label << 8 | cat), kNone if the set is empty
  uint32_t G, app;
  uint32_t lo = 0;   // application-choice order: the lists holding an output label (z > tau)
  int64_t row;
  int n;             // rows held (warp-uniform)
};

// Dense gradient rows of a batch not yet written (kDefer epilogues of the TMA-ring kernel) are
// parked in a per-warp shared-memory slab (kPendSlab bytes at EvalParams::pend_off; nothing
// held in registers) and written a few at a time between stages (dense_drain) instead of as
// one 32-row burst per batch.  Slab: {int32 np (rows parked), int32 pt (next to write), pad},
// the rows' indices (int64 [32]), then {c0, c1, v0, v1} per row (16 B [32]).
__device__ __forceinline__ uint32_t pend_slab(const EvalParams& p) {
  extern __shared__ __align__(128) uint8_t smem[];
  return smem_addr(smem) + static_cast<uint32_t>(p.pend_off) + ((threadIdx.x >> 5) - 1u) * kPendSlab;
}

// One dense gradient row (a9, optional dense layout): zeros except columns c0 / c1, written
// coalesced by the warp with streaming 16-B stores.
__device__ __forceinline__ void dense_row_store(const EvalParams& p, int64_t row, int32_t c0, int32_t c1, float v0,
                                                float v1, int lane) {
  float* out = p.grad_dense + row * p.ld;
  const int32_t nv = static_cast<int32_t>(p.ld >> 2);
  for (int32_t v = lane; v < nv; v += 32) {
    float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int32_t c = 4 * v + q;
      if (c == c0) e[q] = v0;
      if (c == c1) e[q] = v1;
    }
    st_cs_f4(out + 4 * v, make_float4(e[0], e[1], e[2], e[3]));
  }
}

// Write up to `upto` parked dense gradient rows of this warp (call with the whole warp).
__device__ __forceinline__ void dense_drain(const EvalParams& p, int lane, int upto) {
  const uint32_t slab = pend_slab(p);
  uint32_t np, pt;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(np), "=r"(pt) : "r"(slab));
  if (pt >= np) return;  // warp-uniform
  const uint32_t end = np < pt + static_cast<uint32_t>(upto) ? np : pt + static_cast<uint32_t>(upto);
  for (uint32_t t = pt; t < end; ++t) {
    int64_t row;
    uint32_t c0, c1, v0, v1;
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(row) : "r"(slab + 16u + 8u * t));
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(c0), "=r"(c1), "=r"(v0), "=r"(v1)
                 : "r"(slab + 272u + 16u * t));
    dense_row_store(p, row, static_cast<int32_t>(c0), static_cast<int32_t>(c1), __uint_as_float(v0),
                    __uint_as_float(v1), lane);
  }
  __syncwarp();
  if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(slab + 4u), "r"(end) : "memory");
  __syncwarp();
}

// The batch's dense gradient rows: written now, or (kDefer, when the kernel planned slabs)
// parked after the previous batch's leftovers are flushed; the caller drains them.
template <bool kDefer>
__device__ __forceinline__ void dense_pair_rows(const EvalParams& p, RowBatch& b, int lane, int32_t i0, int32_t i1,
                                                float g0, float g1) {
  if (kDefer && p.pend_off >= 0) {
    dense_drain(p, lane, 32);
    const uint32_t slab = pend_slab(p), l = static_cast<uint32_t>(lane);
    if (lane < b.n) {
      asm volatile("st.shared.s64 [%0], %1;" ::"r"(slab + 16u + 8u * l), "l"(b.row) : "memory");
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(slab + 272u + 16u * l), "r"(i0), "r"(i1),
                   "r"(__float_as_uint(g0)), "r"(__float_as_uint(g1))
                   : "memory");
    }
    if (lane == 0)
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(slab), "r"(static_cast<uint32_t>(b.n)), "r"(0u) : "memory");
    __syncwarp();
  } else {
    for (int t = 0; t < b.n; ++t)
      dense_row_store(p, __shfl_sync(kFull, b.row, t), __shfl_sync(kFull, i0, t), __shfl_sync(kFull, i1, t),
                      __shfl_sync(kFull, g0, t), __shfl_sync(kFull, g1, t), lane);
  }
}

template <bool kDefer = false>
__device__ __forceinline__ void finish_batch(const EvalParams& p, RowBatch& b, const float* wtab_smem, int lane) {
  const bool active = lane < b.n;
  const unsigned act = __ballot_sync(kFull, active);
  const float tau = p.ctx.tau;
  uint32_t dec = 0, correct = 1;
  float L = 0.f, g0 = 0.f, g1 = 0.f;
  int32_t i0 = -1, i1 = -1;
  if (active) {
    const uint32_t D = __ldg(p.ctx.nlists + b.app);
    const bool has_p = b.kp != kNone, has_m = b.km != kNone;
    const bool take_p = has_p && (!has_m || beats(b.zp, b.kp, b.zm, b.km));
    const float zs = take_p ? b.zp : b.zm;
    const uint32_t ks = take_p ? b.kp : b.km;
    // a3: first mapped label in confidence order, if it is an API output (z > tau)
    dec = ((has_p || has_m) && zs > tau) ? (ks & 0xFFu) : D;
    const bool y = b.G != 0;
    // a5: Decision(API(x)) ∈ Decision(ŷ) (reading A7)
    correct = y ? (dec < D && ((b.G >> dec) & 1u)) : (dec == D);
    if (p.decision) p.decision[b.row] = static_cast<uint8_t>(dec);
    if (p.want_loss) {
      // a8/a9: Eq. api_output and its gradient
      const float wi = p.w ? (wtab_smem ? wtab_smem[b.G] : __ldg(p.w + b.app * 256u + b.G)) : 1.f;
      const float k = p.ctx.k;
      if (y && has_p) {  // y_i = 1 implies 𝒲_i ≠ ∅ for a G consistent with the context
        const float pp = sigmoid_f(b.zp);
        const bool m_over = has_m && b.zm > tau;
        const float am = m_over ? sigmoid_f(b.zm) : p.ctx.theta;  // max(P⁻, θ)
        const float x = am - pp;
        const float ell = sigmoid_f(k * x);                          // S(x)
        const float ds = k * dsigmoid_f(k * x);                      // S'(x)
        L = wi * ell;
        g0 = -wi * ds * dsigmoid_f(b.zp) * p.grad_scale;
        i0 = static_cast<int32_t>(b.kp >> 8);
        if (m_over) {
          g1 = wi * ds * dsigmoid_f(b.zm) * p.grad_scale;
          i1 = static_cast<int32_t>(b.km >> 8);
        }
      } else if (!y && has_m) {
        const float x = sigmoid_f(b.zm) - p.ctx.theta;               // P⁻ − θ
        const float ell = sigmoid_f(k * x);
        const float ds = k * dsigmoid_f(k * x);
        L = wi * ell;
        g1 = wi * ds * dsigmoid_f(b.zm) * p.grad_scale;
        i1 = static_cast<int32_t>(b.km >> 8);
      }
      if (p.loss_row) p.loss_row[b.row] = L;
      if (p.grad_idx) {  // label ids (i0 / i1 are logit columns, which differ for compacted rows)
        p.grad_idx[2 * b.row] = out_label(p.ctx, i0);
        p.grad_idx[2 * b.row + 1] = out_label(p.ctx, i1);
      }
      if (p.grad_val) {
        p.grad_val[2 * b.row] = g0;
        p.grad_val[2 * b.row + 1] = g1;
      }
    }
  }
  // a6 / a5 counters: one atomic per distinct (app, bin) in the warp.
  if (p.hist_pred && active) {
    const uint32_t key = b.app * 256u + dec;
    const unsigned peers = __match_any_sync(act, key);
    if (lane == __ffs(peers) - 1) atomicAdd(p.hist_pred + key, static_cast<unsigned long long>(__popc(peers)));
  }
  if (p.has_gt) {
    if (p.hist_gt && active) {
      const uint32_t key = b.app * 256u + b.G;
      const unsigned peers = __match_any_sync(act, key);
      if (lane == __ffs(peers) - 1) atomicAdd(p.hist_gt + key, static_cast<unsigned long long>(__popc(peers)));
    }
    const unsigned inc = __ballot_sync(kFull, active && !correct);
    if (p.n_incorrect && (inc >> lane & 1u)) {
      const unsigned peers = __match_any_sync(inc, b.app);
      if (lane == __ffs(peers) - 1) atomicAdd(p.n_incorrect + b.app, static_cast<unsigned long long>(__popc(peers)));
    }
    if (p.loss_sum && p.want_loss) {
      const uint32_t app0 = __shfl_sync(kFull, b.app, 0);
      if (__all_sync(kFull, !active || b.app == app0)) {
        double s = active ? static_cast<double>(L) : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
        if (lane == 0) atomicAdd(p.loss_sum + app0, s);
      } else if (active) {
        atomicAdd(p.loss_sum + b.app, static_cast<double>(L));
      }
    }
  }
  // dense gradient: the warp writes each row coalesced (zeros + <= 2 entries)
  if (p.grad_dense) dense_pair_rows<kDefer>(p, b, lane, i0, i1, g0, g1);
  b.n = 0;
}

// a3-a9 epilogue of the per-list patterns for the batch's rows, one row per lane, from each
// row's per-list arg maxima (zj[j], kj[j]) (P_j of PAPER.md:2026, :2050): the application-choice
// order (Eq. app_choice) and Multi-Select (Eq. multi-select); counters as in finish_batch.
// Used by the eval / gather kernels (sc_kernels.cu) and the fused head (sc_head.cu).
__device__ __forceinline__ void finish_lists_core(const EvalParams& p, RowBatch& b, const float (&zj)[8],
                                                  const uint32_t (&kj)[8], const float* wtab_smem, int lane) {
  const bool active = lane < b.n;
  const unsigned act = __ballot_sync(kFull, active);
  const float tau = p.ctx.tau, theta = p.ctx.theta, k = p.ctx.k;
  const bool ms = p.ctx.order == kMultiSelect;
  const int S = ms ? 8 : 2;
  uint32_t dec = 0, correct = 1;
  float L = 0.f;
  int32_t gi[8];
  float gv[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) { gi[q] = -1; gv[q] = 0.f; }
  if (active) {
    const int D = __ldg(p.ctx.nlists + b.app);
    const uint32_t G = b.G;
    const bool y = G != 0;
    const float wi = p.w ? (wtab_smem ? wtab_smem[G] : __ldg(p.w + b.app * 256u + G)) : 1.f;
    if (!ms) {
      // application-choice order: the first list (code order) holding an output label
      dec = static_cast<uint32_t>(D);
#pragma unroll
      for (int j = 7; j >= 0; --j)
        if (kj[j] != kNone && zj[j] > tau) dec = static_cast<uint32_t>(j);
      const int kk = y ? __ffs(G) - 1 : D;  // the ground truth's decision
      correct = dec == static_cast<uint32_t>(kk);
      if (p.want_loss) {
        // competitor: lists j < k when y = 1 (P_{k⁻}), every list when y = 0 (P)
        float zc = -CUDART_INF_F;
        uint32_t kc = kNone;
        float zk = -CUDART_INF_F;
        uint32_t kk_key = kNone;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j == kk) { zk = zj[j]; kk_key = kj[j]; }
          const bool compete = y ? (j < kk) : (j < D);
          if (compete && kj[j] != kNone && beats(zj[j], kj[j], zc, kc)) { zc = zj[j]; kc = kj[j]; }
        }
        if (y && kk_key != kNone) {
          const bool c_over = kc != kNone && zc > tau;
          const float am = c_over ? sigmoid_f(zc) : theta;  // max(θ, P_{k⁻})
          const float x = am - sigmoid_f(zk);
          const float ds = k * dsigmoid_f(k * x);
          L = wi * sigmoid_f(k * x);
          gi[0] = static_cast<int32_t>(kk_key >> 8);
          gv[0] = -wi * ds * dsigmoid_f(zk) * p.grad_scale;
          if (c_over) {
            gi[1] = static_cast<int32_t>(kc >> 8);
            gv[1] = wi * ds * dsigmoid_f(zc) * p.grad_scale;
          }
        } else if (!y && kc != kNone) {
          const float x = sigmoid_f(zc) - theta;  // P − θ
          L = wi * sigmoid_f(k * x);
          gi[1] = static_cast<int32_t>(kc >> 8);
          gv[1] = wi * k * dsigmoid_f(k * x) * dsigmoid_f(zc) * p.grad_scale;
        }
      }
    } else {
      // Multi-Select: every list holding an output label; exact match with G
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (kj[j] != kNone && zj[j] > tau) dec |= 1u << j;
      correct = dec == G;
      if (p.want_loss) {
        float ell = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (kj[j] != kNone) {
            float pj, dpj, sx, dsx;
            sig_dsig_f(zj[j], pj, dpj);
            const bool yj = (G >> j) & 1u;
            const float x = yj ? theta - pj : pj - theta;
            sig_dsig_f(k * x, sx, dsx);
            ell += sx;
            const float g = wi * k * dsx * dpj * p.grad_scale;
            gi[j] = static_cast<int32_t>(kj[j] >> 8);
            gv[j] = yj ? -g : g;
          }
        }
        L = wi * ell;
      }
    }
    if (p.decision) p.decision[b.row] = static_cast<uint8_t>(dec);
    if (p.want_loss) {
      if (p.loss_row) p.loss_row[b.row] = L;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < S) {
          if (p.grad_idx) p.grad_idx[S * b.row + q] = out_label(p.ctx, gi[q]);  // gi: logit columns
          if (p.grad_val) p.grad_val[S * b.row + q] = gv[q];
        }
      }
    }
  }
  if (p.hist_pred && active) {
    const uint32_t key = b.app * 256u + dec;
    const unsigned peers = __match_any_sync(act, key);
    if (lane == __ffs(peers) - 1) atomicAdd(p.hist_pred + key, static_cast<unsigned long long>(__popc(peers)));
  }
  if (p.has_gt) {
    if (p.hist_gt && active) {
      const uint32_t key = b.app * 256u + b.G;
      const unsigned peers = __match_any_sync(act, key);
      if (lane == __ffs(peers) - 1) atomicAdd(p.hist_gt + key, static_cast<unsigned long long>(__popc(peers)));
    }
    const unsigned inc = __ballot_sync(kFull, active && !correct);
    if (p.n_incorrect && (inc >> lane & 1u)) {
      const unsigned peers = __match_any_sync(inc, b.app);
      if (lane == __ffs(peers) - 1) atomicAdd(p.n_incorrect + b.app, static_cast<unsigned long long>(__popc(peers)));
    }
    if (p.loss_sum && p.want_loss) {
      double sl = active ? static_cast<double>(L) : 0.0;
      const uint32_t app0 = __shfl_sync(kFull, b.app, 0);
      if (__all_sync(kFull, !active || b.app == app0)) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sl += __shfl_xor_sync(kFull, sl, off);
        if (lane == 0) atomicAdd(p.loss_sum + app0, sl);
      } else if (active) {
        atomicAdd(p.loss_sum + b.app, sl);
      }
    }
  }
  if (p.grad_dense) {
    for (int t = 0; t < b.n; ++t) {
      const int64_t row = __shfl_sync(kFull, b.row, t);
      int32_t ci[8];
      float cv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        ci[q] = __shfl_sync(kFull, gi[q], t);
        cv[q] = __shfl_sync(kFull, gv[q], t);
      }
      float* out = p.grad_dense + row * p.ld;
      const int64_t nv = p.ld >> 2;
      for (int64_t v = lane; v < nv; v += 32) {
        float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int64_t c = 4 * v + q4;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (c == ci[q]) e[q4] += cv[q];  // Multi-Select: one label may lead several lists
        }
        st_cs_f4(out + 4 * v, make_float4(e[0], e[1], e[2], e[3]));
      }
    }
  }
  __syncwarp();
  b.n = 0;
}

__device__ __forceinline__ void deposit(RowBatch& b, int lane, float zp, uint32_t kp, float zm, uint32_t km,
                                        uint32_t G, uint32_t a, int64_t row, uint32_t lo = 0) {
  if (lane == b.n) {
    b.zp = zp; b.kp = kp; b.zm = zm; b.km = km; b.G = G; b.app = a; b.row = row; b.lo = lo;
  }
  ++b.n;
}

// The application-choice order (Eq. app_choice, reading A21) from two
// arg maxima per row instead of one per list: with k = the lowest list of G_i, (zp, kp) is
// the arg max over list k (P_k) and (zm, km) the arg max over lists j < k (P_{k⁻}); for
// G_i = ∅ (zm, km) is over all of 𝕎 (P).  The decision is the first list holding an output
// label (b.lo: lists with some z > tau).  Same formulas, in the same order, as the per-list
// epilogue (finish_lists_core), so both give identical values.
template <bool kDefer = false>
__device__ __forceinline__ void finish_app_choice(const EvalParams& p, RowBatch& b, const float* wtab_smem, int lane) {
  const bool active = lane < b.n;
  const unsigned act = __ballot_sync(kFull, active);
  const float tau = p.ctx.tau, theta = p.ctx.theta, k = p.ctx.k;
  uint32_t dec = 0, correct = 1;
  float L = 0.f, g0 = 0.f, g1 = 0.f;
  int32_t i0 = -1, i1 = -1;
  if (active) {
    const uint32_t D = __ldg(p.ctx.nlists + b.app);
    const uint32_t G = b.G;
    const bool y = G != 0;
    dec = b.lo ? static_cast<uint32_t>(__ffs(b.lo) - 1) : D;
    const uint32_t kk = y ? static_cast<uint32_t>(__ffs(G) - 1) : D;
    correct = dec == kk;
    if (p.decision) p.decision[b.row] = static_cast<uint8_t>(dec);
    if (p.want_loss) {
      const float wi = p.w ? (wtab_smem ? wtab_smem[G] : __ldg(p.w + b.app * 256u + G)) : 1.f;
      if (y && b.kp != kNone) {
        const bool c_over = b.km != kNone && b.zm > tau;
        const float am = c_over ? sigmoid_f(b.zm) : theta;  // max(θ, P_{k⁻})
        const float x = am - sigmoid_f(b.zp);
        const float ds = k * dsigmoid_f(k * x);
        L = wi * sigmoid_f(k * x);
        i0 = static_cast<int32_t>(b.kp >> 8);
        g0 = -wi * ds * dsigmoid_f(b.zp) * p.grad_scale;
        if (c_over) {
          i1 = static_cast<int32_t>(b.km >> 8);
          g1 = wi * ds * dsigmoid_f(b.zm) * p.grad_scale;
        }
      } else if (!y && b.km != kNone) {
        const float x = sigmoid_f(b.zm) - theta;  // P − θ
        L = wi * sigmoid_f(k * x);
        i1 = static_cast<int32_t>(b.km >> 8);
        g1 = wi * k * dsigmoid_f(k * x) * dsigmoid_f(b.zm) * p.grad_scale;
      }
      if (p.loss_row) p.loss_row[b.row] = L;
      if (p.grad_idx) {
        p.grad_idx[2 * b.row] = out_label(p.ctx, i0);
        p.grad_idx[2 * b.row + 1] = out_label(p.ctx, i1);
      }
      if (p.grad_val) {
        p.grad_val[2 * b.row] = g0;
        p.grad_val[2 * b.row + 1] = g1;
      }
    }
  }
  if (p.hist_pred && active) {
    const uint32_t key = b.app * 256u + dec;
    const unsigned peers = __match_any_sync(act, key);
    if (lane == __ffs(peers) - 1) atomicAdd(p.hist_pred + key, static_cast<unsigned long long>(__popc(peers)));
  }
  if (p.has_gt) {
    if (p.hist_gt && active) {
      const uint32_t key = b.app * 256u + b.G;
      const unsigned peers = __match_any_sync(act, key);
      if (lane == __ffs(peers) - 1) atomicAdd(p.hist_gt + key, static_cast<unsigned long long>(__popc(peers)));
    }
    const unsigned inc = __ballot_sync(kFull, active && !correct);
    if (p.n_incorrect && (inc >> lane & 1u)) {
      const unsigned peers = __match_any_sync(inc, b.app);
      if (lane == __ffs(peers) - 1) atomicAdd(p.n_incorrect + b.app, static_cast<unsigned long long>(__popc(peers)));
    }
    if (p.loss_sum && p.want_loss) {
      double sl = active ? static_cast<double>(L) : 0.0;
      const uint32_t app0 = __shfl_sync(kFull, b.app, 0);
      if (__all_sync(kFull, !active || b.app == app0)) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sl += __shfl_xor_sync(kFull, sl, off);
        if (lane == 0) atomicAdd(p.loss_sum + app0, sl);
      } else if (active) {
        atomicAdd(p.loss_sum + b.app, sl);
      }
    }
  }
  if (p.grad_dense) dense_pair_rows<kDefer>(p, b, lane, i0, i1, g0, g1);
  __syncwarp();
  b.n = 0;
}

// Shared-memory loads by 32-bit shared address (no generic-to-shared conversion per load).
// volatile keeps them after the mbarrier wait that makes the TMA bytes visible.
template <bool BF16>
__device__ __forceinline__ float lds_z(uint32_t a) {
  if constexpr (BF16) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return __uint_as_float(static_cast<uint32_t>(v) << 16);
  } else {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
  }
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

}  // namespace
}  // namespace sc
