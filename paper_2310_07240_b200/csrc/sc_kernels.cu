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

// Lexicographic max over (z, -label): keys are c << 8 | cat, ordered like c.
__device__ __forceinline__ bool beats(float zo, uint32_t ko, float z, uint32_t k) {
  return zo > z || (zo == z && ko < k);
}

__device__ __forceinline__ void warp_lexmax(float& z, uint32_t& k) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float zo = __shfl_xor_sync(kFull, z, off);
    const uint32_t ko = __shfl_xor_sync(kFull, k, off);
    if (beats(zo, ko, z, k)) {
      z = zo;
      k = ko;
    }
  }
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
  for (int64_t t = b + lane; t < e; t += 32) {
    const uint8_t v = __ldg(cat + __ldg(p.gt_lab + t));
    if (v != kCatNone) G |= 1u << v;
  }
  return __reduce_or_sync(kFull, G);
}

// ------------------------------------------------------------------ per-warp row batch

// Results of up to 32 reduced rows, one row per lane, finished together.
struct RowBatch {
  float zp, zm;      // max logit over 𝒲_i (P⁺ side) and over 𝕎∖𝒲_i (P⁻ side)
  uint32_t kp, km;   // their keys (label << 8 | cat), kNone if the set is empty
  uint32_t G, app;
  int64_t row;
  int n;             // rows held (warp-uniform)
};

// a3-a9 epilogue for the rows in the batch: decision, correctness, loss and
// gradient; per-row outputs and warp-aggregated counter atomics.
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
      if (p.grad_idx) {
        p.grad_idx[2 * b.row] = i0;
        p.grad_idx[2 * b.row + 1] = i1;
      }
      if (p.grad_val) {
        p.grad_val[2 * b.row] = g0;
        p.grad_val[2 * b.row + 1] = g1;
      }
    }
  }
  // a6 / a5 counters: one atomic per distinct (app, bin) in the warp.
  if (p.hist_pred && active) {
    const uint32_t key = b.app * 16u + dec;
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
  if (p.grad_dense) {
    for (int t = 0; t < b.n; ++t) {
      const int64_t row = __shfl_sync(kFull, b.row, t);
      const int32_t c0 = __shfl_sync(kFull, i0, t), c1 = __shfl_sync(kFull, i1, t);
      const float v0 = __shfl_sync(kFull, g0, t), v1 = __shfl_sync(kFull, g1, t);
      float* out = p.grad_dense + row * p.ld;
      const int64_t nv = p.ld >> 2;
      for (int64_t v = lane; v < nv; v += 32) {
        float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t c = 4 * v + q;
          if (c == c0) e[q] = v0;
          if (c == c1) e[q] = v1;
        }
        st_cs_f4(out + 4 * v, make_float4(e[0], e[1], e[2], e[3]));
      }
    }
  }
  b.n = 0;
}

__device__ __forceinline__ void deposit(RowBatch& b, int lane, float zp, uint32_t kp, float zm, uint32_t km,
                                        uint32_t G, uint32_t a, int64_t row) {
  if (lane == b.n) {
    b.zp = zp; b.kp = kp; b.zm = zm; b.km = km; b.G = G; b.app = a; b.row = row;
  }
  ++b.n;
}

// ------------------------------------------------------------------ fused evaluation kernel

__global__ void __launch_bounds__(kThreads, 1) eval_kernel(const EvalParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- prologue: barriers, context entries and weights into shared memory
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps);
    }
    fence_mbar_init();
  }
  uint32_t* ent_smem = reinterpret_cast<uint32_t*>(smem + p.ent_smem_off);
  if (p.ent_mode == 0) {
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
      const uint64_t pol = evict_first_policy();
      int s = 0;
      uint32_t phase = 0;
      for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x) {
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
            if (p.gt_mask) {
              const uintptr_t lo = reinterpret_cast<uintptr_t>(p.gt_mask + r0) & ~uintptr_t(15);
              const uintptr_t hi = (reinterpret_cast<uintptr_t>(p.gt_mask + r0 + nr) + 15) & ~uintptr_t(15);
              src_m = reinterpret_cast<const uint8_t*>(lo);
              nb_m = static_cast<uint32_t>(hi - lo);
            }
            if (p.app) {
              const uintptr_t lo = reinterpret_cast<uintptr_t>(p.app + r0) & ~uintptr_t(15);
              const uintptr_t hi = (reinterpret_cast<uintptr_t>(p.app + r0 + nr) + 15) & ~uintptr_t(15);
              src_a = reinterpret_cast<const uint8_t*>(lo);
              nb_a = static_cast<uint32_t>(hi - lo);
            }
          }
          if (p.nchunks == 1) {
            bytes = static_cast<uint32_t>(nr * p.ld_bytes);
          } else {
            const int rem = p.copy_row_bytes - kc * p.chunk_bytes;
            const uint32_t cb = static_cast<uint32_t>(rem < p.chunk_bytes ? rem : p.chunk_bytes);
            bytes = cb * nr;
          }
          mbar_arrive_expect_tx(full + s, bytes + nb_m + nb_a);
          if (p.nchunks == 1) {
            bulk_g2s(st, p.logits + r0 * p.ld_bytes, bytes, full + s, pol);
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

  auto row_app_mask = [&](const uint8_t* st, int64_t r0, int64_t row, uint32_t& a, uint32_t& G) {
    a = 0;
    if (p.app) {
      const uintptr_t lo = reinterpret_cast<uintptr_t>(p.app + r0) & ~uintptr_t(15);
      a = *reinterpret_cast<const uint16_t*>(st + p.app_off + (reinterpret_cast<uintptr_t>(p.app + row) - lo));
    }
    G = 0;
    if (p.gt_mask) {
      const uintptr_t lo = reinterpret_cast<uintptr_t>(p.gt_mask + r0) & ~uintptr_t(15);
      G = st[p.mask_off + (reinterpret_cast<uintptr_t>(p.gt_mask + row) - lo)];
    } else if (p.has_gt) {
      G = warp_gt_mask(p, row, a, lane);
    }
  };

  int s = 0;
  uint32_t phase = 0;
  for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x) {
    const int64_t r0 = u * p.R;
    const int nr = static_cast<int>((p.rows - r0 < p.R ? p.rows - r0 : (int64_t)p.R));
    if (p.nchunks == 1) {
      mbar_wait(full + s, phase);
      const uint8_t* st = smem + static_cast<size_t>(s) * p.stage_bytes;
      for (int j = cw; j < nr; j += kConsumerWarps) {
        const int64_t row = r0 + j;
        uint32_t a, G;
        row_app_mask(st, r0, row, a, G);
        select_app(a);
        const uint8_t* rowp = st + static_cast<int64_t>(j) * p.ld_bytes;
        float zp = -CUDART_INF_F, zm = -CUDART_INF_F;
        uint32_t kp = kNone, km = kNone;
        // a3/a4: scan only the mapped labels, ascending ids per lane
        for (int e = lane; e < n_ent; e += 32) {
          const uint32_t key = ents[e];
          const float z = load_logit(rowp, key >> 8, p.bf16);
          if ((G >> (key & 0xFFu)) & 1u) {
            if (z > zp) { zp = z; kp = key; }
          } else {
            if (z > zm) { zm = z; km = key; }
          }
        }
        warp_lexmax(zp, kp);
        warp_lexmax(zm, km);
        deposit(b, lane, zp, kp, zm, km, G, a, row);
        if (b.n == 32) finish_batch(p, b, wtab, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (++s == p.stages) { s = 0; phase ^= 1u; }
    } else {
      // split rows: R == W, warp cw owns row r0 + cw across all chunks
      const bool mine = cw < nr;
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
            row_app_mask(st, r0, row, a, G);
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
            const float z = load_logit(rowp, col - c_lo, p.bf16);
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
        warp_lexmax(zp, kp);
        warp_lexmax(zm, km);
        deposit(b, lane, zp, kp, zm, km, G, a, row);
        if (b.n == 32) finish_batch(p, b, wtab, lane);
      }
    }
  }
  if (b.n > 0) finish_batch(p, b, wtab, lane);
}

// ------------------------------------------------------------------ GT-only pre-pass

__global__ void __launch_bounds__(256) hist_kernel(const HistParams p) {
  extern __shared__ unsigned long long sh_hist[];
  const int lane = threadIdx.x & 31;
  const int nbins = p.ctx.n_apps * 256;
  if (p.smem_hist) {
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t start = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t iters = (p.rows + stride - 1) / stride;  // uniform trip count for warp-wide intrinsics
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t row = start + it * stride;
    const bool active = row < p.rows;
    uint32_t key = 0;
    if (active) {
      const uint32_t a = p.app ? __ldg(p.app + row) : 0u;
      const uint8_t* cat = p.ctx.cat + static_cast<int64_t>(a) * p.ctx.C;
      uint32_t G = 0;
      for (int64_t t = __ldg(p.gt_off + row), e = __ldg(p.gt_off + row + 1); t < e; ++t) {
        const uint8_t v = __ldg(cat + __ldg(p.gt_lab + t));
        if (v != kCatNone) G |= 1u << v;
      }
      if (p.gt_mask_out) p.gt_mask_out[row] = static_cast<uint8_t>(G);
      key = a * 256u + G;
    }
    if (p.hist_gt) {
      const unsigned act = __ballot_sync(kFull, active);
      if (active) {
        const unsigned peers = __match_any_sync(act, key);
        if (lane == __ffs(peers) - 1) {
          if (p.smem_hist) atomicAdd(sh_hist + key, static_cast<unsigned long long>(__popc(peers)));
          else atomicAdd(p.hist_gt + key, static_cast<unsigned long long>(__popc(peers)));
        }
      }
    }
  }
  if (p.smem_hist && p.hist_gt) {
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x)
      if (sh_hist[i]) atomicAdd(p.hist_gt + i, sh_hist[i]);
  }
}

// ------------------------------------------------------------------ weights (a7)

// One CTA per app.  F = subset-sum (zeta) transform of H over 8 bits, so
// F[s] = #inputs whose G ⊆ s.  N(m) = M − F[~m] counts the inputs whose G
// intersects m; N(0) = H[0] counts non-target inputs (:2014).
__global__ void __launch_bounds__(256) weights_kernel(const unsigned long long* hist, float* w) {
  __shared__ unsigned long long F[256];
  const int m = threadIdx.x;
  const unsigned long long* H = hist + static_cast<int64_t>(blockIdx.x) * 256;
  const unsigned long long h = H[m];
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
  w[static_cast<int64_t>(blockIdx.x) * 256 + m] = N ? static_cast<float>(static_cast<double>(M) / static_cast<double>(N)) : 0.f;
}

}  // namespace

cudaError_t set_eval_smem_limit(size_t smem) {
  return cudaFuncSetAttribute(eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}

cudaError_t launch_eval(const EvalParams& p, int grid, size_t smem, cudaStream_t st) {
  eval_kernel<<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_hist(const HistParams& p, int grid, size_t smem, cudaStream_t st) {
  hist_kernel<<<grid, 256, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_weights(const unsigned long long* hist, float* w, int n_apps, cudaStream_t st) {
  weights_kernel<<<n_apps, 256, 0, st>>>(hist, w);
  return cudaGetLastError();
}

}  // namespace sc
