// sc_ranges.cu — value-ranges applications, SURVEY.md §8(f) NEXT f1.
//
// An API returning a score O_i (e.g. sentiment); the application checks, in code order,
// whether it lies in each of its ranges [l_j, h_j] (reading A22: closed, first containing
// range wins, none -> default m).  Loss:
//   L_i = w[r_i] ( S(l_{r_i} − O_i) + S(O_i − h_{r_i}) ),  w[r] = M / N_r,
// r_i = the range the ground-truth score lies in (no target range -> L_i = 0).
// HBM-bound element-wise pass: 4 B score + 1 B ground-truth range in, 1 B decision + 4 B
// loss + 4 B gradient out per row, four rows per thread (128-bit / 32-bit accesses);
// histograms of <= 32 bins counted with warp ballots into lane-owned registers.
#include "sc.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <string>

struct sc_ranges_s {
  int32_t m = 0;
  float k = 10.f;
  float* d_lo = nullptr;  // [m]
  float* d_hi = nullptr;  // [m]
  int device = 0;
  int sorted = 0;         // lo[j] < lo[j+1] and hi[j] <= lo[j+1] for all j (see range_lookup)
};

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kMaxRanges = 255;

thread_local std::string g_rerr;

sc_status rfail(sc_status st, const char* msg) {
  g_rerr = msg;
  return st;
}

// σ and σ' in overflow-free, branch-free forms (e = e^{-|z|} in (0, 1], so 1 + e in (1, 2]),
// fast reciprocal divisions (<= 2 ulp) keep the element-wise pass memory-bound.
// σ(z) and σ'(z) from one exponential: e = e^{-|z|}, r = 1/(1+e); σ = r or e·r, σ' = e·r².
// e^{-|z|} = 2^{-|z| log2 e}: one multiply + ex2.approx.f32 (2 ulp, subnormals kept) instead
// of expf's range reduction.  Relative error of e, by source: the rounded product and the
// rounded log2 e constant move the exponent by <= |z|·(2^-24 + 1.3e-8)·log2 e (<= 6e-8·|z|
// relative in e), ex2.approx <= 2.4e-7; and the caller's argument z = k·(x − y), rounded
// twice in fp32, carries <= 1.2e-7·|z| more.  Total <= 1.9e-7·|z| + 5e-7, inside the 1e-5
// bar for |z| <= kFastArg = 24; larger arguments take sig_dsig_arg's fp64 path.
__device__ __forceinline__ void sig_dsig(float z, float& s, float& ds) {
  const float e = exp2f(__fmul_rn(-fabsf(z), 1.4426950408889634f));
  const float r = __fdividef(1.f, 1.f + e);
  s = z >= 0.f ? r : e * r;
  ds = e * r * r;
}

constexpr float kFastArg = 24.f;

// σ(z), σ'(z) for z = k(x − y) with |z| > kFastArg (a score deep inside or far outside its
// ground-truth range; never in the bench's workload), in fp32 with error-free transforms:
// x − y as an exact two-term sum (TwoSum), k times it as zh + zl (FMA residual), the exponent
// −|z| log2 e as yh + yl with log2 e split in two floats, and e^{-|z|} = 2^yh (1 + yl ln 2).
// Relative error of e <= ~5e-7 at any |z| (ex2.approx and the final roundings), subnormal
// results keep their absolute accuracy.  Register-light, so the cold branch does not change
// the hot loop's occupancy (an fp64 version took the kernel from 61 to 98 registers).
__device__ __forceinline__ void sig_dsig_far(float k, float x, float y, float& s, float& ds) {
  const float d = x - y;
  const float bb = d - x;
  const float dl = (x - (d - bb)) + (-y - bb);           // x − y = d + dl exactly
  const float zh = k * d;
  const float zl = fmaf(k, d, -zh) + k * dl;              // k(x − y) = zh + zl (to ~2^-48 |z|)
  const float sg = zh >= 0.f ? 1.f : -1.f;                // |zl| << |zh| here: the sign is zh's
  const float ah = fabsf(zh), al = sg * zl;               // |z| = ah + al
  constexpr float kL2E = 1.44269502162933349609375f;      // log2 e rounded to float
  constexpr float kL2ELo = 1.925963033500011e-8f;         // log2 e − kL2E
  const float yh = -ah * kL2E;
  const float yl = fmaf(-ah, kL2E, -yh) - ah * kL2ELo - al * kL2E;
  const float e0 = exp2f(yh);
  const float e = fmaf(e0, yl * 0.693147180559945f, e0);  // 2^yl = 1 + yl ln 2 (|yl| < 1e-5)
  const float r = 1.f / (1.f + e);
  s = zh >= 0.f ? r : e * r;
  ds = e * r * r;
}

// Eight consecutive rows per thread per pass (2 x float4 / uint2 accesses when aligned): two
// 128-bit loads in flight per thread keep enough bytes in flight for an element-wise pass.
constexpr int kV = 8;

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return static_cast<uint32_t>(a) | static_cast<uint32_t>(b) << 8 | static_cast<uint32_t>(c) << 16 |
         static_cast<uint32_t>(d) << 24;
}

// The range each of kV scores lies in: the first containing range in code order (reading
// A22), else m.  sorted (lo strictly ascending, hi[j] <= lo[j+1]: ranges in code order that
// at most touch): the last range whose lo <= s, found by a branch-free binary search
// (ceil(log2 m) steps, the same trip count in every lane), or the one before it when s
// sits on their shared bound; otherwise a scan of every range.
template <int V>
__device__ __forceinline__ void range_lookup(const float (&sv)[V], int (&r)[V], const float* lo, const float* hi,
                                             int m, bool sorted) {
  if (sorted) {
    int base[V];
#pragma unroll
    for (int q = 0; q < V; ++q) base[q] = 0;
    for (int n = m; n > 1;) {  // uniform
      const int half = n >> 1;
#pragma unroll
      for (int q = 0; q < V; ++q) base[q] = lo[base[q] + half] <= sv[q] ? base[q] + half : base[q];
      n -= half;
    }
#pragma unroll
    for (int q = 0; q < V; ++q) {
      int b = base[q];  // the last range with lo[b] <= s (when s >= lo[0])
      // ranges may touch (hi[b-1] == lo[b]): a score on the shared bound is in b-1 first
      if (b > 0 && sv[q] <= hi[b - 1]) b -= 1;
      r[q] = (lo[b] <= sv[q] && sv[q] <= hi[b]) ? b : m;
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < V; ++q) r[q] = m;
  for (int j = m - 1; j >= 0; --j) {
    const float l = lo[j], u = hi[j];
#pragma unroll
    for (int q = 0; q < V; ++q)
      if (sv[q] >= l && sv[q] <= u) r[q] = j;
  }
}

// Histogram counters, by number of bins:
//   <= 8 (PACKED): each thread counts its own rows in 16-bit fields of two registers (bins
//     0-3 / 4-7), reduced over the warp at the end — one shift and add per row;
//   <= 32 (SMALL): lane j of each warp owns bin j and adds the popcount of the warp's ballot;
//   more: match + shared atomics.
__device__ __forceinline__ void count_packed(bool act, int v, unsigned long long (&pk)[2]) {
  if (act) {
    const unsigned long long inc = 1ull << (16 * (v & 3));
    if (v < 4) pk[0] += inc;
    else pk[1] += inc;
  }
}

template <bool SMALL>
__device__ __forceinline__ void count_bins(int nb, bool act, int v, int lane, unsigned long long& mine,
                                           unsigned long long* h_s) {
  if constexpr (SMALL) {
    for (int j = 0; j < nb; ++j) {  // nb is uniform
      const unsigned c = __popc(__ballot_sync(kFull, act && v == j));
      if (lane == j) mine += c;
    }
  } else {
    const unsigned a = __ballot_sync(kFull, act);
    if (act) {
      const unsigned peers = __match_any_sync(a, v);
      if (lane == __ffs(peers) - 1) atomicAdd(h_s + v, static_cast<unsigned long long>(__popc(peers)));
    }
  }
}

// Packed per-thread counters -> warp sums -> lane j owns bin j (mine); fields never overflow:
// the host caps a thread's rows per launch below 2^16 (grid_for).
__device__ __forceinline__ void flush_packed(const unsigned long long (&pk)[2], int lane, unsigned long long& mine) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    unsigned c = static_cast<unsigned>((pk[j >> 2] >> (16 * (j & 3))) & 0xFFFFull);
    c = __reduce_add_sync(kFull, c);
    if (lane == j) mine += c;
  }
}

template <bool SMALL>
__global__ void __launch_bounds__(256) ranges_hist_kernel(const float* lo_g, const float* hi_g, int m, int sorted,
                                                         const float* gt_score, int64_t rows,
                                                         unsigned long long* hist, uint8_t* gt_range) {
  __shared__ float lo[kMaxRanges], hi[kMaxRanges];
  __shared__ unsigned long long h[kMaxRanges + 1];
  for (int j = threadIdx.x; j < m; j += blockDim.x) { lo[j] = lo_g[j]; hi[j] = hi_g[j]; }
  for (int j = threadIdx.x; j <= m; j += blockDim.x) h[j] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned long long mine = 0;
  const bool packed = SMALL && m + 1 <= 8;
  unsigned long long pk[2] = {0ull, 0ull};
  const bool vec = (reinterpret_cast<uintptr_t>(gt_score) % 16 == 0) &&
                   (!gt_range || reinterpret_cast<uintptr_t>(gt_range) % 8 == 0);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * kV;
  const int64_t iters = (rows + stride - 1) / stride;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i0 = it * stride + (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kV;
    float sv[kV];
    int r[kV];
    // rows of this pass held by the thread (32-bit: one compare per row below)
    const int nv = i0 >= rows ? 0 : (rows - i0 < kV ? static_cast<int>(rows - i0) : kV);
    if (vec && nv == kV) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(gt_score + i0));
      const float4 f2 = __ldg(reinterpret_cast<const float4*>(gt_score + i0 + 4));
      sv[0] = f.x; sv[1] = f.y; sv[2] = f.z; sv[3] = f.w;
      sv[4] = f2.x; sv[5] = f2.y; sv[6] = f2.z; sv[7] = f2.w;
    } else {
#pragma unroll
      for (int q = 0; q < kV; ++q) sv[q] = q < nv ? __ldg(gt_score + i0 + q) : 0.f;
    }
    range_lookup<kV>(sv, r, lo, hi, m, sorted);  // the first containing range in code order
    if (gt_range) {
      if (vec && nv == kV) {
        *reinterpret_cast<uint2*>(gt_range + i0) = make_uint2(pack4(r[0], r[1], r[2], r[3]), pack4(r[4], r[5], r[6], r[7]));
      } else {
#pragma unroll
        for (int q = 0; q < kV; ++q)
          if (q < nv) gt_range[i0 + q] = static_cast<uint8_t>(r[q]);
      }
    }
    if (hist) {
      if (packed) {
#pragma unroll
        for (int q = 0; q < kV; ++q) count_packed(q < nv, r[q], pk);
      } else {
#pragma unroll
        for (int q = 0; q < kV; ++q) count_bins<SMALL>(m + 1, q < nv, r[q], lane, mine, h);
      }
    }
  }
  if (packed && hist) flush_packed(pk, lane, mine);
  if (SMALL && hist && lane <= m && mine) atomicAdd(h + lane, mine);
  __syncthreads();
  if (hist)
    for (int j = threadIdx.x; j <= m; j += blockDim.x)
      if (h[j]) atomicAdd(hist + j, h[j]);
}

__global__ void ranges_weights_kernel(const unsigned long long* hist, int m, float* w) {
  __shared__ unsigned long long M;
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int j = 0; j <= m; ++j) s += hist[j];
    M = s;
  }
  __syncthreads();
  for (int j = threadIdx.x; j <= m; j += blockDim.x)
    w[j] = hist[j] ? static_cast<float>(static_cast<double>(M) / static_cast<double>(hist[j])) : 0.f;
}

template <bool SMALL>
__global__ void __launch_bounds__(256) ranges_loss_kernel(const float* lo_g, const float* hi_g, int m, int sorted, float k,
                                                         const float* score, const uint8_t* gt_range, int64_t rows,
                                                         const float* w, float grad_scale, double* loss_sum,
                                                         float* loss_row, float* grad, uint8_t* decision,
                                                         unsigned long long* n_incorrect,
                                                         unsigned long long* hist_pred) {
  __shared__ float lo[kMaxRanges], hi[kMaxRanges], ws[kMaxRanges + 1];
  __shared__ unsigned long long hp[kMaxRanges + 1];
  __shared__ unsigned long long ninc;
  __shared__ double lsum;
  for (int j = threadIdx.x; j < m; j += blockDim.x) { lo[j] = lo_g[j]; hi[j] = hi_g[j]; }
  for (int j = threadIdx.x; j <= m; j += blockDim.x) { ws[j] = w ? w[j] : 1.f; hp[j] = 0; }
  if (threadIdx.x == 0) { ninc = 0; lsum = 0.0; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const bool vec = (reinterpret_cast<uintptr_t>(score) % 16 == 0) && (reinterpret_cast<uintptr_t>(gt_range) % 8 == 0) &&
                   (!decision || reinterpret_cast<uintptr_t>(decision) % 8 == 0) &&
                   (!loss_row || reinterpret_cast<uintptr_t>(loss_row) % 16 == 0) &&
                   (!grad || reinterpret_cast<uintptr_t>(grad) % 16 == 0);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * kV;
  const int64_t iters = (rows + stride - 1) / stride;
  double my_loss = 0.0;
  unsigned long long my_inc = 0, mine = 0;
  const bool packed = SMALL && m + 1 <= 8;
  unsigned long long pk[2] = {0ull, 0ull};
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i0 = it * stride + (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kV;
    const int nv = i0 >= rows ? 0 : (rows - i0 < kV ? static_cast<int>(rows - i0) : kV);
    const bool full = vec && nv == kV;
    float sv[kV];
    int r[kV], d[kV];
    if (full) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(score + i0));
      const float4 f2 = __ldg(reinterpret_cast<const float4*>(score + i0 + 4));
      const uint2 g = __ldg(reinterpret_cast<const uint2*>(gt_range + i0));
      sv[0] = f.x; sv[1] = f.y; sv[2] = f.z; sv[3] = f.w;
      sv[4] = f2.x; sv[5] = f2.y; sv[6] = f2.z; sv[7] = f2.w;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        r[q] = (g.x >> (8 * q)) & 0xFFu;
        r[4 + q] = (g.y >> (8 * q)) & 0xFFu;
      }
    } else {
#pragma unroll
      for (int q = 0; q < kV; ++q) {
        sv[q] = q < nv ? __ldg(score + i0 + q) : 0.f;
        r[q] = q < nv ? __ldg(gt_range + i0 + q) : m;
      }
    }
    range_lookup<kV>(sv, d, lo, hi, m, sorted);  // Decision(API(x)): the first containing range in code order
    float L[kV], g[kV];
    float part = 0.f;  // this pass's 8 losses in fp32, then one fp64 add (rel. error ~5e-7)
    bool far = false;  // some row's S argument leaves the fast path's accuracy range
#pragma unroll
    for (int q = 0; q < kV; ++q) {
      const bool act = q < nv;
      L[q] = 0.f;
      g[q] = 0.f;
      if (act && r[q] < m) {
        const float a = k * (lo[r[q]] - sv[q]), b = k * (sv[q] - hi[r[q]]);  // S(l − O), S(O − h)
        float sa, da, sb, db;
        sig_dsig(a, sa, da);
        sig_dsig(b, sb, db);
        L[q] = ws[r[q]] * (sa + sb);
        g[q] = ws[r[q]] * k * (db - da) * grad_scale;
        far |= fabsf(a) > kFastArg || fabsf(b) > kFastArg;
      }
      part += L[q];
      my_inc += (act && d[q] != r[q]) ? 1u : 0u;
    }
    my_loss += static_cast<double>(part);
    if (full) {
      if (decision)
        *reinterpret_cast<uint2*>(decision + i0) = make_uint2(pack4(d[0], d[1], d[2], d[3]), pack4(d[4], d[5], d[6], d[7]));
      if (loss_row) {
        *reinterpret_cast<float4*>(loss_row + i0) = make_float4(L[0], L[1], L[2], L[3]);
        *reinterpret_cast<float4*>(loss_row + i0 + 4) = make_float4(L[4], L[5], L[6], L[7]);
      }
      if (grad) {
        *reinterpret_cast<float4*>(grad + i0) = make_float4(g[0], g[1], g[2], g[3]);
        *reinterpret_cast<float4*>(grad + i0 + 4) = make_float4(g[4], g[5], g[6], g[7]);
      }
    } else {
#pragma unroll
      for (int q = 0; q < kV; ++q) {
        if (q >= nv) continue;
        if (decision) decision[i0 + q] = static_cast<uint8_t>(d[q]);
        if (loss_row) loss_row[i0 + q] = L[q];
        if (grad) grad[i0 + q] = g[q];
      }
    }
    if (hist_pred) {
      if (packed) {
#pragma unroll
        for (int q = 0; q < kV; ++q) count_packed(q < nv, d[q], pk);
      } else {
#pragma unroll
        for (int q = 0; q < kV; ++q) count_bins<SMALL>(m + 1, q < nv, d[q], lane, mine, hp);
      }
    }
    if (far) {  // rare (see sig_dsig_far): this thread's rows again, operands re-read (L1-hot), results overwritten
#pragma unroll 1
      for (int q = 0; q < nv; ++q) {
        const int r_q = __ldg(gt_range + i0 + q);
        if (r_q >= m) continue;
        const float s_q = __ldg(score + i0 + q);
        const float a = k * (lo[r_q] - s_q), b = k * (s_q - hi[r_q]);
        if (!(fabsf(a) > kFastArg || fabsf(b) > kFastArg)) continue;
        float sa, da, sb, db;
        sig_dsig(a, sa, da);
        sig_dsig(b, sb, db);
        my_loss -= static_cast<double>(ws[r_q] * (sa + sb));  // the fast value already in part
        sig_dsig_far(k, lo[r_q], s_q, sa, da);
        sig_dsig_far(k, s_q, hi[r_q], sb, db);
        const float Lq = ws[r_q] * (sa + sb);
        my_loss += static_cast<double>(Lq);
        if (loss_row) loss_row[i0 + q] = Lq;
        if (grad) grad[i0 + q] = ws[r_q] * k * (db - da) * grad_scale;
      }
    }
  }
  if (packed && hist_pred) flush_packed(pk, lane, mine);
  if (SMALL && hist_pred && lane <= m && mine) atomicAdd(hp + lane, mine);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    my_loss += __shfl_xor_sync(kFull, my_loss, off);
    my_inc += __shfl_xor_sync(kFull, my_inc, off);
  }
  if (lane == 0) {
    atomicAdd(&lsum, my_loss);
    atomicAdd(&ninc, my_inc);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (loss_sum) atomicAdd(loss_sum, lsum);
    if (n_incorrect) atomicAdd(n_incorrect, ninc);
  }
  if (hist_pred)
    for (int j = threadIdx.x; j <= m; j += blockDim.x)
      if (hp[j]) atomicAdd(hist_pred + j, hp[j]);
}

int grid_for(int64_t rows) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t g = (rows + 256 * kV - 1) / (256 * kV);
  if (g > static_cast<int64_t>(sms) * 8) g = static_cast<int64_t>(sms) * 8;
  // packed 16-bit per-thread counters: < 2^16 rows per thread per launch
  const int64_t g_min = (rows + 256LL * 65535 - 1) / (256LL * 65535);
  if (g < g_min) g = g_min;
  return g < 1 ? 1 : static_cast<int>(g);
}

}  // namespace

extern "C" {

sc_status sc_ranges_load(int32_t m, const float* lo, const float* hi, float k, sc_ranges* out) {
  if (!out) return rfail(SC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (m < 1 || m > kMaxRanges) return rfail(SC_ERR_INVALID_ARG, "m must be in [1, 255]");
  if (!lo || !hi) return rfail(SC_ERR_INVALID_ARG, "lo / hi is NULL");
  if (!(k > 0.f) || !std::isfinite(k)) return rfail(SC_ERR_INVALID_ARG, "k must be finite and > 0");
  for (int j = 0; j < m; ++j)
    if (!std::isfinite(lo[j]) || !std::isfinite(hi[j]) || lo[j] > hi[j])
      return rfail(SC_ERR_INVALID_ARG, "each range needs finite lo <= hi");
  auto* r = new sc_ranges_s();
  r->m = m;
  r->k = k;
  // binary-search lookup only pays for many ranges: a scan loads each bound once for all
  // of a thread's rows, the search needs a dependent shared-memory load per row and step
  // (B200, 7 ranges: 0.460 ms either way; the hist kernel is ALU-bound at ~65 instr/row)
  r->sorted = m > 16 ? 1 : 0;
  for (int j = 0; j + 1 < m; ++j)
    if (!(lo[j] < lo[j + 1] && hi[j] <= lo[j + 1])) r->sorted = 0;
  cudaError_t e = cudaGetDevice(&r->device);
  if (!e) e = cudaMalloc(&r->d_lo, m * sizeof(float));
  if (!e) e = cudaMalloc(&r->d_hi, m * sizeof(float));
  if (!e) e = cudaMemcpy(r->d_lo, lo, m * sizeof(float), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(r->d_hi, hi, m * sizeof(float), cudaMemcpyHostToDevice);
  if (e) {
    cudaFree(r->d_lo);
    cudaFree(r->d_hi);
    delete r;
    return rfail(e == cudaErrorMemoryAllocation ? SC_ERR_OOM : SC_ERR_CUDA, cudaGetErrorString(e));
  }
  *out = r;
  return SC_OK;
}

sc_status sc_ranges_free(sc_ranges r) {
  if (!r) return SC_OK;
  cudaFree(r->d_lo);
  cudaFree(r->d_hi);
  delete r;
  return SC_OK;
}

sc_status sc_ranges_hist(sc_ranges r, const float* gt_score, int64_t rows, uint64_t* hist_gt, uint8_t* gt_range_out,
                         sc_stream stream) {
  if (!r) return rfail(SC_ERR_INVALID_ARG, "ranges is NULL");
  if (rows < 0) return rfail(SC_ERR_INVALID_ARG, "rows < 0");
  if (rows == 0 || (!hist_gt && !gt_range_out)) return SC_OK;
  if (!gt_score) return rfail(SC_ERR_INVALID_ARG, "gt_score is NULL");
  auto kern = r->m + 1 <= 32 ? ranges_hist_kernel<true> : ranges_hist_kernel<false>;
  kern<<<grid_for(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      r->d_lo, r->d_hi, r->m, r->sorted, gt_score, rows, reinterpret_cast<unsigned long long*>(hist_gt), gt_range_out);
  if (cudaError_t e = cudaGetLastError()) return rfail(SC_ERR_CUDA, cudaGetErrorString(e));
  return SC_OK;
}

sc_status sc_ranges_weights(sc_ranges r, const uint64_t* hist_gt, float* w, sc_stream stream) {
  if (!r || !hist_gt || !w) return rfail(SC_ERR_INVALID_ARG, "NULL argument");
  ranges_weights_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const unsigned long long*>(hist_gt), r->m, w);
  if (cudaError_t e = cudaGetLastError()) return rfail(SC_ERR_CUDA, cudaGetErrorString(e));
  return SC_OK;
}

sc_status sc_ranges_loss_fwd_bwd(sc_ranges r, const float* score, const uint8_t* gt_range, int64_t rows,
                                 const float* w, float grad_scale, double* loss_sum, float* loss_row, float* grad,
                                 uint8_t* decision, uint64_t* n_incorrect, uint64_t* hist_pred, sc_stream stream) {
  if (!r) return rfail(SC_ERR_INVALID_ARG, "ranges is NULL");
  if (rows < 0) return rfail(SC_ERR_INVALID_ARG, "rows < 0");
  if (rows == 0) return SC_OK;
  if (!score || !gt_range) return rfail(SC_ERR_INVALID_ARG, "score / gt_range is NULL");
  auto kern = r->m + 1 <= 32 ? ranges_loss_kernel<true> : ranges_loss_kernel<false>;
  kern<<<grid_for(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      r->d_lo, r->d_hi, r->m, r->sorted, r->k, score, gt_range, rows, w, grad_scale, loss_sum, loss_row, grad, decision,
      reinterpret_cast<unsigned long long*>(n_incorrect), reinterpret_cast<unsigned long long*>(hist_pred));
  if (cudaError_t e = cudaGetLastError()) return rfail(SC_ERR_CUDA, cudaGetErrorString(e));
  return SC_OK;
}

const char* sc_ranges_last_error(void) { return g_rerr.c_str(); }

}  // extern "C"
