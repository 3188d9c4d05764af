// sc_ranges.cu — value-ranges applications, SURVEY.md §8(f) NEXT f1.
//
// An API returning a score O_i (e.g. sentiment); the application checks, in code order,
// whether it lies in each of its ranges [l_j, h_j] (reading A22: closed, first containing
// range wins, none -> default m).  Loss:
//   L_i = w[r_i] ( S(l_{r_i} − O_i) + S(O_i − h_{r_i}) ),  w[r] = M / N_r,
// r_i = the range the ground-truth score lies in (no target range -> L_i = 0).
// HBM-bound element-wise pass: 4 B score + 1 B ground-truth range in, 1 B decision + 4 B
// gradient out per row; counters aggregated per warp.
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
};

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kMaxRanges = 255;

thread_local std::string g_rerr;

sc_status rfail(sc_status st, const char* msg) {
  g_rerr = msg;
  return st;
}

__device__ __forceinline__ int range_of(const float* lo, const float* hi, int m, float s) {
  int r = m;
  for (int j = m - 1; j >= 0; --j)
    if (s >= lo[j] && s <= hi[j]) r = j;  // the first containing range in code order
  return r;
}

__device__ __forceinline__ float sig(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

__device__ __forceinline__ float dsig(float z) {
  const float t = expf(-fabsf(z));
  const float d = 1.f + t;
  return t / (d * d);
}

__global__ void __launch_bounds__(256) ranges_hist_kernel(const float* lo_g, const float* hi_g, int m,
                                                         const float* gt_score, int64_t rows,
                                                         unsigned long long* hist, uint8_t* gt_range) {
  __shared__ float lo[kMaxRanges], hi[kMaxRanges];
  __shared__ unsigned long long h[kMaxRanges + 1];
  for (int j = threadIdx.x; j < m; j += blockDim.x) { lo[j] = lo_g[j]; hi[j] = hi_g[j]; }
  for (int j = threadIdx.x; j <= m; j += blockDim.x) h[j] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t iters = (rows + stride - 1) / stride;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = it * stride + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool act = i < rows;
    int r = 0;
    if (act) {
      r = range_of(lo, hi, m, __ldg(gt_score + i));
      if (gt_range) gt_range[i] = static_cast<uint8_t>(r);
    }
    if (hist) {
      const unsigned a = __ballot_sync(kFull, act);
      if (act) {
        const unsigned peers = __match_any_sync(a, r);
        if (lane == __ffs(peers) - 1) atomicAdd(h + r, static_cast<unsigned long long>(__popc(peers)));
      }
    }
  }
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

__global__ void __launch_bounds__(256) ranges_loss_kernel(const float* lo_g, const float* hi_g, int m, float k,
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
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t iters = (rows + stride - 1) / stride;
  double my_loss = 0.0;
  unsigned my_inc = 0;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = it * stride + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool act = i < rows;
    int d = 0;
    if (act) {
      const float s = __ldg(score + i);
      const int r = __ldg(gt_range + i);
      d = range_of(lo, hi, m, s);
      my_inc += d != r;
      float L = 0.f, g = 0.f;
      if (r < m) {
        const float a = k * (lo[r] - s), b = k * (s - hi[r]);
        L = ws[r] * (sig(a) + sig(b));
        g = ws[r] * k * (dsig(b) - dsig(a)) * grad_scale;
      }
      my_loss += L;
      if (decision) decision[i] = static_cast<uint8_t>(d);
      if (loss_row) loss_row[i] = L;
      if (grad) grad[i] = g;
    }
    if (hist_pred) {
      const unsigned a = __ballot_sync(kFull, act);
      if (act) {
        const unsigned peers = __match_any_sync(a, d);
        if (lane == __ffs(peers) - 1) atomicAdd(hp + d, static_cast<unsigned long long>(__popc(peers)));
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    my_loss += __shfl_xor_sync(kFull, my_loss, off);
    my_inc += __shfl_xor_sync(kFull, my_inc, off);
  }
  if (lane == 0) {
    atomicAdd(&lsum, my_loss);
    atomicAdd(&ninc, static_cast<unsigned long long>(my_inc));
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
  int64_t g = (rows + 255) / 256;
  if (g > static_cast<int64_t>(sms) * 8) g = static_cast<int64_t>(sms) * 8;
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
  ranges_hist_kernel<<<grid_for(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      r->d_lo, r->d_hi, r->m, gt_score, rows, reinterpret_cast<unsigned long long*>(hist_gt), gt_range_out);
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
  ranges_loss_kernel<<<grid_for(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      r->d_lo, r->d_hi, r->m, r->k, score, gt_range, rows, w, grad_scale, loss_sum, loss_row, grad, decision,
      reinterpret_cast<unsigned long long*>(n_incorrect), reinterpret_cast<unsigned long long*>(hist_pred));
  if (cudaError_t e = cudaGetLastError()) return rfail(SC_ERR_CUDA, cudaGetErrorString(e));
  return SC_OK;
}

const char* sc_ranges_last_error(void) { return g_rerr.c_str(); }

}  // extern "C"
