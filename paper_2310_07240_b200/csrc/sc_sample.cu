// sc_sample.cu — rebalanced training-data sampler.
//
// The strawman of PAPER.md:1989-1990 (abstract PAPER.md:19-20): re-train on a re-sampled
// training set that rebalances the application's target classes.  Draws are i.i.d. with
// q_i = w[G_i] / Σ_j w[G_j] (w = M/N).  Mapping of two uniforms to a row
// (reading A24): rows grouped by G in ascending mask
// order (row order inside a group), bucket weights count_m·w[m] summed in double in
// ascending m; bucket = first m with u1·ΣW < cumulative W; row = number
// min(count_m − 1, floor(u2·count_m)) of the bucket.
//
// Five launches: per-chunk mask counts; per-mask scans over the chunks (one CTA per mask);
// bucket starts and the CDF in the oracle's summation order (one CTA); a stable scatter (one
// 1024-thread CTA per 1024-row chunk: per-warp ranks from __match_any_sync, a per-mask
// prefix over the chunk's 32 warps in shared memory); the draws (one thread per draw, CDF in
// shared memory).  Row ids are int32 in the bucket order (rows < 2^31).
#include "sc.h"

#include <cuda_runtime.h>

#include <string>

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int64_t kChunk = 1024;  // rows per chunk of the counting sort (one scatter warp each)

thread_local std::string g_serr;

sc_status sfail(sc_status st, const char* msg) {
  g_serr = msg;
  return st;
}

struct Workspace {  // carved from the caller's buffer
  unsigned* chunk_cnt;   // [nchunks][256]
  int64_t* chunk_off;    // [nchunks][256]  first slot of (chunk, mask) within mask m's bucket
  int64_t* count;        // [256]
  int64_t* start;        // [256]
  double* cum;           // [256]
  int32_t* order;        // [rows] row ids in bucket order
  int* status;           // [1]  0 ok, 1 all weights zero
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t layout(int64_t rows, Workspace* ws, uint8_t* base) {
  const int64_t nch = (rows + kChunk - 1) / kChunk;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return base ? base + o : nullptr;
  };
  uint8_t* p;
  p = take(sizeof(unsigned) * 256 * (nch > 0 ? nch : 1));
  if (ws) ws->chunk_cnt = reinterpret_cast<unsigned*>(p);
  p = take(sizeof(int64_t) * 256 * (nch > 0 ? nch : 1));
  if (ws) ws->chunk_off = reinterpret_cast<int64_t*>(p);
  p = take(sizeof(int64_t) * 256);
  if (ws) ws->count = reinterpret_cast<int64_t*>(p);
  p = take(sizeof(int64_t) * 256);
  if (ws) ws->start = reinterpret_cast<int64_t*>(p);
  p = take(sizeof(double) * 256);
  if (ws) ws->cum = reinterpret_cast<double*>(p);
  p = take(sizeof(int32_t) * (rows > 0 ? rows : 1));
  if (ws) ws->order = reinterpret_cast<int32_t*>(p);
  p = take(sizeof(int));
  if (ws) ws->status = reinterpret_cast<int*>(p);
  return off;
}

__global__ void __launch_bounds__(256) chunk_count_kernel(const uint8_t* gt_mask, int64_t rows, unsigned* chunk_cnt) {
  __shared__ unsigned h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t lo = static_cast<int64_t>(blockIdx.x) * kChunk;
  const int64_t hi = lo + kChunk < rows ? lo + kChunk : rows;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(h + gt_mask[i], 1u);
  __syncthreads();
  chunk_cnt[static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x] = h[threadIdx.x];
}

// One CTA per mask m: exclusive scan of chunk_cnt[., m] over the chunks (256 at a time,
// warp shuffles + one shared-memory pass), total count of m.
__global__ void __launch_bounds__(256) chunk_scan_kernel(const unsigned* chunk_cnt, int64_t nch, Workspace ws) {
  __shared__ int64_t warp_sum[8];
  __shared__ int64_t carry_s;
  const int m = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t k0 = 0; k0 < nch; k0 += 256) {
    const int64_t k = k0 + threadIdx.x;
    const int64_t v = k < nch ? static_cast<int64_t>(chunk_cnt[k * 256 + m]) : 0;
    int64_t x = v;  // inclusive warp scan
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) warp_sum[wid] = x;
    __syncthreads();
    int64_t before = carry_s;
    for (int q = 0; q < wid; ++q) before += warp_sum[q];
    if (k < nch) ws.chunk_off[k * 256 + m] = before + x - v;
    __syncthreads();
    if (threadIdx.x == 255) carry_s = before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) ws.count[m] = carry_s;
}

// One CTA: bucket starts (an exclusive scan of the counts) and the CDF.  The products
// count_m·w[m] are formed in parallel; their running sum is taken by one thread in ascending m
// from shared memory (the oracle's summation order, so both compare identical doubles).
__global__ void __launch_bounds__(256) starts_kernel(const float* w, Workspace ws) {
  __shared__ int64_t cnt[256];
  __shared__ double prod[256];
  __shared__ int64_t wsum[8];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t c = ws.count[t];
  cnt[t] = c;
  prod[t] = static_cast<double>(c) * static_cast<double>(w[t]);
  int64_t x = c;  // inclusive warp scan of the counts
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  int64_t before = 0;
  for (int q = 0; q < wid; ++q) before += wsum[q];
  ws.start[t] = before + x - c;
  if (t == 0) {
    double tot = 0.0;
    for (int q = 0; q < 256; ++q) {
      tot += prod[q];
      prod[q] = tot;
    }
    *ws.status = tot > 0.0 ? 0 : 1;
  }
  __syncthreads();
  ws.cum[t] = prod[t];
}

// One CTA per chunk (32 warps x 32 rows): a row's slot in its mask's bucket = bucket start +
// rows of that mask in earlier chunks (chunk_off) + in earlier warps of this chunk (prefix of
// the per-warp counts) + earlier lanes of its warp with the same mask (__match_any_sync), so
// equal masks keep row order (stable).
__global__ void __launch_bounds__(kChunk) scatter_kernel(const uint8_t* gt_mask, int64_t rows, Workspace ws) {
  __shared__ uint16_t cnt[32][256];  // per warp and mask: count, then exclusive prefix over the warps
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t chunk = blockIdx.x;
  for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t i = chunk * kChunk + threadIdx.x;
  const bool act = i < rows;
  const unsigned am = __ballot_sync(kFull, act);
  unsigned key = 0, rank = 0;
  if (act) {
    key = gt_mask[i];
    const unsigned peers = __match_any_sync(am, key);
    rank = __popc(peers & ((1u << lane) - 1u));
    if (lane == __ffs(peers) - 1) cnt[wid][key] = static_cast<uint16_t>(__popc(peers));
  }
  __syncthreads();
  if (threadIdx.x < 256) {
    unsigned run = 0;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) {
      const unsigned v = cnt[w][threadIdx.x];
      cnt[w][threadIdx.x] = static_cast<uint16_t>(run);
      run += v;
    }
  }
  __syncthreads();
  if (act) {
    const int64_t slot = ws.start[key] + ws.chunk_off[chunk * 256 + key] + cnt[wid][key] + rank;
    ws.order[slot] = static_cast<int32_t>(i);
  }
}

__global__ void __launch_bounds__(256) draw_kernel(const double* u, int64_t n, Workspace ws, int64_t* out) {
  __shared__ double cum[256];
  __shared__ int64_t cnt[256], st[256];
  cum[threadIdx.x] = ws.cum[threadIdx.x];
  cnt[threadIdx.x] = ws.count[threadIdx.x];
  st[threadIdx.x] = ws.start[threadIdx.x];
  __syncthreads();
  const double total = cum[255];
  for (int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; d < n;
       d += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!(total > 0.0)) { out[d] = -1; continue; }
    const double t = u[2 * d] * total;
    int lo = 0, hi = 255;  // first m with t < cum[m]
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (t < cum[mid]) hi = mid;
      else lo = mid + 1;
    }
    const int64_t c = cnt[lo];
    int64_t pos = static_cast<int64_t>(floor(u[2 * d + 1] * static_cast<double>(c)));
    if (pos > c - 1) pos = c - 1;
    out[d] = ws.order[st[lo] + pos];
  }
}

}  // namespace

extern "C" {

size_t sc_sample_workspace_bytes(int64_t rows) { return layout(rows < 0 ? 0 : rows, nullptr, nullptr) + 256; }

sc_status sc_rebalance_sample(const uint8_t* gt_mask, int64_t rows, const float* w, const double* u, int64_t n,
                              int64_t* out, void* workspace, size_t workspace_bytes, sc_stream stream) {
  if (rows <= 0) return sfail(SC_ERR_INVALID_ARG, "rows must be > 0");
  if (rows > INT32_MAX) return sfail(SC_ERR_INVALID_ARG, "rows must be < 2^31");
  if (n < 0) return sfail(SC_ERR_INVALID_ARG, "n < 0");
  if (!gt_mask || !w || !workspace || (n > 0 && (!u || !out))) return sfail(SC_ERR_INVALID_ARG, "NULL argument");
  if (workspace_bytes < sc_sample_workspace_bytes(rows)) return sfail(SC_ERR_INVALID_ARG, "workspace too small");
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
  Workspace ws;
  layout(rows, &ws, base);
  const int64_t nch = (rows + kChunk - 1) / kChunk;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  chunk_count_kernel<<<static_cast<unsigned>(nch), 256, 0, st>>>(gt_mask, rows, ws.chunk_cnt);
  chunk_scan_kernel<<<256, 256, 0, st>>>(ws.chunk_cnt, nch, ws);
  starts_kernel<<<1, 256, 0, st>>>(w, ws);
  scatter_kernel<<<static_cast<unsigned>(nch), kChunk, 0, st>>>(gt_mask, rows, ws);
  if (n > 0) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    draw_kernel<<<static_cast<unsigned>(g), 256, 0, st>>>(u, n, ws, out);
  }
  if (cudaError_t e = cudaGetLastError()) return sfail(SC_ERR_CUDA, cudaGetErrorString(e));
  return SC_OK;
}

const char* sc_sample_last_error(void) { return g_serr.c_str(); }

}  // extern "C"
