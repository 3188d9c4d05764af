// synth_cuda.cu — CUDA implementation of the seeded input recipe in synth.h.
// Written independently of synth_host.c (same recipe, separate code); tests
// compare the two bit for bit.  Harness only: no decision / loss arithmetic.
#include "synth.h"
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace {

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t h4(uint64_t seed, uint32_t stream, uint64_t a, uint64_t b) {
  return splitmix(splitmix(splitmix(seed ^ ((uint64_t)stream << 56)) ^ a) ^ b);
}

struct Spec {  // by-value copy of synth_spec for kernels
  uint64_t seed; int32_t C, n_apps, layout; int64_t rows_per_app;
  const uint8_t* mapped; const int64_t* wset_off; const int32_t* wset_lab;
};

__device__ __forceinline__ int32_t row_app(const Spec& s, int64_t row) {
  if (s.n_apps <= 1) return 0;
  return s.layout == 1 ? (int32_t)(row % s.n_apps) : (int32_t)((row / s.rows_per_app) % s.n_apps);
}

__global__ void k_apps(Spec s, int64_t row0, int64_t n, uint16_t* app) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    app[j] = (uint16_t)row_app(s, row0 + j);
}

__global__ void k_count(Spec s, int64_t row0, int64_t n, int64_t* cnt) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    cnt[j] = 1 + (int64_t)(h4(s.seed, SYNTH_S_NGT, (uint64_t)(row0 + j), 0) % 4);
}

__global__ void k_fill(Spec s, int64_t row0, int64_t n, const int64_t* off, int32_t* lab) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = row0 + j;
    const int32_t a = row_app(s, row);
    const int64_t wb = s.wset_off[a], wn = s.wset_off[a + 1] - wb;
    const int64_t b = off[j], m = off[j + 1] - b;
    for (int64_t t = 0; t < m; ++t) {
      const uint64_t u = h4(s.seed, SYNTH_S_GTLAB, (uint64_t)row, (uint64_t)t);
      const uint64_t lo = u & 0xffffffffull;
      lab[b + t] = (t == 0 && (u >> 63) && wn > 0) ? s.wset_lab[wb + (int64_t)(lo % (uint64_t)wn)]
                                                   : (int32_t)(lo % (uint64_t)s.C);
    }
  }
}

// One CTA walks rows (grid-stride); threads cover columns.  The row's GT
// labels (few) are staged in shared memory for the membership test.
template <int DT>
__global__ void k_logits(Spec s, int64_t row0, int64_t n, int64_t ld, const int64_t* off,
                         const int32_t* lab, void* out) {
  __shared__ int32_t g[64];
  __shared__ int32_t ng_s;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const int64_t row = row0 + j;
    const int32_t a = row_app(s, row);
    __syncthreads();
    if (threadIdx.x == 0) ng_s = (int32_t)(off[j + 1] - off[j]);
    __syncthreads();
    const int32_t ng = ng_s;
    const bool small = ng <= 64;
    if (small && threadIdx.x < ng) g[threadIdx.x] = lab[off[j] + threadIdx.x];
    __syncthreads();
    for (int64_t c = threadIdx.x; c < ld; c += blockDim.x) {
      float z;
      if (c >= s.C) {
        z = __int_as_float(0x7FC00000);
      } else {
        const uint64_t h = h4(s.seed, SYNTH_S_LOGIT, (uint64_t)row, (uint64_t)c);
        z = DT == 0 ? -12.0f + (float)(h & 0xffff) * (1.0f / 4096.0f)
                    : -8.0f + (float)(h & 0xff) * (1.0f / 16.0f);
        bool in_gt = false;
        for (int32_t t = 0; t < ng; ++t) {
          const int32_t gl = small ? g[t] : lab[off[j] + t];
          in_gt |= (gl == (int32_t)c);
        }
        if (in_gt) {
          if (h4(s.seed, SYNTH_S_TP, (uint64_t)row, (uint64_t)c) % 10 < 8) z += 8.0f;
        } else if (s.mapped[(int64_t)a * s.C + c]) {
          if (h4(s.seed, SYNTH_S_FP, (uint64_t)row, (uint64_t)c) % 100 < 5) z += 8.0f;
        }
      }
      if (DT == 0) static_cast<float*>(out)[j * ld + c] = z;
      else static_cast<uint16_t*>(out)[j * ld + c] = (uint16_t)(__float_as_uint(z) >> 16);
    }
  }
}

Spec to_spec(const synth_spec* p) {
  Spec s;
  s.seed = p->seed; s.C = p->C; s.n_apps = p->n_apps; s.layout = p->layout;
  s.rows_per_app = p->rows_per_app; s.mapped = p->mapped; s.wset_off = p->wset_off; s.wset_lab = p->wset_lab;
  return s;
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

extern "C" int synth_cuda_apps(const synth_spec* p, int64_t row0, int64_t n, uint16_t* app, void* st) {
  if (n <= 0) return 0;
  k_apps<<<grid_for(n, 256), 256, 0, (cudaStream_t)st>>>(to_spec(p), row0, n, app);
  return (int)cudaGetLastError();
}

extern "C" int synth_cuda_gt_count(const synth_spec* p, int64_t row0, int64_t n, int64_t* cnt, void* st) {
  if (n <= 0) return 0;
  k_count<<<grid_for(n, 256), 256, 0, (cudaStream_t)st>>>(to_spec(p), row0, n, cnt);
  return (int)cudaGetLastError();
}

extern "C" int synth_cuda_gt_fill(const synth_spec* p, int64_t row0, int64_t n, const int64_t* off,
                                  int32_t* lab, void* st) {
  if (n <= 0) return 0;
  k_fill<<<grid_for(n, 256), 256, 0, (cudaStream_t)st>>>(to_spec(p), row0, n, off, lab);
  return (int)cudaGetLastError();
}

extern "C" int synth_cuda_logits(const synth_spec* p, int64_t row0, int64_t n, int64_t ld, int32_t dtype,
                                 const int64_t* off, const int32_t* lab, void* out, void* st) {
  if (n <= 0) return 0;
  const int64_t g = n < 148 * 32 ? n : 148 * 32;
  if (dtype == 0) k_logits<0><<<(int)g, 256, 0, (cudaStream_t)st>>>(to_spec(p), row0, n, ld, off, lab, out);
  else            k_logits<1><<<(int)g, 256, 0, (cudaStream_t)st>>>(to_spec(p), row0, n, ld, off, lab, out);
  return (int)cudaGetLastError();
}
