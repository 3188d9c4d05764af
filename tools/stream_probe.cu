// stream_probe.cu — what limits a persistent TMA-bulk streaming kernel on B200?
// One producer lane streams `bytes` through a ring of `stages` x `chunk` shared-memory
// stages; one consumer lane waits each stage and releases it (no compute).  Variants:
//   threads  CTA size (224 as the head kernel, 544 as the eval kernel)
//   tmem     1: allocate 512 TMEM columns first (as the head kernel)
//   spin     number of extra warps spinning on an mbarrier that never completes until the end
//   layout   0: CTA b streams its own contiguous region; 1: round-robin chunks over CTAs
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/stream_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(b)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sa(dst)),
      "l"(src), "r"(n), "r"(sa(b)), "l"(pol)
      : "memory");
}

struct P {
  const uint8_t* src;
  int64_t bytes;
  int chunk, stages, tmem, spin, layout;
  int tc;  // 1: consumer = head-kernel MMA thread (fences, tcgen05.commit per tile, epilogue handshake)
           // 2: same but releases stages with tcgen05.commit instead of a plain arrive
};

__global__ void probe(const P p) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + p.stages * p.chunk);
  uint64_t* empty = full + p.stages;
  uint64_t* never = empty + p.stages;
  uint64_t* tfull = never + 1;
  uint64_t* tempty = tfull + 2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      bar_init(full + s, 1);
      bar_init(empty + s, 1);
    }
    bar_init(never, 1);
    for (int b = 0; b < 2; ++b) {
      bar_init(tfull + b, 1);
      bar_init(tempty + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (p.tmem && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  const int64_t nchunks = p.bytes / p.chunk;
  // chunks of this CTA
  int64_t c0, cstep, cn;
  if (p.layout == 0) {
    const int64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
    c0 = blockIdx.x * per;
    cn = c0 >= nchunks ? 0 : (c0 + per > nchunks ? nchunks - c0 : per);
    cstep = 1;
  } else {
    c0 = blockIdx.x;
    cstep = gridDim.x;
    cn = c0 < nchunks ? (nchunks - c0 + gridDim.x - 1) / gridDim.x : 0;
  }
  // layout 2: 512-KB tiles round-robin over CTAs, each tile read in order (the head kernel's
  // pattern); layout 3: the same with the start chunk inside the tile skewed per CTA
  const int64_t tile_chunks = (512 * 1024) / p.chunk;
  const int64_t n_tiles = nchunks / tile_chunks;
  if (p.layout >= 2) cn = ((n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * tile_chunks;
  auto chunk_of = [&](int64_t i) -> int64_t {
    if (p.layout < 2) return c0 + i * cstep;
    const int64_t t = blockIdx.x + (i / tile_chunks) * gridDim.x;
    int64_t k = i % tile_chunks;
    if (p.layout == 3) k = (k + blockIdx.x) % tile_chunks;
    return t * tile_chunks + k;
  };
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      uint32_t ph = 0;
      for (int64_t i = 0; i < cn; ++i) {
        bar_wait(empty + s, ph ^ 1u);
        bar_expect(full + s, p.chunk);
        bulk(sm + static_cast<size_t>(s) * p.chunk, p.src + chunk_of(i) * p.chunk, p.chunk, full + s, pol);
        if (++s == p.stages) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1 && p.tc) {
    if (lane == 0) {
      int s = 0, b = 0;
      uint32_t ph = 0, tph[2] = {0, 0};
      const int per_tile = 8;
      for (int64_t i = 0; i < cn; ++i) {
        if (i % per_tile == 0) {
          bar_wait(tempty + b, tph[b] ^ 1u);
          tph[b] ^= 1u;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        bar_wait(full + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (p.tc == 2)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(empty + s)) : "memory");
        else
          bar_arrive(empty + s);
        if (++s == p.stages) { s = 0; ph ^= 1u; }
        if (i % per_tile == per_tile - 1 || i == cn - 1) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(tfull + b)) : "memory");
          b ^= 1;
        }
      }
      bar_arrive(never);
    }
  } else if (p.tc && warp >= 2 && warp <= 5) {
    const int per_tile = 8;
    const int64_t tiles = (cn + per_tile - 1) / per_tile;
    int b = 0;
    uint32_t tph[2] = {0, 0};
    for (int64_t t = 0; t < tiles; ++t) {
      bar_wait(tfull + b, tph[b]);
      tph[b] ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(tempty + b);
      b ^= 1;
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t i = 0; i < cn; ++i) {
        bar_wait(full + s, ph);
        bar_arrive(empty + s);
        if (++s == p.stages) { s = 0; ph ^= 1u; }
      }
      bar_arrive(never);
    }
  } else if (warp - 2 < p.spin) {
    bar_wait(never, 0);
  }
  __syncthreads();
  if (p.tmem && warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}

__global__ void fill_random(uint32_t* p, int64_t n, int mode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + 12345;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    uint32_t v = (uint32_t)z;
    if (mode == 2) v &= 0x0F0F0F0Fu;       // half the bits random
    if (mode == 3) v = (uint32_t)(z & 0xFFFF) * 0x00010001u;  // repeated halves
    p[i] = v;
  }
}

#ifndef STREAM_PROBE_LIB
int main(int argc, char** argv) {
  const int64_t bytes = (int64_t)4 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  const int fill = argc > 1 ? atoi(argv[1]) : 0;
  if (fill == 0) cudaMemset(buf, 1, bytes);
  else fill_random<<<4096, 256>>>(reinterpret_cast<uint32_t*>(buf), bytes / 4, fill);
  cudaDeviceSynchronize();
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct V { int threads, chunk, stages, tmem, spin, layout, tc; } vs[] = {
      {224, 65536, 3, 1, 0, 0, 1}, {224, 65536, 3, 1, 0, 2, 1}, {224, 65536, 3, 1, 0, 3, 1}, {224, 16384, 12, 1, 0, 2, 1},
      {224, 16384, 12, 1, 0, 3, 1}};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& v : vs) {
    P p{buf, bytes, v.chunk, v.stages, v.tmem, v.spin, v.layout, v.tc};
    const size_t smem = (size_t)v.stages * v.chunk + 8 * (2 * v.stages + 6);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      probe<<<sms, v.threads, smem>>>(p);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("fill=%d threads=%3d chunk=%6d stages=%2d tmem=%d spin=%2d layout=%d tc=%d : %.3f ms  %.2f TB/s  %s\n", fill, v.threads, v.chunk,
           v.stages, v.tmem, v.spin, v.layout, v.tc, best, bytes / best / 1e9, cudaGetErrorString(e));
  }
  return 0;
}

#endif

// Same streaming on a caller's buffer (ctypes): -> ms of the best of 5 launches.
extern "C" float stream_probe_ptr(const void* src, long long bytes, int chunk, int stages, int layout) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  P p{reinterpret_cast<const uint8_t*>(src), bytes, chunk, stages, 0, 0, layout, 1};
  const size_t smem = (size_t)stages * chunk + 8 * (2 * stages + 6);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    probe<<<sms, 224, smem>>>(p);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}
