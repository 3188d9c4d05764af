// sc_head.cu — the classifier head fused with the evaluation.
//
// z_i = x_i W_𝕎ᵀ + b_𝕎 over the |𝕎| mapped labels only (labels in no list never decide,
// PAPER.md:128-134, :862; Eq. api_output reads maxima over 𝕎 only),
// then the API-output epilogue of sc_loss_fwd_bwd (rows a3-a9) on the accumulators.
//
// One persistent CTA per SM, 128-row tiles, warp-specialised:
//   warp 0      TMA producer: per 64-wide k-block, the x tile [128 x 64] and the compiled
//               head W_𝕎 [n_cols x 64] (both K-major, 128-B swizzle) into a stage of the
//               shared-memory ring (full/empty mbarriers).
//   warp 1      allocates 512 TMEM columns; one lane issues tcgen05.mma (M=128, N=chunk,
//               K=16, bf16 x bf16 -> fp32 in TMEM), frees stages with tcgen05.commit and
//               signals the epilogue per tile (double-buffered accumulators when n_cols <= 256).
//   warps 2-5   epilogue: each thread owns one row (TMEM lane), tcgen05.ld its n_cols
//               accumulators, adds the bias, keeps the split maxima (P⁺ over cat ∈ G_i, P⁻
//               over the rest of 𝕎; ascending label order, so strict > keeps the smallest id
//               on ties, reading A8) and runs finish_batch (decision, counters, loss, grad).
// The features are the only HBM stream (d·2 bytes per row); W_𝕎 stays in L2.
#include "sc_device.cuh"
#include "sc_host.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

namespace sc {
namespace {

constexpr int kBM = 128;           // rows per tile (UMMA M)
constexpr int kBK = 64;            // bf16 elements per k-block = one 128-B swizzle row
constexpr int kHeadThreads = 192;  // 6 warps
constexpr int kMaxCols = 512;      // TMEM columns

struct HeadParams {
  EvalParams ep;            // context, ground truth, loss and output pointers (finish_batch)
  const uint32_t* keys;     // [n_cols] c << 8 | cat, kNone for padding columns
  const float* bias;        // [n_cols]
  int64_t rows, n_tiles;
  int32_t n_kb;             // k-blocks
  int32_t n_cols;           // head columns (multiple of 16)
  int32_t chunk;            // columns per MMA (n_cols or n_cols / 2)
  int32_t n_chunks;
  int32_t acc_bufs;         // 2: double-buffered accumulators
  int32_t stages;
  int32_t stage_bytes;      // A + B
  int32_t tab_off;          // keys / bias in shared memory
  int32_t bar_off;
};

// ------------------------------------------------------------------ tcgen05 / TMA PTX

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar,
                                       uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Shared-memory matrix descriptor, K-major, 128-B swizzle: rows of 128 B, 8-row groups
// 1024 B apart (SBO), LBO unused (1), descriptor version 1 (sm_100), layout 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

// Instruction descriptor, kind::f16: fp32 accumulator, bf16 A and B, both K-major, M=128, N.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(kBM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive once on `bar` when every tcgen05.mma issued so far by this thread has completed.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 32 lanes x 32 bits, 16 consecutive columns -> 16 registers per thread (thread t: lane t).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ kernel

__global__ void __launch_bounds__(kHeadThreads, 1)
    head_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                const HeadParams p) {
  extern __shared__ uint8_t sm_raw[];
  // 1024-B alignment for the 128-B swizzle atoms
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* s_keys = reinterpret_cast<uint32_t*>(sm + p.tab_off);
  float* s_bias = reinterpret_cast<float*>(s_keys + p.n_cols);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + p.bar_off);
  uint64_t* full = bar;                       // [stages]
  uint64_t* empty = bar + p.stages;           // [stages]
  uint64_t* tfull = bar + 2 * p.stages;       // [2]
  uint64_t* tempty = tfull + 2;               // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  for (int i = tid; i < p.n_cols; i += blockDim.x) {
    s_keys[i] = __ldg(p.keys + i);
    s_bias[i] = __ldg(p.bias + i);
  }
  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "n"(kMaxCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t a_bytes = kBM * kBK * 2;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      const uint64_t pol_x = evict_first_policy(), pol_w = evict_last_policy();
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        const int32_t row0 = static_cast<int32_t>(t * kBM);
        for (int kb = 0; kb < p.n_kb; ++kb) {
          mbar_wait(empty + s, ph ^ 1u);
          uint8_t* st = sm + static_cast<size_t>(s) * p.stage_bytes;
          mbar_arrive_expect_tx(full + s, static_cast<uint32_t>(p.stage_bytes));
          tma_2d(st, &map_x, kb * kBK, row0, full + s, pol_x);
          for (int c = 0; c < p.n_chunks; ++c)
            tma_2d(st + a_bytes + c * p.chunk * (kBK * 2), &map_w, kb * kBK, c * p.chunk, full + s, pol_w);
          if (++s == p.stages) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      const uint32_t idesc = idesc_bf16(p.chunk);
      int s = 0, b = 0;
      uint32_t ph = 0, tph[2] = {0, 0};
      for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        mbar_wait(tempty + b, tph[b] ^ 1u);  // the epilogue drained this accumulator
        tph[b] ^= 1u;
        tc_fence_after();
        const uint32_t acc = tmem_base + static_cast<uint32_t>(b * p.n_cols);
        for (int kb = 0; kb < p.n_kb; ++kb) {
          mbar_wait(full + s, ph);
          tc_fence_after();
          const uint32_t sa = smem_addr(sm + static_cast<size_t>(s) * p.stage_bytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = sw128_desc(sa + 32u * k);
            for (int c = 0; c < p.n_chunks; ++c) {
              const uint64_t bd = sw128_desc(sa + a_bytes + c * p.chunk * (kBK * 2) + 32u * k);
              umma_bf16(acc + c * p.chunk, ad, bd, idesc, (kb | k) != 0);
            }
          }
          umma_commit(empty + s);  // stage reusable once these MMAs have read it
          if (++s == p.stages) {
            s = 0;
            ph ^= 1u;
          }
        }
        umma_commit(tfull + b);  // accumulator complete
        if (p.acc_bufs == 2) b ^= 1;
      }
    }
  } else {
    // ---------------- epilogue: one row per thread
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t lane_base = static_cast<uint32_t>(32 * q) << 16;
    const EvalParams& ep = p.ep;
    const uint8_t* cat = ep.ctx.cat;
    int b = 0;
    uint32_t tph[2] = {0, 0};
    RowBatch rb;
    rb.n = 0;
    for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      const int64_t row = t * kBM + 32 * q + lane;
      const bool active = row < p.rows;
      // G_i before waiting on the accumulator (overlaps the MMA)
      uint32_t G = 0;
      if (active) {
        if (ep.gt_mask) {
          G = __ldg(ep.gt_mask + row);
        } else if (ep.gt_off) {
          const int64_t g0 = __ldg(ep.gt_off + row), g1 = __ldg(ep.gt_off + row + 1);
          for (int64_t i = g0; i < g1; ++i) G |= label_lists(__ldg(cat + __ldg(ep.gt_lab + i)), kApiOutput);
        }
      }
      mbar_wait(tfull + b, tph[b]);
      tph[b] ^= 1u;
      tc_fence_after();
      float zp = -CUDART_INF_F, zm = -CUDART_INF_F;
      uint32_t kp = kNone, km = kNone;
      const uint32_t acc = tmem_base + lane_base + static_cast<uint32_t>(b * p.n_cols);
      for (int c0 = 0; c0 < p.n_cols; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(acc + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t key = s_keys[c0 + j];
          if (key == kNone) continue;
          const float z = __uint_as_float(v[j]) + s_bias[c0 + j];
          if ((G >> (key & 0xFFu)) & 1u) {
            if (z > zp) { zp = z; kp = key; }
          } else {
            if (z > zm) { zm = z; km = key; }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + b);  // the MMA may overwrite this accumulator
      if (p.acc_bufs == 2) b ^= 1;
      const int64_t first = t * kBM + 32 * q;
      const int64_t nrow = p.rows - first;
      if (nrow > 0) {
        rb.zp = zp; rb.kp = kp; rb.zm = zm; rb.km = km; rb.G = G; rb.app = 0; rb.row = row;
        rb.n = nrow < 32 ? static_cast<int>(nrow) : 32;
        finish_batch(ep, rb, nullptr, lane);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kMaxCols)
                 : "memory");
  }
}

// Compiled head rows: Wm[j] = W[c_j] (zero padding to d_pad, zero rows past |𝕎|).
__global__ void head_gather_kernel(const uint16_t* W, int64_t ldw, int64_t d, int64_t d_pad, const float* bias,
                                   const uint32_t* ent, int32_t n_mapped, int32_t n_cols, uint16_t* Wm,
                                   float* bias_m, uint32_t* keys) {
  const int j = blockIdx.x;
  const bool mapped = j < n_mapped;
  const uint32_t key = mapped ? ent[j] : kNone;
  const int64_t c = key >> 8;
  for (int64_t i = threadIdx.x; i < d_pad; i += blockDim.x)
    Wm[static_cast<int64_t>(j) * d_pad + i] = (mapped && i < d) ? W[c * ldw + i] : uint16_t(0);
  if (threadIdx.x == 0) {
    keys[j] = key;
    bias_m[j] = (mapped && bias) ? bias[c] : 0.f;
  }
  (void)n_cols;
}

}  // namespace
}  // namespace sc

// ------------------------------------------------------------------ host

struct sc_head_s {
  int device = 0;
  int64_t d = 0, d_pad = 0;
  int32_t n_mapped = 0, n_cols = 0, chunk = 0, n_chunks = 0;
  uint16_t* Wm = nullptr;  // [n_cols][d_pad]
  float* bias = nullptr;   // [n_cols]
  uint32_t* keys = nullptr;
  CUtensorMap map_w;
};

namespace {

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static std::once_flag once;
  static EncodeTiled fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows][ld] matrix: box = box_rows x 64, 128-B swizzle.
bool make_map(CUtensorMap* m, const void* base, int64_t cols, int64_t rows, int64_t ld, int box_rows) {
  EncodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(sc::kBK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr size_t kHeadSmemMax = 227 * 1024;

}  // namespace

extern "C" {

sc_status sc_head_load(sc_context ctx, const uint16_t* weight, int64_t ldw, int64_t d, const float* bias,
                       sc_stream stream, sc_head* out) {
  if (!ctx || !weight || !out) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_load: NULL argument");
  *out = nullptr;
  if (d < 1 || ldw < d) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_load: need d >= 1 and ldw >= d");
  if (ctx->order != SC_ORDER_API_OUTPUT || ctx->n_apps != 1)
    return sc::set_error(SC_ERR_UNSUPPORTED, "sc_head_load: API-output order and one application only");
  const int32_t nm = ctx->n_mapped[0];
  if (nm > sc::kMaxCols)
    return sc::set_error(SC_ERR_UNSUPPORTED, "sc_head_load: |W| = %d mapped labels > %d", nm, sc::kMaxCols);
  if (d > (int64_t(1) << 31) - sc::kBK) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_load: d too large");
  sc_head h = new sc_head_s;
  h->d = d;
  h->d_pad = (d + 7) / 8 * 8;
  h->n_mapped = nm;
  int32_t n = std::max<int32_t>(16, (nm + 15) / 16 * 16);
  if (n <= 256) {
    h->chunk = n;
    h->n_chunks = 1;
  } else {  // two equal MMAs of <= 256 columns (one TMA box size)
    h->chunk = ((n + 1) / 2 + 15) / 16 * 16;
    h->n_chunks = 2;
    n = 2 * h->chunk;
  }
  h->n_cols = n;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaGetDevice(&h->device);
  if (!e) e = cudaMalloc(&h->Wm, static_cast<size_t>(n) * h->d_pad * 2);
  if (!e) e = cudaMalloc(&h->bias, static_cast<size_t>(n) * 4);
  if (!e) e = cudaMalloc(&h->keys, static_cast<size_t>(n) * 4);
  if (!e) {
    sc::head_gather_kernel<<<n, 256, 0, st>>>(weight, ldw, d, h->d_pad, bias, ctx->d_ent, nm, n, h->Wm, h->bias,
                                             h->keys);
    sc::note_launch("head_gather");
    e = cudaGetLastError();
  }
  if (!e) e = cudaStreamSynchronize(st);
  if (e) {
    sc_head_free(h);
    return sc::set_error(e == cudaErrorMemoryAllocation ? SC_ERR_OOM : SC_ERR_CUDA, "sc_head_load: %s",
                         cudaGetErrorString(e));
  }
  if (!make_map(&h->map_w, h->Wm, d, n, h->d_pad, h->chunk)) {
    sc_head_free(h);
    return sc::set_error(SC_ERR_CUDA, "sc_head_load: cuTensorMapEncodeTiled failed");
  }
  *out = h;
  return SC_OK;
}

sc_status sc_head_free(sc_head h) {
  if (!h) return SC_OK;
  cudaFree(h->Wm);
  cudaFree(h->bias);
  cudaFree(h->keys);
  delete h;
  return SC_OK;
}

sc_status sc_head_info(sc_head h, int64_t* d, int32_t* n_cols) {
  if (!h) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_info: NULL head");
  if (d) *d = h->d;
  if (n_cols) *n_cols = h->n_cols;
  return SC_OK;
}

sc_status sc_head_loss_fwd_bwd(sc_context ctx, sc_head head, const sc_head_batch* batch, const float* w,
                               float grad_scale, double* loss_sum, float* loss_row, int32_t* grad_idx,
                               float* grad_val, uint8_t* decision, uint64_t* n_incorrect, uint64_t* hist_pred,
                               uint64_t* hist_gt, sc_stream stream) {
  if (!ctx || !head || !batch) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: NULL argument");
  if (ctx->order != SC_ORDER_API_OUTPUT || ctx->n_apps != 1)
    return sc::set_error(SC_ERR_UNSUPPORTED, "sc_head_loss_fwd_bwd: API-output order and one application only");
  const sc_head_batch& b = *batch;
  if (b.rows < 0) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: rows < 0");
  if (b.rows > (int64_t(1) << 31) - sc::kBM)
    return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: rows >= 2^31");
  if (b.rows > 0 && !b.x) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: x is NULL");
  if (b.ldx < head->d || b.ldx % 8 != 0 || (reinterpret_cast<uintptr_t>(b.x) & 15u))
    return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: need ldx >= d, ldx %% 8 == 0, x 16-B aligned");
  const bool has_gt = b.gt_mask || (b.gt_off && b.gt_lab);
  const bool want_loss = loss_sum || loss_row || grad_idx || grad_val;
  if (!has_gt && (want_loss || n_incorrect || hist_gt))
    return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: the loss and the counters need ground truth");
  if (b.rows == 0) return SC_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != head->device) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: head on another device");

  sc::HeadParams p{};
  sc::EvalParams& ep = p.ep;
  ep.ctx.cat = ctx->d_cat;
  ep.ctx.ent = ctx->d_ent;
  ep.ctx.ent_off = ctx->d_ent_off;
  ep.ctx.nlists = ctx->d_nlists;
  ep.ctx.C = ctx->C;
  ep.ctx.n_apps = ctx->n_apps;
  ep.ctx.max_ent = ctx->max_ent;
  ep.ctx.tau = ctx->tau;
  ep.ctx.theta = ctx->theta;
  ep.ctx.k = ctx->k;
  ep.ctx.order = ctx->order;
  ep.rows = b.rows;
  ep.gt_off = b.gt_mask ? nullptr : b.gt_off;
  ep.gt_lab = b.gt_lab;
  ep.gt_mask = b.gt_mask;
  ep.has_gt = has_gt;
  ep.w = w;
  ep.grad_scale = grad_scale;
  ep.want_loss = want_loss;
  ep.loss_sum = loss_sum;
  ep.loss_row = loss_row;
  ep.grad_idx = grad_idx;
  ep.grad_val = grad_val;
  ep.decision = decision;
  ep.n_incorrect = reinterpret_cast<unsigned long long*>(n_incorrect);
  ep.hist_pred = reinterpret_cast<unsigned long long*>(hist_pred);
  ep.hist_gt = reinterpret_cast<unsigned long long*>(hist_gt);

  p.keys = head->keys;
  p.bias = head->bias;
  p.rows = b.rows;
  p.n_tiles = (b.rows + sc::kBM - 1) / sc::kBM;
  p.n_kb = static_cast<int32_t>((head->d + sc::kBK - 1) / sc::kBK);
  p.n_cols = head->n_cols;
  p.chunk = head->chunk;
  p.n_chunks = head->n_chunks;
  p.acc_bufs = 2 * head->n_cols <= sc::kMaxCols ? 2 : 1;
  p.stage_bytes = sc::kBM * sc::kBK * 2 + head->n_cols * sc::kBK * 2;
  const int tab_bytes = head->n_cols * 8;
  const int bar_bytes = 8 * (2 * 8 + 4) + 16;
  int stages = static_cast<int>((kHeadSmemMax - 1024 - tab_bytes - bar_bytes) / p.stage_bytes);
  stages = std::min(stages, 8);
  if (const char* s = getenv("SC_HEAD_STAGES")) stages = std::max(1, std::min(stages, atoi(s)));
  if (stages < 2) return sc::set_error(SC_ERR_UNSUPPORTED, "sc_head_loss_fwd_bwd: head too wide for the ring");
  p.stages = stages;
  p.tab_off = stages * p.stage_bytes;
  p.bar_off = (p.tab_off + tab_bytes + 7) / 8 * 8;
  const size_t smem = 1024 + p.bar_off + 8 * (2 * stages + 4) + 16;

  CUtensorMap map_x;
  if (!make_map(&map_x, b.x, head->d, b.rows, b.ldx, sc::kBM))
    return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: cuTensorMapEncodeTiled failed");
  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [] {
    attr_err = cudaFuncSetAttribute(sc::head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kHeadSmemMax));
  });
  if (attr_err) return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: %s", cudaGetErrorString(attr_err));
  const int sms = sc::device_sms();
  const int grid = static_cast<int>(std::min<int64_t>(p.n_tiles, sms));
  sc::head_kernel<<<grid, sc::kHeadThreads, smem, static_cast<cudaStream_t>(stream)>>>(map_x, head->map_w, p);
  sc::note_launch("head_tcgen05");
  if (cudaError_t e = cudaGetLastError())
    return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: %s", cudaGetErrorString(e));
  return SC_OK;
}

}  // extern "C"
