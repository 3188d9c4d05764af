// sc_head.cu — the classifier head fused with the evaluation.
//
// z_i = x_i W_𝕎ᵀ + b_𝕎 over the |𝕎| mapped labels only (labels in no list never decide,
// PAPER.md:128-134, :862; Eq. api_output reads maxima over 𝕎 only),
// then the API-output epilogue of sc_loss_fwd_bwd (rows a3-a9) on the accumulators.
//
// Head columns are grouped by list (code order), ascending label id inside a list, each
// list padded to a multiple of 16 columns (zero weights, bias -inf), so the epilogue takes
// per-list arg maxima over whole 16-column TMEM loads with a branch-free tree and never
// looks a column's list up; P⁺ / P⁻ are then arg maxima over the <= 8 list winners.
//
// Persistent CTAs (one per SM), 128-row tiles, warp-specialised:
//   warp 0      x producer: per stage, kbs 64-wide k-blocks of the CTA's x tile [128 x 64]
//               (one 3-D TMA box, K-major, 128-B swizzle, L2 evict-first).
//   warp 6      W producer: one k-block of the compiled head W_𝕎 [n_cols x 64] per stage
//               (k-block-major layout, L2 evict-last: W is re-read for every row tile).
//   warp 1      allocates 512 TMEM columns; one lane issues tcgen05.mma (M=128, N <= 256,
//               K=16, bf16 x bf16 -> fp32 in TMEM) and frees the x / W stages with
//               tcgen05.commit; double-buffered accumulators when n_cols <= 256.
//   warps 2-5   epilogue: each thread owns one row (TMEM lane), tcgen05.ld its columns 16 at
//               a time (the next load in flight while the current one is reduced), adds the
//               bias, per-list arg max, split maxima by G_i, then finish_batch (decision,
//               counters, loss, gradient).
//   warps 7-10  the same for the unit's second row tile: lone CTAs run two 128-row tiles per
//               unit that share every W stage (two accumulators in TMEM, single-buffered),
//               so W_𝕎 — re-read from L2 for every unit — moves half the bytes per row.
// PAIR (opt-in, SC_HEAD_CLUSTER=2): CTA pairs run M = 256 MMAs with cta_group::2, each CTA
// streaming its own 128 rows of x and half of W_𝕎; the leader's barriers count both CTAs'
// bytes and a multicast tcgen05.commit frees the stages of both.
#include "sc_device.cuh"
#include "sc_host.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

namespace sc {
namespace {

constexpr int kBM = 128;           // rows per tile (UMMA M)
constexpr int kBK = 64;            // bf16 elements per k-block = one 128-B swizzle row
constexpr int kHeadThreads = 352;  // 11 warps: x / MMA / 4 epilogue / W / 4 epilogue (second tile)
constexpr int kMaxCols = 512;      // TMEM columns
constexpr int kPassCols = 256;     // columns per pass when a head has more than kMaxCols (one MMA, N <= 256)
constexpr int kMaxHeadCols = 4096; // keys + bias tables in shared memory (32 KB)
constexpr int kMaxLists = 8;

struct HeadParams {
  EvalParams ep;            // context, ground truth, loss and output pointers (finish_batch)
  const uint32_t* keys;     // [n_cols] c << 8 | cat, kNone for padding columns
  const float* bias;        // [n_cols], -inf for padding columns
  int64_t rows;
  int64_t n_units;          // row units: 128 rows (one CTA) or 256 rows (a CTA pair)
  int32_t n_kb;             // k-blocks
  int32_t n_cols;           // head columns (multiple of 32)
  int32_t chunk;            // columns per MMA (n_cols or n_cols / 2)
  int32_t n_chunks;
  int32_t acc_bufs;         // 2: double-buffered accumulators
  int32_t tiles;            // row tiles per unit sharing every W stage (1, or 2 for lone CTAs)
  int32_t kbs;              // k-blocks per x stage (one 3-D TMA box of kbs x [128 x 64])
  int32_t n_xb;             // x stages per unit = ceil(n_kb / kbs)
  int32_t x_stages, w_stages;
  int32_t x_stage_bytes;    // kbs * 16 KB
  int32_t w_stage_bytes;    // W rows this CTA holds * 128 B (one k-block)
  int32_t w_ring_off;       // byte offset of the W ring (after the x ring)
  int32_t x3d;              // x tensor map is 3-D {64, rows, n_kb} (d % 64 == 0), else 2-D
  int32_t tab_off;          // keys / bias in shared memory
  int32_t bar_off;
  int32_t n_lists;          // D'
  int32_t list_col0[kMaxLists];  // first column of list j (multiple of 16)
  int32_t list_nch[kMaxLists];   // 16-column groups of list j
  int32_t probe;            // experiment (SC_HEAD_PROBE): bit 0 skips the epilogue's reduction, bit 1 the MMAs,
                            // bit 2 the x loads, bit 3 the W loads (lone CTAs; results are garbage),
                            // bit 4 the drain's reduction (loads kept), bit 5 the drain's TMEM loads
  int32_t n_pass;           // column passes per row tile: 1 = every column in TMEM at once (n_cols <= 512);
                            // > 1 = pass_w columns per pass, x re-streamed per pass (from L2)
  int32_t pass_w;           // columns per pass (n_pass > 1; = chunk)
  int32_t pat;              // 0: API-output order (split maxima); 1: per-list patterns (finish_lists_core)
  int32_t n_groups;         // 16-column groups holding list columns (the lists back to back)
  unsigned long long* trace;  // experiment (SC_HEAD_TRACE=file): per-unit timeline of CTAs < kTraceCtas, or NULL
};

// Timeline probe (SC_HEAD_TRACE): globaltimer stamps (ns) and wait sums per (CTA, unit) for
// the first kTraceCtas CTAs and kTraceUnits units; slots: 0/1 MMA waits the accumulator
// (start / acquired), 2/3 MMA's summed waits on x / W stages, 4 MMA's last commit of the unit,
// 5/6 epilogue warp 2 waits the accumulator (start / acquired), 7 its drain done, 8 its finish
// done, 9/10 x / W producers' summed waits for free stages, 11/12 epilogue warp 7 acquired /
// drained.
constexpr int kTraceCtas = 8, kTraceUnits = 32, kTraceSlots = 16;
__device__ __forceinline__ unsigned long long tnow() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long* trace_slot(const HeadParams& p, int64_t st) {
  if (p.trace == nullptr || blockIdx.x >= kTraceCtas || st >= kTraceUnits) return nullptr;
  return p.trace + (static_cast<int64_t>(blockIdx.x) * kTraceUnits + st) * kTraceSlots;
}

// ------------------------------------------------------------------ tcgen05 / TMA / cluster PTX

// TMA tile loads.  CG2: the CTA-pair form, whose mbarrier may live in the peer CTA (the
// pair's leader counts the bytes both CTAs load).
template <bool CG2>
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t bar,
                                       uint64_t pol) {
  if constexpr (CG2)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
        : "memory");
}

// 3-D box {64, 128 rows, kbs k-blocks} of x viewed as [n_kb][rows][64]: kbs swizzled
// [128 x 64] tiles back to back, each row's kbs*128 B contiguous in global memory.
template <bool CG2>
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                       uint32_t bar, uint64_t pol) {
  if constexpr (CG2)
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
        : "memory");
}

__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t evict_normal_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of the same shared variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}


__device__ __forceinline__ void mbar_arrive_cl(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
}

// Shared-memory matrix descriptor, K-major, 128-B swizzle: rows of 128 B, 8-row groups
// 1024 B apart (SBO), LBO unused (1), descriptor version 1 (sm_100), layout 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

// Instruction descriptor, kind::f16: fp32 accumulator, bf16 A and B, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

// D (TMEM) (+)= A (smem) · Bᵀ (smem).  CG2: M = 256 over the CTA pair — each CTA holds its
// 128 rows of A and half of B's columns at the same shared-memory offsets, and receives its
// 128 rows x N of D in its own TMEM; issued by the pair's leader only.
// Called by the whole (converged) MMA warp with warp-uniform operands, which then stay in
// uniform registers; one elected lane issues.  (Issued from a lane-0-only branch, every MMA
// was wrapped in an ELECT / R2UR.BROADCAST loop: ~200 cycles per MMA, measured, against a
// ~96-cycle tensor floor for M = 128, N = 192.)
template <bool CG2>
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  if constexpr (CG2)
    asm volatile(
        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// mbarrier wait for a whole converged warp whose loop exit is provably warp-uniform (a vote):
// after it the compiler keeps warp-uniform values (the MMA descriptors) in uniform registers.
// (An asm spin loop with a per-thread branch makes everything after it look divergent.)
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (__all_sync(0xFFFFFFFFu, ok)) break;
  }
}

// One k-block (4 K = 16 steps) of MMAs: NCH column chunks x NTL row tiles, each its own
// accumulator at acc + t*tc_step + c*cc_step; A of tile t at ad + t*t_step, B of chunk c at
// bd + c*c_step (descriptor units).
template <bool CG2, int NCH, int NTL>
__device__ __forceinline__ void mma_kblock(uint32_t acc, uint64_t ad, uint64_t bd, uint64_t t_step, uint64_t c_step,
                                           uint32_t tc_step, uint32_t cc_step, uint32_t idesc, bool first) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t accum = (first && k == 0) ? 0u : 1u;
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
      for (int t = 0; t < NTL; ++t)
        umma_bf16<CG2>(acc + t * tc_step + c * cc_step, ad + t * t_step + 2 * k, bd + c * c_step + 2 * k, idesc,
                       accum);
  }
}

// Arrive once on `bar` (CG2: at `bar`'s offset in both CTAs of the pair) when every
// tcgen05.mma issued so far by this thread has completed.
// Elected like umma_bf16 (called by the whole MMA warp).
template <bool CG2>
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  if constexpr (CG2)
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::
            "r"(smem_addr(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  else
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_addr(bar))
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
// 32 lanes x 32 bits, 32 consecutive columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld32(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                 "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                 "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}


// Arg max of 16 columns (z, index); strict > keeps the lower index on ties (reading A4:
// the lower column of a list is the smaller label id).
__device__ __forceinline__ void argmax16(const float (&z)[16], float& zo, int& io) {
  float a[8];
  int ia[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool r = z[2 * i + 1] > z[2 * i];
    a[i] = r ? z[2 * i + 1] : z[2 * i];
    ia[i] = r ? 2 * i + 1 : 2 * i;
  }
#pragma unroll
  for (int w = 4; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const bool r = a[2 * i + 1] > a[2 * i];
      a[i] = r ? a[2 * i + 1] : a[2 * i];
      ia[i] = r ? ia[2 * i + 1] : ia[2 * i];
    }
  zo = a[0];
  io = ia[0];
}

// ------------------------------------------------------------------ kernel

// PAIR: clusters of two CTAs on one TPC run M = 256 MMAs (cta_group::2): each CTA streams
// its own 128 rows of x and half of W_𝕎, so a CTA moves half the W bytes per row that a lone
// CTA would (W, re-read for every row tile, outweighs x at d = 2048, |𝕎| = 180).
template <bool PAIR>
__global__ void __launch_bounds__(kHeadThreads, 1)
    head_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                const __grid_constant__ HeadParams p) {
  extern __shared__ uint8_t sm_raw[];
  // 1024-B alignment for the 128-B swizzle atoms (the same offsets in both CTAs of a pair)
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* s_keys = reinterpret_cast<uint32_t*>(sm + p.tab_off);
  float* s_bias = reinterpret_cast<float*>(s_keys + p.n_cols);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + p.bar_off);
  uint64_t* xfull = bar;                      // [x_stages]  (PAIR: the leader's counts both CTAs)
  uint64_t* xempty = xfull + p.x_stages;      // [x_stages]
  uint64_t* wfull = xempty + p.x_stages;      // [w_stages]  (PAIR: the leader's counts both CTAs)
  uint64_t* wempty = wfull + p.w_stages;      // [w_stages]
  uint64_t* tfull = wempty + p.w_stages;      // [2]
  uint64_t* tempty = tfull + 2;               // [2]         (PAIR: the leader's counts both CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  // rows per unit: p.tiles row tiles sharing each W stage, of 128 rows (one CTA) or 256 rows
  // (a CTA pair: rows [t*256, t*256 + 128) in CTA 0, the next 128 in CTA 1)
  const int kTileRows = PAIR ? 2 * kBM : kBM;
  const int kUnit = p.tiles * kTileRows;

  for (int i = tid; i < p.n_cols; i += blockDim.x) {
    s_keys[i] = __ldg(p.keys + i);
    s_bias[i] = __ldg(p.bias + i);
  }
  if (tid == 0) {
    for (int s = 0; s < p.x_stages; ++s) {
      mbar_init(xfull + s, 1);  // PAIR: the leader's one arrival expects both CTAs' bytes
      mbar_init(xempty + s, 1);
    }
    for (int s = 0; s < p.w_stages; ++s) {
      mbar_init(wfull + s, 1);
      mbar_init(wempty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, (PAIR ? 8 : 4) * p.tiles);  // one arrive per working epilogue warp (of both CTAs)
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                   "n"(kMaxCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                   "n"(kMaxCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // both CTAs' barriers exist before either signals the other
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t a_bytes = kBM * kBK * 2;
  // units u = unit0 + step * n_grid_units (a pair shares its unit sequence)
  const int64_t unit0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t n_grid_units = PAIR ? gridDim.x / 2 : gridDim.x;
  const int64_t n_steps = unit0 < p.n_units ? (p.n_units - unit0 + n_grid_units - 1) / n_grid_units : 0;
  // the leader's full barriers, in shared::cluster space (its own for a lone CTA)
  const uint32_t xfull_l = PAIR ? mapa(smem_addr(xfull), 0) : smem_addr(xfull);
  const uint32_t wfull_l = PAIR ? mapa(smem_addr(wfull), 0) : smem_addr(wfull);
  const uint32_t tempty_l = PAIR ? mapa(smem_addr(tempty), 0) : smem_addr(tempty);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- x producer: kbs k-blocks of this CTA's 128 rows per stage (from HBM)
      const uint64_t pol_first = evict_first_policy();
      const uint64_t pol_keep = evict_normal_policy();  // column passes: the tile is read again from L2
      const uint32_t tx = static_cast<uint32_t>(p.x_stage_bytes);
      int s = 0;
      uint32_t ph = 0;
      for (int64_t st = 0; st < n_steps; ++st) {
        // may be past the last row: TMA fills zeros, the epilogue skips those rows
        const int32_t row0 = static_cast<int32_t>((unit0 + st * n_grid_units) * kUnit + rank * kBM);
        for (int ps = 0; ps < p.n_pass; ++ps) {
        const uint64_t pol_x = ps + 1 < p.n_pass ? pol_keep : pol_first;
        for (int xb = 0; xb < p.n_xb; ++xb) {
          if (unsigned long long* tr = trace_slot(p, st)) {
            const unsigned long long t0 = tnow();
            mbar_wait(xempty + s, ph ^ 1u);
            tr[9] += tnow() - t0;
          } else {
            mbar_wait(xempty + s, ph ^ 1u);
          }
          uint8_t* stg = sm + static_cast<size_t>(s) * p.x_stage_bytes;
          const uint32_t fb = xfull_l + 8u * s;
          if (!PAIR && (p.probe & 4)) {  // probe: no x traffic, the MMAs run on stale stages
            mbar_arrive(xfull + s);
            if (++s == p.x_stages) {
              s = 0;
              ph ^= 1u;
            }
            continue;
          }
          // CTA pairs: only the leader arrives, expecting both CTAs' bytes (the peer's copies
          // complete their bytes on the leader's barrier).  A remote arrive.expect_tx per stage
          // from the peer (release at cluster scope) serialised its producer: measured, the
          // leader's MMA waited 18 µs of every 32 µs unit on the peer's stages.
          if (rank == 0) mbar_arrive_expect_tx(xfull + s, PAIR ? 2 * tx : tx);
          for (int t = 0; t < p.tiles; ++t) {  // tile t: kbs k-blocks at t * kbs * 16 KB
            uint8_t* dst = stg + static_cast<size_t>(t) * p.kbs * (kBM * kBK * 2);
            if (p.x3d) tma_3d<PAIR>(dst, &map_x, 0, row0 + t * kTileRows, xb * p.kbs, fb, pol_x);
            else tma_2d<PAIR>(dst, &map_x, xb * kBK, row0 + t * kTileRows, fb, pol_x);
          }
          if (++s == p.x_stages) {
            s = 0;
            ph ^= 1u;
          }
        }
        }
      }
    }
  } else if (warp == 6) {
    if (lane == 0) {
      // ---------------- W producer: one k-block of this CTA's W_𝕎 rows per stage (L2-resident)
      const uint64_t pol_w = evict_last_policy();
      const uint32_t tx = static_cast<uint32_t>(p.w_stage_bytes);
      const int rows_c = PAIR ? p.chunk / 2 : p.chunk;  // W rows per MMA chunk held here
      int s = 0;
      uint32_t ph = 0;
      for (int64_t st = 0; st < n_steps; ++st) {
        for (int ps = 0; ps < p.n_pass; ++ps) {
        const int col0 = ps * p.pass_w;  // 0 when n_pass == 1
        for (int kb = 0; kb < p.n_kb; ++kb) {
          if (unsigned long long* tr = trace_slot(p, st)) {
            const unsigned long long t0 = tnow();
            mbar_wait(wempty + s, ph ^ 1u);
            tr[10] += tnow() - t0;
          } else {
            mbar_wait(wempty + s, ph ^ 1u);
          }
          uint8_t* stg = sm + p.w_ring_off + static_cast<size_t>(s) * p.w_stage_bytes;
          const uint32_t fb = wfull_l + 8u * s;
          if (!PAIR && (p.probe & 8)) {  // probe: no W traffic
            mbar_arrive(wfull + s);
            if (++s == p.w_stages) {
              s = 0;
              ph ^= 1u;
            }
            continue;
          }
          if (rank == 0) mbar_arrive_expect_tx(wfull + s, PAIR ? 2 * tx : tx);
          for (int c = 0; c < p.n_chunks; ++c)
            tma_2d<PAIR>(stg + c * rows_c * (kBK * 2), &map_w, 0,
                         kb * p.n_cols + col0 + c * p.chunk + static_cast<int>(rank) * rows_c, fb, pol_w);
          if (++s == p.w_stages) {
            s = 0;
            ph ^= 1u;
          }
        }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (the pair's leader): the whole warp runs the loop (operands
      // warp-uniform, so they live in uniform registers); one elected lane issues
      const uint32_t idesc = idesc_bf16(PAIR ? 2 * kBM : kBM, p.chunk);
      // descriptors advance by address >> 4 in their low bits: x stage, k-block in the
      // stage (16 KB), 32 B per K=16 step; W stage; second MMA's columns
      const uint64_t a_desc0 = sw128_desc(smem_addr(sm));
      const uint64_t b_desc0 = sw128_desc(smem_addr(sm + p.w_ring_off));
      const uint64_t x_step = static_cast<uint32_t>(p.x_stage_bytes) >> 4;
      const uint64_t w_step = static_cast<uint32_t>(p.w_stage_bytes) >> 4;
      const uint64_t c_step = static_cast<uint32_t>((PAIR ? p.chunk / 2 : p.chunk) * kBK * 2) >> 4;
      const int nch = p.n_chunks, ntl = p.tiles;
      const uint64_t t_step = static_cast<uint32_t>(p.kbs * a_bytes) >> 4;  // tile 1 in an x stage
      const bool no_mma = (p.probe & 2) != 0;
      int xs = 0, ws = 0, b = 0;
      uint32_t xph = 0, wph = 0, tph[2] = {0, 0};
      // accumulator buffer b at column b * acc_stride (a column pass holds pass_w columns)
      const int acc_stride = p.n_pass > 1 ? p.pass_w : p.n_cols;
      for (int64_t st = 0; st < n_steps; ++st) {
        for (int ps = 0; ps < p.n_pass; ++ps) {
        // probe stamps: every lane takes the same path (the waits below vote), lane 0 writes
        unsigned long long* tr = ps == 0 ? trace_slot(p, st) : nullptr;
        if (tr && lane == 0) tr[0] = tnow();
        mbar_wait_warp(tempty + b, tph[b] ^ 1u);  // the epilogue(s) drained this accumulator
        if (tr && lane == 0) tr[1] = tnow();
        tph[b] ^= 1u;
        tc_fence_after();
        const uint32_t acc = tmem_base + static_cast<uint32_t>(b * acc_stride);
        for (int xb = 0; xb < p.n_xb; ++xb) {
          if (tr) {
            const unsigned long long t0 = tnow();
            mbar_wait_warp(xfull + xs, xph);
            if (lane == 0) tr[2] += tnow() - t0;
          } else {
            mbar_wait_warp(xfull + xs, xph);
          }
          tc_fence_after();
          const uint64_t ax = a_desc0 + static_cast<uint64_t>(xs) * x_step;
          const int nk = min(p.kbs, p.n_kb - xb * p.kbs);
          for (int kx = 0; kx < nk; ++kx) {
            if (tr) {
              const unsigned long long t0 = tnow();
              mbar_wait_warp(wfull + ws, wph);
              if (lane == 0) tr[3] += tnow() - t0;
            } else {
              mbar_wait_warp(wfull + ws, wph);
            }
            tc_fence_after();
            const uint64_t ad = ax + static_cast<uint64_t>(kx) * (a_bytes >> 4);
            const uint64_t bd = b_desc0 + static_cast<uint64_t>(ws) * w_step;
            if (!no_mma) {
              const bool first = (xb | kx) == 0;
              // column chunk c of row tile t: its own accumulator (t * n_cols + c * chunk), so
              // the nch * ntl MMAs of a k-step are independent chains the tensor pipe overlaps
              // (measured: back-to-back MMAs into one accumulator serialise at ~195 ns each).
              // One straight-line instance per (nch, ntl): a predicated-off tcgen05.mma is not
              // free (measured: 8 guarded MMAs per k-step ran at half the rate).
              const uint32_t tc_step = static_cast<uint32_t>(p.n_cols), cc_step = static_cast<uint32_t>(p.chunk);
              switch (nch * 2 + ntl - 1) {
                case 2: mma_kblock<PAIR, 1, 1>(acc, ad, bd, t_step, c_step, tc_step, cc_step, idesc, first); break;
                case 3: mma_kblock<PAIR, 1, 2>(acc, ad, bd, t_step, c_step, tc_step, cc_step, idesc, first); break;
                case 4: mma_kblock<PAIR, 2, 1>(acc, ad, bd, t_step, c_step, tc_step, cc_step, idesc, first); break;
                case 5: mma_kblock<PAIR, 2, 2>(acc, ad, bd, t_step, c_step, tc_step, cc_step, idesc, first); break;
                case 8: mma_kblock<PAIR, 4, 1>(acc, ad, bd, t_step, c_step, tc_step, cc_step, idesc, first); break;
                default: mma_kblock<PAIR, 4, 2>(acc, ad, bd, t_step, c_step, tc_step, cc_step, idesc, first); break;
              }
            }
            umma_commit<PAIR>(wempty + ws);  // W stage free (in both CTAs) once read
            if (++ws == p.w_stages) {
              ws = 0;
              wph ^= 1u;
            }
          }
          umma_commit<PAIR>(xempty + xs);
          if (++xs == p.x_stages) {
            xs = 0;
            xph ^= 1u;
          }
        }
        umma_commit<PAIR>(tfull + b);  // accumulator complete (in both CTAs)
        if (tr && lane == 0) tr[4] = tnow();
        if (p.acc_bufs == 2) b ^= 1;
        }
      }
    }
  } else if (warp <= 5 || (warp >= 7 && warp <= 10 && p.tiles == 2)) {
    // ---------------- epilogue: one row per thread
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t lane_base = static_cast<uint32_t>(32 * q) << 16;
    const EvalParams& ep = p.ep;
    const uint8_t* cat = ep.ctx.cat;
    const int D = p.n_lists;
    int b = 0;
    uint32_t tph[2] = {0, 0};
    RowBatch rb;
    rb.n = 0;
    const int ntile = p.tiles;
    // two tiles per unit: warps 2-5 drain tile 0, warps 7-10 tile 1 (lane quarters 3,0,1,2);
    // each warp drains one tile
    const int t = ntile == 2 ? (warp >= 7 ? 1 : 0) : 0;
    const int acc_stride = p.n_pass > 1 ? p.pass_w : p.n_cols;
    const uint32_t s_bias_addr = smem_addr(s_bias);
    for (int64_t st = 0; st < n_steps; ++st) {
      const int64_t first = (unit0 + st * n_grid_units) * kUnit + t * kTileRows + rank * kBM + 32 * q;
      const int64_t row = first + lane;
      // G_i of the row before waiting on the accumulator (overlaps the MMA)
      uint32_t G = 0;
      if (row < p.rows) {
        if (ep.gt_mask) {
          G = __ldg(ep.gt_mask + row);
        } else if (ep.gt_off) {
          const int64_t g0 = __ldg(ep.gt_off + row), g1 = __ldg(ep.gt_off + row + 1);
          for (int64_t i = g0; i < g1; ++i) G |= label_lists(__ldg(cat + __ldg(ep.gt_lab + i)), ep.ctx.order);
        }
      }
      // per-list arg max over the list's 16-column groups, in column order (a list's columns
      // hold its labels ascending, so strict > keeps the smaller label on ties); the state
      // (list j, group g, running max) carries across column passes
      float lz[kMaxLists];
      int lc[kMaxLists];
#pragma unroll
      for (int jj = 0; jj < kMaxLists; ++jj) {
        lz[jj] = -CUDART_INF_F;
        lc[jj] = -1;
      }
      // 16-column groups k = 0 .. n_groups-1 run over the lists back to back (each list padded
      // to 16 columns); j = list of the current group, jend = its first group past the list
      int k = 0, j = 0;
      while (j < D && p.list_nch[j] == 0) ++j;
      int jend = j < D ? (p.list_col0[j] >> 4) + p.list_nch[j] : 0;
      const int n_groups = (p.probe & 1) ? 0 : p.n_groups;
      float run_z = -CUDART_INF_F;
      int run_c = -1;
      for (int ps = 0; ps < p.n_pass; ++ps) {
        const int c_lo = p.n_pass > 1 ? ps * p.pass_w : 0;
        const int c_hi = p.n_pass > 1 ? c_lo + p.pass_w : p.n_cols;
        unsigned long long* tr = (ps == 0 && lane == 0 && (warp == 2 || warp == 7)) ? trace_slot(p, st) : nullptr;
        if (tr && warp == 2) tr[5] = tnow();
        mbar_wait(tfull + b, tph[b]);
        if (tr) tr[warp == 2 ? 6 : 11] = tnow();
        tph[b] ^= 1u;
        tc_fence_after();
        // column c of this pass lives at acc + c - c_lo
        const uint32_t acc = tmem_base + lane_base +
                             static_cast<uint32_t>(p.n_pass > 1 ? b * acc_stride : (b + t) * p.n_cols) -
                             static_cast<uint32_t>(c_lo);
        const int khi = min(c_hi >> 4, n_groups);
        // rounds of two groups (one 32-column TMEM load); the next round's load is in flight
        // while this one is reduced (tcgen05.wait::ld waits for every outstanding load)
        uint32_t v[32], vn[32];
        const bool no_ld = (p.probe & 32) != 0, no_red = (p.probe & 16) != 0;  // drain probes
        if (no_ld) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = vn[i] = 0u;
        }
        if (k < khi && !no_ld) {
          if (k + 1 < khi) tmem_ld32(acc + 16 * k, v);
          else tmem_ld16(acc + 16 * k, *reinterpret_cast<uint32_t(*)[16]>(v));
          tmem_wait_ld32(v);
        }
        while (k < khi) {
          const int kn = k + 2;
          if (kn < khi && !no_ld) {
            if (kn + 1 < khi) tmem_ld32(acc + 16 * kn, vn);
            else tmem_ld16(acc + 16 * kn, *reinterpret_cast<uint32_t(*)[16]>(vn));
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int kg = k + h;
            if (kg < khi) {  // warp-uniform
              while (kg >= jend) {  // list j done (lists past it may be empty)
#pragma unroll
                for (int jj = 0; jj < kMaxLists; ++jj)
                  if (jj == j) {
                    lz[jj] = run_z;
                    lc[jj] = run_c;
                  }
                run_z = -CUDART_INF_F;
                run_c = -1;
                ++j;
                jend = j < D ? (p.list_col0[j] >> 4) + p.list_nch[j] : 0x7FFFFFFF;
              }
              const int col = 16 * kg;
              if (no_red) {  // probe: keep only a dependency on the loaded values
                run_z = fmaxf(run_z, __uint_as_float(v[16 * h]));
                continue;
              }
              float z[16];
              // bias: shared-space 16-B loads (a generic pointer compiled to LD.E.128)
              const uint32_t b_addr = s_bias_addr + 4u * static_cast<uint32_t>(col);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                float bb[4];
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(bb[0]), "=f"(bb[1]), "=f"(bb[2]), "=f"(bb[3])
                             : "r"(b_addr + 16u * i));
                z[4 * i + 0] = __uint_as_float(v[16 * h + 4 * i + 0]) + bb[0];
                z[4 * i + 1] = __uint_as_float(v[16 * h + 4 * i + 1]) + bb[1];
                z[4 * i + 2] = __uint_as_float(v[16 * h + 4 * i + 2]) + bb[2];
                z[4 * i + 3] = __uint_as_float(v[16 * h + 4 * i + 3]) + bb[3];
              }
              float zc;
              int ic;
              argmax16(z, zc, ic);
              if (zc > run_z) {  // strict: an earlier group (smaller labels) keeps ties
                run_z = zc;
                run_c = col + ic;
              }
            }
          }
          k = min(kn, khi);
          if (k < khi && !no_ld) {
            tmem_wait_ld32(vn);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = vn[i];
          }
        }
        if (ps + 1 == p.n_pass && j < D) {  // the last list
#pragma unroll
          for (int jj = 0; jj < kMaxLists; ++jj)
            if (jj == j) {
              lz[jj] = run_z;
              lc[jj] = run_c;
            }
        }
        tc_fence_before();
        __syncwarp();
        if (tr) tr[warp == 2 ? 7 : 12] = tnow();
        if (lane == 0) {  // the MMA may overwrite this accumulator
          if (rank == 0) mbar_arrive(tempty + b);
          else mbar_arrive_cl(tempty_l + 8u * b);
        }
        if (p.acc_bufs == 2) b ^= 1;
      }
      const int64_t nrow = p.rows - first;
      if (nrow <= 0) continue;  // warp-uniform
      rb.G = G;
      rb.app = 0;
      rb.row = row;
      rb.n = nrow < 32 ? static_cast<int>(nrow) : 32;
      if (p.pat == 0) {
        // split maxima over the list winners: P⁺ over lists in G_i, P⁻ over the rest (A8)
        float zp = -CUDART_INF_F, zm = -CUDART_INF_F;
        uint32_t kp = kNone, km = kNone;
#pragma unroll
        for (int jj = 0; jj < kMaxLists; ++jj) {
          if (lc[jj] >= 0) {
            const uint32_t key = s_keys[lc[jj]];
            if ((G >> jj) & 1u) {
              if (beats(lz[jj], key, zp, kp)) { zp = lz[jj]; kp = key; }
            } else {
              if (beats(lz[jj], key, zm, km)) { zm = lz[jj]; km = key; }
            }
          }
        }
        rb.zp = zp; rb.kp = kp; rb.zm = zm; rb.km = km;
        finish_batch(ep, rb, nullptr, lane);
        if (warp == 2 && lane == 0)
          if (unsigned long long* tr = trace_slot(p, st)) tr[8] = tnow();
      } else {
        // application-choice order / Multi-Select: the list maxima P_j themselves
        float zj[8];
        uint32_t kj[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          zj[jj] = lz[jj];
          kj[jj] = lc[jj] >= 0 ? s_keys[lc[jj]] : kNone;
        }
        finish_lists_core(ep, rb, zj, kj, nullptr, lane);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // neither CTA leaves while the other may still signal it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kMaxCols)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kMaxCols)
                   : "memory");
  }
}

// Compiled head, k-block major: Wm[kb][j][0..63] = W[label_j][64 kb .. 64 kb + 63] (zeros past
// d and for padding columns), so the W_𝕎 slice of one k-block is one contiguous n_cols x 128 B
// run: every CTA reads the same k-block at about the same time, and a contiguous block spreads
// over all L2 slices where a strided one (4 KB apart) piles onto a few.
__global__ void head_gather_kernel(const uint16_t* W, int64_t ldw, int64_t d, int32_t n_kb, int32_t n,
                                   const float* bias, const int32_t* col_label, uint16_t* Wm, float* bias_m) {
  const int j = blockIdx.x;
  const int32_t c = col_label[j];
  for (int64_t i = threadIdx.x; i < static_cast<int64_t>(n_kb) * 64; i += blockDim.x) {
    const int64_t kb = i >> 6, k = i & 63;
    Wm[(kb * n + j) * 64 + k] = (c >= 0 && i < d) ? W[c * ldw + i] : uint16_t(0);
  }
  if (threadIdx.x == 0) bias_m[j] = c < 0 ? -CUDART_INF_F : (bias ? bias[c] : 0.f);
}

}  // namespace
}  // namespace sc

// ------------------------------------------------------------------ host

struct sc_head_s {
  int device = 0;
  int64_t d = 0, d_pad = 0;
  int32_t n_mapped = 0, n_cols = 0, chunk = 0, n_chunks = 0;
  int32_t n_lists = 0;
  int32_t n_pass = 1, pass_w = 0;  // column passes (n_cols > 512)
  int32_t order = 0;
  int32_t list_col0[sc::kMaxLists] = {}, list_nch[sc::kMaxLists] = {};
  uint16_t* Wm = nullptr;  // [n_kb][n_cols][64]
  float* bias = nullptr;   // [n_cols]
  uint32_t* keys = nullptr;
  int32_t* col_label = nullptr;
  bool pair_ok = false;    // CTA pairs possible: half a chunk per CTA is a whole number of 8-row swizzle atoms
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

// 3-D bf16 tensor map over row-major x [rows][ld] (d % 64 == 0) viewed as {64, rows, d/64}:
// box {64, 128, kbs}, 128-B swizzle -> kbs [128 x 64] K-major tiles back to back.
bool make_map3(CUtensorMap* m, const void* base, int64_t d, int64_t rows, int64_t ld, int kbs) {
  EncodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(sc::kBK), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(d / sc::kBK)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(sc::kBK) * 2};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(sc::kBK), static_cast<cuuint32_t>(sc::kBM),
                             static_cast<cuuint32_t>(kbs)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr size_t kHeadSmemMax = 227 * 1024;

// One CTA per SM; CTA pairs (cta_group::2) with SC_HEAD_CLUSTER=2 when the pairs cover
// >= 90 % of the SMs.  Memoised: the occupancy query costs more
// than a small launch.
struct HeadLaunch {
  bool pair = false;
  int units = 0;  // co-resident CTAs (single) or pairs
};

HeadLaunch pick_launch(size_t smem, int sms, int64_t n_tiles, bool prefer_pair) {
  int forced = 0;
  if (const char* e = std::getenv("SC_HEAD_CLUSTER")) forced = std::atoi(e);
  static std::mutex mu;
  static std::vector<std::pair<std::array<int64_t, 3>, int>> memo;  // (smem, sms, 0) -> pairs
  int pairs = -1;
  {
    const std::array<int64_t, 3> key = {static_cast<int64_t>(smem), sms, 0};
    std::lock_guard<std::mutex> lock(mu);
    for (auto& kv : memo)
      if (kv.first == key) pairs = kv.second;
    if (pairs < 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(2 * (sms / 2)));
      cfg.blockDim = dim3(sc::kHeadThreads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, sc::head_kernel<true>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
      }
      pairs = n;
      memo.emplace_back(key, pairs);
    }
  }
  HeadLaunch hl;
  // CTA pairs with two row tiles per CTA are the default where the pairs cover >= 90 % of the
  // SMs (B200, cfg2: d = 2048 0.800 vs 0.839 ms, d = 1024 0.434 vs 0.444 ms against lone CTAs);
  // pairs with one tile (double-buffered accumulators, but each MMA feeds 128 rows per CTA)
  // are slower (0.91 ms) and opt-in.  SC_HEAD_CLUSTER=1 / 2 forces lone CTAs / pairs.
  const bool pair_ok = pairs >= 1 && (forced == 2 || 2 * pairs * 10 >= sms * 9);
  if ((forced == 2 || (forced == 0 && prefer_pair)) && pair_ok && n_tiles >= 2) {
    hl.pair = true;
    hl.units = pairs;
  } else {
    hl.units = sms;
  }
  return hl;
}

}  // namespace

extern "C" {

sc_status sc_head_load(sc_context ctx, const uint16_t* weight, int64_t ldw, int64_t d, const float* bias,
                       sc_stream stream, sc_head* out) {
  if (!ctx || !weight || !out) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_load: NULL argument");
  *out = nullptr;
  if (d < 1 || ldw < d) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_load: need d >= 1 and ldw >= d");
  if (ctx->n_apps != 1) return sc::set_error(SC_ERR_UNSUPPORTED, "sc_head_load: one application only");
  if (d > (int64_t(1) << 31) - sc::kBK) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_load: d too large");
  const int32_t nm = ctx->n_mapped[0];
  const int32_t D = ctx->nlists[0];
  // mapped labels of the app (sorted by id), grouped by list, each list padded to 16 columns
  std::vector<uint32_t> ent(std::max(nm, 1));
  cudaError_t e = cudaMemcpy(ent.data(), ctx->d_ent, static_cast<size_t>(nm) * 4, cudaMemcpyDeviceToHost);
  if (e) return sc::set_error(SC_ERR_CUDA, "sc_head_load: %s", cudaGetErrorString(e));
  std::vector<int32_t> col_label;
  std::vector<uint32_t> keys;
  sc_head h = new sc_head_s;
  h->n_lists = D;
  h->order = ctx->order;
  // list j's columns: its member labels ascending (Multi-Select: a label sits in every list holding it)
  for (int32_t j = 0; j < D; ++j) {
    h->list_col0[j] = static_cast<int32_t>(col_label.size());
    for (int32_t t = 0; t < nm; ++t)
      if ((sc::label_lists(static_cast<uint8_t>(ent[t] & 0xFFu), ctx->order) >> j) & 1u) {
        col_label.push_back(ctx->compact ? ctx->cols[ent[t] >> 8] : static_cast<int32_t>(ent[t] >> 8));  // W row
        keys.push_back(ent[t]);
      }
    while (col_label.size() % 16) {
      col_label.push_back(-1);
      keys.push_back(sc::kNone);
    }
    h->list_nch[j] = (static_cast<int32_t>(col_label.size()) - h->list_col0[j]) / 16;
  }
  while (col_label.size() < 32 || col_label.size() % 32) {  // W slices of 8-row multiples for q <= 4
    col_label.push_back(-1);
    keys.push_back(sc::kNone);
  }
  if (col_label.size() > static_cast<size_t>(sc::kMaxCols)) {
    // more columns than TMEM holds: equal column passes of <= 256 (a multiple of 32) each,
    // double-buffered in TMEM; the epilogue carries per-list maxima across passes
    const int32_t n0 = static_cast<int32_t>(col_label.size());
    h->n_pass = (n0 + sc::kPassCols - 1) / sc::kPassCols;
    h->pass_w = ((n0 + h->n_pass - 1) / h->n_pass + 31) / 32 * 32;
    while (static_cast<int32_t>(col_label.size()) < h->n_pass * h->pass_w) {
      col_label.push_back(-1);
      keys.push_back(sc::kNone);
    }
  }
  const int32_t n = static_cast<int32_t>(col_label.size());
  if (n > sc::kMaxHeadCols) {
    sc_head_free(h);
    return sc::set_error(SC_ERR_UNSUPPORTED,
                         "sc_head_load: |W| = %d mapped labels need %d head columns (lists padded to 16) > %d", nm, n,
                         sc::kMaxHeadCols);
  }
  h->d = d;
  h->d_pad = (d + 7) / 8 * 8;
  h->n_mapped = nm;
  h->n_cols = n;
  if (h->n_pass > 1) {  // one MMA of pass_w columns per pass
    h->chunk = h->pass_w;
    h->n_chunks = 1;
  } else if (n <= 256) {
    h->chunk = n;
    h->n_chunks = 1;
  } else {  // two MMAs of n/2 <= 256 columns
    h->chunk = n / 2;
    h->n_chunks = 2;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  e = cudaGetDevice(&h->device);
  const int32_t n_kb = static_cast<int32_t>((d + sc::kBK - 1) / sc::kBK);
  if (!e) e = cudaMalloc(&h->Wm, static_cast<size_t>(n) * n_kb * sc::kBK * 2);
  if (!e) e = cudaMalloc(&h->bias, static_cast<size_t>(n) * 4);
  if (!e) e = cudaMalloc(&h->keys, static_cast<size_t>(n) * 4);
  if (!e) e = cudaMalloc(&h->col_label, static_cast<size_t>(n) * 4);
  if (!e) e = cudaMemcpyAsync(h->keys, keys.data(), static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st);
  if (!e) e = cudaMemcpyAsync(h->col_label, col_label.data(), static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st);
  if (!e) {
    sc::head_gather_kernel<<<n, 256, 0, st>>>(weight, ldw, d, n_kb, n, bias, h->col_label, h->Wm, h->bias);
    sc::note_launch("head_gather");
    e = cudaGetLastError();
  }
  if (!e) e = cudaStreamSynchronize(st);
  if (e) {
    sc_head_free(h);
    return sc::set_error(e == cudaErrorMemoryAllocation ? SC_ERR_OOM : SC_ERR_CUDA, "sc_head_load: %s",
                         cudaGetErrorString(e));
  }
  CUtensorMap probe_map;  // the W maps are encoded per launch (their box is the launch's MMA chunk)
  h->pair_ok = (h->chunk / 2) % 8 == 0;
  if (!make_map(&probe_map, h->Wm, sc::kBK, static_cast<int64_t>(n_kb) * n, sc::kBK, h->chunk)) {
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
  cudaFree(h->col_label);
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
  if (ctx->n_apps != 1) return sc::set_error(SC_ERR_UNSUPPORTED, "sc_head_loss_fwd_bwd: one application only");
  if (ctx->order != head->order)
    return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: the head was compiled for another context");
  const sc_head_batch& b = *batch;
  if (b.rows < 0) return sc::set_error(SC_ERR_INVALID_ARG, "sc_head_loss_fwd_bwd: rows < 0");
  if (b.rows > (int64_t(1) << 31) - (int64_t(1) << 20))
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
  ep.ctx.col_label = ctx->d_col_label;  // compacted context: keys hold columns, gradients report labels
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
  p.n_kb = static_cast<int32_t>((head->d + sc::kBK - 1) / sc::kBK);
  p.n_cols = head->n_cols;
  // MMA column chunks: each its own accumulator chain (SC_HEAD_NCHUNK = 1, 2 or 4 overrides)
  {
    const int32_t cols = head->n_pass > 1 ? head->pass_w : head->n_cols;
    int nch = head->n_chunks;
    if (const char* e = std::getenv("SC_HEAD_NCHUNK")) nch = std::atoi(e);
    if (nch != 1 && nch != 2 && nch != 4) nch = head->n_chunks;
    while (nch > 1 && (cols % (nch * 16) != 0 || cols / nch > 256)) nch /= 2;
    if (cols / nch > 256) nch = 2;
    p.n_chunks = nch;
    p.chunk = cols / nch;
  }
  p.n_pass = head->n_pass;
  p.pass_w = head->pass_w;
  p.n_groups = head->n_lists > 0 ? (head->list_col0[head->n_lists - 1] >> 4) + head->list_nch[head->n_lists - 1] : 0;
  p.pat = ctx->order == SC_ORDER_API_OUTPUT ? 0 : 1;
  p.acc_bufs = (p.n_pass > 1 || 2 * head->n_cols <= sc::kMaxCols) ? 2 : 1;
  // lone CTAs: two 128-row tiles per unit share every W stage (W_𝕎, re-read from L2 for each
  // unit, moves half the bytes per row) when both accumulators fit TMEM; then single-buffered
  const char* t2env = std::getenv("SC_HEAD_T2");
  const bool t2_ok = head->n_pass == 1 && 2 * head->n_cols <= sc::kMaxCols &&
                     !(t2env && std::atoi(t2env) == 0);
  p.n_lists = head->n_lists;
  for (int j = 0; j < sc::kMaxLists; ++j) {
    p.list_col0[j] = head->list_col0[j];
    p.list_nch[j] = head->list_nch[j];
  }
  p.probe = std::getenv("SC_HEAD_PROBE") ? std::atoi(std::getenv("SC_HEAD_PROBE")) : 0;
  const char* trace_file = std::getenv("SC_HEAD_TRACE");  // experiment: per-unit timeline, see trace_slot
  const size_t trace_n = static_cast<size_t>(sc::kTraceCtas) * sc::kTraceUnits * sc::kTraceSlots;
  if (trace_file) {
    if (cudaMalloc(&p.trace, trace_n * 8) != cudaSuccess ||
        cudaMemsetAsync(p.trace, 0, trace_n * 8, static_cast<cudaStream_t>(stream)) != cudaSuccess)
      return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: trace buffer");
  }
  const int a_bytes = sc::kBM * sc::kBK * 2;
  const int tab_bytes = head->n_cols * 8;
  const int bar_bytes = 8 * (2 * 32 + 4) + 16;
  const int64_t budget = static_cast<int64_t>(kHeadSmemMax) - 1024 - tab_bytes - bar_bytes;
  const int sms = sc::device_sms();
  const int64_t n_tiles = (b.rows + sc::kBM - 1) / sc::kBM;
  // the launch shape needs the ring's smem size; the ring needs to know whether W is halved:
  // plan for the pair first (the smem size only shrinks for single CTAs' larger W stages)
  bool pair = false;
  HeadLaunch hl;
  bool x3d = false;
  size_t smem = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const bool want_pair = attempt == 0 && head->n_pass == 1;
    if (attempt == 0 && !want_pair) continue;
    // one k-block of the W rows an MMA pass reads (all n_cols, or pass_w in column passes)
    const int32_t pass_cols = p.chunk * p.n_chunks;
    p.w_stage_bytes = (want_pair ? pass_cols / 2 : pass_cols) * sc::kBK * 2;
    // two row tiles per unit share every W stage (lone CTAs by default; CTA pairs with
    // SC_HEAD_PAIR_T2=1: 512 rows per pass over W)
    // two row tiles per unit share every W stage (lone CTAs and, by default, CTA pairs: 512 rows
    // per pass over W; SC_HEAD_PAIR_T2=0 gives pairs one tile and double-buffered accumulators)
    const char* pt2 = std::getenv("SC_HEAD_PAIR_T2");
    p.tiles = (t2_ok && (!want_pair || !(pt2 && std::atoi(pt2) == 0))) ? 2 : 1;
    // x: 3-D boxes of kbs k-blocks (rows read kbs*128 B at a time) when d % 64 == 0; as many
    // x bytes in flight as fit next to >= 3 W stages (>= 2 for wide heads)
    x3d = head->d % sc::kBK == 0 && !(std::getenv("SC_HEAD_X2D"));
    int kbs_max = x3d ? 4 : 1, kbs_min = 1;
    if (const char* e = std::getenv("SC_HEAD_KBS")) kbs_min = kbs_max = std::max(1, std::atoi(e));
    int64_t best_score = -1;
    int best_kbs = 1, best_xs = 0, best_ws = 0;
    for (int tl = p.tiles; tl >= 1 && best_xs < 2; --tl) {  // two tiles per unit, else one
    p.tiles = tl;
    const int xa_bytes = tl * a_bytes;  // x bytes per k-block of a unit
    for (int kbs = kbs_min; kbs <= kbs_max; kbs *= 2) {
      if (kbs > p.n_kb && kbs > 1) break;
      for (int xs = 2; xs <= 16; ++xs) {
        const int64_t xbytes = static_cast<int64_t>(xs) * kbs * xa_bytes;
        const int64_t rest = budget - xbytes;
        if (rest < 0) break;
        const int ws = static_cast<int>(std::min<int64_t>(16, rest / p.w_stage_bytes));
        // measured (cfg2, d = 2048): 5-6 W stages next to ~96 KB of x beat deeper x rings for
        // one tile per unit; two tiles consume W half as fast per x byte
        int ws_min = p.w_stage_bytes > 32 * 1024 ? 2 : (tl == 2 ? 3 : 5);
        if (const char* e = std::getenv("SC_HEAD_WSTAGES")) ws_min = std::max(ws_min, std::atoi(e));
        if (ws < ws_min) break;
        // prefer more x bytes in flight, then longer contiguous runs, then more W stages
        const int64_t score = xbytes * 64 + kbs * 16 + ws;
        if (score > best_score) {
          best_score = score;
          best_kbs = kbs;
          best_xs = xs;
          best_ws = ws;
        }
      }
    }
    }
    if (best_xs < 2) return sc::set_error(SC_ERR_UNSUPPORTED, "sc_head_loss_fwd_bwd: head too wide for the ring");
    if (best_kbs == 1) x3d = false;
    p.kbs = best_kbs;
    p.n_xb = (p.n_kb + p.kbs - 1) / p.kbs;
    p.x_stages = best_xs;
    p.w_stages = best_ws;
    p.x_stage_bytes = p.kbs * p.tiles * a_bytes;
    p.w_ring_off = p.x_stages * p.x_stage_bytes;
    p.tab_off = p.w_ring_off + p.w_stages * p.w_stage_bytes;
    p.bar_off = (p.tab_off + tab_bytes + 7) / 8 * 8;
    smem = 1024 + p.bar_off + 8 * (2 * p.x_stages + 2 * p.w_stages + 4) + 16;
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [] {
      attr_err = cudaFuncSetAttribute(sc::head_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kHeadSmemMax));
      if (!attr_err)
        attr_err = cudaFuncSetAttribute(sc::head_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kHeadSmemMax));
    });
    if (attr_err) return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: %s", cudaGetErrorString(attr_err));
    hl = pick_launch(smem, sms, n_tiles, want_pair && p.tiles == 2);
    if (want_pair && !(hl.pair && head->pair_ok && (p.chunk / 2) % 8 == 0)) continue;  // re-plan for a lone CTA
    pair = want_pair;
    break;
  }
  if (p.tiles == 2) p.acc_bufs = 1;  // both accumulators of a unit in TMEM at once
  const int64_t unit_rows = static_cast<int64_t>(p.tiles) * (pair ? 2 : 1) * sc::kBM;
  p.n_units = (b.rows + unit_rows - 1) / unit_rows;
  CUtensorMap map_x;
  p.x3d = x3d ? 1 : 0;
  if (x3d ? !make_map3(&map_x, b.x, head->d, b.rows, b.ldx, p.kbs)
          : !make_map(&map_x, b.x, head->d, b.rows, b.ldx, sc::kBM))
    return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: cuTensorMapEncodeTiled failed");
  // W boxes: the rows of one MMA chunk (half of them per CTA of a pair)
  CUtensorMap map_w;
  if (!make_map(&map_w, head->Wm, sc::kBK, static_cast<int64_t>(p.n_kb) * head->n_cols, sc::kBK,
                pair ? p.chunk / 2 : p.chunk))
    return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: cuTensorMapEncodeTiled failed");
  const int64_t units = std::max<int64_t>(1, std::min<int64_t>(pair ? hl.units : sms, p.n_units));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t le = cudaSuccess;
  if (pair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * units));
    cfg.blockDim = dim3(sc::kHeadThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    le = cudaLaunchKernelEx(&cfg, sc::head_kernel<true>, map_x, map_w, p);
    sc::note_launch("head_tcgen05_pair");
  } else {
    sc::head_kernel<false><<<static_cast<unsigned>(units), sc::kHeadThreads, smem, st>>>(map_x, map_w, p);
    sc::note_launch("head_tcgen05");
  }
  if (le) return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: %s", cudaGetErrorString(le));
  if (cudaError_t e2 = cudaGetLastError())
    return sc::set_error(SC_ERR_CUDA, "sc_head_loss_fwd_bwd: %s", cudaGetErrorString(e2));
  if (trace_file) {  // experiment only: synchronous, appends one binary record per launch
    std::vector<unsigned long long> h(trace_n);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), p.trace, trace_n * 8, cudaMemcpyDeviceToHost);
    cudaFree(p.trace);
    if (FILE* f = std::fopen(trace_file, "ab")) {
      std::fwrite(h.data(), 8, trace_n, f);
      std::fclose(f);
    }
  }
  return SC_OK;
}

}  // extern "C"
