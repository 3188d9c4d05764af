/* synth.h — seeded synthetic inputs for the software-context hot path.
 *
 * Harness module, NOT part of the method: it holds none of the method's
 * arithmetic (no decision, no category compile, no loss).  It is the one
 * module both sides may use: tests and bench.py feed identical inputs to the
 * CUDA path (libsc) and to the CPU oracle (oracle/).  Two independent
 * implementations of the same integer counter-hash exist — synth_host.c (C)
 * and synth_cuda.cu (CUDA) — and tests check they agree bit for bit.
 *
 * Recipe (DESIGN.md §"Input recipe"); the paper gives no
 * logit or label distributions, only the Heapsortcypher lists,
 * the 9605-label Open Images label space and "applications
 * typically heavily cluster on a small subset of labels":
 *
 *   h(seed, stream, a, b) = mix(mix(mix(seed ^ stream<<56) ^ a) ^ b),
 *   mix = SplitMix64 (add golden gamma, xor-shift-multiply finaliser).
 *
 *   app(i)   layout 0: (i / rows_per_app) % n_apps; layout 1: i % n_apps
 *   n_gt(i)  = 1 + h(seed, S_NGT, i, 0) % 4                      (mean 2.5)
 *   label t  : u = h(seed, S_GTLAB, i, t); if t == 0 and u>>63 and |Wa|>0:
 *              Wa[(u & 0xffffffff) % |Wa|] else (u & 0xffffffff) % C
 *              (Wa = sorted mapped-label set of app(i); duplicates allowed)
 *   z(i,c)   f32 : -12 + (h(seed,S_LOGIT,i,c) & 0xffff) * 2^-12   in [-12, 4)
 *            bf16: -8  + (h(seed,S_LOGIT,i,c) & 0xff) / 16         in [-8, 8)
 *            +8 if c in gt(i) and h(seed,S_TP,i,c) % 10 < 8          (true positive)
 *            +8 if c in Wa \ gt(i) and h(seed,S_FP,i,c) % 100 < 5     (false positive)
 *            columns C..ld-1 (row padding) are NaN, so any read of them shows.
 *   All values are exact in the storage type.
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SYNTH_S_NGT = 1, SYNTH_S_GTLAB = 2, SYNTH_S_LOGIT = 3, SYNTH_S_TP = 4,
       SYNTH_S_FP = 5, SYNTH_S_CTX = 7 };

typedef struct {
  uint64_t seed;
  int32_t  C;
  int32_t  n_apps;
  int32_t  layout;          /* 0: contiguous rows per app, 1: app = row % n_apps */
  int64_t  rows_per_app;    /* layout 0 */
  const uint8_t*  mapped;   /* [n_apps*C] 1 if label is in some list of the app */
  const int64_t*  wset_off; /* [n_apps+1] CSR offsets into wset_lab          */
  const int32_t*  wset_lab; /* sorted mapped labels per app                   */
} synth_spec;               /* pointers are host pointers for synth_host, device pointers for synth_cuda */

/* ---- host implementation (synth_host.c) ---- */
uint64_t synth_hash(uint64_t seed, uint32_t stream, uint64_t a, uint64_t b);
/* Fisher-Yates permutation of [0,C) drawn from h(seed, S_CTX, i, app). */
void synth_perm(uint64_t seed, int32_t app, int32_t C, int32_t* perm);
/* rows [row0, row0+nrows): app ids (uint16), GT counts. */
void synth_host_apps(const synth_spec* s, int64_t row0, int64_t nrows, uint16_t* app);
void synth_host_gt_count(const synth_spec* s, int64_t row0, int64_t nrows, int64_t* cnt);
/* off: CSR offsets [nrows+1] for these rows (absolute indices into lab, any base);
   fills lab[off[j]..off[j+1]) for row row0+j. */
void synth_host_gt_fill(const synth_spec* s, int64_t row0, int64_t nrows,
                        const int64_t* off, int32_t* lab);
/* logits rows [row0,row0+nrows) into out[nrows*ld]; dtype 0 = f32, 1 = bf16 (uint16 bits). */
void synth_host_logits(const synth_spec* s, int64_t row0, int64_t nrows, int64_t ld,
                       int32_t dtype, const int64_t* off, const int32_t* lab, void* out);

/* ---- CUDA implementation (synth_cuda.cu); all array pointers are device pointers ---- */
int synth_cuda_apps(const synth_spec* s, int64_t row0, int64_t nrows, uint16_t* app, void* stream);
int synth_cuda_gt_count(const synth_spec* s, int64_t row0, int64_t nrows, int64_t* cnt, void* stream);
int synth_cuda_gt_fill(const synth_spec* s, int64_t row0, int64_t nrows,
                       const int64_t* off, int32_t* lab, void* stream);
int synth_cuda_logits(const synth_spec* s, int64_t row0, int64_t nrows, int64_t ld,
                      int32_t dtype, const int64_t* off, const int32_t* lab, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
