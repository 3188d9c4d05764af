/* synth_host.c — host (C) implementation of the seeded input recipe in synth.h.
 * Harness only: no decision / loss arithmetic lives here. */
#include "synth.h"
#include <string.h>

static uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t synth_hash(uint64_t seed, uint32_t stream, uint64_t a, uint64_t b) {
  return mix64(mix64(mix64(seed ^ ((uint64_t)stream << 56)) ^ a) ^ b);
}

void synth_perm(uint64_t seed, int32_t app, int32_t C, int32_t* perm) {
  for (int32_t i = 0; i < C; ++i) perm[i] = i;
  for (int32_t i = C - 1; i > 0; --i) {
    uint64_t u = synth_hash(seed, SYNTH_S_CTX, (uint64_t)i, (uint64_t)app);
    int32_t j = (int32_t)(u % (uint64_t)(i + 1));
    int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
}

static int32_t app_of(const synth_spec* s, int64_t row) {
  if (s->n_apps <= 1) return 0;
  if (s->layout == 1) return (int32_t)(row % s->n_apps);
  return (int32_t)((row / s->rows_per_app) % s->n_apps);
}

void synth_host_apps(const synth_spec* s, int64_t row0, int64_t nrows, uint16_t* app) {
  for (int64_t j = 0; j < nrows; ++j) app[j] = (uint16_t)app_of(s, row0 + j);
}

void synth_host_gt_count(const synth_spec* s, int64_t row0, int64_t nrows, int64_t* cnt) {
  for (int64_t j = 0; j < nrows; ++j)
    cnt[j] = 1 + (int64_t)(synth_hash(s->seed, SYNTH_S_NGT, (uint64_t)(row0 + j), 0) % 4);
}

void synth_host_gt_fill(const synth_spec* s, int64_t row0, int64_t nrows,
                        const int64_t* off, int32_t* lab) {
  for (int64_t j = 0; j < nrows; ++j) {
    int64_t row = row0 + j;
    int32_t a = app_of(s, row);
    int64_t wn = s->wset_off[a + 1] - s->wset_off[a];
    int64_t n = off[j + 1] - off[j];
    for (int64_t t = 0; t < n; ++t) {
      uint64_t u = synth_hash(s->seed, SYNTH_S_GTLAB, (uint64_t)row, (uint64_t)t);
      uint64_t lo = u & 0xffffffffull;
      int32_t c;
      if (t == 0 && (u >> 63) && wn > 0) c = s->wset_lab[s->wset_off[a] + (int64_t)(lo % (uint64_t)wn)];
      else c = (int32_t)(lo % (uint64_t)s->C);
      lab[off[j] + t] = c;
    }
  }
}

static uint16_t f32_to_bf16_bits_exact(float f) {  /* inputs are bf16-exact by construction */
  uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16);
}

void synth_host_logits(const synth_spec* s, int64_t row0, int64_t nrows, int64_t ld,
                       int32_t dtype, const int64_t* off, const int32_t* lab, void* out) {
  const uint32_t qnan = 0x7FC00000u;
  float nanf; memcpy(&nanf, &qnan, 4);
  for (int64_t j = 0; j < nrows; ++j) {
    int64_t row = row0 + j;
    int32_t a = app_of(s, row);
    const int32_t* g = lab + off[j];
    int64_t ng = off[j + 1] - off[j];
    for (int64_t c = 0; c < ld; ++c) {
      float z;
      if (c >= s->C) {
        z = nanf;
      } else {
        uint64_t h = synth_hash(s->seed, SYNTH_S_LOGIT, (uint64_t)row, (uint64_t)c);
        if (dtype == 0) z = -12.0f + (float)(h & 0xffff) * (1.0f / 4096.0f);
        else            z = -8.0f + (float)(h & 0xff) * (1.0f / 16.0f);
        int in_gt = 0;
        for (int64_t t = 0; t < ng; ++t) if (g[t] == c) { in_gt = 1; break; }
        if (in_gt) {
          if (synth_hash(s->seed, SYNTH_S_TP, (uint64_t)row, (uint64_t)c) % 10 < 8) z += 8.0f;
        } else if (s->mapped[(int64_t)a * s->C + c]) {
          if (synth_hash(s->seed, SYNTH_S_FP, (uint64_t)row, (uint64_t)c) % 100 < 5) z += 8.0f;
        }
      }
      if (dtype == 0) ((float*)out)[j * ld + c] = z;
      else ((uint16_t*)out)[j * ld + c] = f32_to_bf16_bits_exact(z);
    }
  }
}
