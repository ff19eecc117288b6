/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's DeAR hot path
 * (see dear_oracle.h for the parity status and who may call this).
 * Compiled with -ffp-contract=off so every a*b+c is two rounded operations,
 * as in the reference's Eigen expressions. */
#include "dear_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG --
 * std::mt19937_64 (the standard's parameters) and libstdc++'s
 * generate_canonical<double, 53> for a 64-bit engine: one draw,
 * (double)x / 2^64, then uniform_real_distribution(a, b) = u * (b - a) + a. */
#define MT_N 312
#define MT_M 156
void or_mt64_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = MT_N;
}

uint64_t or_mt64_next(or_mt64* g) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (g->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      const uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % MT_N] & lower);
      uint64_t v = g->mt[(i + MT_M) % MT_N] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

double or_uniform_pm1(or_mt64* g) {
  double u = (double)or_mt64_next(g) / 18446744073709551616.0;
  if (u >= 1.0) u = nextafter(1.0, 0.0);
  return u * 2.0 + -1.0;
}

void or_random_vectors(int P, int64_t d, uint64_t seed, double* out) {
  or_mt64 g;
  or_mt64_seed(&g, seed);
  for (int64_t i = 0; i < (int64_t)P * d; ++i) out[i] = or_uniform_pm1(&g);
}

/* The same draws rounded to fp32 (= or_random_vectors then a cast), without
 * the fp64 array: bench-scale parity inputs (BERT-L: 336M per rank). */
void or_random_vectors_f32(int P, int64_t d, uint64_t seed, float* out) {
  or_mt64 g;
  or_mt64_seed(&g, seed);
  for (int64_t i = 0; i < (int64_t)P * d; ++i) out[i] = (float)or_uniform_pm1(&g);
}

/* -------------------------------------------------------------- presets --
 * model.cpp:80-86 (tensor counts and totals), :90-98 (spread_uniform: first
 * total%count shares get +1), :138-152 (imbalanced: 80% of the parameters in
 * the last max(1, round(0.2 n)) tensors). */
static void spread_uniform(int64_t* out, int64_t count, int64_t total) {
  if (count <= 0) return;
  const int64_t base = total / count, extra = total % count;
  for (int64_t i = 0; i < count; ++i) out[i] = base + (i < extra ? 1 : 0);
}

int or_preset_params(const char* name, int profile, int64_t* out, int cap) {
  static const struct {
    const char* name;
    int tensors;
    int64_t params;
  } presets[] = {
      {"resnet50", 161, 25600000},   {"densenet201", 604, 20000000},
      {"inceptionv4", 449, 42700000}, {"bert_base", 206, 110100000},
      {"bert_large", 398, 336200000},
  };
  for (unsigned k = 0; k < sizeof(presets) / sizeof(presets[0]); ++k) {
    if (strcmp(name, presets[k].name) != 0) continue;
    const int n = presets[k].tensors;
    if (n > cap) return -1;
    if (profile == 0) {
      spread_uniform(out, n, presets[k].params);
    } else {
      int64_t tail = llround(0.2 * (double)n);
      if (tail < 1) tail = 1;
      const int64_t head = n - tail;
      const int64_t tail_params =
          head == 0 ? presets[k].params : llround(0.8 * (double)presets[k].params);
      spread_uniform(out, head, presets[k].params - tail_params);
      spread_uniform(out + head, tail, tail_params);
    }
    return n;
  }
  return -1;
}

/* --------------------------------------------------------- fusion plan --
 * build_fusion_plan (fusion.cpp:29-57): walk from layer L down; layer l joins
 * the open group while acc + bytes(l) <= buffer, otherwise the open group
 * {l+1..high} closes. per_layer_plan (fusion.cpp:59-70) when buffer == 0. */
int or_build_fusion_plan(const int64_t* layer_bytes, int L, int64_t buffer_bytes,
                         int32_t* low, int32_t* high) {
  if (L < 1 || buffer_bytes < 0) return -1;
  for (int i = 0; i < L; ++i)
    if (layer_bytes[i] < 0) return -1;
  int n = 0;
  if (buffer_bytes == 0) {
    for (int l = L; l >= 1; --l, ++n) low[n] = high[n] = l;
    return n;
  }
  int hi = L;
  int64_t acc = layer_bytes[L - 1];
  for (int l = L - 1; l >= 1; --l) {
    const int64_t next = layer_bytes[l - 1];
    if (acc + next <= buffer_bytes) {
      acc += next;
    } else {
      low[n] = l + 1;
      high[n] = hi;
      ++n;
      hi = l;
      acc = next;
    }
  }
  low[n] = 1;
  high[n] = hi;
  return n + 1;
}

/* ------------------------------------------------------- chunk layout --
 * chunk_ranges (collective.cpp:39-57): chunk c has d/P elements, +1 for the
 * first d%P chunks; contiguous. Owner (collective.cpp:94): (c-1) mod P. */
int or_chunk_ranges(int64_t d, int P, int64_t* begin) {
  if (P < 1 || d < 0) return -1;
  const int64_t base = d / P, extra = d % P;
  int64_t at = 0;
  for (int c = 0; c < P; ++c) {
    begin[c] = at;
    at += base + (c < extra ? 1 : 0);
  }
  begin[P] = at;
  return 0;
}

int or_chunk_owner(int c, int P) { return ((c - 1) % P + P) % P; }

/* ------------------------------------------------ ring reduce-scatter --
 * collective.cpp:70-90: in round r worker w adds the chunk (w-1-r) mod P it
 * received from w-1 to its own copy. Chunk c therefore starts on worker c and
 * picks up workers c+1, c+2, ..., c-1 in that order: a left fold. (Each add is
 * commutative in IEEE arithmetic, so state+inbox vs inbox+state is moot.) */
void or_ring_reduce_scatter(int P, int64_t d, const double* in, double* out) {
  int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P + 1));
  or_chunk_ranges(d, P, b);
  for (int c = 0; c < P; ++c) {
    for (int64_t i = b[c]; i < b[c + 1]; ++i) {
      double acc = in[(int64_t)c * d + i];
      for (int k = 1; k < P; ++k) acc += in[(int64_t)((c + k) % P) * d + i];
      out[i] = acc;
    }
  }
  free(b);
}

void or_all_reduce_average(int P, int64_t d, const double* in, double* out) {
  or_ring_reduce_scatter(P, d, in, out);
  const double inv_p = 1.0 / (double)P; /* collective.cpp:161 */
  for (int64_t i = 0; i < d; ++i) out[i] *= inv_p;
}

int or_sgd_step(int P, int64_t d, double lr, double* w, const double* grads) {
  if (P < 1 || d < 0) return -1;
  double* mean = (double*)malloc(sizeof(double) * (size_t)(d > 0 ? d : 1));
  or_all_reduce_average(P, d, grads, mean);
  for (int64_t i = 0; i < d; ++i) w[i] -= lr * mean[i]; /* collective.cpp:190-192 */
  free(mean);
  return 0;
}

/* UNPINNED: torch.optim.SGD's per-element update on the averaged gradient. */
int or_sgd_step_momentum(int P, int64_t d, double lr, double momentum, double dampening,
                         double weight_decay, int nesterov, double* w, double* buf,
                         int* has_buf, const double* grads) {
  if (P < 1 || d < 0) return -1;
  double* g = (double*)malloc(sizeof(double) * (size_t)(d > 0 ? d : 1));
  or_all_reduce_average(P, d, grads, g);
  for (int64_t i = 0; i < d; ++i) {
    double dp = g[i];
    if (weight_decay != 0.0) dp = dp + weight_decay * w[i];
    if (momentum != 0.0) {
      if (!*has_buf)
        buf[i] = dp;
      else
        buf[i] = buf[i] * momentum + (1.0 - dampening) * dp;
      dp = nesterov ? dp + momentum * buf[i] : buf[i];
    }
    w[i] = w[i] - lr * dp;
  }
  if (momentum != 0.0) *has_buf = 1;
  free(g);
  return 0;
}

/* ----------------------------------------------------------- fp32 --- */
void or_ring_reduce_scatter_f32(int P, int64_t d, const float* in, float* out) {
  int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P + 1));
  or_chunk_ranges(d, P, b);
  for (int c = 0; c < P; ++c) {
    for (int64_t i = b[c]; i < b[c + 1]; ++i) {
      float acc = in[(int64_t)c * d + i];
      for (int k = 1; k < P; ++k) acc += in[(int64_t)((c + k) % P) * d + i];
      out[i] = acc;
    }
  }
  free(b);
}

int or_sgd_step_f32(int P, int64_t d, float lr, float momentum, float dampening,
                    float weight_decay, int nesterov, float* w, float* buf, int* has_buf,
                    const float* grads, int prescale) {
  if (P < 1 || d < 0) return -1;
  const float inv_p = 1.0f / (float)P;
  float* src = (float*)malloc(sizeof(float) * (size_t)((int64_t)P * d + 1));
  float* g = (float*)malloc(sizeof(float) * (size_t)(d + 1));
  for (int64_t i = 0; i < (int64_t)P * d; ++i) src[i] = prescale ? grads[i] * inv_p : grads[i];
  or_ring_reduce_scatter_f32(P, d, src, g);
  for (int64_t i = 0; i < d; ++i) {
    float dp = prescale ? g[i] : g[i] * inv_p;
    if (weight_decay != 0.0f) dp = dp + weight_decay * w[i];
    if (momentum != 0.0f) {
      if (!*has_buf)
        buf[i] = dp;
      else
        buf[i] = buf[i] * momentum + (1.0f - dampening) * dp;
      dp = nesterov ? dp + momentum * buf[i] : buf[i];
    }
    w[i] = w[i] - lr * dp;
  }
  if (momentum != 0.0f) *has_buf = 1;
  free(src);
  free(g);
  return 0;
}
