/* synth.c — host implementation of the synthetic input generator described in synth.h.
 * Input generation only; no method arithmetic. The fp32->fp16 RNE conversion here is the generator's own. */
#include "synth.h"
#include <string.h>

static uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static uint64_t stream_of(uint64_t seed, uint64_t tensor_id) {
  return mix64(mix64(seed) ^ (tensor_id * 0xD1B54A32D192ED03ull));
}
static uint64_t u_at(uint64_t stream, uint64_t i) { return mix64(stream + (i + 1) * 0x9E3779B97F4A7C15ull); }
static int32_t v_of(uint64_t u) {
  return (int32_t)((u & 0xFFFF) + ((u >> 16) & 0xFFFF) + ((u >> 32) & 0xFFFF) + (u >> 48)) - 131070;
}
/* fp32 -> fp16 round-to-nearest-even, all cases. */
static uint16_t f32_to_f16(float f) {
  uint32_t x; memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t ex = (x >> 23) & 0xFF, man = x & 0x7FFFFFu;
  if (ex == 0xFF) return (uint16_t)(sign | 0x7C00u | (man ? 0x200u : 0));
  int e = (int)ex - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7C00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    man |= 0x800000u;
    int sh = 14 - e;                       /* 24-bit significand -> subnormal half */
    uint32_t q = man >> sh, rem = man & ((1u << sh) - 1), half = 1u << (sh - 1);
    if (rem > half || (rem == half && (q & 1))) q++;
    return (uint16_t)(sign | q);
  }
  uint32_t q = ((uint32_t)e << 10) | (man >> 13), rem = man & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (q & 1))) q++;   /* carry into exponent is correct (may give inf) */
  return (uint16_t)(sign | q);
}
static float pow2f(int e) { float r = 1.f; if (e >= 0) while (e--) r *= 2.f; else while (e++) r *= 0.5f; return r; }

uint16_t synth_value_host(uint64_t seed, uint64_t tensor_id, int kind, int rows, int cols, int r, int c) {
  uint64_t st = stream_of(seed, tensor_id);
  uint64_t idx = (uint64_t)r * (uint64_t)cols + (uint64_t)c;
  float v = (float)v_of(u_at(st, idx));
  int e;
  if (kind == SYNTH_WEIGHT) {
    uint64_t st2 = stream_of(seed, tensor_id ^ 0x5A5A5A5A00000000ull);
    uint64_t g = (uint64_t)(r / 128) * (uint64_t)cols + (uint64_t)c;
    int out = (u_at(st2, g) % SYNTH_W_OUTLIER_MOD) == 0;
    e = -SYNTH_W_SHIFT + (out ? SYNTH_W_OUTLIER_LOG2 : 0);
  } else {
    uint64_t st3 = stream_of(seed, tensor_id ^ 0xA5A5A5A500000000ull);
    int out = 0;
    for (int j = 0; j < SYNTH_X_OUTLIER_N; ++j) if ((int)(u_at(st3, (uint64_t)j) % (uint64_t)cols) == c) out = 1;
    e = -SYNTH_X_SHIFT + (out ? SYNTH_X_OUTLIER_LOG2 : 0);
  }
  (void)rows;
  return f32_to_f16(v * pow2f(e));
}

int synth_fill_host(uint64_t seed, uint64_t tensor_id, int kind, int rows, int cols, uint16_t* out) {
  if (!out || rows < 0 || cols <= 0 || (kind != SYNTH_WEIGHT && kind != SYNTH_ACT)) return -1;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) out[(size_t)r * cols + c] = synth_value_host(seed, tensor_id, kind, rows, cols, r, c);
  return 0;
}

int synth_fill_host_block(uint64_t seed, uint64_t tensor_id, int kind, int rows, int cols, int r0, int r1, int c0,
                          int c1, uint16_t* out) {
  if (!out || r0 < 0 || c0 < 0 || r1 > rows || c1 > cols || r0 > r1 || c0 > c1 || (kind != SYNTH_WEIGHT && kind != SYNTH_ACT))
    return -1;
  for (int r = r0; r < r1; ++r)
    for (int c = c0; c < c1; ++c)
      out[(size_t)(r - r0) * (c1 - c0) + (c - c0)] = synth_value_host(seed, tensor_id, kind, rows, cols, r, c);
  return 0;
}
