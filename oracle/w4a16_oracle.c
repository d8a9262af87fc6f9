/* w4a16_oracle.c — CPU oracle (TEST INFRASTRUCTURE ONLY; see w4a16_oracle.h for scope and citations).
 *
 * Plain C, written to be checked by eye against the definitions in DESIGN.md §3 / SURVEY §8(c).
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math (fp32 steps of the pack must be IEEE, RNE, unfused).
 */
#include "w4a16_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------------------------------------------------
 * IEEE binary16 conversions (reading R1). half -> wider is exact; wider -> half rounds once, to nearest
 * even, from the exact value (float -> double is exact, so float -> half is a single rounding too).
 * ---------------------------------------------------------------------------------------------------- */
double orc_half_to_double(uint16_t h) {
  int sign = (h >> 15) & 1, e = (h >> 10) & 0x1F, m = h & 0x3FF;
  double v;
  if (e == 0) v = ldexp((double)m, -24);                       /* zero / subnormal: m * 2^-24 */
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = ldexp((double)(1024 + m), e - 25);                  /* (1 + m/1024) * 2^(e-15) */
  return sign ? -v : v;
}

float orc_half_to_float(uint16_t h) { return (float)orc_half_to_double(h); }

uint16_t orc_double_to_half(double d) {
  uint16_t sign = signbit(d) ? 0x8000 : 0;
  if (isnan(d)) return (uint16_t)(sign | 0x7E00);
  double a = fabs(d);
  if (a >= 65520.0) return (uint16_t)(sign | 0x7C00);          /* half-way between 65504 and 2^16 ties to inf */
  if (a == 0.0) return sign;
  int E;
  frexp(a, &E);                                                /* a = f * 2^E, f in [0.5, 1) */
  int e = E - 1;                                               /* a in [2^e, 2^(e+1)) */
  if (e < -14) e = -14;                                        /* subnormal range: quantum 2^-24 */
  double q = ldexp(a, 10 - e);                                 /* a / quantum, exact (power-of-two scaling) */
  double r = nearbyint(q);                                     /* round to nearest, ties to even (default mode) */
  if (r < 1024.0) return (uint16_t)(sign | (uint16_t)r);      /* subnormal (or zero) */
  /* normal: r in [1024, 2048]; r == 2048 carries into the exponent automatically */
  return (uint16_t)(sign | (uint16_t)(((e + 15) << 10) + ((int)r - 1024)));
}

uint16_t orc_float_to_half(float f) { return orc_double_to_half((double)f); }

static int shape_ok(int K, int N, int group) { return K > 0 && N > 0 && group > 0 && K % group == 0; }

/* clamp to [lo, hi]; -0.0 maps to lo (+0.0) so a zero point of 0 is stored as fp16 +0 (reading R2). */
static float clampf(float x, float lo, float hi) {
  if (!(x > lo)) return lo;
  if (x > hi) return hi;
  return x;
}

/* ------------------------------------------------------------------------------------------------------
 * Quantise (GPTQ quantizer conventions). All arithmetic is fp32 (C float,
 * SSE, no contraction): readings R3 (0 representable), R4 (RNE), R5 (codes use the stored fp16 scale),
 * R15 (all-zero group -> range +-1).
 * ---------------------------------------------------------------------------------------------------- */
int orc_quantize(const uint16_t* W, int K, int N, int group, int mode, uint8_t* codes, uint16_t* scales,
                 uint16_t* zeros, int32_t* status) {
  if (!W || !codes || !scales || !shape_ok(K, N, group)) return -1;
  if (mode != ORC_ASYM && mode != ORC_SYM) return -1;
  if (mode == ORC_ASYM && !zeros) return -1;
  int st = ORC_DEV_OK;
  for (int n = 0; n < N; ++n) {
    for (int g = 0; g < K / group; ++g) {
      /* 1. range, always containing 0; non-finite weights flag the status and count as 0 */
      float wmin = 0.0f, wmax = 0.0f;
      for (int k = g * group; k < (g + 1) * group; ++k) {
        float w = orc_half_to_float(W[(size_t)k * N + n]);
        if (!isfinite(w)) { st = ORC_DEV_NONFINITE; continue; }
        if (w < wmin) wmin = w;
        if (w > wmax) wmax = w;
      }
      /* 2. scale s (fp16) and integer zero z */
      float s32, z;
      uint16_t s;
      if (mode == ORC_ASYM) {
        if (wmin == wmax) { wmin = -1.0f; wmax = 1.0f; }
        s = orc_float_to_half((wmax - wmin) / 15.0f);
        if (orc_half_to_float(s) == 0.0f) { wmin = -1.0f; wmax = 1.0f; s = orc_float_to_half((wmax - wmin) / 15.0f); }
        s32 = orc_half_to_float(s);
        z = clampf(rintf(-wmin / s32), 0.0f, 15.0f);
      } else {
        float amax = -wmin > wmax ? -wmin : wmax;
        if (amax == 0.0f) amax = 1.0f;
        s = orc_float_to_half((amax + amax) / 15.0f);
        if (orc_half_to_float(s) == 0.0f) { amax = 1.0f; s = orc_float_to_half((amax + amax) / 15.0f); }
        s32 = orc_half_to_float(s);
        z = 8.0f;
      }
      scales[(size_t)g * N + n] = s;
      if (zeros) zeros[(size_t)g * N + n] = orc_float_to_half(z);
      /* 3. codes q = clamp(rne(w / s) + z, 0, 15) */
      for (int k = g * group; k < (g + 1) * group; ++k) {
        float w = orc_half_to_float(W[(size_t)k * N + n]);
        if (!isfinite(w)) w = 0.0f;
        float q = clampf(rintf(w / s32) + z, 0.0f, 15.0f);
        codes[(size_t)k * N + n] = (uint8_t)(int)q;
      }
    }
  }
  if (status) *status = st;
  return 0;
}

/* w_hat = fp16_rne((q - z) * s): (q - z) is a small integer, the product is exact in double, so this is
 * exactly one rounding. */
static uint16_t dequant(int q, uint16_t s, const uint16_t* zeros, size_t gi, int mode) {
  double z = mode == ORC_SYM ? 8.0 : orc_half_to_double(zeros[gi]);
  return orc_double_to_half(((double)q - z) * orc_half_to_double(s));
}

int orc_dequantize(const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int K, int N, int group,
                   int mode, uint16_t* W_hat) {
  if (!codes || !scales || !W_hat || !shape_ok(K, N, group)) return -1;
  if (mode != ORC_ASYM && mode != ORC_SYM) return -1;
  if (mode == ORC_ASYM && !zeros) return -1;
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) {
      size_t gi = (size_t)(k / group) * N + n;
      W_hat[(size_t)k * N + n] = dequant(codes[(size_t)k * N + n], scales[gi], zeros, gi, mode);
    }
  return 0;
}

/* ------------------------------------------------------------------------------------------------------
 * GEMM reference: dequantise, then matmul, in fp64 with k in order 0..K-1.
 * ---------------------------------------------------------------------------------------------------- */
typedef struct {
  const uint16_t* X; const uint8_t* codes; const uint16_t* sc; const uint16_t* ze;
  int M, K, N, group, mode;
  int exact_w;                           /* 1: weight = (q - z) * s exactly (reading R22); 0: fp16_rne of it */
  const int32_t* cols;                   /* column list (NULL: all columns) */
  double* Y; int ystride;                /* Y[m*ystride + j] */
  int j0, j1;                            /* this worker's column positions [j0, j1) */
} gemm_job;

static void* gemm_worker(void* p) {
  gemm_job* a = (gemm_job*)p;
  double* wcol = (double*)malloc(sizeof(double) * (size_t)a->K);
  for (int j = a->j0; j < a->j1; ++j) {
    int n = a->cols ? a->cols[j] : j;
    for (int k = 0; k < a->K; ++k) {
      size_t gi = (size_t)(k / a->group) * a->N + n;
      if (a->exact_w) {   /* (q - z) * s: a 4-bit integer times an fp16 scale, exact in double */
        double z = a->mode == ORC_SYM ? 8.0 : orc_half_to_double(a->ze[gi]);
        wcol[k] = ((double)a->codes[(size_t)k * a->N + n] - z) * orc_half_to_double(a->sc[gi]);
      } else {
        wcol[k] = orc_half_to_double(dequant(a->codes[(size_t)k * a->N + n], a->sc[gi], a->ze, gi, a->mode));
      }
    }
    for (int m = 0; m < a->M; ++m) {
      const uint16_t* xr = a->X + (size_t)m * a->K;
      double acc = 0.0;
      for (int k = 0; k < a->K; ++k) acc += orc_half_to_double(xr[k]) * wcol[k];
      a->Y[(size_t)m * a->ystride + j] = acc;
    }
  }
  free(wcol);
  return NULL;
}

static int gemm_run(const uint16_t* X, const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int M,
                    int K, int N, int group, int mode, const int32_t* cols, int ncols, double* Y, int nthreads,
                    int exact_w) {
  if (!X || !codes || !scales || !Y || M < 0 || !shape_ok(K, N, group)) return -1;
  if (mode != ORC_ASYM && mode != ORC_SYM) return -1;
  if (mode == ORC_ASYM && !zeros) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > ncols) nthreads = ncols > 0 ? ncols : 1;
  gemm_job* jobs = (gemm_job*)calloc((size_t)nthreads, sizeof(gemm_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    gemm_job j = {X, codes, scales, zeros, M, K, N, group, mode, exact_w, cols, Y, ncols,
                  (int)((long long)ncols * t / nthreads), (int)((long long)ncols * (t + 1) / nthreads)};
    jobs[t] = j;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, gemm_worker, &jobs[t]);
  gemm_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(jobs); free(th);
  return 0;
}

int orc_gemm(const uint16_t* X, const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int M, int K,
             int N, int group, int mode, double* Y, int nthreads) {
  return gemm_run(X, codes, scales, zeros, M, K, N, group, mode, NULL, N, Y, nthreads, 0);
}

/* The same GEMM on the exact quantised weights (reading R22): W[k][n] = (q - z) * s with no fp16 rounding of
 * the product — the value the scale-after-sum kernel families compute with (they apply s to fp32 sums of
 * (q - z) x). Differs from orc_gemm by at most sum_k |x_k| * ulp16(w_hat_k) / 2. */
int orc_gemm_exact(const uint16_t* X, const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int M,
                   int K, int N, int group, int mode, double* Y, int nthreads) {
  return gemm_run(X, codes, scales, zeros, M, K, N, group, mode, NULL, N, Y, nthreads, 1);
}

int orc_gemm_cols(const uint16_t* X, const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int M,
                  int K, int N, int group, int mode, const int32_t* cols, int ncols, double* Ycols) {
  if (!cols || ncols < 0) return -1;
  for (int j = 0; j < ncols; ++j) if (cols[j] < 0 || cols[j] >= N) return -1;
  return gemm_run(X, codes, scales, zeros, M, K, N, group, mode, cols, ncols, Ycols, 1, 0);
}

/* ------------------------------------------------------------------------------------------------------
 * The ABI's packed blob (include/w4a16.h): 128x128 tiles, n-tile major then k-group; per tile 8192 code
 * bytes (row r: 64 bytes at r*64 = four 16-byte chunks, chunk p = k 32p..32p+31 stored at chunk position
 * p XOR ((r/2) % 4); word w of a chunk: k = 32p + 8w .. +7, local index i in nibble slot (i%2)*4 + i/2),
 * then per row r the fp16 scale and (ASYM) fp16 zero side by side: ASYM {s, z} at 8192 + 4r, SYM s at
 * 8192 + 2r. Integers are little-endian.
 * ---------------------------------------------------------------------------------------------------- */
static int layout_ok(int K, int N) { return K > 0 && N > 0 && K % 128 == 0 && N % 128 == 0; }
static size_t tile_bytes(int mode) { return mode == ORC_ASYM ? 8704 : 8448; }
static size_t tile_offset(int K, int mode, int k, int n) {
  return ((size_t)(n / 128) * (size_t)(K / 128) + (size_t)(k / 128)) * tile_bytes(mode);
}

int orc_nibble_slot(int i) { return (i % 2) * 4 + i / 2; }

size_t orc_packed_bytes(int K, int N, int mode) {
  if (!layout_ok(K, N)) return 0;
  return (size_t)(N / 128) * (size_t)(K / 128) * tile_bytes(mode);
}

size_t orc_code_word_offset(int K, int N, int mode, int k, int n) {
  (void)N;
  int r = n % 128, p = (k % 128) / 32, w = (k % 32) / 8;
  int chunk_pos = p ^ ((r / 2) % 4);
  return tile_offset(K, mode, k, n) + (size_t)r * 64 + (size_t)chunk_pos * 16 + (size_t)w * 4;
}

static uint32_t rd32(const uint8_t* p) { return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24; }
static void wr32(uint8_t* p, uint32_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24); }
static uint16_t rd16(const uint8_t* p) { return (uint16_t)(p[0] | p[1] << 8); }
static void wr16(uint8_t* p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }

int orc_layout_pack(const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int K, int N, int mode,
                    uint8_t* packed) {
  if (!codes || !scales || !packed || !layout_ok(K, N) || (mode != ORC_ASYM && mode != ORC_SYM)) return -1;
  if (mode == ORC_ASYM && !zeros) return -1;
  memset(packed, 0, orc_packed_bytes(K, N, mode));
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      uint8_t* w = packed + orc_code_word_offset(K, N, mode, k, n);
      wr32(w, rd32(w) | ((uint32_t)(codes[(size_t)k * N + n] & 0xF) << (4 * orc_nibble_slot(k % 8))));
    }
  for (int g = 0; g < K / 128; ++g)
    for (int n = 0; n < N; ++n) {
      uint8_t* t = packed + tile_offset(K, mode, 128 * g, n);
      if (mode == ORC_ASYM) {
        wr16(t + 8192 + 4 * (n % 128), scales[(size_t)g * N + n]);
        wr16(t + 8192 + 4 * (n % 128) + 2, zeros[(size_t)g * N + n]);
      } else {
        wr16(t + 8192 + 2 * (n % 128), scales[(size_t)g * N + n]);
      }
    }
  return 0;
}

int orc_layout_unpack(const uint8_t* packed, int K, int N, int mode, uint8_t* codes, uint16_t* scales,
                      uint16_t* zeros) {
  if (!packed || !codes || !scales || !layout_ok(K, N) || (mode != ORC_ASYM && mode != ORC_SYM)) return -1;
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      uint32_t w = rd32(packed + orc_code_word_offset(K, N, mode, k, n));
      codes[(size_t)k * N + n] = (uint8_t)((w >> (4 * orc_nibble_slot(k % 8))) & 0xF);
    }
  for (int g = 0; g < K / 128; ++g)
    for (int n = 0; n < N; ++n) {
      const uint8_t* t = packed + tile_offset(K, mode, 128 * g, n);
      if (mode == ORC_ASYM) {
        scales[(size_t)g * N + n] = rd16(t + 8192 + 4 * (n % 128));
        if (zeros) zeros[(size_t)g * N + n] = rd16(t + 8192 + 4 * (n % 128) + 2);
      } else {
        scales[(size_t)g * N + n] = rd16(t + 8192 + 2 * (n % 128));
        if (zeros) zeros[(size_t)g * N + n] = 0x4800; /* 8.0 */
      }
    }
  return 0;
}

/* ------------------------------------------------------------------------------------------------------
 * Greedy acceptance (reading R9). ok[i]: every edge on the root->i path matches the
 * target's argmax at the parent; the accepted node is the deepest ok node (ties: smallest index); the
 * bonus token is the target's argmax at that node.
 * ---------------------------------------------------------------------------------------------------- */
int orc_accept(const int32_t* tokens, const int32_t* parents, const int32_t* target_argmax, int n, int32_t* out) {
  if (!tokens || !parents || !target_argmax || !out || n < 1) return -1;
  for (int i = 0; i < n; ++i) out[3 + i] = -1;
  int bad = parents[0] != -1;
  for (int i = 1; i < n; ++i) if (parents[i] < 0 || parents[i] >= i) bad = 1;
  if (bad) { out[0] = 0; out[1] = -1; out[2] = ORC_DEV_BAD_TREE; return 0; }
  int* ok = (int*)malloc(sizeof(int) * (size_t)n);
  int* depth = (int*)malloc(sizeof(int) * (size_t)n);
  ok[0] = 1; depth[0] = 0;
  for (int i = 1; i < n; ++i) {
    int p = parents[i];
    ok[i] = ok[p] && tokens[i] == target_argmax[p];
    depth[i] = depth[p] + 1;
  }
  int best = 0;
  for (int i = 1; i < n; ++i) if (ok[i] && depth[i] > depth[best]) best = i;
  out[0] = depth[best];
  out[1] = target_argmax[best];
  out[2] = ORC_DEV_OK;
  for (int x = best; x != 0; x = parents[x]) out[3 + depth[x] - 1] = x;
  free(ok); free(depth);
  return 0;
}

/* ------------------------------------------------------------------------------------------------------
 * LM head + greedy argmax (reading R12: FP16 LM head; ties to the lowest id).
 * Straight from the definition: every logit in fp64 (products of fp16 values are exact in fp64), then a
 * left-to-right scan keeping the first maximum.
 * ---------------------------------------------------------------------------------------------------- */
typedef struct {
  const uint16_t* H; const uint16_t* W; int M, K, V;
  double* L;                              /* logits [M][V] */
  int v0, v1;
} lm_job;

static void* lm_worker(void* p) {
  lm_job* a = (lm_job*)p;
  for (int v = a->v0; v < a->v1; ++v) {
    const uint16_t* wr = a->W + (size_t)v * a->K;
    for (int m = 0; m < a->M; ++m) {
      const uint16_t* hr = a->H + (size_t)m * a->K;
      double acc = 0.0;
      for (int k = 0; k < a->K; ++k) acc += orc_half_to_double(hr[k]) * orc_half_to_double(wr[k]);
      a->L[(size_t)m * a->V + v] = acc;
    }
  }
  return NULL;
}

int orc_lmhead_argmax(const uint16_t* H, const uint16_t* W, int M, int K, int V, int32_t* out_idx, double* out_val,
                      double* logits, int nthreads) {
  if (!H || !W || !out_idx || M < 1 || K < 1 || V < 1) return -1;
  double* L = logits ? logits : (double*)malloc(sizeof(double) * (size_t)M * (size_t)V);
  if (!L) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > V) nthreads = V;
  lm_job* jobs = (lm_job*)calloc((size_t)nthreads, sizeof(lm_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    lm_job j = {H, W, M, K, V, L, (int)((long long)V * t / nthreads), (int)((long long)V * (t + 1) / nthreads)};
    jobs[t] = j;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, lm_worker, &jobs[t]);
  lm_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  for (int m = 0; m < M; ++m) {
    const double* row = L + (size_t)m * V;
    int best = 0;
    for (int v = 1; v < V; ++v) if (row[v] > row[best]) best = v;   /* strict: the first maximum wins */
    out_idx[m] = best;
    if (out_val) out_val[m] = row[best];
  }
  free(jobs); free(th);
  if (!logits) free(L);
  return 0;
}

/* ------------------------------------------------------------------------------------------------------
 * Tree-masked verify attention (ancestry mask S:129-132) and KV compaction.
 * Straight from the definitions: for every (row, head) the list of visible cache rows, scores in fp64,
 * softmax with the maximum subtracted, the weighted sum of values in fp64.
 * ---------------------------------------------------------------------------------------------------- */
int orc_tree_attention(const uint16_t* Q, const uint16_t* Kc, const uint16_t* Vc, const int32_t* parents, int M, int L,
                       int Hq, int Hkv, int D, double* O) {
  if (!Q || !Kc || !Vc || !parents || !O || M < 1 || L < 0 || Hq < 1 || Hkv < 1 || D < 1 || Hq % Hkv) return -1;
  if (parents[0] != -1) return -1;
  for (int i = 1; i < M; ++i) if (parents[i] < 0 || parents[i] >= i) return -1;
  const int rows = L + M, grp = Hq / Hkv;
  int* vis = (int*)malloc(sizeof(int) * (size_t)rows);
  double* sc = (double*)malloc(sizeof(double) * (size_t)rows);
  const double scale = 1.0 / sqrt((double)D);
  for (int i = 0; i < M; ++i) {
    int nv = 0;
    for (int r = 0; r < L; ++r) vis[nv++] = r;                            /* the cached prefix */
    for (int a = i; a >= 0; a = a == 0 ? -1 : parents[a]) vis[nv++] = L + a;   /* i and its ancestors */
    for (int h = 0; h < Hq; ++h) {
      const int g = h / grp;
      const uint16_t* q = Q + ((size_t)i * Hq + h) * D;
      double mx = -HUGE_VAL;
      for (int t = 0; t < nv; ++t) {
        const uint16_t* k = Kc + ((size_t)vis[t] * Hkv + g) * D;
        double acc = 0.0;
        for (int d = 0; d < D; ++d) acc += orc_half_to_double(q[d]) * orc_half_to_double(k[d]);
        sc[t] = acc * scale;
        if (sc[t] > mx) mx = sc[t];
      }
      double den = 0.0;
      for (int t = 0; t < nv; ++t) { sc[t] = exp(sc[t] - mx); den += sc[t]; }
      double* o = O + ((size_t)i * Hq + h) * D;
      for (int d = 0; d < D; ++d) o[d] = 0.0;
      for (int t = 0; t < nv; ++t) {
        const uint16_t* v = Vc + ((size_t)vis[t] * Hkv + g) * D;
        const double w = sc[t] / den;
        for (int d = 0; d < D; ++d) o[d] += w * orc_half_to_double(v[d]);
      }
    }
  }
  free(vis); free(sc);
  return 0;
}

int orc_kv_compact(uint16_t* Kc, uint16_t* Vc, int L, int Hkv, int D, const int32_t* accept_out) {
  if (!Kc || !Vc || !accept_out || L < 0 || Hkv < 1 || D < 1) return -1;
  const int n = accept_out[0];
  const size_t row = (size_t)Hkv * D;
  for (int k = 1; k <= n; ++k) {   /* path[k-1] >= k, so ascending k never overwrites a row still to be read */
    const int src = L + accept_out[3 + k - 1], dst = L + k;
    if (src != dst) {
      memmove(Kc + (size_t)dst * row, Kc + (size_t)src * row, row * sizeof(uint16_t));
      memmove(Vc + (size_t)dst * row, Vc + (size_t)src * row, row * sizeof(uint16_t));
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------------------
 * Block Hadamard rotation: the definition, one output at a time.
 * ---------------------------------------------------------------------------------------------------- */
int orc_hadamard(const uint16_t* X, int M, int K, int B, double* Y) {
  if (!X || !Y || M < 1 || B < 1 || (B & (B - 1)) || K < B || K % B) return -1;
  const double norm = 1.0 / sqrt((double)B);
  for (int m = 0; m < M; ++m)
    for (int b = 0; b < K; b += B)
      for (int i = 0; i < B; ++i) {
        double acc = 0.0;
        for (int j = 0; j < B; ++j) {
          const double x = orc_half_to_double(X[(size_t)m * K + b + j]);
          acc += (__builtin_popcount((unsigned)(i & j)) & 1) ? -x : x;
        }
        Y[(size_t)m * K + b + i] = acc * norm;
      }
  return 0;
}

int orc_allreduce(const uint16_t* P, int T, size_t n, uint16_t* out) {
  if (!P || !out || T < 1) return -1;
  for (size_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int r = 0; r < T; ++r) acc += orc_half_to_double(P[(size_t)r * n + i]);
    out[i] = orc_double_to_half(acc);
  }
  return 0;
}

int orc_quantize_act_int8(const uint16_t* X, int M, int K, int8_t* Xq, float* sx, int32_t* xsum) {
  if (!X || !Xq || !sx || !xsum || M < 1 || K < 128 || K % 128) return -1;
  for (int m = 0; m < M; ++m) {
    const uint16_t* xr = X + (size_t)m * K;
    float amax = 0.0f;
    for (int k = 0; k < K; ++k) {
      const float a = fabsf(orc_half_to_float(xr[k]));
      if (a > amax) amax = a;
    }
    const float inv = amax > 0.0f ? 127.0f / amax : 0.0f;
    sx[m] = amax / 127.0f;
    for (int g = 0; g < K / 128; ++g) {
      int32_t sum = 0;
      for (int k = g * 128; k < (g + 1) * 128; ++k) {
        float q = nearbyintf(orc_half_to_float(xr[k]) * inv);   /* default rounding mode: nearest even */
        if (q > 127.0f) q = 127.0f;
        if (q < -127.0f) q = -127.0f;
        Xq[(size_t)m * K + k] = (int8_t)q;
        sum += (int32_t)q;
      }
      xsum[(size_t)m * (K / 128) + g] = sum;
    }
  }
  return 0;
}

int orc_gemm_w4a8(const int8_t* Xq, const float* sx, const uint8_t* codes, const uint16_t* scales, int M, int K, int N,
                  double* Y) {
  if (!Xq || !sx || !codes || !scales || !Y || M < 1 || K < 128 || K % 128 || N < 1) return -1;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0.0;
      for (int g = 0; g < K / 128; ++g) {
        long long dot = 0;
        for (int k = g * 128; k < (g + 1) * 128; ++k)
          dot += (long long)Xq[(size_t)m * K + k] * ((int)codes[(size_t)k * N + n] - 8);
        acc += orc_half_to_double(scales[(size_t)g * N + n]) * (double)dot;
      }
      Y[(size_t)m * N + n] = (double)sx[m] * acc;
    }
  return 0;
}
