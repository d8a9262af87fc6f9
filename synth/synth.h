/* synth.h — seeded, counter-based synthetic INPUT generator (SURVEY §8(d) "Concrete synthetic inputs").
 *
 * This module holds NO arithmetic of the method (no quantisation, no GEMM, no acceptance). It is the only
 * code shared by the CPU oracle side (synth.c) and the GPU side (synth_gpu.cu): both implement the same
 * integer-only generator so that CPU and GPU see bit-identical fp16 inputs without copying tens of GB.
 *
 *   stream(seed, tensor_id) = mix64(mix64(seed) ^ (tensor_id * 0xD1B54A32D192ED03))
 *   u(stream, i)            = mix64(stream + (i + 1) * 0x9E3779B97F4A7C15)          (splitmix64)
 *   v(u)                    = f0 + f1 + f2 + f3 - 131070,  f_j = 16-bit fields of u  (≈ normal, σ≈37837)
 *   value                   = fp16_rne( (float)v * 2^-(shift) * 2^(outlier) )        (all exact before RNE)
 *
 * Weights W[K][N] (row-major, k = in-feature): shift 21 (σ ≈ 0.018, Llama-style init);
 *   2% of (group-of-128-along-k, n) groups are outlier groups scaled ×8.
 * Activations X[M][K]: shift 15 (σ ≈ 1.15); 4 outlier channels (k) scaled ×16.
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { SYNTH_WEIGHT = 0, SYNTH_ACT = 1 };
#define SYNTH_W_SHIFT 21
#define SYNTH_X_SHIFT 15
#define SYNTH_W_OUTLIER_MOD 50   /* 1 in 50 groups (2%) */
#define SYNTH_W_OUTLIER_LOG2 3   /* ×8  */
#define SYNTH_X_OUTLIER_N 4
#define SYNTH_X_OUTLIER_LOG2 4   /* ×16 */

/* Host fill: out[r*cols + c] for r in [0,rows), c in [0,cols). kind = SYNTH_WEIGHT (rows=K, cols=N) or
 * SYNTH_ACT (rows=M, cols=K). Returns 0, or -1 on bad arguments. */
int synth_fill_host(uint64_t seed, uint64_t tensor_id, int kind, int rows, int cols, uint16_t* out);
/* Sub-block [r0,r1) x [c0,c1) of the same tensor (values depend only on (r, c, rows, cols)); out is
 * (r1-r0) x (c1-c0) row-major. */
int synth_fill_host_block(uint64_t seed, uint64_t tensor_id, int kind, int rows, int cols, int r0, int r1, int c0,
                          int c1, uint16_t* out);
/* Single element (used by full-size sampled parity checks). */
uint16_t synth_value_host(uint64_t seed, uint64_t tensor_id, int kind, int rows, int cols, int r, int c);
/* Device fill (synth_gpu.cu): out is a device pointer; async on stream (a cudaStream_t). */
int synth_fill_gpu(uint64_t seed, uint64_t tensor_id, int kind, int rows, int cols, uint16_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
