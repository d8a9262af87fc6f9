/* w4a16_oracle.h — plain, slow, obviously-correct CPU ORACLE for the W4A16 verify path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load or call this library. The product path (paper_2505_22179_b200/) never
 * includes, links or calls it, and this code shares nothing with the CUDA path (no headers, helpers or
 * tables); the only common code is the input generator in synth/, which holds none of the method's
 * arithmetic.
 *
 * What it computes (citations: PAPER.md line numbers "P:n", SPEC.md "S:n"; readings R1..R15 in DESIGN.md §3):
 *   - quantize:   GPTQ-style W4 group quantisation, round-to-nearest ("symmetrically quantize weights
 *                 to 4-bit with a group size of 128"; RTN stands in for GPTQ calibration as in S:95; ASYM per
 *                 BASELINE.json config 1). Arithmetic in IEEE fp32, RNE, no contraction (reading R5).
 *   - dequantize: w_hat = fp16_rne((q - z) * s)   (exact product, one rounding).
 *   - gemm:       Y[m][n] = sum_k X[m][k] * w_hat[k][n], in fp64, sequential k (BASELINE.json north_star:
 *                 "X[M,K] fp16 x packed W[K,N] -> Y[M,N] fp16, fp32 accumulate"; the oracle uses fp64).
 *   - accept:     greedy tree acceptance (P:79-84 draft-then-verify; the rule is not stated by the paper,
 *                 SPEC S:289/S:298 greedy argmax; reading R9).
 *   - lmhead_argmax: the target's greedy token per verify row: logits[m][v] =
 *                 sum_k H[m][k] * W[v][k] in fp64 (FP16 LM head, reading R12), argmax over v with ties to the
 *                 lowest id — the target_argmax input of accept.
 *   - tree_attention: attention of the verify rows over the KV cache with the draft tree's ancestry mask
 *                 (row i sees the cached prefix and the tree rows that are i or
 *                 an ancestor of i; P:80-82 tree drafts), softmax in fp64.
 *   - kv_compact: after acceptance keep the root and the accepted path's rows, in order (S:159-164
 *                 cache_select of the accepted root-to-leaf path).
 *   - w4a8:       per-token int8 activation quantisation and the W4A8 GEMM.
 *   - allreduce:  the sum over tensor-parallel ranks of row-parallel partial products.
 *   - hadamard:   the rotation of W4A16+Rot (QuaRot-style Hadamard rotation):
 *                 block-diagonal normalised Sylvester Hadamard along k, y = x (I (x) H_B) / sqrt(B).
 * The arithmetic works on plain arrays: codes uint8 [K][N], scales/zeros fp16 [K/group][N]. The byte layout
 * of the ABI's packed blob is a separate pair of functions (layout_pack / layout_unpack), re-derived here
 * from its definition in include/w4a16.h (not shared):
 *   the blob is a sequence of 128x128 (k x n) tiles, tile (t = n/128, g = k/128) at byte
 *   (t*(K/128) + g) * TB with TB = 8704 (ASYM) or 8448 (SYM). Inside a tile: bytes [0, 8192) hold codes,
 *   row r = n%128 owns the 64 bytes at r*64, four 16-byte chunks; chunk p (k = 128g + 32p .. +31) sits at
 *   byte r*64 + 16*(p XOR ((r/2) % 4)); inside a chunk, little-endian 32-bit word w holds k = 32p + 8w + i,
 *   i = 0..7, in nibble slot (i%2)*4 + i/2. Then per row r: ASYM: fp16 scale at 8192 + 4r and fp16 zero at
 *   8192 + 4r + 2 (bytes [8192, 8704)); SYM: fp16 scale at 8192 + 2r (bytes [8192, 8448)).
 */
#ifndef W4A16_ORACLE_H
#define W4A16_ORACLE_H
#include <stdint.h>
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORC_ASYM 0
#define ORC_SYM 1
#define ORC_DEV_OK 0
#define ORC_DEV_NONFINITE 1
#define ORC_DEV_BAD_TREE 2

/* IEEE binary16 <-> binary32/binary64, bit-level, round-to-nearest-even (subnormals, inf, NaN). */
float orc_half_to_float(uint16_t h);
double orc_half_to_double(uint16_t h);
uint16_t orc_float_to_half(float f);
uint16_t orc_double_to_half(double d);

/* Quantise fp16 W[K][N] (row-major) per column n and per group of `group` consecutive k.
 * codes: uint8 [K][N] (values 0..15); scales: fp16 [K/group][N]; zeros: fp16 [K/group][N] (ASYM; in SYM mode
 * zeros may be NULL, otherwise it is filled with 8). *status = ORC_DEV_NONFINITE if any W is not finite.
 * Returns 0 or -1 on bad arguments. */
int orc_quantize(const uint16_t* W, int K, int N, int group, int mode, uint8_t* codes, uint16_t* scales,
                 uint16_t* zeros, int32_t* status);

/* W_hat[K][N] fp16 = fp16_rne((q - z) * s) with z = 8 in SYM mode. */
int orc_dequantize(const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int K, int N, int group,
                   int mode, uint16_t* W_hat);

/* Y[M][N] (fp64) = X[M][K] (fp16) * W_hat (dequantised from codes/scales/zeros); k summed in order 0..K-1 in
 * fp64. Columns are independent: nthreads >= 1 splits columns across pthreads, the result is identical. */
int orc_gemm(const uint16_t* X, const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int M, int K,
             int N, int group, int mode, double* Y, int nthreads);

/* Same definition for a list of columns only: Ycols[m*ncols + j] = Y[m][cols[j]]. */
/* Y = X . W with W[k][n] = (q - z) * s exactly (no fp16 rounding; reading R22: the scale-after-sum families). */
int orc_gemm_exact(const uint16_t* X, const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int M,
                   int K, int N, int group, int mode, double* Y, int nthreads);
int orc_gemm_cols(const uint16_t* X, const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int M,
                  int K, int N, int group, int mode, const int32_t* cols, int ncols, double* Ycols);

/* The ABI's packed blob (group 128; K % 128 == 0, N % 128 == 0). */
size_t orc_packed_bytes(int K, int N, int mode);
size_t orc_code_word_offset(int K, int N, int mode, int k, int n);   /* byte offset of the word holding (k, n) */
int orc_nibble_slot(int i);
int orc_layout_pack(const uint8_t* codes, const uint16_t* scales, const uint16_t* zeros, int K, int N, int mode,
                    uint8_t* packed);
int orc_layout_unpack(const uint8_t* packed, int K, int N, int mode, uint8_t* codes, uint16_t* scales,
                      uint16_t* zeros);

/* Greedy acceptance over a draft tree of n nodes (node 0 = root = last committed token, parents[0] = -1,
 * parents[i] < i). out[0] = accepted length, out[1] = bonus token, out[2] = device status,
 * out[3 .. 3+n) = accepted path (node indices, root excluded, root->leaf), padded with -1.
 * Returns 0, or -1 on bad arguments (n < 1 or NULL). A malformed tree gives out = {0, -1, BAD_TREE, -1...}. */
int orc_accept(const int32_t* tokens, const int32_t* parents, const int32_t* target_argmax, int n, int32_t* out);

/* LM head + greedy argmax: H fp16 [M][K], W fp16 [V][K] (row v = token v's output
 * embedding, the nn.Linear weight layout). logits[m][v] = sum_k H[m][k] * W[v][k] in fp64, k in order.
 * out_idx[m] = the smallest v with the largest logit, out_val[m] = that logit; logits (may be NULL)
 * receives all M x V values. nthreads splits the vocabulary; the result does not depend on it. */
int orc_lmhead_argmax(const uint16_t* H, const uint16_t* W, int M, int K, int V, int32_t* out_idx, double* out_val,
                      double* logits, int nthreads);

/* Tree-masked verify attention. Q fp16 [M][Hq][D]; Kc, Vc fp16 [L + M][Hkv][D] (the cached
 * prefix at rows 0..L-1, the M verify rows' own keys/values at L..L+M-1); parents [M] (parents[0] = -1,
 * parents[i] < i). Query row i, head h attends kv head g = h / (Hq / Hkv) at every prefix row and at rows
 * L + j for j = i or an ancestor of i. O fp64 [M][Hq][D] = softmax(q.k / sqrt(D)) . v over those
 * rows, everything in fp64 (scores, max-subtracted exp, normaliser, weighted sum). Returns 0 / -1. */
int orc_tree_attention(const uint16_t* Q, const uint16_t* Kc, const uint16_t* Vc, const int32_t* parents, int M, int L,
                       int Hq, int Hkv, int D, double* O);

/* KV-cache compaction after acceptance (cache_select of the accepted path): with accept_out of
 * orc_accept (out[0] = accepted length n, out[3..3+n) = path node indices), row L + k of Kc and Vc becomes
 * the former row L + path[k-1] for k = 1..n (row L, the root, stays). Rows are Hkv * D fp16 wide. */
int orc_kv_compact(uint16_t* Kc, uint16_t* Vc, int L, int Hkv, int D, const int32_t* accept_out);

/* Block Hadamard rotation (W4A16+Rot): for every row m and block b of B
 * consecutive k (B a power of two dividing K), Y[m][bB + i] = sum_j (-1)^popcount(i & j) X[m][bB + j] / sqrt(B),
 * in fp64 straight from the definition (Sylvester order). Y fp64 [M][K]. Returns 0 / -1. */
int orc_hadamard(const uint16_t* X, int M, int K, int B, double* Y);

/* W4A8 (4-bit weights, 8-bit activations on INT8 tensor cores, QQQ-style
 * symmetric). Reading R21: per-token symmetric int8 activations, decided in IEEE fp32 exactly
 * as written: amax = max_k |x[m][k]|; inv = 127.0f / amax (0 if amax == 0); q = clamp(rne(x * inv), -127, 127);
 * sx[m] = amax / 127.0f; xsum[m][g] = sum of q over k-group g (128). Returns 0 / -1. */
int orc_quantize_act_int8(const uint16_t* X, int M, int K, int8_t* Xq, float* sx, int32_t* xsum);
/* W4A8 GEMM on SYM group-128 weights (codes q in [0,15], z = 8, fp16 scale s[g][n]):
 * Y[m][n] = sx[m] * sum_g s[g][n] * sum_{k in g} Xq[m][k] * (q[k][n] - 8), inner sums exact integers, the rest
 * in fp64. Y fp64 [M][N]. Returns 0 / -1. */
int orc_gemm_w4a8(const int8_t* Xq, const float* sx, const uint8_t* codes, const uint16_t* scales, int M, int K, int N,
                  double* Y);

/* Tensor-parallel all-reduce of row-parallel partial sums (Megatron row-parallel O / down,
 * y = sum over ranks of the rank's K-shard product): out[i] = fp16_rne(sum_{r < T} P[r][i]), the sum in
 * fp64 (exact for T <= 8 fp16 terms of moderate range), rounded once. P fp16 [T][n]. Returns 0 / -1. */
int orc_allreduce(const uint16_t* P, int T, size_t n, uint16_t* out);

#ifdef __cplusplus
}
#endif
#endif
