/* w4a16.h — C ABI of the B200 (sm_100a) W4A16 verification hot path of arXiv 2505.22179 (HierSpec).
 *
 * The path: the target model's multi-token verification forward through W4A16 linear layers (group-128
 * int4 weights, fp16 activations, fp32 accumulate) at draft widths M = 1..64, followed by greedy
 * tree/sequence acceptance.  Citations are PAPER.md lines ("P:n"), SPEC.md lines ("S:n"), SURVEY.md
 * sections; the readings of the paper these calls implement are listed in DESIGN.md §3 (R1..R15).
 *
 * Conventions for every call:
 *   - All tensor pointers are DEVICE pointers (cudaMalloc'd or equivalent), 16-byte aligned.
 *   - fp16 tensors are passed as uint16_t* holding IEEE binary16 bit patterns.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); every call is asynchronous on it, does no
 *     host synchronisation, allocates nothing, and is CUDA-graph capturable.
 *   - The caller owns and allocates every buffer; the library keeps no global state.
 *   - Return value: W4A16_OK (0) or a negative w4a16_status detected on the host (arguments, shapes,
 *     alignment, workspace, launch failure).  Problems only visible on the device are written to a
 *     caller-provided device status word (w4a16_dev_status values).
 *   - Thread safety: calls are re-entrant; concurrent calls must not share output or workspace buffers.
 *   - Residency: the family-A GEMMs (w4a16_gemm at M <= 16, w4a8_gemm at M <= 16) launch one CTA per SM and a
 *     split tile's owner CTA waits for the other CTAs of its tile, so they assume the whole grid becomes
 *     resident: another kernel that occupies SMs indefinitely (a spinning persistent kernel on a concurrent
 *     stream) can delay them until it yields. Ordinary concurrent kernels only delay them.
 *
 * Shapes (GEMM convention of BASELINE.json): Y[M,N] = X[M,K] · W[K,N]; K = in-features, N = out-features.
 * Requirements: group == 128, K % 128 == 0, N % 128 == 0, 1 <= M <= 64 for the GEMM.
 *
 * Packed weight layout (the blob w4a16_pack writes and w4a16_gemm streams; little-endian):
 *   a sequence of 128x128 (k x n) tiles, n-tile major: tile (t = n/128, g = k/128) occupies TB bytes at
 *   byte (t*(K/128) + g) * TB, TB = 8704 (ASYM) or 8448 (SYM). Inside a tile:
 *     bytes [0, 8192):     4-bit codes. Row r = n % 128 owns the 64 bytes at r*64: four 16-byte chunks, chunk
 *                          p (k = 128g + 32p .. +31) stored at byte r*64 + 16*(p XOR ((r/2) % 4)) — the XOR
 *                          makes the 16-byte reads of 8 consecutive rows hit 8 distinct shared-memory bank
 *                          groups. Word w (32-bit) of a chunk holds k = 32p + 8w + i (i = 0..7) with the
 *                          code of local index i in nibble slot (i % 2) * 4 + i / 2 (bits 4*slot..4*slot+3).
 *                          So the two 16-bit halves of (word & 0x000F000F) are the codes of k = 8w and 8w+1,
 *                          of ((word >> 4) & 0x000F000F) those of 8w+2, 8w+3, and so on.
 *                          Canonical logical order is SPEC's "low nibble first" along k;
 *                          example: codes 0..7 of one word are 0x76543210 canonical, 0x75316420 physical.
 *     bytes [8192, ...):   per row r, the fp16 scale s and (ASYM) the fp16 zero point z (an integer in
 *                          [0,15]) side by side, so one 32-bit load fetches both: ASYM {s, z} at 8192 + 4r
 *                          (bytes [8192, 8704)); SYM s at 8192 + 2r (bytes [8192, 8448)).
 *   Codes, scale and zero of a 128x128 tile are adjacent, so a CTA that owns a run of tiles streams one
 *   contiguous byte range. A column shard (n range, multiple of 128) is a contiguous
 *   sub-range of whole tiles. SYM mode: z == 8 and no zero bytes are stored.
 * Dequantised weight (definition): w_hat[k][n] = fp16_rne((q[k][n] - z) * s).
 */
#ifndef W4A16_H
#define W4A16_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  W4A16_OK = 0,
  W4A16_ERR_ARG = -1,        /* NULL pointer, bad mode/group, or value out of range */
  W4A16_ERR_SHAPE = -2,      /* K, N not multiples of 128, M out of [1, 64], n out of [1, 1024] */
  W4A16_ERR_ALIGN = -3,      /* a pointer is not 16-byte aligned */
  W4A16_ERR_WORKSPACE = -4,  /* workspace NULL or smaller than w4a16_gemm_workspace_bytes() */
  W4A16_ERR_CUDA = -5        /* kernel launch or device query failed */
} w4a16_status;

enum { W4A16_ASYM = 0, W4A16_SYM = 1 };
enum { W4A16_DEV_OK = 0, W4A16_DEV_NONFINITE = 1, W4A16_DEV_BAD_TREE = 2 };
enum { W4A16_FAMILY_AUTO = -1, W4A16_FAMILY_MMA_SYNC = 0, W4A16_FAMILY_TCGEN05 = 1, W4A16_FAMILY_MMA_SYNC_S = 2,
       W4A16_FAMILY_TCGEN05_OC = 3 };
#define W4A16_GROUP 128
#define W4A16_MAX_M 64
#define W4A16_MAX_TREE 1024
#define W4A16_MAX_N 1048576   /* N limit: the workspace holds a fixed region of W4A16_MAX_N / 128 tile counters */

typedef struct CUstream_st* w4a16_stream_t;   /* == cudaStream_t */

/* Bytes of the packed blob for a K x N weight (0 on a bad shape/mode/group). */
size_t w4a16_packed_bytes(int K, int N, int group, int mode);

/* w4a16_pack — quantise fp16 W[K][N] (row-major) to int4 codes + per-group fp16 scale/zero.
 * Method: GPTQ W4 group-128 storage format, round-to-nearest in place of GPTQ's calibration
 * (S:95), per column n and group of 128 consecutive k:
 *   ASYM: wmin = min(min w, 0), wmax = max(max w, 0); equal -> (-1, 1); s = fp16_rne((wmax-wmin)/15);
 *         z = clamp(rne(-wmin/s), 0, 15); q = clamp(rne(w/s) + z, 0, 15)     (fp32 arithmetic, RNE)
 *   SYM:  amax = max|w| (0 -> 1); s = fp16_rne(2*amax/15); z = 8; q = clamp(rne(w/s) + 8, 0, 15)
 *         This is the GPTQ / Marlin symmetric storage convention (codes 0..15 around z = 8, so w = -amax may
 *         take code 0 = -8s; reading R1). It is NOT SPEC's symmetric scheme (s = amax/7, half-away rounding,
 *         codes -7..7), which binds only SPEC's CPU program.
 *   A scale that underflows to 0 is recomputed from the range (-1, 1).
 * Output: `packed`, w4a16_packed_bytes(K, N, group, mode) bytes in the layout above.
 * Non-finite weights count as 0 and set *dev_status = W4A16_DEV_NONFINITE; otherwise *dev_status is
 * left untouched (caller zeroes it).  dev_status may be NULL.  Bit-exact with the CPU oracle. */
int w4a16_pack(const uint16_t* W, int K, int N, int group, int mode, void* packed, int32_t* dev_status,
               w4a16_stream_t stream);

/* w4a16_unpack — W_hat[K][N] fp16 = fp16_rne((q - z) * s) (test/debug). Bit-exact with the oracle. */
int w4a16_unpack(const void* packed, int K, int N, int group, int mode, uint16_t* W_hat, w4a16_stream_t stream);

/* Workspace bytes w4a16_gemm needs for this shape. Layout: a fixed region of W4A16_MAX_N / 128 int32 tile
 * counters, one per 128-byte line (1 MiB, the same offset for every shape) followed by the fp32 split-K partials of this shape.
 * Before its first use the workspace must be zero-filled (w4a16_workspace_init); every w4a16_gemm leaves
 * the counters zeroed again, so one workspace, sized by the maximum over the shapes it serves, can be
 * shared by any sequence of calls of any shapes on one stream. Returns 0 on bad shape. */
size_t w4a16_gemm_workspace_bytes(int M, int K, int N, int group);
int w4a16_workspace_init(void* workspace, size_t workspace_bytes, w4a16_stream_t stream);

/* w4a16_gemm — Y[M][N] fp16 = X[M][K] fp16 · W_hat[K][N], fp32 accumulation, one fp32->fp16 RNE at the
 * end (BASELINE.json north_star; reading R8).  Scales are applied per group to fp32 partial sums, so Y
 * equals the oracle's fp64 result within |Y - Y_ref| <= 1e-2 * (1 + |Y_ref|), not bit-for-bit.
 * The split-K / stream-K plan depends only on (K, N, SM count), never on M, and the cross-CTA reduction
 * runs in a fixed order: results are deterministic and row m of Y does not depend on the other rows of X
 * within one kernel family (w4a16_gemm_family). Rows of Y beyond M and bytes outside Y are
 * never written. */
int w4a16_gemm(const uint16_t* X, const void* packed, uint16_t* Y, int M, int K, int N, int group, int mode,
               void* workspace, size_t workspace_bytes, w4a16_stream_t stream);

/* w4a16_gemm_ex — w4a16_gemm with an explicit kernel family: W4A16_FAMILY_AUTO (= w4a16_gemm),
 * W4A16_FAMILY_MMA_SYNC (mma.sync, exact integer codes (q - z) in the MMA operands, group scale applied to
 * the fp32 group sums; M <= 16, else W4A16_ERR_SHAPE), W4A16_FAMILY_MMA_SYNC_S (mma.sync, scale folded into
 * the dequantised fp16 weights w_hat; M <= 16), W4A16_FAMILY_TCGEN05 (5th-gen tensor cores, exact w_hat in
 * TMEM; any M <= 64) or W4A16_FAMILY_TCGEN05_OC (5th-gen tensor cores, exact (q - z) codes in TMEM, per-unit
 * TMEM accumulator, group scale applied in fp32; any M <= 64). The families that scale group sums compute
 * sum_g s_g * sum_k (q - z) x (the exact weight, reading R22), the others sum_k w_hat x; both are within the
 * tolerance above of the oracle and results are batch-invariant within one family. */
int w4a16_gemm_ex(const uint16_t* X, const void* packed, uint16_t* Y, int M, int K, int N, int group, int mode,
                  void* workspace, size_t workspace_bytes, int family, w4a16_stream_t stream);

/* w4a16_gemm_strided — w4a16_gemm_ex whose X rows are ldx elements apart (row m at X + m * ldx), e.g. the
 * attention-output slice of a fused QKV projection read in place. ldx >= K and ldx % 8 == 0 (rows stay
 * 16-byte aligned), else W4A16_ERR_ARG; ldx = K is w4a16_gemm_ex. Only elements [m][0, K) are read; the
 * result is bitwise the one w4a16_gemm_ex gives for the same rows stored contiguously. */
int w4a16_gemm_strided(const uint16_t* X, int ldx, const void* packed, uint16_t* Y, int M, int K, int N, int group,
                       int mode, void* workspace, size_t workspace_bytes, int family, w4a16_stream_t stream);

/* verify_accept — greedy acceptance of a draft tree against the target's argmax (rule per
 * S:289/S:298, reading R9).  n nodes, node 0 = root (the last committed token, row 0 of the verify
 * forward), parents[0] = -1, 0 <= parents[i] < i.  target_argmax[i] = target's greedy token after node i.
 * ok(i) = every edge p->c on the root->i path has tokens[c] == target_argmax[p]; the accepted node is the
 * deepest ok node (ties: smallest index). Writes (device int32) out[0] = accepted length (root excluded),
 * out[1] = bonus token = target_argmax[accepted node], out[2] = device status, out[3 .. 3+n) = accepted
 * path as node indices root->leaf, padded with -1.  A malformed tree writes {0, -1, BAD_TREE, -1 ...}.
 * A sequence draft is parents[i] = i - 1 (longest matching prefix). 1 <= n <= W4A16_MAX_TREE. */
int verify_accept(const int32_t* tokens, const int32_t* parents, const int32_t* target_argmax, int n, int32_t* out,
                  w4a16_stream_t stream);

/* w4a16_lmhead_argmax — the target's greedy token for every verify row (the argmax the
 * greedy acceptance rule compares drafts with): out_argmax[m] = the smallest v maximising
 * logit[m][v] = sum_k H[m][k] * W_lm[v][k], out_max[m] = that logit (may be NULL). FP16 LM head (the paper
 * keeps the drafter FP16; reading R12), fp32 accumulation, ties -> lowest id; the logits are
 * reduced in the GEMM epilogue and never written. H: fp16 [M][K] (the verify rows' final hidden states);
 * W_lm: fp16 [V][K] row-major (the nn.Linear weight layout: row v = token v); out_argmax: int32 [M], the
 * target_argmax input of verify_accept. 1 <= M <= 64, K % 128 == 0, V % 128 == 0. workspace: zero-filled
 * once, w4a16_lmhead_workspace_bytes() bytes; every call leaves it re-armed. Because fp32 sums decide the
 * argmax, a row whose top two logits are closer than the accumulation error may pick either. */
size_t w4a16_lmhead_workspace_bytes(int M, int K, int V);
int w4a16_lmhead_argmax(const uint16_t* H, const uint16_t* W_lm, int M, int K, int V, int32_t* out_argmax,
                        float* out_max, void* workspace, size_t workspace_bytes, w4a16_stream_t stream);

/* w4a16_tree_attention — tree-masked verify attention: the M verify rows (root + draft
 * tree) attend the cached prefix and, inside the tree, themselves and their ancestors only (the
 * ancestry mask). Q: fp16 [M][Hq][D]; Kc, Vc: fp16 [L + M][Hkv][D] (prefix rows 0..L-1, the verify
 * rows' own keys/values at L..L+M-1); parents: int32 [M] on the device, a valid tree (parents[0] = -1,
 * parents[i] < i; verify_accept reports malformed trees). O[m][h] = softmax_j(q.k_j / sqrt(D)) . v_j over the
 * visible rows j, kv head h / (Hq / Hkv) (GQA); fp32 scores / softmax / accumulation, fp16 probabilities and
 * output. D == 128, 1 <= M <= 64, Hq % Hkv == 0, Hq <= 512, L >= 0. workspace:
 * w4a16_tree_attention_workspace_bytes(); its first 65536 bytes (the split-merge counters) must be zero before
 * the first call, and every call leaves them zero. One cooperative launch: the CTAs of a call must all be
 * resident (the splits are merged inside the kernel).
 * A row m whose ancestry walk meets a parent outside [-1, m) (a malformed tree) sees the prefix and itself
 * only; the walk never loops (each valid step strictly decreases the row index). */
size_t w4a16_tree_attention_workspace_bytes(int M, int L, int Hq, int Hkv, int D);
int w4a16_tree_attention(const uint16_t* Q, const uint16_t* Kc, const uint16_t* Vc, const int32_t* parents, int M,
                         int L, int Hq, int Hkv, int D, uint16_t* O, void* workspace, size_t workspace_bytes,
                         w4a16_stream_t stream);
/* w4a16_kv_compact — after verify_accept, keep the accepted path in the cache (S:159-164 cache_select):
 * rows L + k of Kc and Vc (each Hkv * D fp16) become the former rows L + path[k-1], k = 1..accepted, where
 * accept_out is verify_accept's device output (read on the device: no host synchronisation). Row L (the root)
 * stays. Call once per layer. D % 8 == 0. */
int w4a16_kv_compact(uint16_t* Kc, uint16_t* Vc, int L, int Hkv, int D, const int32_t* accept_out,
                     w4a16_stream_t stream);

/* w4a16_hadamard — the online activation rotation of W4A16+Rot (QuaRot-style):
 * Y[m][bB + i] = fp16_rne(sum_j (-1)^popcount(i & j) X[m][bB + j] / sqrt(B)) for every row m and block b of
 * B consecutive k (block-diagonal normalised Sylvester Hadamard; H is symmetric and orthogonal, so with the
 * weights rotated offline the same way, W' = H W before w4a16_pack, X W = (X H)(H W)). fp32 arithmetic.
 * X, Y: fp16 [M][K]; Y may equal X (in place). block in {64, 128, 256, 512, 1024}, K % block == 0, M >= 1. */
int w4a16_hadamard(const uint16_t* X, uint16_t* Y, int M, int K, int block, w4a16_stream_t stream);

/* w4a16_silu_mul — Llama MLP glue between the fused gate-up GEMM and the down GEMM of the verify forward
 * (not a step of the paper's method): GU is fp16 [M][2F] holding [gate | up] per row (the
 * rank-local shard layout of tp.py), out is fp16 [M][F], out[m][j] = fp16_rne(silu(gate) * up) in fp32.
 * F % 8 == 0, M >= 1. */
int w4a16_silu_mul(const uint16_t* GU, int M, int F, uint16_t* out, w4a16_stream_t stream);
/* w4a16_silu_mul_blocked — the same glue for a gate-up output whose columns come in blocks: GU[m] holds, for
 * b = 0 .. F/block - 1, `block` gate columns then the matching `block` up columns; out[m][b*block + i] =
 * fp16_rne(silu(GU[m][2b*block + i]) * GU[m][(2b+1)*block + i]) in fp32. block = F is w4a16_silu_mul; block = 64
 * is the layout W4A16_OP_GEMM_SILU fuses. block % 8 == 0, F % block == 0. */
int w4a16_silu_mul_blocked(const uint16_t* GU, int M, int F, int block, uint16_t* out, w4a16_stream_t stream);

/* ---- Chains: a verify forward's whole sequence of ops in ONE persistent launch ----------------------
 * A verify forward is a long sequence of small W4A16 GEMMs (4 per decoder layer, 320 for Llama-3-70B)
 * whose weights never depend on earlier ops. Launched one by one, every GEMM pays its own pipeline fill
 * and drain (a fixed ~8 us per GEMM on B200). A chain runs the sequence in one persistent
 * kernel (one CTA per SM): the weight stream (TMA) runs ahead across op boundaries, and an op waits
 * only where it reads a buffer an earlier op writes (RAW), or writes a buffer an earlier op reads or
 * writes (WAR / WAW). The dependencies are derived on the host from the ops' buffer ranges.
 * Each GEMM op computes exactly what w4a16_gemm_ex of the same family computes (same split plan, same
 * reduction order: bit-identical results); each SILU_MUL op exactly what w4a16_silu_mul computes.
 * All G CTAs of a chain must be co-resident: do not run other kernels concurrently with a chain on the
 * same device (it is launched as a cooperative kernel). */
enum { W4A16_OP_GEMM = 0, W4A16_OP_SILU_MUL = 1, W4A16_OP_ALLREDUCE = 2, W4A16_OP_GEMM_SILU = 3 };
/* W4A16_OP_GEMM_SILU: the Llama MLP's gate-up GEMM with SiLU*mul fused into its epilogue (family A chains).
 * The weight's N columns come in 128-column tiles of [64 gate | 64 up] (w4a16_silu_mul_blocked's block = 64
 * layout); Y is [M][N/2]: Y[m][64 t + i] = fp16_rne(silu(g) * u), g = fp16(G[m][128 t + i]),
 * u = fp16(G[m][128 t + 64 + i]), G = X . W_hat — exactly w4a16_gemm followed by w4a16_silu_mul_blocked. */
typedef struct {
  int kind;            /* W4A16_OP_GEMM, W4A16_OP_GEMM_SILU, W4A16_OP_SILU_MUL or W4A16_OP_ALLREDUCE */
  const void* X;       /* GEMM: X [M][K] fp16.  SILU_MUL: GU [M][2N] fp16 ([gate | up] per row).
                        * ALLREDUCE: this rank's partial P [M][N] fp16, inside its symmetric region */
  const void* packed;  /* GEMM: packed weight blob of w4a16_pack (K x N, `mode`).  SILU_MUL: NULL.
                        * ALLREDUCE: HOST pointer to the w4a16_peer_group (read by w4a16_chain_plan only) */
  void* Y;             /* GEMM: Y [M][N] fp16.  GEMM_SILU: Y [M][N/2] fp16.  SILU_MUL: out [M][N] fp16.
                        * ALLREDUCE: out [M][N] fp16 */
  int K, N;            /* GEMM: as w4a16_gemm.  SILU_MUL: K = 2N, N = F (N % 8 == 0).  ALLREDUCE: K = N, N % 8 == 0 */
  int mode;            /* GEMM: W4A16_ASYM or W4A16_SYM; every GEMM of a chain uses the same mode */
  int ldx;             /* GEMM: row stride of X in elements; 0 = K (contiguous), else ldx >= K and ldx % 8 == 0
                        * (e.g. the first K columns of a wider [M][ldx] buffer). Other kinds: 0 */
} w4a16_op;

/* ---- Tensor-parallel all-reduce inside a chain ------------------------------
 * The row-parallel GEMMs of a t-way tensor-parallel verify forward (O and down: each rank multiplies its
 * K-shard, Megatron layout) produce partial sums P_r that are summed over the ranks. An
 * ALLREDUCE op does that sum INSIDE the chain, one-shot over peer memory, so a whole tensor-parallel forward
 * stays one persistent launch per rank instead of 2 launches + 2 NCCL all-reduces per layer:
 *   out[m][n] = fp16_rne( sum over ranks of (float) P_r[m][n] )   (fp32 sum, one rounding)
 * Fused with the GEMM that produces P, tile by tile: when this rank's GEMM has written 128-column tile t of P
 * it bumps tile t's ready counter in EVERY rank's flag area (system-scope release: one NVLS multimem.red
 * through the group's multicast mapping, else one red per peer mapping); the ALLREDUCE op's CTA for tile t
 * waits until its local counter shows all `world` ranks for this run and reduces that tile at once —
 * through the multicast mapping (multimem.ld_reduce: the NVSwitch adds the ranks' fp16 values with fp32
 * accumulation and returns the sum; order inside the switch unspecified, so ranks agree but the sum is not
 * bit-pinned to rank order) or, without multicast, with one 16-byte load per peer mapping, summed in fp32
 * in rank order (bit-identical on every rank). Each reduced tile then publishes its own ready flag, so the
 * next GEMM starts on the tiles that are done: no grid-wide wait anywhere in the all-reduce.
 * Symmetric region: each rank owns one device region of the same size with the P buffers and a flag area
 * (w4a16_peer_flag_bytes, at the same offset on every rank) in it, mapped by every peer (CUDA IPC:
 * w4a16_ipc_alloc / w4a16_ipc_open) and/or bound to one multicast object (NVLS: w4a16_mc_*). Rules (checked
 * by w4a16_chain_plan): every ALLREDUCE of a chain names the same group; its X is exactly the Y of the GEMM
 * right before it (N <= 128 * W4A16_AR_MAX_TILES); X lies inside base[rank]; and cyclically between an
 * ALLREDUCE that reads a buffer and the next op that writes it there is another ALLREDUCE (a rank publishes
 * that op's tile counters only after it has finished the earlier ALLREDUCE — so peers are done reading —
 * two alternating partial buffers, as in a decoder layer's O and down, satisfy it). Every rank runs the same
 * sequence of chains over the group. A wait that does not complete within ~60 s (a peer that never
 * arrives) traps the kernel instead of hanging the device. */
#define W4A16_MAX_PEERS 8
#define W4A16_AR_MAX_TILES 128
typedef struct {
  void* base[W4A16_MAX_PEERS];   /* every rank's symmetric region as mapped in this process; base[rank] is local
                                  * (peers may be NULL when mc_base is set: the multicast path never maps them) */
  size_t bytes;                  /* region size (identical on every rank) */
  size_t flag_offset;            /* flag area offset inside each region (identical on every rank, 256-B aligned) */
  int flag_slots;                /* ALLREDUCE ops the flag area serves (per chain: one slot per ALLREDUCE op) */
  int world, rank;               /* 1 <= world <= W4A16_MAX_PEERS, 0 <= rank < world */
  void* mc_base;                 /* the multicast (NVLS) mapping of the group's regions (w4a16_mc_bind), or
                                  * NULL: peer loads through base[] */
} w4a16_peer_group;
/* Bytes of a flag area for `flag_slots` ALLREDUCE ops (a run counter plus W4A16_AR_MAX_TILES tile counters
 * per slot). */
size_t w4a16_peer_flag_bytes(int flag_slots);
/* Symmetric-region plumbing (CUDA IPC; one process per GPU). w4a16_ipc_alloc: cudaMalloc `bytes` on the
 * current device, zero it, and write its 64-byte IPC handle to handle_out. w4a16_ipc_open: map a peer's
 * region (handle from w4a16_ipc_alloc in another process) into this process, peer access enabled.
 * w4a16_ipc_close / w4a16_ipc_free undo them. W4A16_ERR_CUDA on failure. */
int w4a16_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out);
int w4a16_ipc_open(const void* handle, void** dev_ptr);
int w4a16_ipc_close(void* dev_ptr);
int w4a16_ipc_free(void* dev_ptr);
/* Symmetric regions bound to one multicast object (NVLS, NVSwitch systems; one process per GPU):
 *   w4a16_mc_supported()  1 if the current device supports multicast objects and fabric handles, else 0.
 *   w4a16_mc_create(bytes, world, handle_out, mc_out)   rank 0: create a multicast object for `world`
 *       devices of size round_up(bytes, granularity) and export its 64-byte fabric handle.
 *   w4a16_mc_import(handle, bytes, world, mc_out)   the other ranks: import it (same bytes and world).
 *   w4a16_mc_add_device(mc)   every rank, before any rank binds: add the current device.
 *   w4a16_mc_bind(mc, bytes, uc_out, mc_va_out)   every rank, after every rank has added its device:
 *       allocate `bytes` (rounded as in create) of this device's memory, map it (uc_out: the rank's region, zero-filled),
 *       bind it to the object and map the multicast address range (mc_va_out = w4a16_peer_group.mc_base).
 *   w4a16_mc_free(mc, uc, mc_va, bytes)   unmap and release (after every rank's last use).
 * `mc` is an opaque host handle. Driver API through cudaGetDriverEntryPoint (no link-time libcuda).
 * W4A16_ERR_CUDA on any driver failure, W4A16_ERR_ARG on bad arguments. */
int w4a16_mc_supported(void);
int w4a16_mc_create(size_t bytes, int world, void* handle_out, void** mc_out);
int w4a16_mc_import(const void* handle, size_t bytes, int world, void** mc_out);
int w4a16_mc_add_device(void* mc);
int w4a16_mc_bind(void* mc, size_t bytes, void** uc_out, void** mc_va_out);
int w4a16_mc_free(void* mc, void* uc, void* mc_va, size_t bytes);

/* Bytes of the plan (host buffer) for n_ops ops. */
size_t w4a16_chain_plan_bytes(int n_ops);
/* Workspace bytes of a chain (tile counters per op, op completion counters, split partials). Zero-fill it
 * once (w4a16_workspace_init); every chain run leaves its counters zeroed again. 0 on bad arguments. */
size_t w4a16_chain_workspace_bytes(const w4a16_op* ops, int n_ops, int M, int family);
/* Encode the chain (job table with TMA descriptors of every X, dependency indices) for width M into the
 * HOST buffer `plan` (w4a16_chain_plan_bytes(n_ops) bytes). The caller copies it to device memory once
 * (e.g. cudaMemcpy) and passes that copy to w4a16_chain_run for as long as the buffers stay where they
 * are. family: W4A16_FAMILY_AUTO or an explicit family valid for M (chains serve the mma.sync families,
 * M <= 16). Validates every op like w4a16_gemm / w4a16_silu_mul; in-place ops are rejected. */
int w4a16_chain_plan(const w4a16_op* ops, int n_ops, int M, int family, void* plan, size_t plan_bytes);
/* Run a chain: dev_plan = device copy of the plan for (n_ops, M, family); mode = the GEMMs' mode.
 * workspace: at least w4a16_chain_workspace_bytes(ops, n_ops, M, family) zero-initialised bytes, used by
 * this chain's plan only. Every GEMM of a chain needs (K/128)*(N/128) >= the SM count (every CTA owns a
 * unit). Async on `stream`. */
int w4a16_chain_run(const void* dev_plan, int n_ops, int M, int mode, int family, void* workspace,
                    size_t workspace_bytes, w4a16_stream_t stream);

/* ---- W4A8 variant (4-bit weights with 8-bit activations on INT8 tensor cores,
 * QQQ-style symmetric; reading R21 in DESIGN.md) --------------------------------------------------------
 * w4a8_quantize_act: per-token symmetric int8 activations, decided in IEEE fp32 exactly as
 *   amax = max_k |X[m][k]|; inv = 127 / amax (0 if amax == 0); Xq = clamp(rne(X * inv), -127, 127);
 *   sx[m] = amax / 127; xsum[m][g] = sum of Xq[m][k] over k-group g (128 k).
 *   X fp16 [M][K], Xq int8 [M][K], sx fp32 [M], xsum int32 [M][K/128]; K % 128 == 0, 1 <= M <= W4A16_MAX_M;
 *   all device pointers; Xq 16-byte aligned, sx and xsum 4-byte aligned (else W4A16_ERR_ALIGN).
 * w4a8_gemm: Y[m][n] = fp16_rne(sx[m] * sum_g s[g][n] * (sum_{k in g} Xq[m][k] * q[k][n] - 8 * xsum[m][g]))
 *   on the SYM (z = 8) blob of w4a16_pack (K x N, group 128): int32-exact group sums (INT8 MMA), fp32 group
 *   scaling in k order, per-split partials summed in split order (deterministic). M <= 16 runs on the family-A
 *   pipeline (int8 codes (q - 8) * 16, mma m16n8k32 s8, stream-K; xsum unused), larger M on a k-split kernel
 *   that applies the -8 * xsum correction. workspace: at least w4a8_workspace_bytes(M, K, N) bytes, zeroed
 *   once (w4a16_workspace_init) before its first use; every call leaves it zeroed. Xq, packed and workspace
 *   16-byte aligned (16-byte copies), sx and xsum 4-byte aligned, else W4A16_ERR_ALIGN. */
int w4a8_quantize_act(const uint16_t* X, int M, int K, int8_t* Xq, float* sx, int32_t* xsum, w4a16_stream_t stream);
size_t w4a8_workspace_bytes(int M, int K, int N);
int w4a8_gemm(const int8_t* Xq, const float* sx, const int32_t* xsum, const void* packed, uint16_t* Y, int M, int K, int N,
              void* workspace, size_t workspace_bytes, w4a16_stream_t stream);

/* Human-readable name of a w4a16_status value. */
const char* w4a16_status_string(int status);

/* Kernel family w4a16_gemm uses: W4A16_FAMILY_MMA_SYNC for M <= 16,
 * W4A16_FAMILY_TCGEN05 above. */
int w4a16_gemm_family(int M, int K, int N);

#ifdef __cplusplus
}
#endif
#endif
