// gemm_mma.cu — W4A16 verify GEMM, kernel family A ("decode width", M <= 16): SURVEY §8(a) a2-a6.
//
//   Y[M,N] = X[M,K] · W_hat[K,N]   with W_hat = (q - z) * s per group of 128 k (include/w4a16.h)
//
// Design. At M <= 16 the tensor work per weight is small enough for the legacy
// mma.sync pipe (~540 TFLOP/s measured on B200), and keeping dequant + MMA inside each warp's registers avoids
// the TMEM traffic and cross-warp hand-offs of the tcgen05 families.
//  * Work unit = one 128x128 (n x k) weight tile (8704 / 8448 contiguous bytes of the packed blob: codes,
//    scales, zeros). Units are numbered in blob order, so a CTA's range is one contiguous byte range.
//  * Stream-K: CTA c of G = #SMs (one CTA per SM) owns units [c*U/G, (c+1)*U/G) — a (K, N, SM-count)-only plan.
//  * Warp 16 (producer) streams stages of 4 units with ONE bulk copy each (the TMA engine costs ~100+ cycles
//    per issued copy), plus the units' activation slices with a 3-D TMA (SWIZZLE_128B, rows >= M
//    zero-filled), into a ring of up to 12 stages (as many as fit in shared memory); activation loads wait in
//    a queue for their producing op's tile-ready flags (chains), weights never wait.
//  * Warps 0..15 (consumers) = 2 groups x 8 warps; group g takes units 2g, 2g+1 of every stage; warp w of a
//    group owns tile rows 16w..16w+15 (one m16 MMA tile) and all 128 k of its units. A lane reads one 32-bit
//    word (8 consecutive k of one row) per row and chunk with ldmatrix — conflict-free thanks to the XOR
//    chunk permutation of the layout — dequantises it to EXACT (q - z) fp16 with LOP3 + HSUB2/HFMA2, and
//    issues mma.sync m16n8k16 with weights as the MMA-M operand ("swap AB"; tokens are MMA-N). Inside each
//    32-k chunk a k-permutation lets one lane's 8 consecutive k feed two MMA k-steps, with the activations
//    read as one 16-byte vector per token block.
//  * The group scale is applied after the MMA to the fp32 group sum: Y += s * sum_k X (q - z) (the exact
//    weight, reading R22).
//  * Tile boundary: group 1 hands its sums to group 0 through shared memory; a tile split across CTAs is
//    owned by its first CTA, which handles the tile's head as its LAST segment: the others store fp32
//    partials and bump the tile counter, the owner sums them in CTA order (deterministic) and writes Y.
//  * Releases: tile-ready flags, split-tile counters (M <= 8) and op counts are released by the storing
//    thread right after its group's barrier; warp 17 (publisher) releases the rest (split-tile counters at
//    M = 9..16, ALLREDUCE tile bumps, SiLU-op counts) behind one fence per batch and runs the chain's
//    ALLREDUCE ops. The producer acquires what it polled with an acquire-only fence (no MEMBAR behind its
//    bulk copies). Counters, flags and op counts sit on their own 128-byte lines.
//  * W4A8 (kA8): the same pipeline with int8 activations and int8 codes (q - 8) * 16 on mma m16n8k32.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "tma_host.cuh"
#include "w4a16.h"

// Chain tile counters and tile-ready flags: tile t of an op at ints [kCS (cnt_off + t)] (counter) and
// [kCS (cnt_off + t) + kFO] (flag)
#ifndef W4_MA_CSTRIDE
#define W4_MA_CSTRIDE 64   // 256 B per tile, counter and flag on separate 128-B lines (-4.2 % vs packed 8 B at M = 8)
#endif
#ifndef W4_MA_FOFF
#define W4_MA_FOFF 32
#endif

namespace w4 {
namespace ma {

constexpr int kTileN = 128, kTileK = 128;
constexpr int kCS = W4_MA_CSTRIDE, kFO = W4_MA_FOFF;
constexpr int kDSMax = 32;   // op counts: op j at done[ds j] (GemmParams::ds); exit counter done[-kDSMax] and run
                              // number done[-2 kDSMax] at fixed places: chains of every M that share a workspace share them
#ifndef W4_MA_GROUPS
#define W4_MA_GROUPS 2
#endif
constexpr int kGroups = W4_MA_GROUPS;              // consumer groups sharing one pipeline (1 CTA per SM at 2)
constexpr int kWarps = 8 * kGroups;                // per group: 4 row-quarters x 2 k-halves
constexpr int kProducerWarp = kWarps;
#ifndef W4_MA_PUB
#define W4_MA_PUB 1   // a publisher warp issues the counter increments (fence + red) for the storing warps
#endif
static_assert(W4_MA_PUB == 1, "the chain protocol and ALLREDUCE ops run on the publisher warp");
// Publisher warp (W4_MA_PUB): the release of a tile / op counter costs the issuing thread a GPU-scope fence
// (~1 us under load); the storing warps hand the increment to this warp through a shared-memory ring and
// go straight on to the next units.
template <bool kScaleInA>
__host__ __device__ constexpr int pub_warp() { return kWarps + 1; }
template <bool kScaleInA>
constexpr int threads_for() { return (pub_warp<kScaleInA>() + (W4_MA_PUB ? 1 : 0)) * 32; }
constexpr int kPubSlots = 8;
constexpr int kPubAllReduce = -0x40000000;   // publisher request: run ALLREDUCE op (ptr = its ChainJob)
// Units per consumer group and pipeline stage. It must be the same for every token-block class: the group
// split of a stage's units fixes the fp32 summation order, and results are batch-invariant over M = 1..16.
// (3 at M <= 8 alone: gate-up 54.3 -> 52.1 us and the chain -1.6 %, but M = 16 is faster with 2 and
// splitting the classes broke the invariance; an M-independent pairing with 3 was slower — DESIGN.md §5.1.)
#ifndef W4_MA_UPG1
#define W4_MA_UPG1 2
#endif
#ifndef W4_MA_UPG2
#define W4_MA_UPG2 W4_MA_UPG1
#endif
__host__ __device__ constexpr int kR_for(int ntb) { return (ntb == 1 ? W4_MA_UPG1 : W4_MA_UPG2) * kGroups; }
#ifndef W4_POLL_ACQ
#define W4_POLL_ACQ 0   // A/B only: poll tile flags with one acquire load each (round 1-2 behaviour)
#endif
#ifndef W4_MA_CNTREL
#define W4_MA_CNTREL 1   // split-tile counters released by the storing thread instead of the publisher warp
#endif
#ifndef W4_MA_DONEREL
#define W4_MA_DONEREL 1   // op counts released by the storing thread instead of the publisher warp
#endif
#ifndef W4_MA_WPRE
#define W4_MA_WPRE 1   // consumers: load the WAR op count at the op start (-0.8 % at M = 8)
#endif
#ifndef W4_MA_MAXST
#define W4_MA_MAXST 12   // ring stages cap (as many as fit up to this)
#endif
#ifndef W4_MA_ROT
#define W4_MA_ROT 1   // M <= 8: the two consumer groups take turns owning a flush (combine, store, publish; -0.6 %)
#endif
#ifndef W4_MA_FLAGREL
#define W4_MA_FLAGREL 1   // tile-ready flags released by the storing thread (st.release.gpu) instead of the publisher warp (+0.5 %)
#endif
#ifndef W4_MA_RT
#define W4_MA_RT 1   // 16-row MMA tiles per consumer warp at M <= 8 (2: 4 warps per unit; measured slower)
#endif
#ifndef W4_MA_CTAS
#define W4_MA_CTAS 2
#endif
constexpr int kCtasPerSm = kGroups >= 2 ? 1 : W4_MA_CTAS;   // resident CTAs per SM
constexpr int kSmemBudget = kCtasPerSm == 1 ? 227 * 1024 - 512 : (kCtasPerSm == 2 ? 112 : 74) * 1024;   // 512 B static

static_assert(!W4_MA_ROT || (W4_MA_CNTREL && W4_MA_DONEREL && W4_MA_FLAGREL),
              "a rotating flush owner must not use the publisher ring (thread 0's)");
template <int NTB, bool SYM, bool kA8 = false>
struct Cfg {
  static constexpr int kMpad = 8 * NTB;                           // token rows per TMA box
  static constexpr int kTB = SYM ? 8448 : 8704;
  static constexpr int kXBox = kMpad * 128;                       // one SW128 box: 64 fp16 k (or 128 int8 k) x kMpad rows
  static constexpr int kBPU = kA8 ? 1 : 2;                        // activation boxes per unit (128 k)
  static constexpr int kXUnit = kBPU * kXBox;
  static constexpr int kR = kR_for(NTB);                          // units per pipeline stage
  static constexpr int kStage = (kR * (kXUnit + kTB) + 1023) / 1024 * 1024;
  // consumer geometry (the kWarps = 16 consumer warps): kRT 16-row MMA tiles per warp, kGW warps per unit
  // group, kNG groups, kUPG units per group and stage (W4_MA_RT: row tiles per warp at NTB = 1)
  static constexpr int kRT = NTB == 1 ? W4_MA_RT : 1;
  static constexpr int kGW = 8 / kRT;
  static constexpr int kNG = kWarps / kGW;
  static constexpr int kUPG = kR / kNG;
  static_assert(kUPG * kNG == kR && kGW * kRT == 8, "consumer geometry");
  static constexpr int kRedSlots = kNG == 4 ? 2 : 1;               // group sums combined through shared memory
  static constexpr int kRedFloats = kRedSlots * 8 * NTB * 4 * 32;   // [slot][row tile][tb][e][lane]
  static constexpr int kXchBytes = 4 * NTB * 4 * 32 * 4;          // SiLU epilogue: up values of a tile (fp16 in u32)
  static constexpr int kStagesFit = (kSmemBudget - kRedFloats * 4 - kXchBytes - 1024) / kStage;
  static constexpr int kStages = kStagesFit > W4_MA_MAXST ? W4_MA_MAXST : kStagesFit;
  static constexpr int kSmem = kStages * kStage + kRedFloats * 4 + kXchBytes + 1024;
};

// A single w4a16_gemm is a one-op list whose fields come from GemmParams and the kernel's tensor-map
// parameters; a chain's ops are w4::ChainJob entries (common.cuh).
using w4::ChainJob;
using w4::kOpGemm;
using w4::kOpSilu;
using w4::kOpAllReduce;

struct GemmParams {
  const uint8_t* packed;
  uint16_t* Y;
  float* partials;   // [slots][G][8 row groups][NTB][32 lanes] float4 (a CTA publishes at most its first segment per op)
  int* counters;     // tile counters: [N/128] (single GEMM) or per op at ChainJob::cnt_off (chain)
  int M, K, N;
  int Gk;            // K / 128 groups per n-tile
  int U;             // total units
  int G;             // CTAs
  int dbg;           // diagnostics only (W4A16_MMA_DEBUG, W4A16_MMA_DIAG builds): bit0 skip compute, bit1 skip loads, bit2 backoff waits, bit4 trace
  const ChainJob* jobs;   // chain: the op table (device); nullptr: single GEMM
  int n_jobs;             // 1 for a single GEMM
  int* done;              // chain: [n_jobs] CTAs that finished each op (stride ds); done[-2 kDSMax] = run number,
                          // done[-kDSMax] = exit counter
  int ds;                 // chain: op-count stride in ints (32 = one 128-B line each at M <= 8: -1.9 %; 1 at
                          // M = 9..16, where the spread layout measured +2 %)
                          // (fixed offsets: chains that share a workspace share them)
  int* flags;             // chain: tile-ready flags (one per tile of every GEMM op, at the op's cnt_off): the run
                          // number + 1 of the last run that wrote the tile's Y (run number at done[n_jobs + 1])
  int slots;              // chain: partial-slot ring length in ops (1 for a single GEMM)
  const float* sx;        // W4A8 (kA8): per-token activation scales [M]
  int ldx;                // host only: X row stride in elements (0 = K), read when the X tensor maps are encoded
};

struct JobInfo {
  const uint8_t* packed;
  uint16_t* Y;
  const CUtensorMap* mR;
  const CUtensorMap* m1;
  int* counters;
  int* flags;             // this op's tile-ready flags (chain) or nullptr
  int kind, N, Gk, U, dep_x, dep_y, xf_off, pub_tiles, epi, xf_mul;
  int ar;                 // chain: Y is the partial of the ALLREDUCE op right after this GEMM (tile bumps)
  int cs;                 // counter / flag stride (1: single GEMM; 2: chain, counters and flags interleaved)
};
__device__ __forceinline__ JobInfo job_at(const GemmParams& p, const CUtensorMap* mR, const CUtensorMap* m1, int j) {
  JobInfo J;
  if (p.jobs == nullptr) {
    J.packed = p.packed; J.Y = p.Y; J.mR = mR; J.m1 = m1; J.counters = p.counters; J.flags = nullptr; J.cs = w4::kCounterStride;
    J.kind = kOpGemm; J.N = p.N; J.Gk = p.Gk; J.U = p.U; J.dep_x = -1; J.dep_y = -1; J.xf_off = -1; J.pub_tiles = 0; J.epi = 0; J.xf_mul = 1; J.ar = 0;
  } else {
    const ChainJob* c = p.jobs + j;
    // chain: tile counter and tile-ready flag interleaved per tile (same layout in every chain that shares the
    // workspace, so one chain's flags never land on another's counters)
    J.packed = c->packed; J.Y = c->Y; J.mR = &c->xmapR; J.m1 = &c->xmap1; J.counters = p.counters + kCS * c->cnt_off;
    J.flags = J.counters + kFO;
    J.cs = kCS;
    J.kind = c->kind; J.N = c->N; J.Gk = c->Gk; J.U = c->U; J.dep_x = c->dep_x; J.dep_y = c->dep_y; J.xf_off = c->xf_off;
    J.pub_tiles = c->pub_tiles; J.epi = c->epi; J.xf_mul = c->xf_mul; J.ar = c->ar_world > 0;
  }
  return J;
}
// Op j is complete once every CTA has counted it (CTAs walk the ops in order, so op j complete implies
// every earlier op complete).
__device__ __forceinline__ void wait_op(const GemmParams& p, int j) {
  if (j < 0) return;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_gpu(&p.done[p.ds * j]) < p.G) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > 60000000000ull) __trap();   // never hang the device on a protocol bug
  }
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// Tile t of an ALLREDUCE partial is written on this rank (after a system-scope fence): add 1 to tile t's
// counter of the op's slot in every rank's flag area — one multimem.red through the multicast mapping
// (NVLS), else one red per peer mapping.
__device__ __forceinline__ void ar_bump(const ChainJob* cj, int t) {
  if (cj->ar_tiles_mc != nullptr) {
    multimem_red_add_u32(cj->ar_tiles_mc + t, 1u);
  } else {
    for (int q = 0; q < cj->ar_world; ++q) red_relaxed_sys_add_u32(cj->ar_tiles_peer[q] + t, 1u);
  }
}

// Diagnostics only (W4A16_MMA_DEBUG bit 16): per-CTA %globaltimer stamps (entry, first stage ready, main loop
// done, exit) of consumer warp 0 (tools/probe_tc.py --trace-mma).
constexpr int kTraceCtas = 1024;
__device__ unsigned long long g_trace_ma[kTraceCtas][8];
#ifndef W4A16_MMA_DIAG
#define W4A16_MMA_DIAG 0   // 1: compile the per-CTA timeline trace and consumer-side diagnostics in
#endif
// Diagnostics only (W4A16_MMA_DIAG builds, W4A16_MMA_DEBUG bit 64): per CTA and chain op, %globaltimer when
// consumer warp 0 starts the op, has its first stage, finished its last stage, and has counted the op done.
constexpr int kOpTraceCtas = 296, kOpTraceOps = 512;
#if W4A16_MMA_DIAG
__device__ unsigned long long g_op_trace[kOpTraceCtas][kOpTraceOps][8];
// producer side: when the activation load of the op's first stage of this CTA was issued
__device__ unsigned long long g_prod_trace[kOpTraceCtas][kOpTraceOps];
#endif
__device__ __forceinline__ void trace_op(const GemmParams& p, int job, int ev) {
#if W4A16_MMA_DIAG
  if ((p.dbg & 64) && threadIdx.x == 0 && blockIdx.x < kOpTraceCtas && job < kOpTraceOps) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_op_trace[blockIdx.x][job][ev] = t;
  }
#endif
}
__device__ __forceinline__ void trace_ma(const GemmParams& p, int ev) {
  if (W4A16_MMA_DIAG && (p.dbg & 16) && blockIdx.x < kTraceCtas && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace_ma[blockIdx.x][ev] = t;
    if (ev == 0) {
      unsigned int smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_trace_ma[blockIdx.x][7] = smid;
    }
  }
}

// MMA column j (fragment group g8 = j) carries token pi(j) of its 8-token block: with it, the 8 lanes of each
// quarter-warp phase of an activation LDS.128 read rows {r, r + 4}, whose SWIZZLE_128B chunk positions differ
// in the high bit, instead of rows {r, r + 1}, which collide on the same four bank groups (2-way conflict).
#ifndef W4_MA_EXP
#define W4_MA_EXP 0   // cost experiments only (make variant VDEFS=-DW4_MA_EXP=..; WRONG results): bit0 no per-unit
                      // group accumulator / post-scale, bit1 no dequant (raw words as A), bit2 no activation
                      // loads, bit3 no scale/zero loads
#endif
__device__ __forceinline__ int tok_pi(int j) { return (j >> 1) | ((j & 1) << 2); }

__device__ __forceinline__ int unit_begin(int c, int U, int G) { return (int)(((long long)c * U) / G); }
// CTA owning unit u: largest c with unit_begin(c) <= u.
__device__ __forceinline__ int cta_of_unit(int u, int U, int G) {
  return (int)((((long long)(u + 1) * G) + U - 1) / U) - 1;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint16_t lds16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
// W4A8 (kA8): int8 MMA m16n8k32 with signed operands. The 4-bit codes become int8 (q - 8) * 16 with one
// LOP3 per 4 codes: a code's nibble moved to the top of its byte and its bit 3 flipped is (q - 8) * 16 as a
// two's-complement byte (q ^ 8 read as a signed 4-bit number is q - 8). lo8: the low nibbles of the word's
// bytes (code slots 0, 2, 4, 6 = logical k 0, 4, 1, 5 of the word's 8 k), hi8: the high nibbles (k 2, 6, 3, 7).
__device__ __forceinline__ uint32_t a8_lo(uint32_t w) { return ((w << 4) & 0xF0F0F0F0u) ^ 0x80808080u; }
__device__ __forceinline__ uint32_t a8_hi(uint32_t w) { return (w & 0xF0F0F0F0u) ^ 0x80808080u; }
__device__ __forceinline__ uint32_t prmt_b32(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ void mma_s8_16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                             uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Tensor-parallel all-reduce op of a chain (include/w4a16.h W4A16_OP_ALLREDUCE), fused
// with the GEMM that writes the partial P tile by tile and run by the PUBLISHER warp of each CTA in the
// background: when the consumers reach the op they post one request and go straight on to the next GEMM
// (whose activation loads wait for the reduced tiles' ready flags). CTA c reduces 128-column tiles c, c + G,
// ... of P as soon as tile t's counter in this rank's flag area shows every rank's tile for this run (the
// GEMM's tile writers bump it in every rank's flag area, also through the publisher), writes Y's tile and
// publishes its ready flag. No grid-wide wait, and no all-reduce code in the consumers' loop (a call there
// cost ~5% of the chain, measured). Requests are served in order, so the CTA's own bumps precede it.
__device__ __forceinline__ void allreduce_tiles(const GemmParams& p, int job, int cta, int lane) {
  const ChainJob* cj = p.jobs + job;
  const int world = cj->world, tiles = cj->N / 128;
  const int run = __ldcg(&p.done[-2 * kDSMax]);
  const uint32_t want = (uint32_t)world * (__ldcg(cj->epoch) + 1u);   // counters after this run's bumps
  int* yflags = p.counters + kCS * cj->cnt_off + kFO;                 // Y's tile-ready flags (interleaved)
  if (lane == 0 && cj->dep_y >= 0) wait_op(p, cj->dep_y);            // WAR / WAW on Y
  for (int t = cta; t < tiles; t += p.G) {
    if (lane == 0) {
      const unsigned long long t0 = globaltimer_ns();
      while ((int)(ld_acquire_sys(cj->my_tiles + t) - want) < 0) {
        __nanosleep(64);
        if (globaltimer_ns() - t0 > 60000000000ull) __trap();   // a peer never arrived: fail, do not hang
      }
    }
    __syncwarp();
    for (int i = lane; i < p.M * 16; i += 32) {   // M rows x 16 vectors of 8 fp16
      const size_t off = (size_t)(i >> 4) * cj->N + (size_t)t * 128 + (size_t)(i & 15) * 8;
      uint4 r;
      if (cj->mc_x != nullptr) {
        r = multimem_ld_reduce_f16x8(cj->mc_x + off);
      } else {
        float a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = 0.f;
        for (int q = 0; q < world; ++q) {   // rank order: the same sum on every rank
          const uint4 v = __ldcg(reinterpret_cast<const uint4*>(cj->peer_x[q] + off));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
            a[2 * k] += f.x;
            a[2 * k + 1] += f.y;
          }
        }
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __half2 h = __floats2half2_rn(a[2 * k], a[2 * k + 1]);
          o[k] = *reinterpret_cast<const uint32_t*>(&h);
        }
        r = make_uint4(o[0], o[1], o[2], o[3]);
      }
      *reinterpret_cast<uint4*>(cj->Y + off) = r;
    }
    __syncwarp();
    if (lane == 0 && cj->pub_tiles)
      asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.b32 [%0], %1;" ::"l"(yflags + kCS * t), "r"(run + 1) : "memory");
  }
  __syncwarp();
  if (lane == 0) red_release_gpu_add(&p.done[p.ds * job], 1);
}

template <int NTB, bool SYM, bool kScaleInA, bool kA8>
__global__ void __launch_bounds__(threads_for<kScaleInA>(), kCtasPerSm) gemm_w4a16_mma_kernel(const __grid_constant__ CUtensorMap xmapR,
                                                                      const __grid_constant__ CUtensorMap xmap1,
                                                                      const GemmParams p) {
  using C = Cfg<NTB, SYM, kA8>;
  constexpr int S = C::kStages;
  static_assert(S <= 16, "producer queue holds at most 16 stages");
  // kScaleInA (family W4A16_FAMILY_MMA_SYNC_S): scale inside the A fragments instead of a per-unit group
  // accumulator — fewer registers (NTB = 2 runs at the 96-register cap of 18 warps/SM), 4 more HMUL2 per
  // word. Post-scale (family W4A16_FAMILY_MMA_SYNC) is faster when registers allow (NTB = 1).
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[S];
  __shared__ __align__(8) uint64_t empty_bar[S];
  __shared__ __align__(8) uint64_t pub_full[kPubSlots], pub_empty[kPubSlots];
  __shared__ int* pub_ptr[kPubSlots];
  __shared__ int pub_val[kPubSlots];   // 0: add 1 (counters); else store this value (tile-ready flags)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const bool chain = p.jobs != nullptr;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t smem_base = smem_u32(smem);
  float* red = reinterpret_cast<float*>(smem + S * C::kStage);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], kWarps); }
    for (int s = 0; s < kPubSlots; ++s) { mbar_init(&pub_full[s], 1); mbar_init(&pub_empty[s], 1); }
    fence_mbar_init();
    pdl_launch_dependents();   // the next GEMM's CTAs may take SMs as this grid's CTAs retire
  }
  __syncthreads();

  if (warp == kProducerWarp) {
    // ---------------- producer ----------------
    // Per stage ONE bulk copy of the packed weights (the TMA engine costs ~100+ cycles per issued copy)
    // and a 3-D TMA of the activation slices. Weights never depend on an earlier kernel or op, so they are
    // issued as soon as a ring slot frees; a stage's activations wait in a queue until they may be read
    // (after griddepcontrol.wait for a single GEMM; after the producing op's completion in a chain), so the
    // weight stream runs ahead across op boundaries.
    if (lane == 0) {
      if (!chain) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmapR)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap1)) : "memory");
      }
      const uint64_t pol = policy_evict_first();
      int q_s[16], q_j[16], q_u0[16], q_nu[16];   // stages whose activations are not issued yet (FIFO)
      int q_head = 0, q_n = 0, ok_upto = -1;
      bool pdl_done = chain;                 // a chain is not launched with PDL
      auto issue_x = [&](int s, const JobInfo& J, int u0, int nu) {
        const int g0 = u0 % J.Gk;
        const uint32_t st = smem_base + s * C::kStage;
        if (nu == C::kR && g0 + C::kR <= J.Gk) {
          tma_3d(st, J.mR, 0, 0, C::kBPU * g0, &full_bar[s]);
        } else {
          for (int jj = 0; jj < nu; ++jj) tma_3d(st + jj * C::kXUnit, J.m1, 0, 0, C::kBPU * ((u0 + jj) % J.Gk), &full_bar[s]);
        }
      };
      const int run = chain ? __ldcg(&p.done[-2 * kDSMax]) : 0;   // this launch's run number (tile flags)
      // Tile-level dependency: the stage's activation k-groups are complete once the producing op's tiles
      // xf_off + g are written in this run (their flags reached run + 1).
      // The flags are polled with relaxed loads, all in flight at once (an acquire per flag would serialise
      // them: one L2 round trip each, several us per poll); one acquire fence once all are set.
      auto tiles_ready = [&](const JobInfo& J, int u0, int nu) {
        int g = u0 % J.Gk;
        bool ok = true;
        for (int jj = 0; jj < nu; ++jj) {
          for (int i = 0; i < J.xf_mul; ++i)
            ok &= (W4_POLL_ACQ ? ld_acquire_gpu(&p.counters[kCS * (J.xf_off + J.xf_mul * g + i) + kFO])
                               : ld_relaxed_gpu(&p.counters[kCS * (J.xf_off + J.xf_mul * g + i) + kFO])) > run;
          if (++g == J.Gk) g = 0;
        }
        if (ok) fence_acquire_gpu();
        return ok;
      };
      auto drain = [&](bool block) {   // issue queued activation loads whose producers are done
        while (q_n > 0) {
          if (!pdl_done) {
            if (!block) return;
            pdl_wait();
            pdl_done = true;
          }
          const JobInfo J = job_at(p, &xmapR, &xmap1, q_j[q_head]);
          if (J.dep_x > ok_upto) {
            if ((W4_POLL_ACQ ? ld_acquire_gpu(&p.done[p.ds * J.dep_x]) : ld_relaxed_gpu(&p.done[p.ds * J.dep_x])) >= p.G) {
              if (!W4_POLL_ACQ) fence_acquire_gpu();
              ok_upto = J.dep_x;   // the whole producing op is complete: no more per-tile checks
            } else if (J.xf_off >= 0) {
              if (!tiles_ready(J, q_u0[q_head], q_nu[q_head])) {
                if (!block) return;
                const unsigned long long t0 = globaltimer_ns();
                while (!tiles_ready(J, q_u0[q_head], q_nu[q_head])) {
                  __nanosleep(64);
                  if (globaltimer_ns() - t0 > 60000000000ull) __trap();   // never hang the device
                }
              }
            } else {
              if (!block) return;
              wait_op(p, J.dep_x);
              ok_upto = J.dep_x;
            }
            fence_proxy_async_global();   // generic-proxy stores of other CTAs -> this TMA (async proxy) read
          }
#if W4A16_MMA_DIAG
          if ((p.dbg & 64) && cta < kOpTraceCtas && q_j[q_head] < kOpTraceOps && g_prod_trace[cta][q_j[q_head]] == 0)
            g_prod_trace[cta][q_j[q_head]] = globaltimer_ns();
#endif
          issue_x(q_s[q_head], J, q_u0[q_head], q_nu[q_head]);
          q_head = (q_head + 1) & 15;
          --q_n;
        }
      };
      int s = 0, issued = 0;
      uint32_t ph = 0;
      for (int j = 0; j < p.n_jobs; ++j) {
        const JobInfo J = job_at(p, &xmapR, &xmap1, j);
        if (J.kind != kOpGemm) continue;
        const int u_begin = unit_begin(cta, J.U, p.G), u_end = unit_begin(cta + 1, J.U, p.G);
        for (int u0 = u_begin; u0 < u_end; u0 += C::kR) {
          const int nu = min(C::kR, u_end - u0);
          if (issued >= S) {   // slot s must be released by the consumers first
            if (!pdl_done) drain(true);
            while (!mbar_test_wait(&empty_bar[s], ph ^ 1)) drain(false);
          }
          if (W4A16_MMA_DIAG && (p.dbg & 2)) {   // diagnostics: no memory traffic, stale shared memory
            mbar_arrive(&full_bar[s]);
            ++issued;
            if (++s == S) { s = 0; ph ^= 1; }
            continue;
          }
          mbar_expect_tx(&full_bar[s], nu * (C::kXUnit + C::kTB));
          bulk_g2s(smem + s * C::kStage + C::kR * C::kXUnit, J.packed + (size_t)u0 * C::kTB, nu * C::kTB, &full_bar[s], pol);
          const int e = (q_head + q_n) & 15;
          q_s[e] = s; q_j[e] = j; q_u0[e] = u0; q_nu[e] = nu;
          ++q_n;
          drain(false);
          ++issued;
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
      drain(true);
    }
    return;
  }

  if (W4_MA_PUB && warp == pub_warp<kScaleInA>()) {
    // ---------------- publisher ----------------
    // Requests arrive in order from thread 0 (after a barrier of the threads whose stores they publish):
    // mbarrier release/acquire (CTA scope) hands those stores to this warp; its GPU-scope fence + relaxed
    // red then releases them to the CTAs that acquire the counter. nullptr ends the kernel's requests.
    // Requests that queue up while a fence is in flight are issued together behind ONE fence (a GPU-scope
    // fence costs ~1 us under load; op counts, tile counters and tile-ready flags all come through here).
    int slot = 0, ar_prev_done = -1;
    uint32_t ph = 0;
    for (;;) {
      mbar_wait(&pub_full[slot], ph);
      int n = 1;   // consecutive full slots (at most kPubSlots)
      {
        int s2 = slot + 1 == kPubSlots ? 0 : slot + 1;
        uint32_t p2 = s2 == 0 ? ph ^ 1 : ph;
        while (n < kPubSlots && mbar_test_wait(&pub_full[s2], p2)) {
          ++n;
          if (++s2 == kPubSlots) { s2 = 0; p2 ^= 1; }
        }
      }
      bool stop = false;
      // ALLREDUCE tile bumps (val < 0, ptr = the GEMM's ChainJob, tile -val - 1) go to other GPUs: they need a
      // system-scope fence, and the chain's previous ALLREDUCE must be complete on this rank first
      bool sys = false;
      {
        int s2 = slot;
        for (int i = 0; i < n; ++i) {
          if (pub_ptr[s2] && pub_val[s2] < 0 && pub_val[s2] != kPubAllReduce) {
            sys = true;
            const ChainJob* cj = reinterpret_cast<const ChainJob*>(pub_ptr[s2]);
            if (lane == 0 && cj->ar_prev > ar_prev_done) { wait_op(p, cj->ar_prev); ar_prev_done = cj->ar_prev; }
          }
          if (++s2 == kPubSlots) s2 = 0;
        }
      }
      if (lane == 0) {
        if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      for (int i = 0; i < n; ++i) {
        int* ptr = pub_ptr[slot];
        const int val = pub_val[slot];
        if (ptr && val == kPubAllReduce) {
          // the whole warp reduces this CTA's tiles of the ALLREDUCE op (requests before it are published)
          const int job = (int)(reinterpret_cast<const ChainJob*>(ptr) - p.jobs);
          if (lane == 0) mbar_arrive(&pub_empty[slot]);
          allreduce_tiles(p, job, cta, lane);
        } else if (lane == 0) {
          if (ptr && val == 0) asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(ptr) : "memory");
          if (ptr && val > 0) asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(ptr), "r"(val) : "memory");
          if (ptr && val < 0) ar_bump(reinterpret_cast<const ChainJob*>(ptr), -val - 1);
          mbar_arrive(&pub_empty[slot]);
        }
        stop |= ptr == nullptr;
        if (++slot == kPubSlots) { slot = 0; ph ^= 1; }
      }
      __syncwarp();
      if (stop) break;
    }
    return;
  }

  // ---------------- consumers ----------------
  trace_ma(p, 0);
  const int run_c = chain ? __ldcg(&p.done[-2 * kDSMax]) : 0;   // this launch's run number (tile-ready flags)
  int pub_s = 0;
  uint32_t pub_ph = 0;
  // thread 0 only, after a barrier of the threads whose global stores the increment releases
  auto publish = [&](int* ptr, int val = 0) {
    mbar_wait(&pub_empty[pub_s], pub_ph ^ 1);   // the slot's previous request is consumed
    pub_ptr[pub_s] = ptr;
    pub_val[pub_s] = val;
    mbar_arrive(&pub_full[pub_s]);
    if (++pub_s == kPubSlots) { pub_s = 0; pub_ph ^= 1; }
  };
  pdl_wait();   // Y / workspace writes must follow the preceding kernel (returns at once when satisfied)
  const int g8 = lane >> 2, c4 = lane & 3;   // mma fragment coordinates
  // Unit groups: kNG groups of kGW warps; group grp computes kUPG units of every kR-unit stage
  // (units kUPG grp ..), warp wg of the group owns the kRT 16-row MMA tiles rt = kRT wg .. kRT wg + kRT - 1
  // (tile rows 16 rt .. 16 rt + 15) and all 128 k of those units. At NTB = 1 a warp owns two row tiles: the
  // activation fragments it loads feed twice the MMAs, and the two row tiles are independent MMA chains.
  constexpr int kRT = C::kRT, kGW = C::kGW, kNG = C::kNG, kUPG = C::kUPG;
  const int wg = warp % kGW, grp = warp / kGW;

  float acc[kRT][NTB][4];
  int n_fl = 0, last_og = 0;   // flushes so far; the group that owned the last one (W4_MA_ROT)
  int s = 0;
  uint32_t ph = 0;
  const uint32_t ready_base = smem_u32(&full_bar[0]);
  const uint32_t empty_base = smem_u32(&empty_bar[0]);
  const bool skip_compute = W4A16_MMA_DIAG && (p.dbg & 1);   // diagnostics only

  for (int job = 0; job < p.n_jobs; ++job) {
    trace_op(p, job, 0);
    const JobInfo J = job_at(p, &xmapR, &xmap1, job);
    if (W4A16_MMA_DIAG && (p.dbg & 64)) {   // diagnostics: when the descriptor has arrived
      volatile int sink = J.U + J.Gk;
      (void)sink;
      trace_op(p, job, 7);
    }
    if (J.kind == kOpSilu) {
      // SiLU*mul op of a chain (same arithmetic as w4a16_silu_mul), spread over every consumer thread of
      // every CTA once the gate-up op that writes GU (and the readers of `out`) are done.
      if (threadIdx.x == 0) wait_op(p, max(J.dep_x, J.dep_y));
      named_bar_sync(1, kWarps * 32);
      trace_op(p, job, 1);
      const int F = J.N, vecs = F / 8;
      const long long total = (long long)p.M * vecs;
      const uint16_t* GU = reinterpret_cast<const uint16_t*>(J.packed);
      for (long long i = (long long)cta * (kWarps * 32) + threadIdx.x; i < total; i += (long long)p.G * (kWarps * 32)) {
        const int m = (int)(i / vecs), v = (int)(i % vecs);
        const uint4 g = __ldcg(reinterpret_cast<const uint4*>(GU + (size_t)m * 2 * F + (size_t)v * 8));
        const uint4 u = __ldcg(reinterpret_cast<const uint4*>(GU + (size_t)m * 2 * F + F + (size_t)v * 8));
        *reinterpret_cast<uint4*>(J.Y + (size_t)m * F + (size_t)v * 8) = silu_mul_vec(g, u);
      }
      named_bar_sync(1, kWarps * 32);
      if (threadIdx.x == 0) publish(&p.done[p.ds * job]);
      trace_op(p, job, 2);
      trace_op(p, job, 3);
      continue;
    }
    if (J.kind == kOpAllReduce) {   // run by this CTA's publisher warp (allreduce_tiles)
      if (threadIdx.x == 0) publish(reinterpret_cast<int*>(const_cast<ChainJob*>(p.jobs + job)), kPubAllReduce);
      continue;
    }
    const int u_begin = unit_begin(cta, J.U, p.G), u_end = unit_begin(cta + 1, J.U, p.G);
    const int n_stages = (u_end - u_begin + C::kR - 1) / C::kR;
    int cur_t = -1, seg_u0 = u_begin, boundary = 0;
    bool first_segment = true;
    // Y writes (and this op's partial slot) wait for the earlier ops that read / write the same buffers.
    const int wdep = chain ? max(J.dep_y, job - p.slots) : -1;
    bool y_ready = wdep < 0;
    // the WAR / WAW op count is loaded now and looked at by the first flush (its L2 round trip hides under the
    // op's stages instead of stalling the flush)
    const int wdep_v = (W4_MA_WPRE && threadIdx.x % (kGW * 32) == 0 && wdep >= 0) ? ld_relaxed_gpu(&p.done[p.ds * wdep]) : 0;
    float4* part = reinterpret_cast<float4*>(p.partials) + (size_t)(job % p.slots) * p.G * (8 * NTB * 32);

    auto flush = [&](int t, int sg0, int sg1) {
      // the group that combines, stores and publishes this tile: alternates flush by flush (W4_MA_ROT), so
      // the epilogue work is shared between the groups (a + b == b + a: the result is bit-identical)
      const int og = (W4_MA_ROT && kNG == 2 && NTB == 1 && !J.ar) ? (n_fl & 1) : 0;
      const int lead = og * kGW * 32;
      ++n_fl;
      last_og = og;
      if (!y_ready) {
        if (threadIdx.x == lead) {   // released to the other warps by the barrier below
          if (W4_MA_WPRE && wdep_v >= p.G) fence_acquire_gpu();
          else wait_op(p, wdep);
        }
        y_ready = true;
      }
      // 1. combine the unit groups through shared memory, in a fixed order: ((g0 + g1) + (g2 + g3))
      auto red_put = [&](int slot) {
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb)
#pragma unroll
            for (int e = 0; e < 4; ++e) red[(((slot * 8 + kRT * wg + i) * NTB + tb) * 4 + e) * 32 + lane] = acc[i][tb][e];
      };
      auto red_add = [&](int slot) {
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][tb][e] += red[(((slot * 8 + kRT * wg + i) * NTB + tb) * 4 + e) * 32 + lane];
      };
      if (kNG == 2) {
        if (grp != og) red_put(0);
        named_bar_sync(1, kWarps * 32);
        if (grp == og) red_add(0);
      } else {
        if (grp & 1) red_put(grp >> 1);   // g1 -> slot 0, g3 -> slot 1
        named_bar_sync(1, kWarps * 32);
        if (!(grp & 1)) red_add(grp >> 1);   // g0 += g1, g2 += g3
        named_bar_sync(1, kWarps * 32);
        if (grp == 2) red_put(0);
        named_bar_sync(1, kWarps * 32);
        if (grp == 0) red_add(0);
      }
      named_bar_sync(1, kWarps * 32);
      if (grp != og) return;
      // 2. the group-0 warps own the result
      const int tile_u0 = t * J.Gk, tile_u1 = tile_u0 + J.Gk;
      auto store = [&](float (&v)[kRT][NTB][4]) {
        if (J.epi == 1) {
          // SiLU*mul epilogue (W4A16_OP_GEMM_SILU): tile rows 0..63 (row tiles 0..3) are gate, 64..127 the
          // matching up columns; the up warps hand their fp16-rounded values to the gate warps through a
          // shared-memory area of their own (the other groups may already be writing `red` for their next
          // flush), and the gate warps write Y[m][64 t + row] = fp16(silu(g) * u) — w4a16_silu_mul's arithmetic
          uint32_t* xch = reinterpret_cast<uint32_t*>(smem + S * C::kStage + C::kRedFloats * 4);
          const bool up = wg >= kGW / 2;
          if (up) {
#pragma unroll
            for (int i = 0; i < kRT; ++i)
#pragma unroll
              for (int tb = 0; tb < NTB; ++tb)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  xch[(((kRT * wg + i - 4) * NTB + tb) * 4 + e) * 32 + lane] = __half_as_ushort(__float2half_rn(v[i][tb][e]));
          }
          named_bar_sync(2, kGW * 32);
          if (!up) {
            const int Nh = J.N / 2;
#pragma unroll
            for (int i = 0; i < kRT; ++i) {
              const int rt = kRT * wg + i, c0 = t * 64 + 16 * rt + g8, c1 = c0 + 8;
#pragma unroll
              for (int tb = 0; tb < NTB; ++tb)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float g = __half2float(__float2half_rn(v[i][tb][e]));
                  const float u = __half2float(__ushort_as_half((uint16_t)xch[((rt * NTB + tb) * 4 + e) * 32 + lane]));
                  const int m = tb * 8 + c4 + 4 * (e & 1);
                  if (m < p.M) J.Y[(size_t)m * Nh + ((e >> 1) ? c1 : c0)] = __half_as_ushort(__float2half_rn(g / (1.0f + __expf(-g)) * u));
                }
            }
          }
          named_bar_sync(2, kGW * 32);   // xch is reused by the next flush
          return;
        }
        if constexpr (kA8) {   // the token scale (and the 1/16 of the (q - 8) * 16 codes), once per tile sum
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb) {
            const int m0 = tb * 8 + c4, m1 = m0 + 4;
            const float s0 = m0 < p.M ? __ldg(p.sx + m0) * 0.0625f : 0.f, s1 = m1 < p.M ? __ldg(p.sx + m1) * 0.0625f : 0.f;
#pragma unroll
            for (int i = 0; i < kRT; ++i) {
              v[i][tb][0] *= s0; v[i][tb][2] *= s0;
              v[i][tb][1] *= s1; v[i][tb][3] *= s1;
            }
          }
        }
#pragma unroll
        for (int i = 0; i < kRT; ++i) {
          const int n0 = t * kTileN + 16 * (kRT * wg + i) + g8, n1 = n0 + 8;
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb) {
            const int m0 = tb * 8 + c4, m1 = m0 + 4;   // MMA columns 2c4, 2c4 + 1 = tokens tok_pi(2c4), tok_pi(2c4 + 1)
            if (m0 < p.M) {
              J.Y[(size_t)m0 * J.N + n0] = __half_as_ushort(__float2half_rn(v[i][tb][0]));
              J.Y[(size_t)m0 * J.N + n1] = __half_as_ushort(__float2half_rn(v[i][tb][2]));
            }
            if (m1 < p.M) {
              J.Y[(size_t)m1 * J.N + n0] = __half_as_ushort(__float2half_rn(v[i][tb][1]));
              J.Y[(size_t)m1 * J.N + n1] = __half_as_ushort(__float2half_rn(v[i][tb][3]));
            }
          }
        }
      };
      auto tile_written = [&]() {   // chain: the tile's Y is complete -> its ready flag (tile-level deps)
        if (!chain || (!J.pub_tiles && !J.ar)) return;
        named_bar_sync(2, kGW * 32);
        if (W4_MA_FLAGREL) {   // the tile-ready flag released by this thread (no queue behind the publisher's fences)
          if (threadIdx.x == lead && J.pub_tiles)
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(&J.flags[J.cs * t]), "r"(run_c + 1) : "memory");
        } else if (threadIdx.x == lead && J.pub_tiles) {
          publish(&J.flags[J.cs * t], run_c + 1);
        }
        // Y is an ALLREDUCE's partial: bump tile t's counter in every rank's flag area (publisher warp)
        if (threadIdx.x == 0 && J.ar) publish(reinterpret_cast<int*>(const_cast<ChainJob*>(p.jobs + job)), -t - 1);
      };
      if (sg0 == tile_u0 && sg1 == tile_u1) { store(acc); tile_written(); return; }
      // Split tile: the tile's first CTA c_first owns it. It handles the tile's head as its
      // LAST segment of the op, so it finishes after every other contributor has long published its
      // (first-segment) fp32 partial: contributors store, then release-increment the tile counter and move
      // on (no round trip); the owner acquires the counter, adds the partials in CTA order to its own and
      // writes Y. All G CTAs are co-resident (G = resident capacity), so the owner's wait always completes.
      const int c_first = cta_of_unit(tile_u0, J.U, p.G), c_last = cta_of_unit(tile_u1 - 1, J.U, p.G);
      auto pidx = [&](int c, int rt, int tb) { return (((size_t)c * 8 + rt) * NTB + tb) * 32 + lane; };
      if (cta != c_first) {
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb)
            __stcg(&part[pidx(cta, kRT * wg + i, tb)], make_float4(acc[i][tb][0], acc[i][tb][1], acc[i][tb][2], acc[i][tb][3]));
        named_bar_sync(2, kGW * 32);
        if (threadIdx.x == lead) {
          // direct at M <= 8 (-0.6 %); at M = 9..16 the publisher's queue is 1 % faster (measured)
          if (W4_MA_CNTREL && NTB == 1) red_release_gpu_add(&J.counters[J.cs * t], 1);
          else publish(&J.counters[J.cs * t]);
        }
        return;
      }
      if (threadIdx.x == lead) {
        const int want = c_last - c_first;
        trace_op(p, job, 4);
        while (ld_acquire_gpu(&J.counters[J.cs * t]) != want) __nanosleep(32);
        trace_op(p, job, 5);
        J.counters[J.cs * t] = 0;   // every contributor has arrived: re-arm for the next launch
      }
      named_bar_sync(2, kGW * 32);
      for (int c = c_first + 1; c <= c_last; ++c) {
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb) {
            const float4 v = __ldcg(&part[pidx(c, kRT * wg + i, tb)]);
            acc[i][tb][0] += v.x; acc[i][tb][1] += v.y; acc[i][tb][2] += v.z; acc[i][tb][3] += v.w;
          }
      }
      store(acc);
      tile_written();
    };

    // One unit: all shared-memory loads first (activation fragments, code words, scale/zero pairs), then
    // dequant + 8 MMAs per row tile (one m16 tile x 8 k-steps), then the post-MMA group scale.
    auto process_unit = [&](uint32_t st, int j) {
      const uint32_t xu = st + j * C::kXUnit;                 // activations of this unit: box b holds k 64b..
      const uint32_t ub = st + C::kR * C::kXUnit + j * C::kTB;   // packed tile of this unit
      if constexpr (kA8) {
        // W4A8 (include/w4a16.h w4a8_gemm; reading R21): int8 activations (one 128-k SW128 box), int8 codes
        // (q - 8) * 16, exact int32 group sums from mma m16n8k32, then the fp32 group scale; the token scale
        // sx[m] / 16 is applied to the tile sum at the store. One MMA per 32-k chunk and row tile.
        uint2 xb[4][NTB];   // [32-k chunk][token block]: the 8 int8 activations k = 32 pc + 8 c4 .. +7
#pragma unroll
        for (int pc = 0; pc < 4; ++pc)
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb) {
            const int m = 8 * tb + tok_pi(g8);
            const int ch = 2 * pc + (c4 >> 1);                    // 16-byte chunk of the 128-byte row
            xb[pc][tb] = lds64(xu + m * 128 + ((ch ^ (m & 7)) << 4) + (c4 & 1) * 8);
          }
#pragma unroll
        for (int i = 0; i < kRT; ++i) {
          const int rt = kRT * wg + i;
          uint32_t wq[4][2];
          const int lr = 16 * rt + 8 * ((lane >> 3) & 1) + (lane & 7);
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {
            const int pch = 2 * pp + (lane >> 4);
            ldsm_x4(ub + lr * 64 + ((pch ^ ((lr >> 1) & 3)) << 4), wq[2 * pp][0], wq[2 * pp][1], wq[2 * pp + 1][0],
                    wq[2 * pp + 1][1]);
          }
          float sc[2];
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) sc[hf] = __half2float(__ushort_as_half(lds16(ub + 8192 + 2 * (16 * rt + g8 + 8 * hf))));
          int iacc[NTB][4];
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb) iacc[tb][0] = iacc[tb][1] = iacc[tb][2] = iacc[tb][3] = 0;
#pragma unroll
          for (int pc = 0; pc < 4; ++pc) {
            const uint32_t a0 = a8_lo(wq[pc][0]), a1 = a8_lo(wq[pc][1]), a2 = a8_hi(wq[pc][0]), a3 = a8_hi(wq[pc][1]);
#pragma unroll
            for (int tb = 0; tb < NTB; ++tb) {
              // B bytes in the A fragments' k order: MMA k 4 c4 + j <-> lo byte j (word k 0, 4, 1, 5), MMA k
              // 16 + 4 c4 + j <-> hi byte j (word k 2, 6, 3, 7)
              const uint32_t b0 = prmt_b32(xb[pc][tb].x, xb[pc][tb].y, 0x5140u);
              const uint32_t b1 = prmt_b32(xb[pc][tb].x, xb[pc][tb].y, 0x7362u);
              mma_s8_16832(iacc[tb], a0, a1, a2, a3, b0, b1);
            }
          }
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][tb][e] = fmaf(sc[e >> 1], (float)iacc[tb][e], acc[i][tb][e]);
        }
        return;
      }
      uint4 xr[4][NTB];                                       // [32-k chunk p][token block]
#pragma unroll
      for (int pc = 0; pc < 4; ++pc)
#pragma unroll
        for (int tb = 0; tb < NTB; ++tb) {
          const int m = 8 * tb + tok_pi(g8);                    // MMA column g8 carries token tok_pi(g8)
          const int jx = 4 * (pc & 1) + c4;                     // chunk pc: k 32 pc + 8 c4 .. +7
          if (W4_MA_EXP & 4) xr[pc][tb] = make_uint4(0x3c003c00u + m, 0x3c003c00u, 0x3c003c00u ^ jx, 0x3c003c00u);
          else xr[pc][tb] = lds128(xu + (pc >> 1) * C::kXBox + m * 128 + ((jx ^ (m & 7)) << 4));
        }
      uint32_t wq[kRT][4][2];                                 // [row tile][chunk][row g / g + 8]
      float sc[kRT][2];
      __half2 zp[kRT][2];
#pragma unroll
      for (int i = 0; i < kRT; ++i) {
        const int rt = kRT * wg + i;
        // Two ldmatrix.x4: matrix q = (hf = q & 1, chunk 2 pp + (q >> 1)) is the 8 rows 16 rt + 8 hf + 0..7 of
        // that chunk, and lane (g8, c4) receives word c4 of row g8 — exactly its code word (conflict-free: the
        // XOR chunk layout spreads the 8 rows over all 32 banks).
        const int lr = 16 * rt + 8 * ((lane >> 3) & 1) + (lane & 7);
#pragma unroll
        for (int pp = 0; pp < 2; ++pp) {
          const int pch = 2 * pp + (lane >> 4);
          ldsm_x4(ub + lr * 64 + ((pch ^ ((lr >> 1) & 3)) << 4), wq[i][2 * pp][0], wq[i][2 * pp][1], wq[i][2 * pp + 1][0],
                  wq[i][2 * pp + 1][1]);
        }
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int r = 16 * rt + g8 + 8 * hf;
          if (SYM) {
            sc[i][hf] = __half2float(__ushort_as_half(lds16(ub + 8192 + 2 * r)));
            zp[i][hf] = __floats2half2_rn(72.f, 1032.f);   // z = 8
          } else if (W4_MA_EXP & 8) {
            sc[i][hf] = 0.01f * (r + 1);
            zp[i][hf] = __floats2half2_rn(72.f, 1032.f);
          } else {
            const __half2 sz = u2h2(lds32(ub + 8192 + 4 * r));   // {s, z}
            sc[i][hf] = __low2float(sz);
            zp[i][hf] = zero_pair(__high2half(sz));
          }
        }
      }
      if constexpr (kScaleInA) {
        // w_hat = fp16((q - z) * s) in the A fragments (exactly the oracle's dequantised weight), accumulated
        // straight into acc: no per-unit group accumulator.
#pragma unroll
        for (int i = 0; i < kRT; ++i) {
          __half2 s2[2];
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) s2[hf] = __float2half2_rn(sc[i][hf]);
#pragma unroll
          for (int pc = 0; pc < 4; ++pc)
#pragma unroll
            for (int hs = 0; hs < 2; ++hs) {
              const uint32_t qa = hs ? wq[i][pc][0] >> 8 : wq[i][pc][0];
              const uint32_t qb = hs ? wq[i][pc][1] >> 8 : wq[i][pc][1];
              const uint32_t a0 = h22u(__hmul2(u2h2(dq_lo(qa, zp[i][0])), s2[0]));
              const uint32_t a1 = h22u(__hmul2(u2h2(dq_lo(qb, zp[i][1])), s2[1]));
              const uint32_t a2 = h22u(__hmul2(u2h2(dq_hi(qa, zp[i][0])), s2[0]));
              const uint32_t a3 = h22u(__hmul2(u2h2(dq_hi(qb, zp[i][1])), s2[1]));
#pragma unroll
              for (int tb = 0; tb < NTB; ++tb) {
                const uint32_t* xv = reinterpret_cast<const uint32_t*>(&xr[pc][tb]);
                mma_16816(acc[i][tb], a0, a1, a2, a3, xv[2 * hs], xv[2 * hs + 1]);
              }
            }
        }
      } else {
        // Post-scale with exact codes: the A fragments hold the integers (q - z) (LOP3 +
        // HSUB2 / HFMA2 per pair, exact in fp16), the MMAs sum sum_k (q_k - z) x_k over the unit's 128 k into
        // a fresh fp32 group accumulator per row tile (independent MMA chains), and the group scale multiplies
        // that sum once: Y += s * sum. This is the exact-weight definition (reading R22); no offsets, so no
        // cancellation whatever the activation magnitude.
        float gacc[kRT][NTB][4];
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb)
#pragma unroll
            for (int e = 0; e < 4; ++e) gacc[i][tb][e] = (W4_MA_EXP & 1) ? acc[i][tb][e] : 0.f;
#pragma unroll
        for (int pc = 0; pc < 4; ++pc)
#pragma unroll
          for (int hs = 0; hs < 2; ++hs)
#pragma unroll
            for (int i = 0; i < kRT; ++i) {
              const uint32_t qa = hs ? wq[i][pc][0] >> 8 : wq[i][pc][0];
              const uint32_t qb = hs ? wq[i][pc][1] >> 8 : wq[i][pc][1];
              const uint32_t a0 = (W4_MA_EXP & 2) ? qa : dq_lo(qa, zp[i][0]), a1 = (W4_MA_EXP & 2) ? qb : dq_lo(qb, zp[i][1]);
              const uint32_t a2 = (W4_MA_EXP & 2) ? qa ^ 0x10001u : dq_hi(qa, zp[i][0]);
              const uint32_t a3 = (W4_MA_EXP & 2) ? qb ^ 0x10001u : dq_hi(qb, zp[i][1]);
#pragma unroll
              for (int tb = 0; tb < NTB; ++tb) {
                const uint32_t* xv = reinterpret_cast<const uint32_t*>(&xr[pc][tb]);
                mma_16816_nv(gacc[i][tb], a0, a1, a2, a3, xv[2 * hs], xv[2 * hs + 1]);
              }
            }
#pragma unroll
        for (int i = 0; i < kRT; ++i)
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb) {
            if (W4_MA_EXP & 1) {
              acc[i][tb][0] = gacc[i][tb][0]; acc[i][tb][1] = gacc[i][tb][1]; acc[i][tb][2] = gacc[i][tb][2]; acc[i][tb][3] = gacc[i][tb][3];
              continue;
            }
            acc[i][tb][0] = fmaf(sc[i][0], gacc[i][tb][0], acc[i][tb][0]);
            acc[i][tb][1] = fmaf(sc[i][0], gacc[i][tb][1], acc[i][tb][1]);
            acc[i][tb][2] = fmaf(sc[i][1], gacc[i][tb][2], acc[i][tb][2]);
            acc[i][tb][3] = fmaf(sc[i][1], gacc[i][tb][3], acc[i][tb][3]);
          }
      }
    };
    auto begin_segment = [&](int u) {
      if (cur_t >= 0) {
        if (first_segment) trace_ma(p, 4);
        flush(cur_t, seg_u0, u);
        if (first_segment) trace_ma(p, 5);
        first_segment = false;
      }
      cur_t = cur_t < 0 ? u / J.Gk : cur_t + 1;
      boundary = (cur_t + 1) * J.Gk;
      seg_u0 = u;
#pragma unroll
      for (int i = 0; i < kRT; ++i)
#pragma unroll
        for (int tb = 0; tb < NTB; ++tb) acc[i][tb][0] = acc[i][tb][1] = acc[i][tb][2] = acc[i][tb][3] = 0.f;
    };
    auto stage_begin = [&](int i) {
      if (W4A16_MMA_DIAG && (p.dbg & 4)) mbar_wait_backoff(&full_bar[s], ph, 32);
      else mbar_wait_a(ready_base + 8 * s, ph);
      if (i == 0) { trace_ma(p, 1); trace_op(p, job, 1); }
    };
    auto stage_end = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive_a(empty_base + 8 * s);
      if (++s == S) { s = 0; ph ^= 1; }
    };
    const int n_full = (u_end - u_begin) / C::kR;   // stages holding C::kR units
    // The consumer group of unit u (offset j in its stage): j / kUPG. The stage size must not depend on M, so
    // each group's units — hence the fp32 summation order — depend on the plan (K, N, SMs) only (batch
    // invariance over M = 1..16).
    auto group_of = [&](int u) { return ((u - u_begin) % C::kR) / kUPG; };
    int i = 0;
    while (i < n_stages) {
      // a stage that starts a segment, crosses a tile boundary or is the ragged last one
      {
        const int u0 = u_begin + i * C::kR, nu = min(C::kR, u_end - u0);
        stage_begin(i);
        const uint32_t st = smem_base + s * C::kStage;
        // every warp walks the stage's units in order (tile flushes are joint); each group computes its own
        for (int j = 0; j < nu; ++j) {
          if (u0 + j == boundary || cur_t < 0) begin_segment(u0 + j);
          if (group_of(u0 + j) == grp && !skip_compute) process_unit(st, j);
        }
        stage_end();
        ++i;
      }
      // then the run of full stages inside the current tile: no per-stage bookkeeping
      const int i_end = min(n_full, (boundary - u_begin) / C::kR);
      for (; i < i_end; ++i) {
        stage_begin(i);
        const uint32_t st = smem_base + s * C::kStage;
        if (!skip_compute) {
#pragma unroll
          for (int j = 0; j < kUPG; ++j) process_unit(st, kUPG * grp + j);
        }
        stage_end();
      }
    }
    trace_ma(p, 2);
    trace_op(p, job, 2);
    if (cur_t >= 0) flush(cur_t, seg_u0, u_end);
    trace_op(p, job, 6);
    trace_ma(p, 3);
    // This CTA's share of the op is written: count it. Only the warps that store Y / partials (group 0) take
    // part; the other warps are already streaming the next op.
    if (chain && grp == last_og) {   // the group of the op's last flush has seen every earlier flush's stores
      named_bar_sync(2, kGW * 32);
      if (threadIdx.x == last_og * kGW * 32) {
        if (W4_MA_DONEREL) red_release_gpu_add(&p.done[p.ds * job], 1);
        else publish(&p.done[p.ds * job]);
      }
    }
    trace_op(p, job, 3);
  }
  if (W4_MA_PUB && threadIdx.x == 0) {
    // end the publisher's requests and wait until it has issued every increment
    const int last = pub_s;
    const uint32_t last_ph = pub_ph;
    publish(nullptr);
    mbar_wait(&pub_empty[last], last_ph);
  }
  if (chain && threadIdx.x == 0) {
    // The last CTA out re-arms the op counters for the next run of the chain (every CTA has finished
    // every access to them once it has counted itself out; the fences order its op counts first).
    __threadfence();
    if (atomicAdd(&p.done[-kDSMax], 1) == p.G - 1) {
      __threadfence();
      for (int j = 0; j < p.n_jobs; ++j) p.done[p.ds * j] = 0;
      p.done[-kDSMax] = 0;
      p.done[-2 * kDSMax] += 1;   // the next run's number (tile-ready flags hold run + 1)
      if (p.jobs[0].epoch != nullptr) *p.jobs[0].epoch += 1u;   // the group's next run (ALLREDUCE flags)
      __threadfence();
    }
  }
}

template <int NTB, bool SYM, bool kScaleInA>
static int launch_t(const uint16_t* X, const GemmParams& p, cudaStream_t stream) {
  using C = Cfg<NTB, SYM, false>;
  CUtensorMap mapR, map1;
  if (int e = encode_x_sw128(&mapR, X, p.M, p.K, C::kMpad, 2 * C::kR, p.ldx)) return e;
  if (int e = encode_x_sw128(&map1, X, p.M, p.K, C::kMpad, 2, p.ldx)) return e;
  auto kern = gemm_w4a16_mma_kernel<NTB, SYM, kScaleInA, false>;
  static unsigned long long attr_set = 0;
  if (!ensure_smem_attr(kern, C::kSmem, attr_set)) return W4A16_ERR_CUDA;
  return launch_pdl(kern, dim3(p.G), dim3(threads_for<kScaleInA>()), C::kSmem, stream, mapR, map1, p) == cudaSuccess ? W4A16_OK
                                                                                             : W4A16_ERR_CUDA;
}

template <int NTB, bool SYM, bool kScaleInA>
static int launch_chain_t(const GemmParams& p, bool cooperative, cudaStream_t stream) {
  using C = Cfg<NTB, SYM, false>;
  auto kern = gemm_w4a16_mma_kernel<NTB, SYM, kScaleInA, false>;
  static unsigned long long attr_set = 0;
  if (!ensure_smem_attr(kern, C::kSmem, attr_set)) return W4A16_ERR_CUDA;
  CUtensorMap unused;
  memset(&unused, 0, sizeof(unused));
  // Cooperative: the owner-reduced tile fixup and the op dependencies need all G CTAs co-resident.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(threads_for<kScaleInA>());
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cooperative ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, unused, unused, p) == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

// W4A8 on the family-A pipeline (SYM blob, int8 activations Xq [M][K] viewed as (128 k, M rows, K/128 boxes)).
template <int NTB>
static int launch_a8_t(const int8_t* Xq, const GemmParams& p, cudaStream_t stream) {
  using C = Cfg<NTB, true, true>;
  auto enc = get_encode();
  if (!enc) return W4A16_ERR_CUDA;
  CUtensorMap maps[2];
  const int depth[2] = {C::kR, 1};
  for (int i = 0; i < 2; ++i) {
    const cuuint64_t dims[3] = {128, (cuuint64_t)p.M, (cuuint64_t)(p.K / 128)};
    const cuuint64_t strides[2] = {(cuuint64_t)p.K, 128};
    const cuuint32_t box[3] = {128, (cuuint32_t)C::kMpad, (cuuint32_t)depth[i]};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&maps[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(Xq), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return W4A16_ERR_CUDA;
  }
  auto kern = gemm_w4a16_mma_kernel<NTB, true, false, true>;
  static unsigned long long attr_set = 0;
  if (!ensure_smem_attr(kern, C::kSmem, attr_set)) return W4A16_ERR_CUDA;
  return launch_pdl(kern, dim3(p.G), dim3(threads_for<false>()), C::kSmem, stream, maps[0], maps[1], p) == cudaSuccess
             ? W4A16_OK : W4A16_ERR_CUDA;
}

constexpr int kChainSlots = 8;   // partial-slot ring of a chain, in ops

inline int ntb_of(int M) { return (M + 7) / 8; }
inline size_t chain_partial_bytes(int M, int G) { return (size_t)kChainSlots * G * 4 * ntb_of(M) * 2 * 32 * 16; }
inline size_t chain_done_bytes(int n_ops) { return ((size_t)(n_ops + 2) * kDSMax * 4 + 255) / 256 * 256; }   // run, exit, per op

}  // namespace ma
}  // namespace w4

extern "C" int w4a16_debug_op_trace(void* host, size_t bytes) {
#if W4A16_MMA_DIAG
  return cudaMemcpyFromSymbol(host, w4::ma::g_op_trace, bytes < sizeof(w4::ma::g_op_trace) ? bytes : sizeof(w4::ma::g_op_trace)) ==
                 cudaSuccess ? 0 : -5;
#else
  (void)host; (void)bytes;
  return -1;
#endif
}

extern "C" int w4a16_debug_prod_trace(void* host, size_t bytes, int clear) {
#if W4A16_MMA_DIAG
  if (clear) {
    static unsigned long long zero[w4::ma::kOpTraceCtas][w4::ma::kOpTraceOps];
    return cudaMemcpyToSymbol(w4::ma::g_prod_trace, zero, sizeof(zero)) == cudaSuccess ? 0 : -5;
  }
  return cudaMemcpyFromSymbol(host, w4::ma::g_prod_trace, bytes < sizeof(w4::ma::g_prod_trace) ? bytes : sizeof(w4::ma::g_prod_trace)) ==
                 cudaSuccess ? 0 : -5;
#else
  (void)host; (void)bytes; (void)clear;
  return -1;
#endif
}

extern "C" int w4a16_debug_trace_mma(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, w4::ma::g_trace_ma, bytes < sizeof(w4::ma::g_trace_ma) ? bytes : sizeof(w4::ma::g_trace_ma)) ==
                 cudaSuccess ? 0 : -5;
}

// Plan (depends on K, N and the SM count only).
extern "C" int w4a16_mma_plan_ctas(int K, int N, int num_sms) {
  const long long U = (long long)(N / w4::ma::kTileN) * (K / w4::ma::kTileK);
  long long G = (long long)w4::ma::kCtasPerSm * num_sms;
  if (G > U) G = U;
  return (int)G;
}

extern "C" size_t w4a16_mma_workspace_bytes(int M, int K, int N, int num_sms) {
  const int ntb = (M + 7) / 8;
  const int G = w4a16_mma_plan_ctas(K, N, num_sms);
  const size_t counters = w4::kCounterBytes;
  return counters + (size_t)G * 4 * ntb * 2 * 32 * 16;
}

// ---- chains (include/w4a16.h) ----
namespace {
int chain_family(int M, int family) {
  if (family == W4A16_FAMILY_AUTO) family = W4A16_FAMILY_MMA_SYNC;
  if (M < 1 || M > 16) return W4A16_ERR_SHAPE;   // chains serve the mma.sync families (M <= 16)
  if (family != W4A16_FAMILY_MMA_SYNC && family != W4A16_FAMILY_MMA_SYNC_S) return W4A16_ERR_ARG;
  return family;
}
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
struct Span { uintptr_t a, b; };
bool overlaps(Span x, Span y) { return x.a < y.b && y.a < x.b; }
bool is_gemm(int kind) { return kind == W4A16_OP_GEMM || kind == W4A16_OP_GEMM_SILU; }
int ldx_of(const w4a16_op& o) { return is_gemm(o.kind) && o.ldx > 0 ? o.ldx : o.K; }
int y_cols(const w4a16_op& o) { return o.kind == W4A16_OP_GEMM_SILU ? o.N / 2 : o.N; }   // Y row stride
Span x_span(const w4a16_op& o, int M) {   // rows of X with their row stride (gaps between rows included)
  const uintptr_t a = reinterpret_cast<uintptr_t>(o.X);
  return {a, a + ((size_t)(M - 1) * (size_t)ldx_of(o) + (size_t)o.K) * 2};
}
Span y_span(const w4a16_op& o, int M) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(o.Y);
  return {a, a + (size_t)M * (size_t)y_cols(o) * 2};
}
// Validate the ops; on success return the number of tile counters and the common mode.
int check_ops(const w4a16_op* ops, int n_ops, int M, int G, long long* tiles, int* mode) {
  if (!ops || n_ops < 1) return W4A16_ERR_ARG;
  long long t = 0;
  int n_ar = 0;
  const w4a16_peer_group* group = nullptr;
  *mode = -1;
  for (int j = 0; j < n_ops; ++j) {
    const w4a16_op& o = ops[j];
    if (!o.X || !o.Y) return W4A16_ERR_ARG;
    if (!al16(o.X) || !al16(o.Y)) return W4A16_ERR_ALIGN;
    if (is_gemm(o.kind)) {
      if (!o.packed || (o.mode != W4A16_ASYM && o.mode != W4A16_SYM)) return W4A16_ERR_ARG;
      if (*mode >= 0 && o.mode != *mode) return W4A16_ERR_ARG;
      *mode = o.mode;
      if (!al16(o.packed)) return W4A16_ERR_ALIGN;
      if (o.K <= 0 || o.N <= 0 || o.K % 128 || o.N % 128 || o.N > W4A16_MAX_N) return W4A16_ERR_SHAPE;
      if (o.ldx != 0 && (o.ldx < o.K || o.ldx % 8)) return W4A16_ERR_SHAPE;
      if ((long long)(o.K / 128) * (o.N / 128) < G) return W4A16_ERR_SHAPE;   // every CTA owns >= 1 unit
      t += o.N / 128;
    } else if (o.kind == W4A16_OP_SILU_MUL) {
      if (o.N < 8 || o.N % 8 || o.K != 2 * o.N) return W4A16_ERR_SHAPE;
    } else if (o.kind == W4A16_OP_ALLREDUCE) {
      if (o.N < 128 || o.N % 128 || o.N / 128 > W4A16_AR_MAX_TILES || o.K != o.N) return W4A16_ERR_SHAPE;
      // fused with the GEMM right before it: X is exactly that GEMM's (plain) Y
      if (j == 0 || ops[j - 1].kind != W4A16_OP_GEMM || ops[j - 1].Y != o.X || ops[j - 1].N != o.N) return W4A16_ERR_ARG;
      const w4a16_peer_group* g = reinterpret_cast<const w4a16_peer_group*>(o.packed);
      if (!g) return W4A16_ERR_ARG;
      if (n_ar == 0) group = g;
      else if (g != group) return W4A16_ERR_ARG;   // one group per chain
      ++n_ar;
      if (g->world < 1 || g->world > W4A16_MAX_PEERS || g->rank < 0 || g->rank >= g->world) return W4A16_ERR_ARG;
      if (g->flag_offset % 256 || g->flag_slots < 1) return W4A16_ERR_ARG;
      if (n_ar > g->flag_slots || g->flag_offset + w4a16_peer_flag_bytes(g->flag_slots) > g->bytes) return W4A16_ERR_ARG;
      if (!g->base[g->rank] || !al16(g->base[g->rank]) || (g->mc_base && !al16(g->mc_base))) return W4A16_ERR_ARG;
      if (!g->mc_base)   // the peer-load path reads every rank's mapping
        for (int q = 0; q < g->world; ++q)
          if (!g->base[q] || !al16(g->base[q])) return W4A16_ERR_ARG;
      const uintptr_t b0 = reinterpret_cast<uintptr_t>(g->base[g->rank]);
      const Span xs = x_span(o, M), flags = {b0 + g->flag_offset, b0 + g->flag_offset + w4a16_peer_flag_bytes(g->flag_slots)};
      if (xs.a < b0 || xs.b > b0 + g->bytes || overlaps(xs, flags)) return W4A16_ERR_ARG;   // P inside the region
      t += o.N / 128;   // Y's tile-ready flags
    } else {
      return W4A16_ERR_ARG;
    }
    if (overlaps(x_span(o, M), y_span(o, M))) return W4A16_ERR_ARG;   // in-place ops are not supported
  }
  // Peers read an ALLREDUCE's X after the op's flags: the next op that writes that buffer (cyclically:
  // every rank runs the chain again) must come after another ALLREDUCE, whose flags prove every peer has
  // finished reading it (include/w4a16.h).
  for (int b = 0; b < n_ops; ++b) {
    if (ops[b].kind != W4A16_OP_ALLREDUCE) continue;
    bool fenced = false;
    for (int d = 1; d <= n_ops; ++d) {
      const w4a16_op& c = ops[(b + d) % n_ops];
      if (overlaps(y_span(c, M), x_span(ops[b], M)) && !fenced) return W4A16_ERR_ARG;
      if (c.kind == W4A16_OP_ALLREDUCE && d < n_ops) fenced = true;
      if (fenced) break;
    }
  }
  if (*mode < 0) *mode = W4A16_ASYM;
  *tiles = t;
  return W4A16_OK;
}
int chain_ctas(int sms) { return w4::ma::kCtasPerSm * sms; }   // the tcgen05 family: one CTA per SM too
}  // namespace


extern "C" size_t w4a16_peer_flag_bytes(int flag_slots) {
  return flag_slots > 0 ? ((size_t)(w4::kFlagHead + (size_t)flag_slots * W4A16_AR_MAX_TILES) * 4 + 255) / 256 * 256 : 0;
}

// Test hook (exported, not in the header): validate a chain's ops (w4a16_chain_plan's checks) without
// encoding tensor maps, so the planner's rules are testable on a machine without a GPU.
extern "C" int w4a16_chain_check_sms(const w4a16_op* ops, int n_ops, int M, int family, int sms) {
  const int fam = chain_family(M, family);
  if (fam < 0) return fam;
  if (sms <= 0) return W4A16_ERR_ARG;
  long long tiles = 0;
  int mode = 0;
  return check_ops(ops, n_ops, M, chain_ctas(sms), &tiles, &mode);
}

extern "C" size_t w4a16_chain_plan_bytes(int n_ops) { return n_ops > 0 ? (size_t)n_ops * sizeof(w4::ma::ChainJob) : 0; }

extern "C" size_t w4a16_chain_workspace_bytes_sms(const w4a16_op* ops, int n_ops, int M, int family, int sms) {
  if (chain_family(M, family) < 0 || sms <= 0) return 0;
  long long tiles = 0;
  int mode = 0;
  const int G = chain_ctas(sms);
  if (check_ops(ops, n_ops, M, G, &tiles, &mode) != W4A16_OK) return 0;
  return w4::ma::chain_partial_bytes(M, G) + w4::ma::chain_done_bytes(n_ops) + (size_t)tiles * w4::ma::kCS * 4;   // counters + flags
}

extern "C" int w4a16_chain_plan_sms(const w4a16_op* ops, int n_ops, int M, int family, void* plan, size_t plan_bytes,
                                    int sms) {
  if (!plan) return W4A16_ERR_ARG;
  const int fam = chain_family(M, family);
  if (fam < 0) return fam;
  if (sms <= 0) return W4A16_ERR_CUDA;
  if (plan_bytes < w4a16_chain_plan_bytes(n_ops)) return W4A16_ERR_ARG;
  long long tiles = 0;
  int mode = 0;
  if (int e = check_ops(ops, n_ops, M, chain_ctas(sms), &tiles, &mode)) return e;
  const int mpad = 8 * w4::ma::ntb_of(M), depth = 2 * w4::ma::kR_for(w4::ma::ntb_of(M));   // activation boxes of the stages
  w4::ma::ChainJob* jobs = reinterpret_cast<w4::ma::ChainJob*>(plan);
  int cnt = 0, ar_slot = 0, last_ar = -1;
  uint32_t* epoch = nullptr;   // the group's run counter, advanced by the last CTA of every run
  for (int j = 0; j < n_ops; ++j) {
    const w4a16_op& o = ops[j];
    w4::ma::ChainJob& J = jobs[j];
    memset(&J, 0, sizeof(J));
    J.kind = is_gemm(o.kind) ? W4A16_OP_GEMM : o.kind;
    J.epi = o.kind == W4A16_OP_GEMM_SILU ? 1 : 0;
    J.packed = reinterpret_cast<const uint8_t*>(is_gemm(o.kind) ? o.packed : o.X);
    J.Y = reinterpret_cast<uint16_t*>(o.Y);
    J.K = o.K;
    J.N = o.N;
    if (is_gemm(o.kind)) {
      J.Gk = o.K / 128;
      J.U = (o.N / 128) * J.Gk;
      J.cnt_off = cnt;
      cnt += o.N / 128;
      const uint16_t* X = reinterpret_cast<const uint16_t*>(o.X);
      if (int e = w4::encode_x_sw128(&J.xmapR, X, M, o.K, mpad, depth, ldx_of(o))) return e;
      if (int e = w4::encode_x_sw128(&J.xmap1, X, M, o.K, mpad, 2, ldx_of(o))) return e;
    } else if (o.kind == W4A16_OP_ALLREDUCE) {
      const w4a16_peer_group* g = reinterpret_cast<const w4a16_peer_group*>(o.packed);
      const size_t off = reinterpret_cast<uintptr_t>(o.X) - reinterpret_cast<uintptr_t>(g->base[g->rank]);
      const size_t slot_word = w4::kFlagHead + (size_t)ar_slot * W4A16_AR_MAX_TILES;
      auto flags_of = [&](void* base) {
        return reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(base) + g->flag_offset);
      };
      J.world = g->world;
      J.cnt_off = cnt;   // Y's tile-ready flags
      cnt += o.N / 128;
      J.mc_x = g->mc_base ? reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(g->mc_base) + off) : nullptr;
      for (int q = 0; q < g->world; ++q)
        J.peer_x[q] = g->base[q] ? reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(g->base[q]) + off) : nullptr;
      J.my_tiles = flags_of(g->base[g->rank]) + slot_word;
      J.epoch = flags_of(g->base[g->rank]);
      if (!epoch) epoch = J.epoch;
      // the GEMM right before writes the partial: its tile writers bump tile t's counter in every rank's area
      w4::ma::ChainJob& P = jobs[j - 1];
      P.ar_world = g->world;
      P.ar_prev = last_ar;
      P.ar_tiles_mc = g->mc_base ? flags_of(g->mc_base) + slot_word : nullptr;
      for (int q = 0; q < g->world; ++q) P.ar_tiles_peer[q] = g->base[q] ? flags_of(g->base[q]) + slot_word : nullptr;
      last_ar = j;
      ++ar_slot;
    }
    // dependencies from buffer overlaps: RAW for X; WAR / WAW for Y. Completion of op i implies the
    // completion of every op before it, so the latest conflicting op is enough.
    J.dep_x = -1;
    J.dep_y = -1;
    J.xf_off = -1;
    J.xf_mul = 1;
    for (int i = j - 1; i >= 0 && (J.dep_x < 0 || J.dep_y < 0); --i) {
      if (J.dep_x < 0 && overlaps(y_span(ops[i], M), x_span(o, M))) J.dep_x = i;
      if (J.dep_y < 0 && (overlaps(y_span(ops[i], M), y_span(o, M)) || overlaps(x_span(ops[i], M), y_span(o, M)))) J.dep_y = i;
    }
    // tile-level RAW dependency: X is a whole-tile column range of the producing GEMM's Y with Y's row stride
    // (a GEMM_SILU producer writes 64 output columns per tile: 2 tiles per 128-column k-group)
    if (is_gemm(o.kind) && J.dep_x >= 0 && (is_gemm(ops[J.dep_x].kind) || ops[J.dep_x].kind == W4A16_OP_ALLREDUCE)) {
      const w4a16_op& d = ops[J.dep_x];
      const int per_tile = d.kind == W4A16_OP_GEMM_SILU ? 64 : 128, yc = y_cols(d);
      const uintptr_t xb = reinterpret_cast<uintptr_t>(o.X), yb = reinterpret_cast<uintptr_t>(d.Y);
      if (xb >= yb && (xb - yb) % 256 == 0 && ldx_of(o) == yc && (int)((xb - yb) / 2) + o.K <= yc) {
        J.xf_mul = 128 / per_tile;
        J.xf_off = jobs[J.dep_x].cnt_off + (int)((xb - yb) / 2) / per_tile;
        jobs[J.dep_x].pub_tiles = 1;   // the producing op publishes its tile-ready flags
      }
    }
  }
  jobs[0].epoch = epoch;
  jobs[0].n_tiles = cnt;
  return W4A16_OK;
}

// cooperative = 0 only for tests that run several small chains side by side on one device (simulated
// tensor-parallel ranks, tests/test_gpu_allreduce.py); their grids together fit the device.
extern "C" int w4a16_launch_chain_mma(const void* dev_plan, int n_ops, int M, int mode, int family, void* ws,
                                      size_t ws_bytes, int sms, int cooperative, cudaStream_t stream) {
  const int fam = chain_family(M, family);
  if (fam < 0) return fam;
  if (!dev_plan || !ws || n_ops < 1 || (mode != W4A16_ASYM && mode != W4A16_SYM)) return W4A16_ERR_ARG;
  w4::ma::GemmParams p;
  memset(&p, 0, sizeof(p));
  p.G = chain_ctas(sms);
  p.M = M;
  const size_t pb = w4::ma::chain_partial_bytes(M, p.G), db = w4::ma::chain_done_bytes(n_ops);
  if (ws_bytes < pb + db) return W4A16_ERR_WORKSPACE;
  p.partials = reinterpret_cast<float*>(ws);
  p.ds = w4::ma::ntb_of(M) == 1 ? w4::ma::kDSMax : 1;
  p.done = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + pb) + 2 * w4::ma::kDSMax;   // after the run number and exit counter
  p.counters = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + pb + db);
  p.flags = nullptr;   // interleaved with the counters (JobInfo)
  p.jobs = reinterpret_cast<const w4::ma::ChainJob*>(dev_plan);
  p.n_jobs = n_ops;
  p.slots = w4::ma::kChainSlots;
  static int dbg = -1;
  if (dbg < 0) { const char* e = getenv("W4A16_MMA_DEBUG"); dbg = e ? atoi(e) : 0; }
  p.dbg = dbg;
  const bool sym = mode == W4A16_SYM, s = fam == W4A16_FAMILY_MMA_SYNC_S;
  switch (w4::ma::ntb_of(M)) {
    case 1:
      if (s) return sym ? w4::ma::launch_chain_t<1, true, true>(p, cooperative != 0, stream) : w4::ma::launch_chain_t<1, false, true>(p, cooperative != 0, stream);
      return sym ? w4::ma::launch_chain_t<1, true, false>(p, cooperative != 0, stream) : w4::ma::launch_chain_t<1, false, false>(p, cooperative != 0, stream);
    case 2:
      if (s) return sym ? w4::ma::launch_chain_t<2, true, true>(p, cooperative != 0, stream) : w4::ma::launch_chain_t<2, false, true>(p, cooperative != 0, stream);
      return sym ? w4::ma::launch_chain_t<2, true, false>(p, cooperative != 0, stream) : w4::ma::launch_chain_t<2, false, false>(p, cooperative != 0, stream);
    default:
      return W4A16_ERR_SHAPE;
  }
}

// W4A8 GEMM on the family-A pipeline (include/w4a16.h w4a8_gemm; M <= 16). Workspace: w4a16_mma_workspace_bytes.
extern "C" int w4a8_launch_gemm_mma(const int8_t* Xq, const float* sx, const void* packed, uint16_t* Y, int M, int K, int N,
                                    void* ws, int num_sms, cudaStream_t stream) {
  w4::ma::GemmParams p;
  memset(&p, 0, sizeof(p));
  p.packed = reinterpret_cast<const uint8_t*>(packed);
  p.Y = Y;
  p.M = M; p.K = K; p.N = N;
  p.Gk = K / w4::ma::kTileK;
  p.U = (N / w4::ma::kTileN) * p.Gk;
  p.G = w4a16_mma_plan_ctas(K, N, num_sms);
  p.counters = reinterpret_cast<int*>(ws);
  p.partials = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + w4::kCounterBytes);
  p.n_jobs = 1;
  p.slots = 1;
  p.sx = sx;
  switch ((M + 7) / 8) {
    case 1: return w4::ma::launch_a8_t<1>(Xq, p, stream);
    case 2: return w4::ma::launch_a8_t<2>(Xq, p, stream);
    default: return W4A16_ERR_SHAPE;
  }
}

extern "C" int w4a16_launch_gemm_mma(const uint16_t* X, int ldx, const void* packed, uint16_t* Y, int M, int K, int N,
                                     int mode, bool scale_in_a, void* ws, int num_sms, cudaStream_t stream) {
  w4::ma::GemmParams p;
  memset(&p, 0, sizeof(p));
  p.ldx = ldx;
  p.packed = reinterpret_cast<const uint8_t*>(packed);
  p.Y = Y;
  p.M = M; p.K = K; p.N = N;
  p.Gk = K / w4::ma::kTileK;
  p.U = (N / w4::ma::kTileN) * p.Gk;
  p.G = w4a16_mma_plan_ctas(K, N, num_sms);
  const size_t counters = w4::kCounterBytes;
  p.counters = reinterpret_cast<int*>(ws);
  p.partials = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + counters);
  static int dbg = -1;
  if (dbg < 0) { const char* e = getenv("W4A16_MMA_DEBUG"); dbg = e ? atoi(e) : 0; }
  p.dbg = dbg;
  p.jobs = nullptr;
  p.n_jobs = 1;
  p.done = nullptr;
  p.slots = 1;
  const bool sym = mode == W4A16_SYM;
#define W4_MA_CASE(NTB)                                                                                \
  case NTB:                                                                                             \
    if (scale_in_a) return sym ? w4::ma::launch_t<NTB, true, true>(X, p, stream) : w4::ma::launch_t<NTB, false, true>(X, p, stream); \
    return sym ? w4::ma::launch_t<NTB, true, false>(X, p, stream) : w4::ma::launch_t<NTB, false, false>(X, p, stream);
  switch ((M + 7) / 8) {
    W4_MA_CASE(1)
    W4_MA_CASE(2)
    default: return W4A16_ERR_SHAPE;   // the mma.sync families serve M <= 16
  }
#undef W4_MA_CASE
}
