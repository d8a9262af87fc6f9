// gemm_tp.cu — W4A16 verify GEMM, kernel family T: 5th-gen tensor cores (tcgen05 + TMEM) with exact (q - z)
// codes in TMEM and a per-unit TMEM accumulator, M = 1..64. SURVEY §8(a) a2-a6.
//
//   Y[M,N] = X[M,K] · W_hat[K,N],  W_hat = fp16_rne((q - z) * s)  (include/w4a16.h)
//
// Why this shape. On B200 the int4 -> fp16 conversion, not the MMA, competes with HBM for
// issue slots: at 6.5 TB/s every SM must turn one 128x128 unit (8.7 KB) into MMA operands every ~385 cycles.
// Here the tensor core takes the MMA (one elected thread) and a weight pair costs one LOP3 + one HSUB2:
//   lo nibble slots: (w & 0x000F000F) | 0x64006400 = {1024 + q, 1024 + q'};  - {1024 + z} -> exact q - z
//   hi nibble slots: (w & 0x00F000F0) | 0x54005400 = {  64 + q,   64 + q'};  -   {64 + z} -> exact q - z
// The exact integers (q - z) go to TMEM unscaled; tcgen05.mma (M = 128 weight rows, N = MPAD tokens, K = 16)
// computes per unit D[n][m] = sum_k (q_k - z) x_k[m] into that unit's own TMEM accumulator (no offsets, so no
// cancellation whatever the activation magnitude), and the epilogue applies the group scale in fp32:
//   y[m][n] += s_n * D[n][m]        (group = the unit's 128 k; reading R8: fp32 sums, one RNE at the end)
//
// Work plan (same as the other families): unit u = 128 n x 128 k weight tile (8704 / 8448
// contiguous bytes of the packed blob), stream-K over G = #SMs persistent CTAs, CTA c owns units
// [c*U/G, (c+1)*U/G): a plan of (K, N, SMs) only, hence batch-invariant. A tile split between CTAs is reduced
// by its last-arriving contributor in CTA order (deterministic; no CTA ever waits for another).
//
// Warp roles (one CTA per SM, TMEM 512 columns):
//   warps 0..15    dequant, two groups of 8 taking alternate units (each warp's per-unit chain — shared loads,
//                  LOP3/HSUB2, tcgen05.st, wait::st, arrive — is latency-bound, so two units are in flight):
//                  warp w owns TMEM lanes / tile rows 32(w%4)..+31 and k-half (w/4)%2 of its group's units
//   warps 16..     epilogue (4 or 8): tcgen05.ld of a unit's accumulator, 1 FFMA per output, Y / partials
//   + 1            producer: per stage of kRW units one bulk copy of the packed weights (L2 evict_first) and
//                  one 3-D SW128 TMA of their activation slices (rows >= M zero-filled), on one barrier
//   + 2            MMA issuer: 8 tcgen05.mma per unit (elect.sync), commits release A / stage / accumulator
// The producers and the MMA warp take the highest warp ids (the warp arbiter favours them) and sit on
// different sub-partitions.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tma_host.cuh"
#include "w4a16.h"

namespace w4 {
namespace tp {

using tcx::Ring;
constexpr int kTileN = 128, kTileK = 128;
constexpr int kDqGroups = 2;
constexpr int kDq = 8 * kDqGroups;            // dequant warps
constexpr int kS = 2;                         // units per step (hand-off granularity)
constexpr int kTmemCols = 512;
constexpr int kSmemBudget = 227 * 1024 - 1024;

template <int MPAD>
struct Cfg {
  static constexpr int kEpi = MPAD <= 32 ? 4 : 8;                 // epilogue warps
  static constexpr int kEpiW0 = kDq;
  static constexpr int kWProdW = kDq + kEpi;
  static constexpr int kMmaW = kWProdW + 1;
  static constexpr int kWarps = kMmaW + 1;
  static constexpr int kThreads = kWarps * 32;
  // A step = kS consecutive units of one op: one hand-off per step between the dequant warps, the MMA warp and
  // the epilogue (each hand-off costs ~0.2-0.35 us of latency on the waiting side, traced; per unit the HBM
  // budget is ~0.2 us). A pipeline stage = kRW units: ONE bulk copy of their packed weights plus their
  // activation slices, completing on one barrier — activations loaded on a separate ring queue behind the
  // weight stream in the TMA / L2 path (~3 us round trip, traced) and pace the kernel.
  static constexpr int kRW = MPAD <= 16 ? 4 : 2;                  // units per stage
  static constexpr int kNA = MPAD <= 16 ? 3 : 2;                  // TMEM A buffers (kS units x 64 columns)
  static constexpr int kAccCol0 = kNA * kS * 64;
  static constexpr int kNAccFit = (kTmemCols - kAccCol0) / (kS * MPAD);
  static constexpr int kNAcc = kNAccFit > 8 ? 8 : kNAccFit;       // per-step accumulators (kS x MPAD columns)
  static constexpr int kXBox = MPAD * 128;                        // one 64-k SW128 box of MPAD token rows
  static constexpr int kXUnit = 2 * kXBox;                        // a unit's 128 k
  // Weights and activations live in SEPARATE rings: a weight stage is released as soon as the dequant warps
  // have read it (its HBM refill starts at once), an activation stage when the MMAs that read it complete.
  static constexpr int kStage = kRW * 8704;                        // kRW packed units
  static constexpr int kXStage = kRW * kXUnit;                     // their activation slices
  static constexpr int kAux = kNAcc * kS * 128 * 4;               // the scale s per unit row, per accumulator slot
  static constexpr int kSW0 = (kSmemBudget - kAux - 3 * kXStage) / kStage;
  static constexpr int kSW = kSW0 > 8 ? 8 : kSW0;                 // weight stages
  static constexpr int kSX0 = (kSmemBudget - 1024 - kAux - kSW * kStage) / kXStage;   // (static smem, alignment)
  static constexpr int kSX = kSX0 > 8 ? 8 : kSX0;                 // activation stages
  static constexpr int kSmem = kSW * kStage + kSX * kXStage + kAux + 1024;
  // instruction descriptor: D f32 (bit 4), A/B f16, K-major both, N = MPAD (bits 17-22: N >> 3), M = 128 (bits 24-28: M >> 4)
  static constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(MPAD >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  static_assert(kSW >= 3 && kSX >= 2, "rings too shallow");
  static_assert(kNAcc >= 2, "accumulator ring too shallow");
  static_assert(kRW % kS == 0, "stages hold whole steps");
};

struct Params {
  const uint8_t* packed;
  uint16_t* Y;
  float* partials;      // [slots][2G][MPAD][128] fp32 split-tile partials
  int* counters;        // tile counters: fixed region (single GEMM) or per op at ChainJob::cnt_off (chain)
  int M, K, N, Gk, U, G;
  int ldx;              // host only: X row stride in elements (0 = K), read when the X tensor maps are encoded
  const ChainJob* jobs; // chain op table (device) or nullptr: a single GEMM
  int n_jobs;
  int* done;            // chain: [n_jobs] CTAs that finished each op, then the exit counter
  int slots;            // chain: partial-slot ring length in ops (1 for a single GEMM)
  int dbg;              // diagnostics only (W4A16_TP_DEBUG): bit0 skip MMAs, bit1 skip dequant math, bit2 skip
                        // X loads, bit3 skip accumulator loads, bit4 stream only (stages released on arrival;
                        // wrong results), bit8 per-unit timeline of CTA 0 (g_tp_trace)
};

// Diagnostics only: %globaltimer per unit of CTA 0 at the hand-off points of each role (tools/probe_fam.py --trace).
constexpr int kTraceUnits = 128;
__device__ unsigned long long g_tp_trace[12][kTraceUnits];
__device__ __forceinline__ void trace(const Params& p, int ev, int i) {
  if ((p.dbg & 256) && blockIdx.x == 0 && i < kTraceUnits) g_tp_trace[ev][i] = globaltimer_ns();
}

struct Job {
  const uint8_t* packed;
  uint16_t* Y;
  const CUtensorMap* xmap1;   // one unit's activation boxes (depth 2)
  const CUtensorMap* xmapS;   // a step's (depth 2 kS)
  int* counters;
  int kind, N, Gk, U, dep_x, dep_y;
};
__device__ __forceinline__ Job job_at(const Params& p, const CUtensorMap* xmap1, const CUtensorMap* xmapS, int j) {
  Job J;
  if (p.jobs == nullptr) {
    J.packed = p.packed; J.Y = p.Y; J.xmap1 = xmap1; J.xmapS = xmapS; J.counters = p.counters;
    J.kind = kOpGemm; J.N = p.N; J.Gk = p.Gk; J.U = p.U; J.dep_x = -1; J.dep_y = -1;
  } else {
    const ChainJob* c = p.jobs + j;
    J.packed = c->packed; J.Y = c->Y; J.xmap1 = &c->xmap1; J.xmapS = &c->xmapR; J.counters = p.counters + c->cnt_off;
    J.kind = c->kind; J.N = c->N; J.Gk = c->Gk; J.U = c->U; J.dep_x = c->dep_x; J.dep_y = c->dep_y;
  }
  return J;
}
__device__ __forceinline__ int unit_begin(int c, int U, int G) { return (int)(((long long)c * U) / G); }
__device__ __forceinline__ int cta_of_unit(int u, int U, int G) {
  return (int)((((long long)(u + 1) * G) + U - 1) / U) - 1;
}
__device__ __forceinline__ void wait_op(const Params& p, int j) {
  if (j < 0) return;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_gpu(&p.done[j]) < p.G) {
    __nanosleep(64);
    if (globaltimer_ns() - t0 > 30000000000ull) __trap();   // never hang the device on a protocol bug
  }
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

template <int MPAD, bool SYM>
__global__ void __launch_bounds__(Cfg<MPAD>::kThreads, 1)
    gemm_w4a16_tp_kernel(const __grid_constant__ CUtensorMap xmap1, const __grid_constant__ CUtensorMap xmapS,
                         const Params p) {
  using C = Cfg<MPAD>;
  constexpr int SW = C::kSW, SX = C::kSX, NA = C::kNA, NACC = C::kNAcc, kRW = C::kRW;
  constexpr int TB = SYM ? 8448 : 8704;
  // barriers: wfull/wempty [SW], afull/aempty [NA], accfull/accempty/sfull [NACC]
  __shared__ __align__(8) uint64_t bars[2 * SW + 2 * SX + 2 * NA + 3 * NACC];
  __shared__ uint32_t s_tmem;
  __shared__ int s_last;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t w_base = smem_u32(smem);
  const uint32_t x_base = w_base + SW * C::kStage;            // activation ring
  const uint32_t s_base = x_base + SX * C::kXStage;           // [NACC][kS][128] fp32 scale per unit row
  const uint32_t b0 = smem_u32(&bars[0]);
  const uint32_t WFULL = b0, WEMPTY = WFULL + 8 * SW;
  const uint32_t AFULL = WEMPTY + 8 * SW, AEMPTY = AFULL + 8 * NA, ACCFULL = AEMPTY + 8 * NA;
  const uint32_t ACCEMPTY = ACCFULL + 8 * NACC, SFULL = ACCEMPTY + 8 * NACC;
  const uint32_t XFULL = SFULL + 8 * NACC, XEMPTY = XFULL + 8 * SX;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const bool chain = p.jobs != nullptr;

  if (threadIdx.x == 0) {
    // a weight stage is released by the dequant warps (read), an activation stage by the MMA warp's commit
    for (int i = 0; i < SW; ++i) { tcx::mbar_init_a(WFULL + 8 * i, 1); tcx::mbar_init_a(WEMPTY + 8 * i, kDq); }
    for (int i = 0; i < SX; ++i) { tcx::mbar_init_a(XFULL + 8 * i, 1); tcx::mbar_init_a(XEMPTY + 8 * i, 1); }
    for (int i = 0; i < NA; ++i) { tcx::mbar_init_a(AFULL + 8 * i, 8); tcx::mbar_init_a(AEMPTY + 8 * i, 1); }
    for (int i = 0; i < NACC; ++i) {
      tcx::mbar_init_a(ACCFULL + 8 * i, 1);
      tcx::mbar_init_a(ACCEMPTY + 8 * i, C::kEpi);
      tcx::mbar_init_a(SFULL + 8 * i, 4);   // the step's 4 k-half-0 dequant warps wrote the row scales
    }
    fence_mbar_init();
    if (!chain) pdl_launch_dependents();
  }
  if (warp == C::kMmaW) tcx::tmem_alloc(&s_tmem, kTmemCols);
  tcx::fence_before();
  __syncthreads();
  tcx::fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == C::kWProdW) {
    // ---------------- producer: per stage one bulk copy of kRW packed units + their activation slices ----------
    // Weights never depend on an earlier kernel or op, so they are issued as soon as a stage frees; a stage's
    // activations wait in a FIFO until they may be read (griddepcontrol.wait for a single GEMM; the producing
    // op's completion in a chain), so the weight stream runs ahead across op boundaries.
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      if (!chain) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap1)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmapS)) : "memory");
      }
      int q_j[16], q_u0[16], q_nu[16];   // stages whose activation loads are not issued yet (FIFO)
      int q_head = 0, q_n = 0, ok_upto = -1, n_w = 0, x_issued = 0;
      Ring x{0, 0};
      bool pdl_done = chain;
      auto drain = [&](bool block) {   // issue queued activation loads whose producers are done
        while (q_n > 0) {
          if (!pdl_done) {
            if (!block) return;
            pdl_wait();
            pdl_done = true;
          }
          const Job J = job_at(p, &xmap1, &xmapS, q_j[q_head]);
          if (J.dep_x > ok_upto) {
            if (ld_acquire_gpu(&p.done[J.dep_x]) < p.G) {
              if (!block) return;
              wait_op(p, J.dep_x);
            }
            ok_upto = J.dep_x;
            fence_proxy_async_global();   // generic-proxy stores of other CTAs -> this TMA (async proxy) read
          }
          const int u0 = q_u0[q_head], nu = q_nu[q_head];
          if (x_issued >= SX && !mbar_try_wait(reinterpret_cast<uint64_t*>(__cvta_shared_to_generic(XEMPTY + 8 * x.i)), x.ph ^ 1)) {
            if (!block) return;
            tcx::wait(XEMPTY + 8 * x.i, x.ph ^ 1);   // the MMAs that read this activation slot are complete
          }
          const uint32_t dst = x_base + x.i * C::kXStage, bar = XFULL + 8 * x.i;
          tcx::expect_tx_a(bar, (p.dbg & 4) ? 0 : nu * C::kXUnit);
          const int g = u0 % J.Gk;
          if (p.dbg & 4) {
          } else if (nu == kRW && g + kRW <= J.Gk) {
            tcx::tma_3d(dst, J.xmapS, 0, 0, 2 * g, bar);
          } else {
            for (int jj = 0, gg = g; jj < nu; ++jj, gg = (gg + 1 == J.Gk ? 0 : gg + 1))
              tcx::tma_3d(dst + jj * C::kXUnit, J.xmap1, 0, 0, 2 * gg, bar);
          }
          trace(p, 0, q_u0[q_head] - unit_begin(cta, J.U, p.G));
          q_head = (q_head + 1) & 15;
          --q_n;
          ++x_issued;
          x.next(SX);
        }
      };
      Ring w{0, 0};
      int issued = 0;
      for (int j = 0; j < p.n_jobs; ++j) {
        const Job J = job_at(p, &xmap1, &xmapS, j);
        if (J.kind != kOpGemm) continue;
        const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
        for (int u0 = ub; u0 < ue; u0 += kRW) {
          const int nu = min(kRW, ue - u0);
          if (issued >= SW) {   // the stage must be released first; meanwhile issue pending activation loads
            if (!pdl_done) drain(true);
            const unsigned long long t0 = globaltimer_ns();
            while (!mbar_try_wait(reinterpret_cast<uint64_t*>(__cvta_shared_to_generic(WEMPTY + 8 * w.i)), w.ph ^ 1)) {
              drain(false);
              if (globaltimer_ns() - t0 > 30000000000ull) __trap();   // a protocol bug fails instead of hanging
            }
          }
          trace(p, 1, n_w);
          n_w += nu;
          tcx::expect_tx_a(WFULL + 8 * w.i, nu * TB);
          tcx::bulk_g2s_a(w_base + w.i * C::kStage, J.packed + (size_t)u0 * TB, nu * TB, WFULL + 8 * w.i, pol);
          if (q_n == 16) drain(true);
          const int e = (q_head + q_n) & 15;
          q_j[e] = j; q_u0[e] = u0; q_nu[e] = nu;
          ++q_n;
          drain(false);
          ++issued;
          w.next(SW);
        }
      }
      drain(true);
    }
  } else if (warp == C::kMmaW) {
    // ---------------- MMA issuer: per step 8 x tcgen05.mma (K = 16) per unit, each unit its own accumulator --
    Ring x{0, 0}, a{0, 0}, acc{0, 0};
    int n_u = 0;
    const uint32_t desc_hi = (uint32_t)(tcx::kDescSW128 >> 32);
    for (int j = 0; j < p.n_jobs; ++j) {
      const Job J = job_at(p, &xmap1, &xmapS, j);
      if (J.kind != kOpGemm) continue;
      const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
      for (int u0 = ub; u0 < ue; u0 += kRW) {
        const int nw = min(kRW, ue - u0);
        tcx::wait(XFULL + 8 * x.i, x.ph);
        const uint32_t xs = x_base + x.i * C::kXStage;
        for (int j0 = 0; j0 < nw; j0 += kS) {
          const int nu = min(kS, nw - j0);
          if (p.dbg & 16) {   // diagnostics: stream only (stage released as soon as it lands)
            if (tcx::elect_one() && j0 + kS >= nw) tcx::commit(XEMPTY + 8 * x.i);
            __syncwarp();
            continue;
          }
          tcx::wait(AFULL + 8 * a.i, a.ph);
          tcx::wait(ACCEMPTY + 8 * acc.i, acc.ph ^ 1);
          tcx::fence_after();
          if (lane == 0) trace(p, 5, n_u);
          if (tcx::elect_one()) {
            for (int jj = 0; jj < nu; ++jj) {
              const uint32_t d_tmem = tmem + C::kAccCol0 + (acc.i * kS + jj) * MPAD;
              const uint32_t a_tmem = tmem + (a.i * kS + jj) * 64;
              const uint32_t lo0 = (1u << 16) | ((xs + (j0 + jj) * C::kXUnit) >> 4);   // LBO = 1 | start >> 4
#pragma unroll
              for (int ks = 0; ks < 8; ++ks) {
                const uint32_t lo = lo0 + (uint32_t)(((ks >> 2) * C::kXBox + (ks & 3) * 32) >> 4);
                if (!(p.dbg & 1)) tcx::mma_ts(d_tmem, a_tmem + ks * 8, ((uint64_t)desc_hi << 32) | lo, C::kIdesc, ks > 0 ? 1u : 0u);
              }
            }
            tcx::commit(AEMPTY + 8 * a.i);
            tcx::commit(ACCFULL + 8 * acc.i);
            if (j0 + kS >= nw) tcx::commit(XEMPTY + 8 * x.i);   // the stage's activations are read
          }
          __syncwarp();
          if (lane == 0) trace(p, 6, n_u);
          n_u += nu;
          a.next(NA);
          acc.next(NACC);
        }
        x.next(SX);
      }
    }
  } else if (warp < kDq) {
    // ---------------- dequant: exact (q - z) into a TMEM A buffer; group grp takes every other step ----------
    const int grp = warp >> 3, q = warp & 3, h = (warp >> 2) & 1;
    const int row = q * 32 + lane;
    const int sw = (row >> 1) & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    Ring w{0, 0}, a{0, 0}, acc{0, 0};
    int parity = 0;   // position of the step in this CTA's step sequence, mod 2
    int n_u = 0;
    for (int j = 0; j < p.n_jobs; ++j) {
      const Job J = job_at(p, &xmap1, &xmapS, j);
      if (J.kind != kOpGemm) continue;
      const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
      for (int u0 = ub; u0 < ue; u0 += kRW) {
        const int nw = min(kRW, ue - u0);
        tcx::wait(WFULL + 8 * w.i, w.ph);
        if (lane == 0 && q == 0 && h == 0) trace(p, 2 + grp, n_u);
        const uint32_t st = w_base + w.i * C::kStage;   // the stage's packed units
        for (int j0 = 0; j0 < nw; j0 += kS) {
          const int nu = min(kS, nw - j0);
          if (parity == grp && !(p.dbg & 16)) {
            bool waited = false;
            for (int jj = 0; jj < nu; ++jj) {
              const uint32_t ub_ = st + (j0 + jj) * TB;
              // chunks 2h, 2h+1 of this row (XOR-permuted layout: conflict-free across the warp's 32 rows)
              uint4 w0 = lds128(ub_ + row * 64 + (((2 * h) ^ sw) << 4));
              uint4 w1 = lds128(ub_ + row * 64 + (((2 * h + 1) ^ sw) << 4));
              if (p.dbg & 2) w1 = w0 = make_uint4(lane, row, h, 0);
              float sc;
              __half2 zl, zh;   // {1024 + z} and {64 + z} broadcast pairs
              if (SYM) {
                sc = __half2float(__ushort_as_half(tcx::lds16u(ub_ + 8192 + 2 * row)));
                zl = __float2half2_rn(1032.f);
                zh = __float2half2_rn(72.f);
              } else {
                const __half2 sz = u2h2(tcx::lds32u(ub_ + 8192 + 4 * row));
                sc = __low2float(sz);
                const __half2 z2 = __high2half2(sz);
                zl = __hadd2(z2, __float2half2_rn(1024.f));
                zh = __hadd2(z2, __float2half2_rn(64.f));
              }
              const uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
              uint32_t av[32];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const uint32_t x0 = wv[i], x8 = wv[i] >> 8;
                av[4 * i + 0] = h22u(__hsub2(u2h2(lop3_and_or(x0, 0x000F000Fu, 0x64006400u)), zl));   // k 8i+0, +1
                av[4 * i + 1] = h22u(__hsub2(u2h2(lop3_and_or(x0, 0x00F000F0u, 0x54005400u)), zh));   // k 8i+2, +3
                av[4 * i + 2] = h22u(__hsub2(u2h2(lop3_and_or(x8, 0x000F000Fu, 0x64006400u)), zl));   // k 8i+4, +5
                av[4 * i + 3] = h22u(__hsub2(u2h2(lop3_and_or(x8, 0x00F000F0u, 0x54005400u)), zh));   // k 8i+6, +7
              }
              if (!waited) {
                tcx::wait(AEMPTY + 8 * a.i, a.ph ^ 1);   // the MMAs that last read this A buffer are complete
                if (h == 0) tcx::wait(ACCEMPTY + 8 * acc.i, acc.ph ^ 1);   // and the scale slot is consumed
                tcx::fence_after();
                if (lane == 0 && q == 0 && h == 0) trace(p, 4, n_u);
                waited = true;
              }
              tcx::st_x32(tmem + lane_base + (a.i * kS + jj) * 64 + h * 32, av);
              if (h == 0) sts32f(s_base + ((acc.i * kS + jj) * 128 + row) * 4, sc);
            }
            tcx::wait_st();
            tcx::fence_before();
            __syncwarp();
            if (lane == 0) {
              mbar_arrive_a(AFULL + 8 * a.i);
              if (h == 0) mbar_arrive_a(SFULL + 8 * acc.i);
              if (q == 0 && h == 0) trace(p, 7, n_u);
            }
          }
          parity ^= 1;
          n_u += nu;
          a.next(NA);
          acc.next(NACC);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_a(WEMPTY + 8 * w.i);
        w.next(SW);
      }
    }
  } else {
    // ---------------- epilogue: per-unit group scale in fp32, tile output ----------------
    const int e = warp - C::kEpiW0;
    const int q = e & 3;
    constexpr int kCols = MPAD / (C::kEpi / 4);   // token columns of this warp
    const int col0 = (e >> 2) * kCols;
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t kEpiThreads = C::kEpi * 32;
    const bool epi0 = warp == C::kEpiW0 && lane == 0;
    if (!chain) pdl_wait();   // Y / workspace writes must follow the preceding kernel
    Ring acc{0, 0};
    int n_u = 0;
    for (int j = 0; j < p.n_jobs; ++j) {
      const Job J = job_at(p, &xmap1, &xmapS, j);
      if (J.kind == kOpSilu) {
        // SiLU*mul op of a chain (same arithmetic as w4a16_silu_mul), over every epilogue thread of every CTA
        if (epi0) wait_op(p, max(J.dep_x, J.dep_y));
        named_bar_sync(1, kEpiThreads);
        const int F = J.N, vecs = F / 8;
        const long long total = (long long)p.M * vecs;
        const uint16_t* GU = reinterpret_cast<const uint16_t*>(J.packed);
        const int et = e * 32 + lane;
        for (long long i = (long long)cta * kEpiThreads + et; i < total; i += (long long)p.G * kEpiThreads) {
          const int m = (int)(i / vecs), v = (int)(i % vecs);
          const uint4 gg = __ldcg(reinterpret_cast<const uint4*>(GU + (size_t)m * 2 * F + (size_t)v * 8));
          const uint4 uu = __ldcg(reinterpret_cast<const uint4*>(GU + (size_t)m * 2 * F + F + (size_t)v * 8));
          *reinterpret_cast<uint4*>(J.Y + (size_t)m * F + (size_t)v * 8) = silu_mul_vec(gg, uu);
        }
        named_bar_sync(1, kEpiThreads);
        if (epi0) red_release_gpu_add(&p.done[j], 1);
        continue;
      }
      if (J.kind != kOpGemm) continue;
      const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
      const int wdep = chain ? max(J.dep_y, j - p.slots) : -1;
      bool y_ready = wdep < 0;
      float* part = p.partials + (size_t)(j % p.slots) * 2 * p.G * MPAD * kTileN;
      float y[kCols];
#pragma unroll
      for (int c = 0; c < kCols; ++c) y[c] = 0.f;
      int t = ub / J.Gk, g = ub % J.Gk, seg0 = ub, nseg = 0;
      for (int u0 = ub; u0 < ue && !(p.dbg & 16); u0 += kS) {
        const int nu = min(kS, ue - u0);
        tcx::wait(ACCFULL + 8 * acc.i, acc.ph);
        if (epi0) trace(p, 8, n_u);
        tcx::wait(SFULL + 8 * acc.i, acc.ph);
        tcx::fence_after();
        float sc[kS];
#pragma unroll
        for (int jj = 0; jj < kS; ++jj) sc[jj] = jj < nu ? tcx::lds32f(s_base + ((acc.i * kS + jj) * 128 + row) * 4) : 0.f;
        // the step's accumulators, unit by unit, 8 columns at a time straight into y (few live registers);
        // the slot is released once all are in registers, the segment / tile logic follows per unit
        float yv[kS][kCols];
#pragma unroll
        for (int jj = 0; jj < kS; ++jj) {
          if (jj < nu) {
#pragma unroll
            for (int c = 0; c < kCols; c += 8) {
              uint32_t r8[8];
              if (p.dbg & 8) {
#pragma unroll
                for (int i = 0; i < 8; ++i) r8[i] = 0;
              } else {
                tcx::ld_x8(tmem + lane_base + C::kAccCol0 + (acc.i * kS + jj) * MPAD + col0 + c, r8);
                tcx::wait_ld();
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) yv[jj][c + i] = sc[jj] * __uint_as_float(r8[i]);
            }
          }
        }
        tcx::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_a(ACCEMPTY + 8 * acc.i);
        if (epi0) trace(p, 9, n_u);
        n_u += nu;
        acc.next(NACC);
#pragma unroll
        for (int jj = 0; jj < kS; ++jj) {
          if (jj >= nu) break;
          const int u = u0 + jj;
#pragma unroll
          for (int c = 0; c < kCols; ++c) y[c] += yv[jj][c];
          const bool seg_end = (u + 1 == ue) || (g + 1 == J.Gk);
          if (seg_end) {
            // ---- the segment [seg0, u + 1) of tile t is complete in this CTA ----
            if (!y_ready) {
              if (epi0) wait_op(p, wdep);   // released to the other epilogue threads by the barrier
              named_bar_sync(1, kEpiThreads);
              y_ready = true;
            }
            const int tile_u0 = t * J.Gk, tile_u1 = tile_u0 + J.Gk;
            const int n = t * kTileN + row;
            if (seg0 == tile_u0 && u + 1 == tile_u1) {
#pragma unroll
              for (int c = 0; c < kCols; ++c)
                if (col0 + c < p.M) J.Y[(size_t)(col0 + c) * J.N + n] = __half_as_ushort(__float2half_rn(y[c]));
            } else {
              // split tile: fp32 partial in this CTA's slot, then the last contributor to arrive sums all of
              // them in CTA order (deterministic) and writes Y
              const int slot = 2 * cta + (nseg == 0 ? 0 : 1);
#pragma unroll
              for (int c = 0; c < kCols; ++c) __stcg(&part[((size_t)slot * MPAD + col0 + c) * kTileN + row], y[c]);
              const int c_first = cta_of_unit(tile_u0, J.U, p.G), c_last = cta_of_unit(tile_u1 - 1, J.U, p.G);
              named_bar_sync(1, kEpiThreads);
              if (epi0) {
                __threadfence();
                s_last = atomicAdd(&J.counters[kCounterStride * t], 1) == c_last - c_first;
              }
              named_bar_sync(1, kEpiThreads);
              if (s_last) {
                __threadfence();
                float r[kCols];
#pragma unroll
                for (int c = 0; c < kCols; ++c) r[c] = 0.f;
                for (int cc = c_first; cc <= c_last; ++cc) {
                  const int sl = 2 * cc + (unit_begin(cc, J.U, p.G) >= tile_u0 ? 0 : 1);
#pragma unroll
                  for (int c = 0; c < kCols; ++c) r[c] += __ldcg(&part[((size_t)sl * MPAD + col0 + c) * kTileN + row]);
                }
#pragma unroll
                for (int c = 0; c < kCols; ++c)
                  if (col0 + c < p.M) J.Y[(size_t)(col0 + c) * J.N + n] = __half_as_ushort(__float2half_rn(r[c]));
                if (epi0) J.counters[kCounterStride * t] = 0;   // every contributor has arrived: re-arm for the next launch / run
              }
            }
            ++nseg;
            ++t;
            seg0 = u + 1;
#pragma unroll
            for (int c = 0; c < kCols; ++c) y[c] = 0.f;
          }
          if (++g == J.Gk) g = 0;
        }
      }
      if (chain) {   // this CTA's share of the op is written: count it
        named_bar_sync(1, kEpiThreads);
        if (epi0) red_release_gpu_add(&p.done[j], 1);
      }
    }
    if (chain && epi0) {
      // the last CTA out re-arms the op counters for the next run of the chain
      __threadfence();
      if (atomicAdd(&p.done[p.n_jobs], 1) == p.G - 1) {
        __threadfence();
        for (int jj = 0; jj < p.n_jobs; ++jj) p.done[jj] = 0;
        p.done[p.n_jobs] = 0;
        __threadfence();
      }
    }
  }
  tcx::fence_before();
  __syncthreads();
  if (warp == C::kMmaW) {
    tcx::fence_after();
    tcx::tmem_dealloc(tmem, kTmemCols);
  }
}

// ---- host side ----
inline int mpad_of(int M) { return M <= 8 ? 8 : (M + 15) / 16 * 16; }

template <int MPAD, bool SYM>
int launch(const uint16_t* X, const Params& p, cudaStream_t stream) {
  using C = Cfg<MPAD>;
  CUtensorMap map1, mapS;
  if (int e = encode_x_sw128(&map1, X, p.M, p.K, MPAD, 2, p.ldx)) return e;
  if (int e = encode_x_sw128(&mapS, X, p.M, p.K, MPAD, 2 * C::kRW, p.ldx)) return e;
  auto kern = gemm_w4a16_tp_kernel<MPAD, SYM>;
  static unsigned long long attr = 0;
  if (!ensure_smem_attr(kern, C::kSmem, attr)) return W4A16_ERR_CUDA;
  return launch_pdl(kern, dim3(p.G), dim3(C::kThreads), C::kSmem, stream, map1, mapS, p) == cudaSuccess ? W4A16_OK
                                                                                                      : W4A16_ERR_CUDA;
}

template <int MPAD, bool SYM>
int launch_chain(const Params& p, bool cooperative, cudaStream_t stream) {
  using C = Cfg<MPAD>;
  auto kern = gemm_w4a16_tp_kernel<MPAD, SYM>;
  static unsigned long long attr = 0;
  if (!ensure_smem_attr(kern, C::kSmem, attr)) return W4A16_ERR_CUDA;
  CUtensorMap unused;
  memset(&unused, 0, sizeof(unused));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr1[1];
  attr1[0].id = cudaLaunchAttributeCooperative;
  attr1[0].val.cooperative = 1;
  cfg.attrs = attr1;
  cfg.numAttrs = cooperative ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, unused, unused, p) == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

template <bool SYM>
int dispatch(const uint16_t* X, const Params& p, bool chain, bool cooperative, cudaStream_t stream) {
  const int M = p.M;
#define W4_TP(MP) return chain ? launch_chain<MP, SYM>(p, cooperative, stream) : launch<MP, SYM>(X, p, stream)
  if (M <= 8) W4_TP(8);
  if (M <= 16) W4_TP(16);
  if (M <= 32) W4_TP(32);
  if (M <= 48) W4_TP(48);
  if (M <= 64) W4_TP(64);
#undef W4_TP
  return W4A16_ERR_SHAPE;
}

}  // namespace tp
}  // namespace w4

extern "C" int w4a16_tp_plan_ctas(int K, int N, int num_sms) {
  const long long U = (long long)(N / w4::tp::kTileN) * (K / w4::tp::kTileK);
  return (int)(U < num_sms ? U : num_sms);
}

extern "C" size_t w4a16_tp_workspace_bytes(int M, int K, int N, int num_sms) {
  return w4::kCounterBytes + (size_t)2 * w4a16_tp_plan_ctas(K, N, num_sms) * w4::tp::mpad_of(M) * w4::tp::kTileN * 4;
}

extern "C" int w4a16_launch_gemm_tp(const uint16_t* X, int ldx, const void* packed, uint16_t* Y, int M, int K, int N,
                                    int mode, void* ws, int num_sms, cudaStream_t stream) {
  w4::tp::Params p;
  memset(&p, 0, sizeof(p));
  p.ldx = ldx;
  p.packed = reinterpret_cast<const uint8_t*>(packed);
  p.Y = Y;
  p.M = M; p.K = K; p.N = N;
  p.Gk = K / w4::tp::kTileK;
  p.U = (N / w4::tp::kTileN) * p.Gk;
  p.G = w4a16_tp_plan_ctas(K, N, num_sms);
  p.counters = reinterpret_cast<int*>(ws);
  p.partials = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + w4::kCounterBytes);
  p.jobs = nullptr;
  p.n_jobs = 1;
  p.slots = 1;
  static int dbg = -1;
  if (dbg < 0) { const char* e = getenv("W4A16_TP_DEBUG"); dbg = e ? atoi(e) : 0; }
  p.dbg = dbg;
  return mode == W4A16_SYM ? w4::tp::dispatch<true>(X, p, false, false, stream)
                           : w4::tp::dispatch<false>(X, p, false, false, stream);
}

extern "C" int w4a16_debug_trace_tp(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, w4::tp::g_tp_trace, bytes < sizeof(w4::tp::g_tp_trace) ? bytes : sizeof(w4::tp::g_tp_trace)) ==
                 cudaSuccess ? 0 : -5;
}
