// gemm_tp.cu — W4A16 verify GEMM, kernel family T: 5th-gen tensor cores (tcgen05 + TMEM) with OFFSET CODES
// and a per-unit TMEM accumulator, M = 1..64. SURVEY §8(a) a2-a6.
//
//   Y[M,N] = X[M,K] · W_hat[K,N],  W_hat = fp16_rne((q - z) * s)  (include/w4a16.h)
//
// Why this shape. On B200 the int4 -> fp16 conversion, not the MMA, competes with HBM for
// issue slots: at 6.5 TB/s every SM must turn one 128x128 unit (8.7 KB) into MMA operands every ~385 cycles.
// The mma.sync family spends ~1070 warp-instructions per unit (dequant + HMMA + a per-unit group epilogue in
// registers); here the tensor core takes the MMA (one elected thread) and each weight costs ONE LOP3:
//   lo nibble slots: (w & 0x000F000F) | 0x64006400 = {1024 + q, 1024 + q'}     (exact fp16)
//   hi nibble slots: (w & 0x00F000F0) | 0x54005400 = {  64 + q,   64 + q'}     (exact fp16)
// so A = "offset codes" (1024 + q or 64 + q) goes to TMEM unscaled, and tcgen05.mma (M = 128 weight rows,
// N = MPAD tokens, K = 16) computes per unit D[n][m] = sum_k (off_k + q_k) x_k[m] into its own TMEM
// accumulator. The epilogue restores the definition per unit (group = unit k-range):
//   y[m][n] += s_n * (D[n][m] - C[m] - z_n * S[m]),   C[m] = sum_k off_k x_k[m],  S[m] = sum_k x_k[m]
// with C and S produced per unit by an activation-sum warp (one mma.sync per k-step with a constant B).
// fp32 throughout; one fp32 -> fp16 RNE at the end (reading R8).
//
// Work plan (same as the other families): unit u = 128 n x 128 k weight tile (8704 / 8448
// contiguous bytes of the packed blob), stream-K over G = #SMs persistent CTAs, CTA c owns units
// [c*U/G, (c+1)*U/G): a plan of (K, N, SMs) only, hence batch-invariant. A tile split between CTAs is reduced
// by its last-arriving contributor in CTA order (deterministic, no CTA ever waits for another).
//
// Warp roles (one CTA per SM, TMEM 512 columns):
//   warps 0..7     dequant: warp w owns TMEM lanes / tile rows 32(w%4)..+31 and k-half w/4 of each unit;
//                  LDS.128 x2 -> 32 LOP3/SHF -> one tcgen05.st.32x32b.x32 into a TMEM A buffer
//   warps 8..      epilogue (4 or 8): tcgen05.ld of a unit's accumulator, 3 FFMA per output, Y / partials
//   + 1            activation sums C, S per unit (mma.sync, constant B)
//   + 2            weight producer: one bulk copy (TMA engine) per stage of kRW units, L2 evict_first
//   + 3            activation producer: one 3-D SW128 TMA per unit (rows >= M zero-filled)
//   + 4            MMA issuer: 8 tcgen05.mma per unit (elect.sync), commits release A / X / accumulator
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
constexpr int kDq = 8;                        // dequant warps
constexpr int kRW = 4;                        // units per weight stage (one bulk copy)
constexpr int kTmemCols = 512;
constexpr int kSmemBudget = 227 * 1024 - 1024;

template <int MPAD>
struct Cfg {
  static constexpr int kEpi = MPAD <= 32 ? 4 : 8;                 // epilogue warps
  static constexpr int kEpiW0 = kDq;
  static constexpr int kXsumW = kDq + kEpi;
  static constexpr int kWProdW = kXsumW + 1;
  static constexpr int kXProdW = kXsumW + 2;
  static constexpr int kMmaW = kXsumW + 3;
  static constexpr int kWarps = kMmaW + 1;
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kNA = MPAD <= 16 ? 6 : 4;                  // TMEM A buffers (64 columns = one unit)
  static constexpr int kAccCol0 = kNA * 64;
  static constexpr int kNAccFit = (kTmemCols - kAccCol0) / MPAD;
  static constexpr int kNAcc = kNAccFit > 8 ? 8 : kNAccFit;       // per-unit accumulators (MPAD columns)
  static constexpr int kXBox = MPAD * 128;                        // one 64-k SW128 box of MPAD token rows
  static constexpr int kXSlot = 2 * kXBox;                        // the unit's 128 k
  static constexpr int kNX = MPAD <= 32 ? 8 : 4;                  // activation slots
  static constexpr int kStageW = kRW * 8704;                      // weight stage (ASYM size; SYM uses less)
  static constexpr int kAux = kNAcc * 128 * 8 + kNAcc * MPAD * 8; // {s, z} per row + {C, S} per token, per slot
  static constexpr int kSW0 = (kSmemBudget - kNX * kXSlot - kAux) / kStageW;
  static constexpr int kSW = kSW0 > 8 ? 8 : kSW0;                 // weight stages
  static constexpr int kSmem = kSW * kStageW + kNX * kXSlot + kAux + 1024;
  // instruction descriptor: D f32 (bit 4), A/B f16, K-major both, N = MPAD (bits 17-22: N >> 3), M = 128 (bits 24-28: M >> 4)
  static constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(MPAD >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  static_assert(kSW >= 3, "weight ring too shallow");
  static_assert(kNAcc >= 4, "accumulator ring too shallow");
};

struct Params {
  const uint8_t* packed;
  uint16_t* Y;
  float* partials;      // [slots][2G][MPAD][128] fp32 split-tile partials
  int* counters;        // tile counters: fixed region (single GEMM) or per op at ChainJob::cnt_off (chain)
  int M, K, N, Gk, U, G;
  const ChainJob* jobs; // chain op table (device) or nullptr: a single GEMM
  int n_jobs;
  int* done;            // chain: [n_jobs] CTAs that finished each op, then the exit counter
  int slots;            // chain: partial-slot ring length in ops (1 for a single GEMM)
};

struct Job {
  const uint8_t* packed;
  uint16_t* Y;
  const CUtensorMap* xmap;
  int* counters;
  int kind, N, Gk, U, dep_x, dep_y;
};
__device__ __forceinline__ Job job_at(const Params& p, const CUtensorMap* xmap, int j) {
  Job J;
  if (p.jobs == nullptr) {
    J.packed = p.packed; J.Y = p.Y; J.xmap = xmap; J.counters = p.counters;
    J.kind = kOpGemm; J.N = p.N; J.Gk = p.Gk; J.U = p.U; J.dep_x = -1; J.dep_y = -1;
  } else {
    const ChainJob* c = p.jobs + j;
    J.packed = c->packed; J.Y = c->Y; J.xmap = &c->xmap1; J.counters = p.counters + c->cnt_off;
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
  while (ld_acquire_gpu(&p.done[j]) < p.G) __nanosleep(64);
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

template <int MPAD, int MT, bool SYM>
__global__ void __launch_bounds__(Cfg<MPAD>::kThreads, 1)
    gemm_w4a16_tp_kernel(const __grid_constant__ CUtensorMap xmap, const Params p) {
  using C = Cfg<MPAD>;
  constexpr int SW = C::kSW, NX = C::kNX, NA = C::kNA, NACC = C::kNAcc;
  constexpr int TB = SYM ? 8448 : 8704;
  // barriers: wfull/wempty [SW], xfull/xempty [NX], afull/aempty [NA], accfull/accempty/auxfull [NACC]
  __shared__ __align__(8) uint64_t bars[2 * SW + 2 * NX + 2 * NA + 3 * NACC];
  __shared__ uint32_t s_tmem;
  __shared__ int s_last;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t w_base = smem_u32(smem);
  const uint32_t x_base = w_base + SW * C::kStageW;
  const uint32_t sz_base = x_base + NX * C::kXSlot;           // [NACC][128] {s, z}
  const uint32_t cs_base = sz_base + NACC * 128 * 8;          // [NACC][MPAD] {C, S}
  const uint32_t b0 = smem_u32(&bars[0]);
  const uint32_t WFULL = b0, WEMPTY = WFULL + 8 * SW, XFULL = WEMPTY + 8 * SW, XEMPTY = XFULL + 8 * NX;
  const uint32_t AFULL = XEMPTY + 8 * NX, AEMPTY = AFULL + 8 * NA, ACCFULL = AEMPTY + 8 * NA;
  const uint32_t ACCEMPTY = ACCFULL + 8 * NACC, AUXFULL = ACCEMPTY + 8 * NACC;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const bool chain = p.jobs != nullptr;

  if (threadIdx.x == 0) {
    for (int i = 0; i < SW; ++i) { tcx::mbar_init_a(WFULL + 8 * i, 1); tcx::mbar_init_a(WEMPTY + 8 * i, kDq); }
    for (int i = 0; i < NX; ++i) { tcx::mbar_init_a(XFULL + 8 * i, 1); tcx::mbar_init_a(XEMPTY + 8 * i, 2); }
    for (int i = 0; i < NA; ++i) { tcx::mbar_init_a(AFULL + 8 * i, kDq); tcx::mbar_init_a(AEMPTY + 8 * i, 1); }
    for (int i = 0; i < NACC; ++i) {
      tcx::mbar_init_a(ACCFULL + 8 * i, 1);
      tcx::mbar_init_a(ACCEMPTY + 8 * i, C::kEpi);
      tcx::mbar_init_a(AUXFULL + 8 * i, 4 + 1);   // the 4 k-half-0 dequant warps ({s, z}) + the activation-sum warp
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
    // ---------------- weight producer: one bulk copy per stage of up to kRW units ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      Ring w{0, 0};
      for (int j = 0; j < p.n_jobs; ++j) {
        const Job J = job_at(p, &xmap, j);
        if (J.kind != kOpGemm) continue;
        const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
        for (int u0 = ub; u0 < ue; u0 += kRW) {
          const int nu = min(kRW, ue - u0);
          mbar_wait_a(WEMPTY + 8 * w.i, w.ph ^ 1);
          tcx::expect_tx_a(WFULL + 8 * w.i, nu * TB);
          tcx::bulk_g2s_a(w_base + w.i * C::kStageW, J.packed + (size_t)u0 * TB, nu * TB, WFULL + 8 * w.i, pol);
          w.next(SW);
        }
      }
    }
  } else if (warp == C::kXProdW) {
    // ---------------- activation producer: one 3-D TMA (two 64-k boxes) per unit ----------------
    if (lane == 0) {
      if (!chain) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
        pdl_wait();   // X may be written by the preceding kernel
      }
      Ring x{0, 0};
      int ok_upto = -1;
      for (int j = 0; j < p.n_jobs; ++j) {
        const Job J = job_at(p, &xmap, j);
        if (J.kind != kOpGemm) continue;
        if (J.dep_x > ok_upto) {   // chain: the op that writes this X is complete (all CTAs counted it)
          wait_op(p, J.dep_x);
          ok_upto = J.dep_x;
          fence_proxy_async_global();   // generic-proxy stores of other CTAs -> this TMA (async proxy) read
        }
        const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
        int g = ub % J.Gk;
        for (int u = ub; u < ue; ++u) {
          mbar_wait_a(XEMPTY + 8 * x.i, x.ph ^ 1);
          tcx::expect_tx_a(XFULL + 8 * x.i, C::kXSlot);
          tcx::tma_3d(x_base + x.i * C::kXSlot, J.xmap, 0, 0, 2 * g, XFULL + 8 * x.i);
          x.next(NX);
          if (++g == J.Gk) g = 0;
        }
      }
    }
  } else if (warp == C::kMmaW) {
    // ---------------- MMA issuer: 8 x tcgen05.mma (K = 16) per unit into the unit's own accumulator -------
    Ring x{0, 0}, a{0, 0}, acc{0, 0};
    const uint32_t desc_hi = (uint32_t)(tcx::kDescSW128 >> 32);
    for (int j = 0; j < p.n_jobs; ++j) {
      const Job J = job_at(p, &xmap, j);
      if (J.kind != kOpGemm) continue;
      const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
      for (int u = ub; u < ue; ++u) {
        mbar_wait_a(XFULL + 8 * x.i, x.ph);
        mbar_wait_a(AFULL + 8 * a.i, a.ph);
        mbar_wait_a(ACCEMPTY + 8 * acc.i, acc.ph ^ 1);
        tcx::fence_after();
        if (tcx::elect_one()) {
          const uint32_t d_tmem = tmem + C::kAccCol0 + acc.i * MPAD;
          const uint32_t a_tmem = tmem + a.i * 64;
          const uint32_t lo0 = (1u << 16) | ((x_base + x.i * C::kXSlot) >> 4);   // LBO = 1 | start >> 4
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint32_t lo = lo0 + (uint32_t)(((ks >> 2) * C::kXBox + (ks & 3) * 32) >> 4);
            tcx::mma_ts(d_tmem, a_tmem + ks * 8, ((uint64_t)desc_hi << 32) | lo, C::kIdesc, ks > 0 ? 1u : 0u);
          }
          tcx::commit(AEMPTY + 8 * a.i);
          tcx::commit(XEMPTY + 8 * x.i);
          tcx::commit(ACCFULL + 8 * acc.i);
        }
        __syncwarp();
        x.next(NX);
        a.next(NA);
        acc.next(NACC);
      }
    }
  } else if (warp == C::kXsumW) {
    // ---------------- activation sums: C[m] = sum_k off_k x_k[m], S[m] = sum_k x_k[m] per unit --------------
    // mma.sync m16n8k16 with A = 16 token rows x 16 k (ldmatrix from the SW128 box) and a constant B whose
    // column 0 holds the offsets (1024 on lo nibble slots k%8 in {0,1,4,5}, 64 on hi slots) and column 1 ones:
    // D[m][0] = C[m], D[m][1] = S[m] (products exact, fp32 accumulation).
    const int g8 = lane >> 2, c4 = lane & 3;
    const uint32_t bconst = g8 == 0 ? ((c4 & 1) ? 0x54005400u : 0x64006400u) : (g8 == 1 ? 0x3C003C00u : 0u);
    constexpr int NB = MPAD / 16;
    const int mi = lane >> 3, rr = lane & 7;
    Ring x{0, 0}, acc{0, 0};
    for (int j = 0; j < p.n_jobs; ++j) {
      const Job J = job_at(p, &xmap, j);
      if (J.kind != kOpGemm) continue;
      const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
      for (int u = ub; u < ue; ++u) {
        mbar_wait_a(XFULL + 8 * x.i, x.ph);
        const uint32_t xs = x_base + x.i * C::kXSlot;
        float d[NB][4];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) d[nb][0] = d[nb][1] = d[nb][2] = d[nb][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const int chunk = 2 * (ks & 3) + (mi >> 1);
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const int m = nb * 16 + (mi & 1) * 8 + rr;
            const uint32_t addr = xs + (ks >> 2) * C::kXBox + (m >> 3) * 1024 + (m & 7) * 128 + ((chunk ^ (m & 7)) << 4);
            uint32_t a0, a1, a2, a3;
            tcx::ldsm_x4(addr, a0, a1, a2, a3);
            mma_16816_nv(d[nb], a0, a1, a2, a3, bconst, bconst);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_a(XEMPTY + 8 * x.i);   // this warp's reads of the slot are done
        mbar_wait_a(ACCEMPTY + 8 * acc.i, acc.ph ^ 1);    // the slot's previous unit has been consumed
        if (c4 == 0) {
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const uint32_t at = cs_base + (acc.i * MPAD + nb * 16 + g8) * 8;
            tcx::sts64f(at, d[nb][0], d[nb][1]);
            tcx::sts64f(at + 8 * 8, d[nb][2], d[nb][3]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_a(AUXFULL + 8 * acc.i);
        x.next(NX);
        acc.next(NACC);
      }
    }
  } else if (warp < kDq) {
    // ---------------- dequant: offset codes into a TMEM A buffer ----------------
    const int q = warp & 3, h = warp >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    Ring w{0, 0}, a{0, 0}, acc{0, 0};
    for (int j = 0; j < p.n_jobs; ++j) {
      const Job J = job_at(p, &xmap, j);
      if (J.kind != kOpGemm) continue;
      const int ub = unit_begin(cta, J.U, p.G), ue = unit_begin(cta + 1, J.U, p.G);
      for (int u0 = ub; u0 < ue; u0 += kRW) {
        const int nu = min(kRW, ue - u0);
        mbar_wait_a(WFULL + 8 * w.i, w.ph);
        const uint32_t st = w_base + w.i * C::kStageW;
        for (int jj = 0; jj < nu; ++jj) {
          const uint32_t ub_ = st + jj * TB;
          // chunks 2h, 2h+1 of this row (XOR-permuted layout: conflict-free across the warp's 32 rows)
          const int sw = (row >> 1) & 3;
          const uint4 w0 = lds128(ub_ + row * 64 + (((2 * h) ^ sw) << 4));
          const uint4 w1 = lds128(ub_ + row * 64 + (((2 * h + 1) ^ sw) << 4));
          float sc = 0.f, zf = 8.f;
          if (h == 0) {
            if (SYM) {
              sc = __half2float(__ushort_as_half(tcx::lds16u(ub_ + 8192 + 2 * row)));
            } else {
              const __half2 sz = u2h2(tcx::lds32u(ub_ + 8192 + 4 * row));
              sc = __low2float(sz);
              zf = __high2float(sz);
            }
          }
          const uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
          uint32_t av[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t x0 = wv[i], x8 = wv[i] >> 8;
            av[4 * i + 0] = lop3_and_or(x0, 0x000F000Fu, 0x64006400u);   // k 8i+0, +1: 1024 + q
            av[4 * i + 1] = lop3_and_or(x0, 0x00F000F0u, 0x54005400u);   // k 8i+2, +3:   64 + q
            av[4 * i + 2] = lop3_and_or(x8, 0x000F000Fu, 0x64006400u);   // k 8i+4, +5
            av[4 * i + 3] = lop3_and_or(x8, 0x00F000F0u, 0x54005400u);   // k 8i+6, +7
          }
          mbar_wait_a(AEMPTY + 8 * a.i, a.ph ^ 1);   // the MMAs that last read this A buffer are complete
          tcx::fence_after();
          tcx::st_x32(tmem + lane_base + a.i * 64 + h * 32, av);
          if (h == 0) {   // the unit's {s, z} per row for the epilogue
            mbar_wait_a(ACCEMPTY + 8 * acc.i, acc.ph ^ 1);
            tcx::sts64f(sz_base + (acc.i * 128 + row) * 8, sc, zf);
          }
          tcx::wait_st();
          tcx::fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_a(AFULL + 8 * a.i);
            if (h == 0) mbar_arrive_a(AUXFULL + 8 * acc.i);
          }
          a.next(NA);
          acc.next(NACC);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_a(WEMPTY + 8 * w.i);
        w.next(SW);
      }
    }
  } else {
    // ---------------- epilogue: per-unit scale / offset correction, tile output ----------------
    const int e = warp - C::kEpiW0;
    const int q = e & 3;
    constexpr int kCols = MT / (C::kEpi / 4);   // token columns of this warp
    const int col0 = (e >> 2) * kCols;
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t kEpiThreads = C::kEpi * 32;
    const bool epi0 = warp == C::kEpiW0 && lane == 0;
    if (!chain) pdl_wait();   // Y / workspace writes must follow the preceding kernel
    Ring acc{0, 0};
    for (int j = 0; j < p.n_jobs; ++j) {
      const Job J = job_at(p, &xmap, j);
      if (J.kind == kOpSilu) {
        // SiLU*mul op of a chain (same arithmetic as w4a16_silu_mul), over every epilogue thread of every CTA
        if (epi0) wait_op(p, max(J.dep_x, J.dep_y));
        named_bar_sync(1, kEpiThreads);
        const int F = J.N, vecs = F / 8;
        const long long total = (long long)p.M * vecs;
        const uint16_t* GU = reinterpret_cast<const uint16_t*>(J.packed);
        const int et = (warp - C::kEpiW0) * 32 + lane;
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
      for (int u = ub; u < ue; ++u) {
        mbar_wait_a(ACCFULL + 8 * acc.i, acc.ph);
        mbar_wait_a(AUXFULL + 8 * acc.i, acc.ph);
        tcx::fence_after();
        uint32_t dr[kCols];
#pragma unroll
        for (int c = 0; c < kCols; c += 8) {
          uint32_t r8[8];
          tcx::ld_x8(tmem + lane_base + C::kAccCol0 + acc.i * MPAD + col0 + c, r8);
#pragma unroll
          for (int i = 0; i < 8; ++i) dr[c + i] = r8[i];
        }
        const float2 sz = tcx::lds64f(sz_base + (acc.i * 128 + row) * 8);
        tcx::wait_ld();
#pragma unroll
        for (int c = 0; c < kCols; c += 2) {
          const float4 cs = lds128f(cs_base + (acc.i * MPAD + col0 + c) * 8);   // {C, S} of tokens c, c+1
          const float t0 = fmaf(sz.y, cs.y, cs.x), t1 = fmaf(sz.y, cs.w, cs.z);
          y[c] = fmaf(sz.x, __uint_as_float(dr[c]) - t0, y[c]);
          y[c + 1] = fmaf(sz.x, __uint_as_float(dr[c + 1]) - t1, y[c + 1]);
        }
        tcx::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_a(ACCEMPTY + 8 * acc.i);
        acc.next(NACC);
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
            // split tile: fp32 partial in this CTA's slot, then the last contributor to arrive sums all of them
            // in CTA order (deterministic) and writes Y
            const int slot = 2 * cta + (nseg == 0 ? 0 : 1);
#pragma unroll
            for (int c = 0; c < kCols; ++c) __stcg(&part[((size_t)slot * MPAD + col0 + c) * kTileN + row], y[c]);
            const int c_first = cta_of_unit(tile_u0, J.U, p.G), c_last = cta_of_unit(tile_u1 - 1, J.U, p.G);
            named_bar_sync(1, kEpiThreads);
            if (epi0) {
              __threadfence();
              s_last = atomicAdd(&J.counters[t], 1) == c_last - c_first;
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
              if (epi0) J.counters[t] = 0;   // every contributor has arrived: re-arm for the next launch / run
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
inline int mpad_of(int M) { return M <= 16 ? 16 : (M + 15) / 16 * 16; }

template <int MPAD, int MT, bool SYM>
int launch(const uint16_t* X, const Params& p, cudaStream_t stream) {
  using C = Cfg<MPAD>;
  CUtensorMap map;
  if (int e = encode_x_sw128(&map, X, p.M, p.K, MPAD, 2)) return e;
  auto kern = gemm_w4a16_tp_kernel<MPAD, MT, SYM>;
  static unsigned long long attr = 0;
  if (!ensure_smem_attr(kern, C::kSmem, attr)) return W4A16_ERR_CUDA;
  return launch_pdl(kern, dim3(p.G), dim3(C::kThreads), C::kSmem, stream, map, p) == cudaSuccess ? W4A16_OK
                                                                                                  : W4A16_ERR_CUDA;
}

template <int MPAD, int MT, bool SYM>
int launch_chain(const Params& p, bool cooperative, cudaStream_t stream) {
  using C = Cfg<MPAD>;
  auto kern = gemm_w4a16_tp_kernel<MPAD, MT, SYM>;
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
  return cudaLaunchKernelEx(&cfg, kern, unused, p) == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

template <bool SYM>
int dispatch(const uint16_t* X, const Params& p, bool chain, bool cooperative, cudaStream_t stream) {
  const int M = p.M;
#define W4_TP(MP, MT) return chain ? launch_chain<MP, MT, SYM>(p, cooperative, stream) : launch<MP, MT, SYM>(X, p, stream)
  if (M <= 8) W4_TP(16, 8);
  if (M <= 16) W4_TP(16, 16);
  if (M <= 32) W4_TP(32, 32);
  if (M <= 48) W4_TP(48, 48);
  if (M <= 64) W4_TP(64, 64);
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

extern "C" int w4a16_launch_gemm_tp(const uint16_t* X, const void* packed, uint16_t* Y, int M, int K, int N, int mode,
                                    void* ws, int num_sms, cudaStream_t stream) {
  w4::tp::Params p;
  memset(&p, 0, sizeof(p));
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
  return mode == W4A16_SYM ? w4::tp::dispatch<true>(X, p, false, false, stream)
                           : w4::tp::dispatch<false>(X, p, false, false, stream);
}
