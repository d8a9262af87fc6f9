// common.cuh — sm_100a PTX helpers shared by the w4a16 kernels (mbarrier, bulk copies, fences).
// Internal to libw4a16.so; not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "w4a16.h"

namespace w4 {

// GEMM workspace: a fixed region of tile counters (same offset for every shape, so GEMMs of different N
// can share one workspace), then the fp32 split-K partials (include/w4a16.h).
// Single-GEMM tile counters: one per 128-byte line (counters of neighbouring tiles on one line serialise the
// CTAs' atomics; the chain's sync words showed 4 % from spreading them)
constexpr int kCounterStride = 32;
constexpr size_t kCounterBytes = (size_t)(W4A16_MAX_N / 128) * 4 * kCounterStride;

// One op of a chain: the device copy of a w4a16_chain_plan entry (include/w4a16.h), shared by both GEMM
// families (the activation tensor maps are encoded for the family the plan was made for).
enum { kOpGemm = W4A16_OP_GEMM, kOpSilu = W4A16_OP_SILU_MUL, kOpAllReduce = W4A16_OP_ALLREDUCE };
struct alignas(64) ChainJob {
  CUtensorMap xmapR;       // activation boxes of one stage's units (3-D SWIZZLE_128B)
  CUtensorMap xmap1;       // activation box of one unit
  const uint8_t* packed;   // GEMM: packed weights.  SILU: GU [M][2N]
  uint16_t* Y;             // GEMM: Y [M][N].  SILU: out [M][N]
  int kind, K, N, Gk, U;
  int dep_x;               // earlier op whose completion this op's X reads wait for (-1: none)
  int dep_y;               // earlier op whose completion this op's Y writes wait for (WAR / WAW; -1: none)
  int cnt_off;             // this op's first tile counter (and first tile-ready flag)
  // Tile-level RAW dependency (family A chains): X is a column range of the Y of GEMM op dep_x, so the
  // activation k-group g of this op is complete once that op's tile xf_off + g is written (its ready flag,
  // at flags[xf_off + g], reached the run number). -1: wait for the whole op dep_x instead.
  int xf_off;
  int pub_tiles;           // 1: publish this op's tile-ready flags (a later op reads its Y tile by tile)
  int epi;                 // GEMM: 0 = plain Y, 1 = SiLU*mul of [64 gate | 64 up] tiles into Y [M][N/2]
  int xf_mul;              // producer tiles per activation k-group (1, or 2 when X is a GEMM_SILU output)
  int n_tiles;             // job 0: tiles of all GEMM ops (counters, then as many tile-ready flags, in the workspace)
  // ALLREDUCE (include/w4a16.h): every rank's partial as mapped here (rank order; peer-load path), the
  // multicast address of the partial (NVLS path, else nullptr), this rank's tile counters of the op's slot
  // (local), the group's run counter (local). Job 0 also carries the run counter when the chain has
  // ALLREDUCE ops (advanced at chain end).
  const uint16_t* peer_x[W4A16_MAX_PEERS];
  const uint16_t* mc_x;
  uint32_t* my_tiles;
  uint32_t* epoch;
  int world;
  // GEMM whose Y is the partial of the ALLREDUCE right after it: tile t of Y written -> bump tile t's counter
  // in every rank's flag area (through the multicast address, or through each peer's mapping); ar_prev = the
  // chain's previous ALLREDUCE, complete on this rank before the first bump (peers are done reading).
  uint32_t* ar_tiles_mc;
  uint32_t* ar_tiles_peer[W4A16_MAX_PEERS];
  int ar_world;
  int ar_prev;
};
// Flag area of a peer group (include/w4a16.h): word 0 = the group's run counter, then per ALLREDUCE slot
// W4A16_AR_MAX_TILES tile counters (each rank adds 1 per run: `world` * runs when a tile is complete).
constexpr int kFlagHead = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W4_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W4_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Same wait / arrive on a precomputed shared-memory address (no generic->shared conversion in hot loops).
__device__ __forceinline__ void mbar_wait_a(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W4_WAITA_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W4_WAITA_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Wait with a suspend-time hint: the thread is suspended (not re-issuing polls) until the phase completes
// or the hint (ns) expires.
__device__ __forceinline__ void mbar_wait_suspend(uint64_t* bar, uint32_t parity, uint32_t hint_ns) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W4_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra W4_WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(hint_ns)
      : "memory");
}
// Same wait with a nanosleep back-off between polls (keeps idle warps off the shared-memory pipe).
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe of a phase (mbarrier.test_wait never suspends the thread, unlike try_wait, which may wait
// for a system-dependent time before returning false): for polling loops that interleave other work.
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(ns);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D bulk async copy global -> shared, completion counted on `bar` (TMA engine, SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Programmatic dependent launch (sm_90+): wait for the preceding grid's completion and memory flush /
// allow the next grid in the stream (launched with the PDL attribute) to start scheduling its CTAs.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 ldg128_nc(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// int4 -> fp16 pair tricks. With the nibble interleave of include/w4a16.h:
//   (w & 0x000F000F) | 0x6400_6400 = {1024 + q(k0), 1024 + q(k1)}         (exact fp16)
//   (w & 0x00F000F0) | 0x6400_6400 = {1024 + 16 q(k2), 1024 + 16 q(k3)}   (exact fp16)
// and the same on (w >> 8) for k4..k7. (1024+q) - (1024+z) and (1024+16q)/16 - (64+z) are exact.
__device__ __forceinline__ uint32_t lop3_mask_or(uint32_t w, uint32_t mask) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "r"(mask), "r"(0x64006400u));  // (a & b) | c
  return r;
}
__device__ __forceinline__ uint32_t hsub2_u32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t hfma2_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t hmul2_u32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t h2_bcast(uint16_t h) { return (uint32_t)h | ((uint32_t)h << 16); }
__device__ __forceinline__ __half2 u2h2(uint32_t x) { return *reinterpret_cast<const __half2*>(&x); }
__device__ __forceinline__ uint32_t h22u(__half2 h) { return *reinterpret_cast<const uint32_t*>(&h); }

// Zero-point magic pair for a row: {64 + z, 1024 + z} (exact). With v = (w & 0x000F000F) | 0x64006400 the
// exact (q - z) pair is v - zp.hi; with v = (w & 0x00F000F0) | 0x64006400 it is v / 16 - zp.lo. Written
// with half2 intrinsics so ptxas folds the half broadcasts and the negation into operand modifiers.
__device__ __forceinline__ __half2 zero_pair(__half z) { return __hadd2(__half2half2(z), __floats2half2_rn(64.f, 1024.f)); }
__device__ __forceinline__ uint32_t dq_lo(uint32_t w, __half2 zp) {
  return h22u(__hsub2(u2h2(lop3_mask_or(w, 0x000F000Fu)), __high2half2(zp)));
}
__device__ __forceinline__ uint32_t dq_hi(uint32_t w, __half2 zp) {
  return h22u(__hfma2(u2h2(lop3_mask_or(w, 0x00F000F0u)), __float2half2_rn(0.0625f), __hneg2(__low2half2(zp))));
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts32f(uint32_t addr, float a) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(a) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
// Release-increment of a global counter (prior writes of the CTA, ordered by a preceding barrier, become
// visible first) without waiting for the result; and the matching acquire load.
__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
  asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Relaxed load (no ordering): for polling several flags at once; follow a successful poll with fence_acquire_gpu.
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Acquire-only fence (SASS: CCTL.IVALL, no MEMBAR): after relaxed polls that observed a release, orders the later
// reads. fence.acq_rel.gpu would add a MEMBAR.ALL.GPU, which in a thread with bulk copies in flight cost ~3.5 %
// of the chain (measured with the fence removed).
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acquire.gpu;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// System-scope (cross-GPU, NVLink peer memory) release store / acquire load of a flag word.
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// NVLS (multicast) access: `mc` is an address in a multicast mapping. ld_reduce returns the sum over every
// device bound to the object of 8 fp16 values (fp32 accumulation in the switch, one rounding); red adds to
// the word on every device.
__device__ __forceinline__ uint4 multimem_ld_reduce_f16x8(const void* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
__device__ __forceinline__ void multimem_red_add_u32(uint32_t* mc, uint32_t v) {
  asm volatile("multimem.red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_sys_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// (w & mask) | magic in one LOP3.
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t w, uint32_t mask, uint32_t magic) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "r"(mask), "r"(magic));
  return r;
}
// Same MMA as mma_16816, not volatile: a pure register function the scheduler may interleave freely.
__device__ __forceinline__ void mma_16816_nv(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                             uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// D = A(16x16, row) * B(16x8, col) + C, fp16 inputs, fp32 accumulate (legacy tensor path, SASS HMMA).
__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                          uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// SiLU(gate) * up on 8 fp16 pairs, fp32 arithmetic, one RNE to fp16 (w4a16_silu_mul and chain SILU ops).
__device__ __forceinline__ uint4 silu_mul_vec(uint4 g, uint4 u) {
  const __half2* gh = reinterpret_cast<const __half2*>(&g);
  const __half2* uh = reinterpret_cast<const __half2*>(&u);
  uint4 r;
  __half2* rh = reinterpret_cast<__half2*>(&r);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 gf = __half22float2(gh[j]), uf = __half22float2(uh[j]);
    const float a = gf.x / (1.0f + __expf(-gf.x)) * uf.x;
    const float b = gf.y / (1.0f + __expf(-gf.y)) * uf.y;
    rh[j] = __floats2half2_rn(a, b);
  }
  return r;
}

}  // namespace w4
