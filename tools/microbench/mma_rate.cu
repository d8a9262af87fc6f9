// tcgen05.mma kind::f16 issue/throughput rate vs N, A from TMEM (TS) or SMEM (SS); one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ unsigned long long g_cyc[148];
template <int N, bool TS, int COMMIT, bool FENCE, int NACC = 1>
__global__ void __launch_bounds__(128, 1) k(int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar, bar2;
  int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar2))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = s_tmem;
  if (warp == 1) {
    uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint64_t dbase = ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
    uint64_t bdesc = dbase | ((su(smem) >> 4) & 0x3FFF);
    uint64_t adesc = dbase | ((su(smem + 32768) >> 4) & 0x3FFF);
    uint32_t d = tmem + 256;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t pred;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
      if (pred) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (TS)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                         :: "r"(d + (ks % NACC) * 64), "r"(tmem + ks * 8), "l"(bdesc + ks * 2), "r"(idesc), "r"(1));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                         :: "r"(d), "l"(adesc + ks * 2), "l"(bdesc + ks * 2), "r"(idesc), "r"(1));
        }
      }
      __syncwarp();
      if (FENCE) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (COMMIT && (it % COMMIT) == COMMIT - 1) {
        uint32_t pr;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pr));
        if (pr) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su(&bar2)) : "memory");
        __syncwarp();
      }
    }
    unsigned long long t1 = clock64();
    uint32_t pred;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    if (pred) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su(&bar)) : "memory");
    __syncwarp();
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" :: "r"(su(&bar)) : "memory");
    unsigned long long t2 = clock64();
    if (lane == 0) g_cyc[blockIdx.x] = ((t1 - t0) << 32) | (t2 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
template <int N, bool TS, int COMMIT = 0, bool FENCE = false, int NACC = 1> int run(int grid) {
  auto kern = k<N, TS, COMMIT, FENCE, NACC>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024));
  int iters = 2000;
  kern<<<grid, 128, 70 * 1024>>>(iters); CK(cudaDeviceSynchronize());
  kern<<<grid, 128, 70 * 1024>>>(iters); CK(cudaDeviceSynchronize());
  unsigned long long c[148]; cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
  double issue = (double)(c[0] >> 32) / (iters * 8), total = (double)(c[0] & 0xffffffffull) / (iters * 8);
  printf("nacc %d commit/%d fence %d %s N=%3d grid=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma -> %.0f MAC/cyc/SM\n", NACC, COMMIT, (int)FENCE, TS ? "TS" : "SS", N, grid, issue, total,
         128.0 * N * 16 / total);
  return 0;
}
int main() {
  run<16, true>(148); run<16, true, 0, false, 2>(148); run<16, true, 0, false, 4>(148);
  run<32, true>(148); run<32, true, 0, false, 2>(148); run<64, true, 0, false, 2>(148);
  return 0;
}
