// Does concurrent tcgen05.st (other warps) or TMA bulk traffic slow tcgen05.mma (TS, M=128, N=16)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ unsigned long long g_cyc[148];
__device__ volatile int g_stop[148];
template <int MODE>  // bit0: STTM warps, bit1: bulk-copy producer, bit2: D at col 384 and A rotating over 0..383
__global__ void __launch_bounds__(384, 1) k(const uint8_t* __restrict__ gsrc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t bar, tbar;
  __shared__ volatile int stop;
  int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&tbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
  }
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = s_tmem;
  if (warp == 1) {
    uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint64_t dbase = ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
    uint32_t d = (MODE & 4) ? tmem + 384 : tmem + 256;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t acol = (MODE & 4) ? (it % 6) * 64 : 0;
      uint32_t xs = su(smem) + (it % 4) * 4096;
      uint32_t pred;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
      if (pred) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint64_t bdesc = dbase | (((xs + (ks >> 2) * 2048 + (ks & 3) * 32) >> 4) & 0x3FFF);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                       :: "r"(d), "r"(tmem + acol + ks * 8), "l"(bdesc), "r"(idesc), "r"(1));
        }
      }
      __syncwarp();
    }
    unsigned long long t1 = clock64();
    if (lane == 0) { g_cyc[blockIdx.x] = t1 - t0; stop = 1; }
  } else if (warp >= 4 && (MODE & 1)) {
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = i * lane;
    int q = warp & 3;
    while (!stop) {
      uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (MODE & 4 ? ((warp - 4) >> 2) * 32 + 64 * (1 + (warp & 1)) : 128 + ((warp - 4) >> 2) * 32);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      for (int i = 0; i < 32; ++i) v[i] += 1;
    }
  } else if (warp == 0 && (MODE & 2)) {
    if (lane == 0) {
      uint32_t ph = 0; size_t off = (size_t)blockIdx.x * (64 << 20);
      while (!stop) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&tbar)), "r"(34816));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su(smem + 32768)), "l"(gsrc + off), "r"(34816), "r"(su(&tbar)) : "memory");
        asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" :: "r"(su(&tbar)), "r"(ph) : "memory");
        ph ^= 1; off = (off + 34816) % ((size_t)148 << 26);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
template <int MODE> int run(const uint8_t* g) {
  auto kern = k<MODE>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
  int iters = 4000;
  kern<<<148, 384, 80 * 1024>>>(g, iters); CK(cudaDeviceSynchronize());
  kern<<<148, 384, 80 * 1024>>>(g, iters); CK(cudaDeviceSynchronize());
  unsigned long long c[148]; cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
  double avg = 0; for (int i = 0; i < 148; ++i) avg += c[i]; avg /= 148;
  printf("mode %d (sttm=%d bulk=%d kernel-cols=%d): %.1f cyc/mma\n", MODE, MODE & 1, (MODE >> 1) & 1, (MODE >> 2) & 1, avg / (iters * 8));
  return 0;
}
int main() {
  uint8_t* g; CK(cudaMalloc(&g, (size_t)148 << 26)); CK(cudaMemset(g, 1, (size_t)148 << 26));
  run<0>(g); run<4>(g); run<1>(g); run<5>(g); run<2>(g); run<6>(g); run<7>(g);
  return 0;
}
