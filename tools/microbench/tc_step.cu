// Hand-off cost of the tcgen05 family's A-buffer ring in isolation: NDQ "dequant" warps
// write a 2-unit A step into one of 3 TMEM buffers (optional tcgen05.st), wait::st, fence, arrive on afull;
// one MMA warp waits afull, fences, issues 16 tcgen05.mma (optional, N tokens) and commits aempty (or
// arrives plainly). Reports cycles per A step on SM 0. One CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=;}" :: "r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(b)) : "memory"); }
__device__ unsigned long long g_cyc[148];
template <int N, bool MMA, bool COMMIT, bool ST, int NDQ>
__global__ void __launch_bounds__(32 * (NDQ + 1), 1) k(int steps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t afull[3], aempty[3];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(&afull[i])), "r"(NDQ));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&aempty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  if (warp < NDQ) {   // "dequant" warps: lane quarter warp % 4
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t ph = 0;
    for (int i = 0, b = 0; i < steps; ++i) {
      wait(&aempty[b], ph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (ST) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int h = 0; h < 4 / (NDQ / 4); ++h) {
            const uint32_t addr = tmem + lane_base + b * 128 + u * 64 + ((warp >> 2) * (4 / (NDQ / 4)) + h) * 16;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" :: "r"(addr), "r"(0u));
          }
        asm volatile("tcgen05.wait::st.sync.aligned;");
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) arrive(&afull[b]);
      if (++b == 3) { b = 0; ph ^= 1; }
    }
  } else {   // MMA warp
    uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint64_t dbase = ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
    uint64_t bdesc = dbase | ((su(smem) >> 4) & 0x3FFF);
    const uint32_t d = tmem + 384;
    uint32_t ph = 0;
    unsigned long long t0 = clock64();
    for (int i = 0, b = 0; i < steps; ++i) {
      wait(&afull[b], ph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t pred;
      asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
      if (pred) {
        if (MMA) {
#pragma unroll
          for (int ks = 0; ks < 16; ++ks)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                         :: "r"(d), "r"(tmem + b * 128 + ks * 8), "l"(bdesc + (ks & 7) * 2), "r"(idesc), "r"(1));
        }
        if (COMMIT) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su(&aempty[b])) : "memory");
        else arrive(&aempty[b]);
      }
      __syncwarp();
      if (++b == 3) { b = 0; ph ^= 1; }
    }
    unsigned long long t1 = clock64();
    if (lane == 0) g_cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}
template <int N, bool MMA, bool COMMIT, bool ST, int NDQ> int run(const char* what) {
  auto kern = k<N, MMA, COMMIT, ST, NDQ>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
  const int steps = 4000;
  kern<<<148, 32 * (NDQ + 1), 40 * 1024>>>(steps); CK(cudaDeviceSynchronize());
  kern<<<148, 32 * (NDQ + 1), 40 * 1024>>>(steps); CK(cudaDeviceSynchronize());
  unsigned long long c[148]; cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
  printf("%-44s N=%2d dq warps %2d: %.0f cycles per A step\n", what, N, NDQ, (double)c[0] / steps);
  return 0;
}
int main() {
  run<32, false, false, false, 16>("no MMA, plain arrive, no TMEM stores");
  run<32, false, true, false, 16>("no MMA, commit, no TMEM stores");
  run<32, true, true, false, 16>("16 MMAs, commit, no TMEM stores");
  run<64, true, true, false, 16>("16 MMAs, commit, no TMEM stores");
  run<32, false, true, true, 16>("no MMA, commit, TMEM stores (2 units)");
  run<32, true, true, true, 16>("16 MMAs, commit, TMEM stores (2 units)");
  run<64, true, true, true, 16>("16 MMAs, commit, TMEM stores (2 units)");
  run<32, true, true, true, 4>("16 MMAs, commit, TMEM stores, 4 dq warps");
  return 0;
}
