// How expensive is issuing bulk / tensor TMA copies from one producer thread? (W4A16 weight stream design)
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" :: "r"(su(b)), "r"(ph) : "memory");
}
struct Cfg { int chunk; int nbulk; int ntma; int stages; int nprod; };
__device__ unsigned long long g_cycles[148];

__global__ void k(const uint8_t* __restrict__ p, const __grid_constant__ CUtensorMap xmap, size_t nchunks, Cfg c, int* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  int tid = threadIdx.x, warp = tid / 32;
  int ncons = blockDim.x / 32 - 1;
  if (tid == 0) {
    for (int s = 0; s < c.stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(&empty[s])), "r"(ncons));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  size_t c0 = blockIdx.x * per, cend = min(nchunks, c0 + per);
  int stage_bytes = c.chunk + 16384;
  int acc = 0;
  if (warp == 0) {
    if (tid == 0) {
      unsigned long long cyc = 0;
      int s = 0; uint32_t ph = 0;
      for (size_t i = c0; i < cend; ++i) {
        wait(&empty[s], ph ^ 1);
        unsigned long long t0 = clock64();
        uint32_t fb = su(&full[s]);
        int xbytes = c.ntma * 2048;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(fb), "r"(c.chunk + xbytes));
        for (int t = 0; t < c.ntma; ++t)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       :: "r"(su(smem + s * stage_bytes + c.chunk + t * 2048)), "l"((uint64_t)&xmap), "r"((int)((i * 64 + t * 64) % 8192)), "r"(0), "r"(fb) : "memory");
        int piece = c.chunk / c.nbulk;
        for (int b = 0; b < c.nbulk; ++b)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(su(smem + s * stage_bytes + b * piece)), "l"(p + i * c.chunk + b * piece), "r"(piece), "r"(fb) : "memory");
        cyc += clock64() - t0;
        if (++s == c.stages) { s = 0; ph ^= 1; }
      }
      g_cycles[blockIdx.x] = cyc / (cend - c0);
    }
  } else {
    int s = 0; uint32_t ph = 0;
    for (size_t i = c0; i < cend; ++i) {
      wait(&full[s], ph);
      acc ^= *(const int*)(smem + s * stage_bytes + (tid - 32) * 16);
      __syncwarp();
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(&empty[s])));
      if (++s == c.stages) { s = 0; ph ^= 1; }
    }
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  size_t nbytes = (size_t)4 << 30;
  uint8_t* buf; uint16_t* x; int* io;
  CK(cudaMalloc(&buf, nbytes)); CK(cudaMalloc(&x, 64 * 8192 * 2)); CK(cudaMalloc(&io, 64));
  CK(cudaMemset(buf, 1, nbytes)); CK(cudaMemset(x, 0, 64 * 8192 * 2));
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t dims[2] = {8192, 16}; cuuint64_t str[1] = {8192 * 2}; cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) { printf("enc fail\n"); return 1; }
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  Cfg tests[] = {
    {16384, 1, 0, 8, 1}, {17408, 1, 0, 8, 1}, {17408, 1, 4, 8, 1}, {17408, 2, 0, 8, 1}, {17408, 2, 4, 8, 1},
    {34816, 1, 0, 4, 1}, {34816, 1, 8, 4, 1}, {8704, 1, 2, 12, 1}, {8704, 1, 0, 12, 1}, {34816, 4, 0, 4, 1},
  };
  for (auto& c : tests) {
    size_t nchunks = nbytes / c.chunk;
    int smem = c.stages * (c.chunk + 16384);
    if (smem > 220 * 1024) { printf("skip\n"); continue; }
    k<<<148, 256, smem>>>(buf, map, nchunks, c, io); CK(cudaDeviceSynchronize());
    float best = 1e9, ms;
    for (int r = 0; r < 3; ++r) { cudaEventRecord(e0); k<<<148, 256, smem>>>(buf, map, nchunks, c, io); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    unsigned long long cyc[148]; cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(cyc));
    double avg = 0; for (int i = 0; i < 148; ++i) avg += cyc[i]; avg /= 148;
    printf("chunk %6d bulk %d tma %d stages %2d: %7.1f GB/s (weights), issue %.0f cycles/stage\n", c.chunk, c.nbulk, c.ntma, c.stages,
           (double)(nbytes / c.chunk) * c.chunk / best / 1e6, avg);
  }
  return 0;
}
