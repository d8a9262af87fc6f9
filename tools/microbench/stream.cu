// Streaming-read microbenchmarks for the W4A16 weight stream: which bulk-copy pattern reaches HBM peak?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" :: "r"(su(b)), "r"(ph) : "memory");
}
struct Cfg { int chunk; int stages; int contiguous; int small; int policy; size_t small_stride; };

// one producer lane; NCONS consumer warps touch 16 B per lane and release.
__global__ void stream_kernel(const uint8_t* __restrict__ p, const uint8_t* __restrict__ q, size_t nchunks, Cfg c, int* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
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
  size_t c0 = c.contiguous ? blockIdx.x * per : blockIdx.x;
  size_t step = c.contiguous ? 1 : gridDim.x;
  size_t cend = c.contiguous ? min(nchunks, c0 + per) : nchunks;
  int acc = 0;
  int stage_bytes = c.chunk + 512;
  if (warp == 0) {
    if (tid == 0) {
      uint64_t pol;
      if (c.policy == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      int s = 0; uint32_t ph = 0;
      for (size_t i = c0; i < cend; i += step) {
        wait(&empty[s], ph ^ 1);
        uint32_t fb = su(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(fb), "r"(c.chunk + 256 * c.small));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     :: "r"(su(smem + s * stage_bytes)), "l"(p + i * c.chunk), "r"(c.chunk), "r"(fb), "l"(pol) : "memory");
        for (int j = 0; j < c.small; ++j)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       :: "r"(su(smem + s * stage_bytes + c.chunk + 256 * j)), "l"(q + ((i * 2 + j) * c.small_stride) % (size_t(1) << 30)), "r"(256), "r"(fb), "l"(pol) : "memory");
        if (++s == c.stages) { s = 0; ph ^= 1; }
      }
    }
  } else {
    int s = 0; uint32_t ph = 0;
    for (size_t i = c0; i < cend; i += step) {
      wait(&full[s], ph);
      const int4* v = (const int4*)(smem + s * stage_bytes);
      for (int k = tid - 32; k < c.chunk / 16; k += blockDim.x - 32) acc ^= v[k].x;
      __syncwarp();
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(&empty[s])));
      if (++s == c.stages) { s = 0; ph ^= 1; }
    }
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  size_t nbytes = (size_t)4 << 30;
  uint8_t *buf, *sbuf; int* io;
  CK(cudaMalloc(&buf, nbytes)); CK(cudaMalloc(&sbuf, (size_t)1 << 30)); CK(cudaMalloc(&io, 64));
  CK(cudaMemset(buf, 1, nbytes)); CK(cudaMemset(sbuf, 1, (size_t)1 << 30));
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct T { const char* name; Cfg c; int threads; };
  T tests[] = {
    {"16K x8 interleaved (mb baseline)", {16384, 8, 0, 0, 0, 0}, 256},
    {"16K x8 contiguous", {16384, 8, 1, 0, 0, 0}, 256},
    {"8K x12 contiguous", {8192, 12, 1, 0, 0, 0}, 256},
    {"8K x12 contiguous evict_first", {8192, 12, 1, 0, 1, 0}, 256},
    {"8K x12 contiguous +2x256B strided", {8192, 12, 1, 2, 0, 114688}, 256},
    {"8K x12 contiguous +2x256B strided evict_first", {8192, 12, 1, 2, 1, 114688}, 256},
    {"8K x12 interleaved +2x256B strided", {8192, 12, 0, 2, 0, 114688}, 256},
    {"8K x20 contiguous +2x256B strided", {8192, 20, 1, 2, 0, 114688}, 256},
    {"16K x12 contiguous +2x256B", {16384, 12, 1, 2, 0, 114688}, 256},
    {"8K x12 contiguous 12 warps", {8192, 12, 1, 2, 0, 114688}, 384},
  };
  for (auto& t : tests) {
    size_t nchunks = nbytes / t.c.chunk;
    int smem = t.c.stages * (t.c.chunk + 512);
    stream_kernel<<<148, t.threads, smem>>>(buf, sbuf, nchunks, t.c, io); CK(cudaDeviceSynchronize());
    float best = 1e9, ms;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); stream_kernel<<<148, t.threads, smem>>>(buf, sbuf, nchunks, t.c, io); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    double bytes = (double)nbytes * (1.0 + 512.0 * t.c.small / 2 / t.c.chunk);
    printf("%-50s %8.1f GB/s\n", t.name, bytes / best / 1e6);
  }
  return 0;
}
