// Box microbenchmarks: mma.sync throughput, streaming-read bandwidth
// (LDG.128 and cp.async.bulk), dequant ALU loop. Standalone; not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void mma_tput(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 11;
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 12345.f) out[0] = s;
}

__global__ void ldg_read(const int4* __restrict__ p, size_t n16, int* out) {
  int acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { int4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x7fffffff) out[0] = acc;
}

// cp.async.bulk global->shared ring, one producer thread, consumers just touch data.
template <int STAGES, int CHUNK>
__global__ void bulk_read(const uint8_t* __restrict__ p, size_t nbytes, int* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&full[s])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&empty[s])), "r"(blockDim.x / 32 - 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t nchunks = nbytes / CHUNK;
  int warp = tid / 32;
  int acc = 0;
  if (warp == 0) {
    if (tid == 0) {
      int s = 0; uint32_t ph = 0; int n = 0;
      for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++n) {
        if (n >= STAGES) {
          uint32_t bar = __cvta_generic_to_shared(&empty[s]);
          asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" :: "r"(bar), "r"(ph ^ 1));
        }
        uint32_t fb = __cvta_generic_to_shared(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(fb), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"((uint32_t)__cvta_generic_to_shared(smem + s * CHUNK)), "l"(p + c * CHUNK), "r"(CHUNK), "r"(fb) : "memory");
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    int s = 0; uint32_t ph = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      uint32_t fb = __cvta_generic_to_shared(&full[s]);
      asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" :: "r"(fb), "r"(ph));
      const int4* q = (const int4*)(smem + s * CHUNK);
      for (int i = tid - 32; i < CHUNK / 16; i += blockDim.x - 32) { int4 v = q[i]; acc ^= v.x ^ v.w; }
      __syncwarp();
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&empty[s])));
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

// dequant ALU loop: per u32 word 1 SHF + 4 LOP3 + 2 HSUB2 + 2 HFMA2 (+ optional 4 HMUL2)
template <bool SCALE>
__global__ void dq_loop(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t w = in[threadIdx.x];
  __half2 z = __float2half2_rn(1032.f), z16 = __float2half2_rn(-72.f), inv16 = __float2half2_rn(0.0625f), s = __float2half2_rn(0.01f);
  __half2 acc = __float2half2_rn(0.f);
  for (int it = 0; it < iters; ++it) {
    uint32_t w8 = w >> 8;
    uint32_t r0 = (w & 0x000F000F) | 0x64006400, r1 = (w & 0x00F000F0) | 0x64006400;
    uint32_t r2 = (w8 & 0x000F000F) | 0x64006400, r3 = (w8 & 0x00F000F0) | 0x64006400;
    __half2 h0 = __hsub2(*(__half2*)&r0, z), h2 = __hsub2(*(__half2*)&r2, z);
    __half2 h1 = __hfma2(*(__half2*)&r1, inv16, z16), h3 = __hfma2(*(__half2*)&r3, inv16, z16);
    if (SCALE) { h0 = __hmul2(h0, s); h1 = __hmul2(h1, s); h2 = __hmul2(h2, s); h3 = __hmul2(h3, s); }
    acc = __hadd2(acc, __hadd2(__hadd2(h0, h1), __hadd2(h2, h3)));
    w = w * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = *(uint32_t*)&acc;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d L2 %d MB smem/block optin %zu clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin, clk);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  float* fo; CK(cudaMalloc(&fo, 1024));
  int* io; CK(cudaMalloc(&io, 1024));
  // mma.sync
  for (int wpb : {4, 8, 16}) {
    int iters = 4096, blocks = prop.multiProcessorCount * 4;
    mma_tput<<<blocks, 32 * wpb>>>(fo, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); mma_tput<<<blocks, 32 * wpb>>>(fo, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * blocks * wpb;
    printf("mma.sync m16n8k16 f16->f32: warps/blk %d blocks %d: %.1f TFLOP/s (%.3f ms)\n", wpb, blocks, flops / ms / 1e9, ms);
  }
  // streaming read
  size_t nbytes = (size_t)4 << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, nbytes)); CK(cudaMemset(buf, 1, nbytes));
  for (int bpsm : {2, 4, 8}) {
    int blocks = prop.multiProcessorCount * bpsm;
    ldg_read<<<blocks, 512>>>((const int4*)buf, nbytes / 16, io); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); ldg_read<<<blocks, 512>>>((const int4*)buf, nbytes / 16, io); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("LDG.128 read (unroll4, %d blk/SM x512): %.1f GB/s\n", bpsm, nbytes / best / 1e6);
  }
  {
    auto k = bulk_read<8, 16384>;
    int smem = 8 * 16384;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int bpsm : {1}) {
      int blocks = prop.multiProcessorCount * bpsm;
      k<<<blocks, 256, smem>>>(buf, nbytes, io); CK(cudaDeviceSynchronize());
      float best = 1e9;
      for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k<<<blocks, 256, smem>>>(buf, nbytes, io); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
      printf("cp.async.bulk read (8x16KB ring, 1 blk/SM): %.1f GB/s\n", nbytes / best / 1e6);
    }
  }
  {
    auto k = bulk_read<12, 16384>;
    int smem = 12 * 16384;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int blocks = prop.multiProcessorCount;
    k<<<blocks, 256, smem>>>(buf, nbytes, io); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k<<<blocks, 256, smem>>>(buf, nbytes, io); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("cp.async.bulk read (12x16KB ring, 1 blk/SM): %.1f GB/s\n", nbytes / best / 1e6);
  }
  {
    auto k = bulk_read<6, 16384>;
    int smem = 6 * 16384;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int blocks = prop.multiProcessorCount * 2;
    k<<<blocks, 256, smem>>>(buf, nbytes, io); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k<<<blocks, 256, smem>>>(buf, nbytes, io); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("cp.async.bulk read (6x16KB ring, 2 blk/SM): %.1f GB/s\n", nbytes / best / 1e6);
  }
  // dequant ALU
  {
    uint32_t* dbuf; CK(cudaMalloc(&dbuf, 64 << 20));
    int blocks = prop.multiProcessorCount * 8, iters = 8192;
    for (int sc = 0; sc < 2; ++sc) {
      auto k = sc ? dq_loop<true> : dq_loop<false>;
      k<<<blocks, 256>>>(dbuf, dbuf, 16); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); k<<<blocks, 256>>>(dbuf, dbuf, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double w = 8.0 * iters * blocks * 256;
      printf("dequant loop (scale=%d): %.2f T weights/s\n", sc, w / ms / 1e9);
    }
  }
  return 0;
}
