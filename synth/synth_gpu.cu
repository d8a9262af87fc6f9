// synth_gpu.cu — device implementation of the synthetic input generator in synth.h (bit-identical to
// synth.c). Input generation only; no method arithmetic. Used by tests and bench.py to create inputs
// (up to tens of GB of weights) directly in HBM.
#include "synth.h"
#include <cuda_runtime.h>
#include <cuda_fp16.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t u_at(uint64_t stream, uint64_t i) { return mix64(stream + (i + 1) * 0x9E3779B97F4A7C15ull); }
static uint64_t h_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static uint64_t h_stream(uint64_t seed, uint64_t t) { return h_mix64(h_mix64(seed) ^ (t * 0xD1B54A32D192ED03ull)); }

struct SynthArgs { uint64_t st, st2; int kind, rows, cols; int outc[SYNTH_X_OUTLIER_N]; };

__global__ void synth_kernel(SynthArgs a, uint16_t* __restrict__ out, uint64_t total) {
  for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t u = u_at(a.st, idx);
    int v = (int)((u & 0xFFFF) + ((u >> 16) & 0xFFFF) + ((u >> 32) & 0xFFFF) + (u >> 48)) - 131070;
    int r = (int)(idx / (uint64_t)a.cols), c = (int)(idx % (uint64_t)a.cols);
    int e;
    if (a.kind == SYNTH_WEIGHT) {
      uint64_t g = (uint64_t)(r / 128) * (uint64_t)a.cols + (uint64_t)c;
      e = -SYNTH_W_SHIFT + ((u_at(a.st2, g) % SYNTH_W_OUTLIER_MOD) == 0 ? SYNTH_W_OUTLIER_LOG2 : 0);
    } else {
      int o = 0;
#pragma unroll
      for (int j = 0; j < SYNTH_X_OUTLIER_N; ++j) o |= (a.outc[j] == c);
      e = -SYNTH_X_SHIFT + (o ? SYNTH_X_OUTLIER_LOG2 : 0);
    }
    float f = __fmul_rn((float)v, __int_as_float((127 + e) << 23));   // exact: |v| < 2^18 times a power of two
    __half h = __float2half_rn(f);
    out[idx] = __half_as_ushort(h);
  }
}

extern "C" int synth_fill_gpu(uint64_t seed, uint64_t tensor_id, int kind, int rows, int cols, uint16_t* out, void* stream) {
  if (!out || rows < 0 || cols <= 0 || (kind != SYNTH_WEIGHT && kind != SYNTH_ACT)) return -1;
  SynthArgs a;
  a.st = h_stream(seed, tensor_id);
  a.kind = kind; a.rows = rows; a.cols = cols;
  if (kind == SYNTH_WEIGHT) a.st2 = h_stream(seed, tensor_id ^ 0x5A5A5A5A00000000ull);
  else {
    a.st2 = 0;
    uint64_t st3 = h_stream(seed, tensor_id ^ 0xA5A5A5A500000000ull);
    for (int j = 0; j < SYNTH_X_OUTLIER_N; ++j) a.outc[j] = (int)(h_mix64(st3 + ((uint64_t)j + 1) * 0x9E3779B97F4A7C15ull) % (uint64_t)cols);
  }
  uint64_t total = (uint64_t)rows * (uint64_t)cols;
  if (total == 0) return 0;
  int threads = 256;
  uint64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  synth_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(a, out, total);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
