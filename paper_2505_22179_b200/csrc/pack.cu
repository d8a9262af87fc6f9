// pack.cu — w4a16_pack / w4a16_unpack kernels.
//
// Quantisation follows the GPTQ quantizer conventions (RTN per S:95) exactly as include/w4a16.h
// states them, in IEEE fp32 with explicit round-to-nearest intrinsics (no FMA contraction: this file is
// compiled with --fmad=false), so codes, scales and zeros are bit-identical to the CPU oracle.
#include "common.cuh"
#include "w4a16.h"

namespace w4 {

__device__ __forceinline__ float clamp_lo_hi(float x, float lo, float hi) {
  // !(x > lo) maps -0.0 and NaN to lo, so a zero point is never stored as fp16 -0.
  if (!(x > lo)) return lo;
  if (x > hi) return hi;
  return x;
}

// One thread per (column n, group g); lanes of a warp take consecutive n, so every W read is coalesced.
__host__ __device__ __forceinline__ size_t tile_bytes(int mode) { return mode == W4A16_ASYM ? 8704 : 8448; }

__global__ void __launch_bounds__(256) pack_kernel(const uint16_t* __restrict__ W, int K, int N, int mode,
                                                   uint8_t* __restrict__ packed, int32_t* __restrict__ dev_status) {
  const int groups = K / W4A16_GROUP;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)N * groups) return;
  const int n = (int)(idx % N), g = (int)(idx / N);
  const uint16_t* col = W + (size_t)g * W4A16_GROUP * N + n;

  // 1. range containing 0 (GPTQ: xmin = min(x, 0), xmax = max(x, 0)); non-finite weights count as 0.
  float wmin = 0.0f, wmax = 0.0f;
  bool nonfinite = false;
  for (int k = 0; k < W4A16_GROUP; ++k) {
    float w = __half2float(__ushort_as_half(col[(size_t)k * N]));
    if (!isfinite(w)) { nonfinite = true; continue; }
    if (w < wmin) wmin = w;
    if (w > wmax) wmax = w;
  }
  if (nonfinite && dev_status) atomicExch(dev_status, W4A16_DEV_NONFINITE);

  // 2. scale (fp16, RNE) and integer zero point
  float s32, z;
  __half s;
  if (mode == W4A16_ASYM) {
    if (wmin == wmax) { wmin = -1.0f; wmax = 1.0f; }
    s = __float2half_rn(__fdiv_rn(__fsub_rn(wmax, wmin), 15.0f));
    if (__half2float(s) == 0.0f) { wmin = -1.0f; wmax = 1.0f; s = __float2half_rn(__fdiv_rn(__fsub_rn(wmax, wmin), 15.0f)); }
    s32 = __half2float(s);
    z = clamp_lo_hi(rintf(__fdiv_rn(-wmin, s32)), 0.0f, 15.0f);
  } else {
    float amax = -wmin > wmax ? -wmin : wmax;
    if (amax == 0.0f) amax = 1.0f;
    s = __float2half_rn(__fdiv_rn(__fadd_rn(amax, amax), 15.0f));
    if (__half2float(s) == 0.0f) { amax = 1.0f; s = __float2half_rn(__fdiv_rn(__fadd_rn(amax, amax), 15.0f)); }
    s32 = __half2float(s);
    z = 8.0f;
  }
  uint8_t* tile = packed + ((size_t)(n / 128) * groups + g) * tile_bytes(mode);
  const int r = n % 128;
  if (mode == W4A16_ASYM) {
    reinterpret_cast<uint32_t*>(tile + 8192)[r] =
        (uint32_t)__half_as_ushort(s) | ((uint32_t)__half_as_ushort(__float2half_rn(z)) << 16);   // {s, z}
  } else {
    reinterpret_cast<uint16_t*>(tile + 8192)[r] = __half_as_ushort(s);
  }

  // 3. codes: chunk p (words 4p..4p+3 = k 32p..32p+31) of row r goes to chunk position p ^ ((r/2) % 4)
  uint32_t* dst = reinterpret_cast<uint32_t*>(tile) + (size_t)r * 16;
  for (int j = 0; j < 16; j += 4) {
    uint32_t wq[4];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      uint32_t word = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float w = __half2float(__ushort_as_half(col[(size_t)(8 * (j + jj) + i) * N]));
        if (!isfinite(w)) w = 0.0f;
        float q = clamp_lo_hi(__fadd_rn(rintf(__fdiv_rn(w, s32)), z), 0.0f, 15.0f);
        word |= (uint32_t)(int)q << (4 * ((i % 2) * 4 + i / 2));
      }
      wq[jj] = word;
    }
    *reinterpret_cast<uint4*>(dst + 4 * ((j / 4) ^ ((r >> 1) & 3))) = make_uint4(wq[0], wq[1], wq[2], wq[3]);
  }
}

// One thread per (column n, word j of k); writes W_hat[8j + i][n], i = 0..7 (coalesced along n).
// w_hat = (q - z) * s: q - z is exact in fp16, the multiply rounds once (RNE) -> fp16_rne((q - z) * s).
__global__ void __launch_bounds__(256) unpack_kernel(const uint8_t* __restrict__ packed, int K, int N, int mode,
                                                     uint16_t* __restrict__ W_hat) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)N * (K / 8)) return;
  const int n = (int)(idx % N), kw = (int)(idx / N);
  const int k0 = kw * 8, g = k0 / W4A16_GROUP, r = n % 128;
  const uint8_t* tile = packed + ((size_t)(n / 128) * (K / 128) + g) * tile_bytes(mode);
  const int p = (k0 % 128) / 32, w = (k0 % 32) / 8;
  const uint32_t word = reinterpret_cast<const uint32_t*>(tile)[(size_t)r * 16 + 4 * (p ^ ((r >> 1) & 3)) + w];
  const bool asym = mode == W4A16_ASYM;
  const __half s = __ushort_as_half(reinterpret_cast<const uint16_t*>(tile + 8192)[asym ? 2 * r : r]);
  const __half z = asym ? __ushort_as_half(reinterpret_cast<const uint16_t*>(tile + 8192)[2 * r + 1])
                        : __float2half_rn(8.0f);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int q = (word >> (4 * ((i % 2) * 4 + i / 2))) & 0xF;
    const __half d = __hmul(__hsub(__int2half_rn(q), z), s);
    W_hat[(size_t)(k0 + i) * N + n] = __half_as_ushort(d);
  }
}

}  // namespace w4

extern "C" int w4a16_launch_pack(const uint16_t* W, int K, int N, int mode, void* packed, int32_t* dev_status,
                                 cudaStream_t stream) {
  const long long threads = (long long)N * (K / W4A16_GROUP);
  if (threads == 0) return W4A16_OK;
  w4::pack_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(W, K, N, mode,
                                                                          reinterpret_cast<uint8_t*>(packed), dev_status);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" int w4a16_launch_unpack(const void* packed, int K, int N, int mode, uint16_t* W_hat, cudaStream_t stream) {
  const long long threads = (long long)N * (K / 8);
  if (threads == 0) return W4A16_OK;
  w4::unpack_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(reinterpret_cast<const uint8_t*>(packed), K,
                                                                            N, mode, W_hat);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}
