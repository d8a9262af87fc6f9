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
__global__ void __launch_bounds__(256) pack_kernel(const uint16_t* __restrict__ W, int K, int N, int mode,
                                                   uint32_t* __restrict__ qweight, uint16_t* __restrict__ scales,
                                                   uint16_t* __restrict__ zeros, int32_t* __restrict__ dev_status) {
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
  scales[(size_t)g * N + n] = __half_as_ushort(s);
  if (zeros) zeros[(size_t)g * N + n] = __half_as_ushort(__float2half_rn(z));

  // 3. codes, written as the 16 words of row (n % 128) of tile (n / 128, g)
  uint32_t* dst = qweight + ((size_t)(n / 128) * groups + g) * 2048 + (size_t)(n % 128) * 16;
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
    *reinterpret_cast<uint4*>(dst + j) = make_uint4(wq[0], wq[1], wq[2], wq[3]);
  }
}

// One thread per (column n, word j of k); writes W_hat[8j + i][n], i = 0..7 (coalesced along n).
// w_hat = (q - z) * s: q - z is exact in fp16, the multiply rounds once (RNE) -> fp16_rne((q - z) * s).
__global__ void __launch_bounds__(256) unpack_kernel(const uint32_t* __restrict__ qweight,
                                                     const uint16_t* __restrict__ scales,
                                                     const uint16_t* __restrict__ zeros, int K, int N, int mode,
                                                     uint16_t* __restrict__ W_hat) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)N * (K / 8)) return;
  const int n = (int)(idx % N), kw = (int)(idx / N);
  const int k0 = kw * 8, g = k0 / W4A16_GROUP;
  const uint32_t word =
      qweight[((size_t)(n / 128) * (K / 128) + g) * 2048 + (size_t)(n % 128) * 16 + (size_t)((k0 % 128) / 8)];
  const __half s = __ushort_as_half(scales[(size_t)g * N + n]);
  const __half z = mode == W4A16_SYM ? __float2half_rn(8.0f) : __ushort_as_half(zeros[(size_t)g * N + n]);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int q = (word >> (4 * ((i % 2) * 4 + i / 2))) & 0xF;
    const __half d = __hmul(__hsub(__int2half_rn(q), z), s);
    W_hat[(size_t)(k0 + i) * N + n] = __half_as_ushort(d);
  }
}

}  // namespace w4

extern "C" int w4a16_launch_pack(const uint16_t* W, int K, int N, int mode, uint32_t* qweight, uint16_t* scales,
                                 uint16_t* zeros, int32_t* dev_status, cudaStream_t stream) {
  const long long threads = (long long)N * (K / W4A16_GROUP);
  if (threads == 0) return W4A16_OK;
  w4::pack_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(W, K, N, mode, qweight, scales, zeros,
                                                                          dev_status);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" int w4a16_launch_unpack(const uint32_t* qweight, const uint16_t* scales, const uint16_t* zeros, int K,
                                   int N, int mode, uint16_t* W_hat, cudaStream_t stream) {
  const long long threads = (long long)N * (K / 8);
  if (threads == 0) return W4A16_OK;
  w4::unpack_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(qweight, scales, zeros, K, N, mode, W_hat);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}
