// hadamard.cu — w4a16_hadamard: the online activation rotation of W4A16+Rot.
//
// The paper also evaluates W4A16 with Hadamard rotation (QuaRot-style): the weights are rotated
// offline (W' = H W, then quantised), and the activations are rotated online, x' = x H, so x W = x' W'.
// With the block-diagonal normalised Sylvester Hadamard H_B along k: y[bB + i] = sum_j (-1)^popcount(i&j)
// x[bB + j] / sqrt(B). One warp per (row, block): the B values sit in registers (B/32 per lane, consecutive),
// the fast Walsh-Hadamard butterflies with stride < B/32 run inside a lane and the others through warp
// shuffles (partner lane = lane ^ (stride / (B/32))); fp32 arithmetic, one RNE to fp16. HBM-bound
// (2 bytes in, 2 bytes out per element).
#include "common.cuh"
#include "w4a16.h"

namespace w4 {
namespace hd {

template <int B>
__global__ void __launch_bounds__(256) hadamard_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y, int M,
                                                       int K) {
  constexpr int V = B / 32;   // values per lane (consecutive k)
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);   // (row, block) index
  const int nb = K / B;
  if (w >= (long long)M * nb) return;
  const int m = (int)(w / nb), b = (int)(w % nb);
  const uint16_t* src = X + (size_t)m * K + (size_t)b * B + lane * V;
  float v[V];
#pragma unroll
  for (int i = 0; i < V; i += 2) {
    const __half2 h = *reinterpret_cast<const __half2*>(src + i);
    const float2 f = __half22float2(h);
    v[i] = f.x;
    v[i + 1] = f.y;
  }
  // strides inside a lane
#pragma unroll
  for (int h = 1; h < V; h <<= 1)
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (!(i & h)) {
        const float a = v[i], c = v[i + h];
        v[i] = a + c;
        v[i + h] = a - c;
      }
  // strides across lanes: element (lane, i) pairs with (lane ^ (h / V), i); the lower lane keeps a + c
#pragma unroll
  for (int hl = 1; hl < 32; hl <<= 1) {
    const bool upper = lane & hl;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float o = __shfl_xor_sync(0xffffffffu, v[i], hl);
      v[i] = upper ? o - v[i] : v[i] + o;
    }
  }
  const float norm = rsqrtf((float)B);
  uint16_t* dst = Y + (size_t)m * K + (size_t)b * B + lane * V;
#pragma unroll
  for (int i = 0; i < V; i += 2)
    *reinterpret_cast<__half2*>(dst + i) = __floats2half2_rn(v[i] * norm, v[i + 1] * norm);
}

}  // namespace hd
}  // namespace w4

extern "C" int w4a16_launch_hadamard(const uint16_t* X, uint16_t* Y, int M, int K, int B, cudaStream_t stream) {
  const long long warps = (long long)M * (K / B);
  const unsigned blocks = (unsigned)((warps + 7) / 8);
  switch (B) {
    case 64: w4::hd::hadamard_kernel<64><<<blocks, 256, 0, stream>>>(X, Y, M, K); break;
    case 128: w4::hd::hadamard_kernel<128><<<blocks, 256, 0, stream>>>(X, Y, M, K); break;
    case 256: w4::hd::hadamard_kernel<256><<<blocks, 256, 0, stream>>>(X, Y, M, K); break;
    case 512: w4::hd::hadamard_kernel<512><<<blocks, 256, 0, stream>>>(X, Y, M, K); break;
    case 1024: w4::hd::hadamard_kernel<1024><<<blocks, 256, 0, stream>>>(X, Y, M, K); break;
    default: return W4A16_ERR_SHAPE;
  }
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}
