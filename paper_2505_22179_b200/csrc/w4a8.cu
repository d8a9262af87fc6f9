// w4a8.cu — W4A8 variant (4-bit weights, 8-bit activations on INT8 tensor
// cores, QQQ-style symmetric; reading R21 in DESIGN.md): per-token int8 activation quantisation and the
// W4A8 GEMM on the SYM group-128 blob of w4a16_pack.
//
// GEMM: integer MMA `mma.sync.m16n8k32.row.col.s32.u8.s8.s32` with the weights' raw 4-bit codes q in [0,15]
// as the unsigned A operand (swap-AB: 16 output columns x 32 k) and the int8 activations as B; per k-group
// the exact int32 sum is corrected by -8 * sum(x_q) (precomputed per token and group), scaled by the
// group's fp16 scale into an fp32 accumulator; the token scale and the fp16 rounding come last. First
// correct version: one n-tile x k-range per CTA, code words read straight from global memory.
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tma_host.cuh"
#include "w4a16.h"

namespace w4 {
namespace a8 {

constexpr int kTile = 128;      // n-tile rows = k-group
constexpr int kTB = 8448;       // SYM unit bytes (8192 codes + 128 fp16 scales)
constexpr int kWarps = 8;       // 16 output columns (tile rows) each

// ---- activation quantisation: one CTA per token row ----
// One CTA per token row, kQT threads, one pass over the row: every thread keeps its 8-value chunks (16-byte
// loads) in registers, the row's amax is reduced through shared memory, then each chunk is quantised and a
// 128-k group's sum (16 consecutive chunks = 16 lanes) is reduced with shuffles. The GEMM that follows is
// launched with programmatic dependent launch: this kernel lets it start at once, so its weight stream
// overlaps the quantisation (the GEMM waits for this grid before it reads Xq).
constexpr int kQT = 512;
constexpr int kQChunks = 8;   // 8-value chunks per thread kept in registers: K <= kQT * 8 * kQChunks = 32768
__global__ void __launch_bounds__(kQT) quant_kernel(const __half* __restrict__ X, int K, int8_t* __restrict__ Xq,
                                                    float* __restrict__ sx, int32_t* __restrict__ xsum) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int m = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(X + (size_t)m * K);
  const int nc = K / 8;   // 8-value chunks in the row
  __shared__ float s_red[kQT / 32];
  uint4 v[kQChunks];
  float amax = 0.f;
#pragma unroll
  for (int j = 0; j < kQChunks; ++j) {
    const int c = threadIdx.x + j * kQT;
    v[j] = c < nc ? __ldg(xr + c) : make_uint4(0, 0, 0, 0);
    const __half2* h = reinterpret_cast<const __half2*>(&v[j]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h[e]);
      amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
    }
  }
  for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = s_red[0];
#pragma unroll
  for (int w = 1; w < kQT / 32; ++w) amax = fmaxf(amax, s_red[w]);
  const float inv = amax > 0.f ? __fdiv_rn(127.f, amax) : 0.f;
  if (threadIdx.x == 0) sx[m] = __fdiv_rn(amax, 127.f);
#pragma unroll
  for (int j = 0; j < kQChunks; ++j) {
    const int c = threadIdx.x + j * kQT;   // chunks 16 g .. 16 g + 15 of group g sit on 16 consecutive lanes
    if (j * kQT >= nc) break;
    const __half2* h = reinterpret_cast<const __half2*>(&v[j]);
    int8_t q[8];
    int sum = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h[e]);
      float a = fminf(fmaxf(rintf(__fmul_rn(f.x, inv)), -127.f), 127.f);
      float b = fminf(fmaxf(rintf(__fmul_rn(f.y, inv)), -127.f), 127.f);
      q[2 * e] = (int8_t)(int)a;
      q[2 * e + 1] = (int8_t)(int)b;
      sum += q[2 * e] + q[2 * e + 1];
    }
    if (c < nc) *reinterpret_cast<int2*>(Xq + (size_t)m * K + (size_t)c * 8) = *reinterpret_cast<const int2*>(q);
    for (int o = 8; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);   // 16-lane halves = one group
    if (c < nc && (threadIdx.x & 15) == 0) xsum[(size_t)m * (K / kTile) + c / 16] = sum;
  }
  for (int c0 = kQChunks * kQT; c0 < nc; c0 += kQT) {   // K > 32768: second pass from memory (warp-uniform loop)
    const int c = c0 + threadIdx.x;
    const uint4 w = c < nc ? __ldg(xr + c) : make_uint4(0, 0, 0, 0);
    const __half2* h = reinterpret_cast<const __half2*>(&w);
    int8_t q[8];
    int sum = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h[e]);
      float a = fminf(fmaxf(rintf(__fmul_rn(f.x, inv)), -127.f), 127.f);
      float b = fminf(fmaxf(rintf(__fmul_rn(f.y, inv)), -127.f), 127.f);
      q[2 * e] = (int8_t)(int)a;
      q[2 * e + 1] = (int8_t)(int)b;
      sum += q[2 * e] + q[2 * e + 1];
    }
    if (c < nc) *reinterpret_cast<int2*>(Xq + (size_t)m * K + (size_t)c * 8) = *reinterpret_cast<const int2*>(q);
    for (int o = 8; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (c < nc && (threadIdx.x & 15) == 0) xsum[(size_t)m * (K / kTile) + c / 16] = sum;
  }
}

__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(a), "r"(sel));
  return r;
}
// 8 codes of one 32-bit word (physical nibble slot (i%2)*4 + i/2 holds logical k offset i) -> bytes in
// logical order: lo = k 0..3, hi = k 4..7 (values 0..15).
__device__ __forceinline__ uint32_t codes_lo(uint32_t w) { return prmt((w & 0x000F000Fu) | ((w << 4) & 0x0F000F00u), 0x3120); }
__device__ __forceinline__ uint32_t codes_hi(uint32_t w) {
  return prmt(((w >> 8) & 0x000F000Fu) | ((w >> 4) & 0x0F000F00u), 0x3120);
}

// ---- GEMM: CTA = (n-tile, k-split); warp w owns tile rows 16w..16w+15; NTB token blocks of 8 ----
// A kStages-deep cp.async ring per CTA: each unit's 8 KB of code words (coalesced 16-byte copies by all
// threads) and its M x 128 int8 activation slice (rows padded to 144 B so the 8 token rows of a B
// fragment hit distinct banks); fragments are then read from shared memory.
constexpr int kXRow = 144;
#ifndef W4A8_STAGES
#define W4A8_STAGES 4
#endif
constexpr int kStages = W4A8_STAGES;
#ifndef W4A8_UPS
#define W4A8_UPS 1   // units per CTA barrier (the ring holds kStages units, kStages / W4A8_UPS groups)
#endif
constexpr int kUps = W4A8_UPS;
static_assert(kStages % kUps == 0 && kStages / kUps >= 2, "ring of at least two unit groups");
#ifndef W4A8_MIN_UNITS
#define W4A8_MIN_UNITS 8   // fewest k-groups per split (4: -7 % at M = 64, 16: +25 % at M <= 16)
#endif
template <int NTB>
constexpr int smem_bytes() { return kStages * (kTB + NTB * 8 * kXRow + NTB * 8 * 4); }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NTB>
__global__ void __launch_bounds__(kWarps * 32) gemm_kernel(const int8_t* __restrict__ Xq, const int32_t* __restrict__ xsum,
                                                          const uint8_t* __restrict__ packed, float* __restrict__ part,
                                                          int M, int K, int N, int g_per_split) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* wsm = smem;                                   // [kStages][kTB]: code words + fp16 scales
  uint8_t* xsm = smem + kStages * kTB;                   // [kStages][NTB*8][kXRow]
  int* ssm = reinterpret_cast<int*>(xsm + kStages * NTB * 8 * kXRow);   // [kStages][NTB*8] group sums
  const int t = blockIdx.x, split = blockIdx.y, Gk = K / kTile;
  const int g0 = split * g_per_split, g1 = min(Gk, g0 + g_per_split);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g8 = lane >> 2, c4 = lane & 3;
  const int r0 = warp * 16 + g8, r1 = r0 + 8;   // tile rows of this lane (A rows g / g+8)
  const int sw0 = (r0 >> 1) & 3, sw1 = (r1 >> 1) & 3, wo = (c4 >> 1) * 4;
  // activation rows >= M stay zero
  for (int i = threadIdx.x; i < kStages * NTB * 8 * kXRow / 16; i += kWarps * 32) reinterpret_cast<uint4*>(xsm)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  auto issue = [&](int g) {
    const int st = (g - g0) % kStages;
    const uint8_t* unit = packed + ((size_t)t * Gk + g) * kTB;
    for (int i = threadIdx.x; i < kTB / 16; i += kWarps * 32) cp_async16(wsm + st * kTB + i * 16, unit + i * 16);
    for (int m = threadIdx.x; m < M; m += kWarps * 32) cp_async4(ssm + st * NTB * 8 + m, xsum + (size_t)m * Gk + g);
    for (int i = threadIdx.x; i < M * 8; i += kWarps * 32) {
      const int m = i >> 3, c = i & 7;
      cp_async16(xsm + (st * NTB * 8 + m) * kXRow + c * 16, Xq + (size_t)m * K + g * kTile + c * 16);
    }
  };
  float out[NTB][4];
#pragma unroll
  for (int tb = 0; tb < NTB; ++tb) out[tb][0] = out[tb][1] = out[tb][2] = out[tb][3] = 0.f;
#pragma unroll
  for (int i = 0; i < kStages - kUps; ++i) {
    if (g0 + i < g1) issue(g0 + i);
    if (i % kUps == kUps - 1) cp_commit();
  }
  const uint32_t sh = (c4 & 1) ? 8u : 0u;   // lanes with odd c4 take k 4..7 of each word
  for (int gb = g0; gb < g1; gb += kUps) {
#pragma unroll
    for (int i = 0; i < kUps; ++i)
      if (gb + kStages - kUps + i < g1) issue(gb + kStages - kUps + i);
    cp_commit();
    cp_wait<kStages / kUps - 1>();
    __syncthreads();
#pragma unroll
    for (int ui = 0; ui < kUps; ++ui) {
    const int g = gb + ui;
    if (g >= g1) break;
    const int st = (g - g0) % kStages;
    const uint8_t* wst = wsm + st * kTB;
    const uint8_t* xst = xsm + st * NTB * 8 * kXRow;
    const int* sst = ssm + st * NTB * 8;
    const float s0 = __half2float(reinterpret_cast<const __half*>(wst + 8192)[r0]);
    const float s1 = __half2float(reinterpret_cast<const __half*>(wst + 8192)[r1]);
    int acc[NTB][4];
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb) acc[tb][0] = acc[tb][1] = acc[tb][2] = acc[tb][3] = 0;
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {   // 32 k per MMA
      const uint32_t w0 = *reinterpret_cast<const uint32_t*>(wst + r0 * 64 + ((kb ^ sw0) << 4) + wo);
      const uint32_t w1 = *reinterpret_cast<const uint32_t*>(wst + r0 * 64 + ((kb ^ sw0) << 4) + 8 + wo);
      const uint32_t w2 = *reinterpret_cast<const uint32_t*>(wst + r1 * 64 + ((kb ^ sw1) << 4) + wo);
      const uint32_t w3 = *reinterpret_cast<const uint32_t*>(wst + r1 * 64 + ((kb ^ sw1) << 4) + 8 + wo);
      // k 4..7 of a word are k 0..3 of the word shifted right by 8 (codes_hi(w) == codes_lo(w >> 8))
      const uint32_t a0 = codes_lo(w0 >> sh), a2 = codes_lo(w1 >> sh);
      const uint32_t a1 = codes_lo(w2 >> sh), a3 = codes_lo(w3 >> sh);
#pragma unroll
      for (int tb = 0; tb < NTB; ++tb) {
        const uint8_t* xr = xst + (tb * 8 + g8) * kXRow + kb * 32 + 4 * c4;
        mma_u8s8(acc[tb], a0, a1, a2, a3, *reinterpret_cast<const uint32_t*>(xr), *reinterpret_cast<const uint32_t*>(xr + 16));
      }
    }
    // group epilogue: D[row][col]: d0,d1 = (r0, tokens 2c, 2c+1), d2,d3 = (r1, same tokens)
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb) {
      const int m0 = tb * 8 + 2 * c4, m1 = m0 + 1;
      const int xs0 = m0 < M ? sst[m0] : 0;
      const int xs1 = m1 < M ? sst[m1] : 0;
      out[tb][0] = fmaf(s0, (float)(acc[tb][0] - 8 * xs0), out[tb][0]);
      out[tb][1] = fmaf(s0, (float)(acc[tb][1] - 8 * xs1), out[tb][1]);
      out[tb][2] = fmaf(s1, (float)(acc[tb][2] - 8 * xs0), out[tb][2]);
      out[tb][3] = fmaf(s1, (float)(acc[tb][3] - 8 * xs1), out[tb][3]);
    }
    }
    __syncthreads();   // these stages are refilled by the next iteration's issue
  }
  cp_wait<0>();
  float* P = part + (size_t)split * M * N;
  const int n0 = t * kTile + r0, n1 = t * kTile + r1;
#pragma unroll
  for (int tb = 0; tb < NTB; ++tb) {
    const int m0 = tb * 8 + 2 * c4, m1 = m0 + 1;
    if (m0 < M) { P[(size_t)m0 * N + n0] = out[tb][0]; P[(size_t)m0 * N + n1] = out[tb][2]; }
    if (m1 < M) { P[(size_t)m1 * N + n0] = out[tb][1]; P[(size_t)m1 * N + n1] = out[tb][3]; }
  }
}

// Y[m][n] = fp16_rne(sx[m] * sum over splits in order of part[split][m][n])
__global__ void finish_kernel(const float* __restrict__ part, const float* __restrict__ sx, __half* __restrict__ Y, int M, int N,
                              int splits) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)M * N) return;
  float acc = 0.f;
  for (int s = 0; s < splits; ++s) acc += part[(size_t)s * M * N + i];
  Y[i] = __float2half_rn(sx[i / N] * acc);
}

inline int splits_for(int M, int K, int N, int num_sms) {
  // k-splits that fill the resident CTA slots in whole waves best, each split >= 4 units. Resident CTAs per
  // SM from the kernels' register use (ptxas: ~60 registers up to 32 tokens -> 4 CTAs, ~120 above -> 2)
  const int Gk = K / kTile, tiles = N / kTile, slots = (M <= 32 ? 4 : 2) * num_sms;
  int best = 1;
  double best_eff = 0.0;
  for (int sp = 1; sp <= 16 && sp * W4A8_MIN_UNITS <= Gk; ++sp) {
    const double waves = (double)tiles * sp / slots;
    const double eff = waves / (double)((tiles * sp + slots - 1) / slots);
    if (eff > best_eff + 1e-3) { best_eff = eff; best = sp; }
  }
  return best;
}

}  // namespace a8
}  // namespace w4

extern "C" size_t w4a8_workspace_bytes_sms(int M, int K, int N, int num_sms) {
  return (size_t)w4::a8::splits_for(M, K, N, num_sms) * M * N * 4;
}

extern "C" int w4a8_launch_quantize(const uint16_t* X, int M, int K, int8_t* Xq, float* sx, int32_t* xsum, cudaStream_t stream) {
  w4::a8::quant_kernel<<<M, w4::a8::kQT, 0, stream>>>(reinterpret_cast<const __half*>(X), K, Xq, sx, xsum);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" int w4a8_launch_gemm(const int8_t* Xq, const float* sx, const int32_t* xsum, const void* packed, uint16_t* Y, int M,
                                int K, int N, void* ws, int num_sms, cudaStream_t stream) {
  const int splits = w4::a8::splits_for(M, K, N, num_sms), Gk = K / w4::a8::kTile;
  const int gps = (Gk + splits - 1) / splits;
  const int used = (Gk + gps - 1) / gps;
  float* part = reinterpret_cast<float*>(ws);
  const dim3 grid(N / w4::a8::kTile, used);
  const uint8_t* pk = reinterpret_cast<const uint8_t*>(packed);
  switch ((M + 7) / 8) {
#define W4A8_CASE(T)                                                                                         \
  case T: {                                                                                                  \
    static unsigned long long attr_set = 0;                                                                  \
    if (!w4::ensure_smem_attr(w4::a8::gemm_kernel<T>, w4::a8::smem_bytes<T>(), attr_set)) return W4A16_ERR_CUDA; \
    w4::a8::gemm_kernel<T><<<grid, w4::a8::kWarps * 32, w4::a8::smem_bytes<T>(), stream>>>(Xq, xsum, pk, part, M, K, N, gps); \
    break;                                                                                                   \
  }
    W4A8_CASE(1) W4A8_CASE(2) W4A8_CASE(3) W4A8_CASE(4) W4A8_CASE(5) W4A8_CASE(6) W4A8_CASE(7) W4A8_CASE(8)
#undef W4A8_CASE
    default: return W4A16_ERR_SHAPE;
  }
  const size_t total = (size_t)M * N;
  w4::a8::finish_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(part, sx, reinterpret_cast<__half*>(Y), M, N, used);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}
