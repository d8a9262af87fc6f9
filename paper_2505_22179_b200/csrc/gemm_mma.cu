// gemm_mma.cu — W4A16 verify GEMM, kernel family A ("decode width", M <= 16): SURVEY §8(a) a2-a6.
//
//   Y[M,N] = X[M,K] · W_hat[K,N]   with W_hat = (q - z) * s per group of 128 k (include/w4a16.h)
//
// Design:
//  * Work unit = one 128x128 (n x k) weight tile = 8 KiB of codes + 256 B scales + 256 B zeros. Units are
//    numbered u = tile_n * (K/128) + group, which is exactly their order in qweight, so a CTA's range of
//    units is one contiguous byte range of the packed weights.
//  * Stream-K: CTA c of G owns units [c*U/G, (c+1)*U/G). A (K, N, SM-count)-only plan: no dependence on M.
//  * Warp 8 = producer: one lane streams each unit into a STAGES-deep shared-memory ring with 1-D bulk
//    async copies (TMA engine, mbarrier completion, L2 evict_first for the once-read weights).
//  * Warps 0..7 = consumers: warp w owns rows 16w..16w+15 of the 128-row tile. Per unit a lane reads its
//    two 16-byte chunks (rows g and g+8, k-chunk c), dequantises with LOP3 + HSUB2/HFMA2 to EXACT small
//    integers (q - z) in fp16, and issues mma.sync m16n8k16 with weights as the MMA-M operand ("swap AB";
//    tokens are MMA-N, padded to 8). A k-permutation inside each 32-wide chunk lets one lane's 32
//    consecutive k feed 8 MMAs, so both weights and activations are read as 16-byte vectors.
//  * The group scale is applied after the MMA, to the fp32 group sum: Y += s * sum_k X (q - z). This keeps
//    the dequant at 9 integer/fp16 instructions per 8 weights (no HMUL2), the budget that decides whether
//    B200's ALU can keep up with 7 TB/s of int4 weights.
//  * Split tiles: fp32 partials to the workspace, then the last CTA to arrive (atomic counter per tile)
//    sums the partials in CTA order (fixed, hence deterministic) and writes fp16 Y; it re-zeroes the
//    counter, leaving the workspace ready for the next call.
#include "common.cuh"
#include "w4a16.h"

namespace w4 {

constexpr int kTileN = 128, kTileK = 128;
constexpr int kUnitWBytes = kTileN * kTileK / 2;             // 8192
constexpr int kStageBytes = kUnitWBytes + 2 * kTileN * 2;    // + scales + zeros = 8704
constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;          // 288

struct GemmParams {
  const uint16_t* X;
  const uint32_t* qweight;
  const uint16_t* scales;
  const uint16_t* zeros;
  uint16_t* Y;
  float* partials;   // [2G][NTB][8 warps][32 lanes] float4
  int* counters;     // [N/128]
  int M, K, N;
  int Gk;            // K / 128 groups per n-tile
  int U;             // total units
  int G;             // CTAs
};

__device__ __forceinline__ int unit_begin(int c, int U, int G) { return (int)(((long long)c * U) / G); }
// CTA owning unit u: largest c with unit_begin(c) <= u.
__device__ __forceinline__ int cta_of_unit(int u, int U, int G) {
  return (int)((((long long)(u + 1) * G) + U - 1) / U) - 1;
}

template <int NTB, bool SYM, int STAGES>
__global__ void __launch_bounds__(kThreads, (NTB <= 2 ? 2 : 1)) gemm_w4a16_mma_kernel(const GemmParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int u_begin = unit_begin(cta, p.U, p.G), u_end = unit_begin(cta + 1, p.U, p.G);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], kConsumerWarps); }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer: stream units into the ring ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int u = u_begin; u < u_end; ++u) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        const int t = u / p.Gk, g = u - t * p.Gk;
        uint8_t* st = smem + s * kStageBytes;
        mbar_expect_tx(&full_bar[s], SYM ? kUnitWBytes + 256 : kUnitWBytes + 512);
        bulk_g2s(st, p.qweight + (size_t)u * (kUnitWBytes / 4), kUnitWBytes, &full_bar[s], pol);
        bulk_g2s(st + kUnitWBytes, p.scales + (size_t)g * p.N + (size_t)t * kTileN, 256, &full_bar[s], pol);
        if (!SYM) bulk_g2s(st + kUnitWBytes + 256, p.zeros + (size_t)g * p.N + (size_t)t * kTileN, 256, &full_bar[s], pol);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int g8 = lane >> 2, c4 = lane & 3;   // mma fragment coordinates
  const int r0 = warp * 16 + g8, r1 = r0 + 8; // tile rows (n) owned by this lane
  const uint32_t smem_base = smem_u32(smem);

  float acc[NTB][4];
  int s = 0;
  uint32_t ph = 0;
  int cur_t = -1, seg_first_unit = u_begin;
  bool first_segment = true;

  auto flush = [&](int t, int seg_u0, int seg_u1, bool is_first_seg) {
    const int tile_u0 = t * p.Gk, tile_u1 = tile_u0 + p.Gk;
    const bool whole = (seg_u0 == tile_u0 && seg_u1 == tile_u1);
    const int n0 = t * kTileN + r0, n1 = t * kTileN + r1;
    if (whole) {
#pragma unroll
      for (int tb = 0; tb < NTB; ++tb) {
        const int m0 = tb * 8 + 2 * c4, m1 = m0 + 1;
        if (m0 < p.M) {
          p.Y[(size_t)m0 * p.N + n0] = __half_as_ushort(__float2half_rn(acc[tb][0]));
          p.Y[(size_t)m0 * p.N + n1] = __half_as_ushort(__float2half_rn(acc[tb][2]));
        }
        if (m1 < p.M) {
          p.Y[(size_t)m1 * p.N + n0] = __half_as_ushort(__float2half_rn(acc[tb][1]));
          p.Y[(size_t)m1 * p.N + n1] = __half_as_ushort(__float2half_rn(acc[tb][3]));
        }
      }
      return;
    }
    // split tile: publish the fp32 partial, the last contributor reduces in CTA order.
    const int slot = 2 * cta + (is_first_seg ? 0 : 1);
    float4* part = reinterpret_cast<float4*>(p.partials);
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb)
      __stcg(&part[(((size_t)slot * NTB + tb) * kConsumerWarps + warp) * 32 + lane],
             make_float4(acc[tb][0], acc[tb][1], acc[tb][2], acc[tb][3]));
    __threadfence();
    named_bar_sync(1, kConsumerWarps * 32);
    const int c_first = cta_of_unit(tile_u0, p.U, p.G), c_last = cta_of_unit(tile_u1 - 1, p.U, p.G);
    if (threadIdx.x == 0) s_last = (atomicAdd(&p.counters[t], 1) == c_last - c_first);
    named_bar_sync(1, kConsumerWarps * 32);
    if (!s_last) return;
    __threadfence();
    float sum[NTB][4];
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb) sum[tb][0] = sum[tb][1] = sum[tb][2] = sum[tb][3] = 0.f;
    for (int c = c_first; c <= c_last; ++c) {
      const int sl = 2 * c + (unit_begin(c, p.U, p.G) >= tile_u0 ? 0 : 1);
#pragma unroll
      for (int tb = 0; tb < NTB; ++tb) {
        const float4 v = __ldcg(&part[(((size_t)sl * NTB + tb) * kConsumerWarps + warp) * 32 + lane]);
        sum[tb][0] += v.x; sum[tb][1] += v.y; sum[tb][2] += v.z; sum[tb][3] += v.w;
      }
    }
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb) {
      const int m0 = tb * 8 + 2 * c4, m1 = m0 + 1;
      if (m0 < p.M) {
        p.Y[(size_t)m0 * p.N + n0] = __half_as_ushort(__float2half_rn(sum[tb][0]));
        p.Y[(size_t)m0 * p.N + n1] = __half_as_ushort(__float2half_rn(sum[tb][2]));
      }
      if (m1 < p.M) {
        p.Y[(size_t)m1 * p.N + n0] = __half_as_ushort(__float2half_rn(sum[tb][1]));
        p.Y[(size_t)m1 * p.N + n1] = __half_as_ushort(__float2half_rn(sum[tb][3]));
      }
    }
    if (threadIdx.x == 0) p.counters[t] = 0;   // all contributors have arrived: safe to re-arm
  };

  for (int u = u_begin; u < u_end; ++u) {
    const int t = u / p.Gk, g = u - t * p.Gk;
    if (t != cur_t) {
      if (cur_t >= 0) { flush(cur_t, seg_first_unit, u, first_segment); first_segment = false; }
      cur_t = t;
      seg_first_unit = u;
#pragma unroll
      for (int tb = 0; tb < NTB; ++tb) acc[tb][0] = acc[tb][1] = acc[tb][2] = acc[tb][3] = 0.f;
    }
    // Activations for this unit: lane needs X[m][128g + 32c4 .. +31] for m = 8tb + g8 (L1/L2 resident).
    uint4 xr[NTB][4];
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb) {
      const int m = tb * 8 + g8;
      if (m < p.M) {
        const uint16_t* xp = p.X + (size_t)m * p.K + (size_t)g * kTileK + c4 * 32;
#pragma unroll
        for (int j = 0; j < 4; ++j) xr[tb][j] = ldg128_nc(xp + 8 * j);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) xr[tb][j] = make_uint4(0, 0, 0, 0);
      }
    }
    // Weights for this unit from shared memory.
    mbar_wait(&full_bar[s], ph);
    const uint32_t st = smem_base + s * kStageBytes;
    const uint4 wa = lds128(st + r0 * 64 + c4 * 16);
    const uint4 wb = lds128(st + r1 * 64 + c4 * 16);
    const uint16_t* ssc = reinterpret_cast<const uint16_t*>(smem + s * kStageBytes + kUnitWBytes);
    const float sa = __half2float(__ushort_as_half(ssc[r0])), sb = __half2float(__ushort_as_half(ssc[r1]));
    uint32_t za_lo, zb_lo, za_hi, zb_hi;  // {1024+z} for HSUB2 and {-(64+z)} for HFMA2, per row
    if (SYM) {
      za_lo = zb_lo = 0x64086408u;        // 1032
      za_hi = zb_hi = 0xD480D480u;        // -72
    } else {
      const uint16_t* szr = ssc + kTileN;
      const __half za = __ushort_as_half(szr[r0]), zb = __ushort_as_half(szr[r1]);
      za_lo = h2_bcast(__half_as_ushort(__hadd(za, __float2half_rn(1024.f))));
      zb_lo = h2_bcast(__half_as_ushort(__hadd(zb, __float2half_rn(1024.f))));
      za_hi = h2_bcast(__half_as_ushort(__hneg(__hadd(za, __float2half_rn(64.f)))));
      zb_hi = h2_bcast(__half_as_ushort(__hneg(__hadd(zb, __float2half_rn(64.f)))));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
    if (++s == STAGES) { s = 0; ph ^= 1; }

    float gacc[NTB][4];
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb) gacc[tb][0] = gacc[tb][1] = gacc[tb][2] = gacc[tb][3] = 0.f;
    const uint32_t inv16 = 0x2C002C00u;   // 1/16
    const uint32_t wav[4] = {wa.x, wa.y, wa.z, wa.w}, wbv[4] = {wb.x, wb.y, wb.z, wb.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {          // word j: k = 32c4 + 8j .. +7 (two MMA k-steps)
#pragma unroll
      for (int h = 0; h < 2; ++h) {        // h = 0: k pairs (0,1),(2,3); h = 1: (4,5),(6,7)
        const uint32_t qa = h ? wav[j] >> 8 : wav[j], qb = h ? wbv[j] >> 8 : wbv[j];
        const uint32_t a0 = hsub2_u32(lop3_mask_or(qa, 0x000F000Fu), za_lo);
        const uint32_t a1 = hsub2_u32(lop3_mask_or(qb, 0x000F000Fu), zb_lo);
        const uint32_t a2 = hfma2_u32(lop3_mask_or(qa, 0x00F000F0u), inv16, za_hi);
        const uint32_t a3 = hfma2_u32(lop3_mask_or(qb, 0x00F000F0u), inv16, zb_hi);
        // MMA k-step (j, h) uses physical k = 32c4 + 8j + 4h + {0..3}: logical {2c,2c+1} <- {0,1},
        // {2c+8,2c+9} <- {2,3}; activations use the same permutation.
#pragma unroll
        for (int tb = 0; tb < NTB; ++tb) {
          const uint32_t* xv = reinterpret_cast<const uint32_t*>(&xr[tb][j]);
          mma_16816(gacc[tb], a0, a1, a2, a3, xv[2 * h], xv[2 * h + 1]);
        }
      }
    }
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb) {
      acc[tb][0] = fmaf(sa, gacc[tb][0], acc[tb][0]);
      acc[tb][1] = fmaf(sa, gacc[tb][1], acc[tb][1]);
      acc[tb][2] = fmaf(sb, gacc[tb][2], acc[tb][2]);
      acc[tb][3] = fmaf(sb, gacc[tb][3], acc[tb][3]);
    }
  }
  if (cur_t >= 0) flush(cur_t, seg_first_unit, u_end, first_segment);
}

template <int NTB, bool SYM>
static int launch_t(const GemmParams& p, int stages_unused, cudaStream_t stream) {
  (void)stages_unused;
  constexpr int STAGES = 10;
  auto kern = gemm_w4a16_mma_kernel<NTB, SYM, STAGES>;
  const int smem = STAGES * kStageBytes;
  static bool attr_set = false;   // benign race: idempotent attribute
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return W4A16_ERR_CUDA;
    attr_set = true;
  }
  kern<<<p.G, kThreads, smem, stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

}  // namespace w4

// Plan (depends on K, N and the SM count only).
extern "C" int w4a16_mma_plan_ctas(int K, int N, int num_sms) {
  const long long U = (long long)(N / w4::kTileN) * (K / w4::kTileK);
  long long G = 2LL * num_sms;
  if (G > U) G = U;
  return (int)G;
}

extern "C" size_t w4a16_mma_workspace_bytes(int M, int K, int N, int num_sms) {
  const int ntb = (M + 7) / 8;
  const int G = w4a16_mma_plan_ctas(K, N, num_sms);
  const size_t counters = (((size_t)(N / w4::kTileN) * 4) + 255) / 256 * 256;
  return counters + (size_t)2 * G * ntb * w4::kConsumerWarps * 32 * 16;
}

extern "C" int w4a16_launch_gemm_mma(const uint16_t* X, const uint32_t* qweight, const uint16_t* scales,
                                     const uint16_t* zeros, uint16_t* Y, int M, int K, int N, int mode, void* ws,
                                     int num_sms, cudaStream_t stream) {
  w4::GemmParams p;
  p.X = X; p.qweight = qweight; p.scales = scales; p.zeros = zeros; p.Y = Y;
  p.M = M; p.K = K; p.N = N;
  p.Gk = K / w4::kTileK;
  p.U = (N / w4::kTileN) * p.Gk;
  p.G = w4a16_mma_plan_ctas(K, N, num_sms);
  const size_t counters = (((size_t)(N / w4::kTileN) * 4) + 255) / 256 * 256;
  p.counters = reinterpret_cast<int*>(ws);
  p.partials = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + counters);
  const int ntb = (M + 7) / 8;
  const bool sym = mode == W4A16_SYM;
#define W4_CASE(T)                                                              \
  case T:                                                                       \
    return sym ? w4::launch_t<T, true>(p, 0, stream) : w4::launch_t<T, false>(p, 0, stream);
  switch (ntb) {
    W4_CASE(1) W4_CASE(2) W4_CASE(3) W4_CASE(4) W4_CASE(5) W4_CASE(6) W4_CASE(7) W4_CASE(8)
    default: return W4A16_ERR_SHAPE;
  }
#undef W4_CASE
}
