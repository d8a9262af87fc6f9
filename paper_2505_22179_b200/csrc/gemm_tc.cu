// gemm_tc.cu — W4A16 verify GEMM, kernel family B: 5th-gen tensor cores (tcgen05 + TMEM), M = 1..64.
//
//   Y[M,N] = X[M,K] · W_hat[K,N],  W_hat = fp16_rne((q - z) * s)  (include/w4a16.h)
//
// Why this shape: on B200 the int4->fp16 conversion, not the MMA, competes with HBM for
// time. tcgen05 takes the MMA off the issue slots entirely (one thread issues it) and its cost is nearly
// independent of M <= 64, so the verify GEMM at M = 64 costs about what it costs at M = 1.
//
//  * Same unit / stream-K plan as family A: unit u = 128x128 (n x k) weight tile, CTA c owns units
//    [c*U/G, (c+1)*U/G) with G = #SMs (one persistent CTA per SM); the plan depends on (K, N, SMs) only.
//  * warp 0 (producer): per unit, 1-D bulk copies of the 8 KiB code tile + scales + zeros, and a 2-D TMA
//    (SWIZZLE_128B) of the activation slice X[0:Mpad, 128u_k : 128u_k+128] (rows >= M zero-filled by TMA),
//    into a STAGES-deep shared-memory ring (mbarrier complete_tx).
//  * warps 4..11 (dequant + epilogue): warp w owns TMEM lanes / tile rows 32(w%4)..+31 and k-half
//    (w-4)/4 of the unit. Each thread dequantises 8 words (64 k of one row) with LOP3 + HSUB2/HFMA2 (exact
//    q - z) + HMUL2 (one RNE: exactly the oracle's w_hat), and stores them with one tcgen05.st.32x32b.x32
//    into an A buffer in TMEM (lane = row n, 32-bit column = k pair) — 4 A buffers rotate.
//  * warp 1 (MMA): one thread issues 8 tcgen05.mma.kind::f16 (M=128 rows, N=Mpad tokens, K=16) per unit,
//    A from TMEM, B = X from shared memory (UMMA descriptor, K-major SW128), D = fp32 accumulator in TMEM;
//    tcgen05.commit releases the smem stage and the A buffer, and at a tile boundary signals the epilogue.
//  * epilogue: tcgen05.ld of the accumulator (thread = row), fp16 store of Y, or — for a tile split
//    across CTAs — fp32 partial to the workspace and the ordered last-arriver reduction of family A.
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "w4a16.h"

namespace w4 {
namespace tc {

constexpr int kTileN = 128, kTileK = 128;
constexpr int kUnitWBytes = kTileN * kTileK / 2;  // 8192
constexpr int kNumA = 4;                          // A buffers in TMEM (64 columns each)
constexpr int kDqWarps = 8;
constexpr int kThreads = (4 + kDqWarps) * 32;     // 384: producer, mma, 2 spare, 8 dequant/epilogue
constexpr int kAccCol = kNumA * 64;               // accumulator columns start here
constexpr int kTmemCols = 512;

template <int MPAD>
struct Cfg {
  static constexpr int kXBox = MPAD * 128;                                 // bytes of one 64-k SW128 box
  static constexpr int kXBytes = 2 * kXBox;
  static constexpr int kStage = ((kXBytes + kUnitWBytes + 512) + 1023) / 1024 * 1024;
  static constexpr int kStages = (200 * 1024) / kStage > 12 ? 12 : (200 * 1024) / kStage;
  static constexpr int kSmem = kStages * kStage + 1024;                    // + alignment slack
  static constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(MPAD >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
};

struct Params {
  const uint32_t* qweight;
  const uint16_t* scales;
  const uint16_t* zeros;
  uint16_t* Y;
  float* partials;   // [2G][MPAD][128] fp32
  int* counters;     // [N/128]
  int M, K, N, Gk, U, G;
};

__device__ __forceinline__ int unit_begin(int c, int U, int G) { return (int)(((long long)c * U) / G); }
__device__ __forceinline__ int cta_of_unit(int u, int U, int G) {
  return (int)((((long long)(u + 1) * G) + U - 1) / U) - 1;
}

// ---- tcgen05 / TMA wrappers (PTX ISA 8.7, sm_100a) ----
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, int ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, int ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld_x8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: SBO = 1024 B (8 rows x 128 B), LBO unused (1),
// version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}

template <int MPAD, bool SYM>
__global__ void __launch_bounds__(kThreads, 1) gemm_w4a16_tc_kernel(const __grid_constant__ CUtensorMap xmap,
                                                                     const Params p) {
  using C = Cfg<MPAD>;
  constexpr int S = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[S], empty_bar[S];
  __shared__ __align__(8) uint64_t afull_bar[kNumA], aempty_bar[kNumA];
  __shared__ __align__(8) uint64_t accfull_bar, accempty_bar;
  __shared__ uint32_t s_tmem;
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int u_begin = unit_begin(cta, p.U, p.G), u_end = unit_begin(cta + 1, p.U, p.G);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int b = 0; b < kNumA; ++b) { mbar_init(&afull_bar[b], kDqWarps); mbar_init(&aempty_bar[b], 1); }
    mbar_init(&accfull_bar, 1);
    mbar_init(&accempty_bar, kDqWarps);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&s_tmem, kTmemCols);
  if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int u = u_begin; u < u_end; ++u) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        const int t = u / p.Gk, g = u - t * p.Gk;
        uint8_t* st = smem + s * C::kStage;
        mbar_expect_tx(&full_bar[s], C::kXBytes + kUnitWBytes + (SYM ? 256 : 512));
        tma_2d(st, &xmap, g * kTileK, 0, &full_bar[s]);
        tma_2d(st + C::kXBox, &xmap, g * kTileK + 64, 0, &full_bar[s]);
        bulk_g2s(st + C::kXBytes, p.qweight + (size_t)u * (kUnitWBytes / 4), kUnitWBytes, &full_bar[s], pol);
        bulk_g2s(st + C::kXBytes + kUnitWBytes, p.scales + (size_t)g * p.N + (size_t)t * kTileN, 256, &full_bar[s], pol);
        if (!SYM)
          bulk_g2s(st + C::kXBytes + kUnitWBytes + 256, p.zeros + (size_t)g * p.N + (size_t)t * kTileN, 256, &full_bar[s], pol);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int s = 0, b = 0;
      uint32_t ph = 0, aph = 0, accph = 0;
      int cur_t = -1;
      bool first_seg = true;
      const uint32_t d_tmem = tmem + kAccCol;
      for (int u = u_begin; u < u_end; ++u) {
        const int t = u / p.Gk;
        const bool seg_start = (t != cur_t);
        if (seg_start) {
          if (!first_seg) { mbar_wait(&accempty_bar, accph); accph ^= 1; }   // epilogue drained the accumulator
          first_seg = false;
          cur_t = t;
        }
        const bool seg_end = (u + 1 == u_end) || ((u + 1) / p.Gk != t);
        mbar_wait(&full_bar[s], ph);
        mbar_wait(&afull_bar[b], aph);
        tc_fence_after();
        const uint32_t xs = smem_u32(smem + s * C::kStage);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t bdesc = desc_sw128(xs + (ks >> 2) * C::kXBox + (ks & 3) * 32);
          mma_ts(d_tmem, tmem + b * 64 + ks * 8, bdesc, C::kIdesc, (seg_start && ks == 0) ? 0u : 1u);
        }
        tc_commit(&empty_bar[s]);
        tc_commit(&aempty_bar[b]);
        if (seg_end) tc_commit(&accfull_bar);
        if (++s == S) { s = 0; ph ^= 1; }
        if (++b == kNumA) { b = 0; aph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- dequant + epilogue ----------------
    const int q = warp & 3;           // TMEM lane quarter = tile rows 32q..32q+31
    const int h = (warp - 4) >> 2;    // k-half of the unit: k 64h .. 64h+63
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    int s = 0, b = 0;
    uint32_t ph = 0, aph = 0, accph = 0;
    int cur_t = -1, seg_u0 = u_begin;
    bool first_seg_flag = true;

    auto epilogue = [&](int t, int sg0, int sg1, bool is_first_seg) {
      mbar_wait(&accfull_bar, accph);
      accph ^= 1;
      tc_fence_after();
      constexpr int kCols = MPAD / 2;  // this warp's token columns: [h*kCols, (h+1)*kCols)
      float acc[kCols];
#pragma unroll
      for (int c = 0; c < kCols; c += 8) {
        float v[8];
        tmem_ld_x8(tmem + lane_base + kAccCol + h * kCols + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[c + i] = v[i];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty_bar);
      const int tile_u0 = t * p.Gk, tile_u1 = tile_u0 + p.Gk;
      const int n = t * kTileN + row;
      const int m0 = h * kCols;
      if (sg0 == tile_u0 && sg1 == tile_u1) {
#pragma unroll
        for (int i = 0; i < kCols; ++i)
          if (m0 + i < p.M) p.Y[(size_t)(m0 + i) * p.N + n] = __half_as_ushort(__float2half_rn(acc[i]));
        return;
      }
      const int slot = 2 * blockIdx.x + (is_first_seg ? 0 : 1);
#pragma unroll
      for (int i = 0; i < kCols; ++i) __stcg(&p.partials[((size_t)slot * MPAD + m0 + i) * kTileN + row], acc[i]);
      __threadfence();
      named_bar_sync(1, kDqWarps * 32);
      const int c_first = cta_of_unit(tile_u0, p.U, p.G), c_last = cta_of_unit(tile_u1 - 1, p.U, p.G);
      if (threadIdx.x == 4 * 32) s_last = (atomicAdd(&p.counters[t], 1) == c_last - c_first);
      named_bar_sync(1, kDqWarps * 32);
      if (!s_last) return;
      __threadfence();
#pragma unroll
      for (int i = 0; i < kCols; ++i) acc[i] = 0.f;
      for (int c = c_first; c <= c_last; ++c) {
        const int sl = 2 * c + (unit_begin(c, p.U, p.G) >= tile_u0 ? 0 : 1);
#pragma unroll
        for (int i = 0; i < kCols; ++i) acc[i] += __ldcg(&p.partials[((size_t)sl * MPAD + m0 + i) * kTileN + row]);
      }
#pragma unroll
      for (int i = 0; i < kCols; ++i)
        if (m0 + i < p.M) p.Y[(size_t)(m0 + i) * p.N + n] = __half_as_ushort(__float2half_rn(acc[i]));
      if (threadIdx.x == 4 * 32) p.counters[t] = 0;
    };

    const uint32_t inv16 = 0x2C002C00u;  // 1/16
    for (int u = u_begin; u < u_end; ++u) {
      const int t = u / p.Gk;
      if (t != cur_t) {
        if (cur_t >= 0) { epilogue(cur_t, seg_u0, u, first_seg_flag); first_seg_flag = false; }
        cur_t = t;
        seg_u0 = u;
      }
      mbar_wait(&full_bar[s], ph);
      const uint8_t* st = smem + s * C::kStage;
      const uint32_t wbase = smem_u32(st + C::kXBytes) + row * 64 + h * 32;
      // rotate the two 16-byte reads by row parity: halves the shared-memory bank conflicts of the 64-byte rows
      const int r0 = (row >> 1) & 1;
      const uint4 w0 = lds128(wbase + r0 * 16), w1 = lds128(wbase + (r0 ^ 1) * 16);
      const uint4 wlo = r0 ? w1 : w0, whi = r0 ? w0 : w1;
      const uint16_t* ssc = reinterpret_cast<const uint16_t*>(st + C::kXBytes + kUnitWBytes);
      const uint32_t s2 = h2_bcast(ssc[row]);
      uint32_t zlo, zhi;
      if (SYM) {
        zlo = 0x64086408u;  // 1032
        zhi = 0xD480D480u;  // -72
      } else {
        const __half z = __ushort_as_half(ssc[kTileN + row]);
        zlo = h2_bcast(__half_as_ushort(__hadd(z, __float2half_rn(1024.f))));
        zhi = h2_bcast(__half_as_ushort(__hneg(__hadd(z, __float2half_rn(64.f)))));
      }
      const uint32_t wv[8] = {wlo.x, wlo.y, wlo.z, wlo.w, whi.x, whi.y, whi.z, whi.w};
      uint32_t a[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t w = wv[j], w8 = w >> 8;
        a[4 * j + 0] = hmul2_u32(hsub2_u32(lop3_mask_or(w, 0x000F000Fu), zlo), s2);          // k 8j+0, 8j+1
        a[4 * j + 1] = hmul2_u32(hfma2_u32(lop3_mask_or(w, 0x00F000F0u), inv16, zhi), s2);   // k 8j+2, 8j+3
        a[4 * j + 2] = hmul2_u32(hsub2_u32(lop3_mask_or(w8, 0x000F000Fu), zlo), s2);         // k 8j+4, 8j+5
        a[4 * j + 3] = hmul2_u32(hfma2_u32(lop3_mask_or(w8, 0x00F000F0u), inv16, zhi), s2);  // k 8j+6, 8j+7
      }
      mbar_wait(&aempty_bar[b], aph ^ 1);   // the MMAs that last read this A buffer have completed
      tc_fence_after();
      tmem_st_x32(tmem + lane_base + b * 64 + h * 32, a);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull_bar[b]);
      if (++s == S) { s = 0; ph ^= 1; }
      if (++b == kNumA) { b = 0; aph ^= 1; }
    }
    if (cur_t >= 0) epilogue(cur_t, seg_u0, u_end, first_seg_flag);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// ---- host side ----
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

template <int MPAD, bool SYM>
int launch(const uint16_t* X, const Params& p, cudaStream_t stream) {
  using C = Cfg<MPAD>;
  auto enc = get_encode();
  if (!enc) return W4A16_ERR_CUDA;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)p.K, (cuuint64_t)p.M};
  const cuuint64_t strides[1] = {(cuuint64_t)p.K * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)MPAD};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint16_t*>(X), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return W4A16_ERR_CUDA;
  auto kern = gemm_w4a16_tc_kernel<MPAD, SYM>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem) != cudaSuccess)
      return W4A16_ERR_CUDA;
    attr = true;
  }
  kern<<<p.G, kThreads, C::kSmem, stream>>>(map, p);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

}  // namespace tc
}  // namespace w4

extern "C" int w4a16_tc_plan_ctas(int K, int N, int num_sms) {
  const long long U = (long long)(N / w4::tc::kTileN) * (K / w4::tc::kTileK);
  return (int)(U < num_sms ? U : num_sms);
}

extern "C" size_t w4a16_tc_workspace_bytes(int M, int K, int N, int num_sms) {
  const int mpad = (M + 15) / 16 * 16;
  const size_t counters = (((size_t)(N / w4::tc::kTileN) * 4) + 255) / 256 * 256;
  return counters + (size_t)2 * w4a16_tc_plan_ctas(K, N, num_sms) * mpad * w4::tc::kTileN * 4;
}

extern "C" int w4a16_launch_gemm_tc(const uint16_t* X, const uint32_t* qweight, const uint16_t* scales,
                                    const uint16_t* zeros, uint16_t* Y, int M, int K, int N, int mode, void* ws,
                                    int num_sms, cudaStream_t stream) {
  w4::tc::Params p;
  p.qweight = qweight; p.scales = scales; p.zeros = zeros; p.Y = Y;
  p.M = M; p.K = K; p.N = N;
  p.Gk = K / w4::tc::kTileK;
  p.U = (N / w4::tc::kTileN) * p.Gk;
  p.G = w4a16_tc_plan_ctas(K, N, num_sms);
  const size_t counters = (((size_t)(N / w4::tc::kTileN) * 4) + 255) / 256 * 256;
  p.counters = reinterpret_cast<int*>(ws);
  p.partials = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + counters);
  const int mpad = (M + 15) / 16 * 16;
  const bool sym = mode == W4A16_SYM;
#define W4_TC_CASE(MP) \
  case MP: return sym ? w4::tc::launch<MP, true>(X, p, stream) : w4::tc::launch<MP, false>(X, p, stream);
  switch (mpad) {
    W4_TC_CASE(16) W4_TC_CASE(32) W4_TC_CASE(48) W4_TC_CASE(64)
    default: return W4A16_ERR_SHAPE;
  }
#undef W4_TC_CASE
}
