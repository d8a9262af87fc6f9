// lmhead.cu — w4a16_lmhead_argmax: the target's greedy token for every verify row.
//
//   argmax_v  sum_k H[m][k] * W[v][k]     (FP16 LM head, fp32 accumulation; ties -> lowest id)
//
// The greedy acceptance rule (verify_accept, P:79-84 / S:289) needs the target's argmax after every verify
// row; this is the LM head GEMM [M, K] x [K, V] with the argmax fused into its epilogue, so the M x V logits
// never reach HBM. At M <= 64 the 2.1 GB fp16 head of Llama-3-70B (V = 128256) is HBM-bound (2M flop/B).
//  * Work: 128-row vocabulary tiles, a contiguous run of tiles per CTA, one persistent CTA per SM.
//  * Warp 8 (producer) streams one 128-k chunk of the tile per stage: W as a 3-D SWIZZLE_128B TMA box
//    [2 x 64 k][128 rows] (32 KB) and the matching H box [2 x 64 k][Mpad rows], into a ring of stages.
//  * Warps 0..7: warp w owns rows 16w..16w+15 of the tile. mma.sync m16n8k16 with the vocabulary as MMA-M
//    (A = W rows via ldmatrix.x4) and the tokens as MMA-N (B = H rows via ldmatrix.x2), fp32 accumulators.
//  * Tile epilogue: per token, the (logit, id) maximum over the warp's rows (shuffles), over the 8 warps
//    (shared memory), then into the CTA's running best. The last CTA to finish reduces the per-CTA bests
//    (ordered by (logit desc, id asc), so any order gives the same answer) and writes argmax / max logit.
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "tma_host.cuh"
#include "w4a16.h"

namespace w4 {
namespace lm {

constexpr int kRows = 128;                 // vocabulary rows per tile
constexpr int kWarps = 8;                  // consumer warps (16 rows each)
constexpr int kThreads = (kWarps + 1) * 32;
constexpr int kWBytes = kRows * 128 * 2;   // one 128-k chunk of a tile: 32 KB

template <int NTB>
struct Cfg {
  static constexpr int kMpad = 8 * NTB;
  static constexpr int kXBytes = 2 * kMpad * 128;   // [2 x 64 k][Mpad rows][128 B]
  static constexpr int kStage = kWBytes + kXBytes;  // multiple of 1024 (SW128 atoms)
  static constexpr int kStagesFit = (200 * 1024) / kStage;
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  static constexpr int kSmem = kStages * kStage + 1024;
};

struct Params {
  int M, K, V, G, T;    // T = V / 128 tiles
  int32_t* out_idx;
  float* out_val;
  float* part_val;      // [G][64]
  int* part_idx;        // [G][64]
  int* counter;
};

__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& b0, uint32_t& b1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(addr));
}
// (val, idx) order of the greedy argmax: larger logit first, then the lower id.
__device__ __forceinline__ bool better(float v, int i, float bv, int bi) { return v > bv || (v == bv && i < bi); }

template <int NTB>
__global__ void __launch_bounds__(kThreads, 1) lmhead_argmax_kernel(const __grid_constant__ CUtensorMap wmap,
                                                                    const __grid_constant__ CUtensorMap hmap,
                                                                    const Params p) {
  using C = Cfg<NTB>;
  constexpr int S = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[S], empty_bar[S];
  __shared__ float red_val[kWarps][64];
  __shared__ int red_idx[kWarps][64];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t base = smem_u32(smem);
  const int t0 = (int)((long long)blockIdx.x * p.T / p.G), t1 = (int)((long long)(blockIdx.x + 1) * p.T / p.G);
  const int nk = p.K / 128;
  const int n_stages = (t1 - t0) * nk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], kWarps); }
    fence_mbar_init();
    pdl_launch_dependents();
  }
  __syncthreads();

  if (warp == kWarps) {
    // ---------------- producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&hmap)) : "memory");
      auto load_w = [&](int i, int s) {   // the head's weights never depend on a preceding kernel
        const int t = t0 + i / nk, kc = i % nk;
        mbar_expect_tx(&full_bar[s], C::kStage);
        tma_3d(base + s * C::kStage, &wmap, 0, t * kRows, 2 * kc, &full_bar[s]);
      };
      auto load_h = [&](int i, int s) {
        tma_3d(base + s * C::kStage + kWBytes, &hmap, 0, 0, 2 * (i % nk), &full_bar[s]);
      };
      const int pre = min(S, n_stages);
      for (int i = 0; i < pre; ++i) load_w(i, i);
      pdl_wait();   // H is written by the preceding kernel
      for (int i = 0; i < pre; ++i) load_h(i, i);
      int s = pre % S;
      uint32_t ph = pre == S ? 1 : 0;
      for (int i = pre; i < n_stages; ++i) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        load_w(i, s);
        load_h(i, s);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  pdl_wait();
  const int g8 = lane >> 2, c4 = lane & 3;
  float best_v = -INFINITY;   // running best of token threadIdx.x (threads < M)
  int best_i = 0x7fffffff;
  int s = 0;
  uint32_t ph = 0;
  // ldmatrix row addresses: A = rows 16w + (lane & 15), 16-byte chunk (lane >> 4) of a k16 step;
  // B = token rows (lane & 7), chunk ((lane >> 3) & 1)
  const int ar = 16 * warp + (lane & 15), ac = lane >> 4;
  const int br = lane & 7, bc = (lane >> 3) & 1;
  for (int t = t0; t < t1; ++t) {
    float acc[NTB][4];
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb) acc[tb][0] = acc[tb][1] = acc[tb][2] = acc[tb][3] = 0.f;
    for (int kc = 0; kc < nk; ++kc) {
      mbar_wait(&full_bar[s], ph);
      const uint32_t st = base + s * C::kStage;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        const uint32_t wb = st + kb * (kRows * 128), xb = st + kWBytes + kb * (C::kMpad * 128);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4(wb + ar * 128 + (((2 * ks + ac) ^ (ar & 7)) << 4), a0, a1, a2, a3);
#pragma unroll
          for (int tb = 0; tb < NTB; ++tb) {
            const int m = 8 * tb + br;
            uint32_t b0, b1;
            ldsm_x2(xb + m * 128 + (((2 * ks + bc) ^ (m & 7)) << 4), b0, b1);
            mma_16816_nv(acc[tb], a0, a1, a2, a3, b0, b1);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
    // tile epilogue: lane holds rows (g8, g8 + 8) x tokens (8tb + 2c4, +1)
    const int row0 = t * kRows + 16 * warp + g8;
#pragma unroll
    for (int tb = 0; tb < NTB; ++tb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {   // token 8tb + 2c4 + e: rows g8 (acc e) and g8 + 8 (acc 2 + e)
        float v = acc[tb][e];
        int i = row0;
        if (better(acc[tb][2 + e], row0 + 8, v, i)) { v = acc[tb][2 + e]; i = row0 + 8; }
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {   // across g8
          const float ov = __shfl_xor_sync(0xffffffffu, v, off);
          const int oi = __shfl_xor_sync(0xffffffffu, i, off);
          if (better(ov, oi, v, i)) { v = ov; i = oi; }
        }
        if (g8 == 0) {
          red_val[warp][8 * tb + 2 * c4 + e] = v;
          red_idx[warp][8 * tb + 2 * c4 + e] = i;
        }
      }
    named_bar_sync(1, kWarps * 32);
    if (threadIdx.x < p.M) {
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const float v = red_val[w][threadIdx.x];
        const int i = red_idx[w][threadIdx.x];
        if (better(v, i, best_v, best_i)) { best_v = v; best_i = i; }
      }
    }
    named_bar_sync(1, kWarps * 32);
  }
  // cross-CTA: publish, and the last CTA out reduces
  if (threadIdx.x < p.M) {
    p.part_val[blockIdx.x * 64 + threadIdx.x] = best_v;
    p.part_idx[blockIdx.x * 64 + threadIdx.x] = best_i;
  }
  __threadfence();
  named_bar_sync(1, kWarps * 32);
  if (threadIdx.x == 0) s_last = atomicAdd(p.counter, 1) == p.G - 1;
  named_bar_sync(1, kWarps * 32);
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < p.M) {
    float v = -INFINITY;
    int i = 0x7fffffff;
    for (int c = 0; c < p.G; ++c) {
      const float cv = __ldcg(&p.part_val[c * 64 + threadIdx.x]);
      const int ci = __ldcg(&p.part_idx[c * 64 + threadIdx.x]);
      if (better(cv, ci, v, i)) { v = cv; i = ci; }
    }
    p.out_idx[threadIdx.x] = i;
    if (p.out_val) p.out_val[threadIdx.x] = v;
  }
  if (threadIdx.x == 0) *p.counter = 0;   // re-armed for the next launch
}

template <int NTB>
int launch(const uint16_t* H, const uint16_t* W, const Params& p, cudaStream_t stream) {
  using C = Cfg<NTB>;
  CUtensorMap wmap, hmap;
  if (int e = encode_x_sw128(&wmap, W, p.V, p.K, kRows, 2)) return e;
  if (int e = encode_x_sw128(&hmap, H, p.M, p.K, C::kMpad, 2)) return e;
  auto kern = lmhead_argmax_kernel<NTB>;
  static unsigned long long attr = 0;
  if (!ensure_smem_attr(kern, C::kSmem, attr)) return W4A16_ERR_CUDA;
  return launch_pdl(kern, dim3(p.G), dim3(kThreads), C::kSmem, stream, wmap, hmap, p) == cudaSuccess ? W4A16_OK
                                                                                         : W4A16_ERR_CUDA;
}

}  // namespace lm
}  // namespace w4

extern "C" int w4a16_lmhead_ctas(int V, int num_sms) {
  const int T = V / w4::lm::kRows;
  return T < num_sms ? T : num_sms;
}

extern "C" size_t w4a16_lmhead_workspace_bytes_sms(int num_sms) {
  return 256 + (size_t)num_sms * 64 * 8;   // counter, then [G][64] values and [G][64] ids
}

extern "C" int w4a16_launch_lmhead_argmax(const uint16_t* H, const uint16_t* W, int M, int K, int V, int32_t* out_idx,
                                          float* out_val, void* ws, int num_sms, cudaStream_t stream) {
  w4::lm::Params p;
  p.M = M; p.K = K; p.V = V;
  p.T = V / w4::lm::kRows;
  p.G = w4a16_lmhead_ctas(V, num_sms);
  p.out_idx = out_idx;
  p.out_val = out_val;
  p.counter = reinterpret_cast<int*>(ws);
  p.part_val = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + 256);
  p.part_idx = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + 256 + (size_t)num_sms * 64 * 4);
  switch ((M + 7) / 8) {
    case 1: return w4::lm::launch<1>(H, W, p, stream);
    case 2: return w4::lm::launch<2>(H, W, p, stream);
    case 3: return w4::lm::launch<3>(H, W, p, stream);
    case 4: return w4::lm::launch<4>(H, W, p, stream);
    case 5: return w4::lm::launch<5>(H, W, p, stream);
    case 6: return w4::lm::launch<6>(H, W, p, stream);
    case 7: return w4::lm::launch<7>(H, W, p, stream);
    case 8: return w4::lm::launch<8>(H, W, p, stream);
    default: return W4A16_ERR_SHAPE;
  }
}
