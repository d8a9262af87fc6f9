// tree_attn.cu — tree-masked verify attention and KV compaction.
//
// The other half of the verify forward: the M verify rows (root + draft tree) attend the cached
// prefix and, inside the tree, only themselves and their ancestors (the ancestry mask). After
// verify_accept the accepted root-to-leaf path's keys/values are moved behind the root, so the
// cache again holds a plain sequence.
//
// w4a16_tree_attention: split-KV flash attention on the tensor cores (mma.sync m16n8k16, fp32 softmax), ONE
// cooperative launch.
//  * CTA = (kv head g, block of 64 query rows, KV split). Query row r of head group g is (token m = r / G,
//    head g*G + r % G), G = Hq / Hkv: the G query heads that share a kv head (GQA) share every K/V load.
//  * K/V chunks of 64 positions arrive by TMA (3-D tensor maps over [position][kv head][d], SWIZZLE_128B, rows
//    past L + M zero-filled) into a 2-buffer ring: at the usual split sizes every chunk of the CTA is in flight
//    from its first instruction. 4 warps x 16 query rows: S = Q K^T (ldmatrix + mma), the mask (prefix
//    visible; tree row L + j visible iff j is an ancestor of m or m itself: a 64-bit ancestor mask per token),
//    online softmax in fp32 (exp2), O += P V (P from the S registers, V through ldmatrix.trans).
//  * Split merge in the same launch: each split writes its unnormalised O, running max and sum (fp32), the
//    splits of one (kv head, row block) meet at a sense-reversing counter in the workspace header (all CTAs
//    are co-resident: cooperative launch), then split s merges rows s, s + splits, ... of the block.
// w4a16_kv_compact: for k = 1..accepted, cache row L + k <- row L + path[k-1] (path[k-1] >= k, so ascending
// k never overwrites a row still to be read); reads the acceptance result from device memory.
#include <cstdlib>

#include "common.cuh"
#include "tma_host.cuh"
#include "w4a16.h"

namespace w4 {
namespace ta {

constexpr int kD = 128;             // head dimension
constexpr int kRowsBlk = 64;        // query rows per CTA
constexpr int kKv = 64;             // KV positions per chunk
#ifndef W4_TA_PH
#define W4_TA_PH 2   // 4 (16 warps) measured slower: M = 8 13.9 vs 12.6 us, M = 61 39.1 vs 36.9 us
#endif
constexpr int kPH = W4_TA_PH;        // position slices of every chunk (one warp each per row quarter)
constexpr int kWarps = 4 * kPH;      // 4 row quarters (16 rows) x kPH position slices
constexpr int kThreads = 32 * kWarps;
constexpr int kPW = kKv / kPH;       // positions per warp and chunk
constexpr int kJ = kPW / 8;          // 8-position MMA n-tiles per warp and chunk
static_assert(kJ % 2 == 0 || kJ == 1, "K fragments are loaded two n-tiles at a time");
constexpr int kTileBytes = 64 * kD * 2;   // 16 KB: 64 rows x 256 B, as two SW128 halves of 64 rows x 128 B
constexpr int kKvBufs = 4;                // K/V chunk ring
constexpr int kSmem = kTileBytes * (1 + 2 * kKvBufs) + 64 * 8 + 64 * 4 + 1024;   // Q, (K, V) x bufs, masks, parents
constexpr int kCtasPerSmEst = 1;
constexpr int kHeaderBytes = 65536;       // workspace header: per (kv head, row block) {count, generation} on its own
constexpr int kMaxGroups = kHeaderBytes / 128;   // 128-byte line (the splits' atomics of neighbouring groups do not meet)

struct Params {
  const uint16_t* Q;
  const int32_t* parents;
  uint16_t* O;
  int M, L, Hq, Hkv, G, R;   // R = M * G query rows per kv head
  int qblocks, splits, chunks_per_split;
  int* bar;                  // workspace header: [Hkv * qblocks][8] ints
  float* o_part;             // [splits][Hkv][qblocks * 64][kD]
  float* m_part;             // [splits][Hkv][qblocks * 64]
  float* l_part;
  float scale_log2;          // log2(e) / sqrt(D)
};

// row r, 16-byte chunk c (0..15) of a 64-row tile stored as two SW128 halves [d 0..63 | d 64..127] of
// 64 rows x 128 B (the TMA box layout): chunk c & 7 of row r sits at position (c & 7) ^ (r & 7)
__device__ __forceinline__ uint32_t tile_off(int r, int c) { return (c >> 3) * 8192 + r * 128 + (((c & 7) ^ (r & 7)) << 4); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) { return h22u(__floats2half2_rn(a, b)); }
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) tree_attn_kernel(const __grid_constant__ CUtensorMap kmap,
                                                                           const __grid_constant__ CUtensorMap vmap,
                                                                           const Params p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[kKvBufs];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem), sK0 = sQ + kTileBytes, sV0 = sQ + (1 + kKvBufs) * kTileBytes;
  unsigned long long* anc = reinterpret_cast<unsigned long long*>(smem + (1 + 2 * kKvBufs) * kTileBytes);
  const int split = blockIdx.x, qb = blockIdx.y, g = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, c4 = lane & 3;
  const int wq = warp & 3, ph = warp >> 2;   // row quarter (rows 16 wq ..) and position half (32 ph .. of a chunk)
  const int P = p.L + p.M;
  const int ch0 = split * p.chunks_per_split;
  const int ch1 = min(ch0 + p.chunks_per_split, (P + kKv - 1) / kKv);
  const int nch = ch1 - ch0;

  // chunk i of this split -> ring buffer i % kKvBufs: K and V, each two SW128 boxes (d 0..63, d 64..127)
  auto issue = [&](int i) {
    const int b = i % kKvBufs, pos = (ch0 + i) * kKv;
    const uint32_t bar = smem_u32(&full[b]);
    mbar_expect_tx(&full[b], 2 * kTileBytes);
    tma_3d(sK0 + b * kTileBytes, &kmap, 0, g, pos, bar);
    tma_3d(sK0 + b * kTileBytes + 8192, &kmap, 64, g, pos, bar);
    tma_3d(sV0 + b * kTileBytes, &vmap, 0, g, pos, bar);
    tma_3d(sV0 + b * kTileBytes + 8192, &vmap, 64, g, pos, bar);
  };
  if (tid == 0) {
    for (int b = 0; b < kKvBufs; ++b) mbar_init(&full[b], 1);
    fence_mbar_init();
    for (int i = 0; i < nch && i < kKvBufs; ++i) issue(i);
  }

  // ancestor masks: bit j of anc[m] <=> tree row j is m or an ancestor of m. The parents go to shared
  // memory in one parallel load; then each token walks up its own path (depth <= M) in shared memory.
  int* spar = reinterpret_cast<int*>(anc + 64);
  if (tid < p.M) spar[tid] = p.parents[tid];
  __syncthreads();   // also publishes the barrier initialisation
  if (tid < p.M) {
    // A parent outside [-1, x) is invalid: such a row sees the prefix and itself only. Every step of a valid
    // walk strictly decreases x, so the walk ends within M steps (no hang on a cyclic "tree").
    unsigned long long a = 1ull << tid;
    for (int x = tid; x >= 0;) {
      const int px = spar[x];
      if (px < -1 || px >= x) { a = 1ull << tid; break; }
      if (px >= 0) a |= 1ull << px;
      x = px;
    }
    anc[tid] = a;
  }
  // Q block: row r -> (token m = r / G, head g*G + r % G)
  {
    // thread tid loads 16-byte chunk c = tid & 15 of rows r = tid / 16 + 16 k; (token, head) of the row are
    // stepped incrementally (no integer division per element)
    constexpr int kStep = kThreads / 16;
    const int c = tid & 15;
    int r = tid >> 4, rr = qb * kRowsBlk + r, m = rr / p.G, j = rr - m * p.G;
    for (; r < kRowsBlk; r += kStep, rr += kStep) {
      const bool ok = rr < p.R;
      cp_async16(sQ + tile_off(r, c), p.Q + ((size_t)(ok ? m : 0) * p.Hq + (ok ? g * p.G + j : 0)) * kD + c * 8, ok);
      for (j += kStep; j >= p.G; j -= p.G) ++m;
    }
  }
  cp_async_commit();
  cp_async_wait0();
  __syncthreads();

  // this lane's two query rows (g8, g8 + 8 of the warp's 16) and their tokens
  const int r_lo = qb * kRowsBlk + 16 * wq + g8, r_hi = r_lo + 8;
  const int m_lo = min(r_lo / p.G, p.M - 1), m_hi = min(r_hi / p.G, p.M - 1);
  float o[16][4];
#pragma unroll
  for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mx[2] = {-INFINITY, -INFINITY}, sum[2] = {0.f, 0.f};

  for (int i = 0; i < nch; ++i) {
    const int ch = ch0 + i, buf = i % kKvBufs;
    mbar_wait(&full[buf], (uint32_t)((i / kKvBufs) & 1));
    const uint32_t sK = sK0 + buf * kTileBytes, sV = sV0 + buf * kTileBytes;
    // S = Q K^T: 16 rows x 32 positions (this warp's half of the chunk)
    float s[kJ][4];
#pragma unroll
    for (int j = 0; j < kJ; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(sQ + tile_off(16 * wq + (lane & 15), 2 * ks + (lane >> 4)), a0, a1, a2, a3);
#pragma unroll
      for (int j = 0; j < kJ; j += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sK + tile_off(kPW * ph + 8 * j + (lane & 7) + ((lane >> 4) << 3), 2 * ks + ((lane >> 3) & 1)), b0, b1, b2, b3);
        mma_16816_nv(s[j], a0, a1, a2, a3, b0, b1);
        mma_16816_nv(s[j + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // mask, scale, online softmax (rows lo = e 0,1; hi = e 2,3)
    float cmax[2] = {-INFINITY, -INFINITY};
    if ((ch + 1) * kKv <= p.L) {   // the whole chunk is cached prefix: visible to every row
#pragma unroll
      for (int j = 0; j < kJ; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          s[j][e] *= p.scale_log2;
          cmax[e >> 1] = fmaxf(cmax[e >> 1], s[j][e]);
        }
    } else {
      const unsigned long long al = anc[m_lo], ah = anc[m_hi];
#pragma unroll
      for (int j = 0; j < kJ; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int pos = ch * kKv + kPW * ph + 8 * j + 2 * c4 + (e & 1);
          const unsigned long long a = (e < 2) ? al : ah;
          const bool vis = pos < p.L || (pos < P && ((a >> (pos - p.L)) & 1ull));
          const float v = vis ? s[j][e] * p.scale_log2 : -INFINITY;
          s[j][e] = v;
          cmax[e >> 1] = fmaxf(cmax[e >> 1], v);
        }
    }
    float corr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 1));
      cmax[h] = fmaxf(cmax[h], __shfl_xor_sync(0xffffffffu, cmax[h], 2));
      const float mnew = fmaxf(mx[h], cmax[h]);
      corr[h] = mnew == -INFINITY ? 1.f : exp2f(mx[h] - mnew);
      mx[h] = mnew;
      sum[h] *= corr[h];
    }
#pragma unroll
    for (int j = 0; j < kJ; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float m_ = mx[e >> 1];
        const float pr = m_ == -INFINITY ? 0.f : exp2f(s[j][e] - m_);
        s[j][e] = pr;
        sum[e >> 1] += pr;
      }
#pragma unroll
    for (int n = 0; n < 16; ++n) {
      o[n][0] *= corr[0]; o[n][1] *= corr[0]; o[n][2] *= corr[1]; o[n][3] *= corr[1];
    }
    // O += P V: P (16 x 32) from the S registers as the A operand, V^T through ldmatrix.trans
#pragma unroll
    for (int t = 0; t < kJ / 2; ++t) {
      const uint32_t a0 = pack_h2(s[2 * t][0], s[2 * t][1]), a1 = pack_h2(s[2 * t][2], s[2 * t][3]);
      const uint32_t a2 = pack_h2(s[2 * t + 1][0], s[2 * t + 1][1]), a3 = pack_h2(s[2 * t + 1][2], s[2 * t + 1][3]);
#pragma unroll
      for (int n = 0; n < 16; n += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sV + tile_off(kPW * ph + 16 * t + (lane & 7) + (((lane >> 3) & 1) << 3), n + (lane >> 4)), b0, b1, b2, b3);
        mma_16816_nv(o[n], a0, a1, a2, a3, b0, b1);
        mma_16816_nv(o[n + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();   // every warp is done with this buffer: refill it
    if (tid == 0 && i + kKvBufs < nch) issue(i + kKvBufs);
  }
  // row sums across the 4 lanes of a row
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    sum[h] += __shfl_xor_sync(0xffffffffu, sum[h], 1);
    sum[h] += __shfl_xor_sync(0xffffffffu, sum[h], 2);
  }
  // combine the position slices (the K/V ring is free now): slices 1.. hand (max, sum, O) to slice 0
  {
    // slot q - 1 holds slice q: [4 warps][16 n][4][32 lanes] of O, then [4][4][32] of (max, sum)
    constexpr int kSlot = 4 * 64 * 32 + 4 * 4 * 32;
    float* xo = reinterpret_cast<float*>(smem + kTileBytes) + (ph > 0 ? ph - 1 : 0) * kSlot;
    float* xm = xo + 4 * 64 * 32;
    const int base = wq * 64 * 32 + lane;
    if (ph > 0) {
#pragma unroll
      for (int n = 0; n < 16; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) xo[base + (4 * n + e) * 32] = o[n][e];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        xm[(wq * 4 + h) * 32 + lane] = mx[h];
        xm[(wq * 4 + 2 + h) * 32 + lane] = sum[h];
      }
    }
    __syncthreads();
    if (ph > 0) {
      if (p.splits == 1) return;
    } else {
      for (int q = 1; q < kPH; ++q, xo += kSlot, xm += kSlot)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float m2 = xm[(wq * 4 + h) * 32 + lane], l2 = xm[(wq * 4 + 2 + h) * 32 + lane];
        const float mn = fmaxf(mx[h], m2);
        const float c1 = mx[h] == -INFINITY ? 0.f : exp2f(mx[h] - mn), c2 = m2 == -INFINITY ? 0.f : exp2f(m2 - mn);
        mx[h] = mn;
        sum[h] = sum[h] * c1 + l2 * c2;
#pragma unroll
        for (int n = 0; n < 16; ++n) {
          o[n][2 * h] = o[n][2 * h] * c1 + xo[base + (4 * n + 2 * h) * 32] * c2;
          o[n][2 * h + 1] = o[n][2 * h + 1] * c1 + xo[base + (4 * n + 2 * h + 1) * 32] * c2;
        }
      }
    }
  }
  const int rl = qb * kRowsBlk + 16 * wq + g8;
  if (p.splits == 1) {   // the whole prefix in one CTA: normalise and write O
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = rl + 8 * h;
      if (r >= p.R) continue;
      const float inv = 1.f / sum[h];
      uint16_t* out = p.O + ((size_t)(r / p.G) * p.Hq + g * p.G + r % p.G) * kD;
#pragma unroll
      for (int n = 0; n < 16; ++n)
        *reinterpret_cast<uint32_t*>(out + 8 * n + 2 * c4) = pack_h2(o[n][2 * h] * inv, o[n][2 * h + 1] * inv);
    }
    return;
  }
  // this split's partial results (half-0 warps)
  const int Rpad = p.qblocks * kRowsBlk;
  const size_t base = ((size_t)split * p.Hkv + g) * Rpad;
#pragma unroll
  for (int h = 0; h < 2 && ph == 0; ++h) {
    const int r = rl + 8 * h;
    float* op = p.o_part + (base + r) * kD;
#pragma unroll
    for (int n = 0; n < 16; ++n) __stcg(reinterpret_cast<float2*>(op + 8 * n + 2 * c4), make_float2(o[n][2 * h], o[n][2 * h + 1]));
    if (c4 == 0) {
      __stcg(&p.m_part[base + r], mx[h]);
      __stcg(&p.l_part[base + r], sum[h]);
    }
  }
  // meet the other splits of this (kv head, row block): sense-reversing counter (the count returns to 0)
  __syncthreads();
  if (tid == 0) {
    int* cnt = p.bar + 32 * (g * p.qblocks + qb);
    int* gen = cnt + 1;
    const int g0 = ld_relaxed_gpu(gen);
    int arrived;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(arrived) : "l"(cnt) : "memory");
    if (arrived == p.splits - 1) {
      *cnt = 0;
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(gen), "r"(g0 + 1) : "memory");
    } else {
      const unsigned long long t0 = globaltimer_ns();
      while (ld_acquire_gpu(gen) == g0) {
        __nanosleep(32);
        if (globaltimer_ns() - t0 > 10000000000ull) __trap();   // never hang the device on a protocol bug
      }
    }
  }
  __syncthreads();
  // merge: O = sum_s 2^(m_s - m*) O_s / sum_s 2^(m_s - m*) l_s, fp16 out; this split takes rows split,
  // split + splits, ... of the block, one warp per row (lanes over the 128 head dims as float4)
  for (int lr = split + warp * p.splits; lr < kRowsBlk; lr += kWarps * p.splits) {
    const int r = qb * kRowsBlk + lr;
    if (r >= p.R) break;
    float mstar = -INFINITY;
    for (int sp = lane; sp < p.splits; sp += 32) mstar = fmaxf(mstar, __ldcg(&p.m_part[((size_t)sp * p.Hkv + g) * Rpad + r]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mstar = fmaxf(mstar, __shfl_xor_sync(0xffffffffu, mstar, off));
    float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
    float den = 0.f;
    constexpr int kB = 9;    // splits' loads in flight at a time
    for (int sp0 = 0; sp0 < p.splits; sp0 += kB) {
      float ms[kB], l[kB];
      float4 v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const bool in = sp0 + u < p.splits;   // no loads past the last split
        const size_t ix = ((size_t)(in ? sp0 + u : 0) * p.Hkv + g) * Rpad + r;
        ms[u] = in ? __ldcg(&p.m_part[ix]) : -INFINITY;
        l[u] = in ? __ldcg(&p.l_part[ix]) : 0.f;
        v[u] = in ? __ldcg(reinterpret_cast<const float4*>(p.o_part + ix * kD) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (ms[u] == -INFINITY) continue;
        const float w = exp2f(ms[u] - mstar);
        num.x += w * v[u].x; num.y += w * v[u].y; num.z += w * v[u].z; num.w += w * v[u].w;
        den += w * l[u];
      }
    }
    const float inv = 1.f / den;
    const int m = r / p.G, h = g * p.G + r % p.G;
    uint2 out;
    out.x = pack_h2(num.x * inv, num.y * inv);
    out.y = pack_h2(num.z * inv, num.w * inv);
    *reinterpret_cast<uint2*>(p.O + ((size_t)m * p.Hq + h) * kD + 4 * lane) = out;
  }
}

__global__ void kv_compact_kernel(uint16_t* K, uint16_t* V, int L, int row_vec, const int32_t* __restrict__ acc) {
  const int n = acc[0];
  const int c = blockIdx.x * blockDim.x + threadIdx.x;   // 16-byte chunk of a row
  if (c >= row_vec) return;
  uint4* K4 = reinterpret_cast<uint4*>(K);
  uint4* V4 = reinterpret_cast<uint4*>(V);
  for (int k = 1; k <= n; ++k) {   // ascending k: path[k-1] >= k, so no row is overwritten before it is read
    const size_t src = (size_t)(L + acc[3 + k - 1]) * row_vec + c, dst = (size_t)(L + k) * row_vec + c;
    const uint4 kv = K4[src], vv = V4[src];
    K4[dst] = kv;
    V4[dst] = vv;
  }
}

}  // namespace ta
}  // namespace w4

namespace {
void plan_splits(int M, int L, int Hq, int Hkv, int sms, int* qblocks, int* splits, int* cps) {
  const int G = Hq / Hkv, R = M * G;
  *qblocks = (R + w4::ta::kRowsBlk - 1) / w4::ta::kRowsBlk;
  const int chunks = (L + M + w4::ta::kKv - 1) / w4::ta::kKv;
  // every CTA of a call must be resident (the splits are merged in-kernel): at most kCtasPerSmEst per SM
  int s = (w4::ta::kCtasPerSmEst * sms) / (Hkv * *qblocks);
  static int min_cps = -1;   // diagnostics: W4A16_TA_CPS overrides the minimum chunks per split
  if (min_cps < 0) { const char* e = getenv("W4A16_TA_CPS"); min_cps = e ? atoi(e) : 2; if (min_cps < 1) min_cps = 1; }
  const int max_s = (chunks + min_cps - 1) / min_cps;   // at least two chunks per split where there are two (fewer partials)
  s = s < 1 ? 1 : s > max_s ? max_s : s;
  *cps = (chunks + s - 1) / s;
  *splits = (chunks + *cps - 1) / *cps;
}
}  // namespace

extern "C" size_t w4a16_tree_attention_workspace_bytes_sms(int M, int L, int Hq, int Hkv, int sms) {
  int qb, sp, cps;
  plan_splits(M, L, Hq, Hkv, sms, &qb, &sp, &cps);
  const size_t rows = (size_t)sp * Hkv * qb * w4::ta::kRowsBlk;
  return w4::ta::kHeaderBytes + rows * (w4::ta::kD + 2) * 4;
}

namespace {
// Kc / Vc [P][Hkv][128] fp16 viewed as 3-D (d, kv head, position) with box (64 d, 1 head, 64 positions), SW128:
// one TMA lands a [64 positions][128 B] half of a chunk; positions >= P are zero-filled.
int encode_kv(CUtensorMap* map, const uint16_t* base, int P, int Hkv) {
  auto enc = w4::get_encode();
  if (!enc) return W4A16_ERR_CUDA;
  const cuuint64_t dims[3] = {(cuuint64_t)w4::ta::kD, (cuuint64_t)Hkv, (cuuint64_t)P};
  const cuuint64_t strides[2] = {(cuuint64_t)w4::ta::kD * 2, (cuuint64_t)Hkv * w4::ta::kD * 2};
  const cuuint32_t box[3] = {64, 1, (cuuint32_t)w4::ta::kKv};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<uint16_t*>(base), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return W4A16_ERR_CUDA;
  return W4A16_OK;
}
}  // namespace

extern "C" int w4a16_launch_tree_attention(const uint16_t* Q, const uint16_t* K, const uint16_t* V, const int32_t* parents,
                                           int M, int L, int Hq, int Hkv, uint16_t* O, void* ws, int sms,
                                           cudaStream_t stream) {
  using namespace w4::ta;
  static unsigned long long attr = 0;
  if (!w4::ensure_smem_attr(tree_attn_kernel, kSmem, attr)) return W4A16_ERR_CUDA;
  // the split merge needs every CTA resident (cooperative launch): plan with the real occupancy, never more
  // CTAs per SM than the workspace was sized for
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tree_attn_kernel, kThreads, kSmem) != cudaSuccess || occ < 1)
    return W4A16_ERR_CUDA;
  Params p;
  p.Q = Q; p.parents = parents; p.O = O;
  p.M = M; p.L = L; p.Hq = Hq; p.Hkv = Hkv; p.G = Hq / Hkv; p.R = M * p.G;
  plan_splits(M, L, Hq, Hkv, sms * (occ < kCtasPerSmEst ? occ : kCtasPerSmEst) / kCtasPerSmEst, &p.qblocks, &p.splits,
              &p.chunks_per_split);
  if (Hkv * p.qblocks > kMaxGroups) return W4A16_ERR_SHAPE;
  const size_t rows = (size_t)p.splits * Hkv * p.qblocks * kRowsBlk;
  p.bar = reinterpret_cast<int*>(ws);
  p.o_part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + kHeaderBytes);
  p.m_part = p.o_part + rows * kD;
  p.l_part = p.m_part + rows;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)kD);
  CUtensorMap kmap, vmap;
  if (int e = encode_kv(&kmap, K, L + M, Hkv)) return e;
  if (int e = encode_kv(&vmap, V, L + M, Hkv)) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.splits, p.qblocks, Hkv);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeCooperative;
  la[0].val.cooperative = 1;
  cfg.attrs = la;
  cfg.numAttrs = p.splits > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, tree_attn_kernel, kmap, vmap, p) == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" int w4a16_launch_kv_compact(uint16_t* K, uint16_t* V, int L, int Hkv, int D, const int32_t* accept_out,
                                       cudaStream_t stream) {
  const int row_vec = Hkv * D / 8;
  w4::ta::kv_compact_kernel<<<(row_vec + 127) / 128, 128, 0, stream>>>(K, V, L, row_vec, accept_out);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}
