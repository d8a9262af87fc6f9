// tree_attn.cu — tree-masked verify attention and KV compaction.
//
// The other half of the verify forward: the M verify rows (root + draft tree) attend the cached
// prefix and, inside the tree, only themselves and their ancestors (the ancestry mask). After
// verify_accept the accepted root-to-leaf path's keys/values are moved behind the root, so the
// cache again holds a plain sequence.
//
// w4a16_tree_attention: split-KV flash attention on the tensor cores (mma.sync m16n8k16, fp32 softmax).
//  * CTA = (kv head g, block of 64 query rows, KV split). Query row r of head group g is (token m = r / G,
//    head g*G + r % G), G = Hq / Hkv: the G query heads that share a kv head (GQA) share every K/V load.
//  * 4 warps x 16 query rows. Per 64-position KV chunk (cp.async into one buffer — three CTAs per SM hide
//    the latency better than double-buffering, measured —, XOR-swizzled rows):
//    S = Q K^T (ldmatrix + mma), the mask (prefix visible; tree row L + j visible iff j is an ancestor of m
//    or m itself: a 64-bit ancestor mask per token), online softmax in fp32 (exp2), O += P V (P from the S
//    registers, V through ldmatrix.trans).
//  * Each split writes its unnormalised O, running max and sum (fp32); tree_attn_combine merges the splits.
// w4a16_kv_compact: for k = 1..accepted, cache row L + k <- row L + path[k-1] (path[k-1] >= k, so ascending
// k never overwrites a row still to be read); reads the acceptance result from device memory.
#include "common.cuh"
#include "tma_host.cuh"
#include "w4a16.h"

namespace w4 {
namespace ta {

constexpr int kD = 128;             // head dimension
constexpr int kRowsBlk = 64;        // query rows per CTA
constexpr int kKv = 64;             // KV positions per chunk
constexpr int kThreads = 128;       // 4 warps x 16 rows
constexpr int kTileBytes = 64 * kD * 2;   // 16 KB: 64 rows x 256 B
#ifndef W4_TA_BUFS
#define W4_TA_BUFS 1
#endif
constexpr int kKvBufs = W4_TA_BUFS;       // K/V chunk buffers: 2 = double-buffered, 1 = more CTAs per SM
constexpr int kSmem = kTileBytes * (1 + 2 * kKvBufs) + 64 * 8 + 64 * 4 + 1024;   // Q, (K, V) x bufs, masks, parents
constexpr int kCtasPerSmEst = kKvBufs == 2 ? 2 : 3;

struct Params {
  const uint16_t* Q;
  const uint16_t* K;
  const uint16_t* V;
  const int32_t* parents;
  int M, L, Hq, Hkv, G, R;   // R = M * G query rows per kv head
  int qblocks, splits, chunks_per_split;
  float* o_part;             // [splits][Hkv][qblocks * 64][kD]
  float* m_part;             // [splits][Hkv][qblocks * 64]
  float* l_part;
  float scale_log2;          // log2(e) / sqrt(D)
};

// row r, 16-byte chunk c (0..15) of a [64][256 B] tile: XOR-swizzled within each 128-byte half
__device__ __forceinline__ uint32_t tile_off(int r, int c) { return r * 256 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) { return h22u(__floats2half2_rn(a, b)); }

__global__ void __launch_bounds__(kThreads) tree_attn_kernel(const Params p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the merge kernel may launch and wait
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem), sK0 = sQ + kTileBytes, sV0 = sQ + (1 + kKvBufs) * kTileBytes;
  unsigned long long* anc = reinterpret_cast<unsigned long long*>(smem + (1 + 2 * kKvBufs) * kTileBytes);
  const int split = blockIdx.x, qb = blockIdx.y, g = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, c4 = lane & 3;
  const int P = p.L + p.M;
  const int ch0 = split * p.chunks_per_split;
  const int ch1 = min(ch0 + p.chunks_per_split, (P + kKv - 1) / kKv);

  // ancestor masks: bit j of anc[m] <=> tree row j is m or an ancestor of m. The parents go to shared
  // memory in one parallel load; then each token walks up its own path (depth <= M) in shared memory.
  int* spar = reinterpret_cast<int*>(anc + 64);
  if (tid < p.M) spar[tid] = p.parents[tid];
  __syncthreads();
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
  for (int i = tid; i < kRowsBlk * 16; i += kThreads) {
    const int r = i >> 4, c = i & 15, rr = qb * kRowsBlk + r;
    const int m = rr / p.G, h = g * p.G + rr % p.G;
    const bool ok = rr < p.R;
    cp_async16(sQ + tile_off(r, c), p.Q + ((size_t)(ok ? m : 0) * p.Hq + (ok ? h : 0)) * kD + c * 8, ok);
  }
  auto load_kv = [&](int chunk, int buf) {
    for (int i = tid; i < kKv * 16; i += kThreads) {
      const int r = i >> 4, c = i & 15, pos = chunk * kKv + r;
      const bool ok = pos < P;
      const size_t off = ((size_t)(ok ? pos : 0) * p.Hkv + g) * kD + c * 8;
      cp_async16(sK0 + buf * kTileBytes + tile_off(r, c), p.K + off, ok);
      cp_async16(sV0 + buf * kTileBytes + tile_off(r, c), p.V + off, ok);
    }
  };
  if (kKvBufs == 2 && ch0 < ch1) load_kv(ch0, 0);
  cp_async_commit();

  // this lane's two query rows (g8, g8 + 8 of the warp's 16) and their tokens
  const int r_lo = qb * kRowsBlk + 16 * warp + g8, r_hi = r_lo + 8;
  const int m_lo = min(r_lo / p.G, p.M - 1), m_hi = min(r_hi / p.G, p.M - 1);
  float o[16][4];
#pragma unroll
  for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float mx[2] = {-INFINITY, -INFINITY}, sum[2] = {0.f, 0.f};

  for (int ch = ch0; ch < ch1; ++ch) {
    const int buf = kKvBufs == 2 ? (ch - ch0) & 1 : 0;
    if (kKvBufs == 2) {
      if (ch + 1 < ch1) load_kv(ch + 1, buf ^ 1);
      cp_async_commit();
      cp_async_wait1();
    } else {
      load_kv(ch, 0);
      cp_async_commit();
      cp_async_wait0();
    }
    __syncthreads();
    const uint32_t sK = sK0 + buf * kTileBytes, sV = sV0 + buf * kTileBytes;
    // S = Q K^T: 16 rows x 64 positions per warp
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4(sQ + tile_off(16 * warp + (lane & 15), 2 * ks + (lane >> 4)), a0, a1, a2, a3);
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sK + tile_off(8 * j + (lane & 7) + ((lane >> 4) << 3), 2 * ks + ((lane >> 3) & 1)), b0, b1, b2, b3);
        mma_16816_nv(s[j], a0, a1, a2, a3, b0, b1);
        mma_16816_nv(s[j + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    // mask, scale, online softmax (rows lo = e 0,1; hi = e 2,3)
    const unsigned long long al = anc[m_lo], ah = anc[m_hi];
    float cmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int pos = ch * kKv + 8 * j + 2 * c4 + (e & 1);
        const unsigned long long a = (e < 2) ? al : ah;
        const bool vis = pos < p.L || (pos < P && ((a >> (pos - p.L)) & 1ull));
        const float v = vis ? s[j][e] * p.scale_log2 : -INFINITY;
        s[j][e] = v;
        cmax[e >> 1] = fmaxf(cmax[e >> 1], v);
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
    for (int j = 0; j < 8; ++j)
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
    // O += P V: P (16 x 64) from the S registers as the A operand, V^T through ldmatrix.trans
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t a0 = pack_h2(s[2 * t][0], s[2 * t][1]), a1 = pack_h2(s[2 * t][2], s[2 * t][3]);
      const uint32_t a2 = pack_h2(s[2 * t + 1][0], s[2 * t + 1][1]), a3 = pack_h2(s[2 * t + 1][2], s[2 * t + 1][3]);
#pragma unroll
      for (int n = 0; n < 16; n += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(sV + tile_off(16 * t + (lane & 7) + (((lane >> 3) & 1) << 3), n + (lane >> 4)), b0, b1, b2, b3);
        mma_16816_nv(o[n], a0, a1, a2, a3, b0, b1);
        mma_16816_nv(o[n + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();   // the buffer is refilled by the next iteration's load
  }
  cp_async_wait0();
  // row sums across the 4 lanes of a row, then the split's partial results
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    sum[h] += __shfl_xor_sync(0xffffffffu, sum[h], 1);
    sum[h] += __shfl_xor_sync(0xffffffffu, sum[h], 2);
  }
  const int Rpad = p.qblocks * kRowsBlk;
  const size_t base = ((size_t)split * p.Hkv + g) * Rpad;
  const int rl = qb * kRowsBlk + 16 * warp + g8;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = rl + 8 * h;
    float* op = p.o_part + (base + r) * kD;
#pragma unroll
    for (int n = 0; n < 16; ++n)
      *reinterpret_cast<float2*>(op + 8 * n + 2 * c4) = make_float2(o[n][2 * h], o[n][2 * h + 1]);
    if (c4 == 0) {
      p.m_part[base + r] = mx[h];
      p.l_part[base + r] = sum[h];
    }
  }
}

// Merge the splits: O = sum_s 2^(m_s - m*) O_s / sum_s 2^(m_s - m*) l_s, fp16 out.
// Merge the splits: O = sum_s 2^(m_s - m*) O_s / sum_s 2^(m_s - m*) l_s, fp16 out. One warp per query row
// (lanes over the 128 head dims as float4), 8 rows per block.
__global__ void __launch_bounds__(256) tree_attn_combine(const Params p, uint16_t* __restrict__ O) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // launched with PDL: the split partials are complete
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + warp, g = blockIdx.y;
  if (r >= p.R) return;
  const int Rpad = p.qblocks * kRowsBlk;
  float mstar = -INFINITY;
  for (int sp = lane; sp < p.splits; sp += 32) mstar = fmaxf(mstar, __ldcg(&p.m_part[((size_t)sp * p.Hkv + g) * Rpad + r]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mstar = fmaxf(mstar, __shfl_xor_sync(0xffffffffu, mstar, off));
  float4 num = make_float4(0.f, 0.f, 0.f, 0.f);
  float den = 0.f;
  constexpr int kB = 9;    // splits' loads in flight at a time (one or two L2 round trips for the usual splits)
  for (int sp0 = 0; sp0 < p.splits; sp0 += kB) {
    float ms[kB], l[kB];
    float4 v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const bool in = sp0 + u < p.splits;   // no loads past the last split
      const size_t i = ((size_t)(in ? sp0 + u : 0) * p.Hkv + g) * Rpad + r;
      ms[u] = in ? __ldcg(&p.m_part[i]) : -INFINITY;
      l[u] = in ? __ldcg(&p.l_part[i]) : 0.f;
      v[u] = in ? __ldcg(reinterpret_cast<const float4*>(p.o_part + i * kD) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
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
  *reinterpret_cast<uint2*>(O + ((size_t)m * p.Hq + h) * kD + 4 * lane) = out;
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
  int s = (w4::ta::kCtasPerSmEst * sms + Hkv * *qblocks - 1) / (Hkv * *qblocks);
  const int max_s = (chunks + 1) / 2;   // at least two chunks per split where there are two (fewer partials to merge)
  s = s < 1 ? 1 : s > max_s ? max_s : s;
  *cps = (chunks + s - 1) / s;
  *splits = (chunks + *cps - 1) / *cps;
}
}  // namespace

extern "C" size_t w4a16_tree_attention_workspace_bytes_sms(int M, int L, int Hq, int Hkv, int sms) {
  int qb, sp, cps;
  plan_splits(M, L, Hq, Hkv, sms, &qb, &sp, &cps);
  const size_t rows = (size_t)sp * Hkv * qb * w4::ta::kRowsBlk;
  return rows * (w4::ta::kD + 2) * 4;
}

extern "C" int w4a16_launch_tree_attention(const uint16_t* Q, const uint16_t* K, const uint16_t* V, const int32_t* parents,
                                           int M, int L, int Hq, int Hkv, uint16_t* O, void* ws, int sms,
                                           cudaStream_t stream) {
  w4::ta::Params p;
  p.Q = Q; p.K = K; p.V = V; p.parents = parents;
  p.M = M; p.L = L; p.Hq = Hq; p.Hkv = Hkv; p.G = Hq / Hkv; p.R = M * p.G;
  plan_splits(M, L, Hq, Hkv, sms, &p.qblocks, &p.splits, &p.chunks_per_split);
  const size_t rows = (size_t)p.splits * Hkv * p.qblocks * w4::ta::kRowsBlk;
  p.o_part = reinterpret_cast<float*>(ws);
  p.m_part = p.o_part + rows * w4::ta::kD;
  p.l_part = p.m_part + rows;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)w4::ta::kD);
  static unsigned long long attr = 0;
  if (!w4::ensure_smem_attr(w4::ta::tree_attn_kernel, w4::ta::kSmem, attr)) return W4A16_ERR_CUDA;
  w4::ta::tree_attn_kernel<<<dim3(p.splits, p.qblocks, Hkv), w4::ta::kThreads, w4::ta::kSmem, stream>>>(p);
  if (cudaGetLastError() != cudaSuccess) return W4A16_ERR_CUDA;
  return w4::launch_pdl(w4::ta::tree_attn_combine, dim3((p.R + 7) / 8, Hkv), dim3(256), 0, stream, p, O) == cudaSuccess
             ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" int w4a16_launch_kv_compact(uint16_t* K, uint16_t* V, int L, int Hkv, int D, const int32_t* accept_out,
                                       cudaStream_t stream) {
  const int row_vec = Hkv * D / 8;
  w4::ta::kv_compact_kernel<<<(row_vec + 127) / 128, 128, 0, stream>>>(K, V, L, row_vec, accept_out);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}
