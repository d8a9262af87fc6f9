// accept.cu — verify_accept kernel (greedy acceptance, reading R9).
//
// One CTA, one thread per tree node (n <= 1024). Node i is accepted-reachable ("ok") when every edge on
// its root path matches the target's argmax at the parent; the result is the deepest ok
// node, ties to the smallest index. Depth and ok are computed for all nodes at once by pointer jumping
// (ceil(log2 n) rounds); the jump tables double as a binary-lifting table, so each node decides in
// O(log n) whether it lies on the accepted path and writes its own slot of the path. No host sync.
#include "common.cuh"
#include "w4a16.h"

namespace w4 {

constexpr int kMaxLevels = 10;  // 2^10 = W4A16_MAX_TREE

__global__ void __launch_bounds__(1024) accept_kernel(const int32_t* __restrict__ tokens,
                                                      const int32_t* __restrict__ parents,
                                                      const int32_t* __restrict__ target_argmax, int n,
                                                      int32_t* __restrict__ out) {
  __shared__ int16_t s_lev[kMaxLevels + 1][W4A16_MAX_TREE];  // s_lev[l][i] = 2^l-th ancestor (root -> root)
  __shared__ int16_t s_up[W4A16_MAX_TREE];
  __shared__ int16_t s_dist[W4A16_MAX_TREE];
  __shared__ uint8_t s_good[W4A16_MAX_TREE];
  __shared__ int s_warp_best[32];
  __shared__ int s_best;

  const int i = threadIdx.x;
  const bool valid = i < n;
  int p = -1, bad = 0;
  if (valid) {
    p = parents[i];
    bad = (i == 0) ? (p != -1) : (p < 0 || p >= i);
  }
  if (__syncthreads_or(bad)) {
    if (i == 0) { out[0] = 0; out[1] = -1; out[2] = W4A16_DEV_BAD_TREE; }
    if (valid) out[3 + i] = -1;
    return;
  }
  if (valid) {
    s_up[i] = (int16_t)(i == 0 ? 0 : p);
    s_dist[i] = (int16_t)(i == 0 ? 0 : 1);
    s_good[i] = (uint8_t)(i == 0 ? 1 : (tokens[i] == target_argmax[p]));
  }
  __syncthreads();
  int levels = 0;
  while ((1 << levels) < n) ++levels;
  for (int l = 0; l < levels; ++l) {
    int up = 0, dist = 0, good = 0;
    if (valid) {
      const int u = s_up[i];
      s_lev[l][i] = (int16_t)u;
      good = s_good[i] & s_good[u];
      dist = s_dist[i] + s_dist[u];
      up = s_up[u];
    }
    __syncthreads();
    if (valid) { s_up[i] = (int16_t)up; s_dist[i] = (int16_t)dist; s_good[i] = (uint8_t)good; }
    __syncthreads();
  }
  // After the rounds every jump pointer reached the root: s_dist = depth, s_good = ok.
  const int depth = valid ? s_dist[i] : 0;
  const int key = (valid && s_good[i]) ? (depth << 11) | (2047 - i) : -1;  // max depth, then min index
  int best = key;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((i & 31) == 0) s_warp_best[i >> 5] = best;
  __syncthreads();
  if (i < 32) {
    int b = (i < (int)((blockDim.x + 31) >> 5)) ? s_warp_best[i] : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    if (i == 0) s_best = b;
  }
  __syncthreads();
  const int bkey = s_best;  // root is always ok, so bkey >= 0
  const int bnode = 2047 - (bkey & 2047), blen = bkey >> 11;
  if (i == 0) { out[0] = blen; out[1] = target_argmax[bnode]; out[2] = W4A16_DEV_OK; }
  if (valid) {
    if (i >= blen) out[3 + i] = -1;  // padding slots [blen, n)
    if (i != 0 && depth <= blen) {
      // lift bnode by (blen - depth) levels; i is on the path iff it lands on i
      int x = bnode, d = blen - depth;
      for (int l = 0; d; ++l, d >>= 1)
        if (d & 1) x = s_lev[l][x];
      if (x == i) out[3 + depth - 1] = i;
    }
  }
}

}  // namespace w4

extern "C" int w4a16_launch_accept(const int32_t* tokens, const int32_t* parents, const int32_t* target_argmax, int n,
                                   int32_t* out, cudaStream_t stream) {
  const int threads = ((n + 31) / 32) * 32;
  w4::accept_kernel<<<1, threads, 0, stream>>>(tokens, parents, target_argmax, n, out);
  return cudaGetLastError() == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}
