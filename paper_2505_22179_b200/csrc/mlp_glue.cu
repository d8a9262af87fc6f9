// mlp_glue.cu — w4a16_silu_mul: the elementwise step between the fused gate-up GEMM and the down GEMM of
// a Llama MLP in the verify forward. GU[m] = [gate_0..gate_{F-1} | up_0..up_{F-1}] (the
// rank-local gate-up shard), out[m][j] = fp16_rne(silu(gate_j) * up_j), computed in fp32.
#include "common.cuh"
#include "tma_host.cuh"
#include "w4a16.h"

namespace w4 {

__global__ void __launch_bounds__(256) silu_mul_kernel(const uint16_t* __restrict__ GU, int M, int F, int block,
                                                       uint16_t* __restrict__ out) {
  // programmatic dependent launch: the next GEMM may start streaming its weights now (it waits for this
  // grid before it reads `out`); GU comes from the previous kernel, so wait for it before reading
  pdl_launch_dependents();
  pdl_wait();
  const int vecs = F / 8;  // 8 halves per 16-byte vector
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)M * vecs;
       i += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(i / vecs), v = (int)(i % vecs);
    const int b = (v * 8) / block, o = v * 8 - b * block;   // block b, offset o inside it
    const uint16_t* row = GU + (size_t)m * 2 * F + (size_t)2 * b * block + o;
    const uint4 g = *reinterpret_cast<const uint4*>(row);
    const uint4 u = *reinterpret_cast<const uint4*>(row + block);
    *reinterpret_cast<uint4*>(out + (size_t)m * F + (size_t)v * 8) = silu_mul_vec(g, u);
  }
}

}  // namespace w4

extern "C" int w4a16_launch_silu_mul(const uint16_t* GU, int M, int F, int block, uint16_t* out, cudaStream_t stream) {
  const long long work = (long long)M * (F / 8);
  if (work == 0) return W4A16_OK;
  long long blocks = (work + 255) / 256;
  static int sms = 0;   // grid-stride loop: at most 8 blocks of 256 per SM of this device
  if (sms <= 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
  }
  if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
  return w4::launch_pdl(w4::silu_mul_kernel, dim3((unsigned)blocks), dim3(256), 0, stream, GU, M, F, block, out) == cudaSuccess
             ? W4A16_OK : W4A16_ERR_CUDA;
}
