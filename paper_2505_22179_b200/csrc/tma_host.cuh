// tma_host.cuh — host-side TMA tensor-map encoding shared by the GEMM kernels (driver entry point, no libcuda link).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "w4a16.h"

namespace w4 {

inline PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

// X [M][K] fp16 viewed as 3-D (64 k-in-box, M rows, K/64 boxes) with box (64, mpad, depth) and 128B swizzle:
// one TMA lands `depth` consecutive 64-k boxes as [box][row][128 B] = back-to-back K-major SW128 atoms
// (16-byte chunk j of row m stored at chunk position j ^ (m % 8)); rows >= M are zero-filled.
// ldx: row stride of X in elements (0 = K; else >= K and a multiple of 8 so rows stay 16-byte aligned).
inline int encode_x_sw128(CUtensorMap* map, const uint16_t* X, int M, int K, int mpad, int depth, int ldx = 0) {
  auto enc = get_encode();
  if (!enc) return W4A16_ERR_CUDA;
  const cuuint64_t dims[3] = {64, (cuuint64_t)M, (cuuint64_t)(K / 64)};
  const cuuint64_t strides[2] = {(cuuint64_t)(ldx > 0 ? ldx : K) * 2, 128};
  const cuuint32_t box[3] = {64, (cuuint32_t)mpad, (cuuint32_t)depth};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<uint16_t*>(X), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return W4A16_ERR_CUDA;
  return W4A16_OK;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is per device,
// so a process driving several GPUs must set it on each (the flag word is per template instance).
template <typename Kern>
inline bool ensure_smem_attr(Kern kern, int bytes, unsigned long long& done_mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  const unsigned long long bit = 1ull << dev;
  if (__atomic_load_n(&done_mask, __ATOMIC_ACQUIRE) & bit) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  __atomic_fetch_or(&done_mask, bit, __ATOMIC_RELEASE);
  return true;
}

// Launch with programmatic stream serialization: the kernel may begin while the previous kernel in the
// stream drains; it must call griddepcontrol.wait before touching anything that kernel writes.
template <typename Kern, typename... Args>
inline cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace w4
