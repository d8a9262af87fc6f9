// abi.cu — the C-ABI entry points of libw4a16.so (include/w4a16.h): host-side validation, planning and
// dispatch to the kernels in pack.cu, gemm_mma.cu, gemm_tc.cu and accept.cu. No device allocation, no
// host synchronisation, no global state beyond a per-device SM-count cache.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include "w4a16.h"
#include "common.cuh"

extern "C" int w4a16_launch_pack(const uint16_t*, int, int, int, void*, int32_t*, cudaStream_t);
extern "C" int w4a16_launch_unpack(const void*, int, int, int, uint16_t*, cudaStream_t);
extern "C" int w4a16_launch_accept(const int32_t*, const int32_t*, const int32_t*, int, int32_t*, cudaStream_t);
extern "C" int w4a16_launch_silu_mul(const uint16_t*, int, int, int, uint16_t*, cudaStream_t);
extern "C" size_t w4a16_mma_workspace_bytes(int M, int K, int N, int num_sms);
extern "C" size_t w4a16_tc_workspace_bytes(int M, int K, int N, int num_sms);
extern "C" int w4a16_launch_gemm_tc(const uint16_t*, int, const void*, uint16_t*, int, int, int, int, void*, int, cudaStream_t);
extern "C" size_t w4a16_tp_workspace_bytes(int M, int K, int N, int num_sms);
extern "C" int w4a16_launch_gemm_tp(const uint16_t*, int, const void*, uint16_t*, int, int, int, int, void*, int, cudaStream_t);
extern "C" size_t w4a16_lmhead_workspace_bytes_sms(int num_sms);
extern "C" int w4a16_launch_hadamard(const uint16_t*, uint16_t*, int, int, int, cudaStream_t);
extern "C" size_t w4a16_tree_attention_workspace_bytes_sms(int M, int L, int Hq, int Hkv, int sms);
extern "C" int w4a16_launch_tree_attention(const uint16_t*, const uint16_t*, const uint16_t*, const int32_t*, int, int,
                                           int, int, uint16_t*, void*, int, cudaStream_t);
extern "C" int w4a16_launch_kv_compact(uint16_t*, uint16_t*, int, int, int, const int32_t*, cudaStream_t);
extern "C" int w4a16_launch_lmhead_argmax(const uint16_t*, const uint16_t*, int, int, int, int32_t*, float*, void*, int,
                                          cudaStream_t);
extern "C" size_t w4a16_chain_workspace_bytes_sms(const w4a16_op*, int, int, int, int);
extern "C" int w4a16_chain_plan_sms(const w4a16_op*, int, int, int, void*, size_t, int);
extern "C" int w4a16_launch_chain_mma(const void*, int, int, int, int, void*, size_t, int, int, cudaStream_t);
extern "C" size_t w4a8_workspace_bytes_sms(int, int, int, int);
extern "C" int w4a8_launch_quantize(const uint16_t*, int, int, int8_t*, float*, int32_t*, cudaStream_t);
extern "C" int w4a8_launch_gemm_mma(const int8_t*, const float*, const void*, uint16_t*, int, int, int, void*, int, cudaStream_t);
extern "C" int w4a8_launch_gemm(const int8_t*, const float*, const int32_t*, const void*, uint16_t*, int, int, int, void*, int,
                                cudaStream_t);
extern "C" int w4a16_launch_gemm_mma(const uint16_t*, int, const void*, uint16_t*, int, int, int, int, bool, void*, int,
                                     cudaStream_t);

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int num_sms_of_current_device() {
  static int cache[64] = {0};   // benign race: every writer stores the same value
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return -1;
  if (dev < 64 && cache[dev] > 0) return cache[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return -1;
  if (dev < 64) cache[dev] = n;
  return n;
}

int check_kn(int K, int N, int group) {
  if (group != W4A16_GROUP) return W4A16_ERR_ARG;
  if (K <= 0 || N <= 0 || K % 128 != 0 || N % 128 != 0 || N > W4A16_MAX_N) return W4A16_ERR_SHAPE;
  return W4A16_OK;
}

}  // namespace

bool mode_ok(int mode) { return mode == W4A16_ASYM || mode == W4A16_SYM; }

extern "C" size_t w4a16_packed_bytes(int K, int N, int group, int mode) {
  if (check_kn(K, N, group) != W4A16_OK || !mode_ok(mode)) return 0;
  return (size_t)(N / 128) * (size_t)(K / 128) * (mode == W4A16_ASYM ? 8704 : 8448);
}

extern "C" int w4a16_pack(const uint16_t* W, int K, int N, int group, int mode, void* packed, int32_t* dev_status,
                          w4a16_stream_t stream) {
  if (!W || !packed || !mode_ok(mode)) return W4A16_ERR_ARG;
  if (int e = check_kn(K, N, group)) return e;
  if (!aligned16(W) || !aligned16(packed)) return W4A16_ERR_ALIGN;
  return w4a16_launch_pack(W, K, N, mode, packed, dev_status, (cudaStream_t)stream);
}

extern "C" int w4a16_unpack(const void* packed, int K, int N, int group, int mode, uint16_t* W_hat,
                            w4a16_stream_t stream) {
  if (!packed || !W_hat || !mode_ok(mode)) return W4A16_ERR_ARG;
  if (int e = check_kn(K, N, group)) return e;
  if (!aligned16(packed) || !aligned16(W_hat)) return W4A16_ERR_ALIGN;
  return w4a16_launch_unpack(packed, K, N, mode, W_hat, (cudaStream_t)stream);
}

extern "C" size_t w4a16_gemm_workspace_bytes(int M, int K, int N, int group) {
  if (check_kn(K, N, group) != W4A16_OK || M < 1 || M > W4A16_MAX_M) return 0;
  const int sms = num_sms_of_current_device();
  if (sms <= 0) return 0;
  const size_t a = w4a16_mma_workspace_bytes(M, K, N, sms), b = w4a16_tc_workspace_bytes(M, K, N, sms);
  const size_t c = w4a16_tp_workspace_bytes(M, K, N, sms);
  return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

extern "C" int w4a16_workspace_init(void* workspace, size_t workspace_bytes, w4a16_stream_t stream) {
  if (!workspace) return W4A16_ERR_ARG;
  return cudaMemsetAsync(workspace, 0, workspace_bytes, (cudaStream_t)stream) == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

// Family choice: mma.sync with exact (q - z) codes and the group scale applied to fp32 group
// sums for M <= 16, tcgen05/TMEM above (MMA cost nearly independent of M).
extern "C" int w4a16_gemm_family(int M, int K, int N) {
  (void)K; (void)N;
  if (M <= 16) return W4A16_FAMILY_MMA_SYNC;
  return W4A16_FAMILY_TCGEN05;
}

extern "C" int w4a16_gemm_strided(const uint16_t* X, int ldx, const void* packed, uint16_t* Y, int M, int K, int N,
                                  int group, int mode, void* workspace, size_t workspace_bytes, int family,
                                  w4a16_stream_t stream) {
  if (!X || !packed || !Y || !mode_ok(mode)) return W4A16_ERR_ARG;
  if (int e = check_kn(K, N, group)) return e;
  if (ldx < K || ldx % 8) return W4A16_ERR_ARG;
  if (M < 1 || M > W4A16_MAX_M) return W4A16_ERR_SHAPE;
  if (!aligned16(X) || !aligned16(packed) || !aligned16(Y) || !aligned16(workspace)) return W4A16_ERR_ALIGN;
  const int sms = num_sms_of_current_device();
  if (sms <= 0) return W4A16_ERR_CUDA;
  if (family == W4A16_FAMILY_AUTO) family = w4a16_gemm_family(M, K, N);
  if (family == W4A16_FAMILY_MMA_SYNC || family == W4A16_FAMILY_MMA_SYNC_S) {
    if (M > 16) return W4A16_ERR_SHAPE;
    if (!workspace || workspace_bytes < w4a16_mma_workspace_bytes(M, K, N, sms)) return W4A16_ERR_WORKSPACE;
    return w4a16_launch_gemm_mma(X, ldx, packed, Y, M, K, N, mode, family == W4A16_FAMILY_MMA_SYNC_S, workspace, sms,
                                 (cudaStream_t)stream);
  }
  if (family == W4A16_FAMILY_TCGEN05) {
    if (!workspace || workspace_bytes < w4a16_tc_workspace_bytes(M, K, N, sms)) return W4A16_ERR_WORKSPACE;
    return w4a16_launch_gemm_tc(X, ldx, packed, Y, M, K, N, mode, workspace, sms, (cudaStream_t)stream);
  }
  if (family == W4A16_FAMILY_TCGEN05_OC) {
    if (!workspace || workspace_bytes < w4a16_tp_workspace_bytes(M, K, N, sms)) return W4A16_ERR_WORKSPACE;
    return w4a16_launch_gemm_tp(X, ldx, packed, Y, M, K, N, mode, workspace, sms, (cudaStream_t)stream);
  }
  return W4A16_ERR_ARG;
}

extern "C" int w4a16_gemm_ex(const uint16_t* X, const void* packed, uint16_t* Y, int M, int K, int N, int group,
                             int mode, void* workspace, size_t workspace_bytes, int family, w4a16_stream_t stream) {
  return w4a16_gemm_strided(X, K, packed, Y, M, K, N, group, mode, workspace, workspace_bytes, family, stream);
}

extern "C" int w4a16_gemm(const uint16_t* X, const void* packed, uint16_t* Y, int M, int K, int N, int group, int mode,
                          void* workspace, size_t workspace_bytes, w4a16_stream_t stream) {
  return w4a16_gemm_ex(X, packed, Y, M, K, N, group, mode, workspace, workspace_bytes, W4A16_FAMILY_AUTO, stream);
}

extern "C" int verify_accept(const int32_t* tokens, const int32_t* parents, const int32_t* target_argmax, int n,
                             int32_t* out, w4a16_stream_t stream) {
  if (!tokens || !parents || !target_argmax || !out) return W4A16_ERR_ARG;
  if (n < 1 || n > W4A16_MAX_TREE) return W4A16_ERR_SHAPE;
  return w4a16_launch_accept(tokens, parents, target_argmax, n, out, (cudaStream_t)stream);
}

extern "C" int w4a16_silu_mul(const uint16_t* GU, int M, int F, uint16_t* out, w4a16_stream_t stream) {
  if (!GU || !out) return W4A16_ERR_ARG;
  if (M < 1 || F < 8 || F % 8 != 0) return W4A16_ERR_SHAPE;
  if (!aligned16(GU) || !aligned16(out)) return W4A16_ERR_ALIGN;
  return w4a16_launch_silu_mul(GU, M, F, F, out, (cudaStream_t)stream);
}

extern "C" int w4a16_silu_mul_blocked(const uint16_t* GU, int M, int F, int block, uint16_t* out, w4a16_stream_t stream) {
  if (!GU || !out) return W4A16_ERR_ARG;
  if (M < 1 || F < 8 || F % 8 != 0 || block < 8 || block % 8 != 0 || F % block != 0) return W4A16_ERR_SHAPE;
  if (!aligned16(GU) || !aligned16(out)) return W4A16_ERR_ALIGN;
  return w4a16_launch_silu_mul(GU, M, F, block, out, (cudaStream_t)stream);
}

extern "C" size_t w4a16_chain_workspace_bytes(const w4a16_op* ops, int n_ops, int M, int family) {
  const int sms = num_sms_of_current_device();
  return sms > 0 ? w4a16_chain_workspace_bytes_sms(ops, n_ops, M, family, sms) : 0;
}

extern "C" int w4a16_chain_plan(const w4a16_op* ops, int n_ops, int M, int family, void* plan, size_t plan_bytes) {
  const int sms = num_sms_of_current_device();
  if (sms <= 0) return W4A16_ERR_CUDA;
  return w4a16_chain_plan_sms(ops, n_ops, M, family, plan, plan_bytes, sms);
}

extern "C" int w4a16_chain_run(const void* dev_plan, int n_ops, int M, int mode, int family, void* workspace,
                               size_t workspace_bytes, w4a16_stream_t stream) {
  if (!dev_plan || !workspace) return W4A16_ERR_ARG;
  if (!aligned16(dev_plan) || !aligned16(workspace)) return W4A16_ERR_ALIGN;
  const int sms = num_sms_of_current_device();
  if (sms <= 0) return W4A16_ERR_CUDA;
  return w4a16_launch_chain_mma(dev_plan, n_ops, M, mode, family, workspace, workspace_bytes, sms, 1, (cudaStream_t)stream);
}

// Test hook (not part of include/w4a16.h): a chain planned with w4a16_chain_plan_sms for `sms` SMs, launched
// without the cooperative attribute so that several such chains can share one device side by side
// (tests/test_gpu_allreduce.py simulates tensor-parallel ranks that way on a single GPU).
extern "C" int w4a16_chain_run_sms(const void* dev_plan, int n_ops, int M, int mode, int family, void* workspace,
                                   size_t workspace_bytes, int sms, w4a16_stream_t stream) {
  if (!dev_plan || !workspace) return W4A16_ERR_ARG;
  if (!aligned16(dev_plan) || !aligned16(workspace)) return W4A16_ERR_ALIGN;
  const int dev_sms = num_sms_of_current_device();
  if (dev_sms <= 0) return W4A16_ERR_CUDA;
  if (sms < 1 || sms > dev_sms) return W4A16_ERR_ARG;
  return w4a16_launch_chain_mma(dev_plan, n_ops, M, mode, family, workspace, workspace_bytes, sms, 0, (cudaStream_t)stream);
}

// ---- symmetric regions (CUDA IPC) ----
extern "C" int w4a16_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out || bytes == 0) return W4A16_ERR_ARG;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return W4A16_ERR_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess || cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
    cudaFree(p);
    return W4A16_ERR_CUDA;
  }
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  *dev_ptr = p;
  return W4A16_OK;
}

extern "C" int w4a16_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return W4A16_ERR_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" int w4a16_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return W4A16_ERR_ARG;
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" int w4a16_ipc_free(void* dev_ptr) {
  if (!dev_ptr) return W4A16_ERR_ARG;
  return cudaFree(dev_ptr) == cudaSuccess ? W4A16_OK : W4A16_ERR_CUDA;
}

// ---- symmetric regions bound to a multicast object (NVLS) ----
// Driver entry points resolved at run time (cudaGetDriverEntryPoint), so the library never links libcuda.
namespace {
struct McApi {
  bool ok = false;
  CUresult (*create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  CUresult (*granularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
  CUresult (*add_device)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*bind_mem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t, unsigned long long);
  CUresult (*unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*export_handle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
  CUresult (*import_handle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*mem_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*mem_release)(CUmemGenericAllocationHandle);
  CUresult (*alloc_granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*addr_free)(CUdeviceptr, size_t);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*attr)(int*, CUdevice_attribute, CUdevice);
};
template <class F>
bool entry(const char* name, F& f) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) return false;
  f = reinterpret_cast<F>(p);
  return true;
}
const McApi& mc_api() {
  static McApi a = [] {
    McApi m;
    m.ok = entry("cuMulticastCreate", m.create) && entry("cuMulticastGetGranularity", m.granularity) &&
           entry("cuMulticastAddDevice", m.add_device) && entry("cuMulticastBindMem", m.bind_mem) &&
           entry("cuMulticastUnbind", m.unbind) && entry("cuMemExportToShareableHandle", m.export_handle) &&
           entry("cuMemImportFromShareableHandle", m.import_handle) && entry("cuMemCreate", m.mem_create) &&
           entry("cuMemRelease", m.mem_release) && entry("cuMemGetAllocationGranularity", m.alloc_granularity) &&
           entry("cuMemAddressReserve", m.reserve) && entry("cuMemAddressFree", m.addr_free) && entry("cuMemMap", m.map) &&
           entry("cuMemUnmap", m.unmap) && entry("cuMemSetAccess", m.set_access) && entry("cuDeviceGetAttribute", m.attr);
    return m;
  }();
  return a;
}
// Diagnostics: the last failing driver call of the w4a16_mc_* functions (printed when W4A16_MC_DEBUG is set).
CUresult g_mc_err = CUDA_SUCCESS;
const char* g_mc_where = "";
bool mc_ok(CUresult r, const char* where) {
  if (r == CUDA_SUCCESS) return true;
  g_mc_err = r;
  g_mc_where = where;
  if (getenv("W4A16_MC_DEBUG")) fprintf(stderr, "w4a16_mc: %s failed: CUresult %d\n", where, (int)r);
  return false;
}
// Size of a multicast object for `bytes` and `world` devices: the same on every rank (same query).
int mc_size(const McApi& a, size_t bytes, int world, size_t* size) {
  CUmulticastObjectProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.numDevices = (unsigned)world;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
  size_t gran = 0;
  if (!mc_ok(a.granularity(&gran, &prop, CU_MULTICAST_GRANULARITY_MINIMUM), "granularity") || gran == 0) return W4A16_ERR_CUDA;
  *size = (bytes + gran - 1) / gran * gran;
  return W4A16_OK;
}
struct McObject {
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  size_t size = 0;
  int world = 0;
  CUdevice dev = 0;
  bool bound = false;
};
int current_device(CUdevice* d) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return W4A16_ERR_CUDA;
  *d = (CUdevice)dev;
  return W4A16_OK;
}
}  // namespace

// Test hook (exported, not in the header): the last failing driver call of the w4a16_mc_* functions.
extern "C" int w4a16_mc_last_error(const char** where) {
  if (where) *where = g_mc_where;
  return (int)g_mc_err;
}

extern "C" int w4a16_mc_supported(void) {
  const McApi& a = mc_api();
  CUdevice d;
  if (!a.ok || current_device(&d) != W4A16_OK) return 0;
  cudaFree(nullptr);   // make sure the primary context exists
  int mc = 0, fabric = 0;
  if (!mc_ok(a.attr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d), "attr")) return 0;
  if (!mc_ok(a.attr(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d), "attr")) return 0;
  return mc && fabric ? 1 : 0;
}

extern "C" int w4a16_mc_create(size_t bytes, int world, void* handle_out, void** mc_out) {
  const McApi& a = mc_api();
  if (!handle_out || !mc_out || bytes == 0 || world < 1 || world > W4A16_MAX_PEERS) return W4A16_ERR_ARG;
  if (!a.ok) return W4A16_ERR_CUDA;
  CUmulticastObjectProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.numDevices = (unsigned)world;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
  if (mc_size(a, bytes, world, &prop.size) != W4A16_OK) return W4A16_ERR_CUDA;
  McObject* o = new McObject;
  o->size = prop.size;
  o->world = world;
  CUmemFabricHandle fh;
  if (!mc_ok(a.create(&o->mc, &prop), "create")) { delete o; return W4A16_ERR_CUDA; }
  if (!mc_ok(a.export_handle(&fh, o->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0), "export_handle")) {
    a.mem_release(o->mc);
    delete o;
    return W4A16_ERR_CUDA;
  }
  static_assert(sizeof(fh) == 64, "fabric handle size");
  memcpy(handle_out, &fh, sizeof(fh));
  *mc_out = o;
  return W4A16_OK;
}

extern "C" int w4a16_mc_import(const void* handle, size_t bytes, int world, void** mc_out) {
  const McApi& a = mc_api();
  if (!handle || !mc_out || bytes == 0 || world < 1 || world > W4A16_MAX_PEERS) return W4A16_ERR_ARG;
  if (!a.ok) return W4A16_ERR_CUDA;
  CUmemFabricHandle fh;
  memcpy(&fh, handle, sizeof(fh));
  McObject* o = new McObject;
  o->world = world;
  if (mc_size(a, bytes, world, &o->size) != W4A16_OK) { delete o; return W4A16_ERR_CUDA; }
  if (!mc_ok(a.import_handle(&o->mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC), "import_handle")) { delete o; return W4A16_ERR_CUDA; }
  *mc_out = o;
  return W4A16_OK;
}

extern "C" int w4a16_mc_add_device(void* mc) {
  const McApi& a = mc_api();
  McObject* o = reinterpret_cast<McObject*>(mc);
  if (!o) return W4A16_ERR_ARG;
  if (!a.ok || current_device(&o->dev) != W4A16_OK) return W4A16_ERR_CUDA;
  cudaFree(nullptr);
  return mc_ok(a.add_device(o->mc, o->dev), "add_device") ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" int w4a16_mc_bind(void* mc, size_t bytes, void** uc_out, void** mc_va_out) {
  const McApi& a = mc_api();
  McObject* o = reinterpret_cast<McObject*>(mc);
  if (!o || !uc_out || !mc_va_out || bytes == 0) return W4A16_ERR_ARG;
  if (!a.ok) return W4A16_ERR_CUDA;
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = (int)o->dev;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
  size_t gran = 0;
  if (!mc_ok(a.alloc_granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "alloc_granularity") || gran == 0) return W4A16_ERR_CUDA;
  size_t size = (bytes + gran - 1) / gran * gran;
  size = o->size > size ? o->size : size;
  if (size % gran) size = (size + gran - 1) / gran * gran;
  CUdeviceptr uc = 0, mva = 0;
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = (int)o->dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  int err = W4A16_ERR_CUDA;
  if (!mc_ok(a.mem_create(&o->mem, size, &prop, 0), "mem_create")) return W4A16_ERR_CUDA;
  if (mc_ok(a.reserve(&uc, size, gran, 0, 0), "reserve")) {
    if (mc_ok(a.map(uc, size, 0, o->mem, 0), "map") && mc_ok(a.set_access(uc, size, &acc, 1), "set_access") &&
        cudaMemset(reinterpret_cast<void*>(uc), 0, size) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess &&
        mc_ok(a.bind_mem(o->mc, 0, o->mem, 0, o->size, 0), "bind_mem")) {
      o->bound = true;
      if (mc_ok(a.reserve(&mva, o->size, gran, 0, 0), "reserve")) {
        if (mc_ok(a.map(mva, o->size, 0, o->mc, 0), "map") && mc_ok(a.set_access(mva, o->size, &acc, 1), "set_access")) {
          err = W4A16_OK;
        } else {
          a.unmap(mva, o->size);
          a.addr_free(mva, o->size);
          mva = 0;
        }
      }
    }
    if (err != W4A16_OK) {
      if (o->bound) a.unbind(o->mc, o->dev, 0, o->size);
      o->bound = false;
      a.unmap(uc, size);
      a.addr_free(uc, size);
    }
  }
  if (err != W4A16_OK) {
    a.mem_release(o->mem);
    o->mem = 0;
    return err;
  }
  *uc_out = reinterpret_cast<void*>(uc);
  *mc_va_out = reinterpret_cast<void*>(mva);
  return W4A16_OK;
}

extern "C" int w4a16_mc_free(void* mc, void* uc, void* mc_va, size_t bytes) {
  const McApi& a = mc_api();
  McObject* o = reinterpret_cast<McObject*>(mc);
  if (!o) return W4A16_ERR_ARG;
  if (!a.ok) return W4A16_ERR_CUDA;
  cudaDeviceSynchronize();
  bool ok = true;
  if (mc_va) ok &= mc_ok(a.unmap((CUdeviceptr)mc_va, o->size), "unmap") && mc_ok(a.addr_free((CUdeviceptr)mc_va, o->size), "addr_free");
  if (o->bound) ok &= mc_ok(a.unbind(o->mc, o->dev, 0, o->size), "unbind");
  if (uc) {
    CUmemAllocationProp prop;
    memset(&prop, 0, sizeof(prop));
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = (int)o->dev;
    size_t gran = 1;
    a.alloc_granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    size_t size = (bytes + gran - 1) / gran * gran;
    size = o->size > size ? o->size : size;
    ok &= mc_ok(a.unmap((CUdeviceptr)uc, size), "unmap") && mc_ok(a.addr_free((CUdeviceptr)uc, size), "addr_free");
  }
  if (o->mem) ok &= mc_ok(a.mem_release(o->mem), "mem_release");
  ok &= mc_ok(a.mem_release(o->mc), "mem_release");
  delete o;
  return ok ? W4A16_OK : W4A16_ERR_CUDA;
}

extern "C" size_t w4a16_lmhead_workspace_bytes(int M, int K, int V) {
  if (M < 1 || M > W4A16_MAX_M || K <= 0 || K % 128 || V <= 0 || V % 128) return 0;
  const int sms = num_sms_of_current_device();
  return sms > 0 ? w4a16_lmhead_workspace_bytes_sms(sms) : 0;
}

extern "C" int w4a16_lmhead_argmax(const uint16_t* H, const uint16_t* W_lm, int M, int K, int V, int32_t* out_argmax,
                                   float* out_max, void* workspace, size_t workspace_bytes, w4a16_stream_t stream) {
  if (!H || !W_lm || !out_argmax || !workspace) return W4A16_ERR_ARG;
  if (M < 1 || M > W4A16_MAX_M || K <= 0 || K % 128 || V <= 0 || V % 128) return W4A16_ERR_SHAPE;
  if (!aligned16(H) || !aligned16(W_lm) || !aligned16(workspace) || (reinterpret_cast<uintptr_t>(out_argmax) & 3) ||
      (reinterpret_cast<uintptr_t>(out_max) & 3))
    return W4A16_ERR_ALIGN;
  const int sms = num_sms_of_current_device();
  if (sms <= 0) return W4A16_ERR_CUDA;
  if (workspace_bytes < w4a16_lmhead_workspace_bytes_sms(sms)) return W4A16_ERR_WORKSPACE;
  return w4a16_launch_lmhead_argmax(H, W_lm, M, K, V, out_argmax, out_max, workspace, sms, (cudaStream_t)stream);
}

namespace {
int check_attn(int M, int L, int Hq, int Hkv, int D) {
  if (M < 1 || M > W4A16_MAX_M || L < 0 || Hq < 1 || Hq > 512 || Hkv < 1 || Hq % Hkv || D != 128) return W4A16_ERR_SHAPE;
  return W4A16_OK;
}
}  // namespace

extern "C" size_t w4a16_tree_attention_workspace_bytes(int M, int L, int Hq, int Hkv, int D) {
  if (check_attn(M, L, Hq, Hkv, D) != W4A16_OK) return 0;
  const int sms = num_sms_of_current_device();
  return sms > 0 ? w4a16_tree_attention_workspace_bytes_sms(M, L, Hq, Hkv, sms) : 0;
}

extern "C" int w4a16_tree_attention(const uint16_t* Q, const uint16_t* Kc, const uint16_t* Vc, const int32_t* parents,
                                    int M, int L, int Hq, int Hkv, int D, uint16_t* O, void* workspace,
                                    size_t workspace_bytes, w4a16_stream_t stream) {
  if (!Q || !Kc || !Vc || !parents || !O || !workspace) return W4A16_ERR_ARG;
  if (int e = check_attn(M, L, Hq, Hkv, D)) return e;
  if (!aligned16(Q) || !aligned16(Kc) || !aligned16(Vc) || !aligned16(O) || !aligned16(workspace) ||
      (reinterpret_cast<uintptr_t>(parents) & 3))
    return W4A16_ERR_ALIGN;
  const int sms = num_sms_of_current_device();
  if (sms <= 0) return W4A16_ERR_CUDA;
  if (workspace_bytes < w4a16_tree_attention_workspace_bytes_sms(M, L, Hq, Hkv, sms)) return W4A16_ERR_WORKSPACE;
  return w4a16_launch_tree_attention(Q, Kc, Vc, parents, M, L, Hq, Hkv, O, workspace, sms, (cudaStream_t)stream);
}

extern "C" int w4a16_kv_compact(uint16_t* Kc, uint16_t* Vc, int L, int Hkv, int D, const int32_t* accept_out,
                                w4a16_stream_t stream) {
  if (!Kc || !Vc || !accept_out) return W4A16_ERR_ARG;
  if (L < 0 || Hkv < 1 || D < 8 || D % 8) return W4A16_ERR_SHAPE;
  if (!aligned16(Kc) || !aligned16(Vc) || (reinterpret_cast<uintptr_t>(accept_out) & 3)) return W4A16_ERR_ALIGN;
  return w4a16_launch_kv_compact(Kc, Vc, L, Hkv, D, accept_out, (cudaStream_t)stream);
}

extern "C" int w4a16_hadamard(const uint16_t* X, uint16_t* Y, int M, int K, int block, w4a16_stream_t stream) {
  if (!X || !Y) return W4A16_ERR_ARG;
  if (M < 1 || block < 64 || block > 1024 || (block & (block - 1)) || K < block || K % block) return W4A16_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(X) & 3) || (reinterpret_cast<uintptr_t>(Y) & 3)) return W4A16_ERR_ALIGN;
  return w4a16_launch_hadamard(X, Y, M, K, block, (cudaStream_t)stream);
}

extern "C" const char* w4a16_status_string(int status) {
  switch (status) {
    case W4A16_OK: return "W4A16_OK";
    case W4A16_ERR_ARG: return "W4A16_ERR_ARG: invalid argument";
    case W4A16_ERR_SHAPE: return "W4A16_ERR_SHAPE: unsupported shape";
    case W4A16_ERR_ALIGN: return "W4A16_ERR_ALIGN: pointer not 16-byte aligned";
    case W4A16_ERR_WORKSPACE: return "W4A16_ERR_WORKSPACE: workspace missing or too small";
    case W4A16_ERR_CUDA: return "W4A16_ERR_CUDA: CUDA launch or query failed";
    default: return "unknown w4a16 status";
  }
}

// ---- W4A8 (f4) ----
extern "C" int w4a8_quantize_act(const uint16_t* X, int M, int K, int8_t* Xq, float* sx, int32_t* xsum, w4a16_stream_t stream) {
  if (!X || !Xq || !sx || !xsum) return W4A16_ERR_ARG;
  if (M < 1 || M > W4A16_MAX_M || K < 128 || K % 128) return W4A16_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(Xq) & 15u) || (reinterpret_cast<uintptr_t>(X) & 1u) || (reinterpret_cast<uintptr_t>(sx) & 3u) ||
      (reinterpret_cast<uintptr_t>(xsum) & 3u))
    return W4A16_ERR_ALIGN;
  return w4a8_launch_quantize(X, M, K, Xq, sx, xsum, (cudaStream_t)stream);
}

extern "C" size_t w4a8_workspace_bytes(int M, int K, int N) {
  if (M < 1 || M > W4A16_MAX_M || K < 128 || K % 128 || N < 128 || N % 128 || N > W4A16_MAX_N) return 0;
  const int sms = num_sms_of_current_device();
  if (sms <= 0) return 0;
  // the k-split kernel's partials start after the family-A tile counters, so one workspace serves both paths
  const size_t a = w4::kCounterBytes + w4a8_workspace_bytes_sms(M, K, N, sms), b = M <= 16 ? w4a16_mma_workspace_bytes(M, K, N, sms) : 0;
  return a > b ? a : b;
}

namespace {
// impl: 0 = auto (the family-A pipeline for M <= 16, the round-1 INT8 kernel above), 1 = family-A pipeline,
// 2 = round-1 kernel
int w4a8_gemm_impl(const int8_t* Xq, const float* sx, const int32_t* xsum, const void* packed, uint16_t* Y, int M, int K,
                   int N, void* workspace, size_t workspace_bytes, int impl, cudaStream_t stream) {
  if (!Xq || !sx || !xsum || !packed || !Y || !workspace) return W4A16_ERR_ARG;
  if (M < 1 || M > W4A16_MAX_M || K < 128 || K % 128 || N < 128 || N % 128 || N > W4A16_MAX_N) return W4A16_ERR_SHAPE;
  // the GEMMs stream Xq and the blob with 16-byte copies: a smaller alignment would fault on the device
  if ((reinterpret_cast<uintptr_t>(Xq) & 15u) || (reinterpret_cast<uintptr_t>(packed) & 15u) || (reinterpret_cast<uintptr_t>(Y) & 1u) ||
      (reinterpret_cast<uintptr_t>(workspace) & 15u) || (reinterpret_cast<uintptr_t>(sx) & 3u) ||
      (reinterpret_cast<uintptr_t>(xsum) & 3u))
    return W4A16_ERR_ALIGN;
  const int sms = num_sms_of_current_device();
  if (sms <= 0) return W4A16_ERR_CUDA;
  if (impl == 0) impl = M <= 16 ? 1 : 2;
  if (impl == 1) {
    if (M > 16) return W4A16_ERR_SHAPE;
    if (workspace_bytes < w4a16_mma_workspace_bytes(M, K, N, sms)) return W4A16_ERR_WORKSPACE;
    return w4a8_launch_gemm_mma(Xq, sx, packed, Y, M, K, N, workspace, sms, stream);
  }
  if (workspace_bytes < w4::kCounterBytes + w4a8_workspace_bytes_sms(M, K, N, sms)) return W4A16_ERR_WORKSPACE;
  return w4a8_launch_gemm(Xq, sx, xsum, packed, Y, M, K, N, reinterpret_cast<uint8_t*>(workspace) + w4::kCounterBytes, sms,
                          stream);
}
}  // namespace

extern "C" int w4a8_gemm(const int8_t* Xq, const float* sx, const int32_t* xsum, const void* packed, uint16_t* Y, int M, int K, int N,
                         void* workspace, size_t workspace_bytes, w4a16_stream_t stream) {
  return w4a8_gemm_impl(Xq, sx, xsum, packed, Y, M, K, N, workspace, workspace_bytes, 0, (cudaStream_t)stream);
}

// Test hook (exported, not in the header): w4a8_gemm with an explicit implementation (see w4a8_gemm_impl).
extern "C" int w4a8_gemm_ex(const int8_t* Xq, const float* sx, const int32_t* xsum, const void* packed, uint16_t* Y, int M, int K,
                            int N, void* workspace, size_t workspace_bytes, int impl, w4a16_stream_t stream) {
  return w4a8_gemm_impl(Xq, sx, xsum, packed, Y, M, K, N, workspace, workspace_bytes, impl, (cudaStream_t)stream);
}
