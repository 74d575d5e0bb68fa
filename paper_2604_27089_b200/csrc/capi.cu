// C ABI plumbing of libautosp.so: error text, device info, symmetric (IPC-mapped)
// memory.  The compute entry points live next to their kernels (a2a.cu, attn_*.cu).
#include <cstdarg>
#include <cstdio>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/autosp.h"

static thread_local char g_err[512] = "";

extern "C" void autosp_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int cuda_fail(cudaError_t e, const char* what) {
  autosp_set_error("%s: %s", what, cudaGetErrorString(e));
  return AUTOSP_ERR_CUDA;
}

extern "C" int autosp_abi_version(void) { return AUTOSP_ABI_VERSION; }
extern "C" const char* autosp_last_error(void) { return g_err; }

extern "C" int autosp_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return -1; }
  int sms = 0, ma = 0, mi = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, dev);
  if (sm_count) *sm_count = sms;
  if (cc_major) *cc_major = ma;
  if (cc_minor) *cc_minor = mi;
  return 0;
}

extern "C" int autosp_symm_alloc(size_t bytes, void** dev_ptr, void* ipc_handle_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == AUTOSP_IPC_HANDLE_BYTES, "ipc handle size");
  if (!dev_ptr || bytes == 0) {
    autosp_set_error("symm_alloc: bad arguments");
    return AUTOSP_ERR_VALIDATION;
  }
  cudaError_t e = cudaMalloc(dev_ptr, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "symm_alloc cudaMalloc");
  e = cudaMemset(*dev_ptr, 0, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "symm_alloc cudaMemset");
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, *dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    memcpy(ipc_handle_out, &h, sizeof(h));
  }
  return AUTOSP_OK;
}

extern "C" int autosp_symm_open(const void* ipc_handle, void** dev_ptr) {
  if (!ipc_handle || !dev_ptr) {
    autosp_set_error("symm_open: bad arguments");
    return AUTOSP_ERR_VALIDATION;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  return AUTOSP_OK;
}

extern "C" int autosp_symm_close(void* peer_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(peer_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return AUTOSP_OK;
}

extern "C" int autosp_symm_free(void* dev_ptr) {
  cudaError_t e = cudaFree(dev_ptr);
  if (e != cudaSuccess) return cuda_fail(e, "symm_free cudaFree");
  return AUTOSP_OK;
}

extern "C" int autosp_memset_async(void* dev_ptr, int value, size_t bytes, void* stream) {
  cudaError_t e = cudaMemsetAsync(dev_ptr, value, bytes, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "memset_async");
  return AUTOSP_OK;
}

// Minimal DLPack (v0.8) ABI: what torch.utils.dlpack.from_dlpack reads from a "dltensor"
// capsule.  The struct and its shape live in one C allocation freed by the C deleter.
namespace {
struct DLDevice { int device_type; int device_id; };
struct DLDataType { uint8_t code; uint8_t bits; uint16_t lanes; };
struct DLTensor {
  void* data; DLDevice device; int ndim; DLDataType dtype;
  int64_t* shape; int64_t* strides; uint64_t byte_offset;
};
struct DLManagedTensor {
  DLTensor dl_tensor; void* manager_ctx; void (*deleter)(DLManagedTensor*);
};
struct Wrapped { DLManagedTensor mt; int64_t shape[1]; };
void wrapped_deleter(DLManagedTensor* mt) { delete reinterpret_cast<Wrapped*>(mt); }
}  // namespace

extern "C" void* autosp_dlpack_wrap(void* ptr, int64_t nbytes, int device_type, int device_id) {
  if (!ptr || nbytes < 0) {
    autosp_set_error("dlpack_wrap: bad arguments");
    return nullptr;
  }
  Wrapped* w = new Wrapped{};
  w->shape[0] = nbytes;
  w->mt.dl_tensor.data = ptr;
  w->mt.dl_tensor.device = DLDevice{device_type, device_id};
  w->mt.dl_tensor.ndim = 1;
  w->mt.dl_tensor.dtype = DLDataType{1, 8, 1};  // kDLUInt, 8 bits
  w->mt.dl_tensor.shape = w->shape;
  w->mt.dl_tensor.strides = nullptr;
  w->mt.dl_tensor.byte_offset = 0;
  w->mt.manager_ctx = nullptr;
  w->mt.deleter = wrapped_deleter;
  static_assert(offsetof(Wrapped, mt) == 0, "DLManagedTensor first");
  return &w->mt;
}

int autosp_preload_a2a();
int autosp_preload_fwd();
int autosp_preload_bwd();
int autosp_preload_fused();
int autosp_preload_gemm();

extern "C" int autosp_preload_kernels(void) {
  int rc = autosp_preload_a2a() | autosp_preload_fwd() | autosp_preload_bwd() |
           autosp_preload_fused() | autosp_preload_gemm();
  if (rc) {
    autosp_set_error("preloading kernels failed: %s", cudaGetErrorString(cudaGetLastError()));
    return AUTOSP_ERR_CUDA;
  }
  return AUTOSP_OK;
}
