// api.cu -- error plumbing and library identity for libdfx.
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"

namespace dfx {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

dfx_status fail(dfx_status code, const std::string& msg) {
  g_err = msg;
  return code;
}

dfx_status cuda_status(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return DFX_CUDA_ERROR;
}

}  // namespace dfx

extern "C" {

const char* dfx_last_error(void) { return dfx::g_err.c_str(); }

const char* dfx_version(void) { return "dfx 0.1 sm_100a"; }

dfx_status dfx_event_create(void** ev) {
  cudaEvent_t e;
  DFX_CUDA(cudaEventCreate(&e));
  *ev = e;
  return DFX_OK;
}

dfx_status dfx_event_destroy(void* ev) {
  DFX_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
  return DFX_OK;
}

dfx_status dfx_event_record(void* ev, dfx_stream stream) {
  DFX_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), stream));
  return DFX_OK;
}

dfx_status dfx_event_elapsed_ms(void* b, void* e, float* ms) {
  DFX_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(e)));
  DFX_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(b), static_cast<cudaEvent_t>(e)));
  return DFX_OK;
}

}  // extern "C"

// ---- peer memory (CUDA IPC over NVLink) ----------------------------------------------------------------
#include <dlfcn.h>

#include <map>
#include <mutex>

namespace {
std::mutex g_ipc_mu;
std::map<std::pair<int, std::string>, void*> g_ipc_open;  // (device, handle bytes) -> mapped base
}  // namespace

extern "C" {

dfx_status dfx_ipc_open(const void* handle, size_t handle_bytes, void** base) {
  if (!handle || handle_bytes != sizeof(cudaIpcMemHandle_t) || !base)
    return dfx::fail(DFX_INVALID_ARGUMENT, "dfx_ipc_open: bad handle");
  int dev = 0;
  DFX_CUDA(cudaGetDevice(&dev));
  const std::string key(static_cast<const char*>(handle), handle_bytes);
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc_open.find({dev, key});
  if (it != g_ipc_open.end()) {
    *base = it->second;
    return DFX_OK;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  DFX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  g_ipc_open[{dev, key}] = p;
  *base = p;
  return DFX_OK;
}

// base of the cudaMalloc allocation containing ptr: driver cuMemGetAddressRange, resolved at run time so the
// library has no link-time dependency on libcuda (it must load on CPU-only hosts)
typedef int (*GetRangeFn)(unsigned long long*, size_t*, unsigned long long);

dfx_status dfx_ipc_export(const void* ptr, void* handle_out, uint64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return dfx::fail(DFX_INVALID_ARGUMENT, "dfx_ipc_export: null argument");
  static GetRangeFn get_range = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    return h ? reinterpret_cast<GetRangeFn>(dlsym(h, "cuMemGetAddressRange_v2")) : nullptr;
  }();
  if (!get_range) return dfx::fail(DFX_CUDA_ERROR, "dfx_ipc_export: cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0)
    return dfx::fail(DFX_CUDA_ERROR, "dfx_ipc_export: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  DFX_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (uint64_t)((uintptr_t)ptr - (uintptr_t)base);
  return DFX_OK;
}

dfx_status dfx_copy_async(void* dst, const void* src, size_t bytes, dfx_stream stream) {
  if (bytes == 0) return DFX_OK;
  DFX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream));
  return DFX_OK;
}

dfx_status dfx_copy_batch(int64_t n, const uint64_t* dst, const uint64_t* src, const uint64_t* bytes,
                          dfx_stream stream) {
  for (int64_t i = 0; i < n; ++i) {
    if (bytes[i] == 0) continue;
    DFX_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(dst[i]), reinterpret_cast<const void*>(src[i]), bytes[i],
                             cudaMemcpyDefault, stream));
  }
  return DFX_OK;
}

}  // extern "C"
