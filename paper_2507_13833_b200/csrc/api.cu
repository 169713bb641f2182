#include <algorithm>
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
// (device, handle bytes) -> mapped base + reference count. Every dfx_ipc_open takes a reference, dfx_ipc_close
// drops one and unmaps at zero, so a long run with changing producer allocations does not accumulate mappings
// (which would pin the producers' freed segments and leak the consumer's address space).
struct IpcMap {
  void* base;
  int64_t refs;
};
std::mutex g_ipc_mu;
std::map<std::pair<int, std::string>, IpcMap> g_ipc_open;
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
    ++it->second.refs;
    *base = it->second.base;
    return DFX_OK;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  DFX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  g_ipc_open[{dev, key}] = IpcMap{p, 1};
  *base = p;
  return DFX_OK;
}

dfx_status dfx_ipc_close(void* base) {
  int dev = 0;
  DFX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (auto it = g_ipc_open.begin(); it != g_ipc_open.end(); ++it) {
    if (it->first.first != dev || it->second.base != base) continue;
    if (--it->second.refs > 0) return DFX_OK;
    g_ipc_open.erase(it);
    DFX_CUDA(cudaIpcCloseMemHandle(base));
    return DFX_OK;
  }
  return dfx::fail(DFX_INVALID_ARGUMENT, "dfx_ipc_close: not a mapping opened by dfx_ipc_open on this device");
}

int64_t dfx_ipc_open_count(void) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  return (int64_t)g_ipc_open.size();
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

}  // extern "C"

namespace {
// Same-device copy on the SMs (HBM -> HBM at ~3 TB/s; a copy-engine D2D copy runs at ~0.5 TB/s): 16-byte
// vectors when both ends are 16-byte aligned, else 4-byte words, else bytes.
__global__ void __launch_bounds__(256) copy_sm_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                                      uint64_t n, int width) {
  const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (uint64_t)gridDim.x * blockDim.x;
  if (width == 16) {
    for (uint64_t i = i0; i < n / 16; i += step)
      reinterpret_cast<uint4*>(dst)[i] = __ldcs(reinterpret_cast<const uint4*>(src) + i);
    for (uint64_t i = (n / 16) * 16 + i0; i < n; i += step) dst[i] = src[i];
  } else if (width == 4) {
    for (uint64_t i = i0; i < n / 4; i += step) reinterpret_cast<uint32_t*>(dst)[i] = __ldcs(reinterpret_cast<const uint32_t*>(src) + i);
    for (uint64_t i = (n / 4) * 4 + i0; i < n; i += step) dst[i] = src[i];
  } else {  // different 16-byte phases: 16-byte stores assembled from the aligned source vectors
    dfx::copy_shift16<false>(dst, src, n, (uint32_t)i0, (uint32_t)step);
  }
}
// record metadata of a view of records [r0, r1): group_off rebased to its first rollout, roll_group to r0
__global__ void __launch_bounds__(256) view_meta_kernel(const int32_t* __restrict__ go, const int32_t* __restrict__ rg,
                                                        int64_t r0, int64_t r1, int32_t* __restrict__ go_out,
                                                        int32_t* __restrict__ rg_out) {
  const int32_t s0 = go[r0], s1 = go[r1];
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0; i <= r1 - r0; i += step) go_out[i] = go[r0 + i] - s0;
  for (int64_t j = i0; j < s1 - s0; j += step) rg_out[j] = rg[s0 + j] - (int32_t)r0;
}
// Many copies in one launch (sources in this GPU's HBM or mapped from a peer over NVLink): every copy is cut into
// 64 KB chunks, block b copies chunk b (found by a search over the per-copy chunk prefix), 16-byte vectors when
// both ends are aligned. Local and remote copies run concurrently on the SMs instead of serially on one copy
// engine queue, with no per-copy launch cost.
constexpr int kCopyMany = 96;
constexpr uint64_t kCopyChunk = 65536;
struct CopyMany {
  int n;
  uint64_t dst[kCopyMany], src[kCopyMany], bytes[kCopyMany], chunk0[kCopyMany + 1];
};
__global__ void __launch_bounds__(256) copy_many_kernel(CopyMany c) {
  const uint64_t ch = blockIdx.x;
  int lo = 0, hi = c.n;  // last copy with chunk0 <= ch
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (c.chunk0[mid] <= ch) lo = mid;
    else hi = mid;
  }
  const uint64_t off = (ch - c.chunk0[lo]) * kCopyChunk;
  const uint64_t n = min(kCopyChunk, c.bytes[lo] - off);
  uint8_t* dst = reinterpret_cast<uint8_t*>(c.dst[lo]) + off;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(c.src[lo]) + off;
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src);
  if ((a & 15u) == 0) {
    for (uint64_t i = threadIdx.x; i < n / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = __ldcs(reinterpret_cast<const uint4*>(src) + i);
    for (uint64_t i = (n / 16) * 16 + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  } else {  // different 16-byte phases: 16-byte stores assembled from the aligned source vectors
    dfx::copy_shift16<false>(dst, src, n, threadIdx.x, blockDim.x);
  }
}
}  // namespace

extern "C" {

dfx_status dfx_copy_many(int64_t n, const uint64_t* dst, const uint64_t* src, const uint64_t* bytes,
                         dfx_stream stream) {
  for (int64_t i0 = 0; i0 < n; i0 += kCopyMany) {
    CopyMany c{};
    uint64_t chunks = 0;
    for (int64_t i = i0; i < std::min<int64_t>(n, i0 + kCopyMany); ++i) {
      if (bytes[i] == 0) continue;
      c.dst[c.n] = dst[i];
      c.src[c.n] = src[i];
      c.bytes[c.n] = bytes[i];
      c.chunk0[c.n] = chunks;
      chunks += (bytes[i] + kCopyChunk - 1) / kCopyChunk;
      ++c.n;
    }
    if (c.n == 0) continue;
    c.chunk0[c.n] = chunks;
    copy_many_kernel<<<(unsigned)chunks, 256, 0, stream>>>(c);
    DFX_LAUNCH_CHECK("copy_many_kernel");
  }
  return DFX_OK;
}

dfx_status dfx_view_meta(const int32_t* group_off, const int32_t* roll_group, int64_t r0, int64_t r1, int64_t n_roll,
                         int32_t* group_off_out, int32_t* roll_group_out, dfx_stream stream) {
  if (r1 < r0) return dfx::fail(DFX_INVALID_ARGUMENT, "dfx_view_meta: r1 < r0");
  const int64_t n = std::max<int64_t>(r1 - r0 + 1, n_roll);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 1184);
  view_meta_kernel<<<grid, 256, 0, stream>>>(group_off, roll_group, r0, r1, group_off_out, roll_group_out);
  DFX_LAUNCH_CHECK("view_meta_kernel");
  return DFX_OK;
}

dfx_status dfx_copy_sm(void* dst, const void* src, size_t bytes, dfx_stream stream) {
  if (bytes == 0) return DFX_OK;
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src);
  const int width = (a & 15u) == 0 ? 16 : 1;  // (1: copy_shift16)
  const uint64_t units = bytes / uint64_t(width) + 1;
  const unsigned grid = (unsigned)std::min<uint64_t>((units + 255) / 256, 148ull * 8);
  copy_sm_kernel<<<grid, 256, 0, stream>>>(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes, width);
  DFX_LAUNCH_CHECK("copy_sm_kernel");
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
