// api.cu -- error plumbing and library identity for libdfx.
#include <cstdio>
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
