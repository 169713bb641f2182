// NVLink read vs write rate between two GPUs driven concurrently (one process, peer access): each GPU pulls
// (SM loads of the peer's memory), pushes (SM stores into the peer's memory) or copy-engine copies 64 MB at the
// same time as the other. Diagnostic for the distributed DataBuffer's transport (csrc/dstore.cu).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rw_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  const size_t step = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * step < n; i += 4 * step) {
    uint4 a = src[i], b = src[i + step], c = src[i + 2 * step], d = src[i + 3 * step];
    dst[i] = a; dst[i + step] = b; dst[i + 2 * step] = c; dst[i + 3 * step] = d;
  }
  for (; i < n; i += step) dst[i] = src[i];
}

int main() {
  const size_t bytes = 64ull << 20, n = bytes / 16;
  uint4 *loc[2], *oth[2];
  cudaStream_t st[2];
  for (int g = 0; g < 2; ++g) {
    cudaSetDevice(g);
    cudaDeviceEnablePeerAccess(1 - g, 0);
    cudaMalloc(&loc[g], bytes);
    cudaMalloc(&oth[g], bytes);
    cudaMemset(loc[g], g, bytes);
    cudaStreamCreate(&st[g]);
  }
  for (int mode = 0; mode < 3; ++mode) {
    for (int ctas : {148, 296, 592}) {
      if (mode == 2 && ctas != 148) continue;
      cudaEvent_t e0[2], e1[2];
      for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaEventCreate(&e0[g]); cudaEventCreate(&e1[g]); }
      for (int rep = 0; rep < 6; ++rep) {
        for (int g = 0; g < 2; ++g) {
          cudaSetDevice(g);
          if (rep == 5) cudaEventRecord(e0[g], st[g]);
          if (mode == 0) rw_kernel<<<ctas, 512, 0, st[g]>>>(oth[g], loc[1 - g], n);       // pull: read peer
          else if (mode == 1) rw_kernel<<<ctas, 512, 0, st[g]>>>(oth[1 - g], loc[g], n);  // push: write peer
          else cudaMemcpyAsync(oth[g], loc[1 - g], bytes, cudaMemcpyDefault, st[g]);       // CE pull
          if (rep == 5) cudaEventRecord(e1[g], st[g]);
        }
      }
      for (int g = 0; g < 2; ++g) {
        cudaSetDevice(g);
        cudaEventSynchronize(e1[g]);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0[g], e1[g]);
        std::printf("%s ctas %d gpu %d: %.1f us -> %.0f GB/s\n", mode == 0 ? "pull(SM loads)" : mode == 1 ? "push(SM stores)" : "CE pull", ctas, g, ms * 1e3, bytes / (ms / 1e3) / 1e9);
      }
    }
  }
  return 0;
}
