// NVLink all-to-all rate among N GPUs of one box (one process, peer access), every GPU moving `per_pair` bytes
// to / from each of its N-1 peers at once, as the distributed DataBuffer's reshard does at N = 4:
//   pull: each GPU's SMs load its peers' memory (one kernel; the peers interleaved per CTA)
//   push: each GPU's SMs store into its peers' memory
//   ce:   one cudaMemcpyPeerAsync per peer, each on its own stream
// Prints the per-GPU ingress rate. Diagnostic for csrc/dstore.cu's transport choice.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

struct Ptrs {
  uint4* dst[8];
  const uint4* src[8];
  int n;
};

// CTA b works on pair (b % n); within a pair, a grid-stride copy with 4 x 16 B in flight per thread
__global__ void a2a_kernel(Ptrs p, size_t n16) {
  const int pr = blockIdx.x % p.n;
  const int cta_per = gridDim.x / p.n;
  const int b = blockIdx.x / p.n;
  uint4* __restrict__ dst = p.dst[pr];
  const uint4* __restrict__ src = p.src[pr];
  const size_t step = size_t(cta_per) * blockDim.x;
  size_t i = size_t(b) * blockDim.x + threadIdx.x;
  for (; i + 3 * step < n16; i += 4 * step) {
    uint4 a = src[i], c = src[i + step], d = src[i + 2 * step], e = src[i + 3 * step];
    dst[i] = a; dst[i + step] = c; dst[i + 2 * step] = d; dst[i + 3 * step] = e;
  }
  for (; i < n16; i += step) dst[i] = src[i];
}

// TMA pull: each CTA streams its share of a pair's bytes through shared memory with bulk copies (peer global ->
// shared, shared -> local global), 4 stages of 16 KB in flight
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32) a2a_tma_kernel(Ptrs p, size_t bytes) {
  constexpr int kStages = 4;
  constexpr unsigned kChunk = 16384;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[kStages];
  const int pr = blockIdx.x % p.n, cta_per = gridDim.x / p.n, b = blockIdx.x / p.n;
  const unsigned char* src = reinterpret_cast<const unsigned char*>(p.src[pr]);
  unsigned char* dst = reinterpret_cast<unsigned char*>(p.dst[pr]);
  const size_t n_chunks = bytes / kChunk;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned phase = 0;
    size_t issued = 0, done = 0;
    const size_t mine = (n_chunks > (size_t)b) ? (n_chunks - b + cta_per - 1) / cta_per : 0;
    auto issue = [&](size_t k) {
      const size_t c = b + k * cta_per;
      const int st = (int)(k % kStages);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"(kChunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + st * kChunk)), "l"(src + c * kChunk), "r"(kChunk), "r"(smem_u32(&bar[st])) : "memory");
    };
    for (; issued < mine && issued < kStages; ++issued) issue(issued);
    for (; done < mine; ++done) {
      const int st = (int)(done % kStages);
      const unsigned par = (unsigned)((done / kStages) & 1);
      asm volatile("{\n .reg .pred P;\n W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W;\n}" ::"r"(smem_u32(&bar[st])), "r"(par) : "memory");
      const size_t c = b + done * cta_per;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * kChunk), "r"(smem_u32(sm + st * kChunk)), "r"(kChunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (issued < mine) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        issue(issued++);
      }
      (void)phase;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main(int argc, char** argv) {
  int N = 0;
  cudaGetDeviceCount(&N);
  if (argc > 1) N = std::min(N, atoi(argv[1]));
  if (N < 2) { std::printf("needs 2+ GPUs\n"); return 0; }
  const size_t per_pair = 32ull << 20, n16 = per_pair / 16;
  std::vector<uint4*> in(N), out(N);  // in[g]: N slots of per_pair (one per peer); out[g]: N slots
  std::vector<std::vector<cudaStream_t>> st(N, std::vector<cudaStream_t>(N));
  for (int g = 0; g < N; ++g) {
    cudaSetDevice(g);
    for (int h = 0; h < N; ++h) if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    cudaMalloc(&in[g], per_pair * N);
    cudaMalloc(&out[g], per_pair * N);
    cudaMemset(out[g], g + 1, per_pair * N);
    for (int h = 0; h < N; ++h) cudaStreamCreateWithFlags(&st[g][h], cudaStreamNonBlocking);
  }
  const char* names[4] = {"pull(SM loads)", "push(SM stores)", "ce(peer memcpy)", "pull(TMA bulk)"};
  for (int g = 0; g < N; ++g) {
    cudaSetDevice(g);
    cudaFuncSetAttribute(a2a_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
  }
  for (int mode = 0; mode < 4; ++mode) {
    for (int ctas : {148, 296, 592}) {
      if (mode == 2 && ctas != 148) continue;
      std::vector<cudaEvent_t> e0(N), e1(N);
      for (int g = 0; g < N; ++g) {
        cudaSetDevice(g);
        cudaEventCreate(&e0[g]);
        cudaEventCreate(&e1[g]);
      }
      for (int rep = 0; rep < 6; ++rep) {
        for (int g = 0; g < N; ++g) cudaSetDevice(g), cudaDeviceSynchronize();
        for (int g = 0; g < N; ++g) {
          cudaSetDevice(g);
          cudaEventRecord(e0[g], st[g][0]);
          Ptrs p{};
          p.n = N - 1;
          int k = 0;
          for (int h = 0; h < N; ++h) {
            if (h == g) continue;
            if (mode == 0) {  // g reads h's out slot g into its in slot h
              p.src[k] = out[h] + size_t(g) * n16;
              p.dst[k] = in[g] + size_t(h) * n16;
            } else {  // g writes its out slot h into h's in slot g
              p.src[k] = out[g] + size_t(h) * n16;
              p.dst[k] = in[h] + size_t(g) * n16;
            }
            if (mode == 2) {
              cudaStreamWaitEvent(st[g][h], e0[g], 0);
              cudaMemcpyPeerAsync(in[g] + size_t(h) * n16, g, out[h] + size_t(g) * n16, h, per_pair, st[g][h]);
            }
            ++k;
          }
          if (mode < 2) a2a_kernel<<<(ctas / (N - 1)) * (N - 1), 512, 0, st[g][0]>>>(p, n16);
          if (mode == 3) {  // (same direction as the SM pull: g reads h's slot)
            a2a_tma_kernel<<<(ctas * 2 / (N - 1)) * (N - 1), 32, 4 * 16384, st[g][0]>>>(p, per_pair);
          }
          if (mode == 2) {
            for (int h = 0; h < N; ++h) {
              if (h == g) continue;
              cudaEvent_t ev;
              cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
              cudaEventRecord(ev, st[g][h]);
              cudaStreamWaitEvent(st[g][0], ev, 0);
              cudaEventDestroy(ev);
            }
          }
          cudaEventRecord(e1[g], st[g][0]);
        }
      }
      double worst = 0;
      for (int g = 0; g < N; ++g) {
        cudaSetDevice(g);
        cudaEventSynchronize(e1[g]);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0[g], e1[g]);
        worst = std::max(worst, (double)ms);
      }
      std::printf("N=%d %s ctas %d: %.1f us (slowest GPU) -> %.0f GB/s per GPU (%zu MB from each of %d peers)\n", N,
                  names[mode], ctas, worst * 1e3, per_pair * (N - 1) / (worst / 1e3) / 1e9, per_pair >> 20, N - 1);
    }
  }
  return 0;
}
