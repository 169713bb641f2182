// bench_store.cpp -- BASELINE config 4 through the C++ device DataBuffer (include/dfx_store.hpp), in the
// reference's own process model: one process drives the box's GPUs, B stores x W logical workers.
//
// The round trip DP 8 -> 4 (tp 2) -> 8 of a 16.8M-token batch (1024 prompts x 16 x 1024 tokens; payload
// token_id, lp, old_lp, ref_lp = 16 B/token + reward / advantage channels), one DataBuffer per GPU (B = N;
// logical world 8, or 16 at N = 8). Prints one JSON line: round-trip time, bytes copied across GPUs, GB/s.
// usage: bench_store [n_gpus] [iters]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "dfx_store.hpp"

int main(int argc, char** argv) {
  int avail = 0;
  if (cudaGetDeviceCount(&avail) != cudaSuccess || avail == 0) {
    std::printf("{\"skipped\": \"no CUDA device\"}\n");
    return 0;
  }
  const int N = argc > 1 ? std::min(std::atoi(argv[1]), avail) : avail;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 20;
  const uint32_t logical = N == 8 ? 16 : 8, B = uint32_t(N), W = logical / B, dp = logical;
  std::vector<int> gpu(logical);
  for (uint32_t w = 0; w < logical; ++w) gpu[w] = int(w / W);
  std::map<std::string, dfx::StagePlan> stages;
  stages["s"] = dfx::StagePlan{{dp, 1}, true, {dp / 2, 2}};
  stages["t"] = dfx::StagePlan{{dp / 2, 2}, true, {dp, 1}};
  dfx::DeviceBufferStore store(B, W, gpu, stages);
  // producer group p: 1024/dp prompts x 16 rollouts x 1024 tokens on the GPU of its lead worker
  const uint32_t per = 1024 / dp, R = 16, L = 1024;
  std::vector<dfx::DeviceBatch> prod;
  for (uint32_t p = 0; p < dp; ++p) {
    std::vector<uint64_t> ids(per);
    std::vector<int32_t> go(per + 1);
    std::vector<int64_t> cu(per * R + 1);
    for (uint32_t r = 0; r < per; ++r) ids[r] = p * per + r;
    for (uint32_t r = 0; r <= per; ++r) go[r] = int32_t(r * R);
    for (uint32_t s = 0; s <= per * R; ++s) cu[s] = int64_t(s) * L;
    std::map<std::string, std::vector<double>> ch{{"advantage", std::vector<double>(per * R, -0.5)},
                                                  {"reward", std::vector<double>(per * R, 0.25)}};
    std::map<std::string, std::pair<std::vector<uint8_t>, size_t>> st;
    for (const char* n : {"token_id", "lp", "old_lp", "ref_lp"})
      st[n] = {std::vector<uint8_t>(size_t(per) * R * L * 4, uint8_t(p)), 4};
    prod.push_back(dfx::DeviceBatch::upload(gpu[p], ids, go, cu, ch, st));
  }
  cudaDeviceSynchronize();
  double t_ex_s = 0, t_ex_t = 0, t_rest = 0;
  using clk = std::chrono::steady_clock;
  auto since = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
  auto trip = [&](uint32_t it) {
    auto a = clk::now();
    for (uint32_t p = 0; p < dp; ++p) store.put("s", it, p, 0, prod[p]);
    cudaSetDevice(gpu[0]);
    store.ensure_ready("s", it, dfx::Layout{dp / 2, 2});  // the exchange (the first consumer's get runs it)
    t_ex_s += since(a);
    a = clk::now();
    for (uint32_t w = 0; w < logical; ++w) {  // every worker's get on its GPU
      cudaSetDevice(gpu[w]);
      const uint32_t d = w / 2;
      dfx::DeviceBatch b = store.get("s", it, d, dfx::Layout{dp / 2, 2});
      store.put("t", it, d, w % 2, b);
    }
    t_rest += since(a);
    a = clk::now();
    store.ensure_ready("t", it, dfx::Layout{dp, 1});
    t_ex_t += since(a);
    a = clk::now();
    for (uint32_t w = 0; w < logical; ++w) {
      cudaSetDevice(gpu[w]);
      (void)store.get("t", it, w, dfx::Layout{dp, 1});
    }
    for (uint32_t w = 0; w < logical; ++w) store.worker_done(it);
    t_rest += since(a);
  };
  for (uint32_t it = 0; it < 3; ++it) trip(it);
  t_ex_s = t_ex_t = t_rest = 0;
  const uint64_t c0 = store.bytes_copied();
  const auto t0 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; ++it) trip(3 + it);
  const auto t1 = std::chrono::steady_clock::now();
  const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / iters;
  const double copied = double(store.bytes_copied() - c0) / iters;  // all GPUs, local + peer
  std::printf("{\"workload\": \"C4 round trip dp%u -> dp%u (tp2) -> dp%u, 16.8M tokens x 16 B, B=%u W=%u, %d GPU, "
              "C++ device DataBuffer (one process)\", \"ms_per_trip\": %.4f, \"tokens_per_s\": %.4g, "
              "\"bytes_copied_per_trip\": %.0f, \"copy_GBs_per_gpu\": %.1f, \"exchange_s_ms\": %.4f, "
              "\"exchange_t_ms\": %.4f, \"other_ms\": %.4f}\n",
              dp, dp / 2, dp, B, W, N, ms, 16777216.0 / (ms / 1e3), copied, copied / N / (ms / 1e3) / 1e9,
              t_ex_s / iters, t_ex_t / iters, t_rest / iters);
  return 0;
}
