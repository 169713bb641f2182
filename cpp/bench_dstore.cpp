// bench_dstore.cpp -- BASELINE config 4 through the C++ host of the distributed DataBuffer (include/dfx_dstore.hpp),
// in the reference's fork-per-node process model (runner.hpp:655-742): one process per GPU, forked here; rank 0
// makes the communicator id and hands it to the others through pipes. No Python anywhere.
//
// The round trip DP 8 -> 4 (tp 2) -> 8 of a 16.8M-token batch (1024 prompts x 16 x 1024 tokens; payload token_id,
// lp, old_lp, ref_lp = 16 B/token + reward / advantage channels), one DataBuffer per GPU (B = N; logical world 8,
// or 16 at N = 8). Each process times its steps with CUDA events on its stream; rank 0 prints ONE JSON line with
// the max over ranks and the NVLink bytes each GPU pulled per round trip.
// usage: bench_dstore [n_gpus] [steps] [warmup] [pull|nccl]
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dfx_dstore.hpp"

namespace {

struct Result {
  double ms;
  double pulled;  // bytes received per round trip
  int ok;
};

uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// a device batch of R records x 16 rollouts x L tokens with views of its producer groups
struct Prod {
  std::vector<std::shared_ptr<uint8_t>> keep;
  dfx_batch whole{};
  std::vector<int32_t> hgo;
  std::vector<int64_t> hcu;
};

Prod make_batch(int dev, uint64_t first_id, uint32_t R, uint32_t n, uint32_t L, cudaStream_t st) {
  Prod p;
  const uint64_t S = uint64_t(R) * n, T = S * L;
  std::vector<uint64_t> ids(R);
  std::vector<double> reward(S);
  p.hgo.resize(R + 1);
  p.hcu.resize(S + 1);
  for (uint32_t r = 0; r < R; ++r) ids[r] = first_id + r;
  for (uint32_t r = 0; r <= R; ++r) p.hgo[r] = int32_t(r * n);
  for (uint64_t s = 0; s <= S; ++s) p.hcu[s] = int64_t(s * L);
  for (uint64_t s = 0; s < S; ++s) reward[s] = double(mix64(11 ^ (first_id * 16 + s)) >> 11) * (1.0 / 9007199254740992.0);
  std::vector<int32_t> rg(S);
  for (uint64_t s = 0; s < S; ++s) rg[s] = int32_t(s / n);
  auto up = [&](const void* src, size_t bytes, size_t pad) {
    auto m = dfx::device_alloc(dev, bytes + pad, true);
    if (src && bytes) dfx::store_cuda(cudaMemcpy(m.get(), src, bytes, cudaMemcpyHostToDevice), "H2D");
    p.keep.push_back(m);
    return m.get();
  };
  dfx_batch& b = p.whole;
  b.n_records = R;
  b.n_rollouts = int64_t(S);
  b.token_base = 0;
  b.token_span = int64_t(T);
  b.ids = reinterpret_cast<uint64_t*>(up(ids.data(), R * 8, 0));
  b.group_off = reinterpret_cast<int32_t*>(up(p.hgo.data(), (R + 1) * 4, 0));
  b.roll_group = reinterpret_cast<int32_t*>(up(rg.data(), S * 4, 0));
  b.cu_seqlens = reinterpret_cast<int64_t*>(up(p.hcu.data(), (S + 1) * 8, 0));
  double* rew = reinterpret_cast<double*>(up(reward.data(), S * 8, 0));
  double* adv = reinterpret_cast<double*>(up(nullptr, S * 8, 0));
  b.ch[0] = adv;  // schema: advantage, reward
  b.ch[1] = rew;
  float* lp = reinterpret_cast<float*>(up(nullptr, T * 4, 256));
  float* old = reinterpret_cast<float*>(up(nullptr, T * 4, 256));
  float* ref = reinterpret_cast<float*>(up(nullptr, T * 4, 256));
  int32_t* tid = reinterpret_cast<int32_t*>(up(nullptr, T * 4, 256));
  b.st[0] = tid;
  b.st[1] = lp;
  b.st[2] = old;
  b.st[3] = ref;
  uint64_t* dids = const_cast<uint64_t*>(b.ids);
  dfx::store_check(dfx_synth_tokens(11, dids, R, int32_t(n), b.cu_seqlens, 0, int64_t(T), lp, old, ref, nullptr,
                                    nullptr, nullptr, tid, st));
  dfx_packed pk{};
  pk.n_records = R;
  pk.n_rollouts = int64_t(S);
  pk.group_off = b.group_off;
  pk.reward = rew;
  dfx::store_check(dfx_grpo_advantage(&pk, 1e-6, adv, nullptr, st));  // fn_group_advantage on the device
  dfx::store_cuda(cudaStreamSynchronize(st), "sync");
  return p;
}

// view of records [r0, r1) of a batch (rebased record metadata on the device)
struct View {
  dfx_batch b{};
  std::vector<int32_t> hgo;
  std::vector<int64_t> hcu;
  std::shared_ptr<uint8_t> meta;
};
View make_view(int dev, const Prod& p, int64_t r0, int64_t r1, cudaStream_t st) {
  View v;
  const int32_t s0 = p.hgo[r0], s1 = p.hgo[r1];
  v.b = p.whole;
  v.b.n_records = r1 - r0;
  v.b.n_rollouts = s1 - s0;
  v.b.ids = p.whole.ids + r0;
  v.b.cu_seqlens = p.whole.cu_seqlens + s0;
  for (int c = 0; c < 2; ++c) v.b.ch[c] = p.whole.ch[c] + s0;
  v.b.token_base = p.hcu[s0];
  v.b.token_span = p.hcu[s1] - p.hcu[s0];
  v.hgo.resize(size_t(r1 - r0 + 1));
  for (int64_t r = r0; r <= r1; ++r) v.hgo[size_t(r - r0)] = p.hgo[r] - s0;
  v.hcu.assign(p.hcu.begin() + s0, p.hcu.begin() + s1 + 1);
  v.meta = dfx::device_alloc(dev, size_t(r1 - r0 + 1) * 4 + size_t(s1 - s0) * 4 + 256);
  int32_t* go = reinterpret_cast<int32_t*>(v.meta.get());
  int32_t* rg = reinterpret_cast<int32_t*>(v.meta.get() + ((size_t(r1 - r0 + 1) * 4 + 255) & ~size_t(255)));
  dfx::store_check(dfx_view_meta(p.whole.group_off, p.whole.roll_group, r0, r1, s1 - s0, go, rg, st));
  v.b.group_off = go;
  v.b.roll_group = rg;
  v.b.h_group_off = v.hgo.data();
  v.b.h_cu = v.hcu.data();
  return v;
}

Result run_rank(int rank, int N, int steps, int warmup, int transport, const std::array<char, DFX_COMM_ID_BYTES>& id) {
  dfx::store_cuda(cudaSetDevice(rank), "cudaSetDevice");
  cudaStream_t st;
  dfx::store_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  dfx::Comm comm(N, rank, id);
  const uint32_t logical = N == 8 ? 16 : 8, W = logical / uint32_t(N), dp = logical;
  std::vector<int32_t> row(logical);
  for (uint32_t w = 0; w < logical; ++w) row[w] = int32_t(w / W);
  const uint32_t B = N == 1 ? 1 : uint32_t(N), Wn = N == 1 ? logical : W;
  std::map<std::string, dfx::DStageCfg> stages;
  stages["s"] = dfx::DStageCfg{{dp, 1}, {dp / 2, 2}};
  stages["t"] = dfx::DStageCfg{{dp / 2, 2}, {dp, 1}};
  dfx::DistBufferStore store(comm, B, Wn, row, stages, {4, 4, 4, 4}, 2, st, transport);
  const uint32_t R = 1024 / uint32_t(N);
  Prod prod = make_batch(rank, uint64_t(rank) * R, R, 16, 1024, st);
  std::vector<uint32_t> local_p;
  for (uint32_t p = 0; p < dp; ++p)
    if (row[p] == rank) local_p.push_back(p);
  const uint32_t per = R / uint32_t(local_p.size());
  std::vector<View> views;
  for (size_t j = 0; j < local_p.size(); ++j) views.push_back(make_view(rank, prod, j * per, (j + 1) * per, st));
  std::vector<uint32_t> mine_s;
  for (uint32_t d = 0; d < dp / 2; ++d)
    if (row[d * 2] == rank || row[d * 2 + 1] == rank) mine_s.push_back(d);
  uint32_t local_workers = 0;
  for (uint32_t w = 0; w < logical; ++w) local_workers += row[w] == rank ? 1 : 0;
  const dfx::Layout to_s{dp / 2, 2}, to_t{dp, 1};
  uint64_t it = 0;
  auto step = [&] {
    for (size_t j = 0; j < local_p.size(); ++j) store.put("s", it, local_p[j], 0, views[j].b);
    store.ensure_ready("s", it, to_s);
    for (uint32_t d : mine_s) {
      const dfx_batch b = store.get("s", it, d, to_s);
      for (uint32_t t = 0; t < 2; ++t)
        if (row[d * 2 + t] == rank) store.put("t", it, d, t, b);
    }
    store.ensure_ready("t", it, to_t);
    for (uint32_t w = 0; w < local_workers; ++w) store.worker_done(it);
    ++it;
  };
  for (int i = 0; i < warmup; ++i) step();
  dfx::store_cuda(cudaStreamSynchronize(st), "sync");
  const auto s0 = store.stats();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int i = 0; i < steps; ++i) step();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const auto s1 = store.stats();
  Result res{ms / steps, double(s1[2] - s0[2]) / steps, 1};
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return res;
}

}  // namespace

int main(int argc, char** argv) {
  const int N = argc > 1 ? std::atoi(argv[1]) : 2;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 50;
  const int warmup = argc > 3 ? std::atoi(argv[3]) : 5;
  const int transport = argc > 4 && std::string(argv[4]) == "nccl" ? DFX_TRANSPORT_NCCL : DFX_TRANSPORT_PULL;
  // no CUDA call in the parent before the fork; rank 0 creates the id after it
  std::vector<int> id_pipe(2 * N), res_pipe(2 * N);
  for (int r = 0; r < N; ++r) {
    if (pipe(&id_pipe[2 * r]) || pipe(&res_pipe[2 * r])) return 1;
  }
  std::vector<pid_t> kids;
  for (int r = 0; r < N; ++r) {
    const pid_t pid = fork();
    if (pid == 0) {
      Result res{0, 0, 0};
      try {
        std::array<char, DFX_COMM_ID_BYTES> id{};
        if (r == 0) {
          id = dfx::Comm::unique_id();
          for (int q = 1; q < N; ++q)
            if (write(id_pipe[2 * q + 1], id.data(), id.size()) != ssize_t(id.size())) _exit(2);
        } else if (read(id_pipe[2 * r], id.data(), id.size()) != ssize_t(id.size())) {
          _exit(2);
        }
        res = run_rank(r, N, steps, warmup, transport, id);
      } catch (const std::exception& ex) {
        std::fprintf(stderr, "rank %d: %s\n", r, ex.what());
      }
      if (write(res_pipe[2 * r + 1], &res, sizeof(res)) != ssize_t(sizeof(res))) _exit(3);
      _exit(res.ok ? 0 : 1);
    }
    kids.push_back(pid);
  }
  double ms = 0, pulled = 0;
  int ok = 1;
  for (int r = 0; r < N; ++r) {
    Result res{};
    if (read(res_pipe[2 * r], &res, sizeof(res)) != ssize_t(sizeof(res))) ok = 0;
    ok &= res.ok;
    ms = std::max(ms, res.ms);
    pulled = std::max(pulled, res.pulled);
  }
  for (pid_t k : kids) {
    int status = 0;
    waitpid(k, &status, 0);
  }
  if (!ok) {
    std::printf("{\"error\": \"a rank failed\"}\n");
    return 1;
  }
  const double tokens = 1024.0 * 16 * 1024;
  std::printf("{\"bench\": \"cpp/bench_dstore (C++ host, fork per GPU)\", \"n_gpus\": %d, \"transport\": \"%s\", "
              "\"steps\": %d, \"ms_per_round_trip\": %.5f, \"tokens_per_s\": %.1f, \"nvlink_bytes_per_gpu\": %.0f, "
              "\"nvlink_gbs\": %.1f, \"nvlink_frac_of_770\": %.4f}\n",
              N, transport == DFX_TRANSPORT_NCCL ? "nccl" : "pull", steps, ms, tokens / (ms / 1e3), pulled,
              pulled / (ms / 1e3) / 1e9, pulled / (ms / 1e3) / 1e9 / 770.0);
  return 0;
}
