// bench_e2e.cpp -- the C++ operator API on the measured path: the reference's own runtime (preset_dag("grpo") ->
// registry_bind -> run_iteration over BufferStore + InprocFabric, one thread per worker, runner.hpp:525-530) with
// the GPU stage functions of include/dfx_distflow.hpp bound in (gpu_registry()), on BASELINE config 2 from host
// buffers: 1024 prompts x 16 rollouts x UNIFORM[1,4096] tokens (~33.5M tokens), logical dp8 -> actor_train dp4/tp2,
// every worker on GPU 0.
//
// The hot path is the DAG slice group_advantage_compute -> DataBuffer (reference BufferStore) -> actor_train (the
// fused clipped surrogate + k3 KL on the GPU). Its wall time per iteration is taken from run_iteration's own node
// timings (worker.hpp:219-255, with the cost-model sleep set to zero): from the first worker entering
// group_advantage_compute to the last worker leaving actor_train. The same program runs the chain with the
// reference's builtin_registry() (CPU fn_group_advantage / fn_train) for comparison. Generation upstream is a
// bench-only CPU generator that fills the 17 B/token payload (token_id | lp | old_lp | ref_lp | mask,
// DESIGN.md §3) with valid values; it is outside the timed slice.
// A third run takes the same slice through the device-resident operator API (include/dfx_device_chain.hpp):
// one upload per batch, then the DataBuffer and both nodes on the GPU.
// usage: bench_e2e [iterations] [prompts]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <thread>

#include "distflow/dag.hpp"
#include "distflow/planner.hpp"
#include "distflow/worker.hpp"
#include "dfx_device_chain.hpp"
#include "dfx_distflow.hpp"

using namespace distflow;

namespace {

// bench-only generator: the reference's draw_tokens lengths, payload of valid f32 log-probs (cheap LCG values)
void bench_generate(const NodeSpec& node, SampleBatch& batch, StageContext& ctx) {
  (void)node;
  for (auto& rec : batch.records) {
    rec.rollouts.resize(ctx.gen.rollouts_per_prompt);
    for (uint32_t r = 0; r < ctx.gen.rollouts_per_prompt; ++r) {
      Rollout& ro = rec.rollouts[r];
      const uint32_t L = detail::draw_tokens(ctx.gen.response_tokens, ctx.run_seed, rec.sample_id, r);
      ro.token_count = L;
      ro.payload.assign(size_t(L) * dfx_distflow::kPayloadBytesPerToken, 0);
      uint64_t z = keyed_hash(ctx.run_seed, "bench_tok", rec.sample_id, r);
      float* lp = reinterpret_cast<float*>(ro.payload.data() + 4 * size_t(L));
      float* old = lp + L;
      float* ref = old + L;
      uint8_t* mask = reinterpret_cast<uint8_t*>(ref + L);
      for (uint32_t t = 0; t < L; ++t) {
        z = z * 6364136223846793005ull + 1442695040888963407ull;
        const float u = float(z >> 40) * (1.0f / 16777216.0f), v = float((z >> 16) & 0xffffff) * (1.0f / 16777216.0f);
        lp[t] = -4.0f * u;
        old[t] = lp[t] + 0.25f * (2.0f * v - 1.0f);
        ref[t] = lp[t] + 0.1f * (2.0f * u - 1.0f);
        mask[t] = t >= L / 10 ? 1 : 0;
      }
    }
  }
}

FunctionRegistry with_generator(bool gpu) {
  FunctionRegistry reg;
  reg.register_fn("actor_generate", bench_generate);
  reg.register_fn("ref_logprob", fn_ref_logprob);
  reg.register_fn("value_inference", fn_value);
  reg.register_fn("reward_compute", fn_reward);
  reg.register_fn("group_advantage", gpu ? dfx_distflow::gpu_group_advantage : StageFn(fn_group_advantage));
  reg.register_fn("ppo_advantage", gpu ? dfx_distflow::gpu_ppo_advantage : StageFn(fn_ppo_advantage));
  reg.register_fn("train_actor", gpu ? dfx_distflow::gpu_train : StageFn(fn_train));
  reg.register_fn("train_critic", gpu ? dfx_distflow::gpu_train : StageFn(fn_train));
  return reg;
}

struct Result {
  double hot_ms = 0, iter_ms = 0;
  uint64_t tokens = 0;
};

Result run(bool gpu, uint32_t iterations, uint64_t prompts) {
  const ClusterTopology topo{1, 8};
  const TaskChain chain = serialize_graph(preset_dag(Algorithm::GRPO));
  std::map<std::string, ParallelLayout> layouts;
  for (const auto& n : chain.nodes) layouts[n.node_id] = ParallelLayout{8, 1};
  layouts["actor_train"] = ParallelLayout{4, 2};
  InprocFabric fabric(topo);
  std::map<std::string, StoreStagePlan> stages;
  for (size_t i = 0; i < chain.nodes.size(); ++i) {
    StoreStagePlan p;
    p.produced = layouts.at(chain.nodes[i].node_id);
    if (i + 1 < chain.nodes.size()) p.consumed = layouts.at(chain.nodes[i + 1].node_id);
    p.tag = tags::kRedistBase + uint32_t(i);
    stages[chain.nodes[i].node_id] = p;
  }
  BufferStore store(topo, 0, &fabric, stages);
  const FunctionRegistry reg = with_generator(gpu);
  std::vector<std::vector<IterationMetrics>> per_worker(topo.world_size());
  std::vector<std::thread> threads;
  std::mutex mu;
  std::string err;
  for (uint32_t rk = 0; rk < topo.world_size(); ++rk) {
    threads.emplace_back([&, rk] {
      try {
        if (gpu) dfx_distflow::cuda_check(cudaSetDevice(0), "cudaSetDevice");
        WorkerState st;
        st.rank = rk;
        st.topo = topo;
        st.chain = registry_bind(chain, reg, layouts);
        st.store = &store;
        st.fabric = &fabric;
        st.global_batch = prompts;
        st.ctx.gen.rollouts_per_prompt = 16;
        st.ctx.gen.response_tokens.kind = TokenDist::Kind::UNIFORM;
        st.ctx.gen.response_tokens.min = 1;
        st.ctx.gen.response_tokens.max = 4096;
        st.ctx.gen.bytes_per_token = dfx_distflow::kPayloadBytesPerToken;
        st.ctx.cost = CostModel{0, 0, 0, 0, 0, 0};
        st.init(1);
        const ParallelLayout& g = st.chain.nodes.front().layout;
        DatasetSpec spec;
        spec.synthetic_n = prompts;
        st.loader = make_group_loader(spec, g, g.dp_rank(rk), 1);
        for (uint32_t it = 0; it < iterations; ++it) per_worker[rk].push_back(run_iteration(st, it));
      } catch (const std::exception& e) {
        std::lock_guard lk(mu);
        if (err.empty()) err = e.what();
      }
    });
  }
  for (auto& t : threads) t.join();
  if (!err.empty()) {
    std::fprintf(stderr, "chain error: %s\n", err.c_str());
    std::exit(1);
  }
  // per iteration: first entry into group_advantage_compute .. last exit from actor_train, over the workers;
  // iterations 0 and 1 are warm-up (arena growth, first-touch)
  Result res;
  uint32_t counted = 0;
  for (uint32_t it = std::min<uint32_t>(2, iterations - 1); it < iterations; ++it) {
    uint64_t b = UINT64_MAX, e = 0, ib = UINT64_MAX, ie = 0, tok = 0;
    for (uint32_t rk = 0; rk < topo.world_size(); ++rk) {
      for (const auto& n : per_worker[rk][it].nodes) {
        ib = std::min(ib, n.start_ns);
        ie = std::max(ie, n.end_ns);
        if (n.node_id == "group_advantage_compute") {
          b = std::min(b, n.start_ns);
          tok += n.tokens;
        }
        if (n.node_id == "actor_train") e = std::max(e, n.end_ns);
      }
    }
    res.hot_ms += double(e - b) / 1e6;
    res.iter_ms += double(ie - ib) / 1e6;
    res.tokens = tok;
    ++counted;
  }
  res.hot_ms /= counted;
  res.iter_ms /= counted;
  return res;
}

// The same DAG slice with device-resident batches (include/dfx_device_chain.hpp): each worker's generated host
// batch crosses to the GPU once (upload_batch: the AoS payload packed into pinned staging, one H2D per array),
// then group_advantage_compute -> the device DataBuffer (dfx::DeviceBufferStore: the reference placement, zero-copy
// views here) -> actor_train run on the device through run_iteration_device.
struct DevResult {
  double hot_ms = 0, upload_ms = 0;
  double loss = 0;
};
DevResult run_device(uint32_t iterations, uint64_t prompts) {
  const uint32_t W = 8;
  const TaskChain chain = serialize_graph(preset_dag(Algorithm::GRPO));
  std::map<std::string, ParallelLayout> layouts;
  std::vector<NodeSpec> upstream, slice;
  for (const auto& n : chain.nodes) {
    layouts[n.node_id] = ParallelLayout{8, 1};
    (n.node_id == "group_advantage_compute" || n.node_id == "actor_train" ? slice : upstream).push_back(n);
  }
  layouts["actor_train"] = ParallelLayout{4, 2};
  std::map<std::string, dfx::StagePlan> stages;
  stages["group_advantage_compute"] = dfx::StagePlan{{8, 1}, true, {4, 2}};
  dfx::DeviceBufferStore store(1, W, std::vector<int>(W, 0), stages);
  auto pool = std::make_shared<dfx::DevicePool>();
  const FunctionRegistry host_reg = with_generator(false);
  const auto dev_reg = dfx_distflow::device_registry();
  struct Span {
    uint64_t up0, up1, hot0, hot1;
  };
  std::vector<std::vector<Span>> spans(W);
  std::vector<double> loss(W);
  std::vector<std::thread> threads;
  std::mutex mu;
  std::string err;
  for (uint32_t rk = 0; rk < W; ++rk) {
    threads.emplace_back([&, rk] {
      try {
        dfx_distflow::cuda_check(cudaSetDevice(0), "cudaSetDevice");
        StageContext hctx;
        hctx.gen.rollouts_per_prompt = 16;
        hctx.gen.response_tokens.kind = TokenDist::Kind::UNIFORM;
        hctx.gen.response_tokens.min = 1;
        hctx.gen.response_tokens.max = 4096;
        hctx.gen.bytes_per_token = dfx_distflow::kPayloadBytesPerToken;
        hctx.run_seed = 1;
        TaskChain up_chain;
        up_chain.nodes = upstream;
        const ExecutableChain up = registry_bind(up_chain, host_reg, layouts);
        dfx_distflow::DeviceWorker w;
        w.rank = rk;
        w.chain = dfx_distflow::device_registry_bind(slice, dev_reg, layouts);
        w.store = &store;
        w.ctx.arena = &dfx_distflow::worker_arena();
        w.ctx.pool = pool;
        const ParallelLayout& g = layouts.at(upstream.front().node_id);
        DatasetSpec spec;
        spec.synthetic_n = prompts;
        DataLoader loader = make_group_loader(spec, g, g.dp_rank(rk), 1);
        for (uint32_t it = 0; it < iterations; ++it) {
          SampleBatch b;
          b.records = loader.next_batch(it, prompts);
          for (const auto& bn : up.nodes) detail::invoke_node(bn, b, hctx);  // generation, ref, reward (CPU)
          Span sp{};
          sp.up0 = detail::now_ns();
          const dfx::DeviceBatch db = dfx_distflow::upload_batch(b, {"reward"}, w.ctx);
          sp.up1 = sp.hot0 = detail::now_ns();
          dfx_distflow::run_iteration_device(w, it, &db);
          sp.hot1 = detail::now_ns();
          spans[rk].push_back(sp);
        }
        loss[rk] = w.ctx.last_loss.loss;
      } catch (const std::exception& e) {
        std::lock_guard lk(mu);
        if (err.empty()) err = e.what();
      }
    });
  }
  for (auto& t : threads) t.join();
  if (!err.empty()) {
    std::fprintf(stderr, "device chain error: %s\n", err.c_str());
    std::exit(1);
  }
  DevResult res;
  uint32_t counted = 0;
  for (uint32_t it = std::min<uint32_t>(2, iterations - 1); it < iterations; ++it) {
    uint64_t u0 = UINT64_MAX, u1 = 0, h0 = UINT64_MAX, h1 = 0;
    for (uint32_t rk = 0; rk < W; ++rk) {
      u0 = std::min(u0, spans[rk][it].up0);
      u1 = std::max(u1, spans[rk][it].up1);
      h0 = std::min(h0, spans[rk][it].hot0);
      h1 = std::max(h1, spans[rk][it].hot1);
    }
    res.upload_ms += double(u1 - u0) / 1e6;
    res.hot_ms += double(h1 - h0) / 1e6;
    ++counted;
  }
  res.upload_ms /= counted;
  res.hot_ms /= counted;
  res.loss = loss[0];
  return res;
}

}  // namespace

int main(int argc, char** argv) {
  int avail = 0;
  if (cudaGetDeviceCount(&avail) != cudaSuccess || avail == 0) {
    std::printf("{\"skipped\": \"no CUDA device\"}\n");
    return 0;
  }
  const uint32_t iterations = argc > 1 ? uint32_t(std::atoi(argv[1])) : 6;
  const uint64_t prompts = argc > 2 ? uint64_t(std::atoll(argv[2])) : 1024;
  const DevResult d = run_device(iterations, prompts);
  const Result g = run(true, iterations, prompts);
  const Result c = run(false, std::max<uint32_t>(3, iterations / 2), prompts);
  std::printf("{\"bench\": \"cpp/bench_e2e (reference run_iteration + gpu_registry, host SampleBatches)\", "
              "\"workload\": \"C2: %llu prompts x 16 x UNIFORM[1,4096], logical dp8 -> actor_train dp4/tp2, 8 worker "
              "threads on GPU 0\", \"tokens\": %llu, \"gpu_hot_slice_ms\": %.3f, \"gpu_tokens_per_s\": %.1f, "
              "\"gpu_iteration_ms\": %.3f, \"cpu_hot_slice_ms\": %.3f, \"cpu_tokens_per_s\": %.1f, "
              "\"cpu_iteration_ms\": %.3f, \"speedup_hot_slice\": %.2f, \"device_chain_hot_slice_ms\": %.3f, "
              "\"device_chain_tokens_per_s\": %.1f, \"device_chain_upload_ms\": %.3f, "
              "\"device_chain_e2e_tokens_per_s\": %.1f, \"device_chain_loss\": %.9f}\n",
              (unsigned long long)prompts, (unsigned long long)g.tokens, g.hot_ms, g.tokens / (g.hot_ms / 1e3),
              g.iter_ms, c.hot_ms, c.tokens / (c.hot_ms / 1e3), c.iter_ms, c.hot_ms / g.hot_ms, d.hot_ms,
              g.tokens / (d.hot_ms / 1e3), d.upload_ms, g.tokens / ((d.hot_ms + d.upload_ms) / 1e3), d.loss);
  return 0;
}
