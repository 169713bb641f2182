// test_shims.cpp -- the C++ drop-in (include/dfx_distflow.hpp) inside the reference's own runtime.
//
// Built here against the unmodified reference headers (cpp/Makefile), run on the GPU box by
// tests/test_cpp_shims.py. Checks, printing "PASS <name>" per check and exiting non-zero on failure:
//   1. gpu_group_advantage == fn_group_advantage bit for bit (functions.hpp:143-161) on generated batches
//   2. the reference's exception types: MissingRolloutsError, MissingChannelError, frozen-role Error
//   3. registry_bind(preset chain, gpu_registry(), layouts) + run_iteration (worker.hpp:208-258) over
//      BufferStore/InprocFabric with one thread per worker: the captured final records equal those of the same
//      run with builtin_registry(), byte for byte (GRPO 1x4 dp2->dp2/tp2 and PPO 2x2)
//   4. gpu_train's fused loss on token-stream payloads equals the oracle's f64 loss within 1e-5
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <thread>

#include "distflow/dag.hpp"
#include "distflow/planner.hpp"
#include "distflow/worker.hpp"
#include "dfx_distflow.hpp"
#include "../oracle/dfx_oracle.h"

using namespace distflow;

static int failures = 0;
#define CHECK(cond, name)                                              \
  do {                                                                 \
    if (cond) {                                                        \
      std::printf("PASS %s\n", name);                                  \
    } else {                                                           \
      std::printf("FAIL %s (%s:%d)\n", name, __FILE__, __LINE__);      \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static NodeSpec compute_node() {
  NodeSpec n;
  n.node_id = "adv";
  return n;
}

static SampleBatch generated(uint64_t seed, uint32_t n_records, uint32_t n_roll, uint32_t lo, uint32_t hi) {
  StageContext ctx;
  ctx.run_seed = seed;
  ctx.gen.rollouts_per_prompt = n_roll;
  ctx.gen.response_tokens.kind = TokenDist::Kind::UNIFORM;
  ctx.gen.response_tokens.min = lo;
  ctx.gen.response_tokens.max = hi;
  ctx.gen.bytes_per_token = 0;
  SampleBatch b;
  for (uint32_t i = 0; i < n_records; ++i) {
    SampleRecord r;
    r.sample_id = 1000 + i;
    b.records.push_back(r);
  }
  fn_generate(compute_node(), b, ctx);
  fn_reward(compute_node(), b, ctx);
  fn_value(compute_node(), b, ctx);
  return b;
}

static void test_advantage() {
  for (uint64_t seed : {1ull, 7ull, 11ull}) {
    SampleBatch a = generated(seed, 300, 16, 1, 4096), b = a;
    StageContext ctx;
    fn_group_advantage(compute_node(), a, ctx);
    dfx_distflow::gpu_group_advantage(compute_node(), b, ctx);
    CHECK(serialize_batch(a) == serialize_batch(b), "gpu_group_advantage bit-exact vs fn_group_advantage");
    SampleBatch c = generated(seed, 100, 3, 1, 8), d = c;
    fn_ppo_advantage(compute_node(), c, ctx);
    dfx_distflow::gpu_ppo_advantage(compute_node(), d, ctx);
    CHECK(serialize_batch(c) == serialize_batch(d), "gpu_ppo_advantage bit-exact vs fn_ppo_advantage");
  }
  // tests/test_functions.cpp:134-155 KATs
  SampleBatch k;
  SampleRecord r;
  for (double x : {1.0, 0.0, 1.0, 0.0}) {
    Rollout ro;
    ro.channels["reward"] = x;
    r.rollouts.push_back(ro);
  }
  k.records.push_back(r);
  StageContext z;
  z.advantage_eps = 0.0;
  dfx_distflow::gpu_group_advantage(compute_node(), k, z);
  CHECK(k.records[0].rollouts[0].channels.at("advantage") == 1.0 &&
            k.records[0].rollouts[1].channels.at("advantage") == -1.0,
        "KAT [1,0,1,0] eps 0 -> [1,-1,1,-1]");
}

static void test_errors() {
  StageContext ctx;
  SampleBatch empty;
  empty.records.push_back(SampleRecord{});
  bool ok = false;
  try {
    dfx_distflow::gpu_group_advantage(compute_node(), empty, ctx);
  } catch (const MissingRolloutsError&) {
    ok = true;
  }
  CHECK(ok, "MissingRolloutsError for a record without rollouts");
  SampleBatch nov = generated(3, 2, 2, 4, 8);
  for (auto& rec : nov.records)
    for (auto& ro : rec.rollouts) ro.channels.erase("value");
  ok = false;
  try {
    dfx_distflow::gpu_ppo_advantage(compute_node(), nov, ctx);
  } catch (const MissingChannelError& e) {
    ok = e.channel == "value";
  }
  CHECK(ok, "MissingChannelError('value') for ppo_advantage");
  NodeSpec frozen;
  frozen.node_id = "r";
  frozen.role = Role::REWARD;
  frozen.node_type = NodeType::MODEL_TRAIN;
  ok = false;
  try {
    dfx_distflow::gpu_train(frozen, nov, ctx);
  } catch (const Error&) {
    ok = true;
  }
  CHECK(ok, "frozen role cannot train");
}

// ---- whole chain through the reference worker loop ----------------------------------------------------
static std::vector<uint8_t> run_chain(Algorithm algo, ClusterTopology topo,
                                      std::map<std::string, ParallelLayout> layouts, const FunctionRegistry& reg,
                                      uint64_t global_batch, uint32_t iterations) {
  const TaskChain chain = serialize_graph(preset_dag(algo));
  InprocFabric fabric(topo);
  std::map<std::string, StoreStagePlan> stages;
  for (size_t i = 0; i < chain.nodes.size(); ++i) {
    StoreStagePlan p;
    p.produced = layouts.at(chain.nodes[i].node_id);
    if (i + 1 < chain.nodes.size()) p.consumed = layouts.at(chain.nodes[i + 1].node_id);
    p.tag = tags::kRedistBase + uint32_t(i);
    stages[chain.nodes[i].node_id] = p;
  }
  std::vector<std::unique_ptr<BufferStore>> stores;
  for (uint32_t b = 0; b < topo.num_nodes; ++b)
    stores.push_back(std::make_unique<BufferStore>(topo, b, &fabric, stages));
  CaptureSink sink;
  std::vector<std::thread> threads;
  std::mutex mu;
  std::string err;
  for (uint32_t rk = 0; rk < topo.world_size(); ++rk) {
    threads.emplace_back([&, rk] {
      try {
        WorkerState st;
        st.rank = rk;
        st.topo = topo;
        st.chain = registry_bind(chain, reg, layouts);
        st.store = stores[topo.node_of(rk)].get();
        st.fabric = &fabric;
        st.capture = &sink;
        st.global_batch = global_batch;
        st.ctx.gen.rollouts_per_prompt = 4;
        st.ctx.gen.response_tokens.kind = TokenDist::Kind::UNIFORM;
        st.ctx.gen.response_tokens.min = 8;
        st.ctx.gen.response_tokens.max = 40;
        st.ctx.cost = CostModel{0, 0, 0, 0, 0, 0};
        st.init(21);
        const ParallelLayout& g = st.chain.nodes.front().layout;
        DatasetSpec spec;
        spec.synthetic_n = global_batch;
        st.loader = make_group_loader(spec, g, g.dp_rank(rk), 21);
        for (uint32_t it = 0; it < iterations; ++it) run_iteration(st, it);
      } catch (const std::exception& e) {
        std::lock_guard lk(mu);
        if (err.empty()) err = e.what();
      }
    });
  }
  for (auto& t : threads) t.join();
  if (!err.empty()) {
    std::printf("chain error: %s\n", err.c_str());
    return {};
  }
  std::vector<uint8_t> all;
  for (auto& [it, recs] : sink.take()) {
    std::sort(recs.begin(), recs.end(), [](const SampleRecord& a, const SampleRecord& b) {
      return a.sample_id < b.sample_id;
    });
    auto blob = serialize_records(recs);
    all.insert(all.end(), blob.begin(), blob.end());
  }
  return all;
}

static void test_chain() {
  {
    std::map<std::string, ParallelLayout> l;
    const TaskChain c = serialize_graph(preset_dag(Algorithm::GRPO));
    for (const auto& n : c.nodes) l[n.node_id] = ParallelLayout{4, 1};
    l["actor_train"] = ParallelLayout{2, 2};  // configs/grpo_small.json:7-8
    const auto a = run_chain(Algorithm::GRPO, ClusterTopology{1, 4}, l, builtin_registry(), 16, 3);
    const auto b = run_chain(Algorithm::GRPO, ClusterTopology{1, 4}, l, dfx_distflow::gpu_registry(), 16, 3);
    CHECK(!a.empty() && a == b, "GRPO 1x4 run_iteration: gpu_registry captures == builtin_registry captures");
  }
  {
    std::map<std::string, ParallelLayout> l;
    const TaskChain c = serialize_graph(preset_dag(Algorithm::PPO));
    for (const auto& n : c.nodes) l[n.node_id] = ParallelLayout{2, 2};  // configs/ppo_cross.json
    const auto a = run_chain(Algorithm::PPO, ClusterTopology{2, 2}, l, builtin_registry(), 16, 3);
    const auto b = run_chain(Algorithm::PPO, ClusterTopology{2, 2}, l, dfx_distflow::gpu_registry(), 16, 3);
    CHECK(!a.empty() && a == b, "PPO 2x2 run_iteration: gpu_registry captures == builtin_registry captures");
  }
}

// ---- fused loss on token-stream payloads -------------------------------------------------------------
static void test_loss() {
  const uint32_t R = 40, n = 4;
  std::vector<uint64_t> ids(R);
  for (uint32_t i = 0; i < R; ++i) ids[i] = i;
  dfo_token_dist dist{DFO_UNIFORM, 0, 1, 700};
  std::vector<int64_t> cu(R * n + 1);
  dfo_synth_lengths(&dist, 5, ids.data(), R, n, cu.data());
  const int64_t T = cu.back();
  std::vector<float> lp(T + 16), old(T + 16), ref(T + 16);
  std::vector<uint8_t> mask(T + 16);
  std::vector<int32_t> tid(T + 16);
  std::vector<double> reward(R * n), value(R * n);
  dfo_synth_tokens(5, ids.data(), R, n, cu.data(), lp.data(), old.data(), ref.data(), nullptr, nullptr, mask.data(),
                   tid.data(), 1);
  dfo_synth_rollout_scalars(5, ids.data(), R, n, reward.data(), value.data());
  std::vector<int32_t> go(R + 1);
  for (uint32_t r = 0; r <= R; ++r) go[r] = int32_t(r * n);
  std::vector<double> adv(R * n);
  dfo_grpo_advantage(R, go.data(), reward.data(), 1e-6, adv.data());
  SampleBatch b;
  for (uint32_t r = 0; r < R; ++r) {
    SampleRecord rec;
    rec.sample_id = r;
    for (uint32_t j = 0; j < n; ++j) {
      const int64_t s = r * n + j, a = cu[s], L = cu[s + 1] - a;
      Rollout ro;
      ro.token_count = uint32_t(L);
      ro.payload.resize(size_t(L) * 17);
      uint8_t* p = ro.payload.data();
      std::memcpy(p, tid.data() + a, 4 * L);
      std::memcpy(p + 4 * L, lp.data() + a, 4 * L);
      std::memcpy(p + 8 * L, old.data() + a, 4 * L);
      std::memcpy(p + 12 * L, ref.data() + a, 4 * L);
      std::memcpy(p + 16 * L, mask.data() + a, L);
      ro.channels["reward"] = reward[s];
      ro.channels["advantage"] = adv[s];
      rec.rollouts.push_back(ro);
    }
    b.records.push_back(rec);
  }
  NodeSpec train;
  train.node_id = "actor_train";
  train.role = Role::ACTOR;
  train.node_type = NodeType::MODEL_TRAIN;
  std::map<Role, uint64_t> versions;
  StageContext ctx;
  ctx.model_versions = &versions;
  dfx_distflow::gpu_train(train, b, ctx);
  const dfx_loss_out got = dfx_distflow::last_loss();
  std::vector<float> adv_tok(T + 16);
  dfo_broadcast_advantage(R * n, cu.data(), adv.data(), mask.data(), adv_tok.data());
  dfo_loss_cfg cfg{0.2, 0.2, 0.001, DFO_KL_K3, DFO_AGG_TOKEN_MEAN, 0, 0};
  dfo_loss_out ref_out{};
  dfo_ppo_loss(R * n, cu.data(), lp.data(), old.data(), ref.data(), adv_tok.data(), mask.data(), &cfg, &ref_out,
               nullptr);
  CHECK(got.n_tokens == ref_out.n_tokens, "gpu_train token count == oracle");
  CHECK(std::fabs(got.loss - ref_out.loss) <= 1e-5 * std::max(std::fabs(ref_out.loss), 1.0),
        "gpu_train loss == oracle within 1e-5");
  CHECK(versions[Role::ACTOR] == 1, "gpu_train bumps the ACTOR model version");
}

int main() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    std::printf("SKIP no CUDA device\n");
    return 0;
  }
  test_advantage();
  test_errors();
  test_chain();
  test_loss();
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASSED", failures);
  return failures ? 1 : 0;
}
