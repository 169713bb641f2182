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
//   5. dfx::DeviceBufferStore (include/dfx_store.hpp) == the reference BufferStore + InprocFabric: for several
//      (B, W, produced, consumed) layouts, every destination group's batch -- read on every GPU that hosts one of
//      its TP workers, by one thread per worker -- serializes to the same bytes as the reference get()
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <thread>

#include "distflow/dag.hpp"
#include "distflow/planner.hpp"
#include "distflow/worker.hpp"
#include "dfx_distflow.hpp"
#include "dfx_store.hpp"
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

// gpu_generate (device draw_tokens + hash_bytes) == fn_generate, payload bytes included; same errors
static void test_generate() {
  for (int kind = 0; kind < 2; ++kind) {
    StageContext ctx;
    ctx.run_seed = 17;
    ctx.gen.rollouts_per_prompt = 5;
    ctx.gen.response_tokens.kind = kind ? TokenDist::Kind::UNIFORM : TokenDist::Kind::CONSTANT;
    ctx.gen.response_tokens.value = 37;
    ctx.gen.response_tokens.min = 1;
    ctx.gen.response_tokens.max = 300;
    ctx.gen.bytes_per_token = 3;
    SampleBatch a, b;
    for (uint32_t i = 0; i < 64; ++i) {
      SampleRecord r;
      r.sample_id = 77 + 13 * i;
      a.records.push_back(r);
    }
    b = a;
    fn_generate(compute_node(), a, ctx);
    dfx_distflow::gpu_generate(compute_node(), b, ctx);
    CHECK(serialize_batch(a) == serialize_batch(b), kind ? "gpu_generate (UNIFORM) bit-exact vs fn_generate"
                                                          : "gpu_generate (CONSTANT) bit-exact vs fn_generate");
  }
  StageContext bad;
  bad.gen.response_tokens.kind = TokenDist::Kind::UNIFORM;
  bad.gen.response_tokens.min = 9;
  bad.gen.response_tokens.max = 8;
  SampleBatch one;
  one.records.push_back(SampleRecord{});
  bool threw = false;
  try {
    dfx_distflow::gpu_generate(compute_node(), one, bad);
  } catch (const Error&) {
    threw = true;
  }
  CHECK(threw, "gpu_generate: max < min throws like fn_generate");
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

// ---- 5. device DataBuffer vs the reference BufferStore ---------------------------------------------------------
static const char* kStreamOrder[5] = {"token_id", "lp", "old_lp", "ref_lp", "mask"};  // payload layout, 17 B/token
static const size_t kStreamElem[5] = {4, 4, 4, 4, 1};

static std::vector<SampleRecord> store_records(uint32_t G) {
  std::vector<SampleRecord> recs;
  for (uint32_t i = 0; i < G; ++i) {
    SampleRecord r;
    r.sample_id = 7000 + i;
    const uint32_t nr = 1 + i % 3;
    for (uint32_t j = 0; j < nr; ++j) {
      Rollout ro;
      ro.token_count = (i * 37 + j * 11) % 50;
      ro.payload.resize(size_t(ro.token_count) * 17);
      for (size_t k = 0; k < ro.payload.size(); ++k) ro.payload[k] = uint8_t((i * 131 + j * 17 + k * 7) & 0xff);
      ro.channels["reward"] = i + 0.25 * j;
      ro.channels["advantage"] = -double(i) - 0.5 * j;
      r.rollouts.push_back(ro);
    }
    recs.push_back(r);
  }
  return recs;
}

static dfx::DeviceBatch upload_records(int dev, const std::vector<SampleRecord>& recs) {
  std::vector<uint64_t> ids;
  std::vector<int32_t> go{0};
  std::vector<int64_t> cu{0};
  std::map<std::string, std::vector<double>> ch;
  std::map<std::string, std::pair<std::vector<uint8_t>, size_t>> st;
  for (int k = 0; k < 5; ++k) st[kStreamOrder[k]].second = kStreamElem[k];
  for (const auto& r : recs) {
    ids.push_back(r.sample_id);
    for (const auto& ro : r.rollouts) {
      const size_t L = ro.token_count;
      size_t off = 0;
      for (int k = 0; k < 5; ++k) {
        auto& v = st[kStreamOrder[k]].first;
        v.insert(v.end(), ro.payload.begin() + off, ro.payload.begin() + off + L * kStreamElem[k]);
        off += L * kStreamElem[k];
      }
      for (const auto& [n, x] : ro.channels) ch[n].push_back(x);
      cu.push_back(cu.back() + int64_t(L));
    }
    go.push_back(int32_t(cu.size() - 1));
  }
  return dfx::DeviceBatch::upload(dev, ids, go, cu, ch, st);
}

static std::vector<SampleRecord> download_records(const dfx::DeviceBatch& b) {
  auto d2h = [](const void* p, size_t bytes) {
    std::vector<uint8_t> v(bytes);
    if (bytes) dfx::store_cuda(cudaMemcpy(v.data(), p, bytes, cudaMemcpyDeviceToHost), "D2H");
    return v;
  };
  const auto ids = d2h(b.ids, size_t(b.n_records) * 8);
  const auto cu = d2h(b.cu, size_t(b.n_rollouts + 1) * 8);
  const auto go = d2h(b.group_off, size_t(b.n_records + 1) * 4);
  std::map<std::string, std::vector<uint8_t>> ch, st;
  for (const auto& [n, p] : b.channels) ch[n] = d2h(p, size_t(b.n_rollouts) * 8);
  for (const auto& [n, s] : b.streams) st[n] = d2h(s.base, size_t(b.token_base + b.token_span) * s.elem);
  std::vector<SampleRecord> out;
  const int64_t* c = reinterpret_cast<const int64_t*>(cu.data());
  const int32_t* g = reinterpret_cast<const int32_t*>(go.data());
  for (int64_t r = 0; r < b.n_records; ++r) {
    SampleRecord rec;
    std::memcpy(&rec.sample_id, ids.data() + 8 * r, 8);
    for (int32_t s = g[r]; s < g[r + 1]; ++s) {
      Rollout ro;
      ro.token_count = uint32_t(c[s + 1] - c[s]);
      for (int k = 0; k < 5; ++k) {
        const auto& v = st.at(kStreamOrder[k]);
        ro.payload.insert(ro.payload.end(), v.begin() + c[s] * int64_t(kStreamElem[k]),
                          v.begin() + c[s + 1] * int64_t(kStreamElem[k]));
      }
      for (const auto& [n, v] : ch) {
        double x;
        std::memcpy(&x, v.data() + 8 * s, 8);
        ro.channels[n] = x;
      }
      rec.rollouts.push_back(ro);
    }
    out.push_back(rec);
  }
  return out;
}

static void test_device_store() {
  int n_gpu = 0;
  cudaGetDeviceCount(&n_gpu);
  struct Cfg {
    uint32_t B, W, dp_p, tp_p, dp_c, tp_c, G;
  };
  const Cfg cfgs[] = {{1, 4, 4, 1, 2, 2, 24}, {1, 8, 8, 1, 4, 2, 64}, {2, 2, 4, 1, 2, 2, 16},
                      {2, 4, 2, 4, 8, 1, 32}, {2, 4, 8, 1, 2, 4, 48}, {1, 4, 2, 2, 4, 1, 20}};
  for (const Cfg& c : cfgs) {
    const auto recs = store_records(c.G);
    const ClusterTopology topo{c.B, c.W};
    const ParallelLayout produced{c.dp_p, c.tp_p}, consumed{c.dp_c, c.tp_c};
    // the reference: B stores over one InprocFabric
    InprocFabric fabric(topo);
    std::map<std::string, StoreStagePlan> stages;
    stages["s"] = StoreStagePlan{produced, consumed, tags::kRedistBase};
    std::vector<std::unique_ptr<BufferStore>> stores;
    std::vector<BufferStore*> ptrs;
    for (uint32_t b = 0; b < c.B; ++b) {
      stores.push_back(std::make_unique<BufferStore>(topo, b, &fabric, stages));
      ptrs.push_back(stores.back().get());
    }
    // the device store: logical worker w on GPU w * n_gpu / (B W)
    const uint32_t world = c.B * c.W;
    std::vector<int> gpu(world);
    for (uint32_t w = 0; w < world; ++w) gpu[w] = int(uint64_t(w) * uint64_t(n_gpu) / world);
    std::map<std::string, dfx::StagePlan> dstages;
    dstages["s"] = dfx::StagePlan{{c.dp_p, c.tp_p}, true, {c.dp_c, c.tp_c}};
    dfx::DeviceBufferStore dstore(c.B, c.W, gpu, dstages);
    const uint32_t per = c.G / c.dp_p;
    for (uint32_t p = 0; p < c.dp_p; ++p) {
      SampleBatch batch;
      batch.stage_id = "s";
      batch.records.assign(recs.begin() + p * per, recs.begin() + (p + 1) * per);
      const uint32_t lead = produced.group_lead(p);
      const dfx::DeviceBatch db = upload_records(gpu[lead], batch.records);
      for (uint32_t t = 0; t < c.tp_p; ++t) {
        stores[topo.node_of(lead)]->put("s", 0, p, t, batch);
        dstore.put("s", 0, p, t, db);
      }
    }
    redistribute(ptrs, "s", 0, consumed);
    // one thread per logical worker reads its consumer group on its GPU (SPMD, like run_iteration)
    std::vector<std::vector<uint8_t>> got(world);
    std::vector<std::string> errs(world);
    std::vector<std::thread> th;
    for (uint32_t w = 0; w < world; ++w)
      th.emplace_back([&, w] {
        try {
          cudaSetDevice(gpu[w]);
          const dfx::DeviceBatch b = dstore.get("s", 0, consumed.dp_rank(w), dfx::Layout{c.dp_c, c.tp_c});
          got[w] = serialize_records(download_records(b));
          dstore.worker_done(0);
        } catch (const std::exception& e) {
          errs[w] = e.what();
        }
      });
    for (auto& t : th) t.join();
    bool ok = true;
    for (uint32_t w = 0; w < world; ++w) {
      if (!errs[w].empty()) {
        std::printf("  worker %u: %s\n", w, errs[w].c_str());
        ok = false;
        continue;
      }
      const uint32_t d = consumed.dp_rank(w);
      const SampleBatch want = stores[topo.node_of(consumed.group_lead(d))]->get("s", 0, d, consumed);
      ok = ok && got[w] == serialize_records(want.records);
    }
    ok = ok && dstore.suppressed_count() == uint64_t(c.dp_p) * (c.tp_p - 1);
    char name[160];
    std::snprintf(name, sizeof(name), "device store == reference BufferStore (B%u W%u dp%u tp%u -> dp%u tp%u, %d GPU)",
                  c.B, c.W, c.dp_p, c.tp_p, c.dp_c, c.tp_c, n_gpu);
    CHECK(ok, name);
  }
  // semantics: stale puts / gets and NotReadyError, as the reference
  std::map<std::string, dfx::StagePlan> st1;
  st1["s"] = dfx::StagePlan{{2, 1}, true, {1, 2}};
  dfx::DeviceBufferStore s1(1, 2, {0, 0}, st1);
  bool not_ready = false, stale = false, unknown = false;
  try {
    s1.ensure_ready("s", 0, dfx::Layout{1, 2}, std::chrono::milliseconds(20));
  } catch (const dfx::StoreError& e) {
    not_ready = e.code == DFX_NOT_READY;
  }
  s1.worker_done(0);
  s1.worker_done(0);
  try {
    s1.put("s", 0, 0, 0, upload_records(0, store_records(2)));
  } catch (const dfx::StoreError& e) {
    stale = e.code == DFX_STALE_ITERATION;
  }
  try {
    s1.put("nope", 1, 0, 0, upload_records(0, store_records(2)));
  } catch (const dfx::StoreError& e) {
    unknown = e.code == DFX_UNKNOWN_STAGE;
  }
  CHECK(not_ready && stale && unknown, "device store errors: NotReady / StaleIteration / UnknownStage");
}

int main() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    std::printf("SKIP no CUDA device\n");
    return 0;
  }
  test_advantage();
  test_generate();
  test_errors();
  test_chain();
  test_loss();
  test_device_store();
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASSED", failures);
  return failures ? 1 : 0;
}
