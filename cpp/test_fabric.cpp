// test_fabric.cpp -- the NCCL-backed Fabric (include/dfx_fabric.hpp) under the reference's own runtime in its
// fork-per-node process model (runner.hpp:655-742): one process per node (B = 2), each with its GPU, its
// BufferStore(topo, node, &fabric) and one thread per local worker running run_iteration (worker.hpp:208-258).
// The captured final records of both processes, merged, must equal byte for byte those of the same run in ONE
// process over InprocFabric (the reference's own backend), and the cross-node traffic counters must agree.
// Prints "PASS <name>" per check; exits non-zero on failure. Needs 2 GPUs (skips otherwise).
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <thread>

#include "distflow/dag.hpp"
#include "distflow/planner.hpp"
#include "distflow/worker.hpp"
#include "dfx_fabric.hpp"

using namespace distflow;

namespace {

struct Config {
  const char* name;
  Algorithm algo;
  std::map<std::string, ParallelLayout> layouts;
};

std::map<std::string, StoreStagePlan> stage_plans(const TaskChain& chain, const std::map<std::string, ParallelLayout>& l) {
  std::map<std::string, StoreStagePlan> stages;
  for (size_t i = 0; i < chain.nodes.size(); ++i) {
    StoreStagePlan p;
    p.produced = l.at(chain.nodes[i].node_id);
    if (i + 1 < chain.nodes.size()) p.consumed = l.at(chain.nodes[i + 1].node_id);
    p.tag = tags::kRedistBase + uint32_t(i);
    stages[chain.nodes[i].node_id] = p;
  }
  return stages;
}

// run the workers of `nodes` (all, or one node) over `fabric`; returns the captured records
std::vector<SampleRecord> run_workers(const Config& cfg, const ClusterTopology& topo, Fabric& fabric,
                                      const std::vector<uint32_t>& nodes, uint32_t iterations) {
  const TaskChain chain = serialize_graph(preset_dag(cfg.algo));
  const auto stages = stage_plans(chain, cfg.layouts);
  std::vector<std::unique_ptr<BufferStore>> stores;
  for (uint32_t b : nodes) stores.push_back(std::make_unique<BufferStore>(topo, b, &fabric, stages));
  CaptureSink sink;
  std::vector<std::thread> threads;
  std::mutex mu;
  std::string err;
  const FunctionRegistry reg = builtin_registry();
  for (size_t k = 0; k < nodes.size(); ++k) {
    for (uint32_t w = 0; w < topo.workers_per_node; ++w) {
      const uint32_t rk = nodes[k] * topo.workers_per_node + w;
      BufferStore* store = stores[k].get();
      threads.emplace_back([&, rk, store] {
        try {
          WorkerState st;
          st.rank = rk;
          st.topo = topo;
          st.chain = registry_bind(chain, reg, cfg.layouts);
          st.store = store;
          st.fabric = &fabric;
          st.capture = &sink;
          st.global_batch = 16;
          st.ctx.gen.rollouts_per_prompt = 4;
          st.ctx.gen.response_tokens.kind = TokenDist::Kind::UNIFORM;
          st.ctx.gen.response_tokens.min = 8;
          st.ctx.gen.response_tokens.max = 40;
          st.ctx.gen.bytes_per_token = 2;
          st.ctx.cost = CostModel{0, 0, 0, 0, 0, 0};
          st.init(21);
          const ParallelLayout& g = st.chain.nodes.front().layout;
          DatasetSpec spec;
          spec.synthetic_n = 16;
          st.loader = make_group_loader(spec, g, g.dp_rank(rk), 21);
          for (uint32_t it = 0; it < iterations; ++it) run_iteration(st, it);
        } catch (const std::exception& e) {
          std::lock_guard lk(mu);
          if (err.empty()) err = e.what();
        }
      });
    }
  }
  for (auto& t : threads) t.join();
  if (!err.empty()) throw Error("chain: " + err);
  std::vector<SampleRecord> all;
  for (auto& [it, recs] : sink.take())
    for (auto& r : recs) all.push_back(std::move(r));
  return all;
}

std::vector<uint8_t> canonical(std::vector<SampleRecord> recs) {
  std::sort(recs.begin(), recs.end(), [](const SampleRecord& a, const SampleRecord& b) { return a.sample_id < b.sample_id; });
  return serialize_records(recs);
}

}  // namespace

int main() {
  // (no CUDA call in this process before the forks: a CUDA context does not survive fork)
  const ClusterTopology topo{2, 2};
  std::vector<Config> cfgs;
  {
    Config c{"PPO 2x2 dp2/tp2", Algorithm::PPO, {}};
    for (const auto& n : serialize_graph(preset_dag(c.algo)).nodes) c.layouts[n.node_id] = ParallelLayout{2, 2};
    cfgs.push_back(c);
  }
  {
    Config c{"GRPO 2x2 dp4 -> actor_train dp2/tp2 (cross-node exchange)", Algorithm::GRPO, {}};
    for (const auto& n : serialize_graph(preset_dag(c.algo)).nodes) c.layouts[n.node_id] = ParallelLayout{4, 1};
    c.layouts["actor_train"] = ParallelLayout{2, 2};
    cfgs.push_back(c);
  }
  int failures = 0;
  for (const Config& cfg : cfgs) {
    const uint32_t iterations = 3;
    // the reference backend, one process
    std::vector<uint8_t> want;
    uint64_t want_egress = 0;
    {
      InprocFabric inproc(topo);
      want = canonical(run_workers(cfg, topo, inproc, {0, 1}, iterations));
      want_egress = inproc.traffic().total_egress();
    }
    // fork per node over the NCCL fabric
    int id_pipe[2], res_pipe[2][2];
    if (pipe(id_pipe) || pipe(res_pipe[0]) || pipe(res_pipe[1])) return 1;
    std::vector<pid_t> kids;
    for (uint32_t node = 0; node < 2; ++node) {
      const pid_t pid = fork();
      if (pid == 0) {
        std::vector<uint8_t> blob;
        uint64_t egress = 0, rounds = 0;
        int ok = 1;
        try {
          int avail = 0;
          if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 2) {
            const uint64_t hdr[4] = {2, 0, 0, 0};  // skip
            if (write(res_pipe[node][1], hdr, sizeof(hdr)) != ssize_t(sizeof(hdr))) _exit(3);
            _exit(0);
          }
          dfx::store_cuda(cudaSetDevice(int(node)), "cudaSetDevice");
          std::array<char, DFX_COMM_ID_BYTES> id{};
          if (node == 0) {
            id = dfx::Comm::unique_id();
            if (write(id_pipe[1], id.data(), id.size()) != ssize_t(id.size())) _exit(2);
          } else if (read(id_pipe[0], id.data(), id.size()) != ssize_t(id.size())) {
            _exit(2);
          }
          dfx::Comm comm(2, int32_t(node), id);
          dfx_distflow::NcclFabric fabric(topo, node, comm);
          blob = serialize_records(run_workers(cfg, topo, fabric, {node}, iterations));
          egress = fabric.traffic().node_egress[node];
          fabric.close();
          rounds = fabric.rounds();
        } catch (const std::exception& ex) {
          std::fprintf(stderr, "node %u: %s\n", node, ex.what());
          ok = 0;
        }
        const uint64_t hdr[4] = {uint64_t(ok), blob.size(), egress, rounds};
        if (write(res_pipe[node][1], hdr, sizeof(hdr)) != ssize_t(sizeof(hdr))) _exit(3);
        size_t off = 0;
        while (off < blob.size()) {
          const ssize_t w = write(res_pipe[node][1], blob.data() + off, blob.size() - off);
          if (w <= 0) _exit(3);
          off += size_t(w);
        }
        _exit(ok ? 0 : 1);
      }
      kids.push_back(pid);
    }
    std::vector<SampleRecord> merged;
    uint64_t egress = 0, rounds = 0;
    bool ok = true, skip = false;
    for (uint32_t node = 0; node < 2; ++node) {
      uint64_t hdr[4] = {0, 0, 0, 0};
      if (read(res_pipe[node][0], hdr, sizeof(hdr)) != ssize_t(sizeof(hdr))) ok = false;
      std::vector<uint8_t> blob(hdr[1]);
      size_t off = 0;
      while (off < blob.size()) {
        const ssize_t r = read(res_pipe[node][0], blob.data() + off, blob.size() - off);
        if (r <= 0) break;
        off += size_t(r);
      }
      skip = skip || hdr[0] == 2;
      ok = ok && hdr[0] == 1;
      egress += hdr[2];
      rounds += hdr[3];
      if (!blob.empty()) {
        auto recs = deserialize_records(blob);
        for (auto& r : recs) merged.push_back(std::move(r));
      }
    }
    for (pid_t k : kids) {
      int status = 0;
      waitpid(k, &status, 0);
      ok = ok && WIFEXITED(status) && WEXITSTATUS(status) == 0;
    }
    if (skip) {  // (node 0 may block on the id pipe if node 1 skipped first: both skip on the same count)
      std::printf("SKIP test_fabric: needs 2 GPUs\n");
      return 0;
    }
    const bool same = ok && canonical(merged) == want && !want.empty();
    std::printf("%s %s: fork-per-node NcclFabric captures == InprocFabric captures (%zu bytes, %llu rounds)\n",
                same ? "PASS" : "FAIL", cfg.name, want.size(), (unsigned long long)rounds);
    failures += same ? 0 : 1;
    const bool traffic = ok && egress == want_egress;
    std::printf("%s %s: cross-node framed bytes %llu == reference %llu\n", traffic ? "PASS" : "FAIL", cfg.name,
                (unsigned long long)egress, (unsigned long long)want_egress);
    failures += traffic ? 0 : 1;
  }
  return failures ? 1 : 0;
}
