// dfx_device_chain.hpp -- the reference's operator API with device-resident batches end to end.
//
// The reference's runtime moves AoS SampleBatches (record.hpp:17-41) through a CPU BufferStore; with the GPU
// StageFns of dfx_distflow.hpp bound into it (gpu_registry()), every node re-packs its batch host->device and the
// CPU store copies every payload byte between stages -- cpp/bench_e2e measures that path (store-bound). This header
// keeps the same DAG vocabulary (NodeSpec / TaskChain / ParallelLayout / dispatch keys, preset_dag, the registry-
// bind errors, run_iteration's get -> invoke -> put -> worker_done loop of worker.hpp:208-258) over DEVICE batches:
//   DeviceStageFn      void(const NodeSpec&, dfx::DeviceBatch&, DeviceStageContext&) -- the StageFn of
//                      functions.hpp:63 with the batch on the GPU; the context carries the per-worker arena (the
//                      "new field" SURVEY §8(b) asks for) and the worker's stream
//   device_registry()  the hot-path nodes under the reference's keys (functions.hpp:201-219)
//   run_iteration_device  get from a dfx::DeviceBufferStore (include/dfx_store.hpp: the reference placement,
//                      zero-copy views or NVLink/HBM copies) -> invoke -> put, per node; the first node's batch is
//                      uploaded ONCE from the host SampleBatch (pinned staging, pooled device memory)
// Nothing allocates in a steady state (pooled device blocks, grow-only arenas) and no node re-packs AoS data.
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dfx_distflow.hpp"
#include "dfx_store.hpp"
#include "distflow/dag.hpp"

namespace dfx_distflow {

struct DeviceStageContext {
  double advantage_eps = 1e-6;           // StageContext::advantage_eps (functions.hpp:59)
  std::map<distflow::Role, uint64_t>* model_versions = nullptr;
  Arena* arena = nullptr;                // the worker's arena (stream, workspaces, staging)
  std::shared_ptr<dfx::DevicePool> pool; // device blocks for channels a node adds
  dfx_loss_out last_loss{};              // the actor loss of the last train call (the reference has no slot)
};
using DeviceStageFn = std::function<void(const distflow::NodeSpec&, dfx::DeviceBatch&, DeviceStageContext&)>;

class DeviceFunctionRegistry {
 public:
  void register_fn(const std::string& key, DeviceStageFn fn) {
    if (!fns_.emplace(key, std::move(fn)).second)
      throw distflow::Error("duplicate registration for key '" + key + "'");  // functions.hpp:187-189
  }
  const DeviceStageFn* find(const std::string& key) const {
    auto it = fns_.find(key);
    return it == fns_.end() ? nullptr : &it->second;
  }

 private:
  std::map<std::string, DeviceStageFn> fns_;
};

inline dfx_packed packed_of(const dfx::DeviceBatch& b) { return b.packed(); }

// a new f64 rollout channel on the batch's device from the pool (owned by the batch)
inline double* add_channel(dfx::DeviceBatch& b, const std::string& name, DeviceStageContext& ctx) {
  auto it = b.channels.find(name);
  if (it != b.channels.end()) return it->second;
  auto m = ctx.pool->get(b.device, sizeof(double) * size_t(b.n_rollouts) + 8);
  b.keep.push_back(m);
  double* p = reinterpret_cast<double*>(m.get());
  b.channels[name] = p;
  return p;
}

// fn_group_advantage (functions.hpp:143-161) on a device batch: bit-identical f64 channel "advantage"
inline void dev_group_advantage(const distflow::NodeSpec&, dfx::DeviceBatch& b, DeviceStageContext& ctx) {
  if (!b.channels.count("reward")) throw distflow::MissingChannelError("reward");
  double* adv = add_channel(b, "advantage", ctx);
  const dfx_packed p = packed_of(b);
  auto* flags = static_cast<int32_t*>(ctx.arena->device("flags", sizeof(int32_t)));
  cuda_check(cudaMemsetAsync(flags, 0, sizeof(int32_t), ctx.arena->stream), "memset");
  check(dfx_grpo_advantage(&p, ctx.advantage_eps, adv, flags, ctx.arena->stream));
  check(dfx_check_flags(flags, ctx.arena->stream));  // MissingRolloutsError, like require_rollouts
}

// fn_ppo_advantage (functions.hpp:163-172)
inline void dev_ppo_advantage(const distflow::NodeSpec&, dfx::DeviceBatch& b, DeviceStageContext& ctx) {
  if (!b.channels.count("reward")) throw distflow::MissingChannelError("reward");
  if (!b.channels.count("value")) throw distflow::MissingChannelError("value");
  double* adv = add_channel(b, "advantage", ctx);
  const dfx_packed p = packed_of(b);
  check(dfx_ppo_advantage(&p, adv, ctx.arena->stream));
}

// fn_train (functions.hpp:176-182): the fused clipped surrogate + KL over the batch's own token streams
inline void dev_train(const distflow::NodeSpec& node, dfx::DeviceBatch& b, DeviceStageContext& ctx) {
  if (node.role != distflow::Role::ACTOR && node.role != distflow::Role::CRITIC)
    throw distflow::Error("role " + std::string(distflow::to_string(node.role)) + " is frozen and cannot train");
  if (node.role == distflow::Role::ACTOR && b.n_rollouts > 0) {
    auto adv = b.channels.find("advantage");
    if (adv == b.channels.end()) throw distflow::MissingChannelError("advantage");
    const dfx_packed p = packed_of(b);
    const LossConfig& lc = loss_config();
    dfx_loss_cfg cfg{lc.clip_low, lc.clip_high, lc.beta, ctx.advantage_eps, lc.kl_type, lc.agg, DFX_ADV_ROLLOUT, 0};
    auto* out = static_cast<dfx_loss_out*>(ctx.arena->device("loss_out", sizeof(dfx_loss_out)));
    dfx_loss_args a{};
    a.adv_roll = adv->second;
    a.n_loss_groups = 1;
    a.out = out;
    const size_t ws = dfx_ppo_loss_workspace_bytes(b.n_rollouts, b.token_span, 1);
    check(dfx_ppo_loss(&p, b.token_base, b.token_span, &cfg, &a, ctx.arena->device("loss_ws", ws), ws,
                       ctx.arena->stream));
    auto* host = static_cast<dfx_loss_out*>(ctx.arena->pinned("loss_out", sizeof(dfx_loss_out)));
    cuda_check(cudaMemcpyAsync(host, out, sizeof(dfx_loss_out), cudaMemcpyDeviceToHost, ctx.arena->stream), "D2H");
    cuda_check(cudaStreamSynchronize(ctx.arena->stream), "sync");
    ctx.last_loss = *host;
  }
  if (ctx.model_versions) ++(*ctx.model_versions)[node.role];
}

inline DeviceFunctionRegistry device_registry() {
  DeviceFunctionRegistry reg;
  reg.register_fn("group_advantage", dev_group_advantage);
  reg.register_fn("ppo_advantage", dev_ppo_advantage);
  reg.register_fn("train_actor", dev_train);
  reg.register_fn("train_critic", dev_train);
  reg.register_fn("ACTOR/MODEL_TRAIN", dev_train);
  reg.register_fn("CRITIC/MODEL_TRAIN", dev_train);
  return reg;
}

struct DeviceBoundNode {
  distflow::NodeSpec spec;
  std::string key;
  DeviceStageFn fn;
  distflow::ParallelLayout layout;
};

// registry_bind (functions.hpp:234-249) for the device nodes of a chain slice
inline std::vector<DeviceBoundNode> device_registry_bind(const std::vector<distflow::NodeSpec>& nodes,
                                                         const DeviceFunctionRegistry& reg,
                                                         const std::map<std::string, distflow::ParallelLayout>& layouts) {
  std::vector<DeviceBoundNode> out;
  for (const auto& spec : nodes) {
    const std::string key = spec.dispatch_key();
    const DeviceStageFn* fn = reg.find(key);
    if (!fn) throw distflow::UnboundNodeError(spec.node_id, key);
    auto lit = layouts.find(spec.node_id);
    if (lit == layouts.end()) throw distflow::LayoutError("no layout for stage '" + spec.node_id + "'");
    out.push_back({spec, key, *fn, lit->second});
  }
  return out;
}

// Upload a host SampleBatch (the token-stream payload layout of dfx_distflow.hpp, and the named f64 channels)
// into pooled device memory on the calling thread's device: the chain's single host->device crossing.
inline dfx::DeviceBatch upload_batch(const distflow::SampleBatch& batch, const std::vector<std::string>& channels,
                                     DeviceStageContext& ctx) {
  Arena& ar = *ctx.arena;
  const DevicePacked d = pack(batch, PackOptions{channels, true}, ar);
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  dfx::DeviceBatch b;
  b.device = dev;
  b.n_records = d.n_records;
  b.n_rollouts = d.n_rollouts;
  b.token_base = 0;
  b.token_span = d.n_tokens;
  const size_t R = size_t(d.n_records), S = size_t(d.n_rollouts), T = size_t(d.n_tokens);
  auto take = [&](size_t bytes) {
    auto m = ctx.pool->get(dev, bytes + 64);
    b.keep.push_back(m);
    return m.get();
  };
  auto copy = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ar.stream), "D2D");
  };
  // the arena's staging arrays are reused by the next pack: move this batch into its own pooled blocks
  std::vector<uint64_t> ids(R);
  for (size_t r = 0; r < R; ++r) ids[r] = batch.records[r].sample_id;
  b.ids = reinterpret_cast<uint64_t*>(take(R * 8));
  cuda_check(cudaMemcpyAsync(b.ids, ids.data(), R * 8, cudaMemcpyHostToDevice, ar.stream), "H2D");
  b.group_off = reinterpret_cast<int32_t*>(take((R + 1) * 4));
  copy(b.group_off, d.view.group_off, (R + 1) * 4);
  b.roll_group = reinterpret_cast<int32_t*>(take(S * 4));
  copy(b.roll_group, d.view.roll_group, S * 4);
  b.cu = reinterpret_cast<int64_t*>(take((S + 1) * 8));
  copy(b.cu, d.view.cu_seqlens, (S + 1) * 8);
  for (const auto& [name, p] : d.ch) {
    double* c = reinterpret_cast<double*>(take(S * 8));
    copy(c, p, S * 8);
    b.channels[name] = c;
  }
  const std::pair<const char*, std::pair<const void*, size_t>> st[] = {
      {"lp", {d.view.lp, 4}}, {"old_lp", {d.view.old_lp, 4}}, {"ref_lp", {d.view.ref_lp, 4}}, {"mask", {d.view.mask, 1}}};
  for (const auto& [name, pe] : st) {
    uint8_t* m = static_cast<uint8_t*>(take((T + 16) * pe.second));
    copy(m, pe.first, T * pe.second);
    b.streams[name] = dfx::DeviceBatch::Stream{m, pe.second};
  }
  // host offsets (the store plans from them)
  b.h_group_off.assign(R + 1, 0);
  b.h_cu.assign(S + 1, 0);
  size_t s = 0;
  for (size_t r = 0; r < R; ++r) {
    for (const auto& ro : batch.records[r].rollouts) {
      b.h_cu[s + 1] = b.h_cu[s] + ro.token_count;
      ++s;
    }
    b.h_group_off[r + 1] = int32_t(s);
  }
  cuda_check(cudaStreamSynchronize(ar.stream), "sync");  // the batch is complete before it enters the store
  return b;
}

// run_iteration (worker.hpp:208-258) over device batches: node 0 consumes `first` (uploaded by the caller, e.g.
// upload_batch), node i > 0 gets the previous node's output from the device store under the previous node's id;
// every node's output is put back under its own id; TP != 0 puts are suppressed by the store like the reference's.
struct DeviceWorker {
  uint32_t rank = 0;
  std::vector<DeviceBoundNode> chain;
  dfx::DeviceBufferStore* store = nullptr;
  DeviceStageContext ctx;
};
inline void run_iteration_device(DeviceWorker& w, uint32_t iteration, const dfx::DeviceBatch* first) {
  for (size_t i = 0; i < w.chain.size(); ++i) {
    const DeviceBoundNode& bn = w.chain[i];
    const uint32_t dp = bn.layout.dp_rank(w.rank), tp = bn.layout.tp_rank(w.rank);
    dfx::DeviceBatch batch;
    if (i == 0) {
      if (!first) throw distflow::Error("first chain node requires a batch");
      batch = *first;
    } else {
      const auto& prev = w.chain[i - 1].spec.node_id;
      batch = w.store->get(prev, iteration, dp, dfx::Layout{bn.layout.dp_size, bn.layout.tp_size});
    }
    try {
      bn.fn(bn.spec, batch, w.ctx);
    } catch (const distflow::FunctionError&) {
      throw;
    } catch (const std::exception& e) {
      throw distflow::FunctionError(bn.spec.node_id, e.what());  // invoke_node (worker.hpp:192-200)
    }
    if (i + 1 < w.chain.size()) {
      cuda_check(cudaStreamSynchronize(w.ctx.arena->stream), "sync");  // complete before the store copies it
      w.store->put(bn.spec.node_id, iteration, dp, tp, std::move(batch));
    }
  }
  w.store->worker_done(iteration);
}

}  // namespace dfx_distflow
