// dfx_distflow.hpp -- drop-in GPU stage functions for the DistFlow simulator's operator API.
//
// Header-only C++20 shim over the C ABI in dfx.h. It includes the reference's own headers
// (distflow/functions.hpp, record.hpp, errors.hpp, add -I<reference>/proj/include) and provides StageFns with
// exactly the reference signature (distflow/functions.hpp:63)
//     void(const NodeSpec&, SampleBatch&, StageContext&)
// registered under the reference's registry keys (functions.hpp:201-219), so a DAG from preset_dag binds to
// them unchanged via registry_bind (functions.hpp:234-249) and runs inside run_iteration (worker.hpp:208-258).
// Errors surface as the reference's exception types (errors.hpp): a dfx_status is rethrown as
// MissingChannelError / MissingRolloutsError / IndivisibleError / LayoutError / Error, so invoke_node's wrapping
// (worker.hpp:192-200) behaves identically.
//
// Packing: a SampleBatch (AoS, std::map channels) is packed into the device SoA layout (dfx_packed) per call
// and results are written back as f64 channels -- the reference's channel type -- so the GPU advantage equals
// fn_group_advantage bit for bit. Per-token streams for the loss come from the rollout payload when it follows
// the documented layout: token_id i32[L] | lp f32[L] | old_lp f32[L] | ref_lp f32[L] | mask u8[L]
// (17 bytes per token).
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dfx.h"
#include "distflow/errors.hpp"
#include "distflow/functions.hpp"
#include "distflow/record.hpp"

namespace dfx_distflow {

// ---- errors ------------------------------------------------------------------------------------------
inline void check(dfx_status st) {
  if (st == DFX_OK) return;
  const std::string msg = dfx_last_error();
  switch (st) {
    case DFX_MISSING_CHANNEL: {
      const auto a = msg.find('\''), b = msg.rfind('\'');
      throw distflow::MissingChannelError(a != std::string::npos && b > a ? msg.substr(a + 1, b - a - 1) : msg);
    }
    case DFX_MISSING_ROLLOUTS: throw distflow::MissingRolloutsError(msg);
    case DFX_INDIVISIBLE_ERROR: throw distflow::IndivisibleError(msg);
    case DFX_LAYOUT_ERROR: throw distflow::LayoutError(msg);
    case DFX_STALE_ITERATION: throw distflow::StaleIterationError(msg);
    case DFX_NOT_READY: throw distflow::NotReadyError(msg);
    case DFX_UNKNOWN_STAGE: throw distflow::UnknownStageError(msg);
    default: throw distflow::Error("dfx: " + msg);
  }
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw distflow::Error(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

// ---- device memory -----------------------------------------------------------------------------------
struct DeviceBuffer {
  void* p = nullptr;
  size_t n = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes, bool zero = false) : n(bytes) {
    if (bytes) {
      cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
      if (zero) cuda_check(cudaMemset(p, 0, bytes), "cudaMemset");
    }
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    return *this;
  }
  ~DeviceBuffer() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

template <typename T>
DeviceBuffer upload(const std::vector<T>& v, size_t pad_elems = 0) {
  DeviceBuffer b((v.size() + pad_elems) * sizeof(T), pad_elems != 0);
  if (!v.empty()) cuda_check(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  return b;
}

template <typename T>
std::vector<T> download(const DeviceBuffer& b, size_t n) {
  std::vector<T> v(n);
  if (n) cuda_check(cudaMemcpy(v.data(), b.p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  return v;
}

// ---- packed batch ----------------------------------------------------------------------------------------
struct PackOptions {
  std::vector<std::string> channels;  // rollout channels to upload (f64), e.g. {"reward"}
  bool token_streams = false;         // decode lp/old_lp/ref_lp/mask from the payload layout above
};

struct DevicePacked {
  int64_t n_records = 0, n_rollouts = 0, n_tokens = 0;
  DeviceBuffer group_off, roll_group, cu;
  std::map<std::string, DeviceBuffer> ch;
  DeviceBuffer lp, old_lp, ref_lp, mask;
  dfx_packed view{};
};

constexpr uint32_t kPayloadBytesPerToken = 17;

// Packs a reference SampleBatch into device SoA. Follows detail::require_rollouts / channel_of
// (functions.hpp:82-93): a record without rollouts raises MissingRolloutsError, a rollout without a requested
// channel raises MissingChannelError.
inline DevicePacked pack(const distflow::SampleBatch& batch, const PackOptions& opt) {
  DevicePacked d;
  std::vector<int32_t> go{0}, rg;
  std::vector<int64_t> cu{0};
  std::map<std::string, std::vector<double>> ch;
  std::vector<float> lp, old_lp, ref_lp;
  std::vector<uint8_t> mask;
  for (size_t r = 0; r < batch.records.size(); ++r) {
    const auto& rec = batch.records[r];
    distflow::detail::require_rollouts(rec);
    for (const auto& ro : rec.rollouts) {
      for (const auto& name : opt.channels) ch[name].push_back(distflow::detail::channel_of(ro, name));
      int64_t L = 0;
      if (opt.token_streams) {
        L = ro.token_count;
        if (ro.payload.size() != uint64_t(L) * kPayloadBytesPerToken)
          throw distflow::Error("payload of record " + std::to_string(rec.sample_id) +
                                " does not follow the 17 B/token stream layout");
        const uint8_t* p = ro.payload.data() + 4 * L;  // skip token ids
        auto append_f32 = [&](std::vector<float>& dst, const uint8_t* src) {
          const size_t at = dst.size();
          dst.resize(at + size_t(L));
          std::memcpy(dst.data() + at, src, size_t(L) * 4);
        };
        append_f32(lp, p);
        append_f32(old_lp, p + 4 * L);
        append_f32(ref_lp, p + 8 * L);
        mask.insert(mask.end(), p + 12 * L, p + 13 * L);
      }
      cu.push_back(cu.back() + L);
      rg.push_back(int32_t(r));
    }
    go.push_back(int32_t(rg.size()));
  }
  d.n_records = int64_t(batch.records.size());
  d.n_rollouts = int64_t(rg.size());
  d.n_tokens = cu.back();
  d.group_off = upload(go);
  d.roll_group = upload(rg);
  d.cu = upload(cu);
  for (auto& [name, v] : ch) d.ch.emplace(name, upload(v));
  const size_t pad = 16;  // aligned over-read slack (dfx.h packed-batch contract)
  if (opt.token_streams) {
    d.lp = upload(lp, pad);
    d.old_lp = upload(old_lp, pad);
    d.ref_lp = upload(ref_lp, pad);
    d.mask = upload(mask, pad);
  }
  dfx_packed& v = d.view;
  v.n_records = d.n_records;
  v.n_rollouts = d.n_rollouts;
  v.group_off = d.group_off.as<int32_t>();
  v.roll_group = d.roll_group.as<int32_t>();
  v.cu_seqlens = d.cu.as<int64_t>();
  auto chp = [&](const char* n) { auto it = d.ch.find(n); return it == d.ch.end() ? nullptr : it->second.as<double>(); };
  v.reward = chp("reward");
  v.value = chp("value");
  v.lp = d.lp.as<float>();
  v.old_lp = d.old_lp.as<float>();
  v.ref_lp = d.ref_lp.as<float>();
  v.mask = d.mask.as<uint8_t>();
  return d;
}

// Write a per-rollout f64 device array back as channel `name` (std::map insert, like the reference).
inline void write_channel(distflow::SampleBatch& batch, const std::string& name, const DeviceBuffer& dev, int64_t n) {
  const auto host = download<double>(dev, size_t(n));
  size_t s = 0;
  for (auto& rec : batch.records)
    for (auto& ro : rec.rollouts) ro.channels[name] = host[s++];
}

// ---- loss configuration (the reference has none) -----------------------------------------------
struct LossConfig {
  double clip_low = 0.2, clip_high = 0.2, beta = 0.001;
  int32_t kl_type = DFX_KL_K3, agg = DFX_AGG_TOKEN_MEAN;
};
inline LossConfig& loss_config() {
  static LossConfig c;
  return c;
}

// Last loss computed by gpu_train on this thread (the reference StageContext has no slot for it).
inline dfx_loss_out& last_loss() {
  static thread_local dfx_loss_out o{};
  return o;
}

// ---- stage functions (exact StageFn signature, functions.hpp:63) ------------------------------------------------
// fn_group_advantage (functions.hpp:143-161) on the GPU: bit-identical f64 channel "advantage".
inline void gpu_group_advantage(const distflow::NodeSpec& node, distflow::SampleBatch& batch,
                                distflow::StageContext& ctx) {
  (void)node;
  DevicePacked d = pack(batch, PackOptions{{"reward"}, false});
  DeviceBuffer adv(sizeof(double) * size_t(d.n_rollouts));
  DeviceBuffer flags(sizeof(int32_t), true);
  check(dfx_grpo_advantage(&d.view, ctx.advantage_eps, adv.as<double>(), flags.as<int32_t>(), nullptr));
  check(dfx_check_flags(flags.as<int32_t>(), nullptr));
  write_channel(batch, "advantage", adv, d.n_rollouts);
}

// fn_ppo_advantage (functions.hpp:163-172): advantage = reward - value.
inline void gpu_ppo_advantage(const distflow::NodeSpec& node, distflow::SampleBatch& batch,
                              distflow::StageContext& ctx) {
  (void)node;
  (void)ctx;
  DevicePacked d = pack(batch, PackOptions{{"reward", "value"}, false});
  DeviceBuffer adv(sizeof(double) * size_t(d.n_rollouts));
  check(dfx_ppo_advantage(&d.view, adv.as<double>(), nullptr));
  cuda_check(cudaDeviceSynchronize(), "sync");
  write_channel(batch, "advantage", adv, d.n_rollouts);
}

// fn_train (functions.hpp:176-182) with the loss on the GPU: when the rollouts carry the token-stream payload and
// an "advantage" channel, the fused clipped surrogate + KL runs (result in last_loss()); the role's model version
// is bumped exactly like the reference, frozen roles still throw.
inline void gpu_train(const distflow::NodeSpec& node, distflow::SampleBatch& batch, distflow::StageContext& ctx) {
  if (node.role != distflow::Role::ACTOR && node.role != distflow::Role::CRITIC)
    throw distflow::Error("role " + std::string(distflow::to_string(node.role)) + " is frozen and cannot train");
  bool streams = node.role == distflow::Role::ACTOR && !batch.records.empty();
  for (const auto& rec : batch.records)
    for (const auto& ro : rec.rollouts)
      if (ro.payload.size() != uint64_t(ro.token_count) * kPayloadBytesPerToken || !ro.channels.count("advantage"))
        streams = false;
  if (streams) {
    DevicePacked d = pack(batch, PackOptions{{"advantage"}, true});
    const LossConfig& lc = loss_config();
    dfx_loss_cfg cfg{lc.clip_low, lc.clip_high, lc.beta, ctx.advantage_eps, lc.kl_type, lc.agg, DFX_ADV_ROLLOUT, 0};
    DeviceBuffer out(sizeof(dfx_loss_out));
    dfx_loss_args a{};
    a.adv_roll = d.ch.at("advantage").as<double>();
    a.n_loss_groups = 1;
    a.out = out.as<dfx_loss_out>();
    const size_t ws = dfx_ppo_loss_workspace_bytes(d.n_rollouts, d.n_tokens, 1);
    DeviceBuffer work(ws, true);
    check(dfx_ppo_loss(&d.view, 0, d.n_tokens, &cfg, &a, work.p, ws, nullptr));
    last_loss() = download<dfx_loss_out>(out, 1)[0];
  }
  if (ctx.model_versions) ++(*ctx.model_versions)[node.role];
}

// builtin_registry (functions.hpp:201-219) with the hot-path nodes on the GPU. The generation / inference
// stand-ins upstream of the hot path stay the reference's own CPU functions.
inline distflow::FunctionRegistry gpu_registry() {
  distflow::FunctionRegistry reg;
  reg.register_fn("actor_generate", distflow::fn_generate);
  reg.register_fn("ref_logprob", distflow::fn_ref_logprob);
  reg.register_fn("value_inference", distflow::fn_value);
  reg.register_fn("reward_compute", distflow::fn_reward);
  reg.register_fn("group_advantage", gpu_group_advantage);
  reg.register_fn("ppo_advantage", gpu_ppo_advantage);
  reg.register_fn("train_actor", gpu_train);
  reg.register_fn("train_critic", gpu_train);
  reg.register_fn("ACTOR/MODEL_INFERENCE", distflow::fn_generate);
  reg.register_fn("REFERENCE/MODEL_INFERENCE", distflow::fn_ref_logprob);
  reg.register_fn("CRITIC/MODEL_INFERENCE", distflow::fn_value);
  reg.register_fn("REWARD/COMPUTE", distflow::fn_reward);
  reg.register_fn("ACTOR/MODEL_TRAIN", gpu_train);
  reg.register_fn("CRITIC/MODEL_TRAIN", gpu_train);
  return reg;
}

}  // namespace dfx_distflow
