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
// Packing: a SampleBatch (AoS, std::map channels) is packed into the device SoA layout (dfx_packed) through the
// calling worker thread's arena (pinned staging + grow-only device buffers + the worker's stream: no allocation
// in a steady state) and results are written back as f64 channels -- the reference's channel type -- so the GPU
// advantage equals fn_group_advantage bit for bit. Per-token streams for the loss come from the rollout payload when it follows
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

// ---- per-worker device arena ---------------------------------------------------------------------------------
// The reference's StageContext (functions.hpp:55-61) has no slot for device state, and one OS thread runs each
// worker's chain (runner.hpp:525-530): the arena is thread-local -- the worker's own stream, grow-only device
// buffers and pinned host staging, reused by every node call, so a steady-state run_iteration allocates nothing
// and every host<->device copy is an async pinned transfer on the worker's stream (one synchronization per node).
struct PinnedBuffer {
  void* p = nullptr;
  size_t n = 0;
  PinnedBuffer() = default;
  PinnedBuffer(const PinnedBuffer&) = delete;
  PinnedBuffer& operator=(const PinnedBuffer&) = delete;
  ~PinnedBuffer() {
    if (p) cudaFreeHost(p);
  }
};

struct Arena {
  cudaStream_t stream = nullptr;
  std::map<std::string, DeviceBuffer> dev;
  std::map<std::string, PinnedBuffer> host;
  uint64_t grows = 0;  // allocations so far (a steady state stops growing)
  Arena() { cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate"); }
  ~Arena() {
    if (stream) cudaStreamDestroy(stream);
  }
  // device buffer `name` of at least `bytes` (zero-filled when it grows: workspaces rely on it)
  void* device(const std::string& name, size_t bytes) {
    DeviceBuffer& d = dev[name];
    if (d.n < bytes) {
      d = DeviceBuffer(std::max<size_t>(bytes, 2 * d.n), true);
      ++grows;
    }
    return d.p;
  }
  void* pinned(const std::string& name, size_t bytes) {
    PinnedBuffer& h = host[name];
    if (h.n < bytes) {
      if (h.p) cudaFreeHost(h.p);
      h.n = std::max<size_t>(bytes, 2 * h.n);
      cuda_check(cudaMallocHost(&h.p, h.n), "cudaMallocHost");
      ++grows;
    }
    return h.p;
  }
};
inline Arena& worker_arena() {
  static thread_local Arena a;
  return a;
}

// ---- packed batch ----------------------------------------------------------------------------------------
struct PackOptions {
  std::vector<std::string> channels;  // rollout channels to upload (f64), e.g. {"reward"}
  bool token_streams = false;         // decode lp/old_lp/ref_lp/mask from the payload layout above
};

struct DevicePacked {
  int64_t n_records = 0, n_rollouts = 0, n_tokens = 0;
  std::map<std::string, double*> ch;  // device channel arrays (arena)
  dfx_packed view{};
};

constexpr uint32_t kPayloadBytesPerToken = 17;

// Packs a reference SampleBatch into device SoA through the worker's arena: one pass over the records writes
// the SoA arrays into pinned staging, then one async H2D copy per array on the worker's stream. Follows
// detail::require_rollouts / channel_of (functions.hpp:82-93): a record without rollouts raises
// MissingRolloutsError, a rollout without a requested channel raises MissingChannelError.
inline DevicePacked pack(const distflow::SampleBatch& batch, const PackOptions& opt, Arena& ar = worker_arena()) {
  DevicePacked d;
  int64_t R = int64_t(batch.records.size()), S = 0, T = 0;
  for (const auto& rec : batch.records) {
    distflow::detail::require_rollouts(rec);
    S += int64_t(rec.rollouts.size());
    if (opt.token_streams)
      for (const auto& ro : rec.rollouts) {
        if (ro.payload.size() != uint64_t(ro.token_count) * kPayloadBytesPerToken)
          throw distflow::Error("payload of record " + std::to_string(rec.sample_id) +
                                " does not follow the 17 B/token stream layout");
        T += ro.token_count;
      }
  }
  const size_t pad = 16;  // aligned over-read slack (dfx.h packed-batch contract)
  auto* go = static_cast<int32_t*>(ar.pinned("go", size_t(R + 1) * 4));
  auto* rg = static_cast<int32_t*>(ar.pinned("rg", size_t(S) * 4 + 4));
  auto* cu = static_cast<int64_t*>(ar.pinned("cu", size_t(S + 1) * 8));
  std::vector<double*> chh;
  for (const auto& name : opt.channels) chh.push_back(static_cast<double*>(ar.pinned("ch:" + name, size_t(S) * 8 + 8)));
  float *lp = nullptr, *old = nullptr, *ref = nullptr;
  uint8_t* mask = nullptr;
  if (opt.token_streams) {
    lp = static_cast<float*>(ar.pinned("lp", size_t(T) * 4 + 4));
    old = static_cast<float*>(ar.pinned("old", size_t(T) * 4 + 4));
    ref = static_cast<float*>(ar.pinned("ref", size_t(T) * 4 + 4));
    mask = static_cast<uint8_t*>(ar.pinned("mask", size_t(T) + 1));
  }
  go[0] = 0;
  cu[0] = 0;
  int64_t s = 0, t = 0;
  for (size_t r = 0; r < batch.records.size(); ++r) {
    for (const auto& ro : batch.records[r].rollouts) {
      for (size_t c = 0; c < opt.channels.size(); ++c) chh[c][s] = distflow::detail::channel_of(ro, opt.channels[c]);
      int64_t L = 0;
      if (opt.token_streams) {
        L = ro.token_count;
        const uint8_t* p = ro.payload.data() + 4 * L;  // skip token ids
        std::memcpy(lp + t, p, size_t(L) * 4);
        std::memcpy(old + t, p + 4 * L, size_t(L) * 4);
        std::memcpy(ref + t, p + 8 * L, size_t(L) * 4);
        std::memcpy(mask + t, p + 12 * L, size_t(L));
      }
      t += L;
      cu[s + 1] = t;
      rg[s++] = int32_t(r);
    }
    go[r + 1] = int32_t(s);
  }
  auto up = [&](const char* name, const void* src, size_t bytes, size_t dev_bytes) {
    void* dst = ar.device(name, dev_bytes);
    if (bytes) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ar.stream), "H2D");
    return dst;
  };
  d.n_records = R;
  d.n_rollouts = S;
  d.n_tokens = T;
  dfx_packed& v = d.view;
  v.n_records = R;
  v.n_rollouts = S;
  v.group_off = static_cast<int32_t*>(up("go", go, size_t(R + 1) * 4, size_t(R + 1) * 4));
  v.roll_group = static_cast<int32_t*>(up("rg", rg, size_t(S) * 4, size_t(S) * 4 + 4));
  v.cu_seqlens = static_cast<int64_t*>(up("cu", cu, size_t(S + 1) * 8, size_t(S + 1) * 8));
  for (size_t c = 0; c < opt.channels.size(); ++c)
    d.ch[opt.channels[c]] = static_cast<double*>(up(("ch:" + opt.channels[c]).c_str(), chh[c], size_t(S) * 8, size_t(S) * 8 + 8));
  auto chp = [&](const char* n) { auto it = d.ch.find(n); return it == d.ch.end() ? nullptr : it->second; };
  v.reward = chp("reward");
  v.value = chp("value");
  if (opt.token_streams) {
    v.lp = static_cast<float*>(up("lp", lp, size_t(T) * 4, (size_t(T) + pad) * 4));
    v.old_lp = static_cast<float*>(up("old", old, size_t(T) * 4, (size_t(T) + pad) * 4));
    v.ref_lp = static_cast<float*>(up("ref", ref, size_t(T) * 4, (size_t(T) + pad) * 4));
    v.mask = static_cast<uint8_t*>(up("mask", mask, size_t(T), size_t(T) + pad));
  }
  return d;
}

// Write a per-rollout f64 device array back as channel `name` (std::map insert, like the reference): one async
// D2H into pinned staging, one synchronization of the worker's stream.
inline void write_channel(distflow::SampleBatch& batch, const std::string& name, const double* dev, int64_t n,
                          Arena& ar = worker_arena()) {
  auto* host = static_cast<double*>(ar.pinned("out:" + name, size_t(n) * 8 + 8));
  if (n) cuda_check(cudaMemcpyAsync(host, dev, size_t(n) * 8, cudaMemcpyDeviceToHost, ar.stream), "D2H");
  cuda_check(cudaStreamSynchronize(ar.stream), "sync");
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
// fn_generate (functions.hpp:108-123) on the GPU: token counts (draw_tokens) and hash_bytes payloads computed by
// dfx_generate_counts / dfx_generate_payload, bit-identical, then handed to the host records (the reference's
// SampleBatch owns its payload bytes). Same errors: rollouts_per_prompt < 1, max < min.
inline void gpu_generate(const distflow::NodeSpec& node, distflow::SampleBatch& batch, distflow::StageContext& ctx) {
  (void)node;
  if (ctx.gen.rollouts_per_prompt < 1) throw distflow::Error("rollouts_per_prompt must be >= 1");
  const auto& td = ctx.gen.response_tokens;
  const bool uni = td.kind == distflow::TokenDist::Kind::UNIFORM;
  if (uni && td.max < td.min) throw distflow::Error("token distribution max < min");
  Arena& ar = worker_arena();
  const int64_t R = int64_t(batch.records.size()), n_roll = ctx.gen.rollouts_per_prompt, S = R * n_roll;
  if (R == 0) return;
  auto* hid = static_cast<uint64_t*>(ar.pinned("gen:ids", size_t(R) * 8));
  for (int64_t r = 0; r < R; ++r) hid[r] = batch.records[size_t(r)].sample_id;
  auto* did = static_cast<uint64_t*>(ar.device("gen:ids", size_t(R) * 8));
  auto* dcnt = static_cast<uint32_t*>(ar.device("gen:counts", size_t(S) * 4));
  auto* hcnt = static_cast<uint32_t*>(ar.pinned("gen:counts", size_t(S) * 4));
  cuda_check(cudaMemcpyAsync(did, hid, size_t(R) * 8, cudaMemcpyHostToDevice, ar.stream), "H2D");
  check(dfx_generate_counts(ctx.run_seed, uni ? 1 : 0, td.value, td.min, td.max, did, R, int32_t(n_roll), dcnt,
                            ar.stream));
  cuda_check(cudaMemcpyAsync(hcnt, dcnt, size_t(S) * 4, cudaMemcpyDeviceToHost, ar.stream), "D2H");
  cuda_check(cudaStreamSynchronize(ar.stream), "sync");
  auto* hoff = static_cast<int64_t*>(ar.pinned("gen:off", size_t(S + 1) * 8));
  hoff[0] = 0;
  for (int64_t s = 0; s < S; ++s) hoff[s + 1] = hoff[s] + int64_t(hcnt[s]) * ctx.gen.bytes_per_token;
  const size_t total = size_t(hoff[S]);
  auto* hpl = static_cast<uint8_t*>(ar.pinned("gen:payload", total + 1));
  if (total) {
    auto* doff = static_cast<int64_t*>(ar.device("gen:off", size_t(S + 1) * 8));
    auto* dpl = static_cast<uint8_t*>(ar.device("gen:payload", total));
    cuda_check(cudaMemcpyAsync(doff, hoff, size_t(S + 1) * 8, cudaMemcpyHostToDevice, ar.stream), "H2D");
    check(dfx_generate_payload(ctx.run_seed, did, R, int32_t(n_roll), doff, dpl, ar.stream));
    cuda_check(cudaMemcpyAsync(hpl, dpl, total, cudaMemcpyDeviceToHost, ar.stream), "D2H");
    cuda_check(cudaStreamSynchronize(ar.stream), "sync");
  }
  int64_t s = 0;
  for (auto& rec : batch.records) {
    rec.rollouts.clear();
    rec.rollouts.reserve(size_t(n_roll));
    for (int64_t r = 0; r < n_roll; ++r, ++s) {
      distflow::Rollout ro;
      ro.token_count = hcnt[s];
      ro.payload.assign(hpl + hoff[s], hpl + hoff[s + 1]);
      rec.rollouts.push_back(std::move(ro));
    }
  }
}


// fn_group_advantage (functions.hpp:143-161) on the GPU: bit-identical f64 channel "advantage".
inline void gpu_group_advantage(const distflow::NodeSpec& node, distflow::SampleBatch& batch,
                                distflow::StageContext& ctx) {
  (void)node;
  Arena& ar = worker_arena();
  DevicePacked d = pack(batch, PackOptions{{"reward"}, false}, ar);
  auto* adv = static_cast<double*>(ar.device("adv", sizeof(double) * size_t(d.n_rollouts) + 8));
  auto* flags = static_cast<int32_t*>(ar.device("flags", sizeof(int32_t)));
  cuda_check(cudaMemsetAsync(flags, 0, sizeof(int32_t), ar.stream), "memset");
  check(dfx_grpo_advantage(&d.view, ctx.advantage_eps, adv, flags, ar.stream));
  check(dfx_check_flags(flags, ar.stream));
  write_channel(batch, "advantage", adv, d.n_rollouts, ar);
}

// fn_ppo_advantage (functions.hpp:163-172): advantage = reward - value.
inline void gpu_ppo_advantage(const distflow::NodeSpec& node, distflow::SampleBatch& batch,
                              distflow::StageContext& ctx) {
  (void)node;
  (void)ctx;
  Arena& ar = worker_arena();
  DevicePacked d = pack(batch, PackOptions{{"reward", "value"}, false}, ar);
  auto* adv = static_cast<double*>(ar.device("adv", sizeof(double) * size_t(d.n_rollouts) + 8));
  check(dfx_ppo_advantage(&d.view, adv, ar.stream));
  write_channel(batch, "advantage", adv, d.n_rollouts, ar);
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
    Arena& ar = worker_arena();
    DevicePacked d = pack(batch, PackOptions{{"advantage"}, true}, ar);
    const LossConfig& lc = loss_config();
    dfx_loss_cfg cfg{lc.clip_low, lc.clip_high, lc.beta, ctx.advantage_eps, lc.kl_type, lc.agg, DFX_ADV_ROLLOUT, 0};
    auto* out = static_cast<dfx_loss_out*>(ar.device("loss_out", sizeof(dfx_loss_out)));
    dfx_loss_args a{};
    a.adv_roll = d.ch.at("advantage");
    a.n_loss_groups = 1;
    a.out = out;
    const size_t ws = dfx_ppo_loss_workspace_bytes(d.n_rollouts, d.n_tokens, 1);
    void* work = ar.device("loss_ws", ws);  // zero-filled when it grows; the kernels keep their tickets zeroed
    check(dfx_ppo_loss(&d.view, 0, d.n_tokens, &cfg, &a, work, ws, ar.stream));
    auto* host = static_cast<dfx_loss_out*>(ar.pinned("loss_out", sizeof(dfx_loss_out)));
    cuda_check(cudaMemcpyAsync(host, out, sizeof(dfx_loss_out), cudaMemcpyDeviceToHost, ar.stream), "D2H");
    cuda_check(cudaStreamSynchronize(ar.stream), "sync");
    last_loss() = *host;
  }
  if (ctx.model_versions) ++(*ctx.model_versions)[node.role];
}

// builtin_registry (functions.hpp:201-219) with the hot-path nodes on the GPU. The generation / inference
// stand-ins upstream of the hot path stay the reference's own CPU functions.
inline distflow::FunctionRegistry gpu_registry() {
  distflow::FunctionRegistry reg;
  reg.register_fn("actor_generate", gpu_generate);
  reg.register_fn("ref_logprob", distflow::fn_ref_logprob);
  reg.register_fn("value_inference", distflow::fn_value);
  reg.register_fn("reward_compute", distflow::fn_reward);
  reg.register_fn("group_advantage", gpu_group_advantage);
  reg.register_fn("ppo_advantage", gpu_ppo_advantage);
  reg.register_fn("train_actor", gpu_train);
  reg.register_fn("train_critic", gpu_train);
  reg.register_fn("ACTOR/MODEL_INFERENCE", gpu_generate);
  reg.register_fn("REFERENCE/MODEL_INFERENCE", distflow::fn_ref_logprob);
  reg.register_fn("CRITIC/MODEL_INFERENCE", distflow::fn_value);
  reg.register_fn("REWARD/COMPUTE", distflow::fn_reward);
  reg.register_fn("ACTOR/MODEL_TRAIN", gpu_train);
  reg.register_fn("CRITIC/MODEL_TRAIN", gpu_train);
  return reg;
}

}  // namespace dfx_distflow
