// dfx_store.hpp -- C++ host side of the DataBuffer reshard for device-resident batches.
//
// A header-only C++17 mirror of the reference's BufferStore (distflow/data_plane.hpp:225-457) over the C ABI in
// dfx.h, for C++ callers that keep rollouts on the GPUs. Same verbs and semantics:
//   put(stage, iteration, dp, tp, batch)   TP != 0 puts are suppressed and counted (:245-248); a duplicate put
//                                          raises (:256-258); iterations below the low-water mark raise
//                                          StaleIterationError (:241-244)
//   ensure_ready(stage, iteration, to)     once every producer group has put, the first consumer runs the
//                                          exchange while the others wait (mutex + condition variable, :296-346);
//                                          NotReadyError after the timeout naming the outstanding puts
//   get(stage, iteration, dest_dp, to)     the destination group's batch on the CALLING THREAD's CUDA device --
//                                          TP peers of a group read identical bytes (:266-292)
//   worker_done(iteration)                 when every worker has reported, entries at or below it are purged and
//                                          the low-water mark advances (:351-367)
// The model is the reference's own: one process, one thread per logical worker (runner.hpp:525-530), all B x W
// logical workers of the box in this process, each bound to a GPU (gpu_of_worker). The record placement is the
// reference's computed natively as segments (dfx_reshard_segments); a consumer group that is one
// run of one producer batch on its GPU is a zero-copy view, otherwise it is assembled on its GPU: token streams by
// one copy kernel per batch (dfx_copy_many: local HBM and peer memory over NVLink), record/rollout metadata
// rebased by dfx_reshard_unpack reading the producer's arrays through peer access. Errors are dfx::StoreError carrying the dfx_status code that
// include/dfx_distflow.hpp maps to the reference's exception types.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dfx.h"

namespace dfx {

struct StoreError : std::runtime_error {
  dfx_status code;
  StoreError(dfx_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void store_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw StoreError(DFX_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
inline void store_check(dfx_status st) {
  if (st != DFX_OK) throw StoreError(st, dfx_last_error());
}

// Device memory on one GPU, freed on that GPU when the last owner goes.
inline std::shared_ptr<uint8_t> device_alloc(int device, size_t bytes, bool zero = false) {
  int prev = 0;
  store_cuda(cudaGetDevice(&prev), "cudaGetDevice");
  store_cuda(cudaSetDevice(device), "cudaSetDevice");
  void* p = nullptr;
  if (bytes) store_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  if (bytes && zero) store_cuda(cudaMemset(p, 0, bytes), "cudaMemset");
  store_cuda(cudaSetDevice(prev), "cudaSetDevice");
  return std::shared_ptr<uint8_t>(static_cast<uint8_t*>(p), [device](uint8_t* q) {
    if (!q) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaFree(q);
    cudaSetDevice(cur);
  });
}

// Size-bucketed free lists of device blocks per GPU: a block returns here when its last owner drops it, so a
// steady-state reshard loop allocates nothing (cudaMalloc / cudaFree synchronise the device).
class DevicePool : public std::enable_shared_from_this<DevicePool> {
 public:
  ~DevicePool() {
    for (auto& kv : free_)
      for (uint8_t* p : kv.second) {
        cudaSetDevice(kv.first.first);
        cudaFree(p);
      }
  }
  std::shared_ptr<uint8_t> get(int device, size_t bytes) {
    const size_t b = bytes <= (1u << 20) ? ((bytes + 4095) & ~size_t(4095)) : ((bytes + (2u << 20) - 1) & ~size_t((2u << 20) - 1));
    uint8_t* p = nullptr;
    {
      std::lock_guard lk(mu_);
      auto& fl = free_[{device, b}];
      if (!fl.empty()) {
        p = fl.back();
        fl.pop_back();
      }
    }
    if (!p) {
      int prev = 0;
      store_cuda(cudaGetDevice(&prev), "cudaGetDevice");
      store_cuda(cudaSetDevice(device), "cudaSetDevice");
      void* q = nullptr;
      store_cuda(cudaMalloc(&q, b), "cudaMalloc");
      store_cuda(cudaSetDevice(prev), "cudaSetDevice");
      p = static_cast<uint8_t*>(q);
    }
    std::weak_ptr<DevicePool> self = shared_from_this();
    return std::shared_ptr<uint8_t>(p, [self, device, b](uint8_t* q) {
      if (auto pool = self.lock()) {
        std::lock_guard lk(pool->mu_);
        pool->free_[{device, b}].push_back(q);
      } else {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaFree(q);
        cudaSetDevice(cur);
      }
    });
  }

 private:
  std::mutex mu_;
  std::map<std::pair<int, size_t>, std::vector<uint8_t*>> free_;
};

// A device-resident packed batch: records [group_off[r], group_off[r+1]) of rollouts, rollouts
// [cu[s], cu[s+1]) of tokens in ABSOLUTE token coordinates of the streams. Host copies of group_off / cu travel
// with it (views and the placement need them, no device reads).
struct DeviceBatch {
  int device = 0;
  int64_t n_records = 0, n_rollouts = 0, token_base = 0, token_span = 0;
  uint64_t* ids = nullptr;
  int32_t* group_off = nullptr;   // relative: group_off[0] == 0
  int32_t* roll_group = nullptr;
  int64_t* cu = nullptr;
  std::map<std::string, double*> channels;                        // f64 [n_rollouts]
  struct Stream {
    uint8_t* base;  // element 0 of the token coordinate system
    size_t elem;    // bytes per element
  };
  std::map<std::string, Stream> streams;
  std::vector<int32_t> h_group_off;
  std::vector<int64_t> h_cu;
  std::vector<std::shared_ptr<uint8_t>> keep;  // owners of the memory the pointers above point into

  dfx_packed packed() const {
    dfx_packed p{};
    p.n_records = n_records;
    p.n_rollouts = n_rollouts;
    p.group_off = group_off;
    p.roll_group = roll_group;
    p.cu_seqlens = cu;
    auto ch = [&](const char* n) { auto it = channels.find(n); return it == channels.end() ? nullptr : it->second; };
    auto st = [&](const char* n) -> const void* {
      auto it = streams.find(n);
      return it == streams.end() ? nullptr : it->second.base;
    };
    p.reward = ch("reward");
    p.value = ch("value");
    p.lp = static_cast<const float*>(st("lp"));
    p.old_lp = static_cast<const float*>(st("old_lp"));
    p.ref_lp = static_cast<const float*>(st("ref_lp"));
    p.value_tok = static_cast<const float*>(st("value_tok"));
    p.token_reward = static_cast<const float*>(st("token_reward"));
    p.mask = static_cast<const uint8_t*>(st("mask"));
    return p;
  }

  // Upload a host packed batch to `device`: streams are given as raw bytes of n_tokens elements each and are
  // padded (aligned over-read slack, dfx.h contract).
  static DeviceBatch upload(int device, const std::vector<uint64_t>& ids, const std::vector<int32_t>& group_off,
                            const std::vector<int64_t>& cu, const std::map<std::string, std::vector<double>>& ch,
                            const std::map<std::string, std::pair<std::vector<uint8_t>, size_t>>& st) {
    DeviceBatch b;
    b.device = device;
    b.n_records = int64_t(ids.size());
    b.n_rollouts = int64_t(cu.size()) - 1;
    b.token_base = cu.front();
    b.token_span = cu.back() - cu.front();
    b.h_group_off = group_off;
    b.h_cu = cu;
    auto up = [&](const void* src, size_t bytes, size_t pad = 0) {
      auto m = device_alloc(device, bytes + pad, pad != 0);
      if (bytes) store_cuda(cudaMemcpy(m.get(), src, bytes, cudaMemcpyHostToDevice), "H2D");
      b.keep.push_back(m);
      return m.get();
    };
    std::vector<int32_t> rg;
    for (size_t r = 0; r + 1 < group_off.size(); ++r)
      for (int32_t s = group_off[r]; s < group_off[r + 1]; ++s) rg.push_back(int32_t(r));
    b.ids = reinterpret_cast<uint64_t*>(up(ids.data(), ids.size() * 8));
    b.group_off = reinterpret_cast<int32_t*>(up(group_off.data(), group_off.size() * 4));
    b.roll_group = reinterpret_cast<int32_t*>(up(rg.data(), rg.size() * 4));
    b.cu = reinterpret_cast<int64_t*>(up(cu.data(), cu.size() * 8));
    for (const auto& [name, v] : ch) b.channels[name] = reinterpret_cast<double*>(up(v.data(), v.size() * 8));
    for (const auto& [name, pe] : st) b.streams[name] = Stream{up(pe.first.data(), pe.first.size(), 16 * pe.second + 64), pe.second};
    return b;
  }

  // Zero-copy view of records [r0, r1): streams and channels shared, group_off / roll_group rebased.
  DeviceBatch view(int64_t r0, int64_t r1, DevicePool* pool = nullptr, cudaStream_t stream = nullptr) const {
    if (r0 == 0 && r1 == n_records) return *this;
    DeviceBatch v;
    v.device = device;
    v.keep = keep;
    const int32_t s0 = h_group_off[size_t(r0)], s1 = h_group_off[size_t(r1)];
    v.n_records = r1 - r0;
    v.n_rollouts = s1 - s0;
    v.h_cu.assign(h_cu.begin() + s0, h_cu.begin() + s1 + 1);
    v.h_group_off.resize(size_t(r1 - r0 + 1));
    for (int64_t r = r0; r <= r1; ++r) v.h_group_off[size_t(r - r0)] = h_group_off[size_t(r)] - s0;
    v.token_base = v.h_cu.front();
    v.token_span = v.h_cu.back() - v.h_cu.front();
    v.ids = ids + r0;
    v.cu = cu + s0;
    for (const auto& [n, p] : channels) v.channels[n] = p + s0;
    v.streams = streams;
    // rebased group_off / roll_group built on the device (no host round trip)
    const size_t gob = size_t(r1 - r0 + 1) * 4 + size_t(s1 - s0) * 4 + 16;
    auto go = pool ? pool->get(device, gob) : device_alloc(device, gob);
    v.group_off = reinterpret_cast<int32_t*>(go.get());
    v.roll_group = reinterpret_cast<int32_t*>(go.get() + ((size_t(r1 - r0 + 1) * 4 + 15) & ~size_t(15)));
    int prev = 0;
    store_cuda(cudaGetDevice(&prev), "cudaGetDevice");
    store_cuda(cudaSetDevice(device), "cudaSetDevice");
    store_check(dfx_view_meta(group_off, roll_group, r0, r1, s1 - s0, v.group_off, v.roll_group, stream));
    if (!stream) store_cuda(cudaStreamSynchronize(nullptr), "cudaStreamSynchronize");
    store_cuda(cudaSetDevice(prev), "cudaSetDevice");
    v.keep.push_back(go);
    return v;
  }
};

struct Layout {
  uint32_t dp = 1, tp = 1;
};
struct StagePlan {  // distflow::StoreStagePlan (data_plane.hpp:216-220)
  Layout produced;
  bool has_consumed = false;
  Layout consumed;
};

class DeviceBufferStore {
 public:
  // num_nodes x workers_per_node logical workers, all in this process; gpu_of_worker[w] = CUDA device of worker w.
  DeviceBufferStore(uint32_t num_nodes, uint32_t workers_per_node, std::vector<int> gpu_of_worker,
                    std::map<std::string, StagePlan> stages)
      : B_(num_nodes), W_(workers_per_node), gpu_(std::move(gpu_of_worker)), stages_(std::move(stages)),
        pool_(std::make_shared<DevicePool>()) {
    if (gpu_.size() != size_t(B_) * W_) throw StoreError(DFX_LAYOUT_ERROR, "gpu_of_worker must map every worker");
    std::set<int> devs(gpu_.begin(), gpu_.end());
    for (int d : devs) {  // one copy / unpack stream per GPU for the store's lifetime
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(d);
      cudaStream_t st;
      store_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
      streams_[d] = st;
      cudaSetDevice(prev);
    }
    for (int a : devs)  // peer access between every pair of the box's GPUs (NVLink / NVSwitch)
      for (int b : devs)
        if (a != b) {
          int ok = 0;
          cudaDeviceCanAccessPeer(&ok, a, b);
          if (ok) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(a);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) store_cuda(e, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
            cudaSetDevice(prev);
          }
        }
  }

  ~DeviceBufferStore() {
    for (auto& kv : streams_) cudaStreamDestroy(kv.second);
  }
  DeviceBufferStore(const DeviceBufferStore&) = delete;
  DeviceBufferStore& operator=(const DeviceBufferStore&) = delete;

  // The batches put must be complete on the device (the store copies them on its own streams).
  bool put(const std::string& stage, uint32_t iteration, uint32_t dp, uint32_t tp, DeviceBatch batch) {
    std::unique_lock lk(mu_);
    const StagePlan& plan = stage_plan(stage);
    if (iteration < low_water_)
      throw StoreError(DFX_STALE_ITERATION, "put for iteration " + std::to_string(iteration) + " below low water " +
                                                std::to_string(low_water_));
    if (tp != 0) {
      ++suppressed_;
      return false;
    }
    if (dp >= plan.produced.dp) throw StoreError(DFX_ERROR, "put from dp group " + std::to_string(dp) + " out of range");
    Entry& e = entries_[{stage, iteration}];
    if (e.by_group.count(dp))
      throw StoreError(DFX_ERROR, "duplicate put for stage '" + stage + "' group " + std::to_string(dp));
    e.by_group.emplace(dp, std::move(batch));
    lk.unlock();
    cv_.notify_all();
    return true;
  }

  void ensure_ready(const std::string& stage, uint32_t iteration, const Layout& fallback,
                    std::chrono::milliseconds timeout = std::chrono::milliseconds(60000)) {
    const auto deadline = std::chrono::steady_clock::now() + timeout;
    std::unique_lock lk(mu_);
    const StagePlan& plan = stage_plan(stage);
    const Layout to = plan.has_consumed ? plan.consumed : fallback;
    const size_t expected = plan.produced.dp;
    for (;;) {
      if (iteration < low_water_)
        throw StoreError(DFX_STALE_ITERATION, "get for iteration " + std::to_string(iteration) +
                                                  " below low water " + std::to_string(low_water_));
      Entry& e = entries_[{stage, iteration}];
      if (!e.error.empty()) throw StoreError(e.error_code, "redistribution failed: " + e.error);
      if (e.state == State::READY) return;
      if (e.state == State::COLLECTING && e.by_group.size() == expected) {
        e.state = State::EXCHANGING;
        std::map<uint32_t, DeviceBatch> src = e.by_group;  // shared memory, not copies
        lk.unlock();
        std::map<std::pair<uint32_t, int>, DeviceBatch> out;
        StoreError failure(DFX_OK, "");
        try {
          out = exchange(plan, to, src);
        } catch (const StoreError& ex) {
          failure = ex;
        } catch (const std::exception& ex) {
          failure = StoreError(DFX_ERROR, ex.what());
        }
        lk.lock();
        Entry& e2 = entries_[{stage, iteration}];
        if (failure.code == DFX_OK) {
          e2.ready = std::move(out);
          e2.by_group.clear();
          e2.state = State::READY;
        } else {
          e2.error = failure.what();
          e2.error_code = failure.code;
        }
        lk.unlock();
        cv_.notify_all();
        if (failure.code != DFX_OK) throw failure;
        return;
      }
      if (cv_.wait_until(lk, deadline) == std::cv_status::timeout) {
        const size_t have = entries_[{stage, iteration}].by_group.size();
        throw StoreError(DFX_NOT_READY, "stage '" + stage + "' iteration " + std::to_string(iteration) +
                                            " not ready: " + std::to_string(expected - std::min(expected, have)) +
                                            " puts outstanding");
      }
    }
  }

  // The destination group's batch on the calling thread's CUDA device.
  DeviceBatch get(const std::string& stage, uint32_t iteration, uint32_t dest_dp, const Layout& to,
                  std::chrono::milliseconds timeout = std::chrono::milliseconds(60000)) {
    ensure_ready(stage, iteration, to, timeout);
    int dev = 0;
    store_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard lk(mu_);
    const Entry& e = entries_.at({stage, iteration});
    auto it = e.ready.find({dest_dp, dev});
    if (it == e.ready.end())
      throw StoreError(DFX_ERROR, "dp group " + std::to_string(dest_dp) + " has no worker on device " +
                                      std::to_string(dev));
    return it->second;
  }

  void worker_done(uint32_t iteration) {
    {
      std::lock_guard lk(mu_);
      const uint32_t c = ++done_[iteration];
      if (c < B_ * W_) return;
      done_.erase(iteration);
      low_water_ = std::max(low_water_, iteration + 1);
      for (auto it = entries_.begin(); it != entries_.end();) {
        if (it->first.second < low_water_) it = entries_.erase(it);
        else ++it;
      }
    }
    cv_.notify_all();
  }

  uint64_t suppressed_count() const {
    std::lock_guard lk(mu_);
    return suppressed_;
  }
  uint64_t bytes_copied() const {
    std::lock_guard lk(mu_);
    return copied_;
  }

 private:
  enum class State { COLLECTING, EXCHANGING, READY };
  struct Entry {
    std::map<uint32_t, DeviceBatch> by_group;
    std::map<std::pair<uint32_t, int>, DeviceBatch> ready;  // (consumer group, device) -> batch
    State state = State::COLLECTING;
    std::string error;
    dfx_status error_code = DFX_ERROR;
  };

  const StagePlan& stage_plan(const std::string& stage) const {
    auto it = stages_.find(stage);
    if (it == stages_.end()) throw StoreError(DFX_UNKNOWN_STAGE, "stage '" + stage + "' not in plan");
    return it->second;
  }

  std::map<std::pair<uint32_t, int>, DeviceBatch> exchange(const StagePlan& plan, const Layout& to,
                                                           const std::map<uint32_t, DeviceBatch>& src) {
    std::vector<uint64_t> counts(plan.produced.dp);
    for (const auto& [p, b] : src) counts[p] = uint64_t(b.n_records);
    const int64_t n = dfx_reshard_segments(B_, W_, plan.produced.dp, plan.produced.tp, to.dp, to.tp, counts.data(),
                                           nullptr, 0);
    if (n < 0) store_check(dfx_status(-n));
    std::vector<dfx_segment> segs(size_t(std::max<int64_t>(n, 1)));
    dfx_reshard_segments(B_, W_, plan.produced.dp, plan.produced.tp, to.dp, to.tp, counts.data(), segs.data(), n);
    std::map<std::pair<uint32_t, int>, DeviceBatch> out;
    uint64_t copied = 0;
    for (uint32_t d = 0; d < to.dp; ++d) {
      std::vector<const dfx_segment*> mine;
      for (int64_t i = 0; i < n; ++i)
        if (segs[size_t(i)].dst_group == d) mine.push_back(&segs[size_t(i)]);
      std::set<int> devs;
      for (uint32_t t = 0; t < to.tp; ++t) devs.insert(gpu_[size_t(d) * to.tp + t]);  // lead = d * tp (topology.hpp:50)
      for (int dev : devs) {
        if (mine.size() == 1 && src.at(mine[0]->src_group).device == dev) {  // one local run: a view
          const DeviceBatch& b = src.at(mine[0]->src_group);
          out.emplace(std::make_pair(d, dev),
                      b.view(int64_t(mine[0]->src_rec), int64_t(mine[0]->src_rec + mine[0]->count), pool_.get(),
                             streams_.at(dev)));
          continue;
        }
        out.emplace(std::make_pair(d, dev), assemble(dev, mine, src, copied));
      }
    }
    for (auto& kv : streams_) store_cuda(cudaStreamSynchronize(kv.second), "cudaStreamSynchronize");
    std::lock_guard lk(mu_);
    copied_ += copied;
    return out;
  }

  // Concatenate the segments into a new batch on `dev`: token streams by peer copies, metadata by unpack.
  DeviceBatch assemble(int dev, const std::vector<const dfx_segment*>& segs, const std::map<uint32_t, DeviceBatch>& src,
                       uint64_t& copied) {
    const DeviceBatch& first = src.at(segs[0]->src_group);
    int64_t R = 0, S = 0, T = 0;
    std::vector<int32_t> hgo{0};
    std::vector<int64_t> hcu{0};
    for (const dfx_segment* sg : segs) {
      const DeviceBatch& b = src.at(sg->src_group);
      const int64_t r0 = int64_t(sg->src_rec), r1 = r0 + int64_t(sg->count);
      const int32_t s0 = b.h_group_off[size_t(r0)], s1 = b.h_group_off[size_t(r1)];
      for (int64_t r = r0; r < r1; ++r) hgo.push_back(hgo.back() + b.h_group_off[size_t(r + 1)] - b.h_group_off[size_t(r)]);
      for (int32_t s = s0; s < s1; ++s) hcu.push_back(hcu.back() + b.h_cu[size_t(s + 1)] - b.h_cu[size_t(s)]);
      R += r1 - r0;
      S += s1 - s0;
      T += b.h_cu[size_t(s1)] - b.h_cu[size_t(s0)];
    }
    DeviceBatch o;
    o.device = dev;
    o.n_records = R;
    o.n_rollouts = S;
    o.token_base = 0;
    o.token_span = T;
    o.h_group_off = hgo;
    o.h_cu = hcu;
    auto meta = pool_->get(dev, size_t(R) * 8 + size_t(R + 1) * 4 + size_t(S) * 4 + size_t(S + 1) * 8 +
                                    first.channels.size() * size_t(S) * 8 + 64);
    o.keep.push_back(meta);
    uint8_t* m = meta.get();
    o.ids = reinterpret_cast<uint64_t*>(m);
    o.cu = reinterpret_cast<int64_t*>(m + size_t(R) * 8);
    size_t off = size_t(R) * 8 + size_t(S + 1) * 8;
    std::vector<double*> dst_ch;
    for (const auto& kv : first.channels) {
      o.channels[kv.first] = reinterpret_cast<double*>(m + off);
      dst_ch.push_back(o.channels[kv.first]);
      off += size_t(S) * 8;
    }
    o.group_off = reinterpret_cast<int32_t*>(m + off);
    off += size_t(R + 1) * 4;
    o.roll_group = reinterpret_cast<int32_t*>(m + off);
    for (const auto& kv : first.streams) {
      auto sm = pool_->get(dev, size_t(T) * kv.second.elem + 16 * kv.second.elem + 64);  // padding: over-read slack
      o.keep.push_back(sm);
      o.streams[kv.first] = DeviceBatch::Stream{sm.get(), kv.second.elem};
    }
    int prev = 0;
    store_cuda(cudaGetDevice(&prev), "cudaGetDevice");
    store_cuda(cudaSetDevice(dev), "cudaSetDevice");
    cudaStream_t st = streams_.at(dev);
    std::vector<dfx_seg_meta> metas;
    std::vector<uint64_t> cp_dst, cp_src, cp_n;
    int64_t dr = 0, ds = 0, dt = 0;
    for (const dfx_segment* sg : segs) {
      const DeviceBatch& b = src.at(sg->src_group);
      const int64_t r0 = int64_t(sg->src_rec), r1 = r0 + int64_t(sg->count);
      const int32_t s0 = b.h_group_off[size_t(r0)], s1 = b.h_group_off[size_t(r1)];
      const int64_t t0 = b.h_cu[size_t(s0)], t1 = b.h_cu[size_t(s1)];
      for (const auto& kv : b.streams) {
        const size_t e = kv.second.elem;
        if (t1 > t0) {  // all of this batch's copies (local HBM or a peer over NVLink) go out in one launch
          cp_dst.push_back(uint64_t(reinterpret_cast<uintptr_t>(o.streams.at(kv.first).base + size_t(dt) * e)));
          cp_src.push_back(uint64_t(reinterpret_cast<uintptr_t>(kv.second.base + size_t(t0) * e)));
          cp_n.push_back(uint64_t(t1 - t0) * e);
          copied += uint64_t(t1 - t0) * e;
        }
      }
      dfx_seg_meta sm{};
      sm.ids = b.ids + r0;
      sm.group_off = b.group_off + r0;
      sm.cu = b.cu + s0;
      int c = 0;
      for (const auto& kv : first.channels) sm.ch[c++] = b.channels.at(kv.first) + s0;
      sm.n_rec = r1 - r0;
      sm.n_roll = s1 - s0;
      sm.dst_rec = dr;
      sm.dst_roll = ds;
      sm.dst_tok = dt;
      metas.push_back(sm);
      dr += r1 - r0;
      ds += s1 - s0;
      dt += t1 - t0;
    }
    store_check(dfx_copy_many(int64_t(cp_n.size()), cp_dst.data(), cp_src.data(), cp_n.data(), st));
    store_check(dfx_reshard_unpack(metas.data(), int32_t(metas.size()), int32_t(dst_ch.size()), o.ids, o.group_off,
                                   o.roll_group, o.cu, dst_ch.data(), st));
    store_cuda(cudaSetDevice(prev), "cudaSetDevice");  // completion: the exchange synchronises every stream
    return o;
  }

  uint32_t B_, W_;
  std::vector<int> gpu_;
  std::map<std::string, StagePlan> stages_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::pair<std::string, uint32_t>, Entry> entries_;
  std::map<uint32_t, uint32_t> done_;
  uint32_t low_water_ = 0;
  uint64_t suppressed_ = 0;
  uint64_t copied_ = 0;
  std::shared_ptr<DevicePool> pool_;
  std::map<int, cudaStream_t> streams_;
};

}  // namespace dfx
