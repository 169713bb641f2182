// dfx_dstore.hpp -- C++ host side of the distributed DataBuffer (one process per GPU), over the C ABI in dfx.h.
//
// The reference's BufferStore verbs (distflow/data_plane.hpp:225-457) for the reference's fork-per-node mode
// (runner.hpp:655-742) with device-resident batches: every process owns one GPU and the logical workers mapped to
// it, the exchange is native (libdfx: shared-memory host metadata, copy-engine pulls over NVLink or NCCL send/recv,
// one unpack kernel). Errors are dfx::StoreError carrying the dfx_status (include/dfx_distflow.hpp maps them to
// the reference's exception types).
//
//   dfx::Comm comm = dfx::Comm::create(n_ranks, rank, id_bytes);  // id from dfx::Comm::unique_id() on rank 0
//   dfx::DistBufferStore store(comm, topology, stages, schema, stream);
//   store.put(stage, it, dp, tp, batch);  store.ensure_ready(stage, it, layout);  store.get(stage, it, d, layout);
//   store.worker_done(it);
#pragma once

#include <array>
#include <map>
#include <string>
#include <vector>

#include "dfx.h"
#include "dfx_store.hpp"

namespace dfx {

class Comm {
 public:
  static std::array<char, DFX_COMM_ID_BYTES> unique_id() {
    std::array<char, DFX_COMM_ID_BYTES> id{};
    store_check(dfx_comm_unique_id(id.data()));
    return id;
  }
  // collective: every rank calls it with the same id, its device current
  Comm(int32_t n_ranks, int32_t rank, const std::array<char, DFX_COMM_ID_BYTES>& id) {
    store_check(dfx_comm_init(id.data(), n_ranks, rank, &c_));
  }
  ~Comm() { dfx_comm_destroy(c_); }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  dfx_comm* get() const { return c_; }
  int32_t rank() const { return dfx_comm_rank(c_); }
  int32_t size() const { return dfx_comm_size(c_); }

 private:
  dfx_comm* c_ = nullptr;
};

struct DStageCfg {
  Layout produced;
  Layout consumed;  // dp == 0: given to ensure_ready
};

class DistBufferStore {
 public:
  // rank_of_worker[w]: the process (GPU) hosting logical worker w of the B x W world; streams: element sizes of the
  // token streams (schema order); n_channels f64 rollout channels; all work on `stream`
  DistBufferStore(const Comm& comm, uint32_t num_nodes, uint32_t workers_per_node, std::vector<int32_t> rank_of_worker,
                  const std::map<std::string, DStageCfg>& stages, std::vector<uint32_t> stream_esz, int32_t n_channels,
                  cudaStream_t stream, int32_t transport = DFX_TRANSPORT_PULL)
      : rank_of_worker_(std::move(rank_of_worker)), esz_(std::move(stream_esz)) {
    for (const auto& [name, sc] : stages) {
      names_.push_back(name);
      pdp_.push_back(sc.produced.dp);
      ptp_.push_back(sc.produced.tp);
      cdp_.push_back(sc.consumed.dp);
      ctp_.push_back(sc.consumed.tp);
    }
    std::vector<const char*> cn;
    for (const auto& n : names_) cn.push_back(n.c_str());
    dfx_dstore_cfg cfg{};
    cfg.num_nodes = num_nodes;
    cfg.workers_per_node = workers_per_node;
    cfg.rank_of_worker = rank_of_worker_.data();
    cfg.n_streams = int32_t(esz_.size());
    cfg.stream_esz = esz_.data();
    cfg.n_ch = n_channels;
    cfg.n_stages = int32_t(names_.size());
    cfg.stage_names = cn.data();
    cfg.produced_dp = pdp_.data();
    cfg.produced_tp = ptp_.data();
    cfg.consumed_dp = cdp_.data();
    cfg.consumed_tp = ctp_.data();
    cfg.transport = transport;
    store_check(dfx_dstore_create(&cfg, comm.get(), stream, &s_));
  }
  ~DistBufferStore() { dfx_dstore_destroy(s_); }
  DistBufferStore(const DistBufferStore&) = delete;
  DistBufferStore& operator=(const DistBufferStore&) = delete;

  bool put(const std::string& stage, uint64_t it, uint32_t dp, uint32_t tp, const dfx_batch& b) {
    int32_t acc = 0;
    store_check(dfx_dstore_put(s_, stage.c_str(), it, dp, tp, &b, &acc));
    return acc != 0;
  }
  void ensure_ready(const std::string& stage, uint64_t it, const Layout& to) {
    store_check(dfx_dstore_ensure_ready(s_, stage.c_str(), it, to.dp, to.tp));
  }
  dfx_batch get(const std::string& stage, uint64_t it, uint32_t dest_dp, const Layout& to) {
    dfx_batch b{};
    store_check(dfx_dstore_get(s_, stage.c_str(), it, dest_dp, to.dp, to.tp, &b));
    return b;
  }
  void worker_done(uint64_t it) { store_check(dfx_dstore_worker_done(s_, it)); }
  std::array<uint64_t, 5> stats() const {
    std::array<uint64_t, 5> o{};
    store_check(dfx_dstore_stats(s_, o.data()));
    return o;
  }

 private:
  dfx_dstore* s_ = nullptr;
  std::vector<int32_t> rank_of_worker_;
  std::vector<uint32_t> esz_;
  std::vector<std::string> names_;
  std::vector<uint32_t> pdp_, ptp_, cdp_, ctp_;
};

}  // namespace dfx
