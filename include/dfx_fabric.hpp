// dfx_fabric.hpp -- an NCCL-backed implementation of the reference's message Fabric (distflow/transport.hpp:215-246).
//
// The reference's TcpFabric hosts one node's endpoints (its workers + its store endpoint) per process and carries
// cross-node envelopes over loopback sockets; NcclFabric keeps the same contract -- send() never blocks, recv()
// matches (src, tag, iteration) FIFO from the endpoint's mailbox with the reference's timeout and PeerClosedError,
// intra-node envelopes never leave the process and are not counted, cross-node ones are counted in the reference's
// framed sizes (TrafficCounters) -- and moves the cross-node bytes between the node processes' GPUs with NCCL:
// one progress thread per process (the only thread touching the communicator) runs bulk-synchronous rounds with
// every other node: (1) a device all-reduce of the per-destination byte counts and the closing flags, (2) if
// anything is pending, the outgoing envelopes packed per destination node into one pinned buffer, one H2D copy,
// ONE grouped all-to-all-v over NVLink (dfx_comm_alltoallv), one D2H copy, and delivery into the destination
// endpoints' mailboxes. close() lets the rounds drain every pending envelope on every node before the thread exits.
// Use: one process per node, each with its GPU current and a dfx::Comm over the node processes (rank = node).
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "dfx.h"
#include "dfx_dstore.hpp"
#include "distflow/transport.hpp"

namespace dfx_distflow {

class NcclFabric final : public distflow::Fabric {
 public:
  NcclFabric(const distflow::ClusterTopology& topo, uint32_t node_index, dfx::Comm& comm,
             uint32_t max_frame_bytes = distflow::kDefaultMaxFrameBytes)
      : Fabric(topo, max_frame_bytes), node_(node_index), comm_(comm), counters_(topo) {
    if (node_ >= topo_.num_nodes) throw distflow::Error("node index out of range");
    if (uint32_t(comm.size()) != topo_.num_nodes || uint32_t(comm.rank()) != node_)
      throw distflow::Error("NcclFabric: the communicator must have one rank per node, rank = node index");
    boxes_.resize(topo_.endpoint_count());
    for (auto& b : boxes_) b = std::make_unique<distflow::detail::Mailbox>();
    dfx::store_cuda(cudaGetDevice(&device_), "cudaGetDevice");
    dfx::store_cuda(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    progress_ = std::thread([this] { progress_loop(); });
  }
  ~NcclFabric() override {
    close();
    if (progress_.joinable()) progress_.join();
    for (void* p : {dsend_, drecv_})
      if (p) cudaFree(p);
    for (void* p : {hsend_, hrecv_})
      if (p) cudaFreeHost(p);
    cudaStreamDestroy(stream_);
  }

  void send(distflow::Envelope env) override {
    check_endpoint(env.src_rank, "src");
    check_endpoint(env.dst_rank, "dst");
    const uint32_t dn = topo_.endpoint_node(env.dst_rank);
    if (dn == node_) {  // the shared-memory fast path of the reference: in-process, not counted
      boxes_[env.dst_rank]->push(std::move(env));
      return;
    }
    const uint64_t framed = distflow::wire::framed_size(env.payload.size(), max_frame_bytes_);
    counters_.on_sent(env.src_rank, env.dst_rank, framed);
    std::lock_guard lk(mu_);
    if (closing_) throw distflow::PeerClosedError("fabric closed");
    out_.push_back(std::move(env));
  }

  distflow::Envelope recv(uint32_t self_rank, uint32_t src_rank, uint32_t tag, uint32_t iteration,
                          std::chrono::milliseconds timeout = distflow::kDefaultRecvTimeout) override {
    check_endpoint(self_rank, "self");
    check_endpoint(src_rank, "src");
    return boxes_[self_rank]->pop_match(src_rank, tag, iteration, timeout);
  }

  distflow::TrafficReport traffic() const override { return counters_.snapshot(); }

  // Collective in effect: the progress threads keep running rounds until every node has called close() and no
  // envelope is pending anywhere; then the mailboxes close.
  void close() override {
    {
      std::lock_guard lk(mu_);
      closing_ = true;
    }
    if (progress_.joinable() && std::this_thread::get_id() != progress_.get_id()) progress_.join();
    for (auto& b : boxes_) b->close();
  }

  uint64_t rounds() const { return rounds_.load(); }

 private:
  static constexpr size_t kHdr = 5;  // src, dst, tag, iteration, payload bytes (u64 each)

  void reserve(void*& dptr, void*& hptr, size_t& cap, size_t bytes) {
    if (bytes <= cap) return;
    const size_t n = std::max(bytes, 2 * cap);
    if (dptr) cudaFree(dptr);
    if (hptr) cudaFreeHost(hptr);
    dfx::store_cuda(cudaMalloc(&dptr, n), "cudaMalloc");
    dfx::store_cuda(cudaMallocHost(&hptr, n), "cudaMallocHost");
    cap = n;
  }

  void progress_loop() {
    try {
      dfx::store_cuda(cudaSetDevice(device_), "cudaSetDevice");
      const uint32_t n = topo_.num_nodes;
      std::vector<int64_t> tab(size_t(n) * n + n), sum(tab.size());
      for (;;) {
        std::deque<distflow::Envelope> batch;
        bool closing;
        {
          std::lock_guard lk(mu_);
          batch.swap(out_);
          closing = closing_;
        }
        // per destination node: packed size
        std::vector<std::vector<const distflow::Envelope*>> per(n);
        std::vector<uint64_t> sbytes(n, 0);
        for (const auto& e : batch) {
          const uint32_t dn = topo_.endpoint_node(e.dst_rank);
          per[dn].push_back(&e);
          sbytes[dn] += 8 * kHdr + ((e.payload.size() + 7) & ~size_t(7));
        }
        std::fill(tab.begin(), tab.end(), 0);
        for (uint32_t p = 0; p < n; ++p) tab[size_t(node_) * n + p] = int64_t(sbytes[p]);
        tab[size_t(n) * n + node_] = closing ? 1 : 0;
        dfx::store_check(dfx_comm_allreduce_i64(comm_.get(), tab.data(), sum.data(), int64_t(tab.size()), stream_));
        ++rounds_;
        bool any = false, all_closing = true;
        for (uint32_t a = 0; a < n; ++a) {
          all_closing = all_closing && sum[size_t(n) * n + a] != 0;
          for (uint32_t b = 0; b < n; ++b) any = any || sum[size_t(a) * n + b] != 0;
        }
        if (!any) {
          if (all_closing) return;
          std::this_thread::sleep_for(std::chrono::microseconds(200));
          continue;
        }
        // pack, one H2D, one all-to-all-v, one D2H, deliver
        std::vector<uint64_t> soff(n), roff(n), rbytes(n);
        uint64_t st = 0, rt = 0;
        for (uint32_t p = 0; p < n; ++p) {
          soff[p] = st;
          st += sbytes[p];
          rbytes[p] = uint64_t(sum[size_t(p) * n + node_]);
          roff[p] = rt;
          rt += rbytes[p];
        }
        reserve(dsend_, hsend_, scap_, std::max<uint64_t>(st, 8));
        reserve(drecv_, hrecv_, rcap_, std::max<uint64_t>(rt, 8));
        for (uint32_t p = 0; p < n; ++p) {
          uint8_t* w = static_cast<uint8_t*>(hsend_) + soff[p];
          for (const distflow::Envelope* e : per[p]) {
            const uint64_t h[kHdr] = {e->src_rank, e->dst_rank, e->tag, e->iteration, e->payload.size()};
            std::memcpy(w, h, sizeof(h));
            w += sizeof(h);
            if (!e->payload.empty()) std::memcpy(w, e->payload.data(), e->payload.size());
            w += (e->payload.size() + 7) & ~size_t(7);
          }
        }
        if (st) dfx::store_cuda(cudaMemcpyAsync(dsend_, hsend_, st, cudaMemcpyHostToDevice, stream_), "H2D");
        dfx::store_check(dfx_comm_alltoallv(comm_.get(), dsend_, soff.data(), sbytes.data(), drecv_, roff.data(),
                                            rbytes.data(), stream_));
        if (rt) dfx::store_cuda(cudaMemcpyAsync(hrecv_, drecv_, rt, cudaMemcpyDeviceToHost, stream_), "D2H");
        dfx::store_cuda(cudaStreamSynchronize(stream_), "sync");
        const uint8_t* r = static_cast<const uint8_t*>(hrecv_);
        const uint8_t* end = r + rt;
        while (r < end) {
          uint64_t h[kHdr];
          std::memcpy(h, r, sizeof(h));
          r += sizeof(h);
          distflow::Envelope env;
          env.src_rank = uint32_t(h[0]);
          env.dst_rank = uint32_t(h[1]);
          env.tag = uint32_t(h[2]);
          env.iteration = uint32_t(h[3]);
          env.payload.assign(r, r + h[4]);
          r += (h[4] + 7) & ~uint64_t(7);
          counters_.on_received(env.src_rank, env.dst_rank,
                                distflow::wire::framed_size(env.payload.size(), max_frame_bytes_));
          boxes_[env.dst_rank]->push(std::move(env));
        }
      }
    } catch (const std::exception& ex) {
      std::fprintf(stderr, "NcclFabric progress thread (node %u): %s\n", node_, ex.what());
      for (auto& b : boxes_) b->close();  // waiting receivers see PeerClosedError instead of hanging
    }
  }

  uint32_t node_;
  dfx::Comm& comm_;
  distflow::detail::TrafficCounters counters_;
  std::vector<std::unique_ptr<distflow::detail::Mailbox>> boxes_;
  std::mutex mu_;
  std::deque<distflow::Envelope> out_;
  bool closing_ = false;
  std::thread progress_;
  std::atomic<uint64_t> rounds_{0};
  int device_ = 0;
  cudaStream_t stream_ = nullptr;
  void *dsend_ = nullptr, *drecv_ = nullptr, *hsend_ = nullptr, *hrecv_ = nullptr;
  size_t scap_ = 0, rcap_ = 0;
};

}  // namespace dfx_distflow
