// dstore.cu -- the distributed DataBuffer: the reference's BufferStore (distflow/data_plane.hpp:225-457) for one
// process per GPU, native end to end (include/dfx.h "Distributed DataBuffer").
//
// One ensure_ready = the reference's exchange (data_plane.hpp:400-442 -> transport.hpp:718-754 all_to_all):
//   1. sizes: one int64 all-reduce over the communicator of the producer groups' record counts -- plus, for the
//      segments of the plan those counts produced last time, each segment's (rollouts, tokens, first token) filled
//      by its owner. When the counts repeat (a training loop), the plan and every segment's size are known after
//      this single round; otherwise the placement is recomputed (dfx_reshard_segments) and a second
//      round fills the new segments' sizes.
//   2. layout: this rank's consumer groups in dp order. A group that is one local run of one producer batch is a
//      zero-copy view (rebased record metadata only). The others are carved out of ONE pooled allocation
//      (cudaMallocFromPoolAsync: stream-ordered, no device synchronization).
//   3. data, all on the caller's stream: one pack kernel writes the metadata of every segment this rank sends;
//      ONE grouped NCCL call posts every cross-GPU send and receive -- token streams go straight from the
//      producer's streams into the consumer's (16-byte aligned ends) or through an aligned staging superset;
//      local segments are copied by one copy kernel on a forked stream, overlapping the transfers; one unpack
//      kernel rebases group_off / cu_seqlens / roll_group and fills ids and channels; the consumer's offsets come
//      back to the host by one small D2H (get() waits for it).
// Ordering needs no barriers: a send reads the producer's streams in its stream order, a receive completes before
// the unpack in the consumer's. Errors map to the reference's types (dfx_status).
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "common.cuh"

#define DFX_NCCL(call)                                                                                   \
  do {                                                                                                   \
    ncclResult_t _r = (call);                                                                            \
    if (_r != ncclSuccess) return ::dfx::fail(DFX_NCCL_ERROR, std::string(#call) + ": " + ncclGetErrorString(_r)); \
  } while (0)

struct dfx_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0, n = 1, device = 0;
  int64_t* d_buf = nullptr;  // small all-reduces
  int64_t* h_buf = nullptr;  // pinned
  int64_t cap = 0;
};

namespace dfx {
namespace {

dfx_status comm_reserve(dfx_comm* c, int64_t n) {
  if (n <= c->cap) return DFX_OK;
  const int64_t cap = std::max<int64_t>(n, 4096);
  if (c->d_buf) cudaFree(c->d_buf);
  if (c->h_buf) cudaFreeHost(c->h_buf);
  c->d_buf = nullptr;
  c->h_buf = nullptr;
  DFX_CUDA(cudaMalloc(&c->d_buf, size_t(cap) * 8));
  DFX_CUDA(cudaMallocHost(&c->h_buf, size_t(cap) * 8));
  c->cap = cap;
  return DFX_OK;
}

// ---- unpack into per-group relative metadata -------------------------------------------------------------------
// One entry per segment: source metadata (a local producer's arrays or a received metadata buffer) and the
// destination arrays of its consumer group, already offset to the segment's first record / rollout.
struct XSeg {
  const uint64_t* ids;
  const int32_t* go;
  const int64_t* cu;
  const double* ch[DFX_MAX_CH];
  int64_t n_rec, n_roll;
  uint64_t* d_ids;
  int32_t* d_go;     // group's group_off + record offset in the group
  int32_t* d_rg;     // group's roll_group + rollout offset in the group
  int64_t* d_cu;     // group's cu + rollout offset in the group
  double* d_ch[DFX_MAX_CH];
  int32_t rec_base;  // record offset of the segment in its group (roll_group values)
  int32_t roll_base; // rollout offset in its group (group_off values)
  int64_t tok_base;  // absolute token index of the segment's first token in the consumer's streams
};
constexpr int kXSegs = 32;
struct XSegBatch {
  XSeg s[kXSegs];
};

__global__ void __launch_bounds__(256) xunpack_kernel(const XSegBatch b, int n_ch) {
  const XSeg& m = b.s[blockIdx.x];
  const int64_t i = int64_t(blockIdx.y) * blockDim.x + threadIdx.x;
  if (i > m.n_rec && i > m.n_roll) return;
  const int64_t g0 = m.go[0], c0 = m.cu[0];
  if (i <= m.n_rec) {
    const int64_t gi = m.go[i];
    m.d_go[i] = (int32_t)(gi - g0 + m.roll_base);
    if (i < m.n_rec) {
      m.d_ids[i] = m.ids[i];
      const int64_t ge = m.go[i + 1];
      for (int64_t j = gi; j < ge; ++j) m.d_rg[j - g0] = m.rec_base + (int32_t)i;
    }
  }
  if (i <= m.n_roll) {
    m.d_cu[i] = m.cu[i] - c0 + m.tok_base;
    if (i < m.n_roll)
      for (int c = 0; c < n_ch; ++c) m.d_ch[c][i] = m.ch[c][i];
  }
}

dfx_status xunpack(const std::vector<XSeg>& segs, int n_ch, cudaStream_t st) {
  for (size_t s0 = 0; s0 < segs.size(); s0 += kXSegs) {
    const size_t n = std::min<size_t>(kXSegs, segs.size() - s0);
    XSegBatch b{};
    int64_t span = 1;
    for (size_t i = 0; i < n; ++i) {
      b.s[i] = segs[s0 + i];
      span = std::max<int64_t>(span, std::max(segs[s0 + i].n_rec, segs[s0 + i].n_roll) + 1);
    }
    xunpack_kernel<<<dim3(unsigned(n), unsigned((span + 255) / 256)), 256, 0, st>>>(b, n_ch);
    DFX_LAUNCH_CHECK("xunpack_kernel");
  }
  return DFX_OK;
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct StageCfg {
  uint32_t pdp, ptp, cdp, ctp;
};

// a put batch: the caller's device pointers + our copy of its host offsets
struct Held {
  dfx_batch b{};
  std::vector<int32_t> hgo;
  std::vector<int64_t> hcu;
};

// a consumer group on this rank
struct Group {
  dfx_batch b{};
  int32_t* pin_go = nullptr;  // pinned host copies (filled by the D2H after the unpack) -- or owned vectors
  int64_t* pin_cu = nullptr;
  std::vector<int32_t> hgo;   // views: rebased on the host at once
  std::vector<int64_t> hcu;
};

struct Ready {
  std::map<uint32_t, Group> groups;
  std::vector<void*> dev_mem;   // pooled device allocations (freed stream-ordered at retire)
  void* pinned = nullptr;       // pinned host block of the consumer offsets
  size_t pinned_bytes = 0;
  cudaEvent_t meta_ev = nullptr;
  bool meta_synced = true;
  uint32_t to_dp = 0, to_tp = 0;
};

struct Entry {
  std::map<uint32_t, Held> by_group;
  bool ready = false;
  Ready r;
};

struct PSeg {
  uint32_t dst, src;
  uint64_t dst_rec, src_rec, count;
  int64_t n_roll = 0, n_tok = 0, t0 = 0;  // sizes + the owner's first token (alignment decisions)
};

struct PlanCache {
  bool valid = false;
  uint32_t to_dp = 0, to_tp = 0;
  std::vector<uint64_t> counts;
  std::vector<PSeg> segs;
};

}  // namespace
}  // namespace dfx

struct dfx_dstore {
  dfx_comm* comm = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // local copies, overlapping the NCCL transfers
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaMemPool_t pool = nullptr;
  int device = 0;
  uint32_t B = 1, W = 1;
  std::vector<int32_t> rank_of_worker;
  int32_t n_streams = 0, n_ch = 0;
  std::vector<uint32_t> esz;
  std::map<std::string, dfx::StageCfg> stages;
  std::map<std::pair<std::string, uint64_t>, dfx::Entry> entries;
  std::map<std::string, dfx::PlanCache> plans;
  std::map<uint64_t, uint32_t> done;
  uint64_t low_water = 0;
  uint32_t local_workers = 0;
  uint64_t suppressed = 0, sent = 0, recvd = 0, copied = 0, plan_hits = 0;
  std::vector<void*> pinned_free;  // recycled pinned blocks (size in pinned_size)
  std::map<void*, size_t> pinned_size;
};

namespace dfx {
namespace {

void* pinned_get(dfx_dstore* s, size_t bytes) {
  for (size_t i = 0; i < s->pinned_free.size(); ++i) {
    void* p = s->pinned_free[i];
    if (s->pinned_size[p] >= bytes) {
      s->pinned_free.erase(s->pinned_free.begin() + long(i));
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, std::max<size_t>(bytes, 1 << 16)) != cudaSuccess) return nullptr;
  s->pinned_size[p] = std::max<size_t>(bytes, 1 << 16);
  return p;
}

dfx_status dev_alloc(dfx_dstore* s, size_t bytes, void** p) {
  DFX_CUDA(cudaMallocFromPoolAsync(p, std::max<size_t>(bytes, 256), s->pool, s->stream));
  return DFX_OK;
}

void retire(dfx_dstore* s, Ready& r) {
  for (void* p : r.dev_mem) cudaFreeAsync(p, s->stream);
  r.dev_mem.clear();
  if (r.meta_ev) {
    cudaEventSynchronize(r.meta_ev);  // the pinned block may still be a D2H target
    cudaEventDestroy(r.meta_ev);
    r.meta_ev = nullptr;
  }
  if (r.pinned) s->pinned_free.push_back(r.pinned);
  r.pinned = nullptr;
}

bool rank_holds_worker(const dfx_dstore* s, uint32_t w) { return s->rank_of_worker[w] == s->comm->rank; }

// ranks that host a TP worker of consumer group d (lead = d * tp, topology.hpp:50)
std::vector<int> dst_ranks(const dfx_dstore* s, uint32_t d, uint32_t tp) {
  std::set<int> r;
  for (uint32_t t = 0; t < tp; ++t) r.insert(s->rank_of_worker[size_t(d) * tp + t]);
  return std::vector<int>(r.begin(), r.end());
}

// sizes of segment sg from its owner's host metadata
void seg_sizes(const Held& h, PSeg& sg) {
  const int64_t r0 = int64_t(sg.src_rec), r1 = r0 + int64_t(sg.count);
  const int32_t s0 = h.hgo[size_t(r0)], s1 = h.hgo[size_t(r1)];
  sg.n_roll = s1 - s0;
  sg.t0 = h.hcu[size_t(s0)];
  sg.n_tok = h.hcu[size_t(s1)] - sg.t0;
}

dfx_status plan_segments(const dfx_dstore* s, const StageCfg& c, uint32_t to_dp, uint32_t to_tp,
                         const std::vector<uint64_t>& counts, std::vector<PSeg>& out) {
  const int64_t n = dfx_reshard_segments(s->B, s->W, c.pdp, c.ptp, to_dp, to_tp, counts.data(), nullptr, 0);
  if (n < 0) return dfx_status(-n);
  std::vector<dfx_segment> segs(size_t(std::max<int64_t>(n, 1)));
  dfx_reshard_segments(s->B, s->W, c.pdp, c.ptp, to_dp, to_tp, counts.data(), segs.data(), n);
  out.clear();
  for (int64_t i = 0; i < n; ++i) {
    PSeg p;
    p.dst = segs[size_t(i)].dst_group;
    p.src = segs[size_t(i)].src_group;
    p.dst_rec = segs[size_t(i)].dst_rec;
    p.src_rec = segs[size_t(i)].src_rec;
    p.count = segs[size_t(i)].count;
    out.push_back(p);
  }
  return DFX_OK;
}

// element range moved for a segment's stream k: exact when both ends are 16-byte aligned, else the 8-element
// aligned superset into a staging buffer (NCCL point-to-point runs far slower on misaligned buffers)
bool seg_direct(int64_t t0, int64_t dt, uint32_t esz) {
  return ((t0 * int64_t(esz)) & 15) == 0 && ((dt * int64_t(esz)) & 15) == 0;
}

dfx_status run_exchange(dfx_dstore* s, const StageCfg& c, uint32_t to_dp, uint32_t to_tp, Entry& e,
                        const std::vector<PSeg>& segs) {
  const int me = s->comm->rank;
  cudaStream_t st = s->stream;
  Ready& r = e.r;
  r.to_dp = to_dp;
  r.to_tp = to_tp;
  std::vector<int> src_rank(c.pdp);
  for (uint32_t p = 0; p < c.pdp; ++p) src_rank[p] = s->rank_of_worker[size_t(p) * c.ptp];
  std::vector<std::vector<int>> dranks(to_dp);
  std::vector<uint32_t> local_dst;
  for (uint32_t d = 0; d < to_dp; ++d) {
    dranks[d] = dst_ranks(s, d, to_tp);
    if (std::find(dranks[d].begin(), dranks[d].end(), me) != dranks[d].end()) local_dst.push_back(d);
  }
  std::vector<std::vector<size_t>> seg_of(to_dp);
  for (size_t i = 0; i < segs.size(); ++i) seg_of[segs[i].dst].push_back(i);

  // ---- layout of this rank's consumer groups ----
  struct GL {
    bool view = false;
    int64_t R = 0, S = 0, T = 0;
    size_t o_ids = 0, o_go = 0, o_rg = 0, o_cu = 0, o_ch = 0;  // element offsets into the shared arrays
    int64_t tok = 0;                                           // first token in the shared streams
  };
  std::map<uint32_t, GL> gl;
  int64_t R = 0, S = 0, T = 0, NG = 0;
  for (uint32_t d : local_dst) {
    GL g;
    const auto& ix = seg_of[d];
    g.view = ix.size() == 1 && src_rank[segs[ix[0]].src] == me;
    for (size_t i : ix) {
      g.R += int64_t(segs[i].count);
      g.S += segs[i].n_roll;
      g.T += segs[i].n_tok;
    }
    if (!g.view) {
      g.o_ids = size_t(R);
      g.o_go = size_t(R + NG);
      g.o_rg = size_t(S);
      g.o_cu = size_t(S + NG);
      g.o_ch = size_t(S);
      g.tok = T;
      R += g.R;
      S += g.S;
      T += g.T;
      ++NG;
    }
    gl[d] = g;
  }
  // one allocation: ids | go | rg | cu | ch | streams (each 256-byte aligned, streams padded for over-reads)
  size_t off = 0;
  const size_t b_ids = off; off += al256(size_t(R) * 8);
  const size_t b_go = off; off += al256(size_t(R + NG) * 4);
  const size_t b_rg = off; off += al256(size_t(S) * 4);
  const size_t b_cu = off; off += al256(size_t(S + NG) * 8);
  std::vector<size_t> b_ch(s->n_ch), b_st(s->n_streams);
  for (int c2 = 0; c2 < s->n_ch; ++c2) { b_ch[c2] = off; off += al256(size_t(S) * 8); }
  for (int k = 0; k < s->n_streams; ++k) { b_st[k] = off; off += al256(size_t(T + 64) * s->esz[k]); }
  uint8_t* mem = nullptr;
  if (NG > 0) {
    void* p = nullptr;
    dfx_status stt = dev_alloc(s, off, &p);
    if (stt) return stt;
    mem = static_cast<uint8_t*>(p);
    r.dev_mem.push_back(p);
  }

  // ---- views and group descriptors ----
  for (uint32_t d : local_dst) {
    GL& g = gl[d];
    Group grp;
    if (g.view) {
      const PSeg& sg = segs[seg_of[d][0]];
      const Held& h = e.by_group.at(sg.src);
      const int64_t r0 = int64_t(sg.src_rec), r1 = r0 + int64_t(sg.count);
      const int32_t s0 = h.hgo[size_t(r0)], s1 = h.hgo[size_t(r1)];
      dfx_batch v = h.b;
      v.n_records = r1 - r0;
      v.n_rollouts = s1 - s0;
      v.ids = h.b.ids + r0;
      v.cu_seqlens = h.b.cu_seqlens + s0;
      for (int c2 = 0; c2 < s->n_ch; ++c2) v.ch[c2] = h.b.ch[c2] ? h.b.ch[c2] + s0 : nullptr;
      v.token_base = h.hcu[size_t(s0)];
      v.token_span = h.hcu[size_t(s1)] - v.token_base;
      grp.hcu.assign(h.hcu.begin() + s0, h.hcu.begin() + s1 + 1);
      grp.hgo.resize(size_t(r1 - r0 + 1));
      for (int64_t q = r0; q <= r1; ++q) grp.hgo[size_t(q - r0)] = h.hgo[size_t(q)] - s0;
      if (r0 != 0 || r1 != h.b.n_records) {  // rebased record metadata on the device
        void* p = nullptr;
        const size_t nb = al256(size_t(r1 - r0 + 1) * 4) + size_t(s1 - s0) * 4 + 16;
        dfx_status stt = dev_alloc(s, nb, &p);
        if (stt) return stt;
        r.dev_mem.push_back(p);
        int32_t* go = static_cast<int32_t*>(p);
        int32_t* rg = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(p) + al256(size_t(r1 - r0 + 1) * 4));
        stt = dfx_view_meta(h.b.group_off, h.b.roll_group, r0, r1, s1 - s0, go, rg, st);
        if (stt) return stt;
        v.group_off = go;
        v.roll_group = rg;
      }
      v.h_group_off = grp.hgo.data();
      v.h_cu = grp.hcu.data();
      grp.b = v;
    } else {
      dfx_batch v{};
      v.n_records = g.R;
      v.n_rollouts = g.S;
      v.token_base = g.tok;
      v.token_span = g.T;
      v.ids = reinterpret_cast<uint64_t*>(mem + b_ids) + g.o_ids;
      v.group_off = reinterpret_cast<int32_t*>(mem + b_go) + g.o_go;
      v.roll_group = reinterpret_cast<int32_t*>(mem + b_rg) + g.o_rg;
      v.cu_seqlens = reinterpret_cast<int64_t*>(mem + b_cu) + g.o_cu;
      for (int c2 = 0; c2 < s->n_ch; ++c2) v.ch[c2] = reinterpret_cast<double*>(mem + b_ch[c2]) + g.o_ch;
      for (int k = 0; k < s->n_streams; ++k) v.st[k] = mem + b_st[k];
      grp.b = v;
    }
    r.groups[d] = std::move(grp);
  }
  for (auto& kv : r.groups) {  // (vectors moved: refresh host pointers of views)
    if (gl[kv.first].view) {
      kv.second.b.h_group_off = kv.second.hgo.data();
      kv.second.b.h_cu = kv.second.hcu.data();
    }
  }

  // ---- transfers ----
  // sends: every segment whose producer group lives here, to every other rank hosting a TP worker of its group
  struct Send {
    size_t seg;
    int to;
  };
  struct Recv {
    size_t seg;
    int from;
  };
  std::vector<Send> sends;
  std::vector<Recv> recvs;
  for (size_t i = 0; i < segs.size(); ++i) {
    const PSeg& sg = segs[i];
    const int src = src_rank[sg.src];
    for (int rk : dranks[sg.dst]) {
      if (src == me && rk != me) sends.push_back({i, rk});
      if (rk == me && src != me) recvs.push_back({i, src});
    }
  }
  // destination token position (absolute in the consumer streams) of every segment of a local, non-view group
  std::vector<int64_t> seg_dt(segs.size(), -1), seg_dr(segs.size(), 0), seg_ds(segs.size(), 0);
  for (uint32_t d : local_dst) {
    const GL& g = gl[d];
    if (g.view) continue;
    int64_t dr = 0, ds = 0, dt = g.tok;
    for (size_t i : seg_of[d]) {
      seg_dr[i] = dr;
      seg_ds[i] = ds;
      seg_dt[i] = dt;
      dr += int64_t(segs[i].count);
      ds += segs[i].n_roll;
      dt += segs[i].n_tok;
    }
  }
  // the destination token position of a segment on ANOTHER rank (the sender needs it for the alignment rule):
  // every rank lays out its groups the same way, so recompute it for the receiver
  auto remote_dt = [&](size_t i, int rk) -> int64_t {
    int64_t t = 0;
    for (uint32_t d = 0; d < to_dp; ++d) {
      if (std::find(dranks[d].begin(), dranks[d].end(), rk) == dranks[d].end()) continue;
      const auto& ix = seg_of[d];
      const bool view = ix.size() == 1 && src_rank[segs[ix[0]].src] == rk;
      if (view) continue;
      for (size_t j : ix) {
        if (j == i) return t;
        t += segs[j].n_tok;
      }
    }
    return 0;
  };

  const int64_t n_ch = s->n_ch;
  auto meta_bytes = [&](const PSeg& sg) { return size_t(dfx_reshard_pack_bytes(int64_t(sg.count), sg.n_roll, int32_t(n_ch))); };
  // scratch: send metadata, receive metadata, staging supersets -- one pooled block, freed after the unpack
  size_t scratch = 0;
  std::vector<size_t> o_send(sends.size()), o_recv(recvs.size());
  std::vector<std::vector<size_t>> o_stage(recvs.size(), std::vector<size_t>(s->n_streams, SIZE_MAX));
  for (size_t q = 0; q < sends.size(); ++q) { o_send[q] = scratch; scratch += al256(meta_bytes(segs[sends[q].seg])); }
  for (size_t q = 0; q < recvs.size(); ++q) {
    const PSeg& sg = segs[recvs[q].seg];
    o_recv[q] = scratch;
    scratch += al256(meta_bytes(sg));
    if (sg.n_tok == 0) continue;
    for (int k = 0; k < s->n_streams; ++k) {
      if (seg_direct(sg.t0, seg_dt[recvs[q].seg], s->esz[k])) continue;
      const int64_t a0 = sg.t0 & ~int64_t(7), a1 = (sg.t0 + sg.n_tok + 7) & ~int64_t(7);
      o_stage[q][k] = scratch;
      scratch += al256(size_t(a1 - a0) * s->esz[k]);
    }
  }
  uint8_t* scr = nullptr;
  if (scratch) {
    void* p = nullptr;
    dfx_status stt = dev_alloc(s, scratch, &p);
    if (stt) return stt;
    scr = static_cast<uint8_t*>(p);
  }
  if (!sends.empty()) {  // metadata of every sent segment, one pack launch
    std::vector<dfx_seg_meta> pm(sends.size());
    std::vector<uint8_t*> outp(sends.size());
    for (size_t q = 0; q < sends.size(); ++q) {
      const PSeg& sg = segs[sends[q].seg];
      const Held& h = e.by_group.at(sg.src);
      const int64_t r0 = int64_t(sg.src_rec);
      const int32_t s0 = h.hgo[size_t(r0)];
      dfx_seg_meta m{};
      m.ids = h.b.ids + r0;
      m.group_off = h.b.group_off + r0;
      m.cu = h.b.cu_seqlens + s0;
      for (int c2 = 0; c2 < s->n_ch; ++c2) m.ch[c2] = h.b.ch[c2] + s0;
      m.n_rec = int64_t(sg.count);
      m.n_roll = sg.n_roll;
      pm[q] = m;
      outp[q] = scr + o_send[q];
    }
    dfx_status stt = dfx_reshard_pack(pm.data(), int32_t(pm.size()), s->n_ch, outp.data(), st);
    if (stt) return stt;
  }
  // local segments of non-view groups: one copy kernel on the side stream, concurrent with the transfers
  std::vector<uint64_t> cp_dst, cp_src, cp_n;
  for (uint32_t d : local_dst) {
    if (gl[d].view) continue;
    for (size_t i : seg_of[d]) {
      const PSeg& sg = segs[i];
      if (src_rank[sg.src] != me || sg.n_tok == 0) continue;
      const Held& h = e.by_group.at(sg.src);
      for (int k = 0; k < s->n_streams; ++k) {
        const size_t es = s->esz[k];
        cp_dst.push_back(uint64_t(reinterpret_cast<uintptr_t>(mem + b_st[k] + size_t(seg_dt[i]) * es)));
        cp_src.push_back(uint64_t(reinterpret_cast<uintptr_t>(static_cast<const uint8_t*>(h.b.st[k]) + size_t(sg.t0) * es)));
        cp_n.push_back(uint64_t(sg.n_tok) * es);
        s->copied += uint64_t(sg.n_tok) * es;
      }
    }
  }
  if (!cp_n.empty()) {
    DFX_CUDA(cudaEventRecord(s->ev_fork, st));
    DFX_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
    dfx_status stt = dfx_copy_many(int64_t(cp_n.size()), cp_dst.data(), cp_src.data(), cp_n.data(), s->side);
    if (stt) return stt;
    DFX_CUDA(cudaEventRecord(s->ev_join, s->side));
  }
  if (!sends.empty() || !recvs.empty()) {
    DFX_NCCL(ncclGroupStart());
    // per peer, both sides post in global segment order: metadata, then the streams in schema order
    for (size_t q = 0; q < sends.size(); ++q) {
      const PSeg& sg = segs[sends[q].seg];
      const int to = sends[q].to;
      DFX_NCCL(ncclSend(scr + o_send[q], meta_bytes(sg), ncclUint8, to, s->comm->nccl, st));
      s->sent += meta_bytes(sg);
      if (sg.n_tok == 0) continue;
      const Held& h = e.by_group.at(sg.src);
      const int64_t dt = remote_dt(sends[q].seg, to);
      for (int k = 0; k < s->n_streams; ++k) {
        const size_t es = s->esz[k];
        const uint8_t* base = static_cast<const uint8_t*>(h.b.st[k]);
        if (seg_direct(sg.t0, dt, s->esz[k])) {
          DFX_NCCL(ncclSend(base + size_t(sg.t0) * es, size_t(sg.n_tok) * es, ncclUint8, to, s->comm->nccl, st));
          s->sent += size_t(sg.n_tok) * es;
        } else {
          const int64_t a0 = sg.t0 & ~int64_t(7), a1 = (sg.t0 + sg.n_tok + 7) & ~int64_t(7);
          DFX_NCCL(ncclSend(base + size_t(a0) * es, size_t(a1 - a0) * es, ncclUint8, to, s->comm->nccl, st));
          s->sent += size_t(a1 - a0) * es;
        }
      }
    }
    for (size_t q = 0; q < recvs.size(); ++q) {
      const PSeg& sg = segs[recvs[q].seg];
      const int from = recvs[q].from;
      DFX_NCCL(ncclRecv(scr + o_recv[q], meta_bytes(sg), ncclUint8, from, s->comm->nccl, st));
      s->recvd += meta_bytes(sg);
      if (sg.n_tok == 0) continue;
      for (int k = 0; k < s->n_streams; ++k) {
        const size_t es = s->esz[k];
        if (o_stage[q][k] == SIZE_MAX) {
          DFX_NCCL(ncclRecv(mem + b_st[k] + size_t(seg_dt[recvs[q].seg]) * es, size_t(sg.n_tok) * es, ncclUint8,
                            from, s->comm->nccl, st));
          s->recvd += size_t(sg.n_tok) * es;
        } else {
          const int64_t a0 = sg.t0 & ~int64_t(7), a1 = (sg.t0 + sg.n_tok + 7) & ~int64_t(7);
          DFX_NCCL(ncclRecv(scr + o_stage[q][k], size_t(a1 - a0) * es, ncclUint8, from, s->comm->nccl, st));
          s->recvd += size_t(a1 - a0) * es;
        }
      }
    }
    DFX_NCCL(ncclGroupEnd());
  }
  // staged supersets -> exact destination ranges
  {
    std::vector<uint64_t> pd, ps, pn;
    for (size_t q = 0; q < recvs.size(); ++q) {
      const PSeg& sg = segs[recvs[q].seg];
      for (int k = 0; k < s->n_streams; ++k) {
        if (sg.n_tok == 0 || o_stage[q][k] == SIZE_MAX) continue;
        const size_t es = s->esz[k];
        const int64_t head = sg.t0 - (sg.t0 & ~int64_t(7));
        pd.push_back(uint64_t(reinterpret_cast<uintptr_t>(mem + b_st[k] + size_t(seg_dt[recvs[q].seg]) * es)));
        ps.push_back(uint64_t(reinterpret_cast<uintptr_t>(scr + o_stage[q][k] + size_t(head) * es)));
        pn.push_back(uint64_t(sg.n_tok) * es);
      }
    }
    if (!pn.empty()) {
      dfx_status stt = dfx_copy_many(int64_t(pn.size()), pd.data(), ps.data(), pn.data(), st);
      if (stt) return stt;
    }
  }
  // metadata of every segment of the non-view groups: one unpack
  std::vector<XSeg> xs;
  std::map<size_t, size_t> recv_of;
  for (size_t q = 0; q < recvs.size(); ++q) recv_of[recvs[q].seg] = q;
  for (uint32_t d : local_dst) {
    const GL& g = gl[d];
    if (g.view) continue;
    const Group& grp = r.groups[d];
    for (size_t i : seg_of[d]) {
      const PSeg& sg = segs[i];
      XSeg x{};
      if (src_rank[sg.src] == me) {
        const Held& h = e.by_group.at(sg.src);
        const int64_t r0 = int64_t(sg.src_rec);
        const int32_t s0 = h.hgo[size_t(r0)];
        x.ids = h.b.ids + r0;
        x.go = h.b.group_off + r0;
        x.cu = h.b.cu_seqlens + s0;
        for (int c2 = 0; c2 < s->n_ch; ++c2) x.ch[c2] = h.b.ch[c2] + s0;
      } else {  // received metadata: ids u64[n_rec] | cu i64[n_roll+1] | ch f64[n_ch][n_roll] | go i32[n_rec+1]
        const uint8_t* b = scr + o_recv[recv_of.at(i)];
        const int64_t nr = int64_t(sg.count), ns = sg.n_roll;
        x.ids = reinterpret_cast<const uint64_t*>(b);
        x.cu = reinterpret_cast<const int64_t*>(b + 8 * nr);
        for (int c2 = 0; c2 < s->n_ch; ++c2)
          x.ch[c2] = reinterpret_cast<const double*>(b + 8 * nr + 8 * (ns + 1) + 8 * c2 * ns);
        x.go = reinterpret_cast<const int32_t*>(b + 8 * nr + 8 * (ns + 1) + 8 * n_ch * ns);
      }
      x.n_rec = int64_t(sg.count);
      x.n_roll = sg.n_roll;
      x.d_ids = const_cast<uint64_t*>(grp.b.ids) + seg_dr[i];
      x.d_go = const_cast<int32_t*>(grp.b.group_off) + seg_dr[i];
      x.d_rg = const_cast<int32_t*>(grp.b.roll_group) + seg_ds[i];
      x.d_cu = const_cast<int64_t*>(grp.b.cu_seqlens) + seg_ds[i];
      for (int c2 = 0; c2 < s->n_ch; ++c2) x.d_ch[c2] = const_cast<double*>(grp.b.ch[c2]) + seg_ds[i];
      x.rec_base = int32_t(seg_dr[i]);
      x.roll_base = int32_t(seg_ds[i]);
      x.tok_base = seg_dt[i];
      xs.push_back(x);
    }
  }
  if (!cp_n.empty()) DFX_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
  if (!xs.empty()) {
    dfx_status stt = xunpack(xs, s->n_ch, st);
    if (stt) return stt;
  }
  if (scr) DFX_CUDA(cudaFreeAsync(scr, st));
  // consumer offsets back to the host (get() waits for them)
  if (NG > 0) {
    size_t pb = 0;
    for (uint32_t d : local_dst)
      if (!gl[d].view) pb += al256(size_t(gl[d].R + 1) * 4) + al256(size_t(gl[d].S + 1) * 8);
    r.pinned = pinned_get(s, pb);
    if (!r.pinned) return fail(DFX_CUDA_ERROR, "cudaMallocHost failed");
    uint8_t* hp = static_cast<uint8_t*>(r.pinned);
    for (uint32_t d : local_dst) {
      if (gl[d].view) continue;
      Group& grp = r.groups[d];
      grp.pin_go = reinterpret_cast<int32_t*>(hp);
      hp += al256(size_t(gl[d].R + 1) * 4);
      grp.pin_cu = reinterpret_cast<int64_t*>(hp);
      hp += al256(size_t(gl[d].S + 1) * 8);
      DFX_CUDA(cudaMemcpyAsync(grp.pin_go, grp.b.group_off, size_t(gl[d].R + 1) * 4, cudaMemcpyDeviceToHost, st));
      DFX_CUDA(cudaMemcpyAsync(grp.pin_cu, grp.b.cu_seqlens, size_t(gl[d].S + 1) * 8, cudaMemcpyDeviceToHost, st));
      grp.b.h_group_off = grp.pin_go;
      grp.b.h_cu = grp.pin_cu;
    }
    DFX_CUDA(cudaEventCreateWithFlags(&r.meta_ev, cudaEventDisableTiming));
    DFX_CUDA(cudaEventRecord(r.meta_ev, st));
    r.meta_synced = false;
  }
  return DFX_OK;
}

}  // namespace
}  // namespace dfx

using namespace dfx;

extern "C" {

dfx_status dfx_comm_unique_id(void* id_out) {
  if (!id_out) return fail(DFX_INVALID_ARGUMENT, "dfx_comm_unique_id: null");
  static_assert(sizeof(ncclUniqueId) == DFX_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  DFX_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return DFX_OK;
}

dfx_status dfx_comm_init(const void* id, int32_t n_ranks, int32_t rank, dfx_comm** out) {
  if (!id || !out || n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(DFX_INVALID_ARGUMENT, "dfx_comm_init: bad argument");
  auto c = std::make_unique<dfx_comm>();
  DFX_CUDA(cudaGetDevice(&c->device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  DFX_NCCL(ncclCommInitRank(&c->nccl, n_ranks, uid, rank));
  c->rank = rank;
  c->n = n_ranks;
  dfx_status st = comm_reserve(c.get(), 4096);
  if (st) return st;
  *out = c.release();
  return DFX_OK;
}

dfx_status dfx_comm_destroy(dfx_comm* c) {
  if (!c) return DFX_OK;
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->d_buf) cudaFree(c->d_buf);
  if (c->h_buf) cudaFreeHost(c->h_buf);
  delete c;
  return DFX_OK;
}

int32_t dfx_comm_rank(const dfx_comm* c) { return c ? c->rank : -1; }
int32_t dfx_comm_size(const dfx_comm* c) { return c ? c->n : 0; }

dfx_status dfx_comm_allreduce_i64(dfx_comm* c, const int64_t* in, int64_t* out, int64_t n, dfx_stream stream) {
  if (!c || (n > 0 && (!in || !out))) return fail(DFX_INVALID_ARGUMENT, "dfx_comm_allreduce_i64: bad argument");
  if (n <= 0) return DFX_OK;
  dfx_status st = comm_reserve(c, n);
  if (st) return st;
  std::memcpy(c->h_buf, in, size_t(n) * 8);
  DFX_CUDA(cudaMemcpyAsync(c->d_buf, c->h_buf, size_t(n) * 8, cudaMemcpyHostToDevice, stream));
  DFX_NCCL(ncclAllReduce(c->d_buf, c->d_buf, size_t(n), ncclInt64, ncclSum, c->nccl, stream));
  DFX_CUDA(cudaMemcpyAsync(c->h_buf, c->d_buf, size_t(n) * 8, cudaMemcpyDeviceToHost, stream));
  DFX_CUDA(cudaStreamSynchronize(stream));
  std::memcpy(out, c->h_buf, size_t(n) * 8);
  return DFX_OK;
}

dfx_status dfx_dstore_create(const dfx_dstore_cfg* cfg, dfx_comm* comm, dfx_stream stream, dfx_dstore** out) {
  if (!cfg || !comm || !out || !cfg->rank_of_worker) return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_create: null argument");
  if (cfg->num_nodes == 0 || cfg->workers_per_node == 0)
    return fail(DFX_LAYOUT_ERROR, "topology must have at least one node and one worker per node");
  if (cfg->n_streams < 0 || cfg->n_streams > DFX_MAX_STREAMS || cfg->n_ch < 0 || cfg->n_ch > DFX_MAX_CH)
    return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_create: too many streams or channels");
  auto s = std::make_unique<dfx_dstore>();
  s->comm = comm;
  s->stream = stream;
  s->B = cfg->num_nodes;
  s->W = cfg->workers_per_node;
  const uint32_t world = s->B * s->W;
  s->rank_of_worker.assign(cfg->rank_of_worker, cfg->rank_of_worker + world);
  for (uint32_t w = 0; w < world; ++w) {
    if (s->rank_of_worker[w] < 0 || s->rank_of_worker[w] >= comm->n)
      return fail(DFX_LAYOUT_ERROR, "rank_of_worker maps a worker outside the communicator");
    if (s->rank_of_worker[w] == comm->rank) ++s->local_workers;
  }
  s->n_streams = cfg->n_streams;
  s->n_ch = cfg->n_ch;
  s->esz.assign(cfg->stream_esz, cfg->stream_esz + cfg->n_streams);
  for (int32_t i = 0; i < cfg->n_stages; ++i)
    s->stages[cfg->stage_names[i]] = StageCfg{cfg->produced_dp[i], cfg->produced_tp[i],
                                              cfg->consumed_dp ? cfg->consumed_dp[i] : 0u,
                                              cfg->consumed_tp ? cfg->consumed_tp[i] : 0u};
  DFX_CUDA(cudaGetDevice(&s->device));
  DFX_CUDA(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
  DFX_CUDA(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
  DFX_CUDA(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = s->device;
  DFX_CUDA(cudaMemPoolCreate(&s->pool, &props));
  uint64_t keep = UINT64_MAX;  // keep freed blocks for reuse: a steady-state loop allocates nothing
  DFX_CUDA(cudaMemPoolSetAttribute(s->pool, cudaMemPoolAttrReleaseThreshold, &keep));
  *out = s.release();
  return DFX_OK;
}

dfx_status dfx_dstore_destroy(dfx_dstore* s) {
  if (!s) return DFX_OK;
  for (auto& kv : s->entries) retire(s, kv.second.r);
  cudaStreamSynchronize(s->stream);
  for (void* p : s->pinned_free) cudaFreeHost(p);
  if (s->pool) cudaMemPoolDestroy(s->pool);
  if (s->side) cudaStreamDestroy(s->side);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  delete s;
  return DFX_OK;
}

dfx_status dfx_dstore_put(dfx_dstore* s, const char* stage, uint64_t it, uint32_t dp, uint32_t tp, const dfx_batch* b,
                          int32_t* accepted) {
  if (!s || !stage || !b) return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_put: null argument");
  if (accepted) *accepted = 0;
  auto sc = s->stages.find(stage);
  if (sc == s->stages.end()) return fail(DFX_UNKNOWN_STAGE, std::string("stage '") + stage + "' not in plan");
  if (it < s->low_water)
    return fail(DFX_STALE_ITERATION, "put for iteration " + std::to_string(it) + " below low water " +
                                         std::to_string(s->low_water));  // data_plane.hpp:241-244
  if (tp != 0) {  // only TP rank 0 puts (:245-248)
    ++s->suppressed;
    return DFX_OK;
  }
  if (dp >= sc->second.pdp) return fail(DFX_ERROR, "put from dp group " + std::to_string(dp) + " out of range");
  if (s->rank_of_worker[size_t(dp) * sc->second.ptp] != s->comm->rank)
    return fail(DFX_ERROR, "put from dp group " + std::to_string(dp) + " not local to rank " +
                               std::to_string(s->comm->rank));  // :249-254
  Entry& e = s->entries[{stage, it}];
  if (e.by_group.count(dp) || e.ready)
    return fail(DFX_ERROR, std::string("duplicate put for stage '") + stage + "' group " + std::to_string(dp));  // :256-258
  if (b->n_records > 0 && (!b->h_group_off || !b->h_cu))
    return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_put: the batch needs its host offsets (h_group_off, h_cu)");
  if (b->n_records > 0 && (!b->ids || !b->group_off || !b->roll_group || !b->cu_seqlens))
    return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_put: the batch needs ids, group_off, roll_group and cu_seqlens");
  for (int32_t c = 0; c < s->n_ch && b->n_rollouts > 0; ++c)
    if (!b->ch[c]) return fail(DFX_MISSING_CHANNEL, "dfx_dstore_put: channel " + std::to_string(c) + " missing");
  for (int32_t k = 0; k < s->n_streams && b->token_span > 0; ++k)
    if (!b->st[k]) return fail(DFX_MISSING_CHANNEL, "dfx_dstore_put: token stream " + std::to_string(k) + " missing");
  Held h;
  h.b = *b;
  h.hgo.assign(b->h_group_off, b->h_group_off + b->n_records + 1);
  h.hcu.assign(b->h_cu, b->h_cu + b->n_rollouts + 1);
  if (b->n_records == 0) {
    h.hgo.assign(1, 0);
    h.hcu.assign(1, b->token_base);
  }
  e.by_group.emplace(dp, std::move(h));
  if (accepted) *accepted = 1;
  return DFX_OK;
}

dfx_status dfx_dstore_ensure_ready(dfx_dstore* s, const char* stage, uint64_t it, uint32_t to_dp, uint32_t to_tp) {
  if (!s || !stage) return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_ensure_ready: null argument");
  auto sc = s->stages.find(stage);
  if (sc == s->stages.end()) return fail(DFX_UNKNOWN_STAGE, std::string("stage '") + stage + "' not in plan");
  const StageCfg& c = sc->second;
  if (c.cdp) {
    to_dp = c.cdp;
    to_tp = c.ctp;
  }
  if (to_dp == 0 || to_tp == 0) return fail(DFX_LAYOUT_ERROR, "dp_size and tp_size must be positive for stage '" +
                                                                  std::string(stage) + "'");
  if (it < s->low_water)
    return fail(DFX_STALE_ITERATION, "get for iteration " + std::to_string(it) + " below low water " +
                                         std::to_string(s->low_water));
  Entry& e = s->entries[{stage, it}];
  if (e.ready) return DFX_OK;
  const int me = s->comm->rank;
  std::vector<uint32_t> local_p;
  for (uint32_t p = 0; p < c.pdp; ++p)
    if (s->rank_of_worker[size_t(p) * c.ptp] == me) local_p.push_back(p);
  size_t missing = 0;
  for (uint32_t p : local_p) missing += e.by_group.count(p) ? 0 : 1;
  if (missing)
    return fail(DFX_NOT_READY, std::string("stage '") + stage + "' iteration " + std::to_string(it) +
                                   " not ready: " + std::to_string(missing) + " puts outstanding");  // :340-344

  // ---- sizes: one all-reduce (speculating on last time's plan), a second only when the counts changed ----
  PlanCache& pc = s->plans[stage];
  const bool spec = pc.valid && pc.to_dp == to_dp && pc.to_tp == to_tp;
  const size_t nsp = spec ? pc.segs.size() : 0;
  std::vector<int64_t> tab(c.pdp + 3 * nsp, 0), sum(tab.size());
  for (uint32_t p : local_p) tab[p] = e.by_group.at(p).b.n_records;
  if (spec) {
    for (size_t i = 0; i < nsp; ++i) {
      PSeg sg = pc.segs[i];
      auto h = e.by_group.find(sg.src);
      if (h == e.by_group.end() || sg.src_rec + sg.count > uint64_t(h->second.b.n_records)) continue;
      seg_sizes(h->second, sg);
      tab[c.pdp + 3 * i] = sg.n_roll;
      tab[c.pdp + 3 * i + 1] = sg.n_tok;
      tab[c.pdp + 3 * i + 2] = sg.t0;
    }
  }
  dfx_status st = dfx_comm_allreduce_i64(s->comm, tab.data(), sum.data(), int64_t(tab.size()), s->stream);
  if (st) return st;
  std::vector<uint64_t> counts(c.pdp);
  for (uint32_t p = 0; p < c.pdp; ++p) counts[p] = uint64_t(sum[p]);
  std::vector<PSeg> segs;
  if (spec && counts == pc.counts) {
    segs = pc.segs;
    for (size_t i = 0; i < nsp; ++i) {
      segs[i].n_roll = sum[c.pdp + 3 * i];
      segs[i].n_tok = sum[c.pdp + 3 * i + 1];
      segs[i].t0 = sum[c.pdp + 3 * i + 2];
    }
    ++s->plan_hits;
  } else {
    st = plan_segments(s, c, to_dp, to_tp, counts, segs);
    if (st) return st;
    std::vector<int64_t> t2(3 * segs.size(), 0), s2(t2.size());
    for (size_t i = 0; i < segs.size(); ++i) {
      auto h = e.by_group.find(segs[i].src);
      if (h == e.by_group.end()) continue;
      seg_sizes(h->second, segs[i]);
      t2[3 * i] = segs[i].n_roll;
      t2[3 * i + 1] = segs[i].n_tok;
      t2[3 * i + 2] = segs[i].t0;
    }
    st = dfx_comm_allreduce_i64(s->comm, t2.data(), s2.data(), int64_t(t2.size()), s->stream);
    if (st) return st;
    for (size_t i = 0; i < segs.size(); ++i) {
      segs[i].n_roll = s2[3 * i];
      segs[i].n_tok = s2[3 * i + 1];
      segs[i].t0 = s2[3 * i + 2];
    }
    pc.valid = true;
    pc.to_dp = to_dp;
    pc.to_tp = to_tp;
    pc.counts = counts;
    pc.segs = segs;
  }
  st = run_exchange(s, c, to_dp, to_tp, e, segs);
  if (st) return st;
  e.ready = true;
  return DFX_OK;
}

dfx_status dfx_dstore_get(dfx_dstore* s, const char* stage, uint64_t it, uint32_t dest_dp, uint32_t to_dp,
                          uint32_t to_tp, dfx_batch* out) {
  if (!out) return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_get: null output");
  dfx_status st = dfx_dstore_ensure_ready(s, stage, it, to_dp, to_tp);
  if (st) return st;
  Entry& e = s->entries[{stage, it}];
  auto g = e.r.groups.find(dest_dp);
  if (g == e.r.groups.end())
    return fail(DFX_ERROR, "dp group " + std::to_string(dest_dp) + " not local to rank " +
                               std::to_string(s->comm->rank));  // :276-280
  if (!e.r.meta_synced) {
    DFX_CUDA(cudaEventSynchronize(e.r.meta_ev));
    e.r.meta_synced = true;
  }
  *out = g->second.b;
  return DFX_OK;
}

dfx_status dfx_dstore_worker_done(dfx_dstore* s, uint64_t it) {
  if (!s) return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_worker_done: null");
  const uint32_t n = ++s->done[it];
  if (n < s->local_workers) return DFX_OK;
  s->done.erase(it);
  s->low_water = std::max(s->low_water, it + 1);
  for (auto kv = s->entries.begin(); kv != s->entries.end();) {
    if (kv->first.second < s->low_water) {
      retire(s, kv->second.r);
      kv = s->entries.erase(kv);
    } else {
      ++kv;
    }
  }
  return DFX_OK;
}

dfx_status dfx_dstore_stats(const dfx_dstore* s, uint64_t* out) {
  if (!s || !out) return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_stats: null");
  out[0] = s->suppressed;
  out[1] = s->sent;
  out[2] = s->recvd;
  out[3] = s->copied;
  out[4] = s->plan_hits;
  return DFX_OK;
}

}  // extern "C"
