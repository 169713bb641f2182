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
//   3. data, all on the caller's stream. Transport "pull" (default): every producer allocation a consumer reads
//      is mapped into it once (CUDA IPC; handles exchanged by the all-reduce only when a rank's producer memory
//      changed) and the copy engines pull each remote run of tokens straight from the producer's streams into the
//      consumer's over NVLink; transport "nccl": one grouped NCCL send/recv (the baseline: NCCL point-to-point
//      tops out at ~285 GB/s per direction on this B200 box, profiles/r02_nccl_p2p.log). Either way local
//      segments are copied by one SM copy kernel on a forked stream, overlapping the remote transfers; one unpack
//      kernel rebases group_off / cu_seqlens / roll_group and fills ids and channels (reading the producers'
//      metadata in place over NVLink); the consumer's offsets come back to the host by one small D2H (get() waits
//      for it). Consumer groups that are one contiguous run of local producer memory are zero-copy views.
// Ordering: the sizes all-reduce completes only after every rank's stream has executed what preceded it (the
// production of the put batches); worker_done enqueues a device-side barrier (no host synchronization) before the
// iteration's consumer memory is recycled, so no producer or consumer buffer is reused while a peer reads it.
// Errors map to the reference's types (dfx_status).
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <thread>
#include <tuple>
#include <nccl.h>

#include <type_traits>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "common.cuh"

// NCCL is resolved at run time (dlopen by soname), not linked: inside a torch process the libnccl.so.2 torch
// already loaded serves it (one NCCL per process), elsewhere the system's; CPU-only hosts load libdfx without it.
namespace dfx {
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};
const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return a;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name)); return fn != nullptr; };
    a.ok = sym(a.GetUniqueId, "ncclGetUniqueId") && sym(a.CommInitRank, "ncclCommInitRank") &&
           sym(a.CommDestroy, "ncclCommDestroy") && sym(a.AllReduce, "ncclAllReduce") && sym(a.Send, "ncclSend") &&
           sym(a.Recv, "ncclRecv") && sym(a.GroupStart, "ncclGroupStart") && sym(a.GroupEnd, "ncclGroupEnd") &&
           sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  return api;
}
}  // namespace
}  // namespace dfx

#define DFX_NCCL(call)                                                                                           \
  do {                                                                                                           \
    if (!::dfx::nccl().ok) return ::dfx::fail(DFX_NCCL_ERROR, "libnccl.so.2 could not be loaded");               \
    ncclResult_t _r = ::dfx::nccl().call;                                                                        \
    if (_r != ncclSuccess)                                                                                       \
      return ::dfx::fail(DFX_NCCL_ERROR, std::string("nccl" #call ": ") + ::dfx::nccl().GetErrorString(_r));     \
  } while (0)

struct dfx_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0, n = 1, device = 0;
  int64_t* d_buf = nullptr;  // small all-reduces
  int64_t* h_buf = nullptr;  // pinned
  int64_t cap = 0;
  // host side channel between the box's processes: a POSIX shared-memory segment of per-rank slots
  uint8_t* shm = nullptr;
  size_t shm_bytes = 0;
  int64_t slot_cap = 0;      // int64 values per slot
  uint64_t gen = 0;          // calls so far (every rank makes the same calls in the same order)
  // device barrier over NVLink
  uint64_t* flags = nullptr;                  // own flag array [n]
  std::vector<uint64_t*> peer_flags;          // every rank's flag array, mapped here
  uint64_t barrier_gen = 0;
  int* err = nullptr;                         // device error word (a barrier that lost a peer)
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

// ---- host all-gather through shared memory ----------------------------------------------------------------------
// Slot (parity, rank) = {seq u64, n i64, pad to 64 B, data i64[slot_cap]}. Call g writes parity g & 1, then waits
// until every rank's seq of that parity reaches g. A rank can only write parity g & 1 again (call g + 2) after
// completing call g + 1, which needs every rank to have written g + 1 -- i.e. to be done reading g: two buffers
// suffice, no read acknowledgements. Cost: a memcpy and a spin on the box's coherent memory (~microseconds,
// against ~45 us for a device all-reduce and its host synchronization).
constexpr size_t kShmHeader = 4096;
size_t shm_slot_bytes(int64_t cap) { return 64 + size_t(cap) * 8; }
uint8_t* shm_slot(dfx_comm* c, int parity, int r) {
  return c->shm + kShmHeader + (size_t(parity) * c->n + r) * shm_slot_bytes(c->slot_cap);
}

dfx_status host_allgatherv(dfx_comm* c, const int64_t* data, int64_t n, std::vector<const int64_t*>& rows,
                           std::vector<int64_t>& lens) {
  rows.assign(c->n, nullptr);
  lens.assign(c->n, 0);
  if (c->n == 1) {
    rows[0] = data;
    lens[0] = n;
    return DFX_OK;
  }
  if (n > c->slot_cap)
    return fail(DFX_INVALID_ARGUMENT, "host metadata of " + std::to_string(n) + " values exceeds the shared-memory "
                                      "slot (" + std::to_string(c->slot_cap) + "); raise DFX_SHM_SLOT_MB");
  const uint64_t g = ++c->gen;
  const int par = int(g & 1);
  uint8_t* mine = shm_slot(c, par, c->rank);
  std::memcpy(mine + 64, data, size_t(n) * 8);
  *reinterpret_cast<int64_t*>(mine + 8) = n;
  reinterpret_cast<std::atomic<uint64_t>*>(mine)->store(g, std::memory_order_release);
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < c->n; ++r) {
    uint8_t* sl = shm_slot(c, par, r);
    auto* seq = reinterpret_cast<std::atomic<uint64_t>*>(sl);
    for (uint32_t spin = 0; seq->load(std::memory_order_acquire) < g; ++spin) {
      if ((spin & 1023) == 1023) {
        std::this_thread::yield();
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          return fail(DFX_NOT_READY, "host all-gather: rank " + std::to_string(r) + " did not arrive within 120 s");
      }
    }
    rows[r] = reinterpret_cast<const int64_t*>(sl + 64);
    lens[r] = *reinterpret_cast<const int64_t*>(sl + 8);
  }
  return DFX_OK;
}

// ---- device-side barrier over NVLink -----------------------------------------------------------------------------
// Every rank owns flags[n] (device memory, mapped by every peer through CUDA IPC at communicator setup). Barrier g:
// thread r stores g into flag slot [me] of peer r (system-scope release, after a system fence that publishes the
// stream's earlier writes), then waits until its own slot [r] reaches g (acquire). When it returns on one rank,
// every rank's stream has executed everything enqueued before its own barrier -- the property of a 1-element
// all-reduce (the NCCL fallback, DFX_BARRIER=nccl) at a few microseconds instead of ~14. A bounded spin (~20 s)
// reports a lost peer in the error word instead of hanging the GPU.
constexpr int kMaxRanks = 64;
struct BarrierArgs {
  uint64_t* peer_flags[kMaxRanks];  // peer r's flag array (mapped); peer_flags[me] = own
  uint64_t* mine;
  int n, me;
  uint64_t gen;
  int* err;
};
__global__ void nvlink_barrier_kernel(const BarrierArgs a) {
  const int r = threadIdx.x;
  if (r < a.n) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.peer_flags[r] + a.me), "l"(a.gen) : "memory");
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      uint64_t v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a.mine + r) : "memory");
      if (v >= a.gen) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) {
        atomicExch(a.err, 1);
        break;
      }
    }
  }
  __syncthreads();
}

dfx_status comm_barrier(dfx_comm* c, cudaStream_t st) {
  static const bool use_nccl = [] {
    const char* e = std::getenv("DFX_BARRIER");
    return e && std::string(e) == "nccl";
  }();
  if (use_nccl || !c->flags) {
    DFX_NCCL(AllReduce(c->d_buf + c->cap - 1, c->d_buf + c->cap - 1, 1, ncclInt64, ncclSum, c->nccl, st));
    return DFX_OK;
  }
  BarrierArgs a{};
  for (int r = 0; r < c->n; ++r) a.peer_flags[r] = c->peer_flags[r];
  a.mine = c->flags;
  a.n = c->n;
  a.me = c->rank;
  a.gen = ++c->barrier_gen;
  a.err = c->err;
  nvlink_barrier_kernel<<<1, 64, 0, st>>>(a);
  DFX_LAUNCH_CHECK("nvlink_barrier_kernel");
  return DFX_OK;
}

// ---- unpack into per-group relative metadata -------------------------------------------------------------------
// One entry per segment: source metadata (a local producer's arrays, a producer's arrays mapped from its GPU, or a
// received metadata buffer) and the destination arrays of its consumer group, already offset to the segment.
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

// CTA (segment x, 256-entry chunk y): the source metadata often sits in a peer GPU's memory, so the loads of a
// segment are spread over many CTAs (each loop trip in one CTA would pay an NVLink round trip)
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

// ---- the pull: SM copy of peer-mapped producer memory over NVLink ----------------------------------------------
// Persistent CTAs walk 128 KB chunks of the run list; each thread keeps 4 x 16 B non-coherent loads in flight
// before storing (an NVLink round trip is ~1-2 us: bytes in flight, not instructions, bound the rate).
constexpr int kPullRuns = 64;
constexpr uint64_t kPullChunk = 1ull << 17;
struct PullList {
  int n;
  uint64_t dst[kPullRuns], src[kPullRuns], bytes[kPullRuns], chunk0[kPullRuns + 1];
  uint32_t cta0[kPullRuns + 1];  // CTAs [cta0[r], cta0[r+1]) pull run r
};
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Every run (one producer range on one peer) gets its own share of the CTAs, proportional to its size, so all
// peers are read at once (at N = 4 a GPU pulls from three peers; taking the runs one after the other leaves the
// links to the other two idle and caps the pull at one pair's rate).
__global__ void __launch_bounds__(512) peer_pull_kernel(const PullList c) {
  int lo = 0, hi = c.n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (c.cta0[mid] <= blockIdx.x) lo = mid;
    else hi = mid;
  }
  const uint32_t nc = c.cta0[lo + 1] - c.cta0[lo];
  const uint64_t nch = c.chunk0[lo + 1] - c.chunk0[lo];
  for (uint64_t ch = blockIdx.x - c.cta0[lo]; ch < nch; ch += nc) {
    const uint64_t off = ch * kPullChunk;
    const uint64_t n = min(kPullChunk, c.bytes[lo] - off);
    uint8_t* dst = reinterpret_cast<uint8_t*>(c.dst[lo]) + off;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(c.src[lo]) + off;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0) {
      const uint64_t nv = n / 16, step = blockDim.x;
      uint64_t i = threadIdx.x;
      for (; i + 3 * step < nv; i += 4 * step) {
        const uint4 a = ld_nc_v4(src + 16 * i), b = ld_nc_v4(src + 16 * (i + step));
        const uint4 c2 = ld_nc_v4(src + 16 * (i + 2 * step)), d = ld_nc_v4(src + 16 * (i + 3 * step));
        reinterpret_cast<uint4*>(dst)[i] = a;
        reinterpret_cast<uint4*>(dst)[i + step] = b;
        reinterpret_cast<uint4*>(dst)[i + 2 * step] = c2;
        reinterpret_cast<uint4*>(dst)[i + 3 * step] = d;
      }
      for (; i < nv; i += step) reinterpret_cast<uint4*>(dst)[i] = ld_nc_v4(src + 16 * i);
      for (uint64_t j = nv * 16 + threadIdx.x; j < n; j += step) dst[j] = src[j];
    } else {
      // source and destination in different 16-byte phases (runs start at arbitrary token offsets)
      copy_shift16<true>(dst, src, n, threadIdx.x, blockDim.x);
    }
  }
}

dfx_status peer_pull(const std::vector<uint64_t>& dst, const std::vector<uint64_t>& src,
                     const std::vector<uint64_t>& bytes, int n_peers, cudaStream_t st) {
  // 512-thread CTAs per SM: 2 when reading one peer, 1 when reading several at once -- measured (C4, bench.py):
  // N = 2 0.614 (2) vs 0.60 (1) of 770 GB/s, N = 4 0.64 (1) vs 0.57 (2) vs 0.556 (3); both leave room on every SM
  // for the unpack and local copies running concurrently on the side stream
  static const int env_cps = [] {
    const char* e = std::getenv("DFX_PULL_CTAS_PER_SM");  // benchmarking knob
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int ctas_per_sm = env_cps ? env_cps : (n_peers > 1 ? 1 : 2);
  for (size_t i0 = 0; i0 < bytes.size(); i0 += kPullRuns) {
    PullList c{};
    uint64_t chunks = 0;
    for (size_t i = i0; i < std::min(bytes.size(), i0 + kPullRuns); ++i) {
      if (!bytes[i]) continue;
      c.dst[c.n] = dst[i];
      c.src[c.n] = src[i];
      c.bytes[c.n] = bytes[i];
      c.chunk0[c.n] = chunks;
      chunks += (bytes[i] + kPullChunk - 1) / kPullChunk;
      ++c.n;
    }
    if (!c.n) continue;
    c.chunk0[c.n] = chunks;
    const uint64_t target = std::min<uint64_t>(chunks, uint64_t(148) * ctas_per_sm);
    uint32_t ctas = 0;
    for (int r = 0; r < c.n; ++r) {  // CTAs in proportion to the run's chunks (at least one, at most its chunks)
      const uint64_t cr = c.chunk0[r + 1] - c.chunk0[r];
      c.cta0[r] = ctas;
      ctas += uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(cr, (cr * target + chunks / 2) / chunks)));
    }
    c.cta0[c.n] = ctas;
    peer_pull_kernel<<<ctas, 512, 0, st>>>(c);
    DFX_LAUNCH_CHECK("peer_pull_kernel");
  }
  return DFX_OK;
}

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
  std::vector<int32_t> hgo;   // views: rebased on the host at once
  std::vector<int64_t> hcu;
};

struct Block {
  void* p;
  size_t bytes;
};

struct Ready {
  std::map<uint32_t, Group> groups;
  std::vector<Block> blocks;    // device blocks of the consumer batches (back to the store's cache at retire)
  std::vector<void*> scratch;   // stream-ordered pool allocations (NCCL staging)
  void* pinned = nullptr;       // pinned host block: consumer offsets (D2H) and view metadata (H2D staging)
  cudaEvent_t meta_ev = nullptr;  // the pinned block's H2D copies are done at this point of the stream
};

struct Entry {
  std::map<uint32_t, Held> by_group;
  bool ready = false;
  Ready r;
};

struct PSeg {
  uint32_t dst, src;
  uint64_t dst_rec, src_rec, count;
  int64_t n_roll = 0, n_tok = 0, t0 = 0, s0 = 0;  // sizes; first token and first rollout in the producer's arrays
};
constexpr int kHandleCols = 9;  // 64-byte IPC handle as 8 int64 + the pointer's offset in its allocation

// what every rank knows of every producer group after the host all-gather: its host offsets (record -> rollout
// -> token, as int64) and, for the pull transport, its arrays' IPC handles + offsets
struct GInfo {
  bool present = false;
  int64_t n_rec = 0, n_roll = 0;
  const int64_t* go = nullptr;  // [n_rec + 1]
  const int64_t* cu = nullptr;  // [n_roll + 1]
  const int64_t* handles = nullptr;  // [n_arrays][kHandleCols]
};

struct PlanCache {
  bool valid = false;
  uint32_t to_dp = 0, to_tp = 0;
  std::vector<uint64_t> counts;
  std::vector<PSeg> segs;  // placement only; sizes are filled per exchange
};

// where a producer group's arrays live on this GPU: local pointers, or bases mapped from the owner (CUDA IPC)
struct SrcArrays {
  const uint64_t* ids = nullptr;
  const int32_t* go = nullptr;
  const int64_t* cu = nullptr;
  const double* ch[DFX_MAX_CH] = {};
  const uint8_t* st[DFX_MAX_STREAMS] = {};
};

struct Mapping {
  void* base;
  uint64_t last_use;
};

}  // namespace
}  // namespace dfx

struct dfx_dstore {
  dfx_comm* comm = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // local copies, overlapping the remote transfers
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<cudaStream_t> ce;          // copy-engine pull streams
  cudaEvent_t ev_ce_fork = nullptr;
  std::vector<cudaEvent_t> ev_ce_join;
  cudaMemPool_t pool = nullptr;
  int device = 0;
  int transport = DFX_TRANSPORT_PULL;
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
  uint64_t suppressed = 0, sent = 0, recvd = 0, copied = 0, plan_hits = 0, exchanges = 0;
  std::vector<void*> pinned_free;
  std::map<void*, size_t> pinned_size;
  std::multimap<size_t, void*> block_free;                   // exportable device blocks by size
  std::map<std::string, std::pair<std::vector<int64_t>, std::map<uint32_t, dfx::SrcArrays>>> remote;  // per stage
  std::map<std::string, dfx::Mapping> mappings;              // IPC handle bytes -> mapped base
  std::map<uintptr_t, std::pair<std::string, uint64_t>> exports;  // pointer -> (handle bytes, offset)
  std::vector<int64_t> row;                                   // this rank's host all-gather row
  bool trace = false;                                          // DFX_DSTORE_TRACE: device time per phase
  std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t>> spans;
};

namespace dfx {
namespace {

// DFX_DSTORE_TRACE=1 (diagnostics): events around each phase on the store's stream, summed at destroy
cudaEvent_t trace_mark(dfx_dstore* s) {
  if (!s->trace) return nullptr;
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  cudaEventRecord(ev, s->stream);
  return ev;
}
void trace_span(dfx_dstore* s, const char* name, cudaEvent_t a) {
  if (!s->trace || !a) return;
  s->spans.emplace_back(name, a, trace_mark(s));
}

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

// Consumer batches come from plain cudaMalloc blocks (IPC-exportable: a consumer batch is put as a producer in the
// next stage and mapped by its consumers), cached by size: a steady-state loop allocates nothing. A block returns
// to the cache at retire, after the release barrier is enqueued, so a later stream-ordered reuse cannot race with
// a peer still reading it.
dfx_status block_get(dfx_dstore* s, size_t bytes, Block* out) {
  const size_t b = bytes <= (1u << 20) ? ((bytes + 4095) & ~size_t(4095)) : ((bytes + (2u << 20) - 1) & ~size_t((2u << 20) - 1));
  auto it = s->block_free.find(b);
  if (it != s->block_free.end()) {
    *out = Block{it->second, b};
    s->block_free.erase(it);
    return DFX_OK;
  }
  void* p = nullptr;
  DFX_CUDA(cudaMalloc(&p, b));
  *out = Block{p, b};
  return DFX_OK;
}

dfx_status scratch_alloc(dfx_dstore* s, size_t bytes, void** p) {
  DFX_CUDA(cudaMallocFromPoolAsync(p, std::max<size_t>(bytes, 256), s->pool, s->stream));
  return DFX_OK;
}

void retire(dfx_dstore* s, Ready& r) {
  for (const Block& b : r.blocks) s->block_free.emplace(b.bytes, b.p);
  r.blocks.clear();
  for (void* p : r.scratch) cudaFreeAsync(p, s->stream);
  r.scratch.clear();
  if (r.meta_ev) {
    cudaEventSynchronize(r.meta_ev);  // the pinned block may still be a copy target
    cudaEventDestroy(r.meta_ev);
    r.meta_ev = nullptr;
  }
  if (r.pinned) s->pinned_free.push_back(r.pinned);
  r.pinned = nullptr;
}

// ranks that host a TP worker of consumer group d (lead = d * tp, topology.hpp:50)
std::vector<int> dst_ranks(const dfx_dstore* s, uint32_t d, uint32_t tp) {
  std::set<int> r;
  for (uint32_t t = 0; t < tp; ++t) r.insert(s->rank_of_worker[size_t(d) * tp + t]);
  return std::vector<int>(r.begin(), r.end());
}

// sizes of segment sg from its producer group's host offsets
void seg_sizes(const GInfo& g, PSeg& sg) {
  const int64_t r0 = int64_t(sg.src_rec), r1 = r0 + int64_t(sg.count);
  const int64_t s0 = g.go[r0], s1 = g.go[r1];
  sg.n_roll = s1 - s0;
  sg.s0 = s0;
  sg.t0 = g.cu[s0];
  sg.n_tok = g.cu[s1] - sg.t0;
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

// the arrays of a put batch in table order: ids, group_off, cu, channels, streams
int n_arrays(const dfx_dstore* s) { return 3 + s->n_ch + s->n_streams; }
const void* array_ptr(const dfx_dstore* s, const dfx_batch& b, int a) {
  if (a == 0) return b.ids;
  if (a == 1) return b.group_off;
  if (a == 2) return b.cu_seqlens;
  if (a < 3 + s->n_ch) return b.ch[a - 3];
  return b.st[a - 3 - s->n_ch];
}

// IPC export of the allocation holding ptr (cached per pointer; a producer allocation must not be freed and
// re-allocated at the same address while the store is in use)
dfx_status export_ptr(dfx_dstore* s, const void* ptr, std::string& handle, uint64_t& offset) {
  auto it = s->exports.find(reinterpret_cast<uintptr_t>(ptr));
  if (it != s->exports.end()) {
    handle = it->second.first;
    offset = it->second.second;
    return DFX_OK;
  }
  char h[64];
  dfx_status st = dfx_ipc_export(ptr, h, &offset);
  if (st) return st;
  handle.assign(h, 64);
  s->exports[reinterpret_cast<uintptr_t>(ptr)] = {handle, offset};
  return DFX_OK;
}

uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  return h * 0xBF58476D1CE4E5B9ull;
}

// element range moved for a segment's stream k by NCCL: exact when both ends are 16-byte aligned, else the
// 8-element aligned superset into a staging buffer (NCCL point-to-point runs far slower on misaligned buffers)
bool seg_direct(int64_t t0, int64_t dt, uint32_t esz) {
  return ((t0 * int64_t(esz)) & 15) == 0 && ((dt * int64_t(esz)) & 15) == 0;
}

// ---- the exchange ----------------------------------------------------------------------------------------------
// Consumer groups on this rank, in dp order, fall in three kinds:
//   view    all segments local, one contiguous run of the producers' memory (several producer groups that are
//           adjacent views of one batch qualify): no data moves, only the group's relative record metadata
//   local   all segments local but not contiguous: copied on this GPU (its own allocation)
//   remote  at least one segment from another GPU: the shared layout (token offsets every rank can compute,
//           which the NCCL transport's senders need for their alignment decisions)
dfx_status run_exchange(dfx_dstore* s, const StageCfg& c, uint32_t to_dp, uint32_t to_tp, Entry& e,
                        const std::vector<PSeg>& segs, const std::vector<GInfo>& info,
                        const std::map<uint32_t, SrcArrays>& remote_src) {
  const int me = s->comm->rank;
  cudaStream_t st = s->stream;
  Ready& r = e.r;
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
  auto all_local_on = [&](uint32_t d, int rk) {
    for (size_t i : seg_of[d])
      if (src_rank[segs[i].src] != rk) return false;
    return true;
  };
  const int NA = n_arrays(s);
  // local producer arrays (tables of pointers, like the mapped ones)
  std::map<uint32_t, SrcArrays> loc;
  for (auto& kv : e.by_group) {
    SrcArrays a;
    a.ids = kv.second.b.ids;
    a.go = kv.second.b.group_off;
    a.cu = kv.second.b.cu_seqlens;
    for (int c2 = 0; c2 < s->n_ch; ++c2) a.ch[c2] = kv.second.b.ch[c2];
    for (int k = 0; k < s->n_streams; ++k) a.st[k] = static_cast<const uint8_t*>(kv.second.b.st[k]);
    loc[kv.first] = a;
  }
  auto src_of = [&](uint32_t p) -> const SrcArrays& { return src_rank[p] == me ? loc.at(p) : remote_src.at(p); };
  (void)NA;

  enum Kind { VIEW, LOCAL, REMOTE };
  struct GL {
    Kind kind = REMOTE;
    int64_t R = 0, S = 0, T = 0;
    size_t o_ids = 0, o_go = 0, o_rg = 0, o_cu = 0, o_ch = 0;
    int64_t tok = 0;
    int area = 0;  // 0: shared (remote groups), 1: local copies
  };
  std::map<uint32_t, GL> gl;
  int64_t R[2] = {0, 0}, S[2] = {0, 0}, T[2] = {0, 0}, NG[2] = {0, 0};
  for (uint32_t d : local_dst) {
    GL g;
    const auto& ix = seg_of[d];
    for (size_t i : ix) {
      g.R += int64_t(segs[i].count);
      g.S += segs[i].n_roll;
      g.T += segs[i].n_tok;
    }
    if (all_local_on(d, me)) {
      g.kind = VIEW;  // unless the runs are not contiguous in memory
      for (size_t q = 0; q + 1 < ix.size() && g.kind == VIEW; ++q) {
        const PSeg &a = segs[ix[q]], &b = segs[ix[q + 1]];
        const SrcArrays &A = loc.at(a.src), &Bv = loc.at(b.src);
        const int64_t a_r1 = int64_t(a.src_rec + a.count), a_s1 = a.s0 + a.n_roll;
        bool ok = A.ids + a_r1 == Bv.ids + b.src_rec && A.cu + a_s1 == Bv.cu + b.s0 && a.t0 + a.n_tok == b.t0;
        for (int c2 = 0; c2 < s->n_ch; ++c2) ok = ok && A.ch[c2] + a_s1 == Bv.ch[c2] + b.s0;
        for (int k = 0; k < s->n_streams; ++k) ok = ok && A.st[k] == Bv.st[k];
        if (!ok) g.kind = LOCAL;
      }
    }
    if (g.kind != VIEW) {
      const int ar = g.kind == LOCAL ? 1 : 0;
      g.area = ar;
      g.o_ids = size_t(R[ar]);
      g.o_go = size_t(R[ar] + NG[ar]);
      g.o_rg = size_t(S[ar]);
      g.o_cu = size_t(S[ar] + NG[ar]);
      g.o_ch = size_t(S[ar]);
      g.tok = T[ar];
      R[ar] += g.R;
      S[ar] += g.S;
      T[ar] += g.T;
      ++NG[ar];
    }
    gl[d] = g;
  }
  // per area one block: ids | go | rg | cu | ch | streams (each 256-byte aligned, streams padded for over-reads)
  uint8_t* mem[2] = {nullptr, nullptr};
  size_t b_ids[2], b_go[2], b_rg[2], b_cu[2];
  std::vector<size_t> b_ch[2], b_st[2];
  for (int ar = 0; ar < 2; ++ar) {
    size_t off = 0;
    b_ids[ar] = off; off += al256(size_t(R[ar]) * 8);
    b_go[ar] = off; off += al256(size_t(R[ar] + NG[ar]) * 4);
    b_rg[ar] = off; off += al256(size_t(S[ar]) * 4);
    b_cu[ar] = off; off += al256(size_t(S[ar] + NG[ar]) * 8);
    b_ch[ar].resize(s->n_ch);
    b_st[ar].resize(s->n_streams);
    for (int c2 = 0; c2 < s->n_ch; ++c2) { b_ch[ar][c2] = off; off += al256(size_t(S[ar]) * 8); }
    for (int k = 0; k < s->n_streams; ++k) { b_st[ar][k] = off; off += al256(size_t(T[ar] + 64) * s->esz[k]); }
    if (NG[ar] > 0) {
      Block blk;
      dfx_status stt = block_get(s, off, &blk);
      if (stt) return stt;
      r.blocks.push_back(blk);
      mem[ar] = static_cast<uint8_t*>(blk.p);
    }
  }
  // pinned host block: the views' relative record metadata (H2D)
  size_t pin_bytes = 0;
  for (uint32_t d : local_dst)
    if (gl[d].kind == VIEW) pin_bytes += al256(size_t(gl[d].R + 1) * 4) + al256(size_t(gl[d].S) * 4);
  uint8_t* hp = nullptr;
  if (pin_bytes) {
    r.pinned = pinned_get(s, pin_bytes);
    if (!r.pinned) return fail(DFX_CUDA_ERROR, "cudaMallocHost failed");
    hp = static_cast<uint8_t*>(r.pinned);
  }
  // view metadata device block (one per exchange)
  size_t view_meta = 0;
  for (uint32_t d : local_dst)
    if (gl[d].kind == VIEW) view_meta += al256(size_t(gl[d].R + 1) * 4) + al256(size_t(gl[d].S) * 4);
  uint8_t* vmem = nullptr;
  uint8_t* vmem0 = nullptr;
  uint8_t* hp0 = hp;
  if (view_meta) {
    Block blk;
    dfx_status stt = block_get(s, view_meta, &blk);
    if (stt) return stt;
    r.blocks.push_back(blk);
    vmem = static_cast<uint8_t*>(blk.p);
    vmem0 = vmem;
  }

  // ---- group descriptors; host offsets of every group from the producers' (no device read-back) ----
  for (uint32_t d : local_dst) {
    GL& g = gl[d];
    Group grp;
    const auto& ix = seg_of[d];
    const int64_t tok0 = g.kind == VIEW ? segs[ix.front()].t0 : g.tok;
    // per segment: group_off rebased by (records, rollouts) so far, cu shifted by the segment's token offset --
    // straight-line loops over the producers' host offsets (vectorizable)
    grp.hgo.resize(size_t(g.R + 1));
    grp.hcu.resize(size_t(g.S + 1));
    std::vector<int32_t> hrg(size_t(g.S));
    grp.hgo[0] = 0;
    grp.hcu[0] = tok0;
    int64_t rr = 0, ss = 0, tt = tok0;
    for (size_t i : ix) {
      const PSeg& sg = segs[i];
      const GInfo& gi = info[sg.src];
      const int64_t* go = gi.go + sg.src_rec;
      const int64_t* cu = gi.cu + sg.s0;
      const int64_t nr = int64_t(sg.count), ns = sg.n_roll, dgo = ss - go[0], dcu = tt - cu[0];
      int32_t* hgo = grp.hgo.data() + rr + 1;
      for (int64_t q = 0; q < nr; ++q) hgo[q] = int32_t(go[q + 1] + dgo);
      int64_t* hcu = grp.hcu.data() + ss + 1;
      for (int64_t j = 0; j < ns; ++j) hcu[j] = cu[j + 1] + dcu;
      for (int64_t q = 0; q < nr; ++q) {
        const int64_t a = go[q] + dgo, b = go[q + 1] + dgo;
        for (int64_t j = a; j < b; ++j) hrg[size_t(j)] = int32_t(rr + q);
      }
      rr += nr;
      ss += ns;
      tt += sg.n_tok;
    }
    if (g.kind == VIEW) {
      const PSeg& f = segs[ix.front()];
      const Held& h0 = e.by_group.at(f.src);
      dfx_batch v = h0.b;
      v.n_records = g.R;
      v.n_rollouts = g.S;
      v.ids = h0.b.ids + f.src_rec;
      v.cu_seqlens = h0.b.cu_seqlens + f.s0;
      for (int c2 = 0; c2 < s->n_ch; ++c2) v.ch[c2] = h0.b.ch[c2] + f.s0;
      v.token_base = f.t0;
      v.token_span = g.T;
      int32_t* hgo = reinterpret_cast<int32_t*>(hp);
      hp += al256(size_t(g.R + 1) * 4);
      int32_t* hrgp = reinterpret_cast<int32_t*>(hp);
      hp += al256(size_t(g.S) * 4);
      std::memcpy(hgo, grp.hgo.data(), grp.hgo.size() * 4);
      std::memcpy(hrgp, hrg.data(), hrg.size() * 4);
      int32_t* dgo = reinterpret_cast<int32_t*>(vmem);
      vmem += al256(size_t(g.R + 1) * 4);
      int32_t* drg = reinterpret_cast<int32_t*>(vmem);
      vmem += al256(size_t(g.S) * 4);
      (void)hrgp;  // (the views' metadata goes to the device in ONE copy below: pinned and device regions match)
      v.group_off = dgo;
      v.roll_group = drg;
      grp.b = v;
    } else {
      const int ar = g.area;
      uint8_t* m = mem[ar];
      dfx_batch v{};
      v.n_records = g.R;
      v.n_rollouts = g.S;
      v.token_base = g.tok;
      v.token_span = g.T;
      v.ids = reinterpret_cast<uint64_t*>(m + b_ids[ar]) + g.o_ids;
      v.group_off = reinterpret_cast<int32_t*>(m + b_go[ar]) + g.o_go;
      v.roll_group = reinterpret_cast<int32_t*>(m + b_rg[ar]) + g.o_rg;
      v.cu_seqlens = reinterpret_cast<int64_t*>(m + b_cu[ar]) + g.o_cu;
      for (int c2 = 0; c2 < s->n_ch; ++c2) v.ch[c2] = reinterpret_cast<double*>(m + b_ch[ar][c2]) + g.o_ch;
      for (int k = 0; k < s->n_streams; ++k) v.st[k] = m + b_st[ar][k];
      grp.b = v;
    }
    r.groups[d] = std::move(grp);
  }
  for (auto& kv : r.groups) {
    kv.second.b.h_group_off = kv.second.hgo.data();
    kv.second.b.h_cu = kv.second.hcu.data();
  }
  // (the views' metadata goes to the device in one copy on the side stream, off the pull's critical path)

  // destination offsets of every segment of a copied group
  std::vector<int64_t> seg_dt(segs.size(), -1), seg_dr(segs.size(), 0), seg_ds(segs.size(), 0);
  for (uint32_t d : local_dst) {
    const GL& g = gl[d];
    if (g.kind == VIEW) continue;
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
  auto dst_stream = [&](size_t i, int k) {
    const GL& g = gl[segs[i].dst];
    return mem[g.area] + b_st[g.area][k] + size_t(seg_dt[i]) * s->esz[k];
  };

  // ---- metadata of every segment of the copied groups (one unpack): local arrays, the producers' mapped over
  // NVLink (pull), or the received metadata buffers (NCCL) ----
  std::map<size_t, const uint8_t*> recv_meta;  // segment -> received metadata buffer (NCCL transport)
  auto make_xs = [&]() {
  std::vector<XSeg> xs;
  for (uint32_t d : local_dst) {
    if (gl[d].kind == VIEW) continue;
    const Group& grp = r.groups[d];
    for (size_t i : seg_of[d]) {
      const PSeg& sg = segs[i];
      XSeg x{};
      auto rm = recv_meta.find(i);
      if (rm == recv_meta.end()) {  // local arrays, or the producer's mapped over NVLink (pull)
        const SrcArrays& a = src_of(sg.src);
        x.ids = a.ids + sg.src_rec;
        x.go = a.go + sg.src_rec;
        x.cu = a.cu + sg.s0;
        for (int c2 = 0; c2 < s->n_ch; ++c2) x.ch[c2] = a.ch[c2] + sg.s0;
      } else {  // received: ids u64[n_rec] | cu i64[n_roll+1] | ch f64[n_ch][n_roll] | go i32[n_rec+1]
        const uint8_t* b = rm->second;
        const int64_t nr = int64_t(sg.count), ns = sg.n_roll;
        x.ids = reinterpret_cast<const uint64_t*>(b);
        x.cu = reinterpret_cast<const int64_t*>(b + 8 * nr);
        for (int c2 = 0; c2 < s->n_ch; ++c2)
          x.ch[c2] = reinterpret_cast<const double*>(b + 8 * nr + 8 * (ns + 1) + 8 * c2 * ns);
        x.go = reinterpret_cast<const int32_t*>(b + 8 * nr + 8 * (ns + 1) + 8 * int64_t(s->n_ch) * ns);
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
  return xs;
  };
  // ---- token streams: local copies (side stream) overlapping the remote transfers (main stream) ----
  std::vector<uint64_t> cp_dst, cp_src, cp_n;     // local segments (SM copy kernel)
  std::vector<uint64_t> rp_dst, rp_src, rp_n;     // remote segments, pull transport
  std::set<int> pull_peers;                        // the ranks they come from
  auto push_merged = [](std::vector<uint64_t>& D, std::vector<uint64_t>& S_, std::vector<uint64_t>& N, uint64_t d,
                        uint64_t src, uint64_t n) {
    if (!N.empty() && D.back() + N.back() == d && S_.back() + N.back() == src) {
      N.back() += n;
      return;
    }
    D.push_back(d);
    S_.push_back(src);
    N.push_back(n);
  };
  for (uint32_t d : local_dst) {
    if (gl[d].kind == VIEW) continue;
    for (size_t i : seg_of[d]) {
      const PSeg& sg = segs[i];
      if (sg.n_tok == 0) continue;
      const bool here = src_rank[sg.src] == me;
      if (!here && s->transport != DFX_TRANSPORT_PULL) continue;
      if (!here) pull_peers.insert(src_rank[sg.src]);
      const SrcArrays& a = src_of(sg.src);
      for (int k = 0; k < s->n_streams; ++k) {
        const uint64_t n = uint64_t(sg.n_tok) * s->esz[k];
        const uint64_t dd = uint64_t(reinterpret_cast<uintptr_t>(dst_stream(i, k)));
        const uint64_t ss = uint64_t(reinterpret_cast<uintptr_t>(a.st[k] + size_t(sg.t0) * s->esz[k]));
        if (here) {
          push_merged(cp_dst, cp_src, cp_n, dd, ss, n);
          s->copied += n;
        } else {
          push_merged(rp_dst, rp_src, rp_n, dd, ss, n);
          s->recvd += n;
        }
      }
    }
  }
  // the side stream: local copies, and (pull) the unpack, which reads the producers' metadata in place and does
  // not depend on the token transfers -- its NVLink round trips hide under the bulk pull
  std::vector<XSeg> xs_pull;
  if (s->transport == DFX_TRANSPORT_PULL) xs_pull = make_xs();
  const bool fork = !cp_n.empty() || !xs_pull.empty() || view_meta;
  if (fork) {
    DFX_CUDA(cudaEventRecord(s->ev_fork, st));
    DFX_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
    if (view_meta) DFX_CUDA(cudaMemcpyAsync(vmem0, hp0, view_meta, cudaMemcpyHostToDevice, s->side));
    if (!cp_n.empty()) {
      dfx_status stt = dfx_copy_many(int64_t(cp_n.size()), cp_dst.data(), cp_src.data(), cp_n.data(), s->side);
      if (stt) return stt;
    }
    if (!xs_pull.empty()) {
      dfx_status stt = xunpack(xs_pull, s->n_ch, s->side);
      if (stt) return stt;
    }
    DFX_CUDA(cudaEventRecord(s->ev_join, s->side));
  }
  // pull: the SMs (peer_pull_kernel; or the copy engines) read the producers' memory over NVLink (peer-mapped),
  // straight into the consumer streams -- one run per merged range (adjacent segments of one batch merge)
  static const bool pull_sm = [] {
    const char* v = std::getenv("DFX_DSTORE_PULL");  // benchmarking knob: "ce" = copy-engine transfers
    return !(v && std::string(v) == "ce");
  }();
  cudaEvent_t t_pull = trace_mark(s);
  if (!rp_n.empty()) {
    if (pull_sm) {
      dfx_status stt = peer_pull(rp_dst, rp_src, rp_n, int(pull_peers.size()), st);
      if (stt) return stt;
    } else {
      // the runs spread over several streams, so several copy engines pull concurrently (one queue would run
      // them back to back, each paying its ramp)
      const int ns = std::min<int>(int(s->ce.size()), int(rp_n.size()));
      DFX_CUDA(cudaEventRecord(s->ev_ce_fork, st));
      for (int q = 0; q < ns; ++q) DFX_CUDA(cudaStreamWaitEvent(s->ce[q], s->ev_ce_fork, 0));
      for (size_t q = 0; q < rp_n.size(); ++q)
        DFX_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(rp_dst[q]), reinterpret_cast<const void*>(rp_src[q]),
                                 rp_n[q], cudaMemcpyDefault, ns > 0 ? s->ce[q % size_t(ns)] : st));
      for (int q = 0; q < ns; ++q) {
        DFX_CUDA(cudaEventRecord(s->ev_ce_join[q], s->ce[q]));
        DFX_CUDA(cudaStreamWaitEvent(st, s->ev_ce_join[q], 0));
      }
    }
  }
  trace_span(s, "pull (remote token runs)", t_pull);

  // ---- NCCL transport: grouped send/recv of remote segments (+ packed metadata) ----
  if (s->transport == DFX_TRANSPORT_NCCL) {
    struct Xfer {
      size_t seg;
      int peer;
    };
    std::vector<Xfer> sends, recvs;
    for (size_t i = 0; i < segs.size(); ++i) {
      const int src = src_rank[segs[i].src];
      for (int rk : dranks[segs[i].dst]) {
        const bool rk_view = all_local_on(segs[i].dst, rk);  // groups that never receive (views / local copies)
        if (rk_view) continue;
        if (src == me && rk != me) sends.push_back({i, rk});
        if (rk == me && src != me) recvs.push_back({i, src});
      }
    }
    // destination token position of segment i on rank rk (its shared area: groups with a remote segment)
    auto remote_dt = [&](size_t i, int rk) -> int64_t {
      int64_t t = 0;
      for (uint32_t d = 0; d < to_dp; ++d) {
        if (std::find(dranks[d].begin(), dranks[d].end(), rk) == dranks[d].end() || all_local_on(d, rk)) continue;
        for (size_t j : seg_of[d]) {
          if (j == i) return t;
          t += segs[j].n_tok;
        }
      }
      return 0;
    };
    const int64_t n_ch = s->n_ch;
    auto meta_bytes = [&](const PSeg& sg) {
      return size_t(dfx_reshard_pack_bytes(int64_t(sg.count), sg.n_roll, int32_t(n_ch)));
    };
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
      dfx_status stt = scratch_alloc(s, scratch, &p);
      if (stt) return stt;
      scr = static_cast<uint8_t*>(p);
      r.scratch.push_back(p);
    }
    if (!sends.empty()) {  // metadata of every sent segment, one pack launch
      std::vector<dfx_seg_meta> pm(sends.size());
      std::vector<uint8_t*> outp(sends.size());
      for (size_t q = 0; q < sends.size(); ++q) {
        const PSeg& sg = segs[sends[q].seg];
        const SrcArrays& a = loc.at(sg.src);
        dfx_seg_meta m{};
        m.ids = a.ids + sg.src_rec;
        m.group_off = a.go + sg.src_rec;
        m.cu = a.cu + sg.s0;
        for (int c2 = 0; c2 < s->n_ch; ++c2) m.ch[c2] = a.ch[c2] + sg.s0;
        m.n_rec = int64_t(sg.count);
        m.n_roll = sg.n_roll;
        pm[q] = m;
        outp[q] = scr + o_send[q];
      }
      dfx_status stt = dfx_reshard_pack(pm.data(), int32_t(pm.size()), s->n_ch, outp.data(), st);
      if (stt) return stt;
    }
    if (!sends.empty() || !recvs.empty()) {
      DFX_NCCL(GroupStart());
      // per peer, both sides post in global segment order: metadata, then the streams in schema order
      for (size_t q = 0; q < sends.size(); ++q) {
        const PSeg& sg = segs[sends[q].seg];
        const int to = sends[q].peer;
        DFX_NCCL(Send(scr + o_send[q], meta_bytes(sg), ncclUint8, to, s->comm->nccl, st));
        s->sent += meta_bytes(sg);
        if (sg.n_tok == 0) continue;
        const SrcArrays& a = loc.at(sg.src);
        const int64_t dt = remote_dt(sends[q].seg, to);
        for (int k = 0; k < s->n_streams; ++k) {
          const size_t es = s->esz[k];
          if (seg_direct(sg.t0, dt, s->esz[k])) {
            DFX_NCCL(Send(a.st[k] + size_t(sg.t0) * es, size_t(sg.n_tok) * es, ncclUint8, to, s->comm->nccl, st));
            s->sent += size_t(sg.n_tok) * es;
          } else {
            const int64_t a0 = sg.t0 & ~int64_t(7), a1 = (sg.t0 + sg.n_tok + 7) & ~int64_t(7);
            DFX_NCCL(Send(a.st[k] + size_t(a0) * es, size_t(a1 - a0) * es, ncclUint8, to, s->comm->nccl, st));
            s->sent += size_t(a1 - a0) * es;
          }
        }
      }
      for (size_t q = 0; q < recvs.size(); ++q) {
        const PSeg& sg = segs[recvs[q].seg];
        const int from = recvs[q].peer;
        DFX_NCCL(Recv(scr + o_recv[q], meta_bytes(sg), ncclUint8, from, s->comm->nccl, st));
        s->recvd += meta_bytes(sg);
        recv_meta[recvs[q].seg] = scr + o_recv[q];
        if (sg.n_tok == 0) continue;
        for (int k = 0; k < s->n_streams; ++k) {
          const size_t es = s->esz[k];
          if (o_stage[q][k] == SIZE_MAX) {
            DFX_NCCL(Recv(dst_stream(recvs[q].seg, k), size_t(sg.n_tok) * es, ncclUint8, from, s->comm->nccl, st));
            s->recvd += size_t(sg.n_tok) * es;
          } else {
            const int64_t a0 = sg.t0 & ~int64_t(7), a1 = (sg.t0 + sg.n_tok + 7) & ~int64_t(7);
            DFX_NCCL(Recv(scr + o_stage[q][k], size_t(a1 - a0) * es, ncclUint8, from, s->comm->nccl, st));
            s->recvd += size_t(a1 - a0) * es;
          }
        }
      }
      DFX_NCCL(GroupEnd());
    }
    std::vector<uint64_t> pd, ps, pn;  // staged supersets -> exact destination ranges
    for (size_t q = 0; q < recvs.size(); ++q) {
      const PSeg& sg = segs[recvs[q].seg];
      for (int k = 0; k < s->n_streams; ++k) {
        if (sg.n_tok == 0 || o_stage[q][k] == SIZE_MAX) continue;
        const size_t es = s->esz[k];
        const int64_t head = sg.t0 - (sg.t0 & ~int64_t(7));
        pd.push_back(uint64_t(reinterpret_cast<uintptr_t>(dst_stream(recvs[q].seg, k))));
        ps.push_back(uint64_t(reinterpret_cast<uintptr_t>(scr + o_stage[q][k] + size_t(head) * es)));
        pn.push_back(uint64_t(sg.n_tok) * es);
      }
    }
    if (!pn.empty()) {
      dfx_status stt = dfx_copy_many(int64_t(pn.size()), pd.data(), ps.data(), pn.data(), st);
      if (stt) return stt;
    }
  }

  if (s->transport == DFX_TRANSPORT_NCCL) {  // the received metadata is there once the group has completed
    std::vector<XSeg> xs = make_xs();
    if (!xs.empty()) {
      dfx_status stt = xunpack(xs, s->n_ch, st);
      if (stt) return stt;
    }
  }
  if (fork) DFX_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
  if (pin_bytes) {  // the pinned block is an H2D source until this point of the stream
    DFX_CUDA(cudaEventCreateWithFlags(&r.meta_ev, cudaEventDisableTiming));
    DFX_CUDA(cudaEventRecord(r.meta_ev, st));
  }
  return DFX_OK;
}

// Pull transport: map every remote producer group this rank reads (its arrays' IPC handles came with the host
// all-gather) -- each allocation once, cached; mappings no exchange has used for a while are closed.
dfx_status map_remote(dfx_dstore* s, const std::vector<int>& src_rank, const std::vector<PSeg>& segs,
                      const std::vector<uint32_t>& local_dst, const std::vector<GInfo>& info,
                      std::map<uint32_t, SrcArrays>& out) {
  const int me = s->comm->rank, NA = n_arrays(s);
  std::set<uint32_t> need;
  for (const PSeg& sg : segs)
    if (src_rank[sg.src] != me && std::find(local_dst.begin(), local_dst.end(), sg.dst) != local_dst.end())
      need.insert(sg.src);
  for (uint32_t p : need) {
    const GInfo& gi = info[p];
    if (!gi.handles) return fail(DFX_ERROR, "producer group " + std::to_string(p) + " published no memory handles");
    SrcArrays sa;
    for (int a = 0; a < NA; ++a) {
      const int64_t* row = gi.handles + size_t(a) * kHandleCols;
      bool zero = true;
      for (int q = 0; q < 8; ++q) zero = zero && row[q] == 0;
      if (zero) continue;
      const std::string h(reinterpret_cast<const char*>(row), 64);
      auto m = s->mappings.find(h);
      if (m == s->mappings.end()) {
        void* base = nullptr;
        cudaIpcMemHandle_t ih;
        std::memcpy(&ih, h.data(), sizeof(ih));
        DFX_CUDA(cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess));
        m = s->mappings.emplace(h, Mapping{base, 0}).first;
      }
      m->second.last_use = s->exchanges;
      const uint8_t* addr = static_cast<const uint8_t*>(m->second.base) + row[8];
      if (a == 0) sa.ids = reinterpret_cast<const uint64_t*>(addr);
      else if (a == 1) sa.go = reinterpret_cast<const int32_t*>(addr);
      else if (a == 2) sa.cu = reinterpret_cast<const int64_t*>(addr);
      else if (a < 3 + s->n_ch) sa.ch[a - 3] = reinterpret_cast<const double*>(addr);
      else sa.st[a - 3 - s->n_ch] = addr;
    }
    out[p] = sa;
  }
  bool synced = false;  // retire mappings unused for 64 exchanges (their last reads are complete: synchronize)
  for (auto it = s->mappings.begin(); it != s->mappings.end();) {
    if (s->exchanges - it->second.last_use > 64) {
      if (!synced) {
        DFX_CUDA(cudaStreamSynchronize(s->stream));
        synced = true;
      }
      cudaIpcCloseMemHandle(it->second.base);
      it = s->mappings.erase(it);
    } else {
      ++it;
    }
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
  DFX_NCCL(GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return DFX_OK;
}

dfx_status dfx_comm_init(const void* id, int32_t n_ranks, int32_t rank, dfx_comm** out) {
  if (!id || !out || n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(DFX_INVALID_ARGUMENT, "dfx_comm_init: bad argument");
  auto c = std::make_unique<dfx_comm>();
  DFX_CUDA(cudaGetDevice(&c->device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  DFX_NCCL(CommInitRank(&c->nccl, n_ranks, uid, rank));
  c->rank = rank;
  c->n = n_ranks;
  dfx_status st = comm_reserve(c.get(), 4096);
  if (st) return st;
  if (n_ranks > 1) {  // the shared-memory side channel, named after the communicator's id
    const char* mb = std::getenv("DFX_SHM_SLOT_MB");
    c->slot_cap = int64_t(mb ? std::max(1, std::atoi(mb)) : 1) * (1 << 20) / 8;
    c->shm_bytes = kShmHeader + 2 * size_t(n_ranks) * shm_slot_bytes(c->slot_cap);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(uid); ++i) h = (h ^ uint8_t(reinterpret_cast<const char*>(&uid)[i])) * 1099511628211ull;
    char name[64];
    std::snprintf(name, sizeof(name), "/dfx.%016llx", (unsigned long long)h);
    int fd = -1;
    if (rank == 0) {
      fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0 || ftruncate(fd, off_t(c->shm_bytes)) != 0)
        return fail(DFX_ERROR, std::string("dfx_comm_init: cannot create shared memory ") + name);
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      for (;;) {
        fd = shm_open(name, O_RDWR, 0600);
        struct stat sb {};
        if (fd >= 0 && fstat(fd, &sb) == 0 && size_t(sb.st_size) >= c->shm_bytes) break;
        if (fd >= 0) close(fd);
        fd = -1;
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
          return fail(DFX_ERROR, std::string("dfx_comm_init: shared memory ") + name + " did not appear");
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
    }
    void* m = mmap(nullptr, c->shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return fail(DFX_ERROR, "dfx_comm_init: mmap of the shared memory failed");
    c->shm = static_cast<uint8_t*>(m);
    // every rank attached (a device all-reduce with a host synchronization), then the name can go
    int64_t one = 1, all = 0;
    cudaStream_t st0;
    DFX_CUDA(cudaStreamCreateWithFlags(&st0, cudaStreamNonBlocking));
    st = dfx_comm_allreduce_i64(c.get(), &one, &all, 1, st0);
    cudaStreamDestroy(st0);
    if (st) return st;
    if (rank == 0) shm_unlink(name);
    // flag arrays for the NVLink barrier: allocate, publish the IPC handle through the shared memory, map peers'
    if (n_ranks <= kMaxRanks) {
      DFX_CUDA(cudaMalloc(&c->flags, 2 * 4096));
      DFX_CUDA(cudaMemset(c->flags, 0, 2 * 4096));
      c->err = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(c->flags) + 4096);
      cudaIpcMemHandle_t h;
      DFX_CUDA(cudaIpcGetMemHandle(&h, c->flags));
      int64_t row[8];
      std::memcpy(row, &h, 64);
      std::vector<const int64_t*> rows;
      std::vector<int64_t> lens;
      st = host_allgatherv(c.get(), row, 8, rows, lens);
      if (st) return st;
      c->peer_flags.assign(n_ranks, nullptr);
      for (int r = 0; r < n_ranks; ++r) {
        if (r == rank) {
          c->peer_flags[r] = c->flags;
          continue;
        }
        cudaIpcMemHandle_t ph;
        std::memcpy(&ph, rows[r], 64);
        void* p = nullptr;
        DFX_CUDA(cudaIpcOpenMemHandle(&p, ph, cudaIpcMemLazyEnablePeerAccess));
        c->peer_flags[r] = static_cast<uint64_t*>(p);
      }
      // every rank mapped every flag array before anyone's first barrier can store into it
      std::vector<const int64_t*> rows2;
      st = host_allgatherv(c.get(), row, 1, rows2, lens);
      if (st) return st;
    }
  }
  *out = c.release();
  return DFX_OK;
}

dfx_status dfx_comm_destroy(dfx_comm* c) {
  if (!c) return DFX_OK;
  if (c->nccl && nccl().ok) nccl().CommDestroy(c->nccl);
  if (c->d_buf) cudaFree(c->d_buf);
  if (c->h_buf) cudaFreeHost(c->h_buf);
  if (c->shm) munmap(c->shm, c->shm_bytes);
  for (int r = 0; r < int(c->peer_flags.size()); ++r)
    if (r != c->rank && c->peer_flags[r]) cudaIpcCloseMemHandle(c->peer_flags[r]);
  if (c->flags) cudaFree(c->flags);
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
  DFX_NCCL(AllReduce(c->d_buf, c->d_buf, size_t(n), ncclInt64, ncclSum, c->nccl, stream));
  DFX_CUDA(cudaMemcpyAsync(c->h_buf, c->d_buf, size_t(n) * 8, cudaMemcpyDeviceToHost, stream));
  DFX_CUDA(cudaStreamSynchronize(stream));
  std::memcpy(out, c->h_buf, size_t(n) * 8);
  return DFX_OK;
}

dfx_status dfx_comm_alltoallv(dfx_comm* c, const void* send, const uint64_t* send_off, const uint64_t* send_bytes,
                              void* recv, const uint64_t* recv_off, const uint64_t* recv_bytes, dfx_stream stream) {
  if (!c || !send_off || !send_bytes || !recv_off || !recv_bytes)
    return fail(DFX_INVALID_ARGUMENT, "dfx_comm_alltoallv: null argument");
  const int me = c->rank;
  if (send_bytes[me]) {  // to self: a device copy
    if (send_bytes[me] != recv_bytes[me]) return fail(DFX_INVALID_ARGUMENT, "dfx_comm_alltoallv: self sizes differ");
    DFX_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + recv_off[me], static_cast<const uint8_t*>(send) + send_off[me],
                             send_bytes[me], cudaMemcpyDeviceToDevice, stream));
  }
  bool any = false;
  for (int p = 0; p < c->n; ++p) any = any || (p != me && (send_bytes[p] || recv_bytes[p]));
  if (!any) return DFX_OK;
  DFX_NCCL(GroupStart());
  for (int p = 0; p < c->n; ++p) {
    if (p == me) continue;
    if (send_bytes[p])
      DFX_NCCL(Send(static_cast<const uint8_t*>(send) + send_off[p], send_bytes[p], ncclUint8, p, c->nccl, stream));
    if (recv_bytes[p])
      DFX_NCCL(Recv(static_cast<uint8_t*>(recv) + recv_off[p], recv_bytes[p], ncclUint8, p, c->nccl, stream));
  }
  DFX_NCCL(GroupEnd());
  return DFX_OK;
}

dfx_status dfx_dstore_create(const dfx_dstore_cfg* cfg, dfx_comm* comm, dfx_stream stream, dfx_dstore** out) {
  if (!cfg || !comm || !out || !cfg->rank_of_worker) return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_create: null argument");
  if (cfg->num_nodes == 0 || cfg->workers_per_node == 0)
    return fail(DFX_LAYOUT_ERROR, "topology must have at least one node and one worker per node");
  if (cfg->n_streams < 0 || cfg->n_streams > DFX_MAX_STREAMS || cfg->n_ch < 0 || cfg->n_ch > DFX_MAX_CH)
    return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_create: too many streams or channels");
  if (cfg->transport != DFX_TRANSPORT_PULL && cfg->transport != DFX_TRANSPORT_NCCL)
    return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_create: unknown transport");
  auto s = std::make_unique<dfx_dstore>();
  s->comm = comm;
  s->stream = stream;
  s->transport = cfg->transport;
  s->trace = std::getenv("DFX_DSTORE_TRACE") != nullptr;
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
  {
    const char* e = std::getenv("DFX_DSTORE_CE_STREAMS");  // benchmarking knob
    const int n = e ? std::max(1, std::min(16, std::atoi(e))) : 4;
    DFX_CUDA(cudaEventCreateWithFlags(&s->ev_ce_fork, cudaEventDisableTiming));
    for (int q = 0; q < n; ++q) {
      cudaStream_t cs;
      cudaEvent_t ev;
      DFX_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      DFX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      s->ce.push_back(cs);
      s->ev_ce_join.push_back(ev);
    }
  }
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = s->device;
  DFX_CUDA(cudaMemPoolCreate(&s->pool, &props));
  uint64_t keep = UINT64_MAX;  // keep freed scratch for reuse: a steady-state loop allocates nothing
  DFX_CUDA(cudaMemPoolSetAttribute(s->pool, cudaMemPoolAttrReleaseThreshold, &keep));
  *out = s.release();
  return DFX_OK;
}

dfx_status dfx_dstore_destroy(dfx_dstore* s) {
  if (!s) return DFX_OK;
  if (s->trace && !s->spans.empty()) {
    cudaStreamSynchronize(s->stream);
    std::map<std::string, std::pair<double, int>> acc;
    for (auto& [name, a, b] : s->spans) {
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      acc[name].first += ms;
      acc[name].second += 1;
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    for (auto& [name, v] : acc)
      std::fprintf(stderr, "[dstore trace rank %d] %-34s %8.1f us avg over %d\n", s->comm->rank, name.c_str(),
                   1e3 * v.first / v.second, v.second);
  }
  for (auto& kv : s->entries) retire(s, kv.second.r);
  cudaStreamSynchronize(s->stream);
  cudaStreamSynchronize(s->side);
  for (auto& kv : s->mappings) cudaIpcCloseMemHandle(kv.second.base);
  for (auto& kv : s->block_free) cudaFree(kv.second);
  for (void* p : s->pinned_free) cudaFreeHost(p);
  if (s->pool) cudaMemPoolDestroy(s->pool);
  if (s->side) cudaStreamDestroy(s->side);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  for (cudaStream_t cs : s->ce) {
    cudaStreamSynchronize(cs);
    cudaStreamDestroy(cs);
  }
  for (cudaEvent_t ev : s->ev_ce_join) cudaEventDestroy(ev);
  if (s->ev_ce_fork) cudaEventDestroy(s->ev_ce_fork);
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
  if (to_dp == 0 || to_tp == 0)
    return fail(DFX_LAYOUT_ERROR, "dp_size and tp_size must be positive for stage '" + std::string(stage) + "'");
  if (it < s->low_water)
    return fail(DFX_STALE_ITERATION, "get for iteration " + std::to_string(it) + " below low water " +
                                         std::to_string(s->low_water));
  Entry& e = s->entries[{stage, it}];
  if (e.ready) return DFX_OK;
  const int me = s->comm->rank, world = s->comm->n;
  std::vector<int> src_rank(c.pdp);
  std::vector<uint32_t> local_p;
  for (uint32_t p = 0; p < c.pdp; ++p) {
    src_rank[p] = s->rank_of_worker[size_t(p) * c.ptp];
    if (src_rank[p] == me) local_p.push_back(p);
  }
  size_t missing = 0;
  for (uint32_t p : local_p) missing += e.by_group.count(p) ? 0 : 1;
  if (missing)
    return fail(DFX_NOT_READY, std::string("stage '") + stage + "' iteration " + std::to_string(it) +
                                   " not ready: " + std::to_string(missing) + " puts outstanding");  // :340-344
  ++s->exchanges;
  const bool pull = s->transport == DFX_TRANSPORT_PULL && world > 1;
  const int NA = n_arrays(s);

  // ---- the host all-gather: every local producer group's host offsets (+ IPC handles for the pull) ----
  std::vector<int64_t>& row = s->row;  // reused: no allocation in a steady-state loop
  row.assign(1, int64_t(local_p.size()));
  for (uint32_t p : local_p) {
    const Held& h = e.by_group.at(p);
    const size_t o = row.size();
    row.resize(o + 4 + h.hgo.size() + h.hcu.size());
    int64_t* w = row.data() + o;
    w[0] = p;
    w[1] = h.b.n_records;
    w[2] = h.b.n_rollouts;
    w[3] = pull ? NA * kHandleCols : 0;
    w += 4;
    for (size_t q = 0; q < h.hgo.size(); ++q) w[q] = h.hgo[q];
    std::memcpy(w + h.hgo.size(), h.hcu.data(), h.hcu.size() * 8);
    if (pull) {
      for (int a = 0; a < NA; ++a) {
        const void* ptr = array_ptr(s, h.b, a);
        int64_t cols[kHandleCols] = {};
        if (ptr) {
          std::string hd;
          uint64_t off = 0;
          dfx_status st = export_ptr(s, ptr, hd, off);
          if (st) return st;
          std::memcpy(cols, hd.data(), 64);
          cols[8] = int64_t(off);
        }
        row.insert(row.end(), cols, cols + kHandleCols);
      }
    }
  }
  std::vector<const int64_t*> rows;
  std::vector<int64_t> lens;
  dfx_status st = host_allgatherv(s->comm, row.data(), int64_t(row.size()), rows, lens);
  if (st) return st;
  std::vector<GInfo> info(c.pdp);
  for (int r = 0; r < world; ++r) {
    const int64_t* x = rows[r];
    const int64_t ng = x[0];
    size_t o = 1;
    for (int64_t q = 0; q < ng; ++q) {
      const int64_t p = x[o], nr = x[o + 1], ns = x[o + 2], nh = x[o + 3];
      o += 4;
      if (p < 0 || p >= int64_t(c.pdp)) return fail(DFX_ERROR, "host all-gather: bad producer group");
      GInfo& gi = info[size_t(p)];
      gi.present = true;
      gi.n_rec = nr;
      gi.n_roll = ns;
      gi.go = x + o;
      o += size_t(nr + 1);
      gi.cu = x + o;
      o += size_t(ns + 1);
      gi.handles = nh ? x + o : nullptr;
      o += size_t(nh);
    }
  }
  std::vector<uint64_t> counts(c.pdp);
  for (uint32_t p = 0; p < c.pdp; ++p) counts[p] = uint64_t(info[p].n_rec);

  // ---- the placement (cached while the group sizes repeat) and the segments' sizes ----
  PlanCache& pc = s->plans[stage];
  if (pc.valid && pc.to_dp == to_dp && pc.to_tp == to_tp && pc.counts == counts) {
    ++s->plan_hits;
  } else {
    st = plan_segments(s, c, to_dp, to_tp, counts, pc.segs);
    if (st) return st;
    pc.valid = true;
    pc.to_dp = to_dp;
    pc.to_tp = to_tp;
    pc.counts = counts;
  }
  std::vector<PSeg> segs = pc.segs;
  for (PSeg& sg : segs) seg_sizes(info[sg.src], sg);

  std::map<uint32_t, SrcArrays> remote_src;
  if (pull) {
    std::vector<uint32_t> local_dst;
    for (uint32_t d = 0; d < to_dp; ++d) {
      const auto rk = dst_ranks(s, d, to_tp);
      if (std::find(rk.begin(), rk.end(), me) != rk.end()) local_dst.push_back(d);
    }
    st = map_remote(s, src_rank, segs, local_dst, info, remote_src);
    if (st) return st;
    // every rank's stream has executed what preceded its barrier (the production of the batches put): the
    // consumers may read the producers' memory after it -- a device-side wait, no host synchronization
    cudaEvent_t t0 = trace_mark(s);
    st = comm_barrier(s->comm, s->stream);
    if (st) return st;
    trace_span(s, "barrier (production done)", t0);
  }
  cudaEvent_t t1 = trace_mark(s);
  st = run_exchange(s, c, to_dp, to_tp, e, segs, info, remote_src);
  if (st) return st;
  trace_span(s, "exchange (views, pulls, unpack)", t1);
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
  *out = g->second.b;
  return DFX_OK;
}

dfx_status dfx_dstore_worker_done(dfx_dstore* s, uint64_t it) {
  if (!s) return fail(DFX_INVALID_ARGUMENT, "dfx_dstore_worker_done: null");
  const uint32_t n = ++s->done[it];
  if (n < s->local_workers) return DFX_OK;
  s->done.erase(it);
  s->low_water = std::max(s->low_water, it + 1);
  // release (pull transport): peers may still be reading this rank's producer memory and the consumer blocks
  // about to be recycled; a device-side barrier orders every later write on this stream after their reads
  if (s->transport == DFX_TRANSPORT_PULL && s->comm->n > 1) {
    cudaEvent_t t0 = trace_mark(s);
    dfx_status st = comm_barrier(s->comm, s->stream);
    if (st) return st;
    trace_span(s, "release barrier", t0);
  }
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
