// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference implementation.
//
// TEST INFRASTRUCTURE ONLY. Compiled by oracle/Makefile against the headers
// where they lie (/root/reference/proj/include) into oracle/_ref/, which is
// git-ignored. Used by tests/ (to pin the C restatement and to generate
// golden fixtures) and by bench.py's reference / cpu_baseline arm. Nothing in
// the product links it.
//
// Every entry point calls the reference's own functions:
//   fn_generate / fn_reward / fn_value      distflow/functions.hpp:108-138
//   fn_group_advantage / fn_ppo_advantage   distflow/functions.hpp:143-172
//   BufferStore put / redistribute / get    distflow/data_plane.hpp:237-479
//   serialize_records                       distflow/record.hpp:151-156
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "distflow/data_plane.hpp"
#include "distflow/functions.hpp"
#include "distflow/record.hpp"
#include "distflow/topology.hpp"
#include "distflow/transport.hpp"

using namespace distflow;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const LayoutError*>(&e)) return 2;
  if (dynamic_cast<const IndivisibleError*>(&e)) return 3;
  if (dynamic_cast<const MissingRolloutsError*>(&e)) return 4;
  if (dynamic_cast<const MissingChannelError*>(&e)) return 5;
  if (dynamic_cast<const StaleIterationError*>(&e)) return 6;
  if (dynamic_cast<const NotReadyError*>(&e)) return 7;
  if (dynamic_cast<const UnknownStageError*>(&e)) return 8;
  return 1;
}

NodeSpec compute_node() {
  NodeSpec n;
  n.node_id = "n";
  n.role = Role::NONE;
  n.node_type = NodeType::COMPUTE;
  return n;
}

// Packed SoA batch -> reference AoS records. Payload of rollout s is the
// concatenation of the token streams' slices (our documented payload layout).
struct PackedView {
  uint32_t n_records;
  const uint64_t* ids;
  const int64_t* meta_off;
  const uint8_t* meta_blob;
  const int32_t* group_off;
  const uint32_t* tok_count;
  const int64_t* cu;
  int n_streams;
  const void* const* streams;
  const uint32_t* esz;
  int n_ch;
  const char* const* ch_names;
  const double* const* ch_vals;
};

SampleRecord record_of(const PackedView& v, uint32_t r) {
  SampleRecord rec;
  rec.sample_id = v.ids[r];
  if (v.meta_off) {
    // meta section bytes are u32 count + (str,str)*; parse with the reference reader
    const uint8_t* p = v.meta_blob + v.meta_off[r];
    const size_t n = size_t(v.meta_off[r + 1] - v.meta_off[r]);
    blob::Reader in(p, n);
    const uint32_t nm = in.u32();
    for (uint32_t i = 0; i < nm; ++i) {
      std::string k = in.str();
      rec.meta[k] = in.str();
    }
  }
  for (int32_t s = v.group_off[r]; s < v.group_off[r + 1]; ++s) {
    Rollout ro;
    ro.token_count = v.tok_count[s];
    const int64_t L = v.cu[s + 1] - v.cu[s];
    for (int k = 0; k < v.n_streams; ++k) {
      const uint8_t* b = static_cast<const uint8_t*>(v.streams[k]) + uint64_t(v.cu[s]) * v.esz[k];
      ro.payload.insert(ro.payload.end(), b, b + uint64_t(L) * v.esz[k]);
    }
    for (int c = 0; c < v.n_ch; ++c) ro.channels[v.ch_names[c]] = v.ch_vals[c][s];
    rec.rollouts.push_back(std::move(ro));
  }
  return rec;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_splitmix64(uint64_t z) { return splitmix64(z); }
uint64_t ref_keyed_hash2(uint64_t seed, const char* dom, uint64_t a, uint64_t b) {
  return keyed_hash(seed, dom, a, b);
}
uint64_t ref_keyed_hash3(uint64_t seed, const char* dom, uint64_t a, uint64_t b, uint64_t c) {
  return keyed_hash(seed, dom, a, b, c);
}
double ref_unit_from_hash(uint64_t h) { return unit_from_hash(h); }
double ref_symmetric_from_hash(uint64_t h) { return symmetric_from_hash(h); }
void ref_hash_bytes(uint64_t key, uint8_t* out, size_t n) {
  auto v = hash_bytes(key, n);
  std::memcpy(out, v.data(), n);
}

// fn_generate over records ids[0..n) with rollouts_per_prompt n_roll; writes
// per-rollout token counts and (optionally) payload bytes.
int ref_generate(uint64_t seed, int kind, uint32_t value, uint32_t mn, uint32_t mx, uint32_t n_roll,
                 uint32_t bytes_per_token, const uint64_t* ids, uint32_t n_records,
                 uint32_t* token_counts, uint8_t* payload_out) {
  try {
    StageContext ctx;
    ctx.run_seed = seed;
    ctx.gen.rollouts_per_prompt = n_roll;
    ctx.gen.bytes_per_token = bytes_per_token;
    ctx.gen.response_tokens.kind = kind == 0 ? TokenDist::Kind::CONSTANT : TokenDist::Kind::UNIFORM;
    ctx.gen.response_tokens.value = value;
    ctx.gen.response_tokens.min = mn;
    ctx.gen.response_tokens.max = mx;
    SampleBatch b;
    for (uint32_t r = 0; r < n_records; ++r) {
      SampleRecord rec;
      rec.sample_id = ids[r];
      b.records.push_back(std::move(rec));
    }
    fn_generate(compute_node(), b, ctx);
    uint64_t s = 0, off = 0;
    for (const auto& rec : b.records)
      for (const auto& ro : rec.rollouts) {
        token_counts[s++] = ro.token_count;
        if (payload_out) {
          std::memcpy(payload_out + off, ro.payload.data(), ro.payload.size());
          off += ro.payload.size();
        }
      }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// make_group_loader(synthetic dataset of dataset_n rows, dp, dp_rank, seed, shuffle).next_batch(iteration,
// global_batch): writes the sample ids of the batch (global_batch / dp of them) into out_ids.
int ref_loader_ids(uint64_t dataset_n, uint32_t dp, uint32_t dp_rank, uint64_t seed, int shuffle,
                   uint32_t iteration, uint64_t global_batch, uint64_t* out_ids) {
  try {
    DatasetSpec spec;
    spec.synthetic_n = dataset_n;
    spec.prompt_tokens = 1;
    ParallelLayout layout;
    layout.dp_size = dp;
    const DataLoader loader = make_group_loader(spec, layout, dp_rank, seed, shuffle != 0);
    const auto recs = loader.next_batch(iteration, global_batch);
    for (size_t i = 0; i < recs.size(); ++i) out_ids[i] = recs[i].sample_id;
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// fn_reward / fn_value / fn_ref_logprob on records with n_roll empty rollouts.
int ref_fill_channels(uint64_t seed, const uint64_t* ids, uint32_t n_records, uint32_t n_roll,
                      double* reward, double* value, double* ref_logprob) {
  try {
    StageContext ctx;
    ctx.run_seed = seed;
    SampleBatch b;
    for (uint32_t r = 0; r < n_records; ++r) {
      SampleRecord rec;
      rec.sample_id = ids[r];
      rec.rollouts.resize(n_roll);
      b.records.push_back(std::move(rec));
    }
    fn_reward(compute_node(), b, ctx);
    fn_value(compute_node(), b, ctx);
    fn_ref_logprob(compute_node(), b, ctx);
    uint64_t s = 0;
    for (const auto& rec : b.records)
      for (const auto& ro : rec.rollouts) {
        reward[s] = ro.channels.at("reward");
        value[s] = ro.channels.at("value");
        ref_logprob[s] = ro.channels.at("ref_logprob");
        ++s;
      }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// fn_group_advantage (ppo=0) or fn_ppo_advantage (ppo=1). value may be NULL
// (then the channel is absent, exercising MissingChannelError).
int ref_advantage(int ppo, uint32_t n_records, const int32_t* group_off, const double* reward,
                  const double* value, double eps, double* adv) {
  try {
    StageContext ctx;
    ctx.advantage_eps = eps;
    SampleBatch b;
    for (uint32_t r = 0; r < n_records; ++r) {
      SampleRecord rec;
      rec.sample_id = r;
      for (int32_t s = group_off[r]; s < group_off[r + 1]; ++s) {
        Rollout ro;
        if (reward) ro.channels["reward"] = reward[s];
        if (value) ro.channels["value"] = value[s];
        rec.rollouts.push_back(std::move(ro));
      }
      b.records.push_back(std::move(rec));
    }
    if (ppo) fn_ppo_advantage(compute_node(), b, ctx);
    else fn_group_advantage(compute_node(), b, ctx);
    uint64_t s = 0;
    for (const auto& rec : b.records)
      for (const auto& ro : rec.rollouts) adv[s++] = ro.channels.at("advantage");
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// serialize_records of a packed batch.
int64_t ref_serialize_packed(uint32_t n_records, const uint64_t* ids, const int64_t* meta_off,
                             const uint8_t* meta_blob, const int32_t* group_off,
                             const uint32_t* tok_count, const int64_t* cu, int n_streams,
                             const void* const* streams, const uint32_t* esz, int n_ch,
                             const char* const* ch_names, const double* const* ch_vals,
                             uint8_t* out, int64_t cap) {
  PackedView v{n_records, ids, meta_off, meta_blob, group_off, tok_count, cu,
               n_streams,  streams, esz, n_ch, ch_names, ch_vals};
  std::vector<SampleRecord> recs;
  for (uint32_t r = 0; r < n_records; ++r) recs.push_back(record_of(v, r));
  auto blob = serialize_records(recs);
  if (out && int64_t(blob.size()) <= cap) std::memcpy(out, blob.data(), blob.size());
  return int64_t(blob.size());
}

// Full reference reshard: B stores x W workers over one InprocFabric.
// Producer group p puts records [goff[p], goff[p+1]) of the packed batch
// (p's TP-0 worker puts; TP peers' puts are suppressed). Then every store runs
// ensure_ready (redistribute) and each destination group d gets its batch.
// Outputs: dest_counts[d] = #records; dest_ids (dest-major) = sample ids;
// if blob_out: serialize_records(get(d).records) concatenated, blob_off[d].
// stats[0..B) = redistribution_bytes_sent per store, stats[B..2B) received.
int ref_reshard(uint32_t B, uint32_t W, uint32_t dp_p, uint32_t tp_p, uint32_t dp_c, uint32_t tp_c,
                const uint64_t* group_counts, uint32_t n_records, const uint64_t* ids,
                const int64_t* meta_off, const uint8_t* meta_blob, const int32_t* group_off,
                const uint32_t* tok_count, const int64_t* cu, int n_streams,
                const void* const* streams, const uint32_t* esz, int n_ch,
                const char* const* ch_names, const double* const* ch_vals, uint64_t* dest_counts,
                uint64_t* dest_ids, uint8_t* blob_out, int64_t blob_cap, int64_t* blob_off,
                uint64_t* stats) {
  try {
    const ClusterTopology topo{B, W};
    topo.validate();
    const ParallelLayout produced{dp_p, tp_p}, consumed{dp_c, tp_c};
    check_layout(produced, topo, "produced");
    check_layout(consumed, topo, "consumed");
    PackedView v{n_records, ids, meta_off, meta_blob, group_off, tok_count, cu,
                 n_streams,  streams, esz, n_ch, ch_names, ch_vals};
    InprocFabric fabric(topo);
    std::map<std::string, StoreStagePlan> stages;
    stages["s"] = StoreStagePlan{produced, consumed, tags::kRedistBase};
    std::vector<std::unique_ptr<BufferStore>> stores;
    std::vector<BufferStore*> ptrs;
    for (uint32_t b = 0; b < B; ++b) {
      stores.push_back(std::make_unique<BufferStore>(topo, b, &fabric, stages));
      ptrs.push_back(stores.back().get());
    }
    uint64_t first = 0;
    for (uint32_t p = 0; p < dp_p; ++p) {
      SampleBatch batch;
      batch.stage_id = "s";
      for (uint64_t i = 0; i < group_counts[p]; ++i) batch.records.push_back(record_of(v, uint32_t(first + i)));
      first += group_counts[p];
      const uint32_t lead = produced.group_lead(p);
      const uint32_t node = topo.node_of(lead);
      for (uint32_t t = 0; t < tp_p; ++t) stores[node]->put("s", 0, p, t, batch);
    }
    redistribute(ptrs, "s", 0, consumed);
    uint64_t w = 0;
    int64_t boff = 0;
    for (uint32_t d = 0; d < dp_c; ++d) {
      const uint32_t node = topo.node_of(consumed.group_lead(d));
      const SampleBatch got = stores[node]->get("s", 0, d, consumed);
      dest_counts[d] = got.records.size();
      for (const auto& r : got.records) dest_ids[w++] = r.sample_id;
      if (blob_out) {
        auto bl = serialize_records(got.records);
        if (boff + int64_t(bl.size()) > blob_cap) throw Error("blob capacity exceeded");
        std::memcpy(blob_out + boff, bl.data(), bl.size());
        blob_off[d] = boff;
        boff += int64_t(bl.size());
        blob_off[d + 1] = boff;
      }
    }
    if (stats) {
      for (uint32_t b = 0; b < B; ++b) {
        stats[b] = stores[b]->redistribution_bytes_sent();
        stats[B + b] = stores[b]->redistribution_bytes_received();
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// ---- CPU baseline timing (reference code on this host's cores) -------------
//
// Times the reference's own implementation of the path on a prebuilt batch:
// fn_group_advantage over nthreads partitions of records (one thread per
// logical worker, as runner.hpp:525-530 runs workers), then a BufferStore
// put -> redistribute -> get reshard from (B,W,dp_p,tp_p) to (dp_c,tp_c).
// Returns seconds per repetition for each phase in out[0] (advantage),
// out[1] (reshard).
int ref_bench(uint32_t n_records, const uint64_t* ids, const int32_t* group_off,
              const uint32_t* tok_count, const int64_t* cu, const double* reward, int n_streams,
              const void* const* streams, const uint32_t* esz, uint32_t B, uint32_t W,
              uint32_t dp_p, uint32_t tp_p, uint32_t dp_c, uint32_t tp_c, int nthreads, int reps,
              double* out) {
  try {
    const char* names[1] = {"reward"};
    const double* vals[1] = {reward};
    PackedView v{n_records, ids, nullptr, nullptr, group_off, tok_count, cu,
                 n_streams,  streams, esz, 1, names, vals};
    // one batch per producing DP group (contiguous record ranges)
    const ClusterTopology topo{B, W};
    const ParallelLayout produced{dp_p, tp_p}, consumed{dp_c, tp_c};
    check_layout(produced, topo, "produced");
    check_layout(consumed, topo, "consumed");
    if (n_records % dp_p) throw IndivisibleError("global batch", n_records, dp_p);
    const uint32_t per = n_records / dp_p;
    std::vector<SampleBatch> groups(dp_p);
    for (uint32_t p = 0; p < dp_p; ++p) {
      groups[p].stage_id = "s";
      for (uint32_t i = 0; i < per; ++i) groups[p].records.push_back(record_of(v, p * per + i));
    }
    double t_adv = 0, t_rs = 0;
    for (int rep = 0; rep < reps; ++rep) {
      std::vector<SampleBatch> work = groups;  // fresh copy, not timed
      auto t0 = std::chrono::steady_clock::now();
      {
        std::vector<std::thread> th;
        const int nt = std::max(1, std::min<int>(nthreads, int(dp_p)));
        for (int k = 0; k < nt; ++k)
          th.emplace_back([&, k] {
            StageContext ctx;
            for (uint32_t p = uint32_t(k); p < dp_p; p += uint32_t(nt))
              fn_group_advantage(compute_node(), work[p], ctx);
          });
        for (auto& t : th) t.join();
      }
      auto t1 = std::chrono::steady_clock::now();
      InprocFabric fabric(topo);
      std::map<std::string, StoreStagePlan> stages;
      stages["s"] = StoreStagePlan{produced, consumed, tags::kRedistBase};
      std::vector<std::unique_ptr<BufferStore>> stores;
      for (uint32_t b = 0; b < B; ++b)
        stores.push_back(std::make_unique<BufferStore>(topo, b, &fabric, stages));
      auto t2 = std::chrono::steady_clock::now();
      // one thread per worker rank, like run_iteration's put then get
      {
        std::vector<std::thread> th;
        for (uint32_t rank = 0; rank < topo.world_size(); ++rank)
          th.emplace_back([&, rank] {
            const uint32_t dp = produced.dp_rank(rank), tp = produced.tp_rank(rank);
            const uint32_t node = topo.node_of(rank);
            SampleBatch mine = tp == 0 ? std::move(work[dp]) : SampleBatch{};
            stores[node]->put("s", 0, dp, tp, std::move(mine));
            SampleBatch got = stores[node]->get("s", 0, consumed.dp_rank(rank), consumed);
            (void)got;
          });
        for (auto& t : th) t.join();
      }
      auto t3 = std::chrono::steady_clock::now();
      t_adv += std::chrono::duration<double>(t1 - t0).count();
      t_rs += std::chrono::duration<double>(t3 - t2).count();
    }
    out[0] = t_adv / reps;
    out[1] = t_rs / reps;
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

}  // extern "C"
