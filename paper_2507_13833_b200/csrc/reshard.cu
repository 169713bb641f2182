// reshard.cu -- DataBuffer DP m->n reshard: placement plan (host) + pack/unpack kernels (device).
//
// Placement restates BufferStore::exchange/get (distflow/data_plane.hpp:237-442) with the layout checks of
// distflow/topology.hpp:53-68: store b holds producer groups [b*gpn_p, (b+1)*gpn_p) in dp order; if the dp size
// changes every store's list is cut into B equal parts and part k of every store, in store order, forms store
// k's holdings; destination group d (store k = d / gpn_c) receives the contiguous slice
// [(d - k*gpn_c)*r, +r) of H_k. The plan is expressed as segments: maximal runs of consecutive records of one
// producer group landing consecutively in one destination group. Data moves per segment: token streams as
// contiguous byte ranges (NCCL P2P or device copies, driven by the host runtime), record/rollout metadata through
// the pack/unpack kernels below, which rebase offsets into the destination batch.
#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"

namespace dfx {

namespace {

dfx_status check_layout(uint32_t dp, uint32_t tp, uint32_t world, uint32_t W, const char* which) {
  const std::string where = std::string(" for stage '") + which + "'";
  if (dp == 0 || tp == 0) return fail(DFX_LAYOUT_ERROR, "dp_size and tp_size must be positive" + where);
  if (dp * tp != world)
    return fail(DFX_LAYOUT_ERROR, "dp_size * tp_size = " + std::to_string(dp * tp) + " != world_size " +
                                      std::to_string(world) + where);
  if (W % tp != 0)
    return fail(DFX_LAYOUT_ERROR, "tp_size " + std::to_string(tp) + " does not divide workers_per_node " +
                                      std::to_string(W) + where);
  return DFX_OK;
}

dfx_status indivisible(const std::string& what, uint64_t dividend, uint64_t divisor) {
  return fail(DFX_INDIVISIBLE_ERROR, what + ": " + std::to_string(divisor) + " does not divide " + std::to_string(dividend));
}

// Destination index list (dest-major) as indices into ordered = L_0 || ... || L_{dp_p-1}.
dfx_status placement(uint32_t B, uint32_t W, uint32_t dp_p, uint32_t tp_p, uint32_t dp_c, uint32_t tp_c,
                     const uint64_t* gc, std::vector<uint64_t>& dest_counts, std::vector<uint64_t>& idx) {
  if (B == 0 || W == 0) return fail(DFX_LAYOUT_ERROR, "topology must have at least one node and one worker per node");
  const uint32_t world = B * W;
  dfx_status st = check_layout(dp_p, tp_p, world, W, "produced");
  if (st) return st;
  st = check_layout(dp_c, tp_c, world, W, "consumed");
  if (st) return st;
  const uint32_t gpn_p = W / tp_p, gpn_c = W / tp_c;
  std::vector<uint64_t> goff(dp_p + 1, 0);
  for (uint32_t p = 0; p < dp_p; ++p) goff[p + 1] = goff[p] + gc[p];
  // store b's ordered list O_b = [goff[b*gpn_p], goff[(b+1)*gpn_p])
  std::vector<std::vector<uint64_t>> H(B);
  if (dp_c == dp_p) {  // fast path (data_plane.hpp:411-413)
    for (uint32_t b = 0; b < B; ++b)
      for (uint64_t i = goff[b * gpn_p]; i < goff[(b + 1) * gpn_p]; ++i) H[b].push_back(i);
  } else {
    for (uint32_t b = 0; b < B; ++b) {
      const uint64_t n = goff[(b + 1) * gpn_p] - goff[b * gpn_p];
      if (n % B) return indivisible("per-store record count", n, B);  // :414-416
    }
    for (uint32_t k = 0; k < B; ++k)
      for (uint32_t j = 0; j < B; ++j) {
        const uint64_t o = goff[j * gpn_p], q = (goff[(j + 1) * gpn_p] - o) / B;
        for (uint64_t i = 0; i < q; ++i) H[k].push_back(o + uint64_t(k) * q + i);  // :418-435
      }
  }
  dest_counts.assign(dp_c, 0);
  idx.clear();
  for (uint32_t k = 0; k < B; ++k)
    if (H[k].size() % gpn_c) return indivisible("store holdings", H[k].size(), gpn_c);  // :281-283
  for (uint32_t d = 0; d < dp_c; ++d) {
    const uint32_t k = d / gpn_c;
    const uint64_t r = H[k].size() / gpn_c, at = uint64_t(d - k * gpn_c) * r;
    dest_counts[d] = r;
    idx.insert(idx.end(), H[k].begin() + at, H[k].begin() + at + r);
  }
  return DFX_OK;
}

}  // namespace

// ---- metadata pack / unpack --------------------------------------------------------------
// Grid (segment, 256-entry chunk); the segment table travels by value in the kernel parameters (no H2D copy, no
// host sync).
// Unpack rebases: dst_go[dr+i] = go[i]-go[0]+droll ; dst_cu[droll+j] = cu[j]-cu[0]+dtok ;
// roll_group[droll+j] = dr + (record of rollout j) ; ids / channels copied. Source pointers may be peer-mapped
// (NVLink pull transport): the kernel then reads the producer GPU's metadata directly.
constexpr int kSegsPerLaunch = 48;
struct SegBatch {
  dfx_seg_meta seg[kSegsPerLaunch];
  double* dst_ch[4];
  uint8_t* out[kSegsPerLaunch];
};

__global__ void unpack_kernel(const SegBatch sb, int n_ch, uint64_t* dst_ids, int32_t* dst_go, int32_t* dst_rg,
                              int64_t* dst_cu) {
  // CTA (segment x, chunk y) handles records and rollouts [y*B, y*B + B): the source metadata often sits in a
  // peer GPU's memory, so the loads of a segment are spread over many CTAs instead of looping in one (each loop
  // trip would pay an NVLink round trip)
  const dfx_seg_meta& m = sb.seg[blockIdx.x];
  double* const* dst_ch = sb.dst_ch;
  const int64_t i = int64_t(blockIdx.y) * blockDim.x + threadIdx.x;
  if (i > m.n_rec && i > m.n_roll) return;
  const int64_t g0 = m.group_off[0], c0 = m.cu[0];
  if (i <= m.n_rec) {
    const int64_t gi = m.group_off[i];
    dst_go[m.dst_rec + i] = (int32_t)(gi - g0 + m.dst_roll);
    if (i < m.n_rec) {
      dst_ids[m.dst_rec + i] = m.ids[i];
      const int64_t ge = m.group_off[i + 1];
      for (int64_t j = gi; j < ge; ++j) dst_rg[m.dst_roll + (j - g0)] = (int32_t)(m.dst_rec + i);
    }
  }
  if (i <= m.n_roll) {
    dst_cu[m.dst_roll + i] = m.cu[i] - c0 + m.dst_tok;
    if (i < m.n_roll)
      for (int c = 0; c < n_ch; ++c) dst_ch[c][m.dst_roll + i] = m.ch[c][i];
  }
}

__global__ void pack_kernel(const SegBatch sb, int n_ch) {
  const dfx_seg_meta& m = sb.seg[blockIdx.x];
  const int64_t i = int64_t(blockIdx.y) * blockDim.x + threadIdx.x;  // chunked like unpack_kernel
  if (i > m.n_rec && i > m.n_roll) return;
  uint8_t* o = sb.out[blockIdx.x];
  uint64_t* ids = reinterpret_cast<uint64_t*>(o);
  int64_t* cu = reinterpret_cast<int64_t*>(ids + m.n_rec);
  double* ch = reinterpret_cast<double*>(cu + m.n_roll + 1);
  int32_t* go = reinterpret_cast<int32_t*>(ch + int64_t(n_ch) * m.n_roll);
  if (i <= m.n_rec) {
    go[i] = m.group_off[i];
    if (i < m.n_rec) ids[i] = m.ids[i];
  }
  if (i <= m.n_roll) {
    cu[i] = m.cu[i];
    if (i < m.n_roll)
      for (int c = 0; c < n_ch; ++c) ch[int64_t(c) * m.n_roll + i] = m.ch[c][i];
  }
}

}  // namespace dfx

using namespace dfx;

extern "C" {

dfx_status dfx_reshard_placement(uint32_t B, uint32_t W, uint32_t dp_p, uint32_t tp_p, uint32_t dp_c, uint32_t tp_c,
                                 const uint64_t* group_counts, uint64_t* dest_counts, uint64_t* src_index) {
  std::vector<uint64_t> dc, idx;
  const dfx_status st = placement(B, W, dp_p, tp_p, dp_c, tp_c, group_counts, dc, idx);
  if (st) return st;
  std::copy(dc.begin(), dc.end(), dest_counts);
  if (src_index) std::copy(idx.begin(), idx.end(), src_index);
  return DFX_OK;
}

int64_t dfx_reshard_segments(uint32_t B, uint32_t W, uint32_t dp_p, uint32_t tp_p, uint32_t dp_c, uint32_t tp_c,
                             const uint64_t* group_counts, dfx_segment* out, int64_t cap) {
  std::vector<uint64_t> dc, idx;
  const dfx_status st = placement(B, W, dp_p, tp_p, dp_c, tp_c, group_counts, dc, idx);
  if (st) return -int64_t(st);
  std::vector<uint64_t> goff(dp_p + 1, 0);
  for (uint32_t p = 0; p < dp_p; ++p) goff[p + 1] = goff[p] + group_counts[p];
  std::vector<dfx_segment> segs;
  uint64_t w = 0;
  for (uint32_t d = 0; d < dp_c; ++d) {
    for (uint64_t i = 0; i < dc[d]; ++i, ++w) {
      const uint64_t g = idx[w];
      const uint32_t p = uint32_t(std::upper_bound(goff.begin(), goff.end(), g) - goff.begin()) - 1;
      const uint64_t off = g - goff[p];
      if (!segs.empty()) {
        dfx_segment& last = segs.back();
        if (last.dst_group == d && last.src_group == p && last.src_rec + last.count == off &&
            last.dst_rec + last.count == i) {
          ++last.count;
          continue;
        }
      }
      segs.push_back(dfx_segment{d, p, i, off, 1});
    }
  }
  const int64_t n = int64_t(segs.size());
  if (out) std::copy(segs.begin(), segs.begin() + std::min<int64_t>(n, cap), out);
  return n;
}

dfx_status dfx_reshard_unpack(const dfx_seg_meta* segs, int32_t n_segs, int32_t n_ch, uint64_t* dst_ids,
                              int32_t* dst_group_off, int32_t* dst_roll_group, int64_t* dst_cu,
                              double* const* dst_ch, dfx_stream stream) {
  if (n_segs <= 0) return DFX_OK;
  if (!segs || !dst_ids || !dst_group_off || !dst_roll_group || !dst_cu || (n_ch > 0 && !dst_ch) || n_ch > 4)
    return fail(DFX_INVALID_ARGUMENT, "dfx_reshard_unpack: bad argument");
  for (int32_t s0 = 0; s0 < n_segs; s0 += kSegsPerLaunch) {
    const int32_t n = std::min<int32_t>(kSegsPerLaunch, n_segs - s0);
    SegBatch sb{};
    int64_t span = 1;
    for (int32_t i = 0; i < n; ++i) {
      sb.seg[i] = segs[s0 + i];
      span = std::max<int64_t>(span, std::max(segs[s0 + i].n_rec, segs[s0 + i].n_roll) + 1);
    }
    for (int32_t c = 0; c < n_ch; ++c) sb.dst_ch[c] = dst_ch[c];
    unpack_kernel<<<dim3(n, unsigned((span + 255) / 256)), 256, 0, stream>>>(sb, n_ch, dst_ids, dst_group_off,
                                                                           dst_roll_group, dst_cu);
    DFX_LAUNCH_CHECK("unpack_kernel");
  }
  return DFX_OK;
}

dfx_status dfx_reshard_pack(const dfx_seg_meta* segs, int32_t n_segs, int32_t n_ch, uint8_t* const* out,
                            dfx_stream stream) {
  if (n_segs <= 0) return DFX_OK;
  if (!segs || !out || n_ch > 4) return fail(DFX_INVALID_ARGUMENT, "dfx_reshard_pack: bad argument");
  for (int32_t s0 = 0; s0 < n_segs; s0 += kSegsPerLaunch) {
    const int32_t n = std::min<int32_t>(kSegsPerLaunch, n_segs - s0);
    SegBatch sb{};
    int64_t span = 1;
    for (int32_t i = 0; i < n; ++i) {
      sb.seg[i] = segs[s0 + i];
      sb.out[i] = out[s0 + i];
      span = std::max<int64_t>(span, std::max(segs[s0 + i].n_rec, segs[s0 + i].n_roll) + 1);
    }
    pack_kernel<<<dim3(n, unsigned((span + 255) / 256)), 256, 0, stream>>>(sb, n_ch);
    DFX_LAUNCH_CHECK("pack_kernel");
  }
  return DFX_OK;
}

int64_t dfx_reshard_pack_bytes(int64_t n_rec, int64_t n_roll, int32_t n_ch) {
  const int64_t b = 8 * n_rec + 8 * (n_roll + 1) + 8 * int64_t(n_ch) * n_roll + 4 * (n_rec + 1);
  return (b + 15) & ~int64_t(15);
}

}  // extern "C"
