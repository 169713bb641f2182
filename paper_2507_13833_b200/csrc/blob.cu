// blob.cu -- the reference's record wire format on the device.
//
// serialize_records (distflow/record.hpp:109-127, 151-156) of a packed batch, written by the GPU straight from the
// SoA token streams into the little-endian blob that CPU peers (Fabric, BufferStore::exchange) read:
//   u32 n_records; per record: u64 sample_id | meta section (u32 count + (str, str)*) | u32 n_rollouts;
//   per rollout: u32 token_count | u64 payload_len | payload | u32 n_channels | (u32 len, name, f64 bits)*
// The payload of rollout s is the concatenation, stream by stream, of its tokens' elements (token_id
// i32 | lp f32 | old f32 | ref f32 | mask u8). Record offsets come from a host plan (dfx_serialize_plan: every size
// is known from the host copies of group_off / cu), so every rollout finds its offset in O(1) and one CTA per
// rollout writes its header, payload and channels in parallel. Payload bytes land at arbitrary byte offsets: the
// interior is written as aligned 32-bit words assembled with funnel shifts from aligned source words, the
// (at most two) partial words at either end byte by byte, so neighbouring writers never share a store.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace dfx {

constexpr int kBlobMaxStreams = 8;
constexpr int kBlobMaxCh = 8;
constexpr int kBlobMaxName = 48;

struct BlobParams {
  int64_t n_records, n_rollouts;
  const uint64_t* ids;
  const int32_t* group_off;
  const int32_t* roll_group;  // nullable: the record of each rollout (else a binary search over group_off)
  const int64_t* cu;
  const uint32_t* tok_count;  // nullable: cu[s+1] - cu[s]
  int n_streams;
  const uint8_t* streams[kBlobMaxStreams];
  uint32_t esz[kBlobMaxStreams];
  uint32_t E;                 // sum of esz
  int n_ch;
  const double* ch[kBlobMaxCh];
  uint32_t name_len[kBlobMaxCh];
  char names[kBlobMaxCh][kBlobMaxName];
  uint32_t CH;                // bytes of one rollout's channel entries
  const uint8_t* meta;        // nullable: per-record pre-serialized meta sections
  const int64_t* meta_off;
  const int64_t* rec_off;     // [n_records + 1] blob offset of each record (after the leading u32)
  uint8_t* out;
};

__device__ __forceinline__ void put_le(uint8_t* p, uint64_t v, int n) {
#pragma unroll 8
  for (int i = 0; i < n; ++i) p[i] = uint8_t(v >> (8 * i));
}

// Copy n bytes src -> dst (any alignment) with the block's threads. The 16-byte-aligned interior of dst is written
// with 128-bit stores, each assembled from five aligned 32-bit source words with funnel shifts; the bytes before
// and after it byte by byte (they may share a word with a neighbouring writer).
__device__ __forceinline__ void block_copy(uint8_t* dst, const uint8_t* src, uint64_t n, uint32_t tid,
                                           uint32_t nthr) {
  if (n == 0) return;
  const uintptr_t d0 = reinterpret_cast<uintptr_t>(dst), d1 = d0 + n;
  const uintptr_t a0 = (d0 + 15) & ~uintptr_t(15), a1 = d1 & ~uintptr_t(15);
  if (a1 <= a0) {  // no whole aligned 16-byte unit
    for (uint64_t i = tid; i < n; i += nthr) dst[i] = src[i];
    return;
  }
  const uint64_t head = a0 - d0, tail = d1 - a1;
  if (tid < head) dst[tid] = src[tid];
  if (tid < tail) dst[n - tail + tid] = src[n - tail + tid];
  // unit u covers source bytes [head + 16u, head + 16u + 16)
  const uintptr_t sa = reinterpret_cast<uintptr_t>(src + head);
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(sa & ~uintptr_t(3));
  const uint32_t sh = uint32_t(sa & 3u) * 8u;
  uint4* dv = reinterpret_cast<uint4*>(a0);
  const uint64_t nu = (a1 - a0) / 16;
  // four units per thread in flight (all loads issued before the first store)
  constexpr int kU = 4;
  uint64_t u = tid;
  for (; u + (kU - 1) * nthr < nu; u += kU * nthr) {
    uint32_t w[kU][5];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const uint32_t* q = sw + 4 * (u + j * nthr);
      w[j][0] = __ldg(q);
      w[j][1] = __ldg(q + 1);
      w[j][2] = __ldg(q + 2);
      w[j][3] = __ldg(q + 3);
      w[j][4] = sh ? __ldg(q + 4) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kU; ++j)
      dv[u + j * nthr] = make_uint4(__funnelshift_r(w[j][0], w[j][1], sh), __funnelshift_r(w[j][1], w[j][2], sh),
                                          __funnelshift_r(w[j][2], w[j][3], sh), __funnelshift_r(w[j][3], w[j][4], sh));
  }
  for (; u < nu; u += nthr) {
    const uint32_t* q = sw + 4 * u;
    const uint32_t w0 = __ldg(q), w1 = __ldg(q + 1), w2 = __ldg(q + 2), w3 = __ldg(q + 3);
    const uint32_t w4 = sh ? __ldg(q + 4) : 0u;
    dv[u] = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                       __funnelshift_r(w3, w4, sh));
  }
}

__global__ void __launch_bounds__(256) serialize_kernel(BlobParams p) {
  const int64_t b = blockIdx.x;
  if (b == 0 && threadIdx.x == 0) put_le(p.out, uint64_t(p.n_records), 4);
  // record header of record b (every record, including ones without rollouts)
  if (b < p.n_records) {
    uint8_t* o = p.out + 4 + p.rec_off[b];
    const int32_t g0 = p.group_off[b], g1 = p.group_off[b + 1];
    int64_t mlen = 4;
    if (p.meta) {
      mlen = p.meta_off[b + 1] - p.meta_off[b];
      block_copy(o + 8, p.meta + p.meta_off[b], uint64_t(mlen), threadIdx.x, blockDim.x);
    }
    if (threadIdx.x == 0) {
      put_le(o, p.ids[b], 8);
      if (!p.meta) put_le(o + 8, 0, 4);
      put_le(o + 8 + mlen, uint64_t(g1 - g0), 4);
    }
  }
  if (b >= p.n_rollouts) return;
  // rollout b: its record by a binary search over group_off, then its offset in O(1)
  __shared__ int64_t s_rec;
  if (threadIdx.x == 0) {
    if (p.roll_group) {
      s_rec = p.roll_group[b];
    } else {
      int64_t lo = 0, hi = p.n_records;  // last record with group_off[r] <= b
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (p.group_off[mid] <= b) lo = mid;
        else hi = mid;
      }
      while (lo + 1 < p.n_records && p.group_off[lo + 1] <= b) ++lo;  // skip empty records
      s_rec = lo;
    }
  }
  __syncthreads();
  const int64_t r = s_rec;
  const int32_t g0 = p.group_off[r];
  const int64_t mlen = p.meta ? p.meta_off[r + 1] - p.meta_off[r] : 4;
  const int64_t t0 = p.cu[b], t1 = p.cu[b + 1], L = t1 - t0;
  // record header: u64 id + meta section + u32 n_rollouts = 12 + mlen; each rollout: 16 + payload + channels
  const uint64_t off = uint64_t(p.rec_off[r]) + 12 + uint64_t(mlen) + uint64_t(b - g0) * (16u + p.CH) +
                       uint64_t(t0 - p.cu[g0]) * p.E;
  uint8_t* o = p.out + 4 + off;
  const uint64_t plen = uint64_t(L) * p.E;
  if (threadIdx.x == 0) {
    put_le(o, p.tok_count ? p.tok_count[b] : uint32_t(L), 4);
    put_le(o + 4, plen, 8);
  }
  // the streams are copied concurrently: warp w copies stream w % n_streams (with the other warps of that stream),
  // so the rollout's loads are in flight together instead of one stream after the other
  if (p.n_streams > 0) {
    const int ns = p.n_streams, w = int(threadIdx.x >> 5), nw = int(blockDim.x >> 5);
    const int k = w % ns, cnt = (nw - k + ns - 1) / ns;
    uint64_t po = 12;
    for (int j = 0; j < k; ++j) po += uint64_t(L) * p.esz[j];
    block_copy(o + po, p.streams[k] + uint64_t(t0) * p.esz[k], uint64_t(L) * p.esz[k],
               uint32_t(w / ns) * 32u + (threadIdx.x & 31u), uint32_t(cnt) * 32u);
  }
  uint8_t* c = o + 12 + plen;
  if (threadIdx.x == 0) put_le(c, uint64_t(p.n_ch), 4);
  uint64_t co = 4;
  for (int k = 0; k < p.n_ch; ++k) {
    const uint32_t nl = p.name_len[k];
    if (threadIdx.x == 0) put_le(c + co, nl, 4);
    for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) c[co + 4 + i] = uint8_t(p.names[k][i]);
    if (threadIdx.x == 0) put_le(c + co + 4 + nl, uint64_t(__double_as_longlong(p.ch[k][b])), 8);
    co += 12 + nl;
  }
}

}  // namespace dfx

using namespace dfx;

extern "C" {

int64_t dfx_serialize_plan(int64_t n_records, const int32_t* h_group_off, const int64_t* h_cu,
                           const int64_t* h_meta_off, int32_t n_streams, const uint32_t* esz, int32_t n_ch,
                           const char* const* ch_names, int64_t* rec_off) {
  if (n_records < 0 || !h_group_off || (n_records > 0 && !h_cu) || !rec_off) {
    set_error("dfx_serialize_plan: bad argument");
    return -DFX_INVALID_ARGUMENT;
  }
  uint64_t E = 0, CH = 0;
  for (int32_t k = 0; k < n_streams; ++k) E += esz[k];
  for (int32_t c = 0; c < n_ch; ++c) CH += 12 + std::strlen(ch_names[c]);
  int64_t o = 0;
  for (int64_t r = 0; r < n_records; ++r) {
    rec_off[r] = o;
    const int32_t g0 = h_group_off[r], g1 = h_group_off[r + 1];
    const int64_t meta = h_meta_off ? h_meta_off[r + 1] - h_meta_off[r] : 4;
    o += 12 + meta + int64_t(g1 - g0) * int64_t(16 + CH) + (h_cu[g1] - h_cu[g0]) * int64_t(E);
  }
  rec_off[n_records] = o;
  return 4 + o;  // leading u32 record count
}

dfx_status dfx_serialize_records(const dfx_packed* b, const uint64_t* ids, const uint32_t* tok_count, int32_t n_streams,
                                 const void* const* streams, const uint32_t* esz, int32_t n_ch,
                                 const char* const* ch_names, const double* const* ch, const uint8_t* meta_blob,
                                 const int64_t* meta_off, const int64_t* rec_off, uint8_t* out, dfx_stream stream) {
  if (!b || !ids || !out || !rec_off || n_streams < 0 || n_streams > kBlobMaxStreams || n_ch < 0 || n_ch > kBlobMaxCh ||
      (n_streams && (!streams || !esz)) || (n_ch && (!ch_names || !ch)) || (meta_blob && !meta_off))
    return fail(DFX_INVALID_ARGUMENT, "dfx_serialize_records: bad argument");
  if (b->n_records > 0 && (!b->group_off || !b->cu_seqlens))
    return fail(DFX_INVALID_ARGUMENT, "dfx_serialize_records: packed batch lacks group_off/cu_seqlens");
  BlobParams p{};
  p.n_records = b->n_records;
  p.n_rollouts = b->n_rollouts;
  p.ids = ids;
  p.group_off = b->group_off;
  p.roll_group = b->roll_group;
  p.cu = b->cu_seqlens;
  p.tok_count = tok_count;
  p.n_streams = n_streams;
  for (int k = 0; k < n_streams; ++k) {
    p.streams[k] = static_cast<const uint8_t*>(streams[k]);
    p.esz[k] = esz[k];
    p.E += esz[k];
  }
  p.n_ch = n_ch;
  for (int k = 0; k < n_ch; ++k) {
    const size_t nl = std::strlen(ch_names[k]);
    if (nl >= size_t(kBlobMaxName)) return fail(DFX_INVALID_ARGUMENT, "dfx_serialize_records: channel name too long");
    std::memcpy(p.names[k], ch_names[k], nl);
    p.name_len[k] = uint32_t(nl);
    p.ch[k] = ch[k];
    p.CH += 12 + uint32_t(nl);
  }
  p.meta = meta_blob;
  p.meta_off = meta_off;
  p.rec_off = rec_off;
  p.out = out;
  const int64_t grid = std::max<int64_t>(std::max<int64_t>(p.n_records, p.n_rollouts), 1);
  serialize_kernel<<<(unsigned)grid, 256, 0, stream>>>(p);
  DFX_LAUNCH_CHECK("serialize_kernel");
  return DFX_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------------------------
// deserialize_records (record.hpp:129-149, 158-165) into a packed batch: the CPU walks the headers (an index of
// record ids, rollout token counts and the byte offsets of every payload and channel block -- a sequential parse,
// microseconds per thousand rollouts), the GPU gathers the payload bytes into the SoA token streams and the f64
// channels (one CTA per rollout, unaligned source reads assembled with funnel shifts).
// ---------------------------------------------------------------------------------------------------------------
namespace dfx {

struct UnblobParams {
  int64_t n_rollouts;
  const uint8_t* blob;
  const int64_t* payload_off;  // [S]
  const int64_t* ch_off;       // [S] offset of the f64 of channel 0 entry block (after u32 n_channels)
  const int64_t* cu;           // [S+1] destination token offsets
  int n_streams;
  uint8_t* streams[kBlobMaxStreams];
  uint32_t esz[kBlobMaxStreams];
  int n_ch;
  uint32_t ch_val_off[kBlobMaxCh];  // byte offset of channel c's f64 within the channel block
  double* ch[kBlobMaxCh];
};

// 4-byte-aligned dst: 32-bit stores assembled by funnel shifts from aligned source words; else copy_shift16
__device__ __forceinline__ void block_gather(uint8_t* dst, const uint8_t* src, uint64_t n) {
  const uintptr_t sa = reinterpret_cast<uintptr_t>(src);
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(sa & ~uintptr_t(3));
  const uint32_t sh = uint32_t(sa & 3u) * 8u;
  const uint64_t nw = n / 4;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst);
  if (reinterpret_cast<uintptr_t>(dst) & 3u) {  // (byte streams at an odd token offset)
    copy_shift16<false>(dst, src, n, threadIdx.x, blockDim.x);
    return;
  }
  for (uint64_t w = threadIdx.x; w < nw; w += blockDim.x)
    dw[w] = sh ? __funnelshift_r(__ldg(sw + w), __ldg(sw + w + 1), sh) : __ldg(sw + w);
  for (uint64_t i = nw * 4 + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

__global__ void __launch_bounds__(256) unblob_kernel(UnblobParams p) {
  const int64_t s = blockIdx.x;
  if (s >= p.n_rollouts) return;
  const int64_t t0 = p.cu[s], L = p.cu[s + 1] - t0;
  const uint8_t* src = p.blob + p.payload_off[s];
  for (int k = 0; k < p.n_streams; ++k) {
    block_gather(p.streams[k] + uint64_t(t0) * p.esz[k], src, uint64_t(L) * p.esz[k]);
    src += uint64_t(L) * p.esz[k];
  }
  if (threadIdx.x < p.n_ch) {
    const uint8_t* v = p.blob + p.ch_off[s] + p.ch_val_off[threadIdx.x];
    uint64_t bits = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) bits |= uint64_t(v[i]) << (8 * i);
    p.ch[threadIdx.x][s] = __longlong_as_double((long long)bits);
  }
}

}  // namespace dfx

extern "C" {

// Host-side header walk of a record blob. First call with every output NULL returns counts in *n_records /
// *n_rollouts / *n_tokens (and checks the format); the second fills the arrays. Every rollout must carry the
// channels ch_names (in blob order, i.e. sorted) and a payload of token_count * bytes_per_token bytes.
dfx_status dfx_blob_index(const uint8_t* blob, uint64_t size, uint32_t bytes_per_token, int32_t n_ch,
                          const char* const* ch_names, int64_t* n_records, int64_t* n_rollouts, int64_t* n_tokens,
                          uint64_t* ids, int64_t* meta_range, int32_t* group_off, int64_t* cu, uint32_t* tok_count,
                          int64_t* payload_off, int64_t* ch_off) {
  if (!blob || !n_records || !n_rollouts || !n_tokens) return fail(DFX_INVALID_ARGUMENT, "dfx_blob_index: null argument");
  uint64_t pos = 0;
  auto need = [&](uint64_t n) {
    if (pos + n > size) throw std::string("record blob truncated");  // blob::Reader::need (record.hpp:99-101)
  };
  auto u32 = [&]() {
    need(4);
    uint32_t v = uint32_t(blob[pos]) | uint32_t(blob[pos + 1]) << 8 | uint32_t(blob[pos + 2]) << 16 |
                 uint32_t(blob[pos + 3]) << 24;
    pos += 4;
    return v;
  };
  auto u64 = [&]() {
    const uint64_t lo = u32();
    return lo | uint64_t(u32()) << 32;
  };
  try {
    const uint32_t R = u32();
    int64_t S = 0, T = 0;
    if (group_off) group_off[0] = 0;
    if (cu) cu[0] = 0;
    for (uint32_t r = 0; r < R; ++r) {
      const uint64_t id = u64();
      if (ids) ids[r] = id;
      if (meta_range) meta_range[2 * r] = int64_t(pos);
      const uint32_t nmeta = u32();
      for (uint32_t m = 0; m < 2 * nmeta; ++m) {
        const uint32_t n = u32();
        need(n);
        pos += n;
      }
      if (meta_range) meta_range[2 * r + 1] = int64_t(pos);
      const uint32_t nroll = u32();
      for (uint32_t j = 0; j < nroll; ++j, ++S) {
        const uint32_t tc = u32();
        const uint64_t plen = u64();
        if (bytes_per_token == 0 || plen % bytes_per_token)
          throw std::string("payload of rollout " + std::to_string(S) + " is not a whole number of tokens");
        const int64_t L = int64_t(plen / bytes_per_token);
        need(plen);
        if (payload_off) payload_off[S] = int64_t(pos);
        if (tok_count) tok_count[S] = tc;
        pos += plen;
        T += L;
        if (cu) cu[S + 1] = T;
        const uint32_t nch = u32();
        if (int32_t(nch) != n_ch) throw std::string("rollout " + std::to_string(S) + " has a different channel set");
        if (ch_off) ch_off[S] = int64_t(pos);
        for (uint32_t c = 0; c < nch; ++c) {
          const uint32_t nl = u32();
          need(nl);
          if (ch_names && (std::strlen(ch_names[c]) != nl || std::memcmp(blob + pos, ch_names[c], nl) != 0))
            throw std::string("rollout " + std::to_string(S) + " channel " + std::to_string(c) + " is not '" +
                              ch_names[c] + "'");
          pos += nl;
          need(8);
          pos += 8;
        }
      }
      if (group_off) group_off[r + 1] = int32_t(S);
    }
    if (pos != size) throw std::string("trailing bytes after the last record");
    *n_records = R;
    *n_rollouts = S;
    *n_tokens = T;
  } catch (const std::string& e) {
    return fail(DFX_ERROR, "dfx_blob_index: " + e);  // distflow::ParseError
  }
  return DFX_OK;
}

// Gather payloads and channels of an indexed blob (device copy of the blob, device copies of the index arrays)
// into the token streams (element k of rollout s at streams[k] + (cu[s] + i) * esz[k]) and f64 channels.
dfx_status dfx_blob_unpack(const uint8_t* blob, int64_t n_rollouts, const int64_t* cu, const int64_t* payload_off,
                           const int64_t* ch_off, int32_t n_streams, void* const* streams, const uint32_t* esz,
                           int32_t n_ch, const char* const* ch_names, double* const* ch, dfx_stream stream) {
  if (n_rollouts <= 0) return DFX_OK;
  if (!blob || !cu || !payload_off || n_streams < 0 || n_streams > kBlobMaxStreams || n_ch < 0 || n_ch > kBlobMaxCh ||
      (n_ch && (!ch_off || !ch || !ch_names)))
    return fail(DFX_INVALID_ARGUMENT, "dfx_blob_unpack: bad argument");
  UnblobParams p{};
  p.n_rollouts = n_rollouts;
  p.blob = blob;
  p.payload_off = payload_off;
  p.ch_off = ch_off;
  p.cu = cu;
  p.n_streams = n_streams;
  for (int k = 0; k < n_streams; ++k) {
    p.streams[k] = static_cast<uint8_t*>(streams[k]);
    p.esz[k] = esz[k];
  }
  p.n_ch = n_ch;
  uint32_t o = 0;
  for (int c = 0; c < n_ch; ++c) {
    const uint32_t nl = uint32_t(std::strlen(ch_names[c]));
    p.ch_val_off[c] = o + 4 + nl;
    p.ch[c] = ch[c];
    o += 12 + nl;
  }
  unblob_kernel<<<(unsigned)n_rollouts, 256, 0, stream>>>(p);
  DFX_LAUNCH_CHECK("unblob_kernel");
  return DFX_OK;
}

}  // extern "C"
