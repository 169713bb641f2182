// synth.cu -- on-device synthetic rollouts.
//
// Same counter-keyed SplitMix64 values as the CPU generator
// (oracle/dfx_oracle.h, following fill_channel distflow/functions.hpp:95-104
// and the token-counter convention :52-54), bit-exact: integer hashing plus
// f64 arithmetic with explicit round-to-nearest intrinsics (no FMA
// contraction), rounded to f32 once.
#include "common.cuh"

namespace dfx {

struct SynthParams {
  SlotGeom g;
  int64_t n_slots;
  const uint64_t* ids;
  int32_t n_roll;
  uint64_t dom[7];  // hash_str(seed, domain): tok_lp, tok_old, tok_ref, tok_value, tok_id, tok_mask, reward
  float *lp, *old_lp, *ref_lp, *value_tok, *token_reward;
  uint8_t* mask;
  int32_t* token_id;
};

__global__ void __launch_bounds__(256) synth_kernel(SynthParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (u >= p.n_slots) return;
  int64_t s, t0, t1;
  if (!slot_unit(p.g, u, lane, s, t0, t1)) return;
  const uint64_t id = __ldg(p.ids + s / p.n_roll);
  const uint64_t j = (uint64_t)(s % p.n_roll);
  const int64_t a = __ldg(p.g.cu + s), L = __ldg(p.g.cu + s + 1) - a;
  uint64_t base[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) base[k] = hash_combine(hash_combine(p.dom[k], id), j);
  const uint64_t pm = hash_combine(hash_combine(p.dom[5], id), j) % (uint64_t)(L / 5 + 1);
  const float rew = (float)unit_from_hash(hash_combine(hash_combine(p.dom[6], id), j));
  for (int64_t t = t0 + lane; t < t1; t += 32) {
    const uint64_t tr = (uint64_t)(t - a);
    const float lp = (float)__dmul_rn(-4.0, unit_from_hash(hash_combine(base[0], tr)));
    if (p.lp) p.lp[t] = lp;
    if (p.old_lp)
      p.old_lp[t] = (float)__dadd_rn((double)lp, __dmul_rn(0.25, symmetric_from_hash(hash_combine(base[1], tr))));
    if (p.ref_lp)
      p.ref_lp[t] = (float)__dadd_rn((double)lp, __dmul_rn(0.1, symmetric_from_hash(hash_combine(base[2], tr))));
    if (p.value_tok) p.value_tok[t] = (float)symmetric_from_hash(hash_combine(base[3], tr));
    if (p.token_reward) p.token_reward[t] = ((int64_t)tr == L - 1) ? rew : 0.0f;
    if (p.mask) p.mask[t] = tr >= pm ? 1 : 0;
    if (p.token_id) p.token_id[t] = (int32_t)(hash_combine(base[4], tr) % 151936ull);
  }
}

// fn_generate (distflow/functions.hpp:108-123) on the device: the rollout token counts (draw_tokens,
// functions.hpp:67-80, + SKEWED) and the rollout payloads hash_bytes(keyed_hash(seed, "payload", id, r),
// token_count * bytes_per_token) (hash.hpp:48-59): byte i of a payload is byte i % 8 of splitmix64(key + i / 8).
__global__ void __launch_bounds__(256) gen_counts_kernel(uint64_t dom, const uint64_t* __restrict__ ids, int64_t S,
                                                         int32_t n_roll, int kind, uint32_t value, uint32_t mn,
                                                         uint32_t mx, uint32_t* __restrict__ out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  if (kind == 0) {  // CONSTANT
    out[s] = value;
    return;
  }
  const uint64_t h = hash_combine(hash_combine(dom, __ldg(ids + s / n_roll)), (uint64_t)(s % n_roll));
  const uint64_t span = (uint64_t)mx - mn + 1;
  if (kind == 1) {  // UNIFORM
    out[s] = mn + (uint32_t)(h % span);
  } else {  // SKEWED: min + floor(span * prod / 2^63), prod the product of three 21-bit fields (< 2^63)
    const uint64_t prod = (h & 0x1FFFFFull) * ((h >> 21) & 0x1FFFFFull) * ((h >> 42) & 0x1FFFFFull);
    const uint64_t lo = span * prod, hi = __umul64hi(span, prod);
    out[s] = mn + (uint32_t)((hi << 1) | (lo >> 63));
  }
}

// warp per rollout; lane l writes the 8-byte blocks l, l + 32, ... (byte stores: payloads start at any offset)
__global__ void __launch_bounds__(256) gen_payload_kernel(uint64_t dom, const uint64_t* __restrict__ ids, int64_t S,
                                                          int32_t n_roll, const int64_t* __restrict__ off,
                                                          uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= S) return;
  const int64_t o0 = __ldg(off + s), n = __ldg(off + s + 1) - o0;
  const uint64_t key = hash_combine(hash_combine(dom, __ldg(ids + s / n_roll)), (uint64_t)(s % n_roll));
  uint8_t* dst = out + o0;
  for (int64_t c = lane; 8 * c < n; c += 32) {
    const uint64_t blk = splitmix64(key + (uint64_t)c);
    const int nb = (int)min((int64_t)8, n - 8 * c);
    for (int b = 0; b < nb; ++b) dst[8 * c + b] = (uint8_t)(blk >> (8 * b));
  }
}

// host-side reference hash_str (distflow/hash.hpp:25-29) for the domain bases
static uint64_t h_splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t h_hash_str(uint64_t seed, const char* s) {
  uint64_t h = seed;
  for (const unsigned char* q = (const unsigned char*)s; *q; ++q)
    h = h_splitmix(h ^ (uint64_t(*q) + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2)));
  return h;
}

}  // namespace dfx

using namespace dfx;

extern "C" dfx_status dfx_synth_tokens(uint64_t seed, const uint64_t* ids, int64_t n_records, int32_t n_roll,
                                       const int64_t* cu_seqlens, int64_t token_base, int64_t token_span,
                                       float* lp, float* old_lp, float* ref_lp, float* value_tok,
                                       float* token_reward, uint8_t* mask, int32_t* token_id, dfx_stream stream) {
  if (!ids || !cu_seqlens || n_roll < 1) return fail(DFX_INVALID_ARGUMENT, "dfx_synth_tokens: bad arguments");
  const int64_t S = n_records * n_roll;
  if (S <= 0) return DFX_OK;
  SynthParams p{};
  p.g.cu = cu_seqlens;
  p.g.n_seq = S;
  p.g.base = token_base & ~int64_t(3);
  p.g.sh = 11;
  p.n_slots = slot_count(S, token_span, p.g.sh);
  p.ids = ids;
  p.n_roll = n_roll;
  const char* doms[7] = {"tok_lp", "tok_old", "tok_ref", "tok_value", "tok_id", "tok_mask", "reward"};
  for (int k = 0; k < 7; ++k) p.dom[k] = h_hash_str(seed, doms[k]);
  p.lp = lp;
  p.old_lp = old_lp;
  p.ref_lp = ref_lp;
  p.value_tok = value_tok;
  p.token_reward = token_reward;
  p.mask = mask;
  p.token_id = token_id;
  synth_kernel<<<(unsigned)((p.n_slots + 7) / 8), 256, 0, stream>>>(p);
  DFX_LAUNCH_CHECK("synth_kernel");
  return DFX_OK;
}

extern "C" dfx_status dfx_generate_counts(uint64_t seed, int32_t kind, uint32_t value, uint32_t min_tokens,
                                          uint32_t max_tokens, const uint64_t* ids, int64_t n_records, int32_t n_roll,
                                          uint32_t* tok_count, dfx_stream stream) {
  if (n_roll < 1) return fail(DFX_INVALID_ARGUMENT, "rollouts_per_prompt must be >= 1");
  if (kind < 0 || kind > 2 || !ids || !tok_count) return fail(DFX_INVALID_ARGUMENT, "dfx_generate_counts: bad argument");
  if (kind != 0 && max_tokens < min_tokens) return fail(DFX_INVALID_ARGUMENT, "token distribution max < min");
  const int64_t S = n_records * n_roll;
  if (S <= 0) return DFX_OK;
  gen_counts_kernel<<<(unsigned)((S + 255) / 256), 256, 0, stream>>>(h_hash_str(seed, "gen_tokens"), ids, S, n_roll,
                                                                      kind, value, min_tokens, max_tokens, tok_count);
  DFX_LAUNCH_CHECK("gen_counts_kernel");
  return DFX_OK;
}

extern "C" dfx_status dfx_generate_payload(uint64_t seed, const uint64_t* ids, int64_t n_records, int32_t n_roll,
                                           const int64_t* payload_off, uint8_t* payload, dfx_stream stream) {
  if (n_roll < 1 || !ids || !payload_off || !payload)
    return fail(DFX_INVALID_ARGUMENT, "dfx_generate_payload: bad argument");
  const int64_t S = n_records * n_roll;
  if (S <= 0) return DFX_OK;
  gen_payload_kernel<<<(unsigned)((S + 7) / 8), 256, 0, stream>>>(h_hash_str(seed, "payload"), ids, S, n_roll,
                                                                   payload_off, payload);
  DFX_LAUNCH_CHECK("gen_payload_kernel");
  return DFX_OK;
}
