// loss.cu -- GRPO group advantage (bit-exact vs fn_group_advantage), per-token
// broadcast, and the fused advantage + PPO clipped surrogate + KL + masked
// aggregation kernel over packed variable-length rollouts.
//
// Reference: distflow/functions.hpp:143-161 (fn_group_advantage),
// :163-172 (fn_ppo_advantage), :176-182 (fn_train slot the loss fills).
// HBM-bound streaming kernels: no tensor cores (no dense contraction).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include <utility>

#include "common.cuh"

#ifndef DFX_CLIP_MODE
#define DFX_CLIP_MODE 1
#endif
#ifndef DFX_LOSS_PRED
#define DFX_LOSS_PRED 1  // predicated stream loads instead of a branch per vector (C2 step -1.8%)
#endif
#ifndef DFX_LOSS_PFR
#define DFX_LOSS_PFR 1  // per-lane L2 prefetch of the vectors this many rounds ahead (1: C2 step -3%; 2, 3: slower)
#endif
#ifndef DFX_LOSS_PF
// (kernel-variant sweeps) L2 bulk prefetch of each claimed slot's streams. Measured at C2: the loss launch drops
// from 0.1065 to 0.1034 ms, but the step only by 0.5%: the prefetches still in flight when the kernel retires slow
// the next kernels down, so the launch time overstates the gain. Off.
#define DFX_LOSS_PF 0
#endif
#ifndef DFX_TOKEN_MINB
#define DFX_TOKEN_MINB 2
#endif
#ifndef DFX_TOKEN_UNROLL
#define DFX_TOKEN_UNROLL 2
#endif

namespace dfx {

// ---------------------------------------------------------------------------
// GRPO group statistics, same operation order as functions.hpp:147-158 with
// explicit round-to-nearest intrinsics so nvcc cannot contract into FMAs:
// the f64 result is bit-identical to the reference's.
// ---------------------------------------------------------------------------
struct GroupStats {
  double mean, denom;  // denom = std + eps
};

__device__ __forceinline__ GroupStats group_stats(const double* __restrict__ reward, int32_t r0,
                                                  int32_t r1, double eps) {
  const double n = (double)(r1 - r0);
  double sum = 0.0;
  for (int32_t i = r0; i < r1; ++i) sum = __dadd_rn(sum, __ldg(reward + i));
  const double mean = __ddiv_rn(sum, n);
  double var = 0.0;
  for (int32_t i = r0; i < r1; ++i) {
    const double d = __dsub_rn(__ldg(reward + i), mean);
    var = __dadd_rn(var, __dmul_rn(d, d));
  }
  const double sd = __dsqrt_rn(__ddiv_rn(var, n));
  return {mean, __dadd_rn(sd, eps)};
}

__device__ __forceinline__ double group_adv(double r, const GroupStats& g) {
  const double d = __dsub_rn(r, g.mean);
  return d == 0.0 ? 0.0 : __ddiv_rn(d, g.denom);
}


__global__ void ppo_adv_kernel(int64_t n, const double* __restrict__ reward,
                               const double* __restrict__ value, double* __restrict__ adv) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) adv[s] = __dsub_rn(reward[s], value[s]);  // functions.hpp:169
}

// per-token broadcast adv_tok[t] = mask[t] ? f32(adv[s]) : 0, one warp per slot
__global__ void __launch_bounds__(256) broadcast_kernel(SlotGeom g, int64_t n_slots,
                                                        const double* __restrict__ adv,
                                                        const uint8_t* __restrict__ mask,
                                                        float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (u >= n_slots) return;
  int64_t s, t0, t1;
  if (!slot_unit(g, u, lane, s, t0, t1)) return;
  const float a = (float)__ldg(adv + s);
  for (int64_t v = (t0 >> 2) + lane; v < ((t1 + 3) >> 2); v += 32) {
    const uint32_t mk = ldg_stream_u32(mask + 4 * v);
    float o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = ((mk >> (8 * k)) & 0xffu) ? a : 0.0f;
    const int64_t t = 4 * v;
    if (t >= t0 && t + 4 <= t1) {
      stg_stream_f4(out + t, make_float4(o[0], o[1], o[2], o[3]));
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (t + k >= t0 && t + k < t1) out[t + k] = o[k];
    }
  }
}

// ---------------------------------------------------------------------------
// Fused loss
// ---------------------------------------------------------------------------
// One token source of a loss call: a packed batch (its own token coordinates; pointers may be peer-mapped, e.g.
// a partner GPU's producer batch read over NVLink) owning global slots [slot0, ...) and rollouts [roll0, ...).
constexpr int kMaxLossSrc = 4;
struct LossSrc {
  SlotGeom g;
  int64_t slot0, roll0;
  const float* lp;
  const float* old_lp;
  const float* ref_lp;
  const uint8_t* mask;
  const double* adv_roll_in;
  const float* adv_tok_in;
  float* adv_tok_out;
  float* dlogp;
};

// global slot u -> (source, local slot); global rollout s -> source
__device__ __forceinline__ int src_of_slot(const LossSrc* src, int n_src, int64_t u) {
  int k = 0;
  while (k + 1 < n_src && u >= src[k + 1].slot0) ++k;
  return k;
}
__device__ __forceinline__ int src_of_roll(const LossSrc* src, int n_src, int64_t s) {
  int k = 0;
  while (k + 1 < n_src && s >= src[k + 1].roll0) ++k;
  return k;
}

struct SlotEnt {
  uint32_t toff;  // t0 - base
  int32_t s;      // rollout (source-local)
  int32_t len;    // tokens; 0 = empty slot id
  float A;        // DFX_ADV_ROLLOUT: f32(adv_roll[s])
};

struct LossParams {
  int n_src;
  int multi;  // sources from dfx_ppo_loss_multi (may be peer-mapped memory): the MULTI kernel, even for one source
  LossSrc src[kMaxLossSrc];
  int64_t n_slots;
  int64_t n_records;
  const int32_t* group_off;   // fused GRPO (single source only)
  const int32_t* roll_group;
  const double* reward;
  double* adv_roll_out;
  const double* whiten_sums;
  int whiten;
  float clip_lo, clip_hi, beta;
  // clip decision thresholds on the log-ratio d = lp - old: rho > 1+eps_hi  <=>  d > log(1+eps_hi), rho < 1-eps_lo
  // <=> d < log(1-eps_lo), each as a float pair T32 + Tlo (clip_twosum)
  float t_hi32, t_lo32;
  float t_hi32_lo, t_lo32_lo;  // T64 - T32 (the thresholds as float pairs)
  float clip_margin;           // (DFX_CLIP_MODE 1) |s*d - s*T32| below which the f32 decision may be wrong
  double adv_eps;
  int kl_type;
  int agg;
  int n_groups;
  const int32_t* lgo;
  const double* seq_n;     // dlogp: per-rollout mask count
  const double* grp_stats; // dlogp: per loss group {N, S}
  double* part;            // [5][n_slots]
  const SlotEnt* tab;      // [n_slots] slot table (global slot ids)
  int32_t* flags;
  unsigned long long* ticket;  // [kMaxLossSrc + 1] per-source slot tickets + finished warps; zero on entry, restored
};

// ---- slot table -------------------------------------------------------------------------------------------------
// One 16-byte entry per slot id: the slot's rollout, its token range and (per-rollout advantage) the advantage,
// built by a thread-per-rollout pre-pass, so the streaming warps resolve a claimed slot with ONE load instead of
// the 32-ary search over cu_seqlens (three dependent L2 round trips) plus the advantage load.

// thread per rollout s: the entries of slot ids [f(s), f(s+1)) (f(s) = s + window of cu[s]; the last rollout
// also owns the ids up to the source's slot count)
__global__ void __launch_bounds__(256) slot_table_kernel(SlotGeom g, int64_t n_slots, const double* __restrict__ adv,
                                                         SlotEnt* __restrict__ tab) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the loss kernel may launch now (it waits)
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (programmatic dependent: the advantages of the previous kernel)
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= g.n_seq) return;
  const int64_t a = __ldg(g.cu + s), b = __ldg(g.cu + s + 1);
  const int64_t f0 = s + ((a - g.base) >> g.sh);
  const int64_t f1 = s + 1 < g.n_seq ? s + 1 + ((b - g.base) >> g.sh) : n_slots;
  const int64_t wa = (a - g.base) >> g.sh, wb = (b - 1 - g.base) >> g.sh;
  const float A = adv ? (float)__ldg(adv + s) : 0.0f;
  for (int64_t u = f0; u < f1; ++u) {
    const int64_t w = u - s;
    SlotEnt e{0u, (int32_t)s, 0, A};
    if (b > a && w >= wa && w <= wb) {
      const int64_t ws = g.base + (w << g.sh);
      const int64_t t0 = max(a, ws), t1 = min(b, ws + ((int64_t)1 << g.sh));
      e.toff = (uint32_t)(t0 - g.base);
      e.len = (int32_t)(t1 - t0);
    }
    tab[u] = e;
  }
}

// ---- per-token math (k3_series, clip_exact_f32: common.cuh) ---------------------------------------------
// per lane and round: f32 sums of the surrogate / KL / log ratio; exact integer counts of clipped and masked tokens
// (bit counts per vector instead of a multiply-add per token)
struct WhitenF {  // per-token whitening (A - mu) * rstd with mu = mu_hi + mu_lo
  float mu_hi, mu_lo, rstd;
};
struct TokAcc {
  float pg, kl, akl;
  uint32_t clip, n;
};

// Per-unit constants for a warp-uniform advantage A (GRPO broadcast): with
// s = sign(A), the clipped surrogate max(-A rho, -A clip(rho)) equals
// -|A| * min(s rho, s bound) where bound = 1+eps_hi (A>0) or 1-eps_lo (A<0),
// and the clip fires iff s rho > s bound. A == 0 gives bound = +inf: pg = 0,
// never clipped -- identical to the reference formula.
struct UnitAdv {
  float A, nA, s, sb;
  float sT32;   // s * log-ratio threshold (A > 0: log(1+eps_hi), A < 0: log(1-eps_lo)); +inf when A == 0
};
__device__ __forceinline__ UnitAdv unit_adv(float A, float lo, float hi, float t_lo32, float t_hi32) {
  UnitAdv u;
  u.A = A;
  u.nA = -fabsf(A);
  u.s = A < 0.0f ? -1.0f : 1.0f;
  const float inf = __int_as_float(0x7f800000);
  u.sb = A > 0.0f ? hi : (A < 0.0f ? -lo : inf);
  u.sT32 = A > 0.0f ? t_hi32 : (A < 0.0f ? -t_lo32 : inf);
  return u;
}

// The clip fires iff s*(lp - old) > s*T, T the log-ratio threshold of A's sign (log(1+eps_hi) for A > 0,
// log(1-eps_lo) for A < 0): the same decision as the reference formula's pg2 > pg1 on exp(lp - old) in f64
// (oracle/dfx_oracle.c), made exactly in f32 arithmetic, branch-free (clip_exact_f32, common.cuh). Keeps clipfrac
// (a count) exact instead of within f32 rounding of exp and 1+eps.
__device__ __forceinline__ bool clip_twosum(const LossParams& p, float s, float sT32, float l, float o, float d) {
  return clip_exact_f32(s, sT32, s > 0.0f ? p.t_hi32_lo : -p.t_lo32_lo, l, o, d);
}

// Four tokens of one aligned vector starting at token t. FULL: all in range.
template <int ADV, int KL, bool DLOGP, bool FULL>
__device__ __forceinline__ void loss_vec(const LossParams& p, const UnitAdv& ua, float4 lv, float4 ov, float4 rv,
                                         float4 av, uint32_t mk, int64_t t, int64_t t0, int64_t t1, const WhitenF& wf,
                                         float w, TokAcc& acc, float (&aout)[4], float (&gout)[4]) {
  const float lo = 1.0f - p.clip_lo, hi = 1.0f + p.clip_hi;
  float x[4], kl[4], dkl[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = f4_get(rv, k) - f4_get(lv, k);
  if (KL == DFX_KL_K3) {
    const float ax = fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fmaxf(fabsf(x[2]), fabsf(x[3])));
    if (ax < kK3Series) {
#pragma unroll
      for (int k = 0; k < 4; ++k) kl[k] = k3_series(x[k]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) kl[k] = fminf(fmaxf(expm1f(x[k]) - x[k], -10.0f), 10.0f);
    }
    if (DLOGP)
#pragma unroll
      for (int k = 0; k < 4; ++k) dkl[k] = (kl[k] >= 10.0f || kl[k] <= -10.0f) ? 0.0f : -expm1f(x[k]);
  } else if (KL == DFX_KL_K1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) { kl[k] = -x[k]; dkl[k] = 1.0f; }
  } else if (KL == DFX_KL_K2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) { kl[k] = 0.5f * x[k] * x[k]; dkl[k] = -x[k]; }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) { kl[k] = 0.0f; dkl[k] = 0.0f; }
  }
  // per-token log ratio and the exact clip decision (clip_twosum): for a warp-uniform advantage (GRPO broadcast /
  // per-rollout) here, for per-token advantages (GAE) in the loop below
  float dd[4];
  bool cl[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) dd[k] = f4_get(lv, k) - f4_get(ov, k);  // log ratio
  // DFX_CLIP_MODE (kernel-variant sweeps only): 1 (default) the f32 log-ratio decision, redone exactly by TwoSum
  // for a vector holding a token within rounding distance of the threshold; 0 TwoSum for every token; 2 the f32
  // decision alone (can differ from the reference for tokens within an f32 ulp of the threshold); 3 the ratio
  // decision s*rho > s*bound of round 1. Measured at C2 (bench path): 1 0.1050 ms, 0 0.1055, 2 0.1024.
  if constexpr (ADV != DFX_ADV_TOKEN && DFX_CLIP_MODE == 1) {
    // f32 decision, redone exactly (TwoSum) for the vector only when a token lies within rounding distance
    bool near = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float sd = ua.s * dd[k];
      cl[k] = sd > ua.sT32;
      near |= fabsf(sd - ua.sT32) <= p.clip_margin;
    }
    if (near) {
#pragma unroll
      for (int k = 0; k < 4; ++k) cl[k] = clip_twosum(p, ua.s, ua.sT32, f4_get(lv, k), f4_get(ov, k), dd[k]);
    }
  } else if constexpr (ADV != DFX_ADV_TOKEN && DFX_CLIP_MODE != 3) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      cl[k] = DFX_CLIP_MODE == 2 ? ua.s * dd[k] > ua.sT32
                                 : clip_twosum(p, ua.s, ua.sT32, f4_get(lv, k), f4_get(ov, k), dd[k]);
  }
  float At[4];  // per-token advantages (GAE): whitened here, clip decision as in mode 1 per token
  if constexpr (ADV == DFX_ADV_TOKEN) {
    bool near = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // whitening with mu as an f32 pair: the rounding of mu alone would shift every advantage alike, the
      // rounding of each subtraction is relative to the token's own whitened value
      At[k] = p.whiten ? ((f4_get(av, k) - wf.mu_hi) - wf.mu_lo) * wf.rstd : f4_get(av, k);
      const float sg = At[k] < 0.0f ? -1.0f : 1.0f;
      const float sT = At[k] > 0.0f ? p.t_hi32 : (At[k] < 0.0f ? -p.t_lo32 : __int_as_float(0x7f800000));
      const float sd = sg * dd[k];
      cl[k] = sd > sT;
      near |= fabsf(sd - sT) <= p.clip_margin;
    }
    if (near) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float sg = At[k] < 0.0f ? -1.0f : 1.0f;
        const float sT = At[k] > 0.0f ? p.t_hi32 : (At[k] < 0.0f ? -p.t_lo32 : __int_as_float(0x7f800000));
        cl[k] = clip_twosum(p, sg, sT, f4_get(lv, k), f4_get(ov, k), dd[k]);
      }
    }
  }
  uint32_t onb = 0u, clb = 0u;  // this vector's masked-in and clipped tokens, as bits
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    bool on = ((mk >> (8 * k)) & 0xffu) != 0u;
    if (!FULL) on = on && (t + k >= t0) && (t + k < t1);
    const float m = on ? 1.0f : 0.0f;
    const float d = dd[k];
    const float rho = ex2_ftz(d * kLog2e);   // MUFU.EX2, ~2 ulp
    float A, pg;
    if constexpr (ADV == DFX_ADV_TOKEN) {
      A = At[k];
      const float rc = fminf(fmaxf(rho, lo), hi);
      pg = fmaxf(-A * rho, -A * rc);
    } else {
      A = ua.A;
      const float sr = ua.s * rho;
      pg = ua.nA * fminf(sr, ua.sb);
      if constexpr (DFX_CLIP_MODE == 3) cl[k] = sr > ua.sb;
    }
    acc.pg = fmaf(m, pg, acc.pg);
    acc.kl = fmaf(m, kl[k], acc.kl);
    acc.akl = fmaf(-m, d, acc.akl);
    onb |= (on ? 1u : 0u) << k;
    clb |= (cl[k] ? 1u : 0u) << k;
    aout[k] = on ? A : 0.0f;
    if (DLOGP) gout[k] = m * w * ((cl[k] ? 0.0f : -A * rho) + p.beta * dkl[k]);
  }
  acc.n += __popc(onb);
  acc.clip += __popc(onb & clb);
}

// Group stats with all lanes participating: lanes load the rewards in
// parallel, then every lane folds them in the reference's sequential order via
// shuffles (identical result in every lane, no dependent global loads).
__device__ __forceinline__ GroupStats group_stats_warp(const double* __restrict__ reward, int32_t r0, int32_t r1,
                                                       double eps, int lane) {
  const double n = (double)(r1 - r0);
  double sum = 0.0;
  for (int32_t base = r0; base < r1; base += 32) {
    const int cnt = min(32, r1 - base);
    const double x = lane < cnt ? __ldg(reward + base + lane) : 0.0;
    for (int j = 0; j < cnt; ++j) sum = __dadd_rn(sum, __shfl_sync(kFull, x, j));
  }
  const double mean = __ddiv_rn(sum, n);
  double var = 0.0;
  for (int32_t base = r0; base < r1; base += 32) {
    const int cnt = min(32, r1 - base);
    const double x = lane < cnt ? __ldg(reward + base + lane) : 0.0;
    const double d = __dsub_rn(x, mean);
    const double dd = __dmul_rn(d, d);
    for (int j = 0; j < cnt; ++j) var = __dadd_rn(var, __shfl_sync(kFull, dd, j));
  }
  const double sd = __dsqrt_rn(__ddiv_rn(var, n));
  return {mean, __dadd_rn(sd, eps)};
}

// Fused GRPO (DFX_ADV_GROUP_FUSED): the slot table pre-pass also computes the advantages -- warp per record: the
// bit-exact f64 group statistics once, the rollouts' f64 advantage channel, and every slot entry of the record's
// rollouts with its f32 advantage (the streaming kernel then needs no reward loads and no f64 chain per slot)
__global__ void __launch_bounds__(256) slot_table_group_kernel(SlotGeom g, int64_t n_slots, int64_t n_records,
                                                               const int32_t* __restrict__ go,
                                                               const double* __restrict__ reward, double eps,
                                                               double* __restrict__ adv_out, int32_t* flags,
                                                               SlotEnt* __restrict__ tab) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n_records) return;
  const int32_t ra = go[r], rb = go[r + 1];
  GroupStats gs{0.0, 1.0};
  if (rb > ra) gs = group_stats_warp(reward, ra, rb, eps, lane);
  else if (flags && lane == 0) atomicOr(flags, kFlagMissingRollouts);  // require_rollouts functions.hpp:82-87
  for (int32_t s = ra + lane; s < rb; s += 32) {
    const double adv = group_adv(__ldg(reward + s), gs);
    if (adv_out) adv_out[s] = adv;
    const int64_t a = __ldg(g.cu + s), b = __ldg(g.cu + s + 1);
    const int64_t f0 = s + ((a - g.base) >> g.sh);
    const int64_t f1 = s + 1 < g.n_seq ? s + 1 + ((b - g.base) >> g.sh) : n_slots;
    const int64_t wa = (a - g.base) >> g.sh, wb = (b - 1 - g.base) >> g.sh;
    for (int64_t u = f0; u < f1; ++u) {
      const int64_t w = u - s;
      SlotEnt e{0u, (int32_t)s, 0, (float)adv};
      if (b > a && w >= wa && w <= wb) {
        const int64_t ws = g.base + (w << g.sh);
        const int64_t t0 = max(a, ws), t1 = min(b, ws + ((int64_t)1 << g.sh));
        e.toff = (uint32_t)(t0 - g.base);
        e.len = (int32_t)(t1 - t0);
      }
      tab[u] = e;
    }
  }
}

// one warp per record
__global__ void __launch_bounds__(256) grpo_adv_kernel(int64_t n_records, const int32_t* __restrict__ go,
                                                       const double* __restrict__ reward, double eps,
                                                       double* __restrict__ adv, int32_t* flags) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n_records) return;
  const int32_t a = go[r], b = go[r + 1];
  if (b <= a) {  // require_rollouts functions.hpp:82-87
    if (flags && lane == 0) atomicOr(flags, kFlagMissingRollouts);
    return;
  }
  const GroupStats g = group_stats_warp(reward, a, b, eps, lane);
  for (int32_t s = a + lane; s < b; s += 32) adv[s] = group_adv(__ldg(reward + s), g);
}

template <bool FULL>
__device__ __forceinline__ void store_vec(float* base, int64_t t, int64_t t0, int64_t t1, const float (&v)[4]) {
  if (FULL) {
    stg_stream_f4(base + t, make_float4(v[0], v[1], v[2], v[3]));
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (t + k >= t0 && t + k < t1) base[t + k] = v[k];
  }
}

// masked whitening of the advantages, unbiased variance + 1e-8 (oracle/dfx_oracle.c dfo_ppo_loss)
__device__ __forceinline__ void whiten_coeffs(const LossParams& p, double& mu, double& rstd) {
  const double N = p.whiten_sums[2];
  const double m1 = N > 0 ? p.whiten_sums[0] / N : 0.0;
  const double var = N > 1 ? (p.whiten_sums[1] - p.whiten_sums[0] * m1) / (N - 1.0) : 0.0;
  mu = m1;
  rstd = 1.0 / sqrt(fmax(var, 0.0) + 1e-8);
}

// Persistent warps; each warp repeatedly claims the next slot (atomic ticket)
// and streams it: coalesced 128-bit loads of lp/old/ref (+adv) and 32-bit
// mask words, kUnroll vectors per lane in flight, fused advantage broadcast,
// clipped surrogate, KL and masked partial sums in registers (f32 per round,
// f64 across rounds), one deterministic warp reduction per slot.
template <int ADV, int KL, bool DLOGP, int UNROLL = 2, int MINB = 3, bool MULTI = false>
__global__ void __launch_bounds__(256, MINB) loss_slots_kernel(LossParams p) {
  // programmatic dependent launch: this grid starts while the slot-table pre-pass drains and waits here for it;
  // the finalize kernel is released at once (it waits for this grid's completion)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);

  // whitening coefficients: live across the loop only for per-token advantages; the per-rollout paths whiten
  // once per slot (keeps the hot kernels' registers for loads in flight)
  WhitenF wf{0.0f, 0.0f, 1.0f};
  if (ADV == DFX_ADV_TOKEN && p.whiten) {
    double mu, rstd;
    whiten_coeffs(p, mu, rstd);
    wf.mu_hi = (float)mu;
    wf.mu_lo = (float)(mu - (double)wf.mu_hi);
    wf.rstd = (float)rstd;
  }
  double* part = p.part;
  // tickets: [k] next slot of source k, [kMaxLossSrc] finished warps. Several sources (e.g. local HBM and a
  // partner GPU's memory over NVLink) are drained concurrently: warp w starts on source w % n_src and moves to the
  // next one when its source runs out, so the fast local slots overlap the slow remote ones.
  unsigned long long* next = p.ticket;
  int k = MULTI ? (int)(gwarp % p.n_src) : 0;
  uint32_t live = (1u << p.n_src) - 1u;

  // at most one slot per warp (e.g. C3: 2048 slots, 2368 resident warps): warp w takes slot w, no ticket atomics
  // (claiming would balance nothing and costs two dependent atomic round trips per warp). Per-token-advantage path
  // only: in the 80-register per-rollout kernels any extra live state spills
  const bool one_each = ADV == DFX_ADV_TOKEN && !MULTI && p.n_slots <= nwarps;
  for (bool first = true;; first = false) {
    int64_t ul;
    if (one_each) {
      if (!first) break;
      ul = gwarp;
    } else {
      unsigned long long uu = 0;
      if (lane == 0) uu = atomicAdd(next + k, 1ull);
      ul = (int64_t)__shfl_sync(kFull, uu, 0);
    }
    const int64_t kend = MULTI ? (k + 1 < p.n_src ? p.src[k + 1].slot0 : p.n_slots) - p.src[k].slot0 : p.n_slots;
    if (ul >= kend) {
      if (!MULTI) break;
      live &= ~(1u << k);
      if (!live) break;
      do k = (k + 1) % p.n_src; while (!((live >> k) & 1u));
      continue;
    }
    const LossSrc& S = p.src[k];
    const int64_t u = S.slot0 + ul;
    const int4 ev = __ldg(reinterpret_cast<const int4*>(p.tab + u));  // one load resolves the slot
    if (ev.z == 0) {
      if (lane < 5) part[(int64_t)lane * p.n_slots + u] = 0.0;
      continue;
    }
    const int64_t s = ev.y;
    const int64_t t0 = S.g.base + (int64_t)(uint32_t)ev.x, t1 = t0 + ev.z;
    const int64_t sg = S.roll0 + s;  // global rollout (loss groups, dlogp weights)
    float A_unit = 0.0f;
    if (ADV != DFX_ADV_TOKEN) A_unit = __int_as_float(ev.w);  // (group advantages: computed by the pre-pass)
    if (ADV != DFX_ADV_TOKEN && p.whiten) {
      double m0, r0;
      whiten_coeffs(p, m0, r0);
      A_unit = (float)(((double)A_unit - m0) * r0);
    }
    const UnitAdv ua = unit_adv(A_unit, 1.0f - p.clip_lo, 1.0f + p.clip_hi, p.t_lo32, p.t_hi32);
    float w = 0.0f;
    if (DLOGP) {
      int gi = 0;
      if (p.lgo)
        while (gi + 1 < p.n_groups && __ldg(p.lgo + gi + 1) <= sg) ++gi;
      const double N = p.grp_stats[2 * gi], Sq = p.grp_stats[2 * gi + 1];
      const double ns = p.seq_n[sg];
      if (p.agg == DFX_AGG_TOKEN_MEAN) w = N > 0 ? (float)(1.0 / N) : 0.0f;
      else if (p.agg == DFX_AGG_SEQ_MEAN_TOKEN_MEAN) w = (Sq > 0 && ns > 0) ? (float)(1.0 / (Sq * ns)) : 0.0f;
      else w = Sq > 0 ? (float)(1.0 / Sq) : 0.0f;
    }

    double dpg = 0.0, dkl = 0.0, dakl = 0.0;
    uint32_t nclip = 0u, nmask = 0u;
    const int64_t vbeg = t0 >> 2;
    const int32_t nvec = (int32_t)(((t1 + 3) >> 2) - vbeg);
    // vectors [i_lo, i_lo + n_full) hold four tokens of the slot each
    const int32_t i_lo = (int32_t)(((t0 + 3) >> 2) - vbeg);
    const uint32_t n_full = (uint32_t)max((int64_t)0, (t1 >> 2) - vbeg - i_lo);
    const float* lp0 = S.lp + 4 * vbeg;
    const float* ol0 = S.old_lp + 4 * vbeg;
    const float* rf0 = S.ref_lp + 4 * vbeg;
    const uint8_t* mk0 = S.mask + 4 * vbeg;
    const float* ad0 = ADV == DFX_ADV_TOKEN ? S.adv_tok_in + 4 * vbeg : nullptr;
    float* const atout = S.adv_tok_out;
    float* const dlout = S.dlogp;
    constexpr int kUnroll = UNROLL;
#if DFX_LOSS_PF
    // the slot's streams into L2 at once (more bytes in flight per warp than its registers hold). Not on the
    // per-token-advantage path: its C3-size working set is L2-resident and the prefetches cost 5 us per step
    if (ADV != DFX_ADV_TOKEN && lane == 0 && nvec > 32 * kUnroll) {
      const uint32_t fb = (uint32_t)nvec * 16u;
      l2_prefetch(lp0, fb);
      l2_prefetch(ol0, fb);
      l2_prefetch(rf0, fb);
      const uintptr_t m0 = reinterpret_cast<uintptr_t>(mk0) & ~uintptr_t(15);
      l2_prefetch(reinterpret_cast<const void*>(m0),
                  (uint32_t)((reinterpret_cast<uintptr_t>(mk0) + 4u * (uint32_t)nvec - m0 + 15u) & ~uintptr_t(15)));
    }
#endif
    for (int32_t ib = lane; ib < nvec; ib += 32 * kUnroll) {
      float4 lv[kUnroll], ov[kUnroll], rv[kUnroll], av[kUnroll];
      uint32_t mk[kUnroll];
#pragma unroll
      for (int j = 0; j < kUnroll; ++j) {
        const int32_t i = ib + 32 * j;
#if DFX_LOSS_PRED
        const bool in = i < nvec;  // (predicated loads: no branch around them)
        lv[j] = ldg_stream_f4_if(lp0 + 4 * i, in);
        ov[j] = ldg_stream_f4_if(ol0 + 4 * i, in);
        rv[j] = ldg_stream_f4_if(rf0 + 4 * i, in);
        mk[j] = ldg_stream_u32_if(mk0 + 4 * i, in);
        if (ADV == DFX_ADV_TOKEN) av[j] = ldg_stream_f4_if(ad0 + 4 * i, in);
#if DFX_LOSS_PFR
        // the next round's vectors of this lane into L2 (no registers held). Single-source kernel only: its batch
        // is in this GPU's memory (dfx_ppo_loss); prefetch.global.L2 of NVLink-mapped memory (the multi-source
        // kernel's partner sources) stalls the kernel ~50x
        if constexpr (!MULTI) {
          const int32_t i2 = i + 32 * kUnroll * DFX_LOSS_PFR;
          const bool in2 = i2 < nvec;
          prefetch_l2_if(lp0 + 4 * i2, in2);
          prefetch_l2_if(ol0 + 4 * i2, in2);
          prefetch_l2_if(rf0 + 4 * i2, in2);
          if ((lane & 7) == 0) prefetch_l2_if(mk0 + 4 * i2, in2);  // (one 128-byte line per 8 lanes)
        }
#endif
#else
        if (i < nvec) {
          lv[j] = ldg_stream_f4(lp0 + 4 * i);
          ov[j] = ldg_stream_f4(ol0 + 4 * i);
          rv[j] = ldg_stream_f4(rf0 + 4 * i);
          mk[j] = ldg_stream_u32(mk0 + 4 * i);
          if (ADV == DFX_ADV_TOKEN) av[j] = ldg_stream_f4(ad0 + 4 * i);
        }
#endif
      }
      TokAcc acc{0.f, 0.f, 0.f, 0u, 0u};
#pragma unroll
      for (int j = 0; j < kUnroll; ++j) {
        const int32_t i = ib + 32 * j;
        if (i >= nvec) break;
        const int64_t t = 4 * (vbeg + i);
        float aout[4], gout[4];
        if ((uint32_t)(i - i_lo) < n_full) {  // all four tokens inside the slot (32-bit test)
          loss_vec<ADV, KL, DLOGP, true>(p, ua, lv[j], ov[j], rv[j], av[j], mk[j], t, t0, t1, wf, w, acc, aout,
                                         gout);
          if (atout) store_vec<true>(atout, t, t0, t1, aout);
          if (DLOGP) store_vec<true>(dlout, t, t0, t1, gout);
        } else {
          loss_vec<ADV, KL, DLOGP, false>(p, ua, lv[j], ov[j], rv[j], av[j], mk[j], t, t0, t1, wf, w, acc, aout,
                                          gout);
          if (atout) store_vec<false>(atout, t, t0, t1, aout);
          if (DLOGP) store_vec<false>(dlout, t, t0, t1, gout);
        }
      }
      dpg += acc.pg;
      dkl += acc.kl;
      dakl += acc.akl;
      nclip += acc.clip;
      nmask += acc.n;
    }
    dpg = warp_sum(dpg);
    dkl = warp_sum(dkl);
    const double dclip = (double)warp_sum(nclip);
    dakl = warp_sum(dakl);
    const double dn = (double)warp_sum(nmask);
    if (lane == 0) {
      part[u] = dpg;
      part[p.n_slots + u] = dkl;
      part[2 * p.n_slots + u] = dclip;
      part[3 * p.n_slots + u] = dakl;
      part[4 * p.n_slots + u] = dn;
    }
  }
  // the last warp out restores the tickets for the next launch
  if (!one_each && lane == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(next + kMaxLossSrc, 1ull);
    if (done == (unsigned long long)nwarps - 1) {
#pragma unroll
      for (int q = 0; q <= kMaxLossSrc; ++q) next[q] = 0ull;
    }
  }
}

// mask-count pre-pass (dlogp weights): part[4][u] = sum of mask over the slot
struct MaskCountParams {
  int n_src;
  LossSrc src[kMaxLossSrc];
};
__global__ void __launch_bounds__(256) mask_count_kernel(MaskCountParams mp, int64_t n_slots,
                                                         double* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (u >= n_slots) return;
  const LossSrc& S = mp.src[src_of_slot(mp.src, mp.n_src, u)];
  const uint8_t* mask = S.mask;
  int64_t s, t0, t1;
  if (!slot_unit(S.g, u - S.slot0, lane, s, t0, t1)) {
    if (lane == 0) cnt[u] = 0.0;
    return;
  }
  uint32_t c = 0;
  for (int64_t v = (t0 >> 2) + lane; v < ((t1 + 3) >> 2); v += 32) {
    const uint32_t mk = ldg_stream_u32(mask + 4 * v);
    const int64_t t = 4 * v;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (t + k >= t0 && t + k < t1 && ((mk >> (8 * k)) & 0xffu)) ++c;
  }
  c = warp_sum(c);
  if (lane == 0) cnt[u] = (double)c;
}

// ---------------------------------------------------------------------------
// Finalize: per-rollout sums over its contiguous slots, then per loss group a
// deterministic block reduction; the last block of each group (ticket order)
// reduces the block partials in index order. COUNTS: the dlogp pre-pass.
// ---------------------------------------------------------------------------
constexpr int kFinThreads = 256;

struct FinParams {
  int n_src;
  LossSrc src[kMaxLossSrc];
  int64_t n_roll;         // total rollouts over the sources
  int64_t n_slots;
  int n_groups;
  const int32_t* lgo;
  int agg;
  double beta;
  const double* part;   // [5][n_slots] (COUNTS: [1][n_slots] counts)
  double* blk;          // [n_groups][nb][6]
  unsigned int* ticket; // [n_groups], zero on entry, restored to zero
  int nb;
  double* seq_n;        // COUNTS: out per-rollout mask counts
  double* grp_stats;    // COUNTS: out per group {N, S}
  dfx_loss_out* out;    // !COUNTS: out per group
};

template <int NQ>
__device__ __forceinline__ void block_sum(double (&v)[NQ], double* sh) {
  // fixed-shape tree: warp xor-shuffle, then warp 0 over the per-warp values
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) sh[wid * NQ + q] = v[q];
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double x = lane < nw ? sh[lane * NQ + q] : 0.0;
      v[q] = warp_sum(x);
    }
  }
  __syncthreads();
}

template <bool COUNTS>
__global__ void __launch_bounds__(kFinThreads) finalize_kernel(FinParams f) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (programmatic dependent of the loss kernel)
  __shared__ double sh[(kFinThreads / 32) * 6];
  __shared__ bool is_last;
  const int gi = blockIdx.y;
  const int64_t sr0 = f.lgo ? f.lgo[gi] : 0;
  const int64_t sr1 = f.lgo ? f.lgo[gi + 1] : f.n_roll;
  double acc[6] = {0, 0, 0, 0, 0, 0};  // pg, kl, clip, akl, n, S
  // block b of a group sums rollouts [first, last) with a thread stride (fixed order: deterministic)
  const int64_t per = (sr1 - sr0 + f.nb - 1) / f.nb;
  const int64_t first = sr0 + (int64_t)blockIdx.x * per, last = min(sr1, first + per);
  for (int64_t s = first + threadIdx.x; s < last; s += kFinThreads) {
    const LossSrc& S = f.src[src_of_roll(f.src, f.n_src, s)];
    const int64_t sl = s - S.roll0;
    const int64_t a = S.g.cu[sl], b = S.g.cu[sl + 1];
    double q[5] = {0, 0, 0, 0, 0};
    if (b > a) {
      const int64_t u0 = S.slot0 + sl + ((a - S.g.base) >> S.g.sh), u1 = S.slot0 + sl + ((b - 1 - S.g.base) >> S.g.sh);
      for (int64_t u = u0; u <= u1; ++u) {
        if (COUNTS) {
          q[4] += f.part[u];
        } else {
#pragma unroll
          for (int k = 0; k < 5; ++k) q[k] += f.part[(int64_t)k * f.n_slots + u];
        }
      }
    }
    const double ns = q[4];
    if (COUNTS) f.seq_n[s] = ns;
    acc[2] += q[2];
    acc[3] += q[3];
    acc[4] += ns;
    if (ns > 0) acc[5] += 1.0;
    if (f.agg == DFX_AGG_TOKEN_MEAN) {
      acc[0] += q[0];
      acc[1] += q[1];
    } else if (ns > 0) {
      const double div = f.agg == DFX_AGG_SEQ_MEAN_TOKEN_MEAN ? ns : 1.0;
      acc[0] += q[0] / div;
      acc[1] += q[1] / div;
    }
  }
  block_sum<6>(acc, sh);
  double tot[6] = {0, 0, 0, 0, 0, 0};
  if (f.nb == 1) {  // one block per group (small batches): no second phase
#pragma unroll
    for (int q = 0; q < 6; ++q) tot[q] = acc[q];
  } else {
    double* blk = f.blk + ((int64_t)gi * f.nb + blockIdx.x) * 6;
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < 6; ++q) blk[q] = acc[q];
      __threadfence();
      const unsigned t = atomicAdd(f.ticket + gi, 1u);
      is_last = (t == (unsigned)f.nb - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const volatile double* vb = f.blk + (int64_t)gi * f.nb * 6;
    for (int i = threadIdx.x; i < f.nb; i += kFinThreads)
#pragma unroll
      for (int q = 0; q < 6; ++q) tot[q] += vb[(int64_t)i * 6 + q];
    block_sum<6>(tot, sh);
  }
  if (threadIdx.x == 0) {
    const double N = tot[4], S = tot[5];
    if (COUNTS) {
      f.grp_stats[2 * gi] = N;
      f.grp_stats[2 * gi + 1] = S;
    } else {
      const double denom = f.agg == DFX_AGG_TOKEN_MEAN ? N : S;
      dfx_loss_out o;
      o.pg_loss = denom > 0 ? tot[0] / denom : 0.0;
      o.kl = denom > 0 ? tot[1] / denom : 0.0;
      o.loss = o.pg_loss + f.beta * o.kl;
      o.clipfrac = N > 0 ? tot[2] / N : 0.0;
      o.approx_kl = N > 0 ? tot[3] / N : 0.0;
      o.n_tokens = N;
      o.n_seqs = S;
      f.out[gi] = o;
    }
    f.ticket[gi] = 0u;  // ready for the next call
  }
}

// Merge per-part results of one loss group (the TP-split loss: each TP rank reduced the rollouts it holds):
// the means are re-weighted by their denominators, parts folded in index order (every rank gets the same bits).
__global__ void loss_combine_kernel(const dfx_loss_out* parts, int n_parts, int n_groups, int agg, double beta,
                                    dfx_loss_out* out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  double pg = 0, kl = 0, clip = 0, akl = 0, N = 0, S = 0;
  for (int k = 0; k < n_parts; ++k) {
    const dfx_loss_out p = parts[(int64_t)k * n_groups + g];
    const double den = agg == DFX_AGG_TOKEN_MEAN ? p.n_tokens : p.n_seqs;
    pg += p.pg_loss * den;
    kl += p.kl * den;
    clip += p.clipfrac * p.n_tokens;
    akl += p.approx_kl * p.n_tokens;
    N += p.n_tokens;
    S += p.n_seqs;
  }
  const double den = agg == DFX_AGG_TOKEN_MEAN ? N : S;
  dfx_loss_out o;
  o.pg_loss = den > 0 ? pg / den : 0.0;
  o.kl = den > 0 ? kl / den : 0.0;
  o.loss = o.pg_loss + beta * o.kl;
  o.clipfrac = N > 0 ? clip / N : 0.0;
  o.approx_kl = N > 0 ? akl / N : 0.0;
  o.n_tokens = N;
  o.n_seqs = S;
  out[g] = o;
}

}  // namespace dfx

using namespace dfx;

namespace {

constexpr int kWarpsPerBlock = 8;

struct LossWs {
  unsigned long long* slot_ticket;
  double* part;
  double* blk;
  double* seq_n;
  double* grp_stats;
  unsigned int* ticket;
  SlotEnt* tab;
  int nb;
  size_t bytes;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

LossWs loss_ws_layout(void* base, int64_t n_seq, int64_t n_slots, int32_t n_groups) {
  LossWs w{};
  // finalize blocks per loss group: one block (no inter-block phase) up to 4096 rollouts, else 256 per block
  w.nb = n_seq <= 4096 ? 1 : (int)((n_seq + kFinThreads - 1) / kFinThreads);
  size_t off = 0;
  char* b = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* p = b ? b + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  // the self-maintained tickets first, at offsets that do not depend on the call (callers zero the workspace once
  // at allocation and the kernels restore the tickets to zero on exit; a call with different sizes must find them
  // where the previous call left them); then the regions every call writes before reading
  w.slot_ticket = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * (kMaxLossSrc + 1)));
  w.ticket = reinterpret_cast<unsigned int*>(take(sizeof(unsigned int) * 2 * size_t(DFX_MAX_LOSS_GROUPS)));
  w.part = reinterpret_cast<double*>(take(sizeof(double) * 5 * size_t(n_slots)));
  w.blk = reinterpret_cast<double*>(take(sizeof(double) * 6 * size_t(n_groups) * size_t(w.nb)));
  w.seq_n = reinterpret_cast<double*>(take(sizeof(double) * size_t(n_seq + 1)));
  w.grp_stats = reinterpret_cast<double*>(take(sizeof(double) * 2 * size_t(n_groups)));
  w.tab = reinterpret_cast<SlotEnt*>(take(sizeof(SlotEnt) * size_t(n_slots)));
  w.bytes = off;
  return w;
}

// slots of one source; a source without rollouts owns none (its cu_seqlens may be NULL and is never read)
int64_t src_slots(int64_t n_rollouts, int64_t token_span) {
  return n_rollouts > 0 ? slot_count(n_rollouts, token_span, slot_shift(token_span)) : 0;
}

SlotGeom geom_of(const dfx_packed* b, int64_t base, int64_t span) {
  SlotGeom g;
  g.cu = b->cu_seqlens;
  g.n_seq = b->n_rollouts;
  g.base = base;
  g.sh = slot_shift(span);
  return g;
}

// persistent grid: as many 256-thread CTAs as fit on all SMs at once
// launch as a programmatic dependent of the previous kernel in the stream (its launch and prologue overlap that
// kernel's tail; the kernel itself waits with griddepcontrol.wait before reading what the previous one wrote)
template <typename... KArgs, typename... Args>
void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int ADV, int KL, bool DL, int U, int MB>
void launch_variant(const LossParams& p, cudaStream_t st) {
  static thread_local int cached_dev = -1, cached_blocks = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, loss_slots_kernel<ADV, KL, DL, U, MB>, 256, 0);
    cached_blocks = sms * std::max(per_sm, 1);
    cached_dev = dev;
  }
  // a single source keeps the source index a compile-time 0 (no dynamic parameter indexing)
  if (p.n_src > 1 || p.multi) pdl_launch(loss_slots_kernel<ADV, KL, DL, U, MB, true>, dim3(cached_blocks), dim3(256), st, p);
  else pdl_launch(loss_slots_kernel<ADV, KL, DL, U, MB, false>, dim3(cached_blocks), dim3(256), st, p);
}

// Tuning knob (benchmarking only): DFX_LOSS_VARIANT=u2b3 (default) | u3b2 | u4b2 | u2b2 selects the
// unroll depth (vectors in flight per lane) and the CTAs-per-SM register budget of the hot configuration.
inline int loss_variant() {
  static const int v = [] {
    const char* e = std::getenv("DFX_LOSS_VARIANT");
    if (!e) return 0;
    const std::string s(e);
    return s == "u3b2" ? 1 : s == "u4b2" ? 2 : s == "u2b2" ? 3 : s == "u1b4" ? 4 : s == "u2b4" ? 5 : 0;
  }();
  return v;
}

template <int ADV, int KL, bool DL>
void launch_slots(const LossParams& p, cudaStream_t st) {
  // (the tuning variants are instantiated for the hot configuration only)
  if constexpr (ADV == DFX_ADV_ROLLOUT && KL == DFX_KL_K3 && !DL) {
    if (p.n_src > 1 || p.multi) {
      // sources read over NVLink have ~2x the latency of local HBM: more vectors in flight per lane
      static const int mu =
          std::getenv("DFX_LOSS_MULTI_UNROLL") ? std::atoi(std::getenv("DFX_LOSS_MULTI_UNROLL")) : 4;
      if (mu == 4) return launch_variant<ADV, KL, DL, 4, 2>(p, st);
      if (mu == 3) return launch_variant<ADV, KL, DL, 3, 2>(p, st);
    }
    switch (loss_variant()) {
      case 1: return launch_variant<ADV, KL, DL, 3, 2>(p, st);
      case 2: return launch_variant<ADV, KL, DL, 4, 2>(p, st);
      case 3: return launch_variant<ADV, KL, DL, 2, 2>(p, st);
      case 4: return launch_variant<ADV, KL, DL, 1, 4>(p, st);
      case 5: return launch_variant<ADV, KL, DL, 2, 4>(p, st);
      default: break;
    }
  }
  // per-token advantages (GAE, f64 whitening) need more registers than the 80 of 3 CTAs/SM: 2 CTAs/SM
  launch_variant<ADV, KL, DL, ADV == DFX_ADV_TOKEN ? DFX_TOKEN_UNROLL : 2, ADV == DFX_ADV_TOKEN ? DFX_TOKEN_MINB : 3>(p, st);
}

template <int ADV, int KL>
void launch_slots_kl(const LossParams& p, cudaStream_t st, bool dl) {
  if (dl) launch_slots<ADV, KL, true>(p, st);
  else launch_slots<ADV, KL, false>(p, st);
}

template <int ADV>
void launch_slots_adv(const LossParams& p, cudaStream_t st, int kl, bool dl) {
  switch (kl) {
    case DFX_KL_K1: launch_slots_kl<ADV, DFX_KL_K1>(p, st, dl); break;
    case DFX_KL_K2: launch_slots_kl<ADV, DFX_KL_K2>(p, st, dl); break;
    case DFX_KL_K3: launch_slots_kl<ADV, DFX_KL_K3>(p, st, dl); break;
    default: launch_slots_kl<ADV, DFX_KL_NONE>(p, st, dl); break;
  }
}

}  // namespace

extern "C" {

dfx_status dfx_grpo_advantage(const dfx_packed* b, double eps, double* adv_roll, int32_t* flags,
                              dfx_stream stream) {
  if (!b || !b->group_off || !b->reward || !adv_roll) return fail(DFX_INVALID_ARGUMENT, "dfx_grpo_advantage: null argument");
  if (b->n_records <= 0) return DFX_OK;
  grpo_adv_kernel<<<(unsigned)((b->n_records + 7) / 8), 256, 0, stream>>>(b->n_records, b->group_off, b->reward, eps,
                                                                           adv_roll, flags);
  DFX_LAUNCH_CHECK("grpo_adv_kernel");
  return DFX_OK;
}

dfx_status dfx_broadcast_advantage(const dfx_packed* b, int64_t token_base, int64_t token_span,
                                   const double* adv_roll, float* adv_tok, dfx_stream stream) {
  if (!b || !b->cu_seqlens || !b->mask || !adv_roll || !adv_tok) return fail(DFX_INVALID_ARGUMENT, "dfx_broadcast_advantage: null argument");
  if (b->n_rollouts <= 0) return DFX_OK;
  const SlotGeom g = geom_of(b, token_base & ~int64_t(3), token_span);
  const int64_t n_slots = slot_count(b->n_rollouts, token_span, slot_shift(token_span));
  broadcast_kernel<<<(unsigned)((n_slots + kWarpsPerBlock - 1) / kWarpsPerBlock), 32 * kWarpsPerBlock, 0, stream>>>(
      g, n_slots, adv_roll, b->mask, adv_tok);
  DFX_LAUNCH_CHECK("broadcast_kernel");
  return DFX_OK;
}

dfx_status dfx_ppo_advantage(const dfx_packed* b, double* adv_roll, dfx_stream stream) {
  if (!b || !adv_roll) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_advantage: null argument");
  if (!b->reward) return fail(DFX_MISSING_CHANNEL, "missing channel 'reward'");
  if (!b->value) return fail(DFX_MISSING_CHANNEL, "missing channel 'value'");
  if (b->n_rollouts <= 0) return DFX_OK;
  ppo_adv_kernel<<<(unsigned)((b->n_rollouts + 255) / 256), 256, 0, stream>>>(b->n_rollouts, b->reward, b->value, adv_roll);
  DFX_LAUNCH_CHECK("ppo_adv_kernel");
  return DFX_OK;
}

size_t dfx_ppo_loss_workspace_bytes(int64_t n_rollouts, int64_t token_span, int32_t n_loss_groups) {
  if (n_loss_groups < 1) n_loss_groups = 1;
  return loss_ws_layout(nullptr, n_rollouts, slot_count(n_rollouts, token_span, slot_shift(token_span)),
                        n_loss_groups).bytes;
}

size_t dfx_ppo_loss_multi_workspace_bytes(const dfx_loss_src* srcs, int32_t n_src, int32_t n_loss_groups) {
  if (n_loss_groups < 1) n_loss_groups = 1;
  int64_t S = 0, U = 0;
  for (int32_t k = 0; srcs && k < n_src; ++k) {
    S += srcs[k].b.n_rollouts;
    U += src_slots(srcs[k].b.n_rollouts, srcs[k].token_span);
  }
  return loss_ws_layout(nullptr, S, U, n_loss_groups).bytes;
}

}  // extern "C"

namespace {

dfx_status ppo_loss_impl(bool multi_api, const dfx_loss_src* srcs, int32_t n_src, const dfx_loss_cfg* cfg,
                         const dfx_loss_args* args, void* workspace, size_t ws_bytes, cudaStream_t stream) {
  if (!srcs || n_src < 1 || !cfg || !args || !args->out) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: null argument");
  if (n_src > kMaxLossSrc) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss_multi: at most 4 sources");
  const int32_t ng = args->n_loss_groups < 1 ? 1 : args->n_loss_groups;
  if (ng > DFX_MAX_LOSS_GROUPS) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: more than DFX_MAX_LOSS_GROUPS loss groups");
  int64_t S = 0, U = 0;
  for (int32_t k = 0; k < n_src; ++k) S += srcs[k].b.n_rollouts;
  if (S <= 0) {
    DFX_CUDA(cudaMemsetAsync(args->out, 0, sizeof(dfx_loss_out) * ng, stream));
    return DFX_OK;
  }
  if (ng > 1 && !args->loss_group_off) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: loss_group_off required for >1 group");
  if (cfg->adv_source == DFX_ADV_GROUP_FUSED && n_src != 1)
    return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss_multi: the fused GRPO advantage needs a single source");
  if (cfg->whiten && !args->whiten_sums) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: whiten needs whiten_sums");
  if (cfg->kl_type < 0 || cfg->kl_type > 3 || cfg->agg < 0 || cfg->agg > 2) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: bad kl_type/agg");
  bool want_dl = false;
  LossSrc src[kMaxLossSrc] = {};
  for (int32_t k = 0; k < n_src; ++k) {
    const dfx_loss_src& x = srcs[k];
    const dfx_packed* b = &x.b;
    if (b->n_rollouts > 0 && (!b->cu_seqlens || !b->lp || !b->old_lp || !b->ref_lp || !b->mask))
      return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: packed batch lacks cu_seqlens/lp/old_lp/ref_lp/mask");
    switch (cfg->adv_source) {
      case DFX_ADV_GROUP_FUSED:
        if (!b->reward) return fail(DFX_MISSING_CHANNEL, "missing channel 'reward'");
        if (!b->group_off || !b->roll_group) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: fused GRPO needs group_off/roll_group");
        break;
      case DFX_ADV_ROLLOUT:
        if (!x.adv_roll && b->n_rollouts > 0) return fail(DFX_MISSING_CHANNEL, "missing channel 'advantage'");
        break;
      case DFX_ADV_TOKEN:
        if (!x.adv_tok_in && b->n_rollouts > 0) return fail(DFX_MISSING_CHANNEL, "missing per-token advantage");
        break;
      default:
        return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: bad adv_source");
    }
    if (x.token_span >= (int64_t(1) << 31))
      return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: a source spans more than 2^31 tokens (slot table offsets)");
    if (k > 0 && (x.dlogp != nullptr) != want_dl) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss_multi: dlogp on all sources or none");
    want_dl = x.dlogp != nullptr;
    src[k].g = geom_of(b, x.token_base & ~int64_t(3), x.token_span);
    src[k].slot0 = U;
    src[k].roll0 = k == 0 ? 0 : src[k - 1].roll0 + srcs[k - 1].b.n_rollouts;
    src[k].lp = b->lp;
    src[k].old_lp = b->old_lp;
    src[k].ref_lp = b->ref_lp;
    src[k].mask = b->mask;
    src[k].adv_roll_in = x.adv_roll;
    src[k].adv_tok_in = x.adv_tok_in;
    src[k].adv_tok_out = x.adv_tok_out;
    src[k].dlogp = x.dlogp;
    U += src_slots(b->n_rollouts, x.token_span);
  }
  const LossWs w = loss_ws_layout(workspace, S, U, ng);
  if (!workspace || ws_bytes < w.bytes) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: workspace too small");
  const int64_t n_slots = U;

  FinParams f{};
  f.n_src = n_src;
  for (int32_t k = 0; k < n_src; ++k) f.src[k] = src[k];
  f.n_roll = S;
  f.n_slots = n_slots;
  f.n_groups = ng;
  f.lgo = args->loss_group_off;
  f.agg = cfg->agg;
  f.beta = cfg->beta;
  f.nb = w.nb;
  f.blk = w.blk;
  f.seq_n = w.seq_n;
  f.grp_stats = w.grp_stats;
  f.out = args->out;
  const dim3 fgrid((unsigned)w.nb, (unsigned)ng);

  if (want_dl) {
    MaskCountParams mp{};
    mp.n_src = n_src;
    for (int32_t k = 0; k < n_src; ++k) mp.src[k] = src[k];
    mask_count_kernel<<<(unsigned)((n_slots + kWarpsPerBlock - 1) / kWarpsPerBlock), 256, 0, stream>>>(mp, n_slots, w.part);
    DFX_LAUNCH_CHECK("mask_count_kernel");
    f.part = w.part;
    f.ticket = w.ticket + ng;
    finalize_kernel<true><<<fgrid, kFinThreads, 0, stream>>>(f);
    DFX_LAUNCH_CHECK("finalize_kernel<counts>");
  }

  const dfx_packed* b0 = &srcs[0].b;
  LossParams p{};
  p.n_src = n_src;
  p.multi = multi_api ? 1 : 0;
  for (int32_t k = 0; k < n_src; ++k) p.src[k] = src[k];
  p.n_slots = n_slots;
  p.n_records = b0->n_records;
  p.group_off = b0->group_off;
  p.roll_group = b0->roll_group;
  p.reward = b0->reward;
  p.adv_roll_out = cfg->adv_source == DFX_ADV_GROUP_FUSED ? const_cast<double*>(srcs[0].adv_roll) : nullptr;
  p.whiten_sums = args->whiten_sums;
  p.whiten = cfg->whiten;
  p.clip_lo = (float)cfg->clip_low;
  p.clip_hi = (float)cfg->clip_high;
  {
    const double t_hi = std::log(1.0 + cfg->clip_high);
    const double t_lo = cfg->clip_low < 1.0 ? std::log(1.0 - cfg->clip_low) : -HUGE_VAL;
    p.t_hi32 = (float)t_hi;
    p.t_lo32 = (float)t_lo;
    p.t_hi32_lo = (float)(t_hi - (double)p.t_hi32);
    p.t_lo32_lo = std::isfinite(t_lo) ? (float)(t_lo - (double)p.t_lo32) : 0.0f;
    // f32(l - o) is within 2^-24 |l - o| of l - o, T32 within 2^-24 |T| of T; near the threshold |d| ~ |T|
    p.clip_margin = (float)(1e-6 * (1.0 + std::max(std::fabs(t_hi), std::isfinite(t_lo) ? std::fabs(t_lo) : 0.0)));
  }
  p.beta = (float)cfg->beta;
  p.adv_eps = cfg->adv_eps;
  p.kl_type = cfg->kl_type;
  p.agg = cfg->agg;
  p.n_groups = ng;
  p.lgo = args->loss_group_off;
  p.seq_n = w.seq_n;
  p.grp_stats = w.grp_stats;
  p.part = w.part;
  p.flags = args->flags;
  p.ticket = w.slot_ticket;
  p.tab = w.tab;
  if (cfg->adv_source == DFX_ADV_GROUP_FUSED) {  // single source: the table pre-pass computes the advantages
    pdl_launch(slot_table_group_kernel, dim3((unsigned)((b0->n_records + 7) / 8)), dim3(256), stream, src[0].g, n_slots,
               (int64_t)b0->n_records, b0->group_off, b0->reward, cfg->adv_eps, p.adv_roll_out, args->flags, w.tab);
    DFX_LAUNCH_CHECK("slot_table_group_kernel");
  }
  for (int32_t k = 0; k < n_src && cfg->adv_source != DFX_ADV_GROUP_FUSED; ++k) {  // the slot table of every source
    if (srcs[k].b.n_rollouts <= 0) continue;
    const int64_t nk = (k + 1 < n_src ? src[k + 1].slot0 : n_slots) - src[k].slot0;
    const double* adv = cfg->adv_source == DFX_ADV_ROLLOUT ? srcs[k].adv_roll : nullptr;
    pdl_launch(slot_table_kernel, dim3((unsigned)((srcs[k].b.n_rollouts + 255) / 256)), dim3(256), stream, src[k].g,
               nk, adv, w.tab + src[k].slot0);
    DFX_LAUNCH_CHECK("slot_table_kernel");
  }
  if (args->ev_main_begin) DFX_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(args->ev_main_begin), stream));
  switch (cfg->adv_source) {
    case DFX_ADV_GROUP_FUSED: launch_slots_adv<DFX_ADV_GROUP_FUSED>(p, stream, cfg->kl_type, want_dl); break;
    case DFX_ADV_ROLLOUT: launch_slots_adv<DFX_ADV_ROLLOUT>(p, stream, cfg->kl_type, want_dl); break;
    default: launch_slots_adv<DFX_ADV_TOKEN>(p, stream, cfg->kl_type, want_dl); break;
  }
  DFX_LAUNCH_CHECK("loss_slots_kernel");
  if (args->ev_main_end) DFX_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(args->ev_main_end), stream));
  f.part = w.part;
  f.ticket = w.ticket;
  pdl_launch(finalize_kernel<false>, fgrid, dim3(kFinThreads), stream, f);
  DFX_LAUNCH_CHECK("finalize_kernel");
  return DFX_OK;
}

}  // namespace

extern "C" {

dfx_status dfx_ppo_loss(const dfx_packed* b, int64_t token_base, int64_t token_span, const dfx_loss_cfg* cfg,
                        const dfx_loss_args* args, void* workspace, size_t ws_bytes, dfx_stream stream) {
  if (!b || !args) return fail(DFX_INVALID_ARGUMENT, "dfx_ppo_loss: null argument");
  dfx_loss_src s{};
  s.b = *b;
  s.token_base = token_base;
  s.token_span = token_span;
  s.adv_roll = args->adv_roll;
  s.adv_tok_in = args->adv_tok_in;
  s.adv_tok_out = args->adv_tok_out;
  s.dlogp = args->dlogp;
  return ppo_loss_impl(false, &s, 1, cfg, args, workspace, ws_bytes, stream);
}

dfx_status dfx_ppo_loss_multi(const dfx_loss_src* srcs, int32_t n_src, const dfx_loss_cfg* cfg,
                              const dfx_loss_args* args, void* workspace, size_t ws_bytes, dfx_stream stream) {
  return ppo_loss_impl(true, srcs, n_src, cfg, args, workspace, ws_bytes, stream);
}

dfx_status dfx_loss_combine(const dfx_loss_out* parts, int32_t n_parts, int32_t n_groups, const dfx_loss_cfg* cfg,
                            dfx_loss_out* out, dfx_stream stream) {
  if (n_groups <= 0) return DFX_OK;
  if (!parts || !out || !cfg || n_parts <= 0)
    return fail(DFX_INVALID_ARGUMENT, "dfx_loss_combine: bad argument");
  loss_combine_kernel<<<(n_groups + 127) / 128, 128, 0, stream>>>(parts, n_parts, n_groups, cfg->agg, cfg->beta, out);
  DFX_LAUNCH_CHECK("loss_combine_kernel");
  return DFX_OK;
}

dfx_status dfx_check_flags(const int32_t* flags, dfx_stream stream) {
  int32_t h = 0;
  DFX_CUDA(cudaMemcpyAsync(&h, flags, sizeof(h), cudaMemcpyDeviceToHost, stream));
  DFX_CUDA(cudaStreamSynchronize(stream));
  if (h & kFlagMissingRollouts) return fail(DFX_MISSING_ROLLOUTS, "a record has no rollouts; generation has not run");
  if (h) return fail(DFX_ERROR, "device reported invalid input");
  return DFX_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------------------------
// Per-iteration reward statistics: detail::record_reward_stats (worker.hpp:177-190) on the
// device -- count, sum and sum of squares of the rollouts' "reward" channel -- so aggregate_metrics
// (worker.hpp:275-325) becomes one scalar all-reduce instead of a JSON gather. One block, fixed-shape tree:
// deterministic (f64; the reference's sequential order is not reproduced bit for bit).
// ---------------------------------------------------------------------------------------------------------------
namespace dfx {
__global__ void __launch_bounds__(1024) reward_stats_kernel(int64_t n, const double* __restrict__ reward,
                                                            double* __restrict__ out) {
  __shared__ double sh[32][2];
  double s = 0.0, q = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) {
    const double r = reward[i];
    s += r;
    q = fma(r, r, q);
  }
  s = warp_sum(s);
  q = warp_sum(q);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sh[wid][0] = s;
    sh[wid][1] = q;
  }
  __syncthreads();
  if (wid == 0) {
    s = warp_sum(sh[lane][0]);
    q = warp_sum(sh[lane][1]);
    if (lane == 0) {
      out[0] = (double)n;
      out[1] = s;
      out[2] = q;
    }
  }
}
}  // namespace dfx

extern "C" dfx_status dfx_reward_stats(const dfx_packed* b, double* out, dfx_stream stream) {
  if (!b || !out) return fail(DFX_INVALID_ARGUMENT, "dfx_reward_stats: null argument");
  if (!b->reward) return fail(DFX_MISSING_CHANNEL, "missing channel 'reward'");
  reward_stats_kernel<<<1, 1024, 0, stream>>>(b->n_rollouts, b->reward, out);
  DFX_LAUNCH_CHECK("reward_stats_kernel");
  return DFX_OK;
}
