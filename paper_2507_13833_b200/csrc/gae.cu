// gae.cu -- GAE as a reverse affine scan over packed variable-length rollouts.
//
// The reference has no GAE; it fills the PPO node advantage_compute / func ppo_advantage slot
// (distflow/dag.hpp:333-334). Convention (oracle/dfx_oracle.h dfo_gae):
//   m1 = t+1<L ? mask[t+1] : 0 ; v1 = t+1<L ? V[t+1] : 0
//   delta_t = r_t + gamma*m1*v1 - V_t ; A_t = delta_t + gamma*lam*m1*A_{t+1} ; R_t = A_t + V_t
// Each token is the affine map f_t(X) = delta_t + c_t X (c_t = gamma*lam*m1) and A_t = (f_t o f_{t+1} o ...)(0).
// At the last token of a rollout m1 = v1 = 0, so c = 0 and the chain breaks by itself: GAE over a packed batch is
// ONE reverse scan over the whole token line, no per-rollout segmentation.
//
// Three launches, all stream-ordered (graph-capturable):
//   gae_prep_kernel    thread per rollout: sets the rollout-end bit of its last token in a token bitmap and
//                      advances the look-back epoch (safe here: the previous scan has completed); it releases the
//                      scan as a programmatic dependent launch, so the scan's loads overlap it;
//   gae_smem_kernel    single-pass decoupled look-back scan. One CTA per 4096-token tile, NOT persistent: block b
//                      scans tile n_tiles-1-b, so the tiles it looks back at belong to lower block indices, which
//                      are dispatched first (the forward-progress argument of CUB's single-pass scan). The tile is
//                      bulk-loaded (TMA) into shared memory; each thread owns 32 tokens; every input (r, V, mask,
//                      end bits, the token after the tile) is read without any dependent global load before the
//                      look-back, and each thread clears the end-bit word it consumed, leaving the bitmap zero;
//   gae_finish_kernel  (whitening only) reduces the per-tile masked sums in tile order: deterministic.
// Tile state is one 16-byte record per tile {f64 x ; f32 c ; u32 tag} written and polled with single relaxed
// 128-bit accesses, so value and status are never seen out of order and no fence is needed (on sm_100 a gpu-scope
// fence or acquire invalidates L1: CCTL.IVALL, measured as the top stall of a fenced version).
// Arithmetic: f32 inputs and outputs; deltas, chunk maps, scans and the per-token recurrence in f64. HBM-bound:
// 17 B/token (r, V, mask in; A, R out) + 1 bit/token end map. Design history: profiles/r01_gae_experiments.md.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace dfx {

struct GaeParams {
  const int64_t* cu;
  int64_t n_seq;
  int64_t begin, end;             // token span [begin, end)
  int64_t base;                   // tile origin (begin & ~15)
  int64_t n_tiles;
  int64_t pf_dist;                // L2 prefetch distance in tiles (0: off)
  const float* rew;
  const float* val;
  const uint8_t* mask;
  double gamma, gl;
  float* adv;
  float* ret;
  double* whiten;                 // nullable [3]
  // workspace
  unsigned long long* ticket;     // [2] look-back epoch
  ulonglong2* rec;                // [n_tiles] published tile state
  double* part;                   // [3][n_tiles] whitening partials
  uint8_t* ends;                  // bit (t - base): token t is the last token of its rollout; all-zero between calls
  // fused GAE + PPO loss (dfx_gae_ppo_loss): the clipped surrogate + KL of every token from its advantage as the
  // scan produces it -- the advantage never goes to HBM
  const float* lp;
  const float* old_lp;
  const float* ref_lp;
  float lo1, hi1;                 // 1 - eps_lo, 1 + eps_hi
  float t_hi32, t_lo32, t_hi32_lo, t_lo32_lo;  // log-ratio thresholds as float pairs (clip_exact_f32)
  int kl_type;
  double* lpart;                  // [5][n_tiles] per-tile loss sums {pg, kl, approx_kl, clip, n}
  uint8_t* seq_has;               // [n_seq] rollout has a masked token (prep), summed in order by the finish
};

struct Aff {
  double d, c;  // X -> d + c X
};
// (f o g)(X) = f(g(X))
__device__ __forceinline__ Aff compose(const Aff& f, const Aff& g) { return {fma(f.c, g.d, f.d), f.c * g.c}; }

__device__ __forceinline__ void rec_store(ulonglong2* p, double x, float c, unsigned int tag) {
  const unsigned long long hi = ((unsigned long long)tag << 32) | (unsigned long long)__float_as_uint(c);
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(__double_as_longlong(x)), "l"(hi)
               : "memory");
}
__device__ __forceinline__ ulonglong2 rec_load(const ulonglong2* p) {
  ulonglong2 r;
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ unsigned int rec_tag(const ulonglong2& r) { return (unsigned int)(r.y >> 32); }
__device__ __forceinline__ double rec_x(const ulonglong2& r) { return __longlong_as_double((long long)r.x); }
__device__ __forceinline__ double rec_c(const ulonglong2& r) { return (double)__uint_as_float((unsigned int)r.y); }

// ---- prep: rollout-end bitmap + epoch ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gae_prep_kernel(const int64_t* __restrict__ cu, int64_t n_seq, int64_t base,
                                                       uint32_t* __restrict__ ends, unsigned long long* ticket) {
  // the scan kernel is launched as a programmatic dependent: let it start its loads now; it waits for this
  // grid's completion (griddepcontrol.wait) before reading the bitmap or the epoch
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) ticket[2] = (ticket[2] + 1ull) & 0x3fffffffull;
  if (s >= n_seq) return;
  const int64_t a = __ldg(cu + s), b = __ldg(cu + s + 1);
  if (b <= a) return;  // empty rollouts own no token
  const int64_t e = b - 1 - base;
  atomicOr(ends + (e >> 5), 1u << (e & 31));
}

// fused variant: warp per rollout -- the end bit, the look-back epoch, and whether the rollout has a masked token
// (the sequence count of the loss), found with 16-byte mask loads and an early exit
__global__ void __launch_bounds__(256) gae_prep_loss_kernel(const int64_t* __restrict__ cu, int64_t n_seq,
                                                            int64_t base, uint32_t* __restrict__ ends,
                                                            unsigned long long* ticket,
                                                            const uint8_t* __restrict__ mask, uint8_t* seq_has) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s == 0 && lane == 0) ticket[2] = (ticket[2] + 1ull) & 0x3fffffffull;
  if (s >= n_seq) return;
  const int64_t a = __ldg(cu + s), b = __ldg(cu + s + 1);
  bool has = false;
  if (b > a) {
    if (lane == 0) {
      const int64_t e = b - 1 - base;
      atomicOr(ends + (e >> 5), 1u << (e & 31));
    }
    for (int64_t t0 = a & ~int64_t(15); t0 < b && !has; t0 += 512) {
      const int64_t t = t0 + 16 * lane;
      uint32_t any = 0;
      if (t < b) {
        const uint4 v = *reinterpret_cast<const uint4*>(mask + t);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t tq = t + q;
          if (tq >= a && tq < b && ((w[q >> 2] >> (8 * (q & 3))) & 0xffu)) any = 1;
        }
      }
      has = __any_sync(kFull, any);
    }
  }
  if (lane == 0) seq_has[s] = has ? 1 : 0;
}

// ---- the scan ---------------------------------------------------------------------------------------------------
// Deterministic look-back (warp 0 of the block): the carry X = A at the first token after `tile`.
// The carry must not depend on which predecessor records happen to be published when the warp polls (f64
// composition is not associative), so its definition is fixed by the data alone:
//   * only tiles whose index is a multiple of 32 ("checkpoints") publish an inclusive record derived from a
//     carry; every other tile publishes exactly one record, its aggregate -- tagged inclusive when its map is
//     constant (c == 0: a rollout ends inside the tile, a "natural" inclusive that needs no carry);
//   * tile t composes the aggregates of tiles t+1 .. W-1 with the inclusive of the next checkpoint W above t, or
//     stops at the first natural inclusive before W -- the same elements, composed by the same shuffle tree, on
//     every run.
// By induction every checkpoint's inclusive, hence every carry and every output bit, is run-to-run identical.
// Checkpoints chain (W waits for W+32) only across stretches with no rollout end: one L2 round trip per 32 tiles.
constexpr int64_t kGaeCheckpoint = 32;

__device__ __forceinline__ double gae_lookback(const GaeParams& p, int64_t tile, unsigned int F_AGG,
                                               unsigned int F_INC, int lane) {
  if (tile >= p.n_tiles - 1) return 0.0;
  const int64_t W = (tile / kGaeCheckpoint + 1) * kGaeCheckpoint;
  const int cnt = (int)(W - tile);  // lanes [0, cnt): tiles tile+1 .. W
  const int64_t j = tile + 1 + lane;
  const bool live = lane < cnt && j < p.n_tiles;
  ulonglong2 rr = make_ulonglong2(0ull, (unsigned long long)F_INC << 32);  // past the end (or unused): A = 0
  if (live) rr = rec_load(p.rec + j);
  uint32_t inc_m;
  for (;;) {
    const unsigned int tg = rec_tag(rr);
    inc_m = __ballot_sync(kFull, lane < cnt && tg == F_INC);
    const uint32_t rdy_m = __ballot_sync(kFull, lane < cnt && (tg == F_AGG || tg == F_INC));
    if (inc_m) {
      const uint32_t need = ((inc_m & (0u - inc_m)) << 1) - 1u;
      if ((rdy_m & need) == need) break;
    }
    // non-checkpoint tiles publish once (aggregate or natural inclusive); the checkpoint lane waits for F_INC
    const bool final_rec = tg == F_INC || (tg == F_AGG && lane < cnt - 1);
    if (live && !final_rec) rr = rec_load(p.rec + j);
  }
  const int first = __ffs(inc_m) - 1;
  Aff a{0.0, 1.0};
  if (lane < first) a = Aff{rec_x(rr), rec_c(rr)};
  else if (lane == first) a = Aff{rec_x(rr), 0.0};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double od = __shfl_down_sync(kFull, a.d, o), oc = __shfl_down_sync(kFull, a.c, o);
    if (lane + o < 32) a = compose(a, Aff{od, oc});
  }
  return __shfl_sync(kFull, a.d, 0);
}

// ---------------------------------------------------------------------------------------------------------------
// Shared-memory tiles (default): a tile of THREADS*32 tokens is bulk-loaded (TMA) into shared memory and each
// thread owns 32 consecutive tokens = 8 chunks of 4. A tile is 4-8x longer than a register tile, so the fixed
// cost of its look-back (L2 round trips) is spread over more tokens, while registers stay low because values are
// re-read from shared memory. Chunks are visited in a per-lane rotated order (chunk (j + lane) & 7), which makes
// the 128-bit shared accesses of a warp conflict-free; the in-order dependency is restored by composing the
// eight chunk maps in order afterwards (pass 1) and by deriving every chunk's carry-in before pass 2. Interior
// tiles write A and R back over r and V in shared memory and store them with two bulk copies; the (at most two)
// boundary tiles store per token.
// ---------------------------------------------------------------------------------------------------------------
template <int THREADS>
struct SmemTile {
  static constexpr int TILE = THREADS * 32;
  static constexpr uint32_t kR = 0, kV = TILE * 4 + 16, kM = 2 * (TILE * 4 + 16), kBytes = kM + TILE + 16;
  // fused loss: lp, old, ref of the tile after the mask
  static constexpr uint32_t kL = (kBytes + 127) & ~127u, kO = kL + TILE * 4, kF = kO + TILE * 4,
                            kBytesLoss = kF + TILE * 4;
};

#ifndef DFX_GAE_LOSS_SMEM
#define DFX_GAE_LOSS_SMEM 0  // fused loss inputs: 0 = L2 prefetch + per-thread loads, 1 = TMA into shared memory
#endif
constexpr bool kLossSmem = DFX_GAE_LOSS_SMEM != 0;

template <int THREADS, int MINB, bool WHITEN, bool LOSS = false>
__global__ void __launch_bounds__(THREADS, MINB) gae_smem_kernel(GaeParams p) {
  using L = SmemTile<THREADS>;
  constexpr int TILE = L::TILE, NW = THREADS / 32;
  extern __shared__ __align__(128) uint8_t sm[];
  float* s_r = reinterpret_cast<float*>(sm + L::kR);
  float* s_v = reinterpret_cast<float*>(sm + L::kV);
  uint8_t* s_m = sm + L::kM;
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ Aff s_warp[NW];
  __shared__ double s_X;
  __shared__ double s_red[NW][LOSS ? 5 : 3];
  const float* s_l = reinterpret_cast<const float*>(sm + L::kL);
  const float* s_o = reinterpret_cast<const float*>(sm + L::kO);
  const float* s_f = reinterpret_cast<const float*>(sm + L::kF);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t tile = p.n_tiles - 1 - (int64_t)blockIdx.x;
  const int64_t T0 = p.base + tile * TILE;
  const int64_t rd_end = (p.end + 15) & ~int64_t(15);
  const uint32_t n = (uint32_t)min((int64_t)TILE, rd_end - T0);  // tokens resident in shared memory (16-multiple)
  const bool interior = T0 >= p.begin && T0 + TILE <= p.end;
  const int64_t c0 = T0 + (int64_t)tid * 32;

  if (tid == 0) {
    mbar_init(&s_bar, 1);
    mbar_fence_init();
    mbar_arrive_expect_tx(&s_bar, (LOSS && kLossSmem ? 21u : 9u) * n);
    tma_load_1d(s_r, p.rew + T0, 4u * n, &s_bar);
    tma_load_1d(s_v, p.val + T0, 4u * n, &s_bar);
    tma_load_1d(s_m, p.mask + T0, n, &s_bar);
    if (LOSS && kLossSmem) {
      tma_load_1d(sm + L::kL, p.lp + T0, 4u * n, &s_bar);
      tma_load_1d(sm + L::kO, p.old_lp + T0, 4u * n, &s_bar);
      tma_load_1d(sm + L::kF, p.ref_lp + T0, 4u * n, &s_bar);
    } else if (LOSS) {  // into L2 now, read per thread in pass 2 (keeps shared memory -- and occupancy -- as GAE's)
      l2_prefetch(p.lp + T0, 4u * n);
      l2_prefetch(p.old_lp + T0, 4u * n);
      l2_prefetch(p.ref_lp + T0, 4u * n);
    }
    // the token after the tile (V, mask) sits one past the tile in shared memory
    const int64_t tn = T0 + TILE;
    s_v[TILE] = tn < p.end ? __ldg(p.val + tn) : 0.0f;
    s_m[TILE] = tn < p.end ? __ldg(p.mask + tn) : (uint8_t)0;
    if (p.pf_dist > 0 && tile >= p.pf_dist) {  // keep HBM busy: the next wave's tile into L2
      const int64_t T0p = p.base + (tile - p.pf_dist) * TILE;
      const uint32_t np = (uint32_t)min((int64_t)TILE, rd_end - T0p);
      l2_prefetch(p.rew + T0p, 4u * np);
      l2_prefetch(p.val + T0p, 4u * np);
      l2_prefetch(p.mask + T0p, np);
    }
  }
  // (programmatic dependent launch: everything above overlapped the prep kernel; the bitmap and epoch need it done)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // this thread's rollout-end bits (32 tokens = one aligned 32-bit word of the bitmap), cleared once read
  uint32_t last = 0u;
  if (c0 < rd_end) {
    uint32_t* ew = reinterpret_cast<uint32_t*>(p.ends) + ((c0 - p.base) >> 5);
    last = __ldcg(ew);
    if (last) *ew = 0u;
  }
  uint32_t ident = 0u;
  if (!(c0 >= p.begin && c0 + 32 <= p.end)) {
    for (int q = 0; q < 32; ++q)
      if (c0 + q < p.begin || c0 + q >= p.end) ident |= 1u << q;
  }
  unsigned int epoch;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(epoch) : "l"(p.ticket + 2) : "memory");
  const unsigned int F_AGG = (epoch << 2) | 1u, F_INC = (epoch << 2) | 2u;
  // f64 deltas and maps: with lambda = 1 the f32 rounding of each delta (~eps |V|) does not telescope and
  // would dominate returns that are small against the values
  const double gamd = p.gamma, gld = p.gl;
  __syncthreads();  // s_bar initialised, next-token slot written
  mbar_wait(&s_bar, 0);

  // pass 1: chunk maps in a per-lane rotated order starting at chunk s = lane & 7 (conflict-free 128-bit shared
  // reads), folded into tail = C_s o ... o C_7 and head = C_0 o ... o C_(s-1); the thread map is head o tail.
  // link bit q: token q's successor is in the same rollout and unmasked. Tokens outside the batch are identities
  // (ident) and never stored.
  const int s0 = lane & 7;
  const float vn_cross = s_v[tid * 32 + 32];  // first V of the next thread (or the token after the tile)
  double Hd = 0.0, Hc = 1.0, Td = 0.0, Tc = 1.0;  // the thread's 32-token map, f64
  uint32_t link = 0u, mbits = 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int ch = (s0 + j) & 7;
    const int i0 = tid * 32 + ch * 4;
    const float4 r4 = *reinterpret_cast<const float4*>(s_r + i0);
    const float4 v4 = *reinterpret_cast<const float4*>(s_v + i0);
    const uint32_t m4 = *reinterpret_cast<const uint32_t*>(s_m + i0);
    const float vnx = ch == 7 ? vn_cross : s_v[i0 + 4];
    const uint32_t mnx = s_m[i0 + 4] ? 1u : 0u;
    const float rr[4] = {r4.x, r4.y, r4.z, r4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
    double fd = 0.0, fc = 1.0;
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      const int q = ch * 4 + k;
      const uint32_t mnext = k == 3 ? mnx : (((m4 >> (8 * (k + 1))) & 0xffu) ? 1u : 0u);
      const bool lk = mnext && !((last >> q) & 1u);
      const float vnext = k == 3 ? vnx : vv[k + 1];
      const double dq = (lk ? fma(gamd, (double)vnext, (double)rr[k]) : (double)rr[k]) - (double)vv[k];
      if (!((ident >> q) & 1u)) {
        fd = lk ? fma(gld, fd, dq) : dq;
        fc = lk ? fc * gld : 0.0;
      }
      link |= (lk ? 1u : 0u) << q;
      mbits |= (((m4 >> (8 * k)) & 0xffu) ? 1u : 0u) << q;
    }
    if (ch >= s0) {  // append on the right: F o C
      Td = fma(Tc, fd, Td);
      Tc *= fc;
    } else {
      Hd = fma(Hc, fd, Hd);
      Hc *= fc;
    }
  }
  Aff S{fma(Hc, Td, Hd), Hc * Tc};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double od = __shfl_down_sync(kFull, S.d, o), oc = __shfl_down_sync(kFull, S.c, o);
    if (lane + o < 32) S = compose(S, Aff{od, oc});
  }
  if (lane == 0) s_warp[wid] = S;
  Aff E{__shfl_down_sync(kFull, S.d, 1), __shfl_down_sync(kFull, S.c, 1)};
  if (lane == 31) E = Aff{0.0, 1.0};
  __syncthreads();
  if (wid == 0) {
    Aff tot{0.0, 1.0};
#pragma unroll
    for (int w = NW - 1; w >= 0; --w) tot = compose(s_warp[w], tot);
    if (lane == 0) rec_store(p.rec + tile, tot.d, (float)tot.c, tot.c == 0.0 ? F_INC : F_AGG);
    const double X = gae_lookback(p, tile, F_AGG, F_INC, lane);
    if (lane == 0) {
      if (tot.c != 0.0 && tile % kGaeCheckpoint == 0) rec_store(p.rec + tile, fma(tot.c, X, tot.d), 0.0f, F_INC);
      s_X = X;
    }
  }
  __syncthreads();
  double Xd = s_X;
#pragma unroll
  for (int w = NW - 1; w >= 0; --w)
    if (w > wid) Xd = fma(s_warp[w].c, Xd, s_warp[w].d);
  // pass 2 in descending cyclic order from chunk s-1: chunks s-1 .. 0 start from the carry tail(X_in), chunks
  // 7 .. s from X_in. Interior tiles write A over r at once and R over V one chunk late, after the chunk below
  // has read this chunk's first V as its successor value.
  // the per-token recurrence runs in f64 from the carry: A_t = delta_t + gl A_{t+1} keeps the oracle's accuracy
  // where long discounted sums cancel (values stored as f32 once)
  const double Xin = fma(E.c, Xd, E.d);
  double X = fma(Tc, Xin, Td);
  float wa = 0.0f, wa2 = 0.0f;
  float lpg = 0.0f, lkl = 0.0f, lakl = 0.0f, lclip = 0.0f;  // fused loss sums over this thread's tokens
  float4 pendR = make_float4(0.f, 0.f, 0.f, 0.f);
  int pend_i = -1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int ch = (s0 - 1 - j) & 7;
    if (j == s0) X = Xin;
    const int i0 = tid * 32 + ch * 4;
    const float4 r4 = *reinterpret_cast<const float4*>(s_r + i0);
    const float4 v4 = *reinterpret_cast<const float4*>(s_v + i0);
    const float vnx = ch == 7 ? vn_cross : s_v[i0 + 4];
    if (interior && pend_i >= 0) *reinterpret_cast<float4*>(s_v + pend_i) = pendR;
    const float rr[4] = {r4.x, r4.y, r4.z, r4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
    float4 l4 = make_float4(0.f, 0.f, 0.f, 0.f), o4 = l4, f4 = l4;
    if (LOSS && !kLossSmem && T0 + tid * 32 + ch * 4 + 4 <= rd_end) {  // (L2 hits: prefetched at the start)
      const int64_t g = T0 + tid * 32 + ch * 4;
      l4 = *reinterpret_cast<const float4*>(p.lp + g);
      o4 = *reinterpret_cast<const float4*>(p.old_lp + g);
      f4 = *reinterpret_cast<const float4*>(p.ref_lp + g);
    }
    float oa[4], orr[4];
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      const int q = ch * 4 + k;
      const bool lk = (link >> q) & 1u;
      const float vnext = k == 3 ? vnx : vv[k + 1];
      const double dq = (lk ? fma(gamd, (double)vnext, (double)rr[k]) : (double)rr[k]) - (double)vv[k];
      const double A = lk ? fma(gld, X, dq) : dq;
      X = ((ident >> q) & 1u) ? X : A;
      oa[k] = (float)X;
      orr[k] = (float)(X + (double)vv[k]);
      if (WHITEN) {
        const float mw = ((mbits & ~ident) >> q) & 1u ? 1.0f : 0.0f;
        wa = fmaf(mw, oa[k], wa);
        wa2 = fmaf(mw * oa[k], oa[k], wa2);
      }
      if (LOSS && (((mbits & ~ident) >> q) & 1u)) {  // the PPO terms of a masked token (oracle dfo_ppo_loss)
        const int i = i0 + k;
        const float l = kLossSmem ? s_l[i] : f4_get(l4, k), o = kLossSmem ? s_o[i] : f4_get(o4, k),
                    rf = kLossSmem ? s_f[i] : f4_get(f4, k), A = oa[k];
        const float d = l - o;
        const float rho = exp2f(d * kLog2e);
        const float rc = fminf(fmaxf(rho, p.lo1), p.hi1);
        lpg += fmaxf(-A * rho, -A * rc);
        const float sg = A < 0.0f ? -1.0f : 1.0f;
        const float sT = A > 0.0f ? p.t_hi32 : (A < 0.0f ? -p.t_lo32 : __int_as_float(0x7f800000));
        lclip += clip_exact_f32(sg, sT, sg > 0.0f ? p.t_hi32_lo : -p.t_lo32_lo, l, o, d) ? 1.0f : 0.0f;
        const float x = rf - l;
        float kl = 0.0f;
        if (p.kl_type == DFX_KL_K3) kl = fabsf(x) < kK3Series ? k3_series(x) : fminf(fmaxf(expm1f(x) - x, -10.0f), 10.0f);
        else if (p.kl_type == DFX_KL_K1) kl = -x;
        else if (p.kl_type == DFX_KL_K2) kl = 0.5f * x * x;
        lkl += kl;
        lakl -= d;
      }
    }
    if (interior) {
      *reinterpret_cast<float4*>(s_r + i0) = make_float4(oa[0], oa[1], oa[2], oa[3]);
      pendR = make_float4(orr[0], orr[1], orr[2], orr[3]);
      pend_i = i0;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!((ident >> (ch * 4 + k)) & 1u)) {
          if (!LOSS || p.adv) p.adv[c0 + ch * 4 + k] = oa[k];
          p.ret[c0 + ch * 4 + k] = orr[k];
        }
      }
    }
  }
  if (interior) *reinterpret_cast<float4*>(s_v + pend_i) = pendR;
  if (interior) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      if (!LOSS || p.adv) tma_store_1d(p.adv + T0, s_r, 4u * TILE);  // (fused: the advantage stays on chip)
      tma_store_1d(p.ret + T0, s_v, 4u * TILE);
      tma_store_commit_and_wait();
    }
  }
  if (LOSS) {  // per-tile loss sums: fixed-shape block reduction, summed over tiles in order by the finish kernel
    const double v5[5] = {warp_sum((double)lpg), warp_sum((double)lkl), warp_sum((double)lakl),
                          warp_sum((double)lclip), warp_sum((double)__popc(mbits & ~ident))};
    if (lane == 0)
      for (int q = 0; q < 5; ++q) s_red[wid][q] = v5[q];
    __syncthreads();
    if (tid < 5) {
      double t5 = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) t5 += s_red[w][tid];
      p.lpart[(int64_t)tid * p.n_tiles + tile] = t5;
    }
  }
  if (WHITEN) {
    const double wad = warp_sum((double)wa), wa2d = warp_sum((double)wa2);
    const double wm = warp_sum((double)__popc(mbits & ~ident));
    if (lane == 0) {
      s_red[wid][0] = wad;
      s_red[wid][1] = wa2d;
      s_red[wid][2] = wm;
    }
    __syncthreads();
    if (tid < 3) {
      double t3 = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) t3 += s_red[w][tid];
      p.part[(int64_t)tid * p.n_tiles + tile] = t3;
    }
  }
}

// ---- whitening sums: fixed-shape reduction of the per-tile partials ---------------------------------------------
__global__ void __launch_bounds__(256) gae_finish_kernel(const double* __restrict__ part, int64_t n_tiles,
                                                         double* __restrict__ whiten) {
  __shared__ double s_red[8][3];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double tot[3] = {0.0, 0.0, 0.0};
  for (int64_t i = tid; i < n_tiles; i += 256)
#pragma unroll
    for (int q = 0; q < 3; ++q) tot[q] += part[(int64_t)q * n_tiles + i];
#pragma unroll
  for (int q = 0; q < 3; ++q) tot[q] = warp_sum(tot[q]);
  if (lane == 0)
    for (int q = 0; q < 3; ++q) s_red[wid][q] = tot[q];
  __syncthreads();
  if (tid == 0) {
    double t3[3] = {0.0, 0.0, 0.0};
    for (int w = 0; w < 8; ++w)
      for (int q = 0; q < 3; ++q) t3[q] += s_red[w][q];
    for (int q = 0; q < 3; ++q) whiten[q] = t3[q];
  }
}

// fused loss: the per-tile sums in tile order (fixed-shape tree) -> token-mean dfx_loss_out; the sequence count
// from the prep kernel's per-rollout flags
__global__ void __launch_bounds__(256) gae_loss_finish_kernel(const double* __restrict__ lpart, int64_t n_tiles,
                                                              const uint8_t* __restrict__ seq_has, int64_t n_seq,
                                                              double beta, dfx_loss_out* out) {
  __shared__ double s_red[8][6];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double tot[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t i = tid; i < n_tiles; i += 256)
#pragma unroll
    for (int q = 0; q < 5; ++q) tot[q] += lpart[(int64_t)q * n_tiles + i];
  for (int64_t s = tid; s < n_seq; s += 256) tot[5] += seq_has[s] ? 1.0 : 0.0;
#pragma unroll
  for (int q = 0; q < 6; ++q) tot[q] = warp_sum(tot[q]);
  if (lane == 0)
    for (int q = 0; q < 6; ++q) s_red[wid][q] = tot[q];
  __syncthreads();
  if (tid == 0) {
    double t6[6] = {0, 0, 0, 0, 0, 0};
    for (int w = 0; w < 8; ++w)
      for (int q = 0; q < 6; ++q) t6[q] += s_red[w][q];
    const double N = t6[4];
    dfx_loss_out o;
    o.pg_loss = N > 0 ? t6[0] / N : 0.0;
    o.kl = N > 0 ? t6[1] / N : 0.0;
    o.loss = o.pg_loss + beta * o.kl;
    o.approx_kl = N > 0 ? t6[2] / N : 0.0;
    o.clipfrac = N > 0 ? t6[3] / N : 0.0;
    o.n_tokens = N;
    o.n_seqs = t6[5];
    *out = o;
  }
}

int64_t gae_tiles(int64_t token_base, int64_t token_span, int64_t tile) {
  const int64_t base = token_base & ~int64_t(15);
  return (token_base + token_span - base + tile - 1) / tile;
}

constexpr int64_t kGaeMinTile = 2048;  // smallest tile of any variant (s64: 64 x 32 tokens; workspace sizing)

struct GaeWs {
  size_t ticket, ends, rec, part, lpart, bytes;
  int64_t cap_tiles;
};
// The layout is a function of the tile CAPACITY only, never of the call's span: the self-maintained state (the
// epoch ticket and the all-zero end bitmap) must sit at the same offsets on every call that reuses a workspace, or
// a call with a smaller span would OR its end bits onto a previous call's tile records / whitening partials.
// Order: ticket, end bitmap (both kept consistent by the kernels), then the regions written before being read;
// the fused loss's per-rollout flags follow the capacity part (written before read as well).
GaeWs gae_ws_layout_cap(int64_t cap_tiles) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  GaeWs w{};
  w.cap_tiles = cap_tiles;
  w.ticket = 0;
  w.ends = al(3 * sizeof(unsigned long long));
  w.rec = w.ends + al(size_t(cap_tiles) * kGaeMinTile / 8 + 16);
  w.part = w.rec + al(16 * size_t(cap_tiles));
  w.lpart = w.part + al(24 * size_t(cap_tiles));
  w.bytes = w.lpart + al(40 * size_t(cap_tiles));
  return w;
}
// tiles needed for a span (tile count depends on token_base & 15 as well: size for the worst case)
int64_t gae_tiles_needed(int64_t token_span) { return (token_span + 15) / kGaeMinTile + 2; }
// the largest capacity whose layout fits in ws_bytes (the caller's buffer size fixes the layout)
GaeWs gae_ws_layout_fit(size_t ws_bytes) {
  int64_t cap = (int64_t)(ws_bytes / (kGaeMinTile / 8 + 16 + 24 + 40));  // an upper bound; step down to the fit
  while (cap > 0 && gae_ws_layout_cap(cap).bytes > ws_bytes) --cap;
  return gae_ws_layout_cap(cap);
}

// Tuning knob (benchmarking only): DFX_GAE_VARIANT = s128 (default: 128 threads x 32 tokens, 5 CTAs/SM) |
// s128b4 | s256 | s64 (the register-tile designs it replaced are in profiles/r01_gae_experiments.md)
inline int gae_variant() {
  static const int v = [] {
    const char* e = std::getenv("DFX_GAE_VARIANT");
    if (!e) return 0;
    const std::string s(e);
    return s == "s128b4" ? 1 : s == "s256" ? 2 : s == "s64" ? 3 : 0;
  }();
  return v;
}

template <int THREADS, int MINB, bool LOSS = false>
void gae_launch_smem(GaeParams& p, cudaStream_t st) {
  using L = SmemTile<THREADS>;
  constexpr uint32_t kSmem = LOSS && kLossSmem ? L::kBytesLoss : L::kBytes;
  p.n_tiles = gae_tiles(p.begin, p.end - p.begin, L::TILE);
  static thread_local int cached_dev = -1, resident = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    int sms = 0, per_sm = 0;
    cudaFuncSetAttribute(gae_smem_kernel<THREADS, MINB, true, LOSS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    cudaFuncSetAttribute(gae_smem_kernel<THREADS, MINB, false, LOSS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_smem_kernel<THREADS, MINB, true, LOSS>, THREADS, kSmem);
    resident = sms * std::max(per_sm, 1);
    cached_dev = dev;
  }
  static const int pf_env = std::getenv("DFX_GAE_PF") ? std::atoi(std::getenv("DFX_GAE_PF")) : 100;
  p.pf_dist = LOSS ? 0 : (int64_t)resident * pf_env / 100;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)p.n_tiles);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap launch + loads with gae_prep_kernel
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (p.whiten) cudaLaunchKernelEx(&cfg, gae_smem_kernel<THREADS, MINB, true, LOSS>, p);
  else cudaLaunchKernelEx(&cfg, gae_smem_kernel<THREADS, MINB, false, LOSS>, p);
}


}  // namespace dfx

using namespace dfx;

extern "C" {

size_t dfx_gae_workspace_bytes(int64_t n_rollouts, int64_t token_span) {
  (void)n_rollouts;
  return gae_ws_layout_cap(gae_tiles_needed(token_span)).bytes;
}

dfx_status dfx_gae(const dfx_packed* b, int64_t token_base, int64_t token_span, double gamma, double lam, float* adv,
                   float* ret, double* whiten, void* workspace, size_t ws_bytes, dfx_stream stream) {
  if (!b || !b->cu_seqlens || !b->token_reward || !b->value_tok || !b->mask || !adv || !ret)
    return fail(DFX_INVALID_ARGUMENT, "dfx_gae: packed batch lacks cu_seqlens/token_reward/value_tok/mask or null output");
  if (b->n_rollouts <= 0 || token_span <= 0) {
    if (whiten) DFX_CUDA(cudaMemsetAsync(whiten, 0, 3 * sizeof(double), stream));
    return DFX_OK;
  }
  const GaeWs wl = gae_ws_layout_fit(ws_bytes);
  if (!workspace || wl.cap_tiles < gae_tiles_needed(token_span))
    return fail(DFX_INVALID_ARGUMENT, "dfx_gae: workspace too small");
  char* w = static_cast<char*>(workspace);
  GaeParams p{};
  p.cu = b->cu_seqlens;
  p.n_seq = b->n_rollouts;
  p.begin = token_base;
  p.end = token_base + token_span;
  p.base = token_base & ~int64_t(15);
  p.ticket = reinterpret_cast<unsigned long long*>(w + wl.ticket);
  p.rec = reinterpret_cast<ulonglong2*>(w + wl.rec);
  p.part = reinterpret_cast<double*>(w + wl.part);
  p.ends = reinterpret_cast<uint8_t*>(w + wl.ends);
  p.rew = b->token_reward;
  p.val = b->value_tok;
  p.mask = b->mask;
  p.gamma = gamma;
  p.gl = gamma * lam;
  p.adv = adv;
  p.ret = ret;
  p.whiten = whiten;
  gae_prep_kernel<<<(unsigned)((p.n_seq + 255) / 256), 256, 0, stream>>>(p.cu, p.n_seq, p.base,
                                                                          reinterpret_cast<uint32_t*>(p.ends), p.ticket);
  DFX_LAUNCH_CHECK("gae_prep_kernel");
  switch (gae_variant()) {
    case 1: gae_launch_smem<128, 4>(p, stream); break;
    case 2: gae_launch_smem<256, 2>(p, stream); break;
    case 3: gae_launch_smem<64, 8>(p, stream); break;
    default: gae_launch_smem<128, 5>(p, stream); break;
  }
  DFX_LAUNCH_CHECK("gae_smem_kernel");
  if (whiten) {
    gae_finish_kernel<<<1, 256, 0, stream>>>(p.part, p.n_tiles, whiten);
    DFX_LAUNCH_CHECK("gae_finish_kernel");
  }
  return DFX_OK;
}


// (the fused pass keeps its per-rollout flags in the whitening-partials region, 24 bytes per tile of capacity)
size_t dfx_gae_ppo_loss_workspace_bytes(int64_t n_rollouts, int64_t token_span) {
  return gae_ws_layout_cap(std::max(gae_tiles_needed(token_span), std::max<int64_t>(n_rollouts, 0) / 24 + 1)).bytes;
}

dfx_status dfx_gae_ppo_loss(const dfx_packed* b, int64_t token_base, int64_t token_span, double gamma, double lam,
                            const dfx_loss_cfg* cfg, float* ret, float* adv, dfx_loss_out* out, void* workspace,
                            size_t ws_bytes, dfx_stream stream) {
  if (!b || !cfg || !out || !ret || !b->cu_seqlens || !b->token_reward || !b->value_tok || !b->mask || !b->lp ||
      !b->old_lp || !b->ref_lp)
    return fail(DFX_INVALID_ARGUMENT, "dfx_gae_ppo_loss: the batch needs cu_seqlens, token_reward, value_tok, mask, "
                                      "lp, old_lp, ref_lp; ret and out are required");
  if (cfg->agg != DFX_AGG_TOKEN_MEAN || cfg->whiten)
    return fail(DFX_INVALID_ARGUMENT, "dfx_gae_ppo_loss: the fused pass computes the token-mean loss of unwhitened "
                                      "advantages (whitening or sequence means need dfx_gae + dfx_ppo_loss)");
  if (cfg->kl_type < 0 || cfg->kl_type > 3) return fail(DFX_INVALID_ARGUMENT, "dfx_gae_ppo_loss: bad kl_type");
  if (b->n_rollouts <= 0 || token_span <= 0) {
    DFX_CUDA(cudaMemsetAsync(out, 0, sizeof(dfx_loss_out), stream));
    return DFX_OK;
  }
  const GaeWs wl = gae_ws_layout_fit(ws_bytes);
  if (!workspace || wl.cap_tiles < gae_tiles_needed(token_span) || 24 * wl.cap_tiles < b->n_rollouts)
    return fail(DFX_INVALID_ARGUMENT, "dfx_gae_ppo_loss: workspace too small");
  char* w = static_cast<char*>(workspace);
  GaeParams p{};
  p.cu = b->cu_seqlens;
  p.n_seq = b->n_rollouts;
  p.begin = token_base;
  p.end = token_base + token_span;
  p.base = token_base & ~int64_t(15);
  p.ticket = reinterpret_cast<unsigned long long*>(w + wl.ticket);
  p.rec = reinterpret_cast<ulonglong2*>(w + wl.rec);
  p.part = reinterpret_cast<double*>(w + wl.part);
  p.ends = reinterpret_cast<uint8_t*>(w + wl.ends);
  p.lpart = reinterpret_cast<double*>(w + wl.lpart);
  p.seq_has = reinterpret_cast<uint8_t*>(w + wl.part);  // (no whitening here: the partials region is free)
  p.rew = b->token_reward;
  p.val = b->value_tok;
  p.mask = b->mask;
  p.gamma = gamma;
  p.gl = gamma * lam;
  p.adv = adv;
  p.ret = ret;
  p.whiten = nullptr;
  p.lp = b->lp;
  p.old_lp = b->old_lp;
  p.ref_lp = b->ref_lp;
  p.lo1 = 1.0f - (float)cfg->clip_low;
  p.hi1 = 1.0f + (float)cfg->clip_high;
  const double t_hi = std::log(1.0 + cfg->clip_high);
  const double t_lo = cfg->clip_low < 1.0 ? std::log(1.0 - cfg->clip_low) : -HUGE_VAL;
  p.t_hi32 = (float)t_hi;
  p.t_lo32 = (float)t_lo;
  p.t_hi32_lo = (float)(t_hi - (double)p.t_hi32);
  p.t_lo32_lo = std::isfinite(t_lo) ? (float)(t_lo - (double)p.t_lo32) : 0.0f;
  p.kl_type = cfg->kl_type;
  gae_prep_loss_kernel<<<(unsigned)((p.n_seq + 7) / 8), 256, 0, stream>>>(
      p.cu, p.n_seq, p.base, reinterpret_cast<uint32_t*>(p.ends), p.ticket, p.mask, p.seq_has);
  DFX_LAUNCH_CHECK("gae_prep_loss_kernel");
  switch (gae_variant()) {
    case 1: gae_launch_smem<128, 4, true>(p, stream); break;
    case 3: gae_launch_smem<64, 8, true>(p, stream); break;
    default: gae_launch_smem<128, 5, true>(p, stream); break;
  }
  DFX_LAUNCH_CHECK("gae_smem_kernel<loss>");
  gae_loss_finish_kernel<<<1, 256, 0, stream>>>(p.lpart, p.n_tiles, p.seq_has, p.n_seq, cfg->beta, out);
  DFX_LAUNCH_CHECK("gae_loss_finish_kernel");
  return DFX_OK;
}

}  // extern "C"
