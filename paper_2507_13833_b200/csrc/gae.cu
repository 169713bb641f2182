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
//   gae_prep_kernel    thread per rollout: sets the rollout-end bit of its last token in a token bitmap, writes
//                      the segment bounds (below) and advances the publish epoch (safe here: the previous scan has
//                      completed); it releases the scan as a programmatic dependent launch;
//   the scan           dfx_gae: gae_seg_kernel (rollout-aligned segments, persistent, TMA ring, no look-back for
//                      rollouts up to 64K tokens); the fused dfx_gae_ppo_loss: gae_smem_kernel (one 4096-token
//                      tile per CTA, single-pass decoupled look-back; block b scans tile n_tiles-1-b, so the tiles it
//                      looks back at belong to lower block indices, dispatched first -- the forward-progress
//                      argument of CUB's single-pass scan). Both stage their tiles with bulk copies (TMA) and every
//                      reader clears the end bits it consumed, leaving the bitmap zero between calls;
//   gae_finish_kernel  (whitening only) reduces the per-segment / per-tile masked sums in order: deterministic.
// Tile state is one 16-byte record per tile {f64 x ; f32 c ; u32 tag} written and polled with single relaxed
// 128-bit accesses, so value and status are never seen out of order and no fence is needed (on sm_100 a gpu-scope
// fence or acquire invalidates L1: CCTL.IVALL, measured as the top stall of a fenced version).
// Arithmetic: f32 inputs and outputs; deltas, chunk maps, scans and the per-token recurrence in f64. HBM-bound:
// 17 B/token (r, V, mask in; A, R out) + 1 bit/token end map. Design history: profiles/r01_gae_experiments.md,
// profiles/r02_gae_segments.md.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

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
  // rollout-aligned segments (gae_seg_kernel)
  int64_t seg_len;                // nominal segment length S
  int64_t n_segs;
  unsigned long long* seg_start;  // [n_segs + 1] segment starts (bit 62: the start cuts a rollout)
  unsigned long long* trace;      // (DFX_GAE_TRACE, diagnostics only) per-CTA globaltimer stamps
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

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
__device__ __forceinline__ void seg_bounds_from_start(const GaeParams& p, int64_t s);

__global__ void __launch_bounds__(256) gae_prep_kernel(GaeParams p) {
  // the scan kernel is launched as a programmatic dependent: let it start now; it waits for this grid's
  // completion (griddepcontrol.wait) before reading the bitmap, the segment bounds or the epoch
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) {
    p.ticket[2] = (p.ticket[2] + 1ull) & 0x3fffffffull;
    p.ticket[0] = 0ull;  // segment claims
  }
  if (s > p.n_seq) return;
  if (p.seg_start) seg_bounds_from_start(p, s);
  if (s == p.n_seq) return;
  const int64_t a = __ldg(p.cu + s), b = __ldg(p.cu + s + 1);
  if (b <= a) return;  // empty rollouts own no token
  const int64_t e = b - 1 - p.base;
  atomicOr(reinterpret_cast<uint32_t*>(p.ends) + (e >> 5), 1u << (e & 31));
}

// fused variant: warp per rollout -- the end bit, the segment bounds, the epoch, and whether the rollout has a
// masked token (the sequence count of the loss), found with 16-byte mask loads and an early exit
__global__ void __launch_bounds__(256) gae_prep_loss_kernel(GaeParams p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s == 0 && lane == 0) {
    p.ticket[2] = (p.ticket[2] + 1ull) & 0x3fffffffull;
    p.ticket[0] = 0ull;
  }
  if (s > p.n_seq) return;
  if (lane == 0 && p.seg_start) seg_bounds_from_start(p, s);
  if (s == p.n_seq) return;
  const int64_t a = __ldg(p.cu + s), b = __ldg(p.cu + s + 1);
  bool has = false;
  if (b > a) {
    if (lane == 0) {
      const int64_t e = b - 1 - p.base;
      atomicOr(reinterpret_cast<uint32_t*>(p.ends) + (e >> 5), 1u << (e & 31));
    }
    for (int64_t t0 = a & ~int64_t(15); t0 < b && !has; t0 += 512) {
      const int64_t t = t0 + 16 * lane;
      uint32_t any = 0;
      if (t < b) {
        const uint4 v = *reinterpret_cast<const uint4*>(p.mask + t);
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
  if (lane == 0) p.seq_has[s] = has ? 1 : 0;
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
};


// Fused loss terms of one tile after pass 2 (oracle dfo_ppo_loss per masked token), read coalesced: thread tid
// takes the 4-token vectors tid, tid + THREADS, ... -- A and the mask from shared memory (pass 2 wrote A over r),
// lp / old / ref from L2 (prefetched when the tile's loads were issued). Tokens outside [rb, re) are another
// tile's or segment's. Exact integer counts of clipped and masked tokens.
template <int THREADS>
__device__ __forceinline__ void gae_tile_loss(const GaeParams& p, int64_t T0, uint32_t n, int64_t rb, int64_t re,
                                              const float* s_a, const uint8_t* s_m, float& lpg, float& lkl,
                                              float& lakl, uint32_t& lclip, uint32_t& lcnt) {
  constexpr int kU = 4;  // vectors in flight per thread
  const int32_t lo = (int32_t)max((int64_t)-1, min((int64_t)n, rb - T0));
  const int32_t hi = (int32_t)max((int64_t)0, min((int64_t)n, re - T0));
  for (uint32_t i0 = 4u * threadIdx.x; i0 < n; i0 += 4u * THREADS * kU) {
    float4 l4[kU], o4[kU], f4[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + 4u * THREADS * u;
      if (i < n) {
        l4[u] = __ldcg(reinterpret_cast<const float4*>(p.lp + T0 + i));
        o4[u] = __ldcg(reinterpret_cast<const float4*>(p.old_lp + T0 + i));
        f4[u] = __ldcg(reinterpret_cast<const float4*>(p.ref_lp + T0 + i));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + 4u * THREADS * u;
      if (i >= n) break;
      const float4 a4 = *reinterpret_cast<const float4*>(s_a + i);
      const uint32_t m4 = *reinterpret_cast<const uint32_t*>(s_m + i);
      uint32_t onb = 0u, clb = 0u;
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // (branch-free: masked-out tokens contribute zero)
        const int32_t ti = (int32_t)i + k;
        const bool on = ((m4 >> (8 * k)) & 0xffu) && ti >= lo && ti < hi;
        const float m = on ? 1.0f : 0.0f;
        const float l = f4_get(l4[u], k), o = f4_get(o4[u], k), rf = f4_get(f4[u], k), A = f4_get(a4, k);
        const float d = l - o;
        const float rho = ex2_ftz(d * kLog2e);
        const float rc = fminf(fmaxf(rho, p.lo1), p.hi1);
        lpg = fmaf(m, fmaxf(-A * rho, -A * rc), lpg);
        const float sg = A < 0.0f ? -1.0f : 1.0f;
        const float sT = A > 0.0f ? p.t_hi32 : (A < 0.0f ? -p.t_lo32 : __int_as_float(0x7f800000));
        const bool cl = clip_exact_f32(sg, sT, sg > 0.0f ? p.t_hi32_lo : -p.t_lo32_lo, l, o, d);
        const float x = rf - l;
        float kl = 0.0f;
        if (p.kl_type == DFX_KL_K3) kl = fabsf(x) < kK3Series ? k3_series(x) : fminf(fmaxf(expm1f(x) - x, -10.0f), 10.0f);
        else if (p.kl_type == DFX_KL_K1) kl = -x;
        else if (p.kl_type == DFX_KL_K2) kl = 0.5f * x * x;
        lkl = fmaf(m, kl, lkl);
        lakl = fmaf(-m, d, lakl);
        onb |= (on ? 1u : 0u) << k;
        clb |= (cl ? 1u : 0u) << k;
      }
      lcnt += __popc(onb);
      lclip += __popc(onb & clb);
    }
  }
}

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
    mbar_arrive_expect_tx(&s_bar, 9u * n);
    tma_load_1d(s_r, p.rew + T0, 4u * n, &s_bar);
    tma_load_1d(s_v, p.val + T0, 4u * n, &s_bar);
    tma_load_1d(s_m, p.mask + T0, n, &s_bar);
    if (LOSS) {  // into L2 now, read per thread in pass 2 (keeps shared memory -- and occupancy -- as GAE's)
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
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the finish kernel waits for this grid
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
  const uint32_t mn_cross = s_m[tid * 32 + 32] ? 1u : 0u;
  double Hd = 0.0, Hc = 1.0, Td = 0.0, Tc = 1.0;  // the thread's 32-token map, f64
  uint32_t link = 0u, mbits = 0u;
  // the successor (V, mask) of chunk ch is the first token of chunk ch + 1: from the next chunk in the rotated
  // order, loaded one step ahead (scalar shared loads at the 128-byte thread stride are 32-way bank conflicts);
  // chunk s's first V and mask are kept for the wrap-around and for pass 2
  float4 r4n = *reinterpret_cast<const float4*>(s_r + tid * 32 + s0 * 4);
  float4 v4n = *reinterpret_cast<const float4*>(s_v + tid * 32 + s0 * 4);
  uint32_t m4n = *reinterpret_cast<const uint32_t*>(s_m + tid * 32 + s0 * 4);
  const float v_s0first = v4n.x;
  const uint32_t m_s0first = (m4n & 0xffu) ? 1u : 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int ch = (s0 + j) & 7;
    const float4 r4 = r4n, v4 = v4n;
    const uint32_t m4 = m4n;
    if (j < 7) {
      const int chn = (s0 + j + 1) & 7;
      r4n = *reinterpret_cast<const float4*>(s_r + tid * 32 + chn * 4);
      v4n = *reinterpret_cast<const float4*>(s_v + tid * 32 + chn * 4);
      m4n = *reinterpret_cast<const uint32_t*>(s_m + tid * 32 + chn * 4);
    }
    const float vnx = ch == 7 ? vn_cross : (j < 7 ? v4n.x : v_s0first);
    const uint32_t mnx = ch == 7 ? mn_cross : (j < 7 ? ((m4n & 0xffu) ? 1u : 0u) : m_s0first);
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
  float vprev = v_s0first;  // the first V of the chunk processed before (chunk ch + 1); position 0: chunk s
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int ch = (s0 - 1 - j) & 7;
    if (j == s0) X = Xin;
    const int i0 = tid * 32 + ch * 4;
    const float4 r4 = *reinterpret_cast<const float4*>(s_r + i0);
    const float4 v4 = *reinterpret_cast<const float4*>(s_v + i0);
    const float vnx = ch == 7 ? vn_cross : vprev;
    vprev = v4.x;
    const float rr[4] = {r4.x, r4.y, r4.z, r4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
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
    }
    if (interior || LOSS) *reinterpret_cast<float4*>(s_r + i0) = make_float4(oa[0], oa[1], oa[2], oa[3]);
    if (interior) {  // (every successor value of this thread is in registers: R over V at once)
      *reinterpret_cast<float4*>(s_v + i0) = make_float4(orr[0], orr[1], orr[2], orr[3]);
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
  if (interior || LOSS) {
    fence_proxy_async_smem();
    __syncthreads();
    if (interior && tid == 0) {
      if (!LOSS || p.adv) tma_store_1d(p.adv + T0, s_r, 4u * TILE);  // (fused: the advantage stays on chip)
      tma_store_1d(p.ret + T0, s_v, 4u * TILE);
      tma_store_commit_and_wait();
    }
  }
  if (LOSS) {  // per-tile loss sums: fixed-shape block reduction, summed over tiles in order by the finish kernel
    float lpg = 0.0f, lkl = 0.0f, lakl = 0.0f;
    uint32_t lclip = 0u, lcnt = 0u;
    gae_tile_loss<THREADS>(p, T0, n, p.begin, p.end, s_r, s_m, lpg, lkl, lakl, lclip, lcnt);
    const double v5[5] = {warp_sum((double)lpg), warp_sum((double)lkl), warp_sum((double)lakl),
                          (double)warp_sum(lclip), (double)warp_sum(lcnt)};
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

// ---------------------------------------------------------------------------------------------------------------
// Rollout-aligned segments (default). The token line is cut into segments of about S tokens whose boundaries are
// rollout starts: segment j = [b_j, b_(j+1)), b_j = the first rollout start at or after begin + j*S -- unless that
// start is more than kSegMaxNoCut tokens away (a rollout that long is cut at begin + j*S, flagged). A segment that
// ends at a rollout start needs no carry from anywhere (its last token is a rollout end), so a persistent CTA
// streams it alone, right to left, in 2048-token tiles through a 3-stage TMA ring, the carry between its tiles in
// a register: no look-back, no inter-CTA wait. Only a segment ending inside a (> kSegMaxNoCut) rollout waits for
// the published value at its right neighbour's first token. Segments are claimed in descending order (ticket), so
// the neighbour a CTA waits for is always already running. Per tile: pass 1 (thread maps, f64) -> block scan ->
// pass 2 from the carry (A written over r, R over V in shared memory) -> bulk stores (edge tiles: per token) ->
// fused loss terms (dfx_gae_ppo_loss) read coalesced -> the stage is refilled with the tile 3 ahead.
// Everything a CTA computes is a fixed sequence of operations on its segment: run-to-run bit-identical; the
// whitening / loss partials are per segment, summed in segment order by the finish kernels.
// ---------------------------------------------------------------------------------------------------------------
constexpr int kSegThreads = 128, kSegTPT = 16, kSegTile = kSegThreads * kSegTPT, kSegStages = 3;
constexpr int64_t kSegMaxNoCut = 65536;
constexpr unsigned long long kSegCut = 1ull << 62;
struct SegStage {  // r, V (+ the successor), mask (+ the successor), the rollout-end bitmap slice
  static constexpr uint32_t kR = 0, kV = kSegTile * 4 + 16, kM = kV + kSegTile * 4 + 16, kE = kM + kSegTile + 16,
                            kBytes = (kE + kSegTile / 8 + 32 + 127) & ~127u;
};

// segment starts owned by rollout start s (s == n_seq: the span end, a virtual start): the segments whose nominal
// start P_j lies in (cu[s-1], cu[s]]
__device__ __forceinline__ void seg_bounds_from_start(const GaeParams& p, int64_t s) {
  const auto cl = [&](int64_t x) { return max(p.begin, min(p.end, x)); };
  const int64_t c = s < p.n_seq ? cl(__ldg(p.cu + s)) : p.end;
  const int64_t jlo = s > 0 ? (cl(__ldg(p.cu + s - 1)) - p.begin) / p.seg_len + 1 : 0;
  const int64_t jhi = min((c - p.begin) / p.seg_len, p.n_segs - 1);
  for (int64_t j = jlo; j <= jhi; ++j) {
    const int64_t P = p.begin + j * p.seg_len;
    p.seg_start[j] = c - P <= kSegMaxNoCut ? (unsigned long long)c : ((unsigned long long)P | kSegCut);
  }
  if (s == p.n_seq) p.seg_start[p.n_segs] = (unsigned long long)p.end;
}

// bit k set iff byte k of w is nonzero
__device__ __forceinline__ uint32_t nz_bytes4(uint32_t w) {
  const uint32_t x = __vcmpne4(w, 0u) & 0x01010101u;
  return (x | (x >> 7) | (x >> 14) | (x >> 21)) & 0xfu;
}

// (thread 0) the bulk loads of one tile into a stage: r, V, mask, and the 16-byte-aligned slice of the rollout-end
// bitmap that covers it (its bit (T0 - base) sits at byte seg_ebyte(T0, base) of the stage's copy)
__device__ __forceinline__ int64_t seg_ebyte16(int64_t T0, int64_t base) { return ((T0 - base) >> 3) & ~int64_t(15); }

template <bool LOSS>
__device__ __forceinline__ void seg_issue_load(const GaeParams& p, uint8_t* st, uint64_t* bar, int64_t T0, uint32_t n) {
  float* s_v = reinterpret_cast<float*>(st + SegStage::kV);
  uint8_t* s_m = st + SegStage::kM;
  // the token after the tile (16-aligned): its V and mask land one past the tile in shared memory, by the same
  // bulk copies extended by 16 bytes; past the batch it is never read (the batch's last token ends a rollout)
  const int64_t tn = T0 + n;
  const uint32_t xs = tn < p.end ? 16u : 0u;
  const int64_t eb0 = seg_ebyte16(T0, p.base);
  const uint32_t ebytes = (uint32_t)((((T0 - p.base + n + 7) >> 3) - eb0 + 15) & ~int64_t(15));
  mbar_arrive_expect_tx(bar, 9u * n + 2u * xs + ebytes);
  tma_load_1d(st + SegStage::kR, p.rew + T0, 4u * n, bar);
  tma_load_1d(s_v, p.val + T0, 4u * n + xs, bar);
  tma_load_1d(s_m, p.mask + T0, n + xs, bar);
  tma_load_1d(st + SegStage::kE, p.ends + eb0, ebytes, bar);
  if (LOSS) {  // the loss phase reads these coalesced from L2
    l2_prefetch(p.lp + T0, 4u * n);
    l2_prefetch(p.old_lp + T0, 4u * n);
    l2_prefetch(p.ref_lp + T0, 4u * n);
  }
}

template <bool WHITEN, bool LOSS>
__global__ void __launch_bounds__(kSegThreads, 4) gae_seg_kernel(GaeParams p) {
  constexpr int NW = kSegThreads / 32;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t s_full[kSegStages];
  __shared__ Aff s_warp[NW];
  __shared__ double s_X;
  __shared__ double s_red[NW][5];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int s0 = lane & 3;
  if (tid == 0) {
    for (int i = 0; i < kSegStages; ++i) mbar_init(&s_full[i], 1);
    mbar_fence_init();
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the prep grid: bitmap, bounds, epoch, ticket reset
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the finish kernel waits for this grid
  unsigned long long* tr = p.trace ? p.trace + 32 * blockIdx.x : nullptr;
  int nseg_done = 0;
  if (tr && tid == 0) tr[0] = gtimer();
  unsigned int epoch;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(epoch) : "l"(p.ticket + 2) : "memory");
  const unsigned int F_INC = (epoch << 2) | 2u;
  const double gamd = p.gamma, gld = p.gl, gld4 = (p.gl * p.gl) * (p.gl * p.gl);
  uint32_t phase = 0u;  // parity bit per stage
  for (;;) {
    // static assignment, descending: CTA c takes segments n_segs-1-c, n_segs-1-c-grid, ...; a segment that waits
    // for its right neighbour waits for a lower (CTA, round) pair, so every wait chain ends
    const int64_t j = p.n_segs - 1 - (int64_t)blockIdx.x - (int64_t)nseg_done * gridDim.x;
    ++nseg_done;
    if (tr && tid == 0) {
      if (nseg_done == 1) tr[1] = gtimer();
      tr[22] = (unsigned long long)nseg_done;
    }
    if (j < 0) break;
    const unsigned long long sb = p.seg_start[j], se = p.seg_start[j + 1];
    const int64_t b = (int64_t)(sb & ~kSegCut), e = (int64_t)(se & ~kSegCut);
    const int64_t lo16 = b & ~int64_t(15), e16 = (e + 15) & ~int64_t(15);
    const int ntl = e > b ? (int)((e16 - lo16 + kSegTile - 1) / kSegTile) : 0;
    auto tile_T0 = [&](int k) { return max(lo16, e16 - (int64_t)(k + 1) * kSegTile); };
    if (tid == 0)
      for (int k = 0; k < min(ntl, kSegStages - 1); ++k) {
        const int64_t T0 = tile_T0(k);
        seg_issue_load<LOSS>(p, sm + k * SegStage::kBytes, &s_full[k], T0, (uint32_t)(e16 - (int64_t)k * kSegTile - T0));
      }
    if (tid == 0) {
      double X = 0.0;
      if (ntl > 0 && (se & kSegCut)) {  // ends inside a rollout: the value at the next segment's first token
        ulonglong2 r = rec_load(p.rec + j + 1);
        while (rec_tag(r) != F_INC) {
          __nanosleep(64);
          r = rec_load(p.rec + j + 1);
        }
        X = rec_x(r);
      }
      s_X = X;
    }
    double wsum = 0.0, wsq = 0.0;
    uint32_t wcnt = 0u;
    double lsum[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    __syncthreads();  // s_X
    for (int k = 0; k < ntl; ++k) {
      const int stg = k % kSegStages;
      uint8_t* st = sm + stg * SegStage::kBytes;
      float* s_r = reinterpret_cast<float*>(st + SegStage::kR);
      float* s_v = reinterpret_cast<float*>(st + SegStage::kV);
      const uint8_t* s_m = st + SegStage::kM;
      const int64_t T0 = tile_T0(k);
      const uint32_t n = (uint32_t)(e16 - (int64_t)k * kSegTile - T0);
      const bool interior = T0 >= b && T0 + n <= e;
      const int64_t c0 = T0 + (int64_t)tid * kSegTPT;
      // this thread's tokens outside the segment or past the tile are identities; its rollout-end bits (half a
      // bitmap word)
      const int64_t te = min(e, T0 + (int64_t)n);
      uint32_t ident = 0u, last = 0u;
      if (!(c0 >= b && c0 + kSegTPT <= te)) {
        for (int q = 0; q < kSegTPT; ++q)
          if (c0 + q < b || c0 + q >= te) ident |= 1u << q;
      }
      mbar_wait(&s_full[stg], (phase >> stg) & 1u);
      phase ^= 1u << stg;
      if (tr && tid == 0 && nseg_done == 1 && k < 8) tr[4 + k] = gtimer();
      if (ident != 0xffffu) {  // this thread's 16 end bits from the stage's bitmap slice; cleared in global memory
        const int64_t ob = c0 - p.base;
        last = (uint32_t)*reinterpret_cast<const uint16_t*>(st + SegStage::kE + ((ob >> 3) - seg_ebyte16(T0, p.base))) &
               ~ident;
        if (last)  // (own bits only: a word can be shared with a neighbouring segment; the bitmap is zero between calls)
          atomicAnd(reinterpret_cast<uint32_t*>(p.ends) + (ob >> 5), ~(last << (int)(((ob >> 4) & 1) * 16)));
      }
      // link bits: token q's successor is unmasked and in the same rollout (16 tokens + the next thread's first)
      uint32_t lkb, onm;  // (onm: masked-in tokens of the segment)
      {
        const uint4 mw = *reinterpret_cast<const uint4*>(s_m + tid * kSegTPT);
        const uint32_t on = nz_bytes4(mw.x) | nz_bytes4(mw.y) << 4 | nz_bytes4(mw.z) << 8 | nz_bytes4(mw.w) << 12;
        const uint32_t nx = s_m[tid * kSegTPT + kSegTPT] ? 1u : 0u;
        lkb = ((on >> 1) | (nx << 15)) & ~last & 0xffffu;
        onm = on & ~ident;
      }
      // pass 1: chunk maps in the per-lane rotated order (conflict-free 128-bit shared reads); a chunk of four
      // linked tokens inside the segment (the common case) takes the select-free path
      // The successor value of chunk ch (the first V of chunk ch + 1) comes from registers: the next chunk in the
      // rotated order is loaded one step ahead (a scalar shared load at the 64-byte thread stride would be a 16-way
      // bank conflict); chunk s's first V is kept for the wrap-around and for pass 2
      const float vn_cross = s_v[tid * kSegTPT + kSegTPT];
      double Hd = 0.0, Hc = 1.0, Td = 0.0, Tc = 1.0;
      float4 r4n = *reinterpret_cast<const float4*>(s_r + tid * kSegTPT + s0 * 4);
      float4 v4n = *reinterpret_cast<const float4*>(s_v + tid * kSegTPT + s0 * 4);
      const float v_s0first = v4n.x;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int ch = (s0 + jj) & 3;
        const float4 r4 = r4n, v4 = v4n;
        if (jj < 3) {
          const int chn = (s0 + jj + 1) & 3;
          r4n = *reinterpret_cast<const float4*>(s_r + tid * kSegTPT + chn * 4);
          v4n = *reinterpret_cast<const float4*>(s_v + tid * kSegTPT + chn * 4);
        }
        const float vnx = ch == 3 ? vn_cross : (jj < 3 ? v4n.x : v_s0first);
        const float rr[4] = {r4.x, r4.y, r4.z, r4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
        const uint32_t l4 = (lkb >> (4 * ch)) & 0xfu, id4 = (ident >> (4 * ch)) & 0xfu;
        double fd = 0.0, fc = 1.0;
        if (l4 == 0xfu && id4 == 0u) {
          double vn = (double)vnx;
#pragma unroll
          for (int kk = 3; kk >= 0; --kk) {
            const double v = (double)vv[kk];
            fd = fma(gld, fd, fma(gamd, vn, (double)rr[kk]) - v);
            vn = v;
          }
          fc = gld4;
        } else {
#pragma unroll
          for (int kk = 3; kk >= 0; --kk) {
            const int q = ch * 4 + kk;
            const bool lk = (lkb >> q) & 1u;
            const float vnext = kk == 3 ? vnx : vv[kk + 1];
            const double dq = (lk ? fma(gamd, (double)vnext, (double)rr[kk]) : (double)rr[kk]) - (double)vv[kk];
            if (!((ident >> q) & 1u)) {
              fd = lk ? fma(gld, fd, dq) : dq;
              fc = lk ? fc * gld : 0.0;
            }
          }
        }
        if (ch >= s0) {
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
      __syncthreads();  // s_warp; every thread has read its successor value (vn_cross)
      double Xd = s_X;
#pragma unroll
      for (int w = NW - 1; w >= 0; --w)
        if (w > wid) Xd = fma(s_warp[w].c, Xd, s_warp[w].d);
      const double Xin = fma(E.c, Xd, E.d);
      double X = fma(Tc, Xin, Td);
      float wa = 0.0f, wa2 = 0.0f;
      uint32_t wn = 0u;
      float vprev = v_s0first;  // the first V of the chunk processed before (chunk ch + 1); position 0: chunk s
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int ch = (s0 - 1 - jj) & 3;
        if (jj == s0) X = Xin;
        const int i0 = tid * kSegTPT + ch * 4;
        const float4 r4 = *reinterpret_cast<const float4*>(s_r + i0);
        const float4 v4 = *reinterpret_cast<const float4*>(s_v + i0);
        const float vnx = ch == 3 ? vn_cross : vprev;
        vprev = v4.x;
        const float rr[4] = {r4.x, r4.y, r4.z, r4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
        float oa[4], orr[4];
        const uint32_t l4 = (lkb >> (4 * ch)) & 0xfu, id4 = (ident >> (4 * ch)) & 0xfu;
        if (l4 == 0xfu && id4 == 0u) {
          double vn = (double)vnx;
#pragma unroll
          for (int kk = 3; kk >= 0; --kk) {
            const double v = (double)vv[kk];
            X = fma(gld, X, fma(gamd, vn, (double)rr[kk]) - v);
            oa[kk] = (float)X;
            orr[kk] = (float)(X + v);
            vn = v;
          }
        } else {
#pragma unroll
          for (int kk = 3; kk >= 0; --kk) {
            const int q = ch * 4 + kk;
            const bool lk = (lkb >> q) & 1u;
            const float vnext = kk == 3 ? vnx : vv[kk + 1];
            const double dq = (lk ? fma(gamd, (double)vnext, (double)rr[kk]) : (double)rr[kk]) - (double)vv[kk];
            const double A = lk ? fma(gld, X, dq) : dq;
            X = ((ident >> q) & 1u) ? X : A;
            oa[kk] = (float)X;
            orr[kk] = (float)(X + (double)vv[kk]);
          }
        }
        if (WHITEN) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float mw = ((onm >> (ch * 4 + kk)) & 1u) ? 1.0f : 0.0f;
            wa = fmaf(mw, oa[kk], wa);
            wa2 = fmaf(mw * oa[kk], oa[kk], wa2);
          }
          wn += __popc((onm >> (4 * ch)) & 0xfu);
        }
        *reinterpret_cast<float4*>(s_r + i0) = make_float4(oa[0], oa[1], oa[2], oa[3]);
        if (interior) {  // (every successor value of this thread is in registers: R over V at once)
          *reinterpret_cast<float4*>(s_v + i0) = make_float4(orr[0], orr[1], orr[2], orr[3]);
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (!((ident >> (ch * 4 + kk)) & 1u)) {
              if (!LOSS || p.adv) p.adv[c0 + ch * 4 + kk] = oa[kk];
              p.ret[c0 + ch * 4 + kk] = orr[kk];
            }
          }
        }
      }
      if (WHITEN) {
        wsum += (double)wa;
        wsq += (double)wa2;
        wcnt += wn;
      }
      fence_proxy_async_smem();
      __syncthreads();  // the tile's A and R in shared memory; every thread has read s_X
      if (tr && tid == 0 && nseg_done == 1 && k < 8) tr[12 + k] = gtimer();
      if (tid == 0) {
        s_X = X;  // thread 0's first token: the value at the tile's first segment token = the next tile's carry
        if (interior) {
          if (!LOSS || p.adv) tma_store_1d(p.adv + T0, s_r, 4u * n);
          tma_store_1d(p.ret + T0, s_v, 4u * n);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // (one group per tile, possibly empty)
        if (k + kSegStages - 1 < ntl) {  // refill the previous tile's stage once its stores have read it
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          const int kn = k + kSegStages - 1;
          const int64_t T0n = tile_T0(kn);
          seg_issue_load<LOSS>(p, sm + (kn % kSegStages) * SegStage::kBytes, &s_full[kn % kSegStages], T0n,
                               (uint32_t)(e16 - (int64_t)kn * kSegTile - T0n));
        }
      }
      if (LOSS) {
        float lpg = 0.0f, lkl = 0.0f, lakl = 0.0f;
        uint32_t lclip = 0u, lcnt = 0u;
        gae_tile_loss<kSegThreads>(p, T0, n, b, e, s_r, s_m, lpg, lkl, lakl, lclip, lcnt);
        lsum[0] += (double)lpg;
        lsum[1] += (double)lkl;
        lsum[2] += (double)lakl;
        lsum[3] += (double)lclip;
        lsum[4] += (double)lcnt;
      }
      // (no barrier here: the next refill targets this tile's stage only after the next tile's barriers)
    }
    if (tr && tid == 0 && nseg_done == 1) {
      tr[2] = (unsigned long long)j;
      tr[3] = (unsigned long long)ntl;
      tr[20] = gtimer();
    }
    if (tid == 0) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // (the stores complete before the CTA exits)
      rec_store(p.rec + j, s_X, 0.0f, F_INC);  // the value at b: the carry of segment j-1 if b cuts a rollout
    }
    if (WHITEN || LOSS) {  // per-segment partials: fixed-shape block reduction
      double v[5];
      if (LOSS) {
#pragma unroll
        for (int q = 0; q < 5; ++q) v[q] = warp_sum(lsum[q]);
      } else {
        v[0] = warp_sum(wsum);
        v[1] = warp_sum(wsq);
        v[2] = (double)warp_sum(wcnt);
        v[3] = v[4] = 0.0;
      }
      if (lane == 0)
        for (int q = 0; q < 5; ++q) s_red[wid][q] = v[q];
      __syncthreads();
      if (tid < (LOSS ? 5 : 3)) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += s_red[w][tid];
        if (LOSS) p.lpart[(int64_t)tid * p.n_segs + j] = t;
        else p.part[(int64_t)tid * p.n_segs + j] = t;
      }
    }
  }
  if (tr && tid == 0) tr[21] = gtimer();
}

// ---- whitening sums: fixed-shape reduction of the per-tile partials ---------------------------------------------
__global__ void __launch_bounds__(256) gae_finish_kernel(const double* __restrict__ part, int64_t n_tiles,
                                                         double* __restrict__ whiten) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (programmatic dependent of the scan)
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
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (programmatic dependent of the scan)
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
  size_t ticket, ends, rec, part, lpart, segs, bytes;
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
  w.segs = w.lpart + al(40 * size_t(cap_tiles));
  w.bytes = w.segs + al(8 * size_t(cap_tiles + 1));
  return w;
}
// tiles needed for a span (tile count depends on token_base & 15 as well: size for the worst case)
int64_t gae_tiles_needed(int64_t token_span) { return (token_span + 15) / kGaeMinTile + 2; }
// the largest capacity whose layout fits in ws_bytes (the caller's buffer size fixes the layout)
GaeWs gae_ws_layout_fit(size_t ws_bytes) {
  int64_t cap = (int64_t)(ws_bytes / (kGaeMinTile / 8 + 16 + 24 + 40 + 8));  // an upper bound; step down to the fit
  while (cap > 0 && gae_ws_layout_cap(cap).bytes > ws_bytes) --cap;
  return gae_ws_layout_cap(cap);
}

// Tuning knob (benchmarking only): DFX_GAE_VARIANT = seg (rollout-aligned segments: the default of dfx_gae) |
// lb (one 4096-token tile per CTA with a decoupled look-back: the default of the fused dfx_gae_ppo_loss, whose
// per-tile loss phase needs the latency hiding of 5 independent CTAs per SM) | lb64 (64 x 32)
inline int gae_variant(bool fused) {
  static const int v = [] {
    const char* e = std::getenv("DFX_GAE_VARIANT");
    if (!e) return -1;
    const std::string s(e);
    return s == "lb" ? 1 : s == "lb64" ? 2 : 0;
  }();
  return v >= 0 ? v : (fused ? 1 : 0);
}

// one 256-thread CTA as a programmatic dependent of the previous kernel (the finish kernels)
template <typename... A>
void gae_pdl_launch(void (*kernel)(A...), cudaStream_t st, A... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <typename K>
void gae_set_smem(K kernel, uint32_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int THREADS, int MINB, bool LOSS = false>
void gae_launch_smem(GaeParams& p, cudaStream_t st) {
  using L = SmemTile<THREADS>;
  constexpr uint32_t kSmem = L::kBytes;
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



// segments: about one per resident CTA (at least one tile); the prep kernel writes their bounds
template <bool LOSS>
void gae_seg_plan(GaeParams& p, unsigned long long* seg_start) {
  static thread_local int cached_dev = -1, resident = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  constexpr uint32_t kSmem = kSegStages * SegStage::kBytes;
  if (dev != cached_dev) {
    int sms = 0, per_sm = 0;
    gae_set_smem(gae_seg_kernel<true, LOSS>, kSmem);
    gae_set_smem(gae_seg_kernel<false, LOSS>, kSmem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_seg_kernel<false, LOSS>, kSegThreads, kSmem);
    resident = sms * std::max(per_sm, 1);
    cached_dev = dev;
  }
  const int64_t span = p.end - p.begin;
  p.seg_len = std::max<int64_t>(kSegTile, (span + resident - 1) / resident);  // about one segment per CTA
  p.n_segs = (span + p.seg_len - 1) / p.seg_len;
  p.n_tiles = resident;  // (grid)
  p.seg_start = seg_start;
}

// DFX_GAE_TRACE=1 (diagnostics only, synchronises): per-CTA phase times of the segment kernel to stderr
inline void gae_seg_trace_report(const GaeParams& p, unsigned grid, cudaStream_t st) {
  std::vector<unsigned long long> h(size_t(grid) * 32);
  cudaStreamSynchronize(st);
  cudaMemcpy(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, tend = 0;
  for (unsigned c = 0; c < grid; ++c) {
    t0 = std::min(t0, h[32 * c]);
    tend = std::max(tend, h[32 * c + 21]);
  }
  auto med = [&](int slot, bool only_real) {
    std::vector<double> v;
    for (unsigned c = 0; c < grid; ++c)
      if (h[32 * c + slot] && (!only_real || h[32 * c + 3] > 0)) v.push_back((h[32 * c + slot] - t0) * 1e-3);
    if (v.empty()) return -1.0;
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  std::fprintf(stderr, "[gae trace] grid %u n_segs %lld S %lld span %.3f us | median us: entry %.2f claim %.2f", grid,
               (long long)p.n_segs, (long long)p.seg_len, (tend - t0) * 1e-3, med(0, false), med(1, false));
  for (int k = 0; k < 8; ++k) std::fprintf(stderr, " | t%d ready %.2f done %.2f", k, med(4 + k, true), med(12 + k, true));
  std::fprintf(stderr, " | seg end %.2f exit %.2f\n", med(20, true), med(21, false));
}

template <bool LOSS>
void gae_launch_seg(GaeParams& p, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)std::min<int64_t>(p.n_segs, p.n_tiles));
  cfg.blockDim = dim3(kSegThreads);
  cfg.dynamicSmemBytes = kSegStages * SegStage::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const bool trace = std::getenv("DFX_GAE_TRACE") != nullptr;
  static unsigned long long* tbuf = nullptr;
  if (trace) {
    if (!tbuf) cudaMalloc(&tbuf, 32 * 8 * 4096);
    cudaMemsetAsync(tbuf, 0, 32 * 8 * cfg.gridDim.x, st);
    p.trace = tbuf;
  }
  if (p.whiten) cudaLaunchKernelEx(&cfg, gae_seg_kernel<true, LOSS>, p);
  else cudaLaunchKernelEx(&cfg, gae_seg_kernel<false, LOSS>, p);
  if (trace) gae_seg_trace_report(p, cfg.gridDim.x, st);
  p.trace = nullptr;
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
  const int v = gae_variant(false);
  if (v == 0) gae_seg_plan<false>(p, reinterpret_cast<unsigned long long*>(w + wl.segs));
  gae_prep_kernel<<<(unsigned)((p.n_seq + 1 + 255) / 256), 256, 0, stream>>>(p);
  DFX_LAUNCH_CHECK("gae_prep_kernel");
  switch (v) {
    case 1: gae_launch_smem<128, 5>(p, stream); break;
    case 2: gae_launch_smem<64, 8>(p, stream); break;
    default: gae_launch_seg<false>(p, stream); break;
  }
  DFX_LAUNCH_CHECK("gae scan");
  if (whiten) {
    gae_pdl_launch(gae_finish_kernel, stream, (const double*)p.part, (int64_t)(v == 0 ? p.n_segs : p.n_tiles),
                   whiten);
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
  const int v = gae_variant(true);
  if (v == 0) gae_seg_plan<true>(p, reinterpret_cast<unsigned long long*>(w + wl.segs));
  gae_prep_loss_kernel<<<(unsigned)((p.n_seq + 1 + 7) / 8), 256, 0, stream>>>(p);
  DFX_LAUNCH_CHECK("gae_prep_loss_kernel");
  switch (v) {
    case 1: gae_launch_smem<128, 5, true>(p, stream); break;
    case 2: gae_launch_smem<64, 8, true>(p, stream); break;
    default: gae_launch_seg<true>(p, stream); break;
  }
  DFX_LAUNCH_CHECK("gae scan<loss>");
  gae_pdl_launch(gae_loss_finish_kernel, stream, (const double*)p.lpart, (int64_t)(v == 0 ? p.n_segs : p.n_tiles),
                 (const uint8_t*)p.seq_has, p.n_seq, cfg->beta, out);
  DFX_LAUNCH_CHECK("gae_loss_finish_kernel");
  return DFX_OK;
}

}  // extern "C"
