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
// Single-pass decoupled look-back scan (CUB-style) over 4096-token CTA tiles claimed in decreasing order:
// each thread owns 16 contiguous tokens (four 128-bit loads per stream), composes their maps, a block suffix
// scan (warp shuffles + shared memory) gives the tile aggregate, warp 0 publishes it and resolves the tile's
// carry-in with a warp-parallel look-back over the following tiles, and every thread re-walks its tokens.
// Tile state is published as one 16-byte record per tile (no fences; see rec_store). Scan arithmetic is f64,
// outputs f32; masked whitening sums are per-tile partials reduced in tile order by the last CTA.
// HBM-bound: 17 B/token (r, V, mask in; A, R out).
#include <algorithm>

#include "common.cuh"

namespace dfx {

constexpr int kGaeThreads = 256;
constexpr int kGaeTpt = 16;                          // tokens per thread
constexpr int kGaeTile = kGaeThreads * kGaeTpt;      // 4096 tokens

struct GaeParams {
  const int64_t* cu;
  int64_t n_seq;
  int64_t begin, end;             // token span [begin, end)
  int64_t base;                   // tile origin (begin & ~15)
  int64_t n_tiles;
  const float* rew;
  const float* val;
  const uint8_t* mask;
  double gamma, gl;
  float* adv;
  float* ret;
  double* whiten;                 // nullable [3]
  // workspace
  unsigned long long* ticket;     // [0] reverse tile ticket, [1] finished CTAs, [2] epoch
  ulonglong2* rec;                // [n_tiles] published tile state
  double* part;                   // [3][n_tiles] whitening partials
};

struct Aff {
  double d, c;  // X -> d + c X
};
// (f o g)(X) = f(g(X))
__device__ __forceinline__ Aff compose(const Aff& f, const Aff& g) { return {fma(f.c, g.d, f.d), f.c * g.c}; }

// A tile publishes its state as ONE 16-byte record {f64 x ; f32 c ; u32 tag}, written and polled with single
// relaxed 128-bit accesses, so value and status can never be seen out of order and no fence is needed (on
// sm_100 a gpu-scope fence or acquire invalidates L1: CCTL.IVALL, measured as the top stall of a fenced
// version). tag = (epoch << 2) | state: 1 = aggregate map (x = d, c), 2 = inclusive (x = A at the tile's start).
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

// shared-memory stage: one tile of r (f32), V (f32), mask (u8)
constexpr uint32_t kStR = 0, kStV = kGaeTile * 4, kStM = kGaeTile * 8, kStage = kGaeTile * 9;
constexpr uint32_t kGaeSmem = 2 * kStage;

// TMA: bulk-load tile `tile` into stage buffer `st` (thread 0)
__device__ __forceinline__ void gae_issue(const GaeParams& p, uint8_t* st, uint64_t* bar, int64_t tile) {
  const int64_t T0 = p.base + tile * kGaeTile;
  const int64_t readable = ((p.end + 15) & ~int64_t(15)) - T0;
  const uint32_t n = (uint32_t)min((int64_t)kGaeTile, readable);  // multiple of 16 tokens
  mbar_arrive_expect_tx(bar, 9u * n);
  tma_load_1d(st + kStR, p.rew + T0, 4u * n, bar);
  tma_load_1d(st + kStV, p.val + T0, 4u * n, bar);
  tma_load_1d(st + kStM, p.mask + T0, n, bar);
}

__global__ void __launch_bounds__(kGaeThreads, 2) gae_kernel(GaeParams p) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ long long s_next;
  __shared__ uint32_t s_last[kGaeTile / 32 + 1];   // bit t: token T0+t is the last token of its rollout
  __shared__ Aff s_warp[kGaeThreads / 32];
  __shared__ double s_X;
  __shared__ double s_red[kGaeThreads / 32][3];
  __shared__ long long s_tile;
  __shared__ bool is_last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned int epoch = (unsigned int)*((volatile unsigned long long*)(p.ticket + 2));
  const unsigned int F_AGG = (epoch << 2) | 1u, F_INC = (epoch << 2) | 2u;

  // two-stage TMA ring: tile i+1 streams into shared memory while tile i is scanned
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
    const long long k0 = (long long)atomicAdd(p.ticket, 1ull);
    s_next = k0;
    if (k0 < p.n_tiles) gae_issue(p, dsm, &s_bar[0], p.n_tiles - 1 - k0);
  }
  __syncthreads();
  for (uint32_t it = 0;; ++it) {
    const long long k = s_next;
    if (k >= p.n_tiles) break;
    const uint32_t stg = it & 1u;
    uint8_t* st = dsm + stg * kStage;
    if (tid == 0) s_tile = k;
    for (int i = tid; i <= kGaeTile / 32; i += kGaeThreads) s_last[i] = 0u;
    __syncthreads();  // everyone has read s_next
    if (tid == 0) {  // claim and prefetch the next tile into the other stage (released at the end of it-1)
      const long long kn = (long long)atomicAdd(p.ticket, 1ull);
      s_next = kn;
      if (kn < p.n_tiles) {
        fence_proxy_async_smem();
        gae_issue(p, dsm + (stg ^ 1u) * kStage, &s_bar[stg ^ 1u], p.n_tiles - 1 - kn);
      }
    }
    const int64_t tile = p.n_tiles - 1 - k;  // decreasing: the tiles to the right were claimed earlier
    const int64_t T0 = p.base + tile * kGaeTile;
    const int64_t T1 = min(T0 + (int64_t)kGaeTile, p.end);

    // rollout ends inside [T0, T1): warp 0 finds the first rollout ending at or after T0, then the block marks
    // every rollout end e = cu[s+1]-1 < T1
    if (wid == 0) {
      // 32-ary lower bound: count of rollouts with cu[s+1] <= T0 (a prefix, cu is nondecreasing)
      int64_t lo = 0, hi = p.n_seq;  // invariant: true below lo, false at and above hi
      while (lo < hi) {
        const int64_t step = (hi - lo + 31) >> 5;
        const int64_t sp = lo + (int64_t)lane * step;
        const bool pred = sp < hi && __ldg(p.cu + sp + 1) <= T0;
        const int cnt = __popc(__ballot_sync(kFull, pred));
        if (cnt == 0) break;  // false at lo
        const int64_t nlo = lo + (int64_t)(cnt - 1) * step + 1;
        const int64_t nhi = lo + (int64_t)cnt * step;
        lo = nlo;
        if (cnt < 32 && nhi < hi) hi = nhi;
      }
      if (lane == 0) s_X = __longlong_as_double((long long)lo);  // stash the first rollout index
    }
    __syncthreads();
    {
      const int64_t s_first = (int64_t)__double_as_longlong(s_X);
      for (int64_t sq = s_first + tid; sq < p.n_seq; sq += kGaeThreads) {
        const int64_t e = __ldg(p.cu + sq + 1) - 1;
        if (e >= T1) break;
        if (e >= T0 && e >= __ldg(p.cu + sq)) atomicOr(&s_last[(e - T0) >> 5], 1u << ((e - T0) & 31));
      }
    }
    // this thread's 16 tokens, from the tile's shared-memory stage (tokens past the span are never used)
    const int64_t c0 = T0 + (int64_t)tid * kGaeTpt;
    mbar_wait(&s_bar[stg], (it >> 1) & 1u);
    float r[kGaeTpt], v[kGaeTpt];
    uint32_t mb = 0;
    {
      const float4* sr = reinterpret_cast<const float4*>(st + kStR) + tid * (kGaeTpt / 4);
      const float4* sv = reinterpret_cast<const float4*>(st + kStV) + tid * (kGaeTpt / 4);
#pragma unroll
      for (int q = 0; q < kGaeTpt; q += 4) {
        const float4 a = sr[q / 4];
        const float4 bb = sv[q / 4];
        r[q] = a.x; r[q + 1] = a.y; r[q + 2] = a.z; r[q + 3] = a.w;
        v[q] = bb.x; v[q + 1] = bb.y; v[q + 2] = bb.z; v[q + 3] = bb.w;
      }
      const uint4 mk = reinterpret_cast<const uint4*>(st + kStM)[tid];
      const uint32_t w4[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
      for (int q = 0; q < kGaeTpt; ++q) mb |= (((w4[q >> 2] >> (8 * (q & 3))) & 0xffu) ? 1u : 0u) << q;
    }
    // the token after this thread's chunk: next thread's first token, or (last thread) token T0 + kGaeTile
    float vn = __shfl_down_sync(kFull, v[0], 1);
    uint32_t mn = __shfl_down_sync(kFull, mb & 1u, 1);
    __syncthreads();  // s_last complete
    if (lane == 31) {
      const int64_t tn = c0 + kGaeTpt;
      if (wid == kGaeThreads / 32 - 1) {
        vn = tn < p.end ? __ldg(p.val + tn) : 0.0f;
        mn = tn < p.end ? (__ldg(p.mask + tn) ? 1u : 0u) : 0u;
      } else {
        vn = 0.0f;  // filled from shared memory below
        mn = 0u;
      }
    }
    // cross-warp neighbours: first token of the next warp's lane 0
    __shared__ float s_v0[kGaeThreads / 32];
    __shared__ uint32_t s_m0[kGaeThreads / 32];
    if (lane == 0) {
      s_v0[wid] = v[0];
      s_m0[wid] = mb & 1u;
    }
    __syncthreads();
    if (lane == 31 && wid < kGaeThreads / 32 - 1) {
      vn = s_v0[wid + 1];
      mn = s_m0[wid + 1];
    }
    const uint32_t lastbits = (s_last[(tid * kGaeTpt) >> 5] >> ((tid * kGaeTpt) & 31)) & 0xffffu;

    auto tok = [&](int q) -> Aff {
      const int64_t t = c0 + q;
      if (t < p.begin || t >= p.end) return Aff{0.0, 1.0};  // outside the batch: identity
      const bool last = (lastbits >> q) & 1u;
      const double m1 = last ? 0.0 : (double)(q < kGaeTpt - 1 ? ((mb >> (q + 1)) & 1u) : mn);
      const double vv1 = last ? 0.0 : (double)(q < kGaeTpt - 1 ? v[q + 1] : vn);
      return Aff{fma(p.gamma * m1, vv1, (double)r[q]) - (double)v[q], p.gl * m1};
    };
    Aff F = tok(kGaeTpt - 1);
#pragma unroll
    for (int q = kGaeTpt - 2; q >= 0; --q) F = compose(tok(q), F);
    // block suffix scan: warp level, then across warps
    Aff S = F;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double od = __shfl_down_sync(kFull, S.d, o), oc = __shfl_down_sync(kFull, S.c, o);
      if (lane + o < 32) S = compose(S, Aff{od, oc});
    }
    if (lane == 0) s_warp[wid] = S;
    Aff E{__shfl_down_sync(kFull, S.d, 1), __shfl_down_sync(kFull, S.c, 1)};
    if (lane == 31) E = Aff{0.0, 1.0};
    __syncthreads();
    // tile aggregate and carry-in (warp 0)
    if (wid == 0) {
      Aff tot{0.0, 1.0};
      for (int w = kGaeThreads / 32 - 1; w >= 0; --w) tot = compose(s_warp[w], tot);
      double X = 0.0;
      // A tile containing a rollout end has c == 0: its inclusive value does not depend on the tiles to its
      // right, so it is published at once (tiles to the left stop their look-back here). The carry X is still
      // resolved below: tokens after the tile's last rollout end need it.
      if (lane == 0) rec_store(p.rec + tile, tot.d, (float)tot.c, tot.c == 0.0 ? F_INC : F_AGG);
      if (tile < p.n_tiles - 1) {
        Aff G{0.0, 1.0};
        for (int64_t j0 = tile + 1;; j0 += 32) {
          const int64_t j = j0 + lane;
          const bool valid = j < p.n_tiles;
          ulonglong2 rr = make_ulonglong2(0ull, (unsigned long long)F_INC << 32);  // past the end: A = 0
          if (valid) rr = rec_load(p.rec + j);
          for (;;) {
            const unsigned int tg = rec_tag(rr);
            const uint32_t inc_m = __ballot_sync(kFull, tg == F_INC);
            const uint32_t rdy_m = __ballot_sync(kFull, tg == F_AGG || tg == F_INC);
            const uint32_t need = inc_m ? ((inc_m & (0u - inc_m)) << 1) - 1u : kFull;
            if ((rdy_m & need) == need) break;
            if (valid && tg != F_AGG && tg != F_INC) rr = rec_load(p.rec + j);
          }
          const uint32_t inc_m = __ballot_sync(kFull, rec_tag(rr) == F_INC);
          const int first = inc_m ? __ffs(inc_m) - 1 : 32;
          Aff a{0.0, 1.0};
          if (lane < first) a = Aff{rec_x(rr), rec_c(rr)};
          else if (lane == first) a = Aff{rec_x(rr), 0.0};
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double od = __shfl_down_sync(kFull, a.d, o), oc = __shfl_down_sync(kFull, a.c, o);
            if (lane + o < 32) a = compose(a, Aff{od, oc});
          }
          G = compose(G, Aff{__shfl_sync(kFull, a.d, 0), __shfl_sync(kFull, a.c, 0)});
          if (first < 32) {
            X = G.d;
            break;
          }
        }
      }
      if (lane == 0) {
        rec_store(p.rec + tile, fma(tot.c, X, tot.d), 0.0f, F_INC);
        s_X = X;
      }
    }
    __syncthreads();
    // carry into this thread: (warps after mine) then (lanes after mine) applied to the tile carry
    double X = s_X;
    for (int w = kGaeThreads / 32 - 1; w > wid; --w) X = fma(s_warp[w].c, X, s_warp[w].d);
    X = fma(E.c, X, E.d);
    double wa = 0.0, wa2 = 0.0, wm = 0.0;
    float oa[kGaeTpt], orr[kGaeTpt];
#pragma unroll
    for (int q = kGaeTpt - 1; q >= 0; --q) {
      const Aff f = tok(q);
      X = fma(f.c, X, f.d);
      oa[q] = (float)X;
      orr[q] = (float)(X + (double)v[q]);
      const int64_t t = c0 + q;
      if (t >= p.begin && t < p.end && ((mb >> q) & 1u)) {
        wa += X;
        wa2 += X * X;
        wm += 1.0;
      }
    }
    if (c0 >= p.begin && c0 + kGaeTpt <= p.end) {
#pragma unroll
      for (int q = 0; q < kGaeTpt; q += 4) {
        *reinterpret_cast<float4*>(p.adv + c0 + q) = make_float4(oa[q], oa[q + 1], oa[q + 2], oa[q + 3]);
        *reinterpret_cast<float4*>(p.ret + c0 + q) = make_float4(orr[q], orr[q + 1], orr[q + 2], orr[q + 3]);
      }
    } else {
#pragma unroll
      for (int q = 0; q < kGaeTpt; ++q) {
        const int64_t t = c0 + q;
        if (t >= p.begin && t < p.end) {
          p.adv[t] = oa[q];
          p.ret[t] = orr[q];
        }
      }
    }
    if (p.whiten) {
      wa = warp_sum(wa);
      wa2 = warp_sum(wa2);
      wm = warp_sum(wm);
      if (lane == 0) {
        s_red[wid][0] = wa;
        s_red[wid][1] = wa2;
        s_red[wid][2] = wm;
      }
      __syncthreads();
      if (tid < 3) {
        double t3 = 0.0;
        for (int w = 0; w < kGaeThreads / 32; ++w) t3 += s_red[w][tid];
        p.part[(int64_t)tid * p.n_tiles + tile] = t3;
      }
    }
    __syncthreads();
  }

  // last CTA out: reduce the whitening partials in tile order, reset the ticket, advance the epoch
  if (tid == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(p.ticket + 1, 1ull);
    is_last = done == (unsigned long long)gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (p.whiten) {
    double tot[3] = {0.0, 0.0, 0.0};
    for (int64_t i = tid; i < p.n_tiles; i += kGaeThreads)
#pragma unroll
      for (int q = 0; q < 3; ++q) tot[q] += __ldcg(p.part + (int64_t)q * p.n_tiles + i);
#pragma unroll
    for (int q = 0; q < 3; ++q) tot[q] = warp_sum(tot[q]);
    if (lane == 0)
      for (int q = 0; q < 3; ++q) s_red[wid][q] = tot[q];
    __syncthreads();
    if (tid == 0) {
      double t3[3] = {0.0, 0.0, 0.0};
      for (int w = 0; w < kGaeThreads / 32; ++w)
        for (int q = 0; q < 3; ++q) t3[q] += s_red[w][q];
      for (int q = 0; q < 3; ++q) p.whiten[q] = t3[q];
    }
  }
  if (tid == 0) {
    p.ticket[0] = 0ull;
    p.ticket[1] = 0ull;
    p.ticket[2] = (unsigned long long)((epoch + 1u) & 0x3fffffffu);
  }
}

int64_t gae_tiles(int64_t token_base, int64_t token_span) {
  const int64_t base = token_base & ~int64_t(15);
  return (token_base + token_span - base + kGaeTile - 1) / kGaeTile;
}

size_t gae_ws_bytes(int64_t n_tiles) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return al(3 * sizeof(unsigned long long)) + al(16 * size_t(n_tiles)) + al(24 * size_t(n_tiles));
}

}  // namespace dfx

using namespace dfx;

extern "C" {

size_t dfx_gae_workspace_bytes(int64_t n_rollouts, int64_t token_span) {
  (void)n_rollouts;
  // tile count depends on token_base & 15 as well: size for the worst case (one extra tile)
  return gae_ws_bytes((token_span + 15) / kGaeTile + 2);
}

dfx_status dfx_gae(const dfx_packed* b, int64_t token_base, int64_t token_span, double gamma, double lam, float* adv,
                   float* ret, double* whiten, void* workspace, size_t ws_bytes, dfx_stream stream) {
  if (!b || !b->cu_seqlens || !b->token_reward || !b->value_tok || !b->mask || !adv || !ret)
    return fail(DFX_INVALID_ARGUMENT, "dfx_gae: packed batch lacks cu_seqlens/token_reward/value_tok/mask or null output");
  if (b->n_rollouts <= 0 || token_span <= 0) {
    if (whiten) DFX_CUDA(cudaMemsetAsync(whiten, 0, 3 * sizeof(double), stream));
    return DFX_OK;
  }
  GaeParams p{};
  p.cu = b->cu_seqlens;
  p.n_seq = b->n_rollouts;
  p.begin = token_base;
  p.end = token_base + token_span;
  p.base = token_base & ~int64_t(15);
  p.n_tiles = gae_tiles(token_base, token_span);
  const size_t need = gae_ws_bytes(p.n_tiles);
  if (!workspace || ws_bytes < need) return fail(DFX_INVALID_ARGUMENT, "dfx_gae: workspace too small");
  char* w = static_cast<char*>(workspace);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  p.ticket = reinterpret_cast<unsigned long long*>(w);
  w += al(3 * sizeof(unsigned long long));
  p.rec = reinterpret_cast<ulonglong2*>(w);
  w += al(16 * size_t(p.n_tiles));
  p.part = reinterpret_cast<double*>(w);
  p.rew = b->token_reward;
  p.val = b->value_tok;
  p.mask = b->mask;
  p.gamma = gamma;
  p.gl = gamma * lam;
  p.adv = adv;
  p.ret = ret;
  p.whiten = whiten;
  static thread_local int cached_dev = -1, cached_blocks = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    int sms = 0, per_sm = 0;
    DFX_CUDA(cudaFuncSetAttribute(gae_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGaeSmem));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_kernel, kGaeThreads, kGaeSmem);
    cached_blocks = sms * (per_sm > 0 ? per_sm : 1);
    cached_dev = dev;
  }
  const int64_t grid = std::min<int64_t>(cached_blocks, p.n_tiles);
  gae_kernel<<<(unsigned)grid, kGaeThreads, kGaeSmem, stream>>>(p);
  DFX_LAUNCH_CHECK("gae_kernel");
  return DFX_OK;
}

}  // extern "C"
