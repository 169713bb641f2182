// gae.cu -- GAE as a reverse affine scan over packed variable-length rollouts.
//
// The reference has no GAE; it fills the PPO node
// advantage_compute / func ppo_advantage slot (distflow/dag.hpp:333-334).
// Convention (oracle/dfx_oracle.h dfo_gae):
//   m1 = t+1<L ? mask[t+1] : 0 ; v1 = t+1<L ? V[t+1] : 0
//   delta_t = r_t + gamma*m1*v1 - V_t ; A_t = delta_t + gamma*lam*m1*A_{t+1} ; R_t = A_t + V_t
// Each token is the affine map f_t(X) = delta_t + c_t X (c_t = gamma*lam*m1);
// A_t = (f_t o f_{t+1} o ... )(0). One CTA per rollout walks 2048-token tiles
// from the end: each thread composes the maps of its 8 contiguous tokens, a
// warp-shuffle + shared-memory suffix scan composes across threads, and each
// thread re-walks its tokens with its exact carry-in. All scan arithmetic is
// f64 (B200 FP64 runs at half the FP32 rate, far above this kernel's need);
// outputs are stored f32. HBM-bound: 17 B/token.
#include "common.cuh"

namespace dfx {

constexpr int kGaeThreads = 256;
constexpr int kGaeTpt = 8;                           // tokens per thread (one 8-aligned chunk)

struct GaeParams {
  const int64_t* cu;
  int64_t n_seq;
  const float* rew;
  const float* val;
  const uint8_t* mask;
  double gamma, gl;
  float* adv;
  float* ret;
  double* blk;           // [n_seq][3] whitening partials
  unsigned int* ticket;  // zero on entry, restored
  double* whiten;        // nullable [3]
};

struct Aff {
  double d, c;  // X -> d + c X
};
// (f o g)(X) = f(g(X))
__device__ __forceinline__ Aff compose(const Aff& f, const Aff& g) { return {fma(f.c, g.d, f.d), f.c * g.c}; }

// affine map of token k of the thread's chunk (m1/v1 of the last token come
// from the next chunk's first token)
__device__ __forceinline__ Aff tok_map(const GaeParams& p, const float (&r)[kGaeTpt], const float (&v)[kGaeTpt],
                                       uint32_t mb, int k, double m_next, double v_next) {
  const double m1 = k == kGaeTpt - 1 ? m_next : (double)((mb >> (k + 1)) & 1u);
  const double v1 = k == kGaeTpt - 1 ? v_next : (double)v[k + 1];
  return {fma(p.gamma * m1, v1, (double)r[k]) - (double)v[k], p.gl * m1};
}

__global__ void __launch_bounds__(kGaeThreads, 4) gae_kernel(GaeParams p) {
  __shared__ double s_first_m[kGaeThreads + 1];
  __shared__ double s_first_v[kGaeThreads + 1];
  __shared__ Aff s_warp[kGaeThreads / 32];
  __shared__ double s_carryA;
  __shared__ double s_red[(kGaeThreads / 32) * 3];
  __shared__ bool is_last;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t s = blockIdx.x;
  const int64_t a = p.cu[s], b = p.cu[s + 1];
  double wsA = 0.0, wsA2 = 0.0, wsm = 0.0;

  if (b > a) {
    const int64_t c_first = a >> 3, c_last = (b - 1) >> 3;  // absolute 8-token chunks
    if (tid == 0) {
      s_first_m[kGaeThreads] = 0.0;  // beyond the rollout: m = 0, V = 0
      s_first_v[kGaeThreads] = 0.0;
      s_carryA = 0.0;
    }
    for (int64_t cb = c_last - (kGaeThreads - 1);; cb -= kGaeThreads) {
      const int64_t c = cb + tid;
      const int64_t t0 = c * kGaeTpt;
      float r[kGaeTpt], v[kGaeTpt];
      uint32_t mb = 0;  // bit k = mask of token t0+k
      const bool any = (c >= c_first) && (c <= c_last);
      if (any) {
        const float4 r0 = __ldg(reinterpret_cast<const float4*>(p.rew + t0));
        const float4 r1 = __ldg(reinterpret_cast<const float4*>(p.rew + t0 + 4));
        const float4 v0 = __ldg(reinterpret_cast<const float4*>(p.val + t0));
        const float4 v1 = __ldg(reinterpret_cast<const float4*>(p.val + t0 + 4));
        const uint2 mk = __ldg(reinterpret_cast<const uint2*>(p.mask + t0));
        r[0] = r0.x; r[1] = r0.y; r[2] = r0.z; r[3] = r0.w; r[4] = r1.x; r[5] = r1.y; r[6] = r1.z; r[7] = r1.w;
        v[0] = v0.x; v[1] = v0.y; v[2] = v0.z; v[3] = v0.w; v[4] = v1.x; v[5] = v1.y; v[6] = v1.z; v[7] = v1.w;
#pragma unroll
        for (int k = 0; k < kGaeTpt; ++k) {
          const uint32_t word = k < 4 ? mk.x : mk.y;
          mb |= (((word >> (8 * (k & 3))) & 0xffu) ? 1u : 0u) << k;
        }
      }
#pragma unroll
      for (int k = 0; k < kGaeTpt; ++k) {
        const int64_t t = t0 + k;
        if (!any || t < a || t >= b) {  // outside the rollout: m = 0, V = 0, r = 0
          r[k] = 0.0f;
          v[k] = 0.0f;
          mb &= ~(1u << k);
        }
      }
      __syncthreads();  // previous tile finished reading s_first_* / s_carryA
      s_first_m[tid] = (double)(mb & 1u);
      s_first_v[tid] = v[0];
      __syncthreads();
      const double m_next = s_first_m[tid + 1];
      const double v_next = s_first_v[tid + 1];

      // thread map F = f_{t0} o ... o f_{t0+7}, applied to X = A at t0+8
      Aff F{0.0, 1.0};
#pragma unroll
      for (int k = kGaeTpt - 1; k >= 0; --k) F = compose(tok_map(p, r, v, mb, k, m_next, v_next), F);
      // inclusive suffix scan within the warp: lane gets F_lane o ... o F_31
      Aff S = F;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double od = __shfl_down_sync(kFull, S.d, o);
        const double oc = __shfl_down_sync(kFull, S.c, o);
        if (lane + o < 32) S = compose(S, Aff{od, oc});
      }
      if (lane == 0) s_warp[wid] = S;
      // exclusive within the warp: F_{lane+1} o ... o F_31
      Aff E{__shfl_down_sync(kFull, S.d, 1), __shfl_down_sync(kFull, S.c, 1)};
      if (lane == 31) E = Aff{0.0, 1.0};
      __syncthreads();
      // carry into this warp: (warps w+1..7) applied to the tile carry
      double X = s_carryA;
      for (int w2 = kGaeThreads / 32 - 1; w2 > wid; --w2) X = fma(s_warp[w2].c, X, s_warp[w2].d);
      X = fma(E.c, X, E.d);  // A at t0 + 8
      // walk right to left, store, accumulate whitening sums
      float outA[kGaeTpt], outR[kGaeTpt];
#pragma unroll
      for (int k = kGaeTpt - 1; k >= 0; --k) {
        const Aff f = tok_map(p, r, v, mb, k, m_next, v_next);  // recomputed: cheaper than 32 live registers
        X = fma(f.c, X, f.d);
        outA[k] = (float)X;
        outR[k] = (float)(X + (double)v[k]);
        const int64_t t = t0 + k;
        if ((mb >> k) & 1u) {  // mb is zero outside [a, b)
          wsA += X;
          wsA2 += X * X;
          wsm += 1.0;
        }
      }
      if (any) {
        if (t0 >= a && t0 + kGaeTpt <= b) {
          float4* pa = reinterpret_cast<float4*>(p.adv + t0);
          float4* pr = reinterpret_cast<float4*>(p.ret + t0);
          pa[0] = make_float4(outA[0], outA[1], outA[2], outA[3]);
          pa[1] = make_float4(outA[4], outA[5], outA[6], outA[7]);
          pr[0] = make_float4(outR[0], outR[1], outR[2], outR[3]);
          pr[1] = make_float4(outR[4], outR[5], outR[6], outR[7]);
        } else {
#pragma unroll
          for (int k = 0; k < kGaeTpt; ++k) {
            const int64_t t = t0 + k;
            if (t >= a && t < b) {
              p.adv[t] = outA[k];
              p.ret[t] = outR[k];
            }
          }
        }
      }
      if (cb <= c_first) break;
      __syncthreads();  // everyone done with s_first_* and s_carryA of this tile
      if (tid == 0) {
        s_carryA = X;  // thread 0 holds A at its first token = leftmost of this tile
        s_first_m[kGaeThreads] = (double)(mb & 1u);
        s_first_v[kGaeThreads] = v[0];
      }
    }
  }

  if (!p.whiten) return;
  // deterministic whitening sums: block tree, then the last block (ticket) sums
  // the per-rollout partials in rollout order
  double q[3] = {wsA, wsA2, wsm};
#pragma unroll
  for (int k = 0; k < 3; ++k) q[k] = warp_sum(q[k]);
  __syncthreads();
  if (lane == 0)
    for (int k = 0; k < 3; ++k) s_red[wid * 3 + k] = q[k];
  __syncthreads();
  if (tid == 0) {
    double t3[3] = {0, 0, 0};
    for (int w2 = 0; w2 < kGaeThreads / 32; ++w2)
      for (int k = 0; k < 3; ++k) t3[k] += s_red[w2 * 3 + k];
    for (int k = 0; k < 3; ++k) p.blk[s * 3 + k] = t3[k];
    __threadfence();
    const unsigned tk = atomicAdd(p.ticket, 1u);
    is_last = tk == (unsigned)p.n_seq - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const volatile double* vb = p.blk;
  double tot[3] = {0, 0, 0};
  for (int64_t i = tid; i < p.n_seq; i += kGaeThreads)
    for (int k = 0; k < 3; ++k) tot[k] += vb[i * 3 + k];
  for (int k = 0; k < 3; ++k) tot[k] = warp_sum(tot[k]);
  if (lane == 0)
    for (int k = 0; k < 3; ++k) s_red[wid * 3 + k] = tot[k];
  __syncthreads();
  if (tid == 0) {
    double t3[3] = {0, 0, 0};
    for (int w2 = 0; w2 < kGaeThreads / 32; ++w2)
      for (int k = 0; k < 3; ++k) t3[k] += s_red[w2 * 3 + k];
    for (int k = 0; k < 3; ++k) p.whiten[k] = t3[k];
    *p.ticket = 0u;
  }
}

}  // namespace dfx

using namespace dfx;

extern "C" {

size_t dfx_gae_workspace_bytes(int64_t n_rollouts) {
  return 256 + ((sizeof(double) * 3 * size_t(n_rollouts < 1 ? 1 : n_rollouts) + 255) & ~size_t(255));
}

dfx_status dfx_gae(const dfx_packed* b, double gamma, double lam, float* adv, float* ret, double* whiten,
                   void* workspace, size_t ws_bytes, dfx_stream stream) {
  if (!b || !b->cu_seqlens || !b->token_reward || !b->value_tok || !b->mask || !adv || !ret)
    return fail(DFX_INVALID_ARGUMENT, "dfx_gae: packed batch lacks cu_seqlens/token_reward/value_tok/mask or null output");
  if (b->n_rollouts <= 0) {
    if (whiten) DFX_CUDA(cudaMemsetAsync(whiten, 0, 3 * sizeof(double), stream));
    return DFX_OK;
  }
  if (whiten && (!workspace || ws_bytes < dfx_gae_workspace_bytes(b->n_rollouts)))
    return fail(DFX_INVALID_ARGUMENT, "dfx_gae: workspace too small");
  GaeParams p;
  p.cu = b->cu_seqlens;
  p.n_seq = b->n_rollouts;
  p.rew = b->token_reward;
  p.val = b->value_tok;
  p.mask = b->mask;
  p.gamma = gamma;
  p.gl = gamma * lam;
  p.adv = adv;
  p.ret = ret;
  p.ticket = whiten ? static_cast<unsigned int*>(workspace) : nullptr;
  p.blk = whiten ? reinterpret_cast<double*>(static_cast<char*>(workspace) + 256) : nullptr;
  p.whiten = whiten;
  gae_kernel<<<(unsigned)b->n_rollouts, kGaeThreads, 0, stream>>>(p);
  DFX_LAUNCH_CHECK("gae_kernel");
  return DFX_OK;
}

}  // extern "C"
