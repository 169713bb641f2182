// common.cuh -- shared device helpers for libdfx (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

#include "../../include/dfx.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libdfx is written for sm_100a (B200) only"
#endif

namespace dfx {

// ---- error plumbing (thread-local message, see dfx_last_error) -------------
void set_error(const std::string& msg);
dfx_status fail(dfx_status code, const std::string& msg);
dfx_status cuda_status(cudaError_t e, const char* what);

#define DFX_CUDA(call)                                            \
  do {                                                            \
    cudaError_t _e = (call);                                      \
    if (_e != cudaSuccess) return ::dfx::cuda_status(_e, #call);  \
  } while (0)

#define DFX_LAUNCH_CHECK(what)                                        \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::dfx::cuda_status(_e, what);       \
  } while (0)

constexpr int kWarp = 32;
constexpr uint32_t kFull = 0xffffffffu;

// device error flags (bit per condition), reported by dfx_check_flags
enum : int32_t { kFlagMissingRollouts = 1, kFlagBadInput = 2 };

// ---- 128-bit streaming loads (read once: bypass L1 allocation) --------------
__device__ __forceinline__ float4 ldg_stream_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ldg_stream_u32(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
// predicated forms: no load when pred is false (the outputs are then undefined and must not be used) -- a
// predicated instruction instead of a branch around the asm, which the compiler cannot if-convert
__device__ __forceinline__ float4 ldg_stream_f4_if(const float* p, bool pred) {
  float4 r;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n\t}"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "r"((int)pred));
  return r;
}
__device__ __forceinline__ uint32_t ldg_stream_u32_if(const void* p, bool pred) {
  uint32_t r;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.L1::no_allocate.u32 %0, [%1];\n\t}"
               : "=r"(r)
               : "l"(p), "r"((int)pred));
  return r;
}
__device__ __forceinline__ void prefetch_l2_if(const void* p, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t@q prefetch.global.L2 [%0];\n\t}" ::"l"(p), "r"((int)pred));
}
__device__ __forceinline__ void stg_stream_f4(float* p, float4 v) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ float f4_get(const float4& v, int k) {
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---- TMA bulk copies + mbarriers (sm_90+ async proxy; SASS UBLKCP / SYNCS) ---------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}"
      ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16), completes on bar
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 1-D bulk copy shared -> global (16-byte aligned, size a multiple of 16), tracked by the bulk-group counter
__device__ __forceinline__ void tma_store_1d(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit_and_wait() {
  asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group 0;" ::: "memory");
}
// bulk prefetch of [p, p+bytes) into L2 (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// order earlier generic-proxy shared-memory accesses before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Copy n bytes src -> dst when the two are in different 16-byte phases: aligned 16-byte stores to dst, each
// assembled (funnel shifts) from the two aligned 16-byte source vectors it straddles, and the unaligned ends byte by
// byte. Threads tid, tid + nthr, ... with nthr a multiple of 32 and whole warps calling (warp shuffles).
// NC: read-only non-coherent loads (peer memory over NVLink), else streaming loads.
template <bool NC>
__device__ __forceinline__ uint4 ld_v4_src(const uint8_t* p) {
  uint4 r;
  if (NC)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  else
    r = __ldcs(reinterpret_cast<const uint4*>(p));
  return r;
}
template <bool NC>
__device__ __forceinline__ void copy_shift16(uint8_t* dst, const uint8_t* src, uint64_t n, uint32_t tid,
                                             uint32_t nthr) {
  const uintptr_t d0 = reinterpret_cast<uintptr_t>(dst), a0 = (d0 + 15) & ~uintptr_t(15);
  const uint64_t head = (uint64_t)min((uintptr_t)n, a0 - d0);
  const uint64_t nu = (n - head) / 16, tail0 = head + 16 * nu;
  for (uint64_t j = tid; j < head; j += nthr) dst[j] = src[j];
  for (uint64_t j = tail0 + tid; j < n; j += nthr) dst[j] = src[j];
  const uintptr_t s1 = reinterpret_cast<uintptr_t>(src + head);  // the source of the first aligned unit
  const uint8_t* sv = reinterpret_cast<const uint8_t*>(s1 & ~uintptr_t(15));
  const uint32_t ph = (uint32_t)(s1 & 15u), q = ph >> 2, sh = (ph & 3u) * 8u;
  const uintptr_t send = reinterpret_cast<uintptr_t>(src + n);
  // warp-uniform rounds of two units per lane: lane l takes units base + l and base + nthr + l, and gets the vector
  // after each from lane l + 1 by a shuffle, so every source vector is read once (lane 31 reads its second vectors
  // itself); both units' loads are in flight together
  const uint32_t lane = tid & 31u;
  for (uint64_t base = tid - lane; base < nu; base += 2 * (uint64_t)nthr) {
    uint4 va[2];
    bool in[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint64_t u = base + (uint64_t)r * nthr + lane;
      in[r] = u < nu;
      va[r] = make_uint4(0u, 0u, 0u, 0u);
      if (in[r]) va[r] = ld_v4_src<NC>(sv + 16 * u);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint64_t u = base + (uint64_t)r * nthr + lane;
      uint4 vb;
      vb.x = __shfl_down_sync(0xffffffffu, va[r].x, 1);
      vb.y = __shfl_down_sync(0xffffffffu, va[r].y, 1);
      vb.z = __shfl_down_sync(0xffffffffu, va[r].z, 1);
      vb.w = __shfl_down_sync(0xffffffffu, va[r].w, 1);
      if (lane == 31 || u + 1 >= nu) {  // (the second vector is only needed when the unit straddles two)
        vb = make_uint4(0u, 0u, 0u, 0u);
        if (in[r] && ph != 0 && reinterpret_cast<uintptr_t>(sv + 16 * u + 16) < send)
          vb = ld_v4_src<NC>(sv + 16 * u + 16);
      }
      if (!in[r]) continue;
      const uint32_t w[8] = {va[r].x, va[r].y, va[r].z, va[r].w, vb.x, vb.y, vb.z, vb.w};
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // source bytes ph .. ph + 15 of the 32: words q + k and q + k + 1, >> sh bits
        const uint32_t lo = q == 0 ? w[k] : q == 1 ? w[k + 1] : q == 2 ? w[k + 2] : w[k + 3];
        const uint32_t hi = q == 0 ? w[k + 1] : q == 1 ? w[k + 2] : q == 2 ? w[k + 3] : w[k + 4];
        o[k] = __funnelshift_r(lo, hi, sh);
      }
      reinterpret_cast<uint4*>(dst + head)[u] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// ---- per-token loss math shared by the loss kernels (loss.cu) and the fused GAE + loss scan (gae.cu) ---------
// k3 = e^x - x - 1 (x = ref - lp) by its Taylor series for |x| < 1/8 (truncation < 1.2e-8 relative); callers
// fall back to expm1f(x) - x, which has no cancellation, for larger |x|.
__device__ __forceinline__ float k3_series(float x) {
  float q = 1.0f / 720.0f;
  q = fmaf(q, x, 1.0f / 120.0f);
  q = fmaf(q, x, 1.0f / 24.0f);
  q = fmaf(q, x, 1.0f / 6.0f);
  q = fmaf(q, x, 0.5f);
  return (x * x) * q;
}
constexpr float kK3Series = 0.125f;
// 2^x by MUFU.EX2 alone (flush-to-zero): exp2f's extra range reduction only matters below 2^-126, where the ratio
// (and every term it enters) is zero for the loss anyway; identical bits elsewhere
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f;

// Exact clip decision s*(l - o) > s*T for f32 inputs l, o (d = f32(l - o)) against a threshold given as the float
// pair sT32 + sTl (= s*T to ~2^-48): TwoSum gives d + e == l - o exactly, and s*d - sT32 is exact wherever the sign
// of the total is in doubt (Sterbenz). sT32 = +inf: never.
__device__ __forceinline__ bool clip_exact_f32(float s, float sT32, float sTl, float l, float o, float d) {
  const float bb = d - l;
  const float e = (l - (d - bb)) + (-o - bb);
  return (s * d - sT32) + (s * e - sTl) > 0.0f;
}

// ---- reference hash (distflow/hash.hpp), integer-exact on device ------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t hash_combine(uint64_t seed, uint64_t v) {
  return splitmix64(seed ^ (v + 0x9E3779B97F4A7C15ull + (seed << 6) + (seed >> 2)));
}
__device__ __forceinline__ double unit_from_hash(uint64_t h) {
  return __dmul_rn((double)(h >> 11), 1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double symmetric_from_hash(uint64_t h) {
  return __dadd_rn(__dmul_rn(2.0, unit_from_hash(h)), -1.0);
}

// ---- slot decomposition of a packed token range ------------------------------
// Work units are the non-empty pieces "rollout s  ∩  window w" of the token
// line, windows being 2^sh-token aligned blocks starting at base = cu[0] & ~3.
// Piece (s, w) gets slot id s + w; slot ids are unique and increase along the
// token line, so each rollout's pieces occupy contiguous slots
// [s + w_first(s), s + w_last(s)] and a warp recovers (s, w) from its slot id
// with a search over f(s) = s + ((cu[s] - base) >> sh), which is strictly
// increasing. Slots whose piece is empty (a rollout starting exactly on a
// window edge skips one id; zero-length rollouts own no slot) are no-ops.
struct SlotGeom {
  const int64_t* cu;
  int64_t n_seq;
  int64_t base;
  int sh;
};

__device__ __forceinline__ int64_t slot_f(const SlotGeom& g, int64_t s) {
  return s + ((__ldg(g.cu + s) - g.base) >> g.sh);
}

// Warp-cooperative 32-ary search: largest s in [0, n_seq) with f(s) <= u.
__device__ __forceinline__ int64_t slot_find_seq(const SlotGeom& g, int64_t u, int lane) {
  int64_t lo = 0, hi = g.n_seq;
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) >> 5;
    const int64_t s = lo + (int64_t)lane * step;
    const bool pred = (s < hi) && (slot_f(g, s) <= u);
    const uint32_t m = __ballot_sync(kFull, pred);
    const int k = 31 - __clz(m);  // lane 0 is always true: f(lo) <= u
    lo = lo + (int64_t)k * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// Resolve slot u to (s, [t0, t1)); returns false for an empty slot.
__device__ __forceinline__ bool slot_unit(const SlotGeom& g, int64_t u, int lane, int64_t& s,
                                          int64_t& t0, int64_t& t1) {
  s = slot_find_seq(g, u, lane);
  const int64_t a = __ldg(g.cu + s), b = __ldg(g.cu + s + 1);
  if (b <= a) return false;
  const int64_t w = u - s;
  const int64_t wa = (a - g.base) >> g.sh, wb = (b - 1 - g.base) >> g.sh;
  if (w < wa || w > wb) return false;
  const int64_t ws = g.base + (w << g.sh);
  t0 = max(a, ws);
  t1 = min(b, ws + ((int64_t)1 << g.sh));
  return true;
}

// Host: window size of the streaming kernels, a function of the token span only (the workspace sizing and the
// launch must agree): 2048-token windows, 1024 for spans of 7.3M..21.8M tokens. Measured on B200: shorter
// windows lose more to per-slot setup (claim + table load + reduction + partials) than they gain in balance at C2's
// 33.5M tokens (1024: 0.81 vs 2048: 0.843 of HBM), and gain at C5's 16.9M (0.7555 vs 0.7303); 512-token windows
// made the C3 step 20% slower (profiles/r02_clip_sweep2.log).
// Benchmarking knobs: DFX_SLOT_SHIFT forces the window; DFX_SLOT_TARGET=k halves it until there are k windows per
// resident warp.
inline int slot_shift(int64_t token_span) {
  static const int forced = [] {
    const char* e = std::getenv("DFX_SLOT_SHIFT");
    const int v = e ? std::atoi(e) : 0;
    return v >= 8 && v <= 14 ? v : 0;
  }();
  if (forced) return forced;
  static const int64_t target = [] {
    const char* e = std::getenv("DFX_SLOT_TARGET");
    const int v = e ? std::atoi(e) : 0;
    return int64_t(v >= 1 && v <= 64 ? v : 0) * 148 * 24;
  }();
  if (target) {
    int sh = 11;
    while (sh > 8 && (token_span >> sh) < target) --sh;
    return sh;
  }
  // 2..6k tokens per resident warp (3 x 8 warps on 148 SMs): 1024-token windows, so the last windows are short
  // enough to balance (C5 per-GPU share, 16.9M tokens: 0.73 -> 0.76 of HBM). Above (C2, 33.5M) 2048 stays best;
  // below (C3, 4.2M) the doubled slot table and partials cost more than the balance gains (step +9%).
  const int64_t per_warp = token_span / (int64_t(148) * 24);
  return per_warp >= 2048 && per_warp < 6144 ? 10 : 11;
}

// Host: number of slots for n_seq rollouts spanning token_span tokens.
inline int64_t slot_count(int64_t n_seq, int64_t token_span, int sh) {
  const int64_t win = ((token_span + 3) >> sh) + 2;  // base may start up to 3 before cu[0]
  return n_seq + win;
}

}  // namespace dfx
