/*
 * dfx_oracle.h -- CPU restatement of DistFlow's post-rollout hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2507_13833_b200/,
 * include/, the CUDA library) may include, link or call this. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * use it, and only as the checker or the timed CPU baseline.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/).
 *
 * Parity status:
 *   - hash, draw_tokens, group advantage, ppo advantage, reshard placement
 *     and the LE record blob are PINNED: tests check them against the
 *     reference's own known-answer tests and against the reference headers
 *     compiled into oracle/_ref (see oracle/Makefile).
 *   - GAE, PPO clipped surrogate, KL and loss aggregation do not exist in the
 *     reference. Their restatement here is PARITY UNPINNED: it
 *     is pinned only by our own hand-computed known-answer tests.
 *
 * Build: plain C11, -O2 -ffp-contract=off (no FMA contraction, so f64
 * results are IEEE-reproducible).
 */
#ifndef DFX_ORACLE_H
#define DFX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference's typed exceptions (distflow/errors.hpp) */
enum {
  DFO_OK = 0,
  DFO_ERROR = 1,                 /* Error */
  DFO_LAYOUT_ERROR = 2,          /* LayoutError, errors.hpp:32 */
  DFO_INDIVISIBLE_ERROR = 3,     /* IndivisibleError, errors.hpp:52 */
  DFO_MISSING_ROLLOUTS = 4,      /* MissingRolloutsError, errors.hpp:123 */
  DFO_MISSING_CHANNEL = 5,       /* MissingChannelError, errors.hpp:116 */
};

/* ---- hash.hpp ---------------------------------------------------------- */
uint64_t dfo_splitmix64(uint64_t z);                        /* hash.hpp:14-19 */
uint64_t dfo_hash_combine(uint64_t seed, uint64_t v);       /* hash.hpp:21-23 */
uint64_t dfo_hash_str(uint64_t seed, const char* s);        /* hash.hpp:25-29 */
/* keyed_hash(seed, domain, counters...) hash.hpp:31-37 */
uint64_t dfo_keyed_hash(uint64_t seed, const char* domain, int n, const uint64_t* counters);
double dfo_unit_from_hash(uint64_t h);                      /* hash.hpp:40-42 */
double dfo_symmetric_from_hash(uint64_t h);                 /* hash.hpp:45 */
void dfo_hash_bytes(uint64_t key, uint8_t* out, size_t n);  /* hash.hpp:48-59 */

/* ---- functions.hpp: token distribution ----------------------------------- */
enum { DFO_CONSTANT = 0, DFO_UNIFORM = 1, DFO_SKEWED = 2 };
typedef struct {
  int32_t kind;
  uint32_t value; /* CONSTANT */
  uint32_t min;   /* UNIFORM / SKEWED, inclusive */
  uint32_t max;
} dfo_token_dist;

/* draw_tokens functions.hpp:67-80. SKEWED is new (the reference has only
 * CONSTANT/UNIFORM): L = min + floor(span * a*b*c / 2^63) with a,b,c the three
 * 21-bit fields of the same keyed hash -- a product of three uniforms, heavy
 * toward short lengths with a long tail to max. Integer-exact everywhere. */
int dfo_draw_tokens(const dfo_token_dist* d, uint64_t seed, uint64_t sample_id,
                    uint32_t rollout, uint32_t* out);

/* ---- synthetic rollout batch ---------------------------
 * Records r=0..R-1 with sample ids ids[r], each with n rollouts.
 * Lengths from draw_tokens; rollout scalars exactly as fill_channel
 * (functions.hpp:95-104): reward = unit(kh(seed,"reward",id,j)),
 * value = sym(kh(seed,"value",id,j)). Per-token streams use a token counter
 * appended to the same keyed-hash scheme (functions.hpp:52-54):
 *   lp      = f32(-4 * unit(kh(seed,"tok_lp",id,j,t)))
 *   old_lp  = f32(f64(lp) + 0.25 * sym(kh(seed,"tok_old",id,j,t)))
 *   ref_lp  = f32(f64(lp) + 0.1  * sym(kh(seed,"tok_ref",id,j,t)))
 *   value_t = f32(sym(kh(seed,"tok_value",id,j,t)))
 *   token_reward = t==L-1 ? f32(reward) : 0
 *   mask    = t >= p, p = kh(seed,"tok_mask",id,j) % (L/5 + 1)   (~10% prefix)
 *   token_id= kh(seed,"tok_id",id,j,t) % 151936
 * Every value is rounded to f32 once; consumers promote those f32 to f64. */
int dfo_synth_lengths(const dfo_token_dist* d, uint64_t seed, const uint64_t* ids,
                      uint32_t n_records, uint32_t n_roll, int64_t* cu_seqlens /* R*n+1 */);
void dfo_synth_rollout_scalars(uint64_t seed, const uint64_t* ids, uint32_t n_records,
                               uint32_t n_roll, double* reward, double* value);
/* any output pointer may be NULL. nthreads<=1: single thread. */
void dfo_synth_tokens(uint64_t seed, const uint64_t* ids, uint32_t n_records, uint32_t n_roll,
                      const int64_t* cu_seqlens, float* lp, float* old_lp, float* ref_lp,
                      float* value_tok, float* token_reward, uint8_t* mask, int32_t* token_id,
                      int nthreads);

/* ---- advantages -------------------------------------------------------------- */
/* fn_group_advantage functions.hpp:143-161. group_off: R+1 rollout offsets.
 * Returns DFO_MISSING_ROLLOUTS for an empty group. */
int dfo_grpo_advantage(uint32_t n_records, const int32_t* group_off, const double* reward,
                       double eps, double* adv);
/* fn_ppo_advantage functions.hpp:163-172 */
void dfo_ppo_advantage(uint32_t n_rollouts, const double* reward, const double* value, double* adv);
/* per-token broadcast (new): adv_tok[t] = mask[t] ? f32(adv[s]) : 0 */
void dfo_broadcast_advantage(uint32_t n_seq, const int64_t* cu_seqlens, const double* adv,
                             const uint8_t* mask, float* adv_tok);

/* GAE (new; PARITY UNPINNED). Per sequence, reverse in t:
 *   m1 = t+1<L ? mask[t+1] : 0 ; v1 = t+1<L ? V[t+1] : 0
 *   delta_t = r_t + gamma*m1*v1 - V_t
 *   A_t = delta_t + gamma*lam*m1*A_{t+1}      R_t = A_t + V_t
 * whiten (optional, out[3] = {sum m*A, sum m*A^2, sum m}). */
void dfo_gae(uint32_t n_seq, const int64_t* cu_seqlens, const float* token_reward,
             const float* value, const uint8_t* mask, double gamma, double lam, double* adv,
             double* ret, double* whiten_sums);

/* PPO clipped surrogate + KL + masked aggregation (new; PARITY UNPINNED). */
enum { DFO_KL_NONE = 0, DFO_KL_K1 = 1, DFO_KL_K2 = 2, DFO_KL_K3 = 3 };
enum { DFO_AGG_TOKEN_MEAN = 0, DFO_AGG_SEQ_MEAN_TOKEN_MEAN = 1, DFO_AGG_SEQ_MEAN_TOKEN_SUM = 2 };
typedef struct {
  double clip_low;   /* eps_low: ratio clipped to [1-clip_low, 1+clip_high] */
  double clip_high;
  double beta;       /* KL coefficient */
  int32_t kl_type;
  int32_t agg;
  int32_t whiten;    /* 1: A_w = (A - mu) / sqrt(var_unbiased + 1e-8) over masked tokens */
  int32_t pad;
} dfo_loss_cfg;
typedef struct {
  double loss, pg_loss, kl, clipfrac, approx_kl, n_tokens, n_seqs;
} dfo_loss_out;
/* adv: per-token f32 advantage. dlogp (nullable): d loss / d lp per token. */
int dfo_ppo_loss(uint32_t n_seq, const int64_t* cu_seqlens, const float* lp, const float* old_lp,
                 const float* ref_lp, const float* adv, const uint8_t* mask,
                 const dfo_loss_cfg* cfg, dfo_loss_out* out, double* dlogp);
/* timing-only: sequences split over nthreads (CPU baseline); unwhitened, no dlogp, else single-thread. */
int dfo_ppo_loss_mt(uint32_t n_seq, const int64_t* cu_seqlens, const float* lp, const float* old_lp,
                    const float* ref_lp, const float* adv, const uint8_t* mask,
                    const dfo_loss_cfg* cfg, dfo_loss_out* out, int nthreads);

/* ---- topology.hpp + data_plane.hpp: reshard placement ----
 * Producer groups p=0..dp_p-1 hold group_counts[p] records. Returns, for every
 * destination group d (0..dp_c-1), dest_counts[d] and the records it receives
 * as indices into ordered = L_0 || ... || L_{dp_p-1}, written dest-major into
 * src_index (length sum(group_counts)). Errors: DFO_LAYOUT_ERROR
 * (check_layout topology.hpp:53-68), DFO_INDIVISIBLE_ERROR
 * (data_plane.hpp:414-416 and :281-283). */
int dfo_reshard_placement(uint32_t B, uint32_t W, uint32_t dp_p, uint32_t tp_p, uint32_t dp_c,
                          uint32_t tp_c, const uint64_t* group_counts, uint64_t* dest_counts,
                          uint64_t* src_index);

/* ---- record.hpp: LE record blob -------------------------------------------
 * serialize_records (record.hpp:109-127,151-156) of a packed batch.
 * Record r: sample_id ids[r]; meta = the record's pre-serialized meta section
 * bytes meta_blob[meta_off[r]..meta_off[r+1]) (u32 count + (str,str)*), or an
 * empty map when meta_off is NULL; rollouts group_off[r]..group_off[r+1].
 * Rollout s: token_count = tok_count[s]; payload = concatenation over the
 * n_streams token streams of stream bytes [cu[s]*esz, cu[s+1]*esz);
 * channels: n_ch (name, f64 per rollout), names given in sorted order.
 * If out is NULL only the size is returned. Returns total bytes. */
uint64_t dfo_serialize_packed(uint32_t n_records, const uint64_t* ids, const int64_t* meta_off,
                              const uint8_t* meta_blob, const int32_t* group_off,
                              const uint32_t* tok_count, const int64_t* cu_seqlens, int n_streams,
                              const void* const* streams, const uint32_t* stream_esz, int n_ch,
                              const char* const* ch_names, const double* const* ch_vals,
                              uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
