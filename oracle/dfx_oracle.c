/*
 * dfx_oracle.c -- CPU restatement of the DistFlow post-rollout hot path.
 * TEST INFRASTRUCTURE ONLY (see dfx_oracle.h). Reference paths are relative to
 * /root/reference/proj/include/.
 */
#include "dfx_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- hash.hpp ------------------------------------------------------------ */

uint64_t dfo_splitmix64(uint64_t z) { /* hash.hpp:14-19 */
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t dfo_hash_combine(uint64_t seed, uint64_t v) { /* hash.hpp:21-23 */
  return dfo_splitmix64(seed ^ (v + 0x9E3779B97F4A7C15ull + (seed << 6) + (seed >> 2)));
}

uint64_t dfo_hash_str(uint64_t seed, const char* s) { /* hash.hpp:25-29: bytes as uint8 */
  uint64_t h = seed;
  for (const unsigned char* p = (const unsigned char*)s; *p; ++p) h = dfo_hash_combine(h, *p);
  return h;
}

uint64_t dfo_keyed_hash(uint64_t seed, const char* domain, int n, const uint64_t* c) {
  uint64_t h = dfo_hash_str(seed, domain); /* hash.hpp:31-37 */
  for (int i = 0; i < n; ++i) h = dfo_hash_combine(h, c[i]);
  return h;
}

double dfo_unit_from_hash(uint64_t h) { /* hash.hpp:40-42 */
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

double dfo_symmetric_from_hash(uint64_t h) { return 2.0 * dfo_unit_from_hash(h) - 1.0; }

void dfo_hash_bytes(uint64_t key, uint8_t* out, size_t n) { /* hash.hpp:48-59 */
  size_t i = 0;
  uint64_t counter = 0;
  while (i < n) {
    uint64_t block = dfo_splitmix64(key + counter++);
    for (int b = 0; b < 8 && i < n; ++b, ++i) out[i] = (uint8_t)(block >> (8 * b));
  }
}

static uint64_t kh2(uint64_t seed, const char* dom, uint64_t a, uint64_t b) {
  const uint64_t c[2] = {a, b};
  return dfo_keyed_hash(seed, dom, 2, c);
}

/* ---- functions.hpp:67-80 draw_tokens (+ SKEWED) -------------------------- */

int dfo_draw_tokens(const dfo_token_dist* d, uint64_t seed, uint64_t sample_id, uint32_t rollout,
                    uint32_t* out) {
  switch (d->kind) {
    case DFO_CONSTANT:
      *out = d->value;
      return DFO_OK;
    case DFO_UNIFORM: {
      if (d->max < d->min) return DFO_ERROR; /* "token distribution max < min" */
      const uint64_t span = (uint64_t)d->max - d->min + 1;
      *out = d->min + (uint32_t)(kh2(seed, "gen_tokens", sample_id, rollout) % span);
      return DFO_OK;
    }
    case DFO_SKEWED: {
      if (d->max < d->min) return DFO_ERROR;
      const uint64_t span = (uint64_t)d->max - d->min + 1;
      const uint64_t h = kh2(seed, "gen_tokens", sample_id, rollout);
      const uint64_t prod = (h & 0x1FFFFFull) * ((h >> 21) & 0x1FFFFFull) * ((h >> 42) & 0x1FFFFFull);
      const unsigned __int128 w = (unsigned __int128)span * prod; /* < span * 2^63 */
      *out = d->min + (uint32_t)(uint64_t)(w >> 63);
      return DFO_OK;
    }
  }
  *out = d->value;
  return DFO_OK;
}

/* ---- synthetic batch ----------------------------------------------------- */

int dfo_synth_lengths(const dfo_token_dist* d, uint64_t seed, const uint64_t* ids,
                      uint32_t n_records, uint32_t n_roll, int64_t* cu) {
  cu[0] = 0;
  uint64_t s = 0;
  for (uint32_t r = 0; r < n_records; ++r) {
    for (uint32_t j = 0; j < n_roll; ++j, ++s) {
      uint32_t L;
      int st = dfo_draw_tokens(d, seed, ids[r], j, &L);
      if (st) return st;
      cu[s + 1] = cu[s] + L;
    }
  }
  return DFO_OK;
}

void dfo_synth_rollout_scalars(uint64_t seed, const uint64_t* ids, uint32_t n_records,
                               uint32_t n_roll, double* reward, double* value) {
  /* fill_channel functions.hpp:95-104 (reward unit-range :135-138, value symmetric :130-133) */
  uint64_t s = 0;
  for (uint32_t r = 0; r < n_records; ++r) {
    for (uint32_t j = 0; j < n_roll; ++j, ++s) {
      if (reward) reward[s] = dfo_unit_from_hash(kh2(seed, "reward", ids[r], j));
      if (value) value[s] = dfo_symmetric_from_hash(kh2(seed, "value", ids[r], j));
    }
  }
}

typedef struct {
  uint64_t seed;
  const uint64_t* ids;
  uint32_t r0, r1, n_roll;
  const int64_t* cu;
  float *lp, *old_lp, *ref_lp, *value_tok, *token_reward;
  uint8_t* mask;
  int32_t* token_id;
} synth_job;

static void synth_range(const synth_job* j) {
  const uint64_t h_lp = dfo_hash_str(j->seed, "tok_lp");
  const uint64_t h_old = dfo_hash_str(j->seed, "tok_old");
  const uint64_t h_ref = dfo_hash_str(j->seed, "tok_ref");
  const uint64_t h_val = dfo_hash_str(j->seed, "tok_value");
  const uint64_t h_id = dfo_hash_str(j->seed, "tok_id");
  for (uint32_t r = j->r0; r < j->r1; ++r) {
    const uint64_t id = j->ids[r];
    for (uint32_t k = 0; k < j->n_roll; ++k) {
      const uint64_t s = (uint64_t)r * j->n_roll + k;
      const int64_t b = j->cu[s], L = j->cu[s + 1] - b;
      const uint64_t blp = dfo_hash_combine(dfo_hash_combine(h_lp, id), k);
      const uint64_t bold = dfo_hash_combine(dfo_hash_combine(h_old, id), k);
      const uint64_t bref = dfo_hash_combine(dfo_hash_combine(h_ref, id), k);
      const uint64_t bval = dfo_hash_combine(dfo_hash_combine(h_val, id), k);
      const uint64_t bid = dfo_hash_combine(dfo_hash_combine(h_id, id), k);
      const uint64_t p = kh2(j->seed, "tok_mask", id, k) % (uint64_t)(L / 5 + 1);
      const float rew = (float)dfo_unit_from_hash(kh2(j->seed, "reward", id, k));
      for (int64_t t = 0; t < L; ++t) {
        const float lp = (float)(-4.0 * dfo_unit_from_hash(dfo_hash_combine(blp, (uint64_t)t)));
        if (j->lp) j->lp[b + t] = lp;
        if (j->old_lp)
          j->old_lp[b + t] =
              (float)((double)lp + 0.25 * dfo_symmetric_from_hash(dfo_hash_combine(bold, (uint64_t)t)));
        if (j->ref_lp)
          j->ref_lp[b + t] =
              (float)((double)lp + 0.1 * dfo_symmetric_from_hash(dfo_hash_combine(bref, (uint64_t)t)));
        if (j->value_tok)
          j->value_tok[b + t] = (float)dfo_symmetric_from_hash(dfo_hash_combine(bval, (uint64_t)t));
        if (j->token_reward) j->token_reward[b + t] = (t == L - 1) ? rew : 0.0f;
        if (j->mask) j->mask[b + t] = (uint64_t)t >= p ? 1 : 0;
        if (j->token_id) j->token_id[b + t] = (int32_t)(dfo_hash_combine(bid, (uint64_t)t) % 151936ull);
      }
    }
  }
}

static void* synth_thread(void* arg) {
  synth_range((const synth_job*)arg);
  return NULL;
}

void dfo_synth_tokens(uint64_t seed, const uint64_t* ids, uint32_t n_records, uint32_t n_roll,
                      const int64_t* cu, float* lp, float* old_lp, float* ref_lp, float* value_tok,
                      float* token_reward, uint8_t* mask, int32_t* token_id, int nthreads) {
  synth_job base = {seed, ids, 0, n_records, n_roll, cu, lp, old_lp, ref_lp, value_tok, token_reward,
                    mask, token_id};
  if (nthreads <= 1 || n_records < 2) {
    synth_range(&base);
    return;
  }
  if ((uint32_t)nthreads > n_records) nthreads = (int)n_records;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  synth_job* jobs = (synth_job*)malloc(sizeof(synth_job) * (size_t)nthreads);
  for (int i = 0; i < nthreads; ++i) {
    jobs[i] = base;
    jobs[i].r0 = (uint32_t)((uint64_t)n_records * i / nthreads);
    jobs[i].r1 = (uint32_t)((uint64_t)n_records * (i + 1) / nthreads);
    pthread_create(&th[i], NULL, synth_thread, &jobs[i]);
  }
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  free(jobs);
}

/* ---- advantages ------------------------------------------------------------ */

int dfo_grpo_advantage(uint32_t n_records, const int32_t* go, const double* reward, double eps,
                       double* adv) {
  /* fn_group_advantage functions.hpp:143-161: sequential f64 sums, population
   * std (divide by n), eps added to std, zero numerator short-circuited. */
  for (uint32_t r = 0; r < n_records; ++r) {
    const int32_t a = go[r], b = go[r + 1];
    if (b <= a) return DFO_MISSING_ROLLOUTS; /* require_rollouts :82-87 */
    const double n = (double)(b - a);
    double sum = 0;
    for (int32_t s = a; s < b; ++s) sum += reward[s];
    const double mean = sum / n;
    double var = 0;
    for (int32_t s = a; s < b; ++s) {
      const double d = reward[s] - mean;
      var += d * d;
    }
    const double sd = sqrt(var / n);
    for (int32_t s = a; s < b; ++s) {
      const double d = reward[s] - mean;
      adv[s] = d == 0.0 ? 0.0 : d / (sd + eps);
    }
  }
  return DFO_OK;
}

void dfo_ppo_advantage(uint32_t n, const double* reward, const double* value, double* adv) {
  for (uint32_t s = 0; s < n; ++s) adv[s] = reward[s] - value[s]; /* functions.hpp:169 */
}

void dfo_broadcast_advantage(uint32_t n_seq, const int64_t* cu, const double* adv,
                             const uint8_t* mask, float* adv_tok) {
  for (uint32_t s = 0; s < n_seq; ++s) {
    const float a = (float)adv[s];
    for (int64_t t = cu[s]; t < cu[s + 1]; ++t) adv_tok[t] = mask[t] ? a : 0.0f;
  }
}

void dfo_gae(uint32_t n_seq, const int64_t* cu, const float* rew, const float* val,
             const uint8_t* mask, double gamma, double lam, double* adv, double* ret,
             double* wsum) {
  double sA = 0, sA2 = 0, sm = 0;
  for (uint32_t s = 0; s < n_seq; ++s) {
    const int64_t b = cu[s], e = cu[s + 1];
    double A = 0;
    for (int64_t t = e - 1; t >= b; --t) {
      const double m1 = (t + 1 < e) ? (double)mask[t + 1] : 0.0;
      const double v1 = (t + 1 < e) ? (double)val[t + 1] : 0.0;
      const double delta = (double)rew[t] + gamma * m1 * v1 - (double)val[t];
      A = delta + gamma * lam * m1 * A;
      adv[t] = A;
      ret[t] = A + (double)val[t];
      if (mask[t]) {
        sA += A;
        sA2 += A * A;
        sm += 1.0;
      }
    }
  }
  if (wsum) {
    wsum[0] = sA;
    wsum[1] = sA2;
    wsum[2] = sm;
  }
}

/* ---- PPO loss (new; parity unpinned) --------------------------------------- */

int dfo_ppo_loss(uint32_t n_seq, const int64_t* cu, const float* lp, const float* old_lp,
                 const float* ref_lp, const float* adv, const uint8_t* mask, const dfo_loss_cfg* c,
                 dfo_loss_out* out, double* dlogp) {
  double mu = 0.0, rstd = 1.0;
  double N = 0;
  for (uint32_t s = 0; s < n_seq; ++s)
    for (int64_t t = cu[s]; t < cu[s + 1]; ++t) N += mask[t] ? 1.0 : 0.0;
  if (c->whiten) {
    double sA = 0;
    for (uint32_t s = 0; s < n_seq; ++s)
      for (int64_t t = cu[s]; t < cu[s + 1]; ++t)
        if (mask[t]) sA += (double)adv[t];
    mu = N > 0 ? sA / N : 0.0;
    double ss = 0;
    for (uint32_t s = 0; s < n_seq; ++s)
      for (int64_t t = cu[s]; t < cu[s + 1]; ++t)
        if (mask[t]) ss += ((double)adv[t] - mu) * ((double)adv[t] - mu);
    const double var = N > 1 ? ss / (N - 1) : 0.0;
    rstd = 1.0 / sqrt(var + 1e-8);
  }
  double S = 0;
  for (uint32_t s = 0; s < n_seq; ++s) {
    double ns = 0;
    for (int64_t t = cu[s]; t < cu[s + 1]; ++t) ns += mask[t] ? 1.0 : 0.0;
    if (ns > 0) S += 1.0;
  }
  double pg_tot = 0, kl_tot = 0, clip_tot = 0, akl_tot = 0;
  for (uint32_t s = 0; s < n_seq; ++s) {
    double pg_s = 0, kl_s = 0, ns = 0;
    for (int64_t t = cu[s]; t < cu[s + 1]; ++t) ns += mask[t] ? 1.0 : 0.0;
    for (int64_t t = cu[s]; t < cu[s + 1]; ++t) {
      const double m = mask[t] ? 1.0 : 0.0;
      const double l = lp[t], o = old_lp[t], rf = ref_lp[t];
      const double A = c->whiten ? ((double)adv[t] - mu) * rstd : (double)adv[t];
      const double rho = exp(l - o);
      const double rc = fmin(fmax(rho, 1.0 - c->clip_low), 1.0 + c->clip_high);
      const double pg1 = -A * rho, pg2 = -A * rc;
      const int clipped = pg2 > pg1;
      const double pg = clipped ? pg2 : pg1;
      double kl = 0, dkl = 0;
      switch (c->kl_type) {
        case DFO_KL_K1: kl = l - rf; dkl = 1.0; break;
        case DFO_KL_K2: kl = 0.5 * (l - rf) * (l - rf); dkl = l - rf; break;
        case DFO_KL_K3: {
          const double x = rf - l;
          kl = exp(x) - x - 1.0;
          dkl = -(exp(x) - 1.0);
          if (kl > 10.0) { kl = 10.0; dkl = 0.0; }
          if (kl < -10.0) { kl = -10.0; dkl = 0.0; }
          break;
        }
        default: break;
      }
      pg_s += m * pg;
      kl_s += m * kl;
      clip_tot += m * (double)clipped;
      akl_tot += m * (o - l);
      if (dlogp) {
        double w = 0;
        if (m != 0.0) {
          if (c->agg == DFO_AGG_TOKEN_MEAN) w = 1.0 / N;
          else if (c->agg == DFO_AGG_SEQ_MEAN_TOKEN_MEAN) w = 1.0 / (S * ns);
          else w = 1.0 / S;
        }
        const double dpg = clipped ? 0.0 : -A * rho;
        dlogp[t] = w * (dpg + c->beta * dkl);
      }
    }
    if (c->agg == DFO_AGG_TOKEN_MEAN) {
      pg_tot += pg_s;
      kl_tot += kl_s;
    } else if (ns > 0) {
      const double div = c->agg == DFO_AGG_SEQ_MEAN_TOKEN_MEAN ? ns : 1.0;
      pg_tot += pg_s / div;
      kl_tot += kl_s / div;
    }
  }
  const double denom = c->agg == DFO_AGG_TOKEN_MEAN ? N : S;
  out->pg_loss = denom > 0 ? pg_tot / denom : 0.0;
  out->kl = denom > 0 ? kl_tot / denom : 0.0;
  out->loss = out->pg_loss + c->beta * out->kl;
  out->clipfrac = N > 0 ? clip_tot / N : 0.0;
  out->approx_kl = N > 0 ? akl_tot / N : 0.0;
  out->n_tokens = N;
  out->n_seqs = S;
  return DFO_OK;
}

/* Timing-only parallel form of dfo_ppo_loss for the CPU baseline (bench.py): sequences split into nthreads
 * contiguous slices, each slice run through dfo_ppo_loss, slice means re-weighted by their denominators in slice
 * order. Same arithmetic per token; the final sums differ from the single-thread order only in rounding.
 * Unwhitened, no dlogp (both need global denominators first) -- otherwise the single-thread path. */
typedef struct {
  uint32_t n_seq;
  const int64_t* cu;
  const float *lp, *old_lp, *ref_lp, *adv;
  const uint8_t* mask;
  const dfo_loss_cfg* c;
  dfo_loss_out out;
  int rc;
} loss_job;

static void* loss_thread(void* a) {
  loss_job* j = (loss_job*)a;
  j->rc = dfo_ppo_loss(j->n_seq, j->cu, j->lp, j->old_lp, j->ref_lp, j->adv, j->mask, j->c, &j->out, NULL);
  return NULL;
}

int dfo_ppo_loss_mt(uint32_t n_seq, const int64_t* cu, const float* lp, const float* old_lp,
                    const float* ref_lp, const float* adv, const uint8_t* mask, const dfo_loss_cfg* c,
                    dfo_loss_out* out, int nthreads) {
  if (nthreads <= 1 || c->whiten || n_seq < 2)
    return dfo_ppo_loss(n_seq, cu, lp, old_lp, ref_lp, adv, mask, c, out, NULL);
  if ((uint32_t)nthreads > n_seq) nthreads = (int)n_seq;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  loss_job* jobs = (loss_job*)malloc(sizeof(loss_job) * (size_t)nthreads);
  for (int i = 0; i < nthreads; ++i) {
    const uint32_t s0 = (uint32_t)((uint64_t)n_seq * (uint64_t)i / (uint64_t)nthreads);
    const uint32_t s1 = (uint32_t)((uint64_t)n_seq * (uint64_t)(i + 1) / (uint64_t)nthreads);
    loss_job j = {s1 - s0, cu + s0, lp, old_lp, ref_lp, adv, mask, c, {0}, 0};
    jobs[i] = j;
    pthread_create(&th[i], NULL, loss_thread, &jobs[i]);
  }
  double N = 0, S = 0, pg = 0, kl = 0, clip = 0, akl = 0;
  int rc = DFO_OK;
  for (int i = 0; i < nthreads; ++i) {
    pthread_join(th[i], NULL);
    const dfo_loss_out* o = &jobs[i].out;
    if (jobs[i].rc != DFO_OK) rc = jobs[i].rc;
    const double d = c->agg == DFO_AGG_TOKEN_MEAN ? o->n_tokens : o->n_seqs;
    pg += o->pg_loss * d;
    kl += o->kl * d;
    clip += o->clipfrac * o->n_tokens;
    akl += o->approx_kl * o->n_tokens;
    N += o->n_tokens;
    S += o->n_seqs;
  }
  free(th);
  free(jobs);
  const double denom = c->agg == DFO_AGG_TOKEN_MEAN ? N : S;
  out->pg_loss = denom > 0 ? pg / denom : 0.0;
  out->kl = denom > 0 ? kl / denom : 0.0;
  out->loss = out->pg_loss + c->beta * out->kl;
  out->clipfrac = N > 0 ? clip / N : 0.0;
  out->approx_kl = N > 0 ? akl / N : 0.0;
  out->n_tokens = N;
  out->n_seqs = S;
  return rc;
}

/* ---- reshard placement (topology.hpp, data_plane.hpp) ----------------------- */

static int check_layout(uint32_t dp, uint32_t tp, uint32_t world, uint32_t W) {
  if (dp == 0 || tp == 0) return DFO_LAYOUT_ERROR;     /* topology.hpp:56-58 */
  if (dp * tp != world) return DFO_LAYOUT_ERROR;       /* :59-62 */
  if (W % tp != 0) return DFO_LAYOUT_ERROR;            /* :63-67 */
  return DFO_OK;
}

int dfo_reshard_placement(uint32_t B, uint32_t W, uint32_t dp_p, uint32_t tp_p, uint32_t dp_c,
                          uint32_t tp_c, const uint64_t* gc, uint64_t* dest_counts,
                          uint64_t* src_index) {
  if (B == 0 || W == 0) return DFO_LAYOUT_ERROR; /* topology.hpp:28-32 */
  const uint32_t world = B * W;
  int st = check_layout(dp_p, tp_p, world, W);
  if (st) return st;
  st = check_layout(dp_c, tp_c, world, W);
  if (st) return st;
  const uint32_t gpn_p = W / tp_p, gpn_c = W / tp_c;
  uint64_t* goff = (uint64_t*)calloc(dp_p + 1, sizeof(uint64_t));
  for (uint32_t p = 0; p < dp_p; ++p) goff[p + 1] = goff[p] + gc[p];
  /* O_b: store b's groups [b*gpn_p, (b+1)*gpn_p) in dp order (data_plane.hpp:403-409);
   * as indices into `ordered` they are the contiguous range [goff[b*gpn_p], goff[(b+1)*gpn_p]). */
  uint64_t* ob0 = (uint64_t*)malloc(sizeof(uint64_t) * B);
  uint64_t* obn = (uint64_t*)malloc(sizeof(uint64_t) * B);
  for (uint32_t b = 0; b < B; ++b) {
    ob0[b] = goff[b * gpn_p];
    obn[b] = goff[(b + 1) * gpn_p] - ob0[b];
  }
  const uint64_t G = goff[dp_p];
  uint64_t* H = (uint64_t*)malloc(sizeof(uint64_t) * (G ? G : 1));
  uint64_t* h0 = (uint64_t*)calloc(B + 1, sizeof(uint64_t));
  st = DFO_OK;
  if (dp_c == dp_p) {
    /* fast path: H_b = O_b (:411-413) */
    uint64_t w = 0;
    for (uint32_t b = 0; b < B; ++b) {
      h0[b] = w;
      for (uint64_t i = 0; i < obn[b]; ++i) H[w++] = ob0[b] + i;
    }
    h0[B] = w;
  } else {
    for (uint32_t b = 0; b < B; ++b)
      if (obn[b] % B != 0) st = DFO_INDIVISIBLE_ERROR; /* :414-416 */
    if (!st) {
      /* H_k = ||_j O_j[k*q_j, (k+1)*q_j) (:418-435) */
      uint64_t w = 0;
      for (uint32_t k = 0; k < B; ++k) {
        h0[k] = w;
        for (uint32_t j = 0; j < B; ++j) {
          const uint64_t q = obn[j] / B;
          for (uint64_t i = 0; i < q; ++i) H[w++] = ob0[j] + (uint64_t)k * q + i;
        }
      }
      h0[B] = w;
    }
  }
  if (!st) {
    /* get (:273-291): dest d on store k = d / gpn_c receives H_k[(d-k*gpn_c)*r, +r) */
    for (uint32_t k = 0; k < B && !st; ++k)
      if ((h0[k + 1] - h0[k]) % gpn_c != 0) st = DFO_INDIVISIBLE_ERROR; /* :281-283 */
    if (!st) {
      uint64_t w = 0;
      for (uint32_t d = 0; d < dp_c; ++d) {
        const uint32_t k = d / gpn_c;
        const uint64_t r = (h0[k + 1] - h0[k]) / gpn_c;
        const uint64_t at = h0[k] + (uint64_t)(d - k * gpn_c) * r;
        dest_counts[d] = r;
        for (uint64_t i = 0; i < r; ++i) src_index[w++] = H[at + i];
      }
    }
  }
  free(goff);
  free(ob0);
  free(obn);
  free(H);
  free(h0);
  return st;
}

/* ---- record.hpp LE blob ------------------------------------------------------- */

typedef struct {
  uint8_t* out;
  uint64_t n;
} wbuf;

static void w_bytes(wbuf* w, const void* p, uint64_t n) {
  if (w->out && n) memcpy(w->out + w->n, p, n);
  w->n += n;
}
static void w_u32(wbuf* w, uint32_t v) { /* blob::put_u32 record.hpp:45-50 (LE) */
  uint8_t b[4] = {(uint8_t)v, (uint8_t)(v >> 8), (uint8_t)(v >> 16), (uint8_t)(v >> 24)};
  w_bytes(w, b, 4);
}
static void w_u64(wbuf* w, uint64_t v) { /* :52-55 */
  w_u32(w, (uint32_t)v);
  w_u32(w, (uint32_t)(v >> 32));
}

uint64_t dfo_serialize_packed(uint32_t n_records, const uint64_t* ids, const int64_t* meta_off,
                              const uint8_t* meta_blob, const int32_t* go, const uint32_t* tok_count,
                              const int64_t* cu, int n_streams, const void* const* streams,
                              const uint32_t* esz, int n_ch, const char* const* ch_names,
                              const double* const* ch_vals, uint8_t* out) {
  wbuf w = {out, 0};
  w_u32(&w, n_records); /* serialize_records :151-156 */
  for (uint32_t r = 0; r < n_records; ++r) {
    w_u64(&w, ids[r]); /* serialize_record :109-127 */
    if (meta_off) {
      w_bytes(&w, meta_blob + meta_off[r], (uint64_t)(meta_off[r + 1] - meta_off[r]));
    } else {
      w_u32(&w, 0);
    }
    w_u32(&w, (uint32_t)(go[r + 1] - go[r]));
    for (int32_t s = go[r]; s < go[r + 1]; ++s) {
      w_u32(&w, tok_count[s]);
      uint64_t plen = 0;
      for (int k = 0; k < n_streams; ++k) plen += (uint64_t)(cu[s + 1] - cu[s]) * esz[k];
      w_u64(&w, plen);
      for (int k = 0; k < n_streams; ++k)
        w_bytes(&w, (const uint8_t*)streams[k] + (uint64_t)cu[s] * esz[k],
                (uint64_t)(cu[s + 1] - cu[s]) * esz[k]);
      w_u32(&w, (uint32_t)n_ch);
      for (int c = 0; c < n_ch; ++c) {
        const uint32_t nl = (uint32_t)strlen(ch_names[c]);
        w_u32(&w, nl);
        w_bytes(&w, ch_names[c], nl);
        uint64_t bits;
        memcpy(&bits, &ch_vals[c][s], 8); /* put_f64 :57-59 (bit_cast) */
        w_u64(&w, bits);
      }
    }
  }
  return w.n;
}
