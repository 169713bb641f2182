/*
 * dfx.h -- C ABI of the B200-native DistFlow post-rollout hot path (libdfx.so).
 *
 * Plain C types, device pointers and sizes only; no torch types. Every entry
 * point names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/). The C++ drop-in shims
 * that keep the reference's StageFn / FunctionRegistry / BufferStore API are
 * in include/dfx_distflow.hpp; the Python mirror is paper_2507_13833_b200/.
 *
 * Conventions
 *   - Return value: dfx_status (0 = OK). On failure dfx_last_error() returns a
 *     thread-local message. Codes mirror the reference's typed exceptions
 *     (distflow/errors.hpp), so shims can rethrow the same types.
 *   - All compute calls are asynchronous on the given CUDA stream and never
 *     allocate: scratch comes from a caller-provided workspace sized by the
 *     matching *_workspace_bytes() query. Calls are re-entrant across threads
 *     and devices (no global mutable state besides the error message).
 *   - Kernels launch on the calling thread's current device, which must own
 *     the stream and the (non-peer) buffers (cudaSetDevice first when one
 *     thread drives several GPUs; the Python layer does this per batch).
 *   - There is no CPU fallback: without a CUDA device every compute call
 *     returns DFX_CUDA_ERROR.
 */
#ifndef DFX_H
#define DFX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dfx_stream; /* == cudaStream_t */
typedef int32_t dfx_status;

enum {
  DFX_OK = 0,
  DFX_ERROR = 1,                 /* distflow::Error                errors.hpp:10 */
  DFX_LAYOUT_ERROR = 2,          /* LayoutError                    errors.hpp:32 */
  DFX_INDIVISIBLE_ERROR = 3,     /* IndivisibleError               errors.hpp:52 */
  DFX_MISSING_ROLLOUTS = 4,      /* MissingRolloutsError           errors.hpp:123 */
  DFX_MISSING_CHANNEL = 5,       /* MissingChannelError            errors.hpp:116 */
  DFX_STALE_ITERATION = 6,       /* StaleIterationError            errors.hpp:99 */
  DFX_NOT_READY = 7,             /* NotReadyError                  errors.hpp:104 */
  DFX_UNKNOWN_STAGE = 8,         /* UnknownStageError              errors.hpp:109 */
  DFX_INVALID_ARGUMENT = 9,
  DFX_CUDA_ERROR = 10,
  DFX_NCCL_ERROR = 11,
};

const char* dfx_last_error(void);
const char* dfx_version(void);

/* ---------------------------------------------------------------------------
 * Packed batch (device SoA). Replaces the AoS SampleBatch / SampleRecord /
 * Rollout model (distflow/record.hpp:17-41) on the device.
 *
 * A batch is n_records prompt records; record r owns rollouts
 * [group_off[r], group_off[r+1]) (records are atomic, record.hpp:25-26);
 * rollout s owns tokens [cu_seqlens[s], cu_seqlens[s+1]).
 * cu_seqlens values are ABSOLUTE indices into the token streams, so a view of
 * a sub-range of rollouts is just a pointer offset into group_off/cu_seqlens
 * with the same token stream base pointers (zero-copy slicing).
 * Token streams must be 16-byte aligned at index 0 and readable on
 * [cu_seqlens[0] & ~7, (cu_seqlens[n_rollouts] + 7) & ~7) (kernels issue
 * aligned 128-bit loads and discard the out-of-range lanes).
 * Calls take token_base = cu_seqlens[0] and token_span =
 * cu_seqlens[n_rollouts] - cu_seqlens[0] from the host (the packer knows them),
 * so no call ever reads device memory on the host.
 * Rollout channels are f64 (the reference's channel type, record.hpp:20).
 * Pointers not needed by a call may be NULL.
 * ------------------------------------------------------------------------- */
typedef struct dfx_packed {
  int64_t n_records;
  int64_t n_rollouts;
  const int32_t* group_off;   /* [n_records+1] rollout offsets, group_off[0]==0 */
  const int32_t* roll_group;  /* [n_rollouts] record index of each rollout */
  const int64_t* cu_seqlens;  /* [n_rollouts+1] absolute token offsets */
  const double* reward;       /* [n_rollouts] channel "reward" */
  const double* value;        /* [n_rollouts] channel "value" */
  const float* lp;            /* current-policy log-probs */
  const float* old_lp;        /* rollout-policy log-probs */
  const float* ref_lp;        /* reference-policy log-probs */
  const float* value_tok;     /* per-token critic values (GAE) */
  const float* token_reward;  /* per-token rewards (GAE) */
  const uint8_t* mask;        /* response mask, 0/1 */
} dfx_packed;

/* ---------------------------------------------------------------------------
 * Advantages
 * ------------------------------------------------------------------------- */

/* Replaces fn_group_advantage (distflow/functions.hpp:143-161).
 * Per record: f64 mean and population std of the rollouts' rewards,
 * adv = d == 0 ? 0 : d / (std + eps). Bit-identical to the reference (same
 * operation order, no FMA contraction). Writes adv_roll[n_rollouts] (f64).
 * An empty record sets kFlagMissingRollouts in *flags (device, nullable);
 * dfx_check_flags() turns it into DFX_MISSING_ROLLOUTS. */
dfx_status dfx_grpo_advantage(const dfx_packed* b, double eps, double* adv_roll, int32_t* flags,
                              dfx_stream stream);

/* Per-token broadcast (new): adv_tok[t] = mask[t] ? f32(adv_roll[s]) : 0 for
 * every token t of rollout s, indexed like the token streams. */
dfx_status dfx_broadcast_advantage(const dfx_packed* b, int64_t token_base, int64_t token_span,
                                   const double* adv_roll, float* adv_tok, dfx_stream stream);

/* Replaces fn_ppo_advantage (distflow/functions.hpp:163-172): adv = reward - value. */
dfx_status dfx_ppo_advantage(const dfx_packed* b, double* adv_roll, dfx_stream stream);

/* GAE reverse scan (new; the reference has none). Per rollout:
 *   m1 = t+1<L ? mask[t+1] : 0, v1 = t+1<L ? V[t+1] : 0
 *   delta_t = r_t + gamma*m1*v1 - V_t ;  A_t = delta_t + gamma*lam*m1*A_{t+1} ;  R_t = A_t + V_t
 * computed in f64 inside the kernel, stored f32. Optionally writes the masked
 * whitening sums whiten[3] = {sum m*A, sum m*A^2, sum m} (device f64). */
/* One reverse affine scan over the whole token line (the chain breaks at rollout
 * ends by itself): a prep kernel marks rollout ends in a token bitmap and cuts
 * the line into rollout-aligned segments (about one per resident CTA); a
 * persistent CTA scans its segment right to left in 2048-token tiles through a
 * TMA ring, the carry in a register (a segment that cuts a rollout longer than
 * 64K tokens takes the value its right neighbour publishes); f32
 * inputs/outputs, deltas and recurrences in f64; with whitening a finish kernel
 * reduces the per-segment sums in segment order. Outputs are bit-identical run
 * to run. Workspace (dfx_gae_workspace_bytes) must be zero-filled once at
 * allocation; the kernels keep it consistent across calls (epoch-tagged
 * records, the end bitmap cleared as it is consumed), so it can be reused --
 * by calls of any span up to its capacity: its layout depends only on
 * ws_bytes -- and graph-captured. */
size_t dfx_gae_workspace_bytes(int64_t n_rollouts, int64_t token_span);
dfx_status dfx_gae(const dfx_packed* b, int64_t token_base, int64_t token_span, double gamma, double lam,
                   float* adv, float* ret, double* whiten, void* workspace, size_t ws_bytes, dfx_stream stream);

/* GAE fused with the PPO loss (new): one scan pass computes every token's
 * advantage and, from it, the clipped surrogate + KL terms -- the advantage
 * never goes to HBM (adv may be NULL; ret is written for the critic). Token-
 * mean aggregation of unwhitened advantages only (cfg->agg ==
 * DFX_AGG_TOKEN_MEAN, cfg->whiten == 0: whitening needs the global advantage
 * statistics first -- use dfx_gae then dfx_ppo_loss). The scan is the
 * 4096-token-tile decoupled look-back (its per-tile loss phase is hidden by five
 * independent CTAs per SM); numerics as dfx_gae followed by dfx_ppo_loss with
 * DFX_ADV_TOKEN, within f64 rounding, deterministic.
 * Workspace zero-filled once at allocation (as dfx_gae's). */
typedef struct dfx_loss_cfg dfx_loss_cfg;
typedef struct dfx_loss_out dfx_loss_out;
size_t dfx_gae_ppo_loss_workspace_bytes(int64_t n_rollouts, int64_t token_span);
dfx_status dfx_gae_ppo_loss(const dfx_packed* b, int64_t token_base, int64_t token_span, double gamma, double lam,
                            const dfx_loss_cfg* cfg, float* ret, float* adv, dfx_loss_out* out, void* workspace,
                            size_t ws_bytes, dfx_stream stream);

/* ---------------------------------------------------------------------------
 * PPO / GRPO clipped surrogate + KL + masked aggregation (new; fills the
 * fn_train slot, distflow/functions.hpp:176-182, node actor_train dag.hpp:335)
 * ------------------------------------------------------------------------- */
#define DFX_MAX_LOSS_GROUPS 16384
enum { DFX_KL_NONE = 0, DFX_KL_K1 = 1, DFX_KL_K2 = 2, DFX_KL_K3 = 3 };
enum { DFX_AGG_TOKEN_MEAN = 0, DFX_AGG_SEQ_MEAN_TOKEN_MEAN = 1, DFX_AGG_SEQ_MEAN_TOKEN_SUM = 2 };
enum {
  DFX_ADV_GROUP_FUSED = 0, /* GRPO: group stats from b->reward computed in-kernel (bit-exact) */
  DFX_ADV_ROLLOUT = 1,     /* per-rollout f64 advantage (adv_roll), broadcast to tokens */
  DFX_ADV_TOKEN = 2,       /* per-token f32 advantage (adv_tok_in), e.g. from dfx_gae */
};

typedef struct dfx_loss_cfg {
  double clip_low;   /* ratio clipped to [1-clip_low, 1+clip_high] */
  double clip_high;
  double beta;       /* KL coefficient */
  double adv_eps;    /* DFX_ADV_GROUP_FUSED: StageContext::advantage_eps (functions.hpp:59) */
  int32_t kl_type;   /* DFX_KL_* ; k3 is clamped to [-10, 10] */
  int32_t agg;       /* DFX_AGG_* */
  int32_t adv_source;/* DFX_ADV_* */
  int32_t whiten;    /* 1: A_w = (A - mu) * rsqrt(var_unbiased + 1e-8), from whiten_sums */
} dfx_loss_cfg;

/* One per loss group (device memory), all f64. */
typedef struct dfx_loss_out {
  double loss, pg_loss, kl, clipfrac, approx_kl, n_tokens, n_seqs;
} dfx_loss_out;

typedef struct dfx_loss_args {
  double* adv_roll;              /* DFX_ADV_ROLLOUT input; DFX_ADV_GROUP_FUSED output (nullable) */
  const float* adv_tok_in;       /* DFX_ADV_TOKEN input */
  const double* whiten_sums;     /* cfg.whiten: {sum m*A, sum m*A^2, sum m} (device) */
  float* adv_tok_out;            /* nullable: per-token advantage actually used (after whitening) */
  float* dlogp;                  /* nullable: d loss / d lp per token (extra mask pre-pass) */
  int32_t n_loss_groups;         /* >=1; 0 treated as 1 */
  const int32_t* loss_group_off; /* device [n_loss_groups+1] rollout offsets, NULL for one group */
  dfx_loss_out* out;             /* device [n_loss_groups] */
  int32_t* flags;                /* nullable device error flags (fused GRPO: empty record) */
  void* ev_main_begin;           /* nullable cudaEvent_t recorded right before / after the streaming */
  void* ev_main_end;             /*   kernel (roofline timing of the dominant kernel on its stream) */
} dfx_loss_args;

/* Workspace must be zero-filled once at allocation; every call leaves its
 * ticket counters zeroed again. The tickets sit at fixed offsets (any batch
 * size, at most DFX_MAX_LOSS_GROUPS loss groups), so a workspace can be reused
 * by calls of any size up to ws_bytes. One launch of the fused streaming kernel plus
 * one finalize launch (two more when dlogp is requested). */
size_t dfx_ppo_loss_workspace_bytes(int64_t n_rollouts, int64_t token_span, int32_t n_loss_groups);
dfx_status dfx_ppo_loss(const dfx_packed* b, int64_t token_base, int64_t token_span,
                        const dfx_loss_cfg* cfg,
                        const dfx_loss_args* args, void* workspace, size_t ws_bytes,
                        dfx_stream stream);

/* Multi-source loss (the reshard's consumer side fused with the loss): one call
 * over up to 4 packed batches, each in its own token coordinates -- e.g. the
 * local producer group and the TP partner's producer group mapped from the
 * partner GPU (dfx_ipc_open), read over NVLink by the streaming kernel itself
 * instead of being copied first. Rollouts are numbered across the sources in
 * order; loss_group_off (args) uses that numbering. Per-token inputs/outputs
 * are per source: args->adv_roll/adv_tok_in/adv_tok_out/dlogp are ignored.
 * DFX_ADV_GROUP_FUSED needs a single source. */
typedef struct dfx_loss_src {
  dfx_packed b;              /* cu_seqlens, lp, old_lp, ref_lp, mask (device or peer-mapped pointers) */
  int64_t token_base, token_span;
  const double* adv_roll;    /* DFX_ADV_ROLLOUT: this source's per-rollout advantages */
  const float* adv_tok_in;   /* DFX_ADV_TOKEN */
  float* adv_tok_out;        /* nullable; indexed like this source's token streams */
  float* dlogp;              /* nullable (all sources or none); likewise */
} dfx_loss_src;
size_t dfx_ppo_loss_multi_workspace_bytes(const dfx_loss_src* srcs, int32_t n_src, int32_t n_loss_groups);
dfx_status dfx_ppo_loss_multi(const dfx_loss_src* srcs, int32_t n_src, const dfx_loss_cfg* cfg,
                              const dfx_loss_args* args, void* workspace, size_t ws_bytes, dfx_stream stream);

/* TP-split loss: when a consumer group's records sit on several GPUs (its TP
 * workers' producers), each TP rank runs the loss over the rollouts it holds
 * and the ranks exchange their dfx_loss_out rows (an all-gather of 56 B per
 * group); this folds parts[n_parts][n_groups] (device, rank order) into the
 * group results, re-weighting each mean by its denominator. Every rank gets
 * the same bits. Token-mean / sequence-mean aggregations (no whitening/dlogp,
 * which need group-wide statistics before the streaming pass). */
dfx_status dfx_loss_combine(const dfx_loss_out* parts, int32_t n_parts, int32_t n_groups, const dfx_loss_cfg* cfg,
                            dfx_loss_out* out, dfx_stream stream);

/* Per-iteration reward statistics, replacing detail::record_reward_stats
 * (worker.hpp:177-190): out[0..3) = {count, sum, sum of squares} of the
 * rollouts' "reward" channel (device f64), so the cluster reduction of
 * aggregate_metrics (worker.hpp:275-325) is one scalar all-reduce. */
dfx_status dfx_reward_stats(const dfx_packed* b, double* out, dfx_stream stream);

/* Device-side error flags written by kernels (e.g. an empty record seen by the
 * fused GRPO path). Reads flags (device int32) and returns the status. Syncs. */
dfx_status dfx_check_flags(const int32_t* flags, dfx_stream stream);

/* ---------------------------------------------------------------------------
 * Synthetic rollouts on device: the same counter-keyed
 * SplitMix64 values as the CPU generator (oracle/dfx_oracle.h), bit-exact.
 * ids: device [n_records] sample ids; n_roll rollouts per record;
 * cu_seqlens: device [n_records*n_roll+1]. Any output may be NULL.
 * ------------------------------------------------------------------------- */
dfx_status dfx_synth_tokens(uint64_t seed, const uint64_t* ids, int64_t n_records, int32_t n_roll,
                            const int64_t* cu_seqlens, int64_t token_base, int64_t token_span, float* lp,
                            float* old_lp, float* ref_lp, float* value_tok, float* token_reward,
                            uint8_t* mask, int32_t* token_id, dfx_stream stream);

/* fn_generate (distflow/functions.hpp:108-123) on the device, bit-exact.
 * dfx_generate_counts: tok_count[s] (device u32, s = r * n_roll + j) =
 *   draw_tokens(dist, seed, ids[r], j) (functions.hpp:67-80; kind 0 CONSTANT
 *   (value), 1 UNIFORM [min, max], 2 SKEWED [min, max]). Errors as the
 *   reference: rollouts_per_prompt < 1, max < min -> DFX_INVALID_ARGUMENT.
 * dfx_generate_payload: payload bytes [payload_off[s], payload_off[s+1]) =
 *   hash_bytes(keyed_hash(seed, "payload", ids[r], j), len) (hash.hpp:48-59);
 *   payload_off: device i64 [n_records*n_roll + 1], the exclusive prefix of
 *   tok_count * bytes_per_token. ids: device. */
dfx_status dfx_generate_counts(uint64_t seed, int32_t kind, uint32_t value, uint32_t min_tokens, uint32_t max_tokens,
                               const uint64_t* ids, int64_t n_records, int32_t n_roll, uint32_t* tok_count,
                               dfx_stream stream);
dfx_status dfx_generate_payload(uint64_t seed, const uint64_t* ids, int64_t n_records, int32_t n_roll,
                                const int64_t* payload_off, uint8_t* payload, dfx_stream stream);

/* ---------------------------------------------------------------------------
 * DataBuffer reshard (DP m->n), replacing BufferStore::exchange/get
 * (distflow/data_plane.hpp:237-442) and all_to_all (distflow/transport.hpp:718-754)
 * for device-resident batches.
 * ------------------------------------------------------------------------- */

/* Host-only. The reference placement as an index list: for every consumer
 * group d (dest-major) the records it receives, as indices into
 * ordered = L_0 || ... || L_{dp_p-1} (L_p = producer group p's records).
 * Errors: DFX_LAYOUT_ERROR (topology.hpp:53-68), DFX_INDIVISIBLE_ERROR
 * (data_plane.hpp:414-416, :281-283). src_index may be NULL. */
dfx_status dfx_reshard_placement(uint32_t num_nodes, uint32_t workers_per_node, uint32_t dp_p, uint32_t tp_p,
                                 uint32_t dp_c, uint32_t tp_c, const uint64_t* group_counts,
                                 uint64_t* dest_counts, uint64_t* src_index);

/* One maximal run of consecutive records: producer group src_group's records
 * [src_rec, src_rec+count) become consumer group dst_group's records
 * [dst_rec, dst_rec+count). */
typedef struct dfx_segment {
  uint32_t dst_group;
  uint32_t src_group;
  uint64_t dst_rec;
  uint64_t src_rec;
  uint64_t count;
} dfx_segment;

/* Host-only. Writes up to cap segments (dest-major order) and returns the
 * total count, or -status on a layout/divisibility error. */
int64_t dfx_reshard_segments(uint32_t num_nodes, uint32_t workers_per_node, uint32_t dp_p, uint32_t tp_p,
                             uint32_t dp_c, uint32_t tp_c, const uint64_t* group_counts, dfx_segment* out,
                             int64_t cap);

/* Device-side metadata of one segment: pointers at the slice start of the
 * source arrays (a local producer batch, or a received pack buffer): ids
 * [n_rec], group_off [n_rec+1] and cu_seqlens [n_roll+1] (source-absolute
 * values), up to 4 f64 rollout channels [n_roll]; plus destination offsets
 * (records, rollouts, absolute token index in the destination streams). */
typedef struct dfx_seg_meta {
  const uint64_t* ids;
  const int32_t* group_off;
  const int64_t* cu;
  const double* ch[4];
  int64_t n_rec, n_roll;
  int64_t dst_rec, dst_roll, dst_tok;
} dfx_seg_meta;

/* Pack segments' metadata into contiguous send buffers (one CTA per segment):
 * ids u64[n_rec] | cu i64[n_roll+1] | ch f64[n_ch][n_roll] | group_off i32[n_rec+1].
 * segs and out are HOST arrays (the table travels in the kernel parameters);
 * the pointers inside may be device or peer-mapped addresses. n_ch <= 4. */
int64_t dfx_reshard_pack_bytes(int64_t n_rec, int64_t n_roll, int32_t n_ch);
dfx_status dfx_reshard_pack(const dfx_seg_meta* segs, int32_t n_segs, int32_t n_ch, uint8_t* const* out,
                            dfx_stream stream);
/* Unpack into the destination batch, rebasing group_off / cu_seqlens and
 * rebuilding roll_group. segs and dst_ch are HOST arrays (n_ch <= 4 channel
 * pointers into the destination). */
dfx_status dfx_reshard_unpack(const dfx_seg_meta* segs, int32_t n_segs, int32_t n_ch, uint64_t* dst_ids,
                              int32_t* dst_group_off, int32_t* dst_roll_group, int64_t* dst_cu,
                              double* const* dst_ch, dfx_stream stream);

/* ---------------------------------------------------------------------------
 * The reference's record wire format on the device:
 * serialize_records (distflow/record.hpp:109-127, 151-156) of a packed batch,
 * byte-identical to the CPU serializer, so device batches can be handed to CPU
 * peers (Fabric / BufferStore::exchange) without a host repack.
 * Payload of rollout s: for each stream k in order, its tokens' elements
 * (esz[k] bytes each) -- e.g. token_id i32 | lp f32 | old f32 | ref f32 | mask u8.
 * Channels in the given order (pass them sorted by name: std::map order).
 * meta_blob/meta_off (device, nullable): each record's pre-serialized meta
 * section (u32 count + (str, str)*); NULL writes an empty section.
 * tok_count (device, nullable): Rollout::token_count, default cu[s+1]-cu[s].
 * dfx_serialize_plan (host-only) fills rec_off[n_records+1] (byte offset of
 * each record after the leading u32) from host copies of group_off / cu /
 * meta_off and returns the blob size, or -status. Copy rec_off to the device
 * for dfx_serialize_records. meta_blob must be readable 4 bytes past its end.
 * ------------------------------------------------------------------------- */
int64_t dfx_serialize_plan(int64_t n_records, const int32_t* h_group_off, const int64_t* h_cu,
                           const int64_t* h_meta_off, int32_t n_streams, const uint32_t* esz, int32_t n_ch,
                           const char* const* ch_names, int64_t* rec_off);
dfx_status dfx_serialize_records(const dfx_packed* b, const uint64_t* ids, const uint32_t* tok_count,
                                 int32_t n_streams, const void* const* streams, const uint32_t* esz, int32_t n_ch,
                                 const char* const* ch_names, const double* const* ch, const uint8_t* meta_blob,
                                 const int64_t* meta_off, const int64_t* rec_off, uint8_t* out, dfx_stream stream);

/* deserialize_records (record.hpp:129-149, 158-165) into a packed batch: a
 * host header walk builds the index (call once with every output NULL for
 * the counts, then with arrays: ids[R], meta_range[2R] (start, end of record
 * r's meta section in the blob), group_off[R+1], cu[S+1], tok_count[S], payload_off[S], ch_off[S]);
 * every rollout must carry the channels ch_names (blob order) and a payload of
 * a whole number of bytes_per_token. A truncated or malformed blob returns
 * DFX_ERROR (the reference's ParseError). dfx_blob_unpack then gathers, on the
 * device, every payload into the token streams and the channel values into
 * f64 arrays (blob, cu, payload_off, ch_off: device copies). */
dfx_status dfx_blob_index(const uint8_t* blob, uint64_t size, uint32_t bytes_per_token, int32_t n_ch,
                          const char* const* ch_names, int64_t* n_records, int64_t* n_rollouts, int64_t* n_tokens,
                          uint64_t* ids, int64_t* meta_range, int32_t* group_off, int64_t* cu, uint32_t* tok_count,
                          int64_t* payload_off, int64_t* ch_off);
dfx_status dfx_blob_unpack(const uint8_t* blob, int64_t n_rollouts, const int64_t* cu, const int64_t* payload_off,
                           const int64_t* ch_off, int32_t n_streams, void* const* streams, const uint32_t* esz,
                           int32_t n_ch, const char* const* ch_names, double* const* ch, dfx_stream stream);

/* Peer memory for the NVLink pull transport. dfx_ipc_export returns the IPC
 * handle of the allocation containing ptr and ptr's offset in it; a peer maps
 * it with dfx_ipc_open. Map a peer process's allocation
 * (cudaIpcMemHandle_t bytes, handle_bytes == 64) into the CURRENT device's
 * context with lazy peer access, cached per (device, handle) -- no context is
 * created on the peer device. dfx_copy_async is cudaMemcpyAsync(Default) so
 * peer-mapped sources copy over NVLink on the caller's stream. */
dfx_status dfx_ipc_export(const void* ptr, void* handle_out /* 64 bytes */, uint64_t* offset_out);
dfx_status dfx_ipc_open(const void* handle, size_t handle_bytes, void** base);
/* Drop one reference taken by dfx_ipc_open on the current device; the mapping
 * is closed (cudaIpcCloseMemHandle) when the last reference goes. The caller
 * must have completed every read of it (stream-synchronized). */
dfx_status dfx_ipc_close(void* base);
int64_t dfx_ipc_open_count(void); /* live mappings in this process (tests) */
dfx_status dfx_copy_async(void* dst, const void* src, size_t bytes, dfx_stream stream);
/* Record metadata of a zero-copy view of records [r0, r1) of a batch, on the device: group_off rebased to the
 * view's first rollout ([r1-r0+1]) and roll_group rebased to r0 ([n_roll] = group_off[r1]-group_off[r0]). */
dfx_status dfx_view_meta(const int32_t* group_off, const int32_t* roll_group, int64_t r0, int64_t r1, int64_t n_roll,
                         int32_t* group_off_out, int32_t* roll_group_out, dfx_stream stream);
/* Same-device copy by a kernel (HBM to HBM on the SMs; the copy engines' D2D path is ~6x slower). */
dfx_status dfx_copy_sm(void* dst, const void* src, size_t bytes, dfx_stream stream);
/* n copies (dst[i] <- src[i], bytes[i]; addresses as integers, device or peer-mapped) by ONE kernel launch per
 * 96 copies: local and NVLink-mapped sources copied concurrently by the SMs in 64 KB chunks. */
dfx_status dfx_copy_many(int64_t n, const uint64_t* dst, const uint64_t* src, const uint64_t* bytes,
                         dfx_stream stream);
/* n copies (dst[i] <- src[i], bytes[i]; addresses as integers, device or peer-mapped) in one call. */
dfx_status dfx_copy_batch(int64_t n, const uint64_t* dst, const uint64_t* src, const uint64_t* bytes,
                          dfx_stream stream);

/* ---------------------------------------------------------------------------
 * Distributed DataBuffer: the reference's BufferStore (distflow/data_plane.hpp:
 * 225-457) for one process per GPU, native end to end. Replaces put /
 * ensure_ready / exchange / get and the all_to_all behind them
 * (data_plane.hpp:400-442, transport.hpp:718-754): one host call per verb, no
 * Python and no host-side collective library on the data path.
 *
 * Communicator: an NCCL communicator over the participating GPUs (one rank per
 * process). Rank 0 makes the id (dfx_comm_unique_id) and ships its bytes to the
 * others by any side channel (a pipe, a file, torch's TCPStore); every rank
 * then calls dfx_comm_init with its device current.
 * ------------------------------------------------------------------------- */
#define DFX_COMM_ID_BYTES 128
#define DFX_MAX_CH 4
#define DFX_MAX_STREAMS 8
typedef struct dfx_comm dfx_comm;
dfx_status dfx_comm_unique_id(void* id_out /* DFX_COMM_ID_BYTES */);
dfx_status dfx_comm_init(const void* id, int32_t n_ranks, int32_t rank, dfx_comm** out);
dfx_status dfx_comm_destroy(dfx_comm* comm);
int32_t dfx_comm_rank(const dfx_comm* comm);
int32_t dfx_comm_size(const dfx_comm* comm);
/* Sum of n int64 values over the ranks, host in / host out (one device
 * all-reduce on the stream + a D2H read; synchronizes the stream). */
dfx_status dfx_comm_allreduce_i64(dfx_comm* comm, const int64_t* in, int64_t* out, int64_t n, dfx_stream stream);

/* All-to-all of device byte buffers: this rank sends send_bytes[p] bytes at
 * send + send_off[p] to every rank p and receives recv_bytes[p] bytes into
 * recv + recv_off[p] (sizes agreed beforehand, e.g. through
 * dfx_comm_allreduce_i64). One grouped NCCL call on the stream; the self part
 * is a device copy. The transport under dfx_distflow::NcclFabric. */
dfx_status dfx_comm_alltoallv(dfx_comm* comm, const void* send, const uint64_t* send_off, const uint64_t* send_bytes,
                              void* recv, const uint64_t* recv_off, const uint64_t* recv_bytes, dfx_stream stream);

/* A device batch in a store's schema (generic form of dfx_packed): streams and
 * channels in the schema's order; group_off is relative (group_off[0] == 0);
 * cu_seqlens are absolute token indices into the streams (st[k] points at token
 * 0 of the coordinate system). h_group_off / h_cu: host copies (the store plans
 * from them; it never reads device metadata on the host). */
typedef struct dfx_batch {
  int64_t n_records, n_rollouts, token_base, token_span;
  const uint64_t* ids;
  const int32_t* group_off;
  const int32_t* roll_group;
  const int64_t* cu_seqlens;
  const double* ch[DFX_MAX_CH];
  const void* st[DFX_MAX_STREAMS];
  const int32_t* h_group_off;
  const int64_t* h_cu;
} dfx_batch;

/* Transports of remote segments: PULL maps the producers' allocations (CUDA IPC)
 * and the consumer's copy engines read them over NVLink; NCCL posts one grouped
 * ncclSend/ncclRecv per exchange (the library baseline, ~2.5x slower here). */
enum { DFX_TRANSPORT_PULL = 0, DFX_TRANSPORT_NCCL = 1 };
typedef struct dfx_dstore_cfg {
  uint32_t num_nodes, workers_per_node;  /* the reference's B x W logical world (topology.hpp:11-35) */
  const int32_t* rank_of_worker;         /* [B*W]: the process (GPU) rank hosting each logical worker */
  int32_t n_streams;                     /* token streams per rollout (<= DFX_MAX_STREAMS) */
  const uint32_t* stream_esz;            /* their element sizes in bytes */
  int32_t n_ch;                          /* f64 rollout channels (<= DFX_MAX_CH) */
  int32_t n_stages;
  const char* const* stage_names;        /* StoreStagePlan per stage (data_plane.hpp:216-220) */
  const uint32_t* produced_dp;
  const uint32_t* produced_tp;
  const uint32_t* consumed_dp;           /* 0: the layout is given to ensure_ready (fallback_to_layout) */
  const uint32_t* consumed_tp;
  int32_t transport;                     /* DFX_TRANSPORT_PULL (default) or DFX_TRANSPORT_NCCL */
} dfx_dstore_cfg;
typedef struct dfx_dstore dfx_dstore;

/* All work is enqueued on `stream` (the caller's compute stream, so consumers
 * are ordered after the exchange with no extra synchronization). */
dfx_status dfx_dstore_create(const dfx_dstore_cfg* cfg, dfx_comm* comm, dfx_stream stream, dfx_dstore** out);
dfx_status dfx_dstore_destroy(dfx_dstore* s);
/* BufferStore::put (data_plane.hpp:237-264): TP != 0 is suppressed (*accepted
 * = 0); the group must be local to this rank; duplicates and stale iterations
 * are errors. The batch's memory must stay valid until ensure_ready returns
 * (the exchange reads it on the stream). */
dfx_status dfx_dstore_put(dfx_dstore* s, const char* stage, uint64_t iteration, uint32_t dp, uint32_t tp,
                          const dfx_batch* batch, int32_t* accepted);
/* BufferStore::ensure_ready / exchange (:296-346, :400-442), collective over
 * the communicator: one all-reduce of the producer sizes (cached plan when they
 * repeat; the producers' IPC handles travel only when their memory changed),
 * then the reshard on the stream -- remote token runs pulled by the copy
 * engines over NVLink (or NCCL send/recv), local segments by one copy kernel on
 * a forked stream, one unpack kernel. Consumer groups that are one contiguous
 * run of local producer memory are zero-copy views. DFX_NOT_READY if a local
 * producer group has not put. Put batches must stay unmodified until
 * worker_done retires the iteration (peers may read them until then). */
dfx_status dfx_dstore_ensure_ready(dfx_dstore* s, const char* stage, uint64_t iteration, uint32_t to_dp,
                                   uint32_t to_tp);
/* BufferStore::get (:269-292): consumer group dest_dp's batch on this GPU (TP
 * peers on one GPU share it), valid until worker_done retires the iteration. */
dfx_status dfx_dstore_get(dfx_dstore* s, const char* stage, uint64_t iteration, uint32_t dest_dp, uint32_t to_dp,
                          uint32_t to_tp, dfx_batch* out);
/* BufferStore::worker_done (:351-367): once per local logical worker. */
dfx_status dfx_dstore_worker_done(dfx_dstore* s, uint64_t iteration);
/* {suppressed puts, NVLink bytes sent, NVLink bytes received, local bytes copied, plan cache hits} */
dfx_status dfx_dstore_stats(const dfx_dstore* s, uint64_t* out5);

/* ---------------------------------------------------------------------------
 * Timing helpers (cudaEvent_t as void*), so ctypes callers can bracket a
 * kernel on the stream it runs on.
 * ------------------------------------------------------------------------- */
dfx_status dfx_event_create(void** ev);
dfx_status dfx_event_destroy(void* ev);
dfx_status dfx_event_record(void* ev, dfx_stream stream);
dfx_status dfx_event_elapsed_ms(void* ev_begin, void* ev_end, float* ms); /* syncs ev_end */

#ifdef __cplusplus
}
#endif
#endif
