/*
 * tt.h — the drop-in C ABI of the B200 draft+verify exploration round.
 *
 * Every entry point is extern "C", takes plain pointers and sizes, and
 * returns an int status (TT_OK = 0). The error codes mirror tiletune::Error
 * codes (proj/core/include/tiletune/common.hpp:44-50) plus TT_E_CUDA; the
 * message of the last failure on a context is tt_last_error(ctx). Each
 * function names the reference interface it replaces.
 *
 * Memory: arguments named *_dev are device pointers, *_host host pointers;
 * everything is caller-owned. A context owns one CUDA stream (or adopts the
 * caller's via tt_ctx_set_stream) plus its scratch; calls on one context are
 * serialised on its stream, distinct contexts are independent. Functions
 * documented "async" only enqueue work on the stream.
 *
 * There is no CPU fallback: every compute entry point launches sm_100a
 * kernels and fails with TT_E_CUDA when no device is usable.
 */
#ifndef TT_TT_H_
#define TT_TT_H_

#include <stdint.h>

#include "tt_types.h"

#ifdef __cplusplus
extern "C" {
#endif

enum tt_status {
  TT_OK = 0,
  TT_E_PARSE = 1,    /* tiletune::err::kParse */
  TT_E_VALIDATE = 2, /* tiletune::err::kValidate */
  TT_E_CONFIG = 3,   /* tiletune::err::kConfig */
  TT_E_STATE = 4,    /* tiletune::err::kState */
  TT_E_IO = 5,       /* tiletune::err::kIo */
  TT_E_CUDA = 6,     /* device / launch failure */
  TT_E_NCCL = 7      /* collective failure (tt_comm_*) */
};

/* tt_round_result.status bits above the selector's own (low byte) */
enum tt_round_flags {
  TT_ROUND_BAND_RERUN = 1 << 16 /* bf16 error on the rescored set exceeded the band: re-run in fp64 */
};

/* PaCM arithmetic for tt_pacm_score / tt_round */
enum tt_precision {
  TT_PREC_FP64 = 0, /* CUDA-core fp64, reference accumulation order (parity mode) */
  TT_PREC_BF16 = 1  /* tcgen05 tensor cores, bf16 operands, fp32 TMEM accumulators */
};

typedef struct tt_ctx tt_ctx;

/* "E_VALIDATE" etc. — the reference's stable code strings */
const char* tt_status_code(int status);
const char* tt_version(void);
/* Number of CUDA kernels this library has launched (process-wide). */
uint64_t tt_kernel_launches(void);

/* ------------------------------------------------------------ context -- */
int tt_ctx_create(int device, tt_ctx** out);
void tt_ctx_destroy(tt_ctx* ctx);
const char* tt_last_error(const tt_ctx* ctx);
int tt_ctx_set_stream(tt_ctx* ctx, void* cuda_stream); /* NULL restores the ctx stream */
void* tt_ctx_stream(const tt_ctx* ctx);
int tt_ctx_sync(tt_ctx* ctx);

/* ------------------------------------------------ problem model (host) -- */
/* generate_sketch(op, elementwise_fallback) (schedule.cpp:150-164) incl.
 * validate_op (workload.cpp:49-93); unroll choices {1,4,16}. */
int tt_sketch_from_op(const tt_op_spec* op, int elementwise_fallback, tt_sketch* out);
/* validate_device (device.cpp:105-122) */
int tt_validate_device(const tt_device_spec* dev);
/* space_size (schedule.cpp:188-195), saturating */
uint64_t tt_space_size(const tt_sketch* sketch);
/* RNG draws random_init consumes per schedule (one per (axis, prime) + 1) */
int tt_draws_per_schedule(const tt_sketch* sketch);

/* ------------------------------------------------ K0 population (async) -- */
/* random_init(sketch, n, RngStream(seed)) (schedule.cpp:166-186), schedules
 * [first, first + n) of the stream, written as SoA columns (tt_types.h).
 * identity_dev (nullable) receives each schedule's exact 64-bit identity. */
int tt_population_generate(tt_ctx* ctx, const tt_sketch* sketch, uint64_t seed, int64_t first, int64_t n,
                           int32_t* soa_dev, int64_t ld, uint64_t* identity_dev);
/* Exact identity <-> schedule (the replacement for schedule_key /
 * schedule_from_key identity, schedule.cpp:280-338). Requires
 * tt_space_size < 2^64. */
int tt_schedule_identity(tt_ctx* ctx, const tt_sketch* sketch, const int32_t* soa_dev, int64_t ld, int64_t n,
                         uint64_t* identity_dev);
int tt_schedule_from_identity(tt_ctx* ctx, const tt_sketch* sketch, const uint64_t* identity_dev, int64_t n,
                              int32_t* soa_dev, int64_t ld);

/* ---------------------------------------------------- K1 SA draft cost -- */
/* draft_cost(sketch, sched, device, toggles).total (draft.cpp:129-154) for n
 * schedules; bit-exact fp64. Synchronous: TT_E_VALIDATE if any schedule
 * fails validate_schedule (schedule.cpp:242-278), as the reference throws. */
int tt_draft_cost(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const int32_t* soa_dev,
                  int64_t ld, int64_t n, int toggles, double* cost_dev);

/* --------------------------------------------- K2 PriorFilter (top-K) -- */
/* explore(op, dev, n_steps = 1, draft_size = k, ...) semantics
 * (draft.cpp:156-221): the k lowest UNIQUE schedules by (cost, first index),
 * ascending. Population given explicitly. Outputs: population index
 * (+ index_base), cost, identity; *count_host = min(k, unique). Synchronous. */
int tt_draft_topk(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const int32_t* soa_dev,
                  int64_t ld, int64_t n, int64_t k, int toggles, int64_t index_base, int64_t* idx_dev,
                  double* cost_dev, uint64_t* identity_dev, int64_t* count_host);
/* The same over the counter-based population random_init(., RngStream(seed))
 * restricted to schedules [first, first + n): K0+K1+K2 fused, the
 * population is never materialised. This is explore(n_steps = 1). */
int tt_explore1(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, uint64_t seed, int64_t first,
                int64_t n, int64_t k, int toggles, int64_t* idx_dev, double* cost_dev, uint64_t* identity_dev,
                int64_t* count_host);
/* explore(op, dev, n_steps, draft_size = k, pop_size = n, RngStream(seed),
 * toggles) with any n_steps >= 1 — the reference's genetic draft loop
 * (draft.cpp:156-221; replaces tiletune::explore, draft.hpp). For
 * n <= 8192 every generation — mutate() (schedule.cpp:340-396) on the
 * reference's RNG stream, identities, draft costs — runs in one persistent
 * device kernel and the host folds each generation into the pool as it
 * lands; larger populations run mutate() on the host between device
 * generations. Bit-identical to the reference either way.
 * HOST outputs, sorted by (cost, discovery): soa_host (ld = k, nullable),
 * cost_host, identity_host (nullable); *count_host = pool size (<= k);
 * *evaluations = n_steps * n. Synchronous. */
int tt_explore(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, int n_steps, int64_t k, int64_t n,
               uint64_t seed, int toggles, int32_t* soa_host, double* cost_host, uint64_t* identity_host,
               int64_t* count_host, uint64_t* evaluations);
/* The tuner's per-round draft set (Tuner::build_draft_set, tuner.cpp:294-323):
 * explore(n_steps, n_spec = max(1, llround((1 - random_mix) * draft_size)),
 * pop_size, RngStream(explore_seed)) followed by the draft_size - n_spec
 * schedules of random_init(., RngStream(mix_seed)) not already in the set,
 * in that order. HOST outputs (capacity draft_size): identities and draft
 * costs; *count_host = set size. Score it with tt_pacm_score and pick with
 * tt_select_top (tuner.cpp:361-396). Synchronous. */
int tt_draft_set(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, int n_steps, int64_t draft_size,
                 int64_t pop_size, double random_mix, uint64_t explore_seed, uint64_t mix_seed, int toggles,
                 uint64_t* identity_host, double* cost_host, int64_t* count_host, uint64_t* evaluations);
/* One whole tuner round at its defaults' shape (Tuner round body,
 * tuner.cpp:294-396): tt_draft_set, then features + PaCM scores of the set
 * (precision TT_PREC_FP64 or TT_PREC_BF16) and select_top(scores, drafts,
 * none excluded, b) — the drafted identities never leave the device between
 * the steps and one device->host read returns the picks. HOST outputs:
 * sel_idx[b] (indices into the draft set, in select_top order), sel_scores[b]
 * and sel_identity[b] (nullable; the schedules to measure, decodable with
 * tt_schedule_from_identity), *n_candidates = draft-set size. E_STATE when
 * the set holds fewer than b candidates (as tt_select_top). Synchronous. */
int tt_tuner_round(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, int n_steps, int64_t draft_size,
                   int64_t pop_size, double random_mix, uint64_t explore_seed, uint64_t mix_seed, int64_t b,
                   int precision, int64_t* sel_idx, double* sel_scores, uint64_t* sel_identity,
                   int64_t* n_candidates);
/* Merge R rank-local top-k lists (C1's consumer): m entries of (cost,
 * global index, identity), global index < 0 = empty slot. Same semantics as
 * one explore over the union. Synchronous. */
int tt_topk_merge(tt_ctx* ctx, const double* cost_dev, const int64_t* gidx_dev, const uint64_t* identity_dev,
                  int64_t m, int64_t k, int64_t* idx_dev, double* out_cost_dev, uint64_t* out_identity_dev,
                  int64_t* count_host);

/* ------------------------------------------------- features & PaCM -- */
/* extract_features (features.cpp:98-257), fp64: stmt [k][S][24], block
 * [k][B][23] with S = tt_n_statements, B = tt_n_blocks. Async. */
int tt_features(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const uint64_t* identity_dev,
                int64_t k, double* stmt_dev, double* block_dev);
int tt_features_soa(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const int32_t* soa_dev,
                    int64_t ld, const int64_t* idx_dev, int64_t k, double* stmt_dev, double* block_dev);
/* Load RankerParams (ranker.hpp:48-58) flattened in for_each_tensor order
 * (tt_types.h) from host or device memory; hidden width h. */
int tt_pacm_load(tt_ctx* ctx, const double* params, int h);
/* score() for k drafted candidates given by identity (ranker.cpp:370-373);
 * advances tt_forward_calls by k. Async. */
int tt_pacm_score(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const uint64_t* identity_dev,
                  int64_t k, int precision, double* score_dev);
/* score_batch(params, feats, opts) on given features (ranker.cpp:375-381). */
int tt_pacm_score_features(tt_ctx* ctx, const double* stmt_dev, const double* block_dev, int n_stmt, int n_block,
                           int64_t k, int attention_identity, double* score_dev);
/* forward_calls / reset_forward_calls (ranker.hpp:88-90), process-wide */
uint64_t tt_forward_calls(void);
void tt_reset_forward_calls(void);

/* ----------------------------------------------------- K2b select_top -- */
/* select_top (ranker.cpp:514-532): b best by (score desc, draft asc, index
 * asc), excluded (nullable, 1 = excluded) never chosen. Synchronous;
 * TT_E_STATE "requested b but only m unmeasured candidates available". */
int tt_select_top(tt_ctx* ctx, const double* scores_dev, const double* drafts_dev, const uint8_t* excluded_dev,
                  int64_t n, int64_t b, int64_t* idx_host);

/* ------------------------------------------------------------- K4 MoA -- */
/* train(params, {one task}, cfg) (ranker.cpp:459-512) on the device, fp64:
 * dataset loss -> for each epoch: batch of <= `batch` records drawn by the
 * partial Fisher-Yates of RngStream(derive_seed(seed, "rain")), forward,
 * LambdaRank loss + score gradient (ranker.cpp:394-441, device, see
 * tt_rank_loss), per-sample score_backward (ranker.cpp:211-261), gradients
 * summed in the reference's sample/row order, p -= lr * g. No host round
 * trip between epochs (batches drawn up front); scratch cached on the
 * context. params_dev (flattened RankerParams) is updated in place; features
 * are device rows [n][n_stmt][24] / [n][n_block][23]; latencies host.
 * Synchronous. */
int tt_pacm_train(tt_ctx* ctx, double* params_dev, int h, const double* stmt_dev, const double* block_dev, int n_stmt,
                  int n_block, const double* latencies_host, int64_t n, int epochs, double lr, int batch,
                  uint64_t seed, int attention_identity, double* initial_loss_host, double* final_loss_host);
/* lambda_rank_loss(scores, latencies) (ranker.cpp:394-441) on the device:
 * loss to the host, d loss / d score into grad_dev (may be NULL). Pair terms
 * are the reference's expressions; each item's gradient and the loss are
 * summed in a fixed order of their own (deterministic, equal to the
 * reference up to summation order). TT_E_STATE for n < 2 or a latency <= 0,
 * as the reference. Synchronous. */
int tt_rank_loss(tt_ctx* ctx, const double* scores_dev, const double* latencies_dev, int64_t n, double* loss_host,
                 double* grad_dev);
/* train's GD update p -= lr * g (ranker.cpp:502-506). Async. */
int tt_gd_step(tt_ctx* ctx, double* params_dev, const double* grads_dev, int64_t n, double lr);
/* momentum_update phi' = t + m (phi - t) (momentum.cpp:28-46); TT_E_STATE
 * unless 0 <= m < 1. Async. */
int tt_momentum_update(tt_ctx* ctx, double* phi_dev, const double* target_dev, int64_t n, double m);

/* ------------------------------------------- simulated hardware (§8f #2) -- */
/* noiseless_latency (oracle.cpp:105-111) of n schedules (SoA): draft cost
 * under the hidden spec x stride multiplier (oracle.cpp:82-95) x occupancy
 * multiplier (oracle.cpp:97-103) + launch overhead; bit-exact. Async. */
int tt_oracle_latency(tt_ctx* ctx, const tt_sketch* sketch, const tt_oracle_spec* oracle, const int32_t* soa_dev,
                      int64_t ld, int64_t n, double* latency_dev);
/* measure (oracle.cpp:113-121) as the tuner draws it (tuner.cpp:202-203):
 * schedule i is trial (trial0 + i) of task `task_hash` (hash_str of the
 * task name), latency = noiseless x exp(sigma x normal()) from
 * RngStream(derive_seed(seed, 0x6d656173, task_hash, trial0 + i)). Async. */
int tt_oracle_measure(tt_ctx* ctx, const tt_sketch* sketch, const tt_oracle_spec* oracle, const int32_t* soa_dev,
                      int64_t ld, int64_t n, uint64_t task_hash, uint64_t trial0, double* latency_dev,
                      double* noiseless_dev);
/* oracle_best (oracle.cpp:123-135): the minimal noiseless latency over the
 * whole schedule space (enumerated by identity on the device) and the
 * identity of a schedule attaining it (the lowest such identity).
 * TT_E_CONFIG when the space exceeds 2^40 schedules. Synchronous. */
int tt_oracle_best(tt_ctx* ctx, const tt_sketch* sketch, const tt_oracle_spec* oracle, uint64_t* best_identity_host,
                   double* best_latency_host);

/* ------------------------------------------------------------- round -- */
typedef struct tt_round_config {
  int64_t n;          /* candidates drafted this round (this rank's shard) */
  int64_t k;          /* draft_size handed to PaCM (tuner.hpp:38, 512) */
  int64_t b;          /* measurement batch (tuner.hpp:37, 10) */
  int32_t toggles;    /* TT_TOGGLES_ALL */
  int32_t precision;  /* tt_precision */
  double band;        /* TT_PREC_BF16: certified |score error| bound, > 0 (TT_E_CONFIG otherwise) */
  int64_t first;      /* seeded source: first schedule index of the shard */
} tt_round_config;

typedef struct tt_round_result {
  int64_t selected; /* min(b, drafted) */
  int64_t drafted;  /* unique drafted candidates (<= k) */
  int64_t rescored; /* fp64-rescored candidates (certification band) */
  int32_t status;   /* selector flags (low byte, 0 when clean) | tt_round_flags */
  int32_t retries;  /* selector re-runs (device threshold retries + host re-runs) */
  double band_err;  /* TT_PREC_BF16: max |bf16 - fp64| score over the rescored set */
} tt_round_result;

/* One draft+verify round (tuner.cpp:361-396 minus the measurement):
 * SA draft over n candidates -> dedup top-k -> features + PaCM over the
 * drafted set -> select_top(b). The population is soa_dev (explicit, may be
 * NULL) or the counter-based random_init stream of `seed`. Requires
 * tt_pacm_load. Outputs b entries (host): population index, score, draft
 * cost, identity. Synchronous (one small device->host copy at the end). */
int tt_round(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const tt_round_config* cfg,
             const int32_t* soa_dev, int64_t ld, uint64_t seed, int64_t* sel_index_host, double* sel_score_host,
             double* sel_cost_host, uint64_t* sel_identity_host, tt_round_result* result_host);
/* Async variant: enqueue only. Up to 16 rounds may be in flight on one
 * context (each copies its record into its own pinned slot); a 17th enqueue
 * fails with TT_E_STATE until the oldest is collected. tt_round_collect
 * returns the OLDEST uncollected round, waiting for that round only; the
 * output buffers hold `capacity` entries each (TT_E_CONFIG, round kept in
 * flight, when that round's b exceeds it). A round whose selector ran out of
 * margin is re-run here (result.retries); a bf16 round whose observed error
 * on its rescored set exceeds cfg.band is re-run in fp64
 * (TT_ROUND_BAND_RERUN). tt_round (synchronous) requires no rounds in flight. */
int tt_round_async(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const tt_round_config* cfg,
                   const int32_t* soa_dev, int64_t ld, uint64_t seed);
int tt_round_collect(tt_ctx* ctx, int64_t capacity, int64_t* sel_index_host, double* sel_score_host,
                     double* sel_cost_host, uint64_t* sel_identity_host, tt_round_result* result_host);

/* Sharded round, draft half (async): this rank's K-entry list of (cost,
 * global index, identity) for the all-gather, ascending by (cost, index);
 * unused slots get index -1. A rank whose selector could not certify its
 * list (more than 4096 schedules tied at the threshold) writes index -2 in
 * slot 0, and every rank's merged round then fails with TT_E_STATE; a rank
 * whose explicit population holds an invalid schedule writes -3, and every
 * rank's merged round fails with TT_E_VALIDATE.
 * cfg->first = global index of this shard's first candidate. */
int tt_round_local_async(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev,
                         const tt_round_config* cfg, const int32_t* soa_dev, int64_t ld, uint64_t seed,
                         double* cost_dev, int64_t* gidx_dev, uint64_t* identity_dev);
/* ------------------------------------------ multi-GPU -- */
/* One process per GPU. Rank 0 creates a unique id (128 bytes) and shares it
 * with the others out of band (MPI, a file, torch.distributed...); every rank
 * then calls tt_comm_init on its context. NCCL (libnccl.so.2) is loaded at
 * run time: TT_E_NCCL when it is missing or a collective fails. */
int tt_comm_unique_id(uint8_t* id_out /* 128 bytes */);
int tt_comm_init(tt_ctx* ctx, int nranks, int rank, const uint8_t* id /* 128 bytes */);
int tt_comm_destroy(tt_ctx* ctx);
/* The sharded round in one call (tuner.cpp:361-396 over R GPUs): cfg->n is
 * the GLOBAL population, split by index range (the first n % R ranks take one
 * extra candidate, cfg->first offsets the whole range); this rank drafts its
 * shard (soa_shard = its slice with ld, or NULL for the counter-based
 * stream of `seed`), one ncclAllGather of the K-entry (cost, global index,
 * identity) lists on the context stream, merge, verify, select — every rank
 * returns the same selection, equal to tt_round over the whole population.
 * A rank whose device selector overflowed makes every rank re-run its draft
 * half with tt_round_local. Synchronous, collective. */
int tt_round_sharded(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const tt_round_config* cfg,
                     const int32_t* soa_shard_dev, int64_t ld, uint64_t seed, int64_t* sel_index_host,
                     double* sel_score_host, double* sel_cost_host, uint64_t* sel_identity_host,
                     tt_round_result* result_host);
/* Synchronous draft half (same payload): the selector's host-driven retries
 * (doubled margin, then the hash path for > 4096 ties) and the population
 * check run here, so it fails only where tt_round fails (TT_E_VALIDATE for
 * an invalid schedule, TT_E_STATE when even the hash path overflows). A
 * merged round whose collect reports a rank's selector overflow is re-run
 * with this on every rank (all ranks see the same merged status). */
int tt_round_local(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev, const tt_round_config* cfg,
                   const int32_t* soa_dev, int64_t ld, uint64_t seed, double* cost_dev, int64_t* gidx_dev,
                   uint64_t* identity_dev);
/* Sharded round, verify half, async: merge + features + PaCM + select;
 * read with tt_round_collect. m <= 4096 entries in any order, or up to
 * 65,536 as m / k whole per-rank lists (tt_round_local_async's layout). The
 * gathered lists must stay valid until the round is collected. */
int tt_round_finish_merged_async(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev,
                                 const tt_round_config* cfg, const double* cost_dev, const int64_t* gidx_dev,
                                 const uint64_t* identity_dev, int64_t m);
/* Stage timing with CUDA events on the context stream (0 draft select,
 * 1 PaCM (features + model), 2 certification rescoring, 3 select_top + record, 4 merge, 5 PaCM kernel
 * alone, 6 feature rows alone, 7 the K1 draft-cost kernel alone).
 * tt_profile_read synchronises, returns per-stage summed ms and counts
 * since the last read. */
int tt_profile_enable(tt_ctx* ctx, int on);
int tt_profile_read(tt_ctx* ctx, double* ms_sum, int64_t* count, int n_stages);

/* Sharded round, verify half: after the all-gather of every rank's local
 * top-k (cost, global index, identity) lists, merge them and finish the
 * round (features -> PaCM -> select_top) on identical data on every rank. */
int tt_round_finish_merged(tt_ctx* ctx, const tt_sketch* sketch, const tt_device_spec* dev,
                           const tt_round_config* cfg, const double* cost_dev, const int64_t* gidx_dev,
                           const uint64_t* identity_dev, int64_t m, int64_t* sel_index_host,
                           double* sel_score_host, double* sel_cost_host, uint64_t* sel_identity_host,
                           tt_round_result* result_host);

/* Device views of the last round's drafted set (valid until the next round). */
int tt_round_drafted(const tt_ctx* ctx, const int64_t** idx_dev, const double** cost_dev,
                     const uint64_t** identity_dev, const double** score_dev);

#ifdef __cplusplus
}
#endif

#endif /* TT_TT_H_ */
