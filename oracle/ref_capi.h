/*
 * ref_capi.h — extern "C" wrapper over the UNMODIFIED reference tiletune core
 * (compiled from /root/reference/proj/core/src by oracle/Makefile into
 * oracle/_ref/). TEST INFRASTRUCTURE ONLY: used to pin the oracle
 * (tests/golden), and as bench.py's `--impl reference` arm, which times the
 * reference's own public API on the host cores.
 */
#ifndef TT_REF_CAPI_H_
#define TT_REF_CAPI_H_
#include <stdint.h>

#include "../include/tt/tt_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* every function returns 0 on success, -1 on a tiletune::Error (message via
 * ref_last_error) */
const char* ref_last_error(void);
int ref_random_init(const tt_sketch* sk, uint64_t seed, int64_t n, int32_t* soa, int64_t ld);
int ref_draft_cost(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa,
                   int64_t ld, int64_t n, int toggles, int threads, double* cost);
int ref_trace(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
              int64_t i, int64_t* symbols, double* penalties, double* stmt_cost, double* total);
/* explore(op, dev, n_steps, K, N, RngStream(seed), toggles, threads): writes
 * the drafted schedules (SoA, ld = K) and costs; returns the count in *count */
int ref_explore(const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t k,
                int64_t n, uint64_t seed, int threads, int32_t* soa_out, double* cost_out,
                int64_t* count, uint64_t* evaluations);
int ref_features(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
                 const int64_t* idx, int64_t k, double* stmt_out, double* block_out);
int ref_init_params(int h, uint64_t seed, double* params);
int ref_score_batch(const double* params, int h, int n_stmt, int n_block, const double* stmt,
                    const double* block, int64_t k, int attention_identity, int threads,
                    double* out, uint64_t* forward_calls);
int ref_select_top(const double* scores, const double* drafts, const uint8_t* excluded,
                   int64_t n, int64_t b, int64_t* idx_out);
int ref_momentum_update(double* phi, const double* target, int h, double m);
/* lambda_rank_loss (ranker.cpp:394-441): loss and score gradient */
int ref_rank_loss(const double* scores, const double* latencies, int64_t n, double* loss, double* grad);
/* train(params, {one task}, cfg) with labels given (ranker.cpp:459-512) */
int ref_train(double* params, int h, int n_stmt, int n_block, const double* stmt,
              const double* block, const double* latencies, int64_t k, int epochs, double lr,
              int batch, uint64_t seed, double* initial_loss, double* final_loss);
int ref_noiseless_latency(const tt_sketch* sk, const tt_device_spec* hidden, double stride_coeff,
                          double occupancy_coeff, double launch_overhead_s, const int32_t* soa,
                          int64_t ld, int64_t n, double* out);

/* measure(sketch, sched, oracle, RngStream(derive_seed(seed, "meas", task,
 * trial0 + i))) for column i (oracle.cpp:113-121, tuner.cpp:202-203) */
int ref_measure(const tt_sketch* sk, const tt_oracle_spec* o, const int32_t* soa, int64_t ld, int64_t n,
                uint64_t task_hash, uint64_t trial0, double* latency, double* noiseless);
/* oracle_best(sketch, oracle, cap) (oracle.cpp:123-135): argmin schedule (SoA, ld 1) + latency */
int ref_oracle_best(const tt_sketch* sk, const tt_oracle_spec* o, uint64_t cap, int32_t* argmin_soa,
                    double* latency);

/* model / Siamese checkpoints (ranker.cpp:534-548, momentum.cpp:58-86) */
int ref_serialize_params(const double* params, int h, char* buf, int64_t cap, int64_t* len);
int ref_parse_params(const char* text, double* params, int* h);
int ref_serialize_siamese(const double* params, int h, double m, int evolved, char* buf, int64_t cap,
                          int64_t* len);
int ref_parse_siamese(const char* text, double* params, int* h, double* m, int* evolved);

/* The tuner's real round: build_draft_set (tuner.cpp:294-323: GA explore of
 * n_spec + unseen random mix) -> extract_features -> score_batch ->
 * select_top(b). sel_idx = positions in the candidate list; seconds[0] the
 * draft set, seconds[1] features + scores + select. */
int ref_tuner_round(const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t draft_size,
                    int64_t pop_size, double random_mix, uint64_t explore_seed, uint64_t mix_seed, int64_t b,
                    const double* params, int h, int threads, int64_t* sel_idx, double* sel_scores,
                    int64_t* n_candidates, double* seconds);

/* measurement records JSONL (tuner.cpp:577-645) for one task named `task`,
 * axes named s0.., r0.. (the names this wrapper gives the op's axes) */
int ref_records_to_jsonl(const tt_sketch* sk, const char* task, const int32_t* soa, int64_t ld, int64_t n,
                         const int32_t* rounds, const double* lat, const double* draft, const double* score,
                         char* buf, int64_t cap, int64_t* len);
int ref_records_from_jsonl(const tt_sketch* sk, const char* task, const char* text, int32_t* soa, int64_t ld,
                           int32_t* rounds, double* lat, double* draft, double* score, int64_t cap, int64_t* n);

/* The reference-API draft+verify round of SURVEY.md §3.2, timed inside:
 * explore(n_steps=1) -> extract_features x K -> score_batch -> select_top.
 * Writes the selected b schedules' ranks into sel_idx (positions within the
 * drafted list) and wall seconds per stage into seconds[4]. */
/* strict CPU bound of the round over a given population (see ref_capi.cpp) */
int ref_round_strict(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld, int64_t n,
                     int64_t k, int64_t b, const double* params, int h, int threads, int64_t* sel_pop_idx,
                     double* seconds);
int ref_round(const tt_sketch* sk, const tt_device_spec* dev, int64_t n, int64_t k, int64_t b,
              uint64_t seed, const double* params, int h, int threads, int64_t* sel_idx,
              double* sel_scores, int32_t* drafted_soa, double* drafted_cost,
              int64_t* drafted_count, double* seconds);

#ifdef __cplusplus
}
#endif
#endif
