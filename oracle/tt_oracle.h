/*
 * tt_oracle.h — CPU restatement of the reference draft+verify path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it. The shipped path is the CUDA library behind
 * include/tt/tt.h, which never links or calls anything in oracle/.
 *
 * Parity pinning: every function here is checked in tests/test_oracle_golden.py
 * against golden vectors produced by the reference itself (compiled from
 * /root/reference/proj/core/src by oracle/Makefile into oracle/_ref, dumped by
 * oracle/make_golden.py into tests/golden/) and against the KATs the
 * reference's own doctest suite asserts (proj/tests/test_*.cpp).
 */
#ifndef TT_ORACLE_H_
#define TT_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/tt/tt_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* RngStream / derive_seed / hash_str (common.hpp:52-119) */
uint64_t tto_derive_seed(uint64_t base, uint64_t a);
uint64_t tto_hash_str(const char* s);

/* generate_sketch(op, true) with the default unroll choices {1,4,16}
 * (schedule.cpp:150-164). */
void tto_sketch_init(const tt_op_spec* op, tt_sketch* out);

/* Draws per schedule consumed by random_init: one per (axis, distinct prime)
 * plus one for unroll (schedule.cpp:49-68,141-148,166-186). */
int tto_draws_per_schedule(const tt_sketch* sk);

/* uint64 saturating space size (schedule.cpp:188-195). */
uint64_t tto_space_size(const tt_sketch* sk);

/* Schedules [first, first+n) of random_init(sketch, ., RngStream(seed))
 * written to the SoA layout of tt_types.h. */
void tto_random_init(const tt_sketch* sk, uint64_t seed, int64_t first, int64_t n,
                     int32_t* soa, int64_t ld);

/* draft_cost(...).total for each column i < n (draft.cpp:129-154). */
void tto_draft_cost(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa,
                    int64_t ld, int64_t n, int toggles, double* cost);

/* Per-statement trace of one schedule: symbols s1..s8 [S][8], penalties
 * [S][7] (p_l0_m,p_l0_c,p_l1_m,p_l1_c,alpha,p_l2_c,p_l2_m) and statement
 * costs [S][4] (l_c,l_m,u_p,u_m). Returns the statement count S. */
int tto_trace(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
              int64_t i, int toggles, int64_t* symbols, double* penalties, double* stmt_cost,
              double* total);

/* Exact 64-bit schedule identity: mixed-radix value of the per-(axis,prime)
 * composition ranks and the unroll index (the very draws random_init
 * consumes). Requires tto_space_size < 2^64 (returns 0 and sets *ok = 0
 * otherwise). */
uint64_t tto_identity(const tt_sketch* sk, const int32_t* soa, int64_t ld, int64_t i, int* ok);

/* explore(op, dev, 1, K, N, ...) semantics: the K lowest unique schedules by
 * (cost, first index), ascending (draft.cpp:156-221). Returns the count
 * written (min(K, unique)). */
int64_t tto_draft_topk(const tt_sketch* sk, const double* cost, const int32_t* soa, int64_t ld,
                       int64_t n, int64_t k, int64_t* idx_out, double* cost_out);

/* explore(op, dev, n_steps, K, N, RngStream(seed), toggles) for any
 * n_steps (draft.cpp:156-221, mutate schedule.cpp:340-396): the pool sorted
 * by (cost, discovery), SoA ld = K. Returns the pool size (<= K). */
int64_t tto_explore(const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t k, int64_t n,
                    uint64_t seed, int toggles, int32_t* soa_out, double* cost_out);

/* extract_features for columns idx[0..k) (features.cpp:98-257):
 * stmt_out [k][S][24], block_out [k][B][23]. */
void tto_features(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
                  const int64_t* idx, int64_t k, double* stmt_out, double* block_out);

/* init_params(h, RngStream(seed)) flattened (ranker.cpp:305-326). */
void tto_init_params(int h, uint64_t seed, double* params);

/* run_forward(...).score for each feature set (ranker.cpp:159-209). */
void tto_score(const double* params, int h, int n_stmt, int n_block, const double* stmt,
               const double* block, int64_t k, int attention_identity, double* score_out);

/* select_top (ranker.cpp:514-532). Returns 0, or -1 when fewer than b
 * unexcluded candidates exist. */
int tto_select_top(const double* scores, const double* drafts, const uint8_t* excluded,
                   int64_t n, int64_t b, int64_t* idx_out);

/* momentum_update element-wise (momentum.cpp:28-46) and the GD update of
 * train (ranker.cpp:502-506). */
void tto_momentum_update(double* phi, const double* target, int64_t n, double m);
void tto_gd_step(double* params, const double* grads, int64_t n, double lr);
/* lambda_rank_loss (ranker.cpp:394-441), literal: the n^2 pairs in (i, j)
 * order, one running loss, grad[i] -= slope / grad[j] += slope as they come.
 * Returns 0, or -1 for n < 2 or a latency <= 0 (the reference's kState). */
int tto_rank_loss(const double* scores, const double* latencies, int64_t n, double* loss, double* grad);

#ifdef __cplusplus
}
#endif

#endif /* TT_ORACLE_H_ */
