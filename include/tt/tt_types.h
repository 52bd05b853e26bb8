/*
 * tt_types.h — plain-C POD mirrors of the reference tiletune problem model.
 *
 * These are the structs that cross the drop-in C ABI (include/tt/tt.h). They
 * carry exactly the information the reference's C++ value types carry for
 * the draft+verify path, flattened so that no STL or torch type appears in a
 * signature:
 *
 *   tt_device_spec  <- tiletune::DeviceSpec   (proj/core/include/tiletune/device.hpp:29-39)
 *   tt_buffer_spec  <- tiletune::BufferSpec   (proj/core/include/tiletune/workload.hpp:30-34)
 *   tt_op_spec      <- tiletune::TensorOpSpec (proj/core/include/tiletune/workload.hpp:47-57)
 *                      axis names become ids: spatial axes 0..n_spatial-1 in
 *                      op order, reduction axes n_spatial.. in op order.
 *   tt_sketch       <- tiletune::Sketch       (proj/core/include/tiletune/schedule.hpp:36-50)
 *                      as produced by generate_sketch(op, true)
 *                      (schedule.cpp:150-164): spatial arity 4 for tiled ops,
 *                      2 for element-wise ops, plus the unroll choices.
 *
 * Schedule population layout (tiletune::Schedule, schedule.hpp:56-60, turned
 * into structure-of-arrays): int32 column-major matrix soa[col * ld + i] with
 *   cols 4a..4a+3            = (b, t, o, v) of spatial axis a
 *   cols 4*n_sp + 3r .. +2   = (ra, rb, rc) of reduction axis r
 *   col  4*n_sp + 3*n_red    = unroll value (not its index)
 * i.e. tt_schedule_cols(sketch) = 4*n_sp + 3*n_red + 1 int32 columns.
 * Element-wise sketches keep 4 spatial columns with o = v = 1, exactly like
 * the reference's padded (b, t, 1, 1) tuples.
 */
#ifndef TT_TYPES_H_
#define TT_TYPES_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TT_MAX_AXES 8
#define TT_MAX_BUFFERS 6
#define TT_MAX_UNROLL 4
#define TT_MAX_PRIMES 24 /* distinct (axis, prime) pairs over the whole op */

#define TT_IO_INPUT 0
#define TT_IO_OUTPUT 1

#define TT_OP_TILED 0
#define TT_OP_ELEMENTWISE 1

/* statement / block geometry of the hybrid feature (features.hpp:28-29) */
#define TT_STMT_WIDTH 24
#define TT_BLOCK_WIDTH 23

typedef struct tt_device_spec {
  int64_t m_l0;
  int64_t m_l1;
  int64_t pu_l1;
  int64_t n_l1; /* power of two (device.cpp:105-108) */
  int64_t pu_l2;
  int64_t n_l2; /* power of two */
  double t_p;
  double t_m;
  int64_t element_bytes;
} tt_device_spec;

typedef struct tt_buffer_spec {
  int32_t io;
  int32_t n_axes;
  int32_t axes[TT_MAX_AXES]; /* last entry = innermost (contiguous) axis */
} tt_buffer_spec;

typedef struct tt_op_spec {
  int32_t n_spatial;
  int32_t n_reduction;
  int64_t extent[TT_MAX_AXES];
  int32_t n_buffers;
  int32_t fused_elementwise;
  int32_t kind;
  int32_t _pad;
  tt_buffer_spec buffers[TT_MAX_BUFFERS];
} tt_op_spec;

typedef struct tt_sketch {
  tt_op_spec op;
  int32_t n_unroll;
  int32_t _pad;
  int64_t unroll[TT_MAX_UNROLL];
} tt_sketch;

/* The simulated hardware of the reference (tiletune::OracleDevice,
 * oracle.hpp:40-47): the hidden device spec plus the latency model's
 * coefficients and the measurement noise. */
typedef struct tt_oracle_spec {
  tt_device_spec hidden;
  double stride_coeff;      /* default 0.35 */
  double occupancy_coeff;   /* default 1.5 */
  double launch_overhead_s; /* default 2e-6 */
  double noise_sigma;       /* default 0.03 */
  uint64_t seed;
} tt_oracle_spec;

/* Penalty ablation switches (draft.hpp:83-86). Bit 0 = compute side
 * enabled, bit 1 = memory side enabled; TT_TOGGLES_ALL is the default. */
#define TT_TOGGLE_COMPUTE 1
#define TT_TOGGLE_MEMORY 2
#define TT_TOGGLES_ALL 3

static inline int tt_schedule_cols(const tt_sketch* s) {
  return 4 * s->op.n_spatial + 3 * s->op.n_reduction + 1;
}

/* statements per candidate: 2 per input + compute + store (draft.cpp:42-106) */
static inline int tt_n_inputs(const tt_op_spec* op) {
  int n = 0;
  for (int i = 0; i < op->n_buffers; ++i) n += op->buffers[i].io == TT_IO_INPUT;
  return n;
}
static inline int tt_n_statements(const tt_op_spec* op) { return 2 * tt_n_inputs(op) + 2; }
/* dataflow blocks: loads + per-operand compute + accumulation + store, or a
 * single zero block for element-wise ops (features.cpp:153-158) */
static inline int tt_n_blocks(const tt_op_spec* op) {
  return op->kind == TT_OP_ELEMENTWISE ? 1 : 3 * tt_n_inputs(op) + 2;
}

/* RankerParams flattened in for_each_tensor order (ranker.cpp:339-356):
 * stmt_w1[24h] stmt_b1[h] stmt_w2[h*h] stmt_b2[h] embed_w[23h] embed_b[h]
 * attn_wq[h*h] attn_bq[h] attn_wk[h*h] attn_bk[h] attn_wv[h*h] attn_bv[h]
 * head_w1[2h*h] head_b1[h] head_w2[h] head_b2[1]; all row-major. */
static inline int64_t tt_param_count(int h) {
  return (int64_t)24 * h + h + (int64_t)h * h + h + (int64_t)23 * h + h +
         3 * ((int64_t)h * h + h) + (int64_t)2 * h * h + h + h + 1;
}

#ifdef __cplusplus
}
#endif

#endif /* TT_TYPES_H_ */
