// tt_features.cuh — hybrid feature rows on the device (features.cpp:98-257).
//
// feature_row() produces ONE row of a candidate's hybrid feature: rows
// 0..S-1 are the 24-wide statement vectors (features.cpp:122-151), rows
// S..S+B-1 the 23-wide dataflow blocks (features.cpp:153-255), so a CTA can
// build all rows of a candidate in parallel (one thread per row) and write
// them straight into shared memory as GEMM operands. R = double reproduces
// the reference's fp64 arithmetic (log1p of exactly the same arguments);
// R = float is the tensor-core path's feature precision.
#pragma once

#include "tt_device.cuh"
#include "tt_kernels.h"

namespace tt {

// log1p is ~80 SASS instructions; a feature row calls it up to 17 times, so
// one out-of-line copy keeps the row code small enough to stay in the
// instruction cache (the kernels that build rows are latency-bound).
static __device__ __noinline__ double log1p_ool(double x) { return log1p(x); }
static __device__ __noinline__ float log1pf_ool(float x) { return log1pf(x); }

template <typename R>
__device__ __forceinline__ R lg(R x);
template <>
__device__ __forceinline__ double lg<double>(double x) {
  return log1p_ool(x);
}
template <>
__device__ __forceinline__ float lg<float>(float x) {
  return log1pf_ool(x);
}

template <typename R>
__device__ __forceinline__ R rdiv(R a, R b);
template <>
__device__ __forceinline__ double rdiv<double>(double a, double b) {
  return ddiv_inrange(a, b);  // ratios of counts: integers in [0, 2^63], divisors >= 1
}
template <>
__device__ __forceinline__ float rdiv<float>(float a, float b) {
  return __fdiv_rn(a, b);
}

// Factors of drafted position `pos` (explicit SoA, counter stream or identity).
template <int NSP, int NRED>
__device__ __forceinline__ void feat_load(const DevSketch& S, const CandRef& r, int64_t pos, Factors<NSP, NRED>& F) {
  if (r.soa) {
    load_factors<NSP, NRED>(r.soa, r.ld, r.idx[pos] - r.index_base, F, true);
  } else if (r.seeded) {
    generate<NSP, NRED>(S, r.s0, (uint64_t)r.idx[pos], F);
  } else {
    from_identity<NSP, NRED>(S, r.id[pos], F);
  }
}

// Everything a candidate's rows share; computed once per thread.
template <int NSP, int NRED>
struct CandInfo {
  Tiles<NSP, NRED> T;
  Symbols y;
  Penalties p;
  int64_t s5_in[kMaxIn];
  int64_t traffic;
  int32_t unroll;
};

template <int NSP, int NRED>
__device__ __forceinline__ void cand_info(const DevSketch& S, const DevDevice& D,
                                          const Factors<NSP, NRED>& F, CandInfo<NSP, NRED>& C) {
  constexpr int NA = NSP + NRED;
  build_tiles(F, C.T);
  C.y = symbols_of(S, C.T);
  C.p = penalties(C.y, D);
  C.traffic = 0;
#pragma unroll
  for (int q = 0; q < kMaxIn; ++q) {
    C.s5_in[q] = 0;
    if (q < S.n_in) {
      C.s5_in[q] = fp_mask<NA>(C.T.l1, S.in_mask[q]) * C.T.s6 * C.T.prod_ra;
      C.traffic += C.s5_in[q];
    }
  }
  C.traffic += S.output_size;  // store statement s5
  C.unroll = F.unroll;
}

template <int NA>
__device__ __forceinline__ int64_t inner_vec(const int32_t (&vin)[NA], uint32_t mask) {
  return fp_mask<NA>(vin, mask);
}

// The arguments of row `row` (statement rows first): out value k is
// lg(arg[k]) where bit k of *logm is set, arg[k] itself otherwise — so the
// (expensive) log1p calls of a row can be spread over lanes. feature_row
// applies them in place.
template <typename R, int NSP, int NRED>
__device__ __forceinline__ void feature_args(const DevSketch& S, const DevDevice& D,
                                             const CandInfo<NSP, NRED>& C, int row, R* out, uint32_t* logm) {
  uint32_t lm = 0;
  constexpr int NA = NSP + NRED;
  const int n_in = S.n_in;
  const int n_stmt = 2 * n_in + 2;
  const auto& T = C.T;
  const int64_t lanes = T.s4 * T.s6;
  if (row < n_stmt) {
    // statement order: L2->L1 per input, L1->L0 per input, compute, store
    int kind, q = 0;
    if (row < n_in) kind = 0, q = row;
    else if (row < 2 * n_in) kind = 1, q = row - n_in;
    else if (row == 2 * n_in) kind = 2;
    else kind = 3;
    int64_t s5 = 0, s7 = 0, s8 = 0;
    uint32_t lastmask = 0;
    if (kind == 0) {
#pragma unroll
      for (int t = 0; t < kMaxIn; ++t)
        if (t == q) s5 = C.s5_in[t], lastmask = (uint32_t)S.in_last[t];
      s7 = pick<NA>(T.l1, (int)lastmask);
    } else if (kind == 1) {
      s7 = pick<NA>(T.l0, S.in_last[q]);
    } else if (kind == 2) {
      s8 = S.flops;
    } else {
      s5 = S.output_size;
      s7 = pick<NA>(T.l0, S.out_last);
    }
    const Symbols& y = C.y;
    const Penalties& p = C.p;
    out[0] = (R)y.s1;
    lm |= 1u << 0;
    out[1] = (R)y.s2;
    lm |= 1u << 1;
    out[2] = (R)y.s3;
    lm |= 1u << 2;
    out[3] = (R)y.s4;
    lm |= 1u << 3;
    out[4] = (R)s5;
    lm |= 1u << 4;
    out[5] = (R)y.s6;
    lm |= 1u << 5;
    out[6] = (R)s7;
    lm |= 1u << 6;
    out[7] = (R)s8;
    lm |= 1u << 7;
    out[8] = (R)p.p_l0_m;
    out[9] = (R)p.p_l0_c;
    lm |= 1u << 9;
    out[10] = (R)p.p_l1_m;
    out[11] = (R)p.p_l1_c;
    out[12] = (R)p.alpha;
    out[13] = (R)p.p_l2_c;
    out[14] = (R)p_l2_m_of(s7, D);
    out[15] = (R)S.flops;
    lm |= 1u << 15;
    out[16] = (R)C.traffic;
    lm |= 1u << 16;
    out[17] = rdiv<R>((R)s8, (R)(s5 > 1 ? s5 : 1));
    lm |= 1u << 17;
    out[18] = rdiv<R>((R)y.s4, (R)D.pu_l1_n_l1);
    out[19] = rdiv<R>((R)y.s6, (R)D.pu_l2);
    lm |= 1u << 19;
    out[20] = (R)C.unroll;
    lm |= 1u << 20;
    out[21] = (R)S.fused;
    out[22] = (R)kind / (R)4;
    out[23] = (R)1;
    *logm = lm;
    return;
  }
  // ---- dataflow blocks ----
  const int b = row - n_stmt;
#pragma unroll
  for (int t = 0; t < TT_BLOCK_WIDTH; ++t) out[t] = (R)0;
  out[22] = (R)1;
  if (S.kind == TT_OP_ELEMENTWISE) {  // single zero block (features.cpp:153-158)
    *logm = 0;
    return;
  }
  int flow, access, rank, depth;
  int64_t alloc, volume, distinct, stride, per_lane, s7;
  bool contiguous, red;
  const int n_sp = S.n_sp, n_red = S.n_red;
  const int depth_c = 2 * (n_sp + n_red) + n_red + 2 * n_sp;
  int q = 0;
  int kind;
  if (b < n_in) kind = 0, q = b;
  else if (b < 2 * n_in) kind = 1, q = b - n_in;
  else if (b < 3 * n_in) kind = 2, q = b - 2 * n_in;
  else if (b == 3 * n_in) kind = 3;
  else kind = 4;
  uint32_t mask = 0;
  int last = 0, brank = 0, bred = 0;
  int64_t bsize = 1, s5q = 0;
#pragma unroll
  for (int t = 0; t < kMaxIn; ++t)
    if (t == q) mask = S.in_mask[t], last = S.in_last[t], brank = S.in_rank[t], bred = S.in_has_red[t],
                bsize = S.in_size[t], s5q = C.s5_in[t];
  const int64_t reg_stride = last == S.innermost_spatial ? 1 : (int64_t)pick<NA>(T.l1, last);
  if (kind == 0) {  // load L2 -> L1
    flow = 0, access = 0;
    alloc = fp_mask<NA>(T.l1, mask);
    volume = s5q;
    distinct = bsize;
    stride = 1;
    s7 = pick<NA>(T.l1, last);
    contiguous = (s7 & (D.n_l2 - 1)) == 0;
    per_lane = (alloc + T.s4 - 1) / T.s4;
    rank = brank, depth = n_sp + n_red, red = bred;
  } else if (kind == 1) {  // load L1 -> L0
    flow = 1, access = 0;
    alloc = fp_mask<NA>(T.l0, mask);
    volume = lanes * S.red_total * alloc;
    distinct = bsize;
    stride = reg_stride;
    contiguous = stride == 1;
    per_lane = inner_vec<NA>(T.vin, mask);
    rank = brank, depth = 2 * (n_sp + n_red), red = bred;
    s7 = pick<NA>(T.l0, last);
  } else if (kind == 2) {  // compute operand q
    flow = 2, access = 0;
    alloc = fp_mask<NA>(T.l0, mask);
    volume = S.flops;
    distinct = bsize;
    stride = reg_stride;
    contiguous = stride == 1;
    per_lane = inner_vec<NA>(T.vin, mask);
    rank = brank, depth = depth_c, red = bred;
    s7 = 0;
  } else if (kind == 3) {  // intra-L0 accumulation
    flow = 5, access = 2;
    alloc = fp_mask<NA>(T.l0, S.out_mask);
    volume = S.flops;
    distinct = S.output_size;
    stride = 1;
    contiguous = true;
    per_lane = inner_vec<NA>(T.vin, S.out_mask);
    rank = S.out_rank, depth = depth_c, red = true;
    s7 = 0;
  } else {  // store L0 -> L2
    flow = 3, access = 1;
    alloc = S.output_size;
    volume = S.output_size;
    distinct = S.output_size;
    stride = 1;
    s7 = pick<NA>(T.l0, S.out_last);
    contiguous = (s7 & (D.n_l2 - 1)) == 0;
    per_lane = fp_mask<NA>(T.l0, S.out_mask);
    rank = S.out_rank, depth = 4 * n_sp, red = false;
  }
  out[flow] = (R)1;
  out[6 + access] = (R)1;
  out[9] = (R)alloc;
  lm |= 1u << 9;
  out[10] = (R)volume;
  lm |= 1u << 10;
  out[11] = rdiv<R>((R)volume, (R)(distinct > 1 ? distinct : 1));
  lm |= 1u << 11;
  out[12] = (R)stride;
  lm |= 1u << 12;
  out[13] = contiguous ? (R)1 : (R)0;
  out[14] = rdiv<R>((R)S.flops, (R)(volume > 1 ? volume : 1));
  lm |= 1u << 14;
  out[15] = (R)lanes;
  lm |= 1u << 15;
  out[16] = (R)per_lane;
  lm |= 1u << 16;
  out[17] = (R)rank / (R)8;
  out[18] = (R)depth / (R)16;
  out[19] = red ? (R)1 : (R)0;
  out[20] = (R)C.unroll;
  lm |= 1u << 20;
  out[21] = (R)s7;
  lm |= 1u << 21;
  *logm = lm;
}

// Writes row `row` (statement rows first) into out[0..width).
template <typename R, int NSP, int NRED>
__device__ __forceinline__ void feature_row(const DevSketch& S, const DevDevice& D,
                                            const CandInfo<NSP, NRED>& C, int row, R* out) {
  uint32_t lm;
  feature_args<R, NSP, NRED>(S, D, C, row, out, &lm);
#pragma unroll
  for (int k = 0; k < TT_STMT_WIDTH; ++k)
    if (lm >> k & 1u) out[k] = lg<R>(out[k]);
}

}  // namespace tt
