// k_pacm64.cu — fp64 PaCM forward on CUDA cores ("parity mode").
//
// Restates run_forward (ranker.cpp:159-209) with the reference's exact
// accumulation order — affine() accumulates k in order from +0.0 skipping
// zero inputs, then adds the bias (ranker.cpp:59-75); attention logits are
// full dot products scaled afterwards, softmax subtracts the row max and
// divides by the sequential sum; pooling sums rows in order — so scores
// agree with the reference to the last bit except where CUDA's fp64
// tanh/exp/log1p differ from glibc by an ulp. It serves as the exact
// scorer for small K and as the certification rescorer for the
// tensor-core path (rescoring only the candidates near the selection
// boundary).
//
// One CTA per candidate; the candidate's hybrid feature (features.cpp) is
// built in shared memory one row per thread, never touching HBM.
#include <cstdint>

#include "tt_features.cuh"
#include "tt_kernels.h"

namespace tt {

struct Params64 {
  const double *w1, *b1, *w2, *b2, *we, *be, *wq, *bq, *wk, *bk, *wv, *bv, *hw1, *hb1, *hw2, *hb2;
};

__host__ __device__ inline Params64 split_params(const double* p, int h) {
  Params64 P;
  P.w1 = p, P.b1 = P.w1 + 24 * h, P.w2 = P.b1 + h, P.b2 = P.w2 + h * h;
  P.we = P.b2 + h, P.be = P.we + 23 * h, P.wq = P.be + h, P.bq = P.wq + h * h;
  P.wk = P.bq + h, P.bk = P.wk + h * h, P.wv = P.bk + h, P.bv = P.wv + h * h;
  P.hw1 = P.bv + h, P.hb1 = P.hw1 + 2 * h * h, P.hw2 = P.hb1 + h, P.hb2 = P.hw2 + h;
  return P;
}

constexpr int kThreads64 = 192;  // 3 x 64: the fused Q|K|V layer has 192 columns at h = 64
constexpr int kMaxRows = 20;     // dataflow blocks of a 6-input op (3 * 6 + 2)

// Y_s (n x q) = act(X (n x m) · W_s (m x q) + b_s) for up to three weight
// sets s laid side by side (Q|K|V). Work item = (column, row group): each
// thread keeps one accumulator per row in registers, so one weight load
// feeds every row and the row chains run in parallel. Every (row, column)
// still accumulates k = 0..m-1 in order from +0.0 and adds the bias last —
// the reference's affine() order (ranker.cpp:59-75). Skipping zero inputs,
// as the reference does, cannot change a finite sum (x*w = ±0 and the
// running sum starts at +0.0), so the branch is dropped.
// Weights are read straight from L2 (every CTA of the launch shares them);
// chunks of kPre loads are issued before any is consumed so one L2 round
// trip covers kPre steps of the k loop. MAXR bounds the rows per thread.
constexpr int kPre = 16;

template <int MAXR>
__device__ __forceinline__ void affine64(const double* x, int n, int m, const double* __restrict__ w0,
                                         const double* __restrict__ w1, const double* __restrict__ w2,
                                         const double* __restrict__ b0, const double* __restrict__ b1,
                                         const double* __restrict__ b2, int q, int sets, bool act, double* y0,
                                         double* y1, double* y2) {
  const int p = q * sets;
  const int G = p >= kThreads64 ? 1 : kThreads64 / p;
  for (int item = threadIdx.x; item < p * G; item += blockDim.x) {
    const int g = item / p, j = item % p;
    const int s = j / q, col = j % q;
    const double* __restrict__ w = s == 0 ? w0 : (s == 1 ? w1 : w2);
    const double bj = __ldg((s == 0 ? b0 : (s == 1 ? b1 : b2)) + col);
    double* y = s == 0 ? y0 : (s == 1 ? y1 : y2);
    double acc[MAXR];
#pragma unroll
    for (int r = 0; r < MAXR; ++r) acc[r] = 0.0;
    for (int k0 = 0; k0 < m; k0 += kPre) {
      double wv[kPre];
#pragma unroll
      for (int u = 0; u < kPre; ++u) wv[u] = k0 + u < m ? __ldg(w + (k0 + u) * q + col) : 0.0;
#pragma unroll
      for (int u = 0; u < kPre; ++u) {
        if (k0 + u < m) {
#pragma unroll
          for (int r = 0; r < MAXR; ++r) {
            const int i = g + r * G;
            if (i < n) acc[r] = __dadd_rn(acc[r], __dmul_rn(x[i * m + k0 + u], wv[u]));
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < MAXR; ++r) {
      const int i = g + r * G;
      if (i < n) {
        const double z = __dadd_rn(acc[r], bj);
        y[i * q + col] = act ? tanh(z) : z;
      }
    }
  }
  __syncthreads();
}

template <int MAXR>
__device__ __forceinline__ void affine64(const double* x, int n, int m, const double* __restrict__ w,
                                         const double* __restrict__ b, int p, bool act, double* y) {
  affine64<MAXR>(x, n, m, w, w, w, b, b, b, p, 1, act, y, y, y);
}

struct Smem64 {
  double *xs, *xb, *z1, *z2, *e, *q, *k, *v, *pr, *ao, *cat, *g, *s;
};

__host__ __device__ inline size_t smem64_doubles(int S, int B, int h) {
  return (size_t)S * 24 + B * 23 + 2 * S * h + 5 * B * h + B * B + 2 * h + h + 1;
}

__device__ inline Smem64 carve64(double* base, int S, int B, int h) {
  Smem64 m;
  m.xs = base;
  m.xb = m.xs + S * 24;
  m.z1 = m.xb + B * 23;
  m.z2 = m.z1 + S * h;
  m.e = m.z2 + S * h;
  m.q = m.e + B * h;
  m.k = m.q + B * h;
  m.v = m.k + B * h;
  m.ao = m.v + B * h;
  m.pr = m.ao + B * h;
  m.cat = m.pr + B * B;
  m.g = m.cat + 2 * h;
  m.s = m.g + h;
  return m;
}

// run_forward on the rows already in m.xs / m.xb. RS / RB / RQ bound the
// rows one thread owns in the statement layers, the block layers and the
// fused Q|K|V layer (chosen by the launcher from n_in and h).
template <int RS, int RB, int RQ>
__device__ double forward64(const Params64& P, int h, int S, int B, bool identity, Smem64& m) {
  affine64<RS>(m.xs, S, 24, P.w1, P.b1, h, true, m.z1);
  affine64<RS>(m.z1, S, h, P.w2, P.b2, h, true, m.z2);
  affine64<RB>(m.xb, B, 23, P.we, P.be, h, true, m.e);
  const double* pooled = m.e;
  if (!identity) {
    affine64<RQ>(m.e, B, h, P.wq, P.wk, P.wv, P.bq, P.bk, P.bv, h, 3, false, m.q, m.k, m.v);
    const double scale = __ddiv_rn(1.0, sqrt((double)h));
    for (int t = threadIdx.x; t < B * B; t += blockDim.x) {  // matmul_nt (ranker.cpp:102-111)
      const int i = t / B, j = t % B;
      double acc = 0.0;
      for (int c = 0; c < h; ++c) acc = __dadd_rn(acc, __dmul_rn(m.q[i * h + c], m.k[j * h + c]));
      m.pr[t] = __dmul_rn(acc, scale);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < B; i += blockDim.x) {  // softmax rows (ranker.cpp:181-191)
      double* row = m.pr + i * B;
      double mx = row[0];
      for (int j = 1; j < B; ++j) mx = row[j] > mx ? row[j] : mx;
      double sum = 0.0;
      for (int j = 0; j < B; ++j) {
        const double ex = exp(__dadd_rn(row[j], -mx));
        row[j] = ex;
        sum = __dadd_rn(sum, ex);
      }
      for (int j = 0; j < B; ++j) row[j] = __ddiv_rn(row[j], sum);
    }
    __syncthreads();
    {  // matmul (ranker.cpp:113-122); (column, row) items spread over the CTA
      for (int item = threadIdx.x; item < h * B; item += blockDim.x) {
        const int j = item % h, i = item / h;
        double acc = 0.0;
        for (int t = 0; t < B; ++t) acc = __dadd_rn(acc, __dmul_rn(m.pr[i * B + t], m.v[t * h + j]));
        m.ao[i * h + j] = acc;
      }
    }
    __syncthreads();
    pooled = m.ao;
  }
  const double inv_n = __ddiv_rn(1.0, (double)B);
  for (int j = threadIdx.x; j < h; j += blockDim.x) {  // concat (ranker.cpp:196-200)
    double s = 0.0;
    for (int i = 0; i < S; ++i) s = __dadd_rn(s, m.z2[i * h + j]);
    m.cat[j] = s;
    double d = 0.0;
    for (int i = 0; i < B; ++i) d = __dadd_rn(d, __dmul_rn(pooled[i * h + j], inv_n));
    m.cat[h + j] = d;
  }
  __syncthreads();
  affine64<1>(m.cat, 1, 2 * h, P.hw1, P.hb1, h, true, m.g);
  affine64<1>(m.g, 1, h, P.hw2, P.hb2, 1, false, m.s);
  return m.s[0];
}

// row bounds per variant: 0 = (n_in <= 2, h <= 64), 1 = (n_in <= 6, h <= 64), 2 = generic
template <int V>
struct Rows;
template <>
struct Rows<0> {
  static constexpr int S = 2, B = 3, Q = 8;
};
template <>
struct Rows<1> {
  static constexpr int S = 5, B = 7, Q = 20;
};
template <>
struct Rows<2> {
  static constexpr int S = 14, B = 20, Q = 20;
};

__host__ inline int rows_variant(int n_in, int h) {
  if (h > 64) return 2;
  return n_in <= 2 ? 0 : 1;
}

template <int V>
__device__ __forceinline__ double forward64v(const Params64& P, int h, int S, int B, bool identity, Smem64& m) {
  return forward64<Rows<V>::S, Rows<V>::B, Rows<V>::Q>(P, h, S, B, identity, m);
}

template <int NSP, int NRED>
__device__ __forceinline__ void load_ref(const DevSketch& S, const CandRef& r, int64_t pos, Factors<NSP, NRED>& F) {
  if (r.soa) {
    load_factors<NSP, NRED>(r.soa, r.ld, r.idx[pos] - r.index_base, F, true);
  } else if (r.seeded) {
    generate<NSP, NRED>(S, r.s0, (uint64_t)r.idx[pos], F);
  } else {
    from_identity<NSP, NRED>(S, r.id[pos], F);
  }
}

template <int NSP, int NRED>
__device__ __forceinline__ void rows64(const DevSketch& S, const DevDevice& D, const CandRef& r, int64_t pos,
                                       double* xs, double* xb) {
  const int n_stmt = 2 * S.n_in + 2;
  const int n_block = S.kind == TT_OP_ELEMENTWISE ? 1 : 3 * S.n_in + 2;
  if (threadIdx.x < n_stmt + n_block) {
    Factors<NSP, NRED> F;
    load_ref<NSP, NRED>(S, r, pos, F);
    CandInfo<NSP, NRED> C;
    cand_info<NSP, NRED>(S, D, F, C);
    const int row = threadIdx.x;
    double* out = row < n_stmt ? xs + row * 24 : xb + (row - n_stmt) * 23;
    feature_row<double, NSP, NRED>(S, D, C, row, out);
  }
  __syncthreads();
}

template <int NSP, int NRED>
__global__ void __launch_bounds__(64) k_features64(DevSketch S, DevDevice D, CandRef r, int64_t k,
                                                   double* __restrict__ stmt_out, double* __restrict__ block_out) {
  const int n_stmt = 2 * S.n_in + 2;
  const int n_block = S.kind == TT_OP_ELEMENTWISE ? 1 : 3 * S.n_in + 2;
  for (int64_t pos = blockIdx.x; pos < k; pos += gridDim.x) {
    if (threadIdx.x < n_stmt + n_block) {
      Factors<NSP, NRED> F;
      load_ref<NSP, NRED>(S, r, pos, F);
      CandInfo<NSP, NRED> C;
      cand_info<NSP, NRED>(S, D, F, C);
      const int row = threadIdx.x;
      double* out = row < n_stmt ? stmt_out + (pos * n_stmt + row) * 24 : block_out + (pos * n_block + row - n_stmt) * 23;
      feature_row<double, NSP, NRED>(S, D, C, row, out);
    }
  }
}

template <int NSP, int NRED, int V>
__global__ void __launch_bounds__(kThreads64) k_pacm64(DevSketch S, DevDevice D, CandRef r, const int64_t* count_dev,
                                                       const int32_t* sublist, const int* sublist_count,
                                                       const double* __restrict__ params, int h, int identity,
                                                       double* __restrict__ score_out) {
  extern __shared__ __align__(16) double sm64[];
  const int n_stmt = 2 * S.n_in + 2;
  const int n_block = S.kind == TT_OP_ELEMENTWISE ? 1 : 3 * S.n_in + 2;
  int64_t pos = blockIdx.x;
  if (sublist) {
    if ((int)blockIdx.x >= *sublist_count) return;
    pos = sublist[blockIdx.x];
  }
  if (count_dev && pos >= *count_dev) return;
  Smem64 m = carve64(sm64, n_stmt, n_block, h);
  rows64<NSP, NRED>(S, D, r, pos, m.xs, m.xb);
  const Params64 P = split_params(params, h);
  const double s = forward64v<V>(P, h, n_stmt, n_block, identity != 0, m);
  if (threadIdx.x == 0) score_out[pos] = s;
}

template <int V>
__global__ void __launch_bounds__(kThreads64) k_pacm64_feats(const double* __restrict__ stmt, const double* __restrict__ block,
                                                             int n_stmt, int n_block, const double* __restrict__ params,
                                                             int h, int identity, double* __restrict__ score_out) {
  extern __shared__ __align__(16) double sm64[];
  const int64_t pos = blockIdx.x;
  Smem64 m = carve64(sm64, n_stmt, n_block, h);
  for (int t = threadIdx.x; t < n_stmt * 24; t += blockDim.x) m.xs[t] = stmt[pos * n_stmt * 24 + t];
  for (int t = threadIdx.x; t < n_block * 23; t += blockDim.x) m.xb[t] = block[pos * n_block * 23 + t];
  __syncthreads();
  const Params64 P = split_params(params, h);
  const double s = forward64v<V>(P, h, n_stmt, n_block, identity != 0, m);
  if (threadIdx.x == 0) score_out[pos] = s;
}

template <int NSP, int NRED, int V>
static void run_pacm64(const DevSketch& S, const DevDevice& D, CandRef ref, const int64_t* count_dev, int64_t k_max,
                       const int32_t* sublist, const int* sublist_count, const double* params, int h, int identity,
                       double* score_out, size_t sm, cudaStream_t st) {
  static size_t set = 0;
  if (sm > set) {
    cudaFuncSetAttribute(k_pacm64<NSP, NRED, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    set = sm;
  }
  tt::note_launch();
  k_pacm64<NSP, NRED, V><<<(unsigned)k_max, kThreads64, sm, st>>>(S, D, ref, count_dev, sublist, sublist_count, params,
                                                                  h, identity, score_out);
}

static int n_blocks_of(const DevSketch& S) { return S.kind == TT_OP_ELEMENTWISE ? 1 : 3 * S.n_in + 2; }

int launch_features64(const DevSketch& S, const DevDevice& D, CandRef ref, int64_t k, double* stmt_out,
                      double* block_out, cudaStream_t st) {
  if (k <= 0) return 0;
  const int g = (int)(k < 148 * 64 ? k : 148 * 64);
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_features64<NSP, NRED><<<g, 64, 0, st>>>(S, D, ref, k, stmt_out, block_out)));
}

int launch_pacm64(const DevSketch& S, const DevDevice& D, CandRef ref, const int64_t* count_dev, int64_t k_max,
                  const int32_t* sublist, const int* sublist_count, const double* params, int h,
                  int attention_identity, double* score_out, cudaStream_t st) {
  if (k_max <= 0) return 0;
  const int n_stmt = 2 * S.n_in + 2, n_block = n_blocks_of(S);
  const size_t sm = smem64_doubles(n_stmt, n_block, h) * sizeof(double);
  const int v = rows_variant(S.n_in, h);
#define TT_PACM64_ARGS S, D, ref, count_dev, k_max, sublist, sublist_count, params, h, attention_identity, score_out, sm, st
  if (v == 0) return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_pacm64<NSP, NRED, 0>(TT_PACM64_ARGS)));
  if (v == 1) return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_pacm64<NSP, NRED, 1>(TT_PACM64_ARGS)));
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_pacm64<NSP, NRED, 2>(TT_PACM64_ARGS)));
#undef TT_PACM64_ARGS
}

int launch_pacm64_feats(const double* stmt, const double* block, int n_stmt, int n_block, int64_t k,
                        const double* params, int h, int attention_identity, double* score_out, cudaStream_t st) {
  if (k <= 0) return 0;
  if (n_stmt > 14 || n_block > 20) return -1;
  const size_t sm = smem64_doubles(n_stmt, n_block, h) * sizeof(double);
  const int v = h > 64 ? 2 : (n_stmt <= 6 && n_block <= 8 ? 0 : 1);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    tt::note_launch();
    kern<<<(unsigned)k, kThreads64, sm, st>>>(stmt, block, n_stmt, n_block, params, h, attention_identity, score_out);
  };
  if (v == 0) go(k_pacm64_feats<0>);
  else if (v == 1) go(k_pacm64_feats<1>);
  else go(k_pacm64_feats<2>);
  return 0;
}

}  // namespace tt
