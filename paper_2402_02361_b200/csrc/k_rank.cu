// k_rank.cu — LambdaRank loss and its score gradient on the device
// (lambda_rank_loss, ranker.cpp:394-441), the per-epoch step of train()
// (ranker.cpp:459-512) and of the dataset loss (ranker.cpp:445-455).
//
// The reference walks the n^2 pairs (i, j) in order, one running loss sum
// and grad[i] -= slope, grad[j] += slope as it goes. Here every item k owns
// its gradient: threads (k, chunk of j) evaluate both roles of k in the pairs
// of their chunk — k faster (grad -= slope, loss += w softplus(-d)) and k
// slower (grad += slope) — and the chunk partials are summed in chunk order.
// Each slope is computed twice (once per endpoint) so no atomics are needed:
// the result is deterministic, and equal to the reference's up to the
// summation order (the pair terms themselves are the same expressions:
// gain = exp2(min_lat / lat) - 1, discount = 1 / log2(position + 2) under the
// score ranking descending with index ties, max DCG over the gains sorted
// descending). Kernels:
//   k_rank_min    one CTA: min latency (exact) and the positivity check
//   k_rank_gain   gain per item
//   k_rank_pos    score position -> discount, gain position -> ideal term
//   k_rank_dcg    one CTA: max DCG = sum of the ideal terms (fixed tree)
//   k_rank_pairs  (k, j-chunk) partial gradient / loss
//   k_rank_fold   per k: chunk partials in order -> dscore[k]; loss partials
//   k_rank_loss   one CTA: total loss (fixed tree) -> *loss (+ accumulate)
#include <cstdint>

#include "tt_kernels.h"

namespace tt {

namespace {

constexpr int kRankThreads = 256;

__device__ __forceinline__ double softplus_d(double x) { return x > 30.0 ? x : log1p(exp(x)); }
__device__ __forceinline__ double sigmoid_d(double x) {
  if (x >= 0) {
    const double e = exp(-x);
    return 1.0 / (1.0 + e);
  }
  const double e = exp(x);
  return e / (1.0 + e);
}
__device__ __forceinline__ double log2d_d(double x) { return __dmul_rn(log(x), 1.4426950408889634074); }

// Fixed-order block sum of v over the CTA (blockDim.x a power of two <= 1024).
__device__ __forceinline__ double block_sum_fixed(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  return red[0];
}

__device__ __forceinline__ double lat_of(const double* lat, const int32_t* list, int i) {
  return lat[list ? list[i] : i];
}

__global__ void __launch_bounds__(1024) k_rank_min(const double* __restrict__ lat, const int32_t* __restrict__ list,
                                                   int m, double* __restrict__ ws, int* __restrict__ bad) {
  __shared__ double red[1024];
  double mn = lat_of(lat, list, 0);
  int b = 0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double l = lat_of(lat, list, i);
    b |= !(l > 0.0);
    mn = l < mn ? l : mn;
  }
  red[threadIdx.x] = mn;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (b) atomicOr(bad, 1);
  if (threadIdx.x == 0) ws[0] = red[0];
}

// ws layout (doubles): [0] min lat, [1] max dcg, then gain[m], disc[m], term[m]
__global__ void k_rank_gain(const double* __restrict__ lat, const int32_t* __restrict__ list, int m,
                            double* __restrict__ ws) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) ws[2 + i] = __dsub_rn(exp2(__ddiv_rn(ws[0], lat_of(lat, list, i))), 1.0);
}

__global__ void k_rank_pos(const double* __restrict__ sc, int m, double* __restrict__ ws) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double* gain = ws + 2;
  const double si = sc[i], gi = gain[i];
  int pos = 0, gpos = 0;
  for (int j = 0; j < m; ++j) {
    const double sj = sc[j], gj = gain[j];
    pos += sj > si || (sj == si && j < i);
    gpos += gj > gi || (gj == gi && j < i);
  }
  ws[2 + m + i] = __ddiv_rn(1.0, log2d_d((double)pos + 2.0));                  // discount under the scores
  ws[2 + 2 * m + gpos] = __ddiv_rn(gi, log2d_d((double)gpos + 2.0));          // ideal DCG term at its rank
}

__global__ void __launch_bounds__(1024) k_rank_dcg(int m, double* __restrict__ ws) {
  __shared__ double red[1024];
  const double* term = ws + 2 + 2 * m;
  const int per = (m + blockDim.x - 1) / blockDim.x;
  double v = 0.0;
  for (int q = 0; q < per; ++q) {
    const int p = threadIdx.x * per + q;
    if (p < m) v = __dadd_rn(v, term[p]);
  }
  const double tot = block_sum_fixed(v, red);
  if (threadIdx.x == 0) ws[1] = tot;
}

// thread (k, c): pairs of item k with items j of chunk c
__global__ void k_rank_pairs(const double* __restrict__ sc, const double* __restrict__ lat,
                             const int32_t* __restrict__ list, int m, int chunk, int nchunk,
                             const double* __restrict__ ws, double* __restrict__ gpart, double* __restrict__ lpart) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= m * nchunk) return;
  const int k = g % m, c = g / m;
  const double* gain = ws + 2;
  const double* disc = gain + m;
  const double maxdcg = ws[1];
  const double lk = lat_of(lat, list, k), sk = sc[k], gk = gain[k], dk = disc[k];
  double gr = 0.0, lo = 0.0;
  const int j1 = (c + 1) * chunk < m ? (c + 1) * chunk : m;
  for (int j = c * chunk; j < j1; ++j) {
    const double lj = lat_of(lat, list, j);
    const bool faster = lk < lj, slower = lj < lk;
    if (!faster && !slower) continue;
    // w = |gain_i - gain_j| |disc_i - disc_j| / maxdcg, i the faster item
    const double w = __ddiv_rn(__dmul_rn(fabs(__dsub_rn(faster ? gk : gain[j], faster ? gain[j] : gk)),
                                         fabs(__dsub_rn(faster ? dk : disc[j], faster ? disc[j] : dk))),
                               maxdcg);
    if (w == 0.0) continue;
    const double d = faster ? __dsub_rn(sk, sc[j]) : __dsub_rn(sc[j], sk);  // s_i - s_j
    const double slope = __dmul_rn(w, sigmoid_d(-d));
    if (faster) {
      lo = __dadd_rn(lo, __dmul_rn(w, softplus_d(-d)));
      gr = __dsub_rn(gr, slope);
    } else {
      gr = __dadd_rn(gr, slope);
    }
  }
  gpart[(size_t)c * m + k] = gr;
  lpart[(size_t)c * m + k] = lo;
}

__global__ void k_rank_fold(int m, int nchunk, const double* __restrict__ gpart, double* __restrict__ lpart,
                            double* __restrict__ dscore) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double gr = 0.0, lo = 0.0;
  for (int c = 0; c < nchunk; ++c) {
    gr = __dadd_rn(gr, gpart[(size_t)c * m + k]);
    lo = __dadd_rn(lo, lpart[(size_t)c * m + k]);
  }
  if (dscore) dscore[k] = gr;
  lpart[k] = lo;  // chunk 0's row now holds the per-item loss
}

__global__ void __launch_bounds__(1024) k_rank_loss(int m, const double* __restrict__ lpart,
                                                    double* __restrict__ loss, int accumulate) {
  __shared__ double red[1024];
  const int per = (m + blockDim.x - 1) / blockDim.x;
  double v = 0.0;
  for (int q = 0; q < per; ++q) {
    const int p = threadIdx.x * per + q;
    if (p < m) v = __dadd_rn(v, lpart[p]);
  }
  const double tot = block_sum_fixed(v, red);
  if (threadIdx.x == 0) *loss = accumulate ? __dadd_rn(*loss, tot) : tot;
}

}  // namespace

size_t rank_work_doubles(int m) {
  const int nchunk = rank_chunks(m);
  return 2 + 3 * (size_t)m + 2 * (size_t)nchunk * m;
}

int rank_chunks(int m) {
  const int chunk = m / 64 > 32 ? m / 64 : 32;
  return (m + chunk - 1) / chunk;
}

int launch_rank_loss(const double* scores, const double* lat, const int32_t* list, int m, double* work, int* bad,
                     double* loss, int accumulate, double* dscore, cudaStream_t st) {
  if (m < 2) return -1;
  const int nchunk = rank_chunks(m), chunk = (m + nchunk - 1) / nchunk;
  double* ws = work;
  double* gpart = ws + 2 + 3 * (size_t)m;
  double* lpart = gpart + (size_t)nchunk * m;
  const unsigned gm = (unsigned)((m + kRankThreads - 1) / kRankThreads);
  const unsigned gp = (unsigned)(((size_t)m * nchunk + kRankThreads - 1) / kRankThreads);
  k_rank_min<<<1, 1024, 0, st>>>(lat, list, m, ws, bad);
  k_rank_gain<<<gm, kRankThreads, 0, st>>>(lat, list, m, ws);
  k_rank_pos<<<gm, kRankThreads, 0, st>>>(scores, m, ws);
  k_rank_dcg<<<1, 1024, 0, st>>>(m, ws);
  k_rank_pairs<<<gp, kRankThreads, 0, st>>>(scores, lat, list, m, chunk, nchunk, ws, gpart, lpart);
  k_rank_fold<<<gm, kRankThreads, 0, st>>>(m, nchunk, gpart, lpart, dscore);
  k_rank_loss<<<1, 1024, 0, st>>>(m, lpart, loss, accumulate);
  for (int q = 0; q < 7; ++q) tt::note_launch();
  return cudaGetLastError() != cudaSuccess;
}

}  // namespace tt
