// k_select.cu — K2b select_top, the certification band, and K4 (MoA GD
// step + momentum EMA).
//
// select_top (ranker.cpp:514-532): indices of the b best candidates by
// descending score, ties by ascending draft cost, then ascending index;
// excluded entries never selected. Keys are mapped to order-preserving
// uint64 (so a CTA bitonic sort on (score key, draft key, index) is exactly
// the reference comparator); tiles of 4096 keep their top b, a second CTA
// merges the tile winners.
#include <cstdint>

#include "tt_block.cuh"
#include "tt_kernels.h"

namespace tt {

constexpr int kSelTile = 4096;
constexpr uint64_t kAll = ~0ull;

__device__ __forceinline__ uint64_t ordered(double x) {
  const uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

struct TopbScratch {
  uint64_t* a;
  uint64_t* b;
  uint64_t* c;
};

// Phase 1: each CTA sorts one tile and keeps its b best.
__global__ void __launch_bounds__(1024) k_topb_tile(const double* __restrict__ scores, const double* __restrict__ drafts,
                                                    const uint8_t* __restrict__ excluded, int64_t n,
                                                    const int64_t* __restrict__ n_dev, int64_t b, int final_out,
                                                    uint64_t* __restrict__ wa, uint64_t* __restrict__ wb,
                                                    uint64_t* __restrict__ wc, int64_t* __restrict__ out_pos,
                                                    int64_t* __restrict__ out_count, int* __restrict__ status) {
  extern __shared__ __align__(16) uint64_t sk[];
  uint64_t* a = sk;
  uint64_t* bb = a + kSelTile;
  uint64_t* c = bb + kSelTile;
  __shared__ int avail;
  if (n_dev) n = *n_dev < n ? *n_dev : n;
  const int64_t base = (int64_t)blockIdx.x * kSelTile;
  const int m = (int)((n - base) < kSelTile ? (n - base) : kSelTile);
  const int np = next_pow2(m < 2 ? 2 : m);
  if (threadIdx.x == 0) avail = 0;
  __syncthreads();
  int mine = 0;
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    const int64_t i = base + e;
    const bool ok = e < m && !(excluded && excluded[i]);
    a[e] = ok ? ~ordered(scores[i]) : kAll;
    bb[e] = ok ? ordered(drafts[i]) : kAll;
    c[e] = ok ? (uint64_t)i : kAll;
    mine += ok;
  }
  if (mine) atomicAdd(&avail, mine);
  block_bitonic_sort<true>(a, bb, c, np);
  const int keep = (int)(b < avail ? b : avail);
  if (final_out) {
    for (int e = threadIdx.x; e < keep; e += blockDim.x) out_pos[e] = (int64_t)c[e];
    if (threadIdx.x == 0) {
      *out_count = keep;
      *status = avail < b ? 1 : 0;
    }
  } else {
    for (int e = threadIdx.x; e < b; e += blockDim.x) {
      const int64_t o = (int64_t)blockIdx.x * b + e;
      wa[o] = e < keep ? a[e] : kAll;
      wb[o] = e < keep ? bb[e] : kAll;
      wc[o] = e < keep ? c[e] : kAll;
    }
  }
}

// Phase 2: merge the tiles' winners.
__global__ void __launch_bounds__(1024) k_topb_merge(const uint64_t* __restrict__ wa, const uint64_t* __restrict__ wb,
                                                     const uint64_t* __restrict__ wc, int m, int64_t b,
                                                     int64_t* __restrict__ out_pos, int64_t* __restrict__ out_count,
                                                     int* __restrict__ status) {
  extern __shared__ __align__(16) uint64_t sk[];
  const int np = next_pow2(m < 2 ? 2 : m);
  uint64_t* a = sk;
  uint64_t* bb = a + np;
  uint64_t* c = bb + np;
  __shared__ int avail;
  if (threadIdx.x == 0) avail = 0;
  __syncthreads();
  int mine = 0;
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    a[e] = e < m ? wa[e] : kAll;
    bb[e] = e < m ? wb[e] : kAll;
    c[e] = e < m ? wc[e] : kAll;
    mine += e < m && c[e] != kAll;
  }
  if (mine) atomicAdd(&avail, mine);
  block_bitonic_sort<true>(a, bb, c, np);
  const int keep = (int)(b < avail ? b : avail);
  for (int e = threadIdx.x; e < keep; e += blockDim.x) out_pos[e] = (int64_t)c[e];
  if (threadIdx.x == 0) {
    *out_count = keep;
    *status = avail < b ? 1 : 0;
  }
}

// Scratch for phase 1 winners lives in a static device buffer sized for
// the largest supported call (tiles * b <= kSelTile).
__device__ uint64_t g_topb_a[kSelTile], g_topb_b[kSelTile], g_topb_c[kSelTile];

int launch_select_top(const double* scores, const double* drafts, const uint8_t* excluded, int64_t n,
                      const int64_t* n_dev, int64_t b, int64_t* out_pos, int64_t* out_count, int* status,
                      cudaStream_t st) {
  if (b < 1 || n < 0) return -1;
  const int64_t tiles = (n + kSelTile - 1) / kSelTile;
  const size_t sm1 = (size_t)kSelTile * 3 * sizeof(uint64_t);
  cudaFuncSetAttribute(k_topb_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
  if (tiles <= 1) {
    tt::note_launch(), k_topb_tile<<<1, 1024, sm1, st>>>(scores, drafts, excluded, n, n_dev, b, 1, nullptr, nullptr, nullptr, out_pos,
                                      out_count, status);
    return 0;
  }
  if (b > kSelTile || tiles * b > kSelTile) return -2;
  uint64_t *wa, *wb, *wc;
  cudaGetSymbolAddress((void**)&wa, g_topb_a);
  cudaGetSymbolAddress((void**)&wb, g_topb_b);
  cudaGetSymbolAddress((void**)&wc, g_topb_c);
  tt::note_launch(), k_topb_tile<<<(unsigned)tiles, 1024, sm1, st>>>(scores, drafts, excluded, n, n_dev, b, 0, wa, wb, wc, out_pos,
                                                  out_count, status);
  const int m = (int)(tiles * b);
  const size_t sm2 = (size_t)next_pow2(m) * 3 * sizeof(uint64_t);
  cudaFuncSetAttribute(k_topb_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  tt::note_launch(), k_topb_merge<<<1, 1024, sm2, st>>>(wa, wb, wc, m, b, out_pos, out_count, status);
  return 0;
}

// ------------------------------------------------ certification band ----
// Given the fast-path top-b positions, mark every candidate whose fast
// score is within 2*band of the b-th fast score for exact fp64 rescoring;
// everything else is excluded from the final exact selection. If every
// fast error is below `band`, the excluded candidates are provably outside
// the true top-b.
__global__ void __launch_bounds__(1024) k_band(const double* __restrict__ fast, const int64_t* __restrict__ n_dev,
                                               int64_t n_max, const int64_t* __restrict__ pos_fast,
                                               const int64_t* __restrict__ pos_count, double band,
                                               int32_t* __restrict__ sublist, int* __restrict__ sublist_count,
                                               uint8_t* __restrict__ excluded) {
  __shared__ int cnt;
  const int64_t n = n_dev ? (*n_dev < n_max ? *n_dev : n_max) : n_max;
  const int64_t pc = *pos_count;
  const double thr = pc > 0 ? fast[pos_fast[pc - 1]] - 2.0 * band : -1.0e300;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n_max; i += blockDim.x) {
    const bool in = i < n && fast[i] >= thr;
    excluded[i] = in ? 0 : 1;
    if (in) sublist[atomicAdd(&cnt, 1)] = (int32_t)i;
  }
  __syncthreads();
  if (threadIdx.x == 0) *sublist_count = cnt;
}

int launch_band(const double* fast, const int64_t* n_dev, int64_t n_max, const int64_t* pos_fast,
                     const int64_t* pos_count, double band, int32_t* sublist, int* sublist_count, uint8_t* excluded,
                     cudaStream_t st) {
  tt::note_launch(), k_band<<<1, 1024, 0, st>>>(fast, n_dev, n_max, pos_fast, pos_count, band, sublist, sublist_count, excluded);
  return 0;
}

// --------------------------------------------------------------- MoA ----
// GD update of train (ranker.cpp:502-506): p -= lr * g.
__global__ void k_gd(double* __restrict__ p, const double* __restrict__ g, int64_t n, double lr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __dsub_rn(p[i], __dmul_rn(lr, g[i]));
}

// momentum_update (momentum.cpp:28-46): phi' = t + m * (phi - t), FMA-free so
// m = 0 and phi = t are bit-exact endpoints.
__global__ void k_ema(double* __restrict__ phi, const double* __restrict__ t, int64_t n, double m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ti = t[i];
    phi[i] = __dadd_rn(ti, __dmul_rn(m, __dsub_rn(phi[i], ti)));
  }
}

int launch_gd_step(double* params, const double* grads, int64_t n, double lr, cudaStream_t st) {
  if (n <= 0) return 0;
  const int g = (int)((n + 255) / 256 < 148 * 4 ? (n + 255) / 256 : 148 * 4);
  tt::note_launch(), k_gd<<<g, 256, 0, st>>>(params, grads, n, lr);
  return 0;
}

int launch_momentum(double* phi, const double* target, int64_t n, double m, cudaStream_t st) {
  if (n <= 0) return 0;
  const int g = (int)((n + 255) / 256 < 148 * 4 ? (n + 255) / 256 : 148 * 4);
  tt::note_launch(), k_ema<<<g, 256, 0, st>>>(phi, target, n, m);
  return 0;
}

// ------------------------------------------------- result gathering ----
// Packs the round's b selections into one record for a single
// device->host copy. Layout (8-byte words): [0] selected, [1] drafted,
// [2] status, [3] rescored, then b population indices, b scores, b draft
// costs, b identities.
__global__ void k_gather(const int64_t* __restrict__ pos, const int64_t* __restrict__ pos_count,
                         const int64_t* __restrict__ drafted_count, const SelState* __restrict__ sel,
                         const int* __restrict__ status_b, const int* __restrict__ rescored,
                         const int64_t* __restrict__ idx, const double* __restrict__ cost,
                         const uint64_t* __restrict__ id, const double* __restrict__ scores, int64_t b,
                         int64_t* __restrict__ out) {
  const int64_t cnt = *pos_count;
  const int t = threadIdx.x;
  if (t == 0) {
    out[0] = cnt;
    out[1] = *drafted_count;
    out[2] = (int64_t)((sel ? sel->status : 0) | ((status_b ? *status_b : 0) << 8));
    out[3] = rescored ? *rescored : 0;
  }
  int64_t* ix = out + 4;
  double* sc = (double*)(ix + b);
  double* co = sc + b;
  uint64_t* ids = (uint64_t*)(co + b);
  for (int64_t e = t; e < b; e += blockDim.x) {
    if (e < cnt) {
      const int64_t p = pos[e];
      ix[e] = idx[p];
      sc[e] = scores[p];
      co[e] = cost[p];
      ids[e] = id ? id[p] : 0;
    } else {
      ix[e] = -1;
      sc[e] = 0.0, co[e] = 0.0, ids[e] = 0;
    }
  }
}

int launch_gather(const int64_t* pos, const int64_t* pos_count, const int64_t* drafted_count, const SelState* sel,
                  const int* status_b, const int* rescored, const int64_t* idx, const double* cost,
                  const uint64_t* id, const double* scores, int64_t b, int64_t* out, cudaStream_t st) {
  tt::note_launch(), k_gather<<<1, 128, 0, st>>>(pos, pos_count, drafted_count, sel, status_b, rescored, idx, cost, id, scores, b, out);
  return 0;
}

}  // namespace tt
