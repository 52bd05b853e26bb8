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
#include "tt_finish.cuh"
#include "tt_kernels.h"

namespace tt {

constexpr int kSelTile = 4096;

constexpr int kTopbE = 4;  // keys per thread

// Phase 1: each CTA sorts one tile of up to 4 * blockDim keys
// (~score, draft, index) in registers and keeps its b best. With
// final_out the CTA writes the answer directly.
__global__ void __launch_bounds__(1024) k_topb_tile(const double* __restrict__ scores, const double* __restrict__ drafts,
                                                    const uint8_t* __restrict__ excluded, int64_t n,
                                                    const int64_t* __restrict__ n_dev, int64_t b, int final_out,
                                                    Key3* __restrict__ win, int64_t* __restrict__ out_pos,
                                                    int64_t* __restrict__ out_count, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char sraw[];
  Key3* xchg = (Key3*)sraw;
  __shared__ int avail;
  if (n_dev) n = *n_dev < n ? *n_dev : n;
  const int tile = kTopbE * blockDim.x;
  const int64_t base = (int64_t)blockIdx.x * tile;
  if (threadIdx.x == 0) avail = 0;
  __syncthreads();
  int mine = 0;
  Key3 kk[kTopbE];
#pragma unroll
  for (int e = 0; e < kTopbE; ++e) {
    const int64_t i = base + e * blockDim.x + threadIdx.x;
    const bool ok = i < n && !(excluded && excluded[i]);
    kk[e].a = ok ? ~ordered(scores[i]) : kAll;
    kk[e].b = ok ? ordered(drafts[i]) : kAll;
    kk[e].c = ok ? (uint32_t)i : 0xffffffffu;
    mine += ok;
  }
  if (mine) atomicAdd(&avail, mine);
  block_sort_reg<kTopbE, Key3>(kk, xchg);
  const int keep = (int)(b < avail ? b : avail);
#pragma unroll
  for (int e = 0; e < kTopbE; ++e) {
    const int p = e * blockDim.x + threadIdx.x;
    if (p < b) {
      if (final_out) {
        if (p < keep) out_pos[p] = (int64_t)kk[e].c;
      } else {
        Key3 w = kk[e];
        if (p >= keep) w.a = kAll, w.b = kAll, w.c = 0xffffffffu;
        win[(int64_t)blockIdx.x * b + p] = w;
      }
    }
  }
  if (final_out && threadIdx.x == 0) {
    *out_count = keep;
    *status = avail < b ? 1 : 0;
  }
}

// Phase 2: merge the tiles' winners (all of them fit one CTA).
__global__ void __launch_bounds__(1024) k_topb_merge(const Key3* __restrict__ win, int m, int64_t b,
                                                     int64_t* __restrict__ out_pos, int64_t* __restrict__ out_count,
                                                     int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char sraw[];
  Key3* xchg = (Key3*)sraw;
  __shared__ int avail;
  if (threadIdx.x == 0) avail = 0;
  __syncthreads();
  int mine = 0;
  Key3 kk[kTopbE];
#pragma unroll
  for (int e = 0; e < kTopbE; ++e) {
    const int p = e * blockDim.x + threadIdx.x;
    if (p < m) kk[e] = win[p];
    else kk[e].a = kAll, kk[e].b = kAll, kk[e].c = 0xffffffffu;
    mine += p < m && kk[e].a != kAll;
  }
  if (mine) atomicAdd(&avail, mine);
  block_sort_reg<kTopbE, Key3>(kk, xchg);
  const int keep = (int)(b < avail ? b : avail);
#pragma unroll
  for (int e = 0; e < kTopbE; ++e) {
    const int p = e * blockDim.x + threadIdx.x;
    if (p < keep) out_pos[p] = (int64_t)kk[e].c;
  }
  if (threadIdx.x == 0) {
    *out_count = keep;
    *status = avail < b ? 1 : 0;
  }
}

// Small b over one tile (the round's case: b = 10 of K = 512): b rounds of
// a CTA-wide arg-min over the (~score, draft, index) keys — O(b * n) work
// instead of a full sorting network.
constexpr int kArgThreads = 256;

__device__ __forceinline__ Key3 kmin(const Key3& x, const Key3& y) { return y.lt(x) ? y : x; }

__global__ void __launch_bounds__(kArgThreads) k_topb_argmin(const double* __restrict__ scores,
                                                             const double* __restrict__ drafts,
                                                             const uint8_t* __restrict__ excluded, int64_t n,
                                                             const int64_t* __restrict__ n_dev, int64_t b,
                                                             int64_t* __restrict__ out_pos,
                                                             int64_t* __restrict__ out_count, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char sraw[];
  Key3* ks = (Key3*)sraw;
  __shared__ Key3 wbest[kArgThreads / 32];
  __shared__ int avail;
  if (n_dev) n = *n_dev < n ? *n_dev : n;
  if (threadIdx.x == 0) avail = 0;
  __syncthreads();
  int mine = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const bool ok = !(excluded && excluded[i]);
    Key3 k;
    k.a = ok ? ~ordered(scores[i]) : kAll;
    k.b = ok ? ordered(drafts[i]) : kAll;
    k.c = ok ? (uint32_t)i : 0xffffffffu;
    ks[i] = k;
    mine += ok;
  }
  if (mine) atomicAdd(&avail, mine);
  __syncthreads();
  const int keep = (int)(b < avail ? b : avail);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int it = 0; it < keep; ++it) {
    Key3 best;
    best.a = kAll, best.b = kAll, best.c = 0xffffffffu;
    for (int i = threadIdx.x; i < n; i += blockDim.x) best = kmin(best, ks[i]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) best = kmin(best, best.shfl_xor(off));
    if (lane == 0) wbest[warp] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
      Key3 m = wbest[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = kmin(m, wbest[w]);
      out_pos[it] = (int64_t)m.c;
      ks[m.c].a = kAll, ks[m.c].b = kAll, ks[m.c].c = 0xffffffffu;  // taken
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out_count = keep;
    *status = avail < b ? 1 : 0;
  }
}

// Scratch for phase-1 winners (tiles * b <= kSelTile).
__device__ Key3 g_topb_win[kSelTile];

static int threads_for(int64_t m) {
  int nt = 32;
  while (nt < 1024 && (int64_t)kTopbE * nt < m) nt <<= 1;
  return nt;
}

int launch_select_top(const double* scores, const double* drafts, const uint8_t* excluded, int64_t n,
                      const int64_t* n_dev, int64_t b, int64_t* out_pos, int64_t* out_count, int* status,
                      cudaStream_t st) {
  if (b < 1 || n < 0 || n >= (int64_t{1} << 32)) return -1;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_topb_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSelTile * sizeof(Key3)));
    cudaFuncSetAttribute(k_topb_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSelTile * sizeof(Key3)));
    init = true;
  }
  const int64_t tiles = (n + kSelTile - 1) / kSelTile;
  if (tiles <= 1 && b <= 32) {
    static bool init2 = false;
    if (!init2) {
      cudaFuncSetAttribute(k_topb_argmin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSelTile * sizeof(Key3)));
      init2 = true;
    }
    tt::note_launch();
    k_topb_argmin<<<1, kArgThreads, (n > 0 ? n : 1) * sizeof(Key3), st>>>(scores, drafts, excluded, n, n_dev, b,
                                                                          out_pos, out_count, status);
    return 0;
  }
  if (tiles <= 1) {
    const int nt = threads_for(n);
    tt::note_launch();
    k_topb_tile<<<1, nt, kTopbE * nt * sizeof(Key3), st>>>(scores, drafts, excluded, n, n_dev, b, 1, nullptr, out_pos,
                                                           out_count, status);
    return 0;
  }
  if (b > kSelTile || tiles * b > kSelTile) return -2;
  Key3* win;
  cudaGetSymbolAddress((void**)&win, g_topb_win);
  tt::note_launch();
  k_topb_tile<<<(unsigned)tiles, 1024, kSelTile * sizeof(Key3), st>>>(scores, drafts, excluded, n, n_dev, b, 0, win,
                                                                      out_pos, out_count, status);
  const int m = (int)(tiles * b);
  const int nt = threads_for(m);
  tt::note_launch();
  k_topb_merge<<<1, nt, kTopbE * nt * sizeof(Key3), st>>>(win, m, b, out_pos, out_count, status);
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

// ------------------------------------------------------------ finish ----
__global__ void __launch_bounds__(1024) k_finish(const double* __restrict__ scores, const double* __restrict__ drafts,
                                                 const uint8_t* __restrict__ excluded, int64_t n_max,
                                                 const int64_t* __restrict__ n_dev, int64_t b,
                                                 const int64_t* __restrict__ idx, const uint64_t* __restrict__ id,
                                                 const SelState* __restrict__ sel, const int* __restrict__ rescored,
                                                 const double* __restrict__ fast, RecRing out,
                                                 int* __restrict__ invalid) {
  __shared__ FinishSmem fs;
  finish_block(scores, drafts, excluded, n_max, n_dev, b, idx, id, sel, rescored, fast, out, invalid, fs);
}

// Certification band for the tensor-core path, one CTA (n <= 1024,
// b <= 32): the b-th best fast key by select_top's order (warp sorts + a
// tournament, as k_finish), then every candidate whose fast score is within
// 2 * band of it goes on the fp64 rescoring sublist; the rest are excluded
// from the final selection. If every fast error is below `band`, excluded
// candidates are provably outside the true top-b.
__global__ void __launch_bounds__(1024) k_cert_band(const double* __restrict__ fast,
                                                    const double* __restrict__ drafts, int64_t n_max,
                                                    const int64_t* __restrict__ n_dev, int64_t b, double band,
                                                    int32_t* __restrict__ sublist, int* __restrict__ sublist_count,
                                                    uint8_t* __restrict__ excluded) {
  __shared__ Key3 lists[32][33];
  __shared__ double thr;
  __shared__ int cnt;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  const int64_t n = n_dev ? (*n_dev < n_max ? *n_dev : n_max) : n_max;
  const bool ok = t < n;
  Key3 k;
  k.a = ok ? ~ordered(fast[t]) : kAll;
  k.b = ok ? ordered(drafts[t]) : kAll;
  k.c = ok ? (uint32_t)t : 0xffffffffu;
  warp_sort32(k);
  lists[warp][lane] = k;
  if (lane == 0) lists[warp][32].a = kAll, lists[warp][32].b = kAll, lists[warp][32].c = 0xffffffffu, cnt = 0;
  if (t == 0) thr = -1.0e300;
  __syncthreads();
  if (warp == 0) {
    int head = 0;
    uint32_t last = 0xffffffffu;
    const int64_t keep = b < n ? b : n;
    for (int it = 0; it < keep; ++it) {
      Key3 h;
      if (lane < nw) h = lists[lane][head];
      else h.a = kAll, h.b = kAll, h.c = 0xffffffffu;
      Key3 m = h;
      int who = lane;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const Key3 o = m.shfl_xor(off);
        const int ow = __shfl_xor_sync(0xffffffffu, who, off);
        if (o.lt(m)) m = o, who = ow;
      }
      last = m.c;
      if (lane == who) ++head;
    }
    if (lane == 0 && last != 0xffffffffu) thr = fast[last] - 2.0 * band;
  }
  __syncthreads();
  if (t < n_max) {
    const bool in = ok && fast[t] >= thr;
    excluded[t] = in ? 0 : 1;
    if (in) sublist[atomicAdd(&cnt, 1)] = t;
  }
  __syncthreads();
  if (t == 0) *sublist_count = cnt;
}

int launch_cert_band(const double* fast, const double* drafts, int64_t n_max, const int64_t* n_dev, int64_t b,
                     double band, int32_t* sublist, int* sublist_count, uint8_t* excluded, cudaStream_t st) {
  if (n_max > 1024 || b > 32) return -1;
  const int nt = (int)((n_max + 31) / 32 * 32);
  tt::note_launch();
  k_cert_band<<<1, nt, 0, st>>>(fast, drafts, n_max, n_dev, b, band, sublist, sublist_count, excluded);
  return 0;
}

int launch_finish(const double* scores, const double* drafts, const uint8_t* excluded, int64_t n_max,
                  const int64_t* n_dev, int64_t b, const int64_t* idx, const uint64_t* id, const SelState* sel,
                  const int* rescored, const double* fast, RecRing out, int* invalid, cudaStream_t st) {
  if (n_max > 1024 || b > 32 || b > n_max) return -1;
  const int nt = (int)((n_max + 31) / 32 * 32);
  tt::note_launch();
  k_finish<<<1, nt, 0, st>>>(scores, drafts, excluded, n_max, n_dev, b, idx, id, sel, rescored, fast, out, invalid);
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
                         const uint64_t* __restrict__ id, const double* __restrict__ scores,
                         const double* __restrict__ fast, const uint8_t* __restrict__ excluded, int64_t n_max,
                         int64_t b, RecRing ring, int* __restrict__ invalid) {
  __shared__ unsigned long long band_err;
  __shared__ int s_slot;
  int64_t* __restrict__ out = ring_slot(ring, &s_slot);
  const int64_t cnt = *pos_count;
  const int t = threadIdx.x;
  if (t == 0) band_err = 0ull;
  __syncthreads();
  if (fast) {  // max |exact - fast| over the rescored (not excluded) candidates
    const int64_t nd = *drafted_count < n_max ? *drafted_count : n_max;
    double err = 0.0;
    for (int64_t i = t; i < nd; i += blockDim.x)
      if (!(excluded && excluded[i])) err = fmax(err, fabs(scores[i] - fast[i]));
    if (err > 0.0) atomicMax(&band_err, (unsigned long long)__double_as_longlong(err));
  }
  __syncthreads();
  if (t == 0) {
    out[0] = cnt;
    out[1] = *drafted_count;
    out[2] = (int64_t)((sel ? sel->status : 0) | ((status_b ? *status_b : 0) << 8));
    out[3] = rescored ? *rescored : 0;
    out[4] = 0;
    out[5] = (int64_t)band_err;
    if (invalid) out[6] = *(volatile int*)invalid, *invalid = 0;
    else out[6] = 0;
  }
  int64_t* ix = out + kRecHead;
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
                  const uint64_t* id, const double* scores, const double* fast, const uint8_t* excluded,
                  int64_t n_max, int64_t b, RecRing out, int* invalid, cudaStream_t st) {
  tt::note_launch(), k_gather<<<1, 128, 0, st>>>(pos, pos_count, drafted_count, sel, status_b, rescored, idx, cost, id,
                                                 scores, fast, excluded, n_max, b, out, invalid);
  return 0;
}

}  // namespace tt
