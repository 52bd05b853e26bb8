// tt_finish.cuh — the round's finish (select_top, ranker.cpp:514-532, fused
// with the round-record gather) as a block-level device function: run by
// k_finish (k_select.cu) and by the last CTA of k_verify64 (k_verify.cu).
#pragma once

#include <cstdint>

#include "tt_block.cuh"
#include "tt_kernels.h"

namespace tt {

constexpr uint64_t kAll = ~0ull;

// -0.0 and +0.0 map to one key: the reference comparator (scores[a] !=
// scores[c]) treats them as equal and falls through to the draft cost
__device__ __forceinline__ uint64_t ordered(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// ------------------------------------------------------------ finish ----
// The round's select_top (ranker.cpp:514-532: score desc, draft cost asc,
// position asc; excluded never chosen) fused with the record gather for the
// single device->host copy: [0] selected, [1] drafted, [2] status, [3]
// rescored, then b population indices, b scores, b draft costs, b
// identities. n <= 1024, b <= 32: the keys no larger than the b-th smallest
// warp minimum (a bound on the b-th best) are the only candidates; they are
// ranked among each other by counting.
__device__ __forceinline__ void warp_sort32(Key3& k) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const Key3 o = k.shfl_xor(stride);
      const bool lower = (lane & stride) == 0, up = (lane & size) == 0;
      const bool take = (lower == up) ? o.lt(k) : k.lt(o);
      if (take) k = o;
    }
  }
}

// The body, for a CTA of >= n_max threads (a multiple of 32); shared scratch
// passed in (FinishSmem), so a kernel can run it in memory it is done with.
static __device__ long long g_fin_clk[8];  // finish_block phase marks (thread 0; probe)

// this round's slot of the record ring (one thread takes it, all get it)
__device__ __forceinline__ int64_t* ring_slot(const RecRing& r, int* s_slot) {
  if (threadIdx.x == 0) *s_slot = (int)(atomicAdd(r.seq, 1u) % (unsigned)kRingSlots);
  __syncthreads();
  return r.base + (int64_t)(*s_slot) * r.stride;
}

struct FinishSmem {
  int slot;
  Key3 lists[32][33];
  int16_t rank_of[1024];  // output position of each selected candidate, -1 otherwise
  int cnt[1024];          // candidates' ranks among the warps' b best
  int avail;
  unsigned long long band_err;
};

__device__ __forceinline__ void finish_block(const double* __restrict__ scores, const double* __restrict__ drafts,
                                             const uint8_t* __restrict__ excluded, int64_t n_max,
                                             const int64_t* __restrict__ n_dev, int64_t b,
                                             const int64_t* __restrict__ idx, const uint64_t* __restrict__ id,
                                             const SelState* __restrict__ sel, const int* __restrict__ rescored,
                                             const double* __restrict__ fast, RecRing ring,
                                             int* __restrict__ invalid, FinishSmem& fs) {
  auto& lists = fs.lists;
  auto& avail = fs.avail;
  auto& band_err = fs.band_err;
  auto& rank_of = fs.rank_of;
  int64_t* __restrict__ out = ring_slot(ring, &fs.slot);
  if (threadIdx.x == 0) g_fin_clk[4] = clock64();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  // every global read issued up front, independent of each other (one
  // memory round trip): the count, this thread's candidate, and the record
  // fields it writes if it is selected
  const int64_t nd = n_dev ? *n_dev : n_max;
  const bool in = t < n_max;
  const double s_t = in ? __ldcg(scores + t) : 0.0, d_t = in ? __ldcg(drafts + t) : 0.0;
  const bool ex_t = in && excluded && excluded[t];
  const int64_t ix_t = in ? __ldcg(idx + t) : -1;
  const uint64_t id_t = in && id ? __ldcg(id + t) : 0;
  const int64_t st = t == 0 && sel ? (int64_t)sel->status : 0;
  const int64_t rs = t == 0 && rescored ? (int64_t)*rescored : 0;
  const double f_t = in && fast ? fast[t] : 0.0;
  if (t == 0) avail = 0, band_err = 0ull;
  rank_of[t] = -1;
  __syncthreads();
  if (threadIdx.x == 0) g_fin_clk[0] = clock64();
  const int64_t n = nd < n_max ? nd : n_max;
  const bool ok = t < n && !ex_t;
  if (fast) {  // the certification's premise, checked on the rescored set
    double err = ok ? fabs(s_t - f_t) : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) err = fmax(err, __shfl_xor_sync(0xffffffffu, err, off));
    if (lane == 0 && err > 0.0) atomicMax(&band_err, (unsigned long long)__double_as_longlong(err));
  }
  Key3 k;
  k.a = ok ? ~ordered(s_t) : kAll;
  k.b = ok ? ordered(d_t) : kAll;
  k.c = ok ? (uint32_t)t : 0xffffffffu;
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  if (lane == 0 && bal) atomicAdd(&avail, __popc(bal));
  // filter: M = the b-th smallest of the warps' minima (select_top's order is
  // ascending Key3). At least b keys are <= M (those b warp minima), so the
  // b best are all <= M; when fewer than b warps hold a key, every key is a
  // candidate. Only the candidates are ranked, by counting.
  Key3 mn = k;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Key3 o = mn.shfl_xor(off);
    if (o.lt(mn)) mn = o;
  }
  Key3* wmin = &lists[0][0];   // [nw <= 32] warp minima
  Key3* cand = &lists[0][32];  // the candidates: <= 32 b <= 1024 (the keys of the <= b warps whose minimum is <= M)
  if (lane == 0) wmin[warp] = mn;
  if (t == 0) fs.cnt[0] = 0;  // candidate count
  __syncthreads();
  if (threadIdx.x == 0) g_fin_clk[1] = clock64();
  if (warp == 0) {  // lane w: rank of warp w's minimum among the minima
    Key3 me;
    me.a = kAll, me.b = kAll, me.c = 0xffffffffu;
    if (lane < nw) me = wmin[lane];
    int r = 0;
    for (int q = 0; q < nw; ++q) r += wmin[q].lt(me) ? 1 : 0;
    const unsigned hit = __ballot_sync(0xffffffffu, me.c != 0xffffffffu && r == (int)b - 1);
    if (lane == 0) fs.cnt[1] = hit ? (int)(__ffs(hit) - 1) : -1;  // the warp whose minimum is M, or none
  }
  __syncthreads();
  const int mw = fs.cnt[1];
  Key3 M;
  M.a = kAll, M.b = kAll, M.c = 0xffffffffu;
  if (mw >= 0) M = wmin[mw];
  if (k.c != 0xffffffffu && !M.lt(k)) cand[atomicAdd(&fs.cnt[0], 1)] = k;  // k <= M
  __syncthreads();
  if (threadIdx.x == 0) g_fin_clk[2] = clock64();
  const int64_t keep = b < avail ? b : avail;
  const int m = fs.cnt[0];
  if (threadIdx.x == 0) g_fin_clk[5] = m, g_fin_clk[6] = mw;
  for (int i = t; i < m; i += blockDim.x) {  // rank among the candidates (a strict total order)
    const Key3 me = cand[i];
    int r = 0;
    for (int q = 0; q < m; ++q) r += cand[q].lt(me) ? 1 : 0;
    if (r < keep) rank_of[me.c] = (int16_t)r;
  }
  __syncthreads();
  if (threadIdx.x == 0) g_fin_clk[3] = clock64();
  int64_t* ix = out + kRecHead;
  double* sc = (double*)(ix + b);
  double* co = sc + b;
  uint64_t* ids = (uint64_t*)(co + b);
  const int r = rank_of[t];
  if (r >= 0) ix[r] = ix_t, sc[r] = s_t, co[r] = d_t, ids[r] = id_t;  // the selected candidate writes its own entry
  if (t >= keep && t < b) ix[t] = -1, sc[t] = 0.0, co[t] = 0.0, ids[t] = 0;
  if (t == 0) {
    out[0] = keep;
    out[1] = n;
    out[2] = st;
    out[3] = rs;
    out[4] = 0;
    out[5] = (int64_t)band_err;
    if (invalid) out[6] = *(volatile int*)invalid, *invalid = 0;  // K1 set it earlier in this round
    else out[6] = 0;
  }
}


}  // namespace tt
