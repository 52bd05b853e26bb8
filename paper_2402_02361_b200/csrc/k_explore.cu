// k_explore.cu — one generation of the genetic explorer on the device:
// mutate(population, sketch, costs, rng) (schedule.cpp:340-396), bit-exact.
//
// mutate() is written as one sequential RNG stream: child j draws a parent
// (uniform_real), a slot (uniform_index), then — depending on that parent's
// factors — 0, 1 or 2 more values. Its draws start where child j-1's ended,
// so the reference loop is inherently serial. Here it is split into
//   1. a parallel "length" pass: for EVERY stream offset o that could start a
//      child, the number of draws L(o) in {2, 3, 4} a child starting there
//      consumes (parent and slot are functions of draws o, o+1 only — the
//      stream is counter based);
//   2. one thread walks the chain o_1 = 0, o_{j+1} = o_j + L(o_j) over L in
//      shared memory (n - 1 dependent shared loads);
//   3. a parallel apply pass: child j re-derives its draws at o_j and writes
//      its factors.
// The roulette-wheel prefix sum is one thread's fp64 chain in the reference
// order (the weights are computed in parallel first), so `total` and every
// cumulative bound are the reference's bits. Built with --fmad=false.
//
// One CTA per generation (n <= kMutateMaxN); the population is tiny (512 at
// the TunerConfig defaults) and the generation chain is latency bound, so
// the kernel's job is to remove the host round trip from the GA loop.
#include <cuda_runtime.h>

#include "tt_kernels.h"

namespace tt {

namespace {

constexpr int kMutThreads = 1024;

__device__ __forceinline__ int64_t upper_bound_d(const double* cum, int64_t n, double r) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cum[mid] > r) hi = mid; else lo = mid + 1;
  }
  return lo < n - 1 ? lo : n - 1;
}

__device__ __forceinline__ int slot_col0(const DevSketch& S, int slot) {
  return slot < S.n_sp ? 4 * slot : 4 * S.n_sp + 3 * (slot - S.n_sp);
}

// Moves of factor tuple f (positions 0..arity-1) in the reference's order:
// position ascending, prime ascending, repeated by multiplicity
// (schedule.cpp:377-381). Returns the count; if `pick` >= 0 also returns the
// pick-th move's (position, prime).
__device__ __forceinline__ int moves_of(const DevSketch& S, int slot, const uint32_t* f, int arity, int pick,
                                        int* pos, int64_t* prime) {
  int cnt = 0;
  for (int q = 0; q < arity; ++q) {
    uint32_t v = f[q];
    for (int t = 0; t < S.n_prime && v > 1; ++t) {
      if (S.pr_axis[t] != slot) continue;
      int e = 0;
      if (S.pr_p[t] == 2) {
        e = __ffs(v) - 1;
        v >>= e;
      } else {
        for (uint32_t qv = v * S.pr_inv[t]; qv <= S.pr_lim[t]; qv = v * S.pr_inv[t]) v = qv, ++e;
      }
      if (pick >= cnt && pick < cnt + e) *pos = q, *prime = S.pr_p[t];
      cnt += e;
    }
  }
  return cnt;
}

__global__ void __launch_bounds__(kMutThreads) k_mutate(DevSketch S, const int32_t* __restrict__ pop,
                                                        const double* __restrict__ cost, int n,
                                                        uint64_t* __restrict__ state, int32_t* __restrict__ next) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* cum = (double*)smem;                 // [n]
  int32_t* off = (int32_t*)(cum + n);           // [n] stream offset of child j
  uint8_t* len = (uint8_t*)(off + n);           // [4n] draws a child starting at o consumes
  __shared__ uint64_t s_state;
  __shared__ double s_total;
  __shared__ double s_bc[32];
  __shared__ int s_bi[32];
  const int tid = threadIdx.x;
  if (tid == 0) s_state = *state;
  // weights 1 / (cost + eps) (schedule.cpp:347-351) and the elite: first argmin
  double bc = __longlong_as_double(0x7ff0000000000000LL);
  int bi = n;
  for (int i = tid; i < n; i += kMutThreads) {
    const double c = cost[i];
    cum[i] = 1.0 / __dadd_rn(c, 1e-12);
    if (c < bc) bc = c, bi = i;
  }
  for (int o = 16; o; o >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oc < bc || (oc == bc && oi < bi)) bc = oc, bi = oi;
  }
  if ((tid & 31) == 0) s_bc[tid >> 5] = bc, s_bi[tid >> 5] = bi;
  __syncthreads();
  if (tid < 32) {
    bc = s_bc[tid], bi = s_bi[tid];
    for (int o = 16; o; o >>= 1) {
      const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oc < bc || (oc == bc && oi < bi)) bc = oc, bi = oi;
    }
    if (tid == 0) s_bi[0] = bi;
    // the running total in the reference's order: one dependent DADD chain,
    // operands staged through registers 16 at a time
    if (tid == 0) {
      double t = 0.0;
      int i = 0;
      for (; i + 16 <= n; i += 16) {
        double w[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) w[q] = cum[i + q];
#pragma unroll
        for (int q = 0; q < 16; ++q) t = __dadd_rn(t, w[q]), w[q] = t;
#pragma unroll
        for (int q = 0; q < 16; ++q) cum[i + q] = w[q];
      }
      for (; i < n; ++i) t = __dadd_rn(t, cum[i]), cum[i] = t;
      s_total = t;
    }
  }
  __syncthreads();
  const uint64_t s0 = s_state;
  const double total = s_total;
  const int n_axes = S.n_axes;
  // 1. draw count of a child starting at every offset the chain can reach
  const int n_off = 4 * (n - 1);
  for (int o = tid; o < n_off; o += kMutThreads) {
    const double r = __dmul_rn((double)(draw(s0, (uint64_t)o) >> 11) * 0x1.0p-53, total);
    const int64_t par = upper_bound_d(cum, n, r);
    const int slot = (int)uniform_index(draw(s0, (uint64_t)o + 1), (uint64_t)n_axes + 1);
    int L = 3;
    if (slot != n_axes) {
      const int c0 = slot_col0(S, slot), arity = S.arity[slot];
      uint32_t f[4];
      for (int q = 0; q < arity; ++q) f[q] = (uint32_t)pop[(int64_t)(c0 + q) * n + par];
      int pos;
      int64_t prime;
      L = moves_of(S, slot, f, arity, -1, &pos, &prime) > 0 && arity > 1 ? 4 : 2;
    }
    len[o] = (uint8_t)L;
  }
  __syncthreads();
  // 2. the chain of child start offsets
  if (tid == 0) {
    int o = 0;
    for (int j = 1; j < n; ++j) {
      off[j] = o;
      o += len[o];
    }
    *state = s0 + (uint64_t)o * kGolden;  // RngStream state after mutate()
  }
  __syncthreads();
  // 3. children: elite at 0 (schedule.cpp:368), the rest from their draws
  const int cols = S.cols, ucol = 4 * S.n_sp + 3 * S.n_red;
  const int best = s_bi[0];
  for (int j = tid; j < n; j += kMutThreads) {
    int64_t par = best;
    int slot = -1, from = 0, to = 0, c0 = 0;
    int64_t prime = 1, unroll = 0;
    if (j > 0) {
      const uint64_t o = (uint64_t)off[j];
      const double r = __dmul_rn((double)(draw(s0, o) >> 11) * 0x1.0p-53, total);
      par = upper_bound_d(cum, n, r);
      slot = (int)uniform_index(draw(s0, o + 1), (uint64_t)n_axes + 1);
      if (slot == n_axes) {
        unroll = S.unroll[uniform_index(draw(s0, o + 2), (uint64_t)S.n_unroll)];
      } else {
        c0 = slot_col0(S, slot);
        const int arity = S.arity[slot];
        uint32_t f[4];
        for (int q = 0; q < arity; ++q) f[q] = (uint32_t)pop[(int64_t)(c0 + q) * n + par];
        const int nm = moves_of(S, slot, f, arity, -1, &from, &prime);
        if (nm > 0 && arity > 1) {
          const int m = (int)uniform_index(draw(s0, o + 2), (uint64_t)nm);
          moves_of(S, slot, f, arity, m, &from, &prime);
          to = (int)uniform_index(draw(s0, o + 3), (uint64_t)arity - 1);
          if (to >= from) ++to;
        } else {
          slot = -1;  // nothing movable: the child is the parent
        }
      }
    }
    for (int c = 0; c < cols; ++c) {
      int64_t v = pop[(int64_t)c * n + par];
      if (slot == n_axes && c == ucol) v = unroll;
      if (slot >= 0 && slot < n_axes) {
        if (c == c0 + from) v /= prime;
        if (c == c0 + to) v *= prime;
      }
      next[(int64_t)c * n + j] = (int32_t)v;
    }
  }
}

}  // namespace

size_t mutate_smem_bytes(int64_t n) { return (size_t)n * 8 + (size_t)n * 4 + (size_t)n * 4 + 16; }

int launch_mutate(const DevSketch& S, const int32_t* pop, const double* cost, int64_t n, uint64_t* state,
                  int32_t* next, cudaStream_t st) {
  if (n < 2 || n > kMutateMaxN) return 1;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(k_mutate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mutate_smem_bytes(kMutateMaxN));
    init = true;
  }
  tt::note_launch();
  k_mutate<<<1, kMutThreads, mutate_smem_bytes(n), st>>>(S, pop, cost, (int)n, state, next);
  return 0;
}

}  // namespace tt
