// tt_block.cuh — CTA-wide primitives staged in shared memory: bitonic sort
// of (key1, key2, payload) triples and an exclusive scan. Used by the
// draft top-K finalisation, the cross-rank merge and select_top.
#pragma once

#include <cstdint>

namespace tt {

// Ascending lexicographic (a, b[, c]) bitonic sort of n = 2^m entries, all
// in shared memory, executed by the whole CTA. With KEY3 = false, c is a
// payload carried along.
template <bool KEY3 = false>
__device__ __forceinline__ void block_bitonic_sort(uint64_t* a, uint64_t* b, uint64_t* c, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t a0 = a[lo], a1 = a[hi], b0 = b[lo], b1 = b[hi];
        const uint64_t c0 = c[lo], c1 = c[hi];
        bool gt = a0 > a1 || (a0 == a1 && b0 > b1);
        bool lt = a0 < a1 || (a0 == a1 && b0 < b1);
        if (KEY3 && a0 == a1 && b0 == b1) gt = c0 > c1, lt = c0 < c1;
        if (up ? gt : lt) {
          a[lo] = a1, a[hi] = a0;
          b[lo] = b1, b[hi] = b0;
          c[lo] = c1, c[hi] = c0;
        }
      }
    }
  }
  __syncthreads();
}

// Exclusive prefix sum over flags[0..n) (n <= 32 * blockDim, values small),
// result in out[0..n) and the total returned to every thread. `warp_tot`
// needs 32 ints of shared memory.
__device__ __forceinline__ int block_exclusive_scan(const int* flags, int* out, int n, int* warp_tot) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int beg = threadIdx.x * per;
  int local = 0;
  for (int q = 0; q < per; ++q)
    if (beg + q < n) local += flags[beg + q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    int v = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v += u;
    }
    if (lane < nw) warp_tot[lane] = v;  // inclusive warp prefix
  }
  __syncthreads();
  int run = (warp ? warp_tot[warp - 1] : 0) + incl - local;
  for (int q = 0; q < per; ++q)
    if (beg + q < n) {
      out[beg + q] = run;
      run += flags[beg + q];
    }
  const int nw = (blockDim.x + 31) >> 5;
  const int total = warp_tot[nw - 1];
  __syncthreads();
  return total;
}

// ---- register/shuffle bitonic sort -------------------------------------
// Every thread holds E keys at positions p = e * NT + t (NT = blockDim.x, a
// multiple of 32). Exchanges with partner p ^ stride run in registers when
// stride >= NT, through warp shuffles when stride < 32, and through shared
// memory otherwise — so most of the log^2 n stages never touch shared
// memory. Keys must be strictly ordered (the callers append a unique index).
// The comparators are written branch-free: with the short-circuit form,
// ptxas 12.9 -O3 produced a network that duplicated tied-prefix keys at
// 1024 threads under register pressure (tools/dbg_sort.cu reproduces it;
// -Xptxas -O0 and the branch-free form both sort correctly).
struct Key2 {  // (a, b) lexicographic
  uint64_t a, b;
  __host__ __device__ __forceinline__ bool lt(const Key2& o) const {
    const bool alt = a < o.a, aeq = a == o.a, blt = b < o.b;
    return alt | (aeq & blt);
  }
  __device__ __forceinline__ Key2 shfl_xor(int m) const {
    Key2 r;
    r.a = __shfl_xor_sync(0xffffffffu, a, m);
    r.b = __shfl_xor_sync(0xffffffffu, b, m);
    return r;
  }
};

struct Key3 {  // (a, b, c) lexicographic
  uint64_t a, b;
  uint32_t c;
  __host__ __device__ __forceinline__ bool lt(const Key3& o) const {
    // branch-free form (see block_sort_reg note on ptxas)
    const bool alt = a < o.a, aeq = a == o.a, blt = b < o.b, beq = b == o.b, clt = c < o.c;
    return alt | (aeq & (blt | (beq & clt)));
  }
  __device__ __forceinline__ Key3 shfl_xor(int m) const {
    Key3 r;
    r.a = __shfl_xor_sync(0xffffffffu, a, m);
    r.b = __shfl_xor_sync(0xffffffffu, b, m);
    r.c = __shfl_xor_sync(0xffffffffu, c, m);
    return r;
  }
};

// Sorts the n = E * blockDim.x keys ascending; `xchg` = shared scratch of n keys.
template <int E, typename K>
__device__ __forceinline__ void block_sort_reg(K (&k)[E], K* xchg) {
  const int NT = blockDim.x;
  const int t = threadIdx.x;
  const int n = E * NT;
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= NT) {
        // in-register stage; ES is a compile-time constant in every branch so
        // k[] stays in registers (a runtime register index would spill it)
        const int es = stride / NT;
#pragma unroll
        for (int ES = 1; ES < E; ES <<= 1) {
          if (es == ES) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const int f = e ^ ES;
              if (f > e) {
                const int p = e * NT + t;
                const bool up = (p & size) == 0;
                const bool sw = up ? k[f].lt(k[e]) : k[e].lt(k[f]);
                if (sw) {
                  const K tmp = k[e];
                  k[e] = k[f];
                  k[f] = tmp;
                }
              }
            }
          }
        }
      } else if (stride >= 32) {
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) xchg[e * NT + t] = k[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int p = e * NT + t;
          const K o = xchg[p ^ stride];
          const bool lower = (p & stride) == 0, up = (p & size) == 0;
          const bool take = (lower == up) ? o.lt(k[e]) : k[e].lt(o);
          if (take) k[e] = o;
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int p = e * NT + t;
          const K o = k[e].shfl_xor(stride);
          const bool lower = (p & stride) == 0, up = (p & size) == 0;
          const bool take = (lower == up) ? o.lt(k[e]) : k[e].lt(o);
          if (take) k[e] = o;
        }
      }
    }
  }
  __syncthreads();
}

__host__ __device__ __forceinline__ int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace tt
