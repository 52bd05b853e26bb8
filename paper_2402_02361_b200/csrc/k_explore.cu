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
//   2. the chain o_1 = 0, o_{j+1} = o_j + L(o_j) over L in shared memory,
//      walked per segment from each of the 4 possible entry offsets, stitched
//      by one thread, then re-walked to write every child's offset;
//   3. a parallel apply pass: child j re-derives its draws at o_j and writes
//      its factors.
// The roulette-wheel prefix sum is one thread's fp64 chain in the reference
// order (the weights are computed in parallel first), so `total` and every
// cumulative bound are the reference's bits. Built with --fmad=false.
//
// One persistent thread-block cluster runs every generation (n <=
// kMutateMaxN): each CTA derives the wheel and the offset chain itself and
// produces a slice of the children with their draft costs; a child's identity
// is its parent's with one mixed-radix digit updated. The population is tiny
// (512 at the TunerConfig defaults) and the generation chain is latency
// bound, so the kernel's job is to remove every host round trip from the loop.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "tt_kernels.h"

namespace tt {

namespace {

constexpr int kMutThreads = 512;
constexpr int kWork = kMutThreads - 32;  // warps 0..14 work; warp 15 publishes generations to the host
constexpr int kMain = 224;               // warps 0..6: this generation's wheel and children
constexpr int kPrep = kWork - kMain;     // warps 7..14: the next generation's offset chain and draws
constexpr int kSegs = 128;               // offset-chain segments
// CTAs of the explore cluster and the children slice of each (rounded up to
// even so the arrays after it stay 8-byte aligned)
__host__ __device__ constexpr int cluster_of(int64_t n) { return n > 448 ? 8 : (int)((n + 63) / 64); }
__host__ __device__ constexpr int explore_per_cap(int64_t n) {
  return (int)(((n + cluster_of(n) - 1) / cluster_of(n) + 1) & ~1LL);
}
constexpr int kMaxCols = 4 * 4 + 3 * 3 + 1;  // 4 spatial x 4 + 3 reduction x 3 + unroll

// clock64 marks of thread 0 at the phase boundaries (ttdbg_mutate_clocks)
// of generation g_mut_gen (ttdbg_mutate_probe)
__device__ long long g_clk_mut[26];
__device__ int g_mut_gen = 1;
// debugging: when set (ttdbg_explore_watch), lane 0 of every warp writes
// (generation << 8 | phase) to its word of this mapped host array as it goes
__device__ unsigned* g_mut_prog = nullptr;
#define MUT_PROG(ph)                                                          \
  do {                                                                        \
    if (prog && (tid & 31) == 0) *(volatile unsigned*)(prog + cr * 16 + (tid >> 5)) = (unsigned)(g << 8 | (ph)); \
  } while (0)
__device__ unsigned long long g_mut_ns[4];  // globaltimer at kernel start / generation 1 start / loop end; clock64 span
#define MUT_MARK_T(i, t)                                            \
  do {                                                              \
    if (tid == (t)) {                                               \
      long long c_;                                                 \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)::"memory"); \
      s_clk[i] = c_;                                                \
    }                                                               \
  } while (0)
#define MUT_MARK(i) MUT_MARK_T(i, 0)

__device__ __forceinline__ int upper_bound_d(const double* cum, int n, double r) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cum[mid] > r) hi = mid; else lo = mid + 1;
  }
  return lo < n - 1 ? lo : n - 1;
}

__device__ __forceinline__ int slot_col0(const DevSketch& S, int slot) {
  return slot < S.n_sp ? 4 * slot : 4 * S.n_sp + 3 * (slot - S.n_sp);
}

// The m-th move of factor tuple f (positions 0..arity-1) in the reference's
// order: position ascending, prime ascending, repeated by multiplicity
// (schedule.cpp:377-381). Only the axis' own primes (t0 .. t0+np-1 of the
// sketch's prime table) can divide its factors. The move count itself is
// Omega(extent) — the factors multiply to the extent — so it needs no pass.
// The sketch's prime table, copied to shared memory once: the apply pass
// indexes it with per-lane (divergent) indices, which the kernel-parameter
// bank would serialise.
struct PrimeTab {
  int32_t p[TT_MAX_PRIMES], e[TT_MAX_PRIMES];
  uint32_t inv[TT_MAX_PRIMES], lim[TT_MAX_PRIMES];
  int32_t arity[TT_MAX_AXES], unroll[TT_MAX_UNROLL];
  int32_t len[TT_MAX_AXES + 1];  // draws a child consumes by slot
};

// f[q] without a dynamic register index (the loops over positions stay loops)
__device__ __forceinline__ uint32_t sel4(const uint32_t (&f)[4], int q) {
  return q == 0 ? f[0] : q == 1 ? f[1] : q == 2 ? f[2] : f[3];
}

__device__ __forceinline__ void pick_move(const PrimeTab& S, int t0, int np, const uint32_t (&f)[4], int arity,
                                          int m, int* pos, int32_t* prime, int* tsel) {
  int cnt = 0;
#pragma unroll 1
  for (int q = 0; q < arity; ++q) {
    uint32_t v = sel4(f, q);
    for (int t = t0; t < t0 + np && v > 1; ++t) {
      int e = 0;
      if (S.p[t] == 2) {
        e = __ffs(v) - 1;
        v >>= e;
      } else {
        for (uint32_t qv = v * S.inv[t]; qv <= S.lim[t]; qv = v * S.inv[t]) v = qv, ++e;
      }
      if (m >= cnt && m < cnt + e) {
        *pos = q, *prime = (int32_t)S.p[t], *tsel = t;
        return;
      }
      cnt += e;
    }
  }
}

__device__ __forceinline__ void named_barrier(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void named_barrier_arrive(int id, int threads) {
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// the non-.aligned form: lanes of one warp may reach it from different code
// (a child loop whose trip count differs across the warp's lanes)
__device__ __forceinline__ void named_barrier_divergent(int id, int threads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// the arity factors of `slot` of population member `par` (SoA, ld n)
__device__ __forceinline__ void load_slot(const int32_t* pop, int n, int c0, int arity, int par,
                                          uint32_t (&f)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) f[q] = q < arity ? (uint32_t)pop[(size_t)(c0 + q) * n + par] : 1u;
}

// Factors of member i (SoA, ld n). The generation slots are rewritten while
// the kernel runs (and by other CTAs of the cluster), so reads are ordinary
// coherent loads (ordered by the cluster barrier's acquire), never the
// non-coherent read-only path: the pointers are deliberately not
// const __restrict__.
template <int NSP, int NRED>
__device__ __forceinline__ void load_factors_cg(const int32_t* soa, int n, int i, Factors<NSP, NRED>& F) {
#pragma unroll
  for (int q = 0; q < Factors<NSP, NRED>::kN; ++q) F.f[q] = soa[(size_t)q * n + i];
  F.unroll = soa[(size_t)Factors<NSP, NRED>::kN * n + i];
}

// exponents of prime table entry t in the arity factors f
__device__ __forceinline__ void exps_of(const PrimeTab& S, int t, const uint32_t (&f)[4], int arity, int (&e)[4]) {
  e[0] = e[1] = e[2] = e[3] = 0;
#pragma unroll 1
  for (int q = 0; q < arity; ++q) {
    uint32_t v = sel4(f, q);
    int x = 0;
    if (S.p[t] == 2) {
      x = __ffs(v) - 1;
    } else {
      for (uint32_t qv = v * S.inv[t]; qv <= S.lim[t]; qv = v * S.inv[t]) v = qv, ++x;
    }
    e[q] = x;
  }
}

struct GenDev {
  int32_t* soa;  // [cols][n]
  double* cost;
  uint64_t* id;
};
struct GenOut {  // pinned host slots: generation g at base + g * stride
  char* base;
  size_t stride, cost_off;
};

// generation g's device slot
__device__ __forceinline__ GenDev gen_dev(const GenOut& d, int g, int n) {
  char* b = d.base + (size_t)g * d.stride;
  GenDev r;
  r.soa = (int32_t*)b;
  r.cost = (double*)(b + d.cost_off);
  r.id = (uint64_t*)(r.cost + n);
  return r;
}

// Writes generation g's member j: factors, cost and identity to its device
// slot (every generation keeps its own). The pinned host mirror is written
// by the publishing warp (publish_slice), so no working thread has a
// system-memory write in flight at a cluster barrier.
template <int NSP, int NRED>
__device__ __forceinline__ void emit(int n, const GenDev& d, int j, const Factors<NSP, NRED>& F, double c, uint64_t id,
                                     bool write_dev_soa) {
  constexpr int kN = Factors<NSP, NRED>::kN;
  if (write_dev_soa) {
#pragma unroll
    for (int q = 0; q < kN; ++q) d.soa[(size_t)q * n + j] = F.f[q];
    d.soa[(size_t)kN * n + j] = F.unroll;
  }
  d.cost[j] = c, d.id[j] = id;
}

// One warp: this CTA's slice [jlo, jhi) of generation g (device slot d,
// written by this CTA before a barrier the warp has passed) copied to the
// pinned host slot, then the slice's system-scope flag. Lane 0's release
// fence is cumulative over the lanes' writes it observed through the
// warp barrier.
__device__ __forceinline__ void publish_slice(const GenOut& h, const GenDev& d, int g, int n, int jlo, int jhi,
                                              volatile uint32_t* flag) {
  const int lane = threadIdx.x & 31;
  char* hb = h.base + (size_t)g * h.stride;
  double* hc = (double*)(hb + h.cost_off);
  uint64_t* hi = (uint64_t*)(hc + n);
  for (int j = jlo + lane; j < jhi; j += 32) hc[j] = d.cost[j], hi[j] = d.id[j];
  __syncwarp();
  if (lane == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    *flag = 1u;
  }
}

// Segment maps of the offset chain: entry e in [0, 4) (offset lo + e) ->
// (exit relative to the next segment's lo, children started inside), four
// 16-bit fields (exit << 14 | count). Composition is associative, so the
// chain's entry into every segment is a scan.
__device__ __forceinline__ uint64_t seg_map(const int32_t* seg_exit, const int32_t* seg_cnt, int s, int W) {
  uint64_t m = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t x = (uint32_t)(seg_exit[4 * s + e] - (s + 1) * W) & 3u;
    m |= (uint64_t)(x << 14 | (uint32_t)seg_cnt[4 * s + e]) << (16 * e);
  }
  return m;
}
__device__ __forceinline__ uint64_t map_compose(uint64_t a, uint64_t b) {  // a, then b
  uint64_t r = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t fa = (uint32_t)(a >> (16 * e)) & 0xffffu;
    const uint32_t fb = (uint32_t)(b >> (16 * (fa >> 14))) & 0xffffu;
    r |= (uint64_t)((fb & 0xc000u) | ((fa & 0x3fffu) + (fb & 0x3fffu))) << (16 * e);
  }
  return r;
}
constexpr uint64_t kMapIdentity = (uint64_t)1 << 30 | (uint64_t)2 << 46 | (uint64_t)3 << 62;

// All generations of one explore in one thread-block cluster (<= 8 CTAs):
// generation 0 is the random_init population already in device slot 0
// (k_generate); generation g >= 1 is mutate(generation g-1) in slot g. Every
// member's draft cost and identity are computed by the thread that produced
// it, and each CTA's slice of a generation is published to pinned host
// memory followed by a system-scope flag (flags[g * clusters + rank]), so the
// host folds the generation into the pool while the device moves on.
//
// Warp roles (the generation chain is latency bound, so the work that does
// not depend on the costs is taken off it):
//   main  (warps 0..6)   weights, the DADD running total (warp 0) while
//                        warps 1..6 stage the parents in shared memory, then
//                        the children of this CTA's slice;
//   prep  (warps 7..14)  the NEXT generation's parent-independent part: the
//                        draw count at every stream offset, the offset chain
//                        (segment walks per entry, a warp scan of the
//                        segment maps, re-walks) and every child's draws;
//   publish (warp 15)    the previous generation's host copy and flag.
template <int NSP, int NRED, bool U32 = false>
__global__ void __launch_bounds__(kMutThreads, 1)
    k_explore_gens(DevSketch S, DevDevice D, int toggles, int n, int n_steps, GenOut dv, uint64_t s_init, GenOut h,
                   volatile uint32_t* flags, int mode) {
  constexpr int kN = Factors<NSP, NRED>::kN;
  extern __shared__ __align__(16) unsigned char smem[];
  const int per_cap = explore_per_cap(n);
  const bool staged = (mode & 1) != 0, spec = (mode & 2) != 0;
  double* cum = (double*)smem;                          // [n] the wheel: running sums in the reference's order
  double* wts = spec ? cum + n : cum;                   // [n] weights (in place without speculation)
  double* cum_sp = spec ? wts + n : nullptr;            // [n] the approximate wheel (parallel scan)
  double* ch_u = cum + (spec ? 3 : 1) * (size_t)n;      // [2][per_cap] roulette uniform of child jlo + c
  int32_t* ch_p = (int32_t*)(ch_u + 2 * per_cap);       // [2][per_cap] slot + 1 | move / unroll draws
  int32_t* off = ch_p + 2 * per_cap;                    // [n] stream offset of child j
  int32_t* seg_exit = off + n;                          // [kSegs][4]
  int32_t* seg_cnt = seg_exit + 4 * kSegs;              // [kSegs][4]
  int32_t* seg_entry = seg_cnt + 4 * kSegs;             // [kSegs]
  int32_t* seg_base = seg_entry + kSegs;                // [kSegs]
  uint8_t* len = (uint8_t*)(seg_base + kSegs);          // [4n] draws a child starting at offset o consumes
  // staged copy of the previous generation (when it fits): parents are read
  // at random by the apply pass, so they come from shared memory
  uint64_t* id_s = (uint64_t*)(len + 4 * (size_t)n);    // [n] (4n is a multiple of 8)
  int32_t* pop_s = (int32_t*)(id_s + n);                // [cols][n]
  __shared__ double s_total, s_total_sp;
  __shared__ int s_best;
  __shared__ int s_t0[TT_MAX_AXES], s_np[TT_MAX_AXES], s_omega[TT_MAX_AXES];
  __shared__ uint64_t s_w[TT_MAX_PRIMES];  // identity weight of each (axis, prime) digit
  __shared__ PrimeTab tab;
  __shared__ double s_bc[kMain / 32];
  __shared__ int s_bi[kMain / 32];
  __shared__ long long s_clk[26];  // phase marks of generation probe_g, written out at the end
  const int tid = threadIdx.x;
  const int n_axes = S.n_axes;
  const int probe_g = g_mut_gen;
  unsigned* const prog = g_mut_prog;
  unsigned long long ns0 = 0;
  long long ck0 = 0;
  if (tid == 0 && blockIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0)::"memory");
    ck0 = clock64();
  }
  // the grid is one thread-block cluster: every CTA derives the generation's
  // wheel and offset chain itself (identical, deterministic) and produces its
  // own slice of the children; generations are separated by cluster barriers
  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  const int nc = (int)gridDim.x, cr = (int)blockIdx.x;
  const int per = (n + nc - 1) / nc, jlo = min(n, cr * per), jhi = min(n, jlo + per);
  if (tid < n_axes) {  // each axis' slice of the prime table and Omega(extent)
    int t0 = 0, np = 0, om = 0;
    for (int t = S.n_prime - 1; t >= 0; --t)
      if (S.pr_axis[t] == tid) t0 = t, ++np, om += S.pr_e[t];
    s_t0[tid] = t0, s_np[tid] = np, s_omega[tid] = om;
  }
  if (tid < S.n_prime) {
    tab.p[tid] = (int32_t)S.pr_p[tid], tab.e[tid] = S.pr_e[tid];
    tab.inv[tid] = S.pr_inv[tid], tab.lim[tid] = S.pr_lim[tid];
  }
  if (tid < TT_MAX_AXES) tab.arity[tid] = S.arity[tid];
  if (tid < TT_MAX_UNROLL) tab.unroll[tid] = (int32_t)S.unroll[tid];
  if (tid <= n_axes)
    tab.len[tid] = tid == n_axes ? 3 : (S.extent[tid] > 1 && S.arity[tid] > 1 ? 4 : 2);
  if (tid == 32) {  // identity = mixed radix (digit per (axis, prime), then the unroll index)
    uint64_t w = (uint64_t)S.n_unroll;
    for (int t = S.n_prime - 1; t >= 0; --t) s_w[t] = w, w *= S.pr_count[t];
  }
  __syncthreads();

  const int n_off = 4 * (n - 1);  // child n-1 starts at offset <= 4(n-2)
  // segment count balancing the walks (~W/2.5 steps) against the scan
  const int segs = min(kSegs, max(1, (int)sqrtf(1.67f * (float)n_off)));
  const int W = (n_off + segs - 1) / segs;
  // The prep team's pass for the generation whose mutate() starts at RNG
  // state sp: its children's draws into ch_*[buf]; returns the state after it.
  auto prep = [&](uint64_t sp, int buf, bool mark) -> uint64_t {
    const int p = tid - kMain;
    if (mark) MUT_MARK_T(15, kMain);
    // A child consumes parent + slot draws, then 1 (unroll) or, for an axis
    // slot, 2 more iff it has a movable prime — and the slot's factors
    // multiply to the axis extent, so that is "extent > 1", independent of
    // the parent. So the draw count at every offset is known up front.
    for (int o = p; o < n_off; o += kPrep)
      len[o] = (uint8_t)tab.len[(int)uniform_index(draw(sp, (uint64_t)o + 1), (uint64_t)n_axes + 1)];
    named_barrier(3, kPrep);
    if (mark) MUT_MARK_T(16, kMain);
    // the chain o_1 = 0, o_{j+1} = o_j + len[o_j]: segment s covers offsets
    // [s W, (s + 1) W) and the chain enters it at one of its first 4 offsets
    // (len <= 4): each (segment, entry) walked by its own thread
    for (int q = p; q < 4 * segs; q += kPrep) {
      const int sg = q >> 2, hi = min(sg * W + W, n_off);
      int o = sg * W + (q & 3), c = 0;
      while (o < hi) o += len[o], ++c;
      seg_exit[q] = o, seg_cnt[q] = c;
    }
    named_barrier(3, kPrep);
    if (mark) MUT_MARK_T(17, kMain);
    if (p < 32) {  // scan of the segment maps: entry offset and first child of every segment
      const int qn = (segs + 31) >> 5, s_lo = min(segs, p * qn), s_hi = min(segs, s_lo + qn);
      uint64_t m = kMapIdentity;
      for (int sg = s_lo; sg < s_hi; ++sg) m = map_compose(m, seg_map(seg_exit, seg_cnt, sg, W));
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, m, d);
        if (p >= d) m = map_compose(o, m);
      }
      uint64_t pre = __shfl_up_sync(0xffffffffu, m, 1);
      if (p == 0) pre = kMapIdentity;
      int e = (int)(pre >> 14) & 3, j = 1 + (int)(pre & 0x3fffu);  // the chain starts at offset 0, child 1
      for (int sg = s_lo; sg < s_hi; ++sg) {
        seg_entry[sg] = sg * W + e, seg_base[sg] = j;
        const uint32_t f = (uint32_t)(seg_map(seg_exit, seg_cnt, sg, W) >> (16 * e)) & 0xffffu;
        e = (int)(f >> 14), j += (int)(f & 0x3fffu);
      }
    }
    named_barrier(3, kPrep);
    if (mark) MUT_MARK_T(18, kMain);
    // every segment re-walked from its entry to place its children's offsets
    for (int sg = p; sg < segs; sg += kPrep) {
      const int hi = min(sg * W + W, n_off);
      int o = seg_entry[sg], j = seg_base[sg];
      while (o < hi && j < n) off[j] = o, o += len[o], ++j;
    }
    named_barrier(3, kPrep);
    if (mark) MUT_MARK_T(19, kMain);
    // the parent-independent draws of this CTA's children: the roulette
    // uniform, the slot and the move / unroll draws
    for (int j = jlo + p; j < jhi; j += kPrep) {
      if (j == 0) continue;
      const uint64_t o = (uint64_t)off[j];
      ch_u[buf * per_cap + j - jlo] = (double)(draw(sp, o) >> 11) * 0x1.0p-53;
      const int slot = (int)uniform_index(draw(sp, o + 1), (uint64_t)n_axes + 1);
      int pk = 0;  // slot + 1, 0 = nothing movable (the child is the parent)
      if (slot == n_axes) {
        pk = (slot + 1) | (int)uniform_index(draw(sp, o + 2), (uint64_t)S.n_unroll) << 8;
      } else if (s_omega[slot] > 0 && tab.arity[slot] > 1) {
        const int m = (int)uniform_index(draw(sp, o + 2), (uint64_t)s_omega[slot]);
        const int to = (int)uniform_index(draw(sp, o + 3), (uint64_t)tab.arity[slot] - 1);
        pk = (slot + 1) | m << 8 | to << 24;
      }
      ch_p[buf * per_cap + j - jlo] = pk;
    }
    const int last = off[n - 1];
    const uint64_t nx = sp + (uint64_t)(last + len[last]) * kGolden;  // RngStream state after mutate()
    named_barrier(3, kPrep);  // off / len read before the next pass rewrites them
    if (mark) MUT_MARK_T(20, kMain);
    return nx;
  };

  // generation 0: cost the random_init population; the prep team prepares
  // generation 1 meanwhile
  uint64_t s_prep = s_init;
  if (tid < kMain) {
    const GenDev d0 = gen_dev(dv, 0, n);
    for (int j = jlo + tid; j < jhi; j += kMain) {
      Factors<NSP, NRED> F;
      load_factors_cg<NSP, NRED>(d0.soa, n, j, F);
      emit<NSP, NRED>(n, d0, j, F, draft_cost_of<NSP, NRED, false, std::conditional_t<U32, uint32_t, int64_t>>(S, D, F, toggles), d0.id[j], false);
    }
  } else if (tid < kWork && n_steps > 1) {
    s_prep = prep(s_prep, 1, false);
  }
  cluster.sync();
  if (tid == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    g_mut_ns[1] = t - ns0;
  }
  for (int g = 1; g < n_steps; ++g) {
    const GenDev prev = gen_dev(dv, g - 1, n);
    if (g == probe_g) MUT_MARK(0);
    MUT_PROG(1);
    if (tid >= kWork) {
      // warp 15 publishes the previous generation (this CTA's slice) to the
      // host while the others build this one: the system fence waits for the
      // host writes' PCIe completions, so no working warp carries them
      publish_slice(h, prev, g - 1, n, jlo, jhi, flags + (g - 1) * nc + cr);
    } else if (tid >= kMain) {
      if (g + 1 < n_steps) s_prep = prep(s_prep, (g + 1) & 1, g == probe_g);
    } else {
      const GenDev cur = gen_dev(dv, g, n);
      const int32_t* pop = staged ? pop_s : prev.soa;
      const uint64_t* pid = staged ? id_s : prev.id;
      // A. weights 1 / (cost + eps) (schedule.cpp:347-351) and the elite
      // (first argmin, :360-362)
      double bc = __longlong_as_double(0x7ff0000000000000LL);
      int bi = n;
      for (int i = tid; i < n; i += kMain) {
        const double c = prev.cost[i];
        wts[i] = 1.0 / __dadd_rn(c, 1e-12);
        if (c < bc) bc = c, bi = i;
      }
      for (int o = 16; o; o >>= 1) {
        const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oc < bc || (oc == bc && oi < bi)) bc = oc, bi = oi;
      }
      if ((tid & 31) == 0) s_bc[tid >> 5] = bc, s_bi[tid >> 5] = bi;
      if (g == probe_g) MUT_MARK(14);
      MUT_PROG(2);
      named_barrier(2, kMain);
      MUT_PROG(3);
      // B. warp 0: the running total in the reference's order — one
      // dependent DADD chain (~12 cycles a step) — then it releases barrier 4.
      // The children do not wait for it: warp 6 builds an approximate wheel
      // (a parallel scan: the same sums in another order, a few ulps off),
      // warps 1..5 stage the parents, and warps 1..6 build every child from
      // the parent the approximate wheel picks. Once the exact wheel is out
      // each child checks its draw against it and is rebuilt in the rare
      // case the draw fell between the two wheels' bounds.
      if (tid < 32) {
        if (tid == 0) {
          double t = 0.0;
          int i = 0;
          for (; i + 16 <= n; i += 16) {
            double w[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) w[q] = wts[i + q];
#pragma unroll
            for (int q = 0; q < 16; ++q) t = __dadd_rn(t, w[q]), w[q] = t;
#pragma unroll
            for (int q = 0; q < 16; ++q) cum[i + q] = w[q];
          }
          for (; i < n; ++i) t = __dadd_rn(t, wts[i]), cum[i] = t;
          s_total = t;
          if (g == probe_g) MUT_MARK(22);
        }
        __syncwarp();
        named_barrier_arrive(4, kMain);
      } else {
        if (tid >= kMain - 32) {  // warp 6: the elite and the approximate wheel
          const int l = tid & 31;
          bc = l < kMain / 32 ? s_bc[l] : __longlong_as_double(0x7ff0000000000000LL);
          bi = l < kMain / 32 ? s_bi[l] : n;
          for (int o = 16; o; o >>= 1) {
            const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oc < bc || (oc == bc && oi < bi)) bc = oc, bi = oi;
          }
          if (spec) {
            const int ch = (n + 31) >> 5, i0 = min(n, l * ch), i1 = min(n, i0 + ch);
            double t = 0.0;
            for (int i = i0; i < i1; ++i) t += wts[i];
            double incl = t;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const double o = __shfl_up_sync(0xffffffffu, incl, d);
              if (l >= d) incl += o;
            }
            t = incl - t;  // exclusive prefix
            for (int i = i0; i < i1; ++i) t += wts[i], cum_sp[i] = t;
            if (l == 31) s_total_sp = incl;
          }
          if (l == 0) s_best = bi;
        } else if (staged) {  // warps 1..5: the parents into shared memory
          // async copies, all in flight at once, no register staging; every
          // generation has its own device slot, so no stale L1 line can hit
          const int nt = kMain - 64, t = tid - 32;
          const uint32_t sp = (uint32_t)__cvta_generic_to_shared(pop_s);
          const uint32_t si = (uint32_t)__cvta_generic_to_shared(id_s);
          for (int i = t; i < (kN + 1) * n; i += nt)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sp + 4u * i), "l"(prev.soa + i) : "memory");
          for (int i = t; i < n; i += nt)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(si + 8u * i), "l"(prev.id + i) : "memory");
          asm volatile("cp.async.wait_all;" ::: "memory");
          if (g == probe_g) MUT_MARK_T(21, 32);
        }
        MUT_PROG(4);
        named_barrier(5, kMain - 32);
        MUT_PROG(5);
        if (g == probe_g) MUT_MARK_T(3, 32);
        // D. children: elite at 0 (schedule.cpp:368), the rest from their draws
        const double* cu = ch_u + (g & 1) * per_cap;
        const int32_t* cpk = ch_p + (g & 1) * per_cap;
        const int best = s_best;
        // child j from parent par (factors, identity, draft cost)
        auto build = [&](int j, int par, Factors<NSP, NRED>& F, uint64_t& id_j) -> double {
          const int pk = j > 0 ? cpk[j - jlo] : 0;
          const int slot = (pk & 0xff) - 1;
          // all columns loaded before any store: one round trip per child
          load_factors_cg<NSP, NRED>(pop, n, par, F);
          id_j = pid[par];
          int c_from = -1, c_to = -1;
          uint32_t v_from = 0, v_to = 0;
          if (slot == n_axes) {  // the unroll digit
            const int uidx = pk >> 8;
            int uold = 0;
#pragma unroll 1
            for (int u = 0; u < S.n_unroll; ++u)
              if (tab.unroll[u] == F.unroll) uold = u;
            id_j += (uint64_t)uidx - (uint64_t)uold;
            F.unroll = tab.unroll[uidx];
          } else if (slot >= 0) {  // a prime moved between two positions of the slot
            const int c0 = slot_col0(S, slot), arity = tab.arity[slot];
            uint32_t f[4] = {1u, 1u, 1u, 1u};
            load_slot(pop, n, c0, arity, par, f);
            int from = 0, tsel = 0;
            int32_t prime = 1;
            pick_move(tab, s_t0[slot], s_np[slot], f, arity, (pk >> 8) & 0xffff, &from, &prime, &tsel);
            int to = pk >> 24;
            if (to >= from) ++to;
            int e[4];
            exps_of(tab, tsel, f, arity, e);
            const int d_old = rank_composition_cf(tab.e[tsel], arity, e);
            e[from] -= 1, e[to] += 1;
            const int d_new = rank_composition_cf(tab.e[tsel], arity, e);
            id_j += (uint64_t)(int64_t)(d_new - d_old) * s_w[tsel];
            c_from = c0 + from, c_to = c0 + to;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (q == from) v_from = f[q];
              if (q == to) v_to = f[q];
            }
            v_from /= (uint32_t)prime, v_to *= (uint32_t)prime;
          }
#pragma unroll
          for (int q = 0; q < kN; ++q) F.f[q] = q == c_from ? (int32_t)v_from : q == c_to ? (int32_t)v_to : F.f[q];
          return draft_cost_of<NSP, NRED, !U32, std::conditional_t<U32, uint32_t, int64_t>>(S, D, F, toggles);
        };
        bool exact = !spec;  // past barrier 4: the exact wheel is in cum / s_total
        if (exact) named_barrier(4, kMain);
        for (int j = jlo + tid - 32; j < jhi; j += kMain - 32) {
          const double u = j > 0 ? cu[j - jlo] : 0.0;
          int par = best;
          if (j > 0) par = exact ? upper_bound_d(cum, n, __dmul_rn(u, s_total))
                                 : upper_bound_d(cum_sp, n, __dmul_rn(u, s_total_sp));
          if (g == probe_g) MUT_MARK_T(12, 32);
          Factors<NSP, NRED> F;
          uint64_t id_j;
          double c_j;
          for (;;) {  // one pass, two when the approximate wheel picked another parent
            c_j = build(j, par, F, id_j);
            if (exact) break;
            if (g == probe_g) MUT_MARK_T(6, 32);
            MUT_PROG(6);
            named_barrier_divergent(4, kMain);
            MUT_PROG(7);
            exact = true;
            if (g == probe_g) MUT_MARK_T(8, 32);
            if (j == 0) break;
            const double r = __dmul_rn(u, s_total);  // upper_bound_d's answer is par iff
            if ((par == 0 || cum[par - 1] <= r) && (par == n - 1 || cum[par] > r)) break;
            par = upper_bound_d(cum, n, r);
          }
          emit<NSP, NRED>(n, cur, j, F, c_j, id_j, true);
        }
        MUT_PROG(8);
        if (!exact) named_barrier_divergent(4, kMain);
        MUT_PROG(9);
        if (g == probe_g) MUT_MARK_T(4, 32);
      }
    }
    if (g == probe_g) MUT_MARK(10);
    MUT_PROG(10);
    cluster.sync();  // generation g complete in every CTA before anyone reads it
    if (g == probe_g) MUT_MARK(11);
  }
  // the last generation (every earlier one was published by warp 15)
  __syncthreads();
  if (tid >= kWork) publish_slice(h, gen_dev(dv, n_steps - 1, n), n_steps - 1, n, jlo, jhi, flags + (n_steps - 1) * nc + cr);
  if (cr == 0 && tid < 26 && probe_g < n_steps) g_clk_mut[tid] = s_clk[tid];
  if (tid == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    g_mut_ns[2] = t - ns0, g_mut_ns[3] = (unsigned long long)(clock64() - ck0);
  }
}

}  // namespace

size_t mutate_smem_bytes(int64_t n, int cols, bool staged, bool spec) {
  return (size_t)n * (spec ? 32 : 16) + (size_t)kSegs * 10 * 4 + (size_t)explore_per_cap(n) * 24 +
         (staged ? (size_t)n * (8 + 4 * (size_t)cols) : 0) + 16;
}
constexpr size_t kSmemCap = 220 * 1024;

int launch_explore_gens(const DevSketch& S, const DevDevice& D, int toggles, int64_t n, int n_steps,
                        void* dev_base, size_t dev_stride, size_t dev_cost_off, uint64_t s_init, void* host_base, size_t host_stride, size_t host_cost_off,
                        volatile uint32_t* flags, cudaStream_t st) {
  if (n < 2 || n > kMutateMaxN) return 1;
  GenOut dv{(char*)dev_base, dev_stride, dev_cost_off};
  GenOut h{(char*)host_base, host_stride, host_cost_off};
  // staged parents and the speculative wheel when they fit, in that order
  int mode = 0;
  for (int m : {3, 1, 2, 0})
    if (mutate_smem_bytes(n, S.cols, m & 1, m & 2) <= kSmemCap) {
      mode = m;
      break;
    }
  const size_t sm = mutate_smem_bytes(n, S.cols, mode & 1, mode & 2);
  cudaError_t err = cudaSuccess;
  const int rc = TT_DISPATCH_SHAPE(S.n_sp, S.n_red, ({
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(k_explore_gens<NSP, NRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
      cudaFuncSetAttribute(k_explore_gens<NSP, NRED, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
      init = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(explore_cluster_size(n));
    cfg.blockDim = dim3(kMutThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = explore_cluster_size(n), at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
    cfg.attrs = at, cfg.numAttrs = 1;
    tt::note_launch();
    // the 32-bit draft-cost mode (uint32 products, branch-free divisions)
    // when the sketch and device allow it, as in the round's selector
    if (fits_u32(S, D))
      err = cudaLaunchKernelEx(&cfg, k_explore_gens<NSP, NRED, true>, S, D, toggles, (int)n, n_steps, dv, s_init, h,
                               flags, mode);
    else
      err = cudaLaunchKernelEx(&cfg, k_explore_gens<NSP, NRED>, S, D, toggles, (int)n, n_steps, dv, s_init, h, flags,
                               mode);
  }));
  return rc ? rc : (err != cudaSuccess ? 2 : 0);
}

int explore_cluster_size(int64_t n) { return cluster_of(n); }

}  // namespace tt

extern "C" int ttdbg_mutate_clocks(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_clk_mut, sizeof(long long) * (n < 26 ? n : 26));
}
extern "C" int ttdbg_mutate_ns(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_mut_ns, sizeof(unsigned long long) * 4);
}
extern "C" int ttdbg_mutate_watch(unsigned* mapped) {
  return (int)cudaMemcpyToSymbol(tt::g_mut_prog, &mapped, sizeof(mapped));
}
extern "C" int ttdbg_mutate_probe(int g) { return (int)cudaMemcpyToSymbol(tt::g_mut_gen, &g, sizeof(int)); }
