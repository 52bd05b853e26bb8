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

#include "tt_kernels.h"

namespace tt {

namespace {

constexpr int kMutThreads = 512;
constexpr int kSegs = 128;  // offset-chain segments (stitched by one thread)
constexpr int kMaxCols = 4 * 4 + 3 * 3 + 1;  // 4 spatial x 4 + 3 reduction x 3 + unroll

// clock64 marks of thread 0 at the phase boundaries (ttdbg_mutate_clocks)
__device__ long long g_clk_mut[8];
#define MUT_MARK(i)                          \
  do {                                       \
    if (tid == 0 && blockIdx.x == 0) g_clk_mut[i] = clock64(); \
  } while (0)

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

__device__ __forceinline__ void pick_move(const PrimeTab& S, int t0, int np, const uint32_t (&f)[4], int arity,
                                          int m, int* pos, int32_t* prime, int* tsel) {
  int cnt = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q >= arity) break;
    uint32_t v = f[q];
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
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t v = f[q];
    int x = 0;
    if (q < arity) {
      if (S.p[t] == 2) {
        x = __ffs(v) - 1;
      } else {
        for (uint32_t qv = v * S.inv[t]; qv <= S.lim[t]; qv = v * S.inv[t]) v = qv, ++x;
      }
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

// every thread's host writes, then one system-scope flag per generation:
// the CTA barrier orders the block's writes before thread 0's fence, and the
// (cumulative) fence orders them before the flag, as in a grid barrier
__device__ __forceinline__ void publish(volatile uint32_t* flags, int g) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    flags[g] = 1u;
  }
}

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
// slot (every generation keeps its own), cost and identity to the pinned
// host mirror the pool is built from.
template <int NSP, int NRED>
__device__ __forceinline__ void emit(const GenOut& h, int g, int n, const GenDev& d, int j, const Factors<NSP, NRED>& F,
                                     double c, uint64_t id, bool write_dev_soa) {
  constexpr int kN = Factors<NSP, NRED>::kN;
  char* hb = h.base + (size_t)g * h.stride;
  double* hc = (double*)(hb + h.cost_off);
  uint64_t* hi = (uint64_t*)(hc + n);
  if (write_dev_soa) {
#pragma unroll
    for (int q = 0; q < kN; ++q) d.soa[(size_t)q * n + j] = F.f[q];
    d.soa[(size_t)kN * n + j] = F.unroll;
  }
  d.cost[j] = c, d.id[j] = id;
  hc[j] = c, hi[j] = id;
}

// All generations of one explore in one thread-block cluster (<= 8 CTAs):
// generation 0 is the random_init
// population already in slot 0 (k_generate); generation g >= 1 is
// mutate(generation g-1) written into slot g & 1. Every member's draft cost
// and identity are computed by the thread that produced it, and each CTA's
// slice of a generation is published to pinned host memory followed by a
// system-scope flag (flags[g * clusters + rank]), so the host folds the
// generation into the pool while the device moves on.
template <int NSP, int NRED>
__global__ void __launch_bounds__(kMutThreads, 1)
    k_explore_gens(DevSketch S, DevDevice D, int toggles, int n, int n_steps, GenOut dv, uint64_t s_init,
                   GenOut h, volatile uint32_t* flags, int staged) {
  constexpr int kN = Factors<NSP, NRED>::kN;
  extern __shared__ __align__(16) unsigned char smem[];
  double* cum = (double*)smem;        // [n] weights, then their running sums
  int32_t* off = (int32_t*)(cum + n);  // [n] stream offset of child j
  uint8_t* len = (uint8_t*)(off + n);  // [4n] draws a child starting at offset o consumes
  int32_t* seg_exit = (int32_t*)(len + 4 * (size_t)n);  // [kSegs][4]
  int32_t* seg_cnt = seg_exit + 4 * kSegs;              // [kSegs][4]
  int32_t* seg_entry = seg_cnt + 4 * kSegs;             // [kSegs]
  int32_t* seg_base = seg_entry + kSegs;                // [kSegs]
  // staged copy of the previous generation (when it fits): parents are read
  // at random by the apply pass, so they come from shared memory
  uint64_t* id_s = (uint64_t*)(seg_base + kSegs);  // [n]
  int32_t* pop_s = (int32_t*)(id_s + n);            // [cols][n]
  __shared__ double s_total;
  __shared__ uint64_t s_state;
  __shared__ int s_t0[TT_MAX_AXES], s_np[TT_MAX_AXES], s_omega[TT_MAX_AXES];
  __shared__ uint64_t s_w[TT_MAX_PRIMES];  // identity weight of each (axis, prime) digit
  __shared__ PrimeTab tab;
  __shared__ double s_bc[kMutThreads / 32];
  __shared__ int s_bi[kMutThreads / 32];
  const int tid = threadIdx.x;
  const int n_axes = S.n_axes;
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
  // generation 0: cost the random_init population
  for (int j = jlo + tid; j < jhi; j += kMutThreads) {
    Factors<NSP, NRED> F;
    const GenDev d0 = gen_dev(dv, 0, n);
    load_factors_cg<NSP, NRED>(d0.soa, n, j, F);
    emit<NSP, NRED>(h, 0, n, d0, j, F, draft_cost_of<NSP, NRED>(S, D, F, toggles), d0.id[j], false);
  }
  publish(flags, cr);
  cluster.sync();
  uint64_t s0 = s_init;
  const int n_off = 4 * (n - 1);  // child n-1 starts at offset <= 4(n-2)
  for (int g = 1; g < n_steps; ++g) {
  const GenDev prev = gen_dev(dv, g - 1, n);
  const GenDev cur = gen_dev(dv, g, n);
  const double* cost = prev.cost;
  if (g == 1) MUT_MARK(0);
  if (staged) {
    for (int i = tid; i < (kN + 1) * n; i += kMutThreads) pop_s[i] = prev.soa[i];
    for (int i = tid; i < n; i += kMutThreads) id_s[i] = prev.id[i];
  }
  const int32_t* pop = staged ? pop_s : prev.soa;
  const uint64_t* pid = staged ? id_s : prev.id;
  // A. weights 1 / (cost + eps) (schedule.cpp:347-351), the elite (first
  // argmin, :360-362) and the draw count of a child starting at every offset.
  // A child consumes parent + slot draws, then 1 (unroll) or, for an axis
  // slot, 2 more iff it has a movable prime — and the slot's factors multiply
  // to the axis extent, so that is "extent > 1", independent of the parent.
  double bc = __longlong_as_double(0x7ff0000000000000LL);
  int bi = n;
  for (int i = tid; i < n; i += kMutThreads) {
    const double c = cost[i];
    cum[i] = 1.0 / __dadd_rn(c, 1e-12);
    if (c < bc) bc = c, bi = i;
  }
  for (int o = tid; o < n_off; o += kMutThreads) {
    const int slot = (int)uniform_index(draw(s0, (uint64_t)o + 1), (uint64_t)n_axes + 1);
    len[o] = (uint8_t)tab.len[slot];
  }
  for (int o = 16; o; o >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oc < bc || (oc == bc && oi < bi)) bc = oc, bi = oi;
  }
  if ((tid & 31) == 0) s_bc[tid >> 5] = bc, s_bi[tid >> 5] = bi;
  __syncthreads();
  if (g == 1) MUT_MARK(1);
  // B. warp 0: the elite, then the running total in the reference's order
  // (one dependent DADD chain, operands staged through registers).
  // Meanwhile the other warps build the chain of child start offsets
  // o_1 = 0, o_{j+1} = o_j + len[o_j]: segment s covers offsets
  // [s*W, (s+1)*W) and the chain enters it at one of its first 4 offsets
  // (len <= 4), so each segment is walked from all 4 entries (exit, child
  // count), one thread stitches the true entries, and every segment is
  // re-walked from its entry to write the offsets.
  // segment count balancing the walks (~5W/3 steps) against the stitch (segs steps)
  const int segs = min(kSegs, max(1, (int)sqrtf(1.67f * (float)n_off)));
  const int W = (n_off + segs - 1) / segs;
  if (tid < 32) {
    bc = tid < kMutThreads / 32 ? s_bc[tid] : __longlong_as_double(0x7ff0000000000000LL);
    bi = tid < kMutThreads / 32 ? s_bi[tid] : n;
    for (int o = 16; o; o >>= 1) {
      const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (oc < bc || (oc == bc && oi < bi)) bc = oc, bi = oi;
    }
    if (tid == 0) {
      s_bi[0] = bi;
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
  } else {
    // warps 1..: the offset chain, synchronised among themselves only, so
    // it runs under warp 0's DADD chain
    const int sg = tid - 32;
    if (sg < segs) {
      const int lo = sg * W, hi = min(lo + W, n_off);
      for (int e = 0; e < 4; ++e) {
        int o = lo + e, c = 0;
        while (o < hi) o += len[o], ++c;
        seg_exit[sg * 4 + e] = o, seg_cnt[sg * 4 + e] = c;
      }
    }
    named_barrier(1, kMutThreads - 32);
    // stitch: the true entry offset and first child of every segment
    if (sg == 0) {
      int o = 0, j = 1;
      for (int g = 0; g < segs; ++g) {
        seg_entry[g] = o, seg_base[g] = j;
        const int lo = g * W;
        if (o < lo + W && lo < n_off) {
          const int e = o - lo;
          j += seg_cnt[g * 4 + e];
          o = seg_exit[g * 4 + e];
        }
      }
    }
    named_barrier(1, kMutThreads - 32);
    // every segment re-walked from its entry to place its children's offsets
    if (sg < segs) {
      const int hi = min(sg * W + W, n_off);
      int o = seg_entry[sg], j = seg_base[sg];
      while (o < hi && j < n) off[j] = o, o += len[o], ++j;
    }
  }
  __syncthreads();
  if (g == 1) MUT_MARK(2);
  if (g == 1) MUT_MARK(3);
  if (tid == 0) {
    const int last = off[n - 1];
    s_state = s0 + (uint64_t)(last + len[last]) * kGolden;  // RngStream state after mutate()
  }
  // D. children: elite at 0 (schedule.cpp:368), the rest from their draws
  const double total = s_total;
  const int best = s_bi[0];
  for (int j = jlo + tid; j < jhi; j += kMutThreads) {
    int par = best;
    int slot = -1, from = 0, to = 0, c0 = 0, tsel = 0, uidx = 0;
    int32_t prime = 1, unroll = 0;
    uint32_t f[4] = {1u, 1u, 1u, 1u};
    if (j > 0) {
      const uint64_t o = (uint64_t)off[j];
      const double r = __dmul_rn((double)(draw(s0, o) >> 11) * 0x1.0p-53, total);
      par = upper_bound_d(cum, n, r);
      slot = (int)uniform_index(draw(s0, o + 1), (uint64_t)n_axes + 1);
      if (slot == n_axes) {
        uidx = (int)uniform_index(draw(s0, o + 2), (uint64_t)S.n_unroll);
        unroll = tab.unroll[uidx];
      } else {
        c0 = slot_col0(S, slot);
        const int arity = tab.arity[slot];
        const int nm = s_omega[slot];
        if (nm > 0 && arity > 1) {
          load_slot(pop, n, c0, arity, par, f);
          const int m = (int)uniform_index(draw(s0, o + 2), (uint64_t)nm);
          pick_move(tab, s_t0[slot], s_np[slot], f, arity, m, &from, &prime, &tsel);
          to = (int)uniform_index(draw(s0, o + 3), (uint64_t)arity - 1);
          if (to >= from) ++to;
        } else {
          slot = -1;  // nothing movable: the child is the parent
        }
      }
    }
    const bool mv = slot >= 0 && slot < n_axes;
    const int c_from = mv ? c0 + from : -1, c_to = mv ? c0 + to : -1, c_un = slot == n_axes ? kN : -1;
    // all columns loaded before any store: one L2 round trip per child
    Factors<NSP, NRED> F;
    load_factors_cg<NSP, NRED>(pop, n, par, F);
    // the child's identity from its parent's: one digit changes (the moved
    // prime's exponent composition, or the unroll index)
    uint64_t id_j = pid[par];
    if (c_un == kN) {
      int uold = 0;
      for (int u = 0; u < S.n_unroll; ++u)
        if (tab.unroll[u] == F.unroll) uold = u;
      id_j += (uint64_t)uidx - (uint64_t)uold;
    } else if (mv) {
      const int arity = tab.arity[slot];
      int e[4];
      exps_of(tab, tsel, f, arity, e);
      const uint64_t d_old = rank_composition(tab.e[tsel], arity, e);
      e[from] -= 1, e[to] += 1;
      const uint64_t d_new = rank_composition(tab.e[tsel], arity, e);
      id_j += (d_new - d_old) * s_w[tsel];
    }
    if (c_un == kN) F.unroll = unroll;
#pragma unroll
    for (int q = 0; q < kN; ++q) {
      if (q == c_from) F.f[q] /= prime;
      if (q == c_to) F.f[q] *= prime;
    }
    if (g == 1) MUT_MARK(5);
    const double c_j = draft_cost_of<NSP, NRED>(S, D, F, toggles);
    if (g == 1 && c_j > 0) MUT_MARK(6);
    if (g == 1 && id_j != 1) MUT_MARK(7);
    emit<NSP, NRED>(h, g, n, cur, j, F, c_j, id_j, true);
  }
  if (g == 1) MUT_MARK(4);
  publish(flags, g * nc + cr);
  cluster.sync();  // generation g complete in every CTA before anyone reads it
  s0 = s_state;
  }
}

}  // namespace

size_t mutate_smem_bytes(int64_t n, int cols, bool staged) {
  return (size_t)n * 16 + (size_t)kSegs * 10 * 4 + (staged ? (size_t)n * (8 + 4 * (size_t)cols) : 0) + 16;
}
constexpr size_t kSmemCap = 220 * 1024;

int launch_explore_gens(const DevSketch& S, const DevDevice& D, int toggles, int64_t n, int n_steps,
                        void* dev_base, size_t dev_stride, size_t dev_cost_off, uint64_t s_init, void* host_base, size_t host_stride, size_t host_cost_off,
                        volatile uint32_t* flags, cudaStream_t st) {
  if (n < 2 || n > kMutateMaxN) return 1;
  GenOut dv{(char*)dev_base, dev_stride, dev_cost_off};
  GenOut h{(char*)host_base, host_stride, host_cost_off};
  const bool staged = mutate_smem_bytes(n, S.cols, true) <= kSmemCap;
  const size_t sm = mutate_smem_bytes(n, S.cols, staged);
  cudaError_t err = cudaSuccess;
  const int rc = TT_DISPATCH_SHAPE(S.n_sp, S.n_red, ({
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(k_explore_gens<NSP, NRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
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
    err = cudaLaunchKernelEx(&cfg, k_explore_gens<NSP, NRED>, S, D, toggles, (int)n, n_steps, dv, s_init, h, flags,
                             (int)staged);
  }));
  return rc ? rc : (err != cudaSuccess ? 2 : 0);
}

int explore_cluster_size(int64_t n) { return (int)std::min<int64_t>(8, std::max<int64_t>(1, (n + 63) / 64)); }

}  // namespace tt

extern "C" int ttdbg_mutate_clocks(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_clk_mut, sizeof(long long) * (n < 8 ? n : 8));
}
