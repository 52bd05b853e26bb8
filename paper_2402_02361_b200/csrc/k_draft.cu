// k_draft.cu — K0 population generator, K1 SA draft cost, schedule
// identities and K2 the deduplicating draft top-K selector (PriorFilter).
//
// Reference path: random_init (schedule.cpp:166-186), draft_cost
// (draft.cpp:129-154) and explore(..., n_steps = 1, ...) (draft.cpp:156-221)
// whose pool keeps the first occurrence of every schedule key and trims to
// the draft_size lowest (cost, discovery) entries.
//
// K2 design (HBM-bound, no full sort of N):
//   * N <= 4096: one CTA computes every cost into shared memory, sorts
//     (cost, index) bitonically, dedups and emits — a single launch.
//   * N  > 4096: K1 writes costs and a 4096-bin shared-memory histogram of
//     the cost bit pattern (positive doubles order like their bits); a 1-CTA
//     scan finds the bin holding the K-th key; up to two refine passes
//     narrow it 12 bits at a time until at most kSurvivorCap keys survive;
//     a compaction pass inserts survivors into a hash table keyed by their
//     exact 64-bit identity (atomicMin keeps the first index: the reference's
//     "first discovery wins" dedup); a 1-CTA finalisation sorts the unique
//     survivors by (cost, index) and emits the K lowest.
// Identical schedules have identical costs, so the threshold never splits
// a duplicate group; selection is exact for any input.
#include <cstdint>

#include "tt_block.cuh"
#include "tt_device.cuh"
#include "tt_kernels.h"

namespace tt {

constexpr int kHistBins = 4096;
constexpr int kSurvivorCap = 4096;   // unique survivors the finaliser sorts
constexpr int kTableCap = 16384;     // hash slots (load <= 0.25 at the cap)
constexpr uint64_t kEmpty = ~0ull;

struct Src {
  const int32_t* soa;
  int64_t ld;
  uint64_t s0;        // RNG base state (seeded source)
  int64_t first;      // seeded source: global schedule index of local 0
  int64_t index_base; // added to local indices in outputs
};

template <int NSP, int NRED, bool SEED>
__device__ __forceinline__ uint64_t load_cand(const DevSketch& S, const Src& src, int64_t i,
                                              Factors<NSP, NRED>& F, bool with_unroll) {
  if constexpr (SEED) {
    return generate<NSP, NRED>(S, src.s0, (uint64_t)(src.first + i), F);
  } else {
    load_factors<NSP, NRED>(src.soa, src.ld, i, F, with_unroll);
    return 0;
  }
}

// validate_schedule (schedule.cpp:242-278) on the register copy
template <int NSP, int NRED>
__device__ __forceinline__ bool valid_factors(const DevSketch& S, const Factors<NSP, NRED>& F) {
  bool ok = true;
#pragma unroll
  for (int a = 0; a < NSP; ++a) {
    int64_t prod = 1;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      ok &= F.f[4 * a + t] >= 1;
      prod *= F.f[4 * a + t];
    }
    ok &= prod == S.extent[a];
    if (S.arity[a] == 2) ok &= F.f[4 * a + 2] == 1 && F.f[4 * a + 3] == 1;
  }
#pragma unroll
  for (int r = 0; r < NRED; ++r) {
    int64_t prod = 1;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      ok &= F.f[4 * NSP + 3 * r + t] >= 1;
      prod *= F.f[4 * NSP + 3 * r + t];
    }
    ok &= prod == S.extent[NSP + r];
  }
  return ok;
}

// ------------------------------------------------------------------ K0 ----
template <int NSP, int NRED>
__global__ void __launch_bounds__(256) k_generate(DevSketch S, uint64_t s0, int64_t first, int64_t n,
                                                  int32_t* __restrict__ soa, int64_t ld,
                                                  uint64_t* __restrict__ id_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Factors<NSP, NRED> F;
    const uint64_t id = generate<NSP, NRED>(S, s0, (uint64_t)(first + i), F);
    if (soa) store_factors<NSP, NRED>(soa, ld, i, F);
    if (id_out) id_out[i] = id;
  }
}

template <int NSP, int NRED>
__global__ void __launch_bounds__(256) k_identity(DevSketch S, const int32_t* __restrict__ soa, int64_t ld,
                                                  int64_t n, uint64_t* __restrict__ id_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Factors<NSP, NRED> F;
    load_factors<NSP, NRED>(soa, ld, i, F, true);
    id_out[i] = identity_of<NSP, NRED>(S, F);
  }
}

template <int NSP, int NRED>
__global__ void __launch_bounds__(256) k_from_identity(DevSketch S, const uint64_t* __restrict__ id, int64_t n,
                                                       int32_t* __restrict__ soa, int64_t ld) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Factors<NSP, NRED> F;
    from_identity<NSP, NRED>(S, id[i], F);
    store_factors<NSP, NRED>(soa, ld, i, F);
  }
}

// ------------------------------------------------------------------ K1 ----
// One candidate per thread; SoA factor columns are read coalesced (thread i
// of a warp reads element i of every column). With a histogram pointer the
// kernel also bins the cost bit pattern for the top-K selector.
template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(256) k_draft_cost(DevSketch S, DevDevice D, Src src, int64_t n, int toggles,
                                                    double* __restrict__ cost, uint32_t* __restrict__ hist,
                                                    int* __restrict__ invalid) {
  __shared__ uint32_t sh[kHistBins];
  if (hist) {
    for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) sh[b] = 0;
    __syncthreads();
  }
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Factors<NSP, NRED> F;
    load_cand<NSP, NRED, SEED>(S, src, i, F, false);
    if constexpr (!SEED) bad |= !valid_factors<NSP, NRED>(S, F);
    const double c = draft_cost_of<NSP, NRED>(S, D, F, toggles);
    cost[i] = c;
    if (hist) atomicAdd(&sh[(cost_key(c) >> 51) & (kHistBins - 1)], 1u);
  }
  if (bad) atomicOr(invalid, 1);
  if (hist) {
    __syncthreads();
    for (int b = threadIdx.x; b < kHistBins; b += blockDim.x)
      if (sh[b]) atomicAdd(&hist[b], sh[b]);
  }
}

// --------------------------------------------------------- K2 selector ----
// Scan: find the histogram bin that contains the need-th smallest key.
__global__ void __launch_bounds__(1024) k_sel_scan(uint32_t* __restrict__ hist, SelState* __restrict__ st,
                                                   int64_t need, int64_t n, int level) {
  __shared__ int counts[kHistBins];
  __shared__ int excl[kHistBins];
  __shared__ int wt[32];
  __shared__ int found;
  if (level > 0 && st->done) return;  // refine not needed: nothing to do (hist untouched)
  if (level == 0 && threadIdx.x == 0) {
    st->prefix = 0, st->shift = 64, st->below = 0, st->done = 0, st->all = 0, st->status = 0;
    st->need = need;
    st->survivors = 0, st->unique = 0, st->count = 0;
  }
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) {
    counts[b] = (int)hist[b];
    hist[b] = 0;  // keep the zero invariant for the next pass
  }
  if (threadIdx.x == 0) found = -1;
  __syncthreads();
  const int total = block_exclusive_scan(counts, excl, kHistBins, wt);
  const int64_t below = level == 0 ? 0 : st->below;
  const int64_t want = (level == 0 ? need : st->need) - below;
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x)
    if (counts[b] > 0 && excl[b] < want && excl[b] + counts[b] >= want) found = b;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int width = level == 0 ? 12 : 12;
  const int new_shift = level == 0 ? 51 : (st->shift - width < 0 ? 0 : st->shift - width);
  if (found < 0) {  // fewer keys than needed in range: everything survives
    if (level == 0) {
      st->all = 1;
      st->done = 1;
      st->survivors = (uint32_t)(total < 0 ? 0 : total);
    } else {
      // cannot happen (the refined bin held >= want keys); keep whole bin
      st->done = 1;
    }
    return;
  }
  const int64_t surv = below + excl[found] + counts[found];
  const uint64_t prefix = level == 0 ? (uint64_t)found : ((st->prefix << (st->shift - new_shift)) | (uint64_t)found);
  st->prefix = prefix;
  st->shift = new_shift;
  if (surv <= kSurvivorCap || new_shift == 0 || level >= 2) {
    st->done = 1;
    st->survivors = (uint32_t)(surv > 0xffffffffLL ? 0xffffffffu : surv);
  } else {
    st->below = below + excl[found];
  }
  (void)n;
}

// Refine: histogram the next 12 bits of the keys inside the current bin.
__global__ void __launch_bounds__(256) k_sel_refine(const double* __restrict__ cost, int64_t n,
                                                    const SelState* __restrict__ st, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kHistBins];
  if (st->done) return;
  const uint64_t prefix = st->prefix;
  const int shift = st->shift;
  const int nshift = shift - 12 < 0 ? 0 : shift - 12;
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = cost_key(__ldg(cost + i));
    if ((k >> shift) == prefix) atomicAdd(&sh[(k >> nshift) & ((1u << (shift - nshift)) - 1u)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

__device__ __forceinline__ uint64_t slot_hash(uint64_t id) { return scramble64(id + kGolden); }

// Compaction: survivors → identity-keyed hash table (first index wins).
template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(256) k_sel_compact(DevSketch S, Src src, const double* __restrict__ cost,
                                                     int64_t n, SelState* __restrict__ st,
                                                     uint64_t* __restrict__ tkeys, uint64_t* __restrict__ tvals) {
  const uint64_t prefix = st->prefix;
  const int shift = st->shift;
  const bool all = st->all != 0;
  int local_unique = 0;
  bool overflow = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = cost_key(__ldg(cost + i));
    const bool keep = all || shift >= 64 || (k >> shift) <= prefix;
    if (!keep) continue;
    Factors<NSP, NRED> F;
    uint64_t id = load_cand<NSP, NRED, SEED>(S, src, i, F, true);
    if constexpr (!SEED) id = identity_of<NSP, NRED>(S, F);
    uint64_t h = slot_hash(id) & (kTableCap - 1);
    int probes = 0;
    while (true) {
      const uint64_t prev = atomicCAS((unsigned long long*)&tkeys[h], (unsigned long long)kEmpty,
                                      (unsigned long long)id);
      if (prev == kEmpty || prev == id) {
        atomicMin((unsigned long long*)&tvals[h], (unsigned long long)i);
        local_unique += prev == kEmpty;
        break;
      }
      h = (h + 1) & (kTableCap - 1);
      if (++probes >= kTableCap) {
        overflow = true;
        break;
      }
    }
  }
  if (local_unique) atomicAdd(&st->unique, (uint32_t)local_unique);
  if (overflow) atomicOr(&st->status, TT_SEL_OVERFLOW);
}

// Sort (cost, index, identity) entries, drop later duplicates of an
// identity (duplicates share the cost, so they are adjacent runs of the
// (cost, index) order), emit the first K. Entries >= nvalid are padding.
__device__ void sort_dedup_emit(uint64_t* a, uint64_t* b, uint64_t* c, int* flag, int* pos, int* wt,
                                int nvalid, int npow2, int64_t k, int64_t index_base,
                                int64_t* __restrict__ out_idx, double* __restrict__ out_cost,
                                uint64_t* __restrict__ out_id, int64_t* __restrict__ out_count) {
  for (int e = threadIdx.x + nvalid; e < npow2; e += blockDim.x) a[e] = kEmpty, b[e] = kEmpty, c[e] = kEmpty;
  block_bitonic_sort(a, b, c, npow2);
  for (int e = threadIdx.x; e < npow2; e += blockDim.x) {
    int keep = e < nvalid;
    for (int q = e - 1; keep && q >= 0 && a[q] == a[e]; --q)
      if (c[q] == c[e]) keep = 0;
    flag[e] = keep;
  }
  __syncthreads();
  const int total = block_exclusive_scan(flag, pos, npow2, wt);
  for (int e = threadIdx.x; e < npow2; e += blockDim.x) {
    if (flag[e] && pos[e] < k) {
      const int o = pos[e];
      out_idx[o] = (int64_t)b[e] + index_base;
      out_cost[o] = key_cost(a[e]);
      if (out_id) out_id[o] = c[e];
    }
  }
  if (threadIdx.x == 0) *out_count = total < k ? total : k;
}

// Finalise: unique survivors from the hash table → sorted top-K.
__global__ void __launch_bounds__(1024) k_sel_finalize(const double* __restrict__ cost, SelState* __restrict__ st,
                                                       uint64_t* __restrict__ tkeys, uint64_t* __restrict__ tvals,
                                                       int64_t k, int64_t n, int64_t index_base,
                                                       int64_t* __restrict__ out_idx, double* __restrict__ out_cost,
                                                       uint64_t* __restrict__ out_id, int64_t* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* a = (uint64_t*)smem;
  uint64_t* b = a + kSurvivorCap;
  uint64_t* c = b + kSurvivorCap;
  int* flag = (int*)(c + kSurvivorCap);
  int* pos = flag + kSurvivorCap;
  __shared__ int wt[32];
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  bool overflow = false;
  for (int s = threadIdx.x; s < kTableCap; s += blockDim.x) {
    const uint64_t id = tkeys[s];
    if (id == kEmpty) continue;
    const uint64_t idx = tvals[s];
    tkeys[s] = kEmpty;  // restore the empty-table invariant
    tvals[s] = kEmpty;
    const int e = atomicAdd(&cnt, 1);
    if (e < kSurvivorCap) {
      a[e] = cost_key(cost[idx]);
      b[e] = idx;
      c[e] = id;
    } else {
      overflow = true;
    }
  }
  if (overflow) atomicOr(&st->status, TT_SEL_OVERFLOW);
  __syncthreads();
  const int u = cnt < kSurvivorCap ? cnt : kSurvivorCap;
  const int np = next_pow2(u < 2 ? 2 : u);
  sort_dedup_emit(a, b, c, flag, pos, wt, u, np, k, index_base, out_idx, out_cost, out_id, out_count);
  if (threadIdx.x == 0) {
    // fewer unique survivors than K while keys were cut off: raise the target
    const bool everything = st->all || (int64_t)st->survivors >= n;
    if (u < k && !everything) atomicOr(&st->status, TT_SEL_NEED_MORE);
    st->count = u < k ? u : k;
  }
}

// N <= 4096: the whole selection in one CTA.
template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(1024) k_sel_small(DevSketch S, DevDevice D, Src src, int64_t n, int toggles,
                                                    int64_t k, SelState* __restrict__ st,
                                                    int64_t* __restrict__ out_idx, double* __restrict__ out_cost,
                                                    uint64_t* __restrict__ out_id, int64_t* __restrict__ out_count,
                                                    int* __restrict__ invalid) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int np = next_pow2(n < 2 ? 2 : (int)n);
  uint64_t* a = (uint64_t*)smem;
  uint64_t* b = a + np;
  uint64_t* c = b + np;
  int* flag = (int*)(c + np);
  int* pos = flag + np;
  __shared__ int wt[32];
  bool bad = false;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    Factors<NSP, NRED> F;
    const uint64_t id = load_cand<NSP, NRED, SEED>(S, src, i, F, false);
    if constexpr (!SEED) bad |= !valid_factors<NSP, NRED>(S, F);
    a[i] = cost_key(draft_cost_of<NSP, NRED>(S, D, F, toggles));
    b[i] = (uint64_t)i;
    c[i] = id;
  }
  if (bad) atomicOr(invalid, 1);
  for (int e = threadIdx.x + (int)n; e < np; e += blockDim.x) a[e] = kEmpty, b[e] = kEmpty, c[e] = kEmpty;
  block_bitonic_sort(a, b, c, np);
  if constexpr (!SEED) {
    // identities only where a cost tie makes them matter
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const bool tie = (e > 0 && a[e - 1] == a[e]) || (e + 1 < n && a[e + 1] == a[e]);
      if (tie) {
        Factors<NSP, NRED> F;
        load_factors<NSP, NRED>(src.soa, src.ld, (int64_t)b[e], F, true);
        c[e] = identity_of<NSP, NRED>(S, F);
      } else {
        c[e] = kEmpty - 1 - (uint64_t)e;  // unique placeholder, never compared equal
      }
    }
    __syncthreads();
  }
  sort_dedup_emit(a, b, c, flag, pos, wt, (int)n, np, k, src.index_base, out_idx, out_cost, out_id, out_count);
  if constexpr (!SEED) {
    if (out_id) {
      __syncthreads();
      const int64_t cnt = *out_count;
      for (int o = threadIdx.x; o < cnt; o += blockDim.x) {
        Factors<NSP, NRED> F;
        load_factors<NSP, NRED>(src.soa, src.ld, out_idx[o] - src.index_base, F, true);
        out_id[o] = identity_of<NSP, NRED>(S, F);
      }
    }
  }
  if (threadIdx.x == 0 && st) {
    st->status = 0;
    st->count = *out_count;
  }
}

// Cross-rank merge (C1's consumer): R lists of (cost, global index, id).
__global__ void __launch_bounds__(1024) k_merge(const double* __restrict__ cost, const int64_t* __restrict__ gidx,
                                                const uint64_t* __restrict__ id, int m, int64_t k,
                                                int64_t* __restrict__ out_idx, double* __restrict__ out_cost,
                                                uint64_t* __restrict__ out_id, int64_t* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int np = next_pow2(m < 2 ? 2 : m);
  uint64_t* a = (uint64_t*)smem;
  uint64_t* b = a + np;
  uint64_t* c = b + np;
  int* flag = (int*)(c + np);
  int* pos = flag + np;
  __shared__ int wt[32];
  for (int e = threadIdx.x; e < m; e += blockDim.x) {
    a[e] = gidx[e] < 0 ? kEmpty : cost_key(cost[e]);  // negative index = empty slot
    b[e] = gidx[e] < 0 ? kEmpty : (uint64_t)gidx[e];
    c[e] = gidx[e] < 0 ? kEmpty : id[e];
  }
  __shared__ int valid;
  if (threadIdx.x == 0) valid = 0;
  __syncthreads();
  int mine = 0;
  for (int e = threadIdx.x; e < m; e += blockDim.x) mine += gidx[e] >= 0;
  if (mine) atomicAdd(&valid, mine);
  __syncthreads();
  // empty slots carry all-ones keys, sort last and fall outside `valid`
  sort_dedup_emit(a, b, c, flag, pos, wt, valid, np, k, 0, out_idx, out_cost, out_id, out_count);
}

// ------------------------------------------------------------ launchers ----
size_t small_select_smem(int64_t n);
static int grid_for(int64_t n, int threads, int max_blocks) {
  int64_t g = (n + threads - 1) / threads;
  if (g > max_blocks) g = max_blocks;
  return (int)(g < 1 ? 1 : g);
}

int launch_generate(const DevSketch& S, uint64_t s0, int64_t first, int64_t n, int32_t* soa, int64_t ld,
                    uint64_t* id_out, cudaStream_t st) {
  const int g = grid_for(n, 256, 148 * 16);
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_generate<NSP, NRED><<<g, 256, 0, st>>>(S, s0, first, n, soa, ld, id_out)));
}

int launch_identity(const DevSketch& S, const int32_t* soa, int64_t ld, int64_t n, uint64_t* id_out,
                    cudaStream_t st) {
  const int g = grid_for(n, 256, 148 * 16);
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_identity<NSP, NRED><<<g, 256, 0, st>>>(S, soa, ld, n, id_out)));
}

int launch_from_identity(const DevSketch& S, const uint64_t* id, int64_t n, int32_t* soa, int64_t ld,
                         cudaStream_t st) {
  const int g = grid_for(n, 256, 148 * 16);
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_from_identity<NSP, NRED><<<g, 256, 0, st>>>(S, id, n, soa, ld)));
}

int launch_draft_cost(const DevSketch& S, const DevDevice& D, const int32_t* soa, int64_t ld, uint64_t s0,
                      int64_t first, bool seeded, int64_t n, int toggles, double* cost, uint32_t* hist,
                      int* invalid, cudaStream_t st) {
  const int g = grid_for(n, 256, 148 * 8);
  Src src{soa, ld, s0, first, 0};
  if (seeded)
    return TT_DISPATCH_SHAPE(S.n_sp, S.n_red,
                             (tt::note_launch(), k_draft_cost<NSP, NRED, true><<<g, 256, 0, st>>>(S, D, src, n, toggles, cost, hist, invalid)));
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red,
                           (tt::note_launch(), k_draft_cost<NSP, NRED, false><<<g, 256, 0, st>>>(S, D, src, n, toggles, cost, hist, invalid)));
}

template <int NSP, int NRED, bool SEED>
static void run_small(const DevSketch& S, const DevDevice& D, const Src& src, int64_t n, int toggles, int64_t k,
                      SelScratch& w, int64_t* out_idx, double* out_cost, uint64_t* out_id, int64_t* out_count,
                      size_t sm, cudaStream_t st) {
  auto f = k_sel_small<NSP, NRED, SEED>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  tt::note_launch(), f<<<1, 1024, sm, st>>>(S, D, src, n, toggles, k, w.state, out_idx, out_cost, out_id, out_count, w.invalid);
}

size_t small_select_smem(int64_t n) {
  const int np = next_pow2(n < 2 ? 2 : (int)n);
  return (size_t)np * (3 * sizeof(uint64_t) + 2 * sizeof(int));
}

int launch_select(const DevSketch& S, const DevDevice& D, const int32_t* soa, int64_t ld, uint64_t s0,
                  int64_t first, bool seeded, int64_t n, int64_t k, int64_t need, int toggles,
                  int64_t index_base, SelScratch& w, int64_t* out_idx, double* out_cost, uint64_t* out_id,
                  int64_t* out_count, cudaStream_t st) {
  Src src{soa, ld, s0, first, index_base};
  if (n <= kSmallSelectMax) {
    const size_t sm = small_select_smem(n);
    if (seeded)
      return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_small<NSP, NRED, true>(S, D, src, n, toggles, k, w, out_idx, out_cost, out_id, out_count, sm, st)));
    return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_small<NSP, NRED, false>(S, D, src, n, toggles, k, w, out_idx, out_cost, out_id, out_count, sm, st)));
  }
  {
    int rc = launch_draft_cost(S, D, soa, ld, s0, first, seeded, n, toggles, w.cost, w.hist, w.invalid, st);
    if (rc) return rc;
  }
  tt::note_launch(), k_sel_scan<<<1, 1024, 0, st>>>(w.hist, w.state, need, n, 0);
  for (int lv = 1; lv <= 2; ++lv) {
    const int g = grid_for(n, 256, 148 * 8);
    tt::note_launch(), k_sel_refine<<<g, 256, 0, st>>>(w.cost, n, w.state, w.hist);
    tt::note_launch(), k_sel_scan<<<1, 1024, 0, st>>>(w.hist, w.state, need, n, lv);
  }
  {
    const int g = grid_for(n, 256, 148 * 8);
    int rc;
    if (seeded)
      rc = TT_DISPATCH_SHAPE(S.n_sp, S.n_red,
                             (tt::note_launch(), k_sel_compact<NSP, NRED, true><<<g, 256, 0, st>>>(S, src, w.cost, n, w.state, w.tkeys, w.tvals)));
    else
      rc = TT_DISPATCH_SHAPE(S.n_sp, S.n_red,
                             (tt::note_launch(), k_sel_compact<NSP, NRED, false><<<g, 256, 0, st>>>(S, src, w.cost, n, w.state, w.tkeys, w.tvals)));
    if (rc) return rc;
  }
  const size_t sm = (size_t)kSurvivorCap * (3 * sizeof(uint64_t) + 2 * sizeof(int));
  cudaFuncSetAttribute(k_sel_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  tt::note_launch(), k_sel_finalize<<<1, 1024, sm, st>>>(w.cost, w.state, w.tkeys, w.tvals, k, n, index_base, out_idx, out_cost,
                                      out_id, out_count);
  return 0;
}

int launch_merge(const double* cost, const int64_t* gidx, const uint64_t* id, int m, int64_t k, int64_t* out_idx,
                 double* out_cost, uint64_t* out_id, int64_t* out_count, cudaStream_t st) {
  if (m > kSurvivorCap) return -1;
  const int np = next_pow2(m < 2 ? 2 : m);
  const size_t sm = (size_t)np * (3 * sizeof(uint64_t) + 2 * sizeof(int));
  cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  tt::note_launch(), k_merge<<<1, 1024, sm, st>>>(cost, gidx, id, m, k, out_idx, out_cost, out_id, out_count);
  return 0;
}

}  // namespace tt
