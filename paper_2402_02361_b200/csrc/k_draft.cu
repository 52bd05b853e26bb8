// k_draft.cu — K0 population generator, K1 SA draft cost, schedule
// identities and K2 the deduplicating draft top-K selector (PriorFilter).
//
// Reference path: random_init (schedule.cpp:166-186), draft_cost
// (draft.cpp:129-154) and explore(..., n_steps = 1, ...) (draft.cpp:156-221)
// whose pool keeps the first occurrence of every schedule key and trims to
// the draft_size lowest (cost, discovery) entries.
//
// K2 design (HBM-bound, no full sort of N):
//   * N <= 4096: one CTA computes every cost in registers, sorts (cost,
//     index) with a register/shuffle bitonic network, dedups, emits.
//   * N  > 4096: K1 writes costs and a 4096-bin shared-memory histogram of
//     the cost bit pattern (positive doubles order like their bits); a 1-CTA
//     scan finds the bin holding the need-th key; up to two refine passes
//     narrow it 12 bits at a time until at most kSurvivorTarget keys
//     survive; a compaction pass appends the survivors; a 1-CTA finaliser
//     sorts them, resolves identities only inside equal-cost runs, drops
//     later duplicates ("first discovery wins") and emits the K lowest.
//   * Pathological ties (> kSurvivorCap keys sharing a 36-bit cost prefix)
//     switch to an identity-keyed hash-table compaction that deduplicates
//     on insert (atomicMin keeps the first index).
// Identical schedules have identical costs, so the threshold never splits
// a duplicate group; selection is exact for any input.
#include <cstdint>

#include "tt_block.cuh"
#include "tt_device.cuh"
#include "tt_kernels.h"

namespace tt {

constexpr int kHistBins = 4096;
constexpr int kSurvivorTarget = 1024;  // refine while more keys survive
constexpr int kFinalCap = 1024;        // survivors the (append-path) finaliser sorts
constexpr int kSurvivorCap = 4096;     // entries the hash-path finaliser / merge sort
constexpr int kTableCap = 16384;       // hash slots of the fallback path
constexpr int kSortE = 4;              // keys per thread in the 4096-entry sorts
constexpr int kFinalE = 1;             // keys per thread in the 1024-entry sorts (1024 threads)
constexpr uint64_t kEmpty = ~0ull;
constexpr int kFastCap = 4096;               // survivors the fast path ranks
constexpr int kSampleMax = 32768;            // sampled cost keys (top 32 bits) for the threshold
constexpr int64_t kFastMaxN = int64_t{16} << 20;  // fast path population limit

static int grid_for(int64_t n, int threads, int max_blocks) {
  int64_t g = (n + threads - 1) / threads;
  if (g > max_blocks) g = max_blocks;
  return (int)(g < 1 ? 1 : g);
}

template <typename F>
static void set_smem(F* f, size_t bytes) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

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

template <int NSP, int NRED, bool SEED>
__device__ __forceinline__ uint64_t identity_at(const DevSketch& S, const Src& src, int64_t i) {
  Factors<NSP, NRED> F;
  const uint64_t id = load_cand<NSP, NRED, SEED>(S, src, i, F, true);
  if constexpr (SEED) return id;
  return identity_of<NSP, NRED>(S, F);
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
                                                   int64_t need, int level) {
  __shared__ int counts[kHistBins];
  __shared__ int excl[kHistBins];
  __shared__ int wt[32];
  __shared__ int found;
  if (level > 0 && st->done) return;  // nothing to refine (hist untouched)
  if (level == 0 && threadIdx.x == 0) {
    st->prefix = 0, st->shift = 64, st->below = 0, st->done = 0, st->all = 0, st->status = 0;
    st->need = need;
    st->survivors = 0, st->unique = 0, st->count = 0, st->nsurv = 0;
  }
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) {
    counts[b] = (int)hist[b];
    hist[b] = 0;  // keep the zero invariant for the next pass
  }
  if (threadIdx.x == 0) found = -1;
  __syncthreads();
  const int total = block_exclusive_scan(counts, excl, kHistBins, wt);
  const int64_t below = level == 0 ? 0 : st->below;
  const int64_t want = need - below;
  for (int b = threadIdx.x; b < kHistBins; b += blockDim.x)
    if (counts[b] > 0 && excl[b] < want && excl[b] + counts[b] >= want) found = b;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int new_shift = level == 0 ? 51 : (st->shift - 12 < 0 ? 0 : st->shift - 12);
  if (found < 0) {  // fewer keys than needed: everything in range survives
    if (level == 0) {
      st->all = 1;
      st->survivors = (uint32_t)total;
    }
    st->done = 1;
    return;
  }
  const int64_t surv = below + excl[found] + counts[found];
  const uint64_t prefix = level == 0 ? (uint64_t)found : ((st->prefix << (st->shift - new_shift)) | (uint64_t)found);
  st->prefix = prefix;
  st->shift = new_shift;
  if (surv <= kSurvivorTarget || new_shift == 0 || level >= 2) {
    st->done = 1;
    st->survivors = (uint32_t)(surv > 0xffffffffLL ? 0xffffffffu : surv);
  } else {
    st->below = below + excl[found];
  }
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

__device__ __forceinline__ bool survives(uint64_t k, const SelState& st) {
  return st.all || st.shift >= 64 || (k >> st.shift) <= st.prefix;
}

// Compaction: append survivors (warp-aggregated atomics). Order is
// irrelevant: the finaliser sorts by (cost, index).
__global__ void __launch_bounds__(256) k_sel_compact(const double* __restrict__ cost, int64_t n,
                                                     SelState* __restrict__ st, uint64_t* __restrict__ skey,
                                                     int64_t* __restrict__ sidx) {
  const SelState s = *st;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint64_t k = 0;
    bool keep = false;
    if (i < n) {
      k = cost_key(__ldg(cost + i));
      keep = survives(k, s);
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    uint32_t pos0 = 0;
    if (lane == 0) pos0 = atomicAdd(&st->nsurv, (uint32_t)__popc(m));
    pos0 = __shfl_sync(0xffffffffu, pos0, 0);
    if (keep) {
      const uint32_t p = pos0 + __popc(m & ((1u << lane) - 1u));
      if (p < kSurvivorCap) skey[p] = k, sidx[p] = i;
    }
  }
}

// Dedup + emit over sorted shared arrays a (cost key), b (local index),
// c (identity; valid wherever an equal-cost neighbour exists).
__device__ void dedup_emit(const uint64_t* a, const uint64_t* b, const uint64_t* c, int* flag, int* pos, int* wt,
                           int nvalid, int np, int64_t k, int64_t index_base, int64_t* __restrict__ out_idx,
                           double* __restrict__ out_cost, uint64_t* __restrict__ out_id,
                           int64_t* __restrict__ out_count) {
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    int keep = e < nvalid;
    for (int q = e - 1; keep && q >= 0 && a[q] == a[e]; --q)
      if (c[q] == c[e]) keep = 0;
    flag[e] = keep;
  }
  __syncthreads();
  const int total = block_exclusive_scan(flag, pos, np, wt);
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    if (flag[e] && pos[e] < k) {
      const int o = pos[e];
      out_idx[o] = (int64_t)b[e] + index_base;
      out_cost[o] = key_cost(a[e]);
      if (out_id) out_id[o] = c[e];
    }
  }
  if (threadIdx.x == 0) *out_count = total < k ? total : k;
}

struct SortSmem {
  Key2* xchg;
  uint64_t *a, *b, *c;
  int *flag, *pos;
};

__host__ __device__ inline size_t sort_smem_bytes(int n) {
  return (size_t)n * (sizeof(Key2) + 3 * sizeof(uint64_t) + 2 * sizeof(int));
}

__device__ inline SortSmem carve_sort(unsigned char* base, int n) {
  SortSmem s;
  s.xchg = (Key2*)base;
  s.a = (uint64_t*)(s.xchg + n);
  s.b = s.a + n;
  s.c = s.b + n;
  s.flag = (int*)(s.c + n);
  s.pos = s.flag + n;
  return s;
}

// Sorted keys → shared arrays, identities for the entries of equal-cost
// runs (duplicates can only hide there), dedup, emit. Requires
// kSortE * blockDim.x == kSurvivorCap.
template <int NSP, int NRED, bool SEED>
__device__ void sort_ties_emit(const DevSketch& S, const Src& src, Key2 (&kk)[kFinalE], SortSmem& sm, int nvalid,
                               int64_t k, int64_t* out_idx, double* out_cost, uint64_t* out_id,
                               int64_t* out_count, int* wt) {
  block_sort_reg<kFinalE, Key2>(kk, sm.xchg);
  const int NT = blockDim.x;
#pragma unroll
  for (int e = 0; e < kFinalE; ++e) {
    const int p = e * NT + threadIdx.x;
    sm.a[p] = kk[e].a;
    sm.b[p] = kk[e].b;
  }
  __syncthreads();
  const int np = kFinalE * NT;
  // identities only inside equal-cost runs: the only place duplicates hide
  for (int p = threadIdx.x; p < np; p += NT) {
    uint64_t id = kEmpty - 1 - (uint64_t)p;  // unique placeholder, never compared equal
    if (p < nvalid) {
      const bool tie = (p > 0 && sm.a[p - 1] == sm.a[p]) || (p + 1 < nvalid && sm.a[p + 1] == sm.a[p]);
      if (tie) id = identity_at<NSP, NRED, SEED>(S, src, (int64_t)sm.b[p]);
    }
    sm.c[p] = id;
  }
  __syncthreads();
  dedup_emit(sm.a, sm.b, sm.c, sm.flag, sm.pos, wt, nvalid, np, k, src.index_base, out_idx, out_cost, nullptr,
             out_count);
  if (out_id) {  // identities of the emitted entries, one per thread
    __syncthreads();
    const int64_t cnt = *out_count;
    for (int o = threadIdx.x; o < cnt; o += NT)
      out_id[o] = identity_at<NSP, NRED, SEED>(S, src, out_idx[o] - src.index_base);
  }
}

// Finalise (append path): survivors → sorted, deduplicated top-K.
template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(1024) k_sel_finalize(DevSketch S, Src src, SelState* __restrict__ st,
                                                       const uint64_t* __restrict__ skey,
                                                       const int64_t* __restrict__ sidx, int64_t k, int64_t n,
                                                       int64_t* __restrict__ out_idx, double* __restrict__ out_cost,
                                                       uint64_t* __restrict__ out_id, int64_t* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  SortSmem sm = carve_sort(smem, kFinalCap);
  __shared__ int wt[32];
  const uint32_t ns = st->nsurv;
  if (ns > (uint32_t)kFinalCap) {  // heavy ties: hash path (host retries)
    if (threadIdx.x == 0) {
      st->status |= TT_SEL_OVERFLOW;
      *out_count = 0;
    }
    return;
  }
  const int m = (int)ns;
  Key2 kk[kFinalE];
#pragma unroll
  for (int e = 0; e < kFinalE; ++e) {
    const int p = e * blockDim.x + threadIdx.x;
    kk[e].a = p < m ? skey[p] : kEmpty;
    kk[e].b = p < m ? (uint64_t)sidx[p] : kEmpty;
  }
  sort_ties_emit<NSP, NRED, SEED>(S, src, kk, sm, m, k, out_idx, out_cost, out_id, out_count, wt);
  if (threadIdx.x == 0) {
    const int64_t cnt = *out_count;
    const bool everything = st->all || (int64_t)m >= n;
    if (cnt < k && !everything) st->status |= TT_SEL_NEED_MORE;  // duplicates ate the margin
    st->count = cnt;
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
  SortSmem sm = carve_sort(smem, kFinalCap);
  __shared__ int wt[32];
  bool bad = false;
  Key2 kk[kFinalE];
#pragma unroll
  for (int e = 0; e < kFinalE; ++e) {
    const int p = e * blockDim.x + threadIdx.x;
    kk[e].a = kEmpty, kk[e].b = kEmpty;
    if (p < n) {
      Factors<NSP, NRED> F;
      load_cand<NSP, NRED, SEED>(S, src, p, F, false);
      if constexpr (!SEED) bad |= !valid_factors<NSP, NRED>(S, F);
      kk[e].a = cost_key(draft_cost_of<NSP, NRED>(S, D, F, toggles));
      kk[e].b = (uint64_t)p;
    }
  }
  if (bad) atomicOr(invalid, 1);
  sort_ties_emit<NSP, NRED, SEED>(S, src, kk, sm, (int)n, k, out_idx, out_cost, out_id, out_count, wt);
  if (threadIdx.x == 0 && st) {
    st->status = 0;
    st->count = *out_count;
  }
}

// ------------------------------------------- fast path (sampled threshold) ----
// N > 1024, four short kernels and no CTA-wide sorting network (a bitonic
// sort of 4096 keys costs ~60 us on one SM; everything here is either
// grid-wide or O(log) passes):
//   k_fsel_cost:    K1 over the population, costs to HBM, a strided sample of
//                   4096..32768 cost keys (top 32 bits); the last CTA (ticket) radix-selects the
//                   sample key of rank ceil(1.5 need ns / n) + 3 as the
//                   survivor threshold (~1.5x need survivors expected).
//   k_fsel_compact: keys <= threshold appended (warp-aggregated) with a
//                   schedule fingerprint (seeded: the exact identity the
//                   generator returns; explicit: a 64-bit hash of the factor
//                   columns, confirmed column by column on a match).
//   k_fsel_rank:    all-pairs over the <= 4096 survivors, spread over the GPU:
//                   each (survivor, 256-chunk) thread counts the keys below
//                   it ((cost, index) order) and flags a duplicate when an
//                   equal-cost survivor with a lower index is the same
//                   schedule ("first discovery wins", draft.cpp:200-203).
//   k_fsel_emit:    one CTA scatters survivors to their ranks and emits the K
//                   lowest unique in ascending (cost, index) order.
// Exactness never depends on the sample: every key <= threshold survives,
// so whenever >= K unique schedules survive they include the true top-K;
// otherwise NEED_MORE (the host retries with a larger need); > 4096
// survivors report OVERFLOW (the identity-keyed hash path takes over).
constexpr int kFastThreads = 1024;

// %globaltimer marks (ns) of the fast selector's phases, read by ttdbg_select_clocks:
// [0] first CTA start, [1] K1 done (last CTA begins the threshold), [2] threshold done,
// [3] compact start, [4] rank start, [5] emit start, [6] emit end
__device__ unsigned long long g_sel_ns[12];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int kFastE = kFastCap / kFastThreads;  // 4 keys per thread
constexpr int kRankChunk = 128;

__device__ __forceinline__ bool last_cta(SelState* st) {
  __shared__ int am_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    am_last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last != 0;
}

// Upper bound of the 64-bit cost key whose top 32 bits have rank r (0-based)
// among keys[0..n) in shared memory: MSB-first radix select, 8 bits per pass
// (four passes), the low 32 bits filled with ones. Whole CTA.
__device__ uint64_t block_radix_select(const uint32_t* keys, int n, int r, int* hist) {
  __shared__ uint32_t s_prefix;
  __shared__ int s_r;
  uint32_t prefix = 0, mask = 0;
  int rr = r;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[d] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const uint32_t k = keys[e];
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // one warp scans 256 bins, 8 per lane
      const int lane = threadIdx.x;
      int c[8], tot = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q] = hist[lane * 8 + q], tot += c[q];
      int incl = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      int run = incl - tot;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (run <= rr && rr < run + c[q]) s_prefix = (uint32_t)(lane * 8 + q), s_r = rr - run;
        run += c[q];
      }
    }
    __syncthreads();
    prefix |= s_prefix << shift;
    mask |= 255u << shift;
    rr = s_r;
    __syncthreads();
  }
  // the top 32 bits (sign, exponent, 20 mantissa bits) of the rank-r key,
  // rounded up: a threshold >= that key, loose by < 2^-20 relative
  return ((uint64_t)prefix << 32) | 0xffffffffull;
}

// Survivor threshold from the sample, in one histogram pass: the keys'
// range [min, max] is cut into <= 4096 bins of width 2^shift (data-adaptive,
// so equal high bytes do not pile onto one bin), and the threshold is the
// top of the bin where the count reaches r + 1. Any threshold is correct
// (every key <= it survives); this one keeps ~(r + 1 + bin load) samples'
// worth of survivors. Whole CTA; every thread gets the 64-bit threshold.
__device__ uint64_t block_sample_threshold(const uint32_t* keys, int n, int r, int* hist, int* hsum, int* wt) {
  __shared__ uint32_t s_min, s_max;
  __shared__ int s_bin;
  if (threadIdx.x == 0) s_min = 0xffffffffu, s_max = 0u, s_bin = 4095;
  __syncthreads();
  uint32_t lo = 0xffffffffu, hi = 0u;
  for (int e = threadIdx.x; e < n; e += blockDim.x) lo = min(lo, keys[e]), hi = max(hi, keys[e]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) atomicMin(&s_min, lo), atomicMax(&s_max, hi);
  for (int d = threadIdx.x; d < 4096; d += blockDim.x) hist[d] = 0;
  __syncthreads();
  const uint32_t kmin = s_min, span = s_max - s_min;
  int shift = 0;
  while ((span >> shift) >= 4096u) ++shift;
  for (int e = threadIdx.x; e < n; e += blockDim.x) atomicAdd(&hist[(keys[e] - kmin) >> shift], 1);
  __syncthreads();
  block_exclusive_scan(hist, hsum, 4096, wt);
  for (int d = threadIdx.x; d < 4096; d += blockDim.x)
    if (hsum[d] <= r && r < hsum[d] + hist[d]) s_bin = d;
  __syncthreads();
  const uint64_t top = (uint64_t)kmin + ((uint64_t)(s_bin + 1) << shift) - 1;
  const uint32_t key32 = top > 0xffffffffull ? 0xffffffffu : (uint32_t)top;
  return ((uint64_t)key32 << 32) | 0xffffffffull;
}

template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(kFastThreads) k_fsel_cost(DevSketch S, DevDevice D, Src src, int64_t n,
                                                            int toggles, int64_t need, double* __restrict__ cost,
                                                            uint32_t* __restrict__ sample, SelState* __restrict__ st,
                                                            int* __restrict__ rank_acc, int* __restrict__ dup,
                                                            int* __restrict__ invalid) {
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* keys = (uint32_t*)smem;  // the last CTA's copy of the sample
  if (blockIdx.x == 0 && threadIdx.x == 0) g_sel_ns[0] = gtimer();
  __shared__ int hist[4096], hsum[4096], wt[32];
  // n / 256 samples, clamped to [4096, 32768]: each sample stands for <= 512
  // candidates, so the rank-r threshold keeps ~(r + 1) * stride survivors
  const int64_t want = n / 256 > kFastCap ? (n / 256 < kSampleMax ? n / 256 : kSampleMax) : kFastCap;
  int64_t stride = 1;  // a power of two: the per-candidate sample test is a mask, not a 64-bit modulo
  while (stride * want < n) stride <<= 1;
  bool bad = false;
  // a contiguous chunk per CTA, so small populations still spread over every
  // SM (the per-candidate fp64 division chains share each SM's fp64 pipe)
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t i_end = (blockIdx.x + 1) * chunk < n ? (blockIdx.x + 1) * chunk : n;
  for (int64_t i = blockIdx.x * chunk + threadIdx.x; i < i_end; i += blockDim.x) {
    Factors<NSP, NRED> F;
    load_cand<NSP, NRED, SEED>(S, src, i, F, false);
    if constexpr (!SEED) bad |= !valid_factors<NSP, NRED>(S, F);
    const double c = draft_cost_of<NSP, NRED>(S, D, F, toggles);
    cost[i] = c;
    if ((i & (stride - 1)) == 0) sample[i / stride] = (uint32_t)(cost_key(c) >> 32);
  }
  // zero the rank kernel's accumulators for this round
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kFastCap; e += gridDim.x * blockDim.x)
    rank_acc[e] = 0, dup[e] = 0;
  if (bad) atomicOr(invalid, 1);
  if (!last_cta(st)) return;
  if (threadIdx.x == 0) g_sel_ns[1] = gtimer();
  const int ns = (int)((n + stride - 1) / stride);
  for (int e = threadIdx.x; e < ns; e += blockDim.x) keys[e] = __ldcg(sample + e);
  __syncthreads();
  // expected survivors ~1.5x need (+3 samples): below need only ~3.5 sigma out
  // (then NEED_MORE and a retry with a larger need)
  int64_t r = (3 * need * ns + 2 * n - 1) / (2 * n) + 3;
  const bool all = r >= ns - 1;
  const uint64_t thr = all ? ~0ull : block_sample_threshold(keys, ns, (int)r, hist, hsum, wt);
  if (threadIdx.x == 0) {
    g_sel_ns[2] = gtimer();
    st->prefix = thr;
    st->shift = 0;
    st->all = all ? 1 : 0;
    st->need = need;
    st->nsurv = 0;
    st->status = 0;
    st->count = 0;
    st->done = 1;
    st->ticket = 0;
  }
}

// 64-bit fingerprint of a schedule's factor columns (explicit populations)
template <int NSP, int NRED>
__device__ __forceinline__ uint64_t fingerprint(const Factors<NSP, NRED>& F) {
  uint64_t h = scramble64((uint64_t)(uint32_t)F.unroll + kGolden);
#pragma unroll
  for (int q = 0; q < Factors<NSP, NRED>::kN; ++q) h = scramble64(h ^ ((uint64_t)(uint32_t)F.f[q] + kGolden));
  return h;
}

template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(256) k_fsel_compact(DevSketch S, Src src, const double* __restrict__ cost,
                                                      int64_t n, SelState* __restrict__ st,
                                                      uint64_t* __restrict__ skey, int64_t* __restrict__ sidx,
                                                      uint64_t* __restrict__ sfp) {
  pdl_wait();
  pdl_trigger();
  const uint64_t thr = st->prefix;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) g_sel_ns[3] = gtimer();
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint64_t key = 0;
    bool keep = false;
    if (i < n) {
      key = cost_key(__ldcg(cost + i));
      keep = key <= thr;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    uint32_t pos0 = 0;
    if (lane == 0) pos0 = atomicAdd(&st->nsurv, (uint32_t)__popc(m));
    pos0 = __shfl_sync(0xffffffffu, pos0, 0);
    if (keep) {
      const uint32_t p = pos0 + __popc(m & ((1u << lane) - 1u));
      if (p < (uint32_t)kFastCap) {
        Factors<NSP, NRED> F;
        const uint64_t id = load_cand<NSP, NRED, SEED>(S, src, i, F, true);
        skey[p] = key, sidx[p] = i;
        sfp[p] = SEED ? id : fingerprint<NSP, NRED>(F);
      }
    }
  }
}

template <int NSP, int NRED, bool SEED>
__device__ __forceinline__ bool same_schedule(const DevSketch& S, const Src& src, int64_t i, int64_t j) {
  if constexpr (SEED) return true;  // seeded fingerprints are exact identities
  Factors<NSP, NRED> Fi, Fj;
  load_cand<NSP, NRED, SEED>(S, src, i, Fi, true);
  load_cand<NSP, NRED, SEED>(S, src, j, Fj, true);
  bool same = Fj.unroll == Fi.unroll;
#pragma unroll
  for (int q = 0; q < Factors<NSP, NRED>::kN; ++q) same &= Fj.f[q] == Fi.f[q];
  return same;
}

template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(kRankChunk) k_fsel_rank(DevSketch S, Src src, const SelState* __restrict__ st,
                                                          const uint64_t* __restrict__ skey,
                                                          const int64_t* __restrict__ sidx,
                                                          const uint64_t* __restrict__ sfp,
                                                          int* __restrict__ rank_acc, int* __restrict__ dup) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint64_t ck[kRankChunk], cf[kRankChunk];
  __shared__ int64_t ci[kRankChunk];
  const int m = (int)min(*(volatile const uint32_t*)&st->nsurv, (uint32_t)kFastCap);
  if (blockIdx.x == 0 && threadIdx.x == 0) g_sel_ns[4] = gtimer();
  const int chunks = (m + kRankChunk - 1) / kRankChunk;
  for (int blk = blockIdx.x; blk < chunks * chunks; blk += gridDim.x) {
    const int ce = blk / chunks, cj = blk - ce * chunks;  // element chunk, comparison chunk
    const int j0 = cj * kRankChunk;
    __syncthreads();
    if (j0 + (int)threadIdx.x < m) {
      ck[threadIdx.x] = skey[j0 + threadIdx.x];
      ci[threadIdx.x] = sidx[j0 + threadIdx.x];
      cf[threadIdx.x] = sfp[j0 + threadIdx.x];
    }
    __syncthreads();
    const int e = ce * kRankChunk + threadIdx.x;
    if (e >= m) continue;
    const uint64_t ke = skey[e], fe = sfp[e];
    const int64_t ie = sidx[e];
    const int jn = min(kRankChunk, m - j0);
    int below = 0;
    bool d = false;
    for (int q = 0; q < jn; ++q) {
      const uint64_t kq = ck[q];
      const int64_t iq = ci[q];
      const bool lt = kq < ke || (kq == ke && iq < ie);
      below += lt;
      if (kq == ke && iq < ie && cf[q] == fe && !d) d = same_schedule<NSP, NRED, SEED>(S, src, ie, iq);
    }
    if (below) atomicAdd(rank_acc + e, below);
    if (d) atomicOr(dup + e, 1);
  }
}

// WITH_ID: also write identities of the emitted entries (sharded rounds);
// a separate instantiation keeps the common kernel's code small.
template <int NSP, int NRED, bool SEED, bool WITH_ID>
__global__ void __launch_bounds__(kFastThreads) k_fsel_emit(DevSketch S, Src src, int64_t n, int64_t k,
                                                            SelState* __restrict__ st,
                                                            const uint64_t* __restrict__ skey,
                                                            const int64_t* __restrict__ sidx,
                                                            const int* __restrict__ rank_acc,
                                                            const int* __restrict__ dup,
                                                            int64_t* __restrict__ out_idx,
                                                            double* __restrict__ out_cost,
                                                            uint64_t* __restrict__ out_id,
                                                            int64_t* __restrict__ out_count) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* a = (uint64_t*)smem;
  int64_t* bi = (int64_t*)(a + kFastCap);
  int* flag = (int*)(bi + kFastCap);
  int* pos = flag + kFastCap;
  __shared__ int wt[32];
  // the survivor count and every survivor slot are read together (one memory
  // round trip): the slot arrays hold kFastCap entries, those >= nsurv unused
  const uint32_t nsurv = st->nsurv;
  int r_[kFastE], d_[kFastE];
  uint64_t k_[kFastE];
  int64_t b_[kFastE];
#pragma unroll
  for (int q = 0; q < kFastE; ++q) {
    const int e = threadIdx.x + q * kFastThreads;
    r_[q] = rank_acc[e], k_[q] = skey[e], b_[q] = sidx[e], d_[q] = dup[e];
  }
  if (threadIdx.x == 0) g_sel_ns[5] = gtimer(), g_sel_ns[7] = nsurv;
  if (nsurv > (uint32_t)kFastCap) {
    if (threadIdx.x == 0) st->status |= TT_SEL_OVERFLOW, *out_count = 0;
    return;
  }
  const int m = (int)nsurv;
  for (int e = threadIdx.x; e < kFastCap; e += blockDim.x) flag[e] = 0;
  __syncthreads();
  if (threadIdx.x == 0) g_sel_ns[8] = gtimer();
#pragma unroll
  for (int q = 0; q < kFastE; ++q) {
    const int e = threadIdx.x + q * kFastThreads;
    if (e < m) {
      const int r = r_[q];  // a permutation of 0..m-1: (cost, index) keys are distinct
      a[r] = k_[q];
      bi[r] = b_[q];
      flag[r] = d_[q] ? 0 : 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) g_sel_ns[9] = gtimer();
  const int total = block_exclusive_scan(flag, pos, kFastCap, wt);
  if (threadIdx.x == 0) g_sel_ns[10] = gtimer();
  for (int e = threadIdx.x; e < m; e += blockDim.x) {
    if (flag[e] && pos[e] < k) {
      const int o = pos[e];
      out_idx[o] = bi[e] + src.index_base;
      out_cost[o] = key_cost(a[e]);
      if constexpr (WITH_ID) out_id[o] = identity_at<NSP, NRED, SEED>(S, src, bi[e]);
    }
  }
  if (threadIdx.x == 0) g_sel_ns[11] = gtimer();
  if (threadIdx.x == 0) {
    const int64_t cnt = total < k ? total : k;
    *out_count = cnt;
    st->count = cnt;
    const bool everything = st->all || (int64_t)m >= n;
    if (cnt < k && !everything) st->status |= TT_SEL_NEED_MORE;  // duplicates ate the margin
    g_sel_ns[6] = gtimer();
  }
}

template <int NSP, int NRED, bool SEED>
static void run_fast(const DevSketch& S, const DevDevice& D, const Src& src, int64_t n, int toggles, int64_t k,
                     int64_t need, SelScratch& w, int64_t* out_idx, double* out_cost, uint64_t* out_id,
                     int64_t* out_count, cudaStream_t st) {
  if (w.k1_ev[0]) cudaEventRecord(w.k1_ev[0], st);
  tt::note_launch();
  static bool init_cost = false;
  if (!init_cost) set_smem(k_fsel_cost<NSP, NRED, SEED>, kSampleMax * sizeof(uint32_t)), init_cost = true;
  k_fsel_cost<NSP, NRED, SEED><<<grid_for(n, 128, 148), kFastThreads, kSampleMax * sizeof(uint32_t), st>>>(S, D, src, n, toggles, need, w.cost, w.sample, w.state,
                                                          w.rank, w.dup, w.invalid);
  if (w.k1_ev[1]) cudaEventRecord(w.k1_ev[1], st);
  tt::note_launch();
  launch_pdl(k_fsel_compact<NSP, NRED, SEED>, dim3(grid_for(n, 256, 148 * 4)), dim3(256), 0, st, S, src, w.cost, n,
             w.state, w.skey, w.sidx, w.sfp);
  tt::note_launch();
  launch_pdl(k_fsel_rank<NSP, NRED, SEED>, dim3(2 * 148), dim3(kRankChunk), 0, st, S, src, w.state, w.skey, w.sidx,
             w.sfp, w.rank, w.dup);
  constexpr size_t emit_smem = (size_t)kFastCap * (2 * sizeof(uint64_t) + 2 * sizeof(int));
  static bool init = false;
  if (!init) set_smem(k_fsel_emit<NSP, NRED, SEED, true>, emit_smem), set_smem(k_fsel_emit<NSP, NRED, SEED, false>, emit_smem), init = true;
  tt::note_launch();
  if (out_id)
    launch_pdl(k_fsel_emit<NSP, NRED, SEED, true>, dim3(1), dim3(kFastThreads), emit_smem, st, S, src, n, k, w.state, w.skey, w.sidx, w.rank, w.dup,
                                                          out_idx, out_cost, out_id, out_count);
  else
    launch_pdl(k_fsel_emit<NSP, NRED, SEED, false>, dim3(1), dim3(kFastThreads), emit_smem, st, S, src, n, k, w.state, w.skey, w.sidx, w.rank, w.dup,
                                                          out_idx, out_cost, out_id, out_count);
}

// ---------------------------------------------- hash fallback (ties) ----
__device__ __forceinline__ uint64_t slot_hash(uint64_t id) { return scramble64(id + kGolden); }

template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(256) k_sel_compact_hash(DevSketch S, Src src, const double* __restrict__ cost,
                                                          int64_t n, SelState* __restrict__ st,
                                                          uint64_t* __restrict__ tkeys, uint64_t* __restrict__ tvals) {
  const SelState s = *st;
  bool overflow = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!survives(cost_key(__ldg(cost + i)), s)) continue;
    const uint64_t id = identity_at<NSP, NRED, SEED>(S, src, i);
    uint64_t h = slot_hash(id) & (kTableCap - 1);
    for (int probes = 0;; ++probes) {
      const uint64_t prev = atomicCAS((unsigned long long*)&tkeys[h], (unsigned long long)kEmpty,
                                      (unsigned long long)id);
      if (prev == kEmpty || prev == id) {
        atomicMin((unsigned long long*)&tvals[h], (unsigned long long)i);
        break;
      }
      h = (h + 1) & (kTableCap - 1);
      if (probes >= kTableCap) {
        overflow = true;
        break;
      }
    }
  }
  if (overflow) atomicOr(&st->status, TT_SEL_OVERFLOW);
}

__global__ void __launch_bounds__(1024) k_sel_finalize_hash(const double* __restrict__ cost, SelState* __restrict__ st,
                                                            uint64_t* __restrict__ tkeys, uint64_t* __restrict__ tvals,
                                                            int64_t k, int64_t n, int64_t index_base,
                                                            int64_t* __restrict__ out_idx,
                                                            double* __restrict__ out_cost,
                                                            uint64_t* __restrict__ out_id,
                                                            int64_t* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  SortSmem sm = carve_sort(smem, kSurvivorCap);
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
    if (e < kSurvivorCap) sm.a[e] = cost_key(cost[idx]), sm.b[e] = idx, sm.c[e] = id;
    else overflow = true;
  }
  __syncthreads();
  const int u = cnt < kSurvivorCap ? cnt : kSurvivorCap;
  // sort key: (cost, index << 12 | collection slot); the slot finds the
  // identity again after the sort
  Key2 kk[kSortE];
#pragma unroll
  for (int e = 0; e < kSortE; ++e) {
    const int p = e * blockDim.x + threadIdx.x;
    kk[e].a = p < u ? sm.a[p] : kEmpty;
    kk[e].b = p < u ? (((uint64_t)sm.b[p]) << 12) | (uint64_t)p : kEmpty;
  }
  __syncthreads();
  block_sort_reg<kSortE, Key2>(kk, sm.xchg);
  const int NT = blockDim.x;
  for (int p = threadIdx.x; p < kSurvivorCap; p += NT) sm.a[p] = sm.c[p];  // identities by slot
  __syncthreads();
#pragma unroll
  for (int e = 0; e < kSortE; ++e) {
    const int p = e * NT + threadIdx.x;
    const bool v = p < u;
    sm.c[p] = v ? sm.a[(int)(kk[e].b & 4095u)] : kEmpty - 1 - (uint64_t)p;
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < kSortE; ++e) {
    const int p = e * NT + threadIdx.x;
    sm.a[p] = kk[e].a;
    sm.b[p] = kk[e].a == kEmpty ? kEmpty : (kk[e].b >> 12);
  }
  __syncthreads();
  dedup_emit(sm.a, sm.b, sm.c, sm.flag, sm.pos, wt, u, kSurvivorCap, k, index_base, out_idx, out_cost, out_id,
             out_count);
  if (threadIdx.x == 0) {
    if (overflow) st->status |= TT_SEL_OVERFLOW;
    else st->status &= ~TT_SEL_OVERFLOW;
    const bool everything = st->all || (int64_t)st->survivors >= n;
    if (u < k && !everything) st->status |= TT_SEL_NEED_MORE;
    else st->status &= ~TT_SEL_NEED_MORE;
    st->count = *out_count;
  }
}

// Cross-rank merge (C1's consumer): R lists of (cost, global index, id).
__global__ void __launch_bounds__(1024) k_merge(const double* __restrict__ cost, const int64_t* __restrict__ gidx,
                                                const uint64_t* __restrict__ id, int m, int64_t k,
                                                int64_t* __restrict__ out_idx, double* __restrict__ out_cost,
                                                uint64_t* __restrict__ out_id, int64_t* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  SortSmem sm = carve_sort(smem, kSurvivorCap);
  __shared__ int wt[32];
  __shared__ int valid;
  if (threadIdx.x == 0) valid = 0;
  __syncthreads();
  Key2 kk[kSortE];
  int mine = 0;
#pragma unroll
  for (int e = 0; e < kSortE; ++e) {
    const int p = e * blockDim.x + threadIdx.x;
    const bool v = p < m && gidx[p] >= 0;  // negative index = empty slot
    // position p in the low 12 bits finds the identity after the sort;
    // global indices < 2^51 keep the (index, p) order = index order
    kk[e].a = v ? cost_key(cost[p]) : kEmpty;
    kk[e].b = v ? (((uint64_t)gidx[p]) << 12) | (uint64_t)p : kEmpty;
    mine += v;
  }
  if (mine) atomicAdd(&valid, mine);
  block_sort_reg<kSortE, Key2>(kk, sm.xchg);
  const int NT = blockDim.x;
#pragma unroll
  for (int e = 0; e < kSortE; ++e) {
    const int p = e * NT + threadIdx.x;
    const bool v = kk[e].a != kEmpty;
    sm.a[p] = kk[e].a;
    sm.b[p] = v ? (kk[e].b >> 12) : kEmpty;
    sm.c[p] = v ? id[kk[e].b & 4095u] : kEmpty - 1 - (uint64_t)p;
  }
  __syncthreads();
  dedup_emit(sm.a, sm.b, sm.c, sm.flag, sm.pos, wt, valid, kSurvivorCap, k, 0, out_idx, out_cost, out_id, out_count);
}

// ------------------------------------------------------------ launchers ----

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
                      cudaStream_t st) {
  const size_t sm = sort_smem_bytes(kFinalCap);
  static bool init = false;
  if (!init) set_smem(k_sel_small<NSP, NRED, SEED>, sm), init = true;
  if (w.k1_ev[0]) cudaEventRecord(w.k1_ev[0], st);  // the whole one-CTA selection stands in for K1
  tt::note_launch();
  k_sel_small<NSP, NRED, SEED><<<1, kFinalCap / kFinalE, sm, st>>>(S, D, src, n, toggles, k, w.state, out_idx,
                                                                   out_cost, out_id, out_count, w.invalid);
  if (w.k1_ev[1]) cudaEventRecord(w.k1_ev[1], st);
}

template <int NSP, int NRED, bool SEED>
static void run_tail(const DevSketch& S, const Src& src, int64_t n, int64_t k, bool hash, SelScratch& w,
                     int64_t* out_idx, double* out_cost, uint64_t* out_id, int64_t* out_count, cudaStream_t st) {
  const size_t sm = sort_smem_bytes(kSurvivorCap);
  const int g = grid_for(n, 256, 148 * 8);
  if (!hash) {
    tt::note_launch();
    k_sel_compact<<<g, 256, 0, st>>>(w.cost, n, w.state, w.skey, w.sidx);
    const size_t smf = sort_smem_bytes(kFinalCap);
    static bool init = false;
    if (!init) set_smem(k_sel_finalize<NSP, NRED, SEED>, smf), init = true;
    tt::note_launch();
    k_sel_finalize<NSP, NRED, SEED><<<1, kFinalCap / kFinalE, smf, st>>>(S, src, w.state, w.skey, w.sidx, k, n,
                                                                         out_idx, out_cost, out_id, out_count);
  } else {
    tt::note_launch();
    k_sel_compact_hash<NSP, NRED, SEED><<<g, 256, 0, st>>>(S, src, w.cost, n, w.state, w.tkeys, w.tvals);
    static bool init = false;
    if (!init) set_smem(k_sel_finalize_hash, sm), init = true;
    tt::note_launch();
    k_sel_finalize_hash<<<1, kSurvivorCap / kSortE, sm, st>>>(w.cost, w.state, w.tkeys, w.tvals, k, n,
                                                              src.index_base, out_idx, out_cost, out_id, out_count);
  }
}

int launch_select(const DevSketch& S, const DevDevice& D, const int32_t* soa, int64_t ld, uint64_t s0,
                  int64_t first, bool seeded, int64_t n, int64_t k, int64_t need, int toggles,
                  int64_t index_base, SelScratch& w, int64_t* out_idx, double* out_cost, uint64_t* out_id,
                  int64_t* out_count, cudaStream_t st, bool hash) {
  Src src{soa, ld, s0, first, index_base};
  if (n <= kSmallSelectMax) {
    if (seeded)
      return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_small<NSP, NRED, true>(S, D, src, n, toggles, k, w, out_idx, out_cost, out_id, out_count, st)));
    return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_small<NSP, NRED, false>(S, D, src, n, toggles, k, w, out_idx, out_cost, out_id, out_count, st)));
  }
  // the sampled threshold keeps ~(r + 1) * n / ns survivors: within the 4096-entry
  // cap up to ~16M candidates; larger populations use the histogram path
  if (!hash && n <= kFastMaxN) {
    if (seeded)
      return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_fast<NSP, NRED, true>(S, D, src, n, toggles, k, need, w, out_idx, out_cost, out_id, out_count, st)));
    return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_fast<NSP, NRED, false>(S, D, src, n, toggles, k, need, w, out_idx, out_cost, out_id, out_count, st)));
  }
  {
    if (w.k1_ev[0]) cudaEventRecord(w.k1_ev[0], st);
    int rc = launch_draft_cost(S, D, soa, ld, s0, first, seeded, n, toggles, w.cost, w.hist, w.invalid, st);
    if (w.k1_ev[1]) cudaEventRecord(w.k1_ev[1], st);
    if (rc) return rc;
  }
  tt::note_launch();
  k_sel_scan<<<1, 1024, 0, st>>>(w.hist, w.state, need, 0);
  for (int lv = 1; lv <= 2; ++lv) {
    const int g = grid_for(n, 256, 148 * 8);
    tt::note_launch();
    k_sel_refine<<<g, 256, 0, st>>>(w.cost, n, w.state, w.hist);
    tt::note_launch();
    k_sel_scan<<<1, 1024, 0, st>>>(w.hist, w.state, need, lv);
  }
  if (seeded)
    return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_tail<NSP, NRED, true>(S, src, n, k, hash, w, out_idx, out_cost, out_id, out_count, st)));
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (run_tail<NSP, NRED, false>(S, src, n, k, hash, w, out_idx, out_cost, out_id, out_count, st)));
}

// Identities of the drafted set (positions [0, *count)), written to id[].
// Runs on the context's side stream, overlapped with features + PaCM: the
// exact identity (mixed-radix composition ranks) is a long serial chain per
// candidate and only the b selections' identities are reported.
template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(128) k_drafted_identity(DevSketch S, Src src, const int64_t* __restrict__ idx,
                                                          const int64_t* __restrict__ count_dev, int64_t k_max,
                                                          uint64_t* __restrict__ out) {
  const int64_t cnt = count_dev ? (*count_dev < k_max ? *count_dev : k_max) : k_max;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < cnt; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = identity_at<NSP, NRED, SEED>(S, src, idx[p] - src.index_base);
}

int launch_drafted_identity(const DevSketch& S, const int32_t* soa, int64_t ld, uint64_t s0, int64_t first,
                            bool seeded, const int64_t* idx, const int64_t* count_dev, int64_t k_max, uint64_t* out,
                            cudaStream_t st) {
  if (k_max <= 0) return 0;
  Src src{soa, ld, s0, first, first};
  const int g = grid_for(k_max, 128, 148);
  if (seeded)
    return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_drafted_identity<NSP, NRED, true><<<g, 128, 0, st>>>(S, src, idx, count_dev, k_max, out)));
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_drafted_identity<NSP, NRED, false><<<g, 128, 0, st>>>(S, src, idx, count_dev, k_max, out)));
}

int launch_merge(const double* cost, const int64_t* gidx, const uint64_t* id, int m, int64_t k, int64_t* out_idx,
                 double* out_cost, uint64_t* out_id, int64_t* out_count, cudaStream_t st) {
  if (m > kSurvivorCap) return -1;
  const size_t sm = sort_smem_bytes(kSurvivorCap);
  static bool init = false;
  if (!init) set_smem(k_merge, sm), init = true;
  tt::note_launch();
  k_merge<<<1, kSurvivorCap / kSortE, sm, st>>>(cost, gidx, id, m, k, out_idx, out_cost, out_id, out_count);
  return 0;
}

}  // namespace tt

extern "C" int ttdbg_select_clocks(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_sel_ns, sizeof(unsigned long long) * (n < 12 ? n : 12));
}
