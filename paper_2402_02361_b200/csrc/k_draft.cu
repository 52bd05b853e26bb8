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
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include <cooperative_groups.h>

#include "tt_block.cuh"
#include "tt_device.cuh"
#include "tt_kernels.h"

namespace cg = cooperative_groups;

namespace tt {

constexpr int kHistBins = 4096;
constexpr int kSurvivorTarget = 1024;  // refine while more keys survive
constexpr int kFinalCap = 1024;        // survivors the (append-path) finaliser sorts
constexpr int kSurvivorCap = 4096;     // entries the hash-path finaliser / merge sort
constexpr int kTableCap = 16384;       // hash slots of the fallback path
constexpr int kSortE = 4;              // keys per thread in the 4096-entry sorts
constexpr int kFinalE = 1;             // keys per thread in the 1024-entry sorts (1024 threads)
constexpr uint64_t kEmpty = ~0ull;
constexpr int kFastCap = 8192;               // survivors the fast path ranks
constexpr int kSampleMin = 4096;             // sampled cost keys (top 32 bits) for the threshold
constexpr int kSampleMax = 32768;
constexpr int64_t kFastMaxN = int64_t{16} << 20;  // fast path population limit
constexpr int kL2TabMax = kSampleMax * 4 / 8;      // p_l2_m table entries (overlays the sample)
constexpr int64_t kL2TabMinChunk = 4 * 1024;         // candidates per CTA that amortise filling it

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
// N > 1024: ONE cooperative kernel (one 1024-thread CTA per SM, grid-wide
// barriers between phases; no CTA-wide sorting network and no host round
// trip):
//   A  K1 over the population (a contiguous chunk per CTA), costs to HBM and
//      a strided sample of 4096..32768 cost keys (top 32 bits).
//   B  every CTA loads the whole sample and computes the same survivor
//      threshold: the sample key of rank ceil(1.5 need ns / n) + 3 (~1.5x
//      need survivors expected).
//   C  keys <= threshold appended (warp-aggregated) with a schedule
//      fingerprint (seeded: the exact identity the generator returns;
//      explicit: a 64-bit hash of the factor columns, confirmed column by
//      column on a match).
//   D  all-pairs over the <= 8192 survivors in 32 x 32 blocks, one per warp,
//      spread over the GPU: each survivor counts the keys below it ((cost,
//      index) order) and flags a duplicate when an equal-cost survivor with a
//      lower index is the same schedule ("first discovery wins",
//      draft.cpp:200-203).
//      Too few unique survivors (duplicates ate the margin): need doubles and
//      B-D repeat over the costs already in HBM (K1 is never re-run).
//   E  the CTAs holding survivors write the K lowest unique in ascending
//      (cost, index) order: position = rank - duplicates ranked below.
// Exactness never depends on the sample: every key <= threshold survives,
// so whenever >= K unique schedules survive they include the true top-K;
// > 8192 survivors (or no convergence) report OVERFLOW and the host takes
// the identity-keyed hash path.
constexpr int kFastThreads = 1024;
constexpr int kMaxAttempts = 8;

// %globaltimer marks (ns) of the fused selector's phases (CTA 0), read by
// ttdbg_select_clocks (tools/probe_select.py): [0] start, [1] K1 done (all
// CTAs), [2] threshold, [3] compact done, [4] rank done, [5] emit done,
// [6] survivors, [7] attempts; [8 + 2b] CTA 0's arrival at barrier b,
// [9 + 2b] the latest arrival (first attempt)

__device__ unsigned long long g_sel_ns[24];
// timeline ring of the last 64 selector launches: [start, emit end]
__device__ unsigned long long g_tl[64][2];
__device__ unsigned g_tl_n[1];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Grid-wide barrier of the cooperative launch (every CTA co-resident):
// cooperative_groups' grid sync, 1.25 us on B200 at 148 CTAs against 2.3 us
// for an atomic generation counter polled by one thread per CTA
// (tools/barrier_bench.cu). mark >= 0 records CTA 0's arrival and the latest
// arrival (probe).
__device__ __forceinline__ void grid_barrier(int mark = -1) {
  if (mark >= 0 && threadIdx.x == 0) {
    const unsigned long long now = gtimer();
    if (blockIdx.x == 0) g_sel_ns[8 + 2 * mark] = now;
    atomicMax(&g_sel_ns[9 + 2 * mark], now);
  }
  cg::this_grid().sync();
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

// 64-bit fingerprint of a schedule's factor columns (explicit populations)
template <int NSP, int NRED>
__device__ __forceinline__ uint64_t fingerprint(const Factors<NSP, NRED>& F) {
  uint64_t h = scramble64((uint64_t)(uint32_t)F.unroll + kGolden);
#pragma unroll
  for (int q = 0; q < Factors<NSP, NRED>::kN; ++q) h = scramble64(h ^ ((uint64_t)(uint32_t)F.f[q] + kGolden));
  return h;
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

template <int NSP, int NRED, bool SEED, bool WITH_ID, bool U32 = false>
__global__ void __launch_bounds__(kFastThreads, 1)
    k_fsel(DevSketch S, DevDevice D, Src src, int64_t n, int toggles, int64_t k, int64_t need,
           double* __restrict__ cost, uint32_t* __restrict__ sample, SelState* __restrict__ st,
           uint64_t* __restrict__ skey, int64_t* __restrict__ sidx, uint64_t* __restrict__ sfp,
           int* __restrict__ rank_acc, int* __restrict__ dup, int* __restrict__ invalid,
           int64_t* __restrict__ out_idx, double* __restrict__ out_cost, uint64_t* __restrict__ out_id,
           int64_t* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* keys = (uint32_t*)smem;  // the whole sample, every CTA
  __shared__ int hist[4096], hsum[4096], wt[32];
  __shared__ uint32_t dmask[kFastCap / 32];
  __shared__ int dcnt[kFastCap / 32], dpre[kFastCap / 32];
  const int t = threadIdx.x;
  if (blockIdx.x == 0 && t == 0) {
    g_sel_ns[0] = gtimer();
    for (int q = 9; q < 16; q += 2) g_sel_ns[q] = 0;
    const unsigned r = atomicAdd(&g_tl_n[0], 1u) & 63u;  // timeline ring (tools/probe_round_timeline.py)
    g_tl[r][0] = g_sel_ns[0];
  }
  // n / 256 samples, clamped to [4096, 32768]: each sample stands for <= 512
  // candidates, so the rank-r threshold keeps ~(r + 1) * stride survivors
  const int64_t want = n / 256 > kSampleMin ? (n / 256 < kSampleMax ? n / 256 : kSampleMax) : kSampleMin;
  int64_t stride = 1;  // a power of two: the per-candidate sample test is a mask
  while (stride * want < n) stride <<= 1;
  // ---- A: K1, a contiguous chunk per CTA (small populations still spread
  // over every SM: the per-candidate fp64 division chains share each SM's pipe)
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t i_beg = blockIdx.x * chunk;
  const int64_t i_end = i_beg + chunk < n ? i_beg + chunk : n;
  bool bad = false;
  // large chunks: p_l2_m from a table in the (not yet used) sample region
  // instead of three divisions per GEMM candidate; the sample overwrites it
  // after the grid barrier
  double* l2tab = (double*)smem;
  int n_tab = 0;
  if (i_end - i_beg >= kL2TabMinChunk) {
    int64_t mx = 0;
    for (int a = 0; a < S.n_axes; ++a) mx = S.extent[a] > mx ? S.extent[a] : mx;
    n_tab = (int)(mx + 1 < kL2TabMax ? mx + 1 : kL2TabMax);
    l2m_table_fill(l2tab, n_tab, D);
    __syncthreads();
  }
  for (int64_t i = i_beg + t; i < i_end; i += blockDim.x) {
    Factors<NSP, NRED> F;
    load_cand<NSP, NRED, SEED>(S, src, i, F, false);
    if constexpr (!SEED) bad |= !valid_factors<NSP, NRED>(S, F);
    const double c = draft_cost_of<NSP, NRED, false, std::conditional_t<U32, uint32_t, int64_t>>(S, D, F, toggles,
                                                                                                   l2tab, n_tab);
    cost[i] = c;
    if ((i & (stride - 1)) == 0) sample[i / stride] = (uint32_t)(cost_key(c) >> 32);
  }
  for (int e = blockIdx.x * blockDim.x + t; e < kFastCap; e += gridDim.x * blockDim.x) rank_acc[e] = 0, dup[e] = 0;
  if (blockIdx.x == 0 && t < kMaxAttempts) st->att_surv[t] = 0, st->att_dup[t] = 0;
  if (bad) atomicOr(invalid, 1);
  grid_barrier(0);
  if (blockIdx.x == 0 && t == 0) g_sel_ns[1] = gtimer();
  // ---- B: the sample, every CTA
  const int ns = (int)((n + stride - 1) / stride);
  for (int e0 = t; e0 < ns; e0 += 8 * blockDim.x) {  // eight loads in flight, then the stores
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * (int)blockDim.x;
      v[u] = e < ns ? __ldcg(sample + e) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * (int)blockDim.x;
      if (e < ns) keys[e] = v[u];
    }
  }
  __syncthreads();
  const int lane = t & 31;
  int status = 0, attempt = 0, m = 0, uniq = 0;
  bool all = false;
  for (;; ++attempt) {
    // expected survivors ~1.5x need (+3 samples): below need only ~3.5 sigma out
    const int64_t r = (3 * need * ns + 2 * n - 1) / (2 * n) + 3;
    all = r >= ns - 1;
    if (blockIdx.x == 0 && t == 0) g_sel_ns[19] = gtimer();
    const uint64_t thr = all ? ~0ull : block_sample_threshold(keys, ns, (int)r, hist, hsum, wt);
    if (blockIdx.x == 0 && t == 0) g_sel_ns[2] = gtimer();
    if (attempt > 0)
      for (int e = blockIdx.x * blockDim.x + t; e < kFastCap; e += gridDim.x * blockDim.x) rank_acc[e] = 0, dup[e] = 0;
    // ---- C: compact this CTA's chunk (its costs are still in L2)
    uint32_t* surv = &st->att_surv[attempt];
    auto visit = [&](int64_t i, uint64_t key) {  // warp-uniform call
      const bool keep = i < i_end && key <= thr;
      const unsigned msk = __ballot_sync(0xffffffffu, keep);
      if (!msk) return;
      uint32_t pos0 = 0;
      if (lane == 0) pos0 = atomicAdd(surv, (uint32_t)__popc(msk));
      pos0 = __shfl_sync(0xffffffffu, pos0, 0);
      if (keep) {
        const uint32_t p = pos0 + __popc(msk & ((1u << lane) - 1u));
        if (p < (uint32_t)kFastCap) {
          Factors<NSP, NRED> F;
          const uint64_t id = load_cand<NSP, NRED, SEED>(S, src, i, F, true);
          skey[p] = key, sidx[p] = i;
          sfp[p] = SEED ? id : fingerprint<NSP, NRED>(F);
        }
      }
    };
    if (n <= ((int64_t)6 << 20)) {  // the cost array (<= 48 MB) is still in L2 from K1
      for (int64_t base = i_beg; base < i_end; base += blockDim.x) {
        const int64_t i = base + t;
        visit(i, i < i_end ? cost_key(__ldcg(cost + i)) : 0ull);
      }
    } else {
      // larger cost arrays stream from HBM: kCompactU cost loads in flight per
      // thread (one load per round trip is latency bound); survivor positions
      // come from an atomic, so the scan order does not matter
      constexpr int kCompactU = 8;
      for (int64_t base = i_beg; base < i_end; base += (int64_t)kCompactU * blockDim.x) {
        uint64_t kv[kCompactU];
#pragma unroll
        for (int u = 0; u < kCompactU; ++u) {
          const int64_t i = base + (int64_t)u * blockDim.x + t;
          kv[u] = i < i_end ? cost_key(__ldcg(cost + i)) : 0ull;
        }
#pragma unroll 1
        for (int u = 0; u < kCompactU; ++u) visit(base + (int64_t)u * blockDim.x + t, kv[u]);
      }
    }
    grid_barrier(attempt == 0 ? 1 : -1);
    if (blockIdx.x == 0 && t == 0) g_sel_ns[3] = gtimer();
    const uint32_t m_raw = *(volatile uint32_t*)surv;
    if (m_raw > (uint32_t)kFastCap) {
      status = TT_SEL_OVERFLOW;
      break;
    }
    m = (int)m_raw;
    // ---- D: all-pairs ranking in 32 x 32 blocks, one per warp (comparison
    // keys broadcast by shuffles); block b runs on CTA b % grid, warp b / grid,
    // so every SM takes one block before any takes two
    {
      const int warp = t >> 5;
      const int chunks = (m + 31) >> 5;
      for (int blk = warp * gridDim.x + blockIdx.x; blk < chunks * chunks; blk += gridDim.x * (kFastThreads / 32)) {
        const int ce = blk / chunks, cj = blk - ce * chunks;  // element chunk, comparison chunk
        const int e = ce * 32 + lane, j = cj * 32 + lane;
        const bool ev = e < m;
        const uint64_t ke = ev ? __ldcg(skey + e) : ~0ull, fe = ev ? __ldcg(sfp + e) : 0;
        const int64_t ie = ev ? __ldcg(sidx + e) : -1;
        const uint64_t kj = j < m ? __ldcg(skey + j) : ~0ull, fj = j < m ? __ldcg(sfp + j) : 0;
        const int64_t ij = j < m ? __ldcg(sidx + j) : INT64_MAX;
        const int jn = min(32, m - cj * 32);
        int below = 0;
        bool d = false;
        for (int q = 0; q < jn; ++q) {
          const uint64_t kq = __shfl_sync(0xffffffffu, kj, q);
          const int64_t iq = __shfl_sync(0xffffffffu, ij, q);
          const uint64_t fq = __shfl_sync(0xffffffffu, fj, q);
          const bool lt_ = kq < ke || (kq == ke && iq < ie);
          below += lt_;
          if (ev && kq == ke && iq < ie && fq == fe && !d) d = same_schedule<NSP, NRED, SEED>(S, src, ie, iq);
        }
        if (ev && below) atomicAdd(rank_acc + e, below);
        if (ev && d && atomicOr(dup + e, 1) == 0) atomicAdd(&st->att_dup[attempt], 1u);
      }
    }
    grid_barrier(attempt == 0 ? 2 : -1);
    if (blockIdx.x == 0 && t == 0) g_sel_ns[4] = gtimer();
    uniq = m - (int)*(volatile uint32_t*)&st->att_dup[attempt];
    const bool everything = all || (int64_t)m >= n;
    if (uniq >= k || everything) break;
    if (attempt + 1 == kMaxAttempts) {  // no convergence: the host takes the hash path
      status = TT_SEL_OVERFLOW;
      break;
    }
    need *= 2;  // duplicates ate the margin: a looser threshold over the same costs
  }
  if (status) {
    if (blockIdx.x == 0 && t == 0) {
      st->status = status;
      st->count = 0;
      *out_count = 0;
      if constexpr (WITH_ID) out_idx[0] = kRankFailed;  // sharded: the merge reports it on every rank
      g_sel_ns[5] = gtimer(), g_sel_ns[6] = m, g_sel_ns[7] = attempt + 1;
    }
    return;
  }
  // the dependent verify kernel may launch now (its weight copies overlap the emit)
  pdl_trigger();
  // ---- E: emit. Position of a unique survivor = its rank minus the
  // duplicates ranked below it (a bitmap over ranks, prefix popcounts).
  if (blockIdx.x > 0 && (int64_t)blockIdx.x * blockDim.x >= m) return;
  if (blockIdx.x == 0 && t == 0) g_sel_ns[16] = gtimer();
  // this thread's survivor, loaded up front (its L2 round trips overlap the
  // duplicate bitmap and the scan instead of following them)
  const int e = blockIdx.x * blockDim.x + t;
  int e_dup = 1, e_rank = 0;
  int64_t e_idx = 0;
  uint64_t e_key = 0;
  if (e < m) e_dup = __ldcg(dup + e), e_rank = __ldcg(rank_acc + e), e_idx = __ldcg(sidx + e), e_key = __ldcg(skey + e);
  for (int w = t; w < kFastCap / 32; w += blockDim.x) dmask[w] = 0;
  __syncthreads();
  for (int e = t; e < m; e += blockDim.x)
    if (__ldcg(dup + e)) {
      const int r = __ldcg(rank_acc + e);
      atomicOr(&dmask[r >> 5], 1u << (r & 31));
    }
  __syncthreads();
  if (blockIdx.x == 0 && t == 0) g_sel_ns[17] = gtimer();
  for (int w = t; w < kFastCap / 32; w += blockDim.x) dcnt[w] = __popc(dmask[w]);
  __syncthreads();
  block_exclusive_scan(dcnt, dpre, kFastCap / 32, wt);
  __syncthreads();
  if (blockIdx.x == 0 && t == 0) g_sel_ns[18] = gtimer();
  if (e < m && !e_dup) {
    const int r = e_rank;
    const int o = r - (dpre[r >> 5] + __popc(dmask[r >> 5] & ((1u << (r & 31)) - 1u)));
    if (o < k) {
      const int64_t i = e_idx;
      out_idx[o] = i + src.index_base;
      out_cost[o] = key_cost(e_key);
      if constexpr (WITH_ID) out_id[o] = SEED ? __ldcg(sfp + e) : identity_at<NSP, NRED, SEED>(S, src, i);
    }
  }
  if (blockIdx.x == 0 && t == 0) {
    const int64_t cnt = uniq < k ? uniq : k;
    *out_count = cnt;
    st->count = cnt;
    st->status = 0;
    st->all = all ? 1 : 0;
    st->need = need;
    g_sel_ns[5] = gtimer(), g_sel_ns[6] = m, g_sel_ns[7] = attempt + 1;
    g_tl[(g_tl_n[0] - 1u) & 63u][1] = g_sel_ns[5];
  }
}

static int g_num_sms = 0;


template <int NSP, int NRED, bool SEED>
static void run_fast(const DevSketch& S, const DevDevice& D, const Src& src, int64_t n, int toggles, int64_t k,
                     int64_t need, SelScratch& w, int64_t* out_idx, double* out_cost, uint64_t* out_id,
                     int64_t* out_count, cudaStream_t st) {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  constexpr size_t smem = kSampleMax * sizeof(uint32_t);
  static bool init = false;
  if (!init) {
    set_smem(k_fsel<NSP, NRED, SEED, true>, smem), set_smem(k_fsel<NSP, NRED, SEED, false>, smem);
    set_smem(k_fsel<NSP, NRED, SEED, false, true>, smem), set_smem(k_fsel<NSP, NRED, SEED, true, true>, smem);
    init = true;
  }
  // one CTA per SM (co-resident: a cooperative launch), >= 64 candidates each
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(g_num_sms, n / 64));
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeCooperative;
  attr.val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid), cfg.blockDim = dim3(kFastThreads), cfg.dynamicSmemBytes = smem, cfg.stream = st;
  cfg.attrs = &attr, cfg.numAttrs = 1;
  if (w.k1_ev[0]) cudaEventRecord(w.k1_ev[0], st);
  tt::note_launch();
  const bool u32 = fits_u32(S, D);
  if (out_id && u32)
    cudaLaunchKernelEx(&cfg, k_fsel<NSP, NRED, SEED, true, true>, S, D, src, n, toggles, k, need, w.cost, w.sample,
                       w.state, w.skey, w.sidx, w.sfp, w.rank, w.dup, w.invalid, out_idx, out_cost, out_id,
                       out_count);
  else if (out_id)
    cudaLaunchKernelEx(&cfg, k_fsel<NSP, NRED, SEED, true>, S, D, src, n, toggles, k, need, w.cost, w.sample, w.state,
                       w.skey, w.sidx, w.sfp, w.rank, w.dup, w.invalid, out_idx, out_cost, out_id, out_count);
  else if (u32)
    cudaLaunchKernelEx(&cfg, k_fsel<NSP, NRED, SEED, false, true>, S, D, src, n, toggles, k, need, w.cost, w.sample,
                       w.state, w.skey, w.sidx, w.sfp, w.rank, w.dup, w.invalid, out_idx, out_cost, out_id,
                       out_count);
  else
    cudaLaunchKernelEx(&cfg, k_fsel<NSP, NRED, SEED, false>, S, D, src, n, toggles, k, need, w.cost, w.sample,
                       w.state, w.skey, w.sidx, w.sfp, w.rank, w.dup, w.invalid, out_idx, out_cost, out_id,
                       out_count);
  if (w.k1_ev[1]) cudaEventRecord(w.k1_ev[1], st);
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
                                                uint64_t* __restrict__ out_id, int64_t* __restrict__ out_count,
                                                SelState* __restrict__ st) {
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
    if (st && p < m && gidx[p] == kRankFailed) atomicOr(&st->status, TT_SEL_OVERFLOW);
    if (st && p < m && gidx[p] == kRankInvalid) atomicOr(&st->status, TT_SEL_INVALID);
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

// Merge of R = m / k per-rank lists, each ascending by (cost key, global
// index) with its valid entries first (what tt_round_local_async emits):
// m up to kMergeMax, beyond the one-CTA sort. Global indices are disjoint
// across ranks, so (cost, index) keys are distinct and an entry's merged rank
// is its own list position plus, for every other list, the number of that
// list's entries below it. CTA (r, q) stages list q in shared memory and
// binary-searches it for every entry of list r; an entry is a duplicate when
// an equal-cost entry of another list with a lower index carries the same
// identity (same schedule => same cost). Within a list entries are unique.
constexpr int kMergeListMax = 8192;  // entries per list staged in shared memory

__global__ void __launch_bounds__(512) k_merge_rank(const double* __restrict__ cost, const int64_t* __restrict__ gidx,
                                                    const uint64_t* __restrict__ id, int R, int64_t k,
                                                    int32_t* __restrict__ rank, int32_t* __restrict__ dup,
                                                    SelState* __restrict__ st) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* qk = (uint64_t*)smem;  // list q: cost keys
  int64_t* qi = (int64_t*)(qk + k);  // list q: global indices
  __shared__ int lq;
  const int r = blockIdx.x / R, q = blockIdx.x - (blockIdx.x / R) * R;
  const int64_t* gq = gidx + (int64_t)q * k;
  const int64_t* gr = gidx + (int64_t)r * k;
  if (threadIdx.x == 0) lq = (int)k;
  __syncthreads();
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const int64_t g = gq[j];
    qk[j] = cost_key(cost[(int64_t)q * k + j]);
    qi[j] = g;
    if (g < 0 && (j == 0 || gq[j - 1] >= 0)) lq = (int)j;  // the first empty slot
  }
  if (st && q == r && threadIdx.x == 0 && gr[0] == kRankFailed) atomicOr(&st->status, TT_SEL_OVERFLOW);
  if (st && q == r && threadIdx.x == 0 && gr[0] == kRankInvalid) atomicOr(&st->status, TT_SEL_INVALID);
  __syncthreads();
  const int L = lq;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const int64_t ge = gr[j];
    if (ge < 0) continue;
    const int64_t e = (int64_t)r * k + j;
    if (q == r) {  // own list: its position
      atomicAdd(rank + e, (int)j);
      continue;
    }
    const uint64_t ke = cost_key(cost[e]);
    int lo = 0, hi = L;  // first position with (key, index) >= (ke, ge)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const bool below = qk[mid] < ke || (qk[mid] == ke && qi[mid] < ge);
      if (below) lo = mid + 1;
      else hi = mid;
    }
    if (lo) atomicAdd(rank + e, lo);
    // equal-cost entries of list q with a lower index, nearest first
    const uint64_t ie = id[e];
    for (int p = lo - 1; p >= 0 && qk[p] == ke; --p)
      if (id[(int64_t)q * k + p] == ie) {
        atomicOr(dup + e, 1);
        break;
      }
  }
}

// Scatter to merged order and emit the first kout non-duplicates (one CTA;
// merged positions are walked in chunks until kout entries are out).
__global__ void __launch_bounds__(1024) k_merge_emit(const double* __restrict__ cost, const int64_t* __restrict__ gidx,
                                                     const uint64_t* __restrict__ id, int64_t m, int64_t kout,
                                                     const int32_t* __restrict__ rank, const int32_t* __restrict__ dup,
                                                     int32_t* __restrict__ ord, int64_t* __restrict__ out_idx,
                                                     double* __restrict__ out_cost, uint64_t* __restrict__ out_id,
                                                     int64_t* __restrict__ out_count) {
  __shared__ int flag[1024], pos[1024], wt[32], nvalid;
  if (threadIdx.x == 0) nvalid = 0;
  __syncthreads();
  int mine = 0;
  for (int64_t e = threadIdx.x; e < m; e += blockDim.x)
    if (gidx[e] >= 0) ord[rank[e]] = (int32_t)e, ++mine;
  if (mine) atomicAdd(&nvalid, mine);
  __threadfence_block();
  __syncthreads();
  const int M = nvalid;
  int64_t done = 0;
  for (int base = 0; base < M && done < kout; base += blockDim.x) {
    const int p = base + threadIdx.x;
    const int e = p < M ? ord[p] : -1;
    flag[threadIdx.x] = e >= 0 && !dup[e];
    __syncthreads();
    const int tot = block_exclusive_scan(flag, pos, blockDim.x, wt);
    if (e >= 0 && flag[threadIdx.x] && done + pos[threadIdx.x] < kout) {
      const int64_t o = done + pos[threadIdx.x];
      out_idx[o] = gidx[e];
      out_cost[o] = cost[e];
      if (out_id) out_id[o] = id[e];
    }
    done += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_count = done < kout ? done : kout;
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
// sync (optional, the fused verify's handshake): sync[1] block ticket, sync[2]
// completed-kernel epoch, advanced once every identity is written.
template <int NSP, int NRED, bool SEED>
__global__ void __launch_bounds__(128) k_drafted_identity(DevSketch S, Src src, const int64_t* __restrict__ idx,
                                                          const int64_t* __restrict__ count_dev, int64_t k_max,
                                                          uint64_t* __restrict__ out, unsigned* __restrict__ sync) {
  const int64_t cnt = count_dev ? (*count_dev < k_max ? *count_dev : k_max) : k_max;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < cnt; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = identity_at<NSP, NRED, SEED>(S, src, idx[p] - src.index_base);
  if (!sync) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(&sync[1], 1u) == gridDim.x - 1) {
    sync[1] = 0u;
    __threadfence();
    atomicAdd(&sync[2], 1u);
  }
}

int launch_drafted_identity(const DevSketch& S, const int32_t* soa, int64_t ld, uint64_t s0, int64_t first,
                            bool seeded, const int64_t* idx, const int64_t* count_dev, int64_t k_max, uint64_t* out,
                            cudaStream_t st, unsigned* sync) {
  if (k_max <= 0) return 0;
  Src src{soa, ld, s0, first, first};
  const int g = grid_for(k_max, 128, 148);
  if (seeded)
    return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_drafted_identity<NSP, NRED, true><<<g, 128, 0, st>>>(S, src, idx, count_dev, k_max, out, sync)));
  return TT_DISPATCH_SHAPE(S.n_sp, S.n_red, (tt::note_launch(), k_drafted_identity<NSP, NRED, false><<<g, 128, 0, st>>>(S, src, idx, count_dev, k_max, out, sync)));
}

__global__ void k_mark_invalid(int* __restrict__ invalid, int64_t* __restrict__ out_idx) {
  if (*invalid) out_idx[0] = kRankInvalid, *invalid = 0;  // the flag is zero between calls
}

int launch_mark_invalid(int* invalid, int64_t* out_idx, cudaStream_t st) {
  k_mark_invalid<<<1, 1, 0, st>>>(invalid, out_idx);
  return cudaGetLastError() != cudaSuccess;
}

int launch_merge(const double* cost, const int64_t* gidx, const uint64_t* id, int64_t m, int64_t k, int64_t* out_idx,
                 double* out_cost, uint64_t* out_id, int64_t* out_count, SelState* state, int32_t* scratch,
                 cudaStream_t st) {
  if (m <= kSurvivorCap) {
    const size_t sm = sort_smem_bytes(kSurvivorCap);
    static bool init = false;
    if (!init) set_smem(k_merge, sm), init = true;
    tt::note_launch();
    k_merge<<<1, kSurvivorCap / kSortE, sm, st>>>(cost, gidx, id, (int)m, k, out_idx, out_cost, out_id, out_count,
                                                  state);
    return 0;
  }
  if (m > kMergeMax || k < 1 || k > kMergeListMax || m % k) return -1;
  const int R = (int)(m / k);
  int32_t* rank = scratch;
  int32_t* dup = scratch + m;
  if (cudaMemsetAsync(scratch, 0, sizeof(int32_t) * 2 * m, st) != cudaSuccess) return -1;
  const size_t sm = (size_t)k * 16;
  static bool init = false;
  if (!init) set_smem(k_merge_rank, (size_t)kMergeListMax * 16), init = true;
  tt::note_launch();
  k_merge_rank<<<R * R, 512, sm, st>>>(cost, gidx, id, R, k, rank, dup, state);
  // merged order reuses the duplicate flags' successor: ord lives after rank/dup
  tt::note_launch();
  k_merge_emit<<<1, 1024, 0, st>>>(cost, gidx, id, m, k, rank, dup, scratch + 2 * m, out_idx, out_cost, out_id,
                                   out_count);
  return 0;
}

}  // namespace tt

extern "C" int ttdbg_select_timeline(unsigned long long* out, unsigned* n) {
  int rc = (int)cudaMemcpyFromSymbol(out, tt::g_tl, sizeof(unsigned long long) * 128);
  return rc ? rc : (int)cudaMemcpyFromSymbol(n, tt::g_tl_n, sizeof(unsigned));
}
extern "C" int ttdbg_select_clocks(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, tt::g_sel_ns, sizeof(unsigned long long) * (n < 24 ? n : 24));
}

// ttdbg_div_check (tests/test_gpu_parity.py): ddiv_inrange against
// __ddiv_rn over n pseudo-random operand pairs per kind — 0: integers in
// [1, 2^32), 1: an integer over a double in [2^-400, 2^400] (the draft
// cost's s5 / u_m shape), 2: both doubles in [2^-400, 2^400], 3: integers
// whose quotient is near 1 (round-up ratios). Returns the mismatch count
// (0 expected), or -1 on a CUDA error.
namespace tt {
__global__ void k_div_check(int64_t n, uint64_t seed, unsigned long long* bad) {
  unsigned long long my = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = scramble64(seed + 2 * (uint64_t)i * kGolden), y = scramble64(seed + (2 * (uint64_t)i + 1) * kGolden);
    const auto dbl = [](uint64_t r) {  // exponent in [-400, 400], random mantissa
      const int e = (int)((r >> 52) % 801) - 400;
      return __longlong_as_double((long long)(((uint64_t)(e + 1023) << 52) | (r & ((1ull << 52) - 1))));
    };
    double a, b;
    switch (i & 3) {
      case 0: a = (double)((x >> 32) | 1), b = (double)((y >> 32) | 1); break;
      case 1: a = (double)((x >> 32) | 1), b = dbl(y); break;
      case 2: a = dbl(x), b = dbl(y); break;
      default: {
        const uint32_t s = (uint32_t)(x >> 33) | 1u, d = (uint32_t)(y % 64) + 1;
        a = (double)s, b = (double)((s + d - 1) / d * d);
      }
    }
    const double f = ddiv_inrange(a, b), r = __ddiv_rn(a, b);
    my += __double_as_longlong(f) != __double_as_longlong(r);
  }
  if (my) atomicAdd(bad, my);
}
}  // namespace tt

extern "C" long long ttdbg_div_check(long long n, unsigned long long seed) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(unsigned long long)) != cudaSuccess) return -1;
  cudaMemset(d, 0, sizeof(unsigned long long));
  tt::k_div_check<<<148 * 8, 256>>>(n, seed, d);
  unsigned long long h = 0;
  const cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? (long long)h : -1;
}
