// tt_kernels.h — internal launcher interface between the C-ABI layer
// (tt_api.cu) and the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "tt_device.cuh"

namespace tt {

// Kernel launches issued by this library (tt_kernel_launches()).
void note_launch();

// Programmatic dependent launch. A kernel launched with launch_pdl may be
// scheduled while its predecessor on the stream is still running; it must
// call pdl_wait() before touching anything the predecessor reads or writes
// (griddepcontrol.wait returns once the predecessor grid has completed and
// its memory is visible). Kernels call pdl_trigger() early so their
// dependents' launch overlaps their tail. Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid, cfg.blockDim = block, cfg.dynamicSmemBytes = smem, cfg.stream = st;
  cfg.attrs = &attr, cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

constexpr int64_t kSmallSelectMax = 1024;

// Round record, 8-byte words, written by the round's finishing kernel straight
// into the context's mapped pinned ring slot (no device->host copy):
// [0] selected, [1] drafted, [2] status, [3] rescored, [4] selector retries
// (host), [5] band error bits (max |fast - fp64| over the rescored set), [6]
// the explicit population failed validate_schedule (K1's flag, which the
// finisher resets for the next round), then b population indices, b scores,
// b draft costs, b identities.
constexpr int64_t kRecHead = 7;
// The ring of round records in mapped pinned memory: the finishing kernel of
// a round takes slot (*seq)++ % kRingSlots, so rounds land in enqueue order;
// the host hands out the same sequence (tt_ctx ring_next).
constexpr int kRingSlots = 16;
struct RecRing {
  int64_t* base;    // kRingSlots slots of `stride` words (device address of the mapped buffer)
  int64_t stride;
  unsigned* seq;    // device counter of finished rounds
};
inline int64_t record_words(int64_t b) { return kRecHead + 4 * b; }

enum : int { TT_SEL_OVERFLOW = 1, TT_SEL_NEED_MORE = 2, TT_SEL_INVALID = 4 };

// Device-resident state of one top-K selection (k_draft.cu).
struct SelState {
  uint64_t prefix;  // threshold: keys with (key >> shift) <= prefix survive
  int32_t shift;
  int32_t done;
  int64_t below;
  int64_t need;
  int32_t all;
  int32_t status;
  uint32_t survivors;
  uint32_t unique;
  int64_t count;
  uint32_t nsurv;   // appended survivors
  uint32_t ticket;  // CTAs finished in the current kernel (last one finalises)
  uint32_t bar_count, bar_gen;  // grid barrier of the cooperative fast selector (self-resetting)
  uint32_t att_surv[8], att_dup[8];  // fast selector: survivors / duplicates per threshold attempt
};

struct SelScratch {
  double* cost = nullptr;  // N costs
  int64_t cost_cap = 0;
  uint32_t* hist = nullptr;  // 4096 bins, zero between uses
  uint64_t* skey = nullptr;  // 4096 survivor keys
  int64_t* sidx = nullptr;   // 4096 survivor indices
  uint32_t* sample = nullptr;  // <= 32768 sampled cost keys, top 32 bits (fast path threshold)
  uint64_t* sfp = nullptr;     // 4096 survivor fingerprints (fast path)
  int* rank = nullptr;         // 4096 survivor ranks (fast path, zeroed per round)
  int* dup = nullptr;          // 4096 survivor duplicate flags
  uint64_t* tkeys = nullptr;  // hash table (tie fallback), all-ones between uses
  uint64_t* tvals = nullptr;
  SelState* state = nullptr;
  int* invalid = nullptr;
  int32_t* mscratch = nullptr;  // cross-rank merge: 3 * kMergeMax words
  cudaEvent_t k1_ev[2] = {nullptr, nullptr};  // optional: recorded around the K1 cost kernel (profiling)
};

// k_draft.cu
int launch_generate(const DevSketch& S, uint64_t s0, int64_t first, int64_t n, int32_t* soa, int64_t ld,
                    uint64_t* id_out, cudaStream_t st);
int launch_identity(const DevSketch& S, const int32_t* soa, int64_t ld, int64_t n, uint64_t* id_out,
                    cudaStream_t st);
int launch_from_identity(const DevSketch& S, const uint64_t* id, int64_t n, int32_t* soa, int64_t ld,
                         cudaStream_t st);
int launch_draft_cost(const DevSketch& S, const DevDevice& D, const int32_t* soa, int64_t ld, uint64_t s0,
                      int64_t first, bool seeded, int64_t n, int toggles, double* cost, uint32_t* hist,
                      int* invalid, cudaStream_t st);
int launch_select(const DevSketch& S, const DevDevice& D, const int32_t* soa, int64_t ld, uint64_t s0,
                  int64_t first, bool seeded, int64_t n, int64_t k, int64_t need, int toggles,
                  int64_t index_base, SelScratch& w, int64_t* out_idx, double* out_cost, uint64_t* out_id,
                  int64_t* out_count, cudaStream_t st, bool hash = false);
// k_explore.cu: all GA generations of one explore in one persistent cluster
// (n <= kMutateMaxN): generation 0 = device slot 0 as generated (soa +
// identity), then mutate() bit-exact from RNG state s_init; generation g is
// written to device slot g (dev_base + g * dev_stride: soa | cost at
// dev_cost_off | identity) and its costs + identities to pinned host memory
// at host_base + g * host_stride (same layout), then flags[g * C + rank] = 1 per
// CTA of the C = explore_cluster_size(n) CTA cluster.
constexpr int64_t kMutateMaxN = 8192;
int explore_cluster_size(int64_t n);  // CTAs of the explore cluster (flags per generation)
int launch_explore_gens(const DevSketch& S, const DevDevice& D, int toggles, int64_t n, int n_steps,
                        void* dev_base, size_t dev_stride, size_t dev_cost_off, uint64_t s_init, void* host_base, size_t host_stride, size_t host_cost_off,
                        volatile uint32_t* flags, cudaStream_t st);
// Cross-rank merge of gathered (cost, global index, identity) lists: the k
// lowest unique by (cost, index). m <= 4096: any order (one-CTA sort); larger
// m: m / k per-rank lists of k, each ascending with empty slots (index -1)
// at its tail, as tt_round_local_async emits them. An index of -2 marks a
// rank whose selector failed: the merge ORs TT_SEL_OVERFLOW into *state; -3
// a rank whose explicit population held an invalid schedule (TT_SEL_INVALID).
constexpr int64_t kMergeMax = 1 << 16;
constexpr int64_t kMergeSortMax = 4096;  // one-CTA sort path (any order)
constexpr int64_t kRankFailed = -2;      // index word of a rank whose selector failed
constexpr int64_t kRankInvalid = -3;     // index word of a rank whose population failed validate_schedule
// sharded draft half, explicit population: slot 0's index <- kRankInvalid when K1 flagged a schedule
int launch_mark_invalid(int* invalid, int64_t* out_idx, cudaStream_t st);
int launch_merge(const double* cost, const int64_t* gidx, const uint64_t* id, int64_t m, int64_t k, int64_t* out_idx,
                 double* out_cost, uint64_t* out_id, int64_t* out_count, SelState* state, int32_t* scratch,
                 cudaStream_t st);
// identities of the drafted set (side stream)
int launch_drafted_identity(const DevSketch& S, const int32_t* soa, int64_t ld, uint64_t s0, int64_t first,
                            bool seeded, const int64_t* idx, const int64_t* count_dev, int64_t k_max, uint64_t* out,
                            cudaStream_t st, unsigned* sync = nullptr);
// How a kernel finds drafted candidate `pos`. Candidates are addressed by identity (population-independent) or by
// (soa, ld, local index). `list`/`count` optionally restrict scoring to a
// device-side sublist of positions (count read on device).
struct CandRef {
  const int32_t* soa;  // explicit population (SoA) ...
  int64_t ld;
  const int64_t* idx;  // population index per position (soa: minus index_base)
  int64_t index_base;
  const uint64_t* id;  // ... or identities per position ...
  uint64_t s0;         // ... or the counter-based stream: schedule idx[pos]
  int32_t seeded;
  int32_t _pad;
};
// k_feat.cu — feature rows of the drafted set (fp64 rows and/or the bf16
// tensor-core tile image, kFeatTileBytes per 16 candidates)
constexpr int64_t kFeatTileBytes = 16384;
int launch_feat_rows(const DevSketch& S, const DevDevice& D, CandRef ref, const int64_t* count_dev, int64_t k_max,
                     const int32_t* sublist, const int* sublist_count, double* stmt, double* block, uint8_t* tiles,
                     cudaStream_t st);

// k_pacm64.cu — fp64 PaCM on feature rows (parity mode / certification)
// k_rank.cu: LambdaRank loss + score gradient (lambda_rank_loss,
// ranker.cpp:394-441) of m <= 2^20 items, scores[i] with latency
// lat[list ? list[i] : i]; *loss (+)= the loss, dscore[i] = the gradient (may
// be null); *bad |= 1 when a latency is not positive. work: rank_work_doubles.
int rank_chunks(int m);
size_t rank_work_doubles(int m);
int launch_rank_loss(const double* scores, const double* lat, const int32_t* list, int m, double* work, int* bad,
                     double* loss, int accumulate, double* dscore, cudaStream_t st);
// k_verify.cu: features + fp64 PaCM of the drafted set in one kernel (h = 64,
// <= 8 statement rows and dataflow blocks, attention on); -1 = not applicable
// vf (optional): the round's finish fused in — identities written to
// id_write (if set), then the last CTA runs select_top + the record gather
// (k_max <= 512, b <= 32; -1 otherwise).
// sync: [0] the verify CTAs' ticket, [1] the identity kernel's block ticket,
// [2] identity kernels completed, [3] fused finishes started (epochs; all zero
// at context creation). With wait_ids the last CTA waits for the side-stream
// identity kernel (k_drafted_identity launched with the same sync) before the
// finish, computing the identities itself if that takes longer than 2 ms.
inline bool verify64_finish_ok(int64_t k, int64_t b) { return k <= 512 && b <= 32 && b <= k; }
struct VerifyFinish {
  const double* drafts;
  const int64_t* idx;
  uint64_t* ids;
  const SelState* sel;
  int64_t b;
  RecRing record;
  unsigned* sync;
  int wait_ids;
  int* invalid;  // K1's population flag: copied into the record, then reset
};
int launch_verify64(const DevSketch& S, const DevDevice& D, CandRef ref, const int64_t* count_dev, int64_t k_max,
                    const double* params, int h, double* score_out, cudaStream_t st,
                    const VerifyFinish* vf = nullptr);
int launch_pacm64(const double* stmt, const double* block, int n_stmt, int n_block, const int64_t* count_dev,
                  int64_t k_max, const int32_t* sublist, const int* sublist_count, const double* params, int h,
                  int attention_identity, double* score_out, cudaStream_t st);

// k_pacm_tc.cu — tcgen05/TMEM fast path (bf16 operands, fp32 accumulators)
bool pacm_tc_supported(int n_stmt, int n_block, int h);
size_t pacm_tc_packed_bytes(int h);
int launch_pacm_tc_pack(const double* params, int h, void* packed, cudaStream_t st);
int launch_pacm_tc(const uint8_t* tiles, int n_stmt, int n_block, const int64_t* count_dev, int64_t k_max,
                   const void* packed, int h, double* score_out, cudaStream_t st);

// k_oracle.cu — simulated hardware (oracle.cpp:82-135)
struct DevOracle {
  DevDevice hidden;
  double stride_coeff, occupancy_coeff, launch, sigma;
  uint64_t seed;
};
int launch_oracle_latency(const DevSketch& S, const DevOracle& O, const int32_t* soa, int64_t ld, int64_t n,
                          int measure, uint64_t task, uint64_t trial0, double* latency, double* noiseless,
                          cudaStream_t st);
int launch_oracle_best(const DevSketch& S, const DevOracle& O, uint64_t* scratch_lat, uint64_t* scratch_id,
                       int max_ctas, uint64_t* out2, cudaStream_t st);

// k_train.cu — PaCM training (score_backward + ordered gradient sums)
size_t train_slot_doubles(int S, int B, int h);
size_t train_work_doubles(int S, int B, int h, int ctas);
int launch_train_fwd(const double* stmt, const double* block, int S, int B, const int32_t* list, int m,
                     const double* params, int h, int identity, double* slots, double* scores, cudaStream_t st);
int launch_train_bwd(int S, int B, int m, const double* params, int h, int identity, const double* dscore,
                     double* slots, double* work, int ctas, cudaStream_t st);
int launch_train_accum(int S, int B, int m, int h, int identity, const double* slots, double* grads,
                       cudaStream_t st);

// k_select.cu
int launch_select_top(const double* scores, const double* drafts, const uint8_t* excluded, int64_t n,
                      const int64_t* n_dev, int64_t b, int64_t* out_pos, int64_t* out_count, int* status,
                      cudaStream_t st);
int launch_band(const double* fast, const int64_t* n_dev, int64_t n_max, const int64_t* pos_fast,
                const int64_t* pos_count, double band, int32_t* sublist, int* sublist_count, uint8_t* excluded,
                cudaStream_t st);
int launch_gd_step(double* params, const double* grads, int64_t n, double lr, cudaStream_t st);
int launch_momentum(double* phi, const double* target, int64_t n, double m, cudaStream_t st);
// select_top + the round record in one CTA (n <= 1024, b <= 32); -1 otherwise
// fast (nullable): the tensor-core scores; record word [5] = max |scores - fast| over
// the candidates not excluded (the fp64-rescored set)
int launch_finish(const double* scores, const double* drafts, const uint8_t* excluded, int64_t n_max,
                  const int64_t* n_dev, int64_t b, const int64_t* idx, const uint64_t* id, const SelState* sel,
                  const int* rescored, const double* fast, RecRing out, int* invalid, cudaStream_t st);
// fast top-b + certification band in one CTA (n <= 1024, b <= 32); -1 otherwise
int launch_cert_band(const double* fast, const double* drafts, int64_t n_max, const int64_t* n_dev, int64_t b,
                     double band, int32_t* sublist, int* sublist_count, uint8_t* excluded, cudaStream_t st);
int launch_gather(const int64_t* pos, const int64_t* pos_count, const int64_t* drafted_count, const SelState* sel,
                  const int* status_b, const int* rescored, const int64_t* idx, const double* cost,
                  const uint64_t* id, const double* scores, const double* fast, const uint8_t* excluded,
                  int64_t n_max, int64_t b, RecRing out, int* invalid, cudaStream_t st);

}  // namespace tt
