// tt_api.cu — the C ABI of include/tt/tt.h: context, validation, plan
// compilation (tt_sketch -> DevSketch) and the round orchestration.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is dlopen()ed by tt_comm_init

#include <algorithm>
#include <chrono>
#include <limits>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <deque>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

#include "../../include/tt/tt.h"
#include "tt_kernels.h"

using namespace tt;

struct tt_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // identities of the drafted set, overlapped with verify
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::string err;
  SelScratch sel;
  // drafted set of the current round
  int64_t k_cap = 0;
  int64_t* d_idx = nullptr;
  double* d_cost = nullptr;
  uint64_t* d_id = nullptr;
  double* d_score = nullptr;
  double* d_score_fast = nullptr;
  int64_t* d_count = nullptr;
  uint8_t* d_excluded = nullptr;
  int32_t* d_sublist = nullptr;
  int* d_sublist_count = nullptr;
  // selection
  int64_t b_cap = 0;
  int64_t* d_pos = nullptr;
  int64_t* d_pos_count = nullptr;
  int64_t* d_pos_fast = nullptr;
  int64_t* d_pos_fast_count = nullptr;
  int* d_status = nullptr;
  int64_t* d_record = nullptr;
  unsigned* d_ticket = nullptr;  // k_verify64's last-CTA ticket (zero between launches)
  // PaCM params
  double* d_params = nullptr;
  int h = 0;
  int64_t n_params = 0;
  void* d_packed = nullptr;
  bool packed_ok = false;
  // feature rows of the drafted set (fp64) and the bf16 tensor-core tile image
  int64_t feat_cap = 0;
  double* d_xs = nullptr;
  double* d_xb = nullptr;
  uint8_t* d_tiles = nullptr;
  // merge inputs
  int64_t m_cap = 0;
  // training scratch (tt_pacm_train / tt_rank_loss), grow-only
  struct Train {
    double *slots = nullptr, *work = nullptr, *grads = nullptr, *dscore = nullptr, *scores = nullptr,
           *rank = nullptr, *lat = nullptr, *loss = nullptr;
    int32_t* list = nullptr;
    int* bad = nullptr;
    int64_t slots_cap = 0, work_cap = 0, grads_cap = 0, dscore_cap = 0, scores_cap = 0, rank_cap = 0, lat_cap = 0,
            loss_cap = 0, list_cap = 0, bad_cap = 0;
  } tr;
  double* h_loss = nullptr;  // pinned: training losses read back once per call
  int64_t h_loss_cap = 0;
  // NCCL communicator of tt_round_sharded (tt_comm_init); payload / gathered
  // [R][3][K] / merged [3][R K] int64 device buffers
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  int64_t* d_gather = nullptr;
  int64_t gather_cap = 0;
  // multi-step explore (GA): one generation on the device, its pinned host mirror
  size_t ex_dcap = 0, ex_hcap = 0;
  void* d_ex = nullptr;  // two device generation slots + the RNG state
  void* h_ex = nullptr;  // pinned generation slots: soa | cost | identity
  std::vector<cudaEvent_t> ex_ev;  // one per generation in flight
  void* d_mix = nullptr;           // random-mix schedules of a draft set: soa | cost | identity
  size_t mix_cap = 0;
  void* h_mix = nullptr;  // pinned: the mix's costs | identities
  size_t h_mix_cap = 0;
  // tt_tuner_round: the draft set on the device (identities | costs | scores)
  // and its pinned host image (identities | costs | picks | pick scores)
  void* d_tr = nullptr;
  void* h_tr = nullptr;
  int64_t tr_cap = 0;
  // rounds in flight: each enqueued round copies its record into its own
  // pinned ring slot and records its own event, so a caller can keep up to
  // kRing rounds in flight and collect them in order (a 17th enqueue fails
  // with E_STATE until the oldest is collected)
  static constexpr int kRing = 16;
  struct Pending {
    int slot;
    int64_t b, k, need, ld;
    bool hash, merged;
    tt_round_config cfg;
    tt_sketch sketch;
    tt_device_spec dev;
    const int32_t* soa;
    uint64_t seed;
    // merged rounds: the gathered lists (caller-owned until collected)
    const double* m_cost;
    const int64_t* m_gidx;
    const uint64_t* m_id;
    int64_t m;
  };
  std::deque<Pending> pend;
  int ring_next = 0;
  // the record ring: one mapped pinned buffer of kRing slots; the finishing
  // kernel of a round writes its record into slot (d_seq++ % kRing), the host
  // hands out the same sequence (ring_next), so no device->host copy is queued
  int64_t* h_ring = nullptr;
  int64_t* d_ring = nullptr;  // its device address
  int64_t* h_rec[kRing] = {};  // h_ring + r * stride
  unsigned* d_seq = nullptr;
  cudaEvent_t ev_rec[kRing] = {};
  // CUDA graphs of whole rounds, keyed by every argument that shapes the
  // enqueued work (sketch, device, config, population pointer, seed, need);
  // cleared whenever scratch is reallocated
  bool graphs = true;
  std::map<std::string, std::pair<cudaGraphExec_t, uint64_t>> graph_cache;  // exec, kernel launches
  std::set<std::string> graph_seen;  // argument sets run once eagerly: captured on their second use
  // stage profiling with CUDA events on the ctx stream
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_live;
  cudaEvent_t ev_open[8] = {};
};

namespace {
constexpr int kStages = 8;  // 0 select, 1 pacm, 2 certify, 3 finish, 4 merge

cudaEvent_t ev_get(tt_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_begin(tt_ctx* c, int stage) {
  if (!c->prof) return;
  c->ev_open[stage] = ev_get(c);
  cudaEventRecord(c->ev_open[stage], c->stream);
}

// K1 events handed to the selector (recorded around its cost kernel)
void prof_k1_arm(tt_ctx* c) {
  if (!c->prof) return;
  c->sel.k1_ev[0] = ev_get(c);
  c->sel.k1_ev[1] = ev_get(c);
}
void prof_k1_collect(tt_ctx* c) {
  if (!c->sel.k1_ev[0]) return;
  c->ev_live.push_back({7, {c->sel.k1_ev[0], c->sel.k1_ev[1]}});
  c->sel.k1_ev[0] = c->sel.k1_ev[1] = nullptr;
}

void prof_drop(tt_ctx* c, int stage) {  // an opened stage that did not run
  if (!c->ev_open[stage]) return;
  c->ev_pool.push_back(c->ev_open[stage]);
  c->ev_open[stage] = nullptr;
}
void prof_end(tt_ctx* c, int stage) {
  if (!c->prof || !c->ev_open[stage]) return;
  cudaEvent_t e = ev_get(c);
  cudaEventRecord(e, c->stream);
  c->ev_live.push_back({stage, {c->ev_open[stage], e}});
  c->ev_open[stage] = nullptr;
}
}  // namespace

namespace {
std::atomic<uint64_t> g_launches{0};
}

void tt::note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" uint64_t tt_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

namespace {

std::atomic<uint64_t> g_forward_calls{0};

int fail(tt_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

#define TT_CUDA(ctx, call)                                                                   \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) return fail(ctx, TT_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

#define TT_LAUNCHED(ctx)                                                                     \
  do {                                                                                       \
    cudaError_t e_ = cudaGetLastError();                                                     \
    if (e_ != cudaSuccess) return fail(ctx, TT_E_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
  } while (0)

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
int log2i(int64_t v) {
  int l = 0;
  while ((int64_t{1} << l) < v) ++l;
  return l;
}

void factorize(int64_t n, std::vector<std::pair<int64_t, int>>& out) {
  out.clear();
  for (int64_t p = 2; p * p <= n; ++p)
    if (n % p == 0) {
      int e = 0;
      while (n % p == 0) n /= p, ++e;
      out.emplace_back(p, e);
    }
  if (n > 1) out.emplace_back(n, 1);
}

uint64_t binom_sat(int64_t n, int64_t k) {
  if (k < 0 || k > n) return 0;
  if (n - k < k) k = n - k;
  unsigned __int128 r = 1;
  for (int64_t i = 1; i <= k; ++i) {
    r = r * (unsigned __int128)(n - k + i) / (unsigned __int128)i;
    if (r > (unsigned __int128)UINT64_MAX) return UINT64_MAX;
  }
  return (uint64_t)r;
}

uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a == 0 || b == 0) return 0;
  if (a > UINT64_MAX / b) return UINT64_MAX;
  return a * b;
}

// validate_op (workload.cpp:49-93) on the POD form + the limits of this build.
int validate_op(tt_ctx* ctx, const tt_op_spec& op) {
  const int na = op.n_spatial + op.n_reduction;
  if (op.n_spatial < 0 || op.n_reduction < 0 || na > TT_MAX_AXES)
    return fail(ctx, TT_E_VALIDATE, "op: bad axis counts");
  if (op.kind == TT_OP_TILED && op.n_spatial == 0)
    return fail(ctx, TT_E_VALIDATE, "op: a tiled op needs at least one spatial axis");
  if (op.n_spatial > kMaxSp || op.n_reduction > kMaxRed)
    return fail(ctx, TT_E_VALIDATE, "op: this build supports at most 4 spatial and 3 reduction axes");
  for (int a = 0; a < na; ++a) {
    if (op.extent[a] < 1)
      return fail(ctx, TT_E_VALIDATE, "op: axis " + std::to_string(a) + " extent must be >= 1, got " +
                                          std::to_string(op.extent[a]));
    if (op.extent[a] >= (int64_t{1} << 31)) return fail(ctx, TT_E_VALIDATE, "op: extent exceeds int32 factors");
  }
  if (op.n_buffers < 1 || op.n_buffers > TT_MAX_BUFFERS) return fail(ctx, TT_E_VALIDATE, "op: no buffers");
  int outputs = 0;
  uint32_t referenced = 0;
  for (int b = 0; b < op.n_buffers; ++b) {
    const tt_buffer_spec& bs = op.buffers[b];
    if (bs.n_axes < 1 || bs.n_axes > TT_MAX_AXES)
      return fail(ctx, TT_E_VALIDATE, "op: buffer " + std::to_string(b) + " has no axes");
    uint32_t seen = 0;
    for (int q = 0; q < bs.n_axes; ++q) {
      const int ax = bs.axes[q];
      if (ax < 0 || ax >= na)
        return fail(ctx, TT_E_VALIDATE, "op: buffer " + std::to_string(b) + " references unknown axis");
      if (seen & (1u << ax)) return fail(ctx, TT_E_VALIDATE, "op: buffer " + std::to_string(b) + " repeats axis");
      seen |= 1u << ax;
    }
    referenced |= seen;
    if (bs.io == TT_IO_OUTPUT) ++outputs;
  }
  if (outputs != 1)
    return fail(ctx, TT_E_VALIDATE, "op: exactly one output buffer required, got " + std::to_string(outputs));
  for (int a = 0; a < na; ++a)
    if (!(referenced & (1u << a)))
      return fail(ctx, TT_E_VALIDATE, "op: axis " + std::to_string(a) + " referenced by no buffer");
  if (op.fused_elementwise < 0) return fail(ctx, TT_E_VALIDATE, "op: fused_elementwise must be >= 0");
  return TT_OK;
}

int compile_sketch(tt_ctx* ctx, const tt_sketch* sk, DevSketch& S) {
  if (!sk) return fail(ctx, TT_E_STATE, "null sketch");
  const tt_op_spec& op = sk->op;
  int rc = validate_op(ctx, op);
  if (rc) return rc;
  if (sk->n_unroll < 1 || sk->n_unroll > TT_MAX_UNROLL) return fail(ctx, TT_E_VALIDATE, "sketch: bad unroll choices");
  std::memset(&S, 0, sizeof(S));
  S.n_sp = op.n_spatial, S.n_red = op.n_reduction, S.n_axes = op.n_spatial + op.n_reduction;
  S.cols = 4 * S.n_sp + 3 * S.n_red + 1;
  S.kind = op.kind, S.n_unroll = sk->n_unroll, S.fused = op.fused_elementwise;
  for (int a = 0; a < S.n_axes; ++a) {
    S.extent[a] = op.extent[a];
    S.arity[a] = a < S.n_sp ? (op.kind == TT_OP_ELEMENTWISE ? 2 : 4) : 3;
  }
  for (int u = 0; u < TT_MAX_UNROLL; ++u) S.unroll[u] = u < sk->n_unroll ? sk->unroll[u] : sk->unroll[0];
  S.innermost_spatial = S.n_sp - 1;
  int out_buf = -1;
  for (int b = 0; b < op.n_buffers; ++b)
    if (op.buffers[b].io == TT_IO_OUTPUT && out_buf < 0) out_buf = b;
  auto mask_of = [&](const tt_buffer_spec& bs) {
    uint32_t m = 0;
    for (int q = 0; q < bs.n_axes; ++q) m |= 1u << bs.axes[q];
    return m;
  };
  const tt_buffer_spec& ob = op.buffers[out_buf];
  S.out_mask = mask_of(ob);
  S.out_last = ob.axes[ob.n_axes - 1];
  S.out_rank = ob.n_axes;
  S.n_in = 0;
  for (int b = 0; b < op.n_buffers; ++b) {
    const tt_buffer_spec& bs = op.buffers[b];
    if (bs.io != TT_IO_INPUT) continue;
    const int q = S.n_in++;
    S.in_mask[q] = mask_of(bs);
    S.in_last[q] = bs.axes[bs.n_axes - 1];
    S.in_rank[q] = bs.n_axes;
    int64_t size = 1;
    int red = 0;
    for (int t = 0; t < bs.n_axes; ++t) {
      size *= op.extent[bs.axes[t]];
      red |= bs.axes[t] >= S.n_sp;
    }
    S.in_size[q] = size;
    S.in_has_red[q] = red;
  }
  S.output_size = 1;
  for (int a = 0; a < S.n_sp; ++a) S.output_size *= op.extent[a];
  S.red_total = 1;
  for (int r = 0; r < S.n_red; ++r) S.red_total *= op.extent[S.n_sp + r];
  S.flops = S.output_size * (op.kind == TT_OP_TILED ? S.red_total : 1);
  // random_init draw plan + identity radix
  std::vector<std::pair<int64_t, int>> pf;
  S.n_prime = 0;
  uint64_t space = 1;
  for (int a = 0; a < S.n_axes; ++a) {
    factorize(op.extent[a], pf);
    for (auto& [p, e] : pf) {
      if (S.n_prime >= TT_MAX_PRIMES) return fail(ctx, TT_E_VALIDATE, "op: too many distinct prime factors");
      const int q = S.n_prime++;
      S.pr_axis[q] = a, S.pr_e[q] = e, S.pr_p[q] = p;
      if (p & 1) {  // modular inverse of odd p mod 2^32 (Newton), divisibility limit
        uint32_t inv = (uint32_t)p;
        for (int it = 0; it < 5; ++it) inv *= 2u - (uint32_t)p * inv;
        S.pr_inv[q] = inv;
        S.pr_lim[q] = 0xffffffffu / (uint32_t)p;
      }
      S.pr_count[q] = binom_sat(e + S.arity[a] - 1, S.arity[a] - 1);
      space = sat_mul(space, S.pr_count[q]);
    }
  }
  S.space = sat_mul(space, (uint64_t)sk->n_unroll);
  for (int q = 0; q < S.n_prime; ++q) S.pr_cinv[q] = UINT64_MAX / (S.pr_count[q] ? S.pr_count[q] : 1);
  S.unroll_cinv = UINT64_MAX / (uint64_t)S.n_unroll;
  S.id_exact = S.space != UINT64_MAX;
  return TT_OK;
}

int compile_device(tt_ctx* ctx, const tt_device_spec* d, DevDevice& D) {
  if (!d) return fail(ctx, TT_E_STATE, "null device");
  int rc = tt_validate_device(d);
  if (rc) return fail(ctx, rc, "device: invalid device spec (validate_device)");
  D.m_l0 = d->m_l0, D.m_l1 = d->m_l1, D.pu_l1 = d->pu_l1, D.n_l1 = d->n_l1;
  D.pu_l2 = d->pu_l2, D.n_l2 = d->n_l2, D.t_p = d->t_p, D.t_m = d->t_m;
  D.log2_nl1 = log2i(d->n_l1), D.log2_nl2 = log2i(d->n_l2);
  D.pu_l1_n_l1 = d->pu_l1 * d->n_l1;
  D.pu_l1_magic = d->pu_l1 > 1 ? UINT64_MAX / (uint64_t)d->pu_l1 + 1 : 0;
  D.pu_l2_magic = d->pu_l2 > 1 ? UINT64_MAX / (uint64_t)d->pu_l2 + 1 : 0;
  return TT_OK;
}

void graphs_clear(tt_ctx* ctx) {
  for (auto& kv : ctx->graph_cache) cudaGraphExecDestroy(kv.second.first);
  ctx->graph_cache.clear();
  ctx->graph_seen.clear();
}

template <typename T>
int grow(tt_ctx* ctx, T*& p, int64_t& cap, int64_t want) {
  if (want <= cap && p) return TT_OK;
  graphs_clear(ctx);
  if (p) cudaFree(p);
  p = nullptr;
  TT_CUDA(ctx, cudaMalloc((void**)&p, sizeof(T) * (size_t)(want > 0 ? want : 1)));
  cap = want;
  return TT_OK;
}

int ensure_k(tt_ctx* ctx, int64_t k) {
  if (k <= ctx->k_cap) return TT_OK;
  graphs_clear(ctx);
  cudaFree(ctx->d_idx), cudaFree(ctx->d_cost), cudaFree(ctx->d_id), cudaFree(ctx->d_score);
  cudaFree(ctx->d_score_fast), cudaFree(ctx->d_excluded), cudaFree(ctx->d_sublist);
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_idx, sizeof(int64_t) * k));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_cost, sizeof(double) * k));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_id, sizeof(uint64_t) * k));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_score, sizeof(double) * k));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_score_fast, sizeof(double) * k));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_excluded, k));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_sublist, sizeof(int32_t) * k));
  ctx->k_cap = k;
  return TT_OK;
}

int ensure_b(tt_ctx* ctx, int64_t b) {
  if (b <= ctx->b_cap) return TT_OK;
  // rounds in flight copy their records into the old pinned slots: let them
  // land, then carry each pending record over into the new, larger slot
  for (const auto& p : ctx->pend) TT_CUDA(ctx, cudaEventSynchronize(ctx->ev_rec[p.slot]));
  graphs_clear(ctx);
  cudaFree(ctx->d_pos), cudaFree(ctx->d_pos_fast), cudaFree(ctx->d_record);
  ctx->d_pos = ctx->d_pos_fast = nullptr, ctx->d_record = nullptr;
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_pos, sizeof(int64_t) * b));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_pos_fast, sizeof(int64_t) * b));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_record, sizeof(int64_t) * record_words(b)));
  int64_t* nh = nullptr;
  TT_CUDA(ctx, cudaHostAlloc((void**)&nh, sizeof(int64_t) * record_words(b) * tt_ctx::kRing, cudaHostAllocMapped));
  for (int r = 0; r < tt_ctx::kRing; ++r) {
    if (ctx->h_ring) std::memcpy(nh + r * record_words(b), ctx->h_rec[r], sizeof(int64_t) * record_words(ctx->b_cap));
    ctx->h_rec[r] = nh + r * record_words(b);
  }
  if (ctx->h_ring) cudaFreeHost(ctx->h_ring);
  ctx->h_ring = nh;
  TT_CUDA(ctx, cudaHostGetDevicePointer((void**)&ctx->d_ring, nh, 0));
  ctx->b_cap = b;
  return TT_OK;
}

// Claims the next ring slot for a round about to be enqueued (record_copy
// lands its record and validity flag there). A full ring is an error: the
// caller collects before enqueueing a 17th round.
int ring_claim(tt_ctx* ctx, int* slot) {
  for (const auto& p : ctx->pend)
    if (p.slot == ctx->ring_next)
      return fail(ctx, TT_E_STATE, "round: 16 rounds already in flight on this context (tt_round_collect first)");
  *slot = ctx->ring_next;
  return TT_OK;
}

void ring_push(tt_ctx* ctx, tt_ctx::Pending p) {
  ctx->pend.push_back(p);
  ctx->ring_next = (p.slot + 1) % tt_ctx::kRing;
}

int ensure_cost(tt_ctx* ctx, int64_t n) { return grow(ctx, ctx->sel.cost, ctx->sel.cost_cap, n); }

// room for the feature rows of k candidates (statement rows <= 14, dataflow
// blocks <= 20: ops with up to 6 inputs) and their tensor-core tile image
int ensure_feat(tt_ctx* ctx, int64_t k) {
  if (k <= ctx->feat_cap) return TT_OK;
  graphs_clear(ctx);
  cudaFree(ctx->d_xs), cudaFree(ctx->d_xb), cudaFree(ctx->d_tiles);
  ctx->d_xs = nullptr, ctx->d_xb = nullptr, ctx->d_tiles = nullptr;
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_xs, sizeof(double) * 14 * TT_STMT_WIDTH * k));
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_xb, sizeof(double) * 20 * TT_BLOCK_WIDTH * k));
  // k_feat_rows writes whole 32-candidate passes = 2 tiles
  TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_tiles, (size_t)kFeatTileBytes * 2 * ((k + 31) / 32)));
  ctx->feat_cap = k;
  return TT_OK;
}

int n_stmt_of(const DevSketch& S) { return 2 * S.n_in + 2; }
int n_block_of(const DevSketch& S) { return S.kind == TT_OP_ELEMENTWISE ? 1 : 3 * S.n_in + 2; }

int sync_check(tt_ctx* ctx) {
  TT_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  TT_CUDA(ctx, cudaGetLastError());
  return TT_OK;
}

// Runs the selector with retries (NEED_MORE: duplicates ate into the
// target; the threshold is raised until k unique survive or all pass).
int select_sync(tt_ctx* ctx, const DevSketch& S, const DevDevice& D, const int32_t* soa, int64_t ld, uint64_t s0,
                int64_t first, bool seeded, int64_t n, int64_t k, int toggles, int64_t index_base, int64_t* idx,
                double* cost, uint64_t* id, int64_t* count_host) {
  int64_t need = k + k / 8 + 16;
  bool hash = false;
  for (int attempt = 0; attempt < 64; ++attempt) {
    TT_CUDA(ctx, cudaMemsetAsync(ctx->sel.invalid, 0, sizeof(int), ctx->stream));
    if (n > kSmallSelectMax) {
      int rc = ensure_cost(ctx, n);
      if (rc) return rc;
    }
    if (launch_select(S, D, soa, ld, s0, first, seeded, n, k, need, toggles, index_base, ctx->sel, idx, cost, id,
                      ctx->d_count, ctx->stream, hash))
      return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
    TT_LAUNCHED(ctx);
    SelState st;
    int invalid = 0;
    TT_CUDA(ctx, cudaMemcpyAsync(&st, ctx->sel.state, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream));
    TT_CUDA(ctx, cudaMemcpyAsync(&invalid, ctx->sel.invalid, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    int rc = sync_check(ctx);
    if (rc) return rc;
    if (invalid) return fail(ctx, TT_E_VALIDATE, "schedule does not satisfy validate_schedule (factor products / unroll)");
    if (n > kSmallSelectMax && (st.status & TT_SEL_OVERFLOW)) {
      if (hash)
        return fail(ctx, TT_E_STATE, "draft selector overflow: more than 4096 unique schedules tie at the threshold");
      hash = true;  // > 4096 keys share the threshold prefix: dedup on insert
      continue;
    }
    if (n > kSmallSelectMax && (st.status & TT_SEL_NEED_MORE)) {
      need *= 2;
      continue;
    }
    TT_CUDA(ctx, cudaMemcpy(count_host, ctx->d_count, sizeof(int64_t), cudaMemcpyDeviceToHost));
    return TT_OK;
  }
  return fail(ctx, TT_E_STATE, "draft selector did not converge");
}

uint64_t seed_state(uint64_t seed) { return seed ? seed : kGolden; }

}  // namespace

extern "C" {

const char* tt_version(void) { return "paper_2402_02361_b200 0.1 (sm_100a)"; }

const char* tt_status_code(int s) {
  switch (s) {
    case TT_OK: return "OK";
    case TT_E_PARSE: return "E_PARSE";
    case TT_E_VALIDATE: return "E_VALIDATE";
    case TT_E_CONFIG: return "E_CONFIG";
    case TT_E_STATE: return "E_STATE";
    case TT_E_IO: return "E_IO";
    case TT_E_CUDA: return "E_CUDA";
    case TT_E_NCCL: return "E_NCCL";
  }
  return "E_UNKNOWN";
}

int tt_ctx_create(int device, tt_ctx** out) {
  if (!out) return TT_E_STATE;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return TT_E_CUDA;
  if (device < 0 || device >= n) return TT_E_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return TT_E_CUDA;
  tt_ctx* c = new tt_ctx();
  c->device = device;
  auto bad = [&](cudaError_t e) {
    if (e != cudaSuccess) {
      tt_ctx_destroy(c);
      return true;
    }
    return false;
  };
  if (bad(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking))) return TT_E_CUDA;
  if (bad(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking))) return TT_E_CUDA;
  if (bad(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming))) return TT_E_CUDA;
  if (bad(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming))) return TT_E_CUDA;
  for (int r = 0; r < tt_ctx::kRing; ++r) {
    if (bad(cudaEventCreateWithFlags(&c->ev_rec[r], cudaEventDisableTiming))) return TT_E_CUDA;
  }
  c->stream = c->own;
  if (const char* g = getenv("TT_GRAPHS")) c->graphs = g[0] != '0';
  if (bad(cudaMalloc((void**)&c->sel.hist, 4096 * sizeof(uint32_t)))) return TT_E_CUDA;
  if (bad(cudaMemset(c->sel.hist, 0, 4096 * sizeof(uint32_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.skey, 8192 * sizeof(uint64_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.sidx, 8192 * sizeof(int64_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.sample, 32768 * sizeof(uint32_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.sfp, 8192 * sizeof(uint64_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.rank, 8192 * sizeof(int)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.dup, 8192 * sizeof(int)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.mscratch, kMergeMax * 3 * sizeof(int32_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.tkeys, 16384 * sizeof(uint64_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.tvals, 16384 * sizeof(uint64_t)))) return TT_E_CUDA;
  if (bad(cudaMemset(c->sel.tkeys, 0xff, 16384 * sizeof(uint64_t)))) return TT_E_CUDA;
  if (bad(cudaMemset(c->sel.tvals, 0xff, 16384 * sizeof(uint64_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.state, sizeof(SelState)))) return TT_E_CUDA;
  if (bad(cudaMemset(c->sel.state, 0, sizeof(SelState)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->sel.invalid, sizeof(int)))) return TT_E_CUDA;
  if (bad(cudaMemset(c->sel.invalid, 0, sizeof(int)))) return TT_E_CUDA;  // seeded rounds copy it unset
  if (bad(cudaMalloc((void**)&c->d_count, sizeof(int64_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->d_pos_count, sizeof(int64_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->d_pos_fast_count, sizeof(int64_t)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->d_status, 2 * sizeof(int)))) return TT_E_CUDA;
  if (bad(cudaMalloc((void**)&c->d_ticket, 8 * sizeof(unsigned)))) return TT_E_CUDA;  // VerifyFinish::sync | ring seq
  if (bad(cudaMemset(c->d_ticket, 0, 8 * sizeof(unsigned)))) return TT_E_CUDA;
  c->d_seq = c->d_ticket + 4;
  if (bad(cudaMalloc((void**)&c->d_sublist_count, sizeof(int)))) return TT_E_CUDA;
  if (bad(cudaMemset(c->d_sublist_count, 0, sizeof(int)))) return TT_E_CUDA;
  if (bad(cudaDeviceSynchronize())) return TT_E_CUDA;
  *out = c;
  return TT_OK;
}

void tt_ctx_destroy(tt_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) tt_comm_destroy(c);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (auto& pr : c->ev_live) cudaEventDestroy(pr.second.first), cudaEventDestroy(pr.second.second);
  void* ptrs[] = {c->sel.cost, c->sel.hist, c->sel.skey, c->sel.sidx, c->sel.sample, c->sel.sfp, c->sel.rank, c->sel.dup, c->sel.tkeys, c->sel.tvals, c->sel.state, c->sel.mscratch,
                  c->sel.invalid,
                  c->d_idx, c->d_cost, c->d_id, c->d_score, c->d_score_fast, c->d_count, c->d_excluded,
                  c->d_sublist, c->d_sublist_count, c->d_pos, c->d_pos_count, c->d_pos_fast,
                  c->d_pos_fast_count, c->d_status, c->d_record, c->d_params, c->d_packed, c->d_xs, c->d_xb,
                  c->d_tiles, c->d_ex, c->d_mix, c->tr.slots, c->tr.work, c->tr.grads, c->tr.dscore,
                  c->tr.scores, c->tr.rank, c->tr.lat, c->tr.loss, c->tr.list, c->tr.bad, c->d_gather,
                  c->d_ticket};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (int r = 0; r < tt_ctx::kRing; ++r) {
    if (c->ev_rec[r]) cudaEventDestroy(c->ev_rec[r]);
  }
  if (c->h_ex) cudaFreeHost(c->h_ex);
  if (c->h_ring) cudaFreeHost(c->h_ring);
  if (c->h_loss) cudaFreeHost(c->h_loss);
  if (c->h_mix) cudaFreeHost(c->h_mix);
  if (c->h_tr) cudaFreeHost(c->h_tr);
  if (c->d_tr) cudaFree(c->d_tr);
  for (cudaEvent_t e : c->ex_ev) cudaEventDestroy(e);
  graphs_clear(c);
  if (c->side) cudaStreamSynchronize(c->side), cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
}

const char* tt_last_error(const tt_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int tt_ctx_set_stream(tt_ctx* ctx, void* s) {
  if (!ctx) return TT_E_STATE;
  ctx->stream = s ? (cudaStream_t)s : ctx->own;
  return TT_OK;
}

void* tt_ctx_stream(const tt_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int tt_ctx_sync(tt_ctx* ctx) {
  if (!ctx) return TT_E_STATE;
  return sync_check(ctx);
}

int tt_sketch_from_op(const tt_op_spec* op, int elementwise_fallback, tt_sketch* out) {
  if (!op || !out) return TT_E_STATE;
  int rc = validate_op(nullptr, *op);
  if (rc) return rc;
  if (op->kind == TT_OP_ELEMENTWISE && !elementwise_fallback) return TT_E_VALIDATE;
  std::memset(out, 0, sizeof(*out));
  out->op = *op;
  out->n_unroll = 3;
  out->unroll[0] = 1, out->unroll[1] = 4, out->unroll[2] = 16;
  return TT_OK;
}

int tt_validate_device(const tt_device_spec* d) {
  if (!d) return TT_E_STATE;
  if (d->m_l0 <= 0 || d->m_l1 <= 0 || d->pu_l1 <= 0 || d->n_l1 <= 0 || d->pu_l2 <= 0 || d->n_l2 <= 0 ||
      !(d->t_p > 0.0) || !(d->t_m > 0.0) || d->element_bytes <= 0)
    return TT_E_VALIDATE;
  if (!is_pow2(d->n_l1) || !is_pow2(d->n_l2)) return TT_E_VALIDATE;
  if (d->t_p == __builtin_inf() || d->t_m == __builtin_inf()) return TT_E_VALIDATE;
  return TT_OK;
}

uint64_t tt_space_size(const tt_sketch* sk) {
  DevSketch S;
  if (compile_sketch(nullptr, sk, S)) return 0;
  return S.space;
}

int tt_draws_per_schedule(const tt_sketch* sk) {
  DevSketch S;
  if (compile_sketch(nullptr, sk, S)) return -1;
  return S.n_prime + 1;
}

int tt_population_generate(tt_ctx* ctx, const tt_sketch* sk, uint64_t seed, int64_t first, int64_t n,
                           int32_t* soa, int64_t ld, uint64_t* id) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if (n < 0 || first < 0 || (soa && ld < n)) return fail(ctx, TT_E_STATE, "population: bad n/ld");
  if (launch_generate(S, seed_state(seed), first, n, soa, ld, id, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_schedule_identity(tt_ctx* ctx, const tt_sketch* sk, const int32_t* soa, int64_t ld, int64_t n, uint64_t* id) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if (!S.id_exact) return fail(ctx, TT_E_STATE, "identity: schedule space exceeds 2^64");
  if (launch_identity(S, soa, ld, n, id, ctx->stream)) return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_schedule_from_identity(tt_ctx* ctx, const tt_sketch* sk, const uint64_t* id, int64_t n, int32_t* soa,
                              int64_t ld) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if (!S.id_exact) return fail(ctx, TT_E_STATE, "identity: schedule space exceeds 2^64");
  if (launch_from_identity(S, id, n, soa, ld, ctx->stream)) return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_draft_cost(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
                  int64_t n, int toggles, double* cost) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if (n < 0 || ld < n) return fail(ctx, TT_E_STATE, "draft_cost: bad n/ld");
  if (n == 0) return TT_OK;
  TT_CUDA(ctx, cudaMemsetAsync(ctx->sel.invalid, 0, sizeof(int), ctx->stream));
  if (launch_draft_cost(S, D, soa, ld, 0, 0, false, n, toggles, cost, nullptr, ctx->sel.invalid, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  int invalid = 0;
  TT_CUDA(ctx, cudaMemcpyAsync(&invalid, ctx->sel.invalid, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  if ((rc = sync_check(ctx))) return rc;
  if (invalid) {  // the flag is zero between calls
    TT_CUDA(ctx, cudaMemsetAsync(ctx->sel.invalid, 0, sizeof(int), ctx->stream));
    return fail(ctx, TT_E_VALIDATE, "schedule does not satisfy validate_schedule (factor products / unroll)");
  }
  return TT_OK;
}

int tt_draft_topk(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
                  int64_t n, int64_t k, int toggles, int64_t index_base, int64_t* idx, double* cost, uint64_t* id,
                  int64_t* count) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if (k < 1) return fail(ctx, TT_E_STATE, "explore: draft_size must be >= 1");
  if (n < 2) return fail(ctx, TT_E_STATE, "explore: pop_size must be >= 2");
  if (ld < n) return fail(ctx, TT_E_STATE, "draft_topk: ld < n");
  if (!S.id_exact) return fail(ctx, TT_E_STATE, "draft_topk: schedule space exceeds 2^64 identities");
  return select_sync(ctx, S, D, soa, ld, 0, 0, false, n, k, toggles, index_base, idx, cost, id, count);
}

int tt_explore1(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, uint64_t seed, int64_t first,
                int64_t n, int64_t k, int toggles, int64_t* idx, double* cost, uint64_t* id, int64_t* count) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if (k < 1) return fail(ctx, TT_E_STATE, "explore: draft_size must be >= 1");
  if (n < 2) return fail(ctx, TT_E_STATE, "explore: pop_size must be >= 2");
  if (!S.id_exact) return fail(ctx, TT_E_STATE, "explore1: schedule space exceeds 2^64 identities");
  return select_sync(ctx, S, D, nullptr, 0, seed_state(seed), first, true, n, k, toggles, first, idx, cost, id, count);
}

int tt_topk_merge(tt_ctx* ctx, const double* cost, const int64_t* gidx, const uint64_t* id, int64_t m, int64_t k,
                  int64_t* idx, double* out_cost, uint64_t* out_id, int64_t* count) {
  if (!ctx) return TT_E_STATE;
  if (m < 0 || m > kMergeMax)
    return fail(ctx, TT_E_STATE, "merge: at most " + std::to_string(kMergeMax) + " gathered entries per call");
  if (m > kMergeSortMax && (k < 1 || m % k))
    return fail(ctx, TT_E_STATE, "merge: more than 4096 entries must be whole per-rank lists of k");
  if (launch_merge(cost, gidx, id, m, k, idx, out_cost, out_id, ctx->d_count, nullptr, ctx->sel.mscratch,
                   ctx->stream))
    return fail(ctx, TT_E_STATE, "merge: launch");
  TT_LAUNCHED(ctx);
  TT_CUDA(ctx, cudaMemcpyAsync(count, ctx->d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  return sync_check(ctx);
}

int tt_features(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const uint64_t* id, int64_t k,
                double* stmt, double* block) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  CandRef r{nullptr, 0, nullptr, 0, id};
  if (launch_feat_rows(S, D, r, nullptr, k, nullptr, nullptr, stmt, block, nullptr, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_features_soa(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
                    const int64_t* idx, int64_t k, double* stmt, double* block) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  CandRef r{soa, ld, idx, 0, nullptr};
  if (launch_feat_rows(S, D, r, nullptr, k, nullptr, nullptr, stmt, block, nullptr, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_pacm_load(tt_ctx* ctx, const double* params, int h) {
  if (!ctx) return TT_E_STATE;
  if (h < 1 || h > 512) return fail(ctx, TT_E_STATE, "hidden width must be in [1, 512]");
  const int64_t np = tt_param_count(h);
  if (ctx->h != h) {
    graphs_clear(ctx);
    if (ctx->d_params) cudaFree(ctx->d_params);
    if (ctx->d_packed) cudaFree(ctx->d_packed);
    ctx->d_params = nullptr, ctx->d_packed = nullptr;
    TT_CUDA(ctx, cudaMalloc((void**)&ctx->d_params, sizeof(double) * np));
    ctx->h = h;
    ctx->n_params = np;
  }
  TT_CUDA(ctx, cudaMemcpyAsync(ctx->d_params, params, sizeof(double) * np, cudaMemcpyDefault, ctx->stream));
  ctx->packed_ok = false;
  return TT_OK;
}

uint64_t tt_forward_calls(void) { return g_forward_calls.load(std::memory_order_relaxed); }
void tt_reset_forward_calls(void) { g_forward_calls.store(0, std::memory_order_relaxed); }

}  // extern "C"

namespace {

int ensure_packed(tt_ctx* ctx) {
  if (ctx->packed_ok) return TT_OK;
  if (!ctx->d_packed) {
    graphs_clear(ctx);
    TT_CUDA(ctx, cudaMalloc(&ctx->d_packed, pacm_tc_packed_bytes(ctx->h)));
  }
  if (launch_pacm_tc_pack(ctx->d_params, ctx->h, ctx->d_packed, ctx->stream))
    return fail(ctx, TT_E_CONFIG, "tensor-core PaCM: packing failed");
  TT_LAUNCHED(ctx);
  ctx->packed_ok = true;
  return TT_OK;
}

// Scores the drafted set (positions [0, *count_dev)) into ctx->d_score:
// features (k_feat_rows) -> PaCM. fp64: exact scores. bf16: tensor-core
// scores, then certified selection — the top-b by the fast score and every
// candidate within `band` of the b-th fast score are rescored in fp64 (their
// rows rebuilt in fp64 for just that sublist); the final select_top only
// considers exactly rescored candidates (d_excluded marks the rest).
int score_drafted(tt_ctx* ctx, const DevSketch& S, const DevDevice& D, CandRef ref, int64_t k_max, int precision,
                  int64_t b, double band, const int64_t* count_dev) {
  const int ns = n_stmt_of(S), nb = n_block_of(S);
  int rc = ensure_feat(ctx, k_max);
  if (rc) return rc;
  if (precision == TT_PREC_FP64) {
    prof_begin(ctx, 1);
    prof_begin(ctx, 5);
    // the tuner geometry: features + PaCM in one kernel (k_verify64)
    const int fused = launch_verify64(S, D, ref, count_dev, k_max, ctx->d_params, ctx->h, ctx->d_score, ctx->stream);
    if (fused == 0) {
      prof_end(ctx, 5);
      prof_end(ctx, 1);
      TT_LAUNCHED(ctx);
      TT_CUDA(ctx, cudaMemsetAsync(ctx->d_sublist_count, 0, sizeof(int), ctx->stream));
      return TT_OK;
    }
    prof_begin(ctx, 6);
    if (launch_feat_rows(S, D, ref, count_dev, k_max, nullptr, nullptr, ctx->d_xs, ctx->d_xb, nullptr, ctx->stream))
      return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
    prof_end(ctx, 6);
    if (launch_pacm64(ctx->d_xs, ctx->d_xb, ns, nb, count_dev, k_max, nullptr, nullptr, ctx->d_params, ctx->h, 0,
                      ctx->d_score, ctx->stream))
      return fail(ctx, TT_E_CONFIG, "fp64 PaCM: hidden width too large for shared memory");
    prof_end(ctx, 5);
    prof_end(ctx, 1);
    TT_LAUNCHED(ctx);
    TT_CUDA(ctx, cudaMemsetAsync(ctx->d_sublist_count, 0, sizeof(int), ctx->stream));
    return TT_OK;
  }
  if (precision != TT_PREC_BF16) return fail(ctx, TT_E_CONFIG, "unknown precision");
  if (!pacm_tc_supported(ns, nb, ctx->h)) return fail(ctx, TT_E_CONFIG, "tensor-core PaCM: unsupported shape/width");
  if ((rc = ensure_packed(ctx))) return rc;
  prof_begin(ctx, 1);
  prof_begin(ctx, 6);
  // fp64 rows as well: the certification rescoring reads them (no second feature pass)
  if (launch_feat_rows(S, D, ref, count_dev, k_max, nullptr, nullptr, b > 0 ? ctx->d_xs : nullptr,
                       b > 0 ? ctx->d_xb : nullptr, ctx->d_tiles, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  prof_end(ctx, 6);
  prof_begin(ctx, 5);
  if (launch_pacm_tc(ctx->d_tiles, ns, nb, count_dev, k_max, ctx->d_packed, ctx->h, ctx->d_score_fast, ctx->stream))
    return fail(ctx, TT_E_CONFIG, "tensor-core PaCM launch");
  prof_end(ctx, 5);
  prof_end(ctx, 1);
  TT_LAUNCHED(ctx);
  if (b > 0) {
    prof_begin(ctx, 2);
    if (launch_cert_band(ctx->d_score_fast, ctx->d_cost, k_max, count_dev, b, band, ctx->d_sublist,
                         ctx->d_sublist_count, ctx->d_excluded, ctx->stream)) {
      launch_select_top(ctx->d_score_fast, ctx->d_cost, nullptr, k_max, count_dev, b, ctx->d_pos_fast,
                        ctx->d_pos_fast_count, ctx->d_status + 1, ctx->stream);
      launch_band(ctx->d_score_fast, count_dev, k_max, ctx->d_pos_fast, ctx->d_pos_fast_count, band, ctx->d_sublist,
                  ctx->d_sublist_count, ctx->d_excluded, ctx->stream);
    }
    TT_CUDA(ctx, cudaMemcpyAsync(ctx->d_score, ctx->d_score_fast, sizeof(double) * k_max, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
    if (launch_pacm64(ctx->d_xs, ctx->d_xb, ns, nb, count_dev, k_max, ctx->d_sublist, ctx->d_sublist_count,
                      ctx->d_params, ctx->h, 0, ctx->d_score, ctx->stream))
      return fail(ctx, TT_E_CONFIG, "fp64 PaCM: hidden width too large for shared memory");
    prof_end(ctx, 2);
    TT_LAUNCHED(ctx);
  } else {
    TT_CUDA(ctx, cudaMemcpyAsync(ctx->d_score, ctx->d_score_fast, sizeof(double) * k_max, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
  }
  return TT_OK;
}

// Everything after the drafted set exists on the device.
// ref: how the drafted candidates are addressed (SoA / counter stream /
// identities). Identities of the b selections come from d_id for merged
// rounds, otherwise they are computed for those b only.
int verify_and_select(tt_ctx* ctx, const DevSketch& S, const DevDevice& D, const tt_round_config* cfg,
                      CandRef ref, int slot) {
  (void)slot;  // the finishing kernel takes the ring's next slot = slot (same sequence)
  const RecRing record{ctx->d_ring, record_words(ctx->b_cap), ctx->d_seq};
  const bool by_id = ref.id != nullptr;
  if (cfg->precision == TT_PREC_FP64 && ctx->h == 64 && n_stmt_of(S) <= 8 && n_block_of(S) <= 8 &&
      verify64_finish_ok(cfg->k, cfg->b)) {
    // the tuner geometry: features, PaCM and the finish in ONE kernel
    // (k_verify64; its last CTA runs select_top + the record once the
    // side-stream identities of the drafted set have landed)
    if (!by_id) {
      TT_CUDA(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
      TT_CUDA(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
      if (launch_drafted_identity(S, ref.soa, ref.ld, ref.s0, ref.seeded ? cfg->first : ref.index_base,
                                  ref.seeded != 0, ctx->d_idx, ctx->d_count, cfg->k, ctx->d_id, ctx->side,
                                  ctx->d_ticket))
        return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
      TT_LAUNCHED(ctx);
      TT_CUDA(ctx, cudaEventRecord(ctx->ev_join, ctx->side));
    }
    const VerifyFinish vf{ctx->d_cost, ctx->d_idx, ctx->d_id,     ctx->sel.state,   cfg->b,
                          record,      ctx->d_ticket, by_id ? 0 : 1, ctx->sel.invalid};
    prof_begin(ctx, 1);
    prof_begin(ctx, 5);
    if (launch_verify64(S, D, ref, ctx->d_count, cfg->k, ctx->d_params, ctx->h, ctx->d_score, ctx->stream, &vf))
      return fail(ctx, TT_E_VALIDATE, "fused verify: unsupported op shape");
    prof_end(ctx, 5);
    prof_end(ctx, 1);
    TT_LAUNCHED(ctx);
    // join (the identity kernel is long done: the finish waited for it)
    if (!by_id) TT_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
    return TT_OK;
  }
  if (!by_id) {  // fork: identities of the drafted set on the side stream
    TT_CUDA(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
    TT_CUDA(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    if (launch_drafted_identity(S, ref.soa, ref.ld, ref.s0, ref.seeded ? cfg->first : ref.index_base,
                                ref.seeded != 0, ctx->d_idx, ctx->d_count, cfg->k, ctx->d_id, ctx->side))
      return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
    TT_LAUNCHED(ctx);
    TT_CUDA(ctx, cudaEventRecord(ctx->ev_join, ctx->side));
  }
  int rc = score_drafted(ctx, S, D, ref, cfg->k, cfg->precision, cfg->b, cfg->band,
                         ctx->d_count);
  if (rc) return rc;
  const bool certified = cfg->precision != TT_PREC_FP64;
  prof_begin(ctx, 3);
  if (!by_id) TT_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));  // join
  const uint8_t* excl = certified ? ctx->d_excluded : nullptr;
  const double* fast = certified ? ctx->d_score_fast : nullptr;
  if (launch_finish(ctx->d_score, ctx->d_cost, excl, cfg->k, ctx->d_count, cfg->b, ctx->d_idx, ctx->d_id,
                    ctx->sel.state, ctx->d_sublist_count, fast, record, ctx->sel.invalid, ctx->stream)) {
    // large draft sets / batches: tiled select_top, then the record gather
    if (launch_select_top(ctx->d_score, ctx->d_cost, excl, cfg->k, ctx->d_count, cfg->b, ctx->d_pos,
                          ctx->d_pos_count, ctx->d_status, ctx->stream))
      return fail(ctx, TT_E_CONFIG, "select_top: draft_size too large for the batch");
    launch_gather(ctx->d_pos, ctx->d_pos_count, ctx->d_count, ctx->sel.state, nullptr, ctx->d_sublist_count,
                  ctx->d_idx, ctx->d_cost, ctx->d_id, ctx->d_score, fast, excl, cfg->k, cfg->b, record,
                  ctx->sel.invalid, ctx->stream);
  }
  prof_end(ctx, 3);
  TT_LAUNCHED(ctx);
  return TT_OK;
}

// The round's record and validity flag into its ring slot, then its event.
// Outside any graph (the slot changes every round; the graphs do not).
int record_copy(tt_ctx* ctx, int slot, int64_t) {
  // the record is already in its mapped slot (written by the finishing
  // kernel): the slot's event marks when it is complete
  TT_CUDA(ctx, cudaEventRecord(ctx->ev_rec[slot], ctx->stream));
  return TT_OK;
}

int check_round_cfg(tt_ctx* ctx, const tt_round_config* cfg) {
  if (!cfg) return fail(ctx, TT_E_STATE, "null round config");
  if (cfg->k < 1) return fail(ctx, TT_E_CONFIG, "draft_size must be >= 1");
  if (cfg->b < 1) return fail(ctx, TT_E_CONFIG, "batch must be >= 1");
  if (cfg->k < cfg->b) return fail(ctx, TT_E_CONFIG, "draft_size must be >= batch");
  if (cfg->n < 2) return fail(ctx, TT_E_CONFIG, "pop_size must be >= 2");
  if (cfg->precision == TT_PREC_BF16 && !(cfg->band > 0.0))
    return fail(ctx, TT_E_CONFIG, "bf16 round: the certification band must be > 0 (a bound on |bf16 - fp64| scores)");
  if (!ctx->d_params) return fail(ctx, TT_E_STATE, "round: tt_pacm_load first");
  return TT_OK;
}

// The device work of one round (select -> verify -> finish -> record copy),
// enqueued on ctx->stream. Scratch must already be sized (no allocation
// here), so the sequence can be captured into a CUDA graph.
int round_body(tt_ctx* ctx, const DevSketch& S, const DevDevice& D, const tt_round_config* cfg, const int32_t* soa,
               int64_t ld, uint64_t seed, int64_t need, bool hash, int slot) {
  const bool seeded = soa == nullptr;
  // sel.invalid is zero between calls (every reader resets it): no memset node
  prof_begin(ctx, 0);
  prof_k1_arm(ctx);
  if (launch_select(S, D, soa, ld, seed_state(seed), cfg->first, seeded, cfg->n, cfg->k, need, cfg->toggles,
                    cfg->first, ctx->sel, ctx->d_idx, ctx->d_cost, nullptr, ctx->d_count, ctx->stream, hash))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  prof_k1_collect(ctx);
  prof_end(ctx, 0);
  TT_LAUNCHED(ctx);
  // the verifier re-derives each drafted candidate from its population
  // index: a SoA gather, or a counter-based regeneration
  CandRef ref = seeded ? CandRef{nullptr, 0, ctx->d_idx, 0, nullptr, seed_state(seed), 1, 0}
                       : CandRef{soa, ld, ctx->d_idx, cfg->first, nullptr, 0, 0, 0};
  return verify_and_select(ctx, S, D, cfg, ref, slot);
}

// retry_slot >= 0: a synchronous re-run of a collected round into its own
// (already popped) ring slot; nothing is pushed
int round_enqueue(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
                  const int32_t* soa, int64_t ld, uint64_t seed, int64_t need, bool hash = false,
                  int* retry_slot = nullptr) {
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if ((rc = check_round_cfg(ctx, cfg))) return rc;
  if (!S.id_exact) return fail(ctx, TT_E_STATE, "round: schedule space exceeds 2^64 identities");
  if ((rc = ensure_k(ctx, cfg->k))) return rc;
  if ((rc = ensure_b(ctx, cfg->b))) return rc;
  if ((rc = ensure_feat(ctx, cfg->k))) return rc;
  if (cfg->n > kSmallSelectMax && (rc = ensure_cost(ctx, cfg->n))) return rc;
  if (cfg->precision == TT_PREC_BF16 && (rc = ensure_packed(ctx))) return rc;
  // the ring's next slot (a synchronous re-run of a collected round takes it
  // too: the device hands out slots in launch order)
  int slot = -1;
  if ((rc = ring_claim(ctx, &slot))) return rc;
  if (!ctx->graphs || ctx->prof) {
    if ((rc = round_body(ctx, S, D, cfg, soa, ld, seed, need, hash, slot))) return rc;
  } else {
    // graph cache: the key is every byte that shapes the enqueued work
    std::string key;
    auto put = [&](const void* p, size_t n) { key.append((const char*)p, n); };
    put(sk, sizeof(*sk)), put(dev, sizeof(*dev)), put(cfg, sizeof(*cfg)), put(&soa, sizeof(soa)), put(&ld, 8);
    put(&seed, 8), put(&need, 8), put(&hash, 1), put(&ctx->h, sizeof(ctx->h));
    auto it = ctx->graph_cache.find(key);
    // capturing costs ~1 ms: a round whose arguments never repeat (a fresh
    // seed every tuner round) runs eagerly; repeats are captured and replayed
    if (ctx->graph_seen.size() > 4096) ctx->graph_seen.clear();  // bounded memory over long tuning runs
    const bool repeat = it != ctx->graph_cache.end() || !ctx->graph_seen.insert(key).second;
    if (!repeat) {
      if ((rc = round_body(ctx, S, D, cfg, soa, ld, seed, need, hash, slot))) return rc;
    } else if (it == ctx->graph_cache.end()) {
      cudaStream_t launch = ctx->stream;
      const uint64_t l0 = tt_kernel_launches();
      TT_CUDA(ctx, cudaStreamBeginCapture(ctx->own, cudaStreamCaptureModeRelaxed));
      ctx->stream = ctx->own;
      rc = round_body(ctx, S, D, cfg, soa, ld, seed, need, hash, slot);
      ctx->stream = launch;
      cudaGraph_t g = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(ctx->own, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (ec != cudaSuccess) return fail(ctx, TT_E_CUDA, std::string("round capture: ") + cudaGetErrorString(ec));
      cudaGraphExec_t ex = nullptr;
      const cudaError_t ei = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      if (ei != cudaSuccess) return fail(ctx, TT_E_CUDA, std::string("round graph: ") + cudaGetErrorString(ei));
      it = ctx->graph_cache.emplace(key, std::make_pair(ex, tt_kernel_launches() - l0)).first;
    } else {
      for (uint64_t q = 0; q < it->second.second; ++q) tt::note_launch();  // the replay launches them again
    }
    if (repeat) TT_CUDA(ctx, cudaGraphLaunch(it->second.first, ctx->stream));
  }
  // outside any capture: the record into this round's ring slot, then its event
  if ((rc = record_copy(ctx, slot, cfg->b))) return rc;
  if (!retry_slot)
    ring_push(ctx, tt_ctx::Pending{slot, cfg->b, cfg->k, need, ld, hash, false, *cfg, *sk, *dev, soa, seed,
                                   nullptr, nullptr, nullptr, 0});
  else
    *retry_slot = slot, ctx->ring_next = (slot + 1) % tt_ctx::kRing;
  return TT_OK;
}

int merged_enqueue(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
                   const double* cost, const int64_t* gidx, const uint64_t* id, int64_t m, int* retry_slot = nullptr);

// The oldest round in flight into the caller's buffers (capacity entries
// each). A round whose selector ran out of margin (NEED_MORE: duplicates;
// OVERFLOW: > 4096 ties at the threshold) is re-run synchronously with a
// larger target / the hash path; a tensor-core round whose observed score
// error on the rescored set exceeds its band is re-run in fp64. Both re-runs
// reuse the round's own ring slot.
int round_collect(tt_ctx* ctx, int64_t capacity, int64_t* sel_index, double* sel_score, double* sel_cost,
                  uint64_t* sel_id, tt_round_result* res, bool allow_retry) {
  if (ctx->pend.empty()) return fail(ctx, TT_E_STATE, "round: nothing enqueued");
  const tt_ctx::Pending p = ctx->pend.front();
  if (p.b > capacity)
    return fail(ctx, TT_E_CONFIG, "round_collect: the oldest round selects " + std::to_string(p.b) +
                                      " candidates, the buffers hold " + std::to_string(capacity));
  ctx->pend.pop_front();
  int slot = p.slot;  // a re-run lands in the ring's next slot
  // wait for this round only (the stream may already hold later rounds)
  auto wait_slot = [&]() -> int {
    const cudaError_t e1 = cudaEventSynchronize(ctx->ev_rec[slot]);
    const cudaError_t e2 = cudaGetLastError();
    if (e1 != cudaSuccess || e2 != cudaSuccess)
      return fail(ctx, TT_E_CUDA, std::string("round: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    return TT_OK;
  };
  int rc = wait_slot();
  if (rc) return rc;
  const int64_t b = p.b;
  const int64_t* rec = ctx->h_rec[slot];  // mapped: complete once the slot's event fired
  int retries = 0, extra = 0;
  const int retry_mask = TT_SEL_NEED_MORE | TT_SEL_OVERFLOW;
  if (((int)rec[2] & retry_mask) && allow_retry && !p.merged) {
    int64_t need = p.need;
    bool hash = p.hash;
    bool ok = false;
    for (int attempt = 0; attempt < 62 && !ok; ++attempt) {
      const int st = (int)rec[2];
      if (st & TT_SEL_OVERFLOW) {
        if (hash) break;
        hash = true;
      } else {
        need *= 2;
      }
      tt_round_config cfg = p.cfg;
      if ((rc = round_enqueue(ctx, &p.sketch, &p.dev, &cfg, p.soa, p.ld, p.seed, need, hash, &slot))) return rc;
      if ((rc = wait_slot())) return rc;
      rec = ctx->h_rec[slot];
      ++retries;
      ok = !((int)rec[2] & retry_mask);
    }
    if (!ok && ((int)rec[2] & TT_SEL_NEED_MORE))
      return fail(ctx, TT_E_STATE, "draft selector did not converge");
  }
  if ((int)rec[2] & TT_SEL_INVALID)
    return fail(ctx, TT_E_VALIDATE, "a rank's population holds a schedule that fails validate_schedule");
  if ((int)rec[2] & TT_SEL_OVERFLOW)
    return fail(ctx, TT_E_STATE, p.merged ? "draft selector overflow on a rank: re-run the draft half with tt_round_local"
                                          : "draft selector overflow: more than 4096 unique schedules tie at the threshold");
  if (p.soa && rec[6]) return fail(ctx, TT_E_VALIDATE, "schedule does not satisfy validate_schedule");
  double band_err;
  std::memcpy(&band_err, rec + 5, sizeof(double));
  if (p.cfg.precision != TT_PREC_FP64 && band_err > p.cfg.band && allow_retry) {
    // the observed bf16 error on the rescored set exceeds the certified band:
    // the exclusions are not certified, so the round is re-run in fp64
    tt_round_config cfg = p.cfg;
    cfg.precision = TT_PREC_FP64;
    rc = p.merged ? merged_enqueue(ctx, &p.sketch, &p.dev, &cfg, p.m_cost, p.m_gidx, p.m_id, p.m, &slot)
                  : round_enqueue(ctx, &p.sketch, &p.dev, &cfg, p.soa, p.ld, p.seed, p.need, p.hash, &slot);
    if (rc) return rc;
    if ((rc = wait_slot())) return rc;
    rec = ctx->h_rec[slot];
    extra |= TT_ROUND_BAND_RERUN;
    if ((int)rec[2] & retry_mask) return fail(ctx, TT_E_STATE, "draft selector: fp64 re-run did not converge");
  }
  const int64_t selected = rec[0];
  const int64_t* ix = rec + kRecHead;
  const double* sc = (const double*)(ix + b);
  const double* co = sc + b;
  const uint64_t* ids = (const uint64_t*)(co + b);
  for (int64_t e = 0; e < b; ++e) {
    if (sel_index) sel_index[e] = ix[e];
    if (sel_score) sel_score[e] = sc[e];
    if (sel_cost) sel_cost[e] = co[e];
    if (sel_id) sel_id[e] = ids[e];
  }
  if (res) {
    res->selected = selected;
    res->drafted = rec[1];
    res->rescored = rec[3];
    res->status = (int32_t)rec[2] | extra;
    res->retries = retries + (int32_t)rec[4];
    res->band_err = band_err;
  }
  g_forward_calls.fetch_add((uint64_t)rec[1], std::memory_order_relaxed);
  return TT_OK;
}

int merged_enqueue(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
                   const double* cost, const int64_t* gidx, const uint64_t* id, int64_t m, int* retry_slot) {
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if ((rc = check_round_cfg(ctx, cfg))) return rc;
  if (m < 0 || m > kMergeMax)
    return fail(ctx, TT_E_STATE, "merge: at most " + std::to_string(kMergeMax) + " gathered entries per call");
  if (m > kMergeSortMax && m % cfg->k)
    return fail(ctx, TT_E_STATE, "merge: more than 4096 entries must be whole per-rank lists of k");
  if ((rc = ensure_k(ctx, cfg->k))) return rc;
  if ((rc = ensure_b(ctx, cfg->b))) return rc;
  if (cfg->precision == TT_PREC_BF16 && (rc = ensure_packed(ctx))) return rc;
  int slot = -1;
  if ((rc = ring_claim(ctx, &slot))) return rc;
  prof_begin(ctx, 4);
  if (launch_merge(cost, gidx, id, m, cfg->k, ctx->d_idx, ctx->d_cost, ctx->d_id, ctx->d_count, ctx->sel.state,
                   ctx->sel.mscratch, ctx->stream))
    return fail(ctx, TT_E_STATE, "merge launch");
  prof_end(ctx, 4);
  TT_LAUNCHED(ctx);
  CandRef ref{nullptr, 0, nullptr, 0, ctx->d_id};
  if ((rc = verify_and_select(ctx, S, D, cfg, ref, slot))) return rc;
  if ((rc = record_copy(ctx, slot, cfg->b))) return rc;
  // no selector retry: the local lists are the ranks' own (a rank that could
  // not certify its list marks it, and the merge reports OVERFLOW)
  if (!retry_slot)
    ring_push(ctx, tt_ctx::Pending{slot, cfg->b, cfg->k, -1, 0, false, true, *cfg, *sk, *dev, nullptr, 0, cost, gidx,
                                   id, m});
  else
    *retry_slot = slot, ctx->ring_next = (slot + 1) % tt_ctx::kRing;
  return TT_OK;
}

}  // namespace

extern "C" {

int tt_pacm_score(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const uint64_t* id, int64_t k,
                  int precision, double* score) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if (!ctx->d_params) return fail(ctx, TT_E_STATE, "score: tt_pacm_load first");
  if (k <= 0) return TT_OK;
  const int ns = n_stmt_of(S), nb = n_block_of(S);
  if (precision == TT_PREC_BF16) {
    if (!pacm_tc_supported(ns, nb, ctx->h)) return fail(ctx, TT_E_CONFIG, "tensor-core PaCM: unsupported shape/width");
    if ((rc = ensure_packed(ctx))) return rc;
  } else if (precision != TT_PREC_FP64) {
    return fail(ctx, TT_E_CONFIG, "unknown precision");
  }
  // chunks bound the feature scratch (fp64 rows ~6.4 KB, bf16 tiles 1 KB per candidate)
  const int64_t chunk = precision == TT_PREC_FP64 ? (int64_t)1 << 16 : (int64_t)1 << 20;
  if ((rc = ensure_feat(ctx, k < chunk ? k : chunk))) return rc;
  for (int64_t off = 0; off < k; off += chunk) {
    const int64_t m = k - off < chunk ? k - off : chunk;
    CandRef ref{nullptr, 0, nullptr, 0, id + off};
    if (precision == TT_PREC_FP64) {
      if (launch_feat_rows(S, D, ref, nullptr, m, nullptr, nullptr, ctx->d_xs, ctx->d_xb, nullptr, ctx->stream))
        return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
      if (launch_pacm64(ctx->d_xs, ctx->d_xb, ns, nb, nullptr, m, nullptr, nullptr, ctx->d_params, ctx->h, 0,
                        score + off, ctx->stream))
        return fail(ctx, TT_E_CONFIG, "fp64 PaCM: hidden width too large for shared memory");
    } else {
      if (launch_feat_rows(S, D, ref, nullptr, m, nullptr, nullptr, nullptr, nullptr, ctx->d_tiles, ctx->stream))
        return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
      if (launch_pacm_tc(ctx->d_tiles, ns, nb, nullptr, m, ctx->d_packed, ctx->h, score + off, ctx->stream))
        return fail(ctx, TT_E_CONFIG, "tensor-core PaCM launch");
    }
  }
  TT_LAUNCHED(ctx);
  g_forward_calls.fetch_add((uint64_t)k, std::memory_order_relaxed);
  return TT_OK;
}

int tt_pacm_score_features(tt_ctx* ctx, const double* stmt, const double* block, int n_stmt, int n_block, int64_t k,
                           int attention_identity, double* score) {
  if (!ctx) return TT_E_STATE;
  if (!ctx->d_params) return fail(ctx, TT_E_STATE, "score: tt_pacm_load first");
  if (n_stmt < 1 || n_block < 1)
    return fail(ctx, TT_E_STATE, "feature must have at least one statement and one dataflow block");
  if (n_stmt > 14 || n_block > 20) return fail(ctx, TT_E_STATE, "at most 14 statements and 20 dataflow blocks");
  if (launch_pacm64(stmt, block, n_stmt, n_block, nullptr, k, nullptr, nullptr, ctx->d_params, ctx->h,
                    attention_identity, score, ctx->stream))
    return fail(ctx, TT_E_CONFIG, "fp64 PaCM: hidden width too large for shared memory");
  TT_LAUNCHED(ctx);
  g_forward_calls.fetch_add((uint64_t)(k > 0 ? k : 0), std::memory_order_relaxed);
  return TT_OK;
}

int tt_select_top(tt_ctx* ctx, const double* scores, const double* drafts, const uint8_t* excluded, int64_t n,
                  int64_t b, int64_t* idx_host) {
  if (!ctx) return TT_E_STATE;
  if (b < 1) return fail(ctx, TT_E_STATE, "select_top: b must be >= 1");
  int rc = ensure_b(ctx, b);
  if (rc) return rc;
  if (launch_select_top(scores, drafts, excluded, n, nullptr, b, ctx->d_pos, ctx->d_pos_count, ctx->d_status,
                        ctx->stream))
    return fail(ctx, TT_E_STATE, "select_top: n too large for b (tiles * b must be <= 4096)");
  TT_LAUNCHED(ctx);
  int status = 0;
  int64_t cnt = 0;
  TT_CUDA(ctx, cudaMemcpyAsync(&status, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TT_CUDA(ctx, cudaMemcpyAsync(&cnt, ctx->d_pos_count, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  if ((rc = sync_check(ctx))) return rc;
  if (status)
    return fail(ctx, TT_E_STATE, "select_top: requested " + std::to_string(b) + " but only " + std::to_string(cnt) +
                                     " unmeasured candidates available");
  TT_CUDA(ctx, cudaMemcpy(idx_host, ctx->d_pos, sizeof(int64_t) * b, cudaMemcpyDeviceToHost));
  return TT_OK;
}

// ---------------------------------------------------- simulated hardware --
}  // extern "C"

namespace {
int compile_oracle(tt_ctx* ctx, const tt_oracle_spec* o, DevOracle& O) {
  if (!o) return fail(ctx, TT_E_STATE, "null oracle spec");
  int rc = compile_device(ctx, &o->hidden, O.hidden);
  if (rc) return rc;
  // validate_oracle (oracle.cpp:25-36)
  if (o->stride_coeff < 0.0 || o->occupancy_coeff < 0.0 || o->launch_overhead_s < 0.0 || o->noise_sigma < 0.0)
    return fail(ctx, TT_E_VALIDATE, "oracle coefficients must be non-negative");
  O.stride_coeff = o->stride_coeff, O.occupancy_coeff = o->occupancy_coeff;
  O.launch = o->launch_overhead_s, O.sigma = o->noise_sigma, O.seed = o->seed;
  return TT_OK;
}
}  // namespace

extern "C" {

int tt_oracle_latency(tt_ctx* ctx, const tt_sketch* sk, const tt_oracle_spec* o, const int32_t* soa, int64_t ld,
                      int64_t n, double* latency) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevOracle O;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_oracle(ctx, o, O))) return rc;
  if (launch_oracle_latency(S, O, soa, ld, n, 0, 0, 0, nullptr, latency, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_oracle_measure(tt_ctx* ctx, const tt_sketch* sk, const tt_oracle_spec* o, const int32_t* soa, int64_t ld,
                      int64_t n, uint64_t task_hash, uint64_t trial0, double* latency, double* noiseless) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevOracle O;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_oracle(ctx, o, O))) return rc;
  if (launch_oracle_latency(S, O, soa, ld, n, 1, task_hash, trial0, latency, noiseless, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_oracle_best(tt_ctx* ctx, const tt_sketch* sk, const tt_oracle_spec* o, uint64_t* best_id, double* best_lat) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevOracle O;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_oracle(ctx, o, O))) return rc;
  if (!S.id_exact || S.space > (uint64_t{1} << 40))
    return fail(ctx, TT_E_CONFIG, "oracle_best: schedule space exceeds 2^40");
  // CTA winners in the selector's survivor scratch (4096 entries), result in its hash table
  if (launch_oracle_best(S, O, ctx->sel.skey, (uint64_t*)ctx->sel.sidx, 4096, ctx->sel.tkeys, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);
  uint64_t out[2];
  TT_CUDA(ctx, cudaMemcpyAsync(out, ctx->sel.tkeys, sizeof(out), cudaMemcpyDeviceToHost, ctx->stream));
  TT_CUDA(ctx, cudaMemsetAsync(ctx->sel.tkeys, 0xff, sizeof(out), ctx->stream));  // hash-table invariant
  if ((rc = sync_check(ctx))) return rc;
  if (best_id) *best_id = out[1];
  if (best_lat) std::memcpy(best_lat, &out[0], sizeof(double));
  return TT_OK;
}

// ------------------------------------------------------------- training --
}  // extern "C"

namespace {

// RngStream (common.hpp:87-119) on the host: the batch sampling of train()
struct HostRng {
  uint64_t s;
  explicit HostRng(uint64_t seed) : s(seed ? seed : kGolden) {}
  uint64_t next() {
    s += kGolden;
    return scramble64(s);
  }
  uint64_t index(uint64_t n) { return (uint64_t)(((unsigned __int128)next() * n) >> 64); }
};

uint64_t mix64_h(uint64_t x) { return scramble64(x + kGolden); }
uint64_t derive_seed_h(uint64_t base, uint64_t a) { return mix64_h(base ^ mix64_h(a)); }

// grow-only scratch, doubling (the MoA loop's dataset grows by b records a
// round; no graph invalidation: training is never captured)
template <class T>
int tgrow(tt_ctx* ctx, T*& p, int64_t& cap, int64_t want) {
  if (want <= cap && p) return TT_OK;
  if (want < 2 * cap) want = 2 * cap;
  if (p) cudaFree(p);
  p = nullptr, cap = 0;
  TT_CUDA(ctx, cudaMalloc((void**)&p, sizeof(T) * (size_t)(want > 0 ? want : 1)));
  cap = want;
  return TT_OK;
}

}  // namespace

extern "C" {

int tt_rank_loss(tt_ctx* ctx, const double* scores, const double* latencies, int64_t n, double* loss_host,
                 double* grad) {
  if (!ctx) return TT_E_STATE;
  if (n < 2) return fail(ctx, TT_E_STATE, "rank loss: need at least two items");
  if (n > (int64_t)1 << 20) return fail(ctx, TT_E_CONFIG, "rank loss: at most 2^20 items");
  auto& T = ctx->tr;
  int rc;
  if ((rc = tgrow(ctx, T.rank, T.rank_cap, (int64_t)rank_work_doubles((int)n)))) return rc;
  if ((rc = tgrow(ctx, T.loss, T.loss_cap, 1))) return rc;
  if ((rc = tgrow(ctx, T.bad, T.bad_cap, 1))) return rc;
  TT_CUDA(ctx, cudaMemsetAsync(T.bad, 0, sizeof(int), ctx->stream));
  if (launch_rank_loss(scores, latencies, nullptr, (int)n, T.rank, T.bad, T.loss, 0, grad, ctx->stream))
    return fail(ctx, TT_E_CUDA, "rank loss launch");
  TT_LAUNCHED(ctx);
  int bad = 0;
  double l = 0.0;
  TT_CUDA(ctx, cudaMemcpyAsync(&bad, T.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TT_CUDA(ctx, cudaMemcpyAsync(&l, T.loss, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  if ((rc = sync_check(ctx))) return rc;
  if (bad) return fail(ctx, TT_E_STATE, "rank loss: latencies must be positive");
  if (loss_host) *loss_host = l;
  return TT_OK;
}

// train(params, {one task}, cfg) (ranker.cpp:459-512), entirely on the
// device: every epoch's batch indices are drawn on the host up front (the
// reference's RngStream and partial Fisher-Yates) and uploaded once; each
// epoch is forward (k_train_fwd) -> LambdaRank loss + score gradient
// (k_rank_*) -> score_backward + gradient sums (k_train_bwd/accum) -> GD,
// with no host round trip; the losses come back in one copy at the end.
// Scratch is cached on the context.
int tt_pacm_train(tt_ctx* ctx, double* params, int h, const double* stmt, const double* block, int n_stmt,
                  int n_block, const double* latencies, int64_t n, int epochs, double lr, int batch, uint64_t seed,
                  int attention_identity, double* initial_loss, double* final_loss) {
  if (!ctx) return TT_E_STATE;
  if (n < 2) return fail(ctx, TT_E_STATE, "train: dataset needs at least two labeled schedules");
  if (epochs < 0) return fail(ctx, TT_E_STATE, "train: epochs must be >= 0");
  if (h < 1 || n_stmt < 1 || n_block < 1 || n_stmt > 14 || n_block > 20)
    return fail(ctx, TT_E_STATE, "train: unsupported model / feature geometry");
  if (n > (int64_t)1 << 20) return fail(ctx, TT_E_CONFIG, "train: at most 2^20 records");
  for (int64_t i = 0; i < n; ++i)
    if (!(latencies[i] > 0.0)) return fail(ctx, TT_E_STATE, "rank loss: latencies must be positive");
  const int64_t take = (batch > 0 && batch < n) ? batch : n;
  const size_t slot = train_slot_doubles(n_stmt, n_block, h);
  const int64_t np = tt_param_count(h);
  const int ctas = 8 * 148;
  auto& T = ctx->tr;
  int rc;
  if ((rc = tgrow(ctx, T.slots, T.slots_cap, (int64_t)(slot * n)))) return rc;
  if ((rc = tgrow(ctx, T.work, T.work_cap, (int64_t)train_work_doubles(n_stmt, n_block, h, ctas)))) return rc;
  if ((rc = tgrow(ctx, T.grads, T.grads_cap, np))) return rc;
  if ((rc = tgrow(ctx, T.dscore, T.dscore_cap, n))) return rc;
  if ((rc = tgrow(ctx, T.scores, T.scores_cap, n))) return rc;
  if ((rc = tgrow(ctx, T.rank, T.rank_cap, (int64_t)rank_work_doubles((int)n)))) return rc;
  if ((rc = tgrow(ctx, T.lat, T.lat_cap, n))) return rc;
  if ((rc = tgrow(ctx, T.loss, T.loss_cap, (int64_t)epochs + 2))) return rc;
  if ((rc = tgrow(ctx, T.list, T.list_cap, take * (int64_t)(epochs > 0 ? epochs : 1)))) return rc;
  if ((rc = tgrow(ctx, T.bad, T.bad_cap, 1))) return rc;
  if (ctx->h_loss_cap < (int64_t)epochs + 2) {
    if (ctx->h_loss) cudaFreeHost(ctx->h_loss);
    ctx->h_loss = nullptr, ctx->h_loss_cap = 0;
    TT_CUDA(ctx, cudaMallocHost((void**)&ctx->h_loss, sizeof(double) * (epochs + 2)));
    ctx->h_loss_cap = epochs + 2;
  }
  // every epoch's batch (ranker.cpp:475-486), host RNG, one upload
  std::vector<int32_t> lists((size_t)take * (epochs > 0 ? epochs : 1));
  {
    HostRng rng(derive_seed_h(seed, 0x7261696eULL));
    std::vector<int32_t> idx((size_t)n);
    for (int e = 0; e < epochs; ++e) {
      for (int64_t i = 0; i < n; ++i) idx[i] = (int32_t)i;
      if (take < n)  // partial Fisher-Yates
        for (int64_t i = 0; i < take; ++i) std::swap(idx[i], idx[i + (int64_t)rng.index((uint64_t)(n - i))]);
      std::copy(idx.begin(), idx.begin() + take, lists.begin() + (size_t)e * take);
    }
  }
  TT_CUDA(ctx, cudaMemcpyAsync(T.lat, latencies, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  if (epochs > 0)
    TT_CUDA(ctx, cudaMemcpyAsync(T.list, lists.data(), sizeof(int32_t) * lists.size(), cudaMemcpyHostToDevice,
                                 ctx->stream));
  TT_CUDA(ctx, cudaMemsetAsync(T.bad, 0, sizeof(int), ctx->stream));
  auto dataset_loss = [&](double* out) -> int {  // ranker.cpp:445-455
    launch_train_fwd(stmt, block, n_stmt, n_block, nullptr, (int)n, params, h, attention_identity, T.slots,
                     T.scores, ctx->stream);
    TT_LAUNCHED(ctx);
    if (launch_rank_loss(T.scores, T.lat, nullptr, (int)n, T.rank, T.bad, out, 0, nullptr, ctx->stream))
      return fail(ctx, TT_E_CUDA, "rank loss launch");
    return TT_OK;
  };
  if ((rc = dataset_loss(T.loss))) return rc;
  for (int e = 0; e < epochs; ++e) {
    const int32_t* list = T.list + (size_t)e * take;
    launch_train_fwd(stmt, block, n_stmt, n_block, list, (int)take, params, h, attention_identity, T.slots, T.scores,
                     ctx->stream);
    TT_LAUNCHED(ctx);
    // epoch loss (ranker.cpp:491-492) into loss[2 + e], score gradient into dscore
    if (launch_rank_loss(T.scores, T.lat, list, (int)take, T.rank, T.bad, T.loss + 2 + e, 0,
                         lr == 0.0 ? nullptr : T.dscore, ctx->stream))
      return fail(ctx, TT_E_CUDA, "rank loss launch");
    if (lr == 0.0) continue;
    launch_train_bwd(n_stmt, n_block, (int)take, params, h, attention_identity, T.dscore, T.slots, T.work, ctas,
                     ctx->stream);
    launch_train_accum(n_stmt, n_block, (int)take, h, attention_identity, T.slots, T.grads, ctx->stream);
    launch_gd_step(params, T.grads, np, lr, ctx->stream);  // p -= lr * g (ranker.cpp:502-506)
    TT_LAUNCHED(ctx);
  }
  if ((rc = dataset_loss(T.loss + 1))) return rc;
  TT_CUDA(ctx, cudaMemcpyAsync(ctx->h_loss, T.loss, sizeof(double) * (epochs + 2), cudaMemcpyDeviceToHost,
                               ctx->stream));
  int bad = 0;
  TT_CUDA(ctx, cudaMemcpyAsync(&bad, T.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  if ((rc = sync_check(ctx))) return rc;
  if (bad) return fail(ctx, TT_E_STATE, "rank loss: latencies must be positive");
  if (initial_loss) *initial_loss = ctx->h_loss[0];
  if (final_loss) *final_loss = ctx->h_loss[1];
  return TT_OK;
}

int tt_gd_step(tt_ctx* ctx, double* params, const double* grads, int64_t n, double lr) {
  if (!ctx) return TT_E_STATE;
  launch_gd_step(params, grads, n, lr, ctx->stream);
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_momentum_update(tt_ctx* ctx, double* phi, const double* target, int64_t n, double m) {
  if (!ctx) return TT_E_STATE;
  if (!(m >= 0.0 && m < 1.0)) return fail(ctx, TT_E_STATE, "momentum must lie in [0, 1)");
  launch_momentum(phi, target, n, m, ctx->stream);
  TT_LAUNCHED(ctx);
  return TT_OK;
}

int tt_round_async(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
                   const int32_t* soa, int64_t ld, uint64_t seed) {
  if (!ctx) return TT_E_STATE;
  if (!cfg) return fail(ctx, TT_E_STATE, "null round config");
  return round_enqueue(ctx, sk, dev, cfg, soa, ld, seed, cfg->k + cfg->k / 8 + 16);
}

int tt_round_collect(tt_ctx* ctx, int64_t capacity, int64_t* sel_index, double* sel_score, double* sel_cost,
                     uint64_t* sel_id, tt_round_result* res) {
  if (!ctx) return TT_E_STATE;
  return round_collect(ctx, capacity, sel_index, sel_score, sel_cost, sel_id, res, true);
}

int tt_round(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
             const int32_t* soa, int64_t ld, uint64_t seed, int64_t* sel_index, double* sel_score, double* sel_cost,
             uint64_t* sel_id, tt_round_result* res) {
  if (ctx && !ctx->pend.empty())
    return fail(ctx, TT_E_STATE, "tt_round: rounds still in flight on this context (tt_round_collect them first)");
  int rc = tt_round_async(ctx, sk, dev, cfg, soa, ld, seed);
  if (rc) return rc;
  return round_collect(ctx, cfg->b, sel_index, sel_score, sel_cost, sel_id, res, true);
}

int tt_round_local_async(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
                         const int32_t* soa, int64_t ld, uint64_t seed, double* cost_out, int64_t* gidx_out,
                         uint64_t* id_out) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if ((rc = check_round_cfg(ctx, cfg))) return rc;
  if (!S.id_exact) return fail(ctx, TT_E_STATE, "round: schedule space exceeds 2^64 identities");
  const bool seeded = soa == nullptr;
  if (cfg->n > kSmallSelectMax && (rc = ensure_cost(ctx, cfg->n))) return rc;
  TT_CUDA(ctx, cudaMemsetAsync(gidx_out, 0xff, sizeof(int64_t) * cfg->k, ctx->stream));  // -1 = empty slot
  TT_CUDA(ctx, cudaMemsetAsync(cost_out, 0, sizeof(double) * cfg->k, ctx->stream));
  TT_CUDA(ctx, cudaMemsetAsync(id_out, 0, sizeof(uint64_t) * cfg->k, ctx->stream));
  if (S.space < (uint64_t)cfg->n * 64) {
    // a small schedule space: duplicates may exhaust the device selector's
    // margin (> 4096 tied survivors), so select synchronously with the
    // host-driven hash fallback rather than fail the merged round
    int64_t cnt = 0;
    return select_sync(ctx, S, D, soa, ld, seed_state(seed), cfg->first, seeded, cfg->n, cfg->k, cfg->toggles,
                       cfg->first, gidx_out, cost_out, id_out, &cnt);
  }
  prof_begin(ctx, 0);  // sel.invalid is zero between calls; k_mark_invalid resets it
  if (launch_select(S, D, soa, ld, seed_state(seed), cfg->first, seeded, cfg->n, cfg->k,
                    cfg->k + cfg->k / 8 + 16, cfg->toggles, cfg->first, ctx->sel, gidx_out, cost_out, id_out,
                    ctx->d_count, ctx->stream))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  prof_end(ctx, 0);
  TT_LAUNCHED(ctx);
  // an explicit population with an invalid schedule marks the payload: every
  // rank's merged round then fails with TT_E_VALIDATE
  if (!seeded) {
    if (launch_mark_invalid(ctx->sel.invalid, gidx_out, ctx->stream)) return fail(ctx, TT_E_CUDA, "mark launch");
    TT_LAUNCHED(ctx);
  }
  return TT_OK;
}

int tt_round_local(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
                   const int32_t* soa, int64_t ld, uint64_t seed, double* cost_out, int64_t* gidx_out,
                   uint64_t* id_out) {
  if (!ctx) return TT_E_STATE;
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if ((rc = check_round_cfg(ctx, cfg))) return rc;
  if (!S.id_exact) return fail(ctx, TT_E_STATE, "round: schedule space exceeds 2^64 identities");
  TT_CUDA(ctx, cudaMemsetAsync(gidx_out, 0xff, sizeof(int64_t) * cfg->k, ctx->stream));
  TT_CUDA(ctx, cudaMemsetAsync(cost_out, 0, sizeof(double) * cfg->k, ctx->stream));
  TT_CUDA(ctx, cudaMemsetAsync(id_out, 0, sizeof(uint64_t) * cfg->k, ctx->stream));
  int64_t cnt = 0;
  return select_sync(ctx, S, D, soa, ld, seed_state(seed), cfg->first, soa == nullptr, cfg->n, cfg->k, cfg->toggles,
                     cfg->first, gidx_out, cost_out, id_out, &cnt);
}

int tt_round_finish_merged_async(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev,
                                 const tt_round_config* cfg, const double* cost, const int64_t* gidx,
                                 const uint64_t* id, int64_t m) {
  if (!ctx) return TT_E_STATE;
  return merged_enqueue(ctx, sk, dev, cfg, cost, gidx, id, m);
}

int tt_round_finish_merged(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
                           const double* cost, const int64_t* gidx, const uint64_t* id, int64_t m, int64_t* sel_index,
                           double* sel_score, double* sel_cost, uint64_t* sel_id, tt_round_result* res) {
  if (ctx && !ctx->pend.empty())
    return fail(ctx, TT_E_STATE, "tt_round_finish_merged: rounds still in flight (tt_round_collect them first)");
  int rc = tt_round_finish_merged_async(ctx, sk, dev, cfg, cost, gidx, id, m);
  if (rc) return rc;
  return round_collect(ctx, cfg->b, sel_index, sel_score, sel_cost, sel_id, res, true);
}

int tt_profile_enable(tt_ctx* ctx, int on) {
  if (!ctx) return TT_E_STATE;
  ctx->prof = on != 0;
  return TT_OK;
}

int tt_profile_read(tt_ctx* ctx, double* ms_sum, int64_t* count, int n_stages) {
  if (!ctx) return TT_E_STATE;
  int rc = sync_check(ctx);
  if (rc) return rc;
  for (int s = 0; s < n_stages; ++s) ms_sum[s] = 0.0, count[s] = 0;
  for (auto& [stage, pr] : ctx->ev_live) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pr.first, pr.second);
    if (stage < n_stages) ms_sum[stage] += ms, count[stage] += 1;
    ctx->ev_pool.push_back(pr.first);
    ctx->ev_pool.push_back(pr.second);
  }
  ctx->ev_live.clear();
  return TT_OK;
}

int tt_round_drafted(const tt_ctx* ctx, const int64_t** idx, const double** cost, const uint64_t** id,
                     const double** score) {
  if (!ctx || !ctx->d_idx) return TT_E_STATE;
  if (idx) *idx = ctx->d_idx;
  if (cost) *cost = ctx->d_cost;
  if (id) *id = ctx->d_id;
  if (score) *score = ctx->d_score;
  return TT_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------
// explore() with n_steps > 1: the reference's genetic draft loop
// (draft.cpp:156-221). Each generation's draft costs and identities are
// computed on the device (K1 + identity kernels, bit-exact); the pool
// bookkeeping and mutate() (schedule.cpp:340-396) stay on the host because
// mutate consumes ONE sequential RngStream whose draw count per child depends
// on the parent it picked — every child's offset in the stream depends on all
// earlier children. The pool is keyed by the exact 64-bit identity, which is
// injective, hence equivalent to schedule_key's string (schedule.cpp:280-296).
namespace {

// One generation in a flat slot (device or pinned host): soa (ld n) |
// cost [n] | identity [n]; a whole slot moves in one copy.
struct GenSlot {
  int32_t* soa;
  double* cost;
  uint64_t* id;
};
size_t gen_bytes(int64_t n, int cols) { return (((size_t)n * cols * 4 + 15) & ~(size_t)15) + 16 * (size_t)n; }
GenSlot gen_slot(void* base, int64_t n, int cols, int which) {
  char* p = (char*)base + (size_t)which * gen_bytes(n, cols);
  GenSlot g;
  g.soa = (int32_t*)p;
  g.cost = (double*)(p + (((size_t)n * cols * 4 + 15) & ~(size_t)15));
  g.id = (uint64_t*)(g.cost + n);
  return g;
}

int ensure_explore(tt_ctx* ctx, int64_t n, int cols, int host_slots, int nflag) {
  const size_t dwant = (size_t)std::max(2, host_slots) * gen_bytes(n, cols) + 16;  // device path: one slot per generation
  const size_t hwant = (size_t)host_slots * gen_bytes(n, cols) + 4 * (size_t)host_slots * nflag + 16;  // + flags
  if (dwant > ctx->ex_dcap) {
    cudaFree(ctx->d_ex);
    ctx->d_ex = nullptr, ctx->ex_dcap = 0;
    TT_CUDA(ctx, cudaMalloc(&ctx->d_ex, dwant));
    ctx->ex_dcap = dwant;
  }
  if (hwant > ctx->ex_hcap) {
    if (ctx->h_ex) cudaFreeHost(ctx->h_ex);
    ctx->h_ex = nullptr, ctx->ex_hcap = 0;
    TT_CUDA(ctx, cudaMallocHost(&ctx->h_ex, hwant));
    ctx->ex_hcap = hwant;
  }
  while ((int)ctx->ex_ev.size() < host_slots) {
    cudaEvent_t e;
    TT_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->ex_ev.push_back(e);
  }
  return TT_OK;
}

// mutate(population, sketch, costs, rng) (schedule.cpp:340-396) on SoA
// columns: pop (ld n) -> next (ld n), same draw sequence as the reference.
void mutate_h(const DevSketch& S, const tt_sketch* sk, const int32_t* pop, const double* costs, int64_t n,
              HostRng& rng, int32_t* next) {
  constexpr double kEps = 1e-12;
  std::vector<double> cumulative((size_t)n);
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    total += 1.0 / (costs[i] + kEps);
    cumulative[(size_t)i] = total;
  }
  int64_t best = 0;
  for (int64_t i = 1; i < n; ++i)
    if (costs[i] < costs[best]) best = i;
  const int cols = S.cols, n_axes = S.n_axes;
  const int ucol = 4 * S.n_sp + 3 * S.n_red;
  for (int c = 0; c < cols; ++c) next[(int64_t)c * n] = pop[(int64_t)c * n + best];  // elite
  int32_t f[4];
  int mv_pos[64];
  int64_t mv_p[64];
  for (int64_t j = 1; j < n; ++j) {
    const double r = (double)(rng.next() >> 11) * 0x1.0p-53 * total;
    int64_t par = std::upper_bound(cumulative.begin(), cumulative.end(), r) - cumulative.begin();
    if (par > n - 1) par = n - 1;
    for (int c = 0; c < cols; ++c) next[(int64_t)c * n + j] = pop[(int64_t)c * n + par];
    const int slot = (int)rng.index((uint64_t)n_axes + 1);
    if (slot == n_axes) {
      next[(int64_t)ucol * n + j] = sk->unroll[rng.index((uint64_t)sk->n_unroll)];
      continue;
    }
    const int col0 = slot < S.n_sp ? 4 * slot : 4 * S.n_sp + 3 * (slot - S.n_sp);
    const int arity = S.arity[slot];
    for (int q = 0; q < arity; ++q) f[q] = next[(int64_t)(col0 + q) * n + j];
    // prime_factorize(f[q]) (schedule.cpp:93-108): every factor divides the
    // axis extent, so only the extent's primes (ascending) occur; exponents
    // by ctz for 2 and by exact-division inverses for odd primes (no idiv)
    int n_moves = 0;
    for (int q = 0; q < arity; ++q) {
      uint32_t v = (uint32_t)f[q];
      for (int t = 0; t < S.n_prime && v > 1; ++t) {
        if (S.pr_axis[t] != slot) continue;
        const int32_t p = (int32_t)S.pr_p[t];
        int e = 0;
        if (p == 2) {
          e = __builtin_ctz(v);
          v >>= e;
        } else {
          for (uint32_t qv = v * S.pr_inv[t]; qv <= S.pr_lim[t]; qv = v * S.pr_inv[t]) v = qv, ++e;
        }
        for (int rep = 0; rep < e && n_moves < 64; ++rep) mv_pos[n_moves] = q, mv_p[n_moves++] = p;
      }
    }
    if (n_moves > 0 && arity > 1) {
      const int m = (int)rng.index((uint64_t)n_moves);
      const int from = mv_pos[m];
      const int64_t prime = mv_p[m];
      int to = (int)rng.index((uint64_t)arity - 1);
      if (to >= from) ++to;
      next[(int64_t)(col0 + from) * n + j] = (int32_t)(f[from] / prime);
      next[(int64_t)(col0 + to) * n + j] = (int32_t)(f[to] * prime);
    }
  }
}

}  // namespace

namespace {
double g_ex_stamp[8];  // host timeline of the last tt_explore (ttdbg_explore_stamps), microseconds
double g_ex_watch_s = 0;  // debugging: give up on a generation flag after this many seconds
inline double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace
extern "C" int ttdbg_explore_watch(double seconds) {
  g_ex_watch_s = seconds;
  return 0;
}
extern "C" int ttdbg_explore_stamps(double* out) {
  for (int i = 0; i < 8; ++i) out[i] = g_ex_stamp[i] - g_ex_stamp[0];
  return 0;
}

int tt_explore(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t k, int64_t n,
               uint64_t seed, int toggles, int32_t* soa_host, double* cost_host, uint64_t* id_host,
               int64_t* count_host, uint64_t* evaluations) {
  g_ex_stamp[0] = now_us();
  if (!ctx) return TT_E_STATE;
  if (n_steps < 1) return fail(ctx, TT_E_STATE, "explore: n_steps must be >= 1");
  if (k < 1) return fail(ctx, TT_E_STATE, "explore: draft_size must be >= 1");
  if (n < 2) return fail(ctx, TT_E_STATE, "explore: pop_size must be >= 2");
  if (!count_host || !cost_host) return fail(ctx, TT_E_STATE, "explore: null output");
  DevSketch S;
  DevDevice D;
  int rc = compile_sketch(ctx, sk, S);
  if (rc) return rc;
  if ((rc = compile_device(ctx, dev, D))) return rc;
  if (!S.id_exact) return fail(ctx, TT_E_STATE, "explore: schedule space exceeds 2^64 identities");
  if (n > (int64_t)1 << 31) return fail(ctx, TT_E_STATE, "explore: pop_size too large");
  const int cols = S.cols;
  // Device generations (mutate on the GPU, nothing on the host's critical
  // path) when one CTA holds the roulette wheel and the pinned mirror of all
  // generations stays modest; otherwise mutate() runs on the host between
  // device generations.
  const bool on_device = n <= kMutateMaxN && (size_t)n_steps * gen_bytes(n, cols) <= ((size_t)1 << 30);
  const int host_slots = on_device ? n_steps : 2;
  const int nflag = on_device ? explore_cluster_size(n) : 1;  // flags per generation
  if ((rc = ensure_explore(ctx, n, cols, host_slots, nflag))) return rc;
  GenSlot dgen[1] = {gen_slot(ctx->d_ex, n, cols, 0)};  // generation 0 (device path: slot g holds generation g)
  volatile uint32_t* h_flags = (volatile uint32_t*)((char*)ctx->h_ex + (size_t)host_slots * gen_bytes(n, cols));
  auto hgen = [&](int i) { return gen_slot(ctx->h_ex, n, cols, i); };
  const uint64_t s0 = seed_state(seed);
  // random_init(sketch, n, rng) consumes n * draws_per_schedule draws of the
  // stream; mutate() continues from there
  const uint64_t s_init = s0 + (uint64_t)n * (uint64_t)(S.n_prime + 1) * kGolden;
  cudaStream_t st = ctx->stream;
  auto cost_and_copy = [&](GenSlot& d, GenSlot& h, cudaEvent_t ev) -> int {
    if (launch_draft_cost(S, D, d.soa, n, 0, 0, false, n, toggles, d.cost, nullptr, ctx->sel.invalid, st))
      return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
    TT_LAUNCHED(ctx);
    TT_CUDA(ctx, cudaMemcpyAsync(h.soa, d.soa, gen_bytes(n, cols), cudaMemcpyDeviceToHost, st));
    TT_CUDA(ctx, cudaEventRecord(ev, st));
    return TT_OK;
  };
  if (launch_generate(S, s0, 0, n, dgen[0].soa, n, dgen[0].id, st))
    return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
  TT_LAUNCHED(ctx);

  // the pool (draft.cpp:166-170): (cost, discovery, identity, where its
  // factors are) entries, trimmed in place with nth_element; membership by an
  // open-addressing table over identities, cleared in O(1) per trim by
  // bumping its epoch. On the device path every generation's pinned slot
  // stays alive, so an entry just points at its column (generation * n +
  // index); the host path copies factor rows into an arena.
  struct PE {
    double cost;
    uint64_t disc, id, ref;
  };
  const int64_t cap = k + n;
  std::vector<PE> pool;
  pool.reserve((size_t)cap);
  std::vector<int32_t> rows, rows_t;  // host path only
  if (!on_device) rows.resize((size_t)(cap * cols)), rows_t.resize((size_t)(k * cols));
  int hbits = 4;
  while (((int64_t)1 << hbits) < 2 * cap) ++hbits;
  const uint64_t hmask = ((uint64_t)1 << hbits) - 1;
  std::vector<uint64_t> h_key((size_t)hmask + 1);
  std::vector<uint32_t> h_epoch((size_t)hmask + 1, 0);
  uint32_t epoch = 1;
  auto h_insert = [&](uint64_t id) -> bool {  // true if id was new
    for (uint64_t h = scramble64(id) & hmask;; h = (h + 1) & hmask) {
      if (h_epoch[h] != epoch) {
        h_epoch[h] = epoch, h_key[h] = id;
        return true;
      }
      if (h_key[h] == id) return false;
    }
  };
  uint64_t discovery = 0;
  auto by_cost = [](const PE& a, const PE& b) { return a.cost != b.cost ? a.cost < b.cost : a.disc < b.disc; };
  // pool insertion in population order (first discovery wins,
  // draft.cpp:198-204) + trim to the k smallest (cost, discovery) (:174-191)
  // Once the pool is full, an entry whose cost is >= the worst kept cost
  // can never survive a trim (k kept entries precede it in (cost, discovery)
  // order: its discovery is later), so it is skipped before the membership
  // probe. Discovery numbers then have gaps, which keeps their order.
  double bar = std::numeric_limits<double>::infinity();
  auto consume = [&](const GenSlot& g, int gen) {
    for (int64_t i = 0; i < n; ++i) {
      if (!(g.cost[i] < bar)) continue;
      if (!h_insert(g.id[i])) continue;
      PE e{g.cost[i], discovery++, g.id[i], 0};
      if (on_device) {
        e.ref = (uint64_t)gen * (uint64_t)n + (uint64_t)i;
      } else {
        e.ref = pool.size();
        for (int c = 0; c < cols; ++c) rows[e.ref * cols + c] = g.soa[(int64_t)c * n + i];
      }
      pool.push_back(e);
    }
    if ((int64_t)pool.size() > k) {
      std::nth_element(pool.begin(), pool.begin() + k, pool.end(), by_cost);
      pool.resize((size_t)k);
      ++epoch;
      for (size_t q = 0; q < pool.size(); ++q) {
        h_insert(pool[q].id);
        if (!on_device) {
          std::memcpy(&rows_t[q * cols], &rows[pool[q].ref * cols], sizeof(int32_t) * cols);
          pool[q].ref = q;
        }
      }
      if (!on_device) std::copy(rows_t.begin(), rows_t.begin() + (size_t)k * cols, rows.begin());
    }
    if ((int64_t)pool.size() == k) {
      bar = pool[0].cost;
      for (const PE& e : pool) bar = e.cost > bar ? e.cost : bar;
    }
  };

  if (on_device) {
    // one persistent CTA runs every generation (mutate -> identity -> draft
    // cost) and publishes each to its pinned slot + flag; the host folds
    // generation g into the pool as soon as its flag is up
    for (int g = 0; g < n_steps * nflag; ++g) h_flags[g] = 0u;
    g_ex_stamp[1] = now_us();
    const size_t cost_off = (size_t)((char*)hgen(0).cost - (char*)ctx->h_ex);
    const int lrc = launch_explore_gens(S, D, toggles, n, n_steps, ctx->d_ex, gen_bytes(n, cols), cost_off, s_init,
                                        ctx->h_ex, gen_bytes(n, cols), cost_off, h_flags, st);
    if (lrc == 2) return fail(ctx, TT_E_CUDA, std::string("explore: cluster launch: ") +
                                                  cudaGetErrorString(cudaGetLastError()));
    if (lrc) return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
    TT_LAUNCHED(ctx);
    g_ex_stamp[2] = now_us();
    for (int g = 0; g < n_steps; ++g) {
      if (g == 1) g_ex_stamp[3] = now_us();
      if (g == n_steps - 1) g_ex_stamp[4] = now_us();
      for (int f = g * nflag; f < (g + 1) * nflag; ++f)
      for (uint64_t spin = 0; h_flags[f] == 0u; ++spin) {
        if (g_ex_watch_s > 0 && (spin & 0xffff) == 0xffff && now_us() - g_ex_stamp[0] > 1e6 * g_ex_watch_s)
          return fail(ctx, TT_E_STATE, "explore: generation " + std::to_string(g) + " flag " + std::to_string(f) +
                                           " not published within the watch limit (kernel stuck)");
        if ((spin & 1023) == 1023) {  // a faulted or finished kernel never raises the flag
          const cudaError_t q = cudaStreamQuery(st);
          if (q != cudaErrorNotReady && h_flags[f] == 0u) {
            if (q != cudaSuccess) return fail(ctx, TT_E_CUDA, cudaGetErrorString(q));
            return fail(ctx, TT_E_STATE, "explore: generation kernel ended without publishing");
          }
        }
      }
      std::atomic_thread_fence(std::memory_order_acquire);
      if (g == n_steps - 1) g_ex_stamp[5] = now_us();
      consume(hgen(g), g);
    }
    if ((rc = sync_check(ctx))) return rc;
    g_ex_stamp[6] = now_us();
    // factor columns stay in the device slots; fetched only when asked for
    if (soa_host) {
      TT_CUDA(ctx, cudaMemcpyAsync(ctx->h_ex, ctx->d_ex, (size_t)n_steps * gen_bytes(n, cols), cudaMemcpyDeviceToHost,
                                   st));
      if ((rc = sync_check(ctx))) return rc;
    }
  } else {
    GenSlot h0 = hgen(0);
    if ((rc = cost_and_copy(dgen[0], h0, ctx->ex_ev[0]))) return rc;
    if ((rc = sync_check(ctx))) return rc;
    HostRng rng(s0);
    rng.s = s_init;
    int cur = 0;
    for (int step = 0; step < n_steps; ++step) {
      GenSlot g = hgen(cur), nx = hgen(cur ^ 1);
      const bool more = step + 1 < n_steps;
      if (more) {  // critical path: mutate on the host, the next generation's device work
        mutate_h(S, sk, g.soa, g.cost, n, rng, nx.soa);
        TT_CUDA(ctx, cudaMemcpyAsync(dgen[0].soa, nx.soa, sizeof(int32_t) * n * cols, cudaMemcpyHostToDevice, st));
        if (launch_identity(S, dgen[0].soa, n, n, dgen[0].id, st))
          return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
        TT_LAUNCHED(ctx);
        if ((rc = cost_and_copy(dgen[0], nx, ctx->ex_ev[cur ^ 1]))) return rc;
      }
      consume(g, step);  // overlaps the device
      if (more) {
        if ((rc = sync_check(ctx))) return rc;
        cur ^= 1;
      }
    }
  }
  std::sort(pool.begin(), pool.end(), by_cost);
  const int64_t cnt = (int64_t)pool.size();
  for (int64_t q = 0; q < cnt; ++q) {
    const PE& e = pool[(size_t)q];
    cost_host[q] = e.cost;
    if (id_host) id_host[q] = e.id;
    if (soa_host) {
      if (on_device) {
        const GenSlot g = hgen((int)(e.ref / (uint64_t)n));
        const int64_t i = (int64_t)(e.ref % (uint64_t)n);
        for (int c = 0; c < cols; ++c) soa_host[(int64_t)c * k + q] = g.soa[(int64_t)c * n + i];
      } else {
        for (int c = 0; c < cols; ++c) soa_host[(int64_t)c * k + q] = rows[e.ref * cols + c];
      }
    }
  }
  *count_host = cnt;
  if (evaluations) *evaluations = (uint64_t)n_steps * (uint64_t)n;
  g_ex_stamp[7] = now_us();
  return TT_OK;
}

// The tuner's draft set (Tuner::build_draft_set, tuner.cpp:294-323): the
// explore() pool of n_spec = max(1, llround((1 - random_mix) * draft_size))
// schedules, then draft_size - n_spec fresh random_init schedules of the mix
// stream, each appended (with its draft cost) unless its key was seen.
int tt_draft_set(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t draft_size,
                 int64_t pop_size, double random_mix, uint64_t explore_seed, uint64_t mix_seed, int toggles,
                 uint64_t* id_host, double* cost_host, int64_t* count_host, uint64_t* evaluations) {
  if (!ctx) return TT_E_STATE;
  if (!(random_mix >= 0.0 && random_mix < 1.0)) return fail(ctx, TT_E_CONFIG, "random_mix must be in [0, 1)");
  if (draft_size < 1) return fail(ctx, TT_E_CONFIG, "draft_size must be >= 1");
  if (!id_host || !cost_host || !count_host) return fail(ctx, TT_E_STATE, "draft_set: null output");
  const int64_t n_spec = std::max<int64_t>(1, std::llround((1.0 - random_mix) * (double)draft_size));
  const int64_t n_random = draft_size - n_spec;
  int64_t cnt = 0;
  int rc = TT_OK;
  // the random mix does not depend on the explore: it is generated and costed
  // on the side stream while the GA cluster kernel runs (8 SMs of 148)
  double* mc = nullptr;
  uint64_t* mi = nullptr;
  if (n_random > 0) {
    DevSketch S;
    DevDevice D;
    if ((rc = compile_sketch(ctx, sk, S))) return rc;
    if ((rc = compile_device(ctx, dev, D))) return rc;
    const size_t want = gen_bytes(n_random, S.cols);
    if (want > ctx->mix_cap) {
      cudaFree(ctx->d_mix);
      ctx->d_mix = nullptr, ctx->mix_cap = 0;
      TT_CUDA(ctx, cudaMalloc(&ctx->d_mix, want));
      ctx->mix_cap = want;
    }
    const size_t hwant = (size_t)n_random * 16;
    if (hwant > ctx->h_mix_cap) {
      cudaFreeHost(ctx->h_mix);
      ctx->h_mix = nullptr, ctx->h_mix_cap = 0;
      TT_CUDA(ctx, cudaHostAlloc(&ctx->h_mix, hwant, cudaHostAllocDefault));
      ctx->h_mix_cap = hwant;
    }
    mc = (double*)ctx->h_mix, mi = (uint64_t*)(mc + n_random);
    GenSlot m = gen_slot(ctx->d_mix, n_random, S.cols, 0);
    TT_CUDA(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
    TT_CUDA(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    if (launch_generate(S, seed_state(mix_seed), 0, n_random, m.soa, n_random, m.id, ctx->side))
      return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
    TT_LAUNCHED(ctx);
    if (launch_draft_cost(S, D, m.soa, n_random, 0, 0, false, n_random, toggles, m.cost, nullptr, ctx->sel.invalid,
                          ctx->side))
      return fail(ctx, TT_E_VALIDATE, "unsupported op shape");
    TT_LAUNCHED(ctx);
    TT_CUDA(ctx, cudaMemcpyAsync(mc, m.cost, sizeof(double) * n_random, cudaMemcpyDeviceToHost, ctx->side));
    TT_CUDA(ctx, cudaMemcpyAsync(mi, m.id, sizeof(uint64_t) * n_random, cudaMemcpyDeviceToHost, ctx->side));
  }
  rc = tt_explore(ctx, sk, dev, n_steps, n_spec, pop_size, explore_seed, toggles, nullptr, cost_host, id_host, &cnt,
                  evaluations);
  if (n_random > 0) {
    const cudaError_t e = cudaStreamSynchronize(ctx->side);
    if (rc) return rc;
    if (e != cudaSuccess) return fail(ctx, TT_E_CUDA, cudaGetErrorString(e));
    // membership: open addressing over the identities (insertion order kept)
    int hb = 4;
    while (((int64_t)1 << hb) < 2 * (cnt + n_random)) ++hb;
    const uint64_t hm = ((uint64_t)1 << hb) - 1;
    std::vector<uint64_t> key((size_t)hm + 1);
    std::vector<uint8_t> used((size_t)hm + 1, 0);
    auto insert = [&](uint64_t id) {
      for (uint64_t q = scramble64(id) & hm;; q = (q + 1) & hm) {
        if (!used[q]) return used[q] = 1, key[q] = id, true;
        if (key[q] == id) return false;
      }
    };
    for (int64_t i = 0; i < cnt; ++i) insert(id_host[i]);
    for (int64_t i = 0; i < n_random; ++i)
      if (insert(mi[i])) id_host[cnt] = mi[i], cost_host[cnt++] = mc[i];
  }
  if (rc) return rc;
  *count_host = cnt;
  return TT_OK;
}

int tt_tuner_round(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t draft_size,
                   int64_t pop_size, double random_mix, uint64_t explore_seed, uint64_t mix_seed, int64_t b,
                   int precision, int64_t* sel_idx, double* sel_scores, uint64_t* sel_identity,
                   int64_t* n_candidates) {
  if (!ctx) return TT_E_STATE;
  if (!sel_idx || !n_candidates) return fail(ctx, TT_E_STATE, "tuner_round: null output");
  if (b < 1) return fail(ctx, TT_E_STATE, "select_top: b must be >= 1");
  if (draft_size < 1) return fail(ctx, TT_E_CONFIG, "draft_size must be >= 1");
  if (!ctx->d_params) return fail(ctx, TT_E_STATE, "score: tt_pacm_load first");
  int rc = TT_OK;
  if (draft_size > ctx->tr_cap) {
    cudaFree(ctx->d_tr), cudaFreeHost(ctx->h_tr);
    ctx->d_tr = ctx->h_tr = nullptr, ctx->tr_cap = 0;
    TT_CUDA(ctx, cudaMalloc(&ctx->d_tr, (size_t)draft_size * 24));
    TT_CUDA(ctx, cudaHostAlloc(&ctx->h_tr, (size_t)draft_size * 32 + 64, cudaHostAllocDefault));
    ctx->tr_cap = draft_size;
  }
  if ((rc = ensure_b(ctx, b))) return rc;
  uint64_t* d_id = (uint64_t*)ctx->d_tr;
  double* d_cost = (double*)(d_id + draft_size);
  double* d_score = d_cost + draft_size;
  uint64_t* h_id = (uint64_t*)ctx->h_tr;
  double* h_cost = (double*)(h_id + draft_size);
  double* h_score = h_cost + draft_size;  // the whole set's scores (sel_scores is gathered from it)
  int64_t* h_pos = (int64_t*)(h_score + draft_size);
  int* h_status = (int*)(h_pos + b);
  int64_t cnt = 0;
  if ((rc = tt_draft_set(ctx, sk, dev, n_steps, draft_size, pop_size, random_mix, explore_seed, mix_seed,
                         TT_TOGGLES_ALL, h_id, h_cost, &cnt, nullptr)))
    return rc;
  cudaStream_t st = ctx->stream;
  TT_CUDA(ctx, cudaMemcpyAsync(d_id, h_id, sizeof(uint64_t) * cnt, cudaMemcpyHostToDevice, st));
  TT_CUDA(ctx, cudaMemcpyAsync(d_cost, h_cost, sizeof(double) * cnt, cudaMemcpyHostToDevice, st));
  if ((rc = tt_pacm_score(ctx, sk, dev, d_id, cnt, precision, d_score))) return rc;
  if (launch_select_top(d_score, d_cost, nullptr, cnt, nullptr, b, ctx->d_pos, ctx->d_pos_count, ctx->d_status, st))
    return fail(ctx, TT_E_STATE, "select_top: n too large for b (tiles * b must be <= 4096)");
  TT_LAUNCHED(ctx);
  TT_CUDA(ctx, cudaMemcpyAsync(h_status, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, st));
  TT_CUDA(ctx, cudaMemcpyAsync(h_pos, ctx->d_pos, sizeof(int64_t) * b, cudaMemcpyDeviceToHost, st));
  if (sel_scores) TT_CUDA(ctx, cudaMemcpyAsync(h_score, d_score, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
  if ((rc = sync_check(ctx))) return rc;
  *n_candidates = cnt;
  if (*h_status)
    return fail(ctx, TT_E_STATE, "select_top: requested " + std::to_string(b) + " but only " + std::to_string(cnt) +
                                     " candidates in the draft set");
  for (int64_t i = 0; i < b; ++i) {
    sel_idx[i] = h_pos[i];
    if (sel_scores) sel_scores[i] = h_score[h_pos[i]];
    if (sel_identity) sel_identity[i] = h_id[h_pos[i]];
  }
  return TT_OK;
}

// ------------------------------------------------------------------------
// NCCL: the sharded round inside the C ABI. libnccl is loaded
// at run time (dlopen), so the library has no link-time NCCL dependency;
// in a process that already loaded NCCL (e.g. torch), the same library is used.
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
    a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
    a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_gather && a.comm_destroy && a.error_string;
    if (!a.ok) a.why = "libnccl lacks a required symbol";
    return a;
  }();
  return api;
}
int nccl_fail(tt_ctx* ctx, ncclResult_t r, const char* what) {
  return fail(ctx, TT_E_NCCL, std::string(what) + ": " + nccl().error_string(r));
}
}  // namespace

extern "C" {

int tt_comm_unique_id(uint8_t* id_out) {
  NcclApi& a = nccl();
  if (!a.ok) return TT_E_NCCL;
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) return TT_E_NCCL;
  std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return TT_OK;
}

int tt_comm_init(tt_ctx* ctx, int nranks, int rank, const uint8_t* id) {
  if (!ctx) return TT_E_STATE;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, TT_E_CONFIG, "comm: rank outside [0, nranks)");
  if (ctx->comm) return fail(ctx, TT_E_STATE, "comm: already initialised on this context");
  NcclApi& a = nccl();
  if (!a.ok) return fail(ctx, TT_E_NCCL, "comm: " + a.why);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  cudaSetDevice(ctx->device);
  const ncclResult_t r = a.comm_init_rank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclCommInitRank");
  ctx->comm = c, ctx->nranks = nranks, ctx->rank = rank;
  return TT_OK;
}

int tt_comm_destroy(tt_ctx* ctx) {
  if (!ctx) return TT_E_STATE;
  if (!ctx->comm) return TT_OK;
  cudaStreamSynchronize(ctx->stream);
  const ncclResult_t r = nccl().comm_destroy((ncclComm_t)ctx->comm);
  ctx->comm = nullptr, ctx->nranks = 1, ctx->rank = 0;
  return r == ncclSuccess ? TT_OK : nccl_fail(ctx, r, "ncclCommDestroy");
}

int tt_round_sharded(tt_ctx* ctx, const tt_sketch* sk, const tt_device_spec* dev, const tt_round_config* cfg,
                     const int32_t* soa_shard, int64_t ld, uint64_t seed, int64_t* sel_index, double* sel_score,
                     double* sel_cost, uint64_t* sel_id, tt_round_result* res) {
  if (!ctx) return TT_E_STATE;
  if (!cfg) return fail(ctx, TT_E_STATE, "null round config");
  if (!ctx->comm) return fail(ctx, TT_E_STATE, "round_sharded: tt_comm_init first");
  if (!ctx->pend.empty())
    return fail(ctx, TT_E_STATE, "round_sharded: rounds still in flight (tt_round_collect them first)");
  const int R = ctx->nranks, r = ctx->rank;
  const int64_t k = cfg->k, n = cfg->n;
  if (n < R) return fail(ctx, TT_E_CONFIG, "round_sharded: fewer candidates than ranks");
  if ((int64_t)R * k > kMergeMax) return fail(ctx, TT_E_CONFIG, "round_sharded: ranks * draft_size > 65536");
  // shard_range (sharded.py): the first n % R ranks take one extra candidate
  const int64_t base = n / R, extra = n % R;
  tt_round_config local = *cfg;
  local.first = cfg->first + r * base + std::min<int64_t>(r, extra);
  local.n = base + (r < extra ? 1 : 0);
  int rc;
  if ((rc = tgrow(ctx, ctx->d_gather, ctx->gather_cap, 3 * k * (int64_t)(2 * R + 1)))) return rc;
  int64_t* payload = ctx->d_gather;             // [3][k]: cost bits, global index, identity
  int64_t* gathered = payload + 3 * k;          // [R][3][k]
  int64_t* merged = gathered + 3 * k * R;       // [3][R k]
  auto draft = [&](bool sync) {
    return (sync ? tt_round_local : tt_round_local_async)(ctx, sk, dev, &local, soa_shard, ld, seed, (double*)payload,
                                                          payload + k, (uint64_t*)(payload + 2 * k));
  };
  for (int attempt = 0; attempt < 2; ++attempt) {
    if ((rc = draft(attempt > 0))) return rc;
    const ncclResult_t nr = nccl().all_gather(payload, gathered, (size_t)(3 * k), ncclInt64, (ncclComm_t)ctx->comm,
                                              ctx->stream);
    if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclAllGather");
    for (int row = 0; row < 3; ++row)  // R consecutive [3][k] payloads -> one [3][R k] table
      TT_CUDA(ctx, cudaMemcpy2DAsync(merged + row * R * k, k * 8, gathered + row * k, 3 * k * 8, k * 8, R,
                                     cudaMemcpyDeviceToDevice, ctx->stream));
    tt_round_config m = *cfg;
    m.first = 0;
    rc = tt_round_finish_merged(ctx, sk, dev, &m, (const double*)merged, merged + R * k,
                                (const uint64_t*)(merged + 2 * R * k), R * k, sel_index, sel_score, sel_cost, sel_id,
                                res);
    // a rank's selector overflow is seen by every rank in the merged status:
    // all re-run the draft half synchronously (host-driven retries, hash path)
    if (rc == TT_E_STATE && attempt == 0 && ctx->err.find("tt_round_local") != std::string::npos) continue;
    return rc;
  }
  return rc;
}

}  // extern "C"
