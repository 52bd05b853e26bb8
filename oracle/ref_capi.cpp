// ref_capi.cpp — extern "C" adapter over the unmodified reference tiletune
// core. TEST INFRASTRUCTURE ONLY (see ref_capi.h). Every call goes through
// the reference's own public headers (proj/core/include/tiletune/*.hpp).
#include "ref_capi.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "tiletune/common.hpp"
#include "tiletune/device.hpp"
#include "tiletune/draft.hpp"
#include "tiletune/features.hpp"
#include "tiletune/momentum.hpp"
#include "tiletune/oracle.hpp"
#include "tiletune/ranker.hpp"
#include "tiletune/schedule.hpp"
#include "tiletune/tuner.hpp"
#include "tiletune/workload.hpp"

using namespace tiletune;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

std::string axis_name(const tt_op_spec& op, int a) {
  return a < op.n_spatial ? "s" + std::to_string(a) : "r" + std::to_string(a - op.n_spatial);
}

TensorOpSpec to_op(const tt_op_spec& o) {
  TensorOpSpec op;
  op.name = "op";
  for (int a = 0; a < o.n_spatial; ++a) op.spatial_axes.push_back({axis_name(o, a), o.extent[a]});
  for (int r = 0; r < o.n_reduction; ++r)
    op.reduction_axes.push_back({axis_name(o, o.n_spatial + r), o.extent[o.n_spatial + r]});
  for (int b = 0; b < o.n_buffers; ++b) {
    BufferSpec bs;
    bs.name = "b" + std::to_string(b);
    for (int q = 0; q < o.buffers[b].n_axes; ++q) bs.axes.push_back(axis_name(o, o.buffers[b].axes[q]));
    bs.io = o.buffers[b].io == TT_IO_OUTPUT ? BufferIo::kOutput : BufferIo::kInput;
    op.buffers.push_back(bs);
  }
  op.fused_elementwise = o.fused_elementwise;
  op.kind = o.kind == TT_OP_ELEMENTWISE ? OpKind::kElementwise : OpKind::kTiled;
  return op;
}

Sketch to_sketch(const tt_sketch& s) {
  Sketch sk = generate_sketch(to_op(s.op), true);
  sk.unroll_choices.assign(s.unroll, s.unroll + s.n_unroll);
  return sk;
}

DeviceSpec to_dev(const tt_device_spec& d) {
  DeviceSpec dev;
  dev.m_l0 = d.m_l0, dev.m_l1 = d.m_l1, dev.pu_l1 = d.pu_l1, dev.n_l1 = d.n_l1;
  dev.pu_l2 = d.pu_l2, dev.n_l2 = d.n_l2, dev.t_p = d.t_p, dev.t_m = d.t_m;
  dev.element_bytes = d.element_bytes;
  return dev;
}

Schedule get_sched(const tt_sketch& s, const int32_t* soa, int64_t ld, int64_t i) {
  Schedule sc;
  for (int a = 0; a < s.op.n_spatial; ++a) {
    std::vector<int64_t> f(4);
    for (int q = 0; q < 4; ++q) f[q] = soa[(int64_t)(4 * a + q) * ld + i];
    sc.spatial_factors.push_back(f);
  }
  for (int r = 0; r < s.op.n_reduction; ++r) {
    std::vector<int64_t> f(3);
    for (int q = 0; q < 3; ++q) f[q] = soa[(int64_t)(4 * s.op.n_spatial + 3 * r + q) * ld + i];
    sc.reduction_factors.push_back(f);
  }
  sc.unroll = soa[(int64_t)(tt_schedule_cols(&s) - 1) * ld + i];
  return sc;
}

void put_sched(const tt_sketch& s, const Schedule& sc, int32_t* soa, int64_t ld, int64_t i) {
  for (int a = 0; a < s.op.n_spatial; ++a)
    for (int q = 0; q < 4; ++q) soa[(int64_t)(4 * a + q) * ld + i] = (int32_t)sc.spatial_factors[a][q];
  for (int r = 0; r < s.op.n_reduction; ++r)
    for (int q = 0; q < 3; ++q)
      soa[(int64_t)(4 * s.op.n_spatial + 3 * r + q) * ld + i] = (int32_t)sc.reduction_factors[r][q];
  soa[(int64_t)(tt_schedule_cols(&s) - 1) * ld + i] = (int32_t)sc.unroll;
}

void flatten(const RankerParams& p, double* out) {
  for_each_tensor(p, [&](const std::string&, const Tensor& t) {
    std::memcpy(out, t.v.data(), t.v.size() * sizeof(double));
    out += t.v.size();
  });
}

RankerParams unflatten(const double* in, int h) {
  RngStream dummy(1);
  RankerParams p = zeros_like(init_params(h, dummy));
  for_each_tensor(p, [&](const std::string&, Tensor& t) {
    std::memcpy(t.v.data(), in, t.v.size() * sizeof(double));
    in += t.v.size();
  });
  return p;
}

HybridFeature make_feat(int S, int B, const double* stmt, const double* block) {
  HybridFeature f;
  f.statements.resize(S);
  f.dataflow.resize(B);
  for (int s = 0; s < S; ++s)
    for (int q = 0; q < kStatementFeatureWidth; ++q) f.statements[s][q] = stmt[s * kStatementFeatureWidth + q];
  for (int b = 0; b < B; ++b)
    for (int q = 0; q < kDataflowFeatureWidth; ++q) f.dataflow[b][q] = block[b * kDataflowFeatureWidth + q];
  return f;
}

double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_random_init(const tt_sketch* sk, uint64_t seed, int64_t n, int32_t* soa, int64_t ld) {
  return guard([&] {
    Sketch s = to_sketch(*sk);
    RngStream rng(seed);
    auto pop = random_init(s, n, rng);
    for (int64_t i = 0; i < n; ++i) put_sched(*sk, pop[i], soa, ld, i);
  });
}

int ref_draft_cost(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa,
                   int64_t ld, int64_t n, int toggles, int threads, double* cost) {
  return guard([&] {
    Sketch s = to_sketch(*sk);
    DeviceSpec d = to_dev(*dev);
    PenaltyToggles tg{(toggles & TT_TOGGLE_COMPUTE) != 0, (toggles & TT_TOGGLE_MEMORY) != 0};
    std::vector<Schedule> pop(n);
    for (int64_t i = 0; i < n; ++i) pop[i] = get_sched(*sk, soa, ld, i);
    parallel_for(n, threads, [&](std::size_t i) { cost[i] = draft_cost(s, pop[i], d, tg).total; });
  });
}

int ref_trace(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
              int64_t i, int64_t* symbols, double* penalties, double* stmt_cost, double* total) {
  return guard([&] {
    Sketch s = to_sketch(*sk);
    DeviceSpec d = to_dev(*dev);
    Schedule sc = get_sched(*sk, soa, ld, i);
    auto syms = extract_symbols(s, sc);
    DraftCost c = draft_cost(s, sc, d);
    for (std::size_t q = 0; q < syms.size(); ++q) {
      const SymbolSet& y = syms[q].symbols;
      int64_t v[8] = {y.s1, y.s2, y.s3, y.s4, y.s5, y.s6, y.s7, y.s8};
      std::memcpy(symbols + 8 * q, v, sizeof(v));
      PenaltySet p = compute_penalties(y, d);
      double pv[7] = {p.p_l0_m, p.p_l0_c, p.p_l1_m, p.p_l1_c, p.alpha_l1, p.p_l2_c, p.p_l2_m};
      std::memcpy(penalties + 7 * q, pv, sizeof(pv));
      const auto& st = c.per_statement[q];
      double cv[4] = {st.l_c, st.l_m, st.u_p, st.u_m};
      std::memcpy(stmt_cost + 4 * q, cv, sizeof(cv));
    }
    *total = c.total;
  });
}

int ref_explore(const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t k,
                int64_t n, uint64_t seed, int threads, int32_t* soa_out, double* cost_out,
                int64_t* count, uint64_t* evaluations) {
  return guard([&] {
    RngStream rng(seed);
    ExploreResult r = explore(to_op(sk->op), to_dev(*dev), n_steps, (int)k, (int)n, rng, {}, threads);
    *count = (int64_t)r.drafted.size();
    *evaluations = r.evaluations;
    for (std::size_t i = 0; i < r.drafted.size(); ++i) {
      put_sched(*sk, r.drafted[i], soa_out, k, (int64_t)i);
      cost_out[i] = r.draft_costs[i];
    }
  });
}

int ref_features(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
                 const int64_t* idx, int64_t k, double* stmt_out, double* block_out) {
  return guard([&] {
    Sketch s = to_sketch(*sk);
    DeviceSpec d = to_dev(*dev);
    int S = tt_n_statements(&sk->op), B = tt_n_blocks(&sk->op);
    for (int64_t q = 0; q < k; ++q) {
      HybridFeature f = extract_features(s, get_sched(*sk, soa, ld, idx[q]), d);
      for (int st = 0; st < S; ++st)
        std::memcpy(stmt_out + (q * S + st) * TT_STMT_WIDTH, f.statements[st].data(), sizeof(double) * TT_STMT_WIDTH);
      for (int b = 0; b < B; ++b)
        std::memcpy(block_out + (q * B + b) * TT_BLOCK_WIDTH, f.dataflow[b].data(), sizeof(double) * TT_BLOCK_WIDTH);
    }
  });
}

int ref_init_params(int h, uint64_t seed, double* params) {
  return guard([&] {
    RngStream rng(seed);
    flatten(init_params(h, rng), params);
  });
}

int ref_score_batch(const double* params, int h, int n_stmt, int n_block, const double* stmt,
                    const double* block, int64_t k, int attention_identity, int threads,
                    double* out, uint64_t* forward_calls_delta) {
  return guard([&] {
    RankerParams p = unflatten(params, h);
    std::vector<HybridFeature> feats(k);
    for (int64_t q = 0; q < k; ++q)
      feats[q] = make_feat(n_stmt, n_block, stmt + q * n_stmt * TT_STMT_WIDTH, block + q * n_block * TT_BLOCK_WIDTH);
    ScoreOptions o;
    o.attention_identity = attention_identity != 0;
    uint64_t before = forward_calls();
    auto s = score_batch(p, feats, o, threads);
    if (forward_calls_delta) *forward_calls_delta = forward_calls() - before;
    std::memcpy(out, s.data(), sizeof(double) * k);
  });
}

int ref_select_top(const double* scores, const double* drafts, const uint8_t* excluded,
                   int64_t n, int64_t b, int64_t* idx_out) {
  return guard([&] {
    std::vector<double> s(scores, scores + n), d(drafts, drafts + n);
    std::vector<char> e(n, 0);
    if (excluded)
      for (int64_t i = 0; i < n; ++i) e[i] = excluded[i] ? 1 : 0;
    auto r = select_top(s, d, e, (std::size_t)b);
    for (int64_t i = 0; i < b; ++i) idx_out[i] = (int64_t)r[i];
  });
}

int ref_momentum_update(double* phi, const double* target, int h, double m) {
  return guard([&] {
    SiameseState st;
    st.params = unflatten(phi, h);
    st.momentum = m;
    SiameseState next = momentum_update(st, unflatten(target, h));
    flatten(next.params, phi);
  });
}

int ref_rank_loss(const double* scores, const double* latencies, int64_t n, double* loss, double* grad) {
  return guard([&] {
    RankLossResult r = lambda_rank_loss(std::vector<double>(scores, scores + n),
                                        std::vector<double>(latencies, latencies + n));
    *loss = r.loss;
    if (grad) std::memcpy(grad, r.grad.data(), sizeof(double) * (size_t)n);
  });
}

int ref_train(double* params, int h, int n_stmt, int n_block, const double* stmt,
              const double* block, const double* latencies, int64_t k, int epochs, double lr,
              int batch, uint64_t seed, double* initial_loss, double* final_loss) {
  return guard([&] {
    RankerParams p = unflatten(params, h);
    TaskSamples ts;
    ts.task = "op";
    for (int64_t q = 0; q < k; ++q) {
      ts.features.push_back(make_feat(n_stmt, n_block, stmt + q * n_stmt * TT_STMT_WIDTH, block + q * n_block * TT_BLOCK_WIDTH));
      ts.latencies.push_back(latencies[q]);
    }
    TrainConfig cfg;
    cfg.epochs = epochs, cfg.lr = lr, cfg.batch = batch, cfg.seed = seed;
    TrainReport r = train(p, {ts}, cfg);
    if (initial_loss) *initial_loss = r.initial_loss;
    if (final_loss) *final_loss = r.final_loss;
    flatten(p, params);
  });
}

int ref_noiseless_latency(const tt_sketch* sk, const tt_device_spec* hidden, double stride_coeff,
                          double occupancy_coeff, double launch_overhead_s, const int32_t* soa,
                          int64_t ld, int64_t n, double* out) {
  return guard([&] {
    Sketch s = to_sketch(*sk);
    OracleDevice o;
    o.hidden = to_dev(*hidden);
    o.stride_coeff = stride_coeff;
    o.occupancy_coeff = occupancy_coeff;
    o.launch_overhead_s = launch_overhead_s;
    for (int64_t i = 0; i < n; ++i) out[i] = noiseless_latency(s, get_sched(*sk, soa, ld, i), o);
  });
}

static OracleDevice to_oracle(const tt_oracle_spec& o) {
  OracleDevice r;
  r.hidden = to_dev(o.hidden);
  r.stride_coeff = o.stride_coeff;
  r.occupancy_coeff = o.occupancy_coeff;
  r.launch_overhead_s = o.launch_overhead_s;
  r.noise_sigma = o.noise_sigma;
  r.seed = o.seed;
  return r;
}

int ref_measure(const tt_sketch* sk, const tt_oracle_spec* o, const int32_t* soa, int64_t ld, int64_t n,
                uint64_t task_hash, uint64_t trial0, double* latency, double* noiseless) {
  return guard([&] {
    Sketch s = to_sketch(*sk);
    OracleDevice od = to_oracle(*o);
    for (int64_t i = 0; i < n; ++i) {
      RngStream mrng(derive_seed(od.seed, 0x6d656173ULL, task_hash, trial0 + (uint64_t)i));  // tuner.cpp:202
      Measurement m = measure(s, get_sched(*sk, soa, ld, i), od, mrng);
      latency[i] = m.latency_s;
      noiseless[i] = m.noiseless_latency_s;
    }
  });
}

int ref_oracle_best(const tt_sketch* sk, const tt_oracle_spec* o, uint64_t cap, int32_t* argmin_soa,
                    double* latency) {
  return guard([&] {
    OracleBest b = oracle_best(to_sketch(*sk), to_oracle(*o), cap);
    put_sched(*sk, b.argmin, argmin_soa, 1, 0);
    *latency = b.latency_s;
  });
}

// serialize_params / parse_params (ranker.cpp:534-548) and the Siamese
// checkpoint (momentum.cpp:58-86): text via a caller buffer
int ref_serialize_params(const double* params, int h, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    std::string t = serialize_params(unflatten(params, h));
    *len = (int64_t)t.size();
    if ((int64_t)t.size() < cap) std::memcpy(buf, t.c_str(), t.size() + 1);
  });
}

int ref_parse_params(const char* text, double* params, int* h) {
  return guard([&] {
    RankerParams p = parse_params(text);
    *h = p.hidden;
    if (params) flatten(p, params);
  });
}

int ref_serialize_siamese(const double* params, int h, double m, int evolved, char* buf, int64_t cap,
                          int64_t* len) {
  return guard([&] {
    SiameseState s;
    s.params = unflatten(params, h);
    s.momentum = m;
    s.provenance = evolved ? SiameseState::Provenance::kEvolved : SiameseState::Provenance::kPretrained;
    std::string t = serialize_siamese(s);
    *len = (int64_t)t.size();
    if ((int64_t)t.size() < cap) std::memcpy(buf, t.c_str(), t.size() + 1);
  });
}

int ref_parse_siamese(const char* text, double* params, int* h, double* m, int* evolved) {
  return guard([&] {
    SiameseState s = parse_siamese(text);
    *h = s.params.hidden;
    if (params) flatten(s.params, params);
    *m = s.momentum;
    *evolved = s.provenance == SiameseState::Provenance::kEvolved;
  });
}

int ref_round(const tt_sketch* sk, const tt_device_spec* dev, int64_t n, int64_t k, int64_t b,
              uint64_t seed, const double* params, int h, int threads, int64_t* sel_idx,
              double* sel_scores, int32_t* drafted_soa, double* drafted_cost,
              int64_t* drafted_count, double* seconds) {
  return guard([&] {
    TensorOpSpec op = to_op(sk->op);
    DeviceSpec d = to_dev(*dev);
    RankerParams p = unflatten(params, h);
    auto t0 = std::chrono::steady_clock::now();
    RngStream rng(seed);
    ExploreResult ex = explore(op, d, 1, (int)k, (int)n, rng, {}, threads);  // draft.cpp:156-221
    seconds[0] = secs_since(t0);
    auto t1 = std::chrono::steady_clock::now();
    std::vector<HybridFeature> feats(ex.drafted.size());
    parallel_for(feats.size(), threads, [&](std::size_t i) {  // tuner.cpp:366-369
      feats[i] = extract_features(ex.sketch, ex.drafted[i], d);
    });
    seconds[1] = secs_since(t1);
    auto t2 = std::chrono::steady_clock::now();
    std::vector<double> scores = score_batch(p, feats, {}, threads);  // ranker.cpp:375-381
    seconds[2] = secs_since(t2);
    auto t3 = std::chrono::steady_clock::now();
    std::vector<char> excluded(scores.size(), 0);
    auto sel = select_top(scores, ex.draft_costs, excluded, (std::size_t)b);  // ranker.cpp:514-532
    seconds[3] = secs_since(t3);
    for (int64_t i = 0; i < b; ++i) {
      sel_idx[i] = (int64_t)sel[i];
      if (sel_scores) sel_scores[i] = scores[sel[i]];
    }
    *drafted_count = (int64_t)ex.drafted.size();
    if (drafted_soa)
      for (std::size_t i = 0; i < ex.drafted.size(); ++i) put_sched(*sk, ex.drafted[i], drafted_soa, k, (int64_t)i);
    if (drafted_cost)
      for (std::size_t i = 0; i < ex.drafted.size(); ++i) drafted_cost[i] = ex.draft_costs[i];
  });
}

/* A strict CPU bound for the round: the reference's own
 * per-schedule functions composed by hand, without explore()'s serial
 * string-key bookkeeping. The population is given (resident, like the
 * device's `value`); draft_cost over it in parallel_for; the k lowest unique
 * by (cost, index) via nth_element + sort + exact factor comparison among
 * equal costs (equal schedules have equal costs; the lowest index is the
 * first discovery, as in explore); extract_features in parallel;
 * score_batch; select_top. Same drafted set and selection as ref_round on
 * the same population. seconds: [0] draft + top-k, [1] features, [2] scores,
 * [3] select. sel_pop_idx: population indices of the b selections. */
int ref_round_strict(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld, int64_t n,
                     int64_t k, int64_t b, const double* params, int h, int threads, int64_t* sel_pop_idx,
                     double* seconds) {
  return guard([&] {
    Sketch s = to_sketch(*sk);
    DeviceSpec d = to_dev(*dev);
    RankerParams p = unflatten(params, h);
    std::vector<Schedule> pop((size_t)n);
    parallel_for((size_t)n, threads, [&](std::size_t i) { pop[i] = get_sched(*sk, soa, ld, (int64_t)i); });
    auto t0 = std::chrono::steady_clock::now();
    std::vector<double> cost((size_t)n);
    parallel_for((size_t)n, threads, [&](std::size_t i) { cost[i] = draft_cost(s, pop[i], d).total; });
    auto before = [&](int64_t a, int64_t c) { return cost[a] != cost[c] ? cost[a] < cost[c] : a < c; };
    auto same = [&](const Schedule& x, const Schedule& y) {
      return x.unroll == y.unroll && x.spatial_factors == y.spatial_factors &&
             x.reduction_factors == y.reduction_factors;
    };
    std::vector<int64_t> ord((size_t)n), kept;
    int64_t want = std::min<int64_t>(n, 2 * k + 64);
    for (;;) {
      for (int64_t i = 0; i < n; ++i) ord[i] = i;
      std::nth_element(ord.begin(), ord.begin() + (want - 1), ord.end(), before);
      std::sort(ord.begin(), ord.begin() + want, before);
      kept.clear();
      for (int64_t q = 0; q < want && (int64_t)kept.size() < k; ++q) {
        const int64_t i = ord[q];
        bool dup = false;
        for (auto it = kept.rbegin(); it != kept.rend() && cost[*it] == cost[i]; ++it)
          if (same(pop[*it], pop[i])) {
            dup = true;
            break;
          }
        if (!dup) kept.push_back(i);
      }
      if ((int64_t)kept.size() >= k || want == n) break;
      want = std::min<int64_t>(n, 2 * want);
    }
    seconds[0] = secs_since(t0);
    auto t1 = std::chrono::steady_clock::now();
    std::vector<HybridFeature> feats(kept.size());
    parallel_for(feats.size(), threads, [&](std::size_t i) { feats[i] = extract_features(s, pop[kept[i]], d); });
    seconds[1] = secs_since(t1);
    auto t2 = std::chrono::steady_clock::now();
    std::vector<double> scores = score_batch(p, feats, {}, threads);
    seconds[2] = secs_since(t2);
    auto t3 = std::chrono::steady_clock::now();
    std::vector<double> dcost(kept.size());
    for (std::size_t i = 0; i < kept.size(); ++i) dcost[i] = cost[kept[i]];
    std::vector<char> excluded(scores.size(), 0);
    auto sel = select_top(scores, dcost, excluded, (std::size_t)b);
    seconds[3] = secs_since(t3);
    for (int64_t i = 0; i < b; ++i) sel_pop_idx[i] = kept[sel[i]];
  });
}

/* The tuner's real round (build_draft_set tuner.cpp:294-323 restated over the
 * reference's own functions, then tuner.cpp:366-384): GA explore + random
 * mix -> features -> score_batch -> select_top. seconds[0] draft set,
 * [1] features + scores + select. */
int ref_tuner_round(const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t draft_size,
                    int64_t pop_size, double random_mix, uint64_t explore_seed, uint64_t mix_seed, int64_t b,
                    const double* params, int h, int threads, int64_t* sel_idx, double* sel_scores,
                    int64_t* n_candidates, double* seconds) {
  return guard([&] {
    TensorOpSpec op = to_op(sk->op);
    DeviceSpec d = to_dev(*dev);
    RankerParams p = unflatten(params, h);
    auto t0 = std::chrono::steady_clock::now();
    int64_t n_spec = std::llround((1.0 - random_mix) * (double)draft_size);
    if (n_spec < 1) n_spec = 1;
    const int64_t n_random = draft_size - n_spec;
    RngStream erng(explore_seed);
    ExploreResult ex = explore(op, d, n_steps, (int)n_spec, (int)pop_size, erng, {}, threads);
    std::vector<Schedule> cands;
    std::vector<double> drafts;
    std::set<std::string> seen;
    for (std::size_t i = 0; i < ex.drafted.size(); ++i)
      if (seen.insert(schedule_key(ex.sketch, ex.drafted[i])).second)
        cands.push_back(ex.drafted[i]), drafts.push_back(ex.draft_costs[i]);
    if (n_random > 0) {
      RngStream mrng(mix_seed);
      for (auto& s : random_init(ex.sketch, n_random, mrng))
        if (seen.insert(schedule_key(ex.sketch, s)).second)
          cands.push_back(s), drafts.push_back(draft_cost(ex.sketch, s, d).total);
    }
    seconds[0] = secs_since(t0);
    auto t1 = std::chrono::steady_clock::now();
    std::vector<HybridFeature> feats(cands.size());
    parallel_for(feats.size(), threads, [&](std::size_t i) { feats[i] = extract_features(ex.sketch, cands[i], d); });
    std::vector<double> scores = score_batch(p, feats, {}, threads);
    std::vector<char> excluded(scores.size(), 0);
    auto sel = select_top(scores, drafts, excluded, (std::size_t)b);
    seconds[1] = secs_since(t1);
    for (int64_t i = 0; i < b && i < (int64_t)sel.size(); ++i) {
      sel_idx[i] = (int64_t)sel[i];
      if (sel_scores) sel_scores[i] = scores[sel[i]];
    }
    *n_candidates = (int64_t)cands.size();
  });
}

}  // extern "C"

/* ---- measurement records JSONL (tuner.cpp:577-645), one task named `task` ---- */
int ref_records_to_jsonl(const tt_sketch* sk, const char* task, const int32_t* soa, int64_t ld, int64_t n,
                         const int32_t* rounds, const double* lat, const double* draft, const double* score,
                         char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    std::map<std::string, Sketch> sketches{{task, to_sketch(*sk)}};
    std::vector<TuningRecord> recs;
    for (int64_t i = 0; i < n; ++i) {
      TuningRecord r;
      r.task = task, r.round = rounds[i], r.schedule = get_sched(*sk, soa, ld, i);
      r.latency_s = lat[i], r.draft_cost = draft[i], r.model_score = score[i];
      recs.push_back(std::move(r));
    }
    std::string t = records_to_jsonl(recs, sketches);
    *len = (int64_t)t.size();
    if ((int64_t)t.size() < cap) std::memcpy(buf, t.c_str(), t.size() + 1);
  });
}

int ref_records_from_jsonl(const tt_sketch* sk, const char* task, const char* text, int32_t* soa, int64_t ld,
                           int32_t* rounds, double* lat, double* draft, double* score, int64_t cap, int64_t* n) {
  return guard([&] {
    std::map<std::string, Sketch> sketches{{task, to_sketch(*sk)}};
    std::vector<TuningRecord> recs = records_from_jsonl(text, sketches);
    *n = (int64_t)recs.size();
    for (int64_t i = 0; i < (int64_t)recs.size() && i < cap; ++i) {
      put_sched(*sk, recs[i].schedule, soa, ld, i);
      rounds[i] = recs[i].round, lat[i] = recs[i].latency_s, draft[i] = recs[i].draft_cost;
      score[i] = recs[i].model_score;
    }
  });
}
