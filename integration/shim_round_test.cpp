// shim_round_test.cpp — one reference-API round through the shim against the
// reference's own composition of the same round (tuner.cpp:302-305,366-384:
// explore(n_steps = 1) -> extract_features -> score_batch -> select_top), on
// the same op / device / seed / parameters; then one train() through the
// shim against the reference's train(). Exit 0 iff the selected schedules
// are identical and the trained parameters agree within 1e-11 relative.
#include <cmath>
#include <cstdio>
#include <set>
#include <string>

#include "b200_shim.hpp"
#include "tiletune/common.hpp"
#include "tiletune/draft.hpp"
#include "tiletune/features.hpp"
#include "tiletune/schedule.hpp"

using namespace tiletune;

static TensorOpSpec conv(int64_t f, int64_t y, int64_t x, int64_t c, int64_t r) {  // test_helpers.hpp:89-101
  TensorOpSpec op;
  op.name = "conv";
  op.spatial_axes = {{"f", f}, {"y", y}, {"x", x}};
  op.reduction_axes = {{"c", c}, {"r", r}};
  op.buffers = {{"I", {"c", "y", "x"}, BufferIo::kInput},
                {"W", {"f", "c", "r"}, BufferIo::kInput},
                {"O", {"f", "y", "x"}, BufferIo::kOutput}};
  return op;
}

static bool same(const Schedule& a, const Schedule& b) {
  return a.unroll == b.unroll && a.spatial_factors == b.spatial_factors && a.reduction_factors == b.reduction_factors;
}

int main() {
  DeviceSpec dev;  // test_helpers.hpp reference_device()
  dev.m_l0 = 256, dev.m_l1 = 4096, dev.pu_l1 = 4, dev.n_l1 = 32, dev.pu_l2 = 8, dev.n_l2 = 32;
  dev.t_p = 1.0e12, dev.t_m = 1.0e11, dev.element_bytes = 4;
  const TensorOpSpec op = conv(64, 56, 56, 64, 9);
  const int N = 65536, K = 512, b = 10;
  const uint64_t seed = 1234;
  RngStream prng(77);
  RankerParams target = init_params(64, prng);
  int fails = 0;

  // ---- the reference's round
  RngStream rng(seed);
  ExploreResult ex = explore(op, dev, 1, K, N, rng, {}, 8);
  std::vector<HybridFeature> feats;
  for (const auto& s : ex.drafted) feats.push_back(extract_features(ex.sketch, s, dev));
  std::vector<double> scores = score_batch(target, feats, {}, 8);
  std::vector<char> excluded(scores.size(), 0);
  auto sel = select_top(scores, ex.draft_costs, excluded, b);

  // ---- the same round through the shim (B200)
  b200::B200Round round(0);
  std::vector<double> sc;
  std::vector<int64_t> idx = round.run(op, dev, target, N, K, b, seed, &sc);
  RngStream rng2(seed);
  std::vector<Schedule> pop = random_init(ex.sketch, N, rng2);  // index i of the device population
  if (idx.size() != sel.size()) ++fails;
  for (std::size_t e = 0; e < idx.size() && e < sel.size(); ++e) {
    const bool ok = same(pop[idx[e]], ex.drafted[sel[e]]) && std::fabs(sc[e] - scores[sel[e]]) <= 1e-12;
    std::printf("selection %zu: population %lld score %.17g | reference %.17g %s\n", e, (long long)idx[e], sc[e],
                scores[sel[e]], ok ? "ok" : "MISMATCH");
    fails += !ok;
  }

  // ---- the tuner's real round (GA draft set, tuner.cpp:294-323) through the
  // shim vs the reference's own functions composed the same way
  {
    const int steps = 32, dsize = 512, pop = 512, bb = 10;
    const double mix = 0.2;
    const uint64_t es = 2000, ms = 2001;
    int64_t n_spec = std::llround((1.0 - mix) * (double)dsize);
    if (n_spec < 1) n_spec = 1;
    RngStream erng(es);
    ExploreResult gx = explore(op, dev, steps, (int)n_spec, pop, erng, {}, 8);
    std::vector<Schedule> cands;
    std::vector<double> drafts;
    std::set<std::string> seen;
    for (std::size_t i = 0; i < gx.drafted.size(); ++i)
      if (seen.insert(schedule_key(gx.sketch, gx.drafted[i])).second)
        cands.push_back(gx.drafted[i]), drafts.push_back(gx.draft_costs[i]);
    RngStream mrng(ms);
    for (auto& s : random_init(gx.sketch, dsize - n_spec, mrng))
      if (seen.insert(schedule_key(gx.sketch, s)).second)
        cands.push_back(s), drafts.push_back(draft_cost(gx.sketch, s, dev).total);
    std::vector<HybridFeature> gf;
    for (const auto& s : cands) gf.push_back(extract_features(gx.sketch, s, dev));
    std::vector<double> gs = score_batch(target, gf, {}, 8);
    std::vector<char> gexcl(gs.size(), 0);
    auto gsel = select_top(gs, drafts, gexcl, bb);
    std::vector<double> tsc;
    int64_t tcnt = 0;
    std::vector<int64_t> tsel = round.tuner_round(op, dev, target, steps, dsize, pop, mix, es, ms, bb, &tsc, nullptr,
                                                  &tcnt);
    bool ok = tcnt == (int64_t)cands.size() && tsel.size() == gsel.size();
    for (std::size_t e = 0; ok && e < tsel.size(); ++e)
      ok = tsel[e] == (int64_t)gsel[e] && std::fabs(tsc[e] - gs[gsel[e]]) <= 1e-12 * std::fabs(gs[gsel[e]]) + 1e-300;
    std::printf("tuner round: %lld candidates (reference %zu), picks %s\n", (long long)tcnt, cands.size(),
                ok ? "identical" : "MISMATCH");
    fails += !ok;
  }

  // ---- train() through the shim vs the reference's train() on the drafted set
  std::vector<double> lat(ex.drafted.size()), st, bl;
  for (std::size_t i = 0; i < ex.drafted.size(); ++i) {
    lat[i] = 1e-4 * (1.0 + ex.draft_costs[i] * 1e3 + 0.1 * std::sin((double)i));
    for (const auto& row : feats[i].statements) st.insert(st.end(), row.begin(), row.end());
    for (const auto& row : feats[i].dataflow) bl.insert(bl.end(), row.begin(), row.end());
  }
  TrainConfig cfg;
  cfg.epochs = 3, cfg.batch = 128, cfg.seed = 5;
  RankerParams mine = target, theirs = target;
  auto [l0, l1] = round.train(mine, st, bl, (int)feats[0].statements.size(), (int)feats[0].dataflow.size(), lat, cfg);
  TaskSamples ts;
  ts.task = op.name, ts.features = feats, ts.latencies = lat;
  TrainReport rep = train(theirs, {ts}, cfg);
  const auto pm = b200::flatten(mine), pt = b200::flatten(theirs);
  double dmax = 0.0, pmax = 0.0;
  for (std::size_t i = 0; i < pm.size(); ++i) dmax = std::fmax(dmax, std::fabs(pm[i] - pt[i])), pmax = std::fmax(pmax, std::fabs(pt[i]));
  const bool tok = dmax <= 1e-11 * pmax && std::fabs(l1 - rep.final_loss) <= 1e-11 * std::fabs(rep.final_loss);
  std::printf("train: loss %.17g -> %.17g | reference %.17g -> %.17g | max |dp| / max |p| = %.3g %s\n", l0, l1,
              rep.initial_loss, rep.final_loss, pmax > 0 ? dmax / pmax : 0.0, tok ? "ok" : "MISMATCH");
  fails += !tok;
  std::printf("%s\n", fails ? "FAILED" : "PASSED");
  return fails ? 1 : 0;
}
